export AB_BRIEF=1 AB_REPS=3
timeout 900 python tools/ab_batch.py 4096 "CQP_BATCH_LEGACY=1" "" | grep -E "^==|compute_ms|vs first"
timeout 900 python tools/ab_batch.py 300 "CQP_BATCH_LEGACY=1" "" | grep -E "^==|compute_ms|vs first"
AB_NU=10 timeout 900 python tools/ab_batch.py 700 "CQP_BATCH_LEGACY=1" "" | grep -E "^==|compute_ms|vs first"
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_mpc_server.py -x -q 2>&1 | tail -3
