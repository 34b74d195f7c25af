export AB_BRIEF=1 AB_REPS=1 AB_NU=10
echo "### nu=10 B=200 full solve"
timeout 900 python tools/ab_batch.py 200 "CQP_BATCH_LEGACY=1" "" "CQP_BATCH_FORCE_CFG=3" "CQP_BATCH_FORCE_CFG=7" "CQP_BATCH_FORCE_CFG=4" | grep -E "^==|compute_ms|vs first"
