export CQP_B200_LIB=$PWD/build/trace/libcqp_b200.so
python - <<'PY'
import sys, ctypes as C, numpy as np
sys.path.insert(0, '.')
from paper_2311_18056_b200 import problems, solver as S, _lib
wl = problems.config1(seed=0); base = wl.base_problem()
gpu = S.Solver(base.H, base.g, base.G, base.c, base.d); gpu.set_mpc_template(wl.tmpl, wl.limits)
q = wl.problem_at(wl.x0(1.0)); gpu.update_vectors(q.g, q.c, q.d); gpu.cold_start(); gpu.solve()
gpu.mpc_server_start(1)
x = np.ascontiguousarray(wl.x0(1.0)); u0 = np.zeros(wl.sys.nu)
A, B = wl.sys.A, wl.sys.B
# find mailbox: not exposed; read stamps through a debug hook: the stamps live in the host-mapped mailbox -> expose via ctypes on the handle? use cqp_mpc_server_last_timing only
for t in range(200):
    gpu.mpc_step_x0_fast(x, 1, u0); x = np.ascontiguousarray(A @ x + B @ u0)
print("timing", gpu.mpc_server_last_timing())
lib = _lib.load()
buf = (C.c_ulonglong * 8)()
lib.cqp_debug_server_stamps.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong)]
lib.cqp_debug_server_stamps(gpu._h, buf)
print("stamps ns: pushed, g complete, bias, iterations, results, sysfence:", list(buf)[:6])
PY
