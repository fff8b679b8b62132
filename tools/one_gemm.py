"""One matmul single-op plan, replayed as CUDA graph steps (ncu target):
  python tools/one_gemm.py m n k ta tb [group] [steps]"""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2301_08984_b200 as pb  # noqa: E402
from plan_builder import grouped_matmul_plan  # noqa: E402

m, n, k, ta, tb = (int(x) for x in sys.argv[1:6])
g = int(sys.argv[6]) if len(sys.argv) > 6 else 1
steps = int(sys.argv[7]) if len(sys.argv) > 7 else 3
plan = grouped_matmul_plan(g, m, n, k, bool(ta), bool(tb))
rng = np.random.default_rng(0)
inp = {}
for i in range(g):
    inp[3 * i] = rng.integers(-1, 2, size=(k, m) if ta else (m, k)).astype(np.float64)
    inp[3 * i + 1] = rng.integers(-1, 2, size=(n, k) if tb else (k, n)).astype(np.float64)
with pb.Executor(plan, lane_gpus=[0]) as ex:
    ex.set_inputs(inp)
    ex.run(2)
    print(m, n, k, ta, tb, g, "ms/step", ex.run(steps), pb.gemm_schedule(m, n, k, bool(ta), bool(tb), group=g))
