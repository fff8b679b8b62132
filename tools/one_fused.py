"""One GEMM(+add) plan for ncu: `python tools/one_fused.py [fused|sep|gemm] [m n k]`."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2301_08984_b200 as pb  # noqa: E402
from plan_builder import matmul_add_plan, matmul_plan  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "fused"
m, n, k = (int(x) for x in sys.argv[2:5]) if len(sys.argv) > 4 else (8192, 8192, 2048)
rng = np.random.default_rng(0)
inp = {0: rng.integers(-1, 2, size=(m, k)).astype(np.float64), 1: rng.integers(-1, 2, size=(k, n)).astype(np.float64)}
if mode == "gemm":
    plan = matmul_plan(m, n, k)[0]
else:
    plan = matmul_add_plan(m, n, k)[0]
    inp[3] = rng.integers(-1, 2, size=(m, n)).astype(np.float64)
with pb.Executor(plan, lane_gpus=[0], flags=(pb.FUSE_EPILOGUES if mode == "fused" else pb.NO_FUSION) | pb.NO_GRAPH) as ex:
    ex.set_inputs(inp)
    ex.run(3)
