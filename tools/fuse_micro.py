"""GEMM + elementwise-add: separate kernels vs the fused tcgen05 epilogue,
per C2 shape and tile width. Development / evidence tool."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2301_08984_b200 as pb  # noqa: E402
from plan_builder import matmul_add_plan, matmul_plan  # noqa: E402

T, H, F = 8192, 2048, 8192
SHAPES = [("X.W", T, H, H, False, False), ("X2.W1", T, F, H, False, False), ("F.W2", T, H, F, False, False),
          ("dY.W2^T", T, F, H, False, True), ("Fa^T.dY", F, H, T, True, False)]


def run(plan, inputs, flags, iters=30):
    with pb.Executor(plan, lane_gpus=[0], flags=flags) as ex:
        ex.set_inputs(inputs)
        ex.run(5)
        return ex.run(iters)


rows = []
rng = np.random.default_rng(0)
for name, m, n, k, ta, tb in SHAPES:
    a = rng.integers(-1, 2, size=(k, m) if ta else (m, k)).astype(np.float64)
    b = rng.integers(-1, 2, size=(n, k) if tb else (k, n)).astype(np.float64)
    d = rng.integers(-1, 2, size=(m, n)).astype(np.float64)
    row = {"gemm": name, "m": m, "n": n, "k": k}
    for bn in ("auto", "128"):
        if bn == "auto":
            os.environ.pop("PLANC_B200_GEMM_BN", None)
        else:
            os.environ["PLANC_B200_GEMM_BN"] = bn
        row[f"gemm_only_{bn}_ms"] = round(run(matmul_plan(m, n, k, ta, tb)[0], {0: a, 1: b}, 0), 4)
        p = matmul_add_plan(m, n, k, ta, tb)[0]
        row[f"sep_{bn}_ms"] = round(run(p, {0: a, 1: b, 3: d}, pb.SERIAL_LANES | pb.NO_FUSION), 4)
        row[f"fused_{bn}_ms"] = round(run(p, {0: a, 1: b, 3: d}, pb.FUSE_EPILOGUES), 4)
    os.environ.pop("PLANC_B200_GEMM_BN", None)
    rows.append(row)
    print(json.dumps(row), flush=True)
