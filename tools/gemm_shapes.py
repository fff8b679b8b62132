"""Per-shape tcgen05 GEMM throughput for the C2 block's GEMMs (single-op
plans replayed as CUDA graphs) next to cuBLAS (torch.matmul) on the same
shapes and transposes. Development / evidence tool."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2301_08984_b200 as pb  # noqa: E402
from plan_builder import matmul_plan  # noqa: E402

T, H, F = 8192, 2048, 8192
SHAPES = [  # (name, m, n, k, ta, tb)
    ("fwd X.W (q/k/o)", T, H, H, False, False),
    ("fwd X2.W1", T, F, H, False, False),
    ("fwd F.W2", T, H, F, False, False),
    ("bwd dY.W2^T", T, F, H, False, True),
    ("bwd dF1.W1^T", T, H, F, False, True),
    ("bwd dQ.Wq^T", T, H, H, False, True),
    ("bwd Fa^T.dY", F, H, T, True, False),
    ("bwd X2^T.dF1", H, F, T, True, False),
    ("bwd X^T.dQ", H, H, T, True, False),
    ("c4 shard X.W1", 16384, 512, 512, False, False),
    ("c4 shard dT^T", 512, 512, 16384, True, False),
    ("c5 mb X.W", 8192, 256, 256, False, False),
    ("c5 mb dX", 8192, 256, 256, False, True),
]


def ours(m, n, k, ta, tb, iters=30):
    plan, _ = matmul_plan(m, n, k, ta, tb)
    rng = np.random.default_rng(0)
    a = rng.integers(-1, 2, size=(k, m) if ta else (m, k)).astype(np.float64)
    b = rng.integers(-1, 2, size=(n, k) if tb else (k, n)).astype(np.float64)
    with pb.Executor(plan, lane_gpus=[0]) as ex:
        ex.set_inputs({0: a, 1: b})
        ex.run(5)
        return ex.run(iters)


def cublas(m, n, k, ta, tb, iters=30):
    a = torch.randn((k, m) if ta else (m, k), device="cuda", dtype=torch.bfloat16)
    b = torch.randn((n, k) if tb else (k, n), device="cuda", dtype=torch.bfloat16)
    A = a.t() if ta else a
    B = b.t() if tb else b
    for _ in range(5):
        torch.matmul(A, B)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        torch.matmul(A, B)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


import os  # noqa: E402

rows = []
for name, m, n, k, ta, tb in SHAPES:
    fl = 2.0 * m * n * k
    row = {"gemm": name, "m": m, "n": n, "k": k, "ta": ta, "tb": tb}
    for bn in ("auto", "256", "128", "64"):
        if bn == "auto":
            os.environ.pop("PLANC_B200_GEMM_BN", None)
        else:
            os.environ["PLANC_B200_GEMM_BN"] = bn
        o = ours(m, n, k, ta, tb)
        row[f"ours_{bn}_tflops"] = round(fl / o / 1e9, 1)
    os.environ.pop("PLANC_B200_GEMM_BN", None)
    c = cublas(m, n, k, ta, tb)
    row["cublas_tflops"] = round(fl / c / 1e9, 1)
    rows.append(row)
print(json.dumps(rows, indent=1))
