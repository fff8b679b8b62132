"""Stream-K vs data-parallel tcgen05 GEMM per shape and tile width (single-op
plans replayed as CUDA graphs), with the scheduler's own pick, next to cuBLAS.
Development / evidence tool: python tools/gemm_streamk.py > out.json"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2301_08984_b200 as pb  # noqa: E402
from plan_builder import matmul_plan  # noqa: E402

SHAPES = [  # (name, m, n, k, ta, tb)
    ("c2 X.W", 8192, 2048, 2048, False, False),
    ("c2 X^T.dQ", 2048, 2048, 8192, True, False),
    ("c2 X2^T.dF1", 2048, 8192, 8192, True, False),
    ("c2 F.W2", 8192, 2048, 8192, False, False),
    ("c3 mb X.W", 2048, 2048, 2048, False, False),
    ("c3 mb X.W2", 2048, 2048, 8192, False, False),
    ("c4 X.W1", 16384, 512, 512, False, False),
    ("c4 dW", 512, 512, 16384, True, False),
    ("c5 X.W", 8192, 256, 256, False, False),
    ("c5 dW", 256, 256, 8192, True, False),
]


def ours(m, n, k, ta, tb, iters=50):
    plan, _ = matmul_plan(m, n, k, ta, tb)
    rng = np.random.default_rng(0)
    a = rng.integers(-1, 2, size=(k, m) if ta else (m, k)).astype(np.float64)
    b = rng.integers(-1, 2, size=(n, k) if tb else (k, n)).astype(np.float64)
    with pb.Executor(plan, lane_gpus=[0]) as ex:
        ex.set_inputs({0: a, 1: b})
        ex.run(5)
        return ex.run(iters)


def cublas(m, n, k, ta, tb, iters=50):
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


rows = []
for name, m, n, k, ta, tb in SHAPES:
    fl = 2.0 * m * n * k
    row = {"gemm": name, "m": m, "n": n, "k": k, "ta": ta, "tb": tb,
           "auto_schedule": pb.gemm_schedule(m, n, k, ta, tb)}
    for bn in ("auto", "256", "128", "64"):
        for sk in ("0", "2"):
            if bn == "auto":
                os.environ.pop("PLANC_B200_GEMM_BN", None)
            else:
                os.environ["PLANC_B200_GEMM_BN"] = bn
            os.environ["PLANC_B200_STREAMK"] = sk
            o = ours(m, n, k, ta, tb)
            row[f"bn{bn}_sk{sk}_us"] = round(o * 1e3, 2)
    os.environ.pop("PLANC_B200_GEMM_BN", None)
    os.environ.pop("PLANC_B200_STREAMK", None)
    o = ours(m, n, k, ta, tb)
    row["auto_us"] = round(o * 1e3, 2)
    row["auto_tflops"] = round(fl / o / 1e9, 1)
    c = cublas(m, n, k, ta, tb)
    row["cublas_us"] = round(c * 1e3, 2)
    row["cublas_tflops"] = round(fl / c / 1e9, 1)
    rows.append(row)
    print(json.dumps(row), flush=True)
