"""fp32 GEMM throughput: the 3xTF32 tcgen05 path (gemm_x3.cu) and the SIMT
FFMA tile (NO_TENSOR_CORES) on single-op fp32 plans replayed as CUDA graphs,
next to cuBLAS fp32 (torch, allow_tf32 off: FFMA SGEMM) and cuBLAS TF32
(allow_tf32 on: one TF32 product, the tensor-pipe peak for 32-bit operands)
on the same shapes. Also the accuracy of each against float64.
Development / evidence tool: prints one JSON document."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2301_08984_b200 as pb  # noqa: E402
from plan_builder import matmul_plan  # noqa: E402

SHAPES = [(4096, 4096, 4096, False, False), (8192, 8192, 8192, False, False), (8192, 2048, 2048, False, False),
          (2048, 2048, 8192, True, False), (4096, 4096, 4096, False, True), (4096, 4096, 4096, True, True)]


def ours(m, n, k, ta, tb, flags=0, iters=10):
    plan, out_pt = matmul_plan(m, n, k, ta, tb, in_elem=4, out_elem=4)
    rng = np.random.default_rng(0)
    a = rng.standard_normal((k, m) if ta else (m, k)).astype(np.float32).astype(np.float64)
    b = rng.standard_normal((n, k) if tb else (k, n)).astype(np.float32).astype(np.float64)
    with pb.Executor(plan, lane_gpus=[0], flags=flags) as ex:
        ex.set_inputs({0: a, 1: b})
        ex.run(3)
        ms = ex.run(iters)
        out = ex.get_output(out_pt)
        st = ex.stats()
    A = torch.from_numpy(a).cuda()
    B = torch.from_numpy(b).cuda()
    ref = ((A.t() if ta else A) @ (B.t() if tb else B)).cpu().numpy()
    err = float(np.abs(out - ref).max() / np.abs(ref).max())
    return ms, err, st["gemm_tc_per_step"]


def cublas(m, n, k, ta, tb, tf32, iters=10):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn((k, m) if ta else (m, k), device="cuda", dtype=torch.float32)
    b = torch.randn((n, k) if tb else (k, n), device="cuda", dtype=torch.float32)
    A = a.t() if ta else a
    B = b.t() if tb else b
    for _ in range(3):
        torch.matmul(A, B)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        torch.matmul(A, B)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    ref = (A.double() @ B.double())
    err = float(((A @ B).double() - ref).abs().max() / ref.abs().max())
    torch.backends.cuda.matmul.allow_tf32 = False
    return ms, err


rows = []
for m, n, k, ta, tb in SHAPES:
    fl = 2.0 * m * n * k
    row = {"m": m, "n": n, "k": k, "ta": ta, "tb": tb}
    ms, err, tc = ours(m, n, k, ta, tb)
    row.update(x3_tflops=round(fl / ms / 1e9, 1), x3_err=err, x3_tc=tc)
    if m * n * k <= 4096 ** 3:
        ms, err, tc = ours(m, n, k, ta, tb, flags=pb.NO_TENSOR_CORES, iters=3)
        row.update(simt_tflops=round(fl / ms / 1e9, 1), simt_err=err)
    ms, err = cublas(m, n, k, ta, tb, False)
    row.update(cublas_fp32_tflops=round(fl / ms / 1e9, 1), cublas_fp32_err=err)
    ms, err = cublas(m, n, k, ta, tb, True)
    row.update(cublas_tf32_tflops=round(fl / ms / 1e9, 1), cublas_tf32_err=err)
    rows.append(row)
    print(json.dumps(row), file=sys.stderr)
print(json.dumps(rows, indent=1))
