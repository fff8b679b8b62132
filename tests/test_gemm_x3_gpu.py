"""fp32 GEMMs on the tensor cores: the 3xTF32 tcgen05 kernel (gemm_x3.cu).

Bar (north_star: "1e-5 fp32"): normwise relative error
max|C - C_fp64| / max|C_fp64| <= 1e-5 on random-normal fp32 operands, and
no worse than 4x the SIMT FFMA kernel's own fp32 error on the same inputs
(3xTF32 keeps ~fp32 accuracy, one TF32 product would not: ~1e-3).
Integer-valued operands below 2^11 split exactly (x_lo = 0): the products
are exact and fp32 accumulation keeps them so while partial sums stay below
2^24 — the reference's integer parity inputs stay bit-exact.
"""
import numpy as np
import pytest

import paper_2301_08984_b200 as pb
from plan_builder import matmul_plan

pytestmark = pytest.mark.gpu

SHAPES = [(128, 128, 64), (304, 520, 200), (1000, 1000, 1000), (136, 264, 40), (2048, 512, 4096), (512, 384, 36)]


def run(plan, inputs, out_pt, flags=0):
    with pb.Executor(plan, lane_gpus=[0], flags=flags) as ex:
        ex.set_inputs(inputs)
        ex.run(2)
        return ex.get_output(out_pt), ex.stats()


@pytest.mark.parametrize("m,n,k", SHAPES)
@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
def test_gemm_x3_vs_fp64(m, n, k, ta, tb):
    rng = np.random.default_rng(m * 5 + n * 3 + k)
    plan, out_pt = matmul_plan(m, n, k, ta, tb, in_elem=4, out_elem=4)
    a = rng.standard_normal((k, m) if ta else (m, k)).astype(np.float32).astype(np.float64)
    b = rng.standard_normal((n, k) if tb else (k, n)).astype(np.float32).astype(np.float64)
    out, st = run(plan, {0: a, 1: b}, out_pt)
    assert st["gemm_tc_per_step"] == 1
    ref = (a.T if ta else a) @ (b.T if tb else b)
    err = np.abs(out - ref).max() / np.abs(ref).max()
    simt, st2 = run(plan, {0: a, 1: b}, out_pt, flags=pb.NO_TENSOR_CORES)
    assert st2["gemm_tc_per_step"] == 0
    err_simt = np.abs(simt - ref).max() / np.abs(ref).max()
    assert err <= 1e-5, (err, err_simt)
    assert err <= 4 * err_simt + 1e-7, (err, err_simt)


@pytest.mark.parametrize("m,n,k,ta,tb", [(304, 520, 200, False, False), (1000, 1000, 1000, True, False),
                                         (512, 384, 4096, True, True), (2048, 256, 512, False, True)])
def test_gemm_x3_integer_exact(m, n, k, ta, tb):
    rng = np.random.default_rng(k)
    plan, out_pt = matmul_plan(m, n, k, ta, tb, in_elem=4, out_elem=4)
    a = rng.integers(-4, 5, size=(k, m) if ta else (m, k)).astype(np.float64)
    b = rng.integers(-4, 5, size=(n, k) if tb else (k, n)).astype(np.float64)
    out, st = run(plan, {0: a, 1: b}, out_pt)
    assert st["gemm_tc_per_step"] == 1
    assert np.array_equal(out, (a.T if ta else a) @ (b.T if tb else b))


def test_gemm_x3_config():
    assert pb.gemm_config(1024, 1024, 1024, a_bf16=False, b_bf16=False, c_bf16=False) == \
        {"tensor_cores": True, "tile_n": 128}
    # mixed element types and tiny shapes stay on the SIMT kernel
    assert not pb.gemm_config(1024, 1024, 1024, a_bf16=False, b_bf16=True, c_bf16=False)["tensor_cores"]
    assert not pb.gemm_config(64, 64, 64, a_bf16=False, b_bf16=False, c_bf16=False)["tensor_cores"]


def test_gemm_x3_disabled_falls_to_simt(monkeypatch):
    monkeypatch.setenv("PLANC_B200_TF32X3", "0")
    plan, out_pt = matmul_plan(256, 256, 256, in_elem=4, out_elem=4)
    rng = np.random.default_rng(1)
    a = rng.integers(-4, 5, size=(256, 256)).astype(np.float64)
    b = rng.integers(-4, 5, size=(256, 256)).astype(np.float64)
    out, st = run(plan, {0: a, 1: b}, out_pt)
    assert st["gemm_tc_per_step"] == 0
    assert np.array_equal(out, a @ b)
