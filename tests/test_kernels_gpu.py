"""Kernel-level GPU tests through single-op plans (C ABI).

GEMM: the tcgen05 path (bf16 operands, fp32 TMEM accumulation) against a
float64 matmul of the same bf16-rounded operands, over all transpose
combinations, tile tails, persistent multi-tile grids and fp32 output;
normwise tolerance 2^-8 (one bf16 rounding of the output). The SIMT path is
checked the same way with NO_TENSOR_CORES. Memory-bound kernels: exact on
integer data.
"""
import numpy as np
import pytest

import paper_2301_08984_b200 as pb
from plan_builder import matmul_plan, single_op_plan

pytestmark = pytest.mark.gpu


def bf16_round(x):
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16 << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def run_single(plan, inputs, out_pt, flags=0):
    with pb.Executor(plan, lane_gpus=[0], flags=flags) as ex:
        ex.set_inputs(inputs)
        ex.run(0)
        st = ex.stats()
        return ex.get_output(out_pt), st


GEMM_SHAPES = [
    (128, 256, 64), (256, 512, 128), (304, 520, 200), (1000, 1000, 1000),
    (2048, 2048, 8192), (8192, 2048, 2048), (1024, 8192, 512), (136, 264, 40),
]


@pytest.mark.parametrize("m,n,k", GEMM_SHAPES)
@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
def test_gemm_tcgen05_vs_fp64(m, n, k, ta, tb):
    if m * n * k > 2 ** 33 and (ta, tb) != (False, False):
        pytest.skip("one transpose variant at the largest shapes")
    rng = np.random.default_rng(m * 7 + n * 3 + k)
    plan, out_pt = matmul_plan(m, n, k, ta, tb)
    a = bf16_round(rng.standard_normal((k, m) if ta else (m, k)))
    b = bf16_round(rng.standard_normal((n, k) if tb else (k, n)))
    out, st = run_single(plan, {0: a, 1: b}, out_pt)
    assert st["gemm_tc_per_step"] == 1
    ref = (a.T if ta else a) @ (b.T if tb else b)
    err = np.abs(out - ref).max() / max(1.0, np.abs(ref).max())
    assert err < 2.0 ** -8, err


@pytest.mark.parametrize("bn", ["256", "128", "64"])
@pytest.mark.parametrize("m,n,k,ta,tb", [(304, 520, 200, False, False), (1000, 1000, 1000, True, False),
                                         (2048, 512, 4096, False, True), (512, 128, 384, True, True)])
def test_gemm_tcgen05_every_tile_width(bn, m, n, k, ta, tb, monkeypatch):
    monkeypatch.setenv("PLANC_B200_GEMM_BN", bn)
    rng = np.random.default_rng(m + n + k)
    plan, out_pt = matmul_plan(m, n, k, ta, tb)
    a = bf16_round(rng.standard_normal((k, m) if ta else (m, k)))
    b = bf16_round(rng.standard_normal((n, k) if tb else (k, n)))
    out, st = run_single(plan, {0: a, 1: b}, out_pt, flags=pb.NO_GRAPH)
    assert st["gemm_tc_per_step"] == 1
    ref = (a.T if ta else a) @ (b.T if tb else b)
    err = np.abs(out - ref).max() / max(1.0, np.abs(ref).max())
    assert err < 2.0 ** -8, err


@pytest.mark.parametrize("ta,tb", [(False, False), (True, True)])
def test_gemm_tcgen05_fp32_output(ta, tb):
    m, n, k = 384, 512, 320
    rng = np.random.default_rng(5)
    plan, out_pt = matmul_plan(m, n, k, ta, tb, in_elem=2, out_elem=4)
    a = rng.integers(-4, 5, size=(k, m) if ta else (m, k)).astype(np.float64)
    b = rng.integers(-4, 5, size=(n, k) if tb else (k, n)).astype(np.float64)
    out, st = run_single(plan, {0: a, 1: b}, out_pt)
    assert st["gemm_tc_per_step"] == 1
    ref = (a.T if ta else a) @ (b.T if tb else b)
    assert np.array_equal(out, ref)  # integer products, fp32 accumulate: exact


# Stream-K tail (PLANC_B200_STREAMK=2 forces it wherever it applies): shapes
# whose tiles do not fill whole waves, k not a multiple of a stream-K range,
# tails in m / n / k, several CTAs per tile and several tiles per CTA.
SK_SHAPES = [(512, 512, 16384, True, False), (256, 256, 8192, True, False), (8192, 2048, 2048, False, False),
             (2048, 2048, 8192, True, False), (1000, 1000, 3000, False, True), (304, 520, 4200, True, True),
             (136, 264, 1000, False, False)]


@pytest.mark.parametrize("bn", ["256", "128", "64"])
@pytest.mark.parametrize("m,n,k,ta,tb", SK_SHAPES)
def test_gemm_streamk_vs_fp64(bn, m, n, k, ta, tb, monkeypatch):
    monkeypatch.setenv("PLANC_B200_GEMM_BN", bn)
    monkeypatch.setenv("PLANC_B200_STREAMK", "2")
    sched = pb.gemm_schedule(m, n, k, ta, tb)
    rng = np.random.default_rng(m + 3 * n + k)
    plan, out_pt = matmul_plan(m, n, k, ta, tb)
    a = bf16_round(rng.standard_normal((k, m) if ta else (m, k)))
    b = bf16_round(rng.standard_normal((n, k) if tb else (k, n)))
    with pb.Executor(plan, lane_gpus=[0]) as ex:
        ex.set_inputs({0: a, 1: b})
        ex.run(3)  # graph replays: the tile counters must be re-armed each launch
        out = ex.get_output(out_pt)
        ex.run(2)
        again = ex.get_output(out_pt)
    ref = (a.T if ta else a) @ (b.T if tb else b)
    err = np.abs(out - ref).max() / max(1.0, np.abs(ref).max())
    assert err < 2.0 ** -8, (err, sched)
    assert np.array_equal(out, again)  # fixed reduction order: same bits every step


@pytest.mark.parametrize("m,n,k,ta,tb", [(512, 512, 16384, True, False), (304, 520, 4200, True, True)])
def test_gemm_streamk_fp32_exact(m, n, k, ta, tb, monkeypatch):
    """Integer operands: every partial and the k-ordered sum are exact."""
    monkeypatch.setenv("PLANC_B200_STREAMK", "2")
    monkeypatch.setenv("PLANC_B200_SPLITK", "0")
    assert pb.gemm_schedule(m, n, k, ta, tb, c_bf16=False)["sk_ctas"] > 0
    rng = np.random.default_rng(11)
    plan, out_pt = matmul_plan(m, n, k, ta, tb, in_elem=2, out_elem=4)
    a = rng.integers(-4, 5, size=(k, m) if ta else (m, k)).astype(np.float64)
    b = rng.integers(-4, 5, size=(n, k) if tb else (k, n)).astype(np.float64)
    out, st = run_single(plan, {0: a, 1: b}, out_pt)
    assert st["gemm_tc_per_step"] == 1
    assert np.array_equal(out, (a.T if ta else a) @ (b.T if tb else b))


@pytest.mark.parametrize("m,n,k", [(37, 53, 29), (128, 256, 64), (300, 200, 100)])
@pytest.mark.parametrize("ta,tb", [(False, False), (True, True), (True, False)])
@pytest.mark.parametrize("elem", [2, 4])
def test_gemm_simt(m, n, k, ta, tb, elem):
    rng = np.random.default_rng(m + n + k)
    plan, out_pt = matmul_plan(m, n, k, ta, tb, in_elem=elem, out_elem=4)
    a = rng.integers(-4, 5, size=(k, m) if ta else (m, k)).astype(np.float64)
    b = rng.integers(-4, 5, size=(n, k) if tb else (k, n)).astype(np.float64)
    out, st = run_single(plan, {0: a, 1: b}, out_pt, flags=pb.NO_TENSOR_CORES)
    assert st["gemm_tc_per_step"] == 0
    assert np.array_equal(out, (a.T if ta else a) @ (b.T if tb else b))


@pytest.mark.parametrize("kind,fn", [("add", np.add), ("mul", np.multiply), ("max", np.maximum)])
@pytest.mark.parametrize("n_in,shape,elem", [(2, (1031,), 4), (3, (64, 72), 2), (9, (8, 16), 4),
                                             (2, (4096, 2048), 2)])
def test_elementwise(kind, fn, n_in, shape, elem):
    rng = np.random.default_rng(n_in)
    plan, out_pt = single_op_plan(kind, [shape] * n_in, shape, elem, elem)
    ins = {i: rng.integers(-3, 4, size=shape).astype(np.float64) for i in range(n_in)}
    out, _ = run_single(plan, ins, out_pt)
    ref = ins[0]
    for i in range(1, n_in):
        ref = fn(ref, ins[i])
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("shape,axis", [((5, 7), 0), ((5, 7), 1), ((3, 4, 5), 1), ((9,), 0), ((2048, 1024), 1)])
def test_reduce_sum(shape, axis):
    rng = np.random.default_rng(3)
    out_shape = tuple(e for i, e in enumerate(shape) if i != axis) or (1,)
    plan, out_pt = single_op_plan("reduce-sum", [shape], out_shape, 4, 4, {"axis": axis})
    x = rng.integers(-4, 5, size=shape).astype(np.float64)
    out, _ = run_single(plan, {0: x}, out_pt)
    assert np.array_equal(out.reshape(-1), x.sum(axis=axis).reshape(-1))


# Column reductions split the axis over blocks (fp32 partials, summed in
# split order) and vectorise along the kept inner axis; row reductions load
# 16-byte vectors. Exact on integer data; same bits on every run.
@pytest.mark.parametrize("shape,axis,elem", [((8192, 2048), 0, 4), ((3, 4096, 520), 1, 4), ((64, 300, 40), 1, 4),
                                             ((200, 2048), 0, 2), ((7, 130, 33), 1, 2), ((4096, 1000), 1, 2),
                                             ((1000, 4096), 1, 4), ((65536, 8), 0, 4)])
def test_reduce_sum_vectorised(shape, axis, elem):
    rng = np.random.default_rng(sum(shape))
    out_shape = tuple(e for i, e in enumerate(shape) if i != axis) or (1,)
    plan, out_pt = single_op_plan("reduce-sum", [shape], out_shape, elem, elem, {"axis": axis})
    x = rng.integers(-1, 2, size=shape).astype(np.float64)
    with pb.Executor(plan, lane_gpus=[0]) as ex:
        ex.set_inputs({0: x})
        ex.run(2)
        out = ex.get_output(out_pt)
        ex.run(1)
        again = ex.get_output(out_pt)
    assert np.array_equal(out.reshape(-1), x.sum(axis=axis).reshape(-1))
    assert np.array_equal(out, again)


@pytest.mark.parametrize("h,elem", [(2048, 2), (100, 2), (512, 4), (33, 4)])
def test_embedding_lookup_vectorised(h, elem):
    """Gather of table rows (16-byte vectors when h allows), out-of-shard
    indices give zero rows (refexec.cpp:216-232)."""
    from plan_builder import embedding_plan

    vocab, n, lo, rows = 1000, 4096, 200, 500
    plan, out_pt = embedding_plan(n, vocab, h, lo, rows, elem)
    rng = np.random.default_rng(h)
    idx = rng.integers(0, vocab, size=n).astype(np.float64)
    table = rng.integers(-4, 5, size=(vocab, h)).astype(np.float64)
    out, _ = run_single(plan, {0: idx, 1: table}, out_pt)
    ref = np.where(((idx >= lo) & (idx < lo + rows))[:, None], table[idx.astype(int)], 0.0)
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("g,m,n,k,ta,tb", [(4, 16384, 512, 512, False, False), (3, 304, 520, 200, False, True),
                                           (4, 512, 512, 16384, True, False), (8, 1024, 256, 256, False, False),
                                           (2, 8192, 2048, 2048, False, True)])
def test_grouped_gemm_vs_fp64(g, m, n, k, ta, tb):
    """Independent same-shape GEMMs of a lane run as ONE grouped tcgen05
    launch (stream-K tail included); each member equals its own product."""
    from plan_builder import grouped_matmul_plan

    plan = grouped_matmul_plan(g, m, n, k, ta, tb)
    desc = pb.describe(plan)
    assert [i["group"] for i in desc["instrs"] if i["kind"] == "gemm"] == [g]
    rng = np.random.default_rng(g * 1000 + m + n + k)
    inputs = {}
    for i in range(g):
        inputs[3 * i] = bf16_round(rng.standard_normal((k, m) if ta else (m, k)))
        inputs[3 * i + 1] = bf16_round(rng.standard_normal((n, k) if tb else (k, n)))
    outs = {}
    for flags in (0, pb.NO_GROUPING):
        with pb.Executor(plan, lane_gpus=[0], flags=flags) as ex:
            ex.set_inputs(inputs)
            ex.run(2)
            assert ex.stats()["gemm_tc_per_step"] == (1 if flags == 0 else g)
            outs[flags] = {i: ex.get_output(3 * i + 2) for i in range(g)}
    for i in range(g):
        a, b = inputs[3 * i], inputs[3 * i + 1]
        ref = (a.T if ta else a) @ (b.T if tb else b)
        err = np.abs(outs[0][i] - ref).max() / max(1.0, np.abs(ref).max())
        assert err < 2.0 ** -8, (i, err)
        assert np.array_equal(outs[0][i], outs[pb.NO_GROUPING][i]) or err < 2.0 ** -8


@pytest.mark.parametrize("g,m,n,k,ta,tb", [(1, 256, 256, 8192, True, False), (4, 512, 512, 16384, True, False),
                                           (1, 304, 520, 2000, False, True), (2, 136, 264, 4096, True, True),
                                           (1, 256, 256, 8192, False, False)])
@pytest.mark.parametrize("c_fp32", [False, True])
def test_splitk_gemm_vs_fp64(g, m, n, k, ta, tb, c_fp32, monkeypatch):
    """Split-K (PLANC_B200_SPLITK=2 forces it): k-range partials in fp32,
    summed in split order by the reduce kernel; single and grouped launches."""
    from plan_builder import grouped_matmul_plan

    monkeypatch.setenv("PLANC_B200_SPLITK", "2")
    monkeypatch.setenv("PLANC_B200_STREAMK", "0")
    plan = grouped_matmul_plan(g, m, n, k, ta, tb, out_elem=4 if c_fp32 else 2)
    rng = np.random.default_rng(g * 7 + m + n + k)
    inputs = {}
    for i in range(g):
        inputs[3 * i] = bf16_round(rng.standard_normal((k, m) if ta else (m, k)))
        inputs[3 * i + 1] = bf16_round(rng.standard_normal((n, k) if tb else (k, n)))
    with pb.Executor(plan, lane_gpus=[0]) as ex:
        ex.set_inputs(inputs)
        ex.run(3)
        st = ex.stats()
        outs = [ex.get_output(3 * i + 2) for i in range(g)]
    assert st["gemm_tc_per_step"] == 1 and st["kernels_per_step"] == 2  # GEMM + split-K reduce
    for i in range(g):
        a, b = inputs[3 * i], inputs[3 * i + 1]
        ref = (a.T if ta else a) @ (b.T if tb else b)
        err = np.abs(outs[i] - ref).max() / max(1.0, np.abs(ref).max())
        assert err < (2.0 ** -16 if c_fp32 else 2.0 ** -8), (i, err)


@pytest.mark.parametrize("g,m,n,k,ta,tb", [(1, 8192, 256, 256, False, False), (1, 304, 520, 200, True, True),
                                           (3, 1024, 384, 512, False, True), (1, 2048, 64, 1024, True, False),
                                           (2, 4096, 1024, 2048, False, False)])
def test_two_ctas_per_sm_variant_vs_fp64(g, m, n, k, ta, tb, monkeypatch):
    """The short-k variant (two CTAs per SM, ~76 KB ring, BN <= 128; forced
    here with PLANC_B200_OCC2=2, incl. a long-k shape) against fp64."""
    from plan_builder import grouped_matmul_plan

    monkeypatch.setenv("PLANC_B200_OCC2", "2")
    monkeypatch.setenv("PLANC_B200_SPLITK", "0")
    assert pb.gemm_schedule(m, n, k, ta, tb, group=g)["ctas_per_sm"] == 2
    plan = grouped_matmul_plan(g, m, n, k, ta, tb)
    rng = np.random.default_rng(g + m + n + k)
    inputs = {}
    for i in range(g):
        inputs[3 * i] = bf16_round(rng.standard_normal((k, m) if ta else (m, k)))
        inputs[3 * i + 1] = bf16_round(rng.standard_normal((n, k) if tb else (k, n)))
    with pb.Executor(plan, lane_gpus=[0]) as ex:
        ex.set_inputs(inputs)
        ex.run(2)
        outs = [ex.get_output(3 * i + 2) for i in range(g)]
    for i in range(g):
        a, b = inputs[3 * i], inputs[3 * i + 1]
        ref = (a.T if ta else a) @ (b.T if tb else b)
        assert np.abs(outs[i] - ref).max() / max(1.0, np.abs(ref).max()) < 2.0 ** -8


@pytest.mark.parametrize("g,m,n,k,ta,tb", [(1, 8192, 2048, 2048, False, False), (1, 1000, 1000, 1000, True, False),
                                           (2, 2048, 512, 4096, False, True), (1, 384, 256, 512, True, True)])
def test_cluster_pair_multicast_variant_vs_fp64(g, m, n, k, ta, tb, monkeypatch):
    """Clusters of two CTAs along M sharing each B tile by TMA multicast
    (forced with PLANC_B200_CLUSTER=2; odd M-block counts give a zero tile
    whose stores are clipped) against fp64."""
    from plan_builder import grouped_matmul_plan

    monkeypatch.setenv("PLANC_B200_CLUSTER", "2")
    monkeypatch.setenv("PLANC_B200_EPI8", "0")
    plan = grouped_matmul_plan(g, m, n, k, ta, tb)
    rng = np.random.default_rng(g + 3 * m + n + k)
    inputs = {}
    for i in range(g):
        inputs[3 * i] = bf16_round(rng.standard_normal((k, m) if ta else (m, k)))
        inputs[3 * i + 1] = bf16_round(rng.standard_normal((n, k) if tb else (k, n)))
    with pb.Executor(plan, lane_gpus=[0]) as ex:
        ex.set_inputs(inputs)
        ex.run(2)
        outs = [ex.get_output(3 * i + 2) for i in range(g)]
    for i in range(g):
        a, b = inputs[3 * i], inputs[3 * i + 1]
        ref = (a.T if ta else a) @ (b.T if tb else b)
        assert np.abs(outs[i] - ref).max() / max(1.0, np.abs(ref).max()) < 2.0 ** -8


@pytest.mark.parametrize("g,m,n,k,ta,tb", [(1, 4096, 2048, 2048, False, False), (1, 1000, 1024, 1000, True, False),
                                           (2, 2048, 512, 1536, False, True), (1, 384, 256, 512, True, True)])
def test_two_sm_variant_vs_fp64(g, m, n, k, ta, tb, monkeypatch):
    """The 2-SM variant (a CTA pair issuing one 256-row tcgen05.mma with
    cta_group::2; forced with PLANC_B200_2SM=2; odd M-block counts give a
    zero half tile whose stores are clipped) against fp64."""
    from plan_builder import grouped_matmul_plan

    monkeypatch.setenv("PLANC_B200_2SM", "2")
    monkeypatch.setenv("PLANC_B200_SPLITK", "0")
    monkeypatch.setenv("PLANC_B200_OCC2", "0")
    monkeypatch.setenv("PLANC_B200_EPI8", "0")
    plan = grouped_matmul_plan(g, m, n, k, ta, tb)
    rng = np.random.default_rng(g + 5 * m + n + k)
    inputs = {}
    for i in range(g):
        inputs[3 * i] = bf16_round(rng.standard_normal((k, m) if ta else (m, k)))
        inputs[3 * i + 1] = bf16_round(rng.standard_normal((n, k) if tb else (k, n)))
    with pb.Executor(plan, lane_gpus=[0]) as ex:
        ex.set_inputs(inputs)
        ex.run(2)
        outs = [ex.get_output(3 * i + 2) for i in range(g)]
    for i in range(g):
        a, b = inputs[3 * i], inputs[3 * i + 1]
        ref = (a.T if ta else a) @ (b.T if tb else b)
        assert np.abs(outs[i] - ref).max() / max(1.0, np.abs(ref).max()) < 2.0 ** -8


@pytest.mark.parametrize("two_sm", ["0", "2"])
@pytest.mark.parametrize("m,n,k,ta,tb", [(4096, 1024, 2048, False, False), (1000, 512, 768, True, False),
                                         (384, 256, 512, False, True),
                                         # several tiles per CTA with a partial last wave (the
                                         # epilogue's operand prefetch runs across tile boundaries)
                                         (8192, 2048, 2048, False, False), (2000, 1536, 1024, False, True),
                                         # short k: eight epilogue warps (C4's shape)
                                         (16384, 512, 512, False, False), (16384, 512, 512, False, True),
                                         (8192, 64, 512, False, False)])
def test_fused_epilogue_vs_fp64(m, n, k, ta, tb, two_sm, monkeypatch):
    """C = op(A)·op(B), E = C + D with the add fused into the GEMM's epilogue
    (default lowering), on the one-CTA and the 2-SM variant: C and E equal
    the separate kernels' bits (E = bf16(bf16(C) + D))."""
    from plan_builder import matmul_add_plan

    monkeypatch.setenv("PLANC_B200_2SM", two_sm)
    monkeypatch.setenv("PLANC_B200_SPLITK", "0")
    plan, out = matmul_add_plan(m, n, k, ta, tb)
    rng = np.random.default_rng(m + n + k + int(two_sm))
    a = bf16_round(rng.standard_normal((k, m) if ta else (m, k)))
    b = bf16_round(rng.standard_normal((n, k) if tb else (k, n)))
    d = bf16_round(rng.standard_normal((m, n)))
    res = {}
    for flags in (0, pb.NO_FUSION):
        with pb.Executor(plan, lane_gpus=[0], flags=flags) as ex:
            ex.set_inputs({0: a, 1: b, 3: d})
            ex.run(2)
            res[flags] = (ex.read_buffer(2).reshape(m, n), ex.get_output(out))
    assert pb.describe(plan)["instrs"][0]["label"] == "op+add"  # one fused launch
    ref = (a.T if ta else a) @ (b.T if tb else b)
    assert np.abs(res[0][0] - ref).max() / max(1.0, np.abs(ref).max()) < 2.0 ** -8
    assert np.array_equal(res[0][0], res[pb.NO_FUSION][0])
    assert np.array_equal(res[0][1], res[pb.NO_FUSION][1])


@pytest.mark.parametrize("two_sm", ["0", "2"])
@pytest.mark.parametrize("m,n,k", [(4096, 1024, 2048), (1000, 512, 768)])
def test_fused_gelu_epilogue(m, n, k, two_sm, monkeypatch):
    """G = gelu(op(A)·op(B)) with GELU in the GEMM's epilogue (both
    variants): C and G equal the separate kernels' bits (one GELU
    definition, gelu.cuh, applied to the bf16-rounded C), G within bf16 of
    the fp64 erf GELU of C."""
    from math import erf

    from plan_builder import matmul_gelu_plan

    monkeypatch.setenv("PLANC_B200_2SM", two_sm)
    plan, out = matmul_gelu_plan(m, n, k)
    assert pb.describe(plan, flags=pb.FUSE_ACT)["instrs"][0]["label"] == "op+act"
    rng = np.random.default_rng(m + n + k + 7 * int(two_sm))
    a = bf16_round(rng.standard_normal((m, k)) / 16)
    b = bf16_round(rng.standard_normal((k, n)))
    res = {}
    for flags in (pb.FUSE_ACT, pb.NO_FUSION):
        with pb.Executor(plan, lane_gpus=[0], flags=flags) as ex:
            ex.set_inputs({0: a, 1: b})
            ex.run(2)
            res[flags] = (ex.read_buffer(2).reshape(m, n), ex.get_output(out))
    assert np.array_equal(res[pb.FUSE_ACT][0], res[pb.NO_FUSION][0])
    assert np.array_equal(res[pb.FUSE_ACT][1], res[pb.NO_FUSION][1])
    c = res[pb.FUSE_ACT][0]
    ref = c * 0.5 * (1 + np.vectorize(erf)(c / np.sqrt(2)))
    assert np.abs(res[pb.FUSE_ACT][1] - ref).max() <= 2.0 ** -7 * max(1.0, np.abs(ref).max())
