"""Fused attention kind (schema extension) on the GPU:
the tcgen05 flash-attention kernel (attention.cu) against the float64
oracle (oracle/planc_oracle.py attention) on bf16-rounded operands.

Bar: normwise max|O - O_fp64| / max|O_fp64| <= 1e-2 (P is rounded to bf16
before the P·V product, as in every bf16 flash-attention kernel; the
output is bf16). Unsupported shapes raise UsageError at open.
"""
import numpy as np
import pytest

import paper_2301_08984_b200 as pb
from oracle import planc_oracle
from plan_builder import single_op_plan

pytestmark = pytest.mark.gpu


def bf16_round(x):
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16 << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def attention_plan(T, D, dh, seq, causal, elem=2):
    return single_op_plan("attention", [(T, D)] * 3, (T, D), elem, elem, {"head_dim": dh, "seq": seq, "causal": causal})


@pytest.mark.parametrize("T,heads,dh,seq,causal", [(256, 2, 128, 256, False), (512, 4, 64, 256, True),
                                                   (1024, 2, 128, 512, True), (768, 3, 64, 384, False),
                                                   (2048, 1, 128, 2048, False), (4096, 2, 128, 2048, True)])
def test_attention_vs_fp64(T, heads, dh, seq, causal):
    rng = np.random.default_rng(T + heads + dh)
    D = heads * dh
    plan, out_pt = attention_plan(T, D, dh, seq, causal)
    q, k, v = (bf16_round(rng.standard_normal((T, D))) for _ in range(3))
    with pb.Executor(plan, lane_gpus=[0]) as ex:
        ex.set_inputs({0: q, 1: k, 2: v})
        ex.run(2)
        out = ex.get_output(out_pt)
        prof = ex.profile()
    ref = planc_oracle.attention(q, k, v, dh, seq, causal)
    err = np.abs(out - ref).max() / np.abs(ref).max()
    assert err <= 1e-2, err
    assert any(p["kind"] == "attention" for p in prof)


def test_attention_large_scores():
    """Scores far from 0 (online-softmax rescaling across key blocks)."""
    T, dh, seq = 1024, 128, 1024
    rng = np.random.default_rng(7)
    plan, out_pt = attention_plan(T, dh, dh, seq, False)
    q = bf16_round(4 * rng.standard_normal((T, dh)))
    k = bf16_round(4 * rng.standard_normal((T, dh)))
    v = bf16_round(rng.standard_normal((T, dh)))
    with pb.Executor(plan, lane_gpus=[0]) as ex:
        ex.set_inputs({0: q, 1: k, 2: v})
        ex.run(0)
        out = ex.get_output(out_pt)
    ref = planc_oracle.attention(q, k, v, dh, seq, False)
    assert np.abs(out - ref).max() / np.abs(ref).max() <= 1e-2


@pytest.mark.parametrize("T,D,dh,seq,elem,why", [(256, 128, 128, 256, 4, "bf16"), (256, 192, 96, 256, 2, "head_dim"),
                                                 (320, 128, 128, 160, 2, "multiple of 128")])
def test_attention_unsupported_shapes(T, D, dh, seq, elem, why):
    plan, _ = attention_plan(T, D, dh, seq, False, elem)
    with pytest.raises(pb.PlancError, match=why):
        pb.Executor(plan, lane_gpus=[0])


@pytest.mark.parametrize("T,heads,dh,seq,causal", [(256, 2, 128, 256, False), (512, 2, 64, 256, True),
                                                   (1024, 2, 128, 512, True), (768, 1, 128, 384, False)])
@pytest.mark.parametrize("wrt", ["q", "k", "v"])
def test_attention_grad_vs_fp64(T, heads, dh, seq, causal, wrt):
    """attention-grad (statistics pass, then the dQ or dK / dV kernel) against
    the float64 gradient (pinned against torch autograd in
    tests/test_ext_oracle.py) — normwise <= 2e-2 (bf16 P and dS operands)."""
    rng = np.random.default_rng(T + heads + dh + ord(wrt))
    D = heads * dh
    q, k, v, do = (bf16_round(rng.standard_normal((T, D))) for _ in range(4))
    o = bf16_round(planc_oracle.attention(q, k, v, dh, seq, causal))
    plan, out_pt = single_op_plan("attention-grad", [(T, D)] * 5, (T, D), 2, 2,
                                  {"head_dim": dh, "seq": seq, "causal": causal, "wrt": wrt})
    with pb.Executor(plan, lane_gpus=[0]) as ex:
        ex.set_inputs({0: q, 1: k, 2: v, 3: o, 4: do})
        ex.run(2)
        out = ex.get_output(out_pt)
        prof = ex.profile()
    ref = planc_oracle.attention_grad(q, k, v, o, do, dh, seq, causal, wrt)
    err = np.abs(out - ref).max() / np.abs(ref).max()
    assert err <= 2e-2, err
    assert any(p["kind"] == "attention_grad" for p in prof)
