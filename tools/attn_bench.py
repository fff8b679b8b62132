"""Fused attention throughput (attention.cu) on single-op plans replayed as
CUDA graphs, next to torch scaled_dot_product_attention (cuDNN / flash
backends) on the same bf16 shapes. FLOPs = 4 * T * seq * D (x 0.5 causal).
Development / evidence tool: prints one JSON document."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2301_08984_b200 as pb  # noqa: E402
from plan_builder import attention_grad_plan, single_op_plan  # noqa: E402

ITERS = 20


def ours(T, D, dh, seq, causal):
    plan, _ = single_op_plan("attention", [(T, D)] * 3, (T, D), 2, 2, {"head_dim": dh, "seq": seq, "causal": causal})
    rng = np.random.default_rng(0)
    with pb.Executor(plan, lane_gpus=[0]) as ex:
        ex.set_inputs({i: rng.standard_normal((T, D)) for i in range(3)})
        ex.run(3)
        return ex.run(ITERS)


def ours_bwd(T, D, dh, seq, causal):
    plan, _ = attention_grad_plan(T, D, dh, seq, causal)
    rng = np.random.default_rng(0)
    with pb.Executor(plan, lane_gpus=[0]) as ex:
        ex.set_inputs({i: rng.standard_normal((T, D)) for i in range(5)})
        ex.run(3)
        return ex.run(ITERS)


def sdpa_bwd(T, D, dh, seq, causal):
    b, h = T // seq, D // dh
    q, k, v = (torch.randn(b, h, seq, dh, device="cuda", dtype=torch.bfloat16, requires_grad=True) for _ in range(3))
    o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=causal)
    g = torch.randn_like(o)
    f = lambda: torch.autograd.grad(o, (q, k, v), g, retain_graph=True)  # noqa: E731
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(ITERS):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / ITERS


def sdpa(T, D, dh, seq, causal):
    b, h = T // seq, D // dh
    q, k, v = (torch.randn(b, h, seq, dh, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    f = lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=causal)  # noqa: E731
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(ITERS):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / ITERS


rows = []
for T, heads, dh, seq, causal in [(8192, 16, 128, 2048, False), (8192, 16, 128, 2048, True),
                                  (16384, 16, 128, 4096, True), (8192, 32, 64, 2048, False)]:
    D = heads * dh
    fl = 4.0 * T * seq * D * (0.5 if causal else 1.0)
    r = {"tokens": T, "heads": heads, "head_dim": dh, "seq": seq, "causal": causal}
    ms = ours(T, D, dh, seq, causal)
    r.update(ours_ms=ms, ours_tflops=fl / ms / 1e9)
    ms = sdpa(T, D, dh, seq, causal)
    r.update(sdpa_ms=ms, sdpa_tflops=fl / ms / 1e9)
    # backward: algorithmic 2.5x the forward's flops (dQ, dK, dV and dP; FA convention)
    ms = ours_bwd(T, D, dh, seq, causal)
    r.update(bwd_ours_ms=ms, bwd_ours_tflops=2.5 * fl / ms / 1e9)
    ms = sdpa_bwd(T, D, dh, seq, causal)
    r.update(bwd_sdpa_ms=ms, bwd_sdpa_tflops=2.5 * fl / ms / 1e9)
    rows.append(r)
    print(json.dumps(r), file=sys.stderr)
print(json.dumps(rows, indent=1))
