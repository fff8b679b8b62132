"""Micro-benchmark: the executor's memory-bound kernels on single-op plans
replayed as CUDA graphs (inputs >> L2 where the shape allows), achieved
GB/s of algorithmic bytes (inputs read once + output written once) against
the measured HBM peak (MEASURED_PEAKS.json), next to torch on the same op.
Development / evidence tool: prints one JSON document."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2301_08984_b200 as pb  # noqa: E402
from plan_builder import embedding_plan, single_op_plan  # noqa: E402

ITERS = 30


def ours_plan(plan, inputs):
    with pb.Executor(plan, lane_gpus=[0]) as ex:
        ex.set_inputs(inputs)
        ex.run(3)
        return ex.run(ITERS)


def ours(kind, shapes, out_shape, elem=2, attrs=None):
    plan, _ = single_op_plan(kind, shapes, out_shape, elem, elem, attrs)
    rng = np.random.default_rng(0)
    return ours_plan(plan, {i: rng.integers(-2, 3, size=s).astype(np.float64) for i, s in enumerate(shapes)})


def torch_time(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(ITERS):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / ITERS


peaks = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "MEASURED_PEAKS.json")))
HBM = peaks["hbm_gbs"]
res = []


def row(op, shape, nbytes, ms, tms=None, **kw):
    r = {"op": op, "shape": list(shape), "bytes": nbytes, "ours_ms": ms, "ours_gbs": nbytes / ms / 1e6,
         "frac_hbm": nbytes / ms / 1e6 / HBM}
    if tms is not None:
        r.update(torch_ms=tms, torch_gbs=nbytes / tms / 1e6)
    r.update(kw)
    res.append(r)
    print(json.dumps(r), file=sys.stderr)


bf = torch.bfloat16
for (r, c) in [(8192, 8192), (16384, 8192)]:
    nb = r * c * 2
    x, y, w = (torch.randn(r, c, device="cuda", dtype=bf) for _ in range(3))
    z = torch.empty_like(x)
    row("add", (r, c), 3 * nb, ours("add", [(r, c), (r, c)], (r, c)), torch_time(lambda: torch.add(x, y, out=z)))
    row("add3", (r, c), 4 * nb, ours("add", [(r, c)] * 3, (r, c)), torch_time(lambda: torch.add(torch.add(x, y), w, out=z)))
    row("max", (r, c), 3 * nb, ours("max", [(r, c), (r, c)], (r, c)), torch_time(lambda: torch.maximum(x, y, out=z)))
    row("copy", (r, c), 2 * nb, ours("identity", [(r, c)], (r, c)), torch_time(lambda: z.copy_(x)))
    row("reduce_rows", (r, c), nb + r * 2, ours("reduce-sum", [(r, c)], (r,), attrs={"axis": 1}),
        torch_time(lambda: x.sum(dim=1)))
    row("reduce_cols", (r, c), nb + c * 2, ours("reduce-sum", [(r, c)], (c,), attrs={"axis": 0}),
        torch_time(lambda: x.sum(dim=0)))
    for kind, seg, attrs in [("softmax", 2048, {"segment": 2048}), ("layernorm", c, {"eps": 1e-5})]:
        row(kind, (r, c), 2 * nb, ours(kind, [(r, c)], (r, c), attrs=attrs),
            torch_time(lambda: torch.softmax(x.view(-1, seg), dim=-1)) if kind == "softmax" else
            torch_time(lambda: torch.nn.functional.layer_norm(x, (c,))))
    row("gelu", (r, c), 2 * nb, ours("gelu", [(r, c)], (r, c)), torch_time(lambda: torch.nn.functional.gelu(x)))
    row("gelu_grad", (r, c), 3 * nb, ours("gelu-grad", [(r, c), (r, c)], (r, c)))
# embedding lookup: n rows of h gathered from a [vocab, h] shard
for n, h in [(65536, 2048), (262144, 512)]:
    vocab = 50304
    plan, _ = embedding_plan(n, vocab, h, 0, vocab, 2)
    rng = np.random.default_rng(1)
    idx = rng.integers(0, vocab, size=n).astype(np.float64)
    table = rng.integers(-2, 3, size=(vocab, h)).astype(np.float64)
    ms = ours_plan(plan, {0: idx, 1: table})
    ti = torch.from_numpy(idx.astype(np.int64)).cuda()
    tt = torch.randn(vocab, h, device="cuda", dtype=bf)
    row("emb_lookup", (n, h), n * 4 + 2 * n * h * 2, ms, torch_time(lambda: torch.nn.functional.embedding(ti, tt)))
print(json.dumps({"hbm_peak_gbs": HBM, "rows": res}, indent=1))
