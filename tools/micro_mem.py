"""Micro-benchmark: memory-bound kernels of the executor vs torch on the
same shapes (single-op plans replayed as CUDA graphs). Development tool."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2301_08984_b200 as pb  # noqa: E402
from plan_builder import single_op_plan  # noqa: E402


def ours(kind, shapes, out_shape, elem=2, iters=50, attrs=None):
    plan, out_pt = single_op_plan(kind, shapes, out_shape, elem, elem, attrs)
    rng = np.random.default_rng(0)
    with pb.Executor(plan, lane_gpus=[0]) as ex:
        ex.set_inputs({i: rng.integers(-2, 3, size=s).astype(np.float64) for i, s in enumerate(shapes)})
        ex.run(5)
        return ex.run(iters)


def torch_time(fn, iters=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


res = []
for (r, c) in [(8192, 2048), (8192, 8192)]:
    nbytes = r * c * 2
    ms = ours("add", [(r, c), (r, c)], (r, c))
    x = torch.randn(r, c, device="cuda", dtype=torch.bfloat16)
    y = torch.randn(r, c, device="cuda", dtype=torch.bfloat16)
    z = torch.empty_like(x)
    tms = torch_time(lambda: torch.add(x, y, out=z))
    res.append({"op": "add", "shape": [r, c], "ours_ms": ms, "ours_gbs": 3 * nbytes / ms / 1e6,
                "torch_ms": tms, "torch_gbs": 3 * nbytes / tms / 1e6})
    ms = ours("identity", [(r, c)], (r, c))
    tms = torch_time(lambda: z.copy_(x))
    res.append({"op": "copy", "shape": [r, c], "ours_ms": ms, "ours_gbs": 2 * nbytes / ms / 1e6,
                "torch_ms": tms, "torch_gbs": 2 * nbytes / tms / 1e6})
print(json.dumps(res, indent=1))
