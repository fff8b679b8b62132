"""One fused-attention single-op plan replayed as CUDA graph steps (ncu target):
  python tools/one_attn.py T heads head_dim seq causal [steps]"""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2301_08984_b200 as pb  # noqa: E402
from plan_builder import single_op_plan  # noqa: E402

T, heads, dh, seq, causal = (int(x) for x in sys.argv[1:6])
steps = int(sys.argv[6]) if len(sys.argv) > 6 else 3
D = heads * dh
plan, _ = single_op_plan("attention", [(T, D)] * 3, (T, D), 2, 2, {"head_dim": dh, "seq": seq, "causal": bool(causal)})
rng = np.random.default_rng(0)
with pb.Executor(plan, lane_gpus=[0]) as ex:
    ex.set_inputs({i: rng.standard_normal((T, D)) for i in range(3)})
    ex.run(2)
    print(T, heads, dh, seq, causal, "ms/step", ex.run(steps))
