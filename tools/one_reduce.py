"""One column reduce-sum plan (8192 x 8192 bf16, axis 0) replayed a few
steps — for an ncu capture of reduce_cols_kernel. Development tool."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2301_08984_b200 as pb  # noqa: E402
from plan_builder import single_op_plan  # noqa: E402

r, c = (int(x) for x in (sys.argv[1:3] if len(sys.argv) > 2 else (8192, 8192)))
plan, _ = single_op_plan("reduce-sum", [(r, c)], (c,), 2, 2, {"axis": 0})
rng = np.random.default_rng(0)
with pb.Executor(plan, lane_gpus=[0]) as ex:
    ex.set_inputs({0: rng.integers(-2, 3, size=(r, c)).astype(np.float64)})
    ex.run(2)
    print(ex.run(5))
