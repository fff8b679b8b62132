"""Debug: C3 partitioned vs unpartitioned under launch-mode flags."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import bench  # noqa: E402
import paper_2301_08984_b200 as pb  # noqa: E402
from test_fullsize_gpu import init_inputs, terminal_outputs  # noqa: E402
import json  # noqa: E402

base = sys.argv[1] if len(sys.argv) > 1 else "c3_ref1"
part = sys.argv[2] if len(sys.argv) > 2 else "c3_pp4dp2"
plan0, _ = bench.load_plan(base)
inputs = init_inputs(plan0)
ids = terminal_outputs(plan0)


def run(plan, flags):
    nl = len(json.loads(plan)["lanes"])
    with pb.Executor(plan, lane_gpus=[0] * nl, flags=flags) as ex:
        ex.set_inputs(inputs)
        ex.run(0)
        return {i: ex.get_output(i) for i in ids}


ref = run(plan0, 0)
print("ref finite:", {i: bool(np.isfinite(ref[i]).all()) for i in ids})
plan, _ = bench.load_plan(part)
for flags in (pb.SERIAL_LANES | pb.NO_GRAPH, pb.SERIAL_LANES, pb.NO_GRAPH, 0):
    got = run(plan, flags)
    fin = {i: bool(np.isfinite(got[i]).all()) for i in ids}
    ok, msg = pb.compare_outputs(ref, got, 2e-2, normwise=True)
    print("flags", flags, "finite", fin, ok, msg[:200])
