"""Per-family serialised kernel times of the C2 step with / without epilogue fusion."""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2301_08984_b200 as pb  # noqa: E402

plan, meta = bench.load_plan(sys.argv[1] if len(sys.argv) > 1 else "c2_tp1")
inp = bench.synthetic_inputs(plan)
for flags in (0, pb.FUSE_EPILOGUES):
    with pb.Executor(plan, lane_gpus=[0], flags=flags) as ex:
        ex.set_inputs(inp)
        ex.run(3)
        ex.profile()
        prof = ex.profile()
    print("flags", flags, json.dumps(prof))
