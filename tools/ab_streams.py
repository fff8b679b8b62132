"""A/B of launch options on the C2 TP=1 step (stream spreading, epilogue fusion)."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2301_08984_b200 as pb  # noqa: E402

plan, meta = bench.load_plan(sys.argv[1] if len(sys.argv) > 1 else "c2_tp1")
inp = bench.synthetic_inputs(plan)
for flags in (0, pb.FUSE_EPILOGUES, pb.SERIAL_LANES, pb.SERIAL_LANES | pb.FUSE_EPILOGUES, 0, pb.FUSE_EPILOGUES):
    with pb.Executor(plan, lane_gpus=[0], flags=flags) as ex:
        ex.set_inputs(inp)
        ex.run(5)
        ms = ex.run(30)
    print("flags", flags, "ms/step", round(ms, 4), "samples/s", round(meta["samples_per_step"] / ms * 1e3))
