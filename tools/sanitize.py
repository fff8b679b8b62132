"""Runs a few golden plans (eager issue) for compute-sanitizer sweeps:
  compute-sanitizer --tool memcheck  python tools/sanitize.py
  compute-sanitizer --tool racecheck python tools/sanitize.py
  compute-sanitizer --tool synccheck python tools/sanitize.py
Checks results too, so a sanitizer-clean run is also a correct one."""
import json
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import golden_cases  # noqa: E402
import paper_2301_08984_b200 as pb  # noqa: E402

CASES = sys.argv[1:] or ["mlp_dp2", "gpt_block_tp2", "embed_shard2", "adapt_d1_to_d0_4", "gpt_block_fwd_tp2_mma",
                         "mlp_1f1b_dp2"]
bad = 0
for name in CASES:
    g = golden_cases.load(name)
    n = len(json.loads(g["plan"])["lanes"])
    with pb.Executor(g["plan"], lane_gpus=[0] * n, flags=pb.NO_GRAPH) as ex:
        ex.set_inputs(g["inputs"])
        ex.run(1)
        ok, msg = pb.compare_outputs(g["expected"], ex.outputs(), g["meta"]["rel_tol"], normwise=True)
    print(name, "ok" if ok else msg)
    bad += not ok
sys.exit(1 if bad else 0)
