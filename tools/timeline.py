"""Measured vs simulated step timeline.

Runs one step of a benchmark plan with per-task CUDA events
(planc_b200_timeline) and, when the reference library is present
(oracle/_ref travels with the repo), the reference simulator's prediction
for the same plan (cluster constants of the plan: NVLink 900 GB/s,
1.39 PFLOP/s). Writes both in the simulator's timeline_json shape plus a
per-kind summary:  python tools/timeline.py c2_tp1 [out.json]
"""
import json
import sys
from collections import defaultdict

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2301_08984_b200 as pb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2_tp1"
out_path = sys.argv[2] if len(sys.argv) > 2 else f"gpurun_out/timeline_{name}.json"
plan, meta = bench.load_plan(name)
nl = len(json.loads(plan)["lanes"])
with pb.Executor(plan, lane_gpus=[0] * nl) as ex:
    ex.set_inputs(bench.synthetic_inputs(plan))
    ex.run(3)
    ex.timeline()  # warm
    measured = ex.timeline()


def summarize(tl):
    by = defaultdict(float)
    for e in tl:
        by[e["kind"]] += e["end"] - e["start"]
    span = max(e["end"] for e in tl) - min(e["start"] for e in tl)
    return {"makespan_s": span, "busy_s_by_kind": dict(by)}


res = {"plan": name, "measured": summarize(measured), "measured_timeline": measured}
try:
    from oracle import refpy

    sim = refpy.simulate(plan)
    res["simulated"] = {"makespan_s": sim["report"]["makespan"], "devices": sim["report"]["devices"]}
    res["simulated_timeline"] = sim["timeline"]
    res["measured_over_simulated"] = res["measured"]["makespan_s"] / sim["report"]["makespan"]
except Exception as e:  # reference library not shipped
    res["simulated"] = {"unavailable": str(e)[:200]}
with open(out_path, "w") as f:
    json.dump(res, f)
print(json.dumps({k: v for k, v in res.items() if not k.endswith("timeline")}, indent=1))
