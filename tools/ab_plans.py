"""A/B of executor options across benchmark plans: each variant is
(label, flags, {env}), measured round-robin `rounds` times as graph-replayed
steps (CUDA events inside the library); prints one JSON line per plan with
the median ms/step per variant. Development / evidence tool.

  python tools/ab_plans.py c2_tp1 c4_coshard4 c5_3f1b
"""
import json
import os
import statistics
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2301_08984_b200 as pb  # noqa: E402

VARIANTS = [
    ("base", 0, {}),
    ("no_grouping", pb.NO_GROUPING, {}),
    ("no_occ2", 0, {"PLANC_B200_OCC2": "0"}),
    ("two_sm", 0, {"PLANC_B200_2SM": "2"}),
    ("no_fusion", pb.NO_FUSION, {}),
]


if os.environ.get("AB_VARIANTS"):  # [[label, flags, {env}], ...]
    VARIANTS = [tuple(v) for v in json.loads(os.environ["AB_VARIANTS"])]


def run_variant(plan, inp, flags, env, steps=20):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        with pb.Executor(plan, lane_gpus=[0], flags=flags) as ex:
            ex.set_inputs(inp)
            ex.run(5)
            return ex.run(steps)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def main():
    names = sys.argv[1:] or ["c2_tp1"]
    rounds = int(os.environ.get("AB_ROUNDS", "3"))
    for name in names:
        plan, meta = bench.load_plan(name)
        inp = bench.synthetic_inputs(plan)
        res = {label: [] for label, _, _ in VARIANTS}
        for _ in range(rounds):
            for label, flags, env in VARIANTS:
                res[label].append(run_variant(plan, inp, flags, env))
        out = {"plan": name, "samples_per_step": meta["samples_per_step"]}
        for label in res:
            out[label + "_ms"] = round(statistics.median(res[label]), 4)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
