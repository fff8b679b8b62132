"""Loader for the committed golden fixtures (tests/golden/<case>/)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names():
    with open(os.path.join(GOLDEN, "index.json")) as f:
        return json.load(f)


def load(name):
    d = os.path.join(GOLDEN, name)
    with open(os.path.join(d, "plan.json")) as f:
        plan = f.read()
    with open(os.path.join(d, "graph.json")) as f:
        graph = f.read()
    with open(os.path.join(d, "meta.json")) as f:
        meta = json.load(f)
    io = np.load(os.path.join(d, "io.npz"))
    pick = lambda p: {int(k[len(p):]): io[k] for k in io.files if k.startswith(p)}  # noqa: E731
    return dict(name=name, plan=plan, graph=graph, meta=meta, inputs=pick("in_"), expected=pick("exp_"),
                ref_plan=pick("ref_"), emulated=pick("emu_"))
