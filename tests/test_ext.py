"""Schema extension (softmax / layernorm / GELU and gradients) on CPU: the
executor's lowering of the extended kinds, interpreted in numpy
(tests/program_emu.py), reproduces the float64 graph-level oracle; the
partitioned oracle run agrees; misaligned pieces are rejected like the
reference rejects bad plans (UsageError)."""
import json
import os

import numpy as np
import pytest

import golden_cases
import paper_2301_08984_b200 as pb
from oracle import planc_oracle as po
from program_emu import run_program

EXT = json.load(open(os.path.join(golden_cases.GOLDEN, "index_ext.json")))


@pytest.mark.parametrize("name", EXT)
def test_ext_lowering_reproduces_oracle(name):
    g = golden_cases.load(name)
    desc = pb.describe(g["plan"])
    kinds = {i["kind"] for i in desc["instrs"]}
    assert kinds & {"rowwise", "attention"}
    out = run_program(desc, json.loads(g["plan"]), g["inputs"])
    # float64 interpretation vs the float64 graph run (the fixture's bf16
    # cases store bf16-rounded expectations for the GPU comparison)
    ok, msg = pb.compare_outputs(po.run_graph(g["graph"], g["inputs"]), out, 1e-9, normwise=True)
    assert ok, msg


@pytest.mark.parametrize("name", EXT)
def test_ext_partitioned_oracle_matches_graph_oracle(name):
    g = golden_cases.load(name)
    ok, msg = po.compare_outputs(po.run_graph(g["graph"], g["inputs"]), po.run_plan(g["plan"], g["inputs"]), 1e-9)
    if g["meta"]["spec"]["elem_size"] == 4:
        ok, msg = po.compare_outputs(g["expected"], po.run_plan(g["plan"], g["inputs"]), 1e-9)
        assert ok, msg
    assert ok, msg


def test_ext_segments_follow_heads():
    g = golden_cases.load("ext_block_tp2")
    desc = pb.describe(g["plan"])
    rows = [i for i in desc["instrs"] if i["kind"] == "rowwise"]
    sm = [i for i in rows if i["row_op"] in (0, 1)]
    ln = [i for i in rows if i["row_op"] in (2, 3)]
    assert sm and ln
    assert all(i["seg"] == 4 for i in sm)           # one attention head per segment
    assert all(i["seg"] == 16 for i in ln)          # layernorm over the whole hidden axis
    assert all(i["count"] % i["seg"] == 0 for i in sm + ln)


def test_ext_misaligned_piece_is_usage_error():
    g = golden_cases.load("ext_block_tp2")
    p = json.loads(g["plan"])
    for op in p["ops"]:
        if op["kind"] == "softmax":
            op["segment"] = 3  # 16 / 2 ranks = 8 columns per piece: not whole segments of 3
    with pytest.raises(pb.UsageError, match="segment"):
        pb.describe(json.dumps(p))


def test_ext_layernorm_on_split_rows_is_usage_error():
    g = golden_cases.load("ext_block_tp2")
    p = json.loads(g["plan"])
    for op in p["ops"]:
        if op["kind"] == "softmax":
            op["kind"] = "layernorm"  # a column-split piece cannot hold whole LayerNorm rows
            op.pop("segment", None)
    with pytest.raises(pb.UsageError):
        pb.describe(json.dumps(p))


def test_ext_unknown_kind_is_schema_error():
    g = golden_cases.load("ext_block_tp1")
    p = json.loads(g["plan"])
    p["ops"][0]["kind"] = "rotary-embedding"
    with pytest.raises(pb.SchemaError):
        pb.describe(json.dumps(p))


def test_attention_lowering_and_piece_rules():
    """Fused attention (schema extension): head (TP) and sequence splits lower
    to one attention instruction per lane; a piece cutting a sequence is a
    UsageError at lowering; the lowered program interpreted in numpy equals
    the float64 graph oracle."""
    import json

    import numpy as np

    from oracle import docs, planc_oracle, refpy
    from program_emu import run_program

    doc = docs.attention_doc(512, 2, 128, 256, causal=True)
    stand = docs.dumps(docs.standin_doc(doc))
    for spec in (dict(strategy="megatron_tp", devices=2), dict(strategy="manual", devices=2, target_ops="tpattn@s0")):
        plan = docs.rewrite_plan(refpy.compile_plan(stand, **spec), doc)
        d = pb.describe(plan)
        att = [i for i in d["instrs"] if i["kind"] == "attention"]
        assert len(att) == 2 and all(i["att"]["causal"] for i in att)
        rng = np.random.default_rng(1)
        inputs = {i: rng.standard_normal((512, 256)) for i in range(3)}
        out = run_program(d, json.loads(plan), inputs)
        ref = planc_oracle.run_graph(docs.dumps(doc), inputs)
        assert np.abs(out[3] - ref[3]).max() < 1e-12
    bad = docs.rewrite_plan(refpy.compile_plan(stand, strategy="manual", devices=4, target_ops="tpattn@s0"), doc)
    with pytest.raises(pb.UsageError, match="whole sequences"):
        pb.describe(bad)
