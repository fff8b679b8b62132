"""Host-side lowering and the C-ABI library, on CPU (no compute calls).

The executor compiles a plan into buffers + instructions + box cell
programs + issue order without touching CUDA (planc_b200_describe). A numpy
interpreter of that program (tests/program_emu.py, test-only) must reproduce
the reference outputs for every golden plan; error behaviour must match the
reference's exception classes.
"""
import ctypes
import json
import os
import re

import numpy as np
import pytest

import golden_cases
import paper_2301_08984_b200 as pb
from oracle import planc_oracle as po
from oracle import refpy
from program_emu import run_program

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "planc_b200.h")).read()
    declared = set(re.findall(r"\b(planc_b200_[a-z0-9_]+)\s*\(", header))
    assert len(declared) >= 15
    lib = ctypes.CDLL(pb.library_path())
    for sym in sorted(declared):
        assert hasattr(lib, sym), sym
    assert "sm_100a" in pb.version()


@pytest.mark.parametrize("flags", [0, pb.NO_FUSION])
@pytest.mark.parametrize("name", golden_cases.names())
def test_lowered_program_reproduces_reference(name, flags):
    g = golden_cases.load(name)
    desc = pb.describe(g["plan"], flags=flags)
    out = run_program(desc, json.loads(g["plan"]), g["inputs"])
    # float64 interpretation: exact unless values outgrow 2^53 (summation order)
    tol = 0.0 if g["meta"].get("max_abs", 0) < 2.0 ** 53 else 1e-12
    ok, msg = pb.compare_outputs(g["expected"], out, tol, normwise=True)
    assert ok, msg


@pytest.mark.parametrize("name", golden_cases.names())
def test_lowering_invariants(name):
    g = golden_cases.load(name)
    desc = pb.describe(g["plan"])
    writers = {}
    for ins in desc["instrs"]:
        for b in ins["out"]:
            writers.setdefault(b, []).append(ins["id"])
        for d in ins["deps"]:
            assert d < ins["id"], "dependencies point backwards in issue order"
    assert desc["issue_order"] == sorted(desc["issue_order"])
    # Every buffer element is written exactly once per step: a buffer with
    # several writers (two-phase all-reduce) is covered by disjoint box cells,
    # and its last writer depends on the others.
    nel = {b["id"]: b["bytes"] // (2 if b["dtype"] == "bf16" else 4) for b in desc["buffers"]}
    for b, ws in writers.items():
        if len(ws) == 1:
            continue
        hit = np.zeros(nel[b], dtype=np.int64)
        for w in ws:
            ins = desc["instrs"][w]
            assert ins["kind"] == "box" and ins["out"] == [b]
            for c in ins["cells"]:
                idx = c["dst_off"] + sum(np.arange(e).reshape([-1 if i == d else 1 for i in range(len(c["ext"]))]) * st
                                         for d, (e, st) in enumerate(zip(c["ext"], c["dst_str"])))
                np.add.at(hit, np.asarray(idx).reshape(-1), 1)
        assert (hit == 1).all(), f"buffer {b}: box writers overlap or leave gaps"
        assert set(ws[:-1]) <= set(desc["instrs"][ws[-1]]["deps"])
    for b in desc["buffers"]:
        assert b["offset"] % 256 == 0
        if b.get("dead"):  # replaced by reduce-scatter receive slices: nobody touches it
            assert b["id"] not in writers
            assert not any(b["id"] in i["in"] for i in desc["instrs"])
            continue
        if not b["graph_input"]:
            assert b["id"] in writers
    # Every box cell is in bounds of its source and destination buffers.
    size = {b["id"]: b["bytes"] // (2 if b["dtype"] == "bf16" else 4) for b in desc["buffers"]}
    for ins in desc["instrs"]:
        for c in ins["cells"]:
            hi = c["dst_off"] + sum((e - 1) * s for e, s in zip(c["ext"], c["dst_str"]))
            assert 0 <= c["dst_off"] and hi < size[ins["out"][0]]
            for t in c["terms"]:
                thi = t["off"] + sum((e - 1) * s for e, s in zip(c["ext"], t["str"]))
                assert 0 <= t["off"] and thi < size[t["buf"]]


def test_allreduce_runs_as_reduce_scatter_then_all_gather():
    g = golden_cases.load("adapt_v_to_r4")
    desc = pb.describe(g["plan"])
    rs = [i for i in desc["instrs"] if i["label"].endswith("#rs")]
    ag = [i for i in desc["instrs"] if i["label"].endswith("#ag")]
    assert len(rs) == 4 and len(ag) == 4
    for j, (r, a) in enumerate(zip(rs, ag)):
        assert r["lane"] == a["lane"] and r["out"] == a["out"]
        # phase 1: one slice, all four partials added in the same order
        assert len(r["cells"]) == 1 and len(r["cells"][0]["terms"]) == 4
        assert all(t["add"] for t in r["cells"][0]["terms"])
        # phase 2: the three other members' reduced slices, copied
        assert len(a["cells"]) == 3 and all(len(c["terms"]) == 1 and not c["terms"][0]["add"] for c in a["cells"])
        assert {t["buf"] for c in a["cells"] for t in c["terms"]} == {x["out"][0] for x in rs if x is not r}
        assert {x["id"] for x in rs} <= set(a["deps"])
        assert r["wire_bytes"] + a["wire_bytes"] > 0
    # the NCCL exchange lowering keeps one whole-buffer ncclAllReduce instead
    nccl = pb.describe(g["plan"], lane_rank=[0, 1, 2, 3])
    assert any(i["kind"] == "xfer" and i["allreduce"] for i in nccl["instrs"])


@pytest.mark.parametrize("name", ["adapt_v_to_r4", "mlp_dp2", "gpt_block_tp2", "mlp_1f1b_dp2", "three_pass_3f1b"])
def test_peer_sync_schedule(name):
    # Peer-memory rank mode: every cross-rank dependency edge is one flag
    # slot on the consumer's rank, signalled once by the producer.
    g = golden_cases.load(name)
    plan = json.loads(g["plan"])
    nl = len(plan["lanes"])
    for world in (2, nl):
        lane_rank = pb.lanes_round_robin(nl, world)
        desc = pb.describe(g["plan"], lane_rank=lane_rank, flags=pb.PEER_MEMORY)
        ps = desc["peer_sync"]
        assert not any(i["kind"] == "xfer" for i in desc["instrs"])
        rank_of = lambda i: lane_rank[desc["instrs"][i]["lane"]]  # noqa: E731
        expect_waits = 0
        seen = {}
        for ins in desc["instrs"]:
            cross = [d for d in ins["deps"] if desc["instrs"][d]["kind"] != "nop" and rank_of(d) != rank_of(ins["id"])]
            if ins["kind"] == "nop":
                cross = []
            assert len(ps["waits"][ins["id"]]) == len(cross)
            expect_waits += len(cross)
            for d, slot in zip(cross, ps["waits"][ins["id"]]):
                key = (d, rank_of(ins["id"]))
                assert seen.setdefault(key, slot) == slot
                assert [rank_of(ins["id"]), slot] in ps["signals"][d]
        for r in range(world):
            used = sorted({s for (d, rr), s in seen.items() if rr == r})
            assert used == list(range(ps["slots"][r]))
        if nl > 1 and world > 1:
            assert expect_waits > 0


def test_collectives_become_single_fused_box_per_member():
    g = golden_cases.load("adapt_v_to_d4")
    desc = pb.describe(g["plan"])
    coll = [i for i in desc["instrs"] if ":" in i["label"]]
    assert len(coll) == 4
    for i in coll:
        assert i["kind"] == "box" and i["stream"] == 1
        # reduce-scatter: each member's slice sums the 4 partial pieces
        assert all(len(c["terms"]) == 4 and all(t["add"] for t in c["terms"]) for c in i["cells"])
        assert len({b for b in i["in"]}) == 4


def test_allgather_cells_copy_each_slice():
    g = golden_cases.load("adapt_d_to_r4")
    desc = pb.describe(g["plan"])
    coll = [i for i in desc["instrs"] if i["label"].startswith("all-gather")]
    assert coll
    for i in coll:
        assert len(i["cells"]) == 4
        assert all(len(c["terms"]) == 1 and not c["terms"][0]["add"] for c in i["cells"])


@pytest.mark.parametrize("name", golden_cases.names())
def test_strict_value_mode_matches_reference_rule(name):
    """With the reference rule (STRICT_VALUE) the V(m*v)->V(v) extension is
    off. Plans the reference executor runs lower identically in both modes;
    the fact-6 plans (reference run_plan throws) fail to lower strictly with
    the reference's InternalError and lower with the extension."""
    g = golden_cases.load(name)
    if g["meta"]["reference_run_plan"] == "ok":
        assert pb.describe(g["plan"])["instrs"] == pb.describe(g["plan"], strict_value=True)["instrs"]
    else:
        with pytest.raises(pb.InternalError, match="not fully covered"):
            pb.describe(g["plan"], strict_value=True)
        desc = pb.describe(g["plan"])
        # the chained reduce-scatters sum value sub-parts
        assert any(t["add"] for i in desc["instrs"] for c in i["cells"] for t in c["terms"])


def _two_row_parallel_doc(T=256, H=128):
    """Two independent row-parallel (value-split) GEMMs of one shape whose
    all-reduced outputs meet in an add (group_gemms must not merge
    reduce-scatter GEMMs)."""
    pts = [{"id": 0, "shape": [T, H], "elem_size": 2, "kind": "activation"},
           {"id": 1, "shape": [H, H], "elem_size": 2, "kind": "weight"},
           {"id": 2, "shape": [H, H], "elem_size": 2, "kind": "weight"},
           {"id": 3, "shape": [T, H], "elem_size": 2, "kind": "activation"},
           {"id": 4, "shape": [T, H], "elem_size": 2, "kind": "activation"},
           {"id": 5, "shape": [T, H], "elem_size": 2, "kind": "activation"}]
    ops = [{"id": "rowa", "kind": "matmul", "inputs": [0, 1], "outputs": [3], "direction": "forward",
            "flops": 2.0 * T * H * H},
           {"id": "rowb", "kind": "matmul", "inputs": [0, 2], "outputs": [4], "direction": "forward",
            "flops": 2.0 * T * H * H},
           {"id": "res", "kind": "add", "inputs": [3, 4], "outputs": [5], "direction": "forward", "flops": T * H}]
    return json.dumps({"ptensors": pts, "ops": ops})


@pytest.mark.skipif(not refpy.available(), reason="oracle/_ref not built")
def test_reduce_scatter_gemms_are_never_grouped():
    doc = _two_row_parallel_doc()
    plan = refpy.compile_plan(doc, strategy="megatron_tp", devices=2)
    desc = pb.describe(plan, lane_rank=[0, 1], flags=pb.PEER_MEMORY)
    scat = [i for i in desc["instrs"] if i["kind"] == "gemm" and i["scatter"]]
    assert len(scat) == 4  # two GEMMs x two lanes, each its own launch
    for i in scat:
        assert i["group"] == 1 and len(i["out"]) == i["scatter"]
    inputs = refpy.random_integer_inputs(doc, 3, 1)
    out = run_program(desc, json.loads(plan), inputs)
    ok, msg = pb.compare_outputs(refpy.run_reference(doc, inputs), out, 2e-2, normwise=True)
    assert ok, msg


def test_fusion_requires_bf16_operands():
    """an elementwise consumer with an fp32 operand is not fused
    into a bf16 GEMM epilogue (which reads every operand as bf16)."""
    from plan_builder import matmul_add_plan

    plan, _ = matmul_add_plan(256, 256, 256)
    p = json.loads(plan)
    assert any(f for i in pb.describe(plan)["instrs"] for f in i["fused"])
    for pt in p["ptensors"]:
        if pt["id"] == 3:
            pt["elem_size"] = 4
    desc = pb.describe(json.dumps(p))
    assert not any(f for i in desc["instrs"] for f in i["fused"])


def test_malformed_plan_is_schema_error():
    with pytest.raises(pb.SchemaError):
        pb.describe("{not json")
    with pytest.raises(pb.SchemaError):
        pb.describe(json.dumps({"ptensors": []}))
    plan = json.loads(golden_cases.load("mlp_dp2")["plan"])
    plan["ops"][0]["kind"] = "rotary-embedding"  # not a kind (softmax, attention are the schema extension, tests/test_ext.py)
    with pytest.raises(pb.SchemaError):
        pb.describe(json.dumps(plan))


def test_missing_feed_is_internal_error():
    plan = json.loads(golden_cases.load("mlp_dp2")["plan"])
    plan["feeds"] = plan["feeds"][1:]
    with pytest.raises(pb.InternalError, match="no feed"):
        pb.describe(json.dumps(plan))


def test_crossed_recvs_deadlock_like_run_plan():
    # test_simulate.cpp:188-221 style negative control: swap the order of a
    # lane's recvs against its peer's sends -> pairing deadlock.
    g = golden_cases.load("mlp_dp2_naive")
    plan = json.loads(g["plan"])
    # make lane 0 wait for a channel that lane 1 only sends after waiting on lane 0
    recvs = {}
    for lane in plan["lanes"]:
        for t in lane["tasks"]:
            if t["kind"] == "recv":
                recvs.setdefault(lane["device"], []).append(t)
    lane0 = plan["lanes"][0]["tasks"]
    lane1 = plan["lanes"][1]["tasks"]
    first_recv0 = next(i for i, t in enumerate(lane0) if t["kind"] == "recv")
    first_recv1 = next(i for i, t in enumerate(lane1) if t["kind"] == "recv")
    lane0.insert(0, lane0.pop(first_recv0))
    lane1.insert(0, lane1.pop(first_recv1))
    with pytest.raises(pb.InternalError, match="deadlock"):
        pb.describe(json.dumps(plan))
    with pytest.raises(po.InternalError, match="deadlock"):
        po.run_plan(json.dumps(plan), g["inputs"])


def test_corrupted_channels_are_detected():
    # test_refexec.cpp:142-181: swap two same-shaped value-part sends.
    g = golden_cases.load("mlp_dp2_naive")
    plan = json.loads(g["plan"])
    vts = {v["id"]: v for v in plan["vtensors"]}
    sends = [o for o in plan["ops"] if o["kind"] == "send" and vts[o["inputs"][0]]["value"][1] > 1]
    assert len(sends) >= 2
    s0, s1 = sends[0], sends[1]
    s0["channel"], s1["channel"] = s1["channel"], s0["channel"]
    for lane in plan["lanes"]:
        for t in lane["tasks"]:
            if t["op"] == s0["id"]:
                t["channel"] = s0["channel"]
            if t["op"] == s1["id"]:
                t["channel"] = s1["channel"]
    text = json.dumps(plan)
    try:
        out = run_program(pb.describe(text), plan, g["inputs"])
        assert not po.compare_outputs(g["expected"], out)[0]
    except pb.PlancError:
        pass


def test_unsupported_elem_size_is_usage_error():
    plan = json.loads(golden_cases.load("mlp_dp2")["plan"])
    plan["ptensors"][0]["elem_size"] = 8
    with pytest.raises(pb.UsageError):
        pb.describe(json.dumps(plan))


def test_partial_value_graph_input_is_usage_error():
    plan = json.loads(golden_cases.load("reduce_sum")["plan"])
    for v in plan["vtensors"]:
        if v["ptensor"] == 0:
            v["value"] = [0, 2]
    with pytest.raises(pb.UsageError, match="partial value"):
        pb.describe(json.dumps(plan))


def test_accounting_matches_masks():
    g = golden_cases.load("gpt_block_tp2")
    desc = pb.describe(g["plan"])
    flops = sum(i["flops"] for i in desc["instrs"] if i["kind"] == "gemm")
    T, H = 16, 8
    assert flops == pytest.approx(3 * 22 * T * H * H)  # fwd + 2x bwd GEMMs of the block


@pytest.mark.parametrize("m,n,k,ta", [(8192, 2048, 2048, False), (512, 512, 16384, True), (256, 256, 8192, True),
                                      (2048, 2048, 8192, True), (1000, 1000, 3000, False), (136, 264, 1000, False)])
@pytest.mark.parametrize("sk_mode", ["1", "2"])
def test_gemm_schedule_covers_every_k_block_once(m, n, k, ta, sk_mode, monkeypatch):
    """The tcgen05 GEMM's work split (host-only): data-parallel tiles plus
    stream-K ranges cover every (tile, k-block) exactly once, and every
    shared tile's segments come from consecutive CTAs (the fixed reduction
    order)."""
    monkeypatch.setenv("PLANC_B200_STREAMK", sk_mode)
    monkeypatch.setenv("PLANC_B200_SPLITK", "1" if sk_mode == "1" else "0")
    sms = 148
    sc = pb.gemm_schedule(m, n, k, ta, False, sms=sms)
    bn = sc["tile_n"]
    tiles = -(-m // 128) * -(-n // bn)
    num_k = -(-k // 64)
    assert 0 < sc["grid"] <= sms * sc["ctas_per_sm"]
    if sc["ctas_per_sm"] == 2:  # short-k variant: data-parallel only, <= 128-wide tiles, <= 16 k-blocks
        assert sc["tile_n"] <= 128 and num_k <= 16 and sc["sk_ctas"] == 0 and sc["splits"] == 0
        bn = sc["tile_n"]
        tiles = -(-m // 128) * -(-n // bn)
    seen = {}
    if sc["half_items"]:
        # half-width tail: whole tiles, then both halves of every remaining tile
        assert sc["sk_ctas"] == 0 and sc["half_items"] == 2 * (tiles - sc["dp_tiles"])
        assert sc["dp_tiles"] % sms == 0 and sc["half_items"] <= sms
        halves = {}
        for x in range(sc["dp_tiles"] + sc["half_items"]):
            if x >= sc["dp_tiles"]:
                h = x - sc["dp_tiles"]
                halves.setdefault(sc["dp_tiles"] + h // 2, set()).add(h % 2)
        assert all(v == {0, 1} for v in halves.values()) and len(halves) == tiles - sc["dp_tiles"]
        return
    for b in range(sc["grid"]):
        for t in range(b, sc["dp_tiles"], sc["grid"]):
            for kb in range(num_k):
                seen.setdefault((t, kb), []).append(b)
    if sc["splits"] > 1:
        # split-K: item (tile t, split s) = k-blocks [s*K/S, (s+1)*K/S); no whole tiles
        seen = {}
        S = sc["splits"]
        assert sc["grid"] == tiles * S and sc["ws_bytes"] >= S * tiles * 128 * bn * 4
        for x in range(tiles * S):
            t, s = divmod(x, S)
            for kb in range(s * num_k // S, (s + 1) * num_k // S):
                seen.setdefault((t, kb), []).append(x)
            assert (s * num_k // S * S + num_k - 1) // num_k == s  # the epilogue's split index
        assert sorted(seen) == [(t, kb) for t in range(tiles) for kb in range(num_k)]
        assert all(len(v) == 1 for v in seen.values())
        return
    if sc["sk_ctas"]:
        assert sc["ws_bytes"] > 0 and sc["dp_tiles"] % sms == 0
        iters = (tiles - sc["dp_tiles"]) * num_k
        lo = [b * iters // sc["sk_ctas"] for b in range(sc["sk_ctas"] + 1)]
        for b in range(sc["sk_ctas"]):
            for x in range(lo[b], lo[b + 1]):
                seen.setdefault((sc["dp_tiles"] + x // num_k, x % num_k), []).append(b)
    else:
        assert sc["ws_bytes"] == 0 and sc["dp_tiles"] == tiles
    assert sorted(seen) == [(t, kb) for t in range(tiles) for kb in range(num_k)]
    assert all(len(v) == 1 for v in seen.values())
    for t in range(sc["dp_tiles"], tiles):
        owners = sorted({seen[(t, kb)][0] for kb in range(num_k)})
        assert owners == list(range(owners[0], owners[-1] + 1))
    if sk_mode == "2" and tiles % sms:
        assert sc["sk_ctas"] > 0 or (tiles - sc["dp_tiles"]) * num_k < 8


def test_opt_in_gelu_epilogue_fusion():
    """The FUSE_ACT flag moves GELU into its GEMM's epilogue (fused op
    ew 3); the lowered program still computes the same values."""
    g = golden_cases.load("ext_block_fwd_tp2_mma")
    plan = json.loads(g["plan"])
    base = run_program(pb.describe(g["plan"]), plan, g["inputs"])
    assert not any(f["ew"] == 3 for i in pb.describe(g["plan"])["instrs"] for f in i["fused"])
    desc = pb.describe(g["plan"], flags=pb.FUSE_ACT)
    assert any(f["ew"] == 3 for i in desc["instrs"] for f in i["fused"])
    out = run_program(desc, plan, g["inputs"])
    ok, msg = pb.compare_outputs(base, out, 0.0, normwise=True)
    assert ok, msg


def _happens_before_clocks(desc, ns=4):
    """Vector clocks of the executed step, recomputed here from the lowered
    program: stream FIFO order (describe's stream assignment) plus every
    dependency edge. done[i][s] = last sequence number of stream s complete
    when instruction i completes."""
    instrs = desc["instrs"]
    streams = desc["memory_plan"]["streams"]
    S = desc["num_lanes"] * ns
    sid = {}
    seq = {}
    count = [0] * S
    last = [-1] * S
    prev = {}
    for i in desc["issue_order"]:
        s = instrs[i]["lane"] * ns + streams[i]
        sid[i], seq[i], prev[i] = s, count[s], last[s]
        count[s] += 1
        last[s] = i
    done = np.full((len(instrs), S), -1, dtype=np.int64)
    for i in desc["issue_order"]:
        v = np.full(S, -1, dtype=np.int64)
        for d in instrs[i]["deps"] + ([prev[i]] if prev[i] >= 0 else []):
            v = np.maximum(v, done[d])
        v[sid[i]] = seq[i]
        done[i] = v
    return sid, seq, done, prev


def _uses(ins):
    for b in ins["in"]:
        yield b, False
    for b in ins["out"]:
        yield b, True
    for c in ins["cells"]:
        for t in c["terms"]:
            yield t["buf"], False
    for f in ins["fused"]:
        for b in f["in"]:
            yield b, False
        yield f["out"], True


@pytest.mark.parametrize("name", ["c5_3f1b_dap", "c4_coshard4_dp8", "c2_tp1"])
def test_timed_memory_plan_never_overlaps_live_buffers(name):
    """REUSE_MEMORY (the plan's free tasks made real): two buffers sharing
    arena bytes must be ordered — every use of one happens before every write
    of the other, by dependency edges and stream order — and terminal
    results / graph inputs are never overwritten. Checked independently of
    the C++ planner from the lowered program."""
    import bench

    plan, _ = bench.load_plan(name)
    desc = pb.describe(plan, flags=pb.REUSE_MEMORY)
    mp = desc["memory_plan"]
    assert mp["reused"] > 0 and mp["bytes_after"] < mp["bytes_before"]
    sid, seq, done, prev = _happens_before_clocks(desc)
    uses, writes = {}, {}
    for ins in desc["instrs"]:
        for b, w in _uses(ins):
            uses.setdefault(b, []).append(ins["id"])
            if w:
                writes.setdefault(b, []).append(ins["id"])

    def start_clock(i):
        ins = desc["instrs"][i]
        v = np.full(done.shape[1], -1, dtype=np.int64)
        for d in ins["deps"] + ([prev[i]] if prev[i] >= 0 else []):
            v = np.maximum(v, done[d])
        return v

    def before(x, y):  # every use of x completes before every write of y starts
        clocks = [start_clock(w) for w in writes.get(y, [])]
        return all(c[sid[u]] >= seq[u] for u in uses.get(x, []) for c in clocks)

    bufs = desc["buffers"]
    off = mp["offset"]
    by_lane = {}
    for b in bufs:
        if b["dead"] or b["id"] not in uses:
            continue
        by_lane.setdefault(b["lane"], []).append(b["id"])
    checked = 0
    for lane, ids in by_lane.items():
        ids.sort(key=lambda b: off[b])
        for i, x in enumerate(ids):
            xend = off[x] + bufs[x]["bytes"]
            for y in ids[i + 1:]:
                if off[y] >= xend:
                    break
                checked += 1
                assert before(x, y) or before(y, x), (name, x, y)
                assert not (bufs[x]["graph_input"] or bufs[y]["graph_input"])
    assert checked >= mp["reused"] // 2
    # results the step hands back keep their bytes
    consumed = {v["ptensor"] for o in json.loads(plan)["ops"] for vid in o["inputs"]
                for v in [next(vv for vv in json.loads(plan)["vtensors"] if vv["id"] == vid)]} if name == "c2_tp1" else None
    if consumed is not None:
        for pt, pieces in desc["outputs"]:
            if pt not in consumed:
                assert not any(mp["overwritten"][b] for b in pieces)


def test_box_elementwise_fusion_lowering():
    """C5's all-to-all -> max gate: the max runs as fold terms of the
    all-to-all's box (operand order kept, the adapter output buffer dead),
    and the lowered program still reproduces the reference bit for bit."""
    g = golden_cases.load("c5_3f1b_dap")
    fused = pb.describe(g["plan"])
    plain = pb.describe(g["plan"], flags=pb.NO_BOX_EW)
    n_ew = lambda d: sum(1 for i in d["instrs"] if i["kind"] == "ew")  # noqa: E731
    boxes = [i for i in fused["instrs"] if i["kind"] == "box" and
             any(t["fold"] >= 0 for c in i["cells"] for t in c["terms"])]
    assert boxes and n_ew(fused) == n_ew(plain) - len(boxes)
    for b in boxes:
        for c in b["cells"]:
            assert c["terms"][0]["fold"] == -1 and all(t["fold"] >= 0 for t in c["terms"][1:])
    dead = {b["id"] for b in fused["buffers"] if b.get("dead")}
    assert dead
    for ins in fused["instrs"]:
        assert not dead & set(ins["in"]) and not dead & set(ins["out"])
    a = run_program(fused, json.loads(g["plan"]), g["inputs"])
    b = run_program(plain, json.loads(g["plan"]), g["inputs"])
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    ok, msg = pb.compare_outputs(g["expected"], a, 0.0)
    assert ok, msg


def test_column_gather_lowering():
    """GATHER_COLS: concats of column blocks along K feeding tensor-core GEMMs
    become column-gathered operands (pieces of 64k stored columns, the concat
    buffer dead); the lowered program still reproduces the reference."""
    g = golden_cases.load("c5_3f1b_dap_mma")
    desc = pb.describe(g["plan"], flags=pb.GATHER_COLS)
    cols = [i for i in desc["instrs"] if i["kind"] == "gemm" and any(x["cols"] for x in i["gather"])]
    assert cols
    for i in cols:
        for j, x in enumerate(i["gather"]):
            if x["cols"]:
                assert x["cols"] % 64 == 0 and x["rows"] == 0 and len(x["pieces"]) >= 2
                assert (not i["ta"]) if j == 0 else i["tb"]  # K is the stored column axis
    assert not any(any(x["cols"] for x in i["gather"]) for i in pb.describe(g["plan"])["instrs"]
                   if i["kind"] == "gemm")  # opt-in
    out = run_program(desc, json.loads(g["plan"]), g["inputs"])
    tol = 0.0 if g["meta"].get("max_abs", 0) < 2.0 ** 53 else 1e-12
    ok, msg = pb.compare_outputs(g["expected"], out, tol, normwise=True)
    assert ok, msg
