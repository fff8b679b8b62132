"""TEST INFRASTRUCTURE — numpy restatement of the reference plan executor.

This is the CHECKER, never the product: only tests/, ``__graft_entry__.smoke()``
and bench.py's ``cpu_baseline`` leg may import it. It restates, in float64
numpy, the reference's CPU executor ``planc::run_plan`` and its helpers:

* ``reconstruct``      — reference proj/src/refexec.cpp:102-140
* ``eval_compute``     — refexec.cpp:142-257 (matmul 142-168, elementwise
                         178-193, reduce-sum 194-215, embedding 216-250,
                         identity 251-252)
* ``run_plan``         — refexec.cpp:361-557 (lane cursor loop 483-522,
                         collective rendezvous 459-481, reassembly 532-556)
* ``compare_outputs``  — refexec.cpp:604-631

Two deliberate extensions over the reference, both
off by default so the restatement is bit-compatible with the reference:

* ``vv=True``: a piece whose value_count is a multiple m of the target's
  contributes (summed) to target value index vi when piece_vi // m == vi —
  the multi-step V(4)->V(2)->V(1) reductions the reference throws on
  (slot arithmetic of rvd.cpp:226-251).
* ``return_vtensors=True`` additionally returns every produced vTensor's
  value (the reference only returns reassembled pTensors).

Parity pinning: tests/test_oracle.py checks this module against the compiled
reference (oracle/_ref) and the golden fixtures in tests/golden/.

Schema extension (NOT part of the reference, whose
document.cpp:43-53 rejects these kinds): row-wise sub-operators of a
transformer block over the last axis, in segments of ``segment`` elements
(default: the whole last axis) — ``softmax`` / ``softmax-grad`` (per
attention head when segment = head width), ``layernorm`` / ``layernorm-grad``
(no affine, ``eps`` default 1e-5, population variance) and elementwise
``gelu`` / ``gelu-grad`` (erf form). ``eval_ext`` restates them in float64;
``run_graph`` evaluates a graph document op by op (the run_reference shape,
refexec.cpp:264-350) for the extended vocabulary. Parity of these kinds is
pinned against torch's float64 implementations (tests/test_ext_oracle.py),
not against the reference, which has none.
"""
from __future__ import annotations

import json

import numpy as np


class UsageError(RuntimeError):
    pass


class InternalError(RuntimeError):
    pass


def _region_intersect(a, b):
    out = []
    for (alo, ahi), (blo, bhi) in zip(a, b):
        lo, hi = max(alo, blo), min(ahi, bhi)
        if lo >= hi:
            return None
        out.append((lo, hi))
    return out


def _vol(region):
    v = 1
    for lo, hi in region:
        v *= hi - lo
    return v


def _sl(region, origin):
    return tuple(slice(lo - o[0], hi - o[0]) for (lo, hi), o in zip(region, origin))


def reconstruct(target, pieces, ctx="", vv=False):
    """refexec.cpp:102-140. target/pieces masks are dicts with region, vi, vc.

    With ``vv``, value sub-parts (vc = m * target vc) are summed only into
    elements no exact-match piece covers: where the reference's own copy
    rule (refexec.cpp:110-112) applies, its result stands and the sub-parts
    are skipped as in refexec.cpp:115-117, whatever the piece order."""
    treg = target["region"]
    out = np.zeros([hi - lo for lo, hi in treg], dtype=np.float64)
    sub = np.zeros_like(out) if vv else None
    copied = np.zeros(out.shape, dtype=bool) if vv else None
    touched = 0
    for mask, value in pieces:
        part = False
        if mask["vc"] == target["vc"] and mask["vi"] == target["vi"]:
            copy = True
        elif target["vc"] == 1 and mask["vc"] > 1:
            copy = False
        elif (vv and mask["vc"] > target["vc"] and mask["vc"] % target["vc"] == 0
              and mask["vi"] // (mask["vc"] // target["vc"]) == target["vi"]):
            copy, part = False, True
        else:
            continue
        ov = _region_intersect(mask["region"], treg)
        if ov is None:
            continue
        dst = _sl(ov, treg)
        src = value[_sl(ov, mask["region"])]
        if part:
            sub[dst] += src
        elif copy:
            out[dst] = src
            if vv:
                copied[dst] = True
        else:
            out[dst] += src
        touched += _vol(ov)
    if touched < _vol(treg):
        raise InternalError(f"reconstruct: region {treg} not fully covered ({ctx})")
    if vv:
        out = np.where(copied, out, out + sub)
    return out


def eval_compute(op, ins, in_masks, out_masks):
    """refexec.cpp:172-257."""
    kind = op["kind"]
    if kind == "matmul":
        a, b = ins[0], ins[1]
        a = a.T if op.get("transpose_a") else a
        b = b.T if op.get("transpose_b") else b
        if a.shape[1] != b.shape[0]:
            raise InternalError("matmul operand inner extents differ in " + op["id"])
        return [a @ b]
    if kind in ("add", "mul", "max"):
        out = ins[0].copy()
        for x in ins[1:]:
            if x.shape != out.shape:
                raise InternalError("elementwise shape mismatch in " + op["id"])
            if kind == "add":
                out = out + x
            elif kind == "mul":
                out = out * x
            else:
                out = np.maximum(out, x)
        return [out]
    if kind == "reduce-sum":
        axis = op.get("axis", 0)
        out = ins[0].sum(axis=axis)
        if out.ndim == 0:
            out = out.reshape(1)
        return [out]
    if kind == "embedding-lookup":
        idx, table = ins[0], ins[1]
        lo = in_masks[1]["region"][0][0]
        rows, h = table.shape
        ids = idx.astype(np.int64)
        out = np.zeros((idx.shape[0], h))
        ok = (ids >= lo) & (ids < lo + rows)
        out[ok] = table[ids[ok] - lo]
        return [out]
    if kind == "embedding-grad":
        idx, gout = ins[0], ins[1]
        (lo, hi) = out_masks[0]["region"][0]
        rows = hi - lo
        out = np.zeros((rows, gout.shape[1]))
        ids = idx.astype(np.int64)
        for j in range(ids.shape[0]):
            if lo <= ids[j] < lo + rows:
                out[ids[j] - lo] += gout[j]
        return [out]
    if kind == "identity":
        return [ins[0].copy()]
    if kind == "attention":
        return [attention(ins[0], ins[1], ins[2], op.get("head_dim", 0), op.get("seq", 0), op.get("causal", False),
                          in_masks)]
    if kind == "attention-grad":
        return [attention_grad(*ins[:5], op.get("head_dim", 0), op.get("seq", 0), op.get("causal", False),
                               op.get("wrt", "q"), in_masks)]
    if kind in EXT_KINDS:
        return [eval_ext(kind, ins, op.get("segment", 0), op.get("eps", 1e-5), in_masks)]
    raise UsageError(f"refexec: unsupported op kind {kind} ({op['id']})")


EXT_KINDS = ("softmax", "softmax-grad", "layernorm", "layernorm-grad", "gelu", "gelu-grad")


def attention(q, k, v, head_dim, seq, causal=False, in_masks=None):
    """Schema extension (not in the reference): O = softmax(Q·Kᵀ/sqrt(d) [+
    causal mask])·V per sequence of ``seq`` rows and head of ``head_dim``
    columns of the [T, D] operands, in float64. The executor's rule for a
    piece: whole sequences and whole heads, Q/K/V/O on the same region."""
    q, k, v = (np.asarray(x, dtype=np.float64) for x in (q, k, v))
    T, D = q.shape
    if head_dim <= 0 or seq <= 0 or T % seq or D % head_dim:
        raise UsageError(f"attention: piece [{T}, {D}] does not hold whole sequences of {seq} / heads of {head_dim}")
    if in_masks is not None:
        r = in_masks[0]["region"]
        if r[0][0] % seq or r[1][0] % head_dim or any(m["region"] != r for m in in_masks):
            raise UsageError("attention: pieces not aligned to whole sequences / heads or not the same region")
    nb, nh = T // seq, D // head_dim
    qs = q.reshape(nb, seq, nh, head_dim).transpose(0, 2, 1, 3)
    ks = k.reshape(nb, seq, nh, head_dim).transpose(0, 2, 1, 3)
    vs = v.reshape(nb, seq, nh, head_dim).transpose(0, 2, 1, 3)
    s = qs @ ks.transpose(0, 1, 3, 2) / np.sqrt(head_dim)
    if causal:
        s = np.where(np.tril(np.ones((seq, seq), dtype=bool)), s, -np.inf)
    p = np.exp(s - s.max(axis=-1, keepdims=True))
    p /= p.sum(axis=-1, keepdims=True)
    return (p @ vs).transpose(0, 2, 1, 3).reshape(T, D)


def attention_grad(q, k, v, o, do, head_dim, seq, causal=False, wrt="q", in_masks=None):
    """Gradient of attention (schema extension) with respect to Q, K or V,
    given the forward output O and its incoming gradient dO, in float64:
    P = softmax(Q·Kᵀ/sqrt(d) [causal]); D = rowsum(dO ∘ O);
    dV = Pᵀ·dO; dS = P ∘ (dO·Vᵀ − D); dQ = dS·K/sqrt(d); dK = dSᵀ·Q/sqrt(d).
    (D uses the supplied O, as the executor's kernels do.)"""
    q, k, v, o, do = (np.asarray(x, dtype=np.float64) for x in (q, k, v, o, do))
    T, D = q.shape
    if head_dim <= 0 or seq <= 0 or T % seq or D % head_dim:
        raise UsageError(f"attention-grad: piece [{T}, {D}] does not hold whole sequences / heads")
    if in_masks is not None:
        r = in_masks[0]["region"]
        if r[0][0] % seq or r[1][0] % head_dim or any(m["region"] != r for m in in_masks):
            raise UsageError("attention-grad: pieces not aligned to whole sequences / heads or not the same region")
    nb, nh = T // seq, D // head_dim
    sh = lambda x: x.reshape(nb, seq, nh, head_dim).transpose(0, 2, 1, 3)  # noqa: E731
    qs, ks, vs, os_, dos = sh(q), sh(k), sh(v), sh(o), sh(do)
    sc = 1.0 / np.sqrt(head_dim)
    s = qs @ ks.transpose(0, 1, 3, 2) * sc
    if causal:
        s = np.where(np.tril(np.ones((seq, seq), dtype=bool)), s, -np.inf)
    p = np.exp(s - s.max(axis=-1, keepdims=True))
    p /= p.sum(axis=-1, keepdims=True)
    if wrt == "v":
        g = p.transpose(0, 1, 3, 2) @ dos
    else:
        dd = (dos * os_).sum(axis=-1, keepdims=True)
        ds = p * (dos @ vs.transpose(0, 1, 3, 2) - dd)
        g = (ds @ ks if wrt == "q" else ds.transpose(0, 1, 3, 2) @ qs) * sc
    return g.transpose(0, 2, 1, 3).reshape(T, D)


def _erf(x):
    try:
        from scipy.special import erf

        return erf(x)
    except ImportError:  # pragma: no cover
        import math

        return np.vectorize(math.erf)(x)


def eval_ext(kind, ins, segment=0, eps=1e-5, in_masks=None):
    """Extended kinds in float64. Row-wise kinds work on segments of
    ``segment`` elements of the last axis (0 = the whole last axis); a piece
    must hold whole segments (its last-axis region aligned to the segment)."""
    x = np.asarray(ins[0], dtype=np.float64)
    if kind == "gelu":
        return 0.5 * x * (1.0 + _erf(x / np.sqrt(2.0)))
    if kind == "gelu-grad":  # ins = (x, dy)
        dy = np.asarray(ins[1], dtype=np.float64)
        cdf = 0.5 * (1.0 + _erf(x / np.sqrt(2.0)))
        pdf = np.exp(-0.5 * x * x) / np.sqrt(2.0 * np.pi)
        return dy * (cdf + x * pdf)
    n = x.shape[-1]
    seg = segment or n
    if n % seg != 0:
        raise UsageError(f"{kind}: last-axis extent {n} is not a multiple of the segment {seg}")
    if in_masks is not None and segment and in_masks[0]["region"][-1][0] % seg != 0:
        raise UsageError(f"{kind}: piece does not start on a segment boundary")
    shp = x.shape
    xs = x.reshape(-1, seg)
    if kind == "softmax":
        e = np.exp(xs - xs.max(axis=1, keepdims=True))
        return (e / e.sum(axis=1, keepdims=True)).reshape(shp)
    if kind == "softmax-grad":  # ins = (y, dy)
        dy = np.asarray(ins[1], dtype=np.float64).reshape(-1, seg)
        return (xs * (dy - (dy * xs).sum(axis=1, keepdims=True))).reshape(shp)
    mean = xs.mean(axis=1, keepdims=True)
    var = ((xs - mean) ** 2).mean(axis=1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    xhat = (xs - mean) * rstd
    if kind == "layernorm":
        return xhat.reshape(shp)
    if kind == "layernorm-grad":  # ins = (x, dy)
        dy = np.asarray(ins[1], dtype=np.float64).reshape(-1, seg)
        return (rstd * (dy - dy.mean(axis=1, keepdims=True) - xhat * (dy * xhat).mean(axis=1, keepdims=True))
                ).reshape(shp)
    raise UsageError(f"unsupported extended kind {kind}")


def bf16_round(x):
    """Round-to-nearest-even to bfloat16, returned as float64."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16 << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def run_graph(doc, inputs, round_bf16=False):
    """Graph-level evaluation (the shape of run_reference, refexec.cpp:264-350)
    for documents using the extended kinds: every op in document order on
    whole pTensors; returns every produced pTensor. ``round_bf16``: outputs of
    2-byte pTensors are rounded to bfloat16 (the executor's storage points),
    each op computing in float64 from rounded operands."""
    g = json.loads(doc) if isinstance(doc, str) else doc
    vals = {int(k): np.asarray(v, dtype=np.float64) for k, v in inputs.items()}
    shapes = {p["id"]: tuple(p["shape"]) for p in g["ptensors"]}
    half = {p["id"] for p in g["ptensors"] if p["elem_size"] == 2}
    out = {}
    for op in g["ops"]:
        attrs = dict(op.get("attrs", {}))
        o = dict(op, **attrs)
        ins = [vals[i] for i in op["inputs"]]
        masks = [{"region": [[0, e] for e in shapes[i]], "value": [0, 1]} for i in op["inputs"]]
        omasks = [{"region": [[0, e] for e in shapes[i]], "value": [0, 1]} for i in op["outputs"]]
        res = eval_compute(o, ins, masks, omasks)
        for pid, v in zip(op["outputs"], res):
            vals[pid] = v.reshape(shapes[pid])
            if round_bf16 and pid in half:
                vals[pid] = bf16_round(vals[pid])
            out[pid] = vals[pid]
    return out


class Plan:
    """Parsed plan.json (wire form of ExecutionPlan, simulate.cpp:492-602)."""

    def __init__(self, doc):
        j = json.loads(doc) if isinstance(doc, str) else doc
        self.ptensors = {p["id"]: p for p in j["ptensors"]}
        self.vtensors = {}
        for v in j["vtensors"]:
            self.vtensors[v["id"]] = {
                "id": v["id"], "pt": v["ptensor"],
                "region": [tuple(iv) for iv in v["region"]],
                "vi": v["value"][0], "vc": v["value"][1], "owner": v["owner"],
            }
        self.ops = j["ops"]
        self.op = {o["id"]: o for o in self.ops}
        self.assignment = j["assignment"]
        self.feeds = {c: p for c, p in j["feeds"]}
        self.coll_groups = {g["id"]: g for g in j["coll_groups"]}
        self.lanes = j["lanes"]
        self.sync_edges = j.get("sync_edges", [])
        produced = set()
        for o in self.ops:
            for v in o["outputs"]:
                produced.add(self.vtensors[v]["pt"])
        self.graph_inputs = {p for p in self.ptensors if p not in produced}


class InexactBf16(RuntimeError):
    """round_bf16 emulation left the range where fp32 accumulation is exact."""


def run_plan(plan, inputs, vv=False, return_vtensors=False, round_bf16=False):
    """refexec.cpp:361-557 restated. ``plan`` is a Plan or plan.json text.

    ``round_bf16``: every vTensor of a 2-byte pTensor is rounded to bfloat16
    where the B200 executor stores it (op outputs, every reconstruct / adapter
    output, graph-input placement); the final reassembly of produced pTensors
    stays in float64 (the executor reassembles on the host in double,
    refexec.cpp:532-556). On integer inputs every stored bf16 value is an
    integer, so when every matmul's |A|·|B| stays below 2^24 each fp32
    accumulation on the GPU is exact in ANY summation order and the
    executor's bf16 results must equal this emulation bit for bit; the run
    raises ``InexactBf16`` otherwise (the golden generator then rejects the
    case)."""
    if not isinstance(plan, Plan):
        plan = Plan(plan)
    g = plan
    vt_values = {}
    channel_values = {}
    half = {p for p, d in g.ptensors.items() if d["elem_size"] == 2} if round_bf16 else set()

    def store(v, val):
        if g.vtensors[v]["pt"] in half:
            if val.size and (np.abs(val).max() >= 2.0 ** 24 or not np.all(val == np.round(val))):
                raise InexactBf16(f"vtensor {v}: value outside the exact fp32 integer range")
            val = bf16_round(val)
        vt_values[v] = val

    def input_value(vt):
        if vt["pt"] not in inputs:
            raise UsageError(f"run_plan: missing input tensor {vt['pt']}")
        if vt["vc"] != 1:
            raise UsageError("run_plan: graph input consumed as partial value")
        val = np.asarray(inputs[vt["pt"]], dtype=np.float64)[_sl(vt["region"], [(0, 0)] * len(vt["region"]))].copy()
        return bf16_round(val) if vt["pt"] in half else val

    def feed_ready(cvt):
        vt = g.vtensors[cvt]
        if vt["pt"] in g.graph_inputs:
            return True
        if cvt not in g.feeds:
            raise InternalError(f"run_plan: consumer view {cvt} of op {vt['owner']} has no feed")
        return g.feeds[cvt] in vt_values

    def feed_value(cvt):
        if cvt in g.feeds:
            return vt_values[g.feeds[cvt]]
        return input_value(g.vtensors[cvt])

    def mask(v):
        return g.vtensors[v]

    members = {gid: set(grp["ops"]) for gid, grp in g.coll_groups.items()}
    cursor = [0] * len(g.lanes)
    op_pos = {}
    for l, lane in enumerate(g.lanes):
        for t, task in enumerate(lane["tasks"]):
            op_pos[task["op"]] = (l, t)

    def arrived(oid):
        l, t = op_pos[oid]
        return cursor[l] == t

    def exec_op(op):
        k = op["kind"]
        if k == "free":
            return
        if k == "send":
            channel_values[op["channel"]] = feed_value(op["inputs"][0])
            return
        if k == "recv":
            store(op["outputs"][0], channel_values[op["channel"]])
            return
        if k in ("split", "concat", "reduce-assemble"):
            pieces = [(mask(v), feed_value(v)) for v in op["inputs"]]
            for out in op["outputs"]:
                store(out, reconstruct(mask(out), pieces, "op " + op["id"], vv))
            return
        ins = [feed_value(v) for v in op["inputs"]]
        if round_bf16 and k == "matmul":
            a = ins[0].T if op.get("transpose_a") else ins[0]
            b = ins[1].T if op.get("transpose_b") else ins[1]
            bound = float((np.abs(a) @ np.abs(b)).max()) if a.size and b.size else 0.0
            if bound >= 2.0 ** 24 or not (np.all(a == np.round(a)) and np.all(b == np.round(b))):
                raise InexactBf16(f"matmul {op['id']}: |A|.|B| reaches {bound} (fp32 sums not exact)")
        outs = eval_compute(op, ins, [mask(v) for v in op["inputs"]], [mask(v) for v in op["outputs"]])
        for v, val in zip(op["outputs"], outs):
            store(v, val)

    def exec_collective(grp):
        pieces = []
        for oid in grp["ops"]:
            for v in g.op[oid]["inputs"]:
                pieces.append((mask(v), feed_value(v)))
        for oid in grp["ops"]:
            for out in g.op[oid]["outputs"]:
                store(out, reconstruct(mask(out), pieces, "collective " + oid, vv))

    progress = True
    while progress:
        progress = False
        for l, lane in enumerate(g.lanes):
            tasks = lane["tasks"]
            while cursor[l] < len(tasks):
                op = g.op[tasks[cursor[l]]["op"]]
                if op["kind"] == "recv":
                    ready = op["channel"] in channel_values
                elif op["kind"] == "collective":
                    ready = all(arrived(m) for m in members[op["coll_group"]])
                    if ready:
                        ready = all(feed_ready(v) for m in members[op["coll_group"]] for v in g.op[m]["inputs"])
                else:
                    ready = all(feed_ready(v) for v in op["inputs"])
                if not ready:
                    break
                if op["kind"] == "collective":
                    exec_collective(g.coll_groups[op["coll_group"]])
                    for m in members[op["coll_group"]]:
                        ml, mt = op_pos[m]
                        cursor[ml] = mt + 1
                else:
                    exec_op(op)
                    cursor[l] += 1
                progress = True
    for l, lane in enumerate(g.lanes):
        if cursor[l] < len(lane["tasks"]):
            raise InternalError(f"run_plan: pairing deadlock at task {lane['tasks'][cursor[l]]['op']} "
                                f"on device {lane['device']}")

    outputs = {}
    piece_vts = {}
    for op in g.ops:
        if op["inserted"]:
            continue
        for v in op["outputs"]:
            piece_vts.setdefault(mask(v)["pt"], []).append(v)
    for pt_id, vts in sorted(piece_vts.items()):
        seen = set()
        pieces = []
        for v in vts:
            m = mask(v)
            key = (tuple(m["region"]), m["vi"], m["vc"])
            if key in seen:
                continue
            seen.add(key)
            pieces.append((m, vt_values[v]))
        shape = g.ptensors[pt_id]["shape"]
        full = {"region": [(0, e) for e in shape], "vi": 0, "vc": 1}
        outputs[pt_id] = reconstruct(full, pieces, f"output {pt_id}", vv)
    if return_vtensors:
        return outputs, vt_values
    return outputs


def compare_outputs(expected, actual, rel_tol=0.0):
    """refexec.cpp:604-631: |e-a| <= tol*max(1,|e|), exact when tol == 0."""
    for pid in sorted(expected):
        e = np.asarray(expected[pid])
        if pid not in actual or tuple(np.shape(actual[pid])) != tuple(e.shape):
            return False, f"mismatch on tensor {pid} (missing or shape)"
        a = np.asarray(actual[pid], dtype=np.float64)
        if rel_tol == 0.0:
            bad = e != a
        else:
            bad = np.abs(e - a) > rel_tol * np.maximum(1.0, np.abs(e))
        if bad.any():
            idx = np.unravel_index(int(np.argmax(bad)), e.shape)
            return False, (f"mismatch on tensor {pid} at {list(map(int, idx))}: "
                           f"expected {e[idx]}, got {a[idx]}")
    return True, "ok"
