"""TEST INFRASTRUCTURE — numpy interpreter of the executor's lowered program.

Runs the JSON from ``planc_b200.describe(plan)`` (buffers, instructions, box
cells, issue order) on the CPU in float64 so the host-side lowering — feeds,
placement, cell decomposition of every adapter, issue order, output
reassembly table — is checked against the reference oracle without a GPU.
It is a checker for tests only; the product never executes on the CPU.
"""
from __future__ import annotations

import numpy as np


def _strided_view(flat, offset, strides, extents):
    idx = np.full(tuple(extents), offset, dtype=np.int64)
    for d, (s, e) in enumerate(zip(strides, extents)):
        shape = [1] * len(extents)
        shape[d] = e
        idx = idx + (np.arange(e, dtype=np.int64) * s).reshape(shape)
    return idx


def buffer_shapes(desc: dict) -> dict:
    return {b["id"]: [hi - lo for lo, hi in b["region"]] for b in desc["buffers"]}


def _fold(op, v, x):
    return (v + x, v * x, np.maximum(v, x))[op]


def exec_instr(ins: dict, data: dict, shape: dict):
    """One compute / box instruction on the flat float64 buffers in ``data``
    (results are assigned to data[out]; a box writes only its cells)."""
    k = ins["kind"]
    if k == "gemm":
        gathered = ins.get("gather", [{"pieces": []}, {"pieces": []}])

        def operand(j, buf):
            # all-gather / concat -> GEMM prologue: the row pieces in order
            if gathered[j]["pieces"]:  # row pieces, or column pieces ("cols" > 0)
                axis = 1 if gathered[j].get("cols", 0) else 0
                return np.concatenate([data[p].reshape(shape[p]) for p in gathered[j]["pieces"]], axis=axis)
            return data[buf].reshape(shape[buf])

        for g in range(ins.get("group", 1)):  # grouped launch: member g = (in[2g], in[2g+1]) -> out[g]
            a = operand(0, ins["in"][2 * g])
            b = operand(1, ins["in"][2 * g + 1])
            a = a.T if ins["ta"] else a
            b = b.T if ins["tb"] else b
            c = a @ b
            if ins.get("scatter", 0):  # reduce-scatter epilogue: row slice i -> out[i]
                rp = ins["scatter_rows"]
                for i, ob in enumerate(ins["out"]):
                    data[ob] = c[i * rp:(i + 1) * rp].reshape(-1)
            else:
                data[ins["out"][g]] = c.reshape(-1)
        for f in ins.get("fused", []):  # elementwise consumers run in the GEMM epilogue
            if f["ew"] >= 3:  # GELU (3) / GELU-grad (4, operands x, dy)
                from oracle import planc_oracle as po

                xs = [data[x].reshape(-1, 1) for x in f["in"]]
                data[f["out"]] = po.eval_ext(("gelu", "gelu-grad")[f["ew"] - 3], xs, 1, 0.0).reshape(-1)
                continue
            out = data[f["in"][0]].copy()
            for x in f["in"][1:]:
                out = (out + data[x], out * data[x], np.maximum(out, data[x]))[f["ew"]]
            data[f["out"]] = out
    elif k == "ew":
        out = data[ins["in"][0]].copy()
        for x in ins["in"][1:]:
            out = (out + data[x], out * data[x], np.maximum(out, data[x]))[ins["ew"]]
        data[ins["out"][0]] = out
    elif k == "reduce":
        x = data[ins["in"][0]].reshape(ins["outer"], ins["axis_len"], ins["inner"])
        data[ins["out"][0]] = x.sum(axis=1).reshape(-1)
    elif k == "emb_lookup":
        idx = data[ins["in"][0]].astype(np.int64)
        tab = data[ins["in"][1]].reshape(ins["rows"], ins["h"])
        out = np.zeros((ins["n_idx"], ins["h"]))
        ok = (idx >= ins["lo"]) & (idx < ins["lo"] + ins["rows"])
        out[ok] = tab[idx[ok] - ins["lo"]]
        data[ins["out"][0]] = out.reshape(-1)
    elif k == "emb_grad":
        idx = data[ins["in"][0]].astype(np.int64)
        g = data[ins["in"][1]].reshape(ins["n_idx"], ins["h"])
        out = np.zeros((ins["rows"], ins["h"]))
        for j in range(ins["n_idx"]):
            if ins["lo"] <= idx[j] < ins["lo"] + ins["rows"]:
                out[idx[j] - ins["lo"]] += g[j]
        data[ins["out"][0]] = out.reshape(-1)
    elif k == "rowwise":  # schema extension: row-wise sub-operators / GELU
        from oracle import planc_oracle as po

        names = ["softmax", "softmax-grad", "layernorm", "layernorm-grad", "gelu", "gelu-grad"]
        seg = ins["seg"] if ins["row_op"] < 4 else 1
        xs = [data[b].reshape(-1, seg) for b in ins["in"]]
        data[ins["out"][0]] = po.eval_ext(names[ins["row_op"]], xs, seg, ins["eps"]).reshape(-1)
    elif k == "attention":  # schema extension: fused attention
        from oracle import planc_oracle as po

        a = ins["att"]
        ops = [data[b].reshape(a["rows"], a["cols"]) for b in ins["in"]]
        if not a.get("grad"):
            data[ins["out"][0]] = po.attention(*ops, a["head_dim"], a["seq"], a["causal"]).reshape(-1)
        else:  # attention gradient: dQ / dK / dV into grad_out[0..2]
            for w, ob in zip("qkv", a["grad_out"]):
                if ob >= 0:
                    data[ob] = po.attention_grad(*ops, a["head_dim"], a["seq"], a["causal"], w).reshape(-1)
    elif k == "box":
        ob = ins["out"][0]
        out = data[ob].copy()  # a box writes only its cells (two-phase all-reduce: two boxes per output)
        for c in ins["cells"]:
            di = _strided_view(out, c["dst_off"], c["dst_str"], c["ext"])
            v = np.zeros(di.shape)
            for t in c["terms"]:
                si = _strided_view(data[t["buf"]], t["off"], t["str"], c["ext"])
                x = data[t["buf"]][si]
                f = t.get("fold", -1)
                if f >= 0:  # an elementwise op folded into the box (fuse_box_elementwise)
                    v = _fold(f, v, x)
                else:
                    v = v + x if t["add"] else x.copy()
            out[di] = v
        data[ob] = out


def run_program(desc: dict, plan: dict, inputs: dict, owned_lanes=None, exchange=None, return_buffers=False):
    """Interpret the lowered program. With ``owned_lanes`` only those lanes'
    instructions run (one rank of the one-process-per-GPU mode) and ``xfer``
    exchange steps call ``exchange(instr, data)`` to move cross-rank pieces."""
    bufs = {b["id"]: b for b in desc["buffers"]}
    lane_ok = (lambda lane: True) if owned_lanes is None else (lambda lane: lane in owned_lanes)
    data = {}
    for b in desc["buffers"]:
        n = 1
        for lo, hi in b["region"]:
            n *= hi - lo
        data[b["id"]] = np.zeros(n)
        if b["graph_input"] and lane_ok(b["lane"]):
            x = np.asarray(inputs[b["pt"]], dtype=np.float64)
            sl = tuple(slice(lo, hi) for lo, hi in b["region"])
            data[b["id"]] = x[sl].reshape(-1).copy()
    shape = buffer_shapes(desc)
    for iid in desc["issue_order"]:
        ins = desc["instrs"][iid]
        k = ins["kind"]
        if k == "xfer":
            if exchange is not None:
                exchange(ins, data)
            elif ins.get("allreduce"):  # single process: every member gets the sum
                total = sum(data[x["src"]] for x in ins["xfers"])
                for x in ins["xfers"]:
                    data[x["dst"]] = total.copy()
            else:  # single process: the movement is a plain copy
                for x in ins["xfers"]:
                    data[x["dst"]] = data[x["src"]].copy()
            continue
        if not lane_ok(ins["lane"]):
            continue
        exec_instr(ins, data, shape)
    if return_buffers:
        return data
    return reassemble(desc, plan, data)


def reassemble(desc: dict, plan: dict, data: dict) -> dict:
    """refexec.cpp:532-556 over the (gathered) buffer values."""
    bufs = {b["id"]: b for b in desc["buffers"]}
    shape = {b["id"]: [hi - lo for lo, hi in b["region"]] for b in desc["buffers"]}
    outputs = {}
    for pt, blist in desc["outputs"]:
        full_shape = next(p["shape"] for p in plan["ptensors"] if p["id"] == pt)
        res = np.zeros(full_shape)
        # Pieces: same copy/add rule as reconstruct, in order.
        acc_set = np.zeros(full_shape, dtype=bool)
        for b in blist:
            bd = bufs[b]
            sl = tuple(slice(lo, hi) for lo, hi in bd["region"])
            piece = data[b].reshape(shape[b])
            if bd["value"][1] == 1:
                res[sl] = piece
            else:
                res[sl] = res[sl] + piece
            acc_set[sl] = True
        outputs[pt] = res
    return outputs
