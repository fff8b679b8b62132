"""Graph documents for the benchmark/parity configurations.

Written in the reference's own graph-document vocabulary (reference
proj/src/document.cpp:43-53: matmul / add / mul / max / reduce-sum /
embedding-lookup / embedding-grad / identity), so the unmodified reference
front end compiles them and the reference oracle (run_reference) checks them.
These are plan-generation inputs (test infrastructure), not product code.

Op-id prefixes drive the ``megatron_tp`` sProgram registered by
oracle/ref_capi.cpp: ``col*`` column-parallel GEMM (split output dim 1),
``row*`` row-parallel GEMM (value split -> partial sums -> all-reduce),
``tp*`` elementwise op between them (split dim 1), ``optc*`` / ``optr*``
optimizer adds split like their column / row-parallel weight, anything else
replicated.
"""
from __future__ import annotations

import json


def _pt(i, shape, kind, elem, grad_of=None):
    p = {"id": i, "shape": list(shape), "elem_size": elem, "kind": kind}
    if grad_of is not None:
        p["grad_of"] = grad_of
    return p


def _op(i, kind, ins, outs, direction, flops, attrs=None, backward_of=None):
    o = {"id": i, "kind": kind, "inputs": ins, "outputs": outs,
         "direction": direction, "flops": float(flops)}
    if attrs:
        o["attrs"] = attrs
    if backward_of:
        o["backward_of"] = backward_of
    return o


def gpt_stack_doc(layers: int, tokens: int, hidden: int, elem_size: int = 2) -> dict:
    """`layers` chained GPT blocks (train step) — SURVEY §8d config C3.

    Layer l's input is layer l-1's OUT; the gradient arriving at layer l's
    OUT is layer l+1's input gradient, so one backward chain runs through the
    stack. Every op carries its `layer`, which the pipeline sPrograms group
    into stages (reference strategies.cpp:168-276).
    """
    stride = 200
    pts, ops = [], []
    for l in range(layers):
        base = l * stride
        x_in = None if l == 0 else (l - 1) * stride + 19  # previous OUT
        g_out = None if l == layers - 1 else (l + 1) * stride + 100 + 12  # next layer's dX
        d = gpt_block_doc(tokens, hidden, elem_size, True, layer=l, prefix=f"L{l}.", base=base, x_in=x_in,
                          g_out=g_out)
        pts += d["ptensors"]
        ops += d["ops"]
    return {"ptensors": pts, "ops": ops}


def gpt_block_doc(tokens: int, hidden: int, elem_size: int = 2, train: bool = True,
                  layer: int = 0, prefix: str = "", base: int = 0, x_in=None, g_out=None) -> dict:
    """GPT-3-style transformer block proxy.

    Forward: Q = X·Wq, K = X·Wk (column-parallel), S = Q*K (attention proxy),
    O = S·Wo (row-parallel), X2 = O + X, F1 = X2·W1 [H,4H] (column-parallel),
    F = max(F1, Z) (ReLU proxy), Y = F·W2 [4H,H] (row-parallel), OUT = Y + X2.
    ``train`` adds the mlp_doc-style backward (transposed GEMMs; reference
    proj/tests/testutil.cpp:55-154) and one optimizer add per weight.
    """
    T, H, F = tokens, hidden, 4 * hidden
    e = elem_size
    b = base
    X = x_in if x_in is not None else b + 0
    ids = dict(Wq=b + 1, Wk=b + 2, Wo=b + 3, W1=b + 4, W2=b + 5, Q=b + 10, K=b + 11, S=b + 12,
               O=b + 13, X2=b + 14, F1=b + 15, Z=b + 16, Fa=b + 17, Y=b + 18, OUT=b + 19)
    pts = []
    if x_in is None:
        pts.append(_pt(X, (T, H), "activation", e))
    for w, shp in (("Wq", (H, H)), ("Wk", (H, H)), ("Wo", (H, H)), ("W1", (H, F)), ("W2", (F, H))):
        pts.append(_pt(ids[w], shp, "weight", e))
    for a, shp in (("Q", (T, H)), ("K", (T, H)), ("S", (T, H)), ("O", (T, H)), ("X2", (T, H)),
                   ("F1", (T, F)), ("Z", (T, F)), ("Fa", (T, F)), ("Y", (T, H)), ("OUT", (T, H))):
        pts.append(_pt(ids[a], shp, "activation", e))
    p = prefix
    A = {"layer": layer, "batch_dim": 0}
    mm = lambda m, n, k: 2.0 * m * n * k  # noqa: E731
    ops = [
        _op(p + "colq", "matmul", [X, ids["Wq"]], [ids["Q"]], "forward", mm(T, H, H), A),
        _op(p + "colk", "matmul", [X, ids["Wk"]], [ids["K"]], "forward", mm(T, H, H), A),
        _op(p + "tpmul", "mul", [ids["Q"], ids["K"]], [ids["S"]], "forward", T * H, A),
        _op(p + "rowo", "matmul", [ids["S"], ids["Wo"]], [ids["O"]], "forward", mm(T, H, H), A),
        _op(p + "res1", "add", [ids["O"], X], [ids["X2"]], "forward", T * H, A),
        _op(p + "colf1", "matmul", [ids["X2"], ids["W1"]], [ids["F1"]], "forward", mm(T, F, H), A),
        _op(p + "tprelu", "max", [ids["F1"], ids["Z"]], [ids["Fa"]], "forward", T * F, A),
        _op(p + "roww2", "matmul", [ids["Fa"], ids["W2"]], [ids["Y"]], "forward", mm(T, H, F), A),
        _op(p + "res2", "add", [ids["Y"], ids["X2"]], [ids["OUT"]], "forward", T * H, A),
    ]
    if train:
        g = {k: b + 100 + v for k, v in dict(OUT=0, Y=1, Fa=2, F1=3, X2a=4, X2=5, O=6, S=7, Q=8,
                                               K=9, Xq=10, Xk=11, X=12).items()}
        if g_out is not None:
            g["OUT"] = g_out  # produced by the next layer's backward (declared there)
        gw = {k: b + 120 + v for k, v in dict(Wq=0, Wk=1, Wo=2, W1=3, W2=4).items()}
        nw = {k: b + 130 + v for k, v in dict(Wq=0, Wk=1, Wo=2, W1=3, W2=4).items()}
        for item in ((() if g_out is not None else ("OUT", (T, H), ids["OUT"])), ("Y", (T, H), ids["Y"]),
                     ("Fa", (T, F), ids["Fa"]), ("F1", (T, F), ids["F1"]),
                     ("X2a", (T, H), ids["X2"]), ("X2", (T, H), ids["X2"]),
                     ("O", (T, H), ids["O"]), ("S", (T, H), ids["S"]),
                     ("Q", (T, H), ids["Q"]), ("K", (T, H), ids["K"]),
                     ("Xq", (T, H), X), ("Xk", (T, H), X), ("X", (T, H), X)):
            if not item:
                continue
            name, shp, of = item
            pts.append(_pt(g[name], shp, "gradient", e, of))
        for w, shp in (("Wq", (H, H)), ("Wk", (H, H)), ("Wo", (H, H)), ("W1", (H, F)), ("W2", (F, H))):
            pts.append(_pt(gw[w], shp, "gradient", e, ids[w]))
            pts.append(_pt(nw[w], shp, "weight", e))
        B = {"layer": layer}
        TA = dict(B, transpose_a=True)
        TB = dict(B, transpose_b=True)
        ops += [
            _op(p + "gres2", "identity", [g["OUT"]], [g["Y"]], "backward", 0, B, p + "res2"),
            _op(p + "gw2a", "matmul", [g["Y"], ids["W2"]], [g["Fa"]], "backward", mm(T, F, H), TB, p + "roww2"),
            _op(p + "gw2w", "matmul", [ids["Fa"], g["Y"]], [gw["W2"]], "backward", mm(F, H, T), TA, p + "roww2"),
            _op(p + "grelu", "mul", [g["Fa"], ids["Z"]], [g["F1"]], "backward", T * F, B, p + "tprelu"),
            _op(p + "gf1a", "matmul", [g["F1"], ids["W1"]], [g["X2a"]], "backward", mm(T, H, F), TB, p + "colf1"),
            _op(p + "gf1w", "matmul", [ids["X2"], g["F1"]], [gw["W1"]], "backward", mm(H, F, T), TA, p + "colf1"),
            _op(p + "gres2x", "add", [g["X2a"], g["OUT"]], [g["X2"]], "backward", T * H, B, p + "res2"),
            _op(p + "gres1", "identity", [g["X2"]], [g["O"]], "backward", 0, B, p + "res1"),
            _op(p + "gwoa", "matmul", [g["O"], ids["Wo"]], [g["S"]], "backward", mm(T, H, H), TB, p + "rowo"),
            _op(p + "gwow", "matmul", [ids["S"], g["O"]], [gw["Wo"]], "backward", mm(H, H, T), TA, p + "rowo"),
            _op(p + "gmulq", "mul", [g["S"], ids["K"]], [g["Q"]], "backward", T * H, B, p + "tpmul"),
            _op(p + "gmulk", "mul", [g["S"], ids["Q"]], [g["K"]], "backward", T * H, B, p + "tpmul"),
            _op(p + "gqa", "matmul", [g["Q"], ids["Wq"]], [g["Xq"]], "backward", mm(T, H, H), TB, p + "colq"),
            _op(p + "gqw", "matmul", [X, g["Q"]], [gw["Wq"]], "backward", mm(H, H, T), TA, p + "colq"),
            _op(p + "gka", "matmul", [g["K"], ids["Wk"]], [g["Xk"]], "backward", mm(T, H, H), TB, p + "colk"),
            _op(p + "gkw", "matmul", [X, g["K"]], [gw["Wk"]], "backward", mm(H, H, T), TA, p + "colk"),
            _op(p + "gres1x", "add", [g["Xq"], g["Xk"], g["X2"]], [g["X"]], "backward", 2 * T * H, B, p + "res1"),
        ]
        for w, kind in (("Wq", "optc"), ("Wk", "optc"), ("W1", "optc"), ("Wo", "optr"), ("W2", "optr")):
            shp = next(q["shape"] for q in pts if q["id"] == ids[w])
            ops.append(_op(p + kind + w.lower(), "add", [ids[w], gw[w]], [nw[w]], "optimizer",
                           shp[0] * shp[1], B))
    return {"ptensors": pts, "ops": ops}


def dumps(doc: dict) -> str:
    return json.dumps(doc)
