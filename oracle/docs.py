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
                  layer: int = 0, prefix: str = "", base: int = 0, x_in=None, g_out=None,
                  seq_parallel: bool = False) -> dict:
    """GPT-3-style transformer block proxy.

    Forward: Q = X·Wq, K = X·Wk (column-parallel), S = Q*K (attention proxy),
    O = S·Wo (row-parallel), X2 = O + X, F1 = X2·W1 [H,4H] (column-parallel),
    F = max(F1, Z) (ReLU proxy), Y = F·W2 [4H,H] (row-parallel), OUT = Y + X2.
    ``train`` adds the mlp_doc-style backward (transposed GEMMs; reference
    proj/tests/testutil.cpp:55-154) and one optimizer add per weight.
    ``seq_parallel`` names the residual adds "spres1" / "spres2" so the
    megatron_tp sProgram splits them on the token dim (Megatron sequence
    parallelism: reduce-scatter after the row-parallel GEMMs, all-gather
    before the column-parallel ones).
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
    r1, r2 = ("spres1", "spres2") if seq_parallel else ("res1", "res2")
    A = {"layer": layer, "batch_dim": 0}
    mm = lambda m, n, k: 2.0 * m * n * k  # noqa: E731
    ops = [
        _op(p + "colq", "matmul", [X, ids["Wq"]], [ids["Q"]], "forward", mm(T, H, H), A),
        _op(p + "colk", "matmul", [X, ids["Wk"]], [ids["K"]], "forward", mm(T, H, H), A),
        _op(p + "tpmul", "mul", [ids["Q"], ids["K"]], [ids["S"]], "forward", T * H, A),
        _op(p + "rowo", "matmul", [ids["S"], ids["Wo"]], [ids["O"]], "forward", mm(T, H, H), A),
        _op(p + r1, "add", [ids["O"], X], [ids["X2"]], "forward", T * H, A),
        _op(p + "colf1", "matmul", [ids["X2"], ids["W1"]], [ids["F1"]], "forward", mm(T, F, H), A),
        _op(p + "tprelu", "max", [ids["F1"], ids["Z"]], [ids["Fa"]], "forward", T * F, A),
        _op(p + "roww2", "matmul", [ids["Fa"], ids["W2"]], [ids["Y"]], "forward", mm(T, H, F), A),
        _op(p + r2, "add", [ids["Y"], ids["X2"]], [ids["OUT"]], "forward", T * H, A),
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
            _op(p + "gres2", "identity", [g["OUT"]], [g["Y"]], "backward", 0, B, p + r2),
            _op(p + "gw2a", "matmul", [g["Y"], ids["W2"]], [g["Fa"]], "backward", mm(T, F, H), TB, p + "roww2"),
            _op(p + "gw2w", "matmul", [ids["Fa"], g["Y"]], [gw["W2"]], "backward", mm(F, H, T), TA, p + "roww2"),
            _op(p + "grelu", "mul", [g["Fa"], ids["Z"]], [g["F1"]], "backward", T * F, B, p + "tprelu"),
            _op(p + "gf1a", "matmul", [g["F1"], ids["W1"]], [g["X2a"]], "backward", mm(T, H, F), TB, p + "colf1"),
            _op(p + "gf1w", "matmul", [ids["X2"], g["F1"]], [gw["W1"]], "backward", mm(H, F, T), TA, p + "colf1"),
            _op(p + "gres2x", "add", [g["X2a"], g["OUT"]], [g["X2"]], "backward", T * H, B, p + r2),
            _op(p + "gres1", "identity", [g["X2"]], [g["O"]], "backward", 0, B, p + r1),
            _op(p + "gwoa", "matmul", [g["O"], ids["Wo"]], [g["S"]], "backward", mm(T, H, H), TB, p + "rowo"),
            _op(p + "gwow", "matmul", [ids["S"], g["O"]], [gw["Wo"]], "backward", mm(H, H, T), TA, p + "rowo"),
            _op(p + "gmulq", "mul", [g["S"], ids["K"]], [g["Q"]], "backward", T * H, B, p + "tpmul"),
            _op(p + "gmulk", "mul", [g["S"], ids["Q"]], [g["K"]], "backward", T * H, B, p + "tpmul"),
            _op(p + "gqa", "matmul", [g["Q"], ids["Wq"]], [g["Xq"]], "backward", mm(T, H, H), TB, p + "colq"),
            _op(p + "gqw", "matmul", [X, g["Q"]], [gw["Wq"]], "backward", mm(H, H, T), TA, p + "colq"),
            _op(p + "gka", "matmul", [g["K"], ids["Wk"]], [g["Xk"]], "backward", mm(T, H, H), TB, p + "colk"),
            _op(p + "gkw", "matmul", [X, g["K"]], [gw["Wk"]], "backward", mm(H, H, T), TA, p + "colk"),
            _op(p + "gres1x", "add", [g["Xq"], g["Xk"], g["X2"]], [g["X"]], "backward", 2 * T * H, B, p + r1),
        ]
        for w, kind in (("Wq", "optc"), ("Wk", "optc"), ("W1", "optc"), ("Wo", "optr"), ("W2", "optr")):
            shp = next(q["shape"] for q in pts if q["id"] == ids[w])
            ops.append(_op(p + kind + w.lower(), "add", [ids[w], gw[w]], [nw[w]], "optimizer",
                           shp[0] * shp[1], B))
    return {"ptensors": pts, "ops": ops}


def dumps(doc: dict) -> str:
    return json.dumps(doc)


# ---- schema extension --------------------------------------
# Kinds the reference front end rejects (document.cpp:43-53) are compiled
# through stand-ins with the same data flow and partitioning — unary ops as
# `identity`, binary gradient ops as `mul` — and written back into the
# compiled plan by rewrite_plan (op ids are preserved by op-trans as
# "<id>/<i>" and "<id>~rc").
EXT_STANDIN = {"softmax": "identity", "layernorm": "identity", "gelu": "identity",
               "softmax-grad": "mul", "layernorm-grad": "mul", "gelu-grad": "mul",
               # attention(Q, K, V) partitions like a 3-operand elementwise op:
               # head (column) and sequence (row) splits carry over; the
               # executor rejects pieces that cut a sequence or a head
               "attention": "add",
               # attention-grad(Q, K, V, O, dO) -> dQ | dK | dV ("wrt"): a 5-operand add
               "attention-grad": "add"}
EXT_ATTRS = ("segment", "eps", "head_dim", "seq", "causal")


def gpt_block_ext_doc(tokens: int, hidden: int, head: int, elem_size: int = 2, train: bool = True) -> dict:
    """Transformer block with the extended sub-operators (config C2x):
    N1 = LN(X); Q = N1·Wq, K = N1·Wk (column-parallel); P = softmax over
    each `head`-wide segment of Q (per attention head, split with the heads);
    S = P*K; O = S·Wo (row-parallel); X2 = O + X; N2 = LN(X2);
    F1 = N2·W1 (column-parallel); Fa = GELU(F1); Y = Fa·W2 (row-parallel);
    OUT = Y + X2. LayerNorms are replicated (full rows), as in Megatron.
    ``train`` adds the backward (softmax-grad / layernorm-grad / gelu-grad and
    the transposed GEMMs) and one optimizer add per weight."""
    T, H, Fd = tokens, hidden, 4 * hidden
    e = elem_size
    ids = dict(X=0, Wq=1, Wk=2, Wo=3, W1=4, W2=5, N1=10, Q=11, K=12, P=13, S=14, O=15, X2=16, N2=17, F1=18,
               Fa=19, Y=20, OUT=21)
    pts = [_pt(ids["X"], (T, H), "activation", e)]
    for w, shp in (("Wq", (H, H)), ("Wk", (H, H)), ("Wo", (H, H)), ("W1", (H, Fd)), ("W2", (Fd, H))):
        pts.append(_pt(ids[w], shp, "weight", e))
    for a, shp in (("N1", (T, H)), ("Q", (T, H)), ("K", (T, H)), ("P", (T, H)), ("S", (T, H)), ("O", (T, H)),
                   ("X2", (T, H)), ("N2", (T, H)), ("F1", (T, Fd)), ("Fa", (T, Fd)), ("Y", (T, H)),
                   ("OUT", (T, H))):
        pts.append(_pt(ids[a], shp, "activation", e))
    A = {"layer": 0, "batch_dim": 0}
    SEG = dict(A, segment=head)
    mm = lambda m, n, k: 2.0 * m * n * k  # noqa: E731
    ops = [
        _op("ln1", "layernorm", [ids["X"]], [ids["N1"]], "forward", 8 * T * H, A),
        _op("colq", "matmul", [ids["N1"], ids["Wq"]], [ids["Q"]], "forward", mm(T, H, H), A),
        _op("colk", "matmul", [ids["N1"], ids["Wk"]], [ids["K"]], "forward", mm(T, H, H), A),
        _op("tpsm", "softmax", [ids["Q"]], [ids["P"]], "forward", 8 * T * H, SEG),
        _op("tpmul", "mul", [ids["P"], ids["K"]], [ids["S"]], "forward", T * H, A),
        _op("rowo", "matmul", [ids["S"], ids["Wo"]], [ids["O"]], "forward", mm(T, H, H), A),
        _op("res1", "add", [ids["O"], ids["X"]], [ids["X2"]], "forward", T * H, A),
        _op("ln2", "layernorm", [ids["X2"]], [ids["N2"]], "forward", 8 * T * H, A),
        _op("colf1", "matmul", [ids["N2"], ids["W1"]], [ids["F1"]], "forward", mm(T, Fd, H), A),
        _op("tpgelu", "gelu", [ids["F1"]], [ids["Fa"]], "forward", 8 * T * Fd, A),
        _op("roww2", "matmul", [ids["Fa"], ids["W2"]], [ids["Y"]], "forward", mm(T, H, Fd), A),
        _op("res2", "add", [ids["Y"], ids["X2"]], [ids["OUT"]], "forward", T * H, A),
    ]
    if train:
        g = {k: 100 + v for k, v in dict(OUT=0, Y=1, Fa=2, F1=3, N2=4, X2a=5, X2=6, O=7, S=8, P=9, K=10, Q=11,
                                         N1q=12, N1k=13, N1=14, X1=15, X=16).items()}
        of = dict(OUT="OUT", Y="Y", Fa="Fa", F1="F1", N2="N2", X2a="X2", X2="X2", O="O", S="S", P="P", K="K",
                  Q="Q", N1q="N1", N1k="N1", N1="N1", X1="X", X="X")
        for name, src in of.items():
            shp = next(q["shape"] for q in pts if q["id"] == ids[src])
            pts.append(_pt(g[name], shp, "gradient", e, ids[src]))
        gw = {k: 130 + v for k, v in dict(Wq=0, Wk=1, Wo=2, W1=3, W2=4).items()}
        nw = {k: 140 + v for k, v in dict(Wq=0, Wk=1, Wo=2, W1=3, W2=4).items()}
        for w, shp in (("Wq", (H, H)), ("Wk", (H, H)), ("Wo", (H, H)), ("W1", (H, Fd)), ("W2", (Fd, H))):
            pts.append(_pt(gw[w], shp, "gradient", e, ids[w]))
            pts.append(_pt(nw[w], shp, "weight", e))
        B = {"layer": 0}
        TA = dict(B, transpose_a=True)
        TB = dict(B, transpose_b=True)
        ops += [
            _op("gres2", "identity", [g["OUT"]], [g["Y"]], "backward", 0, B, "res2"),
            _op("gw2a", "matmul", [g["Y"], ids["W2"]], [g["Fa"]], "backward", mm(T, Fd, H), TB, "roww2"),
            _op("gw2w", "matmul", [ids["Fa"], g["Y"]], [gw["W2"]], "backward", mm(Fd, H, T), TA, "roww2"),
            _op("ggelu", "gelu-grad", [ids["F1"], g["Fa"]], [g["F1"]], "backward", 8 * T * Fd, B, "tpgelu"),
            _op("gf1a", "matmul", [g["F1"], ids["W1"]], [g["N2"]], "backward", mm(T, H, Fd), TB, "colf1"),
            _op("gf1w", "matmul", [ids["N2"], g["F1"]], [gw["W1"]], "backward", mm(H, Fd, T), TA, "colf1"),
            _op("gln2", "layernorm-grad", [ids["X2"], g["N2"]], [g["X2a"]], "backward", 8 * T * H, B, "ln2"),
            _op("gres2x", "add", [g["X2a"], g["OUT"]], [g["X2"]], "backward", T * H, B, "res2"),
            _op("gres1", "identity", [g["X2"]], [g["O"]], "backward", 0, B, "res1"),
            _op("gwoa", "matmul", [g["O"], ids["Wo"]], [g["S"]], "backward", mm(T, H, H), TB, "rowo"),
            _op("gwow", "matmul", [ids["S"], g["O"]], [gw["Wo"]], "backward", mm(H, H, T), TA, "rowo"),
            _op("gmulp", "mul", [g["S"], ids["K"]], [g["P"]], "backward", T * H, B, "tpmul"),
            _op("gmulk", "mul", [g["S"], ids["P"]], [g["K"]], "backward", T * H, B, "tpmul"),
            _op("gsm", "softmax-grad", [ids["P"], g["P"]], [g["Q"]], "backward", 8 * T * H, dict(B, segment=head),
                "tpsm"),
            _op("gqa", "matmul", [g["Q"], ids["Wq"]], [g["N1q"]], "backward", mm(T, H, H), TB, "colq"),
            _op("gqw", "matmul", [ids["N1"], g["Q"]], [gw["Wq"]], "backward", mm(H, H, T), TA, "colq"),
            _op("gka", "matmul", [g["K"], ids["Wk"]], [g["N1k"]], "backward", mm(T, H, H), TB, "colk"),
            _op("gkw", "matmul", [ids["N1"], g["K"]], [gw["Wk"]], "backward", mm(H, H, T), TA, "colk"),
            _op("gln1s", "add", [g["N1q"], g["N1k"]], [g["N1"]], "backward", T * H, B, "ln1"),
            _op("gln1", "layernorm-grad", [ids["X"], g["N1"]], [g["X1"]], "backward", 8 * T * H, B, "ln1"),
            _op("gres1x", "add", [g["X1"], g["X2"]], [g["X"]], "backward", T * H, B, "res1"),
        ]
        for w, kind in (("Wq", "optc"), ("Wk", "optc"), ("W1", "optc"), ("Wo", "optr"), ("W2", "optr")):
            shp = next(q["shape"] for q in pts if q["id"] == ids[w])
            ops.append(_op(kind + w.lower(), "add", [ids[w], gw[w]], [nw[w]], "optimizer", shp[0] * shp[1], B))
    return {"ptensors": pts, "ops": ops}


def standin_doc(doc: dict) -> dict:
    """The document the reference front end accepts: extended kinds replaced
    by their stand-ins (same operands, same partitioning behaviour)."""
    out = json.loads(json.dumps(doc))
    for op in out["ops"]:
        if op["kind"] in EXT_STANDIN:
            op["kind"] = EXT_STANDIN[op["kind"]]
            for a in ("segment", "head_dim", "seq", "causal", "wrt"):
                op.get("attrs", {}).pop(a, None)
    return out


def rewrite_plan(plan_json: str, doc: dict) -> str:
    """Writes the extended kinds (and their segment / eps) back into a plan
    compiled from standin_doc(doc)."""
    ext = {op["id"]: op for op in doc["ops"] if op["kind"] in EXT_STANDIN}
    p = json.loads(plan_json)
    n = 0
    for op in p["ops"]:
        base = op["id"].split("/")[0].split("~")[0]
        if base in ext:
            src = ext[base]
            op["kind"] = src["kind"]
            attrs = src.get("attrs", {})
            if attrs.get("segment"):
                op["segment"] = attrs["segment"]
            for a in ("eps", "head_dim", "seq", "causal", "wrt"):
                if a in attrs:
                    op[a] = attrs[a]
            n += 1
    if n == 0:
        raise ValueError("rewrite_plan: no extended op found in the plan")
    return json.dumps(p)


def gpt_block_attn_doc(tokens: int, hidden: int, head_dim: int, seq: int, elem_size: int = 2) -> dict:
    """Transformer block forward with real attention (config C2a, inference
    prefill): N1 = LN(X); Q, K, V = N1·Wq, N1·Wk, N1·Wv (column-parallel);
    A = attention(Q, K, V) (causal, per head, split with the heads); O = A·Wo
    (row-parallel); X2 = O + X; N2 = LN(X2); F1 = N2·W1 (column-parallel);
    Fa = GELU(F1); Y = Fa·W2 (row-parallel); OUT = Y + X2."""
    T, H, Fd = tokens, hidden, 4 * hidden
    e = elem_size
    ids = dict(X=0, Wq=1, Wk=2, Wv=3, Wo=4, W1=5, W2=6, N1=10, Q=11, K=12, V=13, A=14, O=15, X2=16, N2=17, F1=18,
               Fa=19, Y=20, OUT=21)
    pts = [_pt(ids["X"], (T, H), "activation", e)]
    for w, shp in (("Wq", (H, H)), ("Wk", (H, H)), ("Wv", (H, H)), ("Wo", (H, H)), ("W1", (H, Fd)), ("W2", (Fd, H))):
        pts.append(_pt(ids[w], shp, "weight", e))
    for a, shp in (("N1", (T, H)), ("Q", (T, H)), ("K", (T, H)), ("V", (T, H)), ("A", (T, H)), ("O", (T, H)),
                   ("X2", (T, H)), ("N2", (T, H)), ("F1", (T, Fd)), ("Fa", (T, Fd)), ("Y", (T, H)),
                   ("OUT", (T, H))):
        pts.append(_pt(ids[a], shp, "activation", e))
    A = {"layer": 0, "batch_dim": 0}
    mm = lambda m, n, k: 2.0 * m * n * k  # noqa: E731
    ops = [
        _op("ln1", "layernorm", [ids["X"]], [ids["N1"]], "forward", 8 * T * H, A),
        _op("colq", "matmul", [ids["N1"], ids["Wq"]], [ids["Q"]], "forward", mm(T, H, H), A),
        _op("colk", "matmul", [ids["N1"], ids["Wk"]], [ids["K"]], "forward", mm(T, H, H), A),
        _op("colv", "matmul", [ids["N1"], ids["Wv"]], [ids["V"]], "forward", mm(T, H, H), A),
        _op("tpattn", "attention", [ids["Q"], ids["K"], ids["V"]], [ids["A"]], "forward", 2.0 * T * seq * H,
            dict(A, head_dim=head_dim, seq=seq, causal=True)),
        _op("rowo", "matmul", [ids["A"], ids["Wo"]], [ids["O"]], "forward", mm(T, H, H), A),
        _op("res1", "add", [ids["O"], ids["X"]], [ids["X2"]], "forward", T * H, A),
        _op("ln2", "layernorm", [ids["X2"]], [ids["N2"]], "forward", 8 * T * H, A),
        _op("colf1", "matmul", [ids["N2"], ids["W1"]], [ids["F1"]], "forward", mm(T, Fd, H), A),
        _op("tpgelu", "gelu", [ids["F1"]], [ids["Fa"]], "forward", 8 * T * Fd, A),
        _op("roww2", "matmul", [ids["Fa"], ids["W2"]], [ids["Y"]], "forward", mm(T, H, Fd), A),
        _op("res2", "add", [ids["Y"], ids["X2"]], [ids["OUT"]], "forward", T * H, A),
    ]
    return {"ptensors": pts, "ops": ops}


def gpt_block_attn_train_doc(tokens: int, hidden: int, head_dim: int, seq: int, elem_size: int = 2) -> dict:
    """The C2a block (LayerNorm, Q/K/V projections, fused causal attention,
    Wo, GELU MLP) as a train step (config C2at): forward, the backward with
    attention-grad (dQ, dK, dV) and the other extended gradients, and one
    optimizer add per weight. Megatron TP: Q/K/V/W1 column-parallel (split
    with the heads), Wo/W2 row-parallel, LayerNorms replicated."""
    T, H, Fd = tokens, hidden, 4 * hidden
    e = elem_size
    doc = gpt_block_attn_doc(tokens, hidden, head_dim, seq, elem_size)
    pts, ops = doc["ptensors"], doc["ops"]
    ids = dict(X=0, Wq=1, Wk=2, Wv=3, Wo=4, W1=5, W2=6, N1=10, Q=11, K=12, V=13, A=14, O=15, X2=16, N2=17, F1=18,
               Fa=19, Y=20, OUT=21)
    names = ["OUT", "Y", "Fa", "F1", "N2", "X2a", "X2", "O", "A", "Q", "K", "V", "N1q", "N1k", "N1v", "N1", "X1", "X"]
    g = {n: 100 + i for i, n in enumerate(names)}
    of = dict(OUT="OUT", Y="Y", Fa="Fa", F1="F1", N2="N2", X2a="X2", X2="X2", O="O", A="A", Q="Q", K="K", V="V",
              N1q="N1", N1k="N1", N1v="N1", N1="N1", X1="X", X="X")
    for n, src in of.items():
        shp = next(q["shape"] for q in pts if q["id"] == ids[src])
        pts.append(_pt(g[n], shp, "gradient", e, ids[src]))
    W = {"Wq": (H, H), "Wk": (H, H), "Wv": (H, H), "Wo": (H, H), "W1": (H, Fd), "W2": (Fd, H)}
    gw = {w: 130 + i for i, w in enumerate(W)}
    nw = {w: 140 + i for i, w in enumerate(W)}
    for w, shp in W.items():
        pts.append(_pt(gw[w], shp, "gradient", e, ids[w]))
        pts.append(_pt(nw[w], shp, "weight", e))
    B = {"layer": 0}
    TA = dict(B, transpose_a=True)
    TB = dict(B, transpose_b=True)
    AT = dict(B, head_dim=head_dim, seq=seq, causal=True)
    mm = lambda m, n, k: 2.0 * m * n * k  # noqa: E731
    fa = 2.0 * T * seq * H
    ops += [
        _op("gres2", "identity", [g["OUT"]], [g["Y"]], "backward", 0, B, "res2"),
        _op("gw2a", "matmul", [g["Y"], ids["W2"]], [g["Fa"]], "backward", mm(T, Fd, H), TB, "roww2"),
        _op("gw2w", "matmul", [ids["Fa"], g["Y"]], [gw["W2"]], "backward", mm(Fd, H, T), TA, "roww2"),
        _op("ggelu", "gelu-grad", [ids["F1"], g["Fa"]], [g["F1"]], "backward", 8 * T * Fd, B, "tpgelu"),
        _op("gf1a", "matmul", [g["F1"], ids["W1"]], [g["N2"]], "backward", mm(T, H, Fd), TB, "colf1"),
        _op("gf1w", "matmul", [ids["N2"], g["F1"]], [gw["W1"]], "backward", mm(H, Fd, T), TA, "colf1"),
        _op("gln2", "layernorm-grad", [ids["X2"], g["N2"]], [g["X2a"]], "backward", 8 * T * H, B, "ln2"),
        _op("gres2x", "add", [g["X2a"], g["OUT"]], [g["X2"]], "backward", T * H, B, "res2"),
        _op("gres1", "identity", [g["X2"]], [g["O"]], "backward", 0, B, "res1"),
        _op("gwoa", "matmul", [g["O"], ids["Wo"]], [g["A"]], "backward", mm(T, H, H), TB, "rowo"),
        _op("gwow", "matmul", [ids["A"], g["O"]], [gw["Wo"]], "backward", mm(H, H, T), TA, "rowo"),
    ]
    for w in "qkv":
        ops.append(_op("gattn" + w, "attention-grad", [ids["Q"], ids["K"], ids["V"], ids["A"], g["A"]],
                       [g[w.upper()]], "backward", fa, dict(AT, wrt=w), "tpattn"))
    for w, n in (("q", "N1q"), ("k", "N1k"), ("v", "N1v")):
        W_ = "W" + w
        ops.append(_op("g" + w + "a", "matmul", [g[w.upper()], ids[W_]], [g[n]], "backward", mm(T, H, H), TB,
                       "col" + w))
        ops.append(_op("g" + w + "w", "matmul", [ids["N1"], g[w.upper()]], [gw[W_]], "backward", mm(H, H, T), TA,
                       "col" + w))
    ops += [
        _op("gln1s", "add", [g["N1q"], g["N1k"], g["N1v"]], [g["N1"]], "backward", 2 * T * H, B, "ln1"),
        _op("gln1", "layernorm-grad", [ids["X"], g["N1"]], [g["X1"]], "backward", 8 * T * H, B, "ln1"),
        _op("gres1x", "add", [g["X1"], g["X2"]], [g["X"]], "backward", T * H, B, "res1"),
    ]
    for w, kind in (("Wq", "optc"), ("Wk", "optc"), ("Wv", "optc"), ("W1", "optc"), ("Wo", "optr"), ("W2", "optr")):
        shp = W[w]
        ops.append(_op(kind + w.lower(), "add", [ids[w], gw[w]], [nw[w]], "optimizer", shp[0] * shp[1], B))
    return {"ptensors": pts, "ops": ops}


def attention_doc(tokens: int, heads: int, head_dim: int, seq: int, causal: bool = False, elem_size: int = 2,
                  prefix: str = "tp") -> dict:
    """One fused attention op O = attention(Q, K, V) over [tokens, heads x
    head_dim] operands (sequences of ``seq`` tokens). ``prefix`` "tp" makes
    megatron_tp split it by heads (dim 1)."""
    T, D = tokens, heads * head_dim
    pts = [_pt(i, (T, D), "activation", elem_size) for i in range(4)]
    ops = [_op(prefix + "attn", "attention", [0, 1, 2], [3], "forward", 4.0 * T * seq * D,
               {"batch_dim": 0, "head_dim": head_dim, "seq": seq, "causal": causal})]
    return {"ptensors": pts, "ops": ops}


def attention_train_doc(tokens: int, heads: int, head_dim: int, seq: int, causal: bool = True,
                        elem_size: int = 2) -> dict:
    """O = attention(Q, K, V) and its three gradients dQ, dK, dV from dO
    (attention-grad with wrt = q / k / v, each the backward of the forward
    op): the executor merges the three per lane into one instruction."""
    T, D = tokens, heads * head_dim
    pts = [_pt(i, (T, D), "activation", elem_size) for i in range(4)] + [_pt(4, (T, D), "gradient", elem_size, 3)]
    pts += [_pt(5 + i, (T, D), "gradient", elem_size, i) for i in range(3)]
    A = {"batch_dim": 0, "head_dim": head_dim, "seq": seq, "causal": causal}
    fl = 4.0 * T * seq * D * (0.5 if causal else 1.0)
    ops = [_op("tpattn", "attention", [0, 1, 2], [3], "forward", fl, A)]
    for i, w in enumerate("qkv"):
        ops.append(_op("tpg" + w, "attention-grad", [0, 1, 2, 3, 4], [5 + i], "backward", fl, dict(A, wrt=w), "tpattn"))
    return {"ptensors": pts, "ops": ops}


# ---- C4 / C5 benchmark documents ------------------------------------


def swin_stage_doc(tokens: int, hidden: int, elem_size: int = 2) -> dict:
    """Swin-Transformer stage block proxy (config C4): the
    GPT-style block of ``gpt_block_doc`` (window-attention proxy Q / K / S /
    O, FFN 4H with ReLU proxy) as a train step, plus one ``agw*`` identity op
    per updated weight — the parameter publication of a sharded (ZeRO-style)
    optimizer: every data-parallel rank updates a row slice of each weight
    and the next step's replicas read the whole updated weight. Under the
    ``coshard_dp`` sProgram the weight gradients therefore leave each rank as
    reduce-scatters (V(dp) -> D(dp)) and the updates come back as
    all-gathers (D(dp) -> R(dp)), the adapters Dijkstra picks for sharded
    weight updates (reference rvd.cpp:194-284)."""
    d = gpt_block_doc(tokens, hidden, elem_size, train=True)
    pts, ops = d["ptensors"], d["ops"]
    H, F = hidden, 4 * hidden
    for v, (w, shp) in enumerate((("wq", (H, H)), ("wk", (H, H)), ("wo", (H, H)), ("w1", (H, F)), ("w2", (F, H)))):
        pts.append(_pt(140 + v, shp, "weight", elem_size))
        ops.append(_op("agw" + w, "identity", [130 + v], [140 + v], "optimizer", 0, {"layer": 0}))
    return {"ptensors": pts, "ops": ops}


def evoformer_doc(layers: int, msa: tuple, pair: tuple, micro_batches: int = 1, elem_size: int = 2) -> dict:
    """AlphaFold2 Evoformer proxy (config C5) in the
    three-forward-passes-plus-one-backward shape of the reference's
    ``three_pass_doc`` (proj/tests/testutil.cpp:298-368: passes 1-3 with
    their own weights, gradients only through pass 3), with two streams per
    layer: the MSA representation M [Nm, Cm] and the pair representation
    Z [Np, Cz]. Each stream, per layer, pass and micro-batch:

      R = X·Wr       row-attention proxy    (``row*``: DAP splits rows, dim 0)
      C = max(R, G)  column-attention proxy (``col*``: DAP splits channels, dim 1)
      X' = C·Wt      transition             (``row*``: rows again)

    so DAP (``threef1b_dap``) switches the layout D(2,1) -> D(1,2) -> D(2,1)
    twice per stream and layer: the all-to-all layout adapters of
    rvd.cpp:286-326. Micro-batches are explicit in the document (op ids end
    in ``#k``; activations of micro-batch k are their own pTensors of Nr/K
    rows; weights are shared): the reference's collective pattern matching
    works per pTensor family (rvd.cpp:785-870) and only finds collectives
    when one family is one micro-batch. Backward (pass 3, reverse layer
    order, per micro-batch) declares dX / dW GEMMs (transposed operands) and
    the gate gradient mul(dC, G); the K weight gradients of a pass-3 weight
    are accumulated by one ``gacc`` add and applied by one optimizer add."""
    e = elem_size
    L, K = layers, micro_batches
    pts, ops = [], []
    for s, (Nr, Cc), base in (("m", msa, 0), ("z", pair, 500000)):
        if Nr % K:
            raise ValueError("rows must divide into micro-batches")
        rows = Nr // K
        # activations of micro-batch k: base + 10000*k + 100*p + 10*l + {0: X_in, 1: R, 2: C, 3: X'}
        act = lambda k, p, l, j, base=base: base + 10000 * k + 100 * p + 10 * l + j  # noqa: E731
        wt = lambda p, l, j, base=base: base + 100000 + 100 * p + 10 * l + j  # noqa: E731  (0 Wr, 1 Wt, 2 G)
        gx = lambda k, l, base=base: base + 200000 + 10000 * k + 10 * l  # noqa: E731  (+0 dX_in, +1 dR, +2 dC)
        gw = lambda k, l, j, base=base: base + 300000 + 1000 * k + 10 * l + j  # noqa: E731
        for p in (1, 2, 3):
            for l in range(L):
                for j in (0, 1):
                    pts.append(_pt(wt(p, l, j), (Cc, Cc), "weight", e))
                pts.append(_pt(wt(p, l, 2), (rows, Cc), "activation", e))  # gate, shared by the micro-batches
        for l in range(L):
            for j in (0, 1):
                pts.append(_pt(gw(K, l, j), (Cc, Cc), "gradient", e, wt(3, l, j)))  # accumulated
                pts.append(_pt(gw(K + 1, l, j), (Cc, Cc), "weight", e))  # updated
        mm = 2.0 * rows * Cc * Cc
        for k in range(K):
            pts.append(_pt(act(k, 1, 0, 0), (rows, Cc), "activation", e))
            for p in (1, 2, 3):
                for l in range(L):
                    for j in (1, 2, 3):
                        pts.append(_pt(act(k, p, l, j), (rows, Cc), "activation", e))
            for p in (1, 2, 3):
                for l in range(L):
                    x_in = act(k, 1, 0, 0) if (p == 1 and l == 0) else (
                        act(k, p - 1, L - 1, 3) if l == 0 else act(k, p, l - 1, 3))
                    A = {"layer": l, "batch_dim": 0, "pass": p}
                    f = f"{s}{p}_{l}"
                    ops.append(_op(f"{f}.rowr#{k}", "matmul", [x_in, wt(p, l, 0)], [act(k, p, l, 1)], "forward", mm, A))
                    ops.append(_op(f"{f}.colg#{k}", "max", [act(k, p, l, 1), wt(p, l, 2)], [act(k, p, l, 2)],
                                   "forward", rows * Cc, A))
                    ops.append(_op(f"{f}.rowt#{k}", "matmul", [act(k, p, l, 2), wt(p, l, 1)], [act(k, p, l, 3)],
                                   "forward", mm, A))
            for l in range(L):
                x_in = act(k, 2, L - 1, 3) if l == 0 else act(k, 3, l - 1, 3)
                pts.append(_pt(gx(k, l), (rows, Cc), "gradient", e, x_in))
                pts.append(_pt(gx(k, l) + 1, (rows, Cc), "gradient", e, act(k, 3, l, 1)))
                pts.append(_pt(gx(k, l) + 2, (rows, Cc), "gradient", e, act(k, 3, l, 2)))
                for j in (0, 1):
                    pts.append(_pt(gw(k, l, j), (Cc, Cc), "gradient", e, wt(3, l, j)))
            pts.append(_pt(gx(k, L), (rows, Cc), "gradient", e, act(k, 3, L - 1, 3)))
            for l in reversed(range(L)):
                x_in = act(k, 2, L - 1, 3) if l == 0 else act(k, 3, l - 1, 3)
                B = {"layer": l}
                TA, TB = dict(B, transpose_a=True), dict(B, transpose_b=True)
                f = f"{s}3_{l}"
                ops += [
                    _op(f"{f}.growt#{k}", "matmul", [gx(k, l + 1), wt(3, l, 1)], [gx(k, l) + 2], "backward", mm, TB,
                        f"{f}.rowt#{k}"),
                    _op(f"{f}.growtw#{k}", "matmul", [act(k, 3, l, 2), gx(k, l + 1)], [gw(k, l, 1)], "backward", mm,
                        TA, f"{f}.rowt#{k}"),
                    _op(f"{f}.gcolg#{k}", "mul", [gx(k, l) + 2, wt(3, l, 2)], [gx(k, l) + 1], "backward", rows * Cc,
                        B, f"{f}.colg#{k}"),
                    _op(f"{f}.growr#{k}", "matmul", [gx(k, l) + 1, wt(3, l, 0)], [gx(k, l)], "backward", mm, TB,
                        f"{f}.rowr#{k}"),
                    _op(f"{f}.growrw#{k}", "matmul", [x_in, gx(k, l) + 1], [gw(k, l, 0)], "backward", mm, TA,
                        f"{f}.rowr#{k}"),
                ]
        for l in range(L):
            for j in (0, 1):
                ops.append(_op(f"{s}3_{l}.gacc{j}", "add", [gw(k, l, j) for k in range(K)], [gw(K, l, j)],
                               "optimizer", K * Cc * Cc, {"layer": l}))
                ops.append(_op(f"{s}3_{l}.opt{j}", "add", [wt(3, l, j), gw(K, l, j)], [gw(K + 1, l, j)],
                               "optimizer", Cc * Cc, {"layer": l}))
    return {"ptensors": pts, "ops": ops}
