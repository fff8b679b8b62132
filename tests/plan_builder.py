"""TEST INFRASTRUCTURE — minimal plan.json documents for single sub-operators.

Builds ExecutionPlan wire documents (reference simulate.cpp:492-602 schema)
for one op on one lane, so kernel-level tests can run on the GPU box where
the reference front end is absent. Used only by tests.
"""
import json


def single_op_plan(kind, in_shapes, out_shape, in_elem=2, out_elem=2, attrs=None):
    attrs = attrs or {}
    pts, vts, feeds = [], [], []
    ins = []
    for i, shp in enumerate(in_shapes):
        pts.append({"id": i, "shape": list(shp), "elem_size": in_elem if not isinstance(in_elem, list) else in_elem[i],
                    "kind": "activation"})
        vts.append({"id": 100 + i, "ptensor": i, "region": [[0, e] for e in shp], "value": [0, 1],
                    "replica": [0, 1], "side": "in", "owner": "op"})
        ins.append(100 + i)
    out_pt = len(in_shapes)
    pts.append({"id": out_pt, "shape": list(out_shape), "elem_size": out_elem, "kind": "activation"})
    vts.append({"id": 200, "ptensor": out_pt, "region": [[0, e] for e in out_shape], "value": [0, 1],
                "replica": [0, 1], "side": "out", "owner": "op"})
    op = {"id": "op", "kind": kind, "inputs": ins, "outputs": [200], "direction": "forward", "flops": 0.0,
          "doc_order": 0, "inserted": False}
    op.update(attrs)
    doc = {"ptensors": pts, "vtensors": vts, "ops": [op], "assignment": {"op": 0}, "feeds": feeds,
           "coll_groups": [], "sync_edges": [],
           "lanes": [{"device": 0, "tasks": [{"kind": "compute", "op": "op", "duration": 0.0, "bytes": 0}]}],
           "cluster": {"devices": [{"id": 0, "group": 0, "memory": 1 << 34}],
                       "intra_link": {"bandwidth": 1e11, "latency": 1e-6},
                       "inter_link": {"bandwidth": 1e10, "latency": 1e-5}, "device_throughput": 1e12}}
    return json.dumps(doc), out_pt


def matmul_plan(m, n, k, ta=False, tb=False, in_elem=2, out_elem=2):
    a = (k, m) if ta else (m, k)
    b = (n, k) if tb else (k, n)
    attrs = {}
    if ta:
        attrs["transpose_a"] = True
    if tb:
        attrs["transpose_b"] = True
    return single_op_plan("matmul", [a, b], (m, n), in_elem, out_elem, attrs)


def matmul_add_plan(m, n, k, ta=False, tb=False):
    """C = op(A)·op(B); E = C + D (bf16): a GEMM with one fusable consumer."""
    doc = json.loads(matmul_plan(m, n, k, ta, tb)[0])
    doc["ptensors"] += [{"id": 3, "shape": [m, n], "elem_size": 2, "kind": "activation"},
                        {"id": 4, "shape": [m, n], "elem_size": 2, "kind": "activation"}]
    full = [[0, m], [0, n]]
    doc["vtensors"] += [
        {"id": 201, "ptensor": 2, "region": full, "value": [0, 1], "replica": [0, 1], "side": "in", "owner": "add"},
        {"id": 202, "ptensor": 3, "region": full, "value": [0, 1], "replica": [0, 1], "side": "in", "owner": "add"},
        {"id": 203, "ptensor": 4, "region": full, "value": [0, 1], "replica": [0, 1], "side": "out", "owner": "add"}]
    doc["ops"].append({"id": "add", "kind": "add", "inputs": [201, 202], "outputs": [203], "direction": "forward",
                       "flops": 0.0, "doc_order": 1, "inserted": False})
    doc["assignment"]["add"] = 0
    doc["feeds"].append([201, 200])
    doc["lanes"][0]["tasks"].append({"kind": "compute", "op": "add", "duration": 0.0, "bytes": 0})
    return json.dumps(doc), 4


def grouped_matmul_plan(g, m, n, k, ta=False, tb=False, out_elem=2):
    """g independent matmuls of one shape on one lane: C_i = op(A_i)·op(B_i)
    (pTensors A_i = 3i, B_i = 3i+1, C_i = 3i+2) — one grouped GEMM launch."""
    doc = json.loads(matmul_plan(m, n, k, ta, tb, 2, out_elem)[0])
    base = {"pt": doc["ptensors"], "vt": doc["vtensors"], "op": doc["ops"][0]}
    doc["ptensors"], doc["vtensors"], doc["ops"], doc["lanes"][0]["tasks"] = [], [], [], []
    doc["assignment"] = {}
    for i in range(g):
        for j, pt in enumerate(base["pt"]):
            doc["ptensors"].append(dict(pt, id=3 * i + j))
        for vt in base["vt"]:
            v = dict(vt, id=vt["id"] + 1000 * i, ptensor=3 * i + vt["ptensor"], owner=f"op{i}")
            doc["vtensors"].append(v)
        op = dict(base["op"], id=f"op{i}", inputs=[x + 1000 * i for x in base["op"]["inputs"]],
                  outputs=[x + 1000 * i for x in base["op"]["outputs"]], doc_order=i)
        doc["ops"].append(op)
        doc["assignment"][f"op{i}"] = 0
        doc["lanes"][0]["tasks"].append({"kind": "compute", "op": f"op{i}", "duration": 0.0, "bytes": 0})
    return json.dumps(doc)


def matmul_gelu_plan(m, n, k, ta=False, tb=False):
    """C = op(A)·op(B); G = gelu(C) (bf16; schema-extension kind): a GEMM
    whose activation runs in its epilogue."""
    doc = json.loads(matmul_plan(m, n, k, ta, tb)[0])
    doc["ptensors"].append({"id": 3, "shape": [m, n], "elem_size": 2, "kind": "activation"})
    full = [[0, m], [0, n]]
    doc["vtensors"] += [
        {"id": 201, "ptensor": 2, "region": full, "value": [0, 1], "replica": [0, 1], "side": "in", "owner": "act"},
        {"id": 203, "ptensor": 3, "region": full, "value": [0, 1], "replica": [0, 1], "side": "out", "owner": "act"}]
    doc["ops"].append({"id": "act", "kind": "gelu", "inputs": [201], "outputs": [203], "direction": "forward",
                       "flops": 0.0, "doc_order": 1, "inserted": False})
    doc["assignment"]["act"] = 0
    doc["feeds"].append([201, 200])
    doc["lanes"][0]["tasks"].append({"kind": "compute", "op": "act", "duration": 0.0, "bytes": 0})
    return json.dumps(doc), 3


def embedding_plan(n, vocab, h, lo, rows, elem=2):
    """out[j] = table[idx[j]] for idx in the shard [lo, lo + rows) of a
    [vocab, h] table, else 0 (refexec.cpp:216-232): one lane holding table
    rows [lo, lo + rows)."""
    doc = json.loads(single_op_plan("embedding-lookup", [(n,), (vocab, h)], (n, h), [4, elem], elem)[0])
    doc["vtensors"][1]["region"] = [[lo, lo + rows], [0, h]]
    return json.dumps(doc), 2


def attention_grad_plan(T, D, head_dim, seq, causal):
    """dQ, dK, dV = attention-grad(Q, K, V, O, dO) on one lane (three ops the
    executor merges into one instruction): pTensors 0..4 in, 5, 6, 7 out."""
    attrs = {"head_dim": head_dim, "seq": seq, "causal": causal, "wrt": "q"}
    doc = json.loads(single_op_plan("attention-grad", [(T, D)] * 5, (T, D), 2, 2, attrs)[0])
    full = [[0, T], [0, D]]
    for i, w in ((1, "k"), (2, "v")):
        pt = 5 + i
        doc["ptensors"].append({"id": pt, "shape": [T, D], "elem_size": 2, "kind": "activation"})
        ins = []
        for j in range(5):
            vid = 300 + 10 * i + j
            doc["vtensors"].append({"id": vid, "ptensor": j, "region": full, "value": [0, 1], "replica": [0, 1],
                                    "side": "in", "owner": "op" + w})
            ins.append(vid)
        oid = 300 + 10 * i + 9
        doc["vtensors"].append({"id": oid, "ptensor": pt, "region": full, "value": [0, 1], "replica": [0, 1],
                                "side": "out", "owner": "op" + w})
        op = {"id": "op" + w, "kind": "attention-grad", "inputs": ins, "outputs": [oid], "direction": "backward",
              "flops": 0.0, "doc_order": i, "inserted": False}
        op.update(dict(attrs, wrt=w))
        doc["ops"].append(op)
        doc["assignment"]["op" + w] = 0
        doc["lanes"][0]["tasks"].append({"kind": "compute", "op": "op" + w, "duration": 0.0, "bytes": 0})
    return json.dumps(doc), (5, 6, 7)
