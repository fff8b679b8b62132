"""Golden fixtures for the schema extension (softmax / layernorm / GELU and
their gradients) — test infrastructure.

The reference has no such op kinds (document.cpp:43-53 rejects them), so:

  plan.json   the UNMODIFIED reference front end (oracle/_ref compile(),
              megatron_tp sProgram) on the stand-in document
              (oracle/docs.py standin_doc: unary kinds as `identity`, binary
              gradients as `mul` — same operands, same partitioning), with the
              real kinds written back (docs.rewrite_plan)
  graph.json  the extended graph document
  io.npz      in_<pt>: the reference's random_integer_inputs (refexec.cpp:559)
              exp_<pt>: oracle/planc_oracle.py run_graph — every op on whole
                        pTensors in float64 (eval_ext, pinned against torch in
                        tests/test_ext_oracle.py); for bf16 plans every op
                        output rounded to bf16, where the executor stores it
  meta.json   tolerance (normwise), provenance

and planc_oracle.run_plan of the partitioned plan must agree with run_graph
(checked here and in tests/test_ext.py). Run:
  python tests/golden/make_golden_ext.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import docs, planc_oracle, refpy  # noqa: E402

CASES = [
    # name, (tokens, hidden, head, elem, train), devices, seed, rel_tol (normwise)
    ("ext_block_tp1", (16, 16, 4, 4, True), 1, 81, 1e-4),
    ("ext_block_tp2", (16, 16, 4, 4, True), 2, 82, 1e-4),
    ("ext_block_tp4", (16, 16, 4, 4, True), 4, 84, 1e-4),
    ("ext_block_tp2_bf16", (32, 32, 8, 2, True), 2, 85, 2e-2),
    ("ext_block_fwd_tp2_mma", (256, 128, 32, 2, False), 2, 86, 2e-2),
]


# Fused attention (bf16): name, (tokens, heads, head_dim, seq, causal), strategy spec, seed, rel_tol
ATTN_CASES = [
    ("attn_heads_tp2_bf16", (512, 4, 64, 256, False), dict(strategy="megatron_tp", devices=2), 91, 2e-2),
    ("attn_causal_tp2_bf16", (512, 2, 128, 256, True), dict(strategy="megatron_tp", devices=2), 92, 2e-2),
    ("attn_seq_split2_bf16", (1024, 2, 128, 512, True), dict(strategy="manual", devices=2, target_ops="tpattn@s0"),
     93, 2e-2),
]


def cases():
    for name, (T, H, hd, e, train), k, seed, tol in CASES:
        yield name, docs.gpt_block_ext_doc(T, H, hd, elem_size=e, train=train), dict(strategy="megatron_tp", devices=k), \
            seed, tol, e, dict(tokens=T, hidden=H, head=hd, elem_size=e, train=train)
    for name, (T, nh, hd, seq, causal), spec, seed, tol in ATTN_CASES:
        yield name, docs.attention_doc(T, nh, hd, seq, causal), spec, seed, tol, 2, \
            dict(tokens=T, heads=nh, head_dim=hd, seq=seq, causal=causal, elem_size=2)
    # fused attention forward + backward (dQ, dK, dV merged per lane), heads split over 2 lanes
    yield "attn_train_tp2_bf16", docs.attention_train_doc(512, 2, 128, 256, True), \
        dict(strategy="megatron_tp", devices=2), 95, 2e-2, 2, dict(tokens=512, heads=2, head_dim=128, seq=256, elem_size=2)
    # C2at: the block train step with fused attention and attention-grad, Megatron TP 2
    yield "attn_block_train_tp2_mma", docs.gpt_block_attn_train_doc(256, 256, 128, 128), \
        dict(strategy="megatron_tp", devices=2), 96, 2e-2, 2, dict(tokens=256, hidden=256, head_dim=128, seq=128, elem_size=2)
    # C2a: the transformer block forward with fused causal attention, Megatron TP 2
    yield "attn_block_fwd_tp2_mma", docs.gpt_block_attn_doc(512, 256, 128, 256), \
        dict(strategy="megatron_tp", devices=2), 94, 2e-2, 2, dict(tokens=512, hidden=256, head_dim=128, seq=256, elem_size=2)


def main():
    index = []
    only = set(sys.argv[1:])
    for name, doc, spec, seed, tol, e, shape in cases():
        if only and name not in only:
            index.append(name)
            continue
        stand = docs.dumps(docs.standin_doc(doc))
        plan = docs.rewrite_plan(refpy.compile_plan(stand, **spec), doc)
        if name.startswith("attn_block"):
            # full blocks at tensor-core widths: integer inputs would grow past
            # bf16's exact range through the GEMM chain (one-ulp rounding
            # differences become percent-level); standard init instead —
            # weights N(0, 1/fan_in), activations / incoming gradients N(0, 1)
            rng = np.random.default_rng(seed)
            produced = {o for op in doc["ops"] for o in op["outputs"]}
            inputs = {}
            for p_ in doc["ptensors"]:
                if p_["id"] in produced:
                    continue
                x = rng.standard_normal(p_["shape"])
                inputs[p_["id"]] = x / np.sqrt(p_["shape"][0]) if p_["kind"] == "weight" else x
        else:
            inputs = refpy.random_integer_inputs(stand, seed, 1)
        got = planc_oracle.run_plan(plan, inputs)
        ok, msg = planc_oracle.compare_outputs(planc_oracle.run_graph(doc, inputs), got, 1e-9)
        if not ok:
            raise SystemExit(f"{name}: partitioned oracle run disagrees with the graph run: {msg}")
        # bf16 plans: expected values rounded to bf16 at every op output (the
        # executor's storage points), so the stated tolerance measures the
        # kernels, not bf16 storage itself.
        expected = planc_oracle.run_graph(doc, inputs, round_bf16=(e == 2))
        d = os.path.join(HERE, name)
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, "graph.json"), "w") as f:
            f.write(docs.dumps(doc))
        with open(os.path.join(d, "plan.json"), "w") as f:
            f.write(plan)
        arrays = {f"in_{kk}": v for kk, v in inputs.items()}
        arrays.update({f"exp_{kk}": v for kk, v in expected.items()})
        np.savez_compressed(os.path.join(d, "io.npz"), **arrays)
        pj = json.loads(plan)
        meta = dict(name=name, seed=seed, rel_tol=tol, normwise=True, extension=True,
                    provenance="schema extension: reference front end on stand-ins + rewrite_plan; "
                               "expected = planc_oracle.run_graph (float64, torch-pinned)",
                    spec=dict(spec, **shape),
                    max_abs=max(float(np.abs(v).max()) for v in expected.values()),
                    lanes=len(pj["lanes"]), tasks=sum(len(lane["tasks"]) for lane in pj["lanes"]),
                    collectives=sorted({g["primitive"] for g in pj["coll_groups"]}),
                    op_kinds=sorted({o["kind"] for o in pj["ops"]}))
        with open(os.path.join(d, "meta.json"), "w") as f:
            json.dump(meta, f, indent=1)
        index.append(name)
        print(f"{name:24s} lanes={meta['lanes']} tasks={meta['tasks']:4d} coll={meta['collectives']}")
    with open(os.path.join(HERE, "index_ext.json"), "w") as f:
        json.dump(index, f, indent=1)


if __name__ == "__main__":
    main()
