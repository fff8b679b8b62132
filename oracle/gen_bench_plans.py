"""Generates the benchmark plans in plans/ with the UNMODIFIED reference
front end (oracle/_ref: load_graph -> sProgram -> compile -> save_plan).

Plans are the executor's INPUT (what the reference compiler emits); they are
generated once here, where /root/reference exists, and committed — the GPU
box has no reference. Shapes follow SURVEY.md §8d:

  c2   GPT-3-style block (oracle/docs.py gpt_block_doc), train step,
       T=8192 tokens (4 seq x 2048), H=2048, FFN=4H, bf16,
       Megatron TP = 1/2/4/8 (megatron_tp sProgram)
  c1l  2-layer MLP (reference mlp_doc) B=16384, H=4096, bf16, DP = 1/2/4/8
  c2x  the schema-extension transformer block (docs.gpt_block_ext_doc: LN,
       per-head softmax, GELU and their gradients), T=8192, H=2048, 16 heads
       of 128, bf16, Megatron TP = 1/2/4/8 — compiled by the reference front
       end on the stand-in document and rewritten (docs.rewrite_plan); the
       *_cpu_standin plan keeps the stand-ins so the reference CPU executor
       (which has no LN / softmax / GELU) can be timed on the same data flow
  *_cpu  the same graphs at the reduced shape the CPU executor can run
       (T=H=128; SURVEY §8d "CPU baseline")

Run:  python oracle/gen_bench_plans.py [config ...]   (default: all)
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle import docs, refpy  # noqa: E402

OUT = os.path.join(ROOT, "plans")


def write(name, graph, plan, meta):
    if len(plan) > (2 << 20):  # large plans (C3) are stored gzipped
        import gzip

        with open(os.path.join(OUT, name + ".plan.json.gz"), "wb") as raw:
            with gzip.GzipFile(fileobj=raw, mode="wb", compresslevel=9, mtime=0) as f:  # deterministic bytes
                f.write(plan.encode())
    else:
        with open(os.path.join(OUT, name + ".plan.json"), "w") as f:
            f.write(plan)
    with open(os.path.join(OUT, name + ".graph.json"), "w") as f:
        f.write(graph)
    pj = json.loads(plan)
    meta = dict(meta, lanes=len(pj["lanes"]), tasks=sum(len(l["tasks"]) for l in pj["lanes"]),
                collectives=sorted({g["primitive"] for g in pj["coll_groups"]}))
    with open(os.path.join(OUT, name + ".meta.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(name, meta["lanes"], meta["tasks"], meta["collectives"])


def gen_c2x():
    for T, H, hd, tag in ((8192, 2048, 128, ""), (128, 128, 32, "_cpu")):
        doc = docs.gpt_block_ext_doc(T, H, hd, elem_size=2, train=True)
        stand = docs.dumps(docs.standin_doc(doc))
        meta = dict(config="c2x", tokens=T, hidden=H, head=hd, dtype="bf16", samples_per_step=T,
                    sample="token (row of X)", extension=True)
        for k in (1, 2, 4, 8):
            if tag and k > 1:
                continue
            plan = refpy.compile_plan(stand, strategy="megatron_tp", devices=k)
            write(f"c2x_tp{k}{tag}", docs.dumps(doc), docs.rewrite_plan(plan, doc), dict(meta, tp=k))
            if tag:
                write(f"c2x_tp{k}{tag}_standin", stand, plan, dict(meta, tp=k, standin=True))


def main():
    os.makedirs(OUT, exist_ok=True)
    only = set(sys.argv[1:])
    if only:
        if "c2x" in only:
            gen_c2x()
        return
    gen_c2x()
    for T, H, tag in ((8192, 2048, ""), (128, 128, "_cpu")):
        g = docs.dumps(docs.gpt_block_doc(T, H, elem_size=2, train=True))
        for k in (1, 2, 4, 8):
            if tag and k > 1:
                continue
            plan = refpy.compile_plan(g, strategy="megatron_tp", devices=k)
            write(f"c2_tp{k}{tag}", g, plan, dict(config="c2", tokens=T, hidden=H, tp=k, dtype="bf16",
                                                  samples_per_step=T, sample="token (row of X)"))
    # C3: GPT stack, 1F1B pipeline S=4 x inner DP 2 (8 lanes), K=8 micro-batches.
    # (8 layers = 2 per stage keeps the plan ~10^4 tasks; SURVEY §7 "plan scale".)
    for L, T, H, tag in ((8, 32768, 2048, ""), (4, 256, 64, "_cpu")):
        g = docs.dumps(docs.gpt_stack_doc(L, T, H, elem_size=2))
        plan = refpy.compile_plan(g, strategy="1f1b", devices=8, stages=4, micro_batches=8, inner_dp=2)
        write(f"c3_pp4dp2{tag}", g, plan, dict(config="c3", layers=L, tokens=T, hidden=H, stages=4, inner_dp=2,
                                                micro_batches=8, dtype="bf16", samples_per_step=T,
                                                sample="token (row of X)"))
    # C4: co-shard x4 of the FFN-like pair (op1, op2) on one device (Swin stage proxy).
    for B, H, M, tag in ((16384, 512, 2048, ""), (128, 64, 256, "_cpu")):
        g = refpy.with_elem_size(refpy.coshard_doc(batch=B, hidden=H, middle=M), 2)
        plan = refpy.compile_plan(g, strategy="coshard", devices=1, shards=4, target_ops="op1,op2")
        write(f"c4_coshard4{tag}", g, plan, dict(config="c4", batch=B, hidden=H, middle=M, shards=4, dtype="bf16",
                                                  samples_per_step=B, sample="row of the batch"))
    # C5: three chained forward passes + one backward (Evoformer proxy), 3F1B S=2.
    for B, H, tag in ((32768, 256, ""), (128, 32, "_cpu")):
        g = refpy.with_elem_size(refpy.three_pass_doc(layers=4, batch=B, hidden=H), 2)
        plan = refpy.compile_plan(g, strategy="3f1b", devices=2, stages=2, micro_batches=4)
        write(f"c5_3f1b{tag}", g, plan, dict(config="c5", batch=B, hidden=H, stages=2, micro_batches=4,
                                              dtype="bf16", samples_per_step=B, sample="row of the MSA batch"))
    # Unpartitioned single-lane plans of the C3/C4/C5 graphs at full size: the
    # partition-invariance property tests compare the partitioned plans
    # against them (tests/test_fullsize_gpu.py).
    for name, g in (("c3_ref1", docs.dumps(docs.gpt_stack_doc(8, 32768, 2048, elem_size=2))),
                    ("c4_ref1", refpy.with_elem_size(refpy.coshard_doc(batch=16384, hidden=512, middle=2048), 2)),
                    ("c5_ref1", refpy.with_elem_size(refpy.three_pass_doc(layers=4, batch=32768, hidden=256), 2))):
        plan = refpy.compile_plan(g, strategy="none", devices=1)
        write(name, g, plan, dict(config=name[:2], strategy="none", dtype="bf16"))
    for B, H, tag in ((16384, 4096, ""), (128, 128, "_cpu")):
        g = refpy.with_elem_size(refpy.mlp_doc(layers=2, batch=B, hidden=H), 2)
        for k in (1, 2, 4, 8):
            if tag and k > 1:
                continue
            plan = refpy.compile_plan(g, strategy="data_parallel", devices=k)
            write(f"c1l_dp{k}{tag}", g, plan, dict(config="c1l", batch=B, hidden=H, dp=k, dtype="bf16",
                                                   samples_per_step=B, sample="row of the batch"))


if __name__ == "__main__":
    main()
