"""Generates the benchmark plans in plans/ with the UNMODIFIED reference
front end (oracle/_ref: load_graph -> sProgram -> compile -> save_plan).

Plans are the executor's INPUT (what the reference compiler emits); they are
generated once here, where /root/reference exists, and committed — the GPU
box has no reference. Shapes follow SURVEY.md §8d:

  c2   GPT-3-style block (oracle/docs.py gpt_block_doc), train step,
       T=8192 tokens (4 seq x 2048), H=2048, FFN=4H, bf16,
       Megatron TP = 1/2/4/8 (megatron_tp sProgram)
  c1l  2-layer MLP (reference mlp_doc) B=16384, H=4096, bf16, DP = 1/2/4/8
  c4   Swin stage block (docs.swin_stage_doc), 8-way DP x co-shard 4
       (coshard_dp sProgram), 131072 tokens, H=512, bf16
  c5   Evoformer proxy (docs.evoformer_doc), MSA [32768,256] + pair
       [65536,128], 3F1B over 4 stages x 2-way DAP (threef1b_dap), bf16
  c2sp the C2 block under Megatron TP + sequence parallelism (megatron_tp
       "sp" role: residual adds split on the token dim -> reduce-scatter
       after the row-parallel GEMMs, all-gather (send/recv + concat) before
       the column-parallel ones), TP = 2/4/8
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


# C4: Swin stage block (H=512, FFN 2048) as a train step, 16384 tokens per GPU
# x 8-way data parallelism = 131072 tokens; co-shard x4 of the FFN chain on
# every rank (coshard_dp, oracle/ref_capi.cpp). Weight gradients leave the
# ranks as reduce-scatters (attention weights; Dijkstra's pick) or naive
# send/recv + reduce-assemble chains (the co-sharded FFN weights: the
# reference's RVD matcher skips families whose ranks hold several pieces,
# rvd.cpp:825-846); the updated weights come back as all-gathers.
C4_SHAPE = (8 * 16384, 512)
C4_SPEC = dict(strategy="coshard_dp", devices=8, shards=4, target_ops="colf1+tprelu+roww2")
# C5: Evoformer proxy, MSA [32768, 256] + pair [65536, 128], 4 layers, three
# forward passes + one backward, K=4 micro-batches, 3F1B over 4 stages x
# 2-way DAP (threef1b_dap): all-to-all layout switches, reduce-scatter weight
# gradients inside each DAP pair, P2P between stages.
C5_SHAPE = (4, (32768, 256), (65536, 128), 4)
C5_SPEC = dict(strategy="threef1b_dap", devices=8, stages=4, micro_batches=4, inner_dp=2)


def gen_c3_l24():
    """C3 at the GPT-3 1.3B shape: 24 layers (6 per stage), H=2048, 16 x 2048
    tokens, 1F1B S=4 x inner DP 2, K=8. Its step holds ~190 GiB of buffers
    when nothing is freed; the bench runs it with REUSE_MEMORY (the plan's
    free tasks honoured: ~80 GiB)."""
    # (no reduced-shape twin: the reference executor needs ~1 min per step
    # for the 26704-task plan at any shape — per-task lookups, SURVEY fact 10;
    # the CPU baseline of c3 runs c3_pp4dp2_cpu)
    for L, T, H, tag in ((24, 32768, 2048, ""),):
        g = docs.dumps(docs.gpt_stack_doc(L, T, H, elem_size=2))
        plan = refpy.compile_plan(g, strategy="1f1b", devices=8, stages=4, micro_batches=8, inner_dp=2)
        write(f"c3_pp4dp2_l24{tag}", g, plan, dict(config="c3", layers=L, tokens=T, hidden=H, stages=4, inner_dp=2,
                                                    micro_batches=8, dtype="bf16", samples_per_step=T,
                                                    sample="token (row of X)"))


def gen_c4():
    for T, H, tag in (C4_SHAPE + ("",), (8 * 32, 64, "_cpu")):
        g = docs.dumps(docs.swin_stage_doc(T, H))
        plan = refpy.compile_plan(g, **C4_SPEC)
        write(f"c4_coshard4_dp8{tag}", g, plan,
              dict(config="c4", tokens=T, hidden=H, middle=4 * H, shards=4, dp=8, dtype="bf16",
                   samples_per_step=T, sample="token (row of the stage input)", spec=C4_SPEC))


def gen_c5():
    for shape, tag in ((C5_SHAPE, ""), ((4, (512, 32), (1024, 16), 4), "_cpu")):
        L, msa, pair, K = shape
        g = docs.dumps(docs.evoformer_doc(L, msa, pair, K))
        plan = refpy.compile_plan(g, **C5_SPEC)
        write(f"c5_3f1b_dap{tag}", g, plan,
              dict(config="c5", layers=L, msa=list(msa), pair=list(pair), batch=msa[0], hidden=msa[1],
                   micro_batches=K, stages=4, dap=2, dtype="bf16", samples_per_step=msa[0],
                   sample="MSA row (sequence x residue) of the batch", spec=C5_SPEC))


def gen_ref1():
    # Unpartitioned single-lane plans of the C3/C4/C5 graphs at full size: the
    # partition-invariance property tests compare the partitioned plans
    # against them (tests/test_fullsize_gpu.py).
    for name, g in (("c3_ref1", docs.dumps(docs.gpt_stack_doc(8, 32768, 2048, elem_size=2))),
                    ("c4_ref1", docs.dumps(docs.swin_stage_doc(*C4_SHAPE))),
                    ("c5_ref1", docs.dumps(docs.evoformer_doc(*C5_SHAPE)))):
        plan = refpy.compile_plan(g, strategy="none", devices=1)
        write(name, g, plan, dict(config=name[:2], strategy="none", dtype="bf16"))


def gen_c2a():
    """C2a: the block forward with real (fused, causal) attention — 4
    sequences of 2048 tokens, 16 heads of 128 — Megatron TP 1/2/4/8; the
    *_cpu twin (T=256: 2 sequences of 128, H=128, 1 head) and its stand-in
    plan for the reference CPU executor."""
    for T, H, hd, seq, tag in ((8192, 2048, 128, 2048, ""), (256, 128, 128, 128, "_cpu")):
        doc = docs.gpt_block_attn_doc(T, H, hd, seq)
        stand = docs.dumps(docs.standin_doc(doc))
        meta = dict(config="c2a", tokens=T, hidden=H, head=hd, seq=seq, dtype="bf16", samples_per_step=T,
                    sample="token (row of X)", extension=True, note="forward only (inference prefill)")
        for k in (1, 2, 4, 8):
            if tag and k > 1:
                continue
            plan = refpy.compile_plan(stand, strategy="megatron_tp", devices=k)
            write(f"c2a_tp{k}{tag}", docs.dumps(doc), docs.rewrite_plan(plan, doc), dict(meta, tp=k))
            if tag:
                write(f"c2a_tp{k}{tag}_standin", stand, plan, dict(meta, tp=k, standin=True))


def gen_c2at():
    """C2at: the C2a block as a train step (fused attention forward and
    attention-grad, LN / GELU gradients, optimizer), Megatron TP 1/2/4/8, and
    its reduced-shape stand-in twin for the reference CPU executor."""
    for T, H, hd, seq, tag in ((8192, 2048, 128, 2048, ""), (256, 128, 128, 128, "_cpu")):
        doc = docs.gpt_block_attn_train_doc(T, H, hd, seq)
        stand = docs.dumps(docs.standin_doc(doc))
        meta = dict(config="c2at", tokens=T, hidden=H, head=hd, seq=seq, dtype="bf16", samples_per_step=T,
                    sample="token (row of X)", extension=True, note="train step with fused attention and its gradient")
        for k in (1, 2, 4, 8):
            if tag and k > 1:
                continue
            plan = refpy.compile_plan(stand, strategy="megatron_tp", devices=k)
            write(f"c2at_tp{k}{tag}", docs.dumps(doc), docs.rewrite_plan(plan, doc), dict(meta, tp=k))
            if tag:
                write(f"c2at_tp{k}{tag}_standin", stand, plan, dict(meta, tp=k, standin=True))


def gen_c2sp():
    g = docs.dumps(docs.gpt_block_doc(8192, 2048, elem_size=2, train=True, seq_parallel=True))
    for k in (2, 4, 8):
        plan = refpy.compile_plan(g, strategy="megatron_tp", devices=k)
        write(f"c2sp_tp{k}", g, plan, dict(config="c2sp", tokens=8192, hidden=2048, tp=k, dtype="bf16",
                                            samples_per_step=8192, sample="token (row of X)",
                                            parallelism="Megatron TP + sequence parallel"))


def main():
    os.makedirs(OUT, exist_ok=True)
    only = set(sys.argv[1:])
    if only:
        for name, fn in (("c2x", gen_c2x), ("c2sp", gen_c2sp), ("c2a", gen_c2a), ("c2at", gen_c2at), ("c3l24", gen_c3_l24), ("c4", gen_c4), ("c5", gen_c5)):
            if name in only:
                fn()
        if "ref1" in only:
            gen_ref1()
        return
    gen_c2x()
    gen_c2sp()
    gen_c2a()
    gen_c2at()
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
    gen_c3_l24()
    gen_c4()
    gen_c5()
    gen_ref1()
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
