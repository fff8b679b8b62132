"""Runs golden plans (eager issue) for compute-sanitizer sweeps:
  compute-sanitizer --tool memcheck  python tools/sanitize.py
  compute-sanitizer --tool racecheck python tools/sanitize.py
  compute-sanitizer --tool synccheck python tools/sanitize.py
Covers the SIMT and tcgen05 GEMM variants (default, two CTAs per SM,
cluster pairs, split-K, 8 epilogue warps, fused epilogues), the row-wise
extension kernels, box adapters and — through one-rank peer mode — the
reduce-scatter GEMM epilogue and the flag kernels. Checks results too, so a
sanitizer-clean run is also a correct one."""
import json
import os
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import golden_cases  # noqa: E402
import paper_2301_08984_b200 as pb  # noqa: E402

CASES = sys.argv[1:] or ["mlp_dp2", "gpt_block_tp2", "embed_shard2", "adapt_d1_to_d0_4", "gpt_block_fwd_tp2_mma",
                         "mlp_1f1b_dp2", "ext_block_tp2", "ext_block_fwd_tp2_mma", "coshard4_recompute"]
VARIANTS = [{}, {"PLANC_B200_OCC2": "2"}, {"PLANC_B200_CLUSTER": "2", "PLANC_B200_EPI8": "0"},
            {"PLANC_B200_SPLITK": "2", "PLANC_B200_STREAMK": "0"}, {"PLANC_B200_EPI8": "2"}]
bad = 0


def check(name, ex, g, tag):
    global bad
    ok, msg = pb.compare_outputs(g["expected"], ex.outputs(), g["meta"]["rel_tol"], normwise=True)
    print(name, tag, "ok" if ok else msg, flush=True)
    bad += not ok


for name in CASES:
    g = golden_cases.load(name)
    n = len(json.loads(g["plan"])["lanes"])
    for env in (VARIANTS if "mma" in name else [{}]):
        os.environ.update(env)
        with pb.Executor(g["plan"], lane_gpus=[0] * n, flags=pb.NO_GRAPH) as ex:
            ex.set_inputs(g["inputs"])
            ex.run(1)
            check(name, ex, g, ",".join(f"{k[11:]}={v}" for k, v in env.items()) or "default")
        for k in env:
            os.environ.pop(k)
    if "mma" in name:  # one-rank peer mode: scatter epilogue + flag kernels
        with pb.Executor(g["plan"], flags=pb.NO_GRAPH, rank=0, world=1, lane_rank=[0] * n, local_gpu=0,
                         peer_exchange=lambda blob: [blob]) as ex:
            ex.set_inputs(g["inputs"])
            ex.run(1)
            check(name, ex, g, "peer")
sys.exit(1 if bad else 0)
