"""Peer-memory one-process-per-GPU mode on the GPU: several ranks (processes).

Each rank opens the plan with ``planc_b200_open_rank(..., PEER_MEMORY)``, the
ranks all-gather their export blobs over torch.distributed (gloo) and import
them: every rank then maps the other ranks' lane arenas through CUDA IPC,
box kernels read other ranks' pieces in place, and cross-rank dependencies
are device flags with a step-end barrier. All ranks share cuda:0 here (CUDA
IPC works between processes on one device; NVLink between GPUs on the
8-GPU box). Rank 0 reads every rank's pieces through the mappings and the
reassembled plan outputs must equal the reference's — after one step, after
replayed CUDA-graph steps, eagerly, and around the profiling / timeline
paths that issue instructions one at a time.
"""
import json
import os
import socket

import pytest

import golden_cases

pytestmark = pytest.mark.gpu

CASES = ["mlp_dp2", "tp_value_split", "gpt_block_tp2", "gpt_block_tp2_bf16", "adapt_v_to_r4", "adapt_v_to_d4",
         "adapt_d1_to_d0_4", "adapt_d_to_r4", "adapt_r_to_d4", "embed_shard2", "three_pass_3f1b", "mlp_1f1b_dp2",
         "mlp_dp2_naive", "cross_group_rs", "cross_group_copy", "mlp_dp4", "gpt_block_tp4", "gpt_stack2_1f1b_bf16",
         "coshard4_recompute", "embed_interlaced", "ext_block_tp2", "ext_block_tp4", "ext_block_tp2_bf16",
         "gpt_block_fwd_tp2_mma", "ext_block_fwd_tp2_mma"]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, names, flags, result_q):
    import sys
    import traceback

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    sys.path.insert(0, here)
    os.environ["PLANC_B200_PEER_TIMEOUT_S"] = "30"
    import torch.distributed as dist

    import golden_cases as gc
    import paper_2301_08984_b200 as pb

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def exchange(blob):
        out = [None] * world
        dist.all_gather_object(out, blob)
        return out

    report = {}
    try:
        for name in names:
            g = gc.load(name)
            nl = len(json.loads(g["plan"])["lanes"])
            if nl < world:
                continue
            lane_rank = pb.lanes_round_robin(nl, world)
            res = []
            try:
                ex = pb.Executor(g["plan"], flags=flags, rank=rank, world=world, lane_rank=lane_rank, local_gpu=0,
                                 peer_exchange=exchange)
                ex.set_inputs(g["inputs"])
                ex.run(0)
                if rank == 0:
                    res.append(pb.compare_outputs(g["expected"], ex.outputs(), g["meta"]["rel_tol"], normwise=True))
                dist.barrier()
                ex.run(3)  # replayed steps: epochs advance, barrier orders buffer reuse
                ex.profile()
                ex.timeline()
                ex.run(0)
                if rank == 0:
                    res.append(pb.compare_outputs(g["expected"], ex.outputs(), g["meta"]["rel_tol"], normwise=True))
                    res.append((ex.stats()["kernels_per_step"] > 0, "no kernels"))
                dist.barrier()  # nobody unmaps / frees while rank 0 still reads
                ex.close()
            except Exception:
                res.append((False, traceback.format_exc()[-2000:]))
            report[name] = res
    finally:
        result_q.put((rank, report))
        dist.destroy_process_group()


def _run_world(world, names, flags=0):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, names, flags, q)) for r in range(world)]
    for p in procs:
        p.start()
    reports = {}
    for _ in range(world):
        r, rep = q.get(timeout=900)
        reports[r] = rep
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return reports


def _assert_ok(reports, names, world):
    ran = 0
    for name in names:
        nl = len(json.loads(golden_cases.load(name)["plan"])["lanes"])
        if nl < world:
            continue
        ran += 1
        for r, rep in reports.items():
            for ok, msg in rep[name]:
                assert ok, f"{name} (world {world}, rank {r}): {msg}"
    assert ran > 0


@pytest.mark.timeout(1200)
def test_peer_memory_two_ranks():
    reps = _run_world(2, CASES)
    _assert_ok(reps, CASES, 2)


@pytest.mark.timeout(1200)
def test_peer_memory_four_ranks():
    names = [n for n in CASES if len(json.loads(golden_cases.load(n)["plan"])["lanes"]) >= 4]
    reps = _run_world(4, names)
    _assert_ok(reps, names, 4)


@pytest.mark.timeout(900)
def test_peer_memory_launch_modes():
    import paper_2301_08984_b200 as pb

    names = ["gpt_block_tp2", "adapt_v_to_r4", "mlp_1f1b_dp2"]
    for flags in (pb.NO_GRAPH, pb.SERIAL_LANES, pb.NO_FUSION):
        reps = _run_world(2, names, flags)
        _assert_ok(reps, names, 2)


@pytest.mark.slow
@pytest.mark.timeout(1500)
# (c3's 24-layer plan needs ~190 GiB across its ranks without timed-mode
# reuse — one GPU cannot hold 8 ranks of it; c2sp puts the gather prologue
# and the sequence-parallel reduce-scatters on peer memory)
@pytest.mark.parametrize("config,world", [("c2", 8), ("c2sp", 8), ("c5", 8), ("c4", 8)])
def test_peer_memory_bench_under_torchrun(config, world):
    """bench.py under torchrun with the peer-memory transport at full size,
    every rank on cuda:0: persistent tcgen05 GEMMs (all SMs' shared memory)
    interleaved with cross-rank flag waits must not starve each other (a
    programmatic-dependent launch behind a spinning wait once deadlocked the
    8-rank pipeline plan)."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PLANC_B200_BENCH_SAME_GPU="1", PLANC_B200_PEER_TIMEOUT_S="120")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", str(world),
           "--steps", "2", "--warmup", "3", "--config", config]
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=1400)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == world and line["value"] > 0
    assert line["config"]["transport"].startswith("peer memory")
