"""One-process-per-GPU path on CPU: world_size 2 over gloo.

Each rank lowers the plan with ``describe(plan, lane_rank=...)`` (the same
C++ localisation the GPU ranks use), interprets only its own lanes, and
moves cross-rank pieces at every ``xfer`` exchange step with gloo
point-to-point operations — exactly the sends/receives the GPU ranks post to
NCCL at that step. Rank 0 gathers every rank's buffers, reassembles the plan
outputs and compares them with the reference (bit-exact).
"""
import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import golden_cases

CASES = ["mlp_dp2", "mlp_dp2_naive", "tp_value_split", "gpt_block_tp2", "adapt_d1_to_d0_4", "adapt_v_to_d4",
         "embed_shard2", "three_pass_3f1b", "mlp_1f1b_dp2", "cross_group_rs", "adapt_d_to_r4"]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, names, result_q):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    sys.path.insert(0, here)
    import golden_cases as gc
    import paper_2301_08984_b200 as pb
    from program_emu import reassemble, run_program

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        report = {}
        for name in names:
            g = gc.load(name)
            plan = json.loads(g["plan"])
            lane_rank = pb.lanes_round_robin(len(plan["lanes"]), world)
            desc = pb.describe(g["plan"], lane_rank=lane_rank)
            owned = {l for l, r in enumerate(lane_rank) if r == rank}
            n_steps = [0]

            def exchange(ins, data):
                if ins["allreduce"]:  # ncclAllReduce over the world: one member per rank
                    mine = [x for x in ins["xfers"] if lane_rank[x["src_lane"]] == rank]
                    assert len(mine) == 1
                    t = torch.from_numpy(data[mine[0]["src"]].copy())
                    dist.all_reduce(t)
                    data[mine[0]["dst"]] = t.numpy().copy()
                    n_steps[0] += 1
                    return
                ops, recvs = [], []
                for x in ins["xfers"]:
                    src_r, dst_r = lane_rank[x["src_lane"]], lane_rank[x["dst_lane"]]
                    if src_r == rank and dst_r != rank:
                        ops.append(dist.P2POp(dist.isend, torch.from_numpy(data[x["src"]].copy()), dst_r))
                    elif dst_r == rank and src_r != rank:
                        t = torch.empty(data[x["dst"]].shape[0], dtype=torch.float64)
                        ops.append(dist.P2POp(dist.irecv, t, src_r))
                        recvs.append((x["dst"], t))
                if ops:
                    for req in dist.batch_isend_irecv(ops):
                        req.wait()
                    n_steps[0] += 1
                for b, t in recvs:
                    data[b] = t.numpy().copy()

            data = run_program(desc, plan, g["inputs"], owned_lanes=owned, exchange=exchange, return_buffers=True)
            mine = {b["id"]: data[b["id"]] for b in desc["buffers"] if b["lane"] in owned}
            gathered = [None] * world if rank == 0 else None
            dist.gather_object(mine, gathered, dst=0)
            if rank == 0:
                allbufs = {}
                for part in gathered:
                    allbufs.update(part)
                out = reassemble(desc, plan, allbufs)
                ok = all(np.array_equal(g["expected"][k], out[k]) for k in g["expected"])
                bad = [k for k in g["expected"] if not np.array_equal(g["expected"][k], out[k])]
                report[name] = (ok, bad, n_steps[0], sum(1 for i in desc["instrs"] if i["kind"] == "xfer"))
        if rank == 0:
            result_q.put(report)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_exchange_schedule_matches_reference():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, CASES, q)) for r in range(2)]
    for p in procs:
        p.start()
    report = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for name in CASES:
        ok, bad, steps, xfers = report[name]
        assert ok, f"{name}: tensors {bad} differ"
        assert xfers > 0 and steps > 0, f"{name}: no cross-rank exchange exercised"


def test_localised_program_invariants():
    import paper_2301_08984_b200 as pb

    for name in CASES:
        g = golden_cases.load(name)
        plan = json.loads(g["plan"])
        lane_rank = pb.lanes_round_robin(len(plan["lanes"]), 2)
        desc = pb.describe(g["plan"], lane_rank=lane_rank)
        for ins in desc["instrs"]:
            if ins["kind"] == "box":
                # after localisation every term lives on the consumer's rank
                for c in ins["cells"]:
                    for t in c["terms"]:
                        assert lane_rank[desc["buffers"][t["buf"]]["lane"]] == lane_rank[ins["lane"]]
            if ins["kind"] == "xfer":
                for x in ins["xfers"]:
                    if ins["allreduce"]:
                        assert x["src_lane"] == x["dst_lane"]  # one member per rank
                    else:
                        assert lane_rank[x["src_lane"]] != lane_rank[x["dst_lane"]]
                    assert desc["buffers"][x["dst"]]["bytes"] == x["bytes"]
                if ins["allreduce"]:
                    assert sorted(lane_rank[x["src_lane"]] for x in ins["xfers"]) == [0, 1]
        # single-rank ownership needs no exchange at all
        solo = pb.describe(g["plan"], lane_rank=[0] * len(plan["lanes"]))
        assert not any(i["kind"] == "xfer" for i in solo["instrs"])
