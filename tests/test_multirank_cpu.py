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


# ---- peer-memory transport, emulated on CPU -----------------------------------
# Every rank is a process owning the buffers of its lanes in a shared-memory
# block (the "arena" the GPU ranks export through CUDA IPC) plus a flag block
# (ready slots + step barrier). Each rank walks the GLOBAL program of
# describe(plan, lane_rank, PEER_MEMORY) in issue order, running only its own
# lanes' instructions: before one it spins until its ready slots reach the
# step epoch, it reads other ranks' pieces in place from their blocks, after
# one it writes the epoch into the consumers' slots (peer_sync signals) — the
# exact schedule the GPU ranks run as flag kernels. Two steps (epochs 1, 2)
# with the step-end barrier; rank 0 then reassembles every output by reading
# all ranks' blocks and compares with the reference, bit-exact.

PEER_CASES = ["mlp_dp2", "tp_value_split", "gpt_block_tp2", "adapt_v_to_r4", "adapt_v_to_d4", "adapt_d1_to_d0_4",
              "embed_shard2", "three_pass_3f1b", "mlp_1f1b_dp2", "cross_group_rs", "mlp_dp2_naive", "ext_block_tp2",
              "gpt_block_fwd_tp2_mma"]


def _peer_worker(rank, world, port, names, result_q):
    import sys
    import time
    from multiprocessing import shared_memory

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    sys.path.insert(0, here)
    import golden_cases as gc
    import paper_2301_08984_b200 as pb
    from program_emu import buffer_shapes, exec_instr, reassemble

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    report = {}
    try:
        for name in names:
            g = gc.load(name)
            plan = json.loads(g["plan"])
            lane_rank = pb.lanes_round_robin(len(plan["lanes"]), world)
            desc = pb.describe(g["plan"], lane_rank=lane_rank, flags=pb.PEER_MEMORY)
            ps = desc["peer_sync"]
            owner = lambda b: lane_rank[desc["buffers"][b]["lane"]]  # noqa: E731
            elems = {b["id"]: int(np.prod([hi - lo for lo, hi in b["region"]])) for b in desc["buffers"]}
            mine = [b["id"] for b in desc["buffers"] if owner(b["id"]) == rank]
            offs, total = {}, 0
            for b in mine:
                offs[b] = total
                total += elems[b]
            nflags = 64 + world + max(ps["slots"]) + 1  # [0] epoch, [64 + r] barrier of rank r, then ready slots
            arena = shared_memory.SharedMemory(create=True, size=max(8, 8 * total))
            flags = shared_memory.SharedMemory(create=True, size=8 * nflags)
            np.ndarray((nflags,), np.int64, flags.buf)[:] = 0
            names_all = [None] * world
            dist.all_gather_object(names_all, (arena.name, flags.name, offs))  # the IPC blob exchange
            arenas = {rank: (arena, offs)}
            fl = {rank: flags}
            for r, (an, fn, of) in enumerate(names_all):
                if r != rank:
                    arenas[r] = (shared_memory.SharedMemory(name=an), of)
                    fl[r] = shared_memory.SharedMemory(name=fn)
            F = {r: np.ndarray((nflags,), np.int64, fl[r].buf) for r in fl}

            def view(b):
                shm, of = arenas[owner(b)]
                return np.ndarray((elems[b],), np.float64, shm.buf, offset=8 * of[b])

            for bd in desc["buffers"]:  # placement of this rank's graph inputs
                if bd["graph_input"] and owner(bd["id"]) == rank:
                    x = np.asarray(g["inputs"][bd["pt"]], dtype=np.float64)
                    view(bd["id"])[:] = x[tuple(slice(lo, hi) for lo, hi in bd["region"])].reshape(-1)
            shape = buffer_shapes(desc)
            waited = signalled = 0
            for epoch in (1, 2):
                F[rank][0] = epoch
                for iid in desc["issue_order"]:
                    ins = desc["instrs"][iid]
                    if ins["kind"] == "nop" or lane_rank[ins["lane"]] != rank:
                        continue
                    for slot in ps["waits"][iid]:
                        t0 = time.time()
                        while F[rank][64 + world + slot] < epoch:
                            assert time.time() - t0 < 60, f"{name}: rank {rank} stuck at instr {iid} slot {slot}"
                            time.sleep(0.0002)
                        waited += 1
                    data = {b: view(b) for b in set(ins["in"]) | set(ins["out"]) |
                            {t["buf"] for c in ins["cells"] for t in c["terms"]} |
                            {x for f in ins.get("fused", []) for x in f["in"] + [f["out"]]}}
                    exec_instr(ins, data, shape)
                    outs = list(ins["out"]) + [f["out"] for f in ins.get("fused", [])]
                    for b in outs:  # own pieces, or (reduce-scatter epilogue) slices stored into a peer's block
                        view(b)[:] = data[b]
                    for r, slot in ps["signals"][iid]:
                        F[r][64 + world + slot] = epoch
                        signalled += 1
                for r in range(world):  # step-end barrier
                    F[r][64 + rank] = epoch
                for r in range(world):
                    t0 = time.time()
                    while F[rank][64 + r] < epoch:
                        assert time.time() - t0 < 60, f"{name}: rank {rank} stuck in the barrier"
                        time.sleep(0.0002)
            if rank == 0:
                allbufs = {bd["id"]: view(bd["id"]).copy() for bd in desc["buffers"]}
                out = reassemble(desc, plan, allbufs)
                tol = g["meta"]["rel_tol"]
                ok, msg = pb.compare_outputs(g["expected"], out, tol, normwise=tol > 0)
                report[name] = (ok, msg, waited, signalled)
            dist.barrier()  # nobody unlinks while rank 0 reads
            for r in arenas:
                arenas[r][0].close()
                fl[r].close()
            arena.unlink()
            flags.unlink()
    finally:
        if rank == 0:
            result_q.put(report)
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_rank_peer_memory_protocol_matches_reference():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, 2, port, PEER_CASES, q)) for r in range(2)]
    for p in procs:
        p.start()
    report = q.get(timeout=500)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for name in PEER_CASES:
        ok, msg, waited, signalled = report[name]
        assert ok, f"{name}: {msg}"
        assert waited > 0 and signalled > 0, f"{name}: no cross-rank edge exercised"
