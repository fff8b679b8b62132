#!/usr/bin/env python3
"""Plan-step benchmark of the B200 SuperScaler plan executor.

Metric (BASELINE.json): plan-step samples/sec at 1/2/4/8 B200 (% roofline),
adapter bus GB/s vs NVLink. A step is one execution of every lane's tasks of
a plan emitted by the reference front end (plans/*.plan.json); samples are
rows of the graph's batch dimension (tokens for C2).

Default workload (configs[1]): GPT-3-style transformer block,
Megatron tensor-parallel plan, train step (forward + backward + optimizer),
T=8192 tokens, H=2048, FFN=4H, bf16; TP degree = number of GPUs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c1l]
  python bench.py --impl reference ...   # the reference's CPU run_plan

Multi-GPU: under torchrun one process per GPU — rank r runs plan lane r on
LOCAL_RANK's GPU. Transport (--transport): `peer` (default) maps every
other rank's lane arenas through CUDA IPC, so adapter box kernels read the
peer GPU's pieces in place over NVLink (all-reduces as a reduce-scatter
phase + an all-gather phase) and cross-rank order is kept by device flags;
`nccl` moves whole pieces in NCCL exchange steps (all-reduce groups as
ncclAllReduce). Times are the max over ranks (CUDA events per rank).
Without torchrun, --gpus N drives N GPUs from one process (lanes read each
other's buffers over NVLink peer mappings). Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PLANS = os.path.join(ROOT, "plans")


def plan_name(config: str, n: int) -> str:
    """c2 / c1l plans are compiled per GPU count (TP / DP degree n); the
    pipeline (c3: pp4 x dp2), co-shard x DP (c4: dp8 x co-shard 4) and 3F1B
    x DAP (c5: 4 stages x dap 2) plans have 8 lanes — with fewer GPUs, lanes
    share GPUs (round robin)."""
    return {"c2": f"c2_tp{n}", "c2x": f"c2x_tp{n}", "c1l": f"c1l_dp{n}", "c3": "c3_pp4dp2_l24", "c4": "c4_coshard4_dp8",
            "c5": "c5_3f1b_dap", "c2sp": f"c2sp_tp{max(n, 2)}", "c2a": f"c2a_tp{n}",
            "c2at": f"c2at_tp{n}"}[config]


def nvlink_peer_bandwidth(nbytes: int = 512 << 20, reps: int = 5):
    """Peer copy bandwidth GPU 0 -> GPU 1 (and both directions at once) over
    NVLink with CUDA events: the measured ceiling beside the nominal 900 GB/s
    per direction that adapter_bus_gbs is reported against. None with fewer
    than two visible GPUs."""
    import torch

    if torch.cuda.device_count() < 2:
        return {"value": None, "note": "fewer than two visible GPUs"}
    a0 = torch.empty(nbytes, dtype=torch.uint8, device="cuda:0")
    b1 = torch.empty(nbytes, dtype=torch.uint8, device="cuda:1")
    a1 = torch.empty(nbytes, dtype=torch.uint8, device="cuda:1")
    b0 = torch.empty(nbytes, dtype=torch.uint8, device="cuda:0")
    s1 = torch.cuda.Stream(device="cuda:1")
    out = {}
    for name in ("uni", "bidir"):
        best = 0.0
        for _ in range(reps):
            torch.cuda.synchronize(0)
            torch.cuda.synchronize(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(torch.cuda.current_stream(0))
            b1.copy_(a0, non_blocking=True)
            if name == "bidir":
                with torch.cuda.stream(s1):
                    b0.copy_(a1, non_blocking=True)
                torch.cuda.current_stream(0).wait_stream(s1)
            e1.record(torch.cuda.current_stream(0))
            e1.synchronize()
            moved = nbytes * (2 if name == "bidir" else 1)
            best = max(best, moved / (e0.elapsed_time(e1) / 1e3) / 1e9)
        out[name] = round(best, 1)
    return {"value": out["uni"], "bidir_gbs": out["bidir"], "unit": "GB/s", "nbytes": nbytes,
            "via": "torch peer copy cuda:0 -> cuda:1 (CUDA events, best of %d)" % reps}


def cpu_plan_name(config: str) -> str:
    """Reduced-shape twin of the config's plan for the reference CPU executor
    (SURVEY §8d). c3's 24-layer plan has none (the reference needs ~1 min per
    step for its 26704 tasks at any shape): the 4-layer stack under the same
    1F1B pp4 x dp2 strategy stands in."""
    if config == "c3":
        return "c3_pp4dp2_cpu"
    if config == "c2sp":
        return "c2_tp1_cpu"  # the same graph (sequence parallelism only renames the residual ops' split)
    return plan_name(config, 1) + "_cpu" + ("_standin" if config in ("c2x", "c2a", "c2at") else "")


def load_plan(name):
    path = os.path.join(PLANS, name + ".plan.json")
    if os.path.exists(path):
        with open(path) as f:
            plan = f.read()
    else:  # large plans are stored gzipped
        import gzip

        with gzip.open(path + ".gz", "rt") as f:
            plan = f.read()
    with open(os.path.join(PLANS, name + ".meta.json")) as f:
        meta = json.load(f)
    return plan, meta


def synthetic_inputs(plan_json: str, seed: int = 0, only=None) -> dict:
    """Full-entropy inputs for every graph-input pTensor (or the ids in
    ``only``: one rank's inputs): weights N(0, 1/fan_in), activations and
    incoming gradients N(0, 0.1^2) — random mantissas (low-entropy operands
    would understate tensor-core power draw), magnitudes that stay finite in
    bf16 through the stacked blocks. Each tensor draws from its own seeded
    stream, so a rank's subset equals the same tensors of the full set."""
    p = json.loads(plan_json)
    produced = set()
    vts = {v["id"]: v for v in p["vtensors"]}
    for o in p["ops"]:
        for v in o["outputs"]:
            produced.add(vts[v]["ptensor"])
    out = {}
    for pt in p["ptensors"]:
        if pt["id"] in produced or (only is not None and pt["id"] not in only):
            continue
        x = np.random.default_rng([seed, pt["id"]]).standard_normal(pt["shape"])
        out[pt["id"]] = x / np.sqrt(pt["shape"][0]) if pt["kind"] == "weight" else 0.1 * x
    return out


DATA_NOTE = "synthetic: weights N(0,1/fan_in), activations / gradients N(0,0.01), full-entropy bf16 mantissas"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = gpus
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        # One continuously sampling nvidia-smi (every 50 ms) for the timed region.
        cmd = ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "50",
               "-i", ",".join(map(str, self.gpus))]
        try:
            self._proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            return
        for line in self._proc.stdout:
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                self.samples.append(f)
            if self._stop.is_set():
                break

    def __enter__(self):
        self._proc = None
        self._t = None
        if not self.gpus:  # only rank 0 samples
            return self
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        deadline = time.time() + 3.0
        while not self.samples and time.time() < deadline:  # sampler is live before timing starts
            time.sleep(0.01)
        return self

    def __exit__(self, *a):
        if self._t is None:
            return
        time.sleep(0.06)  # at least one sample after the timed region ends
        self._stop.set()
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()
        self._t.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return dict(hbm=j["hbm_gbs"], bf16=j["bf16_tflops"], bf16_sus=j["bf16_tflops_sustained"], src="measured")
    except Exception:
        return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback")


NVLINK_GBS = 900.0  # nominal per direction per GPU (measured peer copy 770)


def pcie_bandwidth(device: int, nbytes: int = 256 << 20, reps: int = 3):
    """Measured pinned host<->device copy bandwidth (GB/s) of this GPU's link:
    the bound of the end-to-end arm, whose steps move their inputs / results
    across it."""
    import torch

    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{device}")
    out = {}
    for name, (dst, src) in (("h2d", (d, h)), ("d2h", (h, d))):
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize(device)
        best = 0.0
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            dst.copy_(src, non_blocking=True)
            b.record()
            b.synchronize()
            best = max(best, nbytes / (a.elapsed_time(b) / 1e3) / 1e9)
        out[name] = best
    return out


def cpu_baseline(config: str, budget_s: float = 20.0):
    """The reference's own CPU executor (oracle/_ref run_plan, 1 thread) on the
    reduced-shape plan of the same graph, bounded in time."""
    from oracle import refpy  # checker / baseline only

    name = cpu_plan_name(config)
    note = ""
    if config in ("c2x", "c2a", "c2at"):
        # The reference executor has no layernorm / softmax / GELU / attention:
        # it runs the stand-in plan (identity / mul / add in their place, same data flow).
        note = "; stand-in plan: identity/mul/add where the extension has LN/softmax/GELU/attention"
    if config == "c3":
        note = "; 4-layer stack (the 24-layer plan takes the reference ~1 min per step)"
    plan, meta = load_plan(name)
    inputs = synthetic_inputs(plan, 1)
    _, secs = refpy.run_plan(plan, inputs, iters=1)
    iters = max(1, min(50, int(budget_s / max(secs, 1e-6))))
    _, secs = refpy.run_plan(plan, inputs, iters=iters)
    sps = meta["samples_per_step"] / secs
    return dict(value=sps, unit="samples/s", cores=1, host_cores=os.cpu_count(), kind="reference",
                sample=f"{iters} x run_plan of {name} ({shape_str(meta)}, same graph at reduced shape; "
                       f"{secs:.3f} s/step, single-threaded reference executor{note})"), secs


def shape_str(meta):
    keys = [k for k in ("tokens", "batch", "hidden", "msa", "pair", "layers") if k in meta]
    return ",".join(f"{k}={meta[k]}" for k in keys)


def run_reference_arm(args, rank, world):
    """--impl reference: the reference's CPU executor (oracle/_ref run_plan,
    the unmodified refexec.cpp) on the reduced-shape plan of the same graph,
    with every host thread: a step is one run_plan per thread, concurrently
    (run_plan is single-threaded and reentrant), so samples/s is
    the host's whole-CPU throughput. Exactly --warmup + --steps steps run."""
    if rank != 0:
        return
    from concurrent.futures import ThreadPoolExecutor

    from oracle import refpy  # reference arm only

    name = cpu_plan_name(args.config)
    plan, meta = load_plan(name)
    inputs = synthetic_inputs(plan, 1)
    threads = os.cpu_count() or 1
    calls = 0

    def one(_):
        refpy.run_plan(plan, inputs, iters=1)  # ctypes releases the GIL for the call

    with ThreadPoolExecutor(threads) as pool:
        for _ in range(args.warmup):
            list(pool.map(one, range(threads)))
            calls += threads
        t0 = time.perf_counter()
        for _ in range(args.steps):
            list(pool.map(one, range(threads)))
            calls += threads
        secs = (time.perf_counter() - t0) / max(args.steps, 1)
    value = threads * meta["samples_per_step"] / secs
    sample = (f"{args.warmup} + {args.steps} steps, each {threads} concurrent run_plan calls (one per host thread) "
              f"of {name} ({shape_str(meta)}, same graph at reduced shape); {calls} run_plan calls in total")
    line = {"metric": "plan step samples/sec", "value": value, "unit": "samples/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": DATA_NOTE, "config": {"workload": name, "config": args.config},
            "cpu_baseline": {"value": value, "unit": "samples/s", "cores": threads, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def dropin_e2e(ex, inputs, samples_per_step, steps=2):
    """The run_plan(plan, TensorMap) contract end to end through the C ABI
    (refexec.cpp:361-557): every graph input handed over as float64 host
    data (planc_b200_set_input: region placement + conversion), one step,
    every produced pTensor reassembled in float64 on the host
    (planc_b200_get_output). Timed on the host clock around whole calls."""
    ids = ex.output_ids()
    h2d = sum(v.nbytes for v in inputs.values())
    # the caller's TensorMap storage, allocated (and first touched) once
    outs = {i: np.zeros(ex.shape(i), dtype=np.float64) for i in ids}

    split = {"set_input_ms": 0.0, "run_ms": 0.0, "get_output_ms": 0.0}

    def once():
        t0 = time.perf_counter()
        ex.set_inputs(inputs)
        t1 = time.perf_counter()
        ex.run(0)
        t2 = time.perf_counter()
        n = sum(ex.get_output(i, outs[i]).nbytes for i in ids)
        t3 = time.perf_counter()
        for k, v in zip(split, (t1 - t0, t2 - t1, t3 - t2)):
            split[k] += v * 1e3 / steps
        return n

    once()
    split = dict.fromkeys(split, 0.0)
    t0 = time.perf_counter()
    for _ in range(steps):
        d2h = once()
    ms = (time.perf_counter() - t0) / steps * 1e3
    return {"value": samples_per_step / (ms / 1e3), "unit": "samples/s", "ms_per_step": ms, "steps": steps,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "split": split,
            "via": "planc_b200_set_input (float64 TensorMap) -> planc_b200_run -> planc_b200_get_output "
                   "(every produced pTensor, float64, into the caller's reused arrays): the reference "
                   "run_plan contract"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=["c2", "c2x", "c1l", "c3", "c4", "c5", "c2sp", "c2a", "c2at"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sustain-s", type=float, default=3.0, help="seconds of the sustained timed region")
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"],
                    help="one-process-per-GPU data path (torchrun): CUDA-IPC peer memory or NCCL exchange steps")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    dist = None
    if world > 1:
        import torch.distributed as dist  # noqa: F811

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo")

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    n = args.gpus
    name = plan_name(args.config, n)
    plan, meta = load_plan(name)
    result = None
    import paper_2301_08984_b200 as pb

    peaks = measured_peaks()
    nlanes = len(json.loads(plan)["lanes"])
    transport = None
    # C3 at 24 layers holds ~190 GiB of step buffers when nothing is freed:
    # one process driving every lane runs it honouring the plan's frees
    # (REUSE_MEMORY, ~80 GiB). One process per GPU holds 1/N of the lanes.
    reuse_flags = pb.REUSE_MEMORY if (args.config == "c3" and not dist) else 0
    reuse_flags |= int(os.environ.get("PLANC_B200_BENCH_FLAGS", "0"), 0)  # A/B experiments only
    if dist:
        # One process per GPU: this rank runs lanes l with l % world == rank
        # on its local GPU; cross-rank pieces move over NVLink (peer memory or
        # NCCL).
        import torch

        local = int(os.environ.get("LOCAL_RANK", rank))
        if os.environ.get("PLANC_B200_BENCH_SAME_GPU"):  # test hook: every rank on GPU 0
            local = 0
        torch.cuda.set_device(local)
        lane_rank = pb.lanes_round_robin(nlanes, world)
        transport = args.transport
        ex = None
        if transport == "peer":
            def exchange(blob):
                out = [None] * world
                dist.all_gather_object(out, blob)
                return out

            try:
                ex = pb.Executor(plan, rank=rank, world=world, lane_rank=lane_rank, local_gpu=local,
                                 peer_exchange=exchange)
            except pb.PlancError as e:  # e.g. no CUDA IPC between these GPUs
                transport = "nccl (peer memory unavailable: %s)" % str(e)[:120]
            ok = torch.tensor([1 if ex is not None else 0])
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if ok.item() == 0 and ex is not None:
                ex.close()
                ex = None
                transport = "nccl (peer memory unavailable on another rank)"
        if ex is None:
            box = [pb.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(box, src=0)
            ex = pb.Executor(plan, rank=rank, world=world, lane_rank=lane_rank, local_gpu=local, nccl_id=box[0])
    else:
        ex = pb.Executor(plan, lane_gpus=list(range(n)), flags=reuse_flags)
    # each rank generates and binds only the inputs its lanes place
    inputs = synthetic_inputs(plan, only=set(ex.input_ids()))
    ex.set_inputs(inputs)
    ex.run(args.warmup)  # warm-up (graph capture + W steps)
    st = ex.stats()

    def max_over_ranks(v):
        if not dist:
            return v
        import torch

        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    if dist:
        dist.barrier()
    with ClockSampler(list(range(n)) if rank == 0 else []) as clk:
        ms = ex.run(args.steps)
    ms = max_over_ranks(ms)
    clocks = clk.summary()
    e2e_ms, h2d, d2h = ex.run_e2e(args.steps)
    e2e_ms = max_over_ranks(e2e_ms)
    # Sustained: a seconds-long timed region (power / clocks settle), clocks
    # sampled throughout.
    sus_iters = max(args.steps, int(args.sustain_s * 1e3 / max(ms, 1e-3)))
    if dist:
        dist.barrier()
    with ClockSampler(list(range(n)) if rank == 0 else []) as clk2:
        sus_ms = ex.run(sus_iters)
    sus_ms = max_over_ranks(sus_ms)
    sustained = {"ms_per_step": sus_ms, "steps": sus_iters, "seconds": sus_ms * sus_iters / 1e3,
                 "value": meta["samples_per_step"] / (sus_ms / 1e3), "clocks": clk2.summary()}
    dropin = None
    if not dist and not reuse_flags:  # one process owns every lane: the whole TensorMap round trip
        dropin = dropin_e2e(ex, inputs, meta["samples_per_step"])
    prof = [ex.profile() for _ in range(3)]  # every rank: exchange steps pair up
    if dist:
        dist.barrier()  # peer memory: no rank unmaps / frees while another still reads
    ex.close()
    e2e_bound = {}
    if rank == 0:
        try:  # the link bound of the e2e arm: max(H2D, D2H, device step) with copies overlapped
            bw = pcie_bandwidth(int(os.environ.get("LOCAL_RANK", 0)) if dist else 0)
            t_link = max(h2d / (bw["h2d"] * 1e9), d2h / (bw["d2h"] * 1e9)) * 1e3
            e2e_bound = {"pcie_gbs": {k: round(v, 1) for k, v in bw.items()},
                         "bound_ms": max(t_link, ms), "frac_of_bound": max(t_link, ms) / e2e_ms}
        except Exception as e:  # torch / pinned memory unavailable
            e2e_bound = {"pcie_gbs": None, "note": str(e)[:100]}
    if rank == 0:
        sps = meta["samples_per_step"] / (ms / 1e3)
        # Dominant kernel (largest share of the serialised step) and its roofline.
        fam = {}
        for pr in prof:
            for p in pr:
                f = fam.setdefault(p["kind"], dict(ms=0.0, launches=0, flops=0.0, bytes=0.0, wire=0.0))
                f["ms"] += p["ms"] / len(prof)
                f["launches"] += p["launches"] / len(prof)
                f["flops"] += p["flops"] / len(prof)
                f["bytes"] += p["bytes"] / len(prof)
                f["wire"] += p["wire_bytes"] / len(prof)
        total_prof = sum(f["ms"] for f in fam.values())
        top = max(fam, key=lambda k: fam[k]["ms"])
        t = fam[top]
        # DRAM traffic per launch of the dominant kernel from the committed
        # ncu --set full capture of this workload (profiles/latest_traffic.json).
        traffic, traffic_src = None, None
        try:
            with open(os.path.join(ROOT, "profiles", "latest_traffic.json")) as f:
                tj = json.load(f)
            if args.config == "c2" and n == 1 and top in tj:
                traffic, traffic_src = tj[top]["mean"], tj["source"]
        except Exception:
            pass
        if top.startswith("gemm") or top.startswith("attention"):
            achieved = t["flops"] / (t["ms"] / 1e3) / 1e12
            # fused elementwise epilogues add their operand / result bytes at
            # HBM speed to the tensor-bound time (0 without fusion)
            t_bound_s = t["flops"] / (peaks["bf16"] * 1e12) + t["bytes"] / (peaks["hbm"] * 1e9)
            roof = {"kernel": top, "bound": "tensor (+ fused-epilogue bytes at HBM)", "achieved": achieved,
                    "peak": peaks["bf16"], "unit": "TFLOP/s", "frac": t_bound_s / (t["ms"] / 1e3),
                    "frac_tensor_only": achieved / peaks["bf16"],
                    "fused_epilogue_gb_per_step": t["bytes"] / 1e9, "traffic": traffic,
                    "traffic_source": traffic_src,
                    "peak_source": peaks["src"] + " burst (kernels timed individually)",
                    "share_of_step": t["ms"] / total_prof,
                    "per_launch": {"flops": t["flops"] / max(t["launches"], 1),
                                   "ms": t["ms"] / max(t["launches"], 1)}}
        else:
            achieved = t["bytes"] / (t["ms"] / 1e3) / 1e9
            roof = {"kernel": top, "bound": "hbm", "achieved": achieved, "peak": peaks["hbm"], "unit": "GB/s",
                    "frac": achieved / peaks["hbm"], "traffic": None, "peak_source": peaks["src"],
                    "share_of_step": t["ms"] / total_prof}
        # Plan-level roofline: max over GPUs of
        # F/P + M/HBM vs W/NVLink, against the measured sustained peaks, from
        # the host lowering's per-instruction algorithmic work. Lanes sharing
        # a GPU add up; their adapter bytes then stay in HBM (no NVLink).
        # algorithmic work of the PLAN (every elementwise op and copy counted,
        # whatever the executor fuses, groups or aliases)
        desc = pb.describe(plan, flags=pb.NO_FUSION | pb.NO_GROUPING | pb.NO_GATHER)
        gpu_of = [lane % n for lane in range(nlanes)]
        F, M, W = [0.0] * n, [0.0] * n, [0.0] * n
        for ins in desc["instrs"]:
            gidx = gpu_of[ins["lane"]]
            if ins["kind"] in ("gemm", "attention"):  # tensor-core work (attention: QK^T and PV, and its gradient)
                F[gidx] += ins["flops"]
                if ins["kind"] == "attention":
                    M[gidx] += ins["bytes"]
            else:
                M[gidx] += ins["bytes"]
            if n > 1:
                W[gidx] += ins["wire_bytes"]
        t_roof = max(max(F[i] / (peaks["bf16_sus"] * 1e12) + M[i] / (peaks["hbm"] * 1e9),
                         W[i] / (NVLINK_GBS * 1e9)) for i in range(n))
        families = {k: {"ms": round(v["ms"], 4), "launches": v["launches"],
                        "tflops" if k.startswith(("gemm", "attention")) else "gbs":
                            round((v["flops"] / 1e12 if k.startswith(("gemm", "attention")) else v["bytes"] / 1e9)
                                  / max(v["ms"] / 1e3, 1e-12), 2)} for k, v in fam.items()}
        # Adapter bus bandwidth: wire bytes (NCCL bus-bandwidth convention) of
        # the cross-GPU adapter launches over their device time.
        adapters = [fam[k] for k in ("box_collective", "box_p2p", "xfer_nccl") if k in fam]
        coll = None
        if adapters:
            coll = {"wire": sum(a["wire"] for a in adapters), "ms": sum(a["ms"] for a in adapters)}
        result = {
            "metric": "plan step samples/sec", "value": sps, "unit": "samples/s", "n_gpus": n,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": DATA_NOTE,
            "config": {"workload": name, "config": args.config, "plan": f"plans/{name}.plan.json",
                       "shape": {k: meta[k] for k in ("tokens", "batch", "hidden", "middle", "layers", "head", "msa", "pair",
                                                                  "micro_batches") if k in meta},
                       "parallelism": {"c2": f"tp{n}", "c2x": f"tp{n}", "c1l": f"dp{n}", "c3": "pp4 x dp2 (1F1B, K=8)",
                                       "c2sp": f"tp{max(n, 2)} + sequence parallel", "c2a": f"tp{n} (forward)",
                                       "c2at": f"tp{n}",
                                       "c4": "dp8 x co-shard 4 (FFN)",
                                       "c5": "3F1B pp4 x dap2 (K=4)"}[args.config],
                       "lanes_per_gpu": nlanes / max(n, 1),
                       "sample": meta["sample"], "l2": "step working set " +
                       f"{st['device_bytes'] / 2**30:.1f} GiB > 126 MB L2 (no flush needed)",
                       "transport": (("peer memory (CUDA IPC over NVLink, device flags)" if transport == "peer"
                                      else transport) if dist else "single process"),
                       "memory": ("timed-mode reuse of freed buffers (REUSE_MEMORY)" if reuse_flags
                                  else "every buffer resident for the step"),
                       "lanes": st["num_lanes"], "tasks": st["num_tasks"], "launch": (
                           "CUDA graph" if st["graph_captured"] else "eager")},
            "roofline": roof,
            "plan_roofline": {"t_roof_ms": t_roof * 1e3, "frac": t_roof * 1e3 / ms,
                              "gemm_tflop_per_step": sum(F) / 1e12, "hbm_gb_per_step": sum(M) / 1e9,
                              "wire_gb_per_step": sum(W) / 1e9,
                              "work": "the plan's algorithmic work (describe with NO_FUSION | NO_GROUPING): every "
                                      "elementwise op and copy counted, whatever the executor fuses or aliases",
                              "peaks": {"bf16_tflops": peaks["bf16_sus"], "hbm_gbs": peaks["hbm"],
                                        "nvlink_gbs": NVLINK_GBS, "source": peaks["src"] + " (sustained bf16)"}},
            "adapter_bus_gbs": (None if not coll or coll["wire"] == 0 else
                                {"value": coll["wire"] / (coll["ms"] / 1e3) / 1e9, "vs_nvlink_gbs": NVLINK_GBS}),
            "nvlink_peer_copy": nvlink_peer_bandwidth() if n > 1 else None,
            "kernel_families": families,
            "e2e": {"value": meta["samples_per_step"] / (e2e_ms / 1e3), "unit": "samples/s",
                    "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "via": "planc_b200_run_e2e (C ABI): pinned H2D of step inputs, graph step, D2H of results",
                    **e2e_bound},
            "sustained": sustained,
            "dropin": dropin,
            "host_cores": os.cpu_count(),
            "gpu_launches": st["kernels_per_step"] * args.steps,
            "gemm_tc_launches_per_step": st["gemm_tc_per_step"],
            "clocks": clocks,
        }
        if not args.no_cpu_baseline and n == 1:
            try:
                cb, _ = cpu_baseline(args.config)
                small, smeta = load_plan(cpu_plan_name(args.config).replace("_standin", ""))
                with pb.Executor(small, lane_gpus=[0]) as sx:
                    sx.set_inputs(synthetic_inputs(small, 1))
                    sx.run(3)
                    sms = sx.run(20)
                cb["gpu_value_same_shape"] = smeta["samples_per_step"] / (sms / 1e3)
                result["cpu_baseline"] = cb
            except Exception as e:  # reference library not shipped
                result["cpu_baseline"] = {"value": None, "unavailable": str(e)[:200]}
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if result:
        print(json.dumps(result))


if __name__ == "__main__":
    main()
