"""GPU parity: every golden plan through the CUDA executor (C ABI).

All lanes of a plan run on cuda:0 (each lane with its own streams); the
outputs must equal the reference's run_reference outputs — bit-exact for
fp32 plans on integer inputs (all partial sums < 2^24), within the stated
relative tolerance (meta.json rel_tol, 2e-2) for bf16 plans.
"""
import json

import numpy as np
import pytest

import golden_cases
import paper_2301_08984_b200 as pb
from oracle import planc_oracle as po

pytestmark = pytest.mark.gpu


def _run(plan, inputs, flags=0, lanes=None):
    n = len(json.loads(plan)["lanes"])
    with pb.Executor(plan, lane_gpus=lanes or [0] * n, flags=flags) as ex:
        ex.set_inputs(inputs)
        ex.run(0)
        return ex.outputs(), ex.stats()


@pytest.mark.parametrize("name", golden_cases.names())
def test_golden_plan_parity(name):
    g = golden_cases.load(name)
    out, st = _run(g["plan"], g["inputs"])
    ok, msg = pb.compare_outputs(g["expected"], out, g["meta"]["rel_tol"], normwise=True)
    assert ok, msg
    assert st["kernels_per_step"] > 0


@pytest.mark.parametrize("name", ["mlp_dp2", "gpt_block_tp2", "embed_shard2", "adapt_d1_to_d0_4",
                                  "three_pass_3f1b", "gpt_block_fwd_tp2_mma"])
@pytest.mark.parametrize("flags", [pb.NO_GRAPH, pb.NO_TENSOR_CORES, pb.SERIAL_LANES, pb.NO_GRAPH | pb.SERIAL_LANES,
                                   pb.NO_FUSION, pb.NO_FUSION | pb.NO_GRAPH, pb.NO_ALIAS, pb.NO_GROUPING,
                                   pb.NO_SCATTER])
def test_parity_across_launch_modes(name, flags):
    g = golden_cases.load(name)
    out, _ = _run(g["plan"], g["inputs"], flags=flags)
    ok, msg = pb.compare_outputs(g["expected"], out, g["meta"]["rel_tol"], normwise=True)
    assert ok, msg


def test_repeated_steps_are_idempotent():
    g = golden_cases.load("gpt_block_tp2")
    n = len(json.loads(g["plan"])["lanes"])
    with pb.Executor(g["plan"], lane_gpus=[0] * n) as ex:
        ex.set_inputs(g["inputs"])
        ex.run(5)
        first = ex.outputs()
        ex.run(3)
        second = ex.outputs()
        assert ex.stats()["graph_captured"] == 1
    for k in first:
        assert np.array_equal(first[k], second[k])
    ok, msg = pb.compare_outputs(g["expected"], first, 0.0)
    assert ok, msg


def test_gpu_matches_numpy_oracle_vtensor_level():
    g = golden_cases.load("mlp_1f1b_dp2")
    out, _ = _run(g["plan"], g["inputs"])
    ok, msg = po.compare_outputs(po.run_plan(g["plan"], g["inputs"]), out, 0.0)
    assert ok, msg


def test_missing_input_is_usage_error():
    g = golden_cases.load("mlp_dp2")
    inputs = dict(g["inputs"])
    inputs.pop(0)
    with pytest.raises(pb.UsageError, match="missing input"):
        _run(g["plan"], inputs)


def test_run_plan_dropin():
    g = golden_cases.load("tp_value_split")
    out = pb.run_plan(g["plan"], g["inputs"], lane_gpus=[0, 0])
    ok, msg = pb.compare_outputs(g["expected"], out)
    assert ok, msg


def test_e2e_counts_bytes():
    g = golden_cases.load("gpt_block_tp2_bf16")
    with pb.Executor(g["plan"], lane_gpus=[0, 0]) as ex:
        ex.set_inputs(g["inputs"])
        ms, h2d, d2h = ex.run_e2e(3)
        assert ms > 0 and h2d > 0 and d2h > 0
        out = ex.outputs()
    ok, msg = pb.compare_outputs(g["expected"], out, 2e-2, normwise=True)
    assert ok, msg


@pytest.mark.parametrize("name", ["gpt_block_tp2", "mlp_1f1b_dp2", "embed_shard2"])
def test_rank_mode_single_rank(name):
    """One-process-per-GPU entry point (NCCL communicator, world = 1)."""
    g = golden_cases.load(name)
    n = len(json.loads(g["plan"])["lanes"])
    with pb.Executor(g["plan"], rank=0, world=1, lane_rank=[0] * n, local_gpu=0,
                     nccl_id=pb.nccl_unique_id()) as ex:
        ex.set_inputs(g["inputs"])
        ex.run(2)
        out = ex.outputs()
    ok, msg = pb.compare_outputs(g["expected"], out, g["meta"]["rel_tol"], normwise=True)
    assert ok, msg


def test_profile_reports_kernel_families():
    g = golden_cases.load("gpt_block_tp2")
    with pb.Executor(g["plan"], lane_gpus=[0, 0]) as ex:
        ex.set_inputs(g["inputs"])
        prof = ex.profile()
    kinds = {p["kind"] for p in prof}
    assert "box_collective" in kinds and any(k.startswith("gemm") for k in kinds)


def test_same_gpu_copies_become_aliases():
    """A recv whose send lane shares the GPU and identity ops launch nothing
    (the output aliases the source); results unchanged; NO_ALIAS copies."""
    g = golden_cases.load("mlp_1f1b_dp2")
    n = len(json.loads(g["plan"])["lanes"])
    outs, kernels = {}, {}
    for flags in (0, pb.NO_ALIAS):
        with pb.Executor(g["plan"], lane_gpus=[0] * n, flags=flags) as ex:
            ex.set_inputs(g["inputs"])
            ex.run(2)
            outs[flags] = ex.outputs()
            kernels[flags] = ex.stats()["kernels_per_step"]
            kinds = {p["kind"] for p in ex.profile()}
        assert ("alias" in kinds) == (flags == 0)
    assert kernels[0] < kernels[pb.NO_ALIAS]
    for k in outs[0]:
        assert np.array_equal(outs[0][k], outs[pb.NO_ALIAS][k])
    ok, msg = pb.compare_outputs(g["expected"], outs[0], 0.0)
    assert ok, msg


@pytest.mark.parametrize("name", ["gpt_block_fwd_tp2_mma", "ext_block_fwd_tp2_mma"])
def test_reduce_scatter_gemm_epilogue(name):
    """Row-parallel GEMMs feeding an all-reduce store their row slices into
    the owners' receive buffers (scatter epilogue); same results as storing
    the partials whole (NO_SCATTER)."""
    g = golden_cases.load(name)
    desc = pb.describe(g["plan"])
    assert any(i["kind"] == "gemm" and i["scatter"] for i in desc["instrs"])
    n = len(json.loads(g["plan"])["lanes"])
    outs = {}
    # Single process, every lane on cuda:0: the executor keeps whole partials
    # (no GPU boundary to cross) unless told the lanes sit on distinct devices;
    # one rank per lane (world 1, every lane owned) takes the scatter path.
    for flags in (0, pb.NO_SCATTER):
        with pb.Executor(g["plan"], flags=flags | pb.PEER_MEMORY, rank=0, world=1, lane_rank=[0] * n,
                         local_gpu=0, peer_exchange=lambda blob: [blob]) as ex:
            ex.set_inputs(g["inputs"])
            ex.run(2)
            outs[flags] = ex.outputs()
        ok, msg = pb.compare_outputs(g["expected"], outs[flags], g["meta"]["rel_tol"], normwise=True)
        assert ok, msg
    for k in outs[0]:
        assert np.array_equal(outs[0][k], outs[pb.NO_SCATTER][k]), k
