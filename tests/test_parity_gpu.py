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
    if g["emulated"]:
        # bf16 plans in the exact-integer regime: bit for bit the plan's bf16
        # emulation (rounding wherever the executor stores; tests/golden
        # make_golden.py), whatever the kernels' fp32 summation order.
        ok, msg = pb.compare_outputs(g["emulated"], out, 0.0)
        assert ok, "bf16 emulation: " + msg


REF_OK = [n for n in golden_cases.names() if golden_cases.load(n)["meta"]["reference_run_plan"] == "ok"]
REF_THROWS = [n for n in golden_cases.names() if golden_cases.load(n)["meta"]["reference_run_plan"] != "ok"]


@pytest.mark.parametrize("name", REF_OK)
def test_value_split_extension_is_inert_where_the_reference_runs(name):
    """The V(m*v)->V(v) extension (default on) changes nothing on any plan
    the reference executor itself runs: bit-identical to STRICT_VALUE (the
    reference's refexec.cpp:110-117 rule)."""
    g = golden_cases.load(name)
    out, _ = _run(g["plan"], g["inputs"])
    strict, _ = _run(g["plan"], g["inputs"], flags=pb.STRICT_VALUE)
    assert sorted(out) == sorted(strict)
    for k in out:
        assert np.array_equal(out[k], strict[k]), k


@pytest.mark.parametrize("name", REF_THROWS)
def test_fact6_plans_match_the_graph_reference(name):
    """Dijkstra chains k=2 reduce-scatters (V(4)->V(2)->D);
    the reference run_plan throws (meta), STRICT_VALUE throws the same
    InternalError, the default executes the plan and equals run_reference on
    the graph bit for bit (fp32, integer inputs)."""
    g = golden_cases.load(name)
    assert g["meta"]["reference_run_plan"].startswith("throws: reconstruct")
    with pytest.raises(pb.InternalError, match="not fully covered"):
        _run(g["plan"], g["inputs"], flags=pb.STRICT_VALUE)
    out, _ = _run(g["plan"], g["inputs"])
    ok, msg = pb.compare_outputs(g["expected"], out, 0.0)
    assert ok, msg
    ok, msg = po.compare_outputs(po.run_plan(g["plan"], g["inputs"], vv=True), out, 0.0)
    assert ok, msg


@pytest.mark.parametrize("name", ["gpt_block_train_tp1_mma", "gpt_block_train_tp2_mma", "c2_cpu_tp1"])
def test_train_step_gemms_take_tensor_cores(name):
    """Every GEMM of the bf16 train step — forward, the transposed-operand
    dX / dW GEMMs of the backward, fused optimizer epilogues — runs on the
    tcgen05 path, and the step equals the bf16 emulation bit for bit."""
    g = golden_cases.load(name)
    desc = pb.describe(g["plan"])
    gemms = [i for i in desc["instrs"] if i["kind"] == "gemm"]
    assert any(i["ta"] for i in gemms) and any(i["tb"] for i in gemms)  # dW / dX shapes present
    out, st = _run(g["plan"], g["inputs"])
    assert st["gemm_tc_per_step"] == len(gemms), (st["gemm_tc_per_step"], len(gemms))
    ok, msg = pb.compare_outputs(g["emulated"], out, 0.0)
    assert ok, msg


@pytest.mark.parametrize("name", ["mlp_dp2", "gpt_block_tp2", "embed_shard2", "adapt_d1_to_d0_4",
                                  "three_pass_3f1b", "gpt_block_fwd_tp2_mma"])
@pytest.mark.parametrize("flags", [pb.NO_GRAPH, pb.NO_TENSOR_CORES, pb.SERIAL_LANES, pb.NO_GRAPH | pb.SERIAL_LANES,
                                   pb.NO_FUSION, pb.NO_FUSION | pb.NO_GRAPH, pb.NO_ALIAS, pb.NO_GROUPING,
                                   pb.NO_SCATTER, pb.BATCH, pb.BATCH | pb.NO_GRAPH, pb.NO_GATHER])
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


def test_gpu_matches_numpy_oracle_ptensor_level():
    g = golden_cases.load("mlp_1f1b_dp2")
    out, _ = _run(g["plan"], g["inputs"])
    ok, msg = po.compare_outputs(po.run_plan(g["plan"], g["inputs"]), out, 0.0)
    assert ok, msg


@pytest.mark.parametrize("name", ["mlp_1f1b_dp2", "gpt_block_tp2", "adapt_vv_rs2x2", "embed_shard2"])
def test_gpu_matches_numpy_oracle_vtensor_level(name):
    """Every produced vTensor (every piece every lane holds, adapters'
    intermediate results included) read back from its device buffer equals
    the restatement's per-vTensor value (planc_oracle return_vtensors)."""
    g = golden_cases.load(name)
    _, vts = po.run_plan(g["plan"], g["inputs"], vv=True, return_vtensors=True)
    desc = pb.describe(g["plan"])
    n = len(json.loads(g["plan"])["lanes"])
    checked = 0
    with pb.Executor(g["plan"], lane_gpus=[0] * n, flags=pb.NO_ALIAS) as ex:
        ex.set_inputs(g["inputs"])
        ex.run(0)
        for vt, buf in enumerate(desc["vt_buffer"]):
            if buf < 0 or vt not in vts or desc["buffers"][buf]["dead"]:
                continue
            got = ex.read_buffer(buf).reshape(vts[vt].shape)
            assert np.array_equal(got, vts[vt]), f"vtensor {vt} (buffer {buf})"
            checked += 1
    assert checked >= len(vts) // 2


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


@pytest.mark.parametrize("name", ["mlp_1f1b_dp2", "three_pass_3f1b", "adapt_d1_to_d0_4", "gpt_stack2_1f1b_bf16",
                                  "cross_group_scatter", "mlp_dp2_naive", "c4_coshard_dp8_bf16", "c5_3f1b_dap_bf16"])
def test_box_batching_same_bits_fewer_launches(name):
    """Adapter / elementwise instructions pending together in issue order
    share launches (BATCH, ExecOptions::batch_boxes; off by default): the
    same bits as one launch per instruction, and no more kernels per step."""
    g = golden_cases.load(name)
    outs, kernels = {}, {}
    for flags in (0, pb.BATCH):
        out, st = _run(g["plan"], g["inputs"], flags=flags)
        outs[flags], kernels[flags] = out, st["kernels_per_step"]
    assert kernels[pb.BATCH] <= kernels[0]
    for k in outs[0]:
        assert np.array_equal(outs[0][k], outs[pb.BATCH][k]), k
    ok, msg = pb.compare_outputs(g["expected"], outs[pb.BATCH], g["meta"]["rel_tol"], normwise=True)
    assert ok, msg


@pytest.mark.parametrize("name", ["gpt_block_sp_tp2_mma", "gpt_block_sp_tp4_mma", "gpt_block_train_tp2_mma",
                                  "c5_3f1b_dap_mma"])
def test_gathered_gemm_operands(name):
    """All-gather / concat -> GEMM prologue: a concat of
    row pieces feeding only tensor-core GEMMs is dropped and the GEMMs' TMA
    loads read the pieces in place. Same operands, same bits as the
    materialised concat (NO_GATHER), and the bf16 plan emulation's bits."""
    g = golden_cases.load(name)
    on = pb.GATHER_COLS if name.startswith("c5_") else 0  # column pieces: opt-in
    desc = pb.describe(g["plan"], flags=on)
    gathers = [i for i in desc["instrs"] if i["kind"] == "gemm" and any(x["pieces"] for x in i["gather"])]
    assert gathers, "the plan has no gathered GEMM operand"
    outs, kernels = {}, {}
    for flags in (on, pb.NO_GATHER):
        out, st = _run(g["plan"], g["inputs"], flags=flags)
        outs[flags], kernels[flags] = out, st["kernels_per_step"]
    # (a single-piece "gather" reads an identity's source: on one GPU that
    # copy is already an alias, so no kernel is saved there)
    assert kernels[on] <= kernels[pb.NO_GATHER]
    if "_sp_" in name or on:
        assert kernels[on] < kernels[pb.NO_GATHER]
    for k in outs[on]:
        assert np.array_equal(outs[on][k], outs[pb.NO_GATHER][k]), k
    ok, msg = pb.compare_outputs(g["expected"], outs[on], g["meta"]["rel_tol"], normwise=True)
    assert ok, msg
    if g["meta"].get("bf16_exact"):
        for k, v in g["emulated"].items():
            assert np.array_equal(outs[on][k], v), k


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


@pytest.mark.parametrize("name", [n for n in golden_cases.names() if golden_cases.load(n)["meta"]["lanes"] > 1])
def test_timed_mode_memory_reuse(name):
    """REUSE_MEMORY (the plan's frees honoured within the step): every output
    whose bytes survive the step is bit-identical to the resident run, the
    rest raise UsageError instead of returning reused bytes; a second step
    gives the same bits (released bytes are rewritten before they are read)."""
    g = golden_cases.load(name)
    n = len(json.loads(g["plan"])["lanes"])
    ref, _ = _run(g["plan"], g["inputs"])
    with pb.Executor(g["plan"], lane_gpus=[0] * n, flags=pb.REUSE_MEMORY) as ex:
        ex.set_inputs(g["inputs"])
        for steps in (0, 3):
            ex.run(steps)
            kept = 0
            for pt in ex.output_ids():
                try:
                    v = ex.get_output(pt)
                except pb.UsageError as e:
                    assert "REUSE_MEMORY" in str(e)
                    continue
                assert np.array_equal(v, ref[pt]), pt
                kept += 1
            assert kept > 0


@pytest.mark.parametrize("name", ["c5_3f1b_dap", "c5_3f1b_dap_bf16", "c5_3f1b_dap_mma", "c4_coshard_dp8_bf16",
                                  "embed_shard2"])
def test_box_elementwise_fusion(name):
    """An add / mul / max on a pure-copy adapter output (C5's all-to-all ->
    max gate) runs inside the adapter's box launch as fold terms: fewer
    kernels, and the same bits as the separate elementwise kernel
    (NO_BOX_EW) and as the reference."""
    g = golden_cases.load(name)
    desc = pb.describe(g["plan"])
    fused = [i for i in desc["instrs"] if i["kind"] == "box" and
             any(t["fold"] >= 0 for c in i["cells"] for t in c["terms"])]
    assert fused, "the plan has no box -> elementwise pattern"
    outs, kernels = {}, {}
    for flags in (0, pb.NO_BOX_EW):
        out, st = _run(g["plan"], g["inputs"], flags=flags)
        outs[flags], kernels[flags] = out, st["kernels_per_step"]
    assert kernels[0] < kernels[pb.NO_BOX_EW]
    for k in outs[0]:
        assert np.array_equal(outs[0][k], outs[pb.NO_BOX_EW][k]), k
    ok, msg = pb.compare_outputs(g["expected"], outs[0], g["meta"]["rel_tol"], normwise=True)
    assert ok, msg


@pytest.mark.parametrize("name", ["c5_3f1b_dap", "c5_3f1b_dap_bf16"])
def test_same_gpu_splits_become_views(name):
    """A copy of a contiguous sub-range (C5's DAP splits feeding the
    all-to-all) launches nothing on one GPU: the output is a view of the
    source range. Same bits as copying it (NO_ALIAS_VIEWS)."""
    g = golden_cases.load(name)
    outs, kernels = {}, {}
    for flags in (0, pb.NO_ALIAS_VIEWS):
        out, st = _run(g["plan"], g["inputs"], flags=flags)
        outs[flags], kernels[flags] = out, st["kernels_per_step"]
    assert kernels[0] < kernels[pb.NO_ALIAS_VIEWS]
    for k in outs[0]:
        assert np.array_equal(outs[0][k], outs[pb.NO_ALIAS_VIEWS][k]), k
    ok, msg = pb.compare_outputs(g["expected"], outs[0], g["meta"]["rel_tol"], normwise=True)
    assert ok, msg


@pytest.mark.parametrize("name", ["c5_3f1b_dap", "c2sp_tp2"])
def test_gathered_operands_at_full_size(name):
    """The gather prologue at the benchmark shapes (C5: column pieces of the
    DAP channel halves, incl. the 2-SM dW GEMMs whose zero tile reads past
    the last piece; C2-SP: row pieces): the terminal outputs are bit-equal
    to the materialised concats' (NO_GATHER)."""
    from test_fullsize_gpu import init_inputs, terminal_outputs  # (puts the repo root on sys.path)
    import bench

    plan, _ = bench.load_plan(name)
    inputs = init_inputs(plan)
    ids = terminal_outputs(plan)
    nl = len(json.loads(plan)["lanes"])
    on = pb.GATHER_COLS if name.startswith("c5_") else 0  # column pieces: opt-in
    outs = {}
    for flags in (on, pb.NO_GATHER):
        with pb.Executor(plan, lane_gpus=[0] * nl, flags=flags) as ex:
            ex.set_inputs(inputs)
            ex.run(0)
            outs[flags] = {i: ex.get_output(i) for i in ids}
    for i in ids:
        assert np.isfinite(outs[on][i]).all(), i
        assert np.array_equal(outs[on][i], outs[pb.NO_GATHER][i]), i

