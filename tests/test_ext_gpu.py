"""GPU parity of the schema extension (softmax / layernorm / GELU and their
gradients, row-wise warp-per-segment kernels) against the float64 graph
oracle, normwise tolerance from meta.json (1e-4 fp32, 2e-2 bf16 against the bf16-rounded oracle), across
launch modes; kernel-level checks of every row-wise op at odd shapes."""
import json
import os

import numpy as np
import pytest

import golden_cases
import paper_2301_08984_b200 as pb
from oracle import planc_oracle as po
from plan_builder import single_op_plan

pytestmark = pytest.mark.gpu

EXT = json.load(open(os.path.join(golden_cases.GOLDEN, "index_ext.json")))


@pytest.mark.parametrize("name", EXT)
@pytest.mark.parametrize("flags", [0, pb.NO_GRAPH | pb.SERIAL_LANES, pb.NO_TENSOR_CORES])
def test_ext_golden_parity(name, flags):
    g = golden_cases.load(name)
    n = len(json.loads(g["plan"])["lanes"])
    with pb.Executor(g["plan"], lane_gpus=[0] * n, flags=flags) as ex:
        ex.set_inputs(g["inputs"])
        ex.run(2)
        out = ex.outputs()
        prof = ex.profile()
    ok, msg = pb.compare_outputs(g["expected"], out, g["meta"]["rel_tol"], normwise=True)
    assert ok, msg
    assert any(p["kind"] in ("rowwise", "attention") for p in prof)


def bf16_round(x):
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16 << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


@pytest.mark.parametrize("kind", ["softmax", "softmax-grad", "layernorm", "layernorm-grad", "gelu", "gelu-grad"])
@pytest.mark.parametrize("shape,seg", [((33, 128), 0), ((7, 2048), 0), ((5, 96), 32), ((9, 7), 0), ((3, 4096), 0),
                                       ((2, 6000), 1000), ((4, 2056), 0), ((3, 8192), 0), ((2, 24576), 0),
                                       ((2, 40000), 0)])
@pytest.mark.parametrize("elem", [4, 2])
def test_rowwise_kernels_vs_fp64(kind, shape, seg, elem):
    binary = kind.endswith("-grad")
    rng = np.random.default_rng(shape[0] * shape[1] + seg)
    x = rng.standard_normal(shape) * 2
    dy = rng.standard_normal(shape)
    if kind == "softmax-grad":
        x = po.eval_ext("softmax", [x], seg)
    if elem == 2:
        x, dy = bf16_round(x), bf16_round(dy)
    plan, out_pt = single_op_plan(kind, [shape, shape] if binary else [shape], shape, elem, elem,
                                  {"segment": seg} if seg else {})
    with pb.Executor(plan, lane_gpus=[0]) as ex:
        ex.set_inputs({0: x, 1: dy} if binary else {0: x})
        ex.run(0)
        got = ex.get_output(out_pt)
    ref = po.eval_ext(kind, [x, dy] if binary else [x], seg)
    err = np.abs(got - ref).max() / max(1.0, np.abs(ref).max())
    assert err < (2e-5 if elem == 4 else 1e-2), err
