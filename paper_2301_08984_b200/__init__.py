"""planc_b200 — B200-native executor for SuperScaler parallelization plans.

Python face of the C ABI in ``include/planc_b200.h`` (the product is the
C++/CUDA library ``_lib/libplanc_b200.so``; this module only binds it).
The API mirrors the reference's plan-execution interface
(reference proj/include/planc/refexec.hpp:38-60):

    run_plan(plan_json, inputs) -> outputs      # refexec.hpp:43
    compare_outputs(expected, actual, rel_tol)  # refexec.hpp:58 (pure host)

``inputs`` / ``outputs`` are TensorMaps: ``dict[int, numpy.ndarray]`` keyed
by pTensor id (refexec.hpp:34), values dense row-major float64 like
ConcreteTensor. Errors raise the reference's exception classes
(SchemaError / UsageError / InternalError, util.hpp:17-29); device failures
raise CudaError. There is no CPU fallback: without the built library or a
GPU every call raises.
"""
from __future__ import annotations

import ctypes
import json
import os

import numpy as np

__all__ = [
    "Executor", "run_plan", "describe", "compare_outputs", "library_path",
    "SchemaError", "UsageError", "InternalError", "CudaError",
    "NO_GRAPH", "NO_TENSOR_CORES", "STRICT_VALUE",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_lib", "libplanc_b200.so")

NO_GRAPH = 0x1
NO_TENSOR_CORES = 0x2
STRICT_VALUE = 0x4
SERIAL_LANES = 0x8
FUSE_EPILOGUES = 0x10  # default on; NO_FUSION turns it off
PEER_MEMORY = 0x20
NO_GROUPING = 0x40
NO_FUSION = 0x80
NO_ALIAS = 0x100
NO_SCATTER = 0x200
FUSE_ACT = 0x400
REUSE_MEMORY = 0x800
BATCH = 0x1000
NO_GATHER = 0x2000
NO_BOX_EW = 0x4000
NO_ALIAS_VIEWS = 0x8000
GATHER_COLS = 0x10000


class PlancError(RuntimeError):
    pass


class SchemaError(PlancError):
    pass


class UsageError(PlancError):
    pass


class InternalError(PlancError):
    pass


class CudaError(PlancError):
    pass


class _Stats(ctypes.Structure):
    _fields_ = [
        ("num_lanes", ctypes.c_int), ("num_tasks", ctypes.c_int), ("num_instructions", ctypes.c_int),
        ("kernels_per_step", ctypes.c_int), ("gemm_tc_per_step", ctypes.c_int), ("graph_captured", ctypes.c_int),
        ("flops", ctypes.c_double), ("hbm_bytes", ctypes.c_double), ("wire_bytes", ctypes.c_double),
        ("max_lane_gemm_flops", ctypes.c_double), ("max_lane_hbm_bytes", ctypes.c_double),
        ("max_lane_wire_bytes", ctypes.c_double), ("device_bytes", ctypes.c_int64),
    ]


_lib = None


def library_path() -> str:
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise RuntimeError(
            f"planc_b200: native library missing ({_LIB_PATH}); build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` — there is no CPU fallback")
    L = ctypes.CDLL(_LIB_PATH)
    c_int, c_i64, c_dbl, vp = ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
    P = ctypes.POINTER
    L.planc_b200_last_error.restype = ctypes.c_char_p
    L.planc_b200_version.restype = ctypes.c_char_p
    L.planc_b200_open.argtypes = [ctypes.c_char_p, P(c_int), c_int, ctypes.c_uint32, P(vp)]
    L.planc_b200_close.argtypes = [vp]
    L.planc_b200_set_input.argtypes = [vp, c_int, P(c_dbl), P(c_i64), c_int]
    L.planc_b200_run.argtypes = [vp, c_int, P(c_dbl)]
    L.planc_b200_run_e2e.argtypes = [vp, c_int, P(c_dbl), P(c_i64), P(c_i64)]
    L.planc_b200_num_outputs.argtypes = [vp]
    L.planc_b200_output_ids.argtypes = [vp, P(c_int), c_int]
    L.planc_b200_num_inputs.argtypes = [vp]
    L.planc_b200_input_ids.argtypes = [vp, P(c_int), c_int]
    L.planc_b200_ptensor_shape.argtypes = [vp, c_int, P(c_i64), c_int, P(c_int)]
    L.planc_b200_get_output.argtypes = [vp, c_int, P(c_dbl), c_i64]
    L.planc_b200_get_stats.argtypes = [vp, P(_Stats)]
    L.planc_b200_read_buffer.argtypes = [vp, c_int, P(c_dbl), c_i64]
    L.planc_b200_read_buffer.restype = c_i64
    L.planc_b200_profile.argtypes = [vp, P(ctypes.c_char_p)]
    L.planc_b200_timeline.argtypes = [vp, P(vp)]
    L.planc_b200_describe.argtypes = [ctypes.c_char_p, ctypes.c_uint32, P(vp)]
    L.planc_b200_describe_rank.argtypes = [ctypes.c_char_p, P(c_int), c_int, ctypes.c_uint32, P(vp)]
    L.planc_b200_nccl_unique_id.argtypes = [ctypes.c_char_p]
    L.planc_b200_open_rank.argtypes = [ctypes.c_char_p, c_int, c_int, P(c_int), c_int, c_int, ctypes.c_char_p,
                                       ctypes.c_uint32, P(vp)]
    L.planc_b200_peer_blob_bytes.argtypes = [vp]
    L.planc_b200_peer_blob_bytes.restype = c_i64
    L.planc_b200_peer_export.argtypes = [vp, ctypes.c_char_p, c_i64]
    L.planc_b200_peer_import.argtypes = [vp, ctypes.c_char_p, c_i64]
    L.planc_b200_gemm_schedule.argtypes = [c_i64, c_i64, c_i64, c_int, c_int, c_int, c_int, c_int, P(c_int),
                                           P(c_int), P(c_int), P(c_int), P(c_int), P(c_int), P(c_int), P(c_i64)]
    L.planc_b200_gemm_config.argtypes = [c_i64, c_i64, c_i64, c_int, c_int, c_int, c_int, c_int, P(c_int), P(c_int)]
    L.planc_b200_free.argtypes = [vp]
    _lib = L
    return L


def _check(rc: int):
    if rc == 0:
        return
    msg = _load().planc_b200_last_error().decode()
    if rc == 4:
        raise (SchemaError if msg.startswith("SchemaError") else UsageError)(msg)
    if rc == 2:
        raise CudaError(msg)
    raise InternalError(msg)


def version() -> str:
    return _load().planc_b200_version().decode()


def describe(plan_json: str, strict_value: bool = False, lane_rank=None, flags: int = 0) -> dict:
    """Host-only lowering of a plan (no GPU): buffers, instructions, cells.

    With ``lane_rank`` (owner rank per plan lane) the one-process-per-GPU
    program is returned: cross-rank pieces become ``xfer`` exchange steps
    (NCCL transport), or — with ``flags`` including PEER_MEMORY — the global
    program plus its cross-rank flag schedule (``peer_sync``).
    """
    L = _load()
    out = ctypes.c_void_p()
    flags = flags | (STRICT_VALUE if strict_value else 0)
    if lane_rank is None:
        _check(L.planc_b200_describe(plan_json.encode(), flags, ctypes.byref(out)))
    else:
        arr = (ctypes.c_int * len(lane_rank))(*lane_rank)
        _check(L.planc_b200_describe_rank(plan_json.encode(), arr, len(lane_rank), flags, ctypes.byref(out)))
    s = ctypes.string_at(out.value).decode()
    L.planc_b200_free(out)
    return json.loads(s)


def gemm_schedule(m: int, n: int, k: int, ta: bool = False, tb: bool = False, c_bf16: bool = True,
                  sms: int = 148, group: int = 1) -> dict:
    """Host-only: the tcgen05 GEMM's launch schedule (tile width, grid, whole
    tiles, stream-K CTAs or split-K splits, workspace bytes) for `group`
    bf16 matmuls of this shape in one launch."""
    L = _load()
    bn, grid, dp, sk, sp, hf, occ = (ctypes.c_int() for _ in range(7))
    ws = ctypes.c_int64()
    _check(L.planc_b200_gemm_schedule(m, n, k, int(ta), int(tb), int(c_bf16), sms, group, ctypes.byref(bn),
                                      ctypes.byref(grid), ctypes.byref(dp), ctypes.byref(sk), ctypes.byref(sp),
                                      ctypes.byref(hf), ctypes.byref(occ), ctypes.byref(ws)))
    return {"tile_n": bn.value, "grid": grid.value, "dp_tiles": dp.value, "sk_ctas": sk.value, "splits": sp.value,
            "half_items": hf.value, "variant": occ.value, "ctas_per_sm": 2 if occ.value == 2 else 1,
            "ws_bytes": ws.value}


def gemm_config(m: int, n: int, k: int, ta: bool = False, tb: bool = False, a_bf16: bool = True,
                b_bf16: bool = True, c_bf16: bool = True) -> dict:
    """Host-only: whether a matmul of this shape and these element types
    takes the tensor cores (bf16: tcgen05 kind::f16; fp32 operands and
    output: 3xTF32 kind::tf32) and the tile width."""
    L = _load()
    tc, bn = ctypes.c_int(), ctypes.c_int()
    _check(L.planc_b200_gemm_config(m, n, k, int(ta), int(tb), int(a_bf16), int(b_bf16), int(c_bf16),
                                    ctypes.byref(tc), ctypes.byref(bn)))
    return {"tensor_cores": bool(tc.value), "tile_n": bn.value}


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId (rank 0 creates it, the caller broadcasts it)."""
    buf = ctypes.create_string_buffer(128)
    _check(_load().planc_b200_nccl_unique_id(buf))
    return buf.raw


def lanes_round_robin(num_lanes: int, world: int):
    """Default lane -> rank ownership: lane l runs on rank l % world."""
    return [lane % world for lane in range(num_lanes)]


class Executor:
    """One compiled plan on the GPU(s). ``lane_gpus[i]`` runs plan lane i.

    ``rank``/``world``/``lane_rank`` select the one-process-per-GPU mode: this
    process runs the lanes it owns on ``local_gpu``. Transport: NCCL exchange
    steps (``nccl_id`` from rank 0), or peer memory (``peer_exchange``: a
    callable all-gathering one ``bytes`` blob per rank, e.g. over
    torch.distributed — every rank maps the others' arenas via CUDA IPC).
    """

    def __init__(self, plan_json: str, lane_gpus=None, flags: int = 0, rank=None, world=None, lane_rank=None,
                 local_gpu: int = 0, nccl_id: bytes = None, peer_exchange=None):
        L = _load()
        self._h = ctypes.c_void_p()
        if rank is not None:
            arr = (ctypes.c_int * len(lane_rank))(*lane_rank)
            if peer_exchange is not None:
                flags |= PEER_MEMORY
            _check(L.planc_b200_open_rank(plan_json.encode(), rank, world, arr, len(lane_rank), local_gpu,
                                          nccl_id, flags, ctypes.byref(self._h)))
            if peer_exchange is not None:
                n = L.planc_b200_peer_blob_bytes(self._h)
                blob = ctypes.create_string_buffer(n)
                _check(L.planc_b200_peer_export(self._h, blob, n))
                blobs = list(peer_exchange(blob.raw))
                if len(blobs) != world or any(len(b) != n for b in blobs):
                    raise UsageError("peer_exchange must return one blob per rank")
                _check(L.planc_b200_peer_import(self._h, b"".join(blobs), n))
            return
        arr, n = None, 0
        if lane_gpus:
            n = len(lane_gpus)
            arr = (ctypes.c_int * n)(*lane_gpus)
        _check(L.planc_b200_open(plan_json.encode(), arr, n, flags, ctypes.byref(self._h)))

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            _load().planc_b200_close(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- inputs / outputs ------------------------------------------------
    def input_ids(self):
        L = _load()
        n = L.planc_b200_num_inputs(self._h)
        ids = (ctypes.c_int * max(n, 1))()
        L.planc_b200_input_ids(self._h, ids, n)
        return list(ids[:n])

    def output_ids(self):
        L = _load()
        n = L.planc_b200_num_outputs(self._h)
        ids = (ctypes.c_int * max(n, 1))()
        L.planc_b200_output_ids(self._h, ids, n)
        return list(ids[:n])

    def shape(self, ptensor: int):
        shp = (ctypes.c_int64 * 16)()
        rank = ctypes.c_int()
        _check(_load().planc_b200_ptensor_shape(self._h, ptensor, shp, 16, ctypes.byref(rank)))
        return tuple(shp[: rank.value])

    def set_input(self, ptensor: int, value):
        a = np.ascontiguousarray(value, dtype=np.float64)
        shp = (ctypes.c_int64 * max(a.ndim, 1))(*a.shape)
        _check(_load().planc_b200_set_input(self._h, ptensor, a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                            shp, a.ndim))

    def set_inputs(self, inputs: dict):
        for pid, v in inputs.items():
            self.set_input(int(pid), v)

    def get_output(self, ptensor: int, out: np.ndarray = None) -> np.ndarray:
        """Reassembled value of a produced pTensor (float64). ``out``: a
        C-contiguous float64 array of the pTensor's shape to fill instead of
        allocating one (a caller reusing its TensorMap storage across steps)."""
        shp = self.shape(ptensor)
        if out is None:
            out = np.empty(shp, dtype=np.float64)
        elif out.dtype != np.float64 or out.shape != tuple(shp) or not out.flags.c_contiguous:
            raise UsageError("get_output: out must be a C-contiguous float64 array of shape %s" % (shp,))
        _check(_load().planc_b200_get_output(self._h, ptensor, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                             out.size))
        return out

    def read_buffer(self, buffer: int) -> np.ndarray:
        L = _load()
        n = L.planc_b200_read_buffer(self._h, buffer, None, 0)
        if n < 0:
            _check(1)
        out = np.empty(n, dtype=np.float64)
        L.planc_b200_read_buffer(self._h, buffer, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), n)
        return out

    def outputs(self) -> dict:
        return {pid: self.get_output(pid) for pid in self.output_ids()}

    # -- execution --------------------------------------------------------
    def run(self, iters: int = 0) -> float:
        ms = ctypes.c_double()
        _check(_load().planc_b200_run(self._h, iters, ctypes.byref(ms)))
        return ms.value

    def run_e2e(self, iters: int):
        ms = ctypes.c_double()
        hb, db = ctypes.c_int64(), ctypes.c_int64()
        _check(_load().planc_b200_run_e2e(self._h, iters, ctypes.byref(ms), ctypes.byref(hb), ctypes.byref(db)))
        return ms.value, hb.value, db.value

    def stats(self) -> dict:
        s = _Stats()
        _check(_load().planc_b200_get_stats(self._h, ctypes.byref(s)))
        return {k: getattr(s, k) for k, _ in _Stats._fields_}

    def timeline(self):
        """Measured per-task timeline of one step (simulator timeline shape)."""
        L = _load()
        out = ctypes.c_void_p()
        _check(L.planc_b200_timeline(self._h, ctypes.byref(out)))
        s = ctypes.string_at(out.value).decode()
        L.planc_b200_free(out)
        return json.loads(s)

    def profile(self):
        out = ctypes.c_char_p()
        L = _load()
        _check(L.planc_b200_profile(self._h, ctypes.byref(out)))
        return json.loads(out.value.decode())


def run_plan(plan_json: str, inputs: dict, lane_gpus=None, flags: int = 0) -> dict:
    """Drop-in for ``planc::run_plan(plan, inputs)`` (refexec.hpp:43)."""
    with Executor(plan_json, lane_gpus, flags) as ex:
        ex.set_inputs(inputs)
        ex.run(0)
        return ex.outputs()


def compare_outputs(expected: dict, actual: dict, rel_tol: float = 0.0, normwise: bool = False):
    """``planc::compare_outputs`` (refexec.cpp:604-631): |e-a| <= tol*max(1,|e|).

    ``normwise=True`` scales the tolerance by the tensor's magnitude instead,
    |e-a| <= tol*max(1, max|e|) — the stated bf16 criterion: after a bf16
    rounding of partial sums, elementwise relative error is unbounded where
    the exact result cancels to near zero.
    """
    for pid in sorted(expected):
        e = np.asarray(expected[pid], dtype=np.float64)
        if pid not in actual or tuple(np.shape(actual[pid])) != e.shape:
            return False, f"mismatch on tensor {pid} (missing or shape)"
        a = np.asarray(actual[pid], dtype=np.float64)
        nan_e, nan_a = np.isnan(e), np.isnan(a)
        if rel_tol == 0.0:
            bad = (e != a) & ~(nan_e & nan_a)
        else:
            with np.errstate(invalid="ignore"):
                if normwise:
                    fin = np.abs(e[np.isfinite(e)])
                    scale = max(1.0, float(fin.max())) if fin.size else 1.0
                    bad = ~(np.abs(e - a) <= rel_tol * scale)
                else:
                    bad = ~(np.abs(e - a) <= rel_tol * np.maximum(1.0, np.abs(e)))
            bad &= ~((nan_e & nan_a) | (np.isinf(e) & (e == a)))
        bad |= nan_e != nan_a  # a NaN on one side only is always a mismatch
        if bad.any():
            idx = np.unravel_index(int(np.argmax(bad)), e.shape)
            return False, (f"mismatch on tensor {pid} at {list(map(int, idx))}: "
                           f"expected {e[idx]}, got {a[idx]}")
    return True, "ok"
