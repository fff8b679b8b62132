"""TEST INFRASTRUCTURE — ctypes view of the reference planc library.

Loads ``oracle/_ref/libplanc_ref.so`` (the unmodified reference sources under
/root/reference/proj built by ``oracle/Makefile`` plus the ``ref_capi.cpp``
shim). Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline /
``--impl reference`` legs may use this module; the product path never does.

TensorMaps are ``dict[int, numpy.ndarray(float64)]`` keyed by pTensor id, the
Python spelling of ``planc::TensorMap`` (reference include/planc/refexec.hpp:34).
"""
from __future__ import annotations

import ctypes
import json
import os
import struct

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libplanc_ref.so")
_lib = None


class RefError(RuntimeError):
    pass


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RefError(f"reference oracle not built: {LIB_PATH} (run make -C oracle)")
        L = ctypes.CDLL(LIB_PATH)
        vp, cp, i64, i64p = ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)
        L.ref_last_error.restype = cp
        L.ref_free.argtypes = [vp]
        for name, args in [
            ("ref_mlp_doc", [ctypes.c_int, i64, i64, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
            ("ref_coshard_doc", [i64, i64, i64]),
            ("ref_embed_doc", [ctypes.c_int, i64, i64, i64]),
            ("ref_three_pass_doc", [ctypes.c_int, i64, i64]),
            ("ref_chain_doc", []),
            ("ref_compile", [cp, cp]),
            ("ref_roundtrip_plan", [cp]),
            ("ref_simulate", [cp]),
        ]:
            f = getattr(L, name)
            f.argtypes = args
            f.restype = vp
        L.ref_random_inputs.argtypes = [cp, ctypes.c_uint64, ctypes.c_int, i64p]
        L.ref_random_inputs.restype = vp
        L.ref_run_reference.argtypes = [cp, cp, i64p]
        L.ref_run_reference.restype = vp
        L.ref_run_plan.argtypes = [cp, cp, ctypes.c_int, ctypes.POINTER(ctypes.c_double), i64p]
        L.ref_run_plan.restype = vp
        L.ref_compare.argtypes = [cp, cp, ctypes.c_double]
        L.ref_compare.restype = ctypes.c_int
        _lib = L
    return _lib


def _take_str(p) -> str:
    if not p:
        raise RefError(lib().ref_last_error().decode())
    s = ctypes.string_at(p).decode()
    lib().ref_free(p)
    return s


def _take_blob(p, n) -> dict:
    if not p:
        raise RefError(lib().ref_last_error().decode())
    raw = ctypes.string_at(p, n.value)
    lib().ref_free(p)
    return decode_tensors(raw)


def encode_tensors(tm: dict) -> bytes:
    out = [struct.pack("<q", len(tm))]
    for pid in sorted(tm):
        a = np.ascontiguousarray(tm[pid], dtype=np.float64)
        out.append(struct.pack("<qq", pid, a.ndim))
        out.append(np.asarray(a.shape, dtype=np.int64).tobytes())
        out.append(a.tobytes())
    return b"".join(out)


def decode_tensors(raw: bytes) -> dict:
    off = 0
    (count,) = struct.unpack_from("<q", raw, off)
    off += 8
    tm = {}
    for _ in range(count):
        pid, rank = struct.unpack_from("<qq", raw, off)
        off += 16
        shape = tuple(np.frombuffer(raw, dtype=np.int64, count=rank, offset=off))
        off += 8 * rank
        vol = int(np.prod(shape)) if rank else 1
        data = np.frombuffer(raw, dtype=np.float64, count=vol, offset=off).copy()
        off += 8 * vol
        tm[int(pid)] = data.reshape(shape)
    return tm


# --- reference fixtures (proj/tests/testutil.cpp) ---------------------------

def mlp_doc(layers=2, batch=4, hidden=4, optimizer=True, bias=False, weight_grads=True) -> str:
    return _take_str(lib().ref_mlp_doc(layers, batch, hidden, int(optimizer), int(bias), int(weight_grads)))


def coshard_doc(batch=4, hidden=4, middle=16) -> str:
    return _take_str(lib().ref_coshard_doc(batch, hidden, middle))


def embed_doc(stage_layers=2, batch=4, vocab=4, hidden=4) -> str:
    return _take_str(lib().ref_embed_doc(stage_layers, batch, vocab, hidden))


def three_pass_doc(layers=2, batch=4, hidden=4) -> str:
    return _take_str(lib().ref_three_pass_doc(layers, batch, hidden))


def chain_doc() -> str:
    return _take_str(lib().ref_chain_doc())


def with_elem_size(doc: str, elem_size: int) -> str:
    """Same graph document with every pTensor's elem_size replaced (bf16 = 2)."""
    j = json.loads(doc)
    for p in j["ptensors"]:
        p["elem_size"] = elem_size
    return json.dumps(j)


# --- front end / oracle -----------------------------------------------------

def compile_plan(graph_doc: str, **spec) -> str:
    """Reference compile() (proj/src/compile.cpp:7) -> save_plan() JSON text."""
    s = ";".join(f"{k}={','.join(v) if isinstance(v, (list, tuple)) else v}" for k, v in spec.items())
    return _take_str(lib().ref_compile(graph_doc.encode(), s.encode()))


def roundtrip_plan(plan_json: str) -> str:
    return _take_str(lib().ref_roundtrip_plan(plan_json.encode()))


def simulate(plan_json: str) -> dict:
    """Reference simulator (simulate.cpp:102): {"report": ..., "timeline": [...]}."""
    return json.loads(_take_str(lib().ref_simulate(plan_json.encode())))


def random_integer_inputs(graph_doc: str, seed: int, magnitude: int = 4) -> dict:
    n = ctypes.c_int64()
    return _take_blob(lib().ref_random_inputs(graph_doc.encode(), seed, magnitude, ctypes.byref(n)), n)


def run_reference(graph_doc: str, inputs: dict) -> dict:
    n = ctypes.c_int64()
    return _take_blob(lib().ref_run_reference(graph_doc.encode(), encode_tensors(inputs), ctypes.byref(n)), n)


def run_plan(plan_json: str, inputs: dict, iters: int = 1):
    """Reference CPU executor (refexec.cpp:361). Returns (outputs, seconds_per_call)."""
    n = ctypes.c_int64()
    secs = ctypes.c_double()
    out = _take_blob(lib().ref_run_plan(plan_json.encode(), encode_tensors(inputs), iters,
                                        ctypes.byref(secs), ctypes.byref(n)), n)
    return out, secs.value


def compare_outputs(expected: dict, actual: dict, rel_tol: float = 0.0):
    """Reference compare_outputs (refexec.cpp:604). Returns (ok, message)."""
    rc = lib().ref_compare(encode_tensors(expected), encode_tensors(actual), rel_tol)
    return rc == 0, lib().ref_last_error().decode()
