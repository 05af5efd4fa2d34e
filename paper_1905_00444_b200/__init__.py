"""B200-native sliced tensor-network amplitude path (qFlex-style RQC simulator).

Python face of ``libqsg.so`` (C ABI in ``include/qsg.h``).  Names, argument
meaning and error behaviour mirror the reference's ``qsim`` API
(/root/reference/proj/include/qsim/*.hpp) so the parity tests read like the
reference's own.  All numeric work runs in the sm_100a kernels behind the C
ABI; there is no CPU fallback -- compute calls raise ``QsgError`` (CUDA) when
no GPU is present, and importing fails loudly when the library is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QSG_LIB") or os.path.join(_HERE, "libqsg.so")  # QSG_LIB: A/B builds only

__all__ = [
    "QsgError", "CircuitError", "lib", "mix_seed", "flop_count", "generate_rqc", "canonical_circuit",
    "circuit_info", "plan_json", "fold_worldlines", "select_slices", "draw_x1", "xeb_score", "transpose", "contract", "normalize_inplace",
    "Engine", "PLAN_JSON", "PLAN_REF7X7", "PLAN_GREEDY", "device_count",
]

PLAN_JSON, PLAN_REF7X7, PLAN_GREEDY = 0, 1, 2
_ERRS = {1: "invalid_argument", 2: "length_error", 3: "out_of_range", 4: "runtime_error", 5: "cuda", 6: "oom",
         7: "circuit"}


class QsgError(RuntimeError):
    """Failure reported through the C ABI; ``kind`` names the reference exception type."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code
        self.kind = _ERRS.get(code, "unknown")


class CircuitError(QsgError):
    """qsim::CircuitError (include/qsim/circuit.hpp:68-74): carries the 1-based line."""

    def __init__(self, code: int, msg: str, line: int):
        super().__init__(code, msg)
        self.line = line


class InvalidArgument(QsgError, ValueError):
    pass


class LengthError(QsgError, ValueError):
    pass


class JobError(QsgError):
    """A run_amplitudes job failed; slice_id = the lowest failing task's
    slice (the reference's JobError, include/qsim/engine.hpp:81-84)."""

    def __init__(self, code, msg, slice_id):
        super().__init__(code, msg)
        self.slice_id = slice_id


class OutOfRange(QsgError, IndexError):
    pass


class _OpProfile(C.Structure):
    _fields_ = [("kind", C.c_int32), ("step", C.c_int32), ("m", C.c_int64), ("n", C.c_int64), ("k", C.c_int64),
                ("flops", C.c_uint64), ("bytes", C.c_int64), ("ms_total", C.c_double), ("executions", C.c_int64),
                ("tensor_cores", C.c_int32), ("pad", C.c_int32)]


class _EngineInfo(C.Structure):
    _fields_ = [("num_qubits", C.c_int64), ("num_slices", C.c_int64), ("batch_size", C.c_int64),
                ("num_steps", C.c_int64), ("max_rank", C.c_int64), ("peak_memory", C.c_int64),
                ("arena_bytes", C.c_int64), ("node_bytes", C.c_int64), ("flops_per_slice", C.c_uint64),
                ("num_ops", C.c_int64)]


class _SampleStats(C.Structure):
    _fields_ = [("x1_draws", C.c_uint64), ("redraws", C.c_uint64), ("cap_hits", C.c_uint64),
                ("candidates", C.c_uint64), ("exact_count", C.c_int64), ("uniform_count", C.c_int64)]


class _XebReport(C.Structure):
    _fields_ = [("n", C.c_int32), ("hog_available", C.c_int32), ("size", C.c_int64), ("zero_excluded", C.c_int64),
                ("mean_log_prob", C.c_double), ("cross_entropy", C.c_double), ("fidelity_estimate", C.c_double),
                ("hog_fraction", C.c_double)]


def _struct_dict(s):
    return {f[0]: getattr(s, f[0]) for f in s._fields_}


_lib = None


def lib():
    """Loads libqsg.so (built by ``make -C paper_1905_00444_b200``); raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libqsg.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    i32, i64, u64, P = C.c_int, C.c_int64, C.c_uint64, C.POINTER
    cp, vp, fp, dp = C.c_char_p, C.c_void_p, P(C.c_float), P(C.c_double)
    sig = {
        "qsg_last_error": (cp, []),
        "qsg_last_error_line": (i32, []),
        "qsg_last_error_slice": (i64, []),
        "qsg_version": (cp, []),
        "qsg_device_count": (i32, [P(i32)]),
        "qsg_mix_seed": (u64, [u64, u64]),
        "qsg_flop_count": (i32, [u64, u64, u64, P(u64)]),
        "qsg_generate_rqc": (i32, [i32, i32, i32, u64, i32, cp, i64, P(i64)]),
        "qsg_canonical_circuit": (i32, [cp, cp, i64, P(i64)]),
        "qsg_generate_rqc_masked": (i32, [i32, i32, cp, i32, u64, i32, cp, i64, P(i64)]),
        "qsg_bristlecone_mask": (i32, [i32, cp, i64, P(i64)]),
        "qsg_circuit_info": (i32, [cp, P(i32), P(i32), P(i32), P(i32)]),
        "qsg_plan_json": (i32, [cp, P(i32), i32, i32, cp, i64, cp, i64, P(i64)]),
        "qsg_fold_qtns": (i32, [cp, P(i32), i32, cp, i64, cp, i64, P(i64)]),
        "qsg_select_slices": (i32, [i64, i64, i64, u64, P(i64)]),
        "qsg_draw_x1": (i32, [i32, P(i32), i32, u64, u64, P(i32)]),
        "qsg_permute_dev": (i32, [vp, i64, vp, i32, P(i64), P(i64), vp]),
        "qsg_cgemm_dev": (i32, [vp, vp, vp, i64, i64, i64, i32, i32, vp]),
        "qsg_cgemm_tc_workspace_bytes": (i64, [i64, i64, i64, i32]),
        "qsg_cgemm_tc_dev": (i32, [vp, vp, vp, i64, i64, i64, i32, vp, i64, vp]),
        "qsg_accumulate_dev": (i32, [vp, C.c_double, i64, vp, vp, vp]),
        "qsg_transpose": (i32, [i32, P(i64), fp, P(i32), fp]),
        "qsg_contract": (i32, [i32, P(i32), P(i64), fp, C.c_double, i32, P(i32), P(i64), fp, C.c_double, i32, P(i32),
                               fp, dp, P(u64), i32]),
        "qsg_normalize": (i32, [fp, i64, dp, P(i32)]),
        "qsg_engine_create": (i32, [cp, i32, cp, P(i32), i32, i32, i32, P(vp)]),
        "qsg_engine_create_ex": (i32, [cp, i32, cp, P(i32), i32, i32, i32, i64, i32, P(vp)]),
        "qsg_program_listing_ex": (i32, [cp, i32, cp, P(i32), i32, i32, i64, i64, cp, i64, P(i64)]),
        "qsg_engine_destroy": (i32, [vp]),
        "qsg_program_listing": (i32, [cp, i32, cp, P(i32), i32, i32, cp, i64, P(i64)]),
        "qsg_engine_get_info": (i32, [vp, P(_EngineInfo)]),
        "qsg_engine_plan_json": (i32, [vp, cp, i64, P(i64)]),
        "qsg_engine_describe": (i32, [vp, cp, i64, P(i64)]),
        "qsg_engine_open_qubits": (i32, [vp, P(i32)]),
        "qsg_engine_prepare": (i32, [vp, P(i32), i32, P(i64)]),
        "qsg_engine_fold_nodes": (i32, [vp, cp, vp, i64]),
        "qsg_engine_load_nodes": (i32, [vp, vp, i64]),
        "qsg_engine_export_nodes": (i32, [vp, vp, i64]),
        "qsg_engine_run": (i32, [vp, P(i64), i64, i32, i32]),
        "qsg_engine_results": (i32, [vp, dp, dp]),
        "qsg_engine_stream": (i32, [vp, P(vp)]),
        "qsg_engine_synchronize": (i32, [vp]),
        "qsg_engine_launches": (i32, [vp, P(i64)]),
        "qsg_engine_per_slice_rows": (i32, [vp, P(i64)]),
        "qsg_engine_profile": (i32, [vp, P(_OpProfile), i32, P(i32)]),
        "qsg_engine_reset_profile": (i32, [vp]),
        "qsg_engine_set_profile": (i32, [vp, i32]),
        "qsg_amplitude_batch": (i32, [vp, P(i32), i32, P(i64), i64, dp, cp]),
        "qsg_widen_plan": (i32, [cp, i32, cp, P(i32), i32, P(i32), i32, cp, i64, P(i64)]),
        "qsg_reassociate_plan": (i32, [cp, i32, cp, P(i32), i32, cp, i64, P(i64), P(i32)]),
        "qsg_amplitude_batches": (i32, [vp, P(i32), i32, P(i32), i32, i32, P(i64), i64, dp, cp]),
        "qsg_amplitude_batches_submit": (i32, [vp, P(i32), i32, P(i32), i32, i32, P(i64), i64, i32]),
        "qsg_amplitude_batches_collect": (i32, [vp, P(i32), i32, P(i32), i32, i32, i32, dp, cp]),
        "qsg_run_amplitudes": (i32, [vp, cp, i32, i32, i64, i64, u64, dp, P(i64), P(u64)]),
        "qsg_sample": (i32, [vp, i64, i64, i64, i32, C.c_double, u64, cp, dp, P(_SampleStats), P(_XebReport)]),
        "qsg_xeb_score": (i32, [i32, dp, i64, i32, C.c_double, P(_XebReport)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def exported_symbols():
    """Names declared in include/qsg.h (checked by the CPU tests)."""
    import re
    hdr = os.path.join(os.path.dirname(_HERE), "include", "qsg.h")
    with open(hdr) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(qsg_[a-z0-9_]+)\s*\(", text)))


def _check(rc: int):
    if rc == 0:
        return
    L = lib()
    msg = L.qsg_last_error().decode()
    if rc == 7:
        raise CircuitError(rc, msg, L.qsg_last_error_line())
    if rc == 1:
        raise InvalidArgument(rc, msg)
    if rc == 2:
        raise LengthError(rc, msg)
    if rc == 3:
        raise OutOfRange(rc, msg)
    slice_id = L.qsg_last_error_slice()
    if slice_id >= 0:
        raise JobError(rc, msg, slice_id)
    raise QsgError(rc, msg)


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _i32(seq):
    a = np.ascontiguousarray(np.asarray(list(seq), dtype=np.int32))
    return a, _p(a, C.c_int)


def _text(fn, *args):
    n = C.c_int64(0)
    _check(fn(*args, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(fn(*args, buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def device_count() -> int:
    n = C.c_int(0)
    _check(lib().qsg_device_count(C.byref(n)))
    return n.value


# ---- host model (bit-exact with qsim) ----------------------------------------

def mix_seed(seed: int, stream: int) -> int:
    """qsim::mix_seed (include/qsim/types.hpp:25-30)."""
    return int(lib().qsg_mix_seed(seed, stream))


def flop_count(v0: int, v1: int, v2: int) -> int:
    """qsim::flop_count, Eq.(1) (include/qsim/contraction.hpp:46-56)."""
    out = C.c_uint64(0)
    _check(lib().qsg_flop_count(v0, v1, v2, C.byref(out)))
    return int(out.value)


def generate_rqc(rows: int, cols: int, m: int, seed: int, t_only_first: bool = True) -> str:
    """serialize_circuit(generate_rqc(...)) (src/circuit.cpp:243-294)."""
    return _text(lib().qsg_generate_rqc, rows, cols, m, seed, 1 if t_only_first else 0)


def generate_rqc_masked(rows: int, cols: int, mask: str, m: int, seed: int, t_only_first: bool = True) -> str:
    """generate_rqc on a masked grid (mask: rows*cols '0'/'1'); inactive cells only get the outer H layers."""
    return _text(lib().qsg_generate_rqc_masked, rows, cols, mask.encode(), m, seed, 1 if t_only_first else 0)


def bristlecone_mask(active: int = 70) -> str:
    """11x12 diamond mask with 72, 70 or 60 active cells (the Bristlecone construction of SURVEY 8d)."""
    return _text(lib().qsg_bristlecone_mask, active)


def canonical_circuit(text: str) -> str:
    """serialize_circuit(parse_circuit(text)) (src/circuit.cpp:128-220)."""
    return _text(lib().qsg_canonical_circuit, text.encode())


def circuit_info(text: str):
    r, c, q, cy = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    _check(lib().qsg_circuit_info(text.encode(), C.byref(r), C.byref(c), C.byref(q), C.byref(cy)))
    return {"rows": r.value, "cols": c.value, "qubits": q.value, "cycles": cy.value}


def plan_json(circuit_text: str, open_qubits=(), kind: int = PLAN_JSON, plan_text: str = "", budget: int = 0) -> str:
    """Annotated plan JSON (plan_from_json / reference_plan_7x7 / plan_contraction + plan_to_json)."""
    a, p = _i32(open_qubits)
    return _text(lib().qsg_plan_json, circuit_text.encode(), p, len(a), kind, plan_text.encode(), budget)


def _parse_qtns(blob: bytes):
    import struct
    out, off = [], 0
    while off < len(blob):
        assert blob[off:off + 4] == b"QTNS"
        _, rank = struct.unpack_from("<II", blob, off + 4)
        off += 12
        labels, dims = [], []
        for _ in range(rank):
            (ln,) = struct.unpack_from("<H", blob, off)
            off += 2
            labels.append(blob[off:off + ln].decode())
            off += ln
            (d,) = struct.unpack_from("<Q", blob, off)
            off += 8
            dims.append(d)
        (ls,) = struct.unpack_from("<d", blob, off)
        off += 8
        vol = int(np.prod(dims)) if dims else 1
        data = np.frombuffer(blob, dtype=np.complex64, count=vol, offset=off).copy()
        off += 8 * vol
        out.append((labels, dims, ls, data.reshape(dims) if dims else data.reshape(())))
    return out


def fold_worldlines(circuit_text: str, out_bits, plan_text: str = "", slice_id: int = 0):
    """fold_worldlines (+ apply_cut) as [(labels, dims, log_scale, ndarray)] (src/network.cpp:106-149)."""
    a, p = _i32(out_bits)
    n = C.c_int64(0)
    L = lib()
    _check(L.qsg_fold_qtns(circuit_text.encode(), p, len(a), plan_text.encode(), slice_id, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value)
    _check(L.qsg_fold_qtns(circuit_text.encode(), p, len(a), plan_text.encode(), slice_id, buf, n.value, C.byref(n)))
    return _parse_qtns(buf.raw[: n.value])


def select_slices(num: int, den: int, num_slices: int, seed: int):
    """select_slices (src/engine.cpp:285-298)."""
    out = np.zeros(max(num, 0), dtype=np.int64)
    _check(lib().qsg_select_slices(num, den, num_slices, seed, _p(out, C.c_int64)))
    return [int(x) for x in out]


def draw_x1(n: int, open_qubits, seed: int, index: int):
    """x1 of sampling task `index` (src/sampler.cpp:70-82): -1 on open qubits."""
    a, p = _i32(open_qubits)
    out = np.zeros(n, dtype=np.int32)
    _check(lib().qsg_draw_x1(n, p, len(a), seed, index, _p(out, C.c_int)))
    return [int(x) for x in out]


# ---- tensor operations (computed on the GPU) -------------------------------

def transpose(data: np.ndarray, perm) -> np.ndarray:
    """qsim::transpose (include/qsim/tensor.hpp:135-197); perm[i] = input axis at output i."""
    data = np.ascontiguousarray(data, dtype=np.complex64)
    dims = np.asarray(data.shape, dtype=np.int64)
    pa, pp = _i32(perm)
    if len(pa) != data.ndim:
        raise InvalidArgument(1, "transpose: order rank mismatch")
    out = np.zeros(data.size, dtype=np.complex64)
    _check(lib().qsg_transpose(data.ndim, _p(dims, C.c_int64), _p(data.view(np.float32), C.c_float), pp,
                               _p(out.view(np.float32), C.c_float)))
    return out.reshape([data.shape[i] for i in pa])


def contract(llab, ldata, lscale, rlab, rdata, rscale, olab=None, normalize=False):
    """contract_ttgt (+ normalize_inplace) on int-labelled tensors; returns (data, log_scale, flops)."""
    ldata = np.ascontiguousarray(ldata, dtype=np.complex64)
    rdata = np.ascontiguousarray(rdata, dtype=np.complex64)
    la, lp = _i32(llab)
    ra, rp = _i32(rlab)
    dims = dict(zip(list(llab), ldata.shape))
    dims.update(zip(list(rlab), rdata.shape))
    if olab is None:
        olab = [x for x in llab if x not in set(rlab)] + [x for x in rlab if x not in set(llab)]
    oa, op = _i32(olab)
    oshape = [dims[x] for x in olab]
    out = np.zeros(int(np.prod(oshape)) if oshape else 1, dtype=np.complex64)
    ld = np.asarray(ldata.shape, dtype=np.int64)
    rd = np.asarray(rdata.shape, dtype=np.int64)
    osc = C.c_double(0)
    fl = C.c_uint64(0)
    _check(lib().qsg_contract(len(la), lp, _p(ld, C.c_int64), _p(ldata.view(np.float32), C.c_float), lscale,
                              len(ra), rp, _p(rd, C.c_int64), _p(rdata.view(np.float32), C.c_float), rscale,
                              len(oa), op, _p(out.view(np.float32), C.c_float), C.byref(osc), C.byref(fl),
                              1 if normalize else 0))
    return out.reshape(oshape), osc.value, int(fl.value)


def normalize_inplace(data: np.ndarray, log_scale: float = 0.0):
    """normalize_inplace (include/qsim/tensor.hpp:209-224): returns (nonzero, log_scale); data rescaled in place."""
    if data.dtype != np.complex64 or not data.flags.c_contiguous:
        raise ValueError("normalize_inplace needs a C-contiguous complex64 array")
    ls = C.c_double(log_scale)
    nz = C.c_int(0)
    _check(lib().qsg_normalize(_p(data.view(np.float32), C.c_float), data.size, C.byref(ls), C.byref(nz)))
    return bool(nz.value), ls.value


def program_listing(circuit_text: str, plan_text: str = "", kind: int = PLAN_JSON, open_qubits=(),
                    tensor_cores: bool = True, memory_budget: int = 0, device_memory: int = 0) -> str:
    """Device program the engine would run (no GPU needed): ops, GEMM shapes/paths, arena bytes;
    with memory_budget > 0 the out-of-core placement (host arena, piece counts); memory_budget=-1
    picks it automatically for a device of device_memory bytes (default 180 GB)."""
    a, p = _i32(open_qubits)
    return _text(lib().qsg_program_listing_ex, circuit_text.encode(), kind, plan_text.encode(), p, len(a),
                 0 if tensor_cores else 2, int(memory_budget), int(device_memory))


def widen_plan(circuit_text: str, plan_text: str, extra_open, kind: int = PLAN_JSON, open_qubits=()) -> str:
    """The plan with extra qubits opened (same order and cut), as JSON -- an
    engine built on it serves many x1 draws in one contraction
    (Engine.amplitude_batches)."""
    a, p = _i32(open_qubits)
    e, pe = _i32(extra_open)
    return _text(lib().qsg_widen_plan, circuit_text.encode(), kind, plan_text.encode(), p, len(a), pe, len(e))


def reassociate_plan(circuit_text: str, plan_text: str = "", kind: int = PLAN_JSON, open_qubits=()):
    """Opt-in contraction-tree rewrite (no reference counterpart): (A x B) x C
    -> A x (B x C) where that cuts the pair's Eq.(1) flops by >= 25% without a
    larger intermediate, to a fixed point.  Returns (plan JSON, rewrites);
    same cut, slices and amplitudes up to rounding."""
    a, p = _i32(open_qubits)
    r = C.c_int(0)
    n = C.c_int64(0)
    args = (circuit_text.encode(), kind, plan_text.encode(), p, len(a))
    _check(lib().qsg_reassociate_plan(*args, None, 0, C.byref(n), C.byref(r)))
    buf = C.create_string_buffer(n.value + 1)
    _check(lib().qsg_reassociate_plan(*args, buf, n.value + 1, C.byref(n), C.byref(r)))
    return buf.value.decode(), r.value


def xeb_score(n: int, probs, hog_median=None) -> dict:
    """xeb_score (src/sampler.cpp:187-215): cross entropy, 2^n<p>-1 fidelity, HOG fraction."""
    a = np.ascontiguousarray(np.asarray(probs, dtype=np.float64))
    r = _XebReport()
    _check(lib().qsg_xeb_score(n, _p(a, C.c_double), len(a), 0 if hog_median is None else 1,
                               0.0 if hog_median is None else float(hog_median), C.byref(r)))
    return _struct_dict(r)


# ---- engine ---------------------------------------------------------------

def _buffer(buf):
    """(pointer, bytes) of a contiguous numpy array or host torch tensor."""
    if isinstance(buf, np.ndarray):
        if not buf.flags["C_CONTIGUOUS"]:
            raise ValueError("buffer must be contiguous")
        return buf.ctypes.data, buf.nbytes
    if hasattr(buf, "data_ptr"):
        if buf.is_cuda or not buf.is_contiguous():
            raise ValueError("buffer must be a contiguous host tensor")
        return buf.data_ptr(), buf.numel() * buf.element_size()
    raise TypeError("buffer must be a numpy array or a torch tensor")


@dataclass
class EngineInfo:
    num_qubits: int
    num_slices: int
    batch_size: int
    num_steps: int
    max_rank: int
    peak_memory: int
    arena_bytes: int
    node_bytes: int
    flops_per_slice: int
    num_ops: int


class Engine:
    """One GPU's compiled contraction program for (circuit, plan).

    ``kind``: PLAN_JSON (plan_text = plan file contents), PLAN_REF7X7, or
    PLAN_GREEDY (open_qubits, reference greedy planner).
    """

    PROFILE = 1
    NO_TENSOR_CORES = 2

    def __init__(self, circuit_text: str, plan_text: str = "", kind: int = PLAN_JSON, open_qubits=(), device: int = 0,
                 profile: bool = False, tensor_cores: bool = True, memory_budget: int = 0, pipeline_depth: int = 2):
        """memory_budget / pipeline_depth: the reference's ExecOptions (include/qsim/engine.hpp:22-27) --
        steps whose working set exceeds the budget run out of core (host-resident tensors, device pieces)."""
        self._h = C.c_void_p(0)
        a, p = _i32(open_qubits)
        flags = (self.PROFILE if profile else 0) | (0 if tensor_cores else self.NO_TENSOR_CORES)
        _check(lib().qsg_engine_create_ex(circuit_text.encode(), kind, plan_text.encode(), p, len(a), device, flags,
                                          int(memory_budget), int(pipeline_depth), C.byref(self._h)))
        info = _EngineInfo()
        _check(lib().qsg_engine_get_info(self._h, C.byref(info)))
        self.info = EngineInfo(*[getattr(info, f[0]) for f in _EngineInfo._fields_])
        oq = np.zeros(max(1, self.info.batch_size.bit_length() - 1), dtype=np.int32)
        _check(lib().qsg_engine_open_qubits(self._h, _p(oq, C.c_int)))
        self.open_qubits = [int(x) for x in oq[: self.info.batch_size.bit_length() - 1]]
        self.n = self.info.num_qubits

    def close(self):
        if self._h:
            lib().qsg_engine_destroy(self._h)
            self._h = C.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def plan_json(self) -> str:
        return _text(lib().qsg_engine_plan_json, self._h)

    def describe(self) -> str:
        return _text(lib().qsg_engine_describe, self._h)

    def prepare(self, x1_bits) -> int:
        a, p = _i32(x1_bits)
        b = C.c_int64(0)
        _check(lib().qsg_engine_prepare(self._h, p, len(a), C.byref(b)))
        return b.value

    def fold_nodes(self, circuit_text: str, out=None):
        """Host open fold of another instance of this circuit layout, packed
        as the engine's node region (complex64, node_bytes); `out` may be a
        caller buffer (numpy array or a pinned torch tensor)."""
        nb = self.info.node_bytes
        if out is None:
            out = np.empty(nb // 8, dtype=np.complex64)
        ptr, size = _buffer(out)
        if size != nb:
            raise ValueError(f"fold_nodes: buffer is {size} B, node region is {nb} B")
        _check(lib().qsg_engine_fold_nodes(self._h, circuit_text.encode(), ptr, nb))
        return out

    def load_nodes(self, host_nodes):
        """Async H2D of a node region on the engine stream (pinned host memory
        overlaps; keep it alive until the next synchronize)."""
        ptr, size = _buffer(host_nodes)
        _check(lib().qsg_engine_load_nodes(self._h, ptr, size))
        return size

    def export_nodes(self):
        out = np.empty(self.info.node_bytes // 8, dtype=np.complex64)
        _check(lib().qsg_engine_export_nodes(self._h, out.ctypes.data, out.nbytes))
        return out

    def run(self, slice_ids, reset: bool = True, per_slice: bool = False):
        ids = np.ascontiguousarray(np.asarray(list(slice_ids), dtype=np.int64))
        _check(lib().qsg_engine_run(self._h, _p(ids, C.c_int64), len(ids), 1 if reset else 0, 1 if per_slice else 0))

    def per_slice_rows(self) -> int:
        """Slices whose contributions the engine's last run kept (0 if none)."""
        n = C.c_int64(0)
        _check(lib().qsg_engine_per_slice_rows(self._h, C.byref(n)))
        return n.value

    def results(self, per_slice=None):
        """Amplitudes of the last run; with per-slice contributions as well when
        that run kept them (or always when per_slice=True, which raises if the
        last run -- e.g. an internal amplitude_batch -- did not)."""
        rows = self.per_slice_rows()
        if per_slice and rows == 0:
            raise InvalidArgument("results: the last run kept no per-slice contributions")
        want = rows > 0 if per_slice is None else bool(per_slice)
        amps = np.zeros(2 * self.info.batch_size, dtype=np.float64)
        ps = np.zeros(2 * self.info.batch_size * rows, dtype=np.float64) if want else None
        _check(lib().qsg_engine_results(self._h, _p(amps, C.c_double), _p(ps, C.c_double) if ps is not None else None))
        out = amps.view(np.complex128)
        if ps is not None:
            return out, ps.view(np.complex128).reshape(rows, self.info.batch_size)
        return out

    def stream(self) -> int:
        s = C.c_void_p(0)
        _check(lib().qsg_engine_stream(self._h, C.byref(s)))
        return s.value or 0

    def synchronize(self):
        _check(lib().qsg_engine_synchronize(self._h))

    def launches(self) -> int:
        n = C.c_int64(0)
        _check(lib().qsg_engine_launches(self._h, C.byref(n)))
        return n.value

    def profile(self):
        n = C.c_int(0)
        _check(lib().qsg_engine_profile(self._h, None, 0, C.byref(n)))
        arr = (_OpProfile * max(n.value, 1))()
        _check(lib().qsg_engine_profile(self._h, arr, n.value, C.byref(n)))
        return [{f[0]: getattr(arr[i], f[0]) for f in _OpProfile._fields_ if f[0] != "pad"} for i in range(n.value)]

    def set_profile(self, on: bool):
        _check(lib().qsg_engine_set_profile(self._h, 1 if on else 0))

    def reset_profile(self):
        _check(lib().qsg_engine_reset_profile(self._h))

    def amplitude_batch(self, x1_bits, slice_ids):
        """amplitude_batch (src/sampler.cpp:111-120): (bitstrings, complex128 amplitudes)."""
        a, p = _i32(x1_bits)
        ids = np.ascontiguousarray(np.asarray(list(slice_ids), dtype=np.int64))
        amps = np.zeros(2 * self.info.batch_size, dtype=np.float64)
        bits = C.create_string_buffer(len(a) * self.info.batch_size)
        _check(lib().qsg_amplitude_batch(self._h, p, len(a), _p(ids, C.c_int64), len(ids), _p(amps, C.c_double), bits))
        raw = bits.raw
        n = len(a)
        return [raw[i * n:(i + 1) * n].decode() for i in range(self.info.batch_size)], amps.view(np.complex128)

    def amplitude_batches(self, base_open, x1_list, slice_ids, bitstrings: bool = True):
        """amplitude_batch for many x1 draws in ONE contraction on an engine built
        from widen_plan(...): per draw (bitstrings, complex128 amplitudes), or with
        bitstrings=False the [draws, 2^|open|] amplitude array alone."""
        b, pb = _i32(base_open)
        xs = np.ascontiguousarray(np.asarray(x1_list, dtype=np.int32))
        nx1, n = xs.shape
        ids = np.ascontiguousarray(np.asarray(list(slice_ids), dtype=np.int64))
        per = 1 << len(b)
        amps = np.empty(2 * per * nx1, dtype=np.float64)  # every entry is written
        bits = C.create_string_buffer(max(1, n * per * nx1)) if bitstrings else None
        _check(lib().qsg_amplitude_batches(self._h, pb, len(b), _p(xs, C.c_int), nx1, n, _p(ids, C.c_int64), len(ids),
                                           _p(amps, C.c_double), bits))
        amps = amps.view(np.complex128).reshape(nx1, per)
        if not bitstrings:
            return amps
        raw = bits.raw
        return [([raw[(t * per + j) * n:(t * per + j + 1) * n].decode() for j in range(per)], amps[t])
                for t in range(nx1)]

    def amplitude_batches_submit(self, base_open, x1_list, slice_ids, slot: int = 0):
        """Pipelined amplitude_batches: enqueue the contraction and the D2H of its
        batch into staging slot 0/1 and return; amplitude_batches_collect(slot)
        later returns the [draws, 2^|open|] amplitudes (or (bitstrings, amps))."""
        b, pb = _i32(base_open)
        xs = np.ascontiguousarray(np.asarray(x1_list, dtype=np.int32))
        nx1, n = xs.shape
        ids = np.ascontiguousarray(np.asarray(list(slice_ids), dtype=np.int64))
        _check(lib().qsg_amplitude_batches_submit(self._h, pb, len(b), _p(xs, C.c_int), nx1, n, _p(ids, C.c_int64),
                                                  len(ids), slot))
        self._pending = getattr(self, "_pending", {})
        self._pending[slot] = (b, xs)

    def amplitude_batches_collect(self, slot: int = 0, bitstrings: bool = False):
        b, xs = self._pending.pop(slot)
        nx1, n = xs.shape
        per = 1 << len(b)
        amps = np.empty(2 * per * nx1, dtype=np.float64)
        bits = C.create_string_buffer(max(1, n * per * nx1)) if bitstrings else None
        _check(lib().qsg_amplitude_batches_collect(self._h, _p(b, C.c_int), len(b), _p(xs, C.c_int), nx1, n, slot,
                                                   _p(amps, C.c_double), bits))
        amps = amps.view(np.complex128).reshape(nx1, per)
        if not bitstrings:
            return amps
        raw = bits.raw
        return [([raw[(t * per + j) * n:(t * per + j + 1) * n].decode() for j in range(per)], amps[t])
                for t in range(nx1)]

    def sample(self, num_samples: int, fraction=(0, 0), amplitude_fraction: bool = False, cap: float = 6.0,
               seed: int = 0):
        """sample / sample_amplitude_fraction (src/sampler.cpp:122-185):
        (bitstrings, probabilities, stats, self_xeb)."""
        n = self.n
        bits = C.create_string_buffer(max(1, num_samples * n))
        probs = np.zeros(max(1, num_samples), dtype=np.float64)
        st, xr = _SampleStats(), _XebReport()
        _check(lib().qsg_sample(self._h, num_samples, fraction[0], fraction[1], 1 if amplitude_fraction else 0, cap,
                                seed, bits, _p(probs, C.c_double), C.byref(st), C.byref(xr)))
        raw = bits.raw
        return ([raw[i * n:(i + 1) * n].decode() for i in range(num_samples)], probs[:num_samples],
                _struct_dict(st), _struct_dict(xr))

    def run_amplitudes(self, bitstrings, fraction=(0, 0), seed: int = 0):
        """run_amplitudes (src/engine.cpp:300-378): (amplitudes, slice_ids, flops)."""
        n = self.n
        joined = "".join(bitstrings).encode()
        out = np.zeros(2 * len(bitstrings), dtype=np.float64)
        k = fraction[0] if fraction[1] > 0 else self.info.num_slices
        ids = np.zeros(max(k, 1), dtype=np.int64)
        fl = C.c_uint64(0)
        _check(lib().qsg_run_amplitudes(self._h, joined, len(bitstrings), n, fraction[0], fraction[1], seed,
                                        _p(out, C.c_double), _p(ids, C.c_int64), C.byref(fl)))
        return out.view(np.complex128), [int(x) for x in ids[:k]], int(fl.value)
