"""ctypes binding to oracle/_ref/libqsim_ref.so -- the UNMODIFIED reference
library (/root/reference/proj/src) built by oracle/Makefile.

TEST INFRASTRUCTURE ONLY.  Imported by tests/, oracle/gen_golden.py and the
CPU-baseline leg of bench.py, as the checker / the timed reference arm.  The
product (paper_1905_00444_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import struct

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# QSIM_REF_LIB selects another build of the same library, e.g.
# _ref/libqsim_relink.so (the reference relinked onto libqsg.so,
# oracle/Makefile `relink`).
LIB_PATH = os.environ.get("QSIM_REF_LIB") or os.path.join(_HERE, "_ref", "libqsim_ref.so")
RELINK_PATH = os.path.join(_HERE, "_ref", "libqsim_relink.so")

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"reference oracle not built: {LIB_PATH} (run make -C oracle)")
        L = C.CDLL(LIB_PATH)
        i64, u64, i32 = C.c_int64, C.c_uint64, C.c_int
        P = C.POINTER
        L.ref_last_error.restype = C.c_char_p
        L.ref_mix_seed.restype = u64
        L.ref_mix_seed.argtypes = [u64, u64]
        L.ref_set_blas_threads.argtypes = [i32]
        L.ref_generate_rqc.argtypes = [i32, i32, i32, u64, C.c_char_p, i64, P(i64)]
        L.ref_canonical_circuit.argtypes = [C.c_char_p, C.c_char_p, i64, P(i64)]
        L.ref_evolve.argtypes = [C.c_char_p, P(C.c_double), i64]
        L.ref_plan_json.argtypes = [C.c_char_p, P(i32), i32, i32, C.c_char_p, i64, C.c_char_p, i64, P(i64)]
        L.ref_fold_qtns.argtypes = [C.c_char_p, P(i32), i32, C.c_char_p, i64, C.c_char_p, i64, P(i64)]
        L.ref_select_slices.argtypes = [i64, i64, i64, u64, P(i64)]
        L.ref_amplitude_batch.argtypes = [C.c_char_p, C.c_char_p, i32, P(i32), i32, P(i64), i64,
                                          P(C.c_double), C.c_char_p]
        L.ref_run_amplitudes.argtypes = [C.c_char_p, C.c_char_p, i32, C.c_char_p, i32, i32, i64, i64,
                                         i32, u64, P(C.c_double), P(i64), P(u64)]
        L.ref_transpose.argtypes = [i32, P(i64), P(C.c_float), P(i32), P(C.c_float)]
        L.ref_contract_step.argtypes = [i32, P(i32), P(i64), P(C.c_float), C.c_double,
                                        i32, P(i32), P(i64), P(C.c_float), C.c_double,
                                        i32, P(i32), P(C.c_float), P(C.c_double), P(u64), i32]
        L.ref_execute_prefix.argtypes = [C.c_char_p, C.c_char_p, i32, P(i32), i32, i32, i32, i32, u64,
                                         P(C.c_double), P(u64)]
        L.ref_sample.argtypes = [C.c_char_p, C.c_char_p, i64, i64, i64, i32, C.c_double, u64, C.c_char_p,
                                 P(C.c_double)]
        L.ref_sample.restype = i32
        for name in ("ref_generate_rqc", "ref_canonical_circuit", "ref_evolve", "ref_plan_json",
                     "ref_fold_qtns", "ref_select_slices", "ref_amplitude_batch", "ref_run_amplitudes",
                     "ref_transpose", "ref_contract_step", "ref_execute_prefix"):
            getattr(L, name).restype = i32
        L.ref_set_blas_threads(1)  # mirrors EIGEN_DONT_PARALLELIZE (proj/CMakeLists.txt:15-17)
        _lib = L
    return _lib


class RefError(RuntimeError):
    pass


def _check(rc):
    if rc != 0:
        raise RefError(lib().ref_last_error().decode())


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _i32(seq):
    a = np.ascontiguousarray(np.asarray(seq, dtype=np.int32))
    return a, _ptr(a, C.c_int)


def _string_call(fn, *args):
    n = C.c_int64(0)
    _check(fn(*args, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(fn(*args, buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def mix_seed(seed: int, stream: int) -> int:
    return int(lib().ref_mix_seed(seed, stream))


def generate_rqc(rows: int, cols: int, m: int, seed: int) -> str:
    return _string_call(lib().ref_generate_rqc, rows, cols, m, seed)


def canonical_circuit(text: str) -> str:
    return _string_call(lib().ref_canonical_circuit, text.encode())


def evolve(text: str, n: int) -> np.ndarray:
    out = np.zeros(2 << n, dtype=np.float64)
    _check(lib().ref_evolve(text.encode(), _ptr(out, C.c_double), 1 << n))
    return out.view(np.complex128)


PLAN_JSON, PLAN_REF7X7, PLAN_GREEDY = 0, 1, 2


def plan_json(text: str, open_qubits, kind=PLAN_JSON, plan_text: str = "", budget: int = 0) -> str:
    a, p = _i32(open_qubits)
    return _string_call(lib().ref_plan_json, text.encode(), p, len(a), kind, plan_text.encode(), budget)


def parse_qtns(blob: bytes):
    """QTNS dumps (include/qsim/tensor_io.hpp:12-41) -> list of (labels, dims, log_scale, data)."""
    out, off = [], 0
    while off < len(blob):
        assert blob[off:off + 4] == b"QTNS"
        ver, rank = struct.unpack_from("<II", blob, off + 4)
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


def fold(text: str, out_bits, plan_text: str = "", slice_id: int = 0):
    a, p = _i32(out_bits)
    n = C.c_int64(0)
    _check(lib().ref_fold_qtns(text.encode(), p, len(a), plan_text.encode(), slice_id, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value)
    _check(lib().ref_fold_qtns(text.encode(), p, len(a), plan_text.encode(), slice_id, buf, n.value, C.byref(n)))
    return parse_qtns(buf.raw[: n.value])


def select_slices(num: int, den: int, num_slices: int, seed: int) -> list[int]:
    out = np.zeros(num, dtype=np.int64)
    _check(lib().ref_select_slices(num, den, num_slices, seed, _ptr(out, C.c_int64)))
    return [int(x) for x in out]


def amplitude_batch(text: str, plan_text: str, x1, slice_ids, kind=PLAN_JSON):
    """(bitstrings, complex128 amplitudes) of src/sampler.cpp:111-120."""
    a, p = _i32(x1)
    n = len(a)
    nopen = int((a < 0).sum())
    ids = np.ascontiguousarray(np.asarray(slice_ids, dtype=np.int64))
    out = np.zeros(2 << nopen, dtype=np.float64)
    bits = C.create_string_buffer(n * (1 << nopen))
    _check(lib().ref_amplitude_batch(text.encode(), plan_text.encode(), kind, p, n, _ptr(ids, C.c_int64),
                                     len(ids), _ptr(out, C.c_double), bits))
    raw = bits.raw
    bs = [raw[i * n:(i + 1) * n].decode() for i in range(1 << nopen)]
    return bs, out.view(np.complex128)


def run_amplitudes(text: str, plan_text: str, bitstrings, frac=(0, 0), workers=1, seed=0, kind=PLAN_JSON):
    n = len(bitstrings[0])
    joined = "".join(bitstrings).encode()
    out = np.zeros(2 * len(bitstrings), dtype=np.float64)
    k = frac[0] if frac[1] > 0 else 0
    ids = np.zeros(max(k, 1) if k else 1 << 16, dtype=np.int64)
    flops = C.c_uint64(0)
    _check(lib().ref_run_amplitudes(text.encode(), plan_text.encode(), kind, joined, len(bitstrings), n,
                                    frac[0], frac[1], workers, seed, _ptr(out, C.c_double),
                                    _ptr(ids, C.c_int64), C.byref(flops)))
    return out.view(np.complex128), int(flops.value)


def transpose(data: np.ndarray, perm) -> np.ndarray:
    """qsim::transpose (include/qsim/tensor.hpp:135-197); perm[i] = input axis at output i."""
    data = np.ascontiguousarray(data, dtype=np.complex64)
    dims = np.asarray(data.shape, dtype=np.int64)
    pa, pp = _i32(perm)
    out = np.zeros(data.size, dtype=np.complex64)
    _check(lib().ref_transpose(data.ndim, _ptr(dims, C.c_int64), _ptr(data.view(np.float32), C.c_float), pp,
                               _ptr(out.view(np.float32), C.c_float)))
    return out.reshape([data.shape[i] for i in perm])


def contract_step(llab, ldata, lscale, rlab, rdata, rscale, olab, normalize=True):
    """contract_ttgt + normalize_inplace (src/engine.cpp:211-233) on int-labelled tensors."""
    ldata = np.ascontiguousarray(ldata, dtype=np.complex64)
    rdata = np.ascontiguousarray(rdata, dtype=np.complex64)
    la, lp = _i32(llab)
    ra, rp = _i32(rlab)
    oa, op = _i32(olab)
    ld = np.asarray(ldata.shape, dtype=np.int64)
    rd = np.asarray(rdata.shape, dtype=np.int64)
    dims = {}
    for lab, d in zip(llab, ldata.shape):
        dims[lab] = d
    for lab, d in zip(rlab, rdata.shape):
        dims[lab] = d
    oshape = [dims[x] for x in olab]
    out = np.zeros(int(np.prod(oshape)) if oshape else 1, dtype=np.complex64)
    osc = C.c_double(0)
    fl = C.c_uint64(0)
    _check(lib().ref_contract_step(len(la), lp, _ptr(ld, C.c_int64), _ptr(ldata.view(np.float32), C.c_float),
                                   lscale, len(ra), rp, _ptr(rd, C.c_int64),
                                   _ptr(rdata.view(np.float32), C.c_float), rscale, len(oa), op,
                                   _ptr(out.view(np.float32), C.c_float), C.byref(osc), C.byref(fl),
                                   1 if normalize else 0))
    return out.reshape(oshape), osc.value, int(fl.value)


def execute_prefix(text: str, plan_text: str, open_qubits, nsteps: int, ntasks: int, threads: int,
                   seed: int = 0, kind=PLAN_JSON):
    """Times the reference's step kernels over the first nsteps plan steps of ntasks slices."""
    a, p = _i32(open_qubits)
    sec = C.c_double(0)
    fl = C.c_uint64(0)
    _check(lib().ref_execute_prefix(text.encode(), plan_text.encode(), kind, p, len(a), nsteps, ntasks, threads,
                                    seed, C.byref(sec), C.byref(fl)))
    return sec.value, int(fl.value)


def sample(text: str, plan_text: str, num_samples: int, frac=(0, 0), amplitude_mode=False, cap=6.0, seed=0):
    """The reference sample() (src/sampler.cpp:122-178): (bitstrings, probabilities)."""
    n = int(text.split("\n", 1)[0])
    bits = C.create_string_buffer(num_samples * n)
    probs = np.zeros(num_samples, dtype=np.float64)
    _check(lib().ref_sample(text.encode(), plan_text.encode(), num_samples, frac[0], frac[1],
                            1 if amplitude_mode else 0, cap, seed, bits, _ptr(probs, C.c_double)))
    raw = bits.raw
    return [raw[i * n:(i + 1) * n].decode() for i in range(num_samples)], probs
