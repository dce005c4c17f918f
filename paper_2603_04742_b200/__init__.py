"""B200-native RNS-BFV evaluation of the CSSC encrypted SpMV (arxiv 2603.04742).

Thin ctypes layer over the in-tree native library ``lib/libcssc_he.so``
(CUDA sm_100a kernels + C++ host, C-ABI in ``include/spmvgpu.h``).  There is
no Python or CPU fallback: importing works without a GPU (so the C-ABI can be
inspected), but every compute call goes through the native library and fails
loudly when it is missing or when no CUDA device is present.

Mirrors of the reference API (``/root/reference/proj/include/spmv``):
  Context           ~ HeParams + SimBackend construction (he.hpp:35-43, 119-139)
  Context.encrypt / decrypt / add / mul_relin / mul_plain / rotate
                    ~ HeBackend virtuals (he.hpp:95-114)
  spmv_partitioned  ~ spmv::spmv_partitioned (protocol.hpp:69-71)
  spmv_batch        ~ several independent spmv_partitioned runs in shared launches
  Job               staged pack/encrypt -> cloud -> decrypt, for benchmarking
"""
from __future__ import annotations

import ctypes as C
import os
import weakref
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
# CSSC_LIB selects another build of the same library (the sanitizer build of
# tools/asan_check.sh); the default is the in-tree product build
LIB_PATH = Path(os.environ["CSSC_LIB"]) if os.environ.get("CSSC_LIB") else _PKG / "lib" / "libcssc_he.so"

u64p = C.POINTER(C.c_uint64)
i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)
u32p = C.POINTER(C.c_uint32)


class SpmvgpuParams(C.Structure):
    _fields_ = [("logn", C.c_int), ("L", C.c_int), ("K", C.c_int), ("alpha", C.c_int),
                ("qbits", C.c_int), ("pbits", C.c_int), ("t", C.c_uint64), ("seed", C.c_uint64),
                ("device", C.c_int), ("ciphertext_size_mb", C.c_double),
                ("noise_initial", C.c_int), ("noise_ct_ct", C.c_int), ("noise_ct_pt", C.c_int),
                ("noise_add", C.c_int), ("noise_rot", C.c_int)]


class PlanStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "chunks", "slices", "levels", "kernels_per_run", "limb_ntts_per_run", "rotations",
        "distinct_keys", "hbm_bytes_algorithmic", "key_bytes_per_run", "relin_folded")]


class Ledger(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("n_mult_cc", "n_mult_cp", "n_rot", "n_add", "n_enc", "n_dec")]


class Message(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("from_", "to", "kind", "payload_bytes", "ciphertext_count")]


class PhaseC(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("us", C.c_double), ("items", C.c_uint64), ("bytes", C.c_uint64),
                ("limb_ntts", C.c_uint64), ("sources", C.c_uint64),
                ("acc_items", C.c_uint64), ("mac_terms", C.c_uint64)]


class KernelTimingC(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("group", C.c_int32), ("us", C.c_double)]


class CsrC(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("cols", C.c_uint64), ("row_ptrs", i64p),
                ("col_indices", i64p), ("values", i64p)]


class ResultC(C.Structure):
    _fields_ = [("ledger", Ledger), ("n_ct", C.c_uint64), ("noise_model_bits", C.c_int32),
                ("noise_measured_bits", C.c_int32), ("n_messages", C.c_uint64)]


# C-ABI symbol table: name -> (restype, argtypes).  tests check every entry
# against include/spmvgpu.h.
_SIGS = {
    "spmvgpu_last_error": (C.c_char_p, []),
    "spmvgpu_default_params": (None, [C.c_int, C.POINTER(SpmvgpuParams)]),
    "spmvgpu_ctx_create": (C.c_int, [C.POINTER(SpmvgpuParams), C.POINTER(C.c_void_p)]),
    "spmvgpu_ctx_destroy": (None, [C.c_void_p]),
    "spmvgpu_ctx_primes": (C.c_int, [C.c_void_p, u64p, C.c_int, C.POINTER(C.c_int)]),
    "spmvgpu_ctx_sizes": (C.c_int, [C.c_void_p, u64p, u64p, u64p, u64p, C.POINTER(C.c_int)]),
    "spmvgpu_sync": (C.c_int, [C.c_void_p]),
    "spmvgpu_set_option": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int64]),
    "spmvgpu_stream": (C.c_void_p, [C.c_void_p]),
    "spmvgpu_galois_keys": (C.c_int, [C.c_void_p, i64p, C.c_size_t]),
    "spmvgpu_galois_element": (C.c_uint32, [C.c_void_p, C.c_int64]),
    "spmvgpu_download_sk": (C.c_int, [C.c_void_p, i64p]),
    "spmvgpu_download_pk": (C.c_int, [C.c_void_p, u64p]),
    "spmvgpu_download_ksk": (C.c_int, [C.c_void_p, C.c_uint32, u64p]),
    "spmvgpu_ct_alloc": (C.c_int, [C.c_void_p, C.c_size_t, u64p]),
    "spmvgpu_ct_free": (C.c_int, [C.c_void_p, u64p, C.c_size_t]),
    "spmvgpu_ct_upload": (C.c_int, [C.c_void_p, C.c_uint64, u64p]),
    "spmvgpu_ct_download": (C.c_int, [C.c_void_p, C.c_uint64, u64p]),
    "spmvgpu_ct_wire_size": (C.c_int, [C.c_void_p, C.POINTER(C.c_size_t)]),
    "spmvgpu_ct_serialize": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(C.c_uint8), C.c_size_t,
                                       C.POINTER(C.c_size_t)]),
    "spmvgpu_ct_deserialize": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint8), C.c_size_t, C.c_uint64]),
    "spmvgpu_encrypt": (C.c_int, [C.c_void_p, i64p, u64p, u64p, u64p, C.c_size_t]),
    "spmvgpu_encrypt_cssc": (C.c_int, [C.c_void_p, i64p, i64p, C.c_uint64, i64p, C.c_uint64, i32p, C.c_uint64,
                                       i32p, C.c_uint64, i32p, C.c_uint64, u64p, C.c_size_t]),
    "spmvgpu_decrypt": (C.c_int, [C.c_void_p, u64p, C.c_size_t, u64p, i32p]),
    "spmvgpu_add": (C.c_int, [C.c_void_p, u64p, u64p, u64p, C.c_size_t]),
    "spmvgpu_mul_relin": (C.c_int, [C.c_void_p, u64p, u64p, u64p, C.c_size_t]),
    "spmvgpu_rotate": (C.c_int, [C.c_void_p, u64p, i64p, u64p, C.c_size_t]),
    "spmvgpu_rotate_add": (C.c_int, [C.c_void_p, u64p, u64p, i64p, u64p, C.c_size_t]),
    "spmvgpu_mul_plain": (C.c_int, [C.c_void_p, u64p, i64p, u64p, u64p, C.c_size_t]),
    "spmvgpu_ntt": (C.c_int, [C.c_void_p, C.c_int, u64p, C.c_size_t, C.c_int]),
    "spmvgpu_probe_ntt": (C.c_int, [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.POINTER(C.c_double)]),
    "spmvgpu_probe_butterfly_peak": (C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    "spmvgpu_plan_create": (C.c_int, [C.c_void_p, C.c_size_t, u64p, u64p, u32p, C.c_size_t,
                                      u64p, u64p, u64p, C.POINTER(C.c_void_p)]),
    "spmvgpu_plan_run": (C.c_int, [C.c_void_p]),
    "spmvgpu_plan_capture": (C.c_int, [C.c_void_p]),
    "spmvgpu_plan_stats_get": (C.c_int, [C.c_void_p, C.POINTER(PlanStats)]),
    "spmvgpu_plan_profile": (C.c_int, [C.c_void_p, C.POINTER(PhaseC), C.c_int, C.POINTER(C.c_int)]),
    "spmvgpu_plan_profile_kernels": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, C.POINTER(KernelTimingC), C.c_int,
                                               C.POINTER(C.c_int)]),
    "spmvgpu_plan_destroy": (None, [C.c_void_p]),
    "cssc_spmv_partitioned": (C.c_int, [C.c_void_p, C.POINTER(CsrC), i64p, C.c_uint64, C.c_uint64,
                                        C.c_int, i64p, C.POINTER(ResultC), C.POINTER(Message),
                                        C.c_uint64]),
    "cssc_spmv": (C.c_int, [C.c_void_p, C.POINTER(CsrC), i64p, C.c_uint64, C.c_uint64, C.c_int, i64p,
                            C.POINTER(ResultC), C.POINTER(Message), C.c_uint64]),
    "cssc_diag_spmv": (C.c_int, [C.c_void_p, C.POINTER(CsrC), i64p, C.c_uint64, C.c_int, i64p,
                                 C.POINTER(ResultC), C.POINTER(Message), C.c_uint64]),
    "spmvgpu_sum": (C.c_int, [C.c_void_p, u64p, C.c_size_t, C.c_uint64]),
    "cssc_speculate": (C.c_int, [C.c_void_p]),
    "cssc_spmv_batch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                  C.c_uint64, C.c_int, C.c_void_p, C.c_void_p]),
    "cssc_job_create": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                  C.c_uint64, C.POINTER(C.c_void_p)]),
    "cssc_job_create_shard": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint64,
                                        C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "cssc_job_result_words": (C.c_int, [C.c_void_p, u64p, C.c_uint64, u64p]),
    "cssc_job_finish_words": (C.c_int, [C.c_void_p, u64p, C.c_void_p, C.c_void_p]),
    "cssc_job_result_words_dev": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, u64p]),
    "cssc_job_finish_words_dev": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "spmvgpu_fold_mod": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64]),
    "cssc_job_encrypt": (C.c_int, [C.c_void_p]),
    "cssc_job_cloud": (C.c_int, [C.c_void_p, C.c_int]),
    "cssc_job_cloud_timed": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]),
    "cssc_job_finish": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "cssc_job_run": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "cssc_job_plan_stats": (C.c_int, [C.c_void_p, C.POINTER(PlanStats)]),
    "cssc_job_profile": (C.c_int, [C.c_void_p, C.POINTER(PhaseC), C.c_int, C.POINTER(C.c_int)]),
    "cssc_job_profile_kernels": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, C.POINTER(KernelTimingC), C.c_int,
                                           C.POINTER(C.c_int)]),
    "cssc_job_input_bytes": (C.c_int, [C.c_void_p, u64p, u64p]),
    "cssc_job_destroy": (None, [C.c_void_p]),
    "cssc_pack_chunks": (C.c_int64, [C.POINTER(CsrC), C.c_uint64, i64p, i64p, i64p, i64p, i64p, u64p]),
    "cssc_rotation_schedule": (C.c_int, [C.c_uint64, C.c_uint64, u64p, i32p]),
    "cssc_convert_binary": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, u64p]),
    "cssc_convert_json": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, u64p]),
    "cssc_load_binary": (C.c_int, [C.c_void_p, C.c_uint64, u64p, u64p, u64p, u64p, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p]),
}

_lib = None


def lib() -> C.CDLL:
    """Load the native library (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"native library missing: {LIB_PATH} (run __graft_entry__.build())")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


STATUS = {-1: ValueError, -2: "OverLengthError", -3: "NoiseExhaustedError", -4: "DimensionMismatchError",
          -5: "ColumnTooTallError", -6: "IndexOutOfRangeError", -7: "DuplicateEntryError",
          -8: RuntimeError, -9: RuntimeError, -10: "NonSquareError", -11: "ParseError"}


class SpmvError(RuntimeError):
    def __init__(self, status: int, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.status, self.kind = status, kind


def check(status: int) -> None:
    if status != 0:
        kind = STATUS.get(status, RuntimeError)
        name = kind if isinstance(kind, str) else kind.__name__
        raise SpmvError(status, name, lib().spmvgpu_last_error().decode())


def _p(a: np.ndarray, t):
    """Typed pointer to a's data (keeps a alive); from_buffer is ~4x cheaper
    than ndarray.ctypes.data_as, which stays as the fallback (read-only or
    empty arrays)."""
    try:
        return C.pointer(t._type_.from_buffer(a))
    except (TypeError, ValueError, BufferError):
        return a.ctypes.data_as(t)


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def default_params(logn: int) -> SpmvgpuParams:
    p = SpmvgpuParams()
    lib().spmvgpu_default_params(logn, C.byref(p))
    return p


class Context:
    """Device-resident RNS-BFV context (keys generated on the GPU).  seed=None
    (default) draws a 256-bit key from OS entropy; an integer seed gives the
    deterministic key the CPU oracle restates (tests, known answers)."""

    def __init__(self, logn: int = 14, seed: int | None = None, device: int = 0, **overrides):
        p = default_params(logn)
        p.seed = 0 if seed is None else int(seed)
        if seed is not None and p.seed == 0:
            raise ValueError("seed must be nonzero (None draws the key from OS entropy)")
        p.device = device
        for k, v in overrides.items():
            setattr(p, k, v)
        self.params = p
        h = C.c_void_p()
        check(lib().spmvgpu_ctx_create(C.byref(p), C.byref(h)))
        self.h = h
        n, s, ctw, kw = (C.c_uint64() for _ in range(4))
        dn = C.c_int()
        check(lib().spmvgpu_ctx_sizes(h, C.byref(n), C.byref(s), C.byref(ctw), C.byref(kw), C.byref(dn)))
        self.n, self.slots, self.ct_words, self.ksk_words, self.dnum = n.value, s.value, ctw.value, kw.value, dn.value
        buf = np.zeros(64, np.uint64)
        cnt = C.c_int()
        check(lib().spmvgpu_ctx_primes(h, _p(buf, u64p), 64, C.byref(cnt)))
        self.primes = [int(x) for x in buf[:cnt.value]]
        self.L, self.K = p.L, p.K

    def close(self):
        if getattr(self, "h", None):
            lib().spmvgpu_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- memory
    def alloc(self, n: int) -> np.ndarray:
        hs = np.zeros(n, np.uint64)
        if n:
            check(lib().spmvgpu_ct_alloc(self.h, n, _p(hs, u64p)))
        return hs

    def free(self, hs) -> None:
        hs = _u64(hs)
        if hs.size:
            check(lib().spmvgpu_ct_free(self.h, _p(hs, u64p), hs.size))

    def upload(self, ct: int, words: np.ndarray) -> None:
        w = _u64(words)
        assert w.size == self.ct_words
        check(lib().spmvgpu_ct_upload(self.h, int(ct), _p(w, u64p)))

    def download(self, ct: int) -> np.ndarray:
        w = np.zeros(self.ct_words, np.uint64)
        check(lib().spmvgpu_ct_download(self.h, int(ct), _p(w, u64p)))
        return w

    # ---- wire format
    @property
    def wire_size(self) -> int:
        b = C.c_size_t()
        check(lib().spmvgpu_ct_wire_size(self.h, C.byref(b)))
        return b.value

    def serialize(self, ct: int) -> bytes:
        buf = np.zeros(self.wire_size, np.uint8)
        w = C.c_size_t()
        check(lib().spmvgpu_ct_serialize(self.h, int(ct), buf.ctypes.data_as(C.POINTER(C.c_uint8)), buf.size,
                                         C.byref(w)))
        return buf[: w.value].tobytes()

    def deserialize(self, data: bytes) -> int:
        buf = np.frombuffer(data, np.uint8).copy()
        out = self.alloc(1)
        try:
            check(lib().spmvgpu_ct_deserialize(self.h, buf.ctypes.data_as(C.POINTER(C.c_uint8)), buf.size,
                                               int(out[0])))
        except Exception:
            self.free(out)
            raise
        return int(out[0])

    # ---- keys
    def download_sk(self) -> np.ndarray:
        s = np.zeros(self.n, np.int64)
        check(lib().spmvgpu_download_sk(self.h, _p(s, i64p)))
        return s

    def download_pk(self) -> np.ndarray:
        w = np.zeros(2 * self.L * self.n, np.uint64)
        check(lib().spmvgpu_download_pk(self.h, _p(w, u64p)))
        return w

    def download_ksk(self, which: int) -> np.ndarray:
        w = np.zeros(self.ksk_words, np.uint64)
        check(lib().spmvgpu_download_ksk(self.h, which, _p(w, u64p)))
        return w

    def galois_element(self, step: int) -> int:
        return int(lib().spmvgpu_galois_element(self.h, step))

    # ---- batched ops
    def encrypt(self, values, streams=None) -> np.ndarray:
        vals = [_i64(v) for v in values]
        offs = np.zeros(len(vals) + 1, np.uint64)
        offs[1:] = np.cumsum([v.size for v in vals])
        flat = _i64(np.concatenate(vals)) if vals and offs[-1] else np.zeros(1, np.int64)
        out = self.alloc(len(vals))
        st = _u64(streams) if streams is not None else None
        check(lib().spmvgpu_encrypt(self.h, _p(flat, i64p), _p(offs, u64p),
                                    _p(st, u64p) if st is not None else None, _p(out, u64p), len(vals)))
        return out

    def encrypt_cssc(self, col_indices, values, vec, rows, slices, cols, n_chunks: int) -> np.ndarray:
        """Device pack + encrypt (spmvgpu_encrypt_cssc); returns 2 n_chunks handles
        (value chunks, then vector chunks)."""
        ci, va, v = _i64(col_indices), _i64(values), _i64(vec)
        r, sl, co = (np.ascontiguousarray(x, np.int32).reshape(-1) for x in (rows, slices, cols))
        out = self.alloc(2 * n_chunks)
        try:
            check(lib().spmvgpu_encrypt_cssc(self.h, _p(ci, i64p), _p(va, i64p), ci.size, _p(v, i64p), v.size,
                                             _p(r, i32p), r.size // 4, _p(sl, i32p), sl.size // 2,
                                             _p(co, i32p), co.size // 4, _p(out, u64p), n_chunks))
        except Exception:
            self.free(out)
            raise
        return out

    def decrypt(self, cts):
        cts = _u64(cts)
        slots = np.zeros((cts.size, self.slots), np.uint64)
        b = np.zeros(cts.size, np.int32)
        check(lib().spmvgpu_decrypt(self.h, _p(cts, u64p), cts.size, _p(slots, u64p), _p(b, i32p)))
        return slots, b

    def sum(self, cts) -> int:
        """One ciphertext = the sum of `cts` (one launch); caller frees it."""
        cts = _u64(cts)
        out = self.alloc(1)
        check(lib().spmvgpu_sum(self.h, _p(cts, u64p) if cts.size else None, cts.size, int(out[0])))
        return int(out[0])

    def add(self, a, b) -> np.ndarray:
        a, b = _u64(a), _u64(b)
        out = self.alloc(a.size)
        check(lib().spmvgpu_add(self.h, _p(a, u64p), _p(b, u64p), _p(out, u64p), a.size))
        return out

    def mul_relin(self, a, b) -> np.ndarray:
        a, b = _u64(a), _u64(b)
        out = self.alloc(a.size)
        check(lib().spmvgpu_mul_relin(self.h, _p(a, u64p), _p(b, u64p), _p(out, u64p), a.size))
        return out

    def rotate(self, a, steps) -> np.ndarray:
        a, st = _u64(a), _i64(steps)
        out = self.alloc(a.size)
        check(lib().spmvgpu_rotate(self.h, _p(a, u64p), _p(st, i64p), _p(out, u64p), a.size))
        return out

    def rotate_add(self, acc, src, steps) -> np.ndarray:
        acc, src, st = _u64(acc), _u64(src), _i64(steps)
        out = self.alloc(acc.size)
        check(lib().spmvgpu_rotate_add(self.h, _p(acc, u64p), _p(src, u64p), _p(st, i64p), _p(out, u64p),
                                       acc.size))
        return out

    def mul_plain(self, a, values) -> np.ndarray:
        a = _u64(a)
        vals = [_i64(v) for v in values]
        offs = np.zeros(len(vals) + 1, np.uint64)
        offs[1:] = np.cumsum([v.size for v in vals])
        flat = _i64(np.concatenate(vals)) if offs[-1] else np.zeros(1, np.int64)
        out = self.alloc(a.size)
        check(lib().spmvgpu_mul_plain(self.h, _p(a, u64p), _p(flat, i64p), _p(offs, u64p), _p(out, u64p),
                                      a.size))
        return out

    def ntt(self, prime_index: int, data: np.ndarray, inverse: bool = False) -> np.ndarray:
        d = _u64(data).copy()
        limbs = d.size // self.n
        check(lib().spmvgpu_ntt(self.h, prime_index, _p(d, u64p), limbs, int(inverse)))
        return d

    def sync(self):
        check(lib().spmvgpu_sync(self.h))

    def set_option(self, name: str, value: int) -> None:
        check(lib().spmvgpu_set_option(self.h, name.encode(), int(value)))

    def stream_ptr(self) -> int:
        return int(lib().spmvgpu_stream(self.h) or 0)

    def probe_ntt_us(self, limbs: int, inverse: bool = False, reps: int = 20) -> float:
        us = C.c_double()
        check(lib().spmvgpu_probe_ntt(self.h, limbs, int(inverse), reps, C.byref(us)))
        return us.value

    def probe_butterfly_peak(self) -> float:
        bps = C.c_double()
        check(lib().spmvgpu_probe_butterfly_peak(self.h, C.byref(bps)))
        return bps.value


def cloud_plan(ctx: Context, r_list, c_list, slice_ids, n_slices: int, a_cts, b_cts, graph: bool = False,
               stats: dict | None = None):
    """Run the batched cloud phase on raw ciphertext handles (device level):
    returns one result-ciphertext handle per slice (caller frees them); `stats`
    (optional dict) receives the plan's statistics."""
    n = len(r_list)
    r = _u64(r_list)
    c = _u64(c_list)
    s = np.ascontiguousarray(np.asarray(slice_ids, dtype=np.uint32))
    a, b = _u64(a_cts), _u64(b_cts)
    out = ctx.alloc(n_slices)
    h = C.c_void_p()
    check(lib().spmvgpu_plan_create(ctx.h, n, _p(r, u64p), _p(c, u64p), _p(s, u32p), n_slices, _p(a, u64p),
                                    _p(b, u64p), _p(out, u64p), C.byref(h)))
    try:
        if graph:
            check(lib().spmvgpu_plan_capture(h))
        check(lib().spmvgpu_plan_run(h))
        ctx.sync()
        if stats is not None:
            ps = PlanStats()
            check(lib().spmvgpu_plan_stats_get(h, C.byref(ps)))
            stats.update({k: int(getattr(ps, k)) for k, _ in PlanStats._fields_})
    finally:
        lib().spmvgpu_plan_destroy(h)
    return out


@dataclass
class Csr:
    """CSR matrix (reference CsrMatrix, sparse.hpp).  Every entry point also
    accepts any object with these five attributes."""
    rows: int
    cols: int
    row_ptrs: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.row_ptrs[-1]) if self.rows else 0

    def dense(self) -> np.ndarray:
        d = np.zeros((self.rows, self.cols), np.int64)
        rows = np.repeat(np.arange(self.rows), np.diff(_i64(self.row_ptrs)))
        d[rows, _i64(self.col_indices)[: rows.size]] = _i64(self.values)[: rows.size]
        return d

    @staticmethod
    def from_dense(d) -> "Csr":
        d = np.asarray(d, dtype=np.int64)
        rows, cols = d.shape if d.ndim == 2 else (0, 0)
        rp, ci, va = [0], [], []
        for i in range(rows):
            for j in range(cols):
                if d[i, j]:
                    ci.append(j)
                    va.append(int(d[i, j]))
            rp.append(len(va))
        return Csr(rows, cols, _i64(rp), _i64(ci), _i64(va))


def _csr_c(m, keep: list) -> CsrC:
    """C view of a CSR matrix; the converted arrays are appended to `keep`,
    which the caller holds until the C call returns."""
    rp, ci, va = _i64(m.row_ptrs), _i64(m.col_indices), _i64(m.values)
    if va.size == 0:
        ci = va = np.zeros(1, np.int64)
    keep += [rp, ci, va]
    return CsrC(int(m.rows), int(m.cols), _p(rp, i64p), _p(ci, i64p), _p(va, i64p))


def _addr(a: np.ndarray) -> int:
    """Data address of a C-contiguous array (from_buffer is ~3x cheaper than
    __array_interface__; read-only arrays take the slow path)."""
    try:
        return C.addressof(C.c_char.from_buffer(a))
    except (TypeError, ValueError, BufferError):
        return a.__array_interface__["data"][0]


_ONE0 = np.zeros(1, np.int64)
_CSR_DT = np.dtype([("rows", "<u8"), ("cols", "<u8"), ("rp", "<u8"), ("ci", "<u8"), ("va", "<u8")])
_RES_DT = np.dtype([("led", "<u8", 6), ("n_ct", "<u8"), ("model", "<i4"), ("measured", "<i4"), ("nmsg", "<u8")])
assert _CSR_DT.itemsize == C.sizeof(CsrC) and _RES_DT.itemsize == C.sizeof(ResultC)
_LEDGER_KEYS = tuple(k for k, _ in Ledger._fields_)


# Marshalling cache: (matrix row, addresses) per CSR object, valid while the
# object still holds the very same arrays (identity-checked on every call;
# the cache entry keeps them alive, so their addresses cannot be reused).
# In-place edits of the arrays need no invalidation: the C side reads the
# contents at call time.
_CSR_CACHE: dict = {}  # id(matrix) -> (weakref, row_ptrs, col_indices, values, row, arrays)
_VEC_CACHE: dict = {}  # id(vector) -> (weakref, entry)


def _cache_put(cache: dict, obj, value) -> None:
    key = id(obj)
    try:
        ref = weakref.ref(obj, lambda _r, k=key: cache.pop(k, None))
    except TypeError:  # not weak-referenceable: no caching
        return
    cache[key] = (ref,) + value


def _csr_row(m):
    hit = _CSR_CACHE.get(id(m))
    if hit is not None and hit[0]() is m and hit[1] is m.row_ptrs and hit[2] is m.col_indices \
            and hit[3] is m.values and hit[4][0] == m.rows and hit[4][1] == m.cols:
        return hit[4], hit[5]
    rp, ci, va = _i64(m.row_ptrs), _i64(m.col_indices), _i64(m.values)
    if va.size == 0:
        ci = va = _ONE0
    row = (int(m.rows), int(m.cols), _addr(rp), _addr(ci), _addr(va))
    arrays = (rp, ci, va)
    if rp is m.row_ptrs and (va is _ONE0 or (ci is m.col_indices and va is m.values)):
        # only when no conversion copy was made (a copy would go stale on in-place edits)
        _cache_put(_CSR_CACHE, m, (m.row_ptrs, m.col_indices, m.values, row, arrays))
    return row, arrays


def _csr_table(ms, keep: list) -> np.ndarray:
    """cssc_csr[] for a batch as one numpy record array (addresses of int64
    copies kept alive in `keep`); a few us per matrix instead of ctypes objects."""
    rows = []
    for m in ms:
        row, arrays = _csr_row(m)
        keep.append(arrays)
        rows.append(row)
    t = np.array(rows, dtype=_CSR_DT) if rows else np.zeros(1, _CSR_DT)
    keep.append(t)
    return t


def _vec_entry(v):
    hit = _VEC_CACHE.get(id(v))
    if hit is not None and hit[0]() is v:
        return hit[1]
    a = _i64(v)
    ent = (a.size, _addr(a if a.size else _ONE0), a if a.size else _ONE0)
    if a is v:  # no conversion copy (a copy would go stale on in-place edits)
        _cache_put(_VEC_CACHE, v, (ent,))
    return ent


def _vectors(ms, vs, keep: list):
    """Addresses of int64 copies of the vectors and their lengths (the C-ABI
    raises DimensionMismatchError on a length != cols, reference protocol.cpp:77-81)."""
    ms, vs = list(ms), list(vs)
    if len(ms) != len(vs):
        raise SpmvError(-4, "DimensionMismatchError",
                        f"spmv_batch: {len(ms)} matrices but {len(vs)} vectors")
    ents = [_vec_entry(v) for v in vs]
    lens = np.array([e[0] for e in ents] or [0], dtype=np.uint64)
    ptrs = np.array([e[1] for e in ents] or [0], dtype=np.uint64)
    keep.append(ents)
    keep += (ptrs, lens)
    return _addr(ptrs), _addr(lens)


def _outputs(ms, keep: list):
    """One int64 buffer for every matrix's rows, the per-matrix address table
    and a cssc_result[] record array."""
    rows = [int(m.rows) for m in ms]
    off = np.zeros(len(rows) + 1, np.int64)
    off[1:] = np.cumsum([max(r, 1) for r in rows])
    buf = np.empty(int(off[-1]) or 1, np.int64)  # the library writes every row of every matrix
    ptrs = (off[:-1] * 8 + _addr(buf)).astype(np.uint64) if rows else np.zeros(1, np.uint64)
    res = np.zeros(max(len(rows), 1), _RES_DT)
    keep += (buf, ptrs, res)
    return buf, off, rows, _addr(ptrs), res


def _results(buf, off, rows, res) -> list:
    n = len(rows)
    led, nct = res["led"][:n].tolist(), res["n_ct"][:n].tolist()
    model, meas, offs = res["model"][:n].tolist(), res["measured"][:n].tolist(), off.tolist()
    return [{"values": buf[offs[i]: offs[i] + rows[i]], "n_ct": nct[i], "noise": model[i],
             "measured_noise": meas[i], "ledger": dict(zip(_LEDGER_KEYS, led[i]))} for i in range(n)]


def _result(r: ResultC, values: np.ndarray, msgs=None) -> dict:
    led = r.ledger
    out = {"values": values, "n_ct": int(r.n_ct), "noise": int(r.noise_model_bits),
           "measured_noise": int(r.noise_measured_bits),
           "ledger": {k: int(getattr(led, k)) for k, _ in Ledger._fields_}}
    if msgs is not None:
        out["messages"] = [(m.from_, m.to, m.kind, m.payload_bytes, m.ciphertext_count)
                           for m in msgs[: int(r.n_messages)]]
    return out


def spmv_partitioned(ctx: Context, m: Csr, v, chunk_size: int | None = None, key_holder: int = 0) -> dict:
    vv = _i64(v)
    chunk = ctx.slots if chunk_size is None else chunk_size
    vals = np.zeros(max(m.rows, 1), np.int64)
    res = ResultC()
    cap = 5 * (m.rows // max(chunk, 1) + 2)
    msgs = (Message * cap)()
    keep: list = []
    csr = _csr_c(m, keep)
    vp = vv if vv.size else np.zeros(1, np.int64)
    check(lib().cssc_spmv_partitioned(ctx.h, C.byref(csr), _p(vp, i64p), vv.size, chunk, key_holder,
                                      _p(vals, i64p), C.byref(res), msgs, cap))
    return _result(res, vals[: m.rows], msgs)


def spmv(ctx: Context, m: Csr, v, chunk_size: int | None = None, key_holder: int = 0) -> dict:
    """The reference's spmv (no row partitioning) on the GPU backend."""
    vv = _i64(v)
    chunk = ctx.slots if chunk_size is None else chunk_size
    vals = np.zeros(max(m.rows, 1), np.int64)
    res = ResultC()
    msgs = (Message * 8)()
    keep: list = []
    csr = _csr_c(m, keep)
    vp = vv if vv.size else np.zeros(1, np.int64)
    check(lib().cssc_spmv(ctx.h, C.byref(csr), _p(vp, i64p), vv.size, chunk, key_holder, _p(vals, i64p),
                          C.byref(res), msgs, 8))
    return _result(res, vals[: m.rows], msgs)


def diag_spmv(ctx: Context, m: Csr, v, key_holder: int = 0) -> dict:
    """The diagonal-method baseline (reference diagonal.cpp) batched on the GPU backend."""
    vv = _i64(v)
    vals = np.zeros(max(m.rows, 1), np.int64)
    res = ResultC()
    msgs = (Message * 8)()
    keep: list = []
    csr = _csr_c(m, keep)
    vp = vv if vv.size else np.zeros(1, np.int64)
    check(lib().cssc_diag_spmv(ctx.h, C.byref(csr), _p(vp, i64p), vv.size, key_holder, _p(vals, i64p),
                               C.byref(res), msgs, 8))
    return _result(res, vals[: m.rows], msgs)


def spmv_batch(ctx: Context, ms, vs, chunk_size: int | None = None, key_holder: int = 0) -> list:
    """Several independent spmv_partitioned runs in shared launches (each result
    equals its own run); party-separated unless the context's pipeline_fuse
    option says otherwise."""
    lib().cssc_speculate(ctx.h)  # the device starts on the previous plan's encryption while this marshals
    chunk = ctx.slots if chunk_size is None else chunk_size
    ms = list(ms)
    keep: list = []
    csrs = _csr_table(ms, keep)
    vptr, vlens = _vectors(ms, vs, keep)
    buf, off, rows, optr, res = _outputs(ms, keep)
    check(lib().cssc_spmv_batch(ctx.h, _addr(csrs), vptr, vlens, len(ms), chunk, key_holder, optr, _addr(res)))
    return _results(buf, off, rows, res)


class Job:
    """Staged evaluation: pack (host) -> encrypt (device) -> cloud (device, repeatable) -> finish."""

    def __init__(self, ctx: Context, ms, vs, chunk_size: int | None = None, rank: int = 0, world: int = 1):
        self.ctx, self.ms = ctx, list(ms)
        chunk = ctx.slots if chunk_size is None else chunk_size
        n = len(self.ms)
        self._keep: list = []  # the job borrows these arrays until it is destroyed
        csrs = _csr_table(self.ms, self._keep)
        vptr, vlens = _vectors(self.ms, vs, self._keep)
        h = C.c_void_p()
        check(lib().cssc_job_create_shard(ctx.h, _addr(csrs), vptr, vlens, n, chunk, rank, world, C.byref(h)))
        self.h = h

    def result_words(self) -> np.ndarray:
        """This shard's per-slice partial result ciphertexts, [results][ct words]."""
        cnt = C.c_uint64()
        check(lib().cssc_job_result_words(self.h, None, 0, C.byref(cnt)))
        w = np.zeros((cnt.value, self.ctx.ct_words), np.uint64)
        if cnt.value:
            check(lib().cssc_job_result_words(self.h, _p(w, u64p), w.size, C.byref(cnt)))
        return w

    def finish_words(self, words: np.ndarray) -> list:
        """Decrypt summed partial results (see result_words) and do the bookkeeping."""
        w = _u64(words)
        keep: list = []
        buf, off, rows, optr, res = _outputs(self.ms, keep)
        check(lib().cssc_job_finish_words(self.h, _p(w, u64p) if w.size else None, optr, _addr(res)))
        return _results(buf, off, rows, res)

    def result_words_dev(self, out=None):
        """This shard's partial result ciphertexts copied into a device tensor
        (torch.int64 [results * ct_words] on the context's GPU; allocated when
        `out` is None) -- the buffer an NCCL all-reduce sums across ranks."""
        import torch

        cnt = C.c_uint64()
        check(lib().cssc_job_result_words_dev(self.h, None, 0, C.byref(cnt)))
        if out is None:
            out = torch.empty(max(cnt.value, 1) * self.ctx.ct_words, dtype=torch.int64,
                              device=torch.device("cuda", self.ctx.params.device))
        if cnt.value:
            check(lib().cssc_job_result_words_dev(self.h, out.data_ptr(), out.numel(), C.byref(cnt)))
        return out

    def finish_words_dev(self, dev) -> list:
        """Fold the summed device words mod q (in place, on the GPU) and decrypt."""
        keep: list = []
        buf, off, rows, optr, res = _outputs(self.ms, keep)
        check(lib().cssc_job_finish_words_dev(self.h, dev.data_ptr(), optr, _addr(res)))
        return _results(buf, off, rows, res)

    def encrypt(self):
        check(lib().cssc_job_encrypt(self.h))

    def cloud(self, graph: bool = True):
        check(lib().cssc_job_cloud(self.h, int(graph)))

    def cloud_timed(self, start, stop, graph: bool = True):
        """cloud() bracketed by two torch.cuda.Event (timing) records issued in the same C call."""
        check(lib().cssc_job_cloud_timed(self.h, int(graph), C.c_void_p(start.cuda_event),
                                         C.c_void_p(stop.cuda_event)))

    def finish(self) -> list:
        keep: list = []
        buf, off, rows, optr, res = _outputs(self.ms, keep)
        check(lib().cssc_job_finish(self.h, optr, _addr(res)))
        return _results(buf, off, rows, res)

    def run(self) -> list:
        """encrypt + cloud + finish in one call (spmv_batch's path: one cached
        graph launch from the second job over the same chunk shapes)."""
        keep: list = []
        buf, off, rows, optr, res = _outputs(self.ms, keep)
        check(lib().cssc_job_run(self.h, optr, _addr(res)))
        return _results(buf, off, rows, res)

    def stats(self) -> dict:
        s = PlanStats()
        check(lib().cssc_job_plan_stats(self.h, C.byref(s)))
        return {k: int(getattr(s, k)) for k, _ in PlanStats._fields_}

    def profile(self) -> list:
        """Device time, compulsory bytes and limb NTTs per launch group (one graph replay)."""
        cap = 64
        ph = (PhaseC * cap)()
        cnt = C.c_int()
        check(lib().cssc_job_profile(self.h, ph, cap, C.byref(cnt)))
        return [{"name": p.name.decode(), "us": p.us, "items": int(p.items), "bytes": int(p.bytes),
                 "limb_ntts": int(p.limb_ntts), "sources": int(p.sources),
                 "acc_items": int(p.acc_items), "mac_terms": int(p.mac_terms)} for p in ph[: min(cnt.value, cap)]]

    def profile_kernels(self, reps: int = 5, flush_bytes: int = 256 << 20) -> list:
        """Mean device time of every kernel launch of the cloud phase over `reps`
        graph replays (L2 flushed before each), with its launch group index."""
        cap = 1024
        kt = (KernelTimingC * cap)()
        cnt = C.c_int()
        check(lib().cssc_job_profile_kernels(self.h, reps, flush_bytes, kt, cap, C.byref(cnt)))
        return [{"name": k.name.decode(), "group": int(k.group), "us": k.us} for k in kt[: min(cnt.value, cap)]]

    def io_bytes(self):
        a, b = C.c_uint64(), C.c_uint64()
        check(lib().cssc_job_input_bytes(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def close(self):
        if getattr(self, "h", None):
            lib().cssc_job_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def rotation_schedule(rows: int, cols: int):
    off = np.zeros(128, np.uint64)
    fa = np.zeros(128, np.int32)
    n = lib().cssc_rotation_schedule(rows, cols, _p(off, u64p), _p(fa, i32p))
    if n < 0:
        check(int(n))
    return [(int(off[i]), bool(fa[i])) for i in range(n)]


def pack_chunks(m: Csr, budget: int) -> dict:
    keep: list = []
    csr = _csr_c(m, keep)
    tot = C.c_uint64()
    n = lib().cssc_pack_chunks(C.byref(csr), budget, None, None, None, None, None, C.byref(tot))
    if n < 0:
        check(int(n))
    r = np.zeros(max(n, 1), np.int64)
    c = np.zeros(max(n, 1), np.int64)
    vf = np.zeros(max(tot.value, 1), np.int64)
    cf = np.zeros(max(tot.value, 1), np.int64)
    rm = np.zeros(max(m.rows, 1), np.int64)
    lib().cssc_pack_chunks(C.byref(csr), budget, _p(r, i64p), _p(c, i64p), _p(vf, i64p), _p(cf, i64p),
                           _p(rm, i64p), C.byref(tot))
    return {"n_ct": int(n), "r": r[:n], "c": c[:n], "vflat": vf[: tot.value], "cflat": cf[: tot.value],
            "row_map": rm[: m.rows]}


# ---- CSSC persistence (the reference's `spmv convert`) ----
def cssc_to_bytes(m) -> bytes:
    """csr_to_cssc + validate_cssc, then the compact binary CSSC form."""
    keep: list = []
    t = _csr_table([m], keep)
    n = C.c_uint64()
    check(lib().cssc_convert_binary(_addr(t), None, 0, C.byref(n)))
    buf = np.zeros(max(n.value, 1), np.uint8)
    check(lib().cssc_convert_binary(_addr(t), _addr(buf), buf.size, C.byref(n)))
    return buf[: n.value].tobytes()


def cssc_to_json(m) -> str:
    """The JSON text `spmv convert` writes for the same matrix (byte for byte)."""
    keep: list = []
    t = _csr_table([m], keep)
    n = C.c_uint64()
    check(lib().cssc_convert_json(_addr(t), None, 0, C.byref(n)))
    buf = np.zeros(max(n.value, 1), np.uint8)
    check(lib().cssc_convert_json(_addr(t), _addr(buf), buf.size, C.byref(n)))
    return buf[: n.value].tobytes().decode()


def cssc_from_bytes(data: bytes) -> dict:
    """The CSSC arrays {rows, cols, va, ci, rm, cp} of a binary buffer."""
    b = np.frombuffer(data, np.uint8).copy() if data else np.zeros(1, np.uint8)
    r, c, nz, L = (C.c_uint64() for _ in range(4))
    check(lib().cssc_load_binary(_addr(b), len(data), C.byref(r), C.byref(c), C.byref(nz), C.byref(L),
                                 None, None, None, None))
    va = np.zeros(max(nz.value, 1), np.int64)
    ci = np.zeros(max(nz.value, 1), np.uint64)
    rm = np.zeros(max(r.value, 1), np.uint64)
    cp = np.zeros(L.value + 1, np.uint64)
    check(lib().cssc_load_binary(_addr(b), len(data), C.byref(r), C.byref(c), C.byref(nz), C.byref(L),
                                 _addr(va), _addr(ci), _addr(rm), _addr(cp)))
    return {"rows": r.value, "cols": c.value, "va": va[: nz.value], "ci": ci[: nz.value].astype(np.int64),
            "rm": rm[: r.value].astype(np.int64), "cp": cp.astype(np.int64)}
