"""ctypes bindings for the TEST-SIDE checkers under oracle/ (never the product).

  BfvOracle  -> oracle/build/liboracle.so  (bfv_oracle.c: CPU RNS-BFV, word level)
  SimOracle  -> oracle/build/liboracle.so  (sim_oracle.c: reference slot semantics)
  RefLib     -> oracle/_ref/libspmv_ref.so (the unmodified reference, compiled in place)
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
import os  # noqa: E402

# CSSC_ORACLE_SO: the sanitizer build of tools/asan_check.sh
ORACLE_SO = Path(os.environ.get("CSSC_ORACLE_SO") or ROOT / "oracle" / "build" / "liboracle.so")
REF_SO = ROOT / "oracle" / "_ref" / "libspmv_ref.so"

u64p = C.POINTER(C.c_uint64)
i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)
ip = C.POINTER(C.c_int)


def _p(a, t):
    return a.ctypes.data_as(t)


def _u64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _i64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


_olib = None


def oracle_lib():
    global _olib
    if _olib is None:
        L = C.CDLL(str(ORACLE_SO))
        L.bfvo_create.restype = C.c_void_p
        L.bfvo_create.argtypes = [C.c_int] * 6 + [C.c_uint64, C.c_uint64]
        L.bfvo_destroy.argtypes = [C.c_void_p]
        L.bfvo_primes.argtypes = [C.c_void_p, u64p]
        L.bfvo_psi.restype = C.c_uint64
        L.bfvo_psi.argtypes = [C.c_void_p, C.c_int]
        for f in ("bfvo_ntt", "bfvo_intt"):
            getattr(L, f).argtypes = [C.c_void_p, C.c_int, u64p]
        L.bfvo_chacha_word.restype = C.c_uint64
        L.bfvo_chacha_word.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64]
        L.bfvo_add_galois_key.argtypes = [C.c_void_p, C.c_uint32]
        L.bfvo_galois_elt.restype = C.c_uint32
        L.bfvo_mul_overq.restype = C.c_int
        L.bfvo_mul_overq.argtypes = [C.c_void_p]
        L.bfvo_galois_elt.argtypes = [C.c_void_p, C.c_int64]
        L.bfvo_get_sk.argtypes = [C.c_void_p, i64p]
        L.bfvo_get_pk.argtypes = [C.c_void_p, u64p]
        L.bfvo_get_ksk.argtypes = [C.c_void_p, C.c_uint32, u64p]
        L.bfvo_encode.argtypes = [C.c_void_p, i64p, C.c_size_t, u64p]
        L.bfvo_decode.argtypes = [C.c_void_p, u64p, u64p]
        L.bfvo_encrypt.argtypes = [C.c_void_p, u64p, C.c_uint64, u64p]
        L.bfvo_decrypt.argtypes = [C.c_void_p, u64p, u64p]
        for f in ("bfvo_add", "bfvo_mul_relin", "bfvo_mul_tensor", "bfvo_mul_plain"):
            getattr(L, f).argtypes = [C.c_void_p, u64p, u64p, u64p]
        L.bfvo_rotate.argtypes = [C.c_void_p, u64p, C.c_int64, u64p]
        L.bfvo_rotate2_add.restype = C.c_int
        L.bfvo_plan_fold.restype = C.c_int
        L.bfvo_plan_fold.argtypes = [C.c_void_p, u64p, C.c_int, i64p, ip, C.c_int, u64p]
        L.bfvo_get_ksk_sq.argtypes = [C.c_void_p, C.c_uint32, u64p]
        L.bfvo_add_galois_key_sq.argtypes = [C.c_void_p, C.c_uint32]
        L.bfvo_mul_relin_z.argtypes = [C.c_void_p, u64p, u64p]
        L.bfvo_rotate2_add.argtypes = [C.c_void_p, u64p, u64p, C.c_int64, C.c_int64, u64p]
        L.bfvo_key_switch.argtypes = [C.c_void_p, C.c_uint32, u64p, u64p, u64p]
        L.bfvo_automorph.argtypes = [C.c_void_p, C.c_uint32, u64p, u64p, C.c_int]
        # sim oracle
        L.simo_to_signed.restype = C.c_int64
        L.simo_to_signed.argtypes = [C.c_uint64, C.c_uint64]
        L.simo_to_residue.restype = C.c_uint64
        L.simo_to_residue.argtypes = [C.c_int64, C.c_uint64]
        L.simo_rotation_schedule.argtypes = [C.c_uint64, C.c_uint64, u64p, ip]
        L.simo_csr_to_cssc.restype = C.c_int64
        L.simo_csr_to_cssc.argtypes = [C.c_uint64, i64p, i64p, i64p, i64p, i64p, i64p, i64p]
        L.simo_generate_chunks.restype = C.c_int64
        L.simo_generate_chunks.argtypes = [C.c_int64, i64p, i64p, i64p, C.c_uint64, i64p, i64p, i64p, i64p, i64p]
        L.simo_spmv_partitioned.restype = C.c_int64
        L.simo_spmv_partitioned.argtypes = [C.c_uint64, C.c_uint64, C.c_double, ip, C.c_uint64, C.c_uint64,
                                            i64p, i64p, i64p, i64p, C.c_uint64, C.c_uint64, C.c_int, i64p,
                                            u64p, i64p, u64p, ip]
        L.simo_rotate.argtypes = [u64p, C.c_int64, C.c_uint64, u64p]
        _olib = L
    return _olib


class BfvOracle:
    """CPU RNS-BFV restatement; ciphertexts are uint64 [2][L][N] coefficient form."""

    def __init__(self, logn, L, K, alpha, qbits, pbits, t=65537, seed=1):
        self.lib = oracle_lib()
        self.h = self.lib.bfvo_create(logn, L, K, alpha, qbits, pbits, t, seed)
        self.n, self.L, self.K = 1 << logn, L, K
        self.dnum = (L + alpha - 1) // alpha
        buf = np.zeros(64, np.uint64)
        cnt = self.lib.bfvo_primes(self.h, _p(buf, u64p))
        self.primes = [int(x) for x in buf[:cnt]]

    @classmethod
    def like(cls, ctx):
        p = ctx.params
        return cls(p.logn, p.L, p.K, p.alpha, p.qbits, p.pbits, p.t, p.seed)

    def __del__(self):
        try:
            self.lib.bfvo_destroy(self.h)
        except Exception:
            pass

    def ntt(self, pi, a, inverse=False):
        a = _u64(a).copy()
        (self.lib.bfvo_intt if inverse else self.lib.bfvo_ntt)(self.h, pi, _p(a, u64p))
        return a

    def sk(self):
        s = np.zeros(self.n, np.int64)
        self.lib.bfvo_get_sk(self.h, _p(s, i64p))
        return s

    def pk(self):
        w = np.zeros(2 * self.L * self.n, np.uint64)
        self.lib.bfvo_get_pk(self.h, _p(w, u64p))
        return w

    def ksk(self, which):
        w = np.zeros(self.dnum * 2 * (self.L + self.K) * self.n, np.uint64)
        self.lib.bfvo_get_ksk(self.h, which, _p(w, u64p))
        return w

    def galois_elt(self, k):
        return int(self.lib.bfvo_galois_elt(self.h, k))

    def encode(self, vals):
        v = _i64(vals)
        m = np.zeros(self.n, np.uint64)
        assert self.lib.bfvo_encode(self.h, _p(v, i64p) if v.size else None, v.size, _p(m, u64p)) == 0
        return m

    def decode(self, m):
        s = np.zeros(self.n // 2, np.uint64)
        self.lib.bfvo_decode(self.h, _p(_u64(m), u64p), _p(s, u64p))
        return s

    def encrypt(self, vals, stream):
        ct = np.zeros(2 * self.L * self.n, np.uint64)
        m = self.encode(vals)
        self.lib.bfvo_encrypt(self.h, _p(m, u64p), stream, _p(ct, u64p))
        return ct

    def decrypt(self, ct):
        m = np.zeros(self.n, np.uint64)
        b = self.lib.bfvo_decrypt(self.h, _p(_u64(ct), u64p), _p(m, u64p))
        return self.decode(m), b

    def _bin(self, f, a, b, outlen=None):
        out = np.zeros(outlen or 2 * self.L * self.n, np.uint64)
        f(self.h, _p(_u64(a), u64p), _p(_u64(b), u64p), _p(out, u64p))
        return out

    def add(self, a, b):
        return self._bin(self.lib.bfvo_add, a, b)

    def mul_relin(self, a, b):
        return self._bin(self.lib.bfvo_mul_relin, a, b)

    def mul_plain(self, a, vals):
        return self._bin(self.lib.bfvo_mul_plain, a, self.encode(vals))

    def rotate(self, a, k):
        out = np.zeros(2 * self.L * self.n, np.uint64)
        self.lib.bfvo_rotate(self.h, _p(_u64(a), u64p), k, _p(out, u64p))
        return out

    def rotate2_add(self, acc, src, k1, k2):
        """acc + rot(acc, k1) + rot(src, k2) with one shared ModDown."""
        out = np.zeros(2 * self.L * self.n, np.uint64)
        r = self.lib.bfvo_rotate2_add(self.h, _p(_u64(acc), u64p), _p(_u64(src), u64p), k1, k2, _p(out, u64p))
        assert r == 0, r
        return out

    def mul_tensor(self, a, b):
        return self._bin(self.lib.bfvo_mul_tensor, a, b, 3 * self.L * self.n)

    def plan_fold_z(self, z, sched, fold_relin):
        """intra_chunk_sum from the product's tensor z as the batched plan evaluates
        it (bfvo_plan_fold); fold_relin: the relinearisation shares level 0's ModDown."""
        out = np.zeros(2 * self.L * self.n, np.uint64)
        offs = np.array([o for o, _ in sched] or [0], np.int64)
        fa = np.array([int(f) for _, f in sched] or [0], np.int32)
        r = self.lib.bfvo_plan_fold(self.h, _p(_u64(z), u64p), len(sched), _p(offs, i64p), _p(fa, ip),
                                    int(fold_relin), _p(out, u64p))  # 0 plain, 1 relin folded, 2 + merged stages
        assert r == 0, r
        return out

    def ksk_sq(self, g):
        w = np.zeros(self.dnum * 2 * (self.L + self.K) * self.n, np.uint64)
        self.lib.bfvo_get_ksk_sq(self.h, g, _p(w, u64p))
        return w

    def plan_fold(self, prod, sched):
        """intra_chunk_sum as the batched plan evaluates it (aggregate.cpp:36-50
        semantics): each doubling step and the odd step right after it share
        one ModDown (rotate2_add); a doubling step without one is rotate + add."""
        acc, i = prod, 0
        while i < len(sched):
            off, from_acc = sched[i]
            if from_acc and i + 1 < len(sched) and not sched[i + 1][1]:
                acc = self.rotate2_add(acc, prod, off, sched[i + 1][0])
                i += 2
            else:
                acc = self.add(acc, self.rotate(acc if from_acc else prod, off))
                i += 1
        return acc


def sim_spmv_partitioned(m, v, slot_count, chunk_size=None, t=65537, ct_mb=0.52,
                         noise=(146, 33, 26, 0, 0), key_holder=0, lib=None):
    """Reference slot semantics (sim_oracle.c) or, with lib=RefLib, the reference itself."""
    L = oracle_lib() if lib is None else lib
    chunk = slot_count if chunk_size is None else chunk_size
    rp, ci, va, vv = _i64(m.row_ptrs), _i64(m.col_indices), _i64(m.values), _i64(v)
    if va.size == 0:
        ci = va = np.zeros(1, np.int64)
    if vv.size == 0:
        vv_p = np.zeros(1, np.int64)
    else:
        vv_p = vv
    out = np.zeros(max(m.rows, 1), np.int64)
    led = np.zeros(6, np.uint64)
    cap = 5 * (m.rows // max(chunk, 1) + 2)
    msgs = np.zeros(5 * cap, np.int64)
    nm = C.c_uint64()
    nz = C.c_int()
    n5 = (C.c_int * 5)(*noise)
    fn = L.simo_spmv_partitioned if lib is None else L.ref_spmv_partitioned
    args = [slot_count, t, ct_mb, n5, m.rows, m.cols, _p(rp, i64p), _p(ci, i64p), _p(va, i64p),
            _p(vv_p, i64p), vv.size, chunk, key_holder, _p(out, i64p), _p(led, u64p), _p(msgs, i64p),
            C.byref(nm)]
    if lib is not None:
        args.append(cap)
    args.append(C.byref(nz))
    r = fn(*args)
    if r < 0:
        return {"error": int(r)}
    keys = ("n_mult_cc", "n_mult_cp", "n_rot", "n_add", "n_enc", "n_dec")
    return {"values": out[: m.rows], "n_ct": int(r), "noise": nz.value,
            "ledger": {k: int(x) for k, x in zip(keys, led)},
            "messages": [tuple(int(x) for x in msgs[5 * i: 5 * i + 5]) for i in range(nm.value)]}


_rlib = None


def ref_lib():
    """The reference library compiled in place (oracle/_ref); None when absent."""
    global _rlib
    if _rlib is None:
        if not REF_SO.exists():
            return None
        L = C.CDLL(str(REF_SO))
        L.ref_last_error.restype = C.c_char_p
        L.ref_spmv_partitioned.restype = C.c_int64
        L.ref_spmv_partitioned.argtypes = [C.c_uint64, C.c_uint64, C.c_double, ip, C.c_uint64, C.c_uint64,
                                           i64p, i64p, i64p, i64p, C.c_uint64, C.c_uint64, C.c_int, i64p,
                                           u64p, i64p, u64p, C.c_uint64, ip]
        L.ref_diag_spmv.restype = C.c_int64
        L.ref_diag_spmv.argtypes = [C.c_uint64, C.c_uint64, C.c_double, ip, C.c_uint64, C.c_uint64, i64p, i64p,
                                    i64p, i64p, C.c_uint64, C.c_int, i64p, u64p, i64p, u64p, C.c_uint64, ip]
        L.ref_time_spmv_partitioned.restype = C.c_double
        L.ref_time_spmv_partitioned.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, i64p, i64p,
                                                i64p, i64p, C.c_uint64, C.c_int]
        L.ref_random_sparse_csr.restype = C.c_int64
        L.ref_random_sparse_csr.argtypes = [C.c_uint64] * 4 + [C.c_int64] * 2 + [i64p] * 3
        L.ref_random_vector.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, i64p]
        L.ref_rotation_schedule.argtypes = [C.c_uint64, C.c_uint64, u64p, ip]
        L.ref_cloud_prepare.restype = C.c_void_p
        L.ref_cloud_prepare.argtypes = [C.c_uint64] * 4 + [i64p] * 4 + [C.c_uint64]
        L.ref_cloud_run.restype = C.c_double
        L.ref_cloud_run.argtypes = [C.c_void_p]
        L.ref_cloud_free.argtypes = [C.c_void_p]
        L.ref_chunks.restype = C.c_int64
        L.ref_chunks.argtypes = [C.c_uint64, C.c_uint64, i64p, i64p, i64p, C.c_uint64, i64p, i64p, i64p, i64p,
                                 i64p, u64p]
        _rlib = L
    return _rlib


def diag_reference(m, v, slot_count, t=65537, ct_mb=0.52, noise=(146, 33, 26, 0, 0), key_holder=0):
    """The reference's diag_spmv (oracle/_ref) or, when absent, a restatement of
    diagonal.cpp:44-104 on exact integers (values, ledger, transcript, model noise)."""
    L = ref_lib()
    if L is not None:
        rp, ci, va, vv = _i64(m.row_ptrs), _i64(m.col_indices), _i64(m.values), _i64(v)
        if va.size == 0:
            ci = va = np.zeros(1, np.int64)
        vv_p = vv if vv.size else np.zeros(1, np.int64)
        out = np.zeros(max(m.rows, 1), np.int64)
        led = np.zeros(6, np.uint64)
        msgs = np.zeros(5 * 8, np.int64)
        nm, nz = C.c_uint64(), C.c_int()
        r = L.ref_diag_spmv(slot_count, t, ct_mb, (C.c_int * 5)(*noise), m.rows, m.cols, _p(rp, i64p),
                            _p(ci, i64p), _p(va, i64p), _p(vv_p, i64p), vv.size, key_holder, _p(out, i64p),
                            _p(led, u64p), _p(msgs, i64p), C.byref(nm), 8, C.byref(nz))
        if r < 0:
            return {"error": int(r)}
        keys = ("n_mult_cc", "n_mult_cp", "n_rot", "n_add", "n_enc", "n_dec")
        return {"values": out[: m.rows], "n_ct": int(r), "noise": nz.value,
                "ledger": {k: int(x) for k, x in zip(keys, led)},
                "messages": [tuple(int(x) for x in msgs[5 * i: 5 * i + 5]) for i in range(nm.value)]}
    n = m.rows
    rows = np.repeat(np.arange(n), np.diff(m.row_ptrs))
    nd = len(set(((np.asarray(m.col_indices) + n - rows) % n).tolist())) if n else 0
    acc = np.zeros(n, np.int64)
    np.add.at(acc, rows, np.asarray(m.values) * np.asarray(v)[m.col_indices])
    r = np.mod(acc, t)
    vals = np.where(r > t // 2, r - t, r)
    price = lambda c: int(round(c * ct_mb * 1048576))  # noqa: E731
    msgs = [(0, 2, 0, price(nd), nd), (1, 2, 0, price(1), 1)]
    if nd:
        msgs.append((2, key_holder, 3, price(1), 1))
    prod = max(0, min(noise[0], max(0, noise[0] - noise[4])) - noise[1])
    noise_v = noise[0]
    for _ in range(nd):
        noise_v = max(0, min(noise_v, prod) - noise[3])
    return {"values": vals, "n_ct": nd, "noise": noise_v,
            "ledger": {"n_mult_cc": nd, "n_mult_cp": 0, "n_rot": nd, "n_add": nd, "n_enc": nd + 1,
                       "n_dec": 1 if nd else 0},
            "messages": msgs}
