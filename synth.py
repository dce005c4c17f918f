"""Seeded synthetic inputs for the five BASELINE.json configs (numpy only).

Benchmark and test data, not product code: the product library
(`paper_2603_04742_b200/lib/libcssc_he.so`) carries no generator, and this
module imports nothing from the product or from `oracle/`, so the bench's
reference arm can build its inputs without loading our library.

* `random_sparse_csr` / `random_vector` reproduce the reference generators'
  draw streams exactly (`/root/reference/proj/src/synthetic.cpp:32-86`,
  `bounded_draw` at `include/spmv/synthetic.hpp:15`, entries ordered as
  `coo_to_csr` does, `src/sparse.cpp:11-53`), so C1, C2 and C5 are
  bit-identical to the reference's matrices.  `tests/test_synth.py` pins them
  against the compiled reference (`oracle/_ref`).
* `random_nonzero_vector`: the same stream with 0 rejected (BASELINE.json's
  "[-8,8] excluding 0"; the reference's `random_vector` includes 0, SURVEY
  Appendix C.8).
* `power_law_csr` (C3) and `stencil27_csr` (C4) are the builder-defined
  generators of SURVEY.md 8(d).

The PRNG is std::mt19937_64 (its published recurrence and tempering), run
block-wise in numpy; only integer PRNG bits are used (no std:: distributions,
reference synthetic.hpp:13-15).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np



class MT19937_64:
    """std::mt19937_64 output stream with look-ahead (`peek`) and `advance`."""

    N, M = 312, 156
    _A = np.uint64(0xB5026F5AA96619E9)
    _UPPER = np.uint64(0xFFFFFFFF80000000)
    _LOWER = np.uint64(0x7FFFFFFF)

    def __init__(self, seed: int):
        mt = [seed & 0xFFFFFFFFFFFFFFFF]
        for i in range(1, self.N):
            p = mt[-1]
            mt.append((6364136223846793005 * (p ^ (p >> 62)) + i) & 0xFFFFFFFFFFFFFFFF)
        self._mt = np.array(mt, dtype=np.uint64)
        self._buf = np.zeros(0, np.uint64)
        self._pos = 0

    def _twist(self) -> np.ndarray:
        mt, n, m = self._mt, self.N, self.M

        def mix(cur, nxt, far):
            x = (cur & self._UPPER) | (nxt & self._LOWER)
            xa = x >> np.uint64(1)
            xa ^= np.where((x & np.uint64(1)) != 0, self._A, np.uint64(0))
            return far ^ xa

        mt[: n - m] = mix(mt[: n - m], mt[1: n - m + 1], mt[m:])
        mt[n - m: n - 1] = mix(mt[n - m: n - 1], mt[n - m + 1:], mt[: m - 1])
        mt[n - 1: n] = mix(mt[n - 1: n], mt[0:1], mt[m - 1: m])
        y = mt.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        return y

    def peek(self, k: int) -> np.ndarray:
        need = self._pos + k - self._buf.size
        if need > 0:
            blocks = [self._buf[self._pos:]]
            got = 0
            while got < need:
                blocks.append(self._twist())
                got += self.N
            self._buf = np.concatenate(blocks)
            self._pos = 0
        return self._buf[self._pos: self._pos + k]

    def advance(self, k: int) -> None:
        self._pos += k

    def take(self, k: int) -> np.ndarray:
        out = self.peek(k).copy()
        self.advance(k)
        return out


@dataclass
class Csr:
    """CSR matrix (the reference's CsrMatrix fields, sparse.hpp)."""
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
        rows = np.repeat(np.arange(self.rows), np.diff(self.row_ptrs))
        d[rows, self.col_indices] = self.values
        return d


def _nonzero_draws(rng: MT19937_64, count: int, lo: int, hi: int) -> np.ndarray:
    """`count` values of the reference's draw_value loop: lo + raw % span, 0
    rejected (synthetic.cpp:14-29)."""
    if count == 0:
        return np.zeros(0, np.int64)
    if lo > hi:
        raise ValueError("draw_value: empty range")
    if lo == 0 and hi == 0:
        raise ValueError("draw_value: range holds only zero")
    span = hi - lo + 1
    out = []
    left = count
    while left:
        k = left + left // max(span - 1, 1) + 64
        raw = rng.peek(k)
        v = (raw % np.uint64(span)).astype(np.int64) + lo
        nz = np.flatnonzero(v != 0)
        if nz.size >= left:
            out.append(v[nz[:left]])
            rng.advance(int(nz[left - 1]) + 1)
            left = 0
        else:
            out.append(v[nz])
            rng.advance(k)
            left -= nz.size
    return np.concatenate(out)


def random_sparse_csr(rows: int, cols: int, nnz: int, seed: int, lo: int = -100, hi: int = 100) -> Csr:
    """Reference random_sparse_csr (synthetic.cpp:32-72): uniform cells without
    replacement, nonzero values, entries sorted by (row, col)."""
    cells = rows * cols
    if nnz > cells:
        raise ValueError("random_sparse_csr: nnz exceeds rows * cols")
    rng = MT19937_64(seed)
    if 2 * nnz >= cells:  # partial Fisher-Yates
        pool = np.arange(cells, dtype=np.uint64)
        raw = rng.take(nnz)
        picks = np.zeros(nnz, np.uint64)
        for i in range(nnz):
            j = i + int(raw[i] % np.uint64(cells - i))
            pool[i], pool[j] = pool[j], pool[i]
            picks[i] = pool[i]
    else:  # rejection of repeated cells, in draw order
        taken = np.zeros(0, np.uint64)
        chunks = []
        while taken.size < nnz:
            need = nnz - taken.size
            k = need + need // 8 + 64
            c = rng.peek(k) % np.uint64(cells)
            _, first = np.unique(c, return_index=True)
            first.sort()
            first = first[~np.isin(c[first], taken)]
            if first.size >= need:
                first = first[:need]
                rng.advance(int(first[-1]) + 1)
            else:
                rng.advance(k)
            chunks.append(c[first])
            taken = np.concatenate([taken, c[first]])
        picks = np.concatenate(chunks) if chunks else np.zeros(0, np.uint64)
    vals = _nonzero_draws(rng, nnz, lo, hi)
    order = np.argsort(picks, kind="stable")
    picks, vals = picks[order], vals[order]
    r = (picks // np.uint64(max(cols, 1))).astype(np.int64)
    ci = (picks % np.uint64(max(cols, 1))).astype(np.int64)
    rp = np.zeros(rows + 1, np.int64)
    np.add.at(rp, r + 1, 1)
    return Csr(rows, cols, np.cumsum(rp), ci, vals.astype(np.int64))


def random_vector(n: int, seed: int, lo: int = -100, hi: int = 100, nonzero: bool = False) -> np.ndarray:
    """Reference random_vector (synthetic.cpp:74-86); nonzero=True rejects 0."""
    if lo > hi:
        raise ValueError("random_vector: empty range")
    rng = MT19937_64(seed ^ 0x9E3779B97F4A7C15)
    if nonzero:
        return _nonzero_draws(rng, n, lo, hi)
    raw = rng.take(n)
    return (raw % np.uint64(hi - lo + 1)).astype(np.int64) + lo


def _unit(raw: np.ndarray) -> np.ndarray:
    return (raw >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def power_law_csr(n: int, mean_degree: float = 12.0, exponent: float = 2.0, seed: int = 3,
                  lo: int = -8, hi: int = 8) -> Csr:
    """C3: row degrees Zipf(exponent) on {1..n} by inverse CDF,
    rescaled to the mean and clamped to [1, n]; columns floor(n u^3) without
    replacement within a row (hub-biased), sorted; then the row's values."""
    if n == 0:
        return Csr(0, 0, np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0, np.int64))
    rng = MT19937_64(seed)
    k = np.arange(1, n + 1, dtype=np.float64)
    cdf = np.cumsum(np.power(k, -exponent))
    cdf = cdf / cdf[-1]
    raw = (np.searchsorted(cdf, _unit(rng.take(n)), side="left") + 1).astype(np.float64)
    total = float(np.add.reduce(raw))  # exact: integers below 2^53
    scale = mean_degree * float(n) / total
    x = raw * scale
    fl = np.floor(x)
    want = np.where(x - fl >= 0.5, fl + 1.0, fl)  # llround for x >= 0
    want = np.clip(want, 1.0, float(n)).astype(np.int64)
    rp = np.zeros(n + 1, np.int64)
    cis, vas = [], []
    fn = float(n)
    for i in range(n):
        w = int(want[i])
        row = np.zeros(0, np.int64)
        while row.size < w:
            need = w - row.size
            kk = 2 * need + 16
            u = _unit(rng.peek(kk))
            c = np.minimum(n - 1, (fn * u * u * u).astype(np.int64))
            _, first = np.unique(c, return_index=True)
            first.sort()
            first = first[~np.isin(c[first], row)]
            if first.size >= need:
                first = first[:need]
                rng.advance(int(first[-1]) + 1)
            else:
                rng.advance(kk)
            row = np.concatenate([row, c[first]])
        row.sort()
        cis.append(row)
        vas.append(_nonzero_draws(rng, w, lo, hi))
        rp[i + 1] = rp[i] + w
    return Csr(n, n, rp, np.concatenate(cis), np.concatenate(vas))


def stencil27_csr(side: int = 32, seed: int = 4, lo: int = -8, hi: int = 8) -> Csr:
    """C4: lexicographic side^3 grid, every row links to its
    in-grid neighbours with max(|dx|,|dy|,|dz|) <= 1 (self included), columns
    ascending, values drawn in row-major entry order."""
    rng = MT19937_64(seed)
    n = side ** 3
    g = np.arange(side)
    x, y, z = (a.reshape(-1) for a in np.meshgrid(g, g, g, indexing="ij"))
    cols = []
    for dx in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dz in (-1, 0, 1):
                nx, ny, nz = x + dx, y + dy, z + dz
                ok = (nx >= 0) & (nx < side) & (ny >= 0) & (ny < side) & (nz >= 0) & (nz < side)
                cols.append(np.where(ok, (nx * side + ny) * side + nz, -1))
    cm = np.stack(cols, axis=1)  # [row][27], -1 outside the grid; ascending per row
    keep = cm >= 0
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum(keep.sum(axis=1))
    ci = cm[keep].astype(np.int64)
    return Csr(n, n, rp, ci, _nonzero_draws(rng, ci.size, lo, hi))


def config(cfg: int) -> dict:
    """Inputs of BASELINE.json config `cfg` (1..5), SURVEY 8(d) seeds."""
    if cfg == 1:
        return dict(name="C1 256x256 uniform 1% (655 nnz)", logn=13,
                    ms=[random_sparse_csr(256, 256, 655, 1, -8, 8)], vs=[random_vector(256, 1, -8, 8, True)])
    if cfg == 2:
        return dict(name="C2 4096x4096 uniform 0.1% (16777 nnz)", logn=14,
                    ms=[random_sparse_csr(4096, 4096, 16777, 2, -8, 8)], vs=[random_vector(4096, 2, -8, 8, True)])
    if cfg == 3:
        return dict(name="C3 16384x16384 power-law Zipf(2) mean 12", logn=14,
                    ms=[power_law_csr(16384, 12.0, 2.0, 3, -8, 8)], vs=[random_vector(16384, 3, -8, 8, True)])
    if cfg == 4:
        return dict(name="C4 32^3 grid 27-point stencil (830584 nnz)", logn=15,
                    ms=[stencil27_csr(32, 4, -8, 8)], vs=[random_vector(32768, 4, -8, 8, True)])
    if cfg == 5:
        return dict(name="C5 64 x 2048x2048 uniform 0.5% (20972 nnz each)", logn=14,
                    ms=[random_sparse_csr(2048, 2048, 20972, 500 + k, -8, 8) for k in range(64)],
                    vs=[random_vector(2048, 500 + k, -8, 8, True) for k in range(64)])
    raise ValueError(cfg)
