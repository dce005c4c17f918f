"""Word-level parity on the five BASELINE configs at their full parameters
(N = 2^13 / 2^14 / 2^15, 58-bit primes): the batched cloud plan's result
ciphertexts equal, word for word, the CPU oracle's op-by-op evaluation of the
reference algorithm (protocol.cpp:121-140: multiply, rotation_schedule
rotate-and-add, mask_plaintext, inter_chunk_sum) on the same encryptions.

Chunks come from the host packing that mirrors the reference (pack_chunks:
csr_to_cssc + generate_chunks; B segments = reorg_vector), encrypted on both
sides with the same stream ids."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np
import pytest

import paper_2603_04742_b200 as pk
from oracle_bindings import BfvOracle

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402

pytestmark = pytest.mark.gpu


def slices_of(m, S):
    """partition_rows (chunk.cpp:55-73) with chunk_size = S."""
    out = []
    for r0 in range(0, m.rows, S):
        r1 = min(m.rows, r0 + S)
        b, e = int(m.row_ptrs[r0]), int(m.row_ptrs[r1])
        out.append(pk.Csr(r1 - r0, m.cols, (m.row_ptrs[r0:r1 + 1] - b).astype(np.int64),
                          m.col_indices[b:e].copy(), m.values[b:e].copy()))
    return out


@pytest.mark.parametrize("cfgno", [1, 2, 3, 4, 5])
def test_config_result_words_match_oracle(cfgno):
    cfg = bench.make_config(cfgno)
    ctx = pk.Context(logn=cfg["logn"], seed=7)
    orc = BfvOracle.like(ctx)
    S = ctx.slots
    r_list, c_list, slice_of, va, vb = [], [], [], [], []
    n_slices = 0
    for m, v in zip(cfg["ms"], cfg["vs"]):
        for part in slices_of(m, S):
            pc = pk.pack_chunks(part, S)
            off = 0
            for r, c in zip(pc["r"], pc["c"]):
                size = int(r * c)
                vf = pc["vflat"][off:off + size]
                cf = pc["cflat"][off:off + size]
                off += size
                r_list.append(int(r))
                c_list.append(int(c))
                slice_of.append(n_slices)
                va.append(vf)
                vb.append(np.where(cf >= 0, np.asarray(v)[np.maximum(cf, 0)], 0))
            if pc["n_ct"]:
                n_slices += 1
    n = len(r_list)
    sa = [10_000 + i for i in range(n)]
    sb = [20_000 + i for i in range(n)]
    ha, hb = ctx.encrypt(va, sa), ctx.encrypt(vb, sb)
    st = {}
    out = pk.cloud_plan(ctx, r_list, c_list, slice_of, n_slices, ha, hb, graph=True, stats=st)
    # Galois keys first (the only oracle state a rotation mutates), then the
    # independent per-chunk chains on all host cores (ctypes drops the GIL)
    scheds = [pk.rotation_schedule(r_list[i], c_list[i]) for i in range(n)]
    for g in sorted({orc.galois_elt(off) for sc in scheds for off, _ in sc}):
        if g != 1:
            orc.lib.bfvo_add_galois_key(orc.h, g)
            if st["relin_folded"]:
                orc.lib.bfvo_add_galois_key_sq(orc.h, g)

    def chain(i):
        z = orc.mul_tensor(orc.encrypt(va[i], sa[i]), orc.encrypt(vb[i], sb[i]))
        acc = orc.plan_fold_z(z, scheds[i], st["relin_folded"])
        return orc.mul_plain(acc, np.ones(r_list[i], np.int64))

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
        parts = list(ex.map(chain, range(n)))
    want = [None] * n_slices
    for i, part in enumerate(parts):
        s = slice_of[i]
        want[s] = part if want[s] is None else orc.add(want[s], part)
    for s in range(n_slices):
        assert np.array_equal(ctx.download(int(out[s])), want[s]), (cfgno, s)
    ctx.free(np.concatenate([ha, hb, out]))
    ctx.close()


@pytest.mark.parametrize("cfgno", [1, 2])
def test_cluster_key_switch_words_match_oracle(cfgno):
    """The opt-in thread-block-cluster key switch (ks_cluster.cu, CSSC_KS_CLUSTER=1)
    produces the same words; run in a child so the env switch is read fresh."""
    import subprocess
    env = dict(os.environ, CSSC_KS_CLUSTER="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        f"{__file__}::test_config_result_words_match_oracle[{cfgno}]"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
