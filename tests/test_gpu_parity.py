"""GPU parity: the sm_100a path against the CPU oracle, word for word (P5),
and decryptions against the reference simulator slot for slot (P1).

Keys and input ciphertexts come from the same seeds on both sides; every
output polynomial is compared in canonical coefficient form."""
import numpy as np
import pytest

import paper_2603_04742_b200 as pk
from oracle_bindings import BfvOracle

pytestmark = pytest.mark.gpu

# (logn, overrides): small rings for speed plus the real C1/C2 parameter sets
SETS = [
    (10, {}),
    (11, dict(L=4, K=2, alpha=2, qbits=58, pbits=58)),
    (12, dict(L=5, K=2, alpha=2, qbits=58, pbits=58)),
    (13, {}),
]


@pytest.fixture(scope="module", params=SETS, ids=lambda s: f"logn{s[0]}")
def pair(request):
    logn, ov = request.param
    ctx = pk.Context(logn=logn, seed=7, **ov)
    orc = BfvOracle.like(ctx)
    return ctx, orc


def rand_vals(n, seed, lo=-8, hi=8):
    rng = np.random.default_rng(seed)
    return rng.integers(lo, hi + 1, n)


def test_primes_match(pair):
    ctx, orc = pair
    assert ctx.primes == orc.primes


def test_ntt_matches_oracle(pair):
    ctx, orc = pair
    rng = np.random.default_rng(1)
    for pi in (0, len(ctx.primes) - 1, len(ctx.primes) - 2):
        q = ctx.primes[pi]
        a = np.array([int(x) for x in rng.integers(0, q, ctx.n, dtype=np.uint64)], np.uint64) % np.uint64(q)
        assert np.array_equal(ctx.ntt(pi, a), orc.ntt(pi, a))
        assert np.array_equal(ctx.ntt(pi, a, inverse=True), orc.ntt(pi, a, inverse=True))


def test_keys_match(pair):
    ctx, orc = pair
    assert np.array_equal(ctx.download_sk(), orc.sk())
    assert np.array_equal(ctx.download_pk(), orc.pk())
    assert np.array_equal(ctx.download_ksk(0), orc.ksk(0))
    g = ctx.galois_element(3)
    assert g == orc.galois_elt(3)
    assert np.array_equal(ctx.download_ksk(g), orc.ksk(g))


def test_encrypt_decrypt_match(pair):
    ctx, orc = pair
    S = ctx.slots
    vals = [rand_vals(S, 1), rand_vals(S // 3, 2), rand_vals(0, 3)]
    streams = [101, 102, 103]
    hs = ctx.encrypt(vals, streams)
    for h, v, s in zip(hs, vals, streams):
        assert np.array_equal(ctx.download(int(h)), orc.encrypt(v, s))
    slots, budgets = ctx.decrypt(hs)
    for row, v in zip(slots, vals):
        want = np.zeros(S, np.int64)
        want[: len(v)] = np.mod(v, 65537)
        assert np.array_equal(row.astype(np.int64), want)
    assert (budgets > 0).all()
    ctx.free(hs)


def test_mul_relin_rotate_mask_match(pair):
    ctx, orc = pair
    S = ctx.slots
    a, b = rand_vals(S, 11), rand_vals(S, 12)
    ha, hb = ctx.encrypt([a, b], [201, 202])
    ca, cb = orc.encrypt(a, 201), orc.encrypt(b, 202)
    hp = ctx.mul_relin([ha], [hb])
    cp = orc.mul_relin(ca, cb)
    assert np.array_equal(ctx.download(int(hp[0])), cp)
    prod = (a * b) % 65537
    for k in (1, 5, S - 1, -3):
        hr = ctx.rotate(hp, [k])
        cr = orc.rotate(cp, k)
        assert np.array_equal(ctx.download(int(hr[0])), cr), k
        sl, bud = ctx.decrypt(hr)
        assert np.array_equal(sl[0].astype(np.int64), np.roll(prod, -k))
        assert bud[0] > 0
        ctx.free(hr)
    # fused rotate-and-add
    hs = ctx.rotate_add(hp, hp, [7])
    cs = orc.add(cp, orc.rotate(cp, 7))
    assert np.array_equal(ctx.download(int(hs[0])), cs)
    # plaintext mask
    hm = ctx.mul_plain(hs, [np.ones(9, np.int64)])
    cm = orc.mul_plain(cs, np.ones(9, np.int64))
    assert np.array_equal(ctx.download(int(hm[0])), cm)
    sl, _ = ctx.decrypt(hm)
    want = (prod + np.roll(prod, -7)) % 65537
    want[9:] = 0
    assert np.array_equal(sl[0].astype(np.int64), want)
    ctx.free(np.concatenate([ha[None], hb[None], hp, hs, hm]))


def test_fused_and_unfused_key_switch_agree():
    """The fused 3-kernel key switch and the 7-launch pipeline give the same words."""
    ctx = pk.Context(logn=14, seed=5)
    S = ctx.slots
    a, b = rand_vals(S, 21), rand_vals(S, 22)
    ha, hb = ctx.encrypt([a, b], [1, 2])
    outs = {}
    for fused in (1, 0):
        ctx.set_option("fused_key_switch", fused)
        hp = ctx.mul_relin([ha], [hb])
        hr = ctx.rotate_add(hp, hp, [129])
        outs[fused] = (ctx.download(int(hp[0])), ctx.download(int(hr[0])))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("graph,shape", [(False, 0), (True, 0), (True, 1)])
def test_cloud_plan_words_match_oracle(graph, shape):
    """The whole batched cloud phase (mult+relin, hoisted rotate-and-add trees,
    masked per-slice accumulation) equals the oracle's op-by-op evaluation of
    the reference algorithm (protocol.cpp:121-140) word for word (P5); shape 1
    is a parameter set without a compile-time specialisation (L=5, K=2, 3 digits)."""
    ctx = pk.Context(logn=10, seed=9) if shape == 0 else pk.Context(logn=12, seed=9, L=5, K=2, alpha=2,
                                                                     qbits=58, pbits=58)
    orc = BfvOracle.like(ctx)
    S = ctx.slots
    shapes = [(7, 13), (3, 6), (5, 7), (11, 2), (1, 64), (40, 12), (2, 1), (8, 3)]
    slices = [0, 0, 1, 1, 1, 0, 2, 2]
    rng = np.random.default_rng(5)
    vals_a = [rng.integers(-8, 9, r * c) for r, c in shapes]
    vals_b = [rng.integers(-8, 9, r * c) for r, c in shapes]
    sa = [1000 + i for i in range(len(shapes))]
    sb = [2000 + i for i in range(len(shapes))]
    ha, hb = ctx.encrypt(vals_a, sa), ctx.encrypt(vals_b, sb)
    st = {}
    out = pk.cloud_plan(ctx, [r for r, _ in shapes], [c for _, c in shapes], slices, 3, ha, hb, graph=graph,
                        stats=st)
    assert st["relin_folded"] == (2 if shape == 0 else 0)  # fixed shape: folded level 0 + merged stages
    want = [None] * 3
    for i, (r, c) in enumerate(shapes):
        z = orc.mul_tensor(orc.encrypt(vals_a[i], sa[i]), orc.encrypt(vals_b[i], sb[i]))
        acc = orc.plan_fold_z(z, pk.rotation_schedule(r, c), st["relin_folded"])
        part = orc.mul_plain(acc, np.ones(r, np.int64))
        want[slices[i]] = part if want[slices[i]] is None else orc.add(want[slices[i]], part)
    for s in range(3):
        assert np.array_equal(ctx.download(int(out[s])), want[s]), s
    ctx.free(np.concatenate([ha, hb, out]))


def test_cloud_plan_fused_and_unfused_agree():
    """The fused plan (fused multiply, K1/K2 key switch, block-phase mask
    accumulation, small-launch tiles, folded level 0) and the launch-per-op
    pipeline (relinearise first) each equal the oracle's plan of their form
    word for word and decrypt to the same slots."""
    shapes = [(7, 13), (3, 6), (5, 7), (11, 2), (1, 64), (2, 1)]
    slices = [0, 0, 1, 1, 1, 0]
    rng = np.random.default_rng(9)
    va = [rng.integers(-8, 9, r * c) for r, c in shapes]
    vb = [rng.integers(-8, 9, r * c) for r, c in shapes]
    outs = {}
    for fused in (1, 0):
        ctx = pk.Context(logn=11, seed=4)
        orc = BfvOracle.like(ctx)
        ctx.set_option("fused_key_switch", fused)
        sa, sb = [300 + i for i in range(len(shapes))], [400 + i for i in range(len(shapes))]
        ha, hb = ctx.encrypt(va, sa), ctx.encrypt(vb, sb)
        st = {}
        out = pk.cloud_plan(ctx, [r for r, _ in shapes], [c for _, c in shapes], slices, 2, ha, hb, graph=True,
                            stats=st)
        assert st["relin_folded"] == 2 * fused
        got = [ctx.download(int(h)) for h in out]
        want = [None] * 2
        for i, (r, c) in enumerate(shapes):
            z = orc.mul_tensor(orc.encrypt(va[i], sa[i]), orc.encrypt(vb[i], sb[i]))
            part = orc.mul_plain(orc.plan_fold_z(z, pk.rotation_schedule(r, c), st["relin_folded"]),
                                 np.ones(r, np.int64))
            want[slices[i]] = part if want[slices[i]] is None else orc.add(want[slices[i]], part)
        assert all(np.array_equal(g, w) for g, w in zip(got, want))
        outs[fused] = [orc.decrypt(g)[0] for g in got]
        ctx.close()
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)


def test_folded_level0_matches_oracle_and_unfolded_values(monkeypatch):
    """Level 0 folded (products unrelinearised; hoisted ModUp + NTT of z1 and
    z2; relinearisation, rotations of z1 / z2 and the odd steps in one ModDown
    per doubling item) equals the oracle's folded plan word for word, and the
    unfolded plan (CSSC_NO_HOIST=1: relinearise, then per-rotation K1/K2)
    equals the oracle's unfolded plan; both decrypt to the same slots."""
    shapes = [(7, 13), (3, 6), (5, 7), (11, 2), (1, 64), (40, 12), (8, 3), (2, 1)]
    slices = [0, 0, 1, 1, 1, 0, 1, 0]
    rng = np.random.default_rng(17)
    va = [rng.integers(-8, 9, r * c) for r, c in shapes]
    vb = [rng.integers(-8, 9, r * c) for r, c in shapes]
    dec = {}
    for off in ("", "1"):
        if off:
            monkeypatch.setenv("CSSC_NO_HOIST", off)
        else:
            monkeypatch.delenv("CSSC_NO_HOIST", raising=False)
        ctx = pk.Context(logn=12, seed=8)
        orc = BfvOracle.like(ctx)
        sa, sb = [500 + i for i in range(len(shapes))], [600 + i for i in range(len(shapes))]
        ha, hb = ctx.encrypt(va, sa), ctx.encrypt(vb, sb)
        st = {}
        out = pk.cloud_plan(ctx, [r for r, _ in shapes], [c for _, c in shapes], slices, 2, ha, hb, graph=True,
                            stats=st)
        assert st["relin_folded"] == (0 if off else 2)
        want = [None] * 2
        for i, (r, c) in enumerate(shapes):
            z = orc.mul_tensor(orc.encrypt(va[i], sa[i]), orc.encrypt(vb[i], sb[i]))
            part = orc.mul_plain(orc.plan_fold_z(z, pk.rotation_schedule(r, c), st["relin_folded"]),
                                 np.ones(r, np.int64))
            want[slices[i]] = part if want[slices[i]] is None else orc.add(want[slices[i]], part)
        got = [ctx.download(int(h)) for h in out]
        for s_ in range(2):
            assert np.array_equal(got[s_], want[s_]), (off, s_)
        dec[off] = [orc.decrypt(g)[0] for g in got]
        ctx.close()
    assert all(np.array_equal(x, y) for x, y in zip(dec[""], dec["1"]))


@pytest.mark.parametrize("merge", [True, False])
def test_deep_trees_merged_stages_match_oracle(monkeypatch, merge):
    """Deep intra-chunk trees (up to 8 doubling steps, odd steps at every
    level): two doubling steps per key-switch stage after level 0 (default)
    and one per stage (CSSC_NO_MERGE=1) each equal the oracle's plan fold word
    for word."""
    if merge:
        monkeypatch.delenv("CSSC_NO_MERGE", raising=False)
    else:
        monkeypatch.setenv("CSSC_NO_MERGE", "1")
    ctx = pk.Context(logn=11, seed=21)
    orc = BfvOracle.like(ctx)
    shapes = [(1, 255), (1, 170), (2, 100), (3, 77), (1, 64), (4, 31), (1, 9), (5, 3)]
    slices = [0, 1, 0, 1, 2, 2, 0, 1]
    rng = np.random.default_rng(33)
    va = [rng.integers(-8, 9, r * c) for r, c in shapes]
    vb = [rng.integers(-8, 9, r * c) for r, c in shapes]
    sa, sb = [700 + i for i in range(len(shapes))], [800 + i for i in range(len(shapes))]
    ha, hb = ctx.encrypt(va, sa), ctx.encrypt(vb, sb)
    st = {}
    out = pk.cloud_plan(ctx, [r for r, _ in shapes], [c for _, c in shapes], slices, 3, ha, hb, graph=True,
                        stats=st)
    assert st["relin_folded"] == (2 if merge else 1)
    want = [None] * 3
    for i, (r, c) in enumerate(shapes):
        z = orc.mul_tensor(orc.encrypt(va[i], sa[i]), orc.encrypt(vb[i], sb[i]))
        part = orc.mul_plain(orc.plan_fold_z(z, pk.rotation_schedule(r, c), st["relin_folded"]),
                             np.ones(r, np.int64))
        want[slices[i]] = part if want[slices[i]] is None else orc.add(want[slices[i]], part)
    for s_ in range(3):
        assert np.array_equal(ctx.download(int(out[s_])), want[s_]), s_
    ctx.close()
