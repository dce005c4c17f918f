"""Known-answer tests that pin the CPU RNS-BFV oracle (oracle/bfv_oracle.c)
before it is trusted as the word-level checker of the GPU path."""
import ctypes as C

import numpy as np
import pytest

from oracle_bindings import BfvOracle, oracle_lib, sim_spmv_partitioned, _u64, _i64
import paper_2603_04742_b200 as pk
import synth

T = 65537


@pytest.fixture(scope="module", params=[(5, 3, 1, 1, 54), (6, 4, 2, 2, 58), (4, 8, 4, 4, 58), (6, 2, 2, 2, 58),
                                        (5, 4, 4, 4, 58)],
                ids=["n32_L3", "n64_L4", "n16_L8", "n64_L2_overq", "n32_L4_overq"])
def orc(request):
    logn, L, K, a, qb = request.param
    return BfvOracle(logn, L, K, a, qb, qb, T, 1234)


def bitrev(x, b):
    return int(format(x, f"0{b}b")[::-1], 2)


def test_chacha20_rfc8439_vector():
    """RFC 8439 section 2.3.2 block-function test vector."""
    L = oracle_lib()
    L.bfvo_chacha_block_raw.argtypes = [C.POINTER(C.c_uint32), C.c_uint32, C.POINTER(C.c_uint32),
                                        C.POINTER(C.c_uint32)]
    key = (C.c_uint32 * 8)(*[int.from_bytes(bytes(range(4 * i, 4 * i + 4)), "little") for i in range(8)])
    nonce = (C.c_uint32 * 3)(0x09000000, 0x4A000000, 0x00000000)
    out = (C.c_uint32 * 16)()
    L.bfvo_chacha_block_raw(key, 1, nonce, out)
    got = b"".join(int(w).to_bytes(4, "little") for w in out).hex()
    want = ("10f1e7e4d13b5915500fdd1fa32071c4c7d1f4c733c068030422aa9ac3d46c4e"
            "d2826446079faa0914c2d705d98b02a2b5129cd1de164eb9cbd083e8a2503c4e")
    assert got == want


def test_primes_are_ntt_friendly(orc):
    n = orc.n
    for q in orc.primes[:-1]:
        assert (q - 1) % (2 * n) == 0 and pow(3, q - 1, q) == 1
    assert len(set(orc.primes)) == len(orc.primes)


def test_ntt_is_evaluation_at_odd_powers(orc):
    rng = np.random.default_rng(0)
    n, lg = orc.n, orc.n.bit_length() - 1
    for pi in (0, len(orc.primes) - 1):
        q = orc.primes[pi]
        psi = int(orc.lib.bfvo_psi(orc.h, pi))
        assert pow(psi, n, q) == q - 1
        a = [int(x) % q for x in rng.integers(0, 2**62, n, dtype=np.uint64)]
        A = orc.ntt(pi, a)
        for p in range(n):
            e = 2 * bitrev(p, lg) + 1
            assert sum(a[j] * pow(psi, e * j, q) for j in range(n)) % q == int(A[p])
        assert [int(x) for x in orc.ntt(pi, A, inverse=True)] == a


def test_ntt_convolution_is_negacyclic(orc):
    rng = np.random.default_rng(1)
    n, q = orc.n, orc.primes[0]
    a = [int(x) % q for x in rng.integers(0, 2**62, n, dtype=np.uint64)]
    b = [int(x) % q for x in rng.integers(0, 2**62, n, dtype=np.uint64)]
    c = orc.ntt(0, np.array([int(x) * int(y) % q for x, y in zip(orc.ntt(0, a), orc.ntt(0, b))], np.uint64),
                inverse=True)
    ref = [0] * n
    for i in range(n):
        for j in range(n):
            k, s = (i + j) % n, -1 if i + j >= n else 1
            ref[k] = (ref[k] + s * a[i] * b[j]) % q
    assert [int(x) for x in c] == ref


def test_encode_encrypt_decrypt_roundtrip(orc):
    rng = np.random.default_rng(2)
    S = orc.n // 2
    for trial in range(3):
        v = rng.integers(-8, 9, S)
        assert np.array_equal(orc.decode(orc.encode(v)).astype(np.int64), np.mod(v, T))
        slots, budget = orc.decrypt(orc.encrypt(v, 100 + trial))
        assert np.array_equal(slots.astype(np.int64), np.mod(v, T)) and budget > 0


def test_homomorphic_ops_match_slot_semantics(orc):
    rng = np.random.default_rng(3)
    S = orc.n // 2
    a, b = rng.integers(-8, 9, S), rng.integers(-8, 9, S)
    ca, cb = orc.encrypt(a, 1), orc.encrypt(b, 2)
    prod = np.mod(a * b, T)
    assert np.array_equal(orc.decrypt(orc.add(ca, cb))[0].astype(np.int64), np.mod(a + b, T))
    cp = orc.mul_relin(ca, cb)
    assert np.array_equal(orc.decrypt(cp)[0].astype(np.int64), prod)
    for k in (1, -1, 3, S - 1, 0, S + 2):
        assert np.array_equal(orc.decrypt(orc.rotate(cp, k))[0].astype(np.int64), np.roll(prod, -k))
    m = orc.decrypt(orc.mul_plain(cp, np.ones(3, np.int64)))[0].astype(np.int64)
    want = prod.copy()
    want[3:] = 0
    assert np.array_equal(m, want)


def test_bfv_protocol_decrypts_to_reference():
    """A whole encrypted SpMV run op by op on the BFV oracle (ring 2^7, S=64)
    decrypts to the reference simulator's values (P1 for the oracle itself)."""
    orc = BfvOracle(7, 3, 1, 1, 54, 54, T, 5)
    S = 64
    for seed in (11, 12):
        m = synth.random_sparse_csr(20, 24, 90, seed, -8, 8)
        v = synth.random_vector(24, seed, -8, 8)
        want = sim_spmv_partitioned(m, v, S, S)
        pc = pk.pack_chunks(m, S)
        res = None
        off = 0
        for i in range(pc["n_ct"]):
            r, c = int(pc["r"][i]), int(pc["c"][i])
            vf = pc["vflat"][off: off + r * c]
            cf = pc["cflat"][off: off + r * c]
            off += r * c
            seg = np.where(cf >= 0, v[np.maximum(cf, 0)], 0)
            prod = orc.mul_relin(orc.encrypt(vf, 2 * i + 1), orc.encrypt(seg, 2 * i + 2))
            acc = prod
            for o, from_acc in pk.rotation_schedule(r, c):
                acc = orc.add(acc, orc.rotate(acc if from_acc else prod, o))
            part = orc.mul_plain(acc, np.ones(r, np.int64))
            res = part if res is None else orc.add(res, part)
        slots, budget = orc.decrypt(res)
        assert budget > 0
        vals = np.zeros(m.rows, np.int64)
        for p in range(m.rows):
            s = int(slots[p])
            vals[int(pc["row_map"][p])] = s - T if s > T // 2 else s
        assert np.array_equal(vals, want["values"])


def test_multiply_method_follows_the_shape():
    """The shapes with specialised GPU kernels multiply over Q u R (E6-E8),
    every other shape over Q u B (HPS)."""
    lib = oracle_lib()
    for (L, K, a), want in (((2, 2, 2), 1), ((4, 4, 4), 1), ((3, 1, 1), 0), ((4, 2, 2), 0), ((2, 2, 1), 0)):
        o = BfvOracle(5, L, K, a, 58, 58, T, 7)
        assert lib.bfvo_mul_overq(o.h) == want


@pytest.mark.parametrize("logn,L", [(13, 2), (14, 2), (15, 4)])
def test_overq_multiply_noise_at_full_size(logn, L):
    """At the default parameters the over-Q product decrypts exactly with a
    wide noise margin (a rotation and a mask still to come)."""
    orc = BfvOracle(logn, L, L, L, 58, 58, T, 99)
    rng = np.random.default_rng(logn)
    S = orc.n // 2
    a, b = rng.integers(-8, 9, S), rng.integers(-8, 9, S)
    cp = orc.mul_relin(orc.encrypt(a, 1), orc.encrypt(b, 2))
    vals, budget = orc.decrypt(cp)
    assert np.array_equal(vals.astype(np.int64), np.mod(a * b, T))
    assert budget >= 40


def test_rotate2_add_decrypts_like_two_rotations(orc):
    """acc + rot(acc, k1) + rot(src, k2) with one shared ModDown (the batched
    plan's fused doubling + odd step) decrypts to the same slots as the two
    separate rotate-and-adds of aggregate.cpp:36-50."""
    rng = np.random.default_rng(11)
    S = orc.n // 2
    a, b = rng.integers(-8, 9, S), rng.integers(-8, 9, S)
    ca, cb = orc.encrypt(a, 5), orc.encrypt(b, 6)
    for k1, k2 in ((1, 2), (3, S - 1), (2, 5)):
        for g in (orc.galois_elt(k1), orc.galois_elt(k2)):
            orc.lib.bfvo_add_galois_key(orc.h, g)
        fused = orc.rotate2_add(ca, cb, k1, k2)
        sep = orc.add(orc.add(ca, orc.rotate(ca, k1)), orc.rotate(cb, k2))
        want = np.mod(a + np.roll(a, -k1) + np.roll(b, -k2), T)
        assert np.array_equal(orc.decrypt(fused)[0].astype(np.int64), want)
        assert np.array_equal(orc.decrypt(sep)[0].astype(np.int64), want)


@pytest.mark.parametrize("r,c", [(1, 7), (3, 5), (2, 13), (4, 2), (1, 1), (1, 15), (1, 27), (1, 16)])
def test_plan_fold_both_forms_decrypt_to_the_intra_chunk_sum(orc, r, c):
    """bfvo_plan_fold from the product's tensor: unfolded (relin first) equals the
    rotate2_add fold of relin(z) word for word; folded (relinearisation inside
    level 0's ModDown, keys for phi_g(s)^2) decrypts to the same slots."""
    S = orc.n // 2
    if r * c > S:
        pytest.skip("chunk exceeds the ring")
    rng = np.random.default_rng(r * 100 + c)
    a, b = rng.integers(-8, 9, S), rng.integers(-8, 9, S)
    z = orc.mul_tensor(orc.encrypt(a, 3), orc.encrypt(b, 4))
    sched = pk.rotation_schedule(r, c)
    p = orc.lib  # noqa: F841
    relin = np.zeros(2 * orc.L * orc.n, np.uint64)
    orc.lib.bfvo_mul_relin_z(orc.h, _u64(z).ctypes.data_as(C.POINTER(C.c_uint64)),
                             relin.ctypes.data_as(C.POINTER(C.c_uint64)))
    unf = orc.plan_fold_z(z, sched, False)
    assert np.array_equal(unf, orc.plan_fold(relin, sched))
    fol = orc.plan_fold_z(z, sched, 1)
    mrg = orc.plan_fold_z(z, sched, 2)  # two doubling steps per key-switch stage after level 0
    prod = np.mod(a * b, T)
    want = np.zeros(S, np.int64)
    for k in range(c):  # blocks of r slots summed: slot i gets sum_k prod[i + k r]
        want += np.roll(prod, -k * r)
    want = np.mod(want, T)
    assert np.array_equal(orc.decrypt(unf)[0].astype(np.int64), want)
    assert np.array_equal(orc.decrypt(fol)[0].astype(np.int64), want)
    assert np.array_equal(orc.decrypt(mrg)[0].astype(np.int64), want)
