"""Ciphertext wire format: serialize -> deserialize is the
identity on the words, the size is the bit-exact residue payload, and foreign
or malformed buffers are rejected."""
import numpy as np
import pytest

import paper_2603_04742_b200 as pk

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("logn", [10, 14])
def test_wire_roundtrip(logn):
    ctx = pk.Context(logn=logn, seed=3)
    vals = np.arange(-50, 50)
    (h,) = ctx.encrypt([vals], [7])
    data = ctx.serialize(h)
    bits = sum(int(q).bit_length() for q in ctx.primes[: ctx.L])
    assert len(data) == ctx.wire_size == 16 + (2 * ctx.n * bits + 7) // 8
    assert len(data) < ctx.ct_words * 8  # denser than the u64 arena
    h2 = ctx.deserialize(data)
    assert np.array_equal(ctx.download(h), ctx.download(h2))
    slots, _ = ctx.decrypt([h2])
    want = np.mod(np.concatenate([vals, np.zeros(ctx.slots - vals.size, np.int64)]), 65537)
    assert np.array_equal(slots[0].astype(np.int64), want)
    bad = bytearray(data)
    bad[0] ^= 1  # magic
    with pytest.raises(pk.SpmvError):
        ctx.deserialize(bytes(bad))
    with pytest.raises(pk.SpmvError):
        ctx.deserialize(data[:-1])
    bad = bytearray(data)
    for i in range(16, 16 + 8):  # first residue -> all ones (>= q0)
        bad[i] = 0xFF
    with pytest.raises(pk.SpmvError):
        ctx.deserialize(bytes(bad))
    other = pk.Context(logn=logn, seed=3, qbits=50)
    with pytest.raises(pk.SpmvError):  # different primes
        other.deserialize(data)
    ctx.free([h, h2])


def spec_encode(words, primes, logn, L):
    """The wire format restated from its spec (include/spmvgpu.h): 16-byte
    header ("CSW1", logn, L, 2 zero bytes, FNV-1a 64 of the L primes' bytes),
    then every residue of poly p, limb j, coefficient k in bitlen(q_j) bits,
    least significant bit first, in one little-endian bit stream."""
    n = 1 << logn
    fp = 1469598103934665603
    for q in primes[:L]:
        for b in range(8):
            fp ^= (int(q) >> (8 * b)) & 0xFF
            fp = (fp * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    head = b"CSW1" + bytes([logn, L, 0, 0]) + fp.to_bytes(8, "little")
    acc, nbits = 0, 0
    w = np.asarray(words, np.uint64).reshape(2, L, n)
    for p in range(2):
        for j in range(L):
            nb = int(primes[j]).bit_length()
            for v in w[p, j].tolist():
                acc |= v << nbits
                nbits += nb
    return head + acc.to_bytes((nbits + 7) // 8, "little")


def test_wire_bytes_equal_the_spec_encoding():
    """Not a self round trip: the library's bytes equal an independent
    encoder of the documented format, for a ciphertext of a real evaluation."""
    ctx = pk.Context(logn=10, seed=5)
    (a, b) = ctx.encrypt([np.arange(100) % 17 - 8, np.arange(100) % 13 - 6], [1, 2])
    (p,) = ctx.mul_relin([a], [b])
    data = ctx.serialize(int(p))
    assert data == spec_encode(ctx.download(int(p)), ctx.primes, 10, ctx.L)
    ctx.free([a, b, p])


def test_wire_transfers_between_party_contexts():
    """The transcript's ResultCiphertext (protocol.cpp:131-132) as real bytes:
    the cloud's context serializes a product, the key holder's own context
    (same key, separately created) deserializes and decrypts it."""
    vals_a, vals_b = np.arange(-40, 40), (np.arange(80) % 9) - 4
    cloud = pk.Context(logn=12, seed=21)
    (a, b) = cloud.encrypt([vals_a, vals_b], [3, 4])
    (p,) = cloud.mul_relin([a], [b])
    data = cloud.serialize(int(p))
    cloud.close()
    holder = pk.Context(logn=12, seed=21)
    h = holder.deserialize(data)
    slots, budget = holder.decrypt([h])
    want = np.mod(vals_a * vals_b, 65537)
    assert np.array_equal(slots[0][:80].astype(np.int64), want) and budget[0] > 0
    assert not slots[0][80:].any()
    holder.free([h])
    holder.close()
