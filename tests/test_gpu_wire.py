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
