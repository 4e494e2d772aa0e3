"""Packed-planes variant: the host layout helper pack_planes must
produce exactly the reference's packed_sequence storage (packed_sequence.hpp:50-53),
checked against planes exported from the reference library itself; the GPU
parity of the packed entry points is in test_gpu_packed_planes.py."""
import numpy as np
import pytest

import paper_1809_07858_b200 as pf


def test_packed_words():
    for m, want in [(1, 3), (64, 3), (65, 6), (100, 6), (150, 9), (250, 12), (256, 12), (257, 15)]:
        assert pf.packed_words(m) == want


def test_pack_planes_known_answer():
    # A=00, C=01, G=10, T=11 (low = bit 0, high = bit 1), N only in the N plane
    out = pf.pack_planes(np.frombuffer(b"ACGTN", np.uint8)[None, :])
    assert out.shape == (1, 3, 1)
    low, high, nn = (int(v) for v in out[0, :, 0])
    assert low == 0b01010 and high == 0b01100 and nn == 0b10000


@pytest.mark.parametrize("m", [1, 5, 63, 64, 65, 100, 150, 250, 300])
def test_pack_planes_matches_reference_storage(reference, m):
    rng = np.random.default_rng(m)
    n = 500
    alpha = np.frombuffer(b"ACGTN", np.uint8)
    t = np.ascontiguousarray(alpha[rng.integers(0, 5, size=(n, m))])
    p = np.ascontiguousarray(alpha[rng.integers(0, 5, size=(n, m))])
    packed = reference.pack(t, p)
    try:
        rt, rp = packed.planes()
    finally:
        packed.free()
    assert (pf.pack_planes(t) == rt).all()
    assert (pf.pack_planes(p) == rp).all()
