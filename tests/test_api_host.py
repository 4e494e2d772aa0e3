"""Host-side mirror of the reference containers and codec contract (no GPU)."""
import numpy as np
import pytest

import paper_1809_07858_b200 as pf


def test_packed_sequence_codec_contract():
    # proj/tests/test_packed_sequence.cpp:11-49
    s = pf.packed_sequence.from_string("ACGTNACGT")
    assert s.size() == 9 and s.to_string() == "ACGTNACGT"
    s = pf.packed_sequence.from_string("ACGT")
    assert [s.code(i) for i in range(4)] == [0, 1, 2, 3]
    s = pf.packed_sequence.from_string("ANGNT")
    assert [s.is_n(i) for i in range(5)] == [False, True, False, True, False]
    assert s.base_at(1) == "N" and s.base_at(4) == "T"
    with pytest.raises(pf.empty_sequence_error):
        pf.packed_sequence.from_string("")
    with pytest.raises(pf.illegal_character_error) as ei:
        pf.packed_sequence.from_string("ACGX")
    assert ei.value.position() == 3 and ei.value.byte() == "X"
    with pytest.raises(pf.illegal_character_error):
        pf.packed_sequence.from_string("acgt")
    assert isinstance(ei.value, pf.error)


def test_bitvector_semantics():
    # proj/tests/test_bitvector.cpp:26-56
    bv = pf.bitvector(70, True)
    assert bv.count_ones() == 70 and len(bv.words()) == 2
    assert int(bv.words()[1]) == (1 << 6) - 1
    w = np.array([0b10000, 0], np.uint64)
    b = pf.bitvector(12, words=w)
    assert b.to_string() == "000010000000" and b.count_zeros() == 11


def test_unpack_bitmap():
    a = np.array([0b101, 1 << 31], np.uint32)
    got = pf.unpack_bitmap(a, 64)
    assert got[0] and not got[1] and got[2] and got[63] and got.sum() == 3


def test_error_hierarchy_mirrors_reference():
    for cls in (pf.empty_sequence_error, pf.illegal_character_error, pf.length_mismatch_error,
                pf.threshold_too_large_error, pf.out_of_band_error, pf.parse_error,
                pf.invalid_parameters_error):
        assert issubclass(cls, pf.error)
    assert pf.parse_error(3, "x").line() == 3
