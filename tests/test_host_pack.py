"""Host packing stage (csrc/host_pack.cpp): ASCII records -> nibble records
(pack.cuh nibble format), both the AVX-512 and the portable path, checked
against a numpy restatement of the format and the reference's validation order
(packed_sequence::from_string, proj/src/packed_sequence.cpp:19-29)."""
import ctypes as C

import numpy as np
import pytest

from paper_1809_07858_b200 import _lib as L


def ref_nibbles(arr):
    """byte q of word w = low nibble of column 8w+q | low nibble of column 8w+q+4 << 4."""
    n, m = arr.shape
    words = (m + 7) // 8
    pad = np.zeros((n, words * 8), np.uint8)
    pad[:, :m] = arr
    blk = pad.reshape(n, words, 8) & 0x0F
    out = blk[:, :, :4] | (blk[:, :, 4:] << 4)
    return out.reshape(n, words * 4)


def host_pack(t, p, simd, stride=None):
    n, m = t.shape[0], t.shape[1] if stride is None else stride
    m = t.shape[1] if stride is None else stride
    np_ = L.lib.pf_nibble_pitch(m)
    ot = np.full((n, np_), 0xEE, np.uint8)
    op = np.full((n, np_), 0xEE, np.uint8)
    err = L.PfError()
    st = L.lib.pf_host_pack_nibbles(t.ctypes.data_as(C.c_void_p), p.ctypes.data_as(C.c_void_p),
                                    t.strides[0], n, m, ot.ctypes.data_as(C.c_void_p),
                                    op.ctypes.data_as(C.c_void_p), simd, C.byref(err))
    return st, ot, op, err


def rand_records(rng, n, m, alphabet=b"ACGTN"):
    a = np.frombuffer(alphabet, np.uint8)
    return np.ascontiguousarray(a[rng.integers(0, len(a), size=(n, m))])


def test_nibble_pitch():
    for m, want in [(1, 4), (8, 4), (9, 8), (100, 52), (128, 64), (150, 76), (250, 128)]:
        assert L.lib.pf_nibble_pitch(m) == want


@pytest.mark.parametrize("simd", [1, 0])
@pytest.mark.parametrize("n,m", [(1, 1), (31, 5), (33, 31), (257, 32), (1000, 33), (300, 64),
                                 (777, 100), (513, 127), (513, 128), (200, 129), (129, 250),
                                 (5000, 100)])
def test_host_pack_matches_format(simd, n, m):
    rng = np.random.default_rng(n * 1000 + m)
    t, p = rand_records(rng, n, m), rand_records(rng, n, m)
    st, ot, op, _ = host_pack(t, p, simd)
    assert st == 0
    assert (ot == ref_nibbles(t)).all()
    assert (op == ref_nibbles(p)).all()


@pytest.mark.parametrize("simd", [1, 0])
def test_host_pack_strided_rows(simd):
    rng = np.random.default_rng(7)
    n, m, stride = 400, 100, 137
    buf_t = rand_records(rng, n, stride, b"ACGT")
    buf_p = rand_records(rng, n, stride, b"ACGT")
    buf_t[:, m:] = ord("x")  # bytes past m are never read
    buf_p[:, m:] = 0
    t, p = buf_t[:, :m], buf_p[:, :m]
    np_ = L.lib.pf_nibble_pitch(m)
    ot = np.zeros((n, np_), np.uint8)
    op = np.zeros((n, np_), np.uint8)
    err = L.PfError()
    st = L.lib.pf_host_pack_nibbles(buf_t.ctypes.data_as(C.c_void_p),
                                    buf_p.ctypes.data_as(C.c_void_p), stride, n, m,
                                    ot.ctypes.data_as(C.c_void_p), op.ctypes.data_as(C.c_void_p),
                                    simd, C.byref(err))
    assert st == 0
    assert (ot == ref_nibbles(np.ascontiguousarray(t))).all()
    assert (op == ref_nibbles(np.ascontiguousarray(p))).all()


@pytest.mark.parametrize("simd", [1, 0])
def test_host_pack_first_illegal_byte(simd):
    rng = np.random.default_rng(3)
    n, m = 7000, 100
    t = rand_records(rng, n, m, b"ACGT")
    p = t.copy()
    p[6000, 3] = ord("x")
    t[6000, 70] = ord("a")  # same pair: text before pattern
    p[100, 99] = 0
    p[100, 98] = ord("U")   # lowest position within the pair
    st, _, _, err = host_pack(t, p, simd)
    assert st == L.PF_ERR_ILLEGAL_CHARACTER
    assert (err.pair, err.field, err.position, err.byte) == (100, 1, 98, ord("U"))
    p[100, 98] = ord("A")
    p[100, 99] = ord("A")
    st, _, _, err = host_pack(t, p, simd)
    assert (err.pair, err.field, err.position, err.byte) == (6000, 0, 70, ord("a"))


@pytest.mark.parametrize("simd", [1, 0])
@pytest.mark.parametrize("byte", [0x00, 0x01, 0x40, 0x61, 0x81, 0xC1, 0xC7, 0xD4, 0xCE, 0x0E,
                                  0x14, ord("n"), ord("t"), 0xFF])
def test_host_pack_rejects_every_illegal_byte(simd, byte):
    """Bytes sharing the low 6 (or low 4) bits with a legal base must still fail."""
    n, m = 64, 130
    t = np.full((n, m), ord("A"), np.uint8)
    p = t.copy()
    p[40, 129] = byte
    st, _, _, err = host_pack(t, p, simd)
    assert st == L.PF_ERR_ILLEGAL_CHARACTER
    assert (err.pair, err.field, err.position, err.byte) == (40, 1, 129, byte)


def test_host_pack_accepts_exactly_the_alphabet():
    n, m = 1, 256
    t = np.arange(256, dtype=np.uint8)[None, :].copy()
    legal = set(b"ACGTN")
    for simd in (1, 0):
        for b in range(256):
            row = np.full((1, m), ord("C"), np.uint8)
            row[0, 200] = b
            st, _, _, _ = host_pack(row, row.copy(), simd)
            assert (st == 0) == (b in legal), (simd, b)
    del t, n


def test_host_pack_errors():
    t = np.zeros((4, 10), np.uint8)
    err = L.PfError()
    out = np.zeros(64, np.uint8)
    vp = t.ctypes.data_as(C.c_void_p)
    op = out.ctypes.data_as(C.c_void_p)
    assert L.lib.pf_host_pack_nibbles(vp, vp, 10, 4, 0, op, op, 1, C.byref(err)) == \
        L.PF_ERR_EMPTY_SEQUENCE
    assert L.lib.pf_host_pack_nibbles(vp, vp, 5, 4, 10, op, op, 1, C.byref(err)) == \
        L.PF_ERR_INVALID_PARAMETERS
    assert L.lib.pf_host_pack_nibbles(None, vp, 10, 4, 10, op, op, 1, C.byref(err)) == \
        L.PF_ERR_NULL_ARGUMENT
    assert L.lib.pf_host_pack_nibbles(vp, vp, 10, 0, 10, op, op, 1, C.byref(err)) == L.PF_OK


@pytest.mark.parametrize("offset", [0, 4, 8, 52, 60])
def test_host_pack_output_alignment(offset):
    """Any destination alignment gives the same bytes and nothing is written
    outside the rows (the 64-byte masked stores stop at each row's end)."""
    rng = np.random.default_rng(offset)
    n, m = 1000, 100
    t, p = rand_records(rng, n, m), rand_records(rng, n, m)
    np_ = L.lib.pf_nibble_pitch(m)
    raw_t = np.full(n * np_ + 192, 0xEE, np.uint8)
    raw_p = np.full(n * np_ + 192, 0xEE, np.uint8)
    base_t = (-raw_t.ctypes.data) % 64 + offset
    base_p = (-raw_p.ctypes.data) % 64 + offset
    err = L.PfError()
    st = L.lib.pf_host_pack_nibbles(t.ctypes.data_as(C.c_void_p), p.ctypes.data_as(C.c_void_p), m,
                                    n, m, C.c_void_p(raw_t.ctypes.data + base_t),
                                    C.c_void_p(raw_p.ctypes.data + base_p), 1, C.byref(err))
    assert st == 0
    assert (raw_t[base_t:base_t + n * np_].reshape(n, np_) == ref_nibbles(t)).all()
    assert (raw_p[base_p:base_p + n * np_].reshape(n, np_) == ref_nibbles(p)).all()
    assert (raw_t[:base_t] == 0xEE).all() and (raw_t[base_t + n * np_:] == 0xEE).all()
    assert (raw_p[:base_p] == 0xEE).all() and (raw_p[base_p + n * np_:] == 0xEE).all()


# ---- dibit records (the default upload format) ---------------------------------------

def ref_dibits(arr):
    """byte q of word w = codes of columns 16w+q, +4, +8, +12 at bits 0-1, 2-3, 4-5, 6-7;
    code = ASCII bits 1-2. N planes: bit c = column c is 'N' (LSB-first u32 words)."""
    n, m = arr.shape
    words = (m + 15) // 16
    pad = np.zeros((n, words * 16), np.uint8)
    pad[:, :m] = arr
    code = (pad >> 1) & 3
    blk = code.reshape(n, words, 4, 4)  # [word][t][q] -> column 16w + 4t + q
    out = np.zeros((n, words, 4), np.uint8)
    for t in range(4):
        out |= (blk[:, :, t, :] << (2 * t)).astype(np.uint8)
    nb = np.zeros((n, ((m + 31) // 32) * 32), np.uint8)
    nb[:, :m] = arr == ord("N")
    nplanes = np.packbits(nb, axis=1, bitorder="little")
    return out.reshape(n, words * 4), nplanes


def host_pack_dib(t, p, simd):
    n, m = t.shape
    dp, npitch = L.lib.pf_dibit_pitch(m), L.lib.pf_nplane_pitch(m)
    bufs = [np.full((n, w), 0xEE, np.uint8) for w in (dp, dp, npitch, npitch)]
    has_n = C.c_int(-1)
    err = L.PfError()
    st = L.lib.pf_host_pack_dibits(t.ctypes.data_as(C.c_void_p), p.ctypes.data_as(C.c_void_p), m,
                                   n, m, *[b.ctypes.data_as(C.c_void_p) for b in bufs],
                                   C.byref(has_n), simd, C.byref(err))
    return st, bufs, has_n.value, err


def test_dibit_pitches():
    for m, dp, npitch in [(1, 4, 4), (16, 4, 4), (17, 8, 4), (100, 28, 16), (150, 40, 20),
                          (250, 64, 32), (256, 64, 32)]:
        assert (L.lib.pf_dibit_pitch(m), L.lib.pf_nplane_pitch(m)) == (dp, npitch)


@pytest.mark.parametrize("simd", [1, 0])
@pytest.mark.parametrize("n,m,alphabet", [(1, 1, b"ACGT"), (33, 15, b"ACGT"), (300, 16, b"ACGTN"),
                                          (777, 100, b"ACGT"), (777, 100, b"ACGTN"),
                                          (513, 127, b"ACGTN"), (200, 129, b"ACGT"),
                                          (129, 250, b"ACGTN"), (5000, 100, b"ACGT")])
def test_host_pack_dibits_matches_format(simd, n, m, alphabet):
    rng = np.random.default_rng(n + m)
    t, p = rand_records(rng, n, m, alphabet), rand_records(rng, n, m, alphabet)
    st, (dt, dq, nt, nq), has_n, _ = host_pack_dib(t, p, simd)
    assert st == 0
    rt, rnt = ref_dibits(t)
    rp, rnp = ref_dibits(p)
    assert (dt == rt).all() and (dq == rp).all()
    assert has_n == int(bool((t == ord("N")).any() or (p == ord("N")).any()))
    if has_n:
        assert (nt == rnt).all() and (nq == rnp).all()
    else:
        assert (nt == 0xEE).all() and (nq == 0xEE).all()  # not written without an N


@pytest.mark.parametrize("simd", [1, 0])
def test_host_pack_dibits_first_illegal_byte(simd):
    rng = np.random.default_rng(5)
    n, m = 7000, 100
    t = rand_records(rng, n, m, b"ACGT")
    p = t.copy()
    p[6000, 3] = ord("x")
    t[6000, 70] = ord("a")
    p[100, 98] = ord("U")
    st, _, _, err = host_pack_dib(t, p, simd)
    assert st == L.PF_ERR_ILLEGAL_CHARACTER
    assert (err.pair, err.field, err.position, err.byte) == (100, 1, 98, ord("U"))
    for b in (0x00, 0xC1, 0x4E | 0x80, ord("n")):
        q = t.copy()
        q[42, 17] = b
        st, _, _, err = host_pack_dib(q, t.copy(), simd)
        assert st == L.PF_ERR_ILLEGAL_CHARACTER and (err.pair, err.field, err.position) == (42, 0, 17)
