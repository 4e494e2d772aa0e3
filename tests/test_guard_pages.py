"""Out-of-bounds checks of the host upload stage with guard pages (compute-sanitizer
is not available on this pool; tests/guard.py): the AVX-512 host pack reads ASCII
records and writes dibit / N-plane / nibble records; every input and output array
here ends (or starts) at an inaccessible page, with the tight stride m, so a load
or store one byte out of bounds crashes the test. Results must equal the same
call on ordinary arrays."""
import ctypes as C

import numpy as np
import pytest

import paper_1809_07858_b200 as pf
from paper_1809_07858_b200 import _lib as L

from guard import host_guarded

ALPHA = np.frombuffer(b"ACGTN", np.uint8)


def _records(rng, n, m, guarded, at_end):
    t = ALPHA[rng.integers(0, 5, size=(n, m))]
    p = ALPHA[rng.integers(0, 5, size=(n, m))]
    if not guarded:
        return t, p
    gt = host_guarded(n * m, at_end).reshape(n, m)
    gp = host_guarded(n * m, at_end).reshape(n, m)
    gt[:] = t
    gp[:] = p
    return gt, gp


def _out(nbytes, guarded, at_end):
    return host_guarded(nbytes, at_end) if guarded else np.zeros(nbytes, np.uint8)


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def _dibits(t, p, n, m, simd, guarded, at_end):
    dp, npp = pf.dibit_pitch(m), pf.nplane_pitch(m)
    dt, dq = _out(n * dp, guarded, at_end), _out(n * dp, guarded, at_end)
    nt, nq = _out(n * npp, guarded, at_end), _out(n * npp, guarded, at_end)
    has_n, err = C.c_int(), L.PfError()
    st = L.lib.pf_host_pack_dibits(_ptr(t), _ptr(p), m, n, m, _ptr(dt), _ptr(dq), _ptr(nt),
                                   _ptr(nq), C.byref(has_n), simd, C.byref(err))
    assert st == 0
    return [x.copy() for x in (dt, dq, nt, nq)]


def _nibbles(t, p, n, m, simd, guarded, at_end):
    npch = pf.nibble_pitch(m)
    ot, op = _out(n * npch, guarded, at_end), _out(n * npch, guarded, at_end)
    err = L.PfError()
    st = L.lib.pf_host_pack_nibbles(_ptr(t), _ptr(p), m, n, m, _ptr(ot), _ptr(op), simd,
                                    C.byref(err))
    assert st == 0
    return [ot.copy(), op.copy()]


@pytest.mark.parametrize("m", [1, 7, 15, 16, 17, 31, 63, 64, 65, 100, 127, 128, 129, 250, 1000])
@pytest.mark.parametrize("at_end", [True, False])
def test_host_pack_stays_in_bounds(m, at_end):
    rng = np.random.default_rng(m)
    for n in (1, 3, 33, 1030):
        for simd in (1, 0):
            t, p = _records(rng, n, m, False, at_end)
            gt, gp = _records(np.random.default_rng(0), n, m, True, at_end)
            gt[:] = t
            gp[:] = p
            want = _dibits(t, p, n, m, simd, False, at_end)
            got = _dibits(gt, gp, n, m, simd, True, at_end)
            for x, y in zip(want, got):
                assert (x == y).all(), (m, n, simd)
            if m <= 4088:
                want = _nibbles(t, p, n, m, simd, False, at_end)
                got = _nibbles(gt, gp, n, m, simd, True, at_end)
                for x, y in zip(want, got):
                    assert (x == y).all(), (m, n, simd)


def test_host_validation_stays_in_bounds():
    # the loader's alphabet check reads the well-formed prefix in place
    rng = np.random.default_rng(3)
    for m in (5, 64, 100, 333):
        n = 257
        t, p = _records(rng, n, m, True, True)
        p[-1, -1] = ord("x")  # the very last byte of the buffer
        with pytest.raises(pf.illegal_character_error) as ex:
            pf.host_pack_dibits(t, p)
        assert (ex.value.pair, ex.value.field, ex.value.position()) == (n - 1, 1, m - 1)
