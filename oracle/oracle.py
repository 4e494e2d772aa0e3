"""TEST INFRASTRUCTURE ONLY — ctypes front end for the two CPU checkers.

* ``Oracle``   — the plain-C restatement (oracle/shouji_oracle.c).
* ``Reference`` — the unmodified reference library compiled from its sources
  (oracle/_ref/libprefilter_ref.so, built by oracle/Makefile); ``None`` when
  that build is absent.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline leg /
``--impl reference`` arm may import this module. The product package never
does: its only compute path is the CUDA extension.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libshouji_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libprefilter_ref.so")

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


class OracleError(Exception):
    def __init__(self, code, pair=0, field=0, position=0, byte=0):
        super().__init__(f"oracle status {code} (pair={pair} field={field} pos={position} byte={byte})")
        self.code, self.pair, self.field, self.position, self.byte = code, pair, field, position, byte


class _SoError(C.Structure):
    _fields_ = [("code", C.c_int), ("pair", C.c_uint64), ("field", C.c_int),
                ("position", C.c_uint64), ("byte", C.c_int)]


def build():
    """Compile the checkers (make -C oracle). Safe to call repeatedly."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _records(text, pattern):
    text = np.ascontiguousarray(text, dtype=np.uint8)
    pattern = np.ascontiguousarray(pattern, dtype=np.uint8)
    assert text.shape == pattern.shape and text.ndim == 2
    return text, pattern


class Oracle:
    """The C restatement (see shouji_oracle.c for the reference file:line map)."""

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            build()
        lib = C.CDLL(path)
        lib.so_shouji_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t, C.c_size_t,
                                        C.c_uint32, C.c_uint, C.c_uint, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.POINTER(_SoError)]
        lib.so_shouji_one.argtypes = [C.c_char_p, C.c_size_t, C.c_char_p, C.c_size_t, C.c_uint32,
                                      C.c_uint, C.c_void_p, C.POINTER(C.c_uint32),
                                      C.POINTER(C.c_int)]
        lib.so_neighborhood.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t, C.c_uint32, C.c_void_p]
        lib.so_generate_pairs.argtypes = [C.c_uint64, C.c_size_t, C.c_size_t, C.c_uint32,
                                          C.c_uint32, C.c_void_p, C.c_void_p, C.c_size_t]
        lib.so_banded_edit_distance.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t, C.c_uint32]
        lib.so_banded_edit_distance.restype = C.c_int32
        lib.so_set_variant.argtypes = [C.c_int]
        lib.so_magnet_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t, C.c_size_t,
                                        C.c_uint32, C.c_uint, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.POINTER(_SoError)]
        lib.so_magnet_one.argtypes = [C.c_char_p, C.c_size_t, C.c_char_p, C.c_size_t, C.c_uint32,
                                      C.c_void_p, C.POINTER(C.c_uint32), C.POINTER(C.c_int)]
        lib.so_recover_subsequences.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t, C.c_uint32,
                                                C.c_uint32, C.c_void_p, C.c_void_p]
        lib.so_recover_subsequences.restype = C.c_size_t
        lib.so_longest_zero_run.argtypes = [C.c_void_p, C.c_size_t, C.c_size_t, C.c_size_t,
                                            C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]
        # config_oracle.c: generator mirror of csrc/datagen.cu + vectorisable restatement
        lib.so_gen_config.argtypes = [C.c_int, C.c_uint64, C.c_uint32, C.c_int, C.c_uint64,
                                      C.c_size_t, C.c_void_p, C.c_void_p, C.c_size_t]
        lib.so_gen_config_rows.argtypes = [C.c_int, C.c_uint64, C.c_uint32, C.c_int, C.c_void_p,
                                           C.c_size_t, C.c_void_p, C.c_void_p, C.c_size_t]
        lib.so_shouji_fast_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t,
                                             C.c_int, C.c_uint32, C.c_uint, C.c_uint, C.c_void_p]
        lib.so_config_estimates.argtypes = [C.c_int, C.c_uint64, C.c_uint32, C.c_int, C.c_uint32,
                                            C.c_uint, C.c_uint64, C.c_size_t, C.c_uint,
                                            C.c_void_p]
        lib.so_shouji_fast_one.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_uint32, C.c_uint,
                                           C.c_void_p, C.POINTER(C.c_uint32), C.POINTER(C.c_int)]
        self.lib = lib

    def set_variant(self, v: int):
        """Mutation-test knob: 0 reference rules; 1 reverse scan; 2 no leading-zero
        tie-break; 3 non-strict commit; 4 pattern/text swapped."""
        self.lib.so_set_variant(v)

    def shouji_batch(self, text, pattern, e, width=4, threads=None, estimates=True, bits=False):
        """Returns (accept_bitmap u32[ceil(n/32)], estimates u32[n] | None, bits u64[n, W64] | None)."""
        text, pattern = _records(text, pattern)
        n, m = text.shape
        threads = threads or os.cpu_count() or 1
        acc = np.zeros((n + 31) // 32, np.uint32)
        est = np.zeros(n, np.uint32) if estimates else None
        bv = np.zeros((n, (m + 63) // 64), np.uint64) if bits else None
        err = _SoError()
        st = self.lib.so_shouji_batch(_ptr(text), _ptr(pattern), m, n, m, e, width, threads,
                                      _ptr(acc), _ptr(est), _ptr(bv), C.byref(err))
        if st:
            raise OracleError(st, err.pair, err.field, err.position, err.byte)
        return acc, est, bv

    # ---- config_oracle.c -----------------------------------------------------------
    def gen_config(self, kind, seed, param, m, begin, count, pitch=None):
        """Pairs [begin, begin+count) of BASELINE config `kind` (1..4), byte-identical
        to the device generator (csrc/datagen.cu). Returns (text, pattern) u8[count, pitch]."""
        pitch = pitch or m
        t = np.zeros((count, pitch), np.uint8)
        p = np.zeros((count, pitch), np.uint8)
        if count and self.lib.so_gen_config(kind, seed, param, m, begin, count, _ptr(t), _ptr(p),
                                            pitch):
            raise OracleError(-1)
        return t, p

    def gen_config_rows(self, kind, seed, param, m, rows):
        """The generator's pairs at arbitrary indices `rows` -> (text, pattern) u8[k, m]."""
        idx = np.ascontiguousarray(rows, dtype=np.uint64)
        t = np.zeros((idx.size, m), np.uint8)
        p = np.zeros((idx.size, m), np.uint8)
        if idx.size and self.lib.so_gen_config_rows(kind, seed, param, m, _ptr(idx), idx.size,
                                                    _ptr(t), _ptr(p), m):
            raise OracleError(-1)
        return t, p

    def shouji_fast_batch(self, text, pattern, e, width=4, threads=None):
        """Estimates u32[n] of validated records by the vectorisable restatement."""
        text, pattern = _records(text, pattern)
        n, m = text.shape
        est = np.zeros(n, np.uint32)
        st = self.lib.so_shouji_fast_batch(_ptr(text), _ptr(pattern), m, n, m, e, width,
                                           threads or os.cpu_count() or 1, _ptr(est))
        if st:
            raise OracleError(st)
        return est

    def config_estimates(self, kind, seed, param, m, e, begin, count, width=4, threads=None):
        """Estimates u32[count] of config pairs [begin, begin+count), generated on the fly."""
        est = np.zeros(count, np.uint32)
        st = self.lib.so_config_estimates(kind, seed, param, m, e, width, begin, count,
                                          threads or os.cpu_count() or 1, _ptr(est))
        if st:
            raise OracleError(st)
        return est

    def shouji_one(self, pattern: str, text: str, e: int, width: int = 4):
        """shouji_filter(seq(pattern), seq(text), e, width) -> (accept, estimate, bits str)."""
        pb, tb = pattern.encode(), text.encode()
        bits = np.zeros(max(len(tb), 1), np.uint8)
        est, acc = C.c_uint32(), C.c_int()
        st = self.lib.so_shouji_one(pb, len(pb), tb, len(tb), e, width, _ptr(bits),
                                    C.byref(est), C.byref(acc))
        if st:
            raise OracleError(st)
        return bool(acc.value), est.value, "".join("1" if b else "0" for b in bits[:len(tb)])

    def neighborhood(self, pattern: str, text: str, e: int):
        """(2e+1, m) uint8 map, row d+e."""
        m = len(text)
        out = np.zeros((2 * e + 1, m), np.uint8)
        self.lib.so_neighborhood(pattern.encode(), text.encode(), m, e, _ptr(out))
        return out

    def generate_pairs(self, seed, count, length, lo, hi):
        """Restated generate_pairs -> (text u8[count, length], pattern u8[count, length])."""
        t = np.zeros((count, length), np.uint8)
        p = np.zeros((count, length), np.uint8)
        st = self.lib.so_generate_pairs(seed, count, length, lo, hi, _ptr(t), _ptr(p), length)
        if st:
            raise OracleError(st)
        return t, p

    def substitution_pairs(self, seed, count, m, max_subs):
        """Restated substitution_pairs (acceptance_tests.cpp:252-276, criterion 7)
        -> (text u8[count, m], pattern u8[count, m])."""
        t = np.zeros((count, m), np.uint8)
        p = np.zeros((count, m), np.uint8)
        self.lib.so_substitution_pairs(C.c_uint64(seed), C.c_size_t(count), C.c_size_t(m),
                                       C.c_uint32(max_subs), _ptr(t), _ptr(p), C.c_size_t(m))
        return t, p

    def banded_edit_distance(self, pattern: bytes, text: bytes, e: int) -> int:
        return self.lib.so_banded_edit_distance(pattern, text, len(text), e)

    # ---- MAGNET (magnet.cpp) ----
    def magnet_batch(self, text, pattern, e, threads=None, estimates=True, bits=False):
        """Returns (accept_bitmap u32[ceil(n/32)], estimates u32[n] | None, bits u64[n, W64] | None)."""
        text, pattern = _records(text, pattern)
        n, m = text.shape
        threads = threads or os.cpu_count() or 1
        acc = np.zeros((n + 31) // 32, np.uint32)
        est = np.zeros(n, np.uint32) if estimates else None
        bv = np.zeros((n, (m + 63) // 64), np.uint64) if bits else None
        err = _SoError()
        st = self.lib.so_magnet_batch(_ptr(text), _ptr(pattern), m, n, m, e, threads, _ptr(acc),
                                      _ptr(est), _ptr(bv), C.byref(err))
        if st:
            raise OracleError(st, err.pair, err.field, err.position, err.byte)
        return acc, est, bv

    def magnet_one(self, pattern: str, text: str, e: int):
        """magnet_filter(seq(pattern), seq(text), e) -> (accept, estimate, bits str)."""
        pb, tb = pattern.encode(), text.encode()
        bits = np.zeros(max(len(tb), 1), np.uint8)
        est, acc = C.c_uint32(), C.c_int()
        st = self.lib.so_magnet_one(pb, len(pb), tb, len(tb), e, _ptr(bits), C.byref(est),
                                    C.byref(acc))
        if st:
            raise OracleError(st)
        return bool(acc.value), est.value, "".join("1" if b else "0" for b in bits[:len(tb)])

    def recover(self, pattern: str, text: str, e: int, budget: int):
        """recover_subsequences(map(pattern, text, e), budget) -> ([(d, start, len, lo, hi)], bits str)."""
        m = len(text)
        bv = np.zeros(m, np.uint8)
        class _X(C.Structure):
            _fields_ = [("diagonal", C.c_int), ("start", C.c_size_t), ("len", C.c_size_t),
                        ("lo", C.c_size_t), ("hi", C.c_size_t)]
        xs = (_X * max(budget, 1))()
        k = self.lib.so_recover_subsequences(pattern.encode(), text.encode(), m, e, budget,
                                             _ptr(bv), C.cast(xs, C.c_void_p))
        ext = [(xs[i].diagonal, xs[i].start, xs[i].len, xs[i].lo, xs[i].hi) for i in range(k)]
        return ext, "".join("1" if b else "0" for b in bv)

    def longest_zero_run(self, bits: str, lo: int, hi: int):
        b = np.frombuffer(bits.encode(), np.uint8) - ord("0")
        b = np.ascontiguousarray(b.astype(np.uint8))
        st, ln = C.c_size_t(), C.c_size_t()
        self.lib.so_longest_zero_run(_ptr(b), len(bits), lo, hi, C.byref(st), C.byref(ln))
        return st.value, ln.value


class Reference:
    """The unmodified reference library (oracle/_ref/libprefilter_ref.so)."""

    def __init__(self, path=REF_SO):
        lib = C.CDLL(path)
        lib.ref_generate_pairs.argtypes = [C.c_uint64, C.c_size_t, C.c_size_t, C.c_uint32,
                                           C.c_uint32, C.c_void_p, C.c_void_p, C.c_size_t]
        lib.ref_pack.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t, C.c_size_t,
                                 C.POINTER(C.c_int), C.POINTER(C.c_uint64), C.POINTER(C.c_int),
                                 C.POINTER(C.c_uint64), C.POINTER(C.c_int)]
        lib.ref_pack.restype = C.c_void_p
        lib.ref_free.argtypes = [C.c_void_p]
        lib.ref_shouji_run.argtypes = [C.c_void_p, C.c_uint32, C.c_uint, C.c_uint, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_size_t]
        lib.ref_magnet_run.argtypes = [C.c_void_p, C.c_uint32, C.c_uint, C.c_void_p, C.c_void_p]
        lib.ref_banded_run.argtypes = [C.c_void_p, C.c_uint32, C.c_uint, C.c_void_p]
        lib.ref_shouji_one.argtypes = [C.c_char_p, C.c_size_t, C.c_char_p, C.c_size_t, C.c_uint32,
                                       C.c_uint, C.POINTER(C.c_int), C.POINTER(C.c_uint32),
                                       C.c_char_p]
        lib.ref_hardware_concurrency.restype = C.c_uint
        lib.ref_load_pairs_tsv.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t),
                                           C.POINTER(C.c_size_t), C.c_char_p, C.c_size_t]
        lib.ref_magnet_one.argtypes = [C.c_char_p, C.c_size_t, C.c_char_p, C.c_size_t, C.c_uint32,
                                       C.POINTER(C.c_int), C.POINTER(C.c_uint32), C.c_char_p,
                                       C.c_int64, C.c_void_p, C.c_size_t,
                                       C.POINTER(C.c_size_t), C.c_char_p]
        lib.ref_export_planes.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        lib.ref_longest_zero_run.argtypes = [C.c_char_p, C.c_size_t, C.c_size_t, C.c_size_t,
                                             C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]
        self.lib = lib

    def load_pairs(self, data: bytes):
        """load_pairs over bytes -> (status, n, m, message)."""
        n, m = C.c_size_t(), C.c_size_t()
        buf = C.create_string_buffer(512)
        st = self.lib.ref_load_pairs_tsv(data, len(data), C.byref(n), C.byref(m), buf, 512)
        return st, n.value, m.value, buf.value.decode(errors="replace")

    @staticmethod
    def available(path=REF_SO):
        return os.path.exists(path)

    def hardware_concurrency(self):
        return self.lib.ref_hardware_concurrency()

    def generate_pairs(self, seed, count, length, lo, hi):
        t = np.zeros((count, length), np.uint8)
        p = np.zeros((count, length), np.uint8)
        st = self.lib.ref_generate_pairs(seed, count, length, lo, hi, _ptr(t), _ptr(p), length)
        if st:
            raise OracleError(st)
        return t, p

    def pack(self, text, pattern):
        """Pack with packed_sequence::from_string; returns a handle (free with .free)."""
        text, pattern = _records(text, pattern)
        n, m = text.shape
        code, pair, field, pos, byte = C.c_int(), C.c_uint64(), C.c_int(), C.c_uint64(), C.c_int()
        h = self.lib.ref_pack(_ptr(text), _ptr(pattern), m, n, m, C.byref(code), C.byref(pair),
                              C.byref(field), C.byref(pos), C.byref(byte))
        if not h:
            raise OracleError(code.value, pair.value, field.value, pos.value, byte.value)
        return _Packed(self, h, n, m)

    def shouji_batch(self, text, pattern, e, width=4, threads=None, estimates=True, bits=False):
        packed = self.pack(text, pattern)
        try:
            return packed.shouji(e, width, threads, estimates, bits)
        finally:
            packed.free()

    def magnet_batch(self, text, pattern, e, threads=None):
        packed = self.pack(text, pattern)
        try:
            return packed.magnet(e, threads)
        finally:
            packed.free()

    def magnet_one(self, pattern: str, text: str, e: int, budget: int | None = None):
        """magnet_filter -> (accept, estimate, bits str); with budget also
        recover_subsequences(map, budget) -> ([(d, start, len, lo, hi)], bits str)."""
        pb, tb = pattern.encode(), text.encode()
        acc, est = C.c_int(), C.c_uint32()
        buf = C.create_string_buffer(len(tb) + 1)
        rbuf = C.create_string_buffer(len(tb) + 1)
        nmax = max(budget or 0, 1)
        ext = (C.c_int64 * (5 * nmax))()
        n_ext = C.c_size_t()
        st = self.lib.ref_magnet_one(pb, len(pb), tb, len(tb), e, C.byref(acc), C.byref(est), buf,
                                     -1 if budget is None else budget, ext, nmax, C.byref(n_ext),
                                     rbuf)
        if st:
            raise OracleError(st)
        out = (bool(acc.value), est.value, buf.value.decode())
        if budget is None:
            return out
        xs = [tuple(int(v) for v in ext[5 * k:5 * k + 5]) for k in range(min(n_ext.value, nmax))]
        return out, (xs, rbuf.value.decode())

    def longest_zero_run(self, bits: str, lo: int, hi: int):
        st, ln = C.c_size_t(), C.c_size_t()
        self.lib.ref_longest_zero_run(bits.encode(), len(bits), lo, hi, C.byref(st), C.byref(ln))
        return st.value, ln.value

    def shouji_one(self, pattern: str, text: str, e: int, width: int = 4):
        pb, tb = pattern.encode(), text.encode()
        acc, est = C.c_int(), C.c_uint32()
        buf = C.create_string_buffer(len(tb) + 1)
        st = self.lib.ref_shouji_one(pb, len(pb), tb, len(tb), e, width, C.byref(acc),
                                     C.byref(est), buf)
        if st:
            raise OracleError(st)
        return bool(acc.value), est.value, buf.value.decode()


class _Packed:
    def __init__(self, ref, handle, n, m):
        self.ref, self.h, self.n, self.m = ref, handle, n, m

    def shouji(self, e, width=4, threads=None, estimates=True, bits=False):
        threads = threads or self.ref.hardware_concurrency() or 1
        acc = np.zeros((self.n + 31) // 32, np.uint32)
        est = np.zeros(self.n, np.uint32) if estimates else None
        wpp = (self.m + 63) // 64
        bv = np.zeros((self.n, wpp), np.uint64) if bits else None
        st = self.ref.lib.ref_shouji_run(self.h, e, width, threads, _ptr(acc), _ptr(est),
                                         _ptr(bv), wpp)
        if st:
            raise OracleError(st)
        return acc, est, bv

    def magnet(self, e, threads=None):
        threads = threads or self.ref.hardware_concurrency() or 1
        acc = np.zeros((self.n + 31) // 32, np.uint32)
        est = np.zeros(self.n, np.uint32)
        st = self.ref.lib.ref_magnet_run(self.h, e, threads, _ptr(acc), _ptr(est))
        if st:
            raise OracleError(st)
        return acc, est

    def planes(self):
        """The reference's own packed_sequence planes: (text, pattern) u64[n, 3, ceil(m/64)]."""
        w = (self.m + 63) // 64
        t = np.zeros((self.n, 3, w), np.uint64)
        p = np.zeros((self.n, 3, w), np.uint64)
        self.ref.lib.ref_export_planes(self.h, _ptr(t), _ptr(p))
        return t, p

    def banded(self, e, threads=None):
        threads = threads or self.ref.hardware_concurrency() or 1
        out = np.zeros(self.n, np.int32)
        st = self.ref.lib.ref_banded_run(self.h, e, threads, _ptr(out))
        if st:
            raise OracleError(st)
        return out

    def free(self):
        if self.h:
            self.ref.lib.ref_free(self.h)
            self.h = None
