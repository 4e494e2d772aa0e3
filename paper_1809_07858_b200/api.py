"""Python mirror of the reference's public interface for the Shouji path.

Names, argument meaning and error behaviour follow ``prefilter`` (C++,
/root/reference/proj/include/prefilter/): ``packed_sequence``, ``bitvector``,
``filter_decision``, ``shouji_filter(pattern, text, e, width=4)``, ``run_filter``
and the ``error`` hierarchy of errors.hpp. Every decision is computed by the
sm_100a kernels behind the C ABI (libshouji_b200.so); this module only moves
buffers and maps status codes onto exceptions.

Batch entry points (``shouji_filter_batch``, ``shouji_filter_device``) are the
fast path: they take N equal-length ASCII records at once, which is how the
reference's callers (evaluate, run_bench, the CLI) drive the filter through
parallel_for_pairs.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib as L

default_window_width = 4
min_window_width = 3
max_window_width = 8


# ---------------------------------------------------------------------------
# Errors (proj/include/prefilter/errors.hpp:11-84)
# ---------------------------------------------------------------------------
class error(RuntimeError):
    """Base of every recoverable error (prefilter::error)."""


class empty_sequence_error(error):
    def __init__(self, msg="empty sequence"):
        super().__init__(msg)


class illegal_character_error(error):
    def __init__(self, position: int, byte: int, pair: int | None = None, field: int | None = None):
        ch = chr(byte) if 32 <= byte < 127 else f"\\x{byte:02x}"
        where = "" if pair is None else f" of {'text' if field == 0 else 'pattern'} {pair}"
        super().__init__(f"illegal character '{ch}' at position {position}{where}")
        self._position, self._byte, self.pair, self.field = position, byte, pair, field

    def position(self) -> int:
        return self._position

    def byte(self) -> str:
        return chr(self._byte)


class length_mismatch_error(error):
    pass


class threshold_too_large_error(error):
    pass


class out_of_band_error(error):
    pass


class parse_error(error):
    def __init__(self, line: int, reason: str):
        super().__init__(f"line {line}: {reason}")
        self._line = line

    def line(self) -> int:
        return self._line


class invalid_parameters_error(error):
    pass


class device_error(RuntimeError):
    """No usable sm_100 device, or a CUDA failure (not a reference error class)."""


def _raise(status: int, err: L.PfError | None = None):
    if status == L.PF_OK:
        return
    msg = err.message.decode(errors="replace") if err is not None else L.lib.pf_status_string(status).decode()
    if status == L.PF_ERR_EMPTY_SEQUENCE:
        raise empty_sequence_error()
    if status == L.PF_ERR_ILLEGAL_CHARACTER:
        raise illegal_character_error(int(err.position), int(err.byte), int(err.pair), int(err.field))
    if status == L.PF_ERR_LENGTH_MISMATCH:
        raise length_mismatch_error(msg)
    if status == L.PF_ERR_PARSE:
        line = int(err.line) if err is not None else 0
        prefix = f"line {line}: "
        raise parse_error(line, msg[len(prefix):] if msg.startswith(prefix) else msg)
    if status == L.PF_ERR_THRESHOLD_TOO_LARGE:
        raise threshold_too_large_error(msg)
    if status == L.PF_ERR_OUT_OF_BAND:
        raise out_of_band_error(msg)
    if status == L.PF_ERR_INVALID_PARAMETERS:
        raise invalid_parameters_error(msg)
    raise device_error(f"{L.lib.pf_status_string(status).decode()}: {msg}")


# ---------------------------------------------------------------------------
# Containers (bitvector.hpp, packed_sequence.hpp, filter_decision.hpp)
# ---------------------------------------------------------------------------
class bitvector:
    """Fixed-length LSB-first bit sequence in uint64 words (bitvector.hpp:16-129)."""

    def __init__(self, nbits: int = 0, value: bool = False, words=None):
        self._n = int(nbits)
        nw = (self._n + 63) // 64
        if words is None:
            self._w = np.full(nw, np.uint64(0xFFFFFFFFFFFFFFFF) if value else 0, np.uint64)
        else:
            self._w = np.array(words, dtype=np.uint64).reshape(-1)[:nw].copy()
        if self._n & 63 and nw:
            self._w[-1] &= np.uint64((1 << (self._n & 63)) - 1)

    def size(self) -> int:
        return self._n

    def get(self, i: int) -> bool:
        return bool((int(self._w[i >> 6]) >> (i & 63)) & 1)

    def count_ones(self) -> int:
        return int(sum(bin(int(w)).count("1") for w in self._w))

    def count_zeros(self) -> int:
        return self._n - self.count_ones()

    def words(self):
        return self._w

    def to_string(self) -> str:
        return "".join("1" if self.get(i) else "0" for i in range(self._n))

    def __eq__(self, other):
        return isinstance(other, bitvector) and self._n == other._n and bool((self._w == other._w).all())

    def __repr__(self):
        return f"bitvector({self.to_string()!r})"


class packed_sequence:
    """A validated A/C/G/T/N sequence (packed_sequence.hpp:17-54).

    ``from_string`` enforces the reference codec's contract (upper case only;
    empty -> empty_sequence_error; first bad byte -> illegal_character_error with
    its 0-based position). The planes themselves are built on the device by the
    filter kernels from the ASCII bytes kept here.
    """

    __slots__ = ("_ascii",)

    def __init__(self, ascii_bytes: bytes = b""):
        self._ascii = ascii_bytes

    @staticmethod
    def from_string(raw) -> "packed_sequence":
        b = raw.encode() if isinstance(raw, str) else bytes(raw)
        if len(b) == 0:
            raise empty_sequence_error()
        arr = np.frombuffer(b, np.uint8)
        ok = np.isin(arr, np.frombuffer(b"ACGTN", np.uint8))
        if not ok.all():
            pos = int(np.argmin(ok))
            raise illegal_character_error(pos, int(arr[pos]))
        return packed_sequence(b)

    def to_string(self) -> str:
        return self._ascii.decode()

    def ascii(self) -> bytes:
        return self._ascii

    def size(self) -> int:
        return len(self._ascii)

    def is_n(self, i: int) -> bool:
        return self._ascii[i] == ord("N")

    def code(self, i: int) -> int:
        return {ord("A"): 0, ord("C"): 1, ord("G"): 2, ord("T"): 3}.get(self._ascii[i], 0)

    def base_at(self, i: int) -> str:
        return chr(self._ascii[i])

    def __eq__(self, other):
        return isinstance(other, packed_sequence) and self._ascii == other._ascii

    def __len__(self):
        return len(self._ascii)


def seq(s) -> packed_sequence:
    """Test shorthand, as in proj/tests/helpers.hpp:17-19."""
    return packed_sequence.from_string(s)


@dataclass
class filter_decision:
    """Outcome of one filter run (filter_decision.hpp:12-16)."""
    accept: bool = False
    edit_estimate: int = 0
    bits: bitvector = field(default_factory=bitvector)


# ---------------------------------------------------------------------------
# Device context
# ---------------------------------------------------------------------------
class Context:
    """A set of devices the batch calls are sharded across (pf_ctx)."""

    def __init__(self, devices: Sequence[int] | None = None):
        self._h = C.c_void_p()
        if devices:
            arr = (C.c_int * len(devices))(*devices)
            st = L.lib.pf_ctx_create(arr, len(devices), C.byref(self._h))
        else:
            st = L.lib.pf_ctx_create(None, 0, C.byref(self._h))
        _raise(st)

    @property
    def handle(self):
        return self._h

    def device_count(self) -> int:
        return L.lib.pf_ctx_device_count(self._h)

    def set_shard_chunk(self, chunk_pairs: int) -> None:
        """0: one contiguous shard per device (default); > 0: chunks of that many pairs
        dealt round-robin over the devices (pf_ctx_set_shard_chunk)."""
        _raise(L.lib.pf_ctx_set_shard_chunk(self._h, int(chunk_pairs)))

    def close(self):
        if self._h:
            L.lib.pf_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Context | None = None
_ctx_lock = threading.Lock()


def default_context() -> Context:
    global _default_ctx
    with _ctx_lock:
        if _default_ctx is None:
            _default_ctx = Context()
        return _default_ctx


def device_count() -> int:
    return L.lib.pf_device_count()


def launch_count() -> int:
    """Kernel launches issued by this process (all contexts)."""
    return int(L.lib.pf_launch_count())


def transfer_bytes() -> tuple[int, int]:
    """(host->device, device->host) bytes moved by the host entry points so far."""
    h2d, d2h = C.c_uint64(), C.c_uint64()
    L.lib.pf_transfer_bytes(C.byref(h2d), C.byref(d2h))
    return int(h2d.value), int(d2h.value)


def host_read_bandwidth(buf: np.ndarray, passes: int = 3) -> float:
    """GB/s at which the host cores stream-read ``buf`` (pf_host_read_bandwidth)."""
    buf = np.ascontiguousarray(buf)
    return float(L.lib.pf_host_read_bandwidth(buf.ctypes.data_as(C.c_void_p), buf.nbytes, passes))


def device_pitch(m: int) -> int:
    return int(L.lib.pf_device_pitch(m))


# ---------------------------------------------------------------------------
# Filter entry points
# ---------------------------------------------------------------------------
def shouji_filter(pattern: packed_sequence, text: packed_sequence, e: int,
                  width: int = default_window_width, ctx: Context | None = None) -> filter_decision:
    """shouji_filter(pattern=read, text=reference segment, e, width) — shouji.hpp:57-59.

    Raises length_mismatch_error, then invalid_parameters_error (width), in the
    reference's order (shouji.cpp:44-47); e >= m accepts with estimate 0.
    """
    ctx = ctx or default_context()
    pb, tb = pattern.ascii(), text.ascii()
    acc, est = C.c_int(), C.c_uint32()
    nbits = len(tb)
    words = np.zeros(max((nbits + 63) // 64, 1), np.uint64)
    err = L.PfError()
    st = L.lib.pf_shouji_filter_one(ctx.handle, pb, len(pb), tb, len(tb), int(e), int(width),
                                    C.byref(acc), C.byref(est), words.ctypes.data_as(C.c_void_p),
                                    C.byref(err))
    _raise(st, err)
    return filter_decision(bool(acc.value), int(est.value), bitvector(nbits, words=words))


def magnet_filter(pattern: packed_sequence, text: packed_sequence, e: int,
                  ctx: Context | None = None) -> filter_decision:
    """magnet_filter(pattern=read, text=reference segment, e) — magnet.hpp:55-57.

    Raises length_mismatch_error (magnet.cpp:79-80); e >= m accepts with estimate 0.
    """
    ctx = ctx or default_context()
    pb, tb = pattern.ascii(), text.ascii()
    acc, est = C.c_int(), C.c_uint32()
    nbits = len(tb)
    words = np.zeros(max((nbits + 63) // 64, 1), np.uint64)
    err = L.PfError()
    st = L.lib.pf_magnet_filter_one(ctx.handle, pb, len(pb), tb, len(tb), int(e), C.byref(acc),
                                    C.byref(est), words.ctypes.data_as(C.c_void_p), C.byref(err))
    _raise(st, err)
    return filter_decision(bool(acc.value), int(est.value), bitvector(nbits, words=words))


def run_filter(algo: str, pattern: packed_sequence, text: packed_sequence, e: int,
               width: int = default_window_width) -> filter_decision:
    """run_filter (evaluate.cpp:13-21): "shouji" or "magnet" (width is Shouji's only)."""
    if algo == "shouji":
        return shouji_filter(pattern, text, e, width)
    if algo == "magnet":
        return magnet_filter(pattern, text, e)
    raise invalid_parameters_error(f"unknown filter '{algo}'")


def _as_records(x, m=None):
    a = np.ascontiguousarray(x, dtype=np.uint8)
    if a.ndim != 2:
        raise invalid_parameters_error("records must be a 2-D uint8 array [n, stride]")
    return a


def shouji_filter_batch(text, pattern, e: int, width: int = default_window_width, m: int | None = None,
                        estimates: bool = False, bits: bool = False, ctx: Context | None = None):
    """Filter N pairs of host ASCII records; text[i] is pair i's reference
    segment, pattern[i] its read (uint8 arrays [n, stride], first m bytes used).

    Returns (accept_bitmap u32[ceil(n/32)], estimates u32[n] | None, bits u64[n, ceil(m/64)] | None).
    """
    ctx = ctx or default_context()
    text = _as_records(text)
    pattern = _as_records(pattern)
    if text.shape != pattern.shape:
        raise length_mismatch_error("text and pattern record arrays differ in shape")
    n, stride = text.shape
    m = stride if m is None else int(m)
    acc = np.zeros((n + 31) // 32, np.uint32)
    est = np.zeros(n, np.uint32) if estimates else None
    bv = np.zeros((n, (m + 63) // 64), np.uint64) if bits else None
    err = L.PfError()
    ptr = lambda a: a.ctypes.data_as(C.c_void_p) if a is not None else None  # noqa: E731
    st = L.lib.pf_shouji_filter_batch(ctx.handle, ptr(text), ptr(pattern), stride, n, m, int(e),
                                      int(width), ptr(acc), ptr(est), ptr(bv), C.byref(err))
    _raise(st, err)
    return acc, est, bv


def packed_words(m: int) -> int:
    """u64 words per sequence per pair in the packed-planes layout (3 * ceil(m/64))."""
    return int(L.lib.pf_packed_words(int(m)))


def pack_planes(records, m: int | None = None) -> np.ndarray:
    """ASCII records u8[n, stride] -> packed_sequence planes u64[n, 3, ceil(m/64)]
    (low, high, N; codes A/C/G/T = 0..3, packed_sequence.cpp:16-30). Host-side
    layout helper for callers and tests; it does not validate (use
    packed_sequence.from_string or the batch entry points for that)."""
    rec = _as_records(records)
    n, stride = rec.shape
    m = stride if m is None else int(m)
    a = rec[:, :m]
    code = np.zeros(a.shape, np.uint8)
    code[a == ord("C")] = 1
    code[a == ord("G")] = 2
    code[a == ord("T")] = 3
    isn = a == ord("N")
    w = (m + 63) // 64
    out = np.zeros((n, 3, w), np.uint64)
    for k, plane in enumerate(((code & 1) == 1, (code & 2) == 2, isn)):
        bits = np.zeros((n, w * 64), np.uint8)
        bits[:, :m] = plane & ~isn if k < 2 else plane
        out[:, k, :] = np.packbits(bits.reshape(n, w, 64), axis=2, bitorder="little").view(np.uint64)[:, :, 0]
    return out


def shouji_filter_packed_batch(text_planes, pattern_planes, m: int, e: int,
                               width: int = default_window_width, estimates: bool = False,
                               bits: bool = False, ctx: Context | None = None):
    """Filter N pre-packed pairs (u64[n, 3, ceil(m/64)] each, see pack_planes)."""
    ctx = ctx or default_context()
    tp = np.ascontiguousarray(text_planes, np.uint64)
    pp = np.ascontiguousarray(pattern_planes, np.uint64)
    n = tp.shape[0]
    if tp.shape != pp.shape or tp.size != n * packed_words(m):
        raise length_mismatch_error("plane arrays must both be [n, 3, ceil(m/64)]")
    acc = np.zeros((n + 31) // 32, np.uint32)
    est = np.zeros(n, np.uint32) if estimates else None
    bv = np.zeros((n, (m + 63) // 64), np.uint64) if bits else None
    err = L.PfError()
    ptr = lambda a: a.ctypes.data_as(C.c_void_p) if a is not None else None  # noqa: E731
    st = L.lib.pf_shouji_filter_packed_batch(ctx.handle, ptr(tp), ptr(pp), n, int(m), int(e),
                                             int(width), ptr(acc), ptr(est), ptr(bv), C.byref(err))
    _raise(st, err)
    return acc, est, bv


def shouji_filter_packed_device(d_text_planes: int, d_pattern_planes: int, n: int, m: int, e: int,
                                d_accept: int, width: int = default_window_width,
                                d_estimates: int | None = None, d_bits: int | None = None,
                                stream: int | None = None, ctx: Context | None = None) -> None:
    """Pre-packed planes already on the device (raw pointers)."""
    ctx = ctx or default_context()
    err = L.PfError()
    st = L.lib.pf_shouji_filter_packed_device(ctx.handle, d_text_planes, d_pattern_planes, n, m,
                                              int(e), int(width), d_accept, d_estimates, d_bits,
                                              stream, C.byref(err))
    _raise(st, err)


def magnet_filter_batch(text, pattern, e: int, m: int | None = None, estimates: bool = False,
                        bits: bool = False, ctx: Context | None = None):
    """MAGNET over N pairs of host ASCII records (same layout and returns as
    shouji_filter_batch)."""
    ctx = ctx or default_context()
    text = _as_records(text)
    pattern = _as_records(pattern)
    if text.shape != pattern.shape:
        raise length_mismatch_error("text and pattern record arrays differ in shape")
    n, stride = text.shape
    m = stride if m is None else int(m)
    acc = np.zeros((n + 31) // 32, np.uint32)
    est = np.zeros(n, np.uint32) if estimates else None
    bv = np.zeros((n, (m + 63) // 64), np.uint64) if bits else None
    err = L.PfError()
    ptr = lambda a: a.ctypes.data_as(C.c_void_p) if a is not None else None  # noqa: E731
    st = L.lib.pf_magnet_filter_batch(ctx.handle, ptr(text), ptr(pattern), stride, n, m, int(e),
                                      ptr(acc), ptr(est), ptr(bv), C.byref(err))
    _raise(st, err)
    return acc, est, bv


def magnet_filter_device(d_text: int, d_pattern: int, pitch: int, n: int, m: int, e: int,
                         d_accept: int, d_estimates: int | None = None, d_bits: int | None = None,
                         stream: int | None = None, ctx: Context | None = None) -> None:
    """MAGNET over device-resident records (raw device pointers)."""
    ctx = ctx or default_context()
    err = L.PfError()
    st = L.lib.pf_magnet_filter_device(ctx.handle, d_text, d_pattern, pitch, n, m, int(e), d_accept,
                                       d_estimates, d_bits, stream, C.byref(err))
    _raise(st, err)


def shouji_filter_device(d_text: int, d_pattern: int, pitch: int, n: int, m: int, e: int,
                         d_accept: int, width: int = default_window_width, d_estimates: int | None = None,
                         d_bits: int | None = None, stream: int | None = None,
                         ctx: Context | None = None) -> None:
    """Device-resident batch (raw device pointers, e.g. torch ``data_ptr()``)."""
    ctx = ctx or default_context()
    err = L.PfError()
    st = L.lib.pf_shouji_filter_device(ctx.handle, d_text, d_pattern, pitch, n, m, int(e), int(width),
                                       d_accept, d_estimates, d_bits, stream, C.byref(err))
    _raise(st, err)


def generate_device(kind: int, seed: int, param: int, d_text: int, d_pattern: int, pitch: int,
                    n: int, m: int, stream: int | None = None, ctx: Context | None = None) -> None:
    """Seeded synthetic pairs for BASELINE configs 1-4, written on the device."""
    ctx = ctx or default_context()
    _raise(L.lib.pf_generate_device(ctx.handle, kind, seed, param, d_text, d_pattern, pitch, n, m,
                                    stream))


def unpack_bitmap(bitmap: np.ndarray, n: int) -> np.ndarray:
    """LSB-first u32 bitmap -> bool[n]."""
    b = np.unpackbits(np.ascontiguousarray(bitmap, np.uint32).view(np.uint8), bitorder="little")
    return b[:n].astype(bool)


def shouji_filter_device_async(d_text: int, d_pattern: int, pitch: int, n: int, m: int, e: int,
                               d_accept: int, d_err_flag: int, width: int = default_window_width,
                               d_estimates: int | None = None, stream: int | None = None,
                               ctx: Context | None = None) -> None:
    """Asynchronous device-resident batch: no host sync; illegal bytes only set *d_err_flag."""
    ctx = ctx or default_context()
    _raise(L.lib.pf_shouji_filter_device_async(ctx.handle, d_text, d_pattern, pitch, n, m, int(e),
                                               int(width), d_accept, d_estimates, d_err_flag, stream))


def nibble_pitch(m: int) -> int:
    """Bytes per nibble record of length m (4 * ceil(m / 8))."""
    return int(L.lib.pf_nibble_pitch(int(m)))


def host_pack_nibbles(text, pattern, m: int | None = None, simd: bool = True):
    """Upload stage on the host's cores: ASCII records -> nibble records
    (u8[n, nibble_pitch(m)] each), validated like packed_sequence::from_string."""
    text = _as_records(text)
    pattern = _as_records(pattern)
    if text.shape != pattern.shape:
        raise length_mismatch_error("text and pattern record arrays differ in shape")
    n, stride = text.shape
    m = stride if m is None else int(m)
    npitch = nibble_pitch(m)
    ot = np.zeros((n, npitch), np.uint8)
    op = np.zeros((n, npitch), np.uint8)
    err = L.PfError()
    ptr = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    st = L.lib.pf_host_pack_nibbles(ptr(text), ptr(pattern), stride, n, m, ptr(ot), ptr(op),
                                    1 if simd else 0, C.byref(err))
    _raise(st, err)
    return ot, op


def dibit_pitch(m: int) -> int:
    """Bytes per dibit record of length m (4 * ceil(m / 16))."""
    return int(L.lib.pf_dibit_pitch(int(m)))


def nplane_pitch(m: int) -> int:
    """Bytes per N-plane record of length m (4 * ceil(m / 32))."""
    return int(L.lib.pf_nplane_pitch(int(m)))


def host_pack_dibits(text, pattern, m: int | None = None, simd: bool = True):
    """Host upload stage in the default format: ASCII records -> dibit records and
    N-plane records (the latter None when no base is N), validated like
    packed_sequence::from_string. Returns (dib_text, dib_pattern, n_text, n_pattern)."""
    text = _as_records(text)
    pattern = _as_records(pattern)
    if text.shape != pattern.shape:
        raise length_mismatch_error("text and pattern record arrays differ in shape")
    n, stride = text.shape
    m = stride if m is None else int(m)
    dt = np.zeros((n, dibit_pitch(m)), np.uint8)
    dq = np.zeros((n, dibit_pitch(m)), np.uint8)
    nt = np.zeros((n, nplane_pitch(m)), np.uint8)
    nq = np.zeros((n, nplane_pitch(m)), np.uint8)
    has_n = C.c_int()
    err = L.PfError()
    ptr = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    st = L.lib.pf_host_pack_dibits(ptr(text), ptr(pattern), stride, n, m, ptr(dt), ptr(dq), ptr(nt),
                                   ptr(nq), C.byref(has_n), 1 if simd else 0, C.byref(err))
    _raise(st, err)
    return (dt, dq, nt, nq) if has_n.value else (dt, dq, None, None)


def shouji_filter_dibits_device(d_text: int, d_pattern: int, n: int, m: int, e: int,
                                d_accept: int, d_ntext: int | None = None,
                                d_npattern: int | None = None, width: int = default_window_width,
                                d_estimates: int | None = None, stream: int | None = None,
                                ctx: Context | None = None) -> None:
    """Filter dibit records (+ optional N-plane records) already on the device."""
    ctx = ctx or default_context()
    err = L.PfError()
    st = L.lib.pf_shouji_filter_dibits_device(ctx.handle, d_text, d_pattern, d_ntext, d_npattern,
                                              n, m, int(e), int(width), d_accept, d_estimates,
                                              stream, C.byref(err))
    _raise(st, err)


def shouji_filter_nibbles_device(d_text: int, d_pattern: int, n: int, m: int, e: int,
                                 d_accept: int, width: int = default_window_width,
                                 d_estimates: int | None = None, stream: int | None = None,
                                 ctx: Context | None = None) -> None:
    """Filter nibble records already on the device (rows of nibble_pitch(m) bytes)."""
    ctx = ctx or default_context()
    err = L.PfError()
    st = L.lib.pf_shouji_filter_nibbles_device(ctx.handle, d_text, d_pattern, n, m, int(e),
                                               int(width), d_accept, d_estimates, stream,
                                               C.byref(err))
    _raise(st, err)


def profile_stages(d_text: int, d_pattern: int, pitch: int, n: int, m: int, e: int, d_accept: int,
                   d_err_flag: int, width: int = default_window_width, reps: int = 3,
                   ctx: Context | None = None) -> tuple[float, float]:
    """(pack ms, search ms) of the device path, timed per stage with CUDA events."""
    ctx = ctx or default_context()
    pk, se = C.c_float(), C.c_float()
    _raise(L.lib.pf_shouji_profile_stages(ctx.handle, d_text, d_pattern, pitch, n, m, int(e),
                                          int(width), d_accept, d_err_flag, int(reps), C.byref(pk),
                                          C.byref(se)))
    return float(pk.value), float(se.value)


def int_peak(op: str = "lop3", ctx: Context | None = None) -> float:
    """Measured integer lane-ops/s of one instruction class on the ctx's device."""
    ctx = ctx or default_context()
    code = {"lop3": 0, "shf": 1, "prmt": 2, "imad": 3}[op]
    out = C.c_double()
    _raise(L.lib.pf_int_peak(ctx.handle, code, C.byref(out)))
    return out.value


# ---------------------------------------------------------------------------
# Exact alignment oracle on the GPU (edit_distance.hpp:13-20)
# ---------------------------------------------------------------------------
def banded_edit_distance_batch(text, pattern, e: int, m: int | None = None,
                               ctx: Context | None = None) -> np.ndarray:
    """banded_edit_distance(pattern[i], text[i], e) for every pair: int32, -1 = out of band."""
    ctx = ctx or default_context()
    text = _as_records(text)
    pattern = _as_records(pattern)
    n, stride = text.shape
    m = stride if m is None else int(m)
    out = np.zeros(n, np.int32)
    err = L.PfError()
    st = L.lib.pf_banded_edit_distance_batch(ctx.handle, text.ctypes.data_as(C.c_void_p),
                                             pattern.ctypes.data_as(C.c_void_p), stride, n, m,
                                             int(e), out.ctypes.data_as(C.c_void_p), C.byref(err))
    _raise(st, err)
    return out


def banded_edit_distance(a: packed_sequence, b: packed_sequence, e: int, ctx: Context | None = None):
    """Distance if <= e else None (edit_distance.cpp:26-70); lengths must match."""
    if a.size() != b.size():
        raise length_mismatch_error(f"length mismatch: {a.size()} vs {b.size()}")
    d = banded_edit_distance_batch(np.frombuffer(b.ascii(), np.uint8)[None, :],
                                   np.frombuffer(a.ascii(), np.uint8)[None, :], e, ctx=ctx)[0]
    return None if d < 0 else int(d)


# ---------------------------------------------------------------------------
# Pair datasets (dataset.hpp:13-58): TSV ingest with GPU validation, generator
# ---------------------------------------------------------------------------
class pair_dataset:
    """n equal-length pairs as fixed-stride ASCII records (pinned host memory)."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle

    def __len__(self):
        return int(L.lib.pf_dataset_size(self._h))

    @property
    def length(self) -> int:
        return int(L.lib.pf_dataset_length(self._h))

    @property
    def source(self) -> str:
        return L.lib.pf_dataset_source(self._h).decode()

    def _view(self, fn):
        n, m = len(self), self.length
        ptr = fn(self._h)
        if not n:
            return np.zeros((0, m), np.uint8)
        buf = (C.c_uint8 * (n * m)).from_address(ptr)
        return np.frombuffer(buf, np.uint8).reshape(n, m)

    def text(self) -> np.ndarray:
        return self._view(L.lib.pf_dataset_text)

    def pattern(self) -> np.ndarray:
        return self._view(L.lib.pf_dataset_pattern)

    def filter(self, e: int, width: int = default_window_width, estimates: bool = False,
               ctx: Context | None = None):
        return shouji_filter_batch(self.text(), self.pattern(), e, width, estimates=estimates, ctx=ctx)

    def write(self, path: str) -> None:
        if L.lib.pf_dataset_write_tsv(self._h, path.encode()) != L.PF_OK:
            raise error(f"cannot open output file: {path}")

    def close(self):
        if self._h:
            L.lib.pf_dataset_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def load_pairs(data, source_name: str = "<stream>", ctx: Context | None = None) -> pair_dataset:
    """load_pairs (dataset.cpp:13-44) over bytes/str; parse_error(line) semantics."""
    ctx = ctx or default_context()
    b = data.encode() if isinstance(data, str) else bytes(data)
    h = C.c_void_p()
    err = L.PfError()
    _raise(L.lib.pf_dataset_load_tsv(ctx.handle, b, len(b), source_name.encode(), C.byref(h),
                                     C.byref(err)), err)
    return pair_dataset(h)


def load_pairs_file(path: str, ctx: Context | None = None) -> pair_dataset:
    ctx = ctx or default_context()
    h = C.c_void_p()
    err = L.PfError()
    _raise(L.lib.pf_dataset_load_tsv_file(ctx.handle, path.encode(), C.byref(h), C.byref(err)), err)
    return pair_dataset(h)


def generate_pairs(seed: int, count: int, length: int, lo: int, hi: int) -> pair_dataset:
    """generate_pairs({seed, count, length, {lo, hi}}) — byte-identical to the reference."""
    h = C.c_void_p()
    err = L.PfError()
    _raise(L.lib.pf_dataset_generate(seed, count, length, lo, hi, C.byref(h), C.byref(err)), err)
    return pair_dataset(h)


def write_pairs(ds: pair_dataset, path: str) -> None:
    ds.write(path)
