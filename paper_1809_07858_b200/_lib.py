"""ctypes binding of the C ABI (include/shouji_b200.h) -> libshouji_b200.so.

The shared library is the product: every filter call runs the sm_100a kernels it
contains. If the library is missing this module raises at import time — there is
no Python or CPU fallback to silently take over.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# PF_LIB_PATH: load another build of the same ABI (A/B experiments)
LIB_PATH = os.environ.get("PF_LIB_PATH") or os.path.join(_HERE, "libshouji_b200.so")

PF_OK = 0
PF_ERR_EMPTY_SEQUENCE = 1
PF_ERR_ILLEGAL_CHARACTER = 2
PF_ERR_LENGTH_MISMATCH = 3
PF_ERR_THRESHOLD_TOO_LARGE = 4
PF_ERR_OUT_OF_BAND = 5
PF_ERR_PARSE = 6
PF_ERR_INVALID_PARAMETERS = 7
PF_ERR_NO_DEVICE = 100
PF_ERR_CUDA = 101
PF_ERR_OUT_OF_MEMORY = 102
PF_ERR_NULL_ARGUMENT = 103

# Every symbol include/shouji_b200.h declares (checked by tests/test_capi_symbols.py).
EXPORTED = [
    "pf_status_string", "pf_version", "pf_device_count", "pf_ctx_create", "pf_ctx_destroy",
    "pf_ctx_device_count", "pf_shouji_filter_batch", "pf_shouji_filter_device", "pf_device_pitch",
    "pf_shouji_filter_one", "pf_host_alloc", "pf_host_free", "pf_generate_device", "pf_launch_count",
    "pf_shouji_filter_device_async", "pf_int_peak",
    "pf_dataset_load_tsv", "pf_dataset_load_tsv_file", "pf_dataset_generate", "pf_dataset_from_records",
    "pf_dataset_size", "pf_dataset_length", "pf_dataset_text", "pf_dataset_pattern",
    "pf_dataset_source", "pf_dataset_write_tsv", "pf_dataset_free", "pf_banded_edit_distance_batch",
    "pf_nibble_pitch", "pf_host_pack_nibbles", "pf_shouji_filter_nibbles_device",
    "pf_transfer_bytes", "pf_dibit_pitch", "pf_nplane_pitch", "pf_host_pack_dibits",
    "pf_shouji_filter_dibits_device", "pf_shouji_profile_stages", "pf_magnet_filter_batch", "pf_magnet_filter_device",
    "pf_magnet_filter_one", "pf_packed_words", "pf_shouji_filter_packed_batch",
    "pf_shouji_filter_packed_device", "pf_host_read_bandwidth", "pf_ctx_set_shard_chunk",
]


class PfError(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("field", C.c_uint32),
        ("pair", C.c_uint64),
        ("position", C.c_uint64),
        ("byte", C.c_uint32),
        ("cuda_error", C.c_int32),
        ("line", C.c_uint64),
        ("message", C.c_char * 160),
    ]


_vp = C.c_void_p
_sz = C.c_size_t
_u32 = C.c_uint32


def _bind(lib):
    sig = {
        "pf_status_string": (C.c_char_p, [C.c_int]),
        "pf_version": (C.c_char_p, []),
        "pf_device_count": (C.c_int, []),
        "pf_ctx_create": (C.c_int, [C.POINTER(C.c_int), C.c_int, C.POINTER(_vp)]),
        "pf_ctx_destroy": (None, [_vp]),
        "pf_ctx_device_count": (C.c_int, [_vp]),
        "pf_shouji_filter_batch": (C.c_int, [_vp, _vp, _vp, _sz, _sz, _u32, _u32, _u32, _vp, _vp,
                                             _vp, C.POINTER(PfError)]),
        "pf_shouji_filter_device": (C.c_int, [_vp, _vp, _vp, _sz, _sz, _u32, _u32, _u32, _vp, _vp,
                                              _vp, _vp, C.POINTER(PfError)]),
        "pf_device_pitch": (_sz, [_u32]),
        "pf_shouji_filter_one": (C.c_int, [_vp, C.c_char_p, _sz, C.c_char_p, _sz, _u32, _u32,
                                           C.POINTER(C.c_int), C.POINTER(_u32), _vp,
                                           C.POINTER(PfError)]),
        "pf_host_alloc": (_vp, [_sz]),
        "pf_host_free": (None, [_vp]),
        "pf_generate_device": (C.c_int, [_vp, C.c_int, C.c_uint64, _u32, _vp, _vp, _sz, _sz, _u32,
                                         _vp]),
        "pf_launch_count": (C.c_uint64, []),
        "pf_shouji_filter_device_async": (C.c_int, [_vp, _vp, _vp, _sz, _sz, _u32, _u32, _u32, _vp,
                                                    _vp, _vp, _vp]),
        "pf_int_peak": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_double)]),
        "pf_dataset_load_tsv": (C.c_int, [_vp, C.c_char_p, _sz, C.c_char_p, C.POINTER(_vp),
                                          C.POINTER(PfError)]),
        "pf_dataset_load_tsv_file": (C.c_int, [_vp, C.c_char_p, C.POINTER(_vp), C.POINTER(PfError)]),
        "pf_dataset_generate": (C.c_int, [C.c_uint64, _sz, _u32, _u32, _u32, C.POINTER(_vp),
                                          C.POINTER(PfError)]),
        "pf_dataset_from_records": (C.c_int, [_vp, _vp, _sz, _sz, _u32, C.c_char_p, C.POINTER(_vp)]),
        "pf_dataset_size": (_sz, [_vp]),
        "pf_dataset_length": (_u32, [_vp]),
        "pf_dataset_text": (_vp, [_vp]),
        "pf_dataset_pattern": (_vp, [_vp]),
        "pf_dataset_source": (C.c_char_p, [_vp]),
        "pf_dataset_write_tsv": (C.c_int, [_vp, C.c_char_p]),
        "pf_dataset_free": (None, [_vp]),
        "pf_banded_edit_distance_batch": (C.c_int, [_vp, _vp, _vp, _sz, _sz, _u32, _u32, _vp,
                                                    C.POINTER(PfError)]),
        "pf_nibble_pitch": (_sz, [_u32]),
        "pf_dibit_pitch": (_sz, [_u32]),
        "pf_shouji_profile_stages": (C.c_int, [_vp, _vp, _vp, _sz, _sz, _u32, _u32, _u32, _vp, _vp,
                                               C.c_int, C.POINTER(C.c_float),
                                               C.POINTER(C.c_float)]),
        "pf_nplane_pitch": (_sz, [_u32]),
        "pf_host_pack_dibits": (C.c_int, [_vp, _vp, _sz, _sz, _u32, _vp, _vp, _vp, _vp,
                                          C.POINTER(C.c_int), C.c_int, C.POINTER(PfError)]),
        "pf_shouji_filter_dibits_device": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _sz, _u32, _u32,
                                                     _u32, _vp, _vp, _vp, C.POINTER(PfError)]),
        "pf_transfer_bytes": (None, [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
        "pf_host_read_bandwidth": (C.c_double, [_vp, _sz, C.c_int]),
        "pf_ctx_set_shard_chunk": (C.c_int, [_vp, _sz]),
        "pf_packed_words": (_sz, [_u32]),
        "pf_shouji_filter_packed_batch": (C.c_int, [_vp, _vp, _vp, _sz, _u32, _u32, _u32, _vp, _vp,
                                                    _vp, C.POINTER(PfError)]),
        "pf_shouji_filter_packed_device": (C.c_int, [_vp, _vp, _vp, _sz, _u32, _u32, _u32, _vp,
                                                     _vp, _vp, _vp, C.POINTER(PfError)]),
        "pf_magnet_filter_batch": (C.c_int, [_vp, _vp, _vp, _sz, _sz, _u32, _u32, _vp, _vp, _vp,
                                             C.POINTER(PfError)]),
        "pf_magnet_filter_device": (C.c_int, [_vp, _vp, _vp, _sz, _sz, _u32, _u32, _vp, _vp, _vp,
                                              _vp, C.POINTER(PfError)]),
        "pf_magnet_filter_one": (C.c_int, [_vp, C.c_char_p, _sz, C.c_char_p, _sz, _u32,
                                           C.POINTER(C.c_int), C.POINTER(_u32), _vp,
                                           C.POINTER(PfError)]),
        "pf_host_pack_nibbles": (C.c_int, [_vp, _vp, _sz, _sz, _u32, _vp, _vp, C.c_int,
                                           C.POINTER(PfError)]),
        "pf_shouji_filter_nibbles_device": (C.c_int, [_vp, _vp, _vp, _sz, _u32, _u32, _u32, _vp,
                                                      _vp, _vp, C.POINTER(PfError)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def load(path: str = LIB_PATH):
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build the sm_100a extension first "
            "(python paper_1809_07858_b200/build.py or __graft_entry__.build()). "
            "There is no CPU fallback.")
    return _bind(C.CDLL(path))


lib = load()
