"""Guard-page buffers for out-of-bounds checks without compute-sanitizer
(closed on this pool): an array placed so that it ENDS (or starts) exactly at
a page boundary with an inaccessible page beyond it, so that any read or write
past the end (or before the start) faults instead of silently passing.

* host_guarded(nbytes)    — anonymous mmap, the next page mprotect(PROT_NONE)
  (a fault kills the test process: the suite fails loudly);
* DeviceGuarded(nbytes)   — CUDA virtual memory: physical memory mapped right
  before an unmapped 2 MiB range (a kernel read/write past the end raises
  cudaErrorIllegalAddress).
"""
import ctypes
import mmap

import numpy as np

_libc = ctypes.CDLL(None, use_errno=True)
_libc.mprotect.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
_keep = []


def host_guarded(nbytes: int, at_end: bool = True, align: int = 1) -> np.ndarray:
    """u8[nbytes] whose last byte is the last accessible byte before a PROT_NONE page
    (at_end=True), or whose first byte follows a PROT_NONE page (at_end=False)."""
    page = mmap.PAGESIZE
    body = (nbytes + page - 1) // page * page
    mm = mmap.mmap(-1, body + 2 * page, prot=mmap.PROT_READ | mmap.PROT_WRITE)
    base = ctypes.addressof(ctypes.c_char.from_buffer(mm))
    assert _libc.mprotect(base, page, 0) == 0
    assert _libc.mprotect(base + page + body, page, 0) == 0
    if at_end:
        off = page + body - (nbytes + align - 1) // align * align
    else:
        off = page
    _keep.append(mm)
    return np.frombuffer(mm, dtype=np.uint8, count=nbytes, offset=off)


class DeviceGuarded:
    """nbytes of device memory ending (at_end) or starting exactly at the edge of a
    mapped VMM range, with unmapped address space on both sides. ptr is 16-byte
    aligned (at_end: the array ends within 15 bytes of the edge when nbytes % 16)."""

    def __init__(self, nbytes: int, device: int = 0, at_end: bool = True):
        from cuda.bindings import driver as d
        self.d = d
        (err,) = d.cuInit(0)
        _ck(err)
        # the device's primary context (the one the CUDA runtime and the library use),
        # current on this thread for the driver calls below
        err, dev = d.cuDeviceGet(device)
        _ck(err)
        err, pctx = d.cuDevicePrimaryCtxRetain(dev)
        _ck(err)
        (err,) = d.cuCtxSetCurrent(pctx)
        _ck(err)
        prop = d.CUmemAllocationProp()
        prop.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        prop.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        prop.location.id = device
        err, gran = d.cuMemGetAllocationGranularity(
            prop, d.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM)
        _ck(err)
        self.size = max(gran, (nbytes + gran - 1) // gran * gran)
        err, self.va = d.cuMemAddressReserve(self.size + 2 * gran, 0, 0, 0)
        _ck(err)
        err, self.handle = d.cuMemCreate(self.size, prop, 0)
        _ck(err)
        self.base = int(self.va) + gran
        (err,) = d.cuMemMap(self.base, self.size, 0, self.handle, 0)
        _ck(err)
        acc = d.CUmemAccessDesc()
        acc.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = device
        acc.flags = d.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        (err,) = d.cuMemSetAccess(self.base, self.size, [acc], 1)
        _ck(err)
        self.gran = gran
        self.ptr = (self.base + self.size - (nbytes + 15) // 16 * 16) if at_end else self.base
        self.nbytes = nbytes

    def upload(self, arr: np.ndarray):
        a = np.ascontiguousarray(arr)
        assert a.nbytes == self.nbytes
        (err,) = self.d.cuMemcpyHtoD(self.ptr, a.ctypes.data, a.nbytes)
        _ck(err)

    def download(self, dtype, shape):
        out = np.empty(shape, dtype)
        assert out.nbytes == self.nbytes
        (err,) = self.d.cuMemcpyDtoH(out.ctypes.data, self.ptr, out.nbytes)
        _ck(err)
        return out

    def fill(self, byte: int):
        (err,) = self.d.cuMemsetD8(self.ptr, byte, self.nbytes)
        _ck(err)

    def free(self):
        d = self.d
        d.cuMemUnmap(self.base, self.size)
        d.cuMemRelease(self.handle)
        d.cuMemAddressFree(self.va, self.size + 2 * self.gran)


def _ck(err):
    from cuda.bindings import driver as d
    if err != d.CUresult.CUDA_SUCCESS:
        raise RuntimeError(f"CUDA driver error {err}")
