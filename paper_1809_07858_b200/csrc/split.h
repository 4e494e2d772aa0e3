// SM-partitioned pack | search pipeline (split.cpp). Internal; not part of the ABI.
#pragma once
#include <string>

#include <cuda_runtime.h>

#include "kernels.cuh"

namespace sb {

struct SplitPipe;

// Green contexts of pack_sms (rounded up by the driver to its SM granularity)
// and the remaining SMs of `device` (which must be current), their streams and
// events. nullptr (with *why) when the driver cannot partition the device.
SplitPipe* split_create(int device, int pack_sms, std::string* why);
void split_destroy(SplitPipe* p);
int split_pack_sms(const SplitPipe* p);
int split_search_sms(const SplitPipe* p);

// The filter over device-resident ASCII records `a` (a.planes unused: the pipe
// owns two chunk-sized plane buffers), chunk by chunk, pack and search
// overlapped on disjoint SMs; ordered after prior work on `s`, and `s` waits
// for its completion.
cudaError_t split_launch(SplitPipe* p, const FilterArgs& a, cudaStream_t s, long long chunk);

}  // namespace sb
