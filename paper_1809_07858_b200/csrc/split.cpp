// SM-partitioned pack | search pipeline (device-resident ASCII records).
//
// The filter step is an HBM-bound pack (records -> pair-sliced planes) followed
// by an ALU-bound search. Run back to back over the whole batch, each stage
// leaves the other's resource idle (ncu: pack 72% DRAM / 50% ALU, search 15% DRAM
// / 86% ALU). Here the device's SMs are split into two green contexts — a pack
// partition and a search partition — and the batch is cut into chunks: while
// the search partition works on chunk i, the pack partition already streams
// chunk i+1's records into the second plane buffer. Each partition has two
// streams (chunk parity) so the next chunk's CTAs fill the tail of the previous
// chunk's launch. Events order every reuse of a plane buffer, and the caller's
// stream waits for the last search, so the call is stream-ordered like the
// serial path. The kernels are the serial path's kernels (launch_filter_stage),
// run on chunk-local views of the records, bitmap and estimates.
//
// Green contexts come from the driver API (cuDevSmResourceSplitByCount,
// cuGreenCtxCreate, cuGreenCtxStreamCreate), reached through
// cudaGetDriverEntryPoint so the library does not link libcuda directly.
#include "split.h"

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "kernels.cuh"
#include "pack.cuh"

namespace sb {

namespace {

struct Driver {
    CUresult (*deviceGet)(CUdevice*, int) = nullptr;
    CUresult (*getDevResource)(CUdevice, CUdevResource*, CUdevResourceType) = nullptr;
    CUresult (*split)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned,
                      unsigned) = nullptr;
    CUresult (*genDesc)(CUdevResourceDesc*, CUdevResource*, unsigned) = nullptr;
    CUresult (*greenCreate)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned) = nullptr;
    CUresult (*greenDestroy)(CUgreenCtx) = nullptr;
    CUresult (*greenStream)(CUstream*, CUgreenCtx, unsigned, int) = nullptr;
    bool ok = false;
};

template <typename F>
bool entry(const char* name, F& fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p) {
        cudaGetLastError();
        return false;
    }
    fn = reinterpret_cast<F>(p);
    return true;
}

const Driver& driver() {
    static const Driver d = [] {
        Driver x;
        x.ok = entry("cuDeviceGet", x.deviceGet) &&
               entry("cuDeviceGetDevResource", x.getDevResource) &&
               entry("cuDevSmResourceSplitByCount", x.split) &&
               entry("cuDevResourceGenerateDesc", x.genDesc) &&
               entry("cuGreenCtxCreate", x.greenCreate) &&
               entry("cuGreenCtxDestroy", x.greenDestroy) &&
               entry("cuGreenCtxStreamCreate", x.greenStream);
        return x;
    }();
    return d;
}

}  // namespace

// Shared mode (pack_sms < 0): no partition — one pack stream (chunks packed
// one after another) and two search streams on the whole device, the pack
// stream at the higher priority, and a ring of kRing plane buffers, so the
// block scheduler can place pack CTAs (shared-memory bound) and search CTAs
// (register bound) on the same SMs.
constexpr int kRing = 3;

struct SplitPipe {
    int device = 0;
    bool shared = false;
    int nbuf = 2;
    CUgreenCtx green[2] = {nullptr, nullptr};  // 0 pack, 1 search
    cudaStream_t ps[kRing] = {nullptr, nullptr, nullptr};  // pack streams (by buffer)
    cudaStream_t ss[kRing] = {nullptr, nullptr, nullptr};  // search streams
    cudaEvent_t in_ev = nullptr;
    cudaEvent_t packed[kRing] = {nullptr, nullptr, nullptr};
    cudaEvent_t searched[kRing] = {nullptr, nullptr, nullptr};
    bool searched_valid[kRing] = {false, false, false};
    uint32_t* planes[kRing] = {nullptr, nullptr, nullptr};
    size_t planes_words = 0;
    int pack_sms = 0, search_sms = 0;
};

int split_pack_sms(const SplitPipe* p) { return p ? p->pack_sms : 0; }
int split_search_sms(const SplitPipe* p) { return p ? p->search_sms : 0; }

void split_destroy(SplitPipe* p) {
    if (!p) return;
    const Driver& drv = driver();
    for (int b = 0; b < kRing; ++b) {
        if (p->ps[b]) cudaStreamSynchronize(p->ps[b]);
        if (p->ss[b]) cudaStreamSynchronize(p->ss[b]);
    }
    for (int b = 0; b < kRing; ++b) {
        if (p->packed[b]) cudaEventDestroy(p->packed[b]);
        if (p->searched[b]) cudaEventDestroy(p->searched[b]);
        cudaFree(p->planes[b]);
        // shared mode aliases streams across buffers: destroy each once
        bool first_ps = true, first_ss = true;
        for (int c = 0; c < b; ++c) {
            if (p->ps[c] == p->ps[b]) first_ps = false;
            if (p->ss[c] == p->ss[b]) first_ss = false;
        }
        if (p->ps[b] && first_ps) cudaStreamDestroy(p->ps[b]);
        if (p->ss[b] && first_ss) cudaStreamDestroy(p->ss[b]);
    }
    if (p->in_ev) cudaEventDestroy(p->in_ev);
    for (auto g : p->green)
        if (g && drv.greenDestroy) drv.greenDestroy(g);
    delete p;
}

SplitPipe* split_create(int device, int pack_sms, std::string* why) {
    const Driver& drv = driver();
    auto fail = [&](const char* msg, SplitPipe* p) -> SplitPipe* {
        if (why) *why = msg;
        split_destroy(p);
        return nullptr;
    };
    if (pack_sms < 0) {  // shared mode: plain priority streams on the whole device
        auto* p = new SplitPipe;
        p->device = device;
        p->shared = true;
        const char* nb = std::getenv("PF_SPLIT_BUFS");
        p->nbuf = nb && std::atoi(nb) == 2 ? 2 : kRing;
        int lo = 0, hi = 0;  // numerically: lo = least priority, hi = greatest
        if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) return fail("priority range", p);
        const char* pr = std::getenv("PF_SPLIT_PRIO");  // "search": search streams first
        const bool search_first = pr && std::strcmp(pr, "search") == 0;
        const int pp = search_first ? lo : hi, sp = search_first ? hi : lo;
        cudaStream_t pack = nullptr, srch[2] = {nullptr, nullptr};
        if (cudaStreamCreateWithPriority(&pack, cudaStreamNonBlocking, pp) != cudaSuccess)
            return fail("cudaStreamCreateWithPriority", p);
        for (int b = 0; b < kRing; ++b) p->ps[b] = pack;
        for (int k = 0; k < 2; ++k)
            if (cudaStreamCreateWithPriority(&srch[k], cudaStreamNonBlocking, sp) != cudaSuccess)
                return fail("cudaStreamCreateWithPriority", p);
        for (int b = 0; b < kRing; ++b) p->ss[b] = srch[b & 1];
        for (int b = 0; b < kRing; ++b)
            if (cudaEventCreateWithFlags(&p->packed[b], cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&p->searched[b], cudaEventDisableTiming) != cudaSuccess)
                return fail("cudaEventCreate", p);
        if (cudaEventCreateWithFlags(&p->in_ev, cudaEventDisableTiming) != cudaSuccess)
            return fail("cudaEventCreate", p);
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        p->pack_sms = p->search_sms = sms;
        return p;
    }
    if (!drv.ok) return fail("green-context driver entry points unavailable", nullptr);
    auto* p = new SplitPipe;
    p->device = device;
    CUdevice dev;
    if (drv.deviceGet(&dev, device) != CUDA_SUCCESS) return fail("cuDeviceGet", p);
    CUdevResource all{}, part{}, rest{};
    if (drv.getDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS)
        return fail("cuDeviceGetDevResource", p);
    unsigned groups = 1;
    if (drv.split(&part, &groups, &all, &rest, 0, static_cast<unsigned>(pack_sms)) !=
            CUDA_SUCCESS ||
        groups != 1 || rest.sm.smCount == 0)
        return fail("cuDevSmResourceSplitByCount", p);
    p->pack_sms = static_cast<int>(part.sm.smCount);
    p->search_sms = static_cast<int>(rest.sm.smCount);
    CUdevResource* res[2] = {&part, &rest};
    for (int k = 0; k < 2; ++k) {
        CUdevResourceDesc desc;
        if (drv.genDesc(&desc, res[k], 1) != CUDA_SUCCESS) return fail("cuDevResourceGenerateDesc", p);
        if (drv.greenCreate(&p->green[k], desc, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS)
            return fail("cuGreenCtxCreate", p);
    }
    for (int b = 0; b < 2; ++b) {
        CUstream a, c;
        if (drv.greenStream(&a, p->green[0], CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS ||
            drv.greenStream(&c, p->green[1], CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS)
            return fail("cuGreenCtxStreamCreate", p);
        p->ps[b] = reinterpret_cast<cudaStream_t>(a);
        p->ss[b] = reinterpret_cast<cudaStream_t>(c);
        if (cudaEventCreateWithFlags(&p->packed[b], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&p->searched[b], cudaEventDisableTiming) != cudaSuccess)
            return fail("cudaEventCreate", p);
    }
    if (cudaEventCreateWithFlags(&p->in_ev, cudaEventDisableTiming) != cudaSuccess)
        return fail("cudaEventCreate", p);
    return p;
}

cudaError_t split_launch(SplitPipe* p, const FilterArgs& a, cudaStream_t s, long long chunk) {
    chunk = (chunk + 4095) / 4096 * 4096;  // whole search CTAs (4096 pairs) and bitmap words
    const size_t words = planes_scratch_words(chunk, a.m);
    const int nbuf = p->nbuf;
    if (words > p->planes_words) {
        for (int b = 0; b < nbuf; ++b) {
            if (p->searched_valid[b]) {
                const cudaError_t st = cudaEventSynchronize(p->searched[b]);
                if (st != cudaSuccess) return st;
            }
            cudaFree(p->planes[b]);
            p->planes[b] = nullptr;
        }
        p->planes_words = 0;
        for (int b = 0; b < nbuf; ++b) {
            const cudaError_t st = cudaMalloc(&p->planes[b], words * sizeof(uint32_t));
            if (st != cudaSuccess) return st;
        }
        p->planes_words = words;
    }
    cudaError_t st = cudaEventRecord(p->in_ev, s);  // inputs (and outputs) ready on s
    if (st != cudaSuccess) return st;
    for (int b = 0; b < nbuf; ++b) {
        if ((st = cudaStreamWaitEvent(p->ps[b], p->in_ev, 0)) != cudaSuccess) return st;
        if ((st = cudaStreamWaitEvent(p->ss[b], p->in_ev, 0)) != cudaSuccess) return st;
    }
    bool used[kRing] = {false, false, false};
    long long i = 0;
    for (long long p0 = 0; p0 < a.n; p0 += chunk, ++i) {
        const int b = static_cast<int>(i % nbuf);
        FilterArgs c = a;
        c.n = std::min<long long>(chunk, a.n - p0);
        c.text = a.text + static_cast<size_t>(p0) * a.pitch;
        c.pattern = a.pattern + static_cast<size_t>(p0) * a.pitch;
        c.accept = a.accept + p0 / 32;
        c.estimates = a.estimates ? a.estimates + p0 : nullptr;
        c.planes = p->planes[b];
        c.planes_words = p->planes_words;
        // plane buffer b is free once the search that last read it is done
        if (p->searched_valid[b] &&
            (st = cudaStreamWaitEvent(p->ps[b], p->searched[b], 0)) != cudaSuccess)
            return st;
        if ((st = launch_filter_stage(c, p->ps[b], 1)) != cudaSuccess) return st;
        if ((st = cudaEventRecord(p->packed[b], p->ps[b])) != cudaSuccess) return st;
        if ((st = cudaStreamWaitEvent(p->ss[b], p->packed[b], 0)) != cudaSuccess) return st;
        if ((st = launch_filter_stage(c, p->ss[b], 2)) != cudaSuccess) return st;
        if ((st = cudaEventRecord(p->searched[b], p->ss[b])) != cudaSuccess) return st;
        p->searched_valid[b] = true;
        used[b] = true;
    }
    for (int b = 0; b < nbuf; ++b)
        if (used[b] && (st = cudaStreamWaitEvent(s, p->searched[b], 0)) != cudaSuccess) return st;
    return cudaSuccess;
}

}  // namespace sb
