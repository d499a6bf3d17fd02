// mgaq_batch.cu -- one launch for all the MGAQ quantizations of a decoder
// layer (the saved activations of FlowCtx::save_nonlinear / save_linear,
// flow.cpp:450-480).
//
// Per-item semantics are exactly the per-tensor entry points':
//   group_size > 0: quantize(x, per_group(G), e4m3)          quantize.cpp:89-111
//   group_size = 0: group_scale_max(x, 128) -> quantize(x, per_tensor, e4m3)
//                                                           quantize.cpp:126-145
// (bit-identical codes and scales; tests/test_gpu_quant.py).
//
// Why one kernel: at B200 bandwidth a 64 MB activation streams in ~10 us, and
// each separate launch pays ~4 us of ramp-up and tail (tools/l2_probe.cu), so
// the 14 launches of a layer lose ~15% to it.  This persistent cooperative
// kernel (grid = #SMs x resident CTAs) runs
//   phase 1: every per-group tile, then the absmax pass of every per-tensor
//            item (loads marked L2::evict_last); per-CTA partial maxima to a
//            workspace;
//   grid barrier;
//   phase 2: per-tensor encode, newest item first (its lines are the ones
//            still in L2), each CTA reducing the item's partial maxima.
#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "act_quant.cuh"
#include "coat_device.cuh"
#include "coat_internal.h"

namespace coat {
namespace {

using namespace aq;
constexpr int kThreads = 256;

struct BItem {
    const void* x;
    uint8_t* codes;
    uint16_t* scales;
    uint32_t* amax_out;
    int64_t nchunks;   // 16-element chunks
    int64_t tiles;
    int32_t dtype;
    int32_t lanes;     // G / 16 for per-group, 0 for per-tensor
    int32_t lshift;    // log2(lanes)
    int32_t pad;
};

struct BParams {
    BItem it[kMgaqMaxItems];
    int32_t n;
    int32_t npt;               // per-tensor items (the last npt entries)
    int64_t tiles1;            // phase-1 tiles (all items)
    int64_t tiles2;            // phase-2 tiles (per-tensor items)
    uint32_t* partials;        // [npt][gridDim.x]
    uint32_t* barrier;         // zeroed by the launcher
    uint32_t* flags;
};

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p);

template <int DT>
__device__ __forceinline__ uint32_t group_tile(const BItem& I, int64_t t, float nz) {
    const int64_t ch = t * kThreads + threadIdx.x;
    const bool valid = ch < I.nchunks;
    RawChunk<DT> raw;
    uint32_t am = 0;
    if (valid) {
        raw = load_raw16<DT, EV_FIRST>(I.x, ch * 16);
        am = absmax_raw<DT, false>(raw);
    }
    for (int off = 1; off < I.lanes; off <<= 1) am = max(am, __shfl_xor_sync(0xFFFFFFFFu, am, off));
    if (!valid) return 0u;
    float s, rs;
    group_scale_fast(am, s, rs);
    reinterpret_cast<uint4*>(I.codes)[ch] = encode16(widen16<DT>(raw), s, rs, nz);
    if ((threadIdx.x & (I.lanes - 1)) == 0) I.scales[ch >> I.lshift] = float_to_bf16_bits_exact(s);
    return am >= 0x7F800000u ? 1u : 0u;
}

template <int DT>
__device__ __forceinline__ uint32_t amax_tile(const BItem& I, int64_t t) {
    const int64_t ch = t * kThreads + threadIdx.x;
    return ch < I.nchunks ? absmax_raw<DT, true>(load_raw16<DT, EV_LAST>(I.x, ch * 16)) : 0u;
}

template <int DT>
__device__ __forceinline__ uint32_t encode_tile(const BItem& I, int64_t t, float s, float rs, float nz) {
    const int64_t ch = t * kThreads + threadIdx.x;
    if (ch >= I.nchunks) return 0u;
    const RawChunk<DT> raw = load_raw16<DT, EV_FIRST>(I.x, ch * 16);
    reinterpret_cast<uint4*>(I.codes)[ch] = encode16(widen16<DT>(raw), s, rs, nz);
    return absmax_raw<DT, false>(raw) >= 0x7F800000u ? 1u : 0u;
}

__global__ void __launch_bounds__(kThreads) mgaq_batch_kernel(const __grid_constant__ BParams P, float nz) {
    __shared__ uint32_t s_pmax[kMgaqMaxItems];
    __shared__ uint32_t s_red[kThreads / 32];
    __shared__ float s_scale[2];
    if (threadIdx.x < kMgaqMaxItems) s_pmax[threadIdx.x] = 0u;
    __syncthreads();
    uint32_t bad = 0;
    const int first_pt = P.n - P.npt;

    // ---------------- phase 1: per-group tiles, then per-tensor absmax tiles
    int item = 0;
    int64_t base = 0;   // first tile of `item`
    for (int64_t t = blockIdx.x; t < P.tiles1; t += gridDim.x) {
        while (t >= base + P.it[item].tiles) base += P.it[item++].tiles;   // uniform per CTA
        const BItem& I = P.it[item];
        if (I.lanes) {
            bad |= I.dtype == 0 ? group_tile<0>(I, t - base, nz) : group_tile<1>(I, t - base, nz);
        } else {
            uint32_t am = I.dtype == 0 ? amax_tile<0>(I, t - base) : amax_tile<1>(I, t - base);
            am = warp_max_u32(am);
            if ((threadIdx.x & 31) == 0 && am) atomicMax(&s_pmax[item - first_pt], am);
        }
    }
    __syncthreads();
    if (threadIdx.x < P.npt) P.partials[threadIdx.x * gridDim.x + blockIdx.x] = s_pmax[threadIdx.x];

    // ---------------- grid barrier (all CTAs are co-resident: cooperative launch)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(P.barrier, 1u);
        while (ld_acquire_u32(P.barrier) < gridDim.x) __nanosleep(64);
    }
    __syncthreads();

    // ---------------- phase 2: per-tensor encode, newest item first
    int cur = -1;
    float s = 1.0f, rs = 1.0f;
    for (int64_t t = blockIdx.x; t < P.tiles2; t += gridDim.x) {
        int j = P.n - 1;
        int64_t b2 = 0;
        while (t >= b2 + P.it[j].tiles) b2 += P.it[j--].tiles;
        if (j != cur) {   // uniform per CTA: reduce this item's partial maxima
            cur = j;
            const uint32_t* pp = P.partials + int64_t(j - first_pt) * gridDim.x;
            uint32_t m = 0;
            for (int i = threadIdx.x; i < (int)gridDim.x; i += kThreads) m = max(m, pp[i]);
            m = warp_max_u32(m);
            if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = m;
            __syncthreads();
            if (threadIdx.x == 0) {
                uint32_t a = 0;
                for (int w = 0; w < kThreads / 32; ++w) a = max(a, s_red[w]);
                const float sc = group_scale(u2f(a));
                s_scale[0] = sc;
                s_scale[1] = __frcp_rn(sc);
                if (t == b2) {   // this CTA owns the item's tile 0: publish scale and absmax
                    P.it[j].scales[0] = float_to_bf16_bits_exact(sc);
                    if (P.it[j].amax_out) *P.it[j].amax_out = a;
                }
            }
            __syncthreads();
            s = s_scale[0];
            rs = s_scale[1];
        }
        const BItem& I = P.it[j];
        bad |= I.dtype == 0 ? encode_tile<0>(I, t - b2, s, rs, nz) : encode_tile<1>(I, t - b2, s, rs, nz);
    }
    if (P.flags && __reduce_or_sync(0xFFFFFFFFu, bad) && (threadIdx.x & 31) == 0) atomicOr(P.flags, kFlagNonFiniteInput);
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

struct Workspace {
    uint32_t* buf = nullptr;
    size_t words = 0;
    int dev = -1;
};

}  // namespace

cudaError_t launch_mgaq_batch(const MgaqItem* items, int n, uint32_t* flags, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    if (n > kMgaqMaxItems) return cudaErrorInvalidValue;
    BParams P{};
    // per-group items first (phase-1 order), per-tensor items last
    int k = 0, npt = 0;
    for (int pass = 0; pass < 2; ++pass) {
        for (int i = 0; i < n; ++i) {
            const MgaqItem& m = items[i];
            const bool pt = m.group_size == 0;
            if (pt != (pass == 1)) continue;
            BItem& b = P.it[k++];
            b.x = m.x;
            b.codes = m.codes;
            b.scales = m.scales;
            b.amax_out = m.amax_out;
            b.nchunks = m.n / 16;
            b.tiles = (b.nchunks + kThreads - 1) / kThreads;
            b.dtype = m.dtype;
            b.lanes = pt ? 0 : int32_t(m.group_size / 16);
            b.lshift = 0;
            while ((1 << b.lshift) < b.lanes) ++b.lshift;
            npt += pt ? 1 : 0;
            P.tiles1 += b.tiles;
            if (pt) P.tiles2 += b.tiles;
        }
    }
    P.n = n;
    P.npt = npt;
    P.flags = flags;

    static Workspace ws;
    static std::mutex mu;
    int dev = 0;
    cudaGetDevice(&dev);
    static int per_sm = 0;
    {
        std::lock_guard<std::mutex> lock(mu);
        if (ws.dev != dev) {
            cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mgaq_batch_kernel, kThreads, 0);
            if (e != cudaSuccess) return e;
            if (ws.buf) cudaFree(ws.buf);
            ws.words = size_t(kMgaqMaxItems) * device_sm_count() * (per_sm > 0 ? per_sm : 1) + 32;
            e = cudaMalloc(&ws.buf, ws.words * sizeof(uint32_t));
            if (e != cudaSuccess) return e;
            ws.dev = dev;
        }
    }
    const int grid = device_sm_count() * (per_sm > 0 ? per_sm : 1);
    P.barrier = ws.buf;
    P.partials = ws.buf + 32;
    cudaError_t e = cudaMemsetAsync(P.barrier, 0, sizeof(uint32_t), st);
    if (e != cudaSuccess) return e;
    float nz = -0.0f;
    void* args[] = {&P, &nz};
    return cudaLaunchCooperativeKernel((void*)mgaq_batch_kernel, dim3(grid), dim3(kThreads), args, 0, st);
}

// ---------------------------------------------------------------------------
// The default schedule of coat_quantize_batch: the records are independent, so
// they are spread over 3 internal streams forked from (and joined back into)
// the caller's stream, each record run by the same kernels as its per-tensor
// entry point (quantize_per_group; group_scale_max + quantize_per_tensor), so
// the results are those of the entry points by construction.  Each per-tensor
// record's encode pass then follows its own stage-1 pass and re-reads it from
// L2, and one kernel's ramp/tail overlaps its neighbours' streaming: 0.31 ms
// for the Llama-2-7B layer vs 0.40 ms for the single cooperative launch above
// (whose phase-1-then-phase-2 order loses the L2 reuse).  Capturable into a
// CUDA graph (fork/join through events).  COAT_MGAQ_BATCH=coop selects the
// cooperative kernel.
namespace {
constexpr int kBatchStreams = 3;
struct StreamSet {
    int dev = -1;
    cudaStream_t s[kBatchStreams] = {};
    cudaEvent_t fork = nullptr, join[kBatchStreams] = {};
    uint32_t* amax_ws = nullptr;   // one Group Scaling word per record without d_amax_bits
};
}  // namespace

bool mgaq_batch_cooperative() {
    static const bool coop = [] {
        const char* e = getenv("COAT_MGAQ_BATCH");
        return e && e[0] == 'c';
    }();
    return coop;
}

cudaError_t launch_mgaq_streams(const MgaqItem* items, int n, uint32_t* flags, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    if (n > kMgaqMaxItems) return cudaErrorInvalidValue;
    static StreamSet sets[16];              // per device, created on first use
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);   // a device's stream set is shared by all callers
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 16) return cudaErrorInvalidDevice;
    StreamSet& ss = sets[dev];
    if (ss.dev != dev) {
        for (int k = 0; k < kBatchStreams; ++k) {
            if ((e = cudaStreamCreateWithFlags(&ss.s[k], cudaStreamNonBlocking)) != cudaSuccess) return e;
            if ((e = cudaEventCreateWithFlags(&ss.join[k], cudaEventDisableTiming)) != cudaSuccess) return e;
        }
        if ((e = cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming)) != cudaSuccess) return e;
        if ((e = cudaMalloc(&ss.amax_ws, kMgaqMaxItems * sizeof(uint32_t))) != cudaSuccess) return e;
        ss.dev = dev;
    }
    if ((e = cudaEventRecord(ss.fork, st)) != cudaSuccess) return e;
    for (int k = 0; k < kBatchStreams; ++k)
        if ((e = cudaStreamWaitEvent(ss.s[k], ss.fork, 0)) != cudaSuccess) return e;
    // Items round-robin over the streams.  (Measured round 2: all per-tensor
    // items on one stream -- one L2-resident tensor at a time -- cuts the
    // layer's DRAM traffic from 1.17x to 1.12x the algorithmic bytes but
    // serialises 8 short kernels: 0.330 vs 0.318 ms.)
    for (int i = 0; i < n; ++i) {
        const MgaqItem& m = items[i];
        cudaStream_t sk = ss.s[i % kBatchStreams];
        if (m.group_size) {
            e = launch_quantize_per_group(m.x, m.dtype, m.n, m.group_size, m.codes, m.scales, flags, sk);
        } else {
            uint32_t* amax = m.amax_out ? m.amax_out : ss.amax_ws + i;
            e = launch_group_amax(m.x, m.dtype, m.n, 128, nullptr, amax, flags, sk);
            if (e == cudaSuccess) e = launch_quantize_per_tensor(m.x, m.dtype, m.n, amax, m.codes, m.scales, flags, sk);
        }
        if (e != cudaSuccess) return e;
    }
    for (int k = 0; k < kBatchStreams; ++k) {
        if ((e = cudaEventRecord(ss.join[k], ss.s[k])) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(st, ss.join[k], 0)) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace coat
