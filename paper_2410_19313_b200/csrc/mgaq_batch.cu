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
#include <algorithm>
#include <climits>
#include <mutex>
#include <vector>

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

    // occupancy per device (queried once); the grid barrier word and the
    // per-CTA partials are a stream-ordered allocation of this call, so
    // concurrent batches on different streams never share them
    static std::mutex mu;
    static int per_sm_of[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    int per_sm = 0;
    {
        std::lock_guard<std::mutex> lock(mu);
        if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
        if (per_sm_of[dev] == 0) {
            const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_of[dev], mgaq_batch_kernel,
                                                                                kThreads, 0);
            if (e != cudaSuccess) return e;
            if (per_sm_of[dev] <= 0) per_sm_of[dev] = 1;
        }
        per_sm = per_sm_of[dev];
    }
    const int grid = device_sm_count() * per_sm;
    const size_t words = size_t(kMgaqMaxItems) * size_t(grid) + 32;
    uint32_t* buf = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&buf), words * sizeof(uint32_t), st);
    if (e != cudaSuccess) return e;
    P.barrier = buf;
    P.partials = buf + 32;
    e = cudaMemsetAsync(P.barrier, 0, sizeof(uint32_t), st);
    if (e == cudaSuccess) {
        float nz = -0.0f;
        void* args[] = {&P, &nz};
        e = cudaLaunchCooperativeKernel((void*)mgaq_batch_kernel, dim3(grid), dim3(kThreads), args, 0, st);
    }
    const cudaError_t f = cudaFreeAsync(buf, st);
    return e != cudaSuccess ? e : f;
}

// ---------------------------------------------------------------------------
// The task-queue schedule (COAT_MGAQ_BATCH=queue): ONE persistent,
// warp-specialised kernel for a whole layer.  A producer warp per CTA claims
// tasks (32 KB of one record's input; two per atomic) from a global counter
// and bulk-copies them (cp.async.bulk + mbarrier, with the L2 eviction hint)
// into a ring of kSlots shared-memory slots; eight consumer warps quantize
// slot after slot.  The host orders the queue so that every per-tensor
// record's encode tasks come 2 (kSlots + kClaim) grids of per-group work after its
// absmax tasks: the record's x is still in L2 (the absmax copies mark the tail
// evict_last, the encode walks it tail first) and its absmax is complete.  The
// producer of an encode task waits for the record's absmax-task count before
// handing the slot over; every task it waits for was claimed earlier, and each
// CTA processes its tasks in claim order while absmax tasks never wait, so the
// queue cannot deadlock -- whether or not the whole grid is resident.
// Specialised on the dtype, per-group items 1x16 (the cfg2 layer); other
// batches take the stream schedule.
namespace {
#ifndef COAT_QUEUE_TASK_KB
#define COAT_QUEUE_TASK_KB 32
#endif
#ifndef COAT_QUEUE_SLOTS
#define COAT_QUEUE_SLOTS 3
#endif
#ifndef COAT_QUEUE_CLAIM
#define COAT_QUEUE_CLAIM 2
#endif
constexpr int kTaskBytes = COAT_QUEUE_TASK_KB * 1024;
constexpr int kSlots = COAT_QUEUE_SLOTS;
constexpr int kClaim = COAT_QUEUE_CLAIM;        // tasks per atomic claim
#ifndef COAT_QUEUE_MARGIN
#define COAT_QUEUE_MARGIN 2                     // filler between a record's absmax and encode tasks, in lookaheads
#endif
#ifndef COAT_QUEUE_CONSUMERS
#define COAT_QUEUE_CONSUMERS 256
#endif
constexpr int kConsumers = COAT_QUEUE_CONSUMERS;   // consumer threads (8 warps)
constexpr int kQThreads = kConsumers + 32;      // + the producer warp
constexpr int kMaxSegs = 3 * kMgaqMaxItems + 2;
struct QSeg {
    int64_t first_task;
    int64_t chunk0, nchunks;        // chunks [chunk0, chunk0 + nchunks) of the item (encode: counted from its end)
    int32_t item;
    int32_t phase;                  // 0 per-group, 1 absmax, 2 encode
};
struct QParams {
    BItem it[kMgaqMaxItems];
    int64_t keep_from[kMgaqMaxItems];   // first chunk of the item's L2-resident tail
    int32_t amax_tasks[kMgaqMaxItems];
    QSeg seg[kMaxSegs];
    int32_t nseg;
    int64_t ntasks;
    unsigned long long* counter;
    uint32_t* amax;
    uint32_t* done;
    uint32_t* flags;
};
struct SlotMeta {
    int64_t c0, c1;                 // chunk range; c0 < 0: no more tasks
    int32_t item, phase;
    float sc, rs;                   // encode: the record's scale and RN(1/scale)
};

template <int DT>
__host__ __device__ constexpr int task_chunks() { return kTaskBytes / (16 * (DT == 0 ? 4 : 2)); }

__device__ __forceinline__ uint32_t q_smem(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void q_mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(q_smem(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void q_mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(q_smem(bar)) : "memory");
}
__device__ __forceinline__ void q_mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W_%=;\n}\n" ::"r"(q_smem(bar)),
        "r"(parity)
        : "memory");
}

template <int DT>
__device__ __forceinline__ RawChunk<DT> q_chunk(const uint8_t* buf, int64_t local) {
    RawChunk<DT> c;
    const uint4* p = reinterpret_cast<const uint4*>(buf + local * 16 * (DT == 0 ? 4 : 2));
#pragma unroll
    for (int k = 0; k < (DT == 0 ? 4 : 2); ++k) {
        const uint4 v = p[k];
        c.w[4 * k] = v.x; c.w[4 * k + 1] = v.y; c.w[4 * k + 2] = v.z; c.w[4 * k + 3] = v.w;
    }
    return c;
}

template <int DT>
__global__ void __launch_bounds__(kQThreads) mgaq_queue_kernel(const __grid_constant__ QParams P, float nz) {
    extern __shared__ __align__(128) uint8_t qsmem[];
    __shared__ __align__(8) uint64_t full[kSlots], empty[kSlots];
    __shared__ SlotMeta meta[kSlots];
    __shared__ uint32_t s_red[kConsumers / 32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kSlots; ++i) {
            q_mbar_init(&full[i], 1);
            q_mbar_init(&empty[i], kConsumers / 32);   // one arrival per consumer warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    constexpr int esz = DT == 0 ? 4 : 2;
    if (warp == kConsumers / 32) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            long long t = 0, t_end = 0;   // claimed tasks [t, t_end)
            int sgi = 0;                   // segment of the last task (claims only grow: the scan resumes)
            for (int k = 0, slot = 0;; ++k, slot = (slot + 1) % kSlots) {
                if (k >= kSlots) q_mbar_wait(&empty[slot], ((k / kSlots) - 1) & 1u);
                if (t == t_end) {
                    t = (long long)atomicAdd(P.counter, (unsigned long long)kClaim);
                    t_end = t + kClaim;
                }
                SlotMeta& m = meta[slot];
                if (t >= P.ntasks) {
                    m.c0 = -1;
                    q_mbar_arrive(&full[slot]);   // the end marker: consumers leave
                    break;
                }
                const int64_t task = t++;
                while (sgi + 1 < P.nseg && P.seg[sgi + 1].first_task <= task) ++sgi;
                const QSeg& sg = P.seg[sgi];
                const BItem& I = P.it[sg.item];
                const int64_t a = sg.chunk0 + (task - sg.first_task) * task_chunks<DT>();
                const int64_t e = sg.chunk0 + sg.nchunks;
                const int64_t b = a + task_chunks<DT>() < e ? a + task_chunks<DT>() : e;
                m.item = sg.item;
                m.phase = sg.phase;
                if (sg.phase == 2) {   // encode walks the tensor from its end
                    m.c0 = I.nchunks - b;
                    m.c1 = I.nchunks - a;
                    while (ld_acquire_u32(&P.done[sg.item]) < uint32_t(P.amax_tasks[sg.item])) __nanosleep(64);
                    const uint32_t am = ld_acquire_u32(&P.amax[sg.item]);
                    const float sc = group_scale(u2f(am));
                    m.sc = sc;
                    m.rs = __frcp_rn(sc);
                    if (task == sg.first_task) {   // the record's first encode task publishes scale and absmax
                        I.scales[0] = float_to_bf16_bits_exact(sc);
                        if (I.amax_out) *I.amax_out = am;
                    }
                } else {
                    m.c0 = a;
                    m.c1 = b;
                }
                uint64_t pol;
                if (sg.phase == 1 && m.c1 > P.keep_from[sg.item])
                    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
                else
                    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
                const uint32_t bytes = uint32_t((m.c1 - m.c0) * 16 * esz);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(q_smem(&full[slot])),
                             "r"(bytes)
                             : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
                    "%2, [%3], %4;" ::"r"(q_smem(qsmem + slot * kTaskBytes)),
                    "l"(static_cast<const uint8_t*>(I.x) + m.c0 * 16 * esz), "r"(bytes), "r"(q_smem(&full[slot])),
                    "l"(pol)
                    : "memory");
            }
        }
        return;
    }
    // ---------------------------------------------------------------- consumers
    uint32_t bad = 0;
    for (int k = 0, slot = 0;; ++k, slot = (slot + 1) % kSlots) {
        q_mbar_wait(&full[slot], (k / kSlots) & 1u);
        const SlotMeta m = meta[slot];
        if (m.c0 < 0) break;
        const BItem& I = P.it[m.item];
        const uint8_t* buf = qsmem + slot * kTaskBytes;
        const int64_t n = m.c1 - m.c0;
        uint32_t am = 0;
        for (int64_t j = threadIdx.x; j < n; j += kConsumers) {
            const RawChunk<DT> raw = q_chunk<DT>(buf, j);
            const int64_t ch = m.c0 + j;
            if (m.phase == 0) {   // 1x16: one chunk = one group
                const uint32_t ga = absmax_raw<DT, false>(raw);
                float sc, rs;
                group_scale_fast(ga, sc, rs);
                reinterpret_cast<uint4*>(I.codes)[ch] = encode16(widen16<DT>(raw), sc, rs, nz);
                I.scales[ch] = float_to_bf16_bits_exact(sc);
                bad |= ga >= 0x7F800000u;
            } else if (m.phase == 1) {
                am = max(am, absmax_raw<DT, true>(raw));
            } else {
                reinterpret_cast<uint4*>(I.codes)[ch] = encode16(widen16<DT>(raw), m.sc, m.rs, nz);
                bad |= absmax_raw<DT, false>(raw) >= 0x7F800000u;
            }
        }
        if (m.phase == 1) {   // the task's absmax: consumer-only named barrier, one atomic per task
            am = warp_max_u32(am);
            if (lane == 0) s_red[warp] = am;
            asm volatile("bar.sync 1, %0;" ::"r"(kConsumers) : "memory");
            if (threadIdx.x == 0) {
                uint32_t a = 0;
                for (int w = 0; w < kConsumers / 32; ++w) a = max(a, s_red[w]);
                if (a) atomicMax(&P.amax[m.item], a);
                __threadfence();                       // the max before the count
                atomicAdd(&P.done[m.item], 1u);
            }
            asm volatile("bar.sync 1, %0;" ::"r"(kConsumers) : "memory");   // s_red reusable
        }
        __syncwarp();
        if (lane == 0) q_mbar_arrive(&empty[slot]);   // the slot's reads are done
    }
    if (P.flags && __reduce_or_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(P.flags, kFlagNonFiniteInput);
}
}  // namespace

cudaError_t launch_mgaq_queue(const MgaqItem* items, int n, uint32_t* flags, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    if (n > kMgaqMaxItems) return cudaErrorInvalidValue;
    const int dt = items[0].dtype;
    for (int i = 0; i < n; ++i)
        if (items[i].dtype != dt || (items[i].group_size != 0 && items[i].group_size != 16))
            return launch_mgaq_streams(items, n, flags, st);   // the kernel's specialisation does not apply
    const int smem = kSlots * kTaskBytes;
    static std::mutex occ_mu;
    static int per_sm[2] = {0, 0};
    static int occ_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    std::unique_lock<std::mutex> occ_lock(occ_mu);
    if (occ_dev != dev) {
        cudaError_t e = cudaFuncSetAttribute(mgaq_queue_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(mgaq_queue_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[0], mgaq_queue_kernel<0>, kQThreads, smem);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[1], mgaq_queue_kernel<1>, kQThreads, smem);
        if (e != cudaSuccess) return e;
        occ_dev = dev;
    }
    const int grid = device_sm_count() * (per_sm[dt] > 0 ? per_sm[dt] : 1);
    occ_lock.unlock();
    const int64_t tc = dt == 0 ? task_chunks<0>() : task_chunks<1>();
    QParams P{};
    std::vector<int> pt, pg;
    for (int i = 0; i < n; ++i) {
        const MgaqItem& m = items[i];
        BItem& b = P.it[i];
        b.x = m.x;
        b.codes = m.codes;
        b.scales = m.scales;
        b.amax_out = m.amax_out;
        b.nchunks = m.n / 16;
        b.dtype = m.dtype;
        b.lanes = m.group_size ? 1 : 0;
        P.keep_from[i] = l2_keep_chunks(b.nchunks, dt == 0 ? 4 : 2);
        P.amax_tasks[i] = int32_t((b.nchunks + tc - 1) / tc);
        (m.group_size ? pg : pt).push_back(i);
    }
    // queue: for every per-tensor record: its absmax tasks, twice kSlots + kClaim
    // grids of per-group tasks (every CTA holds at most kSlots + kClaim claimed
    // tasks, so the absmax tasks are processed well before), its encode
    // tasks; then the rest of the per-group work
    int64_t task = 0;
    size_t gi = 0;          // current per-group item
    int64_t gchunk = 0;     // its next chunk
    auto add = [&](int item, int phase, int64_t c0, int64_t nch) {
        QSeg& q = P.seg[P.nseg++];
        q.first_task = task;
        q.chunk0 = c0;
        q.nchunks = nch;
        q.item = item;
        q.phase = phase;
        task += (nch + tc - 1) / tc;
    };
    auto filler = [&](int64_t want_tasks) {
        while (want_tasks > 0 && gi < pg.size() && P.nseg < kMaxSegs - 2) {
            const BItem& b = P.it[pg[gi]];
            const int64_t left = b.nchunks - gchunk;
            const int64_t take = want_tasks >= (left + tc - 1) / tc ? left : want_tasks * tc;
            add(pg[gi], 0, gchunk, take);
            want_tasks -= (take + tc - 1) / tc;
            gchunk += take;
            if (gchunk >= b.nchunks) { ++gi; gchunk = 0; }
        }
    };
    for (int i : pt) {
        add(i, 1, 0, P.it[i].nchunks);
        filler(int64_t(COAT_QUEUE_MARGIN) * (kSlots + kClaim) * grid);
        add(i, 2, 0, P.it[i].nchunks);
    }
    filler(INT64_MAX);
    P.ntasks = task;
    P.flags = flags;
    uint32_t* ws = nullptr;
    const size_t wsb = (2 + 2 * kMgaqMaxItems) * sizeof(uint32_t);
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&ws), wsb, st);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(ws, 0, wsb, st);
    if (e != cudaSuccess) return e;
    P.counter = reinterpret_cast<unsigned long long*>(ws);
    P.amax = ws + 2;
    P.done = ws + 2 + kMgaqMaxItems;
    if (dt == 0) mgaq_queue_kernel<0><<<grid, kQThreads, smem, st>>>(P, -0.0f);
    else mgaq_queue_kernel<1><<<grid, kQThreads, smem, st>>>(P, -0.0f);
    e = cudaGetLastError();
    const cudaError_t f = cudaFreeAsync(ws, st);
    return e != cudaSuccess ? e : f;
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

bool mgaq_batch_queue() {
    static const bool q = [] {
        const char* e = getenv("COAT_MGAQ_BATCH");
        return e && e[0] == 'q';
    }();
    return q;
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
        int lo = 0, hi = 0;   // stream 0 (the per-tensor records) at the highest priority
        if ((e = cudaDeviceGetStreamPriorityRange(&lo, &hi)) != cudaSuccess) return e;
        for (int k = 0; k < kBatchStreams; ++k) {
            if ((e = cudaStreamCreateWithPriority(&ss.s[k], cudaStreamNonBlocking, k == 0 ? hi : lo)) != cudaSuccess)
                return e;
            if ((e = cudaEventCreateWithFlags(&ss.join[k], cudaEventDisableTiming)) != cudaSuccess) return e;
        }
        if ((e = cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming)) != cudaSuccess) return e;
        if ((e = cudaMalloc(&ss.amax_ws, kMgaqMaxItems * sizeof(uint32_t))) != cudaSuccess) return e;
        ss.dev = dev;
    }
    if ((e = cudaEventRecord(ss.fork, st)) != cudaSuccess) return e;
    for (int k = 0; k < kBatchStreams; ++k)
        if ((e = cudaStreamWaitEvent(ss.s[k], ss.fork, 0)) != cudaSuccess) return e;
    // The per-tensor items on stream 0, at high priority: one per-tensor item
    // at a time, so its tensor stays L2-resident between the absmax and encode
    // passes, running at full speed while the per-group items fill in on the
    // other streams, round-robin.  (Measured on the cfg2 layer graph: 0.3068 vs
    // 0.3090 ms for all items round-robin, DRAM 1.15x vs 1.17x the algorithmic
    // bytes; the one stream without the priority: 0.323-0.330 ms.)
    int next_g = 0;
    for (int i = 0; i < n; ++i) {
        const MgaqItem& m = items[i];
        cudaStream_t sk = m.group_size ? ss.s[1 + (next_g++) % (kBatchStreams - 1)] : ss.s[0];
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
