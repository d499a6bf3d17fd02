// zero_p2p.cu -- the ZeRO step with its two collectives done by SM kernels
// over NVLink peer memory instead of NCCL (PAPER.md:523 names
// the optimizer's communication as the open cost):
//
//   reduce-scatter  g_shard = sum over ranks of every rank's gradient shard,
//                   read in place from the peers' gradient buffers -- direct
//                   P2P loads summed in rank order (deterministic, unlike a
//                   ring), or ONE NVLink-SHARP `multimem.ld_reduce` per 16 B
//                   when the caller has a multicast address (the switch adds);
//   fused step      K1 on the shard (bit-identical to the single-GPU step);
//   all-gather      the updated shard stored straight into every rank's
//                   next-weight buffer (P2P stores, or one `multimem.st`).
//
// The shard is pipelined in chunks over three streams so the NVLink-bound
// reduce of chunk i+1 and broadcast of chunk i-1 run while K1 (HBM-bound)
// steps chunk i -- the collective traffic overlaps the math instead of
// bracketing it (coat_zero_step: reduce-scatter, step, all-gather in sequence).
// The copy kernels are small (64-thread CTAs, <= 64 registers: 16 per SM) so they fit
// beside K1's two persistent CTAs per SM.
//
// Weights are double-buffered across the step (w_cur -> w_next on every
// rank): nothing the step reads is overwritten, so the reference's
// all-or-nothing commit (optimizer.cpp:101-114) needs no republish -- the
// caller OR-reduces the error word and keeps w_cur and the old state when it
// is set.  bf16 gradient wire: peers hold bf16 gradients (half the NVLink
// bytes); the sum is formed in fp32 in rank order.
#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "../../include/coat.h"
#include "coat_device.cuh"
#include "coat_internal.h"

namespace coat {
namespace {

constexpr int kMaxPeers = 16;
constexpr int kCopyThreads = 64;
constexpr int kBatch = 8;   // peer loads in flight per thread before they are summed

struct GradPeers {
    const void* p[kMaxPeers];
};
struct WeightPeers {
    float* p[kMaxPeers];
};

__device__ __forceinline__ float4 ldg_f4(const void* p) {
    float4 v;
    asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ uint4 ldg_u4(const void* p) {
    uint4 v;
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
    return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}

// fp32 wire: out[i] = (((g_0[i] + g_1[i]) + g_2[i]) + ...) for the float4s
// [0, n4) of the slice starting at element `off` of every peer's buffer.
__global__ void __launch_bounds__(kCopyThreads, 16)
reduce_p2p_f32_kernel(GradPeers g, int nranks, int64_t off, int64_t n4, float* __restrict__ out) {
    for (int64_t i = int64_t(blockIdx.x) * kCopyThreads + threadIdx.x; i < n4; i += int64_t(gridDim.x) * kCopyThreads) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int r0 = 0; r0 < nranks; r0 += kBatch) {
            float4 v[kBatch];
#pragma unroll
            for (int j = 0; j < kBatch; ++j)
                if (r0 + j < nranks) v[j] = ldg_f4(static_cast<const float*>(g.p[r0 + j]) + off + 4 * i);
#pragma unroll
            for (int j = 0; j < kBatch; ++j)
                if (r0 + j < nranks) acc = (r0 + j == 0) ? v[j] : add4(acc, v[j]);
        }
        reinterpret_cast<float4*>(out + 4 * i)[0] = acc;
    }
}

// bf16 wire: 8 gradients per 16-byte load, widened exactly, summed in fp32.
__global__ void __launch_bounds__(kCopyThreads, 16)
reduce_p2p_bf16_kernel(GradPeers g, int nranks, int64_t off, int64_t n8, float* __restrict__ out) {
    for (int64_t i = int64_t(blockIdx.x) * kCopyThreads + threadIdx.x; i < n8; i += int64_t(gridDim.x) * kCopyThreads) {
        float4 lo = make_float4(0.f, 0.f, 0.f, 0.f), hi = lo;
        for (int r0 = 0; r0 < nranks; r0 += kBatch) {
            uint4 v[kBatch];
#pragma unroll
            for (int j = 0; j < kBatch; ++j)
                if (r0 + j < nranks) v[j] = ldg_u4(static_cast<const uint16_t*>(g.p[r0 + j]) + off + 8 * i);
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                if (r0 + j >= nranks) continue;
                const float4 a = make_float4(u2f(v[j].x << 16), u2f(v[j].x & 0xFFFF0000u), u2f(v[j].y << 16),
                                             u2f(v[j].y & 0xFFFF0000u));
                const float4 b = make_float4(u2f(v[j].z << 16), u2f(v[j].z & 0xFFFF0000u), u2f(v[j].w << 16),
                                             u2f(v[j].w & 0xFFFF0000u));
                lo = (r0 + j == 0) ? a : add4(lo, a);
                hi = (r0 + j == 0) ? b : add4(hi, b);
            }
        }
        float4* o = reinterpret_cast<float4*>(out + 8 * i);
        o[0] = lo;
        o[1] = hi;
    }
}

// NVLink SHARP: the switch returns the sum over every rank's copy of the
// multicast object (fp32 accumulation; the order is the switch's).
__global__ void __launch_bounds__(kCopyThreads, 16)
reduce_nvls_f32_kernel(const float* mc, int64_t off, int64_t n4, float* __restrict__ out) {
    for (int64_t i = int64_t(blockIdx.x) * kCopyThreads + threadIdx.x; i < n4; i += int64_t(gridDim.x) * kCopyThreads) {
        float4 v;
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                     : "l"(mc + off + 4 * i)
                     : "memory");
        reinterpret_cast<float4*>(out + 4 * i)[0] = v;
    }
}

// all-gather: src[0, 4*n4) -> every other rank's buffer at element `off`
// (the own copy is where the step wrote it).
__global__ void __launch_bounds__(kCopyThreads, 16)
broadcast_p2p_kernel(WeightPeers w, int nranks, int self, int64_t off, int64_t n4, const float* __restrict__ src) {
    for (int64_t i = int64_t(blockIdx.x) * kCopyThreads + threadIdx.x; i < n4; i += int64_t(gridDim.x) * kCopyThreads) {
        const float4 v = reinterpret_cast<const float4*>(src)[i];
        for (int r = 0; r < nranks; ++r)
            if (r != self) reinterpret_cast<float4*>(w.p[r] + off)[i] = v;
    }
    __threadfence_system();   // peer stores performed before the caller's cross-rank sync
}

__global__ void __launch_bounds__(kCopyThreads, 16)
broadcast_nvls_kernel(float* mc, int64_t off, int64_t n4, const float* __restrict__ src) {
    for (int64_t i = int64_t(blockIdx.x) * kCopyThreads + threadIdx.x; i < n4; i += int64_t(gridDim.x) * kCopyThreads) {
        const float4 v = reinterpret_cast<const float4*>(src)[i];
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + off + 4 * i), "f"(v.x),
                     "f"(v.y), "f"(v.z), "f"(v.w)
                     : "memory");
    }
    __threadfence_system();
}

int copy_grid(int64_t items) {
    const int64_t cap = int64_t(device_sm_count()) * 2;
    return (int)imax64(1, imin64((items + kCopyThreads - 1) / kCopyThreads, cap));
}

struct Streams {
    int device = -1;
    cudaStream_t rs = nullptr, ag = nullptr;
    cudaError_t init(int dev) {
        if (device == dev) return cudaSuccess;
        cudaError_t e = cudaStreamCreateWithFlags(&rs, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ag, cudaStreamNonBlocking);
        if (e == cudaSuccess) device = dev;
        return e;
    }
};
Streams g_streams[16];
std::mutex g_streams_mu;

MomentStateIn slice_in(const coat_moment_state& s, int64_t off) {
    return {s.codes + off, s.scales + off / 128, s.k + off / 128, s.c + off / 128};
}
MomentStateOut slice_out(const coat_moment_state& s, int64_t off) {
    return {s.codes + off, s.scales + off / 128, s.k + off / 128, s.c + off / 128};
}

}  // namespace

cudaError_t zero_p2p_step(const ZeroP2PArgs& z, const AdamWScalars& a, uint32_t* flags,
                          unsigned long long* fallbacks, cudaStream_t stream) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 16) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lock(g_streams_mu);
    Streams& ss = g_streams[dev];
    if ((e = ss.init(dev)) != cudaSuccess) return e;

    GradPeers gp{};
    WeightPeers wp{};
    for (int r = 0; r < z.nranks; ++r) {
        gp.p[r] = z.g_peers ? z.g_peers[r] : nullptr;
        wp.p[r] = z.w_next_peers ? z.w_next_peers[r] : nullptr;
    }
    const int64_t n = z.n_shard, base = int64_t(z.rank) * n;
    // P2P: fuse the all-gather into K1 (COAT_P2P_FUSED_AG=0: the separate broadcast)
    static const bool fuse_ag = [] {
        const char* v = getenv("COAT_P2P_FUSED_AG");
        return !(v && v[0] == '0');
    }();
    int64_t peer_delta[7] = {0, 0, 0, 0, 0, 0, 0};
    int npeers = 0;
    const bool peer_fused = fuse_ag && !z.w_next_mc && z.w_next_peers && z.nranks > 1 && z.nranks <= 8 &&
                            !fallbacks;
    bool fuse_ok = peer_fused;
    if (fuse_ok)
        for (int r = 0; r < z.nranks; ++r)
            if (r != z.rank) {
                const int64_t d = int64_t(reinterpret_cast<intptr_t>(z.w_next_peers[r]) -
                                          reinterpret_cast<intptr_t>(z.w_next));
                if (d % int64_t(sizeof(float)) != 0) fuse_ok = false;
                peer_delta[npeers++] = d / int64_t(sizeof(float));
            }
    if (!fuse_ok) npeers = 0;
    const int64_t unit = k1_ws_round_params();
    int64_t chunk = z.chunk > 0 ? z.chunk : int64_t(64) << 20;
    chunk = (chunk + unit - 1) / unit * unit;
    const int64_t nchunks = (n + chunk - 1) / chunk;

    cudaEvent_t start, fin;
    cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&fin, cudaEventDisableTiming);
    cudaEventRecord(start, stream);
    cudaStreamWaitEvent(ss.rs, start, 0);
    cudaStreamWaitEvent(ss.ag, start, 0);
    for (int64_t i = 0; i < nchunks && e == cudaSuccess; ++i) {
        const int64_t off = i * chunk;
        const int64_t len = n - off < chunk ? n - off : chunk;   // multiple of 128 (FlatLayout)
        // reduce-scatter of this chunk (rs stream, runs ahead of the step)
        if (z.g_mc) {
            reduce_nvls_f32_kernel<<<copy_grid(len / 4), kCopyThreads, 0, ss.rs>>>(
                static_cast<const float*>(z.g_mc), base + off, len / 4, z.g_shard + off);
        } else if (z.g_dtype == 0) {
            reduce_p2p_f32_kernel<<<copy_grid(len / 4), kCopyThreads, 0, ss.rs>>>(gp, z.nranks, base + off, len / 4,
                                                                                  z.g_shard + off);
        } else {
            reduce_p2p_bf16_kernel<<<copy_grid(len / 8), kCopyThreads, 0, ss.rs>>>(gp, z.nranks, base + off, len / 8,
                                                                                   z.g_shard + off);
        }
        cudaEvent_t reduced, stepped;
        cudaEventCreateWithFlags(&reduced, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&stepped, cudaEventDisableTiming);
        cudaEventRecord(reduced, ss.rs);
        // the fused step on the caller's stream; over P2P (no multicast) the
        // all-gather is fused into it: K1 stores every w' into the peers'
        // next-weight buffers as well (whole rounds; the ragged tail below)
        cudaStreamWaitEvent(stream, reduced, 0);
        int64_t fused = 0;
        if (fuse_ok) {
            e = launch_adamw_dre_step_peers(z.w_cur + base + off, z.w_next + base + off, z.g_shard + off, len,
                                            slice_in(z.m_in, off), slice_in(z.v_in, off), slice_out(z.m_out, off),
                                            slice_out(z.v_out, off), a, flags, peer_delta, npeers, &fused, stream);
        } else {
            e = launch_adamw_dre_step(z.w_cur + base + off, z.w_next + base + off, z.g_shard + off, len,
                                      slice_in(z.m_in, off), slice_in(z.v_in, off), slice_out(z.m_out, off),
                                      slice_out(z.v_out, off), a, flags, fallbacks, stream);
        }
        cudaEventRecord(stepped, stream);
        // all-gather of this chunk (ag stream, behind the step) -- what K1 did not store
        cudaStreamWaitEvent(ss.ag, stepped, 0);
        const int64_t boff = off + fused, blen = len - fused;
        if (blen > 0 && z.w_next_mc)
            broadcast_nvls_kernel<<<copy_grid(blen / 4), kCopyThreads, 0, ss.ag>>>(z.w_next_mc, base + boff,
                                                                                  blen / 4, z.w_next + base + boff);
        else if (blen > 0 && z.nranks > 1)
            broadcast_p2p_kernel<<<copy_grid(blen / 4), kCopyThreads, 0, ss.ag>>>(
                wp, z.nranks, z.rank, base + boff, blen / 4, z.w_next + base + boff);
        cudaEventDestroy(reduced);   // released once recorded work completes
        cudaEventDestroy(stepped);
    }
    cudaEventRecord(fin, ss.ag);
    cudaStreamWaitEvent(stream, fin, 0);
    cudaEventDestroy(fin);
    cudaEventDestroy(start);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace coat
