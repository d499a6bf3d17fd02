// adamw_dre.cu -- K1: the fused FP8-DRE AdamW step, plus the standalone DRE
// quantize / contract kernels that share its device code.
//
// Reference: coatsim::step (proj/core/src/optimizer.cpp:101-114) with the
// policy {E4M3, expand=true, G=128} for both moments:
//   m,v = unpack_moment(slot)            optimizer.cpp:49-55  (dequantize + contract)
//   adamw_update(w, m, v, g, t)          optimizer.cpp:57-68  (fp32, no FMA)
//   slot.m/v = pack_moment(m/v)          optimizer.cpp:40-47  (measure, expand, quantize)
// The reference makes ~10 full passes over memory; this kernel makes one:
// it reads w, g, the two code arrays and the per-group {scale, k, c}, and
// writes w, the new codes and the new per-group {scale, k, c}:
//   16 B/param (w r/w 8, g 4, codes r/w 2x2) + 40 B per 128-group of metadata
//   = 16.3125 B/param of compulsory HBM traffic.
//
// Work decomposition (B200): one warp owns a "tile" of 4 groups = 512
// params; lane l holds params 4l..4l+3 of every group, so every global access
// is a fully-coalesced 128-bit (w, g) or 32-bit (codes) warp-contiguous load.
// Group extrema are single redux.sync instructions on the fp32 bit patterns
// (non-negative floats order like u32).  The 8 (group, moment) parameter sets
// of a tile (k, c, scale -- double-precision log/sqrt/pow as in the
// reference) are computed by 8 lanes in one pass and shared through shared
// memory.  Grid = a persistent multiple of the SM count.
//
// Error semantics (errors.hpp:8-22): non-finite gradients set
// kFlagNonFiniteGrad; a moment whose expanded values are not finite sets
// kFlagPackM / kFlagPackV.  The state is written to SEPARATE output buffers
// (ping-pong), so the host commits exactly what the reference would have
// committed (see paper_2410_19313_b200/coatsim.py: step()).
#include <cstdint>
#include <cstdlib>

#include "coat_device.cuh"
#include "dre.cuh"
#include "coat_internal.h"

namespace coat {
namespace {

using dre::ContractParams;
using dre::PackParams;

constexpr int kTileGroups = 4;
constexpr int kTile = kTileGroups * dre::kG;   // 512 params per warp tile
constexpr int kWarps = 8;                      // warps per CTA
constexpr int kThreads = kWarps * 32;

struct StepScalars {
    float b1, b2, omb1, omb2, lr, wd, eps, bc1, bc2;
    double log_target;
};

struct WarpShared {
    ContractParams cp[8];   // [moment*TG + group] of the incoming state
    PackParams pp[8];       // [moment*TG + group] of the outgoing state
    uint32_t ext[16];       // lo/hi bit patterns per pair
};

// Load the incoming per-group meta for pair p = mom*4+grp (lanes 0..7).
__device__ __forceinline__ ContractParams load_contract(const MomentStateIn& st, int64_t grp) {
    const float s = bf16_bits_to_float(st.scales[grp]);
    return dre::contract_prepare(s, st.k[grp], st.c[grp]);
}

__device__ __forceinline__ void store_pack(const MomentStateOut& st, int64_t grp, const PackParams& p) {
    st.scales[grp] = float_to_bf16_bits_exact(p.s);
    st.k[grp] = p.k;
    st.c[grp] = p.c;
}

// AdamW on one element, bit-identical to adamw_update (optimizer.cpp:57-68).
__device__ __forceinline__ void adamw_one(float& w, float& m, float& v, float g, const StepScalars& S) {
    m = __fadd_rn(__fmul_rn(S.b1, m), __fmul_rn(S.omb1, g));
    v = __fadd_rn(__fmul_rn(S.b2, v), __fmul_rn(S.omb2, __fmul_rn(g, g)));
    const float mhat = __fdiv_rn(m, S.bc1);
    const float vhat = __fdiv_rn(v, S.bc2);
    const float upd = __fadd_rn(__fdiv_rn(mhat, __fadd_rn(__fsqrt_rn(vhat), S.eps)), __fmul_rn(S.wd, w));
    w = __fsub_rn(w, __fmul_rn(S.lr, upd));
}

// Exact extrema of |x| over nonzero elements; NaN/Inf map above every finite.
__device__ __forceinline__ void extrema4(const float (&x)[4], uint32_t& lo, uint32_t& hi) {
    lo = 0xFFFFFFFFu;
    hi = 0u;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t a = f2u(x[i]) & 0x7FFFFFFFu;
        hi = max(hi, a);
        lo = min(lo, a == 0u ? 0xFFFFFFFFu : a);
    }
}

// Compute pack params for the pairs of this warp from their extrema held in
// ws.ext (lane p < npairs works on pair p), publish through ws.pp.
__device__ __forceinline__ void pack_params_pass(WarpShared& ws, int lane, int npairs, double log_target) {
    if (lane < npairs) {
        const uint32_t lo = ws.ext[2 * lane], hi = ws.ext[2 * lane + 1];
        PackParams p;
        if (hi >= 0x7F800000u) {               // non-finite moment value
            p = dre::pack_prepare(1.0f, 1.0f, log_target);
            p.bad = true;
            p.mode = 2;
        } else {
            p = dre::pack_prepare(u2f(lo), u2f(hi), log_target);
        }
        ws.pp[lane] = p;
    }
    __syncwarp();
}

__device__ __forceinline__ uint32_t pack4(const float (&x)[4], const PackParams& p, uint32_t& fb) {
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) c |= dre::pack_one(x[i], p, fb) << (8 * i);
    return c;
}

__device__ __forceinline__ void contract4(uint32_t codes, const ContractParams& p, float (&x)[4], bool& bad) {
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = dre::contract_one((codes >> (8 * i)) & 0xFFu, p, bad);
}

// ----------------------------------------------------------------------------
// K1: fused step.
// ----------------------------------------------------------------------------
template <int TG>   // groups per warp tile (4; 1 for the short ragged tail after K1: 4x less serial work per lane)
__global__ void __launch_bounds__(kThreads)
adamw_dre_step_kernel(const float* w_in, float* w_out, const float* __restrict__ g, int64_t n,
                      MomentStateIn m_in, MomentStateIn v_in, MomentStateOut m_out,
                      MomentStateOut v_out, StepScalars S, uint32_t* flags,
                      unsigned long long* fallback_counter) {
    __shared__ WarpShared shared[kWarps];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    WarpShared& ws = shared[wid];
    const int64_t ng = (n + dre::kG - 1) / dre::kG;
    const int64_t ntiles = (ng + TG - 1) / TG;
    const int64_t warp_global = int64_t(blockIdx.x) * kWarps + wid;
    const int64_t warp_stride = int64_t(gridDim.x) * kWarps;
    const bool vec_ok = ((reinterpret_cast<uintptr_t>(w_in) | reinterpret_cast<uintptr_t>(w_out) |
                          reinterpret_cast<uintptr_t>(g)) & 15u) == 0;
    uint32_t myflags = 0;
    uint32_t fallbacks = 0;

    for (int64_t tile = warp_global; tile < ntiles; tile += warp_stride) {
        const int64_t g0 = tile * TG;
        const int gvalid = (int)imin64(TG, ng - g0);
        const int64_t base = g0 * dre::kG;
        const bool full = vec_ok && base + TG * dre::kG <= n;

        // ---- incoming per-group meta: lane p = mom*TG + grp
        if (lane < 2 * TG) {
            const int mom = lane / TG, grp = lane % TG;
            if (grp < gvalid) ws.cp[lane] = load_contract(mom ? v_in : m_in, g0 + grp);
        }
        // ---- streaming loads
        float w[TG][4], gr[TG][4];
        uint32_t cm[TG], cv[TG];
#pragma unroll
        for (int j = 0; j < TG; ++j) {
            const int64_t e0 = base + j * dre::kG + 4 * lane;
            if (j < gvalid) {
                cm[j] = ldg_u32(m_in.codes + e0);
                cv[j] = ldg_u32(v_in.codes + e0);
            } else {
                cm[j] = cv[j] = 0u;
            }
            if (full) {
                const float4 a = ldg_f4(w_in + e0);
                const float4 b = ldg_stream_f4(g + e0);
                w[j][0] = a.x; w[j][1] = a.y; w[j][2] = a.z; w[j][3] = a.w;
                gr[j][0] = b.x; gr[j][1] = b.y; gr[j][2] = b.z; gr[j][3] = b.w;
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const bool in = e0 + i < n;
                    w[j][i] = in ? w_in[e0 + i] : 0.0f;
                    gr[j][i] = in ? g[e0 + i] : 0.0f;
                }
            }
        }
        __syncwarp();

        // ---- unpack (dequantize + contract) and AdamW
        float m[TG][4], v[TG][4];
        bool bad_state = false;
#pragma unroll
        for (int j = 0; j < TG; ++j) {
            if (j < gvalid) {
                contract4(cm[j], ws.cp[j], m[j], bad_state);
                contract4(cv[j], ws.cp[TG + j], v[j], bad_state);
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i) m[j][i] = v[j][i] = 0.0f;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if (!isfinite(gr[j][i])) myflags |= kFlagNonFiniteGrad;
                adamw_one(w[j][i], m[j][i], v[j][i], gr[j][i], S);
                if (base + j * dre::kG + 4 * lane + i >= n) m[j][i] = v[j][i] = 0.0f;  // pad_flat
            }
        }
        if (bad_state) myflags |= kFlagContract;

        // ---- group extrema (exact) for both moments: 16 redux.sync
        uint32_t lo[2 * TG], hi[2 * TG];
#pragma unroll
        for (int j = 0; j < TG; ++j) {
            uint32_t l, h;
            extrema4(m[j], l, h);
            lo[j] = warp_min_u32(l);
            hi[j] = warp_max_u32(h);
            extrema4(v[j], l, h);
            lo[TG + j] = warp_min_u32(l);
            hi[TG + j] = warp_max_u32(h);
        }
        if (lane == 0) {
#pragma unroll
            for (int p = 0; p < 2 * TG; ++p) {
                ws.ext[2 * p] = lo[p];
                ws.ext[2 * p + 1] = hi[p];
            }
        }
        __syncwarp();
        pack_params_pass(ws, lane, 2 * TG, S.log_target);

        // ---- outgoing meta (lanes 0..7) + codes + weights
        if (lane < 2 * TG) {
            const int mom = lane / TG, grp = lane % TG;
            if (grp < gvalid) {
                const PackParams& p = ws.pp[lane];
                store_pack(mom ? v_out : m_out, g0 + grp, p);
                if (p.bad) myflags |= mom ? kFlagPackV : kFlagPackM;
            }
        }
#pragma unroll
        for (int j = 0; j < TG; ++j) {
            const int64_t e0 = base + j * dre::kG + 4 * lane;
            if (j < gvalid) {
                stg_u32(m_out.codes + e0, pack4(m[j], ws.pp[j], fallbacks));
                stg_u32(v_out.codes + e0, pack4(v[j], ws.pp[TG + j], fallbacks));
            }
            if (full) {
                stg_stream_f4(w_out + e0, make_float4(w[j][0], w[j][1], w[j][2], w[j][3]));
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (e0 + i < n) w_out[e0 + i] = w[j][i];
            }
        }
        __syncwarp();
    }
    myflags = warp_or_u32(myflags);
    if (lane == 0 && myflags && flags) atomicOr(flags, myflags);
    if (fallback_counter) {
        const uint32_t tot = __reduce_add_sync(0xFFFFFFFFu, fallbacks);
        if (lane == 0 && tot) atomicAdd(fallback_counter, (unsigned long long)tot);
    }
}

// ----------------------------------------------------------------------------
// expand_quantize (expand.cpp:115-135) of a flat fp32 tensor, n % 128 == 0.
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
expand_quantize_kernel(const float* __restrict__ x, int64_t n, MomentStateOut out, double log_target,
                       uint32_t* flags, unsigned long long* fallback_counter) {
    __shared__ WarpShared shared[kWarps];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    WarpShared& ws = shared[wid];
    const int64_t ng = n / dre::kG;
    const int64_t ntiles = (ng + kTileGroups - 1) / kTileGroups;
    uint32_t myflags = 0, fallbacks = 0;
    for (int64_t tile = int64_t(blockIdx.x) * kWarps + wid; tile < ntiles;
         tile += int64_t(gridDim.x) * kWarps) {
        const int64_t g0 = tile * kTileGroups;
        const int gvalid = (int)imin64(kTileGroups, ng - g0);
        const int64_t base = g0 * dre::kG;
        float xv[kTileGroups][4];
#pragma unroll
        for (int j = 0; j < kTileGroups; ++j) {
            if (j < gvalid) {
                const float4 a = ldg_stream_f4(x + base + j * dre::kG + 4 * lane);
                xv[j][0] = a.x; xv[j][1] = a.y; xv[j][2] = a.z; xv[j][3] = a.w;
            } else {
                xv[j][0] = xv[j][1] = xv[j][2] = xv[j][3] = 0.0f;
            }
        }
        uint32_t lo[4], hi[4];
#pragma unroll
        for (int j = 0; j < kTileGroups; ++j) {
            uint32_t l, h;
            extrema4(xv[j], l, h);
            lo[j] = warp_min_u32(l);
            hi[j] = warp_max_u32(h);
        }
        if (lane == 0) {
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                ws.ext[2 * p] = lo[p];
                ws.ext[2 * p + 1] = hi[p];
            }
        }
        __syncwarp();
        pack_params_pass(ws, lane, 4, log_target);
        if (lane < gvalid) {
            store_pack(out, g0 + lane, ws.pp[lane]);
            if (ws.pp[lane].bad) myflags |= kFlagNonFiniteInput;
        }
#pragma unroll
        for (int j = 0; j < kTileGroups; ++j)
            if (j < gvalid) stg_u32(out.codes + base + j * dre::kG + 4 * lane, pack4(xv[j], ws.pp[j], fallbacks));
        __syncwarp();
    }
    myflags = warp_or_u32(myflags);
    if (lane == 0 && myflags && flags) atomicOr(flags, myflags);
    if (fallback_counter) {
        const uint32_t tot = __reduce_add_sync(0xFFFFFFFFu, fallbacks);
        if (lane == 0 && tot) atomicAdd(fallback_counter, (unsigned long long)tot);
    }
}

// ----------------------------------------------------------------------------
// dequantize_contract (expand.cpp:137-141), n % 128 == 0.
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
dequantize_contract_kernel(MomentStateIn in, int64_t n, float* __restrict__ x, uint32_t* flags) {
    __shared__ WarpShared shared[kWarps];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    WarpShared& ws = shared[wid];
    const int64_t ng = n / dre::kG;
    const int64_t ntiles = (ng + kTileGroups - 1) / kTileGroups;
    bool bad = false;
    for (int64_t tile = int64_t(blockIdx.x) * kWarps + wid; tile < ntiles;
         tile += int64_t(gridDim.x) * kWarps) {
        const int64_t g0 = tile * kTileGroups;
        const int gvalid = (int)imin64(kTileGroups, ng - g0);
        const int64_t base = g0 * dre::kG;
        if (lane < gvalid) ws.cp[lane] = load_contract(in, g0 + lane);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < kTileGroups; ++j) {
            if (j < gvalid) {
                const int64_t e0 = base + j * dre::kG + 4 * lane;
                float v[4];
                contract4(ldg_u32(in.codes + e0), ws.cp[j], v, bad);
                stg_stream_f4(x + e0, make_float4(v[0], v[1], v[2], v[3]));
            }
        }
        __syncwarp();
    }
    if (flags && warp_or_u32(bad ? 1u : 0u) && lane == 0) atomicOr(flags, kFlagContract | kFlagNonFiniteInput);
}

// make_slot (optimizer.cpp:90-99): every group degenerate, k = c = 1,
// scale = round_bf16(2^-9) = 2^-9, codes 0.
__global__ void make_slot_kernel(MomentStateOut st, int64_t npad) {
    const int64_t ng = npad / dre::kG;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npad / 16;
         i += int64_t(gridDim.x) * blockDim.x)
        reinterpret_cast<uint4*>(st.codes)[i] = make_uint4(0, 0, 0, 0);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < ng;
         i += int64_t(gridDim.x) * blockDim.x) {
        st.scales[i] = 0x3B00u;   // bf16(2^-9)
        st.k[i] = 1.0f;
        st.c[i] = 1.0f;
    }
}

int grid_for(int64_t tiles, int per_cta) {
    const int sms = device_sm_count();
    const int64_t want = (tiles + per_cta - 1) / per_cta;
    const int64_t cap = int64_t(sms) * 4;   // persistent: 4 CTAs (32 warps) per SM
    return (int)imax64(1, imin64(want, cap));
}

}  // namespace

// ----------------------------------------------------------------------------
// host launchers (called by the C-ABI in api.cu)
// ----------------------------------------------------------------------------
cudaError_t launch_adamw_dre_step_peers(const float* w_in, float* w_out, const float* g, int64_t n,
                                        const MomentStateIn& m_in, const MomentStateIn& v_in,
                                        const MomentStateOut& m_out, const MomentStateOut& v_out,
                                        const AdamWScalars& a, uint32_t* flags, const int64_t* peer_delta,
                                        int npeers, int64_t* fused, cudaStream_t stream) {
    *fused = 0;
    if (n <= 0) return cudaSuccess;
    const int64_t unit = k1_ws_round_params();
    const int64_t nfull = n / unit;
    int64_t done = 0;
    if (nfull > 0) {
        const cudaError_t e =
            launch_k1_ws(w_in, w_out, g, nfull, m_in, v_in, m_out, v_out, a, flags, stream, peer_delta, npeers);
        if (e == cudaSuccess) done = nfull * unit;
        else if (e != cudaErrorNotSupported) return e;
    }
    *fused = done;
    if (done == n) return cudaSuccess;
    const int64_t gdone = done / dre::kG;
    return launch_adamw_dre_step(w_in + done, w_out + done, g + done, n - done,
                                 MomentStateIn{m_in.codes + done, m_in.scales + gdone, m_in.k + gdone, m_in.c + gdone},
                                 MomentStateIn{v_in.codes + done, v_in.scales + gdone, v_in.k + gdone, v_in.c + gdone},
                                 MomentStateOut{m_out.codes + done, m_out.scales + gdone, m_out.k + gdone,
                                                m_out.c + gdone},
                                 MomentStateOut{v_out.codes + done, v_out.scales + gdone, v_out.k + gdone,
                                                v_out.c + gdone},
                                 a, flags, nullptr, stream);
}

cudaError_t launch_adamw_dre_step(const float* w_in, float* w_out, const float* g, int64_t n,
                                  const MomentStateIn& m_in, const MomentStateIn& v_in,
                                  const MomentStateOut& m_out, const MomentStateOut& v_out,
                                  const AdamWScalars& a, uint32_t* flags,
                                  unsigned long long* fallbacks, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    StepScalars S;
    S.b1 = a.beta1;
    S.b2 = a.beta2;
    S.omb1 = 1.0f - a.beta1;
    S.omb2 = 1.0f - a.beta2;
    S.lr = a.lr;
    S.wd = a.weight_decay;
    S.eps = a.eps;
    S.bc1 = a.bc1;
    S.bc2 = a.bc2;
    S.log_target = a.log_target;
    // Whole rounds go through the warp-specialized kernel (k1_ws.cu); the
    // ragged tail (and misaligned buffers, or a fallback count request) through
    // the generic kernel below.
    int64_t done = 0;
    if (!fallbacks) {
        const int64_t unit = k1_ws_round_params();
        const int64_t nfull = n / unit;
        const cudaError_t e = launch_k1_ws(w_in, w_out, g, nfull, m_in, v_in, m_out, v_out, a, flags, stream);
        if (e == cudaSuccess) done = nfull * unit;
        else if (e != cudaErrorNotSupported) return e;
    }
    if (done == n) return cudaSuccess;
    const int64_t gdone = done / dre::kG;
    const MomentStateIn mi{m_in.codes + done, m_in.scales + gdone, m_in.k + gdone, m_in.c + gdone};
    const MomentStateIn vi{v_in.codes + done, v_in.scales + gdone, v_in.k + gdone, v_in.c + gdone};
    const MomentStateOut mo{m_out.codes + done, m_out.scales + gdone, m_out.k + gdone, m_out.c + gdone};
    const MomentStateOut vo{v_out.codes + done, v_out.scales + gdone, v_out.k + gdone, v_out.c + gdone};
    const int64_t rest = n - done;
    const int64_t ng = (rest + dre::kG - 1) / dre::kG;
    if (done > 0 && ng <= 64) {
        // the ragged tail after K1 (< one round): one group per warp, so the
        // per-element literal paths run 4x shorter chains (~40 -> ~10 us)
        adamw_dre_step_kernel<1><<<grid_for(ng, kWarps), kThreads, 0, stream>>>(
            w_in + done, w_out + done, g + done, rest, mi, vi, mo, vo, S, flags, fallbacks);
        return cudaGetLastError();
    }
    const int64_t ntiles = (ng + kTileGroups - 1) / kTileGroups;
    adamw_dre_step_kernel<kTileGroups><<<grid_for(ntiles, kWarps), kThreads, 0, stream>>>(
        w_in + done, w_out + done, g + done, rest, mi, vi, mo, vo, S, flags, fallbacks);
    return cudaGetLastError();
}

cudaError_t launch_expand_quantize(const float* x, int64_t n, const MomentStateOut& out,
                                   double log_target, uint32_t* flags,
                                   unsigned long long* fallbacks, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    int64_t done = 0;
    if (!fallbacks && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(out.codes)) & 15u) == 0) {
        const int64_t nfull = n / kTile;
        const cudaError_t e = launch_expand_quantize_fast(x, nfull, out, log_target, flags, stream);
        if (e != cudaSuccess) return e;
        done = nfull * kTile;
    }
    if (done == n) return cudaSuccess;
    const int64_t gd = done / dre::kG;
    const MomentStateOut o{out.codes + done, out.scales + gd, out.k + gd, out.c + gd};
    const int64_t rest = n - done;
    const int64_t ntiles = (rest / dre::kG + kTileGroups - 1) / kTileGroups;
    expand_quantize_kernel<<<grid_for(ntiles, kWarps), kThreads, 0, stream>>>(x + done, rest, o, log_target,
                                                                               flags, fallbacks);
    return cudaGetLastError();
}

cudaError_t launch_dequantize_contract(const MomentStateIn& in, int64_t n, float* x, uint32_t* flags,
                                       cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    int64_t done = 0;
    if (((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(in.codes)) & 15u) == 0) {
        const int64_t nfull = n / kTile;
        const cudaError_t e = launch_dequantize_contract_fast(in, nfull, x, flags, stream);
        if (e != cudaSuccess) return e;
        done = nfull * kTile;
    }
    if (done == n) return cudaSuccess;
    const int64_t gd = done / dre::kG;
    const MomentStateIn i2{in.codes + done, in.scales + gd, in.k + gd, in.c + gd};
    const int64_t rest = n - done;
    const int64_t ntiles = (rest / dre::kG + kTileGroups - 1) / kTileGroups;
    dequantize_contract_kernel<<<grid_for(ntiles, kWarps), kThreads, 0, stream>>>(i2, rest, x + done, flags);
    return cudaGetLastError();
}

cudaError_t launch_make_slot(const MomentStateOut& st, int64_t npad, cudaStream_t stream) {
    if (npad <= 0) return cudaSuccess;
    const int threads = 256;
    const int64_t work = imax64(npad / 16, npad / dre::kG);
    const int blocks = (int)imin64((work + threads - 1) / threads, int64_t(device_sm_count()) * 8);
    make_slot_kernel<<<max(blocks, 1), threads, 0, stream>>>(st, npad);
    return cudaGetLastError();
}

}  // namespace coat
