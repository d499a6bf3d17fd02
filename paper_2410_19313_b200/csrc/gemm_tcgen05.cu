// gemm_tcgen05.cu -- K4: the per-tensor FP8 linear (and its BF16 backward
// GEMMs) as a hand-written sm_100a tcgen05 / TMEM / TMA kernel.
//
// Reference semantics (flow.cpp):
//   forward  y  = matmul(DQ(Q_t(x)), DQ(Q_t(W)))                flow.cpp:21-33, 548-552
//            = (s_x * s_w) * (codes_x . codes_w)   -- E4M3 x E4M3 products are exact
//   dgrad    dX = bf16(dY . W_used^T)                             flow.cpp:36-46, 636
//   wgrad    dW = X_used^T . dY  (transposed FP8 codes of X)      flow.cpp:360-395, 637
// W is (K, N) row-major (flow.hpp:44-47).  dY stays BF16.
//
// One kernel template:  out[M,N] = alpha * sum_k A[m,k] * B[n,k]
//   A: M x K, K-major (memory [M][K]) or MN-major (memory [K][M])
//   B: N x K, K-major (memory [N][K]) or MN-major (memory [K][N])
//   kind::f8f6f4 (E4M3 x E4M3) or kind::f16 (BF16 x BF16), fp32 accumulate in TMEM.
// Persistent, warp-specialized, TMA (SWIZZLE_128B) -> smem ring of 128-byte K
// slices:
//   warp 0: TMA producer (one elected lane)       full/empty mbarriers per stage
//   warp 1: TMEM allocator + MMA issuer (one lane) tcgen05.mma + tcgen05.commit
//   warps 2-5: epilogue (TMEM lanes 0-127)        double-buffered accumulator
// Two variants (kCta):
//   1: one CTA per SM, 128 x 256 tile, cta_group::1 (small M).
//   2: a CTA pair on the two SMs of a TPC (cluster of 2), 256 x 256 tile,
//      tcgen05.mma.cta_group::2 issued by the leader.  Each CTA stages only its
//      128 rows of A and its 128-column half of B (32 KB per stage instead of
//      48 KB for half the FLOPs), so the L2->SM operand traffic per FLOP drops
//      by a third -- the 1-CTA kernel is operand-bandwidth bound at ~70% of the
//      tensor pipe.  Both CTAs' TMA bytes land on the leader's full barrier
//      (.cta_group::2 TMA, mapa address); commits multicast to both CTAs; both
//      CTAs' epilogues arrive on the leader's TMEM-empty barrier.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "coat_device.cuh"
#include "coat_internal.h"

namespace coat {
namespace gemm {

constexpr int BM = 128;                   // accumulator rows per CTA (TMEM lanes)
constexpr int BN = 256;                   // accumulator columns (MMA N)
constexpr int BKB = 128;                  // K bytes per stage (one 128B swizzle row)
constexpr int A_BYTES = BM * BKB;         // 16 KiB
constexpr int THREADS = 192;
constexpr int ACC_COLS = BN;              // fp32 columns per accumulator
constexpr int TMEM_COLS = 2 * ACC_COLS;   // double buffer = all 512 columns

template <int kCta>
struct Geo {
    static constexpr int BN_L = BN / kCta;                 // B rows staged by this CTA
    static constexpr int B_BYTES = BN_L * BKB;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
#ifndef COAT_GEMM_PAIR_STAGES
#define COAT_GEMM_PAIR_STAGES 6
#endif
    static constexpr int STAGES = kCta == 2 ? COAT_GEMM_PAIR_STAGES : 4;
    static constexpr int TILE_M = BM * kCta;
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

struct Params {
    int M, N, K;               // K in elements
    int tiles_m, tiles_n, k_blocks;
    float alpha;               // epilogue scale
    const uint16_t* scale_a;   // optional BF16 device scalars multiplied into alpha
    const uint16_t* scale_b;
    void* out;
    int64_t ldo;               // elements
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// shared::cluster address of `p` (a local smem object) in cluster CTA `rank`
__device__ __forceinline__ uint32_t cluster_addr(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t caddr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}
// TMA into this CTA's smem, completion bytes counted on the pair leader's barrier
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int x, int y, uint32_t bar_caddr) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
        "%3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(bar_caddr)
        : "memory");
}
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(uint16_t(3))
        : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
template <bool kF8, int kCta>
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    if (kF8 && kCta == 1) {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
    } else if (kCta == 1) {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
    } else if (kF8) {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
    } else {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
    }
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor, SWIZZLE_128B, sm100 version bits.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t((lbo_bytes >> 4) & 0x3FFFu) << 16) |
           (uint64_t((sbo_bytes >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}

// Instruction descriptor: fp32 accumulate, E4M3 (0) or BF16 (1) operands.
__host__ __device__ constexpr uint32_t instr_desc(bool f8, bool a_mn, bool b_mn, int m) {
    return (1u << 4) | ((f8 ? 0u : 1u) << 7) | ((f8 ? 0u : 1u) << 10) | ((a_mn ? 1u : 0u) << 15) |
           ((b_mn ? 1u : 0u) << 16) | (uint32_t(BN >> 3) << 17) | (uint32_t(m >> 4) << 24);
}

template <bool kF8, bool kAMN, bool kBMN, bool kOutBf16, int kCta>
__global__ void __launch_bounds__(THREADS, 1)
gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b, Params P) {
    using G = Geo<kCta>;
    constexpr int STAGES = G::STAGES;
    constexpr int STAGE_BYTES = G::STAGE_BYTES;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int ESZ = kF8 ? 1 : 2;
    constexpr int BK = BKB / ESZ;                  // K elements per stage
    constexpr int UK = 32 / ESZ;                   // K elements per MMA (32 bytes)
    const int ntiles = P.tiles_m * P.tiles_n;
    const uint32_t rank = kCta == 2 ? cluster_rank() : 0u;
    const int tile0 = blockIdx.x / kCta, tstep = gridDim.x / kCta;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4 * kCta);   // one arrive per epilogue warp of the pair
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        if (kCta == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        }
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
    }
    tc_fence_before();
    if (kCta == 2) cluster_sync_all();   // barriers initialised in both CTAs before any remote use
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------ TMA producer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = tile0; tile < ntiles; tile += tstep) {
                const int mb = tile % P.tiles_m, nb = tile / P.tiles_m;
                const int m0 = mb * G::TILE_M + int(rank) * BM;     // this CTA's A rows
                const int n0 = nb * BN + int(rank) * G::BN_L;       // this CTA's B rows
                for (int kb = 0; kb < P.k_blocks; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1u);
                    uint8_t* sa = smem + stage * STAGE_BYTES;
                    uint8_t* sb = sa + A_BYTES;
                    const int k0 = kb * BK;
                    if (kCta == 1) {
                        mbar_expect_tx(&full[stage], STAGE_BYTES);
                        if (!kAMN) {
                            tma_load_2d(sa, &map_a, k0, m0, &full[stage]);
                        } else {
#pragma unroll
                            for (int c = 0; c < BM * ESZ / 128; ++c)
                                tma_load_2d(sa + c * BK * 128, &map_a, m0 + c * (128 / ESZ), k0, &full[stage]);
                        }
                        if (!kBMN) {
                            tma_load_2d(sb, &map_b, k0, n0, &full[stage]);
                        } else {
#pragma unroll
                            for (int c = 0; c < G::BN_L * ESZ / 128; ++c)
                                tma_load_2d(sb + c * BK * 128, &map_b, n0 + c * (128 / ESZ), k0, &full[stage]);
                        }
                    } else {
                        // the leader's full barrier counts both CTAs' bytes
                        if (rank == 0) mbar_expect_tx(&full[stage], 2 * STAGE_BYTES);
                        const uint32_t fb = cluster_addr(&full[stage], 0);
                        if (!kAMN) {
                            tma_load_2d_pair(sa, &map_a, k0, m0, fb);
                        } else {
#pragma unroll
                            for (int c = 0; c < BM * ESZ / 128; ++c)
                                tma_load_2d_pair(sa + c * BK * 128, &map_a, m0 + c * (128 / ESZ), k0, fb);
                        }
                        if (!kBMN) {
                            tma_load_2d_pair(sb, &map_b, k0, n0, fb);
                        } else {
#pragma unroll
                            for (int c = 0; c < G::BN_L * ESZ / 128; ++c)
                                tma_load_2d_pair(sb + c * BK * 128, &map_b, n0 + c * (128 / ESZ), k0, fb);
                        }
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------ MMA issuer (pair: leader only)
        if (lane == 0 && rank == 0) {
            constexpr uint32_t idesc = instr_desc(kF8, kAMN, kBMN, G::TILE_M);
            // per-MMA K advance inside a stage (bytes): K-major +32 B, MN-major +UK rows of 128 B
            constexpr uint32_t a_step = kAMN ? UK * 128 : 32;
            constexpr uint32_t b_step = kBMN ? UK * 128 : 32;
            constexpr uint32_t a_lbo = kAMN ? BK * 128 : 16;
            constexpr uint32_t b_lbo = kBMN ? BK * 128 : 16;
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int tile = tile0; tile < ntiles; tile += tstep) {
                mbar_wait(&tempty[acc], acc_phase ^ 1u);
                tc_fence_after();
                const uint32_t tmem_d = tmem_base + uint32_t(acc * ACC_COLS);
                for (int kb = 0; kb < P.k_blocks; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
                    const uint32_t sb = sa + A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < BK / UK; ++kk) {
                        const uint64_t ad = smem_desc(sa + kk * a_step, a_lbo, 1024);
                        const uint64_t bd = smem_desc(sb + kk * b_step, b_lbo, 1024);
                        tc_mma<kF8, kCta>(tmem_d, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
                    }
                    // frees the smem stage (in both CTAs) when these MMAs retire
                    if (kCta == 1) tc_commit(&empty[stage]);
                    else tc_commit_pair(&empty[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                // accumulator ready for the epilogue(s)
                if (kCta == 1) tc_commit(&tfull[acc]);
                else tc_commit_pair(&tfull[acc]);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1u;
                }
            }
        }
    } else {
        // ------------------------------------------------------ epilogue (warps 2..5)
        const int q = warp & 3;                    // TMEM lane quarter this warp may access
        const int row_in_tile = int(rank) * BM + q * 32 + lane;
        const uint32_t tempty_leader0 = kCta == 2 ? cluster_addr(&tempty[0], 0) : 0u;
        float alpha = P.alpha;
        if (P.scale_a) alpha = __fmul_rn(alpha, bf16_bits_to_float(*P.scale_a));
        if (P.scale_b) alpha = __fmul_rn(alpha, bf16_bits_to_float(*P.scale_b));
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int tile = tile0; tile < ntiles; tile += tstep) {
            const int mb = tile % P.tiles_m, nb = tile / P.tiles_m;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int row = mb * G::TILE_M + row_in_tile;
            const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * ACC_COLS);
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t r[32];
                tmem_ld32(taddr + uint32_t(c * 32), r);
                tmem_wait_ld();
                const int col0 = nb * BN + c * 32;
                if (row < P.M) {
                    if (!kOutBf16) {
                        float* o = static_cast<float*>(P.out) + int64_t(row) * P.ldo + col0;
                        if (col0 + 32 <= P.N) {
#pragma unroll
                            for (int i = 0; i < 32; i += 4)
                                *reinterpret_cast<float4*>(o + i) =
                                    make_float4(__fmul_rn(alpha, u2f(r[i])), __fmul_rn(alpha, u2f(r[i + 1])),
                                                __fmul_rn(alpha, u2f(r[i + 2])), __fmul_rn(alpha, u2f(r[i + 3])));
                        } else {
#pragma unroll
                            for (int i = 0; i < 32; ++i)
                                if (col0 + i < P.N) o[i] = __fmul_rn(alpha, u2f(r[i]));
                        }
                    } else {
                        uint16_t* o = static_cast<uint16_t*>(P.out) + int64_t(row) * P.ldo + col0;
                        if (col0 + 32 <= P.N) {
#pragma unroll
                            for (int i = 0; i < 32; i += 8) {
                                uint32_t w[4];
#pragma unroll
                                for (int j = 0; j < 4; ++j)
                                    w[j] = (f2u(round_bf16(__fmul_rn(alpha, u2f(r[i + 2 * j])))) >> 16) |
                                           (f2u(round_bf16(__fmul_rn(alpha, u2f(r[i + 2 * j + 1])))) & 0xFFFF0000u);
                                *reinterpret_cast<uint4*>(o + i) = make_uint4(w[0], w[1], w[2], w[3]);
                            }
                        } else {
#pragma unroll
                            for (int i = 0; i < 32; ++i)
                                if (col0 + i < P.N) o[i] = uint16_t(f2u(round_bf16(__fmul_rn(alpha, u2f(r[i])))) >> 16);
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (kCta == 1) mbar_arrive(&tempty[acc]);
                else mbar_arrive_cluster(tempty_leader0 + uint32_t(acc * sizeof(uint64_t)));
            }
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1u;
            }
        }
    }
    tc_fence_before();
    if (kCta == 2) cluster_sync_all();   // no CTA of the pair leaves while the other may still signal it
    else __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        if (kCta == 1)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
        else
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
    }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// 2-D tensor map over a row-major matrix [rows][cols] of `esz`-byte elements,
// box = (box_cols, box_rows), 128B swizzle, zero fill out of bounds.
bool make_map(CUtensorMap* m, const void* base, int esz, int64_t rows, int64_t cols, int box_cols, int box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    const cuuint64_t strides[1] = {cuuint64_t(cols) * cuuint64_t(esz)};
    const cuuint32_t box[2] = {cuuint32_t(box_cols), cuuint32_t(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(m, esz == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 2,
                          const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <bool kF8, bool kAMN, bool kBMN, bool kOutBf16, int kCta>
cudaError_t run_cta(const void* a, const void* b, int M, int N, int K, float alpha, const uint16_t* sa,
                    const uint16_t* sb, void* out, int64_t ldo, cudaStream_t stream) {
    using G = Geo<kCta>;
    constexpr int ESZ = kF8 ? 1 : 2;
    constexpr int BK = BKB / ESZ;
    CUtensorMap ma, mb;
    // A logical [M x K]: K-major memory [M][K]; MN-major memory [K][M]
    const bool ok_a = !kAMN ? make_map(&ma, a, ESZ, M, K, BK, BM) : make_map(&ma, a, ESZ, K, M, 128 / ESZ, BK);
    const bool ok_b =
        !kBMN ? make_map(&mb, b, ESZ, N, K, BK, G::BN_L) : make_map(&mb, b, ESZ, K, N, 128 / ESZ, BK);
    if (!ok_a || !ok_b) return cudaErrorInvalidValue;
    auto kern = gemm_kernel<kF8, kAMN, kBMN, kOutBf16, kCta>;
    static int attr_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (attr_dev != dev) {
        const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM_BYTES);
        if (e != cudaSuccess) return e;
        attr_dev = dev;
    }
    Params P;
    P.M = M;
    P.N = N;
    P.K = K;
    P.tiles_m = (M + G::TILE_M - 1) / G::TILE_M;
    P.tiles_n = (N + BN - 1) / BN;
    P.k_blocks = (K + BK - 1) / BK;
    P.alpha = alpha;
    P.scale_a = sa;
    P.scale_b = sb;
    P.out = out;
    P.ldo = ldo;
    const int ntiles = P.tiles_m * P.tiles_n;
    const int units = device_sm_count() / kCta;   // persistent: one CTA (pair) per SM (TPC)
    const int grid = kCta * (ntiles < units ? ntiles : units);
    if (kCta == 1) {
        kern<<<grid, THREADS, G::SMEM_BYTES, stream>>>(ma, mb, P);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = G::SMEM_BYTES;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, ma, mb, P);
}

// COAT_GEMM_CTA=1 forces the single-CTA kernel (A/B comparisons).
inline int pair_mode() {
    static const int v = [] {
        const char* e = getenv("COAT_GEMM_CTA");
        return (e && e[0] == '1') ? 1 : 2;
    }();
    return v;
}

template <bool kF8, bool kAMN, bool kBMN, bool kOutBf16>
cudaError_t run(const void* a, const void* b, int M, int N, int K, float alpha, const uint16_t* sa,
                const uint16_t* sb, void* out, int64_t ldo, cudaStream_t stream) {
    if (M > BM && pair_mode() == 2)
        return run_cta<kF8, kAMN, kBMN, kOutBf16, 2>(a, b, M, N, K, alpha, sa, sb, out, ldo, stream);
    return run_cta<kF8, kAMN, kBMN, kOutBf16, 1>(a, b, M, N, K, alpha, sa, sb, out, ldo, stream);
}

}  // namespace gemm

// y[M,N] (fp32) = (s_x s_w) * codes_x[M,K] . codes_w[K,N]   (W row-major (K,N): MN-major B)
cudaError_t launch_fp8_linear_fwd(const uint8_t* xc, const uint16_t* sx, const uint8_t* wc, const uint16_t* sw, int M,
                                  int K, int N, float* y, cudaStream_t st) {
    return gemm::run<true, false, true, false>(xc, wc, M, N, K, 1.0f, sx, sw, y, N, st);
}
// dX[M,K] (bf16) = s_w * dY[M,N] . Wd[K,N]^T    (Wd = decoded W codes in bf16, exact; B K-major)
cudaError_t launch_linear_dgrad(const uint16_t* dy, const uint16_t* wd, const uint16_t* sw, int M, int K, int N,
                                uint16_t* dx, cudaStream_t st) {
    return gemm::run<false, false, false, true>(dy, wd, M, K, N, 1.0f, sw, nullptr, dx, K, st);
}
// dW[K,N] (fp32) = s_x * Xd[M,K]^T . dY[M,N]     (A = Xd MN-major, B = dY MN-major)
cudaError_t launch_linear_wgrad(const uint16_t* xd, const uint16_t* sx, const uint16_t* dy, int M, int K, int N,
                                float* dw, cudaStream_t st) {
    return gemm::run<false, true, true, false>(xd, dy, K, N, M, 1.0f, sx, nullptr, dw, N, st);
}

}  // namespace coat
