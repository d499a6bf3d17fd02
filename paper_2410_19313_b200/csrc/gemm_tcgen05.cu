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
//   warp 1: TMEM allocator + MMA issuer (the warp  tcgen05.mma + tcgen05.commit
//           runs the loop, elect.sync issues)
//   warps 2-5 (2-17 for the gate/up epilogue):    double-buffered accumulator
//           epilogue, tcgen05.ld -> fp32 output by TMA bulk-tensor stores from
//           swizzled staging tiles (writes spread over the next main loop), or
//           bf16 / per-group 1x16 codes / the gate/up SiLU*mul quantizers
// Tiles are walked in groups of 8 M blocks (the CTAs in flight share operands
// in L2).  Variants (kCta):
//   1: one CTA per SM, 128 x 256 tile, cta_group::1 (small M).
//   2: a CTA pair on the two SMs of a TPC (cluster of 2), 256 x 256 tile,
//      tcgen05.mma.cta_group::2 issued by the leader.  Each CTA stages only its
//      128 rows of A and its 128-column half of B (32 KB per stage instead of
//      48 KB for half the FLOPs), so the L2->SM operand traffic per FLOP drops
//      by a third -- the 1-CTA kernel is operand-bandwidth bound at ~70% of the
//      tensor pipe.  Both CTAs' TMA bytes land on the leader's full barrier
//      (.cta_group::2 TMA, mapa address); commits multicast to both CTAs; both
//      CTAs' epilogues arrive on the leader's TMEM-empty barrier.
//   4: two CTA pairs per cluster sharing B by TMA multicast (COAT_GEMM_CTA=4;
//      parity-tested, measured slower -- DESIGN.md K4).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstring>
#include <cstdlib>
#include <mutex>

#include "act_quant.cuh"
#include "coat_device.cuh"
#include "coat_internal.h"

namespace coat {
namespace gemm {

constexpr int BM = 128;                   // accumulator rows per CTA (TMEM lanes)
constexpr int BN = 256;                   // accumulator columns (MMA N)
constexpr int BKB = 128;                  // K bytes per stage (one 128B swizzle row)
constexpr int A_BYTES = BM * BKB;         // 16 KiB
// Epilogue warps: 4 (one per TMEM lane quarter) -- or 16 for the quantizing
// gate/up epilogue, whose per-element work (three quantizers + SiLU) is longer
// than the MMA main loop of a tile with 4 warps (ncu: tensor pipe 62%); each
// group of four takes a quarter of the accumulator's columns.  (8 warps for
// the plain epilogues measured +-0.)
#ifndef COAT_GEMM_UPGATE_EPI
#define COAT_GEMM_UPGATE_EPI 16
#endif
template <int kOut>
__host__ __device__ constexpr int epi_warps() {
    return kOut == 3 ? COAT_GEMM_UPGATE_EPI : 4;
}
template <int kOut>
__host__ __device__ constexpr int threads_for() { return 64 + 32 * epi_warps<kOut>(); }
// fp32 epilogue through a per-warp shared-memory tile (coalesced row stores)
#ifndef COAT_GEMM_COALESCED
#define COAT_GEMM_COALESCED 1
#endif
// fp32 epilogue by TMA bulk-tensor stores from a swizzled 32 x 32 staging
// tile per warp (double-buffered) instead of STG
#ifndef COAT_GEMM_TMA_STORE
#define COAT_GEMM_TMA_STORE 1
#endif
template <int kOut>
__host__ __device__ constexpr bool tma_store() {
    return (kOut == 0 || kOut == 1) && COAT_GEMM_TMA_STORE;   // fp32 (128B swizzle) / bf16 (64B swizzle)
}
// Gate/up epilogue staging (see the kernel): per TMEM lane quarter and output
// array (silu.in, mul.in.silu, mul.in.up) a 32-row x 128-byte code tile
// (128B-swizzled, 1 KB aligned) and a 32-row x 16-byte scale tile.
constexpr int kUgCodeTile = 32 * 128, kUgScaleTile = 32 * 16;
constexpr int kUgStageBytes = 12 * kUgCodeTile + 12 * kUgScaleTile;
// 1x16 epilogue staging per warp: its 32 rows x 256 codes as two 128B-swizzled
// 32 x 128-byte tiles, and 32 rows x 16 scales (32 bytes)
constexpr int kQ16StageBytes = 2 * kUgCodeTile + 32 * 32;
template <int kOut>
__host__ __device__ constexpr int epi_smem_bytes() {
    // TMA store: the staging tiles start at the next 1 KB boundary after the barriers
    return tma_store<kOut>() ? 768 + epi_warps<kOut>() * 2 * 4096
           : kOut == 3       ? 768 + kUgStageBytes
           : kOut == 2       ? 768 + epi_warps<kOut>() * kQ16StageBytes
           : (kOut == 0 && COAT_GEMM_COALESCED) ? epi_warps<kOut>() * 32 * 36 * 4 : 0;
}
constexpr int ACC_COLS = BN;              // fp32 columns per accumulator
constexpr int TMEM_COLS = 2 * ACC_COLS;   // double buffer = all 512 columns

// kCta: 1 = one CTA, 2 = a CTA pair, 4 = two CTA pairs in a cluster of 4 that
// share the B tile (same N block, adjacent M blocks): each CTA loads half of
// its B half and multicasts it to the same-rank CTA of the other pair, so the
// L2 -> SM operand traffic per FLOP drops by another quarter.
template <int kCta, int kOut = 0>
struct Geo {
    static constexpr int PAIR = kCta >= 2 ? 2 : 1;         // CTAs per MMA
    static constexpr int BN_L = BN / PAIR;                 // B rows staged by this CTA
    static constexpr int B_BYTES = BN_L * BKB;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
#ifndef COAT_GEMM_PAIR_STAGES
#define COAT_GEMM_PAIR_STAGES 6
#endif
    // the gate/up kernel gives one stage to its epilogue staging tiles
    static constexpr int STAGES =
        kCta >= 2 ? ((kOut == 3 || kOut == 2) ? 5 : COAT_GEMM_PAIR_STAGES) : ((kOut == 3 || kOut == 2) ? 3 : 4);
    static constexpr int TILE_M = BM * PAIR;
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

// Epilogue kinds.
enum : int {
    kOutF32 = 0,      // out fp32 [M, N]
    kOutBf16 = 1,     // out bf16 [M, N]
    kOutQ16 = 2,      // per-group (1x16) E4M3 codes + BF16 scales of y (quantize(y, per_group(16)))
    kOutUpGate = 3,   // the fused gate/up projection + SiLU*mul quantizers (see EpiQ)
};

// Quantizing epilogues (kOutQ16 / kOutUpGate).  Row strides: ldc codes per row
// (= N), ldc / 16 scales per row.
//   kOutQ16:    c0/s0 = Q_g16(y);  y0 (may be NULL) = y (fp32)
//   kOutUpGate: B = [W_gate | W_up] per 128-column block (tile n covers gate and
//               up columns [128n, 128n+128)); with g = y_gate, u = y_up:
//               c0/s0 = Q_g16(g) (silu.in), c1/s1 = Q_g16(silu(DQ(c0))) (mul.in.silu),
//               c2/s2 = Q_g16(u) (mul.in.up), *amax_bits = max |DQ(c1) * DQ(c2)|
//               (NaN ignored) for the per-tensor down.in pass; y0 / y1 (may be
//               NULL) = g / u (fp32)
struct EpiQ {
    uint8_t* c0; uint16_t* s0;
    uint8_t* c1; uint16_t* s1;
    uint8_t* c2; uint16_t* s2;
    float* y0; float* y1;
    const uint16_t* scale_b1;   // BF16 device scale of W_up (kOutUpGate)
    uint32_t* amax_bits;
    uint32_t* flags;            // kFlagNonFiniteInput (quantize.cpp:91)
    int64_t ldc;
};

// kOutUpGate with P.ug_tma: TMA store maps of the three code arrays (uint8
// [M, ldc], 128 x 32 boxes, 128B swizzle) and their scale arrays (bf16
// [M, ldc / 16], 8 x 32 boxes)
struct EpiMaps {
    CUtensorMap c[3];
    CUtensorMap s[3];
};

struct Params {
    int M, N, K;               // K in elements
    int tiles_m, tiles_n, k_blocks;
    int group_m;               // tile raster: groups of group_m M-blocks, M fastest inside a group
    float alpha;               // epilogue scale
    const uint16_t* scale_a;   // optional BF16 device scalars multiplied into alpha
    const uint16_t* scale_b;
    void* out;
    int64_t ldo;               // elements
    int tma_out;               // kOutF32 with tma_store(): map_b2 is the output's tensor map
    int ug_tma;                // kOutUpGate / kOutQ16: codes and scales through the staging tiles + emaps
    unsigned epi_pause_ns;     // pause between a warp's epilogue chunks (see epi_pause_ns())
    EpiQ q;
};

// Grouped raster of the persistent tile walk: tiles [g * group_m * tiles_n, ...)
// cover M-blocks [g * group_m, +group_m) x every N-block, M fastest.  The
// CTAs in flight at any moment then cover ~group_m M-blocks x (units /
// group_m) N-blocks instead of every M-block of one or two N columns -- with a
// long K (dgrad: 13824) a 256-row operand block is 7 MB, and the M-fastest
// walk streamed all of dY from DRAM once per wave (ncu: 2.4 GB read vs
// cuBLAS's 0.93 GB on the same shape, and the extra DRAM power cost ~12% of
// the clock).
__device__ __forceinline__ void tile_coords(const Params& P, int tile, int& mb, int& nb) {
    const int span = P.group_m * P.tiles_n;
    const int g = tile / span, r = tile - g * span;
    const int m_first = g * P.group_m;
    const int gm = min(P.tiles_m - m_first, P.group_m);
    nb = r / gm;
    mb = m_first + (r - nb * gm);
#ifndef COAT_GEMM_NO_SNAKE
    // odd groups walk N backwards, so the B blocks at a group seam are still in
    // L2 (ncu, cfg4 dgrad: DRAM reads 1.306 -> 1.219 GB, 723 -> 718 us)
    if (g & 1) nb = P.tiles_n - 1 - nb;
#endif
}

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
#ifdef COAT_GEMM_DEBUG_WAIT
// debug build: bounded waits that report the stuck barrier and trap
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    for (long long i = 0;; ++i) {
        uint32_t ok;
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok) return;
        if (i == (1ll << 24)) {
            uint32_t cr;
            asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(cr));
            printf("stuck: block %d crank %u thread %d bar smem+%u parity %u\n", blockIdx.x, cr, threadIdx.x,
                   smem_u32(bar), parity);
            __trap();
        }
    }
}
#else
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
#endif
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
// one lane of the (converged) warp -- the lowest, so always the same one
__device__ __forceinline__ bool elect_one() {
    uint32_t p;
    asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n" : "=r"(p));
    return p != 0;
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
// The same into the CTAs of `mask` (same smem offset in each); the completion
// bytes land on the barrier of each destination's pair leader.  The mbarrier
// operand is this CTA's own barrier address with the peer bit (bit 24 of a
// shared-window address: the odd CTA of a pair) cleared -- without the mask an
// odd CTA's bytes would count on its own barrier, which nobody waits on.
__device__ __forceinline__ void tma_load_2d_pair_mc(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar,
                                                    uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar) & 0xFEFFFFFFu), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar, uint16_t mask = 3) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
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
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
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

// Per-group (1x16) quantization of one 16-column group of y held by this
// thread (quantize.cpp:89-111 with G = 16: NaN/Inf -> non-finite flag).
__device__ __forceinline__ uint32_t quant16(const aq::Chunk16& y, uint4& cw, uint16_t& sbits, float nz) {
    float m = aq::fmax3_nan_(fabsf(y.v[0]), fabsf(y.v[1]), fabsf(y.v[2]));
#pragma unroll
    for (int i = 3; i < 15; i += 2) m = aq::fmax3_nan_(m, fabsf(y.v[i]), fabsf(y.v[i + 1]));
    m = aq::fmax3_nan_(m, fabsf(y.v[15]), 0.0f);
    float s, rs;
    aq::group_scale_fast(f2u(m), s, rs);
    cw = aq::encode16(y, s, rs, nz);
    sbits = float_to_bf16_bits_exact(s);
    return f2u(m) >= 0x7F800000u ? 1u : 0u;
}

// fp32 output row segment store.  COAT_GEMM_STORE_HINT: 0 plain, 1 streaming
// (.cs), 2 L2 evict_first policy -- the output is written once and never
// re-read by the kernel, so it should not displace the A / B operands in L2.
#ifndef COAT_GEMM_STORE_HINT
#define COAT_GEMM_STORE_HINT 0
#endif
__device__ __forceinline__ void st_out4(float* p, const float4& v, uint64_t policy) {
#if defined(COAT_GEMM_DIAG_NOSTG)
    if (v.x == 1.2345e-38f) *reinterpret_cast<float4*>(p) = v;   // measurement only: (almost) no stores
#elif COAT_GEMM_STORE_HINT == 1
    asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
#elif COAT_GEMM_STORE_HINT == 2
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x),
                 "f"(v.y), "f"(v.z), "f"(v.w), "l"(policy)
                 : "memory");
#else
    (void)policy;
    *reinterpret_cast<float4*>(p) = v;
#endif
}

template <bool kF8, bool kAMN, bool kBMN, int kOut, int kCta>
__global__ void __launch_bounds__(threads_for<kOut>(), 1)
gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
            const __grid_constant__ CUtensorMap map_b2, const __grid_constant__ EpiMaps emaps, Params P) {
    static_assert(kOut != kOutUpGate || (kF8 && kBMN), "gate/up epilogue: FP8 forward, W (K, N) row-major");
    using G = Geo<kCta, kOut>;
    constexpr int STAGES = G::STAGES;
    constexpr int STAGE_BYTES = G::STAGE_BYTES;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
#ifdef COAT_GEMM_DEBUG_WAIT
    if (blockIdx.x == 0 && threadIdx.x == 0)
        printf("barriers: full %u empty %u tfull %u tempty %u (stages %d)\n", smem_u32(full), smem_u32(empty),
               smem_u32(tfull), smem_u32(tempty), STAGES);
#endif

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int ESZ = kF8 ? 1 : 2;
    constexpr int BK = BKB / ESZ;                  // K elements per stage
    constexpr int UK = 32 / ESZ;                   // K elements per MMA (32 bytes)
    const int ntiles = P.tiles_m * P.tiles_n;
    const uint32_t crank = kCta >= 2 ? cluster_rank() : 0u;
    const uint32_t rank = crank & 1u;          // rank inside the CTA pair
    const uint32_t pidx = crank >> 1;          // kCta 4: which pair of the cluster
    const int tile0 = blockIdx.x / kCta, tstep = gridDim.x / kCta;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kCta == 4 ? 2 : 1);   // kCta 4: both pairs' MMAs read the B halves
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], epi_warps<kOut>() * G::PAIR);   // one arrive per epilogue warp of the pair
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
    if (kCta >= 2) cluster_sync_all();   // barriers initialised in every CTA before any remote use
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------ TMA producer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = tile0; tile < ntiles; tile += tstep) {
                int mb, nb;
                tile_coords(P, tile, mb, nb);
                if (kCta == 4) mb = 2 * mb + int(pidx);
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
                        if (kOut == kOutUpGate) {
                            // gate columns then up columns of the same 128-column block
                            tma_load_2d(sb, &map_b, nb * 128, k0, &full[stage]);
                            tma_load_2d(sb + BK * 128, &map_b2, nb * 128, k0, &full[stage]);
                        } else if (!kBMN) {
                            tma_load_2d(sb, &map_b, k0, n0, &full[stage]);
                        } else {
#pragma unroll
                            for (int c = 0; c < G::BN_L * ESZ / 128; ++c)
                                tma_load_2d(sb + c * BK * 128, &map_b, n0 + c * (128 / ESZ), k0, &full[stage]);
                        }
                    } else if (kCta == 4) {
                        // the pair leader's full barrier counts both CTAs' bytes: own A rows,
                        // B half = this CTA's quarter + the other pair's same-rank CTA's quarter
                        if (rank == 0) mbar_expect_tx(&full[stage], 2 * STAGE_BYTES);
                        const uint32_t fb = cluster_addr(&full[stage], crank & ~1u);
                        const uint16_t mc = uint16_t((1u << rank) | (1u << (2 + rank)));
                        if (!kAMN) {
                            tma_load_2d_pair(sa, &map_a, k0, m0, fb);
                        } else {
#pragma unroll
                            for (int c = 0; c < BM * ESZ / 128; ++c)
                                tma_load_2d_pair(sa + c * BK * 128, &map_a, m0 + c * (128 / ESZ), k0, fb);
                        }
                        if (!kBMN) {
                            constexpr int h = G::BN_L / 2;   // B rows per quarter
                            tma_load_2d_pair_mc(sb + int(pidx) * h * 128, &map_b, k0, n0 + int(pidx) * h, &full[stage],
                                                mc);
                        } else {
                            constexpr int h = BK / 2;        // K rows per quarter of each 128-byte column chunk
#pragma unroll
                            for (int c = 0; c < G::BN_L * ESZ / 128; ++c)
                                tma_load_2d_pair_mc(sb + c * BK * 128 + int(pidx) * h * 128, &map_b,
                                                    n0 + c * (128 / ESZ), k0 + int(pidx) * h, &full[stage], mc);
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
                        if (kOut == kOutUpGate) {
                            // the leader stages the gate columns, its partner the up columns
                            tma_load_2d_pair(sb, rank == 0 ? &map_b : &map_b2, nb * 128, k0, fb);
                        } else if (!kBMN) {
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
        // The whole warp runs the loop (warp-uniform control flow, so the
        // descriptors live in uniform registers); one elected lane -- always
        // the same, lane 0 -- issues the MMAs and their commits.  A single-lane
        // loop made the compiler wrap every tcgen05.mma in an elect / R2UR
        // broadcast sequence (~23 SASS instructions per MMA), slow enough that
        // the epilogue warp sharing the scheduler pushed it past the MMA time.
        if (rank == 0) {
            constexpr uint32_t idesc = instr_desc(kF8, kAMN, kBMN, G::TILE_M);
            // per-MMA K advance inside a stage (bytes): K-major +32 B, MN-major +UK rows of 128 B
            constexpr uint32_t a_step = kAMN ? UK * 128 : 32;
            constexpr uint32_t b_step = kBMN ? UK * 128 : 32;
            constexpr uint32_t a_lbo = kAMN ? BK * 128 : 16;
            constexpr uint32_t b_lbo = kBMN ? BK * 128 : 16;
            // stage-0 descriptors; a stage / K step only adds to the address field
            // (bits 0-13 = address >> 4; every smem address < 256 KB, so no carry)
            const uint64_t adesc0 = smem_desc(smem_u32(smem), a_lbo, 1024);
            const uint64_t bdesc0 = smem_desc(smem_u32(smem) + A_BYTES, b_lbo, 1024);
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
                    const uint64_t so = uint64_t(uint32_t(stage * STAGE_BYTES) >> 4);
                    if (elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < BK / UK; ++kk)
                            tc_mma<kF8, kCta>(tmem_d, adesc0 + so + uint64_t((kk * a_step) >> 4),
                                              bdesc0 + so + uint64_t((kk * b_step) >> 4), idesc,
                                              (kb | kk) != 0 ? 1u : 0u);
                        // frees the smem stage (in both CTAs) when these MMAs retire
                        if (kCta == 1) tc_commit(&empty[stage]);
                        else tc_commit_pair(&empty[stage], kCta == 4 ? uint16_t(0xF) : uint16_t(3));
                    }
                    __syncwarp();
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }

                // accumulator ready for the epilogue(s)
                if (elect_one()) {
                    if (kCta == 1) tc_commit(&tfull[acc]);
                    else tc_commit_pair(&tfull[acc], uint16_t(3u << (2 * pidx)));
                }
                __syncwarp();
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1u;
                }
            }
        }
    } else {
        // ------------------------------------------------------ epilogue (warps 2 .. 1 + epi_warps)
        const int q = warp & 3;                    // TMEM lane quarter this warp may access
        const int half = (warp - 2) >> 2;          // which column part (epi_warps / 4 parts)
        const int row_in_tile = int(rank) * BM + q * 32 + lane;
        // kOutF32: this warp's 32 x 36-float staging tile behind the barriers
        const uint32_t stile = smem_u32(smem + STAGES * STAGE_BYTES + 256) + uint32_t((warp - 2) * (32 * 36) * 4);
        // tma_store(): this warp's two 4 KB swizzled staging tiles (1 KB aligned)
        const uint32_t ttile = smem_u32(smem + STAGES * STAGE_BYTES + 1024) + uint32_t((warp - 2) * 8192);
        uint32_t tbuf = 0;
        const uint32_t tempty_leader0 = kCta >= 2 ? cluster_addr(&tempty[0], crank & ~1u) : 0u;
        float alpha = P.alpha;
        if (P.scale_a) alpha = __fmul_rn(alpha, bf16_bits_to_float(*P.scale_a));
        float alpha_u = alpha;
        if (P.scale_b) alpha = __fmul_rn(alpha, bf16_bits_to_float(*P.scale_b));
        if (kOut == kOutUpGate && P.q.scale_b1) alpha_u = __fmul_rn(alpha_u, bf16_bits_to_float(*P.q.scale_b1));
        uint64_t out_policy;
        asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(out_policy));
        uint32_t bad = 0;
        float amp = 0.0f;   // kOutUpGate: max |product| (max.f32: NaN ignored, Inf kept)
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int tile = tile0; tile < ntiles; tile += tstep) {
            int mb, nb;
            tile_coords(P, tile, mb, nb);
            if (kCta == 4) mb = 2 * mb + int(pidx);
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int row = mb * G::TILE_M + row_in_tile;
            const int row_base = row - lane;   // the warp's first accumulator row
            const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * ACC_COLS);
            if (kOut == kOutUpGate) {
                // accumulator columns [0, 128): gate, [128, 256): up, of output columns nb*128 + j
                const bool live = row < P.M;
                const int64_t rq = live ? row : 0;
                constexpr int kGroups = 8 * 4 / epi_warps<kOut>();   // 16-column groups per warp (of 8 per half)
                // P.ug_tma: the four warps of this TMEM lane quarter put their codes and
                // scales into the quarter's staging tiles, and one of them writes each
                // tile to HBM with a TMA store (32 rows x 128 B of codes per array, whole
                // row segments) instead of 32 scattered 16-byte and 2-byte stores per
                // warp instruction (the scattered stores cost the kernel ~14%: ncu, with
                // them removed, 727 vs 843 us, tensor pipe 98 vs 86%)
                const uint32_t ug_code = smem_u32(smem + STAGES * STAGE_BYTES + 1024) + uint32_t(q * 3 * kUgCodeTile);
                const uint32_t ug_scale = smem_u32(smem + STAGES * STAGE_BYTES + 1024) + uint32_t(12 * kUgCodeTile) +
                                          uint32_t(q * 3 * kUgScaleTile);
                const bool ug_issuer = half == 0 && lane == 0;
                auto ug_put = [&](int a, int gi, const uint4& cw, uint16_t sbits) {
                    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(
                                     ug_code + uint32_t(a * kUgCodeTile + lane * 128 + ((gi ^ (lane & 7)) << 4))),
                                 "r"(cw.x), "r"(cw.y), "r"(cw.z), "r"(cw.w)
                                 : "memory");
                    asm volatile("st.shared.u16 [%0], %1;" ::"r"(ug_scale + uint32_t(a * kUgScaleTile + lane * 16 + gi * 2)),
                                 "h"(sbits)
                                 : "memory");
                };
                if (P.ug_tma) {
                    // the previous tile's stores have read the staging tiles
                    if (ug_issuer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    asm volatile("bar.sync %0, %1;" ::"r"(1 + q), "n"(8 * epi_warps<kOut>()) : "memory");
                }
#pragma unroll 1
                for (int gi = half * kGroups; gi < (half + 1) * kGroups; ++gi) {
                    uint32_t rg[16], ru[16];
                    tmem_ld16(taddr + uint32_t(gi * 16), rg);
                    tmem_ld16(taddr + uint32_t(128 + gi * 16), ru);
                    tmem_wait_ld();
                    const int col = nb * 128 + gi * 16;
                    if (col >= P.N) break;   // warp-uniform (N % 16 == 0)
                    aq::Chunk16 gv, uv;
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        gv.v[i] = __fmul_rn(alpha, u2f(rg[i]));
                        uv.v[i] = __fmul_rn(alpha_u, u2f(ru[i]));
                    }
                    if (live && P.q.y0) {
                        float4* o = reinterpret_cast<float4*>(P.q.y0 + rq * P.q.ldc + col);
                        float4* o1 = reinterpret_cast<float4*>(P.q.y1 + rq * P.q.ldc + col);
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            o[k] = make_float4(gv.v[4 * k], gv.v[4 * k + 1], gv.v[4 * k + 2], gv.v[4 * k + 3]);
                            o1[k] = make_float4(uv.v[4 * k], uv.v[4 * k + 1], uv.v[4 * k + 2], uv.v[4 * k + 3]);
                        }
                    }
                    const int64_t co = rq * P.q.ldc + col, so = rq * (P.q.ldc >> 4) + (col >> 4);
                    uint4 cw;
                    uint16_t sbits;
                    float gam;
                    bad |= aq::quant_dq16(gv, cw, sbits, -0.0f, &gam);   // silu.in
                    if (P.ug_tma) ug_put(0, gi, cw, sbits);
                    else if (live) { *reinterpret_cast<uint4*>(P.q.c0 + co) = cw; P.q.s0[so] = sbits; }
                    aq::silu16(gv, -0.0f, gam);
                    bad |= aq::quant_dq16(gv, cw, sbits, -0.0f);   // mul.in.silu
                    if (P.ug_tma) ug_put(1, gi, cw, sbits);
                    else if (live) { *reinterpret_cast<uint4*>(P.q.c1 + co) = cw; P.q.s1[so] = sbits; }
                    bad |= aq::quant_dq16(uv, cw, sbits, -0.0f);   // mul.in.up
                    if (P.ug_tma) ug_put(2, gi, cw, sbits);
                    else if (live) { *reinterpret_cast<uint4*>(P.q.c2 + co) = cw; P.q.s2[so] = sbits; }
                    if (live) {
#pragma unroll
                        for (int i = 0; i < 16; i += 2) {
                            const F2 pr = f2_mul(F2{gv.v[i], gv.v[i + 1]}, F2{uv.v[i], uv.v[i + 1]}, -0.0f);
                            asm("max.f32 %0, %1, %2, %3;" : "=f"(amp) : "f"(amp), "f"(fabsf(pr.x)), "f"(fabsf(pr.y)));
                        }
                    }
                }
                if (P.ug_tma) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    asm volatile("bar.sync %0, %1;" ::"r"(1 + q), "n"(8 * epi_warps<kOut>()) : "memory");
                    if (ug_issuer) {
                        // rows >= M and columns >= N are clipped by the TMA unit
#pragma unroll
                        for (int a = 0; a < 3; ++a) {
                            asm volatile(
                                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                                    &emaps.c[a]),
                                "r"(nb * 128), "r"(row_base), "r"(ug_code + uint32_t(a * kUgCodeTile))
                                : "memory");
                            asm volatile(
                                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                                    &emaps.s[a]),
                                "r"(nb * 8), "r"(row_base), "r"(ug_scale + uint32_t(a * kUgScaleTile))
                                : "memory");
                        }
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                }
            } else {
            // kOutQ16 with P.ug_tma: this warp's staging tiles (free once its previous stores read them)
            const uint32_t q16_code = smem_u32(smem + STAGES * STAGE_BYTES + 1024) + uint32_t((warp - 2) * 2 * kUgCodeTile);
            const uint32_t q16_scale = smem_u32(smem + STAGES * STAGE_BYTES + 1024) +
                                       uint32_t(epi_warps<kOut>() * 2 * kUgCodeTile + (warp - 2) * 1024);
            if (kOut == kOutQ16 && P.ug_tma) {
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                __syncwarp();
            }
#pragma unroll 1
            for (int c = half * (BN / 32) * 4 / epi_warps<kOut>(); c < (half + 1) * (BN / 32) * 4 / epi_warps<kOut>();
                 ++c) {
                // spread the tile's output writes: a pause before every chunk but the first
                if (P.epi_pause_ns && c != half * (BN / 32) * 4 / epi_warps<kOut>()) __nanosleep(P.epi_pause_ns);
                uint32_t r[32];
                tmem_ld32(taddr + uint32_t(c * 32), r);
                tmem_wait_ld();
                const int col0 = nb * BN + c * 32;
#ifdef COAT_GEMM_DIAG_NOEPI
                // measurement only (wrong results): TMEM drained, nothing stored
                if (r[0] == 0x7fc00001u) bad |= 1u;
                continue;
#endif
                if (kOut == kOutQ16) {
                    const bool live = row < P.M;
                    const int64_t rq = live ? row : 0;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int col = col0 + h * 16;
                        if (col >= P.N) break;   // warp-uniform (N % 16 == 0)
                        aq::Chunk16 y;
#pragma unroll
                        for (int i = 0; i < 16; ++i) y.v[i] = __fmul_rn(alpha, u2f(r[16 * h + i]));
                        if (live && P.q.y0) {
                            float4* o = reinterpret_cast<float4*>(P.q.y0 + rq * P.q.ldc + col);
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                o[k] = make_float4(y.v[4 * k], y.v[4 * k + 1], y.v[4 * k + 2], y.v[4 * k + 3]);
                        }
                        uint4 cw;
                        uint16_t sbits;
                        bad |= quant16(y, cw, sbits, -0.0f) & (live ? 1u : 0u);
                        if (P.ug_tma) {
                            // staging: code chunk (col % 128) / 16 of tile col / 128, swizzled; scale col / 16
                            const int tcol = c * 32 + h * 16;   // column within the tile
                            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(
                                             q16_code + uint32_t((tcol >> 7) * kUgCodeTile + lane * 128 +
                                                                 ((((tcol & 127) >> 4) ^ (lane & 7)) << 4))),
                                         "r"(cw.x), "r"(cw.y), "r"(cw.z), "r"(cw.w)
                                         : "memory");
                            asm volatile("st.shared.u16 [%0], %1;" ::"r"(q16_scale + uint32_t(lane * 32 + (tcol >> 4) * 2)),
                                         "h"(sbits)
                                         : "memory");
                        } else if (live) {
                            *reinterpret_cast<uint4*>(P.q.c0 + rq * P.q.ldc + col) = cw;
                            P.q.s0[rq * (P.q.ldc >> 4) + (col >> 4)] = sbits;
                        }
                    }
                } else if (tma_store<kOut>() && P.tma_out) {
                    // rows / columns outside the output are clipped by the TMA unit
                    if (col0 < P.N && row_base < P.M) {
                        const uint32_t buf = ttile + (tbuf & 1u) * 4096u;
                        // the store issued from this buffer two chunks ago has read it
                        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                        __syncwarp();
                        if (kOut == kOutF32) {
#pragma unroll
                            for (int i = 0; i < 8; ++i)   // 16-byte chunk i of this lane's row, 128B-swizzled
                                asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                                                 buf + uint32_t(lane * 128 + ((i ^ (lane & 7)) << 4))),
                                             "f"(__fmul_rn(alpha, u2f(r[4 * i]))),
                                             "f"(__fmul_rn(alpha, u2f(r[4 * i + 1]))),
                                             "f"(__fmul_rn(alpha, u2f(r[4 * i + 2]))),
                                             "f"(__fmul_rn(alpha, u2f(r[4 * i + 3])))
                                             : "memory");
                        } else {
                            // bf16: a 32 x 32 box of 64-byte rows, 64B-swizzled (chunk i ^ ((row >> 1) & 3))
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                uint32_t w[4];
#pragma unroll
                                for (int j = 0; j < 4; ++j)
                                    w[j] = (f2u(round_bf16(__fmul_rn(alpha, u2f(r[8 * i + 2 * j])))) >> 16) |
                                           (f2u(round_bf16(__fmul_rn(alpha, u2f(r[8 * i + 2 * j + 1])))) & 0xFFFF0000u);
                                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(
                                                 buf + uint32_t(lane * 64 + ((i ^ ((lane >> 1) & 3)) << 4))),
                                             "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                                             : "memory");
                            }
                        }
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        __syncwarp();
                        if (lane == 0) {
                            asm volatile(
                                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                                    &map_b2),
#ifdef COAT_GEMM_DIAG_ALIAS
                                "r"(col0), "r"(row_base & 255), "r"(buf)   // measurement only: 256 output rows reused
#else
                                "r"(col0), "r"(row_base), "r"(buf)
#endif
                                : "memory");
                            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                        }
                        ++tbuf;
                    }
                } else if (kOut == kOutF32 && COAT_GEMM_COALESCED && col0 + 32 <= P.N && row_base + 32 <= P.M) {
                    // the warp's 32 rows x 32 columns through a padded shared-memory
                    // tile, so every store instruction writes 4 whole 128-byte row
                    // segments instead of one 16-byte piece of 32 different rows
                    // (row stride 36 floats: both access patterns bank-conflict free)
#pragma unroll
                    for (int i = 0; i < 32; i += 4)
                        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(stile + uint32_t((lane * 36 + i) * 4)),
                                     "f"(__fmul_rn(alpha, u2f(r[i]))), "f"(__fmul_rn(alpha, u2f(r[i + 1]))),
                                     "f"(__fmul_rn(alpha, u2f(r[i + 2]))), "f"(__fmul_rn(alpha, u2f(r[i + 3])))
                                     : "memory");
                    __syncwarp();
                    float* o = static_cast<float*>(P.out) + int64_t(row_base) * P.ldo + col0;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int rr = 4 * j + (lane >> 3), cc = (lane & 7) * 4;
                        float4 v;
                        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                                     : "r"(stile + uint32_t((rr * 36 + cc) * 4))
                                     : "memory");
                        st_out4(o + int64_t(rr) * P.ldo + cc, v, out_policy);
                    }
                    __syncwarp();
                } else if (row < P.M) {
                    if (kOut == kOutF32) {
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
            if (kOut == kOutQ16 && P.ug_tma) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    // rows >= M and columns >= N are clipped by the TMA unit
#pragma unroll
                    for (int t = 0; t < 2; ++t)
                        asm volatile(
                            "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                                &emaps.c[0]),
                            "r"(nb * BN + t * 128), "r"(row_base), "r"(q16_code + uint32_t(t * kUgCodeTile))
                            : "memory");
                    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                                     &emaps.s[0]),
                                 "r"(nb * (BN / 16)), "r"(row_base), "r"(q16_scale)
                                 : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
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
        if (kOut == kOutUpGate) {
            const uint32_t m = warp_max_u32(f2u(amp));
            if (lane == 0 && m) atomicMax(P.q.amax_bits, m);
        }
        if (kOut >= kOutQ16 && P.q.flags && __reduce_or_sync(0xFFFFFFFFu, bad) && lane == 0)
            atomicOr(P.q.flags, kFlagNonFiniteInput);
        if (tma_store<kOut>() && P.tma_out && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        if ((kOut == kOutUpGate || kOut == kOutQ16) && P.ug_tma && lane == 0)
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    tc_fence_before();
    if (kCta >= 2) cluster_sync_all();   // no CTA of the cluster leaves while another may still signal it
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
bool make_map(CUtensorMap* m, const void* base, int esz, int64_t rows, int64_t cols, int box_cols, int box_rows,
              int64_t ld = 0, int swizzle = 128) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    const cuuint64_t strides[1] = {cuuint64_t(ld ? ld : cols) * cuuint64_t(esz)};
    const cuuint32_t box[2] = {cuuint32_t(box_cols), cuuint32_t(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUtensorMapDataType dt = esz == 1   ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                   : esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                              : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    const CUresult r = fn(m, dt, 2,
                          const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          swizzle == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                          : swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                          : CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// Co-resident clusters of 4 (GPC boundaries leave some SMs out).
template <typename K>
int max_clusters4(K kern, int smem, int threads) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(4 * 64);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 4;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) n = 0;
    return n;
}

// Epilogue write spreading.  The CTAs finish their tiles in lock step, and the
// output writes of a whole tile leaving every SM at once compete with the next
// tile's operand loads (ncu: FP8 forward tensor pipe 88% with its fp32 output
// stores, 97% without; the SM -> L2 write traffic, not the DRAM write-back).
// A pause between a warp's 32-column chunks spreads the writes over the next
// main loop: k_blocks * COAT_GEMM_EPI_PAUSE_PER_KB ns for the fp32 outputs
// (default 20: 800 ns per chunk on the cfg4 forward; 7 pauses are ~1/3 of a
// main loop of ~512 cycles per k-block at the power-capped ~1.3 GHz, so the
// epilogue still finishes before its accumulator is needed).  ncu, cfg4
// forward: 399 -> 382 us, tensor pipe 88 -> 95%.  Not for the bf16 dgrad
// output (64 KB per tile over a long K loop: pausing measured -3%).
inline unsigned epi_pause_ns(int k_blocks) {
    static const int per_kb = [] {
        const char* e = getenv("COAT_GEMM_EPI_PAUSE_PER_KB");
        return e ? atoi(e) : 20;
    }();
    const long v = long(per_kb) * long(k_blocks);
    return unsigned(v < 0 ? 0 : v > 8000 ? 8000 : v);
}

// COAT_GEMM_GROUP_M overrides the raster group (A/B; 0 or >= tiles_m = the
// plain M-fastest walk).
inline int raster_group_m(int tiles_m) {
    static const int v = [] {
        const char* e = getenv("COAT_GEMM_GROUP_M");
        return e ? atoi(e) : 8;
    }();
    return (v <= 0 || v > tiles_m) ? tiles_m : v;
}

template <bool kF8, bool kAMN, bool kBMN, int kOut, int kCta>
cudaError_t run_cta(const void* a, const void* b, const void* b2, int M, int N, int K, float alpha,
                    const uint16_t* sa, const uint16_t* sb, void* out, int64_t ldo, const EpiQ& q,
                    cudaStream_t stream) {
    using G = Geo<kCta, kOut>;
    constexpr int ESZ = kF8 ? 1 : 2;
    constexpr int BK = BKB / ESZ;
    CUtensorMap ma, mb, mb2;
    EpiMaps em;
    memset(&em, 0, sizeof(em));
    // kOutUpGate: the codes (uint8 [M, ldc]) and scales (bf16 [M, ldc/16]) as TMA store
    // targets; the scale rows need a 16-byte pitch (ldc % 128 == 0), else direct stores
    int ug_tma = 0;
    if (kOut == kOutUpGate && (q.ldc % 128) == 0) {
        uint8_t* cs[3] = {q.c0, q.c1, q.c2};
        uint16_t* ss[3] = {q.s0, q.s1, q.s2};
        bool ok = true;
        for (int a = 0; a < 3 && ok; ++a)
            ok = make_map(&em.c[a], cs[a], 1, M, N, 128, 32, q.ldc) &&
                 make_map(&em.s[a], ss[a], 2, M, N / 16, 8, 32, q.ldc / 16, 0);
        ug_tma = ok ? 1 : 0;
    }
    // kOutQ16: the same for its one code array (128 x 32 boxes) and scales (16 x 32 boxes)
    if (kOut == kOutQ16 && (q.ldc % 128) == 0)
        ug_tma = (make_map(&em.c[0], q.c0, 1, M, N, 128, 32, q.ldc) &&
                  make_map(&em.s[0], q.s0, 2, M, N / 16, 16, 32, q.ldc / 16, 0))
                     ? 1
                     : 0;
    // A logical [M x K]: K-major memory [M][K]; MN-major memory [K][M]
    const bool ok_a = !kAMN ? make_map(&ma, a, ESZ, M, K, BK, BM) : make_map(&ma, a, ESZ, K, M, 128 / ESZ, BK);
    // kCta 4: the B box is a quarter (half of this CTA's half; see the producer)
    const bool ok_b = !kBMN ? make_map(&mb, b, ESZ, N, K, BK, kCta == 4 ? G::BN_L / 2 : G::BN_L)
                            : make_map(&mb, b, ESZ, K, N, 128 / ESZ, kCta == 4 ? BK / 2 : BK);
    // kOutUpGate: the up weight (same geometry as the gate weight); else a copy of B (unused)
    const bool ok_b2 = kOut == kOutUpGate ? make_map(&mb2, b2, ESZ, K, N, 128 / ESZ, BK) : true;
    if (!ok_a || !ok_b || !ok_b2) return cudaErrorInvalidValue;
    if (kOut != kOutUpGate) mb2 = mb;
    // tma_store(): the output [M, N] (fp32 or bf16) with row pitch ldo as 32 x 32 boxes
    // (128- / 64-byte rows; needs a 16-byte pitch)
    int tma_out = 0;
    constexpr int OSZ = kOut == kOutF32 ? 4 : 2;
    if (tma_store<kOut>() && (ldo * OSZ) % 16 == 0 && (reinterpret_cast<uintptr_t>(out) & 15u) == 0 &&
        make_map(&mb2, out, OSZ, M, N, 32, 32, ldo, OSZ == 4 ? 128 : 64))
        tma_out = 1;
    auto kern = gemm_kernel<kF8, kAMN, kBMN, kOut, kCta>;
    static int attr_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (attr_dev != dev) {
        const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   G::SMEM_BYTES + epi_smem_bytes<kOut>());
        if (e != cudaSuccess) return e;
        attr_dev = dev;
    }
    Params P;
    P.M = M;
    P.N = N;
    P.K = K;
    P.tiles_m = (M + G::TILE_M - 1) / G::TILE_M;
    if (kCta == 4) P.tiles_m = (P.tiles_m + 1) / 2;   // super-blocks of two pair tiles (the odd one out is all OOB)
    P.tiles_n = kOut == kOutUpGate ? (N + 127) / 128 : (N + BN - 1) / BN;
    P.k_blocks = (K + BK - 1) / BK;
    P.group_m = raster_group_m(P.tiles_m);
    P.alpha = alpha;
    P.scale_a = sa;
    P.scale_b = sb;
    P.out = out;
    P.ldo = ldo;
    P.tma_out = tma_out;
    P.ug_tma = ug_tma;
    P.epi_pause_ns = kOut == kOutF32 ? epi_pause_ns(P.k_blocks) : 0u;   // the 4-byte outputs only
    P.q = q;
    const int ntiles = P.tiles_m * P.tiles_n;
    int units = device_sm_count() / kCta;   // persistent: one CTA (pair) per SM (TPC)
    if (kCta == 4) {
        // per kernel instantiation, queried once (thread-safe static initialisation)
        static const int clusters4 = max_clusters4(kern, G::SMEM_BYTES + epi_smem_bytes<kOut>(), threads_for<kOut>());
        units = clusters4;
    }
    if (units <= 0) return cudaErrorInvalidConfiguration;
    const int grid = kCta * (ntiles < units ? ntiles : units);
    if (kCta == 1) {
        kern<<<grid, threads_for<kOut>(), G::SMEM_BYTES + epi_smem_bytes<kOut>(), stream>>>(ma, mb, mb2, em, P);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads_for<kOut>());
    cfg.dynamicSmemBytes = G::SMEM_BYTES + epi_smem_bytes<kOut>();
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kCta;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, ma, mb, mb2, em, P);
}

// COAT_GEMM_CTA=1 forces the single-CTA kernel, =4 the two-pair B-multicast
// cluster (A/B comparisons).
inline int pair_mode() {
    static const int v = [] {
        const char* e = getenv("COAT_GEMM_CTA");
        return (e && e[0] == '1') ? 1 : (e && e[0] == '4') ? 4 : 2;
    }();
    return v;
}

template <bool kF8, bool kAMN, bool kBMN, int kOut>
cudaError_t run(const void* a, const void* b, int M, int N, int K, float alpha, const uint16_t* sa,
                const uint16_t* sb, void* out, int64_t ldo, cudaStream_t stream, const EpiQ& q = EpiQ{},
                const void* b2 = nullptr) {
    if (kOut != kOutUpGate && M > 2 * BM && pair_mode() == 4)
        return run_cta<kF8, kAMN, kBMN, kOut == kOutUpGate ? kOutF32 : kOut, 4>(a, b, b2, M, N, K, alpha, sa, sb, out,
                                                                              ldo, q, stream);
    if (M > BM && pair_mode() >= 2)
        return run_cta<kF8, kAMN, kBMN, kOut, 2>(a, b, b2, M, N, K, alpha, sa, sb, out, ldo, q, stream);
    return run_cta<kF8, kAMN, kBMN, kOut, 1>(a, b, b2, M, N, K, alpha, sa, sb, out, ldo, q, stream);
}

}  // namespace gemm

// y[M,N] (fp32) = (s_x s_w) * codes_x[M,K] . codes_w[K,N]   (W row-major (K,N): MN-major B)
cudaError_t launch_fp8_linear_fwd(const uint8_t* xc, const uint16_t* sx, const uint8_t* wc, const uint16_t* sw, int M,
                                  int K, int N, float* y, cudaStream_t st) {
    return gemm::run<true, false, true, gemm::kOutF32>(xc, wc, M, N, K, 1.0f, sx, sw, y, N, st);
}
// The same y quantized per group of 16 in the epilogue (y never reaches HBM
// unless y_out is given).
cudaError_t launch_fp8_linear_fwd_q16(const uint8_t* xc, const uint16_t* sx, const uint8_t* wc, const uint16_t* sw,
                                      int M, int K, int N, uint8_t* y_codes, uint16_t* y_scales, float* y_out,
                                      uint32_t* flags, cudaStream_t st) {
    gemm::EpiQ q{};
    q.c0 = y_codes;
    q.s0 = y_scales;
    q.y0 = y_out;
    q.flags = flags;
    q.ldc = N;
    return gemm::run<true, false, true, gemm::kOutQ16>(xc, wc, M, N, K, 1.0f, sx, sw, nullptr, N, st, q);
}
// The gate/up projections of the Llama MLP in one GEMM with the SiLU*mul
// block's quantizers in the epilogue; the per-tensor down.in encode follows
// from the codes (silu_mul pass 2).
cudaError_t launch_fp8_upgate_silu(const UpGateArgs& a, cudaStream_t st) {
    gemm::EpiQ q{};
    q.c0 = a.gcodes; q.s0 = a.gscales;
    q.c1 = a.scodes; q.s1 = a.sscales;
    q.c2 = a.ucodes; q.s2 = a.uscales;
    q.y0 = a.gate_out; q.y1 = a.up_out;
    q.scale_b1 = a.s_wu;
    q.amax_bits = a.amax_bits;
    q.flags = a.flags;
    q.ldc = a.I;
    cudaError_t e = cudaMemsetAsync(a.amax_bits, 0, 4, st);
    if (e != cudaSuccess) return e;
    e = gemm::run<true, false, true, gemm::kOutUpGate>(a.xc, a.wg, int(a.M), int(a.I), int(a.H), 1.0f, a.sx, a.s_wg,
                                                        nullptr, a.I, st, q, a.wu);
    if (e != cudaSuccess) return e;
    return launch_silu_mul_pass2(a.scodes, a.sscales, a.ucodes, a.uscales, a.M * a.I, a.amax_bits, a.pcodes, a.pscale,
                                 a.pout, a.flags, st);
}
// dX[M,K] (bf16) = s_w * dY[M,N] . Wd[K,N]^T    (Wd = decoded W codes in bf16, exact; B K-major)
cudaError_t launch_linear_dgrad(const uint16_t* dy, const uint16_t* wd, const uint16_t* sw, int M, int K, int N,
                                uint16_t* dx, cudaStream_t st) {
    return gemm::run<false, false, false, gemm::kOutBf16>(dy, wd, M, K, N, 1.0f, sw, nullptr, dx, K, st);
}
// dW[K,N] (fp32) = s_x * Xd[M,K]^T . dY[M,N]     (A = Xd MN-major, B = dY MN-major)
cudaError_t launch_linear_wgrad(const uint16_t* xd, const uint16_t* sx, const uint16_t* dy, int M, int K, int N,
                                float* dw, cudaStream_t st) {
    return gemm::run<false, true, true, gemm::kOutF32>(xd, dy, K, N, M, 1.0f, sx, nullptr, dw, N, st);
}

}  // namespace coat
