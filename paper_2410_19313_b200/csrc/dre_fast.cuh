// dre_fast.cuh -- table-driven, branch-free DRE building blocks (sm_100a).
// Same results as dre.cuh and the reference, bit for bit; cheaper per element.
//
// Contract (expand.cpp:24-28, x = c * |y|^(1/k), y = decode(code) * s):
//   every E4M3 magnitude is |v| = jj * 2^(ee-10) with jj = mant | (expf?8:0)
//   (1..15) and ee = max(expf, 1) (1..15), so
//       X = sign * c*|y|^(1/k) = T1[sign*16 + jj] * T2[ee],
//       T1[jj] = jj^(1/k) (negated in the upper half),
//       T2[ee] = c * s^(1/k) * 2^((ee-10)/k).
//   The tables (48 doubles per (group, moment)) are built once per tile by 4
//   lanes with a double-precision exp2 (64-entry table + degree-5 polynomial,
//   no SFU).  Each element then costs two LDS.64, one DMUL, one F2F and -- for
//   k != 1 -- a 3-op certification of the float rounding; the ~2e-6 uncertain
//   elements take the literal reference formula behind a warp vote.  For k == 1
//   every product is exact in double, so no certification is needed.
//
// Expand + encode (expand.cpp:18-22, quantize.cpp:19-27):
//   e = (|x|/c)^k on the SFU (lg2/ex2.approx) or |x|*RN(1/c) for k == 1;
//   code = E4M3(e/s) is certified by encoding both ends of an error interval
//   with one cvt.e4m3x2 (certified_code in coat_device.cuh).
#pragma once

#include "coat_device.cuh"
#include "dre.cuh"

namespace coat {
namespace dre {

struct CtaTables {
    double t64[64];    // 2^(i/64)
    double l2b[128];   // log2(1 + i/128)   (bf16 mantissas)
    double l2j[16];    // log2(i), i >= 1
};

__device__ __forceinline__ void init_cta_tables(CtaTables& T, int tid, int nthreads) {
    for (int i = tid; i < 64; i += nthreads) T.t64[i] = exp2((double)i / 64.0);
    for (int i = tid; i < 128; i += nthreads) T.l2b[i] = log2(1.0 + (double)i / 128.0);
    for (int i = tid; i < 16; i += nthreads) T.l2j[i] = i ? log2((double)i) : 0.0;
}

// 2^x for |x| < 1000 on the FP64 pipe only: x*64 = N + r, |r| <= 1/2; rint via
// the 1.5*2^52 magic constant; 2^(r/64) by a degree-5 polynomial (truncation
// error < 2^-54); table entry 2^((N mod 64)/64) with exponent += N div 64.
__device__ __forceinline__ double exp2_fast(double x, const CtaTables& T) {
    constexpr double kMagic = 6755399441055744.0;   // 1.5 * 2^52
    constexpr double c1 = 0.010830424696249145, c2 = 5.864904955056169e-05,
                     c3 = 2.1173137155464774e-07, c4 = 5.732851688640402e-10,
                     c5 = 1.2417843701716923e-12;   // (ln2/64)^i / i!
    const double y = x * 64.0;
    const double z = y + kMagic;
    const int N = __double2loint(z);
    const double r = y - (z - kMagic);
    double p = fma(c5, r, c4);
    p = fma(p, r, c3);
    p = fma(p, r, c2);
    p = fma(p, r, c1);
    p = fma(p, r, 1.0);
    const double t = T.t64[N & 63];
    const double ts = __hiloint2double(__double2hiint(t) + ((N >> 6) << 20), __double2loint(t));
    return ts * p;
}

struct PairContract {
    double t1[32];   // [sign*16 + jj]
    double t2[16];   // [ee]
    float s, k, c;
    int literal;     // 1: every element takes the literal formula
    int exact;       // 1: k == 1, products exact, no certification needed
};

// Lane q (0..3) of the 4 lanes serving one (group, moment) builds entries
// 4q..4q+3.  Must be called by all 32 lanes of the warp together.
__device__ __forceinline__ void build_pair_contract(PairContract& P, int q, float s, float k, float c,
                                                    const CtaTables& T, int lane) {
    const double cd = (double)c;
    const uint32_t sb = f2u(s);
    bool odd = !(s >= 0x1p-100f) || !(s <= 0x1p100f) || !(c > 0.0f) || !(c <= 3.0e38f) ||
               !(k >= 1.0f) || !(k <= 20.0f);
    const bool exact = (k == 1.0f);
    double ik = 1.0, l2s = 0.0, cs = 0.0;
    if (exact) {
        cs = cd * (double)s;   // exact: 24 x 8 significant bits
    } else {
        ik = 1.0 / (double)k;
        l2s = (double)(int((sb >> 23) & 0xFFu) - 127) + T.l2b[(sb >> 16) & 0x7Fu];
    }
#pragma unroll 1
    for (int t = 0; t < 4; ++t) {
        const int i = 4 * q + t;
        double a, b;
        if (exact) {
            // pow(|y|, 1.0) == |y|: X = jj * (c * s * 2^(ee-10)) exactly.
            a = (double)i;
            b = cs * __hiloint2double((1023 + i - 10) << 20, 0);
        } else {
            a = exp2_fast(ik * T.l2j[i], T);
            b = cd * exp2_fast(ik * (l2s + (double)(i - 10)), T);
        }
        if (i == 0) a = b = 0.0;
        P.t1[i] = a;
        P.t1[16 + i] = -a;
        P.t2[i] = b;
    }
    P.t1[16] = 0.0;   // code 0x80: contract_one returns +0
    // Nonzero |X| spans [T1[1]*T2[1], T1[14]*T2[15]] (codes 0x01 .. 0x7E): keep
    // every product in the fp32 normal range or send the whole pair to the
    // literal formula (uniform, rare).
    if (q == 0 && !(P.t2[1] >= 0x1p-125)) odd = true;
    if (q == 3 && !(P.t1[14] * P.t2[15] <= 0x1p126)) odd = true;
    const uint32_t bad = __ballot_sync(0xFFFFFFFFu, odd);
    if (q == 0) {
        P.s = s;
        P.k = k;
        P.c = c;
        P.exact = exact ? 1 : 0;
        P.literal = ((bad >> (lane & ~3)) & 0xFu) ? 1 : 0;
    }
}

// Contract the 4 codes of one packed word (a lane's 4 elements of a group).
// Sets bit i of `unsure` for elements that need the literal formula and
// nanflag for NaN codes (0x7F / 0xFF).
__device__ __forceinline__ void contract_word(uint32_t codes, const PairContract& P, float (&x)[4],
                                              uint32_t& unsure, uint32_t& nanflag) {
    const uint32_t mag = codes & 0x7F7F7F7Fu;
    const uint32_t tt = mag ^ 0x7F7F7F7Fu;
    nanflag |= (tt - 0x01010101u) & ~tt & 0x80808080u;
    const uint32_t expf = (mag >> 3) & 0x0F0F0F0Fu;
    const uint32_t nz = ((expf + 0x0F0F0F0Fu) & 0x10101010u) >> 1;   // 0x08 where expf != 0
    const uint32_t jj = (mag & 0x07070707u) | nz | ((codes >> 3) & 0x10101010u);
    const uint32_t ee = expf | ((~nz >> 3) & 0x01010101u);            // max(expf, 1)
    uint32_t near = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const double X = P.t1[(jj >> (8 * i)) & 0xFFu] * P.t2[(ee >> (8 * i)) & 0xFFu];
        // within 512 double-ulps of a float rounding midpoint?
        near |= (((uint32_t)__double2loint(X) - 0x0FFFFE00u) & 0x1FFFFFFFu) < 0x400u ? (1u << i) : 0u;
        x[i] = __double2float_rn(X);
    }
    unsure |= P.literal ? 0xFu : (P.exact ? 0u : near);
}

// Parameters of a NEW (group, moment) state: measure_group + optimal_k + the
// BF16 group scale (expand.cpp:50-83, quantize.cpp:10-17), from the exact
// extrema of |x| (bit patterns; lo = min over nonzero).  The expanded group
// max feeds only round_bf16(max/448): it is evaluated on the SFU and the BF16
// rounding certified; pow() runs only when uncertain.
static __device__ __noinline__ PackParams pack_prepare_fast(uint32_t lo_bits, uint32_t hi_bits, double log_target) {
    PackParams p;
    p.k = 1.0f;
    p.c = 1.0f;
    p.bad = false;
    p.mode = 0;
    if (hi_bits >= 0x7F800000u) {       // Inf/NaN moment value -> pack throws NonFiniteInput
        p.bad = true;
        p.mode = 2;
        p.s = 1.0f;
        p.inv_c = p.inv_s = 1.0f;
        return p;
    }
    float s;
    if (hi_bits == 0u) {
        s = group_scale(0.0f);
    } else {
        const float lo = u2f(lo_bits), hi = u2f(hi_bits);
        const double lod = (double)lo, hid = (double)hi;
        const double range = hid / lod;
        p.c = (float)sqrt(lod * hid);
        if (range > 1.0) {
            double k = log_target / log(range);
            k = fmin(fmax(k, 1.0), kKMax);
            p.k = (float)k;
        }
        if (p.k == 1.0f) {
            // expand(hi) = float(double(hi)/double(c)) == RN32(hi/c) (innocuous double rounding)
            const float am = __fdiv_rn(hi, p.c);
            if (!isfinite(am)) p.bad = true;
            s = group_scale(am);
            if (range > 0x1p200) p.mode = 2;
        } else {
            p.mode = 1;
            const float r = __fmul_rn(hi, __frcp_rn(p.c));
            const float e = ex2_approx(__fmul_rn(p.k, lg2_approx(r)));
            const float s_lo = group_scale(__fmul_rn(e, 1.0f - kRelMufu));
            const float s_hi = group_scale(__fmul_rn(e, 1.0f + kRelMufu));
            if (s_lo == s_hi) {
                s = s_lo;
            } else {
                const float am = (float)pow(hid / (double)p.c, (double)p.k);
                if (!isfinite(am)) p.bad = true;
                s = group_scale(am);
            }
        }
        if (!(p.c >= 0x1p-100f) || !(p.c <= 0x1p100f) || !(s >= 0x1p-100f)) p.mode = 2;
    }
    p.s = s;
    p.inv_c = __frcp_rn(p.c);
    p.inv_s = __frcp_rn(s);
    return p;
}

// Codes of 4 values of one group; bit i of `unsure` marks an element that
// needs the literal formula.  x must not be -0 (callers canonicalize).  The
// lg2/ex2 inputs are never subnormal here (r in [2^-9, 2^9] for k > 1), so
// the .ftz SFU forms are exact replacements of the non-ftz ones.
__device__ __forceinline__ uint32_t pack_word(const float (&x)[4], const PackParams& p, uint32_t& unsure, float nz) {
    if (p.mode == 0) {
        // k == 1: e = RN(|x|/c) and q = RN(e/s) both EXACTLY via Markstein's
        // correction from RN(1/c), RN(1/s) (tests/test_markstein.py); no
        // certification needed.  c, s in [2^-100, 2^100] (else mode 2).
        uint32_t c2[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const F2 ax{fabsf(x[2 * h]), fabsf(x[2 * h + 1])};
            const F2 e0 = f2_mul(ax, f2s(p.inv_c), nz);
            const F2 e = f2_fma(f2_fma(e0, f2s(-p.c), ax), f2s(p.inv_c), e0);
            const F2 q0 = f2_mul(e, f2s(p.inv_s), nz);
            const F2 qq = f2_fma(f2_fma(q0, f2s(-p.s), e), f2s(p.inv_s), q0);
            c2[h] = cvt_e4m3x2(u2f(f2u(qq.x) | (f2u(x[2 * h]) & 0x80000000u)),
                               u2f(f2u(qq.y) | (f2u(x[2 * h + 1]) & 0x80000000u)));
        }
        return c2[0] | (c2[1] << 16);
    }
    F2 q[2];
    const float rel = p.mode == 0 ? kRelLinear : kRelMufu;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const F2 ax{fabsf(x[2 * h]), fabsf(x[2 * h + 1])};
        const F2 r = f2_mul(ax, f2s(p.inv_c), nz);
        F2 e;
        if (p.mode == 0) {
            e = r;
        } else {
            const F2 l{lg2_approx(r.x), lg2_approx(r.y)};
            const F2 u = f2_mul(l, f2s(p.k), nz);
            e = F2{ex2_approx(u.x), ex2_approx(u.y)};
        }
        const F2 qq = f2_mul(e, f2s(p.inv_s), nz);
        q[h] = F2{u2f(f2u(qq.x) | (f2u(x[2 * h]) & 0x80000000u)), u2f(f2u(qq.y) | (f2u(x[2 * h + 1]) & 0x80000000u))};
    }
    const F2 lo01 = f2_mul(q[0], f2s(1.0f - rel), nz), hi01 = f2_mul(q[0], f2s(1.0f + rel), nz);
    const F2 lo23 = f2_mul(q[1], f2s(1.0f - rel), nz), hi23 = f2_mul(q[1], f2s(1.0f + rel), nz);
    const uint32_t c01 = cvt_e4m3x2(lo01.x, lo01.y), d01 = cvt_e4m3x2(hi01.x, hi01.y);
    const uint32_t c23 = cvt_e4m3x2(lo23.x, lo23.y), d23 = cvt_e4m3x2(hi23.x, hi23.y);
    unsure |= (c01 != d01 ? 0x3u : 0u) | (c23 != d23 ? 0xCu : 0u);
    if (p.mode == 2) unsure = 0xFu;
    return c01 | (c23 << 16);
}

__device__ __forceinline__ void fix_contract(float (&x)[4], uint32_t unsure, uint32_t codes, const PairContract& P) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
        if (unsure & (1u << i)) x[i] = contract_literal((codes >> (8 * i)) & 0xFFu, P.s, P.k, P.c);
}

__device__ __forceinline__ uint32_t fix_pack(const float (&x)[4], uint32_t unsure, uint32_t codes,
                                             const PackParams& p) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (unsure & (1u << i)) {
            const uint32_t c = pack_literal(x[i], p.k, p.c, p.s);
            codes = (codes & ~(0xFFu << (8 * i))) | (c << (8 * i));
        }
    }
    return codes;
}

}  // namespace dre
}  // namespace coat
