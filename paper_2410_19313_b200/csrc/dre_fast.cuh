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
//   lanes in UNIFORM SIMT rounds (every lane evaluates the same double exp2 on
//   its own argument: primes of jj, three T2 anchors; products for the rest),
//   so a warp builds its 8 tables with 3 exp2 rounds.  Each element then costs
//   two LDS.64, one DMUL, one F2F and -- for k != 1 -- a 2-op certification of
//   the float rounding; the ~2e-6 uncertain elements take the literal
//   reference formula behind a warp vote.  For k == 1 every product is exact
//   in double, so no certification is needed.
//
// Expand + encode (expand.cpp:18-22, quantize.cpp:19-27):
//   k == 1: e = RN(|x|/c), q = RN(e/s) exactly (Markstein); else e = (|x|/c)^k
//   on the SFU (lg2/ex2.approx) and the E4M3 code of e/s certified by encoding
//   both ends of an error interval with one cvt.e4m3x2.
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

__device__ __forceinline__ double sel4(int q, double a, double b, double c, double d) {
    return q == 0 ? a : q == 1 ? b : q == 2 ? c : d;
}

// Lane q (0..3) of the 4 lanes serving one (group, moment); must be called by
// all 32 lanes of the warp together (8 pairs x 4 lanes, convergent).  Every
// step below is the same instruction stream on all lanes (no divergence):
//   round 1: T1[{2,3,5,7}[q]]           = exp2(ik * log2 p)
//   round 2: T1[11], T1[13], T2[1], T2[5] = exp2(...)     (q = 0..3)
//   round 3: T2[9], T2[13]                = exp2(...)     (q = 0, 1; 2, 3 idle)
//   products: T1 composites from the primes, T2[e+1..e+3] = T2[e] * u^(1..3)
// Entries are within ~2^-49 of the exact values (<= 4 roundings after exp2),
// well inside the 2^-43 certification margin.  For k == 1 every entry is set
// exactly (T1[j] = j, T2[e] = c*s*2^(e-10)).
__device__ __forceinline__ void build_pair_contract(PairContract& P, int q, float s, float k, float c,
                                                    const CtaTables& T, int lane) {
    const double cd = (double)c;
    const uint32_t sb = f2u(s);
    bool odd = !(s >= 0x1p-100f) || !(s <= 0x1p100f) || !(c > 0.0f) || !(c <= 3.0e38f) ||
               !(k >= 1.0f) || !(k <= 20.0f);
    const bool exact = (k == 1.0f);
    const double ik = exact ? 1.0 : 1.0 / (double)k;
    const double l2s = (double)(int((sb >> 23) & 0xFFu) - 127) + T.l2b[(sb >> 16) & 0x7Fu];
    const double cs = cd * (double)s;          // exact product (24 x 8 bits)

    // ---- round 1: primes 2, 3, 5, 7
    const int p1 = q == 0 ? 2 : q == 1 ? 3 : q == 2 ? 5 : 7;
    const double v1 = exact ? (double)p1 : exp2_fast(ik * T.l2j[p1], T);
    // ---- round 2: T1[11], T1[13], T2[1], T2[5]
    const double e2 = sel4(q, T.l2j[11], T.l2j[13], l2s - 9.0, l2s - 5.0);
    double v2 = exp2_fast(ik * e2, T);
    if (q >= 2) v2 *= cd;
    const double x2 = sel4(q, 11.0, 13.0, cs * 0x1p-9, cs * 0x1p-5);   // exact values for k == 1
    v2 = exact ? x2 : v2;
    // ---- round 3: T2[9], T2[13]
    const double e3 = q == 0 ? l2s - 1.0 : l2s + 3.0;
    double v3 = cd * exp2_fast(ik * e3, T);
    v3 = exact ? (q == 0 ? cs * 0.5 : cs * 8.0) : v3;
    P.t1[p1] = v1;
    if (q < 2) {
        P.t1[q == 0 ? 11 : 13] = v2;
        P.t2[q == 0 ? 9 : 13] = v3;
    } else {
        P.t2[q == 2 ? 1 : 5] = v2;
    }
    __syncwarp();
    // ---- products
    const double u = P.t1[2];                  // 2^(1/k)
    const double t3 = P.t1[3], t5 = P.t1[5], t7 = P.t1[7];
    // T1 composites (2 per lane): 4 6 | 8 9 | 10 12 | 14 15 ; T1[0] = 0, T1[1] = 1
    const int d0 = q == 0 ? 4 : q == 1 ? 8 : q == 2 ? 10 : 14;
    const int d1 = q == 0 ? 6 : q == 1 ? 9 : q == 2 ? 12 : 15;
    const double c0 = q == 0 ? u * u : q == 1 ? (u * u) * u : q == 2 ? u * t5 : u * t7;
    const double c1 = q == 0 ? u * t3 : q == 1 ? t3 * t3 : q == 2 ? (u * u) * t3 : t3 * t5;
    P.t1[d0] = c0;
    P.t1[d1] = c1;
    // T2 chain from the anchors T2[1], T2[5], T2[9], T2[13] (lane q: anchor 4q+1)
    const double anchor = P.t2[4 * q + 1];
    const double a1 = anchor * u, a2 = a1 * u, a3 = a2 * u;
    P.t2[4 * q + 2] = a1;
    P.t2[4 * q + 3] = a2;
    if (q < 3) P.t2[4 * q + 4] = a3;
    if (q == 0) {
        P.t1[0] = 0.0;
        P.t1[1] = 1.0;
        P.t2[0] = 0.0;
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < 4; ++t) P.t1[16 + 4 * q + t] = -P.t1[4 * q + t];
    __syncwarp();
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
    // distance of the low 29 mantissa bits from the float midpoint 2^28, times 8
    // (the multiply shifts the 3 bits above bit 28 out): min over the 4 elements
    uint32_t near = 0xFFFFFFFFu;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const double X = P.t1[(jj >> (8 * i)) & 0xFFu] * P.t2[(ee >> (8 * i)) & 0xFFu];
        near = min(near, ((uint32_t)__double2loint(X) - 0x0FFFFE00u) * 8u);
        x[i] = __double2float_rn(X);
    }
    // any element within 512 double-ulps of a midpoint -> recompute all 4 (rare)
    unsure |= (P.literal || (!P.exact && near < 0x400u * 8u)) ? 0xFu : 0u;
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
            // the SFU evaluation needs a normal RN(1/c): for c outside [2^-100, 2^100]
            // (e.g. subnormal c of a group of subnormal moments, where 1/c overflows)
            // go straight to the reference formula (pow of the double quotient)
            const bool c_ok = p.c >= 0x1p-100f && p.c <= 0x1p100f;
            const float r = c_ok ? __fmul_rn(hi, __frcp_rn(p.c)) : 1.0f;
            const float e = ex2_approx(__fmul_rn(p.k, lg2_approx(r)));
            const float s_lo = group_scale(__fmul_rn(e, 1.0f - kRelMufu));
            const float s_hi = group_scale(__fmul_rn(e, 1.0f + kRelMufu));
            if (c_ok && s_lo == s_hi) {
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

// ---------------------------------------------------------------------------
// Low-latency pack_prepare: same results as pack_prepare_fast (and the
// reference), bit for bit, as one straight-line FP64/FP32 block.
//
// pack_prepare_fast is ~320 dependent instructions (libdevice sqrt / div / log
// with their special-case branches, and the k == 1 and k != 1 scale paths
// serialised by divergence): ~2800 cycles per round on the pack warp, which the
// element warps wait for.  Here every quantity is computed by an approximation
// whose error is bounded well inside what decides the rounded result, and the
// rounding is certified; lanes whose certification fails, or whose inputs are
// special (0, Inf/NaN, extreme ranges that select mode 2), recompute with
// pack_prepare_fast behind a warp vote.
//   c  = (float)sqrt(lo*hi): lo*hi is exact in double; Goldschmidt sqrt from
//        rsqrt.approx (~2^-52); float rounding certified by the 29 dropped
//        mantissa bits being >= 16 double-ulps from the float midpoint.
//   k  = (float)clamp(log_target / log(hi/lo), 1, 20): log2(hi) - log2(lo) by
//        the CTA table l2b[top 7 mantissa bits] + a degree-6 log2(1+u) series
//        (|u| < 2^-7; ~2^-51 absolute), k = (log_target/ln2) / L2 (~2^-49
//        relative, vs ~2^-50 between the reference's own double k and the exact
//        value); the clamp decisions and the float rounding are certified with a
//        2^-43 margin.
//   1/c, hi/c: quotients of 24-bit significands are >= 2^-48 (relative) away
//        from any float midpoint, so a double value within 2^-51 rounds to the
//        correctly rounded float: RN(1/c) and expand(hi) = RN(hi/c) are exact.
//   group_scale: am/448 = am/(7*2^6) is >= 2^-27.8 (relative) from any float
//        midpoint for normal quotients (the bits past the 24th repeat with
//        period 3), so (float)(am * RN64(1/448)) == RN32(am/448); tiny am
//        (< 2^-90, which lead to mode 2 anyway) fall back.
//   1/s: s has an 8-bit significand, 1/s is >= 2^-33 from a float midpoint; one
//        float Newton step from rcp.approx is within 2^-46, hence RN(1/s).
//   k != 1: the SFU evaluation of expand(hi) certified exactly as in
//        pack_prepare_fast (both ends of a 2^-15 interval give the same scale).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double rsqrt_seed_f64(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}
__device__ __forceinline__ double rcp_seed_f64(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}
__device__ __forceinline__ float rcp_approx_f32(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// |low 29 mantissa bits - half| of a double: distance (in double ulps) of its
// value from the nearest float rounding midpoint (normal float range).
__device__ __forceinline__ uint32_t f32_mid_dist(double v) {
    const int32_t low = int32_t(uint32_t(__double2loint(v)) & 0x1FFFFFFFu) - 0x10000000;
    return uint32_t(low < 0 ? -low : low);
}
// 1/x to ~2^-52 relative (x normal, not huge): seed + 2 Newton steps.
__device__ __forceinline__ double rcp_f64_fast(double x) {
    double r = rcp_seed_f64(x);
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}
// log2 pieces of a positive normal double v: returns E and the fractional part
// log2(mantissa) = l2b[i] + P(u) to ~2^-52 absolute.
__device__ __forceinline__ double log2_frac(double v, int& E, const CtaTables& T) {
    const int hw = __double2hiint(v);
    E = ((hw >> 20) & 0x7FF) - 1023;
    const int i = (hw >> 13) & 0x7F;
    const double m = __hiloint2double((hw & 0x000FFFFF) | 0x3FF00000, __double2loint(v));
    const double ci = 1.0 + (double)i * 0.0078125;          // exact
    const double d = m - ci;                                 // exact, [0, 2^-7)
    // u = d / ci: float seed of 1/ci (2^-23) + one FP64 Newton step (2^-46); |u| < 2^-7
    double r = (double)rcp_approx_f32(__double2float_rn(ci));
    r = fma(r, fma(-ci, r, 1.0), r);
    const double u = d * r;
    // log2(1+u) = sum_k (-1)^(k+1) u^k / (k ln2), k <= 6 (truncation < 2^-52)
    constexpr double c1 = 1.4426950408889634, c2 = -0.72134752044448170, c3 = 0.48089834696298783,
                     c4 = -0.36067376022224085, c5 = 0.28853900817779268, c6 = -0.24044917348149390;
    double q = fma(c6, u, c5);
    q = fma(q, u, c4);
    q = fma(q, u, c3);
    q = fma(q, u, c2);
    q = fma(q, u, c1);
    return fma(q, u, T.l2b[i]);
}

static __device__ __noinline__ PackParams pack_prepare_slow(uint32_t lo_bits, uint32_t hi_bits, double log_target) {
    return pack_prepare_fast(lo_bits, hi_bits, log_target);
}

// log2_target = log_target / ln2 (double).  Must be called by all 32 lanes
// (warp vote); give idle lanes any finite positive extrema.
__device__ __forceinline__ PackParams pack_prepare_lowlat(uint32_t lo_bits, uint32_t hi_bits, double log_target,
                                                          double log2_target, const CtaTables& T) {
    const float lo = u2f(lo_bits), hi = u2f(hi_bits);
    const double lod = (double)lo, hid = (double)hi;
    bool ok = hi_bits - 1u < 0x7F7FFFFFu && lo_bits - 1u < 0x7F7FFFFFu;   // both finite and > 0
    // ---- c = (float)sqrt(lo * hi)
    const double x = lod * hid;                              // exact
    const double y0 = rsqrt_seed_f64(x);
    double sq = x * y0, h = 0.5 * y0;
#pragma unroll
    for (int it = 0; it < 3; ++it) {
        const double rr = fma(-sq, h, 0.5);
        sq = fma(sq, rr, sq);
        h = fma(h, rr, h);
    }
    sq = fma(fma(-sq, sq, x), h, sq);
    ok &= sq >= 0x1p-100 && sq <= 0x1p100 && f32_mid_dist(sq) > 16u;
    const float c = __double2float_rn(sq);
    const double cd = (double)c;
    // ---- k
    int eh, el;
    const double fh = log2_frac(hid, eh, T), fl = log2_frac(lod, el, T);
    const double L2 = (double)(eh - el) + (fh - fl);
    ok &= L2 < 199.0;                                        // range > 2^200 selects mode 2
    double ka = hi_bits == lo_bits ? 0.0 : log2_target * rcp_f64_fast(fmax(L2, 0x1p-60));
    constexpr double kM = 0x1p-40;
    const bool k_lo = ka <= 1.0 - kM, k_hi = ka >= kKMax * (1.0 + kM);
    const bool k_mid = ka >= 1.0 + kM && ka <= kKMax * (1.0 - kM);
    ok &= k_lo || k_hi || (k_mid && f32_mid_dist(ka) > 512u);
    const float k = k_lo ? 1.0f : k_hi ? (float)kKMax : __double2float_rn(ka);
    // ---- 1/c and expand(hi) for k == 1
    const double rcd = rcp_f64_fast(cd);
    const float inv_c = __double2float_rn(rcd);
    const double am1d = hid * rcd;
    // ---- k != 1: SFU evaluation of expand(hi), certified through the BF16 scale
    const float rq = __fmul_rn(hi, inv_c);
    const float e = ex2_approx(__fmul_rn(k, lg2_approx(rq)));
    const float e_lo = __fmul_rn(e, 1.0f - kRelMufu), e_hi = __fmul_rn(e, 1.0f + kRelMufu);
    const bool lin = k == 1.0f;
    ok &= am1d < 0x1p127 || !lin;
    const double am1 = (double)__double2float_rn(am1d);   // expand(hi) = RN32(hi / c), exact
    const double aml = lin ? am1 : (double)e_lo, amh = lin ? am1 : (double)e_hi;
    ok &= aml >= 0x1p-90 && amh < 0x1p127;
    constexpr double kInv448 = 1.0 / 448.0;
    const float s = round_bf16(__double2float_rn(aml * kInv448));
    ok &= s == round_bf16(__double2float_rn(amh * kInv448)) && s >= 0x1p-100f;
    // ---- 1/s (s: 8-bit significand)
    const float r0 = rcp_approx_f32(s);
    const float inv_s = __fmaf_rn(r0, __fmaf_rn(-s, r0, 1.0f), r0);
    PackParams p;
    p.k = k;
    p.c = c;
    p.s = s;
    p.inv_c = inv_c;
    p.inv_s = inv_s;
    p.mode = lin ? 0 : 1;
    p.bad = false;
    if (__any_sync(0xFFFFFFFFu, !ok)) {
        if (!ok) p = pack_prepare_slow(lo_bits, hi_bits, log_target);
    }
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
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const F2 ax{fabsf(x[2 * h]), fabsf(x[2 * h + 1])};
        const F2 r = f2_mul(ax, f2s(p.inv_c), nz);
        const F2 l{lg2_approx(r.x), lg2_approx(r.y)};
        const F2 u = f2_mul(l, f2s(p.k), nz);
        const F2 qq = f2_mul(F2{ex2_approx(u.x), ex2_approx(u.y)}, f2s(p.inv_s), nz);
        q[h] = F2{u2f(f2u(qq.x) | (f2u(x[2 * h]) & 0x80000000u)), u2f(f2u(qq.y) | (f2u(x[2 * h + 1]) & 0x80000000u))};
    }
    const F2 lo01 = f2_mul(q[0], f2s(1.0f - kRelMufu), nz), hi01 = f2_mul(q[0], f2s(1.0f + kRelMufu), nz);
    const F2 lo23 = f2_mul(q[1], f2s(1.0f - kRelMufu), nz), hi23 = f2_mul(q[1], f2s(1.0f + kRelMufu), nz);
    const uint32_t c01 = cvt_e4m3x2(lo01.x, lo01.y), d01 = cvt_e4m3x2(hi01.x, hi01.y);
    const uint32_t c23 = cvt_e4m3x2(lo23.x, lo23.y), d23 = cvt_e4m3x2(hi23.x, hi23.y);
    unsure |= (c01 != d01 ? 0x3u : 0u) | (c23 != d23 ? 0xCu : 0u) | (p.mode == 2 ? 0xFu : 0u);
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
