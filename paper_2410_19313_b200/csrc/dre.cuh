// dre.cuh -- Dynamic Range Expansion (DRE) device building blocks for sm_100a.
//
// Reference semantics (paths relative to /root/reference/proj/core/src):
//   measure_group      expand.cpp:57-83   lo/hi over nonzero |x| in double,
//                                          c = float(sqrt(lo*hi)),
//   optimal_k          expand.cpp:50-55   k = float(clamp(log(229376)/log(hi/lo), 1, 20)),
//   expand_one         expand.cpp:18-22   e = float(copysign(pow(|x|/c, k), x)),
//   contract_one       expand.cpp:24-28   x = float(copysign(pow(|y|, 1/k) * c, y)),
//   quantize/encode    quantize.cpp:10-27 s = round_bf16(max|e|/448), code = E4M3(e/s).
//
// The reference evaluates four double-precision pow() per parameter.  Here:
//   * contract runs a short double-precision exp2 (8-entry table + degree-7
//     polynomial) whose result is CERTIFIED against the float rounding
//     boundaries; only uncertain elements (~2e-6) fall back to the literal
//     reference formula (double pow).  Output is bit-identical.
//   * expand runs in fp32 on the SFU (lg2/ex2.approx); only the E4M3 code of
//     e/s is stored, and it is certified with an interval check
//     (certified_code); uncertain elements fall back to the literal formula.
//   * the group scale needs max|e| exactly: expand is monotone in |x|, so
//     max|e| = expand(max|x|), evaluated once per group with the reference
//     formula (double pow).
#pragma once

#include "coat_device.cuh"

namespace coat {
namespace dre {

constexpr int kG = 128;                 // optimizer group
constexpr double kKMax = 20.0;          // expand.hpp:15

// log2(1 + i/8) and 2^(i/8), double, correctly rounded (host-generated).
__device__ __constant__ double kT8L[8] = {
    0.0, 0.16992500144231237, 0.32192809488736235, 0.45943161863729726,
    0.5849625007211562, 0.7004397181410922, 0.8073549220576041, 0.9068905956085185};
__device__ __constant__ double kT8E[8] = {
    1.0, 1.0905077326652577, 1.189207115002721, 1.2968395546510096,
    1.4142135623730951, 1.5422108254079407, 1.681792830507429, 1.8340080864093424};
// 2^(r/8) = sum (r ln2/8)^i / i!
constexpr double kP1 = 0.08664339756999316, kP2 = 0.0037535391712359483,
                 kP3 = 0.00010840646223597964, kP4 = 2.3481760516671086e-06,
                 kP5 = 4.0690790241786014e-08, kP6 = 5.875980527260439e-10,
                 kP7 = 7.2730702419566334e-12;

// Certification margin for contract, in double ulps of the result: the
// table+polynomial evaluation is within ~2^-46.5 relative of |y|^(1/k)*c and
// the reference's pow()*c within ~2^-51, i.e. < 128 ulps together.
constexpr int kContractMarginUlps = 512;
// Relative error bound used to certify SFU-based expand codes (analysis in
// <= ~2^-17 for k <= 20, |k*log2(|x|/c)| <= 8.95); 4x margin.
constexpr float kRelMufu = 0x1p-15f;
// Linear path (k == 1): e = |x| * RN(1/c), q = e * RN(1/s): 4 roundings.
constexpr float kRelLinear = 0x1p-20f;

// Per-(group, moment) parameters of an EXISTING state, prepared for contract.
struct ContractParams {
    double a8;      // 8 * RN(1/k)
    double ab;      // a8 * log2(s)
    double cd;      // (double)c
    float s, k, c;
    int mode;       // 0: all-zero / k==1 linear, 1: table path, 2: literal fallback only
};

__device__ __forceinline__ ContractParams contract_prepare(float s, float k, float c) {
    ContractParams p;
    p.s = s;
    p.k = k;
    p.c = c;
    p.cd = (double)c;
    if (k == 1.0f) {
        p.mode = 0;
        p.a8 = p.ab = 0.0;
    } else if (!(s >= 0x1p-100f) || !(c > 0.0f) || !isfinite(c) || !isfinite(k)) {
        p.mode = 2;  // tiny scales: decode*s may round in fp32 -> use the literal formula
        p.a8 = p.ab = 0.0;
    } else {
        p.mode = 1;
        const double ik = 1.0 / (double)k;
        p.a8 = 8.0 * ik;
        p.ab = p.a8 * log2((double)s);
    }
    return p;
}

// Literal contract_one (expand.cpp:24-28) on y = decode(code)*s (fp32 product,
// quantize.cpp:122).
static __device__ __noinline__ float contract_literal(uint32_t code, float s, float k, float c) {
    const float y = __fmul_rn(e4m3_decode(code), s);
    if (y == 0.0f) return 0.0f;
    const double mag = pow(fabs((double)y), 1.0 / (double)k) * (double)c;
    return (float)copysign(mag, (double)y);
}

// x = contract(decode(code) * s).  Returns false in `ok` when the input is NaN.
__device__ __forceinline__ float contract_one(uint32_t code, const ContractParams& p, bool& bad) {
    const uint32_t mag = code & 0x7Fu;
    if (mag == 0u) return 0.0f;                  // contract_one: y == 0 -> +0
    if (mag == 0x7Fu) { bad = true; return __int_as_float(0x7FC00000); }
    const float neg = (code & 0x80u) ? -1.0f : 1.0f;
    if (p.mode == 0) {
        // pow(|y|, 1.0) == |y| exactly; (float)((double)|y| * c) == RN32(|y|*c)
        // (double rounding is innocuous for a product of two floats).
        const float y = __fmul_rn(e4m3_decode(mag), p.s);
        return neg * __fmul_rn(y, p.c);
    }
    if (p.mode == 2) return contract_literal(code, p.s, p.k, p.c);
    // |y| = v * s with v = decode(mag) = (1 + i/8) * 2^E exactly.
    const uint32_t vb = f2u(e4m3_decode(mag));
    const int E = int((vb >> 23) & 0xFFu) - 127;
    const int i8 = int((vb >> 20) & 7u);
    const double tl = (double)E + kT8L[i8];
    const double t = fma(p.a8, tl, p.ab);        // 8*log2(|y|)/k
    const double N = rint(t);
    const double r = t - N;                      // exact, |r| <= 1/2
    double q = fma(kP7, r, kP6);
    q = fma(q, r, kP5);
    q = fma(q, r, kP4);
    q = fma(q, r, kP3);
    q = fma(q, r, kP2);
    q = fma(q, r, kP1);
    q = fma(q, r, 1.0);                          // 2^(r/8)
    const int Ni = (int)N;
    const double te = kT8E[Ni & 7];
    const double tes = __hiloint2double(__double2hiint(te) + ((Ni >> 3) << 20), __double2loint(te));
    const double X = (tes * p.cd) * q;
    // Certify: X is within 128 double-ulps of the reference's double result;
    // the float rounding is unambiguous unless X is near a float midpoint
    // (low 29 mantissa bits near 2^28) or outside the fp32 normal range.
    const uint32_t hi = (uint32_t)__double2hiint(X);
    const uint32_t lo29 = (uint32_t)__double2loint(X) & 0x1FFFFFFFu;
    const uint32_t ex = (hi >> 20) & 0x7FFu;
    const int dist = (int)lo29 - (1 << 28);
    const bool sure = ex > 1023u - 126u && ex < 1023u + 127u &&
                      (dist > kContractMarginUlps || dist < -kContractMarginUlps);
    if (!sure) return contract_literal(code, p.s, p.k, p.c);
    return neg * __double2float_rn(X);
}

// Per-(group, moment) parameters of a NEW state (measure_group + group scale).
struct PackParams {
    float k, c, s;
    float inv_c, inv_s;
    int mode;       // 0: linear (k == 1), 1: SFU path, 2: literal only
    bool bad;       // non-finite expanded values -> NonFiniteInput
};

// measure_group (expand.cpp:57-83) + optimal_k (expand.cpp:50-55) from the
// exact group extrema, then max|e| = expand(hi) and the BF16 group scale.
__device__ __forceinline__ PackParams pack_prepare(float lo, float hi, double log_target) {
    PackParams p;
    p.k = 1.0f;
    p.c = 1.0f;
    p.bad = false;
    float am = 0.0f;
    if (hi > 0.0f) {
        const double lod = (double)lo, hid = (double)hi;
        const double range = hid / lod;
        p.c = (float)sqrt(lod * hid);
        if (range > 1.0) {
            double k = log_target / log(range);
            k = fmin(fmax(k, 1.0), kKMax);
            p.k = (float)k;
        }
        const double ratio = hid / (double)p.c;
        am = p.k == 1.0f ? (float)ratio : (float)pow(ratio, (double)p.k);
        if (!isfinite(am)) p.bad = true;
    }
    p.s = group_scale(am);
    p.inv_c = __frcp_rn(p.c);
    p.inv_s = __frcp_rn(p.s);
    if (p.k == 1.0f)
        p.mode = 0;
    else
        p.mode = 1;
    if (!(p.s >= 0x1p-100f) || !(p.c >= 0x1p-100f) || !(p.c <= 0x1p100f)) p.mode = 2;
    return p;
}

// Literal expand_one + encode_scaled for one element (expand.cpp:18-22,
// quantize.cpp:19-27).
static __device__ __noinline__ uint32_t pack_literal(float x, float k, float c, float s) {
    if (x == 0.0f) return 0u;
    const double ratio = fabs((double)x) / (double)c;
    const double mag = k == 1.0f ? ratio : pow(ratio, (double)k);
    const float e = (float)copysign(mag, (double)x);
    return e4m3_encode(__fdiv_rn(e, s));
}

__device__ __forceinline__ float lg2_approx(float x) {
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float ex2_approx(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// E4M3 code of expand(x)/s, bit-identical to the reference.
__device__ __forceinline__ uint32_t pack_one(float x, const PackParams& p, uint32_t& fallbacks) {
    if (x == 0.0f) return 0u;
    const float ax = fabsf(x);
    float e, rel;
    if (p.mode == 0) {
        e = __fmul_rn(ax, p.inv_c);
        rel = kRelLinear;
    } else {
        const float r = __fmul_rn(ax, p.inv_c);
        e = ex2_approx(__fmul_rn(p.k, lg2_approx(r)));
        rel = kRelMufu;
    }
    const float q = copysignf(__fmul_rn(e, p.inv_s), x);
    uint32_t code;
    if (p.mode != 2 && e > 0x1p-120f && certified_code(q, rel, code)) return code;
    ++fallbacks;
    return pack_literal(x, p.k, p.c, p.s);
}

}  // namespace dre
}  // namespace coat
