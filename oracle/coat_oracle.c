/* oracle/coat_oracle.c -- TEST INFRASTRUCTURE ONLY (the CPU checker).
 *
 * A plain-C restatement of the reference's hot-path numerics.  Every
 * function cites the reference file:line it follows (paths relative to
 * /root/reference/proj/core).  Compiled with -ffp-contract=off, like the
 * reference (proj/CMakeLists.txt:12-14), so every fp32 operation rounds
 * separately.  Double-precision pow/log/sqrt come from the same libm the
 * reference uses, so results agree bit for bit on the same host.
 */
#include "coat_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

enum { ST_OK = 0, ST_GEOMETRY = 2, ST_NONFINITE_INPUT = 3, ST_NONFINITE_GRAD = 4 };

static inline uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static inline float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* ---------------------------------------------------------------- codec ---- */

/* fp8.cpp:27-51 decode_minifloat for E4M3 (mbits 3, ebits 4, bias 7). */
float oracle_decode_e4m3_one(uint8_t b) {
    const int sign = b >> 7, expf = (b >> 3) & 0xF, mant = b & 7;
    if (expf == 0xF && mant == 7) return NAN;
    float mag = expf == 0 ? ldexpf((float)mant, 1 - 7 - 3) : ldexpf((float)(8 + mant), expf - 7 - 3);
    return sign ? -mag : mag;
}

/* fp8.cpp:53-88 encode_minifloat for E4M3 (delta_max 448, max code 0x7E),
 * fp8.cpp:150-156 encode_byte (non-finite rejected -> -1). */
int oracle_encode_e4m3_one(float value) {
    if (!isfinite(value)) return -1;
    const uint32_t bits = f2u(value);
    const uint8_t sign = (uint8_t)((bits >> 31) << 7);
    const uint32_t absbits = bits & 0x7FFFFFFFu;
    if (absbits == 0) return sign;
    if (fabsf(value) > 448.0f) return sign | 0x7E;
    if ((absbits >> 23) == 0) return sign;            /* fp32 subnormal -> signed zero */
    const int e32 = (int)(absbits >> 23) - 127;
    const uint32_t sig = (absbits & 0x7FFFFFu) | 0x800000u;
    const int e_min_normal = 1 - 7;
    const int ulp_exp = (e32 > e_min_normal ? e32 : e_min_normal) - 3;
    const int shift = ulp_exp - (e32 - 23);
    if (shift > 31) return sign;
    uint32_t q = sig >> shift;
    const uint32_t rem = sig & ((1u << shift) - 1u);
    const uint32_t half = 1u << (shift - 1);
    if (rem > half || (rem == half && (q & 1u))) ++q;
    if (q == 0) return sign;
    uint32_t code = e32 < e_min_normal ? q : (uint32_t)((e32 + 7) << 3) + (q - 8u);
    if (code > 0x7E) code = 0x7E;
    return sign | (uint8_t)code;
}

/* fp8.cpp:209-216 */
float oracle_round_bf16_one(float value) {
    if (isnan(value)) return value;
    uint32_t bits = f2u(value);
    bits += 0x7FFFu + ((bits >> 16) & 1u);
    return u2f(bits & 0xFFFF0000u);
}

int oracle_encode_e4m3(const float* x, uint8_t* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) {
        const int c = oracle_encode_e4m3_one(x[i]);
        if (c < 0) return ST_NONFINITE_INPUT;
        out[i] = (uint8_t)c;
    }
    return ST_OK;
}

int oracle_decode_e4m3(const uint8_t* codes, float* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = oracle_decode_e4m3_one(codes[i]);
    return ST_OK;
}

/* ------------------------------------------------------------ quantizer ---- */

/* quantize.cpp:10-17 group_scale (E4M3, BF16 scales). */
static float group_scale(float am) {
    float s = am > 0.0f ? am / 448.0f : 0x1p-9f;
    s = oracle_round_bf16_one(s);
    if (s == 0.0f) s = u2f(0x00010000u);               /* bf16_min_positive, fp8.cpp:218-220 */
    return s;
}

static int all_finite(const float* x, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        if (!isfinite(x[i])) return 0;
    return 1;
}

/* quantize.cpp:89-111.  G == 0 -> per-tensor (one group of rows*cols). */
int oracle_quantize(const float* x, int64_t rows, int64_t cols, int64_t G, uint8_t* codes,
                    float* scales) {
    const int64_t n = rows * cols;
    if (!all_finite(x, n)) return ST_NONFINITE_INPUT;  /* quantize.cpp:91 */
    if (G < 0 || (G > 0 && cols % G != 0)) return ST_GEOMETRY; /* quantize.cpp:38-46 */
    const int64_t gsz = G == 0 ? n : G;
    const int64_t groups = n / gsz;
    for (int64_t g = 0; g < groups; ++g) {
        const float* xg = x + g * gsz;
        float am = 0.0f;
        for (int64_t i = 0; i < gsz; ++i) am = fmaxf(am, fabsf(xg[i]));
        const float s = group_scale(am);
        scales[g] = s;
        for (int64_t i = 0; i < gsz; ++i) codes[g * gsz + i] = (uint8_t)oracle_encode_e4m3_one(xg[i] / s);
    }
    return ST_OK;
}

/* quantize.cpp:113-124 */
int oracle_dequantize(const uint8_t* codes, const float* scales, int64_t rows, int64_t cols,
                      int64_t G, float* out) {
    const int64_t n = rows * cols;
    if (G < 0 || (G > 0 && cols % G != 0)) return ST_GEOMETRY;
    const int64_t gsz = G == 0 ? n : G;
    for (int64_t i = 0; i < n; ++i) out[i] = oracle_decode_e4m3_one(codes[i]) * scales[i / gsz];
    return ST_OK;
}

/* quantize.cpp:126-145 */
int oracle_group_scale_max(const float* x, int64_t rows, int64_t cols, int64_t G,
                           float* intermediate, float* global) {
    if (G <= 0 || cols % G != 0) return ST_GEOMETRY;
    const int64_t groups = rows * cols / G;
    float gm = 0.0f;
    for (int64_t g = 0; g < groups; ++g) {
        float m = 0.0f;
        for (int64_t i = 0; i < G; ++i) m = fmaxf(m, fabsf(x[g * G + i]));
        intermediate[g] = m;
    }
    for (int64_t g = 0; g < groups; ++g) gm = fmaxf(gm, intermediate[g]);
    *global = gm;
    return ST_OK;
}

/* -------------------------------------------------- range expansion (DRE) -- */

static const double kRangeE4M3 = 229376.0; /* expand.hpp:14 */
static const double kKMax = 20.0;          /* expand.hpp:15 */

/* expand.cpp:50-55 */
void oracle_optimal_k(double range, float* k, int* degenerate) {
    if (!(range > 1.0)) { *k = 1.0f; *degenerate = 1; return; }
    double kk = log(kRangeE4M3) / log(range);
    kk = fmin(fmax(kk, 1.0), kKMax);
    *k = (float)kk;
    *degenerate = 0;
}

/* expand.cpp:57-83 */
void oracle_measure_group(const float* x, int64_t n, float* k, float* c, float* range,
                          int* degenerate) {
    double lo = 0.0, hi = 0.0;
    int any = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (x[i] == 0.0f) continue;
        const double a = fabs((double)x[i]);
        if (!any) { lo = hi = a; any = 1; }
        else { lo = fmin(lo, a); hi = fmax(hi, a); }
    }
    *k = 1.0f; *c = 1.0f; *range = 0.0f; *degenerate = 0;
    if (!any) { *degenerate = 1; return; }
    const double r = hi / lo;
    *range = (float)r;
    *c = (float)sqrt(lo * hi);
    oracle_optimal_k(r, k, degenerate);
}

/* expand.cpp:18-22 */
static inline float expand_one(float x, double k, double c) {
    if (x == 0.0f) return 0.0f;
    const double mag = pow((double)fabsf(x) / c, k);
    return (float)copysign(mag, (double)x);
}

/* expand.cpp:24-28 */
static inline float contract_one(float y, double k, double c) {
    if (y == 0.0f) return 0.0f;
    const double mag = pow((double)fabsf(y), 1.0 / k) * c;
    return (float)copysign(mag, (double)y);
}

/* expand.cpp:115-135: measure every group, expand, then per-group quantize. */
int oracle_expand_quantize(const float* x, int64_t n, int64_t G, uint8_t* codes, float* scales,
                           float* k, float* c) {
    if (G <= 0 || n % G != 0) return ST_GEOMETRY;
    if (!all_finite(x, n)) return ST_NONFINITE_INPUT;
    float* e = (float*)malloc(sizeof(float) * (size_t)(G > 0 ? G : 1));
    int st = ST_OK;
    for (int64_t g = 0; g < n / G && st == ST_OK; ++g) {
        float range; int deg;
        oracle_measure_group(x + g * G, G, &k[g], &c[g], &range, &deg);
        for (int64_t i = 0; i < G; ++i) e[i] = expand_one(x[g * G + i], k[g], c[g]);
        /* quantize(expanded) checks finiteness of the whole expanded tensor (quantize.cpp:91) */
        if (!all_finite(e, G)) { st = ST_NONFINITE_INPUT; break; }
        float am = 0.0f;
        for (int64_t i = 0; i < G; ++i) am = fmaxf(am, fabsf(e[i]));
        const float s = group_scale(am);
        scales[g] = s;
        for (int64_t i = 0; i < G; ++i) codes[g * G + i] = (uint8_t)oracle_encode_e4m3_one(e[i] / s);
    }
    free(e);
    return st;
}

/* expand.cpp:137-141 -> quantize.cpp:113-124 then expand.cpp:100-113 */
int oracle_dequantize_contract(const uint8_t* codes, const float* scales, const float* k,
                               const float* c, int64_t n, int64_t G, float* out) {
    if (G <= 0 || n % G != 0) return ST_GEOMETRY;
    for (int64_t i = 0; i < n; ++i) {
        const float y = oracle_decode_e4m3_one(codes[i]) * scales[i / G];
        if (!isfinite(y)) return ST_NONFINITE_INPUT;   /* contract() checks all_finite(y) */
        out[i] = contract_one(y, k[i / G], c[i / G]);
    }
    return ST_OK;
}

/* ------------------------------------------------------------ optimizer ---- */

/* optimizer.cpp:90-99: pack_moment(zeros) -> every group degenerate. */
int oracle_make_slot(int64_t n, int64_t G, uint8_t* mc, float* ms, float* mk, float* mcc,
                     uint8_t* vc, float* vs, float* vk, float* vcc) {
    if (G <= 0) return ST_GEOMETRY;
    const int64_t npad = (n + G - 1) / G * G;
    float* z = (float*)calloc((size_t)npad, sizeof(float));
    int st = oracle_expand_quantize(z, npad, G, mc, ms, mk, mcc);
    if (st == ST_OK) st = oracle_expand_quantize(z, npad, G, vc, vs, vk, vcc);
    free(z);
    return st;
}

/* optimizer.cpp:57-68 adamw_update (every op rounded separately, no FMA). */
static void adamw_update(float* w, float* m, float* v, const float* g, int64_t n, float b1,
                         float b2, float lr, float wd, float eps, int64_t t) {
    const float bc1 = 1.0f - powf(b1, (float)t);
    const float bc2 = 1.0f - powf(b2, (float)t);
    for (int64_t i = 0; i < n; ++i) {
        m[i] = b1 * m[i] + (1.0f - b1) * g[i];
        v[i] = b2 * v[i] + (1.0f - b2) * (g[i] * g[i]);
        const float mhat = m[i] / bc1;
        const float vhat = v[i] / bc2;
        w[i] = w[i] - lr * (mhat / (sqrtf(vhat) + eps) + wd * w[i]);
    }
}

/* optimizer.cpp:101-114: validate grads, unpack (DQ + contract), AdamW, repack
 * (pad with zeros, measure, expand, quantize).  On NonFiniteInput from the
 * repack, w has been updated but the state is left unchanged (as in the reference). */
int oracle_step(float* w, const float* g, int64_t n, int64_t G, uint8_t* mc, float* ms,
                float* mk, float* mcc, uint8_t* vc, float* vs, float* vk, float* vcc,
                int64_t step_in, float b1, float b2, float lr, float wd, float eps) {
    if (!all_finite(g, n)) return ST_NONFINITE_GRAD;  /* optimizer.cpp:104 */
    const int64_t npad = (n + G - 1) / G * G;
    float* m = (float*)calloc((size_t)npad, sizeof(float));
    float* v = (float*)calloc((size_t)npad, sizeof(float));
    uint8_t* c2 = (uint8_t*)malloc((size_t)npad * 2);
    float* meta = (float*)malloc(sizeof(float) * (size_t)(npad / G) * 6);
    int st = oracle_dequantize_contract(mc, ms, mk, mcc, npad, G, m);
    if (st == ST_OK) st = oracle_dequantize_contract(vc, vs, vk, vcc, npad, G, v);
    if (st == ST_OK) {
        adamw_update(w, m, v, g, n, b1, b2, lr, wd, eps, step_in + 1);
        /* pad_flat: elements past n are zeros again (optimizer.cpp:28-32) */
        for (int64_t i = n; i < npad; ++i) m[i] = v[i] = 0.0f;
        const int64_t ng = npad / G;
        /* slot.m = pack(m); slot.v = pack(v); (optimizer.cpp:111-112): a throw
         * from the second pack leaves the first one committed. */
        st = oracle_expand_quantize(m, npad, G, c2, meta, meta + ng, meta + 2 * ng);
        if (st == ST_OK) {
            memcpy(mc, c2, (size_t)npad);
            memcpy(ms, meta, sizeof(float) * (size_t)ng);
            memcpy(mk, meta + ng, sizeof(float) * (size_t)ng);
            memcpy(mcc, meta + 2 * ng, sizeof(float) * (size_t)ng);
            st = oracle_expand_quantize(v, npad, G, c2 + npad, meta + 3 * ng, meta + 4 * ng, meta + 5 * ng);
        }
        if (st == ST_OK) {
            memcpy(vc, c2 + npad, (size_t)npad);
            memcpy(vs, meta + 3 * ng, sizeof(float) * (size_t)ng);
            memcpy(vk, meta + 4 * ng, sizeof(float) * (size_t)ng);
            memcpy(vcc, meta + 5 * ng, sizeof(float) * (size_t)ng);
        }
    }
    free(m); free(v); free(c2); free(meta);
    return st;
}

/* optimizer.cpp:116-131 */
void oracle_reference_adamw_step(float* w, float* m, float* v, const float* g, int64_t n,
                                 float b1, float b2, float lr, float wd, float eps, int64_t t) {
    adamw_update(w, m, v, g, n, b1, b2, lr, wd, eps, t);
}

/* ------------------------------------------------------- synthetic data ---- */

/* rng.hpp:20-73 SplitMix64 */
typedef struct { uint64_t state; double cached; int have; } sm64;
static uint64_t sm_next(sm64* r) {
    r->state += 0x9E3779B97F4A7C15ULL;
    uint64_t z = r->state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static sm64 sm_make(uint64_t seed) { sm64 r = {seed, 0.0, 0}; return r; }
static sm64 sm_split(uint64_t seed, uint64_t stream) {  /* rng.hpp:24-27 */
    sm64 mixer = sm_make(seed ^ (0x5851F42D4C957F2DULL * (stream + 1)));
    return sm_make(sm_next(&mixer));
}
static double sm_double(sm64* r) { return (double)(sm_next(r) >> 11) * 0x1.0p-53; }
static double sm_uniform(sm64* r, double lo, double hi) { return lo + (hi - lo) * sm_double(r); }
static double sm_normal(sm64* r) {                       /* rng.hpp:54-67 */
    if (r->have) { r->have = 0; return r->cached; }
    double u1 = sm_double(r);
    while (u1 <= 0.0) u1 = sm_double(r);
    const double u2 = sm_double(r);
    const double rr = sqrt(-2.0 * log(u1));
    const double theta = 2.0 * 3.141592653589793 * u2;  /* std::numbers::pi */
    r->cached = rr * sin(theta);
    r->have = 1;
    return rr * cos(theta);
}

uint64_t oracle_splitmix64_at(uint64_t seed, uint64_t i) {
    sm64 r = sm_make(seed + i * 0x9E3779B97F4A7C15ULL);
    return sm_next(&r);
}

/* synthetic.cpp:28-66 */
int oracle_generate(int kind, int64_t rows, int64_t cols, double frac, double scale,
                    uint64_t seed, float* out) {
    const int64_t n = rows * cols;
    if (kind == 0) {
        sm64 values = sm_split(seed, 0), marks = sm_split(seed, 1);
        for (int64_t i = 0; i < n; ++i) {
            double v = sm_normal(&values);
            if (sm_double(&marks) < frac) v *= scale;
            out[i] = (float)v;
        }
    } else if (kind == 1) {
        sm64 values = sm_split(seed, 0), marks = sm_split(seed, 1);
        for (int64_t r = 0; r < rows; ++r) {
            const int hot = sm_double(&marks) < frac;
            const double s = hot ? scale : 1.0;
            for (int64_t c = 0; c < cols; ++c) out[r * cols + c] = (float)(s * sm_normal(&values));
        }
    } else {
        sm64 rng = sm_split(seed, 0);
        const double half_span = 0.5 * log(scale);
        for (int64_t i = 0; i < n; ++i) {
            const double mag = exp(sm_uniform(&rng, -half_span, half_span));
            const int neg = (int)(sm_next(&rng) & 1u);
            out[i] = (float)(neg ? -mag : mag);
        }
    }
    return ST_OK;
}

/* ------------------------------------------------------------ linear ---- */
/* flow.cpp:21-33 matmul: a (m,k) times b (k,n), fp32 accumulation in p order,
 * skipping a == 0 exactly as the reference does. */
void oracle_matmul(const float* a, const float* b, int64_t m, int64_t k, int64_t n, float* out) {
    for (int64_t i = 0; i < m * n; ++i) out[i] = 0.0f;
    for (int64_t i = 0; i < m; ++i)
        for (int64_t p = 0; p < k; ++p) {
            const float av = a[i * k + p];
            if (av == 0.0f) continue;
            for (int64_t j = 0; j < n; ++j) out[i * n + j] += av * b[p * n + j];
        }
}

/* --------------------------------------------------------- producers ---- */
/* flow.cpp:56-71 rmsnorm_forward: per row a sequential fp32 sum of squares,
 * var /= h, rms = sqrtf(var + eps), out = x / rms * w (each op rounded). */
void oracle_rmsnorm(const float* x, const float* w, int64_t rows, int64_t h, float eps, float* out) {
    for (int64_t r = 0; r < rows; ++r) {
        float var = 0.0f;
        for (int64_t j = 0; j < h; ++j) {
            const float v = x[r * h + j];
            var += v * v;
        }
        var /= (float)h;
        const float rms = sqrtf(var + eps);
        for (int64_t j = 0; j < h; ++j) out[r * h + j] = x[r * h + j] / rms * w[j];
    }
}

/* flow.cpp:97-100 sigmoid / silu: x * (1 / (1 + expf(-x))). */
void oracle_silu(const float* x, int64_t n, float* out) {
    for (int64_t i = 0; i < n; ++i) {
        const float s = 1.0f / (1.0f + expf(-x[i]));
        out[i] = x[i] * s;
    }
}
