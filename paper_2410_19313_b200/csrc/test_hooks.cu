// test_hooks.cu -- internal entry points for the GPU tests (not part of the
// reference-facing boundary in include/coat.h).
//
// coat_test_pack_prepare: for n (lo, hi) group extrema (|x| bit patterns),
// runs the K1 pack warp's low-latency pack_prepare_lowlat and the exact
// pack_prepare_fast side by side; out[i] = 7 floats of each
// (k, c, s, inv_c, inv_s, mode, bad).  tests/test_gpu_pack_prepare.py checks
// they agree bit for bit on random and adversarial extrema.
//
// coat_test_expf_neg2: expf_neg2 (the paired expf of the SiLU producer) against
// CUDA's scalar expf(-x) over every float bit pattern in [first, first+count);
// *mismatches counts the bitwise differences.
//
// coat_test_mufu_bounds: exhaustive error of the SFU approximations behind the
// certified expand of the DRE pack (dre.cuh kRelMufu):
// max |lg2.approx.ftz(r) - log2(r)| / (1 + |log2 r|) over every float r in
// [lo_r, hi_r) (an absolute plus a relative part) and max |ex2.approx.ftz(u) /
// 2^u - 1| over every float u with |u| < hi_u, against double log2 / exp2.
//
// coat_test_k1_layout: element warps per CTA of the K1 layout this process
// selected (COAT_K1_EW; tests/test_gpu_k1_layouts.py).
#include <cstdint>
#include <cstring>

#include "coat_device.cuh"
#include "coat_internal.h"
#include "dre_fast.cuh"

namespace coat {
namespace {

__global__ void __launch_bounds__(256) pack_prepare_pair_kernel(const uint32_t* lo, const uint32_t* hi, int64_t n,
                                                              double log_target, float* out) {
    __shared__ dre::CtaTables T;
    dre::init_cta_tables(T, threadIdx.x, blockDim.x);
    __syncthreads();
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint32_t l = i < n ? lo[i] : 0x3F800000u, h = i < n ? hi[i] : 0x3F800000u;
    const dre::PackParams a = dre::pack_prepare_lowlat(l, h, log_target, log_target * 1.4426950408889634, T);
    const dre::PackParams b = dre::pack_prepare_fast(l, h, log_target);
    if (i < n) {
        float* o = out + i * 14;
        const dre::PackParams* ps[2] = {&a, &b};
        for (int j = 0; j < 2; ++j) {
            o[7 * j + 0] = ps[j]->k;
            o[7 * j + 1] = ps[j]->c;
            o[7 * j + 2] = ps[j]->s;
            o[7 * j + 3] = ps[j]->inv_c;
            o[7 * j + 4] = ps[j]->inv_s;
            o[7 * j + 5] = (float)ps[j]->mode;
            o[7 * j + 6] = ps[j]->bad ? 1.0f : 0.0f;
        }
    }
}

__global__ void __launch_bounds__(256) expf_neg2_check_kernel(uint64_t first, uint64_t count, float nz,
                                                              unsigned long long* mismatches) {
    unsigned long long bad = 0;
    for (uint64_t i = 2 * (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x); i < count;
         i += 2 * uint64_t(gridDim.x) * blockDim.x) {
        const float x0 = u2f(uint32_t(first + i)), x1 = u2f(uint32_t(first + i + 1));
        const F2 e = expf_neg2(x0, x1, nz);
        bad += f2u(e.x) != f2u(expf(-x0));
        if (i + 1 < count) bad += f2u(e.y) != f2u(expf(-x1));
    }
    if (bad) atomicAdd(mismatches, bad);
}

__device__ __forceinline__ void atomic_max_nonneg_double(unsigned long long* dst, double v) {
    atomicMax(dst, (unsigned long long)__double_as_longlong(v));   // v >= 0: bit order = value order
}

__global__ void __launch_bounds__(256) mufu_bounds_kernel(uint32_t r0, uint32_t r1, uint32_t u0, uint32_t u1,
                                                          unsigned long long* out) {
    double e_lg = 0.0, e_ex = 0.0;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t b = r0 + blockIdx.x * blockDim.x + threadIdx.x; b < r1; b += stride) {
        const float r = u2f(b);
        const double l = log2((double)r);
        e_lg = fmax(e_lg, fabs((double)dre::lg2_approx(r) - l) / (1.0 + fabs(l)));
    }
    // u in [lo_u, hi_u): positive bit patterns [u0, u1) and their negations
    for (uint32_t b = u0 + blockIdx.x * blockDim.x + threadIdx.x; b < u1; b += stride) {
#pragma unroll
        for (int sg = 0; sg < 2; ++sg) {
            const float u = u2f(b | (sg ? 0x80000000u : 0u));
            e_ex = fmax(e_ex, fabs((double)dre::ex2_approx(u) / exp2((double)u) - 1.0));
        }
    }
    atomic_max_nonneg_double(&out[0], e_lg);
    atomic_max_nonneg_double(&out[1], e_ex);
}

}  // namespace
}  // namespace coat

extern "C" int coat_test_mufu_bounds(float lo_r, float hi_r, float hi_u, unsigned long long* out, void* stream) {
    uint32_t b[3];
    const float f[3] = {lo_r, hi_r, hi_u};
    memcpy(b, f, sizeof(b));
    coat::mufu_bounds_kernel<<<148 * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(b[0], b[1], 0u, b[2], out);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

extern "C" int coat_test_pack_prepare(const uint32_t* lo, const uint32_t* hi, int64_t n, double log_target, float* out,
                                      void* stream) {
    if (n <= 0) return 0;
    const unsigned blocks = unsigned((n + 255) / 256);
    coat::pack_prepare_pair_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(lo, hi, n, log_target, out);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

extern "C" int coat_test_expf_neg2(uint64_t first, uint64_t count, unsigned long long* mismatches, void* stream) {
    if (count == 0) return 0;
    coat::expf_neg2_check_kernel<<<148 * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(first, count, -0.0f,
                                                                                        mismatches);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

namespace coat {
namespace {
__global__ void cta_tables_dump_kernel(double* out) {
    __shared__ dre::CtaTables T;
    dre::init_cta_tables(T, threadIdx.x, blockDim.x);
    __syncthreads();
    const double* src = reinterpret_cast<const double*>(&T);
    for (int i = threadIdx.x; i < int(sizeof(dre::CtaTables) / sizeof(double)); i += blockDim.x) out[i] = src[i];
}
}  // namespace
}  // namespace coat

// coat_test_cta_tables: the CTA constant tables (dre::CtaTables) as the device
// computes them (generator and check of csrc/cta_tables_data.h).
extern "C" int coat_test_cta_tables(double* out, void* stream) {
    coat::cta_tables_dump_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(out);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

extern "C" int coat_test_k1_layout() { return coat::k1_ws_config(); }
