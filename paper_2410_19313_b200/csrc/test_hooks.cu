// test_hooks.cu -- internal entry points for the GPU tests (not part of the
// reference-facing boundary in include/coat.h).
//
// coat_test_pack_prepare: for n (lo, hi) group extrema (|x| bit patterns),
// runs the K1 pack warp's low-latency pack_prepare_lowlat and the exact
// pack_prepare_fast side by side; out[i] = 7 floats of each
// (k, c, s, inv_c, inv_s, mode, bad).  tests/test_gpu_pack_prepare.py checks
// they agree bit for bit on random and adversarial extrema.
#include <cstdint>

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

}  // namespace
}  // namespace coat

extern "C" int coat_test_pack_prepare(const uint32_t* lo, const uint32_t* hi, int64_t n, double log_target, float* out,
                                      void* stream) {
    if (n <= 0) return 0;
    const unsigned blocks = unsigned((n + 255) / 256);
    coat::pack_prepare_pair_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(lo, hi, n, log_target, out);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
