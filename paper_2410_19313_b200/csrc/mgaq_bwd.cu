// mgaq_bwd.cu -- the backward-side MGAQ pieces.
//
//   transpose-dequantize   SavedActivation::used_values_transposed
//                          (flow.cpp:360-395): the wgrad operand X_used^T
//                          [cols, rows] from the saved FP8 codes, with the
//                          per-group scales following the ORIGINAL row-major
//                          grouping; optionally the transposed codes themselves
//                          (the reference caches them, flow.cpp:368-374).
//   requantize_cached      requantize_cached (flow.cpp:487-495): the attention
//                          output re-encoded against the scale cached in the
//                          forward, decode(encode(x / s)) * s, so backward needs
//                          no FP8 copy of it.
// Both are bit-identical to the reference (decode * scale is exact; x / s is
// the exact Markstein quotient of the quantizers, -0 kept).
#include <cstdint>

#include "act_quant.cuh"
#include "coat_device.cuh"
#include "coat_internal.h"

namespace coat {
namespace {

using namespace aq;

constexpr int kT = 64;   // 64 x 64 code tile, 256 threads (4 rows each)

template <int ODT>   // 0: fp32 out, 1: bf16 out
__global__ void __launch_bounds__(256) transpose_dequant_kernel(const uint8_t* __restrict__ codes,
                                                                const uint16_t* __restrict__ scales, int64_t rows,
                                                                int64_t cols, int64_t G, void* __restrict__ out,
                                                                uint8_t* __restrict__ codes_t) {
    __shared__ uint8_t tile[kT][kT + 4];
    __shared__ float stile[kT][kT / 16 + 1];   // per-(row, 16-column chunk) scale (G >= 16 or per-tensor)
    const int64_t r0 = int64_t(blockIdx.y) * kT, c0 = int64_t(blockIdx.x) * kT;
    const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;   // 64 x 4
    const float s_t = G == 0 ? bf16_bits_to_float(scales[0]) : 0.0f;
    for (int i = ty; i < kT; i += 4) {
        const int64_t r = r0 + i, c = c0 + tx;
        tile[i][tx] = (r < rows && c < cols) ? codes[r * cols + c] : 0;
        if (tx < kT / 16) {
            const int64_t cc = c0 + tx * 16;
            float sc = s_t;
            if (G != 0 && r < rows && cc < cols) sc = bf16_bits_to_float(scales[(r * cols + cc) / G]);
            stile[i][tx] = sc;
        }
    }
    __syncthreads();
    for (int j = ty; j < kT; j += 4) {   // output row = source column c0 + j
        const int64_t c = c0 + j, r = r0 + tx;
        if (c >= cols || r >= rows) continue;
        const uint8_t code = tile[tx][j];
        const float v = __fmul_rn(e4m3_decode(code), G == 0 ? s_t : stile[tx][j / 16]);
        if (codes_t) codes_t[c * rows + r] = code;
        if (ODT == 0) static_cast<float*>(out)[c * rows + r] = v;
        else static_cast<uint16_t*>(out)[c * rows + r] = uint16_t(f2u(round_bf16(v)) >> 16);
    }
}

template <int DT, int ODT>
__global__ void __launch_bounds__(256) requantize_kernel(const void* __restrict__ x, int64_t n,
                                                         const uint16_t* scale_bits, void* __restrict__ out,
                                                         uint8_t* __restrict__ codes, uint32_t* flags, float nz) {
    const float s = bf16_bits_to_float(*scale_bits);
    const float rs = __frcp_rn(s);
    uint32_t bad = 0;
    const int64_t nch = n / 16;
    for (int64_t ch = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; ch < nch; ch += int64_t(gridDim.x) * blockDim.x) {
        const RawChunk<DT> raw = load_raw16_a16<DT>(x, ch * 16);
        bad |= absmax_raw<DT, false>(raw) >= 0x7F800000u;
        const uint4 cw = encode16(widen16<DT>(raw), s, rs, nz);
        if (codes) reinterpret_cast<uint4*>(codes)[ch] = cw;
        const uint32_t wd[4] = {cw.x, cw.y, cw.z, cw.w};
        float v[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float2 a = e4m3x2_decode(wd[q] & 0xFFFFu);
            const float2 b = e4m3x2_decode(wd[q] >> 16);
            v[4 * q] = __fmul_rn(a.x, s);
            v[4 * q + 1] = __fmul_rn(a.y, s);
            v[4 * q + 2] = __fmul_rn(b.x, s);
            v[4 * q + 3] = __fmul_rn(b.y, s);
        }
        if (ODT == 0) {
            float4* o = reinterpret_cast<float4*>(static_cast<float*>(out) + ch * 16);
#pragma unroll
            for (int q = 0; q < 4; ++q) o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        } else {
            uint32_t p[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                p[k] = (f2u(round_bf16(v[2 * k])) >> 16) | (f2u(round_bf16(v[2 * k + 1])) & 0xFFFF0000u);
            uint4* o = reinterpret_cast<uint4*>(static_cast<uint16_t*>(out) + ch * 16);
            o[0] = make_uint4(p[0], p[1], p[2], p[3]);
            o[1] = make_uint4(p[4], p[5], p[6], p[7]);
        }
    }
    // tail (n % 16)
    const int64_t t = nch * 16 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (blockIdx.x == 0 && t < n) {
        const float xv = DT == 0 ? static_cast<const float*>(x)[t]
                                 : u2f(uint32_t(static_cast<const uint16_t*>(x)[t]) << 16);
        bad |= (f2u(xv) & 0x7FFFFFFFu) >= 0x7F800000u;
        const uint32_t code = encode_exact(xv, s, rs);
        if (codes) codes[t] = uint8_t(code);
        const float v = __fmul_rn(e4m3_decode(code), s);
        if (ODT == 0) static_cast<float*>(out)[t] = v;
        else static_cast<uint16_t*>(out)[t] = uint16_t(f2u(round_bf16(v)) >> 16);
    }
    if (flags && __reduce_or_sync(0xFFFFFFFFu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, kFlagNonFiniteInput);
}

}  // namespace

cudaError_t launch_transpose_dequant(const uint8_t* codes, const uint16_t* scales, int64_t rows, int64_t cols,
                                     int64_t G, void* out, int out_dtype, uint8_t* codes_t, cudaStream_t st) {
    if (rows <= 0 || cols <= 0) return cudaSuccess;
    const dim3 grid(unsigned((cols + kT - 1) / kT), unsigned((rows + kT - 1) / kT));
    if (out_dtype == 0) transpose_dequant_kernel<0><<<grid, 256, 0, st>>>(codes, scales, rows, cols, G, out, codes_t);
    else transpose_dequant_kernel<1><<<grid, 256, 0, st>>>(codes, scales, rows, cols, G, out, codes_t);
    return cudaGetLastError();
}

cudaError_t launch_requantize_cached(const void* x, int dtype, int64_t n, const uint16_t* scale, void* out,
                                     int out_dtype, uint8_t* codes, uint32_t* flags, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const int blocks = (int)imax64(1, imin64((n / 16 + 255) / 256, int64_t(device_sm_count()) * 8));
#define COAT_RQ(D, O) requantize_kernel<D, O><<<blocks, 256, 0, st>>>(x, n, scale, out, codes, flags, -0.0f)
    if (dtype == 0) {
        if (out_dtype == 0) COAT_RQ(0, 0);
        else COAT_RQ(0, 1);
    } else {
        if (out_dtype == 0) COAT_RQ(1, 0);
        else COAT_RQ(1, 1);
    }
#undef COAT_RQ
    return cudaGetLastError();
}

}  // namespace coat
