// host_pipeline.cu -- coatsim::step with HOST-resident parameters and
// gradients (the drop-in call of the reference's API, where Tensor lives in
// host memory) while the quantized optimizer state stays resident in HBM.
//
// The parameter range is streamed through the GPU in chunks on three CUDA
// streams so PCIe host->device copies, the fused K1 kernel and the
// device->host copy-back of the updated weights overlap:
//
//   h2d stream:   [w_i, g_i -> staging slot i%3] ............
//   compute:           wait h2d_i -> K1(slot) ..................
//   d2h stream:                        wait K1_i -> [w_i -> host out]
//
// Three staging slots (w and g, `chunk` fp32 each) let chunk i+1 upload while
// chunk i computes and chunk i-1 downloads.  Host buffers must be pinned
// (cudaHostAlloc / cudaHostRegister) for the copies to be asynchronous.
// Chunks are multiples of the fused kernel's round (k1_ws_round_params():
// 16 groups of 128 in the default EW = 8 layout), so every chunk starts on a 1x128 group boundary, uses the
// state slice of its own groups, and only the last one has a ragged tail.
#include <cstdint>
#include <mutex>

#include "../../include/coat.h"
#include "coat_internal.h"

namespace coat {
namespace {

constexpr int kSlots = 3;

struct Workspace {
    int device = -1;
    int64_t chunk = 0;
    float* w[kSlots] = {nullptr, nullptr, nullptr};
    float* g[kSlots] = {nullptr, nullptr, nullptr};
    cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
    cudaEvent_t up[kSlots], done[kSlots], down[kSlots];

    cudaError_t init(int dev, int64_t ch) {
        if (device == dev && chunk >= ch) return cudaSuccess;
        release();
        device = dev;
        chunk = ch;
        cudaError_t e = cudaSuccess;
        for (int s = 0; s < kSlots && e == cudaSuccess; ++s) {
            e = cudaMalloc(&w[s], sizeof(float) * size_t(ch));
            if (e == cudaSuccess) e = cudaMalloc(&g[s], sizeof(float) * size_t(ch));
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&up[s], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&done[s], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&down[s], cudaEventDisableTiming);
        }
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&comp, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking);
        return e;
    }

    void release() {
        if (device < 0) return;
        for (int s = 0; s < kSlots; ++s) {
            cudaFree(w[s]);
            cudaFree(g[s]);
            cudaEventDestroy(up[s]);
            cudaEventDestroy(done[s]);
            cudaEventDestroy(down[s]);
            w[s] = g[s] = nullptr;
        }
        cudaStreamDestroy(h2d);
        cudaStreamDestroy(comp);
        cudaStreamDestroy(d2h);
        device = -1;
        chunk = 0;
    }
};

Workspace g_ws[16];
std::mutex g_ws_mu;

MomentStateIn slice_in(const coat_moment_state& s, int64_t off) {
    return {s.codes + off, s.scales + off / 128, s.k + off / 128, s.c + off / 128};
}
MomentStateOut slice_out(const coat_moment_state& s, int64_t off) {
    return {s.codes + off, s.scales + off / 128, s.k + off / 128, s.c + off / 128};
}

}  // namespace

cudaError_t host_pipelined_step(const float* w_host_in, float* w_host_out, const float* g_host, int64_t n,
                                const coat_moment_state& m_in, const coat_moment_state& v_in,
                                const coat_moment_state& m_out, const coat_moment_state& v_out,
                                const AdamWScalars& a, uint32_t* flags, unsigned long long* fallbacks,
                                int64_t chunk, cudaStream_t stream) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 16) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lock(g_ws_mu);
    Workspace& ws = g_ws[dev];
    const int64_t unit = k1_ws_round_params();
    chunk = (chunk + unit - 1) / unit * unit;
    e = ws.init(dev, chunk);
    if (e != cudaSuccess) return e;

    // Order after whatever the caller queued on `stream` (e.g. a flag reset).
    cudaEvent_t start;
    cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
    cudaEventRecord(start, stream);
    cudaStreamWaitEvent(ws.h2d, start, 0);
    cudaStreamWaitEvent(ws.comp, start, 0);

    const int64_t nchunks = (n + chunk - 1) / chunk;
    for (int64_t i = 0; i < nchunks && e == cudaSuccess; ++i) {
        const int s = int(i % kSlots);
        const int64_t off = i * chunk;
        const int64_t len = n - off < chunk ? n - off : chunk;
        // slot drained -- also for the first kSlots chunks: the previous call's
        // D2H of this slot may still be in flight on another caller stream
        // (never-recorded events count as complete)
        cudaStreamWaitEvent(ws.h2d, ws.down[s], 0);
        cudaMemcpyAsync(ws.w[s], w_host_in + off, sizeof(float) * size_t(len), cudaMemcpyHostToDevice, ws.h2d);
        cudaMemcpyAsync(ws.g[s], g_host + off, sizeof(float) * size_t(len), cudaMemcpyHostToDevice, ws.h2d);
        cudaEventRecord(ws.up[s], ws.h2d);
        cudaStreamWaitEvent(ws.comp, ws.up[s], 0);
        e = launch_adamw_dre_step(ws.w[s], ws.w[s], ws.g[s], len, slice_in(m_in, off), slice_in(v_in, off),
                                  slice_out(m_out, off), slice_out(v_out, off), a, flags, fallbacks, ws.comp);
        cudaEventRecord(ws.done[s], ws.comp);
        cudaStreamWaitEvent(ws.d2h, ws.done[s], 0);
        cudaMemcpyAsync(w_host_out + off, ws.w[s], sizeof(float) * size_t(len), cudaMemcpyDeviceToHost, ws.d2h);
        cudaEventRecord(ws.down[s], ws.d2h);
    }
    // The caller's stream resumes once every chunk is back on the host.
    cudaEvent_t fin;
    cudaEventCreateWithFlags(&fin, cudaEventDisableTiming);
    cudaEventRecord(fin, ws.d2h);
    cudaStreamWaitEvent(stream, fin, 0);
    cudaEventDestroy(fin);
    cudaEventDestroy(start);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace coat
