// api.cu -- the extern "C" boundary (include/coat.h) over the sm_100a kernels.
// Host-side validation mirrors the reference's synchronous exceptions
// (GeometryMismatch / ShapeMismatch / InvalidSpec are thrown before any work,
// e.g. quantize.cpp:38-57, optimizer.cpp:102-103); data-dependent errors are
// reported through the device flag word.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <climits>
#include <mutex>

#include "../../include/coat.h"
#include "coat_internal.h"

namespace coat {

static thread_local char g_last_error[256] = "";
static unsigned long long* g_fallback_counter = nullptr;

int device_sm_count() {
    int dev = 0;
    cudaGetDevice(&dev);
    static int cached[64] = {0};
    if (dev < 0 || dev >= 64) return 148;
    if (cached[dev] == 0) {
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = sms > 0 ? sms : 148;
    }
    return cached[dev];
}

static coat_status cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return COAT_OK;
    std::snprintf(g_last_error, sizeof(g_last_error), "CUDA: %s", cudaGetErrorString(e));
    return COAT_ERR_CUDA;
}

static coat_status fail(coat_status s, const char* msg) {
    std::snprintf(g_last_error, sizeof(g_last_error), "%s", msg);
    return s;
}

static cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
static MomentStateIn in_of(const coat_moment_state& s) { return {s.codes, s.scales, s.k, s.c}; }
static MomentStateOut out_of(const coat_moment_state& s) { return {s.codes, s.scales, s.k, s.c}; }
static bool state_ok(const coat_moment_state& s) {
    return s.codes && s.scales && s.k && s.c && (reinterpret_cast<uintptr_t>(s.codes) & 15u) == 0;
}

}  // namespace coat

using namespace coat;

extern "C" {

const char* coat_version(void) { return "coat-b200 0.1.0 (sm_100a)"; }

const char* coat_status_string(coat_status s) {
    switch (s) {
        case COAT_OK: return "ok";
        case COAT_ERR_SHAPE: return "ShapeMismatch";
        case COAT_ERR_GEOMETRY: return "GeometryMismatch";
        case COAT_ERR_NONFINITE_INPUT: return "NonFiniteInput";
        case COAT_ERR_NONFINITE_GRAD: return "NonFiniteGradient";
        case COAT_ERR_INVALID: return "InvalidSpec";
        case COAT_ERR_CUDA: return "CudaError";
        case COAT_ERR_NCCL: return "NcclError";
        case COAT_ERR_OUT_OF_RANGE: return "OutOfRange";
        case COAT_ERR_ALL_ZERO_GROUP: return "AllZeroGroup";
        case COAT_ERR_IO: return "IoError";
        case COAT_ERR_BAD_MAGIC: return "BadMagic";
    }
    return "unknown";
}

const char* coat_last_error(void) { return g_last_error; }

coat_status coat_flags_to_status(uint32_t flags) {
    if (flags & COAT_FLAG_NONFINITE_GRAD) return COAT_ERR_NONFINITE_GRAD;  // checked first, optimizer.cpp:104
    if (flags & (COAT_FLAG_NONFINITE_INPUT | COAT_FLAG_PACK_M | COAT_FLAG_PACK_V | COAT_FLAG_CONTRACT))
        return COAT_ERR_NONFINITE_INPUT;
    return COAT_OK;
}

int coat_device_sm_count(void) { return device_sm_count(); }

coat_status coat_set_fallback_counter(unsigned long long* d_counter) {
    g_fallback_counter = d_counter;
    return COAT_OK;
}

// ------------------------------------------------------------------ codec --
coat_status coat_encode_e4m3(const float* x, uint8_t* codes, int64_t n, uint32_t* d_flags, void* stream) {
    if (n < 0) return fail(COAT_ERR_INVALID, "encode: negative n");
    return cuda_status(launch_encode_e4m3(x, codes, n, d_flags, S(stream)));
}

coat_status coat_decode_e4m3(const uint8_t* codes, float* x, int64_t n, void* stream) {
    if (n < 0) return fail(COAT_ERR_INVALID, "decode: negative n");
    return cuda_status(launch_decode_e4m3(codes, x, n, S(stream)));
}

// -------------------------------------------------------------- quantizer --
static coat_status check_group(int64_t rows, int64_t cols, int64_t G, int dtype) {
    if (rows <= 0 || cols <= 0) return fail(COAT_ERR_INVALID, "tensor dimensions must be positive");
    if (dtype != 0 && dtype != 1) return fail(COAT_ERR_INVALID, "dtype must be 0 (fp32) or 1 (bf16)");
    if (G <= 0) return fail(COAT_ERR_GEOMETRY, "per-group: group size must be positive");
    if (cols % G != 0) return fail(COAT_ERR_GEOMETRY, "per-group: last dim not divisible by group size");
    return COAT_OK;
}

coat_status coat_quantize_per_group(const void* x, int dtype, int64_t rows, int64_t cols, int64_t G,
                                    uint8_t* codes, uint16_t* scales, uint32_t* d_flags, void* stream) {
    const coat_status st = check_group(rows, cols, G, dtype);
    if (st != COAT_OK) return st;
    return cuda_status(launch_quantize_per_group(x, dtype, rows * cols, G, codes, scales, d_flags, S(stream)));
}

coat_status coat_dequantize_per_group(const uint8_t* codes, const uint16_t* scales, int64_t rows, int64_t cols,
                                      int64_t G, void* out, int out_dtype, void* stream) {
    const coat_status st = check_group(rows, cols, G, out_dtype);
    if (st != COAT_OK) return st;
    return cuda_status(launch_dequantize_per_group(codes, scales, rows * cols, G, out, out_dtype, S(stream)));
}

coat_status coat_group_scale_max(const void* x, int dtype, int64_t rows, int64_t cols, int64_t G,
                                 float* intermediate, uint32_t* d_amax_bits, void* stream) {
    const coat_status st = check_group(rows, cols, G, dtype);
    if (st != COAT_OK) return st;
    if (!d_amax_bits) return fail(COAT_ERR_INVALID, "group_scale_max: d_amax_bits is NULL");
    return cuda_status(launch_group_amax(x, dtype, rows * cols, G, intermediate, d_amax_bits, nullptr, S(stream)));
}

coat_status coat_quantize_per_tensor(const void* x, int dtype, int64_t n, const uint32_t* d_amax_bits,
                                     uint8_t* codes, uint16_t* d_scale, uint32_t* d_flags, void* stream) {
    if (n <= 0) return fail(COAT_ERR_INVALID, "tensor dimensions must be positive");
    if (dtype != 0 && dtype != 1) return fail(COAT_ERR_INVALID, "dtype must be 0 (fp32) or 1 (bf16)");
    if (!d_amax_bits) return fail(COAT_ERR_INVALID, "quantize_per_tensor: d_amax_bits is NULL");
    return cuda_status(launch_quantize_per_tensor(x, dtype, n, d_amax_bits, codes, d_scale, d_flags, S(stream)));
}

coat_status coat_dequantize_per_tensor(const uint8_t* codes, const uint16_t* d_scale, int64_t n, void* out,
                                       int out_dtype, void* stream) {
    if (n <= 0) return fail(COAT_ERR_INVALID, "tensor dimensions must be positive");
    if (out_dtype != 0 && out_dtype != 1) return fail(COAT_ERR_INVALID, "dtype must be 0 (fp32) or 1 (bf16)");
    return cuda_status(launch_dequantize_per_group(codes, d_scale, n, n, out, out_dtype, S(stream)));
}

coat_status coat_quantize_batch(const coat_mgaq_item* items, int32_t n_items, uint32_t* d_flags, void* stream) {
    if (n_items <= 0) return COAT_OK;
    if (!items || n_items > kMgaqMaxItems) return fail(COAT_ERR_INVALID, "quantize_batch: 1..16 items");
    MgaqItem it[kMgaqMaxItems];
    for (int i = 0; i < n_items; ++i) {
        const coat_mgaq_item& m = items[i];
        const int64_t G = m.group_size;
        if (G < 0) return fail(COAT_ERR_INVALID, "quantize_batch: negative group size");
        const coat_status st = check_group(m.rows, m.cols, G ? G : m.cols, m.dtype);
        if (st != COAT_OK) return st;
        const int64_t n = m.rows * m.cols;
        if (G) {
            const int64_t l = G / 16;
            if (G % 16 || l > 32 || (l & (l - 1))) return fail(COAT_ERR_INVALID, "quantize_batch: G/16 must be a power of two <= 32");
        }
        if (n % 16 || (reinterpret_cast<uintptr_t>(m.x) & 31u) || (reinterpret_cast<uintptr_t>(m.codes) & 15u) ||
            !m.codes || !m.scales)
            return fail(COAT_ERR_INVALID, "quantize_batch: needs numel % 16 == 0, 32-byte aligned x, 16-byte aligned codes");
        it[i] = MgaqItem{m.x, (int)m.dtype, n, G, m.codes, m.scales, m.d_amax_bits};
    }
    return cuda_status(mgaq_batch_cooperative() ? launch_mgaq_batch(it, n_items, d_flags, S(stream))
                       : mgaq_batch_queue()    ? launch_mgaq_queue(it, n_items, d_flags, S(stream))
                                               : launch_mgaq_streams(it, n_items, d_flags, S(stream)));
}

// ------------------------------------------------------- fused producers -----
static bool a16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

coat_status coat_rmsnorm_quant(const void* x, int32_t dtype, int64_t rows, int64_t h, const float* w, float eps,
                               uint8_t* x_codes, uint16_t* x_scales, uint8_t* y_codes, uint16_t* d_y_scale,
                               float* y_out, float* d_rms, uint32_t* d_amax_bits, uint32_t* d_flags, void* stream) {
    const coat_status st = check_group(rows, h, 16, dtype);
    if (st != COAT_OK) return st;
    if (!x || !w || !x_codes || !x_scales || !y_codes || !d_y_scale || !d_rms || !d_amax_bits)
        return fail(COAT_ERR_INVALID, "rmsnorm_quant: NULL buffer");
    if (!a16(x) || !a16(w) || !a16(x_codes) || !a16(y_codes) || (y_out && !a16(y_out)))
        return fail(COAT_ERR_INVALID, "rmsnorm_quant: buffers must be 16-byte aligned");
    RmsBlockArgs a{x, dtype, rows, h, w, eps, x_codes, x_scales, y_codes, d_y_scale, y_out, d_rms, d_amax_bits, d_flags};
    return cuda_status(launch_rmsnorm_block(a, S(stream)));
}

coat_status coat_silu_mul_quant(const void* gate, const void* up, int32_t dtype, int64_t rows, int64_t cols,
                                uint8_t* g_codes, uint16_t* g_scales, uint8_t* s_codes, uint16_t* s_scales,
                                uint8_t* u_codes, uint16_t* u_scales, uint8_t* p_codes, uint16_t* d_p_scale,
                                float* p_out, uint32_t* d_amax_bits, uint32_t* d_flags, void* stream) {
    const coat_status st = check_group(rows, cols, 16, dtype);
    if (st != COAT_OK) return st;
    if (!gate || !up || !g_codes || !g_scales || !s_codes || !s_scales || !u_codes || !u_scales || !p_codes ||
        !d_p_scale || !d_amax_bits)
        return fail(COAT_ERR_INVALID, "silu_mul_quant: NULL buffer");
    if ((reinterpret_cast<uintptr_t>(gate) & 31u) || (reinterpret_cast<uintptr_t>(up) & 31u) || !a16(g_codes) ||
        !a16(s_codes) || !a16(u_codes) || !a16(p_codes) || (p_out && !a16(p_out)))
        return fail(COAT_ERR_INVALID, "silu_mul_quant: gate/up 32-byte, codes 16-byte aligned");
    SiluBlockArgs a{gate, up, dtype, rows * cols, g_codes, g_scales, s_codes, s_scales, u_codes, u_scales,
                    p_codes, d_p_scale, p_out, d_amax_bits, d_flags};
    return cuda_status(launch_silu_mul_block(a, S(stream)));
}

// ------------------------------------------------- backward-side MGAQ pieces ----
coat_status coat_transpose_dequantize(const uint8_t* codes, const uint16_t* scales, int64_t rows, int64_t cols,
                                      int64_t G, void* out, int32_t out_dtype, uint8_t* codes_t, void* stream) {
    if (rows <= 0 || cols <= 0) return fail(COAT_ERR_INVALID, "tensor dimensions must be positive");
    if (out_dtype != 0 && out_dtype != 1) return fail(COAT_ERR_INVALID, "dtype must be 0 (fp32) or 1 (bf16)");
    if (G < 0 || (G > 0 && (cols % G != 0)))
        return fail(COAT_ERR_GEOMETRY, "per-group: last dim not divisible by group size");
    if (G > 0 && G % 16 != 0) return fail(COAT_ERR_INVALID, "transpose_dequantize: group size must be a multiple of 16");
    if (!codes || !scales || !out) return fail(COAT_ERR_INVALID, "transpose_dequantize: NULL buffer");
    return cuda_status(launch_transpose_dequant(codes, scales, rows, cols, G, out, out_dtype, codes_t, S(stream)));
}

coat_status coat_requantize_cached(const void* x, int32_t dtype, int64_t n, const uint16_t* d_scale, void* out,
                                   int32_t out_dtype, uint8_t* codes, uint32_t* d_flags, void* stream) {
    if (n <= 0) return fail(COAT_ERR_INVALID, "tensor dimensions must be positive");
    if ((dtype != 0 && dtype != 1) || (out_dtype != 0 && out_dtype != 1))
        return fail(COAT_ERR_INVALID, "dtype must be 0 (fp32) or 1 (bf16)");
    if (!x || !d_scale || !out) return fail(COAT_ERR_INVALID, "requantize_cached: NULL buffer");
    if ((reinterpret_cast<uintptr_t>(x) & 15u) || (reinterpret_cast<uintptr_t>(out) & 15u) ||
        (codes && (reinterpret_cast<uintptr_t>(codes) & 15u)))
        return fail(COAT_ERR_INVALID, "requantize_cached: buffers must be 16-byte aligned");
    return cuda_status(launch_requantize_cached(x, dtype, n, d_scale, out, out_dtype, codes, d_flags, S(stream)));
}

// ------------------------------------------------------- slot checkpoints ----
static coat_status check_slot_args(const char* path, const int64_t* shape, int32_t rank, int64_t G,
                                   const coat_moment_state& m, const coat_moment_state& v) {
    if (!path || !shape || rank <= 0) return fail(COAT_ERR_INVALID, "slot io: path/shape required");
    for (int i = 0; i < rank; ++i)
        if (shape[i] <= 0) return fail(COAT_ERR_INVALID, "tensor dimensions must be positive");
    if (G != 128) return fail(COAT_ERR_INVALID, "slot io: the B200 optimizer uses G = 128");
    if (!m.codes || !m.scales || !m.k || !m.c || !v.codes || !v.scales || !v.k || !v.c)
        return fail(COAT_ERR_INVALID, "slot io: NULL state buffer");
    return COAT_OK;
}

coat_status coat_save_slot(const char* path, const int64_t* shape, int32_t rank, int64_t G, coat_moment_state m,
                           coat_moment_state v, const coat_adamw_config* cfg, int64_t step, void* stream) {
    coat_status st = check_slot_args(path, shape, rank, G, m, v);
    if (st != COAT_OK) return st;
    if (!cfg) return fail(COAT_ERR_INVALID, "save_slot: cfg is NULL");
    std::string err;
    st = save_slot_impl(path, shape, rank, G, m, v, *cfg, step, S(stream), err);
    return st == COAT_OK ? st : fail(st, err.c_str());
}

coat_status coat_load_slot(const char* path, const int64_t* shape, int32_t rank, int64_t G, coat_moment_state m,
                           coat_moment_state v, coat_adamw_config* cfg_out, int64_t* step_out, void* stream) {
    coat_status st = check_slot_args(path, shape, rank, G, m, v);
    if (st != COAT_OK) return st;
    if (!cfg_out || !step_out) return fail(COAT_ERR_INVALID, "load_slot: outputs are NULL");
    std::string err;
    st = load_slot_impl(path, shape, rank, G, m, v, cfg_out, step_out, S(stream), err);
    return st == COAT_OK ? st : fail(st, err.c_str());
}

// ------------------------------------------------------------------ DRE -----
static const double kLogTarget = std::log(229376.0);  // expand.cpp:52 log(target_range)

coat_status coat_expand_quantize(const float* x, int64_t n, int64_t G, coat_moment_state out, uint32_t* d_flags,
                                 void* stream) {
    if (G <= 0 || n % G != 0) return fail(COAT_ERR_GEOMETRY, "expand: numel not divisible by group size");
    if (G != 128) return fail(COAT_ERR_INVALID, "expand_quantize: only G = 128 is implemented on B200");
    if (n <= 0) return fail(COAT_ERR_INVALID, "tensor dimensions must be positive");
    if (!state_ok(out) || (reinterpret_cast<uintptr_t>(x) & 15u)) return fail(COAT_ERR_INVALID, "misaligned or NULL buffer");
    return cuda_status(launch_expand_quantize(x, n, out_of(out), kLogTarget, d_flags, g_fallback_counter, S(stream)));
}

coat_status coat_dequantize_contract(coat_moment_state in, int64_t n, int64_t G, float* x, uint32_t* d_flags,
                                     void* stream) {
    if (G <= 0 || n % G != 0) return fail(COAT_ERR_GEOMETRY, "expand: numel not divisible by group size");
    if (G != 128) return fail(COAT_ERR_INVALID, "dequantize_contract: only G = 128 is implemented on B200");
    if (n <= 0) return fail(COAT_ERR_INVALID, "tensor dimensions must be positive");
    if (!state_ok(in) || (reinterpret_cast<uintptr_t>(x) & 15u)) return fail(COAT_ERR_INVALID, "misaligned or NULL buffer");
    return cuda_status(launch_dequantize_contract(in_of(in), n, x, d_flags, S(stream)));
}

// ------------------------------------------------------------ optimizer -----
coat_status coat_make_slot(int64_t n, int64_t G, coat_moment_state m, coat_moment_state v, void* stream) {
    if (n <= 0) return fail(COAT_ERR_INVALID, "tensor dimensions must be positive");
    if (G != 128) return fail(COAT_ERR_INVALID, "make_slot: only G = 128 is implemented on B200");
    if (!state_ok(m) || !state_ok(v)) return fail(COAT_ERR_INVALID, "misaligned or NULL state buffer");
    const int64_t npad = (n + G - 1) / G * G;
    cudaError_t e = launch_make_slot(out_of(m), npad, S(stream));
    if (e == cudaSuccess) e = launch_make_slot(out_of(v), npad, S(stream));
    return cuda_status(e);
}

static coat_status step_args(const coat_adamw_config* cfg, int64_t n, int64_t G, int64_t t,
                             const coat_moment_state& m_in, const coat_moment_state& v_in,
                             const coat_moment_state& m_out, const coat_moment_state& v_out, AdamWScalars& a) {
    if (!cfg) return fail(COAT_ERR_INVALID, "step: cfg is NULL");
    if (n <= 0) return fail(COAT_ERR_INVALID, "tensor dimensions must be positive");
    if (G != 128) return fail(COAT_ERR_INVALID, "step: only G = 128 is implemented on B200");
    if (t < 1) return fail(COAT_ERR_INVALID, "step: t is the 1-based step number");
    if (!state_ok(m_in) || !state_ok(v_in) || !state_ok(m_out) || !state_ok(v_out))
        return fail(COAT_ERR_INVALID, "step: misaligned or NULL state buffer");
    a.beta1 = cfg->beta1;
    a.beta2 = cfg->beta2;
    a.lr = cfg->lr;
    a.weight_decay = cfg->weight_decay;
    a.eps = cfg->eps;
    // optimizer.cpp:58-59: float std::pow on the host, exactly as the reference.
    a.bc1 = 1.0f - std::pow(cfg->beta1, float(t));
    a.bc2 = 1.0f - std::pow(cfg->beta2, float(t));
    a.log_target = kLogTarget;
    return COAT_OK;
}

coat_status coat_adamw_dre_step_host(const float* w_host_in, float* w_host_out, const float* g_host, int64_t n,
                                     int64_t G, coat_moment_state m_in, coat_moment_state v_in,
                                     coat_moment_state m_out, coat_moment_state v_out,
                                     const coat_adamw_config* cfg, int64_t t, uint32_t* d_flags, int64_t chunk,
                                     void* stream) {
    AdamWScalars a;
    const coat_status st = step_args(cfg, n, G, t, m_in, v_in, m_out, v_out, a);
    if (st != COAT_OK) return st;
    if (!w_host_in || !w_host_out || !g_host) return fail(COAT_ERR_INVALID, "step: NULL buffer");
    if (chunk <= 0) chunk = int64_t(32) << 20;
    return cuda_status(host_pipelined_step(w_host_in, w_host_out, g_host, n, m_in, v_in, m_out, v_out, a,
                                           d_flags, g_fallback_counter, chunk, S(stream)));
}

// ------------------------------------------------------------- ZeRO (NCCL) --
static coat_status nccl_status(int r, const char* what) {
    if (r == 0) return COAT_OK;
    std::snprintf(g_last_error, sizeof(g_last_error), "%s: %s", what, nccl_error_string(r));
    return COAT_ERR_NCCL;
}

coat_status coat_nccl_unique_id(uint8_t* out_id) {
    if (!out_id) return fail(COAT_ERR_INVALID, "nccl_unique_id: NULL");
    if (!nccl_available()) return fail(COAT_ERR_NCCL, "NCCL library (libnccl.so.2) not found");
    return nccl_status(nccl_unique_id(out_id), "ncclGetUniqueId");
}

coat_status coat_nccl_comm_init(void** comm, int32_t nranks, const uint8_t* id, int32_t rank) {
    if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks) return fail(COAT_ERR_INVALID, "nccl_comm_init: bad arguments");
    if (!nccl_available()) return fail(COAT_ERR_NCCL, "NCCL library (libnccl.so.2) not found");
    return nccl_status(nccl_comm_init(comm, nranks, id, rank), "ncclCommInitRank");
}

coat_status coat_nccl_comm_destroy(void* comm) {
    if (!comm) return COAT_OK;
    if (!nccl_available()) return fail(COAT_ERR_NCCL, "NCCL library (libnccl.so.2) not found");
    return nccl_status(nccl_comm_destroy(comm), "ncclCommDestroy");
}

coat_status coat_zero_step(float* w_full, const float* g_full, int64_t n_total, int64_t G, coat_moment_state m_in,
                           coat_moment_state v_in, coat_moment_state m_out, coat_moment_state v_out,
                           const coat_adamw_config* cfg, int64_t t, float* g_shard, float* w_scratch,
                           uint32_t* d_flags, void* comm, int32_t rank, int32_t nranks, void* stream) {
    if (!w_full || !g_full || !g_shard || !w_scratch || !d_flags || !comm)
        return fail(COAT_ERR_INVALID, "zero_step: NULL buffer or communicator");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(COAT_ERR_INVALID, "zero_step: bad rank / nranks");
    if (n_total <= 0 || n_total % (128 * int64_t(nranks)) != 0)
        return fail(COAT_ERR_GEOMETRY, "zero_step: n_total must be a positive multiple of 128 * nranks (FlatLayout)");
    if (!nccl_available()) return fail(COAT_ERR_NCCL, "NCCL library (libnccl.so.2) not found");
    const int64_t n = n_total / nranks;
    AdamWScalars a;
    coat_status st = step_args(cfg, n, G, t, m_in, v_in, m_out, v_out, a);
    if (st != COAT_OK) return st;
    const cudaStream_t s = S(stream);
    st = nccl_status(zero_reduce_scatter(g_full, g_shard, n, comm, s), "ncclReduceScatter");
    if (st != COAT_OK) return st;
    const float* w_own = w_full + int64_t(rank) * n;
    st = cuda_status(launch_adamw_dre_step(w_own, w_scratch, g_shard, n, in_of(m_in), in_of(v_in), out_of(m_out),
                                           out_of(v_out), a, d_flags, g_fallback_counter, s));
    if (st != COAT_OK) return st;
    cudaError_t ce = cudaSuccess;
    st = nccl_status(zero_agree_and_select(d_flags, w_own, w_scratch, n, comm,
                                           reinterpret_cast<uint8_t*>(g_shard), s, &ce), "ncclAllReduce");
    if (st != COAT_OK) return st;
    if ((st = cuda_status(ce)) != COAT_OK) return st;
    return nccl_status(zero_all_gather(w_scratch, w_full, n, comm, s), "ncclAllGather");
}

coat_status coat_zero_step_p2p(const void* const* g_peers, const void* g_mc, int32_t g_dtype,
                               float* const* w_next_peers, float* w_next_mc, const float* w_cur, float* w_next,
                               int64_t n_total, int64_t G, coat_moment_state m_in, coat_moment_state v_in,
                               coat_moment_state m_out, coat_moment_state v_out, const coat_adamw_config* cfg,
                               int64_t t, float* g_shard, uint32_t* d_flags, int32_t rank, int32_t nranks,
                               int64_t chunk, void* stream) {
    if (nranks < 1 || nranks > 16 || rank < 0 || rank >= nranks)
        return fail(COAT_ERR_INVALID, "zero_step_p2p: bad rank / nranks (1..16)");
    if (!w_cur || !w_next || !g_shard || !d_flags) return fail(COAT_ERR_INVALID, "zero_step_p2p: NULL buffer");
    if (!g_mc && !g_peers) return fail(COAT_ERR_INVALID, "zero_step_p2p: gradients need g_peers or g_mc");
    if (!w_next_mc && !w_next_peers && nranks > 1)
        return fail(COAT_ERR_INVALID, "zero_step_p2p: weights need w_next_peers or w_next_mc");
    if (g_dtype != 0 && g_dtype != 1) return fail(COAT_ERR_INVALID, "zero_step_p2p: g_dtype 0 (fp32) or 1 (bf16)");
    if (g_mc && g_dtype != 0) return fail(COAT_ERR_INVALID, "zero_step_p2p: the multimem reduce is fp32");
    if (n_total <= 0 || n_total % (128 * int64_t(nranks)) != 0)
        return fail(COAT_ERR_GEOMETRY, "zero_step_p2p: n_total must be a positive multiple of 128 * nranks");
    uintptr_t al = reinterpret_cast<uintptr_t>(w_cur) | reinterpret_cast<uintptr_t>(w_next) |
                   reinterpret_cast<uintptr_t>(g_shard) | reinterpret_cast<uintptr_t>(g_mc) |
                   reinterpret_cast<uintptr_t>(w_next_mc);
    for (int r = 0; r < nranks; ++r) {
        if (g_peers) {
            if (!g_peers[r]) return fail(COAT_ERR_INVALID, "zero_step_p2p: NULL gradient peer");
            al |= reinterpret_cast<uintptr_t>(g_peers[r]);
        }
        if (w_next_peers) {
            if (!w_next_peers[r]) return fail(COAT_ERR_INVALID, "zero_step_p2p: NULL weight peer");
            al |= reinterpret_cast<uintptr_t>(w_next_peers[r]);
        }
    }
    if (al & 15u) return fail(COAT_ERR_INVALID, "zero_step_p2p: buffers must be 16-byte aligned");
    const int64_t n = n_total / nranks;
    AdamWScalars a;
    const coat_status st = step_args(cfg, n, G, t, m_in, v_in, m_out, v_out, a);
    if (st != COAT_OK) return st;
    ZeroP2PArgs z{g_peers, g_mc, int(g_dtype), w_next_peers, w_next_mc, w_cur, w_next, n, m_in, v_in, m_out,
                  v_out, g_shard, int(rank), int(nranks), chunk};
    return cuda_status(zero_p2p_step(z, a, d_flags, g_fallback_counter, S(stream)));
}

coat_status coat_adamw_dre_step(const float* w_in, float* w_out, const float* g, int64_t n, int64_t G,
                                coat_moment_state m_in, coat_moment_state v_in, coat_moment_state m_out,
                                coat_moment_state v_out, const coat_adamw_config* cfg, int64_t t,
                                uint32_t* d_flags, void* stream) {
    AdamWScalars a;
    const coat_status st = step_args(cfg, n, G, t, m_in, v_in, m_out, v_out, a);
    if (st != COAT_OK) return st;
    if (!w_in || !w_out || !g) return fail(COAT_ERR_INVALID, "step: NULL buffer");
    return cuda_status(launch_adamw_dre_step(w_in, w_out, g, n, in_of(m_in), in_of(v_in), out_of(m_out),
                                             out_of(v_out), a, d_flags, g_fallback_counter, S(stream)));
}

}  // extern "C"

// ------------------------------------------------------------ FP8 linear -----
extern "C" {

static coat_status check_linear(int64_t M, int64_t K, int64_t N, const void* a, const void* b, const void* out) {
    if (M <= 0 || K <= 0 || N <= 0) return fail(COAT_ERR_INVALID, "tensor dimensions must be positive");
    if (M > INT32_MAX || K > INT32_MAX || N > INT32_MAX) return fail(COAT_ERR_INVALID, "dimension too large");
    if (K % 16 != 0 || N % 16 != 0) return fail(COAT_ERR_SHAPE, "linear: K and N must be multiples of 16 (TMA strides)");
    if ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) | reinterpret_cast<uintptr_t>(out)) & 15u)
        return fail(COAT_ERR_INVALID, "linear: buffers must be 16-byte aligned");
    return COAT_OK;
}

coat_status coat_fp8_linear_fwd(const uint8_t* x_codes, const uint16_t* d_sx, const uint8_t* w_codes,
                                const uint16_t* d_sw, int64_t M, int64_t K, int64_t N, float* y, void* stream) {
    const coat_status st = check_linear(M, K, N, x_codes, w_codes, y);
    if (st != COAT_OK) return st;
    return cuda_status(launch_fp8_linear_fwd(x_codes, d_sx, w_codes, d_sw, int(M), int(K), int(N), y, S(stream)));
}

coat_status coat_fp8_linear_fwd_q16(const uint8_t* x_codes, const uint16_t* d_sx, const uint8_t* w_codes,
                                    const uint16_t* d_sw, int64_t M, int64_t K, int64_t N, uint8_t* y_codes,
                                    uint16_t* y_scales, float* y_out, uint32_t* d_flags, void* stream) {
    const coat_status st = check_linear(M, K, N, x_codes, w_codes, y_codes);
    if (st != COAT_OK) return st;
    if (!y_scales) return fail(COAT_ERR_INVALID, "linear_fwd_q16: NULL scales");
    if (y_out && !a16(y_out)) return fail(COAT_ERR_INVALID, "linear_fwd_q16: y_out must be 16-byte aligned");
    return cuda_status(launch_fp8_linear_fwd_q16(x_codes, d_sx, w_codes, d_sw, int(M), int(K), int(N), y_codes,
                                                 y_scales, y_out, d_flags, S(stream)));
}

coat_status coat_fp8_upgate_silu_quant(const uint8_t* x_codes, const uint16_t* d_sx, const uint8_t* wg_codes,
                                       const uint16_t* d_swg, const uint8_t* wu_codes, const uint16_t* d_swu,
                                       int64_t M, int64_t H, int64_t I, uint8_t* g_codes, uint16_t* g_scales,
                                       uint8_t* s_codes, uint16_t* s_scales, uint8_t* u_codes, uint16_t* u_scales,
                                       uint8_t* p_codes, uint16_t* d_p_scale, float* gate_out, float* up_out,
                                       float* p_out, uint32_t* d_amax_bits, uint32_t* d_flags, void* stream) {
    coat_status st = check_linear(M, H, I, x_codes, wg_codes, g_codes);
    if (st != COAT_OK) return st;
    if (!wu_codes || !g_scales || !s_codes || !s_scales || !u_codes || !u_scales || !p_codes || !d_p_scale ||
        !d_amax_bits)
        return fail(COAT_ERR_INVALID, "upgate_silu_quant: NULL buffer");
    if (!a16(wu_codes) || !a16(s_codes) || !a16(u_codes) || !a16(p_codes) || (gate_out && !a16(gate_out)) ||
        (up_out && !a16(up_out)) || (p_out && !a16(p_out)) || (!gate_out != !up_out))
        return fail(COAT_ERR_INVALID, "upgate_silu_quant: 16-byte aligned buffers; gate_out and up_out together");
    UpGateArgs a{x_codes, d_sx, wg_codes, d_swg, wu_codes, d_swu, M, H, I, g_codes, g_scales, s_codes, s_scales,
                 u_codes, u_scales, p_codes, d_p_scale, gate_out, up_out, p_out, d_amax_bits, d_flags};
    return cuda_status(launch_fp8_upgate_silu(a, S(stream)));
}

coat_status coat_linear_bwd_dgrad(const uint16_t* dy_bf16, const uint16_t* w_dec_bf16, const uint16_t* d_sw,
                                  int64_t M, int64_t K, int64_t N, uint16_t* dx_bf16, void* stream) {
    const coat_status st = check_linear(M, K, N, dy_bf16, w_dec_bf16, dx_bf16);
    if (st != COAT_OK) return st;
    return cuda_status(launch_linear_dgrad(dy_bf16, w_dec_bf16, d_sw, int(M), int(K), int(N), dx_bf16, S(stream)));
}

coat_status coat_linear_bwd_wgrad(const uint16_t* x_dec_bf16, const uint16_t* d_sx, const uint16_t* dy_bf16,
                                  int64_t M, int64_t K, int64_t N, float* dw, void* stream) {
    const coat_status st = check_linear(M, K, N, x_dec_bf16, dy_bf16, dw);
    if (st != COAT_OK) return st;
    if (M % 16 != 0) return fail(COAT_ERR_SHAPE, "wgrad: M must be a multiple of 16 (TMA strides)");
    return cuda_status(launch_linear_wgrad(x_dec_bf16, d_sx, dy_bf16, int(M), int(K), int(N), dw, S(stream)));
}

coat_status coat_decode_e4m3_bf16(const uint8_t* codes, uint16_t* out_bf16, int64_t n, void* stream) {
    if (n < 0) return fail(COAT_ERR_INVALID, "decode: negative n");
    return cuda_status(launch_decode_e4m3_bf16(codes, out_bf16, n, S(stream)));
}

}  // extern "C"
