/* include/coat.h -- the drop-in C-ABI of the B200-native COAT hot path.
 *
 * Every entry point replaces one operator of the reference's proj/core API
 * (coatsim, /root/reference/proj/core/include/coatsim/), the comment on
 * each cites the reference declaration (file:line) it stands in for.  The
 * reference is a C++ library with no FFI of its own, so this header is the
 * boundary a binding (ctypes, the C++ shim in include/coat/coatsim_compat.hpp,
 * a JNI/cgo stub) links against; INTEGRATION.md shows those bindings.
 *
 * Conventions
 *  - Plain C: extern "C", no exceptions cross this boundary, no CUDA/torch
 *    types in the signatures.  `stream` is a cudaStream_t passed as void*
 *    (NULL = legacy default stream).
 *  - All tensor pointers are caller-owned DEVICE buffers (cudaMalloc'ed or
 *    torch storage) with explicit element counts; calls are asynchronous and
 *    stream-ordered.
 *  - Errors the reference raises from shapes/geometry are returned
 *    synchronously.  Data-dependent errors (non-finite values) are OR-ed as
 *    bits into a caller-provided device word `d_flags` (may be NULL);
 *    coat_flags_to_status() maps the word to the status the reference's
 *    exception would correspond to (errors.hpp:8-22).
 *  - Scales are stored as BF16 bit patterns (uint16_t): the reference's scales
 *    are always BF16-valued (quantize.cpp:10-17), so this is lossless.
 *  - dtype codes: 0 = fp32, 1 = bf16.
 */
#ifndef COAT_H
#define COAT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes, 1:1 with the reference exception taxonomy (errors.hpp:8-22). */
typedef enum coat_status {
    COAT_OK = 0,
    COAT_ERR_SHAPE = 1,             /* ShapeMismatch                     */
    COAT_ERR_GEOMETRY = 2,          /* GeometryMismatch                  */
    COAT_ERR_NONFINITE_INPUT = 3,   /* NonFiniteInput                    */
    COAT_ERR_NONFINITE_GRAD = 4,    /* NonFiniteGradient                 */
    COAT_ERR_INVALID = 5,           /* InvalidSpec                       */
    COAT_ERR_CUDA = 6,              /* (new) CUDA runtime error          */
    COAT_ERR_NCCL = 7,              /* (new) NCCL error                  */
    COAT_ERR_OUT_OF_RANGE = 8,      /* OutOfRange                        */
    COAT_ERR_ALL_ZERO_GROUP = 9,    /* AllZeroGroup                      */
    COAT_ERR_IO = 10,               /* IoError                           */
    COAT_ERR_BAD_MAGIC = 11         /* BadMagic                          */
} coat_status;

/* Device flag bits OR-ed into d_flags. */
#define COAT_FLAG_NONFINITE_INPUT 1u
#define COAT_FLAG_NONFINITE_GRAD 2u
#define COAT_FLAG_PACK_M 4u        /* pack_moment(m) would throw (optimizer.cpp:111) */
#define COAT_FLAG_PACK_V 8u        /* pack_moment(v) would throw (optimizer.cpp:112) */
#define COAT_FLAG_CONTRACT 16u     /* non-finite state on unpack (expand.cpp:104)    */

/* One moment of an E4M3 + DRE optimizer state, 1x128 groups
 * (ExpandedQuantState, expand.hpp:60-63 + QuantizedTensor, quantize.hpp:37-46). */
typedef struct coat_moment_state {
    uint8_t* codes;     /* [npad]   npad = ceil(n/128)*128 */
    uint16_t* scales;   /* [npad/128] BF16 bit patterns    */
    float* k;           /* [npad/128] expansion exponent   */
    float* c;           /* [npad/128] stabilizer           */
} coat_moment_state;

/* AdamWConfig (optimizer.hpp:13-20) minus the step counter (passed as t). */
typedef struct coat_adamw_config {
    float beta1, beta2, lr, weight_decay, eps;
} coat_adamw_config;

const char* coat_version(void);
const char* coat_status_string(coat_status s);
const char* coat_last_error(void);
coat_status coat_flags_to_status(uint32_t flags);
int coat_device_sm_count(void);

/* ---------------------------------------------------------------- codec -- */
/* encode_byte(x, e4m3) elementwise (fp8.hpp:47, fp8.cpp:150-156). */
coat_status coat_encode_e4m3(const float* x, uint8_t* codes, int64_t n, uint32_t* d_flags,
                             void* stream);
/* decode_byte(code, e4m3) elementwise (fp8.hpp:48, fp8.cpp:145-148). */
coat_status coat_decode_e4m3(const uint8_t* codes, float* x, int64_t n, void* stream);

/* ------------------------------------------------------------ quantizer -- */
/* quantize(x, per_group(G), e4m3) on a [rows x cols] tensor (quantize.hpp:70-71);
 * GeometryMismatch unless cols % G == 0.  scales: [rows*cols/G]. */
coat_status coat_quantize_per_group(const void* x, int dtype, int64_t rows, int64_t cols,
                                    int64_t group_size, uint8_t* codes, uint16_t* scales,
                                    uint32_t* d_flags, void* stream);
/* dequantize(QuantizedTensor) for per-group geometry (quantize.hpp:72). */
coat_status coat_dequantize_per_group(const uint8_t* codes, const uint16_t* scales, int64_t rows,
                                      int64_t cols, int64_t group_size, void* out, int out_dtype,
                                      void* stream);
/* group_scale_max(x, G) (quantize.hpp:77): stage 1 per-1xG absmax into
 * `intermediate` [rows*cols/G] (may be NULL), stage 2 global max written as
 * fp32 bits to *d_amax_bits (device). */
coat_status coat_group_scale_max(const void* x, int dtype, int64_t rows, int64_t cols,
                                 int64_t group_size, float* intermediate, uint32_t* d_amax_bits,
                                 void* stream);
/* quantize(x, per_tensor, e4m3) given the absmax from coat_group_scale_max
 * (quantize.hpp:70-71); writes the BF16 scale to *d_scale (device). */
coat_status coat_quantize_per_tensor(const void* x, int dtype, int64_t n,
                                     const uint32_t* d_amax_bits, uint8_t* codes,
                                     uint16_t* d_scale, uint32_t* d_flags, void* stream);
/* dequantize(QuantizedTensor) for per-tensor geometry (quantize.hpp:72). */
coat_status coat_dequantize_per_tensor(const uint8_t* codes, const uint16_t* d_scale, int64_t n,
                                       void* out, int out_dtype, void* stream);

/* ------------------------------------------------- batched MGAQ (layer) -- */
/* Quantize a set of saved activations in ONE launch (the MGAQ call sites of a
 * decoder layer, flow.cpp:450-480).  Per item, identical results to:
 *   group_size > 0: coat_quantize_per_group(x, dtype, rows, cols, group_size)
 *   group_size = 0: coat_group_scale_max(x, 128) + coat_quantize_per_tensor
 *                   (scales -> the one BF16 scale; d_amax_bits, if non-NULL,
 *                   receives the fp32 absmax bits)
 * Requires rows*cols % 16 == 0, x 32-byte and codes 16-byte aligned, G/16 a
 * power of two <= 32; at most 16 items.  d_flags ORs the non-finite flag of
 * every item (COAT_ERR_NONFINITE_INPUT via coat_flags_to_status). */
typedef struct coat_mgaq_item {
    const void* x;
    int32_t dtype;              /* 0 fp32, 1 bf16 */
    int32_t reserved;
    int64_t rows, cols;
    int64_t group_size;         /* > 0 per-group, 0 per-tensor (Group Scaling amax) */
    uint8_t* codes;
    uint16_t* scales;
    uint32_t* d_amax_bits;
} coat_mgaq_item;
coat_status coat_quantize_batch(const coat_mgaq_item* items, int32_t n_items, uint32_t* d_flags,
                                void* stream);

/* ----------------------------------------- fused producers + MGAQ (a17) -- */
/* The RMSNorm block of the COAT forward (flow.cpp:546-549 / 597-599):
 * x [rows, h] (fp32 / bf16) -> x_codes, x_scales = quantize(x, per_group(16))
 * (rmsnorm1.in) and y_codes, *d_y_scale = quantize(rmsnorm(DQ(...), w), per_tensor)
 * (qkv.in).  rmsnorm = flow.cpp:56-71 with the row sum in the reference's
 * sequential order: codes and scales are bit-identical to the reference's tape.
 * y never touches HBM unless y_out (fp32, may be NULL) is given; d_rms [rows]
 * and *d_amax_bits receive the row rms and y's absmax bits.  h % 16 == 0. */
coat_status coat_rmsnorm_quant(const void* x, int32_t dtype, int64_t rows, int64_t h, const float* w, float eps,
                               uint8_t* x_codes, uint16_t* x_scales, uint8_t* y_codes, uint16_t* d_y_scale,
                               float* y_out, float* d_rms, uint32_t* d_amax_bits, uint32_t* d_flags, void* stream);
/* The SiLU*mul block (flow.cpp:603-612): gate, up [rows, cols] ->
 * silu.in = Q_g16(gate), mul.in.silu = Q_g16(silu(DQ(silu.in))), mul.in.up =
 * Q_g16(up), down.in = Q_t(DQ(mul.in.silu) * DQ(mul.in.up)).  silu uses CUDA's
 * expf (the reference: glibc's); every quantizer is exact given its input.
 * p_out (fp32, may be NULL) receives the product.  cols % 16 == 0. */
coat_status coat_silu_mul_quant(const void* gate, const void* up, int32_t dtype, int64_t rows, int64_t cols,
                                uint8_t* g_codes, uint16_t* g_scales, uint8_t* s_codes, uint16_t* s_scales,
                                uint8_t* u_codes, uint16_t* u_scales, uint8_t* p_codes, uint16_t* d_p_scale,
                                float* p_out, uint32_t* d_amax_bits, uint32_t* d_flags, void* stream);

/* -------------------------------------------- backward-side MGAQ pieces -- */
/* SavedActivation::used_values_transposed (flow.cpp:360-395): out [cols, rows]
 * = decode(codes[r, c]) * scale, the per-group scales (group_size % 16 == 0;
 * 0 = per-tensor, one scale) following the original row-major grouping;
 * codes_t (may be NULL) receives the transposed codes.  out_dtype 0 fp32 /
 * 1 bf16.  Exact. */
coat_status coat_transpose_dequantize(const uint8_t* codes, const uint16_t* scales, int64_t rows, int64_t cols,
                                      int64_t group_size, void* out, int32_t out_dtype, uint8_t* codes_t,
                                      void* stream);
/* requantize_cached (flow.cpp:487-495): out = decode(encode(x / s)) * s with
 * the BF16 scale cached in the forward (*d_scale); codes (may be NULL)
 * receives the E4M3 codes.  x and out 16-byte aligned. */
coat_status coat_requantize_cached(const void* x, int32_t dtype, int64_t n, const uint16_t* d_scale, void* out,
                                   int32_t out_dtype, uint8_t* codes, uint32_t* d_flags, void* stream);

/* ------------------------------------------------------ range expansion -- */
/* expand_quantize(x, G=128, e4m3) on a flat tensor (expand.hpp:67-68);
 * GeometryMismatch unless n % G == 0; InvalidSpec for G != 128. */
coat_status coat_expand_quantize(const float* x, int64_t n, int64_t group_size,
                                 coat_moment_state out, uint32_t* d_flags, void* stream);
/* dequantize_contract(state) (expand.hpp:71). */
coat_status coat_dequantize_contract(coat_moment_state in, int64_t n, int64_t group_size,
                                     float* x, uint32_t* d_flags, void* stream);

/* ------------------------------------------------------ slot checkpoint -- */
/* save_slot / load_slot (optimizer.hpp:72-75, optimizer.cpp:196-252): the
 * {E4M3, expand, G} slot of a tensor of the given shape, state resident on the
 * device, in the reference's binary format (u32 JSON header length + header +
 * two ExpandedQuantState records, tensor_io.cpp:96-175).  Files are
 * byte-identical to the reference's for the same state; either side loads the
 * other's.  load: ShapeMismatch when the shape differs, InvalidSpec for another
 * policy, BadMagic / IoError for malformed files. */
coat_status coat_save_slot(const char* path, const int64_t* shape, int32_t rank, int64_t group_size,
                           coat_moment_state m, coat_moment_state v, const coat_adamw_config* cfg,
                           int64_t step, void* stream);
coat_status coat_load_slot(const char* path, const int64_t* shape, int32_t rank, int64_t group_size,
                           coat_moment_state m, coat_moment_state v, coat_adamw_config* cfg_out,
                           int64_t* step_out, void* stream);

/* ------------------------------------------------------------ optimizer -- */
/* make_slot(shape, {E4M3, expand, G} x2) (optimizer.hpp:54) for n params. */
coat_status coat_make_slot(int64_t n, int64_t group_size, coat_moment_state m,
                           coat_moment_state v, void* stream);
/* step(params, grads, slot, cfg) (optimizer.hpp:58) as ONE fused kernel:
 * reads w_in, g and the (m_in, v_in) state, writes w_out and (m_out, v_out).
 * t is the 1-based step being applied (slot.step + 1).  w_out may alias w_in
 * and *_out may alias *_in (in-place), but then a non-finite gradient can no
 * longer leave the parameters untouched as the reference guarantees
 * (optimizer.cpp:104); the ping-pong form keeps that guarantee. */
coat_status coat_adamw_dre_step(const float* w_in, float* w_out, const float* g, int64_t n,
                                int64_t group_size, coat_moment_state m_in,
                                coat_moment_state v_in, coat_moment_state m_out,
                                coat_moment_state v_out, const coat_adamw_config* cfg, int64_t t,
                                uint32_t* d_flags, void* stream);

/* The same step with HOST-resident params/grads (the reference's Tensor lives
 * in host memory) and the state resident in HBM: w/g are streamed through the
 * GPU in `chunk`-parameter pieces on three CUDA streams (H2D, K1, D2H
 * overlapped).  w_host_in/g_host/w_host_out should be pinned host memory;
 * w_host_out may alias w_host_in.  chunk <= 0 selects 32 Mi parameters. */
coat_status coat_adamw_dre_step_host(const float* w_host_in, float* w_host_out, const float* g_host,
                                     int64_t n, int64_t group_size, coat_moment_state m_in,
                                     coat_moment_state v_in, coat_moment_state m_out,
                                     coat_moment_state v_out, const coat_adamw_config* cfg,
                                     int64_t t, uint32_t* d_flags, int64_t chunk, void* stream);

/* ------------------------------------------------------ ZeRO step (NCCL) -- */
/* The ZeRO-sharded step (paper_2410_19313_b200/zero.py is the
 * torch.distributed form).  One process per GPU, comm = this rank's
 * ncclComm_t (as void*) of nranks ranks.  w_full, g_full: the flat [n_total]
 * fp32 buffers (FlatLayout: every tensor 128-aligned, n_total % (128*nranks) ==
 * 0); this rank owns [rank*n, (rank+1)*n), n = n_total / nranks, and only that
 * shard's state (m_in, v_in -> m_out, v_out as in coat_adamw_dre_step).
 * g_shard, w_scratch: n-float device scratch (g_shard is also reused for the
 * error-word lanes once the step has consumed it).  Stream-ordered, no host sync:
 * reduce-scatter (sum) g_full -> g_shard; the fused step on the shard into
 * w_scratch; all-reduce of the error word so *d_flags (zeroed by the caller)
 * is the OR over all ranks; when the step must change nothing
 * (NonFiniteGradient, contract NonFiniteInput) the old shard is republished;
 * all-gather w_scratch -> w_full.  After a sync the caller commits m_out,
 * v_out by coat_flags_to_status exactly as for the single-GPU step.  NCCL is
 * loaded at run time (libnccl.so.2); COAT_ERR_NCCL if absent or failing. */
coat_status coat_zero_step(float* w_full, const float* g_full, int64_t n_total, int64_t group_size,
                           coat_moment_state m_in, coat_moment_state v_in, coat_moment_state m_out,
                           coat_moment_state v_out, const coat_adamw_config* cfg, int64_t t, float* g_shard,
                           float* w_scratch, uint32_t* d_flags, void* nccl_comm, int32_t rank, int32_t nranks,
                           void* stream);
/* The same ZeRO step with the collectives done by SM kernels over NVLink peer
 * memory instead of NCCL, pipelined chunk by chunk with the
 * fused step so the reduce and the broadcast overlap it:
 *   g_shard = sum over ranks r of rank r's gradient slice [rank*n, (rank+1)*n),
 *     read in place: from g_peers[r] (P2P pointers, summed in rank order
 *     r = 0, 1, ..., fp32 or bf16 wire (g_dtype 0 / 1, exact widening)) or,
 *     when g_mc (a multicast address over the fp32 gradient buffers) is
 *     given, by NVLink SHARP multimem.ld_reduce;
 *   w_next[shard] = the fused step of w_cur[shard] (coat_adamw_dre_step);
 *   every rank's next-weight buffer receives the shard: P2P stores into
 *     w_next_peers[r] (r != rank) -- issued by the step kernel itself right
 *     after each local store (up to 8 ranks; a ragged chunk tail and larger
 *     worlds by a broadcast kernel) -- or multimem.st into w_next_mc.
 * n = n_total / nranks as for coat_zero_step; w_cur / w_next are this rank's
 * full buffers (double-buffered: nothing the step reads is overwritten).
 * Stream-ordered; the caller synchronizes the ranks (e.g. an all-reduce of the
 * error word) before reading w_next or rewriting its gradients, then commits
 * m_out, v_out and w_next -- or keeps w_cur and the old state -- by the OR of
 * every rank's *d_flags (coat_flags_to_status), exactly as the reference's
 * step commits or throws as a whole (optimizer.cpp:101-114).  chunk <= 0:
 * 64 Mi parameters.  nranks <= 16. */
coat_status coat_zero_step_p2p(const void* const* g_peers, const void* g_mc, int32_t g_dtype,
                               float* const* w_next_peers, float* w_next_mc, const float* w_cur, float* w_next,
                               int64_t n_total, int64_t group_size, coat_moment_state m_in,
                               coat_moment_state v_in, coat_moment_state m_out, coat_moment_state v_out,
                               const coat_adamw_config* cfg, int64_t t, float* g_shard, uint32_t* d_flags,
                               int32_t rank, int32_t nranks, int64_t chunk, void* stream);
/* Communicator helpers for callers without their own NCCL binding: rank 0
 * creates the 128-byte id, every rank passes it to coat_nccl_comm_init. */
coat_status coat_nccl_unique_id(uint8_t* out_id /* 128 bytes */);
coat_status coat_nccl_comm_init(void** nccl_comm, int32_t nranks, const uint8_t* id, int32_t rank);
coat_status coat_nccl_comm_destroy(void* nccl_comm);

/* ----------------------------------------------------------- FP8 linear -- */
/* The reference's linear (flow.cpp:21-46, no public entry point; SURVEY.md 8(a)
 * a18) on tcgen05/TMEM/TMA.  W is (K, N) row-major as in flow.hpp:44-47.
 * Scales are the BF16 device scalars written by coat_quantize_per_tensor.
 * Constraints: K % 16 == 0, N % 16 == 0, 16-byte aligned buffers. */
/* y[M,N] (fp32) = DQ(x)[M,K] . DQ(W)[K,N] = (s_x s_w) * codes_x . codes_w */
coat_status coat_fp8_linear_fwd(const uint8_t* x_codes, const uint16_t* d_sx, const uint8_t* w_codes,
                                const uint16_t* d_sw, int64_t M, int64_t K, int64_t N, float* y,
                                void* stream);
/* The same y quantized per group of 16 in the GEMM epilogue:
 * y_codes [M,N] / y_scales [M,N/16] = quantize(y, per_group(16)) bit for bit
 * as coat_quantize_per_group would encode coat_fp8_linear_fwd's y; y never
 * reaches HBM unless y_out (fp32, may be NULL) is given.  Non-finite y ->
 * NONFINITE_INPUT in *d_flags (quantize.cpp:91). */
coat_status coat_fp8_linear_fwd_q16(const uint8_t* x_codes, const uint16_t* d_sx, const uint8_t* w_codes,
                                    const uint16_t* d_sw, int64_t M, int64_t K, int64_t N, uint8_t* y_codes,
                                    uint16_t* y_scales, float* y_out, uint32_t* d_flags, void* stream);
/* The MLP's gate/up projections and the SiLU*mul block in one tcgen05 GEMM
 * (flow.cpp:599-610): gate = DQ(x) . DQ(W_gate), up = DQ(x) . DQ(W_up) (W (H, I)
 * row-major), the epilogue writes silu.in = Q_g16(gate), mul.in.silu =
 * Q_g16(silu(DQ(silu.in))), mul.in.up = Q_g16(up) and the product absmax; a
 * second pass encodes down.in = Q_t(DQ(mul.in.silu) * DQ(mul.in.up)) from the
 * codes.  Outputs equal coat_silu_mul_quant applied to the two
 * coat_fp8_linear_fwd outputs.  gate_out / up_out / p_out: optional fp32
 * side outputs (NULL: gate and up never reach HBM).  I % 16 == 0. */
coat_status coat_fp8_upgate_silu_quant(const uint8_t* x_codes, const uint16_t* d_sx, const uint8_t* wg_codes,
                                       const uint16_t* d_swg, const uint8_t* wu_codes, const uint16_t* d_swu,
                                       int64_t M, int64_t H, int64_t I, uint8_t* g_codes, uint16_t* g_scales,
                                       uint8_t* s_codes, uint16_t* s_scales, uint8_t* u_codes, uint16_t* u_scales,
                                       uint8_t* p_codes, uint16_t* d_p_scale, float* gate_out, float* up_out,
                                       float* p_out, uint32_t* d_amax_bits, uint32_t* d_flags, void* stream);
/* dX[M,K] (bf16) = bf16(dY[M,N] . W_used^T), W_used = s_w * w_dec (flow.cpp:636);
 * w_dec = coat_decode_e4m3_bf16(w_codes), exact. */
coat_status coat_linear_bwd_dgrad(const uint16_t* dy_bf16, const uint16_t* w_dec_bf16,
                                  const uint16_t* d_sw, int64_t M, int64_t K, int64_t N,
                                  uint16_t* dx_bf16, void* stream);
/* dW[K,N] (fp32) = X_used^T . dY, X_used = s_x * x_dec (flow.cpp:637, 360-395). */
coat_status coat_linear_bwd_wgrad(const uint16_t* x_dec_bf16, const uint16_t* d_sx,
                                  const uint16_t* dy_bf16, int64_t M, int64_t K, int64_t N,
                                  float* dw, void* stream);
/* decode_byte(code) as BF16 bits (exact: E4M3 values have <= 4 significant bits). */
coat_status coat_decode_e4m3_bf16(const uint8_t* codes, uint16_t* out_bf16, int64_t n, void* stream);

/* Test/diagnostic hook: count elements that took the literal (double pow)
 * fallback in DRE kernels into *d_counter (device u64); NULL disables. */
coat_status coat_set_fallback_counter(unsigned long long* d_counter);

#ifdef __cplusplus
}
#endif
#endif /* COAT_H */
