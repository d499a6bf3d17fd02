// coat_internal.h -- host-side declarations shared by the .cu translation units
// (not part of the public C-ABI; see include/coat.h for that).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace coat {

struct MomentStateIn {
    const uint8_t* codes;     // [npad]
    const uint16_t* scales;   // [npad/128], BF16 bit patterns (scales are BF16-valued)
    const float* k;           // [npad/128]
    const float* c;           // [npad/128]
};

struct MomentStateOut {
    uint8_t* codes;
    uint16_t* scales;
    float* k;
    float* c;
};

struct AdamWScalars {
    float beta1, beta2, lr, weight_decay, eps;
    float bc1, bc2;           // 1 - powf(beta, t), computed on the host like optimizer.cpp:58-59
    double log_target;        // log(229376.0), expand.cpp:52
};

int device_sm_count();

cudaError_t launch_adamw_dre_step(const float* w_in, float* w_out, const float* g, int64_t n,
                                  const MomentStateIn& m_in, const MomentStateIn& v_in,
                                  const MomentStateOut& m_out, const MomentStateOut& v_out,
                                  const AdamWScalars& a, uint32_t* flags,
                                  unsigned long long* fallbacks, cudaStream_t stream);
int k1_ws_config();              // element warps per CTA of the selected layout (COAT_K1_EW)
int64_t k1_ws_round_params();   // parameters per k1_ws round (2048; COAT_K1_EW=7: 1792, =6: 1536)
cudaError_t launch_k1_ws(const float* w_in, float* w_out, const float* g, int64_t nrounds,
                         const MomentStateIn& m_in, const MomentStateIn& v_in, const MomentStateOut& m_out,
                         const MomentStateOut& v_out, const AdamWScalars& a, uint32_t* flags,
                         cudaStream_t stream, const int64_t* peer_delta = nullptr, int npeers = 0);
// The step with the ZeRO all-gather fused into K1: whole rounds also store w'
// into each peer's next-weight buffer (w_out + peer_delta[p], float offsets);
// *fused = how many leading parameters went to the peers (the rest -- a ragged
// tail, or everything when the fused kernel does not apply -- is the caller's
// to broadcast).
cudaError_t launch_adamw_dre_step_peers(const float* w_in, float* w_out, const float* g, int64_t n,
                                        const MomentStateIn& m_in, const MomentStateIn& v_in,
                                        const MomentStateOut& m_out, const MomentStateOut& v_out,
                                        const AdamWScalars& a, uint32_t* flags, const int64_t* peer_delta,
                                        int npeers, int64_t* fused, cudaStream_t stream);
cudaError_t launch_expand_quantize_fast(const float* x, int64_t ntiles, const MomentStateOut& out,
                                        double log_target, uint32_t* flags, cudaStream_t stream);
cudaError_t launch_dequantize_contract_fast(const MomentStateIn& in, int64_t ntiles, float* x, uint32_t* flags,
                                            cudaStream_t stream);
cudaError_t launch_expand_quantize(const float* x, int64_t n, const MomentStateOut& out,
                                   double log_target, uint32_t* flags,
                                   unsigned long long* fallbacks, cudaStream_t stream);
cudaError_t launch_dequantize_contract(const MomentStateIn& in, int64_t n, float* x,
                                       uint32_t* flags, cudaStream_t stream);
cudaError_t launch_make_slot(const MomentStateOut& st, int64_t npad, cudaStream_t stream);

// host_pipeline.cu: host-resident w/g streamed through K1 (state in HBM)
}  // namespace coat
#include "../../include/coat.h"
namespace coat {
// zero_p2p.cu: the ZeRO step with peer-memory (P2P / NVLink SHARP) collectives
struct ZeroP2PArgs {
    const void* const* g_peers;   // [nranks] every rank's full gradient buffer (fp32 / bf16), or NULL with g_mc
    const void* g_mc;             // multicast address of the gradient buffers (fp32), or NULL
    int g_dtype;                  // 0 fp32, 1 bf16 (P2P only)
    float* const* w_next_peers;   // [nranks] every rank's next-weight buffer, or NULL with w_next_mc
    float* w_next_mc;             // multicast address of the next-weight buffers, or NULL
    const float* w_cur;           // this rank's full current weights
    float* w_next;                // this rank's full next-weight buffer
    int64_t n_shard;
    coat_moment_state m_in, v_in, m_out, v_out;
    float* g_shard;               // n_shard floats of scratch: the reduced gradient shard
    int rank, nranks;
    int64_t chunk;
};
cudaError_t zero_p2p_step(const ZeroP2PArgs& z, const AdamWScalars& a, uint32_t* flags,
                          unsigned long long* fallbacks, cudaStream_t stream);
}  // namespace coat
#include <string>
#include "../../include/coat.h"
namespace coat {
cudaError_t host_pipelined_step(const float* w_host_in, float* w_host_out, const float* g_host, int64_t n,
                                const coat_moment_state& m_in, const coat_moment_state& v_in,
                                const coat_moment_state& m_out, const coat_moment_state& v_out,
                                const AdamWScalars& a, uint32_t* flags, unsigned long long* fallbacks,
                                int64_t chunk, cudaStream_t stream);

// slot checkpoints (slot_io.cu)
coat_status save_slot_impl(const char* path, const int64_t* shape, int rank, int64_t G, const coat_moment_state& m,
                           const coat_moment_state& v, const coat_adamw_config& cfg, int64_t step,
                           cudaStream_t s, std::string& err);
coat_status load_slot_impl(const char* path, const int64_t* shape, int rank, int64_t G, const coat_moment_state& m,
                           const coat_moment_state& v, coat_adamw_config* cfg, int64_t* step, cudaStream_t s,
                           std::string& err);

// tcgen05 GEMMs (gemm_tcgen05.cu)
cudaError_t launch_fp8_linear_fwd(const uint8_t* xc, const uint16_t* sx, const uint8_t* wc, const uint16_t* sw, int M,
                                  int K, int N, float* y, cudaStream_t st);
cudaError_t launch_fp8_linear_fwd_q16(const uint8_t* xc, const uint16_t* sx, const uint8_t* wc, const uint16_t* sw,
                                      int M, int K, int N, uint8_t* y_codes, uint16_t* y_scales, float* y_out,
                                      uint32_t* flags, cudaStream_t st);
struct UpGateArgs {
    const uint8_t* xc;      // upgate.in codes [M, H], per-tensor scale *sx
    const uint16_t* sx;
    const uint8_t* wg;      // W_gate codes (H, I) row-major, scale *s_wg
    const uint16_t* s_wg;
    const uint8_t* wu;      // W_up codes (H, I), scale *s_wu
    const uint16_t* s_wu;
    int64_t M, H, I;
    uint8_t* gcodes; uint16_t* gscales;   // silu.in
    uint8_t* scodes; uint16_t* sscales;   // mul.in.silu
    uint8_t* ucodes; uint16_t* uscales;   // mul.in.up
    uint8_t* pcodes; uint16_t* pscale;    // down.in (per-tensor)
    float* gate_out; float* up_out; float* pout;   // optional fp32 side outputs (tests)
    uint32_t* amax_bits;
    uint32_t* flags;
};
cudaError_t launch_fp8_upgate_silu(const UpGateArgs& a, cudaStream_t st);
cudaError_t launch_linear_dgrad(const uint16_t* dy, const uint16_t* wd, const uint16_t* sw, int M, int K, int N,
                                uint16_t* dx, cudaStream_t st);
cudaError_t launch_linear_wgrad(const uint16_t* xd, const uint16_t* sx, const uint16_t* dy, int M, int K, int N,
                                float* dw, cudaStream_t st);
cudaError_t launch_decode_e4m3_bf16(const uint8_t* codes, uint16_t* out, int64_t n, cudaStream_t st);

// batched MGAQ (mgaq_batch.cu): one cooperative launch for a layer's quantizations
constexpr int kMgaqMaxItems = 16;
struct MgaqItem {
    const void* x;
    int dtype;              // 0 fp32, 1 bf16
    int64_t n;              // elements (multiple of 16, 32-byte aligned x)
    int64_t group_size;     // > 0: per-group(G), G/16 a power of two <= 32; 0: per-tensor
    uint8_t* codes;
    uint16_t* scales;       // [n/G] or one BF16 scale
    uint32_t* amax_out;     // per-tensor: fp32 absmax bits (may be NULL)
};
cudaError_t launch_mgaq_batch(const MgaqItem* items, int n, uint32_t* flags, cudaStream_t stream);
cudaError_t launch_mgaq_streams(const MgaqItem* items, int n, uint32_t* flags, cudaStream_t stream);
cudaError_t launch_mgaq_queue(const MgaqItem* items, int n, uint32_t* flags, cudaStream_t stream);
bool mgaq_batch_cooperative();
bool mgaq_batch_queue();
// first 16-element chunk of a per-tensor input kept L2-resident between its
// absmax and encode passes (act_quant.cu; COAT_L2_KEEP_MB)
int64_t l2_keep_chunks(int64_t nchunks, int esz);

// fused producers (producers.cu)
struct RmsBlockArgs {
    const void* x;
    int dtype;
    int64_t rows, h;
    const float* w;
    float eps;
    uint8_t* xcodes;
    uint16_t* xscales;
    uint8_t* ycodes;
    uint16_t* yscale;
    float* yout;        // may be NULL
    float* rms;         // [rows]
    uint32_t* amax_bits;
    uint32_t* flags;
};
struct SiluBlockArgs {
    const void* gate;
    const void* up;
    int dtype;
    int64_t n;
    uint8_t* gcodes;
    uint16_t* gscales;
    uint8_t* scodes;
    uint16_t* sscales;
    uint8_t* ucodes;
    uint16_t* uscales;
    uint8_t* pcodes;
    uint16_t* pscale;
    float* pout;        // may be NULL
    uint32_t* amax_bits;
    uint32_t* flags;
};
cudaError_t launch_rmsnorm_block(const RmsBlockArgs& a, cudaStream_t stream);
cudaError_t launch_silu_mul_block(const SiluBlockArgs& a, cudaStream_t stream);
// pass 2 of the SiLU*mul block alone: down.in = Q_t(DQ(s) * DQ(u)) from the
// global product absmax (*amax_bits)
cudaError_t launch_silu_mul_pass2(const uint8_t* scodes, const uint16_t* sscales, const uint8_t* ucodes,
                                  const uint16_t* uscales, int64_t n, const uint32_t* amax_bits, uint8_t* pcodes,
                                  uint16_t* pscale, float* pout, uint32_t* flags, cudaStream_t stream);

// backward-side MGAQ pieces (mgaq_bwd.cu)
cudaError_t launch_transpose_dequant(const uint8_t* codes, const uint16_t* scales, int64_t rows, int64_t cols,
                                     int64_t G, void* out, int out_dtype, uint8_t* codes_t, cudaStream_t stream);
cudaError_t launch_requantize_cached(const void* x, int dtype, int64_t n, const uint16_t* scale, void* out,
                                     int out_dtype, uint8_t* codes, uint32_t* flags, cudaStream_t stream);

// activation quantizers (act_quant.cu)
cudaError_t launch_encode_e4m3(const float* x, uint8_t* out, int64_t n, uint32_t* flags,
                               cudaStream_t stream);
cudaError_t launch_decode_e4m3(const uint8_t* codes, float* out, int64_t n, cudaStream_t stream);
cudaError_t launch_quantize_per_group(const void* x, int dtype, int64_t n, int64_t G,
                                      uint8_t* codes, uint16_t* scales, uint32_t* flags,
                                      cudaStream_t stream);
cudaError_t launch_dequantize_per_group(const uint8_t* codes, const uint16_t* scales, int64_t n,
                                        int64_t G, void* out, int out_dtype, cudaStream_t stream);
cudaError_t launch_group_amax(const void* x, int dtype, int64_t n, int64_t G, float* intermediate,
                              uint32_t* global_bits, uint32_t* flags, cudaStream_t stream);
cudaError_t launch_quantize_per_tensor(const void* x, int dtype, int64_t n,
                                       const uint32_t* amax_bits, uint8_t* codes,
                                       uint16_t* scale_out, uint32_t* flags, cudaStream_t stream);

// ZeRO collectives (zero_nccl.cu); NCCL results as int (0 = ncclSuccess, -1 = no NCCL library)
bool nccl_available();
const char* nccl_error_string(int r);
int nccl_unique_id(uint8_t* out128);
int nccl_comm_init(void** comm, int nranks, const uint8_t* id128, int rank);
int nccl_comm_destroy(void* comm);
int zero_reduce_scatter(const float* g_full, float* g_shard, int64_t n_shard, void* comm, cudaStream_t st);
int zero_all_gather(const float* w_shard, float* w_full, int64_t n_shard, void* comm, cudaStream_t st);
int zero_agree_and_select(uint32_t* d_flags, const float* w_old, float* w_scratch, int64_t n_shard, void* comm,
                          uint8_t* lanes, cudaStream_t st, cudaError_t* cuda_err);

}  // namespace coat
