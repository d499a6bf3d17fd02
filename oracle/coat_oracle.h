/* oracle/coat_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference (coatsim, /root/reference/proj/core)
 * numerics on the COAT hot path, used as the CPU checker for the CUDA
 * kernels.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it; the product (paper_2410_19313_b200/) never does.
 *
 * Pinned against the compiled reference (oracle/_ref/libcoatsim_ref.so) and
 * the reference's own known-answer tests; see tests/test_oracle.py.
 *
 * Status codes are the coat_status numbering of include/coat.h.
 */
#ifndef COAT_ORACLE_H
#define COAT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* fp8.cpp:53-88 (encode_minifloat), 150-156 (encode_byte): returns -1 for non-finite. */
int oracle_encode_e4m3_one(float x);
float oracle_decode_e4m3_one(uint8_t b);               /* fp8.cpp:27-51 */
float oracle_round_bf16_one(float x);                   /* fp8.cpp:209-216 */
int oracle_encode_e4m3(const float* x, uint8_t* out, int64_t n);
int oracle_decode_e4m3(const uint8_t* codes, float* out, int64_t n);

/* quantize.cpp:89-111, per-group (1xG runs along the last dim) on rows x cols;
 * G == cols*rows with rows==1 or mode per-tensor: pass G = 0 for per-tensor. */
int oracle_quantize(const float* x, int64_t rows, int64_t cols, int64_t G, uint8_t* codes,
                    float* scales);
int oracle_dequantize(const uint8_t* codes, const float* scales, int64_t rows, int64_t cols,
                      int64_t G, float* out);                       /* quantize.cpp:113-124 */
int oracle_group_scale_max(const float* x, int64_t rows, int64_t cols, int64_t G,
                           float* intermediate, float* global);     /* quantize.cpp:126-145 */

/* expand.cpp:50-83 */
void oracle_optimal_k(double range, float* k, int* degenerate);
void oracle_measure_group(const float* x, int64_t n, float* k, float* c, float* range,
                          int* degenerate);
/* expand.cpp:115-141 over a flat tensor of n elements, n % G == 0 */
int oracle_expand_quantize(const float* x, int64_t n, int64_t G, uint8_t* codes, float* scales,
                           float* k, float* c);
int oracle_dequantize_contract(const uint8_t* codes, const float* scales, const float* k,
                               const float* c, int64_t n, int64_t G, float* out);

/* optimizer.cpp:90-114 with the policy {E4M3, expand, G} for both moments.
 * State arrays hold npad = ceil(n/G)*G codes and npad/G scales/k/c. */
int oracle_make_slot(int64_t n, int64_t G, uint8_t* mc, float* ms, float* mk, float* mcc,
                     uint8_t* vc, float* vs, float* vk, float* vcc);
int oracle_step(float* w, const float* g, int64_t n, int64_t G, uint8_t* mc, float* ms,
                float* mk, float* mcc, uint8_t* vc, float* vs, float* vk, float* vcc,
                int64_t step_in, float b1, float b2, float lr, float wd, float eps);
/* optimizer.cpp:116-131 */
void oracle_reference_adamw_step(float* w, float* m, float* v, const float* g, int64_t n,
                                 float b1, float b2, float lr, float wd, float eps, int64_t t);

/* synthetic.cpp:28-66 + rng.hpp:20-73.  kind 0 OptimizerLike, 1 ActivationWithOutliers
 * (rows x cols), 2 UniformLog. */
int oracle_generate(int kind, int64_t rows, int64_t cols, double frac, double scale,
                    uint64_t seed, float* out);
uint64_t oracle_splitmix64_at(uint64_t seed, uint64_t i); /* i-th output of SplitMix64(seed) */
/* flow.cpp:21-33 */
void oracle_matmul(const float* a, const float* b, int64_t m, int64_t k, int64_t n, float* out);

/* producers (flow.cpp:56-71, 97-100) */
void oracle_rmsnorm(const float* x, const float* w, int64_t rows, int64_t h, float eps, float* out);
void oracle_silu(const float* x, int64_t n, float* out);

#ifdef __cplusplus
}
#endif
#endif
