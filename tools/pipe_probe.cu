// pipe_probe.cu -- diagnostic: bandwidth ceiling of K1's TMA round pipeline
// with the math removed.  Same traffic per parameter as K1 (read w, g, m/v
// codes; write w, m/v codes; metadata ignored), same CTA shape (EW consumer
// warps + 1 producer warp), parameterised stage count and round size.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_probe pipe_probe.cu
//   ./pipe_probe [log2 params]
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(unsigned long long* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mb_arrive(unsigned long long* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory"); }
__device__ __forceinline__ void mb_tx(unsigned long long* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void g2s(void* d, const void* s, uint32_t n, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(d)), "l"(s), "r"(n), "r"(su(b)) : "memory"); }
__device__ __forceinline__ void mb_wait(unsigned long long* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n@!p bra W_%=;\n}\n" ::"r"(su(b)), "r"(ph) : "memory"); }

template <int EW, int RG, int NS, int HOLD = 1>   // consumer warps, groups per round, stages, rounds a stage is held after use (K1 parks m', v': 1)
__global__ void __launch_bounds__((EW + 1) * 32) probe(const float* w, float* wo, const float* g, const uint8_t* cm,
    const uint8_t* cv, uint8_t* cmo, uint8_t* cvo, uint32_t nrounds_total) {
  constexpr int R = RG * 128;
  constexpr uint32_t SB = R * 10;
  extern __shared__ __align__(128) uint8_t sm[];
  unsigned long long* bS = (unsigned long long*)sm;
  unsigned long long* bF = bS + NS;
  uint8_t* stg = sm + 256;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { for (int i = 0; i < NS; ++i) { mb_init(&bS[i], 1); mb_init(&bF[i], EW); } asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  const uint32_t nr = blockIdx.x < nrounds_total ? (nrounds_total - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto base = [&](uint32_t r) { return (int64_t(blockIdx.x) + int64_t(r) * gridDim.x) * R; };
  if (warp == EW) {
    if (lane == 0) {
      for (uint32_t r = 0; r < nr; ++r) {
        const int s = r % NS;
        if (r >= NS) mb_wait(&bF[s], ((r / NS) - 1) & 1);
        uint8_t* st = stg + s * SB;
        mb_tx(&bS[s], SB);
        const int64_t b = base(r);
        g2s(st, w + b, R * 4, &bS[s]); g2s(st + R * 4, g + b, R * 4, &bS[s]);
        g2s(st + R * 8, cm + b, R, &bS[s]); g2s(st + R * 9, cv + b, R, &bS[s]);
      }
    }
  } else {
    for (uint32_t r = 0; r < nr; ++r) {
      const int s = r % NS;
      mb_wait(&bS[s], (r / NS) & 1);
      const uint8_t* st = stg + s * SB;
      const int64_t b = base(r);
      for (int gl = warp; gl < RG; gl += EW) {
        const float4 a = *(const float4*)(st + (gl * 128 + 4 * lane) * 4);
        const float4 c = *(const float4*)(st + R * 4 + (gl * 128 + 4 * lane) * 4);
        const uint32_t x = *(const uint32_t*)(st + R * 8 + gl * 128 + 4 * lane);
        const uint32_t y = *(const uint32_t*)(st + R * 9 + gl * 128 + 4 * lane);
        float4 o = make_float4(a.x + c.x, a.y + c.y, a.z + c.z, a.w + c.w);
        asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(wo + b + gl * 128 + 4 * lane), "f"(o.x), "f"(o.y), "f"(o.z), "f"(o.w) : "memory");
        asm volatile("st.global.L1::no_allocate.b32 [%0], %1;" :: "l"(cmo + b + gl * 128 + 4 * lane), "r"(x ^ y) : "memory");
        asm volatile("st.global.L1::no_allocate.b32 [%0], %1;" :: "l"(cvo + b + gl * 128 + 4 * lane), "r"(x + y) : "memory");
      }
      __syncwarp();
      if (lane == 0 && r >= HOLD) mb_arrive(&bF[(r - HOLD) % NS]);
    }
  }
}

template <int EW, int RG, int NS, int HOLD = 1>
void run(const char* name, int64_t n, float* w, float* wo, float* g, uint8_t* cm, uint8_t* cv, uint8_t* cmo, uint8_t* cvo) {
  const size_t smem = 256 + size_t(NS) * RG * 128 * 10;
  cudaFuncSetAttribute(probe<EW, RG, NS, HOLD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, probe<EW, RG, NS, HOLD>, (EW + 1) * 32, smem);
  int dev; cudaGetDevice(&dev); int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t nr = n / (RG * 128);
  const int grid = sms * per;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 2; ++i) probe<EW, RG, NS, HOLD><<<grid, (EW + 1) * 32, smem>>>(w, wo, g, cm, cv, cmo, cvo, nr);
  cudaEventRecord(a);
  const int it = 5;
  for (int i = 0; i < it; ++i) probe<EW, RG, NS, HOLD><<<grid, (EW + 1) * 32, smem>>>(w, wo, g, cm, cv, cmo, cvo, nr);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= it;
  const double bytes = double(n) * 14.0;   // w r/w 8, g 4, codes r/w 2 x 2 ... (w 8 + g 4 + codes 4 = 16; meta excluded) 
  printf("%-28s ctas/SM %d smem %6zu KB  %.3f ms  %.0f GB/s (16 B/param: %.0f GB/s)  err=%s\n", name, per, smem / 1024, ms,
         bytes / ms / 1e6, double(n) * 16.0 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
  const int lg = argc > 1 ? atoi(argv[1]) : 30;
  const int64_t n = int64_t(1) << lg;
  float *w, *wo, *g; uint8_t *cm, *cv, *cmo, *cvo;
  cudaMalloc(&w, n * 4); cudaMalloc(&wo, n * 4); cudaMalloc(&g, n * 4);
  cudaMalloc(&cm, n); cudaMalloc(&cv, n); cudaMalloc(&cmo, n); cudaMalloc(&cvo, n);
  cudaMemset(w, 0, n * 4); cudaMemset(g, 0, n * 4); cudaMemset(cm, 0, n); cudaMemset(cv, 0, n);
  run<8, 16, 3>("EW8 RG16 NS3 (K1 now)", n, w, wo, g, cm, cv, cmo, cvo);
  run<8, 16, 3, 0>("EW8 RG16 NS3 hold0", n, w, wo, g, cm, cv, cmo, cvo);
  run<8, 16, 2>("EW8 RG16 NS2", n, w, wo, g, cm, cv, cmo, cvo);
  run<8, 16, 4>("EW8 RG16 NS4", n, w, wo, g, cm, cv, cmo, cvo);
  run<8, 16, 5>("EW8 RG16 NS5", n, w, wo, g, cm, cv, cmo, cvo);
  run<8, 8, 6>("EW8 RG8 NS6", n, w, wo, g, cm, cv, cmo, cvo);
  run<8, 8, 8>("EW8 RG8 NS8", n, w, wo, g, cm, cv, cmo, cvo);
  run<16, 32, 3>("EW16 RG32 NS3", n, w, wo, g, cm, cv, cmo, cvo);
  run<16, 32, 4>("EW16 RG32 NS4", n, w, wo, g, cm, cv, cmo, cvo);
  run<4, 8, 4>("EW4 RG8 NS4", n, w, wo, g, cm, cv, cmo, cvo);
  run<4, 8, 8>("EW4 RG8 NS8", n, w, wo, g, cm, cv, cmo, cvo);
  return 0;
}
