// Per-SM TMA landing throughput in the batch-1 GEMM regime (development tool, not shipped).
// G CTAs; each loads S stages x 2 boxes of 64 rows x 128 B (the GEMM's B operand of a
// [cout][K] weight matrix, K = 384 halves) into S separate slots, one mbarrier per
// stage, and records when each stage lands (CTA 0) -- mode 0: 2-D tensor-map boxes
// (row-fragmented, 768-B row pitch); mode 1: 1-D cp.async.bulk of the same bytes from a
// pre-tiled (contiguous 8 KB) copy.  Cold = 256 MB written between runs (L2 flushed).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmabw scripts/tma_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr int kMaxS = 8;

__global__ void bench(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap ta,
                      const char* tiled, int S, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[kMaxS];
  uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~uintptr_t(1023));
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint32_t box = 64 * 128;
  const int ntile = blockIdx.x;                   // this CTA's 64 output rows
  unsigned long long t0 = gt();
  for (int s = 0; s < S; ++s) {
    const uint32_t abytes = mode == 2 ? 49 * 128 : (mode == 3 ? 128 * 128 : box);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(abytes + box));
    for (int j = 0; j < 2; ++j) {
      uint8_t* dst = buf + (2 * s + j) * 2 * box;
      const int kstep = 2 * s + j;                // 64-wide K block
      if (mode == 2 && j == 0) {      // 4-D activation box (64 ch, 7 w, 7 h, 1 n): 49 rows
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
                su32(dst)),
            "l"(&ta), "r"(su32(&bar[s])), "r"((kstep % 6) * 64), "r"(0), "r"(0), "r"(0)
            : "memory");
      } else if (mode == 3 && j == 0) {   // 2-D activation box (64 ch, 128 pixel rows), OOB past 49
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                su32(dst)),
            "l"(&ta), "r"(su32(&bar[s])), "r"((kstep % 6) * 64), "r"(0)
            : "memory");
      } else if (mode != 1) {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                su32(dst)),
            "l"(&tm), "r"(su32(&bar[s])), "r"((kstep % 6) * 64), "r"(ntile * 64)
            : "memory");
      } else {
        const char* src = tiled + ((size_t)ntile * 12 + (kstep % 12)) * box;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(dst)),
                     "l"(src), "r"(box), "r"(su32(&bar[s]))
                     : "memory");
      }
    }
  }
  unsigned long long t1 = gt();
  for (int s = 0; s < S; ++s) {
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(su32(&bar[s]))
                   : "memory");
    if (blockIdx.x == 0) out[2 + s] = gt() - t0;
  }
  if (blockIdx.x == 0) out[0] = t1 - t0;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int K = 384, COUT = 148 * 64;             // weights [COUT][K] halves
  const size_t wbytes = size_t(COUT) * K * 2;
  char *w, *tiled, *flush;
  cudaMalloc(&w, wbytes);
  cudaMalloc(&tiled, wbytes * 2);
  cudaMalloc(&flush, 256 << 20);
  cudaMemset(w, 1, wbytes);
  cudaMemset(tiled, 1, wbytes * 2);
  unsigned long long* out;
  cudaMalloc(&out, 8 * 16);
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {cuuint64_t(K), cuuint64_t(COUT)};
  cuuint64_t strides[1] = {cuuint64_t(K) * 2};
  cuuint32_t boxd[2] = {64, 64}, es[2] = {1, 1};
  CUresult r = ((EncFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, w, dims, strides, boxd, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) { printf("encode %d\n", r); return 1; }
  char* act;
  cudaMalloc(&act, 64 * 384 * 2 * 4);
  cudaMemset(act, 1, 64 * 384 * 2 * 4);
  CUtensorMap ta4, ta2;
  {
    cuuint64_t d4[4] = {384, 7, 7, 1}, s4[3] = {384 * 2, 7 * 384 * 2, 49 * 384 * 2};
    cuuint32_t b4[4] = {64, 7, 7, 1}, e4[4] = {1, 1, 1, 1};
    r = ((EncFn)fn)(&ta4, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, act, d4, s4, b4, e4, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("encode4 %d\n", r); return 1; }
    cuuint64_t d2[2] = {384, 49}, s2[1] = {384 * 2};
    cuuint32_t b2[2] = {64, 128}, e2[2] = {1, 1};
    r = ((EncFn)fn)(&ta2, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, act, d2, s2, b2, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("encode2 %d\n", r); return 1; }
  }
  const int smem = 12 * 16384 + 1024;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int S = 6;
  for (int cold = 0; cold < 2; ++cold)
    for (int mode = 0; mode < 4; ++mode)
      for (int G : {1, 36, 148}) {
        const CUtensorMap& ta = mode == 2 ? ta4 : ta2;
        float best = 1e9;
        unsigned long long h[2 + kMaxS];
        for (int rep = 0; rep < 5; ++rep) {
          if (cold) cudaMemset(flush, rep, 256 << 20);
          else bench<<<G, 128, smem>>>(tm, ta, tiled, S, mode, out);
          cudaEventRecord(e0);
          bench<<<G, 128, smem>>>(tm, ta, tiled, S, mode, out);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best) {
            best = ms;
            cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
          }
        }
        const double bytes = double(G) * S * 2 * 64 * 128;
        static const char* mn[4] = {"tma2d ", "bulk1d", "A4d+B2d", "A2d+B2d"};
        printf("%s %s G=%3d: kernel %6.2f us (%6.0f GB/s total, %5.1f GB/s/SM)  CTA0 issue %.2f us, landed:",
               cold ? "cold" : "warm", mn[mode], G, best * 1e3, bytes / (best * 1e-3) / 1e9,
               bytes / G / (best * 1e-3) / 1e9, h[0] / 1e3);
        for (int s = 0; s < S; ++s) printf(" %.2f", h[2 + s] / 1e3);
        printf("\n");
      }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
