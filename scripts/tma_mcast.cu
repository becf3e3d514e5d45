// Batch-1 A-operand landing time when many CTAs read the SAME activation tile
// (development tool, not shipped).  A 1x1-conv A operand of a 7x7 map: P = 49
// pixel rows x K channels (fp16, 128-B swizzled boxes of 64 channels x 49 rows),
// S = K / 64 stages.  G CTAs (one per SM), each needs all S stages:
//   mode 0: every CTA loads the same tile (what gemm_kernel does: the N tiles of
//           one M tile share A, all from the same L2 lines);
//   mode 1: every CTA loads its own copy (distinct lines; the no-contention bound);
//   mode 2: clusters of CL CTAs, CTA rank r issues stages s = r (mod CL) with
//           .multicast::cluster to all CL CTAs (1/CL of the L2 requests).
// Reports per-CTA time from the first issue to the last stage landed (median and
// max over CTAs).  L2 warm (the tile was just read).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmamc scripts/tma_mcast.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release;\nbarrier.cluster.wait.acquire;" ::: "memory");
}

constexpr int kMaxS = 16;

__global__ void bench(const __grid_constant__ CUtensorMap tm, int S, int P, int mode, int CL,
                      unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[kMaxS];
  uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~uintptr_t(1023));
  const uint32_t box_bytes = P * 128;
  const uint32_t stage_pitch = (box_bytes + 1023) & ~1023u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm) : "memory");
  }
  __syncthreads();
  if (mode == 2) cluster_sync();
  if (threadIdx.x != 0) {
    if (mode == 2) cluster_sync();
    return;
  }
  const int row0 = mode == 1 ? blockIdx.x * P : 0;
  const uint32_t rank = mode == 2 ? cluster_rank() : 0;
  const uint16_t mask = (uint16_t)((1u << CL) - 1);
  unsigned long long t0 = gt();
  for (int s = 0; s < S; ++s)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(box_bytes));
  for (int s = 0; s < S; ++s) {
    uint8_t* dst = buf + s * stage_pitch;
    if (mode != 2) {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
              su32(dst)),
          "l"(&tm), "r"(su32(&bar[s])), "r"(s * 64), "r"(row0)
          : "memory");
    } else if ((s % CL) == (int)rank) {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(
              su32(dst)),
          "l"(&tm), "r"(su32(&bar[s])), "r"(s * 64), "r"(row0), "h"(mask)
          : "memory");
    }
  }
  for (int s = 0; s < S; ++s) {
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}"
                   : "=r"(done)
                   : "r"(su32(&bar[s]))
                   : "memory");
  }
  unsigned long long t1 = gt();
  out[blockIdx.x] = t1 - t0;
  if (mode == 2) cluster_sync();
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const int G = 144, P = 49;
  void* d;
  cudaMalloc(&d, (size_t)G * P * 1024 * 2 * 2);
  cudaMemset(d, 0, (size_t)G * P * 1024 * 2 * 2);
  unsigned long long* dout;
  cudaMalloc(&dout, G * sizeof(unsigned long long));
  std::vector<unsigned long long> h(G);
  for (int K : {384, 768, 1024}) {
    const int S = K / 64;
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)G * P};
    cuuint64_t strides[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)P}, es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, d, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", r); return 1; }
    const int smem = S * ((P * 128 + 1023) & ~1023) + 1024;
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(bench, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int mode = 0; mode < 3; ++mode) {
      for (int CL : {2, 4, 8, 16}) {
        if (mode != 2 && CL != 2) continue;
        if (mode == 2 && CL > S) continue;
        std::vector<double> meds;
        double worst = 0;
        for (int rep = 0; rep < 20; ++rep) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(G);
          cfg.blockDim = dim3(64);
          cfg.dynamicSmemBytes = smem;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = mode == 2 ? CL : 1;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          cfg.attrs = at;
          cfg.numAttrs = 1;
          cudaError_t e = cudaLaunchKernelEx(&cfg, bench, tm, S, P, mode, mode == 2 ? CL : 1, dout);
          if (e != cudaSuccess) { printf("launch failed: %s\n", cudaGetErrorString(e)); break; }
          cudaDeviceSynchronize();
          cudaMemcpy(h.data(), dout, G * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
          if (rep < 2) continue;   // first runs warm L2 and the tensor map
          std::vector<unsigned long long> s = h;
          std::sort(s.begin(), s.end());
          meds.push_back(s[G / 2] / 1e3);
          worst = std::max(worst, s[G - 1] / 1e3);
        }
        std::sort(meds.begin(), meds.end());
        printf("K=%4d S=%2d mode=%d CL=%2d  median CTA %.2f us  worst %.2f us\n", K, S, mode, mode == 2 ? CL : 1,
               meds.empty() ? -1.0 : meds[meds.size() / 2], worst);
      }
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("done: %s\n", cudaGetErrorString(e));
  return 0;
}
