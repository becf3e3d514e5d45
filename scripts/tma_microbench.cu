// TMA issue/throughput microbenchmark on one CTA (development tool, not shipped).
// Compares: 2-D tiled TMA boxes (64 x rows, 128-B swizzle) vs cp.async.bulk
// contiguous copies of the same bytes.  Reports issue time and completion time.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmab scripts/tma_microbench.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void bench(const __grid_constant__ CUtensorMap tm, const char* src, int n, int rows, int mode,
                      unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~uintptr_t(1023));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint32_t bytes = rows * 128;
  unsigned long long t0 = gt();
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&bar)), "r"(bytes * n));
  for (int i = 0; i < n; ++i) {
    uint8_t* dst = buf + (i % 8) * bytes;
    if (mode == 0) {
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                   :: "r"(su32(dst)), "l"(&tm), "r"(su32(&bar)), "r"(0), "r"(i * rows) : "memory");
    } else {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(su32(dst)), "l"(src + (size_t)i * bytes), "r"(bytes), "r"(su32(&bar)) : "memory");
    }
  }
  unsigned long long t1 = gt();
  uint32_t done = 0;
  while (!done) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(su32(&bar)) : "memory");
  }
  unsigned long long t2 = gt();
  out[0] = t1 - t0;
  out[1] = t2 - t0;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const size_t total = 64 << 20;
  char* d;
  cudaMalloc(&d, total);
  cudaMemset(d, 1, total);
  unsigned long long* out;
  cudaMalloc(&out, 16);
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int rows : {64, 128, 256}) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {64, total / 128};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, (cuuint32_t)rows};
    cuuint32_t es[2] = {1, 1};
    ((EncFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int mode = 0; mode < 2; ++mode) {
      for (int n : {1, 4, 16}) {
        unsigned long long h[2], best_i = ~0ull, best_c = ~0ull;
        for (int rep = 0; rep < 5; ++rep) {
          bench<<<1, 32, 8 * rows * 128 + 1024>>>(tm, d + ((size_t)rep << 22), n, rows, mode, out);
          cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
          if (rep > 0) { best_i = h[0] < best_i ? h[0] : best_i; best_c = h[1] < best_c ? h[1] : best_c; }
        }
        printf("%-6s rows=%3d n=%2d bytes=%7d  issue %6.2f us  complete %6.2f us  %6.1f GB/s\n",
               mode ? "bulk" : "tiled", rows, n, n * rows * 128, best_i / 1e3, best_c / 1e3,
               n * rows * 128.0 / best_c);
      }
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
