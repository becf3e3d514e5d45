// TMA 2-D vs 4-D activation boxes of the same bytes (development tool, not shipped):
// a 1x1-conv A tile of `rows` pixels x 64 channels read either as a 4-D box
// (c, w, h, n) = (64, W, rows/W, 1) with element strides 1 -- what gemm_kernel
// issues -- or as a 2-D box (64, rows) over [pixels][C].  One CTA, n boxes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma24 scripts/tma_2d4d.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void bench(const __grid_constant__ CUtensorMap t2, const __grid_constant__ CUtensorMap t4, int n,
                      int rows, int W, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~uintptr_t(1023));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  asm volatile("prefetch.tensormap [%0];" :: "l"(mode ? (const void*)&t4 : (const void*)&t2) : "memory");
  const uint32_t bytes = rows * 128;
  unsigned long long t0 = gt();
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&bar)), "r"(bytes * n));
  for (int i = 0; i < n; ++i) {
    uint8_t* dst = buf + (i % 8) * 16384;
    if (mode == 0) {
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                   :: "r"(su32(dst)), "l"(&t2), "r"(su32(&bar)), "r"(0), "r"(i * rows) : "memory");
    } else {
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                   :: "r"(su32(dst)), "l"(&t4), "r"(su32(&bar)), "r"(0), "r"(0), "r"(0), "r"(i) : "memory");
    }
  }
  unsigned long long t1 = gt();
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(su32(&bar)) : "memory");
  out[0] = t1 - t0;
  out[1] = gt() - t0;
}

int main() {
  const size_t total = 64 << 20;
  char* d;
  cudaMalloc(&d, total);
  cudaMemset(d, 1, total);
  unsigned long long* out;
  cudaMalloc(&out, 16);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int W : {7, 14, 56}) {
    const int H = W == 56 ? 2 : W, rows = W * H;          // 49, 196 (->2 boxes of 98?) , 112
    if (rows > 256) continue;
    const uint64_t images = total / (uint64_t(rows) * 128);
    CUtensorMap t2, t4;
    cuuint64_t d2[2] = {64, images * rows}, s2[1] = {128};
    cuuint32_t b2[2] = {64, (cuuint32_t)rows}, e2[2] = {1, 1};
    cuTensorMapEncodeTiled(&t2, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, d, d2, s2, b2, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint64_t d4[4] = {64, (cuuint64_t)W, (cuuint64_t)H, images}, s4[3] = {128, 128ull * W, 128ull * W * H};
    cuuint32_t b4[4] = {64, (cuuint32_t)W, (cuuint32_t)H, 1}, e4[4] = {1, 1, 1, 1};
    cuTensorMapEncodeTiled(&t4, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, d, d4, s4, b4, e4, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int mode = 0; mode < 2; ++mode)
      for (int n : {1, 4, 8}) {
        unsigned long long h[2], bi = ~0ull, bc = ~0ull;
        for (int rep = 0; rep < 6; ++rep) {
          bench<<<1, 32, 8 * 16384 + 1024>>>(t2, t4, n, rows, W, mode, out);
          cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
          if (rep > 0) { bi = h[0] < bi ? h[0] : bi; bc = h[1] < bc ? h[1] : bc; }
        }
        printf("%s W=%2d rows=%3d n=%d  issue %6.2f us  complete %6.2f us\n", mode ? "4d" : "2d", W, rows, n, bi / 1e3, bc / 1e3);
      }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
