// tcgen05.mma issue / execution cost for one CTA (development tool, not shipped).
// One thread issues R back-to-back kind::f16 SS MMAs (M = 128, K = 16, N in {64,128,256})
// from 128B-swizzled K-major smem tiles; clock64 before the loop, after the last issue,
// and after the commit barrier fires.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -o /tmp/mmam scripts/mma_micro.cu
#include <cstdio>
#include "../paper_2410_21120_b200/csrc/dfx_common.cuh"

using namespace dfx;

__global__ void __launch_bounds__(128) mma_bench(int n, int reps, int fence_each, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* a = smem;                 // 128 x 64 halves, SW128
  uint8_t* b = smem + 16384;         // 256 x 64 halves
  for (int i = threadIdx.x; i < (16384 + 32768) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x / 32 == 2) tmem_alloc(&tbase, 256);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (fence_each == 2 && threadIdx.x / 32 == 1) {       // whole warp runs the loop, elect one
    const uint32_t idesc = umma_idesc_f16(uint32_t(n), DFX_F16);
    const uint32_t ab = smem_u32(a), bb = smem_u32(b);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const int kk = r & 3;
      const uint64_t ad = umma_smem_desc(ab + kk * 32, 128);
      const uint64_t bd = umma_smem_desc(bb + kk * 32, 128);
      uint32_t e;
      asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}" : "=r"(e));
      if (e) umma_f16(tbase, ad, bd, idesc, r > 0);
      __syncwarp();
    }
    const long long t1 = clock64();
    if (threadIdx.x == 32) {
      umma_commit(&bar);
      mbar_wait(&bar, 0);
      const long long t2 = clock64();
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  } else if (threadIdx.x == 32) {
    const uint32_t idesc = umma_idesc_f16(uint32_t(n), DFX_F16);
    const uint32_t ab = smem_u32(a), bb = smem_u32(b);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const int kk = r & 3;
      const uint64_t ad = umma_smem_desc(ab + kk * 32, 128);
      const uint64_t bd = umma_smem_desc(bb + kk * 32, 128);
      umma_f16(tbase, ad, bd, idesc, r > 0);
      if (fence_each && (r & 3) == 3) umma_commit(&bar);
    }
    const long long t1 = clock64();
    umma_commit(&bar);
    // the barrier completes one phase per commit; wait for the last one
    const int phases = fence_each ? reps / 4 + 1 : 1;
    mbar_wait(&bar, uint32_t((phases - 1) & 1));
    const long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x / 32 == 2) tmem_dealloc(tbase, 256);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  const int smem = 16384 + 32768 + 1024;
  cudaFuncSetAttribute(mma_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int fe = 0; fe < 3; ++fe)
    for (int n : {64, 128, 256})
      for (int reps : {4, 16, 64}) {
        unsigned long long h[2] = {0, 0};
        for (int it = 0; it < 3; ++it) {
          mma_bench<<<1, 128, smem>>>(n, reps, fe, d);
          cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        }
        printf("N=%3d reps=%3d commit_every4=%d: issue %6llu cyc (%5.1f/mma), done %6llu cyc (%5.1f/mma)\n",
               n, reps, fe, h[0], double(h[0]) / reps, h[1], double(h[1]) / reps);
      }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
