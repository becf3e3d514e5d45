// dfx_fused.cu — multi-node fused kernels built on thread-block clusters.
//
// se_kernel: the squeeze-excitation gate of MobileNetV3 / EfficientNetV2
// (in the reference IR: global_avg_pool -> dense -> act -> dense -> act, the
// kinds of /root/reference/pkg/src/dagfuse/executor.py:56-65, 126-133 plus the
// extension activations) as ONE launch instead of 3-5 dependent nodes.
//
// One 8-CTA cluster per image.  CTA r of the cluster
//   1. pools channel slice r of the image (fixed-order sums, fp32, x fp32(1/HW)),
//   2. after cluster.sync, gathers the whole pooled vector from the 8 CTAs'
//      shared memory over DSMEM and computes hidden units slice r of fc1
//      (+ bias, act1) -- one warp per unit, 16-B weight loads, fixed-order
//      warp reduction,
//   3. after cluster.sync, gathers the hidden vector over DSMEM and computes
//      gate channels slice r of fc2 (+ bias, act2), one thread per channel,
//   4. writes its gate slice (16-bit) and waits for the cluster so no CTA's
//      shared memory disappears while another still reads it.
// Everything is deterministic (fixed summation orders, no atomics).
#include <cooperative_groups.h>

#include "dfx_common.cuh"

namespace cg = cooperative_groups;

namespace dfx {

constexpr int kSeCluster = 8;
constexpr int kSeThreads = 256;
constexpr int kSeMaxC = 4096;      // pooled channels held per CTA
constexpr int kSeMaxCr = 512;      // hidden units held per CTA

template <typename T>
__global__ void __cluster_dims__(kSeCluster, 1, 1) __launch_bounds__(kSeThreads)
    se_kernel(const __grid_constant__ dfx_se_params P) {
  __shared__ float pooled[kSeMaxC];          // full pooled vector (gathered)
  __shared__ float hidden[kSeMaxCr];         // full hidden vector (gathered)
  __shared__ float part[32][64 + 4];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = int(cluster.block_rank());
  const int n = blockIdx.y;
  const dfx_view& in = P.in;
  const int C = in.c, Cr = P.cr;
  const int hw = in.h * in.w;
  // channel slice of this CTA (multiple of 8 wide), hidden-unit slice
  const int cs = ((C + kSeCluster * 8 - 1) / (kSeCluster * 8)) * 8;
  const int c_lo = min(C, rank * cs), c_hi = min(C, c_lo + cs);
  const int hs = (Cr + kSeCluster - 1) / kSeCluster;
  const int h_lo = min(Cr, rank * hs), h_hi = min(Cr, h_lo + hs);

  griddep_wait();
  griddep_launch();

  // ---- 1. pool channels [c_lo, c_hi): 64-channel chunks, 32 spatial rows
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;
  const bool vec_in = (in.coff & 7) == 0;
  for (int cc = c_lo; cc < c_hi; cc += 64) {
    const int c = cc + tx * 8;
    const int nl = max(0, min(8, c_hi - c));
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.f;
    if (nl > 0) {
      const int64_t base = view_pixel_index(in, int64_t(n) * hw, c);
      if (nl == 8 && vec_in) {
        for (int s = ty; s < hw; s += 32) {
          float x[8];
          ld8<T>(in.base, base + int64_t(s) * in.pitch, x);
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] += x[i];
        }
      } else {
        for (int s = ty; s < hw; s += 32)
          for (int i = 0; i < nl; ++i) acc[i] += ld1<T>(in.base, base + int64_t(s) * in.pitch + i);
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) part[ty][tx * 8 + i] = acc[i];
    __syncthreads();
    if (threadIdx.x < 64 && cc + threadIdx.x < c_hi) {
      float s = 0.f;
      for (int r = 0; r < 32; ++r) s += part[r][threadIdx.x];
      pooled[cc + threadIdx.x] = s * (1.0f / float(hw));
    }
    __syncthreads();
  }
  cluster.sync();

  // ---- 2. gather the pooled vector, fc1 slice
  for (int r = 0; r < kSeCluster; ++r) {
    if (r == rank) continue;
    const int lo = min(C, r * cs), hi = min(C, lo + cs);
    const float* remote = cluster.map_shared_rank(pooled, r);
    for (int c = lo + threadIdx.x; c < hi; c += kSeThreads) pooled[c] = remote[c];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const T* w1 = reinterpret_cast<const T*>(P.w1);
  const bool vec_w1 = (C & 7) == 0;
  for (int j = h_lo + warp; j < h_hi; j += kSeThreads / 32) {
    const T* row = w1 + int64_t(j) * C;
    float acc = 0.f;
    if (vec_w1) {
      for (int k = lane * 8; k < C; k += 256) {
        float wv[8];
        ld8<T>(row, k, wv);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc = fmaf(wv[i], pooled[k + i], acc);
      }
    } else {
      for (int k = lane; k < C; k += 32) acc = fmaf(Elt<T>::to_f(row[k]), pooled[k], acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      float v = acc + (P.b1 ? P.b1[j] : 0.f);
      float a[8] = {v, 0, 0, 0, 0, 0, 0, 0};
      act8(P.act1, a);
      hidden[j] = a[0];
    }
  }
  cluster.sync();

  // ---- 3. gather the hidden vector, fc2 slice -> gate
  for (int r = 0; r < kSeCluster; ++r) {
    if (r == rank) continue;
    const int lo = min(Cr, r * hs), hi = min(Cr, lo + hs);
    const float* remote = cluster.map_shared_rank(hidden, r);
    for (int j = lo + threadIdx.x; j < hi; j += kSeThreads) hidden[j] = remote[j];
  }
  __syncthreads();
  const T* w2 = reinterpret_cast<const T*>(P.w2);
  const dfx_view& out = P.out;
  const bool vec_w2 = (Cr & 7) == 0;
  for (int c = c_lo + threadIdx.x; c < c_hi; c += kSeThreads) {
    const T* row = w2 + int64_t(c) * Cr;
    float acc = 0.f;
    if (vec_w2) {
      for (int j = 0; j < Cr; j += 8) {
        float wv[8];
        ld8<T>(row, j, wv);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc = fmaf(wv[i], hidden[j + i], acc);
      }
    } else {
      for (int j = 0; j < Cr; ++j) acc = fmaf(Elt<T>::to_f(row[j]), hidden[j], acc);
    }
    float a[8] = {acc + (P.b2 ? P.b2[c] : 0.f), 0, 0, 0, 0, 0, 0, 0};
    act8(P.act2, a);
    st1<T>(out.base, int64_t(n) * out.pitch + out.coff + c, a[0]);
  }
  cluster.sync();        // keep this CTA's smem alive until every peer finished reading it
}

template __global__ void se_kernel<__nv_bfloat16>(const __grid_constant__ dfx_se_params);
template __global__ void se_kernel<__half>(const __grid_constant__ dfx_se_params);

}  // namespace dfx
