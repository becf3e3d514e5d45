// dfx_fused.cu — multi-node fused kernels built on thread-block clusters.
//
// se_kernel: the squeeze-excitation gate of MobileNetV3 / EfficientNetV2
// (in the reference IR: global_avg_pool -> dense -> act -> dense -> act, the
// kinds of /root/reference/pkg/src/dagfuse/executor.py:56-65, 126-133 plus the
// extension activations) as ONE launch instead of 3-5 dependent nodes.
//
// One CL-CTA cluster per image (CL = 8, or 16 when the weight slices would not
// fit in shared memory).  CTA r of the cluster
//   0. before griddepcontrol.wait (weights are static): one thread bulk-copies
//      its contiguous weight slices -- fc1 rows [h_lo, h_hi) and fc2 rows
//      [c_lo, c_hi) -- into shared memory (cp.async.bulk + mbarrier),
//   1. pools channel slice r of the image (fixed-order sums, fp32, x fp32(1/HW)),
//   2. after cluster.sync, gathers the whole pooled vector from the peers'
//      shared memory over DSMEM and computes hidden units [h_lo, h_hi) of fc1
//      (+ bias, act1): one warp per unit, fixed-order warp reduction,
//   3. after cluster.sync, gathers the hidden vector over DSMEM and computes
//      gate channels [c_lo, c_hi) of fc2 (+ bias, act2), one thread per channel,
//   4. writes its gate slice (16-bit) and waits for the cluster so no CTA's
//      shared memory disappears while a peer still reads it.
// Deterministic: fixed summation orders, no atomics.
#include <cooperative_groups.h>

#include "dfx_common.cuh"

namespace cg = cooperative_groups;

namespace dfx {


template <typename T, int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(kSeThreads)
    se_kernel(const __grid_constant__ dfx_se_params P) {
  __shared__ float pooled[kSeMaxC];          // full pooled vector (gathered)
  __shared__ float hidden[kSeMaxCr];         // full hidden vector (gathered)
  __shared__ float part[32][64 + 4];
  __shared__ __align__(8) uint64_t wbar;
  extern __shared__ __align__(16) uint8_t wsm[];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = int(cluster.block_rank());
  const int n = blockIdx.y;
  const dfx_view& in = P.in;
  const int C = in.c, Cr = P.cr;
  const int hw = in.h * in.w;
  const int cs = se_chan_slice(C, CL);
  const int c_lo = min(C, rank * cs), c_hi = min(C, c_lo + cs);
  const int hs = se_hid_slice(Cr, CL);
  const int h_lo = min(Cr, rank * hs), h_hi = min(Cr, h_lo + hs);
  const T* w1g = reinterpret_cast<const T*>(P.w1);
  const T* w2g = reinterpret_cast<const T*>(P.w2);
  // staged copies (weights rows are contiguous; C, Cr multiples of 8 keep every
  // slice 16-B aligned, otherwise the kernel reads global memory directly)
  const bool staged = (C & 7) == 0 && (Cr & 7) == 0;
  const int b1 = ((hs * C * 2) + 15) & ~15;
  const T* w1s = reinterpret_cast<const T*>(wsm);                 // rows [h_lo, h_hi)
  const T* w2s = reinterpret_cast<const T*>(wsm + b1);            // rows [c_lo, c_hi)

  // ---- 0. weight slices -> smem, issued before the dependency resolves
  if (threadIdx.x == 0) {
    mbar_init(&wbar, 1);
    fence_barrier_init();
    if (staged) {
      const uint32_t n1 = uint32_t(h_hi - h_lo) * C * 2, n2 = uint32_t(c_hi - c_lo) * Cr * 2;
      mbar_arrive_expect_tx(&wbar, n1 + n2);
      if (n1) bulk_load(wsm, w1g + int64_t(h_lo) * C, n1, &wbar);
      if (n2) bulk_load(wsm + b1, w2g + int64_t(c_lo) * Cr, n2, &wbar);
    } else {
      mbar_arrive(&wbar);
    }
  }
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
        int s = ty;
        for (; s + 32 < hw; s += 64) {
          float x0[8], x1[8];
          ld8<T>(in.base, base + int64_t(s) * in.pitch, x0);
          ld8<T>(in.base, base + int64_t(s + 32) * in.pitch, x1);
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] += x0[i] + x1[i];
        }
        for (; s < hw; s += 32) {
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
  for (int r = 0; r < CL; ++r) {
    if (r == rank) continue;
    const int lo = min(C, r * cs), hi = min(C, lo + cs);
    const float* remote = cluster.map_shared_rank(pooled, r);
    for (int c = lo + threadIdx.x; c < hi; c += kSeThreads) pooled[c] = remote[c];
  }
  mbar_wait(&wbar, 0);                       // weight slices landed
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = h_lo + warp; j < h_hi; j += kSeThreads / 32) {
    float acc = 0.f;
    if (staged) {
      const T* row = w1s + int64_t(j - h_lo) * C;
      for (int k = lane * 8; k < C; k += 256) {
        float wv[8];
        ld8<T>(row, k, wv);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc = fmaf(wv[i], pooled[k + i], acc);
      }
    } else {
      const T* row = w1g + int64_t(j) * C;
      for (int k = lane; k < C; k += 32) acc = fmaf(Elt<T>::to_f(row[k]), pooled[k], acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      float a[8] = {acc + (P.b1 ? P.b1[j] : 0.f), 0, 0, 0, 0, 0, 0, 0};
      act8(P.act1, a);
      hidden[j] = a[0];
    }
  }
  cluster.sync();

  // ---- 3. gather the hidden vector, fc2 slice -> gate
  for (int r = 0; r < CL; ++r) {
    if (r == rank) continue;
    const int lo = min(Cr, r * hs), hi = min(Cr, lo + hs);
    const float* remote = cluster.map_shared_rank(hidden, r);
    for (int j = lo + threadIdx.x; j < hi; j += kSeThreads) hidden[j] = remote[j];
  }
  __syncthreads();
  const dfx_view& out = P.out;
  for (int c = c_lo + threadIdx.x; c < c_hi; c += kSeThreads) {
    float acc = 0.f;
    if (staged) {
      const T* row = w2s + int64_t(c - c_lo) * Cr;
      for (int j = 0; j < Cr; j += 8) {
        float wv[8];
        ld8<T>(row, j, wv);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc = fmaf(wv[i], hidden[j + i], acc);
      }
    } else {
      const T* row = w2g + int64_t(c) * Cr;
      for (int j = 0; j < Cr; ++j) acc = fmaf(Elt<T>::to_f(row[j]), hidden[j], acc);
    }
    float a[8] = {acc + (P.b2 ? P.b2[c] : 0.f), 0, 0, 0, 0, 0, 0, 0};
    act8(P.act2, a);
    st1<T>(out.base, int64_t(n) * out.pitch + out.coff + c, a[0]);
  }
  cluster.sync();        // keep this CTA's smem alive until every peer finished reading it
}

#define DFX_SE_INST(T, CL) template __global__ void se_kernel<T, CL>(const __grid_constant__ dfx_se_params);
DFX_SE_INST(__nv_bfloat16, 8)
DFX_SE_INST(__half, 8)
DFX_SE_INST(__nv_bfloat16, 16)
DFX_SE_INST(__half, 16)
#undef DFX_SE_INST

}  // namespace dfx
