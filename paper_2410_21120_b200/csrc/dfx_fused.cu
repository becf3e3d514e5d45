// dfx_fused.cu — multi-node fused kernels built on thread-block clusters.
//
// se_kernel: the squeeze-excitation gate of MobileNetV3 / EfficientNetV2
// (in the reference IR: global_avg_pool -> dense -> act -> dense -> act, the
// kinds of /root/reference/pkg/src/dagfuse/executor.py:56-65, 126-133 plus the
// extension activations) as ONE launch instead of 3-5 dependent nodes.
//
// One CL-CTA cluster per image (CL = 8, or 16 when the weight slices would not
// fit in shared memory).  CTA r owns the channel slice [c_lo, c_hi):
//   0. before griddepcontrol.wait (weights are static) one thread bulk-copies
//      the slice's rows of fc1^T [C][Cr] and fc2 [C][Cr] -- both contiguous --
//      into shared memory (cp.async.bulk + mbarrier);
//   1. pools its channels: every thread's 16-B loads for all of its pixels are
//      issued before any is summed, then a fixed-order smem reduction;
//   2. computes fc1 PARTIAL sums over its own channels for every hidden unit
//      (no gather of the pooled vector), publishes them in smem;
//   3. cluster.sync; reads the CL partial vectors over DSMEM and sums them in
//      rank order (the same order in every CTA -> identical hidden vectors),
//      + bias, act1;
//   4. computes the gate for its channels (8 lanes per channel, 16-B weight
//      reads, shuffle reduction), + bias, act2, 16-bit store;
//   5. optionally (apply = 1) the following channel_scale: each CTA multiplies its
//      channel slice of x by the gate -- no separate elementwise launch;
//   6. cluster.sync so no CTA's smem disappears while a peer still reads it.
// Deterministic: fixed summation orders, no atomics.  Timeline probes
// (-DDFX_TIMELINE): dfx_debug_timeline_se.
#include <cooperative_groups.h>

#ifdef DFX_TIMELINE
__device__ unsigned long long dfx_timeline_se[64];
#define DFX_TL(i)                                                \
  do {                                                           \
    if (blockIdx.x == 0 && blockIdx.y == 0) {                    \
      unsigned long long _t;                                     \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));     \
      dfx_timeline_se[i] = _t;                                   \
    }                                                            \
  } while (0)
#endif

#include "dfx_common.cuh"

extern "C" int dfx_debug_timeline_se(unsigned long long* out, int n) {
#ifdef DFX_TIMELINE
  return cudaMemcpyFromSymbol(out, dfx_timeline_se, sizeof(unsigned long long) * (n < 64 ? n : 64)) ==
                 cudaSuccess
             ? 0
             : -1;
#else
  (void)out;
  (void)n;
  return -4;
#endif
}

namespace cg = cooperative_groups;

namespace dfx {

constexpr int kSeMaxSlice = 512;   // channels per CTA (C <= 4096 -> <= 512 at CL = 8)
__device__ __forceinline__ int out_coff_of(const dfx_se_params& P) { return P.out.coff; }

// IPI images per cluster (large batches): every weight element a CTA reads serves
// IPI images (the FC slices were re-read from L2 once per image: 2.4 MB per image
// for EfficientNetV2-L's last stage), one cluster.sync covers all of them.
template <typename T, int CL, int IPI>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(kSeThreads)
    se_kernel(const __grid_constant__ dfx_se_params P) {
  __shared__ float pooled[IPI][kSeMaxSlice];     // this CTA's channels only (later: gates)
  __shared__ float partial[IPI][kSeMaxCr];       // fc1 partial sums over this CTA's channels
  __shared__ float hidden[IPI][kSeMaxCr];        // full hidden vectors (rank-order reduction)
  __shared__ float red[kSeThreads * 8 + 8];  // pooling reduction scratch
  __shared__ __align__(8) uint64_t wbar;
  extern __shared__ __align__(16) uint8_t wsm[];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = int(cluster.block_rank());
  const int n0 = blockIdx.y * IPI;
  const dfx_view& in = P.in;
  const int nimg = min(IPI, in.n - n0);
  const int C = in.c, Cr = P.cr;
  const int hw = in.h * in.w;
  const int cs = se_chan_slice(C, CL);
  const int c_lo = min(C, rank * cs), c_hi = min(C, c_lo + cs);
  const int nch = c_hi - c_lo;
  const T* w1g = reinterpret_cast<const T*>(P.w1);    // fc1^T  [C][Cr]
  const T* w2g = reinterpret_cast<const T*>(P.w2);    // fc2    [C][Cr]
  // 16-B aligned slices are staged in smem unless apply bit 1 says otherwise (large
  // batches: clusters of smem-heavy CTAs then cannot be co-scheduled, while the
  // weights are L2-resident and shared by every image's cluster anyway)
  const bool aligned = (C & 7) == 0 && (Cr & 7) == 0;
  const bool staged = aligned && !(P.apply & 2);
  // apply bit 2 (split precision, slices beyond the smem budget): stage the fc1
  // slices only, fc2 rows read from L2 (fc1's per-k loads were the phase's cost)
  const bool staged1 = staged || (aligned && (P.apply & 4));
  const bool apply = P.apply & 1;
  const int sb = ((cs * Cr * 2) + 15) & ~15;
  // split precision: FC weights [hi C x Cr][lo C x Cr]; staged, the lo slices follow
  // the two hi slices in smem (w1_lo at +2 sb bytes, w2_lo at +3 sb); fc1 only:
  // [w1 hi][w1 lo]
  const int64_t wlo = !kSplitT<T> ? 0 : staged ? int64_t(sb) : int64_t(C) * Cr;   // w2, elements
  const int64_t wlo1 = !kSplitT<T> ? 0 : staged ? int64_t(sb) : staged1 ? int64_t(sb / 2) : int64_t(C) * Cr;
  const T* w1 = staged1 ? reinterpret_cast<const T*>(wsm) : w1g + int64_t(c_lo) * Cr;
  const T* w2 = staged ? reinterpret_cast<const T*>(wsm + sb) : w2g + int64_t(c_lo) * Cr;

  // ---- 0. weight slices -> smem, before the dependency resolves
  if (threadIdx.x == 0) {
    DFX_TL(0);
    mbar_init(&wbar, 1);
    fence_barrier_init();
    const uint32_t bytes = uint32_t(nch) * Cr * 2;
    if (staged && bytes) {
      mbar_arrive_expect_tx(&wbar, (kSplitT<T> ? 4 : 2) * bytes);
      bulk_load(wsm, w1g + int64_t(c_lo) * Cr, bytes, &wbar);
      bulk_load(wsm + sb, w2g + int64_t(c_lo) * Cr, bytes, &wbar);
      if constexpr (kSplitT<T>) {
        bulk_load(wsm + 2 * sb, w1g + int64_t(C) * Cr + int64_t(c_lo) * Cr, bytes, &wbar);
        bulk_load(wsm + 3 * sb, w2g + int64_t(C) * Cr + int64_t(c_lo) * Cr, bytes, &wbar);
      }
    } else if (staged1 && bytes) {
      mbar_arrive_expect_tx(&wbar, (kSplitT<T> ? 2 : 1) * bytes);
      bulk_load(wsm, w1g + int64_t(c_lo) * Cr, bytes, &wbar);
      if constexpr (kSplitT<T>)
        bulk_load(wsm + sb, w1g + int64_t(C) * Cr + int64_t(c_lo) * Cr, bytes, &wbar);
    }
  }
  griddep_wait();
  griddep_launch();
  if (threadIdx.x == 0) DFX_TL(1);

  // fused scale (apply): when the host sized dynamic smem for it, the CTA's slice
  // of x is kept in smem while pooling, so the scale pass reads smem instead of
  // a second L2 round trip (dfx_api.cu DFX_OP_SE)
  uint32_t dsm;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dsm));
  const int wbytes = staged ? (kSplitT<T> ? 4 : 2) * sb : staged1 ? (kSplitT<T> ? 2 : 1) * sb : 0;
  T* xt = reinterpret_cast<T*>(wsm + wbytes);
  constexpr int kPl = kSplitT<T> ? 2 : 1;            // split: the lo tile follows the hi one
  const bool cache_x = apply && IPI == 1 && ((in.coff | out_coff_of(P) | c_lo | nch) & 7) == 0 &&
                       uint32_t(wbytes + hw * nch * 2 * kPl) <= dsm;
  T* const xtl = xt + hw * nch;                        // lo plane tile (split precision)
  const int64_t xlo = lo_of<T>(in);

  // ---- 1. pool: thread = (channel group g, pixel stripe y); all loads in flight first
  const int G = (nch + 7) / 8;                        // channel groups of this CTA
  const int stripes = G ? kSeThreads / G : 1;
  const int g = threadIdx.x % max(G, 1), y = threadIdx.x / max(G, 1);
  if (P.pooled != nullptr) {
    // the channel means come from the depthwise-epilogue GEMM before (dfx_se_fuse mode 1):
    // no pooling pass; the scale's x tile loads asynchronously behind the FC phases
    if (cache_x && G && y < stripes) {
      const T* ib = reinterpret_cast<const T*>(in.base) + view_pixel_index(in, int64_t(n0) * hw, c_lo + g * 8);
      for (int s = y; s < hw; s += stripes) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(xt + s * nch + g * 8)),
                     "l"(ib + int64_t(s) * in.pitch)
                     : "memory");
        if constexpr (kPl == 2)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(xtl + s * nch + g * 8)),
                       "l"(ib + int64_t(s) * in.pitch + xlo)
                       : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int im = 0; im < nimg; ++im)
      for (int k = threadIdx.x; k < nch; k += kSeThreads)
        pooled[im][k] = __ldcg(P.pooled + int64_t(n0 + im) * C + c_lo + k);
    __syncthreads();
  }
  for (int im = 0; P.pooled == nullptr && im < nimg; ++im) {
  const int n = n0 + im;
  float acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.f;
  if (G && y < stripes) {
    const int c = c_lo + g * 8;
    const int nl = min(8, c_hi - c);
    const int64_t base = view_pixel_index(in, int64_t(n) * hw, c);
    if (cache_x && nl == 8) {
      // every 16-B chunk of this thread's pixels as one async copy into the x tile:
      // all in flight at once (one L2 round trip instead of one per 4 loads), then
      // pooled from smem; the scale pass reuses the tile
      const T* ib = reinterpret_cast<const T*>(in.base) + base;
      for (int s = y; s < hw; s += stripes) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(xt + s * nch + g * 8)),
                     "l"(ib + int64_t(s) * in.pitch)
                     : "memory");
        if constexpr (kPl == 2)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(xtl + s * nch + g * 8)),
                       "l"(ib + int64_t(s) * in.pitch + xlo)
                       : "memory");
      }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
      for (int s = y; s < hw; s += stripes) {
        float x[8];
        unpack8<T>(*reinterpret_cast<const uint4*>(xt + s * nch + g * 8), x);
        if constexpr (kPl == 2) {
          float l[8];
          unpack8<T>(*reinterpret_cast<const uint4*>(xtl + s * nch + g * 8), l);
#pragma unroll
          for (int i = 0; i < 8; ++i) x[i] += l[i];
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += x[i];
      }
    } else if (kSplitT<T> && nl == 8 && ((in.coff + c) & 7) == 0) {
      for (int s = y; s < hw; s += stripes) {
        float x[8];
        ldv8<T>(in, base + int64_t(s) * in.pitch, x);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += x[i];
      }
    } else if (nl == 8 && ((in.coff + c) & 7) == 0) {
      const T* ib = reinterpret_cast<const T*>(in.base) + base;
      int s = y;
      for (; s + 3 * stripes < hw; s += 4 * stripes) {      // 4 independent 16-B loads
        uint4 r[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) r[u] = *reinterpret_cast<const uint4*>(ib + int64_t(s + u * stripes) * in.pitch);
        float x0[8], x1[8], x2[8], x3[8];
        unpack8<T>(r[0], x0);
        unpack8<T>(r[1], x1);
        unpack8<T>(r[2], x2);
        unpack8<T>(r[3], x3);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += (x0[i] + x1[i]) + (x2[i] + x3[i]);
        if (cache_x) {
#pragma unroll
          for (int u = 0; u < 4; ++u) *reinterpret_cast<uint4*>(xt + (s + u * stripes) * nch + g * 8) = r[u];
        }
      }
      for (; s < hw; s += stripes) {
        const uint4 r = *reinterpret_cast<const uint4*>(ib + int64_t(s) * in.pitch);
        float x[8];
        unpack8<T>(r, x);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += x[i];
        if (cache_x) *reinterpret_cast<uint4*>(xt + s * nch + g * 8) = r;
      }
    } else {
      for (int s = y; s < hw; s += stripes)
        for (int i = 0; i < nl; ++i) acc[i] += ldv1<T>(in, base + int64_t(s) * in.pitch + i);
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) red[threadIdx.x * 8 + i] = acc[i];
  __syncthreads();
  for (int k = threadIdx.x; k < nch; k += kSeThreads) {      // fixed stripe order
    const int gg = k / 8, ii = k % 8;
    float s = 0.f;
    for (int yy = 0; yy < stripes; ++yy) s += red[(yy * G + gg) * 8 + ii];
    pooled[im][k] = s * (1.0f / float(hw));
  }
  __syncthreads();                                    // red[] reused by the next image
  }
  if (threadIdx.x == 0) DFX_TL(2);
  if (threadIdx.x == 0 && staged1 && nch * Cr > 0) mbar_wait(&wbar, 0);  // weight slices landed (one poller)
  __syncthreads();
  if (threadIdx.x == 0) DFX_TL(3);

  // ---- 2. fc1 partial sums over this CTA's channels: thread (unit j, k-quarter q);
  // consecutive threads read consecutive units of one row (conflict-free), the
  // KQ k-partitions are combined in fixed order through smem
  {
    const int KQ = Cr >= kSeThreads ? 1 : kSeThreads / Cr;
    const int kq_len = (nch + KQ - 1) / KQ;
    for (int t = threadIdx.x; t < Cr * KQ; t += kSeThreads) {
      const int j = t % Cr, q = t / Cr;
      const int k0 = q * kq_len, k1 = min(nch, k0 + kq_len);
      float sa[IPI];
#pragma unroll
      for (int i = 0; i < IPI; ++i) sa[i] = 0.f;
      for (int k = k0; k < k1; ++k) {
        float wv = Elt<T>::to_f(w1[int64_t(k) * Cr + j]);           // one load, IPI images
        if constexpr (kSplitT<T>) wv += Elt<T>::to_f(w1[int64_t(k) * Cr + j + wlo1]);
#pragma unroll
        for (int i = 0; i < IPI; ++i) sa[i] = fmaf(wv, pooled[i][k], sa[i]);
      }
#pragma unroll
      for (int i = 0; i < IPI; ++i) red[t * IPI + i] = sa[i];
    }
    __syncthreads();
    for (int j = threadIdx.x; j < Cr; j += kSeThreads) {
#pragma unroll
      for (int i = 0; i < IPI; ++i) {
        float s = 0.f;
        for (int q = 0; q < KQ; ++q) s += red[(q * Cr + j) * IPI + i];
        partial[i][j] = s;
      }
    }
  }
  if (threadIdx.x == 0) DFX_TL(4);
  cluster.sync();
  if (threadIdx.x == 0) DFX_TL(5);

  // ---- 3. hidden = act1(b1 + sum over ranks of the partials), rank order
  for (int t = threadIdx.x; t < Cr * IPI; t += kSeThreads) {
    const int i = t / Cr, j = t - i * Cr;
    float v[CL];
#pragma unroll
    for (int r = 0; r < CL; ++r) v[r] = cluster.map_shared_rank(&partial[i][0], r)[j];
    float s = 0.f;
#pragma unroll
    for (int r = 0; r < CL; ++r) s += v[r];
    float a[8] = {s + (P.b1 ? P.b1[j] : 0.f), 0, 0, 0, 0, 0, 0, 0};
    act8<kSplitT<T>>(P.act1, a);
    hidden[i][j] = a[0];
  }
  // every DSMEM read of the peers' partial[] is done: arrive now, wait at exit (the
  // exit barrier then finds the cluster long arrived instead of costing ~0.8 us)
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) DFX_TL(6);

  // ---- 4. gate for this CTA's channels: thread per channel, hidden vector
  // broadcast from smem, weight rows read as 16-B vectors
  const dfx_view& out = P.out;
  for (int k = threadIdx.x; k < nch; k += kSeThreads) {
    const T* row = w2 + int64_t(k) * Cr;
    float sa[IPI], sb[IPI];
#pragma unroll
    for (int i = 0; i < IPI; ++i) sa[i] = sb[i] = 0.f;
    if ((Cr & 7) == 0) {
      for (int j = 0; j < Cr; j += 8) {
        float wv[8];
        ld8<T>(row, j, wlo, wv);                             // one load, IPI images
#pragma unroll
        for (int i = 0; i < IPI; ++i) {
          const float* h = hidden[i] + j;
          sa[i] = fmaf(wv[0], h[0], sa[i]); sb[i] = fmaf(wv[1], h[1], sb[i]);
          sa[i] = fmaf(wv[2], h[2], sa[i]); sb[i] = fmaf(wv[3], h[3], sb[i]);
          sa[i] = fmaf(wv[4], h[4], sa[i]); sb[i] = fmaf(wv[5], h[5], sb[i]);
          sa[i] = fmaf(wv[6], h[6], sa[i]); sb[i] = fmaf(wv[7], h[7], sb[i]);
        }
      }
    } else {
      for (int j = 0; j < Cr; ++j) {
        float wv = Elt<T>::to_f(row[j]);
        if constexpr (kSplitT<T>) wv += Elt<T>::to_f(row[j + wlo]);
#pragma unroll
        for (int i = 0; i < IPI; ++i) sa[i] = fmaf(wv, hidden[i][j], sa[i]);
      }
    }
    const int c = c_lo + k;
#pragma unroll
    for (int i = 0; i < IPI; ++i) {
      if (i >= nimg) break;
      float a[8] = {sa[i] + sb[i] + (P.b2 ? P.b2[c] : 0.f), 0, 0, 0, 0, 0, 0, 0};
      act8<kSplitT<T>>(P.act2, a);
      if (apply)
        pooled[i][k] = a[0];                                 // gate of this CTA's channel k
      else
        stv1<T>(out, int64_t(n0 + i) * out.pitch + out.coff + c, a[0]);
    }
  }
  if (apply) __syncthreads();
  for (int im = 0; apply && im < nimg; ++im) {
    // ---- 5. fused channel_scale: out[n, :, :, slice] = x * gate (x re-read from L2)
    const float* gate = pooled[im];
    const int64_t pb = int64_t(n0 + im) * hw;
    if (cache_x) {
      if (P.pooled != nullptr) {                       // the x tile loaded behind the FCs
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
      }
      const int G8 = nch / 8, total = hw * G8;
      for (int i = threadIdx.x; i < total; i += kSeThreads) {
        const int s = i / G8, g8 = (i - s * G8) * 8;
        float x[8];
        unpack8<T>(*reinterpret_cast<const uint4*>(xt + s * nch + g8), x);
        if constexpr (kPl == 2) {
          float l[8];
          unpack8<T>(*reinterpret_cast<const uint4*>(xtl + s * nch + g8), l);
#pragma unroll
          for (int j = 0; j < 8; ++j) x[j] += l[j];
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] *= gate[g8 + j];
        stv8<T>(out, view_pixel_index(out, pb + s, c_lo + g8), x);
      }
    } else if (kSplitT<T> && ((in.coff | out.coff | c_lo | nch) & 7) == 0) {
      const int G8 = nch / 8, total = hw * G8;
      for (int i = threadIdx.x; i < total; i += kSeThreads) {
        const int s = i / G8, g8 = (i - s * G8) * 8;
        float x[8];
        ldv8<T>(in, view_pixel_index(in, pb + s, c_lo + g8), x);
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] *= gate[g8 + j];
        stv8<T>(out, view_pixel_index(out, pb + s, c_lo + g8), x);
      }
    } else if (((in.coff | out.coff | c_lo | nch) & 7) == 0) {
      // 4 independent 16-B loads in flight per thread before any store (the
      // per-iteration load -> store chain otherwise serialises on L2 latency)
      const int G8 = nch / 8, total = hw * G8;
      for (int i0 = threadIdx.x; i0 < total; i0 += 4 * kSeThreads) {
        uint4 raw[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u * kSeThreads;
          if (i < total) {
            const int s = i / G8, g8 = (i - s * G8) * 8;
            raw[u] = __ldcg(reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(in.base) +
                                                           view_pixel_index(in, pb + s, c_lo + g8)));
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u * kSeThreads;
          if (i < total) {
            const int s = i / G8, g8 = (i - s * G8) * 8;
            float x[8];
            unpack8<T>(raw[u], x);
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] *= gate[g8 + j];
            stv8<T>(out, view_pixel_index(out, pb + s, c_lo + g8), x);
          }
        }
      }
    } else {
      for (int i = threadIdx.x; i < hw * nch; i += kSeThreads) {
        const int s = i / nch, k = i - s * nch;
        stv1<T>(out, view_pixel_index(out, pb + s, c_lo + k),
               ldv1<T>(in, view_pixel_index(in, pb + s, c_lo + k)) * gate[k]);
      }
    }
  }
  if (threadIdx.x == 0) DFX_TL(7);
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");   // peers done with our smem
  if (threadIdx.x == 0) DFX_TL(8);
}

// ---------------------------------------------------------------- dwse_kernel
// An MBConv block's middle -- depthwise conv (+ folded BN + act) -> squeeze-
// excitation gate -> channel scale -- as ONE launch (the three were dwconv,
// se and ew launches, ~14 us of dependent chain per block at batch 1).  One
// 16-CTA cluster per image; CTA r owns channel slice [c_lo, c_hi):
//   0. FC weight slices bulk-copied to smem before griddepcontrol.wait (small
//      batch, P.staged), as in se_kernel;
//   1. depthwise conv of its slice over all output pixels, epilogue, rounded to
//      the 16-bit storage type into an smem tile [HWo][slice] -- the tensor the
//      unfused path would have stored;
//   2. pools the tile per channel (fixed order), fc1 partial sums over its
//      channels, cluster.sync, rank-order DSMEM reduction, act1 (se_kernel 2-3);
//   3. its channels' gate (+b2, act2), rounded like a stored gate;
//   4. out = tile * gate, 16-B stores; cluster.sync so peers' smem stays alive.
constexpr int kDwseCL = 16;

template <typename T>
__global__ void __cluster_dims__(kDwseCL, 1, 1) __launch_bounds__(kSeThreads)
    dwse_kernel(const __grid_constant__ dfx_dwse_params P) {
  constexpr int CL = kDwseCL;
  __shared__ float pooled[kSeMaxSlice];
  __shared__ float partial[kSeMaxCr];
  __shared__ float hidden[kSeMaxCr];
  __shared__ float red[kSeThreads];
  __shared__ __align__(8) uint64_t wbar;
  extern __shared__ __align__(16) uint8_t wsm[];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = int(cluster.block_rank());
  const int n = blockIdx.y;
  const dfx_view& in = P.in;
  const dfx_view& out = P.out;
  const int C = in.c, Cr = P.cr;
  const int OW = out.w, HWo = out.h * out.w;
  const int cs = se_chan_slice(C, CL);
  const int c_lo = min(C, rank * cs), c_hi = min(C, c_lo + cs);
  const int nch = c_hi - c_lo;                       // multiple of 8 (C % 8 == 0)
  const int G = nch >> 3;
  const T* w1g = reinterpret_cast<const T*>(P.w1);
  const T* w2g = reinterpret_cast<const T*>(P.w2);
  const bool staged = P.staged && (Cr & 7) == 0;
  const int sb = ((cs * Cr * 2) + 15) & ~15;
  const T* w1 = staged ? reinterpret_cast<const T*>(wsm) : w1g + int64_t(c_lo) * Cr;
  const T* w2 = staged ? reinterpret_cast<const T*>(wsm + sb) : w2g + int64_t(c_lo) * Cr;
  T* tile = reinterpret_cast<T*>(wsm + (staged ? 2 * sb : 0));     // [HWo][nch]

  if (threadIdx.x == 0) {
    mbar_init(&wbar, 1);
    fence_barrier_init();
    const uint32_t bytes = uint32_t(nch) * Cr * 2;
    if (staged && bytes) {
      mbar_arrive_expect_tx(&wbar, 2 * bytes);
      bulk_load(wsm, w1g + int64_t(c_lo) * Cr, bytes, &wbar);
      bulk_load(wsm + sb, w2g + int64_t(c_lo) * Cr, bytes, &wbar);
    } else {
      mbar_arrive(&wbar);
    }
  }
  griddep_wait();
  griddep_launch();

  // ---- 1. depthwise conv of this slice -> smem tile (16-bit, as a stored tensor)
  const int kh = P.kh, kw = P.kw;
  for (int item = threadIdx.x; item < HWo * G; item += kSeThreads) {
    const int p = item / G, g = item - p * G;
    const int c = c_lo + g * 8;
    const int oh = p / OW, ow = p - oh * OW;
    const int h0 = oh * P.stride_h - P.pad_h, w0 = ow * P.stride_w - P.pad_w;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int ki = 0; ki < kh; ++ki) {
      const int h = h0 + ki;
      if (h < 0 || h >= in.h) continue;
      for (int kj = 0; kj < kw; ++kj) {
        const int w = w0 + kj;
        if (w < 0 || w >= in.w) continue;
        float x[8];
        ldv8<T>(in, view_index(in, n, h, w, c), x);
        const float4* wt = reinterpret_cast<const float4*>(P.dw_weight + (ki * kw + kj) * C + c);
        const float4 lo = __ldg(wt), hi = __ldg(wt + 1);
        acc[0] = fmaf(lo.x, x[0], acc[0]); acc[1] = fmaf(lo.y, x[1], acc[1]);
        acc[2] = fmaf(lo.z, x[2], acc[2]); acc[3] = fmaf(lo.w, x[3], acc[3]);
        acc[4] = fmaf(hi.x, x[4], acc[4]); acc[5] = fmaf(hi.y, x[5], acc[5]);
        acc[6] = fmaf(hi.z, x[6], acc[6]); acc[7] = fmaf(hi.w, x[7], acc[7]);
      }
    }
    epilogue8<T>(P.dw_epi, acc, 0, n, c);
    *reinterpret_cast<uint4*>(tile + p * nch + g * 8) = pack8<T>(acc);
  }
  __syncthreads();

  // ---- 2. pool the tile per channel (pixel order, two interleaved partial sums)
  for (int k = threadIdx.x; k < nch; k += kSeThreads) {
    float s0 = 0.f, s1 = 0.f;
    int p = 0;
    for (; p + 1 < HWo; p += 2) {
      s0 += Elt<T>::to_f(tile[p * nch + k]);
      s1 += Elt<T>::to_f(tile[(p + 1) * nch + k]);
    }
    if (p < HWo) s0 += Elt<T>::to_f(tile[p * nch + k]);
    pooled[k] = (s0 + s1) * (1.0f / float(HWo));
  }
  if (threadIdx.x == 0) mbar_wait(&wbar, 0);
  __syncthreads();
  // fc1 partial sums over this CTA's channels (one hidden unit per thread pass)
  for (int j = threadIdx.x; j < Cr; j += kSeThreads) {
    float s0 = 0.f, s1 = 0.f;
    int k = 0;
    for (; k + 1 < nch; k += 2) {
      s0 = fmaf(Elt<T>::to_f(w1[int64_t(k) * Cr + j]), pooled[k], s0);
      s1 = fmaf(Elt<T>::to_f(w1[int64_t(k + 1) * Cr + j]), pooled[k + 1], s1);
    }
    if (k < nch) s0 = fmaf(Elt<T>::to_f(w1[int64_t(k) * Cr + j]), pooled[k], s0);
    partial[j] = s0 + s1;
  }
  cluster.sync();
  for (int j = threadIdx.x; j < Cr; j += kSeThreads) {
    float s = 0.f;
#pragma unroll
    for (int r = 0; r < CL; ++r) s += cluster.map_shared_rank(partial, r)[j];
    float a[8] = {s + (P.b1 ? P.b1[j] : 0.f), 0, 0, 0, 0, 0, 0, 0};
    act8(P.act1, a);
    hidden[j] = a[0];
  }
  __syncthreads();
  // ---- 3. gate of this CTA's channels, rounded like a stored 16-bit gate
  for (int k = threadIdx.x; k < nch; k += kSeThreads) {
    const T* row = w2 + int64_t(k) * Cr;
    float s0 = 0.f, s1 = 0.f;
    if ((Cr & 7) == 0) {
      for (int j = 0; j < Cr; j += 8) {
        float wv[8];
        ld8<T>(row, j, 0, wv);
        s0 = fmaf(wv[0], hidden[j], s0); s1 = fmaf(wv[1], hidden[j + 1], s1);
        s0 = fmaf(wv[2], hidden[j + 2], s0); s1 = fmaf(wv[3], hidden[j + 3], s1);
        s0 = fmaf(wv[4], hidden[j + 4], s0); s1 = fmaf(wv[5], hidden[j + 5], s1);
        s0 = fmaf(wv[6], hidden[j + 6], s0); s1 = fmaf(wv[7], hidden[j + 7], s1);
      }
    } else {
      for (int j = 0; j < Cr; ++j) s0 = fmaf(Elt<T>::to_f(row[j]), hidden[j], s0);
    }
    float a[8] = {s0 + s1 + (P.b2 ? P.b2[c_lo + k] : 0.f), 0, 0, 0, 0, 0, 0, 0};
    act8(P.act2, a);
    red[k] = Elt<T>::to_f(Elt<T>::from_f(a[0]));
  }
  __syncthreads();
  // ---- 4. out = tile * gate
  for (int item = threadIdx.x; item < HWo * G; item += kSeThreads) {
    const int p = item / G, g = item - p * G;
    float x[8];
    unpack8<T>(*reinterpret_cast<const uint4*>(tile + p * nch + g * 8), x);
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] *= red[g * 8 + k];
    stv8<T>(out, view_pixel_index(out, int64_t(n) * HWo + p, c_lo + g * 8), x);
  }
  cluster.sync();        // peers finished reading this CTA's partial[]
}

template __global__ void dwse_kernel<__nv_bfloat16>(const __grid_constant__ dfx_dwse_params);
template __global__ void dwse_kernel<__half>(const __grid_constant__ dfx_dwse_params);

#define DFX_SE_INST(T, CL, IPI) \
  template __global__ void se_kernel<T, CL, IPI>(const __grid_constant__ dfx_se_params);
DFX_SE_INST(__nv_bfloat16, 8, 1)
DFX_SE_INST(__half, 8, 1)
DFX_SE_INST(__nv_bfloat16, 16, 1)
DFX_SE_INST(__half, 16, 1)
DFX_SE_INST(__nv_bfloat16, 16, 4)
DFX_SE_INST(__half, 16, 4)
DFX_SE_INST(f16x2, 16, 1)
DFX_SE_INST(bf16x2, 16, 1)
DFX_SE_INST(f16x2, 16, 4)
DFX_SE_INST(bf16x2, 16, 4)
#undef DFX_SE_INST

}  // namespace dfx
