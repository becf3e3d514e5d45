// dfx_bw.cu — bandwidth-bound kernels on 16-bit NHWC views.
//
// Reference semantics (/root/reference/pkg/src/dagfuse/executor.py):
//   maxpool2d      :95-109   (+ padding, extension)      -> pool_kernel
//   global_avg_pool:126-133  sum * fp32(1/HW)            -> gap_kernel
//   batchnorm/relu/residual_add/concat copy :112-166      -> ew_kernel
// Extension kinds: depthwise conv (dwconv_kernel), avgpool2d (pool_kernel),
// hardswish/hardsigmoid/silu/sigmoid/channel_scale (ew_kernel epilogue).
// Every kernel moves 8 channels (16 B) per thread when the view's channel
// offset allows it and falls back to scalar lanes for ragged toy shapes.
// Templated on the storage type T (__half or __nv_bfloat16).
#include "dfx_common.cuh"
#include "dfx_epi.cuh"

namespace dfx {

__device__ __forceinline__ int64_t grid_stride_start() {
  return blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
}
__device__ __forceinline__ int64_t grid_stride_step() { return int64_t(gridDim.x) * blockDim.x; }

// ------------------------------------------------------------------ elementwise
template <typename T>
__global__ void ew_kernel(const __grid_constant__ dfx_ew_params P) {
  griddep_wait();
  griddep_launch();
  const dfx_view& in = P.in;
  const dfx_view& out = P.out;
  const int cg = (in.c + 7) / 8;
  const int hw = in.h * in.w;
  const int64_t total = int64_t(in.n) * hw * cg;
  const bool vec_ok_views = ((in.coff | out.coff | (P.epi.binop ? P.epi.other.coff : 0)) & 7) == 0;
  for (int64_t idx = grid_stride_start(); idx < total; idx += grid_stride_step()) {
    const int64_t pix = idx / cg;
    const int c = int(idx - pix * cg) * 8;
    const int n = int(pix / hw);
    if (vec_ok_views && c + 8 <= in.c) {
      float v[8];
      ldv8<T>(in, view_pixel_index(in, pix, c), v);
      epilogue8<T>(P.epi, v, pix, n, c);
      stv8<T>(out, view_pixel_index(out, pix, c), v);
    } else {
      for (int i = 0; i < 8 && c + i < in.c; ++i) {
        const float x = ldv1<T>(in, view_pixel_index(in, pix, c + i));
        stv1<T>(out, view_pixel_index(out, pix, c + i), epilogue<T>(P.epi, x, pix, n, c + i));
      }
    }
  }
}

// Vector form (every view 8-channel aligned, c % 8 == 0): 32-bit indexing, the
// first activation a template parameter, two 16-B items in flight per thread.
// The generic kernel above spent its issue slots on 64-bit divisions and the
// activation switch (DenseNet's pre-activation BN + ReLU copies, 82 launches).
template <typename T, int ACT1>
__global__ void __launch_bounds__(256) ew_vec_kernel(const __grid_constant__ dfx_ew_params P) {
  griddep_wait();
  griddep_launch();
  const dfx_view& in = P.in;
  const dfx_view& out = P.out;
  const dfx_epilogue& e = P.epi;
  const unsigned cg = unsigned(in.c) >> 3;
  const unsigned hw = unsigned(in.h * in.w);
  const unsigned total = unsigned(in.n) * hw * cg;
  const unsigned stride = gridDim.x * blockDim.x;
  const float* alpha = e.alpha;
  const float* beta = e.beta;
  const int binop = e.binop, act2 = e.act2;
  for (unsigned i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < total; i0 += 2 * stride) {
    float v[2][8];
    unsigned pix[2], c[2];
    bool ok[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {                     // both loads issued before any math
      const unsigned idx = i0 + u * stride;
      ok[u] = idx < total;
      pix[u] = ok[u] ? idx / cg : 0u;
      c[u] = (ok[u] ? idx - pix[u] * cg : 0u) * 8u;
      if (ok[u]) ldv8<T>(in, view_pixel_index(in, pix[u], int(c[u])), v[u]);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (!ok[u]) continue;
      float* x = v[u];
      const int cc = int(c[u]);
      if (alpha) {
        const float4 a0 = *reinterpret_cast<const float4*>(alpha + cc), a1 = *reinterpret_cast<const float4*>(alpha + cc + 4);
        x[0] *= a0.x; x[1] *= a0.y; x[2] *= a0.z; x[3] *= a0.w; x[4] *= a1.x; x[5] *= a1.y; x[6] *= a1.z; x[7] *= a1.w;
      }
      if (beta) {
        const float4 b0 = *reinterpret_cast<const float4*>(beta + cc), b1 = *reinterpret_cast<const float4*>(beta + cc + 4);
        x[0] += b0.x; x[1] += b0.y; x[2] += b0.z; x[3] += b0.w; x[4] += b1.x; x[5] += b1.y; x[6] += b1.z; x[7] += b1.w;
      }
      act8_t<ACT1, kSplitT<T>>(x);
      if (binop != DFX_BIN_NONE) {
        const int n = int(pix[u] / hw);
        float o[8];
        ldv8<T>(e.other, binop == DFX_BIN_ADD ? view_pixel_index(e.other, pix[u], cc)
                                                  : int64_t(n) * e.other.pitch + e.other.coff + cc, o);
        if (binop == DFX_BIN_ADD) {
#pragma unroll
          for (int i = 0; i < 8; ++i) x[i] += o[i];
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) x[i] *= o[i];
        }
      }
      if (act2 == DFX_ACT_RELU) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fmaxf(x[i], 0.0f);
      } else if (act2 != DFX_ACT_NONE) {
        act8<kSplitT<T>>(act2, x);
      }
      stv8<T>(out, view_pixel_index(out, pix[u], cc), x);
    }
  }
}

#define DFX_EW_INST(T)                                                                            \
  template __global__ void ew_vec_kernel<T, DFX_ACT_NONE>(const __grid_constant__ dfx_ew_params);  \
  template __global__ void ew_vec_kernel<T, DFX_ACT_RELU>(const __grid_constant__ dfx_ew_params);  \
  template __global__ void ew_vec_kernel<T, DFX_ACT_HARDSWISH>(const __grid_constant__ dfx_ew_params); \
  template __global__ void ew_vec_kernel<T, DFX_ACT_HARDSIGMOID>(const __grid_constant__ dfx_ew_params); \
  template __global__ void ew_vec_kernel<T, DFX_ACT_SILU>(const __grid_constant__ dfx_ew_params);  \
  template __global__ void ew_vec_kernel<T, DFX_ACT_SIGMOID>(const __grid_constant__ dfx_ew_params); \
  template __global__ void ew_vec_kernel<T, DFX_ACT_GELU>(const __grid_constant__ dfx_ew_params);
DFX_EW_INST(__half)
DFX_EW_INST(__nv_bfloat16)
DFX_EW_INST(f16x2)
DFX_EW_INST(bf16x2)
#undef DFX_EW_INST

// ------------------------------------------------------------------ depthwise conv (tiled)
// Square K x K depthwise conv with stride S (the 3x3 / 5x5, stride 1 / 2 layers
// of MobileNetV3 and EfficientNetV2).  One thread = 8 channels (16 B) x QV
// consecutive output pixels of one row: each input row's (QV-1)*S + K columns
// are loaded once and reused by the QV outputs (a 3x3/s1 tap costs 1.5 loads
// per output at QV = 4 instead of 9), the taps of a kernel row are held in
// registers, and all index math is 32-bit (the generic kernel below spends
// most of its issue slots on 64-bit divisions).  Same fold order as the
// generic kernel: for every output, (ki, kj) ascending.
template <typename T, int K, int S, int QV, int ACT>
__global__ void __launch_bounds__(256) dwconv_tile_kernel(const __grid_constant__ dfx_dwconv_params P) {
  griddep_wait();
  griddep_launch();
  const dfx_view& in = P.in;
  const dfx_view& out = P.out;
  constexpr int NCOL = (QV - 1) * S + K;
  const int C = in.c, cg = C >> 3;
  const int OW = out.w, OH = out.h, IW = in.w, IH = in.h;
  const int qb = (OW + QV - 1) / QV;
  const unsigned total = unsigned(out.n) * unsigned(OH) * unsigned(qb) * unsigned(cg);
  const T* ib = reinterpret_cast<const T*>(in.base);
  for (unsigned item = blockIdx.x * blockDim.x + threadIdx.x; item < total;
       item += gridDim.x * blockDim.x) {
    const unsigned cgi = item % unsigned(cg);
    unsigned t = item / unsigned(cg);
    const int qbi = int(t % unsigned(qb));
    t /= unsigned(qb);
    const int p = int(t % unsigned(OH));
    const int n = int(t / unsigned(OH));
    const int c = int(cgi) * 8;
    const int q0 = qbi * QV;
    const int h0 = p * S - P.pad_h, w0 = q0 * S - P.pad_w;
    float acc[QV][8];
#pragma unroll
    for (int v = 0; v < QV; ++v)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[v][i] = 0.0f;
#pragma unroll
    for (int ki = 0; ki < K; ++ki) {
      const int h = h0 + ki;
      if (h < 0 || h >= IH) continue;
      float wv[K][8];
#pragma unroll
      for (int kj = 0; kj < K; ++kj) {
        const float4* wt = reinterpret_cast<const float4*>(P.weight + (ki * K + kj) * C + c);
        const float4 lo = __ldg(wt), hi = __ldg(wt + 1);
        wv[kj][0] = lo.x; wv[kj][1] = lo.y; wv[kj][2] = lo.z; wv[kj][3] = lo.w;
        wv[kj][4] = hi.x; wv[kj][5] = hi.y; wv[kj][6] = hi.z; wv[kj][7] = hi.w;
      }
      const T* row = ib + (int64_t(n) * IH + h) * IW * in.pitch + in.coff + c;
#pragma unroll
      for (int j = 0; j < NCOL; ++j) {
        const int w = w0 + j;
        if (w < 0 || w >= IW) continue;
        float x[8];
        ld8<T>(row, int64_t(w) * in.pitch, lo_of<T>(in), x);
#pragma unroll
        for (int v = 0; v < QV; ++v) {
          const int kj = j - v * S;
          if (kj < 0 || kj >= K) continue;
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[v][i] = fmaf(wv[kj][i], x[i], acc[v][i]);
        }
      }
    }
#pragma unroll
    for (int v = 0; v < QV; ++v) {
      const int q = q0 + v;
      if (q >= OW) break;
      const int64_t pix = (int64_t(n) * OH + p) * OW + q;
      if (P.epi.binop == DFX_BIN_NONE && P.epi.act2 == DFX_ACT_NONE && P.epi.act1 == ACT) {
        // folded BN + the (template) activation: no per-element switch
        float* x = acc[v];
        const float* al = P.epi.alpha;
        const float* be = P.epi.beta;
        if (al) {
          const float4 a0 = *reinterpret_cast<const float4*>(al + c), a1 = *reinterpret_cast<const float4*>(al + c + 4);
          x[0] *= a0.x; x[1] *= a0.y; x[2] *= a0.z; x[3] *= a0.w; x[4] *= a1.x; x[5] *= a1.y; x[6] *= a1.z; x[7] *= a1.w;
        }
        if (be) {
          const float4 b0 = *reinterpret_cast<const float4*>(be + c), b1 = *reinterpret_cast<const float4*>(be + c + 4);
          x[0] += b0.x; x[1] += b0.y; x[2] += b0.z; x[3] += b0.w; x[4] += b1.x; x[5] += b1.y; x[6] += b1.z; x[7] += b1.w;
        }
        act8_t<ACT, kSplitT<T>>(x);
      } else {
        epilogue8<T>(P.epi, acc[v], pix, n, c);
      }
      stv8<T>(out, view_pixel_index(out, pix, c), acc[v]);
    }
  }
}

#define DFX_DW_INST_A(T, K, S, A)                                                                    \
  template __global__ void dwconv_tile_kernel<T, K, S, 1, A>(const __grid_constant__ dfx_dwconv_params); \
  template __global__ void dwconv_tile_kernel<T, K, S, 2, A>(const __grid_constant__ dfx_dwconv_params); \
  template __global__ void dwconv_tile_kernel<T, K, S, 4, A>(const __grid_constant__ dfx_dwconv_params);
#define DFX_DW_INST(T, K, S)                   \
  DFX_DW_INST_A(T, K, S, DFX_ACT_NONE)         \
  DFX_DW_INST_A(T, K, S, DFX_ACT_RELU)         \
  DFX_DW_INST_A(T, K, S, DFX_ACT_HARDSWISH)    \
  DFX_DW_INST_A(T, K, S, DFX_ACT_SILU)
DFX_DW_INST(__half, 3, 1)
DFX_DW_INST(__half, 3, 2)
DFX_DW_INST(__half, 5, 1)
DFX_DW_INST(__half, 5, 2)
DFX_DW_INST(__nv_bfloat16, 3, 1)
DFX_DW_INST(__nv_bfloat16, 3, 2)
DFX_DW_INST(__nv_bfloat16, 5, 1)
DFX_DW_INST(__nv_bfloat16, 5, 2)
DFX_DW_INST(f16x2, 3, 1)
DFX_DW_INST(f16x2, 3, 2)
DFX_DW_INST(f16x2, 5, 1)
DFX_DW_INST(f16x2, 5, 2)
DFX_DW_INST(bf16x2, 3, 1)
DFX_DW_INST(bf16x2, 3, 2)
DFX_DW_INST(bf16x2, 5, 1)
DFX_DW_INST(bf16x2, 5, 2)
#undef DFX_DW_INST_A
#undef DFX_DW_INST

// ------------------------------------------------------------------ depthwise conv (generic)
// One thread = 8 channels of one output pixel; fp32 taps [kh*kw][c].
template <typename T>
__global__ void dwconv_kernel(const __grid_constant__ dfx_dwconv_params P) {
  griddep_wait();
  griddep_launch();
  const dfx_view& in = P.in;
  const dfx_view& out = P.out;
  const int C = in.c;
  const int cg = (C + 7) / 8;
  const int64_t total = int64_t(out.n) * out.h * out.w * cg;
  const bool vec_ok_views = ((in.coff | out.coff) & 7) == 0 && (C & 7) == 0;
  for (int64_t idx = grid_stride_start(); idx < total; idx += grid_stride_step()) {
    const int64_t pix = idx / cg;
    const int c = int(idx - pix * cg) * 8;
    const int q = int(pix % out.w);
    const int p = int((pix / out.w) % out.h);
    const int n = int(pix / (int64_t(out.w) * out.h));
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
    const int h0 = p * P.stride_h - P.pad_h;
    const int w0 = q * P.stride_w - P.pad_w;
    if (vec_ok_views) {
      for (int ki = 0; ki < P.kh; ++ki) {
        const int h = h0 + ki;
        if (h < 0 || h >= in.h) continue;
        for (int kj = 0; kj < P.kw; ++kj) {
          const int w = w0 + kj;
          if (w < 0 || w >= in.w) continue;
          float x[8];
          ldv8<T>(in, view_index(in, n, h, w, c), x);
          const float* wt = P.weight + int64_t(ki * P.kw + kj) * C + c;
          const float4 w_lo = __ldg(reinterpret_cast<const float4*>(wt));
          const float4 w_hi = __ldg(reinterpret_cast<const float4*>(wt + 4));
          acc[0] = fmaf(w_lo.x, x[0], acc[0]); acc[1] = fmaf(w_lo.y, x[1], acc[1]);
          acc[2] = fmaf(w_lo.z, x[2], acc[2]); acc[3] = fmaf(w_lo.w, x[3], acc[3]);
          acc[4] = fmaf(w_hi.x, x[4], acc[4]); acc[5] = fmaf(w_hi.y, x[5], acc[5]);
          acc[6] = fmaf(w_hi.z, x[6], acc[6]); acc[7] = fmaf(w_hi.w, x[7], acc[7]);
        }
      }
      epilogue8<T>(P.epi, acc, pix, n, c);
      stv8<T>(out, view_pixel_index(out, pix, c), acc);
    } else {
      for (int i = 0; i < 8 && c + i < C; ++i) {
        float a = 0.0f;
        for (int ki = 0; ki < P.kh; ++ki) {
          const int h = h0 + ki;
          if (h < 0 || h >= in.h) continue;
          for (int kj = 0; kj < P.kw; ++kj) {
            const int w = w0 + kj;
            if (w < 0 || w >= in.w) continue;
            a = fmaf(P.weight[int64_t(ki * P.kw + kj) * C + c + i],
                     ldv1<T>(in, view_index(in, n, h, w, c + i)), a);
          }
        }
        stv1<T>(out, view_pixel_index(out, pix, c + i), epilogue<T>(P.epi, a, pix, n, c + i));
      }
    }
  }
}

// ------------------------------------------------------------------ pooling
// Index type I: 32-bit when the item count allows (64-bit divisions per item were
// most of the instructions of the bandwidth-bound pools), else 64-bit.
template <typename T, typename I>
__device__ __forceinline__ void pool_body(const dfx_pool_params& P) {
  const dfx_view& in = P.in;
  const dfx_view& out = P.out;
  const int C = in.c;
  const int cg = (C + 7) / 8;
  const I total = I(out.n) * I(out.h) * I(out.w) * I(cg);
  const bool vec = ((in.coff | out.coff) & 7) == 0;
  for (I idx = I(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += I(gridDim.x) * blockDim.x) {
    const I pixi = idx / I(cg);
    const int c = int(idx - pixi * I(cg)) * 8;
    const int q = int(pixi % I(out.w));
    const I pr = pixi / I(out.w);
    const int p = int(pr % I(out.h));
    const int n = int(pr / I(out.h));
    const int64_t pix = int64_t(pixi);
    const int h0 = p * P.stride_h - P.pad_h;
    const int w0 = q * P.stride_w - P.pad_w;
    const int nl = min(8, C - c);
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = P.is_max ? -INFINITY : 0.0f;
    int count = 0;
    for (int ki = 0; ki < P.kh; ++ki) {
      const int h = h0 + ki;
      if (h < 0 || h >= in.h) continue;
      for (int kj = 0; kj < P.kw; ++kj) {
        const int w = w0 + kj;
        if (w < 0 || w >= in.w) continue;
        ++count;
        float x[8];
        if (vec && nl == 8) {
          ldv8<T>(in, view_index(in, n, h, w, c), x);
        } else {
          for (int i = 0; i < 8; ++i) x[i] = i < nl ? ldv1<T>(in, view_index(in, n, h, w, c + i)) : 0.f;
        }
        if (P.is_max) {
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] = fmaxf(acc[i], x[i]);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] += x[i];
        }
      }
    }
    if (!P.is_max) {
      const float inv = 1.0f / float(P.count_include_pad ? P.kh * P.kw : count);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] *= inv;
    }
    if (vec && nl == 8) {
      stv8<T>(out, view_pixel_index(out, pix, c), acc);
    } else {
      for (int i = 0; i < nl; ++i) stv1<T>(out, view_pixel_index(out, pix, c + i), acc[i]);
    }
  }
}

template <typename T>
__global__ void pool_kernel(const __grid_constant__ dfx_pool_params P) {
  griddep_wait();
  griddep_launch();
  const int64_t total = int64_t(P.out.n) * P.out.h * P.out.w * ((P.in.c + 7) / 8);
  if (total < (int64_t(1) << 31))
    pool_body<T, uint32_t>(P);
  else
    pool_body<T, int64_t>(P);
}

// ------------------------------------------------------------------ global average pool
// grid (ceil(C/64), N), 256 threads: 8 lanes x 8 channels cover 64 channels,
// 32 thread rows split the spatial range; fixed-order smem reduction over rows
// (deterministic).  Sum * fp32(1/HW) as the reference (executor.py:129-133).
template <typename T>
__global__ void gap_kernel(const __grid_constant__ dfx_gap_params P) {
  griddep_wait();
  griddep_launch();
  __shared__ float part[32][64 + 4];
  const dfx_view& in = P.in;
  const int n = blockIdx.y;
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;
  const int c = blockIdx.x * 64 + tx * 8;
  const int hw = in.h * in.w;
  const int nl = min(8, in.c - c);
  float acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.f;
  if (nl > 0) {
    const bool vec = nl == 8 && ((in.coff + c) & 7) == 0;
    const int64_t base = view_pixel_index(in, int64_t(n) * hw, c);
    if (vec) {
      int s = ty;
      for (; s + 32 < hw; s += 64) {            // two independent 16-B loads in flight
        float x0[8], x1[8];
        ldv8<T>(in, base + int64_t(s) * in.pitch, x0);
        ldv8<T>(in, base + int64_t(s + 32) * in.pitch, x1);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += x0[i] + x1[i];
      }
      for (; s < hw; s += 32) {
        float x[8];
        ldv8<T>(in, base + int64_t(s) * in.pitch, x);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += x[i];
      }
    } else {
      for (int s = ty; s < hw; s += 32)
        for (int i = 0; i < nl; ++i) acc[i] += ldv1<T>(in, base + int64_t(s) * in.pitch + i);
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) part[ty][tx * 8 + i] = acc[i];
  __syncthreads();
  if (threadIdx.x < 64) {
    const int cc = blockIdx.x * 64 + threadIdx.x;
    if (cc < in.c) {
      float sum = 0.f;
      for (int r = 0; r < 32; ++r) sum += part[r][threadIdx.x];
      const dfx_view& out = P.out;
      stv1<T>(out, int64_t(n) * out.pitch + out.coff + cc, sum * (1.0f / float(hw)));
    }
  }
}

// ------------------------------------------------------------------ layout conversion
// fp32 CHW samples -> 16-bit NHWC (pad channels written as zero).
template <typename T>
__global__ void in_kernel(const __grid_constant__ dfx_in_params P) {
  griddep_wait();
  griddep_launch();
  const dfx_view& o = P.out;
  const int hw = o.h * o.w;
  const int cgp = (kSplitT<T> ? o.pitch / 2 : o.pitch) / 8;   // channel groups incl. padding (one plane)
  const int64_t total = int64_t(o.n) * hw * cgp;
  if (P.kh > 0) {                              // im2col of the entry conv
    const int C = P.c, H = P.h, W = P.w;
    const int64_t HW = int64_t(H) * W;
    for (int64_t idx = grid_stride_start(); idx < total; idx += grid_stride_step()) {
      const int64_t pix = idx / cgp;
      const int c0 = int(idx - pix * cgp) * 8;
      const int n = int(pix / hw);
      const int s = int(pix - int64_t(n) * hw);
      const int y = s / o.w, x = s - (s / o.w) * o.w;
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int cc = c0 + i;
        v[i] = 0.0f;
        if (cc < o.c) {
          const int rs = cc / C, c = cc - rs * C;
          const int r = rs / P.kw, sx = rs - r * P.kw;
          const int iy = y * P.sh - P.ph + r, ix = x * P.sw - P.pw + sx;
          if (iy >= 0 && iy < H && ix >= 0 && ix < W)
            v[i] = __ldg(P.src + (int64_t(n) * C + c) * HW + int64_t(iy) * W + ix);
        }
      }
      stv8<T>(o, pix * o.pitch + c0, v);
    }
    return;
  }
  for (int64_t idx = grid_stride_start(); idx < total; idx += grid_stride_step()) {
    const int64_t pix = idx / cgp;
    const int c = int(idx - pix * cgp) * 8;
    const int n = int(pix / hw);
    const int s = int(pix - int64_t(n) * hw);
    const float* src = P.src + int64_t(n) * o.c * hw + s;
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = (c + i < o.c) ? __ldg(src + int64_t(c + i) * hw) : 0.0f;
    stv8<T>(o, pix * o.pitch + c, v);
  }
}

// im2col of the entry conv (dfx_in_params.kh > 0), one CTA per (row segment of up to
// kIm2colTile output pixels, output row, image): the source window the segment
// needs (C x kh x ((TW-1)*sw + kw) fp32, zero outside the image) is staged in
// shared memory with coalesced loads, then the segment's NHWC bytes -- contiguous,
// TW * pitch halves -- are written with coalesced 16-B stores.
template <typename T>
__global__ void __launch_bounds__(256) in_im2col_kernel(const __grid_constant__ dfx_in_params P) {
  extern __shared__ float win[];
  __shared__ int off[kIm2colMaxK];                  // channel cc -> (c*kh + r)*ww + s
  griddep_wait();
  griddep_launch();
  const dfx_view& o = P.out;
  const int C = P.c, H = P.h, W = P.w, kh = P.kh, kw = P.kw;
  const int x0 = blockIdx.x * kIm2colTile, y = blockIdx.y, n = blockIdx.z;
  const int tw = min(kIm2colTile, o.w - x0);
  const int ww = (tw - 1) * P.sw + kw;              // window width
  const int iy0 = y * P.sh - P.ph, ix0 = x0 * P.sw - P.pw;
  const float* src = P.src + int64_t(n) * C * H * W;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int rc = warp; rc < C * kh; rc += blockDim.x / 32) {   // one window row per warp
    const int r = rc % kh, c = rc / kh;
    const int iy = iy0 + r;
    const bool row_ok = iy >= 0 && iy < H;
    const float* srow = src + (int64_t(c) * H + (row_ok ? iy : 0)) * W;
    for (int col = lane; col < ww; col += 32) {
      const int ix = ix0 + col;
      win[rc * ww + col] = (row_ok && ix >= 0 && ix < W) ? __ldg(srow + ix) : 0.f;
    }
  }
  const int kreal = C * kh * kw;                    // real im2col channels
  const int kb = P.split > 0 ? P.split : o.c;       // channels per block
  for (int cc = threadIdx.x; cc < kb; cc += blockDim.x) {
    const int rs = cc / C, c = cc - rs * C;
    const int r = rs / kw, s = rs - r * kw;
    off[cc] = cc < kreal ? (c * kh + r) * ww + s : -1;
  }
  __syncthreads();
  const int groups = (kSplitT<T> ? o.pitch / 2 : o.pitch) / 8;   // one plane's channel groups
  T* out = reinterpret_cast<T*>(o.base) + ((int64_t(n) * o.h + y) * o.w + x0) * o.pitch;
  for (int i = threadIdx.x; i < tw * groups; i += blockDim.x) {
    const int px = i / groups, c0 = (i - px * groups) * 8;
    const int base = px * P.sw;
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int cc = c0 + j;
      const int blk = cc / kb, k = cc - blk * kb;
      const float x = (cc < o.c && off[k] >= 0) ? win[off[k] + base] : 0.f;
      // split blocks: [x_hi | x_hi | x_lo], x_lo = x - x_hi exactly in fp32
      v[j] = blk == 2 ? x - Elt<T>::to_f(Elt<T>::from_f(x)) : x;
    }
    st8<T>(out, int64_t(px) * o.pitch + c0, lo_of<T>(o), v);
  }
}

// A member's input gate (DFX_OP_GATE): one thread waits for the host's flag, clears it
// for the next query.  The member's IN kernel follows it in the graph.
__global__ void gate_kernel(const __grid_constant__ dfx_gate_params P) {
  if (threadIdx.x == 0) {
    for (uint32_t tries = 0; ld_acquire_u32(P.flag) == 0u; ++tries) {
      __nanosleep(256);
      if (tries > (1u << 24)) __trap();                // ~4 s: never hang the GPU
    }
    *P.flag = 0u;
    __threadfence();
  }
  griddep_launch();
}

// Non-finite logits written by out_kernel since the last reset (per device): an
// fp16 overflow anywhere upstream arrives here as inf / NaN (dfx_common.cuh).
__device__ unsigned long long g_nonfinite_outputs;

// 16-bit NHWC -> fp32 samples in logical CHW order (also the flatten order).
template <typename T>
__global__ void out_kernel(const __grid_constant__ dfx_out_params P) {
  griddep_wait();
  griddep_launch();
  const dfx_view& v = P.in;
  const int hw = v.h * v.w;
  const int64_t per = int64_t(v.c) * hw;
  const int64_t total = int64_t(v.n) * per;
  for (int64_t idx = grid_stride_start(); idx < total; idx += grid_stride_step()) {
    const int n = int(idx / per);
    const int64_t r = idx - int64_t(n) * per;
    const int c = int(r / hw);
    const int s = int(r - int64_t(c) * hw);
    const float y = ldv1<T>(v, view_pixel_index(v, int64_t(n) * hw + s, c));
    P.dst[idx] = y;
    if (!isfinite(y)) atomicAdd(&g_nonfinite_outputs, 1ull);
  }
}

#define DFX_INSTANTIATE(K, P)                                               \
  template __global__ void K<__nv_bfloat16>(const __grid_constant__ P); \
  template __global__ void K<__half>(const __grid_constant__ P);          \
  template __global__ void K<f16x2>(const __grid_constant__ P);           \
  template __global__ void K<bf16x2>(const __grid_constant__ P);
DFX_INSTANTIATE(ew_kernel, dfx_ew_params)
DFX_INSTANTIATE(dwconv_kernel, dfx_dwconv_params)
DFX_INSTANTIATE(pool_kernel, dfx_pool_params)
DFX_INSTANTIATE(gap_kernel, dfx_gap_params)
DFX_INSTANTIATE(in_kernel, dfx_in_params)
DFX_INSTANTIATE(in_im2col_kernel, dfx_in_params)
DFX_INSTANTIATE(out_kernel, dfx_out_params)
#undef DFX_INSTANTIATE

}  // namespace dfx

extern "C" int dfx_nonfinite_count(int device, unsigned long long* count, int reset) {
  if (!count) return DFX_E_ARG;
  if (cudaSetDevice(device) != cudaSuccess) return DFX_E_CUDA;
  if (cudaMemcpyFromSymbol(count, dfx::g_nonfinite_outputs, sizeof(*count)) != cudaSuccess) return DFX_E_CUDA;
  if (reset) {
    const unsigned long long zero = 0;
    if (cudaMemcpyToSymbol(dfx::g_nonfinite_outputs, &zero, sizeof(zero)) != cudaSuccess) return DFX_E_CUDA;
  }
  return 0;
}
