// dfx_dw.cu — column-strip depthwise 3x3 convolution for batched layers.
//
// Replaces the reference's depthwise conv2d evaluation (groups == channels;
// /root/reference/pkg/src/dagfuse/executor.py:56-92 evaluates convs
// channel-by-channel; the depthwise kind is the zoo extension, SURVEY.md §8 KX)
// for the layers the GEMM epilogue does not absorb (batch >= 4).
//
// dwconv_tile_kernel (dfx_bw.cu) computes 8 channels x QV outputs of one row per
// thread and re-reads the 9 fp32 taps (288 B) and a 3-row input window per item.
// Here one thread owns 8 channels of ONE output column and walks a strip of
// output rows top to bottom:
//   * the 9 taps x 8 channels stay in registers for the whole strip;
//   * every input row is loaded once (3 columns, 16 B each) and scattered into
//     the accumulators of the up to ceil(3 / S) output rows that use it, so each
//     output costs S new rows x 3 loads;
//   * those loads travel one output row AHEAD as raw 16-bit vectors (read-only
//     path), so a thread always has a row of loads in flight (without this the
//     strip walk was latency-bound and slower than the tile kernel);
//   * a finished output row gets the folded BN + activation and its 16-B store.
// Measured at batch 32 (scripts/gpu_dwcol_ab.sh): EfficientNetV2-L 14x14x1344
// 20.5 -> 14.3 us, 7x7x3840 13.8 -> 11.8 us, 28x28x768 s2 17.4 -> 13.6 us; the
// 4-model batch-32 step fp16 9.69 -> 9.37 ms, fp16x2 19.39 -> 18.62 ms.
// Summation order per output: kernel rows top to bottom, columns left to right
// (fp32 FMAs), as in the tile kernel (rows outside the map contribute exact zeros).
// Strips: the output rows split (grid.y) only when the columns alone would not
// fill ~2 waves of 128-thread blocks (dw_col_strips, dfx_dw.cuh).
#include <type_traits>

#include "dfx_common.cuh"
#include "dfx_dw.cuh"
#include "dfx_epi.cuh"

namespace dfx {

template <typename T, int S, int ACT>
__global__ void __launch_bounds__(kDwColThreads) dwconv_col_kernel(const __grid_constant__ dfx_dwconv_params P) {
  constexpr int K = 3;
  constexpr int NA = (K + S - 1) / S;       // output rows one input row feeds
  griddep_wait();
  griddep_launch();
  const dfx_view& in = P.in;
  const dfx_view& out = P.out;
  const int C = in.c, cg = C >> 3;
  const int OW = out.w, OH = out.h, IW = in.w, IH = in.h;
  const int strip = (OH + int(gridDim.y) - 1) / int(gridDim.y);
  const unsigned total = unsigned(out.n) * unsigned(OW) * unsigned(cg);
  const unsigned item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= total) return;
  const int cgi = int(item % unsigned(cg));
  unsigned t = item / unsigned(cg);
  const int q = int(t % unsigned(OW));
  const int n = int(t / unsigned(OW));
  const int si = int(blockIdx.y);
  const int c = cgi * 8;
  const int p0 = si * strip, p1 = min(OH, p0 + strip);
  if (p0 >= p1) return;
  const int w0 = q * S - P.pad_w;
  const T* ib = reinterpret_cast<const T*>(in.base) + in.coff + c;
  const int64_t ilo = lo_of<T>(in);
  const int64_t img = int64_t(n) * IH;

  float wv[K][K][8];
#pragma unroll
  for (int ki = 0; ki < K; ++ki)
#pragma unroll
    for (int kj = 0; kj < K; ++kj) {
      const float4* wt = reinterpret_cast<const float4*>(P.weight + (ki * K + kj) * C + c);
      const float4 a = __ldg(wt), b = __ldg(wt + 1);
      wv[ki][kj][0] = a.x; wv[ki][kj][1] = a.y; wv[ki][kj][2] = a.z; wv[ki][kj][3] = a.w;
      wv[ki][kj][4] = b.x; wv[ki][kj][5] = b.y; wv[ki][kj][6] = b.z; wv[ki][kj][7] = b.w;
    }
  float alpha[8], beta[8];
  const bool fast = P.epi.binop == DFX_BIN_NONE && P.epi.act2 == DFX_ACT_NONE && P.epi.act1 == ACT;
  if (fast) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      alpha[i] = P.epi.alpha ? P.epi.alpha[c + i] : 1.0f;
      beta[i] = P.epi.beta ? P.epi.beta[c + i] : 0.0f;
    }
  }

  // acc[j]: output row p + j.  An input row h = p*S - pad + kk feeds output p + j
  // through kernel row ki = kk - j*S.  The per-output order of the FMAs (kernel row
  // ki ascending, then kj) is the tile kernel's.
  float acc[NA][8];
#pragma unroll
  for (int j = 0; j < NA; ++j)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[j][i] = 0.0f;

  // one input row h into the accumulators, kk = its offset from p*S - pad
  auto feed = [&](int h, auto kk_c) {
    constexpr int kk = decltype(kk_c)::value;
    if (h < 0 || h >= IH) return;
    const T* row = ib + (img + h) * int64_t(IW) * in.pitch;
#pragma unroll
    for (int kj = 0; kj < K; ++kj) {
      const int w = w0 + kj;
      if (w < 0 || w >= IW) continue;
      float x[8];
      ld8<T>(row, int64_t(w) * in.pitch, ilo, x);
#pragma unroll
      for (int j = 0; j < NA; ++j) {
        const int ki = kk - j * S;
        if (ki < 0 || ki >= K) continue;
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[j][i] = fmaf(wv[ki][kj][i], x[i], acc[j][i]);
      }
    }
  };
  // prologue: rows kk = 0 .. K-S-1 of the first output (they precede its "new" rows)
  {
    const int hb = p0 * S - P.pad_h;
    if constexpr (K - S >= 1) feed(hb + 0, std::integral_constant<int, 0>{});
    if constexpr (K - S >= 2) feed(hb + 1, std::integral_constant<int, 1>{});
  }
  // The S rows first used by output p (kk = K-S .. K-1) travel as raw 16-bit
  // vectors, loaded one output AHEAD (read-only path, zero outside the map), so
  // each thread keeps a row of loads in flight while it computes the current one.
  constexpr int PL = kSplitT<T> ? 2 : 1;
  uint4 cur[S][K][PL], nxt[S][K][PL];
  auto load_rows = [&](int p, uint4 (&r)[S][K][PL]) {
    const int hb = p * S - P.pad_h;
#pragma unroll
    for (int s2 = 0; s2 < S; ++s2) {
      const int h = hb + (K - S) + s2;
      const bool hok = p < p1 && h >= 0 && h < IH;
      const T* row = ib + (img + h) * int64_t(IW) * in.pitch;
#pragma unroll
      for (int kj = 0; kj < K; ++kj) {
        const int w = w0 + kj;
        const bool ok = hok && w >= 0 && w < IW;
#pragma unroll
        for (int pl = 0; pl < PL; ++pl)
          r[s2][kj][pl] = ok ? __ldg(reinterpret_cast<const uint4*>(row + int64_t(w) * in.pitch + pl * ilo))
                             : make_uint4(0u, 0u, 0u, 0u);
      }
    }
  };
  load_rows(p0, cur);
  for (int p = p0; p < p1; ++p) {
    load_rows(p + 1, nxt);
#pragma unroll
    for (int s2 = 0; s2 < S; ++s2) {
      const int kk = K - S + s2;
#pragma unroll
      for (int kj = 0; kj < K; ++kj) {
        float x[8];
        unpack8<T>(cur[s2][kj][0], x);
        if constexpr (PL == 2) {
          float l[8];
          unpack8<T>(cur[s2][kj][PL - 1], l);
#pragma unroll
          for (int i = 0; i < 8; ++i) x[i] += l[i];
        }
#pragma unroll
        for (int j = 0; j < NA; ++j) {
          const int ki = kk - j * S;
          if (ki < 0 || ki >= K) continue;
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[j][i] = fmaf(wv[ki][kj][i], x[i], acc[j][i]);
        }
      }
    }
    float* x = acc[0];
    const int64_t pix = (int64_t(n) * OH + p) * OW + q;
    if (fast) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {     // the tile kernel's two statements (x *= a; x += b)
        x[i] *= alpha[i];
        x[i] += beta[i];
      }
      act8_t<ACT, kSplitT<T>>(x);
    } else {
      epilogue8<T>(P.epi, x, pix, n, c);
    }
    stv8<T>(out, view_pixel_index(out, pix, c), x);
#pragma unroll
    for (int j = 0; j + 1 < NA; ++j)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[j][i] = acc[j + 1][i];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[NA - 1][i] = 0.0f;
#pragma unroll
    for (int s2 = 0; s2 < S; ++s2)
#pragma unroll
      for (int kj = 0; kj < K; ++kj)
#pragma unroll
        for (int pl = 0; pl < PL; ++pl) cur[s2][kj][pl] = nxt[s2][kj][pl];
  }
}

#define DFX_DWC_INST_A(T, A)                                                                    \
  template __global__ void dwconv_col_kernel<T, 1, A>(const __grid_constant__ dfx_dwconv_params); \
  template __global__ void dwconv_col_kernel<T, 2, A>(const __grid_constant__ dfx_dwconv_params);
#define DFX_DWC_INST(T)                  \
  DFX_DWC_INST_A(T, DFX_ACT_NONE)        \
  DFX_DWC_INST_A(T, DFX_ACT_RELU)        \
  DFX_DWC_INST_A(T, DFX_ACT_HARDSWISH)   \
  DFX_DWC_INST_A(T, DFX_ACT_SILU)
DFX_DWC_INST(__half)
DFX_DWC_INST(__nv_bfloat16)
DFX_DWC_INST(f16x2)
DFX_DWC_INST(bf16x2)
#undef DFX_DWC_INST
#undef DFX_DWC_INST_A

}  // namespace dfx
