// dfx_dw.cuh — launch geometry of the column-strip depthwise kernel (dfx_dw.cu),
// shared by the kernel and its launcher (dfx_api.cu).
#pragma once

namespace dfx {

constexpr int kDwColThreads = 128;

// Row strips per column: whole columns when n * ow * (c / 8) threads already fill
// `waves` waves of 128-thread blocks on 148 SMs, else the rows split until they do
// (every strip re-reads its K - S halo rows, so no more strips than needed).  The
// strip index is blockIdx.y; the kernel derives the strip height from gridDim.y.
inline int dw_col_strips(int n, int oh, int ow, int cg, int waves) {
  const long long cols = (long long)n * ow * cg;
  const long long target = 148LL * waves * kDwColThreads;
  long long ns = (target + cols - 1) / cols;
  if (ns < 1) ns = 1;
  if (ns > oh) ns = oh;
  return int(ns);
}

}  // namespace dfx
