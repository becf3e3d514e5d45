// dfx_epi.cuh — GEMM epilogue drain shared by gemm_kernel and gemm_persist_kernel.
//
// drain_rows (launch flag 4, A/B only) -- one warp owns 32 TMEM lanes = 32 tile rows = 32 output pixels.  Reading the
// accumulator gives each thread ONE pixel's consecutive channels, so storing
// straight from registers makes every warp store touch 32 pixels 16 B each
// (half-used 32-B sectors, ncu: "16.1 of 32 bytes per sector") and every
// residual load likewise.  Here each 16-column chunk goes through a per-warp
// fp32 smem transpose (32 rows x 20 floats, conflict-free for both the row
// writes and the column-group reads) so that lane l then handles pixel
// (l % 16) + 16 i, channels 8 (l / 16) .. +7: a warp store covers 16 pixels x
// 32 contiguous bytes (full sectors), and the residual/scale operand loads
// coalesce the same way.  The TMEM load of chunk c+1 is in flight while chunk
// c is staged and stored.
#pragma once

#include "dfx_common.cuh"

namespace dfx {

constexpr int kEpiStagePitch = 20;                        // floats per staged row
constexpr int kEpiStageWarpBytes = 32 * kEpiStagePitch * 4;   // 2560 B per warp

// Drain accumulator columns c_first, c_first + c_step, ... (16-column chunks,
// c < ncols, ncols a multiple of 16) from TMEM address `taddr` (lane base of
// this warp already folded in).  Two warps sharing a TMEM lane quadrant split
// the chunks (c_step 32) -- the drain is issue-bound, so more warps = faster.  The calling thread's own
// tile row maps to pixel `pix` of image `img`, `valid` if inside the output.
// Output channel of column j is co_base + j.  If `ws` is set the raw fp32 sums
// go to the split-K workspace plane ws[pix * ldw + co] instead.
template <typename T>
DFX_DEV void drain_rows(uint32_t taddr, float* stg, int ncols, int64_t pix, int img, bool valid,
                        int co_base, int cout, const dfx_epilogue& e, const dfx_view& o,
                        bool views_vec, float* ws, int ldw, int c_first, int c_step) {
  if (c_first >= ncols) return;
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  uint32_t cur[16], nxt[16];
  tmem_ld16_issue(taddr + uint32_t(c_first), cur);
  tmem_ld_wait(cur);
  // the two pixels this lane stores (rows lane%16 and lane%16 + 16)
  const int rr0 = lane & 15, cg = lane >> 4;
  int64_t spix[2];
  int simg[2];
  bool sval[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int src = rr0 + 16 * i;
    spix[i] = (int64_t(__shfl_sync(full, int(pix >> 32), src)) << 32) |
              uint32_t(__shfl_sync(full, int(pix & 0xffffffff), src));
    simg[i] = __shfl_sync(full, img, src);
    sval[i] = __shfl_sync(full, int(valid), src) != 0;
  }
  float4* my_row = reinterpret_cast<float4*>(stg + lane * kEpiStagePitch);
  for (int c0 = c_first; c0 < ncols; c0 += c_step) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      my_row[k] = make_float4(__uint_as_float(cur[4 * k]), __uint_as_float(cur[4 * k + 1]),
                              __uint_as_float(cur[4 * k + 2]), __uint_as_float(cur[4 * k + 3]));
    const bool more = c0 + c_step < ncols;
    if (more) tmem_ld16_issue(taddr + uint32_t(c0 + c_step), nxt);
    __syncwarp();
    const int co = co_base + c0 + 8 * cg;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float4* src = reinterpret_cast<const float4*>(stg + (rr0 + 16 * i) * kEpiStagePitch + 8 * cg);
      const float4 a = src[0], b = src[1];
      float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      if (!sval[i] || co >= cout) continue;
      if (ws != nullptr) {
        float4* dst = reinterpret_cast<float4*>(ws + spix[i] * ldw + co);
        dst[0] = a;
        dst[1] = b;
      } else if (views_vec && co + 8 <= cout) {
        epilogue8<T>(e, v, spix[i], simg[i], co);
        stv8<T>(o, view_pixel_index(o, spix[i], co), v);
      } else {
        float tail[8];          // a separate array: taking v's address would spill it on every path
#pragma unroll
        for (int k = 0; k < 8; ++k) tail[k] = v[k];
        epilogue_store_tail<T>(e, o, tail, spix[i], simg[i], co, min(8, cout - co));
      }
    }
    __syncwarp();
    if (more) {
      tmem_ld_wait(nxt);
#pragma unroll
      for (int k = 0; k < 16; ++k) cur[k] = nxt[k];
    }
  }
}

// The unstaged drain (the default): each thread stores its own row's channels
// straight from registers (16 B per thread per store, one pixel per lane).
// Measured faster than drain_rows on every batch-32 layer shape tried
// (scripts/gpu_ab_drain.sh: e.g. 3x3 64->256 55 vs 67 us, 1x1 224->1344 20 vs
// 27 us): the drain is issue-bound, and the transpose's extra shared-memory
// instructions cost more than the half-used store sectors.
//
// Issue-bound means instructions per element set the speed: the first
// activation is a template parameter (the runtime switch compiled to jump
// tables and register shuffles: ncu counted ~184 instructions per 16-column
// chunk on VGG16's first conv), the epilogue fields are copied to registers
// once, and only the ragged channel tail takes the generic path.
template <int ACT, bool P = false>
DFX_DEV void act8_t(float* v) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if constexpr (ACT == DFX_ACT_RELU) v[i] = fmaxf(v[i], 0.0f);
    else if constexpr (ACT == DFX_ACT_HARDSWISH) v[i] = v[i] * hsig_f<P>(v[i]);
    else if constexpr (ACT == DFX_ACT_HARDSIGMOID) v[i] = hsig_f<P>(v[i]);
    else if constexpr (ACT == DFX_ACT_SILU) v[i] = silu_f<P>(v[i]);
    else if constexpr (ACT == DFX_ACT_SIGMOID) v[i] = sigmoid_f<P>(v[i]);
    else if constexpr (ACT == DFX_ACT_GELU) v[i] = gelu_f(v[i]);
  }
}

// lo_cols > 0 (split precision, gemm_kernel): the accumulator is two column halves,
// [0, bn) and [lo_cols, lo_cols + bn), summed on the way out.
template <typename T>
DFX_DEV void tmem_ld16_acc(uint32_t taddr, int lo_cols, uint32_t (&r)[16]) {
  tmem_ld16_issue(taddr, r);
  if (kSplitT<T> && lo_cols > 0) {
    uint32_t q[16];
    tmem_ld16_issue(taddr + uint32_t(lo_cols), q);
    tmem_ld_wait(q);
    tmem_ld_wait(r);
#pragma unroll
    for (int k = 0; k < 16; ++k) r[k] = __float_as_uint(__uint_as_float(r[k]) + __uint_as_float(q[k]));
  } else {
    tmem_ld_wait(r);
  }
}

template <typename T, int ACT1>
DFX_DEV void drain_rows_direct_t(uint32_t taddr, int ncols, int64_t pix, int img, bool valid, int co_base,
                                 int cout, const dfx_epilogue& e, const dfx_view& o, bool views_vec, float* ws,
                                 int ldw, int c_first, int c_step, int lo_cols) {
  const float* const alpha = e.alpha;
  const float* const beta = e.beta;
  const int binop = e.binop, act2 = e.act2;
  void* const obase = o.base;
  const int64_t orow = pix * o.pitch + o.coff;                  // view_pixel_index(o, pix, 0)
  const int64_t olo = lo_of<T>(o), xlo = lo_of<T>(e.other);    // split: lo-plane offsets
  constexpr bool P = kSplitT<T>;
  const void* const xbase = e.other.base;
  const int64_t xrow = binop == DFX_BIN_ADD ? pix * e.other.pitch + e.other.coff
                                            : int64_t(img) * e.other.pitch + e.other.coff;
  // (cout - co_base) % 8 == 0: every chunk is 16 channels but possibly the tile's last,
  // which then holds exactly 8 (cout = 8 mod 16: 24, 40, 72, 120 ... channels)
  if (ws == nullptr && views_vec && ((cout - co_base) & 7) == 0 &&
      (binop == DFX_BIN_NONE || binop == DFX_BIN_ADD) &&
      act2 == DFX_ACT_NONE && (alpha == nullptr || beta != nullptr)) {
    const bool res = binop == DFX_BIN_ADD;
    // the common conv epilogue (bias / folded-BN shift, one activation, 16-B stores)
    // as a branch-free loop: per-chunk checks and reconvergence points were a
    // third of its instructions.  Full 16-channel chunks first; a final chunk with
    // 8 valid channels (cout = 8 mod 16) after the loop
    const int nfull = min(ncols, (cout - co_base) & ~15);
    auto chunk = [&](int c0, bool half) {
      uint32_t r[16];
      tmem_ld16_acc<T>(taddr + uint32_t(c0), lo_cols, r);
      float v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
      const int co = co_base + c0;
      if (alpha != nullptr) {                       // folded BN: one FFMA per element
        const float4* aq = reinterpret_cast<const float4*>(alpha + co);
        const float4* bq = reinterpret_cast<const float4*>(beta + co);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 a4 = aq[q], b4 = bq[q];
          v[4 * q] = fmaf(v[4 * q], a4.x, b4.x); v[4 * q + 1] = fmaf(v[4 * q + 1], a4.y, b4.y);
          v[4 * q + 2] = fmaf(v[4 * q + 2], a4.z, b4.z); v[4 * q + 3] = fmaf(v[4 * q + 3], a4.w, b4.w);
        }
      } else if (beta != nullptr) {
        const float4* bq = reinterpret_cast<const float4*>(beta + co);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 b4 = bq[q];
          v[4 * q] += b4.x; v[4 * q + 1] += b4.y; v[4 * q + 2] += b4.z; v[4 * q + 3] += b4.w;
        }
      }
      act8_t<ACT1, P>(v);
      act8_t<ACT1, P>(v + 8);
      if (valid) {
        if (res) {                                  // residual add (ResNet / MBConv projections)
          float x[16];
          ld8<T>(xbase, xrow + co, xlo, x);
          if (!half) ld8<T>(xbase, xrow + co + 8, xlo, x + 8);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += x[i];
        }
        st8<T>(obase, orow + co, olo, v);
        if (!half) st8<T>(obase, orow + co + 8, olo, v + 8);
      }
    };
    int c0 = c_first;
    for (; c0 < nfull; c0 += c_step) chunk(c0, false);
    if (c0 < ncols) chunk(c0, true);
    return;
  }
  for (int c0 = c_first; c0 < ncols; c0 += c_step) {
    uint32_t r[16];
    tmem_ld16_acc<T>(taddr + uint32_t(c0), lo_cols, r);
    if (!valid) continue;
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
    const int co = co_base + c0;
    if (ws != nullptr) {
      float4* dst = reinterpret_cast<float4*>(ws + pix * ldw + co);
#pragma unroll
      for (int i = 0; i < 4; ++i) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    } else if (views_vec && co + 16 <= cout) {
      if (alpha != nullptr) {
        const float4* a = reinterpret_cast<const float4*>(alpha + co);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 aq = a[q];
          v[4 * q] *= aq.x; v[4 * q + 1] *= aq.y; v[4 * q + 2] *= aq.z; v[4 * q + 3] *= aq.w;
        }
      }
      if (beta != nullptr) {
        const float4* b = reinterpret_cast<const float4*>(beta + co);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 bq = b[q];
          v[4 * q] += bq.x; v[4 * q + 1] += bq.y; v[4 * q + 2] += bq.z; v[4 * q + 3] += bq.w;
        }
      }
      act8_t<ACT1, P>(v);
      act8_t<ACT1, P>(v + 8);
      if (binop != DFX_BIN_NONE) {
        float x[16];
        ld8<T>(xbase, xrow + co, xlo, x);
        ld8<T>(xbase, xrow + co + 8, xlo, x + 8);
        if (binop == DFX_BIN_ADD) {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += x[i];
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] *= x[i];
        }
      }
      if (act2 == DFX_ACT_RELU) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i], 0.0f);
      } else if (act2 != DFX_ACT_NONE) {
        act8<P>(act2, v);
        act8<P>(act2, v + 8);
      }
      st8<T>(obase, orow + co, olo, v);
      st8<T>(obase, orow + co + 8, olo, v + 8);
    } else if (views_vec && co + 8 == cout) {
      // the last 8 channels of a cout = 8 (mod 16) layer (MobileNetV3 / EfficientNetV2:
      // 24, 40, 72, 120, 184, 200 ...): one vector epilogue, not the scalar tail
      epilogue8<T>(e, v, pix, img, co);
      st8<T>(obase, orow + co, olo, v);
    } else {
      float tail[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) tail[i] = v[i];
      epilogue_store_tail<T>(e, o, tail, pix, img, co, min(16, cout - co));
    }
  }
}

template <typename T>
DFX_DEV void drain_rows_direct(uint32_t taddr, int ncols, int64_t pix, int img, bool valid,
                               int co_base, int cout, const dfx_epilogue& e, const dfx_view& o,
                               bool views_vec, float* ws, int ldw, int c_first, int c_step, int lo_cols = 0) {
#define DFX_DRAIN(A)                                                                                  \
  drain_rows_direct_t<T, A>(taddr, ncols, pix, img, valid, co_base, cout, e, o, views_vec, ws, ldw, \
                            c_first, c_step, lo_cols)
  switch (e.act1) {
    case DFX_ACT_RELU: DFX_DRAIN(DFX_ACT_RELU); break;
    case DFX_ACT_HARDSWISH: DFX_DRAIN(DFX_ACT_HARDSWISH); break;
    case DFX_ACT_HARDSIGMOID: DFX_DRAIN(DFX_ACT_HARDSIGMOID); break;
    case DFX_ACT_SILU: DFX_DRAIN(DFX_ACT_SILU); break;
    case DFX_ACT_SIGMOID: DFX_DRAIN(DFX_ACT_SIGMOID); break;
    case DFX_ACT_GELU: DFX_DRAIN(DFX_ACT_GELU); break;
    default: DFX_DRAIN(DFX_ACT_NONE); break;
  }
#undef DFX_DRAIN
}

}  // namespace dfx

namespace dfx {

// ---------------------------------------------------------------- A-operand prologue transform
// Rewrites one pipeline stage's A sub-tiles (nk k-steps of cb channels x 128 rows,
// 16-bit, TMA-swizzled: 16-B chunk bits [4:6] XOR address bits [7:9] for 128-B rows,
// [4:5]/[7:8] for 64-B rows, [4]/[7] for 32-B rows) in place, before the MMA reads
// them (dfx_gemm_desc pre_mode; 1x1 convs, so k-step == channel block).  Chunks of
// channels >= pre_cin (the zero fill of the last block) are left untouched.
template <typename T>
DFX_DEV void pre_transform_stage(uint8_t* a_base, int nk, int cb, int kstep0, const dfx_gemm_desc& D,
                                 int n0, int rows_per_img, int tid, int nthr) {
  // With nthr a multiple of 64, every chunk a thread visits (tid + k * nthr) holds
  // the SAME 8 logical channels of its k-step (the swizzle phase repeats every 8
  // rows): the per-channel vectors are loaded once per k-step, not per chunk.
  const int sub_a = 128 * cb * 2;
  const int cps = sub_a >> 4;                         // 16-B chunks per sub-tile
  const uint32_t m = cb == 64 ? 7u : (cb == 32 ? 3u : 1u);
  const int rshift = cb == 64 ? 7 : (cb == 32 ? 6 : 5);   // log2(row bytes)
  const int mode = D.pre_mode, act = D.pre_act, cin = D.pre_cin;
  const float* sc = static_cast<const float*>(D.pre_scale);
  const float* sh = D.pre_shift;
  const uint32_t a_t = uint32_t(tid) << 4;
  const uint32_t la_t = a_t ^ (((a_t >> 7) & m) << 4);
  const int lchunk = int((la_t & ((1u << rshift) - 1)) >> 4);
  const int row_step = (nthr << 4) >> rshift;          // rows advanced per k
  for (int j = 0; j < nk; ++j) {
    const int c = (kstep0 + j) * cb + lchunk * 8;
    if (c >= cin) continue;
    uint8_t* sub = a_base + j * sub_a;
    if (mode == 1) {
      const float4 a0 = *reinterpret_cast<const float4*>(sc + c), a1 = *reinterpret_cast<const float4*>(sc + c + 4);
      float4 b0 = make_float4(0.f, 0.f, 0.f, 0.f), b1 = b0;
      if (sh) {
        b0 = *reinterpret_cast<const float4*>(sh + c);
        b1 = *reinterpret_cast<const float4*>(sh + c + 4);
      }
      for (int i = tid; i < cps; i += nthr) {
        uint4* p = reinterpret_cast<uint4*>(sub + (i << 4));
        float x[8];
        unpack8<T>(*p, x);
        x[0] = fmaf(x[0], a0.x, b0.x); x[1] = fmaf(x[1], a0.y, b0.y);
        x[2] = fmaf(x[2], a0.z, b0.z); x[3] = fmaf(x[3], a0.w, b0.w);
        x[4] = fmaf(x[4], a1.x, b1.x); x[5] = fmaf(x[5], a1.y, b1.y);
        x[6] = fmaf(x[6], a1.z, b1.z); x[7] = fmaf(x[7], a1.w, b1.w);
        act8(act, x);
        *p = pack8<T>(x);
      }
    } else {
      int row = int(la_t >> rshift), cur_n = -1;
      float g[8];
      for (int i = tid; i < cps; i += nthr, row += row_step) {
        const int n = n0 + row / rows_per_img;
        if (n != cur_n) {
          ld8<T>(D.pre_scale, int64_t(n) * D.pre_pitch + c, 0, g);
          cur_n = n;
        }
        uint4* p = reinterpret_cast<uint4*>(sub + (i << 4));
        float x[8];
        unpack8<T>(*p, x);
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] *= g[k];
        *p = pack8<T>(x);
      }
    }
  }
}

// generic-proxy smem writes -> visible to the tensor core's async proxy
DFX_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
DFX_DEV void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace dfx

namespace dfx {

// ---- depthwise epilogue of a GEMM CTA (dfx_gemm_desc.dw_k > 0)
//
// The CTA's drain left its bn channels of the WHOLE GEMM output map in shared
// memory (xs[((n * P + h) * Q + w) * xp + c], 16-bit, exactly the values the
// unfused GEMM would have stored).  Depthwise convolution is channel-separable,
// so these channels' depthwise outputs need nothing from other CTAs: no halo
// exchange and no HBM round trip of the expanded map.  Arithmetic order is
// dwconv_tile_kernel's (taps (ki, kj) ascending, fmaf, then * alpha + beta and
// the activation), so fused and unfused results are bit-identical.
// Cluster variant (D.mt_p == 2, one M tile per CTA of a 2-CTA cluster): each CTA
// drained its own rows; rows p >= D.tp live in rank 1's shared memory and are read
// over DSMEM, and the output items are split between the two ranks.
template <typename T>
DFX_DEV void se_finish(const dfx_gemm_desc& D, uint8_t* se_smem, const float (*csum)[8], int item0, int total,
                       int N, int OH, int OW, int co_base, int nch, const dfx_view& o, int bn, int tid, int nthr,
                       const uint16_t* wsm, uint64_t* gbar);

DFX_DEV void dw_squeeze(const dfx_gemm_desc& D, uint8_t* scratch, const float (*csum)[8], int item0, int N,
                        int hw, int co_base, int nch, int tid, int nthr);

template <typename T, int K, int S, int ACT>
DFX_DEV void dw_smem_t(const dfx_gemm_desc& D, const T* xs, int xp, int N, int P, int Q, int co_base,
                       int nch, const dfx_view& o, const float* sw, int bn, int tid, int nthr,
                       uint8_t* se_smem, uint64_t* gbar) {
  const int OH = o.h, OW = o.w, cg = nch >> 3, C = D.cout;
  int total = N * OH * OW * cg;
  const bool pair = D.mt_p == 2 && D.m2 == 0;         // 2-CTA cluster, split along p
  const int rank = pair ? int(cluster_ctarank()) : 0;
  int item0 = 0;
  if (pair) {
    const int half = (total + 1) / 2;
    item0 = rank * half;
    total = min(total, item0 + half);
  }
  const int tp_rows = D.tp;
  // taps [K*K][bn] then alpha[bn], beta[bn] (staged in smem; identity when absent)
  const float* const al = sw + K * K * bn;
  const float* const be = al + bn;
  const bool has_al = D.dw_alpha != nullptr, has_be = D.dw_beta != nullptr;
  // split precision: a pixel of the map holds [hi (xp) | lo (xp)]
  constexpr bool kSp = kSplitT<T>;
  const int pp = kSp ? 2 * xp : xp;
  (void)C;
  // SE after the depthwise (D.se): outputs stay in shared memory (ot, stored-tensor
  // rounding) and each thread sums its channel group's rounded values per image
  float csum[2][8];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int i = 0; i < 8; ++i) csum[a][i] = 0.0f;
  T* const ot = reinterpret_cast<T*>(se_smem);
  const int64_t ot_lo = int64_t(N) * OH * OW * nch;   // lo plane of the tile (split)
  for (int item = item0 + tid; item < total; item += nthr) {
    const int cgi = item % cg;
    int t = item / cg;
    const int q = t % OW;
    t /= OW;
    const int p = t % OH;
    const int n = t / OH;
    const int c = cgi * 8, ca = co_base + c;
    const int h0 = p * S - D.dw_pad, w0 = q * S - D.dw_pad;
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
#pragma unroll
    for (int ki = 0; ki < K; ++ki) {
      const int h = h0 + ki;
      if (h < 0 || h >= P) continue;
      const T* row = xs + (n * P + h) * Q * pp + c;
#pragma unroll
      for (int kj = 0; kj < K; ++kj) {
        const int w = w0 + kj;
        if (w < 0 || w >= Q) continue;
        const float4* wt = reinterpret_cast<const float4*>(sw + (ki * K + kj) * bn + c);
        const float4 lo = wt[0], hi = wt[1];
        const float wv[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
        float x[8];
        if (pair) {
          const float4 r4 = dsmem_ld4(row + w * pp, uint32_t(h >= tp_rows));
          unpack8<T>(*reinterpret_cast<const uint4*>(&r4), x);
          if constexpr (kSp) {
            float l[8];
            const float4 l4 = dsmem_ld4(row + w * pp + xp, uint32_t(h >= tp_rows));
            unpack8<T>(*reinterpret_cast<const uint4*>(&l4), l);
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] += l[i];
          }
        } else {
          unpack8<T>(*reinterpret_cast<const uint4*>(row + w * pp), x);
          if constexpr (kSp) {
            float l[8];
            unpack8<T>(*reinterpret_cast<const uint4*>(row + w * pp + xp), l);
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] += l[i];
          }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fmaf(wv[i], x[i], acc[i]);
      }
    }
    if (has_al) {
      const float4 a0 = *reinterpret_cast<const float4*>(al + c), a1 = *reinterpret_cast<const float4*>(al + c + 4);
      acc[0] *= a0.x; acc[1] *= a0.y; acc[2] *= a0.z; acc[3] *= a0.w;
      acc[4] *= a1.x; acc[5] *= a1.y; acc[6] *= a1.z; acc[7] *= a1.w;
    }
    if (has_be) {
      const float4 b0 = *reinterpret_cast<const float4*>(be + c), b1 = *reinterpret_cast<const float4*>(be + c + 4);
      acc[0] += b0.x; acc[1] += b0.y; acc[2] += b0.z; acc[3] += b0.w;
      acc[4] += b1.x; acc[5] += b1.y; acc[6] += b1.z; acc[7] += b1.w;
    }
    act8_t<ACT, kSp>(acc);
    const int64_t pix = (int64_t(n) * OH + p) * OW + q;
    if (se_smem == nullptr) {
      stv8<T>(o, view_pixel_index(o, pix, ca), acc);
    } else if (D.se->mode == 1) {
      // squeeze only: store as usual, sum the stored (rounded) values per channel
      stv8<T>(o, view_pixel_index(o, pix, ca), acc);
      float r[8];
      if constexpr (kSp) {
        uint4 h, l;
        pack8_split<T>(acc, h, l);
        float lv[8];
        unpack8<T>(h, r);
        unpack8<T>(l, lv);
#pragma unroll
        for (int i = 0; i < 8; ++i) r[i] += lv[i];
      } else {
        unpack8<T>(pack8<T>(acc), r);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) csum[n & 1][i] += r[i];
    } else {
      st8<T>(ot, pix * nch + c, ot_lo, acc);
      float r[8];
      ld8<T>(ot, pix * nch + c, ot_lo, r);           // the value a stored tensor would hold
#pragma unroll
      for (int i = 0; i < 8; ++i) csum[n & 1][i] += r[i];
    }
  }
  if (se_smem != nullptr) {
    if (D.se->mode == 1)
      dw_squeeze(D, se_smem, csum, item0, N, OH * OW, co_base, nch, tid, nthr);
    else
      se_finish<T>(D, se_smem, csum, item0, total, N, OH, OW, co_base, nch, o, bn, tid, nthr,
                   reinterpret_cast<const uint16_t*>(sw + (K * K + 2) * bn), gbar);
  }
}

// Channel sums of this CTA's depthwise outputs (csum: per thread, its fixed channel
// group (item0 + tid) % cg) reduced in a fixed order: a butterfly over the lanes of
// equal group (xor cg .. 16), then warps in warp order; a 2-CTA pair adds the
// peer's sums over DSMEM in rank order.  Leaves mean[n * nch + c] (x 1/hw) in smem.
DFX_DEV void dw_channel_means(float* red, float* mean, float* peer, const float (*csum)[8], int item0, int N,
                              int hw, int nch, int tid, int nthr, bool pair) {
  const int cg = nch >> 3;
  const int lane = tid & 31, wid = tid >> 5, nwarps = nthr >> 5;
  float v[16];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int i = 0; i < 8; ++i) v[a * 8 + i] = csum[a][i];
  for (int off = cg; off < 32; off <<= 1)
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], off);
  if (lane < cg)
#pragma unroll
    for (int i = 0; i < 16; ++i) red[(wid * cg + lane) * 16 + i] = v[i];
  __syncthreads();
  const float inv = 1.0f / float(hw);
  for (int k = tid; k < N * nch; k += nthr) {
    const int n = k / nch, c = k - n * nch, g = c >> 3, i = c & 7;
    const int l = ((g - item0) % cg + cg) % cg;        // the lane that held group g
    float s = 0.0f;
    for (int w = 0; w < nwarps; ++w) s += red[(w * cg + l) * 16 + (n & 1) * 8 + i];
    if (pair) peer[k] = s;
    else mean[k] = s * inv;
  }
  if (pair) {
    cluster_sync_all();
    for (int k = tid; k < N * nch; k += nthr) mean[k] = (dsmem_ld1(peer + k, 0) + dsmem_ld1(peer + k, 1)) * inv;
    cluster_sync_all();                                // peers done reading peer[]
  } else {
    __syncthreads();
  }
}

// dfx_se_fuse mode 1: the SE launch after this GEMM reads its channel means from
// D.se->pooled ([n][c]) instead of pooling x (rank 0 of a pair writes).
DFX_DEV void dw_squeeze(const dfx_gemm_desc& D, uint8_t* scratch, const float (*csum)[8], int item0, int N,
                        int hw, int co_base, int nch, int tid, int nthr) {
  float* const red = reinterpret_cast<float*>(scratch);
  float* const mean = red + nthr * 16;
  float* const peer = mean + 2 * nch;
  const bool pair = D.mt_p == 2 && D.m2 == 0;
  dw_channel_means(red, mean, peer, csum, item0, N, hw, nch, tid, nthr, pair);
  if (!pair || cluster_ctarank() == 0) {
    const dfx_se_fuse& F = *D.se;
    for (int k = tid; k < N * nch; k += nthr) {
      const int n = k / nch, c = k - n * nch;
      F.pooled[int64_t(n) * F.c + co_base + c] = mean[k];
    }
  }
}


// The squeeze-excitation of the fused MBConv middle (dfx_gemm_desc.se), after the
// depthwise outputs of this CTA's bn channels sit in `ot` (stored-tensor rounding):
//   1. channel sums: per-thread partials (fixed channel group per thread) reduced in
//      thread order; a 2-CTA pair adds the peer's over DSMEM in rank order; x (1/HW);
//   2. fc1 partial over this CTA's channels (c ascending) -> se->scratch[N tile];
//   3. ONE grid-wide barrier (arrival counter + epoch; every CTA of the grid is
//      resident: the host keeps the grid within its share of the SMs, and the
//      successor launches only after every CTA called launch_dependents);
//   4. hidden = act1(b1 + sum over N tiles in order), gates of this CTA's channels
//      = act2(b2 + fc2 rows . hidden), out = x * gate (the se_kernel apply path).
template <typename T>
DFX_DEV void se_finish(const dfx_gemm_desc& D, uint8_t* se_smem, const float (*csum)[8], int item0, int total,
                       int N, int OH, int OW, int co_base, int nch, const dfx_view& o, int bn, int tid, int nthr,
                       const uint16_t* wsm, uint64_t* gbar) {
  constexpr bool kSp = kSplitT<T>;
  const dfx_se_fuse& F = *D.se;
  const int Cr = F.cr, cg = nch >> 3;
  const int hw = OH * OW;
  const int64_t npix = int64_t(N) * hw;
  T* const ot = reinterpret_cast<T*>(se_smem);
  const int64_t ot_lo = npix * nch;
  float* const red = reinterpret_cast<float*>(se_smem + ((npix * nch * 2 * (kSp ? 2 : 1) + 15) & ~15));
  float* const mean = red + nthr * 16;                 // [2][nch]
  float* const hidden = mean + 2 * bn;                 // [2][Cr]
  float* const gate = hidden + 2 * ((Cr + 3) & ~3);    // [2][nch]
  float* const part = gate + 2 * bn;                   // [N tiles][N][Cr]: the gathered fc1 partials (16-B aligned)
  const bool pair = D.mt_p == 2 && D.m2 == 0;
  const uint32_t rank = pair ? cluster_ctarank() : 0u;
  if (tid == 0) DFX_TL(50);                            // depthwise done
  // 1. channel means (dw_channel_means; gate[] is the pair's exchange buffer)
  dw_channel_means(red, mean, gate, csum, item0, N, hw, nch, tid, nthr, pair);
  if (tid == 0) DFX_TL(51);                            // channel means
  // 2. fc1 partial over this CTA's channels (fc1^T rows staged in smem: wsm =
  // [w1 hi, w2 hi(, w1 lo, w2 lo)] of [bn][Cr]) -> scratch (rank 0 of a pair only)
  const int ntile = co_base / bn;
  const T* w1 = reinterpret_cast<const T*>(wsm);
  const T* w2 = w1 + bn * Cr;
  const int wlo = kSp ? 2 * bn * Cr : 0;
  if (tid == 0) mbar_wait(gbar + 1, 0);               // the staged fc1^T / fc2 rows landed
  __syncthreads();
  if (rank == 0) {
    for (int k = tid; k < N * Cr; k += nthr) {
      const int n = k / Cr, j = k - n * Cr;
      float s = 0.0f;
#pragma unroll 4
      for (int c = 0; c < nch; ++c) {
        const int wi = c * Cr + j;
        float wv = Elt<T>::to_f(w1[wi]);
        if constexpr (kSp) wv += Elt<T>::to_f(w1[wi + wlo]);
        s = fmaf(wv, mean[n * nch + c], s);
      }
      F.scratch[(int64_t(ntile) * N + n) * Cr + j] = s;
    }
  }
  // 3. grid barrier
  __syncthreads();
  if (tid == 0) DFX_TL(52);                            // fc1 partial written
  if (tid == 0) {
    __threadfence();
    uint32_t* sync = F.sync;
    const uint32_t e = ld_acquire_u32(sync + 1);
    const uint32_t a = atomicAdd(sync, 1u) + 1u;
    if (a == uint32_t(F.ctas)) {
      atomicExch(sync, 0u);
      __threadfence();
      atomicAdd(sync + 1, 1u);
    } else {
      for (uint32_t tries = 0; ld_acquire_u32(sync + 1) == e; ++tries)
        if (tries > (1u << 28)) __trap();               // never hang the GPU
    }
    __threadfence();
  }
  __syncthreads();
  if (tid == 0) DFX_TL(53);                            // barrier passed
  // 4. every N tile's partials in ONE bulk copy (global -> smem; the barrier's acquire
  // plus a cross-proxy fence order it after the other CTAs' stores), hidden vector,
  // gates of this CTA's channels, scale
  const int ntiles = D.nt;
  if (tid == 0) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    const uint32_t bytes = (uint32_t(ntiles) * N * Cr * 4 + 15) & ~15u;
    mbar_arrive_expect_tx(gbar, bytes);
    bulk_load(part, F.scratch, bytes, gbar);
    mbar_wait(gbar, 0);
  }
  __syncthreads();
  if (tid == 0) DFX_TL(54);                            // partials gathered
  {                                                    // nparts threads per hidden unit
    const int units = N * Cr;
    const int np = max(1, min(8, nthr / units));
    const int tlen = (ntiles + np - 1) / np;
    for (int k = tid; k < units * np; k += nthr) {
      const int u = k / np, pt = k - u * np;
      const int n = u / Cr, j = u - n * Cr;
      const int t0 = pt * tlen, t1 = min(ntiles, t0 + tlen);
      float s = 0.0f;
      for (int t = t0; t < t1; ++t) s += part[(t * N + n) * Cr + j];
      red[k] = s;
    }
    __syncthreads();
    for (int u = tid; u < units; u += nthr) {
      const int n = u / Cr, j = u - n * Cr;
      float s = 0.0f;
      for (int pt = 0; pt < np; ++pt) s += red[u * np + pt];
      hidden[u] = act_apply<kSp>(F.act1, s + (F.b1 ? F.b1[j] : 0.0f));
    }
  }
  __syncthreads();
  if (tid == 0) DFX_TL(55);                            // hidden
  // fc2 rows of this CTA's channels: nparts threads per (image, channel) over
  // contiguous j ranges, partials combined in part order (deterministic)
  const int items = N * nch;
  const int nparts = max(1, min(8, nthr / items));
  const int jlen = (Cr + nparts - 1) / nparts;
  for (int k = tid; k < items * nparts; k += nthr) {
    const int it = k / nparts, part = k - it * nparts;
    const int n = it / nch, c = it - n * nch;
    const int row = c * Cr;
    const int j0 = part * jlen, j1 = min(Cr, j0 + jlen);
    float s = 0.0f;
#pragma unroll 4
    for (int j = j0; j < j1; ++j) {
      float wv = Elt<T>::to_f(w2[row + j]);
      if constexpr (kSp) wv += Elt<T>::to_f(w2[row + j + wlo]);
      s = fmaf(wv, hidden[n * Cr + j], s);
    }
    red[k] = s;                                        // red[] is free since step 1
  }
  __syncthreads();
  for (int k = tid; k < items; k += nthr) {
    const int n = k / nch, c = k - n * nch;
    float s = 0.0f;
    for (int part = 0; part < nparts; ++part) s += red[k * nparts + part];
    gate[k] = act_apply<kSp>(F.act2, s + (F.b2 ? F.b2[co_base + c] : 0.0f));
  }
  __syncthreads();
  if (tid == 0) DFX_TL(56);                            // gates
  for (int item = item0 + tid; item < total; item += nthr) {
    const int cgi = item % cg;
    int t = item / cg;
    const int q = t % OW;
    t /= OW;
    const int p = t % OH;
    const int n = t / OH;
    const int c = cgi * 8;
    const int64_t pix = (int64_t(n) * OH + p) * OW + q;
    float x[8];
    ld8<T>(ot, pix * nch + c, ot_lo, x);
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] *= gate[n * nch + c + i];
    stv8<T>(o, view_pixel_index(o, pix, co_base + c), x);
  }
  if (tid == 0) DFX_TL(57);                            // scaled output stored
}

template <typename T, int K, int S>
DFX_DEV void dw_smem_k(const dfx_gemm_desc& D, const T* xs, int xp, int N, int P, int Q, int co_base,
                       int nch, const dfx_view& o, const float* sw, int bn, int tid, int nthr, uint8_t* se_smem,
                       uint64_t* gbar) {
  switch (D.dw_act) {
    case DFX_ACT_RELU: dw_smem_t<T, K, S, DFX_ACT_RELU>(D, xs, xp, N, P, Q, co_base, nch, o, sw, bn, tid, nthr, se_smem, gbar); break;
    case DFX_ACT_HARDSWISH:
      dw_smem_t<T, K, S, DFX_ACT_HARDSWISH>(D, xs, xp, N, P, Q, co_base, nch, o, sw, bn, tid, nthr, se_smem, gbar);
      break;
    case DFX_ACT_SILU: dw_smem_t<T, K, S, DFX_ACT_SILU>(D, xs, xp, N, P, Q, co_base, nch, o, sw, bn, tid, nthr, se_smem, gbar); break;
    default: dw_smem_t<T, K, S, DFX_ACT_NONE>(D, xs, xp, N, P, Q, co_base, nch, o, sw, bn, tid, nthr, se_smem, gbar); break;
  }
}

// dispatch on the (host-validated) square kernel size / stride: 3 or 5, 1 or 2
template <typename T>
DFX_DEV void dw_smem(const dfx_gemm_desc& D, const T* xs, int xp, int N, int P, int Q, int co_base, int nch,
                     const dfx_view& o, const float* sw, int bn, int tid, int nthr, uint8_t* se_smem = nullptr,
                     uint64_t* gbar = nullptr) {
  if (D.dw_k == 3) {
    if (D.dw_s == 1) dw_smem_k<T, 3, 1>(D, xs, xp, N, P, Q, co_base, nch, o, sw, bn, tid, nthr, se_smem, gbar);
    else dw_smem_k<T, 3, 2>(D, xs, xp, N, P, Q, co_base, nch, o, sw, bn, tid, nthr, se_smem, gbar);
  } else {
    if (D.dw_s == 1) dw_smem_k<T, 5, 1>(D, xs, xp, N, P, Q, co_base, nch, o, sw, bn, tid, nthr, se_smem, gbar);
    else dw_smem_k<T, 5, 2>(D, xs, xp, N, P, Q, co_base, nch, o, sw, bn, tid, nthr, se_smem, gbar);
  }
}

}  // namespace dfx
