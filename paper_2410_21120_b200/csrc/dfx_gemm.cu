// dfx_gemm.cu — grouped implicit-GEMM convolution on tcgen05 / TMEM, fed by TMA.
//
// Replaces the reference's conv2d and dense evaluation
// (/root/reference/pkg/src/dagfuse/executor.py:56-92): 16-bit operands (fp16 or
// bf16), fp32 accumulation in TMEM, fp32 epilogue (bias / folded batch-norm /
// activation / residual add / channel scale), 16-bit NHWC store at a channel
// offset (zero-copy concat).
//
// One CTA = one (M tile, N tile, K split) of one problem of a grouped launch.
//   M tile : tn x tp x tq output pixels (<= 128 rows, one TMEM lane each)
//   N tile : bn output channels (<= 256 TMEM columns)
//   K      : (r, s, channel block) steps of cb in {16, 32, 64} channels; a
//            pipeline stage packs 64/cb steps = 64 K elements.
// The A tile of a K step is ONE 4-D TMA box over the NHWC activation
// (c, w, h, n) starting at (c0, q0*sw + s - pw, p0*sh + r - ph, n0) with
// element strides (1, sw, sh, 1): TMA's out-of-bounds zero fill implements
// the convolution padding and the channel tail, so no im2col buffer exists.
// The B tile is a 2-D TMA box of the packed [cout][K] weight matrix.
//
// Warp roles (128 threads): warp 0 lane 0 = TMA producer, warp 1 lane 0 =
// MMA issuer, warp 2 = TMEM allocator, warps 2-3 stage the epilogue vectors;
// all four warps run the epilogue (warp w owns TMEM lanes 32w..32w+31 = tile
// rows).  Latency structure (batch-1 layers are latency-bound, measured with
// the DFX_TIMELINE probes below):
//   * a single problem's descriptor and tensor maps are a __grid_constant__
//     kernel parameter (no global round trip before the first TMA);
//   * everything static -- weight tiles of the first `nslots` stages (up to 8
//     deep), the epilogue's folded-BN/bias vectors -- is requested BEFORE
//     griddepcontrol.wait, i.e. while the predecessor kernel still runs;
//   * the descriptor is copied to smem and loops run on register copies of its
//     fields (the PTX "memory" clobbers would otherwise reload them per step).
#ifdef DFX_TIMELINE
// block-0 %globaltimer probes (ns), read back with dfx_debug_timeline
__device__ unsigned long long dfx_timeline[64];
#define DFX_TL(i)                                                \
  do {                                                           \
    if (blockIdx.x == 0 && blockIdx.y == 0) {                    \
      unsigned long long _t;                                     \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));     \
      dfx_timeline[i] = _t;                                      \
    }                                                            \
  } while (0)
// block-0 clock64 probes (cycles) into slots 42..63
#define DFX_TC(i)                                                          \
  do {                                                                     \
    if (blockIdx.x == 0 && (i) < 64) dfx_timeline[i] = clock64();         \
  } while (0)
#else
#define DFX_TC(i) do { } while (0)
#endif

#include "dfx_common.cuh"
#include "dfx_epi.cuh"

// Debug builds (-DDFX_TIMELINE): copy the kernel timeline probes (ns).  Not in
// dfx.h: a development hook, not part of the ABI.
extern "C" int dfx_debug_timeline(unsigned long long* out, int n) {
#ifdef DFX_TIMELINE
  return cudaMemcpyFromSymbol(out, dfx_timeline, sizeof(unsigned long long) * (n < 64 ? n : 64)) ==
                 cudaSuccess
             ? 0
             : -1;
#else
  (void)out;
  (void)n;
  return -4;
#endif
}

namespace dfx {

// L2 prefetch of a global range (16-B aligned, size % 16 == 0): no smem, no barrier
DFX_DEV void l2_prefetch_bulk(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

struct GemmHeader {
  uint64_t full[kMaxSlots];
  uint64_t empty[kMaxSlots];
  uint64_t accum;
  uint64_t ready[kMaxSlots];   // pre_mode: A stage transformed in smem, MMA may read it
  uint32_t tmem_base;
  uint32_t last_split;    // split-K: this CTA arrived last for its output tile
  uint32_t _pad[12];
  dfx_gemm_desc desc;     // 64-B aligned copy of this CTA's problem
};
static_assert(sizeof(GemmHeader) <= kHeaderBytes, "gemm smem header overflow");

// M2 (compile-time): 256-row CTAs, see `m2` below.  A separate instantiation so the
// latency-critical 128-row path carries none of the second tile's bookkeeping.
template <typename T, int M2>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_kernel(const __grid_constant__ dfx_gemm_launch L) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // Dynamic smem base is only guaranteed 16-B aligned: round up to 1024 for swizzles.
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  GemmHeader* hdr = reinterpret_cast<GemmHeader*>(smem);
  float* s_alpha = reinterpret_cast<float*>(smem + kHeaderBytes);
  float* s_beta = s_alpha + 256;
  uint8_t* slots = smem + kSlotsOffset;
  constexpr int m2l = M2;                          // slot / TMEM sizing
  constexpr int planes = kSplitT<T> ? 2 : 1;       // split precision: hi + lo operand tiles
  const int slot_bytes = gemm_slot_bytes(L.bn_max, m2l, planes);
  const int a_lo_off = kStageABytes * (1 + m2l);   // lo A tiles follow the hi ones
  const int a_bytes = a_lo_off * planes;           // A part of a slot (B follows)
  // split precision: each k-step's B sub-tile is [hi bn rows | lo bn rows], so ONE
  // MMA with N = 2 bn computes A_hi*B_hi (TMEM columns [0, bn)) and A_hi*B_lo
  // ([bn, 2 bn)) -- an MMA costs the same at N <= 128 (its SMEM A read bounds
  // it) -- and A_lo*B_hi adds into [0, bn): two MMAs per K=16 step instead of
  // three; the drain sums the two column halves
  const int b_kstride = planes == 2 ? 2 : 1;      // sub-tile pitch in units of sub_b
  const int nslots = L.nslots;
  if (threadIdx.x == 0) DFX_TL(0);                 // CTA start
#ifdef DFX_TIMELINE
  if (threadIdx.x == 0 && blockIdx.x == 0) dfx_timeline[40] = clock64();
#endif

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int bid = blockIdx.x;

  const dfx_gemm_desc* gd;                         // tensor maps are read through this
  if (L.ndesc == 1 && (L.flags & 1) == 0) {
    gd = &L.desc0;                                 // kernel-parameter space
  } else {
    int pi = 0;
    for (int i = 1; i < L.ndesc; ++i)
      if (L.descs[i].tile_begin <= bid) pi = i;
    gd = L.descs + pi;
  }

  // ---- stage the descriptor in smem (32 x 16 B), barriers, TMEM
  if (threadIdx.x < sizeof(dfx_gemm_desc) / 16)
    reinterpret_cast<uint4*>(&hdr->desc)[threadIdx.x] =
        reinterpret_cast<const uint4*>(gd)[threadIdx.x];
  const uint32_t tmem_cols = tmem_cols_for(L.bn_max * (1 + m2l) * planes);
  if (threadIdx.x == 0) {
    DFX_TL(7);                                     // descriptor copied
    for (int i = 0; i < nslots; ++i) {
      mbar_init(&hdr->full[i], 1);
      mbar_init(&hdr->empty[i], 1);
      mbar_init(&hdr->ready[i], 1);
    }
    mbar_init(&hdr->accum, 1);
    fence_barrier_init();
    DFX_TL(8);                                     // barriers initialised
  }
  if (warp == 2) {
    tmem_alloc(&hdr->tmem_base, tmem_cols);
    if (lane == 0) DFX_TL(9);                      // TMEM allocated
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(gd->tmap_a);
    tma_prefetch_desc(gd->tmap_b);
  }
  if (warp == 1 && lane == 0 && L.l2_pf_units) {
    // the member's next weight blobs -> L2, one slice per CTA, while this launch
    // (and its predecessor) run: the next layer's weight TMA then hits L2
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const uint64_t bytes = uint64_t((L.l2_pf_units >> (16 * r)) & 0xFFFFu) << 8;
      if (bytes == 0 || L.l2_pf[r] == nullptr) continue;
      const uint64_t per = ((bytes + gridDim.x - 1) / gridDim.x + 255) & ~uint64_t(255);
      const uint64_t off = per * blockIdx.x;
      if (off < bytes) l2_prefetch_bulk(static_cast<const char*>(L.l2_pf[r]) + off, uint32_t(min(per, bytes - off)));
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) DFX_TL(10);                // prologue barrier passed
  if (L.flags & 16) griddep_launch();              // A/B: release the successor's prologue early
  const uint32_t tmem_base = hdr->tmem_base;
  const dfx_gemm_desc& D = hdr->desc;

  // ---- tile coordinates (M tiles fastest, then K splits, then N tiles)
  const int mt_q = D.mt_q, mt_p = D.mt_p, splits = D.splits;
  const int tn = D.tn, tp = D.tp, tq = D.tq;
  int t = bid - D.tile_begin;
  const int mt_total = D.mt_n * mt_p * mt_q;
  // m2: this CTA owns M tiles 2g and 2g+1 (two TMEM accumulators, columns [0, bn)
  // and [bn, 2bn)); both are multiplied by the same B stage, so the weight bytes
  // per MAC halve -- the lever when the chip-wide TMA/L2 fill rate caps the MMA.
  constexpr int m2 = M2;
  const int mgroups = m2 ? (mt_total + 1) / 2 : mt_total;
  // cluster split-K (flag 8): the `splits` CTAs of one output tile are consecutive
  // blocks = one thread-block cluster, split index = cluster rank
  const bool csplit = !M2 && (L.flags & 8) && splits > 1;
  int split, mi, ntile;
  if (csplit) {
    split = t % splits;
    t /= splits;
    mi = t % mgroups;
    ntile = t / mgroups;
  } else {
    mi = (t % mgroups) << m2;
    t /= mgroups;
    split = t % splits;
    ntile = t / splits;
  }
  const int nhalf = (m2 && mi + 1 < mt_total) ? 2 : 1;   // M tiles in this CTA
  int n0h[1 + M2], p0h[1 + M2], q0h[1 + M2];
#pragma unroll
  for (int h = 0; h < 1 + M2; ++h) {
    const int m = mi + h;
    n0h[h] = (m / (mt_q * mt_p)) * tn;
    p0h[h] = ((m / mt_q) % mt_p) * tp;
    q0h[h] = (m % mt_q) * tq;
  }
  const int bn = D.bn, cb = D.cb, kpack = D.kpack, ksteps = D.ksteps;
  const int st_begin = split * D.stages_per_split;
  const int st_end = min(D.stages, st_begin + D.stages_per_split);
  const int co_base = ntile * bn;
  const int cout = D.cout;

  const int sub_a = 128 * cb * 2;     // bytes of one K-step A sub-tile
  const int sub_b = bn * cb * 2;      // bytes of one K-step B sub-tile

  if (warp == 0 && lane == 0) {
    // ================= TMA producer
    const int cblocks = D.cblocks, S = D.s;
    int qb[1 + M2], pb[1 + M2];
#pragma unroll
    for (int h = 0; h < 1 + M2; ++h) {
      qb[h] = q0h[h] * D.stride_w - D.pad_w;
      pb[h] = p0h[h] * D.stride_h - D.pad_h;
    }
    const uint32_t box_a_bytes = uint32_t(cb) * 2u * tq * tp * tn * nhalf;
    const uint32_t tx_per_k = (box_a_bytes + uint32_t(sub_b)) * planes;
    const void* tma = gd->tmap_a;
    const void* tmb = gd->tmap_b;
    // flags bit 5: every weight tile is read by one or two CTAs (batch-1 layers)
    const uint64_t wpol = (L.flags & 32) ? l2_evict_first() : 0;
    // Weights are static: the first nslots stages' B tiles are requested before
    // the programmatic dependency resolves, overlapping the predecessor's tail.
    const int npre = min(nslots, st_end - st_begin);
    for (int it = 0; it < npre; ++it) {
      const int st = st_begin + it;
      uint8_t* b_dst = slots + it * slot_bytes + a_bytes;
      const int k0 = st * kpack;
      const int nk = min(kpack, ksteps - k0);
      mbar_arrive_expect_tx(&hdr->full[it], nk * tx_per_k);
      for (int j = 0; j < nk; ++j)       // split: one 3-D box, the k-step's hi rows then lo rows
        tma_load_w<planes>(b_dst + j * b_kstride * sub_b, tmb, &hdr->full[it], (k0 + j) * cb, co_base, wpol);
      if (it < 8) DFX_TL(30 + it);                 // B prefetch of stage `it` issued (30..37)
    }
    DFX_TL(1);                                     // weight prefetch issued
    griddep_wait();
    DFX_TL(2);                                     // dependency resolved
    // k-step cursor (channel block, s, r) advanced incrementally: the producer is
    // ONE thread, and integer divisions per k-step (~20-40 instructions each) made
    // its issue loop slower than the MMAs it feeds
    int cblk, sc, rc;
    {
      const int k = st_begin * kpack, rs = k / cblocks;
      cblk = k - rs * cblocks;
      rc = rs / S;
      sc = rs - rc * S;
    }
    int k0 = st_begin * kpack;
    for (int it = 0; it < npre; ++it, k0 += kpack) {
      uint8_t* a_dst = slots + it * slot_bytes;
      const int nk = min(kpack, ksteps - k0);
      for (int j = 0; j < nk; ++j) {
#pragma unroll
        for (int h = 0; h < 1 + M2; ++h)
          if (h < nhalf) {
            if constexpr (planes == 2) {
              tma_load_5d(a_dst + h * kStageABytes + j * sub_a, tma, &hdr->full[it], cblk * cb, qb[h] + sc,
                          pb[h] + rc, n0h[h], 0);
              tma_load_5d(a_dst + a_lo_off + h * kStageABytes + j * sub_a, tma, &hdr->full[it], cblk * cb,
                          qb[h] + sc, pb[h] + rc, n0h[h], 1);
            } else {
              tma_load_4d(a_dst + h * kStageABytes + j * sub_a, tma, &hdr->full[it], cblk * cb, qb[h] + sc,
                          pb[h] + rc, n0h[h]);
            }
          }
        if (++cblk == cblocks) {
          cblk = 0;
          if (++sc == S) {
            sc = 0;
            ++rc;
          }
        }
      }
    }
    DFX_TL(29);                                    // all prefetched stages' A loads issued
    int slot = npre == nslots ? 0 : npre;
    uint32_t par = npre == nslots ? 1u : 0u;
    for (int st = st_begin + npre; st < st_end; ++st, k0 += kpack) {
      mbar_wait(&hdr->empty[slot], par ^ 1);
      uint8_t* a_dst = slots + slot * slot_bytes;
      uint8_t* b_dst = a_dst + a_bytes;
      const int nk = min(kpack, ksteps - k0);
      mbar_arrive_expect_tx(&hdr->full[slot], nk * tx_per_k);
      for (int j = 0; j < nk; ++j) {
#pragma unroll
        for (int h = 0; h < 1 + M2; ++h)
          if (h < nhalf) {
            if constexpr (planes == 2) {
              tma_load_5d(a_dst + h * kStageABytes + j * sub_a, tma, &hdr->full[slot], cblk * cb, qb[h] + sc,
                          pb[h] + rc, n0h[h], 0);
              tma_load_5d(a_dst + a_lo_off + h * kStageABytes + j * sub_a, tma, &hdr->full[slot], cblk * cb,
                          qb[h] + sc, pb[h] + rc, n0h[h], 1);
            } else {
              tma_load_4d(a_dst + h * kStageABytes + j * sub_a, tma, &hdr->full[slot], cblk * cb, qb[h] + sc,
                          pb[h] + rc, n0h[h]);
            }
          }
        tma_load_w<planes>(b_dst + j * b_kstride * sub_b, tmb, &hdr->full[slot], (k0 + j) * cb, co_base, wpol);
        if (++cblk == cblocks) {
          cblk = 0;
          if (++sc == S) {
            sc = 0;
            ++rc;
          }
        }
      }
      if (++slot == nslots) {
        slot = 0;
        par ^= 1u;
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ================= MMA issuer
    const uint32_t idesc = umma_idesc_f16(uint32_t(bn), Elt<T>::kDtype);
    const bool wide = planes == 2 && 2 * bn <= 256;    // hi|lo B rows as one N = 2 bn MMA
    const uint32_t idesc2 = umma_idesc_f16(uint32_t(wide ? 2 * bn : bn), Elt<T>::kDtype);
    const uint32_t row_bytes = uint32_t(cb) * 2u;
    const int kk_n = cb / 16;
    uint32_t accumulate = 0;
    int it = 0;
    uint64_t* const gate_bar = D.pre_mode ? hdr->ready : hdr->full;   // pre_mode: wait for the transform
    int slot = 0;
    uint32_t par = 0;
    for (int st = st_begin; st < st_end; ++st, ++it) {
      mbar_wait(&gate_bar[slot], par);
      if (it == 0) DFX_TL(3);                      // first stage landed
      if (it > 0 && it < 9) DFX_TL(12 + it);       // later stages landed (13..20)
      if (it < 7) DFX_TC(42 + 3 * it);
      tc_fence_after();
      if (it < 7) DFX_TC(43 + 3 * it);
      const uint32_t a_base = smem_u32(slots + slot * slot_bytes);
      const uint32_t b_base = a_base + a_bytes;
      const int nk = min(kpack, ksteps - st * kpack);
      for (int j = 0; j < nk; ++j) {
        for (int kk = 0; kk < kk_n; ++kk) {
          const uint64_t bd = umma_smem_desc(b_base + j * b_kstride * sub_b + kk * 32, row_bytes);
#pragma unroll
          for (int h = 0; h < 1 + M2; ++h) {
            if (h >= nhalf) break;
            const uint64_t ad = umma_smem_desc(a_base + h * kStageABytes + j * sub_a + kk * 32, row_bytes);
#ifndef DFX_EXP_NOMMA
            if constexpr (planes == 2) {
              // [0, bn) += A_hi B_hi, [bn, 2 bn) += A_hi B_lo (one MMA when 2 bn <= 256), then
              // [0, bn) += A_lo B_hi
              const uint64_t adl =
                  umma_smem_desc(a_base + a_lo_off + h * kStageABytes + j * sub_a + kk * 32, row_bytes);
              if (wide) {
                umma_f16(tmem_base, ad, bd, idesc2, accumulate);
              } else {
                const uint64_t bdl = umma_smem_desc(b_base + (2 * j + 1) * sub_b + kk * 32, row_bytes);
                umma_f16(tmem_base, ad, bd, idesc, accumulate);
                umma_f16(tmem_base + uint32_t(bn), ad, bdl, idesc, accumulate);
              }
#ifndef DFX_EXP_SPLIT_1MMA
              umma_f16(tmem_base, adl, bd, idesc, 1u);
#else
              (void)adl;
#endif
            } else {
              umma_f16(tmem_base + uint32_t(h * bn), ad, bd, idesc, accumulate);
            }
#else
            (void)ad; (void)bd; (void)idesc;
#endif
          }
          accumulate = 1;
        }
      }
      if (it < 7) DFX_TC(44 + 3 * it);
      if (it < 8) DFX_TL(21 + it);                 // stage's MMAs issued (21..28)
      umma_commit(&hdr->empty[slot]);
      if (++slot == nslots) {
        slot = 0;
        par ^= 1u;
      }
    }
    umma_commit(&hdr->accum);
    DFX_TL(4);                                     // last MMA issued
  } else if (warp >= 2) {
    const int ti = threadIdx.x - 64, nthr = int(blockDim.x) - 64;
    if (splits == 1) {
      // ================= stage this N tile's epilogue vectors (static data) in smem
      const float* ga = D.epi.alpha;
      const float* gb = D.epi.beta;
      for (int i = ti; i < bn; i += nthr) {
        const int c = co_base + i;
        if (ga) s_alpha[i] = c < cout ? ga[c] : 0.f;
        if (gb) s_beta[i] = c < cout ? gb[c] : 0.f;
      }
      if (D.dw_k > 0) {
        // depthwise epilogue: this CTA's taps [k*k][bn] and BN vectors, after the ring
        float* s_dw = reinterpret_cast<float*>(slots + nslots * slot_bytes);
        const int kk = D.dw_k * D.dw_k;
        for (int i = ti; i < kk * bn; i += nthr) {
          const int tap = i / bn, c = co_base + (i - tap * bn);
          s_dw[i] = c < cout ? D.dw_w[tap * cout + c] : 0.f;
        }
        for (int i = ti; i < bn; i += nthr) {
          const int c = co_base + i;
          s_dw[kk * bn + i] = (D.dw_alpha && c < cout) ? D.dw_alpha[c] : 1.f;
          s_dw[kk * bn + bn + i] = (D.dw_beta && c < cout) ? D.dw_beta[c] : 0.f;
        }
        if (D.se != nullptr && ti == 0) {
          // fused SE: this CTA's rows of fc1^T and fc2 ([bn][Cr] each; split: hi then lo)
          // are static -- bulk copies issued now land while the main loop runs
          // (dfx_epi.cuh se_finish waits on ready[1]); rows are contiguous and 16-B
          // multiples (host-checked: cout % 8 == 0, cr even)
          const dfx_se_fuse& F = *D.se;
          const int Cr = F.cr;
          const int64_t cc = int64_t(F.c) * Cr;
          const uint32_t bytes = uint32_t(min(bn, F.c - co_base)) * Cr * 2;
          uint8_t* dst = reinterpret_cast<uint8_t*>(s_dw + (kk + 2) * bn);
          mbar_arrive_expect_tx(&hdr->ready[1], bytes * 2 * planes);
          for (int mat = 0; mat < 2 * planes; ++mat) {
            const uint16_t* src = reinterpret_cast<const uint16_t*>(mat & 1 ? F.w2 : F.w1) +
                                  (mat >> 1) * cc + int64_t(co_base) * Cr;
            bulk_load(dst + int64_t(mat) * bn * Cr * 2, src, bytes, &hdr->ready[1]);
          }
        }
      }
    }
    if constexpr (!kSplitT<T>) if (D.pre_mode) {
      // ================= A prologue transform: rewrite each landed A stage in smem
      griddep_wait();                                  // the gate vector is a predecessor's output
      int it = 0;
      for (int st = st_begin; st < st_end; ++st, ++it) {
        const int slot = it % nslots;
        if (ti == 0) mbar_wait(&hdr->full[slot], (it / nslots) & 1);
        named_bar_sync(1, nthr);
        pre_transform_stage<T>(slots + slot * slot_bytes, min(kpack, ksteps - st * kpack), cb, st * kpack, D,
                               n0h[0], tp * tq, ti, nthr);
        fence_proxy_async_smem();
        named_bar_sync(1, nthr);
        if (ti == 0) mbar_arrive(&hdr->ready[slot]);
      }
    }
  }
  __syncwarp();

  // ================= epilogue: TMEM -> registers -> 16-bit NHWC (or fp32 split-K partials)
  dfx_epilogue e = D.epi;
  if (splits == 1) {                          // read the smem copies (offset by the tile base)
    if (e.alpha) e.alpha = s_alpha - co_base;
    if (e.beta) e.beta = s_beta - co_base;
  }
  const dfx_view o = D.out;
  const int P = D.p, Q = D.q, N = D.n;
  float* const ws = D.ws;
  const int ldw = D.nt * bn;

  griddep_wait();                              // residual / output buffers of predecessors
  // ONE thread polls the accumulator barrier; the rest park in bar.sync.  (All 128
  // threads spinning on try_wait measurably slowed the producer's TMA issue and
  // the mbarrier transaction updates of the stages still in flight.)
  if (threadIdx.x == 32) mbar_wait(&hdr->accum, 0);
  __syncthreads();                             // accumulator complete, epilogue vectors visible
  if (threadIdx.x == 0) DFX_TL(5);             // accumulator complete
  tc_fence_after();
  if (!(L.flags & 16)) griddep_launch();       // successor may start its prologue now

  const int row = threadIdx.x & 127;           // tile row == TMEM lane (warps w, w+4 share it)
  const int qi = row % tq;
  const int pi_ = (row / tq) % tp;
  const int ni = row / (tq * tp);
  const uint32_t lane_addr = tmem_base + (uint32_t((warp & 3) * 32) << 16);
  const int ncols = min(bn, ((cout - co_base) + 15) & ~15);
  const bool views_vec = vec8_ok(o, 0) && (e.binop == DFX_BIN_NONE || vec8_ok(e.other, 0));

  const int64_t plane = int64_t(N) * P * Q * ldw;      // one split's partials
  if (threadIdx.x == 0) DFX_TL(11);                    // epilogue starts
  if (csplit) {
    // ---- cluster split-K: every rank parks its fp32 partial tile in its own smem
    // (the operand slots are free once the accumulator barrier fired), then rank r
    // reduces rows [r*R/S, (r+1)*R/S) over all ranks IN RANK ORDER through DSMEM
    // (deterministic, same order as splitk_kernel) and runs the epilogue on them.
    // No fp32 workspace round trip through L2 and no second launch.
    float* red = reinterpret_cast<float*>(slots);
    const int rp = bn + 4;                               // row pitch (floats), conflict-free
    const int c_step = 16 * int(blockDim.x >> 7);
    for (int c0 = 16 * (warp >> 2); c0 < ncols; c0 += c_step) {
      uint32_t r[16];
      tmem_ld16_issue(lane_addr + uint32_t(c0), r);
      tmem_ld_wait(r);
      if constexpr (planes == 2) {               // + the A_hi * B_lo column half
        uint32_t q[16];
        tmem_ld16_issue(lane_addr + uint32_t(bn + c0), q);
        tmem_ld_wait(q);
#pragma unroll
        for (int k = 0; k < 16; ++k) r[k] = __float_as_uint(__uint_as_float(r[k]) + __uint_as_float(q[k]));
      }
      float4* dst = reinterpret_cast<float4*>(red + row * rp + c0);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        dst[k] = make_float4(__uint_as_float(r[4 * k]), __uint_as_float(r[4 * k + 1]),
                             __uint_as_float(r[4 * k + 2]), __uint_as_float(r[4 * k + 3]));
    }
    cluster_sync_all();
    const int R = tn * tp * tq;
    const int rows_per = (R + splits - 1) / splits;
    const int r0 = split * rows_per, r1 = min(R, r0 + rows_per);
    const int c8n = ncols / 8;
    for (int item = threadIdx.x; item < (r1 - r0) * c8n; item += int(blockDim.x)) {
      const int rr = r0 + item / c8n;
      const int cc = (item - (rr - r0) * c8n) * 8;
      const int co = co_base + cc;
      const int on = n0h[0] + rr / (tq * tp), op = p0h[0] + (rr / tq) % tp, oq = q0h[0] + rr % tq;
      if (on >= N || op >= P || oq >= Q || co >= cout) continue;
      const float* src = red + rr * rp + cc;
      float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int sr = 0; sr < splits; ++sr) {
        const float4 a = dsmem_ld4(src, uint32_t(sr)), b = dsmem_ld4(src + 4, uint32_t(sr));
        v[0] += a.x; v[1] += a.y; v[2] += a.z; v[3] += a.w;
        v[4] += b.x; v[5] += b.y; v[6] += b.z; v[7] += b.w;
      }
      const int64_t pix = (int64_t(on) * P + op) * Q + oq;
      if (views_vec && co + 8 <= cout) {
        epilogue8<T>(e, v, pix, on, co);
        stv8<T>(o, view_pixel_index(o, pix, co), v);
      } else {
        float tail[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) tail[k] = v[k];
        epilogue_store_tail<T>(e, o, tail, pix, on, co, min(8, cout - co));
      }
    }
    cluster_sync_all();                                  // peers done reading this smem
    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc(tmem_base, tmem_cols);
    return;
  }

  if (D.dw_k > 0) {
    if (threadIdx.x == 0) DFX_TL(48);                  // depthwise-epilogue drain starts
    // ---- depthwise epilogue: this CTA covers every M tile (host-checked), so the
    // drain parks its channels of the whole output map in the (now free) operand
    // slots -- the same epilogue and 16-bit rounding as a global store, through a
    // view whose base is shared memory -- and the consumer depthwise conv runs on
    // it (dfx_epi.cuh dw_smem).  The expanded map never goes to HBM.
    T* xs = reinterpret_cast<T*>(slots);
    const int xp = bn + 8;                             // row pitch: 16 B pad against bank conflicts
    dfx_view sv = o;
    sv.base = xs;
    sv.n = N; sv.h = P; sv.w = Q; sv.c = bn;
    sv.pitch = xp * planes;                            // split: [hi | lo] per pixel
    sv.coff = -co_base;                                // absolute channel -> slot column
#pragma unroll
    for (int h = 0; h < 1 + M2; ++h) {
      if (h >= nhalf) break;
      const int on = n0h[h] + ni, op = p0h[h] + pi_, oq = q0h[h] + qi;
      const bool valid = row < tn * tp * tq && on < N && op < P && oq < Q;
      const int64_t pix = (int64_t(on) * P + op) * Q + oq;
      drain_rows_direct<T>(lane_addr + uint32_t(h * bn), ncols, pix, on, valid, co_base, cout, e, sv, true,
                           nullptr, ldw, 16 * (warp >> 2), 16 * int(blockDim.x >> 7), planes == 2 ? bn : 0);
    }
    tc_fence_before();
    const bool pair = !M2 && mt_total == 2;            // 2-CTA cluster: the peer holds the other rows
    if (pair) cluster_sync_all();
    else __syncthreads();                              // map complete; TMEM reads done
    if (warp == 2) tmem_dealloc(tmem_base, tmem_cols);
    // fused SE (D.se): the depthwise outputs + reduction scratch follow the map
    uint8_t* se_smem = D.se != nullptr
                           ? slots + ((size_t(N) * P * Q * xp * 2 * planes + 15) & ~size_t(15))
                           : nullptr;
    dw_smem<T>(D, xs, xp, N, P, Q, co_base, min(ncols, cout - co_base), o,
               reinterpret_cast<const float*>(slots + nslots * slot_bytes), bn, int(threadIdx.x),
               int(blockDim.x), se_smem, &hdr->ready[0]);   // ready[0]: partials gather, ready[1]: SE weights
    if (pair) cluster_sync_all();                      // the peer finished reading this map
    return;
  }

  // per-warp transpose staging for the coalesced drain: the operand slots are
  // free once the accumulator barrier fired (every TMA load was consumed)
  float* stg = reinterpret_cast<float*>(slots + warp * kEpiStageWarpBytes);
#pragma unroll
  for (int h = 0; h < 1 + M2; ++h) {                   // M tiles of this CTA (m2: two)
    if (h >= nhalf) break;
    const int on = n0h[h] + ni, op = p0h[h] + pi_, oq = q0h[h] + qi;
    const bool valid = row < tn * tp * tq && on < N && op < P && oq < Q;
    const int64_t pix = (int64_t(on) * P + op) * Q + oq;
    float* wsp = splits > 1 ? ws + split * plane : nullptr;
    if (kSplitT<T> || !(L.flags & 4))
      drain_rows_direct<T>(lane_addr + uint32_t(h * bn), ncols, pix, on, valid, co_base, cout, e, o,
                           views_vec, wsp, ldw, 16 * (warp >> 2), 16 * int(blockDim.x >> 7), planes == 2 ? bn : 0);
    else
      drain_rows<T>(lane_addr + uint32_t(h * bn), stg, ncols, pix, on, valid, co_base, cout, e, o,
                    views_vec, wsp, ldw, 16 * (warp >> 2), 16 * int(blockDim.x >> 7));
  }

  if (splits > 1 && D.counters != nullptr) {
    // ---- in-kernel split-K fixup (DFX_SPLITK=fixup): the last CTA to arrive for
    // this output tile sums all splits' partials in split order (deterministic),
    // applies the epilogue and resets the tile's counter for the next replay.
    const int tile_id = mi + mt_total * ntile;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0)
      hdr->last_split = atomicAdd(D.counters + tile_id, 1u) == uint32_t(splits - 1);
    __syncthreads();
    if (hdr->last_split) {
      __threadfence();
      const int c8n = ncols / 8;
      for (int item = threadIdx.x; item < 128 * c8n; item += int(blockDim.x)) {
        const int r = item / c8n;
        const int co = co_base + (item - r * c8n) * 8;
        const int rq = r % tq, rp = (r / tq) % tp, rn = r / (tq * tp);
        const int an = n0h[0] + rn, ap = p0h[0] + rp, aq = q0h[0] + rq;
        if (r >= tn * tp * tq || an >= N || ap >= P || aq >= Q || co >= cout) continue;
        const int64_t rpix = (int64_t(an) * P + ap) * Q + aq;
        const float4* src = reinterpret_cast<const float4*>(ws + rpix * ldw + co);
        const int64_t step = plane / 4;
        float4 a0 = __ldcg(src), a1 = __ldcg(src + 1);
        for (int s = 1; s < splits; ++s) {
          const float4 b0 = __ldcg(src + s * step), b1 = __ldcg(src + s * step + 1);
          a0.x += b0.x; a0.y += b0.y; a0.z += b0.z; a0.w += b0.w;
          a1.x += b1.x; a1.y += b1.y; a1.z += b1.z; a1.w += b1.w;
        }
        float v[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        if (views_vec && co + 8 <= cout) {
          epilogue8<T>(e, v, rpix, an, co);
          stv8<T>(o, view_pixel_index(o, rpix, co), v);
        } else {
          epilogue_store_tail<T>(e, o, v, rpix, an, co, min(8, cout - co));
        }
      }
      if (threadIdx.x == 0) D.counters[tile_id] = 0u;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) DFX_TL(6);             // epilogue stored
#ifdef DFX_TIMELINE
  if (threadIdx.x == 0 && blockIdx.x == 0) dfx_timeline[41] = clock64();
#endif
  if (warp == 2) tmem_dealloc(tmem_base, tmem_cols);
}

// Deterministic split-K reduction (splits summed in ascending order) + epilogue.
template <typename T>
__global__ void splitk_kernel(const __grid_constant__ dfx_splitk_params P) {
  griddep_wait();
  griddep_launch();
  const int cgroups = (P.cout + 7) / 8;
  const int64_t total = int64_t(P.pixels) * cgroups;
  const int hw = P.out.h * P.out.w;
  const int64_t plane = int64_t(P.pixels) * P.ldw;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t pix = idx / cgroups;
    const int c = int(idx - pix * cgroups) * 8;
    const int n = int(pix / hw);
    float v[8];
    const float* src = P.ws + pix * P.ldw + c;
    {
      const float4 a = *reinterpret_cast<const float4*>(src);
      const float4 b = *reinterpret_cast<const float4*>(src + 4);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    }
    for (int s = 1; s < P.splits; ++s) {
      const float* p = src + s * plane;
      const float4 a = *reinterpret_cast<const float4*>(p);
      const float4 b = *reinterpret_cast<const float4*>(p + 4);
      v[0] += a.x; v[1] += a.y; v[2] += a.z; v[3] += a.w; v[4] += b.x; v[5] += b.y; v[6] += b.z; v[7] += b.w;
    }
    const bool vec = c + 8 <= P.cout && vec8_ok(P.out, c) &&
                     (P.epi.binop == DFX_BIN_NONE || vec8_ok(P.epi.other, c));
    if (vec) {
      epilogue8<T>(P.epi, v, pix, n, c);
      stv8<T>(P.out, view_pixel_index(P.out, pix, c), v);
    } else {
      epilogue_store_tail<T>(P.epi, P.out, v, pix, n, c, min(8, P.cout - c));
    }
  }
}

template __global__ void gemm_kernel<__nv_bfloat16, 0>(const __grid_constant__ dfx_gemm_launch);
template __global__ void gemm_kernel<__half, 0>(const __grid_constant__ dfx_gemm_launch);
template __global__ void gemm_kernel<__nv_bfloat16, 1>(const __grid_constant__ dfx_gemm_launch);
template __global__ void gemm_kernel<__half, 1>(const __grid_constant__ dfx_gemm_launch);
template __global__ void splitk_kernel<__nv_bfloat16>(const __grid_constant__ dfx_splitk_params);
template __global__ void splitk_kernel<__half>(const __grid_constant__ dfx_splitk_params);
template __global__ void gemm_kernel<f16x2, 0>(const __grid_constant__ dfx_gemm_launch);
template __global__ void gemm_kernel<bf16x2, 0>(const __grid_constant__ dfx_gemm_launch);
template __global__ void splitk_kernel<f16x2>(const __grid_constant__ dfx_splitk_params);
template __global__ void splitk_kernel<bf16x2>(const __grid_constant__ dfx_splitk_params);

}  // namespace dfx
