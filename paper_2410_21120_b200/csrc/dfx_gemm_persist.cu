// dfx_gemm_persist.cu — persistent variant of the tcgen05 implicit-GEMM conv
// (dfx_gemm.cu) for multi-wave layers (batch >= 8: tens to thousands of
// 128 x bn output tiles).
//
// The one-tile-per-CTA kernel pays per tile: the prologue (descriptor staging,
// barrier init, TMEM alloc), the pipeline fill, and an epilogue that the
// tensor core sits idle through.  Here a grid of <= 2 CTAs per SM walks the
// tile list (M fastest, so concurrently running CTAs share each weight tile in
// L2) and overlaps everything:
//   warp 0  lane 0: TMA producer -- one smem slot ring across ALL of the CTA's
//                   tiles, so the next tile's first stages load while the
//                   current tile's MMAs and the previous tile's epilogue run;
//   warp 1  lane 0: MMA issuer -- a ring of nacc = min(8, 512 / bn) TMEM
//                   accumulators; tile i accumulates into buffer i % nacc once
//                   the epilogue of tile i - nacc released it (acc_empty);
//   warps 2..     : epilogue -- one or two groups of 4 warps (two when the SM
//                   holds one CTA, bn > 64); warp w drains TMEM lanes
//                   32*(w%4)..+31 (the lane quadrant a warp may access) with
//                   coalesced stores (dfx_epi.cuh), then releases the buffer.
//                   The drain is issue-bound: more warps and a deep ring keep
//                   it off the MMA's critical path.
// Split-K never applies (multi-wave layers have enough tiles), so every tile
// finishes in its own epilogue.  Same descriptor (dfx_gemm_desc) and numerics
// as gemm_kernel: K order, fp32 accumulation, epilogue slots.
#include "dfx_common.cuh"
#include "dfx_epi.cuh"

namespace dfx {

constexpr int kPersistThreads = 320;      // producer, MMA, 8 epilogue warps
constexpr int kMaxAcc = 8;                // TMEM accumulator buffers (as many as 512 columns hold)

struct PersistHeader {
  uint64_t full[kMaxSlots];
  uint64_t empty[kMaxSlots];
  uint64_t acc_full[kMaxAcc];
  uint64_t acc_empty[kMaxAcc];
  uint64_t ready[kMaxSlots];     // pre_mode: A stage transformed in smem
  uint32_t tmem_base;
  uint32_t _pad[7];
  dfx_gemm_desc desc;
};
static_assert(sizeof(PersistHeader) <= kHeaderBytes + kEpiBytes, "persistent gemm header overflow");

template <typename T>
__global__ void __launch_bounds__(kPersistThreads, 1)
    gemm_persist_kernel(const __grid_constant__ dfx_gemm_launch L) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  PersistHeader* hdr = reinterpret_cast<PersistHeader*>(smem);
  uint8_t* slots = smem + kSlotsOffset;
  constexpr int planes = kSplitT<T> ? 2 : 1;       // split precision: hi + lo operand tiles
  const int slot_bytes = gemm_slot_bytes(L.bn_max, 0, planes);
  const int a_lo_off = kStageABytes, b_off = kStageABytes * planes;
  // split precision: B sub-tile of k-step j = [hi bn rows | lo bn rows] (lo at (2j + 1)
  // sub_b); "wide" (bn <= 128): A_hi * [B_hi; B_lo] as ONE N = 2 bn MMA into a
  // 2 bn-column accumulator, + A_lo * B_hi into its first half (dfx_gemm.cu)
  const bool wide = planes == 2 && L.bn_max <= 128;
  const int accw = wide ? 2 : 1;                   // accumulator width in units of bn
  const int nslots = L.nslots;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const dfx_gemm_desc* gd = &L.desc0;

  if (threadIdx.x < sizeof(dfx_gemm_desc) / 16)
    reinterpret_cast<uint4*>(&hdr->desc)[threadIdx.x] = reinterpret_cast<const uint4*>(gd)[threadIdx.x];
  // epilogue groups of 4 warps (blockDim = 64 + 128 * groups): with a deep
  // accumulator ring the groups take alternate tiles, else they split each
  // tile's columns (with 2 buffers a tile's drain must finish within one tile).
  // One group = two CTAs per SM: each may hold only half of TMEM (a second
  // CTA's tcgen05.alloc would otherwise block until the first one exits).
  const int groups = (int(blockDim.x) - 64) >> 7;
  const int nacc = max(2, min(kMaxAcc, (groups > 1 ? 512 : 256) / (L.bn_max * accw)));
  // pre_mode (A prologue transform): group 1 transforms A stages, group 0 drains
  const bool pre = !kSplitT<T> && L.desc0.pre_mode != 0;
  const bool alt = groups > 1 && nacc >= 4 && !pre;
  const uint32_t tmem_cols = tmem_cols_for(nacc * L.bn_max * accw);
  if (threadIdx.x == 0) {
    for (int i = 0; i < nslots; ++i) {
      mbar_init(&hdr->full[i], 1);
      mbar_init(&hdr->empty[i], 1);
      mbar_init(&hdr->ready[i], 1);
    }
    for (int b = 0; b < nacc; ++b) {
      mbar_init(&hdr->acc_full[b], 1);
      mbar_init(&hdr->acc_empty[b], (alt || pre) ? 128 : blockDim.x - 64);
    }
    fence_barrier_init();
    tma_prefetch_desc(gd->tmap_a);
    tma_prefetch_desc(gd->tmap_b);
  }
  if (warp == 1) tmem_alloc(&hdr->tmem_base, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = hdr->tmem_base;
  const dfx_gemm_desc& D = hdr->desc;

  const int mt_q = D.mt_q, mt_p = D.mt_p;
  const int tn = D.tn, tp = D.tp, tq = D.tq;
  const int mt_total = D.mt_n * mt_p * mt_q;
  const int total = D.tiles;
  const int bn = D.bn, cb = D.cb, kpack = D.kpack, ksteps = D.ksteps, stages = D.stages;
  const int sub_a = 128 * cb * 2, sub_b = bn * cb * 2;
  const int grid = gridDim.x;

  if (warp == 0) {
    if (lane == 0) {
      // ================= TMA producer: one slot ring across all tiles of this CTA
      const int cblocks = D.cblocks, S = D.s;
      const uint32_t box_a_bytes = uint32_t(cb) * 2u * tq * tp * tn;
      const int cout = D.cout;
      const void* tma = gd->tmap_a;
      const void* tmb = gd->tmap_b;
      // slot / phase and the k-step cursor (channel block, s, r) advance
      // incrementally: this ONE thread feeds the MMA, and per-k-step integer
      // divisions made its issue loop the bottleneck of short-K layers
      int slot = 0, filled = 0;
      uint32_t par = 0;
      bool waited = false;
      for (int tile = blockIdx.x; tile < total; tile += grid) {
        const int mi = tile % mt_total, ntile = tile / mt_total;
        const int n0 = (mi / (mt_q * mt_p)) * tn, p0 = ((mi / mt_q) % mt_p) * tp, q0 = (mi % mt_q) * tq;
        const int qbase = q0 * D.stride_w - D.pad_w, pbase = p0 * D.stride_h - D.pad_h;
        const int co_base = ntile * bn;
        int cblk = 0, sc = 0, rc = 0;
        for (int st = 0, k0 = 0; st < stages; ++st, k0 += kpack) {
          if (filled >= nslots) mbar_wait(&hdr->empty[slot], par ^ 1);
          uint8_t* a_dst = slots + slot * slot_bytes;
          uint8_t* b_dst = a_dst + b_off;
          const int nk = min(kpack, ksteps - k0);
          mbar_arrive_expect_tx(&hdr->full[slot], nk * (box_a_bytes + uint32_t(sub_b)) * planes);
          for (int j = 0; j < nk; ++j) {                // weights: static, before the dependency
            if constexpr (planes == 2)          // hi rows then lo rows, one 3-D box
              tma_load_3d(b_dst + 2 * j * sub_b, tmb, &hdr->full[slot], (k0 + j) * cb, co_base, 0);
            else
              tma_load_2d(b_dst + j * sub_b, tmb, &hdr->full[slot], (k0 + j) * cb, co_base);
          }
          if (!waited) {
            griddep_wait();
            waited = true;
          }
          for (int j = 0; j < nk; ++j) {
            if constexpr (planes == 2) {
              tma_load_5d(a_dst + j * sub_a, tma, &hdr->full[slot], cblk * cb, qbase + sc, pbase + rc, n0, 0);
              tma_load_5d(a_dst + a_lo_off + j * sub_a, tma, &hdr->full[slot], cblk * cb, qbase + sc, pbase + rc,
                          n0, 1);
            } else {
              tma_load_4d(a_dst + j * sub_a, tma, &hdr->full[slot], cblk * cb, qbase + sc, pbase + rc, n0);
            }
            if (++cblk == cblocks) {
              cblk = 0;
              if (++sc == S) {
                sc = 0;
                ++rc;
              }
            }
          }
          ++filled;
          if (++slot == nslots) {
            slot = 0;
            par ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ================= MMA issuer: nacc TMEM accumulators in a ring
      const uint32_t idesc = umma_idesc_f16(uint32_t(bn), Elt<T>::kDtype);
      const uint32_t idesc2 = umma_idesc_f16(uint32_t(accw * bn), Elt<T>::kDtype);
      const uint32_t row_bytes = uint32_t(cb) * 2u;
      const int kk_n = cb / 16;
      int lt = 0, slot = 0, b = 0;
      uint32_t par = 0, apar = 0;
      uint64_t* const gate = pre ? hdr->ready : hdr->full;
      for (int tile = blockIdx.x; tile < total; tile += grid, ++lt) {
        if (lt >= nacc) mbar_wait(&hdr->acc_empty[b], apar ^ 1);
        tc_fence_after();
        const uint32_t acc = tmem_base + uint32_t(b * accw * bn);
        uint32_t accumulate = 0;
        for (int st = 0; st < stages; ++st) {
          mbar_wait(&gate[slot], par);
          tc_fence_after();
          const uint32_t a_base = smem_u32(slots + slot * slot_bytes);
          const uint32_t b_base = a_base + b_off;
          const int nk = min(kpack, ksteps - st * kpack);
          for (int j = 0; j < nk; ++j)
            for (int kk = 0; kk < kk_n; ++kk) {
              const uint64_t ad = umma_smem_desc(a_base + j * sub_a + kk * 32, row_bytes);
              const uint64_t bd = umma_smem_desc(b_base + j * planes * sub_b + kk * 32, row_bytes);
              if constexpr (planes == 2) {
                if (wide) {                        // [0, bn) hi*hi, [bn, 2 bn) hi*lo
                  umma_f16(acc, ad, bd, idesc2, accumulate);
                } else {                           // + hi(A) lo(B) into the same columns
                  umma_f16(acc, ad, bd, idesc, accumulate);
                  umma_f16(acc, ad, umma_smem_desc(b_base + (2 * j + 1) * sub_b + kk * 32, row_bytes), idesc, 1u);
                }
                umma_f16(acc, umma_smem_desc(a_base + a_lo_off + j * sub_a + kk * 32, row_bytes), bd, idesc, 1u);
              } else {
                umma_f16(acc, ad, bd, idesc, accumulate);
              }
              accumulate = 1;
            }
          umma_commit(&hdr->empty[slot]);
          if (++slot == nslots) {
            slot = 0;
            par ^= 1u;
          }
        }
        umma_commit(&hdr->acc_full[b]);
        if (++b == nacc) {
          b = 0;
          apar ^= 1u;
        }
      }
    }
  } else {
    // ================= epilogue warps 2..9: TMEM lane quadrant (warp % 4)
    // the folded-BN / bias vectors (static) staged in smem before the dependency: the
    // drain's per-chunk vector loads were its long-scoreboard stalls from L1/L2
    dfx_epilogue e = D.epi;
    if (D.cout <= kPersistVecMax && (e.alpha || e.beta)) {
      float* s_vec = reinterpret_cast<float*>(slots + nslots * slot_bytes +
                                              ((L.flags & 4) ? 8 * kEpiStageWarpBytes : 0));
      const int cp = (D.cout + 15) & ~15, ti = int(threadIdx.x) - 64, ne = int(blockDim.x) - 64;
      for (int i = ti; i < cp; i += ne) {
        if (e.alpha) s_vec[i] = i < D.cout ? e.alpha[i] : 0.f;
        if (e.beta) s_vec[cp + i] = i < D.cout ? e.beta[i] : 0.f;
      }
      named_bar_sync(2, ne);
      if (e.alpha) e.alpha = s_vec;
      if (e.beta) e.beta = s_vec + cp;
    }
    griddep_wait();                                   // residual operands / output of predecessors
    const int quad = warp & 3;
    const int row = quad * 32 + lane;                 // tile row == TMEM lane
    const int qi = row % tq, pi_ = (row / tq) % tp, ni = row / (tq * tp);
    const dfx_view o = D.out;
    const int P = D.p, Q = D.q, N = D.n, cout = D.cout;
    const bool views_vec = vec8_ok(o, 0) && (e.binop == DFX_BIN_NONE || vec8_ok(e.other, 0));
    const uint32_t lane_addr = tmem_base + (uint32_t(quad * 32) << 16);
    float* stg = reinterpret_cast<float*>(slots + nslots * slot_bytes + (warp - 2) * kEpiStageWarpBytes);
    const int group = (warp - 2) >> 2;
    const int c_first = (alt || pre) ? 0 : 16 * group, c_step = (alt || pre) ? 16 : 16 * groups;
    if (pre && group == 1) {
      // ================= A prologue transform over every stage of every tile of this CTA
      if constexpr (!kSplitT<T>) {
      const int ti = threadIdx.x - 64 - 128;
      int it = 0;
      for (int tile = blockIdx.x; tile < total; tile += grid) {
        const int mi = tile % mt_total;
        const int n0 = (mi / (mt_q * mt_p)) * tn;
        for (int st = 0; st < stages; ++st, ++it) {
          const int slot = it % nslots;
          if (ti == 0) mbar_wait(&hdr->full[slot], (it / nslots) & 1);
          named_bar_sync(1, 128);
          pre_transform_stage<T>(slots + slot * slot_bytes, min(kpack, ksteps - st * kpack), cb, st * kpack, D,
                                 n0, tp * tq, ti, 128);
          fence_proxy_async_smem();
          named_bar_sync(1, 128);
          if (ti == 0) mbar_arrive(&hdr->ready[slot]);
        }
      }
      }
    } else {
    // tile coordinates advance as a mixed-radix counter (q, p, n, N tile) by `grid`
    // per step, the accumulator ring index and phase likewise: the per-tile integer
    // divisions were a quarter of the drain's instructions on narrow (bn = 64) layers
    const int mt_n = D.mt_n;
    int cq, cp, cn, cnt;
    int dq, dp, dn, dnt;
    {
      int t = blockIdx.x;
      cq = t % mt_q; t /= mt_q; cp = t % mt_p; t /= mt_p; cn = t % mt_n; cnt = t / mt_n;
      t = grid;
      dq = t % mt_q; t /= mt_q; dp = t % mt_p; t /= mt_p; dn = t % mt_n; dnt = t / mt_n;
    }
    int lt = 0, b = 0;
    uint32_t aph = 0;
    for (int tile = blockIdx.x; tile < total; tile += grid, ++lt) {
      const int n0 = cn * tn, p0 = cp * tp, q0 = cq * tq;
      const int co_base = cnt * bn;
      const int bcur = b;
      const uint32_t phcur = aph;
      {                                               // advance to this CTA's next tile
        int c = 0;
        cq += dq; if (cq >= mt_q) { cq -= mt_q; c = 1; }
        cp += dp + c; c = 0; if (cp >= mt_p) { cp -= mt_p; c = 1; }
        cn += dn + c; c = 0; if (cn >= mt_n) { cn -= mt_n; c = 1; }
        cnt += dnt + c;
        if (++b == nacc) { b = 0; aph ^= 1u; }
      }
      if (alt && (lt & 1) != group) continue;
      const int on = n0 + ni, op = p0 + pi_, oq = q0 + qi;
      const bool valid = row < tn * tp * tq && on < N && op < P && oq < Q;
      const int64_t pix = (int64_t(on) * P + op) * Q + oq;
      const int ncols = min(bn, ((cout - co_base) + 15) & ~15);
      if (tile + grid >= total) griddep_launch();     // this CTA's last tile
      mbar_wait(&hdr->acc_full[bcur], phcur);
      tc_fence_after();
      if (kSplitT<T> || !(L.flags & 4))
        drain_rows_direct<T>(lane_addr + uint32_t(bcur * accw * bn), ncols, pix, on, valid, co_base, cout, e, o,
                             views_vec, nullptr, 0, c_first, c_step, wide ? bn : 0);
      else
        drain_rows<T>(lane_addr + uint32_t(bcur * bn), stg, ncols, pix, on, valid, co_base, cout, e, o,
                      views_vec, nullptr, 0, c_first, c_step);
      tc_fence_before();
      mbar_arrive(&hdr->acc_empty[bcur]);             // buffer may be overwritten
    }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem_base, tmem_cols);
}

template __global__ void gemm_persist_kernel<__nv_bfloat16>(const __grid_constant__ dfx_gemm_launch);
template __global__ void gemm_persist_kernel<__half>(const __grid_constant__ dfx_gemm_launch);
template __global__ void gemm_persist_kernel<f16x2>(const __grid_constant__ dfx_gemm_launch);
template __global__ void gemm_persist_kernel<bf16x2>(const __grid_constant__ dfx_gemm_launch);

}  // namespace dfx
