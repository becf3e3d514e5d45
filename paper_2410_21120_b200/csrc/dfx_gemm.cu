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
// MMA issuer, warp 2 = TMEM allocator; all four warps run the epilogue
// (warp w owns TMEM lanes 32w..32w+31 = tile rows).
#include "dfx_common.cuh"

namespace dfx {

struct GemmHeader {
  uint64_t full[kSlots];
  uint64_t empty[kSlots];
  uint64_t accum;
  uint32_t tmem_base;
};

template <typename T>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_kernel(const __grid_constant__ dfx_gemm_launch L) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // Dynamic smem base is only guaranteed 16-B aligned: round up to 1024 for swizzles.
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  GemmHeader* hdr = reinterpret_cast<GemmHeader*>(smem);
  uint8_t* slots = smem + kHeaderBytes;
  const int slot_bytes = gemm_slot_bytes(L.bn_max);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int bid = blockIdx.x;

  int pi = 0;
  for (int i = 1; i < L.ndesc; ++i)
    if (L.descs[i].tile_begin <= bid) pi = i;
  const dfx_gemm_desc* d = L.descs + pi;

  // ---- tile coordinates (M tiles fastest, then K splits, then N tiles)
  int t = bid - d->tile_begin;
  const int mt_total = d->mt_n * d->mt_p * d->mt_q;
  const int mi = t % mt_total;
  t /= mt_total;
  const int split = t % d->splits;
  const int ntile = t / d->splits;
  const int mq = mi % d->mt_q;
  const int mp = (mi / d->mt_q) % d->mt_p;
  const int mn = mi / (d->mt_q * d->mt_p);
  const int n0 = mn * d->tn, p0 = mp * d->tp, q0 = mq * d->tq;
  const int bn = d->bn, cb = d->cb, kpack = d->kpack, ksteps = d->ksteps;
  const int st_begin = split * d->stages_per_split;
  const int st_end = min(d->stages, st_begin + d->stages_per_split);
  const uint32_t tmem_cols = tmem_cols_for(L.bn_max);

  if (threadIdx.x == 0) {
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(&hdr->full[i], 1);
      mbar_init(&hdr->empty[i], 1);
    }
    mbar_init(&hdr->accum, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(&hdr->tmem_base, tmem_cols);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(d->tmap_a);
    tma_prefetch_desc(d->tmap_b);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = hdr->tmem_base;

  const int sub_a = 128 * cb * 2;     // bytes of one K-step A sub-tile
  const int sub_b = bn * cb * 2;      // bytes of one K-step B sub-tile
  const uint32_t box_a_bytes = uint32_t(cb) * 2u * d->tq * d->tp * d->tn;

  if (warp == 0 && lane == 0) {
    // ================= TMA producer
    int it = 0;
    for (int st = st_begin; st < st_end; ++st, ++it) {
      const int slot = it % kSlots;
      const uint32_t par = (it / kSlots) & 1;
      mbar_wait(&hdr->empty[slot], par ^ 1);
      uint8_t* a_dst = slots + slot * slot_bytes;
      uint8_t* b_dst = a_dst + kStageABytes;
      const int k0 = st * kpack;
      const int nk = min(kpack, ksteps - k0);
      mbar_arrive_expect_tx(&hdr->full[slot], nk * (box_a_bytes + uint32_t(sub_b)));
      for (int j = 0; j < nk; ++j) {
        const int kstep = k0 + j;
        const int rs = kstep / d->cblocks;
        const int cblk = kstep - rs * d->cblocks;
        const int r = rs / d->s;
        const int s = rs - r * d->s;
        tma_load_4d(a_dst + j * sub_a, d->tmap_a, &hdr->full[slot], cblk * cb,
                    q0 * d->stride_w + s - d->pad_w, p0 * d->stride_h + r - d->pad_h, n0);
        tma_load_2d(b_dst + j * sub_b, d->tmap_b, &hdr->full[slot], kstep * cb, ntile * bn);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ================= MMA issuer
    const uint32_t idesc = umma_idesc_f16(uint32_t(bn), Elt<T>::kDtype);
    const uint32_t row_bytes = uint32_t(cb) * 2u;
    uint32_t accumulate = 0;
    int it = 0;
    for (int st = st_begin; st < st_end; ++st, ++it) {
      const int slot = it % kSlots;
      const uint32_t par = (it / kSlots) & 1;
      mbar_wait(&hdr->full[slot], par);
      tc_fence_after();
      const uint32_t a_base = smem_u32(slots + slot * slot_bytes);
      const uint32_t b_base = a_base + kStageABytes;
      const int nk = min(kpack, ksteps - st * kpack);
      for (int j = 0; j < nk; ++j) {
        for (int kk = 0; kk < cb / 16; ++kk) {
          const uint64_t ad = umma_smem_desc(a_base + j * sub_a + kk * 32, row_bytes);
          const uint64_t bd = umma_smem_desc(b_base + j * sub_b + kk * 32, row_bytes);
          umma_f16(tmem_base, ad, bd, idesc, accumulate);
          accumulate = 1;
        }
      }
      umma_commit(&hdr->empty[slot]);
    }
    umma_commit(&hdr->accum);
  }
  __syncwarp();

  // ================= epilogue: TMEM -> registers -> 16-bit NHWC (or fp32 split-K partials)
  mbar_wait(&hdr->accum, 0);
  tc_fence_after();

  const int row = threadIdx.x;                 // tile row == TMEM lane
  const int qi = row % d->tq;
  const int pi_ = (row / d->tq) % d->tp;
  const int ni = row / (d->tq * d->tp);
  const int on = n0 + ni, op = p0 + pi_, oq = q0 + qi;
  const bool valid = row < d->tn * d->tp * d->tq && on < d->n && op < d->p && oq < d->q;
  const int64_t pix = (int64_t(on) * d->p + op) * d->q + oq;
  const uint32_t lane_addr = tmem_base + (uint32_t(warp * 32) << 16);
  const int co_base = ntile * bn;
  const int ncols = min(bn, ((d->cout - co_base) + 15) & ~15);

  for (int c0 = 0; c0 < ncols; c0 += 16) {
    float v[16];
    tmem_ld16(lane_addr + uint32_t(c0), v);
    if (!valid) continue;
    const int co = co_base + c0;
    if (d->splits > 1) {
      const int ldw = d->nt * bn;
      float4* dst = reinterpret_cast<float4*>(
          d->ws + (int64_t(split) * d->n * d->p * d->q + pix) * ldw + co);
#pragma unroll
      for (int i = 0; i < 4; ++i) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      continue;
    }
    const dfx_epilogue& e = d->epi;
    const dfx_view& o = d->out;
    const bool vec = co + 16 <= d->cout && vec8_ok(o, co) &&
                     (e.binop == DFX_BIN_NONE || vec8_ok(e.other, co));
    if (vec) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        epilogue8<T>(e, v + 8 * h, pix, on, co + 8 * h);
        st8<T>(o.base, view_pixel_index(o, pix, co + 8 * h), v + 8 * h);
      }
    } else {
      for (int i = 0; i < 16 && co + i < d->cout; ++i)
        st1<T>(o.base, view_pixel_index(o, pix, co + i), epilogue<T>(e, v[i], pix, on, co + i));
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem_base, tmem_cols);
}

// Deterministic split-K reduction (splits summed in ascending order) + epilogue.
template <typename T>
__global__ void splitk_kernel(const __grid_constant__ dfx_splitk_params P) {
  const int cgroups = (P.cout + 7) / 8;
  const int64_t total = int64_t(P.pixels) * cgroups;
  const int hw = P.out.h * P.out.w;
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
      const float* p = src + int64_t(s) * P.pixels * P.ldw;
      const float4 a = *reinterpret_cast<const float4*>(p);
      const float4 b = *reinterpret_cast<const float4*>(p + 4);
      v[0] += a.x; v[1] += a.y; v[2] += a.z; v[3] += a.w; v[4] += b.x; v[5] += b.y; v[6] += b.z; v[7] += b.w;
    }
    const bool vec = c + 8 <= P.cout && vec8_ok(P.out, c) &&
                     (P.epi.binop == DFX_BIN_NONE || vec8_ok(P.epi.other, c));
    if (vec) {
      epilogue8<T>(P.epi, v, pix, n, c);
      st8<T>(P.out.base, view_pixel_index(P.out, pix, c), v);
    } else {
      for (int i = 0; i < 8 && c + i < P.cout; ++i)
        st1<T>(P.out.base, view_pixel_index(P.out, pix, c + i), epilogue<T>(P.epi, v[i], pix, n, c + i));
    }
  }
}

template __global__ void gemm_kernel<__nv_bfloat16>(const __grid_constant__ dfx_gemm_launch);
template __global__ void gemm_kernel<__half>(const __grid_constant__ dfx_gemm_launch);
template __global__ void splitk_kernel<__nv_bfloat16>(const __grid_constant__ dfx_splitk_params);
template __global__ void splitk_kernel<__half>(const __grid_constant__ dfx_splitk_params);

}  // namespace dfx
