// dfx_vit.cu — the token kernels of the ViT-B/16 member of the 8-model config
// (SURVEY.md §8 KX "ViT: layernorm, GELU, attention"; there is no reference
// code for them, the semantics are torchvision's VisionTransformer and the
// CPU restatement is oracle/executor_ref.py tokens/layernorm/attention).
//
// Token tensors are NHWC views with h = 1, w = L tokens.  The linear layers of
// the encoder (qkv in-projection, out-projection, MLP) are 1x1 "convs" on
// those views and run on the tcgen05 GEMM (dfx_gemm.cu) with bias / GELU /
// residual-add in its epilogue; what is left is here:
//   ln_kernel      one warp per token row, two-pass mean / variance from
//                  registers, fp32 affine; optional "first out.w rows only"
//                  (layernorm -> select_token 0 reads 1 of 197 rows)
//   tokens_kernel  patch grid -> [class token; patches] + pos_embedding
//   attn_kernel    softmax(q k^T * scale) v per (image, head, 64-query tile),
//                  FlashAttention-2 style: K, V of the head staged in smem,
//                  mma.sync m16n8k16 (fp32 accumulate) with online softmax
//                  over 64-key blocks.  Attention is ~4% of ViT-B/16's FLOPs
//                  at 197 tokens; the warp-level MMA keeps it latency-bound
//                  but short.
#include "dfx_common.cuh"

namespace dfx {

// ------------------------------------------------------------------ layer norm
constexpr int kLnMaxVec = 4;        // in-register path: C <= 32 lanes * 4 * 8 = 1024

template <typename T>
__global__ void __launch_bounds__(256) ln_kernel(const __grid_constant__ dfx_ln_params P) {
  griddep_wait();
  griddep_launch();
  const dfx_view& in = P.in;
  const dfx_view& out = P.out;
  const int lane = threadIdx.x & 31;
  const int64_t row = int64_t(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
  const int64_t rows = int64_t(out.n) * out.w;
  if (row >= rows) return;
  const int img = int(row / out.w), t = int(row % out.w);
  const int C = in.c;
  const int64_t ib = view_index(in, img, 0, t, 0);
  const int64_t ob = view_index(out, img, 0, t, 0);
  const bool vec = (C & 7) == 0 && ((in.coff | out.coff) & 7) == 0 && C <= 32 * 8 * kLnMaxVec;
  if (vec) {
    float x[kLnMaxVec][8];
    const int nv = C / 8;
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < kLnMaxVec; ++k) {
      const int v = lane + 32 * k;
      if (v < nv) {
        ldv8<T>(in, ib + v * 8, x[k]);
#pragma unroll
        for (int i = 0; i < 8; ++i) s += x[k][i];
      }
    }
    if (!P.norm) {
#pragma unroll
      for (int k = 0; k < kLnMaxVec; ++k)
        if (lane + 32 * k < nv) stv8<T>(out, ob + (lane + 32 * k) * 8, x[k]);
      return;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mean = s / float(C);
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < kLnMaxVec; ++k)
      if (lane + 32 * k < nv) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float d = x[k][i] - mean;
          q = fmaf(d, d, q);
        }
      }
#pragma unroll
    for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    const float rstd = rsqrtf(q / float(C) + P.eps);
#pragma unroll
    for (int k = 0; k < kLnMaxVec; ++k) {
      const int v = lane + 32 * k;
      if (v < nv) {
        const float4 g0 = *reinterpret_cast<const float4*>(P.gamma + v * 8);
        const float4 g1 = *reinterpret_cast<const float4*>(P.gamma + v * 8 + 4);
        const float4 b0 = *reinterpret_cast<const float4*>(P.beta + v * 8);
        const float4 b1 = *reinterpret_cast<const float4*>(P.beta + v * 8 + 4);
        const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
        const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
        float y[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) y[i] = fmaf((x[k][i] - mean) * rstd, g[i], b[i]);
        stv8<T>(out, ob + v * 8, y);
      }
    }
    return;
  }
  // generic path (ragged C): two passes over global memory
  float s = 0.f;
  for (int c = lane; c < C; c += 32) s += ldv1<T>(in, ib + c);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mean = s / float(C);
  float q = 0.f;
  for (int c = lane; c < C; c += 32) {
    const float d = ldv1<T>(in, ib + c) - mean;
    q = fmaf(d, d, q);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float rstd = rsqrtf(q / float(C) + P.eps);
  for (int c = lane; c < C; c += 32) {
    const float x = ldv1<T>(in, ib + c);
    stv1<T>(out, ob + c, P.norm ? fmaf((x - mean) * rstd, P.gamma[c], P.beta[c]) : x);
  }
}

// ------------------------------------------------------------------ tokens
// One thread = 8 channels of one output token.
template <typename T>
__global__ void tokens_kernel(const __grid_constant__ dfx_tokens_params P) {
  griddep_wait();
  griddep_launch();
  const dfx_view& in = P.in;
  const dfx_view& out = P.out;
  const int C = out.c, cg = (C + 7) / 8;
  const int L = out.w, hw = in.h * in.w;
  const int64_t total = int64_t(out.n) * L * cg;
  const bool vec = ((C | in.coff | out.coff) & 7) == 0;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = idx / cg;
    const int c = int(idx - r * cg) * 8;
    const int img = int(r / L), t = int(r % L);
    const float* pos = P.pos + int64_t(t) * C;
    const int64_t o = view_index(out, img, 0, t, c);
    if (vec) {
      float x[8];
      if (t == 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = P.cls[c + i];
      } else {
        ldv8<T>(in, view_pixel_index(in, int64_t(img) * hw + t - 1, c), x);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] += pos[c + i];
      stv8<T>(out, o, x);
    } else {
      for (int i = 0; i < 8 && c + i < C; ++i) {
        const float x = t == 0 ? P.cls[c + i]
                               : ldv1<T>(in, view_pixel_index(in, int64_t(img) * hw + t - 1, c + i));
        stv1<T>(out, o + i, x + pos[c + i]);
      }
    }
  }
}

// ------------------------------------------------------------------ attention

template <typename T> struct Mma;
template <> struct Mma<__half> {
  static DFX_DEV void run(float* d, const uint32_t* a, const uint32_t* b) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
};
template <> struct Mma<__nv_bfloat16> {
  static DFX_DEV void run(float* d, const uint32_t* a, const uint32_t* b) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
};

DFX_DEV void ldsm_x4(uint32_t* r, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
DFX_DEV void ldsm_x4_t(uint32_t* r, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}

// grid (ceil(L / 64), heads, n), 128 threads.
template <typename T>
__global__ void __launch_bounds__(128) attn_kernel(const __grid_constant__ dfx_attn_params P) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  T* sq = reinterpret_cast<T*>(smem_raw);                  // [64][kAttnLd]
  const dfx_view& qkv = P.qkv;
  const dfx_view& out = P.out;
  const int L = qkv.w;
  const int Lp = (L + kAttnKB - 1) / kAttnKB * kAttnKB;
  T* sk = sq + kAttnQ * kAttnLd;                           // [Lp][kAttnLd]
  T* sv = sk + Lp * kAttnLd;                               // [Lp][kAttnLd]
  const int q0 = blockIdx.x * kAttnQ, head = blockIdx.y, img = blockIdx.z;
  const int C = out.c;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;

  griddep_wait();
  griddep_launch();
  // ---- stage Q tile, K and V of this head (16-B loads, zero rows past L)
  const int64_t rb = view_index(qkv, img, 0, 0, 0);
  for (int i = threadIdx.x; i < (kAttnQ + 2 * Lp) * 8; i += blockDim.x) {
    const int r = i / 8, c8 = (i % 8) * 8;
    int tok, col;
    T* dst;
    if (r < kAttnQ) {
      tok = q0 + r; col = head * kAttnD; dst = sq + r * kAttnLd;
    } else if (r < kAttnQ + Lp) {
      tok = r - kAttnQ; col = C + head * kAttnD; dst = sk + tok * kAttnLd;
    } else {
      tok = r - kAttnQ - Lp; col = 2 * C + head * kAttnD; dst = sv + tok * kAttnLd;
    }
    uint4 v = make_uint4(0, 0, 0, 0);
    if (tok < L)
      v = *reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(qkv.base) + rb +
                                          int64_t(tok) * qkv.pitch + col + c8);
    *reinterpret_cast<uint4*>(dst + c8) = v;
  }
  __syncthreads();

  // ---- Q fragments (A operand, 16 rows x 64) for this warp
  uint32_t qa[4][4];
  {
    const T* base = sq + (warp * 16 + (lane & 15)) * kAttnLd + (lane >> 4) * 8;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) ldsm_x4(qa[kk], base + kk * 16);
  }
  const float sl2 = P.scale * 1.4426950408889634f;         // softmax in base 2
  float o[8][4];
#pragma unroll
  for (int j = 0; j < 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;   // rows g and g + 8

  for (int kb = 0; kb < Lp; kb += kAttnKB) {
    // S = Q K^T over 64 keys: 8 n-tiles of 8 keys
    float s[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int j2 = 0; j2 < 4; ++j2) {              // pairs of key n-tiles (16 keys)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {            // head-dim k steps of 16
        // x4: matrices (keys 0-7, d 0-7), (keys 0-7, d 8-15), (keys 8-15, d 0-7), (keys 8-15, d 8-15)
        uint32_t b[4];
        const int key = kb + j2 * 16 + (lane & 7) + ((lane >> 4) << 3);
        const int d = kk * 16 + ((lane >> 3) & 1) * 8;
        ldsm_x4(b, sk + key * kAttnLd + d);
        Mma<T>::run(s[2 * j2], qa[kk], b);
        Mma<T>::run(s[2 * j2 + 1], qa[kk], b + 2);
      }
    }
    // mask keys >= L, online softmax (rows g = lane/4 and g + 8; quad-reduced)
    float bm0 = -INFINITY, bm1 = -INFINITY;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int key = kb + j * 8 + (lane & 3) * 2;
      if (key >= L) s[j][0] = s[j][2] = -INFINITY;
      if (key + 1 >= L) s[j][1] = s[j][3] = -INFINITY;
      bm0 = fmaxf(bm0, fmaxf(s[j][0], s[j][1]));
      bm1 = fmaxf(bm1, fmaxf(s[j][2], s[j][3]));
    }
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
      bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, off));
      bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, off));
    }
    const float nm0 = fmaxf(m0, bm0), nm1 = fmaxf(m1, bm1);
    const float c0 = exp2f((m0 - nm0) * sl2), c1 = exp2f((m1 - nm1) * sl2);
    m0 = nm0; m1 = nm1;
    float rs0 = 0.f, rs1 = 0.f;
    uint32_t pa[4][4];                            // P as A fragments (16 x 64 keys)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float p0 = exp2f((s[j][0] - m0) * sl2), p1 = exp2f((s[j][1] - m0) * sl2);
      const float p2 = exp2f((s[j][2] - m1) * sl2), p3 = exp2f((s[j][3] - m1) * sl2);
      rs0 += p0 + p1;
      rs1 += p2 + p3;
      pa[j / 2][(j & 1) * 2 + 0] = Elt<T>::pack2(p0, p1);
      pa[j / 2][(j & 1) * 2 + 1] = Elt<T>::pack2(p2, p3);
    }
    l0 = l0 * c0 + rs0;
    l1 = l1 * c1 + rs1;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      o[j][0] *= c0; o[j][1] *= c0; o[j][2] *= c1; o[j][3] *= c1;
    }
    // O += P V: k = 64 keys (4 steps of 16), n = 64 head dims (8 tiles)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
      for (int j2 = 0; j2 < 4; ++j2) {            // pairs of d n-tiles
        // x4.trans: (keys 0-7, d 0-7), (keys 8-15, d 0-7), (keys 0-7, d 8-15), (keys 8-15, d 8-15)
        uint32_t b[4];
        const int key = kb + kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int d = j2 * 16 + (lane >> 4) * 8;
        ldsm_x4_t(b, sv + key * kAttnLd + d);
        Mma<T>::run(o[2 * j2], pa[kk], b);
        Mma<T>::run(o[2 * j2 + 1], pa[kk], b + 2);
      }
    }
  }
  // ---- normalise and store (rows g, g + 8 of this warp's 16)
#pragma unroll
  for (int off = 1; off <= 2; off <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, off);
    l1 += __shfl_xor_sync(0xffffffffu, l1, off);
  }
  const float il0 = 1.f / l0, il1 = 1.f / l1;
  const int r0 = q0 + warp * 16 + (lane >> 2), r1 = r0 + 8;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int col = head * kAttnD + j * 8 + (lane & 3) * 2;
    T* ob = reinterpret_cast<T*>(out.base);
    if (r0 < L)
      *reinterpret_cast<uint32_t*>(ob + view_index(out, img, 0, r0, col)) =
          Elt<T>::pack2(o[j][0] * il0, o[j][1] * il0);
    if (r1 < L)
      *reinterpret_cast<uint32_t*>(ob + view_index(out, img, 0, r1, col)) =
          Elt<T>::pack2(o[j][2] * il1, o[j][3] * il1);
  }
}

#define DFX_VIT_INST(T)                                                                \
  template __global__ void ln_kernel<T>(const __grid_constant__ dfx_ln_params);        \
  template __global__ void tokens_kernel<T>(const __grid_constant__ dfx_tokens_params); \
  template __global__ void attn_kernel<T>(const __grid_constant__ dfx_attn_params);
DFX_VIT_INST(__nv_bfloat16)
DFX_VIT_INST(__half)
#undef DFX_VIT_INST

}  // namespace dfx
