// dfx_common.cuh — shared device helpers for libdfx (sm_100a only).
//
// Thin inline-PTX wrappers for mbarrier, TMA (cp.async.bulk.tensor), tcgen05
// (alloc / mma / commit / ld) and the bf16 + activation math every epilogue
// uses.  Encodings follow the PTX ISA for sm_100a; the UMMA shared-memory and
// instruction descriptor bit layouts match CUTLASS's cute/arch/mma_sm100_desc.hpp.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/dfx.h"

#define DFX_DEV __device__ __forceinline__

namespace dfx {

// ---------------------------------------------------------------- math
// Activations in fast-math form, each a handful of instructions: the GEMM
// epilogue drain is issue-bound, so instructions per output element set the
// speed of every multi-wave layer.  sigmoid(v) = 0.5 + 0.5 tanh(v / 2) and
// silu(v) = v sigmoid(v) use ONE MUFU.TANH (tanh.approx, ~2^-11 relative --
// the fp16 storage rounding that follows is of the same order, and the parity
// bar is 2e-2); no IEEE division anywhere (x / 6 and 1 / (1 + e) each
// compiled to a division subroutine).
DFX_DEV float tanh_approx(float x) {
  float r;
  asm("tanh.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// P (precise): the split-precision storage types (two 16-bit planes, ~22-bit
// significand) use forms accurate to a few fp32 ulp -- tanh.approx's 2^-11 would
// otherwise be the largest error left in the network.  __expf (ex2.approx) and
// __fdividef are within 2 ulp over the activations' range: 1e-7 relative, below
// the 2^-22 of the storage, at a fraction of the IEEE forms' instructions.
template <bool P = false> DFX_DEV float sigmoid_f(float v) {
  if constexpr (P) return __fdividef(1.0f, 1.0f + __expf(-v));
  else return fmaf(0.5f, tanh_approx(0.5f * v), 0.5f);
}
template <bool P = false> DFX_DEV float silu_f(float v) {
  if constexpr (P) return __fdividef(v, 1.0f + __expf(-v));
  else {
    const float h = 0.5f * v;
    return fmaf(h, tanh_approx(h), h);
  }
}
template <bool P = false> DFX_DEV float hsig_f(float v) {
  if constexpr (P) return __fdividef(fminf(fmaxf(v + 3.0f, 0.0f), 6.0f), 6.0f);
  else return fminf(fmaxf(v + 3.0f, 0.0f), 6.0f) * (1.0f / 6.0f);
}
DFX_DEV float gelu_f(float v) { return 0.5f * v * (1.0f + erff(v * 0.70710678118654752f)); }

template <bool P = false> DFX_DEV float act_apply(int act, float v) {
  switch (act) {
    case DFX_ACT_RELU: return fmaxf(v, 0.0f);
    case DFX_ACT_HARDSWISH: return v * hsig_f<P>(v);
    case DFX_ACT_HARDSIGMOID: return hsig_f<P>(v);
    case DFX_ACT_SILU: return silu_f<P>(v);
    case DFX_ACT_SIGMOID: return sigmoid_f<P>(v);
    case DFX_ACT_GELU: return gelu_f(v);
    default: return v;
  }
}

// Activation over 8 values with the switch hoisted out of the element loop.
template <bool P = false> DFX_DEV void act8(int act, float* v) {
  switch (act) {
    case DFX_ACT_RELU:
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = fmaxf(v[i], 0.0f);
      break;
    case DFX_ACT_HARDSWISH:
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = v[i] * hsig_f<P>(v[i]);
      break;
    case DFX_ACT_HARDSIGMOID:
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = hsig_f<P>(v[i]);
      break;
    case DFX_ACT_SILU:
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = silu_f<P>(v[i]);
      break;
    case DFX_ACT_SIGMOID:
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = sigmoid_f<P>(v[i]);
      break;
    case DFX_ACT_GELU:
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = gelu_f(v[i]);
      break;
    default:
      break;
  }
}

// ---------------------------------------------------------------- storage types
// Activations and GEMM operands are 16-bit: bf16 or IEEE half.  Half stores round
// to nearest WITHOUT saturation: a value beyond the fp16 range becomes +-inf (a
// split value hi + lo becomes NaN), propagates to the logits, and out_kernel counts
// it (dfx_nonfinite_count) -- an overflow is never a silently clamped, finite logit.
//
// Split precision (f16x2 / bf16x2, dtypes DFX_F16X2 / DFX_BF16X2): every value is
// stored as TWO 16-bit planes, x = hi + lo with hi = rn16(x), lo = rn16(x - hi),
// i.e. a 22-bit (fp16) or 16-bit (bf16) significand.  A view's pitch then spans
// both planes of a pixel: hi channel c at pix * pitch + coff + c, lo channel c
// pitch / 2 elements later.  GEMMs multiply three plane products on the tensor
// core (hi*hi + lo*hi + hi*lo, fp32 accumulation): the precision escape of
// SURVEY.md §7 hard part 2 that carries the fp32 reference's top-1 decisions.
// The 2-byte struct makes `T*` arithmetic address the hi plane.
struct f16x2 { unsigned short bits; };
struct bf16x2 { unsigned short bits; };

template <typename T> struct Elt;
template <> struct Elt<__nv_bfloat16> {
  static constexpr int kDtype = DFX_BF16;       // MMA operand type
  static constexpr bool kSplit = false;
  static DFX_DEV float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
  static DFX_DEV __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
  static DFX_DEV uint32_t pack2(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
  static DFX_DEV float2 unpack2(uint32_t u) {
    return __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u));
  }
};
template <> struct Elt<__half> {
  static constexpr int kDtype = DFX_F16;
  static constexpr bool kSplit = false;
  static DFX_DEV float to_f(__half v) { return __half2float(v); }
  static DFX_DEV __half from_f(float v) { return __float2half_rn(v); }
  static DFX_DEV uint32_t pack2(float a, float b) {   // one F2FP: a low, b high
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
    return r;
  }
  static DFX_DEV float2 unpack2(uint32_t u) { return __half22float2(*reinterpret_cast<__half2*>(&u)); }
};
// split types: the per-plane conversions are the 16-bit type's
template <> struct Elt<f16x2> : Elt<__half> {
  static constexpr bool kSplit = true;
  static DFX_DEV float to_f(f16x2 v) { return __half2float(__ushort_as_half(v.bits)); }
  static DFX_DEV f16x2 from_f(float v) { return f16x2{__half_as_ushort(Elt<__half>::from_f(v))}; }
};
template <> struct Elt<bf16x2> : Elt<__nv_bfloat16> {
  static constexpr bool kSplit = true;
  static DFX_DEV float to_f(bf16x2 v) { return __bfloat162float(__ushort_as_bfloat16(v.bits)); }
  static DFX_DEV bf16x2 from_f(float v) { return bf16x2{__bfloat16_as_ushort(__float2bfloat16_rn(v))}; }
};
template <typename T> constexpr bool kSplitT = Elt<T>::kSplit;

template <typename T> DFX_DEV void unpack8(const uint4& u, float* f) {
  float2 t;
  t = Elt<T>::unpack2(u.x); f[0] = t.x; f[1] = t.y;
  t = Elt<T>::unpack2(u.y); f[2] = t.x; f[3] = t.y;
  t = Elt<T>::unpack2(u.z); f[4] = t.x; f[5] = t.y;
  t = Elt<T>::unpack2(u.w); f[6] = t.x; f[7] = t.y;
}

template <typename T> DFX_DEV uint4 pack8(const float* f) {
  uint4 u;
  u.x = Elt<T>::pack2(f[0], f[1]);
  u.y = Elt<T>::pack2(f[2], f[3]);
  u.z = Elt<T>::pack2(f[4], f[5]);
  u.w = Elt<T>::pack2(f[6], f[7]);
  return u;
}

// split form: hi = rn16(f), lo = rn16(f - hi)
template <typename T> DFX_DEV void pack8_split(const float* f, uint4& hi, uint4& lo) {
  hi = pack8<T>(f);
  float h[8], r[8];
  unpack8<T>(hi, h);
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = f[i] - h[i];
  lo = pack8<T>(r);
}

// Loads / stores of activations.  `lo` is the element offset of the lo plane
// (lo_of(view)); ignored for single-plane types.
template <typename T> DFX_DEV int64_t lo_of(const dfx_view& v) {
  if constexpr (kSplitT<T>) return int64_t(v.pitch >> 1);
  else return 0;
}
template <typename T> DFX_DEV float ld1(const void* base, int64_t idx, int64_t lo) {
  const T* p = reinterpret_cast<const T*>(base);
  if constexpr (kSplitT<T>) return Elt<T>::to_f(p[idx]) + Elt<T>::to_f(p[idx + lo]);
  else return Elt<T>::to_f(p[idx]);
}
template <typename T> DFX_DEV void st1(void* base, int64_t idx, int64_t lo, float v) {
  T* p = reinterpret_cast<T*>(base);
  const T h = Elt<T>::from_f(v);
  p[idx] = h;
  if constexpr (kSplitT<T>) p[idx + lo] = Elt<T>::from_f(v - Elt<T>::to_f(h));
}
template <typename T> DFX_DEV void ld8(const void* base, int64_t idx, int64_t lo, float* f) {
  const T* p = reinterpret_cast<const T*>(base) + idx;
  unpack8<T>(*reinterpret_cast<const uint4*>(p), f);
  if constexpr (kSplitT<T>) {
    float l[8];
    unpack8<T>(*reinterpret_cast<const uint4*>(p + lo), l);
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] += l[i];
  }
}
template <typename T> DFX_DEV void st8(void* base, int64_t idx, int64_t lo, const float* f) {
  T* p = reinterpret_cast<T*>(base) + idx;
  if constexpr (kSplitT<T>) {
    uint4 h, l;
    pack8_split<T>(f, h, l);
    *reinterpret_cast<uint4*>(p) = h;
    *reinterpret_cast<uint4*>(p + lo) = l;
  } else {
    *reinterpret_cast<uint4*>(p) = pack8<T>(f);
  }
}
// view forms
template <typename T> DFX_DEV float ldv1(const dfx_view& v, int64_t idx) { return ld1<T>(v.base, idx, lo_of<T>(v)); }
template <typename T> DFX_DEV void stv1(const dfx_view& v, int64_t idx, float x) { st1<T>(v.base, idx, lo_of<T>(v), x); }
template <typename T> DFX_DEV void ldv8(const dfx_view& v, int64_t idx, float* f) { ld8<T>(v.base, idx, lo_of<T>(v), f); }
template <typename T> DFX_DEV void stv8(const dfx_view& v, int64_t idx, const float* f) { st8<T>(v.base, idx, lo_of<T>(v), f); }

DFX_DEV int64_t view_index(const dfx_view& v, int n, int h, int w, int c) {
  return ((int64_t(n) * v.h + h) * v.w + w) * v.pitch + v.coff + c;
}

DFX_DEV int64_t view_pixel_index(const dfx_view& v, int64_t pix, int c) {
  return pix * v.pitch + v.coff + c;
}

// Full epilogue on one value.  `pix` is the flat (n*h*w) pixel index and n the
// image index of the element; `c` its channel.
template <typename T>
DFX_DEV float epilogue(const dfx_epilogue& e, float x, int64_t pix, int n, int c) {
  float v = x;
  if (e.alpha) v = v * e.alpha[c];           // generic loads: alpha/beta may be staged in smem
  if (e.beta) v = v + e.beta[c];
  v = act_apply<kSplitT<T>>(e.act1, v);
  if (e.binop == DFX_BIN_ADD) {
    v += ldv1<T>(e.other, view_pixel_index(e.other, pix, c));
  } else if (e.binop == DFX_BIN_SCALE) {
    v *= ldv1<T>(e.other, int64_t(n) * e.other.pitch + e.other.coff + c);
  }
  return act_apply<kSplitT<T>>(e.act2, v);
}

// Vector form over 8 consecutive channels c..c+7 (caller guarantees alignment).
template <typename T>
DFX_DEV void epilogue8(const dfx_epilogue& e, float* v, int64_t pix, int n, int c) {
  if (e.alpha && e.beta) {                    // folded BN: one FFMA per element
    const float4 a0 = *reinterpret_cast<const float4*>(e.alpha + c);
    const float4 a1 = *reinterpret_cast<const float4*>(e.alpha + c + 4);
    const float4 b0 = *reinterpret_cast<const float4*>(e.beta + c);
    const float4 b1 = *reinterpret_cast<const float4*>(e.beta + c + 4);
    v[0] = fmaf(v[0], a0.x, b0.x); v[1] = fmaf(v[1], a0.y, b0.y);
    v[2] = fmaf(v[2], a0.z, b0.z); v[3] = fmaf(v[3], a0.w, b0.w);
    v[4] = fmaf(v[4], a1.x, b1.x); v[5] = fmaf(v[5], a1.y, b1.y);
    v[6] = fmaf(v[6], a1.z, b1.z); v[7] = fmaf(v[7], a1.w, b1.w);
  } else if (e.alpha) {
    const float4 a0 = *reinterpret_cast<const float4*>(e.alpha + c);
    const float4 a1 = *reinterpret_cast<const float4*>(e.alpha + c + 4);
    v[0] *= a0.x; v[1] *= a0.y; v[2] *= a0.z; v[3] *= a0.w;
    v[4] *= a1.x; v[5] *= a1.y; v[6] *= a1.z; v[7] *= a1.w;
  } else if (e.beta) {
    const float4 b0 = *reinterpret_cast<const float4*>(e.beta + c);
    const float4 b1 = *reinterpret_cast<const float4*>(e.beta + c + 4);
    v[0] += b0.x; v[1] += b0.y; v[2] += b0.z; v[3] += b0.w;
    v[4] += b1.x; v[5] += b1.y; v[6] += b1.z; v[7] += b1.w;
  }
  act8<kSplitT<T>>(e.act1, v);
  if (e.binop != DFX_BIN_NONE) {
    const int64_t idx = e.binop == DFX_BIN_ADD
                            ? view_pixel_index(e.other, pix, c)
                            : int64_t(n) * e.other.pitch + e.other.coff + c;
    float o[8];
    ldv8<T>(e.other, idx, o);
    if (e.binop == DFX_BIN_ADD) {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] += o[i];
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] *= o[i];
    }
  }
  act8<kSplitT<T>>(e.act2, v);
}

// Scalar epilogue + store of `count` (<= 16) consecutive channels starting at c.
// Out of line on purpose: it only serves ragged channel tails / unaligned
// concat offsets, and inlining it per column bloats every kernel's I-cache
// footprint (measured: stalled_no_instructions dominated small GEMMs).
template <typename T>
__device__ __noinline__ void epilogue_store_tail(const dfx_epilogue& e, const dfx_view& o,
                                                 const float* v, int64_t pix, int n, int c,
                                                 int count) {
  for (int i = 0; i < count; ++i)
    stv1<T>(o, view_pixel_index(o, pix, c + i), epilogue<T>(e, v[i], pix, n, c + i));
}

// True when 8-channel vector access at channel c is legal for view v.
DFX_DEV bool vec8_ok(const dfx_view& v, int c) { return ((v.coff + c) & 7) == 0; }

// ---------------------------------------------------------------- debug timeline
// DFX_TL(i): a %globaltimer probe.  dfx_gemm.cu defines it (and the probe array)
// when built with -DDFX_TIMELINE; everywhere else it compiles to nothing.
#ifndef DFX_TL
#define DFX_TL(i) \
  do {            \
  } while (0)
#endif

// ---------------------------------------------------------------- programmatic dependent launch
// Graph edges between libdfx kernels are programmatic: a kernel may start
// (prologue, TMEM/barrier setup, weight prefetch) while its predecessor
// finishes.  griddep_wait() blocks until the predecessor grid completed and
// its writes are visible -- every read of activations and every write must
// come after it.  griddep_launch() lets the successor start its prologue.
// Both are no-ops without a programmatic dependency (eager launches).
DFX_DEV void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
DFX_DEV void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// ---------------------------------------------------------------- PTX wrappers
DFX_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

DFX_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

DFX_DEV void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

DFX_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

DFX_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// try_wait suspends the thread until the phase completes or this many ns pass
// (the hardware wakes it on completion): waiting warps stop spinning through
// try_wait loops that steal issue slots from the drain warps on the same SMSP
// (ncu: 1.7 M loop iterations in one VGG16 batch-32 conv).
constexpr uint32_t kMbarSuspendNs = 100000;

// Blocks until the phase with the given parity completed.  A pipeline bug would
// otherwise hang the GPU; after ~2^26 polls the kernel traps instead.
DFX_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  for (uint32_t tries = 0;; ++tries) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(done)
        : "r"(addr), "r"(parity), "r"(kMbarSuspendNs)
        : "memory");
    if (done) return;
    if (tries > (1u << 24)) __trap();
  }
}

DFX_DEV void tma_load_4d(void* dst, const void* tmap, uint64_t* bar, int c0, int c1, int c2,
                         int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// 5-D box: the split-precision activation map (c, w, h, n, plane)
DFX_DEV void tma_load_5d(void* dst, const void* tmap, uint64_t* bar, int c0, int c1, int c2,
                         int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}

// 3-D box: split-precision weights (k, rows, plane) -> [hi rows | lo rows]
DFX_DEV void tma_load_3d(void* dst, const void* tmap, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

DFX_DEV void tma_load_2d(void* dst, const void* tmap, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// L2 policy for operands read once per query (batch-1 weights): evict_first, so
// streaming hundreds of MB of weights does not push the concurrent members'
// L2-resident activations out to HBM.
DFX_DEV uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

DFX_DEV void tma_load_2d_hint(void* dst, const void* tmap, uint64_t* bar, int c0, int c1, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(pol)
      : "memory");
}

DFX_DEV void tma_load_3d_hint(void* dst, const void* tmap, uint64_t* bar, int c0, int c1, int c2,
                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
      : "memory");
}

// weight (B) tile of one k-step; pol != 0: with that L2 policy
template <int planes>
DFX_DEV void tma_load_w(void* dst, const void* tmap, uint64_t* bar, int c0, int c1, uint64_t pol) {
  if constexpr (planes == 2) {      // one 3-D box: the k-step's hi rows, then its lo rows
    if (pol) tma_load_3d_hint(dst, tmap, bar, c0, c1, 0, pol);
    else tma_load_3d(dst, tmap, bar, c0, c1, 0);
  } else {
    if (pol) tma_load_2d_hint(dst, tmap, bar, c0, c1, pol);
    else tma_load_2d(dst, tmap, bar, c0, c1);
  }
}

// Non-tensor bulk copy global -> own CTA's shared memory (16-B aligned, size % 16 == 0).
DFX_DEV void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

DFX_DEV void tma_prefetch_desc(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}

// thread-block clusters / distributed shared memory ------------------------
DFX_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// all threads of all CTAs of the cluster; orders this CTA's shared-memory writes
// before every peer's subsequent DSMEM reads
DFX_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 16-B load from the same smem offset in CTA `rank` of this cluster
DFX_DEV float4 dsmem_ld4(const void* local, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local)), "r"(rank));
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(remote)
               : "memory");
  return v;
}

DFX_DEV uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
DFX_DEV float dsmem_ld1(const float* local, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local)), "r"(rank));
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote) : "memory");
  return v;
}

// tcgen05 -------------------------------------------------------------------
DFX_DEV void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

DFX_DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}

DFX_DEV void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
DFX_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T, bf16 inputs, fp32 accumulate.
DFX_DEV void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                       uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrive on an mbarrier when all previously issued tcgen05.mma complete.
DFX_DEV void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns per thread.
DFX_DEV void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Split form: issue the load, overlap other work, then wait.  The wait names the
// destination registers as read-write operands so the compiler cannot move any
// use of them above it.
DFX_DEV void tmem_ld16_issue(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
DFX_DEV void tmem_ld_wait(uint32_t (&r)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]),
                 "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]),
                 "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
               :
               : "memory");
}

// UMMA shared-memory descriptor, K-major operand with 32/64/128-byte swizzle.
// rows of `row_bytes` (= swizzle width), 8-row core groups stacked densely.
DFX_DEV uint64_t umma_smem_desc(uint32_t saddr, uint32_t row_bytes) {
  const uint64_t layout = row_bytes == 128 ? 2ull : (row_bytes == 64 ? 4ull : 6ull);
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);            // start address
  d |= uint64_t(1) << 16;                          // LBO (unused for swizzled K-major)
  d |= uint64_t(((8 * row_bytes) >> 4) & 0x3FFF) << 32;  // SBO: 8-row group stride
  d |= uint64_t(1) << 46;                          // version = 1 (sm_100)
  d |= layout << 61;                               // swizzle mode
  return d;
}

// Instruction descriptor: kind::f16, A=B=bf16 (dtype DFX_BF16) or f16, D=f32,
// both K-major, M=128.
DFX_DEV uint32_t umma_idesc_f16(uint32_t n, int dtype) {
  const uint32_t ab = dtype == DFX_BF16 ? 1u : 0u;
  uint32_t d = 0;
  d |= 1u << 4;               // D format f32
  d |= ab << 7;               // A format
  d |= ab << 10;              // B format
  d |= (n >> 3) << 17;        // N
  d |= (128u >> 4) << 24;     // M
  return d;
}

constexpr int kGemmThreads = 256;          // warps 0-3 roles + 4 more for the epilogue drain
constexpr int kMaxSlots = 8;                 // pipeline depth is a launch parameter, 2..8
constexpr int kStageABytes = 128 * 64 * 2;   // 128 rows x 64 16-bit
constexpr int kHeaderBytes = 1024;           // barriers + staged descriptor
constexpr int kEpiBytes = 2048;              // alpha[256] + beta[256] fp32, staged
constexpr int kSlotsOffset = kHeaderBytes + kEpiBytes;   // 1024-B aligned
constexpr int kPersistVecMax = 1024;         // persistent GEMM: epilogue vectors staged up to this cout

// one pipeline slot: A of 1 (or 2, m2) M tiles of 128 rows x 64 K, then B of bn rows x 64 K;
// split precision (`planes` 2): A hi tiles, A lo tiles, B hi, B lo
__host__ __device__ inline int gemm_slot_bytes(int bn_max, int m2 = 0, int planes = 1) {
  return (kStageABytes * (1 + m2) + bn_max * 128) * planes;
}
__host__ __device__ inline int gemm_smem_bytes(int bn_max, int nslots, int m2 = 0, int planes = 1) {
  return kSlotsOffset + nslots * gemm_slot_bytes(bn_max, m2, planes);
}
__host__ __device__ inline bool dtype_split(int dt) { return dt == DFX_F16X2 || dt == DFX_BF16X2; }
// ---- entry-conv im2col (dfx_bw.cu in_im2col_kernel): output pixels per CTA
constexpr int kIm2colTile = 256;           // a whole output row (<= 256 px) per CTA
constexpr int kIm2colMaxK = 2048;          // kh*kw*c of an im2col'ed entry conv
__host__ __device__ inline int im2col_smem_bytes(int c, int kh, int kw, int sw, int ow) {
  const int tw = ow < kIm2colTile ? ow : kIm2colTile;
  return c * kh * ((tw - 1) * sw + kw) * 4;
}
// ---- squeeze-excitation cluster kernel geometry (dfx_fused.cu)
constexpr int kSeThreads = 256;
constexpr int kSeMaxC = 4096;      // pooled channels held per CTA
constexpr int kSeMaxCr = 512;      // hidden units held per CTA
constexpr int kSeSmemBudget = 190 * 1024;
__host__ __device__ inline int se_chan_slice(int C, int cl) { return ((C + cl * 8 - 1) / (cl * 8)) * 8; }
__host__ __device__ inline int se_hid_slice(int Cr, int cl) { return (Cr + cl - 1) / cl; }
// dynamic smem of one CTA: its channel rows of fc1^T and of fc2 (16-bit, [rows][Cr])
// dynamic smem of a dwse_kernel CTA: (staged) FC slices + its 16-bit dw tile [HWo][slice]
__host__ __device__ inline int dwse_smem_bytes(int C, int Cr, int hwo, int staged) {
  const int cs = ((C + 16 * 8 - 1) / (16 * 8)) * 8;
  return (staged ? 2 * (((cs * Cr * 2) + 15) & ~15) : 0) + ((hwo * cs * 2 + 15) & ~15);
}
__host__ __device__ inline int se_smem_bytes(int C, int Cr, int cl) {
  return 2 * (((se_chan_slice(C, cl) * Cr * 2) + 15) & ~15);
}

__host__ __device__ inline uint32_t tmem_cols_for(int bn) {
  uint32_t c = 32;
  while (c < uint32_t(bn)) c <<= 1;
  return c;
}

// ---------------------------------------------------------------- attention geometry (dfx_vit.cu)
constexpr int kAttnD = 64;          // head dim
constexpr int kAttnQ = 64;          // query rows per CTA (4 warps x 16)
constexpr int kAttnKB = 64;         // keys per online-softmax block
constexpr int kAttnLd = kAttnD + 8; // smem row pitch (elements): conflict-free ldmatrix
constexpr int kAttnMaxL = 512;

__host__ __device__ constexpr int attn_smem_bytes(int L) {
  return (kAttnQ + 2 * ((L + kAttnKB - 1) / kAttnKB) * kAttnKB) * kAttnLd * 2;
}

}  // namespace dfx
