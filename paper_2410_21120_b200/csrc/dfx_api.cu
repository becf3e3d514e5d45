// dfx_api.cu — the C ABI of libdfx (declared in include/dfx.h).
//
// Memory, streams, TMA descriptor encoding, kernel dispatch, and the CUDA
// graph that executes a whole fused DAG.  Host-side only; kernels live in
// dfx_gemm.cu and dfx_bw.cu.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX3: ranges cost nothing without a tool attached

#include "dfx_common.cuh"
#include "dfx_dw.cuh"
#include "dfx_epi.cuh"

namespace dfx {
template <typename T, int M2> __global__ void gemm_kernel(const __grid_constant__ dfx_gemm_launch L);
template <typename T> __global__ void gemm_persist_kernel(const __grid_constant__ dfx_gemm_launch L);
template <typename T> __global__ void splitk_kernel(const __grid_constant__ dfx_splitk_params P);
template <typename T> __global__ void ew_kernel(const __grid_constant__ dfx_ew_params P);
template <typename T, int ACT1> __global__ void ew_vec_kernel(const __grid_constant__ dfx_ew_params P);
template <typename T> __global__ void dwconv_kernel(const __grid_constant__ dfx_dwconv_params P);
template <typename T, int K, int S, int QV, int ACT>
__global__ void dwconv_tile_kernel(const __grid_constant__ dfx_dwconv_params P);
template <typename T, int S, int ACT>
__global__ void dwconv_col_kernel(const __grid_constant__ dfx_dwconv_params P);
template <typename T> __global__ void pool_kernel(const __grid_constant__ dfx_pool_params P);
template <typename T> __global__ void gap_kernel(const __grid_constant__ dfx_gap_params P);
template <typename T> __global__ void in_kernel(const __grid_constant__ dfx_in_params P);
template <typename T> __global__ void in_im2col_kernel(const __grid_constant__ dfx_in_params P);
template <typename T> __global__ void out_kernel(const __grid_constant__ dfx_out_params P);
__global__ void gate_kernel(const __grid_constant__ dfx_gate_params P);
template <typename T, int CL, int IPI> __global__ void se_kernel(const __grid_constant__ dfx_se_params P);
template <typename T> __global__ void dwse_kernel(const __grid_constant__ dfx_dwse_params P);
template <typename T> __global__ void ln_kernel(const __grid_constant__ dfx_ln_params P);
template <typename T> __global__ void tokens_kernel(const __grid_constant__ dfx_tokens_params P);
template <typename T> __global__ void attn_kernel(const __grid_constant__ dfx_attn_params P);
}  // namespace dfx

// kernel instantiation for a storage dtype (DFX_F16 / DFX_BF16 / DFX_F16X2 / DFX_BF16X2)
#define DFX_PICK(K, dt)                                                              \
  ((dt) == DFX_F16      ? reinterpret_cast<const void*>(&dfx::K<__half>)           \
   : (dt) == DFX_BF16   ? reinterpret_cast<const void*>(&dfx::K<__nv_bfloat16>)    \
   : (dt) == DFX_F16X2  ? reinterpret_cast<const void*>(&dfx::K<dfx::f16x2>)       \
                        : reinterpret_cast<const void*>(&dfx::K<dfx::bf16x2>))
// kernels without a split-precision instantiation (ViT, fused dw+SE): 16-bit only
#define DFX_PICK16(K, dt) \
  ((dt) == DFX_F16 ? reinterpret_cast<const void*>(&dfx::K<__half>) \
                   : reinterpret_cast<const void*>(&dfx::K<__nv_bfloat16>))

namespace {
// NVTX range for the lifetime of a scope (host side of the ABI entry points)
struct NvtxRange {
  explicit NvtxRange(const char* m) { nvtxRangePushA(m); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

namespace {

const void* gemm_func(int dt, int m2) {
  if (dt == DFX_F16X2) return reinterpret_cast<const void*>(&dfx::gemm_kernel<dfx::f16x2, 0>);
  if (dt == DFX_BF16X2) return reinterpret_cast<const void*>(&dfx::gemm_kernel<dfx::bf16x2, 0>);
  if (m2)
    return dt == DFX_F16 ? reinterpret_cast<const void*>(&dfx::gemm_kernel<__half, 1>)
                         : reinterpret_cast<const void*>(&dfx::gemm_kernel<__nv_bfloat16, 1>);
  return dt == DFX_F16 ? reinterpret_cast<const void*>(&dfx::gemm_kernel<__half, 0>)
                       : reinterpret_cast<const void*>(&dfx::gemm_kernel<__nv_bfloat16, 0>);
}

const void* se_func(int dt, int cl, int ipi = 1) {
  if (dt == DFX_F16X2)
    return ipi == 4 ? reinterpret_cast<const void*>(&dfx::se_kernel<dfx::f16x2, 16, 4>)
                    : reinterpret_cast<const void*>(&dfx::se_kernel<dfx::f16x2, 16, 1>);
  if (dt == DFX_BF16X2)
    return ipi == 4 ? reinterpret_cast<const void*>(&dfx::se_kernel<dfx::bf16x2, 16, 4>)
                    : reinterpret_cast<const void*>(&dfx::se_kernel<dfx::bf16x2, 16, 1>);
  if (ipi == 4)
    return dt == DFX_F16 ? reinterpret_cast<const void*>(&dfx::se_kernel<__half, 16, 4>)
                         : reinterpret_cast<const void*>(&dfx::se_kernel<__nv_bfloat16, 16, 4>);
  if (cl == 16)
    return dt == DFX_F16 ? reinterpret_cast<const void*>(&dfx::se_kernel<__half, 16, 1>)
                         : reinterpret_cast<const void*>(&dfx::se_kernel<__nv_bfloat16, 16, 1>);
  return dt == DFX_F16 ? reinterpret_cast<const void*>(&dfx::se_kernel<__half, 8, 1>)
                       : reinterpret_cast<const void*>(&dfx::se_kernel<__nv_bfloat16, 8, 1>);
}

template <typename T, int A>
const void* dwconv_col_func_a(int s) {
  return s == 1 ? reinterpret_cast<const void*>(&dfx::dwconv_col_kernel<T, 1, A>)
                : reinterpret_cast<const void*>(&dfx::dwconv_col_kernel<T, 2, A>);
}
template <typename T>
const void* dwconv_col_func_t(int s, int act) {
  switch (act) {
    case DFX_ACT_RELU: return dwconv_col_func_a<T, DFX_ACT_RELU>(s);
    case DFX_ACT_HARDSWISH: return dwconv_col_func_a<T, DFX_ACT_HARDSWISH>(s);
    case DFX_ACT_SILU: return dwconv_col_func_a<T, DFX_ACT_SILU>(s);
    default: return dwconv_col_func_a<T, DFX_ACT_NONE>(s);
  }
}
const void* dwconv_col_func(int dt, int s, int act) {
  switch (dt) {
    case DFX_F16: return dwconv_col_func_t<__half>(s, act);
    case DFX_BF16: return dwconv_col_func_t<__nv_bfloat16>(s, act);
    case DFX_F16X2: return dwconv_col_func_t<dfx::f16x2>(s, act);
    case DFX_BF16X2: return dwconv_col_func_t<dfx::bf16x2>(s, act);
    default: return nullptr;
  }
}
// column-strip depthwise kernel for 3x3 layers (dfx_dw.cu); DFX_DW_COL=0: the tile
// kernel everywhere (A/B)
int dw_col_waves() {            // DFX_DW_COL_WAVES: grid size target of the strip split (A/B)
  static const int w = [] {
    const char* e = std::getenv("DFX_DW_COL_WAVES");
    return e ? std::max(1, std::atoi(e)) : 2;
  }();
  return w;
}
bool dw_col_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DFX_DW_COL");
    return !(e && e[0] == '0');
  }();
  return on;
}
template <typename T, int A>
const void* dwconv_tile_func_a(int k, int s, int qv) {
#define DFX_DW_CASE(K, S)                                                                    \
  if (k == K && s == S)                                                                      \
    return qv == 4 ? reinterpret_cast<const void*>(&dfx::dwconv_tile_kernel<T, K, S, 4, A>)  \
         : qv == 2 ? reinterpret_cast<const void*>(&dfx::dwconv_tile_kernel<T, K, S, 2, A>)  \
                   : reinterpret_cast<const void*>(&dfx::dwconv_tile_kernel<T, K, S, 1, A>);
  DFX_DW_CASE(3, 1)
  DFX_DW_CASE(3, 2)
  DFX_DW_CASE(5, 1)
  DFX_DW_CASE(5, 2)
#undef DFX_DW_CASE
  return nullptr;
}
// the epilogue's first activation is a template parameter (the switch per 8 outputs
// was a large share of the kernel's instructions); other activations take NONE's
// instantiation, whose epilogue falls back to the generic switch
template <typename T>
const void* dwconv_tile_func_t(int k, int s, int qv, int act) {
  switch (act) {
    case DFX_ACT_RELU: return dwconv_tile_func_a<T, DFX_ACT_RELU>(k, s, qv);
    case DFX_ACT_HARDSWISH: return dwconv_tile_func_a<T, DFX_ACT_HARDSWISH>(k, s, qv);
    case DFX_ACT_SILU: return dwconv_tile_func_a<T, DFX_ACT_SILU>(k, s, qv);
    default: return dwconv_tile_func_a<T, DFX_ACT_NONE>(k, s, qv);
  }
}
template <typename T>
const void* ew_vec_func_t(int act) {
  switch (act) {
    case DFX_ACT_RELU: return reinterpret_cast<const void*>(&dfx::ew_vec_kernel<T, DFX_ACT_RELU>);
    case DFX_ACT_HARDSWISH: return reinterpret_cast<const void*>(&dfx::ew_vec_kernel<T, DFX_ACT_HARDSWISH>);
    case DFX_ACT_HARDSIGMOID: return reinterpret_cast<const void*>(&dfx::ew_vec_kernel<T, DFX_ACT_HARDSIGMOID>);
    case DFX_ACT_SILU: return reinterpret_cast<const void*>(&dfx::ew_vec_kernel<T, DFX_ACT_SILU>);
    case DFX_ACT_SIGMOID: return reinterpret_cast<const void*>(&dfx::ew_vec_kernel<T, DFX_ACT_SIGMOID>);
    case DFX_ACT_GELU: return reinterpret_cast<const void*>(&dfx::ew_vec_kernel<T, DFX_ACT_GELU>);
    default: return reinterpret_cast<const void*>(&dfx::ew_vec_kernel<T, DFX_ACT_NONE>);
  }
}
const void* ew_vec_func(int dt, int act) {
  switch (dt) {
    case DFX_F16: return ew_vec_func_t<__half>(act);
    case DFX_F16X2: return ew_vec_func_t<dfx::f16x2>(act);
    case DFX_BF16X2: return ew_vec_func_t<dfx::bf16x2>(act);
    default: return ew_vec_func_t<__nv_bfloat16>(act);
  }
}
const void* dwconv_tile_func(int dt, int k, int s, int qv, int act) {
  switch (dt) {
    case DFX_F16: return dwconv_tile_func_t<__half>(k, s, qv, act);
    case DFX_F16X2: return dwconv_tile_func_t<dfx::f16x2>(k, s, qv, act);
    case DFX_BF16X2: return dwconv_tile_func_t<dfx::bf16x2>(k, s, qv, act);
    default: return dwconv_tile_func_t<__nv_bfloat16>(k, s, qv, act);
  }
}

thread_local std::string g_err;
int g_sm_count = 148;
constexpr int kGemmSmemLimit = 227 * 1024;     // opt-in dynamic smem per CTA on sm_100
constexpr int kIm2colSmemLimit = kGemmSmemLimit - int(sizeof(int)) * dfx::kIm2colMaxK;  // - static table

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                       \
  do {                                                                                 \
    cudaError_t _e = (call);                                                           \
    if (_e != cudaSuccess)                                                             \
      return fail(DFX_E_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(_e), __FILE__, \
                  __LINE__);                                                           \
  } while (0)

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// --- cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn g_encode = nullptr;
std::once_flag g_encode_once;

int get_encode() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<EncodeTiledFn>(fn);
  });
  return g_encode ? DFX_OK : fail(DFX_E_CUDA, "cuTensorMapEncodeTiled unavailable");
}

CUtensorMapSwizzle swizzle_for(int cb) {
  return cb == 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                  : (cb == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
}

CUtensorMapDataType tmap_dtype(int dt) {
  return (dt == DFX_F16 || dt == DFX_F16X2) ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                            : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
}

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

unsigned elementwise_grid(int64_t threads, int block) {
  int64_t g = cdiv(threads, block);
  const int64_t cap = int64_t(g_sm_count) * 32;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return unsigned(g);
}

struct LaunchCfg {
  const void* func;
  dim3 grid, block;
  size_t smem;
  unsigned cluster = 1;          // thread-block cluster size along x (1 = none)
};

int config_for(int op, const void* params, size_t size, LaunchCfg* c) {
#define NEED(T)                                                                            \
  if (size != sizeof(T)) return fail(DFX_E_ARG, "op %d: params size %zu != %zu", op, size, \
                                     sizeof(T));
  c->block = dim3(256);
  c->smem = 0;
  switch (op) {
    case DFX_OP_GEMM: {
      NEED(dfx_gemm_launch);
      const auto* p = static_cast<const dfx_gemm_launch*>(params);
      if (p->bn_max < 16 || p->bn_max > 256 || p->total_tiles < 1)
        return fail(DFX_E_ARG, "gemm: bad bn_max %d / tiles %d", p->bn_max, p->total_tiles);
      const int planes = dfx::dtype_split(p->dtype) ? 2 : 1;
      if (planes == 2 && (p->m2 || p->desc0.pre_mode || (p->flags & 4)))
        return fail(DFX_E_UNSUPPORTED, "gemm: split precision without m2 / A transform / staged drain");
      if (p->dtype < DFX_BF16 || p->dtype > DFX_F16X2) return fail(DFX_E_ARG, "gemm: dtype %d", p->dtype);
      c->func = gemm_func(p->dtype, p->m2);
      c->grid = dim3(p->total_tiles);
      c->block = dim3(dfx::kGemmThreads);
      if (p->nslots < 2 || p->nslots > dfx::kMaxSlots)
        return fail(DFX_E_ARG, "gemm: nslots %d", p->nslots);
      if (p->m2 && p->bn_max > 256) return fail(DFX_E_ARG, "gemm: m2 with bn %d", p->bn_max);
      if (p->desc0.pre_mode && (p->m2 || p->ndesc != 1 || p->desc0.r != 1 || p->desc0.s != 1 ||
                                p->desc0.pad_h || p->desc0.pad_w))
        return fail(DFX_E_ARG, "gemm: A prologue transform needs one 1x1 unpadded problem, no m2");
      if (p->flags & 2) {               // persistent: one CTA per SM walks the tile list
        if (p->m2 || p->ndesc != 1 || p->desc0.splits != 1 || p->bn_max > 256)
          return fail(DFX_E_ARG, "gemm: persistent launch needs one problem, no m2 / split-K");
        c->func = DFX_PICK(gemm_persist_kernel, p->dtype);
        // narrow tiles (bn <= 64): two CTAs per SM with one epilogue group each (two
        // producers / MMA issuers per SM); else one CTA per SM with two groups
        // DFX_PERSIST_ONE_CTA_X2=1 (A/B): split precision keeps one CTA per SM with a
        // deeper ring (its slots are twice as large: 2 CTAs x 2 slots otherwise)
        static const bool one_x2 = getenv("DFX_PERSIST_ONE_CTA_X2") && atoi(getenv("DFX_PERSIST_ONE_CTA_X2")) == 1;
        const int per_sm = (p->bn_max <= 64 && !p->desc0.pre_mode && !(planes == 2 && one_x2)) ? 2 : 1;
        const int groups = 3 - per_sm;
        c->smem = dfx::gemm_smem_bytes(p->bn_max, p->nslots, 0, planes) + 1024 +
                  ((p->flags & 4) ? 8 * dfx::kEpiStageWarpBytes : 0) +
                  (p->desc0.cout <= dfx::kPersistVecMax ? 2 * ((p->desc0.cout + 15) & ~15) * 4 : 0);
        int64_t cap = int64_t(per_sm) * g_sm_count;
        if (p->max_ctas > 0) cap = std::min<int64_t>(cap, p->max_ctas);
        c->grid = dim3(unsigned(std::min<int64_t>(p->total_tiles, cap)));
        c->block = dim3(64 + 128 * groups);
      } else {
        c->smem = dfx::gemm_smem_bytes(p->bn_max, p->nslots, p->m2 ? 1 : 0, planes) + 1024;
        if (p->flags & 8) {             // cluster split-K: one cluster per output tile
          const int sp = p->desc0.splits;
          if (p->m2 || p->ndesc != 1 || sp < 2 || sp > 16 || p->total_tiles % sp)
            return fail(DFX_E_ARG, "gemm: cluster split-K needs one problem, no m2, 2..16 splits");
          if (size_t(128) * (p->bn_max + 4) * 4 > size_t(p->nslots) * dfx::gemm_slot_bytes(p->bn_max, 0, planes))
            return fail(DFX_E_ARG, "gemm: cluster split-K partial tile exceeds the %d slots", p->nslots);
          c->cluster = unsigned(sp);
        }
        // 8 warps (4 more drain the epilogue) when shared memory already limits the
        // SM to one CTA; else 4, so small-tile grids keep several CTAs per SM
        c->block = dim3((c->smem > size_t(114 * 1024) || p->desc0.pre_mode) ? dfx::kGemmThreads : 128);
        const dfx_gemm_desc& d0 = p->desc0;
        if (d0.dw_k > 0) {              // depthwise epilogue: one CTA holds the whole map
          const int mtt = d0.mt_n * d0.mt_p * d0.mt_q;
          const bool pair = !p->m2 && mtt == 2;         // one M tile per CTA of a 2-CTA cluster
          if (p->ndesc != 1 || (p->flags & 8) || d0.splits != 1 || (d0.dw_k != 3 && d0.dw_k != 5) ||
              (d0.dw_s != 1 && d0.dw_s != 2) || mtt > 2 || (pair && d0.mt_p != 2) || (d0.cout & 7))
            return fail(DFX_E_ARG, "gemm: depthwise epilogue needs one problem whose M tiles fit one CTA "
                                   "(or a 2-CTA cluster split along p)");
          if (pair) c->cluster = 2;
          size_t need = (size_t(d0.n) * d0.p * d0.q * (p->bn_max + 8) * 2 * planes + 15) & ~size_t(15);
          if (d0.se != nullptr && p->se_cr == 0) {   // SE squeeze only: the means' scratch
            if (p->m2 || d0.n > 2) return fail(DFX_E_ARG, "gemm: SE squeeze needs batch <= 2, no m2");
            need += (size_t(dfx::kGemmThreads) * 16 + 4 * size_t(p->bn_max)) * 4;
          } else if (d0.se != nullptr) {  // fused SE: depthwise-output tile + reduction scratch
            const int oh = d0.out.h, ow = d0.out.w, cr = p->se_cr;
            const int nt = d0.nt;
            if (p->m2 || d0.n > 2 || cr < 1 || cr > 512)
              return fail(DFX_E_ARG, "gemm: fused SE needs batch <= 2, no m2, 1 <= cr <= 512");
            need += ((size_t(d0.n) * oh * ow * p->bn_max * 2 * planes + 15) & ~size_t(15)) +
                    size_t(dfx::kGemmThreads) * 16 * 4 +
                    (4 * size_t(p->bn_max) + 2 * ((cr + 3) & ~3) + size_t(nt) * d0.n * cr + 4) * 4;
            c->smem += size_t(2) * planes * p->bn_max * cr * 2;       // staged fc1^T / fc2 rows
          }
          if (need > size_t(p->nslots) * dfx::gemm_slot_bytes(p->bn_max, p->m2 ? 1 : 0, planes))
            return fail(DFX_E_ARG, "gemm: depthwise epilogue map exceeds the %d slots", p->nslots);
          c->smem += size_t(d0.dw_k * d0.dw_k + 2) * p->bn_max * 4;   // taps + BN vectors
          c->block = dim3(dfx::kGemmThreads);
        }
      }
      if (c->smem > size_t(kGemmSmemLimit))
        return fail(DFX_E_ARG, "gemm: %zu B of shared memory (bn %d x %d slots)", c->smem,
                    p->bn_max, p->nslots);
      return DFX_OK;
    }
    case DFX_OP_SPLITK: {
      NEED(dfx_splitk_params);
      const auto* p = static_cast<const dfx_splitk_params*>(params);
      c->func = DFX_PICK(splitk_kernel, p->out.dtype);
      c->grid = dim3(elementwise_grid(int64_t(p->pixels) * cdiv(p->cout, 8), 256));
      return DFX_OK;
    }
    case DFX_OP_DWCONV: {
      NEED(dfx_dwconv_params);
      const auto* p = static_cast<const dfx_dwconv_params*>(params);
      const int k = p->kh, st = p->stride_h;
      const bool tiled = p->kh == p->kw && (k == 3 || k == 5) && p->stride_w == st &&
                         (st == 1 || st == 2) && (p->in.c & 7) == 0 &&
                         ((p->in.coff | p->out.coff | p->in.pitch) & 7) == 0 &&
                         int64_t(p->out.n) * p->out.h * p->out.w * p->in.c < (int64_t(1) << 34);
      if (tiled && k == 3 && dw_col_enabled()) {
        const int cg = p->in.c / 8;
        const int ns = dfx::dw_col_strips(p->out.n, p->out.h, p->out.w, cg, dw_col_waves());
        const int64_t items = int64_t(p->out.n) * p->out.w * cg;
        c->func = dwconv_col_func(p->in.dtype, st, p->epi.act1);
        c->grid = dim3(unsigned(cdiv(items, dfx::kDwColThreads)), unsigned(ns));
        c->block = dim3(dfx::kDwColThreads);
        return DFX_OK;
      }
      if (tiled) {
        // outputs per thread: as many as keep >= 2 waves of 256-thread blocks
        const int64_t rows = int64_t(p->out.n) * p->out.h * (p->in.c / 8);
        int qv = 4;
        while (qv > 1 && rows * cdiv(p->out.w, qv) < int64_t(2) * g_sm_count * 256) qv >>= 1;
        c->func = dwconv_tile_func(p->in.dtype, k, st, qv, p->epi.act1);
        c->grid = dim3(elementwise_grid(rows * cdiv(p->out.w, qv), 256));
        return DFX_OK;
      }
      c->func = DFX_PICK(dwconv_kernel, p->in.dtype);
      c->grid = dim3(elementwise_grid(int64_t(p->out.n) * p->out.h * p->out.w * cdiv(p->in.c, 8), 256));
      return DFX_OK;
    }
    case DFX_OP_POOL: {
      NEED(dfx_pool_params);
      const auto* p = static_cast<const dfx_pool_params*>(params);
      c->func = DFX_PICK(pool_kernel, p->in.dtype);
      c->grid = dim3(elementwise_grid(int64_t(p->out.n) * p->out.h * p->out.w * cdiv(p->in.c, 8), 256));
      return DFX_OK;
    }
    case DFX_OP_GAP: {
      NEED(dfx_gap_params);
      const auto* p = static_cast<const dfx_gap_params*>(params);
      c->func = DFX_PICK(gap_kernel, p->in.dtype);
      c->grid = dim3(unsigned(cdiv(p->in.c, 64)), unsigned(p->in.n));
      return DFX_OK;
    }
    case DFX_OP_EW: {
      NEED(dfx_ew_params);
      const auto* p = static_cast<const dfx_ew_params*>(params);
      const int64_t items = int64_t(p->in.n) * p->in.h * p->in.w * cdiv(p->in.c, 8);
      const bool vec = (p->in.c & 7) == 0 && items < (int64_t(1) << 31) &&
                       ((p->in.coff | p->out.coff | p->in.pitch | p->out.pitch |
                         (p->epi.binop ? (p->epi.other.coff | p->epi.other.pitch) : 0)) & 7) == 0;
      if (vec) {
        c->func = ew_vec_func(p->in.dtype, p->epi.act1);
        c->grid = dim3(elementwise_grid(cdiv(items, 2), 256));
        return DFX_OK;
      }
      c->func = DFX_PICK(ew_kernel, p->in.dtype);
      c->grid = dim3(elementwise_grid(items, 256));
      return DFX_OK;
    }
    case DFX_OP_IN: {
      NEED(dfx_in_params);
      const auto* p = static_cast<const dfx_in_params*>(params);
      if (p->out.pitch % 8 || p->out.coff) return fail(DFX_E_ARG, "in: pitch/coff");
      if (p->kh > 0) {
        const int kreal = p->kh * p->kw * p->c;
        if (p->split > 0 && dfx::dtype_split(p->out.dtype))
          return fail(DFX_E_ARG, "in: split stem with split-precision storage");
        const bool ok = p->split > 0 ? (p->split >= kreal && p->out.c == 3 * p->split && p->split <= dfx::kIm2colMaxK)
                                     : (p->out.c == kreal && p->out.c <= dfx::kIm2colMaxK);
        if (!ok) return fail(DFX_E_UNSUPPORTED, "in: im2col of %d channels (split %d)", p->out.c, p->split);
        c->func = DFX_PICK(in_im2col_kernel, p->out.dtype);
        c->grid = dim3(unsigned(cdiv(p->out.w, dfx::kIm2colTile)), unsigned(p->out.h), unsigned(p->out.n));
        c->block = dim3(256);
        c->smem = size_t(dfx::im2col_smem_bytes(p->c, p->kh, p->kw, p->sw, p->out.w));
        if (c->smem > size_t(kIm2colSmemLimit))
          return fail(DFX_E_UNSUPPORTED, "in: im2col window of %zu B", c->smem);
        return DFX_OK;
      }
      c->func = DFX_PICK(in_kernel, p->out.dtype);
      const int plane_pitch = dfx::dtype_split(p->out.dtype) ? p->out.pitch / 2 : p->out.pitch;
      c->grid = dim3(elementwise_grid(int64_t(p->out.n) * p->out.h * p->out.w * (plane_pitch / 8), 256));
      return DFX_OK;
    }
    case DFX_OP_OUT: {
      NEED(dfx_out_params);
      const auto* p = static_cast<const dfx_out_params*>(params);
      c->func = DFX_PICK(out_kernel, p->in.dtype);
      c->grid = dim3(elementwise_grid(int64_t(p->in.n) * p->in.h * p->in.w * p->in.c, 256));
      return DFX_OK;
    }
    case DFX_OP_SE: {
      NEED(dfx_se_params);
      const auto* p = static_cast<const dfx_se_params*>(params);
      if (p->in.c > 4096 || p->cr > 512 || p->cr < 1)
        return fail(DFX_E_UNSUPPORTED, "se: c=%d cr=%d beyond the cluster kernel's limits",
                    p->in.c, p->cr);
      // one cluster per image: 8 CTAs, or 16 when the weight slices would not fit in smem
      if ((p->apply & 1) && (p->out.n != p->in.n || p->out.h != p->in.h || p->out.w != p->in.w ||
                       p->out.c != p->in.c))
        return fail(DFX_E_ARG, "se apply: out view must have the input's shape");
      // 16 CTAs per image (measured faster than 8 at batch 1 and 32: smaller slices,
      // more pooling parallelism); DFX_SE_CL=8 for A/B
      static const int cl_env = getenv("DFX_SE_CL") ? atoi(getenv("DFX_SE_CL")) : 16;
      int cl = (cl_env == 8 && dfx::se_smem_bytes(p->in.c, p->cr, 8) <= dfx::kSeSmemBudget) ? 8 : 16;
      // DFX_SE_IPI=4: 4 images per cluster from batch 8 (each FC weight read serves 4
      // images).  Off by default: the lost pooling/scaling parallelism costs more than
      // the weight traffic saves (EfficientNetV2-L batch 32 6.73 vs 6.07 ms)
      static const int ipi_env = getenv("DFX_SE_IPI") ? atoi(getenv("DFX_SE_IPI")) : 1;
      // split precision (DFX_SE_IPI_SPLIT=4, A/B): the hi + lo FC slices double the
      // per-image L2 weight traffic that 4 images per cluster amortise
      static const int ipi_split_env = getenv("DFX_SE_IPI_SPLIT") ? atoi(getenv("DFX_SE_IPI_SPLIT")) : 1;
      const int ipi = (cl == 16 && p->in.n >= 8 &&
                       (dfx::dtype_split(p->in.dtype) ? ipi_split_env == 4 : ipi_env == 4)) ? 4 : 1;
      const bool split = dfx::dtype_split(p->in.dtype);       // hi + lo FC slices, no x tile
      if (split) cl = 16;
      c->func = se_func(p->in.dtype, cl, ipi);
      c->grid = dim3(unsigned(cl), unsigned((p->in.n + ipi - 1) / ipi));
      c->smem = (p->apply & 2) ? ((p->apply & 4) ? size_t(dfx::se_smem_bytes(p->in.c, p->cr, cl)) / 2 * (split ? 2 : 1) : 0)
                               : size_t(dfx::se_smem_bytes(p->in.c, p->cr, cl)) * (split ? 2 : 1);
      // room for the CTA's x slice (latency-bound small batches): the scale reads smem
      // (batch 1: EfficientNetV2-L 2.10 -> 2.08 ms; at batch 32 it costs occupancy)
      static const int xt_batch = getenv("DFX_SE_XTILE_BATCH") ? atoi(getenv("DFX_SE_XTILE_BATCH")) : 8;
      // split precision keeps it at every batch (the scale's second read is of two
      // planes): 4-model batch 32 fp16x2 17.08 -> 16.88 ms
      static const int xt_batch_x2 =
          getenv("DFX_SE_XTILE_BATCH_X2") ? atoi(getenv("DFX_SE_XTILE_BATCH_X2")) : (1 << 30);
      if ((p->apply & 1) && ipi == 1 && p->in.n < (split ? xt_batch_x2 : xt_batch)) {
        const size_t xt = size_t(p->in.h) * p->in.w * dfx::se_chan_slice(p->in.c, cl) * 2 * (split ? 2 : 1);
        if (c->smem + xt <= size_t(dfx::kSeSmemBudget)) c->smem += xt;
      }
      if (c->smem > size_t(dfx::kSeSmemBudget))
        return fail(DFX_E_UNSUPPORTED, "se: c=%d cr=%d needs %zu B of smem", p->in.c, p->cr, c->smem);
      return DFX_OK;
    }
    case DFX_OP_DWSE: {
      NEED(dfx_dwse_params);
      const auto* p = static_cast<const dfx_dwse_params*>(params);
      if (p->in.c > 4096 || (p->in.c & 7) || p->cr > 512 || p->cr < 1 || p->out.c != p->in.c ||
          p->out.n != p->in.n || ((p->in.coff | p->out.coff | p->in.pitch | p->out.pitch) & 7) ||
          p->dw_epi.binop != DFX_BIN_NONE)
        return fail(DFX_E_UNSUPPORTED, "dwse: c=%d cr=%d / views beyond the fused kernel's limits",
                    p->in.c, p->cr);
      if (dfx::dtype_split(p->in.dtype)) return fail(DFX_E_UNSUPPORTED, "dwse: split precision");
      c->func = DFX_PICK16(dwse_kernel, p->in.dtype);
      c->grid = dim3(16u, unsigned(p->in.n));
      c->smem = size_t(dfx::dwse_smem_bytes(p->in.c, p->cr, p->out.h * p->out.w, p->staged));
      if (c->smem > size_t(dfx::kSeSmemBudget))
        return fail(DFX_E_UNSUPPORTED, "dwse: %zu B of smem", c->smem);
      return DFX_OK;
    }
    case DFX_OP_LN: {
      NEED(dfx_ln_params);
      const auto* p = static_cast<const dfx_ln_params*>(params);
      if (p->out.w > p->in.w || p->out.c != p->in.c || p->out.n != p->in.n || p->in.h != 1 ||
          (p->norm && (!p->gamma || !p->beta)))
        return fail(DFX_E_ARG, "ln: bad views/weights");
      if (dfx::dtype_split(p->in.dtype)) return fail(DFX_E_UNSUPPORTED, "ln: split precision");
      c->func = DFX_PICK16(ln_kernel, p->in.dtype);
      c->grid = dim3(unsigned(cdiv(int64_t(p->out.n) * p->out.w, 8)));
      c->block = dim3(256);
      return DFX_OK;
    }
    case DFX_OP_TOKENS: {
      NEED(dfx_tokens_params);
      const auto* p = static_cast<const dfx_tokens_params*>(params);
      if (p->out.w != 1 + p->in.h * p->in.w || p->out.c != p->in.c || p->out.h != 1)
        return fail(DFX_E_ARG, "tokens: out (%d, %d, %d) for grid (%d, %d, %d)", p->out.h, p->out.w,
                    p->out.c, p->in.h, p->in.w, p->in.c);
      if (dfx::dtype_split(p->out.dtype)) return fail(DFX_E_UNSUPPORTED, "tokens: split precision");
      c->func = DFX_PICK16(tokens_kernel, p->out.dtype);
      c->grid = dim3(elementwise_grid(int64_t(p->out.n) * p->out.w * cdiv(p->out.c, 8), 256));
      return DFX_OK;
    }
    case DFX_OP_GATE: {
      NEED(dfx_gate_params);
      const auto* p = static_cast<const dfx_gate_params*>(params);
      if (!p->flag) return fail(DFX_E_ARG, "gate: null flag");
      c->func = reinterpret_cast<const void*>(&dfx::gate_kernel);
      c->grid = dim3(1);
      c->block = dim3(32);
      return DFX_OK;
    }
    case DFX_OP_ATTN: {
      NEED(dfx_attn_params);
      const auto* p = static_cast<const dfx_attn_params*>(params);
      const int L = p->qkv.w;
      if (p->heads < 1 || p->out.c != p->heads * 64 || p->qkv.c != 3 * p->out.c ||
          p->out.w != L || p->qkv.h != 1 || L > dfx::kAttnMaxL || L < 1 ||
          ((p->qkv.pitch | p->qkv.coff | p->out.pitch | p->out.coff) & 7))
        return fail(DFX_E_UNSUPPORTED, "attention: L=%d heads=%d c=%d (head dim 64, L <= %d)", L,
                    p->heads, p->out.c, dfx::kAttnMaxL);
      if (dfx::dtype_split(p->qkv.dtype)) return fail(DFX_E_UNSUPPORTED, "attn: split precision");
      c->func = DFX_PICK16(attn_kernel, p->qkv.dtype);
      c->grid = dim3(unsigned(cdiv(L, 64)), unsigned(p->heads), unsigned(p->qkv.n));
      c->block = dim3(128);
      c->smem = size_t(dfx::attn_smem_bytes(L));
      return DFX_OK;
    }
  }
#undef NEED
  return fail(DFX_E_ARG, "unknown op %d", op);
}

struct Graph {
  cudaGraph_t g = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::vector<cudaGraphNode_t> nodes;
  bool use_priority = false;      // some node carries a priority attribute
  // programmatic dependent launch between nodes; DFX_PDL=0 in the environment
  // turns it off (A/B measurements)
  bool pdl = [] {
    const char* e = getenv("DFX_PDL");
    return !(e && e[0] == '0');
  }();
};

}  // namespace

extern "C" {

const char* dfx_last_error(void) { return g_err.c_str(); }
int dfx_abi_version(void) { return DFX_ABI_VERSION; }

int dfx_sizeof(const char* name) {
  struct {
    const char* n;
    int s;
  } t[] = {{"dfx_view", sizeof(dfx_view)},
           {"dfx_epilogue", sizeof(dfx_epilogue)},
           {"dfx_gemm_desc", sizeof(dfx_gemm_desc)},
           {"dfx_gemm_launch", sizeof(dfx_gemm_launch)},
           {"dfx_splitk_params", sizeof(dfx_splitk_params)},
           {"dfx_dwconv_params", sizeof(dfx_dwconv_params)},
           {"dfx_pool_params", sizeof(dfx_pool_params)},
           {"dfx_gap_params", sizeof(dfx_gap_params)},
           {"dfx_ew_params", sizeof(dfx_ew_params)},
           {"dfx_in_params", sizeof(dfx_in_params)},
           {"dfx_out_params", sizeof(dfx_out_params)},
           {"dfx_se_params", sizeof(dfx_se_params)},
           {"dfx_ln_params", sizeof(dfx_ln_params)},
           {"dfx_tokens_params", sizeof(dfx_tokens_params)},
           {"dfx_attn_params", sizeof(dfx_attn_params)},
           {"dfx_dwse_params", sizeof(dfx_dwse_params)},
           {"dfx_se_fuse", sizeof(dfx_se_fuse)},
           {"dfx_gate_params", sizeof(dfx_gate_params)}};
  for (auto& e : t)
    if (!strcmp(e.n, name)) return e.s;
  return -1;
}

int dfx_init(int device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    return fail(DFX_E_NODEVICE, "no CUDA device visible");
  if (device < 0 || device >= n) return fail(DFX_E_ARG, "device %d of %d", device, n);
  CK(cudaSetDevice(device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(DFX_E_NODEVICE, "device %d is sm_%d%d; libdfx is built for sm_100a", device,
                prop.major, prop.minor);
  g_sm_count = prop.multiProcessorCount;
  for (int dt : {int(DFX_BF16), int(DFX_F16)}) {
    for (int m2 : {0, 1})
      CK(cudaFuncSetAttribute(gemm_func(dt, m2), cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kGemmSmemLimit));
    CK(cudaFuncSetAttribute(DFX_PICK(gemm_persist_kernel, dt), cudaFuncAttributeMaxDynamicSharedMemorySize,
                            kGemmSmemLimit));
    CK(cudaFuncSetAttribute(DFX_PICK(in_im2col_kernel, dt), cudaFuncAttributeMaxDynamicSharedMemorySize,
                            kIm2colSmemLimit));
    for (int cl : {8, 16})
      CK(cudaFuncSetAttribute(se_func(dt, cl), cudaFuncAttributeMaxDynamicSharedMemorySize,
                              dfx::kSeSmemBudget));
    CK(cudaFuncSetAttribute(se_func(dt, 16), cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(se_func(dt, 16, 4), cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(se_func(dt, 16, 4), cudaFuncAttributeMaxDynamicSharedMemorySize,
                            dfx::kSeSmemBudget));
    CK(cudaFuncSetAttribute(DFX_PICK16(dwse_kernel, dt), cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(DFX_PICK16(dwse_kernel, dt), cudaFuncAttributeMaxDynamicSharedMemorySize,
                            dfx::kSeSmemBudget));
    CK(cudaFuncSetAttribute(DFX_PICK16(attn_kernel, dt), cudaFuncAttributeMaxDynamicSharedMemorySize,
                            dfx::attn_smem_bytes(dfx::kAttnMaxL)));
  }
  for (int dt : {int(DFX_BF16X2), int(DFX_F16X2), int(DFX_BF16), int(DFX_F16)})   // 9..16-CTA split-K clusters
    CK(cudaFuncSetAttribute(gemm_func(dt, 0), cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  for (int dt : {int(DFX_BF16X2), int(DFX_F16X2)}) {         // split precision
    CK(cudaFuncSetAttribute(gemm_func(dt, 0), cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmSmemLimit));
    CK(cudaFuncSetAttribute(DFX_PICK(gemm_persist_kernel, dt), cudaFuncAttributeMaxDynamicSharedMemorySize,
                            kGemmSmemLimit));
    CK(cudaFuncSetAttribute(DFX_PICK(in_im2col_kernel, dt), cudaFuncAttributeMaxDynamicSharedMemorySize,
                            kIm2colSmemLimit));
    CK(cudaFuncSetAttribute(se_func(dt, 16), cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(se_func(dt, 16), cudaFuncAttributeMaxDynamicSharedMemorySize, dfx::kSeSmemBudget));
    CK(cudaFuncSetAttribute(se_func(dt, 16, 4), cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(se_func(dt, 16, 4), cudaFuncAttributeMaxDynamicSharedMemorySize,
                            dfx::kSeSmemBudget));
  }
  return get_encode();
}

int dfx_device_info(int device, int* sm_count, int* cc_major, int* cc_minor, size_t* total_mem) {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (cc_major) *cc_major = prop.major;
  if (cc_minor) *cc_minor = prop.minor;
  if (total_mem) *total_mem = prop.totalGlobalMem;
  return DFX_OK;
}

int dfx_mem_info(size_t* free_bytes, size_t* total_bytes) {
  CK(cudaMemGetInfo(free_bytes, total_bytes));
  return DFX_OK;
}

int dfx_malloc(void** dptr, size_t bytes) {
  if (!dptr) return fail(DFX_E_ARG, "null out pointer");
  cudaError_t e = cudaMalloc(dptr, bytes ? bytes : 1);
  if (e != cudaSuccess) return fail(DFX_E_NOMEM, "cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
  return DFX_OK;
}
int dfx_free(void* dptr) {
  CK(cudaFree(dptr));
  return DFX_OK;
}

// Weight-arena pool: one stream-ordered memory pool per device whose release
// threshold is unbounded, so a swapped-out arena's pages stay mapped and the next
// arena (the same DAG again, or another one) is carved from them without a new
// physical mapping.  A fresh cudaMalloc of a re-freed 587 MB arena measured
// 0.5-54 ms depending on the box; a pool allocation of mapped memory is a few us.
static int arena_pool(cudaMemPool_t* out) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail(DFX_E_ARG, "device %d", dev);
  std::lock_guard<std::mutex> g(mu);
  if (!pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    CK(cudaMemPoolCreate(&pools[dev], &props));
    uint64_t keep = ~uint64_t(0);
    CK(cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep));
  }
  *out = pools[dev];
  return DFX_OK;
}

int dfx_pool_malloc(void** dptr, size_t bytes, void* stream) {
  if (!dptr) return fail(DFX_E_ARG, "null out pointer");
  cudaMemPool_t pool;
  int rc = arena_pool(&pool);
  if (rc) return rc;
  CK(cudaMallocFromPoolAsync(dptr, bytes, pool, S(stream)));
  CK(cudaStreamSynchronize(S(stream)));
  return DFX_OK;
}

int dfx_pool_free(void* dptr, void* stream) {
  if (!dptr) return DFX_OK;
  CK(cudaFreeAsync(dptr, S(stream)));
  CK(cudaStreamSynchronize(S(stream)));
  return DFX_OK;
}

int dfx_pool_trim(size_t keep_bytes) {
  cudaMemPool_t pool;
  int rc = arena_pool(&pool);
  if (rc) return rc;
  CK(cudaMemPoolTrimTo(pool, keep_bytes));
  return DFX_OK;
}

int dfx_pool_stats(size_t* reserved, size_t* used) {
  cudaMemPool_t pool;
  int rc = arena_pool(&pool);
  if (rc) return rc;
  uint64_t r = 0, u = 0;
  CK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &r));
  CK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &u));
  if (reserved) *reserved = size_t(r);
  if (used) *used = size_t(u);
  return DFX_OK;
}
int dfx_memset(void* dptr, int value, size_t bytes, void* stream) {
  CK(cudaMemsetAsync(dptr, value, bytes, S(stream)));
  return DFX_OK;
}
int dfx_host_alloc(void** hptr, size_t bytes) {
  cudaError_t e = cudaHostAlloc(hptr, bytes ? bytes : 1, cudaHostAllocDefault);
  if (e != cudaSuccess) return fail(DFX_E_NOMEM, "cudaHostAlloc(%zu): %s", bytes, cudaGetErrorString(e));
  return DFX_OK;
}
int dfx_host_free(void* hptr) {
  CK(cudaFreeHost(hptr));
  return DFX_OK;
}
int dfx_host_register(void* hptr, size_t bytes) {
  CK(cudaHostRegister(hptr, bytes, cudaHostRegisterDefault));
  return DFX_OK;
}
int dfx_host_unregister(void* hptr) {
  CK(cudaHostUnregister(hptr));
  return DFX_OK;
}
int dfx_memcpy_h2d(void* dst, const void* src, size_t bytes, void* stream) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, S(stream)));
  return DFX_OK;
}
int dfx_memcpy_d2h(void* dst, const void* src, size_t bytes, void* stream) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, S(stream)));
  return DFX_OK;
}
int dfx_memcpy_d2d(void* dst, const void* src, size_t bytes, void* stream) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, S(stream)));
  return DFX_OK;
}

int dfx_nvtx_range_push(const char* msg) {
  nvtxRangePushA(msg ? msg : "dfx");
  return DFX_OK;
}
int dfx_nvtx_range_pop(void) {
  nvtxRangePop();
  return DFX_OK;
}

int dfx_arena_upload(const void* pinned_host, size_t bytes, void** dev_arena, void* stream) {
  NvtxRange r("dfx arena upload (swap-in)");
  int rc = dfx_malloc(dev_arena, bytes);
  if (rc) return rc;
  CK(cudaMemcpyAsync(*dev_arena, pinned_host, bytes, cudaMemcpyHostToDevice, S(stream)));
  return DFX_OK;
}

int dfx_stream_create(void** stream) {
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  *stream = s;
  return DFX_OK;
}
int dfx_stream_destroy(void* stream) {
  CK(cudaStreamDestroy(S(stream)));
  return DFX_OK;
}
int dfx_stream_sync(void* stream) {
  CK(cudaStreamSynchronize(S(stream)));
  return DFX_OK;
}
int dfx_event_create(void** ev) {
  cudaEvent_t e;
  CK(cudaEventCreate(&e));
  *ev = e;
  return DFX_OK;
}
int dfx_event_destroy(void* ev) {
  CK(cudaEventDestroy(reinterpret_cast<cudaEvent_t>(ev)));
  return DFX_OK;
}
int dfx_event_record(void* ev, void* stream) {
  CK(cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev), S(stream)));
  return DFX_OK;
}
int dfx_event_elapsed(void* start, void* stop, float* ms) {
  CK(cudaEventSynchronize(reinterpret_cast<cudaEvent_t>(stop)));
  CK(cudaEventElapsedTime(ms, reinterpret_cast<cudaEvent_t>(start),
                          reinterpret_cast<cudaEvent_t>(stop)));
  return DFX_OK;
}

int dfx_tmap_act(void* out128, const dfx_view* v, int cb, int tq, int tp, int tn, int stride_w,
                 int stride_h) {
  int rc = get_encode();
  if (rc) return rc;
  if (!v || !out128) return fail(DFX_E_ARG, "tmap_act: null");
  if (cb != 16 && cb != 32 && cb != 64) return fail(DFX_E_ARG, "tmap_act: cb %d", cb);
  if (v->pitch % 8 || v->coff % 8) return fail(DFX_E_ARG, "tmap_act: pitch %d coff %d", v->pitch, v->coff);
  if (tq * stride_w > 256 || tp * stride_h > 256 || tn > 256 || tq * tp * tn > 128)
    return fail(DFX_E_ARG, "tmap_act: box %dx%dx%d stride %d,%d", tq, tp, tn, stride_w, stride_h);
  void* base = static_cast<char*>(v->base) + int64_t(v->coff) * 2;
  if (reinterpret_cast<uintptr_t>(base) % 16) return fail(DFX_E_ARG, "tmap_act: base alignment");
  // split precision: a 5th dimension selects the plane (hi = 0, lo = 1, pitch/2 elements apart)
  const bool split = dfx::dtype_split(v->dtype);
  if (split && v->pitch % 16) return fail(DFX_E_ARG, "tmap_act: split pitch %d", v->pitch);
  cuuint64_t dims[5] = {cuuint64_t(v->c), cuuint64_t(v->w), cuuint64_t(v->h), cuuint64_t(v->n), 2};
  cuuint64_t strides[4] = {cuuint64_t(v->pitch) * 2, cuuint64_t(v->pitch) * 2 * v->w,
                           cuuint64_t(v->pitch) * 2 * v->w * v->h, cuuint64_t(v->pitch)};
  cuuint32_t box[5] = {cuuint32_t(cb), cuuint32_t(tq * stride_w), cuuint32_t(tp * stride_h),
                       cuuint32_t(tn), 1};
  cuuint32_t estr[5] = {1, cuuint32_t(stride_w), cuuint32_t(stride_h), 1, 1};
  CUresult r = g_encode(reinterpret_cast<CUtensorMap*>(out128), tmap_dtype(v->dtype), split ? 5 : 4,
                        base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swizzle_for(cb), CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(DFX_E_CUDA, "cuTensorMapEncodeTiled(act c=%d w=%d h=%d n=%d pitch=%d cb=%d box=%u,%u,%u,%u) = %d",
                v->c, v->w, v->h, v->n, v->pitch, cb, box[0], box[1], box[2], box[3], int(r));
  return DFX_OK;
}

int dfx_tmap_weights(void* out128, const void* base, int rows, int k, int cb, int bn, int dtype) {
  int rc = get_encode();
  if (rc) return rc;
  if (cb != 16 && cb != 32 && cb != 64) return fail(DFX_E_ARG, "tmap_weights: cb %d", cb);
  if (k % 8 || reinterpret_cast<uintptr_t>(base) % 16)
    return fail(DFX_E_ARG, "tmap_weights: k %d / alignment", k);
  // split precision: `rows` = 2 cout ([hi rows; lo rows]) as a 3-D map (k, cout, plane):
  // ONE box (cb, bn, 2) lands a k-step's hi and lo rows back to back in smem
  const bool split = dfx::dtype_split(dtype);
  if (split && rows % 2) return fail(DFX_E_ARG, "tmap_weights: split rows %d", rows);
  cuuint64_t dims[3] = {cuuint64_t(k), cuuint64_t(split ? rows / 2 : rows), 2};
  cuuint64_t strides[2] = {cuuint64_t(k) * 2, cuuint64_t(k) * 2 * cuuint64_t(rows / 2)};
  cuuint32_t box[3] = {cuuint32_t(cb), cuuint32_t(bn), 2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(reinterpret_cast<CUtensorMap*>(out128), tmap_dtype(dtype), split ? 3 : 2,
                        const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_for(cb),
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(DFX_E_CUDA, "cuTensorMapEncodeTiled(weights rows=%d k=%d cb=%d bn=%d) = %d", rows, k,
                cb, bn, int(r));
  return DFX_OK;
}

int dfx_launch(int op, const void* params, size_t params_size, void* stream) {
  LaunchCfg c;
  int rc = config_for(op, params, params_size, &c);
  if (rc) return rc;
  void* args[1] = {const_cast<void*>(params)};
  if (c.cluster > 1) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = c.grid;
    lc.blockDim = c.block;
    lc.dynamicSmemBytes = c.smem;
    lc.stream = S(stream);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c.cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    CK(cudaLaunchKernelExC(&lc, c.func, args));
    return DFX_OK;
  }
  CK(cudaLaunchKernel(c.func, c.grid, c.block, args, c.smem, S(stream)));
  return DFX_OK;
}

int dfx_graph_create(void** graph) {
  auto* g = new Graph();
  cudaError_t e = cudaGraphCreate(&g->g, 0);
  if (e != cudaSuccess) {
    delete g;
    return fail(DFX_E_CUDA, "cudaGraphCreate: %s", cudaGetErrorString(e));
  }
  *graph = g;
  return DFX_OK;
}

int dfx_graph_add(void* graph, int op, const void* params, size_t params_size, const int* deps,
                  int ndeps, int* node_id) {
  auto* g = static_cast<Graph*>(graph);
  if (!g || g->exec) return fail(DFX_E_STATE, "graph_add after instantiate");
  LaunchCfg c;
  int rc = config_for(op, params, params_size, &c);
  if (rc) return rc;
  std::vector<cudaGraphNode_t> dn;
  for (int i = 0; i < ndeps; ++i) {
    if (deps[i] < 0 || deps[i] >= int(g->nodes.size()))
      return fail(DFX_E_ARG, "graph_add: dependency %d out of range", deps[i]);
    dn.push_back(g->nodes[deps[i]]);
  }
  cudaKernelNodeParams kp = {};
  void* args[1] = {const_cast<void*>(params)};
  kp.func = const_cast<void*>(c.func);
  kp.gridDim = c.grid;
  kp.blockDim = c.block;
  kp.sharedMemBytes = unsigned(c.smem);
  kp.kernelParams = args;
  cudaGraphNode_t node;
  if (g->pdl && !dn.empty()) {
    // programmatic edges: the node may launch once every predecessor block has
    // called griddepcontrol.launch_dependents; it griddepcontrol.wait()s for
    // their completion before touching activations (see dfx_common.cuh)
    CK(cudaGraphAddKernelNode(&node, g->g, nullptr, 0, &kp));
    for (cudaGraphNode_t from : dn) {
      cudaGraphEdgeData ed = {};
      ed.from_port = cudaGraphKernelNodePortProgrammatic;
      ed.type = cudaGraphDependencyTypeProgrammatic;
      CK(cudaGraphAddDependencies_v2(g->g, &from, &node, &ed, 1));
    }
  } else {
    CK(cudaGraphAddKernelNode(&node, g->g, dn.data(), dn.size(), &kp));
  }
  if (c.cluster > 1) {
    cudaLaunchAttributeValue v = {};
    v.clusterDim.x = c.cluster;
    v.clusterDim.y = 1;
    v.clusterDim.z = 1;
    CK(cudaGraphKernelNodeSetAttribute(node, cudaLaunchAttributeClusterDimension, &v));
  }
  g->nodes.push_back(node);
  if (node_id) *node_id = int(g->nodes.size()) - 1;
  return DFX_OK;
}

int dfx_graph_set_priority(void* graph, int node_id, int priority, int* range_out) {
  auto* g = static_cast<Graph*>(graph);
  if (!g || g->exec) return fail(DFX_E_STATE, "graph_set_priority after instantiate");
  int least = 0, greatest = 0;
  CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  if (range_out) {
    range_out[0] = least;
    range_out[1] = greatest;
  }
  if (node_id < 0 || node_id >= int(g->nodes.size()))
    return fail(DFX_E_ARG, "graph_set_priority: node %d out of range", node_id);
  cudaLaunchAttributeValue v = {};
  v.priority = std::min(least, std::max(greatest, priority));
  CK(cudaGraphKernelNodeSetAttribute(g->nodes[node_id], cudaLaunchAttributePriority, &v));
  g->use_priority = true;
  return DFX_OK;
}

int dfx_graph_instantiate(void* graph) {
  NvtxRange r("dfx graph instantiate");
  auto* g = static_cast<Graph*>(graph);
  if (!g) return fail(DFX_E_ARG, "null graph");
  if (g->exec) return DFX_OK;
  CK(cudaGraphInstantiate(&g->exec, g->g,
                          g->use_priority ? cudaGraphInstantiateFlagUseNodePriority : 0));
  return DFX_OK;
}

int dfx_graph_launch(void* graph, void* stream) {
  NvtxRange r("dfx fused DAG graph launch");
  auto* g = static_cast<Graph*>(graph);
  if (!g || !g->exec) return fail(DFX_E_STATE, "graph not instantiated");
  CK(cudaGraphLaunch(g->exec, S(stream)));
  return DFX_OK;
}

int dfx_graph_node_count(void* graph, int* count) {
  auto* g = static_cast<Graph*>(graph);
  if (!g) return fail(DFX_E_ARG, "null graph");
  *count = int(g->nodes.size());
  return DFX_OK;
}

int dfx_graph_destroy(void* graph) {
  auto* g = static_cast<Graph*>(graph);
  if (!g) return DFX_OK;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->g) cudaGraphDestroy(g->g);
  delete g;
  return DFX_OK;
}

int dfx_execute(void* graph, const void* host_in, void* dev_in, size_t in_bytes, void* host_out,
                const void* dev_out, size_t out_bytes, void* stream) {
  CK(cudaMemcpyAsync(dev_in, host_in, in_bytes, cudaMemcpyHostToDevice, S(stream)));
  int rc = dfx_graph_launch(graph, stream);
  if (rc) return rc;
  CK(cudaMemcpyAsync(host_out, dev_out, out_bytes, cudaMemcpyDeviceToHost, S(stream)));
  CK(cudaStreamSynchronize(S(stream)));
  return DFX_OK;
}

}  // extern "C"

namespace {

// ---- host staging pool for dfx_execute_gather
//
// A query's inputs arrive as separate pageable host arrays (one per member or
// sample).  A single thread copies them into the pinned staging buffer at
// ~10 GB/s, which at batch 1 cost more than the H2D itself.  The pool copies
// fixed-size chunks on several threads while the calling thread issues the H2D
// of every completed prefix, so the DMA overlaps the remaining host copies.
// Workers spin for a few ms after a job (queries arrive back to back), then
// sleep on a condition variable.
struct StagePool {
  static constexpr size_t kChunk = size_t(256) << 10;
  static constexpr int kMaxChunks = 4096;
  // One 64-bit word carries the job: bits [27, 40) the chunk count n of the job,
  // bits [0, 27) the next claim index.  A claim (fetch_add) therefore returns the
  // index together with the count of the SAME job: a worker whose claim is >= n
  // drops it without touching chunks[] / done[], whichever job is current by then.
  // A claim < n pins the job: the job cannot end (and chunks[] cannot be rewritten)
  // until that chunk's done flag is set by the claimant.
  static constexpr int kIdxBits = 27;
  static constexpr uint64_t kIdxMask = (uint64_t(1) << kIdxBits) - 1;
  struct Chunk {
    char* dst;
    const char* src;
    size_t bytes;
  };
  std::mutex job_mu;                       // one job at a time uses the workers
  std::mutex mu;
  std::condition_variable cv;
  std::vector<std::thread> workers;
  std::atomic<uint64_t> gen{0};
  std::atomic<uint64_t> claim{0};          // (n << kIdxBits) | next index
  std::atomic<int> done[kMaxChunks];
  Chunk chunks[kMaxChunks];
  bool stop = false;

  explicit StagePool(int nthreads) {
    for (int i = 0; i < nthreads; ++i) workers.emplace_back([this] { loop(); });
  }
  ~StagePool() {
    {
      std::lock_guard<std::mutex> g(mu);
      stop = true;
      gen.fetch_add(1);
    }
    cv.notify_all();
    for (auto& t : workers) t.join();
  }
  // claim one chunk of the current job; -1 when the job has none left
  int take() {
    const uint64_t v = claim.fetch_add(1, std::memory_order_acq_rel);
    const uint64_t idx = v & kIdxMask, n = v >> kIdxBits;
    return idx < n ? int(idx) : -1;
  }
  void copy(int c) {
    std::memcpy(chunks[c].dst, chunks[c].src, chunks[c].bytes);
    done[c].store(1, std::memory_order_release);
  }
  void work() {
    for (int c; (c = take()) >= 0;) copy(c);
  }
  void loop() {
    uint64_t seen = gen.load();
    for (;;) {
      auto t0 = std::chrono::steady_clock::now();
      while (gen.load(std::memory_order_acquire) == seen) {
        if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(3)) {
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&] { return gen.load() != seen; });
          break;
        }
        std::this_thread::yield();
      }
      seen = gen.load(std::memory_order_acquire);
      if (stop) return;
      work();      // a job that already ended (or is being set up) has no claimable chunk
    }
  }
};

StagePool* stage_pool() {
  static StagePool* pool = [] {
    int n = int(std::thread::hardware_concurrency()) / 2;
    if (const char* e = std::getenv("DFX_STAGE_THREADS")) n = std::atoi(e);
    n = std::max(0, std::min(n, 15));
    return new StagePool(n);                    // leaked on purpose: no teardown-order issues
  }();
  return pool;
}

}  // namespace

extern "C" {

int dfx_execute_gather(void* graph, const void* const* srcs, const size_t* sizes, int nsrc, void* host_in,
                       void* dev_in, void* host_out, const void* dev_out, size_t out_bytes, void* stream) {
  NvtxRange r("dfx execute_fused (gather, H2D, graph, D2H)");
  if (nsrc < 0 || (nsrc > 0 && (!srcs || !sizes)) || !host_in) return fail(DFX_E_ARG, "bad gather list");
  size_t total = 0;
  int nch = 0;
  for (int i = 0; i < nsrc; ++i) {
    total += sizes[i];
    nch += int((sizes[i] + StagePool::kChunk - 1) / StagePool::kChunk);
  }
  if (nch > StagePool::kMaxChunks) return fail(DFX_E_ARG, "gather list too large");
  StagePool* P = stage_pool();
  // The pool serves one staging job at a time; a concurrent query whose staging
  // finds it busy copies on its own thread instead of waiting.  Only the staging
  // is serialised: the lock is dropped before the graph launch and the sync.
  std::unique_lock<std::mutex> job(P->job_mu, std::try_to_lock);
  if (!job.owns_lock() || P->workers.empty() || nch <= 1) {
    if (job.owns_lock()) job.unlock();
    size_t off = 0;
    for (int i = 0; i < nsrc; ++i) {
      std::memcpy(static_cast<char*>(host_in) + off, srcs[i], sizes[i]);
      off += sizes[i];
    }
    CK(cudaMemcpyAsync(dev_in, host_in, total, cudaMemcpyHostToDevice, S(stream)));
  } else {
    // no claim of the previous job can be outstanding (it ended with every chunk
    // done); late claimers see n = 0 while the list is rewritten
    P->claim.store(0, std::memory_order_relaxed);
    int n = 0;
    size_t off = 0;
    for (int i = 0; i < nsrc; ++i) {
      for (size_t s = 0; s < sizes[i]; s += StagePool::kChunk) {
        const size_t b = std::min(StagePool::kChunk, sizes[i] - s);
        P->chunks[n] = {static_cast<char*>(host_in) + off + s, static_cast<const char*>(srcs[i]) + s, b};
        P->done[n].store(0, std::memory_order_relaxed);
        ++n;
      }
      off += sizes[i];
    }
    P->claim.store(uint64_t(n) << StagePool::kIdxBits, std::memory_order_release);
    {
      std::lock_guard<std::mutex> g(P->mu);
      P->gen.fetch_add(1, std::memory_order_release);
    }
    P->cv.notify_all();
    // the caller copies chunks too, and issues the H2D of each completed in-order prefix
    int issued = 0;
    cudaError_t err = cudaSuccess;
    while (issued < n) {
      int ready = issued;
      while (ready < n && P->done[ready].load(std::memory_order_acquire)) ++ready;
      if (ready > issued) {
        const size_t b0 = size_t(P->chunks[issued].dst - static_cast<char*>(host_in));
        const size_t b1 = size_t(P->chunks[ready - 1].dst - static_cast<char*>(host_in)) + P->chunks[ready - 1].bytes;
        if (err == cudaSuccess)
          err = cudaMemcpyAsync(static_cast<char*>(dev_in) + b0, static_cast<char*>(host_in) + b0, b1 - b0,
                                cudaMemcpyHostToDevice, S(stream));
        issued = ready;
        continue;
      }
      const int c = P->take();
      if (c >= 0) P->copy(c);
    }
    job.unlock();
    CK(err);
  }
  int rc = dfx_graph_launch(graph, stream);
  if (rc) return rc;
  CK(cudaMemcpyAsync(host_out, dev_out, out_bytes, cudaMemcpyDeviceToHost, S(stream)));
  CK(cudaStreamSynchronize(S(stream)));
  return DFX_OK;
}

int dfx_execute_gated(void* graph, const void* const* srcs, const size_t* sizes, const int* src_member, int nsrc,
                      const size_t* member_off, const size_t* member_bytes, int nmembers, void* host_in,
                      void* dev_in, uint32_t* flags, const uint32_t* one, void* host_out, const void* dev_out,
                      size_t out_bytes, void* stream, void* copy_stream) {
  NvtxRange r("dfx execute_fused (gated: graph first, members' inputs behind it)");
  if (nsrc < 0 || nmembers < 1 || nmembers > 64 || (nsrc > 0 && (!srcs || !sizes || !src_member)) || !host_in ||
      !flags || !one || !member_off || !member_bytes || copy_stream == stream)
    return fail(DFX_E_ARG, "execute_gated: bad arguments");
  // 1. the graph first: every member's gate node waits for its flag
  int rc = dfx_graph_launch(graph, stream);
  if (rc) return rc;
  // 2. sources -> pinned staging, member by member (sources arrive member by member)
  int nch = 0;
  for (int i = 0; i < nsrc; ++i) nch += int((sizes[i] + StagePool::kChunk - 1) / StagePool::kChunk);
  if (nch > StagePool::kMaxChunks) return fail(DFX_E_ARG, "gather list too large");
  std::vector<int> chunk_member(size_t(nch > 0 ? nch : 1));
  std::vector<int> left(size_t(nmembers), 0);            // chunks still to copy, per member
  cudaError_t err = cudaSuccess;
  auto open_gate = [&](int m) {
    if (err != cudaSuccess) return;
    if (member_bytes[m])
      err = cudaMemcpyAsync(static_cast<char*>(dev_in) + member_off[m], static_cast<char*>(host_in) + member_off[m],
                            member_bytes[m], cudaMemcpyHostToDevice, S(copy_stream));
    if (err == cudaSuccess)
      err = cudaMemcpyAsync(flags + m, one, sizeof(uint32_t), cudaMemcpyHostToDevice, S(copy_stream));
  };
  std::vector<size_t> at(size_t(nmembers), 0);
  StagePool* P = stage_pool();
  std::unique_lock<std::mutex> job(P->job_mu, std::try_to_lock);
  if (!job.owns_lock() || P->workers.empty() || nch <= 1) {
    if (job.owns_lock()) job.unlock();
    int i = 0;
    std::vector<char> opened(size_t(nmembers), 0);
    while (i < nsrc) {                                     // member by member, as listed
      const int m = src_member[i];
      for (; i < nsrc && src_member[i] == m; ++i) {
        std::memcpy(static_cast<char*>(host_in) + member_off[m] + at[m], srcs[i], sizes[i]);
        at[m] += sizes[i];
      }
      open_gate(m);
      opened[m] = 1;
    }
    for (int m = 0; m < nmembers; ++m)
      if (!opened[m]) open_gate(m);                      // members with no sources (batch 0)
  } else {
    P->claim.store(0, std::memory_order_relaxed);
    int n = 0;
    for (int i = 0; i < nsrc; ++i) {
      const int m = src_member[i];
      for (size_t s0 = 0; s0 < sizes[i]; s0 += StagePool::kChunk) {
        const size_t b = std::min(StagePool::kChunk, sizes[i] - s0);
        P->chunks[n] = {static_cast<char*>(host_in) + member_off[m] + at[m] + s0,
                        static_cast<const char*>(srcs[i]) + s0, b};
        P->done[n].store(0, std::memory_order_relaxed);
        chunk_member[size_t(n)] = m;
        ++left[size_t(m)];
        ++n;
      }
      at[m] += sizes[i];
    }
    P->claim.store(uint64_t(n) << StagePool::kIdxBits, std::memory_order_release);
    {
      std::lock_guard<std::mutex> g(P->mu);
      P->gen.fetch_add(1, std::memory_order_release);
    }
    P->cv.notify_all();
    // members open in listed order as soon as all their chunks are copied; the
    // caller copies chunks too
    std::vector<char> opened(size_t(nmembers), 0);
    int scan = 0, nopen = 0;
    for (int m = 0; m < nmembers; ++m)
      if (left[size_t(m)] == 0) {
        open_gate(m);
        opened[size_t(m)] = 1;
        ++nopen;
      }
    while (nopen < nmembers) {
      while (scan < n && P->done[scan].load(std::memory_order_acquire)) {
        const int m = chunk_member[size_t(scan)];
        if (--left[size_t(m)] == 0 && !opened[size_t(m)]) {
          open_gate(m);
          opened[size_t(m)] = 1;
          ++nopen;
        }
        ++scan;
      }
      if (nopen == nmembers) break;
      const int c = P->take();
      if (c >= 0) P->copy(c);
    }
    job.unlock();
  }
  CK(err);
  // 3. outputs
  CK(cudaMemcpyAsync(host_out, dev_out, out_bytes, cudaMemcpyDeviceToHost, S(stream)));
  CK(cudaStreamSynchronize(S(stream)));
  return DFX_OK;
}

}  // extern "C"

