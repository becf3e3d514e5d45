/*
 * dfx.h — C ABI of libdfx, the sm_100a execution library behind the fused-DAG
 * path of FusedInf (arXiv 2410.21120).
 *
 * The reference exposes this path only as a Python API (no FFI exists):
 *   fuse_models            /root/reference/pkg/src/dagfuse/fuse.py:165-200
 *   execute_fused          /root/reference/pkg/src/dagfuse/fuse.py:268-291
 *   swap_subgraph          /root/reference/pkg/src/dagfuse/fuse.py:203-242
 *   executor.run/run_batch /root/reference/pkg/src/dagfuse/executor.py:187-201
 *   simulated swap-in      /root/reference/pkg/src/dagfuse/costmodel.py:277-338
 * Python keeps those signatures (paper_2410_21120_b200/fuse.py) and crosses
 * into this library through ctypes (paper_2410_21120_b200/runtime.py); the
 * binding a maintainer would add to the reference is in INTEGRATION.md.
 * Each entry point below names the reference function whose work it does.
 *
 * Conventions: plain pointers and sizes only; every function returns
 * DFX_OK (0) or a negative dfx_status and never throws; dfx_last_error()
 * returns a thread-local message for the last failure on the calling thread.
 * Streams are passed as opaque void* (a cudaStream_t; NULL = legacy default).
 * No function synchronises unless its comment says so.
 *
 * Data layout on the device: activations are 16-bit (fp16 or bf16) NHWC with a channel pitch
 * that is a multiple of 8 elements (16 B); a tensor may be a channel window
 * [coff, coff + C) of a wider buffer (zero-copy concat).  Weights live in one
 * packed arena.
 */
#ifndef DFX_H
#define DFX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DFX_ABI_VERSION 5

typedef enum dfx_status {
  DFX_OK = 0,
  DFX_E_CUDA = -1,         /* a CUDA runtime/driver call failed */
  DFX_E_ARG = -2,          /* invalid argument */
  DFX_E_NOMEM = -3,        /* device or pinned-host allocation failed */
  DFX_E_UNSUPPORTED = -4,  /* shape/feature not supported by the kernels */
  DFX_E_STATE = -5,        /* call out of order (e.g. launch before instantiate) */
  DFX_E_NODEVICE = -6      /* no sm_100 device visible */
} dfx_status;

typedef enum dfx_act {
  DFX_ACT_NONE = 0, DFX_ACT_RELU = 1, DFX_ACT_HARDSWISH = 2,
  DFX_ACT_HARDSIGMOID = 3, DFX_ACT_SILU = 4, DFX_ACT_SIGMOID = 5,
  DFX_ACT_GELU = 6     /* exact: 0.5 x (1 + erf(x / sqrt 2)) */
} dfx_act;

typedef enum dfx_binop {
  DFX_BIN_NONE = 0,
  DFX_BIN_ADD = 1,     /* v += other[n, h, w, c]            (residual_add)   */
  DFX_BIN_SCALE = 2    /* v *= other[n, 0, 0, c]            (channel_scale)  */
} dfx_binop;

typedef enum dfx_op {
  DFX_OP_GEMM = 1,     /* grouped implicit-GEMM conv / dense (tcgen05)      */
  DFX_OP_SPLITK = 2,   /* split-K reduction + epilogue                     */
  DFX_OP_DWCONV = 3,   /* depthwise conv + epilogue                        */
  DFX_OP_POOL = 4,     /* max / avg pool, padded                           */
  DFX_OP_GAP = 5,      /* global average pool                              */
  DFX_OP_EW = 6,       /* affine/act/add/scale/copy on NHWC views          */
  DFX_OP_IN = 7,       /* fp32 CHW samples -> bf16 NHWC                    */
  DFX_OP_OUT = 8,      /* bf16 NHWC -> fp32 samples in logical CHW order   */
  DFX_OP_SE = 9,       /* squeeze-excitation gate: GAP -> FC -> act -> FC -> gate,
                          one 8-CTA cluster per image sharing data over DSMEM */
  DFX_OP_LN = 10,      /* layer norm over channels of token rows (+ token select) */
  DFX_OP_TOKENS = 11,  /* patch grid -> [class token; patches] + pos_embedding */
  DFX_OP_ATTN = 12,    /* multi-head softmax attention over packed q|k|v rows */
  DFX_OP_DWSE = 13,    /* depthwise conv + BN/act -> squeeze-excitation gate -> channel
                          scale, one cluster per image (an MBConv block's middle) */
  DFX_OP_GATE = 14     /* one thread waits until *flag != 0, then clears it: a member's
                          input has landed (dfx_execute_gated) */
} dfx_op;

typedef enum dfx_dtype {
  DFX_BF16 = 0,        /* bfloat16 storage, kind::f16 MMA with BF16 operands */
  DFX_F16 = 1,         /* IEEE half storage (saturating stores), F16 operands */
  /* Split precision: every value stored as two 16-bit planes x = hi + lo
   * (hi = rn(x), lo = rn(x - hi)); a view's pitch spans both planes of a pixel,
   * the lo plane of channel c sits pitch/2 elements after the hi one.  GEMMs
   * accumulate hi*hi + lo*hi + hi*lo on the tensor core (fp32); weights are
   * packed [hi rows; lo rows].  The accurate mode (fp32-class logits). */
  DFX_BF16X2 = 2,
  DFX_F16X2 = 3
} dfx_dtype;

/* A 16-bit NHWC view: element (n, h, w, c) at base[((n*H + h)*W + w)*pitch + coff + c].
 * Every view of one launch has the same dtype. */
typedef struct dfx_view {
  void* base;
  int32_t n, h, w, c;
  int32_t pitch, coff;
  int32_t dtype, _pad;
} dfx_view;

/* Epilogue shared by GEMM / split-K / depthwise / elementwise:
 *   v = x * alpha[c] + beta[c]   (alpha/beta NULL -> identity)
 *   v = act1(v)
 *   v = v (+|*) other            (binop)
 *   v = act2(v)
 * then rounded to bf16 and stored. */
typedef struct dfx_epilogue {
  const float* alpha;
  const float* beta;
  int32_t act1, act2, binop, _pad;
  dfx_view other;
} dfx_epilogue;

/* One implicit-GEMM problem (conv2d groups=1, or dense as a 1x1-output conv).
 *   M = output pixels (n, p, q), tiled as tn x tp x tq <= 128 rows
 *   N = output channels, tiles of bn (multiple of 16, <= 256)
 *   K = r * s * ceil(cin / cb) * cb, consumed in sub-blocks of cb channels
 * tmap_a / tmap_b are CUtensorMap objects written by dfx_tmap_act /
 * dfx_tmap_weights.  Filled by the host, uploaded to device memory. */
typedef struct __attribute__((aligned(64))) dfx_gemm_desc {
  uint64_t tmap_a[16];
  uint64_t tmap_b[16];
  int32_t n, p, q;                 /* output extents */
  int32_t tn, tp, tq;              /* M tile extents */
  int32_t mt_n, mt_p, mt_q;        /* M tiles along n, p, q */
  int32_t nt;                      /* N tiles */
  int32_t r, s, stride_h, stride_w, pad_h, pad_w;
  int32_t cb;                      /* channel block: 16, 32 or 64 */
  int32_t cblocks;                 /* ceil(cin / cb) */
  int32_t ksteps;                  /* r * s * cblocks */
  int32_t kpack;                   /* 64 / cb sub-blocks per pipeline stage */
  int32_t stages;                  /* ceil(ksteps / kpack) */
  int32_t splits;                  /* split-K factor (1 = fused epilogue) */
  int32_t stages_per_split;
  int32_t bn;                      /* N tile width */
  int32_t cout;
  int32_t tile_begin;              /* first blockIdx.x of this problem */
  int32_t tiles;                   /* mt_n*mt_p*mt_q*nt*splits */
  int32_t m2;                      /* 1: the CTA covers M tiles 2i and 2i+1, sharing each B stage */
  dfx_view out;                    /* bf16 output view (n, p, q, cout) */
  dfx_epilogue epi;
  float* ws;                       /* split-K workspace [splits][n*p*q][nt*bn] */
  uint32_t* counters;              /* split-K arrival counters, one per output tile, zeroed
                                      once; the last-arriving CTA of a tile reduces all splits
                                      in split order (deterministic) and resets its counter */
  /* A-operand prologue transform (1x1 convs, r = s = 1, no padding): every A tile
   * is rewritten in shared memory before the MMA reads it, fusing the producer
   * elementwise node into the GEMM:
   *   pre_mode 1: a = act(a * pre_scale[c] + pre_shift[c])   (fp32 vectors, >= cblocks*cb
   *               entries; DenseNet's pre-activation BN + ReLU)
   *   pre_mode 2: a = a * gate[n][c], gate 16-bit at pre_scale + n*pre_pitch + c
   *               (the squeeze-excitation channel scale before a projection conv) */
  const void* pre_scale;
  const float* pre_shift;
  int32_t pre_mode, pre_act, pre_cin, pre_pitch;
  /* Depthwise epilogue (dw_k > 0): the CTA holds the whole
   * GEMM output map (n, p, q) for its bn channels, so the consumer depthwise
   * conv (square dw_k x dw_k, stride dw_s, padding dw_pad; fp32 taps
   * [dw_k*dw_k][cout]) runs on it in shared memory: the GEMM output (after
   * `epi`, rounded to 16 bit exactly as when stored) never reaches HBM, and
   * `out` is the depthwise OUTPUT view, written as act(acc * dw_alpha + dw_beta).
   * Two M tiles split along p (mt_p == 2, m2 == 0) run as a 2-CTA cluster: each
   * CTA drains its own rows and reads the peer's rows over DSMEM. */
  const float* dw_w;
  const float* dw_alpha;
  const float* dw_beta;
  int32_t dw_k, dw_s, dw_pad, dw_act;
  /* Squeeze-excitation after the depthwise epilogue (dw_k > 0, se != NULL; device
   * pointer): the CTAs keep their depthwise outputs in shared memory, pool their
   * channels, add their fc1 partial sums into se->scratch, meet at ONE grid-wide
   * barrier (se->sync), form the hidden vector, their channels' gates, and store
   * x * gate to `out` (the SE's channel_scale output): the SE launch disappears. */
  const struct dfx_se_fuse* se;
} dfx_gemm_desc;

/* Squeeze-excitation fused into a depthwise-epilogue GEMM (dfx_gemm_desc.se). */
typedef struct dfx_se_fuse {
  const void* w1;                      /* fc1^T [c][cr], 16-bit (split: [hi; lo] blocks) */
  const float* b1;                     /* may be NULL */
  const void* w2;                      /* fc2 [c][cr], 16-bit (split: [hi; lo]) */
  const float* b2;                     /* may be NULL */
  float* scratch;                      /* [N tiles][n][cr] fp32 fc1 partial sums */
  uint32_t* sync;                      /* {arrivals, epoch}, zeroed once */
  float* pooled;                       /* mode 1: [n][c] channel means out */
  int32_t c, cr, act1, act2;
  int32_t ctas;                        /* CTAs that meet at the barrier (the grid) */
  int32_t mode;                        /* 0: the whole SE (above); 1: squeeze only -- the
                                          depthwise outputs are stored as usual and the CTA
                                          writes its channels' means to `pooled` for the
                                          SE launch that follows (dfx_se_params.pooled) */
  int32_t _pad[2];
} dfx_se_fuse;

/* Kernel parameter of one GEMM launch.  A single problem travels inline
 * (desc0, ndesc == 1): descriptor and tensor maps then sit in kernel-parameter
 * space, read at launch without a global-memory round trip.  A grouped launch
 * (ndesc > 1) reads `descs` from device memory, sorted by tile_begin. */
typedef struct __attribute__((aligned(64))) dfx_gemm_launch {
  const dfx_gemm_desc* descs;      /* device pointer, ndesc entries (ndesc > 1) */
  int32_t ndesc;
  int32_t total_tiles;             /* grid size */
  int32_t bn_max;                  /* sizes smem / TMEM */
  int32_t dtype;                   /* dfx_dtype of every problem */
  int32_t nslots;                  /* smem pipeline depth, 2..8 */
  int32_t flags;                   /* bit 0: read desc0 from `descs` (debug);
                                      bit 1: persistent kernel (1-2 CTAs/SM walk the
                                      tile list, a ring of TMEM accumulators; one
                                      problem, no split-K, no m2);
                                      bit 2: smem-transposed epilogue drain (A/B only);
                                      bit 3: cluster split-K -- the desc0.splits (2..8)
                                      CTAs of an output tile form a cluster and reduce
                                      their partials over DSMEM (no workspace, no
                                      splitk launch);
                                      bit 5: weight tiles with an L2 evict_first
                                      policy (each read by <= 2 CTAs) */
  int32_t m2;                      /* any problem has m2 = 1 (sizes smem / TMEM) */
  int32_t se_cr;                   /* desc0.se != NULL: its hidden width (sizes smem) */
  int32_t max_ctas;                /* persistent launch: grid cap (0 = 1-2 CTAs per SM) */
  uint32_t l2_pf_units;            /* sizes of l2_pf[0] | l2_pf[1] << 16, in 256-B units */
  const void* l2_pf[2];            /* weights of the member's next launches: each CTA
                                      prefetches its slice into L2 before its dependency
                                      resolves (batch-1 weight streaming off the chain) */
  dfx_gemm_desc desc0;             /* the problem when ndesc == 1 */
} dfx_gemm_launch;

typedef struct dfx_splitk_params {
  const float* ws;
  int32_t splits, pixels, cout, ldw;   /* ws row stride (nt*bn) */
  dfx_view out;                        /* out.n*out.h*out.w == pixels */
  dfx_epilogue epi;
} dfx_splitk_params;

typedef struct dfx_dwconv_params {
  dfx_view in, out;                    /* out.c == in.c */
  const float* weight;                 /* [kh*kw][c] fp32 */
  int32_t kh, kw, stride_h, stride_w, pad_h, pad_w;
  dfx_epilogue epi;
} dfx_dwconv_params;

typedef struct dfx_pool_params {
  dfx_view in, out;
  int32_t kh, kw, stride_h, stride_w, pad_h, pad_w;
  int32_t is_max, count_include_pad;
} dfx_pool_params;

typedef struct dfx_gap_params {
  dfx_view in, out;                    /* out.h == out.w == 1 */
} dfx_gap_params;

typedef struct dfx_ew_params {
  dfx_view in, out;                    /* same n, h, w, c */
  dfx_epilogue epi;
} dfx_ew_params;

/* kh == 0: out[n, h, w, c] = src[n][c][h][w]  (out.c == c, out.h == h, out.w == w).
 * kh > 0 (im2col of the entry conv -- a stem with few input channels, or a
 * patchify conv -- which then runs as a 1x1 GEMM over kh*kw*c channels):
 * out[n, y, x, (r*kw + s)*c + ci] = src[n][ci][y*sh - ph + r][x*sw - pw + s]
 * (0 outside the image); out.h, out.w are the conv's output size. */
typedef struct dfx_in_params {
  const float* src;                    /* n samples, each c*h*w fp32 in CHW order */
  dfx_view out;
  int32_t kh, kw, sh, sw, ph, pw;      /* entry conv geometry (kh = 0: plain copy) */
  int32_t c, h, w;                     /* source sample dims */
  int32_t split;                       /* > 0 (im2col only): out.c = 3*split channels written
                                          as [x_hi | x_hi | x_lo], blocks of `split` channels
                                          (kh*kw*c real ones, zero padded); x = x_hi + x_lo,
                                          both 16-bit: the split-precision stem GEMM */
} dfx_in_params;

typedef struct dfx_out_params {
  dfx_view in;
  float* dst;                          /* n samples, each c*h*w fp32 in CHW order */
} dfx_out_params;

/* gate[n, c] = act2(b2[c] + sum_j w2[c][j] * act1(b1[j] + sum_k w1[j][k] * mean_hw x[n, :, :, k]))
 * (global_avg_pool -> dense -> act -> dense -> act of the reference IR).
 * apply = 0: out = gate (n, 1, 1, c);  apply = 1: out = x * gate (n, h, w, c), i.e. the
 * following channel_scale is fused (each cluster CTA scales its channel slice).
 * apply bit 1 (value 2): read the FC weights from global memory instead of staging
 * each CTA's slice in shared memory (large batches); with bit 2 (value 4) as well,
 * stage only the fc1 slices (split-precision slices of both FCs beyond the budget).
 * w1 [cr][c], w2 [c][cr]: 16-bit, dtype of the views, row-major. */
typedef struct dfx_se_params {
  dfx_view in;                         /* x (n, h, w, c) */
  dfx_view out;                        /* gate (n, 1, 1, c), or x * gate (n, h, w, c) */
  const void* w1;
  const float* b1;                     /* may be NULL */
  const void* w2;
  const float* b2;                     /* may be NULL */
  int32_t cr, act1, act2, apply;
  const float* pooled;                 /* non-NULL: [n][c] channel means of `in`, written by the
                                          depthwise-epilogue GEMM before it (dfx_se_fuse mode 1):
                                          no pooling pass over x */
} dfx_se_params;

/* Depthwise conv (+ epi: folded BN, act) -> SE gate (as dfx_se_params) -> scale, in
 * ONE launch: a 16-CTA cluster per image, CTA r owns a channel slice; the slice's
 * depthwise output stays in shared memory (16-bit, rounded as a stored tensor would
 * be), is pooled there, and is scaled by the gate on the way out.
 * out[n,p,q,c] = dw[n,p,q,c] * gate[n,c]. */
typedef struct dfx_dwse_params {
  dfx_view in, out;                    /* out.c == in.c; out spatial = dw output */
  const float* dw_weight;              /* [kh*kw][c] fp32 taps */
  int32_t kh, kw, stride_h, stride_w, pad_h, pad_w;
  dfx_epilogue dw_epi;                 /* affine + act1 only */
  const void* w1;                      /* fc1^T [c][cr], 16-bit */
  const float* b1;
  const void* w2;                      /* fc2 [c][cr], 16-bit */
  const float* b2;
  int32_t cr, act1, act2, staged;      /* staged: FC slices in smem (small batch) */
} dfx_dwse_params;

/* Token tensors (ViT) are views with h = 1, w = L tokens, c = channels.
 * out[n, 0, t, c] = norm ? (x - mean_t) * rsqrt(var_t + eps) * gamma[c] + beta[c]
 *                        : x                     with x = in[n, 0, t, c],
 * for t < out.w <= in.w (out.w = 1 after "layernorm -> select_token 0");
 * mean/var over the c channels of row t (biased variance). */
typedef struct dfx_ln_params {
  dfx_view in;
  dfx_view out;
  const float* gamma;
  const float* beta;
  float eps;
  int32_t norm, _pad[2];
} dfx_ln_params;

/* out[n, 0, 0, c] = cls[c] + pos[0][c];
 * out[n, 0, 1 + h*W + w, c] = in[n, h, w, c] + pos[1 + h*W + w][c]. */
typedef struct dfx_tokens_params {
  dfx_view in;                         /* patch grid (n, H, W, c) */
  dfx_view out;                        /* tokens (n, 1, 1 + H*W, c) */
  const float* cls;                    /* [c] */
  const float* pos;                    /* [1 + H*W][c] */
} dfx_tokens_params;

/* qkv (n, 1, L, 3C) packed q | k | v (column blocks); per head h (columns
 * h*d .. h*d + d - 1 of each block, d = C / heads, d == 64):
 * out[n, 0, :, h*d : h*d + d] = softmax(q_h k_h^T * scale) v_h. */
typedef struct dfx_attn_params {
  dfx_view qkv;
  dfx_view out;                        /* (n, 1, L, C) */
  int32_t heads;
  float scale;
  int32_t _pad[2];
} dfx_attn_params;

/* Input gate of one member (DFX_OP_GATE): the member's branch of the fused graph
 * starts when its input is on the device -- the host sets the flag (an H2D of a
 * pinned 1 on the copy stream, after the member's input copy) -- so the graph is
 * launched BEFORE the inputs are gathered and each member starts as soon as its own
 * input lands.  The kernel traps after ~4 s instead of hanging the GPU. */
typedef struct dfx_gate_params {
  uint32_t* flag;                      /* device word, 0 = closed */
  int32_t _pad[2];
} dfx_gate_params;

/* ---- library / device ------------------------------------------------- */
const char* dfx_last_error(void);
int dfx_abi_version(void);
/* sizeof() of a struct declared here, by name ("dfx_gemm_desc", ...); -1 if
 * unknown.  Lets bindings verify their mirrored layouts at load time. */
int dfx_sizeof(const char* name);
/* Selects the device on the calling thread, checks sm_100, sets kernel
 * attributes.  Idempotent. */
int dfx_init(int device);
int dfx_device_info(int device, int* sm_count, int* cc_major, int* cc_minor,
                    size_t* total_mem);
int dfx_mem_info(size_t* free_bytes, size_t* total_bytes);
/* Logits that came out non-finite (inf / NaN) on `device` since the last reset:
 * fp16 stores do not saturate, so an activation overflow anywhere in a member
 * reaches its output as inf / NaN and is counted here by the output kernel
 * (reset != 0: read and zero). */
int dfx_nonfinite_count(int device, unsigned long long* count, int reset);

/* NVTX ranges (header-only NVTX3: free unless a profiler is attached).  The library
 * marks swap-in, graph instantiation and execution itself; the Python layer marks
 * fuse_models / load_fused / swap_subgraph with these. */
int dfx_nvtx_range_push(const char* msg);
int dfx_nvtx_range_pop(void);

/* ---- memory ------------------------------------------------------------ */
int dfx_malloc(void** dptr, size_t bytes);
int dfx_free(void* dptr);
int dfx_memset(void* dptr, int value, size_t bytes, void* stream);
/* Weight arenas: allocation from a per-device stream-ordered pool that keeps
 * freed pages mapped (unbounded release threshold), so swap-out / swap-in
 * cycles do not remap physical memory (the cudaMalloc phase of simulate_load,
 * costmodel.py:297-300).  dfx_pool_trim returns mapped-but-free pages to the
 * driver down to keep_bytes. */
int dfx_pool_malloc(void** dptr, size_t bytes, void* stream);
int dfx_pool_free(void* dptr, void* stream);
int dfx_pool_trim(size_t keep_bytes);
/* Bytes the arena pool holds mapped (reserved) and hands out (used): peak-HBM
 * samples taken with cudaMemGetInfo account for the retained pages with it. */
int dfx_pool_stats(size_t* reserved, size_t* used);
int dfx_host_alloc(void** hptr, size_t bytes);          /* pinned */
int dfx_host_free(void* hptr);
int dfx_host_register(void* hptr, size_t bytes);
int dfx_host_unregister(void* hptr);
int dfx_memcpy_h2d(void* dst, const void* src, size_t bytes, void* stream);
int dfx_memcpy_d2h(void* dst, const void* src, size_t bytes, void* stream);
int dfx_memcpy_d2d(void* dst, const void* src, size_t bytes, void* stream);

/* Swap-in (replaces the modelled memcpy phase of simulate_load,
 * costmodel.py:277-305): ONE device allocation and ONE cudaMemcpyAsync of a
 * packed weight arena from pinned host memory. */
int dfx_arena_upload(const void* pinned_host, size_t bytes, void** dev_arena, void* stream);

/* ---- streams / events --------------------------------------------------- */
int dfx_stream_create(void** stream);
int dfx_stream_destroy(void* stream);
int dfx_stream_sync(void* stream);                       /* synchronises */
int dfx_event_create(void** ev);
int dfx_event_destroy(void* ev);
int dfx_event_record(void* ev, void* stream);
int dfx_event_elapsed(void* start, void* stop, float* ms); /* synchronises on stop */

/* ---- tensor maps (TMA descriptors, 128 B written to out128) -------------- */
/* Activation view as a 4-D tiled map (c, w, h, n); box (cb, tq*sw, tp*sh, tn)
 * with element strides (1, sw, sh, 1); 16/32/64-channel boxes use the
 * 32/64/128-byte swizzle; out-of-bounds elements (padding, channel tails)
 * read as zero. */
int dfx_tmap_act(void* out128, const dfx_view* v, int cb, int tq, int tp, int tn,
                 int stride_w, int stride_h);
/* Packed weight matrix [rows][k] of `dtype` (k contiguous); box (cb, bn). */
int dfx_tmap_weights(void* out128, const void* base, int rows, int k, int cb, int bn, int dtype);

/* ---- kernels: direct launch on a stream (tests, eager mode) ------------- */
int dfx_launch(int op, const void* params, size_t params_size, void* stream);

/* ---- CUDA graph of the fused DAG --------------------------------------- */
/* Nodes are kernel launches with explicit dependencies; the executor
 * instantiates one cudaGraphExec per (DAG, batch signature, instance). */
int dfx_graph_create(void** graph);
int dfx_graph_add(void* graph, int op, const void* params, size_t params_size,
                  const int* deps, int ndeps, int* node_id);
/* Scheduling priority of one node (cudaLaunchAttributePriority; lower = more
 * urgent, within cudaDeviceGetStreamPriorityRange).  The executor raises the
 * members with the longest dependent chains so the fused DAG's critical path
 * is not delayed by the other branches' CTAs.  *range_out (optional) receives
 * {least, greatest}. */
int dfx_graph_set_priority(void* graph, int node_id, int priority, int* range_out);
int dfx_graph_instantiate(void* graph);
int dfx_graph_launch(void* graph, void* stream);
int dfx_graph_node_count(void* graph, int* count);
int dfx_graph_destroy(void* graph);

/* End-to-end query (execute_fused, fuse.py:268-291): H2D of the packed fp32
 * inputs, one graph launch, D2H of the packed fp32 outputs, stream sync. */
int dfx_execute(void* graph, const void* host_in, void* dev_in, size_t in_bytes,
                void* host_out, const void* dev_out, size_t out_bytes, void* stream);
/* The same query with the inputs gathered from `nsrc` separate host arrays
 * (one per member or sample, packed in list order): chunks are copied into the
 * pinned staging buffer `host_in` on a pool of host threads
 * (DFX_STAGE_THREADS, default half the cores) while the calling thread issues
 * the H2D of every completed prefix, so the DMA overlaps the host copy.
 * Re-entrant on distinct graphs/streams/staging buffers: only the staging
 * phase uses the shared pool (a caller that finds it busy copies on its own
 * thread); the graph launch and the stream sync run without any global lock. */
int dfx_execute_gather(void* graph, const void* const* srcs, const size_t* sizes, int nsrc,
                       void* host_in, void* dev_in, void* host_out, const void* dev_out,
                       size_t out_bytes, void* stream);

/* End-to-end query with per-member gates (fuse.py execute_fused): the graph (whose
 * members each start with a DFX_OP_GATE node on flags[m]) is launched on `stream`
 * FIRST; then members are gathered into the pinned staging in `order` (the longest
 * chain first), and for each one, once all its sources are copied (thread pool as
 * dfx_execute_gather), its byte range is sent H2D on `copy_stream` followed by its
 * flag (a 4-byte H2D from the pinned word `one`).  Sources are listed member by
 * member in `order`; src_member[i] names the member of source i; member_off /
 * member_bytes give each member's range of host_in / dev_in.  Then the D2H of the
 * outputs on `stream` and a stream sync. */
int dfx_execute_gated(void* graph, const void* const* srcs, const size_t* sizes, const int* src_member, int nsrc,
                      const size_t* member_off, const size_t* member_bytes, int nmembers, void* host_in,
                      void* dev_in, uint32_t* flags, const uint32_t* one, void* host_out, const void* dev_out,
                      size_t out_bytes, void* stream, void* copy_stream);

#ifdef __cplusplus
}
#endif
#endif /* DFX_H */
