/*
 * b2conv — C ABI of the B200-native convolution hot path.
 *
 * This header is the drop-in boundary.  In the reference (cuclgen, pure Python)
 * the device boundary is the call
 *
 *     backend.run_kernel(ir, launch, buffers, meta, engine, thread_order)
 *         -> (buffers, CostReport)                      cuclgen/backend.py:1104-1133
 *
 * made from runner.execute_node (cuclgen/runner.py:73-106, the call at :103)
 * and from runner.run_graph (runner.py:228).  Its arguments are a kernel IR
 * produced by a Variant generator (variants.py:201-220) for one conv node
 * described by ConvParams (frontend.py:56-65) on an input DimsSpec
 * img:chan:y:x (ndarray.py:74-88), plus caller-owned buffers keyed
 * in/filts/bias/out (runner.py:32-36).  The output buffer is written in place.
 *
 * Here the same call is a plain C function over device pointers: the op is a
 * b2c_conv_desc, the variant + TuneParams are a b2c_tune, and the CostReport's
 * wall_ns becomes CUDA-event device time (b2c_conv_time).  All tensors are
 * fp32, dense row-major, canonical layouts: x NCHW (img:chan:y:x), w OIHW
 * (out_chan:in_chan:y:x), bias (out_chan), y NCHW.  No torch types cross this
 * boundary; the Python host mirror (paper_1611_06945_b200/backend.py) binds it
 * with ctypes, and INTEGRATION.md shows the binding a maintainer of the
 * reference would add.
 *
 * Error convention (mirrors cuclgen's exception families):
 *   B2C_OK            0  success
 *   B2C_INAPPLICABLE  1  variant cannot run this op      (variants.Inapplicable, variants.py:31)
 *   B2C_BAD_ARGS      2  inconsistent descriptor/buffers  (oracle.ShapeMismatch, oracle.py:19;
 *                                                          frontend.GraphError, frontend.py:47)
 *   B2C_CUDA_ERROR    3  CUDA runtime / launch failure    (backend.InterpError family, backend.py:61-82)
 *   B2C_UNSUPPORTED   4  precision/feature not built      (CuclgenError, errors.py:1-2)
 * b2c_last_error() returns a thread-local message for the last failing call.
 *
 * Threading: every entry point is re-entrant; launches go to the stream given.
 * The only global state is a mutex-protected per-device attribute cache and
 * the split-K semaphore pool inside caller-provided workspace.
 */
#ifndef B2CONV_H
#define B2CONV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define B2C_OK 0
#define B2C_INAPPLICABLE 1
#define B2C_BAD_ARGS 2
#define B2C_CUDA_ERROR 3
#define B2C_UNSUPPORTED 4

/* Variant ids.  The first four carry the reference's variant names
 * (VARIANTS, variants.py:830-832; ranks at :227, :283, :333, :388);
 * B2C_VAR_UMMA is the B200 tensor-core implicit GEMM. */
#define B2C_VAR_SIMPLE 0 /* "conv_simple": one thread per output, fmaf over ic,ky,kx  (variants.py:223-276) */
#define B2C_VAR_TILED 1  /* "conv_tiled" : register/thread-blocked FFMA implicit GEMM (variants.py:376-685) */
#define B2C_VAR_1X1 2    /* "conv_1x1"   : k=1,pad=0 tcgen05 GEMM                     (variants.py:279-325) */
#define B2C_VAR_FC 3     /* "conv_fc"    : whole-image filter, weight-streaming GEMM  (variants.py:328-373) */
#define B2C_VAR_UMMA 4   /* "conv_umma"  : tcgen05/TMEM 3xTF32 implicit GEMM, k x k      (new, B200)       */
#define B2C_VAR_WINO 6   /* "conv_wino"  : Winograd F(2x2,3x3) for 3x3 / stride-1 / pad <= 1 convs, fp32-exact:
                              input transform V = B^T d B, 16 batched tcgen05 3xTF32 GEMMs against the
                              filter transform U = G g G^T (made by b2c_conv_prepare), output transform
                              A^T M A + bias + ReLU (the paper's gap to cuDNN on 3x3).
                              tile_n 64|128|192, split_k (0 = stream-K), swap_ab; 3 launches */
#define B2C_VAR_FC_STREAM 5 /* "conv_fc_stream": fp32 FFMA weight streaming for ConvFC (HBM-bound at small
                              batch; reads w once).  kb = 1 (batch <= 8): warps split K, mnb0 = warps per
                              block 2|4|8, mnt1 = rows per block 2|4|8; kb = 2 (batch <= 32): x staged in
                              shared memory, mnb0 = warps 4|8, mnt1 = rows per warp 1|2|4 */

/* Precision modes. */
#define B2C_PREC_FP32 0 /* fp32-exact: FFMA, or 3xTF32 split on the tensor cores */
#define B2C_PREC_BF16 1 /* bf16 operands, fp32 accumulate (separately stated tolerance) */
#define B2C_PREC_FP8 2  /* e4m3 operands (round to nearest, saturating at +-448, no scaling), fp32
                           accumulate: tcgen05 kind::f8f6f4 (separately stated tolerance) */

/* One convolution, the C form of (ConvParams, input DimsSpec, fused_activation):
 * ConvParams(ksz, stride, pad, out_chans) frontend.py:56-65; output extent
 * window_out frontend.py:441-442; OpNode.fused_activation frontend.py:100. */
typedef struct b2c_conv_desc {
    int32_t n, c, h, w; /* input img:chan:y:x */
    int32_t k;          /* out_chans */
    int32_t r;          /* ksz (square) */
    int32_t stride, pad;
    int32_t oh, ow; /* must equal (h + 2*pad - r)/stride + 1 (and same for w) */
    int32_t act;    /* 0 none, 1 relu ("(ov > 0) ? ov : 0", variants.py:164) */
    int32_t prec;   /* B2C_PREC_*: 0 fp32-exact, 1 bf16, 2 fp8 (e4m3) */
} b2c_conv_desc;

/* Variant + tuning knobs, the C form of TuneParams (variants.py:39-91).
 * FFMA variants read mnt/mnb/kb/vw with the reference's meaning (register
 * block, thread block, k unroll, vector width).  The tcgen05 variants read
 * tile_n (MMA N), stages (TMA kernel: CTAs per SM, 1 or 2 [2 needs tile_n <= 64];
 * gather kernel: < 0 disables the cooperative L2 prefetch of x/w
 * that small ops get by default), split_k, swap_ab (0: M = output pixels, N =
 * out_chans; 1: M = out_chans, N = output pixels) and drain (K blocks of 32
 * accumulated in one TMEM chunk before it is drained into fp32 registers;
 * 0 = default 4 — bounds the tensor-core accumulation error, see k_umma.cuh).
 * prepared != 0 asserts the workspace already holds this filter tensor packed
 * by b2c_conv_prepare (filters are constant per op; the pack is cached per
 * (filter tensor, variant) as SURVEY.md §8(b) specifies); prepared == 0 makes
 * b2c_conv_fwd pack the filters itself first (one extra launch). */
typedef struct b2c_tune {
    int32_t variant;
    int32_t mnt0, mnt1, mnb0, mnb1, kb, vw;
    int32_t tile_n, stages, split_k, swap_ab, drain, prepared;
    int32_t tma; /* tcgen05 variants: 0 = operands gathered by producer warps from NCHW (k_umma);
                    1 = TMA-fed persistent kernel (k_tconv): im2col TMA on an NHWC copy of x made
                    in the workspace by the same call (first layers, C <= 4: x-window boxes on a
                    padded NHWC4 copy), or 2-D TMA of raw x / w for conv_fc;
                    2 = as 1, but 2-D tiles for 1x1/stride-1 convs and 8-tap 16-byte boxes for C <= 4;
                    3 = 1x1 / stride 1 / pad 0 convs read straight from NCHW x (3-D TMA box
                        [32 ch][128 px] per K block; h*w*4 bytes a multiple of 16; no re-layout launch);
                    4 = k x k stride-1 convs read straight from NCHW x (4-D TMA box of whole output
                        rows, x start rounded down to 16 bytes; input width a multiple of 4);
                    5 = bf16 mode: a bf16 NHWC copy of x and SS MMAs (64-channel K blocks, no split pass);
                    6 = first layers (C <= 4, stride 2..4): space-to-depth -- the conv runs as an
                        R' x R' stride-1 conv (R' = ceil(R/S)) over a C*S*S-channel copy of x with
                        re-arranged filters, on the im2col path of tma=1 */
    int32_t cluster; /* TMA kernel: 2 = CTA pairs (thread-block clusters) take neighbouring pixel tiles of the
                        same filter tile and multicast each filter stage to both (half the filter L2 traffic);
                        3 = 2-SM UMMA pairs: the same two pixel tiles as ONE tcgen05.mma.cta_group::2 of
                        M = 256 issued by the leader CTA, each CTA holding half of the filter tile's rows
                        (half the filter L2 and shared-memory traffic per CTA; tile_n 64 | 128 | 192,
                        fp32-exact mode, tma 1 | 3 | 4);
                        4 = split-K clusters: the split_k (2..8) CTAs of an output tile form one thread-block
                        cluster and the leader sums the partials over distributed shared memory (no global
                        partials / tickets; tile_n 32 | 64 conv tiles with tma 1 | 3 | 4, or the fc swap tile);
                        0/1 = single CTAs.  Pairs need swap_ab = 0 and a conv (not fc) variant. */
} b2c_tune;

/* 0 when `tune` can run `d`; otherwise B2C_INAPPLICABLE / B2C_BAD_ARGS with a
 * reason copied into reason[0..n) (Variant.applies, variants.py:206-210). */
int b2c_conv_applies(const b2c_conv_desc* d, const b2c_tune* t, char* reason, size_t n);

/* Pack the filters w (OIHW fp32) into the workspace in the layout the tcgen05
 * variants stream with cp.async.bulk: per (filter tile, K block) the exact
 * shared-memory image [raw | lo = w - trunc_tf32(w)].  No-op (B2C_OK) for the
 * FFMA variants.  This is the B200 form of ConvTiled.required_formats
 * (variants.py:416-424: K-major padded filters) + the conversion execute_node
 * applies (runner.py:96-98), done once per filter tensor instead of per call.
 * Synchronises `stream` before returning (a one-time setup call), so that
 * launches with prepared != 0 may read the pack without stream ordering. */
int b2c_conv_prepare(const b2c_conv_desc* d, const b2c_tune* t, const float* w, void* workspace,
                     size_t ws_bytes, void* stream);

/* Device workspace bytes b2c_conv_fwd needs (packed filters + split-K partials + semaphores
 * + the NHWC copy of x for the TMA conv path).
 * The workspace MUST be zero-filled once before first use (e.g. cudaMemset after
 * cudaMalloc): the split-K / stream-K tickets in it are counted up by the
 * contributing CTAs and reset to zero by the last one, so garbage there makes
 * the last-arriver reduction misfire and the output silently wrong.  One
 * workspace per concurrently running launch (tickets are per workspace). */
size_t b2c_conv_workspace(const b2c_conv_desc* d, const b2c_tune* t);

/* y = act(conv(x, w) + bias), written in place into caller-allocated y
 * (run_kernel semantics, backend.py:1104-1133).  `stream` is a cudaStream_t
 * (NULL = legacy default stream).  Asynchronous: errors from the kernel
 * itself surface on the next synchronising call. */
int b2c_conv_fwd(const b2c_conv_desc* d, const b2c_tune* t, const float* x, const float* w,
                 const float* bias, float* y, void* workspace, size_t ws_bytes, void* stream);

/* CostReport.wall_ns analogue (backend.py:108, :1125-1132): launches the
 * variant `warmup` times, then times `reps` launches with CUDA events, each
 * optionally preceded by an L2 flush (l2_flush != 0), and returns the median
 * per-launch milliseconds.  Synchronises the stream. */
int b2c_conv_time(const b2c_conv_desc* d, const b2c_tune* t, const float* x, const float* w,
                  const float* bias, float* y, void* workspace, size_t ws_bytes, void* stream,
                  int warmup, int reps, int l2_flush, float* median_ms);

/* End-to-end call over HOST buffers: copies x, w, bias host->device, runs the
 * variant, copies y device->host, all on `stream`, using device scratch the
 * caller provides (dev_scratch of scratch_bytes >= b2c_conv_host_scratch()).
 * This is execute_node (runner.py:73-106) with host NdArrays in and out.
 * dev_scratch may be uninitialised device memory (plain cudaMalloc): the call
 * zeroes the ticket / barrier words of the workspace part on `stream` itself
 * before the launch, and packs the filters it just copied (tune.prepared is
 * ignored).  Host buffers should be pinned for asynchronous copies. */
size_t b2c_conv_host_scratch(const b2c_conv_desc* d, const b2c_tune* t);
int b2c_conv_fwd_host(const b2c_conv_desc* d, const b2c_tune* t, const float* hx, const float* hw,
                      const float* hbias, float* hy, void* dev_scratch, size_t scratch_bytes,
                      void* stream);

/* FLOPs the reference counts for this op: 2*k^2*ic*oc*oy*ox*b
 * (frontend.flops_of, frontend.py:499-514). */
int64_t b2c_conv_flops(const b2c_conv_desc* d);

/* Compulsory HBM bytes: 4*(|x| + |w| + |bias| + |y|). */
int64_t b2c_conv_bytes(const b2c_conv_desc* d);

/* Number of kernel launches one b2c_conv_fwd issues for this (d, t). */
int b2c_conv_launches(const b2c_conv_desc* d, const b2c_tune* t);

/* CTAs of the main conv kernel b2c_conv_fwd launches for (d, t) (0 if inapplicable):
 * with the runtime (the SM-time an op occupies) it is what a concurrent schedule of
 * independent ops packs onto the 148 SMs. */
int b2c_conv_grid(const b2c_conv_desc* d, const b2c_tune* t);

/* Thread-local message for the last non-zero status. */
const char* b2c_last_error(void);

/* Device memory / stream helpers for callers without a CUDA runtime binding of
 * their own (the reference is numpy-only; integration/cuclgen_b200.py binds
 * these with ctypes).  b2c_device_alloc returns zero-filled device memory
 * (cudaMalloc + cudaMemset; NULL and b2c_last_error() on failure) — usable as
 * dev_scratch for b2c_conv_fwd_host or as a b2c_conv_fwd workspace. */
void* b2c_device_alloc(size_t bytes);
int b2c_device_free(void* p);
int b2c_stream_synchronize(void* stream); /* cudaStreamSynchronize; NULL = legacy default stream */

/* Library version string ("b2conv <semver> sm_100a"). */
const char* b2c_version(void);

/* ============================================================================
 * Whole-network forward: the non-conv node kinds.
 * In the reference these are further Variant generators whose kernels
 * runner.run_graph hands to run_kernel (runner.py:200-249): pool_max
 * (variants.py:688-741), activation (variants.py:744-775) and xpose
 * (variants.py:778-827).  Same conventions as the conv entry points: fp32,
 * caller-owned device buffers, asynchronous on `stream`, status codes above.
 * ========================================================================== */

/* Max pooling over img:chan:y:x (PoolParams, frontend.py:68-80): square window r,
 * stride, pad < r; out-of-range taps never win (ref_pool_max pads with -inf,
 * oracle.py:100-116).  oh/ow must equal window_out (frontend.py:441-442). */
typedef struct b2c_pool_desc {
    int32_t n, c, h, w;
    int32_t r, stride, pad;
    int32_t oh, ow;
} b2c_pool_desc;
int b2c_pool_max_fwd(const b2c_pool_desc* d, const float* x, float* y, void* stream);

/* y[i] = (x[i] > 0) ? x[i] : 0 for i < n (Activation "relu", variants.py:744-775;
 * ref_relu, oracle.py:119-121).  x == y (in place) is allowed. */
int b2c_relu_fwd(const float* x, float* y, int64_t n, void* stream);

/* Layout conversion (Xpose, variants.py:778-827 = ndarray.convert_format,
 * ndarray.py:232-253): output dims in output order; for output dim i the
 * same-named source dim has extent src_sizes[i] and element stride
 * src_strides[i].  Output is dense row-major over out_sizes; an index past the
 * source extent reads 0 (growth zero-pads), out_sizes smaller than src_sizes
 * crop. */
#define B2C_XPOSE_MAX_DIMS 8
typedef struct b2c_xpose_desc {
    int32_t ndim;
    int32_t reserved;
    int64_t out_sizes[B2C_XPOSE_MAX_DIMS];
    int64_t src_sizes[B2C_XPOSE_MAX_DIMS];
    int64_t src_strides[B2C_XPOSE_MAX_DIMS];
} b2c_xpose_desc;
int b2c_xpose(const b2c_xpose_desc* d, const float* x, float* y, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* B2CONV_H */
