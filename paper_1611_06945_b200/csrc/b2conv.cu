// b2conv C ABI: descriptor validation, variant applicability, dispatch,
// workspace sizing, CUDA-event timing and the host-buffer end-to-end call.
// See include/b2conv.h for the contract and the reference call it replaces
// (cuclgen/backend.py:1104-1133 run_kernel, via runner.execute_node
// runner.py:73-106).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/b2conv.h"
#include "common.cuh"
#include "k_ffma.cuh"
#include "k_umma.cuh"
#include "k_tma.cuh"
#include "k_fcs.cuh"
#include "k_wino.cuh"
#include "tconv_inst.cuh"

namespace b2c {
__device__ long long g_b2c_trace[256];  // phase trace of k_tconv CTA 0 (debug; TArgs.trace_buf points here)
}  // namespace b2c

using namespace b2c;


namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* where) {
    return fail(B2C_CUDA_ERROR, std::string(where) + ": " + cudaGetErrorString(e));
}

#define B2C_CUDA(call)                                     \
    do {                                                   \
        cudaError_t _e = (call);                           \
        if (_e != cudaSuccess) return cuda_fail(_e, #call); \
    } while (0)

int window_out(int in, int k, int s, int p) { return (in + 2 * p - k) / s + 1; }

int check_desc(const b2c_conv_desc* d) {
    if (!d) return fail(B2C_BAD_ARGS, "null descriptor");
    if (d->n < 1 || d->c < 1 || d->h < 1 || d->w < 1 || d->k < 1 || d->r < 1 || d->stride < 1 || d->pad < 0)
        return fail(B2C_BAD_ARGS, "bad conv params (need n,c,h,w,k,ksz,stride >= 1, pad >= 0)");
    const int oh = window_out(d->h, d->r, d->stride, d->pad);
    const int ow = window_out(d->w, d->r, d->stride, d->pad);
    if (oh < 1 || ow < 1) return fail(B2C_BAD_ARGS, "non-positive output dims");
    if (oh != d->oh || ow != d->ow)
        return fail(B2C_BAD_ARGS, "output extent inconsistent with params (window_out)");
    if (d->act != 0 && d->act != 1) return fail(B2C_BAD_ARGS, "act must be 0 (none) or 1 (relu)");
    const long long xin = (long long)d->n * d->c * d->h * d->w;
    const long long yout = (long long)d->n * d->k * oh * ow;
    const long long wk = (long long)d->k * d->c * d->r * d->r;
    if (xin >= (1ll << 31) || yout >= (1ll << 31) || wk >= (1ll << 31))
        return fail(B2C_UNSUPPORTED, "tensor exceeds 2^31 elements");
    if (d->prec != B2C_PREC_FP32 && d->prec != B2C_PREC_BF16 && d->prec != B2C_PREC_FP8)
        return fail(B2C_BAD_ARGS, "prec must be 0 (fp32), 1 (bf16) or 2 (fp8 e4m3)");
    return B2C_OK;
}

Geom make_geom(const b2c_conv_desc* d) {
    Geom g;
    g.N = d->n; g.C = d->c; g.H = d->h; g.W = d->w;
    g.OC = d->k; g.R = d->r; g.S = d->stride; g.P = d->pad;
    g.OH = d->oh; g.OW = d->ow;
    g.K = d->c * d->r * d->r;
    g.PQ = d->oh * d->ow;
    g.M = d->n * g.PQ;
    g.HW = d->h * d->w;
    g.RR = d->r * d->r;
    g.act = d->act;
    g.fPQ = FastDiv((uint32_t)g.PQ);
    g.fOW = FastDiv((uint32_t)g.OW);
    g.fRR = FastDiv((uint32_t)g.RR);
    g.fR = FastDiv((uint32_t)g.R);
    return g;
}

bool valid_bn(int bn) { return bn == 16 || bn == 32 || bn == 64 || bn == 96 || bn == 128 || bn == 192; }

// K order of the tcgen05 kernels: tap-major (3) when there are >= 32 input
// channels, flat (0) for first layers, flat contiguous (2) for conv_fc.
// K orders: 0 flat (ic,ky,kx) [gather kernel, C < 32]; 2 flat contiguous (fc);
// 3 tap-major, 32 channels per block; first layers (TMA kernel, C <= 4):
// 4 = 8 taps x 4 channels per block (tma=2), 5 = (filter row, 32-float
// x-window chunk) per block (tma=1).
int window_chunks(const b2c_conv_desc* d) { return (d->r * 4 + TM_BK - 1) / TM_BK; }
int kmode_for(const b2c_conv_desc* d, int variant, int tma) {
    if (variant == B2C_VAR_FC) return 2;
    if (tma == 5) return 6;  // bf16 NHWC copy: (tap, 64-channel block) per K block, SS MMAs
    if (tma && tma != 3 && tma != 4 && d->c <= 4) return tma == 2 ? 4 : 5;
    if (variant == B2C_VAR_1X1 || tma) return 3;
    return d->c >= 32 ? 3 : 0;
}

int kblocks_for(const b2c_conv_desc* d, int kmode) {
    if (kmode == 4) return (d->r * d->r + TM_TAPS - 1) / TM_TAPS;
    if (kmode == 5) return d->r * window_chunks(d);
    if (kmode == 3) return d->r * d->r * ((d->c + 31) / 32);
    if (kmode == 6) return d->r * d->r * ((d->c + 63) / 64);
    return (d->c * d->r * d->r + 31) / 32;
}

int is_pow2_in(int v, int lo, int hi) { return v >= lo && v <= hi && (v & (v - 1)) == 0; }

// ----------------------------------------------------------------------------- applicability

// ----------------------------------------------------------------------------- first-layer space-to-depth (tma = 6)
// An R x R stride-S conv with C <= 4 channels is rewritten as an R' x R' stride-1 conv
// (R' = ceil(R/S)) over a space-to-depth copy of x with C*S*S channels (k_s2d_nhwc) and
// re-arranged filters (k_s2d_filters), then run on the ordinary im2col TMA path (tm=1):
// AlexNet / NiN conv1 (11x11 s4, C=3) become 3x3 convs over 48 channels -- 18 K blocks
// per 128-pixel tile instead of 22 per 110-pixel tile with the x-window packing.
struct S2d {
    b2c_conv_desc d2;
    b2c_tune t2;
    int S;
};

bool s2d_of(const b2c_conv_desc* d, const b2c_tune* t, S2d& o) {
    if (!d || !t || t->tma != 6) return false;
    const int S = d->stride, R2 = (d->r + S - 1) / S;
    const int Hs = std::max((d->h + 2 * d->pad + S - 1) / S, d->oh + R2 - 1);
    const int Ws = std::max((d->w + 2 * d->pad + S - 1) / S, d->ow + R2 - 1);
    o.S = S;
    o.d2 = b2c_conv_desc{d->n, d->c * S * S, Hs, Ws, d->k, R2, 1, 0, d->oh, d->ow, d->act, d->prec};
    o.t2 = *t;
    o.t2.tma = 1;
    return true;
}

int applies_impl(const b2c_conv_desc* d, const b2c_tune* t, std::string& why);

int applies_s2d(const b2c_conv_desc* d, const b2c_tune* t, std::string& why) {
    if (t->variant != B2C_VAR_UMMA) { why = "tma=6 (first-layer space-to-depth): conv_umma"; return B2C_INAPPLICABLE; }
    if (d->c > 4 || (d->stride != 2 && d->stride != 4) || d->r <= d->stride || (d->c * d->stride * d->stride) % 4 ||
        d->c * d->stride * d->stride <= 4) {
        why = "tma=6: first layers (C <= 4) with stride 2 or 4 < ksz and C*stride^2 a multiple of 4 above 4"; return B2C_INAPPLICABLE;
    }
    S2d o;
    s2d_of(d, t, o);
    return applies_impl(&o.d2, &o.t2, why);
}

int applies_impl(const b2c_conv_desc* d, const b2c_tune* t, std::string& why) {
    int rc = check_desc(d);
    if (rc) { why = g_last_error; return rc; }
    if (!t) { why = "null tune"; return B2C_BAD_ARGS; }
    const long long M = (long long)d->n * d->oh * d->ow;
    if (d->prec == B2C_PREC_BF16) {
        // bf16 operands / fp32 accumulate: only the TMA tcgen05 kernel with pixels on M
        if (t->variant != B2C_VAR_UMMA && t->variant != B2C_VAR_1X1) {
            why = "bf16 mode: tcgen05 conv_umma / conv_1x1 only"; return B2C_INAPPLICABLE;
        }
        const bool ss_pair = t->tma == 5 && t->cluster == 3;  // bf16 SS on 2-SM pairs
        if (!t->tma || t->swap_ab || (t->cluster >= 2 && !ss_pair) || t->stages == 2 || (t->tma == 2 && d->c <= 4)) {
            why = "bf16 mode: TMA kernel (tma=1|2), swap_ab=0, single CTAs, not the 8-tap first-layer path";
            return B2C_INAPPLICABLE;
        }
        if (t->tile_n != 32 && t->tile_n != 64 && t->tile_n != 128 && t->tile_n != 192) {
            why = "bf16 mode: tile_n in {32, 64, 128, 192}"; return B2C_INAPPLICABLE;
        }
    }
    if (d->prec == B2C_PREC_FP8) {
        // e4m3 operands / fp32 accumulate: the TMA tcgen05 kernel with pixels on M
        if (t->variant != B2C_VAR_UMMA && t->variant != B2C_VAR_1X1) {
            why = "fp8 mode: tcgen05 conv_umma / conv_1x1 only"; return B2C_INAPPLICABLE;
        }
        if (!t->tma || t->tma == 2 || t->swap_ab || t->cluster >= 2 || t->stages == 2) {
            why = "fp8 mode: TMA kernel (tma=1|3|4), swap_ab=0, single CTAs"; return B2C_INAPPLICABLE;
        }
        if (t->tile_n != 32 && t->tile_n != 64 && t->tile_n != 128) {
            why = "fp8 mode: tile_n in {32, 64, 128}"; return B2C_INAPPLICABLE;
        }
    }
    switch (t->variant) {
        case B2C_VAR_SIMPLE:
            return B2C_OK;
        case B2C_VAR_TILED: {
            if (!is_pow2_in(t->mnt0, 1, 8) || !is_pow2_in(t->mnt1, 1, 8)) {
                why = "MNt entries must be 1, 2, 4 or 8"; return B2C_INAPPLICABLE;
            }
            if (t->mnb0 < 1 || t->mnb1 < 1 || t->kb < 1) { why = "bad tune params"; return B2C_BAD_ARGS; }
            const int threads = t->mnb0 * t->mnb1;
            if (threads > 1024) { why = "workgroup exceeds 1024 threads"; return B2C_INAPPLICABLE; }
            if (t->vw != 1 && t->vw != 2 && t->vw != 4 && t->vw != 8) { why = "vector width must be 1,2,4,8"; return B2C_BAD_ARGS; }
            if (t->mnt1 % t->vw) { why = "vector width must divide register block"; return B2C_BAD_ARGS; }
            // Reference applicability (variants.py:391-403).
            if (M < t->mnt0) { why = "fewer output pixels than the register block"; return B2C_INAPPLICABLE; }
            if (d->k < t->mnt1) { why = "fewer output channels than the register block"; return B2C_INAPPLICABLE; }
            if (t->vw > 4) { why = "vector width 8 is not offered"; return B2C_INAPPLICABLE; }
            const size_t sm = tiled_smem_bytes(t->mnb0 * t->mnt0, t->mnb1 * t->mnt1, t->kb);
            if (sm > 200 * 1024) { why = "shared-memory tile too large"; return B2C_INAPPLICABLE; }
            return B2C_OK;
        }
        case B2C_VAR_1X1:
            if (d->r != 1) { why = "kernel size != 1"; return B2C_INAPPLICABLE; }
            if (d->pad != 0) { why = "padding not supported"; return B2C_INAPPLICABLE; }
            break;
        case B2C_VAR_FC:
            if (!(d->r == d->h && d->r == d->w && d->pad == 0 && d->oh == 1 && d->ow == 1)) {
                why = "filters must cover the whole input with 1x1 output"; return B2C_INAPPLICABLE;
            }
            break;
        case B2C_VAR_UMMA:
            break;
        case B2C_VAR_WINO: {  // Winograd F(2x2,3x3): transforms + 16 batched tcgen05 GEMMs (k_wino.cuh)
            if (d->r != 3 || d->stride != 1 || d->pad > 1) { why = "conv_wino needs a 3x3, stride-1 conv with pad 0 or 1"; return B2C_INAPPLICABLE; }
            if (d->prec != B2C_PREC_FP32) { why = "conv_wino: fp32-exact mode only"; return B2C_INAPPLICABLE; }
            if (d->c % 4) { why = "conv_wino needs in_chans % 4 == 0 (16-byte TMA rows of V)"; return B2C_INAPPLICABLE; }
            if (t->tile_n != 64 && t->tile_n != 128 && t->tile_n != 192) { why = "conv_wino: tile_n in {64, 128, 192}"; return B2C_INAPPLICABLE; }
            if (t->split_k < 0) { why = "split_k must be >= 0 (0 = stream-K)"; return B2C_BAD_ARGS; }
            if (t->swap_ab != 0 && t->swap_ab != 1) { why = "swap_ab must be 0 or 1"; return B2C_BAD_ARGS; }
            if (t->drain < 0 || t->drain > 64) { why = "drain must be in [0, 64]"; return B2C_BAD_ARGS; }
            if (t->stages == 2 || t->cluster >= 2) { why = "conv_wino: single CTAs, 1 per SM"; return B2C_INAPPLICABLE; }
            if (t->split_k > (d->c + 31) / 32) { why = "split_k exceeds the number of 32-wide K blocks"; return B2C_INAPPLICABLE; }
            return B2C_OK;
        }
        case B2C_VAR_FC_STREAM: {
            if (!(d->r == d->h && d->r == d->w && d->pad == 0 && d->oh == 1 && d->ow == 1)) {
                why = "filters must cover the whole input with 1x1 output"; return B2C_INAPPLICABLE;
            }
            if (t->kb < 1 || t->kb > 3) { why = "Kb must be 1 (x from L1/L2), 2 (x staged in smem) or 3 (TMA bulk ring)"; return B2C_INAPPLICABLE; }
            if (d->n > (t->kb == 2 ? 32 : 8)) { why = "weight streaming is for batch <= 8 (Kb=1|3) / <= 32 (Kb=2)"; return B2C_INAPPLICABLE; }
            if ((d->c * d->r * d->r) % 4) { why = "ic*h*w % 4 != 0 (16-byte rows)"; return B2C_INAPPLICABLE; }
            if (t->kb == 3) return B2C_OK;  // fixed shape: 8 compute warps, rows per CTA from OC / SMs
            if (t->mnb0 != 2 && t->mnb0 != 4 && t->mnb0 != 8) { why = "warps per block (MNb0) must be 2, 4 or 8"; return B2C_INAPPLICABLE; }
            if (t->kb == 1 && t->mnt1 != 2 && t->mnt1 != 4 && t->mnt1 != 8) { why = "rows per block (MNt1) must be 2, 4 or 8"; return B2C_INAPPLICABLE; }
            if (t->kb == 2 && t->mnt1 != 1 && t->mnt1 != 2 && t->mnt1 != 4) { why = "rows per warp (MNt1) must be 1, 2 or 4"; return B2C_INAPPLICABLE; }
            return B2C_OK;
        }
        default:
            why = "unknown variant";
            return B2C_BAD_ARGS;
    }
    // tcgen05 family
    if (!valid_bn(t->tile_n)) { why = "tile_n must be one of 16,32,64,96,128,192"; return B2C_INAPPLICABLE; }
    if (t->tile_n == 16 && !(t->variant == B2C_VAR_FC && t->swap_ab && t->tma && t->cluster <= 1)) {
        why = "tile_n 16: the swapped TMA fc tile (conv_fc, swap_ab, tma, single CTAs)"; return B2C_INAPPLICABLE;
    }
    if (t->split_k < 0 || (t->split_k == 0 && !t->tma)) { why = "split_k must be >= 1 (0 = stream-K, TMA kernel only)"; return B2C_BAD_ARGS; }
    if (t->cluster < 0 || t->cluster > 4) { why = "cluster must be 0..4"; return B2C_BAD_ARGS; }
    if (t->cluster == 4) {  // split-K over a thread-block cluster, fixup through DSMEM
        if (!t->tma || t->split_k < 2 || t->split_k > 8 || t->stages == 2 || d->prec != B2C_PREC_FP32) {
            why = "cluster split-K (cluster=4): TMA kernel, split_k 2..8, 1 CTA/SM, fp32-exact mode";
            return B2C_INAPPLICABLE;
        }
        const bool fc_swap = t->variant == B2C_VAR_FC && t->swap_ab && t->tile_n == 32;
        const bool conv = t->variant != B2C_VAR_FC && !t->swap_ab && (t->tile_n == 32 || t->tile_n == 64) &&
                          (t->tma == 1 || t->tma == 3 || t->tma == 4) && !(t->tma == 1 && d->c <= 4);
        if (!fc_swap && !conv) {
            why = "cluster split-K: tile_n 32|64 conv tiles (tma 1|3|4, pixels on M) or the fc swap tile (tile_n 32)";
            return B2C_INAPPLICABLE;
        }
    }
    if (t->split_k == 0 && (t->cluster == 2 || t->stages == 2)) { why = "stream-K: single CTAs or 2-SM pairs"; return B2C_INAPPLICABLE; }
    if (t->swap_ab != 0 && t->swap_ab != 1) { why = "swap_ab must be 0 or 1"; return B2C_BAD_ARGS; }
    if (t->drain < 0 || t->drain > 64) { why = "drain must be in [0, 64]"; return B2C_BAD_ARGS; }
    if (t->tma < 0 || t->tma > 6) { why = "tma must be 0..6"; return B2C_BAD_ARGS; }
    if (t->tma == 6) return applies_s2d(d, t, why);
    if (t->tma == 5) {  // bf16 mode: bf16 NHWC copy + SS MMAs (MODE 8)
        if (d->prec != B2C_PREC_BF16) { why = "tma=5 is the bf16 mode's NHWC-bf16 / SS-MMA path"; return B2C_INAPPLICABLE; }
        if (t->variant == B2C_VAR_FC || t->swap_ab || t->cluster == 2 || t->cluster == 4 || t->stages == 2) {
            why = "tma=5: a conv variant, pixels on M, single CTAs or 2-SM pairs, 1 CTA/SM"; return B2C_INAPPLICABLE;
        }
        if (t->cluster == 3 && t->tile_n == 64) { why = "tma=5 pairs: tile_n 128 | 192"; return B2C_INAPPLICABLE; }
        if (d->c % 8 || d->c <= 4) { why = "tma=5 needs in_chans % 8 == 0 (16-byte bf16 NHWC pixels)"; return B2C_INAPPLICABLE; }
        if (t->tile_n != 64 && t->tile_n != 128 && t->tile_n != 192) { why = "tma=5: tile_n in {64, 128, 192}"; return B2C_INAPPLICABLE; }
        if (t->split_k < 0) { why = "split_k must be >= 0"; return B2C_BAD_ARGS; }
    }
    if (t->tma == 4) {  // k x k stride-1 conv read straight from NCHW x (no re-layout launch)
        if (d->stride != 1 || d->r < 2 || t->variant == B2C_VAR_FC) {
            why = "tma=4 (direct NCHW k x k) needs a stride-1 conv with ksz >= 2"; return B2C_INAPPLICABLE;
        }
        if (t->swap_ab || t->cluster == 2) { why = "tma=4: pixels on M (swap_ab=0), no multicast pairs"; return B2C_INAPPLICABLE; }
        if (d->w % 4 || d->ow + 3 > UMMA_M) {
            why = "tma=4: input width must be a multiple of 4 (16-byte TMA rows) and ow <= 125"; return B2C_INAPPLICABLE;
        }
    }
    if (t->tma == 3) {  // 1x1 conv read straight from NCHW x (no re-layout launch)
        if (!(d->r == 1 && d->stride == 1 && d->pad == 0) || t->variant == B2C_VAR_FC) {
            why = "tma=3 (direct NCHW) needs a 1x1, stride 1, pad 0 conv"; return B2C_INAPPLICABLE;
        }
        if (t->swap_ab || t->cluster == 2) { why = "tma=3: pixels on M (swap_ab=0), no multicast pairs"; return B2C_INAPPLICABLE; }
        if (((long long)d->h * d->w * 4) % 16) { why = "tma=3: h*w*4 bytes must be a multiple of 16 (TMA strides)"; return B2C_INAPPLICABLE; }
    }
    if (t->tma && t->stages == 2 && t->tile_n > 64) { why = "two CTAs per SM (stages=2) need tile_n <= 64"; return B2C_INAPPLICABLE; }
    if (t->cluster == 2 && (!t->tma || t->swap_ab || t->variant == B2C_VAR_FC || t->tile_n < 64 || t->stages == 2)) {
        why = "CTA pairs (cluster=2) need the TMA kernel, swap_ab=0, a conv variant, tile_n >= 64, 1 CTA/SM";
        return B2C_INAPPLICABLE;
    }
    if (t->cluster == 2 && t->tma == 2 && d->c <= 4) { why = "CTA pairs: not with the 8-tap first-layer path"; return B2C_INAPPLICABLE; }
    if (t->cluster == 3) {  // 2-SM UMMA (tcgen05 cta_group::2, M = 256)
        if (!t->tma || t->swap_ab || t->variant == B2C_VAR_FC || t->tile_n < 64 || t->stages == 2) {
            why = "2-SM UMMA pairs (cluster=3) need the TMA kernel, swap_ab=0, a conv variant, tile_n >= 64, 1 CTA/SM";
            return B2C_INAPPLICABLE;
        }
        if (t->tma == 2) { why = "2-SM UMMA pairs: not with tma=2 (2-D tiles / 8-tap first-layer boxes)"; return B2C_INAPPLICABLE; }
        if (t->tile_n != 64 && t->tile_n != 96 && t->tile_n != 128 && t->tile_n != 192) { why = "2-SM UMMA pairs: tile_n in {64, 96, 128, 192}"; return B2C_INAPPLICABLE; }
        if (t->tile_n == 96 && t->tma == 5) { why = "tma=5 pairs: tile_n 128 | 192"; return B2C_INAPPLICABLE; }
        if (d->prec != B2C_PREC_FP32 && !(d->prec == B2C_PREC_BF16 && t->tma == 5)) {
            why = "2-SM UMMA pairs: fp32-exact mode, or the bf16 SS path (tma=5)"; return B2C_INAPPLICABLE;
        }
    }
    if (t->tma == 2 && !(d->r == 1 && d->stride == 1 && d->pad == 0) && t->variant != B2C_VAR_FC && d->c > 4) {
        why = "tma=2 (2-D tiled pixels) needs a 1x1, stride 1, pad 0 conv"; return B2C_INAPPLICABLE;
    }
    if (t->tma) {
        if (t->variant == B2C_VAR_FC) {
            if ((d->c * d->r * d->r) % 4) { why = "TMA fc path needs ic*h*w % 4 == 0 (16-byte rows)"; return B2C_INAPPLICABLE; }
        } else {
            if (d->c % 4 && d->c > 4) { why = "TMA conv path needs in_chans % 4 == 0 or <= 4 (16-byte NHWC pixels)"; return B2C_INAPPLICABLE; }
            if (d->pad > 127 || d->r - 1 - d->pad > 128 || d->r > 256) { why = "filter too large for TMA im2col"; return B2C_INAPPLICABLE; }
            if (d->c <= 4 && t->tma != 2 && t->swap_ab) { why = "first-layer TMA path (tma=1) tiles pixels on M (swap_ab=0)"; return B2C_INAPPLICABLE; }
        }
    }
    const int kblocks = kblocks_for(d, kmode_for(d, t->variant, t->tma));
    if (t->split_k > kblocks) { why = "split_k exceeds the number of 32-wide K blocks"; return B2C_INAPPLICABLE; }
    return B2C_OK;
}

// ----------------------------------------------------------------------------- launch plans

struct UmmaPlan {
    int grid_x, grid_y, split, kps, kblocks, cblocks, tiles, kmode, flt_rows, tma;
    int bx, by, tiles_x, tiles_y, hp, wp;  // kmode 5: pixel blocks and the padded NHWC extent
    int box_w;                             // tma = 4: TMA box width (floats) over NCHW rows
    int parts;                             // packed filter halves per K block (2: raw | lo, 1: raw)
    int streamk, sk_grid, sk_maxc;         // split_k == 0: stream-K over the units' K blocks
    size_t wpk_bytes;   // packed filters (offset 0 of the workspace; 0 for the TMA fc path)
    size_t part_off;    // split-K partials
    size_t sems_off;    // split-K tickets
    size_t nhwc_off;    // TMA conv path: NHWC copy of x
    size_t gbar_off;    // TMA path: grid-barrier counter
    size_t ws_bytes;    // total
};

size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

int num_sms();

UmmaPlan umma_plan(const b2c_conv_desc* d, const b2c_tune* t) {
    UmmaPlan p;
    const int M = d->n * d->oh * d->ow;
    const int BN = t->tile_n;
    const int pix_tile = t->swap_ab ? BN : UMMA_M;
    p.flt_rows = t->swap_ab ? UMMA_M : BN;
    p.grid_x = (M + pix_tile - 1) / pix_tile;
    p.grid_y = (d->k + p.flt_rows - 1) / p.flt_rows;
    p.tiles = p.grid_x * p.grid_y;
    p.tma = t->tma;
    p.kmode = kmode_for(d, t->variant, t->tma);
    p.kblocks = kblocks_for(d, p.kmode);
    p.cblocks = p.kmode == 5 ? window_chunks(d) : p.kmode == 6 ? (d->c + 63) / 64 : (d->c + 31) / 32;
    p.bx = p.by = p.tiles_x = p.tiles_y = p.hp = p.wp = p.box_w = 0;
    if (t->tma == 4) {  // MODE 6: whole output rows of one image, the box 3+ floats wider for the aligned start
        p.bx = d->ow;
        p.box_w = (d->ow + 3 + 3) / 4 * 4;
        p.by = std::max(1, std::min(UMMA_M / p.box_w, d->oh));
        p.tiles_x = 1;
        p.tiles_y = (d->oh + p.by - 1) / p.by;
        p.grid_x = d->n * p.tiles_y;
        p.tiles = p.grid_x * p.grid_y;
    }
    if (t->tma == 3) {  // MODE 5: runs of 128 pixels of one image (tiles do not straddle images)
        p.bx = UMMA_M;
        p.by = 1;
        p.tiles_x = (d->oh * d->ow + UMMA_M - 1) / UMMA_M;
        p.tiles_y = 1;
        p.grid_x = d->n * p.tiles_x;
        p.tiles = p.grid_x * p.grid_y;
    }
    if (p.kmode == 5) {
        p.bx = std::min(d->ow, UMMA_M);
        p.by = std::min(UMMA_M / p.bx, d->oh);
        p.tiles_x = (d->ow + p.bx - 1) / p.bx;
        p.tiles_y = (d->oh + p.by - 1) / p.by;
        p.grid_x = d->n * p.tiles_x * p.tiles_y;
        p.tiles = p.grid_x * p.grid_y;
        p.hp = d->h + 2 * d->pad;
        p.wp = std::max(d->w + 2 * d->pad, (d->ow - 1) * d->stride + TM_BK / 4 * window_chunks(d));
    }
    const int want = std::max(1, std::min(t->split_k, p.kblocks));
    p.kps = (p.kblocks + want - 1) / want;
    p.split = (p.kblocks + p.kps - 1) / p.kps;  // every split gets >= 1 block
    // packed filters: raw | lo per K block; raw only when the TMA kernel takes them as its TMEM A operand
    p.parts = (p.tma && t->swap_ab) || d->prec != B2C_PREC_FP32 ? 1 : 2;
    const size_t row_bytes = p.kmode == 6 ? 128 : d->prec == B2C_PREC_BF16 ? UMMA_BK * 2 : d->prec == B2C_PREC_FP8 ? UMMA_BK
                                                                                           : UMMA_BK * sizeof(float);  // per K block
    p.wpk_bytes = (p.tma && p.kmode == 2) ? 0 : (size_t)p.grid_y * p.kblocks * p.parts * p.flt_rows * row_bytes;
    p.streamk = (t->tma && t->split_k == 0) ? 1 : 0;
    p.sk_grid = p.sk_maxc = 0;
    size_t nslots = (p.split > 1 && t->cluster != 4) ? (size_t)p.tiles * p.split : 0;  // cluster split-K: DSMEM
    if (p.streamk) {
        // 2-SM pairs share units (two neighbouring pixel tiles): stream-K over pair-units, one share per pair
        const bool pair = t->cluster == 3;
        const long long units = pair ? (long long)((p.grid_x + 1) / 2) * p.grid_y : p.tiles;
        const long long W = units * p.kblocks;
        const int ctas = (int)std::min<long long>(W, pair ? num_sms() / 2 : num_sms());  // CTAs (pairs)
        p.sk_grid = pair ? 2 * ctas : ctas;
        const long long L = std::max<long long>(1, W / ctas);  // K blocks per CTA / pair (floor)
        p.sk_maxc = (int)((p.kblocks + L - 1) / L + 1);
        nslots = (size_t)p.tiles * p.sk_maxc;
    }
    p.part_off = align256(p.wpk_bytes);
    p.sems_off = p.part_off + (nslots ? align256(nslots * BN * UMMA_M * sizeof(float)) : 0);
    p.nhwc_off = p.sems_off + (nslots ? align256((size_t)p.tiles * sizeof(int)) : 0);
    const bool nhwc = p.tma && p.tma != 3 && p.tma != 4 && (p.kmode == 3 || p.kmode == 4 || p.kmode == 5 || p.kmode == 6);
    const int cp = (p.kmode == 4 || p.kmode == 5) ? 4 : d->c;  // first layers: channels padded to 4 (16-byte pixels)
    const size_t pix = p.kmode == 5 ? (size_t)p.hp * p.wp : (size_t)d->h * d->w;
    const size_t elt = p.kmode == 6 ? 2 : sizeof(float);  // kmode 6: bf16 NHWC copy
    p.gbar_off = p.nhwc_off + (nhwc ? align256((size_t)d->n * cp * pix * elt) : 0);
    p.ws_bytes = p.gbar_off + (p.tma ? 256 : 0);  // grid-barrier counter of the fused re-layout
    return p;
}

using UmmaKernel = void (*)(UmmaArgs);

struct UmmaEntry {
    UmmaKernel fn;
    int smem;
    int stages;
};

template <int BN, bool SWAP, int KMODE>
UmmaEntry umma_entry() {
    return UmmaEntry{&k_umma<BN, SWAP, KMODE>, UmmaCfg<BN, SWAP>::SMEM, UmmaCfg<BN, SWAP>::STAGES};
}

template <bool SWAP, int KMODE>
UmmaEntry umma_pick_bn(int bn) {
    switch (bn) {
        case 32: return umma_entry<32, SWAP, KMODE>();
        case 64: return umma_entry<64, SWAP, KMODE>();
        case 96: return umma_entry<96, SWAP, KMODE>();
        case 128: return umma_entry<128, SWAP, KMODE>();
        case 192: return umma_entry<192, SWAP, KMODE>();
    }
    return UmmaEntry{nullptr, 0, 0};
}

UmmaEntry umma_pick(int bn, int swap, int kmode) {
    if (swap) {
        if (kmode == 0) return umma_pick_bn<true, 0>(bn);
        if (kmode == 2) return umma_pick_bn<true, 2>(bn);
        return umma_pick_bn<true, 3>(bn);
    }
    if (kmode == 0) return umma_pick_bn<false, 0>(bn);
    if (kmode == 2) return umma_pick_bn<false, 2>(bn);
    return umma_pick_bn<false, 3>(bn);
}

bool is_umma(int variant) { return variant == B2C_VAR_UMMA || variant == B2C_VAR_1X1 || variant == B2C_VAR_FC; }

int pack_impl(const b2c_conv_desc* d, const b2c_tune* t, const float* w, void* ws, size_t ws_bytes,
              cudaStream_t st) {
    S2d o;
    if (s2d_of(d, t, o)) {  // re-arrange the filters past the rewritten conv's workspace, then pack those
        const size_t base = umma_plan(&o.d2, &o.t2).ws_bytes;
        const size_t w2b = (size_t)o.d2.k * o.d2.c * o.d2.r * o.d2.r * sizeof(float);
        if (!ws || ws_bytes < base + align256(w2b)) return fail(B2C_BAD_ARGS, "workspace too small (see b2c_conv_workspace)");
        float* w2 = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + base);
        const long long total = (long long)(w2b / sizeof(float));
        k_s2d_filters<<<(unsigned)std::min<long long>((total + 255) / 256, 148LL * 16), 256, 0, st>>>(
            w, w2, d->k, d->c, d->r, o.S, o.d2.r);
        return pack_impl(&o.d2, &o.t2, w2, ws, base, st);
    }
    const UmmaPlan p = umma_plan(d, t);
    if (p.wpk_bytes == 0) return B2C_OK;  // TMA fc path reads raw filters
    if (!ws || ws_bytes < p.ws_bytes) return fail(B2C_BAD_ARGS, "workspace too small (see b2c_conv_workspace)");
    const Geom g = make_geom(d);
    if (d->prec == B2C_PREC_FP8) {
        const long long total = (long long)p.wpk_bytes;
        const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 32);
        k_pack_filters_e4m3<<<blocks, 256, 0, st>>>(g, w, reinterpret_cast<uint8_t*>(ws), p.flt_rows, p.kblocks,
                                                    FastDiv((uint32_t)p.cblocks), p.kmode, total);
        return B2C_OK;
    }
    if (p.kmode == 6) {  // bf16 SW128 images of (tap, 64-channel block) for the SS MMAs
        const long long total = (long long)p.wpk_bytes / 2;
        const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 32);
        k_pack_filters_bf16_sw128<<<blocks, 256, 0, st>>>(g, w, reinterpret_cast<uint16_t*>(ws), p.flt_rows, p.kblocks,
                                                          FastDiv((uint32_t)p.cblocks), total);
        return B2C_OK;
    }
    if (d->prec == B2C_PREC_BF16) {
        const long long total = (long long)p.wpk_bytes / 2;
        const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 32);
        k_pack_filters_bf16<<<blocks, 256, 0, st>>>(g, w, reinterpret_cast<uint16_t*>(ws), p.flt_rows, p.kblocks,
                                                    FastDiv((uint32_t)p.cblocks), p.kmode, total);
        return B2C_OK;
    }
    const long long total = (long long)p.wpk_bytes / 4;
    const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 32);
    k_pack_filters<<<blocks, 256, 0, st>>>(g, w, reinterpret_cast<float*>(ws), p.flt_rows, p.kblocks,
                                           FastDiv((uint32_t)p.cblocks), p.kmode, total,
                                           (p.tma && (p.kmode == 3 || p.kmode == 5)) ? 1 : 0,  // SWIZZLE_128B image
                                           p.parts);
    return B2C_OK;
}

// Per-device "max dynamic smem" attribute of a kernel: the largest size set so
// far is remembered per (kernel, device) and raised whenever a launch needs
// more (k_tiled<MT,NT> / the staged fc kernels take runtime-dependent sizes).
struct AttrRec {
    const void* fn;
    int dev;
    int bytes;
};
std::mutex g_attr_mu;
std::vector<AttrRec> g_attr_done;

int ensure_smem_attr(const void* fn, int bytes) {
    int dev = 0;
    B2C_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_attr_mu);
    AttrRec* rec = nullptr;
    for (auto& e : g_attr_done)
        if (e.fn == fn && e.dev == dev) rec = &e;
    if (rec && rec->bytes >= bytes) return B2C_OK;
    B2C_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    if (rec)
        rec->bytes = bytes;
    else
        g_attr_done.push_back(AttrRec{fn, dev, bytes});
    return B2C_OK;
}

using TiledKernel = void (*)(Geom, const float*, const float*, const float*, float*, int, int, int);

TiledKernel tiled_pick(int mt, int nt) {
#define B2C_T(a, b) \
    if (mt == a && nt == b) return &k_tiled<a, b>;
    B2C_T(1, 1) B2C_T(1, 2) B2C_T(1, 4) B2C_T(1, 8)
    B2C_T(2, 1) B2C_T(2, 2) B2C_T(2, 4) B2C_T(2, 8)
    B2C_T(4, 1) B2C_T(4, 2) B2C_T(4, 4) B2C_T(4, 8)
    B2C_T(8, 1) B2C_T(8, 2) B2C_T(8, 4) B2C_T(8, 8)
#undef B2C_T
    return nullptr;
}

// ----------------------------------------------------------------------------- TMA path

// Tensor-map encoders come from the driver through the runtime's entry-point
// query, so the library needs no -lcuda link.
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
using EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int g_trace_on = 0;
long long* trace_buf() {  // device address of g_b2c_trace (looked up when tracing is on)
    long long* p = nullptr;
    if (g_trace_on & 15) cudaGetSymbolAddress(reinterpret_cast<void**>(&p), b2c::g_b2c_trace);
    return p;
}
std::once_flag g_drv_once;
EncodeTiledFn g_enc_tiled = nullptr;
EncodeIm2colFn g_enc_im2col = nullptr;
int g_drv_version = 0;

int load_tma_encoders() {
    std::call_once(g_drv_once, [] {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_enc_tiled = reinterpret_cast<EncodeTiledFn>(fn);
        fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_enc_im2col = reinterpret_cast<EncodeIm2colFn>(fn);
        cudaDriverGetVersion(&g_drv_version);
    });
    if (!g_enc_tiled || !g_enc_im2col) return fail(B2C_CUDA_ERROR, "cuTensorMapEncode* not available from the driver");
    return B2C_OK;
}

// Known driver issue (<= 13.1) with im2col maps over tensors smaller than
// 128 KiB: clear bit 21 of the second descriptor word (the same workaround
// CUTLASS applies, cute/atom/copy_traits_sm90_im2col.hpp).
void im2col_small_tensor_fix(CUtensorMap* tm, size_t tensor_bytes) {
    if (g_drv_version <= 13010 && tensor_bytes < 131072) reinterpret_cast<uint64_t*>(tm)[1] &= ~(1ull << 21);
}

// NHWC tensor (cp channels per pixel) for im2col loads of `pix_rows` output
// pixels x `cpp` channels; the bounding box corners are the conv padding
// (lower = -pad, upper = pad - (ksz - 1)), the traversal strides the conv stride.
int encode_im2col(CUtensorMap* tm, const b2c_conv_desc* d, const void* xh, int cp, int cpp, int pix_rows, bool sw128,
                  int elt = 4) {
    const cuuint64_t dims[4] = {(cuuint64_t)cp, (cuuint64_t)d->w, (cuuint64_t)d->h, (cuuint64_t)d->n};
    const cuuint64_t strides[3] = {(cuuint64_t)cp * elt, (cuuint64_t)d->w * cp * elt, (cuuint64_t)d->h * d->w * cp * elt};
    const int lower[2] = {-d->pad, -d->pad};
    const int upper[2] = {d->pad - (d->r - 1), d->pad - (d->r - 1)};
    const cuuint32_t estr[4] = {1, (cuuint32_t)d->stride, (cuuint32_t)d->stride, 1};
    CUresult r = g_enc_im2col(tm, elt == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                              const_cast<void*>(xh), dims, strides, lower,
                              upper, (cuuint32_t)cpp, (cuuint32_t)pix_rows, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              sw128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(B2C_CUDA_ERROR, "cuTensorMapEncodeIm2col failed (" + std::to_string((int)r) + ")");
    im2col_small_tensor_fix(tm, (size_t)d->n * cp * d->h * d->w * elt);
    return B2C_OK;
}

// First-layer x-window map over the padded NHWC4 copy: coordinates
// (window float, ox, oy, ky, image) with byte strides (4, 16*S, 16*S*Wp,
// 16*Wp, 16*Hp*Wp) -- deliberately overlapping, so that (ox, oy, ky) address
// the 8 x-taps x 4 channels an output pixel needs for filter row ky as one
// 128-byte row.  Box = 32 floats x bx x by pixels.
int encode_window(CUtensorMap* tm, const b2c_conv_desc* d, const UmmaPlan& p, const float* xp) {
    const cuuint64_t dims[5] = {(cuuint64_t)window_chunks(d) * TM_BK, (cuuint64_t)d->ow, (cuuint64_t)d->oh,
                                (cuuint64_t)d->r, (cuuint64_t)d->n};
    const cuuint64_t strides[4] = {(cuuint64_t)16 * d->stride, (cuuint64_t)16 * d->stride * p.wp, (cuuint64_t)16 * p.wp,
                                   (cuuint64_t)16 * p.hp * p.wp};
    const cuuint32_t box[5] = {(cuuint32_t)TM_BK, (cuuint32_t)p.bx, (cuuint32_t)p.by, 1, 1};
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = g_enc_tiled(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(xp), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(B2C_CUDA_ERROR, "cuTensorMapEncodeTiled (x-window) failed (" + std::to_string((int)r) + ")");
    return B2C_OK;
}

// Row-major [rows][cols] fp32 matrix, box = 32 cols (128 B) x box_rows, SWIZZLE_128B.
int encode_rows(CUtensorMap* tm, const float* base, long long rows, long long cols, int box_rows) {
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
    const cuuint32_t box[2] = {(cuuint32_t)TM_BK, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = g_enc_tiled(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(B2C_CUDA_ERROR, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return B2C_OK;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*fn)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int cluster,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    static const bool no_pdl = std::getenv("B2C_NO_PDL") != nullptr;  // A/B switch for measurements
    if (!no_pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (cluster > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = cluster;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, fn, std::forward<Args>(args)...);
}

// Multiply-shift divisors for the kernel's unit decomposition (unit_of, k_tma.cuh).
void set_unit_divs(TArgs& a) {
    a.fSplit = FastDiv((uint32_t)std::max(1, a.split));
    a.fTilesN = FastDiv((uint32_t)std::max(1, a.tiles_n));
    a.fTilesMN = FastDiv((uint32_t)std::max(1, a.tiles_m * a.tiles_n));
    a.fPerImg = FastDiv((uint32_t)std::max(1, a.tiles_x * a.tiles_y));
    a.fTilesX = FastDiv((uint32_t)std::max(1, a.tiles_x));
}


int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// k_fc_bulk: out_chan rows per CTA (one CTA per SM, <= 32 rows: 4 per compute warp)
int fcb_rows_per_cta(int oc) {
    const int sms = num_sms();
    return std::min(FCB_WARPS * FCB_MAX_RPW, std::max(1, (oc + sms - 1) / sms));
}

int tma_fwd(const b2c_conv_desc* d, const b2c_tune* t, const UmmaPlan& p, const Geom& g, const float* x,
            const float* w, const float* bias, float* y, void* ws, cudaStream_t st,
            const b2c_conv_desc* s2d_src = nullptr) {  // s2d_src: the original first-layer conv (tma = 6)
    int rc = load_tma_encoders();
    if (rc) return rc;
    const bool plain_1x1 = d->r == 1 && d->stride == 1 && d->pad == 0;
    const int mode = t->tma == 5 ? 8 : t->tma == 4 ? 6 : t->tma == 3 ? 5 : p.kmode == 2 ? 1 : p.kmode == 5 ? 4 : p.kmode == 4 ? 3 : (plain_1x1 && t->tma == 2) ? 2 : 0;
    const int occ = t->stages == 2 ? 2 : 1;  // TMA kernel: b2c_tune.stages = CTAs per SM
    const int cl = (t->cluster >= 2 && t->cluster <= 4) ? t->cluster : 1;
    const TconvEntry e = tconv_pick_mode(mode, d->prec, t->tile_n, t->swap_ab, occ, cl);
    if (!e.fn) return fail(B2C_INAPPLICABLE, "no TMA tcgen05 kernel for this tile");
    rc = ensure_smem_attr((const void*)e.fn, e.smem);
    if (rc) return rc;
    const int pix_rows = t->swap_ab ? t->tile_n : TM_M;
    char* wsb = reinterpret_cast<char*>(ws);
    CUtensorMap tm_pix, tm_flt;
    std::memset(&tm_flt, 0, sizeof(tm_flt));
    // x re-layout: a separate PDL-launched kernel (default; measured faster) or,
    // with B2C_FUSED_NHWC set, inside k_tconv before a grid barrier.
    static const bool separate = std::getenv("B2C_FUSED_NHWC") == nullptr;
    int relayout = 0;
    if (mode == 5) {  // 1x1: x itself as [img][chan][pixels], box = 128 pixels x 32 channels
        const cuuint64_t dims[3] = {(cuuint64_t)d->h * d->w, (cuuint64_t)d->c, (cuuint64_t)d->n};
        const cuuint64_t strides[2] = {(cuuint64_t)d->h * d->w * 4, (cuuint64_t)d->c * d->h * d->w * 4};
        const cuuint32_t box[3] = {(cuuint32_t)UMMA_M, (cuuint32_t)TM_BK, 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = g_enc_tiled(&tm_pix, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(x), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(B2C_CUDA_ERROR, "cuTensorMapEncodeTiled (NCHW 1x1) failed (" + std::to_string((int)r) + ")");
    } else if (mode == 6) {  // k x k, stride 1: x itself as [img][chan][y][x]; box = box_w x by pixels x 32 channels
        const cuuint64_t dims[4] = {(cuuint64_t)d->w, (cuuint64_t)d->h, (cuuint64_t)d->c, (cuuint64_t)d->n};
        const cuuint64_t strides[3] = {(cuuint64_t)d->w * 4, (cuuint64_t)d->h * d->w * 4, (cuuint64_t)d->c * d->h * d->w * 4};
        const cuuint32_t box[4] = {(cuuint32_t)p.box_w, (cuuint32_t)p.by, (cuuint32_t)TM_BK, 1};
        const cuuint32_t estr[4] = {1, 1, 1, 1};
        CUresult r = g_enc_tiled(&tm_pix, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(x), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(B2C_CUDA_ERROR, "cuTensorMapEncodeTiled (NCHW kxk) failed (" + std::to_string((int)r) + ")");
    } else if (mode == 4) {
        float* xp = reinterpret_cast<float*>(wsb + p.nhwc_off);
        const long long total = (long long)d->n * p.hp * p.wp;
        if (!separate) relayout = 2;
        else if (!(g_trace_on & 16)) {
            cudaError_t le = launch_pdl(k_to_nhwc4_pad, dim3(d->n * p.hp), dim3(p.wp > 128 ? 256 : 128), 0, st, 1, x, reinterpret_cast<float4*>(xp),
                                        (int)d->c, (int)d->h, (int)d->w, p.hp, p.wp, (int)d->pad, total);
            if (le != cudaSuccess) return cuda_fail(le, "k_to_nhwc4_pad launch");
        }
        rc = encode_window(&tm_pix, d, p, xp);
        if (rc) return rc;
    } else if (mode == 8) {  // bf16 NHWC copy, im2col boxes of 128 pixels x 64 channels (128-byte rows)
        uint16_t* xb = reinterpret_cast<uint16_t*>(wsb + p.nhwc_off);
        const int HW = d->h * d->w;
        if (!(g_trace_on & 16)) {
            dim3 tgrid((HW + 31) / 32, (d->c + 31) / 32, d->n);
            cudaError_t le = launch_pdl(k_nchw_to_nhwc_bf16, tgrid, dim3(256), 0, st, 1, x, xb, (int)d->c, HW);
            if (le != cudaSuccess) return cuda_fail(le, "bf16 NHWC conversion launch");
        }
        rc = encode_im2col(&tm_pix, d, xb, d->c, 64, pix_rows, true, 2);
        if (rc) return rc;
    } else if (mode != 1) {
        float* xh = reinterpret_cast<float*>(wsb + p.nhwc_off);
        const int HW = d->h * d->w;
        const int cp = mode == 3 ? 4 : d->c;
        if (!separate && mode != 3 && !s2d_src) relayout = 1;
        else if (!(g_trace_on & 16)) {  // debug bit 4: reuse the NHWC copy already in the workspace
            cudaError_t le;
            if (mode == 3) {
                const long long total = (long long)d->n * HW;
                le = launch_pdl(k_to_nhwc4_pad, dim3(d->n * d->h), dim3(d->w > 128 ? 256 : 128), 0, st, 1, x, reinterpret_cast<float4*>(xh),
                                (int)d->c, (int)d->h, (int)d->w, (int)d->h, (int)d->w, 0, total);
            } else if (s2d_src) {  // x -> its space-to-depth NHWC copy (d is the rewritten conv)
                auto ks = s2d_src->stride == 4 ? k_s2d_nhwc<4> : k_s2d_nhwc<2>;  // S*S % 4 == 0: float4 stores
                le = launch_pdl(ks, dim3(d->n * d->h), dim3(256), 0, st, 1, x, xh, (int)s2d_src->c, (int)s2d_src->h,
                                (int)s2d_src->w, (int)s2d_src->pad, (int)d->h, (int)d->w);
            } else {
                dim3 tgrid((HW + 31) / 32, (cp + 31) / 32, d->n);
                le = launch_pdl(k_nchw_to_nhwc, tgrid, dim3(256), 0, st, 1, x, xh, (int)d->c, cp, HW);
            }
            if (le != cudaSuccess) return cuda_fail(le, "NHWC conversion launch");
        }
        if (mode == 2)
            rc = encode_rows(&tm_pix, xh, (long long)d->n * d->h * d->w, d->c, pix_rows);
        else
            rc = encode_im2col(&tm_pix, d, xh, cp, mode == 3 ? 4 : TM_BK, pix_rows, mode != 3);
        if (rc) return rc;
    } else {
        rc = encode_rows(&tm_pix, x, d->n, (long long)g.K, pix_rows);
        if (rc) return rc;
        rc = encode_rows(&tm_flt, w, d->k, (long long)g.K, t->swap_ab ? TM_M : t->tile_n);
        if (rc) return rc;
    }
    TArgs a = {};  // every field set below; zero-init guards new ones
    a.g = g;
    a.wpk = reinterpret_cast<const float*>(ws);
    a.bias = bias;
    a.y = y;
    a.split = p.split;
    a.kps = p.kps;
    a.kblocks = p.kblocks;
    a.streamk = p.streamk;
    a.sk_maxc = p.sk_maxc;
    a.tiles_n = p.grid_y;
    a.tiles_m = p.grid_x;
    // CL = 2: units are pair-units (two neighbouring pixel tiles)
    a.units = ((cl == 2 || cl == 3) ? (p.grid_x + 1) / 2 * p.grid_y : p.tiles) * p.split;
    a.bx = p.bx;
    a.by = p.by;
    a.tiles_x = p.tiles_x;
    a.tiles_y = p.tiles_y;
    a.box_w = p.box_w;
    a.fCB = FastDiv((uint32_t)p.cblocks);
    set_unit_divs(a);
    a.drain = t->drain > 0 ? std::max(2, t->drain) : 4;
    a.ws = reinterpret_cast<float*>(wsb + p.part_off);
    a.sems = reinterpret_cast<int*>(wsb + p.sems_off);
    a.trace_buf = trace_buf();
    a.trace = g_trace_on & 15;  // bit0 trace, bit1 hi*hi only, bit2 no B split, bit3 no A->TMEM (experiments)
    a.relayout = (g_trace_on & 16) ? 0 : relayout;
    a.x = x;
    a.xh = reinterpret_cast<float*>(wsb + p.nhwc_off);
    a.hp = p.hp;
    a.wp = p.wp;
    a.pad = d->pad;
    a.gbar = reinterpret_cast<unsigned long long*>(wsb + p.gbar_off);
    a.flt_early = t->prepared ? 1 : 0;  // b2c_conv_prepare synchronises, so a prepared pack is complete
    {
        int period = p.kblocks, valid = g.K - TM_BK * (p.kblocks - 1);  // fc (MODE 1): flat K tail
        if (mode == 8) {  // 64-channel blocks, K = 16 per MMA step
            period = p.cblocks;
            valid = (d->c - 64 * (period - 1) + 1) / 2;  // ceil(valid / 8) below = ceil(channels / 16) MMA steps
        } else if (mode == 0 || mode == 2 || mode == 5 || mode == 6) {
            period = p.cblocks;
            valid = d->c - TM_BK * (period - 1);
        } else if (mode == 4) {
            period = p.cblocks;  // x-window chunks per filter row
            valid = d->r * 4 - TM_BK * (period - 1);
        } else if (mode == 3) {
            valid = 4 * (d->r * d->r - TM_TAPS * (p.kblocks - 1));
        }
        a.kb_period = std::max(1, period);
        a.ksteps_last = std::min(TM_BK / 8, std::max(1, (valid + 7) / 8));
        static const bool no_skip = std::getenv("B2C_NO_KSKIP") != nullptr;  // A/B experiments
        if (no_skip) a.ksteps_last = TM_BK / 8;
    }
    const int grid = p.streamk ? p.sk_grid
                     : cl == 4  ? p.split * std::min(p.tiles, std::max(1, num_sms() / p.split))  // whole clusters
                     : cl >= 2  ? 2 * std::min(a.units, num_sms() / 2)
                                : std::min(a.units, occ * num_sms());
    const int cdim = cl == 4 ? p.split : cl >= 2 ? 2 : 1;
    cudaError_t le = launch_pdl(e.fn, dim3(grid), dim3(e.threads), (size_t)e.smem, st, cdim, tm_pix, tm_flt, a);
    if (le != cudaSuccess) return cuda_fail(le, "k_tconv launch");
    return B2C_OK;
}

// ----------------------------------------------------------------------------- Winograd F(2x2,3x3)

struct WinoPlan {
    int tiles_y, tiles_x, P;   // 2x2 output tiles per image row / column, all tiles
    b2c_conv_desc gd;          // the GEMM as a (P x C) * (OC x C)^T "fc" problem (act none)
    int pix_rows, flt_rows, tiles_m, tiles_n, kblocks, kps, split, streamk, sk_grid, sk_maxc;
    long long units;           // GEMM work units over all 16 z
    size_t u_off, v_off, m_off, zb_off, part_off, sems_off, ws_bytes;
};

WinoPlan wino_plan(const b2c_conv_desc* d, const b2c_tune* t) {
    WinoPlan p;
    p.tiles_y = (d->oh + 1) / 2;
    p.tiles_x = (d->ow + 1) / 2;
    p.P = d->n * p.tiles_y * p.tiles_x;
    // GEMM output M[z]: [P][OC] with swap_ab (its stores run along out channels), else [OC][P]
    // (pixels on M: stores run along p) -- the geometry's PQ sets the stride (see epilogue_unit)
    p.gd = t->swap_ab ? b2c_conv_desc{p.P, d->c, 1, 1, d->k, 1, 1, 0, 1, 1, 0, B2C_PREC_FP32}
                      : b2c_conv_desc{1, d->c, 1, p.P, d->k, 1, 1, 0, 1, p.P, 0, B2C_PREC_FP32};
    p.pix_rows = t->swap_ab ? t->tile_n : UMMA_M;
    p.flt_rows = t->swap_ab ? UMMA_M : t->tile_n;
    p.tiles_m = (p.P + p.pix_rows - 1) / p.pix_rows;
    p.tiles_n = (d->k + p.flt_rows - 1) / p.flt_rows;
    p.kblocks = (d->c + TM_BK - 1) / TM_BK;
    const int want = std::max(1, std::min(t->split_k, p.kblocks));
    p.kps = (p.kblocks + want - 1) / want;
    p.split = (p.kblocks + p.kps - 1) / p.kps;
    const long long tiles = 16ll * p.tiles_m * p.tiles_n;
    p.streamk = t->split_k == 0 ? 1 : 0;
    p.sk_grid = p.sk_maxc = 0;
    size_t nslots = p.split > 1 ? (size_t)tiles * p.split : 0;
    if (p.streamk) {
        p.split = 1;
        p.kps = p.kblocks;
        const long long W = tiles * p.kblocks;
        p.sk_grid = (int)std::min<long long>(W, num_sms());
        const long long L = std::max<long long>(1, W / p.sk_grid);
        p.sk_maxc = (int)((p.kblocks + L - 1) / L + 1);
        nslots = (size_t)tiles * p.sk_maxc;
    }
    p.units = tiles * p.split;
    const size_t f = sizeof(float);
    p.u_off = 0;
    p.v_off = align256(16ull * d->k * d->c * f);
    p.m_off = p.v_off + align256(16ull * p.P * d->c * f);
    p.zb_off = p.m_off + align256(16ull * p.P * d->k * f);
    p.part_off = p.zb_off + align256((size_t)d->k * f);
    p.sems_off = p.part_off + (nslots ? align256(nslots * t->tile_n * UMMA_M * f) : 0);
    p.ws_bytes = p.sems_off + (nslots ? align256((size_t)tiles * sizeof(int)) : 256);
    return p;
}


int wino_filter_impl(const b2c_conv_desc* d, const b2c_tune* t, const float* w, void* ws, size_t ws_bytes,
                     cudaStream_t st) {
    const WinoPlan p = wino_plan(d, t);
    if (!ws || ws_bytes < p.ws_bytes) return fail(B2C_BAD_ARGS, "workspace too small (see b2c_conv_workspace)");
    const long long n = (long long)d->k * d->c;
    k_wino_filter<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(w, reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + p.u_off), d->k, d->c);
    return B2C_OK;
}

int wino_fwd(const b2c_conv_desc* d, const b2c_tune* t, const float* x, const float* w, const float* bias, float* y,
             void* ws, size_t ws_bytes, cudaStream_t st) {
    const WinoPlan p = wino_plan(d, t);
    if (!ws || ws_bytes < p.ws_bytes) return fail(B2C_BAD_ARGS, "workspace too small (see b2c_conv_workspace)");
    int rc = load_tma_encoders();
    if (rc) return rc;
    TconvEntry e = tconv_pick_mode(7, B2C_PREC_FP32, t->tile_n, t->swap_ab, 1, 1);
    if (!e.fn) return fail(B2C_INAPPLICABLE, "no Winograd GEMM kernel for this tile");
    rc = ensure_smem_attr((const void*)e.fn, e.smem);
    if (rc) return rc;
    char* wsb = reinterpret_cast<char*>(ws);
    float* u = reinterpret_cast<float*>(wsb + p.u_off);
    float* v = reinterpret_cast<float*>(wsb + p.v_off);
    float* m = reinterpret_cast<float*>(wsb + p.m_off);
    if (!t->prepared) {
        rc = wino_filter_impl(d, t, w, ws, ws_bytes, st);
        if (rc) return rc;
    }
    // input transform: x -> V[16][P][C]
    {
        const int ws_cols = 2 * p.tiles_x + 2;
        const size_t sm = (size_t)4 * ws_cols * 33 * sizeof(float);
        rc = ensure_smem_attr((const void*)k_wino_input, (int)sm);
        if (rc) return rc;
        cudaError_t le = launch_pdl(k_wino_input, dim3(p.tiles_y, (d->c + WINO_CB - 1) / WINO_CB, d->n), dim3(256), sm, st, 1,
                                    x, v, (int)d->c, (int)d->h, (int)d->w, (int)d->pad, p.tiles_y, p.tiles_x, (long long)p.P);
        if (le != cudaSuccess) return cuda_fail(le, "k_wino_input launch");
    }
    // 16 GEMMs M[z] = V[z] U[z]^T on the tcgen05 3xTF32 kernel (MODE 7)
    {
        CUtensorMap tm_v, tm_u;
        const cuuint64_t vd[3] = {(cuuint64_t)d->c, (cuuint64_t)p.P, 16};
        const cuuint64_t vs[2] = {(cuuint64_t)d->c * 4, (cuuint64_t)p.P * d->c * 4};
        const cuuint32_t vb[3] = {(cuuint32_t)TM_BK, (cuuint32_t)p.pix_rows, 1};
        const cuuint64_t ud[3] = {(cuuint64_t)d->c, (cuuint64_t)d->k, 16};
        const cuuint64_t us[2] = {(cuuint64_t)d->c * 4, (cuuint64_t)d->k * d->c * 4};
        const cuuint32_t ub[3] = {(cuuint32_t)TM_BK, (cuuint32_t)p.flt_rows, 1};
        const cuuint32_t es[3] = {1, 1, 1};
        CUresult r = g_enc_tiled(&tm_v, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, v, vd, vs, vb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(B2C_CUDA_ERROR, "cuTensorMapEncodeTiled (Winograd V) failed (" + std::to_string((int)r) + ")");
        r = g_enc_tiled(&tm_u, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, u, ud, us, ub, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(B2C_CUDA_ERROR, "cuTensorMapEncodeTiled (Winograd U) failed (" + std::to_string((int)r) + ")");
        TArgs a = {};
        a.g = make_geom(&p.gd);
        a.wpk = u;
        a.bias = reinterpret_cast<const float*>(wsb + p.zb_off);  // unused by MODE 7 (no bias in the GEMM)
        a.y = m;
        a.split = p.split;
        a.kps = p.kps;
        a.kblocks = p.kblocks;
        a.streamk = p.streamk;
        a.sk_maxc = p.sk_maxc;
        a.tiles_n = p.tiles_n;
        a.tiles_m = p.tiles_m;
        a.units = (int)p.units;
        a.fCB = FastDiv(1u);
        set_unit_divs(a);
        a.drain = t->drain > 0 ? std::max(2, t->drain) : 4;
        a.ws = reinterpret_cast<float*>(wsb + p.part_off);
        a.sems = reinterpret_cast<int*>(wsb + p.sems_off);
        a.trace_buf = trace_buf();
        a.trace = g_trace_on & 15;
        a.kb_period = p.kblocks;
        a.ksteps_last = std::min(TM_BK / 8, std::max(1, (d->c - TM_BK * (p.kblocks - 1) + 7) / 8));
        const int grid = p.streamk ? p.sk_grid : (int)std::min<long long>(p.units, num_sms());
        cudaError_t le = launch_pdl(e.fn, dim3(grid), dim3(e.threads), (size_t)e.smem, st, 1, tm_v, tm_u, a);
        if (le != cudaSuccess) return cuda_fail(le, "Winograd GEMM launch");
    }
    // output transform: M -> y (+ bias, ReLU)
    {
        const size_t sm = (size_t)WINO_CB * 2 * (2 * p.tiles_x + 1) * sizeof(float);
        auto kout = t->swap_ab ? k_wino_output<false> : k_wino_output<true>;
        rc = ensure_smem_attr((const void*)kout, (int)sm);
        if (rc) return rc;
        cudaError_t le = launch_pdl(kout, dim3(p.tiles_y, (d->k + WINO_CB - 1) / WINO_CB, d->n), dim3(256), sm, st, 1,
                                    (const float*)m, bias, y, (int)d->k, (int)d->oh, (int)d->ow, p.tiles_y, p.tiles_x,
                                    (long long)p.P, (int)d->act);
        if (le != cudaSuccess) return cuda_fail(le, "k_wino_output launch");
    }
    return B2C_OK;
}

int fwd_impl(const b2c_conv_desc* d, const b2c_tune* t, const float* x, const float* w, const float* bias,
             float* y, void* ws, size_t ws_bytes, cudaStream_t st) {
    std::string why;
    int rc = applies_impl(d, t, why);
    if (rc) return fail(rc, why);
    if (!x || !w || !bias || !y) return fail(B2C_BAD_ARGS, "null tensor pointer");
    {
        S2d o;
        if (s2d_of(d, t, o)) {  // first-layer space-to-depth: the rewritten 3x3-class conv on the TMA path
            if (!t->prepared) {
                rc = pack_impl(d, t, w, ws, ws_bytes, st);
                if (rc) return rc;
            }
            const UmmaPlan p2 = umma_plan(&o.d2, &o.t2);
            if (!ws || ws_bytes < p2.ws_bytes) return fail(B2C_BAD_ARGS, "workspace too small (see b2c_conv_workspace)");
            rc = tma_fwd(&o.d2, &o.t2, p2, make_geom(&o.d2), x, w, bias, y, ws, st, d);
            if (rc) return rc;
            cudaError_t le = cudaGetLastError();
            return le == cudaSuccess ? B2C_OK : cuda_fail(le, "kernel launch");
        }
    }
    const Geom g = make_geom(d);
    switch (t->variant) {
        case B2C_VAR_SIMPLE: {
            const long long total = (long long)g.N * g.OC * g.PQ;
            const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 64);
            k_simple<<<blocks, 256, 0, st>>>(g, x, w, bias, y);
            break;
        }
        case B2C_VAR_TILED: {
            TiledKernel fn = tiled_pick(t->mnt0, t->mnt1);
            if (!fn) return fail(B2C_INAPPLICABLE, "no kernel for this register block");
            const int BM = t->mnb0 * t->mnt0, BN = t->mnb1 * t->mnt1;
            const size_t sm = tiled_smem_bytes(BM, BN, t->kb);
            rc = ensure_smem_attr((const void*)fn, (int)sm);
            if (rc) return rc;
            dim3 grid((g.M + BM - 1) / BM, (g.OC + BN - 1) / BN);
            fn<<<grid, t->mnb0 * t->mnb1, sm, st>>>(g, x, w, bias, y, t->mnb0, t->mnb1, t->kb);
            break;
        }
        case B2C_VAR_WINO:
            rc = wino_fwd(d, t, x, w, bias, y, ws, ws_bytes, st);
            if (rc) return rc;
            break;
        case B2C_VAR_FC_STREAM: {
            using FcsKernel = void (*)(const float*, const float*, const float*, float*, int, int, int, int);
            if (t->kb == 3) {  // TMA bulk ring (k_fc_bulk)
                using FcbKernel = void (*)(const float*, const float*, const float*, float*, int, int, int, int, int, int);
                const int nb = d->n <= 1 ? 1 : d->n <= 2 ? 2 : d->n <= 4 ? 4 : 8;
                FcbKernel fn = nb == 1 ? k_fc_bulk<1> : nb == 2 ? k_fc_bulk<2> : nb == 4 ? k_fc_bulk<4> : k_fc_bulk<8>;
                const int rpc = fcb_rows_per_cta(g.OC);
                const int stage_bytes = (rpc + g.N) * FCB_KC * (int)sizeof(float);
                const int nst = std::min(8, (TM_MAX_SMEM - FCB_HDR) / stage_bytes);
                if (nst < 2) return fail(B2C_INAPPLICABLE, "k_fc_bulk: fewer than two stages fit");
                const int sm = FCB_HDR + nst * stage_bytes;
                rc = ensure_smem_attr((const void*)fn, sm);
                if (rc) return rc;
                const int nblocks = (g.OC + rpc - 1) / rpc;
                fn<<<std::min(nblocks, num_sms()), 32 * (FCB_WARPS + 1), sm, st>>>(x, w, bias, y, g.N, g.OC, g.K, g.act, rpc, nst);
                break;
            }
            if (t->kb == 2) {
                const int nb = d->n <= 1 ? 1 : d->n <= 2 ? 2 : d->n <= 4 ? 4 : d->n <= 8 ? 8 : d->n <= 16 ? 16 : d->n <= 20 ? 20 : 32;
                const int R = t->mnt1;
                FcsKernel fn = nullptr;
#define B2C_FCM(NB_, R_) if (nb == NB_ && R == R_) fn = k_fc_smem<NB_, R_>;
                B2C_FCM(1, 1) B2C_FCM(2, 1) B2C_FCM(4, 1) B2C_FCM(8, 1) B2C_FCM(16, 1) B2C_FCM(20, 1) B2C_FCM(32, 1)
                B2C_FCM(1, 2) B2C_FCM(2, 2) B2C_FCM(4, 2) B2C_FCM(8, 2) B2C_FCM(16, 2) B2C_FCM(20, 2) B2C_FCM(32, 2)
                B2C_FCM(1, 4) B2C_FCM(2, 4) B2C_FCM(4, 4) B2C_FCM(8, 4) B2C_FCM(16, 4)
#undef B2C_FCM
                if (!fn) return fail(B2C_INAPPLICABLE, "no staged weight-streaming kernel for this batch / rows");
                const int W = t->mnb0;
                const int sm = 2 * nb * FCS_KC * (int)sizeof(float);
                rc = ensure_smem_attr((const void*)fn, sm);
                if (rc) return rc;
                fn<<<(g.OC + W * R - 1) / (W * R), 32 * W, sm, st>>>(x, w, bias, y, g.N, g.OC, g.K, g.act);
                break;
            }
            const int nb = d->n <= 1 ? 1 : d->n <= 2 ? 2 : d->n <= 4 ? 4 : 8;
            const int R = t->mnt1;
            FcsKernel fn = nullptr;
#define B2C_FCS(NB_, R_) if (nb == NB_ && R == R_) fn = k_fc_stream<NB_, R_>;
            B2C_FCS(1, 2) B2C_FCS(2, 2) B2C_FCS(4, 2) B2C_FCS(8, 2)
            B2C_FCS(1, 4) B2C_FCS(2, 4) B2C_FCS(4, 4) B2C_FCS(8, 4)
            B2C_FCS(1, 8) B2C_FCS(2, 8) B2C_FCS(4, 8) B2C_FCS(8, 8)
#undef B2C_FCS
            if (!fn) return fail(B2C_INAPPLICABLE, "no weight-streaming kernel for this shape");
            const int W = t->mnb0;
            const size_t sm = (size_t)W * R * nb * sizeof(float);
            fn<<<(g.OC + R - 1) / R, 32 * W, sm, st>>>(x, w, bias, y, g.N, g.OC, g.K, g.act);
            break;
        }
        default: {
            const UmmaPlan p = umma_plan(d, t);
            UmmaEntry e = umma_pick(t->tile_n, t->swap_ab, p.kmode);
            if (!e.fn && !t->tma) return fail(B2C_INAPPLICABLE, "no tcgen05 kernel for this tile");  // (TMA tiles: tma_fwd picks)
            if (p.ws_bytes > 0 && (!ws || ws_bytes < p.ws_bytes))
                return fail(B2C_BAD_ARGS, "workspace too small (see b2c_conv_workspace)");
            if (!t->prepared) {
                rc = pack_impl(d, t, w, ws, ws_bytes, st);
                if (rc) return rc;
            }
            if (t->tma) {
                rc = tma_fwd(d, t, p, g, x, w, bias, y, ws, st);
                if (rc) return rc;
                break;
            }
            rc = ensure_smem_attr((const void*)e.fn, e.smem);
            if (rc) return rc;
            UmmaArgs a;
            a.g = g;
            a.x = x;
            a.wpk = reinterpret_cast<const float*>(ws);
            a.bias = bias;
            a.y = y;
            a.split = p.split;
            a.kps = p.kps;
            a.kblocks = p.kblocks;
            a.fCB = FastDiv((uint32_t)p.cblocks);
            a.drain = t->drain > 0 ? std::max(2, t->drain) : 4;
            a.lag = std::max(0, std::min(a.drain - 2, e.stages - 1));
            a.wpk_elems = (long long)p.wpk_bytes / 4;
            {
                const long long op_bytes = 4ll * ((long long)d->n * d->c * d->h * d->w) + (long long)p.wpk_bytes;
                a.prefetch = (t->stages >= 0 && op_bytes <= (48ll << 20)) ? 1 : 0;  // stages < 0: disable
            }
            a.ws = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + p.part_off);
            a.sems = reinterpret_cast<int*>(reinterpret_cast<char*>(ws) + p.sems_off);
            dim3 grid(p.grid_x, p.grid_y, p.split);
            e.fn<<<grid, UMMA_THREADS, e.smem, st>>>(a);
            break;
        }
    }
    cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess) return cuda_fail(le, "kernel launch");
    return B2C_OK;
}

// L2 flush buffer (one per device), larger than the 126 MB L2.
std::mutex g_flush_mu;
std::vector<std::pair<int, void*>> g_flush;
constexpr size_t kFlushBytes = 256ull << 20;

// Reads the flush buffer (2x L2) so that L2 ends up holding clean lines of it.
// A memset flush would leave ~L2-sized dirty data whose write-back the timed
// kernel then pays for (~19 us at HBM peak), which hid the differences between
// HBM-bound candidates in the tuner.
__global__ void __launch_bounds__(256) k_flush_read(const int4* __restrict__ p, long long n, int* sink) {
    int acc = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int4 v = __ldcg(p + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x7fffffff) *sink = acc;  // practically never; keeps the loads alive
}

int flush_l2(cudaStream_t st) {
    int dev = 0;
    B2C_CUDA(cudaGetDevice(&dev));
    void* buf = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_flush_mu);
        for (auto& e : g_flush)
            if (e.first == dev) buf = e.second;
        if (!buf) {
            B2C_CUDA(cudaMalloc(&buf, kFlushBytes + 256));
            B2C_CUDA(cudaMemset(buf, 0, kFlushBytes + 256));
            B2C_CUDA(cudaDeviceSynchronize());
            g_flush.emplace_back(dev, buf);
        }
    }
    k_flush_read<<<num_sms() * 8, 256, 0, st>>>(reinterpret_cast<const int4*>(buf), (long long)(kFlushBytes / 16),
                                                reinterpret_cast<int*>(reinterpret_cast<char*>(buf) + kFlushBytes));
    B2C_CUDA(cudaGetLastError());
    return B2C_OK;
}

}  // namespace

namespace b2c {
// shared with b2net.cu: one thread-local last-error slot for the whole library
int set_last_error(int code, const char* msg) { return fail(code, msg); }
}  // namespace b2c

// ============================================================================ C ABI

extern "C" {

int b2c_conv_applies(const b2c_conv_desc* d, const b2c_tune* t, char* reason, size_t n) {
    std::string why;
    const int rc = applies_impl(d, t, why);
    if (reason && n) {
        std::snprintf(reason, n, "%s", rc ? why.c_str() : "");
    }
    if (rc) g_last_error = why;
    return rc;
}

size_t b2c_conv_workspace(const b2c_conv_desc* d, const b2c_tune* t) {
    std::string why;
    if (applies_impl(d, t, why)) return 0;
    if (t->variant == B2C_VAR_WINO) return wino_plan(d, t).ws_bytes;
    S2d o;
    if (s2d_of(d, t, o))  // the rewritten conv's workspace + the re-arranged filters (used while packing)
        return umma_plan(&o.d2, &o.t2).ws_bytes + align256((size_t)o.d2.k * o.d2.c * o.d2.r * o.d2.r * sizeof(float));
    if (!is_umma(t->variant)) return 0;
    return umma_plan(d, t).ws_bytes;
}

int b2c_conv_prepare(const b2c_conv_desc* d, const b2c_tune* t, const float* w, void* workspace, size_t ws_bytes,
                     void* stream) {
    std::string why;
    int rc = applies_impl(d, t, why);
    if (rc) return fail(rc, why);
    if (!is_umma(t->variant) && t->variant != B2C_VAR_WINO) return B2C_OK;
    if (!w) return fail(B2C_BAD_ARGS, "null filter pointer");
    rc = t->variant == B2C_VAR_WINO
             ? wino_filter_impl(d, t, w, workspace, ws_bytes, reinterpret_cast<cudaStream_t>(stream))
             : pack_impl(d, t, w, workspace, ws_bytes, reinterpret_cast<cudaStream_t>(stream));
    if (rc) return rc;
    cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess) return cuda_fail(le, "pack launch");
    // One-time setup call: complete the pack before returning, so that later
    // launches with prepared != 0 may read it without ordering on the stream
    // (the TMA kernel fetches filters ahead of griddepcontrol.wait).
    le = cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream));
    if (le != cudaSuccess) return cuda_fail(le, "pack synchronize");
    return B2C_OK;
}

int b2c_conv_fwd(const b2c_conv_desc* d, const b2c_tune* t, const float* x, const float* w, const float* bias,
                 float* y, void* workspace, size_t ws_bytes, void* stream) {
    return fwd_impl(d, t, x, w, bias, y, workspace, ws_bytes, reinterpret_cast<cudaStream_t>(stream));
}

int b2c_conv_time(const b2c_conv_desc* d, const b2c_tune* t, const float* x, const float* w, const float* bias,
                  float* y, void* workspace, size_t ws_bytes, void* stream, int warmup, int reps, int l2_flush,
                  float* median_ms) {
    if (!median_ms || reps < 1 || warmup < 0) return fail(B2C_BAD_ARGS, "bad timing arguments");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    for (int i = 0; i < warmup; ++i) {
        int rc = fwd_impl(d, t, x, w, bias, y, workspace, ws_bytes, st);
        if (rc) return rc;
    }
    std::vector<float> ms(reps);
    cudaEvent_t e0, e1;
    B2C_CUDA(cudaEventCreate(&e0));
    B2C_CUDA(cudaEventCreate(&e1));
    int rc = B2C_OK;
    for (int i = 0; i < reps && rc == B2C_OK; ++i) {
        if (l2_flush) rc = flush_l2(st);
        if (rc) break;
        cudaEventRecord(e0, st);
        rc = fwd_impl(d, t, x, w, bias, y, workspace, ws_bytes, st);
        cudaEventRecord(e1, st);
        if (rc) break;
        cudaError_t se = cudaEventSynchronize(e1);
        if (se != cudaSuccess) { rc = cuda_fail(se, "cudaEventSynchronize"); break; }
        cudaEventElapsedTime(&ms[i], e0, e1);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (rc) return rc;
    std::sort(ms.begin(), ms.end());
    *median_ms = ms[reps / 2];
    return B2C_OK;
}

size_t b2c_conv_host_scratch(const b2c_conv_desc* d, const b2c_tune* t) {
    if (check_desc(d)) return 0;
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t xb = (size_t)d->n * d->c * d->h * d->w * 4;
    const size_t wb = (size_t)d->k * d->c * d->r * d->r * 4;
    const size_t bb = (size_t)d->k * 4;
    const size_t yb = (size_t)d->n * d->k * d->oh * d->ow * 4;
    return al(xb) + al(wb) + al(bb) + al(yb) + al(b2c_conv_workspace(d, t));
}

int b2c_conv_fwd_host(const b2c_conv_desc* d, const b2c_tune* t, const float* hx, const float* hw,
                      const float* hbias, float* hy, void* dev_scratch, size_t scratch_bytes, void* stream) {
    int rc = check_desc(d);
    if (rc) return rc;
    if (!hx || !hw || !hbias || !hy || !dev_scratch) return fail(B2C_BAD_ARGS, "null pointer");
    const size_t need = b2c_conv_host_scratch(d, t);
    if (scratch_bytes < need) return fail(B2C_BAD_ARGS, "device scratch too small (b2c_conv_host_scratch)");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t xb = (size_t)d->n * d->c * d->h * d->w * 4;
    const size_t wb = (size_t)d->k * d->c * d->r * d->r * 4;
    const size_t bb = (size_t)d->k * 4;
    const size_t yb = (size_t)d->n * d->k * d->oh * d->ow * 4;
    char* p = reinterpret_cast<char*>(dev_scratch);
    float* dx = reinterpret_cast<float*>(p); p += al(xb);
    float* dw = reinterpret_cast<float*>(p); p += al(wb);
    float* db = reinterpret_cast<float*>(p); p += al(bb);
    float* dy = reinterpret_cast<float*>(p); p += al(yb);
    void* ws = p;
    const size_t wsb = b2c_conv_workspace(d, t);
    // The split-K / stream-K tickets and the grid-barrier counter must be zero at
    // rest; the scratch may be fresh (uninitialised) device memory, so zero them
    // on the stream (a few bytes; the partials themselves need no init).
    if (wsb && t->variant == B2C_VAR_WINO) {
        const WinoPlan wp = wino_plan(d, t);
        B2C_CUDA(cudaMemsetAsync(reinterpret_cast<char*>(ws) + wp.sems_off, 0, wp.ws_bytes - wp.sems_off, st));
    }
    if (wsb && is_umma(t->variant)) {
        S2d o;
        const bool s2d = s2d_of(d, t, o);
        const UmmaPlan up = s2d ? umma_plan(&o.d2, &o.t2) : umma_plan(d, t);
        if (up.nhwc_off > up.sems_off)
            B2C_CUDA(cudaMemsetAsync(reinterpret_cast<char*>(ws) + up.sems_off, 0, up.nhwc_off - up.sems_off, st));
        if (up.ws_bytes > up.gbar_off)
            B2C_CUDA(cudaMemsetAsync(reinterpret_cast<char*>(ws) + up.gbar_off, 0, up.ws_bytes - up.gbar_off, st));
    }
    B2C_CUDA(cudaMemcpyAsync(dx, hx, xb, cudaMemcpyHostToDevice, st));
    B2C_CUDA(cudaMemcpyAsync(dw, hw, wb, cudaMemcpyHostToDevice, st));
    B2C_CUDA(cudaMemcpyAsync(db, hbias, bb, cudaMemcpyHostToDevice, st));
    b2c_tune tt = *t;
    tt.prepared = 0;  // filters arrive fresh from the host: pack them in this call
    rc = fwd_impl(d, &tt, dx, dw, db, dy, ws, wsb, st);
    if (rc) return rc;
    B2C_CUDA(cudaMemcpyAsync(hy, dy, yb, cudaMemcpyDeviceToHost, st));
    return B2C_OK;
}

int64_t b2c_conv_flops(const b2c_conv_desc* d) {
    if (!d) return 0;
    return 2ll * d->r * d->r * d->c * d->k * d->oh * d->ow * d->n;
}

int64_t b2c_conv_bytes(const b2c_conv_desc* d) {
    if (!d) return 0;
    return 4ll * ((int64_t)d->n * d->c * d->h * d->w + (int64_t)d->k * d->c * d->r * d->r + d->k +
                  (int64_t)d->n * d->k * d->oh * d->ow);
}

int b2c_conv_launches(const b2c_conv_desc* d, const b2c_tune* t) {
    (void)d;
    if (!t) return 0;
    if (t->variant == B2C_VAR_WINO) return 3 + (t->prepared ? 0 : 1);  // input transform, GEMM, output transform
    if (t->tma == 6) return 2 + (t->prepared ? 0 : 2);  // s2d copy + conv (+ filter re-arrangement + pack)
    const int pack = (is_umma(t->variant) && !t->prepared && !(t->tma && t->variant == B2C_VAR_FC)) ? 1 : 0;
    const bool sep = std::getenv("B2C_FUSED_NHWC") == nullptr || (t->tma == 2 && d && d->c <= 4);
    const int nhwc = (is_umma(t->variant) && t->tma && t->tma != 3 && t->tma != 4 && t->variant != B2C_VAR_FC && sep) ? 1 : 0;
    return 1 + pack + nhwc;
}

const char* b2c_last_error(void) { return g_last_error.c_str(); }

int b2c_conv_grid(const b2c_conv_desc* d, const b2c_tune* t) {
    std::string why;
    if (applies_impl(d, t, why)) return 0;
    const Geom g = make_geom(d);
    switch (t->variant) {
        case B2C_VAR_SIMPLE:
            return (int)std::min<long long>(((long long)g.N * g.OC * g.PQ + 255) / 256, 148LL * 64);
        case B2C_VAR_TILED: {
            const int BM = t->mnb0 * t->mnt0, BN = t->mnb1 * t->mnt1;
            return ((g.M + BM - 1) / BM) * ((g.OC + BN - 1) / BN);
        }
        case B2C_VAR_WINO: {
            const WinoPlan p = wino_plan(d, t);
            return p.streamk ? p.sk_grid : (int)std::min<long long>(p.units, num_sms());
        }
        case B2C_VAR_FC_STREAM:
            if (t->kb == 3) {
                const int rpc = fcb_rows_per_cta(g.OC);
                return std::min((g.OC + rpc - 1) / rpc, num_sms());
            }
            return t->kb == 2 ? (g.OC + t->mnb0 * t->mnt1 - 1) / (t->mnb0 * t->mnt1) : (g.OC + t->mnt1 - 1) / t->mnt1;
        default: {
            S2d o;
            if (s2d_of(d, t, o)) return b2c_conv_grid(&o.d2, &o.t2);
            const UmmaPlan p = umma_plan(d, t);
            if (!t->tma) return p.grid_x * p.grid_y * p.split;
            const int occ = t->stages == 2 ? 2 : 1, cl = (t->cluster == 2 || t->cluster == 3) ? 2 : 1;
            const int units = (cl == 2 ? (p.grid_x + 1) / 2 * p.grid_y : p.tiles) * p.split;
            if (t->cluster == 4) return p.split * std::min(p.tiles, std::max(1, num_sms() / p.split));
            return p.streamk ? p.sk_grid : cl == 2 ? 2 * std::min(units, num_sms() / 2) : std::min(units, occ * num_sms());
        }
    }
}

void* b2c_device_alloc(size_t bytes) {
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes ? bytes : 1);
    if (e != cudaSuccess) {
        cuda_fail(e, "cudaMalloc");
        return nullptr;
    }
    e = cudaMemset(p, 0, bytes ? bytes : 1);
    if (e != cudaSuccess) {
        cuda_fail(e, "cudaMemset");
        cudaFree(p);
        return nullptr;
    }
    return p;
}

int b2c_device_free(void* p) {
    if (!p) return B2C_OK;
    B2C_CUDA(cudaFree(p));
    return B2C_OK;
}

int b2c_stream_synchronize(void* stream) {
    B2C_CUDA(cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream)));
    return B2C_OK;
}

/* Debug only (not part of include/b2conv.h): enable the phase trace of the
 * TMA kernel's CTA 0 and read it back (256 clock64 stamps). */
void b2c_debug_trace_enable(int on) { g_trace_on = on; }
int b2c_debug_trace_read(long long* out) {
    return cudaMemcpyFromSymbol(out, b2c::g_b2c_trace, sizeof(long long) * 256) == cudaSuccess ? 0 : 3;
}

const char* b2c_version(void) { return "b2conv 0.1.0 sm_100a"; }

}  // extern "C"
