// tcgen05 / TMEM implicit-GEMM convolution, fp32-exact via 3xTF32.
//
// The GEMM view is the reference ConvTiled's (cuclgen/variants.py:376-414):
// M = img*oy*ox output pixels, N = out_chan, K = in_chan*ksz*ksz, with the
// bias/ReLU epilogue of variants.py:160-165 and graphopt.fuse_activations
// (graphopt.py:59-86) fused into the TMEM drain.  The reduction order is
// free at the reference tolerance ("summation order is immaterial",
// oracle.py:69-74), so K is walked in whichever order loads best:
//   KMODE 3  tap-major: K block = (tap ky,kx ; 32 input channels).  Within a
//            block the tap is fixed, so a pixel row needs ONE bounds check and
//            its 32 values are one strided load each.  conv_umma (C >= 32),
//            conv_1x1 (variants.py:279-325).
//   KMODE 0  flat (ic, ky, kx) walk, for first layers with C = 3
//            (AlexNet/NiN conv1, GoogLeNet conv1) where tap-major would pad
//            3 channels to 32.
//   KMODE 2  whole-image filter = one flat contiguous K row per image
//            (conv_fc, variants.py:328-373, K = ic*h*w flattened at :354-356).
// SWAP=false: MMA M = 128 output pixels, MMA N = BN out_chans (TMEM lane =
// pixel, so the NCHW epilogue store is coalesced along pixels).
// SWAP=true : MMA M = 128 out_chans, MMA N = BN pixels (small maps, fc).
//
// Precision: tcgen05 kind::tf32 reads an fp32 operand by truncating it to
// TF32 (measured: tools/tf32_probe.cu).  So the raw fp32 value IS the "hi"
// operand, and producers add lo = x - trunc_tf32(x) (exact in fp32);
// D += Ahi*Bhi + Ahi*Blo + Alo*Bhi ("3xTF32"), lo*lo dropped (~2^-21 rel).
//
// Accumulation precision: the tensor core adds each MMA into the fp32 TMEM
// accumulator with truncation; measured on B200 the error grows ~6.5e-8
// (relative) per MMA issued into one accumulator (~5e-5 at K = 2304, over
// the 1e-5 budget).  So K is accumulated in chunks of `drain` K blocks
// (12*drain MMAs) into one of two TMEM slots; while the tensor core fills
// one slot, the producer warps drain the other with tcgen05.ld into fp32
// round-to-nearest register sums.  Chunk error ~7.8e-7*drain, any K.
//
// Operand staging.  Filters are constant per op, so b2c_conv_prepare packs
// them once (cached in workspace) into "UMMA-ready" tiles:
// per (filter tile, K block) the exact smem image [raw rows][lo rows], which
// warp 9 streams with one cp.async.bulk per stage (TMA engine, no register
// traffic).  Activations are gathered by warps 0-7 in two groups of four
// (group g produces K blocks g, g+2, ...; two K blocks of loads in flight per
// SM): each thread owns one output pixel's im2col row, loads its 32 values
// (tap-major: one bounds check, 32 coalesced-across-lanes strided loads),
// and stores raw + lo as 16-byte chunks.  Every operand uses the K-major
// no-swizzle layout [chunk c = k/4][row][16 B] (LBO = rows*16 B between
// K-adjacent core matrices, SBO = 128 B between 8-row groups), so a warp's
// 32 consecutive rows store as 512 contiguous bytes.  Warp 8 allocates TMEM;
// its lane 0 issues 12 tcgen05.mma per K block (4 K=8 steps x 3 terms) and
// releases stages with tcgen05.commit.  Warps 0-7 drain the TMEM chunks
// (warp w: lane quarter w%4, column half w/4) and run the epilogue: + bias,
// ReLU, NCHW stores.  Split-K CTAs write partials to workspace; the last CTA
// of a tile (atomic ticket) reduces them in split order (deterministic).
#pragma once
#include <cuda_bf16.h>
#include "common.cuh"

namespace b2c {

constexpr int UMMA_M = 128;
constexpr int UMMA_BK = 32;          // fp32 elements of K per pipeline stage
constexpr int UMMA_GROUP = 128;      // pixel-producer threads per group
constexpr int UMMA_GROUPS = 2;       // producer groups (K blocks in flight)
constexpr int UMMA_PRODUCERS = UMMA_GROUP * UMMA_GROUPS;
constexpr int UMMA_MMA_WARP = UMMA_PRODUCERS / 32;      // warp 8
constexpr int UMMA_LOAD_WARP = UMMA_MMA_WARP + 1;       // warp 9
constexpr int UMMA_THREADS = UMMA_PRODUCERS + 64;
constexpr int UMMA_SMEM_HDR = 1024;  // barriers + TMEM slot + flags

template <int BN, bool SWAP>
struct UmmaCfg {
    static_assert(BN % 32 == 0 && BN >= 32 && BN <= 192, "BN: multiple of 32 in [32, 192]");
    static constexpr int A_ROWS = UMMA_M;
    static constexpr int B_ROWS = BN;
    static constexpr int PIX_ROWS = SWAP ? B_ROWS : A_ROWS;   // gathered by producers
    static constexpr int FLT_ROWS = SWAP ? A_ROWS : B_ROWS;   // bulk-copied, pre-packed
    static constexpr int PART = UMMA_BK * 4;                  // bytes per row per part (128)
    static constexpr int A_BYTES = 2 * A_ROWS * PART;         // raw + lo
    static constexpr int B_BYTES = 2 * B_ROWS * PART;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int FLT_STAGE_BYTES = 2 * FLT_ROWS * PART;
    static constexpr int BUDGET = 220 * 1024 - UMMA_SMEM_HDR;
    static constexpr int STAGES = (BUDGET / STAGE_BYTES) > 8 ? 8 : (BUDGET / STAGE_BYTES);
    static constexpr int SMEM = UMMA_SMEM_HDR + STAGES * STAGE_BYTES;
    static constexpr int TMEM_COLS = 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
    static constexpr int NROWS = (PIX_ROWS + UMMA_GROUP - 1) / UMMA_GROUP;
    static constexpr int HALF = BN / 2;  // accumulator columns per producer warp
    static_assert(STAGES >= 2, "need at least two stages");
    static_assert(HALF % 8 == 0, "TMEM drain granularity");
};

struct UmmaArgs {
    Geom g;
    const float* x;
    const float* wpk;   // packed filters [flt tile][K block][raw|lo][chunk][row][4]
    const float* bias;
    float* y;
    float* ws;          // split-K partials [tiles][split][BN][128]
    int* sems;          // split-K tickets [tiles], zero at rest
    int split;          // number of K splits (gridDim.z)
    int kps;            // K blocks per split
    int kblocks;        // K blocks in the whole reduction
    FastDiv fCB;        // KMODE 3: divides by ceil(C/32) channel blocks per tap
    int drain;          // K blocks per TMEM chunk before a register drain (>= 2)
    int lag;            // a group drains chunk c before its first K block >= (c+1)*drain + lag
    int prefetch;       // 1: CTAs cooperatively bulk-prefetch x and packed w into L2 at start
    long long wpk_elems;
};

// Per K block, everything uniform across the CTA.
struct KBlock {
    int k0;      // KMODE 0/2: first flat k
    int ic0;     // KMODE 3: first channel
    int ky, kx;  // KMODE 3: tap
    int nvalid;  // real K entries in this block (<= 32)
};

__device__ __forceinline__ KBlock kblock_info(const Geom& g, int kb, const FastDiv& fcb, int kmode) {
    KBlock k;
    if (kmode == 3) {
        uint32_t tap, cb, ky, kx;
        fcb.divmod((uint32_t)kb, tap, cb);
        g.fR.divmod(tap, ky, kx);
        k.ic0 = (int)cb * UMMA_BK;
        k.ky = (int)ky;
        k.kx = (int)kx;
        k.nvalid = min(UMMA_BK, g.C - k.ic0);
        k.k0 = 0;
    } else {
        k.k0 = kb * UMMA_BK;
        k.ic0 = k.ky = k.kx = 0;
        k.nvalid = min(UMMA_BK, g.K - k.k0);
    }
    return k;
}

// One output pixel's im2col row.
struct PixRow {
    const float* base;  // KMODE 3: x + b*C*HW ; KMODE 0: x + b*C*HW + iy0*W + ix0 ; KMODE 2: x + b*K
    int iy0, ix0;
    bool valid;
};

template <int KMODE>
__device__ __forceinline__ void load_pixel_row(const Geom& g, const PixRow& rs, const KBlock& kb, float (&v)[32]) {
    if (KMODE == 2) {  // whole-image filter: a contiguous K row per image
        if ((g.K & 3) == 0) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const int k = kb.k0 + 4 * c;
                float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
                if (rs.valid && k < g.K) q = __ldg(reinterpret_cast<const float4*>(rs.base + k));
                v[4 * c] = q.x; v[4 * c + 1] = q.y; v[4 * c + 2] = q.z; v[4 * c + 3] = q.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = (rs.valid && j < kb.nvalid) ? __ldg(rs.base + kb.k0 + j) : 0.0f;
        }
    } else if (KMODE == 3) {  // tap-major: fixed tap, 32 channels at stride HW
        const int iy = rs.iy0 + kb.ky, ix = rs.ix0 + kb.kx;
        const bool ok = rs.valid && (unsigned)iy < (unsigned)g.H && (unsigned)ix < (unsigned)g.W;
        const float* p = rs.base + (long long)kb.ic0 * g.HW + iy * g.W + ix;
        if (ok && kb.nvalid == 32) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __ldg(p + (long long)j * g.HW);
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = (ok && j < kb.nvalid) ? __ldg(p + (long long)j * g.HW) : 0.0f;
        }
    } else {  // flat (ic, ky, kx) walk from k0 (first layers, C < 32)
        uint32_t ic, rem, ky, kx;
        g.fRR.divmod((uint32_t)kb.k0, ic, rem);
        g.fR.divmod(rem, ky, kx);
        int koff = (int)ic * g.HW + (int)ky * g.W + (int)kx;
        int iky = (int)ky, ikx = (int)kx;
        const int wrap_x = g.W - g.R, wrap_y = g.HW - g.R * g.W;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const int iy = rs.iy0 + iky, ix = rs.ix0 + ikx;
            const bool ok = rs.valid && (j < kb.nvalid) && (unsigned)iy < (unsigned)g.H && (unsigned)ix < (unsigned)g.W;
            v[j] = ok ? __ldg(rs.base + koff) : 0.0f;
            ++ikx;
            ++koff;
            if (ikx == g.R) {
                ikx = 0;
                ++iky;
                koff += wrap_x;
                if (iky == g.R) {
                    iky = 0;
                    koff += wrap_y;
                }
            }
        }
    }
}

// Store one row's 32 K values as raw fp32 (read as TF32 = hi by the tensor
// core) and lo = x - trunc_tf32(x), chunk c at part_base + c*rows*16.
__device__ __forceinline__ void store_row_split(uint32_t raw_row, uint32_t lo_row, uint32_t chunk_stride,
                                                const float (&v)[32]) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        float l[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            float h;
            split_tf32(v[4 * c + e], h, l[e]);
        }
        sts128(raw_row + c * chunk_stride, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
        sts128(lo_row + c * chunk_stride, l[0], l[1], l[2], l[3]);
    }
}

template <int N>
__device__ __forceinline__ void tmem_add_cols(uint32_t taddr, float* acc) {
    static_assert(N % 8 == 0, "");
    int c = 0;
#pragma unroll
    for (; c + 16 <= N; c += 16) {
        float v[16];
        tmem_ld16(taddr + (uint32_t)c, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[c + j] += v[j];
    }
    if (c < N) {
        float v[8];
        tmem_ld8(taddr + (uint32_t)c, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[c + j] += v[j];
    }
}

// --------------------------------------------------------------------------- filter packing
// packed[((t*KB + kb)*2 + part)*8*ROWS*4 + (c*ROWS + r)*4 + e] =
//   part 0: W[oc][k], part 1: W - trunc_tf32(W), oc = t*ROWS + r, k = k-index(kb, 4c+e)
// swz != 0 writes each (tile, K block, part) as 128-byte rows with 16-byte
// chunks XOR-swizzled by row % 8 (the SWIZZLE_128B image k_tconv reads).
// parts == 1 packs the raw half only (k_tconv computes lo itself when the
// filter tile is its TMEM A operand).
// Filter value at K position kk (0..31) of K block kb for out_chan oc, in the
// K order of `kmode` (see kmode_for in b2conv.cu); 0 past the real K.
__device__ __forceinline__ float packed_k_value(const Geom& g, const float* __restrict__ w, int oc, int kb, int kk,
                                                FastDiv fCB, int kmode) {
    if (oc >= g.OC) return 0.0f;
    if (kmode == 3) {
        uint32_t tap, cb, ky, kx;
        fCB.divmod((uint32_t)kb, tap, cb);
        g.fR.divmod(tap, ky, kx);
        const int ic = (int)cb * UMMA_BK + kk;
        return ic < g.C ? w[(long long)oc * g.K + ((long long)ic * g.R + ky) * g.R + kx] : 0.0f;
    }
    if (kmode == 5) {
        uint32_t ky, kc;
        fCB.divmod((uint32_t)kb, ky, kc);
        const int wi = (int)kc * 32 + kk;
        const int kx = wi >> 2, ch = wi & 3;
        return (kx < g.R && ch < g.C) ? w[(long long)oc * g.K + ((long long)ch * g.R + ky) * g.R + kx] : 0.0f;
    }
    if (kmode == 4) {
        const int tap = kb * 8 + (kk >> 2), ch = kk & 3;
        return (tap < g.RR && ch < g.C) ? w[(long long)oc * g.K + (long long)ch * g.RR + tap] : 0.0f;
    }
    const int k = kb * UMMA_BK + kk;
    return k < g.K ? w[(long long)oc * g.K + k] : 0.0f;
}
#ifndef B2C_INST_TU  // (non-template kernel: defined in b2conv.cu's translation unit only)

// bf16 pack for the TMA kernel's bf16 mode: [filter tile][K block][8-element chunk 0..3][rows][8 x bf16]
// (UMMA no-swizzle K-major core matrices: 8 rows x 16 B contiguous), round to nearest even.
__global__ void __launch_bounds__(256) k_pack_filters_bf16(Geom g, const float* __restrict__ w,
                                                           uint16_t* __restrict__ out, int rows, int kblocks,
                                                           FastDiv fCB, int kmode, long long total) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int e = (int)(i & 7);
        long long t = i >> 3;
        const int r = (int)(t % rows);
        t /= rows;
        const int c = (int)(t & 3);
        t >>= 2;
        const int kb = (int)(t % kblocks);
        const int tile = (int)(t / kblocks);
        const float v = packed_k_value(g, w, tile * rows + r, kb, 8 * c + e, fCB, kmode);
        out[i] = __bfloat16_as_ushort(__float2bfloat16_rn(v));
    }
}
#endif
#ifndef B2C_INST_TU  // (non-template kernel: defined in b2conv.cu's translation unit only)

// bf16 pack for MODE 8 (tm=5): per (filter tile, K block of 64 channels of one tap) the
// SWIZZLE_128B K-major image the SS MMAs read: rows of 128 B (64 bf16), 16-byte chunk c
// (elements 8c..8c+7) stored at chunk position c ^ (row % 8).
__global__ void __launch_bounds__(256) k_pack_filters_bf16_sw128(Geom g, const float* __restrict__ w,
                                                                 uint16_t* __restrict__ out, int rows, int kblocks,
                                                                 FastDiv fCB, long long total) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int e = (int)(i & 7);        // element within the stored 16-byte chunk
        const int pc = (int)((i >> 3) & 7);  // stored chunk position in the 128-byte row
        long long t = i >> 6;
        const int r = (int)(t % rows);
        t /= rows;
        const int kb = (int)(t % kblocks);
        const int tile = (int)(t / kblocks);
        const int c = pc ^ (r & 7);  // logical chunk
        const int oc = tile * rows + r;
        uint32_t tap, cb, ky, kx;
        fCB.divmod((uint32_t)kb, tap, cb);
        g.fR.divmod(tap, ky, kx);
        const int ic = (int)cb * 64 + 8 * c + e;
        const float v = (oc < g.OC && ic < g.C) ? w[(long long)oc * g.K + ((long long)ic * g.R + ky) * g.R + kx] : 0.0f;
        out[i] = __bfloat16_as_ushort(__float2bfloat16_rn(v));
    }
}
#endif
#ifndef B2C_INST_TU  // (non-template kernel: defined in b2conv.cu's translation unit only)

// e4m3 pack for the TMA kernel's fp8 mode: [filter tile][K block][16-element chunk 0..1][rows][16 x e4m3]
// (UMMA no-swizzle K-major core matrices: 8 rows x 16 B contiguous), round to nearest even, saturating.
__global__ void __launch_bounds__(256) k_pack_filters_e4m3(Geom g, const float* __restrict__ w,
                                                           uint8_t* __restrict__ out, int rows, int kblocks,
                                                           FastDiv fCB, int kmode, long long total) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int e = (int)(i & 15);
        long long t = i >> 4;
        const int r = (int)(t % rows);
        t /= rows;
        const int c = (int)(t & 1);
        t >>= 1;
        const int kb = (int)(t % kblocks);
        const int tile = (int)(t / kblocks);
        const float v = packed_k_value(g, w, tile * rows + r, kb, 16 * c + e, fCB, kmode);
        uint16_t two;
        asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(two) : "f"(0.0f), "f"(v));
        out[i] = (uint8_t)(two & 0xFF);
    }
}
#endif
#ifndef B2C_INST_TU  // (non-template kernel: defined in b2conv.cu's translation unit only)

__global__ void __launch_bounds__(256) k_pack_filters(Geom g, const float* __restrict__ w, float* __restrict__ out,
                                                      int rows, int kblocks, FastDiv fCB, int kmode,
                                                      long long total, int swz, int parts) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int e = (int)(i & 3);
        long long t = i >> 2;
        const int r = (int)(t % rows);
        t /= rows;
        const int c = (int)(t & 7);
        t >>= 3;
        const int part = parts == 2 ? (int)(t & 1) : 0;  // parts == 1: raw only
        if (parts == 2) t >>= 1;
        const int kb = (int)(t % kblocks);
        const int tile = (int)(t / kblocks);
        const int oc = tile * rows + r;
        const int kk = 4 * c + e;
        float v = 0.0f;
        if (oc < g.OC) {
            if (kmode == 3) {
                uint32_t tap, cb, ky, kx;
                fCB.divmod((uint32_t)kb, tap, cb);
                g.fR.divmod(tap, ky, kx);
                const int ic = (int)cb * UMMA_BK + kk;
                if (ic < g.C) v = w[(long long)oc * g.K + ((long long)ic * g.R + ky) * g.R + kx];
            } else if (kmode == 5) {  // first layers, x-window: K block = (ky, 32-float window chunk)
                uint32_t ky, kc;
                fCB.divmod((uint32_t)kb, ky, kc);
                const int wi = (int)kc * 32 + kk;  // window float = kx * 4 + channel
                const int kx = wi >> 2, ch = wi & 3;
                if (kx < g.R && ch < g.C) v = w[(long long)oc * g.K + ((long long)ch * g.R + ky) * g.R + kx];
            } else if (kmode == 4) {  // first layers: chunk c = tap kb*8 + c, element e = channel
                const int tap = kb * 8 + c;
                if (tap < g.RR && e < g.C) v = w[(long long)oc * g.K + (long long)e * g.RR + tap];
            } else {
                const int k = kb * UMMA_BK + kk;
                if (k < g.K) v = w[(long long)oc * g.K + k];
            }
        }
        if (part) {
            float h, l;
            split_tf32(v, h, l);
            v = l;
        }
        if (swz) {
            const long long part_base = i - (i % (8LL * rows * 4));
            out[part_base + ((long long)r * 8 + (c ^ (r & 7))) * 4 + e] = v;
        } else {
            out[i] = v;
        }
    }
}
#endif

// --------------------------------------------------------------------------- main kernel

template <int BN, bool SWAP, int KMODE>
__global__ void __launch_bounds__(UMMA_THREADS, 1) k_umma(UmmaArgs a) {
    using Cfg = UmmaCfg<BN, SWAP>;
    constexpr int STAGES = Cfg::STAGES;
    constexpr int HALF = Cfg::HALF;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty_bar = full_bar + STAGES;
    uint64_t* tfull_bar = empty_bar + STAGES;  // [2] chunk in TMEM slot ready
    uint64_t* tempty_bar = tfull_bar + 2;      // [2] TMEM slot drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
    int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);
    uint8_t* tiles = smem + UMMA_SMEM_HDR;

    const Geom& g = a.g;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;

    // Tile coordinates: pixel tile along x, out_chan (filter) tile along y, K split along z.
    const int m0 = blockIdx.x * Cfg::PIX_ROWS;
    const int n0 = blockIdx.y * Cfg::FLT_ROWS;
    const int z = blockIdx.z;
    const int kb_begin = z * a.kps;
    const int kb_end = min(a.kblocks, kb_begin + a.kps);
    const int nkb = kb_end - kb_begin;
    const int G = a.drain;
    const int nchunks = (nkb + G - 1) / G;

    // Operand regions inside a stage: A then B; each [raw rows*128 B][lo rows*128 B].
    constexpr uint32_t PIX_OFF = SWAP ? Cfg::A_BYTES : 0u;
    constexpr uint32_t FLT_OFF = SWAP ? 0u : Cfg::A_BYTES;

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&full_bar[s]), UMMA_GROUP + 1);  // one group + the bulk loader
            mbar_init(smem_u32(&empty_bar[s]), 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(smem_u32(&tfull_bar[s]), 1);
            mbar_init(smem_u32(&tempty_bar[s]), UMMA_PRODUCERS);
        }
        mbar_fence_init();
    }
    if (warp == UMMA_MMA_WARP) tmem_alloc(smem_u32(tmem_slot), Cfg::TMEM_COLS);
    if (warp == UMMA_LOAD_WARP && lane == 0 && a.prefetch) {
        // Whole-grid cooperative L2 prefetch of the operands of small ops: the
        // dependent per-K-block loads then hit L2 instead of DRAM.
        const int ncta = gridDim.x * gridDim.y * gridDim.z;
        const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
        prefetch_share_l2(a.x, (long long)g.N * g.C * g.HW, cta, ncta);
        prefetch_share_l2(a.wpk, a.wpk_elems, cta, ncta);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t tiles_u32 = smem_u32(tiles);

    if (warp < UMMA_MMA_WARP) {
        // ------------------------------------------------------------ pixel producers (+ drain, epilogue)
        const int group = warp >> 2;                 // warps 0-3: group 0, warps 4-7: group 1
        const int gtid = tid & (UMMA_GROUP - 1);
        const int quarter = warp & 3, half = warp >> 2;
        const int c_begin = half * HALF;
        const uint32_t t_row = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c_begin;
        float acc[HALF];
#pragma unroll
        for (int j = 0; j < HALF; ++j) acc[j] = 0.0f;

        PixRow rs[Cfg::NROWS];
#pragma unroll
        for (int q = 0; q < Cfg::NROWS; ++q) {
            const int i = gtid + q * UMMA_GROUP;
            PixRow st;
            st.iy0 = 0;
            st.ix0 = 0;
            st.valid = false;
            st.base = a.x;
            const int m = m0 + i;
            if (i < Cfg::PIX_ROWS && m < g.M) {
                uint32_t b, p, oy, ox;
                g.fPQ.divmod((uint32_t)m, b, p);
                g.fOW.divmod(p, oy, ox);
                st.iy0 = (int)oy * g.S - g.P;
                st.ix0 = (int)ox * g.S - g.P;
                st.valid = true;
                if (KMODE == 2)
                    st.base = a.x + (long long)b * g.K;
                else if (KMODE == 3)
                    st.base = a.x + (long long)b * g.C * g.HW;
                else
                    st.base = a.x + (long long)b * g.C * g.HW + (long long)st.iy0 * g.W + st.ix0;
            }
            rs[q] = st;
        }

        // Drain TMEM chunk c (slot c&1) into the fp32 register sums.
        auto drain_chunk = [&](int c) {
            const int slot = c & 1;
            mbar_wait(smem_u32(&tfull_bar[slot]), (uint32_t)(c >> 1) & 1u);
            tc_fence_after();
            tmem_add_cols<HALF>(t_row + (uint32_t)(slot * BN), acc);
            tc_fence_before();
            mbar_arrive(smem_u32(&tempty_bar[slot]));
        };

        int drained = 0;
        for (int it = group; it < nkb; it += UMMA_GROUPS) {
            while (drained < nchunks && it >= (drained + 1) * G + a.lag) drain_chunk(drained++);
            const KBlock kb = kblock_info(g, kb_begin + it, a.fCB, KMODE);
            const int stage = it % STAGES;
            const uint32_t phase = (uint32_t)(it / STAGES) & 1u;
            const uint32_t pbase = tiles_u32 + (uint32_t)(stage * Cfg::STAGE_BYTES) + PIX_OFF;
#pragma unroll
            for (int q = 0; q < Cfg::NROWS; ++q) {
                const int i = gtid + q * UMMA_GROUP;
                const bool has_row = i < Cfg::PIX_ROWS;
                float v[32];
                if (has_row) load_pixel_row<KMODE>(g, rs[q], kb, v);
                if (q == 0) mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1u);
                if (has_row)
                    store_row_split(pbase + (uint32_t)i * 16u, pbase + (uint32_t)(Cfg::PIX_ROWS * 128 + i * 16),
                                    (uint32_t)(Cfg::PIX_ROWS * 16), v);
            }
            fence_proxy_async_smem();
            mbar_arrive(smem_u32(&full_bar[stage]));
        }
        while (drained < nchunks) drain_chunk(drained++);

        // ------------------------------------------------------------ epilogue
        const int row = quarter * 32 + lane;  // TMEM lane = MMA M row
        long long row_out = 0;                // !SWAP: b*OC*PQ + p ; SWAP: oc
        bool row_ok;
        float row_bias = 0.f;
        if (!SWAP) {
            const int m = m0 + row;
            row_ok = m < g.M;
            if (row_ok) {
                uint32_t b, p;
                g.fPQ.divmod((uint32_t)m, b, p);
                row_out = (long long)b * g.OC * g.PQ + p;
            }
        } else {
            const int oc = n0 + row;
            row_ok = oc < g.OC;
            row_out = oc;
            if (row_ok) row_bias = __ldg(a.bias + oc);
        }

        // emit with a pre-loaded bias (!SWAP: per column; SWAP: row_bias)
        auto emit_b = [&](int col, float v, float bcol) {
            if (!SWAP) {
                const int oc = n0 + col;
                if (row_ok && oc < g.OC) a.y[row_out + (long long)oc * g.PQ] = apply_act(v + bcol, g.act);
            } else {
                const int m = m0 + col;
                if (row_ok && m < g.M) {
                    uint32_t b, p;
                    g.fPQ.divmod((uint32_t)m, b, p);
                    a.y[((long long)b * g.OC + row_out) * g.PQ + p] = apply_act(v + row_bias, g.act);
                }
            }
        };
        auto emit = [&](int col, float v) {
            if (!SWAP) {
                const int oc = n0 + col;
                if (row_ok && oc < g.OC)
                    a.y[row_out + (long long)oc * g.PQ] = apply_act(v + __ldg(a.bias + oc), g.act);
            } else {
                const int m = m0 + col;
                if (row_ok && m < g.M) {
                    uint32_t b, p;
                    g.fPQ.divmod((uint32_t)m, b, p);
                    a.y[((long long)b * g.OC + row_out) * g.PQ + p] = apply_act(v + row_bias, g.act);
                }
            }
        };

        if (a.split == 1) {
            // groups of 8: the 8 bias loads issue before the 8 stores (y may
            // alias bias as far as the compiler knows)
#pragma unroll
            for (int j0 = 0; j0 < HALF; j0 += 8) {
                float bv[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int oc = n0 + c_begin + j0 + j;
                    bv[j] = SWAP ? 0.0f : (oc < g.OC ? __ldg(a.bias + oc) : 0.0f);
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) emit_b(c_begin + j0 + j, acc[j0 + j], bv[j]);
            }
        } else {
            const int tile = blockIdx.y * gridDim.x + blockIdx.x;
            float* part = a.ws + ((size_t)tile * a.split + z) * BN * UMMA_M;
#pragma unroll
            for (int j = 0; j < HALF; ++j) __stcg(part + (size_t)(c_begin + j) * UMMA_M + row, acc[j]);
            __threadfence();
            named_bar_sync(1, UMMA_PRODUCERS);
            if (tid == 0) {
                const int ticket = atomicAdd(a.sems + tile, 1);
                *last_flag = (ticket == a.split - 1);
            }
            named_bar_sync(1, UMMA_PRODUCERS);
            if (*last_flag) {
                __threadfence();
                const float* base = a.ws + (size_t)tile * a.split * BN * UMMA_M;
#pragma unroll 1
                for (int c = c_begin; c < c_begin + HALF; ++c) {
                    float sum = 0.f;
                    for (int zz = 0; zz < a.split; ++zz) sum += __ldcg(base + ((size_t)zz * BN + c) * UMMA_M + row);
                    emit(c, sum);
                }
                if (tid == 0) a.sems[tile] = 0;
            }
        }
    } else if (warp == UMMA_MMA_WARP) {
        if (lane == 0) {
            // ------------------------------------------------------------ MMA issuer
            constexpr uint32_t idesc = umma_idesc(2, UMMA_M, BN);
            constexpr uint32_t A_LBO = UMMA_M * 16, B_LBO = BN * 16;
            for (int it = 0; it < nkb; ++it) {
                const int c = it / G;
                const int slot = c & 1;
                const bool first = (it % G) == 0;
                const bool last = ((it % G) == G - 1) || (it == nkb - 1);
                if (first && c >= 2) {
                    mbar_wait(smem_u32(&tempty_bar[slot]), (uint32_t)((c >> 1) - 1) & 1u);
                    tc_fence_after();
                }
                const int stage = it % STAGES;
                const uint32_t phase = (uint32_t)(it / STAGES) & 1u;
                mbar_wait(smem_u32(&full_bar[stage]), phase);
                tc_fence_after();
                const uint32_t a_raw = tiles_u32 + (uint32_t)(stage * Cfg::STAGE_BYTES);
                const uint32_t a_lo = a_raw + UMMA_M * 128;
                const uint32_t b_raw = a_raw + Cfg::A_BYTES;
                const uint32_t b_lo = b_raw + BN * 128;
                const uint32_t d = tmem_base + (uint32_t)(slot * BN);
#pragma unroll
                for (int s = 0; s < UMMA_BK / 8; ++s) {
                    const uint64_t dah = umma_desc(a_raw + s * 2 * A_LBO, A_LBO, 128);
                    const uint64_t dal = umma_desc(a_lo + s * 2 * A_LBO, A_LBO, 128);
                    const uint64_t dbh = umma_desc(b_raw + s * 2 * B_LBO, B_LBO, 128);
                    const uint64_t dbl = umma_desc(b_lo + s * 2 * B_LBO, B_LBO, 128);
                    mma_tf32(d, dah, dbh, idesc, (first && s == 0) ? 0u : 1u);
                    mma_tf32(d, dah, dbl, idesc, 1u);
                    mma_tf32(d, dal, dbh, idesc, 1u);
                }
                tc_commit(smem_u32(&empty_bar[stage]));
                if (last) tc_commit(smem_u32(&tfull_bar[slot]));
            }
        }
        __syncwarp();
    } else {
        if (lane == 0) {
            // ------------------------------------------------------------ packed-filter bulk loader
            const char* src = reinterpret_cast<const char*>(a.wpk) +
                              ((size_t)blockIdx.y * a.kblocks + kb_begin) * Cfg::FLT_STAGE_BYTES;
            for (int it = 0; it < nkb; ++it) {
                const int stage = it % STAGES;
                const uint32_t phase = (uint32_t)(it / STAGES) & 1u;
                mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1u);
                const uint32_t bar = smem_u32(&full_bar[stage]);
                mbar_arrive_expect_tx(bar, Cfg::FLT_STAGE_BYTES);
                bulk_g2s(tiles_u32 + (uint32_t)(stage * Cfg::STAGE_BYTES) + FLT_OFF,
                         src + (size_t)it * Cfg::FLT_STAGE_BYTES, Cfg::FLT_STAGE_BYTES, bar);
            }
        }
        __syncwarp();
    }
    __syncthreads();
    if (warp == UMMA_MMA_WARP) {
        tc_fence_after();
        tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
    }
}

}  // namespace b2c
