// TMA-fed, persistent tcgen05 / TMEM implicit-GEMM convolution, fp32-exact
// via 3xTF32.
//
// GEMM view of the reference ConvTiled (cuclgen/variants.py:376-414):
// M = img*oy*ox output pixels, N = out_chan, K = in_chan*ksz*ksz, with the
// bias/ReLU epilogue of variants.py:160-165 fused (graphopt.fuse_activations,
// graphopt.py:59-86).  No thread gathers an operand element from global
// memory; the TMA unit does, straight into the layout the tensor core reads:
//
//   * MODE 0 (conv): the activations are re-laid out once per call to NHWC
//     (k_nchw_to_nhwc: the B200 form of the reference's required_formats
//     conversion, variants.py:416-424 / runner.py:96-105, charged to the op)
//     and one TMA *im2col* load per K block brings 128 (or BN) output pixels x
//     32 channels of one filter tap into the K-major SWIZZLE_128B layout; the
//     TMA unit zero-fills the conv padding.  Filters are packed once (cached,
//     b2c_conv_prepare) into the same swizzled layout, raw and lo halves, and
//     streamed with one cp.async.bulk per K block.
//   * MODE 2 (1x1, stride 1, no pad; conv_1x1, variants.py:279-325): the NHWC
//     copy is a plain [pixels][C] matrix; a 2-D tiled box replaces the im2col.
//   * MODE 3 (first layers, C <= 4: AlexNet/NiN conv1, GoogLeNet conv1): NHWC
//     with C padded to 4; a K block is 8 filter taps x 4 channels, loaded as 8
//     im2col boxes of 16-byte pixels into the no-swizzle core-matrix layout
//     [tap][row][16 B] (strides 4 and 2 are the TMA element strides).
//   * MODE 4 (first layers, C <= 4, default): x is copied to a zero-padded
//     NHWC buffer with 4 channels; for one filter row ky, the 8 x-taps x 4
//     channels an output pixel needs are 32 consecutive floats there (128 B).
//     A 5-D tiled tensor map with overlapping strides (window, ox step S*16 B,
//     oy step S rows, ky step 1 row, image) loads a BX x BY block of output
//     pixels x 32 window floats per box into the SWIZZLE_128B layout: 128-byte
//     rows instead of MODE 3's 16-byte ones (the TMA unit issues ~0.75 rows
//     per clock per SM, so row width sets its throughput).
//   * MODE 8 (bf16 mode, tm=5): x re-laid out to a bf16 NHWC copy; one im2col TMA
//     per K block brings 128 output pixels x 64 bf16 channels of one filter tap
//     (128-byte rows, SWIZZLE_128B) and the filters are packed once as bf16 in the
//     same layout, so both MMA operands come straight from shared memory (SS
//     kind::f16 MMAs, four K = 16 steps per block): no split pass at all.
//   * MODE 7 (Winograd F(2x2,3x3), conv_wino): 16 independent GEMMs
//     M[z] = V[z] * U[z]^T over the transformed tiles (k_wino.cuh): MODE 1 with a
//     third TMA coordinate z, no bias / activation (the output transform adds them).
//   * MODE 1 (fc, variants.py:328-373): the whole-image filter makes both
//     operands plain row-major [rows][K] matrices (x as [img][ic*h*w], w as
//     [oc][ic*h*w]), loaded raw by 2-D tiled TMA: the fc6 weights (151 MB)
//     are read from HBM once, with no pack.
//
// Precision (see k_umma.cuh): kind::tf32 truncates an fp32 operand to TF32,
// so raw x is the "hi" operand and lo = x - trunc_tf32(x);
// D += Ahi*Bhi + Ahi*Blo + Alo*Bhi (single-CTA tiles with BN <= 96: Ahi*[Bhi | Blo] as one
// N = 2*BN MMA plus Alo*Bhi into the lo half, summed by the drain).  K is accumulated in TMEM chunks of
// `drain` K blocks into two ping-ponged slots and each finished chunk is
// drained into fp32 round-to-nearest register sums, bounding the tensor
// core's truncating accumulation error for any K.
//
// Persistent: grid = min(work units, SMs); a unit is (pixel tile, filter
// tile, K split).  The smem ring, the TMEM slots and all barrier phases run
// on across units, so the epilogue of one unit overlaps the main loop of the
// next and the pipeline never drains between tiles.
//
// Warp roles:
//   warps 0-3        split: for every stage, lo = x - trunc(x) beside each raw
//                    operand the TMA loaded (elementwise on the tile image).
//   warps 4..4+4DG-1 drain + epilogue (DG = 1, or 2 column halves):
//                    tcgen05.ld finished chunks, fp32 sums, + bias, ReLU,
//                    NCHW stores (or split-K partials + deterministic reduce
//                    behind one acq_rel ticket).
//   next warp        TMEM allocation; one lane issues the tcgen05.mma (12 per
//                    32-wide K block, 8 with the fused issue).
//   last warp(s)     one lane each issues the pixel TMA / the filter loads.
// Launched with programmatic dependent launch: the prologue (barrier init,
// TMEM alloc, tensor-map prefetch, the loaders' first-unit decode) overlaps the
// previous kernel; griddepcontrol.wait precedes every global access.  The role
// dispatch lists the loaders first so that their code follows the prologue.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "k_umma.cuh"  // tmem_add_cols, k_pack_filters

namespace b2c {

constexpr int TM_M = 128;
constexpr int TM_BK = 32;              // fp32 K elements per stage
constexpr int TM_SPLIT_THREADS = 128;  // warps 0-3
constexpr int TM_HDR = 2048;           // barriers, TMEM slot, flags (< 1 KB); unit bias at +1 KB (<= 256 floats)
constexpr int TM_MAX_SMEM = 232448;    // 227 KB opt-in per CTA
constexpr int TM_TAPS = 8;             // MODE 3: filter taps per K block
#ifndef B2C_FUSED_ON
#define B2C_FUSED_ON 1
#endif

// PREC 0: fp32-exact 3xTF32 (kind::tf32, A = raw | lo in TMEM, B = packed raw | lo).
// PREC 2: e4m3 operands, fp32 accumulate (kind::f8f6f4): as PREC 1 with one K = 32 MMA per
//         K block; filters packed as e4m3 in the no-swizzle layout [16-element chunk][rows][16 B].
// PREC 1: bf16 operands, fp32 accumulate (kind::f16): the split warps round the fp32
//         pixel tile to bf16 into TMEM; filters are packed once as bf16 in the
//         no-swizzle core-matrix layout [8-element chunk][rows][16 B].
// CL: 1 single CTAs; 2 CTA pairs (clusters of 2) multicasting each filter stage to both,
// each CTA issuing its own M = 128 MMAs; 3 2-SM UMMA pairs (tcgen05 cta_group::2): the
// leader issues M = 256 MMAs over both CTAs' pixel tiles, each CTA holding half of the
// filter tile (B rows) and its own 128 accumulator rows.
template <int BN, bool SWAP, int MODE, int OCC = 1, int CL = 1, int PREC = 0>
struct TmaCfg {
    static_assert(PREC == 0 || (!SWAP && MODE != 1 && MODE != 3 && MODE != 7 && (CL == 1 || MODE == 8)), "bf16 / fp8: pixels on M, packed filters");
    static constexpr bool RAW_B = MODE == 1 || MODE == 7;  // both operands raw [rows][K] matrices by TMA (no pack)
    static constexpr bool SS = MODE == 8;  // bf16 NHWC copy: A and B straight from shared memory, no split pass
    static_assert(!SS || (PREC == 1 && !SWAP && (CL == 1 || CL == 3) && OCC == 1), "MODE 8: bf16, pixels on M, single CTAs or 2-SM pairs");
    static_assert((MODE != 5 && MODE != 6) || CL != 2, "MODE 5/6: no multicast pairs");
    static_assert(CL == 1 || CL == 4 || ((CL == 2 || CL == 3) && !SWAP && !RAW_B && OCC == 1), "pairs share B = packed filters");
    static_assert(CL != 4 || OCC == 1, "cluster split-K: one CTA per SM (the staging tile)");
    static constexpr bool PAIR = CL == 3;  // 2-SM UMMA
    static constexpr bool TWO_TILES = CL == 2 || CL == 3;  // a unit is two neighbouring pixel tiles
    static constexpr bool CSPLIT = CL == 4;  // the split-K CTAs of a tile form one cluster; fixup over DSMEM
    static constexpr int STG_BYTES = CSPLIT ? TM_M * BN * 4 : 0;  // this CTA's partial, [col][row] fp32
    static_assert(!PAIR || (BN >= 64 && BN <= 192), "2-SM UMMA: N = BN in [64, 192] (two accumulators + A slots in TMEM)");
    static_assert((BN % 32 == 0 && BN >= 32 && BN <= 256) || (BN == 16 && SWAP && MODE == 1),
                  "BN: multiple of 32 in [32, 256] (16: the swapped fc tile for small batches)");
    static_assert(OCC == 1 || (OCC == 2 && BN <= 64), "two CTAs per SM: BN <= 64 (256 TMEM columns each)");
    // drain warp groups (column halves); two groups halve the exposed epilogue
    static constexpr int DG = (OCC == 1 && (BN >= 64 || SWAP)) ? 2 : 1;
    static constexpr int DRAIN_COLS = BN / DG;
    static constexpr int DRAIN_THREADS = 128 * DG;
    static constexpr int MMA_WARP = 4 + 4 * DG;
    static constexpr int LOAD_WARP = MMA_WARP + 1;  // pixel / activation tiles (one TMA per stage: ~200 issue cycles)
    // filter stages from their own warp, issued in parallel with the pixel loads; with two CTAs
    // per SM the extra warp would cost registers the drain warps need, so one warp issues both
    static constexpr bool TWO_LOADERS = OCC == 1;
    static constexpr int FLT_WARP = TWO_LOADERS ? LOAD_WARP + 1 : LOAD_WARP;
    static constexpr int THREADS = 32 * (FLT_WARP + 1);
    static constexpr int PIX_ROWS = SWAP ? BN : TM_M;
    static constexpr int FLT_ROWS = SWAP ? TM_M : BN;
    // The MMA's A operand (M = 128 rows) lives in TMEM: the split warps move
    // it there as raw + lo from the smem image the TMA (or bulk copy) wrote.
    // lo is computed on the way (filters, when they are A, are packed raw-only).
    static constexpr bool A_PRESPLIT = false;
    static constexpr bool B_SPLIT = SWAP || RAW_B;  // B raw from TMA: lo computed into smem
    static constexpr int A_SMEM = (A_PRESPLIT ? 2 : 1) * TM_M * 128;
    static constexpr int B_BYTES = SS ? (PAIR ? BN / 2 : BN) * 128 : PREC == 1 ? BN * 64 : PREC == 2 ? BN * 32
                                                             : (PAIR ? 1 : 2) * BN * 128;  // bf16 SW128 64-K | bf16 | e4m3 | raw + lo (a pair: half the rows each)
    static constexpr int STAGE_BYTES = A_SMEM + B_BYTES;
    static constexpr int PIX_OFF = SWAP ? A_SMEM : 0;
    static constexpr int FLT_OFF = SWAP ? 0 : A_SMEM;
    static constexpr int FLT_STAGE = SS ? FLT_ROWS * 128 : PREC == 1 ? FLT_ROWS * 64 : PREC == 2 ? FLT_ROWS * 32
                                                                 : (SWAP ? 1 : 2) * FLT_ROWS * 128;  // packed filters per K block
    static constexpr int FLT_HALF = FLT_ROWS / 2 * 128;   // 2-SM pair: one CTA's rows of one (raw | lo) image
    static constexpr int FLT_CTA = PAIR ? (SS ? FLT_HALF : 2 * FLT_HALF) : FLT_STAGE;  // filter bytes landing in one CTA per K block
    static constexpr bool SW128 = MODE != 3;
    // Fused 3xTF32 issue (PREC 0, B raw | lo contiguous in one SWIZZLE_128B image): the raw and
    // lo B tiles form one N = 2*BN operand, so Ahi*[Braw | Blo] is ONE MMA and Alo*Braw a second
    // one accumulating into the Blo half: 2 tcgen05.mma per K = 8 step instead of 3 (fewer
    // issue slots for the single MMA-issuing thread).  An accumulator slot is then 2*BN columns
    // [Ahi*Braw | Ahi*Blo + Alo*Braw], summed by the drain; kept where >= 2 A slots still fit.
    static constexpr int TMEM_COLS0 = OCC == 2 ? 256 : 512;
    static constexpr bool FUSED = B2C_FUSED_ON && PREC == 0 && !SS && !PAIR && SW128 && OCC == 1 && 2 * BN <= 256 &&
                                  4 * BN + 128 <= TMEM_COLS0;
    static constexpr int SLOT_COLS = FUSED ? 2 * BN : BN;  // TMEM columns per accumulation slot
    static constexpr int ACC_COLS = 2 * SLOT_COLS;        // two TMEM accumulation slots
    // OCC CTAs per SM share its 228 KB of shared memory (1 KB per CTA is the driver's) and 512 TMEM columns
    static constexpr int BUDGET = (OCC == 1 ? TM_MAX_SMEM : 233472 / OCC - 1024) - TM_HDR - 1024 - STG_BYTES;
    static constexpr int SM_STAGES = BUDGET / STAGE_BYTES;
    static constexpr int STAGES = SM_STAGES < 8 ? SM_STAGES : 8;
    static constexpr int SMEM = TM_HDR + 1024 + STAGES * STAGE_BYTES + STG_BYTES;
    static constexpr int TMEM_COLS = TMEM_COLS0;
    // TMEM A stages (raw | lo: 64 columns each): as many as the columns left beside the two
    // accumulators allow (<= 4), so a split is not held up waiting for the MMAs of the stage
    // two back to release its slot (the 2-slot loop was paced split -> MMA issue -> MMA done).
    static constexpr int A_SLOTS_FIT = (TMEM_COLS - ACC_COLS) / 64;
    static constexpr int A_SLOTS = A_SLOTS_FIT < 4 ? A_SLOTS_FIT : 4;
    static_assert(ACC_COLS + A_SLOTS * 64 <= TMEM_COLS, "TMEM budget");
    static constexpr uint32_t BYTES = PIX_ROWS * 128 + (RAW_B ? FLT_ROWS * 128 : FLT_CTA);
    static constexpr uint32_t FLT_BYTES = RAW_B ? FLT_ROWS * 128 : FLT_CTA;  // the filter warp's bytes per stage
    // barrier arrival counts (a pair's leader counts its peer's split / drain warps too)
    // (SS pairs: one forwarding lane per CTA reports its stage's TMA bytes to the leader)
    static constexpr int SPLIT_ARRIVALS = PAIR ? (SS ? 2 : 2 * (TM_SPLIT_THREADS / 32)) : TM_SPLIT_THREADS;
    static constexpr int DRAIN_ARRIVALS = PAIR ? 2 * (DRAIN_THREADS / 32) : DRAIN_THREADS;
    static_assert(MODE != 4 || !SWAP, "MODE 4 tiles are pixel blocks on M");
    static_assert((MODE != 5 && MODE != 6) || !SWAP, "MODE 5/6 tiles are pixel blocks on M (split warps transpose them)");
    static_assert(STAGES >= 2, "need at least two stages");
    static_assert(DRAIN_COLS % 8 == 0, "TMEM drain granularity");
};

struct TArgs {
    Geom g;
    const float* wpk;   // packed filters [flt tile][K block][raw | lo][rows][128 B]
    const float* bias;
    float* y;
    float* ws;          // split-K partials [tile][split][BN][128]
    int* sems;          // split-K tickets [tile], zero at rest
    int split, kps, kblocks;
    int streamk;        // 1: every CTA takes an equal contiguous range of the units' K blocks (split == 1)
    int sk_maxc;        // stream-K: partial slots per unit (max CTAs sharing one unit)
    int tiles_n;        // filter tiles
    int tiles_m;        // pixel tiles
    int units;          // pixel tiles * filter tiles * split
    int bx, by;         // MODE 4: output-pixel block of a tile (bx * by <= 128 rows)
    int tiles_x, tiles_y;  // MODE 4: blocks per image row / column
    FastDiv fCB;        // MODE 0: channel blocks of 32 per filter tap
    int drain;
    int trace;          // debug: phase clocks of CTA 0 into g_b2c_trace
    long long* trace_buf;  // debug: where (b2conv.cu's g_b2c_trace)
    // In-kernel re-layout of x (instead of a separate conversion launch):
    // 0 none (x already converted / fc), 1 NCHW -> NHWC (C channels),
    // 2 NCHW -> zero-padded NHWC4 [N][hp][wp][4] (first layers).
    int relayout;
    const float* x;
    float* xh;
    int hp, wp, pad;
    unsigned long long* gbar;  // grid barrier counter (monotonic; zero at allocation)
    int flt_early;      // packed filters are complete: the loader may fetch them before griddepcontrol.wait
    // K blocks whose index % kb_period == kb_period - 1 hold only ksteps_last valid
    // groups of 8 K (channel / window / K tail); the MMAs skip the all-zero rest.
    int kb_period, ksteps_last;
    int box_w;  // MODE 6: box width in floats (multiple of 4, >= bx + 3); the box is [32 ch][by][box_w]
    // unit decomposition by multiply-shift (every role walks the units; no runtime integer divides
    // on the loader's path to its first TMA)
    FastDiv fSplit, fTilesN, fTilesMN, fPerImg, fTilesX;
};

// Walks a CTA's work: units blockIdx, +stride, ... ; or, in stream-K mode, the
// contiguous K-block range [c*W/G, (c+1)*W/G) of the W = units*kblocks K
// blocks, cut into per-unit segments.  A unit whose K blocks span several CTAs
// is finished through the split-K partials (contributors in CTA order).
struct UnitCursor {
    long long k, end;
    int u;
};

__device__ __forceinline__ long long sk_start(long long W, int G, int c) { return (long long)c * W / G; }

// Stream-K shares go to CTAs, or to CTA pairs (CL >= 2: both CTAs of a pair walk the same pair-units).
template <int CL>
__device__ __forceinline__ int sk_ctas() { return (int)gridDim.x / ((CL == 2 || CL == 3) ? 2 : 1); }
template <int CL>
__device__ __forceinline__ int sk_me() { return (int)blockIdx.x / ((CL == 2 || CL == 3) ? 2 : 1); }

template <int PIX_ROWS, int FLT_ROWS, int MODE, int CL>
__device__ __forceinline__ UnitCursor cursor_begin(const TArgs& a, int ubase) {
    UnitCursor c;
    c.u = ubase;
    c.k = c.end = 0;
    if (a.streamk) {
        const long long W = (long long)a.units * a.kblocks;
        c.k = sk_start(W, sk_ctas<CL>(), sk_me<CL>());
        c.end = sk_start(W, sk_ctas<CL>(), sk_me<CL>() + 1);
    }
    return c;
}

struct Unit {
    int t, m0, n0, z, kb_begin, nkb;
    int nsplit, pslot0;  // contributors to this tile's output (1 = direct store); first partial slot
    int b, oy0, ox0;  // MODE 4 tile origin
    bool ghost;       // 2-CTA pair whose second pixel tile is past the end: runs the pipeline, stores nothing
};

// Unit u of a CTA (CL = 1), or pair-unit u of a 2-CTA cluster (CL = 2: the two
// CTAs take pixel tiles 2p and 2p+1 with the same filter tile and K range).
template <int PIX_ROWS, int FLT_ROWS, int MODE, int CL = 1>
__device__ __forceinline__ Unit unit_of(const TArgs& a, int u, int rank = 0) {
    Unit w;
    uint32_t t2, zs;
    a.fSplit.divmod((uint32_t)u, t2, zs);
    w.z = (int)zs;
    // MODE 7: tile t2 of the batched GEMM = (z, pixel tile, filter tile), z outermost
    uint32_t zb = 0, t3 = t2;
    if (MODE == 7) a.fTilesMN.divmod(t2, zb, t3);
    uint32_t mq, ntu;
    a.fTilesN.divmod(t3, mq, ntu);
    const int nt = (int)ntu;
    const int mt = (CL == 2 || CL == 3) ? 2 * (int)mq + rank : (int)mq;
    w.ghost = mt >= a.tiles_m;
    w.t = MODE == 7 ? (int)t2 : mt * a.tiles_n + nt;
    w.m0 = mt * PIX_ROWS;
    w.n0 = nt * FLT_ROWS;
    w.kb_begin = w.z * a.kps;
    w.nkb = min(a.kblocks, w.kb_begin + a.kps) - w.kb_begin;
    if (MODE == 4 || MODE == 5 || MODE == 6) {  // MODE 5: tiles_y = by = 1, bx = 128 (pixel runs of one image)
        uint32_t b, r, ty, tx;
        a.fPerImg.divmod((uint32_t)mt, b, r);
        a.fTilesX.divmod(r, ty, tx);
        w.b = (int)b;
        w.oy0 = (int)ty * a.by;
        w.ox0 = (int)tx * a.bx;
    } else {
        w.b = (int)zb;  // MODE 7: the GEMM's z (0 otherwise)
        w.oy0 = w.ox0 = 0;
    }
    w.nsplit = a.split;
    w.pslot0 = w.t * a.split;
    return w;
}

template <int PIX_ROWS, int FLT_ROWS, int MODE, int CL>
__device__ __forceinline__ bool next_unit(const TArgs& a, UnitCursor& cur, int ustride, int rank, Unit& w) {
    if (a.streamk) {
        if (cur.k >= cur.end) return false;
        const int u = (int)(cur.k / a.kblocks);
        const int kb0 = (int)(cur.k - (long long)u * a.kblocks);
        const long long left = cur.end - cur.k;
        const int n = (int)(left < (long long)(a.kblocks - kb0) ? left : (long long)(a.kblocks - kb0));
        w = unit_of<PIX_ROWS, FLT_ROWS, MODE, CL>(a, u, rank);
        w.kb_begin = kb0;
        w.nkb = n;
        // CTAs owning this unit's first and last K block
        const long long W = (long long)a.units * a.kblocks;
        const int G = sk_ctas<CL>();
        const long long x0 = (long long)u * a.kblocks, x1 = x0 + a.kblocks - 1;
        int c0 = (int)(x0 * G / W), c1 = (int)(x1 * G / W);
        while (c0 + 1 < G && sk_start(W, G, c0 + 1) <= x0) ++c0;
        while (c0 > 0 && sk_start(W, G, c0) > x0) --c0;
        while (c1 + 1 < G && sk_start(W, G, c1 + 1) <= x1) ++c1;
        while (c1 > 0 && sk_start(W, G, c1) > x1) --c1;
        w.nsplit = c1 - c0 + 1;
        w.z = sk_me<CL>() - c0;
        w.pslot0 = w.t * a.sk_maxc;
        cur.k += n;
        return true;
    }
    if (cur.u >= a.units) return false;
    w = unit_of<PIX_ROWS, FLT_ROWS, MODE, CL>(a, cur.u, rank);
    cur.u += ustride;
    return true;
}

// ----------------------------------------------------------------------------- NCHW -> NHWC
#ifndef B2C_INST_TU  // (non-template kernel: defined in b2conv.cu's translation unit only)

// x [N][C][HW] -> xh [N][HW][Cp] (Cp >= C, channels C..Cp-1 zero); 32x32 tiles
// through shared memory so the read (along pixels) and the write (along
// channels) are both coalesced.
__global__ void __launch_bounds__(256) k_nchw_to_nhwc(const float* __restrict__ x, float* __restrict__ xh, int C,
                                                      int Cp, int HW) {
    __shared__ float tile[32][33];
    pdl_launch_dependents();
    pdl_wait();
    const int n = blockIdx.z;
    const int p0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const float* src = x + (size_t)n * C * HW;
    float* dst = xh + (size_t)n * HW * Cp;
#pragma unroll
    for (int j = ty; j < 32; j += 8) {
        const int c = c0 + j, p = p0 + tx;
        tile[j][tx] = (c < C && p < HW) ? __ldg(src + (size_t)c * HW + p) : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int j = ty; j < 32; j += 8) {
        const int p = p0 + j, c = c0 + tx;
        if (p < HW && c < Cp) dst[(size_t)p * Cp + c] = tile[tx][j];
    }
}
#endif
#ifndef B2C_INST_TU  // (non-template kernel: defined in b2conv.cu's translation unit only)

// bf16 mode, MODE 8: x [N][C][HW] fp32 -> xh [N][HW][C] bf16 (round to nearest even, the
// rounding the split pass of the TS path applies); same 32x32 smem tiles, 2-byte stores.
__global__ void __launch_bounds__(256) k_nchw_to_nhwc_bf16(const float* __restrict__ x, uint16_t* __restrict__ xh,
                                                           int C, int HW) {
    __shared__ float tile[32][33];
    pdl_launch_dependents();
    pdl_wait();
    const int n = blockIdx.z;
    const int p0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const float* src = x + (size_t)n * C * HW;
    uint16_t* dst = xh + (size_t)n * HW * C;
#pragma unroll
    for (int j = ty; j < 32; j += 8) {
        const int c = c0 + j, p = p0 + tx;
        tile[j][tx] = (c < C && p < HW) ? __ldg(src + (size_t)c * HW + p) : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int j = ty; j < 32; j += 8) {
        const int p = p0 + j, c = c0 + tx;
        if (p < HW && c < C) dst[(size_t)p * C + c] = (uint16_t)(pack_bf16x2(tile[tx][j], 0.0f) & 0xFFFFu);
    }
}
#endif

// First layers, space-to-depth (tm=6): x [N][C][H][W] -> xs [N][H'][W'][C*S*S] with
// xs[n][Y][X][(c*S + dy)*S + dx] = x[n][c][S*Y + dy - P][S*X + dx - P] (0 outside): an
// R x R stride-S conv over x is an R' x R' stride-1 conv over xs (R' = ceil(R/S)) with
// C*S*S channels.  One block per (image, output row Y); the stores run along (X, c').
template <int S>
__global__ void __launch_bounds__(256) k_s2d_nhwc(const float* __restrict__ x, float* __restrict__ xs, int C, int H,
                                                  int W, int P, int Hs, int Ws) {
    pdl_launch_dependents();
    pdl_wait();
    const int n = blockIdx.x / Hs, Y = blockIdx.x - n * Hs;
    const int C2 = C * S * S;
    float* dst = xs + ((size_t)n * Hs + Y) * Ws * C2;
    // one thread per (output pixel X, input channel c): S*S consecutive channels of xs, float4 stores
    for (int i = threadIdx.x; i < Ws * C; i += blockDim.x) {
        const int X = i / C, c = i - X * C;
        const float* src = x + ((size_t)n * C + c) * H * W;
        float v[S * S];
#pragma unroll
        for (int dy = 0; dy < S; ++dy) {
            const int iy = S * Y + dy - P;
#pragma unroll
            for (int dx = 0; dx < S; ++dx) {
                const int ix = S * X + dx - P;
                v[dy * S + dx] = ((unsigned)iy < (unsigned)H && (unsigned)ix < (unsigned)W) ? __ldg(src + (size_t)iy * W + ix) : 0.0f;
            }
        }
        float4* o = reinterpret_cast<float4*>(dst + (size_t)X * C2 + c * S * S);
#pragma unroll
        for (int q = 0; q < S * S / 4; ++q) o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
}
#ifndef B2C_INST_TU  // (non-template kernel: defined in b2conv.cu's translation unit only)

// The matching filter transform (once per filter tensor): w [OC][C][R][R] ->
// ws [OC][C*S*S][R'][R'], ws[oc][(c*S + dy)*S + dx][ky'][kx'] = w[oc][c][S*ky' + dy][S*kx' + dx] (0 past R).
__global__ void __launch_bounds__(256) k_s2d_filters(const float* __restrict__ w, float* __restrict__ w2, int OC, int C,
                                                     int R, int S, int R2) {
    const int C2 = C * S * S;
    const long long total = (long long)OC * C2 * R2 * R2;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const int kx2 = (int)(i % R2);
        long long t = i / R2;
        const int ky2 = (int)(t % R2);
        t /= R2;
        const int c2 = (int)(t % C2);
        const int oc = (int)(t / C2);
        const int dx = c2 % S, u = c2 / S, dy = u % S, c = u / S;
        const int ky = S * ky2 + dy, kx = S * kx2 + dx;
        w2[i] = (ky < R && kx < R) ? w[(((long long)oc * C + c) * R + ky) * R + kx] : 0.0f;
    }
}
#endif
#ifndef B2C_INST_TU  // (non-template kernel: defined in b2conv.cu's translation unit only)

// x [N][C][H][W] (C <= 4) -> xp [N][Hp][Wp][4], image at (pad, pad), zeros
// elsewhere: one thread per padded pixel, coalesced plane reads, float4 writes.
__global__ void __launch_bounds__(256) k_to_nhwc4_pad(const float* __restrict__ x, float4* __restrict__ xp, int C,
                                                      int H, int W, int Hp, int Wp, int pad, long long total) {
    // one block per padded row (image b, row yq): no per-element index divisions
    (void)total;
    pdl_launch_dependents();
    pdl_wait();
    const int row = blockIdx.x;
    const int b = row / Hp, yq = row - (row / Hp) * Hp;
    const int iy = yq - pad;
    const bool yin = (unsigned)iy < (unsigned)H;
    const size_t plane = (size_t)H * W;
    const float* src = x + ((size_t)b * C * H + (yin ? iy : 0)) * W;
    float4* dst = xp + (size_t)row * Wp;
    for (int xq = threadIdx.x; xq < Wp; xq += blockDim.x) {
        const int ix = xq - pad;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (yin && (unsigned)ix < (unsigned)W) {
            v.x = __ldg(src + ix);
            if (C > 1) v.y = __ldg(src + plane + ix);
            if (C > 2) v.z = __ldg(src + 2 * plane + ix);
            if (C > 3) v.w = __ldg(src + 3 * plane + ix);
        }
        dst[xq] = v;
    }
}
#endif

// ----------------------------------------------------------------------------- fused re-layout

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Every CTA converts its share of x into the workspace copy the TMA reads,
// then all CTAs meet at a grid barrier (grid <= #SMs with one CTA per SM, so
// all CTAs are co-resident).  Saves a kernel boundary per op.  `scratch` is
// the (still unused) pipeline smem: a 32 x 33 transpose tile per warp.
static __device__ void fused_relayout(const TArgs& a, uint8_t* scratch) {
    const Geom& g = a.g;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    if (a.relayout == 1) {
        float* tile = reinterpret_cast<float*>(scratch) + warp * (32 * 33);
        const int tp = (g.HW + 31) / 32, tc = (g.C + 31) / 32;
        const long long ntiles = (long long)g.N * tp * tc;
        for (long long t = (long long)blockIdx.x * nwarps + warp; t < ntiles; t += (long long)gridDim.x * nwarps) {
            const int ci = (int)(t % tc);
            const long long r = t / tc;
            const int pi = (int)(r % tp), n = (int)(r / tp);
            const int p0 = pi * 32, c0 = ci * 32;
            const float* src = a.x + (size_t)n * g.C * g.HW;
            float* dst = a.xh + (size_t)n * g.HW * g.C;
#pragma unroll 8
            for (int j = 0; j < 32; ++j) {
                const int c = c0 + j, p = p0 + lane;
                tile[j * 33 + lane] = (c < g.C && p < g.HW) ? __ldg(src + (size_t)c * g.HW + p) : 0.0f;
            }
            __syncwarp();
#pragma unroll 8
            for (int j = 0; j < 32; ++j) {
                const int p = p0 + j, c = c0 + lane;
                if (p < g.HW && c < g.C) dst[(size_t)p * g.C + c] = tile[lane * 33 + j];
            }
            __syncwarp();
        }
    } else if (a.relayout == 2) {
        const long long total = (long long)g.N * a.hp * a.wp;
        float4* dst = reinterpret_cast<float4*>(a.xh);
        for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
             i += (long long)gridDim.x * blockDim.x) {
            const int xq = (int)(i % a.wp);
            const long long t = i / a.wp;
            const int yq = (int)(t % a.hp), b = (int)(t / a.hp);
            const int iy = yq - a.pad, ix = xq - a.pad;
            float v[4] = {0.f, 0.f, 0.f, 0.f};
            if ((unsigned)iy < (unsigned)g.H && (unsigned)ix < (unsigned)g.W) {
                const float* src = a.x + ((size_t)b * g.C * g.H + iy) * g.W + ix;
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (c < g.C) v[c] = __ldg(src + (size_t)c * g.HW);
            }
            dst[i] = make_float4(v[0], v[1], v[2], v[3]);
        }
    }
    // publish (generic-proxy writes -> other CTAs' TMA reads) and meet
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long ticket = atomicAdd(a.gbar, 1ull);
        const unsigned long long target = (ticket / gridDim.x + 1ull) * gridDim.x;
        // Needs every CTA of the grid co-resident (grid <= #SMs, 1 CTA/SM) and no
        // concurrent kernel holding SMs: opt-in (B2C_FUSED_NHWC) experiments only.
        // Bounded like mbar_wait: a grid that is not co-resident faults instead of hanging.
        const long long t0 = clock64();
        while (ld_acquire_u64(a.gbar) < target) {
            __nanosleep(64);
            if (clock64() - t0 > (1ll << 32)) __trap();
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    __syncthreads();
}

// One K block of packed filters into a stage: one bulk copy, or, in a 2-CTA
// pair, each CTA fetches half (raw | lo) and multicasts it to both.
template <int BYTES, int CL, bool ONE_IMAGE = false>
__device__ __forceinline__ void load_filters(uint32_t dst, const char* src, uint32_t bar, int rank) {
    if (CL == 3 && ONE_IMAGE) {  // 2-SM pair, one image per K block (bf16 SS): this CTA's half of its rows
        constexpr uint32_t H = BYTES / 2;
        bulk_g2s(dst, src + (size_t)rank * H, H, bar);
    } else if (CL == 3) {  // 2-SM pair: this CTA's half of the rows of the raw image and of the lo image
        constexpr uint32_t H = BYTES / 4;
        bulk_g2s(dst, src + (size_t)rank * H, H, bar);
        bulk_g2s(dst + H, src + BYTES / 2 + (size_t)rank * H, H, bar);
    } else if (CL == 2) {
        constexpr uint32_t H = BYTES / 2;
        bulk_g2s_mc(dst + (uint32_t)rank * H, src + (size_t)rank * H, H, bar, (uint16_t)0x3);
    } else {
        bulk_g2s(dst, src, BYTES, bar);
    }
}

// ----------------------------------------------------------------------------- split + epilogue helpers

// lo = x - trunc_tf32(x) for a raw operand image of `rows` x 128 B, written
// beside it (at + rows*128).  Elementwise on the image, so the swizzle / core
// matrix layout needs no index math.  128 split threads.
template <int ROWS>
__device__ __forceinline__ void split_tile(uint32_t raw, int tid) {
    const uint32_t lo = raw + (uint32_t)ROWS * 128u;
#pragma unroll
    for (int k = 0; k < ROWS * 8 / TM_SPLIT_THREADS; ++k) {
        const uint32_t off = (uint32_t)(tid + k * TM_SPLIT_THREADS) * 16u;
        const float4 v = lds128(raw + off);
        float h, l0, l1, l2, l3;
        split_tf32(v.x, h, l0);
        split_tf32(v.y, h, l1);
        split_tf32(v.z, h, l2);
        split_tf32(v.w, h, l3);
        sts128(lo + off, l0, l1, l2, l3);
    }
}

// Move this thread's A row (M row = tid, 128 threads) into TMEM as 32 raw +
// 32 lo columns: raw from the smem image at `a` (SWIZZLE_128B rows, or the
// no-swizzle [chunk][128 rows][16 B] image of MODE 3); lo either computed
// (x - trunc_tf32(x)) or, for pre-split filter tiles, read from a + 16 KB.
template <bool SW128, bool PRESPLIT>
__device__ __forceinline__ void a_to_tmem(uint32_t a, int tid, uint32_t tcol) {
    float v[32], l[32];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const uint32_t off = SW128 ? (uint32_t)tid * 128u + (uint32_t)((c ^ (tid & 7)) * 16)
                                   : (uint32_t)(c * TM_M * 16 + tid * 16);
        const float4 q = lds128(a + off);
        v[4 * c] = q.x;
        v[4 * c + 1] = q.y;
        v[4 * c + 2] = q.z;
        v[4 * c + 3] = q.w;
        if (PRESPLIT) {
            const float4 r = lds128(a + TM_M * 128 + off);
            l[4 * c] = r.x;
            l[4 * c + 1] = r.y;
            l[4 * c + 2] = r.z;
            l[4 * c + 3] = r.w;
        }
    }
    if (!PRESPLIT) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            float h;
            split_tf32(v[j], h, l[j]);
        }
    }
    tmem_st32(tcol, v);
    tmem_st32(tcol + 32, l);
}

// bf16 mode: the same 32 fp32 of this thread's row, rounded to bf16 and packed in
// pairs (even K in the low half) into 16 TMEM columns.
template <bool SW128>
__device__ __forceinline__ void a_to_tmem_bf16(uint32_t a, int tid, uint32_t tcol) {
    uint32_t r[16];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const uint32_t off = SW128 ? (uint32_t)tid * 128u + (uint32_t)((c ^ (tid & 7)) * 16)
                                   : (uint32_t)(c * TM_M * 16 + tid * 16);
        const float4 q = lds128(a + off);
        r[2 * c] = pack_bf16x2(q.x, q.y);
        r[2 * c + 1] = pack_bf16x2(q.z, q.w);
    }
    tmem_st16u(tcol, r);
}

// fp8 mode: the same 32 fp32 of this thread's row as 32 e4m3 in 8 TMEM columns.
template <bool SW128>
__device__ __forceinline__ void a_to_tmem_e4m3(uint32_t a, int tid, uint32_t tcol) {
    uint32_t r[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const uint32_t off = SW128 ? (uint32_t)tid * 128u + (uint32_t)((c ^ (tid & 7)) * 16)
                                   : (uint32_t)(c * TM_M * 16 + tid * 16);
        const float4 q = lds128(a + off);
        r[c] = pack_e4m3x4(q.x, q.y, q.z, q.w);
    }
    tmem_st8u(tcol, r);
}

// MODE 5 (1x1 convs read straight from NCHW): the TMA box is [32 channels][128
// pixels] (no swizzle), so thread tid's row is a column of it: 32 scalar smem
// loads at a 512-byte stride (consecutive threads hit consecutive banks).  PREC 0
// stores raw | lo (3xTF32), PREC 1 packs bf16 pairs.
template <int PREC>
__device__ __forceinline__ void a_to_tmem_cmajor(uint32_t a, int idx, uint32_t tcol, int cstride) {
    float v[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) v[c] = lds32(a + (uint32_t)(c * cstride + idx) * 4u);
    if constexpr (PREC == 1) {
        uint32_t r[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) r[j] = pack_bf16x2(v[2 * j], v[2 * j + 1]);
        tmem_st16u(tcol, r);
    } else if constexpr (PREC == 2) {
        uint32_t r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = pack_e4m3x4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        tmem_st8u(tcol, r);
    } else {
        float l[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            float h;
            split_tf32(v[j], h, l[j]);
        }
        tmem_st32(tcol, v);
        tmem_st32(tcol + 32, l);
    }
}

// One unit's output: + bias, ReLU (variants.py:160-165), NCHW stores; with
// split-K, the fp32 partial goes to the workspace and the unit that arrives
// last for its tile (atomic ticket) reduces all partials in split order, so
// results are deterministic.  Called by the NT drain threads; `row` is this
// thread's TMEM lane (MMA M row), columns c_begin .. c_begin+DC.
template <int BN, bool SWAP, int DC, int NT, int MODE, bool CSPLIT>
__device__ __forceinline__ void epilogue_unit(const TArgs& a, const Unit& w, float* acc, int c_begin, int row,
                                              int dtid, int* last_flag, float* bias_s, float bpre, uint32_t stg,
                                              uint64_t* cs_bar, int& cs_uses) {
    const Geom& g = a.g;
    if (!SWAP) {  // the unit's out_chan biases -> smem (bpre was loaded by thread dtid before the drains)
        named_bar_sync(1, NT);  // previous unit's readers are done
        if (dtid < BN) bias_s[dtid] = bpre;
        named_bar_sync(1, NT);
    }
    if (CSPLIT && w.nsplit > 1) {
        // Cluster split-K: the tile's split CTAs are one thread-block cluster (rank = split
        // index).  Each non-leader stages its partial in its own shared memory and signals
        // the leader, which sums the partials over DSMEM in split order (deterministic),
        // frees the peers' staging tiles and stores.  No global partials, no tickets.
        const uint32_t rank = cluster_ctarank();
        const int wl = threadIdx.x & 31;
        if (rank != 0) {
            if (cs_uses > 0) mbar_wait(smem_u32(&cs_bar[1]), (uint32_t)(cs_uses - 1) & 1u);
#pragma unroll
            for (int j = 0; j < DC; ++j) sts32(stg + (uint32_t)(((c_begin + j) * TM_M + row) * 4), acc[j]);
            __syncwarp();
            if (wl == 0) mbar_arrive_cluster(smem_u32(&cs_bar[0]), 0);
            ++cs_uses;
            return;
        }
        mbar_wait_cluster(smem_u32(&cs_bar[0]), (uint32_t)cs_uses & 1u);
        for (int r = 1; r < w.nsplit; ++r) {
            const uint32_t base = dsmem_addr(stg, (uint32_t)r);
            float pv[DC];
#pragma unroll
            for (int j = 0; j < DC; ++j) pv[j] = ld_dsmem(base + (uint32_t)(((c_begin + j) * TM_M + row) * 4));
#pragma unroll
            for (int j = 0; j < DC; ++j) acc[j] += pv[j];
        }
        __syncwarp();
        if (wl == 0)
            for (int r = 1; r < w.nsplit; ++r) mbar_arrive_cluster_relaxed(smem_u32(&cs_bar[1]), (uint32_t)r);
        ++cs_uses;
    } else if (w.nsplit > 1) {
        // Split-K / stream-K fixup: every contributor publishes its fp32 partial
        // to L2, fences and takes a ticket; the one that arrives last reduces
        // all partials in split order (deterministic) and resets the ticket.
        // No CTA ever waits on another, so the fixup is correct whether or not
        // the grid is co-resident (concurrent kernels on other streams).
        // (An owner-waits variant saved one L2 round trip but could deadlock
        // against a concurrent kernel holding the SMs its contributors need.)
        float* part = a.ws + ((size_t)w.pslot0 + w.z) * BN * TM_M;
#pragma unroll
        for (int j = 0; j < DC; ++j) __stcg(part + (size_t)(c_begin + j) * TM_M + row, acc[j]);
        // Ordering without a per-thread SC fence: the barrier orders this CTA's partial stores
        // before the ticket, and the ticket is an acq_rel atomic at gpu scope (its release is
        // cumulative over the barrier; its acquire, by the last contributor, makes every other
        // contributor's partials visible to this CTA's cache-global loads after the next barrier).
        named_bar_sync(1, NT);
        if (dtid == 0) {
            const int ticket = atom_add_acq_rel_gpu(a.sems + w.t, 1);
            *last_flag = (ticket == w.nsplit - 1);
        }
        named_bar_sync(1, NT);
        const bool last = *last_flag != 0;
        named_bar_sync(1, NT);  // last_flag is rewritten by the next unit
        if (!last) return;
        if (dtid == 0) a.sems[w.t] = 0;
#pragma unroll
        for (int j = 0; j < DC; ++j) acc[j] = 0.0f;
        const float* base = a.ws + (size_t)w.pslot0 * BN * TM_M;
        // Partials are summed in split order (deterministic); loads for RG
        // consecutive splits are issued together so that RG L2 round trips
        // overlap (RG * DC <= 64 extra registers).
        constexpr int RG = DC >= 64 ? 1 : 64 / DC;
        int zz = 0;
        for (; zz + RG <= w.nsplit; zz += RG) {
            float pv[RG][DC];
#pragma unroll
            for (int g = 0; g < RG; ++g)
#pragma unroll
                for (int j = 0; j < DC; ++j) pv[g][j] = __ldcg(base + ((size_t)(zz + g) * BN + c_begin + j) * TM_M + row);
#pragma unroll
            for (int g = 0; g < RG; ++g)
#pragma unroll
                for (int j = 0; j < DC; ++j) acc[j] += pv[g][j];
        }
        for (; zz < w.nsplit; ++zz) {
#pragma unroll
            for (int j = 0; j < DC; ++j) acc[j] += __ldcg(base + ((size_t)zz * BN + c_begin + j) * TM_M + row);
        }
    }
    float* __restrict__ yp = a.y + (MODE == 7 ? (long long)w.b * g.M * g.OC : 0ll);  // MODE 7: M[z]
    if (!SWAP) {  // row = output pixel, columns = out_chans
        long long row_out;
        if (MODE == 5) {  // run of 128 pixels of image b starting at ox0
            const int p = w.ox0 + row;
            if (p >= g.PQ) return;
            row_out = (long long)w.b * g.OC * g.PQ + p;
        } else if (MODE == 4 || MODE == 6) {  // rectangular tile: row = y * bx + x
            const int y = row / a.bx, x = row - (row / a.bx) * a.bx;
            const int oy = w.oy0 + y, ox = w.ox0 + x;
            if (y >= a.by || oy >= g.OH || ox >= g.OW) return;
            row_out = (long long)w.b * g.OC * g.PQ + (long long)oy * g.OW + ox;
        } else {
            const int m = w.m0 + row;
            if (m >= g.M) return;
            uint32_t b, p;
            g.fPQ.divmod((uint32_t)m, b, p);
            row_out = (long long)b * g.OC * g.PQ + p;
        }
        // pass 1: + bias (vector smem loads), ReLU; pass 2: stores only, one
        // 64-bit pointer step per out_chan plane (no loads between stores)
        const int act = g.act;
#pragma unroll
        for (int j = 0; j < DC; j += 4) {
            const float4 bq = *reinterpret_cast<const float4*>(bias_s + c_begin + j);
            acc[j] = apply_act(acc[j] + bq.x, act);
            acc[j + 1] = apply_act(acc[j + 1] + bq.y, act);
            acc[j + 2] = apply_act(acc[j + 2] + bq.z, act);
            acc[j + 3] = apply_act(acc[j + 3] + bq.w, act);
        }
        float* yr = yp + row_out + (long long)(w.n0 + c_begin) * g.PQ;
        const long long pq = g.PQ;
        const int nvalid = min(DC, g.OC - (w.n0 + c_begin));
        if (nvalid >= DC) {
#pragma unroll
            for (int j = 0; j < DC; ++j, yr += pq) *yr = acc[j];
        } else {
#pragma unroll
            for (int j = 0; j < DC; ++j, yr += pq)
                if (j < nvalid) *yr = acc[j];
        }
    } else {  // row = out_chan, columns = output pixels
        const int oc = w.n0 + row;
        if (oc >= g.OC) return;
        const float rb = MODE == 7 ? 0.0f : __ldg(a.bias + oc);
        const int act = g.act;
#pragma unroll
        for (int j = 0; j < DC; ++j) acc[j] = apply_act(acc[j] + rb, act);
        const int m_begin = w.m0 + c_begin;
        uint32_t b, p;
        g.fPQ.divmod((uint32_t)min(m_begin, g.M - 1), b, p);
        float* yr = yp + ((long long)b * g.OC + oc) * g.PQ + p;  // walks pixels, hopping images at PQ
        const long long img_hop = (long long)(g.OC - 1) * g.PQ;
        int pp = (int)p;
#pragma unroll
        for (int j = 0; j < DC; ++j) {
            if (m_begin + j < g.M) *yr = acc[j];
            ++yr;
            if (++pp == g.PQ) {
                pp = 0;
                yr += img_hop;
            }
        }
    }
}

// ----------------------------------------------------------------------------- main kernel

template <int BN, bool SWAP, int MODE, int OCC, int CL, int PREC = 0>
__global__ void __launch_bounds__(TmaCfg<BN, SWAP, MODE, OCC, CL, PREC>::THREADS, OCC)
    k_tconv(const __grid_constant__ CUtensorMap tm_pix, const __grid_constant__ CUtensorMap tm_flt, TArgs a) {
    using Cfg = TmaCfg<BN, SWAP, MODE, OCC, CL, PREC>;
    constexpr int STAGES = Cfg::STAGES;
    constexpr int DC = Cfg::DRAIN_COLS;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* raw_full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* split_full = raw_full + STAGES;
    uint64_t* empty_bar = split_full + STAGES;
    uint64_t* tfull_bar = empty_bar + STAGES;  // [2]
    uint64_t* tempty_bar = tfull_bar + 2;      // [2]
    uint64_t* afree_bar = tempty_bar + 2;      // [A_SLOTS] TMEM A slot consumed by the MMAs
    uint64_t* cs_bar = afree_bar + Cfg::A_SLOTS;  // [2] cluster split-K: partials staged (leader), staging free (peers)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cs_bar + 2);
    int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);
    float* bias_s = reinterpret_cast<float*>(smem + 1024);
    const uint32_t tiles_u32 = (smem_u32(smem) + TM_HDR + 1023u) & ~1023u;

    const Geom& g = a.g;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int G = a.drain;
    const int rank = CL >= 2 ? (int)cluster_ctarank() : 0;
    constexpr int NCTA = Cfg::TWO_TILES ? 2 : 1;  // CTAs walking one unit sequence
    const int ubase = (int)blockIdx.x / NCTA, ustride = (int)gridDim.x / NCTA;
    // The loaders decode their first unit before the set-up barrier: it reads only kernel
    // parameters, and their first-touch constant-cache misses (~800 cycles, profiles/r2be)
    // then overlap barrier init / TMEM allocation instead of delaying the first TMA.
    UnitCursor ld_cur{};
    Unit ld_w{};
    bool ld_first = false;
    if ((warp == Cfg::LOAD_WARP || warp == Cfg::FLT_WARP) && lane == 0) {
        ld_cur = cursor_begin<Cfg::PIX_ROWS, Cfg::FLT_ROWS, MODE, CL>(a, ubase);
        ld_first = next_unit<Cfg::PIX_ROWS, Cfg::FLT_ROWS, MODE, CL>(a, ld_cur, ustride, rank, ld_w);
        // touch the rest of the parameter block the loaders' loops read (one field per 64 B): the
        // constant-cache lines are then resident when the loops start after griddepcontrol.wait
        const uint32_t sink = (uint32_t)g.OW + g.fPQ.mul + g.fOW.mul + g.fR.mul + (uint32_t)(size_t)a.wpk +
                              (uint32_t)a.kblocks + (uint32_t)a.bx + (uint32_t)a.by + a.fCB.mul + (uint32_t)a.drain +
                              (uint32_t)a.hp + (uint32_t)a.box_w + (uint32_t)a.kb_period + a.fTilesX.mul + (uint32_t)a.trace;
        asm volatile("" ::"r"(sink));
    }
    // the flags every warp branches on right after griddepcontrol.wait, read here for the same reason
    // (asm volatile pins the reads to this point)
    int relayout_on, flt_early_on;
    asm volatile("mov.b32 %0, %1;" : "=r"(relayout_on) : "r"(a.relayout));
    asm volatile("mov.b32 %0, %1;" : "=r"(flt_early_on) : "r"(a.flt_early));
    if (tid == 0) B2C_TRACE(a.trace, 0);

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&raw_full[s]), Cfg::TWO_LOADERS ? 2 : 1);  // each loader arrives with its bytes
            mbar_init(smem_u32(&split_full[s]), Cfg::SPLIT_ARRIVALS);
            mbar_init(smem_u32(&empty_bar[s]), CL == 2 ? 2 : 1);  // one tcgen05.commit per MMA-issuing CTA
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(smem_u32(&tfull_bar[s]), 1);
            mbar_init(smem_u32(&tempty_bar[s]), Cfg::DRAIN_ARRIVALS);
        }
        for (int s = 0; s < Cfg::A_SLOTS; ++s) mbar_init(smem_u32(&afree_bar[s]), 1);
        if (Cfg::CSPLIT) {
            mbar_init(smem_u32(&cs_bar[0]), (uint32_t)(a.split - 1) * (Cfg::DRAIN_THREADS / 32));
            mbar_init(smem_u32(&cs_bar[1]), Cfg::DRAIN_THREADS / 32);
        }
        mbar_fence_init();
    }
    if (warp == Cfg::MMA_WARP) {
        if (Cfg::PAIR)
            tmem_alloc_pair(smem_u32(tmem_slot), Cfg::TMEM_COLS);
        else
            tmem_alloc(smem_u32(tmem_slot), Cfg::TMEM_COLS);
    }
    if (warp == Cfg::LOAD_WARP && lane == 0) {
        tma_prefetch_desc(&tm_pix);
        if (MODE == 1 || MODE == 7) tma_prefetch_desc(&tm_flt);
    }
    tc_fence_before();
    __syncthreads();
    if (CL >= 2) cluster_sync_all();  // the peer's barriers exist before any multicast / remote arrive reaches them
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (tid == 0) B2C_TRACE(a.trace, 1);
    pdl_launch_dependents();
    // The loader may stream the first stages' packed filters (constant, written
    // by an earlier synchronised b2c_conv_prepare) while the previous kernel
    // (the x re-layout) is still running; everything else waits for it here.
    const bool early = Cfg::TWO_LOADERS && flt_early_on && !Cfg::RAW_B && !relayout_on && warp == Cfg::FLT_WARP;
    if (!early) pdl_wait();
    if (warp == Cfg::LOAD_WARP && lane == 0) B2C_TRACE(a.trace, 14);
    if (relayout_on) fused_relayout(a, smem + TM_HDR + 1024);
    if (tid == 0) B2C_TRACE(a.trace, 3);

    // the loaders first: their code then follows the prologue in the binary (their first TMA is on the
    // critical path of every launch; the other roles wait on barriers behind it)
    if (warp == Cfg::LOAD_WARP && lane == 0) {
        // ------------------------------------------------------------ pixel / activation loader (TMA)
        // (with one loader warp, OCC == 2, it issues each stage's filters too; the early filter
        // prefetch is then off)
        int stage = 0, n = 0;
        uint32_t phase = 0;
        B2C_TRACE(a.trace, 10);
        UnitCursor cur = ld_cur;
        Unit w = ld_w;
        for (bool have = ld_first; have; have = next_unit<Cfg::PIX_ROWS, Cfg::FLT_ROWS, MODE, CL>(a, cur, ustride, rank, w)) {
            if (n == 0) B2C_TRACE(a.trace, 11);
            int pw = 0, ph = 0, pn = 0;  // im2col base of the unit's first pixel
            if (MODE == 0 || MODE == 3 || MODE == 8) {
                uint32_t b, p, oy, ox;
                g.fPQ.divmod((uint32_t)w.m0, b, p);
                g.fOW.divmod(p, oy, ox);
                pw = (int)ox * g.S - g.P;
                ph = (int)oy * g.S - g.P;
                pn = (int)b;
            }
            for (int i = 0; i < w.nkb; ++i, ++n) {
                mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1u);
                if (n == 0) B2C_TRACE(a.trace, 12);
                const uint32_t bar = smem_u32(&raw_full[stage]);
                const uint32_t pix = tiles_u32 + (uint32_t)(stage * Cfg::STAGE_BYTES) + Cfg::PIX_OFF;
                const int kb = w.kb_begin + i;
                // MODE 4 / 6 boxes are bx*by / box_w*by rows (<= 128): the rest of the tile keeps
                // stale (finite) data whose output rows the epilogue discards.
                const uint32_t bytes = (MODE == 4   ? (uint32_t)(a.bx * a.by) * 128u
                                        : MODE == 6 ? (uint32_t)(a.box_w * a.by) * 128u
                                                    : (uint32_t)Cfg::PIX_ROWS * 128u) +
                                       (Cfg::TWO_LOADERS ? 0u : Cfg::FLT_BYTES);
                mbar_arrive_expect_tx(bar, bytes);
                if (!Cfg::TWO_LOADERS) {
                    const uint32_t dst = tiles_u32 + (uint32_t)(stage * Cfg::STAGE_BYTES) + Cfg::FLT_OFF;
                    if (MODE == 1)
                        tma_load_2d(dst, &tm_flt, bar, kb * TM_BK, w.n0);
                    else if (MODE == 7)
                        tma_load_3d(dst, &tm_flt, bar, kb * TM_BK, w.n0, w.b);
                    else
                        load_filters<Cfg::FLT_STAGE, CL, Cfg::SS>(
                            dst, reinterpret_cast<const char*>(a.wpk) +
                                     ((size_t)(w.n0 / Cfg::FLT_ROWS) * a.kblocks + kb) * (size_t)Cfg::FLT_STAGE, bar, rank);
                }
                if (n < 32) B2C_TRACE(a.trace, 176 + n);
                if (MODE == 1 || MODE == 2) {
                    tma_load_2d(pix, &tm_pix, bar, kb * TM_BK, w.m0);
                } else if (MODE == 7) {  // V[z] rows: (k, row, z)
                    tma_load_3d(pix, &tm_pix, bar, kb * TM_BK, w.m0, w.b);
                } else if (MODE == 5) {  // (pixel run, channel block, image) straight from NCHW x
                    tma_load_3d(pix, &tm_pix, bar, w.ox0, kb * TM_BK, w.b);
                } else if (MODE == 6) {  // (x, y, channel block, image) of NCHW x; x start rounded down to 16 B
                    uint32_t tap, cb, ky, kx;
                    a.fCB.divmod((uint32_t)kb, tap, cb);
                    g.fR.divmod(tap, ky, kx);
                    const int dx = w.ox0 + (int)kx - g.P;
                    const int xs = ((dx >= 0 ? dx : dx - 3) / 4) * 4;  // floor to a multiple of 4 floats
                    tma_load_4d(pix, &tm_pix, bar, xs, w.oy0 + (int)ky - g.P, (int)cb * TM_BK, w.b);
                } else if (MODE == 4) {  // (window chunk, ox, oy, ky, image)
                    uint32_t ky, kc;
                    a.fCB.divmod((uint32_t)kb, ky, kc);
                    tma_load_5d(pix, &tm_pix, bar, (int)kc * TM_BK, w.ox0, w.oy0, (int)ky, w.b);
                } else if (MODE == 0 || MODE == 8) {  // MODE 8: 64 bf16 channels per block
                    uint32_t tap, cb, ky, kx;
                    a.fCB.divmod((uint32_t)kb, tap, cb);
                    g.fR.divmod(tap, ky, kx);
                    tma_load_im2col_4d(pix, &tm_pix, bar, (int)cb * (MODE == 8 ? 64 : TM_BK), pw, ph, pn, (uint16_t)kx,
                                       (uint16_t)ky);
                } else {  // MODE 3: 8 taps x 4 channels, one 16-byte-pixel box per tap
#pragma unroll 1
                    for (int j = 0; j < TM_TAPS; ++j) {
                        const int tap = kb * TM_TAPS + j;
                        uint32_t ky = 0, kx = 0;
                        int c = 4;  // taps past R*R: channel 4 is out of bounds -> zeros
                        if (tap < g.RR) {
                            g.fR.divmod((uint32_t)tap, ky, kx);
                            c = 0;
                        }
                        tma_load_im2col_4d(pix + (uint32_t)(j * Cfg::PIX_ROWS * 16), &tm_pix, bar, c, pw, ph, pn,
                                           (uint16_t)kx, (uint16_t)ky);
                    }
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
    } else if (Cfg::TWO_LOADERS && warp == Cfg::FLT_WARP && lane == 0) {
        // ------------------------------------------------------------ filter loader (bulk copies / TMA)
        int stage = 0, n = 0;
        uint32_t phase = 0;
        int npre = 0;  // stages whose filter bytes were issued before griddepcontrol.wait
        if (early) {
            if (ld_first) {
                const Unit& w0 = ld_w;
                npre = min(STAGES, w0.nkb);
                const char* wsrc0 = reinterpret_cast<const char*>(a.wpk) +
                                    ((size_t)(w0.n0 / Cfg::FLT_ROWS) * a.kblocks + w0.kb_begin) * (size_t)Cfg::FLT_STAGE;
                for (int i = 0; i < npre; ++i) {  // fresh stages: no empty wait
                    const uint32_t bar = smem_u32(&raw_full[i]);
                    mbar_arrive_expect_tx(bar, Cfg::FLT_BYTES);
                    load_filters<Cfg::FLT_STAGE, CL, Cfg::SS>(tiles_u32 + (uint32_t)(i * Cfg::STAGE_BYTES) + Cfg::FLT_OFF,
                                                    wsrc0 + (size_t)i * Cfg::FLT_STAGE, bar, rank);
                }
            }
            B2C_TRACE(a.trace, 8);
            pdl_wait();
            B2C_TRACE(a.trace, 9);
        }
        UnitCursor cur = ld_cur;
        Unit w = ld_w;
        for (bool have = ld_first; have; have = next_unit<Cfg::PIX_ROWS, Cfg::FLT_ROWS, MODE, CL>(a, cur, ustride, rank, w)) {
            const char* wsrc = reinterpret_cast<const char*>(a.wpk) +
                               ((size_t)(w.n0 / Cfg::FLT_ROWS) * a.kblocks + w.kb_begin) * (size_t)Cfg::FLT_STAGE;
            for (int i = 0; i < w.nkb; ++i, ++n) {
                if (n >= npre) {  // (stages issued early were armed and loaded above)
                    mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1u);
                    const uint32_t bar = smem_u32(&raw_full[stage]);
                    const uint32_t dst = tiles_u32 + (uint32_t)(stage * Cfg::STAGE_BYTES) + Cfg::FLT_OFF;
                    const int kb = w.kb_begin + i;
                    mbar_arrive_expect_tx(bar, Cfg::FLT_BYTES);
                    if (MODE == 1)
                        tma_load_2d(dst, &tm_flt, bar, kb * TM_BK, w.n0);
                    else if (MODE == 7)  // U[z] rows: (k, row, z)
                        tma_load_3d(dst, &tm_flt, bar, kb * TM_BK, w.n0, w.b);
                    else
                        load_filters<Cfg::FLT_STAGE, CL, Cfg::SS>(dst, wsrc + (size_t)i * Cfg::FLT_STAGE, bar, rank);
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
    } else if (warp < 4) {
        // ------------------------------------------------------------ split: A -> TMEM (raw | lo), B lo -> smem
        if constexpr (Cfg::SS && Cfg::PAIR) {  // SS pair: forward this CTA's stage-full to the leader's MMA warp
            if (warp == 0 && lane == 0) {
                int stage = 0;
                uint32_t phase = 0;
                UnitCursor cur = cursor_begin<Cfg::PIX_ROWS, Cfg::FLT_ROWS, MODE, CL>(a, ubase);
                for (Unit w; next_unit<Cfg::PIX_ROWS, Cfg::FLT_ROWS, MODE, CL>(a, cur, ustride, rank, w);) {
                    for (int i = 0; i < w.nkb; ++i) {
                        mbar_wait(smem_u32(&raw_full[stage]), phase);
                        mbar_arrive_cluster_relaxed(smem_u32(&split_full[stage]), 0);
                        if (++stage == STAGES) {
                            stage = 0;
                            phase ^= 1u;
                        }
                    }
                }
            }
        }
        if constexpr (!Cfg::SS) {  // MODE 8: the MMAs read both operands from shared memory (no split)
        int stage = 0, n = 0;
        uint32_t phase = 0;
        const uint32_t t_lane = tmem_base + ((uint32_t)(warp * 32) << 16);  // this warp's 32 TMEM lanes
        UnitCursor cur = cursor_begin<Cfg::PIX_ROWS, Cfg::FLT_ROWS, MODE, CL>(a, ubase);
        for (Unit w; next_unit<Cfg::PIX_ROWS, Cfg::FLT_ROWS, MODE, CL>(a, cur, ustride, rank, w);) {
            for (int i = 0; i < w.nkb; ++i, ++n) {
                const uint32_t sbase = tiles_u32 + (uint32_t)(stage * Cfg::STAGE_BYTES);
                mbar_wait(smem_u32(&raw_full[stage]), phase);
                if (tid == 0 && n < 32) B2C_TRACE(a.trace, 16 + n);
                const int aslot = n % Cfg::A_SLOTS;
                if (n >= Cfg::A_SLOTS)  // the MMAs of iteration n - A_SLOTS are done with this TMEM slot
                    mbar_wait(smem_u32(&afree_bar[aslot]), (uint32_t)((n / Cfg::A_SLOTS) - 1) & 1u);
                tc_fence_after();
                const uint32_t acol = (uint32_t)(Cfg::ACC_COLS + aslot * 64);
                if (MODE == 5) {  // channel-major box [32 ch][128 px]: this thread's pixel is column tid
                    a_to_tmem_cmajor<PREC>(sbase, tid, t_lane + acol, TM_M);
                } else if (MODE == 6) {  // box [32 ch][by][box_w] starting at the 16-byte-aligned x below this tap
                    uint32_t tap, cb, ky, kx;
                    a.fCB.divmod((uint32_t)(w.kb_begin + i), tap, cb);
                    g.fR.divmod(tap, ky, kx);
                    const int dx = (int)kx - g.P;
                    const int shift = dx - ((dx >= 0 ? dx : dx - 3) / 4) * 4;  // dx - floor(dx / 4) * 4
                    const int y = tid / a.bx, xx = tid - (tid / a.bx) * a.bx;
                    const int idx = y < a.by ? y * a.box_w + xx + shift : 0;  // rows past the tile: any in-box value
                    a_to_tmem_cmajor<PREC>(sbase, idx, t_lane + acol, a.by * a.box_w);
                }
                else if (PREC == 1)
                    a_to_tmem_bf16<Cfg::SW128>(sbase, tid, t_lane + acol);
                else if (PREC == 2)
                    a_to_tmem_e4m3<Cfg::SW128>(sbase, tid, t_lane + acol);
                else if (!(a.trace & 8))
                    a_to_tmem<Cfg::SW128, Cfg::A_PRESPLIT>(sbase, tid, t_lane + acol);  // debug bit 3: skip
                if (Cfg::B_SPLIT && !(a.trace & 4)) split_tile<BN>(sbase + Cfg::A_SMEM, tid);
                fence_proxy_async_smem();
                tmem_st_wait();
                tc_fence_before();
                if (Cfg::PAIR) {  // one arrive per warp on the leader's barrier (relaxed: a release at
                    // cluster scope costs ~1.5k cycles per stage and paced the whole pipeline; the TMEM
                    // stores are complete at tcgen05.wait::st and the smem operand was written by TMA)
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster_relaxed(smem_u32(&split_full[stage]), 0);
                } else {
                    mbar_arrive(smem_u32(&split_full[stage]));
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
        }
    } else if (warp < Cfg::MMA_WARP) {
        // ------------------------------------------------------------ drain + epilogue
        const int dw = warp - 4;
        const int quarter = dw & 3;  // TMEM lane quarter = warp % 4
        const int c_begin = (dw >> 2) * DC;
        const int dtid = tid - 128;
        const int row = quarter * 32 + lane;  // TMEM lane = MMA M row
        const uint32_t t_row = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c_begin;
        int ui = 0;  // unit ordinal (trace slots)
        int cidx = 0;
        int cs_uses = 0;  // cluster split-K: units staged / reduced so far (barrier phases)
        const uint32_t stg = tiles_u32 + (uint32_t)(STAGES * Cfg::STAGE_BYTES);  // staging tile (CSPLIT)
        UnitCursor cur = cursor_begin<Cfg::PIX_ROWS, Cfg::FLT_ROWS, MODE, CL>(a, ubase);
        for (Unit w; next_unit<Cfg::PIX_ROWS, Cfg::FLT_ROWS, MODE, CL>(a, cur, ustride, rank, w);) {
            float acc[DC];
#pragma unroll
            for (int j = 0; j < DC; ++j) acc[j] = 0.0f;
            float bpre = 0.0f;  // this thread's share of the unit's biases, loaded under the main loop
            if (!SWAP && MODE != 7 && dtid < BN && w.n0 + dtid < g.OC) bpre = __ldg(a.bias + w.n0 + dtid);
            const int nch = (w.nkb + G - 1) / G;
            for (int c = 0; c < nch; ++c, ++cidx) {
                const int slot = cidx & 1;
                mbar_wait(smem_u32(&tfull_bar[slot]), (uint32_t)(cidx >> 1) & 1u);
                tc_fence_after();
                tmem_add_cols<DC>(t_row + (uint32_t)(slot * Cfg::SLOT_COLS), acc);
                if (Cfg::FUSED) tmem_add_cols<DC>(t_row + (uint32_t)(slot * Cfg::SLOT_COLS + BN), acc);
                tc_fence_before();
                if (Cfg::PAIR) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster_relaxed(smem_u32(&tempty_bar[slot]), 0);
                } else {
                    mbar_arrive(smem_u32(&tempty_bar[slot]));
                }
            }
            if (dtid == 0 && ui == 0) B2C_TRACE(a.trace, 4);
            if (dtid == 0 && ui < 24) B2C_TRACE(a.trace, 208 + 2 * ui);
            if (!w.ghost)
                epilogue_unit<BN, SWAP, DC, Cfg::DRAIN_THREADS, MODE, Cfg::CSPLIT>(a, w, acc, c_begin, row, dtid, last_flag,
                                                                                 bias_s, bpre, stg, cs_bar, cs_uses);
            if (dtid == 0 && ui < 24) B2C_TRACE(a.trace, 209 + 2 * ui);
            ++ui;
        }
        if (dtid == 0) B2C_TRACE(a.trace, 6);
    } else if (warp == Cfg::MMA_WARP && (!Cfg::PAIR || rank == 0)) {
        // ------------------------------------------------------------ MMA issuer (whole warp waits, one lane issues)
        constexpr uint32_t idesc = umma_idesc(PREC == 1 ? 1 : PREC == 2 ? 0 : 2, Cfg::PAIR ? 2 * TM_M : TM_M, BN);
        int stage = 0, cidx = 0, n = 0;
        uint32_t phase = 0;
        UnitCursor cur = cursor_begin<Cfg::PIX_ROWS, Cfg::FLT_ROWS, MODE, CL>(a, ubase);
        for (Unit w; next_unit<Cfg::PIX_ROWS, Cfg::FLT_ROWS, MODE, CL>(a, cur, ustride, rank, w);) {
            int kin = 0;
            int kph = w.kb_begin % a.kb_period;  // position of this K block within its period
            for (int i = 0; i < w.nkb; ++i, ++n) {
                const int slot = cidx & 1;
                const int nsteps = (kph == a.kb_period - 1) ? a.ksteps_last : TM_BK / 8;
                if (++kph == a.kb_period) kph = 0;
                const bool first = kin == 0;
                const bool last = (kin == G - 1) || (i == w.nkb - 1);
                if (first && cidx >= 2) {
                    if (Cfg::PAIR)
                        mbar_wait_cluster(smem_u32(&tempty_bar[slot]), (uint32_t)((cidx >> 1) - 1) & 1u);
                    else
                        mbar_wait(smem_u32(&tempty_bar[slot]), (uint32_t)((cidx >> 1) - 1) & 1u);
                    tc_fence_after();
                }
                // split_full is armed only after the split threads observed
                // raw_full, so it also covers the TMA / bulk bytes (a pair: both CTAs').
                if (Cfg::PAIR)
                    mbar_wait_cluster(smem_u32(&split_full[stage]), phase);
                else if (Cfg::SS)  // no split pass: wait for the TMA / bulk bytes themselves (a pair: forwarded)
                    mbar_wait(smem_u32(&raw_full[stage]), phase);
                else
                    mbar_wait(smem_u32(&split_full[stage]), phase);
                tc_fence_after();
                if (lane == 0 && n < 32) B2C_TRACE(a.trace, 112 + n);
                if (elect_one_sync()) {
                    const uint32_t a_hi = tmem_base + (uint32_t)(Cfg::ACC_COLS + (n % Cfg::A_SLOTS) * 64);
                    const uint32_t a_lo = a_hi + 32;
                    const uint32_t b_raw = tiles_u32 + (uint32_t)(stage * Cfg::STAGE_BYTES + Cfg::A_SMEM);
                    const uint32_t b_lo = b_raw + (Cfg::PAIR ? BN / 2 : BN) * 128;
                    const uint32_t d = tmem_base + (uint32_t)(slot * Cfg::SLOT_COLS);
                    if constexpr (Cfg::SS) {  // bf16 SS: four K = 16 MMAs per 64-wide K block, +32 B per step
                        const uint32_t a_s = tiles_u32 + (uint32_t)(stage * Cfg::STAGE_BYTES + Cfg::PIX_OFF);
#pragma unroll
                        for (int s = 0; s < 4; ++s) {
                            if (s >= nsteps) break;  // all-zero channel tail
                            if constexpr (Cfg::PAIR)
                                mma_bf16_pair(d, umma_desc_sw128(a_s + s * 32), umma_desc_sw128(b_raw + s * 32), idesc,
                                              (first && s == 0) ? 0u : 1u);
                            else
                                mma_bf16(d, umma_desc_sw128(a_s + s * 32), umma_desc_sw128(b_raw + s * 32), idesc,
                                         (first && s == 0) ? 0u : 1u);
                        }
                    } else if constexpr (PREC == 2) {  // e4m3: one K=32 MMA per K block ([2 chunks][rows][16 B])
                        mma_e4m3_ts(d, a_hi, umma_desc(b_raw, BN * 16, 128), idesc, first ? 0u : 1u);
                    } else if constexpr (PREC == 1) {  // bf16: two K=16 MMAs per 32-wide K block
#pragma unroll
                        for (int s = 0; s < TM_BK / 16; ++s) {
                            if (2 * s >= nsteps) break;
                            const uint64_t db = umma_desc(b_raw + s * 2 * BN * 16, BN * 16, 128);
                            mma_bf16_ts(d, a_hi + 8 * s, db, idesc, (first && s == 0) ? 0u : 1u);
                        }
                    } else {
#pragma unroll
                    for (int s = 0; s < TM_BK / 8; ++s) {
                        if (s >= nsteps) break;  // all-zero K tail of the block (exact: 0 * finite)
                        uint64_t dbh, dbl;
                        if (Cfg::SW128) {
                            dbh = umma_desc_sw128(b_raw + s * 32);
                            dbl = umma_desc_sw128(b_lo + s * 32);
                        } else {  // [16-byte chunk][rows][16 B]: K-adjacent core matrices rows*16 B apart
                            dbh = umma_desc(b_raw + s * 2 * BN * 16, BN * 16, 128);
                            dbl = umma_desc(b_lo + s * 2 * BN * 16, BN * 16, 128);
                        }
                        if constexpr (Cfg::FUSED) {  // [d, d+2BN) = Ahi*[Braw | Blo]; [d+BN, d+2BN) += Alo*Braw
                            constexpr uint32_t idesc2 = umma_idesc(2, TM_M, 2 * BN);
                            mma_tf32_ts(d, a_hi + 8 * s, dbh, idesc2, (first && s == 0) ? 0u : 1u);
                            mma_tf32_ts(d + BN, a_lo + 8 * s, dbh, idesc, 1u);
                        } else if constexpr (Cfg::PAIR) {
                            mma_tf32_ts_pair(d, a_hi + 8 * s, dbh, idesc, (first && s == 0) ? 0u : 1u);
                            if (!(a.trace & 2)) {
                                mma_tf32_ts_pair(d, a_hi + 8 * s, dbl, idesc, 1u);
                                mma_tf32_ts_pair(d, a_lo + 8 * s, dbh, idesc, 1u);
                            }
                        } else {
                        mma_tf32_ts(d, a_hi + 8 * s, dbh, idesc, (first && s == 0) ? 0u : 1u);
                        if (!(a.trace & 2)) {  // debug bit 1: hi*hi only (timing experiments only)
                            mma_tf32_ts(d, a_hi + 8 * s, dbl, idesc, 1u);
                            mma_tf32_ts(d, a_lo + 8 * s, dbh, idesc, 1u);
                        }
                        }
                    }
                    }
                    if (Cfg::PAIR) {  // both CTAs' stage, A slot and accumulator slot
                        tc_commit_pair(smem_u32(&empty_bar[stage]), (uint16_t)0x3);
                        if (!Cfg::SS)  // (SS: no A slots in TMEM, nobody waits on afree)
                            tc_commit_pair(smem_u32(&afree_bar[n % Cfg::A_SLOTS]), (uint16_t)0x3);
                        if (last) tc_commit_pair(smem_u32(&tfull_bar[slot]), (uint16_t)0x3);
                    } else {
                    if (CL == 2)  // the stage's filter half may be refilled by either CTA
                        tc_commit_mc(smem_u32(&empty_bar[stage]), (uint16_t)0x3);
                    else
                        tc_commit(smem_u32(&empty_bar[stage]));
                    if (!Cfg::SS) tc_commit(smem_u32(&afree_bar[n % Cfg::A_SLOTS]));
                    if (last) tc_commit(smem_u32(&tfull_bar[slot]));
                    }
                    if (n < 32) B2C_TRACE(a.trace, 144 + n);
                }
                __syncwarp();
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1u;
                }
                if (last) {
                    kin = 0;
                    ++cidx;
                } else {
                    ++kin;
                }
            }
        }
        if (lane == 0) B2C_TRACE(a.trace, 5);
    }
    if (tid == 0) B2C_TRACE(a.trace, 2);
    __syncthreads();
    if (CL >= 2) cluster_sync_all();  // no multicast or remote commit may still target this CTA
    if (warp == Cfg::MMA_WARP) {
        tc_fence_after();
        if (Cfg::PAIR)
            tmem_dealloc_pair(tmem_base, Cfg::TMEM_COLS);
        else
            tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
    }
    if (tid == 0) B2C_TRACE(a.trace, 7);
}

}  // namespace b2c
