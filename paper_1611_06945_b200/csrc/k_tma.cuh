// TMA-fed tcgen05 / TMEM implicit-GEMM convolution, fp32-exact via 3xTF32.
//
// Same GEMM view and precision scheme as k_umma (cuclgen/variants.py:376-414
// ConvTiled's M = img*oy*ox, N = out_chan, K = in_chan*ksz*ksz; fused
// bias/ReLU epilogue of variants.py:160-165), but no thread ever gathers an
// operand element from global memory:
//
//   * MODE 0 (conv): the activations are re-laid out once per call to NHWC
//     (k_nchw_to_nhwc, the B200 form of the reference's required_formats
//     conversion, variants.py:416-424 / runner.py:96-105, charged to the op)
//     and one TMA *im2col* load per K block brings 128 (or BN) output pixels x
//     32 channels of one filter tap straight into the K-major SWIZZLE_128B
//     layout the tensor core reads; the TMA unit zero-fills the padding.
//     Filters are packed once (cached) into the same swizzled layout, raw and
//     lo halves, and streamed with one cp.async.bulk per K block.
//   * MODE 2 (1x1, stride 1, no pad; conv_1x1, variants.py:279-325): the NHWC
//     copy is a plain [pixels][C] matrix, so a 2-D tiled TMA box replaces
//     the im2col walk (filters as in MODE 0).
//   * MODE 1 (fc, variants.py:328-373): the whole-image filter makes both
//     operands plain row-major [rows][K] matrices (x as [img][ic*h*w], w as
//     [oc][ic*h*w]); both are loaded raw by 2-D tiled TMA, so the 151 MB fc6
//     weight tensor is read from HBM exactly once, with no pack.
//
// Warp roles (320 threads):
//   warps 0-7  split + drain + epilogue.  All 256 threads take every stage
//              (each its 1/256 of the tile; a group that ran ahead over
//              alternate stages could see a stale mbarrier parity, since TMA
//              loads may land out of order): they wait for the TMA bytes, write
//              lo = x - trunc_tf32(x) beside every raw operand the TMA loaded
//              (elementwise on the swizzled tile, so no index math), and
//              drain finished TMEM chunks into fp32 register sums (the
//              accumulation-precision scheme of k_umma.cuh).
//   warp 8     TMEM allocation; lane 0 issues 12 tcgen05.mma.kind::tf32 per
//              K block (4 K=8 steps x {hi*hi, hi*lo, lo*hi}).
//   warp 9     lane 0 issues the TMA / bulk loads.
// Kernels are launched with programmatic dependent launch: the prologue
// (barrier init, TMEM alloc, tensor-map prefetch) overlaps the previous
// kernel's tail; griddepcontrol.wait precedes every global access.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "k_umma.cuh"  // tmem_add_cols, k_pack_filters

namespace b2c {

constexpr int TM_M = 128;
constexpr int TM_BK = 32;                 // fp32 K elements per stage (128-byte rows)
constexpr int TM_SPLIT = 256;             // split / drain / epilogue threads (warps 0-7)
constexpr int TM_MMA_WARP = 8;
constexpr int TM_LOAD_WARP = 9;
constexpr int TM_THREADS = 320;
constexpr int TM_HDR = 256;               // barriers, TMEM slot, flags
constexpr int TM_BIAS = 1024;             // bias of the tile's out_chans (<= 256 floats)
constexpr int TM_MAX_SMEM = 232448;       // 227 KB opt-in per CTA

template <int BN, bool SWAP>
struct TmaCfg {
    static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "BN: multiple of 32 in [32, 256]");
    static constexpr int A_ROWS = TM_M;
    static constexpr int B_ROWS = BN;
    static constexpr int PIX_ROWS = SWAP ? B_ROWS : A_ROWS;
    static constexpr int FLT_ROWS = SWAP ? A_ROWS : B_ROWS;
    static constexpr int A_BYTES = 2 * A_ROWS * 128;  // raw + lo
    static constexpr int B_BYTES = 2 * B_ROWS * 128;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int PIX_OFF = SWAP ? A_BYTES : 0;  // raw part; lo follows at + PIX_ROWS*128
    static constexpr int FLT_OFF = SWAP ? 0 : A_BYTES;
    static constexpr int BUDGET = TM_MAX_SMEM - TM_HDR - TM_BIAS - 1024;
    static constexpr int STAGES = (BUDGET / STAGE_BYTES) > 8 ? 8 : (BUDGET / STAGE_BYTES);
    static constexpr int SMEM = TM_HDR + TM_BIAS + 1024 + STAGES * STAGE_BYTES;
    static constexpr int TMEM_COLS = 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
    static constexpr int HALF = BN / 2;
    static_assert(STAGES >= 2, "need at least two stages");
    static_assert(HALF % 8 == 0, "TMEM drain granularity");
};

struct TArgs {
    Geom g;
    const float* wpk;   // MODE 0: packed filters [flt tile][K block][raw | lo][rows][128 B swizzled]
    const float* bias;
    float* y;
    float* ws;          // split-K partials [tiles][split][BN][128]
    int* sems;          // split-K tickets [tiles], zero at rest
    int split, kps, kblocks;
    FastDiv fCB;        // MODE 0: channel blocks of 32 per filter tap
    int drain, lag;
    int trace;          // debug: record phase clocks of CTA 0 into g_b2c_trace
};

// ----------------------------------------------------------------------------- NCHW -> NHWC

// x [N][C][HW] -> xh [N][HW][C]; 32x32 tiles through shared memory so both the
// read (along pixels) and the write (along channels) are coalesced.
__global__ void __launch_bounds__(256) k_nchw_to_nhwc(const float* __restrict__ x, float* __restrict__ xh, int C,
                                                      int HW) {
    __shared__ float tile[32][33];
    pdl_launch_dependents();
    pdl_wait();
    const int n = blockIdx.z;
    const int p0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const float* src = x + (size_t)n * C * HW;
    float* dst = xh + (size_t)n * HW * C;
#pragma unroll
    for (int j = ty; j < 32; j += 8) {
        const int c = c0 + j, p = p0 + tx;
        tile[j][tx] = (c < C && p < HW) ? __ldg(src + (size_t)c * HW + p) : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int j = ty; j < 32; j += 8) {
        const int p = p0 + j, c = c0 + tx;
        if (p < HW && c < C) dst[(size_t)p * C + c] = tile[tx][j];
    }
}

// ----------------------------------------------------------------------------- split-K
// Write this CTA's fp32 partial tile; returns true in the CTA that arrives
// last for its output tile (it then reduces all partials in split order, so
// the result is deterministic).  Called by all 256 split/epilogue threads.
template <int BN>
__device__ __forceinline__ bool split_reduce_last(const TArgs& a, const float* acc, int c_begin, int row, int z,
                                                  int* last_flag) {
    constexpr int HALF = BN / 2;
    const int tile = blockIdx.y * gridDim.x + blockIdx.x;
    float* part = a.ws + ((size_t)tile * a.split + z) * BN * TM_M;
#pragma unroll
    for (int j = 0; j < HALF; ++j) __stcg(part + (size_t)(c_begin + j) * TM_M + row, acc[j]);
    __threadfence();
    named_bar_sync(1, TM_SPLIT);
    if (threadIdx.x == 0) {
        const int ticket = atomicAdd(a.sems + tile, 1);
        *last_flag = (ticket == a.split - 1);
    }
    named_bar_sync(1, TM_SPLIT);
    const bool last = *last_flag != 0;
    if (last) {
        __threadfence();
        if (threadIdx.x == 0) a.sems[tile] = 0;
    }
    return last;
}

// ----------------------------------------------------------------------------- main kernel

template <int BN, bool SWAP, int MODE>
__global__ void __launch_bounds__(TM_THREADS, 1)
    k_tconv(const __grid_constant__ CUtensorMap tm_pix, const __grid_constant__ CUtensorMap tm_flt, TArgs a) {
    using Cfg = TmaCfg<BN, SWAP>;
    constexpr int STAGES = Cfg::STAGES;
    constexpr int HALF = Cfg::HALF;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* raw_full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* split_full = raw_full + STAGES;
    uint64_t* empty_bar = split_full + STAGES;
    uint64_t* tfull_bar = empty_bar + STAGES;  // [2]
    uint64_t* tempty_bar = tfull_bar + 2;      // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
    int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);
    float* bias_s = reinterpret_cast<float*>(smem + TM_HDR);
    const uint32_t tiles_u32 = (smem_u32(smem) + TM_HDR + TM_BIAS + 1023u) & ~1023u;

    const Geom& g = a.g;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    if (tid == 0) B2C_TRACE(a.trace, 0);

    const int m0 = blockIdx.x * Cfg::PIX_ROWS;
    const int n0 = blockIdx.y * Cfg::FLT_ROWS;
    const int z = blockIdx.z;
    const int kb_begin = z * a.kps;
    const int kb_end = min(a.kblocks, kb_begin + a.kps);
    const int nkb = kb_end - kb_begin;
    const int G = a.drain;
    const int nchunks = (nkb + G - 1) / G;

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&raw_full[s]), 1);
            mbar_init(smem_u32(&split_full[s]), TM_SPLIT);
            mbar_init(smem_u32(&empty_bar[s]), 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(smem_u32(&tfull_bar[s]), 1);
            mbar_init(smem_u32(&tempty_bar[s]), TM_SPLIT);
        }
        mbar_fence_init();
    }
    if (warp == TM_MMA_WARP) tmem_alloc(smem_u32(tmem_slot), Cfg::TMEM_COLS);
    if (warp == TM_LOAD_WARP && lane == 0) {
        tma_prefetch_desc(&tm_pix);
        if (MODE == 1) tma_prefetch_desc(&tm_flt);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (tid == 0) B2C_TRACE(a.trace, 1);
    pdl_launch_dependents();
    pdl_wait();
    if (tid == 0) B2C_TRACE(a.trace, 2);

    if (warp < TM_MMA_WARP) {
        // ------------------------------------------------------------ split + drain + epilogue
        const int gtid = tid;
        const int quarter = warp & 3, half = warp >> 2;
        const int c_begin = half * HALF;
        const uint32_t t_row = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c_begin;
        float acc[HALF];
#pragma unroll
        for (int j = 0; j < HALF; ++j) acc[j] = 0.0f;
        if (!SWAP && tid < BN) {  // the tile's out_chan biases, read by the epilogue from smem
            const int oc = n0 + tid;
            bias_s[tid] = oc < g.OC ? __ldg(a.bias + oc) : 0.0f;
        }

        auto drain_chunk = [&](int c) {
            const int slot = c & 1;
            mbar_wait(smem_u32(&tfull_bar[slot]), (uint32_t)(c >> 1) & 1u);
            tc_fence_after();
            tmem_add_cols<HALF>(t_row + (uint32_t)(slot * BN), acc);
            tc_fence_before();
            mbar_arrive(smem_u32(&tempty_bar[slot]));
        };
        auto split_region = [&](uint32_t raw, int rows) {
            const uint32_t lo = raw + (uint32_t)rows * 128u;
            for (int i = gtid; i < rows * 8; i += TM_SPLIT) {
                const float4 v = lds128(raw + (uint32_t)i * 16u);
                float h, l0, l1, l2, l3;
                split_tf32(v.x, h, l0);
                split_tf32(v.y, h, l1);
                split_tf32(v.z, h, l2);
                split_tf32(v.w, h, l3);
                sts128(lo + (uint32_t)i * 16u, l0, l1, l2, l3);
            }
        };

        int drained = 0;
        for (int it = 0; it < nkb; ++it) {
            while (drained < nchunks && it >= (drained + 1) * G + a.lag) drain_chunk(drained++);
            const int stage = it % STAGES;
            const uint32_t phase = (uint32_t)(it / STAGES) & 1u;
            const uint32_t sbase = tiles_u32 + (uint32_t)(stage * Cfg::STAGE_BYTES);
            mbar_wait(smem_u32(&raw_full[stage]), phase);
            if (gtid == 0 && it < 32) B2C_TRACE(a.trace, 16 + it);
            if (!(a.trace & 4)) {  // debug bit 2: skip the split (timing experiments only)
                split_region(sbase + Cfg::PIX_OFF, Cfg::PIX_ROWS);
                if (MODE == 1) split_region(sbase + Cfg::FLT_OFF, Cfg::FLT_ROWS);
            }
            fence_proxy_async_smem();
            mbar_arrive(smem_u32(&split_full[stage]));
            if (gtid == 0 && it < 32) B2C_TRACE(a.trace, 48 + it);
        }
        while (drained < nchunks) drain_chunk(drained++);
        if (tid == 0) B2C_TRACE(a.trace, 4);

        // ------------------------------------------------------------ epilogue
        // Values are produced in groups of 8 columns (bias from smem first), so
        // no global load sits between the stores.
        float* __restrict__ yp = a.y;
        const int row = quarter * 32 + lane;  // TMEM lane = MMA M row
        named_bar_sync(2, TM_SPLIT);      // bias_s visible
        if (!SWAP) {
            const int m = m0 + row;
            const bool row_ok = m < g.M;
            long long row_out = 0;
            if (row_ok) {
                uint32_t b, p;
                g.fPQ.divmod((uint32_t)m, b, p);
                row_out = (long long)b * g.OC * g.PQ + p;
            }
            auto store8 = [&](int c0, const float* v) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int oc = n0 + c0 + j;
                    if (row_ok && oc < g.OC) yp[row_out + (long long)oc * g.PQ] = apply_act(v[j] + bias_s[c0 + j], g.act);
                }
            };
            if (a.split == 1) {
#pragma unroll
                for (int j0 = 0; j0 < HALF; j0 += 8) store8(c_begin + j0, acc + j0);
            } else if (split_reduce_last<BN>(a, acc, c_begin, row, z, last_flag)) {
                const float* __restrict__ base = a.ws + (size_t)(blockIdx.y * gridDim.x + blockIdx.x) * a.split * BN * TM_M;
#pragma unroll 1
                for (int j0 = 0; j0 < HALF; j0 += 8) {
                    float v[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) v[j] = 0.f;
                    for (int zz = 0; zz < a.split; ++zz)
#pragma unroll
                        for (int j = 0; j < 8; ++j) v[j] += __ldcg(base + ((size_t)zz * BN + c_begin + j0 + j) * TM_M + row);
                    store8(c_begin + j0, v);
                }
            }
        } else {
            const int oc = n0 + row;
            const bool row_ok = oc < g.OC;
            const float rb = row_ok ? __ldg(a.bias + oc) : 0.0f;
            auto store8 = [&](int c0, const float* v) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int m = m0 + c0 + j;
                    if (row_ok && m < g.M) {
                        uint32_t b, p;
                        g.fPQ.divmod((uint32_t)m, b, p);
                        yp[((long long)b * g.OC + oc) * g.PQ + p] = apply_act(v[j] + rb, g.act);
                    }
                }
            };
            if (a.split == 1) {
#pragma unroll
                for (int j0 = 0; j0 < HALF; j0 += 8) store8(c_begin + j0, acc + j0);
            } else if (split_reduce_last<BN>(a, acc, c_begin, row, z, last_flag)) {
                const float* __restrict__ base = a.ws + (size_t)(blockIdx.y * gridDim.x + blockIdx.x) * a.split * BN * TM_M;
#pragma unroll 1
                for (int j0 = 0; j0 < HALF; j0 += 8) {
                    float v[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) v[j] = 0.f;
                    for (int zz = 0; zz < a.split; ++zz)
#pragma unroll
                        for (int j = 0; j < 8; ++j) v[j] += __ldcg(base + ((size_t)zz * BN + c_begin + j0 + j) * TM_M + row);
                    store8(c_begin + j0, v);
                }
            }
        }
    } else if (warp == TM_MMA_WARP) {
        // ------------------------------------------------------------ MMA issuer (whole warp waits, one lane issues)
        constexpr uint32_t idesc = umma_idesc(2, TM_M, BN);
        int stage = 0, kin = 0, cidx = 0;
        uint32_t phase = 0;
        for (int it = 0; it < nkb; ++it) {
            const int slot = cidx & 1;
            const bool first = kin == 0;
            const bool last = (kin == G - 1) || (it == nkb - 1);
            if (first && cidx >= 2) {
                mbar_wait(smem_u32(&tempty_bar[slot]), (uint32_t)((cidx >> 1) - 1) & 1u);
                tc_fence_after();
            }
            if (lane == 0 && it < 32) B2C_TRACE(a.trace, 80 + it);
            // split_full is armed by the split threads only after they observed
            // raw_full, so it also covers the TMA / bulk bytes.
            mbar_wait(smem_u32(&split_full[stage]), phase);
            tc_fence_after();
            if (lane == 0 && it < 32) B2C_TRACE(a.trace, 112 + it);
            if (elect_one_sync()) {
                const uint32_t a_raw = tiles_u32 + (uint32_t)(stage * Cfg::STAGE_BYTES);
                const uint32_t a_lo = a_raw + TM_M * 128;
                const uint32_t b_raw = a_raw + Cfg::A_BYTES;
                const uint32_t b_lo = b_raw + BN * 128;
                const uint32_t d = tmem_base + (uint32_t)(slot * BN);
#pragma unroll
                for (int s = 0; s < TM_BK / 8; ++s) {
                    const uint64_t dah = umma_desc_sw128(a_raw + s * 32);
                    const uint64_t dal = umma_desc_sw128(a_lo + s * 32);
                    const uint64_t dbh = umma_desc_sw128(b_raw + s * 32);
                    const uint64_t dbl = umma_desc_sw128(b_lo + s * 32);
                    mma_tf32(d, dah, dbh, idesc, (first && s == 0) ? 0u : 1u);
                    if (!(a.trace & 2)) {  // debug bit 1: hi*hi only (timing experiments only)
                        mma_tf32(d, dah, dbl, idesc, 1u);
                        mma_tf32(d, dal, dbh, idesc, 1u);
                    }
                }
                tc_commit(smem_u32(&empty_bar[stage]));
                if (last) tc_commit(smem_u32(&tfull_bar[slot]));
                if (it < 32) B2C_TRACE(a.trace, 144 + it);
            }
            __syncwarp();
            if (++stage == STAGES) {
                stage = 0;
                phase ^= 1u;
            }
            if (++kin == G) {
                kin = 0;
                ++cidx;
            }
        }
        if (lane == 0) B2C_TRACE(a.trace, 5);
    } else {
        if (lane == 0) {
            // ------------------------------------------------------------ TMA / bulk loader
            int pw = 0, ph = 0, pn = 0;  // MODE 0: im2col base of the tile's first pixel
            if (MODE == 0) {
                uint32_t b, p, oy, ox;
                g.fPQ.divmod((uint32_t)m0, b, p);
                g.fOW.divmod(p, oy, ox);
                pw = (int)ox * g.S - g.P;
                ph = (int)oy * g.S - g.P;
                pn = (int)b;
            }
            const char* wsrc = reinterpret_cast<const char*>(a.wpk) +
                               ((size_t)blockIdx.y * a.kblocks + kb_begin) * (size_t)(2 * Cfg::FLT_ROWS * 128);
            constexpr uint32_t bytes =
                Cfg::PIX_ROWS * 128 + (MODE != 1 ? 2 * Cfg::FLT_ROWS * 128 : Cfg::FLT_ROWS * 128);
            for (int it = 0; it < nkb; ++it) {
                const int stage = it % STAGES;
                const uint32_t phase = (uint32_t)(it / STAGES) & 1u;
                mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1u);
                const uint32_t bar = smem_u32(&raw_full[stage]);
                const uint32_t sbase = tiles_u32 + (uint32_t)(stage * Cfg::STAGE_BYTES);
                const int kb = kb_begin + it;
                mbar_arrive_expect_tx(bar, bytes);
                if (it < 32) B2C_TRACE(a.trace, 176 + it);
                if (MODE == 2) {  // 1x1, stride 1, no pad: x is a plain [pixels][C] NHWC matrix
                    tma_load_2d(sbase + Cfg::PIX_OFF, &tm_pix, bar, kb * TM_BK, m0);
                    bulk_g2s(sbase + Cfg::FLT_OFF, wsrc + (size_t)it * (2 * Cfg::FLT_ROWS * 128),
                             2 * Cfg::FLT_ROWS * 128, bar);
                } else if (MODE == 0) {
                    uint32_t tap, cb, ky, kx;
                    a.fCB.divmod((uint32_t)kb, tap, cb);
                    g.fR.divmod(tap, ky, kx);
                    tma_load_im2col_4d(sbase + Cfg::PIX_OFF, &tm_pix, bar, (int)cb * TM_BK, pw, ph, pn,
                                       (uint16_t)kx, (uint16_t)ky);
                    bulk_g2s(sbase + Cfg::FLT_OFF, wsrc + (size_t)it * (2 * Cfg::FLT_ROWS * 128),
                             2 * Cfg::FLT_ROWS * 128, bar);
                } else {
                    tma_load_2d(sbase + Cfg::PIX_OFF, &tm_pix, bar, kb * TM_BK, m0);
                    tma_load_2d(sbase + Cfg::FLT_OFF, &tm_flt, bar, kb * TM_BK, n0);
                }
            }
        }
        __syncwarp();
    }
    if (tid == 0) B2C_TRACE(a.trace, 6);
    __syncthreads();
    if (warp == TM_MMA_WARP) {
        tc_fence_after();
        tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
    }
    if (tid == 0) B2C_TRACE(a.trace, 7);
}

}  // namespace b2c
