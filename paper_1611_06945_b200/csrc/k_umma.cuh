// tcgen05 / TMEM implicit-GEMM convolution, fp32-exact via 3xTF32.
//
// The GEMM view is the reference ConvTiled's (cuclgen/variants.py:376-414):
// M = img*oy*ox output pixels, N = out_chan, K = in_chan*ksz*ksz, walked in
// (ic, ky, kx) order, with the bias/ReLU epilogue of variants.py:160-165 and
// graphopt.fuse_activations (graphopt.py:59-86) fused into the TMEM drain.
// Variants map onto template arguments:
//   conv_umma  (k x k, any stride/pad)    KMODE=0  (im2col gather)
//   conv_1x1   (variants.py:279-325)      KMODE=1  (no window, pixel stride)
//   conv_fc    (variants.py:328-373)      KMODE=2  (whole-image filter = flat
//                                                   dot, variants.py:354-356)
// SWAP=false: MMA M = 128 output pixels, MMA N = BN out_chans (TMEM lane =
// pixel, so the NCHW epilogue store is coalesced along pixels).
// SWAP=true : MMA M = 128 out_chans, MMA N = BN pixels, for small-pixel ops
// (7x7/6x6 maps, fc layers) where a 128-pixel tile would be mostly empty.
//
// Precision: tcgen05 kind::tf32 keeps 10 explicit mantissa bits, too few for
// the reference tolerance (rel 1e-5 for K <= 4096, oracle.py:31-38).  Each
// operand x is split in registers into hi = trunc_tf32(x) and lo = x - hi
// (both exact in fp32) and D += Ahi*Bhi + Ahi*Blo + Alo*Bhi accumulates in
// fp32 TMEM ("3xTF32"); the dropped lo*lo term is ~2^-21 relative.
//
// CTA = 9 warps.  Warps 0-7 (256 threads) are producers: each owns one or two
// operand rows (a pixel's im2col row or a filter row) and, per 32-wide K
// block, loads 32 fp32 values, splits them, and stores hi/lo 16-byte chunks
// into the UMMA K-major no-swizzle layout (8-row x 16-byte core matrices;
// LBO = 128 B between K-adjacent core matrices, SBO = 1024 B between 8-row
// groups), then fence.proxy.async + mbarrier arrive.  Warp 8 allocates TMEM
// and one lane issues 12 tcgen05.mma per K block (4 K=8 steps x 3 terms),
// releasing each smem stage with tcgen05.commit.  Warps 0-7 then drain TMEM
// (warp w reads lane quarter w%4, column half w/4), add bias, apply ReLU and
// store NCHW.  Split-K CTAs write partials to workspace; the last CTA of a
// tile (atomic ticket) reduces them in split order, so results are
// deterministic run to run.
#pragma once
#include "common.cuh"

namespace b2c {

constexpr int UMMA_M = 128;
constexpr int UMMA_BK = 32;  // fp32 elements of K per pipeline stage
constexpr int UMMA_PRODUCERS = 256;
constexpr int UMMA_THREADS = UMMA_PRODUCERS + 32;
constexpr int UMMA_SMEM_HDR = 1024;  // barriers + TMEM slot + flags

template <int BN>
struct UmmaCfg {
    static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "BN: multiple of 32 in [32, 256]");
    static constexpr int ROWS = UMMA_M + BN;
    static constexpr int STAGE_BYTES = ROWS * UMMA_BK * 4 * 2;  // hi + lo
    static constexpr int BUDGET = 220 * 1024 - UMMA_SMEM_HDR;
    static constexpr int STAGES = (BUDGET / STAGE_BYTES) > 6 ? 6 : (BUDGET / STAGE_BYTES);
    static constexpr int SMEM = UMMA_SMEM_HDR + STAGES * STAGE_BYTES;
    static constexpr int TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
    static constexpr int NROWS = (ROWS + UMMA_PRODUCERS - 1) / UMMA_PRODUCERS;
    static_assert(STAGES >= 2, "need at least two stages");
};

struct UmmaArgs {
    Geom g;
    const float* x;
    const float* w;
    const float* bias;
    float* y;
    float* ws;    // split-K partials [tiles][split][BN][128]
    int* sems;    // split-K tickets [tiles], zero at rest
    int split;    // number of K splits (gridDim.z)
    int kps;      // K blocks per split
    int kblocks;  // ceil(K / 32)
};

// Which source an operand row reads.
struct RowState {
    const float* base;  // pixel: x + b*C*HW + iy0*W + ix0 ; filter: w + oc*K ; flat: x + b*K
    int iy0, ix0;
    bool valid;
};

template <int KMODE>
__device__ __forceinline__ void load_pixel_row(const Geom& g, const RowState& rs, int k0, float (&v)[32]) {
    if (KMODE == 2) {  // fc: the whole image is one flat K-long row
        if ((g.K & 3) == 0) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const int k = k0 + 4 * c;
                float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
                if (rs.valid && k < g.K) q = __ldg(reinterpret_cast<const float4*>(rs.base + k));
                v[4 * c] = q.x; v[4 * c + 1] = q.y; v[4 * c + 2] = q.z; v[4 * c + 3] = q.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = (rs.valid && k0 + j < g.K) ? __ldg(rs.base + k0 + j) : 0.0f;
        }
    } else if (KMODE == 1) {  // 1x1: k is the input channel
#pragma unroll
        for (int j = 0; j < 32; ++j)
            v[j] = (rs.valid && k0 + j < g.K) ? __ldg(rs.base + (long long)(k0 + j) * g.HW) : 0.0f;
    } else {  // k x k window: walk (ic, ky, kx) incrementally from k0
        uint32_t ic, rem, ky, kx;
        g.fRR.divmod((uint32_t)k0, ic, rem);
        g.fR.divmod(rem, ky, kx);
        int koff = (int)ic * g.HW + (int)ky * g.W + (int)kx;
        int iky = (int)ky, ikx = (int)kx;
        const int wrap_x = g.W - g.R, wrap_y = g.HW - g.R * g.W;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const int iy = rs.iy0 + iky, ix = rs.ix0 + ikx;
            const bool ok =
                rs.valid && (k0 + j < g.K) && (unsigned)iy < (unsigned)g.H && (unsigned)ix < (unsigned)g.W;
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

__device__ __forceinline__ void load_filter_row(const Geom& g, const RowState& rs, int k0, float (&v)[32]) {
    if ((g.K & 3) == 0) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int k = k0 + 4 * c;
            float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
            if (rs.valid && k < g.K) q = __ldg(reinterpret_cast<const float4*>(rs.base + k));
            v[4 * c] = q.x; v[4 * c + 1] = q.y; v[4 * c + 2] = q.z; v[4 * c + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = (rs.valid && k0 + j < g.K) ? __ldg(rs.base + k0 + j) : 0.0f;
    }
}

// Store one operand row's 32 K values as hi/lo 16-byte chunks.
__device__ __forceinline__ void store_row_split(uint32_t hi_row, uint32_t lo_row, const float (&v)[32]) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        float h0, h1, h2, h3, l0, l1, l2, l3;
        split_tf32(v[4 * c + 0], h0, l0);
        split_tf32(v[4 * c + 1], h1, l1);
        split_tf32(v[4 * c + 2], h2, l2);
        split_tf32(v[4 * c + 3], h3, l3);
        sts128(hi_row + c * 128, h0, h1, h2, h3);
        sts128(lo_row + c * 128, l0, l1, l2, l3);
    }
}

__device__ __forceinline__ uint32_t row_offset(int i) { return (uint32_t)((i >> 3) * 1024 + (i & 7) * 16); }

template <int BN, bool SWAP, int KMODE>
__global__ void __launch_bounds__(UMMA_THREADS, 1) k_umma(UmmaArgs a) {
    using Cfg = UmmaCfg<BN>;
    constexpr int STAGES = Cfg::STAGES;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty_bar = full_bar + STAGES;
    uint64_t* done_bar = empty_bar + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done_bar + 1);
    int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);
    uint8_t* tiles = smem + UMMA_SMEM_HDR;

    const Geom& g = a.g;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;

    // Tile coordinates: pixel tile along x, out_chan tile along y, K split along z.
    constexpr int PIX_TILE = SWAP ? BN : UMMA_M;
    constexpr int OC_TILE = SWAP ? UMMA_M : BN;
    const int m0 = blockIdx.x * PIX_TILE;
    const int n0 = blockIdx.y * OC_TILE;
    const int z = blockIdx.z;
    const int kb_begin = z * a.kps;
    const int kb_end = min(a.kblocks, kb_begin + a.kps);
    const int nkb = kb_end - kb_begin;

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&full_bar[s]), UMMA_PRODUCERS);
            mbar_init(smem_u32(&empty_bar[s]), 1);
        }
        mbar_init(smem_u32(done_bar), 1);
        mbar_fence_init();
    }
    if (warp == 8) tmem_alloc(smem_u32(tmem_slot), Cfg::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp < 8) {
        // ------------------------------------------------------------ producers
        RowState rs[Cfg::NROWS];
        bool is_pixel[Cfg::NROWS];
        uint32_t row_hi[Cfg::NROWS], row_lo[Cfg::NROWS];
#pragma unroll
        for (int q = 0; q < Cfg::NROWS; ++q) {
            const int r = tid + q * UMMA_PRODUCERS;
            const bool in_a = r < UMMA_M;
            const int i = in_a ? r : r - UMMA_M;  // row within its operand
            const bool exists = r < Cfg::ROWS;
            // A region: [hi 128 rows][lo 128 rows]; B region follows.
            const uint32_t reg_hi = in_a ? 0u : (uint32_t)(2 * UMMA_M * 128);
            const uint32_t reg_lo = reg_hi + (uint32_t)((in_a ? UMMA_M : BN) * 128);
            row_hi[q] = reg_hi + row_offset(i);
            row_lo[q] = reg_lo + row_offset(i);
            const bool pix = (in_a != SWAP);  // A rows are pixels unless swapped
            is_pixel[q] = pix;
            RowState s;
            s.iy0 = 0;
            s.ix0 = 0;
            s.valid = false;
            s.base = a.x;
            if (exists) {
                if (pix) {
                    const int m = m0 + i;
                    if (m < g.M) {
                        uint32_t b, p, oy, ox;
                        g.fPQ.divmod((uint32_t)m, b, p);
                        g.fOW.divmod(p, oy, ox);
                        s.iy0 = (int)oy * g.S - g.P;
                        s.ix0 = (int)ox * g.S - g.P;
                        s.valid = true;
                        if (KMODE == 2)
                            s.base = a.x + (long long)b * g.K;
                        else
                            s.base = a.x + (long long)b * g.C * g.HW + (long long)s.iy0 * g.W + s.ix0;
                    }
                } else {
                    const int oc = n0 + i;
                    if (oc < g.OC) {
                        s.valid = true;
                        s.base = a.w + (long long)oc * g.K;
                    }
                }
            }
            rs[q] = s;
        }
        const uint32_t tiles_u32 = smem_u32(tiles);
        for (int it = 0; it < nkb; ++it) {
            const int stage = it % STAGES;
            const uint32_t phase = (uint32_t)(it / STAGES) & 1u;
            mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1u);
            const int k0 = (kb_begin + it) * UMMA_BK;
            const uint32_t sbase = tiles_u32 + (uint32_t)(stage * Cfg::STAGE_BYTES);
#pragma unroll
            for (int q = 0; q < Cfg::NROWS; ++q) {
                if (tid + q * UMMA_PRODUCERS < Cfg::ROWS) {
                    float v[32];
                    if (is_pixel[q])
                        load_pixel_row<KMODE>(g, rs[q], k0, v);
                    else
                        load_filter_row(g, rs[q], k0, v);
                    store_row_split(sbase + row_hi[q], sbase + row_lo[q], v);
                }
            }
            fence_proxy_async_smem();
            mbar_arrive(smem_u32(&full_bar[stage]));
        }
    } else {
      if (lane == 0) {
        // ------------------------------------------------------------ MMA issuer
        constexpr uint32_t idesc = umma_idesc(2, UMMA_M, BN);
        const uint32_t tiles_u32 = smem_u32(tiles);
        for (int it = 0; it < nkb; ++it) {
            const int stage = it % STAGES;
            const uint32_t phase = (uint32_t)(it / STAGES) & 1u;
            mbar_wait(smem_u32(&full_bar[stage]), phase);
            tc_fence_after();
            const uint32_t a_hi = tiles_u32 + (uint32_t)(stage * Cfg::STAGE_BYTES);
            const uint32_t a_lo = a_hi + UMMA_M * 128;
            const uint32_t b_hi = a_lo + UMMA_M * 128;
            const uint32_t b_lo = b_hi + BN * 128;
#pragma unroll
            for (int s = 0; s < UMMA_BK / 8; ++s) {
                const uint32_t off = (uint32_t)s * 256u;
                const uint64_t dah = umma_desc(a_hi + off, 128, 1024);
                const uint64_t dal = umma_desc(a_lo + off, 128, 1024);
                const uint64_t dbh = umma_desc(b_hi + off, 128, 1024);
                const uint64_t dbl = umma_desc(b_lo + off, 128, 1024);
                mma_tf32(tmem_base, dah, dbh, idesc, (it > 0 || s > 0) ? 1u : 0u);
                mma_tf32(tmem_base, dah, dbl, idesc, 1u);
                mma_tf32(tmem_base, dal, dbh, idesc, 1u);
            }
            tc_commit(smem_u32(&empty_bar[stage]));
        }
        tc_commit(smem_u32(done_bar));
      }
      __syncwarp();
    }

    if (warp < 8) {
        // ------------------------------------------------------------ epilogue
        mbar_wait(smem_u32(done_bar), 0);
        tc_fence_after();
        const int quarter = warp & 3, half = warp >> 2;
        const int row = quarter * 32 + lane;  // TMEM lane = MMA M row
        const uint32_t t_row = tmem_base + ((uint32_t)(quarter * 32) << 16);
        constexpr int HALF_COLS = BN / 2;
        const int c_begin = half * HALF_COLS;

        // Per-row destination (row is a pixel unless SWAP).
        long long row_out = 0;  // !SWAP: b*OC*PQ + p ; SWAP: oc
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

        auto emit = [&](int col, float acc) {
            if (!SWAP) {
                const int oc = n0 + col;
                if (row_ok && oc < g.OC)
                    a.y[row_out + (long long)oc * g.PQ] = apply_act(acc + __ldg(a.bias + oc), g.act);
            } else {
                const int m = m0 + col;
                if (row_ok && m < g.M) {
                    uint32_t b, p;
                    g.fPQ.divmod((uint32_t)m, b, p);
                    a.y[((long long)b * g.OC + row_out) * g.PQ + p] = apply_act(acc + row_bias, g.act);
                }
            }
        };

        if (a.split == 1) {
#pragma unroll 1
            for (int c0 = c_begin; c0 < c_begin + HALF_COLS; c0 += 16) {
                float v[16];
                tmem_ld16(t_row + (uint32_t)c0, v);
#pragma unroll
                for (int j = 0; j < 16; ++j) emit(c0 + j, v[j]);
            }
        } else {
            const int tile = blockIdx.y * gridDim.x + blockIdx.x;
            float* part = a.ws + ((size_t)tile * a.split + z) * BN * UMMA_M;
#pragma unroll 1
            for (int c0 = c_begin; c0 < c_begin + HALF_COLS; c0 += 16) {
                float v[16];
                tmem_ld16(t_row + (uint32_t)c0, v);
#pragma unroll
                for (int j = 0; j < 16; ++j) __stcg(part + (size_t)(c0 + j) * UMMA_M + row, v[j]);
            }
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
                for (int c = c_begin; c < c_begin + HALF_COLS; ++c) {
                    float s = 0.f;
                    for (int zz = 0; zz < a.split; ++zz) s += __ldcg(base + ((size_t)zz * BN + c) * UMMA_M + row);
                    emit(c, s);
                }
                if (tid == 0) a.sems[tile] = 0;
            }
        }
        tc_fence_before();
    }
    __syncthreads();
    if (warp == 8) {
        tc_fence_after();
        tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
    }
}

}  // namespace b2c
