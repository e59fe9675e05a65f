// k_fcs.cuh — conv_fc_stream: fp32 FFMA weight-streaming kernel for the
// whole-image-filter convs (AlexNet fc6 / fc7, ConvFC, cuclgen/variants.py:328-373)
// at small batch (N <= 8).
//
// At N <= 8 these ops are HBM-bound (fc6: 151 MB of weights for 2*N*37.7M
// FLOP, arithmetic intensity <= 4 FLOP/B against a ridge of ~40 for FFMA):
// the job is to stream w from HBM once at full bandwidth.  Each block takes R
// consecutive out_chan rows; its W warps split K in 512-byte (32 lanes x
// float4) chunks, interleaved so that a warp's lanes read one contiguous 512 B
// segment per row per step (fully coalesced, 16-byte loads marked
// L1::no_allocate: weights are read once).  The image rows x[n][K] are reused
// by every block and stay L1/L2 resident.  Every lane accumulates R x NB fp32
// partial sums; the warp reduces them with a fixed shuffle tree and the block
// sums the W warp partials in warp order, so results are deterministic.
// Bias is added last, ReLU as the reference writes it (variants.py:164).
#pragma once
#include "common.cuh"

namespace b2c {

__device__ __forceinline__ float4 ld_stream4(const float4* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}

template <int NB, int R>
__global__ void __launch_bounds__(256) k_fc_stream(const float* __restrict__ x, const float* __restrict__ w,
                                                   const float* __restrict__ bias, float* __restrict__ y, int N,
                                                   int OC, int K, int act) {
    extern __shared__ float red[];  // [W][R][NB]
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int oc0 = blockIdx.x * R;
    const int K4 = K >> 2;
    const float4* wr[R];
#pragma unroll
    for (int r = 0; r < R; ++r) wr[r] = reinterpret_cast<const float4*>(w + (size_t)min(oc0 + r, OC - 1) * K);
    const float4* x4 = reinterpret_cast<const float4*>(x);
    float acc[R][NB];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int n = 0; n < NB; ++n) acc[r][n] = 0.0f;
    const int step = nw * 32;
#pragma unroll 2
    for (int k = warp * 32 + lane; k < K4; k += step) {
        float4 wv[R];
#pragma unroll
        for (int r = 0; r < R; ++r) wv[r] = ld_stream4(wr[r] + k);
#pragma unroll
        for (int n = 0; n < NB; ++n) {
            if (n < N) {
                const float4 xv = __ldg(x4 + (size_t)n * K4 + k);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    float s = acc[r][n];
                    s = fmaf(wv[r].x, xv.x, s);
                    s = fmaf(wv[r].y, xv.y, s);
                    s = fmaf(wv[r].z, xv.z, s);
                    s = fmaf(wv[r].w, xv.w, s);
                    acc[r][n] = s;
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int n = 0; n < NB; ++n) {
            float v = acc[r][n];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
            if (lane == 0) red[(warp * R + r) * NB + n] = v;
        }
    __syncthreads();
    for (int t = threadIdx.x; t < R * NB; t += blockDim.x) {
        const int r = t / NB, n = t - (t / NB) * NB, oc = oc0 + r;
        if (n >= N || oc >= OC) continue;
        float s = 0.0f;
        for (int j = 0; j < nw; ++j) s += red[(j * R + r) * NB + n];
        y[(size_t)n * OC + oc] = apply_act(s + __ldg(bias + oc), act);
    }
}

// Kb = 2 form (batch <= 32): the image rows x[:, k0:k0+256] are staged in shared
// memory (cp.async, double-buffered) once per block, so x costs one L2 read per
// block instead of one per weight row; each warp owns RPW whole out_chan rows
// (no cross-warp reduction) and streams their weights 512 B per lane-step.
// Every lane accumulates RPW x NB sums over its strided K subset; a fixed
// shuffle tree finishes each row (deterministic).
constexpr int FCS_KC = 256;  // floats of K per staged chunk

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int NB, int RPW>
__global__ void __launch_bounds__(256) k_fc_smem(const float* __restrict__ x, const float* __restrict__ w,
                                                 const float* __restrict__ bias, float* __restrict__ y, int N, int OC,
                                                 int K, int act) {
    extern __shared__ __align__(16) float4 xs[];  // [2][NB][FCS_KC / 4]
    constexpr int C4 = FCS_KC / 4;                 // float4 per image row per chunk
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int K4 = K >> 2;
    const int nchunks = (K4 + C4 - 1) / C4;
    const int oc0 = (blockIdx.x * nw + warp) * RPW;
    const float4* wr[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r) wr[r] = reinterpret_cast<const float4*>(w + (size_t)min(oc0 + r, OC - 1) * K);
    const float4* x4 = reinterpret_cast<const float4*>(x);
    auto stage = [&](int c, int buf) {
        for (int i = threadIdx.x; i < N * C4; i += blockDim.x) {
            const int n = i / C4, q = i - (i / C4) * C4;
            const int k4 = c * C4 + q;
            const bool in = k4 < K4;
            cp_async16(smem_u32(&xs[(buf * NB + n) * C4 + q]), x4 + (size_t)n * K4 + (in ? k4 : 0), in ? 16 : 0);
        }
        cp_async_commit();
    };
    float acc[RPW][NB];
#pragma unroll
    for (int r = 0; r < RPW; ++r)
#pragma unroll
        for (int n = 0; n < NB; ++n) acc[r][n] = 0.0f;
    stage(0, 0);
    for (int c = 0; c < nchunks; ++c) {
        const int buf = c & 1;
        if (c + 1 < nchunks) {
            stage(c + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < C4 / 32; ++j) {
            const int q = lane + 32 * j, k4 = c * C4 + q;
            if (k4 >= K4) break;
            float4 wv[RPW];
#pragma unroll
            for (int r = 0; r < RPW; ++r) wv[r] = ld_stream4(wr[r] + k4);
#pragma unroll
            for (int n = 0; n < NB; ++n) {
                if (n < N) {
                    const float4 xv = xs[(buf * NB + n) * C4 + q];
#pragma unroll
                    for (int r = 0; r < RPW; ++r) {
                        float s = acc[r][n];
                        s = fmaf(wv[r].x, xv.x, s);
                        s = fmaf(wv[r].y, xv.y, s);
                        s = fmaf(wv[r].z, xv.z, s);
                        s = fmaf(wv[r].w, xv.w, s);
                        acc[r][n] = s;
                    }
                }
            }
        }
        __syncthreads();  // this buffer is refilled by the stage() of chunk c + 2
    }
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
        const int oc = oc0 + r;
#pragma unroll
        for (int n = 0; n < NB; ++n) {
            float v = acc[r][n];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
            if (lane == 0 && n < N && oc < OC) y[(size_t)n * OC + oc] = apply_act(v + __ldg(bias + oc), act);
        }
    }
}

// Kb = 3 form (batch <= 8): the weight rows are streamed by the TMA engine
// (cp.async.bulk, one 2 KB copy per row per K chunk) into a deep shared-memory
// ring, so each SM keeps ~150 KB of weights in flight -- the op is bound by HBM
// latency x bytes in flight, which the register-staged loads of Kb = 1 / 2
// cannot reach.  One CTA per SM owns a block of rpc <= 32 consecutive out_chan
// rows (rows warp, warp + 8, ...: at most 4 per compute warp); a stage is the
// block's rows and the N image rows over one 512-float K chunk, both read from
// shared memory by the 8 compute warps (lane = float4 column, conflict-free).
// A producer warp issues the copies; per-stage full / empty mbarriers.  Every
// lane accumulates its rows x N sums over its K columns; a fixed shuffle tree
// finishes each (deterministic).
constexpr int FCB_KC = 512;     // floats of K per stage
constexpr int FCB_WARPS = 8;    // compute warps (+1 producer warp)
constexpr int FCB_MAX_RPW = 4;  // rows per compute warp: rpc <= 32
constexpr int FCB_HDR = 128;    // barriers

template <int NB>
__global__ void __launch_bounds__(32 * (FCB_WARPS + 1), 1)
    k_fc_bulk(const float* __restrict__ x, const float* __restrict__ w, const float* __restrict__ bias,
              float* __restrict__ y, int N, int OC, int K, int act, int rpc, int nst) {
    extern __shared__ __align__(128) uint8_t fsm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(fsm);
    uint64_t* empty = full + nst;
    float* stg = reinterpret_cast<float*>(fsm + FCB_HDR);
    const int stage_floats = (rpc + N) * FCB_KC;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nchunks = (K + FCB_KC - 1) / FCB_KC;
    const int nblocks = (OC + rpc - 1) / rpc;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&empty[s]), FCB_WARPS);
        }
        mbar_fence_init();
    }
    __syncthreads();
    if (warp == FCB_WARPS) {  // producer
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int rb = blockIdx.x; rb < nblocks; rb += gridDim.x) {
                const int r0 = rb * rpc, nr = min(rpc, OC - r0);
                for (int c = 0; c < nchunks; ++c) {
                    mbar_wait(smem_u32(&empty[s]), ph ^ 1u);
                    const int k0 = c * FCB_KC;
                    const uint32_t bytes = (uint32_t)min(FCB_KC, K - k0) * 4u;
                    const uint32_t bar = smem_u32(&full[s]);
                    mbar_arrive_expect_tx(bar, bytes * (uint32_t)(nr + N));
                    float* base = stg + (size_t)s * stage_floats;
                    for (int r = 0; r < nr; ++r)
                        bulk_g2s(smem_u32(base + r * FCB_KC), w + (size_t)(r0 + r) * K + k0, bytes, bar);
                    for (int n = 0; n < N; ++n)
                        bulk_g2s(smem_u32(base + (rpc + n) * FCB_KC), x + (size_t)n * K + k0, bytes, bar);
                    if (++s == nst) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            }
        }
        return;
    }
    int s = 0;
    uint32_t ph = 0;
    for (int rb = blockIdx.x; rb < nblocks; rb += gridDim.x) {
        const int r0 = rb * rpc, nr = min(rpc, OC - r0);
        float acc[FCB_MAX_RPW][NB];
#pragma unroll
        for (int j = 0; j < FCB_MAX_RPW; ++j)
#pragma unroll
            for (int n = 0; n < NB; ++n) acc[j][n] = 0.0f;
        for (int c = 0; c < nchunks; ++c) {
            mbar_wait(smem_u32(&full[s]), ph);
            const float4* base = reinterpret_cast<const float4*>(stg + (size_t)s * stage_floats);
            const int kl4 = min(FCB_KC, K - c * FCB_KC) >> 2;
#pragma unroll
            for (int i = 0; i < FCB_KC / 128; ++i) {
                const int q = lane + 32 * i;
                if (q >= kl4) break;
                float4 xv[NB];
#pragma unroll
                for (int n = 0; n < NB; ++n)
                    if (n < N) xv[n] = base[(rpc + n) * (FCB_KC / 4) + q];
#pragma unroll
                for (int j = 0; j < FCB_MAX_RPW; ++j) {
                    const int r = warp + FCB_WARPS * j;
                    if (r < nr) {
                        const float4 wv = base[r * (FCB_KC / 4) + q];
#pragma unroll
                        for (int n = 0; n < NB; ++n) {
                            if (n < N) {
                                float a = acc[j][n];
                                a = fmaf(wv.x, xv[n].x, a);
                                a = fmaf(wv.y, xv[n].y, a);
                                a = fmaf(wv.z, xv[n].z, a);
                                a = fmaf(wv.w, xv[n].w, a);
                                acc[j][n] = a;
                            }
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&empty[s]));
            if (++s == nst) {
                s = 0;
                ph ^= 1u;
            }
        }
#pragma unroll
        for (int j = 0; j < FCB_MAX_RPW; ++j) {
            const int r = warp + FCB_WARPS * j;
#pragma unroll
            for (int n = 0; n < NB; ++n) {
                float v = acc[j][n];
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                if (lane == 0 && r < nr && n < N) y[(size_t)n * OC + r0 + r] = apply_act(v + __ldg(bias + r0 + r), act);
            }
        }
    }
}

}  // namespace b2c
