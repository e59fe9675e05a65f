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

}  // namespace b2c
