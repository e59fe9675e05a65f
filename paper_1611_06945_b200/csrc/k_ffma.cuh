// CUDA-core (FFMA) convolution kernels: exact fp32, every shape.
//
//  * k_simple  — "conv_simple" (cuclgen/variants.py:223-276): one thread per
//    output, acc = bias[oc], then fmaf over ic -> ky -> kx with zero padding.
//    It is the exact-order device reference the autotuner cross-checks every
//    candidate against (the role oracle.compare plays in tuner._evaluate,
//    tuner.py:311-320).
//  * k_tiled   — "conv_tiled" (variants.py:376-685): register/thread-blocked
//    implicit GEMM, M = img*oy*ox, N = out_chan, K = in_chan*ksz*ksz, with the
//    reference's TuneParams meaning: MNt = per-thread register block, MNb =
//    thread block, Kb = reduction chunk staged in shared memory.  Each output
//    accumulates the same fmaf sequence as k_simple (bias first, k ascending),
//    so tiled == simple bit-for-bit for any tile shape — the B200 form of the
//    reference's "degenerate tiled == simple" property (tests/test_variants.py:173-179).
//    Unlike the reference it reads canonical NCHW/OIHW and writes NCHW
//    directly (no required_formats conversions, variants.py:416-424).
#pragma once
#include "common.cuh"

namespace b2c {

__global__ void __launch_bounds__(256) k_simple(Geom g, const float* __restrict__ x,
                                                const float* __restrict__ w,
                                                const float* __restrict__ bias, float* __restrict__ y) {
    const long long total = (long long)g.N * g.OC * g.PQ;
    for (long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x; gid < total;
         gid += (long long)gridDim.x * blockDim.x) {
        const long long t = gid / g.PQ;
        const int p = (int)(gid - t * g.PQ);
        const int oc = (int)(t % g.OC);
        const int b = (int)(t / g.OC);
        const int oy = p / g.OW, ox = p - (p / g.OW) * g.OW;
        const int iy0 = oy * g.S - g.P, ix0 = ox * g.S - g.P;
        const float* xb = x + (long long)b * g.C * g.HW;
        const float* wp = w + (long long)oc * g.K;
        float acc = bias[oc];
        for (int ic = 0; ic < g.C; ++ic) {
            for (int ky = 0; ky < g.R; ++ky) {
                const int iy = iy0 + ky;
                const bool yok = (unsigned)iy < (unsigned)g.H;
                for (int kx = 0; kx < g.R; ++kx) {
                    const int ix = ix0 + kx;
                    const float v = (yok && (unsigned)ix < (unsigned)g.W) ? __ldg(xb + ic * g.HW + iy * g.W + ix) : 0.0f;
                    acc = fmaf(v, __ldg(wp + (ic * g.R + ky) * g.R + kx), acc);
                }
            }
        }
        y[gid] = apply_act(acc, g.act);
    }
}

// Dynamic smem layout of k_tiled:
//   As   [KB][BM]  im2col tile (k-major rows, pixels contiguous)
//   Bs   [KB][BN]  filter tile
//   pix  [BM] int4 {x offset of (b, iy0, ix0), iy0, ix0, valid}
//   ktab [KB] int4 {ic*HW + ky*W + kx, ky, kx, valid}
__host__ __device__ inline int tiled_tab_offset(int BM, int BN, int KB) {  // in floats, 16-byte aligned
    return (KB * (BM + BN) + 3) & ~3;
}
__host__ __device__ inline size_t tiled_smem_bytes(int BM, int BN, int KB) {
    return (size_t)tiled_tab_offset(BM, BN, KB) * 4 + (size_t)BM * 16 + (size_t)KB * 16;
}

template <int MT, int NT>
__global__ void __launch_bounds__(1024) k_tiled(Geom g, const float* __restrict__ x,
                                                const float* __restrict__ w,
                                                const float* __restrict__ bias, float* __restrict__ y,
                                                int MB, int NB, int KB) {
    extern __shared__ __align__(16) float smf[];
    const int BM = MB * MT, BN = NB * NT;
    float* As = smf;
    float* Bs = smf + KB * BM;
    int4* pix = reinterpret_cast<int4*>(smf + tiled_tab_offset(BM, BN, KB));
    int4* ktab = pix + BM;

    const int tid = threadIdx.x;
    const int nthr = MB * NB;
    // Strided register blocks: thread (tm, tn) owns pixels tm + i*MB and channels
    // tn + j*NB, so a warp's As reads and NCHW stores are unit-stride.
    const int tm = tid % MB, tn = tid / MB;
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;

    for (int i = tid; i < BM; i += nthr) {
        const int m = m0 + i;
        int4 e = make_int4(0, 0, 0, 0);
        if (m < g.M) {
            uint32_t b, p, oy, ox;
            g.fPQ.divmod((uint32_t)m, b, p);
            g.fOW.divmod(p, oy, ox);
            const int iy0 = (int)oy * g.S - g.P, ix0 = (int)ox * g.S - g.P;
            e = make_int4((int)b * g.C * g.HW + iy0 * g.W + ix0, iy0, ix0, 1);
        }
        pix[i] = e;
    }

    float acc[MT][NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) {
        const int n = n0 + tn + j * NB;
        const float bj = (n < g.OC) ? __ldg(bias + n) : 0.0f;
#pragma unroll
        for (int i = 0; i < MT; ++i) acc[i][j] = bj;
    }

    for (int k0 = 0; k0 < g.K; k0 += KB) {
        for (int i = tid; i < KB; i += nthr) {
            const int k = k0 + i;
            int4 e = make_int4(0, 0, 0, 0);
            if (k < g.K) {
                uint32_t ic, rem, ky, kx;
                g.fRR.divmod((uint32_t)k, ic, rem);
                g.fR.divmod(rem, ky, kx);
                e = make_int4((int)ic * g.HW + (int)ky * g.W + (int)kx, (int)ky, (int)kx, 1);
            }
            ktab[i] = e;
        }
        __syncthreads();  // ktab ready; previous chunk's reads of As/Bs done
        for (int e = tid; e < KB * BM; e += nthr) {
            const int kk = e / BM, mm = e - (e / BM) * BM;
            const int4 pe = pix[mm];
            const int4 ke = ktab[kk];
            const int iy = pe.y + ke.y, ix = pe.z + ke.z;
            float v = 0.0f;
            if (pe.w & ke.w && (unsigned)iy < (unsigned)g.H && (unsigned)ix < (unsigned)g.W)
                v = __ldg(x + pe.x + ke.x);
            As[kk * BM + mm] = v;
        }
        for (int e = tid; e < KB * BN; e += nthr) {
            const int nn = e / KB, kk = e - (e / KB) * KB;
            const int n = n0 + nn, k = k0 + kk;
            Bs[kk * BN + nn] = (n < g.OC && k < g.K) ? __ldg(w + (long long)n * g.K + k) : 0.0f;
        }
        __syncthreads();
        const int kend = min(KB, g.K - k0);
        for (int kk = 0; kk < kend; ++kk) {
            float a[MT], bv[NT];
#pragma unroll
            for (int i = 0; i < MT; ++i) a[i] = As[kk * BM + tm + i * MB];
#pragma unroll
            for (int j = 0; j < NT; ++j) bv[j] = Bs[kk * BN + tn + j * NB];
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) acc[i][j] = fmaf(a[i], bv[j], acc[i][j]);
        }
    }

#pragma unroll
    for (int i = 0; i < MT; ++i) {
        const int m = m0 + tm + i * MB;
        if (m >= g.M) continue;
        uint32_t b, p;
        g.fPQ.divmod((uint32_t)m, b, p);
        float* yb = y + (long long)b * g.OC * g.PQ + p;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            const int n = n0 + tn + j * NB;
            if (n < g.OC) yb[(long long)n * g.PQ] = apply_act(acc[i][j], g.act);
        }
    }
}

}  // namespace b2c
