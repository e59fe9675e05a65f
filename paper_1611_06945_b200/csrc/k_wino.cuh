// Winograd F(2x2, 3x3) for the 3x3 / stride-1 convs of the sweep (conv_wino;
// the paper's stated gap to cuDNN).
//
// y = A^T [ (G g G^T) .* (B^T d B) ] A per 2x2 output tile, which for a whole
// layer is 16 independent GEMMs, one per position z = 4*xi + nu of the 4x4
// transformed tile:
//     M[z][p][oc] = sum_c V[z][p][c] * U[z][oc][c]
//   U = G g G^T      filters, once per filter tensor (b2c_conv_prepare)   [16][OC][C]
//   V = B^T d B      input tiles d (4x4, stride 2, zero padded)            [16][P][C]
//   y = A^T M A      + bias, ReLU (variants.py:160-165)                  NCHW
// with P = N * ceil(OH/2) * ceil(OW/2) tiles.  The GEMMs run on the tcgen05
// 3xTF32 kernel (k_tconv MODE 7: fp32-exact products of the fp32 U and V);
// the transforms are exact-coefficient fp32 adds (+-1, 1/2 for U computed in
// fp64), so the result is an fp32-accurate evaluation of the same sum in a
// different order.  2.25x fewer multiplies than direct conv (4 x 4 products per
// 2 x 2 outputs instead of 9 x 4), paid for with V / M traffic through L2/HBM.
#pragma once
#include "common.cuh"

namespace b2c {

constexpr int WINO_CB = 32;  // channels per transform block (one per lane)

// U[z][oc][c] = (G g G^T)[xi][nu], G = [[1,0,0],[1/2,1/2,1/2],[1/2,-1/2,1/2],[0,0,1]];
// one thread per (oc, c), computed in fp64 and rounded once.
__global__ void __launch_bounds__(256) k_wino_filter(const float* __restrict__ w, float* __restrict__ u, int OC,
                                                     int C) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)OC * C) return;
    const float* g = w + i * 9;  // OIHW: [oc][c][3][3]
    double t[4][3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const double g0 = g[j], g1 = g[3 + j], g2 = g[6 + j];
        t[0][j] = g0;
        t[1][j] = 0.5 * (g0 + g1 + g2);
        t[2][j] = 0.5 * (g0 - g1 + g2);
        t[3][j] = g2;
    }
    const size_t plane = (size_t)OC * C;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const double v[4] = {t[a][0], 0.5 * (t[a][0] + t[a][1] + t[a][2]), 0.5 * (t[a][0] - t[a][1] + t[a][2]), t[a][2]};
#pragma unroll
        for (int b = 0; b < 4; ++b) u[(size_t)(a * 4 + b) * plane + i] = (float)v[b];
    }
}

// V[z][p][c] = (B^T d B)[xi][nu], B^T = [[1,0,-1,0],[0,1,1,0],[0,-1,1,0],[0,1,0,-1]].
// Block = (tile row ty, 32-channel block, image n): the 4 input rows of the tile row are
// staged in shared memory (a warp per (channel, row) pair, lanes along x: coalesced, no
// index divisions); then lane = channel, so every V store of a warp is 128 contiguous bytes.
__global__ void __launch_bounds__(256) k_wino_input(const float* __restrict__ x, float* __restrict__ v, int C, int H,
                                                    int W, int pad, int tiles_y, int tiles_x, long long P) {
    extern __shared__ float wx_s[];  // [4 rows][WS cols][33]: channel innermost (+1 pad: conflict-free both ways)
    pdl_launch_dependents();
    pdl_wait();
    const int ty = blockIdx.x, c0 = blockIdx.y * WINO_CB, n = blockIdx.z;
    const int WS = 2 * tiles_x + 2;  // input columns of the tile row
    const int y0 = 2 * ty - pad, x0 = -pad;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int pr = wid; pr < WINO_CB * 4; pr += nw) {
        const int cc = pr >> 2, r = pr & 3;
        const int c = c0 + cc, iy = y0 + r;
        const bool rowok = c < C && (unsigned)iy < (unsigned)H;
        const float* src = x + (((size_t)n * C + (rowok ? c : 0)) * H + (rowok ? iy : 0)) * W;
        for (int col = lane; col < WS; col += 32) {
            const int ix = x0 + col;
            wx_s[(r * WS + col) * 33 + cc] = (rowok && (unsigned)ix < (unsigned)W) ? __ldg(src + ix) : 0.0f;
        }
    }
    __syncthreads();
    const int c = c0 + lane;
    if (c >= C) return;
    const size_t plane = (size_t)P * C;
    for (int tx = wid; tx < tiles_x; tx += nw) {
        float d[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int q = 0; q < 4; ++q) d[r][q] = wx_s[(r * WS + 2 * tx + q) * 33 + lane];
        float s[4][4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            s[0][q] = d[0][q] - d[2][q];
            s[1][q] = d[1][q] + d[2][q];
            s[2][q] = d[2][q] - d[1][q];
            s[3][q] = d[1][q] - d[3][q];
        }
        float* dst = v + (((long long)n * tiles_y + ty) * tiles_x + tx) * C + c;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const float o[4] = {s[a][0] - s[a][2], s[a][1] + s[a][2], s[a][2] - s[a][1], s[a][1] - s[a][3]};
#pragma unroll
            for (int b = 0; b < 4; ++b, dst += plane) *dst = o[b];
        }
    }
}

// y[n][oc][2ty+i][2tx+j] = act((A^T M A)[i][j] + bias[oc]), A^T = [[1,1,1,0],[0,1,-1,-1]].
// M is [16][P][OC] (OC_MAJOR = false: the swap_ab GEMM's coalesced store order) or
// [16][OC][P] (true: the pixels-on-M GEMM's).  Block = (tile row ty, 32-out-channel
// block, image n); loads run along the contiguous index (oc, or tx), the 2 output rows
// go through shared memory and leave coalesced along x.
template <bool OC_MAJOR>
__global__ void __launch_bounds__(256) k_wino_output(const float* __restrict__ m, const float* __restrict__ bias,
                                                     float* __restrict__ y, int OC, int OH, int OW, int tiles_y,
                                                     int tiles_x, long long P, int act) {
    extern __shared__ float wy_s[];  // [32 oc][2 rows][OS]
    pdl_launch_dependents();
    pdl_wait();
    const int ty = blockIdx.x, oc0 = blockIdx.y * WINO_CB, n = blockIdx.z;
    const int OS = 2 * tiles_x + 1;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const long long p0 = ((long long)n * tiles_y + ty) * tiles_x;
    const size_t plane = (size_t)P * OC;
    // work items (oc in block, tx): OC_MAJOR walks tx fastest (contiguous p), else oc fastest
    const int items = WINO_CB * tiles_x;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
        const int cc = OC_MAJOR ? it / tiles_x : (it & 31);
        const int tx = OC_MAJOR ? it - cc * tiles_x : (it >> 5);
        const int oc = oc0 + cc;
        if (oc >= OC) continue;
        const float* src = OC_MAJOR ? m + (size_t)oc * P + p0 + tx : m + (p0 + tx) * OC + oc;
        float q[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c) q[a][c] = __ldcs(src + (size_t)(a * 4 + c) * plane);
        float u[2][4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            u[0][c] = q[0][c] + q[1][c] + q[2][c];
            u[1][c] = q[1][c] - q[2][c] - q[3][c];
        }
        const float b = __ldg(bias + oc);
        float* row = wy_s + cc * 2 * OS;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            row[i * OS + 2 * tx] = apply_act(u[i][0] + u[i][1] + u[i][2] + b, act);
            row[i * OS + 2 * tx + 1] = apply_act(u[i][1] - u[i][2] - u[i][3] + b, act);
        }
    }
    __syncthreads();
    const int rows_out = min(2, OH - 2 * ty);
    for (int pr = wid; pr < WINO_CB * 2; pr += nw) {  // a warp per (out channel, row), lanes along x
        const int cc = pr >> 1, r = pr & 1, o = oc0 + cc;
        if (r >= rows_out || o >= OC) continue;
        float* dst = y + (((size_t)n * OC + o) * OH + 2 * ty + r) * OW;
        const float* srow = wy_s + cc * 2 * OS + r * OS;
        for (int xo = lane; xo < OW; xo += 32) dst[xo] = srow[xo];
    }
}

}  // namespace b2c
