// Semantics check of the 2-SM UMMA (tcgen05.mma.cta_group::2, M = 256) as the conv kernel uses it:
// A (128 rows per CTA, K = 8 tf32) from TMEM or smem, B (N/2 rows per CTA, K-major SWIZZLE_128B)
// from each CTA's smem at the same offset, D rows 0-127 / 128-255 in rank 0's / rank 1's TMEM.
// A[m][k] = (k == m % 8), B[n][k] = n * 8 + k  =>  D[m][n] = n * 8 + m % 8.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/pair_check tools/pair_check.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#include "../paper_1611_06945_b200/csrc/common.cuh"

using namespace b2c;

template <int N, bool TS, bool SPLITB>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) pair_check(int* bad, float* sample) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t rank = cluster_ctarank();
    const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
    const uint32_t a_s = base, b_s = base + 16384;
    // B rows this CTA holds: SPLITB -> N/2 rows (global n = rank*N/2 + r), else all N rows
    constexpr int BR = SPLITB ? N / 2 : N;
    for (int i = tid; i < 128 * 32; i += 128) {  // A image, SW128 K-major, 128 rows x 32 floats (only K 0-7 used)
        const int m = i / 32, k = i % 32;
        const float v = (k < 8 && k == m % 8) ? 1.f : 0.f;
        const int chunk = k / 4, e = k % 4;
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(a_s + m * 128 + ((chunk ^ (m & 7)) * 16) + e * 4), "f"(v));
    }
    for (int i = tid; i < BR * 32; i += 128) {
        const int r = i / 32, k = i % 32;
        const int n = (SPLITB ? (int)rank * (N / 2) : 0) + r;
        const float v = k < 8 ? (float)(n * 8 + k) : 0.f;
        const int chunk = k / 4, e = k % 4;
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(b_s + r * 128 + ((chunk ^ (r & 7)) * 16) + e * 4), "f"(v));
    }
    if (tid == 0) {
        mbar_init(smem_u32(&bar), 1);
        mbar_fence_init();
    }
    if (warp == 0) tmem_alloc_pair(smem_u32(&slot), 512);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (TS) {  // A row tid -> TMEM lane tid, columns 256..263
        float v[32];
        for (int k = 0; k < 32; ++k) v[k] = (k < 8 && k == tid % 8) ? 1.f : 0.f;
        tmem_st32(tmem + ((uint32_t)(warp * 32) << 16) + 256, v);
        tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    if (tid == 0 && rank == 0) {
        constexpr uint32_t idesc = umma_idesc(2, 256, N);
        const uint64_t db = umma_desc_sw128(b_s);
        if (TS)
            mma_tf32_ts_pair(tmem, tmem + 256, db, idesc, 0u);
        else
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                         "l"(umma_desc_sw128(a_s)), "l"(db), "r"(idesc), "r"(0u) : "memory");
        tc_commit_pair(smem_u32(&bar), (uint16_t)3);
    }
    mbar_wait(smem_u32(&bar), 0);
    tc_fence_after();
    const int m = (int)rank * 128 + tid;
    int nbad = 0;
    for (int c = 0; c < N; c += 8) {
        float v[8];
        tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
        for (int j = 0; j < 8; ++j) {
            const int n = c + j;
            const float want = (float)(n * 8 + m % 8);
            if (v[j] != want) ++nbad;
            if (tid < 4 && n < 4) sample[(rank * 4 + tid) * 4 + n] = v[j];
        }
    }
    atomicAdd(bad + rank, nbad);
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc_pair(tmem, 512);
    }
}

template <int N, bool TS, bool SPLITB>
void run() {
    int* bad;
    float* sample;
    cudaMalloc(&bad, 8);
    cudaMalloc(&sample, 32 * 4);
    cudaMemset(bad, 0, 8);
    cudaMemset(sample, 0, 128);
    auto k = pair_check<N, TS, SPLITB>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    k<<<2, 128, 80 * 1024>>>(bad, sample);
    cudaError_t e = cudaDeviceSynchronize();
    int hb[2] = {-1, -1};
    float hs[32];
    cudaMemcpy(hb, bad, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hs, sample, 128, cudaMemcpyDeviceToHost);
    printf("N=%3d A:%s B:%s  err=%s  bad rank0=%d rank1=%d (of %d each)\n", N, TS ? "TMEM" : "smem",
           SPLITB ? "half-per-CTA" : "full-per-CTA", cudaGetErrorString(e), hb[0], hb[1], 128 * N);
    for (int r = 0; r < 2; ++r)
        for (int t = 0; t < 2; ++t)
            printf("   rank%d row%d: D[.,0..3] = %g %g %g %g (want %d %d %d %d)\n", r, t, hs[(r * 4 + t) * 4],
                   hs[(r * 4 + t) * 4 + 1], hs[(r * 4 + t) * 4 + 2], hs[(r * 4 + t) * 4 + 3], t % 8, 8 + t % 8,
                   16 + t % 8, 24 + t % 8);
    cudaFree(bad);
    cudaFree(sample);
}

int main() {
    run<64, false, true>();
    run<64, true, true>();
    run<128, false, true>();
    run<128, true, true>();
    run<128, false, false>();
    run<128, true, false>();
    return 0;
}
