// tcgen05.mma.kind::tf32 issue-rate probe (B200): cycles per MMA for M = 128,
// N in {32..256}, A from TMEM (TS) or shared memory (SS), B from shared memory,
// back-to-back into one accumulator (the conv kernel's pattern) or
// alternating between two accumulators.  One CTA per SM, all SMs busy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_probe tools/mma_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#include "../paper_1611_06945_b200/csrc/common.cuh"

using namespace b2c;

template <int N, bool TS, int NACC>
__global__ void __launch_bounds__(128, 1) probe(int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
    // zero the operand images (finite data)
    for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) sts128(base + i * 16, 0.f, 0.f, 0.f, 0.f);
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar), 1);
        mbar_fence_init();
    }
    if (warp == 0) tmem_alloc(smem_u32(&slot), 512);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc = umma_idesc(2, 128, N);
        const uint32_t a_s = base, b_s = base + 16384;
        const uint32_t a_t = tmem + 448;  // A in TMEM: 32 columns at 448
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint32_t d = tmem + (uint32_t)((i % NACC) * (N > 128 ? 0 : 128));
            const int s = i & 3;
            const uint64_t db = umma_desc_sw128(b_s + s * 32);
            if (TS) {
                mma_tf32_ts(d, a_t + 8 * s, db, idesc, 1u);
            } else {
                mma_tf32(d, umma_desc_sw128(a_s + s * 32), db, idesc, 1u);
            }
        }
        tc_commit(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), 0);
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}


// 2-SM UMMA (cta_group::2, M = 256): a cluster of two CTAs, the leader issues;
// A (128 rows per CTA) in each CTA's TMEM or smem, B split N/2 rows per CTA.
template <int N, bool TS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe2(int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    const uint32_t rank = cluster_ctarank();
    const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
    for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) sts128(base + i * 16, 0.f, 0.f, 0.f, 0.f);
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar), 1);
        mbar_fence_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = slot;
    long long t0 = clock64();
    if (threadIdx.x == 0 && rank == 0) {
        constexpr uint32_t idesc = umma_idesc(2, 256, N);
        const uint32_t a_s = base, b_s = base + 16384;
        const uint32_t a_t = tmem + 448;
        for (int i = 0; i < iters; ++i) {
            const int s = i & 3;
            const uint64_t db = umma_desc_sw128(b_s + s * 32);
            if (TS) {
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                             "r"(a_t + 8 * s), "l"(db), "r"(idesc), "r"(1u) : "memory");
            } else {
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                             "l"(umma_desc_sw128(a_s + s * 32)), "l"(db), "r"(idesc), "r"(1u) : "memory");
            }
        }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                     ::"r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
    }
    if (threadIdx.x == 0) {
        mbar_wait(smem_u32(&bar), 0);
        long long t1 = clock64();
        if (rank == 0) out[blockIdx.x / 2] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    }
}

template <int N, bool TS>
void run2(long long* d_out, int sms) {
    const int iters = 4096;
    auto k = probe2<N, TS>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    k<<<sms, 128, 80 * 1024>>>(iters, d_out);
    k<<<sms, 128, 80 * 1024>>>(iters, d_out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("pair N=%d error %s\n", N, cudaGetErrorString(e));
        return;
    }
    std::vector<long long> h(sms / 2);
    cudaMemcpy(h.data(), d_out, (sms / 2) * 8, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (auto v : h) mx = v > mx ? v : mx;
    const double cyc = (double)mx / iters;
    const double floor = N / 2.0;  // per SM: 128 x N x 8 FMA at 2048 FMA/clk
    printf("PAIR M=256 N=%3d %s: %6.1f cycles/MMA (per-SM floor %5.1f) -> %4.0f%% of tf32 peak\n", N,
           TS ? "A:TMEM" : "A:smem", cyc, floor, 100.0 * floor / cyc);
}

template <int N, bool TS, int NACC>
void run(long long* d_out, int sms) {
    const int iters = 4096;
    auto k = probe<N, TS, NACC>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    k<<<sms, 128, 80 * 1024>>>(iters, d_out);
    k<<<sms, 128, 80 * 1024>>>(iters, d_out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return;
    }
    std::vector<long long> h(sms);
    cudaMemcpy(h.data(), d_out, sms * 8, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (auto v : h) mx = v > mx ? v : mx;
    const double cyc = (double)mx / iters;
    const double floor = N / 2.0;
    printf("N=%3d %s acc=%d: %6.1f cycles/MMA (floor %5.1f) -> %4.0f%% of tf32 peak\n", N, TS ? "A:TMEM" : "A:smem",
           NACC, cyc, floor, 100.0 * floor / cyc);
}

int main() {
    long long* d_out;
    cudaMalloc(&d_out, 1024 * 8);
    int sms = 148;
    run<32, true, 1>(d_out, sms);
    run<64, true, 1>(d_out, sms);
    run<96, true, 1>(d_out, sms);
    run<128, true, 1>(d_out, sms);
    run<192, true, 1>(d_out, sms);
    run<256, true, 1>(d_out, sms);
    run<32, false, 1>(d_out, sms);
    run<64, false, 1>(d_out, sms);
    run<128, false, 1>(d_out, sms);
    run<256, false, 1>(d_out, sms);
    run<64, true, 2>(d_out, sms);
    run<128, true, 2>(d_out, sms);
    run2<64, true>(d_out, sms);
    run2<128, true>(d_out, sms);
    run2<192, true>(d_out, sms);
    run2<256, true>(d_out, sms);
    run2<128, false>(d_out, sms);
    run2<256, false>(d_out, sms);
    return 0;
}
