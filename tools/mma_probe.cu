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
    return 0;
}
