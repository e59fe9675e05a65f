// Probe (debug): does a 4-D tiled TMA load with negative start coordinates and a
// box larger than the tensor's channel extent complete, and what lands in smem?
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tma4d_probe tools/tma4d_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void k_probe(const __grid_constant__ CUtensorMap tm, float* out, int c0, int c1, int c2, int c3, int nbytes) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm);
    float* dst = reinterpret_cast<float*>(sm + 1024);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(nbytes));
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                     ::"r"(su32(dst)), "l"(&tm), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
        unsigned ok = 0;
        long long t0 = clock64();
        while (!ok && clock64() - t0 < (1ll << 28)) {
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                         : "=r"(ok) : "r"(su32(bar)));
        }
        out[0] = ok ? 1.f : -1.f;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nbytes / 4; i += blockDim.x) out[1 + i] = dst[i];
}

int main() {
    const int W = 28, H = 28, C = 32, N = 1, bx = 28, by = 4;
    std::vector<float> hx((size_t)N * C * H * W);
    for (size_t i = 0; i < hx.size(); ++i) hx[i] = (float)(i + 1);
    float *dx, *dout;
    cudaMalloc(&dx, hx.size() * 4);
    cudaMemcpy(dx, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice);
    const int nbytes = bx * by * 32 * 4;
    cudaMalloc(&dout, 4 + nbytes);
    CUtensorMap tm;
    cuuint64_t dims[4] = {W, H, C, N};
    cuuint64_t strides[3] = {W * 4ull, (cuuint64_t)H * W * 4, (cuuint64_t)C * H * W * 4};
    cuuint32_t box[4] = {bx, by, 32, 1}, es[4] = {1, 1, 1, 1};
    cuInit(0);
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, dx, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc=%d\n", (int)r);
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 + nbytes);
    int coords[6][4] = {{0, 0, 0, 0}, {-4, 0, 0, 0}, {0, -1, 0, 0}, {-4, -2, 0, 0}, {4, 26, 0, 0}, {-1, -1, 0, 0}};
    for (auto& c : coords) {
        k_probe<<<1, 128, 1024 + nbytes>>>(tm, dout, c[0], c[1], c[2], c[3], nbytes);
        cudaError_t e = cudaDeviceSynchronize();
        float h[8];
        cudaMemcpy(h, dout, sizeof(h), cudaMemcpyDeviceToHost);
        printf("coords (%d,%d,%d,%d): %s done=%g first=%g %g %g\n", c[0], c[1], c[2], c[3], cudaGetErrorString(e), h[0], h[1], h[2], h[3]);
        if (e != cudaSuccess) return 1;  // sticky: later cases cannot run
    }
    return 0;
}
