// Probe: how does tcgen05.mma kind::tf32 read an fp32 operand with bits below
// the TF32 mantissa — truncation or round-to-nearest?  D[r][n] = A[r][0] * 1.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o tf32_probe tools/tf32_probe.cu
#include <cstdio>
#include "../paper_1611_06945_b200/csrc/common.cuh"
using namespace b2c;

__global__ void probe(float* out) {
    __shared__ __align__(1024) uint8_t sm[4096 + 1024 + 64];
    uint8_t* A = sm;
    uint8_t* B = sm + 4096;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 4096 + 1024);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    const int tid = threadIdx.x, warp = tid >> 5;
    // A: 128 rows x 8 k, K-major no swizzle: group g at g*256, kc at kc*128, row r%8 at 16*(r%8)
    {
        const int r = tid;
        float a = 1.0f + (float)r * (1.0f / 16384.0f);
        float* p0 = reinterpret_cast<float*>(A + (r >> 3) * 256 + (r & 7) * 16);
        float* p1 = reinterpret_cast<float*>(A + (r >> 3) * 256 + 128 + (r & 7) * 16);
        p0[0] = a; p0[1] = 0.f; p0[2] = 0.f; p0[3] = 0.f;
        p1[0] = 0.f; p1[1] = 0.f; p1[2] = 0.f; p1[3] = 0.f;
        if (r < 32) {
            float* q0 = reinterpret_cast<float*>(B + (r >> 3) * 256 + (r & 7) * 16);
            float* q1 = reinterpret_cast<float*>(B + (r >> 3) * 256 + 128 + (r & 7) * 16);
            for (int i = 0; i < 4; ++i) { q0[i] = 1.f; q1[i] = 1.f; }
        }
    }
    if (tid == 0) { mbar_init(smem_u32(bar), 1); mbar_fence_init(); }
    if (warp == 0) tmem_alloc(smem_u32(slot), 32);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    if (tid == 0) {
        uint64_t da = umma_desc(smem_u32(A), 128, 256), db = umma_desc(smem_u32(B), 128, 256);
        mma_tf32(tmem, da, db, umma_idesc(2, 128, 32), 0u);
        tc_commit(smem_u32(bar));
    }
    __syncwarp();
    mbar_wait(smem_u32(bar), 0);
    tc_fence_after();
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16), v);
    out[tid] = v[0];
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 32); }
}

int main() {
    float* d; cudaMalloc(&d, 128 * 4);
    probe<<<1, 128>>>(d);
    float h[128];
    cudaError_t e = cudaMemcpy(h, d, 512, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    int trunc_ok = 1, rn_ok = 1;
    for (int r = 0; r < 128; ++r) {
        const double a = 1.0 + r / 16384.0, ulp = 1.0 / 1024.0;
        const double tr = 1.0 + (r / 16) * ulp;
        const double rn = 1.0 + ((r + 8) / 16) * ulp;  // ties up (r%16==8) ambiguity noted
        if (h[r] != (float)tr) trunc_ok = 0;
        if (r % 16 != 8 && h[r] != (float)rn) rn_ok = 0;
        if (r < 40 || r % 16 == 8) printf("r=%3d a=%.9f D=%.9f\n", r, a, h[r]);
    }
    printf("tf32 operand read: %s\n", trunc_ok ? "TRUNCATION (low 13 bits ignored)" : rn_ok ? "ROUND-TO-NEAREST" : "OTHER");
    return 0;
}
