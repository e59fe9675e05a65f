// TMA throughput probe (B200): per-SM ingest rate of tiled 2-D boxes of various
// shapes vs 1-D bulk copies.  Each CTA streams its own slice of a large fp32
// matrix through a ring of shared-memory stages; prints bytes/cycle per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_probe tools/tma_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(c)); }
__device__ __forceinline__ void expect_tx(uint32_t bar, uint32_t b) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %0;" ::"r"(b), "r"(bar) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(bar), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma2d(uint32_t dst, const void* tm, uint32_t bar, int x, int y) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst), "l"(tm), "r"(bar), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

constexpr int STAGES = 6;

// mode 0: 2-D boxes (bw cols x bh rows); mode 1: bulk copies of bw*bh*4 bytes
__global__ void probe(const __grid_constant__ CUtensorMap tm, const float* base, int mode, int bw, int bh,
                      int cols, int iters, int wrap_tiles, long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    const uint32_t tiles = (smem_u32(smem) + 1024 + 1023) & ~1023u;
    const uint32_t bytes = (uint32_t)bw * bh * 4;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(smem_u32(&bars[s]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const int tiles_x = cols / bw;
    long long t0 = clock64();
    for (int it = 0; it < iters + STAGES; ++it) {
        if (it >= STAGES) mbar_wait(smem_u32(&bars[it % STAGES]), ((it / STAGES) - 1) & 1);
        if (it < iters) {
            const int s = it % STAGES;
            const uint32_t bar = smem_u32(&bars[s]);
            expect_tx(bar, bytes);
            const int t = (blockIdx.x * iters + it) % wrap_tiles;  // this CTA's t-th tile (wraps: L2-resident runs)
            if (mode == 0) {
                tma2d(tiles + s * bytes, &tm, bar, (t % tiles_x) * bw, (t / tiles_x) * bh);
            } else {
                bulk(tiles + s * bytes, base + (size_t)t * bw * bh, bytes, bar);
            }
        }
    }
    cycles[blockIdx.x] = clock64() - t0;
}

// W issuing warps per CTA (lane 0 of each), each with its own STAGES-deep ring: does a second
// issuer double the per-SM box rate (issue-bound) or not (engine / latency-bound)?
__global__ void probe_multi(const __grid_constant__ CUtensorMap tm, int bw, int bh, int cols, int iters, int wrap_tiles,
                            int nw, long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    const uint32_t bytes = (uint32_t)bw * bh * 4;
    const uint32_t tiles = (smem_u32(smem) + 1024 + 1023) & ~1023u;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES * nw; ++s) mbar_init(smem_u32(&bars[s]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (lane != 0 || warp >= nw) return;
    const int tiles_x = cols / bw;
    long long t0 = clock64();
    for (int it = 0; it < iters + STAGES; ++it) {
        const int s = warp * STAGES + it % STAGES;
        if (it >= STAGES) mbar_wait(smem_u32(&bars[s]), ((it / STAGES) - 1) & 1);
        if (it < iters) {
            const uint32_t bar = smem_u32(&bars[s]);
            expect_tx(bar, bytes);
            const int t = ((blockIdx.x * nw + warp) * iters + it) % wrap_tiles;
            tma2d(tiles + s * bytes, &tm, bar, (t % tiles_x) * bw, (t / tiles_x) * bh);
        }
    }
    const long long dt = clock64() - t0;
    atomicMax((unsigned long long*)&cycles[blockIdx.x], (unsigned long long)dt);
}

using EncFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                           const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                           CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    EncFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    const int rows = 16384, cols = 4096;  // 256 MB
    float* d = nullptr;
    cudaMalloc(&d, (size_t)rows * cols * 4);
    cudaMemset(d, 0, (size_t)rows * cols * 4);
    long long* cyc = nullptr;
    cudaMalloc(&cyc, 1024 * sizeof(long long));
    struct Cfg { int mode, bw, bh; CUtensorMapSwizzle sw; const char* name; int stride = 0; };  // stride: row pitch in bytes (0: dense)
    std::vector<Cfg> cfgs = {
        {0, 32, 128, CU_TENSOR_MAP_SWIZZLE_128B, "box 32x128 SW128 (16 KB)"},
        {0, 32, 256, CU_TENSOR_MAP_SWIZZLE_128B, "box 32x256 SW128 (32 KB)"},
        {0, 16, 256, CU_TENSOR_MAP_SWIZZLE_64B, "box 16x256 SW64 (16 KB)"},
        {0, 64, 64, CU_TENSOR_MAP_SWIZZLE_NONE, "box 64x64 none (16 KB)"},
        {0, 256, 16, CU_TENSOR_MAP_SWIZZLE_NONE, "box 256x16 none (16 KB)"},
        {0, 4, 256, CU_TENSOR_MAP_SWIZZLE_NONE, "box 4x256 none (4 KB, 16 B rows)"},
        {1, 32, 128, CU_TENSOR_MAP_SWIZZLE_NONE, "bulk 16 KB"},
        {1, 32, 256, CU_TENSOR_MAP_SWIZZLE_NONE, "bulk 32 KB"},
        // first-layer x-window rows: 128-byte rows whose starts advance by less than 128 B (overlapping,
        // mostly unaligned), as k_tconv MODE 4 reads them for stride-2 / stride-4 convs
        {0, 32, 128, CU_TENSOR_MAP_SWIZZLE_128B, "box 32x128 SW128 pitch 128 B", 128},
        {0, 32, 128, CU_TENSOR_MAP_SWIZZLE_128B, "box 32x128 SW128 pitch 64 B", 64},
        {0, 32, 128, CU_TENSOR_MAP_SWIZZLE_128B, "box 32x128 SW128 pitch 32 B", 32},
        {0, 32, 128, CU_TENSOR_MAP_SWIZZLE_128B, "box 32x128 SW128 pitch 48 B", 48},
    };
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    for (auto& c : cfgs) {
        CUtensorMap tm;
        const int ccols = c.stride ? c.bw : cols;  // pitched maps: one tile column
        const long long crows = c.stride ? ((long long)rows * cols * 4 - 512) / c.stride : rows;
        const cuuint64_t dims[2] = {(cuuint64_t)ccols, (cuuint64_t)crows};
        const cuuint64_t str[1] = {(cuuint64_t)(c.stride ? c.stride : cols * 4)};
        const cuuint32_t box[2] = {(cuuint32_t)c.bw, (cuuint32_t)c.bh};
        const cuuint32_t es[2] = {1, 1};
        if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, c.sw,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            printf("%-34s encode failed\n", c.name);
            continue;
        }
        const int bytes = c.bw * c.bh * 4;
        const int smem = 2048 + STAGES * bytes;
        for (int l2 = 0; l2 < 2; ++l2)
        for (int grid : {1, 16, 148}) {
            const long long total_tiles = c.stride ? crows / c.bh : (long long)rows * cols * 4 / bytes;
            int iters = (int)std::min<long long>(total_tiles / grid, 2048);
            // l2: re-read a 32 MB window (L2-resident after the first pass)
            const int wrap = l2 ? (int)((32ll << 20) / bytes) : (int)total_tiles;
            if (l2) iters = 512;
            for (int rep = 0; rep < 2; ++rep) probe<<<grid, 32, smem>>>(tm, d, c.mode, c.bw, c.bh, ccols, iters, wrap, cyc);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            std::vector<long long> h(grid);
            cudaMemcpy(h.data(), cyc, grid * 8, cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (auto v : h) mx = v > mx ? v : mx;
            printf("%-34s %s grid %3d: %6.1f B/clk/SM  (%d tiles/CTA, %lld cyc)\n", c.name, l2 ? "L2  " : "DRAM", grid,
                   (double)iters * bytes / mx, iters, mx);
        }
    }
    // issue-rate test: 16 KB SW128 boxes re-read from L2, 1 / 2 / 4 issuing warps per CTA (each a 6-deep ring)
    {
        CUtensorMap tm;
        const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
        const cuuint64_t str[1] = {(cuuint64_t)cols * 4};
        const cuuint32_t box[2] = {32, 128};
        const cuuint32_t es[2] = {1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int bytes = 32 * 128 * 4;
        cudaFuncSetAttribute(probe_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        for (int nw : {1, 2}) {
            for (int grid : {1, 148}) {
                const int iters = 256;
                const int smem = 2048 + STAGES * nw * bytes;
                cudaMemset(cyc, 0, 1024 * sizeof(long long));
                for (int rep = 0; rep < 2; ++rep) {
                    cudaMemset(cyc, 0, 1024 * sizeof(long long));
                    probe_multi<<<grid, 32 * nw, smem>>>(tm, 32, 128, cols, iters, (int)((32ll << 20) / bytes), nw, cyc);
                }
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
                std::vector<long long> h(grid);
                cudaMemcpy(h.data(), cyc, grid * 8, cudaMemcpyDeviceToHost);
                long long mx = 0;
                for (auto v : h) mx = v > mx ? v : mx;
                printf("issuers %d grid %3d: %6.1f B/clk/SM, %.0f cycles per box per SM\n", nw, grid,
                       (double)iters * nw * bytes / mx, (double)mx / (iters * nw));
            }
        }
    }
    return 0;
}
