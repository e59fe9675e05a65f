// b2net.cu — the non-conv node kinds of a whole-network forward:
//   max pooling  (PoolMax, cuclgen/variants.py:688-741; oracle ref_pool_max, oracle.py:100-116)
//   ReLU         (Activation, variants.py:744-775; oracle ref_relu, oracle.py:119-121)
//   layout conversion (Xpose, variants.py:778-827; ndarray.convert_format, ndarray.py:232-253)
// All three are HBM-bound byte movers: no tensor cores, coalesced 128-bit
// accesses where the layout allows it, grids sized in multiples of the SM count.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/b2conv.h"

namespace b2c {
int set_last_error(int code, const char* msg);  // b2conv.cu
}

namespace {

int cuda_fail(cudaError_t e, const char* where) {
    std::string m = std::string(where) + ": " + cudaGetErrorString(e);
    return b2c::set_last_error(B2C_CUDA_ERROR, m.c_str());
}

int grid_for(long long work, int per_block, int sms) {
    long long blocks = (work + per_block - 1) / per_block;
    const long long cap = (long long)sms * 16;  // grid-stride beyond 16 CTAs per SM
    if (blocks > cap) blocks = cap;
    return (int)(blocks < 1 ? 1 : blocks);
}

int num_sms_cached() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

// ---------------------------------------------------------------------------- max pooling
// One thread per output (ox fastest, so a warp reads neighbouring windows of one
// row: the k x k taps hit the same L1 lines).  m starts at -FLT_MAX and only
// in-range taps compete — the -inf-padding semantics of ref_pool_max; a window
// always holds at least one in-range tap because pad < ksz (frontend.py:75-80).
__global__ void __launch_bounds__(256) k_pool_max(const float* __restrict__ x, float* __restrict__ y, int n, int c,
                                                  int h, int w, int r, int s, int p, int oh, int ow) {
    const long long total = (long long)n * c * oh * ow;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int ox = (int)(i % ow);
        long long t = i / ow;
        const int oy = (int)(t % oh);
        const long long plane = t / oh;  // img * c + chan
        const float* xp = x + plane * h * w;
        const int y0 = oy * s - p, x0 = ox * s - p;
        float m = -3.402823466e+38f;
        for (int ky = 0; ky < r; ++ky) {
            const int iy = y0 + ky;
            if (iy < 0 || iy >= h) continue;
            const float* row = xp + (long long)iy * w;
            for (int kx = 0; kx < r; ++kx) {
                const int ix = x0 + kx;
                if (ix < 0 || ix >= w) continue;
                const float v = __ldg(row + ix);
                m = (v > m) ? v : m;
            }
        }
        y[i] = m;
    }
}

// ---------------------------------------------------------------------------- ReLU
// (v > 0) ? v : 0 exactly as the reference kernel writes it (variants.py:164).
__device__ __forceinline__ float relu1(float v) { return (v > 0.0f) ? v : 0.0f; }

__global__ void __launch_bounds__(256) k_relu4(const float4* __restrict__ x, float4* __restrict__ y, long long n4) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
        float4 v = __ldcs(x + i);
        v.x = relu1(v.x);
        v.y = relu1(v.y);
        v.z = relu1(v.z);
        v.w = relu1(v.w);
        __stcs(y + i, v);
    }
}

__global__ void __launch_bounds__(256) k_relu1(const float* __restrict__ x, float* __restrict__ y, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        y[i] = relu1(x[i]);
}

// ---------------------------------------------------------------------------- layout conversion
struct XArgs {
    int nd;
    long long osz[B2C_XPOSE_MAX_DIMS];   // output extent per output dim
    long long ssz[B2C_XPOSE_MAX_DIMS];   // source extent of the same-named dim
    long long sst[B2C_XPOSE_MAX_DIMS];   // source stride (elements) of the same-named dim
    long long ost[B2C_XPOSE_MAX_DIMS];   // output row-major stride
};

// Direct form: one thread per output element, used when the output's innermost
// dim is also contiguous in the source (pure pad/crop/outer permutation), so
// reads and writes are both coalesced.
__global__ void __launch_bounds__(256) k_xpose_direct(const float* __restrict__ x, float* __restrict__ y, XArgs a,
                                                      long long total) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        long long rem = i, src = 0;
        bool in = true;
#pragma unroll
        for (int d = B2C_XPOSE_MAX_DIMS - 1; d >= 0; --d) {
            if (d >= a.nd) continue;
            const long long q = rem % a.osz[d];
            rem /= a.osz[d];
            in &= q < a.ssz[d];
            src += q * a.sst[d];
        }
        y[i] = in ? __ldg(x + src) : 0.0f;  // growth zero-pads (ndarray.py:246-251)
    }
}

// Tiled transpose: dims A (output innermost) and B (the output dim that is
// contiguous in the source) form 32 x 32 tiles staged through shared memory —
// source reads run along B, output writes along A, both coalesced.  The other
// dims are flattened into the z loop.
constexpr int XT = 32;

__global__ void __launch_bounds__(256) k_xpose_tiled(const float* __restrict__ x, float* __restrict__ y, XArgs a,
                                                     int dim_b, long long outer) {
    __shared__ float tile[XT][XT + 1];
    const int dim_a = a.nd - 1;
    const long long a0 = (long long)blockIdx.x * XT, b0 = (long long)blockIdx.y * XT;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
    for (long long o = blockIdx.z; o < outer; o += gridDim.z) {
        // decompose o over the dims other than A and B
        long long rem = o, src = 0, dst = 0;
        bool in = true;
        for (int d = a.nd - 1; d >= 0; --d) {
            if (d == dim_a || d == dim_b) continue;
            const long long q = rem % a.osz[d];
            rem /= a.osz[d];
            in &= q < a.ssz[d];
            src += q * a.sst[d];
            dst += q * a.ost[d];
        }
        __syncthreads();
        // load: threads along B (source-contiguous)
        for (int r = ty; r < XT; r += 8) {
            const long long ia = a0 + r, ib = b0 + tx;
            float v = 0.0f;
            if (in && ia < a.ssz[dim_a] && ib < a.ssz[dim_b] && ia < a.osz[dim_a] && ib < a.osz[dim_b])
                v = __ldg(x + src + ia * a.sst[dim_a] + ib);
            tile[r][tx] = v;
        }
        __syncthreads();
        // store: threads along A (output-contiguous)
        for (int r = ty; r < XT; r += 8) {
            const long long ib = b0 + r, ia = a0 + tx;
            if (ia < a.osz[dim_a] && ib < a.osz[dim_b]) y[dst + ib * a.ost[dim_b] + ia] = tile[tx][r];
        }
    }
}

}  // namespace

extern "C" {

int b2c_pool_max_fwd(const b2c_pool_desc* d, const float* x, float* y, void* stream) {
    if (!d || !x || !y) return b2c::set_last_error(B2C_BAD_ARGS, "null pointer");
    if (d->n < 1 || d->c < 1 || d->h < 1 || d->w < 1 || d->r < 1 || d->stride < 1 || d->pad < 0)
        return b2c::set_last_error(B2C_BAD_ARGS, "bad pool descriptor");
    if (d->pad >= d->r) return b2c::set_last_error(B2C_BAD_ARGS, "pool pad must be < window (frontend.py:75-80)");
    const int oh = (d->h + 2 * d->pad - d->r) / d->stride + 1, ow = (d->w + 2 * d->pad - d->r) / d->stride + 1;
    if (oh < 1 || ow < 1 || oh != d->oh || ow != d->ow)
        return b2c::set_last_error(B2C_BAD_ARGS, "pool output extent != window_out");
    const long long total = (long long)d->n * d->c * oh * ow;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    k_pool_max<<<grid_for(total, 256, num_sms_cached()), 256, 0, st>>>(x, y, d->n, d->c, d->h, d->w, d->r, d->stride,
                                                                       d->pad, oh, ow);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? B2C_OK : cuda_fail(e, "k_pool_max launch");
}

int b2c_relu_fwd(const float* x, float* y, int64_t n, void* stream) {
    if (n < 0 || (n > 0 && (!x || !y))) return b2c::set_last_error(B2C_BAD_ARGS, "bad relu arguments");
    if (n == 0) return B2C_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int sms = num_sms_cached();
    const bool vec = (n % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) % 16 == 0);
    if (vec)
        k_relu4<<<grid_for(n / 4, 256, sms), 256, 0, st>>>(reinterpret_cast<const float4*>(x),
                                                          reinterpret_cast<float4*>(y), n / 4);
    else
        k_relu1<<<grid_for(n, 256, sms), 256, 0, st>>>(x, y, n);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? B2C_OK : cuda_fail(e, "k_relu launch");
}

int b2c_xpose(const b2c_xpose_desc* d, const float* x, float* y, void* stream) {
    if (!d || !x || !y) return b2c::set_last_error(B2C_BAD_ARGS, "null pointer");
    if (d->ndim < 1 || d->ndim > B2C_XPOSE_MAX_DIMS) return b2c::set_last_error(B2C_BAD_ARGS, "ndim out of range");
    XArgs a{};
    a.nd = d->ndim;
    long long total = 1;
    for (int i = d->ndim - 1; i >= 0; --i) {
        if (d->out_sizes[i] < 1 || d->src_sizes[i] < 1 || d->src_strides[i] < 0)
            return b2c::set_last_error(B2C_BAD_ARGS, "bad xpose extents");
        a.osz[i] = d->out_sizes[i];
        a.ssz[i] = d->src_sizes[i];
        a.sst[i] = d->src_strides[i];
        a.ost[i] = total;
        total *= d->out_sizes[i];
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int sms = num_sms_cached();
    const int last = d->ndim - 1;
    int dim_b = -1;  // the output dim that is contiguous in the source
    for (int i = 0; i < d->ndim; ++i)
        if (d->src_strides[i] == 1 && d->src_sizes[i] > 1) dim_b = i;
    if (dim_b < 0 || dim_b == last || d->out_sizes[last] < 8) {
        k_xpose_direct<<<grid_for(total, 256, sms), 256, 0, st>>>(x, y, a, total);
    } else {
        const long long outer = total / (a.osz[last] * a.osz[dim_b]);
        dim3 grid((unsigned)((a.osz[last] + XT - 1) / XT), (unsigned)((a.osz[dim_b] + XT - 1) / XT),
                  (unsigned)(outer < 65535 ? outer : 65535));
        if (grid.x > 2147483647u || grid.y > 65535u) return b2c::set_last_error(B2C_UNSUPPORTED, "xpose tile grid too large");
        k_xpose_tiled<<<grid, 256, 0, st>>>(x, y, a, dim_b, outer);
    }
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? B2C_OK : cuda_fail(e, "k_xpose launch");
}

}  // extern "C"
