// The paper's own SIMT kernels, restated from their published descriptions and
// compiled for sm_100a: the baselines the B200 kernels are measured against
// (Table 7.4 compares exactly these on an RTX 5060).
//   transpose_naive      one element per thread, column-strided stores
//   transpose_tile32     Listing 3.6 / the OptiGPU output (PAPER.md:409-433,
//                        1041-1068): unpadded 32x32 shared tile, 32x16 threads,
//                        2 cells per thread, one __syncthreads
//   transpose_nbc        "transposeNoBankConflicts" shape: the
//                        same tile padded to 32x33, 32x8 threads, 4 cells each
//   reduce_optigpu       the OptiGPU tree (PAPER.md:1120-1131 / SURVEY A.5):
//                        adjacent pair load, in-place shared halving tree with a
//                        barrier per level, one partial per 2*blockDim elements
//   reduce3              two block-strided elements per thread, shared tree
//   reduce6              grid-stride accumulation + shared tree + warp shuffles
// Partials are summed by a second launch of the same kernel family (device only).
// Not product code: built by tools/paper_baselines.py into tools/paperk/.
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void transpose_naive(const float *in, float *out, int W, int H) {
    int x = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 32 + threadIdx.y;
    for (int j = 0; j < 32; j += 8)
        if (x < W && y + j < H) out[(size_t)x * H + y + j] = in[(size_t)(y + j) * W + x];
}

__global__ void transpose_tile32(const float *in, float *out, int W, int H) {
    __shared__ float tile[32][32];
    int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int j = 0; j < 32; j += 16)
        tile[threadIdx.y + j][threadIdx.x] = in[(size_t)(by + threadIdx.y + j) * W + bx + threadIdx.x];
    __syncthreads();
    for (int j = 0; j < 32; j += 16)
        out[(size_t)(bx + threadIdx.y + j) * H + by + threadIdx.x] = tile[threadIdx.x][threadIdx.y + j];
}

__global__ void transpose_nbc(const float *in, float *out, int W, int H) {
    __shared__ float tile[32][33];
    int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int j = 0; j < 32; j += 8)
        tile[threadIdx.y + j][threadIdx.x] = in[(size_t)(by + threadIdx.y + j) * W + bx + threadIdx.x];
    __syncthreads();
    for (int j = 0; j < 32; j += 8)
        out[(size_t)(bx + threadIdx.y + j) * H + by + threadIdx.x] = tile[threadIdx.x][threadIdx.y + j];
}

template <int NT>
__global__ void reduce_optigpu(const float *a, float *partial, int64_t n) {
    __shared__ float s[NT];
    int64_t base = (int64_t)blockIdx.x * 2 * NT;
    int t = threadIdx.x;
    int64_t i = base + 2 * t;
    s[t] = (i < n ? a[i] : 0.f) + (i + 1 < n ? a[i + 1] : 0.f);
    __syncthreads();
    for (int h = NT / 2; h > 0; h >>= 1) {
        if (t < h) s[t] = s[t] + s[t + h];
        __syncthreads();
    }
    if (t == 0) partial[blockIdx.x] = s[0];
}

template <int NT>
__global__ void reduce3(const float *a, float *partial, int64_t n) {
    __shared__ float s[NT];
    int t = threadIdx.x;
    int64_t i = (int64_t)blockIdx.x * 2 * NT + t;
    float v = i < n ? a[i] : 0.f;
    if (i + NT < n) v += a[i + NT];
    s[t] = v;
    __syncthreads();
    for (int h = NT / 2; h > 0; h >>= 1) {
        if (t < h) s[t] = v = v + s[t + h];
        __syncthreads();
    }
    if (t == 0) partial[blockIdx.x] = v;
}

template <int NT>
__global__ void reduce6(const float *a, float *partial, int64_t n) {
    __shared__ float s[NT / 32];
    int t = threadIdx.x;
    float v = 0.f;
    for (int64_t i = (int64_t)blockIdx.x * NT * 2 + t; i < n; i += (int64_t)gridDim.x * NT * 2) {
        v += a[i];
        if (i + NT < n) v += a[i + NT];
    }
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((t & 31) == 0) s[t >> 5] = v;
    __syncthreads();
    if (t < 32) {
        v = t < NT / 32 ? s[t] : 0.f;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (t == 0) partial[blockIdx.x] = v;
    }
}

extern "C" {
int pk_transpose(int which, const float *in, float *out, int W, int H, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    dim3 grid((W + 31) / 32, (H + 31) / 32);
    if (which == 0) transpose_naive<<<grid, dim3(32, 8), 0, st>>>(in, out, W, H);
    else if (which == 1) transpose_tile32<<<grid, dim3(32, 16), 0, st>>>(in, out, W, H);
    else transpose_nbc<<<grid, dim3(32, 8), 0, st>>>(in, out, W, H);
    return (int)cudaGetLastError();
}

// which: 0 = OptiGPU tree, 1 = reduce3, 2 = reduce6. tmp holds the partials of
// both passes (>= n / 512 + 2 floats); the sum lands in *out (device).
int pk_reduce(int which, const float *a, int64_t n, float *tmp, float *out, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    constexpr int NT = 256;
    const float *src = a;
    float *dst = tmp;
    int64_t m = n;
    while (true) {
        int64_t blocks = (m + 2 * NT - 1) / (2 * NT);
        if (which == 2) blocks = blocks < 148 * 8 ? blocks : 148 * 8;
        if (blocks < 1) blocks = 1;
        float *o = blocks == 1 ? out : dst;
        if (which == 0) reduce_optigpu<NT><<<(unsigned)blocks, NT, 0, st>>>(src, o, m);
        else if (which == 1) reduce3<NT><<<(unsigned)blocks, NT, 0, st>>>(src, o, m);
        else reduce6<NT><<<(unsigned)blocks, NT, 0, st>>>(src, o, m);
        if (blocks == 1) break;
        src = dst;
        dst = dst + blocks;
        m = blocks;
    }
    return (int)cudaGetLastError();
}
}
