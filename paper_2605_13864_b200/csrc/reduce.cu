// Tree-based parallel sum reduction for sm_100a (B200).
//
// Replaces the reference interpreter executing the OptiGPU reduce programs
// (SURVEY A.2/A.3 naive, A.5 tree form).
//
// reduce_kernel (the HBM-bound hot path), one launch per reduction:
//   1. persistent grid (SMs x resident CTAs), 128-bit ld.global.nc grid-stride
//      loads, U independent loads in flight per thread, per-thread accumulator
//      (int32 -> int64 so the sum is exact like the reference's Python ints;
//      fp32 -> binary64, rounded to binary32 once at the end: the result is the
//      correctly rounded sum up to ~n 2^-53 sum|x|, whatever the conditioning);
//   2. warp __shfl_down_sync tree;
//   3. shared-memory block tree over the warp partials with one __syncthreads per
//      level (the barrier structure the paper verifies);
//   4. single-pass grid combine: partial -> workspace, __threadfence, atomic
//      ticket; the last CTA sums the partials in block order (deterministic) and
//      re-arms the ticket, so the workspace stays zero-filled between calls.
//
// tree512_kernel: the A.5 program's exact fp32 evaluation order, bit-identical
// with the reference interpreter (each warp evaluates one 512-element block's
// tree in registers: the same DAG of binary32 adds as the smem halving loop).
#include <algorithm>
#include <type_traits>

#include "b2_internal.cuh"

namespace b2 {
namespace {

template <typename T>
struct AccOf;
// fp32 cells accumulate in binary64 (every float is exact in a double, and the
// chains below stay far from 2^53 ulps): ~0.5 ulp of the binary32 result instead of
// the ~L u sum|x| of an L-long binary32 chain. Costs one F2F per cell, well under
// the conversion throughput the HBM stream needs (6 cells/clk/SM).
template <>
struct AccOf<float> {
    using type = double;
};
template <>
struct AccOf<int32_t> {
    using type = long long;
};
template <>
struct AccOf<double> {
    using type = double;
};
// int64 cells (the reference's ints are unbounded): 128-bit accumulation, exact
// for any n < 2^64
template <>
struct AccOf<int64_t> {
    using type = __int128;
};

template <typename T, typename A>
__device__ __forceinline__ A vec_sum(const uint4 &v);
template <>
__device__ __forceinline__ double vec_sum<float, double>(const uint4 &v) {
    return ((double)__uint_as_float(v.x) + (double)__uint_as_float(v.y)) +
           ((double)__uint_as_float(v.z) + (double)__uint_as_float(v.w));
}
template <>
__device__ __forceinline__ long long vec_sum<int32_t, long long>(const uint4 &v) {
    return ((long long)(int)v.x + (long long)(int)v.y) + ((long long)(int)v.z + (long long)(int)v.w);
}
template <>
__device__ __forceinline__ double vec_sum<double, double>(const uint4 &v) {
    return __hiloint2double((int)v.y, (int)v.x) + __hiloint2double((int)v.w, (int)v.z);
}
template <>
__device__ __forceinline__ __int128 vec_sum<int64_t, __int128>(const uint4 &v) {
    const long long a = (long long)(((unsigned long long)v.y << 32) | v.x);
    const long long b = (long long)(((unsigned long long)v.w << 32) | v.z);
    return (__int128)a + (__int128)b;
}

__device__ __forceinline__ __int128 shfl_down(__int128 a, int off) {
    const unsigned long long lo = (unsigned long long)a, hi = (unsigned long long)(a >> 64);
    const unsigned long long lo2 = __shfl_down_sync(0xffffffffu, lo, off);
    const unsigned long long hi2 = __shfl_down_sync(0xffffffffu, hi, off);
    return (__int128)(((unsigned __int128)hi2 << 64) | lo2);
}
template <typename A>
__device__ __forceinline__ A shfl_down(A a, int off) {
    return __shfl_down_sync(0xffffffffu, a, off);
}
// partials written by other CTAs: read through L2 (volatile semantics)
template <typename A>
__device__ __forceinline__ A load_partial(const A *p) {
    if constexpr (sizeof(A) == 16) {
        const volatile unsigned long long *q = reinterpret_cast<const volatile unsigned long long *>(p);
        return (__int128)(((unsigned __int128)(unsigned long long)q[1] << 64) | (unsigned long long)q[0]);
    } else {
        return *reinterpret_cast<const volatile A *>(p);
    }
}

// The result cell: fp32 sums are returned as binary32 (one rounding of the binary64
// total) unless the caller asked for the raw accumulator (acc_out: the library's
// own chunked / multi-shard pipelines combine binary64 partials and round once).
template <typename T, typename A>
__device__ __forceinline__ void store_result(void *out, A v, bool acc_out) {
    if constexpr (sizeof(T) == 4 && sizeof(A) == 8 && !std::is_integral<T>::value) {
        if (acc_out) *static_cast<double *>(out) = (double)v;
        else *static_cast<float *>(out) = (float)v;
    } else {
        *static_cast<A *>(out) = v;
    }
}

template <typename A>
__device__ __forceinline__ A warp_tree(A a) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) a += shfl_down(a, off);
    return a;
}

// Warp shuffle tree, then a shared-memory halving tree over the NT/32 warp
// partials with __syncthreads per level. Result valid in thread 0.
template <typename A, int NT>
__device__ __forceinline__ A block_tree(A a, A *sm) {
    constexpr int NW = NT / 32;
    a = warp_tree(a);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) sm[w] = a;
    __syncthreads();
#pragma unroll
    for (int h = NW / 2; h > 0; h >>= 1) {
        if (threadIdx.x < h) sm[threadIdx.x] = sm[threadIdx.x] + sm[threadIdx.x + h];
        __syncthreads();
    }
    return sm[0];
}

// ---- fused cross-GPU combine (mailbox in rank 0's memory, mapped into every rank)
// Layout (bytes): slots[kEpochs][64] x 8 | written[64] u64 | consumed u64 | status u64.
// Rank g's last CTA stores its partial into slots[e % kEpochs][g] over NVLink,
// fences at system scope and publishes written[g] = e (release). Rank 0's last CTA
// waits for written[g] >= e for every g (acquire), sums the slots in rank order
// (deterministic for fp32) and publishes consumed = e. A writer may only reuse a
// slot row after the root consumed the epoch that last used it (window kEpochs).
// Every wait is bounded (fz.spin_ns, tune key reduce.spin_ms, default 20 s): on timeout the status word records the epoch
// (atomicMax: it holds the latest failed epoch, so one timeout does not poison
// later healthy calls) and the kernel exits instead of hanging the device; the
// root still publishes consumed = e, so writers of later epochs are not stalled
// behind the abandoned one.
constexpr int kEpochs = 4;
constexpr int kMaxRanks = 64;

using Fused = FusedCombine;

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// wait until *p >= want; false on timeout (status word set)
__device__ __forceinline__ bool wait_ge(const unsigned long long *p, unsigned long long want,
                                        unsigned long long *status, unsigned long long epoch,
                                        unsigned long long spin_ns) {
    const unsigned long long t0 = gtimer();
    while (ld_acquire_sys(p) < want) {
        if (gtimer() - t0 > spin_ns) {
            atomicMax(status, epoch);
            __threadfence_system();
            return false;
        }
        __nanosleep(200);
    }
    return true;
}

template <typename T, typename A>
__device__ void fused_combine(const Fused &fz, A total, void *out, bool acc_out) {
    unsigned char *mb = static_cast<unsigned char *>(fz.mailbox);
    A *slots = reinterpret_cast<A *>(mb);  // 8-byte slots: A is float, long long or double
    unsigned long long *written = reinterpret_cast<unsigned long long *>(mb + kEpochs * kMaxRanks * 8);
    unsigned long long *consumed = written + kMaxRanks;
    unsigned long long *status = consumed + 1;
    const int row = (int)(fz.epoch % kEpochs) * kMaxRanks * (8 / (int)sizeof(A));
    const int stride = 8 / (int)sizeof(A);
    if (fz.rank != 0 && fz.epoch > kEpochs - 1)  // slot row free again?
        if (!wait_ge(consumed, fz.epoch - (kEpochs - 1), status, fz.epoch, fz.spin_ns)) {
            store_result<T, A>(out, total, acc_out);
            return;
        }
    *reinterpret_cast<volatile A *>(slots + row + fz.rank * stride) = total;
    __threadfence_system();
    st_release_sys(written + fz.rank, fz.epoch);
    if (fz.rank != 0) {
        store_result<T, A>(out, total, acc_out);
        return;
    }
    A s = A(0);
    for (int g = 0; g < fz.nranks; ++g) {
        if (!wait_ge(written + g, fz.epoch, status, fz.epoch, fz.spin_ns)) {
            store_result<T, A>(out, total, acc_out);
            st_release_sys(consumed, fz.epoch);  // abandon this epoch, free its slot row
            return;
        }
        s += *reinterpret_cast<volatile A *>(slots + row + g * stride);
    }
    store_result<T, A>(out, s, acc_out);
    __threadfence_system();
    st_release_sys(consumed, fz.epoch);
}

// W x 128 bits per load: W = 2 uses the 256-bit global loads sm_100 adds
// (LDG.E.256), halving the load instructions per byte.
#ifndef B2_LDG256_QUAL
#define B2_LDG256_QUAL "ld.global.nc.L1::no_allocate.v8.b32"
#endif
#ifndef B2_REDUCE_DEFAULT_W
#define B2_REDUCE_DEFAULT_W 1
#endif
template <int W>
struct alignas(16 * W) VecW {
    uint4 q[W];
};
template <int W>
__device__ __forceinline__ VecW<W> ldg_w(const VecW<W> *p) {
    VecW<W> r;
    if constexpr (W == 1) {
        r.q[0] = ldg_stream(reinterpret_cast<const uint4 *>(p));
    } else {
        asm volatile(B2_LDG256_QUAL " {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r.q[0].x), "=r"(r.q[0].y), "=r"(r.q[0].z), "=r"(r.q[0].w), "=r"(r.q[1].x),
                       "=r"(r.q[1].y), "=r"(r.q[1].z), "=r"(r.q[1].w)
                     : "l"(p));
    }
    return r;
}

template <typename T, int NT, int U, int W = 1>
__global__ void __launch_bounds__(NT)
    reduce_kernel(const T *__restrict__ in, int64_t head, int64_t nvec, int64_t n,
                  void *__restrict__ out, typename AccOf<T>::type *__restrict__ partials,
                  unsigned *__restrict__ ticket, Fused fz, bool acc_out) {
    using A = typename AccOf<T>::type;
    constexpr int V = 16 / sizeof(T);
    __shared__ A sm[NT / 32];
    __shared__ bool last;
    pdl_enter();

    A acc = A(0);
    const VecW<W> *vin = reinterpret_cast<const VecW<W> *>(in + head);
    const int64_t stride = (int64_t)gridDim.x * NT;
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    // main body: U independent (W x 128)-bit loads in flight per thread
    for (; i + (U - 1) * stride < nvec; i += U * stride) {
        VecW<W> v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ldg_w<W>(vin + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int w = 0; w < W; ++w) acc += vec_sum<T, A>(v[u].q[w]);
    }
    // remainder (< U vectors per thread): one batch with all loads in flight together
    // instead of one DRAM round trip per leftover vector. Out-of-range slots re-load
    // the thread's own first vector (unconditional loads keep ptxas from serialising
    // them behind the adds) and are masked out of the sum.
    if (i < nvec) {
        VecW<W> v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ldg_w<W>(vin + (i + u * stride < nvec ? i + u * stride : i));
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i + u * stride < nvec)
#pragma unroll
                for (int w = 0; w < W; ++w) acc += vec_sum<T, A>(v[u].q[w]);
    }
    // unaligned head and ragged tail (< V * W elements each)
    const int64_t g = (int64_t)blockIdx.x * NT + threadIdx.x;
    const int64_t tail0 = head + nvec * V * W;
    if (g < head) acc += A(in[g]);
    if (g < n - tail0) acc += A(in[tail0 + g]);

    A bsum = block_tree<A, NT>(acc, sm);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = bsum;
        __threadfence();
        const unsigned t = atomicAdd(ticket, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;
    // last CTA: combine the per-CTA partials in block order
    __threadfence();
    A a = A(0);
    for (int j = threadIdx.x; j < (int)gridDim.x; j += NT)
        a += load_partial<A>(partials + j);
    __syncthreads();  // sm reuse
    A total = block_tree<A, NT>(a, sm);
    if (threadIdx.x == 0) {
        *ticket = 0u;  // re-arm for the next call on this workspace
        if constexpr (sizeof(A) <= 8) {
            if (fz.mailbox) fused_combine<T, A>(fz, total, out, acc_out);
            else store_result<T, A>(out, total, acc_out);
        } else {
            store_result<T, A>(out, total, acc_out);  // 128-bit results: no cross-GPU combine (8-byte slots)
        }
    }
}

// A.5 and its derivation family (programs.reduce_tree_family): B-element blocks
// (B = 64 .. 2048), one per warp per iteration. Lane l holds s[l + 32j]
// (j < B/64) = a[2t] + a[2t+1]; levels h = B/4 .. 32 pair registers of the same
// lane (t + h = l + 32(j + h/32)), h = 16..1 pair lanes via shuffles. Same adds,
// same operands, same association as the interpreter's smem loop `s[t] = s[t] +
// s[t + h]` -> bit-identical partials (B = 512 is A.5).
template <int B, int NT>
__global__ void __launch_bounds__(NT)
    tree_kernel(const float *__restrict__ in, int64_t nblocks, float *__restrict__ partials) {
    constexpr int K = B / 64;  // float2 pairs per lane
    pdl_enter();
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * NT + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * NT) >> 5;
    for (int64_t b = warp; b < nblocks; b += nwarps) {
        const float2 *p = reinterpret_cast<const float2 *>(in + b * B);
        float2 v[K];
#pragma unroll
        for (int j = 0; j < K; ++j) v[j] = __ldg(p + lane + 32 * j);
        float s[K];
#pragma unroll
        for (int j = 0; j < K; ++j) s[j] = __fadd_rn(v[j].x, v[j].y);
#pragma unroll
        for (int h = K / 2; h >= 1; h >>= 1)  // levels B/4 .. 32, in registers
#pragma unroll
            for (int j = 0; j < h; ++j) s[j] = __fadd_rn(s[j], s[j + h]);
        float x = s[0];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)  // levels 16 .. 1
            x = __fadd_rn(x, __shfl_down_sync(0xffffffffu, x, off));
        if (lane == 0) partials[b] = x;
    }
}

constexpr int kMinNT = 256;  // smallest CTA among the variants (sizes the workspace)

int max_grid(int dev) { return num_sms(dev) * (2048 / kMinNT); }

template <typename T, int NT, int U, int W = 1>
int run_reduce_v(const T *in, int64_t n, void *out, void *ws, int dev, cudaStream_t st,
                 const Fused &fz, bool acc_out) {
    using A = typename AccOf<T>::type;
    constexpr int V = 16 / sizeof(T);
    // head: elements before the first (16 W)-byte boundary; nvec: whole W-vectors
    int64_t head = (int64_t)(((16 * W - ((uintptr_t)in & (16 * W - 1))) & (16 * W - 1)) / sizeof(T));
    head = std::min<int64_t>(head, n);
    const int64_t nvec = (n - head) / (V * W);
    static std::atomic<int> occ[64];  // per-device cache (zero-initialised)
    if (occ[dev] == 0) {
        int o = 0;
        B2_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, reduce_kernel<T, NT, U, W>, NT, 0));
        occ[dev] = o > 0 ? o : 1;
    }
    // Default: 1024 threads per SM (2 x 512). Measured on B200: full occupancy
    // (2048) reads 6.94 TB/s, 1536 7.19 TB/s (profiles/r01_tune.md, isolated); in the
    // bench step 1024 beats 1536 by 1.5 % on the reduction and leaves the next
    // transpose untouched, and isolated it is on par (profiles/r01k_reduce_residency.md).
    const int auto_sm = std::max(1, kReduceThreadsPerSM / NT);
    const int per_sm = std::min(g_tune.r_ctas_per_sm > 0 ? g_tune.r_ctas_per_sm : auto_sm, occ[dev].load());
    const int64_t cap = (int64_t)num_sms(dev) * per_sm;
    const int64_t need = std::max<int64_t>(1, (nvec + NT - 1) / NT);
    const int grid = (int)std::min(cap, need);
    unsigned *ticket = (unsigned *)ws;
    A *partials = (A *)((char *)ws + 64);
    B2_CUDA(launch_kernel(reduce_kernel<T, NT, U, W>, dim3(grid), dim3(NT), 0, st, in, head, nvec, n, out, partials,
                          ticket, fz, acc_out));
    count_launch();
    return B2_OK;
}

// <threads, loads in flight per thread> variants; g_tune.r_variant picks one.
template <typename T>
int run_reduce(const void *in_, int64_t n, void *out, void *ws, size_t ws_bytes, int dev,
               cudaStream_t st, const Fused &fz, bool acc_out) {
    using A = typename AccOf<T>::type;
    const T *in = (const T *)in_;
    if ((uintptr_t)in % sizeof(T)) return fail(B2_ERR_INVALID, "reduce: misaligned input");
    const size_t need = (size_t)max_grid(dev) * sizeof(A) + 64;
    if (ws_bytes < need) return fail(B2_ERR_INVALID, "reduce: workspace too small");
    switch (g_tune.r_variant) {
    case 1: return run_reduce_v<T, 512, 8>(in, n, out, ws, dev, st, fz, acc_out);
    case 2: return run_reduce_v<T, 256, 8>(in, n, out, ws, dev, st, fz, acc_out);
    case 3: return run_reduce_v<T, 1024, 4>(in, n, out, ws, dev, st, fz, acc_out);
    case 4: return run_reduce_v<T, 256, 16>(in, n, out, ws, dev, st, fz, acc_out);
    case 5: return run_reduce_v<T, 512, 4, 2>(in, n, out, ws, dev, st, fz, acc_out);   // 256-bit loads
    case 6: return run_reduce_v<T, 512, 2, 2>(in, n, out, ws, dev, st, fz, acc_out);
    case 7: return run_reduce_v<T, 256, 4, 2>(in, n, out, ws, dev, st, fz, acc_out);
    case 8: return run_reduce_v<T, 1024, 2, 2>(in, n, out, ws, dev, st, fz, acc_out);
    case 9: return run_reduce_v<T, 512, 4>(in, n, out, ws, dev, st, fz, acc_out);
    default:
        // 128-bit loads. The 256-bit variants (5-8) read 1-2 % faster in isolation but
        // slowed the FOLLOWING transpose in the bench step by 4 % (A/B of whole bench
        // steps, profiles/r01j_ldst_variants.md), so they stay opt-in.
        return run_reduce_v<T, 512, 4, B2_REDUCE_DEFAULT_W>(in, n, out, ws, dev, st, fz, acc_out);
    }
}

}  // namespace

// The reference's own evaluation order for the naive fp32 program A.2 (interp.py:
// 262-270: `sum += arr[i]`, one binary32 rounding per step, i ascending): inherently
// sequential, so one warp runs it — all 32 lanes stream 8-KB chunks global -> shared
// with 4-byte cp.async (any alignment) into a double buffer, lane 0 adds each chunk's
// cells in order onto the carried binary32 sum (`*acc`, so chunks of a host pipeline
// chain). ~4 cycles per cell (the FADD dependency): C2's 2^24 cells in ~35 ms,
// bit-identical with the reference (tests/test_gpu_seq_sum.py).
constexpr int kSeqChunk = 2048;
__global__ void __launch_bounds__(32) seq_sum_f32_kernel(const float *__restrict__ in, int64_t n, float *acc) {
    __shared__ __align__(16) float buf[2][kSeqChunk];
    const int lane = threadIdx.x;
    const int64_t nch = (n + kSeqChunk - 1) / kSeqChunk;
    pdl_enter();
    auto issue = [&](int64_t c) {
        const int64_t base = c * kSeqChunk;
        const int cnt = (int)min((int64_t)kSeqChunk, n - base);
        float *b = buf[c & 1];
        for (int j = lane; j < cnt; j += 32) {
            const uint32_t sa = (uint32_t)__cvta_generic_to_shared(b + j);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(in + base + j) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    float s = lane == 0 ? *acc : 0.0f;
    if (nch > 0) issue(0);
    for (int64_t c = 0; c < nch; ++c) {
        if (c + 1 < nch) issue(c + 1);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncwarp();  // every lane's copies of chunk c are visible to lane 0
        if (lane == 0) {
            const float *b = buf[c & 1];
            const int cnt = (int)min((int64_t)kSeqChunk, n - c * kSeqChunk);
            int j = 0;
            for (; j + 4 <= cnt; j += 4) {
                const float4 v = *reinterpret_cast<const float4 *>(b + j);
                s = __fadd_rn(s, v.x);
                s = __fadd_rn(s, v.y);
                s = __fadd_rn(s, v.z);
                s = __fadd_rn(s, v.w);
            }
            for (; j < cnt; ++j) s = __fadd_rn(s, b[j]);
        }
        __syncwarp();  // lane 0 is done with buf[c & 1] before chunk c + 2 refills it
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (lane == 0) *acc = s;
}

int launch_seq_sum_f32(const float *in, int64_t n, float *acc, int dev, cudaStream_t st) {
    (void)dev;
    if (n < 0) return fail(B2_ERR_INVALID, "sequential sum: negative length");
    if ((uintptr_t)in % 4) return fail(B2_ERR_INVALID, "sequential sum: input must be 4-byte aligned");
    B2_CUDA(launch_kernel(seq_sum_f32_kernel, dim3(1), dim3(32), 0, st, in, n, acc));
    count_launch();
    return B2_OK;
}

size_t reduce_ws_bytes(int64_t, int dtype, int dev) {
    size_t a = dtype == B2_I64 ? 16 : 8;  // fp32 partials are binary64
    return (size_t)max_grid(dev) * a + 64;
}

size_t mailbox_bytes() { return 4096; }

int launch_reduce(const void *in, int64_t n, int dtype, void *out, void *ws, size_t ws_bytes,
                  int dev, cudaStream_t st, const FusedCombine &fz, bool acc_out) {
    if (fz.mailbox && (fz.nranks < 1 || fz.nranks > kMaxRanks || fz.rank < 0 || fz.rank >= fz.nranks ||
                       fz.epoch == 0))
        return fail(B2_ERR_INVALID, "fused combine: bad rank / nranks / epoch");
    if (fz.mailbox && fz.spin_ns == 0) {
        FusedCombine f2 = fz;
        f2.spin_ns = (unsigned long long)std::max(1, g_tune.r_spin_ms) * 1000000ull;
        return launch_reduce(in, n, dtype, out, ws, ws_bytes, dev, st, f2, acc_out);
    }
    switch (dtype) {
    case B2_F32: return run_reduce<float>(in, n, out, ws, ws_bytes, dev, st, fz, acc_out);
    case B2_I32: return run_reduce<int32_t>(in, n, out, ws, ws_bytes, dev, st, fz, acc_out);
    case B2_F64: return run_reduce<double>(in, n, out, ws, ws_bytes, dev, st, fz, acc_out);
    case B2_I64:
        if (fz.mailbox) return fail(B2_ERR_UNSUPPORTED, "fused combine: int64 sums are 128-bit");
        return run_reduce<int64_t>(in, n, out, ws, ws_bytes, dev, st, fz, acc_out);
    default: return fail(B2_ERR_UNSUPPORTED, "reduce: dtype must be B2_F32, B2_I32, B2_I64 or B2_F64");
    }
}

template <int B>
int run_tree(const float *in, int64_t nb, float *partials, int dev, cudaStream_t st) {
    constexpr int NT = 256;
    const int64_t grid = std::min<int64_t>((nb + NT / 32 - 1) / (NT / 32), (int64_t)num_sms(dev) * 8);
    B2_CUDA(launch_kernel(tree_kernel<B, NT>, dim3((unsigned)grid), dim3(NT), 0, st, in, nb, partials));
    count_launch();
    B2_CUDA(cudaGetLastError());
    return B2_OK;
}

bool tree_block_supported(int block) {
    return block >= 64 && block <= 2048 && (block & (block - 1)) == 0;
}

int launch_tree(const float *in, int64_t n, int block, float *partials, int dev, cudaStream_t st) {
    if (!tree_block_supported(block))
        return fail(B2_ERR_UNSUPPORTED, "tree: block must be a power of two in 64..2048, not " +
                                            std::to_string(block));
    if (n % block != 0 || n <= 0)
        return fail(B2_ERR_INVALID, "exact_div(" + std::to_string(n) + ", " + std::to_string(block) +
                                        ") is not exact");
    if ((uintptr_t)in % 8) return fail(B2_ERR_INVALID, "tree: input must be 8-byte aligned");
    const int64_t nb = n / block;
    switch (block) {
    case 64: return run_tree<64>(in, nb, partials, dev, st);
    case 128: return run_tree<128>(in, nb, partials, dev, st);
    case 256: return run_tree<256>(in, nb, partials, dev, st);
    case 512: return run_tree<512>(in, nb, partials, dev, st);
    case 1024: return run_tree<1024>(in, nb, partials, dev, st);
    default: return run_tree<2048>(in, nb, partials, dev, st);
    }
}

int launch_tree512(const float *in, int64_t n, float *partials, int dev, cudaStream_t st) {
    return launch_tree(in, n, 512, partials, dev, st);
}

}  // namespace b2
