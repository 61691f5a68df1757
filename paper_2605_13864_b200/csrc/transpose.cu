// Tiled matrix transpose for sm_100a (B200).
//
// Replaces the reference interpreter executing the OptiGPU transpose programs
// (SURVEY A.1 naive nest and A.4 GPU form): out is
// the W x H transpose of the H x W input, a pure permutation, bit-exact for every
// element width.
//
// Large aligned matrices (the C4 hot path) go to the cp.async-loaded tiles of
// transpose_cpa.cu since round 2; this file's register-staged vector path serves the
// smaller aligned ones (and every size with transpose.cpa = 0).
//
// Vector path (16-B aligned pitches):
//   * each thread owns V x V "micro-tiles" (V = 16 / sizeof(elem)): V 128-bit
//     coalesced loads from V consecutive input rows, an in-register V x V
//     transpose (PRMT byte permutes for 2-byte cells), then V 128-bit stores into
//     a shared-memory tile laid out in OUTPUT orientation;
//   * the shared tile is XOR-swizzled at 16-B granularity (phys = col ^ (row/V)&7)
//     so both the transposed STS.128 and the row-wise LDS.128 are bank-conflict
//     free (the B200 equivalent of the paper's +1 padding, without losing 16-B
//     alignment);
//   * one __syncthreads between stage-in and stage-out (the barrier the paper's
//     blocksync() proves), then 128-bit coalesced stores;
//   * persistent grid (a multiple of the SM count) walking tiles; the next tile's
//     loads are issued before the current tile's stores so HBM reads and writes
//     overlap inside every CTA.
// Scalar path (odd pitches / edge strips): the classic padded 32 x 33 tile.
#include "b2_internal.cuh"

namespace b2 {
namespace {

template <int E>
struct Micro {
    static constexpr int V = 16 / E;
};

// In-register V x V transpose of a micro-tile held as V uint4 rows.
__device__ __forceinline__ void micro_transpose4(uint4 (&v)[4]) {  // 4-byte cells
    uint4 o[4];
    o[0] = make_uint4(v[0].x, v[1].x, v[2].x, v[3].x);
    o[1] = make_uint4(v[0].y, v[1].y, v[2].y, v[3].y);
    o[2] = make_uint4(v[0].z, v[1].z, v[2].z, v[3].z);
    o[3] = make_uint4(v[0].w, v[1].w, v[2].w, v[3].w);
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = o[i];
}

__device__ __forceinline__ void micro_transpose8(uint4 (&v)[2]) {  // 8-byte cells
    uint4 o0 = make_uint4(v[0].x, v[0].y, v[1].x, v[1].y);
    uint4 o1 = make_uint4(v[0].z, v[0].w, v[1].z, v[1].w);
    v[0] = o0;
    v[1] = o1;
}

__device__ __forceinline__ uint32_t word(const uint4 &v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

__device__ __forceinline__ void micro_transpose2(uint4 (&v)[8]) {  // 2-byte cells
    // out[j] element k = in[k] element j. Element j of a row lives in word j/2,
    // half j%2; output word m packs elements (2m, j) and (2m+1, j).
    uint4 o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t sel = (j & 1) ? 0x7632u : 0x5410u;
        uint32_t w[4];
#pragma unroll
        for (int m = 0; m < 4; ++m)
            w[m] = __byte_perm(word(v[2 * m], j >> 1), word(v[2 * m + 1], j >> 1), sel);
        o[j] = make_uint4(w[0], w[1], w[2], w[3]);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = o[i];
}

template <int E>
__device__ __forceinline__ void micro_transpose(uint4 (&v)[16 / E]) {
    if constexpr (E == 4) micro_transpose4(v);
    else if constexpr (E == 8) micro_transpose8(v);
    else micro_transpose2(v);
}

// Tile = (TRV*V) input rows x (TCV*V) input columns; NT threads; each thread owns
// MT = TRV*TCV/NT micro-tiles.
template <int E, int TRV, int TCV, int NT>
__global__ void __launch_bounds__(NT)
    transpose_vec_kernel(const uint8_t *__restrict__ in, uint8_t *__restrict__ out,
                         int64_t rows_v, int64_t cols_v, int64_t ld_in_b, int64_t ld_out_b,
                         int64_t tiles_r, int64_t tiles_c, int64_t ntiles, int group) {
    constexpr int V = Micro<E>::V;
    constexpr int TR = TRV * V;  // input rows per tile   (= output vector columns * V)
    constexpr int TC = TCV * V;  // input cols per tile   (= output rows)
    constexpr int MT = TRV * TCV / NT;
    static_assert(MT >= 1 && TRV * TCV % NT == 0, "tile/thread mismatch");
    static_assert(TRV >= 8 && (TRV & (TRV - 1)) == 0, "swizzle needs >= 8 vector columns");
    constexpr int ST = TC * TRV / NT;  // 16-B stores per thread per tile

    extern __shared__ uint4 S[];  // TC * TRV vectors (dynamic: large tiles exceed 48 KB)

    uint4 reg[MT][V];
    pdl_enter();

    // Tile order: bands of `group` tile-rows, walked column by column inside a
    // band; with group = tiles_r (the default) the walk is column-major, so CTAs
    // running at the same time work down one column block and write neighbouring
    // segments of the same output rows.
    auto origin = [&](int64_t tile, int64_t &r0, int64_t &c0) {
        const int64_t per_band = (int64_t)group * tiles_c;
        const int64_t band = tile / per_band, w = tile - band * per_band;
        const int64_t rows_in_band = min((int64_t)group, tiles_r - band * group);
        r0 = (band * group + w % rows_in_band) * TR;
        c0 = (w / rows_in_band) * TC;
    };
    auto load_tile = [&](int64_t tile) {
        int64_t r0, c0;
        origin(tile, r0, c0);
#pragma unroll
        for (int m = 0; m < MT; ++m) {
            const int mt = threadIdx.x + m * NT;
            const int vc = mt % TCV, rg = mt / TCV;
            const int64_t r = r0 + rg * V, c = c0 + vc * V;
            if (r < rows_v && c < cols_v) {
                const uint8_t *p = in + r * ld_in_b + c * E;
#pragma unroll
                for (int k = 0; k < V; ++k)
                    reg[m][k] = ldg_stream(reinterpret_cast<const uint4 *>(p + k * ld_in_b));
            }
        }
    };

    int64_t tile = blockIdx.x;
    if (tile < ntiles) load_tile(tile);
    for (; tile < ntiles; tile += gridDim.x) {
        int64_t r0, c0;
        origin(tile, r0, c0);
        // stage-in: register transpose, swizzled 16-B stores in output orientation
#pragma unroll
        for (int m = 0; m < MT; ++m) {
            const int mt = threadIdx.x + m * NT;
            const int vc = mt % TCV, rg = mt / TCV;
            micro_transpose<E>(reg[m]);
#pragma unroll
            for (int k = 0; k < V; ++k) {
                const int orow = vc * V + k;
                S[orow * TRV + (rg ^ ((orow / V) & 7))] = reg[m][k];
            }
        }
        __syncthreads();
        // prefetch the next tile while this one drains to HBM
        const int64_t next = tile + gridDim.x;
        if (next < ntiles) load_tile(next);
        // stage-out: row-wise 16-B reads, coalesced stores. 4- and 8-byte cells pair two
        // 16-B chunks into one 256-bit store (STG.E.256, sm_100) marked L2 evict-first:
        // +0.8 % in the bench step, +1-1.6 % isolated; plain 256-bit stores and 2-byte
        // cells measured slower (profiles/r01k_st256.md), so those keep 128-bit stores.
        if (E >= 4 && ((uintptr_t)out % 32 == 0) && (ld_out_b % 32 == 0)) {
#pragma unroll
            for (int s = 0; s < ST / 2; ++s) {
                const int idx = threadIdx.x + s * NT;
                const int orow = idx / (TRV / 2), ocp = idx % (TRV / 2);
                const int64_t oc = c0 + orow, orr = r0 + 2 * ocp * V;
                if (oc < cols_v && orr < rows_v) {
                    // Bank-conflict-free pair reads: a quarter-warp (8 lanes x 16 B) must
                    // touch all eight 16-B bank groups. Lanes 0-3 of each quarter read their
                    // even chunk first, lanes 4-7 their odd chunk first (chunk indices mod 8
                    // then cover 0..7), and the pair is put back in order in registers.
                    const int sw = (orow / V) & 7;
                    const int odd_first = (idx >> 2) & 1;
                    const uint4 p0 = S[orow * TRV + ((2 * ocp + odd_first) ^ sw)];
                    const uint4 p1 = S[orow * TRV + ((2 * ocp + 1 - odd_first) ^ sw)];
                    const uint4 a = odd_first ? p1 : p0;
                    if (orr + V < rows_v) {
                        const uint4 b = odd_first ? p0 : p1;
                        asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                                     ::"l"(out + oc * ld_out_b + orr * E),
                                     "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
                                     : "memory");
                    } else {
                        stg_stream(reinterpret_cast<uint4 *>(out + oc * ld_out_b + orr * E), a);
                    }
                }
            }
        } else
#pragma unroll
        for (int s = 0; s < ST; ++s) {
            const int idx = threadIdx.x + s * NT;
            const int orow = idx / TRV, ocv = idx % TRV;
            const int64_t oc = c0 + orow, orr = r0 + ocv * V;
            if (oc < cols_v && orr < rows_v) {
                const uint4 v = S[orow * TRV + (ocv ^ ((orow / V) & 7))];
                stg_stream(reinterpret_cast<uint4 *>(out + oc * ld_out_b + orr * E), v);
            }
        }
        __syncthreads();
    }
}

// Padded tile (the paper's transposeNoBankConflicts shape) over a
// sub-rectangle [r_lo, r_hi) x [c_lo, c_hi); any pitch, any alignment. 64 x 64
// cells per tile, 256 threads, 16 cells per thread in flight; the +PAD column
// keeps the transposed shared-memory reads on distinct banks for every width.
template <typename T, int TC = 64>
__global__ void __launch_bounds__(256)
    transpose_scalar_kernel(const T *__restrict__ in, T *__restrict__ out, int64_t r_lo,
                            int64_t r_hi, int64_t c_lo, int64_t c_hi, int64_t ld_in,
                            int64_t ld_out, int64_t tiles_c, int64_t ntiles) {
    constexpr int TR = 64;        // tile rows; TC tile columns (64, or 128 for narrow cells)
    constexpr int HC = TC / 32;   // column groups per thread
    constexpr int PAD = sizeof(T) == 2 ? 2 : 1;
    __shared__ T tile[TR][TC + PAD];
    pdl_enter();
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    const int64_t tiles_r = ntiles / tiles_c;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        // column-major tile walk, as in the vector path: concurrent tiles share
        // output rows, so the (short) output segments merge into long write runs
        const int64_t r0 = r_lo + (t % tiles_r) * TR, c0 = c_lo + (t / tiles_r) * TC;
        T v[TR / 8][HC];
#pragma unroll
        for (int j = 0; j < TR / 8; ++j) {
            const int64_t r = r0 + ty + 8 * j;
#pragma unroll
            for (int h = 0; h < HC; ++h) {
                const int64_t c = c0 + tx + 32 * h;
                if (r < r_hi && c < c_hi) v[j][h] = in[r * ld_in + c];
            }
        }
#pragma unroll
        for (int j = 0; j < TR / 8; ++j)
#pragma unroll
            for (int h = 0; h < HC; ++h) tile[ty + 8 * j][tx + 32 * h] = v[j][h];
        __syncthreads();
        // out[c][r]: output rows are input columns (TC of them), output columns the
        // TR input rows; 8 warps x (TC / 8) output rows, 32 lanes x 2 output columns
#pragma unroll
        for (int j = 0; j < TC / 8; ++j) {
            const int64_t oc = c0 + ty + 8 * j;  // out row = input col
#pragma unroll
            for (int h = 0; h < TR / 32; ++h) {
                const int64_t orr = r0 + tx + 32 * h;
                if (oc < c_hi && orr < r_hi) out[oc * ld_out + orr] = tile[tx + 32 * h][ty + 8 * j];
            }
        }
        __syncthreads();
    }
}

// Degenerate shapes (one row or one column): the transpose is a strided copy
// out[i * so] = in[i * si]; 128-bit vectors when both sides are contiguous.
template <typename T>
__global__ void __launch_bounds__(256)
    strided_copy_kernel(const T *__restrict__ in, T *__restrict__ out, int64_t n, int64_t si,
                        int64_t so) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    constexpr int V = 16 / sizeof(T);
    if (si == 1 && so == 1 && ((uintptr_t)in % 16 == 0) && ((uintptr_t)out % 16 == 0)) {
        const int64_t nv = n / V;
        for (int64_t k = i; k < nv; k += stride)
            stg_stream(reinterpret_cast<uint4 *>(out) + k, ldg_stream(reinterpret_cast<const uint4 *>(in) + k));
        for (int64_t k = nv * V + i; k < n; k += stride) out[k] = in[k];
        return;
    }
    for (int64_t k = i; k < n; k += stride) out[k * so] = in[k * si];
}

template <typename T>
int run_copy(const void *in, void *out, int64_t n, int64_t si, int64_t so, int dev,
             cudaStream_t st) {
    const int64_t per = 256 * (16 / (int64_t)sizeof(T));
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((n + per - 1) / per, (int64_t)num_sms(dev) * 8));
    strided_copy_kernel<T><<<(unsigned)grid, 256, 0, st>>>((const T *)in, (T *)out, n, si, so);
    count_launch();
    B2_CUDA(cudaGetLastError());
    return B2_OK;
}

template <int E, int TRV, int TCV, int NT>
int run_vec(const void *in, void *out, int64_t rows_v, int64_t cols_v, int64_t ld_in,
            int64_t ld_out, int dev, cudaStream_t st) {
    constexpr int V = 16 / E;
    constexpr int TR = TRV * V, TC = TCV * V;
    const int64_t tiles_r = (rows_v + TR - 1) / TR, tiles_c = (cols_v + TC - 1) / TC;
    const int64_t ntiles = tiles_r * tiles_c;
    if (ntiles == 0) return B2_OK;
    constexpr int kSmem = TC * TRV * 16;
    static std::atomic<int> occ[64];  // per-device cache (zero-initialised)
    if (occ[dev] == 0) {
        if (kSmem > 48 * 1024)
            B2_CUDA(cudaFuncSetAttribute(transpose_vec_kernel<E, TRV, TCV, NT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        int o = 0;
        B2_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &o, transpose_vec_kernel<E, TRV, TCV, NT>, NT, kSmem));
        occ[dev] = o > 0 ? o : 1;
    }
    // Default residency: ~64 KB of tile data in flight per SM. Measured on B200
    // (profiles/r01_tune.md): more resident tiles than that only adds DRAM
    // page/turnaround contention (fp32 64x64: 6 CTAs/SM 5.69 TB/s, 4 CTAs 6.13).
    constexpr int kTileBytes = TR * TC * E;
    const int auto_sm = std::max(1, kInflightBytesPerSM / kTileBytes);
    const int per_sm = std::min(g_tune.t_ctas_per_sm > 0 ? g_tune.t_ctas_per_sm : auto_sm, occ[dev].load());
    const int64_t grid = std::min<int64_t>(ntiles, (int64_t)num_sms(dev) * per_sm);
    // Tile walk. Column-major (band height = all tile-rows) when a column block holds
    // about as many tiles as there are SMs: the tiles in flight then sit in ONE
    // column block and their output rows are written as long contiguous runs
    // (fp32 32768^2 6.37-6.43 TB/s vs 6.01-6.18 row-major, fp64 +5 %, bf16 +3 %;
    // profiles/r01h_colwalk.md). With fewer tile-rows the window would straddle
    // several column blocks, and row-major bands measure better (8192x16384 +4 %,
    // 16384x8192 +7 %, 4096x32768 +3 %; profiles/r01n_midsize.md).
    const bool colwalk = tiles_r * 4 >= (int64_t)num_sms(dev) * 3;
    const int grp = g_tune.t_group > 0 ? g_tune.t_group
                                       : colwalk ? (int)std::min<int64_t>(tiles_r, 1 << 30)
                                                 : (kTileBytes >= 64 * 1024 ? 1 : 4);
    const int group = (int)std::max<int64_t>(1, std::min<int64_t>(grp, tiles_r));
    B2_CUDA(launch_kernel(transpose_vec_kernel<E, TRV, TCV, NT>, dim3((unsigned)grid), dim3(NT), kSmem, st,
                          (const uint8_t *)in, (uint8_t *)out, rows_v, cols_v, ld_in * E, ld_out * E, tiles_r,
                          tiles_c, ntiles, group));
    count_launch();
    return B2_OK;
}

template <typename T, int TC>
int run_scalar_tc(const void *in, void *out, int64_t r_lo, int64_t r_hi, int64_t c_lo,
                  int64_t c_hi, int64_t ld_in, int64_t ld_out, int dev, cudaStream_t st);

template <typename T>
int run_scalar(const void *in, void *out, int64_t r_lo, int64_t r_hi, int64_t c_lo,
               int64_t c_hi, int64_t ld_in, int64_t ld_out, int dev, cudaStream_t st) {
    if (r_hi <= r_lo || c_hi <= c_lo) return B2_OK;
    // 2-byte cells: 64 x 128 tiles (256-B input row runs; 64 x 64 over-fetches ~1.8x
    // from DRAM on odd pitches, profiles/r01_odd.md); transpose.scalar_tile = 64 opts out
    if constexpr (sizeof(T) == 2) {
        if (g_tune.t_scalar_tile != 64) return run_scalar_tc<T, 128>(in, out, r_lo, r_hi, c_lo, c_hi, ld_in, ld_out, dev, st);
    } else if constexpr (sizeof(T) == 4) {
        if (g_tune.t_scalar_tile == 128) return run_scalar_tc<T, 128>(in, out, r_lo, r_hi, c_lo, c_hi, ld_in, ld_out, dev, st);
    }
    return run_scalar_tc<T, 64>(in, out, r_lo, r_hi, c_lo, c_hi, ld_in, ld_out, dev, st);
}

template <typename T, int TC>
int run_scalar_tc(const void *in, void *out, int64_t r_lo, int64_t r_hi, int64_t c_lo,
                  int64_t c_hi, int64_t ld_in, int64_t ld_out, int dev, cudaStream_t st) {
    const int64_t tiles_r = (r_hi - r_lo + 63) / 64, tiles_c = (c_hi - c_lo + TC - 1) / TC;
    const int64_t ntiles = tiles_r * tiles_c;
    // same ~64 KB-of-tiles-in-flight rule as the vector path (profiles/r01_odd.md); the
    // 2-byte 64 x 128 tiles keep 32 KB in flight on large matrices (measured +13-33 %)
    int auto_sm = std::max(1, kInflightBytesPerSM / (64 * TC * (int)sizeof(T)));
    if (sizeof(T) == 2 && TC == 128 && ntiles >= 48 * (int64_t)num_sms(dev)) auto_sm = 2;
    const int per_sm = g_tune.t_scalar_ctas > 0 ? g_tune.t_scalar_ctas : auto_sm;
    const int64_t grid = std::min<int64_t>(ntiles, (int64_t)num_sms(dev) * per_sm);
    B2_CUDA(launch_kernel(transpose_scalar_kernel<T, TC>, dim3((unsigned)grid), dim3(256), 0, st, (const T *)in,
                          (T *)out, r_lo, r_hi, c_lo, c_hi, ld_in, ld_out, tiles_c, ntiles));
    count_launch();
    return B2_OK;
}

template <typename T>
int run_scalar_all(const void *in, void *out, int64_t rows, int64_t cols, int64_t rv,
                   int64_t cv, int64_t ld_in, int64_t ld_out, int dev, cudaStream_t st) {
    // right strip [0,rows) x [cv,cols) and bottom strip [rv,rows) x [0,cv)
    int rc = run_scalar<T>(in, out, 0, rows, cv, cols, ld_in, ld_out, dev, st);
    if (rc) return rc;
    return run_scalar<T>(in, out, rv, rows, 0, cv, ld_in, ld_out, dev, st);
}

// Tile shapes per element size; g_tune.t_variant picks one (0 = default).
//   4-byte: 0: 64x64   1: 128x64 (rows x cols)   2: 64x128   3: 256x32   4: 128x32
//           5: 128x128 (512 thr)  6: 128x128 (256 thr)  7: 256x128 (512 thr, 128 KB smem)
//   2-byte: 0: 128x128 1: 64x128                 2: 128x64
//   8-byte: 0: 64x32   1: 32x32                  2: 64x64
template <int E>
int run_vec_for(const void *in, void *out, int64_t rv, int64_t cv, int64_t ld_in,
                int64_t ld_out, int dev, cudaStream_t st) {
    const int v = g_tune.t_variant;
    // Large matrices: one 128-KB tile per SM (256 x 512 B) — half as many concurrent
    // DRAM row streams, each twice as long, measured +2.5 % for fp32 / fp64
    // (profiles/r01_tune_big.md). Needs enough tiles to keep every SM busy.
    // t_big == 2 forces them whatever the size (sanitizer / test coverage).
    const int64_t big_min_tiles = g_tune.t_big == 2 ? 1 : 8 * (int64_t)num_sms(dev);
    if (v == 0 && g_tune.t_big) {
        if constexpr (E == 4) {
            if (rv >= 256 && cv >= 128 && (rv / 256) * (cv / 128) >= big_min_tiles)
                return run_vec<4, 64, 32, 512>(in, out, rv, cv, ld_in, ld_out, dev, st);
        } else if constexpr (E == 8) {
            if (rv >= 256 && cv >= 64 && (rv / 256) * (cv / 64) >= big_min_tiles)
                return run_vec<8, 128, 32, 512>(in, out, rv, cv, ld_in, ld_out, dev, st);
        }
    }
    if constexpr (E == 4) {
        if (v == 1) return run_vec<4, 32, 16, 256>(in, out, rv, cv, ld_in, ld_out, dev, st);
        if (v == 2) return run_vec<4, 16, 32, 256>(in, out, rv, cv, ld_in, ld_out, dev, st);
        if (v == 3) return run_vec<4, 64, 8, 256>(in, out, rv, cv, ld_in, ld_out, dev, st);
        if (v == 4) return run_vec<4, 32, 8, 256>(in, out, rv, cv, ld_in, ld_out, dev, st);
        if (v == 5) return run_vec<4, 32, 32, 512>(in, out, rv, cv, ld_in, ld_out, dev, st);
        if (v == 6) return run_vec<4, 32, 32, 256>(in, out, rv, cv, ld_in, ld_out, dev, st);
        if (v == 7) return run_vec<4, 64, 32, 512>(in, out, rv, cv, ld_in, ld_out, dev, st);
        if (v == 8) return run_vec<4, 64, 16, 512>(in, out, rv, cv, ld_in, ld_out, dev, st);
        if (v == 9) return run_vec<4, 32, 64, 512>(in, out, rv, cv, ld_in, ld_out, dev, st);
        if (v == 10) return run_vec<4, 64, 32, 1024>(in, out, rv, cv, ld_in, ld_out, dev, st);
        return run_vec<4, 16, 16, 256>(in, out, rv, cv, ld_in, ld_out, dev, st);
    } else if constexpr (E == 2) {
        if (v == 1) return run_vec<2, 8, 16, 128>(in, out, rv, cv, ld_in, ld_out, dev, st);
        if (v == 2) return run_vec<2, 16, 8, 128>(in, out, rv, cv, ld_in, ld_out, dev, st);
        if (v == 7) return run_vec<2, 32, 32, 512>(in, out, rv, cv, ld_in, ld_out, dev, st);
        return run_vec<2, 16, 16, 256>(in, out, rv, cv, ld_in, ld_out, dev, st);
    } else {
        if (v == 1) return run_vec<8, 16, 16, 256>(in, out, rv, cv, ld_in, ld_out, dev, st);
        if (v == 2) return run_vec<8, 32, 32, 256>(in, out, rv, cv, ld_in, ld_out, dev, st);
        if (v == 7) return run_vec<8, 128, 32, 512>(in, out, rv, cv, ld_in, ld_out, dev, st);
        return run_vec<8, 32, 16, 256>(in, out, rv, cv, ld_in, ld_out, dev, st);
    }
}

template <typename T>
int dispatch(const void *in, void *out, int64_t rows, int64_t cols, int64_t ld_in,
             int64_t ld_out, int dev, cudaStream_t st) {
    constexpr int E = sizeof(T);
    constexpr int V = 16 / E;
    // one row: out[c][0] = in[0][c];  one column: out[0][r] = in[r][0]
    if (rows == 1) return run_copy<T>(in, out, cols, 1, ld_out, dev, st);
    if (cols == 1) return run_copy<T>(in, out, rows, ld_in, 1, dev, st);
    if constexpr (E == 4) {
        if (g_tune.t_tma) {
            const int rc = launch_transpose_tma(in, out, rows, cols, ld_in, ld_out, dev, st);
            if (rc != B2_ERR_UNSUPPORTED) return rc;  // else: fall through to the LDG path
        }
    }
    const bool aligned = E >= 2 && ((uintptr_t)in % 16 == 0) && ((uintptr_t)out % 16 == 0) &&
                         (ld_in * E % 16 == 0) && (ld_out * E % 16 == 0);
    if (!aligned) {
        // odd pitches / unaligned views: funnel-shifted 128-bit path (transpose_any.cu)
        if constexpr (E >= 2) {
            if (g_tune.t_any) return launch_transpose_any(in, out, rows, cols, ld_in, ld_out, E, dev, st);
            // cp.async-staged 16-B chunks (transpose_staged.cu) unless the cells themselves
            // are misaligned (then only the scalar tile applies). Auto (t_staged = 1):
            // 2-byte cells from 2^22 cells up, where it measured +27..40 % over the scalar
            // tile (bf16 4097x8191 3.6 -> 4.6 TB/s, 16385x16383 3.76 -> 5.15 TB/s); 4- and
            // 8-byte cells and small matrices stay on the scalar tile, which is on par or
            // faster there (profiles/r02c_odd_staged.md). t_staged = 2 forces it.
            // Round 2: every cell width beyond 256 MB of input, on 128-row tiles
            // (+4..12 % over the scalar tile for 4- / 8-byte cells, profiles/r02s_odd_geom.md).
            const bool use = g_tune.t_staged == 2 ||
                             (g_tune.t_staged == 1 && ((E == 2 && rows * cols >= (int64_t(1) << 22)) ||
                                                       rows * cols * E > (int64_t(256) << 20)));
            if (use && (uintptr_t)in % E == 0 && (uintptr_t)out % E == 0)
                return launch_transpose_staged(in, out, rows, cols, ld_in, ld_out, E, dev, st);
        }
        return run_scalar<T>(in, out, 0, rows, 0, cols, ld_in, ld_out, dev, st);
    }
    const int64_t rv = rows - rows % V, cv = cols - cols % V;
    if constexpr (E >= 2) {
        // aligned interior: cp.async-loaded tiles (transpose_cpa.cu) on large matrices,
        // register-staged LDG tiles below (and with transpose.cpa = 0)
        int rc = transpose_cpa_wanted(rv, cv, E, dev) ? launch_transpose_cpa(in, out, rv, cv, ld_in, ld_out, E, dev, st)
                                                      : run_vec_for<E>(in, out, rv, cv, ld_in, ld_out, dev, st);
        if (rc) return rc;
    }
    return run_scalar_all<T>(in, out, rows, cols, rv, cv, ld_in, ld_out, dev, st);
}

}  // namespace

int launch_transpose(const void *in, void *out, int64_t rows, int64_t cols, int64_t ld_in,
                     int64_t ld_out, int esize, int dev, cudaStream_t st) {
    switch (esize) {
    case 1: return dispatch<uint8_t>(in, out, rows, cols, ld_in, ld_out, dev, st);
    case 2: return dispatch<uint16_t>(in, out, rows, cols, ld_in, ld_out, dev, st);
    case 4: return dispatch<uint32_t>(in, out, rows, cols, ld_in, ld_out, dev, st);
    case 8: return dispatch<uint64_t>(in, out, rows, cols, ld_in, ld_out, dev, st);
    default: return fail(B2_ERR_UNSUPPORTED, "transpose: unsupported element size");
    }
}

}  // namespace b2
