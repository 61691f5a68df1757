// cp.async-staged transpose for odd pitches / unaligned views (any cell width,
// any alignment) on sm_100a — the C5 "non-square / odd-dimension" path.
//
// Why: with an odd row pitch every input row starts at a different 16-B phase,
// so neither 128-bit LDG nor TMA (16-B strides) can load a tile row as aligned
// vectors. The padded scalar tile (transpose.cu) moves one cell per instruction
// on both the load and the store side and keeps its loads in registers: for
// 2-byte cells it is latency-bound at ~3.6 TB/s (warps active 25 %, long-
// scoreboard stalls, profiles/r01p_small_sizes.md).
//
// Design: every tile row is fetched as the 16-B-ALIGNED superset of its cells
// with `cp.async.cg` (16 B per lane, straight from L2 into shared memory: no
// registers, no per-cell load instructions), into an S-stage ring so several
// tiles per CTA are in flight. Shared memory keeps each row's raw bytes in order,
// so cell (i, j) of the tile sits at row_base(i) + (phase(i) + j) * E: the
// transposed read is one LDS per cell at an address that advances by a constant,
// and the store is a coalesced warp-wide run of one output row (64 cells = one
// 128-B segment for 2-byte cells). Rows are placed at a rotation of ROT * (i / 8)
// 16-B slots so the 32 rows a warp reads at one column spread over the banks.
// Brute-forced over every odd pitch class, base phase and column (round 2): 2-byte
// cells ROT = 2 (1.5 wavefronts per LDS.U16, the best any rotation reaches); 4- and
// 8-byte cells ROT = 1 — conflict-free (1 wavefront per LDS.32, 2 per LDS.64, the
// minimum), where ROT = 2 had made every read exactly 2-way (ncu: 9.5 M conflicts of
// 24.7 M wavefronts on fp32 16385x16383).
//
// Loads only touch aligned 16-B chunks that contain at least one cell of the
// row, so they never leave the row's allocation pages.
#include "b2_internal.cuh"

namespace b2 {
namespace {

template <int H>
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void *g, uint64_t pol) {
    if constexpr (H == 1)  // L2 evict-first policy (read-once input)
        asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "l"(pol)
                     : "memory");
    else
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Tile = TR input rows x TC input cells; NT threads; S stages.
template <typename T, int TR, int TC, int NT, int S>
struct Staged {
    static constexpr int E = sizeof(T);
    static constexpr int V = 16 / E;                 // cells per 16-B chunk
    static constexpr int CH = TC / V + 1;            // chunks per staged row (phase < V)
    static constexpr int ROT = E == 2 ? 2 : 1;       // rotation step (slots) per 8 rows
    static constexpr int SLOTS = TR * CH + ROT * (TR / 8 - 1) + 1;  // per stage
    static constexpr int SMEM = S * SLOTS * 16;
    __device__ static __forceinline__ int row_slot(int i) { return i * CH + ROT * (i >> 3); }
};

template <typename T, int TR, int TC, int NT, int S, int H>
__global__ void __launch_bounds__(NT)
    transpose_staged_kernel(const T *__restrict__ in, T *__restrict__ out, int64_t rows, int64_t cols,
                            int64_t ld_in, int64_t ld_out, int64_t tiles_r, int64_t ntiles) {
    using G = Staged<T, TR, TC, NT, S>;
    constexpr int E = G::E, V = G::V, CH = G::CH;
    constexpr int NW = NT / 32;
    constexpr int RPL = TR / 32;  // tile rows per lane: a warp writes TR-cell output segments as RPL 32-lane runs
    static_assert(TR % 32 == 0, "tile rows must be a multiple of the warp width");
    extern __shared__ __align__(16) uint4 sm[];
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t pol = 0;
    if constexpr (H == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    pdl_enter();

    // column-major tile walk: concurrently processed tiles are vertical neighbours,
    // so their 128-B output segments of one output row are contiguous in HBM
    auto origin = [&](int64_t t, int64_t &r0, int64_t &c0) {
        r0 = (t % tiles_r) * TR;
        c0 = (t / tiles_r) * TC;
    };
    auto load = [&](int64_t t, int stage) {
        int64_t r0, c0;
        origin(t, r0, c0);
        const int ncols = (int)(cols - c0 < TC ? cols - c0 : TC);
        const uint32_t st_base = sbase + (uint32_t)(stage * G::SLOTS * 16);
        for (int idx = threadIdx.x; idx < TR * CH; idx += NT) {
            const int i = idx / CH, k = idx - i * CH;
            const int64_t r = r0 + i;
            if (r >= rows) break;  // idx grows with i: the rest of this thread's chunks are past the end too
            const uintptr_t ga = (uintptr_t)(in + r * ld_in + c0);
            const uintptr_t ab = ga & ~(uintptr_t)15;
            const int ph = (int)(ga - ab) / E;
            const int nch = (ph + ncols - 1) / V + 1;
            if (k < nch) cp_async16<H>(st_base + (uint32_t)((G::row_slot(i) + k) * 16), (const void *)(ab + 16 * k), pol);
        }
    };

    // prologue: the first S - 1 tiles of this CTA
    int64_t t = blockIdx.x;
#pragma unroll
    for (int s = 0; s < S - 1; ++s) {
        const int64_t tl = t + (int64_t)s * gridDim.x;
        if (tl < ntiles) load(tl, s);
        cp_async_commit();
    }
    for (int it = 0; t < ntiles; t += gridDim.x, ++it) {
        cp_async_wait<S - 2>();
        __syncthreads();  // tile `it` visible to all; stage (it - 1) % S free again
        {
            const int64_t tl = t + (int64_t)(S - 1) * gridDim.x;
            if (tl < ntiles) load(tl, (it + S - 1) % S);
            cp_async_commit();
        }
        int64_t r0, c0;
        origin(t, r0, c0);
        const int ncols = (int)(cols - c0 < TC ? cols - c0 : TC);
        const int nrows = (int)(rows - r0 < TR ? rows - r0 : TR);
        const char *stage = reinterpret_cast<const char *>(sm) + (size_t)(it % S) * G::SLOTS * 16;
        // this lane's tile rows (i = lane + 32 h): byte address of cell (i, j = 0). The
        // 32 rows one instruction reads are consecutive, so every h sees the bank
        // spread of row_slot's rotation (rows 32 h .. 32 h + 31 are rows 0 .. 31 shifted
        // by a constant number of slots)
        const char *src[RPL];
        bool ok[RPL];
#pragma unroll
        for (int h = 0; h < RPL; ++h) {
            const int i = lane + 32 * h;
            ok[h] = i < nrows;
            const uintptr_t ga = (uintptr_t)(in + (r0 + (ok[h] ? i : 0)) * ld_in + c0);
            src[h] = stage + G::row_slot(i) * 16 + (int)(ga & 15);
        }
        T *dst = out + c0 * ld_out + r0 + lane;
#pragma unroll 4
        for (int j = warp; j < ncols; j += NW) {
            T *d = dst + (int64_t)j * ld_out;
#pragma unroll
            for (int h = 0; h < RPL; ++h)
                if (ok[h]) d[32 * h] = *reinterpret_cast<const T *>(src[h] + j * E);
        }
    }
    cp_async_wait<0>();
}

template <typename T, int TC, int S, int TR = 64, int CTAS = 2, int H = 0>
int run_staged(const void *in, void *out, int64_t rows, int64_t cols, int64_t ld_in, int64_t ld_out,
               int dev, cudaStream_t st) {
    constexpr int NT = 256;
    using G = Staged<T, TR, TC, NT, S>;
    const int64_t tiles_r = (rows + TR - 1) / TR, tiles_c = (cols + TC - 1) / TC;
    const int64_t ntiles = tiles_r * tiles_c;
    if (ntiles == 0) return B2_OK;
    auto kern = transpose_staged_kernel<T, TR, TC, NT, S, H>;
    static std::atomic<int> occ[64];
    if (occ[dev] == 0) {
        if (G::SMEM > 48 * 1024)
            B2_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM));
        int o = 0;
        B2_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, NT, G::SMEM));
        occ[dev] = o > 0 ? o : 1;
    }
    const int want = g_tune.t_staged_ctas > 0 ? g_tune.t_staged_ctas : CTAS;
    const int per_sm = std::min(want, occ[dev].load());
    const int64_t grid = std::min<int64_t>(ntiles, (int64_t)num_sms(dev) * per_sm);
    B2_CUDA(launch_kernel(kern, dim3((unsigned)grid), dim3(NT), G::SMEM, st, (const T *)in, (T *)out, rows, cols,
                          ld_in, ld_out, tiles_r, ntiles));
    count_launch();
    return B2_OK;
}

// Tile geometries behind transpose.staged_geom (tile rows x 256-B rows, stages, CTAs
// per SM, L2 load hint): 1 = 256 rows, 2 stages, 1 CTA; 2 = 128 rows, 2 stages, 2
// CTAs; 3 = 1 + evict-first; 4 = 128 rows, 3 stages, 1 CTA; 5 = 2 + evict-first;
// 6 = 64 rows, t_staged_stages (4) x 2 CTAs. 0 = auto: geometry 2 for inputs beyond
// 256 MB (2x L2), else geometry 6 (profiles/r02s_odd_geom.md: 128-row tiles x 2
// stages x 2 CTAs measured +4..12 % on the large C5 odd shapes of every cell width,
// the 64-row ring stays ahead on mid sizes; the hint costs everywhere).
template <typename T, int TC>
int staged_geom(const void *in, void *out, int64_t rows, int64_t cols, int64_t ld_in, int64_t ld_out, int dev,
                cudaStream_t st) {
    int geom = g_tune.t_staged_geom;
    if (geom == 0) geom = rows * cols * (int64_t)sizeof(T) > (int64_t(256) << 20) ? 2 : 6;
    switch (geom) {
    case 1: return run_staged<T, TC, 2, 256, 1>(in, out, rows, cols, ld_in, ld_out, dev, st);
    case 2: return run_staged<T, TC, 2, 128, 2>(in, out, rows, cols, ld_in, ld_out, dev, st);
    case 3: return run_staged<T, TC, 2, 256, 1, 1>(in, out, rows, cols, ld_in, ld_out, dev, st);
    case 4: return run_staged<T, TC, 3, 128, 1>(in, out, rows, cols, ld_in, ld_out, dev, st);
    case 5: return run_staged<T, TC, 2, 128, 2, 1>(in, out, rows, cols, ld_in, ld_out, dev, st);
    default: break;
    }
    const int s = g_tune.t_staged_stages;
    if (s == 3) return run_staged<T, TC, 3>(in, out, rows, cols, ld_in, ld_out, dev, st);
    if (s == 2) return run_staged<T, TC, 2>(in, out, rows, cols, ld_in, ld_out, dev, st);
    return run_staged<T, TC, 4>(in, out, rows, cols, ld_in, ld_out, dev, st);
}

template <typename T>
int staged_for(const void *in, void *out, int64_t rows, int64_t cols, int64_t ld_in, int64_t ld_out,
               int dev, cudaStream_t st) {
    // 256-B input row runs: 128 cells of 2 bytes, 64 of 4, 32 of 8 (each staged row
    // 17 x 16 B with its alignment phase)
    return staged_geom<T, 256 / (int)sizeof(T)>(in, out, rows, cols, ld_in, ld_out, dev, st);
}

}  // namespace

int launch_transpose_staged(const void *in, void *out, int64_t rows, int64_t cols, int64_t ld_in,
                            int64_t ld_out, int esize, int dev, cudaStream_t st) {
    if ((uintptr_t)in % esize || (uintptr_t)out % esize)
        return fail(B2_ERR_UNSUPPORTED, "staged transpose: cells must be naturally aligned");
    switch (esize) {
    case 2: return staged_for<uint16_t>(in, out, rows, cols, ld_in, ld_out, dev, st);
    case 4: return staged_for<uint32_t>(in, out, rows, cols, ld_in, ld_out, dev, st);
    case 8: return staged_for<uint64_t>(in, out, rows, cols, ld_in, ld_out, dev, st);
    default: return fail(B2_ERR_UNSUPPORTED, "staged transpose: cell width must be 2, 4 or 8 bytes");
    }
}

}  // namespace b2
