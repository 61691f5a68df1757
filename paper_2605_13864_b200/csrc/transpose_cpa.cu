// cp.async-loaded tiled transpose for sm_100a (16-B aligned bases and pitches).
//
// The same permutation as transpose_vec_kernel (transpose.cu; SURVEY A.1 / A.4,
// PAPER.md:1041-1068), with the load side moved off the register file: every
// 16-B chunk of a tile row (CH chunks: 256 B in the default geometry, a warp fetches
// 512 contiguous bytes per instruction) goes global -> shared with `cp.async.cg`
// (LDGSTS, optionally with an L2 evict-first cache policy) into an S-stage ring, so
// S - 1 tiles per CTA are in flight without holding a single register. Default (the
// C4 bench kernel): 256-row x 256-B tiles, 2 stages of 64 KB, 256 threads, 1 CTA/SM,
// evict-first loads for 4- / 8-byte cells (profiles/r02k_cpa.md).
//
//   * shared layout: input orientation, row i of the tile at i * CH chunks, chunk
//     k stored at slot k ^ ((i / R) & 7) (R = 8 rows, 4 for 8-byte cells). The
//     cp.async writes of a row are a permutation of its slots (conflict-free);
//   * stage-out: a warp unit is one chunk column x 64 tile rows; each lane gathers
//     the cells of one output row segment with scalar LDS at a constant stride (all
//     rows of a lane share one swizzle; the rows the warp reads at one instruction
//     hit distinct 16-B bank groups, see Lane below) and writes 32 B with one
//     256-bit L2-evict-first store (2-byte cells: two 16-B stores into two output
//     rows) — the LDG path's store side;
//   * one __syncthreads per tile (the paper's blocksync between the shared-tile
//     write and the transposed read) also frees the stage the next
//     cp.async group refills; persistent grid, column-major tile walk as in the
//     LDG path.
// Edge cells outside the V-multiple interior are left to the padded scalar tile
// (transpose.cu), exactly like the LDG path.
#include "b2_internal.cuh"

namespace b2 {
namespace {

template <int H>
__device__ __forceinline__ void cpa16(uint32_t saddr, const void *g, uint64_t pol) {
    if constexpr (H == 1)  // L2 evict-first policy (read-once input)
        asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "l"(pol)
                     : "memory");
    else if constexpr (H == 2)  // 256-B L2 prefetch
        asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
    else
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void lds64(uint32_t a, uint32_t &x, uint32_t &y) {
    asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(x), "=r"(y) : "r"(a));
}
// 256-bit store, L2 evict-first (the LDG path's stage-out store, transpose.cu)
__device__ __forceinline__ void stg256(uint8_t *p, const uint4 &a, const uint4 &b) {
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
                 "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
                 : "memory");
}

// Per cell width: a warp unit is one 16-B chunk column x 64 tile rows, and every lane
// assembles two 16-B output vectors from 8 (4-byte, 2-byte cells) or 4 (8-byte cells)
// shared loads:
//   4-byte: lane (cw = lane % 4, rg = lane / 4): cell column cw of rows rg*8 .. +7 ->
//           32 B of one output row (8 x LDS.32);
//   8-byte: lane (cw = lane % 2, rg = lane / 2): rows rg*4 .. +3 -> 32 B (4 x LDS.64);
//   2-byte: lane (cwp = lane % 4, rg = lane / 4): the 32-bit word cwp (cell columns
//           2 cwp, 2 cwp + 1) of rows rg*8 .. +7 -> two output rows of 16 B each
//           (8 x LDS.32, PRMT split).
// The lane's rows share one swizzle, and the rows a warp touches at one instruction
// hit distinct 16-B bank groups: swizzle period R = 8 rows (4 for 8-byte cells).
template <int E>
struct Lane {
    static constexpr int R = E == 8 ? 4 : 8;  // tile rows per lane = swizzle period
};

// TR input rows x CH 16-B chunks per tile; NT threads; S stages.
template <int E, int TR, int CH_, int NT, int S>
struct Cpa {
    static constexpr int V = 16 / E;
    static constexpr int CH = CH_;                // 16-B chunks per tile row (256 or 512 B)
    static constexpr int TC = CH * V;             // cells per tile row
    static constexpr int STAGE = TR * CH * 16;    // bytes per stage
    static constexpr int SMEM = S * STAGE;
    static constexpr int LOADS = TR * CH / NT;    // cp.async per thread per tile
    static constexpr int UNITS = CH * (TR / 64);  // warp units (chunk column x 64 rows) per tile
    static_assert(TR % 64 == 0 && (TR * CH) % NT == 0 && S >= 2 && CH % 8 == 0, "tile / thread mismatch");
};

template <int E, int TR, int CH_, int NT, int S, int H>
__global__ void __launch_bounds__(NT)
    transpose_cpa_kernel(const uint8_t *__restrict__ in, uint8_t *__restrict__ out, int64_t rows_v,
                         int64_t cols_v, int64_t ld_in_b, int64_t ld_out_b, int64_t tiles_r, int64_t tiles_c,
                         int64_t ntiles, int group) {
    using G = Cpa<E, TR, CH_, NT, S>;
    constexpr int V = G::V, CH = G::CH, TC = G::TC, NW = NT / 32, R = Lane<E>::R;
    extern __shared__ __align__(128) uint4 smem[];
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t pol = 0;
    if constexpr (H == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    pdl_enter();

    auto origin = [&](int64_t tile, int64_t &r0, int64_t &c0) {
        const int64_t per_band = (int64_t)group * tiles_c;
        const int64_t band = tile / per_band, w = tile - band * per_band;
        const int64_t rows_in_band = min((int64_t)group, tiles_r - band * group);
        r0 = (band * group + w % rows_in_band) * TR;
        c0 = (w / rows_in_band) * TC;
    };
    auto load = [&](int64_t tile, int stage) {
        int64_t r0, c0;
        origin(tile, r0, c0);
        const uint32_t st = sbase + (uint32_t)(stage * G::STAGE);
#pragma unroll
        for (int m = 0; m < G::LOADS; ++m) {
            const int idx = threadIdx.x + m * NT;
            const int i = idx / CH, k = idx % CH;  // a warp fetches 512 B of row runs
            const int64_t r = r0 + i, c = c0 + k * V;
            if (r < rows_v && c < cols_v)
                cpa16<H>(st + (uint32_t)((i * CH + (k ^ ((i / R) & 7))) * 16), in + r * ld_in_b + c * E, pol);
        }
    };

    int64_t t = blockIdx.x;
#pragma unroll
    for (int s = 0; s < S - 1; ++s) {
        const int64_t tl = t + (int64_t)s * gridDim.x;
        if (tl < ntiles) load(tl, s);
        cpa_commit();
    }
    const bool st256 = ((uintptr_t)out % 32 == 0) && (ld_out_b % 32 == 0);
    for (int it = 0; t < ntiles; t += gridDim.x, ++it) {
        cpa_wait<S - 2>();
        __syncthreads();  // tile `it` visible; the stage read in iteration it - 1 is free
        {
            const int64_t tl = t + (int64_t)(S - 1) * gridDim.x;
            if (tl < ntiles) load(tl, (it + S - 1) % S);
            cpa_commit();
        }
        int64_t r0, c0;
        origin(t, r0, c0);
        const uint32_t st = sbase + (uint32_t)((it % S) * G::STAGE);
#pragma unroll 2
        for (int u = warp; u < G::UNITS; u += NW) {  // UNITS / NW = 1-4
            const int kc = u % CH, rb = u / CH;
            if constexpr (E == 2) {
                const int cwp = lane & 3, i0 = rb * 64 + (lane >> 2) * 8;
                const uint32_t a = st + (uint32_t)((i0 * CH + (kc ^ ((i0 / R) & 7))) * 16 + cwp * 4);
                uint32_t w[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) w[k] = lds32(a + k * CH * 16);
                const uint4 lo = make_uint4(__byte_perm(w[0], w[1], 0x5410), __byte_perm(w[2], w[3], 0x5410),
                                            __byte_perm(w[4], w[5], 0x5410), __byte_perm(w[6], w[7], 0x5410));
                const uint4 hi = make_uint4(__byte_perm(w[0], w[1], 0x7632), __byte_perm(w[2], w[3], 0x7632),
                                            __byte_perm(w[4], w[5], 0x7632), __byte_perm(w[6], w[7], 0x7632));
                const int64_t oc = c0 + kc * V + 2 * cwp, orr = r0 + i0;  // oc + 1 < cols_v iff oc < cols_v
                if (oc < cols_v && orr < rows_v) {
                    stg_stream(reinterpret_cast<uint4 *>(out + oc * ld_out_b + orr * E), lo);
                    stg_stream(reinterpret_cast<uint4 *>(out + (oc + 1) * ld_out_b + orr * E), hi);
                }
            } else {
                const int cw = lane % V, i0 = rb * 64 + (lane / V) * R;
                const uint32_t a = st + (uint32_t)((i0 * CH + (kc ^ ((i0 / R) & 7))) * 16 + cw * E);
                uint4 p, q;
                if constexpr (E == 4) {
                    p = make_uint4(lds32(a), lds32(a + CH * 16), lds32(a + 2 * CH * 16), lds32(a + 3 * CH * 16));
                    q = make_uint4(lds32(a + 4 * CH * 16), lds32(a + 5 * CH * 16), lds32(a + 6 * CH * 16),
                                   lds32(a + 7 * CH * 16));
                } else {
                    lds64(a, p.x, p.y);
                    lds64(a + CH * 16, p.z, p.w);
                    lds64(a + 2 * CH * 16, q.x, q.y);
                    lds64(a + 3 * CH * 16, q.z, q.w);
                }
                const int64_t oc = c0 + kc * V + cw, orr = r0 + i0;  // output row / first column
                if (oc < cols_v && orr < rows_v) {
                    uint8_t *d = out + oc * ld_out_b + orr * E;
                    if (orr + V < rows_v) {
                        if (st256) stg256(d, p, q);
                        else {
                            stg_stream(reinterpret_cast<uint4 *>(d), p);
                            stg_stream(reinterpret_cast<uint4 *>(d + 16), q);
                        }
                    } else {
                        stg_stream(reinterpret_cast<uint4 *>(d), p);
                    }
                }
            }
        }
    }
    cpa_wait<0>();
}

template <int E, int TR, int CH, int NT, int S, int H>
int run_cpa(const void *in, void *out, int64_t rv, int64_t cv, int64_t ld_in, int64_t ld_out, int dev,
            cudaStream_t st) {
    using G = Cpa<E, TR, CH, NT, S>;
    const int64_t tiles_r = (rv + TR - 1) / TR, tiles_c = (cv + G::TC - 1) / G::TC;
    const int64_t ntiles = tiles_r * tiles_c;
    if (ntiles == 0) return B2_OK;
    auto kern = transpose_cpa_kernel<E, TR, CH, NT, S, H>;
    static std::atomic<int> occ[64];
    if (occ[dev] == 0) {
        if (G::SMEM > 48 * 1024)
            B2_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM));
        int o = 0;
        B2_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, NT, G::SMEM));
        occ[dev] = o > 0 ? o : 1;
    }
    const int per_sm = std::min(g_tune.t_cpa_ctas > 0 ? g_tune.t_cpa_ctas : occ[dev].load(), occ[dev].load());
    const int64_t grid = std::min<int64_t>(ntiles, (int64_t)num_sms(dev) * per_sm);
    // column-major tile walk at every size (unlike the LDG path's mid-size row bands:
    // with these 256-row tiles the column walk measured level or ahead everywhere,
    // 16384x32768 fp32 +1.8 %; profiles/r02m_shard_shapes.md)
    const int grp = g_tune.t_group > 0 ? g_tune.t_group : (int)std::min<int64_t>(tiles_r, 1 << 30);
    const int group = (int)std::max<int64_t>(1, std::min<int64_t>(grp, tiles_r));
    B2_CUDA(launch_kernel(kern, dim3((unsigned)grid), dim3(NT), G::SMEM, st, (const uint8_t *)in, (uint8_t *)out,
                          rv, cv, ld_in * E, ld_out * E, tiles_r, tiles_c, ntiles, group));
    count_launch();
    return B2_OK;
}

// Geometry. Auto (transpose.cpa = 1): 256 x 256-B tiles, 256 threads, 2 stages for 4-
// and 8-byte cells; 128 x 256-B tiles, 512 threads, 4 stages for 2-byte cells
// (profiles/r02k_cpa.md: two 64-KB stages, i.e. one tile loading while one drains,
// measured best for 4 / 8-byte cells, the ~64 KB in flight per SM of the LDG path's
// residency rule; 2-byte cells keep more in flight). The 4 / 8-byte loads carry an
// L2 evict-first policy (transpose.cpa_hint = 1, default: the input is read once; in
// the bench step that took the transpose + sum from 0.9 % behind the LDG path to
// 0.2-0.5 % ahead, the following reduction included); 0 = no hint, 2 = a 256-B L2
// prefetch hint (slower). transpose.cpa = 2 takes g_tune.t_cpa_variant (tile
// rows x row bytes, threads, stages; shared memory), with the evict-first hint (0-9):
//   0: 256 x 256 B, 512, 2 (128 KB)  1: 128 x 512 B, 512, 2 (128 KB)
//   2: 256 x 256 B, 256, 2 (128 KB)  3: 256 x 256 B, 1024, 2 (128 KB)
//   4: 384 x 256 B, 512, 2 (192 KB)  5: 128 x 256 B, 512, 4 (128 KB)
//   6: 512 x 128 B, 512, 2 (128 KB)  7: 448 x 256 B, 512, 2 (224 KB)
//   8: 256 x 256 B, 128, 2 (128 KB)  9: 192 x 256 B, 256, 2 (96 KB)
//   10 / 11: the auto geometry of the cell width without / with the evict-first hint
template <int E, int H>
int cpa_auto(const void *in, void *out, int64_t rv, int64_t cv, int64_t ld_in, int64_t ld_out, int dev,
             cudaStream_t st) {
    if constexpr (E == 2) return run_cpa<E, 128, 16, 512, 4, H>(in, out, rv, cv, ld_in, ld_out, dev, st);
    else return run_cpa<E, 256, 16, 256, 2, H>(in, out, rv, cv, ld_in, ld_out, dev, st);
}

template <int E>
int cpa_for(const void *in, void *out, int64_t rv, int64_t cv, int64_t ld_in, int64_t ld_out, int dev,
            cudaStream_t st) {
    if (g_tune.t_cpa != 2) {
        // the evict-first hint pays for 4 / 8-byte cells; the 2-byte geometry's four
        // stages measured 11 % slower with it (r02k_cpa.md), so 2-byte loads go unhinted
        if (g_tune.t_cpa_hint == 0 || E == 2) return cpa_auto<E, 0>(in, out, rv, cv, ld_in, ld_out, dev, st);
        if (g_tune.t_cpa_hint == 2) return cpa_auto<E, 2>(in, out, rv, cv, ld_in, ld_out, dev, st);
        return cpa_auto<E, 1>(in, out, rv, cv, ld_in, ld_out, dev, st);
    }
    switch (g_tune.t_cpa_variant) {
    case 1: return run_cpa<E, 128, 32, 512, 2, 1>(in, out, rv, cv, ld_in, ld_out, dev, st);
    case 2: return run_cpa<E, 256, 16, 256, 2, 1>(in, out, rv, cv, ld_in, ld_out, dev, st);
    case 3: return run_cpa<E, 256, 16, 1024, 2, 1>(in, out, rv, cv, ld_in, ld_out, dev, st);
    case 4: return run_cpa<E, 384, 16, 512, 2, 1>(in, out, rv, cv, ld_in, ld_out, dev, st);
    case 5: return run_cpa<E, 128, 16, 512, 4, 1>(in, out, rv, cv, ld_in, ld_out, dev, st);
    case 6: return run_cpa<E, 512, 8, 512, 2, 1>(in, out, rv, cv, ld_in, ld_out, dev, st);
    case 7: return run_cpa<E, 448, 16, 512, 2, 1>(in, out, rv, cv, ld_in, ld_out, dev, st);
    case 8: return run_cpa<E, 256, 16, 128, 2, 1>(in, out, rv, cv, ld_in, ld_out, dev, st);
    case 9: return run_cpa<E, 192, 16, 256, 2, 1>(in, out, rv, cv, ld_in, ld_out, dev, st);
    case 10: return cpa_auto<E, 0>(in, out, rv, cv, ld_in, ld_out, dev, st);  // auto geometry, no hint
    case 11: return cpa_auto<E, 1>(in, out, rv, cv, ld_in, ld_out, dev, st);  // auto geometry, evict-first
    default: return run_cpa<E, 256, 16, 512, 2, 1>(in, out, rv, cv, ld_in, ld_out, dev, st);
    }
}

}  // namespace

// Default dispatch (transpose.cpa = 1): the cp.async path takes aligned interiors
// whose input exceeds twice the 126-MB L2 (it measured level with or ahead of the LDG
// path there: fp32 32768^2 +0.6 %, 32000x32008 +1.5 %, bf16 32768x65536 +2.5 %;
// profiles/r02k_cpa.md) and that hold at least two tiles per SM; smaller ones (fp32
// 4096^2: -1.3 %; C1 1024^2: 64 tiles) keep the LDG path's tiles. transpose.cpa = 2
// forces it, 0 disables it.
bool transpose_cpa_wanted(int64_t rv, int64_t cv, int esize, int dev) {
    if (g_tune.t_cpa == 0) return false;
    if (g_tune.t_cpa == 2) return true;
    const int64_t tr = esize == 2 ? 128 : 256, tc = 256 / esize;  // auto tiles: rows x 256-B rows
    // 256 MB itself (fp32 8192^2, bf16 8192x16384) goes to the cp.async path for 2- / 4-byte
    // cells (+5 % / +1.4 %), not for 8-byte cells (fp64 4096x8192: -2.4 %; r02k_cpa_mid.jsonl)
    const int64_t bytes = rv * cv * esize, lim = int64_t(256) << 20;
    return (esize == 8 ? bytes > lim : bytes >= lim) && (rv / tr) * (cv / tc) >= 2 * (int64_t)num_sms(dev);
}

int launch_transpose_cpa(const void *in, void *out, int64_t rv, int64_t cv, int64_t ld_in, int64_t ld_out,
                         int esize, int dev, cudaStream_t st) {
    switch (esize) {
    case 2: return cpa_for<2>(in, out, rv, cv, ld_in, ld_out, dev, st);
    case 4: return cpa_for<4>(in, out, rv, cv, ld_in, ld_out, dev, st);
    case 8: return cpa_for<8>(in, out, rv, cv, ld_in, ld_out, dev, st);
    default: return fail(B2_ERR_UNSUPPORTED, "cp.async transpose: cell width must be 2, 4 or 8 bytes");
    }
}

}  // namespace b2
