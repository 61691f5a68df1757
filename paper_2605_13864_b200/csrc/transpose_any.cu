// Transpose for ANY alignment and pitch (odd dimensions, unaligned views) with
// 128-bit memory traffic on sm_100a — the C5 "non-square / odd-dimension" path.
//
// A 64x64-cell tile moves through three stages per CTA:
//   1. load: every tile row is covered by 16-B ALIGNED vectors (one lane per
//      vector); neighbouring lanes' vectors are funnel-shifted by the row's byte
//      misalignment (shfl + __funnelshift_r) so each lane holds V cells that start
//      exactly at its column; stored to an input-layout shared tile;
//   2. transpose: the register VxV micro-transpose of transpose.cu, written into
//      an output-layout tile XOR-swizzled at 16-B granularity (conflict-free);
//   3. store: every output row segment is written as 16-B ALIGNED vectors, each
//      funnel-shifted out of two shared vectors; the one or two vectors at the
//      ends of a segment that it shares with neighbouring tiles are written cell
//      by cell (masked), everything else with STG.128.
// Loads only touch aligned 16-B chunks that contain at least one cell of the
// row, so they never leave the row's allocation pages.
#include "b2_internal.cuh"

namespace b2 {
namespace {

constexpr int TS = 64;  // tile side in cells
constexpr int NT = 256;

// bytes [m, m + 16) of the 32-byte concatenation lo:hi (m even, 0..15)
__device__ __forceinline__ uint4 funnel16(const uint4 &lo, const uint4 &hi, int m) {
    const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    const int bs = (m & 3) * 8;
    uint32_t o[4];
    switch (m >> 2) {
#define B2_FUN(WS)                                                                  \
    case WS:                                                                        \
        _Pragma("unroll") for (int k = 0; k < 4; ++k) o[k] =                        \
            __funnelshift_r(w[WS + k], (WS + k + 1 < 8) ? w[WS + k + 1] : 0u, bs);  \
        break;
        B2_FUN(0) B2_FUN(1) B2_FUN(2) B2_FUN(3)
#undef B2_FUN
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
}

__device__ __forceinline__ uint4 shfl_down16(const uint4 &v, int d, int width) {
    return make_uint4(__shfl_down_sync(0xffffffffu, v.x, d, width),
                      __shfl_down_sync(0xffffffffu, v.y, d, width),
                      __shfl_down_sync(0xffffffffu, v.z, d, width),
                      __shfl_down_sync(0xffffffffu, v.w, d, width));
}

template <int E>
__device__ __forceinline__ void micro_t(uint4 (&v)[16 / E]);
template <>
__device__ __forceinline__ void micro_t<4>(uint4 (&v)[4]) {
    uint4 o[4];
    o[0] = make_uint4(v[0].x, v[1].x, v[2].x, v[3].x);
    o[1] = make_uint4(v[0].y, v[1].y, v[2].y, v[3].y);
    o[2] = make_uint4(v[0].z, v[1].z, v[2].z, v[3].z);
    o[3] = make_uint4(v[0].w, v[1].w, v[2].w, v[3].w);
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = o[i];
}
template <>
__device__ __forceinline__ void micro_t<8>(uint4 (&v)[2]) {
    const uint4 o0 = make_uint4(v[0].x, v[0].y, v[1].x, v[1].y);
    const uint4 o1 = make_uint4(v[0].z, v[0].w, v[1].z, v[1].w);
    v[0] = o0;
    v[1] = o1;
}
__device__ __forceinline__ uint32_t wsel(const uint4 &v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}
template <>
__device__ __forceinline__ void micro_t<2>(uint4 (&v)[8]) {
    uint4 o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t sel = (j & 1) ? 0x7632u : 0x5410u;
        uint32_t w[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) w[m] = __byte_perm(wsel(v[2 * m], j >> 1), wsel(v[2 * m + 1], j >> 1), sel);
        o[j] = make_uint4(w[0], w[1], w[2], w[3]);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = o[i];
}

template <int E>
__device__ __forceinline__ void store_cell(uint8_t *p, const uint4 &v, int k) {
    // cell k (E bytes) of the 16-B vector v
    const uint32_t w = wsel(v, (k * E) >> 2);
    if constexpr (E == 2) *reinterpret_cast<uint16_t *>(p) = (uint16_t)(w >> (((k * E) & 3) * 8));
    else if constexpr (E == 4) *reinterpret_cast<uint32_t *>(p) = w;
    else *reinterpret_cast<uint2 *>(p) = make_uint2(w, wsel(v, ((k * E) >> 2) + 1));
}

template <int E>
__global__ void __launch_bounds__(NT)
    transpose_any_kernel(const uint8_t *__restrict__ in, uint8_t *__restrict__ out, int64_t rows,
                         int64_t cols, int64_t ld_in, int64_t ld_out, int64_t tiles_c, int64_t ntiles) {
    constexpr int V = 16 / E;          // cells per vector
    constexpr int NV = TS * E / 16;    // vectors per tile row (8 / 16 / 32)
    constexpr int RPP = NT / NV;       // tile rows loaded per pass
    constexpr int LP = TS / RPP;       // load passes per tile
    constexpr int MTN = (TS / V) * (TS / V);                   // micro-tiles per tile
    constexpr int MT = MTN >= NT ? MTN / NT : 1;               // micro-tiles per thread
    extern __shared__ __align__(16) uint4 smem_any[];
    uint4 *tin = smem_any;              // [TS][NV] input layout
    uint4 *tout = smem_any + TS * NV;   // [TS][NV] output layout, swizzled

    const int g = threadIdx.x % NV;     // vector slot within a row
    const int rl = threadIdx.x / NV;    // row within a pass
    uint4 reg[LP];

    const int64_t ldiE = ld_in * E, ldoE = ld_out * E;
    auto load_tile = [&](int64_t tile) {
        const int64_t r0 = (tile / tiles_c) * TS, c0 = (tile % tiles_c) * TS;
        // per-tile base and extents; per row only a 64-bit multiply-add remains
        const uint8_t *tb = in + r0 * ldiE + c0 * E;
        const int seg = (int)(min(c0 + TS, cols) - c0) * E;  // valid bytes per row segment
        const int nrows = (int)min((int64_t)TS, rows - r0);
#pragma unroll
        for (int p = 0; p < LP; ++p) {
            const int r = p * RPP + rl;
            uint4 v = make_uint4(0, 0, 0, 0), nx = make_uint4(0, 0, 0, 0);
            int m = 0;
            if (r < nrows) {
                const uintptr_t a0 = reinterpret_cast<uintptr_t>(tb + r * ldiE);
                m = (int)(a0 & 15);
                const int rel = 16 * g - m;  // this lane's aligned vector, relative to a0
                const uintptr_t va = a0 - m + 16 * g;
                if (rel < seg) v = ldg_stream(reinterpret_cast<const uint4 *>(va));
                if (g == NV - 1 && rel + 16 < seg) nx = ldg_stream(reinterpret_cast<const uint4 *>(va + 16));
            }
            const uint4 up = shfl_down16(v, 1, NV);
            if (g != NV - 1) nx = up;
            reg[p] = m ? funnel16(v, nx, m) : v;
        }
    };

    int64_t tile = blockIdx.x;
    if (tile < ntiles) load_tile(tile);
    for (; tile < ntiles; tile += gridDim.x) {
        const int64_t r0 = (tile / tiles_c) * TS, c0 = (tile % tiles_c) * TS;
#pragma unroll
        for (int p = 0; p < LP; ++p) tin[(p * RPP + rl) * NV + g] = reg[p];
        __syncthreads();
        // register micro-transpose into the swizzled output-layout tile
#pragma unroll
        for (int t = 0; t < MT; ++t) {
            const int mt = threadIdx.x + t * NT;
            if (mt < MTN) {
                const int vc = mt % (TS / V), rg = mt / (TS / V);
                uint4 v[V];
#pragma unroll
                for (int k = 0; k < V; ++k) v[k] = tin[(rg * V + k) * NV + vc];
                micro_t<E>(v);
#pragma unroll
                for (int k = 0; k < V; ++k) {
                    const int o = vc * V + k;
                    tout[o * NV + (rg ^ ((o / V) & 7))] = v[k];
                }
            }
        }
        __syncthreads();
        const int64_t next = tile + gridDim.x;
        if (next < ntiles) load_tile(next);
        // store: aligned 16-B vectors per output row segment, masked at the ends.
        // NV lanes per output row; the (NV+1)-th vector of a misaligned segment is
        // taken by lane 0 of the row group as a second item.
        const uint8_t *ob = out + c0 * ldoE + r0 * E;
        const int oseg = (int)(min(r0 + TS, rows) - r0) * E;  // valid bytes per out row
        const int orows = (int)min((int64_t)TS, cols - c0);
        constexpr int RPI = NT / NV;                          // out rows per block iteration
#pragma unroll
        for (int it = 0; it < TS / RPI; ++it) {
            const int o = it * RPI + rl;
            if (o >= orows) continue;
            const uintptr_t b0 = reinterpret_cast<uintptr_t>(ob + o * ldoE);
            const int mo = (int)(b0 & 15);
            const int sw = (o / V) & 7;
#pragma unroll
            for (int pass = 0; pass < 2; ++pass) {
                const int gv = pass == 0 ? g : NV;
                if (pass == 1 && (g != 0 || mo == 0)) break;
                const int rel = 16 * gv - mo;  // vector start relative to b0
                if (rel >= oseg) continue;
                const uint4 zero = make_uint4(0, 0, 0, 0);
                const uint4 s1 = gv < NV ? tout[o * NV + (gv ^ sw)] : zero;
                uint4 w = s1;
                if (mo) {
                    const uint4 s0 = gv > 0 ? tout[o * NV + ((gv - 1) ^ sw)] : zero;
                    w = funnel16(s0, s1, 16 - mo);
                }
                uint8_t *va = reinterpret_cast<uint8_t *>(b0 - mo + 16 * gv);
                if (rel >= 0 && rel + 16 <= oseg) {
                    stg_stream(reinterpret_cast<uint4 *>(va), w);
                } else {
#pragma unroll
                    for (int k = 0; k < V; ++k) {
                        const int c = rel + k * E;
                        if (c >= 0 && c < oseg) store_cell<E>(va + k * E, w, k);
                    }
                }
            }
        }
    }
}

template <int E>
int run_any(const void *in, void *out, int64_t rows, int64_t cols, int64_t ld_in, int64_t ld_out,
            int dev, cudaStream_t st) {
    const int64_t tiles_r = (rows + TS - 1) / TS, tiles_c = (cols + TS - 1) / TS;
    const int64_t ntiles = tiles_r * tiles_c;
    if (ntiles == 0) return B2_OK;
    constexpr int smem = 2 * TS * TS * E;
    static std::atomic<int> occ[64];  // per-device cache (zero-initialised)
    if (occ[dev] == 0) {
        if (smem > 48 * 1024)
            B2_CUDA(cudaFuncSetAttribute(transpose_any_kernel<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        int o = 0;
        B2_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, transpose_any_kernel<E>, NT, smem));
        occ[dev] = o > 0 ? o : 1;
    }
    const int auto_sm = std::max(1, kInflightBytesPerSM / (TS * TS * E));
    const int per_sm = std::min(g_tune.t_ctas_per_sm > 0 ? g_tune.t_ctas_per_sm : auto_sm, occ[dev].load());
    const int64_t grid = std::min<int64_t>(ntiles, (int64_t)num_sms(dev) * per_sm);
    transpose_any_kernel<E><<<(unsigned)grid, NT, smem, st>>>((const uint8_t *)in, (uint8_t *)out, rows,
                                                              cols, ld_in, ld_out, tiles_c, ntiles);
    count_launch();
    B2_CUDA(cudaGetLastError());
    return B2_OK;
}

}  // namespace

int launch_transpose_any(const void *in, void *out, int64_t rows, int64_t cols, int64_t ld_in,
                         int64_t ld_out, int esize, int dev, cudaStream_t st) {
    switch (esize) {
    case 2: return run_any<2>(in, out, rows, cols, ld_in, ld_out, dev, st);
    case 4: return run_any<4>(in, out, rows, cols, ld_in, ld_out, dev, st);
    case 8: return run_any<8>(in, out, rows, cols, ld_in, ld_out, dev, st);
    default: return fail(B2_ERR_UNSUPPORTED, "transpose_any: element size must be 2, 4 or 8");
    }
}

}  // namespace b2
