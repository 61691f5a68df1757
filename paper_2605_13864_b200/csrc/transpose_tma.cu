// TMA-staged tiled transpose for sm_100a (4-byte cells).
//
// Same tile algebra as transpose_vec_kernel (transpose.cu), but both HBM
// directions are bulk tensor copies:
//   * TMA loads (cp.async.bulk.tensor.2d, 128-B swizzle) fill a ring of S input
//     stages of 64x64 cells (two 32-column boxes each), completion tracked by one
//     mbarrier per stage (expect_tx);
//   * each thread reads a 4x4 micro-tile with four LDS.128, transposes it in
//     registers and writes four STS.128 into a 128-B-swizzled output tile;
//     lanes of a quarter-warp walk a diagonal (row group i, chunk (i + s) % 8) so
//     both the LDS and the STS hit 8 distinct 16-B bank groups (conflict-free);
//   * fence.proxy.async, one __syncthreads, then thread 0 issues the TMA store of
//     the output tile (two boxes, bulk_group) and the TMA load that refills the
//     freed input stage; output tiles are double-buffered (wait_group.read 1).
// TMA clips out-of-range boxes, so ragged edges need no scalar strips; the only
// requirement is 16-B aligned bases and pitches.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "b2_internal.cuh"

namespace b2 {
namespace {

constexpr int kTile = 64;               // cells per tile side
constexpr int kBox = 32;                // cells per 128-B box row
constexpr int kStageBytes = kTile * kTile * 4;
constexpr int kBoxBytes = kStageBytes / 2;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int x, int y,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *map, const void *src, int x, int y) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(x), "r"(y), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int S>
__global__ void __launch_bounds__(256, 1)
    transpose_tma_kernel(const __grid_constant__ CUtensorMap tin,
                         const __grid_constant__ CUtensorMap tout, int64_t tiles_r,
                         int64_t tiles_c, int64_t ntiles, int group) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                ~uintptr_t(1023));
    uint8_t *in_buf = base;                      // S stages
    uint8_t *out_buf = base + S * kStageBytes;   // 2 output tiles
    __shared__ uint64_t full[S];
    const int tid = threadIdx.x;

    auto origin = [&](int64_t tile, int &r0, int &c0) {
        const int64_t per_band = (int64_t)group * tiles_c;
        const int64_t band = tile / per_band, w = tile - band * per_band;
        const int64_t rows_in_band = min((int64_t)group, tiles_r - band * group);
        r0 = (int)((band * group + w % rows_in_band) * kTile);
        c0 = (int)((w / rows_in_band) * kTile);
    };
    const int64_t my_n = blockIdx.x < ntiles ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    auto issue = [&](int64_t it) {
        int r0, c0;
        origin(blockIdx.x + it * gridDim.x, r0, c0);
        const int s = (int)(it % S);
        mbar_expect_tx(&full[s], kStageBytes);
        tma_load_2d(in_buf + s * kStageBytes, &tin, c0, r0, &full[s]);
        tma_load_2d(in_buf + s * kStageBytes + kBoxBytes, &tin, c0 + kBox, r0, &full[s]);
    };
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int64_t it = 0; it < min((int64_t)S, my_n); ++it) issue(it);
    }
    __syncthreads();

    // quarter-warp diagonal mapping (see header): row group rg, chunk c in box b
    const int q = tid >> 3, i = tid & 7;
    const int rg = i + 8 * (q & 1);
    const int b = (q >> 1) & 1;
    const int c = (i + (q >> 2)) & 7;
    const int vc = 8 * b + c;

    for (int64_t it = 0; it < my_n; ++it) {
        const int s = (int)(it % S);
        mbar_wait(&full[s], (uint32_t)((it / S) & 1));
        const int ob = (int)(it & 1);
        if (tid == 0) bulk_wait_read<1>();  // the store that last used out tile ob is done
        __syncthreads();
        const uint8_t *src = in_buf + s * kStageBytes + b * kBoxBytes;
        uint4 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int row = 4 * rg + k;
            v[k] = *reinterpret_cast<const uint4 *>(src + row * 128 + ((c ^ (row & 7)) << 4));
        }
        // 4x4 register transpose: v[k'] = out row 4*vc + k', in rows 4*rg .. 4*rg+3
        uint4 o[4];
        o[0] = make_uint4(v[0].x, v[1].x, v[2].x, v[3].x);
        o[1] = make_uint4(v[0].y, v[1].y, v[2].y, v[3].y);
        o[2] = make_uint4(v[0].z, v[1].z, v[2].z, v[3].z);
        o[3] = make_uint4(v[0].w, v[1].w, v[2].w, v[3].w);
        uint8_t *dst = out_buf + ob * kStageBytes + (rg >> 3) * kBoxBytes;
        const int oc = rg & 7;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int orow = 4 * vc + k;
            *reinterpret_cast<uint4 *>(dst + orow * 128 + ((oc ^ (orow & 7)) << 4)) = o[k];
        }
        fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            int r0, c0;
            origin(blockIdx.x + it * gridDim.x, r0, c0);
            tma_store_2d(&tout, out_buf + ob * kStageBytes, r0, c0);
            tma_store_2d(&tout, out_buf + ob * kStageBytes + kBoxBytes, r0 + kBox, c0);
            bulk_commit();
            if (it + S < my_n) issue(it + S);
        }
    }
    if (tid == 0) bulk_wait_all();
}

// ---------------------------------------------------------------------------
// TMA-loaded tiles, register transpose, direct 128-bit stores (transpose.tma = 2).
// Only the INPUT is staged in shared memory (S stages of TR x 128 fp32 cells,
// four 32-column 128B-swizzled boxes each), so up to 192 KB of tile data per SM
// is in flight through TMA. Lane l of a warp owns input rows 4l..4l+3 of one
// 4-column micro-column; its four LDS.128 are issued in a lane-rotated row order
// ((k + l/2) & 3) so every quarter-warp touches 8 distinct 16-B bank groups
// under the swizzle; after un-rotating and a 4x4 register transpose each lane
// stores 16 B to four output rows, a warp covering 512 contiguous bytes per row.
// One __syncthreads per tile releases the stage, then thread 0 refills it while
// the stores drain.
template <int TR, int S, int NB = 4>
__global__ void __launch_bounds__(512, 1)
    transpose_tmar_kernel(const __grid_constant__ CUtensorMap tin, uint8_t *__restrict__ out,
                          int64_t rows, int64_t cols, int64_t ld_out_b, int64_t tiles_r,
                          int64_t ntiles) {
    constexpr int TC = 32 * NB;                // input columns per tile (NB boxes of 32)
    constexpr int kBoxB = TR * 128;            // bytes per box
    constexpr int kStage = NB * kBoxB;
    constexpr int G = TR / 4;                  // row groups (4 input rows each) per tile
    constexpr int MPT = G * (TC / 4) / 512;    // micro-tiles per thread
    static_assert(G >= 16 && G % 16 == 0 && MPT >= 1, "the lane-rotated loads assume >= 16 row groups");
    extern __shared__ uint8_t smem_raw[];
    uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                ~uintptr_t(1023));
    __shared__ uint64_t full[S];
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t my_n = blockIdx.x < ntiles ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    auto origin = [&](int64_t it, int &r0, int &c0) {
        const int64_t t = blockIdx.x + it * gridDim.x;  // column-major tile walk
        r0 = (int)((t % tiles_r) * TR);
        c0 = (int)((t / tiles_r) * TC);
    };
    auto issue = [&](int64_t it) {
        int r0, c0;
        origin(it, r0, c0);
        const int st = (int)(it % S);
        mbar_expect_tx(&full[st], kStage);
#pragma unroll
        for (int b = 0; b < NB; ++b) tma_load_2d(base + st * kStage + b * kBoxB, &tin, c0 + 32 * b, r0, &full[st]);
    };
    if (tid == 0) {
        for (int s2 = 0; s2 < S; ++s2) mbar_init(&full[s2], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int64_t it = 0; it < min((int64_t)S, my_n); ++it) issue(it);
    }
    __syncthreads();
    const int rot = (lane >> 1) & 3;
    for (int64_t it = 0; it < my_n; ++it) {
        const int st = (int)(it % S);
        mbar_wait(&full[st], (uint32_t)((it / S) & 1));
        int r0, c0;
        origin(it, r0, c0);
        uint4 v[MPT][4];
#pragma unroll
        for (int q = 0; q < MPT; ++q) {
            const int p = tid + 512 * q;               // micro-tile: row group fastest
            const int g = p % G, m = p / G;            // row group, micro-column 0..31
            const uint8_t *box = base + st * kStage + (m >> 3) * kBoxB;
            const int cc = m & 7;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int row = 4 * g + ((k + rot) & 3);
                v[q][k] = *reinterpret_cast<const uint4 *>(box + row * 128 + ((cc ^ (row & 7)) << 4));
            }
        }
        __syncthreads();  // stage st fully read by every thread
        if (tid == 0 && it + S < my_n) issue(it + S);
#pragma unroll
        for (int q = 0; q < MPT; ++q) {
            // un-rotate: u[i] = v[(i - rot) & 3]
            uint4 u[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint4 a0 = v[q][i], a1 = v[q][(i + 3) & 3], a2 = v[q][(i + 2) & 3], a3 = v[q][(i + 1) & 3];
                u[i] = rot == 0 ? a0 : rot == 1 ? a1 : rot == 2 ? a2 : a3;
            }
            const int p = tid + 512 * q;
            const int g = p % G, m = p / G;
            const int64_t orow0 = (int64_t)c0 + 4 * m;   // output rows = input columns
            const int64_t ocol = (int64_t)r0 + 4 * g;    // output columns = input rows
            const uint4 o[4] = {make_uint4(u[0].x, u[1].x, u[2].x, u[3].x),
                                make_uint4(u[0].y, u[1].y, u[2].y, u[3].y),
                                make_uint4(u[0].z, u[1].z, u[2].z, u[3].z),
                                make_uint4(u[0].w, u[1].w, u[2].w, u[3].w)};
            if (ocol + 3 < rows) {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (orow0 + j < cols)
                        stg_stream(reinterpret_cast<uint4 *>(out + (orow0 + j) * ld_out_b + ocol * 4), o[j]);
            }
        }
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    // resolved once (thread-safe static initialisation); null if the driver lacks it
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        cudaGetLastError();
        return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    }();
    return fn;
}

int make_map(CUtensorMap *m, const void *ptr, int64_t inner, int64_t outer, int64_t pitch_bytes) {
    auto enc = encode_fn();
    if (!enc) return fail(B2_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    cuuint64_t strides[1] = {(cuuint64_t)pitch_bytes};
    cuuint32_t box[2] = {kBox, kTile};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(ptr), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(B2_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return B2_OK;
}

int make_map_box(CUtensorMap *m, const void *ptr, int64_t inner, int64_t outer, int64_t pitch_bytes,
                 int box_inner, int box_outer) {
    auto enc = encode_fn();
    if (!enc) return fail(B2_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    cuuint64_t strides[1] = {(cuuint64_t)pitch_bytes};
    cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void *>(ptr), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(B2_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return B2_OK;
}

template <int TR, int S, int NB = 4>
int run_tmar(const void *in, void *out, int64_t rows, int64_t cols, int64_t ld_in, int64_t ld_out, int dev,
             cudaStream_t st) {
    CUtensorMap tin;
    if (int rc = make_map_box(&tin, in, cols, rows, ld_in * 4, 32, TR)) return rc;
    const int64_t tiles_r = (rows + TR - 1) / TR, tiles_c = (cols + 32 * NB - 1) / (32 * NB);
    const int64_t ntiles = tiles_r * tiles_c;
    const int smem = S * NB * TR * 128 + 1024;
    static std::atomic<bool> attr[64];
    if (!attr[dev]) {
        B2_CUDA(cudaFuncSetAttribute(transpose_tmar_kernel<TR, S, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     smem));
        attr[dev] = true;
    }
    const int64_t grid = std::min<int64_t>(ntiles, (int64_t)num_sms(dev));
    transpose_tmar_kernel<TR, S, NB><<<(unsigned)grid, 512, smem, st>>>(tin, (uint8_t *)out, rows, cols,
                                                                         ld_out * 4, tiles_r, ntiles);
    count_launch();
    B2_CUDA(cudaGetLastError());
    return B2_OK;
}

template <int S>
int run_tma(const void *in, void *out, int64_t rows, int64_t cols, int64_t ld_in, int64_t ld_out,
            int dev, cudaStream_t st) {
    CUtensorMap tin, tout;
    if (int rc = make_map(&tin, in, cols, rows, ld_in * 4)) return rc;
    if (int rc = make_map(&tout, out, rows, cols, ld_out * 4)) return rc;
    const int64_t tiles_r = (rows + kTile - 1) / kTile, tiles_c = (cols + kTile - 1) / kTile;
    const int64_t ntiles = tiles_r * tiles_c;
    const int smem = (S + 2) * kStageBytes + 1024;
    static std::atomic<bool> attr[64];
    if (!attr[dev]) {
        B2_CUDA(cudaFuncSetAttribute(transpose_tma_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr[dev] = true;
    }
    // 2 CTAs x 2 stages per SM (64 KB of tiles in flight) measured best on B200
    // (profiles/r01_tma.md); deeper rings in one CTA serialise on its barriers.
    const int per_sm = g_tune.t_ctas_per_sm > 0 ? g_tune.t_ctas_per_sm : 2;
    const int64_t grid = std::min<int64_t>(ntiles, (int64_t)num_sms(dev) * per_sm);
    const int group = (int)std::max<int64_t>(1, std::min<int64_t>(g_tune.t_group, tiles_r));
    transpose_tma_kernel<S><<<(unsigned)grid, 256, smem, st>>>(tin, tout, tiles_r, tiles_c, ntiles, group);
    count_launch();
    B2_CUDA(cudaGetLastError());
    return B2_OK;
}

}  // namespace

// 4-byte cells, 16-B aligned bases and pitches (else B2_ERR_UNSUPPORTED).
int launch_transpose_tma(const void *in, void *out, int64_t rows, int64_t cols, int64_t ld_in,
                         int64_t ld_out, int dev, cudaStream_t st) {
    if ((uintptr_t)in % 16 || (uintptr_t)out % 16 || (ld_in * 4) % 16 || (ld_out * 4) % 16 ||
        rows >= (1ll << 31) || cols >= (1ll << 31))
        return fail(B2_ERR_UNSUPPORTED, "TMA transpose needs 16-B aligned bases and pitches");
    if (g_tune.t_tma == 2) {  // TMA loads + register transpose + direct stores
        if (rows % 4 || cols % 4) return fail(B2_ERR_UNSUPPORTED, "tmar: rows and cols must be multiples of 4");
        switch (g_tune.t_tma_stages) {
        case 2: return run_tmar<128, 2>(in, out, rows, cols, ld_in, ld_out, dev, st);
        case 4: return run_tmar<64, 4>(in, out, rows, cols, ld_in, ld_out, dev, st);
        case 6: return run_tmar<64, 6>(in, out, rows, cols, ld_in, ld_out, dev, st);
        case 7: return run_tmar<256, 3, 2>(in, out, rows, cols, ld_in, ld_out, dev, st);  // 256 x 64 tiles
        case 8: return run_tmar<256, 2, 2>(in, out, rows, cols, ld_in, ld_out, dev, st);
        default: return run_tmar<128, 3>(in, out, rows, cols, ld_in, ld_out, dev, st);
        }
    }
    switch (g_tune.t_tma_stages) {
    case 2: return run_tma<2>(in, out, rows, cols, ld_in, ld_out, dev, st);
    case 3: return run_tma<3>(in, out, rows, cols, ld_in, ld_out, dev, st);
    case 6: return run_tma<6>(in, out, rows, cols, ld_in, ld_out, dev, st);
    default: return run_tma<4>(in, out, rows, cols, ld_in, ld_out, dev, st);
    }
}

}  // namespace b2
