// Internal helpers shared by the sm_100a kernels and the C-ABI layer.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges cost a null check without a tool

#include "../../include/b2k.h"

namespace b2 {

// NVTX range around an ABI entry point (visible in ncu --nvtx / nsys timelines)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};
#define B2_NVTX(name) ::b2::NvtxRange b2_nvtx_range_(name)

// ---- error state (thread-local message, integer codes at the ABI) ----------
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
int cuda_fail(cudaError_t e, const char *what);

#define B2_CUDA(call)                                  \
    do {                                               \
        cudaError_t e_ = (call);                       \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int num_sms(int dev);

// Runtime tuning knobs (b2_tune_set); defaults are the tuned values.
struct Tuning {
    int t_variant = 0;      // transpose tile shape (see run_vec_for)
    int t_group = 0;        // tile-rows per band in the tile walk order (0 = auto)
    int t_big = 1;          // 1 = 128-KB tiles (1 CTA/SM) for large fp32/fp64 matrices, 2 = always
    int t_ctas_per_sm = 0;  // 0 = auto (~kInflightBytesPerSM of tiles per SM)
    int r_variant = 0;      // reduce <threads, unroll> instantiation
    int r_ctas_per_sm = 0;  // 0 = auto (kReduceThreadsPerSM threads per SM)
    int t_tma = 0;          // 1 = TMA-staged transpose for 4-byte cells (transpose_tma.cu)
    int t_any = 0;          // 1 = funnel-shifted 128-bit path for unaligned pitches, 0 = padded scalar tile
                            //     (measured: the scalar tile is faster, profiles/r01_odd.md)
    int t_scalar_ctas = 0;  // CTAs per SM of the padded scalar tile kernel (0 = auto)
    int h_chunk_mb = 64;    // host-pipeline chunk (MiB) for the *_host entry points
    int t_tma_stages = 2;   // input stages in flight per CTA (2, 3, 4, 6); 2 x 2 CTAs/SM measured best
    int t_scalar_tile = 0;  // padded scalar tile width: 0 = auto (2-byte 128, else 64), 64, 128 (2/4-byte)
    int r_spin_ms = 20000;  // fused combine: bounded wait per epoch before giving up (status word)
    int t_staged = 1;       // odd pitches / unaligned views: cp.async-staged kernel 1 = auto (2-byte cells
                            // from 2^22 cells, any width beyond 256 MB), 2 = always, 0 = never (scalar tile)
    int t_staged_ctas = 0;  // CTAs per SM of the staged kernel (0 = 2)
    int t_staged_stages = 4;  // cp.async ring depth of the staged kernel (2, 3, 4)
    int t_staged_geom = 0;  // staged kernel tile geometry (see staged_geom; 0 = auto by size)
    int c_pipe_kb = 65536;  // generated programs: bytes per copy / kernel pipeline step (KiB; 0 = off)
    int l_pdl = 0;          // 1 = launch the hot kernels with programmatic dependent launch
    int c_coarsen = 8;      // generated programs: largest thread-coarsening factor (1 = off; 8 only packed)
    int c_pack = 2;         // generated programs: most program blocks per CUDA block (1 = off)
    int t_cpa = 1;          // cp.async-loaded tiles for aligned transposes (transpose_cpa.cu): 1 = auto
                            // (large interiors), 2 = always (geometry t_cpa_variant), 0 = LDG path only
    int t_cpa_variant = 0;  // tile geometry of the forced cp.async path (see cpa_for)
    int t_cpa_ctas = 0;     // CTAs per SM of the cp.async path (0 = as many as fit)
    int t_cpa_hint = 1;     // cp.async L2 hint of the auto geometry: 1 = evict-first policy, 0 = none, 2 = 256-B prefetch
};
extern Tuning g_tune;
constexpr int kInflightBytesPerSM = 64 * 1024;
constexpr int kReduceThreadsPerSM = 1024;  // 2 x 512: best in the bench step (profiles/r01k_reduce_residency.md)

// ---- global memory access with explicit cache policy -----------------------
// Streaming 128-bit load that bypasses L1 (read-once data). No L2 prefetch-size
// hint: A/B on one B200 (profiles/r01j_ldst_variants.md) measured the .L2::256B
// hint 0.6-0.9 % slower for the transposes and neutral for the reduction.
#ifndef B2_LDG_QUAL
#define B2_LDG_QUAL "ld.global.nc.L1::no_allocate.v4.u32"
#endif
__device__ __forceinline__ uint4 ldg_stream(const uint4 *p) {
    uint4 r;
    asm volatile(B2_LDG_QUAL " {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// Streaming 128-bit store (the output is written once; no L1 allocation).
#ifndef B2_STG_QUAL
#define B2_STG_QUAL "st.global.L1::no_allocate.v4.u32"
#endif
__device__ __forceinline__ void stg_stream(uint4 *p, const uint4 &v) {
    asm volatile(B2_STG_QUAL " [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// ---- programmatic dependent launch (PDL) -----------------------------------
// With g_tune.l_pdl the hot kernels are launched with programmatic stream
// serialisation: a kernel's CTAs may be scheduled while its predecessor on the
// stream is still running. Every such kernel executes griddepcontrol.wait before
// its first memory access (no input is read before the predecessor has completed
// and flushed, whatever the predecessor was), then immediately allows its own
// dependents to be scheduled: what overlaps is the launch / CTA dispatch of the
// next kernel with the tail of this one, never data access.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_kernel(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                 Args... args) {
    if (!g_tune.l_pdl) {
        kernel<<<grid, block, smem, st>>>(args...);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, ((KArgs)args)...);
}

// ---- kernel launchers (defined in transpose.cu / reduce.cu) ---------------
int launch_transpose(const void *in, void *out, int64_t rows, int64_t cols, int64_t ld_in,
                     int64_t ld_out, int esize, int dev, cudaStream_t st);
int launch_transpose_tma(const void *in, void *out, int64_t rows, int64_t cols, int64_t ld_in,
                         int64_t ld_out, int dev, cudaStream_t st);
int launch_transpose_any(const void *in, void *out, int64_t rows, int64_t cols, int64_t ld_in,
                         int64_t ld_out, int esize, int dev, cudaStream_t st);
int launch_transpose_cpa(const void *in, void *out, int64_t rv, int64_t cv, int64_t ld_in, int64_t ld_out,
                         int esize, int dev, cudaStream_t st);
bool transpose_cpa_wanted(int64_t rv, int64_t cv, int esize, int dev);
int launch_transpose_staged(const void *in, void *out, int64_t rows, int64_t cols, int64_t ld_in,
                            int64_t ld_out, int esize, int dev, cudaStream_t st);

size_t reduce_ws_bytes(int64_t n, int dtype, int dev);
// Cross-GPU combine fused into the reduction's last CTA (reduce.cu): mailbox is a
// mailbox_bytes() region in rank 0's memory, mapped into every rank (CUDA IPC).
struct FusedCombine {
    void *mailbox = nullptr;  // nullptr: plain single-GPU reduction
    int rank = 0, nranks = 1;
    unsigned long long epoch = 0;  // 1, 2, 3, ... identical on every rank
    unsigned long long spin_ns = 0;  // bounded-wait limit (0: g_tune.r_spin_ms)
};
size_t mailbox_bytes();
// acc_out: write the raw accumulator (binary64 for fp32 cells) instead of the
// result type, for the library's own pipelines that combine several partials
int launch_reduce(const void *in, int64_t n, int dtype, void *out, void *ws, size_t ws_bytes,
                  int dev, cudaStream_t st, const FusedCombine &fz = FusedCombine(),
                  bool acc_out = false);
int launch_tree512(const float *in, int64_t n, float *partials, int dev, cudaStream_t st);
// the naive fp32 program's own order: *acc += in[0], in[1], ... in binary32 (one warp)
int launch_seq_sum_f32(const float *in, int64_t n, float *acc, int dev, cudaStream_t st);
// B-element tree blocks (power of two, 64..2048): the A.5 family
bool tree_block_supported(int block);
int launch_tree(const float *in, int64_t n, int block, float *partials, int dev, cudaStream_t st);

}  // namespace b2
