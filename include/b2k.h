/*
 * b2k.h — C ABI of libb200k.so, the B200 (sm_100a) implementation of the two
 * OptiGPU hot-path programs: the tiled matrix transpose and the tree reduction.
 *
 * The reference (arXiv 2605.13864 artifact, /root/reference/pkg/src/minigpu) is
 * pure Python and has no FFI of its own: its only executable form of these
 * programs is the interpreter entry `run_program(program, entry, inputs)`
 * (interp.py:380-387) walking the DSL loop nests (interp.py:248-309). Each entry
 * point below replaces the part of that walk cited beside it; the Python package
 * paper_2605_13864_b200 binds them with ctypes behind a run_program-compatible
 * API (INTEGRATION.md shows the binding a minigpu maintainer would add).
 *
 * Conventions
 *   - Plain pointers and sizes only; no C++ or torch types cross this boundary.
 *   - "dev" functions take DEVICE pointers owned by the caller and a cudaStream_t
 *     passed as void* (NULL = legacy default stream). They are asynchronous.
 *   - "host" functions take HOST pointers (pinned or pageable), stage through
 *     library-owned device buffers with overlapped H2D / kernel / D2H, and return
 *     after the result is in host memory.
 *   - Sizes and pitches are in ELEMENTS, 64-bit. Return 0 on success, a B2_ERR_*
 *     code otherwise; b2_last_error() gives the calling thread's message.
 *   - The library never frees caller memory and never falls back to the CPU.
 */
#ifndef B2K_H
#define B2K_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define B2K_ABI_VERSION 1

#if defined(__GNUC__)
#define B2_API __attribute__((visibility("default")))
#else
#define B2_API
#endif

/* element types (interp cells are binary32 `float` or `int`, intrinsics.py:35;
 * bf16 / fp64 / 64-bit ints are carried as bit patterns) */
enum b2_dtype {
    B2_BF16 = 1,
    B2_F16 = 2,
    B2_F32 = 3,
    B2_F64 = 4,
    B2_I32 = 5,
    B2_I64 = 6,
    B2_U8 = 7,
    B2_U16 = 8,
    B2_U32 = 9,
    B2_U64 = 10
};

enum b2_status {
    B2_OK = 0,
    B2_ERR_INVALID = 1,     /* bad argument (InterpError-class at the Python layer) */
    B2_ERR_UNSUPPORTED = 2, /* dtype / alignment combination not implemented      */
    B2_ERR_CUDA = 3,        /* CUDA runtime error (message in b2_last_error)      */
    B2_ERR_NOMEM = 4        /* device or pinned allocation failed                 */
};

/* ---- library ------------------------------------------------------------- */
B2_API int b2_abi_version(void);
/* sha256 prefix (16 hex digits) of the csrc/ sources, include/b2k.h and the nvcc
 * flags this library was compiled from: the loader compares it with the tree it
 * runs from and refuses a stale build (mtimes are not trusted). */
B2_API const char *b2_build_id(void);
B2_API const char *b2_last_error(void);
B2_API int b2_device_count(int *count);
/* Number of kernels this library has launched in this process (evidence for the
 * bench's gpu_launches claim). */
B2_API uint64_t b2_launch_count(void);
B2_API size_t b2_dtype_size(int dtype);
/* Performance knobs (process-wide; the defaults are the tuned values):
 *   "transpose.cpa" cp.async-loaded tiles for large aligned matrices (1 = auto,
 *   2 = always, 0 = LDG tiles only), "transpose.cpa_variant" / "transpose.cpa_hint"
 *   / "transpose.cpa_ctas" (forced geometry, L2 load hint, CTAs per SM),
 *   "transpose.variant" LDG tile shape, "transpose.group" tile-rows per band of the
 *   tile walk, "transpose.ctas_per_sm", "transpose.staged" / "transpose.staged_geom" /
 *   "transpose.tma" / "transpose.any" alternative paths and geometries, "reduce.variant" <threads, loads in
 *   flight>, "reduce.ctas_per_sm" (0 = occupancy limit), "reduce.spin_ms"
 *   (bounded wait of the fused combine, default 20000), "host.chunk_mb" host
 *   pipeline stage, "codegen.pipe_kb" / "codegen.coarsen" / "codegen.pack"
 *   generated-program pipelining, coarsening and block packing, "launch.pdl".
 *   Results never depend on them. b2_tune_get returns -1 for an unknown key. */
B2_API int b2_tune_set(const char *key, int64_t value);
B2_API int64_t b2_tune_get(const char *key);

/* ---- transpose ------------------------------------------------------------
 * out[c][r] = in[r][c] for r < rows, c < cols; in has pitch ld_in, out has pitch
 * ld_out (elements). Bit-exact permutation for 1/2/4/8-byte elements.
 * Replaces: interp.py:282-300 executing the DSL nest
 *   `for x < W { for y < H { out[x][y] = in[y][x]; } }`
 *   and its GPU form (A.4, PAPER.md:586-618 / 1041-1068), with rows = H, cols = W. */
B2_API int b2_transpose(const void *in, void *out, int64_t rows, int64_t cols, int64_t ld_in,
                 int64_t ld_out, int dtype, int dev, void *stream);

/* Host-buffer form of b2_transpose: chunked, copy/compute-overlapped pipeline.
 * Replaces the host half of A.4: memcpy_host_to_device / device_to_host
 * (interp.py:353-365) around the kernel_launch scope (interp.py:334-347). */
B2_API int b2_transpose_host(const void *in_host, void *out_host, int64_t rows, int64_t cols,
                      int64_t ld_in, int64_t ld_out, int dtype, int dev);

/* ---- reduction ------------------------------------------------------------
 * Single-pass sum: vectorised grid-stride loads, warp shuffle tree, shared-memory
 * block tree with __syncthreads, last-block-done grid combine (deterministic).
 *   dtype B2_F32 -> *out is float   (order differs from the reference's
 *                                     sequential sum: tolerance, not bits)
 *   dtype B2_I32 -> *out is int64_t (exact == the reference's unbounded int sum)
 *   dtype B2_F64 -> *out is double
 *   dtype B2_I64 -> *out is a 16-byte two's-complement integer (little-endian;
 *                   128-bit accumulation: exact for any n, like Python ints).
 *                   Not available in the fused / multi-GPU combines (8-byte slots).
 * Replaces: interp.py:282-300 + :262-270 executing `for i < N { sum += arr[i]; }`
 *   (PAPER.md:155-172).
 * ws: device workspace of b2_reduce_ws_bytes(n, dtype) bytes, zero-filled before
 * first use and left zero-filled on return; ws == NULL uses a library-owned
 * per-device workspace (calls on one device must then be stream-ordered). */
B2_API size_t b2_reduce_ws_bytes(int64_t n, int dtype);
B2_API int b2_reduce_sum(const void *in, int64_t n, int dtype, void *out, void *ws, size_t ws_bytes,
                  int dev, void *stream);

/* Multi-GPU reduction with the cross-GPU combine fused into the kernel (SURVEY 8e
 * "fused variant"; replaces a separate NCCL reduce of the 8-byte partial). Rank 0
 * creates a mailbox in its memory and exports a 64-byte CUDA IPC handle; every
 * other rank opens it (peer-mapped over NVLink). In b2_reduce_sum_fused the last
 * CTA of rank g stores its partial into the mailbox and publishes it (system-scope
 * release); rank 0's last CTA waits for all ranks (acquire, bounded: 20 s) and
 * writes the rank-ordered sum to its *out. b2_mailbox_status returns the latest
 * epoch whose combine timed out (0 = never): a call with epoch e failed iff
 * status >= e, so one timeout does not poison later healthy epochs.
 * epoch = 1, 2, 3, ... must advance identically on every rank. */
B2_API int b2_mailbox_create(int dev, void **mailbox, void *ipc_handle64);
B2_API int b2_mailbox_open(const void *ipc_handle64, int dev, void **mailbox);
B2_API int b2_mailbox_close(void *mailbox, int dev, int owner);
B2_API int b2_mailbox_status(void *mailbox, int dev, uint64_t *status);
B2_API int b2_reduce_sum_fused(const void *in, int64_t n, int dtype, void *out, void *ws,
                               size_t ws_bytes, void *mailbox, int rank, int nranks,
                               uint64_t epoch, int dev, void *stream);

/* Host-buffer form of b2_reduce_sum; *out_host receives float / int64 / double /
 * 16-byte int (B2_I64), as b2_reduce_sum. */
B2_API int b2_reduce_sum_host(const void *in_host, int64_t n, int dtype, void *out_host, int dev);

/* The naive fp32 program A.2 in the reference's OWN order (interp.py:262-270, `sum +=
 * arr[i]`: one binary32 rounding per cell, i ascending) — bit-identical with the
 * reference interpreter, where b2_reduce_sum returns the correctly rounded sum. The
 * order is inherently sequential: one warp, ~4 cycles per cell. *acc (device float)
 * += in[0], ..., in[n - 1]; set it to 0 for a fresh sum, successive calls chain.
 * `in`: device pointer, 4-byte aligned. */
B2_API int b2_reduce_sum_seq_f32(const float *in, int64_t n, float *acc, int dev, void *stream);
/* Host-buffer form: chunked H2D, the chunks summed in order; *result_host receives it. */
B2_API int b2_reduce_sum_seq_f32_host(const float *in_host, int64_t n, float *result_host, int dev);

/* Appendix A.5 order: per 512-element block b,
 * s[t] = a[2t] + a[2t+1], then s[t] = s[t] + s[t + 2^(7-k)] for k = 0..7;
 * partials[b] = s[0]. Bit-identical to the reference interpreter's tree form.
 * Requires 512 | n (exact_div, interp.py:209-214), else B2_ERR_INVALID. */
B2_API int b2_reduce_tree512_partials(const float *in, int64_t n, float *partials, int dev,
                               void *stream);
/* Full A.5 program: partials on the device, memcpy_device_to_host, then the
 * program's host loop `sum += p[i]` in binary32 (bit-exact with the reference).
 * `in` is a device pointer; *result_host receives the float. Synchronous. */
B2_API int b2_reduce_tree512(const float *in, int64_t n, float *result_host, int dev, void *stream);

/* Host-buffer form of the A.5 program: chunked H2D of `in_host`, per-512 partials
 * on the device, D2H of the partials, sequential binary32 host sum. Bit-exact. */
B2_API int b2_reduce_tree512_host(const float *in_host, int64_t n, float *result_host, int dev);

/* The same three entries for the whole A.5 derivation family
 * (programs.reduce_tree_family: B-element blocks, B/2 threads, log2(B/2) halving
 * levels, s[t] = s[t] + s[t + h] for h = B/4 .. 1): `block` = B, a power of two in
 * 64..2048 (else B2_ERR_UNSUPPORTED). Requires block | n (exact_div). The *512
 * entries above are block = 512. */
B2_API int b2_reduce_tree_partials(const float *in, int64_t n, int block, float *partials, int dev,
                                   void *stream);
B2_API int b2_reduce_tree(const float *in, int64_t n, int block, float *result_host, int dev,
                          void *stream);
B2_API int b2_reduce_tree_host(const float *in_host, int64_t n, int block, float *result_host, int dev);

/* Synchronous bulk copies for generated host code (codegen.py), replacing the
 * interpreter's element-wise memcpy_host_to_device / memcpy_device_to_host
 * (interp.py:353-365): pinned host buffers go straight to the DMA engines,
 * pageable ones are staged through the pinned ring by the host copy pool.
 * Like cudaMemcpy they are ordered after the work already queued on the device's
 * legacy default stream (stream NULL), and return when the copy is complete. */
B2_API int b2_copy_h2d(void *dst_dev, const void *src_host, size_t bytes, int dev);
B2_API int b2_copy_d2h(void *dst_host, const void *src_dev, size_t bytes, int dev);
/* Caching device allocator for generated code's gmem_malloc / gmem_free
 * (intrinsics.py:107-161 gmem contracts): 2 MiB-rounded blocks reused across calls.
 * b2_device_free first waits for the legacy default stream (like cudaFree), so a
 * block is never handed out again while queued work still uses it; work the
 * caller queued on its own non-blocking streams must be synchronised first. */
B2_API int b2_device_alloc(size_t bytes, int dev, void **out);
B2_API int b2_device_free(void *ptr, int dev);

/* Chunked copy -> kernel -> copy pipeline for generated programs (
 * replaces the element-wise, strictly sequential memcpy_host_to_device / kernel /
 * memcpy_device_to_host of interp.py:330-377 + intrinsics.py:137-158 and the host
 * listing of). Step c = the H2D copies h2d[h2d_off[c] ..
 * h2d_off[c+1]) on the library's copy stream, then launch(ctx, c, stream) on its
 * compute stream once those copies have landed, then the D2H copies
 * d2h[d2h_off[c] .. d2h_off[c+1]) once that launch has finished. Consecutive steps
 * overlap: step c+1's H2D runs under step c's kernel and D2H, so both PCIe
 * directions stream at once. Each copy is a 2-D region (height rows of width
 * bytes; pitches in bytes); pageable host regions go through the pinned ring and
 * the host copy threads. Ordered after the legacy default stream; returns when
 * every step is complete (0, or the first launch / copy error). */
typedef struct {
    void *host;
    int64_t host_pitch;
    void *dev;
    int64_t dev_pitch;
    int64_t width;
    int64_t height;
} b2_copy2d;
typedef int (*b2_step_fn)(void *ctx, int step, void *stream);
B2_API int b2_pipe_run(int nsteps, const b2_copy2d *h2d, const int64_t *h2d_off, const b2_copy2d *d2h,
                       const int64_t *d2h_off, b2_step_fn launch, void *ctx, int dev);

/* ---- single-process multi-GPU ------------------------------
 * One host thread drives every GPU of the box. Shard g runs on the device that
 * owns its pointer, so the same call covers 1..8 GPUs (or several shards on one
 * GPU). Both calls order after each device's legacy default stream and return
 * when the work is complete.
 * b2_init: create the per-device contexts of devices 0..ndev-1 (ndev <= 0: all)
 *   and enable peer access between every pair that supports it. Optional: the
 *   multi calls initialise what they touch lazily.
 * b2_peer_access: 1 if kernels on `from` can load/store memory of `to`
 *   (enabling it if possible), else 0. */
B2_API int b2_init(int ndev);
B2_API int b2_peer_access(int from, int to);
/* Row-block sharded transpose: shard g is the rows[g] x cols block in[g] (pitch
 * ld_in[g]); its transpose goes to out[g] (cols x rows[g], pitch ld_out[g]), which
 * may live on another GPU (e.g. a column slab of one full W x H matrix: the
 * kernel's stores then cross NVLink). No exchange step.
 * Replaces the A.1 / A.4 nest over a partition of the y loop (interp.py:282-300). */
B2_API int b2_transpose_multi(const void *const *in, void *const *out, const int64_t *rows,
                              int64_t cols, const int64_t *ld_in, const int64_t *ld_out, int dtype,
                              int nshards);
/* Sharded sum: shard g (n[g] elements, device pointer) is reduced on its device;
 * the partials are combined in shard order inside the kernels over NVLink (each
 * shard's last CTA stores into the root's mailbox, root = shard 0's device; the
 * root's last CTA sums them) — or, without peer access, on the host in the same
 * order (identical bits). *host_out receives float / int64 / double as in
 * b2_reduce_sum. Replaces: `for i < N { sum += arr[i]; }` (A.2 / A.3) over
 * contiguous shards + one combine step. */
B2_API int b2_reduce_sum_multi(const void *const *shards, const int64_t *n, int nshards, int dtype,
                               void *host_out);

/* Block until all work this library queued on `stream` of `dev` is done. */
B2_API int b2_sync(int dev, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* B2K_H */
