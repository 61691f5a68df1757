// C ABI of libb200k.so (include/b2k.h): argument validation, per-device context
// (streams, staging buffers, default reduce workspace), and the host-buffer
// pipelines that overlap H2D copy, kernel and D2H copy chunk by chunk.
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <unordered_map>
#include <string>
#include <thread>
#include <vector>

#include "b2_internal.cuh"

namespace b2 {

static thread_local std::string t_err;
std::atomic<uint64_t> g_launches{0};
Tuning g_tune;

void set_error(const std::string &msg) { t_err = msg; }
int fail(int code, const std::string &msg) {
    t_err = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char *what) {
    t_err = std::string(what) + ": " + cudaGetErrorName(e) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? B2_ERR_NOMEM : B2_ERR_CUDA;
}

static std::atomic<int> g_sms[64];  // per-device SM count cache
int num_sms(int dev) {
    if (dev < 0 || dev >= 64) return 148;
    if (g_sms[dev] == 0) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
            n = 148;
        g_sms[dev] = n;
    }
    return g_sms[dev];
}

// ---------------------------------------------------------------- device context
namespace {

constexpr int kStages = 3;

struct DevCtx {
    std::mutex mu;
    bool ready = false;
    cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
    cudaEvent_t ev_in[kStages], ev_comp[kStages], ev_out[kStages];
    cudaEvent_t ev_legacy = nullptr;  // orders bulk copies after the legacy default stream
    void *d_in[kStages] = {nullptr, nullptr, nullptr};
    void *d_out[kStages] = {nullptr, nullptr, nullptr};
    size_t stage_bytes = 0;
    void *ws = nullptr;  // default reduce workspace lent to ws == NULL callers (their streams)
    size_t ws_bytes = 0;
    void *ws_pipe = nullptr;  // the library's own: host pipelines and *_multi on s_comp
                              // (never shared with callers' streams: no ticket races)
    void *d_small = nullptr;  // per-chunk results / tree partials
    size_t small_bytes = 0;
    void *h_small = nullptr;  // pinned mirror of d_small
    void *hs_in[kStages] = {nullptr, nullptr, nullptr};   // pinned staging (pageable sources)
    void *hs_out[kStages] = {nullptr, nullptr, nullptr};  // pinned staging (pageable destinations)
    size_t hs_bytes = 0;
    // single-process multi-GPU entries (b2_*_multi): per-shard result slots, and the
    // fused-combine mailbox when this device is the root
    void *d_slots = nullptr;  // kMaxShards x 8 B
    void *h_slots = nullptr;  // pinned mirror
    void *mailbox = nullptr;
    unsigned long long mb_epoch = 0;
};

// Per device: kLanes independent pipeline contexts ("lanes": streams, events, stage
// buffers, workspace). Lane 0 also owns the device-wide state (the workspace lent to
// ws == NULL callers, the multi-GPU slots and mailbox); the host-buffer pipelines take
// any free lane, so concurrent calls from several host threads (a transpose and a
// reduction) overlap their PCIe traffic instead of serialising on one context.
constexpr int kLanes = 2;
DevCtx g_lanes[64][kLanes];
inline DevCtx &g_ctx_of(int dev) { return g_lanes[dev][0]; }  // lane 0: device-wide state

struct Lane {
    DevCtx *c;
    std::unique_lock<std::mutex> lock;
};
Lane acquire_lane(int dev) {
    for (int i = 0; i < kLanes; ++i) {
        std::unique_lock<std::mutex> l(g_lanes[dev][i].mu, std::try_to_lock);
        if (l.owns_lock()) return {&g_lanes[dev][i], std::move(l)};
    }
    return {&g_lanes[dev][0], std::unique_lock<std::mutex>(g_lanes[dev][0].mu)};
}

int check_dev(int dev) {
    static std::atomic<int> s_count{-1};
    int n = s_count.load(std::memory_order_relaxed);
    if (n < 0) {
        B2_CUDA(cudaGetDeviceCount(&n));
        s_count.store(n, std::memory_order_relaxed);
    }
    if (dev < 0 || dev >= n || dev >= 64)
        return fail(B2_ERR_INVALID, "device " + std::to_string(dev) + " out of range (have " +
                                        std::to_string(n) + ")");
    // cudaSetDevice is per host thread; skip it when this thread is already there
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != dev) B2_CUDA(cudaSetDevice(dev));
    return B2_OK;
}

int ctx_init(DevCtx &c, int dev) {
    if (c.ready) return B2_OK;
    B2_CUDA(cudaStreamCreateWithFlags(&c.s_h2d, cudaStreamNonBlocking));
    B2_CUDA(cudaStreamCreateWithFlags(&c.s_comp, cudaStreamNonBlocking));
    B2_CUDA(cudaStreamCreateWithFlags(&c.s_d2h, cudaStreamNonBlocking));
    for (int k = 0; k < kStages; ++k) {
        B2_CUDA(cudaEventCreateWithFlags(&c.ev_in[k], cudaEventDisableTiming));
        B2_CUDA(cudaEventCreateWithFlags(&c.ev_comp[k], cudaEventDisableTiming));
        B2_CUDA(cudaEventCreateWithFlags(&c.ev_out[k], cudaEventDisableTiming));
    }
    B2_CUDA(cudaEventCreateWithFlags(&c.ev_legacy, cudaEventDisableTiming));
    c.ws_bytes = reduce_ws_bytes(0, B2_I64, dev);  // the widest partial (128-bit int64 sums)
    B2_CUDA(cudaMalloc(&c.ws, c.ws_bytes));
    B2_CUDA(cudaMemset(c.ws, 0, c.ws_bytes));
    B2_CUDA(cudaMalloc(&c.ws_pipe, c.ws_bytes));
    B2_CUDA(cudaMemset(c.ws_pipe, 0, c.ws_bytes));
    c.ready = true;
    return B2_OK;
}

int ensure_stages(DevCtx &c, size_t bytes) {
    if (c.stage_bytes >= bytes) return B2_OK;
    B2_CUDA(cudaStreamSynchronize(c.s_h2d));
    B2_CUDA(cudaStreamSynchronize(c.s_comp));
    B2_CUDA(cudaStreamSynchronize(c.s_d2h));
    for (int k = 0; k < kStages; ++k) {
        if (c.d_in[k]) cudaFree(c.d_in[k]);
        if (c.d_out[k]) cudaFree(c.d_out[k]);
        c.d_in[k] = c.d_out[k] = nullptr;
    }
    c.stage_bytes = 0;
    for (int k = 0; k < kStages; ++k) {
        B2_CUDA(cudaMalloc(&c.d_in[k], bytes));
        B2_CUDA(cudaMalloc(&c.d_out[k], bytes));
    }
    c.stage_bytes = bytes;
    return B2_OK;
}

int ensure_host_stages(DevCtx &c, size_t bytes) {
    if (c.hs_bytes >= bytes) return B2_OK;
    B2_CUDA(cudaStreamSynchronize(c.s_h2d));
    B2_CUDA(cudaStreamSynchronize(c.s_d2h));
    for (int k = 0; k < kStages; ++k) {
        if (c.hs_in[k]) cudaFreeHost(c.hs_in[k]);
        if (c.hs_out[k]) cudaFreeHost(c.hs_out[k]);
        c.hs_in[k] = c.hs_out[k] = nullptr;
    }
    c.hs_bytes = 0;
    for (int k = 0; k < kStages; ++k) {
        B2_CUDA(cudaMallocHost(&c.hs_in[k], bytes));
        B2_CUDA(cudaMallocHost(&c.hs_out[k], bytes));
    }
    c.hs_bytes = bytes;
    return B2_OK;
}

void par_copy2d(void *dst, size_t dpitch, const void *src, size_t spitch, size_t width, size_t height);

// H2D of `height` host rows (`width` bytes, pitch `spitch`) into contiguous device
// memory on c.s_h2d, staged through c.hs_in[k] when the source is pageable.
int h2d_rows(DevCtx &c, int k, bool staged, void *dst, const char *src, size_t spitch, size_t width,
             size_t height) {
    if (!staged) {
        B2_CUDA(cudaMemcpy2DAsync(dst, width, src, spitch, width, height, cudaMemcpyHostToDevice, c.s_h2d));
        return B2_OK;
    }
    B2_CUDA(cudaEventSynchronize(c.ev_in[k]));  // the DMA that last read hs_in[k] is done
    par_copy2d(c.hs_in[k], width, src, spitch, width, height);
    B2_CUDA(cudaMemcpyAsync(dst, c.hs_in[k], width * height, cudaMemcpyHostToDevice, c.s_h2d));
    return B2_OK;
}

int ensure_small(DevCtx &c, size_t bytes) {
    if (c.small_bytes >= bytes) return B2_OK;
    if (c.d_small) cudaFree(c.d_small);
    if (c.h_small) cudaFreeHost(c.h_small);
    c.d_small = c.h_small = nullptr;
    c.small_bytes = 0;
    B2_CUDA(cudaMalloc(&c.d_small, bytes));
    B2_CUDA(cudaMallocHost(&c.h_small, bytes));
    c.small_bytes = bytes;
    return B2_OK;
}

int esize_of(int dtype) { return (int)b2_dtype_size(dtype); }

// ------------------------------------------------ staged copies for pageable host memory
// The DMA engines only stream pinned memory at PCIe speed (55 GB/s measured on the
// B200 box vs 29 / 18 GB/s H2D / D2H from pageable memory, profiles/r01_e2e_chunks.json).
// Pageable buffers are therefore staged through pinned chunks by a small pool of host
// threads, overlapped with the DMA of the neighbouring chunk.
class CopyPool {
  public:
    explicit CopyPool(int n) {
        for (int i = 0; i < n; ++i) th_.emplace_back([this, i] { loop(i + 1); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto &t : th_) t.join();
    }
    int size() const { return (int)th_.size() + 1; }
    // run f(part) for part in [0, size()); the caller runs part 0. One job at a time:
    // concurrent submitters (pipelines on several lanes / devices) queue here.
    void run(const std::function<void(int)> &f) {
        std::lock_guard<std::mutex> one(submit_);
        {
            std::lock_guard<std::mutex> g(m_);
            job_ = &f;
            pending_ = (int)th_.size();
            ++gen_;
        }
        cv_.notify_all();
        f(0);
        std::unique_lock<std::mutex> l(m_);
        done_.wait(l, [this] { return pending_ == 0; });
        job_ = nullptr;
    }

  private:
    void loop(int part) {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(int)> *job;
            {
                std::unique_lock<std::mutex> l(m_);
                cv_.wait(l, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                job = job_;
            }
            (*job)(part);
            {
                std::lock_guard<std::mutex> g(m_);
                if (--pending_ == 0) done_.notify_one();
            }
        }
    }
    std::vector<std::thread> th_;
    std::mutex submit_, m_;
    std::condition_variable cv_, done_;
    const std::function<void(int)> *job_ = nullptr;
    int pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

CopyPool &copy_pool() {
    // host threads for pageable staging copies (incl. the caller): B2K_COPY_THREADS,
    // else every hardware thread up to 32 — the copies are host-memory-bound and the
    // caller is blocked anyway (pageable e2e on the 16-thread box: 8 threads 33 GB/s,
    // 16 threads 42 GB/s; profiles/r01i_pcie.md)
    static CopyPool *p = [] {
        int n = std::max(1, std::min(32, (int)std::thread::hardware_concurrency()));
        const char *e = getenv("B2K_COPY_THREADS");
        if (e && *e) n = std::max(1, std::min(64, atoi(e)));
        return new CopyPool(n - 1);
    }();
    return *p;
}

// rows of `width` bytes, pitches in bytes, copied by all pool threads
void par_copy2d(void *dst, size_t dpitch, const void *src, size_t spitch, size_t width, size_t height) {
    CopyPool &pool = copy_pool();
    const int parts = pool.size();
    if (height == 1 || (dpitch == width && spitch == width)) {  // contiguous: split bytes
        const size_t total = width * height, step = (total + parts - 1) / parts;
        pool.run([&](int p) {
            const size_t b = std::min(total, p * step), e = std::min(total, b + step);
            if (e > b) memcpy((char *)dst + b, (const char *)src + b, e - b);
        });
        return;
    }
    const size_t step = (height + parts - 1) / parts;
    pool.run([&](int p) {
        const size_t b = std::min(height, p * step), e = std::min(height, b + step);
        for (size_t r = b; r < e; ++r) memcpy((char *)dst + r * dpitch, (const char *)src + r * spitch, width);
    });
}

bool is_pinned(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// host-pipeline stage size (b2_tune_set("host.chunk_mb", ...))
inline size_t chunk_bytes() { return size_t(g_tune.h_chunk_mb > 0 ? g_tune.h_chunk_mb : 64) << 20; }

}  // namespace
}  // namespace b2

using namespace b2;

extern "C" {

int b2_abi_version(void) { return B2K_ABI_VERSION; }

#ifndef B2_BUILD_ID
#define B2_BUILD_ID "unknown"
#endif
const char *b2_build_id(void) { return B2_BUILD_ID; }

const char *b2_last_error(void) { return t_err.c_str(); }

uint64_t b2_launch_count(void) { return g_launches.load(); }

static int *tune_slot(const char *key) {
    if (!key) return nullptr;
    const std::string k(key);
    if (k == "transpose.variant") return &g_tune.t_variant;
    if (k == "transpose.group") return &g_tune.t_group;
    if (k == "transpose.big") return &g_tune.t_big;
    if (k == "transpose.ctas_per_sm") return &g_tune.t_ctas_per_sm;
    if (k == "reduce.variant") return &g_tune.r_variant;
    if (k == "reduce.ctas_per_sm") return &g_tune.r_ctas_per_sm;
    if (k == "transpose.tma") return &g_tune.t_tma;
    if (k == "transpose.any") return &g_tune.t_any;
    if (k == "transpose.scalar_ctas") return &g_tune.t_scalar_ctas;
    if (k == "transpose.tma_stages") return &g_tune.t_tma_stages;
    if (k == "transpose.scalar_tile") return &g_tune.t_scalar_tile;
    if (k == "host.chunk_mb") return &g_tune.h_chunk_mb;
    if (k == "reduce.spin_ms") return &g_tune.r_spin_ms;
    if (k == "transpose.staged") return &g_tune.t_staged;
    if (k == "codegen.pipe_kb") return &g_tune.c_pipe_kb;
    if (k == "launch.pdl") return &g_tune.l_pdl;
    if (k == "codegen.coarsen") return &g_tune.c_coarsen;
    if (k == "codegen.pack") return &g_tune.c_pack;
    if (k == "transpose.staged_ctas") return &g_tune.t_staged_ctas;
    if (k == "transpose.staged_stages") return &g_tune.t_staged_stages;
    if (k == "transpose.staged_geom") return &g_tune.t_staged_geom;
    if (k == "transpose.cpa") return &g_tune.t_cpa;
    if (k == "transpose.cpa_variant") return &g_tune.t_cpa_variant;
    if (k == "transpose.cpa_ctas") return &g_tune.t_cpa_ctas;
    if (k == "transpose.cpa_hint") return &g_tune.t_cpa_hint;
    return nullptr;
}

int b2_tune_set(const char *key, int64_t value) {
    int *slot = tune_slot(key);
    if (!slot) return fail(B2_ERR_INVALID, std::string("unknown tuning key ") + (key ? key : "(null)"));
    if (value < 0 || value > 1 << 20) return fail(B2_ERR_INVALID, "tuning value out of range");
    *slot = (int)value;
    return B2_OK;
}

int64_t b2_tune_get(const char *key) {
    int *slot = tune_slot(key);
    return slot ? *slot : -1;
}

int b2_device_count(int *count) {
    if (!count) return fail(B2_ERR_INVALID, "count is NULL");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        *count = 0;
        return cuda_fail(e, "cudaGetDeviceCount");
    }
    *count = n;
    return B2_OK;
}

size_t b2_dtype_size(int dtype) {
    switch (dtype) {
    case B2_U8: return 1;
    case B2_BF16: case B2_F16: case B2_U16: return 2;
    case B2_F32: case B2_I32: case B2_U32: return 4;
    case B2_F64: case B2_I64: case B2_U64: return 8;
    default: return 0;
    }
}

int b2_transpose(const void *in, void *out, int64_t rows, int64_t cols, int64_t ld_in,
                 int64_t ld_out, int dtype, int dev, void *stream) {
    B2_NVTX("b2_transpose");
    const int E = esize_of(dtype);
    if (!E) return fail(B2_ERR_UNSUPPORTED, "transpose: unknown dtype " + std::to_string(dtype));
    if (rows < 0 || cols < 0) return fail(B2_ERR_INVALID, "transpose: negative extent");
    if (rows == 0 || cols == 0) return B2_OK;
    if (!in || !out) return fail(B2_ERR_INVALID, "transpose: NULL buffer");
    if (ld_in < cols || ld_out < rows)
        return fail(B2_ERR_INVALID, "transpose: pitch smaller than row length");
    if (int rc = check_dev(dev)) return rc;
    return launch_transpose(in, out, rows, cols, ld_in, ld_out, E, dev, (cudaStream_t)stream);
}

size_t b2_reduce_ws_bytes(int64_t n, int dtype) {
    int dev = 0;
    cudaGetDevice(&dev);
    return reduce_ws_bytes(n, dtype, dev);
}

int b2_reduce_sum(const void *in, int64_t n, int dtype, void *out, void *ws, size_t ws_bytes,
                  int dev, void *stream) {
    B2_NVTX("b2_reduce_sum");
    if (n < 0) return fail(B2_ERR_INVALID, "reduce: negative length");
    if ((!in && n) || !out) return fail(B2_ERR_INVALID, "reduce: NULL buffer");
    if (int rc = check_dev(dev)) return rc;
    if (!ws) {
        DevCtx &c = g_ctx_of(dev);
        std::lock_guard<std::mutex> g(c.mu);
        if (int rc = ctx_init(c, dev)) return rc;
        ws = c.ws;
        ws_bytes = c.ws_bytes;
    }
    return launch_reduce(in, n, dtype, out, ws, ws_bytes, dev, (cudaStream_t)stream);
}

int b2_reduce_tree_partials(const float *in, int64_t n, int block, float *partials, int dev,
                            void *stream) {
    B2_NVTX("b2_reduce_tree_partials");
    if (!in || !partials) return fail(B2_ERR_INVALID, "tree: NULL buffer");
    if (int rc = check_dev(dev)) return rc;
    return launch_tree(in, n, block, partials, dev, (cudaStream_t)stream);
}

int b2_reduce_tree512_partials(const float *in, int64_t n, float *partials, int dev, void *stream) {
    return b2_reduce_tree_partials(in, n, 512, partials, dev, stream);
}

static int tree_args(int64_t n, int block) {
    if (!tree_block_supported(block))
        return fail(B2_ERR_UNSUPPORTED, "tree: block must be a power of two in 64..2048, not " +
                                            std::to_string(block));
    if (n <= 0 || n % block)
        return fail(B2_ERR_INVALID, "exact_div(" + std::to_string(n) + ", " + std::to_string(block) +
                                        ") is not exact");
    return B2_OK;
}

int b2_reduce_tree(const float *in, int64_t n, int block, float *result_host, int dev, void *stream) {
    B2_NVTX("b2_reduce_tree");
    if (!in || !result_host) return fail(B2_ERR_INVALID, "tree: NULL buffer");
    if (int rc = tree_args(n, block)) return rc;
    if (int rc = check_dev(dev)) return rc;
    DevCtx &c = g_ctx_of(dev);
    std::lock_guard<std::mutex> g(c.mu);
    if (int rc = ctx_init(c, dev)) return rc;
    const int64_t nb = n / block;
    if (int rc = ensure_small(c, (size_t)nb * sizeof(float))) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if (int rc = launch_tree(in, n, block, (float *)c.d_small, dev, st)) return rc;
    B2_CUDA(cudaMemcpyAsync(c.h_small, c.d_small, nb * sizeof(float), cudaMemcpyDeviceToHost, st));
    B2_CUDA(cudaStreamSynchronize(st));
    // The program's host loop: `sum += p[i]` in binary32, i ascending.
    volatile float s = 0.0f;
    const float *p = (const float *)c.h_small;
    for (int64_t i = 0; i < nb; ++i) s = s + p[i];
    *result_host = s;
    return B2_OK;
}

int b2_reduce_tree512(const float *in, int64_t n, float *result_host, int dev, void *stream) {
    return b2_reduce_tree(in, n, 512, result_host, dev, stream);
}

int b2_reduce_tree_host(const float *in_host, int64_t n, int block, float *result_host, int dev) {
    B2_NVTX("b2_reduce_tree_host");
    if (!in_host || !result_host) return fail(B2_ERR_INVALID, "tree: NULL buffer");
    if (int rc = tree_args(n, block)) return rc;
    if (int rc = check_dev(dev)) return rc;
    Lane lane = acquire_lane(dev);  // any free pipeline lane of the device
    DevCtx &c = *lane.c;
    if (int rc = ctx_init(c, dev)) return rc;
    int64_t ce = (int64_t)(chunk_bytes() / sizeof(float));
    ce -= ce % block;
    ce = std::max<int64_t>(block, std::min(ce, n));
    if (int rc = ensure_stages(c, (size_t)ce * sizeof(float))) return rc;
    const int64_t nb = n / block;
    if (int rc = ensure_small(c, (size_t)nb * sizeof(float))) return rc;
    const int64_t nchunks = (n + ce - 1) / ce;
    const bool stage_in = !is_pinned(in_host);
    if (stage_in && ensure_host_stages(c, (size_t)ce * sizeof(float))) return B2_ERR_NOMEM;
    for (int64_t i = 0; i < nchunks; ++i) {
        const int k = (int)(i % kStages);
        const int64_t e0 = i * ce, ne = std::min(ce, n - e0);
        if (i >= kStages) B2_CUDA(cudaStreamWaitEvent(c.s_h2d, c.ev_comp[k], 0));
        if (int rc = h2d_rows(c, k, stage_in, c.d_in[k], (const char *)(in_host + e0), ne * sizeof(float),
                              ne * sizeof(float), 1))
            return rc;
        B2_CUDA(cudaEventRecord(c.ev_in[k], c.s_h2d));
        B2_CUDA(cudaStreamWaitEvent(c.s_comp, c.ev_in[k], 0));
        if (int rc = launch_tree((const float *)c.d_in[k], ne, block, (float *)c.d_small + e0 / block, dev,
                                 c.s_comp))
            return rc;
        B2_CUDA(cudaEventRecord(c.ev_comp[k], c.s_comp));
    }
    B2_CUDA(cudaMemcpyAsync(c.h_small, c.d_small, nb * sizeof(float), cudaMemcpyDeviceToHost, c.s_comp));
    B2_CUDA(cudaStreamSynchronize(c.s_comp));
    volatile float s = 0.0f;  // the program's host loop, binary32, i ascending
    const float *p = (const float *)c.h_small;
    for (int64_t i = 0; i < nb; ++i) s = s + p[i];
    *result_host = s;
    return B2_OK;
}

int b2_reduce_sum_seq_f32(const float *in, int64_t n, float *acc, int dev, void *stream) {
    B2_NVTX("b2_reduce_sum_seq_f32");
    if ((!in && n) || !acc) return fail(B2_ERR_INVALID, "sequential sum: NULL buffer");
    if (int rc = check_dev(dev)) return rc;
    return launch_seq_sum_f32(in, n, acc, dev, (cudaStream_t)stream);
}

int b2_reduce_sum_seq_f32_host(const float *in_host, int64_t n, float *result_host, int dev) {
    B2_NVTX("b2_reduce_sum_seq_f32_host");
    if ((!in_host && n) || !result_host) return fail(B2_ERR_INVALID, "sequential sum: NULL buffer");
    if (n < 0) return fail(B2_ERR_INVALID, "sequential sum: negative length");
    if (int rc = check_dev(dev)) return rc;
    Lane lane = acquire_lane(dev);  // any free pipeline lane of the device
    DevCtx &c = *lane.c;
    if (int rc = ctx_init(c, dev)) return rc;
    const int64_t ce = std::max<int64_t>(1, std::min<int64_t>(std::max<int64_t>(n, 1),
                                                              (int64_t)(chunk_bytes() / sizeof(float))));
    if (int rc = ensure_stages(c, (size_t)ce * sizeof(float))) return rc;
    if (int rc = ensure_small(c, sizeof(float))) return rc;
    B2_CUDA(cudaMemsetAsync(c.d_small, 0, sizeof(float), c.s_comp));
    const int64_t nchunks = (n + ce - 1) / ce;
    const bool stage_in = n > 0 && !is_pinned(in_host);
    if (stage_in && ensure_host_stages(c, (size_t)ce * sizeof(float))) return B2_ERR_NOMEM;
    for (int64_t i = 0; i < nchunks; ++i) {  // chunks in order on one compute stream
        const int k = (int)(i % kStages);
        const int64_t e0 = i * ce, ne = std::min(ce, n - e0);
        if (i >= kStages) B2_CUDA(cudaStreamWaitEvent(c.s_h2d, c.ev_comp[k], 0));
        if (int rc = h2d_rows(c, k, stage_in, c.d_in[k], (const char *)(in_host + e0), ne * sizeof(float),
                              ne * sizeof(float), 1))
            return rc;
        B2_CUDA(cudaEventRecord(c.ev_in[k], c.s_h2d));
        B2_CUDA(cudaStreamWaitEvent(c.s_comp, c.ev_in[k], 0));
        if (int rc = launch_seq_sum_f32((const float *)c.d_in[k], ne, (float *)c.d_small, dev, c.s_comp)) return rc;
        B2_CUDA(cudaEventRecord(c.ev_comp[k], c.s_comp));
    }
    B2_CUDA(cudaMemcpyAsync(c.h_small, c.d_small, sizeof(float), cudaMemcpyDeviceToHost, c.s_comp));
    B2_CUDA(cudaStreamSynchronize(c.s_comp));
    *result_host = *(const float *)c.h_small;
    return B2_OK;
}

int b2_reduce_tree512_host(const float *in_host, int64_t n, float *result_host, int dev) {
    return b2_reduce_tree_host(in_host, n, 512, result_host, dev);
}

int b2_sync(int dev, void *stream) {
    if (int rc = check_dev(dev)) return rc;
    B2_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    return B2_OK;
}

// ------------------------------------------------------------ fused cross-GPU combine
int b2_mailbox_create(int dev, void **mailbox, void *ipc_handle) {
    if (!mailbox || !ipc_handle) return fail(B2_ERR_INVALID, "mailbox: NULL argument");
    if (int rc = check_dev(dev)) return rc;
    B2_CUDA(cudaMalloc(mailbox, mailbox_bytes()));
    B2_CUDA(cudaMemset(*mailbox, 0, mailbox_bytes()));
    B2_CUDA(cudaDeviceSynchronize());
    cudaIpcMemHandle_t h;
    B2_CUDA(cudaIpcGetMemHandle(&h, *mailbox));
    memcpy(ipc_handle, &h, sizeof(h));
    return B2_OK;
}

int b2_mailbox_open(const void *ipc_handle, int dev, void **mailbox) {
    if (!mailbox || !ipc_handle) return fail(B2_ERR_INVALID, "mailbox: NULL argument");
    if (int rc = check_dev(dev)) return rc;
    cudaIpcMemHandle_t h;
    memcpy(&h, ipc_handle, sizeof(h));
    B2_CUDA(cudaIpcOpenMemHandle(mailbox, h, cudaIpcMemLazyEnablePeerAccess));
    return B2_OK;
}

int b2_mailbox_close(void *mailbox, int dev, int owner) {
    if (!mailbox) return B2_OK;
    if (int rc = check_dev(dev)) return rc;
    if (owner) B2_CUDA(cudaFree(mailbox));
    else B2_CUDA(cudaIpcCloseMemHandle(mailbox));
    return B2_OK;
}

int b2_mailbox_status(void *mailbox, int dev, uint64_t *status) {
    if (!mailbox || !status) return fail(B2_ERR_INVALID, "mailbox: NULL argument");
    if (int rc = check_dev(dev)) return rc;
    // layout (reduce.cu): slots 4 x 64 x 8 | written 64 x 8 | consumed 8 | status 8
    B2_CUDA(cudaMemcpy(status, (char *)mailbox + 4 * 64 * 8 + 64 * 8 + 8, 8, cudaMemcpyDeviceToHost));
    return B2_OK;
}

int b2_reduce_sum_fused(const void *in, int64_t n, int dtype, void *out, void *ws, size_t ws_bytes,
                        void *mailbox, int rank, int nranks, uint64_t epoch, int dev, void *stream) {
    B2_NVTX("b2_reduce_sum_fused");
    if (n < 0) return fail(B2_ERR_INVALID, "reduce: negative length");
    if ((!in && n) || !out || !mailbox) return fail(B2_ERR_INVALID, "reduce: NULL buffer");
    if (int rc = check_dev(dev)) return rc;
    if (!ws) {
        DevCtx &c = g_ctx_of(dev);
        std::lock_guard<std::mutex> g(c.mu);
        if (int rc = ctx_init(c, dev)) return rc;
        ws = c.ws;
        ws_bytes = c.ws_bytes;
    }
    FusedCombine fz;
    fz.mailbox = mailbox;
    fz.rank = rank;
    fz.nranks = nranks;
    fz.epoch = epoch;
    return launch_reduce(in, n, dtype, out, ws, ws_bytes, dev, (cudaStream_t)stream, fz);
}

// ------------------------------------------------------------ caching device allocator
// Generated programs gmem_malloc / gmem_free their arrays on every call; cudaMalloc
// and cudaFree of multi-hundred-MB blocks cost milliseconds and synchronise the
// device. Blocks are rounded to 2 MiB, kept per device in size-keyed free lists and
// handed back on the next request of the same rounded size (cache capped at 16 GiB).
namespace {
struct AllocCache {
    std::mutex mu;
    std::multimap<size_t, void *> free_blocks;
    std::unordered_map<void *, size_t> live;
    size_t cached = 0;
};
AllocCache g_alloc[64];
constexpr size_t kAllocGrain = size_t(2) << 20, kAllocCap = size_t(16) << 30;
}  // namespace

int b2_device_alloc(size_t bytes, int dev, void **out) {
    if (!out) return fail(B2_ERR_INVALID, "alloc: NULL out");
    *out = nullptr;
    if (!bytes) return B2_OK;
    if (int rc = check_dev(dev)) return rc;
    const size_t sz = (bytes + kAllocGrain - 1) / kAllocGrain * kAllocGrain;
    AllocCache &a = g_alloc[dev];
    {
        std::lock_guard<std::mutex> g(a.mu);
        auto it = a.free_blocks.find(sz);
        if (it != a.free_blocks.end()) {
            *out = it->second;
            a.free_blocks.erase(it);
            a.cached -= sz;
            a.live[*out] = sz;
            return B2_OK;
        }
    }
    cudaError_t e = cudaMalloc(out, sz);
    if (e != cudaSuccess) {  // release the cache and retry once
        std::lock_guard<std::mutex> g(a.mu);
        for (auto &kv : a.free_blocks) cudaFree(kv.second);
        a.free_blocks.clear();
        a.cached = 0;
        cudaGetLastError();
        e = cudaMalloc(out, sz);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    }
    std::lock_guard<std::mutex> g(a.mu);
    a.live[*out] = sz;
    return B2_OK;
}

int b2_device_free(void *p, int dev) {
    if (!p) return B2_OK;
    if (dev < 0 || dev >= 64) return fail(B2_ERR_INVALID, "free: bad device");
    AllocCache &a = g_alloc[dev];
    std::lock_guard<std::mutex> g(a.mu);
    auto it = a.live.find(p);
    if (it == a.live.end()) return fail(B2_ERR_INVALID, "free: pointer not from b2_device_alloc");
    const size_t sz = it->second;
    a.live.erase(it);
    // like cudaFree: work already queued on the legacy stream may still use the block
    if (int rc = check_dev(dev)) return rc;
    B2_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
    if (a.cached + sz > kAllocCap) {
        B2_CUDA(cudaFree(p));
        return B2_OK;
    }
    a.free_blocks.emplace(sz, p);
    a.cached += sz;
    return B2_OK;
}

// ------------------------------------------------------------ copy / kernel pipeline
int b2_pipe_run(int nsteps, const b2_copy2d *h2d, const int64_t *h2d_off, const b2_copy2d *d2h,
                const int64_t *d2h_off, b2_step_fn launch, void *ctx, int dev) {
    B2_NVTX("b2_pipe_run");
    if (nsteps < 0 || (nsteps && (!h2d_off || !d2h_off || !launch)))
        return fail(B2_ERR_INVALID, "pipe: bad arguments");
    if (nsteps == 0) return B2_OK;
    if (int rc = check_dev(dev)) return rc;
    Lane lane = acquire_lane(dev);  // any free pipeline lane of the device
    DevCtx &c = *lane.c;
    if (int rc = ctx_init(c, dev)) return rc;
    auto bytes = [](const b2_copy2d &x) { return (size_t)x.width * (size_t)x.height; };
    // pinned or pageable, per copy; the largest per-step pageable volume sizes the ring
    std::vector<char> pin_in(h2d_off[nsteps], 0), pin_out(d2h_off[nsteps], 0);
    size_t ring = 0;
    for (int st = 0; st < nsteps; ++st) {
        size_t a = 0, b = 0;
        for (int64_t i = h2d_off[st]; i < h2d_off[st + 1]; ++i) {
            const b2_copy2d &x = h2d[i];
            if (x.width < 0 || x.height < 0 || (bytes(x) && (!x.host || !x.dev)) ||
                (x.height > 1 && (x.host_pitch < x.width || x.dev_pitch < x.width)))
                return fail(B2_ERR_INVALID, "pipe: bad H2D region");
            pin_in[i] = is_pinned(x.host);
            if (!pin_in[i]) a += (bytes(x) + 15) & ~(size_t)15;
        }
        for (int64_t i = d2h_off[st]; i < d2h_off[st + 1]; ++i) {
            const b2_copy2d &x = d2h[i];
            if (x.width < 0 || x.height < 0 || (bytes(x) && (!x.host || !x.dev)) ||
                (x.height > 1 && (x.host_pitch < x.width || x.dev_pitch < x.width)))
                return fail(B2_ERR_INVALID, "pipe: bad D2H region");
            pin_out[i] = is_pinned(x.host);
            if (!pin_out[i]) b += (bytes(x) + 15) & ~(size_t)15;
        }
        ring = std::max(ring, std::max(a, b));
    }
    if (ring && ensure_host_stages(c, ring)) return B2_ERR_NOMEM;
    B2_CUDA(cudaEventRecord(c.ev_legacy, cudaStreamLegacy));
    B2_CUDA(cudaStreamWaitEvent(c.s_h2d, c.ev_legacy, 0));
    B2_CUDA(cudaStreamWaitEvent(c.s_comp, c.ev_legacy, 0));
    // pageable D2H regions of step j land packed in hs_out[j % kStages]; the host
    // unpacks them one step later, overlapped with the next step's DMA
    auto scatter = [&](int j) -> int {
        const int k = j % kStages;
        B2_CUDA(cudaEventSynchronize(c.ev_out[k]));
        size_t off = 0;
        for (int64_t i = d2h_off[j]; i < d2h_off[j + 1]; ++i) {
            const b2_copy2d &x = d2h[i];
            if (pin_out[i] || !bytes(x)) continue;
            par_copy2d(x.host, (size_t)x.host_pitch, (char *)c.hs_out[k] + off, (size_t)x.width, (size_t)x.width,
                       (size_t)x.height);
            off += (bytes(x) + 15) & ~(size_t)15;
        }
        return B2_OK;
    };
    // B2K_PIPE_TRACE=1: per-step H2D / kernel / D2H intervals on stderr (tools/r02_pipe_sweep.py)
    static const bool trace = getenv("B2K_PIPE_TRACE") && getenv("B2K_PIPE_TRACE")[0] == '1';
    std::vector<cudaEvent_t> tev;
    auto mark = [&](cudaStream_t s) {
        if (!trace) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        tev.push_back(e);
    };
    for (int st = 0; st < nsteps; ++st) {
        const int k = st % kStages;
        mark(c.s_h2d);
        bool staged = false;
        for (int64_t i = h2d_off[st]; i < h2d_off[st + 1]; ++i) staged |= !pin_in[i] && bytes(h2d[i]);
        if (staged) B2_CUDA(cudaEventSynchronize(c.ev_in[k]));  // the DMA that last read hs_in[k] is done
        size_t off = 0;
        for (int64_t i = h2d_off[st]; i < h2d_off[st + 1]; ++i) {
            const b2_copy2d &x = h2d[i];
            if (!bytes(x)) continue;
            if (pin_in[i]) {
                B2_CUDA(cudaMemcpy2DAsync(x.dev, (size_t)x.dev_pitch, x.host, (size_t)x.host_pitch, (size_t)x.width,
                                          (size_t)x.height, cudaMemcpyHostToDevice, c.s_h2d));
            } else {
                char *slot = (char *)c.hs_in[k] + off;
                par_copy2d(slot, (size_t)x.width, x.host, (size_t)x.host_pitch, (size_t)x.width, (size_t)x.height);
                B2_CUDA(cudaMemcpy2DAsync(x.dev, (size_t)x.dev_pitch, slot, (size_t)x.width, (size_t)x.width,
                                          (size_t)x.height, cudaMemcpyHostToDevice, c.s_h2d));
                off += (bytes(x) + 15) & ~(size_t)15;
            }
        }
        mark(c.s_h2d);
        B2_CUDA(cudaEventRecord(c.ev_in[k], c.s_h2d));
        B2_CUDA(cudaStreamWaitEvent(c.s_comp, c.ev_in[k], 0));
        mark(c.s_comp);
        if (int rc = launch(ctx, st, (void *)c.s_comp))
            return fail(B2_ERR_CUDA, std::string("pipe: step launch failed: ") + cudaGetErrorString(cudaGetLastError()) +
                                         " (code " + std::to_string(rc) + ")");
        mark(c.s_comp);
        B2_CUDA(cudaEventRecord(c.ev_comp[k], c.s_comp));
        B2_CUDA(cudaStreamWaitEvent(c.s_d2h, c.ev_comp[k], 0));
        mark(c.s_d2h);
        off = 0;
        for (int64_t i = d2h_off[st]; i < d2h_off[st + 1]; ++i) {
            const b2_copy2d &x = d2h[i];
            if (!bytes(x)) continue;
            if (pin_out[i]) {
                B2_CUDA(cudaMemcpy2DAsync(x.host, (size_t)x.host_pitch, x.dev, (size_t)x.dev_pitch, (size_t)x.width,
                                          (size_t)x.height, cudaMemcpyDeviceToHost, c.s_d2h));
            } else {
                B2_CUDA(cudaMemcpy2DAsync((char *)c.hs_out[k] + off, (size_t)x.width, x.dev, (size_t)x.dev_pitch,
                                          (size_t)x.width, (size_t)x.height, cudaMemcpyDeviceToHost, c.s_d2h));
                off += (bytes(x) + 15) & ~(size_t)15;
            }
        }
        mark(c.s_d2h);
        B2_CUDA(cudaEventRecord(c.ev_out[k], c.s_d2h));
        if (st > 0)
            if (int rc = scatter(st - 1)) return rc;
    }
    if (int rc = scatter(nsteps - 1)) return rc;
    B2_CUDA(cudaStreamSynchronize(c.s_d2h));
    B2_CUDA(cudaStreamSynchronize(c.s_comp));
    B2_CUDA(cudaStreamSynchronize(c.s_h2d));
    if (trace && !tev.empty()) {  // ms from the first H2D start: h2d [a, b) kernel [a, b) d2h [a, b)
        for (int st = 0; st < nsteps; ++st) {
            float t[6];
            for (int i = 0; i < 6; ++i) cudaEventElapsedTime(&t[i], tev[0], tev[6 * st + i]);
            fprintf(stderr, "pipe step %d: h2d %.3f-%.3f kernel %.3f-%.3f d2h %.3f-%.3f\n", st, t[0], t[1], t[2],
                    t[3], t[4], t[5]);
        }
        for (cudaEvent_t e : tev) cudaEventDestroy(e);
    }
    return B2_OK;
}

// ------------------------------------------------------------ bulk copies
int b2_copy_h2d(void *dst_dev, const void *src_host, size_t bytes, int dev) {
    B2_NVTX("b2_copy_h2d");
    if (!bytes) return B2_OK;
    if (!dst_dev || !src_host) return fail(B2_ERR_INVALID, "copy: NULL buffer");
    if (int rc = check_dev(dev)) return rc;
    Lane lane = acquire_lane(dev);  // any free pipeline lane of the device
    DevCtx &c = *lane.c;
    if (int rc = ctx_init(c, dev)) return rc;
    // like cudaMemcpy: ordered after the work already queued on the legacy default
    // stream (our copy streams are non-blocking, so this is explicit)
    B2_CUDA(cudaEventRecord(c.ev_legacy, cudaStreamLegacy));
    B2_CUDA(cudaStreamWaitEvent(c.s_h2d, c.ev_legacy, 0));
    const bool staged = !is_pinned(src_host);
    const size_t cb = chunk_bytes();
    if (staged && ensure_host_stages(c, std::min(bytes, cb))) return B2_ERR_NOMEM;
    const size_t nchunks = staged ? (bytes + cb - 1) / cb : 1;
    for (size_t i = 0; i < nchunks; ++i) {
        const int k = (int)(i % kStages);
        const size_t off = i * cb, n = staged ? std::min(cb, bytes - off) : bytes;
        if (int rc = h2d_rows(c, k, staged, (char *)dst_dev + off, (const char *)src_host + off, n, n, 1))
            return rc;
        B2_CUDA(cudaEventRecord(c.ev_in[k], c.s_h2d));
    }
    B2_CUDA(cudaStreamSynchronize(c.s_h2d));
    return B2_OK;
}

int b2_copy_d2h(void *dst_host, const void *src_dev, size_t bytes, int dev) {
    B2_NVTX("b2_copy_d2h");
    if (!bytes) return B2_OK;
    if (!dst_host || !src_dev) return fail(B2_ERR_INVALID, "copy: NULL buffer");
    if (int rc = check_dev(dev)) return rc;
    Lane lane = acquire_lane(dev);  // any free pipeline lane of the device
    DevCtx &c = *lane.c;
    if (int rc = ctx_init(c, dev)) return rc;
    B2_CUDA(cudaEventRecord(c.ev_legacy, cudaStreamLegacy));  // see b2_copy_h2d
    B2_CUDA(cudaStreamWaitEvent(c.s_d2h, c.ev_legacy, 0));
    if (is_pinned(dst_host)) {
        B2_CUDA(cudaMemcpyAsync(dst_host, src_dev, bytes, cudaMemcpyDeviceToHost, c.s_d2h));
        B2_CUDA(cudaStreamSynchronize(c.s_d2h));
        return B2_OK;
    }
    const size_t cb = chunk_bytes();
    if (ensure_host_stages(c, std::min(bytes, cb))) return B2_ERR_NOMEM;
    const size_t nchunks = (bytes + cb - 1) / cb;
    auto drain = [&](size_t j) -> int {  // host copy of chunk j out of its pinned stage
        const int kk = (int)(j % kStages);
        const size_t off = j * cb, n = std::min(cb, bytes - off);
        B2_CUDA(cudaEventSynchronize(c.ev_out[kk]));
        par_copy2d((char *)dst_host + off, n, c.hs_out[kk], n, n, 1);
        return B2_OK;
    };
    for (size_t i = 0; i < nchunks; ++i) {
        const int k = (int)(i % kStages);
        const size_t off = i * cb, n = std::min(cb, bytes - off);
        B2_CUDA(cudaMemcpyAsync(c.hs_out[k], (const char *)src_dev + off, n, cudaMemcpyDeviceToHost, c.s_d2h));
        B2_CUDA(cudaEventRecord(c.ev_out[k], c.s_d2h));
        if (i > 0)
            if (int rc = drain(i - 1)) return rc;
    }
    return drain(nchunks - 1);
}

// ------------------------------------------------------------ host pipelines
int b2_transpose_host(const void *in_host, void *out_host, int64_t rows, int64_t cols,
                      int64_t ld_in, int64_t ld_out, int dtype, int dev) {
    B2_NVTX("b2_transpose_host");
    const int E = esize_of(dtype);
    if (!E) return fail(B2_ERR_UNSUPPORTED, "transpose: unknown dtype " + std::to_string(dtype));
    if (rows < 0 || cols < 0) return fail(B2_ERR_INVALID, "transpose: negative extent");
    if (rows == 0 || cols == 0) return B2_OK;
    if (!in_host || !out_host) return fail(B2_ERR_INVALID, "transpose: NULL buffer");
    if (ld_in < cols || ld_out < rows)
        return fail(B2_ERR_INVALID, "transpose: pitch smaller than row length");
    if (int rc = check_dev(dev)) return rc;
    Lane lane = acquire_lane(dev);  // any free pipeline lane of the device
    DevCtx &c = *lane.c;
    if (int rc = ctx_init(c, dev)) return rc;
    // Chunk = a cr x cc block of the input -> a cc x cr block of the output, both
    // moved as 2-D DMA copies. Rows of either copy shorter than ~4 KB drop the copy
    // engines from 57 to 48 GB/s (profiles/r01i_pcie.md), so cr is at least 4 KB of
    // cells (output rows) and cc takes the rest of the chunk budget (input rows);
    // whole 64-row tiles per chunk where possible.
    const size_t budget = chunk_bytes();
    const int64_t min_run = std::max<int64_t>(64, 4096 / E);
    int64_t cr, cc;
    if ((size_t)cols * E * (size_t)min_run <= budget) {  // full-width row blocks
        cc = cols;
        cr = std::max<int64_t>(min_run, (int64_t)(budget / ((size_t)cols * E)));
    } else {
        cr = min_run;
        cc = std::max<int64_t>(64, (int64_t)(budget / ((size_t)cr * E)));
    }
    if (cr >= 64) cr -= cr % 64;
    if (cc >= 64 && cc < cols) cc -= cc % 64;
    cr = std::min(cr, rows);
    cc = std::min(cc, cols);
    if (int rc = ensure_stages(c, (size_t)cr * cc * E)) return rc;
    const bool stage_in = !is_pinned(in_host), stage_out = !is_pinned(out_host);
    if ((stage_in || stage_out) && ensure_host_stages(c, (size_t)cr * cc * E)) return B2_ERR_NOMEM;
    const char *hin = (const char *)in_host;
    char *hout = (char *)out_host;
    const int64_t nbr = (rows + cr - 1) / cr, nbc = (cols + cc - 1) / cc;
    const int64_t nchunks = nbr * nbc;
    auto block = [&](int64_t i, int64_t &r0, int64_t &nr, int64_t &c0, int64_t &nc) {
        r0 = (i / nbc) * cr;
        c0 = (i % nbc) * cc;
        nr = std::min(cr, rows - r0);
        nc = std::min(cc, cols - c0);
    };
    // pageable destination: the D2H lands in hs_out[k]; the host scatters it into the
    // output block one chunk later, overlapped with the next chunk's DMA
    auto scatter = [&](int64_t j) -> int {
        const int kk = (int)(j % kStages);
        int64_t r0, nr, c0, nc;
        block(j, r0, nr, c0, nc);
        B2_CUDA(cudaEventSynchronize(c.ev_out[kk]));
        par_copy2d(hout + (c0 * ld_out + r0) * E, ld_out * E, c.hs_out[kk], nr * E, nr * E, nc);
        return B2_OK;
    };
    for (int64_t i = 0; i < nchunks; ++i) {
        const int k = (int)(i % kStages);
        int64_t r0, nr, c0, nc;
        block(i, r0, nr, c0, nc);
        if (i >= kStages) B2_CUDA(cudaStreamWaitEvent(c.s_h2d, c.ev_comp[k], 0));  // d_in[k] free
        if (int rc = h2d_rows(c, k, stage_in, c.d_in[k], hin + (r0 * ld_in + c0) * E, ld_in * E, nc * E, nr))
            return rc;
        B2_CUDA(cudaEventRecord(c.ev_in[k], c.s_h2d));
        B2_CUDA(cudaStreamWaitEvent(c.s_comp, c.ev_in[k], 0));
        if (i >= kStages) B2_CUDA(cudaStreamWaitEvent(c.s_comp, c.ev_out[k], 0));  // d_out[k] free
        if (int rc = launch_transpose(c.d_in[k], c.d_out[k], nr, nc, nc, nr, E, dev, c.s_comp))
            return rc;
        B2_CUDA(cudaEventRecord(c.ev_comp[k], c.s_comp));
        B2_CUDA(cudaStreamWaitEvent(c.s_d2h, c.ev_comp[k], 0));
        if (stage_out)
            B2_CUDA(cudaMemcpyAsync(c.hs_out[k], c.d_out[k], (size_t)nr * E * nc, cudaMemcpyDeviceToHost, c.s_d2h));
        else
            B2_CUDA(cudaMemcpy2DAsync(hout + (c0 * ld_out + r0) * E, ld_out * E, c.d_out[k], nr * E, nr * E, nc,
                                      cudaMemcpyDeviceToHost, c.s_d2h));
        B2_CUDA(cudaEventRecord(c.ev_out[k], c.s_d2h));
        if (stage_out && i > 0)
            if (int rc = scatter(i - 1)) return rc;
    }
    if (stage_out)
        if (int rc = scatter(nchunks - 1)) return rc;
    B2_CUDA(cudaStreamSynchronize(c.s_d2h));
    B2_CUDA(cudaStreamSynchronize(c.s_comp));
    return B2_OK;
}

int b2_reduce_sum_host(const void *in_host, int64_t n, int dtype, void *out_host, int dev) {
    B2_NVTX("b2_reduce_sum_host");
    const int E = esize_of(dtype);
    if (dtype != B2_F32 && dtype != B2_I32 && dtype != B2_F64 && dtype != B2_I64)
        return fail(B2_ERR_UNSUPPORTED, "reduce: dtype must be B2_F32, B2_I32, B2_I64 or B2_F64");
    if (n < 0) return fail(B2_ERR_INVALID, "reduce: negative length");
    if ((!in_host && n) || !out_host) return fail(B2_ERR_INVALID, "reduce: NULL buffer");
    if (int rc = check_dev(dev)) return rc;
    Lane lane = acquire_lane(dev);  // any free pipeline lane of the device
    DevCtx &c = *lane.c;
    if (int rc = ctx_init(c, dev)) return rc;
    const int64_t ce = std::min<int64_t>(std::max<int64_t>(n, 1), (int64_t)(chunk_bytes() / E));
    if (int rc = ensure_stages(c, (size_t)ce * E)) return rc;
    const int64_t nchunks = n == 0 ? 1 : (n + ce - 1) / ce;
    if (int rc = ensure_small(c, (size_t)nchunks * 16)) return rc;
    const bool stage_in = n > 0 && !is_pinned(in_host);
    if (stage_in && ensure_host_stages(c, (size_t)ce * E)) return B2_ERR_NOMEM;
    const char *hin = (const char *)in_host;
    for (int64_t i = 0; i < nchunks; ++i) {
        const int k = (int)(i % kStages);
        const int64_t e0 = i * ce, ne = std::min(ce, n - e0);
        if (i >= kStages) B2_CUDA(cudaStreamWaitEvent(c.s_h2d, c.ev_comp[k], 0));
        if (ne > 0)
            if (int rc = h2d_rows(c, k, stage_in, c.d_in[k], hin + e0 * E, ne * E, ne * E, 1)) return rc;
        B2_CUDA(cudaEventRecord(c.ev_in[k], c.s_h2d));
        B2_CUDA(cudaStreamWaitEvent(c.s_comp, c.ev_in[k], 0));
        if (int rc = launch_reduce(c.d_in[k], std::max<int64_t>(ne, 0), dtype,
                                   (char *)c.d_small + i * 16, c.ws_pipe, c.ws_bytes, dev, c.s_comp,
                                   FusedCombine(), /*acc_out=*/true))
            return rc;
        B2_CUDA(cudaEventRecord(c.ev_comp[k], c.s_comp));
    }
    B2_CUDA(cudaMemcpyAsync(c.h_small, c.d_small, nchunks * 16, cudaMemcpyDeviceToHost, c.s_comp));
    B2_CUDA(cudaStreamSynchronize(c.s_comp));
    // host combine of the per-chunk partials, chunk order (deterministic)
    const char *h = (const char *)c.h_small;
    if (dtype == B2_I32) {
        long long s = 0;
        for (int64_t i = 0; i < nchunks; ++i) s += *(const long long *)(h + i * 16);
        *(long long *)out_host = s;
    } else if (dtype == B2_F32) {  // binary64 chunk partials, one rounding at the end
        double s = 0.0;
        for (int64_t i = 0; i < nchunks; ++i) s += *(const double *)(h + i * 16);
        *(float *)out_host = (float)s;
    } else if (dtype == B2_I64) {
        __int128 s = 0;  // exact: 128-bit chunk partials, 128-bit total (lo, hi words)
        for (int64_t i = 0; i < nchunks; ++i) {
            __int128 v;
            memcpy(&v, h + i * 16, 16);
            s += v;
        }
        memcpy(out_host, &s, 16);
    } else {
        double s = 0.0;
        for (int64_t i = 0; i < nchunks; ++i) s += *(const double *)(h + i * 16);
        *(double *)out_host = s;
    }
    return B2_OK;
}


// ------------------------------------------------ single-process multi-GPU entries
// One host thread drives every GPU of the box. Shard g lives on the
// device that owns its pointer (cudaPointerGetAttributes), so the same call runs on
// 1..8 GPUs, or with several shards on one GPU. Transpose: no exchange, each device
// transposes its row block into its column slab (possibly a peer pointer into one
// full matrix: the stores then cross NVLink inside the kernel). Reduction: every
// shard's single-pass kernel combines into the root's mailbox over NVLink (fused
// P2P combine, root = shard 0's device), rank-ordered and deterministic; without
// peer access the per-shard partials go to the host and are summed in the same
// order (identical bits).
static bool g_peer[64][64];
static std::mutex g_multi_mu;
constexpr int kMaxShards = 64;

static int ptr_device(const void *p, int *dev) {
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return cuda_fail(e, "cudaPointerGetAttributes");
    }
    if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged)
        return fail(B2_ERR_INVALID, "multi: shard pointers must be device memory");
    *dev = a.device;
    return B2_OK;
}

static int enable_peer(int from, int to) {
    if (from == to) return 1;
    if (g_peer[from][to]) return 1;
    int can = 0;
    if (cudaDeviceCanAccessPeer(&can, from, to) != cudaSuccess || !can) {
        cudaGetLastError();
        return 0;
    }
    if (check_dev(from)) return 0;
    cudaError_t e = cudaDeviceEnablePeerAccess(to, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return 0;
    }
    cudaGetLastError();
    g_peer[from][to] = true;
    return 1;
}

static int multi_ctx(int dev) {
    if (int rc = check_dev(dev)) return rc;
    DevCtx &c = g_ctx_of(dev);
    if (int rc = ctx_init(c, dev)) return rc;
    if (!c.d_slots) {
        B2_CUDA(cudaMalloc(&c.d_slots, kMaxShards * 8));
        B2_CUDA(cudaMallocHost(&c.h_slots, kMaxShards * 8));
    }
    return B2_OK;
}

// lock the contexts of every device involved, in device order (no lock-order cycles)
struct MultiLock {
    std::vector<std::unique_lock<std::mutex>> locks;
    explicit MultiLock(const std::vector<int> &devs) {
        std::vector<int> d(devs);
        std::sort(d.begin(), d.end());
        d.erase(std::unique(d.begin(), d.end()), d.end());
        for (int x : d) locks.emplace_back(g_ctx_of(x).mu);
    }
};

int b2_init(int ndev) {
    int have = 0;
    if (int rc = b2_device_count(&have)) return rc;
    if (ndev <= 0 || ndev > have) ndev = have;
    std::lock_guard<std::mutex> g(g_multi_mu);
    for (int d = 0; d < ndev; ++d) {
        std::lock_guard<std::mutex> l(g_ctx_of(d).mu);
        if (int rc = multi_ctx(d)) return rc;
    }
    for (int a = 0; a < ndev; ++a)
        for (int b = 0; b < ndev; ++b) enable_peer(a, b);
    return B2_OK;
}

int b2_peer_access(int from, int to) {
    if (from < 0 || to < 0 || from >= 64 || to >= 64) return 0;
    std::lock_guard<std::mutex> g(g_multi_mu);
    return enable_peer(from, to);
}

int b2_transpose_multi(const void *const *in, void *const *out, const int64_t *rows, int64_t cols,
                       const int64_t *ld_in, const int64_t *ld_out, int dtype, int nshards) {
    B2_NVTX("b2_transpose_multi");
    const int E = esize_of(dtype);
    if (!E) return fail(B2_ERR_UNSUPPORTED, "transpose: unknown dtype " + std::to_string(dtype));
    if (nshards <= 0 || nshards > kMaxShards || !in || !out || !rows || !ld_in || !ld_out)
        return fail(B2_ERR_INVALID, "transpose_multi: bad shard arrays");
    if (cols < 0) return fail(B2_ERR_INVALID, "transpose: negative extent");
    std::vector<int> devs(nshards, 0);
    for (int g = 0; g < nshards; ++g) {
        if (rows[g] < 0) return fail(B2_ERR_INVALID, "transpose: negative extent");
        if (rows[g] == 0 || cols == 0) continue;
        if (!in[g] || !out[g]) return fail(B2_ERR_INVALID, "transpose: NULL buffer");
        if (ld_in[g] < cols || ld_out[g] < rows[g])
            return fail(B2_ERR_INVALID, "transpose: pitch smaller than row length");
        if (int rc = ptr_device(in[g], &devs[g])) return rc;
    }
    std::lock_guard<std::mutex> gm(g_multi_mu);
    MultiLock lk(devs);
    for (int g = 0; g < nshards; ++g) {
        if (rows[g] == 0 || cols == 0) continue;
        if (int rc = multi_ctx(devs[g])) return rc;
        int od = devs[g];
        if (int rc = ptr_device(out[g], &od)) return rc;
        if (od != devs[g] && !enable_peer(devs[g], od))
            return fail(B2_ERR_UNSUPPORTED, "transpose_multi: no peer access from device " +
                                                std::to_string(devs[g]) + " to " + std::to_string(od));
    }
    // every device's stream first waits for the legacy stream (inputs produced there)
    for (int g = 0; g < nshards; ++g) {
        if (rows[g] == 0 || cols == 0) continue;
        DevCtx &c = g_ctx_of(devs[g]);
        if (int rc = check_dev(devs[g])) return rc;
        B2_CUDA(cudaEventRecord(c.ev_legacy, cudaStreamLegacy));
        B2_CUDA(cudaStreamWaitEvent(c.s_comp, c.ev_legacy, 0));
        if (int rc = launch_transpose(in[g], out[g], rows[g], cols, ld_in[g], ld_out[g], E, devs[g], c.s_comp))
            return rc;
    }
    for (int g = 0; g < nshards; ++g) {
        if (rows[g] == 0 || cols == 0) continue;
        if (int rc = check_dev(devs[g])) return rc;
        B2_CUDA(cudaStreamSynchronize(g_ctx_of(devs[g]).s_comp));
    }
    return B2_OK;
}

int b2_reduce_sum_multi(const void *const *shards, const int64_t *n, int nshards, int dtype,
                        void *host_out) {
    B2_NVTX("b2_reduce_sum_multi");
    if (dtype != B2_F32 && dtype != B2_I32 && dtype != B2_F64)
        return fail(B2_ERR_UNSUPPORTED, "reduce: dtype must be B2_F32, B2_I32 or B2_F64");
    if (nshards <= 0 || nshards > kMaxShards || !shards || !n || !host_out)
        return fail(B2_ERR_INVALID, "reduce_multi: bad shard arrays");
    std::vector<int> devs(nshards, -1);
    int root = -1;
    for (int g = 0; g < nshards; ++g) {
        if (n[g] < 0) return fail(B2_ERR_INVALID, "reduce: negative length");
        if (n[g] > 0) {
            if (!shards[g]) return fail(B2_ERR_INVALID, "reduce: NULL buffer");
            if (int rc = ptr_device(shards[g], &devs[g])) return rc;
        }
    }
    // empty shards run on the root's device (their partial is 0)
    for (int g = 0; g < nshards && root < 0; ++g) root = devs[g];
    if (root < 0) {
        if (int rc = check_dev(0)) return rc;
        root = 0;
    }
    for (int g = 0; g < nshards; ++g)
        if (devs[g] < 0) devs[g] = root;
    std::lock_guard<std::mutex> gm(g_multi_mu);
    MultiLock lk(devs);
    bool fused = true;
    for (int g = 0; g < nshards; ++g) {
        if (int rc = multi_ctx(devs[g])) return rc;
        fused = fused && enable_peer(devs[g], root);
    }
    DevCtx &rc_ = g_ctx_of(root);
    if (fused && !rc_.mailbox) {
        if (int rc = check_dev(root)) return rc;
        B2_CUDA(cudaMalloc(&rc_.mailbox, mailbox_bytes()));
        B2_CUDA(cudaMemset(rc_.mailbox, 0, mailbox_bytes()));
        B2_CUDA(cudaDeviceSynchronize());
    }
    const unsigned long long epoch = fused ? ++rc_.mb_epoch : 0;
    // non-root shards first: shards sharing the root's device then precede the
    // root's kernel on the same stream, so its wait can never block them
    auto launch = [&](int g) -> int {
        DevCtx &c = g_ctx_of(devs[g]);
        if (int rc = check_dev(devs[g])) return rc;
        B2_CUDA(cudaEventRecord(c.ev_legacy, cudaStreamLegacy));
        B2_CUDA(cudaStreamWaitEvent(c.s_comp, c.ev_legacy, 0));
        FusedCombine fz;
        if (fused) {
            fz.mailbox = rc_.mailbox;
            fz.rank = g;
            fz.nranks = nshards;
            fz.epoch = epoch;
        }
        return launch_reduce(shards[g], n[g], dtype, (char *)c.d_slots + 8 * g, c.ws_pipe, c.ws_bytes,
                             devs[g], c.s_comp, fz, /*acc_out=*/true);
    };
    for (int g = 1; g < nshards; ++g)
        if (int rc = launch(g)) return rc;
    if (int rc = launch(0)) return rc;
    // collect: the root's slot 0 holds the combined value (fused), else every slot
    std::vector<char> part(8 * nshards, 0);
    for (int g = 0; g < nshards; ++g) {
        if (fused && g > 0) continue;
        DevCtx &c = g_ctx_of(devs[g]);
        if (int rc = check_dev(devs[g])) return rc;
        B2_CUDA(cudaMemcpyAsync((char *)c.h_slots + 8 * g, (char *)c.d_slots + 8 * g, 8,
                                cudaMemcpyDeviceToHost, c.s_comp));
    }
    for (int g = 0; g < nshards; ++g) {
        if (int rc = check_dev(devs[g])) return rc;
        B2_CUDA(cudaStreamSynchronize(g_ctx_of(devs[g]).s_comp));
        memcpy(&part[8 * g], (char *)g_ctx_of(devs[g]).h_slots + 8 * g, 8);
    }
    if (fused) {
        uint64_t st = 0;
        if (int rc = check_dev(root)) return rc;
        B2_CUDA(cudaMemcpy(&st, (char *)rc_.mailbox + 4 * 64 * 8 + 64 * 8 + 8, 8, cudaMemcpyDeviceToHost));
        if (st >= epoch) return fail(B2_ERR_CUDA, "reduce_multi: fused combine timed out");
        if (dtype == B2_F32) *(float *)host_out = (float)*(const double *)&part[0];
        else memcpy(host_out, &part[0], 8);
        return B2_OK;
    }
    // host combine, shard order (the fused kernel's order: identical result)
    if (dtype == B2_I32) {
        long long s = 0;
        for (int g = 0; g < nshards; ++g) s += *(const long long *)&part[8 * g];
        *(long long *)host_out = s;
    } else if (dtype == B2_F32) {  // binary64 shard partials (the fused kernel's order)
        double s = 0.0;
        for (int g = 0; g < nshards; ++g) s += *(const double *)&part[8 * g];
        *(float *)host_out = (float)s;
    } else {
        double s = 0.0;
        for (int g = 0; g < nshards; ++g) s += *(const double *)&part[8 * g];
        *(double *)host_out = s;
    }
    return B2_OK;
}

}  // extern "C"
