// ts_capi.cpp -- the C ABI (include/treescore_gpu.h): argument checks that
// mirror the reference's Evaluator errors (ref evaluators.py:204-220), the
// per-segment launch sequence, and the host-buffer pipeline that stands in
// for the reference's generated score_batch (ref codegen.py:115-121).
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <thread>
#include <string>
#include <unordered_map>

#include "ts_internal.h"

namespace ts {

static thread_local std::string g_err;
static std::atomic<long long> g_launches{0};
static std::atomic<int> g_kernel_path{0};  // ts_set_kernel_path

void set_error(const std::string &msg) { g_err = msg; }

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t err, const char *what) {
    char buf[512];
    snprintf(buf, sizeof buf, "%s: %s (%s)", what, cudaGetErrorString(err), cudaGetErrorName(err));
    g_err = buf;
    return TS_ERR_CUDA;
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int kernel_path() { return g_kernel_path.load(std::memory_order_relaxed); }

const DevAttrs &dev_attrs(int device) {
    static DevAttrs cache[64];
    static std::once_flag once[64];
    if (device < 0 || device >= 64) device = 0;
    std::call_once(once[device], [device] {
        cudaDeviceGetAttribute(&cache[device].sms, cudaDevAttrMultiProcessorCount, device);
        cudaDeviceGetAttribute(&cache[device].smem_optin,
                               cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    });
    return cache[device];
}

// The library's own stream-ordered pool for per-call scratch (tree-split
// mode), keeping up to 512 MB between calls so a cudaMallocFromPoolAsync is a
// sub-allocation, not a fresh mapping, and leaving the process's default pool
// settings alone.
cudaMemPool_t scratch_pool(int device) {
    static cudaMemPool_t pools[64];
    static std::once_flag once[64];
    if (device < 0 || device >= 64) device = 0;
    std::call_once(once[device], [device] {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        if (cudaMemPoolCreate(&pools[device], &props) != cudaSuccess) {
            pools[device] = nullptr;
            return;
        }
        // keep up to 2 GB cached between calls: large per-call scratch (the
        // rank path's instance ranks, the small-batch tree split's terms)
        // would otherwise be unmapped and remapped on every call
        uint64_t keep = 2048ull << 20;
        cudaMemPoolSetAttribute(pools[device], cudaMemPoolAttrReleaseThreshold, &keep);
    });
    return pools[device];
}

cudaError_t ensure_smem(const void *kernel, size_t bytes) {
    static std::mutex mu;
    static std::unordered_map<const void *, size_t> granted[64];  // per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    std::lock_guard<std::mutex> lock(mu);
    auto it = granted[dev].find(kernel);
    if (it != granted[dev].end() && it->second >= bytes) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)bytes);
    if (e == cudaSuccess) granted[dev][kernel] = bytes;
    return e;
}

void free_tables(DeviceTables *t);

namespace {

struct DeviceGuard {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) err = cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

int score_device(const ts_model *m, const float *x, int64_t n, int64_t f, int64_t ld,
                 double *out, uint16_t *ord, int64_t ld_ord, int32_t *status,
                 cudaStream_t stream, bool accumulate = false,
                 const PipeArgs *pipe = nullptr, bool x_mapped = false) {
    if (n == 0) return TS_OK;
    ScoreArgs a{};
    a.x = x;
    a.x_mapped = x_mapped ? 1 : 0;
    a.n = n;
    a.ld = ld;
    a.F = m->num_features;
    a.tables = &m->dev;
    a.blob = m->dev.blob;
    a.tree_off16 = m->dev.tree_off16;
    a.depth = m->dev.depth;
    a.weight = m->dev.weight;
    a.unit_w = m->unit_weights ? 1 : 0;
    a.out = out;
    a.ord = ord;
    a.ld_ord = ld_ord;
    a.status = status;
    for (size_t s = 0; s < m->segments.size(); s++) {
        const Segment &seg = m->segments[s];
        a.t0 = seg.t0;
        a.t1 = seg.t1;
        a.accumulate = accumulate || s > 0;
        // Only the first launch of a call needs to flag non-finite input.
        a.status = s == 0 ? status : nullptr;
        if (pipe) a.pipe = *pipe;
        cudaError_t e = launch_segment(seg, a, m->device, stream);
        if (e != cudaSuccess) return cuda_fail(e, "scoring kernel launch");
    }
    return TS_OK;
}

int check_args(const ts_model *m, const float *x, int64_t n, int64_t f, int64_t ld,
               const double *out) {
    if (!m) return fail(TS_ERR_INVALID, "model is NULL");
    if (n < 0) return fail(TS_ERR_SHAPE, "n must be >= 0");
    if (f != m->num_features) {
        char buf[160];
        snprintf(buf, sizeof buf, "dataset has shape (%lld, %lld), expected (n, %d)",
                 (long long)n, (long long)f, m->num_features);
        return fail(TS_ERR_SHAPE, buf);
    }
    if (ld < f) return fail(TS_ERR_SHAPE, "ld must be >= f");
    if (n > 0 && (!x || !out)) return fail(TS_ERR_INVALID, "x/out is NULL");
    return TS_OK;
}

}  // namespace
}  // namespace ts

using namespace ts;

extern "C" int ts_model_get_info(const ts_model *m, ts_model_info *info) {
    if (!m || !info) return fail(TS_ERR_INVALID, "NULL argument");
    *info = m->info;
    return TS_OK;
}

extern "C" int ts_score(const ts_model *m, const float *x, int64_t n, int64_t f, int64_t ld,
                        double *out, uint16_t *ord_out, int64_t ld_ord, int32_t *status,
                        void *stream) {
    int rc = check_args(m, x, n, f, ld, out);
    if (rc) return rc;
    if (ord_out && ld_ord < n) return fail(TS_ERR_SHAPE, "ld_ord must be >= n");
    if (ord_out && m->info.max_depth > TS_MAX_DEPTH)
        return fail(TS_ERR_DEPTH, "predicated ordinals need trees of depth <= MAX_DEPTH");
    DeviceGuard g(m->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    return score_device(m, x, n, f, ld, out, ord_out, ld_ord, status, (cudaStream_t)stream);
}

extern "C" int ts_score_ex(const ts_model *m, const float *x, int64_t n, int64_t f, int64_t ld,
                           double *out, uint16_t *ord_out, int64_t ld_ord, int32_t *status,
                           int accumulate, void *stream) {
    int rc = check_args(m, x, n, f, ld, out);
    if (rc) return rc;
    if (ord_out && ld_ord < n) return fail(TS_ERR_SHAPE, "ld_ord must be >= n");
    if (ord_out && m->info.max_depth > TS_MAX_DEPTH)
        return fail(TS_ERR_DEPTH, "predicated ordinals need trees of depth <= MAX_DEPTH");
    DeviceGuard g(m->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    return score_device(m, x, n, f, ld, out, ord_out, ld_ord, status, (cudaStream_t)stream,
                        accumulate != 0);
}

extern "C" int ts_score_pipe(const ts_model *m, const float *x, int64_t n, int64_t f,
                             int64_t ld, double *out, const ts_pipe *pipe, void *stream) {
    int rc = check_args(m, x, n, f, ld, out);
    if (rc) return rc;
    if (!pipe) return fail(TS_ERR_INVALID, "pipe is NULL");
    if (m->segments.size() != 1 || m->segments[0].layout != kSplit)
        return fail(TS_ERR_UNSUPPORTED,
                    "the fused pipeline needs one streaming segment of complete trees");
    if ((pipe->sums_in == nullptr) != (pipe->flags_in == nullptr) ||
        (pipe->sums_out == nullptr) != (pipe->flags_out == nullptr))
        return fail(TS_ERR_INVALID, "pipe sums and flags must be given together");
    DeviceGuard g(m->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    PipeArgs p;
    p.sums_in = pipe->sums_in;
    p.flags_in = pipe->flags_in;
    p.sums_out = pipe->sums_out;
    p.flags_out = pipe->flags_out;
    p.epoch = pipe->epoch;
    p.nblocks = (n + 31) / 32;
    return score_device(m, x, n, f, ld, out, nullptr, 0, nullptr, (cudaStream_t)stream, false,
                        &p);
}

extern "C" int ts_pipe_alloc(int device, int64_t n, double **sums, uint32_t **flags,
                             void *sums_handle64, void *flags_handle64) {
    if (!sums || !flags || n < 1) return fail(TS_ERR_INVALID, "bad pipe allocation request");
    *sums = nullptr;
    *flags = nullptr;
    DeviceGuard g(device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    const size_t nb = (size_t)(n + 31) / 32;
    cudaError_t e;
    if ((e = cudaMalloc(sums, n * sizeof(double))) ||
        (e = cudaMalloc(flags, nb * sizeof(uint32_t))) ||
        (e = cudaMemset(*flags, 0, nb * sizeof(uint32_t)))) {
        cudaFree(*sums);
        cudaFree(*flags);
        *sums = nullptr;
        *flags = nullptr;
        return cuda_fail(e, "ts_pipe_alloc");
    }
    cudaIpcMemHandle_t hs, hf;
    if (sums_handle64 && (e = cudaIpcGetMemHandle(&hs, *sums)) == cudaSuccess)
        memcpy(sums_handle64, &hs, sizeof hs);
    if (e == cudaSuccess && flags_handle64 && (e = cudaIpcGetMemHandle(&hf, *flags)) == cudaSuccess)
        memcpy(flags_handle64, &hf, sizeof hf);
    if (e != cudaSuccess) {
        cudaFree(*sums);
        cudaFree(*flags);
        *sums = nullptr;
        *flags = nullptr;
        return cuda_fail(e, "cudaIpcGetMemHandle");
    }
    return TS_OK;
}

extern "C" void ts_pipe_free(double *sums, uint32_t *flags) {
    cudaFree(sums);
    cudaFree(flags);
}

extern "C" int ts_ipc_open(const void *handle64, void **dev_ptr) {
    if (!handle64 || !dev_ptr) return fail(TS_ERR_INVALID, "NULL argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, sizeof h);
    cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
    return e == cudaSuccess ? TS_OK : cuda_fail(e, "cudaIpcOpenMemHandle");
}

extern "C" void ts_ipc_close(void *dev_ptr) {
    if (dev_ptr) cudaIpcCloseMemHandle(dev_ptr);
}

namespace {

bool host_pinned(const void *p) {
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();  // clear: an unknown host pointer is just pageable
        return false;
    }
    return attr.type == cudaMemoryTypeHost;
}

// Host copy of a pageable chunk into pinned staging, split over a small
// persistent thread pool (one memcpy thread cannot keep up with PCIe).
class CopyPool {
  public:
    static CopyPool &get() {
        // never destroyed: its workers block on the condition variable for the
        // life of the process, and destroying a condition variable with
        // waiters would hang (or crash) at exit
        static CopyPool *pool = new CopyPool();
        return *pool;
    }
    void copy(void *dst, const void *src, size_t bytes) {
        const size_t parts = bytes < (8u << 20) ? 1 : workers_.size() + 1;
        if (parts == 1) {
            memcpy(dst, src, bytes);
            return;
        }
        std::lock_guard<std::mutex> job(job_mu_);  // one split copy at a time
        const size_t step = (bytes / parts + 4095) & ~(size_t)4095;
        {
            std::lock_guard<std::mutex> l(mu_);
            dst_ = (char *)dst;
            src_ = (const char *)src;
            bytes_ = bytes;
            step_ = step;
            pending_ = workers_.size();
            gen_++;
        }
        cv_.notify_all();
        const size_t off = workers_.size() * step;  // the caller's own share: the last part
        if (off < bytes) memcpy((char *)dst + off, (const char *)src + off, bytes - off);
        std::unique_lock<std::mutex> l(mu_);
        done_.wait(l, [this] { return pending_ == 0; });
    }

  private:
    CopyPool() {
        unsigned hw = std::thread::hardware_concurrency();
        const unsigned n = std::max(1u, std::min(7u, hw > 1 ? hw / 2 : 1u));
        for (unsigned i = 0; i < n; i++) workers_.emplace_back([this, i] { run(i); });
        for (auto &t : workers_) t.detach();  // live for the process
    }
    void run(unsigned i) {
        uint64_t seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> l(mu_);
            cv_.wait(l, [&] { return gen_ != seen; });
            seen = gen_;
            char *dst = dst_;
            const char *src = src_;
            const size_t bytes = bytes_, step = step_;
            l.unlock();
            const size_t off = i * step;
            if (off < bytes) memcpy(dst + off, src + off, std::min(step, bytes - off));
            l.lock();
            if (--pending_ == 0) done_.notify_one();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex job_mu_, mu_;
    std::condition_variable cv_, done_;
    char *dst_ = nullptr;
    const char *src_ = nullptr;
    size_t bytes_ = 0, step_ = 0, pending_ = 0;
    uint64_t gen_ = 0;
};

}  // namespace

// Small batches: rows copied into mapped pinned memory, which the scoring
// kernel reads over PCIe (as its own staging loads); scores and the
// non-finite flag written straight back into mapped memory; one launch and
// one stream synchronisation per call instead of memset + H2D + kernel +
// two D2H commands (each ~2-5 us of command latency at this size).
constexpr int64_t kDirectBytes = 1 << 20;

int score_host_direct(ts_model *m, HostScratch &s, const float *x, int64_t n, int64_t f,
                      double *out) {
    const size_t xb = ((size_t)n * f * sizeof(float) + 255) & ~(size_t)255;
    const size_t need = xb + (((size_t)n * sizeof(double) + 255) & ~(size_t)255) + 256;
    cudaError_t e;
    if (s.map_bytes < need) {
        if (s.map) cudaFreeHost(s.map);
        s.map = nullptr;
        s.map_bytes = 0;
        const size_t cap = std::max<size_t>(need, 16 << 10);
        if ((e = cudaHostAlloc((void **)&s.map, cap, cudaHostAllocMapped)))
            return cuda_fail(e, "cudaHostAlloc(mapped)");
        s.map_bytes = cap;
    }
    unsigned char *dmap = nullptr;
    if ((e = cudaHostGetDevicePointer((void **)&dmap, s.map, 0)))
        return cuda_fail(e, "cudaHostGetDevicePointer");
    float *hx = reinterpret_cast<float *>(s.map);
    double *hout = reinterpret_cast<double *>(s.map + xb);
    volatile int32_t *hstatus = reinterpret_cast<int32_t *>(s.map + s.map_bytes - 256);
    // rows already in page-locked (mapped) memory are read in place; others
    // are copied into the mapped buffer (a small copy: below 64 KB the
    // pointer query costs more than it saves)
    const float *dx = reinterpret_cast<const float *>(dmap);
    const size_t in_bytes = (size_t)n * f * sizeof(float);
    void *dpin = nullptr;
    if (in_bytes > (64u << 10) && host_pinned(x) &&
        cudaHostGetDevicePointer(&dpin, const_cast<float *>(x), 0) == cudaSuccess && dpin)
        dx = static_cast<const float *>(dpin);
    else {
        (void)cudaGetLastError();
        CopyPool::get().copy(hx, x, in_bytes);
    }
    *hstatus = 0;
    int rc = score_device(m, dx, n, f, f,
                          reinterpret_cast<double *>(dmap + xb), nullptr, 0,
                          reinterpret_cast<int32_t *>(dmap + s.map_bytes - 256), s.compute,
                          false, nullptr, true);
    if (rc) {
        cudaStreamSynchronize(s.compute);
        return rc;
    }
    if ((e = cudaStreamSynchronize(s.compute))) return cuda_fail(e, "direct host path (sync)");
    memcpy(out, hout, (size_t)n * sizeof(double));
    if (*hstatus) return fail(TS_ERR_NONFINITE, "dataset contains non-finite values");
    return TS_OK;
}

// A HostScratch for the duration of one ts_score_host call: concurrent host
// callers sharing a model each get their own streams and buffers (created on
// first need, up to ts_model::kMaxHostScratch, then waited for).
struct ScratchLease {
    ts_model *m;
    HostScratch *s;
    explicit ScratchLease(ts_model *mm) : m(mm) {
        std::unique_lock<std::mutex> l(m->scratch_mu);
        m->scratch_cv.wait(l, [&] {
            return !m->scratch_free.empty() ||
                   (int)m->scratch_all.size() < ts_model::kMaxHostScratch;
        });
        if (!m->scratch_free.empty()) {
            s = m->scratch_free.back();
            m->scratch_free.pop_back();
        } else {
            m->scratch_all.emplace_back(new HostScratch());
            s = m->scratch_all.back().get();
        }
    }
    ~ScratchLease() {
        {
            std::lock_guard<std::mutex> l(m->scratch_mu);
            m->scratch_free.push_back(s);
        }
        m->scratch_cv.notify_one();
    }
};

extern "C" int ts_score_host(const ts_model *mc, const float *x, int64_t n, int64_t f,
                             double *out) {
    int rc = check_args(mc, x, n, f, f, out);
    if (rc) return rc;
    if (n == 0) return TS_OK;
    ts_model *m = const_cast<ts_model *>(mc);
    DeviceGuard g(m->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    ScratchLease lease(m);
    HostScratch &s = *lease.s;
    cudaError_t e = cudaSuccess;
    if (!s.compute) {
        if ((e = cudaStreamCreateWithFlags(&s.copy, cudaStreamNonBlocking)) ||
            (e = cudaStreamCreateWithFlags(&s.compute, cudaStreamNonBlocking)))
            return cuda_fail(e, "cudaStreamCreate");
    }
    const int64_t in_bytes = n * f * (int64_t)sizeof(float);
    if (in_bytes <= kDirectBytes) return score_host_direct(m, s, x, n, f, out);
    // Chunk so that H2D of chunk i+1 overlaps the scoring of chunk i (and,
    // for pageable input, the staging copy of chunk i+1 overlaps the DMA of
    // chunk i): 64 MB chunks, but at least four of them once the batch is
    // over 16 MB (a 54 MB batch as one chunk serialised copy, DMA and
    // kernel); smaller batches go in one piece.
    const int64_t row_bytes = f * (int64_t)sizeof(float);
    const int64_t total = n * row_bytes;
    int64_t chunk_bytes = 64ll << 20;
    if (total > (16ll << 20))
        chunk_bytes = std::min<int64_t>(chunk_bytes, std::max<int64_t>(8ll << 20, total / 4));
    int64_t chunk = std::max<int64_t>(4096, chunk_bytes / row_bytes);
    chunk = std::min(chunk, n);
    // Pageable caller buffers go through pinned staging: the pool copies
    // chunk i+1 into one pinned buffer while the DMA engine reads the other
    // (a cudaMemcpyAsync from pageable memory would stage synchronously at
    // ~10 GB/s); results land in pinned memory and are copied out on the host.
    const bool x_pinned = host_pinned(x), out_pinned = host_pinned(out);
    if (!s.copied[0]) {
        for (int i = 0; i < 2; i++) {
            if ((e = cudaEventCreateWithFlags(&s.copied[i], cudaEventDisableTiming)) ||
                (e = cudaEventCreateWithFlags(&s.consumed[i], cudaEventDisableTiming)) ||
                (e = cudaEventCreateWithFlags(&s.d2h[i], cudaEventDisableTiming)))
                return cuda_fail(e, "cudaEventCreate");
        }
        if ((e = cudaMalloc(&s.status, sizeof(int32_t)))) return cuda_fail(e, "cudaMalloc");
    }
    if (s.x_rows < chunk) {
        for (int i = 0; i < 2; i++) {
            cudaFree(s.x[i]);
            s.x[i] = nullptr;
            if ((e = cudaMalloc(&s.x[i], chunk * row_bytes))) return cuda_fail(e, "cudaMalloc(x)");
        }
        s.x_rows = chunk;
    }
    if (s.out_rows < chunk) {
        cudaFree(s.out);
        s.out = nullptr;
        if ((e = cudaMalloc(&s.out, 2 * chunk * sizeof(double))))
            return cuda_fail(e, "cudaMalloc(out)");
        s.out_rows = chunk;
    }
    if (!x_pinned && s.hx_rows < chunk) {
        for (int i = 0; i < 2; i++) {
            cudaFreeHost(s.hx[i]);
            s.hx[i] = nullptr;
            if ((e = cudaMallocHost(&s.hx[i], chunk * row_bytes)))
                return cuda_fail(e, "cudaMallocHost(x staging)");
        }
        s.hx_rows = chunk;
    }
    if (!out_pinned && s.hout_rows < chunk) {
        for (int i = 0; i < 2; i++) {
            cudaFreeHost(s.hout[i]);
            s.hout[i] = nullptr;
            if ((e = cudaMallocHost(&s.hout[i], chunk * sizeof(double))))
                return cuda_fail(e, "cudaMallocHost(out staging)");
        }
        s.hout_rows = chunk;
    }
    if ((e = cudaMemsetAsync(s.status, 0, sizeof(int32_t), s.compute)))
        return cuda_fail(e, "cudaMemsetAsync");
    // The compute stream must not start before the status reset; the copy
    // stream's first wait below orders buffer reuse.
    // On a mid-pipeline error the copies already queued may still read x or
    // write out: drain both streams before handing the buffers back.
    auto drain = [&s](int code) {
        cudaStreamSynchronize(s.copy);
        cudaStreamSynchronize(s.compute);
        return code;
    };
    // results staged in s.hout[k] waiting to be copied into the caller's out
    double *pend_dst[2] = {nullptr, nullptr};
    int64_t pend_rows[2] = {0, 0};
    auto flush = [&](int k) -> cudaError_t {
        if (!pend_dst[k]) return cudaSuccess;
        cudaError_t fe = cudaEventSynchronize(s.d2h[k]);
        if (fe == cudaSuccess) memcpy(pend_dst[k], s.hout[k], pend_rows[k] * sizeof(double));
        pend_dst[k] = nullptr;
        return fe;
    };
    // Full chunks, then halving pieces over the last two chunks' worth of
    // rows, so the part not overlapped with a copy (the last piece's kernel
    // and D2H) is small.
    int k = 0;
    int64_t rows = 0;
    for (int64_t r0 = 0; r0 < n; r0 += rows, k ^= 1) {
        const int64_t left = n - r0;
        rows = left > 2 * chunk ? chunk
                                : std::min(left, std::max<int64_t>(std::min<int64_t>(4096, chunk),
                                                                   (left + 1) / 2));
        const float *src = x + r0 * f;
        // One piece (a batch up to a chunk: the latency case): copy, score
        // and read back on the compute stream alone, no cross-stream events.
        // Every earlier call ended with the compute stream drained, which
        // orders the copy stream's last use of these buffers too.
        const bool single = r0 == 0 && rows == n;
        if (!x_pinned) {
            // staging buffer k is free once its previous H2D completed
            if (!single && (e = cudaEventSynchronize(s.copied[k])))
                return drain(cuda_fail(e, "staging"));
            CopyPool::get().copy(s.hx[k], src, rows * row_bytes);
            src = s.hx[k];
        }
        if (single) {
            if ((e = cudaMemcpyAsync(s.x[k], src, rows * row_bytes, cudaMemcpyHostToDevice,
                                     s.compute)))
                return drain(cuda_fail(e, "host pipeline (H2D)"));
        } else if ((e = cudaStreamWaitEvent(s.copy, s.consumed[k], 0)) ||
                   (e = cudaMemcpyAsync(s.x[k], src, rows * row_bytes, cudaMemcpyHostToDevice,
                                        s.copy)) ||
                   (e = cudaEventRecord(s.copied[k], s.copy)) ||
                   (e = cudaStreamWaitEvent(s.compute, s.copied[k], 0))) {
            return drain(cuda_fail(e, "host pipeline (H2D)"));
        }
        double *dout = s.out + k * chunk;
        rc = score_device(m, s.x[k], rows, f, f, dout, nullptr, 0, s.status, s.compute);
        if (rc) return drain(rc);
        if (!single && (e = cudaEventRecord(s.consumed[k], s.compute)))
            return drain(cuda_fail(e, "host pipeline"));
        if (out_pinned) {
            e = cudaMemcpyAsync(out + r0, dout, rows * sizeof(double), cudaMemcpyDeviceToHost,
                                s.compute);
        } else {
            if ((e = flush(k)) == cudaSuccess &&
                (e = cudaMemcpyAsync(s.hout[k], dout, rows * sizeof(double),
                                     cudaMemcpyDeviceToHost, s.compute)) == cudaSuccess)
                e = cudaEventRecord(s.d2h[k], s.compute);
            pend_dst[k] = out + r0;
            pend_rows[k] = rows;
        }
        if (e != cudaSuccess) return drain(cuda_fail(e, "host pipeline (D2H)"));
    }
    int32_t flag = 0;
    if ((e = cudaMemcpyAsync(&flag, s.status, sizeof(int32_t), cudaMemcpyDeviceToHost,
                             s.compute)) ||
        (e = cudaStreamSynchronize(s.compute)) || (e = flush(0)) || (e = flush(1)))
        return drain(cuda_fail(e, "host pipeline (sync)"));
    if (flag) return fail(TS_ERR_NONFINITE, "dataset contains non-finite values");
    return TS_OK;
}

extern "C" void ts_free(ts_model *m) {
    if (!m) return;
    {
        DeviceGuard g(m->device);
        free_tables(&m->dev);
        for (auto &sp : m->scratch_all) {
            HostScratch &s = *sp;
            if (s.copy) {
                cudaStreamSynchronize(s.copy);
                cudaStreamSynchronize(s.compute);
            }
            cudaFree(s.x[0]);
            cudaFree(s.x[1]);
            cudaFree(s.out);
            cudaFree(s.status);
            cudaFreeHost(s.hx[0]);
            cudaFreeHost(s.hx[1]);
            cudaFreeHost(s.hout[0]);
            cudaFreeHost(s.hout[1]);
            for (int i = 0; i < 2; i++) {
                if (s.copied[i]) cudaEventDestroy(s.copied[i]);
                if (s.consumed[i]) cudaEventDestroy(s.consumed[i]);
                if (s.d2h[i]) cudaEventDestroy(s.d2h[i]);
            }
            if (s.copy) cudaStreamDestroy(s.copy);
            if (s.compute) cudaStreamDestroy(s.compute);
            if (s.map) cudaFreeHost(s.map);
        }
    }
    delete m;
}

extern "C" const char *ts_last_error(void) { return g_err.c_str(); }

extern "C" int64_t ts_launch_count(void) { return g_launches.load(); }

extern "C" const char *ts_version(void) { return "0.1.0 sm_100a"; }

extern "C" int ts_set_kernel_path(int path) {
    if (path < 0 || path > 1) return fail(TS_ERR_INVALID, "path must be 0 (auto) or 1 (L1 only)");
    g_kernel_path = path;
    return TS_OK;
}
