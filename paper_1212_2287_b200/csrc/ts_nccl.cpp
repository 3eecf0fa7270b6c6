// ts_nccl.cpp -- the tree-shard partial-score reduction of the C ABI
// (SURVEY 8(b) `ts_reduce_partials`): one NCCL f64 sum-reduce to the root
// over NVLink / NVSwitch.  NCCL is resolved at run time (dlopen of
// libnccl.so.2, or the copy already loaded into the process, e.g. by torch)
// so the library never pins a second NCCL build next to the caller's.
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <chrono>
#include <mutex>
#include <thread>

#include "ts_internal.h"

namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId *) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, int,
                           ncclComm_t, cudaStream_t) = nullptr;
    const char *(*error_string)(ncclResult_t) = nullptr;
    // async-error polling (optional symbols: NCCL >= 2.4)
    ncclResult_t (*get_async_error)(ncclComm_t, ncclResult_t *) = nullptr;
    ncclResult_t (*comm_abort)(ncclComm_t) = nullptr;
    bool ok = false;
};

const NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
        api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
        api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
        api.reduce = (decltype(api.reduce))dlsym(h, "ncclReduce");
        api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
        api.get_async_error = (decltype(api.get_async_error))dlsym(h, "ncclCommGetAsyncError");
        api.comm_abort = (decltype(api.comm_abort))dlsym(h, "ncclCommAbort");
        api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.reduce &&
                 api.error_string;
    });
    return api;
}

int nccl_fail(ncclResult_t r, const char *what) {
    std::string msg = what;
    msg += ": ";
    msg += nccl().error_string ? nccl().error_string(r) : "NCCL error";
    return ts::fail(TS_ERR_CUDA, msg);
}

int no_nccl() { return ts::fail(TS_ERR_UNSUPPORTED, "NCCL (libnccl.so.2) is not available"); }

// A communicator whose peer died or whose network failed reports it only
// asynchronously (ncclCommGetAsyncError); a reduce enqueued on it would hang
// the stream.  ncclInProgress is a healthy non-blocking communicator.
int async_status(ncclComm_t c, const char *what) {
    if (!nccl().get_async_error) return TS_OK;
    ncclResult_t a = ncclSuccess;
    ncclResult_t r = nccl().get_async_error(c, &a);
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommGetAsyncError");
    if (a != ncclSuccess && a != ncclInProgress) return nccl_fail(a, what);
    return TS_OK;
}

}  // namespace

extern "C" int ts_nccl_get_unique_id(void *id128) {
    if (!id128) return ts::fail(TS_ERR_INVALID, "NULL argument");
    if (!nccl().ok) return no_nccl();
    ncclUniqueId id;
    ncclResult_t r = nccl().get_unique_id(&id);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    memcpy(id128, &id, sizeof id);
    return TS_OK;
}

extern "C" int ts_nccl_comm_init(const void *id128, int nranks, int rank, int device,
                                 void **comm) {
    if (!id128 || !comm || nranks < 1 || rank < 0 || rank >= nranks)
        return ts::fail(TS_ERR_INVALID, "bad communicator arguments");
    *comm = nullptr;
    if (!nccl().ok) return no_nccl();
    int prev = -1;
    cudaGetDevice(&prev);
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return ts::cuda_fail(e, "cudaSetDevice");
    ncclUniqueId id;
    memcpy(&id, id128, sizeof id);
    ncclComm_t c = nullptr;
    ncclResult_t r = nccl().comm_init_rank(&c, nranks, id, rank);
    if (prev >= 0) cudaSetDevice(prev);
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
    *comm = c;
    return TS_OK;
}

extern "C" int ts_reduce_partials(void *comm, const double *partial, double *out, int64_t n,
                                  int root, void *stream) {
    if (!comm || n < 0) return ts::fail(TS_ERR_INVALID, "bad reduction arguments");
    if (n == 0) return TS_OK;
    if (!partial) return ts::fail(TS_ERR_INVALID, "partial is NULL");
    if (!nccl().ok) return no_nccl();
    if (int st = async_status((ncclComm_t)comm, "communicator failed before ncclReduce")) return st;
    ncclResult_t r = nccl().reduce(partial, out, (size_t)n, ncclFloat64, ncclSum, root,
                                   (ncclComm_t)comm, (cudaStream_t)stream);
    if (r != ncclSuccess && r != ncclInProgress) return nccl_fail(r, "ncclReduce");
    return async_status((ncclComm_t)comm, "ncclReduce (async)");
}

extern "C" int ts_nccl_wait(void *comm, void *stream, int64_t timeout_ms) {
    if (!comm) return ts::fail(TS_ERR_INVALID, "bad communicator");
    if (!nccl().ok) return no_nccl();
    const auto t0 = std::chrono::steady_clock::now();
    while (true) {
        const cudaError_t q = cudaStreamQuery((cudaStream_t)stream);
        if (q == cudaSuccess) return async_status((ncclComm_t)comm, "NCCL (async)");
        if (q != cudaErrorNotReady) return ts::cuda_fail(q, "cudaStreamQuery");
        if (int st = async_status((ncclComm_t)comm, "NCCL (async)")) {
            // a failed peer: abort so the enqueued collective releases the stream
            if (nccl().comm_abort) nccl().comm_abort((ncclComm_t)comm);
            return st;
        }
        if (timeout_ms >= 0 &&
            std::chrono::duration_cast<std::chrono::milliseconds>(
                std::chrono::steady_clock::now() - t0).count() > timeout_ms) {
            if (nccl().comm_abort) nccl().comm_abort((ncclComm_t)comm);
            return ts::fail(TS_ERR_CUDA, "NCCL collective timed out; communicator aborted");
        }
        std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
}

extern "C" int ts_nccl_comm_destroy(void *comm) {
    if (!comm) return TS_OK;
    if (!nccl().ok) return no_nccl();
    ncclResult_t r = nccl().comm_destroy((ncclComm_t)comm);
    return r == ncclSuccess ? TS_OK : nccl_fail(r, "ncclCommDestroy");
}
