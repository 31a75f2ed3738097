// sp_runtime.cu -- error reporting, per-call streams, stream-ordered scratch.
#include <stdarg.h>
#include <string.h>

#include <atomic>
#include <mutex>
#include <vector>

#include "sp_common.cuh"

namespace sp {

static thread_local char g_err[1024] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int cuda_fail(cudaError_t e, const char *what, const char *file, int line) {
    set_error("CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
              cudaGetErrorString(e), what, file, line);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        return SP_ERR_OOM;
    }
    return SP_ERR_CUDA;
}

int num_sms(int device) {
    static int cached[64] = {0};
    if (device < 0 || device >= 64) return kNumSMs;
    if (!cached[device]) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0)
            v = kNumSMs;
        cached[device] = v;
    }
    return cached[device];
}

static std::once_flag g_pool_once[64];

static size_t g_persist_max[64];
static size_t g_window_max[64];

static void tune_pool(int device) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;  // keep freed scratch for reuse
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    // L2 set-aside limits for persisting accesses (see Call::persist); the
    // set-aside itself is reserved only while a call holds a window, since
    // it shrinks the L2 every other kernel sees
    int pmax = 0, wmax = 0;
    cudaDeviceGetAttribute(&pmax, cudaDevAttrMaxPersistingL2CacheSize, device);
    cudaDeviceGetAttribute(&wmax, cudaDevAttrMaxAccessPolicyWindowSize, device);
    g_persist_max[device] = pmax > 0 ? (size_t)pmax : 0;
    g_window_max[device] = wmax > 0 ? (size_t)wmax : 0;
    cudaGetLastError();
}

static std::mutex g_persist_mu;
static int g_persist_users[64];  // calls currently holding a persisting window

// Pinned host words for per-iteration flag/counter reads: a process-wide
// free list of kPinnedBlock-byte blocks (cudaMallocHost costs milliseconds,
// so blocks are allocated once and recycled across calls).
static std::mutex g_pinned_mu;
static std::vector<void *> g_pinned_free;

void *pinned_get() {
    {
        std::lock_guard<std::mutex> lk(g_pinned_mu);
        if (!g_pinned_free.empty()) {
            void *p = g_pinned_free.back();
            g_pinned_free.pop_back();
            return p;
        }
    }
    void *p = nullptr;
    if (cudaMallocHost(&p, kPinnedBlock) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}

void pinned_put(void *p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    g_pinned_free.push_back(p);
}

int scratch_alloc(void **p, size_t bytes, cudaStream_t s) {
    cudaError_t e = cudaMallocAsync(p, bytes ? bytes : 16, s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        set_error("device scratch allocation of %zu bytes failed (%s)", bytes,
                  cudaGetErrorString(e));
        return e == cudaErrorMemoryAllocation ? SP_ERR_OOM : SP_ERR_CUDA;
    }
    return SP_OK;
}

// Graph-resident arrays come from the same stream-ordered pool (so graph
// creation/destruction does not pay cudaMalloc/cudaFree, which synchronise
// the device); allocated on the legacy stream and made visible to every
// stream by one synchronisation.
int resident_alloc(void **p, size_t bytes) {
    cudaError_t e = cudaMallocAsync(p, bytes ? bytes : 16, 0);
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *p = nullptr;
        set_error("device allocation of %zu bytes failed (%s)", bytes, cudaGetErrorString(e));
        return e == cudaErrorMemoryAllocation ? SP_ERR_OOM : SP_ERR_CUDA;
    }
    return SP_OK;
}

void resident_free(void *p) {
    if (p) cudaFreeAsync(p, 0);
}

void scratch_free(void *p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

// Per host thread and device: one non-blocking stream and two timing
// events, created on first use and reused by every later call of that
// thread (stream/event creation costs tens of microseconds per call
// otherwise).  Calls from different host threads never share a stream.
struct ThreadRes {
    cudaStream_t stream = nullptr;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    ~ThreadRes() {  // thread exit (e.g. sp_bc's workers): release the stream
        if (stream) cudaStreamDestroy(stream);
        if (t0) cudaEventDestroy(t0);
        if (t1) cudaEventDestroy(t1);
    }
};
static thread_local ThreadRes g_tres[64];

static ThreadRes g_wres[64][kWorkerSlots];
static std::mutex g_wres_mu;
static std::mutex g_wslot_mu[64];

std::mutex &worker_slots_mutex(int dev) { return g_wslot_mu[dev & 63]; }

int Call::begin_worker(int dev, int k) {
    if (dev < 0 || dev >= 64 || k < 0 || k >= kWorkerSlots) return begin(dev);
    device = dev;
    SP_CUDA(cudaSetDevice(dev));
    std::call_once(g_pool_once[dev], tune_pool, dev);
    ThreadRes *r = &g_wres[dev][k];
    {
        std::lock_guard<std::mutex> lk(g_wres_mu);
        if (!r->stream) {
            SP_CUDA(cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking));
            SP_CUDA(cudaEventCreate(&r->t0));
            SP_CUDA(cudaEventCreate(&r->t1));
        }
    }
    stream = r->stream;
    t0 = r->t0;
    t1 = r->t1;
    owned = false;
    SP_CUDA(cudaEventRecord(t0, stream));
    return SP_OK;
}

int Call::begin(int dev) {
    device = dev;
    SP_CUDA(cudaSetDevice(dev));
    if (dev >= 0 && dev < 64) std::call_once(g_pool_once[dev], tune_pool, dev);
    ThreadRes *r = (dev >= 0 && dev < 64) ? &g_tres[dev] : nullptr;
    if (r && r->stream) {
        stream = r->stream;
        t0 = r->t0;
        t1 = r->t1;
        owned = false;
    } else {
        SP_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        SP_CUDA(cudaEventCreate(&t0));
        SP_CUDA(cudaEventCreate(&t1));
        if (r) {
            r->stream = stream;
            r->t0 = t0;
            r->t1 = t1;
            owned = false;
        } else {
            owned = true;
        }
    }
    SP_CUDA(cudaEventRecord(t0, stream));
    return SP_OK;
}

int Call::finish(sp_stats *st) {
    SP_CUDA(cudaEventRecord(t1, stream));
    SP_CUDA(cudaStreamSynchronize(stream));
    SP_CUDA(cudaGetLastError());
    if (st) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, t0, t1);
        st->device_ms = ms;
        st->kernel_launches = launches;
    }
    return SP_OK;
}

void Call::persist(const void *base, size_t bytes) {
    // Opt-in (SP_L2_PERSIST=1): measured on B200 the persisting windows
    // slow every user down (BC cfg4 55.4 -> 59.8 ms, SSSP RMAT-24 5.27 ->
    // 5.65 ms) -- the set-aside shrinks the L2 the other streams gather
    // from -- and small arrays stay L2-resident anyway.
    static const bool enabled = [] {
        const char *e = getenv("SP_L2_PERSIST");
        return e && e[0] == '1';
    }();
    constexpr size_t kPersistMinBytes = size_t(16) << 20;
    if (!enabled || device < 0 || device >= 64 || !g_persist_max[device] ||
        !g_window_max[device] || bytes < kPersistMinBytes)
        return;
    {
        std::lock_guard<std::mutex> lk(g_persist_mu);
        if (g_persist_users[device]++ == 0)
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, g_persist_max[device]);
    }
    const size_t win = bytes < g_window_max[device] ? bytes : g_window_max[device];
    cudaStreamAttrValue v = {};
    v.accessPolicyWindow.base_ptr = const_cast<void *>(base);
    v.accessPolicyWindow.num_bytes = win;
    const double ratio = (double)g_persist_max[device] / (double)win;
    v.accessPolicyWindow.hitRatio = (float)(ratio < 1.0 ? ratio : 1.0);
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cudaStreamSetAttribute(stream, cudaStreamAttributeAccessPolicyWindow, &v);
    persisting = true;  // released in ~Call (also when the window was refused)
    cudaGetLastError();
}

int Call::host(void **p) {
    if (!pinned) pinned = pinned_get();
    SP_CHECK(pinned, SP_ERR_OOM, "pinned host allocation failed");
    *p = pinned;
    return SP_OK;
}

int Call::begin_external(int dev, cudaStream_t s) {
    device = dev;
    SP_CUDA(cudaSetDevice(dev));
    if (dev >= 0 && dev < 64) std::call_once(g_pool_once[dev], tune_pool, dev);
    stream = s;
    owned = false;
    external = true;
    return SP_OK;
}

Call::~Call() {
    if (stream && external) {
        for (int i = 0; i < nbufs; i++) scratch_free(bufs[i], stream);
        pinned_put(pinned);
        return;
    }
    if (stream) {
        for (int i = 0; i < nbufs; i++) scratch_free(bufs[i], stream);
        cudaStreamSynchronize(stream);
        if (persisting) {  // the stream is reused by later calls: drop the window
            cudaStreamAttrValue v = {};
            v.accessPolicyWindow.num_bytes = 0;
            cudaStreamSetAttribute(stream, cudaStreamAttributeAccessPolicyWindow, &v);
            std::lock_guard<std::mutex> lk(g_persist_mu);
            if (--g_persist_users[device] == 0) {  // last holder: give the L2 back
                cudaCtxResetPersistingL2Cache();
                cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
            }
            cudaGetLastError();
        }
        if (owned) cudaStreamDestroy(stream);
    }
    pinned_put(pinned);
    if (owned) {
        if (t0) cudaEventDestroy(t0);
        if (t1) cudaEventDestroy(t1);
    }
}

// Executable graphs of the device-side loops, per host thread, keyed by
// (graph handle, loop kind): a later call captures its body again and
// refreshes the executable with cudaGraphExecUpdate (kernel parameters
// change from call to call, the topology does not), which is far cheaper
// than cudaGraphInstantiate; a topology change falls back to instantiate.
struct ExecEntry {
    const void *key;
    int kind;
    cudaGraphExec_t exec;
};
struct ExecCache {
    std::vector<ExecEntry> v;
    ~ExecCache() {
        for (auto &e : v) cudaGraphExecDestroy(e.exec);
    }
};
static thread_local ExecCache g_exec_cache;

int launch_cached_graph(cudaGraph_t graph, const void *key, int kind, cudaStream_t stream) {
    // the same (graph, kind) first; then any executable of the same kind --
    // a fresh graph (e.g. one per request) usually has the same loop
    // topology, so an update replaces a ~0.1-0.5 ms instantiation
    for (int pass = 0; pass < 2; pass++) {
        for (auto &e : g_exec_cache.v) {
            if (e.kind != kind || (pass == 0 && e.key != key)) continue;
            cudaGraphExecUpdateResultInfo info;
            if (cudaGraphExecUpdate(e.exec, graph, &info) == cudaSuccess) {
                e.key = key;
                SP_CUDA(cudaGraphLaunch(e.exec, stream));
                return SP_OK;
            }
            cudaGetLastError();
            if (pass == 0) {  // this graph's own executable went stale: rebuild it
                cudaGraphExecDestroy(e.exec);
                e.exec = nullptr;
                SP_CUDA(cudaGraphInstantiate(&e.exec, graph, 0));
                SP_CUDA(cudaGraphLaunch(e.exec, stream));
                return SP_OK;
            }
        }
    }
    cudaGraphExec_t exec = nullptr;
    SP_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    if (g_exec_cache.v.size() >= 16) {  // bounded: drop the oldest
        cudaGraphExecDestroy(g_exec_cache.v.front().exec);
        g_exec_cache.v.erase(g_exec_cache.v.begin());
    }
    g_exec_cache.v.push_back(ExecEntry{key, kind, exec});
    SP_CUDA(cudaGraphLaunch(exec, stream));
    return SP_OK;
}

uint64_t next_graph_uid() {
    static std::atomic<uint64_t> next{1};
    return next++;
}

struct ArgExecCache {
    std::vector<ArgExec> v;
    ~ArgExecCache() {
        for (auto &e : v) {
            if (e.exec) cudaGraphExecDestroy(e.exec);
            if (e.args) cudaFree(e.args);
        }
    }
};
static thread_local ArgExecCache g_arg_exec;

int arg_exec_get(uint64_t key, int kind, size_t bytes, int device, ArgExec **out, bool *fresh) {
    for (auto &e : g_arg_exec.v) {
        if (e.key == key && e.kind == kind && e.bytes == bytes && e.exec) {
            *out = &e;
            *fresh = false;
            return SP_OK;
        }
    }
    // another graph's entry of the same kind and layout: handed over with
    // its executable, which the caller refreshes (cudaGraphExecUpdate)
    for (auto &e : g_arg_exec.v) {
        if (e.kind == kind && e.bytes == bytes && e.exec && e.device == device) {
            e.key = key;
            *out = &e;
            *fresh = true;
            return SP_OK;
        }
    }
    if (g_arg_exec.v.size() >= 16) {  // bounded: drop the oldest (calls are synchronous)
        ArgExec &o = g_arg_exec.v.front();
        if (o.exec) cudaGraphExecDestroy(o.exec);
        if (o.args) cudaFree(o.args);
        g_arg_exec.v.erase(g_arg_exec.v.begin());
    }
    ArgExec e;
    e.device = device;
    e.key = key;
    e.kind = kind;
    e.bytes = bytes;
    SP_CUDA(cudaSetDevice(device));
    SP_CUDA(cudaMalloc(&e.args, bytes));
    g_arg_exec.v.push_back(e);
    *out = &g_arg_exec.v.back();
    *fresh = true;
    return SP_OK;
}

int to_device(void *dst, const void *src, size_t bytes, int mem, cudaStream_t s) {
    if (!bytes) return SP_OK;
    SP_CUDA(cudaMemcpyAsync(dst, src, bytes,
                            mem == SP_MEM_DEVICE ? cudaMemcpyDeviceToDevice
                                                 : cudaMemcpyHostToDevice, s));
    return SP_OK;
}

int from_device(void *dst, const void *src, size_t bytes, int mem, cudaStream_t s) {
    if (!bytes) return SP_OK;
    SP_CUDA(cudaMemcpyAsync(dst, src, bytes,
                            mem == SP_MEM_DEVICE ? cudaMemcpyDeviceToDevice
                                                 : cudaMemcpyDeviceToHost, s));
    return SP_OK;
}

}  // namespace sp

extern "C" {

int sp_abi_version(void) { return SP_ABI_VERSION; }

const char *sp_last_error(void) { return sp::g_err; }

int sp_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

}  // extern "C"
