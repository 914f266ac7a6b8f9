// lk_abi.cu -- C ABI (include/loopkit_b200.h) over the device path.
//
// Mirrors proj/include/loopkit/registration.hpp: status codes instead of
// exceptions (errors.hpp), LK_NO_ALIGNMENT instead of std::nullopt. Contexts
// own their device buffers; calls on one context serialise on its mutex, so
// concurrent calls on a shared context stay safe as in the reference.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>
#include <dlfcn.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <condition_variable>
#include <functional>
#include <exception>
#include <future>
#include <type_traits>
#include <vector>

#include "../../include/loopkit_b200.h"
#include "lk_host_math.hpp"
#include "lk_kernels.cuh"

namespace {

thread_local std::string g_err;

lk_status fail(lk_status code, const std::string& msg) {
    g_err = msg;
    return code;
}

struct CudaFail {
    cudaError_t e;
    const char* where;
};
inline void ck(cudaError_t e, const char* where) {
    if (e != cudaSuccess) throw CudaFail{e, where};
}
#define CK(x) ck((x), #x)

// NCCL is opened on first use (dlopen), not linked: a process that imports
// PyTorch after this library must still get PyTorch's own libnccl.so.2 (the
// dynamic linker reuses an already-loaded SONAME, and the system NCCL lacks
// symbols PyTorch's build needs). An NCCL already in the process (PyTorch's)
// is used as is; otherwise LK_NCCL_LIBRARY, otherwise libnccl.so.2 from the
// loader's search path.
struct NcclApi {
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommInitAll) CommInitAll = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclBroadcast) Broadcast = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    std::string error;
};
const NcclApi& nccl() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h)
            if (const char* path = std::getenv("LK_NCCL_LIBRARY")) h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) {
            const char* why = dlerror();
            a.error = std::string("cannot open libnccl.so.2: ") + (why ? why : "unknown");
            return a;
        }
        auto sym = [&](auto& f, const char* name) {
            f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
            if (!f && a.error.empty()) a.error = std::string("libnccl.so.2 has no ") + name;
        };
        sym(a.GetUniqueId, "ncclGetUniqueId");
        sym(a.CommInitRank, "ncclCommInitRank");
        sym(a.CommInitAll, "ncclCommInitAll");
        sym(a.CommDestroy, "ncclCommDestroy");
        sym(a.Broadcast, "ncclBroadcast");
        sym(a.AllReduce, "ncclAllReduce");
        sym(a.GroupStart, "ncclGroupStart");
        sym(a.GroupEnd, "ncclGroupEnd");
        sym(a.GetErrorString, "ncclGetErrorString");
        return a;
    }();
    if (!api.error.empty()) throw lk::Status(LK_NCCL_ERROR, api.error);
    return api;
}

inline void nk(ncclResult_t r, const char* where) {
    if (r != ncclSuccess)
        throw lk::Status(LK_NCCL_ERROR, std::string(where) + ": " + nccl().GetErrorString(r));
}
#define NK(x) nk((x), #x)

// NVTX ranges around every ABI phase (header-only NVTX v3: free when no tool
// is attached; nsys / ncu --nvtx show the prepare sides, the hypotheses and
// the exchanges by name)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

template <class F>
lk_status guarded(F&& fn) {
    try {
        return fn();
    } catch (const lk::Status& s) {
        return fail(static_cast<lk_status>(s.code), s.what());
    } catch (const CudaFail& c) {
        return fail(LK_CUDA_ERROR, std::string(c.where) + ": " + cudaGetErrorString(c.e));
    } catch (const std::bad_alloc&) {
        return fail(LK_INTERNAL_ERROR, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(LK_INTERNAL_ERROR, e.what());
    }
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int select_device(int32_t device) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        throw lk::Status(LK_CUDA_ERROR, "no usable CUDA device (the B200 path has no CPU fallback)");
    }
    int dev = device;
    if (dev < 0) CK(cudaGetDevice(&dev));
    if (dev >= n) throw lk::Status(LK_INVALID_ARGUMENT, "device ordinal out of range");
    CK(cudaSetDevice(dev));
    // keep freed pool memory resident: contexts are created per registration
    static std::once_flag once[64];
    if (dev < 64)
        std::call_once(once[dev], [dev] {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t thr = UINT64_MAX;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
        });
    return dev;
}

// Streams are recycled across contexts (one context per registration is the
// common pattern): creating and destroying two streams per registration costs
// more than the small clouds' kernels, and fresh streams defeat the memory
// pool's same-stream reuse.
std::mutex g_stream_mu;
std::vector<std::pair<int, cudaStream_t>> g_free_streams;

// high = the device's greatest stream priority (the critical path of a
// prepare: the side whose cloud lands last, then the hypotheses), else the
// default priority. Pooled per (device, priority).
cudaStream_t acquire_stream(int dev, bool high = false) {
    int least = 0, greatest = 0;
    CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    const int prio = high ? greatest : 0;
    {
        std::lock_guard<std::mutex> lock(g_stream_mu);
        for (size_t k = g_free_streams.size(); k-- > 0;) {
            int p = 0;
            if (g_free_streams[k].first == dev && cudaStreamGetPriority(g_free_streams[k].second, &p) == cudaSuccess &&
                p == prio) {
                cudaStream_t s = g_free_streams[k].second;
                g_free_streams.erase(g_free_streams.begin() + static_cast<std::ptrdiff_t>(k));
                return s;
            }
        }
    }
    cudaStream_t s = nullptr;
    CK(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, prio));
    return s;
}

void release_stream(int dev, cudaStream_t s) {
    if (!s) return;
    std::lock_guard<std::mutex> lock(g_stream_mu);
    g_free_streams.emplace_back(dev, s);
}

// Host worker threads, recycled: prepare_registration drives the target side
// on one of these while the caller's thread drives the source side. Recycling
// keeps thread start-up (and the OpenMP team a thread builds on first use)
// off the per-registration path.
class Worker {
  public:
    Worker() : th_([this] { loop(); }) { th_.detach(); }
    void post(std::function<void()> f) {
        std::lock_guard<std::mutex> lock(mu_);
        job_ = std::move(f);
        busy_ = true;
        cv_.notify_all();
    }
    void wait() {
        std::unique_lock<std::mutex> lock(mu_);
        cv_.wait(lock, [this] { return !busy_; });
    }

  private:
    void loop() {
        std::unique_lock<std::mutex> lock(mu_);
        while (true) {
            cv_.wait(lock, [this] { return busy_ && job_; });
            std::function<void()> f = std::move(job_);
            job_ = nullptr;
            lock.unlock();
            f();
            lock.lock();
            busy_ = false;
            cv_.notify_all();
        }
    }
    std::mutex mu_;
    std::condition_variable cv_;
    std::function<void()> job_;
    bool busy_ = false;
    std::thread th_;
};

std::mutex g_worker_mu;
std::vector<Worker*> g_free_workers;

Worker* acquire_worker() {
    {
        std::lock_guard<std::mutex> lock(g_worker_mu);
        if (!g_free_workers.empty()) {
            Worker* w = g_free_workers.back();
            g_free_workers.pop_back();
            return w;
        }
    }
    return new Worker();  // lives for the process
}

void release_worker(Worker* w) {
    std::lock_guard<std::mutex> lock(g_worker_mu);
    g_free_workers.push_back(w);
}

// LK_TRACE=2: device-event timeline of prepare_registration (no syncs added;
// printed after the final sync): per mark the device time of the event on its
// stream and the host time it was enqueued, both from the start of prepare.
struct TraceMark {
    std::string name;
    cudaEvent_t ev;
    double host_ms;
};
std::mutex g_trace_mu;
std::vector<TraceMark> g_trace;
cudaEvent_t g_trace_start = nullptr;

int trace_level() {
    static const int lvl = [] {
        const char* v = std::getenv("LK_TRACE");
        return v ? std::atoi(v) : 0;
    }();
    return lvl;
}

double now_ms_since(double t0) { return (now_s() - t0) * 1e3; }

void tmark(const char* name, cudaStream_t s, double t0) {
    if (trace_level() < 2) return;
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, s);
    std::lock_guard<std::mutex> lock(g_trace_mu);
    g_trace.push_back({name, e, now_ms_since(t0)});
}

void tstart(cudaStream_t s) {
    if (trace_level() < 2) return;
    std::lock_guard<std::mutex> lock(g_trace_mu);
    for (auto& m : g_trace) cudaEventDestroy(m.ev);
    g_trace.clear();
    if (!g_trace_start) cudaEventCreate(&g_trace_start);
    cudaEventRecord(g_trace_start, s);
}

void tdump() {
    if (trace_level() < 2) return;
    std::lock_guard<std::mutex> lock(g_trace_mu);
    for (auto& m : g_trace) {
        float ms = -1.f;
        cudaEventSynchronize(m.ev);
        cudaEventElapsedTime(&ms, g_trace_start, m.ev);
        std::fprintf(stderr, "[lk trace] %-26s device %8.3f ms   enqueued %8.3f ms\n", m.name.c_str(), ms, m.host_ms);
        cudaEventDestroy(m.ev);
    }
    g_trace.clear();
}

double g_trace_t0 = 0.0;
thread_local const char* t_trace_tag = "";

bool trace_on() {
    static const bool on = std::getenv("LK_TRACE") != nullptr;
    return on;
}

int sm_count_of(int dev) {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    return sms;
}

template <class T>
T* dev_upload(const T* host, size_t count, cudaStream_t s) {
    T* d = nullptr;
    CK(lkk::pool_alloc(&d, std::max<size_t>(count, 1) * sizeof(T), s));
    if (count) CK(cudaMemcpyAsync(d, host, count * sizeof(T), cudaMemcpyHostToDevice, s));
    return d;
}

// Pageable uploads (the drop-in caller's std::vector clouds): chunks are
// copied by a few host threads into this thread's page-locked staging ring
// and DMA'd from there, the copy of chunk k + 1 overlapping the DMA of chunk
// k. (cudaMemcpyAsync from pageable memory stages through the driver's
// single-threaded bounce buffer and blocks the host for the whole copy.)
struct StageRing {
    static constexpr size_t kChunk = size_t(4) << 20;
    static constexpr int kSlots = 3;
    char* buf[kSlots] = {};
    cudaEvent_t ev[kSlots] = {};
    bool used[kSlots] = {};
    int dev = -1;
    void bind(int device) {
        if (!buf[0])
            for (auto& b : buf) CK(cudaHostAlloc(reinterpret_cast<void**>(&b), kChunk, cudaHostAllocPortable));
        if (dev != device) {
            for (int k = 0; k < kSlots; ++k) {
                if (ev[k]) {
                    if (used[k]) cudaEventSynchronize(ev[k]);
                    cudaEventDestroy(ev[k]);
                }
                CK(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
                used[k] = false;
            }
            dev = device;
        }
    }
    ~StageRing() {
        for (int k = 0; k < kSlots; ++k) {
            if (ev[k]) {
                cudaEventSynchronize(ev[k]);
                cudaEventDestroy(ev[k]);
            }
            if (buf[k]) cudaFreeHost(buf[k]);
        }
    }
};
thread_local StageRing t_ring;

void staged_upload(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    int device = 0;
    CK(cudaGetDevice(&device));
    StageRing& r = t_ring;
    r.bind(device);
    size_t off = 0;
    for (int k = 0; off < bytes; k = (k + 1) % StageRing::kSlots) {
        const size_t len = std::min(StageRing::kChunk, bytes - off);
        if (r.used[k]) CK(cudaEventSynchronize(r.ev[k]));
        const char* from = static_cast<const char*>(src) + off;
        char* to = r.buf[k];
        const int parts = len >= (size_t(1) << 20) ? 4 : 1;  // 6 or 8 measured slower, also with one side staging at a time
#pragma omp parallel for num_threads(parts) schedule(static)
        for (int q = 0; q < parts; ++q) {
            const size_t a = len * q / parts, b = len * (q + 1) / parts;
            std::memcpy(to + a, from + a, b - a);
        }
        CK(cudaMemcpyAsync(static_cast<char*>(dst) + off, to, len, cudaMemcpyHostToDevice, s));
        CK(cudaEventRecord(r.ev[k], s));
        r.used[k] = true;
        off += len;
    }
}

bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (!p || cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

void check_cloud_ptr(const lk_cloud* c, const char* what) {
    if (!c) throw lk::Status(LK_INVALID_ARGUMENT, std::string(what) + ": null cloud");
    if (c->n < 0) throw lk::Status(LK_INVALID_ARGUMENT, std::string(what) + ": negative size");
    if (c->n > 0 && !c->xyz) throw lk::Status(LK_INVALID_ARGUMENT, std::string(what) + ": null positions");
}

double resolved_max_fitness(const lk_reg_params& p) { return p.max_fitness < 0 ? p.d_max * p.d_max / 2.0 : p.max_fitness; }

lkk::ScoreParams score_params(const lk_reg_params& p, int64_t ns, bool early_exit, bool from_distance) {
    lkk::ScoreParams sp{};
    sp.d_max = p.d_max;
    sp.d2_max = p.d_max * p.d_max;
    sp.cos_max = std::cos(p.normal_angle_max);
    sp.min_ratio = p.min_inlier_ratio;
    sp.max_fitness = resolved_max_fitness(p);
    // registration.cpp:259-261
    sp.miss_budget = early_exit ? ns - static_cast<int64_t>(std::ceil(p.min_inlier_ratio * static_cast<double>(ns)))
                                : INT64_MAX;
    sp.fitness_from_distance = from_distance ? 1 : 0;
    return sp;
}

// The FP32 guard-band path is on unless LK_FP64_ONLY=1 (used by the tests to
// check both paths against the oracle).
bool fast_path_enabled() {
    const char* v = std::getenv("LK_FP64_ONLY");
    return !(v && v[0] == '1');
}

double max_norm(const double* xyz, int64_t n) {
    double m = 0.0;
    for (int64_t i = 0; i < n; ++i)
        m = std::max(m, std::sqrt(xyz[3 * i] * xyz[3 * i] + xyz[3 * i + 1] * xyz[3 * i + 1] +
                                  xyz[3 * i + 2] * xyz[3 * i + 2]));
    return m;
}

void record_to_result(const lk_reg_record& r, int64_t ns, lk_reg_result* out) {
    std::memset(out, 0, sizeof(*out));
    out->hypothesis_index = -1;
    if (!r.valid) return;
    std::memcpy(out->R, r.R, sizeof(out->R));
    std::memcpy(out->t, r.t, sizeof(out->t));
    out->inliers = r.inliers;
    out->inlier_ratio = static_cast<double>(r.inliers) / static_cast<double>(ns);
    out->fitness = r.fitness;
    out->hypothesis_index = r.index;
    out->found = 1;
}

// registration.cpp:272-276 on records of one source cloud
bool record_better(const lk_reg_record& a, const lk_reg_record& b) {
    if (a.inliers != b.inliers) return a.inliers > b.inliers;
    if (a.fitness != b.fitness) return a.fitness < b.fitness;
    return a.index < b.index;
}

}  // namespace

void lkk::trace_point(const char* what, cudaStream_t s) {
    if (trace_level() < 2) return;
    tmark((std::string(t_trace_tag) + "   . " + what).c_str(), s, g_trace_t0);
}


// EvalGrid targets from this size on also get a ring grid (explicit candidates)
constexpr int64_t kDenseTarget = 65536;

struct lk_grid {
    int device = 0;
    int sm_count = 0;
    int kind = 0;
    double cell = 0, d_max = 0;
    bool has_normals = false;
    cudaStream_t stream = nullptr;
    lkk::GridStorage g;
    lkk::RingStorage ring;  // dense EvalGrid targets: exact NN by ring shells
    bool has_ring = false;
    lkk::RunBuffers rb;
    lk_reg_record* d_record = nullptr;
    std::mutex mu;
    ~lk_grid() {
        cudaSetDevice(device);
        if (stream) cudaStreamSynchronize(stream);
        g.release();
        ring.release();
        rb.release();
        lkk::pool_free(d_record, stream);
        if (stream) cudaStreamDestroy(stream);
    }
};

struct lk_reg_ctx {
    int device = 0;
    int sm_count = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t aux_stream = nullptr;  // target-side preparation, concurrent with the source side
    cudaStream_t grid_stream = nullptr; // EvalGrid build, concurrent with the target's FPFH
    int64_t ns = 0, nt = 0;
    double *d_spos = nullptr, *d_snrm = nullptr, *d_tpos = nullptr, *d_tnrm = nullptr;
    float *d_sfeat = nullptr, *d_tfeat = nullptr;  // FPFH (prepare_registration only)
    float4* d_spos32 = nullptr;  // FP32 copy of the source for the guard-band scan
    double4* d_spos4 = nullptr;  // (x, y, z, 0) FP64 source records
    float4* d_snrm32 = nullptr;  // FP32 source normals (guarded normal gate)
    double src_max_norm = 0.0;
    int32_t* d_cache = nullptr;
    lkk::GridStorage grid;
    lkk::RunBuffers rb;
    lk_reg_record* d_record = nullptr;
    // multi-GPU: the NCCL communicator of this context's rank
    // and the [nranks x record] exchange buffer; a single-process G-device
    // context keeps the other devices' replicas in `peers` (rank g = peers[g-1])
    ncclComm_t comm = nullptr;
    int32_t nranks = 1, rank = 0;
    lk_reg_record* d_xbuf = nullptr;
    std::vector<lk_reg_ctx*> peers;
    double prepare_seconds = 0.0;
    bool profile = false;
    std::vector<std::array<cudaEvent_t, lkk::kPhaseEvents>> pending;
    double kernel_ms[lkk::kPhaseEvents - 1] = {};
    int64_t profiled_runs = 0;
    std::mutex mu;
    void drain_events() {
        for (auto& ev : pending) {
            cudaEventSynchronize(ev[lkk::kPhaseEvents - 1]);
            for (int k = 0; k < lkk::kPhaseEvents - 1; ++k) {
                float ms = 0.f;
                cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
                kernel_ms[k] += ms;
            }
            for (auto e : ev) cudaEventDestroy(e);
            profiled_runs += 1;
        }
        pending.clear();
    }
    ~lk_reg_ctx() {
        for (lk_reg_ctx* p : peers) delete p;
        peers.clear();
        cudaSetDevice(device);
        drain_events();
        if (comm) nccl().CommDestroy(comm);
        if (stream) cudaStreamSynchronize(stream);
        cudaStream_t s = own_stream;
        lkk::pool_free(d_spos, s);
        lkk::pool_free(d_spos32, s);
        lkk::pool_free(d_spos4, s);
        lkk::pool_free(d_snrm32, s);
        lkk::pool_free(d_snrm, s);
        lkk::pool_free(d_tpos, s);
        lkk::pool_free(d_tnrm, s);
        lkk::pool_free(d_cache, s);
        lkk::pool_free(d_sfeat, s);
        lkk::pool_free(d_tfeat, s);
        grid.release();
        rb.stream = s;  // the caller's stream (synchronised above) may be gone
        rb.release();
        lkk::pool_free(d_record, s);
        lkk::pool_free(d_xbuf, s);
        if (own_stream) cudaStreamSynchronize(own_stream);
        if (aux_stream) cudaStreamSynchronize(aux_stream);
        if (grid_stream) cudaStreamSynchronize(grid_stream);
        release_stream(device, own_stream);
        release_stream(device, aux_stream);
        release_stream(device, grid_stream);
    }
};

namespace {

// Source-side tail shared by both constructors: the FP32 source copy, |p|max
// bound for the guard bands and the record buffer.
void ctx_finish_source(lk_reg_ctx* c, cudaStream_t s = nullptr) {
    if (!s) s = c->stream;
    CK(lkk::pool_alloc(&c->d_spos32, std::max<int64_t>(c->ns, 1) * sizeof(float4), s));
    CK(lkk::make_source32(c->d_spos, c->ns, c->d_spos32, s));
    CK(lkk::pool_alloc(&c->d_spos4, std::max<int64_t>(c->ns, 1) * sizeof(double4), s));
    CK(lkk::pool_alloc(&c->d_snrm32, std::max<int64_t>(c->ns, 1) * sizeof(float4), s));
    CK(lkk::make_records(c->d_spos, c->d_snrm, c->ns, c->d_spos4, c->d_snrm32, s));
    CK(lkk::pool_alloc(&c->d_record, sizeof(lk_reg_record), s));
}

lk_reg_ctx* ctx_new(int32_t device) {
    auto* c = new lk_reg_ctx();
    try {
        c->device = select_device(device);
        c->sm_count = sm_count_of(c->device);
        c->own_stream = acquire_stream(c->device, true);  // source side (lands last), then the run
        c->aux_stream = acquire_stream(c->device);
        c->grid_stream = acquire_stream(c->device);
        c->stream = c->own_stream;
        c->rb.stream = c->own_stream;
    } catch (...) {
        delete c;
        throw;
    }
    return c;
}

// One cloud through voxel_downsample and FPFH on its own stream
// (registration.cpp:226-228, 246-247); the target side also builds the
// EvalGrid (:249). Runs on a host thread of its own; errors are kept, not
// thrown, so both sides finish before the reference's check order decides.
// Orders the two sides' host-staged (pageable) uploads: the target's first,
// so that its side starts while the source's cloud is still being staged.
struct UploadGate {
    std::promise<void> p;
    std::shared_future<void> f = p.get_future().share();
    bool opened = false;
    void open() {
        if (!opened) p.set_value();
        opened = true;
    }
};
struct CloudSide {
    UploadGate* wait_gate = nullptr;  // upload after this gate opens
    UploadGate* open_gate = nullptr;  // opened once this side's upload is enqueued
    const lk_cloud* in = nullptr;
    cudaStream_t s = nullptr;
    double *raw_pos = nullptr, *raw_nrm = nullptr;
    double *pos = nullptr, *nrm = nullptr;
    float* feat = nullptr;
    float4* padded = nullptr;  // feat in the feature match's layout
    float* q2 = nullptr;       // target side: |q|^2 per feature
    int64_t n = 0;
    int status = 0;  // 5: invalid normals
    int64_t usable = 0;
    double max_norm = 0.0;
    unsigned long long* stats = nullptr;  // 2 pinned words of the calling thread: usable normals, |p|max
    bool features = false;                 // feat is being computed on s
    cudaEvent_t ready = nullptr;           // downsampled positions and normals final on s
    std::exception_ptr err;
};

void prepare_side(CloudSide& cs, double feature_radius, double normal_radius, double leaf, lkk::GridStorage* grid,
                  double d_max, int device, double t0, const char* tag, cudaStream_t grid_stream = nullptr) {
    NvtxRange range(tag[0] == 's' ? "lk prepare source side" : "lk prepare target side");
    t_trace_tag = tag;
    auto mark = [&](const char* what) {
        if (trace_level() >= 2) {
            tmark((std::string(tag) + " " + what).c_str(), cs.s, t0);
            return;
        }
        if (!trace_on()) return;
        cudaStreamSynchronize(cs.s);
        std::fprintf(stderr, "[lk prepare %s] %-14s %8.3f ms\n", tag, what, (now_s() - t0) * 1e3);
    };
    try {
        CK(cudaSetDevice(device));
        const int64_t n = cs.in->n;
        if (!cs.raw_pos) {  // not already enqueued by prepare_impl: a pageable caller
            auto up = [&](const double* h) {
                double* d = nullptr;
                CK(lkk::pool_alloc(&d, std::max<int64_t>(3 * n, 1) * sizeof(double), cs.s));
                if (n) {
                    if (is_pinned(h)) CK(cudaMemcpyAsync(d, h, 3 * n * sizeof(double), cudaMemcpyHostToDevice, cs.s));
                    else staged_upload(d, h, 3 * n * sizeof(double), cs.s);
                }
                return d;
            };
            if (cs.wait_gate) cs.wait_gate->f.wait();
            cs.raw_pos = up(cs.in->xyz);
            cs.raw_nrm = cs.in->nxyz ? up(cs.in->nxyz) : nullptr;
        }
        if (cs.open_gate) cs.open_gate->open();
        mark("upload");
        CK(lkk::pool_alloc(&cs.pos, 3 * n * sizeof(double), cs.s));
        CK(lkk::pool_alloc(&cs.nrm, 3 * n * sizeof(double), cs.s));
        // with input normals the downsample also produces the cloud stats
        // (usable normals, |p|max); they land in cs.stats (the calling
        // thread's pinned words) ahead of the FPFH, whose readback synchronises
        CK(lkk::voxel_downsample(cs.raw_pos, cs.raw_nrm, n, leaf, cs.pos, cs.nrm, &cs.n, &cs.status, cs.s,
                                 cs.raw_nrm ? cs.stats : nullptr));
        lkk::pool_free(cs.raw_pos, cs.s);
        lkk::pool_free(cs.raw_nrm, cs.s);
        cs.raw_pos = cs.raw_nrm = nullptr;
        mark("downsample");
        if (cs.status != 0 || cs.n < 4) return;
        if (!cs.in->nxyz) {
            // registration.cpp:232-237: estimate_normals(cloud, normal_radius, origin)
            const double origin[3] = {0.0, 0.0, 0.0};
            CK(lkk::estimate_normals(cs.pos, cs.n, normal_radius, origin, cs.nrm, cs.s));
            mark("normals");
        }
        if (!cs.in->nxyz) CK(lkk::cloud_stats_async(cs.pos, cs.nrm, cs.n, cs.stats, cs.s));
        CK(cudaEventCreateWithFlags(&cs.ready, cudaEventDisableTiming));
        CK(cudaEventRecord(cs.ready, cs.s));
        // the EvalGrid (registration.cpp:249) only needs the downsampled
        // cloud: it is built on its own stream and host thread while this
        // one runs the FPFH
        Worker* gw = nullptr;
        cudaError_t grid_err = cudaSuccess;
        if (grid) {
            CK(cudaStreamWaitEvent(grid_stream, cs.ready, 0));
            gw = acquire_worker();
            const double* pos = cs.pos;
            const double* nrm = cs.nrm;
            const int64_t n = cs.n;
            gw->post([grid, pos, nrm, n, d_max, grid_stream, device, &grid_err, t0] {
                cudaSetDevice(device);
                grid_err = lkk::build_grid(*grid, 0, pos, nrm, n, d_max, d_max, grid_stream);
                tmark("tgt eval grid (own stream)", grid_stream, t0);
            });
        }
        try {
            CK(lkk::pool_alloc(&cs.feat, 33 * cs.n * sizeof(float), cs.s));
            CK(lkk::compute_fpfh(cs.pos, cs.nrm, cs.n, feature_radius, cs.feat, cs.s));
        } catch (...) {
            if (gw) {
                gw->wait();
                release_worker(gw);
            }
            throw;
        }
        // the feature match's per-cloud inputs, on this side's stream (the
        // target's off the source's critical path)
        CK(lkk::pool_alloc(&cs.padded, lkk::fnn_padded_bytes(cs.n), cs.s));
        if (grid) CK(lkk::pool_alloc(&cs.q2, std::max<int64_t>(cs.n, 1) * sizeof(float), cs.s));
        CK(lkk::fnn_prepare(cs.feat, cs.n, cs.padded, cs.q2, cs.s));
        mark("fpfh");
        // no wait here: the feature match is queued behind both sides'
        // streams, and prepare's final sync brings the stats back
        cs.features = true;
        if (gw) {
            gw->wait();
            release_worker(gw);
            CK(grid_err);
            mark("eval grid");
        }
    } catch (...) {
        cs.err = std::current_exception();
    }
    if (cs.open_gate) cs.open_gate->open();  // never leave the other side waiting
}

// Devices of a call (lk_reg_params::device_count): `device` alone, or G
// consecutive devices from it, or every visible device (-1).
std::vector<int> call_devices(int32_t device, int32_t device_count) {
    const int d0 = select_device(device);
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    int g = device_count < 0 ? n - d0 : device_count;
    if (g <= 1) return {d0};
    if (d0 + g > n) throw lk::Status(LK_INVALID_ARGUMENT, "device_count exceeds the visible CUDA devices");
    std::vector<int> devs;
    for (int k = 0; k < g; ++k) devs.push_back(d0 + k);
    return devs;
}

// A single-process G-device context: NCCL communicators over the devices
// (ncclCommInitAll), the prepared context broadcast from device 0
// (ncclBroadcast of the downsampled clouds and the match cache), the source
// records and the EvalGrid rebuilt on each replica from the broadcast target
// (deterministic: bit-identical to device 0's), one exchange buffer per rank.
void make_peers(lk_reg_ctx* c, const std::vector<int>& devs, double d_max) {
    NvtxRange range("lk replicate context (ncclBroadcast)");
    const int G = static_cast<int>(devs.size());
    std::vector<ncclComm_t> comms(G);
    NK(nccl().CommInitAll(comms.data(), G, devs.data()));
    c->comm = comms[0];
    c->nranks = G;
    c->rank = 0;
    for (int g = 1; g < G; ++g) {
        lk_reg_ctx* p = ctx_new(devs[g]);
        c->peers.push_back(p);
        p->comm = comms[g];
        p->nranks = G;
        p->rank = g;
        p->ns = c->ns;
        p->nt = c->nt;
        p->src_max_norm = c->src_max_norm;
        cudaStream_t s = p->stream;
        CK(lkk::pool_alloc(&p->d_spos, 3 * p->ns * sizeof(double), s));
        CK(lkk::pool_alloc(&p->d_snrm, 3 * p->ns * sizeof(double), s));
        CK(lkk::pool_alloc(&p->d_tpos, 3 * p->nt * sizeof(double), s));
        CK(lkk::pool_alloc(&p->d_tnrm, 3 * p->nt * sizeof(double), s));
        CK(lkk::pool_alloc(&p->d_cache, p->ns * sizeof(int32_t), s));
    }
    std::vector<lk_reg_ctx*> all{c};
    all.insert(all.end(), c->peers.begin(), c->peers.end());
    auto bcast = [&](auto member, size_t count, ncclDataType_t type) {
        NK(nccl().GroupStart());
        for (int g = 0; g < G; ++g)
            NK(nccl().Broadcast(all[0]->*member, all[g]->*member, count, type, 0, all[g]->comm, all[g]->stream));
        NK(nccl().GroupEnd());
    };
    bcast(&lk_reg_ctx::d_spos, 3 * c->ns, ncclFloat64);
    bcast(&lk_reg_ctx::d_snrm, 3 * c->ns, ncclFloat64);
    bcast(&lk_reg_ctx::d_tpos, 3 * c->nt, ncclFloat64);
    bcast(&lk_reg_ctx::d_tnrm, 3 * c->nt, ncclFloat64);
    bcast(&lk_reg_ctx::d_cache, c->ns, ncclInt32);
    for (lk_reg_ctx* p : c->peers) {
        CK(cudaSetDevice(p->device));
        ctx_finish_source(p);
        CK(lkk::build_grid(p->grid, 0, p->d_tpos, p->d_tnrm, p->nt, d_max, d_max, p->stream));
    }
    for (lk_reg_ctx* q : all) {
        CK(cudaSetDevice(q->device));
        CK(lkk::pool_alloc(&q->d_xbuf, G * sizeof(lk_reg_record), q->stream));
        CK(cudaStreamSynchronize(q->stream));
    }
    CK(cudaSetDevice(c->device));
}

lk_status prepare_impl(const lk_cloud* src, const lk_cloud* tgt, const lk_reg_params* params, lk_reg_ctx** out) {
    NvtxRange range("lk_reg_prepare");
    if (!params || !out) return fail(LK_INVALID_ARGUMENT, "null argument");
    check_cloud_ptr(src, "source");
    check_cloud_ptr(tgt, "target");
    *out = nullptr;
    double t0 = now_s();
    if (src->n == 0 || tgt->n == 0) return fail(LK_EMPTY_CLOUD, "voxel_downsample: empty cloud");
    if (!(params->leaf > 0.0)) return fail(LK_INVALID_ARGUMENT, "voxel_downsample: leaf must be positive");
    const std::vector<int> devs = call_devices(params->device, params->device_count);
    lk_reg_ctx* c = ctx_new(devs[0]);
    tstart(c->own_stream);
    g_trace_t0 = t0;
    CloudSide S, T;
    UploadGate gate;
    S.in = src;
    S.s = c->own_stream;
    T.in = tgt;
    T.s = c->aux_stream;
    // both sides' stats words belong to the calling thread (the target side's
    // worker is released before they are read)
    thread_local unsigned long long* t_stats = nullptr;
    if (!t_stats) CK(cudaHostAlloc(reinterpret_cast<void**>(&t_stats), 4 * sizeof(unsigned long long), 0));
    S.stats = t_stats;
    T.stats = t_stats + 2;
    auto drop = [&](CloudSide& cs) {
        lkk::pool_free(cs.raw_pos, cs.s);
        lkk::pool_free(cs.raw_nrm, cs.s);
        lkk::pool_free(cs.padded, cs.s);
        lkk::pool_free(cs.q2, cs.s);
        cs.padded = nullptr;
        cs.q2 = nullptr;
        if (cs.ready) cudaEventDestroy(cs.ready);
        cs.ready = nullptr;
    };
    try {
        // page-locked callers: the two uploads are enqueued here back to back,
        // the target's first and the source's after it (an event orders them),
        // so each gets the whole PCIe link and its side starts as soon as its
        // own cloud has landed (two concurrent copies share the link and both
        // land late). Pageable callers: each side's thread stages its own.
        if (is_pinned(src->xyz) && is_pinned(tgt->xyz) && (!src->nxyz || is_pinned(src->nxyz)) &&
            (!tgt->nxyz || is_pinned(tgt->nxyz))) {
            T.raw_pos = dev_upload(tgt->xyz, 3 * tgt->n, T.s);
            T.raw_nrm = tgt->nxyz ? dev_upload(tgt->nxyz, 3 * tgt->n, T.s) : nullptr;
            cudaEvent_t landed;
            CK(cudaEventCreateWithFlags(&landed, cudaEventDisableTiming));
            CK(cudaEventRecord(landed, T.s));
            CK(cudaStreamWaitEvent(S.s, landed, 0));
            cudaEventDestroy(landed);
            S.raw_pos = dev_upload(src->xyz, 3 * src->n, S.s);
            S.raw_nrm = src->nxyz ? dev_upload(src->nxyz, 3 * src->n, S.s) : nullptr;
        } else {
            // host-staged copies share the link and the host's memory
            // bandwidth: the target's first, the source's after it
            T.open_gate = &gate;
            S.wait_gate = &gate;
        }
        // the two clouds are independent until the feature match: the target
        // side (H2D, downsample, FPFH, EvalGrid) runs on a second host thread
        // and stream while this thread does the source side
        Worker* worker = acquire_worker();
        const double fr = params->feature_radius, nr = params->normal_radius, leaf = params->leaf,
                     dm = params->d_max;
        const int dev = c->device;
        lkk::GridStorage* grid = &c->grid;
        cudaStream_t gs = c->grid_stream;
        worker->post([&T, fr, nr, leaf, grid, dm, dev, t0, gs] {
            prepare_side(T, fr, nr, leaf, grid, dm, dev, t0, "tgt", gs);
        });
        prepare_side(S, fr, nr, leaf, nullptr, 0.0, dev, t0, "src");
        worker->wait();
        release_worker(worker);
        if (trace_on() && trace_level() < 2)
            std::fprintf(stderr, "[lk prepare] joined %8.3f ms\n", (now_s() - t0) * 1e3);
        c->d_spos = S.pos;
        c->d_snrm = S.nrm;
        c->d_tpos = T.pos;
        c->d_tnrm = T.nrm;
        c->d_sfeat = S.feat;
        c->d_tfeat = T.feat;
        c->ns = S.n;
        c->nt = T.n;
        if (S.err) std::rethrow_exception(S.err);
        if (T.err) std::rethrow_exception(T.err);
        // feature pre-match (registration.cpp:248) queued behind both sides'
        // streams before any host wait; the checks below decide whether it
        // counts (an error discards the context)
        cudaStream_t s = c->stream;
        if (S.features && T.features) {
            for (CloudSide* cs : {&S, &T}) {
                if (cs->s == s) continue;
                cudaEvent_t done;
                CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
                CK(cudaEventRecord(done, cs->s));
                CK(cudaStreamWaitEvent(s, done, 0));
                cudaEventDestroy(done);
            }
            CK(lkk::pool_alloc(&c->d_cache, c->ns * sizeof(int32_t), s));
            CK(lkk::feature_nn_prepared(c->d_sfeat, S.padded, c->ns, c->d_tfeat, T.padded, T.q2, c->nt, c->d_cache,
                                        s));
            for (CloudSide* cs : {&S, &T}) {
                lkk::pool_free(cs->padded, s);
                lkk::pool_free(cs->q2, s);
                cs->padded = nullptr;
                cs->q2 = nullptr;
            }
            tmark("joined, feature nn start", s, t0);
            // the source's FP32 copy and records need only its downsampled
            // cloud: on the target's stream (idle by now), beside the match
            CK(cudaStreamWaitEvent(T.s, S.ready, 0));
            ctx_finish_source(c, T.s);
            cudaEvent_t fin;
            CK(cudaEventCreateWithFlags(&fin, cudaEventDisableTiming));
            CK(cudaEventRecord(fin, T.s));
            CK(cudaStreamWaitEvent(s, fin, 0));
            cudaEventDestroy(fin);
            tmark("feature nn done", s, t0);
        }
        // no wait for the match: each side's stats were copied ahead of its
        // FPFH, whose list-head readback synchronised that side's stream; a
        // side that stopped early (invalid normals, < 4 points) fails a check
        // below before its stats are read
        if (!(S.features && T.features)) {
            CK(cudaStreamSynchronize(T.s));
            CK(cudaStreamSynchronize(S.s));
        }
        for (CloudSide* cs : {&S, &T}) {
            if (cs->features) lkk::cloud_stats_decode(cs->stats, &cs->usable, &cs->max_norm);
            if (cs->ready) cudaEventDestroy(cs->ready);  // its waits are enqueued
            cs->ready = nullptr;
        }
        c->src_max_norm = S.max_norm;
        // the reference's check order (registration.cpp:226-245)
        if (S.status == 5 || T.status == 5)
            throw lk::Status(LK_MISSING_NORMALS, "normals must be unit length or exactly zero");
        if (c->ns < 4 || c->nt < 4)
            throw lk::Status(LK_TOO_FEW_POINTS, "register_global: fewer than 4 points after downsampling");
        if (S.usable < 4 || T.usable < 4)
            throw lk::Status(LK_MISSING_DATA, "register_global: fewer than 4 points with usable normals");
        if (trace_on()) {
            CK(cudaStreamSynchronize(s));
            tdump();
            std::fprintf(stderr, "[lk prepare] feature nn %8.3f ms\n", (now_s() - t0) * 1e3);
        }
        if (devs.size() > 1) make_peers(c, devs, params->d_max);
    } catch (...) {
        drop(S);
        drop(T);
        delete c;
        throw;
    }
    c->prepare_seconds = now_s() - t0;
    *out = c;
    return LK_OK;
}

lk_status run_range_impl(lk_reg_ctx* c, const lk_reg_params& p, int64_t begin, int64_t end, void* d_record) {
    NvtxRange range("lk run_hypotheses range");
    if (c->ns < 4) return fail(LK_TOO_FEW_POINTS, "sample_quadruple: need >= 4 source points");
    if (!c->d_cache) return fail(LK_MISSING_DATA, "sample_quadruple: no correspondence cache");
    if (begin < 0 || end < begin) return fail(LK_INVALID_ARGUMENT, "bad hypothesis range");
    CK(cudaSetDevice(c->device));
    lkk::SourceView sv{c->d_spos, c->d_snrm, c->d_spos32, c->ns, c->d_spos4, c->d_snrm32};
    lkk::ScoreParams sp = score_params(p, c->ns, true, false);
    if (fast_path_enabled()) lkk::configure_fast_path(sp, c->grid.view, c->src_max_norm);
    cudaEvent_t* ev = nullptr;
    if (c->profile) {
        std::array<cudaEvent_t, lkk::kPhaseEvents> e4;
        for (auto& e : e4) CK(cudaEventCreate(&e));
        c->pending.push_back(e4);
        ev = c->pending.back().data();
    }
    CK(lkk::run_hypotheses_range(sv, c->d_tpos, c->d_cache, c->grid.view, sp, p.seed, p.similarity_tau, begin, end,
                                 c->rb, d_record, c->stream, c->sm_count, ev));
    return LK_OK;
}

// Every rank's share of [0, H) and one ncclAllReduce(sum) over the
// zero-filled [nranks x record] buffers (an exact all-gather: each slot has
// one writer); single-process G-device contexts drive all ranks from here,
// a multi-process rank drives its own. Leaves the records on c's device.
lk_status exchange_run(lk_reg_ctx* c, const lk_reg_params& p) {
    NvtxRange range("lk shares + ncclAllReduce of rank records");
    const int G = c->nranks;
    const int64_t H = p.hypothesis_count;
    const size_t words = G * sizeof(lk_reg_record) / sizeof(int64_t);
    std::vector<lk_reg_ctx*> all;
    if (!c->peers.empty()) {
        all.push_back(c);
        all.insert(all.end(), c->peers.begin(), c->peers.end());
    } else {
        all.push_back(c);
    }
    for (lk_reg_ctx* q : all) {
        CK(cudaSetDevice(q->device));
        CK(cudaMemsetAsync(q->d_xbuf, 0, G * sizeof(lk_reg_record), q->stream));
        const int64_t begin = q->rank * H / G, end = (q->rank + 1) * H / G;
        const lk_status st = run_range_impl(q, p, begin, end, q->d_xbuf + q->rank);
        if (st != LK_OK) return st;
    }
    NK(nccl().GroupStart());
    for (lk_reg_ctx* q : all)
        NK(nccl().AllReduce(q->d_xbuf, q->d_xbuf, words, ncclInt64, ncclSum, q->comm, q->stream));
    NK(nccl().GroupEnd());
    CK(cudaSetDevice(c->device));
    return LK_OK;
}

}  // namespace

extern "C" {

int lk_abi_version(void) { return LK_ABI_VERSION; }
const char* lk_last_error(void) { return g_err.c_str(); }

int lk_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

lk_status lk_reg_prepare(const lk_cloud* src, const lk_cloud* tgt, const lk_reg_params* params, lk_reg_ctx** out) {
    return guarded([&] { return prepare_impl(src, tgt, params, out); });
}

lk_status lk_reg_ctx_create(const lk_cloud* src, const lk_cloud* tgt, const int32_t* cache,
                            const lk_reg_params* params, lk_reg_ctx** out) {
    return guarded([&]() -> lk_status {
        if (!params || !out || !cache) return fail(LK_INVALID_ARGUMENT, "null argument");
        check_cloud_ptr(src, "source");
        check_cloud_ptr(tgt, "target");
        *out = nullptr;
        if (src->n == 0 || tgt->n == 0) return fail(LK_EMPTY_CLOUD, "RegistrationContext: empty cloud");
        if (!src->nxyz || !tgt->nxyz) return fail(LK_MISSING_NORMALS, "RegistrationContext: normals required");
        for (int64_t i = 0; i < src->n; ++i)
            if (cache[i] < 0 || cache[i] >= tgt->n)
                return fail(LK_MISSING_DATA, "RegistrationContext: cache index out of range");
        lk_reg_ctx* c = ctx_new(params->device);
        try {
            cudaStream_t s = c->stream;
            c->ns = src->n;
            c->nt = tgt->n;
            c->d_spos = dev_upload(src->xyz, 3 * src->n, s);
            c->d_snrm = dev_upload(src->nxyz, 3 * src->n, s);
            c->d_tpos = dev_upload(tgt->xyz, 3 * tgt->n, s);
            c->d_tnrm = dev_upload(tgt->nxyz, 3 * tgt->n, s);
            c->d_cache = dev_upload(cache, src->n, s);
            c->src_max_norm = max_norm(src->xyz, src->n);
            ctx_finish_source(c);
            CK(lkk::build_grid(c->grid, 0, c->d_tpos, c->d_tnrm, c->nt, params->d_max, params->d_max, s));
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
        return LK_OK;
    });
}

void lk_reg_ctx_destroy(lk_reg_ctx* ctx) { delete ctx; }

lk_status lk_reg_ctx_set_stream(lk_reg_ctx* ctx, void* stream) {
    if (!ctx) return fail(LK_INVALID_ARGUMENT, "null context");
    std::lock_guard<std::mutex> lock(ctx->mu);
    cudaSetDevice(ctx->device);
    // the run buffers are (re)allocated and freed stream-ordered: finish the
    // old stream's work and move the buffers' stream with the kernels, so a
    // buffer freed on growth is ordered after every kernel that read it
    const cudaError_t e = cudaStreamSynchronize(ctx->stream);
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
    ctx->rb.stream = ctx->stream;
    if (e != cudaSuccess) return fail(LK_CUDA_ERROR, cudaGetErrorString(e));
    return LK_OK;
}

lk_status lk_reg_ctx_set_profiling(lk_reg_ctx* ctx, int32_t enable) {
    if (!ctx) return fail(LK_INVALID_ARGUMENT, "null context");
    std::lock_guard<std::mutex> lock(ctx->mu);
    ctx->profile = enable != 0;
    return LK_OK;
}

lk_status lk_reg_ctx_kernel_times(lk_reg_ctx* ctx, double* ms3, int64_t* runs, int32_t reset) {
    if (!ctx) return fail(LK_INVALID_ARGUMENT, "null context");
    std::lock_guard<std::mutex> lock(ctx->mu);
    cudaSetDevice(ctx->device);
    ctx->drain_events();
    if (ms3) {
        ms3[0] = ctx->kernel_ms[0];
        ms3[1] = ctx->kernel_ms[1];
        ms3[2] = 0.0;
        for (int k = 2; k < lkk::kPhaseEvents - 1; ++k) ms3[2] += ctx->kernel_ms[k];
    }
    if (runs) *runs = ctx->profiled_runs;
    if (reset) {
        for (double& v : ctx->kernel_ms) v = 0.0;
        ctx->profiled_runs = 0;
    }
    return LK_OK;
}

lk_status lk_reg_ctx_phase_times(lk_reg_ctx* ctx, double* ms, int32_t n_phases, int64_t* runs, int32_t reset) {
    if (!ctx) return fail(LK_INVALID_ARGUMENT, "null context");
    if (n_phases < 0 || (n_phases > 0 && !ms)) return fail(LK_INVALID_ARGUMENT, "null argument");
    std::lock_guard<std::mutex> lock(ctx->mu);
    cudaSetDevice(ctx->device);
    ctx->drain_events();
    for (int k = 0; k < n_phases; ++k) ms[k] = k < lkk::kPhaseEvents - 1 ? ctx->kernel_ms[k] : 0.0;
    if (runs) *runs = ctx->profiled_runs;
    if (reset) {
        for (double& v : ctx->kernel_ms) v = 0.0;
        ctx->profiled_runs = 0;
    }
    return LK_OK;
}

lk_status lk_reg_ctx_sizes(const lk_reg_ctx* ctx, int64_t* n_source, int64_t* n_target) {
    if (!ctx) return fail(LK_INVALID_ARGUMENT, "null context");
    if (n_source) *n_source = ctx->ns;
    if (n_target) *n_target = ctx->nt;
    return LK_OK;
}

lk_status lk_reg_ctx_download(const lk_reg_ctx* c, double* src_xyz, double* src_n, double* tgt_xyz, double* tgt_n,
                              int32_t* cache, float* src_features, float* tgt_features) {
    return guarded([&]() -> lk_status {
        if (!c) return fail(LK_INVALID_ARGUMENT, "null context");
        CK(cudaSetDevice(c->device));
        auto cp = [&](void* dst, const void* d, size_t bytes) {
            if (dst && d && bytes) CK(cudaMemcpyAsync(dst, d, bytes, cudaMemcpyDeviceToHost, c->stream));
        };
        cp(src_xyz, c->d_spos, 3 * c->ns * sizeof(double));
        cp(src_n, c->d_snrm, 3 * c->ns * sizeof(double));
        cp(tgt_xyz, c->d_tpos, 3 * c->nt * sizeof(double));
        cp(tgt_n, c->d_tnrm, 3 * c->nt * sizeof(double));
        cp(cache, c->d_cache, c->ns * sizeof(int32_t));
        cp(src_features, c->d_sfeat, 33 * c->ns * sizeof(float));
        cp(tgt_features, c->d_tfeat, 33 * c->nt * sizeof(float));
        CK(cudaStreamSynchronize(c->stream));
        return LK_OK;
    });
}

lk_status lk_reg_run_range(lk_reg_ctx* ctx, const lk_reg_params* params, int64_t begin, int64_t end,
                           lk_reg_record* record, int32_t record_on_device) {
    return guarded([&]() -> lk_status {
        if (!ctx || !params || !record) return fail(LK_INVALID_ARGUMENT, "null argument");
        std::lock_guard<std::mutex> lock(ctx->mu);
        void* target = record_on_device ? static_cast<void*>(record) : static_cast<void*>(ctx->d_record);
        lk_status st = run_range_impl(ctx, *params, begin, end, target);
        if (st != LK_OK) return st;
        if (!record_on_device) {
            CK(cudaMemcpyAsync(record, ctx->d_record, sizeof(lk_reg_record), cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
        }
        return LK_OK;
    });
}

lk_status lk_reg_merge_records(const lk_reg_record* records, int32_t count, int64_t n_source, lk_reg_result* result,
                               lk_hyp_stats* stats) {
    if (!records || count <= 0 || !result || n_source <= 0) return fail(LK_INVALID_ARGUMENT, "bad merge arguments");
    const lk_reg_record* best = nullptr;
    lk_hyp_stats st{};
    for (int32_t g = 0; g < count; ++g) {
        const lk_reg_record& r = records[g];
        st.sampled += r.sampled;
        st.prerejected += r.prerejected;
        st.degenerate += r.degenerate;
        st.evaluated += r.evaluated;
        st.qualified += r.qualified;
        st.w_ref += r.w_ref;
        st.evals_executed += r.evals_executed;
        if (r.valid && (!best || record_better(r, *best))) best = &r;
    }
    lk_reg_record none{};
    record_to_result(best ? *best : none, n_source, result);
    if (stats) {
        double ps = stats->prepare_seconds, hs = stats->hypothesis_seconds;
        *stats = st;
        stats->prepare_seconds = ps;
        stats->hypothesis_seconds = hs;
    }
    return result->found ? LK_OK : LK_NO_ALIGNMENT;
}

lk_status lk_reg_run_hypotheses(lk_reg_ctx* ctx, const lk_reg_params* params, lk_reg_result* result,
                                lk_hyp_stats* stats) {
    return guarded([&]() -> lk_status {
        if (!ctx || !params || !result) return fail(LK_INVALID_ARGUMENT, "null argument");
        if (params->hypothesis_count < 0) return fail(LK_INVALID_ARGUMENT, "negative hypothesis_count");
        std::lock_guard<std::mutex> lock(ctx->mu);
        double t0 = now_s();
        const int G = ctx->nranks;
        std::vector<lk_reg_record> recs(static_cast<size_t>(G));
        auto* hrec = static_cast<lk_reg_record*>(lkk::host_scratch(G * sizeof(lk_reg_record)));
        if (!hrec) CK(cudaErrorMemoryAllocation);
        if (ctx->comm) {
            lk_status st = exchange_run(ctx, *params);
            if (st != LK_OK) return st;
            CK(cudaMemcpyAsync(hrec, ctx->d_xbuf, G * sizeof(lk_reg_record), cudaMemcpyDeviceToHost, ctx->stream));
            for (lk_reg_ctx* q : ctx->peers) {
                CK(cudaSetDevice(q->device));
                CK(cudaStreamSynchronize(q->stream));
            }
            CK(cudaSetDevice(ctx->device));
        } else {
            lk_status st = run_range_impl(ctx, *params, 0, params->hypothesis_count, ctx->d_record);
            if (st != LK_OK) return st;
            CK(cudaMemcpyAsync(hrec, ctx->d_record, sizeof(lk_reg_record), cudaMemcpyDeviceToHost, ctx->stream));
        }
        CK(cudaStreamSynchronize(ctx->stream));
        std::memcpy(recs.data(), hrec, G * sizeof(lk_reg_record));
        double t1 = now_s();
        lk_hyp_stats local{};
        lk_hyp_stats* sp = stats ? stats : &local;
        double prep = sp->prepare_seconds;
        lk_status ms = lk_reg_merge_records(recs.data(), G, ctx->ns, result, sp);
        sp->prepare_seconds = prep;
        sp->hypothesis_seconds = t1 - t0;
        return ms;
    });
}

lk_status lk_nccl_unique_id(uint8_t id[128]) {
    return guarded([&]() -> lk_status {
        if (!id) return fail(LK_INVALID_ARGUMENT, "null argument");
        ncclUniqueId u;
        static_assert(sizeof(u.internal) == 128, "NCCL unique id size");
        NK(nccl().GetUniqueId(&u));
        std::memcpy(id, u.internal, 128);
        return LK_OK;
    });
}

lk_status lk_reg_ctx_attach_comm(lk_reg_ctx* ctx, const uint8_t id[128], int32_t nranks, int32_t rank) {
    return guarded([&]() -> lk_status {
        if (!ctx || !id) return fail(LK_INVALID_ARGUMENT, "null argument");
        if (nranks < 1 || rank < 0 || rank >= nranks) return fail(LK_INVALID_ARGUMENT, "bad rank / nranks");
        std::lock_guard<std::mutex> lock(ctx->mu);
        if (ctx->comm) return fail(LK_INVALID_ARGUMENT, "context already has a communicator");
        CK(cudaSetDevice(ctx->device));
        ncclUniqueId u;
        std::memcpy(u.internal, id, 128);
        NK(nccl().CommInitRank(&ctx->comm, nranks, u, rank));
        ctx->nranks = nranks;
        ctx->rank = rank;
        CK(lkk::pool_alloc(&ctx->d_xbuf, nranks * sizeof(lk_reg_record), ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        return LK_OK;
    });
}

lk_status lk_reg_run_exchange(lk_reg_ctx* ctx, const lk_reg_params* params, lk_reg_record* records_dev) {
    return guarded([&]() -> lk_status {
        if (!ctx || !params || !records_dev) return fail(LK_INVALID_ARGUMENT, "null argument");
        if (params->hypothesis_count < 0) return fail(LK_INVALID_ARGUMENT, "negative hypothesis_count");
        std::lock_guard<std::mutex> lock(ctx->mu);
        if (ctx->comm) {
            const lk_status st = exchange_run(ctx, *params);
            if (st != LK_OK) return st;
            CK(cudaMemcpyAsync(records_dev, ctx->d_xbuf, ctx->nranks * sizeof(lk_reg_record), cudaMemcpyDeviceToDevice,
                               ctx->stream));
            for (lk_reg_ctx* q : ctx->peers) {  // the caller waits on the context stream only
                cudaEvent_t done;
                CK(cudaSetDevice(q->device));
                CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
                CK(cudaEventRecord(done, q->stream));
                CK(cudaSetDevice(ctx->device));
                CK(cudaStreamWaitEvent(ctx->stream, done, 0));
                CK(cudaSetDevice(q->device));
                cudaEventDestroy(done);
            }
            CK(cudaSetDevice(ctx->device));
            return LK_OK;
        }
        return run_range_impl(ctx, *params, 0, params->hypothesis_count, records_dev);
    });
}

lk_status lk_reg_ctx_topology(const lk_reg_ctx* ctx, int32_t* n_devices, int32_t* nranks, int32_t* rank) {
    if (!ctx) return fail(LK_INVALID_ARGUMENT, "null context");
    if (n_devices) *n_devices = 1 + static_cast<int32_t>(ctx->peers.size());
    if (nranks) *nranks = ctx->nranks;
    if (rank) *rank = ctx->rank;
    return LK_OK;
}

lk_status lk_register_global(const lk_cloud* src, const lk_cloud* tgt, const lk_reg_params* params,
                             lk_reg_result* result, lk_hyp_stats* stats) {
    lk_reg_ctx* ctx = nullptr;
    lk_status st = lk_reg_prepare(src, tgt, params, &ctx);
    if (st != LK_OK) return st;
    lk_hyp_stats local{};
    lk_hyp_stats* sp = stats ? stats : &local;
    sp->prepare_seconds = ctx->prepare_seconds;
    st = lk_reg_run_hypotheses(ctx, params, result, sp);
    std::string keep = g_err;
    lk_reg_ctx_destroy(ctx);
    g_err = keep;
    return st;
}

lk_status lk_grid_build(const lk_cloud* target, int32_t kind, double cell, double d_max, int32_t device,
                        lk_grid** out) {
    return guarded([&]() -> lk_status {
        if (!out) return fail(LK_INVALID_ARGUMENT, "null argument");
        check_cloud_ptr(target, "target");
        *out = nullptr;
        if (target->n == 0) return fail(LK_EMPTY_CLOUD, "build_grid: empty cloud");
        if (kind != 0 && kind != 1) return fail(LK_INVALID_ARGUMENT, "grid kind must be 0 or 1");
        if (kind == 0) cell = d_max;
        if (!(cell > 0.0)) return fail(LK_INVALID_ARGUMENT, "build_grid: cell_length must be positive");
        if (!(d_max > 0.0)) return fail(LK_INVALID_ARGUMENT, "build_grid: d_max must be positive");
        auto* g = new lk_grid();
        try {
            g->device = select_device(device);
            g->sm_count = sm_count_of(g->device);
            g->kind = kind;
            g->cell = cell;
            g->d_max = d_max;
            g->has_normals = target->nxyz != nullptr;
            CK(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
            g->rb.stream = g->stream;
            double* d_pos = dev_upload(target->xyz, 3 * target->n, g->stream);
            double* d_nrm = target->nxyz ? dev_upload(target->nxyz, 3 * target->n, g->stream) : nullptr;
            cudaError_t e = lkk::build_grid(g->g, kind, d_pos, d_nrm, target->n, cell, d_max, g->stream);
            // a dense target (full-resolution frames: tens of points per
            // EvalGrid cell) also gets a ring grid for explicit candidates
            if (e == cudaSuccess && kind == 0 && target->n >= kDenseTarget && fast_path_enabled()) {
                e = lkk::build_ring_grid(g->ring, d_pos, target->n, d_max, g->stream);
                g->has_ring = e == cudaSuccess;
            }
            if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
            cudaFree(d_pos);
            cudaFree(d_nrm);
            CK(e);
            CK(cudaMalloc(&g->d_record, sizeof(lk_reg_record)));
        } catch (...) {
            delete g;
            throw;
        }
        *out = g;
        return LK_OK;
    });
}

void lk_grid_destroy(lk_grid* grid) { delete grid; }

lk_status lk_grid_dims(const lk_grid* grid, double* origin3, double* cell, int32_t* dims3, int64_t* ncells,
                       int64_t* npoints) {
    if (!grid) return fail(LK_INVALID_ARGUMENT, "null grid");
    const lkk::GridView& v = grid->g.view;
    if (origin3) {
        origin3[0] = v.ox;
        origin3[1] = v.oy;
        origin3[2] = v.oz;
    }
    if (cell) *cell = v.cell;
    if (dims3) {
        dims3[0] = v.nx;
        dims3[1] = v.ny;
        dims3[2] = v.nz;
    }
    if (ncells) *ncells = grid->g.ncells;
    if (npoints) *npoints = grid->g.npoints;
    return LK_OK;
}

lk_status lk_grid_download(const lk_grid* grid, int32_t* start, int32_t* index, double* slot_xyz, double* slot_n,
                           uint8_t* near_occupied) {
    return guarded([&]() -> lk_status {
        if (!grid) return fail(LK_INVALID_ARGUMENT, "null grid");
        CK(cudaSetDevice(grid->device));
        const lkk::GridStorage& g = grid->g;
        if (start) CK(cudaMemcpy(start, g.start, (g.ncells + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost));
        if (index) CK(cudaMemcpy(index, g.index, g.npoints * sizeof(int32_t), cudaMemcpyDeviceToHost));
        if (slot_xyz) CK(cudaMemcpy(slot_xyz, g.slot_pos, 3 * g.npoints * sizeof(double), cudaMemcpyDeviceToHost));
        if (slot_n) CK(cudaMemcpy(slot_n, g.slot_nrm, 3 * g.npoints * sizeof(double), cudaMemcpyDeviceToHost));
        if (near_occupied) CK(cudaMemcpy(near_occupied, g.near, g.ncells, cudaMemcpyDeviceToHost));
        return LK_OK;
    });
}

lk_status lk_score_candidates(lk_grid* grid, const lk_cloud* src, const double* Rt, int64_t C,
                              const lk_reg_params* params, int32_t early_exit, lk_cand_score* per_cand,
                              lk_reg_result* best, int64_t* qualified) {
    return guarded([&]() -> lk_status {
        if (!grid || !params) return fail(LK_INVALID_ARGUMENT, "null argument");
        check_cloud_ptr(src, "source");
        if (C < 0 || (C > 0 && !Rt)) return fail(LK_INVALID_ARGUMENT, "bad candidate list");
        if (src->n == 0) return fail(LK_EMPTY_CLOUD, "evaluate_hypothesis: empty cloud");
        if (!src->nxyz || !grid->has_normals)
            return fail(LK_MISSING_NORMALS, "evaluate_hypothesis: both clouds need normals");
        std::lock_guard<std::mutex> lock(grid->mu);
        CK(cudaSetDevice(grid->device));
        cudaStream_t s = grid->stream;
        const int64_t ns = src->n;
        double* d_pos = dev_upload(src->xyz, 3 * ns, s);
        double* d_nrm = dev_upload(src->nxyz, 3 * ns, s);
        double* d_rt = dev_upload(Rt, 12 * static_cast<size_t>(C), s);
        int64_t* d_inl = nullptr;
        double* d_sum = nullptr;
        CK(cudaMalloc(&d_inl, std::max<int64_t>(C, 1) * sizeof(int64_t)));
        CK(cudaMalloc(&d_sum, std::max<int64_t>(C, 1) * sizeof(double)));
        float4* d_pos32 = nullptr;
        CK(cudaMalloc(&d_pos32, std::max<int64_t>(ns, 1) * sizeof(float4)));
        CK(lkk::make_source32(d_pos, ns, d_pos32, s));
        lkk::SourceView sv{d_pos, d_nrm, d_pos32, ns};
        lkk::ScoreParams sp = score_params(*params, ns, early_exit != 0, grid->kind == 1);
        if (fast_path_enabled()) lkk::configure_fast_path(sp, grid->g.view, max_norm(src->xyz, ns));
        lk_reg_record rec{};
        std::vector<int64_t> inl(C);
        std::vector<double> sum(C);
        cudaError_t e = lkk::score_candidates(sv, grid->g.view, sp, d_rt, C, grid->rb, d_inl, d_sum, grid->d_record,
                                              s, grid->sm_count, grid->has_ring ? &grid->ring.view : nullptr);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&rec, grid->d_record, sizeof(rec), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess && C)
            e = cudaMemcpyAsync(inl.data(), d_inl, C * sizeof(int64_t), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess && C) e = cudaMemcpyAsync(sum.data(), d_sum, C * sizeof(double), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        cudaFree(d_pos);
        cudaFree(d_nrm);
        cudaFree(d_pos32);
        cudaFree(d_rt);
        cudaFree(d_inl);
        cudaFree(d_sum);
        CK(e);
        if (per_cand) {
            for (int64_t k = 0; k < C; ++k) {
                lk_cand_score& o = per_cand[k];
                o.inliers = inl[k];
                if (inl[k] < 0) {
                    o.inlier_ratio = 0.0;
                    o.fitness = 0.0;
                } else {
                    o.inlier_ratio = static_cast<double>(inl[k]) / static_cast<double>(ns);
                    o.fitness = inl[k] > 0 ? sum[k] / static_cast<double>(inl[k]) : 0.0;
                }
            }
        }
        if (qualified) *qualified = rec.qualified;
        if (best) record_to_result(rec, ns, best);
        return LK_OK;
    });
}

// The pairs' clouds as per-pair host pointers with point offsets (validated).
struct PackedPairs {
    std::vector<const double*> qpos, qnrm, ppos, pnrm;
    std::vector<int64_t> offq, offp;
};

PackedPairs pack_pairs(const lk_cloud* ci, const lk_cloud* cj, int64_t K, bool normals) {
    PackedPairs pk;
    pk.offq.assign(static_cast<size_t>(K) + 1, 0);
    pk.offp.assign(static_cast<size_t>(K) + 1, 0);
    for (int64_t k = 0; k < K; ++k) {
        check_cloud_ptr(&ci[k], "cloud_i");
        check_cloud_ptr(&cj[k], "cloud_j");
        if (ci[k].n == 0 || cj[k].n == 0) throw lk::Status(LK_EMPTY_CLOUD, "edge_info: empty cloud");
        if (normals && (!ci[k].nxyz || !cj[k].nxyz))
            throw lk::Status(LK_MISSING_NORMALS, "evaluate_hypothesis: both clouds need normals");
        pk.offq[k + 1] = pk.offq[k] + ci[k].n;
        pk.offp[k + 1] = pk.offp[k] + cj[k].n;
        pk.qpos.push_back(ci[k].xyz);
        pk.ppos.push_back(cj[k].xyz);
        pk.qnrm.push_back(ci[k].nxyz);
        pk.pnrm.push_back(cj[k].nxyz);
    }
    if (pk.offq[K] > INT32_MAX / 2 || pk.offp[K] > INT32_MAX / 2)
        throw lk::Status(LK_INVALID_ARGUMENT, "verify: batch too large");
    return pk;
}

lk_status lk_propose_loops(const lk_cloud* fragments, const double* poses, int32_t n, const int32_t* loops,
                           int32_t n_loops, const lk_loop_params* params, lk_loop_proposal* out, int64_t capacity,
                           int64_t* n_out) {
    return guarded([&]() -> lk_status {
        if (!params || !n_out || n < 0 || n_loops < 0 || (n > 0 && (!fragments || !poses)) ||
            (n_loops > 0 && !loops) || (capacity > 0 && !out))
            return fail(LK_INVALID_ARGUMENT, "null argument");
        *n_out = 0;
        if (n == 0) return LK_OK;
        // grids in fragment order: build_grid throws EmptyCloud, then rejects the cell (grid.cpp:36-37)
        for (int32_t f = 0; f < n; ++f) {
            check_cloud_ptr(fragments + f, "fragment");
            if (fragments[f].n == 0) return fail(LK_EMPTY_CLOUD, "build_grid: empty cloud");
            if (!(params->overlap_radius > 0.0))
                return fail(LK_INVALID_ARGUMENT, "build_grid: cell_length must be positive");
        }
        NvtxRange range("lk_propose_loops");
        std::vector<int64_t> foff(static_cast<size_t>(n) + 1, 0);
        for (int32_t f = 0; f < n; ++f) foff[f + 1] = foff[f] + fragments[f].n;
        std::vector<double> xyz(static_cast<size_t>(3 * foff[n]));
        for (int32_t f = 0; f < n; ++f)
            std::memcpy(xyz.data() + 3 * foff[f], fragments[f].xyz, 3 * fragments[f].n * sizeof(double));
        // pairs i >= j + 2 not joined by a loop edge in either orientation (fragments.cpp:79-84,89-92)
        std::vector<int32_t> pairs;
        for (int32_t i = 2; i < n; ++i)
            for (int32_t j = 0; j + 2 <= i; ++j) {
                bool linked = false;
                for (int32_t e = 0; e < n_loops && !linked; ++e)
                    linked = (loops[2 * e] == i && loops[2 * e + 1] == j) || (loops[2 * e] == j && loops[2 * e + 1] == i);
                if (!linked) {
                    pairs.push_back(i);
                    pairs.push_back(j);
                }
            }
        const int32_t K = static_cast<int32_t>(pairs.size() / 2);
        std::vector<int64_t> hits(static_cast<size_t>(K > 0 ? K : 1));
        const int dev = select_device(params->device);
        cudaStream_t s = acquire_stream(dev);
        cudaError_t e = lkk::propose_loops(xyz.data(), foff.data(), n, poses, pairs.data(), K,
                                           params->overlap_radius, hits.data(), s);
        release_stream(dev, s);
        CK(e);
        std::vector<lk_loop_proposal> props;
        for (int32_t k = 0; k < K; ++k) {
            const int32_t i = pairs[2 * k], j = pairs[2 * k + 1];
            const double overlap = static_cast<double>(hits[k]) / static_cast<double>(fragments[i].n);
            if (overlap >= params->min_overlap) props.push_back(lk_loop_proposal{i, j, overlap});
        }
        // fragments.cpp:102-107: overlap desc, then i, then j (a strict total order)
        std::sort(props.begin(), props.end(), [](const lk_loop_proposal& a, const lk_loop_proposal& b) {
            if (a.overlap != b.overlap) return a.overlap > b.overlap;
            if (a.i != b.i) return a.i < b.i;
            return a.j < b.j;
        });
        *n_out = static_cast<int64_t>(props.size());
        for (int64_t k = 0; k < *n_out && k < capacity; ++k) out[k] = props[static_cast<size_t>(k)];
        return LK_OK;
    });
}

lk_status lk_edge_info_batched(const lk_cloud* clouds_i, const lk_cloud* clouds_j, const double* Ti, const double* Tj,
                               int64_t n_pairs, double epsilon, int32_t device, double* info, int64_t* pair_count) {
    return guarded([&]() -> lk_status {
        if (n_pairs < 0 || (n_pairs > 0 && (!clouds_i || !clouds_j || !Ti || !Tj || !info || !pair_count)))
            return fail(LK_INVALID_ARGUMENT, "null argument");
        if (!(epsilon > 0.0)) return fail(LK_INVALID_ARGUMENT, "build_grid: cell_length must be positive");
        if (n_pairs == 0) return LK_OK;
        if (n_pairs > INT32_MAX) return fail(LK_INVALID_ARGUMENT, "edge_info: batch too large");
        PackedPairs pk = pack_pairs(clouds_i, clouds_j, n_pairs, false);
        const int dev = select_device(device);
        cudaStream_t s = acquire_stream(dev);
        lkk::VerifyInput in{};
        in.n_pairs = static_cast<int32_t>(n_pairs);
        in.qpos = pk.qpos.data();
        in.ppos = pk.ppos.data();
        in.offq = pk.offq.data();
        in.offp = pk.offp.data();
        in.Ti = Ti;
        in.Tj = Tj;
        in.epsilon = epsilon;
        in.full = 0;
        std::vector<lkk::VerifyOutput> o(static_cast<size_t>(n_pairs));
        cudaError_t e = lkk::verify_batch(in, o.data(), s);
        release_stream(dev, s);
        CK(e);
        for (int64_t k = 0; k < n_pairs; ++k) {
            for (int q = 0; q < 36; ++q) info[36 * k + q] = o[k].info[q];
            pair_count[k] = o[k].pair_count;
        }
        return LK_OK;
    });
}

// One device's share of a verification batch (pairs [k0, k0 + K) of the call).
void verify_share(const lk_cloud* clouds_i, const lk_cloud* clouds_j, const double* Ti, const double* Tj,
                  const double* T, int64_t k0, int64_t K, const lk_verify_params* params, int dev,
                  lk_verify_result* out) {
    NvtxRange range("lk verify share");
    PackedPairs pk = pack_pairs(clouds_i + k0, clouds_j + k0, K, true);
    CK(cudaSetDevice(dev));
    cudaStream_t s = acquire_stream(dev);
    lkk::VerifyInput in{};
    in.n_pairs = static_cast<int32_t>(K);
    in.qpos = pk.qpos.data();
    in.qnrm = pk.qnrm.data();
    in.ppos = pk.ppos.data();
    in.pnrm = pk.pnrm.data();
    in.offq = pk.offq.data();
    in.offp = pk.offp.data();
    in.Ti = Ti + 12 * k0;
    in.Tj = Tj + 12 * k0;
    in.T = T + 12 * k0;
    in.epsilon = params->epsilon;
    in.overlap_radius = params->overlap_radius;
    in.d_max = params->d_max;
    in.grid_cell = params->grid_cell > 0.0 ? params->grid_cell : params->d_max;
    in.cos_max = std::cos(params->normal_angle_max);  // registration.cpp:61
    in.full = 1;
    std::vector<lkk::VerifyOutput> o(static_cast<size_t>(K));
    cudaError_t e = lkk::verify_batch(in, o.data(), s);
    release_stream(dev, s);
    CK(e);
    for (int64_t k = 0; k < K; ++k) {
        lk_verify_result& r = out[k0 + k];
        for (int q = 0; q < 36; ++q) r.info[q] = o[k].info[q];
        r.pair_count = o[k].pair_count;
        r.overlap_hits = o[k].overlap_hits;
        const double np = static_cast<double>(clouds_j[k0 + k].n);
        r.overlap = static_cast<double>(o[k].overlap_hits) / np;
        r.inliers = o[k].inliers;
        r.inlier_ratio = static_cast<double>(o[k].inliers) / np;
        r.fitness = o[k].inliers > 0 ? o[k].sq_sum / static_cast<double>(o[k].inliers) : 0.0;
    }
}

lk_status lk_verify_batch(const lk_cloud* clouds_i, const lk_cloud* clouds_j, const double* Ti, const double* Tj,
                          const double* T, int64_t n_pairs, const lk_verify_params* params, lk_verify_result* out) {
    return guarded([&]() -> lk_status {
        if (!params || n_pairs < 0 || (n_pairs > 0 && (!clouds_i || !clouds_j || !Ti || !Tj || !T || !out)))
            return fail(LK_INVALID_ARGUMENT, "null argument");
        if (!(params->epsilon > 0.0) || !(params->overlap_radius > 0.0) || !(params->d_max > 0.0))
            return fail(LK_INVALID_ARGUMENT, "build_grid: cell_length must be positive");
        if (n_pairs == 0) return LK_OK;
        if (n_pairs > INT32_MAX) return fail(LK_INVALID_ARGUMENT, "verify: batch too large");
        pack_pairs(clouds_i, clouds_j, n_pairs, true);  // validation in pair order, before any device work
        std::vector<int> devs = call_devices(params->device, params->device_count);
        const int G = static_cast<int>(std::min<int64_t>(static_cast<int64_t>(devs.size()), n_pairs));
        if (G <= 1) {
            verify_share(clouds_i, clouds_j, Ti, Tj, T, 0, n_pairs, params, devs[0], out);
            return LK_OK;
        }
        // the pairs are independent: contiguous shares, one host thread per device, no exchange
        std::vector<std::thread> th;
        std::vector<std::exception_ptr> errs(static_cast<size_t>(G));
        for (int g = 0; g < G; ++g) {
            const int64_t k0 = g * n_pairs / G, k1 = (g + 1) * n_pairs / G;
            th.emplace_back([&, g, k0, k1] {
                try {
                    verify_share(clouds_i, clouds_j, Ti, Tj, T, k0, k1 - k0, params, devs[g], out);
                } catch (...) {
                    errs[g] = std::current_exception();
                }
            });
        }
        for (auto& t : th) t.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
        CK(cudaSetDevice(devs[0]));
        return LK_OK;
    });
}

lk_status lk_icp_point_to_plane(const lk_cloud* source, const lk_cloud* target, const double* T0,
                                const lk_icp_params* params, lk_icp_result* result, double* history) {
    return guarded([&]() -> lk_status {
        if (!T0 || !params || !result) return fail(LK_INVALID_ARGUMENT, "null argument");
        check_cloud_ptr(source, "source");
        check_cloud_ptr(target, "target");
        if (source->n == 0 || target->n == 0) return fail(LK_EMPTY_CLOUD, "icp: empty cloud");
        if (!target->nxyz) return fail(LK_MISSING_NORMALS, "icp: target normals required");
        const double dmax = params->max_correspondence_distance;
        if (!(dmax > 0.0)) return fail(LK_INVALID_ARGUMENT, "icp: max_correspondence_distance must be positive");
        if (params->max_iterations < 0) return fail(LK_INVALID_ARGUMENT, "icp: max_iterations must be >= 0");
        const int dev = select_device(params->device);
        const int sms = sm_count_of(dev);
        cudaStream_t s = acquire_stream(dev);
        lkk::RingStorage g;
        double *d_src = nullptr, *d_tp = nullptr, *d_tn = nullptr, *d_hist = nullptr;
        lkk::IcpOutcome o{};
        double R[9], t[3];
        cudaError_t e = cudaSuccess;
        try {
            d_src = dev_upload(source->xyz, 3 * source->n, s);
            d_tp = dev_upload(target->xyz, 3 * target->n, s);
            d_tn = dev_upload(target->nxyz, 3 * target->n, s);
            const int64_t hn = 3 * static_cast<int64_t>(params->max_iterations);
            if (history && hn > 0) CK(cudaMalloc(&d_hist, hn * sizeof(double)));
            e = lkk::build_ring_grid(g, d_tp, target->n, dmax, s, fast_path_enabled());
            if (e == cudaSuccess)
                e = lkk::icp_point_to_plane(d_src, source->n, g, d_tn, dmax, params->max_iterations,
                                            params->convergence_eps, T0, T0 + 9, R, t, &o, d_hist, s, sms);
            if (e == cudaSuccess && d_hist)
                e = cudaMemcpyAsync(history, d_hist, hn * sizeof(double), cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        } catch (...) {
            g.release();
            lkk::pool_free(d_src, s);
            lkk::pool_free(d_tp, s);
            lkk::pool_free(d_tn, s);
            cudaStreamSynchronize(s);
            cudaFree(d_hist);
            release_stream(dev, s);
            throw;
        }
        g.release();
        lkk::pool_free(d_src, s);
        lkk::pool_free(d_tp, s);
        lkk::pool_free(d_tn, s);
        cudaStreamSynchronize(s);
        cudaFree(d_hist);
        release_stream(dev, s);
        CK(e);
        if (o.status == LK_NO_CORRESPONDENCES)
            return fail(LK_NO_CORRESPONDENCES, "icp: fewer than 6 correspondences");
        for (int k = 0; k < 9; ++k) result->R[k] = R[k];
        for (int k = 0; k < 3; ++k) result->t[k] = t[k];
        result->iterations = o.iterations;
        result->converged = o.converged;
        result->correspondences = o.correspondences;
        result->rmse = o.rmse;
        result->fitness = o.fitness;
        return LK_OK;
    });
}

lk_status lk_feature_nn_cache(const float* src_features, int64_t ns, const float* tgt_features, int64_t nt,
                              int32_t device, int32_t* cache) {
    return guarded([&]() -> lk_status {
        if (ns <= 0 || nt <= 0) return fail(LK_MISSING_DATA, "feature_nn_cache: empty feature set");
        if (!src_features || !tgt_features || !cache) return fail(LK_INVALID_ARGUMENT, "null argument");
        select_device(device);
        cudaStream_t s;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        float* d_sf = dev_upload(src_features, 33 * ns, s);
        float* d_tf = dev_upload(tgt_features, 33 * nt, s);
        int32_t* d_out = nullptr;
        cudaError_t e = cudaMalloc(&d_out, ns * sizeof(int32_t));
        if (e == cudaSuccess) e = lkk::feature_nn(d_sf, ns, d_tf, nt, d_out, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(cache, d_out, ns * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        cudaFree(d_sf);
        cudaFree(d_tf);
        cudaFree(d_out);
        cudaStreamDestroy(s);
        CK(e);
        return LK_OK;
    });
}

lk_status lk_estimate_normals(const lk_cloud* cloud, double radius, const double* viewpoint, int32_t device,
                              double* out_normals) {
    return guarded([&]() -> lk_status {
        check_cloud_ptr(cloud, "cloud");
        if (!out_normals) return fail(LK_INVALID_ARGUMENT, "null argument");
        if (cloud->n == 0) return fail(LK_EMPTY_CLOUD, "estimate_normals: empty cloud");
        if (!(radius > 0.0)) return fail(LK_INVALID_ARGUMENT, "build_grid: cell_length must be positive");
        const double origin[3] = {0.0, 0.0, 0.0};
        const int dev = select_device(device);
        cudaStream_t s = acquire_stream(dev);
        double* d_in = nullptr;
        double* d_out = nullptr;
        cudaError_t e = cudaSuccess;
        try {
            d_in = dev_upload(cloud->xyz, 3 * cloud->n, s);
            CK(lkk::pool_alloc(&d_out, 3 * cloud->n * sizeof(double), s));
            e = lkk::estimate_normals(d_in, cloud->n, radius, viewpoint ? viewpoint : origin, d_out, s);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(out_normals, d_out, 3 * cloud->n * sizeof(double), cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        } catch (...) {
            lkk::pool_free(d_in, s);
            lkk::pool_free(d_out, s);
            release_stream(dev, s);
            throw;
        }
        lkk::pool_free(d_in, s);
        lkk::pool_free(d_out, s);
        cudaStreamSynchronize(s);
        release_stream(dev, s);
        CK(e);
        return LK_OK;
    });
}

lk_status lk_voxel_downsample(const lk_cloud* cloud, double leaf, double* out_xyz, double* out_n, int64_t* out_count) {
    return guarded([&]() -> lk_status {
        check_cloud_ptr(cloud, "cloud");
        if (!out_xyz || !out_count) return fail(LK_INVALID_ARGUMENT, "null argument");
        if (cloud->n == 0) return fail(LK_EMPTY_CLOUD, "voxel_downsample: empty cloud");
        if (!(leaf > 0.0)) return fail(LK_INVALID_ARGUMENT, "voxel_downsample: leaf must be positive");
        select_device(-1);
        cudaStream_t s;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        double* d_in = dev_upload(cloud->xyz, 3 * cloud->n, s);
        double* d_inn = cloud->nxyz ? dev_upload(cloud->nxyz, 3 * cloud->n, s) : nullptr;
        double *d_out = nullptr, *d_outn = nullptr;
        cudaError_t e = cudaMalloc(&d_out, 3 * cloud->n * sizeof(double));
        if (e == cudaSuccess && d_inn) e = cudaMalloc(&d_outn, 3 * cloud->n * sizeof(double));
        int st = 0;
        int64_t cnt = 0;
        if (e == cudaSuccess) e = lkk::voxel_downsample(d_in, d_inn, cloud->n, leaf, d_out, d_outn, &cnt, &st, s);
        if (e == cudaSuccess && st == 0)
            e = cudaMemcpyAsync(out_xyz, d_out, 3 * cnt * sizeof(double), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess && st == 0 && out_n && d_outn)
            e = cudaMemcpyAsync(out_n, d_outn, 3 * cnt * sizeof(double), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        cudaFree(d_in);
        cudaFree(d_inn);
        cudaFree(d_out);
        cudaFree(d_outn);
        cudaStreamDestroy(s);
        CK(e);
        if (st == 5) return fail(LK_MISSING_NORMALS, "normals must be unit length or exactly zero");
        *out_count = cnt;
        return LK_OK;
    });
}

lk_status lk_compute_fpfh(const lk_cloud* cloud, double radius, int32_t threads, float* out) {
    (void)threads;  // the device implementation has no host thread knob
    return guarded([&]() -> lk_status {
        check_cloud_ptr(cloud, "cloud");
        if (!out) return fail(LK_INVALID_ARGUMENT, "null argument");
        if (cloud->n == 0) return fail(LK_EMPTY_CLOUD, "compute_fpfh: empty cloud");
        if (!cloud->nxyz) return fail(LK_MISSING_NORMALS, "compute_fpfh: cloud has no normals");
        if (!(radius > 0.0)) return fail(LK_INVALID_ARGUMENT, "build_grid: cell_length must be positive");
        // validate_cloud (proj/src/geometry.cpp:93-103): unit length (1e-6) or exactly zero
        for (int64_t i = 0; i < cloud->n; ++i) {
            const double* q = cloud->nxyz + 3 * i;
            const double len = std::sqrt((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]);
            if (len != 0.0 && std::abs(len - 1.0) > 1e-6)
                return fail(LK_MISSING_NORMALS, "normals must be unit length or exactly zero");
        }
        select_device(-1);
        cudaStream_t s;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        double* d_p = dev_upload(cloud->xyz, 3 * cloud->n, s);
        double* d_n = dev_upload(cloud->nxyz, 3 * cloud->n, s);
        float* d_f = nullptr;
        cudaError_t e = cudaMalloc(&d_f, 33 * cloud->n * sizeof(float));
        if (e == cudaSuccess) e = lkk::compute_fpfh(d_p, d_n, cloud->n, radius, d_f, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(out, d_f, 33 * cloud->n * sizeof(float), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        cudaFree(d_p);
        cudaFree(d_n);
        cudaFree(d_f);
        cudaStreamDestroy(s);
        CK(e);
        return LK_OK;
    });
}

// ---- line-process weight (row a11; host) -----------------------------------
namespace {

lk::Rigid rigid12(const double* T) {
    lk::Rigid r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.R.m[i][j] = T[3 * i + j];
    r.t = {T[9], T[10], T[11]};
    return r;
}

// rotation_angle (geometry.cpp:23-26)
double rotation_angle(const lk::Mat3& r) {
    const double c = ((r.m[0][0] + r.m[1][1]) + r.m[2][2] - 1.0) / 2.0;
    return std::acos(std::clamp(c, -1.0, 1.0));
}

// xi = twist(rel * T_j^-1 * T_i) (line_process.cpp:37-38, geometry.cpp:28-40);
// false when the rotation angle reaches pi/2 (RotationTooLarge)
bool residual_twist(const double* Ti, const double* Tj, const double* rel, double xi[6]) {
    const lk::Rigid d = lk::compose(rigid12(rel), lk::compose(lk::inverse(rigid12(Tj)), rigid12(Ti)));
    if (rotation_angle(d.R) >= M_PI / 2.0) return false;
    xi[1] = std::asin(std::clamp(d.R.m[0][2], -1.0, 1.0));  // beta
    xi[0] = std::atan2(-d.R.m[1][2], d.R.m[2][2]);          // alpha
    xi[2] = std::atan2(-d.R.m[0][1], d.R.m[0][0]);          // gamma
    xi[3] = d.t.x;
    xi[4] = d.t.y;
    xi[5] = d.t.z;
    return true;
}

// xi.dot(info * xi) (line_process.cpp:39) in Eigen 3.4's SSE2 order (the rules
// of oracle/ref_shim/Eigen/Dense, checked against the reference build in
// tests/test_ref_parity.py): the Mat6 * Vec6 lazy product evaluates all six
// rows as packets, k in order (m_i0 x0 + m_i1 x1) + ...; the Vec6 dot reduces
// three packets by halving, lane-wise, then adds the two lanes:
// (p0 + (p2 + p4)) + (p1 + (p3 + p5)) with p_k = xi_k y_k.
double quad_form(const double* info36, const double xi[6]) {
    double y[6];
    for (int i = 0; i < 6; ++i) {
        double a = info36[6 * i] * xi[0];
        for (int k = 1; k < 6; ++k) a = info36[6 * i + k] * xi[k] + a;
        y[i] = a;
    }
    double p[6];
    for (int k = 0; k < 6; ++k) p[k] = xi[k] * y[k];
    return (p[0] + (p[2] + p[4])) + (p[1] + (p[3] + p[5]));
}

double update_weight(double f, double mu) {  // line_process.cpp:42-46
    if (!(mu > 0.0)) return 0.0;
    const double r = mu / (mu + std::max(f, 0.0));
    return std::clamp(r * r, 0.0, 1.0);
}

}  // namespace

lk_status lk_edge_residual(const double* Ti, const double* Tj, const double* rel, const double* info36, double* f) {
    return guarded([&]() -> lk_status {
        if (!Ti || !Tj || !rel || !info36 || !f) return fail(LK_INVALID_ARGUMENT, "null argument");
        double xi[6];
        if (!residual_twist(Ti, Tj, rel, xi))
            return fail(LK_ROTATION_TOO_LARGE, "twist_from_transform: rotation angle >= pi/2");
        *f = quad_form(info36, xi);
        return LK_OK;
    });
}

double lk_update_weight(double f, double mu) { return update_weight(f, mu); }

lk_status lk_loop_weights(int64_t n, const double* Ti, const double* Tj, const double* rel, const double* info36,
                          const int64_t* pair_count, double mu_tau, double threshold, double* weight,
                          int32_t* accepted) {
    return guarded([&]() -> lk_status {
        if (n < 0 || (n > 0 && (!Ti || !Tj || !rel || !info36 || !pair_count || !weight)))
            return fail(LK_INVALID_ARGUMENT, "null argument");
        for (int64_t k = 0; k < n; ++k) {
            const double mu = mu_tau * static_cast<double>(pair_count[k]);
            double xi[6];
            // loop_residual (line_process.cpp:52-60): outside the small-angle
            // regime the edge gets weight 0
            const bool ok = residual_twist(Ti + 12 * k, Tj + 12 * k, rel + 12 * k, xi);
            weight[k] = ok ? update_weight(quad_form(info36 + 36 * k, xi), mu) : 0.0;
            if (accepted) accepted[k] = weight[k] >= threshold ? 1 : 0;
        }
        return LK_OK;
    });
}

}  // extern "C"
