// capi.cu -- the C ABI (include/ffsga_cuda.h): handles, device memory, launch sequences.
//
// Host code here only validates, lays data out for the device and sequences launches; every
// evaluation, breeding step, replacement, archive update and migration runs in kernels.cu.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstddef>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>

#include <nvtx3/nvToolsExt.h>
#include <numeric>
#include <string>
#include <vector>

#include "ffsga_cuda.h"
#include "launch.h"

using namespace ffsga_dev;

namespace {

thread_local std::string g_err;
std::atomic<long long> g_launches{0};

struct Fail {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, std::string msg) { throw Fail{code, std::move(msg)}; }

#define CK(x)                                                                                      \
    do {                                                                                           \
        cudaError_t e_ = (x);                                                                      \
        if (e_ != cudaSuccess) fail(FFSGA_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

template <typename F>
int guard(F&& f) {
    try {
        f();
        return FFSGA_OK;
    } catch (const Fail& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return FFSGA_ERR_CUDA;
    }
}

// Device memory comes from the device's stream-ordered pool with an unbounded release
// threshold: freed island/batch buffers stay mapped and the next instance or island reuses them
// without a new mapping (a solver process that builds several models pays the mapping once).
// Allocation and release keep cudaMalloc/cudaFree's synchronous semantics.
inline void pool_setup_once() {
    static std::once_flag once[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
    std::call_once(once[dev], [dev] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        cudaGetLastError();
    });
}

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    // Stream on which every use of the buffer is ordered (island and batch buffers: the instance
    // stream).  Such a buffer is freed stream-ordered, without blocking the host or other
    // instances' work; an unowned buffer keeps cudaFree's device-wide synchronisation.
    cudaStream_t owner = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) {
            if (owner) {
                cudaFreeAsync(p, owner);
            } else {
                cudaDeviceSynchronize();  // every use of the buffer has completed (cudaFree semantics)
                cudaFreeAsync(p, 0);
            }
        }
        p = nullptr;
        bytes = 0;
    }
    void alloc(size_t n) {
        release();
        if (n == 0) n = 16;
        pool_setup_once();
        cudaError_t e = cudaMallocAsync(&p, n, 0);
        if (e == cudaSuccess) e = cudaStreamSynchronize(0);  // usable from every stream
        if (e != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            fail(e == cudaErrorMemoryAllocation ? FFSGA_ERR_OOM : FFSGA_ERR_CUDA,
                 std::string("device allocation of ") + std::to_string(n) + " bytes failed: " + cudaGetErrorString(e));
        }
        bytes = n;
    }
    void ensure(size_t n) {
        if (n > bytes) alloc(n);
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

template <typename T>
void upload(DevBuf& b, const std::vector<T>& v) {
    b.alloc(sizeof(T) * std::max<size_t>(v.size(), 1));
    if (!v.empty()) CK(cudaMemcpy(b.p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
}

unsigned long long coin_threshold(double p) {  // (u>>11) < ceil(p * 2^53)  <=>  unit(u) < p
    return (unsigned long long)std::ceil(p * 9007199254740992.0);
}

int bit_width_u(unsigned v) {
    int w = 0;
    while (v) {
        ++w;
        v >>= 1;
    }
    return w;
}

std::string gene_error(unsigned long long code) {
    const int stage = (int)((code >> 16) & 0xFFFFull);
    const int job = (int)(code & 0xFFFFull);
    return "decode: machine index out of range at job " + std::to_string(job) + " stage " + std::to_string(stage);
}

constexpr unsigned long long kNoError = ~0ull;

// NVTX range over one C-ABI call (nsys / ncu --nvtx timelines; header-only NVTX 3, no cost
// without a tool attached)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace

// ------------------------------------------------------------------------------ instance
struct ffsga_cuda_instance_t {
    int device = 0;
    int sm_count = 0;
    int J = 0, S = 0, Jpad = 0, maxM = 0;
    std::vector<int> M, stage_off, bps, sbo;
    int bpj = 0, total_bits = 0, words = 0;
    double weight = 0, emax = 0;
    DevInst d{};
    DevBuf dM, dStageOff, dBps, dSbo, dProcT, dRelease, dDue, dRelOrder, dBitStage;
    EvalConfig ec{};       // standalone batches: full-size CTAs
    EvalConfig ec_step{};  // joint GA step (FFSGA_STEP_WARPS: experiments)
    cudaStream_t stream = nullptr;
    std::vector<cudaStream_t> side;      // joint step: streams of step groups 1.. (group 0: stream)
    std::vector<cudaEvent_t> side_join;
    int step_split = 1;                  // joint step: groups per island kind (measured best at C3)
    int step_mix = 0;                    // joint step: > 0 = that many groups holding both kinds
    cudaEvent_t fork = nullptr, join = nullptr;
    // CUDA graph of `graph_chunk` generations of the last joint step (relaunched while the
    // island set and the work-list buffers are unchanged)
    cudaGraphExec_t graph_exec = nullptr;
    std::vector<const void*> graph_key;
    std::mutex mu;
    // joint-step work list
    DevBuf wl_ptrs, wl_obj, wl_fit, wl_count, cell_desc, pseudo_desc;
    // evaluate() staging
    DevBuf ev_in, ev_rows, ev_obj, ev_fit, ev_mk, ev_td, ev_err;
    long long ev_cap = 0;
    // host-batch evaluation pipeline (evaluate_host): pinned staging pair, copy stream, second
    // device input buffer, whole-batch results and per-sub-batch error slots
    void* pin[2] = {nullptr, nullptr};
    size_t pin_bytes = 0;
    cudaStream_t cstream = nullptr;
    cudaEvent_t pin_free[2] = {nullptr, nullptr}, in_ready[2] = {nullptr, nullptr}, in_free[2] = {nullptr, nullptr};
    DevBuf ev_in2, ev_res, ev_errs;
    DevBuf sched;  // K7 schedule of ffsga_cuda_decode (machine, start, completion)
    // migration scratch
    DevBuf mg_keys0, mg_keys1, mg_idx0, mg_idx_a, mg_idx_b, mg_temp;
    // timing: event pairs recorded around launches, resolved lazily (no sync in the timed path)
    bool timing = false;
    double t_ms[3] = {0, 0, 0};
    double t_busy[3] = {0, 0, 0};  // union of the launch intervals (concurrent streams counted once)
    long long t_n[3] = {0, 0, 0};
    struct Pending {
        int which;
        cudaEvent_t a, b;
    };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> pool;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, st0 = nullptr, st1 = nullptr;
    bool step_recorded = false;
    DevBuf eval_total;  // evaluations performed by ffsga_cuda_step (device counter)

    size_t block() const { return (size_t)S * Jpad; }
    void use() const { CK(cudaSetDevice(device)); }
    ~ffsga_cuda_instance_t() {
        cudaSetDevice(device);
        if (cstream) cudaStreamSynchronize(cstream);
        for (int k = 0; k < 2; ++k) {
            if (pin[k]) cudaFreeHost(pin[k]);
            for (cudaEvent_t e : {pin_free[k], in_ready[k], in_free[k]})
                if (e) cudaEventDestroy(e);
        }
        if (cstream) cudaStreamDestroy(cstream);
        if (stream) cudaStreamDestroy(stream);
        for (auto s : side) cudaStreamDestroy(s);
        for (auto e : side_join) cudaEventDestroy(e);
        if (fork) cudaEventDestroy(fork);
        if (join) cudaEventDestroy(join);
        if (graph_exec) cudaGraphExecDestroy(graph_exec);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (st0) cudaEventDestroy(st0);
        if (st1) cudaEventDestroy(st1);
        for (auto& p : pending) {
            cudaEventDestroy(p.a);
            cudaEventDestroy(p.b);
        }
        for (auto e : pool) cudaEventDestroy(e);
    }
    cudaEvent_t take_event() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        return e;
    }
    // brackets a launch with events when timing is enabled (resolved by resolve_timing)
    template <typename F>
    void timed(int which, F&& f) {
        timed_on(which, stream, f);
    }
    template <typename F>
    void timed_on(int which, cudaStream_t st, F&& f) {
        if (!timing) {
            f();
            return;
        }
        Pending p{which, take_event(), take_event()};
        CK(cudaEventRecord(p.a, st));
        f();
        CK(cudaEventRecord(p.b, st));
        pending.push_back(p);
    }
    void resolve_timing() {
        // intervals relative to the first pending start (offsets may be negative: the launches
        // of concurrent streams are recorded in host order, not device order)
        std::vector<std::pair<float, float>> iv[3];
        for (auto& p : pending) {
            CK(cudaEventSynchronize(p.b));
            float ms = 0, at = 0;
            CK(cudaEventElapsedTime(&ms, p.a, p.b));
            CK(cudaEventElapsedTime(&at, pending.front().a, p.a));
            t_ms[p.which] += ms;
            t_n[p.which] += 1;
            iv[p.which].push_back({at, at + ms});
        }
        for (int w = 0; w < 3; ++w) {
            std::sort(iv[w].begin(), iv[w].end());
            double busy = 0;
            float lo = 0, hi = 0;
            bool open = false;
            for (auto& x : iv[w]) {
                if (open && x.first <= hi) {
                    hi = std::max(hi, x.second);
                    continue;
                }
                if (open) busy += hi - lo;
                lo = x.first;
                hi = x.second;
                open = true;
            }
            if (open) busy += hi - lo;
            t_busy[w] += busy;
        }
        for (auto& p : pending) {
            pool.push_back(p.a);
            pool.push_back(p.b);
        }
        pending.clear();
    }
};

namespace {

// Evaluate n device rows into device outputs; returns the first gene error code or kNoError.
void eval_rows(ffsga_cuda_instance_t* I, const uint8_t* rows, long long n, double* obj, double* fit, double* mk,
               double* td, bool check, unsigned long long* err = nullptr) {
    if (n <= 0) return;
    I->ev_err.ensure(sizeof(unsigned long long));
    if (check && !err) CK(cudaMemsetAsync(I->ev_err.p, 0xFF, sizeof(unsigned long long), I->stream));
    EvalItems W{};
    W.n = n;
    W.base = rows;
    W.stride = (long long)I->block();
    W.deal = 1;
    W.obj = obj;
    W.fit = fit;
    W.mk = mk;
    W.td = td;
    W.err = err ? err : I->ev_err.as<unsigned long long>();
    I->timed(0, [&] { CK(launch_eval(I->d, I->ec, W, n, I->sm_count, false, I->stream)); });
    g_launches += 1;
}

unsigned long long read_error(ffsga_cuda_instance_t* I) {
    unsigned long long code = kNoError;
    CK(cudaMemcpyAsync(&code, I->ev_err.p, sizeof(code), cudaMemcpyDeviceToHost, I->stream));
    CK(cudaStreamSynchronize(I->stream));
    return code;
}

void ensure_eval_staging(ffsga_cuda_instance_t* I, long long chunk) {
    if (chunk <= I->ev_cap) return;
    const size_t L = (size_t)I->J * I->S;
    I->ev_in.alloc(chunk * L * sizeof(int32_t));
    I->ev_rows.alloc(chunk * I->block());
    I->ev_obj.alloc(chunk * sizeof(double));
    I->ev_fit.alloc(chunk * sizeof(double));
    I->ev_mk.alloc(chunk * sizeof(double));
    I->ev_td.alloc(chunk * sizeof(double));
    I->ev_cap = chunk;
}

// Host-to-pinned copy of one sub-batch, split over a few threads for large ones (a single
// memcpy thread moves ~10 GB/s, below PCIe).
void staged_copy(void* dst, const void* src, size_t bytes) {
    const size_t per = (size_t)8 << 20;
    const int nt = (int)std::min<size_t>(8, (bytes + per - 1) / per);
    if (nt <= 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    std::vector<std::thread> th;
    const size_t part = (bytes + nt - 1) / nt;
    for (int t = 0; t < nt; ++t) {
        const size_t o = (size_t)t * part;
        if (o >= bytes) break;
        th.emplace_back([=] { std::memcpy((char*)dst + o, (const char*)src + o, std::min(part, bytes - o)); });
    }
    for (auto& x : th) x.join();
}

// Is [p, p + bytes) in memory the copy engines can read in place (page-locked host memory, or
// device / managed memory)?  Both ends are checked; pageable memory reports "unregistered".
bool dma_readable(const void* p, size_t bytes) {
    for (const void* q : {p, (const void*)((const char*)p + bytes - 1)}) {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, q) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        if (a.type != cudaMemoryTypeHost && a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged)
            return false;
    }
    return true;
}

// Evaluator::score over a host batch, pipelined in sub-batches: the host copies sub-batch k+1
// into pinned staging while the copy stream moves sub-batch k to the device and the instance
// stream transposes and decodes the one before; results stay on the device until one copy back.
// A batch already in page-locked (or device) memory skips the staging copy: the copy engine
// reads it in place.
template <typename T>
void evaluate_host(ffsga_cuda_instance_t* I, const T* genes, int64_t n, double* obj, double* fit, double* mk,
                   double* td) {
    if (n < 0) fail(FFSGA_ERR_CONTRACT, "evaluate: negative batch size");
    if (n == 0) return;
    if (!genes || !obj || !fit) fail(FFSGA_ERR_ARG, "evaluate: null pointer");
    const long long L = (long long)I->J * I->S;
    // sub-batches of >= 8192 chromosomes keep every decoder round full; at most ~64 MB staged
    const long long sub = std::min<long long>(n, std::max<long long>(8192, (64ll << 20) / (L * (long long)sizeof(T))));
    const long long nsub = (n + sub - 1) / sub;
    const size_t in_bytes = (size_t)sub * L * sizeof(T);
    const bool direct = dma_readable(genes, (size_t)n * L * sizeof(T));
    ensure_eval_staging(I, sub);
    I->ev_in2.ensure(in_bytes);
    I->ev_res.ensure(sizeof(double) * 4 * (size_t)n);
    I->ev_errs.ensure(sizeof(unsigned long long) * (size_t)nsub);
    if (!I->cstream) {
        CK(cudaStreamCreateWithFlags(&I->cstream, cudaStreamNonBlocking));
        for (int k = 0; k < 2; ++k)
            for (cudaEvent_t* e : {&I->pin_free[k], &I->in_ready[k], &I->in_free[k]})
                CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    if (!direct && I->pin_bytes < in_bytes) {
        for (int k = 0; k < 2; ++k) {
            if (I->pin[k]) CK(cudaFreeHost(I->pin[k]));
            I->pin[k] = nullptr;
        }
        I->pin_bytes = 0;
        for (int k = 0; k < 2; ++k) CK(cudaHostAlloc(&I->pin[k], in_bytes, cudaHostAllocDefault));
        I->pin_bytes = in_bytes;
    }
    double* robj = I->ev_res.as<double>();
    double* rfit = robj + n;
    double* rmk = rfit + n;
    double* rtd = rmk + n;
    unsigned long long* errs = I->ev_errs.as<unsigned long long>();
    CK(cudaMemsetAsync(errs, 0xFF, sizeof(unsigned long long) * (size_t)nsub, I->stream));
    uint8_t* din[2] = {I->ev_in.as<uint8_t>(), I->ev_in2.as<uint8_t>()};
    for (long long k = 0; k < nsub; ++k) {
        const int b = (int)(k & 1);
        const long long first = k * sub, c = std::min<long long>(sub, n - first);
        const size_t bytes = (size_t)c * L * sizeof(T);
        if (!direct) {
            if (k >= 2) CK(cudaEventSynchronize(I->pin_free[b]));  // sub-batch k-2 has left staging
            staged_copy(I->pin[b], genes + first * L, bytes);
        }
        if (k >= 2) CK(cudaStreamWaitEvent(I->cstream, I->in_free[b], 0));  // ... and its device input
        CK(cudaMemcpyAsync(din[b], direct ? (const void*)(genes + first * L) : (const void*)I->pin[b], bytes,
                           cudaMemcpyDefault, I->cstream));
        CK(cudaEventRecord(I->pin_free[b], I->cstream));
        CK(cudaEventRecord(I->in_ready[b], I->cstream));
        CK(cudaStreamWaitEvent(I->stream, I->in_ready[b], 0));
        if (sizeof(T) == 4)
            CK(launch_rows_from_int(I->d, reinterpret_cast<const int32_t*>(din[b]), nullptr, I->ev_rows.as<uint8_t>(), c,
                                    I->stream));
        else
            CK(launch_rows_from_int(I->d, nullptr, din[b], I->ev_rows.as<uint8_t>(), c, I->stream));
        g_launches += 1;
        CK(cudaEventRecord(I->in_free[b], I->stream));
        eval_rows(I, I->ev_rows.as<uint8_t>(), c, robj + first, rfit + first, rmk + first, rtd + first, true,
                  errs + k);
    }
    std::vector<unsigned long long> codes((size_t)nsub);
    CK(cudaMemcpyAsync(codes.data(), errs, sizeof(unsigned long long) * (size_t)nsub, cudaMemcpyDeviceToHost, I->stream));
    CK(cudaMemcpyAsync(obj, robj, sizeof(double) * n, cudaMemcpyDeviceToHost, I->stream));
    CK(cudaMemcpyAsync(fit, rfit, sizeof(double) * n, cudaMemcpyDeviceToHost, I->stream));
    if (mk) CK(cudaMemcpyAsync(mk, rmk, sizeof(double) * n, cudaMemcpyDeviceToHost, I->stream));
    if (td) CK(cudaMemcpyAsync(td, rtd, sizeof(double) * n, cudaMemcpyDeviceToHost, I->stream));
    CK(cudaStreamSynchronize(I->stream));
    for (unsigned long long code : codes)  // the first chromosome in batch order with a bad gene
        if (code != kNoError) fail(FFSGA_ERR_CONTRACT, gene_error(code));
}

}  // namespace

extern "C" {

const char* ffsga_cuda_last_error(void) { return g_err.c_str(); }
int ffsga_cuda_abi_version(void) { return FFSGA_CUDA_ABI_VERSION; }

int ffsga_cuda_device_count(int* count) {
    return guard([&] {
        if (!count) fail(FFSGA_ERR_ARG, "null pointer");
        int n = 0;
        cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
        *count = n;
    });
}

int ffsga_cuda_instance_create(int device, int num_jobs, int num_stages, const int32_t* machines,
                               const double* proc, const double* release, const double* due, double weight,
                               double emax, ffsga_cuda_instance* out) {
    return guard([&] {
        const bool dbg = std::getenv("FFSGA_DEBUG_INIT") != nullptr;
        auto t_last = std::chrono::steady_clock::now();
        auto mark = [&](const char* what) {
            if (!dbg) return;
            const auto t = std::chrono::steady_clock::now();
            std::fprintf(stderr, "instance_create %-24s %.3f ms\n", what,
                         std::chrono::duration<double, std::milli>(t - t_last).count());
            t_last = t;
        };
        if (!out || !machines || !proc || !release || !due) fail(FFSGA_ERR_ARG, "instance_create: null pointer");
        *out = nullptr;
        if (num_jobs < 1) fail(FFSGA_ERR_CONTRACT, "instance: num_jobs must be >= 1");
        if (num_stages < 1) fail(FFSGA_ERR_CONTRACT, "instance: num_stages must be >= 1");
        if (num_jobs > 64000) fail(FFSGA_ERR_CONFIG, "device decoder supports at most 64000 jobs");
        if (num_stages > 65535) fail(FFSGA_ERR_CONFIG, "device decoder supports at most 65535 stages");
        int dev_count = 0;
        cudaError_t e = cudaGetDeviceCount(&dev_count);
        if (e != cudaSuccess || dev_count == 0) {
            cudaGetLastError();
            fail(FFSGA_ERR_CUDA, "no CUDA device available: the FFS hot path runs only on sm_100 GPUs");
        }
        if (device < 0 || device >= dev_count) fail(FFSGA_ERR_ARG, "instance_create: bad device ordinal");
        auto* I = new ffsga_cuda_instance_t();
        std::unique_ptr<ffsga_cuda_instance_t> hold(I);
        I->device = device;
        I->use();
        // two attributes, not cudaGetDeviceProperties (which queries everything: tens of ms)
        int cc_major = 0;
        CK(cudaDeviceGetAttribute(&cc_major, cudaDevAttrComputeCapabilityMajor, device));
        if (cc_major < 10) fail(FFSGA_ERR_CUDA, "device is not sm_100 class (built for sm_100a only)");
        CK(cudaDeviceGetAttribute(&I->sm_count, cudaDevAttrMultiProcessorCount, device));
        const int J = num_jobs, S = num_stages;
        I->J = J;
        I->S = S;
        I->Jpad = (J + 15) & ~15;
        I->M.assign(machines, machines + S);
        I->stage_off.assign(S + 1, 0);
        I->maxM = 0;
        for (int s = 0; s < S; ++s) {
            if (I->M[s] < 1) fail(FFSGA_ERR_CONTRACT, "instance: every stage needs at least one machine");
            if (I->M[s] > kMaxMachines)
                fail(FFSGA_ERR_CONFIG, "device decoder supports at most 32 machines per stage");
            I->stage_off[s + 1] = I->stage_off[s] + I->M[s];
            I->maxM = std::max(I->maxM, I->M[s]);
        }
        const int MT = I->stage_off[S];
        double horizon = 0.0, min_p = INFINITY;
        for (int j = 0; j < J; ++j) horizon = std::max(horizon, release[j]);
        for (int j = 0; j < J; ++j)
            for (int s = 0; s < S; ++s) {
                double worst = 0.0;
                for (int m = 0; m < I->M[s]; ++m) {
                    const double p = proc[(size_t)j * MT + I->stage_off[s] + m];
                    if (!(p > 0.0) || !std::isfinite(p))
                        fail(FFSGA_ERR_CONTRACT, "instance: processing times must be positive");
                    worst = std::max(worst, p);
                    min_p = std::min(min_p, p);
                }
                horizon += worst;
            }
        for (int j = 0; j < J; ++j)
            if (!std::isfinite(release[j]) || !std::isfinite(due[j]))
                fail(FFSGA_ERR_CONTRACT, "instance: release and due times must be finite");
        // completions on a machine must strictly increase for the merge-ordered decoder:
        // x + p > x for every completion x <= horizon iff p >= ulp(horizon)
        // (instances violating it run on the bucket-sort decoder, which needs no such bound)
        const double ulp = std::nextafter(horizon, INFINITY) - horizon;
        const bool merge_ok = min_p >= ulp;
        I->weight = weight;
        I->emax = emax;
        // stage-major proc columns with one zero pad per column
        std::vector<double> procT((size_t)MT * (J + 1), 0.0);
        for (int j = 0; j < J; ++j)
            for (int s = 0; s < S; ++s)
                for (int m = 0; m < I->M[s]; ++m)
                    procT[(size_t)(I->stage_off[s] + m) * (J + 1) + j] = proc[(size_t)j * MT + I->stage_off[s] + m];
        // stage-0 order: jobs by (release, index)  (model.cpp:98-105)
        std::vector<uint16_t> order(J);
        std::iota(order.begin(), order.end(), 0);
        std::sort(order.begin(), order.end(), [&](int a, int b) {
            return release[a] < release[b] || (release[a] == release[b] && a < b);
        });
        // bit layout (chromosome.cpp:10-26)
        I->bps.assign(S, 0);
        I->sbo.assign(S + 1, 0);
        for (int s = 0; s < S; ++s) {
            I->bps[s] = std::max(1, bit_width_u((unsigned)I->M[s] - 1u));
            I->sbo[s + 1] = I->sbo[s] + I->bps[s];
        }
        I->bpj = I->sbo[S];
        const long long tb = (long long)J * I->bpj;
        if (tb > 0x7FFFFFFF) fail(FFSGA_ERR_CONFIG, "bit layout too large");
        I->total_bits = (int)tb;
        I->words = std::max(1, (I->total_bits + 63) / 64);
        std::vector<uint16_t> bit_stage(I->bpj);
        for (int s = 0; s < S; ++s)
            for (int r = I->sbo[s]; r < I->sbo[s + 1]; ++r) bit_stage[r] = (uint16_t)s;
        mark("validate+layout");
        upload(I->dM, I->M);
        upload(I->dStageOff, I->stage_off);
        upload(I->dBps, I->bps);
        upload(I->dSbo, I->sbo);
        upload(I->dProcT, procT);
        upload(I->dRelease, std::vector<double>(release, release + J));
        upload(I->dDue, std::vector<double>(due, due + J));
        upload(I->dRelOrder, order);
        upload(I->dBitStage, bit_stage);
        mark("uploads");
        DevInst& d = I->d;
        d.J = J;
        d.S = S;
        d.Jpad = I->Jpad;
        d.maxM = I->maxM;
        d.bits_per_job = I->bpj;
        d.total_bits = I->total_bits;
        d.words = I->words;
        d.weight = weight;
        d.emax = emax;
        d.M = I->dM.as<int>();
        d.stage_off = I->dStageOff.as<int>();
        d.bps = I->dBps.as<int>();
        d.sbo = I->dSbo.as<int>();
        d.procT = I->dProcT.as<double>();
        d.release = I->dRelease.as<double>();
        d.due = I->dDue.as<double>();
        d.rel_order = I->dRelOrder.as<uint16_t>();
        // CTA-wide stage barriers keep one stage slice of procT hot in L1 for the whole CTA; they
        // pay off when the table does not fit L1 anyway (measured: 500x20 +14 %, 100x10 -11 %)
        d.cta_sync = (size_t)MT * (J + 1) * sizeof(double) > (size_t)128 * 1024 ? 1 : 0;
        d.max_warps = 0;
        if (const char* v = std::getenv("FFSGA_EVAL_SYNC")) d.cta_sync = std::string(v) == "cta" ? 1 : (std::string(v) == "warp" ? 0 : d.cta_sync);
        if (const char* v = std::getenv("FFSGA_EVAL_WARPS")) d.max_warps = std::atoi(v);
        d.algo = merge_ok ? 0 : 1;
        d.bshift = 0;
        if (const char* v = std::getenv("FFSGA_EVAL_ALGO")) {
            if (std::string(v) == "bucket") d.algo = 1;
            if (std::string(v) == "merge") {
                if (!merge_ok) fail(FFSGA_ERR_CONFIG, "merge decoder needs processing times >= ulp(schedule horizon)");
                d.algo = 0;
            }
        }
        if (const char* v = std::getenv("FFSGA_EVAL_BSHIFT")) d.bshift = std::atoi(v);
        d.check_selftest = std::getenv("FFSGA_CHECK_SELFTEST") ? 1 : 0;
        // Packed heads for K1's ready-only pass: a ready time's low bit_width(J) mantissa bits
        // carry the job id, so one fp64 compare orders (ready, job) up to that truncation and the
        // heads move one 64-bit word instead of a value and a job.  Needs sign-clear ready times
        // (release -0.0 would order as a negative number) and a horizon far below the sentinel.
        {
            bool pk = J <= 65534 && horizon < 1e300;
            for (int j = 0; j < J && pk; ++j) pk = !std::signbit(release[j]) && release[j] < 1e300;
            d.pk_bits = pk ? bit_width_u((unsigned)J) : 0;
            if (const char* v = std::getenv("FFSGA_EVAL_PK")) if (std::string(v) == "0") d.pk_bits = 0;
        }
        if (const char* v = std::getenv("FFSGA_STEP_SPLIT")) I->step_split = std::max(1, std::atoi(v));
        if (const char* v = std::getenv("FFSGA_STEP_MIX")) I->step_mix = std::max(0, std::atoi(v));
        mark("devinst");
        int rc = eval_config(d, I->sm_count, d.max_warps, &I->ec);
        if (rc == -1) fail(FFSGA_ERR_CONFIG, "instance too large for the on-chip decoder state (num_jobs)");
        if (rc != 0) fail(FFSGA_ERR_CUDA, std::string("decoder configuration failed: ") + cudaGetErrorString(cudaGetLastError()));
        // The joint GA step runs the cellular and the pseudo decoder launches side by side on two
        // streams.  With the two-pop pipeline a shared-memory-bound standalone CTA (one per SM,
        // L1 left for the procT slice) is also the best step CTA: C3 152.5 generations/s vs 148.7
        // with half-size CTAs that let both launches share an SM (which won before the
        // pipeline: 136.8 vs 127.9).  Small instances, whose standalone CTA is the 16-warp cap,
        // still do better with half-size CTAs (C2: 11.3 k vs 8.7 k generations/s).
        int step_warps = I->ec.warps > 8 ? I->ec.warps / 2 : I->ec.warps;
        if (const char* v = std::getenv("FFSGA_STEP_WARPS")) step_warps = std::max(1, std::atoi(v));
        rc = eval_config(d, I->sm_count, step_warps, &I->ec_step);
        if (rc != 0) fail(FFSGA_ERR_CUDA, std::string("decoder configuration failed: ") + cudaGetErrorString(cudaGetLastError()));
        mark("eval_config");
        CK(cudaStreamCreateWithFlags(&I->stream, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&I->fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&I->join, cudaEventDisableTiming));
        CK(cudaEventCreate(&I->ev0));
        CK(cudaEventCreate(&I->ev1));
        CK(cudaEventCreate(&I->st0));
        CK(cudaEventCreate(&I->st1));
        I->wl_count.alloc(2 * sizeof(long long));  // one item counter per joint-step group (grown on demand)
        I->eval_total.alloc(sizeof(unsigned long long));
        CK(cudaMemsetAsync(I->eval_total.p, 0, sizeof(unsigned long long), I->stream));
        mark("streams+events+bufs");
        *out = hold.release();
    });
}

int ffsga_cuda_instance_destroy(ffsga_cuda_instance inst) {
    return guard([&] { delete inst; });
}

int ffsga_cuda_instance_info(ffsga_cuda_instance inst, int* row_stride, int* group_lanes, int* total_bits,
                             int* smem_per_group) {
    return guard([&] {
        if (!inst) fail(FFSGA_ERR_ARG, "null instance");
        if (row_stride) *row_stride = inst->Jpad;
        if (group_lanes) *group_lanes = inst->ec.G;
        if (total_bits) *total_bits = inst->total_bits;
        if (smem_per_group) *smem_per_group = inst->ec.gl.bytes;
    });
}

int ffsga_cuda_evaluate(ffsga_cuda_instance inst, const int32_t* genes, int64_t n, double* obj, double* fit,
                        double* mk, double* td) {
    return guard([&] {
        NvtxRange nvtx_range("ffsga_cuda_evaluate");
        if (!inst) fail(FFSGA_ERR_ARG, "null instance");
        std::lock_guard<std::mutex> lk(inst->mu);
        inst->use();
        evaluate_host(inst, genes, n, obj, fit, mk, td);
    });
}

int ffsga_cuda_evaluate_device(ffsga_cuda_instance inst, const uint8_t* genes, int64_t n, double* obj, double* fit,
                               double* mk, double* td, void* stream) {
    return guard([&] {
        NvtxRange nvtx_range("ffsga_cuda_evaluate_device");
        if (!inst) fail(FFSGA_ERR_ARG, "null instance");
        if (n < 0) fail(FFSGA_ERR_CONTRACT, "evaluate: negative batch size");
        if (n == 0) return;
        if (!genes || !obj || !fit) fail(FFSGA_ERR_ARG, "evaluate: null pointer");
        std::lock_guard<std::mutex> lk(inst->mu);
        inst->use();
        ffsga_cuda_instance_t* I = inst;
        cudaStream_t user = static_cast<cudaStream_t>(stream);
        // order: caller's queued work -> our stream -> back to the caller's stream
        CK(cudaEventRecord(I->fork, user));
        CK(cudaStreamWaitEvent(I->stream, I->fork, 0));
        const long long L = (long long)I->J * I->S;
        const long long chunk = std::min<long long>(n, 1 << 16);
        ensure_eval_staging(I, chunk);
        for (long long first = 0; first < n; first += chunk) {
            const long long c = std::min<long long>(chunk, n - first);
            CK(launch_rows_from_int(I->d, nullptr, genes + first * L, I->ev_rows.as<uint8_t>(), c, I->stream));
            g_launches += 1;
            eval_rows(I, I->ev_rows.as<uint8_t>(), c, obj + first, fit + first, mk ? mk + first : nullptr,
                      td ? td + first : nullptr, true);
            const unsigned long long code = read_error(I);
            if (code != kNoError)
                fail(FFSGA_ERR_CONTRACT, gene_error(code) + " (chromosome " + std::to_string((code >> 32) + first) + ")");
        }
        CK(cudaEventRecord(I->join, I->stream));
        CK(cudaStreamWaitEvent(user, I->join, 0));
    });
}

int ffsga_cuda_evaluate_u8(ffsga_cuda_instance inst, const uint8_t* genes, int64_t n, double* obj, double* fit,
                           double* mk, double* td) {
    return guard([&] {
        NvtxRange nvtx_range("ffsga_cuda_evaluate_u8");
        if (!inst) fail(FFSGA_ERR_ARG, "null instance");
        std::lock_guard<std::mutex> lk(inst->mu);
        inst->use();
        evaluate_host(inst, genes, n, obj, fit, mk, td);
    });
}

int ffsga_cuda_decode(ffsga_cuda_instance inst, const int32_t* genes, int32_t* machine, double* start,
                      double* completion, double* report5) {
    return guard([&] {
        NvtxRange nvtx_range("ffsga_cuda_decode");
        if (!inst || !genes || !machine || !start || !completion) fail(FFSGA_ERR_ARG, "decode: null pointer");
        std::lock_guard<std::mutex> lk(inst->mu);
        inst->use();
        ffsga_cuda_instance_t* I = inst;
        const size_t L = (size_t)I->J * I->S;
        ensure_eval_staging(I, 1);
        // the schedule lives in the instance (grown once): no allocation or device-wide
        // synchronisation per call
        I->sched.ensure(L * (sizeof(int32_t) + 2 * sizeof(double)) + 16);
        int32_t* smach = reinterpret_cast<int32_t*>(I->sched.p);
        double* sstart = reinterpret_cast<double*>(I->sched.as<char>() + ((L * sizeof(int32_t) + 15) & ~size_t(15)));
        double* scomp = sstart + L;
        CK(cudaMemcpyAsync(I->ev_in.p, genes, L * sizeof(int32_t), cudaMemcpyHostToDevice, I->stream));
        CK(launch_rows_from_int(I->d, I->ev_in.as<int32_t>(), nullptr, I->ev_rows.as<uint8_t>(), 1, I->stream));
        I->ev_err.ensure(sizeof(unsigned long long));
        CK(cudaMemsetAsync(I->ev_err.p, 0xFF, sizeof(unsigned long long), I->stream));
        EvalItems W{};
        W.n = 1;
        W.base = I->ev_rows.as<uint8_t>();
        W.stride = (long long)I->block();
        W.obj = I->ev_obj.as<double>();
        W.fit = I->ev_fit.as<double>();
        W.mk = I->ev_mk.as<double>();
        W.td = I->ev_td.as<double>();
        W.err = I->ev_err.as<unsigned long long>();
        W.smachine = smach;
        W.sstart = sstart;
        W.scomp = scomp;
        CK(launch_eval(I->d, I->ec, W, 1, I->sm_count, true, I->stream));
        g_launches += 2;
        const unsigned long long code = read_error(I);
        if (code != kNoError) fail(FFSGA_ERR_CONTRACT, gene_error(code));
        CK(cudaMemcpyAsync(machine, smach, L * sizeof(int32_t), cudaMemcpyDeviceToHost, I->stream));
        CK(cudaMemcpyAsync(start, sstart, L * sizeof(double), cudaMemcpyDeviceToHost, I->stream));
        CK(cudaMemcpyAsync(completion, scomp, L * sizeof(double), cudaMemcpyDeviceToHost, I->stream));
        CK(cudaStreamSynchronize(I->stream));
        if (report5) {
            double r[4];
            CK(cudaMemcpyAsync(&r[0], I->ev_mk.p, sizeof(double), cudaMemcpyDeviceToHost, I->stream));
            CK(cudaMemcpyAsync(&r[1], I->ev_td.p, sizeof(double), cudaMemcpyDeviceToHost, I->stream));
            CK(cudaMemcpyAsync(&r[2], I->ev_obj.p, sizeof(double), cudaMemcpyDeviceToHost, I->stream));
            CK(cudaMemcpyAsync(&r[3], I->ev_fit.p, sizeof(double), cudaMemcpyDeviceToHost, I->stream));
            CK(cudaStreamSynchronize(I->stream));
            report5[0] = r[0];
            report5[1] = r[1];
            report5[2] = r[2];
            report5[3] = r[3];
            report5[4] = I->emax;
        }
    });
}

}  // extern "C"

// ------------------------------------------------------------------------------ batches
struct ffsga_cuda_batch_t {
    ffsga_cuda_instance_t* inst = nullptr;
    long long cap = 0;
    DevBuf rows, obj, fit, mk, td, err, stage;
    void adopt(cudaStream_t s) {
        for (DevBuf* b : {&rows, &obj, &fit, &mk, &td, &err, &stage}) b->owner = s;
    }
    long long stage_cap = 0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    ~ffsga_cuda_batch_t() {
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
    }
};

namespace {
template <typename T>
void batch_upload(ffsga_cuda_batch b, const T* genes, int64_t n) {
    if (!b || !genes) fail(FFSGA_ERR_ARG, "batch_upload: null pointer");
    if (n < 0 || n > b->cap) fail(FFSGA_ERR_CONTRACT, "batch_upload: n exceeds capacity");
    auto* I = b->inst;
    std::lock_guard<std::mutex> lk(I->mu);  // the instance stream may be capturing a step graph
    I->use();
    const long long L = (long long)I->J * I->S;
    const long long chunk = std::min<long long>(std::max<long long>(n, 1), 1 << 14);
    if (chunk * L * (long long)sizeof(T) > (long long)b->stage.bytes) b->stage.alloc(chunk * L * sizeof(T));
    for (long long f = 0; f < n; f += chunk) {
        const long long c = std::min<long long>(chunk, n - f);
        CK(cudaMemcpyAsync(b->stage.p, genes + f * L, sizeof(T) * c * L, cudaMemcpyHostToDevice, I->stream));
        uint8_t* dst = b->rows.as<uint8_t>() + (size_t)f * I->block();
        if (sizeof(T) == 4)
            CK(launch_rows_from_int(I->d, b->stage.as<int32_t>(), nullptr, dst, c, I->stream));
        else
            CK(launch_rows_from_int(I->d, nullptr, b->stage.as<uint8_t>(), dst, c, I->stream));
        g_launches += 1;
    }
}

}  // namespace

extern "C" {

int ffsga_cuda_batch_create(ffsga_cuda_instance inst, int64_t capacity, ffsga_cuda_batch* out) {
    return guard([&] {
        if (!inst || !out) fail(FFSGA_ERR_ARG, "batch_create: null pointer");
        if (capacity < 1) fail(FFSGA_ERR_CONTRACT, "batch capacity must be >= 1");
        std::lock_guard<std::mutex> lk(inst->mu);
        inst->use();
        auto* b = new ffsga_cuda_batch_t();
        std::unique_ptr<ffsga_cuda_batch_t> hold(b);
        b->inst = inst;
        b->adopt(inst->stream);
        b->cap = capacity;
        b->rows.alloc((size_t)capacity * inst->block());
        b->obj.alloc(sizeof(double) * capacity);
        b->fit.alloc(sizeof(double) * capacity);
        b->mk.alloc(sizeof(double) * capacity);
        b->td.alloc(sizeof(double) * capacity);
        b->err.alloc(sizeof(unsigned long long));
        CK(cudaMemsetAsync(b->err.p, 0xFF, sizeof(unsigned long long), inst->stream));
        CK(cudaEventCreate(&b->e0));
        CK(cudaEventCreate(&b->e1));
        *out = hold.release();
    });
}

int ffsga_cuda_batch_destroy(ffsga_cuda_batch b) {
    return guard([&] { delete b; });
}

int ffsga_cuda_batch_fill_random(ffsga_cuda_batch b, uint64_t base_seed, int64_t first, int64_t n) {
    return guard([&] {
        NvtxRange nvtx_range("ffsga_cuda_batch_fill_random");
        if (!b) fail(FFSGA_ERR_ARG, "null batch");
        if (n < 0 || n > b->cap) fail(FFSGA_ERR_CONTRACT, "batch_fill_random: n exceeds capacity");
        auto* I = b->inst;
        std::lock_guard<std::mutex> lk(I->mu);
        I->use();
        CK(launch_random_rows(I->d, b->rows.as<uint8_t>(), (long long)I->block(), n, base_seed, first, true, I->stream));
        g_launches += 1;
    });
}

int ffsga_cuda_batch_upload(ffsga_cuda_batch b, const int32_t* genes, int64_t n) {
    return guard([&] { batch_upload(b, genes, n); });
}

int ffsga_cuda_batch_upload_u8(ffsga_cuda_batch b, const uint8_t* genes, int64_t n) {
    return guard([&] { batch_upload(b, genes, n); });
}

int ffsga_cuda_batch_evaluate(ffsga_cuda_batch b, int64_t n) {
    return guard([&] {
        NvtxRange nvtx_range("ffsga_cuda_batch_evaluate");
        if (!b) fail(FFSGA_ERR_ARG, "null batch");
        if (n < 0 || n > b->cap) fail(FFSGA_ERR_CONTRACT, "batch_evaluate: n exceeds capacity");
        auto* I = b->inst;
        std::lock_guard<std::mutex> lk(I->mu);
        I->use();
        EvalItems W{};
        W.n = n;
        W.base = b->rows.as<uint8_t>();
        W.stride = (long long)I->block();
        W.deal = 1;
        W.obj = b->obj.as<double>();
        W.fit = b->fit.as<double>();
        W.mk = b->mk.as<double>();
        W.td = b->td.as<double>();
        W.err = b->err.as<unsigned long long>();
        CK(cudaEventRecord(b->e0, I->stream));
        CK(launch_eval(I->d, I->ec, W, n, I->sm_count, false, I->stream));
        CK(cudaEventRecord(b->e1, I->stream));
        g_launches += 1;
    });
}

int ffsga_cuda_batch_last_eval_ms(ffsga_cuda_batch b, float* ms) {
    return guard([&] {
        if (!b || !ms) fail(FFSGA_ERR_ARG, "null pointer");
        b->inst->use();
        CK(cudaEventSynchronize(b->e1));
        CK(cudaEventElapsedTime(ms, b->e0, b->e1));
    });
}

int ffsga_cuda_batch_results(ffsga_cuda_batch b, int64_t n, double* obj, double* fit, double* mk, double* td) {
    return guard([&] {
        if (!b) fail(FFSGA_ERR_ARG, "null batch");
        if (n < 0 || n > b->cap) fail(FFSGA_ERR_CONTRACT, "batch_results: n exceeds capacity");
        auto* I = b->inst;
        std::lock_guard<std::mutex> lk(I->mu);
        I->use();
        const size_t bytes = sizeof(double) * n;
        if (obj) CK(cudaMemcpyAsync(obj, b->obj.p, bytes, cudaMemcpyDeviceToHost, I->stream));
        if (fit) CK(cudaMemcpyAsync(fit, b->fit.p, bytes, cudaMemcpyDeviceToHost, I->stream));
        if (mk) CK(cudaMemcpyAsync(mk, b->mk.p, bytes, cudaMemcpyDeviceToHost, I->stream));
        if (td) CK(cudaMemcpyAsync(td, b->td.p, bytes, cudaMemcpyDeviceToHost, I->stream));
        unsigned long long code = kNoError;
        CK(cudaMemcpyAsync(&code, b->err.p, sizeof(code), cudaMemcpyDeviceToHost, I->stream));
        CK(cudaStreamSynchronize(I->stream));
        if (code != kNoError) {
            CK(cudaMemsetAsync(b->err.p, 0xFF, sizeof(unsigned long long), I->stream));
            fail(FFSGA_ERR_CONTRACT, gene_error(code) + " (chromosome " + std::to_string(code >> 32) + ")");
        }
    });
}

int ffsga_cuda_batch_device_results(ffsga_cuda_batch b, const double** obj, const double** fit) {
    return guard([&] {
        if (!b) fail(FFSGA_ERR_ARG, "null batch");
        if (obj) *obj = b->obj.as<double>();
        if (fit) *fit = b->fit.as<double>();
    });
}

int ffsga_cuda_batch_download(ffsga_cuda_batch b, int64_t first, int64_t n, int32_t* genes) {
    return guard([&] {
        if (!b || !genes) fail(FFSGA_ERR_ARG, "null pointer");
        if (first < 0 || n < 0 || first + n > b->cap) fail(FFSGA_ERR_CONTRACT, "batch_download: range");
        auto* I = b->inst;
        std::lock_guard<std::mutex> lk(I->mu);
        I->use();
        const size_t L = (size_t)I->J * I->S;
        DevBuf out;
        out.alloc(std::max<size_t>(1, n * L * sizeof(int32_t)));
        CK(launch_rows_to_int(I->d, b->rows.as<uint8_t>() + first * I->block(), (long long)I->block(), nullptr,
                              out.as<int32_t>(), n, I->stream));
        g_launches += 1;
        CK(cudaMemcpyAsync(genes, out.p, n * L * sizeof(int32_t), cudaMemcpyDeviceToHost, I->stream));
        CK(cudaStreamSynchronize(I->stream));
    });
}

int ffsga_cuda_batch_sync(ffsga_cuda_batch b) {
    return guard([&] {
        if (!b) fail(FFSGA_ERR_ARG, "null batch");
        std::lock_guard<std::mutex> lk(b->inst->mu);
        b->inst->use();
        CK(cudaStreamSynchronize(b->inst->stream));
    });
}

}  // extern "C"

// ------------------------------------------------------------------------------ islands
struct ffsga_cuda_cellular_t {
    ffsga_cuda_instance_t* inst = nullptr;
    int n = 0, W = 0, H = 0, radius = 1, npc = 0;
    unsigned long long gen = 0;
    std::vector<int> slots_host;
    DevBuf genes, sel, fit, obj, slots, st, trace, desc;
    long long trace_cap = 0;
    CellIsland d{};
    void adopt(cudaStream_t s) {
        for (DevBuf* b : {&genes, &sel, &fit, &obj, &slots, &st, &trace, &desc}) b->owner = s;
    }
    int parity() const { return (int)(gen & 1ull); }
    void push_desc() {
        d.trace = trace.as<double>();
        desc.ensure(sizeof(CellIsland));
        // stream-ordered after any kernel that still reads the old descriptor (pageable: staged)
        CK(cudaMemcpyAsync(desc.p, &d, sizeof(CellIsland), cudaMemcpyHostToDevice, inst->stream));
    }
};

struct ffsga_cuda_pseudo_t {
    ffsga_cuda_instance_t* inst = nullptr;
    int n = 0;
    unsigned long long gen = 0;
    DevBuf words, fit, obj, mslot, rows, archive, st, trace, desc;
    long long trace_cap = 0;
    PseudoIsland d{};
    void adopt(cudaStream_t s) {
        for (DevBuf* b : {&words, &fit, &obj, &mslot, &rows, &archive, &st, &trace, &desc}) b->owner = s;
    }
    void push_desc() {
        d.trace = trace.as<double>();
        desc.ensure(sizeof(PseudoIsland));
        CK(cudaMemcpyAsync(desc.p, &d, sizeof(PseudoIsland), cudaMemcpyHostToDevice, inst->stream));
    }
};

namespace {

void neighborhood_slots(int x, int y, int w, int h, int r, std::vector<int>& out) {
    // cellular.cpp:12-27: dy ascending, dx ascending, centre skipped, toroidal wrap
    for (int dy = -r; dy <= r; ++dy) {
        const int budget = r - std::abs(dy);
        for (int dx = -budget; dx <= budget; ++dx) {
            if (dx == 0 && dy == 0) continue;
            const int nx = ((x + dx) % w + w) % w;
            const int ny = ((y + dy) % h + h) % h;
            out.push_back(ny * w + nx);
        }
    }
}

IslandState read_state(ffsga_cuda_instance_t* I, const DevBuf& st) {
    IslandState s;
    CK(cudaMemcpyAsync(&s, st.p, sizeof(s), cudaMemcpyDeviceToHost, I->stream));
    CK(cudaStreamSynchronize(I->stream));
    return s;
}

void refresh_stats(ffsga_cuda_cellular_t* c, ffsga_cuda_pseudo_t* p, int mode) {
    ffsga_cuda_instance_t* I = c ? c->inst : p->inst;
    CK(launch_island_stats(I->d, c ? c->desc.as<CellIsland>() : nullptr, c ? 1 : 0,
                           p ? p->desc.as<PseudoIsland>() : nullptr, p ? 1 : 0, mode, I->stream));
    g_launches += 1;
}

// storage row block of each cell in the live generation
std::vector<long long> cell_storage_index(ffsga_cuda_cellular_t* c) {
    std::vector<uint8_t> sel(c->n);
    CK(cudaMemcpyAsync(sel.data(), c->sel.as<uint8_t>() + (size_t)c->parity() * c->n, c->n, cudaMemcpyDeviceToHost,
                       c->inst->stream));
    CK(cudaStreamSynchronize(c->inst->stream));
    std::vector<long long> idx(c->n);
    for (int i = 0; i < c->n; ++i) idx[i] = (long long)sel[i] * c->n + i;
    return idx;
}

void pack_host_bits(const uint8_t* bits, int nbits, int words, std::vector<unsigned long long>& out) {
    out.assign(words, 0ull);
    for (int i = 0; i < nbits; ++i)
        if (bits[i] & 1u) out[i >> 6] |= 1ull << (i & 63);
}

void unpack_host_bits(const unsigned long long* w, int nbits, uint8_t* bits) {
    for (int i = 0; i < nbits; ++i) bits[i] = (uint8_t)((w[i >> 6] >> (i & 63)) & 1ull);
}

}  // namespace

extern "C" {

int ffsga_cuda_cellular_create(ffsga_cuda_instance inst, int width, int height, int radius, double xr, double mr,
                               uint64_t seed, const int32_t* init_genes, ffsga_cuda_cellular* out) {
    return guard([&] {
        NvtxRange nvtx_range("ffsga_cuda_cellular_create");
        if (!inst || !out) fail(FFSGA_ERR_ARG, "cellular_create: null pointer");
        *out = nullptr;
        if (width < 1 || height < 1) fail(FFSGA_ERR_CONFIG, "cellular grid shape does not match cell count");
        if (radius < 1) fail(FFSGA_ERR_CONTRACT, "neighborhood: radius must be >= 1");
        if (!(xr >= 0.0 && xr <= 1.0)) fail(FFSGA_ERR_CONFIG, "cellular crossover rate must lie in [0, 1]");
        if (!(mr >= 0.0 && mr <= 1.0)) fail(FFSGA_ERR_CONFIG, "cellular mutation rate must lie in [0, 1]");
        if ((long long)width * height > 0x3FFFFFFF) fail(FFSGA_ERR_CONFIG, "cellular island too large");
        std::lock_guard<std::mutex> lk(inst->mu);
        inst->use();
        ffsga_cuda_instance_t* I = inst;
        auto* c = new ffsga_cuda_cellular_t();
        std::unique_ptr<ffsga_cuda_cellular_t> hold(c);
        c->inst = I;
        c->adopt(I->stream);
        c->W = width;
        c->H = height;
        c->n = width * height;
        c->radius = radius;
        for (int i = 0; i < c->n; ++i) neighborhood_slots(i % width, i / width, width, height, radius, c->slots_host);
        c->npc = (int)(c->slots_host.size() / c->n);
        upload(c->slots, c->slots_host);
        const size_t block = I->block();
        c->genes.alloc(2 * (size_t)c->n * block);  // slot 1 is written by the first breed, pads included
        c->sel.alloc(2 * (size_t)c->n);
        CK(cudaMemsetAsync(c->sel.p, 0, 2 * (size_t)c->n, I->stream));
        c->fit.alloc(2 * sizeof(double) * c->n);
        c->obj.alloc(2 * sizeof(double) * c->n);
        c->st.alloc(sizeof(IslandState));
        IslandState s0{};
        s0.arch_fit = -1.0;
        CK(cudaMemcpyAsync(c->st.p, &s0, sizeof(s0), cudaMemcpyHostToDevice, I->stream));  // pageable: staged
        c->trace_cap = 1;
        c->trace.alloc(sizeof(double));
        if (init_genes) {
            // explicit population (cellular.cpp:90-102), scored on the device
            const long long L = (long long)I->J * I->S;
            DevBuf tmp;
            tmp.alloc(sizeof(int32_t) * L * c->n);
            CK(cudaMemcpy(tmp.p, init_genes, sizeof(int32_t) * L * c->n, cudaMemcpyHostToDevice));
            CK(launch_rows_from_int(I->d, tmp.as<int32_t>(), nullptr, c->genes.as<uint8_t>(), c->n, I->stream));
            g_launches += 1;
        } else {
            // one sequential Rng(island_seed) stream: cell i, gene g = draw i*L + g (cellular.cpp:84-86)
            CK(launch_random_rows(I->d, c->genes.as<uint8_t>(), (long long)block, c->n, seed, 0, false, I->stream));
            g_launches += 1;
        }
        // device-generated genes are in range by construction: only explicit populations are
        // checked (and only then does creation wait for the device)
        eval_rows(I, c->genes.as<uint8_t>(), c->n, c->obj.as<double>(), c->fit.as<double>(), nullptr, nullptr,
                  init_genes != nullptr);
        if (init_genes) {
            const unsigned long long code = read_error(I);
            if (code != kNoError) fail(FFSGA_ERR_CONTRACT, gene_error(code));
        }
        CellIsland& d = c->d;
        d.n = c->n;
        d.width = width;
        d.height = height;
        d.npc = c->npc;
        d.slots = c->slots.as<int>();
        d.genes = c->genes.as<uint8_t>();
        d.sel = c->sel.as<uint8_t>();
        d.fit = c->fit.as<double>();
        d.obj = c->obj.as<double>();
        d.seed = seed;
        d.thr_xr = coin_threshold(xr);
        d.thr_mu = coin_threshold(mr);
        d.st = c->st.as<IslandState>();
        d.item0 = 0;
        d.cell0 = 0;
        c->push_desc();
        refresh_stats(c, nullptr, 0);
        *out = hold.release();  // stream-ordered: every later call on the instance sees the initial state
    });
}

int ffsga_cuda_cellular_destroy(ffsga_cuda_cellular c) {
    return guard([&] {
        if (c) c->inst->use();
        delete c;
    });
}

int ffsga_cuda_cellular_size(ffsga_cuda_cellular c, int* size, int* width, int* height, int* neighbors) {
    return guard([&] {
        if (!c) fail(FFSGA_ERR_ARG, "null island");
        if (size) *size = c->n;
        if (width) *width = c->W;
        if (height) *height = c->H;
        if (neighbors) *neighbors = c->npc;
    });
}

int ffsga_cuda_cellular_generation(ffsga_cuda_cellular c, uint64_t* g) {
    return guard([&] {
        if (!c || !g) fail(FFSGA_ERR_ARG, "null pointer");
        *g = c->gen;
    });
}

int ffsga_cuda_cellular_read(ffsga_cuda_cellular c, double* fit, double* obj) {
    return guard([&] {
        if (!c) fail(FFSGA_ERR_ARG, "null island");
        std::lock_guard<std::mutex> lk(c->inst->mu);
        c->inst->use();
        const size_t off = (size_t)c->parity() * c->n;
        if (fit) CK(cudaMemcpyAsync(fit, c->fit.as<double>() + off, sizeof(double) * c->n, cudaMemcpyDeviceToHost, c->inst->stream));
        if (obj) CK(cudaMemcpyAsync(obj, c->obj.as<double>() + off, sizeof(double) * c->n, cudaMemcpyDeviceToHost, c->inst->stream));
        CK(cudaStreamSynchronize(c->inst->stream));
    });
}

int ffsga_cuda_cellular_genes(ffsga_cuda_cellular c, int index, int32_t* genes) {
    return guard([&] {
        if (!c || !genes) fail(FFSGA_ERR_ARG, "null pointer");
        if (index >= c->n) fail(FFSGA_ERR_CONTRACT, "cell index out of range");
        std::lock_guard<std::mutex> lk(c->inst->mu);
        ffsga_cuda_instance_t* I = c->inst;
        I->use();
        std::vector<long long> idx = cell_storage_index(c);
        if (index >= 0) idx = {idx[index]};
        DevBuf didx, out;
        upload(didx, idx);
        const size_t L = (size_t)I->J * I->S;
        out.alloc(sizeof(int32_t) * L * idx.size());
        CK(launch_rows_to_int(I->d, c->genes.as<uint8_t>(), (long long)I->block(), didx.as<long long>(), out.as<int32_t>(),
                              (long long)idx.size(), I->stream));
        g_launches += 1;
        CK(cudaMemcpyAsync(genes, out.p, sizeof(int32_t) * L * idx.size(), cudaMemcpyDeviceToHost, I->stream));
        CK(cudaStreamSynchronize(I->stream));
    });
}

int ffsga_cuda_cellular_slots(ffsga_cuda_cellular c, int index, int32_t* slots) {
    return guard([&] {
        if (!c || !slots) fail(FFSGA_ERR_ARG, "null pointer");
        if (index < 0 || index >= c->n) fail(FFSGA_ERR_CONTRACT, "cell index out of range");
        for (int k = 0; k < c->npc; ++k) slots[k] = c->slots_host[(size_t)index * c->npc + k];
    });
}

int ffsga_cuda_cellular_best(ffsga_cuda_cellular c, int* index, double* fit, double* obj) {
    return guard([&] {
        if (!c) fail(FFSGA_ERR_ARG, "null island");
        std::lock_guard<std::mutex> lk(c->inst->mu);
        c->inst->use();
        IslandState s = read_state(c->inst, c->st);
        if (index) *index = s.best_idx;
        if (fit) *fit = s.best_fit;
        if (obj) *obj = s.best_obj;
    });
}

int ffsga_cuda_cellular_candidate(ffsga_cuda_cellular c, int index, uint64_t stream_state, int32_t* genes,
                                  double* fit, double* obj, int* replaced, uint64_t* draws_used) {
    return guard([&] {
        if (!c || !genes || !fit || !obj || !replaced) fail(FFSGA_ERR_ARG, "cellular_candidate: null pointer");
        if (index < 0 || index >= c->n) fail(FFSGA_ERR_CONTRACT, "cell index out of range");
        std::lock_guard<std::mutex> lk(c->inst->mu);
        ffsga_cuda_instance_t* I = c->inst;
        I->use();
        const int q = c->parity();
        ensure_eval_staging(I, 1);
        DevBuf draws;
        draws.alloc(sizeof(unsigned long long));
        CK(launch_cell_candidate(I->d, c->d, index, stream_state, q, I->ev_rows.as<uint8_t>(), draws.as<unsigned long long>(),
                                 I->stream));
        g_launches += 1;
        eval_rows(I, I->ev_rows.as<uint8_t>(), 1, I->ev_obj.as<double>(), I->ev_fit.as<double>(), nullptr, nullptr, true);
        const unsigned long long code = read_error(I);
        if (code != kNoError) fail(FFSGA_ERR_CONTRACT, gene_error(code));
        double cf = 0, co = 0, f0 = 0, o0 = 0;
        unsigned long long used = 0;
        CK(cudaMemcpy(&cf, I->ev_fit.p, sizeof(double), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&co, I->ev_obj.p, sizeof(double), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&f0, c->fit.as<double>() + (size_t)q * c->n + index, sizeof(double), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&o0, c->obj.as<double>() + (size_t)q * c->n + index, sizeof(double), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&used, draws.p, sizeof(used), cudaMemcpyDeviceToHost));
        const bool rep = cf > f0;  // strict improvement (cellular.cpp:153)
        const size_t L = (size_t)I->J * I->S;
        DevBuf out, didx;
        out.alloc(sizeof(int32_t) * L);
        const uint8_t* src = I->ev_rows.as<uint8_t>();
        long long row = 0;
        if (!rep) {
            src = c->genes.as<uint8_t>();
            row = cell_storage_index(c)[index];
        }
        std::vector<long long> idx{row};
        upload(didx, idx);
        CK(launch_rows_to_int(I->d, src, (long long)I->block(), didx.as<long long>(), out.as<int32_t>(), 1, I->stream));
        g_launches += 1;
        CK(cudaMemcpyAsync(genes, out.p, sizeof(int32_t) * L, cudaMemcpyDeviceToHost, I->stream));
        CK(cudaStreamSynchronize(I->stream));
        *fit = rep ? cf : f0;
        *obj = rep ? co : o0;
        *replaced = rep ? 1 : 0;
        if (draws_used) *draws_used = used;
    });
}

int ffsga_cuda_cellular_install(ffsga_cuda_cellular c, int index, const int32_t* genes, double fit, double obj) {
    return guard([&] {
        if (!c || !genes) fail(FFSGA_ERR_ARG, "null pointer");
        if (index < 0 || index >= c->n) fail(FFSGA_ERR_CONTRACT, "cell index out of range");
        std::lock_guard<std::mutex> lk(c->inst->mu);
        ffsga_cuda_instance_t* I = c->inst;
        I->use();
        const long long slot = cell_storage_index(c)[index];
        const size_t L = (size_t)I->J * I->S;
        DevBuf tmp;
        tmp.alloc(sizeof(int32_t) * L);
        CK(cudaMemcpy(tmp.p, genes, sizeof(int32_t) * L, cudaMemcpyHostToDevice));
        CK(launch_rows_from_int(I->d, tmp.as<int32_t>(), nullptr, c->genes.as<uint8_t>() + slot * I->block(), 1, I->stream));
        g_launches += 1;
        const size_t off = (size_t)c->parity() * c->n + index;
        CK(cudaMemcpyAsync(c->fit.as<double>() + off, &fit, sizeof(double), cudaMemcpyHostToDevice, I->stream));
        CK(cudaMemcpyAsync(c->obj.as<double>() + off, &obj, sizeof(double), cudaMemcpyHostToDevice, I->stream));
        refresh_stats(c, nullptr, 0);
        CK(cudaStreamSynchronize(I->stream));
    });
}

int ffsga_cuda_pseudo_create(ffsga_cuda_instance inst, int population, double xr, uint64_t seed,
                             ffsga_cuda_pseudo* out) {
    return guard([&] {
        NvtxRange nvtx_range("ffsga_cuda_pseudo_create");
        if (!inst || !out) fail(FFSGA_ERR_ARG, "pseudo_create: null pointer");
        *out = nullptr;
        if (population < 2 || population % 2 != 0)
            fail(FFSGA_ERR_CONFIG, "pseudo island population must be even and >= 2");
        if (!(xr >= 0.0 && xr <= 1.0)) fail(FFSGA_ERR_CONFIG, "pseudo crossover rate must lie in [0, 1]");
        std::lock_guard<std::mutex> lk(inst->mu);
        ffsga_cuda_instance_t* I = inst;
        I->use();
        const bool dbg = std::getenv("FFSGA_DEBUG_INIT") != nullptr;
        auto t_last = std::chrono::steady_clock::now();
        auto mark = [&](const char* what) {
            if (!dbg) return;
            const auto t = std::chrono::steady_clock::now();
            std::fprintf(stderr, "pseudo_create %-24s %.3f ms\n", what,
                         std::chrono::duration<double, std::milli>(t - t_last).count());
            t_last = t;
        };
        auto* p = new ffsga_cuda_pseudo_t();
        std::unique_ptr<ffsga_cuda_pseudo_t> hold(p);
        p->inst = I;
        p->adopt(I->stream);
        p->n = population;
        const int W = I->words;
        p->words.alloc(sizeof(unsigned long long) * (size_t)W * population);
        p->fit.alloc(sizeof(double) * population);
        p->obj.alloc(sizeof(double) * population);
        p->mslot.alloc(sizeof(long long) * population);
        p->archive.alloc(sizeof(unsigned long long) * W);
        CK(cudaMemsetAsync(p->archive.p, 0, sizeof(unsigned long long) * W, I->stream));
        p->st.alloc(sizeof(IslandState));
        IslandState s0{};
        s0.arch_fit = -1.0;  // pseudo.hpp:79
        s0.arch_obj = 0.0;
        CK(cudaMemcpyAsync(p->st.p, &s0, sizeof(s0), cudaMemcpyHostToDevice, I->stream));  // pageable: staged
        p->trace_cap = 1;
        p->trace.alloc(sizeof(double));
        mark("allocs");
        // pairs (x, ~x): x = pair p's chromosome of the sequential init stream (pseudo.cpp:40-47).
        // The island's row storage (gene rows of its crossed members in every generation) holds
        // the initial members' rows for their first evaluation.  An island-sized buffer is
        // recycled by the stream-ordered pool across models (a shared arena regrown by the first
        // step was not: 10-45 ms to map per model).
        const size_t block = I->block();
        p->rows.alloc(block * (size_t)population);
        uint8_t* rows = p->rows.as<uint8_t>();
        mark("rows");
        CK(launch_random_rows(I->d, rows, (long long)block, population / 2, seed, 0, false, I->stream));
        CK(launch_pack_bits(I->d, rows, (long long)block, nullptr, p->words.as<unsigned long long>(), nullptr,
                            population / 2, true, I->dBitStage.as<uint16_t>(), I->stream));
        CK(launch_unpack_rows(I->d, p->words.as<unsigned long long>(), nullptr, rows, (long long)block, nullptr,
                              population, I->stream));
        g_launches += 3;
        mark("init launches");
        eval_rows(I, rows, population, p->obj.as<double>(), p->fit.as<double>(), nullptr, nullptr, false);
        mark("eval_rows");
        PseudoIsland& d = p->d;  // (device-generated genes: in range by construction)
        d.n = population;
        d.words = p->words.as<unsigned long long>();
        d.fit = p->fit.as<double>();
        d.obj = p->obj.as<double>();
        d.mslot = p->mslot.as<long long>();
        d.rows = p->rows.as<uint8_t>();
        d.archive = p->archive.as<unsigned long long>();
        d.seed = seed;
        d.thr_xr = coin_threshold(xr);
        d.st = p->st.as<IslandState>();
        d.pair0 = 0;
        p->push_desc();
        refresh_stats(nullptr, p, 2);  // archive = first max over the scored members
        mark("stats");
        *out = hold.release();          // stream-ordered, as cellular_create
    });
}

int ffsga_cuda_pseudo_destroy(ffsga_cuda_pseudo p) {
    return guard([&] {
        if (p) p->inst->use();
        delete p;
    });
}

int ffsga_cuda_pseudo_size(ffsga_cuda_pseudo p, int* size, int* total_bits) {
    return guard([&] {
        if (!p) fail(FFSGA_ERR_ARG, "null island");
        if (size) *size = p->n;
        if (total_bits) *total_bits = p->inst->total_bits;
    });
}

int ffsga_cuda_pseudo_generation(ffsga_cuda_pseudo p, uint64_t* g) {
    return guard([&] {
        if (!p || !g) fail(FFSGA_ERR_ARG, "null pointer");
        *g = p->gen;
    });
}

int ffsga_cuda_pseudo_read(ffsga_cuda_pseudo p, double* fit, double* obj) {
    return guard([&] {
        if (!p) fail(FFSGA_ERR_ARG, "null island");
        std::lock_guard<std::mutex> lk(p->inst->mu);
        p->inst->use();
        if (fit) CK(cudaMemcpyAsync(fit, p->fit.p, sizeof(double) * p->n, cudaMemcpyDeviceToHost, p->inst->stream));
        if (obj) CK(cudaMemcpyAsync(obj, p->obj.p, sizeof(double) * p->n, cudaMemcpyDeviceToHost, p->inst->stream));
        CK(cudaStreamSynchronize(p->inst->stream));
    });
}

int ffsga_cuda_pseudo_member(ffsga_cuda_pseudo p, int index, uint8_t* bits) {
    return guard([&] {
        if (!p || !bits) fail(FFSGA_ERR_ARG, "null pointer");
        if (index >= p->n) fail(FFSGA_ERR_CONTRACT, "member index out of range");
        std::lock_guard<std::mutex> lk(p->inst->mu);
        ffsga_cuda_instance_t* I = p->inst;
        I->use();
        const int W = I->words, nb = I->total_bits;
        const int first = index < 0 ? 0 : index;
        const int count = index < 0 ? p->n : 1;
        std::vector<unsigned long long> w((size_t)W * count);
        CK(cudaMemcpyAsync(w.data(), p->words.as<unsigned long long>() + (size_t)first * W, sizeof(unsigned long long) * w.size(),
                           cudaMemcpyDeviceToHost, I->stream));
        CK(cudaStreamSynchronize(I->stream));
        for (int i = 0; i < count; ++i) unpack_host_bits(w.data() + (size_t)i * W, nb, bits + (size_t)i * nb);
    });
}

int ffsga_cuda_pseudo_best(ffsga_cuda_pseudo p, int* index, double* fit, double* obj) {
    return guard([&] {
        if (!p) fail(FFSGA_ERR_ARG, "null island");
        std::lock_guard<std::mutex> lk(p->inst->mu);
        p->inst->use();
        IslandState s = read_state(p->inst, p->st);
        if (index) *index = s.best_idx;
        if (fit) *fit = s.best_fit;
        if (obj) *obj = s.best_obj;
    });
}

int ffsga_cuda_pseudo_archive(ffsga_cuda_pseudo p, double* fit, double* obj, uint8_t* bits) {
    return guard([&] {
        if (!p) fail(FFSGA_ERR_ARG, "null island");
        std::lock_guard<std::mutex> lk(p->inst->mu);
        ffsga_cuda_instance_t* I = p->inst;
        I->use();
        IslandState s = read_state(I, p->st);
        if (fit) *fit = s.arch_fit;
        if (obj) *obj = s.arch_obj;
        if (bits) {
            std::vector<unsigned long long> w(I->words);
            CK(cudaMemcpy(w.data(), p->archive.p, sizeof(unsigned long long) * I->words, cudaMemcpyDeviceToHost));
            unpack_host_bits(w.data(), I->total_bits, bits);
        }
    });
}

int ffsga_cuda_pseudo_archive_genes(ffsga_cuda_pseudo p, int32_t* genes) {
    return guard([&] {
        if (!p || !genes) fail(FFSGA_ERR_ARG, "null pointer");
        std::lock_guard<std::mutex> lk(p->inst->mu);
        ffsga_cuda_instance_t* I = p->inst;
        I->use();
        const size_t L = (size_t)I->J * I->S;
        DevBuf rows, out;
        rows.alloc(I->block());
        out.alloc(sizeof(int32_t) * L);
        CK(launch_unpack_rows(I->d, p->archive.as<unsigned long long>(), nullptr, rows.as<uint8_t>(), (long long)I->block(),
                              nullptr, 1, I->stream));
        CK(launch_rows_to_int(I->d, rows.as<uint8_t>(), (long long)I->block(), nullptr, out.as<int32_t>(), 1, I->stream));
        g_launches += 2;
        CK(cudaMemcpyAsync(genes, out.p, sizeof(int32_t) * L, cudaMemcpyDeviceToHost, I->stream));
        CK(cudaStreamSynchronize(I->stream));
    });
}

int ffsga_cuda_pseudo_install(ffsga_cuda_pseudo p, int index, const uint8_t* bits, double fit, double obj) {
    return guard([&] {
        if (!p || !bits) fail(FFSGA_ERR_ARG, "null pointer");
        if (index < 0 || index >= p->n) fail(FFSGA_ERR_CONTRACT, "member index out of range");
        std::lock_guard<std::mutex> lk(p->inst->mu);
        ffsga_cuda_instance_t* I = p->inst;
        I->use();
        std::vector<unsigned long long> w;
        pack_host_bits(bits, I->total_bits, I->words, w);
        CK(cudaMemcpy(p->words.as<unsigned long long>() + (size_t)index * I->words, w.data(),
                      sizeof(unsigned long long) * I->words, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(p->fit.as<double>() + index, &fit, sizeof(double), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(p->obj.as<double>() + index, &obj, sizeof(double), cudaMemcpyHostToDevice));
        IslandState s = read_state(I, p->st);
        if (fit > s.arch_fit) {  // consider_for_archive (pseudo.cpp:106-113)
            s.arch_fit = fit;
            s.arch_obj = obj;
            CK(cudaMemcpy(p->st.p, &s, sizeof(s), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(p->archive.p, w.data(), sizeof(unsigned long long) * I->words, cudaMemcpyHostToDevice));
        }
        refresh_stats(nullptr, p, 0);
        CK(cudaStreamSynchronize(I->stream));
    });
}

int ffsga_cuda_step(const ffsga_cuda_cellular* cells, int nc, const ffsga_cuda_pseudo* pseudos, int np,
                    int generations, double* trace_c, double* trace_p) {
    return guard([&] {
        NvtxRange nvtx_range("ffsga_cuda_step");
        if (nc < 0 || np < 0 || (nc > 0 && !cells) || (np > 0 && !pseudos)) fail(FFSGA_ERR_ARG, "step: bad island list");
        if (generations < 0) fail(FFSGA_ERR_CONTRACT, "step: negative generation count");
        if (nc + np == 0 || generations == 0) return;
        ffsga_cuda_instance_t* I = nc > 0 ? cells[0]->inst : pseudos[0]->inst;
        for (int i = 0; i < nc; ++i)
            if (!cells[i] || cells[i]->inst != I) fail(FFSGA_ERR_ARG, "step: islands must share one instance");
        for (int i = 0; i < np; ++i)
            if (!pseudos[i] || pseudos[i]->inst != I) fail(FFSGA_ERR_ARG, "step: islands must share one instance");
        std::lock_guard<std::mutex> lk(I->mu);
        I->use();
        const bool dbg = std::getenv("FFSGA_DEBUG_STEP") != nullptr;  // host-side phase timing
        auto t_last = std::chrono::steady_clock::now();
        auto mark = [&](const char* what) {
            if (!dbg) return;
            const auto t = std::chrono::steady_clock::now();
            std::fprintf(stderr, "step %-24s %.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t_last).count());
            t_last = t;
        };
        // Descriptors of this joint step.  The islands are split into step groups (up to
        // step_split contiguous groups of each kind) and every group runs its own breed ->
        // evaluate -> commit chain on its own stream: groups never read each other between
        // rendezvous, so the GPU overlaps the integer-bound breeding of one group with the
        // latency-bound decoding of another and fills the tail of every decoder launch.
        // Work-list items: every cell in island order, then per pseudo group a region of
        // 2 x its pairs for the crossed members.
        const int split = std::max(1, I->step_split);
        const int gc = nc ? std::min(nc, split) : 0, gp = np ? std::min(np, split) : 0;
        std::vector<CellIsland> cd(nc);
        std::vector<PseudoIsland> pd(np);
        std::vector<long long> cell_base(nc + 1, 0), pair_base(np + 1, 0);
        for (int i = 0; i < nc; ++i) {
            auto* c = cells[i];
            if (c->trace_cap < generations) {
                c->trace.alloc(sizeof(double) * generations);
                c->trace_cap = generations;
            }
            c->d.trace = c->trace.as<double>();
            cd[i] = c->d;
            cd[i].item0 = cell_base[i];
            cell_base[i + 1] = cell_base[i] + c->n;
            CK(cudaMemcpyAsync(&c->st.as<IslandState>()->seg_start, &c->gen, sizeof(unsigned long long),
                               cudaMemcpyHostToDevice, I->stream));
        }
        for (int i = 0; i < np; ++i) {
            auto* p = pseudos[i];
            if (p->trace_cap < generations) {
                p->trace.alloc(sizeof(double) * generations);
                p->trace_cap = generations;
            }
            p->d.trace = p->trace.as<double>();
            pd[i] = p->d;
            pair_base[i + 1] = pair_base[i] + p->n / 2;
            CK(cudaMemcpyAsync(&p->st.as<IslandState>()->seg_start, &p->gen, sizeof(unsigned long long),
                               cudaMemcpyHostToDevice, I->stream));
        }
        const long long n_cells = cell_base[nc], n_pairs = pair_base[np];
        // A step group owns a range of cellular islands [c0, c1) and of pseudo islands [p0, p1)
        // and a work-list region: its cells first, then its crossed pseudo members (slots from
        // the group counter); every index inside the group's kernels is group-relative.
        struct Group {
            int c0, c1, p0, p1;
            long long cells, pairs;  // units of the group
            long long item0;  // first work-list item
        };
        std::vector<Group> groups;
        auto add_group = [&](int c0, int c1, int p0, int p1) {
            Group G{c0, c1, p0, p1, cell_base[c1] - cell_base[c0], pair_base[p1] - pair_base[p0], 0};
            if (G.cells + G.pairs == 0) return;
            if (!groups.empty()) {
                const Group& L = groups.back();
                G.item0 = L.item0 + L.cells + 2 * L.pairs;
            }
            for (int i = c0; i < c1; ++i) cd[i].item0 = cd[i].cell0 = cell_base[i] - cell_base[c0];
            for (int i = p0; i < p1; ++i) pd[i].pair0 = pair_base[i] - pair_base[p0];
            groups.push_back(G);
        };
        if (I->step_mix > 0) {  // mixed groups: each takes a share of both kinds
            const int S = std::max(1, std::min(I->step_mix, std::max(nc, np)));
            for (int g = 0; g < S; ++g)
                add_group((int)((long long)g * nc / S), (int)((long long)(g + 1) * nc / S),
                          (int)((long long)g * np / S), (int)((long long)(g + 1) * np / S));
        } else {  // kind groups: cellular islands in gc groups, pseudo islands in gp groups
            for (int g = 0; g < gc; ++g)
                add_group((int)((long long)g * nc / gc), (int)((long long)(g + 1) * nc / gc), 0, 0);
            for (int g = 0; g < gp; ++g)
                add_group(0, 0, (int)((long long)g * np / gp), (int)((long long)(g + 1) * np / gp));
        }
        const long long cap = n_cells + 2 * n_pairs;
        I->wl_ptrs.ensure(sizeof(void*) * cap);
        I->wl_obj.ensure(sizeof(double) * cap);
        I->wl_fit.ensure(sizeof(double) * cap);
        I->wl_count.ensure(sizeof(long long) * std::max<size_t>(2, groups.size()));
        I->cell_desc.ensure(sizeof(CellIsland) * std::max(1, nc));
        I->pseudo_desc.ensure(sizeof(PseudoIsland) * std::max(1, np));
        if (nc) CK(cudaMemcpyAsync(I->cell_desc.p, cd.data(), sizeof(CellIsland) * nc, cudaMemcpyHostToDevice, I->stream));
        if (np) CK(cudaMemcpyAsync(I->pseudo_desc.p, pd.data(), sizeof(PseudoIsland) * np, cudaMemcpyHostToDevice, I->stream));
        const CellIsland* cdev = I->cell_desc.as<CellIsland>();
        const PseudoIsland* pdev = I->pseudo_desc.as<PseudoIsland>();
        // group 0 runs on the instance stream, the others on side streams forked from it
        while (I->side.size() + 1 < groups.size()) {
            cudaStream_t s;
            cudaEvent_t e;
            CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            I->side.push_back(s);
            I->side_join.push_back(e);
        }
        struct Chain {
            cudaStream_t st;
            WorkList w;
            EvalItems E;
        };
        std::vector<Chain> chains(groups.size());
        const uint8_t** ptrs = I->wl_ptrs.as<const uint8_t*>();
        double* wobj = I->wl_obj.as<double>();
        double* wfit = I->wl_fit.as<double>();
        for (size_t k = 0; k < groups.size(); ++k) {
            const Group& G = groups[k];
            Chain& ch = chains[k];
            ch.st = k == 0 ? I->stream : I->side[k - 1];
            WorkList w{};
            w.ptrs = ptrs + G.item0;
            w.obj = wobj + G.item0;
            w.fit = wfit + G.item0;
            w.count = I->wl_count.as<long long>() + k;  // gen-begin sets it to the group's cells
            w.total = I->eval_total.as<unsigned long long>();
            EvalItems E{};
            E.ptrs = w.ptrs;
            E.obj = w.obj;
            E.fit = w.fit;
            E.n_dev = w.count;
            E.deal = groups.size() == 1 ? 1 : 0;  // a lone decoder launch owns the GPU
            ch.w = w;
            ch.E = E;
        }
        auto enqueue = [&](int gens, bool timed) {
            CK(cudaEventRecord(I->fork, I->stream));
            for (size_t k = 1; k < chains.size(); ++k) CK(cudaStreamWaitEvent(chains[k].st, I->fork, 0));
            for (int g = 0; g < gens; ++g) {
                for (size_t k = 0; k < chains.size(); ++k) {
                    const Group& G = groups[k];
                    const Chain& ch = chains[k];
                    auto b = [&] {
                        CK(launch_breed(I->d, cdev + G.c0, G.c1 - G.c0, G.cells, pdev + G.p0, G.p1 - G.p0, G.pairs,
                                        ch.w, ch.st));
                    };
                    auto e = [&] {
                        // one group alone owns the GPU: the standalone configuration fits it best
                        const EvalConfig& ec = groups.size() == 1 ? I->ec : I->ec_step;
                        CK(launch_eval(I->d, ec, ch.E, G.cells + 2 * G.pairs, I->sm_count, false, ch.st));
                    };
                    auto c = [&] {
                        CK(launch_commit(I->d, cdev + G.c0, G.c1 - G.c0, pdev + G.p0, G.p1 - G.p0, ch.w, ch.st));
                    };
                    if (timed) {
                        I->timed_on(1, ch.st, b);
                        I->timed_on(0, ch.st, e);
                        I->timed_on(2, ch.st, c);
                    } else {
                        b();
                        e();
                        c();
                    }
                }
            }
            for (size_t k = 1; k < chains.size(); ++k) {
                CK(cudaEventRecord(I->side_join[k - 1], chains[k].st));
                CK(cudaStreamWaitEvent(I->stream, I->side_join[k - 1], 0));
            }
        };
        long long per_gen = 0;
        for (const Group& G : groups) per_gen += 3 + (G.cells ? 1 : 0) + (G.pairs ? 1 : 0);
        // graphs pay off when a generation is launch bound (small islands); capturing costs
        // ~0.1 s, so large work lists run plain launches
        const bool use_graph = !I->timing && generations >= 2 && cap <= 16384 && !std::getenv("FFSGA_NO_GRAPH");
        mark("setup");
        CK(cudaEventRecord(I->st0, I->stream));
        if (use_graph) {
            // the generation sequence is launch-bound for small islands: capture a chunk of
            // generations once (device-side generation counters make it replayable)
            const int chunk = std::min(generations, 16);
            // the captured launches bake in every group's island range, unit counts (grid sizes)
            // and work-list offset, so all of them are part of the key
            std::vector<const void*> key = {cdev, pdev, (const void*)ptrs, (const void*)wobj,
                                            I->wl_count.p, (const void*)groups.size(),
                                            (const void*)(intptr_t)nc, (const void*)(intptr_t)np,
                                            (const void*)(intptr_t)n_cells, (const void*)(intptr_t)n_pairs,
                                            (const void*)(intptr_t)chunk};
            for (const Group& G : groups)
                for (long long v : {(long long)G.c0, (long long)G.c1, (long long)G.p0, (long long)G.p1, G.cells,
                                    G.pairs, G.item0})
                    key.push_back((const void*)(intptr_t)v);
            if (!I->graph_exec || I->graph_key != key) {
                if (I->graph_exec) {
                    CK(cudaGraphExecDestroy(I->graph_exec));
                    I->graph_exec = nullptr;
                }
                cudaGraph_t graph = nullptr;
                CK(cudaStreamBeginCapture(I->stream, cudaStreamCaptureModeThreadLocal));
                enqueue(chunk, false);
                CK(cudaStreamEndCapture(I->stream, &graph));
                cudaError_t e = cudaGraphInstantiate(&I->graph_exec, graph, 0);
                cudaGraphDestroy(graph);
                CK(e);
                I->graph_key = key;
            }
            for (int done = 0; done + chunk <= generations; done += chunk) CK(cudaGraphLaunch(I->graph_exec, I->stream));
            if (generations % chunk) enqueue(generations % chunk, false);
        } else {
            enqueue(generations, true);
        }
        g_launches += per_gen * generations;
        CK(cudaEventRecord(I->st1, I->stream));
        mark("enqueue");
        I->step_recorded = true;
        for (int i = 0; i < nc; ++i) {
            if (trace_c)
                CK(cudaMemcpyAsync(trace_c + (size_t)i * generations, cells[i]->trace.p, sizeof(double) * generations,
                                   cudaMemcpyDeviceToHost, I->stream));
        }
        for (int i = 0; i < np; ++i) {
            if (trace_p)
                CK(cudaMemcpyAsync(trace_p + (size_t)i * generations, pseudos[i]->trace.p, sizeof(double) * generations,
                                   cudaMemcpyDeviceToHost, I->stream));
        }
        CK(cudaStreamSynchronize(I->stream));
        mark("traces+sync");
        for (int i = 0; i < nc; ++i) cells[i]->gen += (unsigned long long)generations;
        for (int i = 0; i < np; ++i) pseudos[i]->gen += (unsigned long long)generations;
    });
}

}  // extern "C"

namespace {

// sort_island order (fitness desc, index asc) of n fitness values into idx_out (device)
void sort_island_dev(ffsga_cuda_instance_t* I, const double* fit, long long n, DevBuf& idx_out) {
    I->mg_keys0.ensure(sizeof(double) * n);
    I->mg_keys1.ensure(sizeof(double) * n);
    I->mg_idx0.ensure(sizeof(long long) * n);
    idx_out.ensure(sizeof(long long) * n);
    const size_t tb = sort_temp_bytes(n);
    I->mg_temp.ensure(std::max<size_t>(tb, 16));
    CK(launch_sort_desc(fit, n, I->mg_keys0.as<double>(), I->mg_keys1.as<double>(), I->mg_idx0.as<long long>(),
                        idx_out.as<long long>(), I->mg_temp.p, tb, I->stream));
    g_launches += 3;
}

void check_count(int k, int a, int b) {  // migration.cpp:40-43
    if (k < 0 || k > a || k > b) fail(FFSGA_ERR_CONTRACT, "migrate: migrant count exceeds an island population");
}

}  // namespace

extern "C" {

int ffsga_cuda_migrate_cellular_to_pseudo(ffsga_cuda_cellular from, ffsga_cuda_pseudo to, int k) {
    return guard([&] {
        NvtxRange nvtx_range("ffsga_cuda_migrate_cellular_to_pseudo");
        if (!from || !to) fail(FFSGA_ERR_ARG, "migrate: null island");
        if (from->inst != to->inst) fail(FFSGA_ERR_ARG, "migrate: islands must share one instance");
        check_count(k, from->n, to->n);
        if (k == 0) return;
        ffsga_cuda_instance_t* I = from->inst;
        std::lock_guard<std::mutex> lk(I->mu);
        I->use();
        const int q = from->parity();
        sort_island_dev(I, from->fit.as<double>() + (size_t)q * from->n, from->n, I->mg_idx_a);
        sort_island_dev(I, to->fit.as<double>(), to->n, I->mg_idx_b);
        CK(launch_migrate_c2p(I->d, from->d, to->d, I->mg_idx_a.as<long long>(), I->mg_idx_b.as<long long>(), k, q,
                              I->dBitStage.as<uint16_t>(), I->stream));
        g_launches += 2;
        refresh_stats(nullptr, to, 0);
        CK(cudaStreamSynchronize(I->stream));
    });
}

int ffsga_cuda_migrate_pseudo_to_cellular(ffsga_cuda_pseudo from, ffsga_cuda_cellular to, int k) {
    return guard([&] {
        NvtxRange nvtx_range("ffsga_cuda_migrate_pseudo_to_cellular");
        if (!from || !to) fail(FFSGA_ERR_ARG, "migrate: null island");
        if (from->inst != to->inst) fail(FFSGA_ERR_ARG, "migrate: islands must share one instance");
        check_count(k, from->n, to->n);
        if (k == 0) return;
        ffsga_cuda_instance_t* I = from->inst;
        std::lock_guard<std::mutex> lk(I->mu);
        I->use();
        const int q = to->parity();
        sort_island_dev(I, from->fit.as<double>(), from->n, I->mg_idx_a);
        sort_island_dev(I, to->fit.as<double>() + (size_t)q * to->n, to->n, I->mg_idx_b);
        CK(launch_migrate_p2c(I->d, from->d, to->d, I->mg_idx_a.as<long long>(), I->mg_idx_b.as<long long>(), k, q,
                              I->stream));
        g_launches += 1;
        refresh_stats(to, nullptr, 0);
        CK(cudaStreamSynchronize(I->stream));
    });
}

}  // extern "C"

namespace {

// ---- migrant packets: [fit[k] fp64][obj[k] fp64][payload] (kernels.cu "Migrant packets")
size_t packet_bytes(const ffsga_cuda_instance_t* I, int from_kind, int k) {
    const size_t payload = from_kind == 0 ? I->block() : sizeof(unsigned long long) * (size_t)I->words;
    return (size_t)k * (2 * sizeof(double) + payload);
}

// Every packet routine runs on the instance stream under I->mu, ordered after the caller's
// stream (fork) and before the caller's later work (join): no host synchronisation.
struct Ordered {
    ffsga_cuda_instance_t* I;
    cudaStream_t user;
    Ordered(ffsga_cuda_instance_t* I_, void* stream) : I(I_), user(static_cast<cudaStream_t>(stream)) {
        CK(cudaEventRecord(I->fork, user));
        CK(cudaStreamWaitEvent(I->stream, I->fork, 0));
    }
    void done() {
        CK(cudaEventRecord(I->join, I->stream));
        CK(cudaStreamWaitEvent(user, I->join, 0));
    }
};

void export_cell_packet(ffsga_cuda_cellular_t* c, int k, unsigned char* packet) {
    ffsga_cuda_instance_t* I = c->inst;
    const int q = c->parity();
    sort_island_dev(I, c->fit.as<double>() + (size_t)q * c->n, c->n, I->mg_idx_a);
    CK(launch_export_cell(I->d, c->d, I->mg_idx_a.as<long long>(), k, q, packet + 2 * sizeof(double) * k,
                          reinterpret_cast<double*>(packet), I->stream));
    g_launches += 1;
}

void export_pseudo_packet(ffsga_cuda_pseudo_t* p, int k, unsigned char* packet) {
    ffsga_cuda_instance_t* I = p->inst;
    sort_island_dev(I, p->fit.as<double>(), p->n, I->mg_idx_a);
    CK(launch_export_pseudo(I->d, p->d, I->mg_idx_a.as<long long>(), k,
                            reinterpret_cast<unsigned long long*>(packet + 2 * sizeof(double) * k),
                            reinterpret_cast<double*>(packet), I->stream));
    g_launches += 1;
}

// a pseudo island's packet installed over the k worst cells (migration.cpp:59-69)
void import_into_cell(ffsga_cuda_cellular_t* c, int k, const unsigned char* packet) {
    ffsga_cuda_instance_t* I = c->inst;
    const int q = c->parity();
    sort_island_dev(I, c->fit.as<double>() + (size_t)q * c->n, c->n, I->mg_idx_b);
    CK(launch_migrate_p2c(I->d, PseudoIsland{}, c->d, nullptr, I->mg_idx_b.as<long long>(), k, q, I->stream,
                          reinterpret_cast<const unsigned long long*>(packet + 2 * sizeof(double) * k),
                          reinterpret_cast<const double*>(packet)));
    g_launches += 1;
    refresh_stats(c, nullptr, 0);
}

// a cellular island's packet installed over the k worst members; the archive absorbs them
// (migration.cpp:47-57, pseudo.cpp:98-113)
void import_into_pseudo(ffsga_cuda_pseudo_t* p, int k, const unsigned char* packet) {
    ffsga_cuda_instance_t* I = p->inst;
    sort_island_dev(I, p->fit.as<double>(), p->n, I->mg_idx_b);
    CK(launch_migrate_c2p(I->d, CellIsland{}, p->d, nullptr, I->mg_idx_b.as<long long>(), k, 0,
                          I->dBitStage.as<uint16_t>(), I->stream, packet + 2 * sizeof(double) * k,
                          reinterpret_cast<const double*>(packet)));
    g_launches += 2;
    refresh_stats(nullptr, p, 0);
}

void check_migrants(int k, int n, const void* ptr) {
    if (k < 0 || k > n) fail(FFSGA_ERR_CONTRACT, "migrate: migrant count exceeds an island population");
    if (k > 0 && !ptr) fail(FFSGA_ERR_ARG, "migrant packet: null pointer");
}

}  // namespace

extern "C" {

int ffsga_cuda_packet_bytes(ffsga_cuda_instance inst, int from_kind, int k, int64_t* bytes) {
    return guard([&] {
        if (!inst || !bytes || (from_kind != 0 && from_kind != 1) || k < 0) fail(FFSGA_ERR_ARG, "packet_bytes: bad argument");
        *bytes = (int64_t)packet_bytes(inst, from_kind, k);
    });
}

int ffsga_cuda_cellular_export_device(ffsga_cuda_cellular c, int k, void* packet, void* stream) {
    return guard([&] {
        NvtxRange nvtx_range("ffsga_cuda_cellular_export_device");
        if (!c) fail(FFSGA_ERR_ARG, "export: null island");
        check_migrants(k, c->n, packet);
        if (k == 0) return;
        std::lock_guard<std::mutex> lk(c->inst->mu);
        c->inst->use();
        Ordered o(c->inst, stream);
        export_cell_packet(c, k, static_cast<unsigned char*>(packet));
        o.done();
    });
}

int ffsga_cuda_pseudo_export_device(ffsga_cuda_pseudo p, int k, void* packet, void* stream) {
    return guard([&] {
        NvtxRange nvtx_range("ffsga_cuda_pseudo_export_device");
        if (!p) fail(FFSGA_ERR_ARG, "export: null island");
        check_migrants(k, p->n, packet);
        if (k == 0) return;
        std::lock_guard<std::mutex> lk(p->inst->mu);
        p->inst->use();
        Ordered o(p->inst, stream);
        export_pseudo_packet(p, k, static_cast<unsigned char*>(packet));
        o.done();
    });
}

int ffsga_cuda_cellular_import_device(ffsga_cuda_cellular c, int k, const void* packet, void* stream) {
    return guard([&] {
        NvtxRange nvtx_range("ffsga_cuda_cellular_import_device");
        if (!c) fail(FFSGA_ERR_ARG, "import: null island");
        check_migrants(k, c->n, packet);
        if (k == 0) return;
        std::lock_guard<std::mutex> lk(c->inst->mu);
        c->inst->use();
        Ordered o(c->inst, stream);
        import_into_cell(c, k, static_cast<const unsigned char*>(packet));
        o.done();
    });
}

int ffsga_cuda_pseudo_import_device(ffsga_cuda_pseudo p, int k, const void* packet, void* stream) {
    return guard([&] {
        NvtxRange nvtx_range("ffsga_cuda_pseudo_import_device");
        if (!p) fail(FFSGA_ERR_ARG, "import: null island");
        check_migrants(k, p->n, packet);
        if (k == 0) return;
        std::lock_guard<std::mutex> lk(p->inst->mu);
        p->inst->use();
        Ordered o(p->inst, stream);
        import_into_pseudo(p, k, static_cast<const unsigned char*>(packet));
        o.done();
    });
}

int ffsga_cuda_cellular_state_device(ffsga_cuda_cellular c, double* out4, void* stream) {
    return guard([&] {
        if (!c || !out4) fail(FFSGA_ERR_ARG, "state_device: null pointer");
        std::lock_guard<std::mutex> lk(c->inst->mu);
        c->inst->use();
        Ordered o(c->inst, stream);
        CK(cudaMemcpyAsync(out4, reinterpret_cast<const char*>(c->st.p) + offsetof(IslandState, best_fit),
                           4 * sizeof(double), cudaMemcpyDeviceToDevice, c->inst->stream));
        o.done();
    });
}

int ffsga_cuda_pseudo_state_device(ffsga_cuda_pseudo p, double* out4, void* stream) {
    return guard([&] {
        if (!p || !out4) fail(FFSGA_ERR_ARG, "state_device: null pointer");
        std::lock_guard<std::mutex> lk(p->inst->mu);
        p->inst->use();
        Ordered o(p->inst, stream);
        CK(cudaMemcpyAsync(out4, reinterpret_cast<const char*>(p->st.p) + offsetof(IslandState, best_fit),
                           4 * sizeof(double), cudaMemcpyDeviceToDevice, p->inst->stream));
        o.done();
    });
}

// ---- host-buffer export/import: the same packets, staged through host memory
int ffsga_cuda_cellular_export(ffsga_cuda_cellular c, int k, int32_t* genes, double* fit, double* obj) {
    return guard([&] {
        NvtxRange nvtx_range("ffsga_cuda_cellular_export");
        if (!c || (k > 0 && (!genes || !fit || !obj))) fail(FFSGA_ERR_ARG, "export: null pointer");
        check_migrants(k, c->n, genes);
        if (k == 0) return;
        ffsga_cuda_instance_t* I = c->inst;
        std::lock_guard<std::mutex> lk(I->mu);
        I->use();
        DevBuf pk, out;
        pk.alloc(packet_bytes(I, 0, k));
        export_cell_packet(c, k, pk.as<unsigned char>());
        const size_t L = (size_t)I->J * I->S;
        out.alloc(sizeof(int32_t) * L * k);
        CK(launch_rows_to_int(I->d, pk.as<uint8_t>() + 2 * sizeof(double) * k, (long long)I->block(), nullptr,
                              out.as<int32_t>(), k, I->stream));
        g_launches += 1;
        CK(cudaMemcpyAsync(genes, out.p, sizeof(int32_t) * L * k, cudaMemcpyDeviceToHost, I->stream));
        CK(cudaMemcpyAsync(fit, pk.p, sizeof(double) * k, cudaMemcpyDeviceToHost, I->stream));
        CK(cudaMemcpyAsync(obj, pk.as<double>() + k, sizeof(double) * k, cudaMemcpyDeviceToHost, I->stream));
        CK(cudaStreamSynchronize(I->stream));
    });
}

int ffsga_cuda_pseudo_export(ffsga_cuda_pseudo p, int k, uint8_t* bits, double* fit, double* obj) {
    return guard([&] {
        NvtxRange nvtx_range("ffsga_cuda_pseudo_export");
        if (!p || (k > 0 && (!bits || !fit || !obj))) fail(FFSGA_ERR_ARG, "export: null pointer");
        check_migrants(k, p->n, bits);
        if (k == 0) return;
        ffsga_cuda_instance_t* I = p->inst;
        std::lock_guard<std::mutex> lk(I->mu);
        I->use();
        DevBuf pk;
        const size_t bytes = packet_bytes(I, 1, k);
        pk.alloc(bytes);
        export_pseudo_packet(p, k, pk.as<unsigned char>());
        std::vector<unsigned char> host(bytes);
        CK(cudaMemcpyAsync(host.data(), pk.p, bytes, cudaMemcpyDeviceToHost, I->stream));  // one copy
        CK(cudaStreamSynchronize(I->stream));
        const double* fo = reinterpret_cast<const double*>(host.data());
        const unsigned long long* w = reinterpret_cast<const unsigned long long*>(host.data() + 2 * sizeof(double) * k);
        for (int i = 0; i < k; ++i) {
            unpack_host_bits(w + (size_t)i * I->words, I->total_bits, bits + (size_t)i * I->total_bits);
            fit[i] = fo[i];
            obj[i] = fo[k + i];
        }
    });
}

int ffsga_cuda_cellular_import(ffsga_cuda_cellular c, int k, const uint8_t* bits, const double* fit, const double* obj) {
    return guard([&] {
        NvtxRange nvtx_range("ffsga_cuda_cellular_import");
        if (!c || (k > 0 && (!bits || !fit || !obj))) fail(FFSGA_ERR_ARG, "import: null pointer");
        check_migrants(k, c->n, bits);
        if (k == 0) return;
        ffsga_cuda_instance_t* I = c->inst;
        std::lock_guard<std::mutex> lk(I->mu);
        I->use();
        const size_t bytes = packet_bytes(I, 1, k);
        std::vector<unsigned char> host(bytes);
        double* fo = reinterpret_cast<double*>(host.data());
        unsigned long long* w = reinterpret_cast<unsigned long long*>(host.data() + 2 * sizeof(double) * k);
        std::vector<unsigned long long> one;
        for (int i = 0; i < k; ++i) {
            pack_host_bits(bits + (size_t)i * I->total_bits, I->total_bits, I->words, one);
            std::copy(one.begin(), one.end(), w + (size_t)i * I->words);
            fo[i] = fit[i];
            fo[k + i] = obj[i];
        }
        DevBuf pk;
        pk.alloc(bytes);
        CK(cudaMemcpyAsync(pk.p, host.data(), bytes, cudaMemcpyHostToDevice, I->stream));
        import_into_cell(c, k, pk.as<unsigned char>());
        CK(cudaStreamSynchronize(I->stream));
    });
}

int ffsga_cuda_pseudo_import(ffsga_cuda_pseudo p, int k, const int32_t* genes, const double* fit, const double* obj) {
    return guard([&] {
        NvtxRange nvtx_range("ffsga_cuda_pseudo_import");
        if (!p || (k > 0 && (!genes || !fit || !obj))) fail(FFSGA_ERR_ARG, "import: null pointer");
        check_migrants(k, p->n, genes);
        if (k == 0) return;
        ffsga_cuda_instance_t* I = p->inst;
        std::lock_guard<std::mutex> lk(I->mu);
        I->use();
        const size_t L = (size_t)I->J * I->S;
        DevBuf gi, pk;
        gi.alloc(sizeof(int32_t) * L * k);
        pk.alloc(packet_bytes(I, 0, k));
        CK(cudaMemcpyAsync(gi.p, genes, sizeof(int32_t) * L * k, cudaMemcpyHostToDevice, I->stream));
        CK(cudaMemcpyAsync(pk.p, fit, sizeof(double) * k, cudaMemcpyHostToDevice, I->stream));
        CK(cudaMemcpyAsync(pk.as<double>() + k, obj, sizeof(double) * k, cudaMemcpyHostToDevice, I->stream));
        CK(launch_rows_from_int(I->d, gi.as<int32_t>(), nullptr, pk.as<uint8_t>() + 2 * sizeof(double) * k, k,
                                I->stream));
        g_launches += 1;
        import_into_pseudo(p, k, pk.as<unsigned char>());
        CK(cudaStreamSynchronize(I->stream));
    });
}

int ffsga_cuda_last_step_ms(ffsga_cuda_instance inst, float* ms) {
    return guard([&] {
        if (!inst || !ms) fail(FFSGA_ERR_ARG, "null pointer");
        if (!inst->step_recorded) fail(FFSGA_ERR_CONTRACT, "no step recorded");
        inst->use();
        CK(cudaEventSynchronize(inst->st1));
        CK(cudaEventElapsedTime(ms, inst->st0, inst->st1));
    });
}

int ffsga_cuda_set_timing(ffsga_cuda_instance inst, int enabled) {
    return guard([&] {
        if (!inst) fail(FFSGA_ERR_ARG, "null instance");
        inst->timing = enabled != 0;
    });
}

int ffsga_cuda_timing(ffsga_cuda_instance inst, int which, double* ms, int64_t* launches) {
    return guard([&] {
        if (!inst || which < 0 || which > 2) fail(FFSGA_ERR_ARG, "timing: bad argument");
        std::lock_guard<std::mutex> lk(inst->mu);
        inst->use();
        inst->resolve_timing();
        if (ms) *ms = inst->t_ms[which];
        if (launches) *launches = inst->t_n[which];
    });
}

int ffsga_cuda_timing_busy(ffsga_cuda_instance inst, int which, double* busy_ms) {
    return guard([&] {
        if (!inst || which < 0 || which > 2 || !busy_ms) fail(FFSGA_ERR_ARG, "timing_busy: bad argument");
        std::lock_guard<std::mutex> lk(inst->mu);
        inst->use();
        inst->resolve_timing();
        *busy_ms = inst->t_busy[which];
    });
}

int ffsga_cuda_evaluations(ffsga_cuda_instance inst, int64_t* count) {
    return guard([&] {
        if (!inst || !count) fail(FFSGA_ERR_ARG, "null pointer");
        std::lock_guard<std::mutex> lk(inst->mu);
        inst->use();
        unsigned long long v = 0;
        CK(cudaMemcpyAsync(&v, inst->eval_total.p, sizeof(v), cudaMemcpyDeviceToHost, inst->stream));
        CK(cudaStreamSynchronize(inst->stream));
        *count = (int64_t)v;
    });
}

int ffsga_cuda_reset_timing(ffsga_cuda_instance inst) {
    return guard([&] {
        if (!inst) fail(FFSGA_ERR_ARG, "null instance");
        std::lock_guard<std::mutex> lk(inst->mu);
        inst->use();
        inst->resolve_timing();
        for (int i = 0; i < 3; ++i) {
            inst->t_ms[i] = 0;
            inst->t_busy[i] = 0;
            inst->t_n[i] = 0;
        }
    });
}

int ffsga_cuda_checked_status(int reset, int64_t* status) {
    return guard([&] {
        if (!status) fail(FFSGA_ERR_ARG, "null pointer");
        CK(cudaDeviceSynchronize());
        long long v = -1;
        CK(checked_status(&v, reset != 0));
        *status = (int64_t)v;
    });
}

int ffsga_cuda_launch_count(int64_t* count) {
    return guard([&] {
        if (!count) fail(FFSGA_ERR_ARG, "null pointer");
        *count = g_launches.load();
    });
}

}  // extern "C"
