// es_runtime.cu — host runtime behind the C-ABI (include/eventscope_b200.h).
//
// One context per GPU (one process per GPU under torchrun / MPI).  A dataset
// is the rank's contiguous block of event rows, resident in HBM in the
// feature-planar layout of es_layout.h.  The EM loop per iteration is
//   em_pass (fused E + M statistics, per-CTA partials)
//   -> fixed-order block reduce -> rank exchange (NCCL all-gather over NVLink)
//   -> finalize (rank-ordered sum, M-step, Cholesky, W = L^-1, logL record)
//   -> 40-byte IterStatus read by the host (convergence / collapse decisions).
// Control semantics follow SPEC.md:291-299,319-326,335 exactly as the CPU
// oracle restates them (oracle/es_oracle.cpp), including the host PRNG
// (SplitMix64) so that Random / k-means++ init and collapse reseeds draw the
// same rows.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: NCCL is resolved at run time (see Nccl below)

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/eventscope_b200.h"
#include "es_kernels.h"

using namespace es;

namespace {

thread_local std::string g_name;
thread_local std::string g_msg;

struct Fail {
    int code;
    std::string name;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& name, const std::string& msg) { throw Fail{code, name, msg}; }
// re-raise the error a nested es_* call just recorded
[[noreturn]] void rethrow_last(int code) { throw Fail{code, g_name, g_msg}; }

void cu_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();  // clear the non-sticky last error so later checks do not re-report it
        fail(ES_ERR_RUNTIME, "CudaError", std::string(what) + ": " + cudaGetErrorString(e));
    }
}
#define CU(x) cu_check((x), #x)

// NCCL is bound lazily with dlopen instead of at link time: a process that
// already loaded a libnccl.so.2 (e.g. PyTorch's bundled 2.28) keeps using it,
// and a process that never builds a multi-GPU context never loads NCCL.
struct Nccl {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl();

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        fail(ES_ERR_RUNTIME, "NcclError", std::string(what) + ": " + nccl().GetErrorString(r));
}
#define NC(x) nccl_check((x), #x)

const Nccl& nccl() {
    static Nccl n;
    static bool loaded = false;
    if (loaded) return n;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) fail(ES_ERR_RUNTIME, "NcclError", std::string("cannot load libnccl.so.2: ") + dlerror());
    auto sym = [&](const char* name) {
        void* p = dlsym(h, name);
        if (!p) fail(ES_ERR_RUNTIME, "NcclError", std::string("missing NCCL symbol ") + name);
        return p;
    };
    n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
    n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
    n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
    n.AllGather = reinterpret_cast<decltype(n.AllGather)>(sym("ncclAllGather"));
    n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(sym("ncclAllReduce"));
    n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
    loaded = true;
    return n;
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return ES_OK;
    } catch (const Fail& e) {
        g_name = e.name;
        g_msg = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_name = "OutOfMemory";
        g_msg = "host allocation failed";
        return ES_ERR_RUNTIME;
    } catch (const std::exception& e) {
        g_name = "RuntimeError";
        g_msg = e.what();
        return ES_ERR_RUNTIME;
    }
}

// SplitMix64 — the documented host PRNG ("named, portable 64-bit
// generator"); identical draws to the oracle's.
struct SplitMix64 {
    uint64_t s;
    explicit SplitMix64(uint64_t seed) : s(seed) {}
    uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    uint64_t below(uint64_t n) { return (uint64_t)(((unsigned __int128)next() * n) >> 64); }
    double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }
};

// Growable device buffer.
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    void* get(size_t bytes) {
        if (bytes > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            CU(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
            cap = std::max<size_t>(bytes, 256);
        }
        return p;
    }
    template <class T>
    T* as(size_t count) {
        return static_cast<T*>(get(count * sizeof(T)));
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace

// ================================================================ structs
struct es_ctx {
    int device = 0, rank = 0, world = 1;
    // the parameters last uploaded and derived into `model` (model_for skips the upload, the
    // Cholesky launch and its status round trip when a call passes the same model again)
    std::vector<double> mkey;
    const double* mkey_dev = nullptr;
    int mode = 0;  // 0 single, 1 nccl, 2 host exchange
    ncclComm_t comm = nullptr;
    es_exchange ex{};
    cudaStream_t stream = nullptr;
    cudaStream_t cstream = nullptr;          // host->device copies of dataset_create (overlap the transposes)
    cudaEvent_t evc[2] = {nullptr, nullptr}, evt[2] = {nullptr, nullptr};
    int num_sms = 148;
    LaunchStats ls;
    int64_t collectives = 0;  // NCCL collectives issued (replays of captured ones included)
    std::vector<es_dataset*> live;  // datasets bound to this context (detached on destroy)
    DevBuf stage2;  // second staging buffer of dataset_create
    // the planes of the last destroyed dataset, kept for the next dataset_create of a
    // similar size (an 8.6 GB cudaMalloc / cudaFree pair per fit-on-fresh-data call is
    // ~20 ms plus a device synchronisation)
    void* plane_cache = nullptr;
    size_t plane_cache_bytes = 0;
    double* take_planes(size_t bytes) {
        if (plane_cache && plane_cache_bytes >= bytes && plane_cache_bytes <= 2 * bytes) {
            void* p = plane_cache;
            plane_cache = nullptr;
            plane_cache_bytes = 0;
            return static_cast<double*>(p);
        }
        void* p = nullptr;
        CU(cudaMalloc(&p, bytes));
        return static_cast<double*>(p);
    }
    void give_planes(void* p, size_t bytes) {
        cudaStreamSynchronize(stream);
        if (plane_cache) cudaFree(plane_cache);
        plane_cache = p;
        plane_cache_bytes = bytes;
    }
    DevBuf partial, stats_local, stats_all, model, model_backup, status, scratch, scratch2, scratch3, out_scratch,
        hist, xbuf, o1, o2, o3, o4, o5, kpp, center;
    std::vector<double> center_host;  // host copy of `center` (scoring kernels' FP64 centre)
    double center_xs = 1.0;           // power of two bringing the model's span into (8, 16]
    int precision = 0;  // 0 = mixed (FP32 whitening, FP64 statistics), 1 = strict FP64
    IterStatus* h_status = nullptr;  // pinned
    std::vector<double> hbuf;
    // optional CUDA-event timing of the hot kernels (bench.py roofline)
    bool timing = false;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    double em_ms = 0.0, score_ms = 0.0;
    int64_t em_launches = 0, score_launches = 0;
    double* t_acc = nullptr;  // measurement pending until the next stream synchronisation
    int64_t* t_cnt = nullptr;
    void t_begin() {
        if (timing) CU(cudaEventRecord(ev0, stream));
    }
    // records the end event only: the elapsed time is collected after the next sync(), so
    // timing adds no host round trip inside an EM iteration
    void t_end(double& acc, int64_t& cnt) {
        if (!timing) return;
        CU(cudaEventRecord(ev1, stream));
        t_acc = &acc;
        t_cnt = &cnt;
    }
    void t_collect() {
        if (!t_acc) return;
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, ev0, ev1));
        *t_acc += ms;
        ++*t_cnt;
        t_acc = nullptr;
    }

    void sync() {
        CU(cudaStreamSynchronize(stream));
        t_collect();
    }
    void check_launch() { CU(cudaGetLastError()); }

    // All-gather count doubles per rank (device in/out).
    void allgather(const double* d_send, double* d_recv, size_t count) {
        if (world == 1 && mode != 1) {
            if (d_send != d_recv) CU(cudaMemcpyAsync(d_recv, d_send, count * 8, cudaMemcpyDeviceToDevice, stream));
        } else if (mode == 1) {
            NC(nccl().AllGather(d_send, d_recv, count, ncclFloat64, comm, stream));
            ++collectives;
        } else {
            std::vector<double> s(count), r(count * world);
            CU(cudaMemcpyAsync(s.data(), d_send, count * 8, cudaMemcpyDeviceToHost, stream));
            sync();
            if (ex.allgather(ex.user, s.data(), r.data(), count * 8) != 0)
                fail(ES_ERR_RUNTIME, "ExchangeError", "allgather callback failed");
            CU(cudaMemcpyAsync(d_recv, r.data(), count * world * 8, cudaMemcpyHostToDevice, stream));
            sync();
        }
    }
    // In-place all-reduce on HOST memory (small control values).
    void allreduce_host(void* buf, size_t count, int dtype, int op) {
        if (world == 1 && mode != 1) return;
        if (mode == 2) {
            if (ex.allreduce(ex.user, buf, count, dtype, op) != 0)
                fail(ES_ERR_RUNTIME, "ExchangeError", "allreduce callback failed");
            return;
        }
        const size_t bytes = count * 8;
        void* d = xbuf.get(bytes);
        CU(cudaMemcpyAsync(d, buf, bytes, cudaMemcpyHostToDevice, stream));
        const ncclDataType_t t = dtype == 0 ? ncclFloat64 : ncclInt64;
        const ncclRedOp_t o = op == 0 ? ncclSum : op == 1 ? ncclMin : ncclMax;
        NC(nccl().AllReduce(d, d, count, t, o, comm, stream));
        ++collectives;
        CU(cudaMemcpyAsync(buf, d, bytes, cudaMemcpyDeviceToHost, stream));
        sync();
    }
    // Rank-ordered all-gather of host values.
    std::vector<double> allgather_host(const double* v, size_t count) {
        std::vector<double> r(count * world);
        if (world == 1 && mode != 1) {
            std::copy(v, v + count, r.begin());
            return r;
        }
        if (mode == 2) {
            if (ex.allgather(ex.user, v, r.data(), count * 8) != 0)
                fail(ES_ERR_RUNTIME, "ExchangeError", "allgather callback failed");
            return r;
        }
        double* d = xbuf.as<double>(count * (world + 1));
        CU(cudaMemcpyAsync(d, v, count * 8, cudaMemcpyHostToDevice, stream));
        NC(nccl().AllGather(d, d + count, count, ncclFloat64, comm, stream));
        ++collectives;
        CU(cudaMemcpyAsync(r.data(), d + count, count * world * 8, cudaMemcpyDeviceToHost, stream));
        sync();
        return r;
    }
};

struct es_dataset {
    es_ctx* ctx = nullptr;
    int64_t n_local = 0, n_global = 0, row_offset = 0, ld = 0;
    int D = 0;
    double* X = nullptr;
    CUtensorMap xmap{};      // TMA descriptor over X (D <= 16), see make_event_tmap
    bool has_xmap = false;
    bool owned_by_cache = false;  // planes from es_ctx::take_planes (returned there on destroy)
    ~es_dataset();
};

es_dataset::~es_dataset() {
    if (ctx) {
        auto& v = ctx->live;
        v.erase(std::remove(v.begin(), v.end(), this), v.end());
    }
    if (!X) return;
    if (owned_by_cache && ctx)
        ctx->give_planes(X, (size_t)ld * D * 8);
    else
        cudaFree(X);  // also after its context was destroyed (ctx == nullptr): no dangling cache
}

struct es_em_state {
    es_ctx* ctx = nullptr;
    es_dataset* ds = nullptr;
    int K = 0, D = 0;
    es_fit_opts opts{};
    double reg = 0.0;
    std::vector<double> S;  // data covariance (D x D)
    std::vector<double> mean;  // data mean: FP64 centre of the mixed-precision path
    double xs = 1.0;           // power of two bringing max|x - mean| into (8, 16] (k_em_mma operand scale)
    bool f32conv = false;      // max|x| <= 4 max|x - mean|: x^ may be formed on the FP32 pipe
    double min_nk = 0.0;       // min_k N_k of the current model (global), selects k_em_mma's record precision
    int last_npass = 0;        // record precision of the last k_em_mma pass (0: other kernel)
    int last_path = -1;        // EmIterPath of the last iteration
    DevBuf dcenter;
    SplitMix64 rng{0};
    std::vector<double> per_iter;
    int t = 0;          // E-steps done
    int iterations = 0; // M-steps kept
    int collapses = 0;
    bool converged = false, done = false;
    double prev = 0.0, last = 0.0;
    // the fit's own device buffers (sized once in em_begin, so the pointers a captured
    // iteration graph holds stay valid for the whole fit) and the graphs per iteration path.
    // The model has three slots: iteration t reads slot `cur` (theta_t) and writes slot
    // cur + 1; the next iteration may already be in flight (writing cur + 2) while the host
    // reads iteration t's status, and theta_t stays intact for a convergence stop.
    DevBuf model, partial, stats_local, stats_all, status, wide_ws, tick;
    size_t part_cap = 0;
    int cur = 0;
    IterRecord* h_rec = nullptr;                    // mapped pinned, one slot per model slot
    cudaEvent_t done_ev[3] = {}, tev[3][2] = {};   // iteration complete / EM-pass timing per slot
    struct Graph {
        int key;
        cudaGraphExec_t exec;
        int64_t launches;     // kernels in one replay (launch accounting)
        int64_t collectives;  // NCCL collectives in one replay
    };
    std::vector<Graph> graphs;
    ~es_em_state() {
        if (ctx) cudaStreamSynchronize(ctx->stream);
        for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
        for (int i = 0; i < 3; ++i) {
            if (done_ev[i]) cudaEventDestroy(done_ev[i]);
            for (int j = 0; j < 2; ++j)
                if (tev[i][j]) cudaEventDestroy(tev[i][j]);
        }
        if (h_rec) cudaFreeHost(h_rec);
    }
};

// ============================================================== helpers
namespace {

int64_t mstride(int K, int D) { return ModelView::size(K, D); }

// model slot i (0..2) of a fit; em_model(st) = theta_t
double* em_model(es_em_state* st, int slot) {
    const int64_t m = mstride(st->K, st->D);
    return st->model.as<double>(3 * (size_t)m) + (size_t)slot * m;
}
double* em_model(es_em_state* st) { return em_model(st, st->cur); }

void fetch_rows(es_ctx* c, es_dataset* ds, const std::vector<int64_t>& rows, std::vector<double>& out) {
    const int D = ds->D;
    const size_t m = rows.size();
    out.assign(m * D, 0.0);
    double* d = c->scratch3.as<double>(std::max<size_t>(m * D, 1));
    bool any = false;
    for (size_t r = 0; r < m; ++r) {
        const int64_t li = rows[r] - ds->row_offset;
        if (li >= 0 && li < ds->n_local) {
            launch_planar_to_rows(ds->X, ds->ld, D, li, 1, d + r * D, c->stream, c->ls);
            any = true;
        }
    }
    if (any) {
        c->check_launch();
        std::vector<double> tmp(m * D);
        CU(cudaMemcpyAsync(tmp.data(), d, m * D * 8, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        for (size_t r = 0; r < m; ++r) {
            const int64_t li = rows[r] - ds->row_offset;
            if (li >= 0 && li < ds->n_local) std::copy(&tmp[r * D], &tmp[r * D] + D, &out[r * D]);
        }
    }
    // exactly one rank owns each row: the sum is exact
    c->allreduce_host(out.data(), out.size(), 0, 0);
}

// Data statistics: mean, S (biased), min/max, non-finite.
struct DataStats {
    std::vector<double> mean, S, mn, mx;
    double nonfinite = 0;
};

DataStats data_stats(es_ctx* c, es_dataset* ds) {
    const int D = ds->D;
    DataStats r;
    double* out = c->scratch2.as<double>(4 * D);
    double* scr = c->scratch.as<double>((size_t)D * 1024 * 4);
    std::vector<double> h(4 * D, 0.0);
    if (ds->n_local > 0) {
        launch_col_stats(ds->X, ds->n_local, ds->ld, D, scr, out, c->num_sms, c->stream, c->ls);
        c->check_launch();
        CU(cudaMemcpyAsync(h.data(), out, 4 * D * 8, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
    } else {
        for (int j = 0; j < D; ++j) {
            h[D + j] = INFINITY;
            h[2 * D + j] = -INFINITY;
        }
    }
    std::vector<double> sums(2 * D);
    for (int j = 0; j < D; ++j) {
        sums[j] = h[j];
        sums[D + j] = h[3 * D + j];
    }
    r.mn.assign(h.begin() + D, h.begin() + 2 * D);
    r.mx.assign(h.begin() + 2 * D, h.begin() + 3 * D);
    // rank-ordered sum of column sums keeps the mean identical on every rank
    std::vector<double> all = c->allgather_host(sums.data(), sums.size());
    std::vector<double> tot(2 * D, 0.0);
    for (int g = 0; g < c->world; ++g)
        for (int j = 0; j < 2 * D; ++j) tot[j] += all[(size_t)g * 2 * D + j];
    c->allreduce_host(r.mn.data(), D, 0, 1);
    c->allreduce_host(r.mx.data(), D, 0, 2);
    for (int j = 0; j < D; ++j) r.nonfinite += tot[D + j];
    r.mean.resize(D);
    for (int j = 0; j < D; ++j) r.mean[j] = tot[j] / (double)ds->n_global;
    r.S.assign((size_t)D * D, 0.0);
    if (r.nonfinite > 0) return r;
    // centered second moments about the mean (one unit-weight stats pass)
    double* dmean = c->scratch2.as<double>(D);
    CU(cudaMemcpyAsync(dmean, r.mean.data(), D * 8, cudaMemcpyHostToDevice, c->stream));
    const int SK = stat_k(D);
    int nblk = 0;
    double* part = c->partial.as<double>((size_t)em_grid(64, 128, c->num_sms) * 4 * (SK + 1));
    std::vector<double> loc(SK + 1, 0.0);
    if (ds->n_local > 0) {
        launch_unit_stats(ds->X, ds->n_local, ds->ld, D, dmean, part, c->num_sms, &nblk, c->stream, c->ls);
        double* red = c->stats_local.as<double>(SK + 1);
        launch_reduce_blocks(part, nblk, SK + 1, red, c->stream, c->ls);
        c->check_launch();
        CU(cudaMemcpyAsync(loc.data(), red, (SK + 1) * 8, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
    }
    std::vector<double> allst = c->allgather_host(loc.data(), SK + 1);
    std::vector<double> st(SK + 1, 0.0);
    for (int g = 0; g < c->world; ++g)
        for (int e = 0; e <= SK; ++e) st[e] += allst[(size_t)g * (SK + 1) + e];
    const double N = (double)ds->n_global;
    const double* s1 = &st[1];
    const double* s2 = &st[1 + D];
    for (int a = 0; a < D; ++a)
        for (int b = a; b < D; ++b) {
            const double v = s2[packed_index(a, b, D)] / N - (s1[a] / N) * (s1[b] / N);
            r.S[(size_t)a * D + b] = v;
            r.S[(size_t)b * D + a] = v;
        }
    return r;
}

double default_reg(const std::vector<double>& S, int D) {
    double tr = 0.0;
    for (int d = 0; d < D; ++d) tr += S[(size_t)d * D + d];
    return 1e-6 * tr / D;
}

// Upload pi/mu/cov into the context model block and derive (Cholesky, W).
void upload_model(es_ctx* c, double* dmodel, int K, int D, const double* pi, const double* mu, const double* cov) {
    ModelView mv{K, D, dmodel};
    CU(cudaMemcpyAsync(mv.pi(), pi, K * 8, cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(mv.mu(), mu, (size_t)K * D * 8, cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(mv.cov(), cov, (size_t)K * D * D * 8, cudaMemcpyHostToDevice, c->stream));
    IterStatus* st = c->status.as<IterStatus>(1);
    CU(cudaMemsetAsync(st, 0, sizeof(IterStatus), c->stream));
    launch_derive(dmodel, D, K, st, c->stream, c->ls);
    c->check_launch();
    CU(cudaMemcpyAsync(c->h_status, st, sizeof(IterStatus), cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    if (c->h_status->not_pd)
        fail(ES_ERR_NUMERIC, "SingularCovariance", "a covariance matrix is not positive definite");
}

void check_params(const es_gmm_params* p, int D) {
    if (!p || !p->weights || !p->means || !p->covariances) fail(ES_ERR_DATA, "InvalidModel", "null parameters");
    if (p->K < 1 || p->K > 128) fail(ES_ERR_DATA, "InvalidModel", "K must be in [1,128]");
    if (p->D != D) fail(ES_ERR_DATA, "DimensionMismatch", "model dimension does not match the data");
    for (int k = 0; k < p->K; ++k)
        if (!(p->weights[k] >= 0.0) || !std::isfinite(p->weights[k]))
            fail(ES_ERR_DATA, "InvalidModel", "weights must be finite and non-negative");
}

double* model_for(es_ctx* c, const es_gmm_params* p, int D) {
    check_params(p, D);
    double* m = c->model.as<double>(mstride(p->K, D));
    const size_t K = (size_t)p->K;
    std::vector<double> key;
    key.reserve(2 + K + K * D + K * D * D);
    key.push_back((double)p->K);
    key.push_back((double)D);
    key.insert(key.end(), p->weights, p->weights + K);
    key.insert(key.end(), p->means, p->means + K * D);
    key.insert(key.end(), p->covariances, p->covariances + K * D * D);
    if (c->mkey_dev == m && key.size() == c->mkey.size() &&
        std::memcmp(key.data(), c->mkey.data(), key.size() * sizeof(double)) == 0)
        return m;  // derived model, centre and scale on the device are those of these parameters
    c->mkey_dev = nullptr;
    upload_model(c, m, p->K, D, p->weights, p->means, p->covariances);
    // FP64 centre for the mixed-precision scorer: the model's mean sum_k pi_k mu_k
    std::vector<double> cen(D, 0.0);
    double z = 0.0;
    for (int k = 0; k < p->K; ++k) z += p->weights[k];
    for (int k = 0; k < p->K; ++k)
        for (int j = 0; j < D; ++j) cen[j] += (z > 0 ? p->weights[k] / z : 1.0 / p->K) * p->means[(size_t)k * D + j];
    double* dc = c->center.as<double>(D);
    CU(cudaMemcpyAsync(dc, cen.data(), D * 8, cudaMemcpyHostToDevice, c->stream));
    // x^ = (x - c) xs for the tcgen05 scorer: the model's span (means +- 8 sigma) maps into
    // (8, 16]; events further out are refined entirely in FP64 by the kernel
    double span = 0.0;
    for (int k = 0; k < p->K; ++k)
        for (int j = 0; j < D; ++j)
            span = std::max(span, std::fabs(p->means[(size_t)k * D + j] - cen[j]) +
                                      8.0 * std::sqrt(std::max(p->covariances[(size_t)k * D * D + j * D + j], 0.0)));
    c->center_host = cen;
    c->center_xs = span > 0.0 && std::isfinite(span) ? std::ldexp(1.0, 4 - (int)std::ceil(std::log2(span))) : 1.0;
    c->mkey.swap(key);
    c->mkey_dev = m;
    return m;
}

// Output staging: device pointers are written directly, host pointers via scratch.
template <class T>
struct Out {
    T* user;
    T* dev;
    size_t count;
    DevBuf* buf;
    Out(T* u, size_t n, DevBuf& b) : user(u), dev(nullptr), count(n), buf(&b) {
        if (!u) return;
        if (is_device_ptr(u)) dev = u;
        else dev = b.as<T>(std::max<size_t>(n, 1));
    }
    void finish(cudaStream_t s) {
        if (user && dev != user && count) CU(cudaMemcpyAsync(user, dev, count * sizeof(T), cudaMemcpyDeviceToHost, s));
    }
};

// Scoring launch: mixed-precision kernel when supported, FP64 team kernel otherwise.
void score_launch(es_ctx* c, const double* X, int64_t n, int64_t ld, int D, int K, const double* dmodel,
                  const double* center, const double* center_host, double xs, const ScoreOut& o, double* bs,
                  int* nblk, const CUtensorMap* xmap = nullptr) {
    // mixture mode decides on ll itself: flags and calibration keys at the
    // threshold then need ll to FP64 accuracy, so that ablation scores on the strict kernel
    if (o.mode == 1)
        launch_score(X, n, ld, D, K, dmodel, o, bs, c->num_sms, nblk, c->stream, c->ls);
    else if (c->precision == 0 && center && center_host && xmap && score_mma_enabled(D, K, o))
        launch_score_mma(xmap, n, D, K, dmodel, center, center_host, xs, o, bs, c->num_sms, nblk, c->stream,
                         c->ls);
    else
        launch_score(X, n, ld, D, K, dmodel, o, bs, c->num_sms, nblk, c->stream, c->ls);
}

size_t score_blocks(es_ctx* c, int D, int K) { return (size_t)2 * std::max(score_grid(D, K, c->num_sms), 2 * c->num_sms) + 2; }

double run_score(es_ctx* c, es_dataset* ds, const double* dmodel, int K, ScoreOut o, const double* center,
                 const double* center_host, double xs, bool need_total = true) {
    const int D = ds->D;
    double* bs = c->scratch.as<double>(score_blocks(c, D, K));
    double loc = 0.0;
    if (ds->n_local > 0) {
        int nblk = 0;
        c->t_begin();
        score_launch(c, ds->X, ds->n_local, ds->ld, D, K, dmodel, center, center_host, xs, o, bs, &nblk,
                     ds->has_xmap ? &ds->xmap : nullptr);
        c->t_end(c->score_ms, c->score_launches);
        if (!need_total) return 0.0;
        double* red = c->scratch2.as<double>(2);
        launch_reduce_blocks(bs, nblk, 2, red, c->stream, c->ls);
        c->check_launch();
        double h[2];
        CU(cudaMemcpyAsync(h, red, 16, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        loc = h[0];
    }
    if (!need_total) return 0.0;  // every rank (empty shards too): no exchange skipped on one rank only
    std::vector<double> all = c->allgather_host(&loc, 1);
    double tot = 0.0;
    for (double v : all) tot += v;
    return tot;
}

// Exact order statistic (global rank r) of FP64 keys by 8-bit radix select.
double radix_select(es_ctx* c, const double* dkeys, int64_t n, int64_t r) {
    unsigned long long* hist = c->hist.as<unsigned long long>(256);
    uint64_t prefix = 0, mask = 0;
    std::vector<long long> h(256);
    for (int pass = 0; pass < 8; ++pass) {
        const int shift = 56 - 8 * pass;
        launch_hist8(dkeys, n, shift, mask, prefix, hist, c->num_sms, c->stream, c->ls);
        c->check_launch();
        CU(cudaMemcpyAsync(h.data(), hist, 256 * 8, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        c->allreduce_host(h.data(), 256, 1, 0);
        long long cum = 0;
        int digit = 255;
        for (int b = 0; b < 256; ++b) {
            if (cum + h[b] > r) {
                digit = b;
                break;
            }
            cum += h[b];
        }
        r -= cum;
        prefix |= (uint64_t)digit << shift;
        mask |= (uint64_t)0xFF << shift;
    }
    const uint64_t u = (prefix >> 63) ? (prefix & 0x7FFFFFFFFFFFFFFFull) : ~prefix;
    double v;
    std::memcpy(&v, &u, 8);
    return v;
}

// ---------------------------------------------------------------- EM core
bool is_diag(const es_em_state* st) { return st->opts.covariance_type == ES_COV_DIAG; }

// k-means++ seeding on the device: first centre uniform; then D^2-weighted
// draws, cumulative sum over global rows in chunk order (4096-row chunks).  Shared by
// fit_em's KMeansPP init and the k-means baseline.
std::vector<int64_t> kmeanspp_device(es_ctx* c, es_dataset* ds, int K, SplitMix64& rng) {
    const int D = ds->D;
    std::vector<int64_t> rows;
    // k-means++ (DESIGN.md): first centre uniform; then D^2-weighted draws,
    // cumulative sum over global rows in chunk order (4096-row chunks).
    rows.push_back((int64_t)rng.below((uint64_t)ds->n_global));
    const int64_t CH = 4096;
    const int64_t nlc = (ds->n_local + CH - 1) / CH;
    double* d2 = c->kpp.as<double>(std::max<int64_t>(ds->n_local, 1) + nlc + 8);
    double* parts = d2 + std::max<int64_t>(ds->n_local, 1);
    double* dcen = c->scratch2.as<double>(D);
    std::vector<double> cen;
    for (int j = 1; j < K; ++j) {
        fetch_rows(c, ds, {rows.back()}, cen);
        CU(cudaMemcpyAsync(dcen, cen.data(), D * 8, cudaMemcpyHostToDevice, c->stream));
        launch_kpp_update(ds->X, ds->n_local, ds->ld, D, dcen, d2, parts, j == 1, c->stream, c->ls);
        c->check_launch();
        std::vector<double> hp(nlc);
        if (nlc) CU(cudaMemcpyAsync(hp.data(), parts, nlc * 8, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        double loc = 0.0;
        for (double v : hp) loc += v;
        std::vector<double> all = c->allgather_host(&loc, 1);
        double total = 0.0;
        for (double v : all) total += v;
        const double u = rng.uniform() * total;
        int64_t pick = -1;
        if (total > 0.0) {
            // owner rank of the crossing point locates the row; others report -1
            double before = 0.0;
            for (int g = 0; g < c->rank; ++g) before += all[g];
            double found = -1.0;
            if (u >= before && u < before + all[c->rank]) {
                double acc = before;
                int64_t ch = 0;
                for (; ch < nlc; ++ch) {
                    if (acc + hp[ch] > u) break;
                    acc += hp[ch];
                }
                if (ch == nlc) ch = nlc - 1;
                const int64_t r0 = ch * CH, nr = std::min(CH, ds->n_local - r0);
                std::vector<double> seg(nr);
                CU(cudaMemcpyAsync(seg.data(), d2 + r0, nr * 8, cudaMemcpyDeviceToHost, c->stream));
                c->sync();
                int64_t li = r0 + nr - 1;
                for (int64_t q = 0; q < nr; ++q) {
                    acc += seg[q];
                    if (acc > u) {
                        li = r0 + q;
                        break;
                    }
                }
                found = (double)(ds->row_offset + li);
            }
            c->allreduce_host(&found, 1, 0, 2);
            pick = (int64_t)found;
        }
        if (pick < 0) pick = (int64_t)rng.below((uint64_t)ds->n_global);
        rows.push_back(pick);
    }
    return rows;
}

void em_init_model(es_em_state* st, const es_gmm_params* init, const DataStats& dsx) {
    es_ctx* c = st->ctx;
    es_dataset* ds = st->ds;
    const int K = st->K, D = st->D;
    std::vector<double> pi(K), mu((size_t)K * D), cov((size_t)K * D * D);
    if (st->opts.init == ES_INIT_GIVEN) {
        check_params(init, D);
        if (init->K != K) fail(ES_ERR_DATA, "DimensionMismatch", "init K differs from requested K");
        std::copy(init->weights, init->weights + K, pi.begin());
        std::copy(init->means, init->means + (size_t)K * D, mu.begin());
        std::copy(init->covariances, init->covariances + (size_t)K * D * D, cov.begin());
    } else {
        std::vector<int64_t> rows;
        if (st->opts.init == ES_INIT_KMEANSPP) {
            rows = kmeanspp_device(c, ds, K, st->rng);
        } else {
            while ((int)rows.size() < K) {
                const int64_t r = (int64_t)st->rng.below((uint64_t)ds->n_global);
                if (std::find(rows.begin(), rows.end(), r) == rows.end()) rows.push_back(r);
            }
        }
        std::vector<double> X0;
        fetch_rows(c, ds, rows, X0);
        for (int k = 0; k < K; ++k) {
            pi[k] = 1.0 / K;
            std::copy(&X0[(size_t)k * D], &X0[(size_t)k * D] + D, &mu[(size_t)k * D]);
            for (int a = 0; a < D; ++a)
                for (int b = 0; b < D; ++b)
                    cov[(size_t)k * D * D + a * D + b] =
                        (is_diag(st) && a != b) ? 0.0 : dsx.S[(size_t)a * D + b] + (a == b ? st->reg : 0.0);
        }
    }
    double* m = em_model(st);
    upload_model(c, m, K, D, pi.data(), mu.data(), cov.data());
    st->min_nk = (double)ds->n_global * *std::min_element(pi.begin(), pi.end());
}

void em_begin(es_em_state* st, const es_gmm_params* init) {
    es_ctx* c = st->ctx;
    es_dataset* ds = st->ds;
    const int K = st->K, D = st->D;
    if (K < 1 || ds->n_global < K) fail(ES_ERR_DATA, "TooFewPoints", "fit_em requires N >= K >= 1");
    if (K > 128) fail(ES_ERR_DATA, "InvalidModel", "K must be <= 128");
    if (st->opts.max_iter < 0) fail(ES_ERR_DATA, "RangeViolation", "max_iter must be >= 0");
    if (st->opts.covariance_type != ES_COV_FULL && st->opts.covariance_type != ES_COV_DIAG)
        fail(ES_ERR_DATA, "RangeViolation", "covariance_type must be ES_COV_FULL or ES_COV_DIAG");
    if (st->opts.covariance_type == ES_COV_DIAG && (K > 32 || D > 32))
        fail(ES_ERR_DATA, "Unsupported", "diagonal covariance supports K <= 32, D <= 32");
    DataStats dsx = data_stats(c, ds);
    if (dsx.nonfinite > 0) fail(ES_ERR_DATA, "NonFiniteInput", "X contains non-finite entries");
    if (K > 1) {
        bool deg = true;
        for (int j = 0; j < D; ++j)
            if (dsx.mn[j] != dsx.mx[j]) deg = false;
        if (deg) fail(ES_ERR_DATA, "DegenerateData", "all points identical and K > 1");
    }
    st->S = dsx.S;
    st->mean = dsx.mean;
    {
        double span = 0.0, mag = 0.0;
        for (int j = 0; j < D; ++j) {
            span = std::max(span, std::max(dsx.mx[j] - dsx.mean[j], dsx.mean[j] - dsx.mn[j]));
            mag = std::max(mag, std::max(std::fabs(dsx.mx[j]), std::fabs(dsx.mn[j])));
        }
        st->xs = span > 0.0 ? std::ldexp(1.0, 4 - (int)std::ceil(std::log2(span))) : 1.0;
        st->f32conv = span > 0.0 && mag <= 4.0 * span && mag < 1e30;
    }
    CU(cudaMemcpyAsync(st->dcenter.as<double>(D), dsx.mean.data(), D * 8, cudaMemcpyHostToDevice, c->stream));
    {  // the fit's buffers at their final sizes (every iteration path), allocated once
        const int NE1 = stat_total(D, K);
        st->part_cap = (size_t)std::max(em_grid(D, K, c->num_sms), 2 * c->num_sms) * NE1;
        st->partial.as<double>(st->part_cap);
        st->stats_local.as<double>(NE1);
        st->stats_all.as<double>((size_t)NE1 * c->world);
        CU(cudaMemsetAsync(st->tick.as<int>(K), 0, K * sizeof(int), c->stream));
        em_model(st, 0);
        if (!st->h_rec) CU(cudaHostAlloc(&st->h_rec, 3 * sizeof(IterRecord), cudaHostAllocMapped));
        for (int i = 0; i < 3; ++i) {
            if (!st->done_ev[i]) CU(cudaEventCreateWithFlags(&st->done_ev[i], cudaEventDisableTiming));
            for (int j = 0; j < 2; ++j)
                if (!st->tev[i][j]) CU(cudaEventCreate(&st->tev[i][j]));
        }
    }
    st->reg = st->opts.reg < 0 ? default_reg(dsx.S, D) : st->opts.reg;
    st->rng = SplitMix64(st->opts.seed);
    em_init_model(st, init, dsx);
}

// The mixed-precision EM passes (tcgen05 E-step) need enough events per component for
// the per-event rounding of the whitening to average out: below
// kMixedMinNk events in some component the iteration runs on the strict FP64 kernel.
bool mixed_em(es_ctx* c, const es_em_state* st) {
    return c->precision == 0 && em_mixed_supported(st->D, st->K) && st->min_nk >= kMixedMinNk;
}

// logL of the current model from one fused tcgen05 E+M pass (statistics discarded): the
// same FP32 log-sum-exp per event as every per-iteration logL, half the cost of the
// refined scorer; used for final_log_likelihood on the mixed path.
bool em_logl_pass(es_em_state* st, double* out) {
    es_ctx* c = st->ctx;
    es_dataset* ds = st->ds;
    const int K = st->K, D = st->D;
    if (is_diag(st) || !mixed_em(c, st) || !em_mma_enabled() || !ds->has_xmap) return false;
    const int NE1 = stat_total(D, K);
    double* dmodel = em_model(st);
    double* loc = st->stats_local.as<double>(NE1);
    if (ds->n_local > 0) {
        int nblk = 0;
        double* part = st->partial.as<double>(st->part_cap);
        const int np = st->min_nk >= kOnePassMinNk ? 1 : 2;
        launch_em_mma(&ds->xmap, ds->n_local, D, K, dmodel, st->dcenter.as<double>(D), st->mean.data(), st->xs,
                      st->f32conv, np, part, c->num_sms, &nblk, c->stream, c->ls);
        launch_reduce_blocks(part, nblk, NE1, loc, c->stream, c->ls);
        c->check_launch();
    } else {
        CU(cudaMemsetAsync(loc, 0, NE1 * 8, c->stream));
    }
    double ll = 0.0;
    CU(cudaMemcpyAsync(&ll, loc + (NE1 - 1), 8, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    const std::vector<double> all = c->allgather_host(&ll, 1);  // rank-ordered sum
    double tot = 0.0;
    for (double v : all) tot += v;
    *out = tot;
    return true;
}

// Iteration paths (the EM pass kernel and its statistics format).
enum EmIterPath {
    kPathEmpty = 0,
    kPathDiag,
    kPathStrict,
    kPathMma1,
    kPathMma2,
    kPathDiagMixed,
    kPathFullMixed,
    kPathWide,   // k_em_wide, one fp16 record per value
    kPathWide2,  // k_em_wide, fp16 hi + lo records
    kPathDiagTc  // k_em_diag_tc (diagonal, tcgen05 E-step quadratic form + M-step moments)
};

// ES_EM_WIDE=0 keeps the FP32 k_em_full_mixed pass where the wide tensor-core pass applies;
// ES_EM_WIDE=3 (diagnostics) also takes k_em_mma's shapes.  (Read per iteration, so a test
// can switch it within one process.)
int em_wide_mode() {
    const char* e = getenv("ES_EM_WIDE");
    return (e && e[0] == '0') ? 0 : (e && e[0] == '3') ? 3 : 1;
}

// Record precision of a k_em_wide iteration: one fp16 record per value once every component
// held >= kOnePassMinNk events in the previous M-step; hi + lo records otherwise, and in the
// first iteration (the initial weights are not event counts).  ES_EM_MMA_PASSES forces it.
int wide_path(const es_em_state* st) {
    int np = em_mma_passes();
    if (!np) np = (st->t > 0 && st->min_nk >= kOnePassMinNk) ? 1 : 2;
    return np == 1 ? kPathWide : kPathWide2;
}

// Full covariances outside the tensor-core pass's shapes: the FP32 k_em_full_mixed pass once
// every component holds >= kMixedMinNk events (as the tensor-core pass), strict FP64 below.
bool mixed_full(const es_ctx* c, const es_em_state* st) {
    return c->precision == 0 && !em_mixed_supported(st->D, st->K) && em_full_mixed_supported(st->D, st->K) &&
           st->min_nk >= kMixedMinNk && em_mma_enabled();
}

// The mixed diagonal pass needs >= kOnePassMinNk events in every component (its per-event FP32
// rounding averages out there), the strict FP64 team kernel otherwise.
bool mixed_diag(const es_ctx* c, const es_em_state* st) {
    return c->precision == 0 && em_diag_mixed_supported(st->D, st->K) && st->min_nk >= kOnePassMinNk;
}

int em_choose_path(const es_em_state* st) {
    es_ctx* c = st->ctx;
    const es_dataset* ds = st->ds;
    if (ds->n_local == 0) return kPathEmpty;
    if (is_diag(st)) {
        if (em_diag_tc_mode() == 2 && c->precision == 0 && em_diag_tc_enabled(st->D, st->K) &&
            st->min_nk >= kMixedMinNk)
            return kPathDiagTc;
        return mixed_diag(c, st) ? (em_diag_tc_enabled(st->D, st->K) ? kPathDiagTc : kPathDiagMixed) : kPathDiag;
    }
    if (em_wide_mode() == 3 && c->precision == 0 && em_wide_supported(st->D, st->K) && st->min_nk >= kMixedMinNk)
        return wide_path(st);
    if (mixed_em(c, st) && em_mma_enabled() && ds->has_xmap) {
        // one fp16 record per value once every component held >= 2^20 events in the previous
        // M-step; hi + lo records otherwise and in the first iteration (the initial weights are
        // not event counts: the bench trajectory's first E-step leaves a component 225k events)
        const int np = em_mma_passes() ? em_mma_passes() : ((st->t > 0 && st->min_nk >= kOnePassMinNk) ? 1 : 2);
        return np == 1 ? kPathMma1 : kPathMma2;
    }
    if (mixed_full(c, st)) {
        if (em_wide_mode() && em_wide_supported(st->D, st->K)) return wide_path(st);
        return kPathFullMixed;
    }
    return kPathStrict;
}

// Enqueues one EM iteration on the context stream, no host synchronisation:
//   EM pass (fused E + M statistics, per-CTA partials) -> fixed-order block reduce ->
//   rank exchange (NCCL all-gather; skipped on one rank) -> k_finalize (rank-ordered sum,
//   M-step, Cholesky, W = L^-1, collapse flags, logL) -> 40-byte IterStatus to pinned host.
// The EM pass of an iteration path: launches it and returns the statistics format for
// k_finalize (*nblk = partial blocks written).
int em_pass_launch(es_em_state* st, int path, int slot, int* nblk) {
    es_ctx* c = st->ctx;
    es_dataset* ds = st->ds;
    const int K = st->K, D = st->D;
    double* dmodel = em_model(st, slot);
    double* part = st->partial.as<double>(st->part_cap);
    *nblk = 0;
    switch (path) {
        case kPathDiag:
            launch_em_diag(ds->X, ds->n_local, ds->ld, D, K, dmodel, part, c->num_sms, nblk, c->stream, c->ls);
            return 2;
        case kPathFullMixed:
            launch_em_full_mixed(ds->X, ds->n_local, ds->ld, D, K, dmodel, st->dcenter.as<double>(D), st->xs, part,
                                 c->num_sms, nblk, c->stream, c->ls);
            return 3;
        case kPathDiagMixed:
            launch_em_diag_mixed(ds->X, ds->n_local, ds->ld, D, K, dmodel, st->dcenter.as<double>(D), part,
                                 c->num_sms, nblk, c->stream, c->ls);
            return 4;
        case kPathDiagTc:
            launch_em_diag_tc(&ds->xmap, ds->n_local, D, K, dmodel, st->dcenter.as<double>(D), st->mean.data(), st->xs,
                              part, c->num_sms, nblk, c->stream, c->ls);
            return 2;
        case kPathWide:
        case kPathWide2:
            launch_em_wide(ds->X, ds->n_local, ds->ld, D, K, dmodel, st->dcenter.as<double>(D), st->mean.data(),
                           st->xs, st->f32conv, path == kPathWide ? 1 : 2, st->wide_ws.get(em_wide_workspace_bytes()),
                           part, c->num_sms, nblk, c->stream, c->ls);
            return 3;
        case kPathMma1:
        case kPathMma2:
            launch_em_mma(&ds->xmap, ds->n_local, D, K, dmodel, st->dcenter.as<double>(D), st->mean.data(), st->xs,
                          st->f32conv, path == kPathMma1 ? 1 : 2, part, c->num_sms, nblk, c->stream, c->ls);
            return 3;
        case kPathStrict: {
            bool wh = true;
            launch_em_pass(ds->X, ds->n_local, ds->ld, D, K, dmodel, part, c->num_sms, nblk, &wh, c->stream, c->ls);
            return wh ? 1 : 0;
        }
        default:  // an empty shard announces the statistics format the other ranks use
            if (is_diag(st)) return (mixed_diag(c, st) && !em_diag_tc_enabled(st->D, st->K)) ? 4 : 2;
            if ((mixed_em(c, st) && em_mma_enabled()) || mixed_full(c, st)) return 3;
            return em_path(D, K) != EmPath::Generic ? 1 : 0;
    }
}

// Everything of an iteration after the EM pass: fixed-order block reduce -> rank exchange
// (NCCL all-gather; skipped on one rank) -> k_finalize (rank-ordered sum, M-step, Cholesky,
// W = L^-1, collapse flags, logL) -> 40-byte IterStatus to pinned host memory.  On one rank
// without NCCL, k_finalize reduces the per-CTA partials itself (same fixed order).
// Model slot `slot` -> slot + 1 (mod 3), status slot `slot`.
void em_tail_launch(es_em_state* st, int path, int slot, int nblk, int whitened) {
    es_ctx* c = st->ctx;
    es_dataset* ds = st->ds;
    const int K = st->K, D = st->D;
    const int NE1 = stat_total(D, K);
    double* part = st->partial.as<double>(st->part_cap);
    double* loc = st->stats_local.as<double>(NE1);
    const double* all = loc;
    int G = c->world;
    if (c->world == 1 && c->mode != 1 && path != kPathEmpty) {
        all = part;
        G = -nblk;
    } else {
        if (path != kPathEmpty)
            launch_reduce_blocks(part, nblk, NE1, loc, c->stream, c->ls);
        else
            CU(cudaMemsetAsync(loc, 0, NE1 * 8, c->stream));
        if (c->world > 1 || c->mode == 1) {
            double* ag = st->stats_all.as<double>((size_t)NE1 * c->world);
            c->allgather(loc, ag, NE1);
            all = ag;
        }
    }
    IterRecord* dst = nullptr;  // the slot's record in mapped host memory (device view)
    CU(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dst), st->h_rec + slot, 0));
    launch_finalize(all, G, D, K, ds->n_global, st->reg, whitened, em_model(st, slot), em_model(st, (slot + 1) % 3),
                    dst, nullptr, st->t, c->stream, c->ls, st->dcenter.as<double>(D), st->xs, loc, st->tick.as<int>(K));
    c->check_launch();
}

// Captures whatever `enqueue` puts on the context stream as a graph (launch and collective
// accounting per replay).
template <class F>
es_em_state::Graph capture_graph(es_ctx* c, int key, F&& enqueue) {
    cudaGraph_t graph = nullptr;
    const int64_t l0 = c->ls.launches, n0 = c->collectives;
    CU(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed));
    try {
        enqueue();
    } catch (...) {
        cudaStreamEndCapture(c->stream, &graph);
        if (graph) cudaGraphDestroy(graph);
        c->ls.launches = l0;
        c->collectives = n0;
        throw;
    }
    CU(cudaStreamEndCapture(c->stream, &graph));
    cudaGraphExec_t ex = nullptr;
    const cudaError_t e = cudaGraphInstantiate(&ex, graph, 0);
    cudaGraphDestroy(graph);
    CU(e);
    es_em_state::Graph g{key, ex, c->ls.launches - l0, c->collectives - n0};
    c->ls.launches = l0;
    c->collectives = n0;
    return g;
}

// ES_GRAPH=0 disables the per-path CUDA graph of the iteration (default on; never in the
// host-exchange mode, whose all-gather is a host callback).
bool graphs_enabled(const es_ctx* c) {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("ES_GRAPH");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1 && c->mode != 2;
}

// Enqueues one EM iteration on model slot `slot` (-> slot + 1, status slot `slot`) as graph
// replays (or the same sequence launched directly), then the slot's completion event; no
// host synchronisation.  Timing mode brackets the EM pass with the slot's timing events
// (the pass and the tail are separate graphs then), so the pass is timed live.
void em_enqueue(es_em_state* st, int path, int slot) {
    es_ctx* c = st->ctx;
    const bool timed = c->timing && path != kPathEmpty;
    st->last_npass = (path == kPathMma1 || path == kPathWide) ? 1 : (path == kPathMma2 || path == kPathWide2) ? 2 : 0;
    st->last_path = path;
    if (!graphs_enabled(c)) {
        int nblk = 0;
        if (timed) CU(cudaEventRecord(st->tev[slot][0], c->stream));
        const int wh = em_pass_launch(st, path, slot, &nblk);
        if (timed) CU(cudaEventRecord(st->tev[slot][1], c->stream));
        em_tail_launch(st, path, slot, nblk, wh);
    } else {
        auto find = [&](int key) -> es_em_state::Graph* {
            for (auto& x : st->graphs)
                if (x.key == key) return &x;
            return nullptr;
        };
        auto replay = [&](es_em_state::Graph* g) {
            CU(cudaGraphLaunch(g->exec, c->stream));
            c->ls.launches += g->launches;
            c->collectives += g->collectives;
        };
        // one graph per (path, slot, timing): timing mode records the slot's events inside it
        const int key = 2 * (3 * path + slot) + (timed ? 1 : 0);
        es_em_state::Graph* g = find(key);
        if (!g) {
            st->graphs.push_back(capture_graph(c, key, [&] {
                int nblk = 0;  // (external event-record nodes: the events are real, timed records)
                if (timed) CU(cudaEventRecordWithFlags(st->tev[slot][0], c->stream, cudaEventRecordExternal));
                const int wh = em_pass_launch(st, path, slot, &nblk);
                if (timed) CU(cudaEventRecordWithFlags(st->tev[slot][1], c->stream, cudaEventRecordExternal));
                em_tail_launch(st, path, slot, nblk, wh);
            }));
            g = &st->graphs.back();
        }
        replay(g);
    }
    CU(cudaEventRecord(st->done_ev[slot], c->stream));
}

// Waits for the iteration on `slot` and returns its status (timing mode: adds its EM pass time).
IterStatus em_wait(es_em_state* st, int slot, int path) {
    es_ctx* c = st->ctx;
    CU(cudaEventSynchronize(st->done_ev[slot]));
    if (c->timing && path != kPathEmpty) {
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, st->tev[slot][0], st->tev[slot][1]));
        c->em_ms += ms;
        ++c->em_launches;
    }
    // the host view of the slot's IterRecord -> IterStatus (min N_k, collapse mask, not-PD count)
    const volatile IterRecord* r = st->h_rec + slot;
    IterStatus s{};
    s.logL = r->logL;
    double mn = INFINITY;
    for (int k = 0; k < st->K; ++k) {
        const double nk = r->nk[k];
        const int32_t f = r->flags[k];
        if (nk >= 0.0) mn = std::min(mn, nk);
        if (f & 1) {
            if (k < 64) s.collapse_lo |= 1ull << k;
            else s.collapse_hi |= 1ull << (k - 64);
        }
        if (f & 2) ++s.not_pd;
    }
    if (mn < INFINITY) s.min_nk_inv = ~(unsigned long long)__builtin_bit_cast(uint64_t, mn);
    return s;
}

// Whether iteration t's status asks for more than recording its logL: a convergence stop,
// an error, or a collapse reseed (each needs the host to act on the model it produced).
bool em_needs_host(const es_em_state* st, const IterStatus& s) {
    if (s.not_pd || s.collapse_lo || s.collapse_hi) return true;
    return st->opts.tol > 0.0 && st->t >= 1 && std::fabs(s.logL - st->prev) < st->opts.tol * (1.0 + std::fabs(s.logL));
}

// Host side of iteration t, whose EM pass used model slot `slot` (theta_t) and whose M-step
// wrote slot + 1: records logL, stops on convergence (theta_t is returned: slot stays
// current), raises SingularCovariance, reseeds collapsed components in
// the new model.  Nothing may be in flight on the stream when this acts on the model.
// Returns true when the loop must stop.
bool em_after(es_em_state* st, const IterStatus& s, int slot) {
    es_ctx* c = st->ctx;
    es_dataset* ds = st->ds;
    const int K = st->K, D = st->D;
    const double cur = s.logL;
    if (s.min_nk_inv) st->min_nk = __builtin_bit_cast(double, ~(unsigned long long)s.min_nk_inv);
    st->per_iter.push_back(cur);
    st->last = cur;
    const int t = st->t++;
    if (st->opts.tol > 0.0 && t >= 1 && std::fabs(cur - st->prev) < st->opts.tol * (1.0 + std::fabs(cur))) {
        st->converged = true;  // theta_t (before this M-step) is returned, final logL = logL_t
        return true;
    }
    st->prev = cur;
    st->cur = (slot + 1) % 3;
    if (s.not_pd) fail(ES_ERR_NUMERIC, "SingularCovariance", "updated covariance is not positive definite");
    if (s.collapse_lo || s.collapse_hi) {
        // reseed mean at a uniform data row, covariance to the
        // data covariance (+reg), weight 1/K then renormalise; at most twice.
        double* dmodel = em_model(st);
        ModelView mv{K, D, dmodel};
        std::vector<double> pi(K), mu((size_t)K * D), cov((size_t)K * D * D);
        CU(cudaMemcpyAsync(pi.data(), mv.pi(), K * 8, cudaMemcpyDeviceToHost, c->stream));
        CU(cudaMemcpyAsync(mu.data(), mv.mu(), (size_t)K * D * 8, cudaMemcpyDeviceToHost, c->stream));
        CU(cudaMemcpyAsync(cov.data(), mv.cov(), (size_t)K * D * D * 8, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        for (int k = 0; k < K; ++k) {
            const bool col = k < 64 ? ((s.collapse_lo >> k) & 1) : ((s.collapse_hi >> (k - 64)) & 1);
            if (!col) continue;
            if (++st->collapses > 2) fail(ES_ERR_NUMERIC, "RepeatedCollapse", "component collapsed more than twice");
            st->min_nk = 0.0;  // a reseeded component: two-pass records next iteration
            const int64_t r = (int64_t)st->rng.below((uint64_t)ds->n_global);
            std::vector<double> row;
            fetch_rows(c, ds, {r}, row);
            std::copy(row.begin(), row.end(), &mu[(size_t)k * D]);
            for (int a = 0; a < D; ++a)
                for (int b = 0; b < D; ++b)
                    cov[(size_t)k * D * D + a * D + b] =
                        (is_diag(st) && a != b) ? 0.0 : st->S[(size_t)a * D + b] + (a == b ? st->reg : 0.0);
            pi[k] = 1.0 / K;
        }
        double z = 0.0;
        for (int k = 0; k < K; ++k) z += pi[k];
        for (int k = 0; k < K; ++k) pi[k] /= z;
        upload_model(c, dmodel, K, D, pi.data(), mu.data(), cov.data());
    }
    st->iterations = t + 1;
    return false;
}

// ES_EM_DEBUG=1: one stderr line per EM iteration (path, min N_k, speculation kept)
bool em_debug() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("ES_EM_DEBUG");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

// ES_EM_SPEC=0 disables enqueueing iteration t + 1 before iteration t's status is read
// (never in the host-exchange mode, whose all-gather is a synchronous host callback).
bool spec_enabled(const es_ctx* c) {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("ES_EM_SPEC");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1 && c->mode != 2;
}

// Whether the path of the next iteration is predictable from the current min N_k: the path
// depends on min N_k only through thresholds (kMixedMinNk, kOnePassMinNk), and min N_k moves
// by up to ~35% per iteration early in a fit.  Near a threshold (within 1.5x) the next
// iteration is not enqueued speculatively: a mispredicted one is a whole discarded EM pass,
// an unspeculated one costs the status round trip (~40 us).
bool path_settled(es_em_state* st, int path) {
    const double m = st->min_nk;
    ++st->t;  // the next iteration's path (k_em_wide keeps hi + lo records at t = 0)
    st->min_nk = m / 1.5;
    const int lo = em_choose_path(st);
    st->min_nk = m * 1.5;
    const int hi = em_choose_path(st);
    st->min_nk = m;
    --st->t;
    return lo == path && hi == path;
}

// Up to n_iter EM iterations.  Iteration t + 1 is enqueued (on the predicted path: the
// path only changes with min N_k) before the host waits for iteration t, so the GPU never
// idles on the host's status read; when iteration t's status needs the host (convergence,
// an error, a collapse reseed) or changes the path, the speculative iteration is drained and
// discarded (it wrote only model slot t + 2 and status slot t + 1) and re-enqueued.
void em_steps(es_em_state* st, int n_iter) {
    es_ctx* c = st->ctx;
    int pend = -1;  // path of the iteration already enqueued for t = st->t on slot st->cur
    for (int i = 0; i < n_iter && !st->done; ++i) {
        if (st->t >= st->opts.max_iter) {
            st->done = true;
            break;
        }
        const int slot = st->cur;
        if (pend < 0) {
            pend = em_choose_path(st);
            em_enqueue(st, pend, slot);
        }
        const int path = pend;
        const bool spec = spec_enabled(c) && i + 1 < n_iter && st->t + 1 < st->opts.max_iter && path_settled(st, path);
        if (spec) em_enqueue(st, path, (slot + 1) % 3);
        const IterStatus s = em_wait(st, slot, path);
        bool live = spec;
        if (live && em_needs_host(st, s)) {
            CU(cudaStreamSynchronize(c->stream));
            live = false;
        }
        if (em_after(st, s, slot)) st->done = true;
        if (live && em_choose_path(st) != path) {
            CU(cudaStreamSynchronize(c->stream));
            live = false;
        }
        if (em_debug())
            fprintf(stderr, "[es em] t=%d path=%d min_nk=%.0f spec=%d kept=%d\n", st->t - 1, path, st->min_nk,
                    (int)spec, (int)live);
        pend = live ? path : -1;
    }
    if (st->t >= st->opts.max_iter) st->done = true;
}

}  // namespace

// ================================================================= C ABI
extern "C" {

const char* es_last_error_name(void) { return g_name.c_str(); }
const char* es_last_error_message(void) { return g_msg.c_str(); }
const char* es_version(void) { return "eventscope-b200 0.1.0 (sm_100a)"; }

static void ctx_common(es_ctx* c, int device) {
    c->device = device;
    CU(cudaSetDevice(device));
    CU(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
        CU(cudaEventCreateWithFlags(&c->evc[i], cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&c->evt[i], cudaEventDisableTiming));
    }
    CU(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));

    CU(cudaMallocHost(&c->h_status, sizeof(IterStatus)));
}

int es_ctx_create(int device, es_ctx** out) {
    return guard([&] {
        auto c = std::make_unique<es_ctx>();
        ctx_common(c.get(), device);
        *out = c.release();
    });
}

int es_nccl_unique_id(unsigned char id[128]) {
    return guard([&] {
        ncclUniqueId u;
        NC(nccl().GetUniqueId(&u));
        static_assert(sizeof(u) == 128, "nccl id size");
        std::memcpy(id, &u, 128);
    });
}

int es_ctx_create_nccl(int device, int rank, int world, const unsigned char id[128], es_ctx** out) {
    return guard([&] {
        if (world < 1 || rank < 0 || rank >= world) fail(ES_ERR_DATA, "RangeViolation", "bad rank/world");
        auto c = std::make_unique<es_ctx>();
        ctx_common(c.get(), device);
        c->rank = rank;
        c->world = world;
        // ES_FORCE_NCCL=1: a one-rank NCCL communicator too (tests the NCCL exchange path
        // on a single GPU)
        const char* fe = std::getenv("ES_FORCE_NCCL");
        if (world > 1 || (fe && fe[0] == '1')) {
            ncclUniqueId u;
            std::memcpy(&u, id, 128);
            NC(nccl().CommInitRank(&c->comm, world, u, rank));
            c->mode = 1;
        }
        *out = c.release();
    });
}

int es_ctx_create_exchange(int device, int rank, int world, const es_exchange* ex, es_ctx** out) {
    return guard([&] {
        if (world < 1 || rank < 0 || rank >= world) fail(ES_ERR_DATA, "RangeViolation", "bad rank/world");
        if (world > 1 && (!ex || !ex->allgather || !ex->allreduce))
            fail(ES_ERR_DATA, "InvalidExchange", "exchange callbacks required");
        auto c = std::make_unique<es_ctx>();
        ctx_common(c.get(), device);
        c->rank = rank;
        c->world = world;
        if (world > 1) {
            c->ex = *ex;
            c->mode = 2;
        }
        *out = c.release();
    });
}

int es_ctx_destroy(es_ctx* c) {
    return guard([&] {
        if (!c) return;
        cudaSetDevice(c->device);
        cudaStreamSynchronize(c->stream);
        for (es_dataset* d : c->live) d->ctx = nullptr;  // live datasets free their own planes later
        c->live.clear();
        if (c->comm) nccl().CommDestroy(c->comm);
        if (c->h_status) cudaFreeHost(c->h_status);
        if (c->ev0) cudaEventDestroy(c->ev0);
        if (c->ev1) cudaEventDestroy(c->ev1);
        cudaStreamSynchronize(c->cstream);
        if (c->plane_cache) cudaFree(c->plane_cache);
        for (int i = 0; i < 2; ++i) {
            if (c->evc[i]) cudaEventDestroy(c->evc[i]);
            if (c->evt[i]) cudaEventDestroy(c->evt[i]);
        }
        cudaStreamDestroy(c->cstream);
        cudaStreamDestroy(c->stream);
        delete c;
    });
}

int es_ctx_stream(es_ctx* c, void** stream) {
    return guard([&] { *stream = (void*)c->stream; });
}

int es_ctx_launch_count(es_ctx* c, int64_t* count) {
    return guard([&] { *count = c->ls.launches; });
}

int es_ctx_collective_count(es_ctx* c, int64_t* count) {
    return guard([&] { *count = c->collectives; });
}

int es_ctx_set_precision(es_ctx* c, int mode) {
    return guard([&] {
        if (mode != 0 && mode != 1) fail(ES_ERR_DATA, "RangeViolation", "precision mode must be 0 or 1");
        c->precision = mode;
    });
}

int es_ctx_set_timing(es_ctx* c, int enable) {
    return guard([&] {
        CU(cudaSetDevice(c->device));
        if (enable && !c->ev0) {
            CU(cudaEventCreate(&c->ev0));
            CU(cudaEventCreate(&c->ev1));
        }
        c->timing = enable != 0;
        c->em_ms = c->score_ms = 0.0;
        c->em_launches = c->score_launches = 0;
    });
}

int es_ctx_kernel_time(es_ctx* c, int which, double* ms, int64_t* launches) {
    return guard([&] {
        *ms = which == 0 ? c->em_ms : c->score_ms;
        *launches = which == 0 ? c->em_launches : c->score_launches;
    });
}

// -------------------------------------------------------------- dataset
static void finish_dataset(es_ctx* c, es_dataset* ds) {
    c->live.push_back(ds);
    ds->has_xmap = ds->n_local > 0 && make_event_tmap(&ds->xmap, ds->X, ds->n_local, ds->ld, ds->D);
    double nl = (double)ds->n_local;
    std::vector<double> all = c->allgather_host(&nl, 1);
    int64_t off = 0, tot = 0;
    for (int g = 0; g < c->world; ++g) {
        if (g < c->rank) off += (int64_t)all[g];
        tot += (int64_t)all[g];
    }
    ds->row_offset = off;
    ds->n_global = tot;
}

int es_dataset_create(es_ctx* c, const double* X, int64_t n_local, int32_t D, int64_t row_stride,
                      int64_t col_stride, es_dataset** out) {
    return guard([&] {
        if (D < 1 || D > 64) fail(ES_ERR_DATA, "DimensionMismatch", "D must be in [1,64]");
        if (n_local < 0) fail(ES_ERR_DATA, "RangeViolation", "negative row count");
        CU(cudaSetDevice(c->device));
        auto ds = std::make_unique<es_dataset>();
        ds->ctx = c;
        ds->n_local = n_local;
        ds->D = D;
        ds->ld = plane_ld(std::max<int64_t>(n_local, 1));
        ds->X = c->take_planes((size_t)ds->ld * D * 8);
        ds->owned_by_cache = true;
        if (n_local > 0) {
            if (!X) fail(ES_ERR_DATA, "InvalidInput", "null matrix");
            const bool dev = is_device_ptr(X);
            std::vector<double> packed;
            const bool row_major = (row_stride == D && col_stride == 1) || n_local == 1;
            const bool col_major = !row_major && row_stride == 1 && col_stride >= n_local;
            if (n_local == 1) {
                row_stride = D;
                col_stride = 1;
            }
            if (!row_major && !col_major) {
                if (dev) fail(ES_ERR_DATA, "UnsupportedLayout", "device input must be row- or column-major");
                packed.resize((size_t)n_local * D);
                for (int64_t i = 0; i < n_local; ++i)
                    for (int j = 0; j < D; ++j) packed[(size_t)i * D + j] = X[i * row_stride + (int64_t)j * col_stride];
                X = packed.data();
                row_stride = D;
                col_stride = 1;
            }
            if (col_major) {
                CU(cudaMemcpy2DAsync(ds->X, ds->ld * 8, X, col_stride * 8, n_local * 8, D, cudaMemcpyDefault,
                                     c->stream));
            } else {
                // 64 MB chunks, two staging buffers: the copy of chunk i + 1 (copy stream)
                // overlaps the row -> plane transpose of chunk i (compute stream)
                const int64_t chunk = std::max<int64_t>(1, (64ll << 20) / (8 * D));
                double* stage[2] = {c->scratch3.as<double>((size_t)std::min(chunk, n_local) * D),
                                    c->stage2.as<double>((size_t)std::min(chunk, n_local) * D)};
                CU(cudaEventRecord(c->evt[0], c->stream));  // the allocation is ordered before the copies
                CU(cudaStreamWaitEvent(c->cstream, c->evt[0], 0));
                int64_t ci = 0;
                for (int64_t r0 = 0; r0 < n_local; r0 += chunk, ++ci) {
                    const int b = (int)(ci & 1);
                    const int64_t nr = std::min(chunk, n_local - r0);
                    if (ci >= 2) CU(cudaStreamWaitEvent(c->cstream, c->evt[b], 0));  // buffer b transposed
                    CU(cudaMemcpyAsync(stage[b], X + r0 * D, (size_t)nr * D * 8, cudaMemcpyDefault, c->cstream));
                    CU(cudaEventRecord(c->evc[b], c->cstream));
                    CU(cudaStreamWaitEvent(c->stream, c->evc[b], 0));
                    launch_rows_to_planar(stage[b], nr, D, ds->X, ds->ld, r0, c->stream, c->ls);
                    c->check_launch();
                    CU(cudaEventRecord(c->evt[b], c->stream));
                }
            }
            c->sync();
        }
        finish_dataset(c, ds.get());
        *out = ds.release();
    });
}

// SYN-v1 true model: host SplitMix64 stream, same algorithm as
// the oracle's eso_syn_model; rows come from the device Philox generator.
static void syn_true_model(uint64_t seed, int D, int K, std::vector<double>& cum, std::vector<double>& mu,
                           std::vector<double>& chol) {
    SplitMix64 rng(seed ^ 0x53594E2D76310000ull);
    auto normal = [&]() {
        const double u1 = 1.0 - rng.uniform(), u2 = rng.uniform();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
    };
    double z = 0.0;
    for (int k = 0; k < K; ++k) z += (double)(k + 1);
    cum.resize(K);
    double acc = 0.0;
    for (int k = 0; k < K; ++k) {
        acc += (double)(k + 1) / z;
        cum[k] = acc;
    }
    mu.resize((size_t)K * D);
    chol.assign((size_t)K * D * D, 0.0);
    std::vector<double> B((size_t)D * D), Sg((size_t)D * D);
    for (int k = 0; k < K; ++k) {
        for (int d = 0; d < D; ++d) mu[(size_t)k * D + d] = -3.0 + 6.0 * rng.uniform();
        for (auto& b : B) b = normal();
        for (int a = 0; a < D; ++a)
            for (int c = 0; c < D; ++c) {
                double s = 0.0;
                for (int p = 0; p < D; ++p) s += B[(size_t)a * D + p] * B[(size_t)c * D + p];
                Sg[(size_t)a * D + c] = s / D + (a == c ? 0.05 : 0.0);
            }
        double* L = &chol[(size_t)k * D * D];
        for (int j = 0; j < D; ++j) {
            double s = Sg[(size_t)j * D + j];
            for (int p = 0; p < j; ++p) s -= L[j * D + p] * L[j * D + p];
            L[j * D + j] = std::sqrt(s);
            for (int i = j + 1; i < D; ++i) {
                double t = Sg[(size_t)i * D + j];
                for (int p = 0; p < j; ++p) t -= L[i * D + p] * L[j * D + p];
                L[i * D + j] = t / L[j * D + j];
            }
        }
    }
}

int es_dataset_generate(es_ctx* c, uint64_t seed, int64_t n_global, int32_t D, int32_t K_true, es_dataset** out) {
    return es_dataset_generate_range(c, seed, 0, n_global, D, K_true, out);
}

int es_dataset_generate_range(es_ctx* c, uint64_t seed, int64_t row0, int64_t n_global, int32_t D, int32_t K_true,
                              es_dataset** out) {
    return guard([&] {
        if (D < 1 || D > 64) fail(ES_ERR_DATA, "DimensionMismatch", "D must be in [1,64]");
        if (K_true < 1 || n_global < 0 || row0 < 0) fail(ES_ERR_DATA, "RangeViolation", "bad generator shape");
        CU(cudaSetDevice(c->device));
        auto ds = std::make_unique<es_dataset>();
        ds->ctx = c;
        ds->D = D;
        const int64_t r0 = row0 + n_global * c->rank / c->world, r1 = row0 + n_global * (c->rank + 1) / c->world;
        ds->n_local = r1 - r0;
        ds->ld = plane_ld(std::max<int64_t>(ds->n_local, 1));
        CU(cudaMalloc(&ds->X, (size_t)ds->ld * D * 8));
        std::vector<double> cum, mu, chol;
        syn_true_model(seed, D, K_true, cum, mu, chol);
        std::vector<double> blob;
        blob.insert(blob.end(), cum.begin(), cum.end());
        blob.insert(blob.end(), mu.begin(), mu.end());
        blob.insert(blob.end(), chol.begin(), chol.end());
        double* dm = c->scratch2.as<double>(blob.size());
        CU(cudaMemcpyAsync(dm, blob.data(), blob.size() * 8, cudaMemcpyHostToDevice, c->stream));
        launch_synth(ds->X, ds->ld, ds->n_local, r0, D, K_true, dm, seed, c->stream, c->ls);
        c->check_launch();
        c->sync();
        finish_dataset(c, ds.get());
        *out = ds.release();
    });
}

// ---------------------------------------------------------------- pipeline
// A dataset sharing `base`'s (or its own) planes, restricted to the global rows [0, n_rows)
// (`own` = false: the view never frees X).
static es_dataset* make_view(es_ctx* c, es_dataset* base, double* X, int64_t n_rows) {
    auto v = std::make_unique<es_dataset>();
    v->ctx = c;
    v->D = base->D;
    v->ld = base->ld;
    v->X = X;
    v->n_local = std::max<int64_t>(0, std::min(base->n_local, n_rows - base->row_offset));
    finish_dataset(c, v.get());
    return v.release();
}

int es_run_pipeline(es_ctx* c, es_dataset* ds, const es_pipeline_cfg* cfg, es_gmm_params* model, es_fit_report* rep,
                    double* std_mean, double* std_scale, double* delta, double* log_delta, uint8_t* flags,
                    int32_t* best_k, double* best_logdens, int64_t* anomaly_indices, int64_t* n_local_flagged,
                    int64_t* n_flagged) {
    struct Views {  // views do not own their planes; the standardized copy is owned here
        es_dataset* train = nullptr;
        es_dataset* all = nullptr;
        es_dataset* ztrain = nullptr;
        double* Z = nullptr;
        ~Views() {
            for (es_dataset* v : {train, ztrain}) {
                if (v) v->X = nullptr;
                delete v;
            }
            if (all) all->X = nullptr;
            delete all;
            if (Z) cudaFree(Z);
        }
    } V;
    int status = guard([&] {
        CU(cudaSetDevice(c->device));
        if (!cfg || !model || !delta || !log_delta) fail(ES_ERR_DATA, "InvalidArgument", "null argument");
        const int D = ds->D, K = cfg->K;
        if (model->K != K || model->D != D) fail(ES_ERR_DATA, "DimensionMismatch", "model buffers do not match K, D");
        if (!(cfg->train_window > 0.0 && cfg->train_window <= 1.0))
            fail(ES_ERR_DATA, "RangeViolation", "train_window must be in (0,1]");
        if (ds->n_global < 1) fail(ES_ERR_DATA, "EmptyLayer", "no events");
        const int64_t n_train = (int64_t)std::floor(cfg->train_window * (double)ds->n_global);
        if (n_train < 10 * (int64_t)K)
            fail(ES_ERR_DATA, "InsufficientTraining", "training split has fewer than 10*K events");
        if (!(cfg->quantile_q > 0.0) && !(cfg->delta > 0.0))
            fail(ES_ERR_DATA, "RangeViolation", "need quantile_q in (0,1) or delta > 0");
        // training-split statistics (rank-ordered sums: identical on every rank)
        std::vector<double> mean(D, 0.0), scale(D, 1.0);
        V.train = make_view(c, ds, ds->X, n_train);
        if (cfg->standardize) {
            const DataStats st = data_stats(c, V.train);
            if (st.nonfinite > 0) fail(ES_ERR_DATA, "NonFiniteFeature", "X contains non-finite entries");
            for (int j = 0; j < D; ++j) {
                mean[j] = st.mean[j];
                const double var = st.S[(size_t)j * D + j];
                scale[j] = var > 0.0 ? std::sqrt(var) : 1.0;  // zero variance: centred only
            }
            // standardized copy of every local row
            CU(cudaMalloc(&V.Z, (size_t)ds->ld * D * 8));
            std::vector<double> ms(2 * D);
            for (int j = 0; j < D; ++j) {
                ms[j] = mean[j];
                ms[D + j] = 1.0 / scale[j];
            }
            double* dms = c->scratch2.as<double>(2 * D);
            CU(cudaMemcpyAsync(dms, ms.data(), 2 * D * 8, cudaMemcpyHostToDevice, c->stream));
            launch_standardize(ds->X, ds->n_local, ds->ld, D, dms, dms + D, V.Z, ds->ld, c->num_sms, c->stream,
                               c->ls);
            c->check_launch();
            V.all = make_view(c, ds, V.Z, ds->n_global);
            V.ztrain = make_view(c, ds, V.Z, n_train);
        }
        es_dataset* fit_ds = cfg->standardize ? V.ztrain : V.train;
        es_dataset* all_ds = cfg->standardize ? V.all : ds;
        es_fit_report r{};
        if (int e = es_gmm_fit(c, fit_ds, K, &cfg->fit, nullptr, model, rep ? rep : &r, nullptr)) rethrow_last(e);
        if (cfg->quantile_q > 0.0) {
            if (int e = es_gmm_calibrate(c, all_ds, model, n_train, cfg->quantile_q, cfg->mode, delta, log_delta))
                rethrow_last(e);
        } else {
            *delta = cfg->delta;
            *log_delta = std::log(cfg->delta);
        }
        if (int e = es_gmm_detect(c, all_ds, model, *log_delta, cfg->mode, flags, best_k, best_logdens,
                                  anomaly_indices, n_local_flagged, n_flagged))
            rethrow_last(e);
        if (std_mean) std::copy(mean.begin(), mean.end(), std_mean);
        if (std_scale) std::copy(scale.begin(), scale.end(), std_scale);
    });
    return status;
}

// k-means baseline (eval-bench): Lloyd's algorithm with k-means++
// seeding on the train split (the first floor(train_window N) rows, as run_pipeline);
// score = distance to the nearest centroid; threshold = (1 - q)-quantile of the train
// scores (linear interpolation, h = (n_train - 1)(1 - q), the calibrate convention);
// flag iff score > threshold.  Lloyd stops when no assignment changes or after max_iter
// steps; an empty cluster keeps its centroid.
int es_kmeans_baseline(es_ctx* c, es_dataset* ds, int32_t K, double q, double train_window, uint64_t seed,
                       int32_t max_iter, double* centroids, double* threshold, uint8_t* flags, double* scores,
                       int64_t* n_flagged, int32_t* iterations) {
    struct View {
        es_dataset* v = nullptr;
        ~View() {
            if (v) v->X = nullptr;
            delete v;
        }
    } V;
    return guard([&] {
        CU(cudaSetDevice(c->device));
        const int D = ds->D;
        if (K < 1) fail(ES_ERR_DATA, "InvalidK", "K must be >= 1");
        if (D > 64) fail(ES_ERR_DATA, "DimensionTooLarge", "k-means baseline supports D <= 64");
        if (!(q > 0.0 && q < 1.0)) fail(ES_ERR_DATA, "RangeViolation", "q must be in (0,1)");
        if (!(train_window > 0.0 && train_window <= 1.0))
            fail(ES_ERR_DATA, "RangeViolation", "train_window must be in (0,1]");
        const int64_t n_train = (int64_t)std::floor(train_window * (double)ds->n_global);
        if (n_train < K) fail(ES_ERR_DATA, "TooFewPoints", "training split has fewer rows than K");
        if ((size_t)(K * D + 8 * (K * (D + 1) + 1)) * 8 > 227 * 1024)
            fail(ES_ERR_DATA, "DimensionTooLarge", "K (D + 1) too large for the k-means kernel");
        if (max_iter <= 0) max_iter = 100;
        V.v = make_view(c, ds, ds->X, n_train);
        es_dataset* tr = V.v;
        SplitMix64 rng(seed);
        const std::vector<int64_t> rows = kmeanspp_device(c, tr, K, rng);
        std::vector<double> cen;
        fetch_rows(c, tr, rows, cen);
        const int L = K * (D + 1) + 1;
        const int grid = lloyd_grid(tr->n_local, c->num_sms);
        double* dcen = c->o1.as<double>((size_t)K * D);
        int32_t* asg = c->o2.as<int32_t>(std::max<int64_t>(tr->n_local, 1));
        double* part = c->o3.as<double>((size_t)grid * L);
        double* red = c->o4.as<double>(L);
        CU(cudaMemsetAsync(asg, 0xFF, std::max<int64_t>(tr->n_local, 1) * 4, c->stream));  // -1: unassigned
        int it = 0;
        std::vector<double> h(L);
        while (it < max_iter) {
            CU(cudaMemcpyAsync(dcen, cen.data(), (size_t)K * D * 8, cudaMemcpyHostToDevice, c->stream));
            if (tr->n_local > 0) {
                launch_lloyd(tr->X, tr->n_local, tr->ld, D, K, dcen, asg, part, nullptr, 0, grid, c->stream, c->ls);
                c->check_launch();
                launch_reduce_blocks(part, grid, L, red, c->stream, c->ls);
                c->check_launch();
                CU(cudaMemcpyAsync(h.data(), red, (size_t)L * 8, cudaMemcpyDeviceToHost, c->stream));
                c->sync();
            } else {
                std::fill(h.begin(), h.end(), 0.0);
            }
            const std::vector<double> all = c->allgather_host(h.data(), L);  // rank-ordered sum
            std::vector<double> tot(L, 0.0);
            for (int g = 0; g < c->world; ++g)
                for (int e = 0; e < L; ++e) tot[e] += all[(size_t)g * L + e];
            ++it;
            for (int k = 0; k < K; ++k) {
                const double cnt = tot[(size_t)k * (D + 1) + D];
                if (cnt > 0.0)
                    for (int a = 0; a < D; ++a) cen[(size_t)k * D + a] = tot[(size_t)k * (D + 1) + a] / cnt;
            }
            if (tot[L - 1] == 0.0) break;  // no assignment changed: the centroids are the ones just used
        }
        // scores of every local row, threshold from the train rows, flags
        CU(cudaMemcpyAsync(dcen, cen.data(), (size_t)K * D * 8, cudaMemcpyHostToDevice, c->stream));
        double* dsc = c->out_scratch.as<double>(std::max<int64_t>(ds->n_local, 1));
        launch_lloyd(ds->X, ds->n_local, ds->ld, D, K, dcen, nullptr, nullptr, dsc, 1,
                     lloyd_grid(ds->n_local, c->num_sms), c->stream, c->ls);
        c->check_launch();
        const double hq = (double)(n_train - 1) * (1.0 - q);
        const int64_t lo = (int64_t)std::floor(hq);
        const int64_t hi = std::min<int64_t>(lo + 1, n_train - 1);
        const int64_t nloc = tr->n_local;
        const double vlo = radix_select(c, dsc, nloc, lo);
        const double vhi = hi == lo ? vlo : radix_select(c, dsc, nloc, hi);
        const double thr = vlo + (hq - (double)lo) * (vhi - vlo);
        uint8_t* dfl = c->o5.as<uint8_t>(std::max<int64_t>(ds->n_local, 1));
        unsigned long long* dcount = c->hist.as<unsigned long long>(256);
        launch_flag_gt(dsc, ds->n_local, thr, dfl, dcount, c->num_sms, c->stream, c->ls);
        c->check_launch();
        unsigned long long cnt = 0;
        CU(cudaMemcpyAsync(&cnt, dcount, 8, cudaMemcpyDeviceToHost, c->stream));
        if (flags && ds->n_local)
            CU(cudaMemcpyAsync(flags, dfl, ds->n_local, cudaMemcpyDefault, c->stream));
        if (scores && ds->n_local)
            CU(cudaMemcpyAsync(scores, dsc, ds->n_local * 8, cudaMemcpyDefault, c->stream));
        c->sync();
        double total = (double)cnt;
        c->allreduce_host(&total, 1, 0, 0);
        if (centroids) std::copy(cen.begin(), cen.end(), centroids);
        if (threshold) *threshold = thr;
        if (n_flagged) *n_flagged = (int64_t)total;
        if (iterations) *iterations = it;
    });
}

// confusion counts of labels against flags (anomaly = positive class);
// host or device arrays; out = {tp, fp, tn, fn}
int es_confusion(es_ctx* c, const uint8_t* labels, const uint8_t* flags, int64_t n, int64_t* out) {
    return guard([&] {
        CU(cudaSetDevice(c->device));
        if (n < 0) fail(ES_ERR_DATA, "LengthMismatch", "negative length");
        if (!out) fail(ES_ERR_DATA, "InvalidArgument", "null output");
        const uint8_t* dl = labels;
        const uint8_t* df = flags;
        if (n > 0 && !is_device_ptr(labels)) {
            uint8_t* t = c->o1.as<uint8_t>(n);
            CU(cudaMemcpyAsync(t, labels, n, cudaMemcpyHostToDevice, c->stream));
            dl = t;
        }
        if (n > 0 && !is_device_ptr(flags)) {
            uint8_t* t = c->o2.as<uint8_t>(n);
            CU(cudaMemcpyAsync(t, flags, n, cudaMemcpyHostToDevice, c->stream));
            df = t;
        }
        unsigned long long* d = c->hist.as<unsigned long long>(256);
        launch_confusion(dl, df, n, d, c->num_sms, c->stream, c->ls);
        c->check_launch();
        unsigned long long h[4] = {0, 0, 0, 0};
        CU(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        for (int j = 0; j < 4; ++j) out[j] = (int64_t)h[j];
    });
}

// extract_features on the device from columnar events: validation of the
// TraceEvent invariants (first violating row reported), the layer filter
// (order-preserving compaction) and the layer's default features, straight into a
// library-owned planar dataset.  Columns may be host or device arrays.
int es_events_extract(es_ctx* c, const es_event_columns* cols, int64_t n, int32_t layer, es_dataset** out,
                      int64_t* event_index, int64_t* bad_row) {
    return guard([&] {
        CU(cudaSetDevice(c->device));
        if (bad_row) *bad_row = -1;
        if (!cols || !out) fail(ES_ERR_DATA, "InvalidArgument", "null argument");
        if (n < 0) fail(ES_ERR_DATA, "RangeViolation", "negative event count");
        if (layer < 0 || layer > 4) fail(ES_ERR_DATA, "UnknownLayer", "layer must be 0..4");
        if (n > 0 && (!cols->layer || !cols->ts_start || !cols->duration_ns))
            fail(ES_ERR_DATA, "MissingField", "layer, ts_start and duration_ns columns are required");
        const int D = layer == ES_LAYER_GPU_SAMPLE ? 3 : (layer == ES_LAYER_NCCL ? 2 : 1);
        // device copies of host columns (8-byte aligned slices of one buffer)
        const int64_t n8 = (n + 7) & ~int64_t(7);
        std::vector<const void*> src = {cols->layer, cols->ts_start, cols->duration_ns, cols->message_bytes,
                                        cols->util_pct, cols->mem_used_mb, cols->temp_c};
        const size_t width[7] = {1, 8, 8, 8, 8, 8, 8};
        size_t tot = 0;
        for (int j = 0; j < 7; ++j) tot += (size_t)n8 * width[j];
        unsigned char* buf = c->o1.as<unsigned char>(std::max<size_t>(tot, 8));
        std::vector<const void*> dptr(7, nullptr);
        size_t off = 0;
        for (int j = 0; j < 7; ++j) {
            if (src[j] && n > 0) {
                if (is_device_ptr(src[j])) {
                    dptr[j] = src[j];
                } else {
                    CU(cudaMemcpyAsync(buf + off, src[j], (size_t)n * width[j], cudaMemcpyHostToDevice, c->stream));
                    dptr[j] = buf + off;
                }
            }
            off += (size_t)n8 * width[j];
        }
        const auto* L = static_cast<const uint8_t*>(dptr[0]);
        const auto* ts = static_cast<const int64_t*>(dptr[1]);
        const auto* du = static_cast<const int64_t*>(dptr[2]);
        const auto* mb = static_cast<const double*>(dptr[3]);
        const auto* ut = static_cast<const double*>(dptr[4]);
        const auto* me = static_cast<const double*>(dptr[5]);
        const auto* te = static_cast<const double*>(dptr[6]);
        uint8_t* keep = c->o2.as<uint8_t>(std::max<int64_t>(n, 1));
        unsigned long long* bad = c->hist.as<unsigned long long>(256);
        launch_event_keep(L, ts, du, mb, ut, me, te, n, layer, keep, bad, c->num_sms, c->stream, c->ls);
        c->check_launch();
        unsigned long long hb = ~0ull;
        CU(cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        if (hb != ~0ull) {
            static const char* names[8] = {"", "layer", "ts_start", "duration_ns", "message_bytes", "util_pct",
                                           "mem_used_mb", "temp_c"};
            const int64_t row = (int64_t)(hb >> 8);
            const int f = (int)(hb & 0xFF);
            if (bad_row) *bad_row = row;
            fail(ES_ERR_DATA, f == 1 ? "UnknownLayer" : (f & 0x10) ? "MissingField" : "RangeViolation",
                 std::string(names[f & 0xF]) + ((f & 0x10) ? " missing" : " out of range") + " at event " +
                     std::to_string(row));
        }
        const int64_t nc = (n + 4095) / 4096;
        int64_t* cnt = c->o3.as<int64_t>(std::max<int64_t>(nc, 1) + 8);
        int64_t* idx = c->o4.as<int64_t>(std::max<int64_t>(n, 1));
        int64_t* dm = cnt + std::max<int64_t>(nc, 1);
        launch_compact(keep, n, 0, cnt, idx, dm, c->stream, c->ls);
        c->check_launch();
        int64_t m = 0;
        CU(cudaMemcpyAsync(&m, dm, 8, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        if (m == 0) fail(ES_ERR_DATA, "EmptyLayer", "no events of the requested layer");
        auto ds = std::make_unique<es_dataset>();
        ds->ctx = c;
        ds->n_local = m;
        ds->D = D;
        ds->ld = plane_ld(m);
        CU(cudaMalloc(&ds->X, (size_t)ds->ld * D * 8));
        launch_event_features(idx, m, du, mb, ut, me, te, layer, ds->X, ds->ld, c->num_sms, c->stream, c->ls);
        c->check_launch();
        if (event_index) CU(cudaMemcpyAsync(event_index, idx, (size_t)m * 8, cudaMemcpyDefault, c->stream));
        c->sync();
        finish_dataset(c, ds.get());
        *out = ds.release();
    });
}

int es_dataset_destroy(es_dataset* ds) {
    return guard([&] { delete ds; });
}

int es_dataset_info(es_dataset* ds, int64_t* n_local, int64_t* n_global, int64_t* row_offset, int32_t* D) {
    return guard([&] {
        if (n_local) *n_local = ds->n_local;
        if (n_global) *n_global = ds->n_global;
        if (row_offset) *row_offset = ds->row_offset;
        if (D) *D = ds->D;
    });
}

int es_dataset_read_rows(es_dataset* ds, int64_t row0, int64_t n, double* out) {
    return guard([&] {
        if (!ds->ctx) fail(ES_ERR_RUNTIME, "ContextDestroyed", "the dataset's context was destroyed");
        if (row0 < 0 || n < 0 || row0 + n > ds->n_local) fail(ES_ERR_DATA, "RangeViolation", "rows out of range");
        es_ctx* c = ds->ctx;
        if (n == 0) return;
        double* d = c->out_scratch.as<double>((size_t)n * ds->D);
        launch_planar_to_rows(ds->X, ds->ld, ds->D, row0, n, d, c->stream, c->ls);
        c->check_launch();
        CU(cudaMemcpyAsync(out, d, (size_t)n * ds->D * 8, cudaMemcpyDefault, c->stream));
        c->sync();
    });
}

// ------------------------------------------------------------------ fit
int es_gmm_em_begin(es_ctx* c, es_dataset* ds, int32_t K, const es_fit_opts* opts, const es_gmm_params* init,
                    es_em_state** out) {
    return guard([&] {
        CU(cudaSetDevice(c->device));
        if (!opts) fail(ES_ERR_DATA, "InvalidOptions", "null options");
        auto st = std::make_unique<es_em_state>();
        st->ctx = c;
        st->ds = ds;
        st->K = K;
        st->D = ds->D;
        st->opts = *opts;
        em_begin(st.get(), init);
        *out = st.release();
    });
}

int es_gmm_em_record_passes(const es_em_state* st, int32_t* passes) {
    return guard([&] {
        if (!st || !passes) fail(ES_ERR_DATA, "InvalidArgument", "null state or output");
        *passes = st->last_npass;
    });
}

int es_gmm_em_last_kernel(const es_em_state* st, const char** name) {
    return guard([&] {
        if (!st || !name) fail(ES_ERR_DATA, "InvalidArgument", "null state or output");
        static const char* names[] = {"none (empty shard)", "k_em_diag (FP64)", "strict FP64 (k_em_team / k_em_generic)",
                                      "k_em_mma<1>", "k_em_mma<2>", "k_em_diag_mixed", "k_em_full_mixed",
                                      "k_em_wide<1>", "k_em_wide<2>", "k_em_diag_tc"};
        *name = st->last_path < 0 ? "" : names[st->last_path];
    });
}

int es_gmm_em_step(es_em_state* st, int32_t n_iter, int32_t* done) {
    return guard([&] {
        CU(cudaSetDevice(st->ctx->device));
        em_steps(st, n_iter);
        if (done) *done = st->done ? 1 : 0;
    });
}

int es_gmm_em_end(es_em_state* st, es_gmm_params* out, es_fit_report* rep, double* per_iter) {
    return guard([&] {
        es_ctx* c = st->ctx;
        CU(cudaSetDevice(c->device));
        const int K = st->K, D = st->D;
        double* dmodel = em_model(st);
        double final_ll = st->last;
        if (!st->converged && !em_logl_pass(st, &final_ll))
            final_ll = run_score(c, st->ds, dmodel, K, ScoreOut{}, st->dcenter.as<double>(D), st->mean.data(), st->xs);
        if (out) {
            if (out->K != K || out->D != D) fail(ES_ERR_DATA, "DimensionMismatch", "output params shape");
            ModelView mv{K, D, dmodel};
            CU(cudaMemcpyAsync(out->weights, mv.pi(), K * 8, cudaMemcpyDeviceToHost, c->stream));
            CU(cudaMemcpyAsync(out->means, mv.mu(), (size_t)K * D * 8, cudaMemcpyDeviceToHost, c->stream));
            CU(cudaMemcpyAsync(out->covariances, mv.cov(), (size_t)K * D * D * 8, cudaMemcpyDeviceToHost, c->stream));
            c->sync();
        }
        if (rep) {
            rep->iterations = st->iterations;
            rep->final_log_likelihood = final_ll;
            rep->converged = st->converged ? 1 : 0;
            rep->seed = st->opts.seed;
            rep->n_per_iter = (int32_t)st->per_iter.size();
            rep->collapses = st->collapses;
            rep->reg_used = st->reg;
        }
        if (per_iter) std::copy(st->per_iter.begin(), st->per_iter.end(), per_iter);
    });
}

int es_gmm_em_free(es_em_state* st) {
    return guard([&] { delete st; });
}

int es_gmm_fit(es_ctx* c, es_dataset* ds, int32_t K, const es_fit_opts* opts, const es_gmm_params* init,
               es_gmm_params* out, es_fit_report* rep, double* per_iter) {
    es_em_state* st = nullptr;
    int s = es_gmm_em_begin(c, ds, K, opts, init, &st);
    if (s) return s;
    int32_t done = 0;
    s = es_gmm_em_step(st, opts->max_iter, &done);
    if (!s) s = es_gmm_em_end(st, out, rep, per_iter);
    delete st;
    return s;
}

// ---------------------------------------------------------------- score
int es_gmm_score(es_ctx* c, es_dataset* ds, const es_gmm_params* p, double* ll, int32_t* predict, int32_t* best_k,
                 double* best_logdens, double* total_ll) {
    return guard([&] {
        CU(cudaSetDevice(c->device));
        double* m = model_for(c, p, ds->D);
        const size_t n = ds->n_local;
        Out<double> o_ll(ll, n, c->o1), o_bl(best_logdens, n, c->o2);
        Out<int32_t> o_pr(predict, n, c->o3), o_bk(best_k, n, c->o4);
        ScoreOut o;
        o.ll = o_ll.dev;
        o.best_ld = o_bl.dev;
        o.predict = o_pr.dev;
        o.best_k = o_bk.dev;
        const double tot = run_score(c, ds, m, p->K, o, c->center.as<double>(ds->D), c->center_host.data(), c->center_xs);
        o_ll.finish(c->stream);
        o_bl.finish(c->stream);
        o_pr.finish(c->stream);
        o_bk.finish(c->stream);
        c->sync();
        if (total_ll) *total_ll = tot;
    });
}

int es_gmm_responsibilities(es_ctx* c, es_dataset* ds, const es_gmm_params* p, double* gamma) {
    return guard([&] {
        CU(cudaSetDevice(c->device));
        double* m = model_for(c, p, ds->D);
        Out<double> o_g(gamma, (size_t)ds->n_local * p->K, c->o1);
        ScoreOut o;
        o.gamma = o_g.dev;
        run_score(c, ds, m, p->K, o, c->center.as<double>(ds->D), c->center_host.data(), c->center_xs);
        o_g.finish(c->stream);
        c->sync();
    });
}

static void single_event(es_ctx* c, const es_gmm_params* p, const double* x, std::vector<double>& lnk, double* ll) {
    check_params(p, p->D);
    const int D = p->D, K = p->K;
    double* m = model_for(c, p, D);
    double* dx = c->scratch3.as<double>(D + (size_t)K + 8);
    double* dl = dx + D;
    double* dll = dl + K;
    CU(cudaMemcpyAsync(dx, x, D * 8, cudaMemcpyHostToDevice, c->stream));
    ScoreOut o;
    o.lnk = dl;
    o.ll = dll;
    double* bs = c->scratch.as<double>((size_t)2 * score_grid(D, K, c->num_sms) + 2);
    int nblk = 0;
    launch_score(dx, 1, 1, D, K, m, o, bs, c->num_sms, &nblk, c->stream, c->ls);
    c->check_launch();
    lnk.resize(K);
    CU(cudaMemcpyAsync(lnk.data(), dl, K * 8, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaMemcpyAsync(ll, dll, 8, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
}

int es_gmm_component_log_density(es_ctx* c, const es_gmm_params* p, const double* x, int32_t k, double* out) {
    return guard([&] {
        CU(cudaSetDevice(c->device));
        if (!p || k < 0 || k >= p->K) fail(ES_ERR_DATA, "DimensionMismatch", "component index out of range");
        std::vector<double> lnk;
        double ll;
        single_event(c, p, x, lnk, &ll);
        *out = lnk[k];
    });
}

int es_gmm_mixture_log_density(es_ctx* c, const es_gmm_params* p, const double* x, double* out) {
    return guard([&] {
        CU(cudaSetDevice(c->device));
        std::vector<double> lnk;
        single_event(c, p, x, lnk, out);
    });
}

// --------------------------------------------------------------- detect
int es_gmm_detect(es_ctx* c, es_dataset* ds, const es_gmm_params* p, double log_delta, int32_t mode, uint8_t* flags,
                  int32_t* best_k, double* best_logdens, int64_t* anomaly_indices, int64_t* n_local_flagged,
                  int64_t* n_flagged) {
    return guard([&] {
        CU(cudaSetDevice(c->device));
        if (mode != 0 && mode != 1) fail(ES_ERR_DATA, "RangeViolation", "mode must be 0 or 1");
        double* m = model_for(c, p, ds->D);
        const size_t n = ds->n_local;
        uint8_t* dflags = flags && is_device_ptr(flags) ? flags : c->o5.as<uint8_t>(std::max<size_t>(n, 1));
        Out<int32_t> o_bk(best_k, n, c->o2);
        Out<double> o_bl(best_logdens, n, c->o3);
        Out<int64_t> o_idx(anomaly_indices, n, c->o4);
        ScoreOut o;
        o.flags = dflags;
        o.best_k = o_bk.dev;
        o.best_ld = o_bl.dev;
        o.log_delta = log_delta;
        o.mode = mode;
        o.sum_ll = 0;  // detect reports no log-likelihood
        run_score(c, ds, m, p->K, o, c->center.as<double>(ds->D), c->center_host.data(), c->center_xs, false);
        int64_t* cnt = c->scratch2.as<int64_t>((n + 4095) / 4096 + 2);
        int64_t* dcount = cnt + (n + 4095) / 4096 + 1;
        launch_compact(dflags, n, ds->row_offset, cnt, o_idx.dev, dcount, c->stream, c->ls);
        c->check_launch();
        int64_t local = 0;
        CU(cudaMemcpyAsync(&local, dcount, 8, cudaMemcpyDeviceToHost, c->stream));
        if (flags && dflags != flags) CU(cudaMemcpyAsync(flags, dflags, n, cudaMemcpyDeviceToHost, c->stream));
        o_bk.finish(c->stream);
        o_bl.finish(c->stream);
        c->sync();
        if (o_idx.user && o_idx.dev != o_idx.user && local) {
            CU(cudaMemcpyAsync(o_idx.user, o_idx.dev, local * 8, cudaMemcpyDeviceToHost, c->stream));
            c->sync();
        }
        if (n == 0) local = 0;
        if (n_local_flagged) *n_local_flagged = local;
        long long g = local;
        c->allreduce_host(&g, 1, 1, 0);
        if (n_flagged) *n_flagged = g;
    });
}

int es_gmm_calibrate(es_ctx* c, es_dataset* ds, const es_gmm_params* p, int64_t n_train, double q, int32_t mode,
                     double* delta, double* log_delta) {
    return guard([&] {
        CU(cudaSetDevice(c->device));
        if (n_train < 1) fail(ES_ERR_DATA, "EmptyTraining", "training split is empty");
        if (n_train > ds->n_global) fail(ES_ERR_DATA, "RangeViolation", "n_train exceeds the dataset");
        if (!(q > 0.0 && q < 1.0)) fail(ES_ERR_DATA, "RangeViolation", "q must be in (0,1)");
        if (mode != 0 && mode != 1) fail(ES_ERR_DATA, "RangeViolation", "mode must be 0 or 1");
        double* m = model_for(c, p, ds->D);
        const int64_t nloc = std::max<int64_t>(0, std::min(ds->n_local, n_train - ds->row_offset));
        double* keys = c->out_scratch.as<double>(std::max<int64_t>(nloc, 1));
        if (nloc > 0) {  // the train rows are the first nloc local rows (planes keep their stride)
            ScoreOut o;
            o.mode = mode;
            o.sum_ll = 0;
            if (mode == 1) o.ll = keys;
            else o.best_ld = keys;
            int nblk = 0;
            double* bs = c->scratch.as<double>(score_blocks(c, ds->D, p->K));
            score_launch(c, ds->X, nloc, ds->ld, ds->D, p->K, m, c->center.as<double>(ds->D), c->center_host.data(),
                         c->center_xs, o, bs, &nblk,
                         ds->has_xmap ? &ds->xmap : nullptr);
            c->check_launch();
        }
        // q-quantile, linear interpolation between order statistics, h = (n-1) q
        const double h = (double)(n_train - 1) * q;
        const int64_t lo = (int64_t)std::floor(h);
        const int64_t hi = std::min<int64_t>(lo + 1, n_train - 1);
        const double vlo = radix_select(c, keys, nloc, lo);
        const double vhi = hi == lo ? vlo : radix_select(c, keys, nloc, hi);
        const double dlo = std::exp(vlo), dhi = std::exp(vhi);
        const double frac = h - (double)lo;
        const double d = dlo + frac * (dhi - dlo);
        *delta = d;
        // one shared log(delta); exact endpoints keep their log
        *log_delta = (d == dlo) ? vlo : (d == dhi) ? vhi : std::log(d);
    });
}

int es_gmm_select_k_bic(es_ctx* c, es_dataset* ds, const int32_t* k_range, int32_t n_k, const es_fit_opts* opts,
                        int32_t* best_k, double* bic) {
    return guard([&] {
        if (n_k < 1) fail(ES_ERR_DATA, "EmptyRange", "k_range is empty");
        int best = -1;
        double best_bic = INFINITY;
        int last = ES_OK;
        std::string ln, lm;
        const int D = ds->D;
        for (int j = 0; j < n_k; ++j) {
            const int K = k_range[j];
            std::vector<double> pi(std::max(K, 1)), mu((size_t)std::max(K, 1) * D),
                cov((size_t)std::max(K, 1) * D * D);
            es_gmm_params outp{K, D, pi.data(), mu.data(), cov.data()};
            es_fit_report rep{};
            const int s = es_gmm_fit(c, ds, K, opts, nullptr, &outp, &rep, nullptr);
            if (s != ES_OK) {  // skip failed K
                bic[j] = NAN;
                last = s;
                ln = g_name;
                lm = g_msg;
                continue;
            }
            const double p = (K - 1) + (double)K * D +
                             (opts->covariance_type == ES_COV_DIAG ? (double)K * D
                                                                   : (double)K * D * (D + 1) / 2.0);
            bic[j] = -2.0 * rep.final_log_likelihood + p * std::log((double)ds->n_global);
            if (bic[j] < best_bic) {
                best_bic = bic[j];
                best = K;
            }
        }
        if (best < 0) fail(last, ln, lm);
        *best_k = best;
    });
}

}  // extern "C"
