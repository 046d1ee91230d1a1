// Internal declarations shared by the libedfa translation units.
#pragma once
#include <chrono>
#include <unordered_map>
#include <mutex>
#include <map>

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/edfa.h"

namespace edfa {

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// EDFA_SLOW_LOG=<ms>: report runtime calls that block the host longer than
// that (diagnostics for host stalls inside the driver)
double slow_log_ms();
void slow_log(double ms, const char* what, const char* file, int line);
inline double host_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

#define EDFA_CUDA(call)                                                          \
    do {                                                                         \
        const double lim_ = ::edfa::slow_log_ms();                               \
        const double t0_ = lim_ > 0 ? ::edfa::host_ms() : 0.0;                   \
        cudaError_t e_ = (call);                                                 \
        if (lim_ > 0) {                                                          \
            double dt_ = ::edfa::host_ms() - t0_;                                \
            if (dt_ > lim_) ::edfa::slow_log(dt_, #call, __FILE__, __LINE__);    \
        }                                                                        \
        if (e_ != cudaSuccess)                                                   \
            throw ::edfa::Error(EDFA_ERR_CUDA, std::string(#call ": ") +         \
                                                  cudaGetErrorString(e_));       \
    } while (0)

inline void require(bool ok, int code, const std::string& msg) {
    if (!ok) throw Error(code, msg);
}

// ---------------------------------------------------------------- context
struct ProfRec {
    const char* name;
    cudaEvent_t t0, t1;
    double bytes;
};

// Algorithm selections of a context.  Defaults are the production choices;
// the alternatives are kept because tests compare them against each other
// (edfa_ctx_set_option; the EDFA_OPT_* environment variables seed them once
// at context creation).
struct CtxOptions {
    int ic_pair = 1;        // fused (L L^T)^-1 chain kernel for chain-structured IC factors
    int fill_fusion = 1;    // the two ILU tile solves pre-fill each other's SENTINELs
    int trsv_levels = 0;    // level-synchronous triangular solves instead of the sync-free ones
    int ilu_levels = 0;     // level-synchronous ILU(0) factorisation instead of the sync-free one
    int tile_direct = -1;   // ILU tile solves: -1 by wavefront width, 0 staged plan (15 warps), 1 direct (7 warps)
    int ilu_wf = -1;        // ILU solves wavefront-packed on one slot layout: -1 by level width, 0 never, 1 always
    int wf_prefetch = 1;    // wavefront-packed solves prefetch the next slice's records into shared memory (k_wf_pf)
};

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    CtxOptions opt;
    int profiling = 0;
    std::string prof_prefix;   // only kernels whose name starts with it are timed
    int64_t launches = 0;
    std::vector<ProfRec> pending;
    std::vector<cudaEvent_t> event_pool;
    struct Acc { std::string name; int64_t n = 0; double ms = 0, bytes = 0; };
    std::vector<Acc> acc;
    // scratch
    void* cub_tmp = nullptr;
    size_t cub_tmp_bytes = 0;
    int* d_scalar_i = nullptr;     // small device int scratch (64 ints)
    double* d_scalar_d = nullptr;  // small device double scratch (4096 doubles)
    double* h_pinned = nullptr;    // pinned host scratch (4096 doubles)
    // caching allocator: device blocks are recycled in stream order on this
    // context's stream and only returned to the driver when the cache is
    // trimmed (driver allocation calls can block the host for a long time)
    std::multimap<size_t, void*> free_blocks;
    std::unordered_map<void*, size_t> block_size;
    size_t cached_bytes = 0;
    std::mutex alloc_mu;

    void* alloc(size_t bytes);
    void free(void* p);
    void trim_cache();             // synchronises the stream, releases cached blocks
    void* cub_scratch(size_t bytes);
    cudaEvent_t get_event();
    void flush_profile();
    // spin-limit flag of the sync-free triangular solves (d_scalar_i[8]):
    // entry points that run solves post an async read-back; the next entry
    // point (or edfa_ctx_sync) raises it once the copy has landed
    int* h_trsv_err = nullptr;     // pinned
    cudaEvent_t trsv_ev = nullptr;
    bool trsv_pending = false;
    void trsv_err_post();          // enqueue the flag's read-back (no host wait)
    void trsv_err_poll();          // raise a landed flag (no host wait)
    void trsv_err_check();         // synchronise, raise and clear
    void trsv_err_reset();         // drop any stale flag before a new solve
};

// RAII guard for library-owned device allocations
template <class T>
struct DevBuf {
    Ctx* ctx = nullptr;
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(Ctx* c, size_t count) { reset(c, count); }
    void reset(Ctx* c, size_t count) {
        release();
        ctx = c;
        n = count;
        p = count ? static_cast<T*>(c->alloc(count * sizeof(T))) : nullptr;
    }
    void release() {
        if (p && ctx) ctx->free(p);
        p = nullptr;
        n = 0;
    }
    ~DevBuf() { release(); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : ctx(o.ctx), p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); ctx = o.ctx; p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
};

// Timed launch scope: records events around the enclosed launches when profiling.
struct Prof {
    Ctx* c;
    const char* name;
    double bytes;
    cudaEvent_t e0 = nullptr;
    bool on = false;
    Prof(Ctx* ctx, const char* nm, double b) : c(ctx), name(nm), bytes(b) {
        c->launches++;
        on = c->profiling && (c->prof_prefix.empty() || strncmp(nm, c->prof_prefix.c_str(), c->prof_prefix.size()) == 0);
        if (on) {
            e0 = c->get_event();
            cudaEventRecord(e0, c->stream);
        }
    }
    ~Prof() {
        if (on) {
            cudaEvent_t e1 = c->get_event();
            cudaEventRecord(e1, c->stream);
            c->pending.push_back({name, e0, e1, bytes});
        }
    }
};

// Host-side phase timer (EDFA_PHASE_TIMING=1): synchronises the stream at
// both ends and prints the phase's wall time -- diagnostics only.
struct PhaseTimer {
    Ctx* c;
    const char* name;
    double t0 = 0;
    bool on;
    static bool enabled() {
        static const bool e = getenv("EDFA_PHASE_TIMING") != nullptr;
        return e;
    }
    static double now() {
        timespec ts;
        clock_gettime(CLOCK_MONOTONIC, &ts);
        return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
    }
    PhaseTimer(Ctx* ctx, const char* nm) : c(ctx), name(nm), on(enabled()) {
        if (on) {
            cudaStreamSynchronize(c->stream);
            t0 = now();
        }
    }
    ~PhaseTimer() {
        if (on) {
            cudaStreamSynchronize(c->stream);
            fprintf(stderr, "[edfa phase] %-28s %9.3f ms\n", name, now() - t0);
        }
    }
};

inline void check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Error(EDFA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------- CSR
struct Csr {
    int32_t n_rows = 0, n_cols = 0;
    int64_t nnz = 0;
    DevBuf<int32_t> ptr, idx;
    DevBuf<double> val;   // may be empty for pattern-only matrices
};

// SELL-32: slices of 32 consecutive rows, entries column-major inside a slice
// (row r's k-th entry at slice_ptr[r/32] + 32*k + r%32), padded with zeros
struct Sell {
    int32_t n_rows = 0, n_cols = 0;
    int64_t nnz = 0, stored = 0;
    int32_t uniform_w = 0;       // > 0: every slice stores exactly this many entries per row
    DevBuf<int64_t> slice_ptr;   // n_slices + 1
    DevBuf<int32_t> col;
    DevBuf<double> val;
};

// light view passed to kernels
struct CsrV {
    int32_t n_rows, n_cols;
    const int32_t* __restrict__ ptr;
    const int32_t* __restrict__ idx;
    const double* __restrict__ val;
};
inline CsrV view(const Csr& A) {
    return CsrV{A.n_rows, A.n_cols, A.ptr.p, A.idx.p, A.val.p};
}

constexpr int WARP = 32;
constexpr int NUM_SMS_B200 = 148;

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// ---------------------------------------------------------------- helpers (sparse_util.cu)
// exclusive scan of int32 counts into int32 row pointers; returns total (syncs)
int64_t scan_counts(Ctx* c, const int32_t* counts, int32_t* ptr_out, int32_t n);
// CSR transpose (sorted rows in the output), values optional
void transpose(Ctx* c, const Csr& A, Csr& AT);
// monolithic block matrix [[A, B], [C, D]]
void block_merge(Ctx* c, const Csr& A, const Csr& B, const Csr& C, const Csr& D, Csr& M);
// y = alpha*A x + beta*y
void spmv(Ctx* c, const CsrV& A, int64_t nnz, const double* x, double* y, double alpha, double beta,
          const char* name = "spmv");
void build_sell(Ctx* c, const Csr& A, Sell& S);
void spmv_sell(Ctx* c, const Sell& A, const double* x, double* y, double alpha, double beta, const char* name);
// S = A - H (row-wise sorted merge, exact zeros dropped, optional row filter)
void csr_sub(Ctx* c, const Csr& A, const Csr& H, double tau, Csr& S);
// row filter (filter_rows, precond.py:138-157): drop |v| < tau*||row||_2 off-diagonal
void csr_filter(Ctx* c, const Csr& A, double tau, Csr& out, bool keep_diag = true);
void copy_csr(Ctx* c, const Csr& A, Csr& out);
void fill(Ctx* c, double* p, int64_t n, double v);
void fill_bits(Ctx* c, double* p, int64_t n, unsigned long long bits);

int set_error(int code, const std::string& msg);

}  // namespace edfa

#define API_BEGIN try {
#define API_END                                                                      \
    }                                                                                \
    catch (const edfa::Error& e) { return edfa::set_error(e.code, e.what()); }       \
    catch (const std::exception& e) { return edfa::set_error(EDFA_ERR_CUDA, e.what()); } \
    return EDFA_OK;

// ---------------------------------------------------------------- opaque handles
struct edfa_ctx { edfa::Ctx c; };
// owning handle (own) or borrowed view of a library-internal matrix (m)
struct edfa_csr {
    edfa::Ctx* ctx = nullptr;
    edfa::Csr own;
    const edfa::Csr* m = nullptr;
};
