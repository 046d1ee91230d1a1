// Context: stream, stream-ordered allocator, scratch, per-kernel event timing.
#include <algorithm>
#include <cstring>

#include "edfa_internal.cuh"

namespace edfa {

double slow_log_ms() {
    static const double v = [] {
        const char* e = getenv("EDFA_SLOW_LOG");
        return e ? atof(e) : 0.0;
    }();
    return v;
}
void slow_log(double ms, const char* what, const char* file, int line) {
    fprintf(stderr, "[edfa slow] %8.2f ms  %s:%d  %s\n", ms, file, line, what);
}

namespace {
// The idle cache is trimmed only when it outgrows 70 % of the device memory (at
// least 48 GiB): a time-step loop that frees one preconditioner and builds the
// next of the same shape then reuses every block instead of paying cudaFree +
// cudaMalloc per system (256^3: ~0.3 s per system).  An allocation that fails
// still hands the whole cache back and retries (alloc).
size_t cache_limit() {
    static const size_t v = [] {
        size_t fr = 0, tot = 0;
        if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) { cudaGetLastError(); tot = 0; }
        return std::max(size_t(48) << 30, tot / 10 * 7);
    }();
    return v;
}

size_t round_block(size_t bytes) {
    if (bytes <= (size_t(1) << 20)) return (bytes + 511) & ~size_t(511);
    return (bytes + (size_t(1) << 20) - 1) & ~((size_t(1) << 20) - 1);
}
}  // namespace

void Ctx::trim_cache() {
    std::lock_guard<std::mutex> lk(alloc_mu);
    if (free_blocks.empty()) return;
    cudaStreamSynchronize(stream);
    for (auto& kv : free_blocks) {
        block_size.erase(kv.second);
        cudaFree(kv.second);
    }
    free_blocks.clear();
    cached_bytes = 0;
}

void* Ctx::alloc(size_t bytes) {
    if (bytes == 0) return nullptr;
    const size_t sz = round_block(bytes);
    {
        std::lock_guard<std::mutex> lk(alloc_mu);
        auto it = free_blocks.lower_bound(sz);
        if (it != free_blocks.end() && it->first <= sz + sz / 8 + (size_t(1) << 20)) {
            void* p = it->second;
            cached_bytes -= it->first;
            free_blocks.erase(it);
            return p;
        }
    }
    void* p = nullptr;
    const double lim = slow_log_ms(), t0 = lim > 0 ? host_ms() : 0.0;
    cudaError_t e = cudaMalloc(&p, sz);
    if (e != cudaSuccess) {                 // give the cache back and retry once
        cudaGetLastError();
        trim_cache();
        e = cudaMalloc(&p, sz);
    }
    if (lim > 0 && host_ms() - t0 > lim) slow_log(host_ms() - t0, "cudaMalloc", __FILE__, __LINE__);
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw Error(EDFA_ERR_CUDA, std::string("device allocation of ") + std::to_string(bytes) +
                                       " bytes failed: " + cudaGetErrorString(e));
    }
    std::lock_guard<std::mutex> lk(alloc_mu);
    block_size[p] = sz;
    return p;
}

void Ctx::free(void* p) {
    if (!p) return;
    bool trim = false;
    {
        std::lock_guard<std::mutex> lk(alloc_mu);
        auto it = block_size.find(p);
        if (it == block_size.end()) return;   // not ours
        free_blocks.emplace(it->second, p);   // reusable in stream order
        cached_bytes += it->second;
        trim = cached_bytes > cache_limit();
    }
    if (trim) trim_cache();
}

void* Ctx::cub_scratch(size_t bytes) {
    if (bytes > cub_tmp_bytes) {
        if (cub_tmp) free(cub_tmp);
        cub_tmp_bytes = std::max(bytes, size_t(1) << 20);
        cub_tmp = alloc(cub_tmp_bytes);
    }
    return cub_tmp;
}

cudaEvent_t Ctx::get_event() {
    if (event_pool.empty()) {
        cudaEvent_t e;
        EDFA_CUDA(cudaEventCreate(&e));
        return e;
    }
    cudaEvent_t e = event_pool.back();
    event_pool.pop_back();
    return e;
}

void Ctx::flush_profile() {
    if (pending.empty()) return;
    EDFA_CUDA(cudaStreamSynchronize(stream));
    for (auto& r : pending) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.t0, r.t1);
        auto it = std::find_if(acc.begin(), acc.end(), [&](const Acc& a) { return a.name == r.name; });
        if (it == acc.end()) {
            acc.push_back(Acc{r.name});
            it = acc.end() - 1;
        }
        it->n += 1;
        it->ms += ms;
        it->bytes += r.bytes;
        event_pool.push_back(r.t0);
        event_pool.push_back(r.t1);
    }
    pending.clear();
}

}  // namespace edfa

using namespace edfa;

static thread_local std::string g_last_error;

namespace edfa {
int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}
}  // namespace edfa


void Ctx::trsv_err_post() {
    EDFA_CUDA(cudaMemcpyAsync(h_trsv_err, d_scalar_i + 8, sizeof(int), cudaMemcpyDeviceToHost, stream));
    EDFA_CUDA(cudaEventRecord(trsv_ev, stream));
    trsv_pending = true;
}

static void raise_trsv(Ctx* c) {
    *c->h_trsv_err = 0;
    c->trsv_pending = false;
    EDFA_CUDA(cudaMemsetAsync(c->d_scalar_i + 8, 0, sizeof(int), c->stream));
    throw Error(EDFA_ERR_CUDA, "triangular solve exceeded its spin limit (dependency never published)");
}

void Ctx::trsv_err_poll() {
    if (!trsv_pending) return;
    const cudaError_t q = cudaEventQuery(trsv_ev);
    if (q == cudaErrorNotReady) return;
    EDFA_CUDA(q);
    trsv_pending = false;
    if (*h_trsv_err) raise_trsv(this);
}

void Ctx::trsv_err_check() {
    EDFA_CUDA(cudaMemcpyAsync(h_trsv_err, d_scalar_i + 8, sizeof(int), cudaMemcpyDeviceToHost, stream));
    EDFA_CUDA(cudaStreamSynchronize(stream));
    trsv_pending = false;
    if (*h_trsv_err) raise_trsv(this);
}

void Ctx::trsv_err_reset() {
    trsv_pending = false;
    *h_trsv_err = 0;
    EDFA_CUDA(cudaMemsetAsync(d_scalar_i + 8, 0, sizeof(int), stream));
}

extern "C" {

int edfa_abi_version(void) { return EDFA_ABI_VERSION; }

const char* edfa_last_error(void) { return g_last_error.c_str(); }

int edfa_ctx_create(int device, void* stream, edfa_ctx** out) {
    API_BEGIN
    require(out != nullptr, EDFA_ERR_VALUE, "out is NULL");
    EDFA_CUDA(cudaSetDevice(device));
    auto* h = new edfa_ctx();
    h->c.device = device;
    h->c.stream = static_cast<cudaStream_t>(stream);
    // algorithm selections: read from the environment once, here
    auto env_opt = [](const char* name, int dflt) {
        const char* e = getenv(name);
        return e ? atoi(e) : dflt;
    };
    h->c.opt.ic_pair = env_opt("EDFA_OPT_IC_PAIR", 1);
    h->c.opt.fill_fusion = env_opt("EDFA_OPT_FILL_FUSION", 1);
    h->c.opt.trsv_levels = env_opt("EDFA_OPT_TRSV_LEVELS", 0);
    h->c.opt.ilu_levels = env_opt("EDFA_OPT_ILU_LEVELS", 0);
    h->c.opt.tile_direct = env_opt("EDFA_OPT_TILE_DIRECT", -1);
    h->c.opt.ilu_wf = env_opt("EDFA_OPT_ILU_WF", -1);
    h->c.opt.wf_prefetch = env_opt("EDFA_OPT_WF_PREFETCH", 1);
    h->c.d_scalar_i = static_cast<int*>(h->c.alloc(64 * sizeof(int)));
    EDFA_CUDA(cudaMemsetAsync(h->c.d_scalar_i, 0, 64 * sizeof(int), h->c.stream));   // [60]: reduction ticket
    h->c.d_scalar_d = static_cast<double*>(h->c.alloc(4096 * sizeof(double)));
    EDFA_CUDA(cudaMallocHost(&h->c.h_pinned, 4096 * sizeof(double)));
    EDFA_CUDA(cudaMallocHost(&h->c.h_trsv_err, sizeof(int)));
    *h->c.h_trsv_err = 0;
    EDFA_CUDA(cudaEventCreateWithFlags(&h->c.trsv_ev, cudaEventDisableTiming));
    *out = h;
    API_END
}

int edfa_ctx_set_stream(edfa_ctx* ctx, void* stream) {
    API_BEGIN
    require(ctx, EDFA_ERR_VALUE, "ctx is NULL");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (s != ctx->c.stream) {
        // cached blocks are recycled in the order of one stream: drain it first
        EDFA_CUDA(cudaStreamSynchronize(ctx->c.stream));
        ctx->c.stream = s;
    }
    API_END
}

int edfa_ctx_set_option(edfa_ctx* ctx, const char* name, int value) {
    API_BEGIN
    require(ctx && name, EDFA_ERR_VALUE, "ctx or name is NULL");
    CtxOptions& o = ctx->c.opt;
    const std::string n = name;
    if (n == "ic_pair") o.ic_pair = value;
    else if (n == "fill_fusion") o.fill_fusion = value;
    else if (n == "trsv_levels") o.trsv_levels = value;
    else if (n == "ilu_levels") o.ilu_levels = value;
    else if (n == "tile_direct") o.tile_direct = value;
    else if (n == "ilu_wf") o.ilu_wf = value;
    else if (n == "wf_prefetch") o.wf_prefetch = value;
    else throw Error(EDFA_ERR_VALUE, "unknown option '" + n + "'");
    API_END
}

int edfa_ctx_get_option(edfa_ctx* ctx, const char* name, int* value) {
    API_BEGIN
    require(ctx && name && value, EDFA_ERR_VALUE, "ctx, name or value is NULL");
    const CtxOptions& o = ctx->c.opt;
    const std::string n = name;
    if (n == "ic_pair") *value = o.ic_pair;
    else if (n == "fill_fusion") *value = o.fill_fusion;
    else if (n == "trsv_levels") *value = o.trsv_levels;
    else if (n == "ilu_levels") *value = o.ilu_levels;
    else if (n == "tile_direct") *value = o.tile_direct;
    else if (n == "ilu_wf") *value = o.ilu_wf;
    else if (n == "wf_prefetch") *value = o.wf_prefetch;
    else throw Error(EDFA_ERR_VALUE, "unknown option '" + n + "'");
    API_END
}

int edfa_ctx_trim(edfa_ctx* ctx) {
    API_BEGIN
    require(ctx, EDFA_ERR_VALUE, "ctx is NULL");
    ctx->c.trim_cache();
    API_END
}

int edfa_ctx_sync(edfa_ctx* ctx) {
    API_BEGIN
    ctx->c.trsv_err_check();   // synchronises; raises a solve that hit its spin limit
    API_END
}

int edfa_ctx_destroy(edfa_ctx* ctx) {
    API_BEGIN
    if (!ctx) return EDFA_OK;
    Ctx& c = ctx->c;
    cudaStreamSynchronize(c.stream);
    c.flush_profile();
    for (auto e : c.event_pool) cudaEventDestroy(e);
    c.free(c.cub_tmp);
    c.free(c.d_scalar_i);
    c.free(c.d_scalar_d);
    cudaFreeHost(c.h_pinned);
    cudaFreeHost(c.h_trsv_err);
    cudaEventDestroy(c.trsv_ev);
    cudaStreamSynchronize(c.stream);
    c.trim_cache();
    delete ctx;
    API_END
}

int edfa_ctx_profile(edfa_ctx* ctx, int enable) {
    API_BEGIN
    ctx->c.flush_profile();
    ctx->c.profiling = enable;
    API_END
}

int edfa_ctx_profile_filter(edfa_ctx* ctx, const char* prefix) {
    API_BEGIN
    ctx->c.flush_profile();
    ctx->c.prof_prefix = prefix ? prefix : "";
    API_END
}

int64_t edfa_ctx_profile_report(edfa_ctx* ctx, char* buf, int64_t cap, int reset) {
    try {
        ctx->c.flush_profile();
        std::string s = "{";
        bool first = true;
        for (auto& a : ctx->c.acc) {
            char line[512];
            snprintf(line, sizeof line, "%s\"%s\": {\"launches\": %lld, \"ms\": %.6f, \"bytes\": %.1f}",
                     first ? "" : ", ", a.name.c_str(), (long long)a.n, a.ms, a.bytes);
            s += line;
            first = false;
        }
        s += "}";
        if (buf && cap > 0) {
            int64_t n = std::min<int64_t>(cap - 1, (int64_t)s.size());
            memcpy(buf, s.data(), n);
            buf[n] = 0;
        }
        if (reset) ctx->c.acc.clear();
        return (int64_t)s.size() + 1;
    } catch (const std::exception& e) {
        edfa::set_error(EDFA_ERR_CUDA, e.what());
        return -1;
    }
}

int64_t edfa_ctx_launch_count(edfa_ctx* ctx) { return ctx ? ctx->c.launches : -1; }

}  // extern "C"
