// K8: sync-free, level-ordered triangular solves (InnerFactorization.apply,
// hx/sparse.py:125-129) and the plan construction they need.
//
// Plan: dependency levels are computed once on the device (sync-free, one
// thread per row); rows are sorted by level and each level is padded to whole
// warps, so a warp never waits on itself; coefficients are stored SELL-32
// (column-major inside 32-row slices) so every coefficient load is coalesced.
// Solve: warps take slices in level order from an atomic ticket (deadlock-free
// without relying on block scheduling order), each thread polls the solution
// entries its row depends on -- the solution vector is sentinel-initialised,
// so the value is its own ready flag -- and publishes its own entry.
#include <cub/cub.cuh>
#include <climits>

#include "dev_util.cuh"
#include "edfa_internal.cuh"
#include "objects.cuh"

namespace edfa {
namespace {

constexpr int LEVEL_UNSET = -1;

// level[i] = 1 + max(level[j], j in deps(i)); rows visited in dependency order
__global__ void k_levels(CsrV D, bool reverse, int* __restrict__ level, int* __restrict__ ticket,
                         int* __restrict__ max_level, int* __restrict__ err) {
    __shared__ int base[8];
    int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) base[wid] = atomicAdd(ticket, 1) * 32;
    __syncwarp();
    int t = base[wid] + lane;
    if (t >= D.n_rows) return;
    int i = reverse ? D.n_rows - 1 - t : t;
    int lv = 0;
    for (int e = D.ptr[i]; e < D.ptr[i + 1]; ++e) {
        int j = D.idx[e];
        int v = ld_relaxed_i(level + j);
        long long spins = 0;
        unsigned ns = 32;
        while (v == LEVEL_UNSET) {   // back off: thousands of pollers share the L2
            if (++spins > SPIN_LIMIT) { atomicExch(err, 1); v = 0; break; }
            __nanosleep(ns);
            if (ns < 512) ns <<= 1;
            v = ld_relaxed_i(level + j);
        }
        lv = max(lv, v + 1);
    }
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(level + i), "r"(lv) : "memory");
    atomicMax(max_level, lv);
}

__global__ void k_fill_int(int* p, int64_t n, int v) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}
__global__ void k_iota_i(int* p, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = i;
}
__global__ void k_level_hist(const int* __restrict__ level, int n, int* __restrict__ cnt) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) atomicAdd(&cnt[level[i]], 1);
}
__global__ void k_pad_counts(const int* __restrict__ cnt, int nl, int* __restrict__ pcnt) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nl) pcnt[i] = (cnt[i] + 31) & ~31;
}
// perm[pstart[L] + (t - ustart[L])] = row
__global__ void k_scatter_perm(const int* __restrict__ skeys, const int* __restrict__ srows, int n,
                               const int* __restrict__ ustart, const int* __restrict__ pstart,
                               int* __restrict__ perm) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    int L = skeys[t];
    perm[pstart[L] + (t - ustart[L])] = srows[t];
}
__global__ void k_slice_width(const int* __restrict__ perm, int n_slices, const int32_t* __restrict__ dptr,
                              int64_t* __restrict__ wbytes) {
    int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (s >= n_slices) return;
    int r = perm[s * 32 + lane];
    int len = r >= 0 ? dptr[r + 1] - dptr[r] : 0;
    len = warp_max(len);
    if (lane == 0) wbytes[s] = (int64_t)len * 32;
}
__global__ void k_max_width(const int64_t* __restrict__ sptr, int n_slices, int* __restrict__ out) {
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < n_slices) atomicMax(out, (int)((sptr[s + 1] - sptr[s]) / 32));
}

__global__ void k_fill_sell(const int* __restrict__ perm, int n_slices, CsrV D, const int64_t* __restrict__ sptr,
                            int32_t* __restrict__ col, double* __restrict__ val, const double* __restrict__ diag,
                            bool unit, double* __restrict__ dinv) {
    int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (s >= n_slices) return;
    int r = perm[s * 32 + lane];
    int64_t b = sptr[s];
    int w = (int)((sptr[s + 1] - b) / 32);
    int e0 = r >= 0 ? D.ptr[r] : 0, len = r >= 0 ? D.ptr[r + 1] - e0 : 0;
    for (int k = 0; k < w; ++k) {
        bool live = k < len;
        if (col) col[b + (int64_t)k * 32 + lane] = live ? D.idx[e0 + k] : -1;
        if (val) val[b + (int64_t)k * 32 + lane] = live && D.val ? D.val[e0 + k] : 0.0;
    }
    if (dinv) dinv[s * 32 + lane] = (r < 0 || unit) ? 1.0 : 1.0 / diag[r];
}

struct SolveArgs {
    const int* perm;
    const int64_t* sptr;
    const int32_t* col;
    const double* val;
    const double* dinv;
    const int* slice_level;
    const int* level_slices;
    int* sync;            // done[n_levels], ticket, finished
    int n_levels;
    int n_slices;
    const double* b;
    double alpha;
    double* x;
    const double* add;
    double* out2;
    int* err;
};

__device__ __forceinline__ void wait_level(const int* done, int L, int need, int* err) {
    // one lane per warp polls the per-level completion counter with backoff
    if (L < 0) return;
    unsigned ns = 16;
    long long spins = 0;
    while (ld_acquire(done + L) < need) {
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
        if (++spins > SPIN_LIMIT) { atomicExch(err, 2); return; }
    }
}

// Level-counter synchronisation: a slice of level L starts once every slice
// of level L-1 has finished; by induction all earlier levels are complete,
// so dependencies are read without per-entry polling.  The last warp to
// finish resets the counters for the next launch (no memset between solves).
template <int U>
__global__ void __launch_bounds__(256) k_trsv(SolveArgs a) {
    __shared__ int base[8];
    int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int* done = a.sync;
    if (lane == 0) base[wid] = atomicAdd(a.sync + a.n_levels, 1);
    __syncwarp();
    int s = base[wid];
    if (s >= a.n_slices) return;
    int L = a.slice_level[s];
    if (lane == 0 && L > 0) wait_level(done, L - 1, a.level_slices[L - 1], a.err);
    __syncwarp();
    int slot = s * 32 + lane;
    int r = a.perm[slot];
    if (r >= 0) {
        int64_t b0 = a.sptr[s];
        int w = (int)((a.sptr[s + 1] - b0) / 32);
        double acc = a.alpha * __ldg(a.b + r);
        const int32_t* cp = a.col + b0 + lane;
        const double* vp = a.val + b0 + lane;
        for (int k0 = 0; k0 < w; k0 += U) {
            int c[U];
            double v[U], xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                bool in = k0 + u < w;
                c[u] = in ? __ldg(cp + (int64_t)(k0 + u) * 32) : -1;
                v[u] = in ? __ldg(vp + (int64_t)(k0 + u) * 32) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) xv[u] = c[u] >= 0 ? __ldcg(a.x + c[u]) : 0.0;
#pragma unroll
            for (int u = 0; u < U; ++u) acc = fma(-v[u], xv[u], acc);
        }
        double xr = acc * a.dinv[slot];
        __stcg(a.x + r, xr);
        if (a.out2) a.out2[r] = xr + a.add[r];
    }
    __syncwarp();
    if (lane == 0) {
        __threadfence();
        atomicAdd(done + L, 1);
        int f = atomicAdd(a.sync + a.n_levels + 1, 1);
        if (f == a.n_slices - 1) {           // last slice of the solve: reset
            for (int l = 0; l < a.n_levels; ++l) done[l] = 0;
            a.sync[a.n_levels] = 0;
            a.sync[a.n_levels + 1] = 0;
            __threadfence();
        }
    }
}

struct LsArgs {
    const int* perm;
    const int64_t* sptr;
    const int32_t* col;
    const double* val;
    const double* dinv;
    const int* level_start;
    int n_levels;
    unsigned* bar;        // [count, generation]
    const double* b;
    double alpha;
    double* x;
    const double* add;
    double* out2;
};

// Level-synchronous persistent solve: all co-resident warps sweep the slices
// of one level, then a software grid barrier; no per-entry polling.
// Row data of one slot, prefetched before the grid barrier that precedes its
// level: only the gather of already-final x entries remains on the critical path.
template <int K>
struct RowPre {
    int r, w;
    int64_t b0;
    int c[K];
    double v[K];
    double bias, dinv;
};

template <int K>
__device__ __forceinline__ void row_prefetch(const LsArgs& a, int s, int lane, RowPre<K>& p) {
    int slot = s * 32 + lane;
    p.r = a.perm[slot];
    p.b0 = a.sptr[s];
    p.w = (int)((a.sptr[s + 1] - p.b0) / 32);
    const int32_t* cp = a.col + p.b0 + lane;
    const double* vp = a.val + p.b0 + lane;
#pragma unroll
    for (int u = 0; u < K; ++u) {
        bool in = u < p.w;
        p.c[u] = in ? __ldg(cp + (int64_t)u * 32) : -1;
        p.v[u] = in ? __ldg(vp + (int64_t)u * 32) : 0.0;
    }
    p.bias = p.r >= 0 ? a.alpha * __ldg(a.b + p.r) : 0.0;
    p.dinv = a.dinv[slot];
}

template <int K>
__device__ __forceinline__ void row_finish(const LsArgs& a, int lane, const RowPre<K>& p) {
    if (p.r < 0) return;
    double xv[K];
#pragma unroll
    for (int u = 0; u < K; ++u) xv[u] = p.c[u] >= 0 ? __ldcg(a.x + p.c[u]) : 0.0;
    double acc = p.bias;
#pragma unroll
    for (int u = 0; u < K; ++u) acc = fma(-p.v[u], xv[u], acc);
    // rows wider than K (rare): remaining entries without prefetch
    const int32_t* cp = a.col + p.b0 + lane;
    const double* vp = a.val + p.b0 + lane;
    for (int k = K; k < p.w; ++k) {
        int c = __ldg(cp + (int64_t)k * 32);
        if (c >= 0) acc = fma(-__ldg(vp + (int64_t)k * 32), __ldcg(a.x + c), acc);
    }
    double xr = acc * p.dinv;
    __stcg(a.x + p.r, xr);
    if (a.out2) a.out2[p.r] = xr + a.add[p.r];
}

template <int K>
__global__ void __launch_bounds__(256) k_trsv_ls(LsArgs a) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    RowPre<K> pre;
    bool have = false;
    {
        int s = a.level_start[0] + gw;
        if (a.n_levels > 0 && s < a.level_start[1]) { row_prefetch<K>(a, s, lane, pre); have = true; }
    }
    for (int L = 0; L < a.n_levels; ++L) {
        int s0 = a.level_start[L], s1 = a.level_start[L + 1];
        if (have) row_finish<K>(a, lane, pre);
        for (int s = s0 + gw + nw; s < s1; s += nw) {   // levels wider than the grid
            RowPre<K> q;
            row_prefetch<K>(a, s, lane, q);
            row_finish<K>(a, lane, q);
        }
        have = false;
        if (L + 1 < a.n_levels) {
            int s = s1 + gw;
            if (s < a.level_start[L + 2]) { row_prefetch<K>(a, s, lane, pre); have = true; }
            grid_barrier(a.bar, a.bar + 1, gridDim.x);
        }
    }
}

__global__ void k_slice_level(const int* __restrict__ pstart, int nl, int* __restrict__ slice_level,
                              int* __restrict__ level_slices, int* __restrict__ level_start) {
    int L = blockIdx.x * blockDim.x + threadIdx.x;
    if (L >= nl) return;
    int s0 = pstart[L] / 32, s1 = pstart[L + 1] / 32;
    level_slices[L] = s1 - s0;
    level_start[L] = s0;
    if (L == nl - 1) level_start[nl] = s1;
    for (int s = s0; s < s1; ++s) slice_level[s] = L;
}

}  // namespace

// Build the level-ordered SELL plan for deps (pattern and, optionally, values).
void build_plan(Ctx* c, const Csr& deps, const double* diag, bool unit, bool reverse, TriPlan& p, bool allow_chain,
                const int32_t* given_level, int given_levels) {
    const int n = deps.n_rows;
    p.n = n;
    p.unit = unit;
    p.is_chain = false;
    if (allow_chain && n > 0 && build_chain(c, deps, diag, unit, p.chain)) {
        p.is_chain = true;
        p.n_dep = deps.nnz;
        p.n_levels = 0;
        return;
    }
    p.n_dep = deps.nnz;
    p.ticket.reset(c, 1);
    if (n == 0) {
        p.n_slots = 0;
        p.n_levels = 0;
        p.perm.release();
        p.slice_ptr.reset(c, 1);
        EDFA_CUDA(cudaMemsetAsync(p.slice_ptr.p, 0, sizeof(int64_t), c->stream));
        return;
    }
    DevBuf<int> level_own, rows(c, n), skeys(c, n), srows(c, n);
    const int* level_p = given_level;
    int nl = given_levels;
    if (!given_level) {
        level_own.reset(c, n);
        int* scal = c->d_scalar_i + 16;   // [ticket, max_level, err]
        EDFA_CUDA(cudaMemsetAsync(scal, 0, 3 * sizeof(int), c->stream));
        {
            Prof pr(c, "trsv_levels", 4.0 * deps.nnz + 8.0 * n);
            k_fill_int<<<ceil_div(n, 256), 256, 0, c->stream>>>(level_own.p, n, LEVEL_UNSET);
            k_levels<<<ceil_div(n, 256), 256, 0, c->stream>>>(view(deps), reverse, level_own.p, scal, scal + 1,
                                                               scal + 2);
            check_launch("k_levels");
        }
        int hs[3];
        EDFA_CUDA(cudaMemcpyAsync(hs, scal, sizeof hs, cudaMemcpyDeviceToHost, c->stream));
        EDFA_CUDA(cudaStreamSynchronize(c->stream));
        require(hs[2] == 0, EDFA_ERR_CUDA, "level computation did not converge (dependency cycle?)");
        nl = hs[1] + 1;
        level_p = level_own.p;
    }
    p.n_levels = nl;
    struct { const int* p; } level{level_p};
    // sort rows by level (stable: natural order inside a level)
    k_iota_i<<<ceil_div(n, 256), 256, 0, c->stream>>>(rows.p, n);
    int bits = 1;
    while ((1 << bits) <= nl) ++bits;
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, level.p, skeys.p, rows.p, srows.p, n, 0, bits, c->stream);
    EDFA_CUDA(cub::DeviceRadixSort::SortPairs(c->cub_scratch(bytes), bytes, level.p, skeys.p, rows.p, srows.p, n, 0,
                                              bits, c->stream));
    DevBuf<int> cnt(c, nl), pcnt(c, nl), ustart(c, nl + 1), pstart(c, nl + 1);
    EDFA_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int) * nl, c->stream));
    k_level_hist<<<ceil_div(n, 256), 256, 0, c->stream>>>(level.p, n, cnt.p);
    k_pad_counts<<<ceil_div(nl, 256), 256, 0, c->stream>>>(cnt.p, nl, pcnt.p);
    check_launch("level hist");
    scan_counts(c, cnt.p, ustart.p, nl);
    int64_t slots = scan_counts(c, pcnt.p, pstart.p, nl);
    p.n_slots = (int32_t)slots;
    p.perm.reset(c, slots);
    k_fill_int<<<ceil_div(slots, 256), 256, 0, c->stream>>>(p.perm.p, slots, -1);
    k_scatter_perm<<<ceil_div(n, 256), 256, 0, c->stream>>>(skeys.p, srows.p, n, ustart.p, pstart.p, p.perm.p);
    check_launch("k_scatter_perm");
    int n_slices = (int)(slots / 32);
    p.slice_level.reset(c, std::max(n_slices, 1));
    p.level_slices.reset(c, nl);
    p.level_start.reset(c, nl + 1);
    k_slice_level<<<ceil_div(nl, 128), 128, 0, c->stream>>>(pstart.p, nl, p.slice_level.p, p.level_slices.p,
                                                           p.level_start.p);
    check_launch("k_slice_level");
    p.sync.reset(c, (size_t)nl + 2);
    EDFA_CUDA(cudaMemsetAsync(p.sync.p, 0, sizeof(int) * (nl + 2), c->stream));
    sell_on_layout(c, p.perm.p, n_slices, deps, diag, unit, p.slice_ptr, p.col, p.val, p.dinv, p.n_stored, p.max_w);
}

// SELL-32 storage of deps' rows on a given slot layout (perm: slot -> row, -1 pad)
void sell_on_layout(Ctx* c, const int32_t* perm, int n_slices, const Csr& deps, const double* diag, bool unit,
                    DevBuf<int64_t>& slice_ptr, DevBuf<int32_t>& col, DevBuf<double>& val, DevBuf<double>& dinv,
                    int64_t& n_stored, int32_t& max_w) {
    const int64_t slots = (int64_t)n_slices * 32;
    DevBuf<int64_t> wb(c, (size_t)n_slices + 1);
    k_slice_width<<<ceil_div((int64_t)n_slices * 32, 256), 256, 0, c->stream>>>(perm, n_slices, deps.ptr.p, wb.p);
    check_launch("k_slice_width");
    slice_ptr.reset(c, (size_t)n_slices + 1);
    {
        size_t b2 = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, b2, wb.p, slice_ptr.p, n_slices + 1, c->stream);
        EDFA_CUDA(cudaMemsetAsync(wb.p + n_slices, 0, sizeof(int64_t), c->stream));
        EDFA_CUDA(cub::DeviceScan::ExclusiveSum(c->cub_scratch(b2), b2, wb.p, slice_ptr.p, n_slices + 1, c->stream));
    }
    int64_t stored = 0;
    int* mw = c->d_scalar_i + 19;
    EDFA_CUDA(cudaMemsetAsync(mw, 0, sizeof(int), c->stream));
    k_max_width<<<ceil_div(n_slices, 256), 256, 0, c->stream>>>(slice_ptr.p, n_slices, mw);
    check_launch("k_max_width");
    int hmw = 0;
    EDFA_CUDA(cudaMemcpyAsync(&stored, slice_ptr.p + n_slices, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaMemcpyAsync(&hmw, mw, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
    n_stored = stored;
    max_w = hmw;
    col.reset(c, std::max<int64_t>(stored, 1));
    val.reset(c, std::max<int64_t>(stored, 1));
    dinv.reset(c, std::max<int64_t>(slots, 1));
    Prof pr(c, "trsv_plan", 12.0 * stored + 8.0 * slots);
    k_fill_sell<<<ceil_div((int64_t)n_slices * 32, 256), 256, 0, c->stream>>>(
        perm, n_slices, view(deps), slice_ptr.p, col.p, deps.val.p ? val.p : nullptr, diag, unit,
        diag || unit ? dinv.p : nullptr);
    check_launch("k_fill_sell");
}

// (Re)load coefficient values and diagonal of an existing plan from deps.
void plan_values(Ctx* c, const Csr& deps, const double* diag, TriPlan& p) {
    if (p.is_chain) {
        chain_values(c, deps, diag, p.chain);
        return;
    }
    int n_slices = p.n_slots / 32;
    if (n_slices == 0) return;
    Prof pr(c, "trsv_plan", 20.0 * p.n_stored);
    k_fill_sell<<<ceil_div((int64_t)n_slices * 32, 256), 256, 0, c->stream>>>(
        p.perm.p, n_slices, view(deps), p.slice_ptr.p, nullptr, p.val.p, diag, p.unit, p.dinv.p);
    check_launch("k_fill_sell values");
}

// Sync-free solve for plans with wide rows (e.g. the Schur factors of dynamic
// patterns on distorted grids, ~70 dependencies per row): one warp per row,
// rows taken from a ticket in level order (topological, so a warp only waits
// on rows held by running warps), lanes gather the row's dependencies in
// parallel and poll each one on the solution vector itself (SENTINEL-filled:
// a stored value is its own ready flag), a warp reduction, one store.  No
// grid barrier per level; the hand-off is one L2 round trip.
__global__ void __launch_bounds__(256) k_trsv_wsf(const int* __restrict__ perm, const int64_t* __restrict__ sptr,
                                                  const int32_t* __restrict__ col, const double* __restrict__ val,
                                                  const double* __restrict__ dinv, int n_slots, int* ticket,
                                                  const double* __restrict__ b, double alpha, double* x,
                                                  const double* __restrict__ add, double* __restrict__ out2,
                                                  int* err) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        int slot = 0;
        if (lane == 0) slot = atomicAdd(ticket, 1);
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if (slot >= n_slots) break;
        const int r = perm[slot];
        if (r < 0) continue;
        const int s = slot >> 5, rr = slot & 31;
        const int64_t b0 = sptr[s];
        const int w = (int)((sptr[s + 1] - b0) / 32);
        // pass 1: every lane loads its coefficients and the current values of
        // its dependencies (most are final long before the row is taken); the
        // missing dependency nearest to the row -- for natural-order stencils
        // the last one to finish -- is polled by one lane, the others are
        // re-read only if they were missing too
        constexpr int PL = 4;                       // entries per lane held in registers
        double acc = 0.0;
        if (w <= 32 * PL) {
            int cc[PL];
            double vv[PL], xv[PL];
            int near = INT_MAX, near_u = -1;
#pragma unroll
            for (int u = 0; u < PL; ++u) {
                const int k = lane + 32 * u;
                cc[u] = k < w ? __ldg(col + b0 + 32 * (int64_t)k + rr) : -1;
                vv[u] = cc[u] >= 0 ? __ldg(val + b0 + 32 * (int64_t)k + rr) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < PL; ++u) {
                xv[u] = cc[u] >= 0 ? ld_relaxed(x + cc[u]) : 0.0;
                if (cc[u] >= 0 && is_sentinel(xv[u]) && abs(cc[u] - r) < near) { near = abs(cc[u] - r); near_u = u; }
            }
            int best = near;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
            if (best != INT_MAX) {
                const unsigned who = __ballot_sync(0xffffffffu, near == best);
                if (lane == __ffs(who) - 1) {
#pragma unroll
                    for (int u = 0; u < PL; ++u)
                        if (u == near_u) {
                            long long spins = 0;
                            while (is_sentinel(xv[u] = ld_relaxed(x + cc[u]))) {
                                if (++spins > SPIN_LIMIT) { atomicExch(err, 3); xv[u] = 0.0; break; }
                                __nanosleep(20);
                            }
                        }
                }
                __syncwarp();
#pragma unroll
                for (int u = 0; u < PL; ++u) {
                    long long spins = 0;
                    while (cc[u] >= 0 && is_sentinel(xv[u])) {
                        if (++spins > SPIN_LIMIT) { atomicExch(err, 3); xv[u] = 0.0; break; }
                        xv[u] = ld_relaxed(x + cc[u]);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < PL; ++u) acc = fma(-vv[u], xv[u], acc);
        } else {
            for (int k = lane; k < w; k += 32) {
                const int cidx = __ldg(col + b0 + 32 * (int64_t)k + rr);
                if (cidx < 0) continue;
                const double v = __ldg(val + b0 + 32 * (int64_t)k + rr);
                double xk = ld_relaxed(x + cidx);
                long long spins = 0;
                while (is_sentinel(xk)) {
                    if (++spins > SPIN_LIMIT) { atomicExch(err, 3); xk = 0.0; break; }
                    xk = ld_relaxed(x + cidx);
                }
                acc = fma(-v, xk, acc);
            }
        }
        acc = warp_sum(acc);
        if (lane == 0) {
            const double xr = (alpha * __ldg(b + r) + acc) * dinv[slot];
            // fire-and-forget reduction performed at L2 (SENTINEL + (x - SENTINEL)):
            // visible to the polling warps sooner than a buffered store
            atomicAdd(reinterpret_cast<unsigned long long*>(x + r),
                      (unsigned long long)__double_as_longlong(publishable(xr)) - SENTINEL_BITS);
            if (out2) out2[r] = xr + add[r];
        }
    }
}

// Sync-free solve for narrow rows: one warp per 32-row slice (rows of one
// level), slices from a ticket in level order, a thread per row polls its
// dependencies on the SENTINEL-filled solution vector.  Coefficient loads are
// coalesced (SELL-32) and issued before the polls; the row arithmetic is the
// level solver's (bias first, entries in stored order) so the results are
// bitwise those of k_trsv_ls.
template <int K>
__global__ void __launch_bounds__(256) k_trsv_tsf(const int* __restrict__ perm, const int64_t* __restrict__ sptr,
                                                  const int32_t* __restrict__ col, const double* __restrict__ val,
                                                  const double* __restrict__ dinv, int n_slices, int* ticket,
                                                  const double* __restrict__ b, double alpha, double* x,
                                                  const double* __restrict__ add, double* __restrict__ out2,
                                                  int* err) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        int s = 0;
        if (lane == 0) s = atomicAdd(ticket, 1);
        s = __shfl_sync(0xffffffffu, s, 0);
        if (s >= n_slices) break;
        const int r = perm[s * 32 + lane];
        const int64_t b0 = sptr[s];
        const int w = (int)((sptr[s + 1] - b0) / 32);
        const bool act = r >= 0;   // pad lanes run along (their records hold no dependencies)
        int cc[K];
        double vv[K];
#pragma unroll
        for (int u = 0; u < K; ++u) {
            const bool in = u < w;
            cc[u] = in ? __ldg(col + b0 + (int64_t)u * 32 + lane) : -1;
            vv[u] = in ? __ldg(val + b0 + (int64_t)u * 32 + lane) : 0.0;
        }
        double acc = act ? alpha * __ldg(b + r) : 0.0;
        double xv[K];
#pragma unroll
        for (int u = 0; u < K; ++u) xv[u] = cc[u] >= 0 ? ld_relaxed(x + cc[u]) : 0.0;   // all in flight at once
        // missing dependencies are re-read as one batch per round (all loads in
        // flight, one warp vote): polling them one after the other left every
        // stale value to be re-read in sequence after the last arrival
        {
            bool miss = false;
#pragma unroll
            for (int u = 0; u < K; ++u) miss |= cc[u] >= 0 && is_sentinel(xv[u]);
            long long spins = 0;
            while (__any_sync(0xffffffffu, miss)) {
#pragma unroll
                for (int u = 0; u < K; ++u)
                    if (cc[u] >= 0 && is_sentinel(xv[u])) xv[u] = ld_relaxed(x + cc[u]);
                miss = false;
#pragma unroll
                for (int u = 0; u < K; ++u) miss |= cc[u] >= 0 && is_sentinel(xv[u]);
                if (++spins > SPIN_LIMIT) {
                    if (miss) {
                        atomicExch(err, 3);
#pragma unroll
                        for (int u = 0; u < K; ++u)
                            if (is_sentinel(xv[u])) xv[u] = 0.0;
                    }
                    break;
                }
            }
        }
#pragma unroll
        for (int u = 0; u < K; ++u) acc = fma(-vv[u], xv[u], acc);
        if (!act) continue;
        const double xr = acc * dinv[s * 32 + lane];
        atomicAdd(reinterpret_cast<unsigned long long*>(x + r),
                  (unsigned long long)__double_as_longlong(publishable(xr)) - SENTINEL_BITS);
        if (out2) out2[r] = xr + add[r];
    }
}

void run_plan(Ctx* c, const TriPlan& p, const double* b, double alpha, double* x, const double* add, double* out2,
              const char* name) {
    if (p.n == 0) return;
    if (p.is_chain) {
        run_chain(c, p.chain, b, alpha, x, add, out2, name);
        return;
    }
    if (p.is_wf) {
        run_wf_natural(c, p, b, alpha, x, add, out2, name);
        return;
    }
    if (p.is_tile) {   // ticket bookkeeping is per plan (serialised on the stream)
        run_tile(c, const_cast<TilePlan&>(p.tile), b, alpha, x, add, out2, name);
        return;
    }
    // wide rows, or levels narrow enough that a grid barrier per level costs
    // more than the rows: sync-free warp-per-row solve
    // (measured on config 3's IC at 128^3, 16k rows per level: 1.95 ms vs 4.09 ms
    // per solve pair for the level-synchronous kernel; at 64^3 1.03 vs 1.76 ms)
    if (x != b && !c->opt.trsv_levels) {
        fill_bits(c, x, p.n, SENTINEL_BITS);
        EDFA_CUDA(cudaMemsetAsync(p.ticket.p, 0, sizeof(int), c->stream));
        int* err = c->d_scalar_i + 8;   // the solve error flag check_trsv_error reads
        Prof pr(c, name, 12.0 * p.n_dep + 8.0 * p.n + 16.0 * p.n + (out2 ? 16.0 * p.n : 0.0));
        static int grid_sf = 0;
        if (!grid_sf) {
            int occ = 0;
            EDFA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_trsv_wsf, 256, 0));
            grid_sf = NUM_SMS_B200 * std::max(1, occ);
        }
        // thread per row while rows fit 32 registers' worth of dependencies and
        // levels are wide enough to fill the warps; warp per row otherwise
        const bool wide_levels = (int64_t)p.n >= 1024ll * std::max(p.n_levels, 1);
        if (p.max_w > 16 && p.max_w <= 32 && wide_levels) {
            k_trsv_tsf<32><<<grid_sf, 256, 0, c->stream>>>(p.perm.p, p.slice_ptr.p, p.col.p, p.val.p, p.dinv.p,
                                                           p.n_slots / 32, p.ticket.p, b, alpha, x, add, out2, err);
            check_launch("k_trsv_tsf");
        } else if (p.max_w > 16) {
            k_trsv_wsf<<<grid_sf, 256, 0, c->stream>>>(p.perm.p, p.slice_ptr.p, p.col.p, p.val.p, p.dinv.p,
                                                       p.n_slots, p.ticket.p, b, alpha, x, add, out2, err);
            check_launch("k_trsv_wsf");
        } else {
            k_trsv_tsf<16><<<grid_sf, 256, 0, c->stream>>>(p.perm.p, p.slice_ptr.p, p.col.p, p.val.p, p.dinv.p,
                                                           p.n_slots / 32, p.ticket.p, b, alpha, x, add, out2, err);
            check_launch("k_trsv_tsf");
        }
        return;
    }
    LsArgs a{p.perm.p, p.slice_ptr.p, p.col.p, p.val.p, p.dinv.p, p.level_start.p, p.n_levels,
             reinterpret_cast<unsigned*>(p.sync.p), b, alpha, x, add, out2};
    double bytes = 12.0 * p.n_dep + 8.0 * p.n + 16.0 * p.n + (out2 ? 16.0 * p.n : 0.0);
    Prof pr(c, name, bytes);
    static int grid = 0;
    if (!grid) {
        int occ = 0;
        EDFA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_trsv_ls<16>, 256, 0));
        grid = NUM_SMS_B200 * std::max(1, std::min(occ, 2));
    }
    void* args[] = {&a};
    EDFA_CUDA(cudaLaunchCooperativeKernel((void*)k_trsv_ls<16>, dim3(grid), dim3(256), args, 0, c->stream));
    check_launch("k_trsv");
}

}  // namespace edfa
