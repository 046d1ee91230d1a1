// Chain-structured triangular systems: when every row has at most one
// dependency and is the dependency of at most one row, the DAG is a set of
// disjoint paths ("chains").  On regular hexahedral grids the IC(0) factor of
// -A_ff is exactly that: -A_ff couples each face only with the opposite face
// of the cells it bounds, so it is tridiagonal along every grid line
// (SURVEY.md §7.3-1).  One thread walks one chain, so the dependency is a
// register, not a memory round trip; loads of the next steps are independent
// of the recurrence and stay in flight.
#include <cub/cub.cuh>

#include "dev_util.cuh"
#include "edfa_internal.cuh"
#include "objects.cuh"

namespace edfa {
namespace {

__global__ void k_chain_check(CsrV D, int* __restrict__ succ, int* __restrict__ bad) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= D.n_rows) return;
    int len = D.ptr[i + 1] - D.ptr[i];
    if (len > 1) { atomicExch(bad, 1); return; }
    if (len == 1) {
        int j = D.idx[D.ptr[i]];
        if (atomicCAS(succ + j, -1, i) != -1) atomicExch(bad, 1);
    }
}

__global__ void k_chain_heads(CsrV D, const int* __restrict__ succ, int* __restrict__ heads,
                              int* __restrict__ n_heads, int* __restrict__ lens) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= D.n_rows) return;
    if (D.ptr[i + 1] != D.ptr[i]) return;     // not a head
    int h = atomicAdd(n_heads, 1);
    heads[h] = i;
    int len = 0;
    for (int r = i; r >= 0; r = succ[r]) ++len;
    lens[h] = len;
}

// lay chain t's k-th row at  gbase[t/32] + k*32 + t%32  (SELL-32 over chains)
__global__ void k_chain_fill(CsrV D, const int* __restrict__ succ, const int* __restrict__ heads, int n_chains,
                             const int64_t* __restrict__ gbase, int* __restrict__ rows, double* __restrict__ coef,
                             double* __restrict__ dinv, const double* __restrict__ diag, bool unit) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_chains) return;
    int64_t base = gbase[t >> 5] + (t & 31);
    int64_t end = gbase[(t >> 5) + 1];
    int64_t p = base;
    for (int r = heads[t]; r >= 0; r = succ[r], p += 32) {
        rows[p] = r;
        int e = D.ptr[r];
        coef[p] = (D.ptr[r + 1] > e && D.val) ? D.val[e] : 0.0;
        dinv[p] = (unit || !diag) ? 1.0 : 1.0 / diag[r];
    }
    for (; p < end; p += 32) rows[p] = -1;
}

__global__ void k_group_width(const int* __restrict__ lens, int n_chains, int64_t* __restrict__ w) {
    int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    int t = g * 32 + lane;
    int len = t < n_chains ? lens[t] : 0;
    len = warp_max(len);
    if (lane == 0 && g * 32 < n_chains) w[g] = (int64_t)len * 32;
}

template <int U>
__global__ void __launch_bounds__(128) k_chain_solve(const int* __restrict__ rows, const double* __restrict__ coef,
                                                     const double* __restrict__ dinv, const int64_t* __restrict__ gbase,
                                                     int n_chains, const double* __restrict__ b, double alpha,
                                                     double* __restrict__ x, const double* __restrict__ add,
                                                     double* __restrict__ out2) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_chains) return;
    int64_t p = gbase[t >> 5] + (t & 31), end = gbase[(t >> 5) + 1];
    double xp = 0.0;
    for (; p < end; p += 32 * U) {
        int r[U];
        double c[U], d[U], bv[U], av[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            int64_t q = p + 32 * u;
            r[u] = q < end ? rows[q] : -1;
            c[u] = q < end ? coef[q] : 0.0;
            d[u] = q < end ? dinv[q] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            bv[u] = r[u] >= 0 ? b[r[u]] : 0.0;
            av[u] = (r[u] >= 0 && out2) ? add[r[u]] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (r[u] >= 0) {
                double v = fma(-c[u], xp, alpha * bv[u]) * d[u];
                x[r[u]] = v;
                if (out2) out2[r[u]] = v + av[u];
                xp = v;
            }
        }
    }
}

// IC(0) along chains: L_{i,prev} = a / L_prev,prev ; d = a_ii - L^2 ; guard ;
// L_ii = sqrt(d) -- the same IEEE operations as the general k_ic0.
__global__ void k_chain_ic0(const int* __restrict__ rows, const int64_t* __restrict__ gbase, int n_chains,
                            const int32_t* __restrict__ Lp, double* __restrict__ Lv, const double* __restrict__ aii,
                            const double* __restrict__ scale, double* __restrict__ diag, int* shifts,
                            double fill_tol) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_chains) return;
    int64_t p = gbase[t >> 5] + (t & 31), end = gbase[(t >> 5) + 1];
    double dprev = 0.0;
    int cnt = 0;
    for (; p < end; p += 32) {
        int i = rows[p];
        if (i < 0) break;
        double d = aii[i];
        int lo = Lp[i];
        if (Lp[i + 1] > lo && fabs(Lv[lo]) < fill_tol * scale[i]) {
            Lv[lo] = 0.0;   // dropped (hx/sparse.py:255-256)
        } else if (Lp[i + 1] > lo) {
            double mult = __ddiv_rn(Lv[lo], dprev);
            Lv[lo] = mult;
            d = sub_mul(d, mult, mult);
        }
        double g = 1e-12 * scale[i];
        if (d < g) {
            d = g;
            ++cnt;
        }
        dprev = __dsqrt_rn(d);
        diag[i] = dprev;
    }
    if (cnt) atomicAdd(shifts, cnt);
}

__global__ void k_max_int(const int* __restrict__ v, int n, int* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) atomicMax(out, v[i]);
}

struct I64 {
    __host__ __device__ int64_t operator()(int v) const { return (int64_t)v; }
};

// lane-interleaved layout for the warp solvers: chain t's k-th row at
// t*32E + (k % E)*32 + k / E, so lane l owns the consecutive segment
// [l*E, l*E + E) and a warp-wide load of step j is one coalesced line
__global__ void k_chain_fill_il(CsrV D, const int* __restrict__ succ, const int* __restrict__ heads, int n_chains,
                                int E, int* __restrict__ rows, double* __restrict__ coef, double* __restrict__ dinv,
                                const double* __restrict__ diag, bool unit) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_chains) return;
    const int64_t base = (int64_t)t * 32 * E;
    int k = 0;
    for (int r = heads[t]; r >= 0; r = succ[r], ++k) {
        const int64_t p = base + (k % E) * 32 + k / E;
        rows[p] = r;
        int e = D.ptr[r];
        coef[p] = (D.ptr[r + 1] > e && D.val) ? D.val[e] : 0.0;
        dinv[p] = (unit || !diag) ? 1.0 : 1.0 / diag[r];
    }
    for (; k < 32 * E; ++k) {
        const int64_t p = base + (k % E) * 32 + k / E;
        rows[p] = -1;
        coef[p] = 0.0;
        dinv[p] = 0.0;
    }
}

// One warp per chain: x_i = d_i (alpha b_i - c_i x_{i-1}) is an affine
// recurrence x_i = a_i + m_i x_{i-1}; lanes compose their segment's maps,
// a warp scan composes across lanes, then every lane replays its segment.
// Depth log2(32) + E instead of the chain length.
template <int E>
__global__ void __launch_bounds__(256) k_chain_scan(const int* __restrict__ rows, const double* __restrict__ coef,
                                                    const double* __restrict__ dinv, int n_chains,
                                                    const double* __restrict__ b, double alpha,
                                                    double* __restrict__ x, const double* __restrict__ add,
                                                    double* __restrict__ out2) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= n_chains) return;
    const int64_t base = (int64_t)w * 32 * E + lane;
    int r[E];
    double al[E], be[E];
#pragma unroll
    for (int j = 0; j < E; ++j) {
        r[j] = rows[base + 32 * j];
        const double d = dinv[base + 32 * j], cf = coef[base + 32 * j];
        al[j] = d;
        be[j] = -cf * d;
    }
#pragma unroll
    for (int j = 0; j < E; ++j) {
        if (r[j] >= 0) al[j] = al[j] * (alpha * b[r[j]]);
        else { al[j] = 0.0; be[j] = 1.0; }
    }
    double A = al[0], B = be[0];
#pragma unroll
    for (int j = 1; j < E; ++j) {
        A = fma(be[j], A, al[j]);
        B = be[j] * B;
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        double Ap = __shfl_up_sync(0xffffffffu, A, off), Bp = __shfl_up_sync(0xffffffffu, B, off);
        if (lane >= off) {
            A = fma(B, Ap, A);
            B = B * Bp;
        }
    }
    double xl = __shfl_up_sync(0xffffffffu, A, 1);
    if (lane == 0) xl = 0.0;
#pragma unroll
    for (int j = 0; j < E; ++j) {
        double v = fma(be[j], xl, al[j]);
        if (r[j] >= 0) {
            x[r[j]] = v;
            if (out2) out2[r[j]] = v + add[r[j]];
        }
        xl = v;
    }
}

// (L L^T)^{-1} on chains in one pass: the IC factor of -A_ff is block
// diagonal by chains, so a warp solves L then L^T for its own chain without any
// global dependency -- forward affine scan (x_i = d_i(alpha b_i - c_i x_{i-1})),
// then the mirrored backward scan (y_i = d_i(x_i - c_{i+1} y_{i+1})), with x
// kept in registers (chains of at most 32*E rows).  Half the launches and no
// HBM round trip for the intermediate vector.
#ifndef EDFA_CHAIN_PAIR_MINB
#define EDFA_CHAIN_PAIR_MINB 5
#endif
template <int E>
__global__ void __launch_bounds__(128, E <= 9 ? EDFA_CHAIN_PAIR_MINB : 2) k_chain_pair(const int* __restrict__ rows,
                                                    const double* __restrict__ coef, const double* __restrict__ dinv,
                                                    int n_chains, const double* b, double alpha, double* x,
                                                    const double* __restrict__ add, double* __restrict__ out2) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= n_chains) return;
    const int64_t base = (int64_t)w * 32 * E + lane;
    int r[E];
    double d[E], cf[E], xv[E];
#pragma unroll
    for (int j = 0; j < E; ++j) {   // coalesced: step j of all 32 lanes is one line
        r[j] = rows[base + 32 * j];
        d[j] = dinv[base + 32 * j];
        cf[j] = coef[base + 32 * j];
    }
    // forward: x_i = al_i + be_i x_{i-1}
    double al[E], be[E];
#pragma unroll
    for (int j = 0; j < E; ++j) {
        if (r[j] >= 0) { al[j] = d[j] * (alpha * b[r[j]]); be[j] = -cf[j] * d[j]; }
        else { al[j] = 0.0; be[j] = 1.0; }
    }
    double A = al[0], B = be[0];
#pragma unroll
    for (int j = 1; j < E; ++j) {
        A = fma(be[j], A, al[j]);
        B = be[j] * B;
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const double Ap = __shfl_up_sync(0xffffffffu, A, off), Bp = __shfl_up_sync(0xffffffffu, B, off);
        if (lane >= off) { A = fma(B, Ap, A); B = B * Bp; }
    }
    double xl = __shfl_up_sync(0xffffffffu, A, 1);
    if (lane == 0) xl = 0.0;
#pragma unroll
    for (int j = 0; j < E; ++j) {
        xv[j] = fma(be[j], xl, al[j]);
        xl = xv[j];
    }
    // backward: y_i = al'_i + be'_i y_{i+1}, al' = d_i x_i, be' = -c_{i+1} d_i
    double cn = __shfl_down_sync(0xffffffffu, cf[0], 1);   // c of the next lane's first row
    if (lane == 31) cn = 0.0;
#pragma unroll
    for (int j = 0; j < E; ++j) {
        const double cnext = j + 1 < E ? cf[j + 1] : cn;
        if (r[j] >= 0) { al[j] = d[j] * xv[j]; be[j] = -cnext * d[j]; }
        else { al[j] = 0.0; be[j] = 0.0; }
    }
    A = al[E - 1];
    B = be[E - 1];
#pragma unroll
    for (int j = E - 2; j >= 0; --j) {
        A = fma(be[j], A, al[j]);
        B = be[j] * B;
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const double Ap = __shfl_down_sync(0xffffffffu, A, off), Bp = __shfl_down_sync(0xffffffffu, B, off);
        if (lane + off < 32) { A = fma(B, Ap, A); B = B * Bp; }
    }
    double yl = __shfl_down_sync(0xffffffffu, A, 1);
    if (lane == 31) yl = 0.0;
#pragma unroll
    for (int j = E - 1; j >= 0; --j) {
        const double y = fma(be[j], yl, al[j]);
        if (r[j] >= 0) {
            if (x) x[r[j]] = y;
            if (out2) out2[r[j]] = y + add[r[j]];
        }
        yl = y;
    }
}

}  // namespace

// Try to build a chain plan for deps; returns false if deps is not chain-structured.
bool build_chain(Ctx* c, const Csr& deps, const double* diag, bool unit, ChainPlan& cp) {
    const int n = deps.n_rows;
    if (n == 0) return false;
    DevBuf<int> succ(c, n), flags(c, 2), heads(c, n), lens(c, n);
    EDFA_CUDA(cudaMemsetAsync(succ.p, 0xff, sizeof(int) * n, c->stream));
    EDFA_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int) * 2, c->stream));
    {
        Prof pr(c, "chain_plan", 16.0 * n);
        k_chain_check<<<ceil_div(n, 256), 256, 0, c->stream>>>(view(deps), succ.p, flags.p);
        check_launch("k_chain_check");
    }
    int hf[2];
    EDFA_CUDA(cudaMemcpyAsync(hf, flags.p, sizeof hf, cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
    if (hf[0]) return false;
    {
        Prof pr(c, "chain_plan", 16.0 * n);
        k_chain_heads<<<ceil_div(n, 256), 256, 0, c->stream>>>(view(deps), succ.p, heads.p, flags.p + 1, lens.p);
        check_launch("k_chain_heads");
    }
    int nc = 0;
    EDFA_CUDA(cudaMemcpyAsync(&nc, flags.p + 1, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
    // deterministic chain order: sort heads ascending (atomic append order is not)
    DevBuf<int> heads_s(c, std::max(nc, 1)), lens_s(c, std::max(nc, 1));
    {
        size_t bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, bytes, heads.p, heads_s.p, lens.p, lens_s.p, nc, 0, 32, c->stream);
        EDFA_CUDA(cub::DeviceRadixSort::SortPairs(c->cub_scratch(bytes), bytes, heads.p, heads_s.p, lens.p, lens_s.p,
                                                  nc, 0, 32, c->stream));
    }
    int ng = ceil_div(nc, 32);
    DevBuf<int64_t> w(c, (size_t)ng + 1);
    EDFA_CUDA(cudaMemsetAsync(w.p, 0, sizeof(int64_t) * (ng + 1), c->stream));
    k_group_width<<<ceil_div((int64_t)ng * 32, 256), 256, 0, c->stream>>>(lens_s.p, nc, w.p);
    cp.gbase.reset(c, (size_t)ng + 1);
    {
        size_t bytes = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, bytes, w.p, cp.gbase.p, ng + 1, c->stream);
        EDFA_CUDA(cub::DeviceScan::ExclusiveSum(c->cub_scratch(bytes), bytes, w.p, cp.gbase.p, ng + 1, c->stream));
    }
    int64_t total = 0;
    EDFA_CUDA(cudaMemcpyAsync(&total, cp.gbase.p + ng, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
    cp.n = n;
    cp.n_chains = nc;
    cp.n_stored = total;
    cp.unit = unit;
    cp.rows.reset(c, std::max<int64_t>(total, 1));
    cp.coef.reset(c, std::max<int64_t>(total, 1));
    cp.dinv.reset(c, std::max<int64_t>(total, 1));
    cp.heads = std::move(heads_s);
    cp.succ = std::move(succ);
    {   // longest chain -> segment length E of the warp solvers (lane-interleaved layout)
        int* mx = c->d_scalar_i + 34;
        EDFA_CUDA(cudaMemsetAsync(mx, 0, sizeof(int), c->stream));
        k_max_int<<<ceil_div(nc, 256), 256, 0, c->stream>>>(lens_s.p, nc, mx);
        EDFA_CUDA(cudaMemcpyAsync(&cp.max_len, mx, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        EDFA_CUDA(cudaStreamSynchronize(c->stream));
    }
    cp.E = chain_segment(cp.max_len);
    if (cp.E == 0) return false;   // chains longer than 512 rows: level plans instead
    const int64_t il = (int64_t)nc * 32 * cp.E;
    cp.crow.reset(c, il);
    cp.ccoef.reset(c, il);
    cp.cdinv.reset(c, il);
    Prof pr(c, "chain_plan", 24.0 * total);
    k_chain_fill<<<ceil_div(nc, 128), 128, 0, c->stream>>>(view(deps), cp.succ.p, cp.heads.p, nc, cp.gbase.p,
                                                           cp.rows.p, cp.coef.p, cp.dinv.p, diag, unit);
    k_chain_fill_il<<<ceil_div(nc, 128), 128, 0, c->stream>>>(view(deps), cp.succ.p, cp.heads.p, nc, cp.E, cp.crow.p,
                                                              cp.ccoef.p, cp.cdinv.p, diag, unit);
    check_launch("k_chain_fill");
    return true;
}

void chain_values(Ctx* c, const Csr& deps, const double* diag, ChainPlan& cp) {
    Prof pr(c, "chain_plan", 24.0 * cp.n_stored);
    k_chain_fill<<<ceil_div(cp.n_chains, 128), 128, 0, c->stream>>>(view(deps), cp.succ.p, cp.heads.p, cp.n_chains,
                                                                    cp.gbase.p, cp.rows.p, cp.coef.p, cp.dinv.p,
                                                                    diag, cp.unit);
    k_chain_fill_il<<<ceil_div(cp.n_chains, 128), 128, 0, c->stream>>>(view(deps), cp.succ.p, cp.heads.p,
                                                                       cp.n_chains, cp.E, cp.crow.p, cp.ccoef.p,
                                                                       cp.cdinv.p, diag, cp.unit);
    check_launch("k_chain_fill");
}

#define EDFA_CHAIN_E(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(12) X(16)

int chain_segment(int max_len) {
    const int need = std::max(1, ceil_div(max_len, 32));
#define EDFA_E_PICK(e) if (need <= e) return e;
    EDFA_CHAIN_E(EDFA_E_PICK)
#undef EDFA_E_PICK
    return 0;
}

void run_chain(Ctx* c, const ChainPlan& cp, const double* b, double alpha, double* x, const double* add, double* out2,
               const char* name) {
    Prof pr(c, name, 12.0 * cp.n + 24.0 * cp.n + (out2 ? 16.0 * cp.n : 0.0));
    const unsigned grid = (unsigned)ceil_div((int64_t)cp.n_chains * 32, 256);
    switch (cp.E) {
#define EDFA_E_CASE(e)                                                                                     \
    case e:                                                                                                \
        k_chain_scan<e><<<grid, 256, 0, c->stream>>>(cp.crow.p, cp.ccoef.p, cp.cdinv.p, cp.n_chains, b, alpha, x, \
                                                     add, out2);                                           \
        break;
        EDFA_CHAIN_E(EDFA_E_CASE)
#undef EDFA_E_CASE
        default: throw Error(EDFA_ERR_CUDA, "chain plan without a segment length");
    }
    check_launch("k_chain_scan");
}

void chain_ic0(Ctx* c, const ChainPlan& cp, const Csr& Lpat, const double* aii, const double* scale, double* diag,
               int* shifts, double fill_tol) {
    Prof pr(c, "ic0_factor", 40.0 * cp.n);
    k_chain_ic0<<<ceil_div(cp.n_chains, 128), 128, 0, c->stream>>>(cp.rows.p, cp.gbase.p, cp.n_chains, Lpat.ptr.p,
                                                                   Lpat.val.p, aii, scale, diag, shifts, fill_tol);
    check_launch("k_chain_ic0");
}

bool run_chain_pair(Ctx* c, const ChainPlan& cp, const double* b, double alpha, double* x, const double* add,
                    double* out2, const char* name) {
    if (cp.n_chains == 0 || cp.E == 0) return false;
    Prof pr(c, name, 12.0 * cp.n + 32.0 * cp.n + (out2 ? 16.0 * cp.n : 0.0) + (x ? 8.0 * cp.n : 0.0));
    // 128-thread blocks: five resident per SM at <= 102 registers (20 warps instead of 16)
    const unsigned grid = (unsigned)ceil_div((int64_t)cp.n_chains * 32, 128);
    switch (cp.E) {
#define EDFA_E_CASE(e)                                                                                     \
    case e:                                                                                                \
        k_chain_pair<e><<<grid, 128, 0, c->stream>>>(cp.crow.p, cp.ccoef.p, cp.cdinv.p, cp.n_chains, b, alpha, x, \
                                                     add, out2);                                           \
        break;
        EDFA_CHAIN_E(EDFA_E_CASE)
#undef EDFA_E_CASE
        default: return false;
    }
    check_launch("k_chain_pair");
    return true;
}

}  // namespace edfa
