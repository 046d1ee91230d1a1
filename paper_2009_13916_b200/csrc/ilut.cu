// Threshold incomplete factorisations with fill-in:
// ilu_factorize / ic_factorize of hx/sparse.py:141-282 with fill_tol > 0
// and/or no_fill=False -- the reference CLI's default inner solves
// (face_drop_tol = schur_drop_tol = 1e-3, no_fill = False, hx/config.py:79-83).
//
// The working row of the reference (a dict plus a heap of pending lower
// columns) becomes an open-addressing hash table in the warp's shared memory:
//   * pivots are taken in increasing column order by a warp-wide min search
//     over the table (the heap), popped entries become tombstones;
//   * the drop test is applied to the unscaled working value, the multiplier
//     is a_ik / u_kk, updates w_j <- w_j - l_ik u_kj run without FMA
//     contraction, new fill enters as -(l_ik u_kj); with no_fill only entries
//     already in the row are updated -- operation for operation the
//     reference's arithmetic, so factors and drop decisions are bit-identical;
//   * the U part keeps |v| >= tau, sorted; the pivot guard is the reference's
//     sign-preserving 1e-12 ||row||_inf shift.
// ILU(tau): sync-free -- warps take rows in natural order from a ticket and
// wait only on their pivot rows' published pivots (a row's U part depends on
// nothing else), so independent rows overlap as in the ILU(0) kernel.
// IC(tau) with fill: row i needs column k of L restricted to rows < i for
// every pivot k, and which rows hold column k is only known once they are
// factored; the kernel therefore walks the rows in order on one warp and
// appends every finished row to per-column lists (the reference's ``cols``).
// Rows are written to padded per-row slots and compacted to CSR afterwards.
#include <cub/cub.cuh>

#include <climits>

#include "dev_util.cuh"
#include "edfa_internal.cuh"
#include "objects.cuh"

namespace edfa {
namespace {

constexpr double PIVOT_GUARD = 1e-12;   // hx/sparse.py:24-25
constexpr int EMPTY = -1, TOMB = -2;
constexpr int ERR_OVERFLOW = 1, ERR_SPIN = 2;

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}

// ---- working row of ILU(tau) / IC(tau): open-addressing table of 2^HB slots per warp
template <int HB>
struct HTab {
    static constexpr int N = 1 << HB;
    static constexpr int MAX = N * 3 / 4;
    int* keys;
    double* vals;
    __device__ __forceinline__ unsigned slot(int j) const { return ((unsigned)j * 2654435761u) >> (32 - HB); }
    __device__ __forceinline__ int find(int j) const {
        unsigned s = slot(j);
        for (int p = 0; p < N; ++p, s = (s + 1) & (N - 1)) {
            const int k = keys[s];
            if (k == j) return (int)s;
            if (k == EMPTY) return -1;
        }
        return -1;
    }
    __device__ __forceinline__ int insert(int j, bool* fresh) const {
        unsigned s = slot(j);
        for (int p = 0; p < N; ++p, s = (s + 1) & (N - 1)) {
            int k = keys[s];
            if (k == j) { *fresh = false; return (int)s; }
            if (k == EMPTY) {
                k = atomicCAS(keys + s, EMPTY, j);
                if (k == EMPTY) { *fresh = true; return (int)s; }
                if (k == j) { *fresh = false; return (int)s; }
            }
        }
        return -1;
    }
    __device__ __forceinline__ unsigned long long next_pivot(int last, int lim, int lane) const {
        unsigned long long best = ~0ull;
        for (int s = lane; s < N; s += 32) {
            const int k = keys[s];
            if (k > last && k < lim) {
                unsigned long long v = ((unsigned long long)(unsigned)k << 32) | (unsigned)s;
                best = v < best ? v : best;
            }
        }
        return warp_min_u64(best);
    }
};

struct IlutOut {
    int* Lcnt;              // per row: multipliers
    int* Ucnt;              // per row: kept U entries (unsorted in the pool)
    int64_t* off;           // per row: first pool slot (L part, then U part)
    int32_t* pcol;          // pool
    double* pval;
    unsigned long long* pool_used;
    int64_t pool_cap;
    int32_t* scol;          // per-warp L staging (MAX entries per warp)
    double* sval;
};

// One warp per row, rows from a ticket in natural order (topological: every
// pivot row precedes the row); a row waits only on its pivot rows' published
// pivots and reads their U parts from the pool in L2.
template <bool NO_FILL, int HB>
__global__ void __launch_bounds__(128) k_ilut(int n, int* ticket, CsrV S, const double* __restrict__ scale,
                                              double fill_tol, IlutOut out, double* __restrict__ udiag,
                                              int* shifts, int* err) {
    using T = HTab<HB>;
    extern __shared__ __align__(16) unsigned char smem[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    T t;
    t.vals = reinterpret_cast<double*>(smem + (size_t)wid * T::N * 12);
    t.keys = reinterpret_cast<int*>(t.vals + T::N);
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int32_t* scol = out.scol + gw * T::MAX;
    double* sval = out.sval + gw * T::MAX;
    for (;;) {
        int i = 0;
        if (lane == 0) i = atomicAdd(ticket, 1);
        i = __shfl_sync(0xffffffffu, i, 0);
        if (i >= n) break;
        for (int q = lane; q < T::N; q += 32) t.keys[q] = EMPTY;
        __syncwarp();
        const int lo = S.ptr[i], hi = S.ptr[i + 1];
        const double norm = scale[i];
        const double tau = fill_tol * norm;
        int live = hi - lo;                     // keys ever inserted (tombstones included)
        bool bad = live > T::MAX;
        if (!bad) {
            for (int e = lo + lane; e < hi; e += 32) {
                bool fresh;
                const int q = t.insert(S.idx[e], &fresh);
                t.vals[q] = S.val[e];
            }
        }
        __syncwarp();
        int nl = 0, last = -1;
        while (!bad) {
            const unsigned long long best = t.next_pivot(last, i, lane);
            if (best == ~0ull) break;
            const int k = (int)(best >> 32), q = (int)(best & 0xffffffffu);
            const double a = t.vals[q];
            __syncwarp();
            if (lane == 0) t.keys[q] = TOMB;   // row.pop(k)
            last = k;
            if (fabs(a) < tau) {               // dropped: no multiplier, no update
                __syncwarp();
                continue;
            }
            double d = 0.0;
            if (lane == 0) {
                d = ld_relaxed(udiag + k);
                long long spins = 0;
                while (is_sentinel(d)) {
                    if (++spins > SPIN_LIMIT) { atomicExch(err, ERR_SPIN); d = 1.0; break; }
                    __nanosleep(32);
                    d = ld_relaxed(udiag + k);
                }
            }
            d = __shfl_sync(0xffffffffu, d, 0);
            __threadfence();                   // pivot row k's U part is read after its pivot was seen
            const double lik = __ddiv_rn(a, d);
            const int cu = __ldcg(out.Ucnt + k);
            const int64_t ok = __ldcg(out.off + k) + __ldcg(out.Lcnt + k);
            int added = 0;
            for (int r = lane; r < cu; r += 32) {
                const int j = __ldcg(out.pcol + ok + r);
                const double u = __ldcg(out.pval + ok + r);
                if (NO_FILL) {
                    const int sj = t.find(j);
                    if (sj >= 0) t.vals[sj] = sub_mul(t.vals[sj], lik, u);
                } else {
                    bool fresh = false;
                    const int sj = t.insert(j, &fresh);
                    if (sj < 0) { bad = true; continue; }
                    if (fresh) {
                        t.vals[sj] = -__dmul_rn(lik, u);
                        ++added;
                    } else {
                        t.vals[sj] = sub_mul(t.vals[sj], lik, u);
                    }
                }
            }
            live += warp_sum(added);
            bad = __any_sync(0xffffffffu, bad) || live > T::MAX;
            if (lane == 0) {
                scol[nl] = k;
                sval[nl] = lik;
            }
            ++nl;
            __syncwarp();
        }
        double piv = 0.0;
        int nu = 0;
        if (!bad) {
            const int sd = t.find(i);          // row.pop(i, 0.0)
            piv = sd >= 0 ? t.vals[sd] : 0.0;
            const double g = PIVOT_GUARD * norm;
            if (fabs(piv) < g) {
                piv = piv >= 0.0 ? g : -g;
                if (lane == 0) atomicAdd(shifts, 1);
            }
            for (int q = lane; q < T::N; q += 32) {
                const int k = t.keys[q];
                nu += k > i && !(fabs(t.vals[q]) < tau);
            }
            nu = warp_sum(nu);
        }
        int64_t base = 0;
        if (!bad && lane == 0) {
            base = (int64_t)atomicAdd(out.pool_used, (unsigned long long)(nl + nu));
            if (base + nl + nu > out.pool_cap) bad = true;
        }
        base = __shfl_sync(0xffffffffu, base, 0);
        bad = __shfl_sync(0xffffffffu, bad, 0);
        if (!bad) {
            __syncwarp();
            for (int r = lane; r < nl; r += 32) {
                out.pcol[base + r] = scol[r];
                out.pval[base + r] = sval[r];
            }
            int m = nl;
            for (int q0 = 0; q0 < T::N; q0 += 32) {   // U part in table order (sorted at compaction)
                const int q = q0 + lane;
                const int k = t.keys[q];
                const bool take = k > i && !(fabs(t.vals[q]) < tau);
                const unsigned bal = __ballot_sync(0xffffffffu, take);
                if (take) {
                    const int64_t pos = base + m + __popc(bal & ((1u << lane) - 1));
                    out.pcol[pos] = k;
                    out.pval[pos] = t.vals[q];
                }
                m += __popc(bal);
            }
        } else {
            if (lane == 0) atomicExch(err, ERR_OVERFLOW);
            nl = nu = 0;
            piv = 1.0;                           // unblock dependants; the factor is discarded
        }
        if (lane == 0) {
            out.off[i] = base;
            out.Lcnt[i] = nl;
            out.Ucnt[i] = nu;
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) st_relaxed(udiag + i, publishable(piv));
    }
}

// IC(tau) with fill of sign*A, rows in order on one warp; finished rows are
// appended to per-column lists (row, L_ik) -- hx/sparse.py:217-282.
__global__ void __launch_bounds__(32) k_ict(int n, CsrV A, double sign, const double* __restrict__ scale,
                                            double fill_tol, int cap, int capc, int* __restrict__ Lcnt,
                                            int32_t* __restrict__ Lcol, double* __restrict__ Lval,
                                            double* __restrict__ diag, int* __restrict__ Ccnt,
                                            int32_t* __restrict__ Crow, double* __restrict__ Cval, int* shifts,
                                            int* err) {
    using T = HTab<10>;
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    T t;
    t.vals = reinterpret_cast<double*>(smem);
    t.keys = reinterpret_cast<int*>(t.vals + T::N);
    int nshift = 0;
    for (int i = 0; i < n; ++i) {
        for (int q = lane; q < T::N; q += 32) t.keys[q] = EMPTY;
        __syncwarp();
        const int lo = A.ptr[i], hi = A.ptr[i + 1];
        const double norm = scale[i];
        const double tau = fill_tol * norm;
        int live = hi - lo;
        bool bad = live > T::MAX;
        double dii = 0.0;                       // row.get(i, 0.0)
        if (!bad) {
            for (int e = lo + lane; e < hi; e += 32) {
                const int j = A.idx[e];
                if (j < i) {
                    bool fresh;
                    const int s = t.insert(j, &fresh);
                    t.vals[s] = sign * A.val[e];
                } else if (j == i) {
                    dii = sign * A.val[e];
                }
            }
            dii = warp_sum(dii);                 // at most one lane holds the diagonal
        }
        __syncwarp();
        const int64_t o = (int64_t)i * cap;
        int nl = 0, last = -1;
        while (!bad) {
            const unsigned long long best = t.next_pivot(last, i, lane);
            if (best == ~0ull) break;
            const int k = (int)(best >> 32), s = (int)(best & 0xffffffffu);
            const double w = t.vals[s];
            __syncwarp();
            if (lane == 0) t.keys[s] = TOMB;
            last = k;
            if (fabs(w) < tau) {
                __syncwarp();
                continue;
            }
            const double lik = __ddiv_rn(w, diag[k]);   // diagonal of row k is stored last
            const int cc = Ccnt[k];
            const int64_t ok = (int64_t)k * capc;
            int added = 0;
            for (int q = lane; q < cc && q < capc; q += 32) {
                const int j = Crow[ok + q];
                if (j <= k || j >= i) continue;
                const double ljk = Cval[ok + q];
                bool fresh = false;
                const int sj = t.insert(j, &fresh);
                if (sj < 0) { bad = true; continue; }
                if (fresh) {
                    t.vals[sj] = -__dmul_rn(lik, ljk);
                    ++added;
                } else {
                    t.vals[sj] = sub_mul(t.vals[sj], lik, ljk);
                }
            }
            live += warp_sum(added);
            bad = __any_sync(0xffffffffu, bad) || live > T::MAX;
            dii = sub_mul(dii, lik, lik);
            if (lane == 0 && nl < cap) {
                Lcol[o + nl] = k;
                Lval[o + nl] = lik;
            }
            ++nl;
            __syncwarp();
            if (nl > cap) bad = true;
        }
        double d = dii;
        if (bad) {
            if (lane == 0) atomicExch(err, ERR_OVERFLOW);
            nl = 0;
            d = 1.0;
        } else if (d < PIVOT_GUARD * norm) {
            d = PIVOT_GUARD * norm;
            ++nshift;
        }
        // the row's entries join their columns' lists (cols[j].append((i, v)))
        __syncwarp();
        if (lane == 0) {
            for (int q = 0; q < nl; ++q) {
                const int k = Lcol[o + q];
                const int pos = Ccnt[k];
                if (pos < capc) {
                    Crow[(int64_t)k * capc + pos] = i;
                    Cval[(int64_t)k * capc + pos] = Lval[o + q];
                } else {
                    atomicExch(err, ERR_OVERFLOW);
                }
                Ccnt[k] = pos + 1;
            }
            Lcnt[i] = nl;
            diag[i] = __dsqrt_rn(d);
        }
        __syncwarp();
    }
    if (lane == 0 && nshift) atomicAdd(shifts, nshift);
}

// padded rows -> CSR (row = [first part | second part], both already sorted)
template <bool FILL>
__global__ void k_pad_to_csr(int n, int cap, const int* __restrict__ c1, const int32_t* __restrict__ col1,
                             const double* __restrict__ val1, const int* __restrict__ c2,
                             const int32_t* __restrict__ col2, const double* __restrict__ val2,
                             int32_t* __restrict__ cnt, const int32_t* __restrict__ ptr, int32_t* __restrict__ idx,
                             double* __restrict__ val) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int a = c1[i], b = c2 ? c2[i] : 0;
    if (!FILL) {
        cnt[i] = a + b;
        return;
    }
    const int64_t o = (int64_t)i * cap;
    int p = ptr[i];
    for (int q = 0; q < a; ++q, ++p) {
        idx[p] = col1[o + q];
        val[p] = val1[o + q];
    }
    for (int q = 0; q < b; ++q, ++p) {
        idx[p] = col2[o + q];
        val[p] = val2[o + q];
    }
}

__global__ void k_row_scale(CsrV A, double* __restrict__ sc) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.n_rows) return;
    double mx = 0.0;
    for (int e = A.ptr[i]; e < A.ptr[i + 1]; ++e) mx = fmax(mx, fabs(A.val[e]));
    sc[i] = A.ptr[i + 1] > A.ptr[i] ? mx : 1.0;
}

void pad_to_csr(Ctx* c, int n, int n_cols, int cap, const int* c1, const int32_t* col1, const double* val1,
                const int* c2, const int32_t* col2, const double* val2, Csr& out) {
    out.n_rows = n;
    out.n_cols = n_cols;
    out.ptr.reset(c, (size_t)n + 1);
    DevBuf<int32_t> cnt(c, std::max(n, 1));
    if (n) {
        k_pad_to_csr<false><<<ceil_div(n, 256), 256, 0, c->stream>>>(n, cap, c1, col1, val1, c2, col2, val2, cnt.p,
                                                                    nullptr, nullptr, nullptr);
        check_launch("k_pad_to_csr");
    }
    out.nnz = scan_counts(c, cnt.p, out.ptr.p, n);
    out.idx.reset(c, out.nnz);
    out.val.reset(c, out.nnz);
    if (n) {
        Prof pr(c, "ilut_compact", 24.0 * out.nnz);
        k_pad_to_csr<true><<<ceil_div(n, 256), 256, 0, c->stream>>>(n, cap, c1, col1, val1, c2, col2, val2, nullptr,
                                                                   out.ptr.p, out.idx.p, out.val.p);
        check_launch("k_pad_to_csr");
    }
}

template <bool FILL>
__global__ void k_nonzero(CsrV A, int32_t* __restrict__ cnt, const int32_t* __restrict__ ptr,
                          int32_t* __restrict__ idx, double* __restrict__ val) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.n_rows) return;
    int o = FILL ? ptr[i] : 0, m = 0;
    for (int e = A.ptr[i]; e < A.ptr[i + 1]; ++e) {
        if (A.val[e] == 0.0) continue;
        if (FILL) {
            idx[o + m] = A.idx[e];
            val[o + m] = A.val[e];
        }
        ++m;
    }
    if (!FILL) cnt[i] = m;
}

int row_cap(Ctx* c, const Csr& A, double fill_tol, bool no_fill) {
    // output slots per row: the longest input row with room for fill, capped
    // by what the working table can hold; complete factorisations (no drop
    // tolerance) of small matrices get whole rows
    const int maxr = A.n_rows ? max_row_nnz(c, A) : 0;
    int cap = 64;
    while (cap < 4 * maxr && cap < 512) cap *= 2;
    if (!no_fill) cap = std::max(cap, std::min(A.n_rows, 512));   // fill: whole table's worth
    return cap;
}

}  // namespace

namespace {
template <bool FILL>
__global__ void k_pool_rows(int n, const int* __restrict__ lc, const int* __restrict__ uc,
                            const int64_t* __restrict__ off, const int32_t* __restrict__ pcol,
                            const double* __restrict__ pval, int32_t* __restrict__ cnt, const int32_t* __restrict__ ptr,
                            int32_t* __restrict__ idx, double* __restrict__ val) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int m = lc[i] + uc[i];
    if (!FILL) {
        cnt[i] = m;
        return;
    }
    const int64_t o = off[i];
    const int p = ptr[i];
    for (int q = 0; q < m; ++q) {
        idx[p + q] = pcol[o + q];
        val[p + q] = pval[o + q];
    }
}
}  // namespace

// pooled rows (L part in pop order, U part unsorted) -> canonical CSR rows
void pool_to_csr(Ctx* c, int n, const int* lc, const int* uc, const int64_t* off, const int32_t* pcol,
                 const double* pval, Csr& out) {
    out.n_rows = out.n_cols = n;
    out.ptr.reset(c, (size_t)n + 1);
    DevBuf<int32_t> cnt(c, std::max(n, 1));
    if (n) {
        k_pool_rows<false><<<ceil_div(n, 256), 256, 0, c->stream>>>(n, lc, uc, off, pcol, pval, cnt.p, nullptr,
                                                                   nullptr, nullptr);
        check_launch("k_pool_rows");
    }
    out.nnz = scan_counts(c, cnt.p, out.ptr.p, n);
    DevBuf<int32_t> idx(c, std::max<int64_t>(out.nnz, 1));
    DevBuf<double> val(c, std::max<int64_t>(out.nnz, 1));
    out.idx.reset(c, std::max<int64_t>(out.nnz, 1));
    out.val.reset(c, std::max<int64_t>(out.nnz, 1));
    if (n && out.nnz) {
        Prof pr(c, "ilut_compact", 48.0 * out.nnz);
        k_pool_rows<true><<<ceil_div(n, 256), 256, 0, c->stream>>>(n, lc, uc, off, pcol, pval, nullptr, out.ptr.p,
                                                                  idx.p, val.p);
        check_launch("k_pool_rows");
        size_t bytes = 0;
        cub::DeviceSegmentedSort::SortPairs(nullptr, bytes, idx.p, out.idx.p, val.p, out.val.p, (int)out.nnz, n,
                                            out.ptr.p, out.ptr.p + 1, c->stream);
        EDFA_CUDA(cub::DeviceSegmentedSort::SortPairs(c->cub_scratch(bytes), bytes, idx.p, out.idx.p, val.p,
                                                      out.val.p, (int)out.nnz, n, out.ptr.p, out.ptr.p + 1,
                                                      c->stream));
    }
}

void drop_zeros(Ctx* c, Csr& A) {
    const int n = A.n_rows;
    Csr out;
    out.n_rows = n;
    out.n_cols = A.n_cols;
    out.ptr.reset(c, (size_t)n + 1);
    DevBuf<int32_t> cnt(c, std::max(n, 1));
    if (n) {
        k_nonzero<false><<<ceil_div(n, 256), 256, 0, c->stream>>>(view(A), cnt.p, nullptr, nullptr, nullptr);
        check_launch("k_nonzero");
    }
    out.nnz = scan_counts(c, cnt.p, out.ptr.p, n);
    out.idx.reset(c, out.nnz);
    out.val.reset(c, out.nnz);
    if (n) {
        k_nonzero<true><<<ceil_div(n, 256), 256, 0, c->stream>>>(view(A), nullptr, out.ptr.p, out.idx.p, out.val.p);
        check_launch("k_nonzero");
    }
    A = std::move(out);
}

void ilut_factor(Ctx* c, const Csr& S, double fill_tol, bool no_fill, IluFactor& f) {
    const int n = S.n_rows;
    f.n = n;
    DevBuf<double> sc(c, std::max(n, 1));
    DevBuf<int> lc(c, std::max(n, 1)), uc(c, std::max(n, 1));
    DevBuf<int64_t> off(c, std::max(n, 1));
    f.udiag.reset(c, std::max(n, 1));
    f.has_diag.reset(c, std::max(n, 1));
    int* flags = c->d_scalar_i + 24;   // [shifts, err]
    unsigned long long* used = reinterpret_cast<unsigned long long*>(c->d_scalar_i + 56);
    // pool: no_fill rows are at most S's rows; with fill start at 4x and grow on overflow
    int64_t pool_cap = no_fill ? S.nnz + 1 : 4 * S.nnz + 64 * (int64_t)n;
    int hb = 10;
    if (n) {
        k_row_scale<<<ceil_div(n, 256), 256, 0, c->stream>>>(view(S), sc.p);
        check_launch("k_row_scale");
    }
    for (int attempt = 0;; ++attempt) {
        DevBuf<int32_t> pcol(c, (size_t)std::max<int64_t>(pool_cap, 1));
        DevBuf<double> pval(c, (size_t)std::max<int64_t>(pool_cap, 1));
        EDFA_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(int), c->stream));
        EDFA_CUDA(cudaMemsetAsync(used, 0, sizeof(unsigned long long), c->stream));
        if (n) {
            fill_bits(c, f.udiag.p, n, SENTINEL_BITS);
            int* tk = c->d_scalar_i + 29;
            EDFA_CUDA(cudaMemsetAsync(tk, 0, sizeof(int), c->stream));
            const int threads = 128;
            auto kern = hb == 10 ? (no_fill ? k_ilut<true, 10> : k_ilut<false, 10>)
                                 : (no_fill ? k_ilut<true, 12> : k_ilut<false, 12>);
            const size_t smem = (size_t)(1 << hb) * 12 * (threads / 32);
            EDFA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            int occ = 0;
            EDFA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
            const int grid = NUM_SMS_B200 * std::max(1, occ);
            const int64_t warps = (int64_t)grid * (threads / 32);
            const int hmax = (1 << hb) * 3 / 4;
            DevBuf<int32_t> scol(c, (size_t)warps * hmax);
            DevBuf<double> sval(c, (size_t)warps * hmax);
            IlutOut o{lc.p, uc.p, off.p, pcol.p, pval.p, used, pool_cap, scol.p, sval.p};
            Prof pr(c, "ilut_factor", 24.0 * S.nnz + 24.0 * n);
            kern<<<grid, threads, smem, c->stream>>>(n, tk, view(S), sc.p, fill_tol, o, f.udiag.p, flags, flags + 1);
            check_launch("k_ilut");
        }
        int h[2];
        unsigned long long hu = 0;
        EDFA_CUDA(cudaMemcpyAsync(h, flags, sizeof h, cudaMemcpyDeviceToHost, c->stream));
        EDFA_CUDA(cudaMemcpyAsync(&hu, used, sizeof hu, cudaMemcpyDeviceToHost, c->stream));
        EDFA_CUDA(cudaStreamSynchronize(c->stream));
        require(h[1] != ERR_SPIN, EDFA_ERR_CUDA, "ILU(tau) factorisation stalled");
        if (h[1] == 0) {
            f.shifts = h[0];
            pool_to_csr(c, n, lc.p, uc.p, off.p, pcol.p, pval.p, f.LU);
            break;
        }
        // overflow: a row outgrew the working table (-> 4096 slots) or the pool (-> larger pool)
        const bool pool_full = (int64_t)hu > pool_cap;
        require(attempt < 4 && (pool_full || hb == 10), EDFA_ERR_UNSUPPORTED,
                "ILU(tau) fill exceeds " + std::to_string((1 << hb) * 3 / 4) +
                    " entries per working row (use a larger drop tolerance)");
        if (pool_full) pool_cap = std::max<int64_t>(2 * pool_cap, (int64_t)hu + n);
        else hb = 12;
    }
    if (n) EDFA_CUDA(cudaMemsetAsync(f.has_diag.p, 0, sizeof(int32_t) * n, c->stream));
}

void ict_factor(Ctx* c, const Csr& A, double sign, double fill_tol, IcFactor& f) {
    const int n = A.n_rows;
    f.n = n;
    const int cap = row_cap(c, A, fill_tol, false);
    const int capc = std::max(2 * cap, fill_tol == 0.0 ? std::min(n, 512) : 0);
    DevBuf<double> sc(c, std::max(n, 1));
    DevBuf<int> lc(c, std::max(n, 1)), cc(c, std::max(n, 1));
    DevBuf<int32_t> lcol(c, (size_t)std::max(n, 1) * cap), crow(c, (size_t)std::max(n, 1) * capc);
    DevBuf<double> lval(c, (size_t)std::max(n, 1) * cap), cval(c, (size_t)std::max(n, 1) * capc);
    f.diag.reset(c, std::max(n, 1));
    int* flags = c->d_scalar_i + 24;
    EDFA_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(int), c->stream));
    if (n) {
        EDFA_CUDA(cudaMemsetAsync(cc.p, 0, sizeof(int) * n, c->stream));
        k_row_scale<<<ceil_div(n, 256), 256, 0, c->stream>>>(view(A), sc.p);
        check_launch("k_row_scale");
        const size_t smem = (size_t)HTab<10>::N * 12;
        EDFA_CUDA(cudaFuncSetAttribute(k_ict, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        Prof pr(c, "ict_factor", 12.0 * A.nnz + 16.0 * n);
        k_ict<<<1, 32, smem, c->stream>>>(n, view(A), sign, sc.p, fill_tol, cap, capc, lc.p, lcol.p, lval.p, f.diag.p,
                                          cc.p, crow.p, cval.p, flags, flags + 1);
        check_launch("k_ict");
    }
    int h[2];
    EDFA_CUDA(cudaMemcpyAsync(h, flags, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
    f.shifts = h[0];
    require(h[1] == 0, EDFA_ERR_UNSUPPORTED,
            "IC(tau) fill exceeds " + std::to_string(cap) + " entries per factor row (use a larger drop tolerance)");
    pad_to_csr(c, n, n, cap, lc.p, lcol.p, lval.p, nullptr, nullptr, nullptr, f.Lpat);
}

}  // namespace edfa
