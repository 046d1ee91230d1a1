// K6/K7: IC(0) of -A_ff and ILU(0) of S~ (hx/sparse.py:141-282 with
// no_fill=True, fill_tol=0) in dependency-level order.
//
// The arithmetic mirrors the reference operation for operation -- pivots in
// increasing column order, multipliers a_ik / d_k, updates
// w_j <- w_j - l_ik * u_kj without FMA contraction, the sign-preserving guard
// |pivot| < 1e-12 * ||row||_inf -- so, given the same input matrix, the
// factors are bit-identical to the reference's pure-Python factorisation.
// Rows are processed level by level of the forward triangular-solve plan (the
// factorisation DAG is the forward-solve DAG): chain-structured factors are
// walked one chain per thread, everything else runs as a persistent
// cooperative kernel with a software grid barrier between levels.
#include <cub/cub.cuh>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "dev_util.cuh"
#include "edfa_internal.cuh"
#include "objects.cuh"

namespace edfa {
namespace {

constexpr double PIVOT_GUARD = 1e-12;

// strictly lower (mode 0) / strictly upper (mode 1) part, values scaled
template <bool FILL>
__global__ void k_select(CsrV A, int mode, double scale, int32_t* __restrict__ cnt, const int32_t* __restrict__ Op,
                         int32_t* __restrict__ Oi, double* __restrict__ Ov) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.n_rows) return;
    int n = 0, o = FILL ? Op[i] : 0;
    for (int e = A.ptr[i]; e < A.ptr[i + 1]; ++e) {
        int j = A.idx[e];
        if (mode == 0 ? j < i : j > i) {
            if (FILL) {
                Oi[o + n] = j;
                if (Ov) Ov[o + n] = A.val ? scale * A.val[e] : 0.0;
            }
            ++n;
        }
    }
    if (!FILL) cnt[i] = n;
}

// diagonal (0 if not stored) and max |row| (1 for an empty row)
__global__ void k_diag_scale(CsrV A, double sign, double* __restrict__ d, double* __restrict__ sc,
                             int32_t* __restrict__ has) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.n_rows) return;
    double dv = 0.0, mx = 0.0;
    int h = 0;
    for (int e = A.ptr[i]; e < A.ptr[i + 1]; ++e) {
        double v = A.val[e];
        mx = fmax(mx, fabs(v));
        if (A.idx[e] == i) { dv = sign * v; h = 1; }
    }
    d[i] = dv;
    sc[i] = A.ptr[i + 1] > A.ptr[i] ? mx : 1.0;
    if (has) has[i] = h;
}

struct LevelArgs {
    const int* perm;          // slot -> row (-1 padding)
    const int* level_start;   // level -> first slice
    int n_levels;
    unsigned* bar;            // [count, generation]
};

// IC(0) of -A_ff, one thread per row; L holds the strictly lower pattern
// initialised with -A values, diag receives L_ii.
__global__ void __launch_bounds__(256) k_ic0(LevelArgs la, const int32_t* __restrict__ Lp,
                                             const int32_t* __restrict__ Li, double* __restrict__ Lv,
                                             const double* __restrict__ aii, const double* __restrict__ scale,
                                             double* __restrict__ diag, int* shifts, double fill_tol) {
    const int nthr = gridDim.x * blockDim.x;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    for (int L = 0; L < la.n_levels; ++L) {
        int t1 = la.level_start[L + 1] * 32;
        for (int t = la.level_start[L] * 32 + tid; t < t1; t += nthr) {
            int i = la.perm[t];
            if (i < 0) continue;
            int lo = Lp[i], hi = Lp[i + 1];
            double d = aii[i];
            const double tau = fill_tol * scale[i];
            for (int p = lo; p < hi; ++p) {
                int k = Li[p];
                if (fabs(Lv[p]) < tau) {   // dropped on the unscaled working value
                    Lv[p] = 0.0;
                    continue;
                }
                double mult = __ddiv_rn(Lv[p], __ldcg(diag + k));
                Lv[p] = mult;
                for (int q = p + 1; q < hi; ++q) {
                    int j = Li[q];
                    int pos = bsearch(Li, Lp[j], Lp[j + 1], k);
                    if (pos >= 0) Lv[q] = sub_mul(Lv[q], mult, __ldcg(Lv + pos));
                }
                d = sub_mul(d, mult, mult);
            }
            double g = PIVOT_GUARD * scale[i];
            if (d < g) {
                d = g;
                atomicAdd(shifts, 1);
            }
            __stcg(diag + i, __dsqrt_rn(d));
        }
        if (L + 1 < la.n_levels) grid_barrier(la.bar, la.bar + 1, gridDim.x);
    }
}

// ILU(0) of S, one warp per row.  LU starts as a copy of S; on exit its
// strictly lower part holds the multipliers and its strictly upper part U;
// pivots go to udiag.
// staged U entries per pivot chunk (the elimination chunks longer pivot sets)
// (rows of at most 40 entries -- static patterns on regular grids: 37 -- stage at most 18 x 19 U entries: the
// smaller working set and 64 registers let four blocks share an SM instead of two)
__host__ __device__ constexpr int ilu0_ecap(int rmax) { return rmax <= 40 ? 352 : rmax <= 64 ? 512 : 1024; }
#ifndef EDFA_ILU0_MINB
#define EDFA_ILU0_MINB 4
#endif
__host__ __device__ constexpr int ilu0_min_blocks(int rmax) { return rmax <= 40 ? EDFA_ILU0_MINB : 1; }
__host__ __device__ constexpr size_t ilu0_warp_smem(int rmax) {
    return ((size_t)(3 * rmax + ilu0_ecap(rmax)) * 8 + (size_t)(4 * rmax + 1 + ilu0_ecap(rmax) + 2) * 4 + 15) &
           ~size_t(15);
}

// position of the first strictly-upper entry of every row
__global__ void k_ustart(CsrV A, int32_t* __restrict__ us) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < A.n_rows) us[i] = lower_bound(A.idx, A.ptr[i], A.ptr[i + 1], i + 1);
}

// one row of the ILU(0): IKJ elimination against the (final) pivot rows.
// SF: sync-free -- pivot rows are awaited through their published pivots
// (udiag is SENTINEL-filled before the launch).
template <int RMAX, bool SF>
__device__ __forceinline__ void ilu0_row(int i, const int32_t* __restrict__ Sp, const int32_t* __restrict__ Si,
                                         const int32_t* __restrict__ ustart, double* __restrict__ LU,
                                         const double* __restrict__ scale, double* __restrict__ udiag, int* shifts,
                                         int* err, unsigned char* base, int lane) {
    constexpr int ECAP = ilu0_ecap(RMAX);
    constexpr int SW = ECAP / 32 < 16 ? ECAP / 32 : 16;   // staged entries per lane per round trip
    double* vals = reinterpret_cast<double*>(base);
    double* pdk = vals + RMAX;
    double* eval = pdk + RMAX;
    int* cols = reinterpret_cast<int*>(eval + ECAP);
    int* pu0 = cols + RMAX;
    int* pcnt = pu0 + RMAX;
    int* poff = pcnt + RMAX;           // RMAX + 1
    int* eslot = poff + RMAX + 1;      // ECAP
    int* misc = eslot + ECAP;          // 2
    int lo = Sp[i], n = Sp[i + 1] - lo;
    if (n > RMAX) {
        if (lane == 0) atomicExch(err, 4);
        if (SF && lane == 0) st_relaxed(udiag + i, 1.0);   // unblock dependants (the factor is discarded)
        return;
    }
    for (int t = lane; t < n; t += 32) {
        cols[t] = Si[lo + t];
        vals[t] = LU[lo + t];
    }
    __syncwarp();
    int nl = lower_bound(cols, 0, n, i);
    // pattern-only work first (U-row extents, chunking, target slots): it
    // needs no pivot values, so it overlaps the wait for the pivot rows and
    // only the value loads and the elimination remain on the critical path
    for (int p = lane; p < nl; p += 32) {
        const int k = cols[p];
        const int u0 = __ldg(ustart + k);
        pu0[p] = u0;
        pcnt[p] = Sp[k + 1] - u0;
    }
    __syncwarp();
    auto chunk = [&](int p0) {   // pivots [p0, misc[0]) whose U entries fit the staging buffer
        if (lane == 0) {
            int acc = 0, p1 = p0;
            while (p1 < nl && (p1 == p0 || acc + pcnt[p1] <= ECAP)) {
                poff[p1 - p0] = acc;
                acc += pcnt[p1];
                ++p1;
            }
            poff[p1 - p0] = acc;
            misc[0] = p1;
            misc[1] = min(acc, ECAP);
        }
        __syncwarp();
    };
    // stage (target slot, global index of u_kj) of every U entry of a chunk
    long long* eidx = reinterpret_cast<long long*>(eval);
    auto stage_slots = [&](int p0) {
        const int p1 = misc[0], tot = misc[1];
        for (int f0 = 0; f0 < tot; f0 += 32 * SW) {
            int e[SW], q[SW];
            int32_t j[SW];
#pragma unroll
            for (int w = 0; w < SW; ++w) {
                int f = f0 + w * 32 + lane;
                q[w] = -1;
                if (f < tot) {
                    int lo2 = 0, hi2 = p1 - p0;      // pivot owning flat entry f
                    while (hi2 - lo2 > 1) {
                        int mid = (lo2 + hi2) >> 1;
                        if (poff[mid] <= f) lo2 = mid;
                        else hi2 = mid;
                    }
                    q[w] = p0 + lo2;
                    e[w] = pu0[q[w]] + (f - poff[lo2]);
                }
            }
#pragma unroll
            for (int w = 0; w < SW; ++w)
                if (q[w] >= 0) j[w] = __ldg(Si + e[w]);
#pragma unroll
            for (int w = 0; w < SW; ++w) {
                int f = f0 + w * 32 + lane;
                if (q[w] >= 0) {
                    eslot[f] = bsearch(cols, q[w] + 1, n, j[w]);
                    eidx[f] = e[w];
                }
            }
        }
        __syncwarp();
    };
    auto stage_values = [&]() {   // u_kj of the staged entries (pivot rows final)
        const int tot = misc[1];
        for (int f = lane; f < tot; f += 32) eval[f] = __ldcg(LU + eidx[f]);
        __syncwarp();
    };
    if (nl > 0) {
        chunk(0);
        stage_slots(0);
    }
    // every pivot row is final (earlier level) or awaited here through its
    // published pivot
    for (int p = lane; p < nl; p += 32) {
        int k = cols[p];
        if (SF) {   // wait for pivot row k (its pivot is published last)
            double d = ld_relaxed(udiag + k);
            long long spins = 0;
            while (is_sentinel(d)) {
                if (++spins > SPIN_LIMIT) { atomicExch(err, 7); d = 1.0; break; }
                __nanosleep(32);
                d = ld_relaxed(udiag + k);
            }
            pdk[p] = d;
        } else {
            pdk[p] = __ldcg(udiag + k);
        }
    }
    if (SF) __threadfence();   // pivot rows' U entries are read after their pivots were seen
    __syncwarp();
    for (int p0 = 0; p0 < nl;) {
        if (p0 > 0) {   // later chunks (rows whose pivots' U parts exceed the buffer)
            chunk(p0);
            stage_slots(p0);
        }
        stage_values();
        const int p1 = misc[0], tot = misc[1];
        // eliminate, pivots in increasing column order (reference IKJ order)
        for (int p = p0; p < p1; ++p) {
            double mult = __ddiv_rn(vals[p], pdk[p]);
            __syncwarp();
            if (lane == 0) vals[p] = mult;
            const int off = poff[p - p0], cnt = min(pcnt[p], tot - off);
            for (int f = lane; f < cnt; f += 32) {
                int sl = eslot[off + f];
                if (sl >= 0) vals[sl] = sub_mul(vals[sl], mult, eval[off + f]);
            }
            __syncwarp();
        }
        p0 = p1;
    }
    int dslot = bsearch(cols, nl, n, i);
    double piv = dslot >= 0 ? vals[dslot] : 0.0;
    double g = PIVOT_GUARD * scale[i];
    if (fabs(piv) < g) {
        piv = piv >= 0.0 ? g : -g;
        if (lane == 0) atomicAdd(shifts, 1);
    }
    for (int t = lane; t < n; t += 32) __stcg(LU + lo + t, vals[t]);
    if (SF) {   // publish: row values, fence, then the pivot (the row's ready flag)
        __threadfence();
        __syncwarp();
        if (lane == 0) st_relaxed(udiag + i, publishable(piv));
    } else if (lane == 0) {
        __stcg(udiag + i, piv);
    }
    __syncwarp();
}

// level-synchronous: rows of one level per grid-barrier phase
template <int RMAX>
__global__ void __launch_bounds__(256) k_ilu0(LevelArgs la, const int32_t* __restrict__ Sp,
                                              const int32_t* __restrict__ Si, const int32_t* __restrict__ ustart,
                                              double* __restrict__ LU, const double* __restrict__ scale,
                                              double* __restrict__ udiag, int* shifts, int* err) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* base = smem + (size_t)wid * ilu0_warp_smem(RMAX);
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (int L = 0; L < la.n_levels; ++L) {
        int t1 = la.level_start[L + 1] * 32;
        for (int slot = la.level_start[L] * 32 + gw; slot < t1; slot += nw) {
            int i = la.perm[slot];
            if (i < 0) continue;
            ilu0_row<RMAX, false>(i, Sp, Si, ustart, LU, scale, udiag, shifts, err, base, lane);
        }
        if (L + 1 < la.n_levels) grid_barrier(la.bar, la.bar + 1, gridDim.x);
    }
}

// sync-free: warps take rows from a ticket in a topological order (every
// dependency of ord[s] precedes it), so a warp only ever waits on rows held by
// running warps -- no grid barrier, no level plan, a row starts as soon as its
// own pivot rows are final
template <int RMAX>
__global__ void __launch_bounds__(256, ilu0_min_blocks(RMAX)) k_ilu0_sf(const int* __restrict__ ord, int n_ord, int* ticket,
                                                 const int32_t* __restrict__ Sp, const int32_t* __restrict__ Si,
                                                 const int32_t* __restrict__ ustart, double* __restrict__ LU,
                                                 const double* __restrict__ scale, double* __restrict__ udiag,
                                                 int* shifts, int* err) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* base = smem + (size_t)wid * ilu0_warp_smem(RMAX);
    for (;;) {
        int s = 0;
        if (lane == 0) s = atomicAdd(ticket, 1);
        s = __shfl_sync(0xffffffffu, s, 0);
        if (s >= n_ord) break;
        const int i = ord[s];
        if (i < 0) continue;
        ilu0_row<RMAX, true>(i, Sp, Si, ustart, LU, scale, udiag, shifts, err, base, lane);
    }
}

// wavefront order of a cell grid: key = i + j + k (x fastest, hx/grid.py:49-50)
__global__ void k_grid_keys(int n, int nx, int ny, int* __restrict__ key, int* __restrict__ row) {
    int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    key[e] = e % nx + (e / nx) % ny + e / (nx * ny);
    row[e] = e;
}
// the order is topological iff every strictly-lower entry has key <= the row's
__global__ void k_grid_order_check(CsrV A, int nx, int ny, int* __restrict__ bad, bool strict = false) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.n_rows) return;
    const int ki = i % nx + (i / nx) % ny + i / (nx * ny);
    for (int e = A.ptr[i]; e < A.ptr[i + 1]; ++e) {
        const int j = A.idx[e];
        if (j >= i) break;
        const int kj = j % nx + (j / nx) % ny + j / (nx * ny);
        if (strict ? kj >= ki : kj > ki) { atomicExch(bad, 1); return; }
    }
}

// exported CSRs in the reference layout: IC L with the diagonal last in each
// row; ILU L = strict lower + unit diagonal (last); U = diagonal first + upper
template <bool FILL>
__global__ void k_export_tri(CsrV P, const double* __restrict__ diag, int mode, int32_t* __restrict__ cnt,
                             const int32_t* __restrict__ Op, int32_t* __restrict__ Oi, double* __restrict__ Ov) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.n_rows) return;
    int n = 0, o = FILL ? Op[i] : 0;
    auto put = [&](int j, double v) {
        if (FILL) { Oi[o + n] = j; Ov[o + n] = v; }
        ++n;
    };
    if (mode == 2) put(i, diag[i]);
    for (int e = P.ptr[i]; e < P.ptr[i + 1]; ++e) {
        int j = P.idx[e];
        if (mode == 2 ? j > i : j < i) put(j, P.val[e]);
    }
    if (mode == 0) put(i, diag[i]);
    if (mode == 1) put(i, 1.0);
    if (!FILL) cnt[i] = n;
}

void select_part(Ctx* c, const Csr& A, int mode, double scale, bool values, Csr& out) {
    int n = A.n_rows;
    out.n_rows = n;
    out.n_cols = A.n_cols;
    out.ptr.reset(c, (size_t)n + 1);
    DevBuf<int32_t> cnt(c, std::max(n, 1));
    if (n) {
        Prof pr(c, "select", 8.0 * A.nnz);
        k_select<false><<<ceil_div(n, 128), 128, 0, c->stream>>>(view(A), mode, scale, cnt.p, nullptr, nullptr,
                                                                nullptr);
        check_launch("k_select");
    }
    out.nnz = scan_counts(c, cnt.p, out.ptr.p, n);
    out.idx.reset(c, out.nnz);
    if (values) out.val.reset(c, out.nnz);
    else out.val.release();
    if (n) {
        Prof pr(c, "select", 8.0 * A.nnz + 12.0 * out.nnz);
        k_select<true><<<ceil_div(n, 128), 128, 0, c->stream>>>(view(A), mode, scale, nullptr, out.ptr.p, out.idx.p,
                                                               values ? out.val.p : nullptr);
        check_launch("k_select");
    }
}

void export_tri(Ctx* c, const Csr& P, const double* diag, int mode, Csr& out) {
    int n = P.n_rows;
    out.n_rows = n;
    out.n_cols = P.n_cols;
    out.ptr.reset(c, (size_t)n + 1);
    DevBuf<int32_t> cnt(c, std::max(n, 1));
    if (n) {
        k_export_tri<false><<<ceil_div(n, 128), 128, 0, c->stream>>>(view(P), diag, mode, cnt.p, nullptr, nullptr,
                                                                    nullptr);
        check_launch("k_export_tri");
    }
    out.nnz = scan_counts(c, cnt.p, out.ptr.p, n);
    out.idx.reset(c, out.nnz);
    out.val.reset(c, out.nnz);
    if (n) {
        k_export_tri<true><<<ceil_div(n, 128), 128, 0, c->stream>>>(view(P), diag, mode, nullptr, out.ptr.p,
                                                                   out.idx.p, out.val.p);
        check_launch("k_export_tri");
    }
}

void read_flags(Ctx* c, const int* dev, int* shifts, int* err) {
    int h[2];
    EDFA_CUDA(cudaMemcpyAsync(h, dev, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
    *shifts = h[0];
    *err = h[1];
}

template <class K>
int coop_grid(K kern, int threads, size_t smem, int cap = 2) {
    int occ = 0;
    EDFA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
    return NUM_SMS_B200 * std::max(1, std::min(occ, cap));
}

}  // namespace

void ilu_plans(Ctx* c, IluFactor& f, const int* dims, bool have_fwd_levels);
bool use_wf_layout(Ctx* c, int n, const int* dims);

// backward plan of an IC factor whose forward plan holds L's values: chains
// and level plans as before; non-chain factors (distorted grids) get the
// wavefront-packed solves, L^T on L's slot layout
static void ic_backward_plan(Ctx* c, IcFactor& f, const Csr& LT) {
    if (!f.fwd.is_chain && f.n > 0 && c->opt.ilu_wf != 0 && !c->opt.trsv_levels &&
        build_wf_plans(c, f.Lpat, LT, f.diag.p, f.fwd, f.bwd))
        return;
    build_plan(c, LT, f.diag.p, false, true, f.bwd);
}

void ic0_factor(Ctx* c, const Csr& A_ff, double drop_tol, IcFactor& f, bool no_fill) {
    require(drop_tol >= 0.0, EDFA_ERR_VALUE, "fill_tol must be >= 0");
    const int n = A_ff.n_rows;
    f.n = n;
    select_part(c, A_ff, 0, -1.0, true, f.Lpat);
    DevBuf<double> aii(c, std::max(n, 1)), sc(c, std::max(n, 1));
    f.diag.reset(c, std::max(n, 1));
    if (n) {
        Prof pr(c, "ic0_prep", 12.0 * A_ff.nnz + 16.0 * n);
        k_diag_scale<<<ceil_div(n, 128), 128, 0, c->stream>>>(view(A_ff), -1.0, aii.p, sc.p, nullptr);
        check_launch("k_diag_scale");
    }
    build_plan(c, f.Lpat, nullptr, false, false, f.fwd);
    // a chain-structured (disjoint paths) pattern has no fill-in, so IC(tau)
    // with fill equals the pattern-restricted factorisation there
    if (!no_fill && n && !f.fwd.is_chain) {
        ict_factor(c, A_ff, -1.0, drop_tol, f);
        f.fwd = TriPlan();
        build_plan(c, f.Lpat, f.diag.p, false, false, f.fwd);
        plan_values(c, f.Lpat, f.diag.p, f.fwd);
        Csr LT;
        transpose(c, f.Lpat, LT);
        ic_backward_plan(c, f, LT);
        return;
    }
    int* flags = c->d_scalar_i + 24;   // [shifts, err]
    EDFA_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(int), c->stream));
    if (n && f.fwd.is_chain) {
        chain_ic0(c, f.fwd.chain, f.Lpat, aii.p, sc.p, f.diag.p, flags, drop_tol);
    } else if (n) {
        LevelArgs la{f.fwd.perm.p, f.fwd.level_start.p, f.fwd.n_levels, reinterpret_cast<unsigned*>(f.fwd.sync.p)};
        Prof pr(c, "ic0_factor", 24.0 * f.Lpat.nnz + 32.0 * n);
        int grid = coop_grid(k_ic0, 256, 0);
        const int32_t* Lp = f.Lpat.ptr.p;
        const int32_t* Li = f.Lpat.idx.p;
        double* Lv = f.Lpat.val.p;
        const double* ap = aii.p;
        const double* sp = sc.p;
        double* dp = f.diag.p;
        int* sh = flags;
        double ft = drop_tol;
        void* args[] = {&la, &Lp, &Li, &Lv, &ap, &sp, &dp, &sh, &ft};
        EDFA_CUDA(cudaLaunchCooperativeKernel((void*)k_ic0, dim3(grid), dim3(256), args, 0, c->stream));
    }
    int err = 0;
    read_flags(c, flags, &f.shifts, &err);
    require(err == 0, EDFA_ERR_CUDA, "IC(0) factorisation failed");
    if (drop_tol > 0.0) {   // dropped entries (exact zeros: kept ones satisfy |w| >= tau > 0) leave the factor
        drop_zeros(c, f.Lpat);
        f.fwd = TriPlan();
        build_plan(c, f.Lpat, f.diag.p, false, false, f.fwd);
    }
    plan_values(c, f.Lpat, f.diag.p, f.fwd);
    Csr LT;
    transpose(c, f.Lpat, LT);
    ic_backward_plan(c, f, LT);
}

void ilu0_factor(Ctx* c, const Csr& S, double drop_tol, IluFactor& f, const int* dims, bool no_fill) {
    require(drop_tol >= 0.0, EDFA_ERR_VALUE, "fill_tol must be >= 0");
    if (drop_tol > 0.0 || !no_fill) {   // threshold ILU (ilut.cu), then the same solve plans
        ilut_factor(c, S, drop_tol, no_fill, f);
        ilu_plans(c, f, dims, false);
        return;
    }
    const int n = S.n_rows;
    f.n = n;
    copy_csr(c, S, f.LU);
    DevBuf<double> dd(c, std::max(n, 1)), sc(c, std::max(n, 1));
    f.udiag.reset(c, std::max(n, 1));
    f.has_diag.reset(c, std::max(n, 1));
    if (n) {
        Prof pr(c, "ilu0_prep", 12.0 * S.nnz + 16.0 * n);
        k_diag_scale<<<ceil_div(n, 128), 128, 0, c->stream>>>(view(S), 1.0, dd.p, sc.p, f.has_diag.p);
        check_launch("k_diag_scale");
    }
    // factorisation schedule: on a cell grid whose lower pattern only reaches
    // back in i+j+k (true for the axial stencils of base/static patterns) the
    // wavefront order (i+j+k, row) is topological and the sync-free kernel
    // runs without a level plan; otherwise rows go level by level
    const bool grid = dims && n > 0 && dims[0] > 0 && dims[1] > 0 && dims[2] > 0 &&
                      (int64_t)dims[0] * dims[1] * dims[2] == n;
    bool sync_free = false;
    DevBuf<int> ord;
    if (grid && !use_wf_layout(c, n, dims)) {
        PhaseTimer pt(c, "ilu0.wavefront_order");
        int* bad = c->d_scalar_i + 28;
        EDFA_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), c->stream));
        k_grid_order_check<<<ceil_div(n, 256), 256, 0, c->stream>>>(view(S), dims[0], dims[1], bad);
        check_launch("k_grid_order_check");
        DevBuf<int> key(c, n), row(c, n), skey(c, n);
        ord.reset(c, n);
        k_grid_keys<<<ceil_div(n, 256), 256, 0, c->stream>>>(n, dims[0], dims[1], key.p, row.p);
        check_launch("k_grid_keys");
        int bits = 1;
        while ((1 << bits) <= dims[0] + dims[1] + dims[2]) ++bits;
        size_t bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, bytes, key.p, skey.p, row.p, ord.p, n, 0, bits, c->stream);
        EDFA_CUDA(cub::DeviceRadixSort::SortPairs(c->cub_scratch(bytes), bytes, key.p, skey.p, row.p, ord.p, n, 0,
                                                  bits, c->stream));
        int hb = 0;
        EDFA_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        EDFA_CUDA(cudaStreamSynchronize(c->stream));
        sync_free = hb == 0 && !c->opt.ilu_levels;
    }
    Csr Lpart;
    auto level_plan = [&]() {
        PhaseTimer pt(c, "ilu0.level_plan");
        select_part(c, S, 0, 1.0, false, Lpart);
        if (grid) {
            // axial stencils: every lower entry lies on an earlier plane i+j+k, so the
            // planes are a valid layering (no sync-free level computation)
            int* bad = c->d_scalar_i + 28;
            EDFA_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), c->stream));
            k_grid_order_check<<<ceil_div(n, 256), 256, 0, c->stream>>>(view(S), dims[0], dims[1], bad, true);
            DevBuf<int> key(c, n), row(c, n);
            k_grid_keys<<<ceil_div(n, 256), 256, 0, c->stream>>>(n, dims[0], dims[1], key.p, row.p);
            check_launch("k_grid_keys");
            int hb = 0;
            EDFA_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
            EDFA_CUDA(cudaStreamSynchronize(c->stream));
            if (!hb) {
                build_plan(c, Lpart, nullptr, true, false, f.fwd, /*allow_chain=*/false, key.p,
                           dims[0] + dims[1] + dims[2] - 2);
                return;
            }
        }
        build_plan(c, Lpart, nullptr, true, false, f.fwd, /*allow_chain=*/false);
    };
    const bool have_levels = !sync_free;
    if (!sync_free) {
        level_plan();
        // rows in level order are topological too: run the sync-free kernel on
        // that order (no grid barrier per level) unless levels are requested
        sync_free = !c->opt.ilu_levels;
    }
    PhaseTimer pt_fact(c, "ilu0.factor+plans");
    int maxr = n ? max_row_nnz(c, S) : 0;
    require(maxr <= 1024, EDFA_ERR_UNSUPPORTED, "Schur rows longer than 1024 entries are not supported");
    int* flags = c->d_scalar_i + 24;
    EDFA_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(int), c->stream));
    if (n) {
        DevBuf<int32_t> ust(c, n);
        k_ustart<<<ceil_div(n, 256), 256, 0, c->stream>>>(view(f.LU), ust.p);
        check_launch("k_ustart");
        const int32_t* Sp = f.LU.ptr.p;
        const int32_t* Si = f.LU.idx.p;
        const int32_t* Us = ust.p;
        double* LUv = f.LU.val.p;
        const double* scp = sc.p;
        double* ud = f.udiag.p;
        int* sh = flags;
        int* er = flags + 1;
        if (sync_free) fill_bits(c, ud, n, SENTINEL_BITS);   // a row's pivot is its ready flag
        Prof pr(c, "ilu0_factor", 24.0 * S.nnz + 24.0 * n);
        LevelArgs la{f.fwd.perm.p, f.fwd.level_start.p, f.fwd.n_levels, reinterpret_cast<unsigned*>(f.fwd.sync.p)};
        const int* op = have_levels ? f.fwd.perm.p : ord.p;
        int n_ord = have_levels ? f.fwd.n_slots : n;
        int* tk = c->d_scalar_i + 29;
        if (sync_free) EDFA_CUDA(cudaMemsetAsync(tk, 0, sizeof(int), c->stream));
        void* args[] = {&la, &Sp, &Si, &Us, &LUv, &scp, &ud, &sh, &er};
        void* args_sf[] = {&op, &n_ord, &tk, &Sp, &Si, &Us, &LUv, &scp, &ud, &sh, &er};
        auto launch = [&](auto kern, auto kern_sf, int rmax) {
            int threads = rmax >= 1024 ? 64 : rmax <= 64 ? 256 : 128;
            size_t smem = ilu0_warp_smem(rmax) * (threads / 32);
            void* k = sync_free ? (void*)kern_sf : (void*)kern;
            if (smem > 48 * 1024)
                EDFA_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            if (sync_free) {
                // persistent warps, every resident slot filled (no co-residency requirement)
                int grid = coop_grid(kern_sf, threads, smem, 8);
                EDFA_CUDA(cudaLaunchKernel(k, dim3(grid), dim3(threads), args_sf, smem, c->stream));
            } else {
                int grid = coop_grid(kern, threads, smem, 4);
                EDFA_CUDA(cudaLaunchCooperativeKernel(k, dim3(grid), dim3(threads), args, smem, c->stream));
            }
        };
        if (maxr <= 40) launch(k_ilu0<40>, k_ilu0_sf<40>, 40);
        else if (maxr <= 64) launch(k_ilu0<64>, k_ilu0_sf<64>, 64);
        else if (maxr <= 256) launch(k_ilu0<256>, k_ilu0_sf<256>, 256);
        else launch(k_ilu0<1024>, k_ilu0_sf<1024>, 1024);
    }
    int err = 0;
    read_flags(c, flags, &f.shifts, &err);
    require(err == 0, EDFA_ERR_CUDA, "ILU(0) factorisation failed");
    ilu_plans(c, f, dims, have_levels);
}

// the wavefront-packed layout pays when levels are wide: decided from the grid
// shape before any plan exists (levels of an axial stencil = nx+ny+nz-2), and
// re-checked against the real level count in ilu_plans.  Measured (config 5
// generator, per solve): the wf solve costs ~1.1 us per level while levels are
// narrow and turns bandwidth-bound when they are wide (382 / 574 / 766 levels at
// 128^3 / 192^3 / 256^3: 0.42 / 0.73 / 1.51 ms), the tile-DAG solve streams at
// ~1.75 TB/s (0.40 / 0.98 / 2.23 ms).  With the prefetching shape (k_wf_pf) the wf solve takes 0.26 / 0.35 ms at
// 96^3 / 128^3 against the tile solver's 0.235 / 0.40 ms, and its plan builds faster (stage 2 at 128^3: 17 vs 28 ms):
// crossover at ~4k rows per level (96^3: 3.1k, 128^3: 5.5k).
constexpr int64_t WF_MIN_ROWS_PER_LEVEL = 4096;
bool use_wf_layout(Ctx* c, int n, const int* dims) {
    if (c->opt.ilu_wf >= 0) return c->opt.ilu_wf == 1 && n > 0;
    if (!dims || dims[0] <= 0) return false;
    return (int64_t)n >= WF_MIN_ROWS_PER_LEVEL * (dims[0] + dims[1] + dims[2]);
}

// triangular-solve plans of an ILU factor (f.LU strict parts + f.udiag);
// have_fwd_levels: f.fwd already holds the level plan of L's pattern
void ilu_plans(Ctx* c, IluFactor& f, const int* dims, bool have_fwd_levels) {
    const int n = f.n;
    Csr Lv, Uv;
    select_part(c, f.LU, 0, 1.0, true, Lv);
    select_part(c, f.LU, 1, 1.0, true, Uv);
    // 1. wide dependency levels on a cell grid (e.g. 256^3: 766 levels of up to 49k
    //    rows): both solves wavefront-packed on the slot layout of L's level plan;
    // 2. otherwise cell-grid factors with an axial stencil: tile-DAG solves;
    // 3. otherwise (general factors, e.g. dynamic patterns on distorted grids:
    //    thousands of narrow levels): wavefront-packed again -- its hand-off per
    //    level is the cheapest of the level-ordered solvers.
    const bool wf_allowed = c->opt.ilu_wf != 0 && !c->opt.trsv_levels;
    bool want_wf = wf_allowed && use_wf_layout(c, n, dims);
    auto fwd_levels = [&]() {
        if (!have_fwd_levels) build_plan(c, Lv, nullptr, true, false, f.fwd, /*allow_chain=*/false);
        have_fwd_levels = true;
    };
    if (want_wf && c->opt.ilu_wf != 1) {
        fwd_levels();
        want_wf = (int64_t)n >= WF_MIN_ROWS_PER_LEVEL * f.fwd.n_levels;
    }
    bool fwd_tile = false, bwd_tile = false;
    if (!want_wf && dims) {
        fwd_tile = build_tile_plan(c, Lv, nullptr, true, false, dims, f.fwd.tile);
        bwd_tile = build_tile_plan(c, Uv, f.udiag.p, false, true, dims, f.bwd.tile);
    }
    if (fwd_tile) {
        f.fwd.is_tile = true;
        f.fwd.n = n;
        f.fwd.n_dep = Lv.nnz;
        f.fwd.n_levels = f.fwd.tile.n_tile_levels;
    } else {
        fwd_levels();
        plan_values(c, Lv, nullptr, f.fwd);
    }
    if (bwd_tile) {
        f.bwd.is_tile = true;
        f.bwd.n = n;
        f.bwd.n_dep = Uv.nnz;
        f.bwd.n_levels = f.bwd.tile.n_tile_levels;
        return;
    }
    if (!fwd_tile && wf_allowed && n > 0 && build_wf_plans(c, Lv, Uv, f.udiag.p, f.fwd, f.bwd)) return;
    build_plan(c, Uv, f.udiag.p, false, true, f.bwd);
}

void ic_export(Ctx* c, IcFactor& f) {
    if (f.export_L.ptr.p) return;
    export_tri(c, f.Lpat, f.diag.p, 0, f.export_L);
}

void ilu_export(Ctx* c, IluFactor& f) {
    if (f.export_L.ptr.p) return;
    export_tri(c, f.LU, f.udiag.p, 1, f.export_L);
    export_tri(c, f.LU, f.udiag.p, 2, f.export_U);
}

}  // namespace edfa
