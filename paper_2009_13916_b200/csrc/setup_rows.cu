// EDFA stage-1 row kernels: restricted SPD solves for the decoupling factors
// (K1, static/base patterns) and residual-driven pattern growth (K2, dynamic).
//
// One warp per cell row m (hx/precond.py:187-201):
//   gather  M = -A_ff[Q,Q] (dense, shared memory, ld = SMAX+1: conflict-free
//           column access for doubles), b_g = A_cf[m,Q], b_f = A_fc[Q,m]
//   factor  right-looking Cholesky in shared memory (LAPACK potrf semantics:
//           a non-positive pivot is a FactorizationError for row m)
//   solve   forward/backward substitution for both right-hand sides
//   dynamic prolonged residual r = b + A_ff R^T x on the candidate support,
//           top-n fresh entries by (|r| desc, index asc), re-solve
//           (hx/precond.py:96-135, Algorithm 1 of P:594-611)
//   write   g~, f~ (pre-filtered) in a per-row slot layout + nonzero counts;
//           a second kernel compacts them into canonical CSR (exact zeros
//           dropped, hx/sparse.py:28-34).
#include <cub/cub.cuh>

#include <mutex>
#include <set>

#include "dev_util.cuh"
#include "edfa_internal.cuh"
#include "objects.cuh"

namespace edfa {

namespace {

enum { ERR_FACT = 1, ERR_CAND = 2, ERR_SIZE = 3 };

struct RowArgs {
    CsrV A;        // A_ff (rows = faces)
    CsrV AT;       // transpose of A_ff (columns of A_ff), for candidate support
    CsrV Acf;      // rhs rows for g (cells x faces)
    CsrV AfcT;     // rhs rows for f (cells x faces)
    const int32_t* q_ptr;  // static sets (CSR pattern), NULL for dynamic
    const int32_t* q_idx;
    int32_t n_rows;
    int32_t n_add, n_ent, sweep_limit;
    double pre_tau;
    const int32_t* slot_ptr;  // output slot start per row
    int32_t* out_q;           // dynamic: final sets in slot layout
    int32_t* out_qsize;
    double* out_g;
    double* out_f;
    int32_t* out_gcnt;
    int32_t* out_fcnt;
    int* err;                 // [code, row]
};

__device__ void report(int* err, int code, int row) {
    atomicCAS(err, 0, code);
    atomicMin(err + 1, row);
}

// The s x s block is kept as its lower triangle, packed by rows (entry (i, j),
// j <= i, at i(i+1)/2 + j): half the shared memory of a padded square tile, so
// more warps are resident per SM (the dynamic kernel is latency-bound).
__device__ __forceinline__ int tri(int i, int j) { return ((i * (i + 1)) >> 1) + j; }

__device__ void gather_M(const CsrV& A, const int* q, int s, double* M, int lane) {
    for (int t = lane; t < tri(s, 0); t += 32) M[t] = 0.0;
    __syncwarp();
    for (int i = lane; i < s; i += 32) {
        int row = q[i];
        for (int e = A.ptr[row]; e < A.ptr[row + 1]; ++e) {
            int j = bsearch(q, 0, i + 1, A.idx[e]);   // lower triangle only
            if (j >= 0) M[tri(i, j)] = -A.val[e];
        }
    }
    __syncwarp();
}

__device__ void gather_rhs(const CsrV& R, int m, const int* q, int s, double* b, int lane) {
    for (int i = lane; i < s; i += 32) b[i] = 0.0;
    __syncwarp();
    for (int e = R.ptr[m] + lane; e < R.ptr[m + 1]; e += 32) {
        int j = bsearch(q, 0, s, R.idx[e]);
        if (j >= 0) b[j] = R.val[e];
    }
    __syncwarp();
}

// in-place lower Cholesky of the packed s x s block; false on a non-positive pivot
__device__ bool cholesky(double* M, int s, int lane) {
    for (int k = 0; k < s; ++k) {
        double d = M[tri(k, k)];
        if (!(d > 0.0)) return false;
        double l = sqrt(d);
        double il = 1.0 / l;
        __syncwarp();
        for (int i = k + 1 + lane; i < s; i += 32) M[tri(i, k)] *= il;
        if (lane == 0) M[tri(k, k)] = l;
        __syncwarp();
        for (int i = k + 1 + lane; i < s; i += 32) {
            double lik = M[tri(i, k)];
            double* Mi = M + tri(i, 0);
            for (int j = k + 1; j <= i; ++j) Mi[j] = fma(-lik, M[tri(j, k)], Mi[j]);
        }
        __syncwarp();
    }
    return true;
}

template <int NRHS>
__device__ void chol_solve(const double* M, int s, double* b1, double* b2, int lane) {
    for (int k = 0; k < s; ++k) {
        __syncwarp();
        double il = 1.0 / M[tri(k, k)];
        double y1 = b1[k] * il, y2 = NRHS > 1 ? b2[k] * il : 0.0;
        __syncwarp();
        for (int i = k + 1 + lane; i < s; i += 32) {
            double l = M[tri(i, k)];
            b1[i] = fma(-l, y1, b1[i]);
            if (NRHS > 1) b2[i] = fma(-l, y2, b2[i]);
        }
        if (lane == 0) {
            b1[k] = y1;
            if (NRHS > 1) b2[k] = y2;
        }
    }
    for (int k = s - 1; k >= 0; --k) {
        __syncwarp();
        double il = 1.0 / M[tri(k, k)];
        double x1 = b1[k] * il, x2 = NRHS > 1 ? b2[k] * il : 0.0;
        __syncwarp();
        for (int i = lane; i < k; i += 32) {
            double l = M[tri(k, i)];
            b1[i] = fma(-l, x1, b1[i]);
            if (NRHS > 1) b2[i] = fma(-l, x2, b2[i]);
        }
        if (lane == 0) {
            b1[k] = x1;
            if (NRHS > 1) b2[k] = x2;
        }
    }
    __syncwarp();
}

// _filter_vector (hx/precond.py:160-165) on a warp-resident vector
__device__ void prefilter(double* v, int s, double tau, int lane) {
    if (tau <= 0.0) return;
    double ss = 0.0;
    for (int i = lane; i < s; i += 32) ss += v[i] * v[i];
    ss = warp_sum(ss);
    double thr = tau * sqrt(ss);
    __syncwarp();
    for (int i = lane; i < s; i += 32)
        if (fabs(v[i]) < thr) v[i] = 0.0;
    __syncwarp();
}

// warp bitonic sort of n (power of two) ints in shared memory
__device__ void warp_sort(int* a, int n, int lane) {
    for (int k = 2; k <= n; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = lane; i < n; i += 32) {
                int l = i ^ j;
                if (l > i) {
                    int x = a[i], y = a[l];
                    bool up = (i & k) == 0;
                    if ((x > y) == up) { a[i] = y; a[l] = x; }
                }
            }
            __syncwarp();
        }
    }
}

template <int SMAX, int CMAX, bool DYN>
__global__ void __launch_bounds__(256) k_setup_rows(RowArgs a) {
    constexpr int MSZ = SMAX * (SMAX + 1) / 2;   // packed lower triangle
    extern __shared__ __align__(16) unsigned char smem[];
    const int warps = blockDim.x >> 5;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr size_t per_warp = sizeof(double) * (MSZ + 2 * SMAX + (DYN ? CMAX : 0)) +
                                sizeof(int) * (SMAX + (DYN ? CMAX + 8 : 0));
    unsigned char* base = smem + per_warp * wid;
    double* M = reinterpret_cast<double*>(base);
    double* bg = M + MSZ;
    double* bf = bg + SMAX;
    double* rv = bf + SMAX;                                   // CMAX (dynamic)
    int* q = reinterpret_cast<int*>(rv + (DYN ? CMAX : 0));   // SMAX
    int* cand = q + SMAX;                                     // CMAX (dynamic)
    int* misc = cand + (DYN ? CMAX : 0);                      // 8 ints

    for (int m = blockIdx.x * warps + wid; m < a.n_rows; m += gridDim.x * warps) {
        int s;
        if (!DYN) {
            int q0 = a.q_ptr[m];
            s = a.q_ptr[m + 1] - q0;
            if (s > SMAX) { if (lane == 0) report(a.err, ERR_SIZE, m); continue; }
            for (int i = lane; i < s; i += 32) q[i] = a.q_idx[q0 + i];
        } else {
            int r0 = a.Acf.ptr[m];
            s = a.Acf.ptr[m + 1] - r0;
            if (s + a.n_ent > SMAX) { if (lane == 0) report(a.err, ERR_SIZE, m); continue; }
            for (int i = lane; i < s; i += 32) q[i] = a.Acf.idx[r0 + i];   // canonical rows: sorted, unique
        }
        __syncwarp();
        gather_M(a.A, q, s, M, lane);
        gather_rhs(a.Acf, m, q, s, bg, lane);
        if (!DYN) gather_rhs(a.AfcT, m, q, s, bf, lane);
        bool ok = cholesky(M, s, lane);
        if (!ok) { if (lane == 0) report(a.err, ERR_FACT, m); continue; }
        if (!DYN) {
            chol_solve<2>(M, s, bg, bf, lane);
        } else {
            chol_solve<1>(M, s, bg, nullptr, lane);
            int added = 0, sweeps = 0;
            bool failed = false;
            while (added < a.n_ent && sweeps < a.sweep_limit) {
                ++sweeps;
                int budget = min(a.n_add, a.n_ent - added);
                // ---- candidate support: rhs pattern U rows touched by columns q (hx/precond.py:98-100)
                if (lane == 0) misc[0] = 0;
                __syncwarp();
                int r0 = a.Acf.ptr[m], r1 = a.Acf.ptr[m + 1];
                for (int e = r0 + lane; e < r1; e += 32) {
                    int p = atomicAdd(misc, 1);
                    if (p < CMAX) cand[p] = a.Acf.idx[e];
                }
                for (int i = lane; i < s; i += 32) {
                    int j = q[i];
                    for (int e = a.AT.ptr[j]; e < a.AT.ptr[j + 1]; ++e) {
                        int p = atomicAdd(misc, 1);
                        if (p < CMAX) cand[p] = a.AT.idx[e];
                    }
                }
                __syncwarp();
                int nc = misc[0];
                if (nc > CMAX) { failed = true; if (lane == 0) report(a.err, ERR_CAND, m); break; }
                int np2 = 32;
                while (np2 < nc) np2 <<= 1;
                for (int i = nc + lane; i < np2; i += 32) cand[i] = INT32_MAX;
                __syncwarp();
                warp_sort(cand, np2, lane);
                // ---- prolonged residual on fresh, unique candidates
                double best_r = 0.0;
                for (int i = lane; i < nc; i += 32) {
                    int c = cand[i];
                    double r = 0.0;
                    bool fresh = (i == 0 || cand[i - 1] != c) && bsearch(q, 0, s, c) < 0;
                    if (fresh) {
                        int p = bsearch(a.Acf.idx, r0, r1, c);
                        if (p >= 0) r = a.Acf.val[p];
                        for (int e = a.A.ptr[c]; e < a.A.ptr[c + 1]; ++e) {
                            int t = bsearch(q, 0, s, a.A.idx[e]);
                            if (t >= 0) r = add_mul(r, a.A.val[e], bg[t]);
                        }
                    }
                    rv[i] = fresh ? fabs(r) : 0.0;
                    best_r = fmax(best_r, rv[i]);
                }
                __syncwarp();
                // ---- pick up to `budget` entries by (|r| desc, index asc)
                int picked = 0;
                for (int t = 0; t < budget; ++t) {
                    double bv = 0.0;
                    int bi = INT32_MAX, bpos = -1;
                    for (int i = lane; i < nc; i += 32) {
                        double v = rv[i];
                        int c = cand[i];
                        if (v > bv || (v == bv && v > 0.0 && c < bi)) { bv = v; bi = c; bpos = i; }
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                        int op = __shfl_xor_sync(0xffffffffu, bpos, o);
                        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; bpos = op; }
                    }
                    if (!(bv > 0.0)) break;
                    if (lane == 0) {
                        rv[bpos] = 0.0;
                        misc[1 + picked] = bi;
                    }
                    __syncwarp();
                    ++picked;
                }
                if (picked == 0) break;   // nothing fresh: growth stops (hx/precond.py:129-130)
                if (lane == 0) {          // sorted insertion of the picks
                    for (int t = 0; t < picked; ++t) {
                        int v = misc[1 + t];
                        int p = s + t;
                        while (p > 0 && q[p - 1] > v) { q[p] = q[p - 1]; --p; }
                        q[p] = v;
                    }
                }
                __syncwarp();
                s += picked;
                added += picked;
                gather_M(a.A, q, s, M, lane);
                gather_rhs(a.Acf, m, q, s, bg, lane);
                if (!cholesky(M, s, lane)) { failed = true; if (lane == 0) report(a.err, ERR_FACT, m); break; }
                chol_solve<1>(M, s, bg, nullptr, lane);
                (void)best_r;
            }
            if (failed) continue;
            gather_rhs(a.AfcT, m, q, s, bf, lane);
            chol_solve<1>(M, s, bf, nullptr, lane);
        }
        prefilter(bg, s, a.pre_tau, lane);
        prefilter(bf, s, a.pre_tau, lane);
        int o = a.slot_ptr[m];
        int ng = 0, nf = 0;
        for (int i0 = 0; i0 < s; i0 += 32) {
            int i = i0 + lane;
            double g = i < s ? bg[i] : 0.0, f = i < s ? bf[i] : 0.0;
            if (i < s) {
                a.out_g[o + i] = g;
                a.out_f[o + i] = f;
                if (DYN) a.out_q[o + i] = q[i];
            }
            ng += __popc(__ballot_sync(0xffffffffu, i < s && g != 0.0));
            nf += __popc(__ballot_sync(0xffffffffu, i < s && f != 0.0));
        }
        if (lane == 0) {
            a.out_gcnt[m] = ng;
            a.out_fcnt[m] = nf;
            if (DYN) a.out_qsize[m] = s;
        }
        __syncwarp();
    }
}

// ---- static / base patterns: register-resident Cholesky (s <= 32)
//
// L = 8, 16 or 32 lanes per row (32 / L rows per warp).  Lane i of a row's
// segment owns row i of M = -A_ff[Q,Q] in registers (a[0..SMAX)); the
// factorisation is right-looking with the column entries l_jk broadcast by
// segment shuffles, so the only shared-memory traffic is the gather (a
// scatter of A_ff's rows into a per-row scratch tile) and the columns of L
// read by the backward substitution.  No __syncwarp per column.
template <int SMAX>
struct RegRow {
    static constexpr int L = SMAX <= 8 ? 8 : (SMAX <= 16 ? 16 : 32);   // lanes per row (>= SMAX)
    static constexpr int RPW = 32 / L;                                  // rows per warp
    static constexpr int LD = SMAX + 1;
    static constexpr size_t BYTES = sizeof(double) * (SMAX * LD + 2 * SMAX) + sizeof(int) * SMAX;
};

// blocks per SM: the static prototype-A rows (s = 18) run at 64 registers, eight blocks = 32 warps per SM
// (config 5, 256^3: 72 -> 64 ms; six blocks 68 ms); wider rows keep their ~100 registers
constexpr int rows_reg_min_blocks(int smax) { return smax == 18 ? 8 : 0; }   // 0: unspecified (the other instances keep their allocation)
template <int SMAX>
__global__ void __launch_bounds__(128, rows_reg_min_blocks(SMAX)) k_setup_rows_reg(RowArgs a) {
    using R = RegRow<SMAX>;
    constexpr int L = R::L, RPW = R::RPW, LD = R::LD;
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, seg = lane / L, li = lane % L;
    const int wid = threadIdx.x >> 5, warps = blockDim.x >> 5;
    const unsigned segmask = (L == 32) ? 0xffffffffu : (((1u << L) - 1u) << (seg * L));
    unsigned char* base = smem + (size_t)(wid * RPW + seg) * R::BYTES;
    double* M = reinterpret_cast<double*>(base);
    double* bg = M + SMAX * LD;
    double* bf = bg + SMAX;
    int* q = reinterpret_cast<int*>(bf + SMAX);
    const int n_groups = (a.n_rows + RPW - 1) / RPW;
    for (int grp = blockIdx.x * warps + wid; grp < n_groups; grp += gridDim.x * warps) {
        const int m = grp * RPW + seg;
        const bool row_ok = m < a.n_rows;
        int s = 0, q0 = 0;
        if (row_ok) {
            q0 = a.q_ptr[m];
            s = a.q_ptr[m + 1] - q0;
        }
        int s_w = s;                                   // warp-uniform loop bound
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s_w = max(s_w, __shfl_xor_sync(0xffffffffu, s_w, o));
        // ---- gather: q, the scratch tile, the two right-hand sides
        if (li < s) q[li] = a.q_idx[q0 + li];
        for (int t = li; t < s * LD; t += L) M[t] = 0.0;
        (void)s_w;
        if (li < SMAX) { bg[li] = 0.0; bf[li] = 0.0; }
        __syncwarp();
        if (li < s) {   // the row's entries are loaded in batches of 12 (all in flight), then
                        // merged with the sorted set (both ascending: one forward walk, no search)
            const int row = q[li];
            const int e0 = a.A.ptr[row], e1 = a.A.ptr[row + 1];
            int j = 0;
            for (int eb = e0; eb < e1; eb += 12) {
                int ci[12];
                double cv[12];
#pragma unroll
                for (int u = 0; u < 12; ++u) {
                    ci[u] = eb + u < e1 ? a.A.idx[eb + u] : INT32_MAX;
                    cv[u] = eb + u < e1 ? a.A.val[eb + u] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 12; ++u) {
                    while (j < s && q[j] < ci[u]) ++j;
                    if (j < s && q[j] == ci[u]) M[li * LD + j] = -cv[u];
                }
            }
        }
        if (row_ok) {
            for (int e = a.Acf.ptr[m] + li; e < a.Acf.ptr[m + 1]; e += L) {
                const int j = bsearch(q, 0, s, a.Acf.idx[e]);
                if (j >= 0) bg[j] = a.Acf.val[e];
            }
            for (int e = a.AfcT.ptr[m] + li; e < a.AfcT.ptr[m + 1]; e += L) {
                const int j = bsearch(q, 0, s, a.AfcT.idx[e]);
                if (j >= 0) bf[j] = a.AfcT.val[e];
            }
        }
        __syncwarp();
        // the s x s block padded to SMAX with an identity: every loop below is
        // straight-line code over the compile-time size (padded unknowns solve to 0)
        double r[SMAX];
#pragma unroll
        for (int j = 0; j < SMAX; ++j) r[j] = (li < s && j < s) ? M[li * LD + j] : (j == li ? 1.0 : 0.0);
        double yg = li < s ? bg[li] : 0.0, yf = li < s ? bf[li] : 0.0;
        // ---- right-looking Cholesky, lane i holds row i; column k of L goes
        // through a shared-memory line (broadcast reads).  Lanes update their
        // whole row (the upper part is never read), so no per-entry predicates.
        double inv_self = 0.0;
        bool bad = false;
        double* colk = bg;                             // bg / bf are in registers now: reuse as the line
        __syncwarp();
#pragma unroll
        for (int k = 0; k < SMAX; ++k) {
            const double dkk = __shfl_sync(0xffffffffu, r[k], seg * L + k);
            bad |= !(dkk > 0.0);
            const double ik = rsqrt(dkk), lkk = dkk * ik;
            if (li > k) r[k] *= ik;
            if (li == k) { r[k] = lkk; inv_self = ik; }
            if (li < SMAX) colk[li] = r[k];
            __syncwarp();
#pragma unroll
            for (int j = k + 1; j < SMAX; ++j) r[j] = fma(-r[k], colk[j], r[j]);
            __syncwarp();
        }
        bad = bad && row_ok;
        if (__any_sync(0xffffffffu, bad)) {
            if (bad && li == 0) report(a.err, ERR_FACT, m);
            continue;                                  // the build raises; values are not used
        }
        // ---- forward substitution L y = b (both right-hand sides)
#pragma unroll
        for (int k = 0; k < SMAX; ++k) {
            if (li == k) { yg *= inv_self; yf *= inv_self; }
            const double vg = __shfl_sync(0xffffffffu, yg, seg * L + k);
            const double vf = __shfl_sync(0xffffffffu, yf, seg * L + k);
            if (li > k) { yg = fma(-r[k], vg, yg); yf = fma(-r[k], vf, yf); }
        }
        // ---- backward substitution L^T x = y: columns of L from the scratch tile
#pragma unroll
        for (int j = 0; j < SMAX; ++j)
            if (j < li && li < SMAX) M[li * LD + j] = r[j];
        __syncwarp();
#pragma unroll
        for (int k = SMAX - 1; k >= 0; --k) {
            if (li == k) { yg *= inv_self; yf *= inv_self; }
            const double vg = __shfl_sync(0xffffffffu, yg, seg * L + k);
            const double vf = __shfl_sync(0xffffffffu, yf, seg * L + k);
            if (li < k) {
                const double l = M[k * LD + li];
                yg = fma(-l, vg, yg);
                yf = fma(-l, vf, yf);
            }
        }
        // ---- pre-filter (hx/precond.py:160-165), slot-layout output, nonzero counts
        if (a.pre_tau > 0.0) {
            double sg = li < s ? yg * yg : 0.0, sf = li < s ? yf * yf : 0.0;
#pragma unroll
            for (int o = L / 2; o > 0; o >>= 1) {
                sg += __shfl_xor_sync(0xffffffffu, sg, o);
                sf += __shfl_xor_sync(0xffffffffu, sf, o);
            }
            const double tg = a.pre_tau * sqrt(sg), tf = a.pre_tau * sqrt(sf);
            if (fabs(yg) < tg) yg = 0.0;
            if (fabs(yf) < tf) yf = 0.0;
        }
        const bool live = row_ok && li < s;
        if (live) {
            const int o = a.slot_ptr[m];
            a.out_g[o + li] = yg;
            a.out_f[o + li] = yf;
        }
        const unsigned bgm = __ballot_sync(0xffffffffu, live && yg != 0.0) & segmask;
        const unsigned bfm = __ballot_sync(0xffffffffu, live && yf != 0.0) & segmask;
        if (row_ok && li == 0) {
            a.out_gcnt[m] = __popc(bgm);
            a.out_fcnt[m] = __popc(bfm);
        }
        __syncwarp();
    }
}

template <int SMAX>
void launch_rows_reg(Ctx* c, const RowArgs& a) {
    using R = RegRow<SMAX>;
    constexpr int warps = 4;
    const size_t sm = R::BYTES * R::RPW * warps;
    auto kern = k_setup_rows_reg<SMAX>;
    static std::mutex mu;
    static std::set<int> done;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (done.insert(c->device).second)
            EDFA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    }
    const int groups = ceil_div(a.n_rows, R::RPW);
    const int blocks = std::max(1, std::min(ceil_div(groups, warps), NUM_SMS_B200 * 64));
    kern<<<blocks, warps * 32, sm, c->stream>>>(a);
    check_launch("k_setup_rows_reg");
}

// compaction of slot-layout values into canonical CSR rows (zeros dropped)
__global__ void k_compact(int32_t n_rows, const int32_t* __restrict__ slot_ptr, const int32_t* __restrict__ qsize,
                          const int32_t* __restrict__ qidx, const double* __restrict__ v,
                          const int32_t* __restrict__ out_ptr, int32_t* __restrict__ out_idx,
                          double* __restrict__ out_val) {
    int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= n_rows) return;
    int o = slot_ptr[w], s = qsize ? qsize[w] : slot_ptr[w + 1] - o, d = out_ptr[w];
    for (int i0 = 0; i0 < s; i0 += 32) {
        int i = i0 + lane;
        double x = i < s ? v[o + i] : 0.0;
        bool keep = i < s && x != 0.0;
        unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            int p = d + __popc(bal & ((1u << lane) - 1));
            out_idx[p] = qidx[o + i];
            out_val[p] = x;
        }
        d += __popc(bal);
    }
}

__global__ void k_slot_ptr_dyn(const int32_t* __restrict__ acf_ptr, int32_t n, int32_t n_ent,
                               int32_t* __restrict__ slot_ptr) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i <= n) slot_ptr[i] = acf_ptr[i] + (int32_t)i * n_ent;
}

// ---- static prototype patterns (hx/patterns.py:63-133), thread per cell
template <bool FILL>
__global__ void k_static_pattern(int32_t n_cells, const int32_t* __restrict__ e2f, const int32_t* __restrict__ nbr,
                                 const int32_t* __restrict__ fidx, char proto, int32_t* __restrict__ cnt,
                                 const int32_t* __restrict__ out_ptr, int32_t* __restrict__ out_idx) {
    int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= n_cells) return;
    int f[64];
    int n = 0;
    auto add = [&](int gface) {
        int r = fidx[gface];
        if (r >= 0 && n < 64) f[n++] = r;
    };
    for (int s = 0; s < 6; ++s) add(e2f[m * 6 + s]);
    auto chain = [&](int slot, int depth) {
        int cur = m;
        for (int t = 0; t < depth; ++t) {
            cur = nbr[cur * 6 + slot];
            if (cur < 0) return;
            add(e2f[cur * 6 + slot]);
        }
    };
    if (proto == 'A' || proto == 'B' || proto == 'E') {
        int depth = proto == 'A' ? 2 : (proto == 'B' ? 3 : 1);
        for (int s = 0; s < 6; ++s) chain(s, depth);
        if (proto == 'E')
            for (int s = 0; s < 6; ++s) {
                int nb = nbr[m * 6 + s];
                if (nb >= 0) add(e2f[nb * 6 + 2 * (((s >> 1) + 1) % 3) + (s & 1)]);
            }
    } else {
        for (int s = 0; s < 6; ++s) {
            int nb = nbr[m * 6 + s];
            if (nb >= 0)
                for (int t = 0; t < 6; ++t) add(e2f[nb * 6 + t]);
        }
        if (proto == 'D')
            for (int s = 0; s < 6; ++s) chain(s, 2);
    }
    for (int i = 1; i < n; ++i) {   // insertion sort
        int v = f[i], j = i - 1;
        while (j >= 0 && f[j] > v) { f[j + 1] = f[j]; --j; }
        f[j + 1] = v;
    }
    int u = 0;
    for (int i = 0; i < n; ++i)
        if (i == 0 || f[i] != f[i - 1]) {
            if (FILL) out_idx[out_ptr[m] + u] = f[i];
            ++u;
        }
    if (!FILL) cnt[m] = u;
}

size_t warp_smem(int smax, int cmax, bool dyn) {
    return sizeof(double) * (smax * (smax + 1) / 2 + 2 * smax + (dyn ? cmax : 0)) +
           sizeof(int) * (smax + (dyn ? cmax + 8 : 0));
}

template <int SMAX, int CMAX, bool DYN>
void launch_rows(Ctx* c, const RowArgs& a) {
    size_t pw = warp_smem(SMAX, CMAX, DYN);
    int warps = (int)std::max<size_t>(1, std::min<size_t>(8, (220 * 1024) / pw));
    size_t sm = pw * warps;
    auto kern = k_setup_rows<SMAX, CMAX, DYN>;
    EDFA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    int per_sm = std::max(1, (int)((227 * 1024) / sm));
    int blocks = std::max(1, std::min(ceil_div(a.n_rows, warps), NUM_SMS_B200 * per_sm * 4));
    kern<<<blocks, warps * 32, sm, c->stream>>>(a);
    check_launch("k_setup_rows");
}

}  // namespace

int max_row_nnz(Ctx* c, const Csr& A);   // objects.cu

void setup_rows(Ctx* c, const SetupInput& in, SetupOutput& out) {
    const int n = in.Acf->n_rows;
    RowArgs a{};
    a.A = view(*in.A);
    a.AT = in.AT ? view(*in.AT) : view(*in.A);
    a.Acf = view(*in.Acf);
    a.AfcT = view(*in.AfcT);
    a.n_rows = n;
    a.pre_tau = in.pre_tau;
    out.slot_ptr.reset(c, (size_t)n + 1);
    out.gcnt.reset(c, std::max(n, 1));
    out.fcnt.reset(c, std::max(n, 1));
    int smax_need;
    const bool dyn = in.pattern == nullptr;
    if (!dyn) {
        a.q_ptr = in.pattern->ptr.p;
        a.q_idx = in.pattern->idx.p;
        EDFA_CUDA(cudaMemcpyAsync(out.slot_ptr.p, in.pattern->ptr.p, sizeof(int32_t) * (n + 1),
                                  cudaMemcpyDeviceToDevice, c->stream));
        smax_need = max_row_nnz(c, *in.pattern);
        out.n_slots = in.pattern->nnz;
    } else {
        a.n_add = in.n_add;
        a.n_ent = in.n_ent;
        a.sweep_limit = in.sweep_limit;
        if (n) k_slot_ptr_dyn<<<ceil_div(n + 1, 256), 256, 0, c->stream>>>(in.Acf->ptr.p, n, in.n_ent, out.slot_ptr.p);
        check_launch("k_slot_ptr_dyn");
        smax_need = max_row_nnz(c, *in.Acf) + in.n_ent;
        out.n_slots = in.Acf->nnz + (int64_t)n * in.n_ent;
        out.q.reset(c, std::max<int64_t>(out.n_slots, 1));
        out.qsize.reset(c, std::max(n, 1));
    }
    out.max_pattern = smax_need;
    require(smax_need <= 128, EDFA_ERR_UNSUPPORTED,
            "restriction sets larger than 128 faces are not supported (got " + std::to_string(smax_need) + ")");
    out.g.reset(c, std::max<int64_t>(out.n_slots, 1));
    out.f.reset(c, std::max<int64_t>(out.n_slots, 1));
    a.slot_ptr = out.slot_ptr.p;
    a.out_q = out.q.p;
    a.out_qsize = out.qsize.p;
    a.out_g = out.g.p;
    a.out_f = out.f.p;
    a.out_gcnt = out.gcnt.p;
    a.out_fcnt = out.fcnt.p;
    int* err = c->d_scalar_i;
    int init[2] = {0, INT32_MAX};
    EDFA_CUDA(cudaMemcpyAsync(err, init, sizeof init, cudaMemcpyHostToDevice, c->stream));
    a.err = err;
    if (n == 0) return;
    int amax = dyn ? max_row_nnz(c, *in.A) : 0;
    int cand_need = dyn ? smax_need * std::max(amax, in.AT ? max_row_nnz(c, *in.AT) : amax) + max_row_nnz(c, *in.Acf) : 0;
    if (PhaseTimer::enabled())
        fprintf(stderr, "[edfa phase] setup_rows: dyn=%d smax_need=%d amax=%d cand_need=%d n_add=%d n_ent=%d\n", (int)dyn,
                smax_need, amax, cand_need, (int)in.n_add, (int)in.n_ent);
    double bytes = 12.0 * in.Acf->nnz + 12.0 * in.AfcT->nnz + 16.0 * out.n_slots + 8.0 * n +
                   (dyn ? 0.0 : 4.0 * out.n_slots) + 12.0 * (double)out.n_slots * 3.0;
    {
        Prof pr(c, dyn ? "setup_rows_dynamic" : "setup_rows_static", bytes);
        if (!dyn) {
            // the smallest register-row size >= the largest set (prototype A: 18, B/E: 24, base: 6-12)
            if (smax_need <= 8) launch_rows_reg<8>(c, a);
            else if (smax_need <= 12) launch_rows_reg<12>(c, a);
            else if (smax_need <= 16) launch_rows_reg<16>(c, a);
            else if (smax_need <= 18) launch_rows_reg<18>(c, a);
            else if (smax_need <= 24) launch_rows_reg<24>(c, a);
            else if (smax_need <= 32) launch_rows_reg<32>(c, a);
            else if (smax_need <= 64) launch_rows<64, 0, false>(c, a);
            else launch_rows<128, 0, false>(c, a);
        } else {
            require(cand_need <= 4096, EDFA_ERR_UNSUPPORTED, "dynamic candidate support exceeds 4096 entries");
            // shared memory per warp sets the residency: <64, 1024> fits one 4-warp block per
            // SM (6 % warps active in ncu, profiles/r02h), <32, 1024> two
            if (smax_need <= 32 && cand_need <= 512) launch_rows<32, 512, true>(c, a);
            else if (smax_need <= 32 && cand_need <= 1024) launch_rows<32, 1024, true>(c, a);
            else if (smax_need <= 64 && cand_need <= 1024) launch_rows<64, 1024, true>(c, a);
            else if (smax_need <= 64) launch_rows<64, 4096, true>(c, a);
            else launch_rows<128, 4096, true>(c, a);
        }
    }
    int h_err[2];
    EDFA_CUDA(cudaMemcpyAsync(h_err, err, sizeof h_err, cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
    if (h_err[0] == ERR_FACT)
        throw Error(EDFA_ERR_FACTORIZATION, "dense Cholesky failed: restricted block of row " +
                                                std::to_string(h_err[1]) + " is not positive definite");
    if (h_err[0] == ERR_CAND)
        throw Error(EDFA_ERR_UNSUPPORTED, "dynamic candidate support overflow at row " + std::to_string(h_err[1]));
    if (h_err[0] == ERR_SIZE)
        throw Error(EDFA_ERR_UNSUPPORTED, "restriction set too large at row " + std::to_string(h_err[1]));
}

void compact_rows(Ctx* c, int32_t n, const DevBuf<int32_t>& slot_ptr, const int32_t* qsize, const int32_t* qidx,
                  const double* vals, const DevBuf<int32_t>& cnt, int32_t n_cols, Csr& out) {
    out.n_rows = n;
    out.n_cols = n_cols;
    out.ptr.reset(c, (size_t)n + 1);
    out.nnz = scan_counts(c, cnt.p, out.ptr.p, n);
    out.idx.reset(c, out.nnz);
    out.val.reset(c, out.nnz);
    if (n == 0) return;
    Prof pr(c, "compact", 12.0 * out.nnz + 12.0 * out.nnz);
    k_compact<<<ceil_div((int64_t)n * 32, 256), 256, 0, c->stream>>>(n, slot_ptr.p, qsize, qidx, vals, out.ptr.p,
                                                                    out.idx.p, out.val.p);
    check_launch("k_compact");
}

void copy_rows(Ctx* c, int32_t n, const int32_t* sp, const int32_t* sz, const int32_t* src, const int32_t* dp,
               int32_t* dst);

void pattern_compact(Ctx* c, int32_t n, const DevBuf<int32_t>& slot_ptr, const DevBuf<int32_t>& qsize,
                     const DevBuf<int32_t>& q, int32_t n_cols, Csr& out) {
    // final dynamic sets as a pattern CSR (values NULL)
    out.n_rows = n;
    out.n_cols = n_cols;
    out.ptr.reset(c, (size_t)n + 1);
    out.nnz = scan_counts(c, qsize.p, out.ptr.p, n);
    out.idx.reset(c, out.nnz);
    out.val.release();
    if (n) copy_rows(c, n, slot_ptr.p, qsize.p, q.p, out.ptr.p, out.idx.p);
}

namespace {
__global__ void k_copy_rows(int32_t n, const int32_t* __restrict__ sp, const int32_t* __restrict__ sz,
                            const int32_t* __restrict__ src, const int32_t* __restrict__ dp,
                            int32_t* __restrict__ dst) {
    int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= n) return;
    for (int i = lane; i < sz[w]; i += 32) dst[dp[w] + i] = src[sp[w] + i];
}
// cell -> faces (narrowed to int32) and cell -> neighbour across each face
// (hx/grid.py:100-129: face_to_elems[f] = (lower cell, upper cell or -1))
template <typename I>
__global__ void k_grid_topology(int32_t n_cells, int32_t n_faces, const I* __restrict__ e2f,
                                const I* __restrict__ f2e, const I* __restrict__ fidx, int32_t* __restrict__ e2f_out,
                                int32_t* __restrict__ nbr_out, int32_t* __restrict__ fidx_out) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < (int64_t)n_cells * 6) {
        const int32_t e = (int32_t)(t / 6);
        const int32_t f = (int32_t)e2f[t];
        const int32_t a = (int32_t)f2e[2 * (int64_t)f], b = (int32_t)f2e[2 * (int64_t)f + 1];
        e2f_out[t] = f;
        nbr_out[t] = a == e ? b : a;
    }
    if (fidx_out && t < n_faces) fidx_out[t] = (int32_t)fidx[t];
}

}  // namespace

void grid_topology(Ctx* c, int32_t n_cells, int32_t n_faces, const void* e2f, const void* f2e, const void* fidx,
                   int index_bytes, int32_t* e2f_out, int32_t* nbr_out, int32_t* fidx_out) {
    require(index_bytes == 4 || index_bytes == 8, EDFA_ERR_VALUE, "index_bytes must be 4 or 8");
    const int64_t work = std::max<int64_t>((int64_t)n_cells * 6, n_faces);
    if (work == 0) return;
    Prof pr(c, "grid_topology", (index_bytes + 12.0) * 6 * n_cells + (index_bytes + 4.0) * n_faces);
    const int blocks = (int)ceil_div(work, (int64_t)256);
    if (index_bytes == 8)
        k_grid_topology<int64_t><<<blocks, 256, 0, c->stream>>>(
            n_cells, n_faces, static_cast<const int64_t*>(e2f), static_cast<const int64_t*>(f2e),
            static_cast<const int64_t*>(fidx), e2f_out, nbr_out, fidx ? fidx_out : nullptr);
    else
        k_grid_topology<int32_t><<<blocks, 256, 0, c->stream>>>(
            n_cells, n_faces, static_cast<const int32_t*>(e2f), static_cast<const int32_t*>(f2e),
            static_cast<const int32_t*>(fidx), e2f_out, nbr_out, fidx ? fidx_out : nullptr);
    check_launch("k_grid_topology");
}

void copy_rows(Ctx* c, int32_t n, const int32_t* sp, const int32_t* sz, const int32_t* src, const int32_t* dp,
               int32_t* dst) {
    Prof pr(c, "compact", 8.0 * n);
    k_copy_rows<<<ceil_div((int64_t)n * 32, 256), 256, 0, c->stream>>>(n, sp, sz, src, dp, dst);
    check_launch("k_copy_rows");
}

void static_pattern(Ctx* c, int32_t n_cells, int32_t n_free, const int32_t* e2f, const int32_t* nbr,
                    const int32_t* fidx, char proto, Csr& out) {
    require(proto >= 'A' && proto <= 'E', EDFA_ERR_VALUE,
            std::string("unknown prototype '") + proto + "'; expected one of A..E");
    out.n_rows = n_cells;
    out.n_cols = n_free;
    out.ptr.reset(c, (size_t)n_cells + 1);
    DevBuf<int32_t> cnt(c, std::max(n_cells, 1));
    if (n_cells) {
        Prof pr(c, "static_pattern", 56.0 * n_cells);
        k_static_pattern<false><<<ceil_div(n_cells, 128), 128, 0, c->stream>>>(n_cells, e2f, nbr, fidx, proto, cnt.p,
                                                                              nullptr, nullptr);
        check_launch("k_static_pattern");
    }
    out.nnz = scan_counts(c, cnt.p, out.ptr.p, n_cells);
    out.idx.reset(c, out.nnz);
    out.val.release();
    if (n_cells) {
        Prof pr(c, "static_pattern", 56.0 * n_cells + 4.0 * out.nnz);
        k_static_pattern<true><<<ceil_div(n_cells, 128), 128, 0, c->stream>>>(n_cells, e2f, nbr, fidx, proto, nullptr,
                                                                             out.ptr.p, out.idx.p);
        check_launch("k_static_pattern");
    }
}

}  // namespace edfa
