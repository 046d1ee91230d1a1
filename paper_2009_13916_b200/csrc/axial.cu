// Pencil solver for cell-indexed triangular factors with an axial stencil
// (InnerFactorization.apply of the Schur ILU, hx/sparse.py:125-129).
//
// With base/static restriction patterns on a structured grid the Schur
// complement couples a cell only to cells on its own grid lines, up to R
// cells away (R = 6 for prototype A), so row (i,j,k) of L depends on
// (i-d,j,k), (i,j-d,k), (i,j,k-d), d = 1..R (U: the mirror image; it is solved
// here in reversed coordinates).  The dependency DAG is a 3-D wavefront of
// depth nx+ny+nz; what limits a GPU solve is the hand-off latency per
// wavefront step, not bandwidth.
//
// Layout: every lane owns one x-pencil (fixed j,k) and walks it cell by cell,
// skewed by j+k inside its CTA, so at every step
//   * the x-neighbours (i-d) are the lane's own previous results (registers),
//   * the y/z-neighbours inside the CTA's 8x8 (j,k) block were produced by
//     other lanes 1..R steps ago (shared-memory ring, one barrier per step),
//   * neighbours in the upstream blocks arrive through a halo ring in shared
//     memory that a loader warp fills from HBM (the solution vector is
//     SENTINEL-filled, so a stored value is its own ready flag).
// Coefficients are permuted once per factorisation into [block][step][slot]
// [lane] order, so one TMA bulk copy per step stages a step's 19 coefficient
// rows (coalesced, prefetched AX_P steps ahead); the right-hand side is
// prefetched AX_PB steps ahead with cp.async.  A step's critical path is one
// shared-memory round trip, three FMAs and a barrier.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "dev_util.cuh"
#include "edfa_internal.cuh"
#include "objects.cuh"

namespace edfa {
namespace {

constexpr int AX_BJ = 8, AX_BK = 8, AX_T = AX_BJ * AX_BK;   // pencils per block
constexpr int AX_CW = 4 * AX_T / 32;                          // compute warps (four lanes per pencil)
constexpr int AX_THREADS = (AX_CW + 1) * 32;                  // + loader warp
constexpr int AX_P = 8;      // coefficient stages in flight (TMA)
constexpr int AX_PB = 8;     // right-hand-side prefetch distance (cp.async)
constexpr int AX_W = 64;     // halo ring length along the pencil
constexpr int AX_RMAX = 8;
#ifndef AX_EXP_NOWAIT
#define AX_EXP_NOWAIT 0    // experiments only: skip the coefficient-stage wait (wrong results)
#endif
#ifndef AX_EXP_NOB
#define AX_EXP_NOB 0       // experiments: right-hand side by direct loads instead of cp.async
#endif

struct AxGeo {
    int nx, ny, nz, NJ, NK, nsteps, R, NC;
    int reverse;
};

__host__ __device__ __forceinline__ int ax_nat(const AxGeo& g, int i, int j, int k) {
    return g.reverse ? (g.nx - 1 - i) + g.nx * ((g.ny - 1 - j) + g.ny * (g.nz - 1 - k)) : i + g.nx * (j + g.ny * k);
}
__device__ __forceinline__ void ax_coords(const AxGeo& g, int row, int& i, int& j, int& k) {
    i = row % g.nx;
    j = (row / g.nx) % g.ny;
    k = row / (g.nx * g.ny);
    if (g.reverse) { i = g.nx - 1 - i; j = g.ny - 1 - j; k = g.nz - 1 - k; }
}

// every dependency must be (i-d,j,k) / (i,j-d,k) / (i,j,k-d) in solver
// coordinates with 1 <= d <= AX_RMAX; maxr = the largest d seen
__global__ void k_ax_check(CsrV D, AxGeo g, int* __restrict__ bad, int* __restrict__ maxr) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= D.n_rows) return;
    int i, j, k;
    ax_coords(g, r, i, j, k);
    int m = 0;
    for (int e = D.ptr[r]; e < D.ptr[r + 1]; ++e) {
        int ci, cj, ck;
        ax_coords(g, D.idx[e], ci, cj, ck);
        const int di = i - ci, dj = j - cj, dk = k - ck;
        const int nz = (di != 0) + (dj != 0) + (dk != 0);
        const int d = di + dj + dk;
        if (nz != 1 || d < 1 || d > AX_RMAX) { atomicExch(bad, 1); return; }
        m = max(m, d);
    }
    if (m) atomicMax(maxr, m);
}

// coef[((blk * nsteps + s) * NC + o) * T + t]: o = x(d-1) | y(R+d-1) | z(2R+d-1) | 1/diag (3R)
__global__ void k_ax_fill(CsrV D, AxGeo g, const double* __restrict__ diag, int unit, double* __restrict__ coef) {
    const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)g.NJ * g.NK * g.nsteps * AX_T;
    if (gid >= total) return;
    const int t = (int)(gid % AX_T);
    const int64_t bs = gid / AX_T;
    const int s = (int)(bs % g.nsteps);
    const int blk = (int)(bs / g.nsteps);
    const int J = blk % g.NJ, K = blk / g.NJ;
    const int jl = t % AX_BJ, kl = t / AX_BJ;
    const int j = J * AX_BJ + jl, k = K * AX_BK + kl, i = s - jl - kl;
    double* out = coef + (bs * g.NC) * AX_T + t;
    for (int o = 0; o < g.NC; ++o) out[(int64_t)o * AX_T] = 0.0;
    if (j >= g.ny || k >= g.nz || i < 0 || i >= g.nx) return;
    const int row = ax_nat(g, i, j, k);
    out[(int64_t)(3 * g.R) * AX_T] = (unit || !diag) ? 1.0 : 1.0 / diag[row];
    for (int e = D.ptr[row]; e < D.ptr[row + 1]; ++e) {
        int ci, cj, ck;
        ax_coords(g, D.idx[e], ci, cj, ck);
        const int di = i - ci, dj = j - cj, dk = k - ck;
        const int o = di ? di - 1 : dj ? g.R + dj - 1 : 2 * g.R + dk - 1;
        out[(int64_t)o * AX_T] = D.val[e];
    }
}

struct AxSolve {
    AxGeo g;
    const double* coef;
    const int* order;     // block ticket order (anti-diagonals)
    int* ticket;
    int ticket_base;
    const double* b;
    double alpha;
    double* x;
    const double* add;
    double* out2;
    int* err;
    long long* dbg;       // diagnostics: [block][nsteps] time after each step's barrier
};

__device__ __forceinline__ long long ax_gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned ax_saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ double ax_lds(const double* p) { return *reinterpret_cast<const volatile double*>(p); }
__device__ __forceinline__ void ax_sts(double* p, double v) { *reinterpret_cast<volatile double*>(p) = v; }
__device__ __forceinline__ double ax_halo(const double* p, int* err) {
    double v = ax_lds(p);
    if (is_sentinel(v)) {
        long long spins = 0;
        do {
            if (++spins > SPIN_LIMIT) { atomicExch(err, 7); return 0.0; }
            __nanosleep(16);
            v = ax_lds(p);
        } while (is_sentinel(v));
    }
    return v;
}
__device__ __forceinline__ bool is_sent_hi(double v) {   // published values are never NaN-boxed like this
    return __double2hiint(v) == (int)(SENTINEL_BITS >> 32);
}
__device__ __forceinline__ void ax_bar() { asm volatile("bar.sync 1, %0;" ::"n"(4 * AX_T) : "memory"); }

template <int R>
__global__ void __launch_bounds__(AX_THREADS) k_ax_solve(AxSolve a) {
    constexpr int NC = 3 * R + 1;
    constexpr int RR = R + 1 <= 8 ? 8 : 16;   // x ring (power of two >= R+1)
    extern __shared__ __align__(128) unsigned char sm[];
    double* cf = reinterpret_cast<double*>(sm);                  // [P][NC][T]
    double* xr = cf + AX_P * NC * AX_T;                           // [RR][T]
    double* hy = xr + RR * AX_T;                                  // [R][BK][W]
    double* hz = hy + R * AX_BK * AX_W;                           // [R][BJ][W]
    double* br = hz + R * AX_BJ * AX_W;                           // [PB][T]
    double* zc = br + AX_PB * AX_T;                               // [R][T] zeros (dummy lanes)
    __shared__ __align__(8) uint64_t mbar[AX_P];
    __shared__ int s_blk;
    __shared__ volatile int s_prog;
    __shared__ int rdy_y[AX_BK], rdy_z[AX_BJ];   // halo pencils present below i (per kl / jl)
    const AxGeo& g = a.g;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int q = 0; q < AX_P; ++q)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(ax_saddr(&mbar[q])), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const double sent = __longlong_as_double((long long)SENTINEL_BITS);
    const unsigned stage_bytes = NC * AX_T * 8;
    const int dstep = g.reverse ? -1 : 1;   // natural-index step along a pencil
    long long gs0 = 0;   // steps issued on this CTA's stage ring so far (slot = gs % P)
    for (;;) {
        if (tid == 0) {
            const int q = atomicAdd(a.ticket, 1) - a.ticket_base;
            s_blk = q < g.NJ * g.NK ? a.order[q] : -1;
            s_prog = -1;
        }
        __syncthreads();
        const int blk = s_blk;
        if (blk < 0) break;
        const int J = blk % g.NJ, K = blk / g.NJ;
        const double* cblk = a.coef + (int64_t)blk * g.nsteps * NC * AX_T;
        // coefficient stage of step s -> ring slot (gs0 + s) % P (TMA bulk copy)
        auto stage = [&](int s) {
            const int q = (int)((gs0 + s) % AX_P);
            uint64_t* mb = &mbar[q];
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ax_saddr(mb)),
                         "r"(stage_bytes) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(ax_saddr(cf + q * NC * AX_T)), "l"(cblk + (int64_t)s * NC * AX_T),
                         "r"(stage_bytes), "r"(ax_saddr(mb)) : "memory");
        };
        const int pre = min(AX_P, g.nsteps);
        if (tid == 0) {   // stage the first P steps; the loader warp stages the rest
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            for (int s = 0; s < pre; ++s) stage(s);
        }
        // halo rings: SENTINEL where an upstream block exists (not read before
        // its ready counter passes it), 0 where the grid ends
        for (int q = tid; q < R * AX_BK * AX_W; q += AX_THREADS) hy[q] = J > 0 ? sent : 0.0;
        for (int q = tid; q < R * AX_BJ * AX_W; q += AX_THREADS) hz[q] = K > 0 ? sent : 0.0;
        for (int q = tid; q < RR * AX_T; q += AX_THREADS) xr[q] = 0.0;   // x history before i = 0
        for (int q = tid; q < R * AX_T; q += AX_THREADS) zc[q] = 0.0;
        if (tid < AX_BK) rdy_y[tid] = (J > 0 && K * AX_BK + tid < g.nz) ? 0 : 1 << 30;
        if (tid < AX_BJ) rdy_z[tid] = (K > 0 && J * AX_BJ + tid < g.ny) ? 0 : 1 << 30;
        __syncthreads();
        if (warp == AX_CW) {
            // ---- loader.  Lane kl (< BK) copies the R y-halo pencils (J*BJ-dd, K*BK+kl),
            // lane BK+jl the R z-halo pencils (J*BJ+jl, K*BK-dd), each walked in
            // pencil order, and publishes (release) how far all R are present.
            // Ring slot i % W is reset once every consumer of i - W has passed it.
            const bool isy = lane < AX_BK, isz = lane >= AX_BK && lane < AX_BK + AX_BJ;
            const int ll = isy ? lane : lane - AX_BK;
            const bool act = (isy && J > 0 && K * AX_BK + ll < g.nz) || (isz && K > 0 && J * AX_BJ + ll < g.ny);
            int cur = act ? 0 : g.nx;
            double* base = isy ? hy + ll * AX_W : hz + ll * AX_W;   // + (dd-1)*{BK,BJ}*W + i%W
            const int dstr = isy ? AX_BK * AX_W : AX_BJ * AX_W;
            int* rdy = isy ? &rdy_y[ll] : &rdy_z[ll];
            int rst = AX_W;    // slots of i < rst hold (or await) the value of i
            int staged = pre;  // lane 0: coefficient stages issued
            long long spins = 0;
            for (;;) {
                bool todo = cur < g.nx, prog = false;
                const int sp = s_prog;
                if (lane == 0 && staged < g.nsteps) {
                    // a slot is free once the compute lanes passed the step that used it
                    if (sp >= staged - AX_P) {
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        while (staged < g.nsteps && sp >= staged - AX_P) stage(staged++);
                        prog = true;
                    }
                    todo |= staged < g.nsteps;
                }
                if (act) {
                    while (rst < g.nx && sp > rst - AX_W + (AX_BJ - 1) + (AX_BK - 1)) {
#pragma unroll
                        for (int dd = 0; dd < R; ++dd) ax_sts(base + dd * dstr + rst % AX_W, sent);
                        ++rst;
                    }
                }
                if (cur < g.nx) {
                    constexpr int LA = 4;
                    const int lim = min(min(cur + LA, g.nx), rst);
                    double v[R][LA];
#pragma unroll
                    for (int dd = 0; dd < R; ++dd) {
                        const int jj = isy ? J * AX_BJ - dd - 1 : J * AX_BJ + ll;
                        const int kk = isy ? K * AX_BK + ll : K * AX_BK - dd - 1;
                        const int r0 = ax_nat(g, cur, jj, kk);
#pragma unroll
                        for (int q = 0; q < LA; ++q)
                            v[dd][q] = cur + q < lim ? ld_relaxed(a.x + r0 + q * dstep) : sent;
                    }
                    int adv = 0;
#pragma unroll
                    for (int q = 0; q < LA; ++q) {
                        bool all = cur + q < lim;
#pragma unroll
                        for (int dd = 0; dd < R; ++dd) all = all && !is_sentinel(v[dd][q]);
                        if (all && adv == q) {
#pragma unroll
                            for (int dd = 0; dd < R; ++dd) ax_sts(base + dd * dstr + (cur + q) % AX_W, v[dd][q]);
                            adv = q + 1;
                        }
                    }
                    if (adv) {
                        cur += adv;
                        prog = true;
                        __threadfence_block();   // values before the counter
                        *reinterpret_cast<volatile int*>(rdy) = cur;
                    }
                }
                if (!__any_sync(0xffffffffu, todo)) break;
                if (!__any_sync(0xffffffffu, prog)) {
                    __nanosleep(20);
                    if (++spins > SPIN_LIMIT) { if (lane == 0) atomicExch(a.err, 7); break; }
                } else {
                    spins = 0;
                }
            }
        } else {
            // ---- compute lanes: four lanes per pencil (j, k), skewed by jl + kl.
            // Lane h folds the neighbours along x (h=0, plus the right-hand side),
            // y (h=1) or z (h=2); h=3 runs the same code on zero coefficients, so
            // every warp executes one uniform instruction stream.  All neighbour
            // values come from the shared ring (this block's pencils, the lane's
            // own pencil for x) or the halo rings (upstream blocks).  Software
            // pipelined over the barrier-separated steps: in step s a lane adds its
            // d = 1 (critical) term to the d >= 2 sum it prepared in step s-1, two
            // shuffles combine the four sums, and the d >= 2 sum of step s+1 is
            // prepared before the barrier.
            const int pc = tid >> 2, h = tid & 3;
            const int jl = pc % AX_BJ, kl = pc / AX_BJ;
            const int j = J * AX_BJ + jl, k = K * AX_BK + kl;
            const bool pen = j < g.ny && k < g.nz;
            const int row0 = pen ? ax_nat(g, 0, j, k) : 0;
            auto prefetch_b = [&](int s) {
                const int i = s - jl - kl;
                if (h == 0 && pen && s < g.nsteps && i >= 0 && i < g.nx)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(ax_saddr(br + (s % AX_PB) * AX_T + pc)),
                                 "l"(a.b + row0 + i * dstep) : "memory");
                asm volatile("cp.async.commit_group;" ::: "memory");
            };
            for (int s = 0; s < AX_PB; ++s) prefetch_b(s);
            // neighbour d along this lane's dimension: ring lane (or halo pencil offset)
            const int ml = h == 1 ? jl : h == 2 ? kl : 1 << 20;   // x / dummy: always in the ring
            const int dl = h == 1 ? 1 : h == 2 ? AX_BJ : 0;       // ring lane step per d
            bool in[R];
            int off[R];
#pragma unroll
            for (int d = 1; d <= R; ++d) {
                in[d - 1] = ml >= d;
                off[d - 1] = ml >= d ? pc - d * dl
                                     : (h == 1 ? ((d - jl - 1) * AX_BK + kl) : ((d - kl - 1) * AX_BJ + jl)) * AX_W;
            }
            const double* halo = h == 1 ? hy : hz;
            const volatile int* rdy = h == 1 ? &rdy_y[kl] : &rdy_z[jl];
            const bool need_halo = (h == 1 || h == 2) && ml < R;
            // coefficient rows of this lane (h=3: a zero block) and its stride
            const double* zrow = zc + pc;
            auto coef_base = [&](int s) -> const double* {
                return h == 3 ? zrow : cf + (int)((gs0 + s) % AX_P) * NC * AX_T + h * R * AX_T + pc;
            };
            auto wait_stage = [&](long long gs) {
                const unsigned par = (unsigned)((gs / AX_P) & 1);
                unsigned ok = 0;
                while (!ok)
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                                 : "=r"(ok) : "r"(ax_saddr(&mbar[(int)(gs % AX_P)])), "r"(par) : "memory");
            };
            auto wait_halo = [&](int i) {   // upstream values below i+1 present
                if (need_halo && *rdy <= i) {
                    long long spins = 0;
                    while (*rdy <= i) {
                        __nanosleep(16);
                        if (++spins > SPIN_LIMIT) { atomicExch(a.err, 7); break; }
                    }
                }
            };
            auto nb = [&](int s, int d, int iw) -> double {   // neighbour d of step s
                return in[d - 1] ? xr[((s - d) & (RR - 1)) * AX_T + off[d - 1]] : ax_lds(halo + off[d - 1] + iw);
            };
            // d >= 2 part of step s (+ -alpha b on the x lane)
            auto old_part = [&](int s) -> double {
                const int i = s - jl - kl;
                if (!pen || i < 0 || i >= g.nx) return 0.0;
                wait_halo(i);
                const double* c = coef_base(s);
                const int iw = i % AX_W;
                double p0 = 0.0, p1 = 0.0;
#pragma unroll
                for (int d = 2; d <= R; ++d) {
                    if (d & 1) p1 = fma(c[(d - 1) * AX_T], nb(s, d, iw), p1);
                    else p0 = fma(c[(d - 1) * AX_T], nb(s, d, iw), p0);
                }
                asm volatile("cp.async.wait_group %0;" ::"n"(AX_PB - 1) : "memory");   // rhs of step s present
                const double bb = h == 0 ? br[(s % AX_PB) * AX_T + pc] : 0.0;
                return fma(-a.alpha, bb, p0 + p1);
            };
            // prologue: stages 0 and 1 present (one waiter, then the barrier), old part of step 0
            if (tid == 0) {
                wait_stage(gs0);
                if (g.nsteps > 1) wait_stage(gs0 + 1);
            }
            ax_bar();
            double old = old_part(0);
            for (int s = 0; s < g.nsteps; ++s) {
                long long k0 = 0, k1 = 0, k2 = 0, k3 = 0, k4 = 0;
                const bool probe = a.dbg && blk == 0 && (tid == 0 || tid == 64 || tid == 193);
                if (probe) k0 = clock64();
                const int i = s - jl - kl;
                const bool act = pen && i >= 0 && i < g.nx;
                double part = old;
                if (act) {   // critical term: the d = 1 neighbour (step s-1)
                    if (!in[0]) wait_halo(i);
                    part = fma(coef_base(s)[0], nb(s, 1, i % AX_W), part);
                }
                if (probe) k1 = clock64();
                double tot = part + __shfl_xor_sync(0xffffffffu, part, 1);
                tot = tot + __shfl_xor_sync(0xffffffffu, tot, 2);   // sum(all deps) - alpha b
                if (act) {
                    const double x = -tot * cf[(int)((gs0 + s) % AX_P) * NC * AX_T + 3 * R * AX_T + pc];
                    if (h == 0) {
                        xr[(s & (RR - 1)) * AX_T + pc] = x;
                        const int row = row0 + i * dstep;
                        __stcg(a.x + row, publishable(x));
                        if (a.out2) a.out2[row] = x + a.add[row];
                    }
                }
                if (probe) k2 = clock64();
                // prepare step s+1 (its old part), then the step barrier; the ring
                // row of step s is read by step s+1's old part only from d >= 2,
                // i.e. rows <= s-1 (written before barrier s-1)
                prefetch_b(s + AX_PB);
                if (s + 1 < g.nsteps) old = old_part(s + 1);   // stage s+1 present since barrier s-1
                if (probe) k3 = clock64();
                // one thread waits for stage s+2; the barrier publishes it to the CTA
                if (tid == 0 && s + 2 < g.nsteps) wait_stage(gs0 + s + 2);
                if (probe) {
                    k4 = clock64();
                    const int ps = tid == 0 ? 0 : tid == 64 ? 1 : 2;
                    long long* q = a.dbg + (int64_t)g.NJ * g.NK * g.nsteps + ((int64_t)s * 3 + ps) * 5;
                    q[0] = k0; q[1] = k1; q[2] = k2; q[3] = k3; q[4] = k4;
                }
                ax_bar();
                if (tid == 0) {
                    s_prog = s;
                    if (a.dbg) a.dbg[(int64_t)blk * g.nsteps + s] = clock64();
                }
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
            if (tid == 0) s_prog = 1 << 30;
        }
        gs0 += g.nsteps;
        __syncthreads();
    }
}

size_t ax_smem(int R) {
    const int NC = 3 * R + 1;
    const int RR = R + 1 <= 8 ? 8 : 16;
    return sizeof(double) * ((size_t)AX_P * NC * AX_T + (size_t)RR * AX_T + (size_t)R * (AX_BK + AX_BJ) * AX_W +
                             (size_t)AX_PB * AX_T + (size_t)R * AX_T);
}

template <int R>
void ax_launch(Ctx* c, AxialPlan& p, AxSolve& a) {
    static std::once_flag once;
    static int grid = 0;
    const size_t smem = ax_smem(R);
    std::call_once(once, [&] {
        EDFA_CUDA(cudaFuncSetAttribute(k_ax_solve<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int occ = 0;
        EDFA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_ax_solve<R>, AX_THREADS, smem));
        grid = NUM_SMS_B200 * std::max(1, occ);
    });
    const int nb = p.NJ * p.NK;
    const int g = std::min(grid, nb);
    a.ticket_base = p.ticket_base;
    p.ticket_base += nb + g;   // every CTA takes exactly one failing ticket
    void* args[] = {&a};
    // cooperative: all CTAs co-resident, so a block never waits on an unscheduled one
    EDFA_CUDA(cudaLaunchCooperativeKernel((void*)k_ax_solve<R>, dim3(g), dim3(AX_THREADS), args, smem, c->stream));
}

}  // namespace

bool build_axial_plan(Ctx* c, const Csr& D, const double* diag, bool unit, bool reverse, const int* dims,
                      AxialPlan& p) {
    // opt-in (EDFA_AXIAL=1): correct, but at ~0.5-1 us per pencil step it does
    // not yet beat the dataflow tile solve (tile.cu) on config 2
    if (!getenv("EDFA_AXIAL")) return false;
    const int n = D.n_rows;
    if (!dims || n == 0 || (int64_t)dims[0] * dims[1] * dims[2] != n) return false;
    AxGeo g{dims[0], dims[1], dims[2], 0, 0, 0, 0, 0, reverse ? 1 : 0};
    int* fl = c->d_scalar_i + 32;   // [bad, maxr]
    EDFA_CUDA(cudaMemsetAsync(fl, 0, 2 * sizeof(int), c->stream));
    {
        Prof pr(c, "axial_plan", 12.0 * D.nnz);
        k_ax_check<<<ceil_div(n, 256), 256, 0, c->stream>>>(view(D), g, fl, fl + 1);
        check_launch("k_ax_check");
    }
    int h[2];
    EDFA_CUDA(cudaMemcpyAsync(h, fl, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
    if (h[0] || h[1] < 1) return false;
    g.R = h[1];
    g.NC = 3 * g.R + 1;
    g.NJ = ceil_div(g.ny, AX_BJ);
    g.NK = ceil_div(g.nz, AX_BK);
    g.nsteps = g.nx + (AX_BJ - 1) + (AX_BK - 1);
    if (ax_smem(g.R) > 220 * 1024) return false;
    p.n = n;
    p.R = g.R;
    p.NJ = g.NJ;
    p.NK = g.NK;
    p.nsteps = g.nsteps;
    p.reverse = reverse;
    p.dims[0] = g.nx; p.dims[1] = g.ny; p.dims[2] = g.nz;
    p.n_dep = D.nnz;
    const int64_t total = (int64_t)g.NJ * g.NK * g.nsteps * AX_T;
    p.coef.reset(c, (size_t)total * g.NC);
    {
        Prof pr(c, "axial_plan", 12.0 * D.nnz + 8.0 * total * g.NC);
        k_ax_fill<<<(unsigned)ceil_div(total, (int64_t)256), 256, 0, c->stream>>>(view(D), g, diag, unit ? 1 : 0,
                                                                                  p.coef.p);
        check_launch("k_ax_fill");
    }
    // blocks by anti-diagonal (J + K), then K, J: a block's upstream blocks come first
    std::vector<int> ord(g.NJ * g.NK);
    for (int b = 0; b < (int)ord.size(); ++b) ord[b] = b;
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) {
        return (x % g.NJ + x / g.NJ) < (y % g.NJ + y / g.NJ);
    });
    p.order.reset(c, ord.size());
    EDFA_CUDA(cudaMemcpyAsync(p.order.p, ord.data(), sizeof(int) * ord.size(), cudaMemcpyHostToDevice, c->stream));
    p.ticket.reset(c, 1);
    EDFA_CUDA(cudaMemsetAsync(p.ticket.p, 0, sizeof(int), c->stream));
    p.ticket_base = 0;
    EDFA_CUDA(cudaStreamSynchronize(c->stream));   // ord is a host temporary
    return true;
}

void run_axial(Ctx* c, AxialPlan& p, const double* b, double alpha, double* x, const double* add, double* out2,
               const char* name) {
    if (p.n == 0) return;
    fill_bits(c, x, p.n, SENTINEL_BITS);   // a cell's value is its own ready flag
    AxGeo g{p.dims[0], p.dims[1], p.dims[2], p.NJ, p.NK, p.nsteps, p.R, 3 * p.R + 1, p.reverse ? 1 : 0};
    AxSolve a{g, p.coef.p, p.order.p, p.ticket.p, 0, b, alpha, x, add, out2, c->d_scalar_i + 8, nullptr};
    static const char* dbg_path = getenv("EDFA_AX_DEBUG");
    DevBuf<long long> dbg;
    const int64_t ndbg = (int64_t)p.NJ * p.NK * p.nsteps + (int64_t)p.nsteps * 15;
    if (dbg_path) {
        dbg.reset(c, ndbg);
        a.dbg = dbg.p;
    }
    Prof pr(c, name, 12.0 * p.n_dep + 24.0 * p.n + (out2 ? 16.0 * p.n : 0.0));
    switch (p.R) {
        case 1: ax_launch<1>(c, p, a); break;
        case 2: ax_launch<2>(c, p, a); break;
        case 3: ax_launch<3>(c, p, a); break;
        case 4: ax_launch<4>(c, p, a); break;
        case 5: ax_launch<5>(c, p, a); break;
        case 6: ax_launch<6>(c, p, a); break;
        case 7: ax_launch<7>(c, p, a); break;
        default: ax_launch<8>(c, p, a); break;
    }
    check_launch("k_ax_solve");
    if (dbg_path) {
        std::vector<long long> h(ndbg);
        EDFA_CUDA(cudaMemcpyAsync(h.data(), dbg.p, ndbg * 8, cudaMemcpyDeviceToHost, c->stream));
        EDFA_CUDA(cudaStreamSynchronize(c->stream));
        FILE* f = fopen(dbg_path, "w");
        if (f) {
            fprintf(f, "%d %d %d\n", p.NJ, p.NK, p.nsteps);
            for (int64_t q = 0; q < (int64_t)p.NJ * p.NK * p.nsteps; ++q) fprintf(f, "%lld\n", h[q]);
            FILE* f2 = fopen((std::string(dbg_path) + ".probe").c_str(), "w");
            if (f2) {
                for (int s = 0; s < p.nsteps; ++s)
                    for (int ps = 0; ps < 3; ++ps) {
                        const long long* q = &h[(int64_t)p.NJ * p.NK * p.nsteps + ((int64_t)s * 3 + ps) * 5];
                        fprintf(f2, "%d %d %lld %lld %lld %lld %lld\n", s, ps, q[0], q[1], q[2], q[3], q[4]);
                    }
                fclose(f2);
            }
            fclose(f);
        }
    }
}

}  // namespace edfa
