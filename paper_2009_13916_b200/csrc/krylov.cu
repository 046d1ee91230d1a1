// K9-K11: EDFA application, right-preconditioned GMRES(m) and Bi-CGStab.
//
// apply  (hx/precond.py:311-320)
//   t_f = -(L L^T)^-1 r_f            two level-ordered solves, sign folded in
//   u_c = r_c - A_cf t_f             SpMV with beta = 1
//   t_c = (L U)^-1 u_c               two level-ordered solves
//   y_f = t_f + (L L^T)^-1 A_fc t_c  SpMV + two solves, "+ t_f" fused into the
//                                    last solve's epilogue
// GMRES: Arnoldi with classical Gram-Schmidt and DGKS selective
// re-orthogonalisation (second pass only when ||w|| drops below ||w0||/sqrt2):
// one fused multi-dot pass over V_0..V_j and one fused multi-axpy(+norm) pass
// per iteration; block partial sums reduced in a fixed order (deterministic).
// Givens rotations and the small triangular solve run on the host.
#include <cmath>
#include <cstdlib>
#include <vector>

#include "dev_util.cuh"
#include "edfa_internal.cuh"
#include "objects.cuh"

namespace edfa {
namespace {

constexpr int RED_BLOCKS = 3 * NUM_SMS_B200;   // fixed grid -> fixed reduction order
constexpr int RED_THREADS = 256;
constexpr int GROUP = 8;                      // vectors per multi-dot block row

// The last block of a reduction kernel to finish (atomic ticket) sums the
// per-block partials in a fixed order -- the same order as a separate
// k_reduce_partials launch, so results are identical and deterministic.
__device__ void last_block_reduce(const double* partial, int nblk, int nvec, double* out, unsigned* counter) {
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x * gridDim.y - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int k = wid; k < nvec; k += nw) {
        double s = 0.0;
        for (int b = lane; b < nblk; b += 32) s += __ldcg(partial + (int64_t)b * 64 + k);
        s = warp_sum(s);
        if (lane == 0) out[k] = s;
    }
    if (threadIdx.x == 0) *counter = 0u;
}

// partial[blk][k] = sum over the block's rows of V[k0+k] . w   (k < GROUP).
// VEC2: pairs of rows per thread with 16-byte loads (V rows and w 16-byte
// aligned, ldv even); the odd tail row is taken by the scalar path.
template <bool VEC2>
__global__ void __launch_bounds__(RED_THREADS) k_multidot(const double* __restrict__ V, int64_t ldv, int nvec,
                                                          const double* __restrict__ w, int64_t n,
                                                          double* __restrict__ partial, double* __restrict__ out,
                                                          unsigned* counter) {
    int k0 = blockIdx.y * GROUP;
    double acc[GROUP];
#pragma unroll
    for (int k = 0; k < GROUP; ++k) acc[k] = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (VEC2) {
        const int64_t n2 = n >> 1;
        const double2* w2 = reinterpret_cast<const double2*>(w);
        for (int64_t i = t0; i < n2; i += stride) {
            double2 wi = w2[i];
            double2 v[GROUP];
#pragma unroll
            for (int k = 0; k < GROUP; ++k)
                if (k0 + k < nvec) v[k] = reinterpret_cast<const double2*>(V + (int64_t)(k0 + k) * ldv)[i];
#pragma unroll
            for (int k = 0; k < GROUP; ++k)
                if (k0 + k < nvec) acc[k] = fma(v[k].y, wi.y, fma(v[k].x, wi.x, acc[k]));
        }
        if ((n & 1) && t0 == 0) {
            double wi = w[n - 1];
#pragma unroll
            for (int k = 0; k < GROUP; ++k)
                if (k0 + k < nvec) acc[k] = fma(V[(int64_t)(k0 + k) * ldv + n - 1], wi, acc[k]);
        }
    } else {
        for (int64_t i = t0; i < n; i += stride) {
            double wi = w[i];
#pragma unroll
            for (int k = 0; k < GROUP; ++k)
                if (k0 + k < nvec) acc[k] = fma(V[(int64_t)(k0 + k) * ldv + i], wi, acc[k]);
        }
    }
    __shared__ double red[GROUP][RED_THREADS / 32];
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < GROUP; ++k) {
        double v = warp_sum(acc[k]);
        if (lane == 0) red[k][wid] = v;
    }
    __syncthreads();
    if (threadIdx.x < GROUP && k0 + threadIdx.x < nvec) {
        double s = 0.0;
        for (int t = 0; t < RED_THREADS / 32; ++t) s += red[threadIdx.x][t];
        partial[(int64_t)blockIdx.x * 64 + k0 + threadIdx.x] = s;
    }
    last_block_reduce(partial, gridDim.x, nvec, out, counter);
}

// out[k] = sum_blk partial[blk][k]   (fixed order)
__global__ void k_reduce_partials(const double* __restrict__ partial, int nblk, int nvec, double* __restrict__ out) {
    int k = blockIdx.x;
    if (k >= nvec) return;
    double s = 0.0;
    for (int b = threadIdx.x; b < nblk; b += 32) s += partial[(int64_t)b * 64 + k];
    s = warp_sum(s);
    if (threadIdx.x == 0) out[k] = s;
}

// w <- w - sum_{k<nv} h[k] V[k]   (or out = sum h[k] V[k] when w_in == NULL),
// partial[blk] = block sum of out^2.  VEC2 as in k_multidot.
template <bool VEC2>
__global__ void __launch_bounds__(RED_THREADS, 3) k_multiaxpy(const double* __restrict__ V, int64_t ldv, int nv,
                                                           const double* __restrict__ h, double hscale,
                                                           const double* w_in, double* out,
                                                           int64_t n, double* __restrict__ partial,
                                                           double* __restrict__ norm2, unsigned* counter) {
    __shared__ double hs[64];
    if (threadIdx.x < nv) hs[threadIdx.x] = h[threadIdx.x] * hscale;
    __syncthreads();
    double ss = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (VEC2) {
        const int64_t n2 = n >> 1;
        for (int64_t i = t0; i < n2; i += stride) {
            double ax = 0.0, ay = 0.0;
            int k = 0;
            for (; k + 8 <= nv; k += 8) {
                double2 a[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) a[u] = reinterpret_cast<const double2*>(V + (int64_t)(k + u) * ldv)[i];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    ax = fma(hs[k + u], a[u].x, ax);
                    ay = fma(hs[k + u], a[u].y, ay);
                }
            }
            for (; k < nv; ++k) {
                double2 a = reinterpret_cast<const double2*>(V + (int64_t)k * ldv)[i];
                ax = fma(hs[k], a.x, ax);
                ay = fma(hs[k], a.y, ay);
            }
            double2 o;
            if (w_in) {
                double2 wv = reinterpret_cast<const double2*>(w_in)[i];
                o.x = wv.x - ax;
                o.y = wv.y - ay;
            } else {
                o.x = ax;
                o.y = ay;
            }
            reinterpret_cast<double2*>(out)[i] = o;
            ss = fma(o.x, o.x, ss);
            ss = fma(o.y, o.y, ss);
        }
        if ((n & 1) && t0 == 0) {
            const int64_t i = n - 1;
            double acc = 0.0;
            for (int k = 0; k < nv; ++k) acc = fma(hs[k], V[(int64_t)k * ldv + i], acc);
            double o = w_in ? w_in[i] - acc : acc;
            out[i] = o;
            ss = fma(o, o, ss);
        }
    } else {
        for (int64_t i = t0; i < n; i += stride) {
            double acc = 0.0;
            int k = 0;
            for (; k + 4 <= nv; k += 4) {
                double a0 = V[(int64_t)k * ldv + i], a1 = V[(int64_t)(k + 1) * ldv + i];
                double a2 = V[(int64_t)(k + 2) * ldv + i], a3 = V[(int64_t)(k + 3) * ldv + i];
                acc = fma(hs[k], a0, acc);
                acc = fma(hs[k + 1], a1, acc);
                acc = fma(hs[k + 2], a2, acc);
                acc = fma(hs[k + 3], a3, acc);
            }
            for (; k < nv; ++k) acc = fma(hs[k], V[(int64_t)k * ldv + i], acc);
            double o = w_in ? w_in[i] - acc : acc;
            out[i] = o;
            ss = fma(o, o, ss);
        }
    }
    __shared__ double red[RED_THREADS / 32];
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int t = 0; t < RED_THREADS / 32; ++t) s += red[t];
        if (partial) partial[(int64_t)blockIdx.x * 64] = s;
    }
    if (partial) last_block_reduce(partial, gridDim.x, 1, norm2, counter);
}

// ---------------------------------------------------------------- DCGS2 Arnoldi step
// One reduction per Arnoldi step (delayed classical Gram-Schmidt with
// re-orthogonalisation; the re-orthogonalisation of u_j is folded into the
// projection of the next Krylov vector).  Step j holds final q_0..q_{j-1}
// (slots 0..j-1), u_j = A P q_{j-1} - Q_j h1 after ONE projection pass (slot
// j, unnormalised) and w = A P u_j (slot j+1).
//   dots:  [Q_j u]^T u = (a, alpha), [Q_j u]^T w = (b, beta)      (one pass)
//   nu = sqrt(alpha - a.a),  q_j = (u - Q_j a) / nu
//   H[:j, j-1] = h1 + a,  H[j, j-1] = nu                 (column j-1 final)
//   A P q_j = (w - Q_{j+1} t) / nu with t = H[:j+1, :j] a  (Arnoldi relation)
//   c = Q_{j+1}^T A P q_j,  u_{j+1} = A P q_j - Q_{j+1} c    (one pass)
// so each step reads the basis twice (dots, update) instead of CGS2's four
// times; in exact arithmetic the columns equal CGS2's.
#ifndef EDFA_D2_GROUP
#define EDFA_D2_GROUP 8
#endif
constexpr int D2_GROUP = EDFA_D2_GROUP;
#ifndef EDFA_DOTS2_WAVE
#define EDFA_DOTS2_WAVE 2
#endif

// DCGS2 step coefficients from the reduced dots (executed by one 256-thread block):
// dot[0..j] = [Q_j u]^T u, dot[64..64+j] = [Q_j u]^T w.  Writes Hessenberg column
// j-1 (H, hcol), the first-pass coefficients h1 of the next step and the update
// weights coef: [0..63] q_j, [64..127] u_{j+1}, [128..130] = (1/nu, 1/nu, -d_j/nu).
__device__ void dcgs2_coeffs_block(const double* dot, int j, int m, double* __restrict__ H, double* __restrict__ h1,
                                   double* __restrict__ coef, double* __restrict__ hcol) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int ld = m + 1, tid = threadIdx.x;
    __shared__ double sa[64], st[64], sd[64], s_aa, s_ab, s_nu;
    if (j == 0) {   // u_0 = q_0 is final: first projection only
        if (tid == 0) {
            const double c0 = dot[64];
            h1[0] = c0;
            coef[128] = 1.0;
            coef[129] = 1.0;
            coef[130] = -c0;
        }
        return;
    }
    if (tid < j) sa[tid] = dot[tid];
    __syncthreads();
    if (wid == 0) {
        double aa = 0.0, ab = 0.0;
        for (int i = lane; i < j; i += 32) {
            aa = fma(sa[i], sa[i], aa);
            ab = fma(sa[i], dot[64 + i], ab);
        }
        aa = warp_sum(aa);
        ab = warp_sum(ab);
        if (lane == 0) {
            s_aa = aa;
            s_ab = ab;
            const double nu2 = dot[j] - aa;
            s_nu = nu2 > 0.0 ? sqrt(nu2) : 0.0;
        }
    }
    __syncthreads();
    const double nu = s_nu;
    double* col = H + (int64_t)(j - 1) * ld;
    if (tid < j) {
        const double v = h1[tid] + sa[tid];
        col[tid] = v;
        hcol[tid] = v;
    }
    if (tid == j) { col[j] = nu; hcol[j] = nu; }
    __syncthreads();
    if (nu == 0.0) {   // happy breakdown: column j-1 ends the cycle
        if (tid < 64) { coef[tid] = 0.0; coef[64 + tid] = 0.0; }
        if (tid == 0) { coef[128] = 0.0; coef[129] = 0.0; coef[130] = 0.0; }
        return;
    }
    const double inv = 1.0 / nu;
    {   // t = H[:j+1, :j] a  (H[r, i] = 0 for r > i + 1): thread (r, quarter) loads
        // its <= 16 entries at once, quarters summed in order
        __shared__ double tq[4][64];
        const int r = tid & 63, qt = tid >> 6;
        double hv[16];
        int ii[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int i = qt + 4 * u;
            ii[u] = i;
            hv[u] = (r <= j && i < j && i >= r - 1) ? H[(int64_t)i * ld + r] : 0.0;
        }
        double t = 0.0;
#pragma unroll
        for (int u = 0; u < 16; ++u)
            if (ii[u] < j) t = fma(hv[u], sa[ii[u]], t);
        tq[qt][r] = t;
        __syncthreads();
        if (tid <= j) st[tid] = ((tq[0][tid] + tq[1][tid]) + tq[2][tid]) + tq[3][tid];
    }
    __syncthreads();
    if (tid <= j) {
        const double c = tid < j ? (dot[64 + tid] - st[tid]) * inv
                                 : ((dot[64 + j] - s_ab) * inv - st[j]) * inv;
        sd[tid] = st[tid] * inv + c;
        h1[tid] = c;
    }
    __syncthreads();
    if (tid < j) {
        coef[tid] = sa[tid] * inv;
        coef[64 + tid] = sd[tid] - sd[j] * sa[tid] * inv;
    }
    if (tid == 0) {
        coef[128] = inv;
        coef[129] = inv;
        coef[130] = -sd[j] * inv;
    }
}

// standalone coefficient kernel (slab path: dots reduced across slabs in between)
__global__ void __launch_bounds__(RED_THREADS) k_dcgs2_coeffs(const double* __restrict__ dots, int j, int m,
                                                              double* __restrict__ H, double* __restrict__ h1,
                                                              double* __restrict__ coef, double* __restrict__ hcol) {
    __shared__ double dot[128];
    if (threadIdx.x < 128) dot[threadIdx.x] = dots[threadIdx.x];
    __syncthreads();
    dcgs2_coeffs_block(dot, j, m, H, h1, coef, hcol);
}

// dots of V_0..V_{nv-1} with u = V_{nv-1} and w = V_{nv}: grid (groups, ranges),
// block-contiguous element ranges so the blocks sharing a range run together
// and u, w come from L2 after the first group.  partial[r][0..63] = u-dots,
// [64..127] = w-dots.
// 2 resident blocks per SM (<= 128 registers): the one-wave grid below assumes it
// (157 registers at minBlocks 1 left half the grid in a second wave: 5.8 -> 4.6 ms/step)
#ifndef DOTS2_MINB
#define DOTS2_MINB EDFA_DOTS2_WAVE
#endif
template <bool VEC2>
__global__ void __launch_bounds__(RED_THREADS, DOTS2_MINB) k_dots2(const double* __restrict__ V, int64_t ldv, int nv, int64_t n,
                                                       int64_t range, double* __restrict__ partial, int pr,
                                                       unsigned* counter, int j, int m, double* __restrict__ H,
                                                       double* __restrict__ h1, double* __restrict__ coef,
                                                       double* __restrict__ hcol) {
    const int k0 = blockIdx.x * D2_GROUP;
    const double* u = V + (int64_t)(nv - 1) * ldv;
    const double* w = V + (int64_t)nv * ldv;
    double au[D2_GROUP], aw[D2_GROUP];
#pragma unroll
    for (int k = 0; k < D2_GROUP; ++k) au[k] = aw[k] = 0.0;
    const int64_t lo = blockIdx.y * range, hi = min(n, lo + range);
    if (VEC2) {   // range is even, rows 16-byte aligned
        const int64_t lo2 = lo >> 1, hi2 = hi >> 1;
        for (int64_t i = lo2 + threadIdx.x; i < hi2; i += RED_THREADS) {
            const double2 ui = reinterpret_cast<const double2*>(u)[i];
            const double2 wi = reinterpret_cast<const double2*>(w)[i];
            double2 v[D2_GROUP];
#pragma unroll
            for (int k = 0; k < D2_GROUP; ++k)
                if (k0 + k < nv) v[k] = reinterpret_cast<const double2*>(V + (int64_t)(k0 + k) * ldv)[i];
#pragma unroll
            for (int k = 0; k < D2_GROUP; ++k)
                if (k0 + k < nv) {
                    au[k] = fma(v[k].y, ui.y, fma(v[k].x, ui.x, au[k]));
                    aw[k] = fma(v[k].y, wi.y, fma(v[k].x, wi.x, aw[k]));
                }
        }
        if ((hi & 1) && hi == n && threadIdx.x == 0) {
            const int64_t i = n - 1;
#pragma unroll
            for (int k = 0; k < D2_GROUP; ++k)
                if (k0 + k < nv) {
                    const double vk = V[(int64_t)(k0 + k) * ldv + i];
                    au[k] = fma(vk, u[i], au[k]);
                    aw[k] = fma(vk, w[i], aw[k]);
                }
        }
    } else {
        for (int64_t i = lo + threadIdx.x; i < hi; i += RED_THREADS) {
            const double ui = u[i], wi = w[i];
#pragma unroll
            for (int k = 0; k < D2_GROUP; ++k)
                if (k0 + k < nv) {
                    const double vk = V[(int64_t)(k0 + k) * ldv + i];
                    au[k] = fma(vk, ui, au[k]);
                    aw[k] = fma(vk, wi, aw[k]);
                }
        }
    }
    __shared__ double red[2 * D2_GROUP][RED_THREADS / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < D2_GROUP; ++k) {
        const double x = warp_sum(au[k]), y = warp_sum(aw[k]);
        if (lane == 0) { red[k][wid] = x; red[D2_GROUP + k][wid] = y; }
    }
    __syncthreads();
    if (threadIdx.x < 2 * D2_GROUP) {
        const int k = threadIdx.x % D2_GROUP, side = threadIdx.x / D2_GROUP;
        if (k0 + k < nv) {
            double t = 0.0;
            for (int q = 0; q < RED_THREADS / 32; ++q) t += red[threadIdx.x][q];
            partial[(int64_t)(side * 64 + k0 + k) * pr + blockIdx.y] = t;   // slot-major
        }
    }
    // last block: fixed-order sum over ranges, then the step's coefficients
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x * gridDim.y - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    // warp w sums the needed slots w, w+8, ... over the ranges (slot-major
    // partials: lanes read consecutive ranges), fixed order: deterministic
    __shared__ double dot[128];
    {
        const int nr = gridDim.y, nw = RED_THREADS / 32;
        for (int q = wid; q < 2 * nv; q += nw) {
            const int slot = q < nv ? q : 64 + (q - nv);
            const double* col = partial + (int64_t)slot * pr;
            double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
            int b = lane;
            for (; b + 96 < nr; b += 128) {
                acc0 += __ldcg(col + b);
                acc1 += __ldcg(col + b + 32);
                acc2 += __ldcg(col + b + 64);
                acc3 += __ldcg(col + b + 96);
            }
            for (; b < nr; b += 32) acc0 += __ldcg(col + b);
            const double t = warp_sum((acc0 + acc1) + (acc2 + acc3));
            if (lane == 0) dot[slot] = t;
        }
    }
    if (threadIdx.x == 0) *counter = 0u;
    __syncthreads();
    if (!coef) {   // dots only (slab-distributed solves reduce them across slabs first)
        const int t = threadIdx.x;
        if (t < 128) hcol[t] = (t < nv || (t >= 64 && t < 64 + nv)) ? dot[t] : 0.0;
        return;
    }
    dcgs2_coeffs_block(dot, j, m, H, h1, coef, hcol);
}

// slot j  <- q_j     = coef[128] u - sum_k coef[k] V_k          (j >= 1)
// slot j+1 <- u_{j+1} = coef[129] w + coef[130] u - sum_k coef[64+k] V_k
template <bool VEC2>
__global__ void __launch_bounds__(RED_THREADS, 3) k_axpy2(double* __restrict__ V, int64_t ldv, int j, int64_t n,
                                                          const double* __restrict__ coef) {
    __shared__ double cq[64], cw[64], sc[3];
    if (threadIdx.x < j) {
        cq[threadIdx.x] = coef[threadIdx.x];
        cw[threadIdx.x] = coef[64 + threadIdx.x];
    }
    if (threadIdx.x < 3) sc[threadIdx.x] = coef[128 + threadIdx.x];
    __syncthreads();
    double* u = V + (int64_t)j * ldv;
    double* w = u + ldv;
    const double su = sc[0], sw = sc[1], suw = sc[2];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (VEC2) {
        const int64_t n2 = n >> 1;
        for (int64_t i = t0; i < n2; i += stride) {
            double qx = 0.0, qy = 0.0, ex = 0.0, ey = 0.0;
            int k = 0;
            for (; k + 8 <= j; k += 8) {
                double2 a[8];
#pragma unroll
                for (int t = 0; t < 8; ++t) a[t] = reinterpret_cast<const double2*>(V + (int64_t)(k + t) * ldv)[i];
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    qx = fma(cq[k + t], a[t].x, qx);
                    qy = fma(cq[k + t], a[t].y, qy);
                    ex = fma(cw[k + t], a[t].x, ex);
                    ey = fma(cw[k + t], a[t].y, ey);
                }
            }
            for (; k < j; ++k) {
                const double2 a = reinterpret_cast<const double2*>(V + (int64_t)k * ldv)[i];
                qx = fma(cq[k], a.x, qx);
                qy = fma(cq[k], a.y, qy);
                ex = fma(cw[k], a.x, ex);
                ey = fma(cw[k], a.y, ey);
            }
            const double2 uv = reinterpret_cast<const double2*>(u)[i];
            const double2 wv = reinterpret_cast<const double2*>(w)[i];
            if (j > 0) reinterpret_cast<double2*>(u)[i] = make_double2(su * uv.x - qx, su * uv.y - qy);
            reinterpret_cast<double2*>(w)[i] =
                make_double2(fma(sw, wv.x, suw * uv.x) - ex, fma(sw, wv.y, suw * uv.y) - ey);
        }
        if ((n & 1) && t0 == 0) {
            const int64_t i = n - 1;
            double q = 0.0, e = 0.0;
            for (int k = 0; k < j; ++k) {
                const double a = V[(int64_t)k * ldv + i];
                q = fma(cq[k], a, q);
                e = fma(cw[k], a, e);
            }
            const double uv = u[i], wv = w[i];
            if (j > 0) u[i] = su * uv - q;
            w[i] = fma(sw, wv, suw * uv) - e;
        }
    } else {
        for (int64_t i = t0; i < n; i += stride) {
            double q = 0.0, e = 0.0;
            for (int k = 0; k < j; ++k) {
                const double a = V[(int64_t)k * ldv + i];
                q = fma(cq[k], a, q);
                e = fma(cw[k], a, e);
            }
            const double uv = u[i], wv = w[i];
            if (j > 0) u[i] = su * uv - q;
            w[i] = fma(sw, wv, suw * uv) - e;
        }
    }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

__global__ void k_axpby(int64_t n, double a, const double* x, double b, double* y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = (b == 0.0) ? a * x[i] : fma(a, x[i], b * y[i]);
}
// w <- w / sqrt(nrm2[0])  (0 when the norm is 0: happy breakdown)
__global__ void k_normalize(int64_t n, const double* __restrict__ nrm2, double* w) {
    const double s2 = *nrm2;
    const double inv = s2 > 0.0 ? 1.0 / sqrt(s2) : 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        w[i] = w[i] * inv;
}
// z = x + a*(y - w*v)   (Bi-CGStab direction update, p = r + beta (p - omega v))
__global__ void k_bicg_p(int64_t n, const double* __restrict__ r, double beta, double omega,
                         const double* __restrict__ v, double* __restrict__ p) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = r[i] + beta * (p[i] - omega * v[i]);
}
__global__ void k_lincomb3(int64_t n, double a, const double* __restrict__ x, double b, const double* __restrict__ y,
                           double* __restrict__ z) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        z[i] = z[i] + a * x[i] + b * y[i];
}

int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(RED_BLOCKS, (n + RED_THREADS - 1) / RED_THREADS)); }

}  // namespace

// ---------------------------------------------------------------- BLAS-1 (host-facing)
struct Blas {
    Ctx* c;
    DevBuf<double> partial;  // RED_BLOCKS x 64
    DevBuf<double> red;      // 64
    explicit Blas(Ctx* ctx) : c(ctx), partial(ctx, (size_t)RED_BLOCKS * 64), red(ctx, 64) {}

    // out_dev[k] = V_k . w for k < nvec
    void multidot(const double* V, int64_t ldv, int nvec, const double* w, int64_t n, double* out_dev) {
        if (nvec == 0) return;
        dim3 grid(grid_for(n), (nvec + GROUP - 1) / GROUP);
        Prof pr(c, "gs_multidot", 8.0 * n * (nvec + 1));
        unsigned* cnt = reinterpret_cast<unsigned*>(c->d_scalar_i + 60);
        if ((ldv % 2 == 0 || nvec == 1) && aligned16(V) && aligned16(w))
            k_multidot<true><<<grid, RED_THREADS, 0, c->stream>>>(V, ldv, nvec, w, n, partial.p, out_dev, cnt);
        else
            k_multidot<false><<<grid, RED_THREADS, 0, c->stream>>>(V, ldv, nvec, w, n, partial.p, out_dev, cnt);
        check_launch("multidot");
    }
    // out = w_in - V h  (or V h); returns nothing, norm^2 in red[0] when want_norm
    void multiaxpy(const double* V, int64_t ldv, int nv, const double* h, double hscale, const double* w_in,
                   double* out, int64_t n, double* norm2_dev) {
        int g = grid_for(n);
        Prof pr(c, "gs_multiaxpy", 8.0 * n * (nv + (w_in ? 2 : 1)));
        const bool v2 = (ldv % 2 == 0 || nv <= 1) && aligned16(V) && aligned16(out) && (!w_in || aligned16(w_in));
        unsigned* cnt = reinterpret_cast<unsigned*>(c->d_scalar_i + 60);
        if (v2)
            k_multiaxpy<true><<<g, RED_THREADS, 0, c->stream>>>(V, ldv, nv, h, hscale, w_in, out, n,
                                                                 norm2_dev ? partial.p : nullptr, norm2_dev, cnt);
        else
            k_multiaxpy<false><<<g, RED_THREADS, 0, c->stream>>>(V, ldv, nv, h, hscale, w_in, out, n,
                                                                  norm2_dev ? partial.p : nullptr, norm2_dev, cnt);
        check_launch("multiaxpy");
    }
    // DCGS2 step j on basis V (ld n): dots + coefficients, then the update
    void dcgs2_step(double* V, int64_t n, int j, int m, double* H, double* h1, double* coef, double* hcol,
                    double* part2, int part2_rows) {
        const int nv = j + 1;
        const int groups = (nv + D2_GROUP - 1) / D2_GROUP;
        // one wave of resident blocks (2 per SM at 128 registers): no tail wave
        int64_t ranges = std::max<int64_t>(1, std::min<int64_t>((EDFA_DOTS2_WAVE * NUM_SMS_B200) / groups,
                                                                (n + 511) / 512));
        ranges = std::min<int64_t>(ranges, part2_rows);
        int64_t range = (n + ranges - 1) / ranges;
        range = (range + 1) & ~int64_t(1);
        ranges = (n + range - 1) / range;
        unsigned* cnt = reinterpret_cast<unsigned*>(c->d_scalar_i + 60);
        const bool v2 = n % 2 == 0 && aligned16(V);
        {
            Prof pr(c, "gs_dots2", 8.0 * n * (nv + 1));
            dim3 grid(groups, (unsigned)ranges);
            if (v2)
                k_dots2<true><<<grid, RED_THREADS, 0, c->stream>>>(V, n, nv, n, range, part2, part2_rows, cnt, j, m, H,
                                                                  h1, coef, hcol);
            else
                k_dots2<false><<<grid, RED_THREADS, 0, c->stream>>>(V, n, nv, n, range, part2, part2_rows, cnt, j, m,
                                                                   H, h1, coef, hcol);
            check_launch("dots2");
        }
        {
            Prof pr(c, "gs_axpy2", 8.0 * n * (nv + 1) + 8.0 * n * (j > 0 ? 2 : 1));
            if (v2)
                k_axpy2<true><<<grid_for(n), RED_THREADS, 0, c->stream>>>(V, n, j, n, coef);
            else
                k_axpy2<false><<<grid_for(n), RED_THREADS, 0, c->stream>>>(V, n, j, n, coef);
            check_launch("axpy2");
        }
    }
    // split DCGS2 step for slab-distributed vectors (ld = ldv)
    void dcgs2_dots(const double* V, int64_t ldv, int64_t n, int j, double* dots_out, double* part2, int part2_rows) {
        const int nv = j + 1;
        const int groups = (nv + D2_GROUP - 1) / D2_GROUP;
        int64_t ranges = std::max<int64_t>(1, std::min<int64_t>((EDFA_DOTS2_WAVE * NUM_SMS_B200) / groups,
                                                                (n + 511) / 512));
        ranges = std::min<int64_t>(ranges, part2_rows);
        int64_t range = (n + ranges - 1) / ranges;
        range = (range + 1) & ~int64_t(1);
        ranges = (n + range - 1) / range;
        unsigned* cnt = reinterpret_cast<unsigned*>(c->d_scalar_i + 60);
        const bool v2 = n % 2 == 0 && ldv % 2 == 0 && aligned16(V);
        Prof pr(c, "gs_dots2", 8.0 * n * (nv + 1));
        dim3 grid(groups, (unsigned)ranges);
        double* Vm = const_cast<double*>(V);
        if (v2)
            k_dots2<true><<<grid, RED_THREADS, 0, c->stream>>>(Vm, ldv, nv, n, range, part2, part2_rows, cnt, j, 0,
                                                              nullptr, nullptr, nullptr, dots_out);
        else
            k_dots2<false><<<grid, RED_THREADS, 0, c->stream>>>(Vm, ldv, nv, n, range, part2, part2_rows, cnt, j, 0,
                                                               nullptr, nullptr, nullptr, dots_out);
        check_launch("dots2");
    }
    void dcgs2_coeffs(const double* dots, int j, int m, double* H, double* h1, double* coef, double* hcol) {
        k_dcgs2_coeffs<<<1, RED_THREADS, 0, c->stream>>>(dots, j, m, H, h1, coef, hcol);
        check_launch("dcgs2_coeffs");
    }
    void dcgs2_update(double* V, int64_t ldv, int64_t n, int j, const double* coef) {
        const bool v2 = n % 2 == 0 && ldv % 2 == 0 && aligned16(V);
        Prof pr(c, "gs_axpy2", 8.0 * n * (j + 2) + 8.0 * n * (j > 0 ? 2 : 1));
        if (v2)
            k_axpy2<true><<<grid_for(n), RED_THREADS, 0, c->stream>>>(V, ldv, j, n, coef);
        else
            k_axpy2<false><<<grid_for(n), RED_THREADS, 0, c->stream>>>(V, ldv, j, n, coef);
        check_launch("axpy2");
    }
    double dot(const double* x, const double* y, int64_t n) {
        // x . y through the multidot path with V = x as a single vector
        multidot(x, 0, 1, y, n, red.p);
        double h;
        EDFA_CUDA(cudaMemcpyAsync(&h, red.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        EDFA_CUDA(cudaStreamSynchronize(c->stream));
        return h;
    }
    void normalize(int64_t n, const double* nrm2_dev, double* w) {
        Prof pr(c, "axpby", 16.0 * n);
        k_normalize<<<grid_for(n), RED_THREADS, 0, c->stream>>>(n, nrm2_dev, w);
        check_launch("normalize");
    }
    void axpby(int64_t n, double a, const double* x, double b, double* y) {
        Prof pr(c, "axpby", 24.0 * n);
        k_axpby<<<grid_for(n), RED_THREADS, 0, c->stream>>>(n, a, x, b, y);
        check_launch("axpby");
    }
};

// ---------------------------------------------------------------- apply
struct ApplyWS {
    DevBuf<double> a_f, t_f, u_c, c_c;
    DevBuf<double> c_s, y_s;        // slot-order cell vectors of the wavefront-packed ILU solves
};

static void precond_apply(Ctx* c, const edfa_system* sys, const edfa_stage1* s1, const edfa_stage2* s2,
                          ApplyWS& ws, const double* r, double* y) {
    const int nf = sys->A_ff->n_rows, nc = sys->A_cc->n_rows;
    if (!ws.a_f.p && nf) {
        ws.a_f.reset(c, nf);
        ws.t_f.reset(c, nf);
    }
    const IluFactor& il = s2->ilu;
    const bool wf = nc && il.fwd.is_wf && il.bwd.is_wf && il.bwd.wf_shared;   // else: natural hand-over (run_plan)
    if (wf && !ws.c_s.p) {
        const int ns = il.fwd.n_slots;
        ws.u_c.reset(c, nc);
        ws.c_s.reset(c, ns);
        ws.y_s.reset(c, ns);
        fill_bits(c, ws.c_s.p, ns, SENTINEL_BITS);   // kept SENTINEL between applies (U resets what it reads)
    }
    if (!wf && !ws.u_c.p && nc) {
        ws.u_c.reset(c, nc);
        ws.c_c.reset(c, nc);
        fill_bits(c, ws.c_c.p, nc, SENTINEL_BITS);   // kept SENTINEL between applies (tile path)
    }
    const double* r_f = r;
    const double* r_c = r + nf;
    double* y_f = y;
    double* y_c = y + nf;
    const IcFactor& ic = s1->ic;
    // (L L^T)^{-1}: one fused chain kernel when the factor is chain-structured
    const bool pair = ic.fwd.is_chain && ic.bwd.is_chain && c->opt.ic_pair;
    if (!pair || !run_chain_pair(c, ic.fwd.chain, r_f, -1.0, ws.t_f.p, nullptr, nullptr, "trsv_ic_pair")) {
        run_plan(c, ic.fwd, r_f, -1.0, ws.a_f.p, nullptr, nullptr, "trsv_ic_L");
        run_plan(c, ic.bwd, ws.a_f.p, 1.0, ws.t_f.p, nullptr, nullptr, "trsv_ic_LT");
    }
    const bool fuse = nc && il.fwd.is_tile && il.bwd.is_tile && c->opt.fill_fusion;
    if (wf) {
        // L gathers its right-hand side by row, both solves keep their vectors in the
        // factor's slot order (c_s, y_s), U scatters y_c back to natural order
        EDFA_CUDA(cudaMemcpyAsync(ws.u_c.p, r_c, sizeof(double) * nc, cudaMemcpyDeviceToDevice, c->stream));
        spmv_sell(c, sys->sAcf, ws.t_f.p, ws.u_c.p, -1.0, 1.0, "spmv_Acf");
        run_wf(c, il.fwd, ws.u_c.p, false, 1.0, ws.c_s.p, false, nullptr, nullptr, nullptr, nullptr, ws.y_s.p,
               "trsv_ilu_L");
        run_wf(c, il.bwd, ws.c_s.p, true, 1.0, ws.y_s.p, false, y_c, nullptr, nullptr, ws.c_s.p, nullptr,
               "trsv_ilu_U");
        spmv_sell(c, sys->sAfc, y_c, ws.a_f.p, 1.0, 0.0, "spmv_Afc");
    } else if (nc) {
        EDFA_CUDA(cudaMemcpyAsync(ws.u_c.p, r_c, sizeof(double) * nc, cudaMemcpyDeviceToDevice, c->stream));
        spmv_sell(c, sys->sAcf, ws.t_f.p, ws.u_c.p, -1.0, 1.0, "spmv_Acf");
        if (fuse) {
            // L writes c_c (SENTINEL since the last apply's U solve consumed it)
            // and pre-fills y_c; U consumes c_c (resets it) and writes y_c
            run_tile_ex(c, const_cast<TilePlan&>(il.fwd.tile), ws.u_c.p, 1.0, ws.c_c.p, nullptr, nullptr, "trsv_ilu_L",
                        true, false, y_c);
            run_tile_ex(c, const_cast<TilePlan&>(il.bwd.tile), ws.c_c.p, 1.0, y_c, nullptr, nullptr, "trsv_ilu_U",
                        true, true, nullptr);
        } else {
            run_plan(c, il.fwd, ws.u_c.p, 1.0, ws.c_c.p, nullptr, nullptr, "trsv_ilu_L");
            run_plan(c, il.bwd, ws.c_c.p, 1.0, y_c, nullptr, nullptr, "trsv_ilu_U");
            if (il.fwd.is_tile) fill_bits(c, ws.c_c.p, nc, SENTINEL_BITS);   // restore the invariant
        }
        spmv_sell(c, sys->sAfc, y_c, ws.a_f.p, 1.0, 0.0, "spmv_Afc");
    } else if (nf) {
        EDFA_CUDA(cudaMemsetAsync(ws.a_f.p, 0, sizeof(double) * nf, c->stream));
    }
    if (nf) {
        const bool done = pair && run_chain_pair(c, ic.fwd.chain, ws.a_f.p, 1.0, nullptr, ws.t_f.p, y_f, "trsv_ic_pair");
        if (!done) {
            run_plan(c, ic.fwd, ws.a_f.p, 1.0, y_f, nullptr, nullptr, "trsv_ic_L");
            // b and out2 alias row-wise only (thread r reads b[r] before writing out2[r])
            run_plan(c, ic.bwd, y_f, 1.0, ws.a_f.p, ws.t_f.p, y_f, "trsv_ic_LT");
        }
    }
}

void inner_apply(Ctx* c, const edfa_stage1* s1, const edfa_stage2* s2, int which, const double* r, double* y) {
    if (which == 0) {
        const IcFactor& ic = s1->ic;
        DevBuf<double> tmp(c, std::max(ic.n, 1));
        run_plan(c, ic.fwd, r, 1.0, tmp.p, nullptr, nullptr, "trsv_ic_L");
        run_plan(c, ic.bwd, tmp.p, 1.0, y, nullptr, nullptr, "trsv_ic_LT");
    } else {
        const IluFactor& il = s2->ilu;
        DevBuf<double> tmp(c, std::max(il.n, 1));
        run_plan(c, il.fwd, r, 1.0, tmp.p, nullptr, nullptr, "trsv_ilu_L");
        run_plan(c, il.bwd, tmp.p, 1.0, y, nullptr, nullptr, "trsv_ilu_U");
    }
}

// ---------------------------------------------------------------- solver plumbing
struct Operator {
    Ctx* c;
    const edfa_system* sys;
    const edfa_stage1* s1;
    const edfa_stage2* s2;
    ApplyWS ws;
    int64_t n;
    void A(const double* x, double* y) { spmv_sell(c, sys->sA, x, y, 1.0, 0.0, "spmv_A"); }
    void P(const double* x, double* y) {
        if (s1 && s2) precond_apply(c, sys, s1, s2, ws, x, y);
        else EDFA_CUDA(cudaMemcpyAsync(y, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
    }
};


void gmres(Ctx* c, const edfa_system* sys, const edfa_stage1* s1, const edfa_stage2* s2, const double* b, double* x,
           double rtol, int m, int max_it, edfa_report* rep, double* hist, int hist_cap) {
    // Right-preconditioned restarted GMRES(m), x0 = 0 (hx/krylov.py
    // conventions), Arnoldi by DCGS2 (k_dots2 / k_axpy2: one
    // reduction and two basis passes per step).  Step s applies A P to u_s and
    // finalises Hessenberg column s-1 on the device; the host enqueues step
    // s+1 before reading column s-1 back (pinned copy + event), applies the
    // Givens rotations and tests the estimate, so the GPU never idles between
    // steps.  Speculatively enqueued steps only touch slots above the ones the
    // solution update reads.  Convergence is confirmed on the true residual.
    require(rtol > 0.0, EDFA_ERR_VALUE, "tol must be positive");
    require(m >= 1 && m <= 62, EDFA_ERR_VALUE, "restart must be in [1, 62]");
    require(max_it >= 0, EDFA_ERR_VALUE, "max_it must be >= 0");
    c->trsv_err_reset();   // a stale flag of an earlier call must not leak into this solve
    const int64_t n = (int64_t)sys->A.n_rows;
    Operator op{c, sys, s1, s2, {}, n};
    Blas bl(c);
    *rep = edfa_report{0, 0, 0, 0, INFINITY};
    auto push_hist = [&](double v) {
        if (hist && rep->n_hist < hist_cap) hist[rep->n_hist] = v;
        rep->n_hist++;
    };
    double bnorm = std::sqrt(bl.dot(b, b, n));
    if (bnorm == 0.0) {
        EDFA_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, c->stream));
        rep->converged = 1;
        rep->final_relres = 0.0;
        push_hist(0.0);
        EDFA_CUDA(cudaStreamSynchronize(c->stream));
        return;
    }
    const int ld = m + 1;
    const int part_rows = 4 * NUM_SMS_B200;
    // device state: basis (m+2 slots), Hessenberg (unrotated, (m+1) x m col-major),
    // first-pass coefficients, update coefficients, per-step column slots (parity s & 1)
    DevBuf<double> V(c, (size_t)(m + 2) * n), z(c, n), r(c, n), Hd(c, (size_t)ld * m), h1(c, 64), coef(c, 192),
        hcol(c, 2 * 64 + 64), part2(c, (size_t)part_rows * 128);
    double* hpin = c->h_pinned;   // 2 x 64 host column slots + 64 for y
    cudaEvent_t ev[2] = {c->get_event(), c->get_event()};
    EDFA_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, c->stream));
    EDFA_CUDA(cudaMemcpyAsync(r.p, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
    double beta = bnorm;
    std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), y(m);
    bool happy = false;
    auto enqueue_step = [&](int st) {
        double* us = V.p + (int64_t)st * n;
        double* w = us + n;
        op.P(us, z.p);
        op.A(z.p, w);
        double* hc = hcol.p + (st & 1) * 64;
        bl.dcgs2_step(V.p, n, st, m, Hd.p, h1.p, coef.p, hc, part2.p, part_rows);
        if (st >= 1) {
            EDFA_CUDA(cudaMemcpyAsync(hpin + (st & 1) * 64, hc, sizeof(double) * (st + 1), cudaMemcpyDeviceToHost,
                                      c->stream));
            EDFA_CUDA(cudaEventRecord(ev[st & 1], c->stream));
        }
    };
    while (rep->n_it < max_it) {
        bl.axpby(n, 1.0 / beta, r.p, 0.0, V.p);
        std::fill(H.begin(), H.end(), 0.0);
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = beta;
        int k = 0;
        const int budget = std::min(m, max_it - rep->n_it);   // columns this cycle
        int enq = 0;                                          // steps enqueued (step s finalises column s-1)
        enqueue_step(enq++);
        enqueue_step(enq++);
        for (int j = 0; j < budget; ++j) {
            if (enq <= budget) enqueue_step(enq++);            // keep one step ahead of the host
            EDFA_CUDA(cudaEventSynchronize(ev[(j + 1) & 1]));
            const double* hp = hpin + ((j + 1) & 1) * 64;
            rep->n_it++;
            for (int i = 0; i <= j + 1; ++i) H[(size_t)i * m + j] = hp[i];
            const double wn = hp[j + 1];
            for (int i = 0; i < j; ++i) {
                double a = H[(size_t)i * m + j], bb = H[(size_t)(i + 1) * m + j];
                H[(size_t)i * m + j] = cs[i] * a + sn[i] * bb;
                H[(size_t)(i + 1) * m + j] = -sn[i] * a + cs[i] * bb;
            }
            double den = std::hypot(H[(size_t)j * m + j], H[(size_t)(j + 1) * m + j]);
            if (den == 0.0) { cs[j] = 1.0; sn[j] = 0.0; }
            else { cs[j] = H[(size_t)j * m + j] / den; sn[j] = H[(size_t)(j + 1) * m + j] / den; }
            H[(size_t)j * m + j] = den;
            H[(size_t)(j + 1) * m + j] = 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            double est = std::fabs(g[j + 1]) / bnorm;
            push_hist(est);
            k = j + 1;
            if (wn == 0.0) { happy = true; break; }
            if (est <= rtol) break;
        }
        // speculatively enqueued steps may still be running: everything below is
        // stream-ordered after them and reads only slots 0..k-1, which they never write
        for (int i = k - 1; i >= 0; --i) {   // back substitution H y = g
            double sacc = g[i];
            for (int t = i + 1; t < k; ++t) sacc -= H[(size_t)i * m + t] * y[t];
            y[i] = H[(size_t)i * m + i] != 0.0 ? sacc / H[(size_t)i * m + i] : 0.0;
        }
        for (int i = 0; i < k; ++i) hpin[128 + i] = y[i];
        double* yd = hcol.p + 128;
        EDFA_CUDA(cudaMemcpyAsync(yd, hpin + 128, sizeof(double) * k, cudaMemcpyHostToDevice, c->stream));
        bl.multiaxpy(V.p, n, k, yd, 1.0, nullptr, r.p, n, nullptr);   // r <- V y (scratch)
        op.P(r.p, z.p);
        bl.axpby(n, 1.0, z.p, 1.0, x);
        op.A(x, r.p);
        bl.axpby(n, 1.0, b, -1.0, r.p);                                   // r = b - A x
        beta = std::sqrt(bl.dot(r.p, r.p, n));
        c->trsv_err_check();
        if (beta / bnorm <= rtol) { rep->converged = 1; break; }
        if (happy || beta == 0.0) { rep->breakdown = 1; break; }
    }
    c->event_pool.push_back(ev[0]);
    c->event_pool.push_back(ev[1]);
    rep->final_relres = beta / bnorm;
    if (rep->n_it == 0) push_hist(beta / bnorm);
}

void bicgstab(Ctx* c, const edfa_system* sys, const edfa_stage1* s1, const edfa_stage2* s2, const double* b,
              double* x, double rtol, int max_it, edfa_report* rep, double* hist, int hist_cap) {
    // operation-for-operation restatement of hx/krylov.py:40-115
    require(rtol > 0.0, EDFA_ERR_VALUE, "tol must be positive");
    c->trsv_err_reset();
    const int64_t n = (int64_t)sys->A.n_rows;
    Operator op{c, sys, s1, s2, {}, n};
    Blas bl(c);
    *rep = edfa_report{0, 0, 0, 0, INFINITY};
    auto push_hist = [&](double v) {
        if (hist && rep->n_hist < hist_cap) hist[rep->n_hist] = v;
        rep->n_hist++;
    };
    double bnorm = std::sqrt(bl.dot(b, b, n));
    EDFA_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, c->stream));
    if (bnorm == 0.0) {
        rep->converged = 1;
        rep->final_relres = 0.0;
        push_hist(0.0);
        EDFA_CUDA(cudaStreamSynchronize(c->stream));
        return;
    }
    DevBuf<double> r(c, n), rh(c, n), p(c, n), v(c, n), ph(c, n), s(c, n), sh(c, n), t(c, n);
    EDFA_CUDA(cudaMemcpyAsync(r.p, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
    EDFA_CUDA(cudaMemcpyAsync(rh.p, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
    EDFA_CUDA(cudaMemsetAsync(p.p, 0, sizeof(double) * n, c->stream));
    EDFA_CUDA(cudaMemsetAsync(v.p, 0, sizeof(double) * n, c->stream));
    double rho = 1.0, alpha = 1.0, omega = 1.0;
    bool any_hist = false;
    while (rep->n_it < max_it) {
        double rho_new = bl.dot(rh.p, r.p, n);
        if (rho_new == 0.0) { rep->breakdown = 1; break; }
        double beta = (rho_new / rho) * (alpha / omega);
        rho = rho_new;
        {
            Prof pr(c, "axpby", 32.0 * n);
            k_bicg_p<<<grid_for(n), RED_THREADS, 0, c->stream>>>(n, r.p, beta, omega, v.p, p.p);
            check_launch("k_bicg_p");
        }
        op.P(p.p, ph.p);
        op.A(ph.p, v.p);
        double den = bl.dot(rh.p, v.p, n);
        if (den == 0.0) { rep->breakdown = 1; break; }
        alpha = rho / den;
        EDFA_CUDA(cudaMemcpyAsync(s.p, r.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
        bl.axpby(n, -alpha, v.p, 1.0, s.p);
        rep->n_it++;
        double snorm = std::sqrt(bl.dot(s.p, s.p, n));
        if (snorm / bnorm <= rtol) {
            bl.axpby(n, alpha, ph.p, 1.0, x);
            push_hist(snorm / bnorm);
            any_hist = true;
            rep->converged = 1;
            break;
        }
        op.P(s.p, sh.p);
        op.A(sh.p, t.p);
        double tt = bl.dot(t.p, t.p, n);
        if (tt == 0.0) { rep->breakdown = 1; break; }
        omega = bl.dot(t.p, s.p, n) / tt;
        {
            Prof pr(c, "axpby", 32.0 * n);
            k_lincomb3<<<grid_for(n), RED_THREADS, 0, c->stream>>>(n, alpha, ph.p, omega, sh.p, x);
            check_launch("k_lincomb3");
        }
        EDFA_CUDA(cudaMemcpyAsync(r.p, s.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
        bl.axpby(n, -omega, t.p, 1.0, r.p);
        double rr = std::sqrt(bl.dot(r.p, r.p, n)) / bnorm;
        push_hist(rr);
        any_hist = true;
        if (rr <= rtol) { rep->converged = 1; break; }
        if (omega == 0.0) { rep->breakdown = 1; break; }
    }
    if (!any_hist) push_hist(std::sqrt(bl.dot(r.p, r.p, n)) / bnorm);
    op.A(x, t.p);
    bl.axpby(n, 1.0, b, -1.0, t.p);
    rep->final_relres = std::sqrt(bl.dot(t.p, t.p, n)) / bnorm;
    c->trsv_err_check();
}

// exported to capi.cu
void apply_entry(Ctx* c, const edfa_system* sys, const edfa_stage1* s1, const edfa_stage2* s2, const double* r,
                 double* y) {
    ApplyWS ws;
    precond_apply(c, sys, s1, s2, ws, r, y);
    // workspace freed stream-ordered on return
}
double dot_entry(Ctx* c, int64_t n, const double* x, const double* y) {
    Blas bl(c);
    return bl.dot(x, y, n);
}
void multidot_entry(Ctx* c, int64_t n, int nvec, const double* V, int64_t ldv, const double* w, double* out_dev) {
    require(nvec >= 0 && nvec <= 64, EDFA_ERR_VALUE, "nvec must be in [0, 64]");
    Blas bl(c);
    bl.multidot(V, ldv, nvec, w, n, out_dev);
}
void multiaxpy_entry(Ctx* c, int64_t n, int nvec, const double* V, int64_t ldv, const double* h, double hscale,
                     const double* w_in, double* out, double* norm2_dev) {
    require(nvec >= 0 && nvec <= 64, EDFA_ERR_VALUE, "nvec must be in [0, 64]");
    Blas bl(c);
    bl.multiaxpy(V, ldv, nvec, h, hscale, w_in, out, n, norm2_dev);
}
void dcgs2_dots_entry(Ctx* c, int64_t n, int j, const double* V, int64_t ldv, double* dots_out) {
    require(j >= 0 && j <= 62, EDFA_ERR_VALUE, "j must be in [0, 62]");
    require(ldv >= n, EDFA_ERR_VALUE, "ldv must be >= n");
    Blas bl(c);
    DevBuf<double> part2(c, (size_t)4 * NUM_SMS_B200 * 128);
    bl.dcgs2_dots(V, ldv, n, j, dots_out, part2.p, 4 * NUM_SMS_B200);
}
void dcgs2_coeffs_entry(Ctx* c, int j, int m, const double* dots, double* H, double* h1, double* coef, double* hcol) {
    require(j >= 0 && j <= m && m >= 1 && m <= 62, EDFA_ERR_VALUE, "need 0 <= j <= m <= 62");
    Blas bl(c);
    bl.dcgs2_coeffs(dots, j, m, H, h1, coef, hcol);
}
void dcgs2_update_entry(Ctx* c, int64_t n, int j, double* V, int64_t ldv, const double* coef) {
    require(j >= 0 && j <= 62, EDFA_ERR_VALUE, "j must be in [0, 62]");
    require(ldv >= n, EDFA_ERR_VALUE, "ldv must be >= n");
    Blas bl(c);
    bl.dcgs2_update(V, ldv, n, j, coef);
}
void axpby_entry(Ctx* c, int64_t n, double a, const double* x, double b, double* y) {
    Blas bl(c);
    bl.axpby(n, a, x, b, y);
}

}  // namespace edfa
