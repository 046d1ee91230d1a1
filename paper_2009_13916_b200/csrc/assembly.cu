// RT0 mixed-hybrid / FV assembly of the 2x2 block system on the device
// (the producer of the EDFA path's inputs).
//
// Restates hx/assembly.py without its per-cell Python loop (252-274):
//   k_elem_ops   B^E by 2x2x2 Gauss with the contravariant Piola map, its
//                inverse cleaned of relative dust < 1e-13 and re-symmetrised,
//                row sums and diagonal                      (hx/assembly.py:57-88)
//   k_face_rows  A_ff = -sum_E P_E Binv^E P_E^T and A_fc from the row sums on
//                free faces; Dirichlet columns go to rhs_f   (186-230, 283-299)
//   k_cell_rows  balance rows with the strong two-sided flux on interior
//                faces and the one-sided flux on the hull: A_cf, A_cc_steady;
//                Dirichlet columns go to rhs_c              (232-281, 283-299)
// update_accumulation (314-333) is A_cc_steady + diag(acc/dt) through the
// canonical csr_sub, and rhs_c = rhs_c_base + acc*p_prev/dt.
//
// One thread per cell / face.  Element operators are stored SoA ([36][n],
// [6][n]) so the row kernels read them coalesced.  Rows come out canonical
// (sorted columns, duplicates summed, exact zeros dropped) as hx/sparse.py:
// 28-34 produces them, built by a count pass, a scan and a fill pass.
#include <cmath>

#include "dev_util.cuh"
#include "edfa_internal.cuh"
#include "objects.cuh"

namespace edfa {
namespace {

constexpr double BINV_CLEAN = 1e-13;   // hx/assembly.py:27 (_BINV_CLEAN)

__device__ __forceinline__ double det3(const double J[3][3]) {
    return J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
           J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
           J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
}

// Elemental operators of every cell.  Corner order and face slots as
// hx/refelem.py:13-26; Gauss points x fastest with unit weights.
__global__ void __launch_bounds__(128) k_elem_ops(int n, const double* __restrict__ xyz,
                                                  const int32_t* __restrict__ e2n, const double* __restrict__ K,
                                                  double gamma, const double* __restrict__ storage,
                                                  double storage_scalar, double* __restrict__ Bi,
                                                  double* __restrict__ rs, double* __restrict__ dg,
                                                  double* __restrict__ vol, double* __restrict__ acc,
                                                  int* __restrict__ bad) {
    int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    double X[8][3];
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        int nd = e2n[8 * (int64_t)e + a];
#pragma unroll
        for (int c = 0; c < 3; ++c) X[a][c] = xyz[3 * (int64_t)nd + c];
    }
    // Kinv = inv(K), symmetrised (hx/assembly.py:79-80)
    double k[3][3], Ki[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) k[a][b] = K[9 * (int64_t)e + 3 * a + b];
    {
        double dk = det3(k);
        double inv = 1.0 / dk;
        Ki[0][0] = (k[1][1] * k[2][2] - k[1][2] * k[2][1]) * inv;
        Ki[0][1] = (k[0][2] * k[2][1] - k[0][1] * k[2][2]) * inv;
        Ki[0][2] = (k[0][1] * k[1][2] - k[0][2] * k[1][1]) * inv;
        Ki[1][0] = (k[1][2] * k[2][0] - k[1][0] * k[2][2]) * inv;
        Ki[1][1] = (k[0][0] * k[2][2] - k[0][2] * k[2][0]) * inv;
        Ki[1][2] = (k[0][2] * k[1][0] - k[0][0] * k[1][2]) * inv;
        Ki[2][0] = (k[1][0] * k[2][1] - k[1][1] * k[2][0]) * inv;
        Ki[2][1] = (k[0][1] * k[2][0] - k[0][0] * k[2][1]) * inv;
        Ki[2][2] = (k[0][0] * k[1][1] - k[0][1] * k[1][0]) * inv;
        // the diagonal tensors of the BASELINE fields invert exactly
        if (k[0][1] == 0.0 && k[0][2] == 0.0 && k[1][0] == 0.0 && k[1][2] == 0.0 && k[2][0] == 0.0 &&
            k[2][1] == 0.0) {
            Ki[0][0] = 1.0 / k[0][0];
            Ki[1][1] = 1.0 / k[1][1];
            Ki[2][2] = 1.0 / k[2][2];
        }
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = a + 1; b < 3; ++b) {
                double s = 0.5 * (Ki[a][b] + Ki[b][a]);
                Ki[a][b] = s;
                Ki[b][a] = s;
            }
    }
    // B = sum_q w M^T Kinv M / det with M[:, f] = J[:, ax(f)] eta_f (hx/assembly.py:57-73).
    // Only the 3x3 P = J^T Kinv J is needed per point: B_fg += eta_f eta_g P[ax_f][ax_g] / det.
    double P6[6][6];
#pragma unroll
    for (int f = 0; f < 6; ++f)
#pragma unroll
        for (int g = 0; g < 6; ++g) P6[f][g] = 0.0;
    double v = 0.0;
    const double G = 0.57735026918962576451;   // 1/sqrt(3)
    bool ok = true;
#pragma unroll 1
    for (int q = 0; q < 8; ++q) {
        const double xi[3] = {(q & 1) ? G : -G, (q & 2) ? G : -G, (q & 4) ? G : -G};
        double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const double s0 = (a == 1 || a == 2 || a == 5 || a == 6) ? 1.0 : -1.0;
            const double s1 = (a == 2 || a == 3 || a == 6 || a == 7) ? 1.0 : -1.0;
            const double s2 = (a >= 4) ? 1.0 : -1.0;
            const double f0 = 1.0 + xi[0] * s0, f1 = 1.0 + xi[1] * s1, f2 = 1.0 + xi[2] * s2;
            const double g0 = s0 * f1 * f2 / 8.0, g1 = s1 * f0 * f2 / 8.0, g2 = s2 * f0 * f1 / 8.0;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                J[c][0] += X[a][c] * g0;
                J[c][1] += X[a][c] * g1;
                J[c][2] += X[a][c] * g2;
            }
        }
        const double det = det3(J);
        if (!(det > 0.0)) ok = false;
        v += det;
        double KJ[3][3];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) KJ[a][b] = Ki[a][0] * J[0][b] + Ki[a][1] * J[1][b] + Ki[a][2] * J[2][b];
        double P[3][3];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) P[a][b] = J[0][a] * KJ[0][b] + J[1][a] * KJ[1][b] + J[2][a] * KJ[2][b];
        double eta[6];
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            eta[2 * ax] = (xi[ax] - 1.0) / 8.0;
            eta[2 * ax + 1] = (xi[ax] + 1.0) / 8.0;
        }
        const double inv_det = 1.0 / det;
#pragma unroll
        for (int f = 0; f < 6; ++f)
#pragma unroll
            for (int g = 0; g < 6; ++g) P6[f][g] += eta[f] * eta[g] * P[f / 2][g / 2] * inv_det;
    }
    if (!ok) atomicMin(bad, e);
    // B *= gamma, symmetrised; Cholesky B = L L^T; Binv = L^-T L^-1
#pragma unroll
    for (int f = 0; f < 6; ++f)
#pragma unroll
        for (int g = f; g < 6; ++g) {
            double s = 0.5 * (gamma * P6[f][g] + gamma * P6[g][f]);
            P6[f][g] = s;
            P6[g][f] = s;
        }
    double Lm[6][6];
#pragma unroll
    for (int j = 0; j < 6; ++j) {
        double d = P6[j][j];
#pragma unroll
        for (int t = 0; t < j; ++t) d -= Lm[j][t] * Lm[j][t];
        if (!(d > 0.0)) {
            ok = false;
            d = 1.0;
        }
        const double ljj = sqrt(d);
        Lm[j][j] = ljj;
#pragma unroll
        for (int i = j + 1; i < 6; ++i) {
            double s = P6[i][j];
#pragma unroll
            for (int t = 0; t < j; ++t) s -= Lm[i][t] * Lm[j][t];
            Lm[i][j] = s / ljj;
        }
    }
    if (!ok) atomicMin(bad, e);
    // W = L^-1 (lower triangular)
    double W[6][6];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
#pragma unroll
        for (int j = 0; j < 6; ++j) W[i][j] = 0.0;
    }
#pragma unroll
    for (int j = 0; j < 6; ++j) {
        W[j][j] = 1.0 / Lm[j][j];
#pragma unroll
        for (int i = j + 1; i < 6; ++i) {
            double s = 0.0;
#pragma unroll
            for (int t = j; t < i; ++t) s += Lm[i][t] * W[t][j];
            W[i][j] = -s / Lm[i][i];
        }
    }
    double Bv[6][6];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int j = i; j < 6; ++j) {
            double s = 0.0;
#pragma unroll
            for (int t = j; t < 6; ++t) s += W[t][i] * W[t][j];
            Bv[i][j] = s;
            Bv[j][i] = s;
        }
    // dust cleaning relative to each row's max, then re-symmetrise (hx/assembly.py:82-85)
    bool keep[6][6];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        double sc = 0.0;
#pragma unroll
        for (int j = 0; j < 6; ++j) sc = fmax(sc, fabs(Bv[i][j]));
#pragma unroll
        for (int j = 0; j < 6; ++j) keep[i][j] = !(fabs(Bv[i][j]) < BINV_CLEAN * sc);
    }
    double C[6][6];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            const double a = keep[i][j] ? Bv[i][j] : 0.0;
            const double b = keep[j][i] ? Bv[j][i] : 0.0;
            C[i][j] = 0.5 * (a + b);
        }
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            Bi[(int64_t)(6 * i + j) * n + e] = C[i][j];
            s += C[i][j];
        }
        rs[(int64_t)i * n + e] = s;
        dg[(int64_t)i * n + e] = C[i][i];
    }
    vol[e] = v;
    acc[e] = v * (storage ? storage[e] : storage_scalar);
}

struct Ent {
    int32_t c;
    double v;
};

// sort by column, sum duplicates in arrival order, drop exact zeros
template <int CAP>
__device__ __forceinline__ int canon(Ent (&a)[CAP], int m) {
    for (int i = 1; i < m; ++i) {
        Ent x = a[i];
        int j = i - 1;
        while (j >= 0 && a[j].c > x.c) {
            a[j + 1] = a[j];
            --j;
        }
        a[j + 1] = x;
    }
    int o = 0;
    for (int i = 0; i < m;) {
        Ent s = a[i++];
        while (i < m && a[i].c == s.c) s.v += a[i++].v;
        if (s.v != 0.0) a[o++] = s;
    }
    return o;
}

// Dirichlet contribution sum_d A[row, d] * p_d in ascending d (a CSR row
// slice times the prescribed values, hx/assembly.py:296-299)
template <int CAP>
__device__ __forceinline__ double dirichlet_sum(Ent (&a)[CAP], int m) {
    canon<CAP>(a, m);
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += a[i].v;
    return s;
}

struct AsmArgs {
    int n_cells, n_faces;
    const int32_t* e2f;
    const int32_t* f2e;
    const int32_t* floc;
    const int32_t* fidx;     // free numbering, -1 = prescribed pressure
    const double* fval;      // prescribed pressure (Dirichlet faces)
    const double* fpi;       // Neumann flux * area per face, or NULL
    const double* Bi;
    const double* rs;
    const double* dg;
    const double* vol;
    const double* src;       // per-cell source, or NULL
};

// Flux-continuity rows of the free faces (A_ff, A_fc, rhs_f).
template <bool FILL>
__global__ void k_face_rows(AsmArgs a, int32_t* __restrict__ cnt_ff, int32_t* __restrict__ cnt_fc,
                            const int32_t* __restrict__ ptr_ff, int32_t* __restrict__ idx_ff,
                            double* __restrict__ val_ff, const int32_t* __restrict__ ptr_fc,
                            int32_t* __restrict__ idx_fc, double* __restrict__ val_fc, double* __restrict__ rhs_f) {
    int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= a.n_faces) return;
    const int row = a.fidx[f];
    if (row < 0) return;
    const int n = a.n_cells;
    Ent ff[12], dd[12], fc[2];
    int nff = 0, ndd = 0, nfc = 0;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
        const int e = a.f2e[2 * f + side];
        if (e < 0) continue;
        const int l = a.floc[2 * f + side];
        for (int m = 0; m < 6; ++m) {
            const int col = a.e2f[6 * (int64_t)e + m];
            const double v = -a.Bi[(int64_t)(6 * l + m) * n + e];
            const int fc_ = a.fidx[col];
            if (fc_ >= 0) ff[nff++] = Ent{fc_, v};
            else dd[ndd++] = Ent{col, v * a.fval[col]};
        }
        fc[nfc++] = Ent{e, a.rs[(int64_t)l * n + e]};
    }
    nff = canon<12>(ff, nff);
    nfc = canon<2>(fc, nfc);
    if (!FILL) {
        cnt_ff[row] = nff;
        cnt_fc[row] = nfc;
        return;
    }
    int o = ptr_ff[row];
    for (int i = 0; i < nff; ++i) {
        idx_ff[o + i] = ff[i].c;
        val_ff[o + i] = ff[i].v;
    }
    o = ptr_fc[row];
    for (int i = 0; i < nfc; ++i) {
        idx_fc[o + i] = fc[i].c;
        val_fc[o + i] = fc[i].v;
    }
    const double pi = a.fpi ? a.fpi[f] : 0.0;
    rhs_f[row] = ndd ? pi - dirichlet_sum<12>(dd, ndd) : pi;
}

// Balance rows of the cells (A_cf, A_cc_steady, rhs_c_base).
template <bool FILL>
__global__ void __launch_bounds__(128) k_cell_rows(AsmArgs a, int32_t* __restrict__ cnt_cf,
                                                   int32_t* __restrict__ cnt_cc, const int32_t* __restrict__ ptr_cf,
                                                   int32_t* __restrict__ idx_cf, double* __restrict__ val_cf,
                                                   const int32_t* __restrict__ ptr_cc, int32_t* __restrict__ idx_cc,
                                                   double* __restrict__ val_cc, double* __restrict__ rhs_c,
                                                   int* __restrict__ bad_w) {
    int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= a.n_cells) return;
    const int n = a.n_cells;
    int nb[6], nl[6], fe[6];
    double w[6], dgs[6];
#pragma unroll
    for (int s = 0; s < 6; ++s) {
        const int f = a.e2f[6 * (int64_t)e + s];
        fe[s] = f;
        const int c0 = a.f2e[2 * f], c1 = a.f2e[2 * f + 1];
        const bool own = c0 == e;
        nb[s] = own ? c1 : c0;
        nl[s] = nb[s] >= 0 ? a.floc[2 * f + (own ? 1 : 0)] : -1;
        dgs[s] = a.dg[(int64_t)s * n + e];
        if (nb[s] >= 0) {
            const double d_o = a.dg[(int64_t)nl[s] * n + nb[s]];
            const double den = dgs[s] + d_o;
            if (!(den > 0.0)) atomicMin(bad_w, e);
            w[s] = d_o / den;
        } else {
            w[s] = 1.0;
        }
    }
    Ent cf[40], dd[40], cc[8];
    int ncf = 0, ndd = 0, ncc = 0;
    double diag = 0.0;
#pragma unroll
    for (int j = 0; j < 6; ++j) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < 6; ++i) s += w[i] * a.Bi[(int64_t)(6 * i + j) * n + e];
        double coef = -s;
        if (nb[j] >= 0) coef += w[j] * dgs[j];
        const int col = a.fidx[fe[j]];
        if (col >= 0) cf[ncf++] = Ent{col, coef};
        else dd[ndd++] = Ent{fe[j], coef * a.fval[fe[j]]};
        diag += w[j] * a.rs[(int64_t)j * n + e];
    }
    cc[ncc++] = Ent{e, diag};
    for (int s = 0; s < 6; ++s) {
        if (nb[s] < 0) continue;
        const int m_ = nb[s], ln = nl[s];
        const double wf = 1.0 - w[s];
        for (int t = 0; t < 6; ++t) {
            if (t == ln) continue;
            const double v = wf * a.Bi[(int64_t)(6 * ln + t) * n + m_];
            if (v == 0.0) continue;
            const int face = a.e2f[6 * (int64_t)m_ + t];
            const int col = a.fidx[face];
            if (col >= 0) cf[ncf++] = Ent{col, v};
            else dd[ndd++] = Ent{face, v * a.fval[face]};
        }
        cc[ncc++] = Ent{m_, -wf * a.rs[(int64_t)ln * n + m_]};
    }
    ncf = canon<40>(cf, ncf);
    ncc = canon<8>(cc, ncc);
    if (!FILL) {
        cnt_cf[e] = ncf;
        cnt_cc[e] = ncc;
        return;
    }
    int o = ptr_cf[e];
    for (int i = 0; i < ncf; ++i) {
        idx_cf[o + i] = cf[i].c;
        val_cf[o + i] = cf[i].v;
    }
    o = ptr_cc[e];
    for (int i = 0; i < ncc; ++i) {
        idx_cc[o + i] = cc[i].c;
        val_cc[o + i] = cc[i].v;
    }
    const double base = a.vol[e] * (a.src ? a.src[e] : 0.0);
    rhs_c[e] = ndd ? base - dirichlet_sum<40>(dd, ndd) : base;
}

__global__ void k_free_flags(int n, const int8_t* __restrict__ bc, int32_t* __restrict__ keep) {
    int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f < n) keep[f] = bc[f] != 1;
}

__global__ void k_face_prep(int n, const int8_t* __restrict__ bc, const double* __restrict__ value,
                            const double* __restrict__ area, const int32_t* __restrict__ ptr,
                            int32_t* __restrict__ fidx, double* __restrict__ fval, double* __restrict__ fpi) {
    int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= n) return;
    const int k = bc[f];
    fidx[f] = k == 1 ? -1 : ptr[f];
    fval[f] = k == 1 ? value[f] : 0.0;
    fpi[f] = k == 2 ? value[f] * area[f] : 0.0;
}

__global__ void k_diag_csr(int n, const double* __restrict__ acc, double dt, int32_t* __restrict__ ptr,
                           int32_t* __restrict__ idx, double* __restrict__ val) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    ptr[i] = i;
    if (i < n) {
        idx[i] = i;
        val[i] = -(acc[i] / dt);   // A + acc/dt == A - (-(acc/dt)) exactly
    }
}

__global__ void k_accum_rhs(int n, const double* __restrict__ base, const double* __restrict__ acc,
                            const double* __restrict__ p_prev, double dt, double* __restrict__ rhs) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) rhs[i] = base[i] + acc[i] * (p_prev ? p_prev[i] : 0.0) / dt;
}

// ---- after the solve (hx/assembly.py:334-387, hx/driver.py:67-71)
__global__ void k_face_pressures(int nf, const int32_t* __restrict__ fidx, const double* __restrict__ fval,
                                 const double* __restrict__ pi, double* __restrict__ out) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f < nf) out[f] = fidx[f] >= 0 ? pi[fidx[f]] : fval[f];
}

// one-sided fluxes q1 = rs p - Binv pi_local and strong-flux numerators lam = q1 + diag pi_local
__global__ void k_cell_flux(int n, const int32_t* __restrict__ e2f, const double* __restrict__ pf,
                            const double* __restrict__ p, const double* __restrict__ Bi,
                            const double* __restrict__ rs, const double* __restrict__ dg, double* __restrict__ q1,
                            double* __restrict__ lam) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    double pl[6];
#pragma unroll
    for (int j = 0; j < 6; ++j) pl[j] = pf[e2f[6 * (int64_t)e + j]];
    const double pe = p[e];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < 6; ++j) s += Bi[(int64_t)(6 * i + j) * n + e] * pl[j];
        const double q = rs[(int64_t)i * n + e] * pe - s;
        q1[(int64_t)i * n + e] = q;
        lam[(int64_t)i * n + e] = q + dg[(int64_t)i * n + e] * pl[i];
    }
}

__global__ void k_face_flux(int nf, int n, const int32_t* __restrict__ f2e, const int32_t* __restrict__ floc,
                            const double* __restrict__ q1, const double* __restrict__ lam,
                            const double* __restrict__ dg, double* __restrict__ q) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nf) return;
    const int o = f2e[2 * f], nb = f2e[2 * f + 1], lo = floc[2 * f];
    if (nb < 0) {
        q[f] = q1[(int64_t)lo * n + o];
        return;
    }
    const int ln = floc[2 * f + 1];
    const double d_o = dg[(int64_t)lo * n + o], d_n = dg[(int64_t)ln * n + nb];
    q[f] = (d_n * lam[(int64_t)lo * n + o] - d_o * lam[(int64_t)ln * n + nb]) / (d_o + d_n);
}

__device__ __forceinline__ void atomic_max_nonneg(double* p, double v) {
    if (!(v >= 0.0)) return;
    atomicMax(reinterpret_cast<unsigned long long*>(p), (unsigned long long)__double_as_longlong(v));
}

// chi = outflow rate * dt / pore volume; max chi and max |p_new - p_old|
__global__ void k_cfl(int n, const int32_t* __restrict__ e2f, const int32_t* __restrict__ f2e,
                      const double* __restrict__ q, const double* __restrict__ vol, const double* __restrict__ phi,
                      double phi_s, double dt, const double* __restrict__ pn, const double* __restrict__ po,
                      double* __restrict__ chi, double* __restrict__ mx) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    double c = 0.0, dp = 0.0;
    if (e < n) {
        double rate = 0.0;
#pragma unroll
        for (int s = 0; s < 6; ++s) {
            const int f = e2f[6 * (int64_t)e + s];
            const double o = (f2e[2 * f] == e ? 1.0 : -1.0) * q[f];
            rate += o > 0.0 ? o : 0.0;
        }
        c = rate * dt / (vol[e] * (phi ? phi[e] : phi_s));
        if (chi) chi[e] = c;
        if (pn && po) dp = fabs(pn[e] - po[e]);
    }
    c = warp_max(c);
    dp = warp_max(dp);
    if ((threadIdx.x & 31) == 0) {
        atomic_max_nonneg(mx, c);
        atomic_max_nonneg(mx + 1, dp);
    }
}

void alloc_rows(Ctx* c, Csr& M, int32_t rows, int32_t cols, const DevBuf<int32_t>& cnt) {
    M.n_rows = rows;
    M.n_cols = cols;
    M.ptr.reset(c, (size_t)rows + 1);
    M.nnz = scan_counts(c, cnt.p, M.ptr.p, rows);
    M.idx.reset(c, M.nnz);
    M.val.reset(c, M.nnz);
}

}  // namespace

void assemble(Ctx* c, const edfa_hex_grid& g, const edfa_assembly_in& in, edfa_assembly_out& out, Csr& A_ff,
              Csr& A_fc, Csr& A_cf, Csr& A_cc) {
    const int n = g.n_cells, nf = g.n_faces;
    require(n > 0 && nf > 0 && g.n_nodes > 0, EDFA_ERR_VALUE, "empty grid");
    require(g.node_coords && g.elem_to_nodes && g.elem_to_faces && g.face_to_elems && g.face_local &&
                g.face_area && in.K && in.face_bc && in.face_value,
            EDFA_ERR_VALUE, "NULL grid or assembly input");
    require(out.face_index && out.rhs_f && out.rhs_c_base && out.elem_volume && out.accumulation, EDFA_ERR_VALUE,
            "NULL assembly output");
    // free numbering (hx/assembly.py:283-290)
    DevBuf<int32_t> keep(c, nf), fptr(c, (size_t)nf + 1);
    DevBuf<double> fval(c, nf), fpi(c, nf);
    {
        Prof pr(c, "asm_faces", 25.0 * nf);
        k_free_flags<<<ceil_div(nf, 256), 256, 0, c->stream>>>(nf, in.face_bc, keep.p);
        check_launch("k_free_flags");
    }
    const int32_t n_free = (int32_t)scan_counts(c, keep.p, fptr.p, nf);
    {
        Prof pr(c, "asm_faces", 33.0 * nf);
        k_face_prep<<<ceil_div(nf, 256), 256, 0, c->stream>>>(nf, in.face_bc, in.face_value, g.face_area, fptr.p,
                                                              out.face_index, fval.p, fpi.p);
        check_launch("k_face_prep");
    }
    // element operators
    DevBuf<double> Bi_own, rs_own, dg_own;
    double* Bi = out.binv;
    double* rs = out.row_sums;
    double* dg = out.diag;
    if (!Bi) { Bi_own.reset(c, 36 * (size_t)n); Bi = Bi_own.p; }
    if (!rs) { rs_own.reset(c, 6 * (size_t)n); rs = rs_own.p; }
    if (!dg) { dg_own.reset(c, 6 * (size_t)n); dg = dg_own.p; }
    int* bad = c->d_scalar_i + 40;
    int* bad_w = c->d_scalar_i + 41;
    {
        const int big = 0x7fffffff;
        int init[2] = {big, big};
        EDFA_CUDA(cudaMemcpyAsync(bad, init, 2 * sizeof(int), cudaMemcpyHostToDevice, c->stream));
    }
    {
        Prof pr(c, "asm_elem_ops", (32.0 + 72 + 8 * 24 + 8 * (36 + 12 + 2)) * n);
        k_elem_ops<<<ceil_div(n, 128), 128, 0, c->stream>>>(n, g.node_coords, g.elem_to_nodes, in.K, in.gamma,
                                                            in.storage, in.storage_scalar, Bi, rs, dg,
                                                            out.elem_volume, out.accumulation, bad);
        check_launch("k_elem_ops");
    }
    AsmArgs a{n, nf, g.elem_to_faces, g.face_to_elems, g.face_local, out.face_index, fval.p, fpi.p, Bi, rs, dg,
              out.elem_volume, in.source};
    DevBuf<int32_t> cff(c, std::max(n_free, 1)), cfc(c, std::max(n_free, 1)), ccf(c, n), ccc(c, n);
    {
        Prof pr(c, "asm_face_rows", 8.0 * nf * 10);
        k_face_rows<false><<<ceil_div(nf, 128), 128, 0, c->stream>>>(a, cff.p, cfc.p, nullptr, nullptr, nullptr,
                                                                     nullptr, nullptr, nullptr, nullptr);
        check_launch("k_face_rows<count>");
    }
    {
        Prof pr(c, "asm_cell_rows", 8.0 * n * 60);
        k_cell_rows<false><<<ceil_div(n, 128), 128, 0, c->stream>>>(a, ccf.p, ccc.p, nullptr, nullptr, nullptr,
                                                                    nullptr, nullptr, nullptr, nullptr, bad_w);
        check_launch("k_cell_rows<count>");
    }
    int hbad[2];
    EDFA_CUDA(cudaMemcpyAsync(hbad, bad, 2 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
    out.bad_element = hbad[0] == 0x7fffffff ? -1 : hbad[0];
    require(hbad[0] == 0x7fffffff, EDFA_ERR_VALUE,
            "element " + std::to_string(hbad[0]) + " has a non-positive Jacobian");
    require(hbad[1] == 0x7fffffff, EDFA_ERR_VALUE,
            "non-positive interface weight at element " + std::to_string(hbad[1]) +
                "; elemental matrices are not SPD");
    alloc_rows(c, A_ff, n_free, n_free, cff);
    alloc_rows(c, A_fc, n_free, n, cfc);
    alloc_rows(c, A_cf, n, n_free, ccf);
    alloc_rows(c, A_cc, n, n, ccc);
    {
        Prof pr(c, "asm_face_rows", 12.0 * (A_ff.nnz + A_fc.nnz) + 8.0 * nf * 10);
        k_face_rows<true><<<ceil_div(nf, 128), 128, 0, c->stream>>>(a, nullptr, nullptr, A_ff.ptr.p, A_ff.idx.p,
                                                                    A_ff.val.p, A_fc.ptr.p, A_fc.idx.p, A_fc.val.p,
                                                                    out.rhs_f);
        check_launch("k_face_rows<fill>");
    }
    {
        Prof pr(c, "asm_cell_rows", 12.0 * (A_cf.nnz + A_cc.nnz) + 8.0 * n * 60);
        k_cell_rows<true><<<ceil_div(n, 128), 128, 0, c->stream>>>(a, nullptr, nullptr, A_cf.ptr.p, A_cf.idx.p,
                                                                   A_cf.val.p, A_cc.ptr.p, A_cc.idx.p, A_cc.val.p,
                                                                   out.rhs_c_base, bad_w);
        check_launch("k_cell_rows<fill>");
    }
    out.n_free = n_free;
}

void update_accumulation(Ctx* c, const Csr& A_cc_steady, const double* acc, const double* rhs_c_base,
                         const double* p_prev, double dt, Csr& A_cc, double* rhs_c) {
    const int n = A_cc_steady.n_rows;
    require(dt > 0.0, EDFA_ERR_VALUE, "dt must be positive (math.inf for steady state)");
    require(A_cc_steady.n_cols == n, EDFA_ERR_VALUE, "A_cc must be square");
    if (std::isinf(dt)) {
        copy_csr(c, A_cc_steady, A_cc);
        if (n) EDFA_CUDA(cudaMemcpyAsync(rhs_c, rhs_c_base, 8 * (size_t)n, cudaMemcpyDeviceToDevice, c->stream));
        return;
    }
    Csr D;
    D.n_rows = D.n_cols = n;
    D.nnz = n;
    D.ptr.reset(c, (size_t)n + 1);
    D.idx.reset(c, n);
    D.val.reset(c, n);
    {
        Prof pr(c, "asm_accumulation", 24.0 * n);
        k_diag_csr<<<ceil_div(n + 1, 256), 256, 0, c->stream>>>(n, acc, dt, D.ptr.p, D.idx.p, D.val.p);
        check_launch("k_diag_csr");
        k_accum_rhs<<<ceil_div(n, 256), 256, 0, c->stream>>>(n, rhs_c_base, acc, p_prev, dt, rhs_c);
        check_launch("k_accum_rhs");
    }
    csr_sub(c, A_cc_steady, D, 0.0, A_cc);
}

}  // namespace edfa

namespace edfa {

void face_fluxes(Ctx* c, const edfa_hex_grid& g, const int32_t* fidx, const double* fval, const double* Bi,
                 const double* rs, const double* dg, const double* pi, const double* p, double* q) {
    const int n = g.n_cells, nf = g.n_faces;
    require(n > 0 && nf > 0 && g.elem_to_faces && g.face_to_elems && g.face_local && fidx && fval && Bi && rs &&
                dg && pi && p && q,
            EDFA_ERR_VALUE, "NULL grid, element operators or vectors");
    DevBuf<double> pf(c, nf), q1(c, 6 * (size_t)n), lam(c, 6 * (size_t)n);
    Prof pr(c, "asm_fluxes", 8.0 * (nf * 4 + n * 60));
    k_face_pressures<<<ceil_div(nf, 256), 256, 0, c->stream>>>(nf, fidx, fval, pi, pf.p);
    k_cell_flux<<<ceil_div(n, 128), 128, 0, c->stream>>>(n, g.elem_to_faces, pf.p, p, Bi, rs, dg, q1.p, lam.p);
    k_face_flux<<<ceil_div(nf, 256), 256, 0, c->stream>>>(nf, n, g.face_to_elems, g.face_local, q1.p, lam.p, dg, q);
    check_launch("face fluxes");
}

void cfl(Ctx* c, const edfa_hex_grid& g, const double* q, const double* vol, const double* phi, double phi_s,
         double dt, const double* pn, const double* po, double* chi, double* out_host) {
    const int n = g.n_cells;
    require(n > 0 && g.elem_to_faces && g.face_to_elems && q && vol && out_host, EDFA_ERR_VALUE,
            "NULL grid or vectors");
    require(phi || phi_s > 0.0, EDFA_ERR_VALUE, "porosity must lie in (0, 1]");
    double* mx = c->d_scalar_d + 4000;
    EDFA_CUDA(cudaMemsetAsync(mx, 0, 2 * sizeof(double), c->stream));
    {
        Prof pr(c, "asm_cfl", 8.0 * (n * 10));
        k_cfl<<<ceil_div(n, 256), 256, 0, c->stream>>>(n, g.elem_to_faces, g.face_to_elems, q, vol, phi, phi_s, dt,
                                                       pn, po, chi, mx);
        check_launch("k_cfl");
    }
    EDFA_CUDA(cudaMemcpyAsync(out_host, mx, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
}

}  // namespace edfa
