/*
 * edfa.h -- C ABI of libedfa.so, the B200 (sm_100a) implementation of the
 * EDFA block preconditioner and the Krylov solves it accelerates.
 *
 * The entry points replace the reference's hot-path Python API
 * (hexflow 0.1.0, paths relative to /root/reference/pkg/src/hexflow):
 *
 *   edfa_csr_create / edfa_csr_export     scipy CSR blocks of BlockSystem
 *                                         (assembly.py:135-183, sparse.py:28-34)
 *   edfa_system_create                    BlockSystem.full_matrix (assembly.py:168-170)
 *   edfa_pattern_static                   patterns.static_patterns (patterns.py:124-133)
 *   edfa_stage1_build                     precond.build_stage1 (precond.py:204-261)
 *   edfa_stage2_build                     precond.build_stage2 (precond.py:264-271)
 *   edfa_precond_apply                    BlockLDUPreconditioner.apply (precond.py:311-320)
 *   edfa_inner_apply                      InnerFactorization.apply (sparse.py:125-129)
 *   edfa_restricted_solve                 precond.solve_restricted_row (precond.py:70-82)
 *   edfa_grow_dynamic                     precond.grow_pattern_dynamic (precond.py:107-135)
 *   edfa_spmv / edfa_system_spmv          sparse.spmv (sparse.py:37-42), A @ v (driver.py:135-139)
 *   edfa_bicgstab                         krylov.bicgstab (krylov.py:40-115)
 *   edfa_gmres                            GMRES(m) -- absent from the reference
 *   edfa_assemble                         assembly.assemble (assembly.py:186-311), the
 *                                         producer of the path's blocks
 *   edfa_update_accumulation              assembly.update_accumulation (assembly.py:314-333)
 *   edfa_face_fluxes / edfa_cfl           assembly.recover_face_fluxes (assembly.py:334-356),
 *                                         driver.cfl (driver.py:67-71)
 *
 * Conventions
 *   - Every call is stream-ordered on the context's stream.  Calls that must
 *     learn a data-dependent size (stage builds, exports of sizes) or a
 *     convergence decision synchronise that stream; nothing else does.
 *   - Vectors passed to apply/spmv/solve entry points are DEVICE pointers.
 *     Matrix uploads/exports take a memory-space flag (host or device).
 *   - Return value: EDFA_OK or an error code; edfa_last_error() returns the
 *     message of the calling thread's last failure.  Error codes map onto the
 *     reference's exceptions: VALUE -> ValueError, FACTORIZATION ->
 *     FactorizationError (hx/errors.py:16), STATE -> RuntimeError.
 *   - Indices are int32 (row pointers and column ids), values IEEE float64.
 */
#ifndef EDFA_H
#define EDFA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EDFA_ABI_VERSION 1

enum edfa_status {
    EDFA_OK = 0,
    EDFA_ERR_VALUE = 1,          /* invalid argument        -> ValueError          */
    EDFA_ERR_FACTORIZATION = 2,  /* non-SPD restricted block -> FactorizationError  */
    EDFA_ERR_STATE = 3,          /* apply before stage 2    -> RuntimeError        */
    EDFA_ERR_CUDA = 4,           /* CUDA runtime failure                            */
    EDFA_ERR_UNSUPPORTED = 5     /* option not implemented on this path            */
};

enum edfa_filtration {           /* precond.FILTRATION_MODES (precond.py:35) */
    EDFA_FILT_NONE = 0,
    EDFA_FILT_PRE = 1,
    EDFA_FILT_POST_SCHUR = 2,
    EDFA_FILT_POST_PRODUCT = 3
};

enum edfa_mem { EDFA_MEM_HOST = 0, EDFA_MEM_DEVICE = 1 };

enum edfa_stage1_part {          /* Stage1 fields (precond.py:168-176) */
    EDFA_S1_G = 0,               /* G~, cells x faces                          */
    EDFA_S1_FT = 1,              /* F~^T, cells x faces (CSR of F~'s columns)  */
    EDFA_S1_H = 2,               /* H~ = G~ A_ff F~, cells x cells             */
    EDFA_S1_Q = 3,               /* restriction sets (values NULL)             */
    EDFA_S1_L = 4,               /* IC factor L of -A_ff, explicit diagonal    */
    EDFA_S1_F = 5                /* F~, faces x cells                          */
};

enum edfa_stage2_part {          /* Stage2 fields (precond.py:179-184) */
    EDFA_S2_S = 0,               /* S~ = A_cc - H~                             */
    EDFA_S2_L = 1,               /* unit lower ILU factor, explicit diagonal   */
    EDFA_S2_U = 2                /* upper ILU factor, diagonal first           */
};

typedef struct edfa_ctx edfa_ctx;
typedef struct edfa_csr edfa_csr;
typedef struct edfa_system edfa_system;
typedef struct edfa_stage1 edfa_stage1;
typedef struct edfa_stage2 edfa_stage2;
typedef struct edfa_factor edfa_factor;

typedef struct edfa_dynamic {    /* precond.DynamicConfig (precond.py:38-67) */
    int32_t n_add;
    int32_t n_ent;
    int32_t it_max;              /* <= 0 means "None" (sweep limit max(n_ent,1)) */
} edfa_dynamic;

typedef struct edfa_stage1_info {
    int64_t nnz_G, nnz_FT, nnz_H, nnz_Q, nnz_L;
    int32_t max_pattern;
    int32_t pivot_shifts;        /* InnerFactorization.pivot_shifts of the IC */
    int32_t trsv_levels;         /* dependency depth of L (and L^T)           */
} edfa_stage1_info;

typedef struct edfa_stage2_info {
    int64_t nnz_S, nnz_L, nnz_U; /* L, U counted like the reference's CSR     */
    int32_t pivot_shifts;
    int32_t levels_L, levels_U;
} edfa_stage2_info;

typedef struct edfa_report {     /* krylov.SolveReport (krylov.py:15-37) */
    int32_t n_it;
    int32_t converged;
    int32_t breakdown;
    int32_t n_hist;              /* entries written to the history buffer      */
    double final_relres;         /* ||b - A x|| / ||b|| recomputed at the end  */
} edfa_report;

/* ---- library / context ------------------------------------------------- */
int         edfa_abi_version(void);
const char* edfa_last_error(void);
int edfa_ctx_create(int device, void* cuda_stream, edfa_ctx** out);
int edfa_ctx_set_stream(edfa_ctx* ctx, void* cuda_stream);
/* Algorithm selections (defaults = production; alternatives for A/B tests):
 * "ic_pair" (1) fused (L L^T)^-1 chain kernel, "fill_fusion" (1) ILU solves
 * pre-fill each other's SENTINELs, "trsv_levels" (0) level-synchronous
 * triangular solves, "ilu_levels" (0) level-synchronous ILU(0), "tile_direct" (-1)
 * ILU tile solves with early records read from L2 (1) / staged (0) / chosen
 * by wavefront width (-1), "ilu_wf" (-1) ILU solves wavefront-packed on one
 * slot layout (1) / tile-DAG or level plans (0) / chosen by level width (-1),
 * "wf_prefetch" (1) wavefront-packed solves prefetch the next slice's records
 * into shared memory by bulk copies (0: records loaded to registers per slice).  Seeded once
 * from EDFA_OPT_<NAME> at context creation.  Unknown name -> EDFA_ERR_VALUE. */
int edfa_ctx_set_option(edfa_ctx* ctx, const char* name, int value);
int edfa_ctx_get_option(edfa_ctx* ctx, const char* name, int* value);
int edfa_ctx_sync(edfa_ctx* ctx);
/* Return the context's cached (freed, stream-ordered) device blocks to the
 * driver -- synchronises the stream. */
int edfa_ctx_trim(edfa_ctx* ctx);
int edfa_ctx_destroy(edfa_ctx* ctx);
/* Per-kernel CUDA-event timing with algorithmic byte counts (roofline). */
int edfa_ctx_profile(edfa_ctx* ctx, int enable);
/* Restrict event timing to kernels whose name starts with prefix ("" = all). */
int edfa_ctx_profile_filter(edfa_ctx* ctx, const char* prefix);
/* JSON {"kernel": {"launches": n, "ms": t, "bytes": b}, ...}; returns needed length. */
int64_t edfa_ctx_profile_report(edfa_ctx* ctx, char* buf, int64_t cap, int reset);
/* Number of library kernel launches issued so far on this context. */
int64_t edfa_ctx_launch_count(edfa_ctx* ctx);

/* ---- matrices ---------------------------------------------------------- */
int edfa_csr_create(edfa_ctx* ctx, int32_t n_rows, int32_t n_cols, int64_t nnz,
                    const int32_t* indptr, const int32_t* indices, const double* data,
                    int mem, edfa_csr** out);
int edfa_csr_info(const edfa_csr* A, int32_t* n_rows, int32_t* n_cols, int64_t* nnz);
int edfa_csr_export(edfa_ctx* ctx, const edfa_csr* A, int32_t* indptr, int32_t* indices,
                    double* data, int mem);
int edfa_csr_destroy(edfa_csr* A);

/* ---- block system ------------------------------------------------------ */
/* Borrows the four blocks (they must outlive the system); builds the
 * monolithic [[A_ff, A_fc], [A_cf, A_cc]] operator on the device. */
int edfa_system_create(edfa_ctx* ctx, const edfa_csr* A_ff, const edfa_csr* A_fc,
                       const edfa_csr* A_cf, const edfa_csr* A_cc, edfa_system** out);
/* update_accumulation: replace A_cc (face blocks untouched; assembly.py:314-333). */
int edfa_system_set_cc(edfa_ctx* ctx, edfa_system* sys, const edfa_csr* A_cc);
/* Optional hint: cells are the natural-order (x fastest) cells of an
 * nx*ny*nz box (hx/grid.py:49-50).  Enables tile-DAG triangular solves of the
 * Schur ILU; results do not depend on it. */
int edfa_system_set_grid(edfa_system* sys, int32_t nx, int32_t ny, int32_t nz);
int edfa_system_destroy(edfa_system* sys);

/* ---- restriction patterns ---------------------------------------------- */
/* Static prototype 'A'..'E' (patterns.py:63-133).  elem_to_faces and
 * neighbors are n_cells x 6 (global face ids / neighbour cell or -1);
 * face_index maps global -> free face (-1 eliminated). */
int edfa_pattern_static(edfa_ctx* ctx, int32_t n_cells, int32_t n_faces,
                        const int32_t* elem_to_faces, const int32_t* neighbors,
                        const int32_t* face_index, char prototype, int mem,
                        edfa_csr** out);

/* Device-side topology for edfa_pattern_static (hexflow grid.py:100-129,
 * what patterns.static_patterns derives per call on the host): narrows
 * elem_to_faces (n_cells x 6) and face_index (n_faces; optional) to int32 and
 * computes neighbors[e][s] = the other cell of face elem_to_faces[e][s] (-1 on
 * the boundary) from face_to_elems (n_faces x 2).  All pointers are device
 * memory; inputs are int32 or int64 (index_bytes 4 / 8). */
int edfa_grid_topology(edfa_ctx* ctx, int32_t n_cells, int32_t n_faces,
                       const void* elem_to_faces, const void* face_to_elems,
                       const void* face_index, int index_bytes,
                       int32_t* elem_to_faces_out, int32_t* neighbors_out,
                       int32_t* face_index_out);

/* ---- EDFA stage 1 / stage 2 -------------------------------------------- */
/* Exactly one of pattern (base/static sets as a CSR pattern over faces) or
 * dyn must be non-NULL (precond.py:217-218). */
int edfa_stage1_build(edfa_ctx* ctx, const edfa_system* sys, const edfa_csr* pattern,
                      const edfa_dynamic* dyn, double tau_filt, int filtration,
                      double face_drop_tol, int no_fill, edfa_stage1** out);
int edfa_stage1_info_get(const edfa_stage1* s1, edfa_stage1_info* info);
/* Materialises (lazily) and returns a borrowed handle to one part. */
int edfa_stage1_part(edfa_ctx* ctx, edfa_stage1* s1, int part, const edfa_csr** out);
int edfa_stage1_destroy(edfa_stage1* s1);

int edfa_stage2_build(edfa_ctx* ctx, const edfa_csr* A_cc, const edfa_stage1* s1,
                      double tau_filt, int filtration, double schur_drop_tol,
                      int no_fill, edfa_stage2** out);
int edfa_stage2_info_get(const edfa_stage2* s2, edfa_stage2_info* info);
int edfa_stage2_part(edfa_ctx* ctx, edfa_stage2* s2, int part, const edfa_csr** out);
int edfa_stage2_destroy(edfa_stage2* s2);

/* ---- application and products (device vectors) ------------------------ */
/* y = P^-1 r, block-triangular factored inverse; s2 == NULL -> EDFA_ERR_STATE. */
int edfa_precond_apply(edfa_ctx* ctx, const edfa_system* sys, const edfa_stage1* s1,
                       const edfa_stage2* s2, const double* r, double* y);
/* which = 0: face inner (L L^T)^-1 of -A_ff;  which = 1: Schur inner (L U)^-1. */
int edfa_inner_apply(edfa_ctx* ctx, const edfa_stage1* s1, const edfa_stage2* s2,
                     int which, const double* r, double* y);
/* y = alpha * A x + beta * y */
int edfa_spmv(edfa_ctx* ctx, const edfa_csr* A, const double* x, double* y,
              double alpha, double beta);
int edfa_system_spmv(edfa_ctx* ctx, const edfa_system* sys, const double* x, double* y);

/* ---- single-row kernels (precond.py:70-135), results on the host --------- */
/* x (length |idx|) solving -A_ff[idx,idx] x = rhs[idx]; rhs_idx/rhs_val sparse. */
int edfa_restricted_solve(edfa_ctx* ctx, const edfa_csr* A_ff, int32_t n_rhs,
                          const int32_t* rhs_idx, const double* rhs_val, int32_t n_idx,
                          const int32_t* idx, double* x_out);
/* Grow one set from the rhs pattern; idx_out (cap entries) and x_out receive
 * the final set / solution, *n_out its size. */
int edfa_grow_dynamic(edfa_ctx* ctx, const edfa_csr* A_ff, int32_t n_rhs,
                      const int32_t* rhs_idx, const double* rhs_val,
                      const edfa_dynamic* dyn, int32_t cap, int32_t* idx_out,
                      double* x_out, int32_t* n_out);

/* ---- Krylov solves (device vectors b, x; host history buffer) ------------ */
/* Right-preconditioned restarted GMRES(restart), x0 = 0, stop on the true
 * residual ||b - A x|| / ||b|| <= rtol.  s1/s2 NULL -> unpreconditioned. */
int edfa_gmres(edfa_ctx* ctx, const edfa_system* sys, const edfa_stage1* s1,
               const edfa_stage2* s2, const double* b, double* x, double rtol,
               int32_t restart, int32_t max_it, edfa_report* rep, double* hist,
               int32_t hist_cap);
/* Right-preconditioned Bi-CGStab exactly as krylov.bicgstab (krylov.py:40-115). */
int edfa_bicgstab(edfa_ctx* ctx, const edfa_system* sys, const edfa_stage1* s1,
                  const edfa_stage2* s2, const double* b, double* x, double rtol,
                  int32_t max_it, edfa_report* rep, double* hist, int32_t hist_cap);

/* ---- BLAS-1 helpers on device vectors (generic-callable Krylov paths) --- */
int edfa_dot(edfa_ctx* ctx, int64_t n, const double* x, const double* y, double* out_host);
int edfa_axpby(edfa_ctx* ctx, int64_t n, double a, const double* x, double b, double* y);

/* ---- z-slab (multi-GPU) building blocks, SURVEY.md §8(e) ------------------
 * A rank computes stage-1 rows on its extended subsystem and keeps
 * block-Jacobi inner factors of its own rows; parallel.py orchestrates. */
/* out = A[rows, :] with column j kept as col_map[j] when col_map[j] >= 0
 * (col_map must be increasing on the kept columns; device arrays). */
int edfa_csr_submatrix(edfa_ctx* ctx, const edfa_csr* A, int32_t n_rows, const int32_t* rows,
                       const int32_t* col_map, int32_t n_cols, edfa_csr** out);
/* filter_rows (hx/precond.py:138-157): out = A with the off-diagonal (or, with
 * keep_diagonal = 0, all) entries |v| < tau * ||row||_2 and exact zeros
 * dropped; A canonical, tau > 0. */
int edfa_csr_filter(edfa_ctx* ctx, const edfa_csr* A, double tau, int keep_diagonal, edfa_csr** out);
/* out = canonical(A - B) with the optional row filter (S~ = A_cc - H~,
 * hx/precond.py:264-271; filter_rows 138-157 when tau > 0). */
int edfa_csr_sub(edfa_ctx* ctx, const edfa_csr* A, const edfa_csr* B, double tau, edfa_csr** out);
/* IC(0) of -A (ic_factorize(-A_ff, no_fill=True), hx/sparse.py:217-282). */
int edfa_factor_ic0(edfa_ctx* ctx, const edfa_csr* A, double drop_tol, edfa_factor** out);
/* ILU(0) of S (ilu_factorize(S, no_fill=True), hx/sparse.py:141-214); nx*ny*nz
 * = n_rows enables the tile-DAG solves (cells in natural order), else 0s. */
int edfa_factor_ilu0(edfa_ctx* ctx, const edfa_csr* S, double drop_tol, int32_t nx, int32_t ny,
                     int32_t nz, edfa_factor** out);
/* General forms: ic_factorize(-A, drop_tol, no_fill) / ilu_factorize(S,
 * drop_tol, no_fill) (hx/sparse.py:141-282) -- no_fill = 0 admits fill-in
 * (threshold factorisations); rows outgrowing the working table ->
 * EDFA_ERR_UNSUPPORTED. */
int edfa_factor_ic(edfa_ctx* ctx, const edfa_csr* A, double drop_tol, int no_fill, edfa_factor** out);
int edfa_factor_ilu(edfa_ctx* ctx, const edfa_csr* S, double drop_tol, int no_fill, int32_t nx, int32_t ny,
                    int32_t nz, edfa_factor** out);
/* InnerFactorization.nnz_stored (hx/sparse.py:118-123), pivot shifts, levels. */
int edfa_factor_info(const edfa_factor* f, int64_t* nnz_stored, int32_t* pivot_shifts,
                     int32_t* levels_fwd, int32_t* levels_bwd);
/* which = 0: L, 1: U (ILU only); borrowed handle. */
int edfa_factor_part(edfa_ctx* ctx, edfa_factor* f, int which, const edfa_csr** out);
/* y = alpha * (L L^T)^-1 r  or  alpha * (L U)^-1 r   (InnerFactorization.apply,
 * hx/sparse.py:125-129). */
int edfa_factor_solve(edfa_ctx* ctx, const edfa_factor* f, const double* r, double alpha, double* y);
int edfa_factor_destroy(edfa_factor* f);
/* One DCGS2 Arnoldi step of a slab-distributed GMRES (the building blocks of
 * edfa_gmres, for vectors whose dot products are summed across slabs/GPUs
 * between the calls).  V holds q_0..q_{j-1}, u_j, w = A P u_j in rows
 * 0..j+1 (leading dimension ldv >= n).
 *   edfa_dcgs2_dots:   dots_dev[0..j] = [Q_j u_j]^T u_j, dots_dev[64..64+j] =
 *                      [Q_j u_j]^T w (local sums, 128 doubles, unused slots 0)
 *   edfa_dcgs2_coeffs: from the globally summed dots: Hessenberg column j-1
 *                      into H_dev ((m+1) x m, column-major) and hcol_dev,
 *                      first-pass coefficients h1_dev (64), update weights
 *                      coef_dev (192)
 *   edfa_dcgs2_update: row j <- q_j, row j+1 <- u_{j+1} (local) */
int edfa_dcgs2_dots(edfa_ctx* ctx, int64_t n, int32_t j, const double* V, int64_t ldv,
                    double* dots_dev);
int edfa_dcgs2_coeffs(edfa_ctx* ctx, int32_t j, int32_t m, const double* dots_dev,
                      double* H_dev, double* h1_dev, double* coef_dev, double* hcol_dev);
int edfa_dcgs2_update(edfa_ctx* ctx, int64_t n, int32_t j, double* V, int64_t ldv,
                      const double* coef_dev);

/* Gram-Schmidt passes on device vectors (GMRES on distributed vectors):
 * out_dev[k] = V_k . w (k < nvec <= 64, V_k = V + k*ldv);
 * out = w_in - hscale * sum_k h_dev[k] V_k (out = hscale * V h when w_in is NULL),
 * norm2_dev[0] = ||out||^2 when norm2_dev is not NULL. */
int edfa_multidot(edfa_ctx* ctx, int64_t n, int32_t nvec, const double* V, int64_t ldv,
                  const double* w, double* out_dev);
int edfa_multiaxpy(edfa_ctx* ctx, int64_t n, int32_t nvec, const double* V, int64_t ldv,
                   const double* h_dev, double hscale, const double* w_in, double* out,
                   double* norm2_dev);
/* out[i] = x[idx[i]]  (halo send buffers). */
/* y[rows[r]] = (A x)[r] for r < rows of A: the halo-dependent (boundary) rows of
 * a slab's SpMV, computed after the halo exchange that the interior rows overlap. */
int edfa_spmv_rows(edfa_ctx* ctx, const edfa_csr* A, const int32_t* rows, const double* x, double* y);
int edfa_gather(edfa_ctx* ctx, int64_t n, const int32_t* idx, const double* x, double* out);

/* ---- RT0 MHFE / FV assembly --------------------------
 * Device arrays of a hexahedral grid in hexflow's numbering (hx/grid.py:22-65):
 * cells x-fastest, faces grouped by family and k-slowest, local slots
 * (-x,+x,-y,+y,-z,+z), face_to_elems[f][0] = owner (lower-indexed cell). */
typedef struct edfa_hex_grid {
    int32_t n_cells, n_faces, n_nodes;
    const double*  node_coords;      /* [n_nodes][3]                          */
    const int32_t* elem_to_nodes;    /* [n_cells][8], hx/refelem.py:13-16     */
    const int32_t* elem_to_faces;    /* [n_cells][6]                          */
    const int32_t* face_to_elems;    /* [n_faces][2], -1 on the hull          */
    const int32_t* face_local;       /* [n_faces][2], -1 on the hull          */
    const double*  face_area;        /* [n_faces]                             */
} edfa_hex_grid;

typedef struct edfa_assembly_in {
    const double* K;                 /* [n_cells][3][3] conductivity tensors   */
    double gamma;                    /* FluidRockProps.gamma                   */
    const int8_t* face_bc;           /* [n_faces] 0 none, 1 pressure, 2 flux   */
    const double* face_value;        /* [n_faces] prescribed pressure / flux   */
    const double* source;            /* [n_cells] or NULL (zero source)        */
    const double* storage;           /* [n_cells] storage coefficient or NULL  */
    double storage_scalar;           /* used when storage is NULL              */
} edfa_assembly_in;

typedef struct edfa_assembly_out {   /* caller-allocated device arrays         */
    int32_t* face_index;             /* [n_faces] free numbering, -1 = Dirichlet */
    double*  rhs_f;                  /* [n_faces] capacity; first n_free used  */
    double*  rhs_c_base;             /* [n_cells]                              */
    double*  elem_volume;            /* [n_cells] 2x2x2 Gauss volumes          */
    double*  accumulation;           /* [n_cells] volume * storage             */
    double*  binv;                   /* [36][n_cells] Binv (SoA) or NULL       */
    double*  row_sums;               /* [6][n_cells] or NULL                   */
    double*  diag;                   /* [6][n_cells] or NULL                   */
    int32_t  n_free;                 /* out: number of free faces              */
    int32_t  bad_element;            /* out: first inverted element or -1      */
} edfa_assembly_out;

/* Steady blocks A_ff, A_fc, A_cf, A_cc_steady (canonical CSR, free faces
 * first) and rhs of assemble(..., dt=inf).  An inverted element or a
 * non-SPD elemental matrix -> EDFA_ERR_VALUE (GeometryError/AssemblyError). */
int edfa_assemble(edfa_ctx* ctx, const edfa_hex_grid* grid, const edfa_assembly_in* in,
                  edfa_assembly_out* out, edfa_csr** A_ff, edfa_csr** A_fc, edfa_csr** A_cf,
                  edfa_csr** A_cc_steady);
/* After the solve (hx/assembly.py:334-356): per-face fluxes q_out[n_faces],
 * positive out of the owner -- strong two-sided flux on interior faces, the
 * owner's one-sided flux on the hull.  face_value holds the prescribed
 * pressures of Dirichlet faces (face_index < 0); binv/row_sums/diag as
 * written by edfa_assemble. */
int edfa_face_fluxes(edfa_ctx* ctx, const edfa_hex_grid* grid, const int32_t* face_index,
                     const double* face_value, const double* binv, const double* row_sums,
                     const double* diag, const double* pi_reduced, const double* p, double* q_out);
/* cfl (hx/driver.py:67-71): chi_out[e] = outflow rate * dt / (volume * porosity)
 * (chi_out may be NULL); max_out (HOST, 2 doubles) = [max chi, max |p_new - p_old|]
 * (the step controller's dp_max, hx/driver.py:215; p_new/p_old may be NULL). */
int edfa_cfl(edfa_ctx* ctx, const edfa_hex_grid* grid, const double* q, const double* elem_volume,
             const double* porosity, double porosity_scalar, double dt, const double* p_new,
             const double* p_old, double* chi_out, double* max_out);
/* A_cc = canonical(A_cc_steady + diag(acc/dt)), rhs_c = rhs_c_base + acc*p_prev/dt
 * (p_prev NULL = zeros; dt = +inf returns the steady pair). */
int edfa_update_accumulation(edfa_ctx* ctx, const edfa_csr* A_cc_steady, const double* accumulation,
                             const double* rhs_c_base, const double* p_prev, double dt,
                             edfa_csr** A_cc, double* rhs_c);

#ifdef __cplusplus
}
#endif
#endif /* EDFA_H */
