// Library objects behind the opaque C handles: system, stage 1, stage 2,
// incomplete factors and their sync-free triangular-solve plans.
#pragma once
#include "edfa_internal.cuh"

namespace edfa {

// ---- stage-1 row kernel I/O (setup_rows.cu)
struct SetupInput {
    const Csr* A = nullptr;        // A_ff
    const Csr* AT = nullptr;       // transpose of A_ff (dynamic), may be NULL -> A
    const Csr* Acf = nullptr;
    const Csr* AfcT = nullptr;     // A_fc^T (cells x faces)
    const Csr* pattern = nullptr;  // static/base sets, NULL -> dynamic
    int32_t n_add = 1, n_ent = 0, sweep_limit = 1;
    double pre_tau = 0.0;
};
struct SetupOutput {
    DevBuf<int32_t> slot_ptr, q, qsize, gcnt, fcnt;
    DevBuf<double> g, f;
    int64_t n_slots = 0;
    int max_pattern = 0;
};
void setup_rows(Ctx* c, const SetupInput& in, SetupOutput& out);
void compact_rows(Ctx* c, int32_t n, const DevBuf<int32_t>& slot_ptr, const int32_t* qsize, const int32_t* qidx,
                  const double* vals, const DevBuf<int32_t>& cnt, int32_t n_cols, Csr& out);
void pattern_compact(Ctx* c, int32_t n, const DevBuf<int32_t>& slot_ptr, const DevBuf<int32_t>& qsize,
                     const DevBuf<int32_t>& q, int32_t n_cols, Csr& out);
void static_pattern(Ctx* c, int32_t n_cells, int32_t n_free, const int32_t* e2f, const int32_t* nbr,
                    const int32_t* fidx, char proto, Csr& out);
void grid_topology(Ctx* c, int32_t n_cells, int32_t n_faces, const void* e2f, const void* f2e, const void* fidx,
                   int index_bytes, int32_t* e2f_out, int32_t* nbr_out, int32_t* fidx_out);
int max_row_nnz(Ctx* c, const Csr& A);
int max_value_plus_one(Ctx* c, const int32_t* v, int n);

// ---- H~ = G~ A_ff F~ (product.cu)
void triple_product(Ctx* c, const Csr& G, const Csr& A, const Csr& F, double post_tau, Csr& H);

// ---- sync-free triangular solve plan (trsv.cu)
// Rows are grouped by dependency level, each level padded to whole warps;
// one thread per row; SELL-32 (column-major inside 32-row slices) so the
// coefficient stream is fully coalesced.  Dependencies are polled on the
// solution vector itself (sentinel-initialised), so there is no flag array.
struct ChainPlan {              // disjoint-path DAGs (chain.cu)
    int32_t n = 0, n_chains = 0, max_len = 0;
    int64_t n_stored = 0;
    bool unit = false;
    DevBuf<int64_t> gbase;      // group of 32 chains -> first stored step
    DevBuf<int32_t> rows;       // SELL-32 over chains: row of step k of chain t
    DevBuf<double> coef, dinv;  // dependency coefficient / inverse diagonal per step
    DevBuf<int32_t> heads, succ;
    int32_t E = 0;              // segment length per lane of the warp solvers (max_len <= 32 E)
    DevBuf<int32_t> crow;       // lane-interleaved: chain t, step k at t*32E + (k%E)*32 + k/E
    DevBuf<double> ccoef, cdinv;
};
int chain_segment(int max_len);   // smallest instantiated E with 32 E >= max_len (0: too long)
bool build_chain(Ctx* c, const Csr& deps, const double* diag, bool unit, ChainPlan& cp);
void chain_values(Ctx* c, const Csr& deps, const double* diag, ChainPlan& cp);
void run_chain(Ctx* c, const ChainPlan& cp, const double* b, double alpha, double* x, const double* add, double* out2,
               const char* name);
// x = (L L^T)^{-1} (alpha b) on the chains of L (out2 = x + add); false when
// the chains are too long for the fused kernel (caller runs the two solves)
// fz (optional): b := fz x (a fused SpMV; rows of fz = rows of the factor), b itself is ignored
bool run_chain_pair(Ctx* c, const ChainPlan& cp, const double* b, double alpha, double* x, const double* add,
                    double* out2, const char* name);
void chain_ic0(Ctx* c, const ChainPlan& cp, const Csr& Lpat, const double* aii, const double* scale, double* diag,
               int* shifts, double fill_tol = 0.0);

struct TilePlan {               // tile-DAG solves of cell-indexed factors (tile.cu)
    int32_t n = 0, n_tiles = 0, n_tile_levels = 0;
    int32_t RC = 0, KD = 0, EC = 0, LC = 0;   // rows / early deps / externals / levels per tile
    int64_t n_dep = 0;
    bool unit = false;
    DevBuf<int32_t> hdr, row_id, ext_id, up_cnt, up_ids, order;   // up_*: tile DAG (schedule order)
    DevBuf<unsigned> ticket;
    DevBuf<short> lev_ptr, dslot, eslot;     // critical / early dependency slots
    DevBuf<double> dcoef, ecoef, dinv;       // critical / early coefficients
    DevBuf<short> xlev_ptr;                  // externals first needed below level l: [0, xlev_ptr[l])
    unsigned ticket_base = 0;                // tickets wrap modulo 2^32
};
// dims = {nx, ny, nz} of the cell grid (rows = cells in natural order) or NULL
bool build_tile_plan(Ctx* c, const Csr& D, const double* diag, bool unit, bool reverse, const int* dims,
                     TilePlan& tp);
void run_tile(Ctx* c, TilePlan& tp, const double* b, double alpha, double* x, const double* add, double* out2,
              const char* name);
// x_prefilled: x already holds SENTINEL; consume_b: b's rows are reset to
// SENTINEL once read; pre_sent: a vector set to SENTINEL row by row (the next
// solve's output) -- lets consecutive solves skip their fill kernels
void run_tile_ex(Ctx* c, TilePlan& tp, const double* b, double alpha, double* x, const double* add, double* out2,
                 const char* name, bool x_prefilled, bool consume_b, double* pre_sent);

struct TriPlan {
    bool is_chain = false;
    ChainPlan chain;
    bool is_tile = false;
    TilePlan tile;
    int32_t n = 0;          // rows
    int32_t n_slots = 0;    // padded thread count (multiple of 32)
    int32_t n_levels = 0;
    int64_t n_dep = 0;      // off-diagonal coefficients (algorithmic)
    int64_t n_stored = 0;   // SELL entries incl. padding
    int32_t max_w = 0;      // widest slice (entries per row); > 16 -> warp-per-row sync-free solve
    bool unit = false;
    DevBuf<int32_t> perm;       // slot -> row (-1 pad)
    DevBuf<int64_t> slice_ptr;  // slice -> first SELL entry
    DevBuf<int32_t> col;
    DevBuf<double> val;
    DevBuf<double> dinv;        // slot -> 1/diag (1 for unit)
    DevBuf<int32_t> slice_level;   // slice -> dependency level
    DevBuf<int32_t> level_slices;  // level -> number of slices
    DevBuf<int32_t> level_start;   // level -> first slice (n_levels + 1)
    // [done[0..n_levels), ticket, finished]; self-resetting at kernel end
    DevBuf<int32_t> sync;
    DevBuf<int32_t> ticket;     // unused (kept for ABI of older plans)
    // wavefront-packed solves (wf.cu): col holds dependency SLOTS, vectors live in slot order
    bool is_wf = false, wf_reverse = false;
    bool wf_shared = false;             // a backward plan on the forward plan's slot layout
    const int32_t* wf_perm = nullptr;   // the shared slot -> row map (the forward plan's perm)
    int32_t wf_slices = 0;
    DevBuf<int32_t> wf_pos;             // row -> slot (forward plan only)
    DevBuf<unsigned> wf_ticket;
    unsigned wf_ticket_base = 0;        // tickets wrap modulo 2^32
};
// deps: row i -> (j, coef) with x_i = (alpha*b_i - sum coef*x_j) * dinv_i;
// reverse = deps point to higher rows (backward substitution).  diag may be
// NULL (values loaded later with plan_values).
// given_level (optional): a layering of the rows computed by the caller (every
// dependency in a strictly earlier layer), given_levels layers
void build_plan(Ctx* c, const Csr& deps, const double* diag, bool unit, bool reverse, TriPlan& plan,
                bool allow_chain = true, const int32_t* given_level = nullptr, int given_levels = 0);
void plan_values(Ctx* c, const Csr& deps, const double* diag, TriPlan& plan);
// SELL-32 storage of deps' rows on a given slot layout (perm: slot -> row, -1 pad)
void sell_on_layout(Ctx* c, const int32_t* perm, int n_slices, const Csr& deps, const double* diag, bool unit,
                    DevBuf<int64_t>& slice_ptr, DevBuf<int32_t>& col, DevBuf<double>& val, DevBuf<double>& dinv,
                    int64_t& n_stored, int32_t& max_w);
// wavefront-packed L / U solves on one slot layout (wf.cu)
bool build_wf_plans(Ctx* c, const Csr& Lv, const Csr& Uv, const double* udiag, TriPlan& fwd, TriPlan& bwd);
void run_wf(Ctx* c, const TriPlan& p, const double* b, bool b_slots, double alpha, double* xs, bool fill_xs,
            double* x_nat, const double* add, double* out2, double* b_sent, double* pre_sent, const char* name);
void run_wf_natural(Ctx* c, const TriPlan& p, const double* b, double alpha, double* x, const double* add,
                    double* out2, const char* name);
// x = solve(b * alpha); if (add) out2 = x + add (fused epilogue)
void run_plan(Ctx* c, const TriPlan& p, const double* b, double alpha, double* x, const double* add, double* out2,
              const char* name);

// ---- incomplete factors (factor.cu)
struct IcFactor {               // IC of -A_ff (no fill)
    int32_t n = 0;
    Csr Lpat;                   // strictly lower part of -A_ff's pattern, values = L
    DevBuf<double> diag;        // L_ii
    int32_t shifts = 0;
    TriPlan fwd, bwd;           // L y = b ; L^T x = y
    Csr export_L;               // materialised on request
};
struct IluFactor {              // ILU of S (no fill)
    int32_t n = 0;
    Csr LU;                     // pattern of S; strict lower = multipliers, strict upper = U
    DevBuf<double> udiag;
    DevBuf<int32_t> has_diag;   // S stores its diagonal (for the exported nnz)
    int32_t shifts = 0;
    TriPlan fwd, bwd;
    Csr export_L, export_U;
};
// IC of -A_ff / ILU of S with the reference's drop tolerance; no_fill = False
// admits fill-in (threshold factorisations, ilut.cu)
void ic0_factor(Ctx* c, const Csr& A_ff, double drop_tol, IcFactor& f, bool no_fill = true);
void ilu0_factor(Ctx* c, const Csr& S, double drop_tol, IluFactor& f, const int* dims, bool no_fill = true);
// threshold kernels (ilut.cu): f.LU / f.Lpat compact, pivots, shifts
void ilut_factor(Ctx* c, const Csr& S, double fill_tol, bool no_fill, IluFactor& f);
void ict_factor(Ctx* c, const Csr& A, double sign, double fill_tol, IcFactor& f);
void drop_zeros(Ctx* c, Csr& A);
void ic_export(Ctx* c, IcFactor& f);
void ilu_export(Ctx* c, IluFactor& f);

}  // namespace edfa

// ---- handle objects
struct edfa_system {
    edfa::Ctx* ctx;
    const edfa::Csr* A_ff;
    const edfa::Csr* A_fc;
    const edfa::Csr* A_cf;
    const edfa::Csr* A_cc;
    edfa::Csr A;            // monolithic operator
    edfa::Sell sA, sAcf, sAfc;   // SELL-32 copies for the SpMVs of the solve
    edfa::Csr AfcT;         // A_fc^T, cells x faces (rows = f-rhs per cell)
    edfa::Csr AffT;         // A_ff^T (columns of A_ff)
    bool have_T = false;
    int dims[3] = {0, 0, 0};   // cell grid (nx, ny, nz) when cells are a natural-order box
};

struct edfa_stage1 {
    edfa::Ctx* ctx;
    edfa::Csr G, FT, H, Q;
    edfa::Csr F;            // faces x cells
    bool have_F = false;
    edfa::IcFactor ic;
    int32_t max_pattern = 0;
    int32_t n_free = 0, n_cells = 0;
    int dims[3] = {0, 0, 0};
    edfa_csr views[6];      // borrowed handles returned by edfa_stage1_part
};

struct edfa_stage2 {
    edfa::Ctx* ctx;
    edfa::Csr S;
    edfa::IluFactor ilu;
    edfa_csr views[3];
};

struct edfa_factor {            // stand-alone IC(0) of -A / ILU(0) of S (slab.cu)
    edfa::Ctx* ctx;
    int kind = 0;               // 0 = IC (factor of -A), 1 = ILU
    edfa::IcFactor ic;
    edfa::IluFactor ilu;
    edfa_csr views[2];
};

namespace edfa {
void stage1_build(Ctx* c, edfa_system* sys, const Csr* pattern, const edfa_dynamic* dyn, double tau, int filt,
                  double face_drop_tol, int no_fill, edfa_stage1* s1);
void stage2_build(Ctx* c, const Csr& A_cc, const edfa_stage1* s1, double tau, int filt, double schur_drop_tol,
                  int no_fill, edfa_stage2* s2);
void ensure_transposes(Ctx* c, edfa_system* sys, bool need_AffT);
void apply_entry(Ctx* c, const edfa_system* sys, const edfa_stage1* s1, const edfa_stage2* s2, const double* r,
                 double* y);
void inner_apply(Ctx* c, const edfa_stage1* s1, const edfa_stage2* s2, int which, const double* r, double* y);
void gmres(Ctx* c, const edfa_system* sys, const edfa_stage1* s1, const edfa_stage2* s2, const double* b, double* x,
           double rtol, int m, int max_it, edfa_report* rep, double* hist, int hist_cap);
void bicgstab(Ctx* c, const edfa_system* sys, const edfa_stage1* s1, const edfa_stage2* s2, const double* b,
              double* x, double rtol, int max_it, edfa_report* rep, double* hist, int hist_cap);
double dot_entry(Ctx* c, int64_t n, const double* x, const double* y);
void multidot_entry(Ctx* c, int64_t n, int nvec, const double* V, int64_t ldv, const double* w, double* out_dev);
void multiaxpy_entry(Ctx* c, int64_t n, int nvec, const double* V, int64_t ldv, const double* h, double hscale,
                     const double* w_in, double* out, double* norm2_dev);
void csr_submatrix(Ctx* c, const Csr& A, const int32_t* rows, int32_t n_out, const int32_t* cmap, int32_t n_cols,
                   Csr& out);
void gather(Ctx* c, int64_t n, const int32_t* idx, const double* x, double* out);
// y[rows[r]] = (A x)[r], A compact (the boundary rows of a slab SpMV)
void spmv_rows(Ctx* c, const Csr& A, const int32_t* rows, const double* x, double* y);
void axpby_entry(Ctx* c, int64_t n, double a, const double* x, double b, double* y);
void dcgs2_dots_entry(Ctx* c, int64_t n, int j, const double* V, int64_t ldv, double* dots_out);
void dcgs2_coeffs_entry(Ctx* c, int j, int m, const double* dots, double* H, double* h1, double* coef, double* hcol);
void dcgs2_update_entry(Ctx* c, int64_t n, int j, double* V, int64_t ldv, const double* coef);
// RT0 MHFE / FV assembly (assembly.cu)
void assemble(Ctx* c, const edfa_hex_grid& g, const edfa_assembly_in& in, edfa_assembly_out& out, Csr& A_ff,
              Csr& A_fc, Csr& A_cf, Csr& A_cc);
void update_accumulation(Ctx* c, const Csr& A_cc_steady, const double* acc, const double* rhs_c_base,
                         const double* p_prev, double dt, Csr& A_cc, double* rhs_c);
void face_fluxes(Ctx* c, const edfa_hex_grid& g, const int32_t* fidx, const double* fval, const double* Bi,
                 const double* rs, const double* dg, const double* pi, const double* p, double* q);
void cfl(Ctx* c, const edfa_hex_grid& g, const double* q, const double* vol, const double* phi, double phi_s,
         double dt, const double* pn, const double* po, double* chi, double* out_host);
}  // namespace edfa
