// extern "C" entry points of libedfa.so (declared in include/edfa.h).
#include <algorithm>
#include <map>
#include <vector>

#include "dev_util.cuh"
#include "edfa_internal.cuh"
#include "objects.cuh"

using namespace edfa;

namespace {

const Csr& M(const edfa_csr* h) {
    require(h != nullptr, EDFA_ERR_VALUE, "matrix handle is NULL");
    return h->m ? *h->m : h->own;
}

void upload(Ctx* c, void* dst, const void* src, size_t bytes, int mem) {
    if (!bytes) return;
    EDFA_CUDA(cudaMemcpyAsync(dst, src, bytes, mem == EDFA_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                              c->stream));
}
void download(Ctx* c, void* dst, const void* src, size_t bytes, int mem) {
    if (!bytes) return;
    EDFA_CUDA(cudaMemcpyAsync(dst, src, bytes, mem == EDFA_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                              c->stream));
}

// single-row helper matrices for the row-level entry points
void host_row(Ctx* c, int32_t n_cols, const std::vector<int32_t>& idx, const std::vector<double>& val, Csr& out) {
    out.n_rows = 1;
    out.n_cols = n_cols;
    out.nnz = (int64_t)idx.size();
    int32_t ptr[2] = {0, (int32_t)idx.size()};
    out.ptr.reset(c, 2);
    EDFA_CUDA(cudaMemcpyAsync(out.ptr.p, ptr, sizeof ptr, cudaMemcpyHostToDevice, c->stream));
    out.idx.reset(c, idx.size());
    out.val.reset(c, idx.size());
    if (!idx.empty()) {
        EDFA_CUDA(cudaMemcpyAsync(out.idx.p, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice, c->stream));
        EDFA_CUDA(cudaMemcpyAsync(out.val.p, val.data(), val.size() * 8, cudaMemcpyHostToDevice, c->stream));
    }
    EDFA_CUDA(cudaStreamSynchronize(c->stream));   // host vectors go out of scope
}

// sort + unique keeping the LAST value of duplicates (numpy fancy assignment)
void unique_last(int32_t n, const int32_t* idx, const double* val, std::vector<int32_t>& oi, std::vector<double>& ov) {
    std::map<int32_t, double> m;
    for (int32_t k = 0; k < n; ++k) m[idx[k]] = val ? val[k] : 0.0;
    oi.clear();
    ov.clear();
    for (auto& kv : m) { oi.push_back(kv.first); ov.push_back(kv.second); }
}

}  // namespace

extern "C" {

// ---------------------------------------------------------------- matrices
int edfa_csr_create(edfa_ctx* ctx, int32_t n_rows, int32_t n_cols, int64_t nnz, const int32_t* indptr,
                    const int32_t* indices, const double* data, int mem, edfa_csr** out) {
    API_BEGIN
    require(ctx && out, EDFA_ERR_VALUE, "NULL argument");
    require(n_rows >= 0 && n_cols >= 0 && nnz >= 0, EDFA_ERR_VALUE, "negative matrix size");
    require(nnz <= INT32_MAX, EDFA_ERR_UNSUPPORTED, "more than 2^31-1 stored entries");
    Ctx* c = &ctx->c;
    auto* h = new edfa_csr();
    h->ctx = c;
    Csr& A = h->own;
    A.n_rows = n_rows;
    A.n_cols = n_cols;
    A.nnz = nnz;
    A.ptr.reset(c, (size_t)n_rows + 1);
    upload(c, A.ptr.p, indptr, sizeof(int32_t) * (n_rows + 1), mem);
    A.idx.reset(c, nnz);
    upload(c, A.idx.p, indices, sizeof(int32_t) * nnz, mem);
    if (data) {
        A.val.reset(c, nnz);
        upload(c, A.val.p, data, sizeof(double) * nnz, mem);
    }
    if (mem == EDFA_MEM_HOST) EDFA_CUDA(cudaStreamSynchronize(c->stream));   // pageable sources
    *out = h;
    API_END
}

int edfa_csr_info(const edfa_csr* A, int32_t* n_rows, int32_t* n_cols, int64_t* nnz) {
    API_BEGIN
    const Csr& m = M(A);
    if (n_rows) *n_rows = m.n_rows;
    if (n_cols) *n_cols = m.n_cols;
    if (nnz) *nnz = m.nnz;
    API_END
}

int edfa_csr_export(edfa_ctx* ctx, const edfa_csr* A, int32_t* indptr, int32_t* indices, double* data, int mem) {
    API_BEGIN
    Ctx* c = &ctx->c;
    const Csr& m = M(A);
    if (indptr) download(c, indptr, m.ptr.p, sizeof(int32_t) * (m.n_rows + 1), mem);
    if (indices) download(c, indices, m.idx.p, sizeof(int32_t) * m.nnz, mem);
    if (data) {
        require(m.val.p != nullptr || m.nnz == 0, EDFA_ERR_VALUE, "matrix has no values (pattern only)");
        download(c, data, m.val.p, sizeof(double) * m.nnz, mem);
    }
    if (mem == EDFA_MEM_HOST) EDFA_CUDA(cudaStreamSynchronize(c->stream));
    API_END
}

int edfa_csr_destroy(edfa_csr* A) {
    API_BEGIN
    delete A;
    API_END
}

// ---------------------------------------------------------------- system
int edfa_system_create(edfa_ctx* ctx, const edfa_csr* A_ff, const edfa_csr* A_fc, const edfa_csr* A_cf,
                       const edfa_csr* A_cc, edfa_system** out) {
    API_BEGIN
    Ctx* c = &ctx->c;
    auto* s = new edfa_system();
    try {
        s->ctx = c;
        s->A_ff = &M(A_ff);
        s->A_fc = &M(A_fc);
        s->A_cf = &M(A_cf);
        s->A_cc = &M(A_cc);
        require(s->A_ff->n_rows == s->A_ff->n_cols, EDFA_ERR_VALUE, "A_ff must be square");
        require(s->A_cc->n_rows == s->A_cc->n_cols, EDFA_ERR_VALUE, "A_cc must be square");
        block_merge(c, *s->A_ff, *s->A_fc, *s->A_cf, *s->A_cc, s->A);
        build_sell(c, s->A, s->sA);
        build_sell(c, *s->A_cf, s->sAcf);
        build_sell(c, *s->A_fc, s->sAfc);
    } catch (...) {
        delete s;
        throw;
    }
    *out = s;
    API_END
}

int edfa_system_set_cc(edfa_ctx* ctx, edfa_system* sys, const edfa_csr* A_cc) {
    API_BEGIN
    Ctx* c = &ctx->c;
    const Csr& cc = M(A_cc);
    require(cc.n_rows == sys->A_cc->n_rows && cc.n_cols == sys->A_cc->n_cols, EDFA_ERR_VALUE, "A_cc shape changed");
    sys->A_cc = &cc;
    block_merge(c, *sys->A_ff, *sys->A_fc, *sys->A_cf, *sys->A_cc, sys->A);
    build_sell(c, sys->A, sys->sA);
    API_END
}

int edfa_system_set_grid(edfa_system* sys, int32_t nx, int32_t ny, int32_t nz) {
    API_BEGIN
    require(sys != nullptr, EDFA_ERR_VALUE, "system is NULL");
    require(nx >= 0 && ny >= 0 && nz >= 0, EDFA_ERR_VALUE, "negative grid dimensions");
    sys->dims[0] = nx;
    sys->dims[1] = ny;
    sys->dims[2] = nz;
    API_END
}

int edfa_system_destroy(edfa_system* sys) {
    API_BEGIN
    delete sys;
    API_END
}

// ---------------------------------------------------------------- patterns
int edfa_pattern_static(edfa_ctx* ctx, int32_t n_cells, int32_t n_faces, const int32_t* elem_to_faces,
                        const int32_t* neighbors, const int32_t* face_index, char prototype, int mem,
                        edfa_csr** out) {
    API_BEGIN
    Ctx* c = &ctx->c;
    require(n_cells >= 0 && n_faces >= 0, EDFA_ERR_VALUE, "negative sizes");
    DevBuf<int32_t> e2f, nbr, fidx;
    const int32_t *pe2f = elem_to_faces, *pnbr = neighbors, *pfidx = face_index;
    int32_t n_free = 0;
    if (mem == EDFA_MEM_HOST) {
        e2f.reset(c, (size_t)n_cells * 6);
        nbr.reset(c, (size_t)n_cells * 6);
        fidx.reset(c, std::max(n_faces, 1));
        upload(c, e2f.p, elem_to_faces, sizeof(int32_t) * 6 * n_cells, mem);
        upload(c, nbr.p, neighbors, sizeof(int32_t) * 6 * n_cells, mem);
        upload(c, fidx.p, face_index, sizeof(int32_t) * n_faces, mem);
        pe2f = e2f.p;
        pnbr = nbr.p;
        pfidx = fidx.p;
        for (int32_t k = 0; k < n_faces; ++k) n_free = std::max(n_free, face_index[k] + 1);
    } else {
        n_free = max_value_plus_one(c, face_index, n_faces);   // device reduction, 4-byte readback
    }
    auto* h = new edfa_csr();
    h->ctx = c;
    try {
        static_pattern(c, n_cells, n_free, pe2f, pnbr, pfidx, prototype, h->own);
    } catch (...) {
        delete h;
        throw;
    }
    *out = h;
    API_END
}

int edfa_grid_topology(edfa_ctx* ctx, int32_t n_cells, int32_t n_faces, const void* elem_to_faces,
                       const void* face_to_elems, const void* face_index, int index_bytes, int32_t* elem_to_faces_out,
                       int32_t* neighbors_out, int32_t* face_index_out) {
    API_BEGIN
    require(n_cells >= 0 && n_faces >= 0, EDFA_ERR_VALUE, "negative sizes");
    require(!face_index == !face_index_out, EDFA_ERR_VALUE, "face_index and face_index_out go together");
    grid_topology(&ctx->c, n_cells, n_faces, elem_to_faces, face_to_elems, face_index, index_bytes,
                  elem_to_faces_out, neighbors_out, face_index_out);
    API_END
}

// ---------------------------------------------------------------- stage 1 / 2
int edfa_stage1_build(edfa_ctx* ctx, const edfa_system* sys, const edfa_csr* pattern, const edfa_dynamic* dyn,
                      double tau_filt, int filtration, double face_drop_tol, int no_fill, edfa_stage1** out) {
    API_BEGIN
    Ctx* c = &ctx->c;
    auto* s1 = new edfa_stage1();
    s1->ctx = c;
    try {
        stage1_build(c, const_cast<edfa_system*>(sys), pattern ? &M(pattern) : nullptr, dyn, tau_filt, filtration,
                     face_drop_tol, no_fill, s1);
    } catch (...) {
        delete s1;
        throw;
    }
    *out = s1;
    API_END
}

int edfa_stage1_info_get(const edfa_stage1* s1, edfa_stage1_info* info) {
    API_BEGIN
    info->nnz_G = s1->G.nnz;
    info->nnz_FT = s1->FT.nnz;
    info->nnz_H = s1->H.nnz;
    info->nnz_Q = s1->Q.nnz;
    info->nnz_L = s1->ic.Lpat.nnz + s1->ic.n;
    info->max_pattern = s1->max_pattern;
    info->pivot_shifts = s1->ic.shifts;
    info->trsv_levels = std::max(s1->ic.fwd.n_levels, s1->ic.bwd.n_levels);
    API_END
}

int edfa_stage1_part(edfa_ctx* ctx, edfa_stage1* s1, int part, const edfa_csr** out) {
    API_BEGIN
    Ctx* c = &ctx->c;
    const Csr* m = nullptr;
    switch (part) {
        case EDFA_S1_G: m = &s1->G; break;
        case EDFA_S1_FT: m = &s1->FT; break;
        case EDFA_S1_H: m = &s1->H; break;
        case EDFA_S1_Q: m = &s1->Q; break;
        case EDFA_S1_L: ic_export(c, s1->ic); m = &s1->ic.export_L; break;
        case EDFA_S1_F: m = &s1->F; break;
        default: throw Error(EDFA_ERR_VALUE, "unknown stage-1 part");
    }
    s1->views[part].ctx = c;
    s1->views[part].m = m;
    *out = &s1->views[part];
    API_END
}

int edfa_stage1_destroy(edfa_stage1* s1) {
    API_BEGIN
    delete s1;
    API_END
}

int edfa_stage2_build(edfa_ctx* ctx, const edfa_csr* A_cc, const edfa_stage1* s1, double tau_filt, int filtration,
                      double schur_drop_tol, int no_fill, edfa_stage2** out) {
    API_BEGIN
    Ctx* c = &ctx->c;
    require(s1 != nullptr, EDFA_ERR_STATE, "stage 1 has not been built");
    auto* s2 = new edfa_stage2();
    s2->ctx = c;
    try {
        stage2_build(c, M(A_cc), s1, tau_filt, filtration, schur_drop_tol, no_fill, s2);
    } catch (...) {
        delete s2;
        throw;
    }
    *out = s2;
    API_END
}

int edfa_stage2_info_get(const edfa_stage2* s2, edfa_stage2_info* info) {
    API_BEGIN
    int64_t n = s2->ilu.n;
    int64_t lower = s2->ilu.fwd.n_dep, upper = s2->ilu.bwd.n_dep;
    info->nnz_S = s2->S.nnz;
    info->nnz_L = lower + n;
    info->nnz_U = upper + n;
    info->pivot_shifts = s2->ilu.shifts;
    info->levels_L = s2->ilu.fwd.n_levels;
    info->levels_U = s2->ilu.bwd.n_levels;
    API_END
}

int edfa_stage2_part(edfa_ctx* ctx, edfa_stage2* s2, int part, const edfa_csr** out) {
    API_BEGIN
    Ctx* c = &ctx->c;
    const Csr* m = nullptr;
    switch (part) {
        case EDFA_S2_S: m = &s2->S; break;
        case EDFA_S2_L: ilu_export(c, s2->ilu); m = &s2->ilu.export_L; break;
        case EDFA_S2_U: ilu_export(c, s2->ilu); m = &s2->ilu.export_U; break;
        default: throw Error(EDFA_ERR_VALUE, "unknown stage-2 part");
    }
    s2->views[part].ctx = c;
    s2->views[part].m = m;
    *out = &s2->views[part];
    API_END
}

int edfa_stage2_destroy(edfa_stage2* s2) {
    API_BEGIN
    delete s2;
    API_END
}

// ---------------------------------------------------------------- apply / products
int edfa_precond_apply(edfa_ctx* ctx, const edfa_system* sys, const edfa_stage1* s1, const edfa_stage2* s2,
                       const double* r, double* y) {
    API_BEGIN
    require(s1 != nullptr, EDFA_ERR_STATE, "stage 1 has not been built");
    require(s2 != nullptr, EDFA_ERR_STATE, "stage 2 has not been built; call refresh()");
    ctx->c.trsv_err_poll();
    apply_entry(&ctx->c, sys, s1, s2, r, y);
    ctx->c.trsv_err_post();
    API_END
}

int edfa_inner_apply(edfa_ctx* ctx, const edfa_stage1* s1, const edfa_stage2* s2, int which, const double* r,
                     double* y) {
    API_BEGIN
    require(which == 0 ? s1 != nullptr : s2 != nullptr, EDFA_ERR_STATE, "factorisation not built");
    ctx->c.trsv_err_poll();
    inner_apply(&ctx->c, s1, s2, which, r, y);
    ctx->c.trsv_err_post();
    API_END
}

int edfa_spmv(edfa_ctx* ctx, const edfa_csr* A, const double* x, double* y, double alpha, double beta) {
    API_BEGIN
    const Csr& m = M(A);
    spmv(&ctx->c, view(m), m.nnz, x, y, alpha, beta, "spmv");
    API_END
}

int edfa_system_spmv(edfa_ctx* ctx, const edfa_system* sys, const double* x, double* y) {
    API_BEGIN
    spmv_sell(&ctx->c, sys->sA, x, y, 1.0, 0.0, "spmv_A");
    API_END
}

// ---------------------------------------------------------------- row-level kernels
int edfa_restricted_solve(edfa_ctx* ctx, const edfa_csr* A_ff, int32_t n_rhs, const int32_t* rhs_idx,
                          const double* rhs_val, int32_t n_idx, const int32_t* idx, double* x_out) {
    API_BEGIN
    Ctx* c = &ctx->c;
    const Csr& A = M(A_ff);
    std::vector<int32_t> ri, qi;
    std::vector<double> rv, qv;
    unique_last(n_rhs, rhs_idx, rhs_val, ri, rv);
    unique_last(n_idx, idx, nullptr, qi, qv);
    require((int32_t)qi.size() == n_idx, EDFA_ERR_VALUE, "idx must be unique");
    for (auto v : qi) require(v >= 0 && v < A.n_rows, EDFA_ERR_VALUE, "row index out of range");
    // rhs entries outside idx are dropped (hx/precond.py:88-92)
    Csr acf, afct, pat;
    host_row(c, A.n_cols, ri, rv, acf);
    host_row(c, A.n_cols, {}, {}, afct);
    host_row(c, A.n_cols, qi, qv, pat);
    SetupInput in;
    in.A = &A;
    in.Acf = &acf;
    in.AfcT = &afct;
    in.pattern = &pat;
    SetupOutput out;
    setup_rows(c, in, out);
    if (n_idx) download(c, x_out, out.g.p, sizeof(double) * n_idx, EDFA_MEM_HOST);
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
    API_END
}

int edfa_grow_dynamic(edfa_ctx* ctx, const edfa_csr* A_ff, int32_t n_rhs, const int32_t* rhs_idx,
                      const double* rhs_val, const edfa_dynamic* dyn, int32_t cap, int32_t* idx_out, double* x_out,
                      int32_t* n_out) {
    API_BEGIN
    Ctx* c = &ctx->c;
    const Csr& A = M(A_ff);
    require(dyn && dyn->n_add >= 1 && dyn->n_ent >= 0, EDFA_ERR_VALUE, "invalid dynamic configuration");
    std::vector<int32_t> ri;
    std::vector<double> rv;
    unique_last(n_rhs, rhs_idx, rhs_val, ri, rv);
    for (auto v : ri) require(v >= 0 && v < A.n_rows, EDFA_ERR_VALUE, "row index out of range");
    Csr acf, afct, AT;
    host_row(c, A.n_cols, ri, rv, acf);
    host_row(c, A.n_cols, {}, {}, afct);
    transpose(c, A, AT);
    SetupInput in;
    in.A = &A;
    in.AT = &AT;
    in.Acf = &acf;
    in.AfcT = &afct;
    in.n_add = dyn->n_add;
    in.n_ent = dyn->n_ent;
    in.sweep_limit = dyn->it_max > 0 ? dyn->it_max : std::max(dyn->n_ent, 1);
    SetupOutput out;
    setup_rows(c, in, out);
    int32_t s = 0;
    download(c, &s, out.qsize.p, sizeof(int32_t), EDFA_MEM_HOST);
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
    require(s <= cap, EDFA_ERR_VALUE, "output capacity too small");
    download(c, idx_out, out.q.p, sizeof(int32_t) * s, EDFA_MEM_HOST);
    download(c, x_out, out.g.p, sizeof(double) * s, EDFA_MEM_HOST);
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
    *n_out = s;
    API_END
}

// ---------------------------------------------------------------- Krylov
int edfa_gmres(edfa_ctx* ctx, const edfa_system* sys, const edfa_stage1* s1, const edfa_stage2* s2, const double* b,
               double* x, double rtol, int32_t restart, int32_t max_it, edfa_report* rep, double* hist,
               int32_t hist_cap) {
    API_BEGIN
    require((s1 == nullptr) == (s2 == nullptr), EDFA_ERR_STATE, "stage 2 has not been built; call refresh()");
    gmres(&ctx->c, sys, s1, s2, b, x, rtol, restart, max_it, rep, hist, hist_cap);
    API_END
}

int edfa_bicgstab(edfa_ctx* ctx, const edfa_system* sys, const edfa_stage1* s1, const edfa_stage2* s2,
                  const double* b, double* x, double rtol, int32_t max_it, edfa_report* rep, double* hist,
                  int32_t hist_cap) {
    API_BEGIN
    require((s1 == nullptr) == (s2 == nullptr), EDFA_ERR_STATE, "stage 2 has not been built; call refresh()");
    bicgstab(&ctx->c, sys, s1, s2, b, x, rtol, max_it, rep, hist, hist_cap);
    API_END
}

int edfa_dot(edfa_ctx* ctx, int64_t n, const double* x, const double* y, double* out_host) {
    API_BEGIN
    *out_host = dot_entry(&ctx->c, n, x, y);
    API_END
}

int edfa_axpby(edfa_ctx* ctx, int64_t n, double a, const double* x, double b, double* y) {
    API_BEGIN
    axpby_entry(&ctx->c, n, a, x, b, y);
    API_END
}

// ---------------------------------------------------------------- slab (multi-GPU) building blocks
int edfa_csr_submatrix(edfa_ctx* ctx, const edfa_csr* A, int32_t n_rows, const int32_t* rows, const int32_t* col_map,
                       int32_t n_cols, edfa_csr** out) {
    API_BEGIN
    require(ctx && out && (n_rows == 0 || rows) && col_map, EDFA_ERR_VALUE, "NULL argument");
    require(n_rows >= 0 && n_cols >= 0, EDFA_ERR_VALUE, "negative size");
    auto* h = new edfa_csr();
    h->ctx = &ctx->c;
    try {
        csr_submatrix(&ctx->c, M(A), rows, n_rows, col_map, n_cols, h->own);
    } catch (...) {
        delete h;
        throw;
    }
    *out = h;
    API_END
}

int edfa_csr_filter(edfa_ctx* ctx, const edfa_csr* A, double tau, int keep_diagonal, edfa_csr** out) {
    API_BEGIN
    require(ctx && A && out, EDFA_ERR_VALUE, "NULL argument");
    require(tau > 0.0, EDFA_ERR_VALUE, "tau must be > 0 (tau <= 0 leaves the matrix unchanged)");
    auto* h = new edfa_csr();
    h->ctx = &ctx->c;
    try {
        csr_filter(&ctx->c, M(A), tau, h->own, keep_diagonal != 0);
    } catch (...) {
        delete h;
        throw;
    }
    *out = h;
    API_END
}

int edfa_csr_sub(edfa_ctx* ctx, const edfa_csr* A, const edfa_csr* B, double tau, edfa_csr** out) {
    API_BEGIN
    require(ctx && out, EDFA_ERR_VALUE, "NULL argument");
    require(tau >= 0.0, EDFA_ERR_VALUE, "tau must be >= 0");
    auto* h = new edfa_csr();
    h->ctx = &ctx->c;
    try {
        csr_sub(&ctx->c, M(A), M(B), tau, h->own);
    } catch (...) {
        delete h;
        throw;
    }
    *out = h;
    API_END
}

int edfa_factor_ic0(edfa_ctx* ctx, const edfa_csr* A, double drop_tol, edfa_factor** out) {
    API_BEGIN
    require(ctx && out, EDFA_ERR_VALUE, "NULL argument");
    require(drop_tol >= 0.0, EDFA_ERR_VALUE, "fill_tol must be >= 0");
    const Csr& a = M(A);
    require(a.n_rows == a.n_cols, EDFA_ERR_VALUE, "IC needs a square matrix");
    auto* f = new edfa_factor();
    f->ctx = &ctx->c;
    f->kind = 0;
    try {
        ic0_factor(&ctx->c, a, drop_tol, f->ic);
    } catch (...) {
        delete f;
        throw;
    }
    *out = f;
    API_END
}

int edfa_factor_ilu0(edfa_ctx* ctx, const edfa_csr* S, double drop_tol, int32_t nx, int32_t ny, int32_t nz,
                     edfa_factor** out) {
    API_BEGIN
    require(ctx && out, EDFA_ERR_VALUE, "NULL argument");
    require(drop_tol >= 0.0, EDFA_ERR_VALUE, "fill_tol must be >= 0");
    const Csr& s = M(S);
    require(s.n_rows == s.n_cols, EDFA_ERR_VALUE, "ILU needs a square matrix");
    int dims[3] = {nx, ny, nz};
    const bool grid = nx > 0 && ny > 0 && nz > 0 && (int64_t)nx * ny * nz == s.n_rows;
    auto* f = new edfa_factor();
    f->ctx = &ctx->c;
    f->kind = 1;
    try {
        ilu0_factor(&ctx->c, s, drop_tol, f->ilu, grid ? dims : nullptr);
    } catch (...) {
        delete f;
        throw;
    }
    *out = f;
    API_END
}

int edfa_factor_ic(edfa_ctx* ctx, const edfa_csr* A, double drop_tol, int no_fill, edfa_factor** out) {
    API_BEGIN
    require(ctx && out, EDFA_ERR_VALUE, "NULL argument");
    require(drop_tol >= 0.0, EDFA_ERR_VALUE, "fill_tol must be >= 0");
    const Csr& a = M(A);
    require(a.n_rows == a.n_cols, EDFA_ERR_VALUE, "IC needs a square matrix");
    auto* f = new edfa_factor();
    f->ctx = &ctx->c;
    f->kind = 0;
    try {
        ic0_factor(&ctx->c, a, drop_tol, f->ic, no_fill != 0);
    } catch (...) {
        delete f;
        throw;
    }
    *out = f;
    API_END
}

int edfa_factor_ilu(edfa_ctx* ctx, const edfa_csr* S, double drop_tol, int no_fill, int32_t nx, int32_t ny,
                    int32_t nz, edfa_factor** out) {
    API_BEGIN
    require(ctx && out, EDFA_ERR_VALUE, "NULL argument");
    require(drop_tol >= 0.0, EDFA_ERR_VALUE, "fill_tol must be >= 0");
    const Csr& s = M(S);
    require(s.n_rows == s.n_cols, EDFA_ERR_VALUE, "ILU needs a square matrix");
    int dims[3] = {nx, ny, nz};
    const bool grid = nx > 0 && ny > 0 && nz > 0 && (int64_t)nx * ny * nz == s.n_rows;
    auto* f = new edfa_factor();
    f->ctx = &ctx->c;
    f->kind = 1;
    try {
        ilu0_factor(&ctx->c, s, drop_tol, f->ilu, grid ? dims : nullptr, no_fill != 0);
    } catch (...) {
        delete f;
        throw;
    }
    *out = f;
    API_END
}

int edfa_factor_info(const edfa_factor* f, int64_t* nnz_stored, int32_t* pivot_shifts, int32_t* levels_fwd,
                     int32_t* levels_bwd) {
    API_BEGIN
    require(f != nullptr, EDFA_ERR_VALUE, "factor handle is NULL");
    const TriPlan& fw = f->kind == 0 ? f->ic.fwd : f->ilu.fwd;
    const TriPlan& bw = f->kind == 0 ? f->ic.bwd : f->ilu.bwd;
    // hx/sparse.py:118-123: IC stores 2 nnz(L) - n, ILU nnz(L) - n + nnz(U)
    if (nnz_stored) {
        if (f->kind == 0) *nnz_stored = 2 * (f->ic.Lpat.nnz + f->ic.n) - f->ic.n;
        else *nnz_stored = f->ilu.fwd.n_dep + f->ilu.bwd.n_dep + f->ilu.n;
    }
    if (pivot_shifts) *pivot_shifts = f->kind == 0 ? f->ic.shifts : f->ilu.shifts;
    if (levels_fwd) *levels_fwd = fw.n_levels;
    if (levels_bwd) *levels_bwd = bw.n_levels;
    API_END
}

int edfa_factor_part(edfa_ctx* ctx, edfa_factor* f, int which, const edfa_csr** out) {
    API_BEGIN
    require(ctx && f && out, EDFA_ERR_VALUE, "NULL argument");
    require(which == 0 || (which == 1 && f->kind == 1), EDFA_ERR_VALUE, "unknown factor part");
    Ctx* c = &ctx->c;
    const Csr* m;
    if (f->kind == 0) {
        ic_export(c, f->ic);
        m = &f->ic.export_L;
    } else {
        ilu_export(c, f->ilu);
        m = which == 0 ? &f->ilu.export_L : &f->ilu.export_U;
    }
    f->views[which].ctx = c;
    f->views[which].m = m;
    *out = &f->views[which];
    API_END
}

int edfa_factor_solve(edfa_ctx* ctx, const edfa_factor* f, const double* r, double alpha, double* y) {
    API_BEGIN
    require(ctx && f, EDFA_ERR_VALUE, "NULL argument");
    Ctx* c = &ctx->c;
    c->trsv_err_poll();
    if (f->kind == 0) {
        // chain-structured factor: (L L^T)^-1 in one fused kernel (no shared state: safe for concurrent calls)
        if (!(f->ic.fwd.is_chain && f->ic.bwd.is_chain &&
              run_chain_pair(c, f->ic.fwd.chain, r, alpha, y, nullptr, nullptr, "trsv_ic_pair"))) {
            DevBuf<double> tmp(c, std::max(f->ic.n, 1));
            run_plan(c, f->ic.fwd, r, alpha, tmp.p, nullptr, nullptr, "trsv_ic_L");
            run_plan(c, f->ic.bwd, tmp.p, 1.0, y, nullptr, nullptr, "trsv_ic_LT");
        }
    } else {
        DevBuf<double> tmp(c, std::max(f->ilu.n, 1));
        run_plan(c, f->ilu.fwd, r, alpha, tmp.p, nullptr, nullptr, "trsv_ilu_L");
        run_plan(c, f->ilu.bwd, tmp.p, 1.0, y, nullptr, nullptr, "trsv_ilu_U");
    }
    c->trsv_err_post();
    API_END
}

int edfa_factor_destroy(edfa_factor* f) {
    API_BEGIN
    delete f;
    API_END
}

int edfa_dcgs2_dots(edfa_ctx* ctx, int64_t n, int32_t j, const double* V, int64_t ldv, double* dots_dev) {
    API_BEGIN
    dcgs2_dots_entry(&ctx->c, n, j, V, ldv, dots_dev);
    API_END
}

int edfa_dcgs2_coeffs(edfa_ctx* ctx, int32_t j, int32_t m, const double* dots_dev, double* H_dev, double* h1_dev,
                      double* coef_dev, double* hcol_dev) {
    API_BEGIN
    dcgs2_coeffs_entry(&ctx->c, j, m, dots_dev, H_dev, h1_dev, coef_dev, hcol_dev);
    API_END
}

int edfa_dcgs2_update(edfa_ctx* ctx, int64_t n, int32_t j, double* V, int64_t ldv, const double* coef_dev) {
    API_BEGIN
    dcgs2_update_entry(&ctx->c, n, j, V, ldv, coef_dev);
    API_END
}

int edfa_multidot(edfa_ctx* ctx, int64_t n, int32_t nvec, const double* V, int64_t ldv, const double* w,
                  double* out_dev) {
    API_BEGIN
    multidot_entry(&ctx->c, n, nvec, V, ldv, w, out_dev);
    API_END
}

int edfa_multiaxpy(edfa_ctx* ctx, int64_t n, int32_t nvec, const double* V, int64_t ldv, const double* h_dev,
                   double hscale, const double* w_in, double* out, double* norm2_dev) {
    API_BEGIN
    multiaxpy_entry(&ctx->c, n, nvec, V, ldv, h_dev, hscale, w_in, out, norm2_dev);
    API_END
}

int edfa_spmv_rows(edfa_ctx* ctx, const edfa_csr* A, const int32_t* rows, const double* x, double* y) {
    API_BEGIN
    require(ctx && A, EDFA_ERR_VALUE, "NULL argument");
    spmv_rows(&ctx->c, M(A), rows, x, y);
    API_END
}

int edfa_gather(edfa_ctx* ctx, int64_t n, const int32_t* idx, const double* x, double* out) {
    API_BEGIN
    gather(&ctx->c, n, idx, x, out);
    API_END
}

int edfa_assemble(edfa_ctx* ctx, const edfa_hex_grid* grid, const edfa_assembly_in* in, edfa_assembly_out* out,
                  edfa_csr** A_ff, edfa_csr** A_fc, edfa_csr** A_cf, edfa_csr** A_cc_steady) {
    API_BEGIN
    require(ctx && grid && in && out && A_ff && A_fc && A_cf && A_cc_steady, EDFA_ERR_VALUE, "NULL argument");
    edfa_csr* h[4];
    for (auto& x : h) {
        x = new edfa_csr();
        x->ctx = &ctx->c;
    }
    try {
        assemble(&ctx->c, *grid, *in, *out, h[0]->own, h[1]->own, h[2]->own, h[3]->own);
    } catch (...) {
        for (auto* x : h) delete x;
        throw;
    }
    *A_ff = h[0];
    *A_fc = h[1];
    *A_cf = h[2];
    *A_cc_steady = h[3];
    API_END
}

int edfa_face_fluxes(edfa_ctx* ctx, const edfa_hex_grid* grid, const int32_t* face_index, const double* face_value,
                     const double* binv, const double* row_sums, const double* diag, const double* pi_reduced,
                     const double* p, double* q_out) {
    API_BEGIN
    require(ctx && grid, EDFA_ERR_VALUE, "NULL argument");
    face_fluxes(&ctx->c, *grid, face_index, face_value, binv, row_sums, diag, pi_reduced, p, q_out);
    API_END
}

int edfa_cfl(edfa_ctx* ctx, const edfa_hex_grid* grid, const double* q, const double* elem_volume,
             const double* porosity, double porosity_scalar, double dt, const double* p_new, const double* p_old,
             double* chi_out, double* max_out) {
    API_BEGIN
    require(ctx && grid, EDFA_ERR_VALUE, "NULL argument");
    cfl(&ctx->c, *grid, q, elem_volume, porosity, porosity_scalar, dt, p_new, p_old, chi_out, max_out);
    API_END
}

int edfa_update_accumulation(edfa_ctx* ctx, const edfa_csr* A_cc_steady, const double* accumulation,
                             const double* rhs_c_base, const double* p_prev, double dt, edfa_csr** A_cc,
                             double* rhs_c) {
    API_BEGIN
    require(ctx && A_cc_steady && accumulation && rhs_c_base && A_cc && rhs_c, EDFA_ERR_VALUE, "NULL argument");
    auto* h = new edfa_csr();
    h->ctx = &ctx->c;
    try {
        update_accumulation(&ctx->c, M(A_cc_steady), accumulation, rhs_c_base, p_prev, dt, h->own, rhs_c);
    } catch (...) {
        delete h;
        throw;
    }
    *A_cc = h;
    API_END
}

}  // extern "C"

