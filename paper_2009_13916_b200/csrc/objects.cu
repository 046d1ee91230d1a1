// Orchestration of the two-stage EDFA build (hx/precond.py:204-271) on the
// device: host code here only sequences kernels and reads back sizes.
#include <cub/cub.cuh>

#include "dev_util.cuh"
#include "edfa_internal.cuh"
#include "objects.cuh"

namespace edfa {
namespace {
__global__ void k_row_len_max(const int32_t* __restrict__ ptr, int n, int* __restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    int v = i < n ? ptr[i + 1] - ptr[i] : 0;
    v = warp_max(v);
    if ((threadIdx.x & 31) == 0 && v > 0) atomicMax(out, v);
}
}  // namespace

namespace {
__global__ void k_max_plus_one(const int32_t* __restrict__ v, int n, int* __restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    int x = i < n ? v[i] + 1 : 0;
    x = warp_max(x);
    if ((threadIdx.x & 31) == 0 && x > 0) atomicMax(out, x);
}
}  // namespace

int max_value_plus_one(Ctx* c, const int32_t* v, int n) {
    if (n <= 0) return 0;
    int* d = c->d_scalar_i + 44;
    EDFA_CUDA(cudaMemsetAsync(d, 0, sizeof(int), c->stream));
    k_max_plus_one<<<ceil_div(n, 256), 256, 0, c->stream>>>(v, n, d);
    check_launch("k_max_plus_one");
    int h = 0;
    EDFA_CUDA(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
    return h;
}

int max_row_nnz(Ctx* c, const Csr& A) {
    if (A.n_rows == 0) return 0;
    int* d = c->d_scalar_i + 40;
    EDFA_CUDA(cudaMemsetAsync(d, 0, sizeof(int), c->stream));
    k_row_len_max<<<ceil_div(A.n_rows, 256), 256, 0, c->stream>>>(A.ptr.p, A.n_rows, d);
    check_launch("k_row_len_max");
    int h = 0;
    EDFA_CUDA(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
    return h;
}

void ensure_transposes(Ctx* c, edfa_system* sys, bool need_AffT) {
    if (!sys->AfcT.ptr.p) transpose(c, *sys->A_fc, sys->AfcT);
    if (need_AffT && !sys->AffT.ptr.p) transpose(c, *sys->A_ff, sys->AffT);
}

void stage1_build(Ctx* c, edfa_system* sys, const Csr* pattern, const edfa_dynamic* dyn, double tau, int filt,
                  double face_drop_tol, int no_fill, edfa_stage1* s1) {
    require((pattern == nullptr) != (dyn == nullptr), EDFA_ERR_VALUE, "give exactly one of patterns or dynamic");
    require(filt >= EDFA_FILT_NONE && filt <= EDFA_FILT_POST_PRODUCT, EDFA_ERR_VALUE,
            "filtration must be one of ('none', 'pre', 'post-schur', 'post-product')");
    require(face_drop_tol >= 0.0, EDFA_ERR_VALUE, "fill_tol must be >= 0");
    const Csr& Aff = *sys->A_ff;
    const int nf = Aff.n_rows, nc = sys->A_cf->n_rows;
    if (pattern) {
        require(pattern->n_rows == nc && pattern->n_cols == nf, EDFA_ERR_VALUE,
                "pattern set must have one set per cell over the free faces");
    } else {
        require(dyn->n_add >= 1, EDFA_ERR_VALUE, "n_add must be >= 1");
        require(dyn->n_ent >= 0, EDFA_ERR_VALUE, "n_ent must be >= 0");
    }
    ensure_transposes(c, sys, dyn != nullptr);
    s1->n_free = nf;
    s1->n_cells = nc;
    for (int d = 0; d < 3; ++d) s1->dims[d] = sys->dims[d];
    SetupInput in;
    in.A = &Aff;
    in.AT = dyn ? &sys->AffT : nullptr;
    in.Acf = sys->A_cf;
    in.AfcT = &sys->AfcT;
    in.pattern = pattern;
    if (dyn) {
        in.n_add = dyn->n_add;
        in.n_ent = dyn->n_ent;
        in.sweep_limit = dyn->it_max > 0 ? dyn->it_max : std::max(dyn->n_ent, 1);
    }
    in.pre_tau = filt == EDFA_FILT_PRE ? tau : 0.0;
    SetupOutput out;
    {
        PhaseTimer pt(c, "stage1.setup_rows");
        setup_rows(c, in, out);
    }
    s1->max_pattern = out.max_pattern;
    const int32_t* qsz = dyn ? out.qsize.p : nullptr;
    const int32_t* qidx = dyn ? out.q.p : pattern->idx.p;
    {
        PhaseTimer pt(c, "stage1.compact+transpose");
        compact_rows(c, nc, out.slot_ptr, qsz, qidx, out.g.p, out.gcnt, nf, s1->G);
        compact_rows(c, nc, out.slot_ptr, qsz, qidx, out.f.p, out.fcnt, nf, s1->FT);
        if (dyn) pattern_compact(c, nc, out.slot_ptr, out.qsize, out.q, nf, s1->Q);
        else copy_csr(c, *pattern, s1->Q);
        transpose(c, s1->FT, s1->F);
        s1->have_F = true;
    }
    {
        PhaseTimer pt(c, "stage1.product");
        triple_product(c, s1->G, Aff, s1->F, filt == EDFA_FILT_POST_PRODUCT ? tau : 0.0, s1->H);
    }
    PhaseTimer pt(c, "stage1.ic0");
    ic0_factor(c, Aff, face_drop_tol, s1->ic, no_fill != 0);
}

void stage2_build(Ctx* c, const Csr& A_cc, const edfa_stage1* s1, double tau, int filt, double schur_drop_tol,
                  int no_fill, edfa_stage2* s2) {
    require(filt >= EDFA_FILT_NONE && filt <= EDFA_FILT_POST_PRODUCT, EDFA_ERR_VALUE,
            "filtration must be one of ('none', 'pre', 'post-schur', 'post-product')");
    require(schur_drop_tol >= 0.0, EDFA_ERR_VALUE, "fill_tol must be >= 0");
    {
        PhaseTimer pt(c, "stage2.schur_sub");
        csr_sub(c, A_cc, s1->H, filt == EDFA_FILT_POST_SCHUR ? tau : 0.0, s2->S);
    }
    PhaseTimer pt(c, "stage2.ilu0_total");
    const int* dims = (int64_t)s1->dims[0] * s1->dims[1] * s1->dims[2] == A_cc.n_rows && s1->dims[0] > 0
                          ? s1->dims : nullptr;
    ilu0_factor(c, s2->S, schur_drop_tol, s2->ilu, dims, no_fill != 0);
}

}  // namespace edfa
