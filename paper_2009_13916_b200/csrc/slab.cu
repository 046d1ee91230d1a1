// Pieces of the z-slab (multi-GPU) EDFA path, §8(e) of SURVEY.md.
//
// A rank owns a contiguous range of cell layers and the faces those cells own.
// Stage 1 rows are computed on the rank's extended subsystem (slab + halo
// layers); the rank then keeps
//   S~_own = A_cc[own, own] - H~[own, own]     (block-Jacobi Schur block)
//   IC(0) of -A_ff[own, own]                   (block-Jacobi face block)
// so the inner triangular solves never cross a slab boundary.  This file holds
// the generic device operations the host orchestration (parallel.py) needs:
// submatrix extraction, stand-alone IC(0)/ILU(0) factor objects and a gather.
#include <vector>

#include "dev_util.cuh"
#include "edfa_internal.cuh"
#include "objects.cuh"

namespace edfa {
namespace {

// counts[r] = #entries of row rows[r] whose column maps to >= 0
__global__ void k_sub_count(CsrV A, const int32_t* __restrict__ rows, int n_out, const int32_t* __restrict__ cmap,
                            int32_t* __restrict__ cnt) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_out) return;
    int i = rows[r];
    int k = 0;
    for (int e = A.ptr[i]; e < A.ptr[i + 1]; ++e) k += cmap[A.idx[e]] >= 0;
    cnt[r] = k;
}

__global__ void k_sub_fill(CsrV A, const int32_t* __restrict__ rows, int n_out, const int32_t* __restrict__ cmap,
                           const int32_t* __restrict__ ptr, int32_t* __restrict__ idx, double* __restrict__ val,
                           int* __restrict__ err) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_out) return;
    int i = rows[r];
    int o = ptr[r], last = -1;
    for (int e = A.ptr[i]; e < A.ptr[i + 1]; ++e) {
        int j = cmap[A.idx[e]];
        if (j < 0) continue;
        if (j <= last) *err = 1;      // the column map must be increasing on kept columns
        last = j;
        idx[o] = j;
        if (val) val[o] = A.val[e];
        ++o;
    }
}

__global__ void k_gather(int64_t n, const int32_t* __restrict__ idx, const double* __restrict__ x,
                         double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = x[idx[i]];
}

// y[rows[r]] = (A x)[r] for a compact CSR A (boundary rows of a slab's SpMV)
__global__ void k_spmv_rows(CsrV A, const int32_t* __restrict__ rows, const double* __restrict__ x,
                            double* __restrict__ y) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= A.n_rows) return;
    double acc = 0.0;
    for (int e = A.ptr[r]; e < A.ptr[r + 1]; ++e) acc = fma(A.val[e], x[A.idx[e]], acc);
    y[rows[r]] = acc;
}

}  // namespace

void spmv_rows(Ctx* c, const Csr& A, const int32_t* rows, const double* x, double* y) {
    if (A.n_rows <= 0) return;
    Prof pr(c, "spmv_rows", 12.0 * A.nnz + 12.0 * A.n_rows + 8.0 * A.nnz);
    k_spmv_rows<<<ceil_div(A.n_rows, 128), 128, 0, c->stream>>>(view(A), rows, x, y);
    check_launch("k_spmv_rows");
}

void csr_submatrix(Ctx* c, const Csr& A, const int32_t* rows, int32_t n_out, const int32_t* cmap, int32_t n_cols,
                   Csr& out) {
    out.n_rows = n_out;
    out.n_cols = n_cols;
    out.ptr.reset(c, (size_t)n_out + 1);
    DevBuf<int32_t> cnt(c, std::max(n_out, 1));
    if (n_out) {
        Prof pr(c, "submatrix", 12.0 * A.nnz * n_out / std::max(A.n_rows, 1) + 4.0 * n_out);
        k_sub_count<<<ceil_div(n_out, 128), 128, 0, c->stream>>>(view(A), rows, n_out, cmap, cnt.p);
        check_launch("k_sub_count");
    }
    out.nnz = scan_counts(c, cnt.p, out.ptr.p, n_out);
    out.idx.reset(c, out.nnz);
    if (A.val.p) out.val.reset(c, out.nnz);
    else out.val.release();
    if (n_out) {
        int* err = c->d_scalar_i + 48;
        EDFA_CUDA(cudaMemsetAsync(err, 0, sizeof(int), c->stream));
        {
            Prof pr(c, "submatrix", 12.0 * out.nnz + 4.0 * n_out);
            k_sub_fill<<<ceil_div(n_out, 128), 128, 0, c->stream>>>(view(A), rows, n_out, cmap, out.ptr.p,
                                                                   out.idx.p, out.val.p, err);
            check_launch("k_sub_fill");
        }
        int h = 0;
        EDFA_CUDA(cudaMemcpyAsync(&h, err, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        EDFA_CUDA(cudaStreamSynchronize(c->stream));
        require(h == 0, EDFA_ERR_VALUE, "column map must be increasing on the kept columns");
    }
}

void gather(Ctx* c, int64_t n, const int32_t* idx, const double* x, double* out) {
    if (n <= 0) return;
    Prof pr(c, "gather", 20.0 * n);
    int blocks = (int)std::min<int64_t>(ceil_div(n, 256), NUM_SMS_B200 * 4);
    k_gather<<<blocks, 256, 0, c->stream>>>(n, idx, x, out);
    check_launch("k_gather");
}

}  // namespace edfa
