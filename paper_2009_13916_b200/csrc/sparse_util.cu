// Sparse plumbing kernels: scans, transpose, block merge, SpMV, S = A - H,
// row filtration.  All HBM-bound integer/FP64 streaming work.
#include <cub/cub.cuh>

#include "dev_util.cuh"
#include "edfa_internal.cuh"

namespace edfa {

namespace {

__global__ void k_incl_to_ptr(const int64_t* __restrict__ incl, int32_t* __restrict__ ptr, int32_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i == 0) ptr[0] = 0;
    if (i < n) ptr[i + 1] = (int32_t)incl[i];
}

struct ToI64 {
    __host__ __device__ int64_t operator()(int32_t v) const { return (int64_t)v; }
};

__global__ void k_fill(double* p, int64_t n, double v) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void k_fill_bits(unsigned long long* p, int64_t n, unsigned long long v) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

// G lanes per row (chosen from the mean row length: short rows keep their lanes busy)
template <int G>
__global__ void k_row_of(const int32_t* __restrict__ ptr, int32_t n, int32_t* __restrict__ row_of) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int w = (int)(t / G), lane = (int)(t % G);
    if (w >= n) return;
    for (int e = ptr[w] + lane; e < ptr[w + 1]; e += G) row_of[e] = w;
}
__global__ void k_iota(int32_t* p, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = (int32_t)i;
}
__global__ void k_col_hist(const int32_t* __restrict__ idx, int64_t nnz, int32_t* __restrict__ cnt) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < nnz) atomicAdd(&cnt[idx[i]], 1);
}
__global__ void k_gather_T(const int32_t* __restrict__ order, const int32_t* __restrict__ row_of,
                           const double* __restrict__ val, int64_t nnz, int32_t* __restrict__ out_idx,
                           double* __restrict__ out_val) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= nnz) return;
    int32_t e = order[p];
    out_idx[p] = row_of[e];
    if (val) out_val[p] = val[e];
}

__global__ void k_merge_ptr(const int32_t* A, const int32_t* B, const int32_t* C, const int32_t* D, int32_t nA,
                            int32_t nC, int32_t* M) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i <= nA) M[i] = A[i] + B[i];
    else if (i <= nA + nC) {
        int k = (int)(i - nA);
        M[i] = A[nA] + B[nA] + C[k] + D[k];
    }
}
template <int G>   // lanes per row
__global__ void k_merge_fill(CsrV A, CsrV B, CsrV C, CsrV D, const int32_t* __restrict__ Mp,
                             int32_t* __restrict__ Mi, double* __restrict__ Mv) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int w = (int)(t / G), lane = (int)(t % G);
    int n = A.n_rows + C.n_rows;
    if (w >= n) return;
    const CsrV& L = w < A.n_rows ? A : C;
    const CsrV& R = w < A.n_rows ? B : D;
    int r = w < A.n_rows ? w : w - A.n_rows;
    int off = A.n_cols;
    int o = Mp[w];
    int l0 = L.ptr[r], l1 = L.ptr[r + 1], r0 = R.ptr[r], r1 = R.ptr[r + 1];
    for (int e = l0 + lane; e < l1; e += G) {
        Mi[o + e - l0] = L.idx[e];
        Mv[o + e - l0] = L.val[e];
    }
    o += l1 - l0;
    for (int e = r0 + lane; e < r1; e += G) {
        Mi[o + e - r0] = R.idx[e] + off;
        Mv[o + e - r0] = R.val[e];
    }
}

// vector-CSR SpMV: G lanes per row
template <int G>
__global__ void __launch_bounds__(256) k_spmv(CsrV A, const double* __restrict__ x, double* __restrict__ y,
                                              double alpha, double beta) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int row = (int)(t / G);
    int sub = (int)(t % G);
    if (row >= A.n_rows) return;
    int e0 = A.ptr[row], e1 = A.ptr[row + 1];
    double s = 0.0;
    for (int e = e0 + sub; e < e1; e += G) s = fma(A.val[e], __ldg(x + A.idx[e]), s);
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, G);
    if (sub == 0) y[row] = (beta == 0.0) ? alpha * s : fma(beta, y[row], alpha * s);
}


// ---------------------------------------------------------------- SELL-32
__global__ void k_sell_width(const int32_t* __restrict__ ptr, int n, int64_t* __restrict__ w) {
    const int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int r = s * 32 + lane;
    int len = r < n ? ptr[r + 1] - ptr[r] : 0;
    len = warp_max(len);
    if (lane == 0 && s * 32 < n) w[s] = (int64_t)len * 32;
}
__global__ void k_sell_fill(CsrV A, const int64_t* __restrict__ sp, int32_t* __restrict__ col,
                            double* __restrict__ val) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= A.n_rows) return;
    const int s = r >> 5, lane = r & 31;
    const int64_t base = sp[s] + lane, end = sp[s + 1];
    const int e0 = A.ptr[r], e1 = A.ptr[r + 1];
    int64_t q = base;
    for (int e = e0; e < e1; ++e, q += 32) {
        col[q] = A.idx[e];
        val[q] = A.val[e];
    }
    for (; q < end; q += 32) {
        col[q] = 0;
        val[q] = 0.0;
    }
}
// thread per row, sequential sum in column order (as CSR row order)
__global__ void __launch_bounds__(256) k_spmv_sell(int n, const int64_t* __restrict__ sp,
                                                   const int32_t* __restrict__ col, const double* __restrict__ val,
                                                   const double* __restrict__ x, double* __restrict__ y, double alpha,
                                                   double beta) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int s = r >> 5, lane = r & 31;
    const int64_t b = sp[s] + lane, e = sp[s + 1];
    double acc = 0.0;
    int64_t q = b;
    for (; q + 3 * 32 < e; q += 4 * 32) {
        const int c0 = col[q], c1 = col[q + 32], c2 = col[q + 64], c3 = col[q + 96];
        const double v0 = val[q], v1 = val[q + 32], v2 = val[q + 64], v3 = val[q + 96];
        acc = fma(v0, __ldg(x + c0), acc);
        acc = fma(v1, __ldg(x + c1), acc);
        acc = fma(v2, __ldg(x + c2), acc);
        acc = fma(v3, __ldg(x + c3), acc);
    }
    for (; q < e; q += 32) acc = fma(val[q], __ldg(x + col[q]), acc);
    y[r] = (beta == 0.0) ? alpha * acc : fma(beta, y[r], alpha * acc);
}

// uniform slice width W (every slice stores exactly W entries per row, e.g. A_fc:
// two cells per face): the slice offset is arithmetic, so the column / value
// loads do not wait for a slice-pointer load, and all W loads are in flight
template <int W>
__global__ void __launch_bounds__(256) k_spmv_ell(int n, const int32_t* __restrict__ col,
                                                  const double* __restrict__ val, const double* __restrict__ x,
                                                  double* __restrict__ y, double alpha, double beta) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int64_t b = (int64_t)(r >> 5) * (32 * W) + (r & 31);
    int c[W];
    double v[W];
#pragma unroll
    for (int k = 0; k < W; ++k) {
        c[k] = col[b + 32 * k];
        v[k] = val[b + 32 * k];
    }
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < W; ++k) acc = fma(v[k], __ldg(x + c[k]), acc);   // same order as k_spmv_sell
    y[r] = (beta == 0.0) ? alpha * acc : fma(beta, y[r], alpha * acc);
}

// w[s] = 32 * (entries per row of slice s): widest slice and the sum of the widths
__global__ void k_sell_max_width(const int64_t* __restrict__ w, int ns, int* __restrict__ out,
                                 unsigned long long* __restrict__ sum) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < ns) {
        atomicMax(out, (int)(w[s] / 32));
        atomicAdd(sum, (unsigned long long)(w[s] / 32));
    }
}
__global__ void k_sell_set_width(int64_t* __restrict__ w, int ns, int64_t v) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < ns) w[s] = v;
}

// S = A - H, thread per row, two passes (count / fill); tau > 0 -> filter_rows
template <bool FILL>
__global__ void k_sub(CsrV A, CsrV H, double tau, int32_t* __restrict__ cnt, const int32_t* __restrict__ Sp,
                      int32_t* __restrict__ Si, double* __restrict__ Sv) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.n_rows) return;
    int a = A.ptr[i], a1 = A.ptr[i + 1], h = H.ptr[i], h1 = H.ptr[i + 1];
    double thr = 0.0;
    if (tau > 0.0) {
        double ss = 0.0;
        int p = a, q = h;
        while (p < a1 || q < h1) {
            int ca = p < a1 ? A.idx[p] : INT32_MAX, ch = q < h1 ? H.idx[q] : INT32_MAX;
            double v;
            if (ca == ch) v = A.val[p++] - H.val[q++];
            else if (ca < ch) v = A.val[p++];
            else v = 0.0 - H.val[q++];
            ss += v * v;
        }
        thr = tau * sqrt(ss);
    }
    int o = FILL ? Sp[i] : 0, n = 0;
    int p = a, q = h;
    while (p < a1 || q < h1) {
        int ca = p < a1 ? A.idx[p] : INT32_MAX, ch = q < h1 ? H.idx[q] : INT32_MAX;
        double v;
        int col;
        if (ca == ch) { col = ca; v = A.val[p++] - H.val[q++]; }
        else if (ca < ch) { col = ca; v = A.val[p++]; }
        else { col = ch; v = 0.0 - H.val[q++]; }
        bool keep = v != 0.0 && (col == i || !(fabs(v) < thr));
        if (keep) {
            if (FILL) { Si[o + n] = col; Sv[o + n] = v; }
            ++n;
        }
    }
    if (!FILL) cnt[i] = n;
}

// S = A - H without a row filter (tau = 0: only exact zeros are dropped), eight
// lanes per row.  Every entry of the union finds its own output position:
// an H entry ranks by its index in H plus the A-only entries left of it, an
// A-only entry by the H entries left of it plus the A-only ones before it; the
// kept entries are compacted through a per-row bit mask in shared memory.
// Rows the fast path does not cover (more than 8 entries in A's row, more than
// SUB_MAX entries in the union) are merged serially by the group's first lane.
constexpr int SUB_G = 8;
constexpr int SUB_MAX = 128;
__device__ __forceinline__ int sub_lower_bound(const int32_t* __restrict__ idx, int lo, int hi, int col) {
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (idx[mid] < col) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}
template <bool FILL>
__global__ void __launch_bounds__(256) k_sub_rows8(CsrV A, CsrV H, int32_t* __restrict__ cnt,
                                                   const int32_t* __restrict__ Sp, int32_t* __restrict__ Si,
                                                   double* __restrict__ Sv) {
    __shared__ unsigned mask_s[256 / SUB_G][SUB_MAX / 32];
    const int g = threadIdx.x % SUB_G, grp = threadIdx.x / SUB_G;
    const int gshift = (threadIdx.x & 31) / SUB_G * SUB_G;
    const int i = blockIdx.x * (256 / SUB_G) + grp;
    const bool live = i < A.n_rows;
    int a0 = 0, a1 = 0, h0 = 0, h1 = 0;
    if (live) { a0 = A.ptr[i]; a1 = A.ptr[i + 1]; h0 = H.ptr[i]; h1 = H.ptr[i + 1]; }
    const int nA = a1 - a0, nH = h1 - h0;
    const bool fast = nA <= SUB_G && nA + nH <= SUB_MAX;
    unsigned* mask = mask_s[grp];
    if (g < SUB_MAX / 32) mask[g] = 0u;
    // A's row: one entry per lane
    int colA = 0, lbH = 0;
    bool a_only = false;
    double vA = 0.0;
    if (fast && g < nA) {
        colA = A.idx[a0 + g];
        lbH = sub_lower_bound(H.idx, h0, h1, colA);
        a_only = !(lbH < h1 && H.idx[lbH] == colA);
        vA = A.val[a0 + g];
    }
    const unsigned onlyA = (__ballot_sync(0xffffffffu, a_only) >> gshift) & ((1u << SUB_G) - 1u);
    __syncwarp();
    if (fast) {
        if (g < nA && a_only && vA != 0.0) {
            const int u = (lbH - h0) + __popc(onlyA & ((1u << g) - 1u));
            atomicOr(&mask[u >> 5], 1u << (u & 31));
        }
        for (int q = h0 + g; q < h1; q += SUB_G) {
            const int col = H.idx[q];
            const int lb = sub_lower_bound(A.idx, a0, a1, col);
            const bool hit = lb < a1 && A.idx[lb] == col;
            const double v = (hit ? A.val[lb] : 0.0) - H.val[q];
            if (v != 0.0) {
                const int u = (q - h0) + __popc(onlyA & ((1u << (lb - a0)) - 1u));
                atomicOr(&mask[u >> 5], 1u << (u & 31));
            }
        }
    }
    __syncwarp();
    if (fast) {
        auto kept_before = [&](int u) {
            int n = 0;
            for (int w = 0; w < (u >> 5); ++w) n += __popc(mask[w]);
            return n + __popc(mask[u >> 5] & ((1u << (u & 31)) - 1u));
        };
        if (!FILL) {
            if (live && g == 0) {
                int n = 0;
#pragma unroll
                for (int w = 0; w < SUB_MAX / 32; ++w) n += __popc(mask[w]);
                cnt[i] = n;
            }
        } else {
            const int o = live ? Sp[i] : 0;
            if (g < nA && a_only && vA != 0.0) {
                const int u = (lbH - h0) + __popc(onlyA & ((1u << g) - 1u));
                const int d = o + kept_before(u);
                Si[d] = colA;
                Sv[d] = vA;
            }
            for (int q = h0 + g; q < h1; q += SUB_G) {
                const int col = H.idx[q];
                const int lb = sub_lower_bound(A.idx, a0, a1, col);
                const bool hit = lb < a1 && A.idx[lb] == col;
                const double v = (hit ? A.val[lb] : 0.0) - H.val[q];
                if (v != 0.0) {
                    const int u = (q - h0) + __popc(onlyA & ((1u << (lb - a0)) - 1u));
                    const int d = o + kept_before(u);
                    Si[d] = col;
                    Sv[d] = v;
                }
            }
        }
    } else if (live && g == 0) {   // serial merge of an oversized row
        int o = FILL ? Sp[i] : 0, n = 0, p = a0, q = h0;
        while (p < a1 || q < h1) {
            const int ca = p < a1 ? A.idx[p] : INT32_MAX, ch = q < h1 ? H.idx[q] : INT32_MAX;
            double v;
            int col;
            if (ca == ch) { col = ca; v = A.val[p++] - H.val[q++]; }
            else if (ca < ch) { col = ca; v = A.val[p++]; }
            else { col = ch; v = 0.0 - H.val[q++]; }
            if (v != 0.0) {
                if (FILL) { Si[o + n] = col; Sv[o + n] = v; }
                ++n;
            }
        }
        if (!FILL) cnt[i] = n;
    }
}

template <bool FILL>
__global__ void k_filter(CsrV A, double tau, bool keep_diag, int32_t* __restrict__ cnt, const int32_t* __restrict__ Sp,
                         int32_t* __restrict__ Si, double* __restrict__ Sv) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.n_rows) return;
    int a = A.ptr[i], a1 = A.ptr[i + 1];
    double ss = 0.0;
    for (int p = a; p < a1; ++p) ss += A.val[p] * A.val[p];
    double thr = tau * sqrt(ss);
    int o = FILL ? Sp[i] : 0, n = 0;
    for (int p = a; p < a1; ++p) {
        double v = A.val[p];
        int col = A.idx[p];
        if (v != 0.0 && ((keep_diag && col == i) || !(fabs(v) < thr))) {
            if (FILL) { Si[o + n] = col; Sv[o + n] = v; }
            ++n;
        }
    }
    if (!FILL) cnt[i] = n;
}

}  // namespace

int64_t scan_counts(Ctx* c, const int32_t* counts, int32_t* ptr_out, int32_t n) {
    if (n == 0) {
        EDFA_CUDA(cudaMemsetAsync(ptr_out, 0, sizeof(int32_t), c->stream));
        return 0;
    }
    DevBuf<int64_t> incl(c, n);
    cub::TransformInputIterator<int64_t, ToI64, const int32_t*> it(counts, ToI64());
    size_t bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, bytes, it, incl.p, n, c->stream);
    void* tmp = c->cub_scratch(bytes);
    {
        Prof pr(c, "scan", 12.0 * n);
        EDFA_CUDA(cub::DeviceScan::InclusiveSum(tmp, bytes, it, incl.p, n, c->stream));
        k_incl_to_ptr<<<ceil_div(n, 256), 256, 0, c->stream>>>(incl.p, ptr_out, n);
        check_launch("k_incl_to_ptr");
    }
    int64_t total = 0;
    EDFA_CUDA(cudaMemcpyAsync(&total, incl.p + (n - 1), sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
    require(total <= INT32_MAX, EDFA_ERR_UNSUPPORTED, "matrix exceeds 2^31-1 stored entries");
    return total;
}

void fill(Ctx* c, double* p, int64_t n, double v) {
    if (n <= 0) return;
    Prof pr(c, "fill", 8.0 * n);
    int blocks = std::min<int64_t>(ceil_div(n, 256), NUM_SMS_B200 * 8);
    k_fill<<<blocks, 256, 0, c->stream>>>(p, n, v);
    check_launch("k_fill");
}
void fill_bits(Ctx* c, double* p, int64_t n, unsigned long long bits) {
    if (n <= 0) return;
    Prof pr(c, "fill", 8.0 * n);
    int blocks = std::min<int64_t>(ceil_div(n, 256), NUM_SMS_B200 * 8);
    k_fill_bits<<<blocks, 256, 0, c->stream>>>(reinterpret_cast<unsigned long long*>(p), n, bits);
    check_launch("k_fill_bits");
}

void transpose(Ctx* c, const Csr& A, Csr& AT) {
    AT.n_rows = A.n_cols;
    AT.n_cols = A.n_rows;
    AT.nnz = A.nnz;
    AT.ptr.reset(c, (size_t)A.n_cols + 1);
    AT.idx.reset(c, A.nnz);
    if (A.val.p) AT.val.reset(c, A.nnz);
    else AT.val.release();
    DevBuf<int32_t> cnt(c, std::max<int32_t>(A.n_cols, 1));
    EDFA_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t) * std::max<int32_t>(A.n_cols, 1), c->stream));
    if (A.nnz == 0) {
        EDFA_CUDA(cudaMemsetAsync(AT.ptr.p, 0, sizeof(int32_t) * (A.n_cols + 1), c->stream));
        return;
    }
    DevBuf<int32_t> row_of(c, A.nnz), ids(c, A.nnz), keys_out(c, A.nnz), order(c, A.nnz);
    {
        Prof pr(c, "transpose", 24.0 * A.nnz + 8.0 * A.n_rows);
        const int64_t mean = A.nnz / std::max(A.n_rows, 1);
        if (mean <= 4)
            k_row_of<4><<<ceil_div((int64_t)A.n_rows * 4, 256), 256, 0, c->stream>>>(A.ptr.p, A.n_rows, row_of.p);
        else if (mean <= 16)
            k_row_of<8><<<ceil_div((int64_t)A.n_rows * 8, 256), 256, 0, c->stream>>>(A.ptr.p, A.n_rows, row_of.p);
        else
            k_row_of<32><<<ceil_div((int64_t)A.n_rows * 32, 256), 256, 0, c->stream>>>(A.ptr.p, A.n_rows, row_of.p);
        k_iota<<<ceil_div(A.nnz, 256), 256, 0, c->stream>>>(ids.p, A.nnz);
        k_col_hist<<<ceil_div(A.nnz, 256), 256, 0, c->stream>>>(A.idx.p, A.nnz, cnt.p);
        check_launch("transpose prep");
    }
    scan_counts(c, cnt.p, AT.ptr.p, A.n_cols);
    int bits = 1;
    while ((1ll << bits) < (int64_t)A.n_cols) ++bits;
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, A.idx.p, keys_out.p, ids.p, order.p, (int)A.nnz, 0, bits,
                                    c->stream);
    void* tmp = c->cub_scratch(bytes);
    {
        Prof pr(c, "transpose", 32.0 * A.nnz);
        EDFA_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, A.idx.p, keys_out.p, ids.p, order.p, (int)A.nnz, 0,
                                                  bits, c->stream));
        k_gather_T<<<ceil_div(A.nnz, 256), 256, 0, c->stream>>>(order.p, row_of.p, A.val.p, A.nnz, AT.idx.p,
                                                                AT.val.p);
        check_launch("k_gather_T");
    }
}

void block_merge(Ctx* c, const Csr& A, const Csr& B, const Csr& C, const Csr& D, Csr& M) {
    require(A.n_rows == B.n_rows && C.n_rows == D.n_rows && A.n_cols == C.n_cols && B.n_cols == D.n_cols,
            EDFA_ERR_VALUE, "block shapes are inconsistent");
    M.n_rows = A.n_rows + C.n_rows;
    M.n_cols = A.n_cols + B.n_cols;
    M.nnz = A.nnz + B.nnz + C.nnz + D.nnz;
    require(M.nnz <= INT32_MAX, EDFA_ERR_UNSUPPORTED, "system exceeds 2^31-1 stored entries");
    M.ptr.reset(c, (size_t)M.n_rows + 1);
    M.idx.reset(c, M.nnz);
    M.val.reset(c, M.nnz);
    Prof pr(c, "block_merge", 24.0 * M.nnz);
    k_merge_ptr<<<ceil_div(M.n_rows + 1, 256), 256, 0, c->stream>>>(A.ptr.p, B.ptr.p, C.ptr.p, D.ptr.p, A.n_rows,
                                                                   C.n_rows, M.ptr.p);
    if (M.nnz <= 16ll * M.n_rows)
        k_merge_fill<8><<<ceil_div((int64_t)M.n_rows * 8, 256), 256, 0, c->stream>>>(view(A), view(B), view(C), view(D),
                                                                                    M.ptr.p, M.idx.p, M.val.p);
    else
        k_merge_fill<32><<<ceil_div((int64_t)M.n_rows * 32, 256), 256, 0, c->stream>>>(
            view(A), view(B), view(C), view(D), M.ptr.p, M.idx.p, M.val.p);
    check_launch("block_merge");
}

void spmv(Ctx* c, const CsrV& A, int64_t nnz, const double* x, double* y, double alpha, double beta,
          const char* name) {
    if (A.n_rows == 0) return;
    double avg = A.n_rows ? double(nnz) / A.n_rows : 0.0;
    Prof pr(c, name, 12.0 * nnz + 4.0 * (A.n_rows + 1) + 8.0 * A.n_cols + 8.0 * A.n_rows * (beta != 0.0 ? 2 : 1));
    auto launch = [&](auto kern, int G) {
        int64_t threads = (int64_t)A.n_rows * G;
        kern<<<ceil_div(threads, 256), 256, 0, c->stream>>>(A, x, y, alpha, beta);
    };
    if (avg <= 3.0) launch(k_spmv<1>, 1);
    else if (avg <= 6.0) launch(k_spmv<2>, 2);
    else if (avg <= 12.0) launch(k_spmv<4>, 4);
    else if (avg <= 24.0) launch(k_spmv<8>, 8);
    else if (avg <= 48.0) launch(k_spmv<16>, 16);
    else launch(k_spmv<32>, 32);
    check_launch("k_spmv");
}


void build_sell(Ctx* c, const Csr& A, Sell& S) {
    const int n = A.n_rows;
    S.n_rows = n;
    S.n_cols = A.n_cols;
    S.nnz = A.nnz;
    const int ns = ceil_div(n, 32);
    S.slice_ptr.reset(c, (size_t)ns + 1);
    DevBuf<int64_t> w(c, (size_t)ns + 1);
    EDFA_CUDA(cudaMemsetAsync(w.p, 0, sizeof(int64_t) * (ns + 1), c->stream));
    if (n) {
        Prof pr(c, "sell_build", 4.0 * n);
        k_sell_width<<<ceil_div((int64_t)ns * 32, 256), 256, 0, c->stream>>>(A.ptr.p, n, w.p);
        check_launch("k_sell_width");
    }
    // narrow matrices whose slices are (almost) all as wide as the widest are stored with
    // ONE width (the few narrower slices padded): the SpMV then needs no slice pointers
    int* mw = c->d_scalar_i + 46;   // [max width, sum of widths (entries per row, 64-bit)]
    int h_mw = 0;
    unsigned long long h_sum = 0;
    EDFA_CUDA(cudaMemsetAsync(mw, 0, 4 * sizeof(int), c->stream));
    if (ns) k_sell_max_width<<<ceil_div(ns, 256), 256, 0, c->stream>>>(w.p, ns, mw,
                                                                       reinterpret_cast<unsigned long long*>(mw + 2));
    EDFA_CUDA(cudaMemcpyAsync(&h_mw, mw, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaMemcpyAsync(&h_sum, mw + 2, sizeof(h_sum), cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
    S.uniform_w = 0;
    if (ns > 0 && (h_mw == 2 || h_mw == 6) && (double)ns * h_mw <= 1.05 * (double)h_sum) {
        S.uniform_w = h_mw;
        k_sell_set_width<<<ceil_div(ns, 256), 256, 0, c->stream>>>(w.p, ns, (int64_t)h_mw * 32);
    }
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, w.p, S.slice_ptr.p, ns + 1, c->stream);
    EDFA_CUDA(cub::DeviceScan::ExclusiveSum(c->cub_scratch(bytes), bytes, w.p, S.slice_ptr.p, ns + 1, c->stream));
    EDFA_CUDA(cudaMemcpyAsync(&S.stored, S.slice_ptr.p + ns, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
    S.col.reset(c, std::max<int64_t>(S.stored, 1));
    S.val.reset(c, std::max<int64_t>(S.stored, 1));
    if (n) {
        Prof pr(c, "sell_build", 24.0 * S.stored);
        k_sell_fill<<<ceil_div(n, 256), 256, 0, c->stream>>>(view(A), S.slice_ptr.p, S.col.p, S.val.p);
        check_launch("k_sell_fill");
    }
}

void spmv_sell(Ctx* c, const Sell& A, const double* x, double* y, double alpha, double beta, const char* name) {
    if (A.n_rows == 0) return;
    Prof pr(c, name, 12.0 * A.nnz + 4.0 * (A.n_rows + 1) + 8.0 * A.n_cols + 8.0 * A.n_rows * (beta != 0.0 ? 2 : 1));
    const int g = ceil_div(A.n_rows, 256);
    if (A.uniform_w == 2) k_spmv_ell<2><<<g, 256, 0, c->stream>>>(A.n_rows, A.col.p, A.val.p, x, y, alpha, beta);
    else if (A.uniform_w == 6) k_spmv_ell<6><<<g, 256, 0, c->stream>>>(A.n_rows, A.col.p, A.val.p, x, y, alpha, beta);
    else
        k_spmv_sell<<<g, 256, 0, c->stream>>>(A.n_rows, A.slice_ptr.p, A.col.p, A.val.p, x, y, alpha, beta);
    check_launch("k_spmv_sell");
}

void csr_sub(Ctx* c, const Csr& A, const Csr& H, double tau, Csr& S) {
    require(A.n_rows == H.n_rows && A.n_cols == H.n_cols, EDFA_ERR_VALUE, "A_cc and H shapes differ");
    int n = A.n_rows;
    S.n_rows = n;
    S.n_cols = A.n_cols;
    S.ptr.reset(c, (size_t)n + 1);
    DevBuf<int32_t> cnt(c, std::max(n, 1));
    if (n) {
        Prof pr(c, "schur_sub", 12.0 * (A.nnz + H.nnz) + 8.0 * n);
        if (tau > 0.0)
            k_sub<false><<<ceil_div(n, 128), 128, 0, c->stream>>>(view(A), view(H), tau, cnt.p, nullptr, nullptr,
                                                                 nullptr);
        else
            k_sub_rows8<false><<<ceil_div(n, 256 / SUB_G), 256, 0, c->stream>>>(view(A), view(H), cnt.p, nullptr,
                                                                               nullptr, nullptr);
        check_launch("k_sub count");
    }
    S.nnz = scan_counts(c, cnt.p, S.ptr.p, n);
    S.idx.reset(c, S.nnz);
    S.val.reset(c, S.nnz);
    if (n) {
        Prof pr(c, "schur_sub", 12.0 * (A.nnz + H.nnz + S.nnz) + 8.0 * n);
        if (tau > 0.0)
            k_sub<true><<<ceil_div(n, 128), 128, 0, c->stream>>>(view(A), view(H), tau, nullptr, S.ptr.p, S.idx.p,
                                                                S.val.p);
        else
            k_sub_rows8<true><<<ceil_div(n, 256 / SUB_G), 256, 0, c->stream>>>(view(A), view(H), nullptr, S.ptr.p,
                                                                              S.idx.p, S.val.p);
        check_launch("k_sub fill");
    }
}

void csr_filter(Ctx* c, const Csr& A, double tau, Csr& out, bool keep_diag) {
    int n = A.n_rows;
    out.n_rows = n;
    out.n_cols = A.n_cols;
    out.ptr.reset(c, (size_t)n + 1);
    DevBuf<int32_t> cnt(c, std::max(n, 1));
    if (n) {
        Prof pr(c, "filter_rows", 12.0 * A.nnz);
        k_filter<false><<<ceil_div(n, 128), 128, 0, c->stream>>>(view(A), tau, keep_diag, cnt.p, nullptr, nullptr, nullptr);
        check_launch("k_filter count");
    }
    out.nnz = scan_counts(c, cnt.p, out.ptr.p, n);
    out.idx.reset(c, out.nnz);
    out.val.reset(c, out.nnz);
    if (n) {
        Prof pr(c, "filter_rows", 12.0 * (A.nnz + out.nnz));
        k_filter<true><<<ceil_div(n, 128), 128, 0, c->stream>>>(view(A), tau, keep_diag, nullptr, out.ptr.p, out.idx.p,
                                                               out.val.p);
        check_launch("k_filter fill");
    }
}

void copy_csr(Ctx* c, const Csr& A, Csr& out) {
    out.n_rows = A.n_rows;
    out.n_cols = A.n_cols;
    out.nnz = A.nnz;
    out.ptr.reset(c, (size_t)A.n_rows + 1);
    out.idx.reset(c, A.nnz);
    EDFA_CUDA(cudaMemcpyAsync(out.ptr.p, A.ptr.p, sizeof(int32_t) * (A.n_rows + 1), cudaMemcpyDeviceToDevice,
                              c->stream));
    if (A.nnz)
        EDFA_CUDA(cudaMemcpyAsync(out.idx.p, A.idx.p, sizeof(int32_t) * A.nnz, cudaMemcpyDeviceToDevice,
                                  c->stream));
    if (A.val.p) {
        out.val.reset(c, A.nnz);
        if (A.nnz)
            EDFA_CUDA(cudaMemcpyAsync(out.val.p, A.val.p, sizeof(double) * A.nnz, cudaMemcpyDeviceToDevice,
                                      c->stream));
    }
}

}  // namespace edfa
