// K3: H~ = G~ A_ff F~ (hx/precond.py:257) with the optional post-product
// filtration fused into the epilogue (hx/precond.py:258-259, 138-157).
//
// Row-wise Gustavson, one warp per cell row m, two passes (count, fill):
//   W_m = sum_{i in G_m, ascending} g_mi * A_ff[i, :]    (scipy csr_matmat order)
//   H_m = sum_{k in W_m} W_mk * F~[k, :], k in reverse first-encounter order
//         (the unsorted row order csr_matmat emits W in)
// Both accumulators are shared-memory open-addressing tables; each
// accumulation step adds the contributions of ONE source entry, whose target
// columns are distinct, so lanes never collide and every sum is formed in a
// fixed order (deterministic, bit-reproducible across runs).  Products are
// not contracted into FMAs, as in the reference's compiled sparsetools.
#include <mutex>
#include <set>

#include "dev_util.cuh"
#include "edfa_internal.cuh"
#include "objects.cuh"

namespace edfa {
namespace {

constexpr int EMPTY = -1;

__device__ __forceinline__ unsigned hslot(int key, int bits) { return ((unsigned)key * 2654435761u) >> (32 - bits); }

// find-or-insert; returns slot or -1 when the table is full (*fresh: inserted now)
__device__ int h_insert(int* keys, int bits, int key, bool* fresh = nullptr) {
    int mask = (1 << bits) - 1;
    unsigned s = hslot(key, bits);
    for (int t = 0; t <= mask; ++t) {
        int cur = keys[s];
        if (cur == key) { if (fresh) *fresh = false; return (int)s; }
        if (cur == EMPTY) {
            int prev = atomicCAS(&keys[s], EMPTY, key);
            if (prev == EMPTY) { if (fresh) *fresh = true; return (int)s; }
            if (prev == key) { if (fresh) *fresh = false; return (int)s; }
        }
        s = (s + 1) & mask;
    }
    return -1;
}

// compact (key, val) of a table into its front, sort by key; returns count
__device__ int h_extract_sorted(int* keys, double* vals, int bits, int* tmpk, double* tmpv, int lane) {
    int n_tab = 1 << bits;
    int n = 0;
    for (int i0 = 0; i0 < n_tab; i0 += 32) {
        int i = i0 + lane;
        bool live = keys[i] != EMPTY;
        unsigned bal = __ballot_sync(0xffffffffu, live);
        if (live) {
            int p = n + __popc(bal & ((1u << lane) - 1));
            tmpk[p] = keys[i];
            tmpv[p] = vals[i];
        }
        n += __popc(bal);
    }
    __syncwarp();
    int np2 = 32;
    while (np2 < n) np2 <<= 1;
    for (int i = n + lane; i < np2; i += 32) tmpk[i] = INT32_MAX;
    __syncwarp();
    for (int k = 2; k <= np2; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = lane; i < np2; i += 32) {
                int l = i ^ j;
                if (l > i) {
                    int a = tmpk[i], b = tmpk[l];
                    bool up = (i & k) == 0;
                    if ((a > b) == up) {
                        tmpk[i] = b; tmpk[l] = a;
                        double va = tmpv[i]; tmpv[i] = tmpv[l]; tmpv[l] = va;
                    }
                }
            }
            __syncwarp();
        }
    return n;
}

struct ProdArgs {
    CsrV G, A, F;
    int32_t n_rows;
    const int32_t* rows;   // optional row list (overflow re-run)
    int32_t n_list;
    double tau;
    int32_t* cnt;          // pass 1
    const int32_t* Hp;     // pass 2
    int32_t* Hi;
    double* Hv;
    int32_t* overflow;     // [count, rows...]
    int32_t cap;           // PADDED: row capacity of the padded output
};

// pass modes: COUNT (row lengths), FILL (into final CSR positions), PADDED
// (single pass: rows of <= cap entries into a padded buffer + their lengths;
// longer rows go to the overflow list like table overflows)
enum { COUNT = 0, FILL = 1, PADDED = 2 };

template <int BITS, int MODE>
__global__ void __launch_bounds__(256) k_product(ProdArgs a) {
    constexpr int T = 1 << BITS;
    extern __shared__ __align__(16) unsigned char smem[];
    const int warps = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // per warp: table keys/vals, sorted W (keys/vals), H table keys/vals
    unsigned char* base = smem + (size_t)wid * T * (4 + 8) * 3;
    double* tv = reinterpret_cast<double*>(base);
    double* wv = tv + T;
    double* hv = wv + T;
    int* tk = reinterpret_cast<int*>(hv + T);
    int* wk = tk + T;
    int* hk = wk + T;
    int n_items = a.rows ? a.n_list : a.n_rows;
    for (int it = blockIdx.x * warps + wid; it < n_items; it += gridDim.x * warps) {
        int m = a.rows ? a.rows[it] : it;
        for (int i = lane; i < T; i += 32) { tk[i] = EMPTY; tv[i] = 0.0; hk[i] = EMPTY; hv[i] = 0.0; }
        __syncwarp();
        bool full = false;
        // ---- W = g_m A_ff; wk records the slots in first-encounter order
        int g0 = a.G.ptr[m], g1 = a.G.ptr[m + 1];
        int nW = 0;
        for (int t = g0; t < g1; ++t) {
            int i = a.G.idx[t];
            double g = a.G.val[t];
            const int e0 = a.A.ptr[i], e1 = a.A.ptr[i + 1];
            for (int eb = e0; eb < e1; eb += 32) {
                const int e = eb + lane;
                bool fresh = false;
                int s = -1;
                if (e < e1) {
                    s = h_insert(tk, BITS, a.A.idx[e], &fresh);
                    if (s < 0) full = true;
                    else tv[s] = add_mul(tv[s], g, a.A.val[e]);
                }
                const unsigned bal = __ballot_sync(0xffffffffu, fresh);
                if (fresh && nW + __popc(bal & ((1u << lane) - 1)) < T) wk[nW + __popc(bal & ((1u << lane) - 1))] = s;
                nW += __popc(bal);
            }
            __syncwarp();
        }
        full = __any_sync(0xffffffffu, full) || nW > T;
        // scipy's csr_matmat emits a row's columns in REVERSE first-encounter
        // order (linked-list head insertion), and (G A_ff) F walks W that way:
        // H sums are formed in exactly the reference's order
        if (!full) {
            for (int q = lane; q < nW; q += 32) hk[q] = wk[q];
            __syncwarp();
            for (int q = lane; q < nW; q += 32) {
                const int sl = hk[nW - 1 - q];
                wk[q] = tk[sl];
                wv[q] = tv[sl];
            }
            __syncwarp();
            for (int q = lane; q < nW; q += 32) hk[q] = EMPTY;
            __syncwarp();
        }
        // ---- H = W F
        if (!full) {
            for (int t = 0; t < nW; ++t) {
                double w = wv[t];
                if (w == 0.0) continue;          // scipy drops exact-zero sums of W
                int k = wk[t];
                for (int e = a.F.ptr[k] + lane; e < a.F.ptr[k + 1]; e += 32) {
                    int s = h_insert(hk, BITS, a.F.idx[e]);
                    if (s < 0) full = true;
                    else hv[s] = add_mul(hv[s], w, a.F.val[e]);
                }
                __syncwarp();
            }
            full = __any_sync(0xffffffffu, full);
        }
        int nH = 0;
        if (!full) {
            nH = h_extract_sorted(hk, hv, BITS, tk, tv, lane);   // sorted H row in (tk, tv)
            if (MODE == PADDED && nH > a.cap) full = true;       // (kept entries <= nH)
        }
        if (full) {
            if (lane == 0) {
                if (MODE != FILL) a.cnt[m] = 0;
                int p = atomicAdd(a.overflow, 1);
                a.overflow[1 + p] = m;
            }
            __syncwarp();
            continue;
        }
        double thr = 0.0;
        if (a.tau > 0.0) {
            double ss = 0.0;
            for (int i = lane; i < nH; i += 32) ss += tv[i] * tv[i];
            thr = a.tau * sqrt(warp_sum(ss));
        }
        const long long o = MODE == FILL     ? (long long)a.Hp[m]
                            : MODE == PADDED ? (long long)(a.rows ? it : m) * a.cap
                                             : 0;
        int n = 0;
        for (int i0 = 0; i0 < nH; i0 += 32) {
            int i = i0 + lane;
            double v = i < nH ? tv[i] : 0.0;
            int col = i < nH ? tk[i] : -1;
            bool keep = i < nH && v != 0.0 && (col == m || !(fabs(v) < thr));
            unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (MODE != COUNT && keep) {
                const long long p = o + n + __popc(bal & ((1u << lane) - 1));
                a.Hi[p] = col;
                a.Hv[p] = v;
            }
            n += __popc(bal);
        }
        if (MODE != FILL && lane == 0) a.cnt[m] = n;
        __syncwarp();
    }
}

// ---- first tier: the same accumulation, operands prefetched.
// k_product walks G_m entry by entry and W_m entry by entry, and every step
// started with dependent global loads (row pointer, then the row) -- ~60
// serialised L2/HBM round trips per row.  Here the warp first loads G_m's
// entries and the row pointers they need in one round, then every A_ff entry
// the row will touch (flattened, all loads in flight) into shared memory, and
// the same for the F~ rows of W_m; the hash accumulation then runs from
// shared memory in exactly k_product's order (bit-identical results).  Rows
// that exceed the tier's capacities go to the overflow list (k_product).
// staged F~ / A_ff entries per cell: 288 keeps a warp's working set at 9.2 KB, so three blocks (24 warps)
// share an SM instead of two (config 5: 123 -> 90 ms; cells with more products take the next tier)
#ifndef EDFA_PF_CAPF
#define EDFA_PF_CAPF 288
#endif
constexpr int PF_BITS = 7, PF_T = 1 << PF_BITS, PF_CAPG = 32, PF_CAPF = EDFA_PF_CAPF, PF_CAP = 64;
constexpr size_t PF_WARP_BYTES = (size_t)PF_T * 12 * 3 + PF_CAPG * (8 + 4 + 4) + (PF_CAPG + 1) * 4 +
                                 (PF_T + 1) * 4 + (size_t)PF_CAPF * 12;

__device__ __forceinline__ int seg_of(const int* off, int n, int p) {   // last t with off[t] <= p
    int lo = 0, hi = n;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (off[mid] <= p) lo = mid;
        else hi = mid;
    }
    return lo;
}

// One chunk of 32 consecutive contributions (lane order = flattened order p)
// added into a hash accumulator with exactly the sequential semantics:
// lanes holding the same key form a match group whose leader (lowest lane)
// inserts, and the group's adds run in lane order, so every sum is formed in
// increasing p (bit-identical to one entry at a time).  Returns the slot and
// whether the leader inserted the key now (first encounter).
__device__ __forceinline__ int chunk_accumulate(int* keys, double* vals, int bits, bool act, int key, double v,
                                                int lane, bool* fresh_out, bool* full) {
    const unsigned am = __ballot_sync(0xffffffffu, act);
    const unsigned grp = __match_any_sync(0xffffffffu, act ? key : INT32_MIN);
    const int leader = __ffs(grp) - 1;
    bool fresh = false;
    int sl = -1;
    if (act && lane == leader) {
        sl = h_insert(keys, bits, key, &fresh);
        if (sl < 0) *full = true;
    }
    sl = __shfl_sync(0xffffffffu, sl, leader);
    const int rank = __popc(grp & am & ((1u << lane) - 1));
    int rmax = act ? rank : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rmax = max(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
    for (int r = 0; r <= rmax; ++r) {
        if (act && sl >= 0 && rank == r) vals[sl] = __dadd_rn(vals[sl], v);
        __syncwarp();
    }
    *fresh_out = fresh;
    return sl;
}

__global__ void __launch_bounds__(256) k_product_pf(ProdArgs a) {
    constexpr int T = PF_T;
    extern __shared__ __align__(16) unsigned char smem[];
    const int warps = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* base = smem + (size_t)wid * PF_WARP_BYTES;
    double* tv = reinterpret_cast<double*>(base);
    double* wv = tv + T;
    double* hv = wv + T;
    double* gv = hv + T;                                 // PF_CAPG
    double* fval = gv + PF_CAPG;                         // PF_CAPF
    int* tk = reinterpret_cast<int*>(fval + PF_CAPF);
    int* wk = tk + T;
    int* hk = wk + T;
    int* ga0 = hk + T;                                   // PF_CAPG
    int* goff = ga0 + PF_CAPG;                           // PF_CAPG + 1
    int* wo = goff + PF_CAPG + 1;                        // T + 1
    int* fcol = wo + T + 1;                              // PF_CAPF
    for (int m = blockIdx.x * warps + wid; m < a.n_rows; m += gridDim.x * warps) {
        for (int i = lane; i < T; i += 32) { tk[i] = EMPTY; tv[i] = 0.0; hk[i] = EMPTY; hv[i] = 0.0; }
        const int g0 = a.G.ptr[m], nG = a.G.ptr[m + 1] - g0;
        bool full = nG > PF_CAPG;
        // ---- G_m entries and the A_ff row extents they select (one round trip each)
        int len = 0;
        if (!full && lane < nG) {
            const int i = a.G.idx[g0 + lane];
            gv[lane] = a.G.val[g0 + lane];
            const int e0 = a.A.ptr[i];
            ga0[lane] = e0;
            len = a.A.ptr[i + 1] - e0;
        }
        int inc = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        const int P = __shfl_sync(0xffffffffu, inc, 31);
        if (lane < nG) goff[lane] = inc - len;
        if (lane == 0) goff[min(nG, PF_CAPG)] = P;
        full = full || P > PF_CAPF;
        __syncwarp();
        // ---- every A_ff entry of the row's W, flattened, loads in flight
        if (!full)
            for (int p = lane; p < P; p += 32) {   // products formed here: acc + (g * a), no contraction
                const int t = seg_of(goff, nG, p);
                const int e = ga0[t] + (p - goff[t]);
                fcol[p] = a.A.idx[e];
                fval[p] = __dmul_rn(gv[t], a.A.val[e]);
            }
        __syncwarp();
        // ---- W = g_m A_ff from shared memory, k_product's order
        int nW = 0;
        if (!full) {
            for (int pb = 0; pb < P; pb += 32) {   // 32 contributions per step, in p order
                const int e = pb + lane;
                bool fresh = false;
                const int sl = chunk_accumulate(tk, tv, PF_BITS, e < P, e < P ? fcol[e] : 0, e < P ? fval[e] : 0.0,
                                                lane, &fresh, &full);
                const unsigned bal = __ballot_sync(0xffffffffu, fresh);
                const int pos = nW + __popc(bal & ((1u << lane) - 1));
                if (fresh && pos < T) wk[pos] = sl;
                nW += __popc(bal);
                __syncwarp();
            }
            full = __any_sync(0xffffffffu, full) || nW > T;
        }
        if (!full) {   // reverse first-encounter order (scipy csr_matmat's emission order)
            for (int q = lane; q < nW; q += 32) hk[q] = wk[q];
            __syncwarp();
            for (int q = lane; q < nW; q += 32) {
                const int sl = hk[nW - 1 - q];
                wk[q] = tk[sl];
                wv[q] = tv[sl];
            }
            __syncwarp();
            for (int q = lane; q < nW; q += 32) hk[q] = EMPTY;
            __syncwarp();
        }
        // ---- F~ rows of W's entries: extents, then every entry, flattened
        int P2 = 0;
        if (!full) {
            int run = 0;
            for (int q0 = 0; q0 < nW; q0 += 32) {
                const int q = q0 + lane;
                int l2 = 0;
                if (q < nW && wv[q] != 0.0) {            // scipy drops exact-zero sums of W
                    const int k = wk[q];
                    const int f0 = a.F.ptr[k];
                    tk[q] = f0;                           // tk is free after the W extraction
                    l2 = a.F.ptr[k + 1] - f0;
                }
                int inc2 = l2;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, inc2, o);
                    if (lane >= o) inc2 += v;
                }
                if (q < nW) wo[q] = run + inc2 - l2;
                run += __shfl_sync(0xffffffffu, inc2, 31);
            }
            if (lane == 0) wo[nW] = run;
            P2 = run;
            full = P2 > PF_CAPF;
            __syncwarp();
            if (!full)
                for (int p = lane; p < P2; p += 32) {
                    const int q = seg_of(wo, nW, p);
                    const int e = tk[q] + (p - wo[q]);
                    fcol[p] = a.F.idx[e];
                    fval[p] = __dmul_rn(wv[q], a.F.val[e]);
                }
            __syncwarp();
        }
        // ---- H = W F from shared memory, k_product's order
        if (!full) {
            for (int pb = 0; pb < P2; pb += 32) {  // zero sums of W contribute nothing (empty ranges)
                const int e = pb + lane;
                bool fresh = false;
                chunk_accumulate(hk, hv, PF_BITS, e < P2, e < P2 ? fcol[e] : 0, e < P2 ? fval[e] : 0.0, lane, &fresh,
                                 &full);
                __syncwarp();
            }
            full = __any_sync(0xffffffffu, full);
        }
        int nH = 0;
        if (!full) {
            nH = h_extract_sorted(hk, hv, PF_BITS, tk, tv, lane);   // sorted H row in (tk, tv)
            if (nH > PF_CAP) full = true;
        }
        if (full) {
            if (lane == 0) {
                a.cnt[m] = 0;
                const int p = atomicAdd(a.overflow, 1);
                a.overflow[1 + p] = m;
            }
            __syncwarp();
            continue;
        }
        double thr = 0.0;
        if (a.tau > 0.0) {
            double ss = 0.0;
            for (int i = lane; i < nH; i += 32) ss += tv[i] * tv[i];
            thr = a.tau * sqrt(warp_sum(ss));
        }
        const long long o = (long long)m * PF_CAP;
        int n = 0;
        for (int i0 = 0; i0 < nH; i0 += 32) {
            const int i = i0 + lane;
            const double v = i < nH ? tv[i] : 0.0;
            const int col = i < nH ? tk[i] : -1;
            const bool keep = i < nH && v != 0.0 && (col == m || !(fabs(v) < thr));
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const long long p = o + n + __popc(bal & ((1u << lane) - 1));
                a.Hi[p] = col;
                a.Hv[p] = v;
            }
            n += __popc(bal);
        }
        if (lane == 0) a.cnt[m] = n;
        __syncwarp();
    }
}

void launch_product_pf(Ctx* c, const ProdArgs& a) {
    constexpr int warps = 8;
    const size_t sm = PF_WARP_BYTES * warps;
    static std::mutex mu;
    static std::set<int> done;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (done.insert(c->device).second)
            EDFA_CUDA(cudaFuncSetAttribute(k_product_pf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    }
    const int per_sm = std::max(1, (int)((227 * 1024) / sm));
    const int blocks = std::max(1, std::min(ceil_div(a.n_rows, warps), NUM_SMS_B200 * per_sm * 8));
    k_product_pf<<<blocks, warps * 32, sm, c->stream>>>(a);
    check_launch("k_product_pf");
}

template <int BITS, int MODE>
void launch_product(Ctx* c, const ProdArgs& a) {
    constexpr int T = 1 << BITS;
    size_t pw = (size_t)T * 12 * 3;
    int warps = (int)std::max<size_t>(1, std::min<size_t>(8, (200 * 1024) / pw));
    size_t sm = pw * warps;
    auto kern = k_product<BITS, MODE>;
    EDFA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    int items = a.rows ? a.n_list : a.n_rows;
    int per_sm = std::max(1, (int)((227 * 1024) / sm));
    int blocks = std::max(1, std::min(ceil_div(items, warps), NUM_SMS_B200 * per_sm * 4));
    kern<<<blocks, warps * 32, sm, c->stream>>>(a);
    check_launch("k_product");
}

__global__ void k_unpad(const int32_t* __restrict__ cnt, const int32_t* __restrict__ Hp, int n, int cap,
                        const int32_t* __restrict__ pi, const double* __restrict__ pv, int32_t* __restrict__ Hi,
                        double* __restrict__ Hv) {
    // one warp per row; rows of the overflow list have cnt 0 here
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= n) return;
    const int c = cnt[w], o = Hp[w];
    const size_t src = (size_t)w * cap;
    for (int i = lane; i < c; i += 32) {
        Hi[o + i] = pi[src + i];
        Hv[o + i] = pv[src + i];
    }
}

// rows of a re-run list, padded by list position
__global__ void k_unpad_list(const int32_t* __restrict__ rows, int nl, const int32_t* __restrict__ cnt,
                             const int32_t* __restrict__ Hp, int cap, const int32_t* __restrict__ pi,
                             const double* __restrict__ pv, int32_t* __restrict__ Hi, double* __restrict__ Hv) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= nl) return;
    const int m = rows[w];
    const int c = cnt[m], o = Hp[m];
    const size_t src = (size_t)w * cap;
    for (int i = lane; i < c; i += 32) {
        Hi[o + i] = pi[src + i];
        Hv[o + i] = pv[src + i];
    }
}

std::vector<int32_t> read_overflow(Ctx* c, int32_t* ovf_dev) {
    int n_ovf = 0;
    EDFA_CUDA(cudaMemcpyAsync(&n_ovf, ovf_dev, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
    std::vector<int32_t> rows(n_ovf);
    if (n_ovf) {
        EDFA_CUDA(cudaMemcpyAsync(rows.data(), ovf_dev + 1, sizeof(int) * n_ovf, cudaMemcpyDeviceToHost, c->stream));
        EDFA_CUDA(cudaStreamSynchronize(c->stream));
    }
    return rows;
}

}  // namespace

void triple_product(Ctx* c, const Csr& G, const Csr& A, const Csr& F, double post_tau, Csr& H) {
    const int n = G.n_rows;
    H.n_rows = n;
    H.n_cols = F.n_cols;
    H.ptr.reset(c, (size_t)n + 1);
    DevBuf<int32_t> cnt(c, std::max(n, 1));
    DevBuf<int32_t> ovf(c, (size_t)n + 1);
    ProdArgs a{};
    a.G = view(G);
    a.A = view(A);
    a.F = view(F);
    a.n_rows = n;
    a.tau = post_tau;
    a.cnt = cnt.p;
    a.overflow = ovf.p;
    constexpr int CAP = PF_CAP;
    a.cap = CAP;
    DevBuf<int32_t> pi(c, (size_t)std::max(n, 1) * CAP);
    DevBuf<double> pv(c, (size_t)std::max(n, 1) * CAP);
    a.Hi = pi.p;
    a.Hv = pv.p;
    std::vector<int32_t> ovf_rows;
    if (n) {
        // single pass into the padded buffer (prefetching tier, 128-slot tables)
        Prof pr(c, "product", 12.0 * (G.nnz + A.nnz + F.nnz) + 12.0 * G.n_rows * 35);
        EDFA_CUDA(cudaMemsetAsync(ovf.p, 0, sizeof(int), c->stream));
        launch_product_pf(c, a);
        ovf_rows = read_overflow(c, ovf.p);
    }
    // first-tier counts (0 for the rows re-run below): what k_unpad copies from
    // the first padded buffer -- the re-runs overwrite cnt with their own counts
    DevBuf<int32_t> cnt1(c, std::max(n, 1));
    if (n) EDFA_CUDA(cudaMemcpyAsync(cnt1.p, cnt.p, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, c->stream));
    // rows beyond the first tier: 1024-slot tables into a second padded
    // buffer (by list position); rows beyond that: 4096-slot count + fill
    constexpr int CAP2 = 512;
    DevBuf<int32_t> rows1(c, std::max<size_t>(ovf_rows.size(), 1)), rows2(c, 1);
    DevBuf<int32_t> pi2;
    DevBuf<double> pv2;
    std::vector<int32_t> ovf2;
    ProdArgs b = a;
    if (!ovf_rows.empty()) {
        EDFA_CUDA(cudaMemcpyAsync(rows1.p, ovf_rows.data(), sizeof(int) * ovf_rows.size(), cudaMemcpyHostToDevice,
                                  c->stream));
        pi2.reset(c, ovf_rows.size() * CAP2);
        pv2.reset(c, ovf_rows.size() * CAP2);
        b.rows = rows1.p;
        b.n_list = (int32_t)ovf_rows.size();
        b.cap = CAP2;
        b.Hi = pi2.p;
        b.Hv = pv2.p;
        EDFA_CUDA(cudaMemsetAsync(ovf.p, 0, sizeof(int), c->stream));
        Prof pr(c, "product_wide", 12.0 * (G.nnz + A.nnz + F.nnz) * b.n_list / std::max(n, 1));
        launch_product<10, PADDED>(c, b);
        ovf2 = read_overflow(c, ovf.p);
    }
    DevBuf<int32_t> cnt2;   // second-tier counts (0 for the rows the third tier re-runs)
    if (!ovf2.empty()) {
        cnt2.reset(c, std::max(n, 1));
        EDFA_CUDA(cudaMemcpyAsync(cnt2.p, cnt.p, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, c->stream));
    }
    ProdArgs b3 = a;
    if (!ovf2.empty()) {
        rows2.reset(c, ovf2.size());
        EDFA_CUDA(cudaMemcpyAsync(rows2.p, ovf2.data(), sizeof(int) * ovf2.size(), cudaMemcpyHostToDevice,
                                  c->stream));
        b3.rows = rows2.p;
        b3.n_list = (int32_t)ovf2.size();
        EDFA_CUDA(cudaMemsetAsync(ovf.p, 0, sizeof(int), c->stream));
        Prof pr(c, "product_wide", 12.0 * (G.nnz + A.nnz + F.nnz) * b3.n_list / std::max(n, 1));
        launch_product<12, COUNT>(c, b3);
        require(read_overflow(c, ovf.p).empty(), EDFA_ERR_UNSUPPORTED, "H~ row exceeds 4096 distinct columns");
    }
    H.nnz = scan_counts(c, cnt.p, H.ptr.p, n);
    H.idx.reset(c, H.nnz);
    H.val.reset(c, H.nnz);
    if (n) {
        Prof pr(c, "product_unpad", 24.0 * H.nnz + 8.0 * n);
        k_unpad<<<ceil_div((int64_t)n * 32, 256), 256, 0, c->stream>>>(cnt1.p, H.ptr.p, n, CAP, pi.p, pv.p, H.idx.p,
                                                                      H.val.p);
        check_launch("k_unpad");
    }
    if (!ovf_rows.empty()) {
        const int nl = (int)ovf_rows.size();
        k_unpad_list<<<ceil_div((int64_t)nl * 32, 256), 256, 0, c->stream>>>(rows1.p, nl, ovf2.empty() ? cnt.p : cnt2.p,
                                                                            H.ptr.p, CAP2, pi2.p, pv2.p, H.idx.p,
                                                                            H.val.p);
        check_launch("k_unpad_list");
    }
    if (!ovf2.empty()) {
        b3.Hp = H.ptr.p;
        b3.Hi = H.idx.p;
        b3.Hv = H.val.p;
        EDFA_CUDA(cudaMemsetAsync(ovf.p, 0, sizeof(int), c->stream));
        Prof pr(c, "product_wide", 12.0 * (G.nnz + A.nnz + F.nnz) * b3.n_list / std::max(n, 1));
        launch_product<12, FILL>(c, b3);
        require(read_overflow(c, ovf.p).empty(), EDFA_ERR_UNSUPPORTED, "H~ row exceeds 4096 distinct columns");
    }
}

}  // namespace edfa
