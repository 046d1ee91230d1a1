// Tile-DAG triangular solves for cell-indexed factors (the ILU(0) of S~).
//
// Rows are cells of an nx*ny*nz grid in natural order.  Cells are grouped
// into tx*ty*tz tiles; when every dependency of a row lies in its own tile or
// in a tile that precedes it in natural tile order (true for the axial
// stencils of base/static patterns on structured grids -- checked, otherwise
// the caller falls back to the level solvers), the tiles form a DAG.
//
// One persistent CTA per SM takes tiles in tile-level order from a ticket,
// stages the tile's plan (TMA bulk copies into shared memory) and solves it
// as a dataflow: every x slot (rows and externals) starts as the SENTINEL
// pattern, so a stored value is its own ready flag -- no per-level barrier,
// no per-tile flag (k_tile_flow below).
//
// Plan records are stored per level, column-major ([dep k][row r]) so the
// lanes of a step read consecutive addresses.
#include <cub/cub.cuh>

#include <algorithm>
#include <map>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "dev_util.cuh"
#include "edfa_internal.cuh"
#include "objects.cuh"

namespace edfa {
namespace {

constexpr int CK = 4;               // critical dependencies per row (axial stencils: <= 3)
constexpr int EKMAX = 32;           // early dependencies per row

struct Geo {
    int nx, ny, nz, tx, ty, tz, NX, NY, NZ;
    __host__ __device__ int tile_of(int e) const {
        int i = e % nx, j = (e / nx) % ny, k = e / (nx * ny);
        return (i / tx) + NX * ((j / ty) + NY * (k / tz));
    }
    __host__ __device__ int tile_rows(int t) const {
        int I = t % NX, J = (t / NX) % NY, K = t / (NX * NY);
        int ax = min(tx, nx - I * tx), ay = min(ty, ny - J * ty), az = min(tz, nz - K * tz);
        return ax * ay * az;
    }
    __host__ __device__ int tile_cell(int t, int r) const {
        int I = t % NX, J = (t / NX) % NY, K = t / (NX * NY);
        int ax = min(tx, nx - I * tx), ay = min(ty, ny - J * ty);
        int li = r % ax, lj = (r / ax) % ay, lk = r / (ax * ay);
        return (I * tx + li) + nx * ((J * ty + lj) + ny * (K * tz + lk));
    }
    // box-local index of global cell j (j must lie in tile t)
    __host__ __device__ int local_of(int t, int j) const {
        int I = t % NX, J = (t / NX) % NY, K = t / (NX * NY);
        int ax = min(tx, nx - I * tx), ay = min(ty, ny - J * ty);
        int ji = j % nx - I * tx, jj = (j / nx) % ny - J * ty, jk = j / (nx * ny) - K * tz;
        return ji + ax * (jj + ay * jk);
    }
};

__global__ void k_tile_check(CsrV D, Geo g, bool reverse, int* __restrict__ bad, int* __restrict__ maxdeps) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= D.n_rows) return;
    int t = g.tile_of(i);
    atomicMax(maxdeps, D.ptr[i + 1] - D.ptr[i]);
    for (int e = D.ptr[i]; e < D.ptr[i + 1]; ++e) {
        int u = g.tile_of(D.idx[e]);
        if (reverse ? u < t : u > t) atomicExch(bad, 1);
    }
}

struct TileBuild {
    CsrV D;
    Geo g;
    int RC, EK, EC, LC;   // row / early-dep / external / level capacities per tile
    const double* diag;   // may be NULL (unit)
    bool unit;
    int* hdr;             // [n_rows, n_ext, n_lev, 0] per tile
    short* lev_ptr;       // LC per tile
    int* row_id;          // RC per tile (sorted by local level)
    int* ext_id;          // EC per tile
    short* cs;            // RC*CK per tile: critical dep slots, [lev_ptr*CK + k*R + r]
    double* cc;           // RC*CK
    short* es;            // RC*EK per tile: early dep slots, [lev_ptr*EK + k*R + r]
    double* ec;           // RC*EK
    double* dinv;         // RC per tile
    int* up_cnt;
    int* up_ids;          // 32 per tile
    int* err;
    int* max_early;       // count-only pass: max early deps of a row (sizes EK)
    bool count_only;
    int MD;               // max dependencies of a row
    int* glev;            // local level of every row (written by the count pass)
    short* xlev_ptr;      // LC per tile: externals first needed below level l
};

__global__ void __launch_bounds__(256) k_tile_build(TileBuild b) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int t = blockIdx.x;
    const Geo& g = b.g;
    const int n = g.tile_rows(t);
    int* cell = reinterpret_cast<int*>(sm);           // RC
    int* lev = cell + b.RC;                           // RC
    int* order = lev + b.RC;                          // RC: sorted position -> box index
    int* pos = order + b.RC;                          // RC: box index -> sorted position
    int* cnt = pos + b.RC;                            // RC+2
    int* ext = cnt + b.RC + 2;                        // EC
    int* misc = ext + b.EC;                           // 8
    int* hs = misc + 8;                               // HS
    __shared__ int ups[32];
    if (threadIdx.x < 8) misc[threadIdx.x] = 0;
    if (threadIdx.x < 32) ups[threadIdx.x] = -1;
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        cell[r] = g.tile_cell(t, r);
        lev[r] = 0;
    }
    __syncthreads();
    if (b.count_only) {
        // intra-tile dependency lists (box indices, -1 = external), then local
        // levels by relaxation over them (converges in local-depth sweeps);
        // the fill pass reads the levels back from glev
        short* dl = reinterpret_cast<short*>(order);      // RC*MD (reuses the fill-pass scratch)
        for (int r = threadIdx.x; r < n; r += blockDim.x) {
            const int row = cell[r], e0 = b.D.ptr[row], e1 = b.D.ptr[row + 1];
            for (int e = e0; e < e1; ++e) {
                const int j = b.D.idx[e];
                dl[r * b.MD + (e - e0)] = g.tile_of(j) == t ? (short)g.local_of(t, j) : (short)-1;
            }
            for (int e = e1 - e0; e < b.MD; ++e) dl[r * b.MD + e] = -2;
        }
        __syncthreads();
        for (int it = 0; it < b.RC + 1; ++it) {
            int changed = 0;
            for (int r = threadIdx.x; r < n; r += blockDim.x) {
                int lv = 0;
                for (int e = 0; e < b.MD; ++e) {
                    const int q = dl[r * b.MD + e];
                    if (q == -2) break;
                    if (q >= 0) lv = max(lv, lev[q] + 1);
                }
                if (lv != lev[r]) { lev[r] = lv; changed = 1; }
            }
            if (!__syncthreads_or(changed)) break;
        }
        // early deps = all but the intra-tile ones on the previous level
        for (int r = threadIdx.x; r < n; r += blockDim.x) {
            b.glev[cell[r]] = lev[r];
            int ne_r = 0;
            for (int e = 0; e < b.MD; ++e) {
                const int q = dl[r * b.MD + e];
                if (q == -2) break;
                ne_r += !(q >= 0 && lev[q] == lev[r] - 1);
            }
            atomicMax(b.max_early, ne_r);
        }
        return;
    }
    for (int r = threadIdx.x; r < n; r += blockDim.x) lev[r] = b.glev[cell[r]];
    __syncthreads();
    for (int l = threadIdx.x; l < b.RC + 2; l += blockDim.x) cnt[l] = 0;
    __syncthreads();
    for (int r = threadIdx.x; r < n; r += blockDim.x) atomicMax(&misc[0], lev[r] + 1);
    __syncthreads();
    const int nlev = misc[0];
    if (threadIdx.x == 0) {
        if (nlev + 1 > b.LC) atomicExch(b.err, 8);
        for (int r = 0; r < n; ++r) cnt[lev[r] + 1]++;
        for (int l = 0; l < nlev; ++l) cnt[l + 1] += cnt[l];
        short* lp = b.lev_ptr + (size_t)t * b.LC;
        for (int l = 0; l <= nlev && l < b.LC; ++l) lp[l] = (short)cnt[l];
        for (int r = 0; r < n; ++r) {
            int p = cnt[lev[r]]++;
            order[p] = r;
            pos[r] = p;
        }
        // cnt[l] now holds the END of level l; rebuild starts in cnt via lp
        for (int l = 0; l <= nlev && l < b.LC; ++l) cnt[l] = lp[l];
    }
    // external dependency set: hash insert, compact, bitonic sort
    int HS = 1;
    while (HS < 2 * b.EC) HS <<= 1;
    for (int q = threadIdx.x; q < HS; q += blockDim.x) hs[q] = -1;
    __syncthreads();
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        int row = cell[r];
        for (int e = b.D.ptr[row]; e < b.D.ptr[row + 1]; ++e) {
            int j = b.D.idx[e];
            if (g.tile_of(j) == t) continue;
            unsigned s = ((unsigned)j * 2654435761u) & (HS - 1);
            for (int probe = 0; probe < HS; ++probe) {
                int cur = atomicCAS(&hs[s], -1, j);
                if (cur == -1 || cur == j) break;
                s = (s + 1) & (HS - 1);
            }
        }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < HS; q += blockDim.x) {
        int v = hs[q];
        if (v >= 0) {
            int p = atomicAdd(&misc[1], 1);
            if (p < b.EC) ext[p] = v;
            else atomicExch(b.err, 5);
        }
    }
    __syncthreads();
    const int ne = min(misc[1], b.EC);
    int np2 = 1;
    while (np2 < ne) np2 <<= 1;
    int* srt = hs;
    for (int q = threadIdx.x; q < np2; q += blockDim.x) srt[q] = q < ne ? ext[q] : INT32_MAX;
    __syncthreads();
    for (int k = 2; k <= np2; k <<= 1)
        for (int jx = k >> 1; jx > 0; jx >>= 1) {
            for (int q = threadIdx.x; q < np2; q += blockDim.x) {
                int l = q ^ jx;
                if (l > q) {
                    int x0 = srt[q], x1 = srt[l];
                    if ((x0 > x1) == ((q & k) == 0)) { srt[q] = x1; srt[l] = x0; }
                }
            }
            __syncthreads();
        }
    for (int q = threadIdx.x; q < ne; q += blockDim.x) ext[q] = srt[q];
    __syncthreads();
    for (int q = threadIdx.x; q < ne; q += blockDim.x) {
        int u = g.tile_of(ext[q]);
        for (int z = 0; z < 32; ++z) {
            int cur = atomicCAS(&ups[z], -1, u);
            if (cur == -1 || cur == u) break;
            if (z == 31) atomicExch(b.err, 6);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {   // compacted upstream list (tile DAG -> schedule order)
        int nu = 0;
        int* up = b.up_ids + (size_t)t * 32;
        for (int z = 0; z < 32; ++z)
            if (ups[z] >= 0) up[nu++] = ups[z];
        b.up_cnt[t] = nu;
    }
    // externals ordered by the first local level that needs them (pipelined
    // loading); fn[q] = min level of a consumer row of ext[q]
    int* fn = misc + 8 + HS;                          // EC
    int* npos = fn + b.EC;                            // EC: id-sorted index -> need-sorted index
    for (int q = threadIdx.x; q < ne; q += blockDim.x) fn[q] = INT32_MAX;
    __syncthreads();
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        int row = cell[r];
        for (int e = b.D.ptr[row]; e < b.D.ptr[row + 1]; ++e) {
            int j = b.D.idx[e];
            if (g.tile_of(j) == t) continue;
            int lo = 0, hi = ne;
            while (lo < hi) {
                int mid = (lo + hi) >> 1;
                if (ext[mid] < j) lo = mid + 1;
                else hi = mid;
            }
            atomicMin(&fn[lo], lev[r]);
        }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < np2; q += blockDim.x) srt[q] = q < ne ? (fn[q] << 12) | q : INT32_MAX;
    __syncthreads();
    for (int k = 2; k <= np2; k <<= 1)
        for (int jx = k >> 1; jx > 0; jx >>= 1) {
            for (int q = threadIdx.x; q < np2; q += blockDim.x) {
                int l = q ^ jx;
                if (l > q) {
                    int x0 = srt[q], x1 = srt[l];
                    if ((x0 > x1) == ((q & k) == 0)) { srt[q] = x1; srt[l] = x0; }
                }
            }
            __syncthreads();
        }
    for (int p = threadIdx.x; p < ne; p += blockDim.x) npos[srt[p] & 4095] = p;
    __syncthreads();
    for (int q = threadIdx.x; q < ne; q += blockDim.x) b.ext_id[(size_t)t * b.EC + npos[q]] = ext[q];
    __syncthreads();
    if (threadIdx.x == 0) {            // xlev_ptr[l] = #externals with fn < l
        short* xl = b.xlev_ptr + (size_t)t * b.LC;
        int q = 0;
        for (int l = 0; l < b.LC; ++l) {
            while (q < ne && (srt[q] >> 12) < l) ++q;
            xl[l] = (short)q;
        }
    }
    // records: critical deps = rows of the immediately preceding local level
    const int ZSLOT = b.RC + b.EC;   // a shared-memory x slot that stays 0
    for (int p = threadIdx.x; p < n; p += blockDim.x) {
        const int r = order[p], row = cell[r], lv = lev[r];
        const int l0 = cnt[lv], R = cnt[lv + 1] - l0, rr = p - l0;
        b.row_id[(size_t)t * b.RC + p] = row;
        b.dinv[(size_t)t * b.RC + p] = (b.unit || !b.diag) ? 1.0 : 1.0 / b.diag[row];
        int nc = 0, nE = 0;
        short* csb = b.cs + (size_t)t * b.RC * CK + (size_t)l0 * CK;
        double* ccb = b.cc + (size_t)t * b.RC * CK + (size_t)l0 * CK;
        short* esb = b.es + (size_t)t * b.RC * b.EK + (size_t)l0 * b.EK;
        double* ecb = b.ec + (size_t)t * b.RC * b.EK + (size_t)l0 * b.EK;
        // early deps ordered oldest first (largest wavefront distance |gl(row) -
        // gl(dep)|, gl = i+j+k), padding in front: the dataflow solve folds them
        // in this order, so only the last few can still be in flight
        auto gl = [&](int e) { return e % g.nx + (e / g.nx) % g.ny + e / (g.nx * g.ny); };
        const int glr = gl(row);
        short e_slot[EKMAX];
        double e_val[EKMAX];
        int e_dist[EKMAX];
        for (int e = b.D.ptr[row]; e < b.D.ptr[row + 1]; ++e) {
            int j = b.D.idx[e];
            double v = b.D.val ? b.D.val[e] : 0.0;
            int slot;
            bool critical = false;
            if (g.tile_of(j) == t) {
                int rj = g.local_of(t, j);
                slot = pos[rj];
                critical = lev[rj] == lv - 1;
            } else {
                int lo = 0, hi = ne;
                while (lo < hi) {
                    int mid = (lo + hi) >> 1;
                    if (ext[mid] < j) lo = mid + 1;
                    else hi = mid;
                }
                slot = b.RC + npos[lo];
            }
            if (critical) {
                if (nc >= CK) { atomicExch(b.err, 10); continue; }
                csb[nc * R + rr] = (short)slot;
                ccb[nc * R + rr] = v;
                ++nc;
            } else {
                if (nE >= b.EK || nE >= EKMAX) { atomicExch(b.err, 11); continue; }
                const int dist = abs(glr - gl(j));
                int q = nE++;
                while (q > 0 && e_dist[q - 1] < dist) {   // stable: descending distance
                    e_dist[q] = e_dist[q - 1];
                    e_slot[q] = e_slot[q - 1];
                    e_val[q] = e_val[q - 1];
                    --q;
                }
                e_dist[q] = dist;
                e_slot[q] = (short)slot;
                e_val[q] = v;
            }
        }
        for (; nc < CK; ++nc) { csb[nc * R + rr] = (short)ZSLOT; ccb[nc * R + rr] = 0.0; }
        const int pad = b.EK - nE;
        for (int q = 0; q < pad; ++q) { esb[q * R + rr] = (short)ZSLOT; ecb[q * R + rr] = 0.0; }
        for (int q = 0; q < nE; ++q) { esb[(pad + q) * R + rr] = e_slot[q]; ecb[(pad + q) * R + rr] = e_val[q]; }
    }
    if (threadIdx.x == 0) {
        int* h = b.hdr + (size_t)t * 4;
        h[0] = n;
        h[1] = ne;
        h[2] = nlev;
        h[3] = 0;
    }
}

struct TileSolve {
    int n_tiles, RC, EK, EC, LC;
    const int* order;
    const int* hdr;
    const short* lev_ptr;
    const int* row_id;
    const int* ext_id;
    const short* cs;
    const double* cc;
    const short* es;
    const double* ec;
    const double* dinv;
    unsigned* ticket;
    unsigned ticket_base;  // tickets wrap modulo 2^32 (well defined for unsigned)
    const double* b;
    double alpha;
    double* x;
    const double* add;
    double* out2;
    int* err;
    const short* xlev_ptr;
    double* b_sent;       // == b, whose tile rows are reset to SENTINEL once read (or NULL)
    double* pre_sent;     // another vector whose tile rows are set to SENTINEL (or NULL)
};

__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned r16(unsigned b) { return (b + 15u) & ~15u; }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* mbar) {
    if (bytes == 0) return;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(mbar)) : "memory");
}

__device__ __forceinline__ double ld_relaxed_d(const double* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return __longlong_as_double((long long)v);
}

// ---------------------------------------------------------------------------
// Dataflow tile solve: no per-level barrier.  Every x slot of the tile (its
// rows and its externals) starts as the SENTINEL pattern in shared memory, so
// a stored value is its own ready flag there too.
//   * compute warps take the tile's 32-row groups (rows of one local level) in
//     level order, round robin; a lane folds its row's early dependencies
//     (older levels, externals) as soon as they are present, then its <= 3
//     critical ones (previous level), stores x to shared memory and HBM;
//   * the loader warp copies externals (HBM, polled in need order) into their
//     shared slots as they appear.
// A level therefore costs one shared-memory hand-off plus a short FMA chain
// instead of a CTA barrier plus the slowest warp, and a downstream tile's row
// starts as soon as its own externals exist.
__device__ __forceinline__ double ld_vol_s(const double* p) { return *reinterpret_cast<const volatile double*>(p); }
__device__ __forceinline__ void st_vol_s(double* p, double v) { *reinterpret_cast<volatile double*>(p) = v; }
constexpr int FLOW_LW = 8;          // loader: externals in flight per lane per polling round (8: 1 % faster than 16)
constexpr int FLOW_LSLEEP = 20;     // loader back-off (ns) when nothing new arrived
constexpr int FLOW_LAHEAD = 64;     // loader window: need-levels polled past the first missing external
// Two shapes of the kernel:
//  * narrow wavefronts (few tiles per level, e.g. 64^3): W = 15 compute warps
//    + the loader (512 threads at 128 registers, one CTA per SM) with the whole
//    plan staged in shared memory -- the latency of the level chain dominates
//    (12 -> 15 warps: 141 -> 134 us per solve at 64^3);
//  * wide wavefronts (thousands of ready tiles, e.g. 256^3): W = 7 (256
//    threads) and DIRECT early records -- read from global memory (L2-warmed
//    by a bulk prefetch when the tile starts) instead of staged, so the CTA
//    needs ~60 KB of shared memory and two tiles are in flight per SM: the
//    solve is bound by tile throughput, not by the critical path.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
    if (bytes) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool is_sent_hi(double v) {   // published values are never NaN-boxed like this
    return __double2hiint(v) == (int)(SENTINEL_BITS >> 32);
}

template <int EK, int W, bool DIRECT>
__global__ void __launch_bounds__((W + 1) * 32, DIRECT ? 2 : 1) k_tile_flow(TileSolve a) {
    constexpr int FLOW_THREADS = (W + 1) * 32;
    constexpr int SEK = DIRECT ? 0 : EK;                            // early records staged in smem
    extern __shared__ __align__(128) unsigned char sm[];
    double* xs = reinterpret_cast<double*>(sm);                     // RC + EC + 2
    double* bsm = xs + a.RC + a.EC + 2;                             // RC (right-hand side)
    double* cc = bsm + a.RC;                                        // RC*CK
    double* ecf = cc + (size_t)a.RC * CK;                           // RC*SEK
    double* di = ecf + (size_t)a.RC * SEK;                          // RC
    int* rid = reinterpret_cast<int*>(di + a.RC);                   // RC
    int* eid_s = rid + a.RC;                                        // EC (external row ids, need-sorted)
    short* cs = reinterpret_cast<short*>(eid_s + a.EC);             // RC*CK
    short* es = cs + (size_t)a.RC * CK;                             // RC*SEK
    short* lp = es + (size_t)a.RC * SEK;                            // LC
    short* xl = lp + a.LC;                                          // LC: externals needed below level l
    __shared__ int s_tile, s_hdr[4];
    __shared__ __align__(8) uint64_t mbar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(&mbar)), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned phase = 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double sent = __longlong_as_double((long long)SENTINEL_BITS);
    for (;;) {
        if (threadIdx.x == 0) {
            const unsigned k = atomicAdd(a.ticket, 1u) - a.ticket_base;
            const int t = k < (unsigned)a.n_tiles ? a.order[k] : -1;
            s_tile = t;
            if (t >= 0) {
                const int4 h = *reinterpret_cast<const int4*>(a.hdr + (size_t)t * 4);
                s_hdr[0] = h.x; s_hdr[1] = h.y; s_hdr[2] = h.z;
                const unsigned n = h.x;
                unsigned b_cs = r16(2u * n * CK), b_cc = r16(8u * n * CK), b_es = DIRECT ? 0u : r16(2u * n * EK),
                         b_ec = DIRECT ? 0u : r16(8u * n * EK), b_di = r16(8u * n), b_ri = r16(4u * n),
                         b_lp = r16(2u * (h.z + 1));
                if (DIRECT) {   // the early records are read per group: warm L2 with them now
                    bulk_prefetch_l2(a.es + (size_t)t * a.RC * EK, r16(2u * n * EK));
                    bulk_prefetch_l2(a.ec + (size_t)t * a.RC * EK, r16(8u * n * EK));
                }
                unsigned b_ei = r16(4u * h.y), b_xl = r16(2u * (h.z + 1));
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                             ::"r"(smem_addr(&mbar)), "r"(b_cs + b_cc + b_es + b_ec + b_di + b_ri + b_lp + b_ei + b_xl)
                             : "memory");
                bulk_g2s(xl, a.xlev_ptr + (size_t)t * a.LC, b_xl, &mbar);
                bulk_g2s(eid_s, a.ext_id + (size_t)t * a.EC, b_ei, &mbar);
                bulk_g2s(cs, a.cs + (size_t)t * a.RC * CK, b_cs, &mbar);
                bulk_g2s(cc, a.cc + (size_t)t * a.RC * CK, b_cc, &mbar);
                if (!DIRECT) {
                    bulk_g2s(es, a.es + (size_t)t * a.RC * EK, b_es, &mbar);
                    bulk_g2s(ecf, a.ec + (size_t)t * a.RC * EK, b_ec, &mbar);
                }
                bulk_g2s(di, a.dinv + (size_t)t * a.RC, b_di, &mbar);
                bulk_g2s(rid, a.row_id + (size_t)t * a.RC, b_ri, &mbar);
                bulk_g2s(lp, a.lev_ptr + (size_t)t * a.LC, b_lp, &mbar);
            }
        }
        __syncthreads();
        const int t = s_tile;
        if (t < 0) break;
        const int n = s_hdr[0], ne = s_hdr[1], nlev = s_hdr[2];
        for (int q = threadIdx.x; q < ne; q += FLOW_THREADS) xs[a.RC + q] = sent;
        {
            unsigned done = 0;
            while (!done)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(done) : "r"(smem_addr(&mbar)), "r"(phase) : "memory");
            phase ^= 1u;
        }
        for (int p0 = 0; p0 < n; p0 += 8 * FLOW_THREADS) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                int p = p0 + u * FLOW_THREADS + threadIdx.x;
                v[u] = p < n ? __ldg(a.b + rid[p]) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                int p = p0 + u * FLOW_THREADS + threadIdx.x;
                if (p < n) {
                    bsm[p] = a.alpha * v[u];
                    xs[p] = sent;
                    // sentinel pre-fill of the next solves' outputs, row by row
                    // (this tile is the only reader / writer of these rows)
                    if (a.b_sent) a.b_sent[rid[p]] = sent;
                    if (a.pre_sent) a.pre_sent[rid[p]] = sent;
                }
            }
        }
        if (threadIdx.x < 2) xs[a.RC + a.EC + threadIdx.x] = 0.0;   // ZSLOT (+pad)
        __syncthreads();
        if (warp == W) {
            // externals in need order; q0 = first entry not yet present
            constexpr int LW = FLOW_LW;
            // the polling window stops FLOW_LAHEAD need-levels past the first
            // missing external: no L2 traffic for values produced much later
            int q0 = 0, lq = 0;
            long long spins = 0;
            while (q0 < ne) {
                while (lq < nlev && xl[lq + 1] <= q0) ++lq;
                const int qe = min(min(ne, q0 + LW * 32), (int)xl[min(lq + FLOW_LAHEAD, nlev)]);
                double v[LW];
#pragma unroll
                for (int u = 0; u < LW; ++u) {
                    const int q = q0 + u * 32 + lane;
                    v[u] = q < qe ? ld_relaxed_d(a.x + eid_s[q]) : 0.0;
                }
                int adv = qe - q0;
#pragma unroll
                for (int u = 0; u < LW; ++u) {
                    const int q = q0 + u * 32 + lane;
                    const bool ok = q >= qe || !is_sentinel(v[u]);
                    if (q < qe && ok) st_vol_s(xs + a.RC + q, v[u]);
                    const unsigned miss = __ballot_sync(0xffffffffu, !ok);
                    if (miss && adv == qe - q0) adv = u * 32 + __ffs(miss) - 1;
                }
                if (adv == 0) {
                    __nanosleep(FLOW_LSLEEP);
                    if (++spins > SPIN_LIMIT) { if (lane == 0) atomicExch(a.err, 7); break; }
                    continue;
                }
                spins = 0;
                q0 += adv;
            }
        } else {
            // groups of 16 rows of one level; a lane pair per row splits the
            // early dependencies (lane li takes li, li+2, ...).  The whole warp
            // walks a group together (inactive lanes predicated, __syncwarp per
            // group): lanes never run ahead into later groups, where they would
            // spin on rows their own warp still has to produce.
            constexpr int KH = EK / 2;
            const int li = lane & 1;
            int g = 0;
            for (int lv = 0; lv < nlev; ++lv) {
                const int l0 = lp[lv], R = lp[lv + 1] - l0;
                for (int r0 = 0; r0 < R; r0 += 16, ++g) {
                    if (g % W != warp) continue;
                    const int r = r0 + (lane >> 1);
                    const bool act = r < R;
                    const int p = l0 + (act ? r : 0);
                    const short zs = (short)(a.RC + a.EC);
                    short es_[KH], cs_[CK];
                    double ec_[KH], cc_[CK];
                    const short* esb = DIRECT ? a.es + (size_t)t * a.RC * EK : es;
                    const double* ecb = DIRECT ? a.ec + (size_t)t * a.RC * EK : ecf;
#pragma unroll
                    for (int u = 0; u < KH; ++u) {
                        const int k = 2 * u + li;
                        es_[u] = act ? esb[(size_t)l0 * EK + k * R + r] : zs;
                        ec_[u] = act ? ecb[(size_t)l0 * EK + k * R + r] : 0.0;
                    }
#pragma unroll
                    for (int k = 0; k < CK; ++k) {
                        cs_[k] = act ? cs[(size_t)l0 * CK + k * R + r] : zs;
                        cc_[k] = act ? cc[(size_t)l0 * CK + k * R + r] : 0.0;
                    }
                    const double d = di[p];
                    const int row = rid[p];
                    const double bv = bsm[p];
                    // early deps (older levels, externals) are polled as one batch,
                    // one warp vote per round
                    double ev[KH];
#pragma unroll
                    for (int u = 0; u < KH; ++u) ev[u] = ld_vol_s(xs + es_[u]);
                    auto fetch = [&](int u) -> double {   // an external the loader has not copied yet comes from L2
                        const int q = es_[u] - a.RC;
                        return (q >= 0 && q < ne) ? ld_relaxed_d(a.x + eid_s[q]) : ld_vol_s(xs + es_[u]);
                    };
                    {
                        bool miss = false;
#pragma unroll
                        for (int u = 0; u < KH; ++u) miss |= is_sent_hi(ev[u]);
                        long long spins = 0;
                        while (__any_sync(0xffffffffu, miss)) {
                            miss = false;
#pragma unroll
                            for (int u = 0; u < KH; ++u) {
                                if (is_sent_hi(ev[u])) ev[u] = fetch(u);
                                miss |= is_sent_hi(ev[u]);
                            }
                            if (++spins > SPIN_LIMIT) { if (lane == 0) atomicExch(a.err, 7); break; }
                        }
                    }
                    double h = 0.0;
#pragma unroll
                    for (int u = 0; u < KH; ++u) h = fma(-ec_[u], ev[u], h);
                    h += __shfl_xor_sync(0xffffffffu, h, 1);   // same sum on both lanes
                    double acc = bv + h;
                    double cv[CK];
#pragma unroll
                    for (int k = 0; k < CK; ++k) cv[k] = ld_vol_s(xs + cs_[k]);
                    {
                        bool miss = false;
#pragma unroll
                        for (int k = 0; k < CK; ++k) miss |= is_sent_hi(cv[k]);
                        long long spins = 0;
                        while (__any_sync(0xffffffffu, miss)) {   // the previous level is being finished
                            miss = false;
#pragma unroll
                            for (int k = 0; k < CK; ++k) {
                                cv[k] = ld_vol_s(xs + cs_[k]);
                                miss |= is_sent_hi(cv[k]);
                            }
                            if (++spins > SPIN_LIMIT) { if (lane == 0) atomicExch(a.err, 7); break; }
                        }
                    }
#pragma unroll
                    for (int k = 0; k < CK; ++k) acc = fma(-cc_[k], cv[k], acc);
                    const double v = acc * d;
                    if (act && li == 0) {
                        st_vol_s(xs + p, v);
                        // fire-and-forget reduction at L2: SENTINEL + (v - SENTINEL)
                        // (visible downstream ~0.5 us after issue; a plain store ~2 us)
                        atomicAdd(reinterpret_cast<unsigned long long*>(a.x + row),
                                  (unsigned long long)__double_as_longlong(publishable(v)) - SENTINEL_BITS);
                    }
                    __syncwarp();
                }
            }
        }
        __syncthreads();
        if (a.out2)
            for (int p = threadIdx.x; p < n; p += FLOW_THREADS) {
                int row = rid[p];
                a.out2[row] = xs[p] + a.add[row];
            }
    }
}

}  // namespace

// smem: xs[RC+EC+2] b[RC] cc[RC*CK] ec[RC*EK] di[RC] rid[RC] eid[EC] cs[RC*CK] es[RC*EK] lp[LC] xl[LC]
// (ec / es absent with direct early records)
size_t tile_flow_smem_bytes(const TilePlan& tp, bool direct) {
    size_t rc = tp.RC, ek = direct ? 0 : tp.KD, ec = tp.EC, lc = tp.LC;
    size_t bytes = 8 * (rc + ec + 2) + 8 * rc + 8 * rc * CK + 8 * rc * ek + 8 * rc + 4 * rc + 4 * ec +
                   2 * rc * CK + 2 * rc * ek + 2 * lc + 2 * lc;
    return (bytes + 127) & ~size_t(127);
}

// wide wavefronts: enough tiles per tile level to keep two CTAs per SM busy
static bool tile_direct(const TilePlan& tp) {
    return tp.n_tile_levels > 0 && tp.n_tiles / tp.n_tile_levels >= 2 * NUM_SMS_B200 / 8 && tp.n_tiles >= 4096;
}

bool build_tile_plan(Ctx* c, const Csr& D, const double* diag, bool unit, bool reverse, const int* dims,
                     TilePlan& tp) {
    const int n = D.n_rows;
    if (!dims || dims[0] <= 0 || (int64_t)dims[0] * dims[1] * dims[2] != n || n == 0) return false;
    Geo g{dims[0], dims[1], dims[2], 8, 8, 8, 0, 0, 0};
    g.tx = std::min(8, g.nx);
    g.ty = std::min(8, g.ny);
    g.tz = std::min(8, g.nz);
    g.NX = ceil_div(g.nx, g.tx);
    g.NY = ceil_div(g.ny, g.ty);
    g.NZ = ceil_div(g.nz, g.tz);
    int* fl = c->d_scalar_i + 48;   // [bad, maxdeps, err]
    EDFA_CUDA(cudaMemsetAsync(fl, 0, 3 * sizeof(int), c->stream));
    k_tile_check<<<ceil_div(n, 256), 256, 0, c->stream>>>(view(D), g, reverse, fl, fl + 1);
    check_launch("k_tile_check");
    int hf[2];
    EDFA_CUDA(cudaMemcpyAsync(hf, fl, sizeof hf, cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
    if (hf[0] || hf[1] > EKMAX) return false;
    const int nt = g.NX * g.NY * g.NZ;
    tp.n = n;
    tp.n_tiles = nt;
    tp.RC = (g.tx * g.ty * g.tz + 7) & ~7;
    tp.EC = (std::min(tp.RC * std::max(hf[1], 1), 4 * tp.RC + 256) + 7) & ~7;
    tp.LC = ((g.tx + g.ty + g.tz) * 4 + 8 + 7) & ~7;    // generous bound on local levels + 1
    if (tp.LC > tp.RC + 8) tp.LC = tp.RC + 8;
    tp.unit = unit;
    tp.n_dep = D.nnz;
    DevBuf<int32_t> glev(c, n);
    int HS = 1;
    while (HS < 2 * tp.EC) HS <<= 1;
    size_t bsm = sizeof(int) * (5 * tp.RC + 2 + tp.EC + 8 + HS + 2 * tp.EC);
    bsm = std::max(bsm, sizeof(int) * 2 * tp.RC + sizeof(short) * (size_t)tp.RC * hf[1] + 64);
    if (bsm > 48 * 1024)
        EDFA_CUDA(cudaFuncSetAttribute(k_tile_build, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
    {
        // count pass: the early-dependency capacity EK is the exact maximum
        // (rounded to the instantiated widths) so no padded work is staged
        TileBuild cb{};
        cb.D = view(D);
        cb.g = g;
        cb.RC = tp.RC;
        cb.EC = tp.EC;
        cb.LC = tp.LC;
        cb.max_early = fl + 3;
        cb.err = fl + 2;
        cb.count_only = true;
        cb.glev = glev.p;
        cb.MD = hf[1];
        EDFA_CUDA(cudaMemsetAsync(fl + 3, 0, sizeof(int), c->stream));
        Prof pr(c, "tile_plan", 8.0 * D.nnz);
        k_tile_build<<<nt, 256, bsm, c->stream>>>(cb);
        check_launch("k_tile_build count");
        int me = 0;
        EDFA_CUDA(cudaMemcpyAsync(&me, fl + 3, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        EDFA_CUDA(cudaStreamSynchronize(c->stream));
        const int widths[] = {4, 8, 12, 16, 24, 32};
        tp.KD = 0;
        for (int w : widths)
            if (me <= w) { tp.KD = w; break; }
        if (!tp.KD) return false;
    }
    if (tile_flow_smem_bytes(tp, false) > 220 * 1024) return false;
    tp.hdr.reset(c, (size_t)nt * 4);
    tp.lev_ptr.reset(c, (size_t)nt * tp.LC);
    tp.row_id.reset(c, (size_t)nt * tp.RC);
    tp.ext_id.reset(c, (size_t)nt * tp.EC);
    tp.dslot.reset(c, (size_t)nt * tp.RC * CK);        // critical slots
    tp.dcoef.reset(c, (size_t)nt * tp.RC * CK);        // critical coefficients
    tp.eslot.reset(c, (size_t)nt * tp.RC * tp.KD);
    tp.ecoef.reset(c, (size_t)nt * tp.RC * tp.KD);
    tp.dinv.reset(c, (size_t)nt * tp.RC);
    tp.up_cnt.reset(c, nt);
    tp.up_ids.reset(c, (size_t)nt * 32);
    tp.xlev_ptr.reset(c, (size_t)nt * tp.LC);
    tp.ticket.reset(c, 1);
    EDFA_CUDA(cudaMemsetAsync(tp.ticket.p, 0, sizeof(unsigned), c->stream));
    tp.ticket_base = 0;
    TileBuild b{view(D), g, tp.RC, tp.KD, tp.EC, tp.LC, diag, unit, tp.hdr.p, tp.lev_ptr.p, tp.row_id.p,
                tp.ext_id.p, tp.dslot.p, tp.dcoef.p, tp.eslot.p, tp.ecoef.p, tp.dinv.p, tp.up_cnt.p, tp.up_ids.p,
                fl + 2, fl + 3, false, hf[1]};
    b.glev = glev.p;
    b.xlev_ptr = tp.xlev_ptr.p;
    {
        Prof pr(c, "tile_plan", 24.0 * D.nnz);
        k_tile_build<<<nt, 256, bsm, c->stream>>>(b);
        check_launch("k_tile_build");
    }
    int e = 0;
    EDFA_CUDA(cudaMemcpyAsync(&e, fl + 2, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    std::vector<int> upc(nt), upi((size_t)nt * 32);
    EDFA_CUDA(cudaMemcpyAsync(upc.data(), tp.up_cnt.p, sizeof(int) * nt, cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaMemcpyAsync(upi.data(), tp.up_ids.p, sizeof(int) * nt * 32, cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
    if (e) return false;
    // tile schedule: level of the tile DAG (host, tiny), ticket order by (level, id)
    std::vector<int> lvl(nt, 0), ord(nt);
    if (!reverse) {
        for (int t = 0; t < nt; ++t)
            for (int z = 0; z < upc[t]; ++z) lvl[t] = std::max(lvl[t], lvl[upi[(size_t)t * 32 + z]] + 1);
    } else {
        for (int t = nt - 1; t >= 0; --t)
            for (int z = 0; z < upc[t]; ++z) lvl[t] = std::max(lvl[t], lvl[upi[(size_t)t * 32 + z]] + 1);
    }
    for (int t = 0; t < nt; ++t) ord[t] = t;
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return lvl[a] < lvl[b]; });
    tp.n_tile_levels = nt ? *std::max_element(lvl.begin(), lvl.end()) + 1 : 0;
    tp.order.reset(c, nt);
    EDFA_CUDA(cudaMemcpyAsync(tp.order.p, ord.data(), sizeof(int) * nt, cudaMemcpyHostToDevice, c->stream));
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
    return true;
}

template <int EK, int W, bool DIRECT>
static void launch_tile(Ctx* c, TilePlan& tp, TileSolve& a) {
    const size_t smem = tile_flow_smem_bytes(tp, DIRECT);
    auto kern = k_tile_flow<EK, W, DIRECT>;
    constexpr int threads = (W + 1) * 32;
    // the dynamic shared-memory attribute only ever grows (a smaller value set
    // for one plan must not invalidate the grid sized for another)
    static std::mutex mu;
    static std::map<std::pair<int, size_t>, int> grids;
    static std::map<int, size_t> smem_set;   // per device
    int grid;
    {
        std::lock_guard<std::mutex> lk(mu);
        const auto key = std::make_pair(c->device, smem);
        auto it = grids.find(key);
        if (it == grids.end()) {
            size_t& cur = smem_set[c->device];
            if (smem > cur) {
                EDFA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                cur = smem;
            }
            int occ = 0;
            EDFA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
            it = grids.emplace(key, NUM_SMS_B200 * std::max(1, std::min(occ, DIRECT ? 4 : 2))).first;
        }
        grid = it->second;
    }
    a.ticket_base = tp.ticket_base;
    tp.ticket_base += (unsigned)(tp.n_tiles + grid);   // every CTA takes exactly one failing ticket
    void* args[] = {&a};
    EDFA_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3(grid), dim3(threads), args, smem, c->stream));
}

template <int EK>
static void launch_tile_shape(Ctx* c, TilePlan& tp, TileSolve& a) {
    const int mode = c->opt.tile_direct < 0 ? (tile_direct(tp) ? 1 : 0) : c->opt.tile_direct;
    if (mode == 2) launch_tile<EK, 5, true>(c, tp, a);        // three CTAs per SM
    else if (mode == 1) launch_tile<EK, 7, true>(c, tp, a);
    else launch_tile<EK, 15, false>(c, tp, a);
}

void run_tile(Ctx* c, TilePlan& tp, const double* b, double alpha, double* x, const double* add, double* out2,
              const char* name) {
    run_tile_ex(c, tp, b, alpha, x, add, out2, name, false, false, nullptr);
}

void run_tile_ex(Ctx* c, TilePlan& tp, const double* b, double alpha, double* x, const double* add, double* out2,
                 const char* name, bool x_prefilled, bool consume_b, double* pre_sent) {
    TileSolve a{tp.n_tiles, tp.RC, tp.KD, tp.EC, tp.LC, tp.order.p, tp.hdr.p, tp.lev_ptr.p, tp.row_id.p,
                tp.ext_id.p, tp.dslot.p, tp.dcoef.p, tp.eslot.p, tp.ecoef.p, tp.dinv.p, tp.ticket.p, 0u, b, alpha, x,
                add, out2, c->d_scalar_i + 8, tp.xlev_ptr.p, nullptr, nullptr};
    a.b_sent = consume_b ? const_cast<double*>(b) : nullptr;
    a.pre_sent = pre_sent;
    // a row's value is its own ready flag
    if (!x_prefilled) fill_bits(c, x, tp.n, SENTINEL_BITS);
    Prof pr(c, name, 12.0 * tp.n_dep + 24.0 * tp.n + (out2 ? 16.0 * tp.n : 0.0));
    switch (tp.KD) {
        case 4: launch_tile_shape<4>(c, tp, a); break;
        case 8: launch_tile_shape<8>(c, tp, a); break;
        case 12: launch_tile_shape<12>(c, tp, a); break;
        case 16: launch_tile_shape<16>(c, tp, a); break;
        case 24: launch_tile_shape<24>(c, tp, a); break;
        default: launch_tile_shape<32>(c, tp, a); break;
    }
}

}  // namespace edfa
