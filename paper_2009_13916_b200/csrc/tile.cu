// Tile-DAG triangular solves for cell-indexed factors (the ILU(0) of S~).
//
// Rows are cells of an nx*ny*nz grid in natural order.  Cells are grouped
// into tx*ty*tz tiles; when every dependency of a row lies in its own tile or
// in a tile that precedes it in natural tile order (true for the axial
// stencils of base/static patterns on structured grids -- checked, otherwise
// the caller falls back to the level-synchronous solver), the tiles form a
// DAG of depth ~ NX+NY+NZ instead of the row DAG's nx+ny+nz.
//
// One persistent CTA per SM takes tiles in tile-level order from a ticket:
//   1. stage the tile's coefficients (slots, values, 1/diag, level bounds)
//      from HBM into shared memory -- independent of the solve, so it runs
//      before the upstream wait;
//   2. wait for the upstream tiles' epoch flags (one poller per upstream);
//   3. gather the external dependencies of the tile into shared memory;
//   4. sweep the tile's local levels with __syncthreads between them, reading
//      every dependency from shared memory;
//   5. write the tile's solution to HBM and publish the tile's flag.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "dev_util.cuh"
#include "edfa_internal.cuh"
#include "objects.cuh"

namespace edfa {
namespace {

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
    // r-th cell (natural order inside the tile box) of tile t
    __host__ __device__ int tile_cell(int t, int r) const {
        int I = t % NX, J = (t / NX) % NY, K = t / (NX * NY);
        int ax = min(tx, nx - I * tx), ay = min(ty, ny - J * ty);
        int li = r % ax, lj = (r / ax) % ay, lk = r / (ax * ay);
        return (I * tx + li) + nx * ((J * ty + lj) + ny * (K * tz + lk));
    }
};

// every external dependency must lie in a tile before (forward) / after
// (backward) the row's tile in natural tile order
__global__ void k_tile_check(CsrV D, Geo g, bool reverse, int* __restrict__ bad, int* __restrict__ maxdeps) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= D.n_rows) return;
    int t = g.tile_of(i);
    int len = D.ptr[i + 1] - D.ptr[i];
    atomicMax(maxdeps, len);
    for (int e = D.ptr[i]; e < D.ptr[i + 1]; ++e) {
        int u = g.tile_of(D.idx[e]);
        if (reverse ? u < t : u > t) atomicExch(bad, 1);
    }
}

// Per-tile analysis: local levels, sort by level, external list, slot-mapped
// dependencies.  One CTA per tile; fixed per-tile capacities:
//   rows <= RC, deps <= RC*KD, externals <= EC.
struct TileBuild {
    CsrV D;
    Geo g;
    bool reverse;
    int RC, KD, EC;
    const double* diag;   // may be NULL (unit or values later)
    bool unit;
    // outputs, tile-major with the fixed capacities
    int* hdr;             // [n_rows, n_ext, n_lev, n_dep] per tile
    short* lev_ptr;       // RC+1 per tile
    int* row_id;          // RC per tile (sorted by local level)
    int* ext_id;          // EC per tile
    int* dptr;            // RC+1 per tile (local dep offsets)
    short* dslot;         // RC*KD per tile
    int* dsrc;            // RC*KD per tile: global CSR position of the dep (for value reloads)
    double* dcoef;        // RC*KD per tile
    double* dinv;         // RC per tile
    int* up_cnt;          // upstream tiles per tile (<= 26)
    int* up_ids;          // 32 per tile
    int* err;
};

__global__ void __launch_bounds__(512) k_tile_build(TileBuild b) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int t = blockIdx.x;
    const Geo& g = b.g;
    const int n = g.tile_rows(t);
    int* cell = reinterpret_cast<int*>(sm);           // RC: tile row r -> global row (box order)
    int* lev = cell + b.RC;                           // RC
    int* order = lev + b.RC;                          // RC: sorted position -> r
    int* pos = order + b.RC;                          // RC: r -> sorted position
    int* cnt = pos + b.RC;                            // RC+2 (level histogram)
    int* ext = cnt + b.RC + 2;                        // EC
    int* misc = ext + b.EC;                           // 8
    if (threadIdx.x < 8) misc[threadIdx.x] = 0;
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        cell[r] = g.tile_cell(t, r);
        lev[r] = 0;
    }
    __syncthreads();
    // local levels by relaxation (converges in local-depth sweeps)
    for (int it = 0; it < b.RC + 1; ++it) {
        int changed = 0;
        for (int r = threadIdx.x; r < n; r += blockDim.x) {
            int e0 = b.D.ptr[cell[r]], e1 = b.D.ptr[cell[r] + 1];
            int lv = 0;
            for (int e = e0; e < e1; ++e) {
                int j = b.D.idx[e];
                if (g.tile_of(j) != t) continue;
                // local index of j inside the box
                int ji = j % g.nx - (t % g.NX) * g.tx;
                int jj = (j / g.nx) % g.ny - ((t / g.NX) % g.NY) * g.ty;
                int jk = j / (g.nx * g.ny) - (t / (g.NX * g.NY)) * g.tz;
                int ax = min(g.tx, g.nx - (t % g.NX) * g.tx), ay = min(g.ty, g.ny - ((t / g.NX) % g.NY) * g.ty);
                int rj = ji + ax * (jj + ay * jk);
                lv = max(lv, lev[rj] + 1);
            }
            if (lv != lev[r]) { lev[r] = lv; changed = 1; }
        }
        changed = __syncthreads_or(changed);
        if (!changed) break;
    }
    // counting sort by level (stable in box order)
    for (int l = threadIdx.x; l < b.RC + 2; l += blockDim.x) cnt[l] = 0;
    __syncthreads();
    for (int r = threadIdx.x; r < n; r += blockDim.x) atomicMax(&misc[0], lev[r] + 1);
    __syncthreads();
    int nlev = misc[0];
    if (threadIdx.x == 0) {
        for (int r = 0; r < n; ++r) cnt[lev[r] + 1]++;
        for (int l = 0; l < nlev; ++l) cnt[l + 1] += cnt[l];
        short* lp = b.lev_ptr + (size_t)t * ((b.RC + 8) & ~7);
        for (int l = 0; l <= nlev; ++l) lp[l] = (short)cnt[l];
        for (int r = 0; r < n; ++r) {
            int p = cnt[lev[r]]++;
            order[p] = r;
            pos[r] = p;
        }
    }
    __syncthreads();
    // external dependency set: hash-set insert, compact, bitonic sort
    int* hs = misc + 8;                 // HS = power of two >= 2*EC
    int HS = 1;
    while (HS < 2 * b.EC) HS <<= 1;
    for (int q = threadIdx.x; q < HS; q += blockDim.x) hs[q] = -1;
    __shared__ int ups[32];
    if (threadIdx.x < 32) ups[threadIdx.x] = -1;
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
    // bitonic sort of ext[0, np2) (pad with INT_MAX; np2 <= EC rounded up fits in hs)
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
    // upstream tiles (unique, <= 32)
    for (int q = threadIdx.x; q < ne; q += blockDim.x) {
        int u = g.tile_of(ext[q]);
        for (int z = 0; z < 32; ++z) {
            int cur = atomicCAS(&ups[z], -1, u);
            if (cur == -1 || cur == u) break;
            if (z == 31) atomicExch(b.err, 6);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int nu = 0;
        int* up = b.up_ids + (size_t)t * 32;
        for (int z = 0; z < 32; ++z)
            if (ups[z] >= 0) up[nu++] = ups[z];
        b.up_cnt[t] = nu;
    }
    for (int q = threadIdx.x; q < ne; q += blockDim.x) b.ext_id[(size_t)t * b.EC + q] = ext[q];
    // per-row dependency counts -> local offsets (thread 0 scan; n <= RC)
    int* dp = b.dptr + (size_t)t * ((b.RC + 4) & ~3);
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int p = 0; p < n; ++p) {
            dp[p] = acc;
            int row = cell[order[p]];
            acc += b.D.ptr[row + 1] - b.D.ptr[row];
        }
        dp[n] = acc;
        misc[2] = acc;
    }
    __syncthreads();
    for (int p = threadIdx.x; p < n; p += blockDim.x) {
        int r = order[p], row = cell[r];
        b.row_id[(size_t)t * b.RC + p] = row;
        double dv = (b.unit || !b.diag) ? 1.0 : 1.0 / b.diag[row];
        b.dinv[(size_t)t * b.RC + p] = dv;
        int o = dp[p];
        for (int e = b.D.ptr[row]; e < b.D.ptr[row + 1]; ++e, ++o) {
            int j = b.D.idx[e];
            int slot;
            if (g.tile_of(j) == t) {
                int ji = j % g.nx - (t % g.NX) * g.tx;
                int jj = (j / g.nx) % g.ny - ((t / g.NX) % g.NY) * g.ty;
                int jk = j / (g.nx * g.ny) - (t / (g.NX * g.NY)) * g.tz;
                int ax = min(g.tx, g.nx - (t % g.NX) * g.tx), ay = min(g.ty, g.ny - ((t / g.NX) % g.NY) * g.ty);
                slot = pos[ji + ax * (jj + ay * jk)];
            } else {
                int lo = 0, hi = ne;
                while (lo < hi) {
                    int mid = (lo + hi) >> 1;
                    if (ext[mid] < j) lo = mid + 1;
                    else hi = mid;
                }
                slot = b.RC + lo;
            }
            size_t q = (size_t)t * b.RC * b.KD + o;
            b.dslot[q] = (short)slot;
            b.dsrc[q] = e;
            b.dcoef[q] = b.D.val ? b.D.val[e] : 0.0;
        }
    }
    if (threadIdx.x == 0) {
        int* h = b.hdr + (size_t)t * 4;
        h[0] = n;
        h[1] = ne;
        h[2] = nlev;
        h[3] = misc[2];
    }
}

// reload coefficients / 1/diag from the CSR positions recorded at build time
__global__ void k_tile_values(int n_tiles, int RC, int KD, const int* __restrict__ hdr, const int* __restrict__ dsrc,
                              const double* __restrict__ val, double* __restrict__ dcoef,
                              const int* __restrict__ row_id, const double* __restrict__ diag, bool unit,
                              double* __restrict__ dinv) {
    int t = blockIdx.x;
    int n = hdr[t * 4], nd = hdr[t * 4 + 3];
    for (int q = threadIdx.x; q < nd; q += blockDim.x) {
        size_t o = (size_t)t * RC * KD + q;
        dcoef[o] = val[dsrc[o]];
    }
    for (int p = threadIdx.x; p < n; p += blockDim.x) {
        size_t o = (size_t)t * RC + p;
        dinv[o] = (unit || !diag) ? 1.0 : 1.0 / diag[row_id[o]];
    }
}

struct TileSolve {
    int n_tiles, RC, KD, EC;
    const int* order;      // ticket -> tile
    const int* hdr;
    const short* lev_ptr;
    const int* row_id;
    const int* ext_id;
    const int* dptr;
    const short* dslot;
    const double* dcoef;
    const double* dinv;
    const int* up_cnt;
    const int* up_ids;
    int* flags;            // per tile: epoch of the last completed solve
    int* ticket;           // [counter]
    int epoch;
    int ticket_base;
    const double* b;
    double alpha;
    double* x;
    const double* add;
    double* out2;
    int* err;
    long long* dbg;        // optional per-tile phase timestamps (globaltimer ns)
};

__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned r16(unsigned b) { return (b + 15u) & ~15u; }
// TMA bulk copy global -> shared, completion signalled on an mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* mbar) {
    if (bytes == 0) return;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(mbar)) : "memory");
}

__global__ void __launch_bounds__(512) k_tile_solve(TileSolve a) {
    extern __shared__ __align__(128) unsigned char sm[];
    // 16-byte aligned sections (capacities padded on the host, see tile_smem_bytes)
    double* xs = reinterpret_cast<double*>(sm);                 // RC + EC
    double* cf = xs + a.RC + a.EC;                              // RC*KD
    double* di = cf + (size_t)a.RC * a.KD;                      // RC
    int* rid = reinterpret_cast<int*>(di + a.RC);               // RC
    int* dp = rid + a.RC;                                       // DPS = RC+1 rounded to 4
    short* sl = reinterpret_cast<short*>(dp + ((a.RC + 4) & ~3));   // RC*KD
    short* lp = sl + (size_t)a.RC * a.KD;                       // LPS = RC+1 rounded to 8
    __shared__ int s_tile, s_hdr[4];
    __shared__ __align__(8) uint64_t mbar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(&mbar)), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned phase = 0;
    const int DPS = (a.RC + 4) & ~3, LPS = (a.RC + 8) & ~7;
    for (;;) {
        if (threadIdx.x == 0) {
            int k = atomicAdd(a.ticket, 1) - a.ticket_base;
            int t = k < a.n_tiles ? a.order[k] : -1;
            s_tile = t;
            if (t >= 0) {
                const int4 h = *reinterpret_cast<const int4*>(a.hdr + (size_t)t * 4);
                s_hdr[0] = h.x; s_hdr[1] = h.y; s_hdr[2] = h.z; s_hdr[3] = h.w;
                // 1. stage the tile's plan with TMA bulk copies (independent of
                //    the solve, overlaps the upstream wait below)
                unsigned b_cf = r16(8u * h.w), b_sl = r16(2u * h.w), b_dp = r16(4u * (h.x + 1));
                unsigned b_lp = r16(2u * (h.z + 1)), b_di = r16(8u * h.x), b_ri = r16(4u * h.x);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                             ::"r"(smem_addr(&mbar)), "r"(b_cf + b_sl + b_dp + b_lp + b_di + b_ri) : "memory");
                bulk_g2s(cf, a.dcoef + (size_t)t * a.RC * a.KD, b_cf, &mbar);
                bulk_g2s(sl, a.dslot + (size_t)t * a.RC * a.KD, b_sl, &mbar);
                bulk_g2s(dp, a.dptr + (size_t)t * DPS, b_dp, &mbar);
                bulk_g2s(lp, a.lev_ptr + (size_t)t * LPS, b_lp, &mbar);
                bulk_g2s(di, a.dinv + (size_t)t * a.RC, b_di, &mbar);
                bulk_g2s(rid, a.row_id + (size_t)t * a.RC, b_ri, &mbar);
            }
        }
        __syncthreads();
        const int t = s_tile;
        if (t < 0) break;
        const int n = s_hdr[0], ne = s_hdr[1], nlev = s_hdr[2];
        if (a.dbg && threadIdx.x == 0) a.dbg[t * 6 + 0] = gtimer();
        // 2. wait for upstream tiles (relaxed polls: no L1 invalidation per poll)
        const int nu = a.up_cnt[t];
        if (threadIdx.x < nu) {
            const int* f = a.flags + a.up_ids[(size_t)t * 32 + threadIdx.x];
            unsigned ns = 8;
            long long spins = 0;
            while (ld_relaxed_i(f) != a.epoch) {
                __nanosleep(ns);
                if (ns < 64) ns <<= 1;
                if (++spins > SPIN_LIMIT) { atomicExch(a.err, 7); break; }
            }
            __threadfence();
            if (a.dbg && threadIdx.x == 0) a.dbg[t * 6 + 1] = gtimer();
        }
        // staged plan must have landed
        {
            unsigned done = 0;
            while (!done)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(done) : "r"(smem_addr(&mbar)), "r"(phase) : "memory");
            phase ^= 1u;
        }
        // rhs into the x slots
        for (int p = threadIdx.x; p < n; p += blockDim.x) xs[p] = a.alpha * __ldg(a.b + rid[p]);
        __syncthreads();
        // 3. gather external dependencies
        for (int q = threadIdx.x; q < ne; q += blockDim.x)
            xs[a.RC + q] = __ldcg(a.x + a.ext_id[(size_t)t * a.EC + q]);
        __syncthreads();
        if (a.dbg && threadIdx.x == 0) a.dbg[t * 6 + 2] = gtimer();
        // 4. local levels: G lanes per row (shuffle-reduced), rows of a level
        //    spread over the CTA
        constexpr int G = 8;
        const int grp = threadIdx.x / G, li = threadIdx.x % G, ngrp = blockDim.x / G;
        for (int l = 0; l < nlev; ++l) {
            int p1 = lp[l + 1];
            for (int base = lp[l]; base < p1; base += ngrp) {   // warp-uniform trip count
                const int p = base + grp;
                const bool act = p < p1;
                double acc = 0.0;
                if (act)
                    for (int q = dp[p] + li; q < dp[p + 1]; q += G) acc = fma(-cf[q], xs[sl[q]], acc);
#pragma unroll
                for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, G);
                if (act && li == 0) xs[p] = (xs[p] + acc) * di[p];
            }
            __syncthreads();
        }
        if (a.dbg && threadIdx.x == 0) a.dbg[t * 6 + 3] = gtimer();
        // 5. write back, publish
        for (int p = threadIdx.x; p < n; p += blockDim.x) {
            int row = rid[p];
            double v = xs[p];
            __stcg(a.x + row, v);
            if (a.out2) a.out2[row] = v + a.add[row];
        }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0)
            asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(a.flags + t), "r"(a.epoch) : "memory");
        if (a.dbg && threadIdx.x == 0) { a.dbg[t * 6 + 4] = gtimer(); a.dbg[t * 6 + 5] = blockIdx.x; }
    }
}

}  // namespace

// smem layout of k_tile_solve: xs[RC+EC] cf[RC*KD] di[RC] rid[RC] dp[DPS] sl[RC*KD] lp[LPS]
// (RC multiple of 8, KD and EC even -> every section starts 16-byte aligned)
size_t tile_smem_bytes(const TilePlan& tp) {
    size_t rc = tp.RC, kd = tp.KD, ec = tp.EC;
    size_t dps = (rc + 4) & ~size_t(3), lps = (rc + 8) & ~size_t(7);
    size_t bytes = 8 * (rc + ec) + 8 * rc * kd + 8 * rc + 4 * rc + 4 * dps + 2 * rc * kd + 2 * lps;
    return (bytes + 127) & ~size_t(127);
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
    if (hf[0] || hf[1] > 64) return false;
    const int nt = g.NX * g.NY * g.NZ;
    tp.n = n;
    tp.n_tiles = nt;
    tp.RC = (g.tx * g.ty * g.tz + 7) & ~7;           // per-tile capacities / strides
    tp.KD = (std::max(hf[1], 1) + 1) & ~1;
    tp.EC = (std::min(tp.RC * tp.KD, 4 * tp.RC + 256) + 1) & ~1;
    tp.unit = unit;
    tp.n_dep = D.nnz;
    size_t smem = tile_smem_bytes(tp);
    if (smem > 200 * 1024) return false;
    const size_t dps = (tp.RC + 4) & ~3, lps = (tp.RC + 8) & ~7;
    tp.hdr.reset(c, (size_t)nt * 4);
    tp.lev_ptr.reset(c, (size_t)nt * lps);
    tp.row_id.reset(c, (size_t)nt * tp.RC);
    tp.ext_id.reset(c, (size_t)nt * tp.EC);
    tp.dptr.reset(c, (size_t)nt * dps);
    tp.dslot.reset(c, (size_t)nt * tp.RC * tp.KD);
    tp.dsrc.reset(c, (size_t)nt * tp.RC * tp.KD);
    tp.dcoef.reset(c, (size_t)nt * tp.RC * tp.KD);
    tp.dinv.reset(c, (size_t)nt * tp.RC);
    tp.up_cnt.reset(c, nt);
    tp.up_ids.reset(c, (size_t)nt * 32);
    tp.flags.reset(c, nt);
    tp.ticket.reset(c, 1);
    EDFA_CUDA(cudaMemsetAsync(tp.flags.p, 0, sizeof(int) * nt, c->stream));
    EDFA_CUDA(cudaMemsetAsync(tp.ticket.p, 0, sizeof(int), c->stream));
    tp.epoch = 0;
    tp.ticket_base = 0;
    TileBuild b{view(D), g, reverse, tp.RC, tp.KD, tp.EC, diag, unit, tp.hdr.p, tp.lev_ptr.p, tp.row_id.p,
                tp.ext_id.p, tp.dptr.p, tp.dslot.p, tp.dsrc.p, tp.dcoef.p, tp.dinv.p, tp.up_cnt.p, tp.up_ids.p,
                fl + 2};
    int HS = 1;
    while (HS < 2 * tp.EC) HS <<= 1;
    size_t bsm = sizeof(int) * (5 * tp.RC + 2 + tp.EC + 8 + HS);
    {
        Prof pr(c, "tile_plan", 24.0 * D.nnz);
        if (bsm > 48 * 1024)
            EDFA_CUDA(cudaFuncSetAttribute(k_tile_build, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
        k_tile_build<<<nt, 256, bsm, c->stream>>>(b);
        check_launch("k_tile_build");
    }
    int e = 0;
    EDFA_CUDA(cudaMemcpyAsync(&e, fl + 2, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    // tile schedule: level of the tile DAG (host, tiny), ticket order by (level, id)
    std::vector<int> upc(nt), upi((size_t)nt * 32);
    EDFA_CUDA(cudaMemcpyAsync(upc.data(), tp.up_cnt.p, sizeof(int) * nt, cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaMemcpyAsync(upi.data(), tp.up_ids.p, sizeof(int) * nt * 32, cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
    if (e) return false;
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
    if (smem > 48 * 1024)
        EDFA_CUDA(cudaFuncSetAttribute(k_tile_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    return true;
}

void tile_values(Ctx* c, const Csr& D, const double* diag, TilePlan& tp) {
    Prof pr(c, "tile_plan", 20.0 * D.nnz);
    k_tile_values<<<tp.n_tiles, 256, 0, c->stream>>>(tp.n_tiles, tp.RC, tp.KD, tp.hdr.p, tp.dsrc.p, D.val.p,
                                                     tp.dcoef.p, tp.row_id.p, diag, tp.unit, tp.dinv.p);
    check_launch("k_tile_values");
}

void run_tile(Ctx* c, TilePlan& tp, const double* b, double alpha, double* x, const double* add, double* out2,
              const char* name) {
    size_t smem = tile_smem_bytes(tp);
    int occ = 0;
    EDFA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tile_solve, 256, smem));
    int grid = NUM_SMS_B200 * std::max(1, std::min(occ, 2));
    tp.epoch += 1;
    TileSolve a{tp.n_tiles, tp.RC, tp.KD, tp.EC, tp.order.p, tp.hdr.p, tp.lev_ptr.p, tp.row_id.p, tp.ext_id.p,
                tp.dptr.p, tp.dslot.p, tp.dcoef.p, tp.dinv.p, tp.up_cnt.p, tp.up_ids.p, tp.flags.p, tp.ticket.p,
                tp.epoch, tp.ticket_base, b, alpha, x, add, out2, c->d_scalar_i + 8, nullptr};
    static const char* dbg_path = getenv("EDFA_TILE_DEBUG");
    DevBuf<long long> dbg;
    if (dbg_path) {
        dbg.reset(c, (size_t)tp.n_tiles * 6);
        a.dbg = dbg.p;
    }
    tp.ticket_base += tp.n_tiles + grid;   // every CTA takes exactly one failing ticket
    Prof pr(c, name, 12.0 * tp.n_dep + 24.0 * tp.n + (out2 ? 16.0 * tp.n : 0.0));
    void* args[] = {&a};
    EDFA_CUDA(cudaLaunchCooperativeKernel((void*)k_tile_solve, dim3(grid), dim3(256), args, smem, c->stream));
    if (dbg_path) {
        std::vector<long long> h((size_t)tp.n_tiles * 6);
        EDFA_CUDA(cudaMemcpyAsync(h.data(), dbg.p, h.size() * 8, cudaMemcpyDeviceToHost, c->stream));
        EDFA_CUDA(cudaStreamSynchronize(c->stream));
        FILE* f = fopen(dbg_path, "w");
        if (f) {
            for (int t = 0; t < tp.n_tiles; ++t)
                fprintf(f, "%d %lld %lld %lld %lld %lld %lld\n", t, h[t * 6], h[t * 6 + 1], h[t * 6 + 2], h[t * 6 + 3],
                        h[t * 6 + 4], h[t * 6 + 5]);
            fclose(f);
        }
    }
}

}  // namespace edfa
