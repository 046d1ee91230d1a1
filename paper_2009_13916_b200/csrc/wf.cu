// Wavefront-packed triangular solves of an ILU factor (InnerFactorization.apply,
// hx/sparse.py:125-129) for factors whose dependency levels are wide (e.g.
// the ILU(0) of S~ at 256^3: 766 levels of up to 49k rows).
//
// Both solves run on ONE slot layout: rows sorted by the dependency level of
// L (natural order inside a level), every level padded to whole warps.  The
// intermediate and the solution live in slot order, and the SELL-32
// coefficient records store dependency SLOTS, so
//   * the plan is streamed once, fully coalesced;
//   * the rows of a level that sit next to each other in a slice depend on
//     rows that sit next to each other in an earlier level (axial stencils),
//     so the dependency gathers are near-coalesced L2 hits;
//   * x is written with one coalesced 8-byte reduction per row.
// U runs the same slices in reverse order (its dependencies are checked to lie
// in later slices).  The solve itself is sync-free: warps take slices from a
// ticket in topological order, a thread per row polls its dependencies on the
// SENTINEL-prefilled slot vector (a stored value is its own ready flag).
// A row is summed bias first, then its records in stored order (sorted by
// dependency level, oldest first): fixed per plan, so solves are reproducible.
#include "dev_util.cuh"
#include "edfa_internal.cuh"
#include "objects.cuh"

namespace edfa {
namespace {

__global__ void k_wf_pos(const int32_t* __restrict__ perm, int n_slots, int32_t* __restrict__ pos) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_slots) return;
    const int r = perm[s];
    if (r >= 0) pos[r] = s;
}
// every dependency of a row must sit in a slice processed earlier
__global__ void k_wf_check(CsrV D, const int32_t* __restrict__ pos, bool reverse, int* __restrict__ bad) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= D.n_rows) return;
    const int si = pos[i] >> 5;
    for (int e = D.ptr[i]; e < D.ptr[i + 1]; ++e) {
        const int sj = pos[D.idx[e]] >> 5;
        if (reverse ? sj <= si : sj >= si) atomicExch(bad, 1);
    }
}
__global__ void k_wf_remap(int32_t* __restrict__ col, int64_t n, const int32_t* __restrict__ pos) {
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        const int c = col[q];
        if (c >= 0) col[q] = pos[c];
    }
}
struct WfArgs {
    const int32_t* perm;
    const int64_t* sptr;
    const int32_t* col;
    const double* val;
    const double* dinv;
    int n_slices;
    unsigned* ticket;
    unsigned ticket_base;
    const double* b;      // slot order (b_slots) or natural order
    int b_slots;
    double alpha;
    double* xs;           // slot-order solution, SENTINEL-prefilled
    double* x_nat;        // optional natural-order copy
    const double* add;    // natural order
    double* out2;         // natural order: x + add
    double* b_sent;       // slot-order rhs, reset to SENTINEL once read (or NULL)
    double* pre_sent;     // slot-order vector set to SENTINEL (or NULL)
    int* err;
};

// Per-row records are sorted so that the dependencies of the nearest level
// come LAST (k_wf_sort_rows) and are loaded right-aligned into the register
// arrays: slots [0, K-NEAR) hold older levels, [K-NEAR, K) the nearest ones.
//   phase 1: the older dependencies -- nearly always present already; warps
//     that run several levels ahead of the frontier wait here with a back-off,
//     so they do not flood the L2 with polls;
//   phase 2: the nearest NEAR dependencies, polled tightly as one batch; after
//     the last arrival only NEAR FMAs and the publish remain.
// The summation order is the stored order (bias first), fixed per plan.
#ifndef EDFA_WF_NEAR
#define EDFA_WF_NEAR 3
#endif
constexpr int WF_NEAR = EDFA_WF_NEAR;
#ifndef EDFA_WF_SLEEP0
#define EDFA_WF_SLEEP0 64
#endif
#ifndef EDFA_WF_SLEEP_MAX
#define EDFA_WF_SLEEP_MAX 512
#endif
constexpr int WF_CHUNK = 16;   // records per batch of the older part of rows wider than the register window

// batch poll of missing values (SENTINEL) among x[U0..U1): re-read all of them
// per round, one warp vote; back_off: sleep between rounds (warps far ahead of
// the frontier)
template <int N, int U0, int U1, bool BACKOFF, unsigned SLEEP0 = EDFA_WF_SLEEP0, unsigned SLEEP_MAX = EDFA_WF_SLEEP_MAX>
__device__ __forceinline__ void wf_poll(const int (&cc)[N], double (&xv)[N], const double* xs, int* err) {
    bool miss = false;
#pragma unroll
    for (int u = U0; u < U1; ++u) miss |= cc[u] >= 0 && is_sentinel(xv[u]);
    long long spins = 0;
    unsigned ns = SLEEP0;
    while (__any_sync(0xffffffffu, miss)) {
        if (BACKOFF) {
            __nanosleep(ns);
            if (ns < SLEEP_MAX) ns <<= 1;
        }
#pragma unroll
        for (int u = U0; u < U1; ++u)
            if (cc[u] >= 0 && is_sentinel(xv[u])) xv[u] = ld_relaxed(xs + cc[u]);
        miss = false;
#pragma unroll
        for (int u = U0; u < U1; ++u) miss |= cc[u] >= 0 && is_sentinel(xv[u]);
        if (++spins > SPIN_LIMIT) {
            if (miss) {
                atomicExch(err, 3);
#pragma unroll
                for (int u = U0; u < U1; ++u)
                    if (is_sentinel(xv[u])) xv[u] = 0.0;
            }
            break;
        }
    }
}

// WIDE: rows may hold more than K records (general factors, e.g. the Schur
// ILU of dynamic patterns on distorted grids: ~110 dependencies per row);
// the records in front of the last K are streamed in batches of WF_CHUNK
// (they belong to old levels and are nearly always present).
// (two blocks per SM: three force the K = 20 window into 80 registers with 168 bytes of spills and are slower,
// 697 / 714 us vs 577 / 653 us per solve at 256^3)
template <int K, bool REV, bool WIDE>
__global__ void __launch_bounds__(256, 2) k_wf(WfArgs a) {
    const int lane = threadIdx.x & 31;
    const double sent = __longlong_as_double((long long)SENTINEL_BITS);
    for (;;) {
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(a.ticket, 1u) - a.ticket_base;
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= (unsigned)a.n_slices) break;
        const int s = REV ? a.n_slices - 1 - (int)t : (int)t;
        const int slot = s * 32 + lane;
        const int r = a.perm[slot];
        const int64_t b0 = a.sptr[s];
        const int w = (int)((a.sptr[s + 1] - b0) / 32);
        const int skip = (WIDE && w > K) ? w - K : 0;  // oldest records beyond the register window
        const int off = K - (w - skip);                // right alignment: record k sits in register k - skip + off
        double acc = 0.0;
        if (r >= 0) acc = a.alpha * (a.b_slots ? a.b[slot] : a.b[r]);   // b may alias out2 row-wise: plain load
        const double di = a.dinv ? a.dinv[slot] : 1.0;
        if (a.b_sent) a.b_sent[slot] = sent;
        if (a.pre_sent) a.pre_sent[slot] = sent;
        if (WIDE) {
            for (int k0 = 0; k0 < skip; k0 += WF_CHUNK) {
                int c[WF_CHUNK];
                double v[WF_CHUNK], x[WF_CHUNK];
#pragma unroll
                for (int u = 0; u < WF_CHUNK; ++u) {
                    const bool in = k0 + u < skip;
                    const int64_t q = b0 + (int64_t)(k0 + u) * 32 + lane;
                    c[u] = in ? __ldg(a.col + q) : -1;
                    v[u] = in ? __ldg(a.val + q) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < WF_CHUNK; ++u) x[u] = c[u] >= 0 ? ld_relaxed(a.xs + c[u]) : 0.0;
                wf_poll<WF_CHUNK, 0, WF_CHUNK, true>(c, x, a.xs, a.err);
#pragma unroll
                for (int u = 0; u < WF_CHUNK; ++u) acc = fma(-v[u], x[u], acc);
            }
        }
        int cc[K];
        double vv[K];
#pragma unroll
        for (int u = 0; u < K; ++u) {
            const bool in = u >= off;
            const int64_t q = b0 + (int64_t)(u - off + skip) * 32 + lane;
            cc[u] = in ? __ldg(a.col + q) : -1;
            vv[u] = in ? __ldg(a.val + q) : 0.0;
        }
        double xv[K];
#pragma unroll
        for (int u = 0; u < K; ++u) xv[u] = cc[u] >= 0 ? ld_relaxed(a.xs + cc[u]) : 0.0;   // all in flight at once
        // ---- phase 1: older levels
        wf_poll<K, 0, K - WF_NEAR, true>(cc, xv, a.xs, a.err);
#pragma unroll
        for (int u = 0; u < K - WF_NEAR; ++u) acc = fma(-vv[u], xv[u], acc);
        // ---- phase 2: the nearest level
        wf_poll<K, K - WF_NEAR, K, false>(cc, xv, a.xs, a.err);
#pragma unroll
        for (int u = K - WF_NEAR; u < K; ++u) acc = fma(-vv[u], xv[u], acc);
        if (r >= 0) {
            const double xr = acc * di;
            // fire-and-forget reduction at L2: SENTINEL + (x - SENTINEL)
            atomicAdd(reinterpret_cast<unsigned long long*>(a.xs + slot),
                      (unsigned long long)__double_as_longlong(publishable(xr)) - SENTINEL_BITS);
            if (a.x_nat) a.x_nat[r] = xr;
            if (a.out2) a.out2[r] = xr + a.add[r];
        }
    }
}

// Prefetching shape of k_wf (rows of at most K records): a warp holds three
// slices at a time --
//   A: being solved; its columns sit in registers, its coefficients in shared memory;
//   B: the next ticket; its records are on their way into the warp's shared-memory
//      stage by two bulk copies (cp.async.bulk, one mbarrier per stage), its
//      right-hand side and diagonal are in flight to registers;
//   C: the ticket after that; its slice pointer and row index are in flight;
// so the DRAM latency of a slice's plan (slice pointer -> records) is paid while the
// previous slice polls its dependencies instead of in front of every slice.
// Tickets are still handed out in topological order and a warp solves its slices
// in ticket order, so the lowest unfinished slice is always some warp's A: no deadlock.
// Per warp: one column stage (read into registers as soon as it lands, then free
// for B) and two coefficient stages.  Summation order as in k_wf.
__device__ __forceinline__ unsigned wf_saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
// back-off of the prefetching shape's phase 1 (A/B at 256^3: 64..512 ns 502/512 ms per step for L/U, 8..32 ns 479/490)
#ifndef EDFA_WF_PF_SLEEP0
#define EDFA_WF_PF_SLEEP0 8
#endif
#ifndef EDFA_WF_PF_SLEEP_MAX
#define EDFA_WF_PF_SLEEP_MAX 32
#endif
#ifndef EDFA_WF_PF_WARPS
#define EDFA_WF_PF_WARPS 8
#endif
#ifndef EDFA_WF_PF_BLOCKS
#define EDFA_WF_PF_BLOCKS 2
#endif
constexpr int WF_PF_WARPS = EDFA_WF_PF_WARPS;
constexpr size_t wf_pf_warp_bytes(int K) { return (size_t)K * 32 * (4 + 2 * 8); }
constexpr size_t wf_pf_smem(int K) { return WF_PF_WARPS * wf_pf_warp_bytes(K) + WF_PF_WARPS * 2 * sizeof(uint64_t); }

template <int K, bool REV>
__global__ void __launch_bounds__(WF_PF_WARPS * 32, EDFA_WF_PF_BLOCKS) k_wf_pf(WfArgs a) {
    extern __shared__ __align__(128) unsigned char wf_smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double* vbuf = reinterpret_cast<double*>(wf_smem) + (size_t)wid * 2 * K * 32;            // [2][K*32]
    int32_t* cbuf = reinterpret_cast<int32_t*>(wf_smem + WF_PF_WARPS * (size_t)2 * K * 32 * 8) + (size_t)wid * K * 32;
    uint64_t* bar = reinterpret_cast<uint64_t*>(wf_smem + WF_PF_WARPS * wf_pf_warp_bytes(K)) + wid * 2;
    const double sent = __longlong_as_double((long long)SENTINEL_BITS);
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(wf_saddr(&bar[0])) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(wf_saddr(&bar[1])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    bool more = true;   // tickets left (a warp stops at its first failing ticket)
    auto take = [&]() -> int {
        if (!more) return -1;
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(a.ticket, 1u) - a.ticket_base;
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= (unsigned)a.n_slices) { more = false; return -1; }
        return REV ? a.n_slices - 1 - (int)t : (int)t;
    };
    // lane 0: records of slice (b0, w) -> column stage and coefficient stage st
    auto issue = [&](int64_t b0, int w, int st) {
        if (lane == 0 && w > 0) {
            const unsigned mb = wf_saddr(&bar[st]);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"((unsigned)w * 32u * 12u)
                         : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(wf_saddr(cbuf)), "l"(a.col + b0), "r"((unsigned)w * 128u), "r"(mb) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(wf_saddr(vbuf + (size_t)st * K * 32)), "l"(a.val + b0), "r"((unsigned)w * 256u), "r"(mb)
                         : "memory");
        }
    };
    // stage C of a slice: pointer pair and row index (loads stay in flight until used)
    int sA = take(), sB = -1, sC = -1;
    int64_t b0A = 0, b0B = 0, b0C = 0;
    int wA = 0, wB = 0, wC = 0, rA = -1, rB = -1, rC = -1;
    double biasA = 0.0, biasB = 0.0, diA = 1.0, diB = 1.0;
    auto stage_c = [&](int s, int64_t& b0, int& w, int& r) {
        if (s < 0) return;
        b0 = a.sptr[s];
        w = (int)((a.sptr[s + 1] - b0) / 32);
        r = a.perm[s * 32 + lane];
    };
    auto stage_b = [&](int s, int r, double& bias, double& di) {
        if (s < 0) return;
        const int slot = s * 32 + lane;
        bias = r >= 0 ? (a.b_slots ? a.b[slot] : a.b[r]) : 0.0;   // b may alias out2 / b_sent row-wise: plain load
        di = a.dinv ? a.dinv[slot] : 1.0;
    };
    stage_c(sA, b0A, wA, rA);
    stage_b(sA, rA, biasA, diA);
    issue(b0A, wA, 0);
    sB = take();
    stage_c(sB, b0B, wB, rB);
    unsigned phase = 0;   // bit st: parity of the next completion of bar[st]
    int st = 0;
    while (sA >= 0) {
        const int slot = sA * 32 + lane;
        const int off = K - wA;   // right alignment: record k sits in register k + off
        int cc[K];
        if (wA > 0) {
            asm volatile("{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
                         "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                         "@!p bra WAIT_%=;\n\t}" ::"r"(wf_saddr(&bar[st])), "r"((phase >> st) & 1u) : "memory");
            phase ^= 1u << st;
        }
#pragma unroll
        for (int u = 0; u < K; ++u) cc[u] = u >= off ? cbuf[(u - off) * 32 + lane] : -1;
        double xv[K];
#pragma unroll
        for (int u = 0; u < K; ++u) xv[u] = cc[u] >= 0 ? ld_relaxed(a.xs + cc[u]) : 0.0;   // all in flight at once
        __syncwarp();   // the column stage is free again
        // B's records into the other stage, B's scalars and C's pointers into registers
        issue(b0B, wB, st ^ 1);
        stage_b(sB, rB, biasB, diB);
        sC = take();
        stage_c(sC, b0C, wC, rC);
        if (a.b_sent) a.b_sent[slot] = sent;
        if (a.pre_sent) a.pre_sent[slot] = sent;
        const double* vv = vbuf + (size_t)st * K * 32 + lane;
        double acc = rA >= 0 ? a.alpha * biasA : 0.0;
        // ---- phase 1: older levels
        wf_poll<K, 0, K - WF_NEAR, true, EDFA_WF_PF_SLEEP0, EDFA_WF_PF_SLEEP_MAX>(cc, xv, a.xs, a.err);
#pragma unroll
        for (int u = 0; u < K - WF_NEAR; ++u)
            if (u >= off) acc = fma(-vv[(u - off) * 32], xv[u], acc);
        // ---- phase 2: the nearest level
        auto publish = [&](double sum) {
            if (rA >= 0) {
                const double xr = sum * diA;
                // fire-and-forget reduction at L2: SENTINEL + (x - SENTINEL)
                atomicAdd(reinterpret_cast<unsigned long long*>(a.xs + slot),
                          (unsigned long long)__double_as_longlong(publishable(xr)) - SENTINEL_BITS);
                if (a.x_nat) a.x_nat[rA] = xr;
                if (a.out2) a.out2[rA] = xr + a.add[rA];
            }
        };
        // (publishing per lane, without the warp vote, measured slower: 495 / 508 vs 479 / 490 ms per step)
        // (two staggered probes in flight per poll round measured slower too: 498 / 508 ms)
        wf_poll<K, K - WF_NEAR, K, false>(cc, xv, a.xs, a.err);
#pragma unroll
        for (int u = K - WF_NEAR; u < K; ++u)
            if (u >= off) acc = fma(-vv[(u - off) * 32], xv[u], acc);
        publish(acc);
        __syncwarp();   // every lane is done with coefficient stage st before it is refilled
        sA = sB; b0A = b0B; wA = wB; rA = rB; biasA = biasB; diA = diB;
        sB = sC; b0B = b0C; wB = wC; rB = rC;
        sC = -1;
        st ^= 1;
    }
}

// Sort every row's records by dependency slot -- ascending for L (older levels
// first), descending for U (run in reverse: larger slots are older) -- pads (-1)
// in front, so the nearest level's dependencies are the last records of the row.
__global__ void k_wf_sort_rows(const int64_t* __restrict__ sptr, int n_slices, int32_t* __restrict__ col,
                               double* __restrict__ val, bool descending) {
    const int slot = blockIdx.x * blockDim.x + threadIdx.x;
    const int s = slot >> 5, lane = slot & 31;
    if (s >= n_slices) return;
    const int64_t b0 = sptr[s];
    const int w = (int)((sptr[s + 1] - b0) / 32);
    // insertion sort in place (w is small; one-time plan work)
    for (int i = 1; i < w; ++i) {
        const int ci = col[b0 + (int64_t)i * 32 + lane];
        const double vi = val[b0 + (int64_t)i * 32 + lane];
        // key: pads first, then by slot in the requested direction
        auto before = [&](int x, int y) {   // x sorts before y
            if (x < 0 || y < 0) return x < 0 && y >= 0;
            return descending ? x > y : x < y;
        };
        int j = i - 1;
        while (j >= 0 && before(ci, col[b0 + (int64_t)j * 32 + lane])) {
            col[b0 + (int64_t)(j + 1) * 32 + lane] = col[b0 + (int64_t)j * 32 + lane];
            val[b0 + (int64_t)(j + 1) * 32 + lane] = val[b0 + (int64_t)j * 32 + lane];
            --j;
        }
        col[b0 + (int64_t)(j + 1) * 32 + lane] = ci;
        val[b0 + (int64_t)(j + 1) * 32 + lane] = vi;
    }
}

template <int K>
void launch_wf_pf(Ctx* c, const TriPlan& p, WfArgs& a) {
    static int grid = 0;
    auto kf = k_wf_pf<K, false>;
    auto kr = k_wf_pf<K, true>;
    const size_t smem = wf_pf_smem(K);
    // per launch: the attribute is per device and the call costs ~1 us against a ~1 ms solve
    EDFA_CUDA(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    EDFA_CUDA(cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (!grid) {
        int occ = 0;
        EDFA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kf, WF_PF_WARPS * 32, smem));
        grid = NUM_SMS_B200 * std::max(1, occ);
    }
    unsigned& base = const_cast<unsigned&>(p.wf_ticket_base);
    a.ticket_base = base;
    base += (unsigned)(a.n_slices + grid * WF_PF_WARPS);   // every warp takes exactly one failing ticket
    if (p.wf_reverse) kr<<<grid, WF_PF_WARPS * 32, smem, c->stream>>>(a);
    else kf<<<grid, WF_PF_WARPS * 32, smem, c->stream>>>(a);
    check_launch("k_wf_pf");
}

template <int K, bool WIDE>
void launch_wf(Ctx* c, const TriPlan& p, WfArgs& a) {
    static int grid = 0;
    auto kf = k_wf<K, false, WIDE>;
    auto kr = k_wf<K, true, WIDE>;
    if (!grid) {
        int occ = 0;
        EDFA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kf, 256, 0));
        grid = NUM_SMS_B200 * std::max(1, occ);
    }
    unsigned& base = const_cast<unsigned&>(p.wf_ticket_base);
    a.ticket_base = base;
    base += (unsigned)(a.n_slices + grid * 8);   // every warp takes exactly one failing ticket
    if (p.wf_reverse) kr<<<grid, 256, 0, c->stream>>>(a);
    else kf<<<grid, 256, 0, c->stream>>>(a);
    check_launch("k_wf");
}

}  // namespace

// A level plan (natural dependency columns, values loaded) becomes a
// wavefront-packed plan on its own slot layout: columns -> slots, records
// sorted oldest level first, slices run in plan order.
static void wf_from_level_plan(Ctx* c, TriPlan& p) {
    const int n_slots = p.n_slots, n_slices = n_slots / 32;
    p.wf_pos.reset(c, std::max(p.n, 1));
    Prof pr(c, "wf_plan", 40.0 * p.n_stored + 8.0 * p.n);
    k_wf_pos<<<ceil_div(n_slots, 256), 256, 0, c->stream>>>(p.perm.p, n_slots, p.wf_pos.p);
    if (p.n_stored > 0)
        k_wf_remap<<<std::min<int64_t>(ceil_div(p.n_stored, 256), NUM_SMS_B200 * 16), 256, 0, c->stream>>>(
            p.col.p, p.n_stored, p.wf_pos.p);
    k_wf_sort_rows<<<ceil_div(n_slots, 256), 256, 0, c->stream>>>(p.slice_ptr.p, n_slices, p.col.p, p.val.p, false);
    check_launch("k_wf_sort_rows");
    p.is_wf = true;
    p.wf_reverse = false;
    p.wf_shared = false;
    p.wf_perm = p.perm.p;
    p.wf_slices = n_slices;
    p.wf_ticket.reset(c, 1);
    EDFA_CUDA(cudaMemsetAsync(p.wf_ticket.p, 0, sizeof(unsigned), c->stream));
    p.wf_ticket_base = 0;
}

// Turn the level plan of L (fwd, built by build_plan on Lv's pattern, values
// loaded) and U's rows into wavefront-packed plans.  When every dependency of
// U lies in a later slice of L's layout (structurally symmetric factors) U
// shares that layout and runs its slices in reverse, so the intermediate
// vector never leaves slot order; otherwise U gets the layout of its own
// level plan and the two solves hand over in natural order.
bool build_wf_plans(Ctx* c, const Csr& Lv, const Csr& Uv, const double* udiag, TriPlan& fwd, TriPlan& bwd) {
    const int n = Lv.n_rows;
    if (n == 0 || fwd.n_slots == 0 || fwd.is_chain) return false;
    const int n_slots = fwd.n_slots, n_slices = n_slots / 32;
    wf_from_level_plan(c, fwd);
    int* bad = c->d_scalar_i + 30;
    EDFA_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), c->stream));
    k_wf_check<<<ceil_div(n, 256), 256, 0, c->stream>>>(view(Uv), fwd.wf_pos.p, true, bad);
    check_launch("k_wf_check");
    int hb = 0;
    EDFA_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    EDFA_CUDA(cudaStreamSynchronize(c->stream));
    if (hb) {   // U on the layout of its own (reverse) level plan
        build_plan(c, Uv, udiag, false, true, bwd, /*allow_chain=*/false);
        if (bwd.n_slots == 0) return true;
        wf_from_level_plan(c, bwd);
        return true;
    }
    // U on L's slots
    bwd.n = n;
    bwd.unit = false;
    bwd.n_dep = Uv.nnz;
    bwd.n_slots = n_slots;
    bwd.n_levels = fwd.n_levels;
    sell_on_layout(c, fwd.perm.p, n_slices, Uv, udiag, false, bwd.slice_ptr, bwd.col, bwd.val, bwd.dinv, bwd.n_stored,
                   bwd.max_w);
    Prof pr(c, "wf_plan", 40.0 * bwd.n_stored);
    if (bwd.n_stored > 0)
        k_wf_remap<<<std::min<int64_t>(ceil_div(bwd.n_stored, 256), NUM_SMS_B200 * 16), 256, 0, c->stream>>>(
            bwd.col.p, bwd.n_stored, fwd.wf_pos.p);
    k_wf_sort_rows<<<ceil_div(n_slots, 256), 256, 0, c->stream>>>(bwd.slice_ptr.p, n_slices, bwd.col.p, bwd.val.p, true);
    check_launch("k_wf_remap");
    bwd.is_wf = true;
    bwd.wf_reverse = true;
    bwd.wf_shared = true;
    bwd.wf_perm = fwd.perm.p;
    bwd.wf_slices = n_slices;
    bwd.wf_ticket.reset(c, 1);
    EDFA_CUDA(cudaMemsetAsync(bwd.wf_ticket.p, 0, sizeof(unsigned), c->stream));
    bwd.wf_ticket_base = 0;
    return true;
}

// One solve on the slot layout.  b: slot order (b_slots) or natural; xs: slot-
// order solution (SENTINEL-prefilled unless fill_xs); x_nat / out2: optional
// natural-order outputs.
void run_wf(Ctx* c, const TriPlan& p, const double* b, bool b_slots, double alpha, double* xs, bool fill_xs,
            double* x_nat, const double* add, double* out2, double* b_sent, double* pre_sent, const char* name) {
    if (fill_xs) fill_bits(c, xs, p.n_slots, SENTINEL_BITS);
    WfArgs a{p.wf_perm, p.slice_ptr.p, p.col.p, p.val.p, p.unit ? nullptr : p.dinv.p, p.wf_slices,
             p.wf_ticket.p, 0u, b, b_slots ? 1 : 0, alpha, xs, x_nat, add, out2, b_sent, pre_sent, c->d_scalar_i + 8};
    Prof pr(c, name, 12.0 * p.n_dep + 24.0 * p.n + (out2 ? 16.0 * p.n : 0.0));
    if (c->opt.wf_prefetch && p.max_w <= 20) {
        if (p.max_w <= 8) launch_wf_pf<8>(c, p, a);
        else if (p.max_w <= 12) launch_wf_pf<12>(c, p, a);
        else launch_wf_pf<20>(c, p, a);
    } else if (p.max_w <= 8) launch_wf<8, false>(c, p, a);
    else if (p.max_w <= 12) launch_wf<12, false>(c, p, a);
    else if (p.max_w <= 20) launch_wf<20, false>(c, p, a);
    else launch_wf<16, true>(c, p, a);
}

// natural-order entry (run_plan): gathers b, scatters x through a slot-order scratch
void run_wf_natural(Ctx* c, const TriPlan& p, const double* b, double alpha, double* x, const double* add,
                    double* out2, const char* name) {
    DevBuf<double> xs(c, p.n_slots);
    run_wf(c, p, b, false, alpha, xs.p, true, x, add, out2, nullptr, nullptr, name);
}

}  // namespace edfa
