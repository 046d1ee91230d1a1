// Microbenchmark: variants of the tile solver's level step in isolation
// (synthetic 22-level tile, 48 rows/level, 3 critical + 8 early deps).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

struct Tile {
    const int* dp; const short* md; const short* sl; const double* cf; const short* lp;
    int nlev, n, nd;
};

__device__ void stage(const Tile& g, double*& xs, double*& cf, int*& dp, short*& sl, short*& lp, short*& md,
                      unsigned char* sm) {
    xs = reinterpret_cast<double*>(sm);
    cf = xs + 4096;
    dp = reinterpret_cast<int*>(cf + g.nd);
    sl = reinterpret_cast<short*>(dp + g.n + 4);
    lp = sl + g.nd;
    md = lp + 64;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) xs[i] = 1.0 + i * 1e-6;
    for (int i = threadIdx.x; i < g.nd; i += blockDim.x) { cf[i] = g.cf[i]; sl[i] = g.sl[i]; }
    for (int i = threadIdx.x; i <= g.n; i += blockDim.x) dp[i] = g.dp[i];
    for (int i = threadIdx.x; i < g.n; i += blockDim.x) md[i] = g.md[i];
    for (int i = threadIdx.x; i <= g.nlev; i += blockDim.x) lp[i] = g.lp[i];
    __syncthreads();
}

// A: current kernel (half critical / half early, one thread per row)
__global__ void k_a(Tile g, long long* cyc, double* out, int reps) {
    extern __shared__ __align__(16) unsigned char sm[];
    double *xs, *cf; int* dp; short *sl, *lp, *md;
    stage(g, xs, cf, dp, sl, lp, md, sm);
    long long t0 = clock64();
    const int HALF = blockDim.x / 2;
    const bool crit = threadIdx.x < HALF;
    const int lid = crit ? threadIdx.x : threadIdx.x - HALF;
    for (int rep = 0; rep < reps; ++rep)
        for (int k = -1; k < g.nlev; ++k) {
            const int lv = crit ? k : k + 1;
            if (lv >= 0 && lv < g.nlev) {
                const int p1 = lp[lv + 1];
                for (int p = lp[lv] + lid; p < p1; p += HALF) {
                    const int qm = dp[p] + md[p];
                    const int q0 = crit ? qm : dp[p], q1 = crit ? dp[p + 1] : qm;
                    double acc = xs[p];
                    for (int q = q0; q < q1; ++q) acc = fma(-cf[q], xs[sl[q]], acc);
                    xs[p] = crit ? acc * 0.5 : acc;
                }
            }
            __syncthreads();
        }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / ((long long)reps * (g.nlev + 1));
    out[threadIdx.x] = xs[threadIdx.x];
}

// B: critical warps prefetch next level's (slot, coef) into registers;
// early work for level k+2 spread over the remaining warps, 2 lanes per row
template <int KC>
__global__ void k_b(Tile g, long long* cyc, double* out, int reps) {
    extern __shared__ __align__(16) unsigned char sm[];
    double *xs, *cf; int* dp; short *sl, *lp, *md;
    stage(g, xs, cf, dp, sl, lp, md, sm);
    long long t0 = clock64();
    const int NC = 64;                          // critical lanes
    const bool crit = threadIdx.x < NC;
    const int nE = blockDim.x - NC, lidE = threadIdx.x - NC;
    for (int rep = 0; rep < reps; ++rep) {
        // prefetch for level 0 (critical part)
        int pr = -1, ns = 0;
        short s[KC];
        double c[KC];
        auto fetch = [&](int lv) {
            pr = -1; ns = 0;
            if (lv < g.nlev) {
                int p = lp[lv] + threadIdx.x;
                if (p < lp[lv + 1]) {
                    pr = p;
                    int qm = dp[p] + md[p];
                    ns = dp[p + 1] - qm;
#pragma unroll
                    for (int u = 0; u < KC; ++u) {
                        s[u] = u < ns ? sl[qm + u] : 0;
                        c[u] = u < ns ? cf[qm + u] : 0.0;
                    }
                }
            }
        };
        if (crit) fetch(0);
        // early partials of levels 0 and 1 before the first step
        for (int lv = 0; lv < 2 && lv < g.nlev; ++lv)
            if (!crit)
                for (int p = lp[lv] + lidE; p < lp[lv + 1]; p += nE) {
                    double acc = xs[p];
                    for (int q = dp[p]; q < dp[p] + md[p]; ++q) acc = fma(-cf[q], xs[sl[q]], acc);
                    xs[p] = acc;
                }
        __syncthreads();
        for (int k = 0; k < g.nlev; ++k) {
            if (crit) {
                if (pr >= 0) {
                    double acc = xs[pr];
#pragma unroll
                    for (int u = 0; u < KC; ++u) acc = fma(-c[u], xs[s[u]], acc);   // padded: c = 0
                    xs[pr] = acc * 0.5;
                }
                fetch(k + 1);
            } else {
                const int lv = k + 2;                 // early deps of level k+2 are at levels <= k
                if (lv < g.nlev) {
                    const int p1 = lp[lv + 1];
                    const int grp = lidE >> 1, li = lidE & 1;
                    for (int base = lp[lv]; base < p1; base += nE / 2) {
                        int p = base + grp;
                        double acc = 0.0;
                        if (p < p1) {
                            int q0 = dp[p], q1 = q0 + md[p];
                            for (int q = q0 + li; q < q1; q += 2) acc = fma(-cf[q], xs[sl[q]], acc);
                        }
                        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
                        if (p < p1 && li == 0) xs[p] += acc;
                    }
                }
            }
            __syncthreads();
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[1] = (t1 - t0) / ((long long)reps * (g.nlev + 1));
    out[threadIdx.x] = xs[threadIdx.x];
}


// C: pieces of the step (mode 0: barrier only, 1: + lp loads, 2: + dp/md, 3: + 1 dep, 4: + all deps)
__global__ void k_c(Tile g, long long* cyc, double* out, int reps, int mode) {
    extern __shared__ __align__(16) unsigned char sm[];
    double *xs, *cf; int* dp; short *sl, *lp, *md;
    stage(g, xs, cf, dp, sl, lp, md, sm);
    long long t0 = clock64();
    const int HALF = blockDim.x / 2;
    const bool crit = threadIdx.x < HALF;
    const int lid = crit ? threadIdx.x : threadIdx.x - HALF;
    double sink = 0.0;
    for (int rep = 0; rep < reps; ++rep)
        for (int k = -1; k < g.nlev; ++k) {
            const int lv = crit ? k : k + 1;
            if (mode >= 1 && lv >= 0 && lv < g.nlev) {
                const int p1 = lp[lv + 1];
                for (int p = lp[lv] + lid; p < p1; p += HALF) {
                    if (mode == 1) { sink += p; continue; }
                    const int qm = dp[p] + md[p];
                    const int q0 = crit ? qm : dp[p], q1 = crit ? dp[p + 1] : qm;
                    if (mode == 2) { sink += q0 + q1; continue; }
                    double acc = xs[p];
                    int qe = mode == 3 ? min(q1, q0 + 1) : q1;
                    for (int q = q0; q < qe; ++q) acc = fma(-cf[q], xs[sl[q]], acc);
                    xs[p] = crit ? acc * 0.5 : acc;
                }
            }
            __syncthreads();
        }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / ((long long)reps * (g.nlev + 1));
    out[threadIdx.x] = xs[threadIdx.x] + sink;
}

int main() {
    const int nlev = 22, per = 48, n = nlev * per, dcrit = 3, dearly = 8, kd = dcrit + dearly, nd = n * kd;
    int* dp = new int[n + 1];
    short* md = new short[n];
    short* sl = new short[nd];
    double* cf = new double[nd];
    short* lp = new short[nlev + 1];
    for (int l = 0; l <= nlev; ++l) lp[l] = (short)(l * per);
    srand(1);
    for (int p = 0; p < n; ++p) {
        dp[p] = p * kd;
        md[p] = dearly;
        int l = p / per;
        for (int q = 0; q < kd; ++q) {
            int slot;
            if (q < dearly) slot = l >= 2 ? (l - 2) * per + rand() % per : 2000 + rand() % 800;
            else slot = l >= 1 ? (l - 1) * per + rand() % per : 2000 + rand() % 800;
            sl[p * kd + q] = (short)slot;
            cf[p * kd + q] = 1e-3 * (q + 1);
        }
    }
    dp[n] = nd;
    Tile g;
    int* d_dp; short *d_md, *d_sl, *d_lp; double *d_cf, *d_out; long long* d_cyc;
    cudaMalloc(&d_dp, 4 * (n + 1)); cudaMalloc(&d_md, 2 * n); cudaMalloc(&d_sl, 2 * nd); cudaMalloc(&d_lp, 2 * (nlev + 1));
    cudaMalloc(&d_cf, 8 * nd); cudaMalloc(&d_out, 8 * 1024); cudaMalloc(&d_cyc, 16);
    cudaMemcpy(d_dp, dp, 4 * (n + 1), cudaMemcpyHostToDevice);
    cudaMemcpy(d_md, md, 2 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(d_sl, sl, 2 * nd, cudaMemcpyHostToDevice);
    cudaMemcpy(d_lp, lp, 2 * (nlev + 1), cudaMemcpyHostToDevice);
    cudaMemcpy(d_cf, cf, 8 * nd, cudaMemcpyHostToDevice);
    g.dp = d_dp; g.md = d_md; g.sl = d_sl; g.cf = d_cf; g.lp = d_lp; g.nlev = nlev; g.n = n; g.nd = nd;
    size_t smem = 8 * 4096 + 8 * nd + 4 * (n + 4) + 2 * nd + 2 * 64 + 2 * n + 64;
    cudaFuncSetAttribute(k_a, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_b<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    long long h[2];
    cudaFuncSetAttribute(k_c, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int mode = 0; mode <= 4; ++mode) {
        k_c<<<1, 128, smem>>>(g, d_cyc, d_out, 100, mode);
        cudaMemcpy(h, d_cyc, 8, cudaMemcpyDeviceToHost);
        printf("C mode %d: %lld cyc/step\n", mode, h[0]);
    }
    for (int th : {128, 256}) {
        k_a<<<1, th, smem>>>(g, d_cyc, d_out, 100);
        k_b<4><<<1, th, smem>>>(g, d_cyc, d_out, 100);
        cudaMemcpy(h, d_cyc, 16, cudaMemcpyDeviceToHost);
        printf("threads=%d: A (current) %lld cyc/step, B (register prefetch + 2-lane early) %lld cyc/step (%s)\n", th,
               h[0], h[1], cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
