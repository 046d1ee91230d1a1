// Microbenchmark: inter-SM hand-off latency through L2 (value as its own flag):
// CTA 0 stores x[i] (st.global.cg), CTA 1 polls it (ld.relaxed.gpu) and answers
// in y[i]; also the same with st.relaxed.gpu stores and with __nanosleep polling.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double ld_rlx(const double* p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rlx(double* p, double v) {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

template <int MODE>   // 0: stcg + spin, 1: st.relaxed + spin, 2: stcg + nanosleep(32)
__global__ void k_pp(double* x, double* y, int iters, long long* out) {
    if (threadIdx.x != 0) return;
    long long t0 = clock64();
    long long g0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    for (int i = 0; i < iters; ++i) {
        double* mine = blockIdx.x == 0 ? x : y;
        double* other = blockIdx.x == 0 ? y : x;
        if (blockIdx.x == 0) {
            if (MODE == 1) st_rlx(mine + i, 1.0 + i); else __stcg(mine + i, 1.0 + i);
            while (ld_rlx(other + i) < 0.0) if (MODE == 2) __nanosleep(32);
        } else {
            while (ld_rlx(other + i) < 0.0) if (MODE == 2) __nanosleep(32);
            if (MODE == 1) st_rlx(mine + i, 1.0 + i); else __stcg(mine + i, 1.0 + i);
        }
    }
    long long g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    if (blockIdx.x == 0) { out[0] = (clock64() - t0) / iters / 2; out[1] = (g1 - g0) / iters / 2; }
}

int main() {
    double *x, *y;
    long long* out;
    const int iters = 2000;
    cudaMalloc(&x, iters * 8);
    cudaMalloc(&y, iters * 8);
    cudaMalloc(&out, 16);
    for (int mode = 0; mode < 3; ++mode) {
        for (int grid : {2, 150}) {   // 150: blocks 0 and 1 likely on different SMs / dies
            cudaMemset(x, 0xff, iters * 8);   // negative NaN? 0xff.. = NaN; use -1 fill below
            double* h = new double[iters];
            for (int i = 0; i < iters; ++i) h[i] = -1.0;
            cudaMemcpy(x, h, iters * 8, cudaMemcpyHostToDevice);
            cudaMemcpy(y, h, iters * 8, cudaMemcpyHostToDevice);
            if (mode == 0) k_pp<0><<<grid, 32>>>(x, y, iters, out);
            if (mode == 1) k_pp<1><<<grid, 32>>>(x, y, iters, out);
            if (mode == 2) k_pp<2><<<grid, 32>>>(x, y, iters, out);
            long long r[2];
            cudaMemcpy(r, out, 16, cudaMemcpyDeviceToHost);
            printf("mode %d grid %d: one hand-off %lld cyc, %lld ns (%s)\n", mode, grid, r[0], r[1],
                   cudaGetErrorString(cudaGetLastError()));
            delete[] h;
        }
    }
    return 0;
}
