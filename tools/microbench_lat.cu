// Microbenchmark: latency of dependent DFMA, dependent LDS.64 chains and
// __syncthreads on B200 (calibrates the tile-solver level-step model).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(double* out, long long* cyc, int iters) {
    __shared__ double s[1024];
    __shared__ int idx[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
        s[i] = 1.0 + i * 1e-9;
        idx[i] = (i * 7 + 3) & 1023;
    }
    __syncthreads();
    double a = out[0], b = 1.0000001, c = 1e-7;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) a = fma(a, b, c);          // dependent DFMA chain
    long long t1 = clock64();
    int p = threadIdx.x;
    for (int i = 0; i < iters; ++i) p = idx[p];                // dependent LDS.32 chain
    long long t2 = clock64();
    double acc = 0.0;
    for (int i = 0; i < iters; ++i) { acc += s[p & 1023]; p = (int)acc & 1023; }   // LDS.64 + dep
    long long t3 = clock64();
    for (int i = 0; i < iters; ++i) __syncthreads();
    long long t4 = clock64();
    if (threadIdx.x == 0) {
        cyc[0] = (t1 - t0) / iters;
        cyc[1] = (t2 - t1) / iters;
        cyc[2] = (t3 - t2) / iters;
        cyc[3] = (t4 - t3) / iters;
    }
    out[1 + threadIdx.x] = a + p + acc;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 4096 * 8);
    cudaMalloc(&cyc, 64);
    cudaMemset(out, 0, 8);
    for (int th : {32, 128, 256}) {
        k_lat<<<1, th>>>(out, cyc, 1000);
        long long h[4];
        cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost);
        printf("threads=%d: DFMA dep %lld cyc, LDS.32 dep %lld cyc, LDS.64+cvt dep %lld cyc, syncthreads %lld cyc (%s)\n",
               th, h[0], h[1], h[2], h[3], cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
