// Microbenchmark: shared-memory hand-off latency between two warps (value as
// its own flag, volatile polling), with and without __nanosleep back-off, and
// the dependent DFMA latency -- calibrates the dataflow tile solve.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double ldv(const double* p) { return *reinterpret_cast<const volatile double*>(p); }
__device__ __forceinline__ void stv(double* p, double v) { *reinterpret_cast<volatile double*>(p) = v; }

template <int SLEEP>
__global__ void k_pingpong(long long* cyc, int iters, double* out) {
    __shared__ double slot[2][1024];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) (&slot[0][0])[i] = -1.0;
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    long long t0 = clock64();
    double v = 0.0;
    if (w < 2) {
        for (int i = 0; i < iters; ++i) {
            // warp 0 writes slot[0][i], warp 1 waits for it then writes slot[1][i]; warp 0 waits for slot[1][i]
            if (w == 0) {
                if (lane == 0) stv(&slot[0][i], v + 1.0);
                double r;
                while ((r = ldv(&slot[1][i])) < 0.0) if (SLEEP) __nanosleep(SLEEP);
                v = r;
            } else {
                double r;
                while ((r = ldv(&slot[0][i])) < 0.0) if (SLEEP) __nanosleep(SLEEP);
                v = r;
                if (lane == 0) stv(&slot[1][i], v + 1.0);
            }
            __syncwarp();
        }
    } else {
        // other warps: spin on a slot that never arrives during the run (polling pressure)
        for (int i = 0; i < iters * 4; ++i) {
            if (ldv(&slot[0][1023]) > 1e300) break;
            if (SLEEP) __nanosleep(SLEEP);
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / iters / 2;   // one hand-off
    out[threadIdx.x] = v;
}

__global__ void k_dfma(long long* cyc, int iters, double* out) {
    double a = out[0], b = 1.0000001, c = 1e-7;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) a = fma(a, b, c);
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[1] = (t1 - t0) / iters;
    out[threadIdx.x + 64] = a;
}

int main() {
    long long* cyc;
    double* out;
    cudaMalloc(&cyc, 64);
    cudaMalloc(&out, 8192 * 8);
    cudaMemset(out, 0, 8192 * 8);
    long long h[2];
    for (int th : {64, 224}) {
        k_pingpong<0><<<1, th>>>(cyc, 500, out);
        cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
        printf("threads=%d spin: hand-off %lld cyc\n", th, h[0]);
        k_pingpong<16><<<1, th>>>(cyc, 500, out);
        cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
        printf("threads=%d nanosleep16: hand-off %lld cyc\n", th, h[0]);
    }
    k_dfma<<<1, 32>>>(cyc, 1000, out);
    cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency %lld cyc (%s)\n", h[1], cudaGetErrorString(cudaGetLastError()));
    return 0;
}
