// Microbenchmark: cost of one software grid barrier on B200 for the
// level-synchronous triangular solves (variants: sleep/no-sleep, grid size).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench_sync.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <int SLEEP>
__device__ void barrier(unsigned* count, unsigned* gen, unsigned nb) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned g = ld_acq(gen);
        __threadfence();
        if (atomicAdd(count, 1u) == nb - 1) {
            *count = 0;
            __threadfence();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gen), "r"(g + 1) : "memory");
        } else {
            while (ld_acq(gen) == g) {
                if (SLEEP) __nanosleep(SLEEP);
            }
        }
    }
    __syncthreads();
}

// red.release + per-block polling of a counter (no reset): arrivals counted
// monotonically, target = (iter+1)*nb
__device__ void barrier_mono(unsigned* count, unsigned nb, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(count, 1u);
        while (ld_acq(count) < target) {
        }
    }
    __syncthreads();
}

template <int SLEEP>
__global__ void k_bar(unsigned* st, int iters) {
    for (int i = 0; i < iters; ++i) barrier<SLEEP>(st, st + 1, gridDim.x);
}
__global__ void k_bar_mono(unsigned* st, int iters) {
    for (int i = 0; i < iters; ++i) barrier_mono(st + 2, gridDim.x, (unsigned)(i + 1) * gridDim.x);
}

// point-to-point hop: block b waits for block b-1's flag then sets its own
__global__ void k_chain(unsigned* flags, int rounds) {
    for (int r = 1; r <= rounds; ++r) {
        if (threadIdx.x == 0) {
            if (blockIdx.x > 0)
                while (ld_acq(flags + blockIdx.x - 1) < (unsigned)r) {
                }
            else if (r > 1)
                while (ld_acq(flags + gridDim.x - 1) < (unsigned)(r - 1)) {
                }
            __threadfence();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x), "r"((unsigned)r)
                         : "memory");
        }
        __syncthreads();
    }
}

int main() {
    unsigned* st;
    cudaMalloc(&st, 4096 * sizeof(unsigned));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 2000;
    for (int blocks : {148, 296}) {
        for (int variant = 0; variant < 4; ++variant) {
            cudaMemset(st, 0, 4096 * sizeof(unsigned));
            void* args[] = {&st, (void*)&iters};
            int it = iters;
            void* args2[] = {&st, &it};
            cudaEventRecord(a);
            if (variant == 0) cudaLaunchCooperativeKernel((void*)k_bar<0>, blocks, 256, args2);
            if (variant == 1) cudaLaunchCooperativeKernel((void*)k_bar<32>, blocks, 256, args2);
            if (variant == 2) cudaLaunchCooperativeKernel((void*)k_bar<200>, blocks, 256, args2);
            if (variant == 3) cudaLaunchCooperativeKernel((void*)k_bar_mono, blocks, 256, args2);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const char* names[] = {"spin", "sleep32", "sleep200", "monotonic"};
            printf("blocks=%d barrier=%s: %.3f us per barrier (%s)\n", blocks, names[variant], ms * 1000 / iters,
                   cudaGetErrorString(cudaGetLastError()));
            (void)args;
        }
    }
    {
        int rounds = 50;
        cudaMemset(st, 0, 4096 * sizeof(unsigned));
        void* args[] = {&st, &rounds};
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_chain, 148, 128, args);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("point-to-point flag hop: %.3f us per hop (%s)\n", ms * 1000 / (rounds * 148.0),
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
