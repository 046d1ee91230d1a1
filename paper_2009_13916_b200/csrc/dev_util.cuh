// Device-side helpers: warp reductions, searches, relaxed/acquire memory ops.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace edfa {

// Sentinel marking "not yet computed" in sync-free solves: a negative
// signalling NaN with a fixed payload.  Arithmetic never produces it (results
// are quieted and canonicalised before they are published).
constexpr unsigned long long SENTINEL_BITS = 0xFFF40000DEADBEEFull;
constexpr long long SPIN_LIMIT = 1ll << 22;   // bounded spins -> error flag, never a hang

__device__ __forceinline__ double ld_relaxed(const double* p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_relaxed_i(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(double* p, double v) {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

__device__ __forceinline__ bool is_sentinel(double v) {
    return (unsigned long long)__double_as_longlong(v) == SENTINEL_BITS;
}
__device__ __forceinline__ double publishable(double v) {
    // canonicalise NaNs so a published value can never equal the sentinel
    return isnan(v) ? __longlong_as_double(0x7FF8000000000000ll) : v;
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
template <class T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        T w = __shfl_xor_sync(0xffffffffu, v, o);
        v = v > w ? v : w;
    }
    return v;
}

// Software grid barrier for cooperative (co-resident) persistent launches:
// one arrival atomic per block, the last arriver bumps the generation.
__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned g;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(gen) : "memory");
        __threadfence();
        if (atomicAdd(count, 1u) == nblocks - 1) {
            *count = 0;
            __threadfence();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gen), "r"(g + 1) : "memory");
        } else {
            unsigned v;
            unsigned ns = 8;
            do {
                __nanosleep(ns);
                if (ns < 64) ns <<= 1;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gen) : "memory");
            } while (v == g);
        }
    }
    __syncthreads();
}

// position of key in sorted a[lo, hi) or -1
__device__ __forceinline__ int bsearch(const int32_t* a, int lo, int hi, int key) {
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        int v = a[mid];
        if (v == key) return mid;
        if (v < key) lo = mid + 1;
        else hi = mid;
    }
    return -1;
}
// first position in sorted a[lo, hi) with a[p] >= key
__device__ __forceinline__ int lower_bound(const int32_t* a, int lo, int hi, int key) {
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// IEEE operations without contraction, used where the reference's scalar
// Python/C arithmetic is mirrored operation for operation.
__device__ __forceinline__ double sub_mul(double a, double b, double c) {
    return __dsub_rn(a, __dmul_rn(b, c));
}
__device__ __forceinline__ double add_mul(double a, double b, double c) {
    return __dadd_rn(a, __dmul_rn(b, c));
}

}  // namespace edfa
