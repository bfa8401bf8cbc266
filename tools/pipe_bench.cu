// Microbenchmark: per-step cost of the producer/consumer mbarrier protocol used
// by k_gconv_tc, without any data movement. NP producer warps arrive on a
// stage's FULL barrier (per-thread cp.async.mbarrier.arrive.noinc, per-thread
// mbarrier.arrive, or one arrive per warp); one consumer warp waits FULL and
// arrives EMPTY. 5 stages. Reports cycles per step (CTA 0).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_bench pipe_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su(b)), "r"(c)); }
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}" :: "r"(su(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" :: "r"(su(b)) : "memory");
}
__device__ __forceinline__ void mb_arrive_noinc(uint64_t* b) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" :: "r"(su(b)) : "memory");
}

template <int NP, int MODE>
__global__ void k_pipe(int steps, long long* out) {
    constexpr int S = 5;
    __shared__ uint64_t full[S], empty[S];
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mb_init(&full[i], MODE == 2 ? NP : NP * 32);
            mb_init(&empty[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (w < NP) {
        int st = 0; uint32_t ph = 0;
        for (int i = 0; i < steps; ++i) {
            mb_wait(&empty[st], ph ^ 1);
            if (MODE == 0) mb_arrive_noinc(&full[st]);
            else if (MODE == 1) mb_arrive(&full[st]);
            else { __syncwarp(); if (lane == 0) mb_arrive(&full[st]); }
            if (++st == S) { st = 0; ph ^= 1; }
        }
    } else if (w == NP) {
        int st = 0; uint32_t ph = 0;
        long long t0 = clock64();
        for (int i = 0; i < steps; ++i) {
            mb_wait(&full[st], ph);
            if (lane == 0) mb_arrive(&empty[st]);
            __syncwarp();
            if (++st == S) { st = 0; ph ^= 1; }
        }
        if (lane == 0 && blockIdx.x == 0) *out = (clock64() - t0) / steps;
    }
}

int main() {
    long long* d; cudaMalloc(&d, 8);
    auto run = [&](auto k, int np, const char* nm) {
        k<<<148, (np + 1) * 32>>>(2000, d);
        k<<<148, (np + 1) * 32>>>(2000, d);
        long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("%-40s NP=%2d  %lld cycles/step\n", nm, np, c);
    };
    run(k_pipe<8, 0>, 8, "per-thread cp.async.mbarrier.arrive.noinc");
    run(k_pipe<16, 0>, 16, "per-thread cp.async.mbarrier.arrive.noinc");
    run(k_pipe<8, 1>, 8, "per-thread mbarrier.arrive");
    run(k_pipe<16, 1>, 16, "per-thread mbarrier.arrive");
    run(k_pipe<8, 2>, 8, "per-warp mbarrier.arrive");
    run(k_pipe<16, 2>, 16, "per-warp mbarrier.arrive");
    return 0;
}
