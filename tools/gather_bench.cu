// Microbenchmark: row-gather -> shared memory throughput per SM on B200.
// X = [N][64] fp16 rows (128 B, L2 resident), random row indices; each CTA
// streams 128-row tiles (16 KB) into an 8-stage smem ring. Variants:
//   1 cp.async.cg 16B (8 lanes per row, 4 warps), wait_group pipelining
//   2 cp.async.ca 16B
//   3 ld.global.v4 -> st.shared.v4 (4 warps)
//   4 TMA tile::gather4, 4 warps x 8 gathers, single issuing thread per warp
//   5 TMA tile::gather4, 8 warps x 4 gathers
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int ROWB = 128, TILE = 128, STAGES = 8;

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128) v_cpasync(const uint4* __restrict__ x, const int* __restrict__ idx,
                                                int tiles, int ca, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int t = threadIdx.x, q = t % 8, r0 = t / 8;
    for (int tile = 0; tile < tiles; ++tile) {
        const int* id = idx + ((size_t)blockIdx.x * tiles + tile) * TILE;
        uint8_t* st = sm + (tile % STAGES) * TILE * ROWB;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            int r = r0 + 16 * i;
            const uint4* src = x + (size_t)id[r] * 8 + q;
            uint32_t dst = su(st + r * ROWB + q * 16);
            if (ca) asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src));
            else asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src));
        }
        asm volatile("cp.async.commit_group;");
        asm volatile("cp.async.wait_group 6;");
    }
    asm volatile("cp.async.wait_group 0;");
    __syncthreads();
    if (t == 0) sink[blockIdx.x] = sm[5];
}

__global__ void __launch_bounds__(128) v_ldg(const uint4* __restrict__ x, const int* __restrict__ idx,
                                            int tiles, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int t = threadIdx.x, q = t % 8, r0 = t / 8;
    for (int tile = 0; tile < tiles; ++tile) {
        const int* id = idx + ((size_t)blockIdx.x * tiles + tile) * TILE;
        uint4* st = reinterpret_cast<uint4*>(sm + (tile % STAGES) * TILE * ROWB);
        uint4 v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __ldg(x + (size_t)id[r0 + 16 * i] * 8 + q);
#pragma unroll
        for (int i = 0; i < 8; ++i) st[(r0 + 16 * i) * 8 + q] = v[i];
    }
    __syncthreads();
    if (t == 0) sink[blockIdx.x] = sm[5];
}

__device__ __forceinline__ void mb_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su(b)), "r"(c)); }
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred P;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" :: "r"(su(b)), "r"(ph) : "memory");
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) v_tma(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx,
                                                     int tiles, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + STAGES * TILE * ROWB);
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    constexpr int G = 32 / WARPS;  // gathers per warp per tile
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mb_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (lane == 0) {
        for (int tile = 0; tile < tiles; ++tile) {
            const int s = tile % STAGES;
            if (tile >= STAGES) mb_wait(&bar[s], ((tile / STAGES) - 1) & 1);
            // all warps need the previous phase done before re-arming
            const int* id = idx + ((size_t)blockIdx.x * tiles + tile) * TILE + w * 4 * G;
            if (w == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su(&bar[s])), "r"(TILE * ROWB));
            uint32_t dst = su(sm + s * TILE * ROWB + w * 4 * G * ROWB);
#pragma unroll
            for (int g = 0; g < G; ++g) {
                int4 r = *reinterpret_cast<const int4*>(id + 4 * g);
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                             :: "r"(dst + g * 4 * ROWB), "l"((uint64_t)&tm), "r"(0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w), "r"(su(&bar[s])) : "memory");
            }
        }
        for (int s = 0; s < STAGES; ++s) {
            int tile = tiles - STAGES + s;
            if (tile >= 0) mb_wait(&bar[tile % STAGES], (tile / STAGES) & 1);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) sink[blockIdx.x] = sm[5];
}

int main() {
    const int N = 100000, SMS = 148, TILES = 512;
    std::vector<uint16_t> hx((size_t)N * 64, 0x3c00);
    std::vector<int> hi((size_t)SMS * TILES * TILE);
    srand(1);
    for (auto& v : hi) v = rand() % N;
    uint4* x; int* idx; unsigned long long* sink;
    CK(cudaMalloc(&x, hx.size() * 2)); CK(cudaMalloc(&idx, hi.size() * 4)); CK(cudaMalloc(&sink, SMS * 8));
    CK(cudaMemcpy(x, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(idx, hi.data(), hi.size() * 4, cudaMemcpyHostToDevice));
    const size_t smem = STAGES * TILE * ROWB + 1024;
    CUtensorMap tm;
    {
        void* f; cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
        auto enc = (CUresult(*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill))f;
        cuuint64_t dims[2] = {64, (cuuint64_t)N}, str[1] = {128};
        cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r) { printf("encode failed %d\n", r); return 1; }
    }
    auto attr = [&](const void* k) { CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); };
    attr((const void*)v_cpasync); attr((const void*)v_ldg); attr((const void*)v_tma<4>); attr((const void*)v_tma<8>); attr((const void*)v_tma<32>);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const double bytes = (double)SMS * TILES * TILE * ROWB;
    for (int v = 1; v <= 6; ++v) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            if (v == 1) v_cpasync<<<SMS, 128, smem>>>(x, idx, TILES, 0, sink);
            if (v == 2) v_cpasync<<<SMS, 128, smem>>>(x, idx, TILES, 1, sink);
            if (v == 3) v_ldg<<<SMS, 128, smem>>>(x, idx, TILES, sink);
            if (v == 4) v_tma<4><<<SMS, 128, smem>>>(tm, idx, TILES, sink);
            if (v == 5) v_tma<8><<<SMS, 256, smem>>>(tm, idx, TILES, sink);
            if (v == 6) v_tma<32><<<SMS, 1024, smem>>>(tm, idx, TILES, sink);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep == 2) {
                const char* nm[] = {"", "cp.async.cg", "cp.async.ca", "ldg+sts", "tma gather4 4w", "tma gather4 8w", "tma gather4 32w"};
                printf("%-16s %8.3f ms  %7.1f GB/s total  %6.1f B/cyc/SM @1.9GHz\n", nm[v], ms, bytes / ms / 1e6,
                       bytes / (ms * 1e-3) / SMS / 1.9e9);
            }
        }
    }
    CK(cudaGetLastError());
    return 0;
}
