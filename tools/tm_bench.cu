// Microbenchmarks for the A-in-TMEM (tcgen05 "TS") gathered GEMM design.
//   part 1: correctness of kind::f16 MMA with A read from TMEM (lane = row,
//           32-bit column = 2 consecutive K elements), B K-major SW128 in smem
//   part 2: MMA issue throughput, A from TMEM vs A from smem, N = 64/128/256
//   part 3: row-gather throughput per SM into TMEM / smem for three index
//           patterns: random over 100k rows (L2), window of 256 rows per
//           tile (L1 reuse), one zero row (sentinel)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tm_bench tm_bench.cu
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su(b)), "r"(c)); }
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}" :: "r"(su(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" :: "r"(su(b)) : "memory");
}
__device__ __forceinline__ void tm_alloc(uint32_t* slot, uint32_t n) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(su(slot)), "r"(n) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tm_dealloc(uint32_t a, uint32_t n) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ void fb() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fa() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bd, uint32_t id, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                 :: "r"(d), "r"(a), "l"(bd), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t ad, uint64_t bd, uint32_t id, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                 :: "r"(d), "l"(ad), "l"(bd), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit(uint64_t* b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su(b)) : "memory");
}
#define R32(r) "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), \
    "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), \
    "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), \
    "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
__device__ __forceinline__ void tm_st32(uint32_t a, const uint32_t (&r)[32]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                 "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" :: "r"(a), R32(r) : "memory");
}
__device__ __forceinline__ void tm_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_ld32(uint32_t a, uint32_t (&r)[32]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                   "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                   "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(a));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// K-major SW128 descriptor (rows of 128 B, 8-row atoms of 1024 B)
__device__ __forceinline__ uint64_t desc128(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint32_t swz128(int r, int q) {
    uint32_t off = (uint32_t)r * 128 + (uint32_t)q * 16;
    return off ^ (((off >> 7) & 7) << 4);
}
__host__ __device__ constexpr uint32_t idesc_f16(int n) {
    // D f32 (bit 4), A/B f16 (fmt 0), K-major both, N>>3 at 17, M>>4 at 24
    return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

// ---------------- part 1: TS correctness (M=128, N=64, K=64) ----------------
__global__ void __launch_bounds__(128) k_ts_check(const __half* A, const __half* B, float* D, int ts) {
    extern __shared__ __align__(1024) uint8_t sb[];  // B 8 KB, A 16 KB, bar, slot
    uint64_t& bar = *reinterpret_cast<uint64_t*>(sb + 24576);
    uint32_t& slot = *reinterpret_cast<uint32_t*>(sb + 24584);
    const int t = threadIdx.x, w = t / 32;
    if (su(sb) & 1023) __trap();
    // B: [64 n][64 k] K-major -> SW128; A (SS mode): [128][64] SW128 after B
    for (int i = t; i < 64 * 8; i += 128) {
        int r = i / 8, q = i % 8;
        *reinterpret_cast<uint4*>(sb + swz128(r, q)) = reinterpret_cast<const uint4*>(B)[r * 8 + q];
    }
    for (int i = t; i < 128 * 8; i += 128) {
        int r = i / 8, q = i % 8;
        *reinterpret_cast<uint4*>(sb + 8192 + swz128(r, q)) = reinterpret_cast<const uint4*>(A)[r * 8 + q];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (t == 0) { mb_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    if (w == 0) tm_alloc(&slot, 256);
    fb(); __syncthreads(); fa();
    const uint32_t tm = slot;
    // thread t = row t: write its 64 halves (32 cols) at column 128
    uint32_t r[32];
    const uint32_t* arow = reinterpret_cast<const uint32_t*>(A + t * 64);
    for (int i = 0; i < 32; ++i) r[i] = arow[i];
    tm_st32(tm + ((uint32_t)(w * 32) << 16) + 128, r);
    tm_st_wait();
    fb(); __syncthreads(); fa();
    if (t == 0) {
        uint64_t bd = desc128(su(sb)), ad = desc128(su(sb + 8192));
        for (int kk = 0; kk < 4; ++kk) {
            if (ts) mma_ts(tm, tm + 128 + kk * 8, bd + kk * 2, idesc_f16(64), kk > 0);
            else mma_ss(tm, ad + kk * 2, bd + kk * 2, idesc_f16(64), kk > 0);
        }
        commit(&bar);
    }
    mb_wait(&bar, 0);
    fa();
    uint32_t o[32];
    for (int c = 0; c < 64; c += 32) {
        tm_ld32(tm + ((uint32_t)(w * 32) << 16) + c, o);
        for (int i = 0; i < 32; ++i) D[t * 64 + c + i] = __uint_as_float(o[i]);
    }
    fb(); __syncthreads(); fa();
    if (w == 0) tm_dealloc(tm, 256);
}

// ---------------- part 2: MMA throughput ----------------
template <int N, bool TS>
__global__ void __launch_bounds__(128) k_mma_rate(int iters, long long* cyc) {
    extern __shared__ __align__(1024) uint8_t sm[];  // A 16 KB + B N*128, bar, slot
    uint64_t& bar = *reinterpret_cast<uint64_t*>(sm + 16384 + N * 128);
    uint32_t& slot = *reinterpret_cast<uint32_t*>(sm + 16384 + N * 128 + 8);
    const int t = threadIdx.x, w = t / 32;
    for (int i = t; i < (16384 + N * 128) / 16; i += 128) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (t == 0) { mb_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    if (w == 0) tm_alloc(&slot, 512);
    fb(); __syncthreads(); fa();
    const uint32_t tm = slot;
    if (t == 0) {
        const uint64_t ad = desc128(su(sm)), bd = desc128(su(sm + 16384));
        long long c0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                if (TS) mma_ts(tm, tm + 256 + kk * 8, bd + kk * 2, idesc_f16(N), 1);
                else mma_ss(tm, ad + kk * 2, bd + kk * 2, idesc_f16(N), 1);
            }
        }
        commit(&bar);
        mb_wait(&bar, 0);
        long long c1 = clock64();
        if (blockIdx.x == 0) cyc[0] = c1 - c0;
    }
    fb(); __syncthreads(); fa();
    if (w == 0) tm_dealloc(tm, 512);
}

// ---------------- part 3: gather into TMEM (thread per row) ----------------
// X [n][64] fp16; idx [tiles][128]; each of NW warps handles lane quadrant
// (w % 4); warps w and w+4 alternate tiles. Stage = 32 TMEM columns.
template <int NW, bool SMEM_T>
__global__ void __launch_bounds__(NW * 32) k_gather_tm(const uint4* __restrict__ x, const int* __restrict__ idx,
                                                      int tiles, unsigned long long* sink) {
    __shared__ uint32_t slot;
    const int t = threadIdx.x, w = t / 32, lane = t % 32, quad = w % 4, grp = w / 4;
    if (w == 0) tm_alloc(&slot, 512);
    fb(); __syncthreads(); fa();
    const uint32_t tm = slot + ((uint32_t)(quad * 32) << 16);
    constexpr int G = NW / 4;
    const int* base = idx + (size_t)blockIdx.x * tiles * 128;
    uint32_t r[32];
    for (int tile = grp; tile < tiles; tile += G) {
        const int row = base[tile * 128 + quad * 32 + lane];
        const uint4* src = x + (size_t)row * 8;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            uint4 v = __ldg(src + q);
            r[4 * q] = v.x; r[4 * q + 1] = v.y; r[4 * q + 2] = v.z; r[4 * q + 3] = v.w;
        }
        tm_st32(tm + (uint32_t)((tile / G) % 8) * 32 + 256 * 0, r);
    }
    tm_st_wait();
    fb(); __syncthreads(); fa();
    if (t == 0) sink[blockIdx.x] = r[3];
    if (w == 0) tm_dealloc(slot, 512);
}

// coalesced gather (8 lanes per row) into registers only (upper bound of LDG path)
template <int NW>
__global__ void __launch_bounds__(NW * 32) k_gather_coal(const uint4* __restrict__ x, const int* __restrict__ idx,
                                                        int tiles, unsigned long long* sink) {
    const int t = threadIdx.x, q = t % 8, r0 = t / 8;
    constexpr int RS = NW * 32 / 8;
    const int* base = idx + (size_t)blockIdx.x * tiles * 128;
    uint32_t acc = 0;
    for (int tile = 0; tile < tiles; ++tile) {
        uint4 v[128 / RS];
#pragma unroll
        for (int i = 0; i < 128 / RS; ++i) v[i] = __ldg(x + (size_t)base[tile * 128 + r0 + i * RS] * 8 + q);
#pragma unroll
        for (int i = 0; i < 128 / RS; ++i) acc ^= v[i].x ^ v[i].w;
    }
    if (acc == 0x12345) sink[blockIdx.x] = acc;
}

// cp.async 16B (8 lanes per row) into a smem ring, NW warps
template <int NW, bool CA>
__global__ void __launch_bounds__(NW * 32) k_gather_cp(const uint4* __restrict__ x, const int* __restrict__ idx,
                                                      int tiles, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int t = threadIdx.x, q = t % 8, r0 = t / 8;
    constexpr int RS = NW * 32 / 8;
    const int* base = idx + (size_t)blockIdx.x * tiles * 128;
    for (int tile = 0; tile < tiles; ++tile) {
        uint8_t* st = sm + (tile % 8) * 16384;
#pragma unroll
        for (int i = 0; i < 128 / RS; ++i) {
            int r = r0 + i * RS;
            const uint4* src = x + (size_t)max(base[tile * 128 + r], 0) * 8 + q;
            uint32_t dst = su(st + swz128(r, q));
            const int id = base[tile * 128 + r];
            if (id < 0) { if (!CA) asm volatile("cp.async.cg.shared.global [%0], [%1], 16, 0;" :: "r"(dst), "l"(x)); }
            else if (CA) asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src));
            else asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src));
        }
        asm volatile("cp.async.commit_group;");
        asm volatile("cp.async.wait_group 6;");
    }
    asm volatile("cp.async.wait_group 0;");
    __syncthreads();
    if (t == 0) sink[blockIdx.x] = sm[5];
}

template <int NW, int MODE>
__global__ void __launch_bounds__(NW * 32) k_scatter(float* __restrict__ y, const int* __restrict__ idx, int tiles,
                                                    unsigned long long* sink) {
    // 128-row tiles of 64 fp32 (256 B rows), 16 lanes per row, v4 each
    const int t = threadIdx.x, q = t % 16, r0 = t / 16;
    constexpr int RS = NW * 32 / 16;
    const int* base = idx + (size_t)blockIdx.x * tiles * 128;
    for (int tile = 0; tile < tiles; ++tile) {
#pragma unroll 4
        for (int r = r0; r < 128; r += RS) {
            float* dst = y + (size_t)base[tile * 128 + r] * 64 + q * 4;
            if (MODE == 0) asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" :: "l"(dst), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
            else *reinterpret_cast<float4*>(dst) = make_float4(1.f, 1.f, 1.f, 1.f);
        }
    }
}

int main() {
    // ---- part 1
    {
        std::vector<__half> hA(128 * 64), hB(64 * 64);
        std::vector<float> fA(128 * 64), fB(64 * 64);
        srand(3);
        for (int i = 0; i < 128 * 64; ++i) { float v = (rand() % 17 - 8) / 8.f; hA[i] = __float2half(v); fA[i] = v; }
        for (int i = 0; i < 64 * 64; ++i) { float v = (rand() % 17 - 8) / 8.f; hB[i] = __float2half(v); fB[i] = v; }
        __half *dA, *dB; float* dD;
        CK(cudaMalloc(&dA, 128 * 64 * 2)); CK(cudaMalloc(&dB, 64 * 64 * 2)); CK(cudaMalloc(&dD, 128 * 64 * 4));
        CK(cudaMemcpy(dA, hA.data(), 128 * 64 * 2, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dB, hB.data(), 64 * 64 * 2, cudaMemcpyHostToDevice));
        for (int ts = 0; ts < 2; ++ts) {
            CK(cudaMemset(dD, 0, 128 * 64 * 4));
            k_ts_check<<<1, 128, 24576 + 64>>>(dA, dB, dD, ts);
            CK(cudaDeviceSynchronize());
            std::vector<float> hD(128 * 64);
            CK(cudaMemcpy(hD.data(), dD, 128 * 64 * 4, cudaMemcpyDeviceToHost));
            double err = 0;
            for (int m = 0; m < 128; ++m)
                for (int n = 0; n < 64; ++n) {
                    double s = 0;
                    for (int k = 0; k < 64; ++k) s += fA[m * 64 + k] * fB[n * 64 + k];
                    err = fmax(err, fabs(s - hD[m * 64 + n]));
                }
            printf("part1 %s max abs err %.3g (D[0]=%f)\n", ts ? "TS (A in TMEM)" : "SS (A in smem)", err, hD[0]);
        }
    }
    // ---- part 2
    {
        long long* dc; CK(cudaMalloc(&dc, 8));
        auto run = [&](auto kern, int n, const char* nm) {
            size_t smem = 16384 + n * 128 + 1024;
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            const int iters = 4096;
            for (int rep = 0; rep < 2; ++rep) kern<<<148, 128, smem>>>(iters, dc);
            CK(cudaDeviceSynchronize());
            long long c; CK(cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost));
            double fma = (double)iters * 4 * 128 * n * 16;
            printf("part2 %-4s N=%3d: %.1f cyc per K=16 MMA, %.0f FMA/cyc/SM\n", nm, n, (double)c / (iters * 4), fma / c);
        };
        run(k_mma_rate<64, false>, 64, "SS"); run(k_mma_rate<64, true>, 64, "TS");
        run(k_mma_rate<128, false>, 128, "SS"); run(k_mma_rate<128, true>, 128, "TS");
        run(k_mma_rate<256, false>, 256, "SS"); run(k_mma_rate<256, true>, 256, "TS");
    }
    // ---- part 3
    {
        const int N = 100000, SMS = 148, TILES = 512;
        std::vector<uint16_t> hx((size_t)(N + 1) * 64, 0x3c00);
        uint4* x; int* idx; unsigned long long* sink;
        CK(cudaMalloc(&x, hx.size() * 2)); CK(cudaMalloc(&idx, (size_t)SMS * TILES * 128 * 4)); CK(cudaMalloc(&sink, SMS * 8));
        CK(cudaMemcpy(x, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice));
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        const double bytes = (double)SMS * TILES * 128 * 128;
        for (int pat = 0; pat < 5; ++pat) {
            std::vector<int> hi((size_t)SMS * TILES * 128);
            srand(1);
            for (size_t i = 0; i < hi.size(); ++i) {
                const size_t tile = i / 128;
                if (pat == 0) hi[i] = rand() % N;
                else if (pat == 1) hi[i] = (int)((tile / 16 * 997) % (N - 256)) + rand() % 256;  // 16 tiles share a 256-row window
                else if (pat == 2) hi[i] = N;
                else if (pat == 3) hi[i] = -1;
                else hi[i] = (rand() % 2) ? -1 : rand() % N;
            }
            CK(cudaMemcpy(idx, hi.data(), hi.size() * 4, cudaMemcpyHostToDevice));
            const char* pn[] = {"random100k", "window256", "zero-row", "zfill-all", "zfill-half"};
            auto run = [&](auto kern, int threads, size_t smem, const char* nm) {
                if (smem) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                float ms = 0;
                for (int rep = 0; rep < 3; ++rep) {
                    cudaEventRecord(a);
                    kern<<<SMS, threads, smem>>>(x, idx, TILES, sink);
                    cudaEventRecord(b);
                    CK(cudaEventSynchronize(b));
                    cudaEventElapsedTime(&ms, a, b);
                }
                CK(cudaGetLastError());
                printf("part3 %-10s %-22s %7.3f ms %7.1f GB/s %6.1f B/cyc/SM @1.9GHz\n", pn[pat], nm, ms, bytes / ms / 1e6,
                       bytes / (ms * 1e-3) / SMS / 1.9e9);
            };
            if (pat < 3) {
            run(k_gather_tm<4, false>, 128, 0, "ldg row/thread->tmem 4w");
            run(k_gather_tm<8, false>, 256, 0, "ldg row/thread->tmem 8w");
            run(k_gather_tm<16, false>, 512, 0, "ldg row/thread->tmem16w");
            run(k_gather_coal<4>, 128, 0, "ldg coalesced 4w");
            run(k_gather_coal<8>, 256, 0, "ldg coalesced 8w");
            run(k_gather_coal<16>, 512, 0, "ldg coalesced 16w");
            }
            run(k_gather_cp<4, false>, 128, 8 * 16384 + 1024, "cp.async.cg 4w");
            run(k_gather_cp<8, false>, 256, 8 * 16384 + 1024, "cp.async.cg 8w");
            run(k_gather_cp<8, true>, 256, 8 * 16384 + 1024, "cp.async.ca 8w");
            run(k_gather_cp<16, true>, 512, 8 * 16384 + 1024, "cp.async.ca 16w(skip)");
            run(k_gather_cp<16, false>, 512, 8 * 16384 + 1024, "cp.async.cg 16w");
            run(k_gather_cp<24, false>, 768, 8 * 16384 + 1024, "cp.async.cg 24w");
            run(k_gather_cp<32, false>, 1024, 8 * 16384 + 1024, "cp.async.cg 32w");
        }
    }
    {
        const int N = 130000, SMS = 148, TILES = 64;
        float* y; int* idx; unsigned long long* sink;
        CK(cudaMalloc(&y, (size_t)N * 64 * 4)); CK(cudaMalloc(&idx, (size_t)SMS * TILES * 128 * 4)); CK(cudaMalloc(&sink, SMS * 8));
        std::vector<int> hi((size_t)SMS * TILES * 128);
        for (auto& v : hi) v = rand() % N;
        CK(cudaMemcpy(idx, hi.data(), hi.size() * 4, cudaMemcpyHostToDevice));
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        const double bytes = (double)SMS * TILES * 128 * 256;
        auto run = [&](auto kern, int threads, const char* nm) {
            float ms = 0;
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(a);
                kern<<<SMS, threads>>>(y, idx, TILES, sink);
                cudaEventRecord(b);
                CK(cudaEventSynchronize(b));
                cudaEventElapsedTime(&ms, a, b);
            }
            printf("part4 %-24s %7.3f ms %7.1f GB/s\n", nm, ms, bytes / ms / 1e6);
        };
        run(k_scatter<4, 0>, 128, "red.add.v4 4w");
        run(k_scatter<8, 0>, 256, "red.add.v4 8w");
        run(k_scatter<4, 1>, 128, "st.v4 4w");
        run(k_scatter<8, 1>, 256, "st.v4 8w");
    }
    return 0;
}
