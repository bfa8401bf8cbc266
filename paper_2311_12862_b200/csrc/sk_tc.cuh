// tcgen05 / TMA / mbarrier helpers shared by the gathered-GEMM (conv.cu),
// dense identity-map (dense.cu) and wgrad kernels. sm_100a only.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "sk_common.cuh"

namespace sk {

// 2D row-major [rows][cols] fp16/bf16 tensor map, box {kc, box_rows}, swizzle
// = kc*2 bytes (conv.cu)
CUtensorMap make_tmap(const void* base, sk_dtype dt, int cols, long long rows, int kc,
                      int box_rows);
CUtensorMap make_tmap_rows(const void* base, CUtensorMapDataType ty, int elem_bytes, long long cols,
                           long long rows, long long ld, int box_cols, int box_rows);

template <typename T>
struct Fmt;
template <>
struct Fmt<__half> {
    static constexpr uint32_t v = 0;
};
template <>
struct Fmt<__nv_bfloat16> {
    static constexpr uint32_t v = 1;
};

__device__ __forceinline__ uint32_t pack2(float a, float b, __half*) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ uint32_t pack2(float a, float b, __nv_bfloat16*) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float2 unpack2(uint32_t u, __half*) {
    return __half22float2(*reinterpret_cast<__half2*>(&u));
}
__device__ __forceinline__ float2 unpack2(uint32_t u, __nv_bfloat16*) {
    return __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u));
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap* tm, int col, int r0,
                                            int r1, int r2, int r3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
        "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_tile2d(uint32_t dst, const CUtensorMap* tm, int c0, int c1,
                                           uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
// whole-warp (uniform) callers: one elected lane issues
__device__ __forceinline__ void tma_gather4_elect(uint32_t dst, const CUtensorMap* tm, int col,
                                                  int r0, int r1, int r2, int r3, uint64_t* bar) {
    asm volatile(
        "{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\n"
        "@P cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n}" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
        "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_tile2d_elect(uint32_t dst, const CUtensorMap* tm, int c0, int c1,
                                                 uint64_t* bar) {
    asm volatile(
        "{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\n"
        "@P cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];\n}" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(dst),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void bulk_g2s_elect(uint32_t dst, const void* src, uint32_t bytes,
                                               uint64_t* bar) {
    asm volatile(
        "{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\n"
        "@P cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n}" ::
            "r"(dst),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// K-major smem descriptor; row = KC*2 bytes, 8-row swizzle atoms (SBO).
template <int KC>
__device__ __forceinline__ uint64_t kmajor_desc(uint32_t saddr) {
    constexpr uint32_t RB = KC * 2;                                  // 32 / 64 / 128
    constexpr uint64_t layout = RB == 128 ? 2 : (RB == 64 ? 4 : 6);  // SW128/SW64/SW32
    constexpr uint64_t sbo = (8 * RB) >> 4;
    return (uint64_t)((saddr >> 4) & 0x3FFF) | (sbo << 32) | (1ull << 46) | (layout << 61);
}

// byte offset of 16B chunk q of row r inside a K-major swizzled tile whose
// base is aligned to the swizzle repeat (Swizzle<B,4,3>: bits[4,4+B) ^= bits[7,7+B))
template <int KC>
__device__ __forceinline__ uint32_t swz(int r, int q) {
    constexpr uint32_t RB = KC * 2;
    constexpr uint32_t B = RB == 128 ? 7 : (RB == 64 ? 3 : 1);
    const uint32_t off = (uint32_t)r * RB + (uint32_t)q * 16;
    return off ^ (((off >> 7) & B) << 4);
}

__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// One K step of both 128-row halves (KC/16 MMAs each, interleaved so they
// share the B stage), then commit -> bar. Called by the whole warp with
// uniform operands; elect.sync picks the issuing lane.
// two == 0: only the first half (an item of one 128-row tile).
template <int KC>
__device__ __forceinline__ void tc_mma_step_f16(uint32_t d0, uint32_t d1, uint64_t a0, uint64_t a1,
                                                uint64_t b, uint32_t idesc, uint32_t accumulate,
                                                uint64_t* bar, uint32_t two = 1) {
#pragma unroll
    for (int kk = 0; kk < KC / 16; ++kk) {
        const uint32_t acc = (kk > 0 || accumulate) ? 1u : 0u;
        asm volatile(
            "{\n.reg .pred E, p, q, E2;\n"
            "elect.sync _|E, 0xffffffff;\n"
            "setp.ne.b32 p, %6, 0;\n"
            "setp.ne.and.b32 E2, %7, 0, E;\n"
            "@E tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %4, %5, p;\n"
            "@E2 tcgen05.mma.cta_group::1.kind::f16 [%1], %3, %4, %5, p;\n"
            "}\n" ::"r"(d0),
            "r"(d1), "l"(a0 + (uint64_t)(kk * 2)), "l"(a1 + (uint64_t)(kk * 2)),
            "l"(b + (uint64_t)(kk * 2)), "r"(idesc), "r"(acc), "r"(two)
            : "memory");
    }
    if (bar)
        asm volatile(
            "{\n.reg .pred E;\nelect.sync _|E, 0xffffffff;\n"
            "@E tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(
                smem_u32(bar))
            : "memory");
}
__device__ __forceinline__ void tc_commit_elect(uint64_t* bar) {
    asm volatile(
        "{\n.reg .pred E;\nelect.sync _|E, 0xffffffff;\n"
        "@E tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(
            smem_u32(bar))
        : "memory");
}

}  // namespace sk
