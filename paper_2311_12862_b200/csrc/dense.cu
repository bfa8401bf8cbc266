// Identity-map layers (K=1, stride 1, one coordinate set): the kernel map is
// the identity, so the layer is a plain dense GEMM y[n][co] = x[n][ci] W[ci][co]
// (dgrad: dx = dy W^T, optionally added into the producer's fp32 gradient sum).
// Reference path: conv_forward -> any executor over the K=1 map
// (exec.cpp:368-383, kmap.cpp:96-136 with K^D = 1).
//
// k_dense_tc: a lean persistent tcgen05 GEMM for these memory-bound shapes
// (rows up to millions, C_in/C_out <= 256 per N tile). Per CTA:
//   warp 0      TMA producer: the N tile's whole B (= W^T, [bn][C_in] K-major)
//               once per N tile, then 128-row A tiles (2D TMA, OOB rows zero)
//               into a ring of KC-channel stages
//   warp 1      TMEM owner + tcgen05.mma issuer (M=128, N=bn, K=16 steps)
//   warps 2-5   epilogue: tcgen05.ld -> fp32 (+ residual) -> T; each warp
//               stages its 32 rows in smem in the TMA-swizzled layout (no
//               bank conflicts) and writes them with TMA tensor stores
//               (cp.reduce.async.bulk.tensor .add for the fp32 gradient sum);
//               residual tiles arrive by TMA into the same staging rows
// Double-buffered TMEM accumulators overlap tile i's epilogue with tile
// i+1's MMAs; the A ring keeps several tiles of loads in flight.
// Algorithmic bytes per launch: rows*(C_in + C_out)*es (+ residual / fp32 RMW).
#include "sk_internal.hpp"
#include "sk_tc.cuh"

namespace sk {

namespace {

constexpr int kDenseM = 128;
constexpr int kDenseThreads = 320;
constexpr int kDenseEpi0 = 2;  // epilogue warps 2..9: TMEM lane quadrant = warp % 4,
                                // column half = (warp - 2) / 4

struct DenseArgs {
#ifdef SK_DENSE_TRACE
    long long* trace;
#endif
    const void* residual;  // out_mode 0: y = x W + residual ([rows][ld_y] T), or null
    void* y;
    long long rows;
    int k_total, n_total, bn, n_nt, m_tiles, items;
    int out_mode;  // 0 store T, 1 store f32, 3 add into f32 (RMW)
    int ld_y;
    int staged;    // epilogue rows contiguous (bn == ld_y): smem + one bulk copy per warp
    int stages;
    int accs;      // TMEM accumulator buffers (2 or 4)
    int cb;        // staged: bytes per row per staging chunk (32 / 64 / 128 = TMA swizzle)
    int csplit;    // epilogue warps per TMEM lane quadrant (2: each takes half the chunks)
};

__device__ __forceinline__ void tma_store2d(const CUtensorMap* tm, int c0, int c1, uint32_t src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(tm)),
                 "r"(c0), "r"(c1), "r"(src)
                 : "memory");
}
__device__ __forceinline__ void tma_store2d_add(const CUtensorMap* tm, int c0, int c1, uint32_t src) {
    asm volatile(
        "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
            reinterpret_cast<uint64_t>(tm)),
        "r"(c0), "r"(c1), "r"(src)
        : "memory");
}
__device__ __forceinline__ void bulk_commit() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <typename T, int KC>
__global__ void __launch_bounds__(kDenseThreads, 2)
    k_dense_tc(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
               const __grid_constant__ CUtensorMap tm_y, const __grid_constant__ CUtensorMap tm_r,
               const DenseArgs p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int BN = p.bn;
#ifdef SK_DENSE_TRACE
    if (blockIdx.x == 0 && threadIdx.x == 0) p.trace[0] = clock64();
#endif
    const int nchunks = (p.k_total + KC - 1) / KC;
    constexpr uint32_t kAStage = kDenseM * KC * 2;
    const uint32_t b_chunk = (uint32_t)BN * KC * 2;  // multiple of 1024 (BN % 16 == 0)
    const uint32_t b_bytes = b_chunk * nchunks;
    const int es_out = p.out_mode == 0 ? (int)sizeof(T) : 4;
    const uint32_t stage_out = p.staged ? (uint32_t)(32 * BN * es_out / p.csplit) : 0u;  // per epilogue warp
    uint8_t* b_smem = smem;
    uint8_t* a_smem = smem + b_bytes;
    uint8_t* o_smem = a_smem + (size_t)p.stages * kAStage;
    uint64_t* bars = reinterpret_cast<uint64_t*>(o_smem + 4 * p.csplit * (size_t)stage_out);
    uint64_t* full = bars;
    uint64_t* empty = bars + p.stages;
    uint64_t* tfull = bars + 2 * p.stages;
    uint64_t* tempty = tfull + 4;
    uint64_t* bfull = tempty + 4;
    uint64_t* bempty = bfull + 1;
    uint64_t* rbars = bempty + 1;  // [8] residual tile landed (per epilogue warp)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbars + 8);

    uint32_t ncols = 32;
    while (ncols < (uint32_t)(p.accs * BN)) ncols <<= 1;
    if (threadIdx.x == 0) {
        if (smem_u32(smem) & 1023) __trap();
        for (int i = 0; i < p.stages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 4; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 128 * p.csplit);
        }
        mbar_init(bfull, 1);
        mbar_init(bempty, 1);
        for (int i = 0; i < 8; ++i) mbar_init(&rbars[i], 1);
        fence_mbar_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_a)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_b)) : "memory");
    }
    if (warp == 1) tmem_alloc(tmem_slot, ncols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // the prologue (barriers, tensor-map prefetch, TMEM) overlapped the
    // predecessor's tail; global memory only after it has completed
    pdl_wait();
#ifdef SK_DENSE_TRACE
    if (blockIdx.x == 0 && threadIdx.x == 0) p.trace[63 * 8] = clock64();
#endif
    const int g = gridDim.x;

    if (warp == 0) {
        // ===== TMA producer =====
        int stage = 0, cur_nt = -1, nb = 0;
        uint32_t phase = 0;
        for (int item = blockIdx.x; item < p.items; item += g) {
            const int nt = item / p.m_tiles, mt = item % p.m_tiles;
            if (nt != cur_nt) {
                if (nb > 0) mbar_wait(bempty, (uint32_t)(nb - 1) & 1u);
                if (lane == 0) mbar_expect_tx(bfull, b_bytes);
                __syncwarp();
                for (int c = 0; c < nchunks; ++c)
                    tma_tile2d_elect(smem_u32(b_smem) + c * b_chunk, &tm_b, c * KC, nt * BN, bfull);
                cur_nt = nt;
                ++nb;
            }
            for (int c = 0; c < nchunks; ++c) {
                mbar_wait(&empty[stage], phase ^ 1);
                if (lane == 0) mbar_expect_tx(&full[stage], kAStage);
                __syncwarp();
                tma_tile2d_elect(smem_u32(a_smem) + stage * kAStage, &tm_a, c * KC, mt * kDenseM,
                                 &full[stage]);
                if (++stage == p.stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer (whole warp, elected lane inside the asm) =====
        const uint32_t idesc = (1u << 4) | (Fmt<T>::v << 7) | (Fmt<T>::v << 10) |
                               ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(kDenseM >> 4) << 24);
        const uint64_t a0 = kmajor_desc<KC>(smem_u32(a_smem));
        const uint64_t b0 = kmajor_desc<KC>(smem_u32(b_smem));
        int stage = 0, local = 0, cur_nt = -1, nb = 0;
        uint32_t phase = 0;
        for (int item = blockIdx.x; item < p.items; item += g, ++local) {
            const int nt = item / p.m_tiles;
            if (nt != cur_nt) {
                mbar_wait(bfull, (uint32_t)nb & 1u);
                cur_nt = nt;
                ++nb;
            }
            const int acc = local % p.accs;
            mbar_wait(&tempty[acc], (uint32_t)((local / p.accs) & 1) ^ 1u);
            tc_fence_after();
            const uint32_t d = tmem + (uint32_t)(acc * BN);
            for (int c = 0; c < nchunks; ++c) {
                mbar_wait(&full[stage], phase);
#ifdef SK_DENSE_TRACE
                if (blockIdx.x == 0 && lane == 0 && local < 60 && c == 0) p.trace[(1 + local) * 8 + 1] = clock64();
#endif
                tc_fence_after();
                const uint64_t da = a0 + (((uint64_t)stage * kAStage) >> 4);
                const uint64_t db = b0 + (((uint64_t)c * b_chunk) >> 4);
#pragma unroll
                for (int kk = 0; kk < KC / 16; ++kk) {
                    const uint32_t accf = (c > 0 || kk > 0) ? 1u : 0u;
                    asm volatile(
                        "{\n.reg .pred E, p;\n"
                        "elect.sync _|E, 0xffffffff;\n"
                        "setp.ne.b32 p, %4, 0;\n"
                        "@E tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
                        "}\n" ::"r"(d),
                        "l"(da + (uint64_t)(kk * 2)), "l"(db + (uint64_t)(kk * 2)), "r"(idesc),
                        "r"(accf)
                        : "memory");
                }
                tc_commit_elect(&empty[stage]);
                if (++stage == p.stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            tc_commit_elect(&tfull[acc]);
#ifdef SK_DENSE_TRACE
            if (blockIdx.x == 0 && lane == 0 && local < 60) p.trace[(1 + local) * 8 + 2] = clock64();
#endif
            const int nxt = item + g;
            if (nxt >= p.items || nxt / p.m_tiles != nt) tc_commit_elect(bempty);
            __syncwarp();
        }
    } else {
        // ===== epilogue: thread owns TMEM lane quad*32+lane = tile row. Staged
        // mode: the warp's 32 rows go to smem in the TMA swizzled layout (chunks
        // of CB bytes per row; 8 consecutive rows hit distinct banks) and leave
        // with one TMA tensor store (or .add reduction) per chunk; a residual
        // tile comes in the same way before the accumulator is read =====
        const int quad = warp & 3;
        const int ew = warp - kDenseEpi0;
        const int half = ew / 4;
        const uint32_t so = smem_u32(o_smem) + (uint32_t)ew * stage_out;
        const uint32_t CB = (uint32_t)p.cb;
        const uint32_t swm = CB == 128 ? 7u : (CB == 64 ? 3u : 1u);
        const int cw = (int)CB / es_out;  // columns per chunk
        const int nch = BN / cw / p.csplit;  // chunks of this warp
        const int ch0 = half * nch;          // first chunk of this warp
        const int c_begin = ch0 * cw, c_end = c_begin + nch * cw;
        uint64_t* rbar = rbars + ew;
        uint32_t rph = 0;
        int local = 0;
        // csplit == 1: one warp per quadrant covers all columns, the others idle
        for (int item = half < p.csplit ? (int)blockIdx.x : p.items; item < p.items; item += g, ++local) {
            const int nt = item / p.m_tiles, mt = item % p.m_tiles;
            const long long row0 = (long long)mt * kDenseM + quad * 32;
            const long long row = row0 + lane;
            const bool live = row < p.rows;
            const int acc = local % p.accs;
            const bool res = p.residual != nullptr;
            if (p.staged) {
                if (local > 0) {  // the previous stores have read the staging rows
                    if (lane == 0) bulk_wait_read0();
                    __syncwarp();
                }
                if (res) {
                    if (lane == 0) mbar_expect_tx(rbar, (uint32_t)nch * 32u * CB);
                    __syncwarp();
                    for (int ch = 0; ch < nch; ++ch)
                        tma_tile2d_elect(so + (uint32_t)ch * 32u * CB, &tm_r,
                                         nt * BN + (ch0 + ch) * cw, (int)row0, rbar);
                }
            }
            mbar_wait(&tfull[acc], (uint32_t)((local / p.accs) & 1));
#ifdef SK_DENSE_TRACE
            if (blockIdx.x == 0 && ew == 0 && lane == 0 && local < 60) p.trace[(1 + local) * 8 + 3] = clock64();
#endif
            tc_fence_after();
            if (p.staged && res) {
                mbar_wait(rbar, rph);
                rph ^= 1;
            }
            auto emit = [&](int c0, uint32_t (&v)[16]) {
                if (p.staged) {
                    const uint32_t byte = (uint32_t)c0 * es_out;
                    const uint32_t base = so + (byte / CB - (uint32_t)ch0) * 32u * CB;
                    const uint32_t roff = (uint32_t)lane * CB + byte % CB;
                    auto sw = [&](uint32_t j) {  // swizzled address of 16 B piece j
                        const uint32_t off = roff + 16u * j;
                        return base + (off ^ (((off >> 7) & swm) << 4));
                    };
                    if (p.out_mode == 0) {
                        if (res) {
#pragma unroll
                            for (uint32_t j = 0; j < 2; ++j) {
                                uint32_t r[4];
                                asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                                             : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                                             : "r"(sw(j)));
#pragma unroll
                                for (int i = 0; i < 4; ++i) {
                                    const float2 f = unpack2(r[i], (T*)nullptr);
                                    const int k = 8 * j + 2 * i;
                                    v[k] = __float_as_uint(__uint_as_float(v[k]) + f.x);
                                    v[k + 1] = __float_as_uint(__uint_as_float(v[k + 1]) + f.y);
                                }
                            }
                        }
#pragma unroll
                        for (uint32_t j = 0; j < 2; ++j) {
                            const int k = 8 * j;
                            asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(sw(j)),
                                         "r"(pack2(__uint_as_float(v[k]), __uint_as_float(v[k + 1]), (T*)nullptr)),
                                         "r"(pack2(__uint_as_float(v[k + 2]), __uint_as_float(v[k + 3]), (T*)nullptr)),
                                         "r"(pack2(__uint_as_float(v[k + 4]), __uint_as_float(v[k + 5]), (T*)nullptr)),
                                         "r"(pack2(__uint_as_float(v[k + 6]), __uint_as_float(v[k + 7]), (T*)nullptr))
                                         : "memory");
                        }
                    } else {
#pragma unroll
                        for (uint32_t j = 0; j < 4; ++j)
                            asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(sw(j)),
                                         "r"(v[4 * j]), "r"(v[4 * j + 1]), "r"(v[4 * j + 2]),
                                         "r"(v[4 * j + 3])
                                         : "memory");
                    }
                    return;
                }
                if (!live) return;
                const int col = nt * BN + c0;
                if (p.out_mode == 0) {
                    if (res) {
                        const uint4* rs = reinterpret_cast<const uint4*>(
                            static_cast<const T*>(p.residual) + (size_t)row * p.ld_y + col);
                        const uint4 r0 = rs[0], r1 = rs[1];
                        const uint32_t rr[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const float2 f = unpack2(rr[i], (T*)nullptr);
                            v[2 * i] = __float_as_uint(__uint_as_float(v[2 * i]) + f.x);
                            v[2 * i + 1] = __float_as_uint(__uint_as_float(v[2 * i + 1]) + f.y);
                        }
                    }
                    uint4 u0, u1;
                    u0.x = pack2(__uint_as_float(v[0]), __uint_as_float(v[1]), (T*)nullptr);
                    u0.y = pack2(__uint_as_float(v[2]), __uint_as_float(v[3]), (T*)nullptr);
                    u0.z = pack2(__uint_as_float(v[4]), __uint_as_float(v[5]), (T*)nullptr);
                    u0.w = pack2(__uint_as_float(v[6]), __uint_as_float(v[7]), (T*)nullptr);
                    u1.x = pack2(__uint_as_float(v[8]), __uint_as_float(v[9]), (T*)nullptr);
                    u1.y = pack2(__uint_as_float(v[10]), __uint_as_float(v[11]), (T*)nullptr);
                    u1.z = pack2(__uint_as_float(v[12]), __uint_as_float(v[13]), (T*)nullptr);
                    u1.w = pack2(__uint_as_float(v[14]), __uint_as_float(v[15]), (T*)nullptr);
                    uint4* dst = reinterpret_cast<uint4*>(static_cast<T*>(p.y) + (size_t)row * p.ld_y + col);
                    dst[0] = u0;
                    dst[1] = u1;
                } else {
                    float* dst = static_cast<float*>(p.y) + (size_t)row * p.ld_y + col;
#pragma unroll
                    for (int i = 0; i < 16; i += 4) {
                        float4 o = make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]),
                                               __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
                        if (p.out_mode == 3) {
                            const float4 q = *reinterpret_cast<const float4*>(dst + i);
                            o.x += q.x; o.y += q.y; o.z += q.z; o.w += q.w;
                        }
                        *reinterpret_cast<float4*>(dst + i) = o;
                    }
                }
            };
            const uint32_t tbase = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * BN);
            for (int c0 = c_begin; c0 < c_end; c0 += 32) {
                // two 16-column loads per wait: TMEM reads overlap
                uint32_t v0[16], v1[16];
                const bool two = c0 + 16 < c_end;
                tmem_ld16(tbase + (uint32_t)c0, v0);
                if (two) tmem_ld16(tbase + (uint32_t)(c0 + 16), v1);
                tmem_ld_wait();
                emit(c0, v0);
                if (two) emit(c0 + 16, v1);
            }
            tc_fence_before();
            mbar_arrive(&tempty[acc]);
#ifdef SK_DENSE_TRACE
            if (blockIdx.x == 0 && ew == 0 && lane == 0 && local < 60) p.trace[(1 + local) * 8 + 4] = clock64();
#endif
            if (p.staged) {
                fence_proxy_async_smem();  // generic-proxy staging writes -> TMA store
                __syncwarp();
                if (lane == 0) {
                    for (int ch = 0; ch < nch; ++ch) {
                        const uint32_t src = so + (uint32_t)ch * 32u * CB;
                        const int cx = nt * BN + (ch0 + ch) * cw;
                        if (p.out_mode == 3) tma_store2d_add(&tm_y, cx, (int)row0, src);
                        else tma_store2d(&tm_y, cx, (int)row0, src);
                    }
                    bulk_commit();
#ifdef SK_DENSE_TRACE
                    if (blockIdx.x == 0 && ew == 0 && local < 60) p.trace[(1 + local) * 8 + 5] = clock64();
#endif
                }
            }
        }
        if (p.staged && lane == 0) bulk_wait0();
    }
    pdl_trigger();  // this CTA's work is done: let the next kernel launch
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
#ifdef SK_DENSE_TRACE
    if (blockIdx.x == 0 && threadIdx.x == 0) p.trace[63 * 8 + 1] = clock64();
#endif
    if (warp == 1) tmem_dealloc(tmem, ncols);
}

template <typename T, int KC>
bool launch_dense(sk_ctx* ctx, sk_dtype dt, DenseArgs a, const void* x, const void* b,
                  cudaStream_t st) {
    const int nchunks = (int)ceil_div(a.k_total, KC);
    const size_t b_bytes = (size_t)a.bn * KC * 2 * nchunks;
    const size_t a_stage = (size_t)kDenseM * KC * 2;
    const int es_out = a.out_mode == 0 ? (int)sizeof(T) : 4;
    const size_t budget = 220 * 1024;
    const size_t bars = (2 * 8 + 18) * 8 + 16;
    const int row_b = a.bn * es_out;
    a.cb = row_b % 128 == 0 ? 128 : (row_b % 64 == 0 ? 64 : 32);
    a.csplit = (row_b / a.cb) % 2 == 0 ? 2 : 1;
    size_t staged_bytes = 4 * (size_t)32 * row_b;
    a.staged = (b_bytes + 3 * a_stage + staged_bytes + bars <= budget) ? 1 : 0;
    if (!a.staged) staged_bytes = 0;
    const size_t room = budget - std::min(budget, b_bytes + staged_bytes + bars);
    a.stages = (int)std::min<size_t>(8, room / a_stage);
    if (a.stages < 2) return false;
    const size_t smem = b_bytes + a.stages * a_stage + staged_bytes + (2 * a.stages + 18) * 8 + 16;
    // TMEM: up to four accumulators; two CTAs per SM when smem and TMEM allow
    // (a second CTA's epilogue and loads overlap the first's)
    a.accs = a.bn <= 64 ? 4 : 2;
    const int cols = a.accs * a.bn <= 128 ? 128 : (a.accs * a.bn <= 256 ? 256 : 512);
    const int per_sm = (smem <= 112 * 1024 && cols <= 256) ? 2 : 1;
    const CUtensorMap ta = make_tmap(x, dt, a.k_total, a.rows, KC, kDenseM);
    const CUtensorMap tb = make_tmap(b, dt, a.k_total, a.n_total, KC, a.bn);
    const CUtensorMapDataType tt = dt == SK_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    const int cw = a.cb / es_out;
    const CUtensorMap ty =
        a.out_mode == 0 ? make_tmap_rows(a.y, tt, 2, a.n_total, a.rows, a.ld_y, cw, 32)
                        : make_tmap_rows(a.y, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, a.n_total, a.rows,
                                         a.ld_y, cw, 32);
    const CUtensorMap tr =
        a.residual ? make_tmap_rows(a.residual, tt, 2, a.n_total, a.rows, a.ld_y, cw, 32) : ty;
    auto kern = k_dense_tc<T, KC>;
    ensure_smem(reinterpret_cast<const void*>(kern), smem);
    const int grid = std::max(1, std::min(a.items, per_sm * ctx->num_sms));
#ifdef SK_DENSE_TRACE
    static long long* trbuf = nullptr;
    if (!trbuf) SK_CUDA(cudaMalloc(&trbuf, 64 * 8 * 8));
    fill_async(trbuf, 0, 64 * 8 * 8, st);
    a.trace = trbuf;
#endif
    launch_pdl(kern, grid, kDenseThreads, smem, st, ta, tb, ty, tr, a);
#ifdef SK_DENSE_TRACE
    {
        std::vector<long long> h(64 * 8);
        SK_CUDA(cudaMemcpyAsync(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost, st));
        SK_CUDA(cudaStreamSynchronize(st));
        fprintf(stderr, "dense trace bn=%d k=%d items=%d grid=%d\n", a.bn, a.k_total, a.items, grid);
        for (int i = 0; i < 64; ++i) {
            bool any = false;
            for (int j = 0; j < 8; ++j) any |= h[i * 8 + j] != 0;
            if (!any) continue;
            fprintf(stderr, "%2d", i);
            for (int j = 0; j < 8; ++j) fprintf(stderr, " %8lld", h[i * 8 + j] ? h[i * 8 + j] - h[0] : -1);
            fprintf(stderr, "\n");
        }
    }
#endif
    return true;
}

}  // namespace

// b: B operand [n_total][k_total] K-major (forward: W^T; dgrad: W), as the
// gathered-GEMM kernel reads it. y_accum != null: y_accum += result (fp32).
bool dense_identity_tc(sk_ctx* ctx, sk_dtype dt, long long rows, int k_total, int n_total,
                       const void* x, const void* b, void* y, const void* residual,
                       float* y_accum, int cta_n, cudaStream_t st) {
    if (dt != SK_F16 && dt != SK_BF16) return false;
    if (rows <= 0 || k_total % 8 != 0 || n_total % 16 != 0) return false;
    DenseArgs a;
    a.residual = y_accum ? nullptr : residual;
    a.y = y_accum ? (void*)y_accum : y;
    a.rows = rows;
    a.k_total = k_total;
    a.n_total = n_total;
    int cap = cta_n > 0 ? std::min(cta_n, 256) : 256;
    cap = std::max(16, cap / 16 * 16);
    a.n_nt = (int)ceil_div(n_total, cap);
    a.bn = (int)ceil_div(ceil_div(n_total, a.n_nt), 16) * 16;
    a.m_tiles = (int)ceil_div(rows, kDenseM);
    if ((long long)a.m_tiles * a.n_nt > INT32_MAX) return false;
    a.items = a.m_tiles * a.n_nt;
    a.out_mode = y_accum ? 3 : 0;
    a.ld_y = n_total;
    a.staged = 0;
    a.stages = 2;
    a.accs = 2;
    a.cb = 128;
    a.csplit = 1;
    const bool h = dt == SK_F16;
    if (k_total % 64 == 0)
        return h ? launch_dense<__half, 64>(ctx, dt, a, x, b, st)
                 : launch_dense<__nv_bfloat16, 64>(ctx, dt, a, x, b, st);
    if (k_total % 32 == 0)
        return h ? launch_dense<__half, 32>(ctx, dt, a, x, b, st)
                 : launch_dense<__nv_bfloat16, 32>(ctx, dt, a, x, b, st);
    return h ? launch_dense<__half, 16>(ctx, dt, a, x, b, st)
             : launch_dense<__nv_bfloat16, 16>(ctx, dt, a, x, b, st);
}

}  // namespace sk
