// sk200 sparse-convolution dataflows on sm_100a (hot path (2)).
//
// All three reference dataflows (exec.cpp:117-257) reduce to one primitive,
// a GATHERED GEMM over 128-row tiles:
//
//   for each work item (tile of 128 rows, N-tile):
//     acc[128 x BN] = sum over k-steps (offset k, channel chunk c) of
//                     A_rows(k)[128 x KC] * B_k[KC x BN]
//     epilogue: rows -> output rows (store / fp32 red.add / fp32 RMW)
//
//  * implicit GEMM (exec.cpp:206-257): rows = prepared OS rows of one split,
//    A row = x[entries[row][k]] (sentinel -> zero-filled), k-steps = offsets
//    whose bit is set in the tile's OR-mask (sorted masks => empty offsets
//    skipped per tile), output row = out_row[row];
//  * fetch-on-demand (exec.cpp:160-201): rows = the WS pairs of one offset,
//    A row = x[in[p]], output row = out[p] accumulated with fp32 red.add;
//  * gather-GEMM-scatter (exec.cpp:117-158): explicit gather kernel, the same
//    GEMM over the gathered buffer (identity rows), scatter-add kernel.
//  * dgrad (exec.cpp:385-396) = the same over the transposed map with the
//    mirrored offset and B = W[k'] read as [c_in][c_out] (already K-major);
//    forward uses B = W^T (a tiny per-call transpose to [k][c_out][c_in]).
//
// fp16/bf16 -> k_gconv_tc: warp-specialised, persistent tcgen05 kernel over
// 256-row work items (two 128-row MMA halves sharing each B stage). Default
// (cp.async) roles, PW = 16 gather warps at one CTA per SM or 8 at two:
//   warps 0..PW-1  producers: warp w gathers only the REAL rows of its
//                  256/PW rows (compacted lists), 16 B cp.async into
//                  128/64/32 B-swizzled K-major stages, completion via
//                  cp.async.mbarrier.arrive.noinc; warp 0 also loads the B
//                  tile (2D TMA, expect_tx)
//   warp PW        TMEM allocator + tcgen05.mma issuer (M=128 x 2 halves,
//                  N = C_out tile <= 256, K=16; elect.sync inside the asm),
//                  tcgen05.commit frees stages
//   warp PW+1      index warp: takes work items from the dynamic item queue
//                  (ItemSrc), walks their active columns (tile OR-masks),
//                  streams each column step's 256 row indices into an 8-slot
//                  smem ring (cp.async.bulk) and compacts them into the
//                  producers' real-row lists one step behind
//   warps PW+2..3  zero warps: st.shared zeros only for sentinel rows that
//                  still hold data from the stage's previous use
//   warps PW+4..7  epilogue: tcgen05.ld 32x32b -> registers -> fp16 store /
//                  fp32 red.add / RMW (+ fused skip add); double-buffered TMEM
//                  accumulators so item i's epilogue overlaps item i+1's MMAs
// The TilePreset picks the variant (launch_tc_kc): cta_m 256 = one CTA per
// SM, cta_k = channels per stage (C_in = 96: three 32-channel slabs),
// load_width 1 = TMA tile::gather4 producers (4 warps, one gather per 4 rows,
// sentinel rows -> out-of-bounds coordinate -> zero fill).
// Measured limits and rejected designs: profiles/r01_gather_pipeline.md,
// r01_gather_paths.md, r02_gather_redesign.md.
// fp32 -> k_gconv_simt: the 1e-5 parity path (FFMA, fp32 accumulate).
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "sk_internal.hpp"
#include "sk_tc.cuh"

namespace sk {

namespace {

constexpr int kItemM = 2 * kTileM;  // rows per work item: two 128-row MMA halves
// Warp roles of k_gconv_tc for PW producer warps (16: one CTA per SM, 768
// threads; 8: two CTAs per SM, 512 threads, <= 64 registers). Epilogue warps
// start at a multiple of 4 (TMEM lane quadrant = warp % 4).
template <int PW>
struct Roles {
    static constexpr int kProducerWarps = PW;           // warps 0..PW-1: cp.async gathers
    static constexpr int kGroupRows = 256 / PW;        // rows per producer warp (16 / 32)
    static constexpr int kMmaWarp = PW;                 // TMEM owner + tcgen05.mma issuer
    static constexpr int kIndexWarp = PW + 1;           // index/descriptor streamer
    static constexpr int kZeroWarp0 = PW + 2;           // 2 zero warps
    static constexpr int kEpiWarp0 = PW + 4;            // 4 epilogue warps
    static constexpr int kThreads = (PW + 8) * 32;
};
// compacted list entries: (A row << kRowBits) | row in the producer group (<= 64)
constexpr uint32_t kRowBits = 6, kRowMask = 63;
constexpr int kTmaWarps = 4;          // warps 0-3: TMA gather4 producers (TMA variant)
constexpr int kZeroWarps = 2;
constexpr int kMaxStages = 10;       // launch_tc_kc caps the stage count
constexpr int kCompactLag = 1;       // index warp compacts slot s-1 after publishing s (3: -1..2% slower)
constexpr int kIdxRing = 8;           // column steps in flight in the index ring (1 KB each)

struct ConvArgs {
    int mode;  // 0 = OS rows (implicit GEMM), 1 = WS pairs (FOD / GGS GEMM)
    // OS mode (prepared map, entries tile-column-major [tile][col][128])
    const int* entries;
    const int* out_row;
    const unsigned long long* tile_masks;
    const int* split_begin;
    int ns, rows_pad, n_tiles, n_rows_valid;
    // WS mode: per-offset pair lists padded to 256-pair tiles (-1 pads)
    const int* ws_tile_ptr;
    const int* in_pad;
    const int* out_pad;
    int a_identity, out_identity;
    int kd;
    // operands
    const void* a;
    int k_total, n_rows_a;
    const void* b;
    int n_total, mirror;
    void* y;
    int out_mode;  // 0 store T, 1 store f32, 2 red.add f32, 3 RMW f32
    int ld_y;
    int n_ntiles, bn;
    const void* residual;  // optional [n_out][ld_y] T added in the epilogue (out_mode 0)
    int items;        // OS mode item count (WS mode: derived on device)
    int split_only;   // >= 0: only items of this split (deterministic sequencing)
    long long* trace; // SK_CONV_TRACE builds: per-step clock64 timeline of CTA 0
    int exp;          // SK_CONV_TRACE builds: SK_EXP bits 1 no A gathers, 2 no zeroing, 4 no MMA, 8 no B TMA
    int offset_only;  // >= 0: WS mode only tiles of this offset
    int* sched;       // dynamic item queue {next item, CTAs done} (self-resetting), or null
    int single;       // OS mode: one 128-row tile per work item (cta_m 64) instead of two
    // tile preferences from the layer's TilePreset (include/sk200.h):
    int cta_m;        // 256: one CTA per SM; otherwise two per SM when C_out <= 128 fits
    int cta_k;        // channels per pipeline stage: 0 auto, 16 / 32 / 64, 96 = 3 x 32 slabs
    int tma_gather;   // load_width == 1: TMA tile::gather4 producers instead of cp.async
};

// one work item = 256 rows (OS: 128-row tiles 2*t2 and 2*t2+1 of split s;
// WS: one 256-pair tile of offset k) x one N-tile
#ifdef SK_CONV_TRACE
#define SK_TR(slot, cond)                                                              \
    do {                                                                               \
        if (p.trace && blockIdx.x == 0 && (cond) && tr_n < 4096)                       \
            p.trace[(size_t)tr_n * 8 + (slot)] = clock64();                            \
    } while (0)
#else
#define SK_TR(slot, cond) do {} while (0)
#endif
#ifdef SK_CONV_TRACE
#define SK_TZ(k)                                                                       \
    do {                                                                               \
        if (p.trace && blockIdx.x == 0 && lane == 0 && zw == 0 && tr_n < 4096)         \
            p.trace[4096 * 8 + (size_t)tr_n * 4 + (k)] = clock64();                    \
    } while (0)
#else
#define SK_TZ(k) do {} while (0)
#endif

#ifdef SK_CONV_TRACE
__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define SK_CTA_REC(k, v)                                                               \
    do {                                                                               \
        if (p.trace && lane == 0 && blockIdx.x < 1024)                                 \
            p.trace[4096 * 16 + blockIdx.x * 4 + (k)] = (v);                           \
    } while (0)
#else
#define SK_CTA_REC(k, v) do {} while (0)
#endif

struct Item {
    int s, t2, nt, k;
    int w;             // split width (OS) or 1 (WS)
    int col_begin;     // global offset of column 0
    long long row0;    // first row: OS row within the split, WS padded pair index
    int halves;        // OS: 128-row tiles present (1 or 2)
    unsigned long long m0, m1;
    int biw0, bw1;
};

__device__ __forceinline__ int pairs_of(int n_tiles) { return (n_tiles + 1) / 2; }

__device__ __forceinline__ int num_items(const ConvArgs& p) {
    if (p.mode != 1) return p.items;
    if (p.offset_only >= 0)
        return (p.ws_tile_ptr[p.offset_only + 1] - p.ws_tile_ptr[p.offset_only]) * p.n_ntiles;
    return p.ws_tile_ptr[p.kd] * p.n_ntiles;
}

__device__ Item decode(const ConvArgs& p, int item) {
    Item it;
    if (p.mode == 2) {  // dense identity map (K=1, stride 1): a plain GEMM
        it.s = 0;
        it.k = 0;
        it.t2 = item / p.n_ntiles;
        it.nt = item % p.n_ntiles;
        it.w = 1;
        it.col_begin = 0;
        it.row0 = (long long)it.t2 * kItemM;
        it.halves = 2;
        it.m0 = 1;
        it.m1 = 0;
        it.biw0 = 1;
        it.bw1 = 0;
        return it;
    }
    if (p.mode == 0) {
        const int tpi = p.single ? 1 : 2;  // 128-row tiles per item
        const int per = (p.single ? p.n_tiles : pairs_of(p.n_tiles)) * p.n_ntiles;
        it.s = p.split_only >= 0 ? p.split_only : item / per;
        const int rem = p.split_only >= 0 ? item : item % per;
        it.t2 = rem / p.n_ntiles;  // item index within the split
        it.nt = rem % p.n_ntiles;
        it.col_begin = p.split_begin[it.s];
        it.w = p.split_begin[it.s + 1] - it.col_begin;
        it.row0 = (long long)it.t2 * tpi * kTileM;
        it.k = -1;
        it.halves = (!p.single && 2 * it.t2 + 1 < p.n_tiles) ? 2 : 1;
        const unsigned long long* tm = p.tile_masks + ((size_t)it.s * p.n_tiles + tpi * it.t2) * 2;
        it.m0 = tm[0];
        it.m1 = tm[1];
        if (it.halves == 2) {
            it.m0 |= tm[2];
            it.m1 |= tm[3];
        }
        it.biw0 = it.w < 64 ? it.w : 64;
        it.bw1 = it.w - 64;
    } else {
        int tile = item / p.n_ntiles;
        it.nt = item % p.n_ntiles;
        int k = 0;
        if (p.offset_only >= 0) {
            k = p.offset_only;
            tile += p.ws_tile_ptr[k];
        } else {
            while (k + 1 <= p.kd && p.ws_tile_ptr[k + 1] <= tile) ++k;
        }
        it.k = k;
        it.s = 0;
        it.t2 = tile;
        it.w = 1;
        it.col_begin = k;
        it.row0 = (long long)tile * kItemM;
        it.halves = 2;
        it.m0 = 1;  // one active "column"
        it.m1 = 0;
        it.biw0 = 1;
        it.bw1 = 0;
    }
    return it;
}

// Active columns in ascending order (big-endian masks, kmap.cpp:38-45); -1 = done.
__device__ __forceinline__ int next_col(unsigned long long& m0, unsigned long long& m1, int biw0,
                                        int bw1) {
    if (m0) {
        int hb = 63 - __clzll((long long)m0);
        m0 &= ~(1ull << hb);
        return biw0 - 1 - hb;
    }
    if (m1) {
        int hb = 63 - __clzll((long long)m1);
        m1 &= ~(1ull << hb);
        return 64 + bw1 - 1 - hb;
    }
    return -1;
}

// the 128 A-row indices of half h of a column step (contiguous, 512B aligned);
// nullptr when the half does not exist
__device__ __forceinline__ const int* idx_column(const ConvArgs& p, const Item& it, int j, int h) {
    if (p.mode == 0) {
        if (h >= it.halves) return nullptr;
        const long long t = (p.single ? 1 : 2) * (long long)it.t2 + h;
        return p.entries + (size_t)p.rows_pad * it.col_begin + ((size_t)t * it.w + j) * kTileM;
    }
    return p.in_pad + it.row0 + h * kTileM;
}

// row r (0..255) of an item
__device__ __forceinline__ int a_index(const ConvArgs& p, const Item& it, int r, int j) {
    if (p.mode == 2) return it.row0 + r < p.n_rows_valid ? (int)(it.row0 + r) : -1;
    if (p.mode == 1 && p.a_identity) return (int)(it.row0 + r);
    const int* col = idx_column(p, it, j, r / kTileM);
    return col ? __ldg(col + (r % kTileM)) : -1;
}

__device__ __forceinline__ long long out_index(const ConvArgs& p, const Item& it, int r) {
    if (p.mode == 2) return it.row0 + r < p.n_rows_valid ? it.row0 + r : -1;
    if (p.mode == 0) {
        if (r / kTileM >= it.halves) return -1;
        return __ldg(p.out_row + (size_t)it.s * p.rows_pad + it.row0 + r);
    }
    const long long pi = it.row0 + r;
    return p.out_identity ? pi : (long long)__ldg(p.out_pad + pi);
}

// position of the k-th (0-based) set bit of r
__device__ __forceinline__ int kth_bit64(uint64_t r, int k) {
    const uint32_t lo = (uint32_t)r, hi = (uint32_t)(r >> 32);
    const int c = __popc(lo);
    return k < c ? (int)__fns(lo, 0, k + 1) : 32 + (int)__fns(hi, 0, k - c + 1);
}

// i-th work item of this CTA. Items come out of the mask sort in roughly
// descending cost, so rounds alternate direction (boustrophedon) to even out
// the per-CTA sums of a static persistent schedule; -1 = no more items.
__device__ __forceinline__ int item_of(int i, int n_items) {
    const int g = gridDim.x;
    const long long it = (long long)i * g + ((i & 1) ? g - 1 - (int)blockIdx.x : (int)blockIdx.x);
    return it < n_items ? (int)it : -1;
}

// Work-item source of one warp (all lanes call next() together).
// Static (p.sched == null): the boustrophedon schedule of item_of. Dynamic:
// the CTA's scheduler warp takes the next item with one global atomic
// (descending-cost order -> greedy LPT balance across CTAs; a static
// schedule left the slowest CTA ~1.4x the mean, tools/trace2.py) and
// publishes it through a kItemRing smem ring that every other item-walking
// warp of the CTA reads in order.
constexpr int kItemRing = 4;  // smem-bound: two CTAs per SM must still fit
struct ItemSrc {
    int kind;  // 0 static, 1 publisher, 2 consumer
    int local, n_items, slot;
    uint32_t ph;
    int* ids;
    uint64_t* full;
    uint64_t* empty;
    int* sched;
    __device__ void init(const ConvArgs& p, int dyn_kind, int n, int* ids_, uint64_t* full_,
                         uint64_t* empty_) {
        kind = p.sched ? dyn_kind : 0;
        local = 0;
        n_items = n;
        slot = 0;
        ph = 0;
        ids = ids_;
        full = full_;
        empty = empty_;
        sched = p.sched;
    }
    __device__ int next() {
        const int lane = threadIdx.x & 31;
        int v;
        if (kind == 0) {
            v = item_of(local, n_items);
        } else if (kind == 1) {
            mbar_wait(&empty[slot], ph ^ 1);
            if (lane == 0) {
                // first item static (no atomic round trip before the CTA's
                // first gather), the rest from the queue
                v = local == 0 ? (int)blockIdx.x : (int)gridDim.x + atomicAdd(sched, 1);
                if (v >= n_items) v = -1;
                ids[slot] = v;
                mbar_arrive(&full[slot]);
            }
            v = __shfl_sync(0xffffffffu, v, 0);
        } else {
            mbar_wait(&full[slot], ph);
            v = ids[slot];
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
        }
        if (kind != 0 && ++slot == kItemRing) {
            slot = 0;
            ph ^= 1;
        }
        ++local;
        return v;
    }
};
// end of a dynamically scheduled launch: the last CTA out re-zeroes the
// queue so the context can hand the slot to a later launch
__device__ __forceinline__ void sched_finish(const ConvArgs& p) {
    if (p.sched && threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(p.sched + 1, 1) == (int)gridDim.x - 1) {
            p.sched[0] = 0;
            p.sched[1] = 0;
            __threadfence();
        }
    }
}

// iterator over the column steps (item, active column) of this CTA
struct Cursor {
    int local, n_items, j;
    Item it;
    unsigned long long m0, m1;
    bool done;
    ItemSrc* src;
    __device__ void load(const ConvArgs& p) {
        for (int item; (item = src->next()) >= 0; ++local) {
            it = decode(p, item);
            m0 = it.m0;
            m1 = it.m1;
            j = next_col(m0, m1, it.biw0, it.bw1);
            if (j >= 0) {
                done = false;
                return;
            }
        }
        done = true;
    }
    __device__ void init(const ConvArgs& p, int n, ItemSrc* s) {
        n_items = n;
        local = 0;
        src = s;
        load(p);
    }
    __device__ void advance(const ConvArgs& p) {
        j = next_col(m0, m1, it.biw0, it.bw1);
        if (j < 0) {
            ++local;
            load(p);
        }
    }
};


// epilogue store of 16 fp32 accumulators (row orow, columns col..col+15)
template <typename T>
__device__ __forceinline__ void store16(const ConvArgs& p, long long orow, int col, uint32_t (&v)[16]) {
    if (p.out_mode == 0) {
        T* dst = static_cast<T*>(p.y) + (size_t)orow * p.ld_y + col;
        if (p.residual) {  // fused skip connection: y = conv + residual
            const uint4* rs = reinterpret_cast<const uint4*>(
                static_cast<const T*>(p.residual) + (size_t)orow * p.ld_y + col);
            const uint4 r0 = rs[0], r1 = rs[1];
            const uint32_t rr[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                float2 f = unpack2(rr[i], (T*)nullptr);
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
        reinterpret_cast<uint4*>(dst)[0] = u0;
        reinterpret_cast<uint4*>(dst)[1] = u1;
    } else {
        float* dst = static_cast<float*>(p.y) + (size_t)orow * p.ld_y + col;
        if (p.out_mode == 2) {
#pragma unroll
            for (int i = 0; i < 16; i += 4)
                red_add_v4(dst + i, __uint_as_float(v[i]), __uint_as_float(v[i + 1]),
                           __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
        } else {
#pragma unroll
            for (int i = 0; i < 16; i += 4) {
                float4 o = make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]),
                                       __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
                if (p.out_mode == 3) {
                    float4 prev = *reinterpret_cast<float4*>(dst + i);
                    o.x += prev.x; o.y += prev.y; o.z += prev.z; o.w += prev.w;
                }
                *reinterpret_cast<float4*>(dst + i) = o;
            }
        }
    }
}


// Per ring slot, built by the index warp from the slot's 256 row indices:
// for each producer warp's 16-row group the list of its real rows
// ((idx << kRowBits) | row-in-group) and their count, and the real-row bitmask of
// every 32-row group (zero warps). Moves the ballot/compaction smem traffic
// off the producers' per-step critical path (their LDS would queue behind
// the SM's LDGSTS backlog in the MIO pipe).
template <int PW>
struct CSlot {
    uint32_t list[PW][256 / PW];
    int cnt[PW];
    uint32_t zmask[kItemM / 32];
};
// index warp: lane l covers rows 8l..8l+7 of the slot; a producer group of
// 256/PW rows spans LPG = 32/PW lanes (prefix over the group's lanes)
template <int PW>
__device__ __forceinline__ void compact_slot(const int* ring, CSlot<PW>& cs, int lane) {
    constexpr int LPG = 32 / PW;
    const int4 a = reinterpret_cast<const int4*>(ring)[2 * lane];
    const int4 b = reinterpret_cast<const int4*>(ring)[2 * lane + 1];
    const int v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint32_t bits = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) bits |= (v[i] >= 0 ? 1u : 0u) << i;
    const int c = __popc(bits);
    int incl = c;  // inclusive scan over the group's lanes
#pragma unroll
    for (int o = 1; o < LPG; o <<= 1) {
        const int up = __shfl_up_sync(0xffffffffu, incl, o);
        if ((lane % LPG) >= o) incl += up;
    }
    int k = incl - c;
    uint32_t* L = cs.list[lane / LPG];
#pragma unroll
    for (int i = 0; i < 8; ++i)
        if (bits >> i & 1u) L[k++] = ((uint32_t)v[i] << kRowBits) | (uint32_t)((lane % LPG) * 8 + i);
    if (lane % LPG == LPG - 1) cs.cnt[lane / LPG] = incl;
    uint32_t m = bits << ((lane & 3) * 8);
    m |= __shfl_xor_sync(0xffffffffu, m, 1);
    m |= __shfl_xor_sync(0xffffffffu, m, 2);
    if ((lane & 3) == 0) cs.zmask[lane >> 2] = m;
}

// per index-ring slot: {brow (first B row of this step, -1 = end of work), unused x3}
struct alignas(16) StepDesc {
    int brow, pad0, pad1, pad2;
};

// USE_TMA = true: producer warps 0-3 issue TMA tile::gather4 (4 rows each,
// sentinel rows -> out-of-bounds coordinate -> zero fill without L2 traffic)
// from uniform warp code (shuffled operands, elect.sync inside the asm), and
// warp 0 loads B with one 2D TMA tile. USE_TMA = false: warps 0-7 gather with
// 16 B cp.async (reference path, kept for A/B measurement).
template <typename T, int KC, bool USE_TMA, int SLABS, int PW>
__global__ void __launch_bounds__(Roles<PW>::kThreads, PW == 16 ? 1 : (PW == 8 ? 2 : 3))
    k_gconv_tc(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
               const ConvArgs p, int stages, int acc_bufs) {
    constexpr int kProducerWarps = Roles<PW>::kProducerWarps;
    constexpr int kGroupRows = Roles<PW>::kGroupRows;
    constexpr int kMmaWarp = Roles<PW>::kMmaWarp;
    constexpr int kIndexWarp = Roles<PW>::kIndexWarp;
    constexpr int kZeroWarp0 = Roles<PW>::kZeroWarp0;
    constexpr int kEpiWarp0 = Roles<PW>::kEpiWarp0;
    // dynamic smem starts 1024B-aligned (no static smem); checked below since
    // the swizzle atoms and UMMA descriptors rely on it
    extern __shared__ __align__(1024) uint8_t smem[];
    const int BN = p.bn;
    const uint32_t a_half = kTileM * KC * 2;   // one 128-row half
    const uint32_t a_bytes = 2 * a_half;       // 256-row A tile
    const uint32_t b_bytes = (uint32_t)BN * KC * 2;
    // a stage holds NSL K-slabs of KC channels (cp.async path: the chunks of
    // one column step together, fewer and fatter pipeline steps): A slabs
    // first, then the B slabs
    constexpr int NSL = USE_TMA ? 1 : SLABS;
    const uint32_t a_all = (uint32_t)NSL * a_bytes;
    const uint32_t stage_bytes = (uint32_t)NSL * (a_bytes + b_bytes);
    uint8_t* stage_base = smem;
    int* idx_ring = reinterpret_cast<int*>(smem + (size_t)stages * stage_bytes);  // [R][256]
    StepDesc* descs = reinterpret_cast<StepDesc*>(idx_ring + kIdxRing * kItemM);   // [R]
    uint64_t* bars = reinterpret_cast<uint64_t*>(descs + kIdxRing);
    uint64_t* full = bars;
    uint64_t* empty = bars + stages;
    uint64_t* tfull = bars + 2 * stages;
    uint64_t* tempty = tfull + 2;
    uint64_t* ifull = tempty + 2;         // [R] ring slot landed (bulk copy / fill)
    uint64_t* iempty = ifull + kIdxRing;  // [R] all gathering warps done with the slot
    uint64_t* cfull = iempty + kIdxRing;  // [R] compacted row lists of the slot ready
    uint64_t* itfull = cfull + kIdxRing;  // [kItemRing] dynamic item queue
    uint64_t* itempty = itfull + kItemRing;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(itempty + kItemRing);
    int* item_ids = reinterpret_cast<int*>(tmem_slot + 4);
    CSlot<PW>* cslots = reinterpret_cast<CSlot<PW>*>(item_ids + kItemRing);  // [R] compacted row lists

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    uint32_t ncols = 32;
    while (ncols < (uint32_t)(acc_bufs * 2 * BN)) ncols <<= 1;

    if (threadIdx.x == 0) {
        if (smem_u32(smem) & 1023) __trap();
        for (int i = 0; i < stages; ++i) {
            // cp.async: one noinc arrival per producer thread; TMA: one
            // expect_tx arrival per gathering warp
#ifdef SK_CONV_TRACE
            const int zw_n = (p.exp & 32) ? 0 : kZeroWarps;
#else
            const int zw_n = kZeroWarps;
#endif
            mbar_init(&full[i], USE_TMA ? kTmaWarps : kProducerWarps * 32 + zw_n + 1);  // + B TMA
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 128);
        }
        for (int i = 0; i < kIdxRing; ++i) {
            mbar_init(&ifull[i], 1);
            mbar_init(&cfull[i], 1);
#ifdef SK_CONV_TRACE
            const int zw_n = (p.exp & 32) ? 0 : kZeroWarps;
#else
            const int zw_n = kZeroWarps;
#endif
            mbar_init(&iempty[i], USE_TMA ? kTmaWarps : kProducerWarps + zw_n);
        }
        for (int i = 0; i < kItemRing; ++i) {
            mbar_init(&itfull[i], 1);
            mbar_init(&itempty[i], 5);  // MMA warp + 4 epilogue warps
        }
        fence_mbar_init();
        if (USE_TMA)
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_a)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_b)) : "memory");
    }
    if (warp == kMmaWarp) tmem_alloc(tmem_slot, ncols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // the prologue (barriers, tensor-map prefetch, TMEM) overlapped the
    // predecessor's tail; global memory only after it has completed
    pdl_wait();
    const int n_items = num_items(p);
    const int nchunks = (p.k_total + KC - 1) / KC;
    const T* __restrict__ A = static_cast<const T*>(p.a);
    const T* __restrict__ Bw = static_cast<const T*>(p.b);

    if (warp == kIndexWarp && p.mode == 0 && !USE_TMA) {
        // ===== index warp, implicit GEMM: per item, the lanes work out the
        // item's active columns in parallel (lane k: k-th set bit of the
        // tile OR-mask, ascending) with their index-column pointers and B
        // rows; the serial part per step is then one ring publish (wait slot,
        // descriptor, expect_tx, one or two 512 B cp.async.bulk). A single
        // warp's dependent address math per step was the pipeline's pace. =====
        int slot = 0;
        uint32_t ph = 0;
        int pub = 0, cmp = 0;  // steps published / compacted (compaction lags kCompactLag)
        auto compact_one = [&]() {
            const int sl = cmp % kIdxRing;
            mbar_wait(&ifull[sl], (uint32_t)(cmp / kIdxRing) & 1u);
            compact_slot(idx_ring + sl * kItemM, cslots[sl], lane);
            __syncwarp();
            if (lane == 0) mbar_arrive(&cfull[sl]);
            ++cmp;
        };
#ifdef SK_CONV_TRACE
        int tr_n = 0;
#endif
        ItemSrc src;
        src.init(p, 1, n_items, item_ids, itfull, itempty);
        // The item queue may block this warp until the MMA / epilogue warps
        // consume earlier items, and they wait on steps this warp has
        // published but not yet compacted: flush before every take.
        auto take = [&]() {
            while (cmp < pub) compact_one();
            return src.next();
        };
        for (int item; (item = take()) >= 0;) {
            const Item it = decode(p, item);
            const uint64_t r0 = it.biw0 > 0 ? (__brevll(it.m0) >> (64 - it.biw0)) : 0ull;
            const uint64_t r1 = it.bw1 > 0 ? (__brevll(it.m1) >> (64 - it.bw1)) : 0ull;
            const int n0 = __popcll(r0), n = n0 + __popcll(r1);
            const int* tile0 = p.entries + (size_t)p.rows_pad * it.col_begin +
                               (size_t)((p.single ? 1 : 2) * it.t2) * it.w * kTileM;
            const int half1 = it.halves == 2 ? it.w * kTileM : -1;  // offset of half 1's column
            for (int base = 0; base < n; base += 32) {
                const int k = base + lane;
                int j = 0;
                if (k < n) j = k < n0 ? kth_bit64(r0, k) : 64 + kth_bit64(r1, k - n0);
                const int kg = it.col_begin + j;
                const int brow_l = (p.mirror ? p.kd - 1 - kg : kg) * p.n_total + it.nt * BN;
                const int cnt = min(32, n - base);
                for (int u = 0; u < cnt; ++u) {
                    const int ju = __shfl_sync(0xffffffffu, j, u);
                    const int brow = __shfl_sync(0xffffffffu, brow_l, u);
                    const int* c0 = tile0 + (size_t)ju * kTileM;
                    mbar_wait_sleep(&iempty[slot], ph ^ 1);
                    int* ring = idx_ring + slot * kItemM;
                    if (half1 < 0) {
                        for (int v = kTileM + lane; v < kItemM; v += 32) ring[v] = -1;  // missing half
                        __syncwarp();
                    }
                    if (lane == 0) {
                        descs[slot].brow = brow;
                        descs[slot].pad0 = half1 >= 0 ? 2 : 1;  // MMA halves of the step
                        mbar_expect_tx(&ifull[slot], (half1 >= 0 ? 2 : 1) * kTileM * 4);
                    }
                    __syncwarp();
                    bulk_g2s_elect(smem_u32(ring), c0, kTileM * 4, &ifull[slot]);
                    if (half1 >= 0)
                        bulk_g2s_elect(smem_u32(ring + kTileM), c0 + half1, kTileM * 4, &ifull[slot]);
                    SK_TR(7, lane == 0);
#ifdef SK_CONV_TRACE
                    ++tr_n;
#endif
                    if (++pub - cmp > kCompactLag) compact_one();
                    if (++slot == kIdxRing) {
                        slot = 0;
                        ph ^= 1;
                    }
                }
            }
        }
        while (cmp < pub) compact_one();
        mbar_wait_sleep(&iempty[slot], ph ^ 1);
        if (lane == 0) {
            descs[slot].brow = -1;
            mbar_arrive(&ifull[slot]);
            mbar_arrive(&cfull[slot]);
        }
    } else if (warp == kIndexWarp) {
        // ===== index warp (FOD/GGS pair tiles, dense, TMA variant): walks the column steps and streams each step's 256
        // A-row indices (cp.async.bulk, 512B per half) + its B row base =====
        Cursor cur;
#ifdef SK_CONV_TRACE
        int tr_n = 0;
#endif
        ItemSrc src;
        src.init(p, 1, n_items, item_ids, itfull, itempty);
        cur.init(p, n_items, &src);
        const bool ident = (p.mode == 1 && p.a_identity) || p.mode == 2;
        int slot = 0;
        uint32_t ph = 0;
        int pub = 0, cmp = 0;
        auto compact_one = [&]() {
            const int sl = cmp % kIdxRing;
            mbar_wait(&ifull[sl], (uint32_t)(cmp / kIdxRing) & 1u);
            compact_slot(idx_ring + sl * kItemM, cslots[sl], lane);
            __syncwarp();
            if (lane == 0) mbar_arrive(&cfull[sl]);
            ++cmp;
        };
        for (;;) {
#ifdef SK_CONV_TRACE
            if (p.trace && blockIdx.x == 0 && lane == 0 && tr_n < 4096)
                p.trace[4096 * 12 + (size_t)tr_n * 2] = clock64();
#endif
            mbar_wait_sleep(&iempty[slot], ph ^ 1);
#ifdef SK_CONV_TRACE
            if (p.trace && blockIdx.x == 0 && lane == 0 && tr_n < 4096)
                p.trace[4096 * 12 + (size_t)tr_n * 2 + 1] = clock64();
#endif
            int* ring = idx_ring + slot * kItemM;
            if (cur.done) {
                if (!USE_TMA)
                    while (cmp < pub) compact_one();
                if (lane == 0) {
                    descs[slot].brow = -1;
                    mbar_arrive(&ifull[slot]);
                    mbar_arrive(&cfull[slot]);
                }
                break;
            }
            const int kg = cur.it.col_begin + cur.j;
            const int kb = p.mirror ? p.kd - 1 - kg : kg;
            const int* c0 = ident ? nullptr : idx_column(p, cur.it, cur.j, 0);
            const int* c1 = ident ? nullptr : idx_column(p, cur.it, cur.j, 1);
            if (ident) {
                for (int u = lane; u < kItemM; u += 32) {
                    const long long rr = cur.it.row0 + u;
                    ring[u] = (p.mode == 2 && rr >= p.n_rows_valid) ? -1 : (int)rr;
                }
            } else if (!c1) {
                for (int u = kTileM + lane; u < kItemM; u += 32) ring[u] = -1;  // missing half
            }
            __syncwarp();
#ifdef SK_CONV_TRACE
            if (p.trace && blockIdx.x == 0 && lane == 0 && tr_n < 4096)
                p.trace[4096 * 14 + (size_t)tr_n * 2] = clock64();
#endif
            if (lane == 0) {
                descs[slot].brow = kb * p.n_total + cur.it.nt * BN;
                descs[slot].pad0 = (ident || c1) ? 2 : 1;  // MMA halves of the step
                if (ident) mbar_arrive(&ifull[slot]);
                else mbar_expect_tx(&ifull[slot], (c1 ? 2 : 1) * kTileM * 4);
            }
            __syncwarp();
#ifdef SK_CONV_TRACE
            if (p.trace && blockIdx.x == 0 && lane == 0 && tr_n < 4096)
                p.trace[4096 * 14 + (size_t)tr_n * 2 + 1] = clock64();
#endif
            if (!ident) {  // uniform issue, elected lane (no per-lane R2UR loops)
                bulk_g2s_elect(smem_u32(ring), c0, kTileM * 4, &ifull[slot]);
                if (c1) bulk_g2s_elect(smem_u32(ring + kTileM), c1, kTileM * 4, &ifull[slot]);
            }
            SK_TR(7, lane == 0);
#ifdef SK_CONV_TRACE
            ++tr_n;
#endif
            ++pub;
            // last column of the item: the advance takes the next item from
            // the queue (may block on the MMA / epilogue warps), so flush the
            // compactions they depend on first
            if (!USE_TMA && (cur.m0 | cur.m1) == 0)
                while (cmp < pub) compact_one();
            cur.advance(p);
            if (!USE_TMA && pub - cmp > kCompactLag) compact_one();
            if (++slot == kIdxRing) {
                slot = 0;
                ph ^= 1;
            }
        }
    } else if (USE_TMA && warp < kTmaWarps) {
        // ===== TMA producers: warp w owns rows [64w, 64w+64) = 16 gather4 per
        // step; lanes 0-15 hold the 4-row index groups, shuffled to the whole
        // warp so the TMA operands are warp-uniform =====
        constexpr int GPW = kItemM / 4 / kTmaWarps;  // gathers per warp per step (16)
        int slot = 0, stage = 0;
        uint32_t ph = 0, phase = 0;
        const uint32_t base_u = smem_u32(stage_base);
        const bool dense = p.mode == 2;  // A rows contiguous: two 128-row 2D tiles
        const uint32_t my_bytes = dense ? (warp == 0 ? a_bytes + b_bytes : 0)
                                        : GPW * 4 * KC * 2 + (warp == 0 ? b_bytes : 0);
        for (;;) {
            mbar_wait(&ifull[slot], ph);
            const int brow = descs[slot].brow;
            if (brow < 0) break;
            int4 g4 = make_int4(-1, -1, -1, -1);
            if (dense) g4.x = __shfl_sync(0xffffffffu, idx_ring[slot * kItemM], 0);
            else if (lane < GPW) g4 = reinterpret_cast<const int4*>(idx_ring + slot * kItemM)[warp * GPW + lane];
            g4.x = g4.x < 0 ? p.n_rows_a : g4.x;  // sentinel -> out of bounds -> zeros
            // (dense: g4.x is the item's first row, always valid)
            g4.y = g4.y < 0 ? p.n_rows_a : g4.y;
            g4.z = g4.z < 0 ? p.n_rows_a : g4.z;
            g4.w = g4.w < 0 ? p.n_rows_a : g4.w;
            __syncwarp();
            if (lane == 0) mbar_arrive(&iempty[slot]);
            for (int c = 0; c < nchunks; ++c) {
                mbar_wait(&empty[stage], phase ^ 1);
                const uint32_t sa = base_u + (uint32_t)stage * stage_bytes;
                if (lane == 0) mbar_expect_tx(&full[stage], my_bytes);
                __syncwarp();
                if (warp == 0) tma_tile2d_elect(sa + a_bytes, &tm_b, c * KC, brow, &full[stage]);
                if (dense) {
                    if (warp == 0) {
                        const int r0 = g4.x;  // first row of the item (identity ring)
                        tma_tile2d_elect(sa, &tm_a, c * KC, r0, &full[stage]);
                        tma_tile2d_elect(sa + a_half, &tm_a, c * KC, r0 + kTileM, &full[stage]);
                    }
                } else
#pragma unroll
                for (int g = 0; g < GPW; ++g) {
                    const int r = (warp * GPW + g) * 4;  // first of the 4 rows
                    const uint32_t dst = sa + (uint32_t)(r / kTileM) * a_half +
                                         (uint32_t)(r % kTileM) * KC * 2;
                    tma_gather4_elect(dst, &tm_a, c * KC, __shfl_sync(0xffffffffu, g4.x, g),
                                      __shfl_sync(0xffffffffu, g4.y, g),
                                      __shfl_sync(0xffffffffu, g4.z, g),
                                      __shfl_sync(0xffffffffu, g4.w, g), &full[stage]);
                }
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (++slot == kIdxRing) {
                slot = 0;
                ph ^= 1;
            }
        }
    } else if (!USE_TMA && warp < kProducerWarps) {
        // ===== producers: warp w owns rows [16w, 16w+16) of every step and
        // gathers only its REAL rows, compacted (ballot + prefix, a 16-entry
        // per-warp list) so every cp.async instruction is fully populated:
        // CH = KC/8 lanes per row, 32/CH rows per instruction. LDGSTS drain
        // cost follows the instruction count, not the active lanes, so
        // predicated-off sentinel lanes would waste it. Stale sentinel rows are
        // the zero warps' job; warp 0 also loads the B tile with one 2D TMA
        // (elected lane, expect_tx). Completion is signalled asynchronously
        // (cp.async.mbarrier.arrive.noinc). =====
        constexpr int CH = KC / 8;        // 16B chunks per row
        constexpr int RPI = 32 / CH;      // rows per cp.async instruction
        constexpr int IT = (kGroupRows + RPI - 1) / RPI;
        constexpr uint32_t RB = KC * 2;   // bytes per stage row
        constexpr uint32_t SWB = RB == 128 ? 7 : (RB == 64 ? 3 : 1);
        const int q = lane % CH, sub = lane / CH;
        const size_t row_bytes = (size_t)p.k_total * sizeof(T);
        const char* __restrict__ Ab = reinterpret_cast<const char*>(A) + q * 16;
        const uint32_t half_off = (uint32_t)(warp * kGroupRows / kTileM) * a_half;
        const uint32_t row0 = (uint32_t)(warp * kGroupRows % kTileM);
#ifdef SK_CONV_TRACE
        const int t = threadIdx.x;
        int tr_n = 0;
#endif
        int slot = 0, stage = 0;
        uint32_t ph = 0, phase = 0;
        const uint32_t base_u = smem_u32(stage_base);
        for (;;) {
#ifdef SK_CONV_TRACE
            if (p.trace && blockIdx.x == 0 && t == 0 && tr_n < 4096)
                p.trace[4096 * 12 + (size_t)tr_n * 2] = clock64();
#endif
            mbar_wait_sleep(&cfull[slot], ph);
#ifdef SK_CONV_TRACE
            if (p.trace && blockIdx.x == 0 && t == 0 && tr_n < 4096)
                p.trace[4096 * 12 + (size_t)tr_n * 2 + 1] = clock64();
#endif
            // descriptor, count and list entries are independent loads issued
            // together: one MIO round trip (the slot is released at the end of
            // the step, so no barrier has to wait for these loads here)
            const int brow = descs[slot].brow;
            const int n = cslots[slot].cnt[warp];
            uint32_t e[IT];
#pragma unroll
            for (int i = 0; i < IT; ++i) e[i] = cslots[slot].list[warp][(sub + i * RPI) % kGroupRows];
            if (brow < 0) break;
#ifdef SK_CONV_TRACE
            const int n_do = (p.exp & 1) ? 0 : n;
#else
            const int n_do = n;
#endif
            for (int c0 = 0; c0 < nchunks; c0 += NSL) {
                SK_TR(0, t == 0);
                mbar_wait_sleep(&empty[stage], phase ^ 1);
                SK_TR(1, t == 0);
                const uint32_t sa = base_u + (uint32_t)stage * stage_bytes;
                if (warp == 0) {
#ifdef SK_CONV_TRACE
                    if (p.exp & 8) { if (lane == 0) mbar_arrive(&full[stage]); } else
#endif
                    {
                    if (lane == 0) mbar_expect_tx(&full[stage], NSL * b_bytes);
                    __syncwarp();
                    for (int sl = 0; sl < NSL; ++sl)
                        tma_tile2d_elect(sa + a_all + sl * b_bytes, &tm_b, (c0 + sl) * KC, brow,
                                         &full[stage]);
                    }
                }
                for (int sl = 0; sl < NSL; ++sl) {
                    const uint32_t sa_w = sa + sl * a_bytes + half_off;
                    const int col = (c0 + sl) * KC + q * 8;
                    const uint32_t nbytes = col < p.k_total ? 16u : 0u;  // channel tail -> zeros
                    const char* src_c = Ab + (size_t)(c0 + sl) * KC * sizeof(T);
#pragma unroll
                    for (int i = 0; i < IT; ++i) {
                        if (sub + i * RPI >= n_do) break;
                        const uint32_t r = row0 + (e[i] & kRowMask);       // row within the half
                        const uint32_t off = r * RB + (uint32_t)q * 16;
                        cp_async16(sa_w + (off ^ (((off >> 7) & SWB) << 4)),
                                   src_c + (size_t)(e[i] >> kRowBits) * row_bytes, nbytes);
                    }
                }
                cp_async_arrive_noinc(&full[stage]);
                SK_TR(2, t == 0);
#ifdef SK_CONV_TRACE
                ++tr_n;
#endif
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&iempty[slot]);
            if (++slot == kIdxRing) {
                slot = 0;
                ph ^= 1;
            }
        }
    } else if (!USE_TMA && warp >= kZeroWarp0 && warp < kZeroWarp0 + kZeroWarps
#ifdef SK_CONV_TRACE
               && !(p.exp & 32)
#endif
               ) {
        // ===== zero warps: st.shared zeros into sentinel rows, but only rows
        // that still hold real data from the previous use of the stage (a
        // per-stage dirty mask per 32-row group): about half of the sentinel
        // rows are already zero. Lane l owns row l of each of its groups
        // (KC/8 16-byte stores, swizzled so 8 consecutive rows hit distinct
        // banks). Then fence.proxy.async so the tensor core (async proxy) sees
        // the zeros; these warps issue no cp.async, so the fence never waits
        // on in-flight gathers. =====
        constexpr int CH = KC / 8;
        constexpr uint32_t RB = KC * 2;
        constexpr uint32_t SWB = RB == 128 ? 7 : (RB == 64 ? 3 : 1);
        constexpr int GROUPS = kItemM / 32 / kZeroWarps;  // 32-row groups per zero warp
        const int zw = warp - kZeroWarp0;
        uint32_t dreg[kMaxStages];  // stage contents unknown at start: all dirty
#pragma unroll
        for (int k = 0; k < kMaxStages; ++k) dreg[k] = ~0u;
#ifdef SK_CONV_TRACE
        int tr_n = 0;
#endif
        int slot = 0, stage = 0;
        uint32_t ph = 0, phase = 0;
        const uint32_t base_u = smem_u32(stage_base);
        for (;;) {
            SK_TZ(0);
            mbar_wait_sleep(&cfull[slot], ph);
            SK_TZ(1);
            const int brow = descs[slot].brow;
            // a one-half step never feeds the MMA's second half: zero warp 1
            // (rows 128-255) leaves those stale rows (and their dirty marks) alone
            const bool idle = zw * GROUPS * 32 >= kTileM && descs[slot].pad0 < 2;
            uint32_t real[GROUPS];
#pragma unroll
            for (int g = 0; g < GROUPS; ++g) real[g] = cslots[slot].zmask[zw * GROUPS + g];
            if (brow < 0) break;
            for (int c0 = 0; c0 < nchunks; c0 += NSL) {
                SK_TZ(2);
                mbar_wait_sleep(&empty[stage], phase ^ 1);
                SK_TZ(3);
                const uint32_t sa = base_u + (uint32_t)stage * stage_bytes;
                // lane g < GROUPS keeps group g's per-stage dirty masks in registers
                uint32_t mine = 0, my_real = 0;
#pragma unroll
                for (int g = 0; g < GROUPS; ++g)
                    if (lane == g) my_real = real[g];
#pragma unroll
                for (int k = 0; k < kMaxStages; ++k)
                    if (k == stage && !idle) {
                        mine = ~my_real & dreg[k];
                        dreg[k] = my_real;
                    }
                uint32_t need[GROUPS];
#pragma unroll
                for (int g = 0; g < GROUPS; ++g) need[g] = __shfl_sync(0xffffffffu, mine, g);
#pragma unroll
                for (int g = 0; g < GROUPS; ++g) {
                    if (!(need[g] >> lane & 1u)) continue;
#ifdef SK_CONV_TRACE
                    if (p.exp & 2) continue;
#endif
                    const int grp = zw * GROUPS + g;
                    const uint32_t r = (uint32_t)(grp * 32 % kTileM + lane);
                    const uint32_t rb = sa + (uint32_t)(grp * 32 / kTileM) * a_half + r * RB;
                    const uint32_t x = ((r * RB >> 7) & SWB) << 4;  // Swizzle<B,4,3> of this row
                    for (int sl = 0; sl < NSL; ++sl)
#pragma unroll
                        for (int qq = 0; qq < CH; ++qq)
                            asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(
                                             rb + sl * a_bytes + (((uint32_t)qq * 16) ^ x)),
                                         "r"(0)
                                         : "memory");
                }
#ifdef SK_CONV_TRACE
                if (!(p.exp & 16))
#endif
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[stage]);
                SK_TR(6, lane == 0 && zw == 0);
#ifdef SK_CONV_TRACE
                ++tr_n;
#endif
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&iempty[slot]);
            if (++slot == kIdxRing) {
                slot = 0;
                ph ^= 1;
            }
        }
    } else if (warp == kMmaWarp) {
        // ===== MMA issuer: the whole warp runs the loop with uniform values
        // and elect.sync picks the issuing lane inside the asm, so descriptors
        // stay in uniform registers (no per-MMA R2UR/elect loops) =====
        const uint32_t idesc = (1u << 4) | (Fmt<T>::v << 7) | (Fmt<T>::v << 10) |
                               ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(kTileM >> 4) << 24);
        int stage = 0;
        uint32_t phase = 0;
        const uint64_t desc0 = kmajor_desc<KC>(smem_u32(stage_base));
#ifdef SK_CONV_TRACE
        int tr_n = 0;
        SK_CTA_REC(0, gtimer());
        {
            uint32_t smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            SK_CTA_REC(3, (long long)smid);
        }
#endif
        int local = 0;
        ItemSrc src;
        src.init(p, 2, n_items, item_ids, itfull, itempty);
        for (int item; (item = src.next()) >= 0; ++local) {
            Item it = decode(p, item);
            const int acc = acc_bufs == 2 ? (local & 1) : 0;
            const uint32_t aph = acc_bufs == 2 ? (uint32_t)((local >> 1) & 1) : (uint32_t)(local & 1);
            mbar_wait(&tempty[acc], aph ^ 1);
            tc_fence_after();
            const uint32_t d0 = tmem + (uint32_t)(acc * 2 * BN);  // half 0; half 1 at +BN
            // the MMA needs only the step count: A and B come from the stage
            const int nsteps = (__popcll(it.m0) + __popcll(it.m1)) * (nchunks / NSL);
            const uint32_t two = it.halves == 2 ? 1u : 0u;  // one-tile items: no second-half MMAs
            uint32_t accumulate = 0;
            for (int st = 0; st < nsteps; ++st) {
                SK_TR(3, lane == 0);
                mbar_wait(&full[stage], phase);
                SK_TR(4, lane == 0);
                tc_fence_after();
                // descriptor start addresses advance in 16B units
                const uint64_t da = desc0 + ((uint64_t)stage * stage_bytes >> 4);
#ifdef SK_CONV_TRACE
                if (p.exp & 4) tc_commit_elect(&empty[stage]); else
#endif
                {
                    for (int sl = 0; sl + 1 < NSL; ++sl) {
                        const uint64_t ds = da + ((uint64_t)(sl * a_bytes) >> 4);
                        tc_mma_step_f16<KC>(d0, d0 + (uint32_t)BN, ds, ds + (a_half >> 4),
                                            da + ((uint64_t)(a_all + sl * b_bytes) >> 4), idesc,
                                            accumulate, nullptr, two);
                        accumulate = 1;
                    }
                    const uint64_t ds = da + ((uint64_t)((NSL - 1) * a_bytes) >> 4);
                    tc_mma_step_f16<KC>(d0, d0 + (uint32_t)BN, ds, ds + (a_half >> 4),
                                        da + ((uint64_t)(a_all + (NSL - 1) * b_bytes) >> 4), idesc,
                                        accumulate, &empty[stage], two);
                }
                SK_TR(5, lane == 0);
#ifdef SK_CONV_TRACE
                ++tr_n;
#endif
                accumulate = 1;
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            tc_commit_elect(&tfull[acc]);
            __syncwarp();
        }
#ifdef SK_CONV_TRACE
        SK_CTA_REC(1, gtimer());
        SK_CTA_REC(2, (long long)tr_n);
#endif
    } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4) {
        // ====== epilogue: thread owns TMEM lane (quad*32+lane) = rows r, 128+r ======
        const int quad = warp & 3;
        const int lr = quad * 32 + lane;
        int local = 0;
        ItemSrc src;
        src.init(p, 2, n_items, item_ids, itfull, itempty);
        for (int item; (item = src.next()) >= 0; ++local) {
            Item it = decode(p, item);
            long long orow[2];
            orow[0] = out_index(p, it, lr);  // issued before the wait
            orow[1] = out_index(p, it, kTileM + lr);
            const int acc = acc_bufs == 2 ? (local & 1) : 0;
            const uint32_t aph = acc_bufs == 2 ? (uint32_t)((local >> 1) & 1) : (uint32_t)(local & 1);
            mbar_wait_sleep<256>(&tfull[acc], aph);
            tc_fence_after();
            const bool empty_tile = (it.m0 | it.m1) == 0;
            const int n0 = it.nt * BN;
#pragma unroll 1
            for (int h = 0; h < it.halves; ++h) {
                for (int c0 = 0; c0 < BN; c0 += 16) {
                    uint32_t v[16];
                    if (!empty_tile) {
                        tmem_ld16(tmem + ((uint32_t)(quad * 32) << 16) +
                                      (uint32_t)(acc * 2 * BN + h * BN + c0),
                                  v);
                        tmem_ld_wait();
                    } else {
#pragma unroll
                        for (int i = 0; i < 16; ++i) v[i] = 0;
                    }
                    const int col = n0 + c0;
                    if (orow[h] < 0 || col >= p.n_total) continue;
                    store16<T>(p, orow[h], col, v);
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty[acc]);
        }
    }
    pdl_trigger();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == kMmaWarp) tmem_dealloc(tmem, ncols);
    sched_finish(p);
}

// ---------------------------------------------------------------------------
// SIMT fp32 path: 128 rows x 64 cols per item, 256 threads, 8x4 per thread.
constexpr int kSimtN = 64;
constexpr int kSimtK = 16;

template <typename T>
__device__ __forceinline__ float to_f(T v) { return (float)v; }
template <>
__device__ __forceinline__ float to_f<__half>(__half v) { return __half2float(v); }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __half from_f<__half>(float v) { return __float2half_rn(v); }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

template <typename T>
__global__ void __launch_bounds__(256) k_gconv_simt(const ConvArgs p) {
    pdl_wait();
    pdl_trigger();
    __shared__ float As[kSimtK][kTileM + 4];
    __shared__ float Bs[kSimtK][kSimtN + 4];
    __shared__ int aidx[kTileM];
    const int tid = threadIdx.x;
    const int tr = tid / 16, tc = tid % 16;  // 16 x 16 threads; rows tr*8.., cols tc*4..
    const T* __restrict__ A = static_cast<const T*>(p.a);
    const T* __restrict__ Bw = static_cast<const T*>(p.b);
    const int n_items = num_items(p);
    for (int iter = blockIdx.x; iter < 2 * n_items; iter += gridDim.x) {
        const int item = iter >> 1, h = iter & 1;  // 128-row half h of a 256-row item
        Item it = decode(p, item);
        const int n0 = it.nt * kSimtN;
        // fp64 accumulators: this is the 1e-5 parity path, so a row's
        // K^D * C_in products must not carry fp32 summation error (the result
        // is rounded once, at the store)
        double acc[8][4];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
        unsigned long long m0 = it.m0, m1 = it.m1;
        for (int j = next_col(m0, m1, it.biw0, it.bw1); j >= 0;
             j = next_col(m0, m1, it.biw0, it.bw1)) {
            const int kg = it.col_begin + j;
            const int kb = p.mirror ? p.kd - 1 - kg : kg;
            __syncthreads();
            if (tid < kTileM) aidx[tid] = a_index(p, it, h * kTileM + tid, j);
            __syncthreads();
            for (int c0 = 0; c0 < p.k_total; c0 += kSimtK) {
                for (int i = tid; i < kTileM * kSimtK; i += 256) {
                    const int r = i / kSimtK, kk = i % kSimtK;
                    const int ai = aidx[r];
                    As[kk][r] = (ai >= 0 && c0 + kk < p.k_total)
                                    ? to_f(A[(size_t)ai * p.k_total + c0 + kk]) : 0.f;
                }
                for (int i = tid; i < kSimtN * kSimtK; i += 256) {
                    const int n = i / kSimtK, kk = i % kSimtK;
                    Bs[kk][n] = (n0 + n < p.n_total && c0 + kk < p.k_total)
                                    ? to_f(Bw[((size_t)kb * p.n_total + n0 + n) * p.k_total + c0 + kk])
                                    : 0.f;
                }
                __syncthreads();
#pragma unroll
                for (int kk = 0; kk < kSimtK; ++kk) {
                    float a[8], b[4];
#pragma unroll
                    for (int i = 0; i < 8; ++i) a[i] = As[kk][tr * 8 + i];
#pragma unroll
                    for (int i = 0; i < 4; ++i) b[i] = Bs[kk][tc * 4 + i];
#pragma unroll
                    for (int i = 0; i < 8; ++i)
#pragma unroll
                        for (int jj = 0; jj < 4; ++jj)
                            acc[i][jj] = fma((double)a[i], (double)b[jj], acc[i][jj]);
                }
                __syncthreads();
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const long long orow = out_index(p, it, h * kTileM + tr * 8 + i);
            if (orow < 0) continue;
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const int col = n0 + tc * 4 + jj;
                if (col >= p.n_total) continue;
                const size_t o = (size_t)orow * p.ld_y + col;
                const double res = p.residual ? (double)to_f(static_cast<const T*>(p.residual)[o]) : 0.0;
                if (p.out_mode == 0) static_cast<T*>(p.y)[o] = from_f<T>((float)(acc[i][jj] + res));
                else if (p.out_mode == 1) static_cast<float*>(p.y)[o] = (float)(acc[i][jj] + res);
                else if (p.out_mode == 2) atomicAdd(static_cast<float*>(p.y) + o, (float)acc[i][jj]);
                else {
                    float* d = static_cast<float*>(p.y) + o;
                    *d = (float)((double)*d + acc[i][jj]);
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// glue kernels

template <typename T>
__global__ void k_transpose_w(const T* __restrict__ w, int kd, int c_in, int c_out,
                              T* __restrict__ wt) {
    pdl_wait();
    pdl_trigger();
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    long long tot = (long long)kd * c_in * c_out;
    if (i >= tot) return;
    int k = (int)(i / ((long long)c_in * c_out));
    int rem = (int)(i % ((long long)c_in * c_out));
    int ci = rem / c_out, co = rem % c_out;
    wt[((size_t)k * c_out + co) * c_in + ci] = w[i];
}

template <typename T>
__global__ void k_convert_out(const float* __restrict__ src, long long n, T* __restrict__ dst,
                              const T* __restrict__ res) {
    pdl_wait();
    pdl_trigger();
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = from_f<T>(src[i] + (res ? to_f(res[i]) : 0.f));
}

// dst[r][0:k_pad] = src[r][0:k] with zero channels k..k_pad (tensor-core
// operands need 16 B rows: C_in % 8 != 0 inputs, e.g. the 4-channel stem)
template <typename T>
__global__ void k_pad_cols(const T* __restrict__ src, long long rows, int k, int k_pad,
                           T* __restrict__ dst) {
    pdl_wait();
    pdl_trigger();
    const long long n = rows * k_pad;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / k_pad;
        const int c = (int)(i % k_pad);
        dst[i] = c < k ? src[r * k + c] : from_f<T>(0.f);
    }
}

// GGS gather over the padded pair lists: buf[i] = x[in_pad[i]] (zeros for pads)
template <typename T>
__global__ void k_gather_rows(const T* __restrict__ x, int c, const int* __restrict__ idx,
                              const int* __restrict__ tile_total, T* __restrict__ buf) {
    pdl_wait();
    pdl_trigger();
    const long long nelem = (long long)(*tile_total) * kItemM * c;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nelem;
         i += (long long)gridDim.x * blockDim.x) {
        long long pr = i / c;
        int cc = (int)(i % c);
        int j = idx[pr];
        buf[i] = j >= 0 ? x[(size_t)j * c + cc] : from_f<T>(0.f);
    }
}

// GGS scatter-add into the fp32 accumulator: y[out_pad[i]] += buf[i] over the
// padded tiles [tile_lo, tile_hi); deterministic = one offset per launch
// (out rows unique within an offset, exec.cpp:140-146) with plain RMW.
__global__ void k_scatter_add(const float* __restrict__ buf, int c, const int* __restrict__ idx,
                              const int* __restrict__ tile_lo, const int* __restrict__ tile_hi,
                              float* __restrict__ y, int deterministic) {
    pdl_wait();
    pdl_trigger();
    const long long a = (long long)(*tile_lo) * kItemM, b = (long long)(*tile_hi) * kItemM;
    const long long nelem = (b - a) * c;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nelem;
         i += (long long)gridDim.x * blockDim.x) {
        long long pr = a + i / c;
        int cc = (int)(i % c);
        int o = idx[pr];
        if (o < 0) continue;
        float v = buf[pr * c + cc];
        float* d = y + (size_t)o * c + cc;
        if (deterministic) *d += v;
        else atomicAdd(d, v);
    }
}

// wgrad SIMT: one block per (offset, ci-tile 32, co-tile 32, pair-chunk);
// dW_k[ci][co] += sum_p x[in[p]][ci] * dy[out[p]][co], fp32 atomics across
// pair chunks (deterministic: one chunk).
// wgrad for tiny C_in (the 4-channel stem): dW[k][ci][co] = sum over offset
// k's pairs of x[in][ci] * dy[out][co]. Lane = output channel (coalesced dy
// row loads), warps stride over the pairs with the CI input values broadcast,
// CI fp32 accumulators per lane; the block's 8 warps reduce in smem and flush
// one red.add per (ci, co). The 32x32-tile SIMT kernel wasted 28 of 32 rows
// of every tile on C_in = 4 (337 us -> tens of us per MinkUNet scan).
template <typename T, int CI>
__global__ void __launch_bounds__(256) k_wgrad_small_cin(const T* __restrict__ x,
                                                         const T* __restrict__ dy, int c_out,
                                                         const long long* __restrict__ ptr,
                                                         const int* __restrict__ ws_in,
                                                         const int* __restrict__ ws_out, int chunk,
                                                         float* __restrict__ dw) {
    pdl_wait();
    pdl_trigger();
    const int k = blockIdx.z;
    const long long b = ptr[k], e = ptr[k + 1];
    const long long p0 = b + (long long)blockIdx.x * chunk;
    const long long p1 = p0 + chunk < e ? p0 + chunk : e;
    if (p0 >= p1) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int co = blockIdx.y * 32 + lane;
    const bool live = co < c_out;
    float acc[CI];
#pragma unroll
    for (int c = 0; c < CI; ++c) acc[c] = 0.f;
    long long p = p0 + warp;
    for (; p + 24 < p1; p += 32) {  // four pairs per trip: loads in flight together
        int ii[4], oo[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            ii[u] = __ldg(ws_in + p + 8 * u);
            oo[u] = __ldg(ws_out + p + 8 * u);
        }
        float g[4], xv[4][CI];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            g[u] = live ? to_f(dy[(size_t)oo[u] * c_out + co]) : 0.f;
#pragma unroll
            for (int c = 0; c < CI; ++c) xv[u][c] = to_f(x[(size_t)ii[u] * CI + c]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int c = 0; c < CI; ++c) acc[c] = fmaf(xv[u][c], g[u], acc[c]);
    }
    for (; p < p1; p += 8) {
        const int i = __ldg(ws_in + p), o = __ldg(ws_out + p);
        const float g = live ? to_f(dy[(size_t)o * c_out + co]) : 0.f;
#pragma unroll
        for (int c = 0; c < CI; ++c) acc[c] = fmaf(to_f(x[(size_t)i * CI + c]), g, acc[c]);
    }
    __shared__ float red[8][CI][32];
#pragma unroll
    for (int c = 0; c < CI; ++c) red[warp][c][lane] = acc[c];
    __syncthreads();
    if (warp < CI && live) {  // warp c flushes input channel c
        float sum = 0.f;
#pragma unroll
        for (int w = 0; w < 8; ++w) sum += red[w][warp][lane];
        atomicAdd(dw + ((size_t)k * CI + warp) * c_out + co, sum);
    }
}

// fp64 accumulation (per thread over its chunk, fp64 atomics across chunks
// into dw64): the fp32 path's dW sums tens of thousands of pairs per cell and
// must stay within 1e-5 of the f64 reference; dw64 is rounded once.
template <typename T>
__global__ void __launch_bounds__(256) k_wgrad_simt(const T* __restrict__ x,
                                                    const T* __restrict__ dy, int c_in, int c_out,
                                                    const long long* __restrict__ ptr,
                                                    const int* __restrict__ ws_in,
                                                    const int* __restrict__ ws_out, int chunk,
                                                    double* __restrict__ dw) {
    pdl_wait();
    pdl_trigger();
    __shared__ float xs[32][33];
    __shared__ float ds[32][33];
    const int k = blockIdx.z;
    const int ci0 = (blockIdx.y / ((c_out + 31) / 32)) * 32;
    const int co0 = (blockIdx.y % ((c_out + 31) / 32)) * 32;
    const long long lo = ptr[k], hi = ptr[k + 1];
    const long long p0 = lo + (long long)blockIdx.x * chunk;
    if (p0 >= hi) return;
    const long long p1 = min(hi, p0 + chunk);
    const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // 32 x 8
    double acc[4] = {0, 0, 0, 0};
    for (long long pb = p0; pb < p1; pb += 32) {
        for (int i = threadIdx.x; i < 32 * 32; i += 256) {
            int pp = i / 32, cc = i % 32;
            long long pr = pb + pp;
            bool ok = pr < p1;
            xs[pp][cc] = (ok && ci0 + cc < c_in) ? to_f(x[(size_t)ws_in[pr] * c_in + ci0 + cc]) : 0.f;
            ds[pp][cc] = (ok && co0 + cc < c_out) ? to_f(dy[(size_t)ws_out[pr] * c_out + co0 + cc]) : 0.f;
        }
        __syncthreads();
#pragma unroll 8
        for (int pp = 0; pp < 32; ++pp) {
            float d = ds[pp][tx];
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[u] = fma((double)xs[pp][ty * 4 + u], (double)d, acc[u]);
        }
        __syncthreads();
    }
    for (int u = 0; u < 4; ++u) {
        int ci = ci0 + ty * 4 + u, co = co0 + tx;
        if (ci < c_in && co < c_out) atomicAdd(&dw[((size_t)k * c_in + ci) * c_out + co], acc[u]);
    }
}

// dw (fp32) = [dw +] dw64, rounded once
__global__ void k_round_f64(const double* __restrict__ src, long long n, float* __restrict__ dw,
                            int accumulate) {
    pdl_wait();
    pdl_trigger();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        dw[i] = accumulate ? (float)((double)dw[i] + src[i]) : (float)src[i];
}

// ---------------------------------------------------------------------------
// tcgen05 wgrad: dW_k[ci][co] = sum_p x[in_p][ci] * dy[out_p][co] (exec.cpp:259-279)
// GEMM with M = C_in (128-channel tiles), N = C_out tile, K = the pairs of one
// offset. Both operands are gathered rows, i.e. MN-major: each pair's row is
// 128 B of channels, 8 pairs form a 1024 B SW128 atom (SBO), 64-channel
// blocks are LBO = 8 KB apart. CTA b owns a contiguous range of virtual tiles
// (mn-tile, 256-pair tile); consecutive tiles of the same (mn, offset)
// accumulate in TMEM and are flushed with fp32 red.add when the run ends.
constexpr int kWgK = 64;            // pairs per k-step
constexpr int kWgThreads = 288;     // warps 0-3 producers, 4 MMA, 5-8 epilogue
constexpr int kWgStepsPerTile = kTileWS / kWgK;

struct WgArgs {
    const void* x;
    const void* dy;
    int c_in, c_out, kd;
    const int* tile_ptr;  // [kd+1], 256-pair tiles per offset
    const int* in_pad;
    const int* out_pad;
    float* dw;
    int m_tiles, n_tiles, bn, nblk_b;
};

__device__ __forceinline__ uint64_t mnmajor_desc(uint32_t saddr) {
    constexpr uint64_t lbo = 8192 >> 4, sbo = 1024 >> 4;
    return (uint64_t)((saddr >> 4) & 0x3FFF) | (lbo << 16) | (sbo << 32) | (1ull << 46) |
           (2ull << 61);
}

__device__ __forceinline__ int wg_offset_of(const int* tp, int kd, int t) {
    int k = 0;
    while (k + 1 <= kd && tp[k + 1] <= t) ++k;
    return k;
}

template <typename T>
__global__ void __launch_bounds__(kWgThreads, 3) k_wgrad_tc(const WgArgs p, int stages) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t a_bytes = 2 * 8192;                   // 128 channels x 64 pairs
    const uint32_t b_bytes = (uint32_t)p.nblk_b * 8192;  // bn channels (64-blocks) x 64 pairs
    const uint32_t stage_bytes = a_bytes + b_bytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)stages * stage_bytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + stages;
    uint64_t* tfull = bars + 2 * stages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int BN = p.bn;
    uint32_t ncols = 32;
    while (ncols < (uint32_t)(2 * BN)) ncols <<= 1;
    if (threadIdx.x == 0) {
        if (smem_u32(smem) & 1023) __trap();
        for (int i = 0; i < stages; ++i) {
            mbar_init(&full[i], 128);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 128);
        }
        fence_mbar_init();
    }
    if (warp == 4) tmem_alloc(tmem_slot, ncols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const long long NT = p.tile_ptr[p.kd];  // 256-pair tiles
    const long long V = NT * p.m_tiles * p.n_tiles;
    const long long v0 = V * blockIdx.x / gridDim.x, v1 = V * (blockIdx.x + 1) / gridDim.x;

    if (warp < 4) {
        // producers: threads 0-63 gather x rows, 64-127 dy rows (pair t % 64),
        // 16 B cp.async per 8 channels; indices prefetched 8 steps ahead
        const int t = threadIdx.x;
        const bool is_x = t < 64;
        const int kk = t & 63;
        const int C = is_x ? p.c_in : p.c_out;
        const T* src = static_cast<const T*>(is_x ? p.x : p.dy);
        const int* idx = is_x ? p.in_pad : p.out_pad;
        const long long nsteps = (v1 - v0) * kWgStepsPerTile;
        auto pair_of = [&](long long g) -> long long {
            const long long v = v0 + g / kWgStepsPerTile;
            return (v % NT) * kTileWS + (g % kWgStepsPerTile) * kWgK + kk;
        };
        // indices for the next group of 8 steps are loaded while the current
        // group is issued (no register shifting: a shift would wait for each
        // load one step later, i.e. a lookahead of one)
        int cur[8], nxt[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) cur[i] = i < nsteps ? __ldg(idx + pair_of(i)) : -1;
        int stage = 0;
        uint32_t phase = 0;
        for (long long g0 = 0; g0 < nsteps; g0 += 8) {
#pragma unroll
            for (int i = 0; i < 8; ++i) nxt[i] = g0 + 8 + i < nsteps ? __ldg(idx + pair_of(g0 + 8 + i)) : -1;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const long long g = g0 + i;
            if (g >= nsteps) break;
            const int row = cur[i];
            const long long v = v0 + g / kWgStepsPerTile;
            const long long mn = v / NT;
            const int c_lo = is_x ? (int)(mn / p.n_tiles) * 128 : (int)(mn % p.n_tiles) * BN;
            const int c_n = min(is_x ? 128 : BN, C - c_lo);
            mbar_wait(&empty[stage], phase ^ 1);
            const uint32_t sbase = smem_u32(smem) + (uint32_t)stage * stage_bytes + (is_x ? 0 : a_bytes);
            const T* rp = src + (size_t)(row < 0 ? 0 : row) * C + c_lo;
            for (int c = 0; c < c_n; c += 8) {
                const uint32_t off = (uint32_t)(c / 64) * 8192 + (uint32_t)(kk / 8) * 1024 +
                                     (uint32_t)(kk % 8) * 128 + (uint32_t)((c % 64) / 8) * 16;
                const uint32_t sw = off ^ (((off >> 7) & 7) << 4);
                cp_async16(sbase + sw, row < 0 ? (const void*)src : (const void*)(rp + c),
                           row < 0 ? 0u : 16u);
            }
            cp_async_arrive_noinc(&full[stage]);
            if (++stage == stages) {
                stage = 0;
                phase ^= 1;
            }
        }
#pragma unroll
            for (int i = 0; i < 8; ++i) cur[i] = nxt[i];
        }
    } else if (warp == 4) {
        // MMA issuer: runs of tiles with the same (mn tile, offset) accumulate
        const uint32_t idesc = (1u << 4) | (Fmt<T>::v << 7) | (Fmt<T>::v << 10) | (1u << 15) |
                               (1u << 16) | ((uint32_t)(BN >> 3) << 17) |
                               ((uint32_t)(kTileM >> 4) << 24);
        int stage = 0;
        uint32_t phase = 0;
        int run = -1;
        long long cur_key = -1;
        uint32_t acc = 0, accumulate = 0;
        for (long long v = v0; v < v1; ++v) {
            const long long mn = v / NT;
            const long long key = mn * (p.kd + 1) + wg_offset_of(p.tile_ptr, p.kd, (int)(v % NT));
            if (key != cur_key) {
                if (run >= 0) tc_commit_elect(&tfull[acc]);
                ++run;
                acc = run & 1;
                mbar_wait(&tempty[acc], (uint32_t)(((run >> 1) & 1) ^ 1));
                tc_fence_after();
                cur_key = key;
                accumulate = 0;
            }
            for (int sidx = 0; sidx < kWgStepsPerTile; ++sidx) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                {
                    // warp-uniform issue, elected lane inside the asm (descriptors
                    // stay in uniform registers); +2048 B per K=16 step
                    const uint32_t sa = smem_u32(smem) + (uint32_t)stage * stage_bytes;
                    const uint64_t da = mnmajor_desc(sa), db = mnmajor_desc(sa + a_bytes);
#pragma unroll
                    for (int k16 = 0; k16 < kWgK / 16; ++k16) {
                        asm volatile(
                            "{\n.reg .pred E, p;\n"
                            "elect.sync _|E, 0xffffffff;\n"
                            "setp.ne.b32 p, %4, 0;\n"
                            "@E tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
                            "}\n" ::"r"(tmem + acc * (uint32_t)BN),
                            "l"(da + (uint64_t)(k16 * 128)), "l"(db + (uint64_t)(k16 * 128)),
                            "r"(idesc), "r"(accumulate)
                            : "memory");
                        accumulate = 1;
                    }
                    tc_commit_elect(&empty[stage]);
                }
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
        if (run >= 0) tc_commit_elect(&tfull[acc]);
        __syncwarp();
    } else {
        // epilogue: TMEM lane = channel ci of the M tile; flush a run with red.add
        const int quad = warp & 3;
        const int lr = quad * 32 + lane;
        int run = -1;
        long long cur_key = -1, cur_mn = 0;
        int cur_k = 0;
        auto flush = [&](int r, long long mn, int k) {
            const uint32_t a = r & 1;
            mbar_wait(&tfull[a], (uint32_t)((r >> 1) & 1));
            tc_fence_after();
            const int ci = (int)(mn / p.n_tiles) * 128 + lr;
            const int co0 = (int)(mn % p.n_tiles) * BN;
            for (int c0 = 0; c0 < BN; c0 += 16) {
                uint32_t v[16];
                tmem_ld16(tmem + ((uint32_t)(quad * 32) << 16) + a * (uint32_t)BN + (uint32_t)c0, v);
                tmem_ld_wait();
                if (ci >= p.c_in) continue;
                float* dst = p.dw + ((size_t)k * p.c_in + ci) * p.c_out + co0 + c0;
                const int lim = min(16, p.c_out - co0 - c0);
                if (lim == 16 && (p.c_out % 4) == 0) {
#pragma unroll
                    for (int i = 0; i < 16; i += 4)
                        red_add_v4(dst + i, __uint_as_float(v[i]), __uint_as_float(v[i + 1]),
                                   __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
                } else {
                    for (int i = 0; i < lim; ++i) atomicAdd(dst + i, __uint_as_float(v[i]));
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty[a]);
        };
        for (long long v = v0; v < v1; ++v) {
            const long long mn = v / NT;
            const int k = wg_offset_of(p.tile_ptr, p.kd, (int)(v % NT));
            const long long key = mn * (p.kd + 1) + k;
            if (key != cur_key) {
                if (run >= 0) flush(run, cur_mn, cur_k);
                ++run;
                cur_key = key;
                cur_mn = mn;
                cur_k = k;
            }
        }
        if (run >= 0) flush(run, cur_mn, cur_k);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 4) tmem_dealloc(tmem, ncols);
}

size_t elem_size(sk_dtype dt) { return dt == SK_F32 ? 4 : 2; }

}  // namespace

// ---- tensor maps (driver entry point resolved once through cudart) ----
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        SK_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
        if (!f || q != cudaDriverEntryPointSuccess)
            fail(SK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<EncodeTiledFn>(f);
    }();
    return fn;
}

// 2D row-major tensor [rows][cols] with row pitch ld (elements), any element
// type, box {box_cols, box_rows}, swizzle = box_cols * elem bytes (32/64/128)
CUtensorMap make_tmap_rows(const void* base, CUtensorMapDataType ty, int elem_bytes, long long cols,
                           long long rows, long long ld, int box_cols, int box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)std::max<long long>(rows, 1)};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * elem_bytes)};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    const int rb = box_cols * elem_bytes;
    CUtensorMapSwizzle sw = rb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                          : rb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
    CUresult r = encode_fn()(&m, ty, 2, const_cast<void*>(base), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(SK_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return m;
}

// 2D row-major [rows][cols] half tensor, box {kc, box_rows}, swizzle = kc*2 bytes
CUtensorMap make_tmap(const void* base, sk_dtype dt, int cols, long long rows, int kc,
                      int box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)std::max<long long>(rows, 1)};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)kc, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUtensorMapSwizzle sw = kc == 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                          : kc == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
    CUresult r = encode_fn()(&m, dt == SK_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                               : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                             2, const_cast<void*>(base), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(SK_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return m;
}

namespace {

template <typename T, int KC, bool TMA, int SLABS, int PW>
void launch_tc_variant(const ConvArgs& a, const CUtensorMap& ta, const CUtensorMap& tb,
                       int grid, int stages, int acc_bufs, size_t stage_bytes,
                       cudaStream_t st) {
    const size_t smem = stages * stage_bytes + kIdxRing * (kItemM * 4 + 16) +
                        (2 * stages + 4 + 3 * kIdxRing + 2 * kItemRing) * 8 + 16 + kItemRing * 4 +
                        kIdxRing * sizeof(CSlot<PW>);
    auto kern = k_gconv_tc<T, KC, TMA, SLABS, PW>;
    ensure_smem(reinterpret_cast<const void*>(kern), smem);
    launch_pdl(kern, grid, Roles<PW>::kThreads, smem, st, ta, tb, a, stages, acc_bufs);
}

template <typename T, int KC>
void launch_tc_kc(const ConvArgs& a, sk_dtype dt, int grid, int num_sms, cudaStream_t st) {
    // Variant choice follows the layer's TilePreset (tuned per group; the
    // defaults are the measured winners, profiles/r01_gather_paths.md,
    // r01_gather_pipeline.md, r02_gather_redesign.md):
    //  * gather: cp.async (default) or TMA tile::gather4 (load_width 1);
    //  * two CTAs per SM (8 gather warps, ~100 KB of stages each) for
    //    C_out <= 128 unless cta_m = 256 asks for one CTA (16 gather warps);
    //  * C_in = 96 runs three 32-channel K-slabs per stage (one CTA per SM)
    //    unless cta_k = 32 asks for single-slab stages.
    constexpr int kMinSlabStages = 3;
    const int bn = a.bn;
    const bool tma = a.tma_gather || a.mode == 2;  // dense A always streams 2D TMA tiles
    const bool two_cta = a.cta_m != 256;
    const int nchunks = (int)ceil_div(a.k_total, KC);
    const size_t slab_bytes = (size_t)kItemM * KC * 2 + (size_t)bn * KC * 2;
    CUtensorMap ta, tb;
    if (tma) ta = make_tmap(a.a, dt, a.k_total, a.n_rows_a, KC, a.mode == 2 ? kTileM : 1);
    else memset(&ta, 0, sizeof(ta));
    tb = make_tmap(a.b, dt, a.k_total, (long long)a.kd * a.n_total, KC, bn);
    const bool slab3 = a.cta_k != 32 && !tma && KC == 32 && nchunks == 3;
    if (!tma && two_cta && bn <= 32 && !slab3) {
        // three CTAs per SM (4 gather warps each, ~64 KB of stages) for
        // C_out <= 32: a third independent pipeline per SM (C=32 lidar layer
        // 44.0 -> 39.9 us). C_out = 64 with 32-channel stages on this path:
        // 58.4 -> 70.6 us (one accumulator pair; measured, not used)
        const int stages = (int)std::min<size_t>(kMaxStages, (64 * 1024) / slab_bytes);
        if (stages >= 2) {
            const int acc3 = 4 * bn <= 128 ? 2 : 1;
            const int g3 = a.mode == 1 ? 3 * num_sms : std::min(a.items, 3 * num_sms);
            launch_tc_variant<T, KC, false, 1, 4>(a, ta, tb, std::max(1, g3), stages, acc3, slab_bytes, st);
            return;
        }
    }
    if (!tma && two_cta && bn <= 128 && !slab3) {
        // TMEM per CTA <= 256 columns: double-buffer only up to BN = 64
        const int acc_bufs = 4 * bn <= 256 ? 2 : 1;
        const int stages = (int)std::min<size_t>(kMaxStages, (96 * 1024) / slab_bytes);
        if (stages >= 2) {
            const int g2 = a.mode == 1 ? 2 * num_sms : std::min(a.items, 2 * num_sms);
            launch_tc_variant<T, KC, false, 1, 8>(a, ta, tb, std::max(1, g2), stages, acc_bufs,
                                                  slab_bytes, st);
            return;
        }
    }
    // C_in = 96 (three 32-channel slabs) is the one width where fusing the
    // chunks pays (measured: C = 64/128 gain nothing, and SLABS stays a
    // compile-time constant so the single-slab kernel keeps its lean loops)
    const int slabs = (slab3 && ((size_t)bn * KC * 2) % 1024 == 0 &&
                       (size_t)kMinSlabStages * 3 * slab_bytes <= 200 * 1024) ? 3 : 1;
    const size_t stage_bytes = slabs * slab_bytes;
    int stages = (int)std::min<size_t>(kMaxStages, (200 * 1024) / stage_bytes);
    stages = std::max(stages, 2);
    const int acc_bufs = 4 * bn <= 512 ? 2 : 1;  // double-buffered TMEM accumulators
    if (tma) launch_tc_variant<T, KC, true, 1, 16>(a, ta, tb, grid, stages, acc_bufs, stage_bytes, st);
    else if (slabs == 3)
        launch_tc_variant<T, KC, false, 3, 16>(a, ta, tb, grid, stages, acc_bufs, stage_bytes, st);
    else launch_tc_variant<T, KC, false, 1, 16>(a, ta, tb, grid, stages, acc_bufs, stage_bytes, st);
}

template <typename T>
void launch_tc(const ConvArgs& a, sk_dtype dt, int grid, int num_sms, cudaStream_t st) {
    // channel step: the widest of 64 / 32 / 16 dividing C_in, or the
    // preset's cta_k when it divides C_in
    const int k = a.k_total;
    const int pref = (a.cta_k == 16 || a.cta_k == 32 || a.cta_k == 64) && k % a.cta_k == 0 ? a.cta_k : 0;
    const int kc = pref ? pref : (k % 64 == 0 ? 64 : (k % 32 == 0 ? 32 : 16));
    if (kc == 64) launch_tc_kc<T, 64>(a, dt, grid, num_sms, st);
    else if (kc == 32) launch_tc_kc<T, 32>(a, dt, grid, num_sms, st);
    else launch_tc_kc<T, 16>(a, dt, grid, num_sms, st);
}

bool tc_ok(sk_dtype dt, int k_total, int n_total) {
    return dt != SK_F32 && k_total % 8 == 0 && n_total % 16 == 0;
}

// N tile: whole C_out when <= 256 (or <= cta_n), else balanced tiles
void pick_n_tiling(int n_total, int cta_n, bool tc, int& bn, int& n_nt) {
    if (!tc) {
        bn = kSimtN;
        n_nt = (int)ceil_div(n_total, kSimtN);
        return;
    }
    int cap = cta_n > 0 ? std::min(cta_n, 256) : 256;
    cap = std::max(16, cap / 16 * 16);
    n_nt = (int)ceil_div(n_total, cap);
    bn = (int)ceil_div(ceil_div(n_total, n_nt), 16) * 16;
}

void launch_gconv(sk_ctx* ctx, sk_dtype dt, const ConvArgs& a_in, cudaStream_t st) {
    ConvArgs a = a_in;
#ifdef SK_CONV_TRACE
    DevBuf tbuf;
    const char* tpath = getenv("SK_TRACE");
    if (tpath) {
        tbuf.alloc((4096 * 16 + 4 * 1024) * 8, st);
        fill_async(tbuf.p, 0, tbuf.bytes, st);
        a.trace = tbuf.as<long long>();
    }
    a.exp = getenv("SK_EXP") ? atoi(getenv("SK_EXP")) : 0;
    struct Dump {
        DevBuf& b; const char* path; cudaStream_t st; const ConvArgs& a;
        ~Dump() {
            if (!path) return;
            std::vector<long long> h(4096 * 16 + 4 * 1024);
            cudaMemcpyAsync(h.data(), b.p, b.bytes, cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            if (FILE* f = fopen(path, "a")) {
                fprintf(f, "# k=%d n=%d bn=%d\n", a.k_total, a.n_total, a.bn);
                for (int i = 0; i < 4096 && h[i * 8 + 4]; ++i) {
                    for (int j = 0; j < 8; ++j) fprintf(f, "%lld ", h[i * 8 + j]);
                    for (int j = 0; j < 4; ++j) fprintf(f, "%lld ", h[4096 * 8 + i * 4 + j]);
                    for (int j = 0; j < 2; ++j) fprintf(f, "%lld ", h[4096 * 12 + i * 2 + j]);
                    for (int j = 0; j < 2; ++j) fprintf(f, "%lld ", h[4096 * 14 + i * 2 + j]);
                    fprintf(f, "\n");
                }
                fprintf(f, "# cta start end stages smid\n");
                for (int c = 0; c < 1024 && h[4096 * 16 + c * 4 + 1]; ++c)
                    fprintf(f, "C %d %lld %lld %lld %lld\n", c, h[4096 * 16 + c * 4], h[4096 * 16 + c * 4 + 1],
                            h[4096 * 16 + c * 4 + 2], h[4096 * 16 + c * 4 + 3]);
                fclose(f);
            }
        }
    } dump{tbuf, tpath, st, a};
#endif
    const bool tc = tc_ok(dt, a.k_total, a.n_total);
    if (tc) a.sched = ctx->sched_slot();  // dynamic item queue (ItemSrc)
    int grid;
    if (a.mode != 1) grid = std::max(1, std::min(a.items, ctx->num_sms * (tc ? 1 : 8)));
    else grid = ctx->num_sms * (tc ? 1 : 8);
    if (tc) {
        if (dt == SK_F16) launch_tc<__half>(a, dt, grid, ctx->num_sms, st);
        else launch_tc<__nv_bfloat16>(a, dt, grid, ctx->num_sms, st);
    } else {
        if (dt == SK_F32) launch_pdl(k_gconv_simt<float>, grid, 256, 0, st, a);
        else if (dt == SK_F16) launch_pdl(k_gconv_simt<__half>, grid, 256, 0, st, a);
        else launch_pdl(k_gconv_simt<__nv_bfloat16>, grid, 256, 0, st, a);
    }
}

template <typename T>
void convert_out(const float* src, long long n, void* dst, const void* res, cudaStream_t st) {
    if (n <= 0) return;
    launch_pdl(k_convert_out<T>, (int)ceil_div(n, 256), 256, 0, st, src, n, static_cast<T*>(dst),
                                                              static_cast<const T*>(res));
}

// fp32 accumulator -> output dtype (+ fused residual)
void convert_from_f32(sk_dtype dt, const float* src, long long n, void* dst, const void* res,
                      cudaStream_t st) {
    if (dt == SK_F16) convert_out<__half>(src, n, dst, res, st);
    else if (dt == SK_BF16) convert_out<__nv_bfloat16>(src, n, dst, res, st);
    else if (res || src != dst) convert_out<float>(src, n, dst, res, st);
}

template <typename T>
void pad_cols(const void* src, long long rows, int k, int k_pad, void* dst, cudaStream_t st) {
    const long long n = rows * k_pad;
    if (n <= 0) return;
    launch_pdl(k_pad_cols<T>, (int)std::min<long long>(ceil_div(n, 256), 148 * 32), 256, 0, st, static_cast<const T*>(src), rows, k, k_pad, static_cast<T*>(dst));
}

// Implicit GEMM on CUDA cores for tiny C_in (<= 8, the 4-channel stem):
// one thread per output row keeps its C_out fp32 accumulators in registers,
// walks the raw OS row (unsorted map) and FMAs the neighbour's C_in values
// against W_k staged in smem as fp32. The tensor-core path would move 16 B
// rows through a 256-row pipeline step for 8 MACs per output channel.
template <typename T, int CI, int CO>
__global__ void __launch_bounds__(256) k_conv_small_cin(
    const int* __restrict__ os, int n_out, int kd, const T* __restrict__ x, const T* __restrict__ w,
    T* __restrict__ y, const T* __restrict__ residual, float* __restrict__ y_accum) {
    pdl_wait();
    pdl_trigger();
    // persistent blocks: W staged once per block as fp32; 4 threads per output
    // row, each owning CO/4 output channels (latency hiding + short tails)
    constexpr int KD = 27, TPR = 4, CQ = CO / TPR;
    extern __shared__ float4 wsh4[];  // [kd][CI][CO/4] fp32
    float* wsh = reinterpret_cast<float*>(wsh4);
    {  // stage W with every element's load in flight at once (one latency, not ~14)
        constexpr int PER = (KD * CI * CO + 255) / 256;
        float v[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int i = threadIdx.x + j * 256;
            v[j] = i < kd * CI * CO ? to_f(w[i]) : 0.f;
        }
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int i = threadIdx.x + j * 256;
            if (i < kd * CI * CO) wsh[i] = v[j];
        }
    }
    __syncthreads();
    const int sub = threadIdx.x % TPR;
    for (int row = (blockIdx.x * blockDim.x + threadIdx.x) / TPR; row < n_out;
         row += gridDim.x * blockDim.x / TPR) {
        float acc[CQ];
#pragma unroll
        for (int c = 0; c < CQ; ++c) acc[c] = 0.f;
        const int* e = os + (size_t)row * kd;
        int nb[KD];
#pragma unroll
        for (int k = 0; k < KD; ++k) nb[k] = k < kd ? __ldg(e + k) : -1;
        // all neighbour rows in flight at once (one load latency per row, not
        // 27 dependent ones: 67 -> ~15 us for the MinkUNet stem)
        uint2 xr[KD];
        if constexpr (CI == 4 && sizeof(T) == 2) {
#pragma unroll
            for (int k = 0; k < KD; ++k)
                xr[k] = nb[k] >= 0 ? __ldg(reinterpret_cast<const uint2*>(x) + nb[k]) : make_uint2(0, 0);
        }
#pragma unroll
        for (int k = 0; k < KD; ++k) {
            if (nb[k] < 0) continue;
            float xv[CI];
            if constexpr (CI == 4 && sizeof(T) == 2) {
                const uint2 u = xr[k];
                const float2 a = unpack2(u.x, (T*)nullptr), b = unpack2(u.y, (T*)nullptr);
                xv[0] = a.x; xv[1] = a.y; xv[2] = b.x; xv[3] = b.y;
            } else {
#pragma unroll
                for (int c = 0; c < CI; ++c) xv[c] = to_f(x[(size_t)nb[k] * CI + c]);
            }
            const float4* wk = wsh4 + k * CI * (CO / 4) + sub * (CQ / 4);
#pragma unroll
            for (int ci = 0; ci < CI; ++ci)
#pragma unroll
                for (int c4 = 0; c4 < CQ / 4; ++c4) {
                    const float4 wv = wk[ci * (CO / 4) + c4];
                    acc[4 * c4 + 0] = fmaf(xv[ci], wv.x, acc[4 * c4 + 0]);
                    acc[4 * c4 + 1] = fmaf(xv[ci], wv.y, acc[4 * c4 + 1]);
                    acc[4 * c4 + 2] = fmaf(xv[ci], wv.z, acc[4 * c4 + 2]);
                    acc[4 * c4 + 3] = fmaf(xv[ci], wv.w, acc[4 * c4 + 3]);
                }
        }
        const size_t o = (size_t)row * CO + sub * CQ;
        if (y_accum) {
#pragma unroll
            for (int c = 0; c < CQ; ++c) y_accum[o + c] += acc[c];
            continue;
        }
#pragma unroll
        for (int c = 0; c < CQ; ++c) {
            const float r = residual ? to_f(residual[o + c]) : 0.f;
            y[o + c] = from_f<T>(acc[c] + r);
        }
    }
}

// Tiny-C_in layers (the stem) as ONE dense tensor-core GEMM: gather every
// output row's K^D neighbour rows into A[row][k*CI + c] (zeros for missing
// neighbours and the pad to K_pad, a multiple of 16), so that
// y = A [n_out x K_pad] . Wc [K_pad x C_out] with Wc[k*CI + c][co] = W[k][c][co]
// runs on k_dense_tc. The CUDA-core path spent ~60 us on the MinkUNet stem
// (low occupancy, LDS-latency-bound FMA chains); the gather writes n_out x
// K_pad halves once and the GEMM streams them.
template <typename T, int CI>
__global__ void __launch_bounds__(256) k_im2col_small(const int* __restrict__ os, int n_out, int kd,
                                                      const T* __restrict__ x, int k_pad,
                                                      T* __restrict__ a) {
    pdl_wait();
    pdl_trigger();
    const long long tot = (long long)n_out * (k_pad / CI);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
         i += (long long)gridDim.x * blockDim.x) {
        const int row = (int)(i / (k_pad / CI)), k = (int)(i % (k_pad / CI));
        const int nb = k < kd ? __ldg(os + (size_t)row * kd + k) : -1;
        T* dst = a + (size_t)row * k_pad + k * CI;
        if constexpr (CI == 4 && sizeof(T) == 2) {
            *reinterpret_cast<uint2*>(dst) =
                nb >= 0 ? __ldg(reinterpret_cast<const uint2*>(x) + nb) : make_uint2(0, 0);
        } else {
#pragma unroll
            for (int c = 0; c < CI; ++c) dst[c] = nb >= 0 ? x[(size_t)nb * CI + c] : from_f<T>(0.f);
        }
    }
}
// Wc^T, K-major: b[co][k*CI + c] = W[k][c][co]; zero pad columns
template <typename T>
__global__ void k_small_cin_weights(const T* __restrict__ w, int kd, int ci, int co, int k_pad,
                                    T* __restrict__ b) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= co * k_pad) return;
    const int o = i / k_pad, kk = i % k_pad;
    const int k = kk / ci, c = kk % ci;
    b[i] = k < kd ? w[((size_t)k * ci + c) * co + o] : from_f<T>(0.f);
}

template <typename T>
bool conv_small_cin_dense(sk_ctx* ctx, sk_dtype dt, const sk_kmap* m, int c_in, int c_out,
                          const void* x, const void* w, void* y, int cta_n, cudaStream_t st) {
    // 8 B neighbour-row loads: the feature rows (4 halves) must be 8 B aligned
    if (c_in != 4 || c_out % 16 != 0 || (reinterpret_cast<uintptr_t>(x) & 7) != 0) return false;
    const int k_pad = (int)ceil_div((long long)m->kd * c_in, 16) * 16;
    DevBuf a, b;
    a.alloc((size_t)m->n_out * k_pad * sizeof(T), st);
    b.alloc((size_t)c_out * k_pad * sizeof(T), st);
    const long long tot = (long long)m->n_out * (k_pad / c_in);
    launch_pdl(k_im2col_small<T, 4>, (int)std::min<long long>(ceil_div(tot, 256), (long long)ctx->num_sms * 16),
               256, 0, st, m->os.as<int>(), m->n_out, m->kd, static_cast<const T*>(x), k_pad, a.as<T>());
    launch_pdl(k_small_cin_weights<T>, (int)ceil_div((long long)c_out * k_pad, 256), 256, 0, st,
               static_cast<const T*>(w), m->kd, c_in, c_out, k_pad, b.as<T>());
    return dense_identity_tc(ctx, dt, m->n_out, k_pad, c_out, a.p, b.p, y, nullptr, nullptr, cta_n, st);
}

template <typename T>
bool conv_small_cin(const sk_kmap* m, int c_in, int c_out, const void* x, const void* w, void* y,
                    const void* residual, float* y_accum, cudaStream_t st) {
    auto launch = [&](auto kern) {
        const size_t smem = (size_t)m->kd * c_in * c_out * 4;
        ensure_smem(reinterpret_cast<const void*>(kern), smem);
        // persistent: each block stages W once, then walks many rows
        const int grid = (int)std::min<int64_t>(ceil_div(m->n_out, 64), (int64_t)m->ctx->num_sms * 2);
        launch_pdl(kern, grid, 256, smem, st, m->os.as<int>(), m->n_out, m->kd, static_cast<const T*>(x), static_cast<const T*>(w),
            static_cast<T*>(y), static_cast<const T*>(residual), y_accum);
        return true;
    };
    if (m->kd > 27) return false;
    // CI = 4 half rows are read as 8 B vectors: the feature base must be 8 B aligned
    if (c_in == 4 && c_out == 32 && (reinterpret_cast<uintptr_t>(x) & 7) == 0)
        return launch(k_conv_small_cin<T, 4, 32>);
    if (c_in == 3 && c_out == 32) return launch(k_conv_small_cin<T, 3, 32>);
    if (c_in == 1 && c_out == 32) return launch(k_conv_small_cin<T, 1, 32>);
    return false;
}

ConvArgs base_args() {
    ConvArgs a;
    memset(&a, 0, sizeof(a));
    a.split_only = -1;
    a.offset_only = -1;
    return a;
}

template <typename T>
void gather_rows(const void* x, int c, const int* idx, const int* tiles, void* buf, int g,
                 cudaStream_t st) {
    launch_pdl(k_gather_rows<T>, g, 256, 0, st, static_cast<const T*>(x), c, idx, tiles,
                                        static_cast<T*>(buf));
}

}  // namespace

void conv_forward_prepare(sk_ctx* ctx, sk_kmap* m, const sk_dataflow_cfg& cfg, sk_dtype dt,
                          int c_in, int c_out, cudaStream_t st) {
    if (m->n_out == 0 || m->graph) return;
    // mirrors conv_forward's (dgrad = false) dispatch below
    if (cfg.kind == SK_IMPLICIT_GEMM && dt != SK_F32 && m->kd <= 27 &&
        ((c_in == 4 && c_out % 16 == 0) || (c_out == 32 && (c_in == 3 || c_in == 1))))
        return;  // the small-C_in paths (im2col + dense GEMM, CUDA cores) read the raw OS map
    int k_eff = c_in;
    if (dt != SK_F32 && c_in % 8 != 0 && c_out % 16 == 0) k_eff = (c_in + 7) / 8 * 8;
    if (m->identity && tc_ok(dt, k_eff, c_out) && !ctx->deterministic) return;  // dense GEMM
    if (cfg.kind == SK_IMPLICIT_GEMM) kmap_prepare(m, cfg.splits, kTileM, st);
    else kmap_ensure_ws(m, st);
}

// Forward (dgrad = false) or dgrad (dgrad = true; m_fwd is the FORWARD map).
void conv_forward(sk_ctx* ctx, sk_kmap* m_fwd, const sk_dataflow_cfg& cfg, sk_dtype dt, int c_in,
                  int c_out, const void* x, const void* w, void* y, bool dgrad, cudaStream_t st,
                  const void* w_kmajor, const void* residual, float* y_accum) {
    validate(c_in >= 1 && c_out >= 1, "channel counts must be >= 1");
    validate(cfg.splits >= 0, "splits must be >= 0");
    validate(cfg.kind >= 0 && cfg.kind <= 2, "unknown dataflow kind");
    contract(!(m_fwd->graph && cfg.kind == SK_IMPLICIT_GEMM),
             "graph maps run through the pair-list dataflows (GGS / FOD) only");
    sk_kmap* m = dgrad ? kmap_transpose(m_fwd, st) : m_fwd;
    // GEMM shape: A rows carry k_total channels, the output n_total
    const int k_total = dgrad ? c_out : c_in;
    const int n_total = dgrad ? c_in : c_out;
    const size_t es = elem_size(dt);
    const long long y_elems = (long long)m->n_out * n_total;
    if (m->n_out == 0) return;
    if (cfg.kind == SK_IMPLICIT_GEMM && !dgrad && dt != SK_F32 && !residual && !y_accum &&
        !ctx->deterministic && m->kd <= 27) {
        // tiny C_in (the 4-channel stem): neighbour gather + one dense tcgen05 GEMM
        const bool done = dt == SK_F16
                              ? conv_small_cin_dense<__half>(ctx, dt, m, c_in, c_out, x, w, y,
                                                             cfg.tile.cta_n, st)
                              : conv_small_cin_dense<__nv_bfloat16>(ctx, dt, m, c_in, c_out, x, w,
                                                                    y, cfg.tile.cta_n, st);
        if (done) return;
    }
    if (cfg.kind == SK_IMPLICIT_GEMM && !dgrad && dt != SK_F32) {
        // tiny C_in (the 4-channel stem): implicit GEMM on CUDA cores, raw OS map
        const bool done = dt == SK_F16
                              ? conv_small_cin<__half>(m, c_in, c_out, x, w, y, residual, y_accum, st)
                              : conv_small_cin<__nv_bfloat16>(m, c_in, c_out, x, w, y, residual,
                                                              y_accum, st);
        if (done) return;
    }

    // B operand [kd][n_total][k_total] (K-major): forward -> W^T per offset;
    // dgrad -> W itself with mirrored offsets (WeightTensor::transposed,
    // exec.cpp:32-43)
    DevBuf wt;
    const void* b = w;
    if (!dgrad && w_kmajor) {
        b = w_kmajor;  // caller keeps W^T [kd][c_out][c_in] (inference weights)
    } else if (!dgrad) {
        wt.alloc((size_t)m->kd * c_in * c_out * es, st);
        long long tot = (long long)m->kd * c_in * c_out;
        const int g = (int)ceil_div(tot, 256);
        if (dt == SK_F32) launch_pdl(k_transpose_w<float>, g, 256, 0, st, (const float*)w, m->kd, c_in, c_out, wt.as<float>());
        else if (dt == SK_F16) launch_pdl(k_transpose_w<__half>, g, 256, 0, st, (const __half*)w, m->kd, c_in, c_out, wt.as<__half>());
        else launch_pdl(k_transpose_w<__nv_bfloat16>, g, 256, 0, st, (const __nv_bfloat16*)w, m->kd, c_in, c_out, wt.as<__nv_bfloat16>());
        b = wt.p;
    }
    // tensor cores need 16 B operand rows: zero-pad C % 8 != 0 channel dims
    // (the 4-channel stem) instead of taking the SIMT path
    DevBuf xpad, bpad;
    int k_eff = k_total;
    if (dt != SK_F32 && k_total % 8 != 0 && n_total % 16 == 0) {
        k_eff = (k_total + 7) / 8 * 8;
        xpad.alloc((size_t)std::max(m->n_in, 1) * k_eff * es, st);
        bpad.alloc((size_t)m->kd * n_total * k_eff * es, st);
        if (dt == SK_F16) {
            pad_cols<__half>(x, m->n_in, k_total, k_eff, xpad.p, st);
            pad_cols<__half>(b, (long long)m->kd * n_total, k_total, k_eff, bpad.p, st);
        } else {
            pad_cols<__nv_bfloat16>(x, m->n_in, k_total, k_eff, xpad.p, st);
            pad_cols<__nv_bfloat16>(b, (long long)m->kd * n_total, k_total, k_eff, bpad.p, st);
        }
        x = xpad.p;
        b = bpad.p;
    }
    const bool tc = tc_ok(dt, k_eff, n_total);
    ConvArgs a = base_args();
    a.kd = m->kd;
    a.a = x;
    a.k_total = k_eff;
    a.n_rows_a = m->n_in;
    a.b = b;
    a.n_total = n_total;
    a.mirror = dgrad ? 1 : 0;
    a.ld_y = n_total;
    pick_n_tiling(n_total, cfg.tile.cta_n, tc, a.bn, a.n_ntiles);
    a.cta_m = cfg.tile.cta_m;
    a.cta_k = cfg.tile.cta_k;
    a.single = cfg.tile.cta_m == 64 ? 1 : 0;
    a.tma_gather = cfg.tile.load_width == 1 ? 1 : 0;
    const bool det = ctx->deterministic;

    if (m->identity && tc && !det &&
        dense_identity_tc(ctx, dt, m->n_out, k_eff, n_total, x, b, y, residual, y_accum,
                          cfg.tile.cta_n, st))
        return;  // plain dense GEMM (dense.cu: k_dense_tc)
    if (m->identity && tc && !det) {
        // K=1 stride-1 layer on one coordinate set: y = x W_0 for every
        // dataflow (the map is the identity), so run it as a dense GEMM
        a.mode = 2;
        a.n_rows_valid = m->n_out;
        a.items = (int)ceil_div(m->n_out, kItemM) * a.n_ntiles;
        a.y = y_accum ? (void*)y_accum : y;
        a.residual = y_accum ? nullptr : residual;
        a.out_mode = y_accum ? 3 : 0;
        launch_gconv(ctx, dt, a, st);
        return;
    }
    if (cfg.kind == SK_IMPLICIT_GEMM) {
        Prepared* pr = kmap_prepare(m, cfg.splits, kTileM, st);
        a.mode = 0;
        a.entries = pr->entries.as<int>();
        a.out_row = pr->out_row.as<int>();
        a.tile_masks = pr->tile_masks.as<unsigned long long>();
        a.split_begin = pr->d_begin.as<int>();
        a.ns = pr->num_splits;
        a.rows_pad = pr->rows_pad;
        a.n_tiles = pr->rows_pad / kTileM;
        a.n_rows_valid = m->n_out;
        // work items: 256 rows (two MMA tiles), or one 128-row tile (cta_m 64)
        const int pairs = a.single ? a.n_tiles : (a.n_tiles + 1) / 2;
        if (pr->num_splits == 1) {
            a.items = pairs * a.n_ntiles;
            a.y = y_accum ? (void*)y_accum : y;
            a.residual = y_accum ? nullptr : residual;
            a.out_mode = y_accum ? 3 : (dt == SK_F32 ? 1 : 0);
            launch_gconv(ctx, dt, a, st);
        } else {
            DevBuf acc;
            float* yf = y_accum ? y_accum : (dt == SK_F32 ? static_cast<float*>(y) : nullptr);
            if (!yf) {
                acc.alloc((size_t)y_elems * 4, st);
                yf = acc.as<float>();
            }
            if (!y_accum) fill_async(yf, 0, (size_t)y_elems * 4, st);
            a.y = yf;
            if (det) {
                // splits accumulate in order so partial sums telescope
                // (implicit_gemm_impl deterministic branch, exec.cpp:240-246)
                a.out_mode = 3;
                a.items = pairs * a.n_ntiles;
                for (int s = 0; s < pr->num_splits; ++s) {
                    a.split_only = s;
                    launch_gconv(ctx, dt, a, st);
                }
            } else {
                a.out_mode = 2;
                a.items = pr->num_splits * pairs * a.n_ntiles;
                launch_gconv(ctx, dt, a, st);
            }
            if (!y_accum && (dt != SK_F32 || residual))
                convert_from_f32(dt, yf, y_elems, y, residual, st);
        }
        return;
    }

    // WS-based dataflows over the per-offset, 128-padded pair lists
    kmap_ensure_ws(m, st);
    DevBuf acc;
    float* yf = y_accum ? y_accum : (dt == SK_F32 ? static_cast<float*>(y) : nullptr);
    if (!yf) {
        acc.alloc((size_t)y_elems * 4, st);
        yf = acc.as<float>();
    }
    if (!y_accum) fill_async(yf, 0, (size_t)y_elems * 4, st);
    a.mode = 1;
    a.ws_tile_ptr = m->ws_tile_ptr.as<int>();
    a.in_pad = m->ws_in_pad.as<int>();
    a.out_pad = m->ws_out_pad.as<int>();
    const int* tile_ptr = m->ws_tile_ptr.as<int>();

    if (cfg.kind == SK_FETCH_ON_DEMAND) {
        a.y = yf;
        if (det) {
            a.out_mode = 3;
            for (int k = 0; k < m->kd; ++k) {
                a.offset_only = k;
                launch_gconv(ctx, dt, a, st);
            }
        } else {
            a.out_mode = 2;
            launch_gconv(ctx, dt, a, st);
        }
    } else {
        // gather -> GEMM -> scatter-add (exec.cpp:117-158)
        const int64_t P = kmap_total_pairs(m, st);
        if (P > 0) {
            const long long rows_pad = P + (long long)m->kd * kItemM;  // >= tiles*256
            DevBuf ga, gc;
            ga.alloc((size_t)rows_pad * a.k_total * es, st);
            gc.alloc((size_t)rows_pad * n_total * 4, st);
            const int g = ctx->num_sms * 8;
            const int kk = a.k_total;  // padded width when the channels were padded
            if (dt == SK_F32) gather_rows<float>(x, kk, a.in_pad, tile_ptr + m->kd, ga.p, g, st);
            else if (dt == SK_F16) gather_rows<__half>(x, kk, a.in_pad, tile_ptr + m->kd, ga.p, g, st);
            else gather_rows<__nv_bfloat16>(x, kk, a.in_pad, tile_ptr + m->kd, ga.p, g, st);
            a.a = ga.p;
            a.n_rows_a = (int)rows_pad;
            a.a_identity = 1;
            a.out_identity = 1;
            a.y = gc.p;
            a.out_mode = 1;
            launch_gconv(ctx, dt, a, st);
            if (det) {
                for (int k = 0; k < m->kd; ++k) {
                    launch_pdl(k_scatter_add, g, 256, 0, st, gc.as<float>(), n_total, a.out_pad,
                                                     tile_ptr + k, tile_ptr + k + 1, yf, 1);
                }
            } else {
                launch_pdl(k_scatter_add, g, 256, 0, st, gc.as<float>(), n_total, a.out_pad, tile_ptr,
                                                 tile_ptr + m->kd, yf, 0);
            }
        }
    }
    if (!y_accum && (dt != SK_F32 || residual)) convert_from_f32(dt, yf, y_elems, y, residual, st);
}

void transpose_weights(sk_dtype dt, const void* w, int kd, int c_in, int c_out, void* wt,
                       cudaStream_t st) {
    const long long tot = (long long)kd * c_in * c_out;
    if (tot == 0) return;
    const int g = (int)ceil_div(tot, 256);
    if (dt == SK_F32) launch_pdl(k_transpose_w<float>, g, 256, 0, st, (const float*)w, kd, c_in, c_out, (float*)wt);
    else if (dt == SK_F16) launch_pdl(k_transpose_w<__half>, g, 256, 0, st, (const __half*)w, kd, c_in, c_out, (__half*)wt);
    else launch_pdl(k_transpose_w<__nv_bfloat16>, g, 256, 0, st, (const __nv_bfloat16*)w, kd, c_in, c_out, (__nv_bfloat16*)wt);
}

void conv_wgrad(sk_ctx* ctx, sk_kmap* m, const sk_dataflow_cfg& cfg, sk_dtype dt, int c_in,
                int c_out, const void* x, const void* dy, float* dw, cudaStream_t st,
                bool accumulate) {
    (void)cfg;  // conv_wgrad ignores cfg.kind in the reference (exec.cpp:398-414)
    validate(c_in >= 1 && c_out >= 1, "channel counts must be >= 1");
    kmap_ensure_ws(m, st);
    if (!accumulate) fill_async(dw, 0, (size_t)m->kd * c_in * c_out * 4, st);
    if (m->n_out == 0 || m->n_in == 0) return;
    if (dt != SK_F32 && !ctx->deterministic && c_in % 8 == 0 && c_out % 8 == 0) {
        // tcgen05 path (fp32 accumulate in TMEM, fp32 red.add flush)
        WgArgs a;
        a.x = x;
        a.dy = dy;
        a.c_in = c_in;
        a.c_out = c_out;
        a.kd = m->kd;
        a.tile_ptr = m->ws_tile_ptr.as<int>();
        a.in_pad = m->ws_in_pad.as<int>();
        a.out_pad = m->ws_out_pad.as<int>();
        a.dw = dw;
        a.m_tiles = (int)ceil_div(c_in, 128);
        a.n_tiles = (int)ceil_div(c_out, 256);  // 128-wide tiles + 2 CTAs/SM: C=256 421 -> 570 us
        a.bn = (int)ceil_div(ceil_div(c_out, a.n_tiles), 16) * 16;
        a.nblk_b = (int)ceil_div(a.bn, 64);
        const size_t stage_bytes = 16384 + (size_t)a.nblk_b * 8192;
        // two or three CTAs per SM (4 gather warps each, a share of the
        // stages) when their accumulator pairs fit in TMEM: the gathers are
        // latency-bound and more pipelines per SM overlap them (lidar scan,
        // tools/wgrad_time.py: C=32 88 -> 61 us, C=64 110 -> 89, C=96 136 ->
        // 126, C=128 165 -> 159)
        const int per_sm = (2 * a.bn <= 128) ? 3 : (2 * a.bn <= 256 ? 2 : 1);
        const size_t budget = per_sm == 3 ? 66 * 1024 : (per_sm == 2 ? 100 * 1024 : 200 * 1024);
        const int stages = (int)std::max<size_t>(2, std::min<size_t>(8, budget / stage_bytes));
        const size_t smem = stages * stage_bytes + (2 * stages + 4) * 8 + 16;
        auto kern = dt == SK_F16 ? k_wgrad_tc<__half> : k_wgrad_tc<__nv_bfloat16>;
        ensure_smem(reinterpret_cast<const void*>(kern), smem);
        launch_pdl(kern, per_sm * ctx->num_sms, kWgThreads, smem, st, a, stages);
        return;
    }
    if (dt != SK_F32 && !ctx->deterministic && c_in <= 8 && !m->graph) {
        // tiny C_in (the stem): lane-per-output-channel kernel; conv maps hold
        // at most n_out pairs per offset
        const int chunk = 1024;
        const dim3 grid((unsigned)ceil_div(std::max(m->n_out, 1), chunk),
                        (unsigned)ceil_div(c_out, 32), (unsigned)m->kd);
        const long long* ptr = m->ws_ptr.as<long long>();
        auto launch = [&](auto tag, auto ci) {
            using T = decltype(tag);
            constexpr int CI = decltype(ci)::value;
            launch_pdl(k_wgrad_small_cin<T, CI>, grid, 256, 0, st, static_cast<const T*>(x), static_cast<const T*>(dy), c_out, ptr,
                m->ws_in.as<int>(), m->ws_out.as<int>(), chunk, dw);
        };
        auto by_ci = [&](auto tag) {
            switch (c_in) {
                case 1: launch(tag, std::integral_constant<int, 1>{}); break;
                case 2: launch(tag, std::integral_constant<int, 2>{}); break;
                case 3: launch(tag, std::integral_constant<int, 3>{}); break;
                case 4: launch(tag, std::integral_constant<int, 4>{}); break;
                case 5: launch(tag, std::integral_constant<int, 5>{}); break;
                case 6: launch(tag, std::integral_constant<int, 6>{}); break;
                case 7: launch(tag, std::integral_constant<int, 7>{}); break;
                default: launch(tag, std::integral_constant<int, 8>{}); break;
            }
        };
        if (dt == SK_F16) by_ci(__half{});
        else by_ci(__nv_bfloat16{});
        return;
    }
    // pair chunking: enough blocks to fill the machine; deterministic mode
    // uses one chunk per offset (no cross-block float atomics on one cell)
    // pairs per offset are bounded by n_out for conv maps (one per (out,
    // offset)); a graph relation can hold up to all E edges
    const int64_t per_off = m->graph ? std::max<int64_t>(m->total_pairs_host, 1) : m->n_out;
    const int chunk = ctx->deterministic ? (int)std::max<int64_t>(1, per_off) : 2048;
    const int chunks = (int)ceil_div(std::max<int64_t>(per_off, 1), chunk);
    dim3 grid(chunks, (unsigned)(ceil_div(c_in, 32) * ceil_div(c_out, 32)), m->kd);
    const long long* ptr = m->ws_ptr.as<long long>();
    const long long cells = (long long)m->kd * c_in * c_out;
    DevBuf dw64;
    dw64.alloc((size_t)cells * 8, st);
    fill_async(dw64.p, 0, (size_t)cells * 8, st);
    double* d64 = dw64.as<double>();
    if (dt == SK_F32)
        launch_pdl(k_wgrad_simt<float>, grid, 256, 0, st, (const float*)x, (const float*)dy, c_in, c_out,
                                                  ptr, m->ws_in.as<int>(), m->ws_out.as<int>(),
                                                  chunk, d64);
    else if (dt == SK_F16)
        launch_pdl(k_wgrad_simt<__half>, grid, 256, 0, st, (const __half*)x, (const __half*)dy, c_in,
                                                   c_out, ptr, m->ws_in.as<int>(),
                                                   m->ws_out.as<int>(), chunk, d64);
    else
        launch_pdl(k_wgrad_simt<__nv_bfloat16>, grid, 256, 0, st, (const __nv_bfloat16*)x, (const __nv_bfloat16*)dy, c_in, c_out, ptr,
            m->ws_in.as<int>(), m->ws_out.as<int>(), chunk, d64);
    launch_pdl(k_round_f64, (int)std::min<long long>(ceil_div(cells, 256), 148 * 16), 256, 0, st, d64, cells, dw, accumulate ? 1 : 0);
}

}  // namespace sk
