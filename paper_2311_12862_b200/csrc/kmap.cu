// sk200 kernel-map construction on sm_100a (hot path (1)).
//
// Data layout in HBM
//   coords      int4 [n]                         (Coord, tensor.hpp:15-20)
//   hash table  16 B slots {u64 key, u32 row, pad} [cap], cap = pow2 >= 2n,
//               linear probing; one 16 B load resolves a probe (key + row)
//   OS map      i32 [rows_pad][KD], -1 sentinel   (KernelMapOS, kmap.hpp:65-93)
//   masks       u64 [rows_pad][words]             (compute_masks, kmap.cpp:34-47)
//   WS lists    CSR over offsets: ptr[KD+1], in[P], out[P], ascending out row
//               per offset (KernelMapWS, kmap.hpp:40-56)
//   prepared    per split s: entries [rows_pad][w_s], out_row [rows_pad],
//               masks [rows_pad][words_s], tile OR-masks [n_tiles][2]
//
// Kernels (one thread per output row unless noted; 128-row blocks match the
// 128-row MMA tiles of the dataflows):
//   k_hash_insert      CoordLookup build (tensor.cpp:80-85): CAS insert,
//                      atomicMin keeps the FIRST row of a duplicate key
//   k_down_insert/...  build_out_coords (kmap.cpp:73-94): floor_div keys,
//                      first-appearance dedup via atomicMin + flag + scan
//   k_kmap_query       build_kmap_ws + ws_to_os + compute_masks
//                      (kmap.cpp:96-183) fused: 8 probes in flight per thread,
//                      tile staged in smem, coalesced OS/mask stores, per
//                      block per offset pair counts for the WS compaction
//   k_ws_*             os_to_ws (kmap.cpp:185-209) as a stable per-offset
//                      stream compaction (ballot + block scan)
//   k_transpose        transpose_map (kmap.cpp:290-315) as a scatter
//   k_split_keys/...   split_and_sort + pad_map (kmap.cpp:211-288): split-local
//                      masks -> stable radix sort on (split, ~mask) -> reorder
#include <cstdlib>

#include "sk_internal.hpp"

namespace sk {

namespace {

constexpr int kQB = 128;  // rows per query block

__device__ __forceinline__ void offset_of(int k, int K, int dims, int& a, int& b, int& c) {
    const int h = K / 2;
    if (dims == 3) {
        a = k / (K * K) - h;
        b = (k / K) % K - h;
        c = k % K - h;
    } else {
        a = k / K - h;
        b = k % K - h;
        c = 0;
    }
}

__device__ __forceinline__ unsigned long long* slot_key(ulonglong2* t, uint64_t s) {
    return &t[s].x;
}
__device__ __forceinline__ unsigned* slot_val(ulonglong2* t, uint64_t s) {
    return reinterpret_cast<unsigned*>(&t[s].y);  // low 32 bits (little endian)
}

__global__ void k_hash_insert(const int4* __restrict__ coords, int n,
                              ulonglong2* __restrict__ table, uint64_t mask,
                              int* __restrict__ err) {
    pdl_wait();
    pdl_trigger();
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int4 c = coords[i];
    if (!packable(c.x, c.y, c.z, c.w)) {  // root sets were range-checked at creation
        if (err) atomicOr(err, 1);
        return;
    }
    unsigned long long key = pack_key(c.x, c.y, c.z, c.w);
    uint64_t s = hash_slot(key, mask);
    for (;;) {
        unsigned long long prev = atomicCAS(slot_key(table, s), (unsigned long long)kEmpty, key);
        if (prev == (unsigned long long)kEmpty || prev == key) {
            atomicMin(slot_val(table, s), (unsigned)i);
            return;
        }
        s = (s + 1) & mask;
    }
}

__global__ void k_coords_check(const int4* __restrict__ coords, int n, int* __restrict__ err) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int4 c = coords[i];
    if (!packable(c.x, c.y, c.z, c.w)) atomicOr(err, 1);
}

__global__ void k_down_insert(const int4* __restrict__ coords, int n, int sx, int sy, int sz,
                              int dims, ulonglong2* __restrict__ table, uint64_t mask,
                              int* __restrict__ slot_out,
                              int4* __restrict__ q_out) {
    pdl_wait();
    pdl_trigger();
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int4 c = coords[i];
    int4 q = c;
    q.y = (int)floor_div(c.y, sx);
    q.z = (int)floor_div(c.z, sy);
    if (dims == 3) q.w = (int)floor_div(c.w, sz);
    q_out[i] = q;
    unsigned long long key = pack_key(q.x, q.y, q.z, q.w);
    uint64_t s = hash_slot(key, mask);
    for (;;) {
        unsigned long long prev = atomicCAS(slot_key(table, s), (unsigned long long)kEmpty, key);
        if (prev == (unsigned long long)kEmpty || prev == key) {
            atomicMin(slot_val(table, s), (unsigned)i);
            slot_out[i] = (int)s;
            return;
        }
        s = (s + 1) & mask;
    }
}

__global__ void k_down_flag(const int* __restrict__ slot, ulonglong2* __restrict__ table, int n,
                            int* __restrict__ flag) {
    pdl_wait();
    pdl_trigger();
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    flag[i] = *slot_val(table, slot[i]) == (unsigned)i ? 1 : 0;
}

__global__ void k_down_compact(const int* __restrict__ flag, const int* __restrict__ pos,
                               const int* __restrict__ slot, const int4* __restrict__ q, int n,
                               ulonglong2* __restrict__ table, int4* __restrict__ out) {
    pdl_wait();
    pdl_trigger();
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !flag[i]) return;
    int p = pos[i];
    out[p] = q[i];
    *slot_val(table, slot[i]) = (unsigned)p;  // the table now maps out-coordinate -> out row
}

// ---- 4x4x4 block index (stride-1 query path) ---------------------------------
constexpr int kBlkEmpty = 0x7FFFFFFF;

// Two passes, no cross-warp waiting. k_block_claim: one lane per distinct
// block key in the warp inserts it (CAS); the winner takes an id from the
// counter, publishes it in the slot and fills the block's 64 cells with
// kBlkEmpty. k_block_fill (next launch: every id is published) looks the id up
// and keeps the FIRST row per cell (atomicMin), like emplace.
__global__ void k_block_claim(const int4* __restrict__ coords, int n, ulonglong2* __restrict__ bt,
                              uint64_t mask, int* __restrict__ dense, int* __restrict__ count) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = i < n;
    const int4 c = live ? coords[i] : make_int4(0, 0, 0, 0);
    const unsigned long long key = live ? pack_key(c.x, c.y >> 2, c.z >> 2, c.w >> 2) : kEmpty;
    // neighbouring voxels mostly share a block: one CAS per distinct key
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const int lane = threadIdx.x & 31;
    bool win = false;
    uint64_t s = hash_slot(key, mask);
    if (live && lane == __ffs(peers) - 1) {
        for (;;) {
            // ~8 warps claim each block: an L2 read finds most keys already
            // there, so only the first claim pays the (same-address) CAS
            const unsigned long long seen = __ldcg(slot_key(bt, s));
            if (seen == key) break;
            if (seen != (unsigned long long)kEmpty) {
                s = (s + 1) & mask;
                continue;
            }
            const unsigned long long prev = atomicCAS(slot_key(bt, s), (unsigned long long)kEmpty, key);
            if (prev == (unsigned long long)kEmpty) {
                win = true;
                break;
            }
            if (prev == key) break;
            s = (s + 1) & mask;
        }
    }
    // ids: one counter add per CTA (per-warp adds serialised on the counter)
    __shared__ unsigned cta_cnt, cta_base;
    if (threadIdx.x == 0) cta_cnt = 0;
    __syncthreads();
    const unsigned wins = __ballot_sync(0xffffffffu, win);
    unsigned woff = 0;
    if (lane == 0 && wins) woff = atomicAdd(&cta_cnt, (unsigned)__popc(wins));
    woff = __shfl_sync(0xffffffffu, woff, 0);
    __syncthreads();
    if (threadIdx.x == 0 && cta_cnt) cta_base = (unsigned)atomicAdd(count, (int)cta_cnt);
    __syncthreads();
    if (!win) return;
    const unsigned base = cta_base + woff;
    const unsigned bid = base + __popc(wins & ((1u << lane) - 1));
    int4* d = reinterpret_cast<int4*>(dense + (size_t)bid * 64);
#pragma unroll
    for (int j = 0; j < 16; ++j) d[j] = make_int4(kBlkEmpty, kBlkEmpty, kBlkEmpty, kBlkEmpty);
    *slot_val(bt, s) = bid;
}

__device__ __forceinline__ int block_lookup(const ulonglong2* __restrict__ bt, uint64_t mask,
                                            unsigned long long key);

__global__ void k_block_fill(const int4* __restrict__ coords, int n, const ulonglong2* __restrict__ bt,
                             uint64_t mask, int* __restrict__ dense) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int4 c = coords[i];
    const int bid = block_lookup(bt, mask, pack_key(c.x, c.y >> 2, c.z >> 2, c.w >> 2));
    const int local = ((c.y & 3) << 4) | ((c.z & 3) << 2) | (c.w & 3);
    atomicMin(dense + (size_t)bid * 64 + local, i);
}

__device__ __forceinline__ int block_lookup(const ulonglong2* __restrict__ bt, uint64_t mask,
                                            unsigned long long key) {
    uint64_t s = hash_slot(key, mask);
    for (;;) {
        const ulonglong2 e = __ldg(&bt[s]);
        if (e.x == key) return (int)(unsigned)e.y;
        if (e.x == (unsigned long long)kEmpty) return -1;
        s = (s + 1) & mask;
    }
}

// Stride-1 (submanifold or generative) query over the input's block index:
// one thread per output row. Per axis the K neighbours span one or two
// blocks (lo, lo+1); the row's 2x2x2 neighbour-block ids are looked up once
// (only distinct ones probe the table). A block's cells are z-minor, so for
// each (x, y) offset the K z-neighbours are read as one or two aligned 16 B
// z-rows (K=3: 9-18 loads per row instead of 27 scattered 4 B loads; K=5: 50
// instead of 125). Same outputs as k_kmap_query: OS tile via smem, big-endian
// masks, per-block counts.
template <int K>
__global__ void __launch_bounds__(kQB) k_kmap_query_blk(
    const int4* __restrict__ out_coords, int n_out, const ulonglong2* __restrict__ bt,
    uint64_t mask, const int* __restrict__ dense, int words, int* __restrict__ os,
    unsigned long long* __restrict__ masks, int* __restrict__ blk_counts) {
    pdl_wait();
    pdl_trigger();
    constexpr int KD = K * K * K, H = K / 2;
    extern __shared__ int q_sh[];
    int* tile = q_sh;            // kQB x KD
    int* cnt = q_sh + kQB * KD;  // KD
    const int t = threadIdx.x;
    const int row = blockIdx.x * kQB + t;
    for (int k = t; k < KD; k += kQB) cnt[k] = 0;
    __syncthreads();
    unsigned long long m0 = 0, m1 = 0;
    // every lane runs the (unrolled) offset loop so the per-offset counts are
    // warp ballots, not 32-way contended shared atomics; rows past n_out see
    // no blocks
    const bool live = row < n_out;
    {
        const int4 q = live ? out_coords[row] : make_int4(0, 0, 0, 0);
        const int lx = q.y & 3, ly = q.z & 3, lz = q.w & 3;
        const int bx = q.y >> 2, by = q.z >> 2, bz = q.w >> 2;
        const int lox = (lx - H) >> 2, loy = (ly - H) >> 2, loz = (lz - H) >> 2;  // -1 or 0
        const int nx = ((lx + H) >> 2) - lox, ny = ((ly + H) >> 2) - loy, nz = ((lz + H) >> 2) - loz;
        // bid[ix][iy][iz]: block (lo+i) per axis, -1 = absent or not needed
        // (an axis whose neighbours stay in one block never selects i = 1)
        int bid[2][2][2];
#pragma unroll
        for (int ix = 0; ix < 2; ++ix)
#pragma unroll
            for (int iy = 0; iy < 2; ++iy)
#pragma unroll
                for (int iz = 0; iz < 2; ++iz) {
                    const int x = bx + lox + ix, y = by + loy + iy, z = bz + loz + iz;
                    bid[ix][iy][iz] = (live && ix <= nx && iy <= ny && iz <= nz && packable(q.x, x, y, z))
                                          ? block_lookup(bt, mask, pack_key(q.x, x, y, z)) : -1;
                }
        // the z window: concat(row at lo, row at lo+1)[zb + c], c = 0..K-1
        const int zb = lz - H - 4 * loz;  // 0..3
        const int4 kE = make_int4(kBlkEmpty, kBlkEmpty, kBlkEmpty, kBlkEmpty);
#pragma unroll
        for (int a = 0; a < K; ++a)
#pragma unroll
            for (int b = 0; b < K; ++b) {
                const int px = lx + a - H, py = ly + b - H;
                const int ix = (px >> 2) - lox, iy = (py >> 2) - loy;
                const int id0 = ix ? (iy ? bid[1][1][0] : bid[1][0][0]) : (iy ? bid[0][1][0] : bid[0][0][0]);
                const int id1 = ix ? (iy ? bid[1][1][1] : bid[1][0][1]) : (iy ? bid[0][1][1] : bid[0][0][1]);
                const int zrow = ((px & 3) << 4) | ((py & 3) << 2);
                const int4 r0 = id0 >= 0 ? __ldg(reinterpret_cast<const int4*>(dense + (size_t)id0 * 64 + zrow)) : kE;
                const int4 r1 = id1 >= 0 ? __ldg(reinterpret_cast<const int4*>(dense + (size_t)id1 * 64 + zrow)) : kE;
                const int w[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
                for (int c = 0; c < K; ++c) {
                    int v = w[c];
#pragma unroll
                    for (int s2 = 1; s2 < 4; ++s2)
                        if (zb == s2) v = w[s2 + c];
                    const int k = (a * K + b) * K + c;  // lexicographic
                    const int j = v == kBlkEmpty ? -1 : v;
                    tile[t * KD + k] = j;
                    const unsigned hit = __ballot_sync(0xffffffffu, j >= 0);
                    if ((t & 31) == 0 && hit) atomicAdd(&cnt[k], __popc(hit));
                    if (j >= 0) {
                        if (k < 64) m0 |= 1ull << ((KD < 64 ? KD : 64) - 1 - k);
                        else m1 |= 1ull << (KD - 64 - 1 - (k - 64));
                    }
                }
            }
    }
    __syncthreads();
    int* dst = os + (size_t)blockIdx.x * kQB * KD;
    for (int i = t; i < kQB * KD; i += kQB) __stcs(dst + i, tile[i]);
    __stcs(masks + (size_t)row * words, m0);
    if (words == 2) __stcs(masks + (size_t)row * words + 1, m1);
    for (int k = t; k < KD; k += kQB) blk_counts[(size_t)blockIdx.x * KD + k] = cnt[k];
}


// ---- quantize (tensor.cpp:87-142): floor(raw / voxel) + first-appearance dedup
// err bit 1: non-finite coordinate, bit 2: outside the packable range
__global__ void k_quant_insert(const double* __restrict__ raw, const int* __restrict__ batch,
                               int m, int dims, double vx, double vy, double vz,
                               ulonglong2* __restrict__ table, uint64_t mask,
                               int* __restrict__ slot_out, int4* __restrict__ q_out,
                               int* __restrict__ err) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const double v[3] = {vx, vy, vz};
    long long c[3] = {0, 0, 0};
    bool finite = true;
    for (int d = 0; d < dims; ++d) {
        const double r = raw[(size_t)i * dims + d];
        finite &= isfinite(r);
        c[d] = finite ? (long long)floor(r / v[d]) : 0;
    }
    const int b = batch ? batch[i] : 0;
    if (!finite) {
        atomicOr(err, 1);
        slot_out[i] = -1;
        return;
    }
    if (!packable(b, (int)max(min(c[0], (long long)INT_MAX), (long long)INT_MIN),
                  (int)max(min(c[1], (long long)INT_MAX), (long long)INT_MIN),
                  (int)max(min(c[2], (long long)INT_MAX), (long long)INT_MIN)) ||
        c[0] != (int)c[0] || c[1] != (int)c[1] || c[2] != (int)c[2]) {
        atomicOr(err, 2);
        slot_out[i] = -1;
        return;
    }
    const int4 q = make_int4(b, (int)c[0], (int)c[1], (int)c[2]);
    q_out[i] = q;
    const unsigned long long key = pack_key(q.x, q.y, q.z, q.w);
    uint64_t s = hash_slot(key, mask);
    for (;;) {
        const unsigned long long prev = atomicCAS(slot_key(table, s), (unsigned long long)kEmpty, key);
        if (prev == (unsigned long long)kEmpty || prev == key) {
            atomicMin(slot_val(table, s), (unsigned)i);
            slot_out[i] = (int)s;
            return;
        }
        s = (s + 1) & mask;
    }
}

// point -> output row (after compaction the table maps key -> out row)
__global__ void k_point_rows(const int* __restrict__ slot, const ulonglong2* __restrict__ table,
                             int m, int* __restrict__ rows) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    rows[i] = (int)*slot_val(const_cast<ulonglong2*>(table), slot[i]);
}

// DedupRule::first: the first point of each row (min point index)
__global__ void k_first_point(const int* __restrict__ rows, int m, int* __restrict__ first) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) atomicMin(first + rows[i], i);
}

template <typename T>
__global__ void k_quant_feats_first(const double* __restrict__ feats, int channels,
                                    const int* __restrict__ first, int n, T* __restrict__ out) {
    pdl_wait();
    pdl_trigger();
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)n * channels) return;
    const int r = (int)(t / channels), c = (int)(t % channels);
    out[t] = (T)feats[(size_t)first[r] * channels + c];
}

// DedupRule::mean: f64 sums and counts (the reference's running mean is the
// same mean up to f64 rounding)
__global__ void k_quant_sum(const double* __restrict__ feats, int channels,
                            const int* __restrict__ rows, int m, double* __restrict__ sum,
                            int* __restrict__ count) {
    pdl_wait();
    pdl_trigger();
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)m * channels) return;
    const int i = (int)(t / channels), c = (int)(t % channels);
    atomicAdd(sum + (size_t)rows[i] * channels + c, feats[t]);
    if (c == 0) atomicAdd(count + rows[i], 1);
}

template <typename T>
__global__ void k_quant_mean(const double* __restrict__ sum, const int* __restrict__ count,
                             int channels, int n, T* __restrict__ out) {
    pdl_wait();
    pdl_trigger();
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)n * channels) return;
    out[t] = (T)(sum[t] / (double)count[t / channels]);
}

template <typename T>
__global__ void k_fill(T* __restrict__ out, long long n, double v) {
    pdl_wait();
    pdl_trigger();
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) out[t] = (T)v;
}


// ---- graph maps (kmap_from_edges, kmap.cpp:317-336) -----------------------------
__global__ void k_edge_keys(const int* __restrict__ edges, int E, int R, int n_in, int n_out,
                            unsigned long long* __restrict__ keys, int* __restrict__ vals,
                            int* __restrict__ counts, int* __restrict__ err) {
    pdl_wait();
    pdl_trigger();
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    const int src = edges[3 * e], dst = edges[3 * e + 1], rel = edges[3 * e + 2];
    if (rel < 0 || rel >= R) atomicOr(err, 1);
    if (src < 0 || src >= n_in || dst < 0 || dst >= n_out) atomicOr(err, 2);
    const int r = min(max(rel, 0), R - 1);
    keys[e] = ((unsigned long long)r << 32) | (unsigned)max(dst, 0);
    vals[e] = e;
    atomicAdd(counts + r, 1);
}

// exclusive scans of the per-relation counts (pairs and 256-pair tiles); one thread
__global__ void k_edge_scan(const int* __restrict__ counts, int R, long long* __restrict__ ptr,
                            int* __restrict__ tile_ptr) {
    pdl_wait();
    pdl_trigger();
    long long acc = 0;
    int tiles = 0;
    for (int r = 0; r < R; ++r) {
        ptr[r] = acc;
        tile_ptr[r] = tiles;
        acc += counts[r];
        tiles += (counts[r] + kTileWS - 1) / kTileWS;
    }
    ptr[R] = acc;
    tile_ptr[R] = tiles;
}

__global__ void k_edge_scatter(const int* __restrict__ edges, const unsigned long long* __restrict__ keys,
                               const int* __restrict__ order, int E, const long long* __restrict__ ptr,
                               const int* __restrict__ tile_ptr, int* __restrict__ ws_in,
                               int* __restrict__ ws_out, int* __restrict__ in_pad,
                               int* __restrict__ out_pad) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= E) return;
    const int e = order[i];
    const int rel = (int)(keys[i] >> 32);
    const long long j = i - ptr[rel];
    ws_in[i] = edges[3 * e];
    ws_out[i] = edges[3 * e + 1];
    const long long pp = (long long)tile_ptr[rel] * kTileWS + j;
    in_pad[pp] = edges[3 * e];
    out_pad[pp] = edges[3 * e + 1];
}


// resolve a probe whose first slot (key + row) is already loaded
__device__ __forceinline__ int probe(const ulonglong2* __restrict__ table, uint64_t mask,
                                     unsigned long long key, uint64_t s, ulonglong2 first) {
    ulonglong2 e = first;
    for (;;) {
        if (e.x == key) return (int)(unsigned)e.y;
        if (e.x == (unsigned long long)kEmpty) return -1;
        // two slots per iteration (usually the same 32 B sector)
        const uint64_t s1 = (s + 1) & mask, s2 = (s + 2) & mask;
        const ulonglong2 e1 = __ldg(&table[s1]);
        const ulonglong2 e2 = __ldg(&table[s2]);
        if (e1.x == key) return (int)(unsigned)e1.y;
        if (e1.x == (unsigned long long)kEmpty) return -1;
        s = s2;
        e = e2;
    }
}

// ---- generalized offsets: per-axis kernel sizes (odd or
// even) and dilation; offsets come from a device table (lexicographic). One
// thread per (row, offset subset); same outputs as k_kmap_query.
template <int TPR>
__global__ void __launch_bounds__(kQB * TPR) k_kmap_query_gen(
    const int4* __restrict__ out_coords, int n_out, const ulonglong2* __restrict__ table,
    uint64_t mask, const int4* __restrict__ offs, int KD, int dims, int sx, int sy, int sz,
    int transposed, int words, int* __restrict__ os, unsigned long long* __restrict__ masks,
    int* __restrict__ blk_counts) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ int q_sh[];
    int* tile = q_sh;                                       // kQB x KD
    int* cnt = q_sh + kQB * KD;                             // KD
    int4* soff = reinterpret_cast<int4*>(cnt + ((KD + 3) & ~3));  // KD
    const int t = threadIdx.x;
    const int rl = t / TPR, sub = t % TPR;
    const int row = blockIdx.x * kQB + rl;
    for (int k = t; k < KD; k += kQB * TPR) {
        cnt[k] = 0;
        soff[k] = offs[k];
    }
    __syncthreads();
    const bool live = row < n_out;
    const int4 q = live ? out_coords[row] : make_int4(0, 0, 0, 0);
    unsigned long long m0 = 0, m1 = 0;
    for (int k = sub; k < KD; k += TPR) {
        int j = -1;
        if (live) {
            const int4 o = soff[k];
            int px, py, pz;
            bool ok = true;
            if (!transposed) {
                px = q.y * sx + o.x;
                py = q.z * sy + o.y;
                pz = q.w * sz + o.z;
            } else {
                const int nx = q.y + o.x, ny = q.z + o.y, nz = q.w + o.z;
                ok = nx % sx == 0 && ny % sy == 0 && (dims != 3 || nz % sz == 0);
                px = nx / sx;
                py = ny / sy;
                pz = dims == 3 ? nz / sz : 0;
            }
            if (ok && packable(q.x, px, py, pz)) {
                const unsigned long long key = pack_key(q.x, px, py, pz);
                const uint64_t s0 = hash_slot(key, mask);
                j = probe(table, mask, key, s0, __ldg(&table[s0]));
            }
        }
        tile[rl * KD + k] = j;
        if (j >= 0) {
            atomicAdd(&cnt[k], 1);
            if (k < 64) m0 |= 1ull << ((KD < 64 ? KD : 64) - 1 - k);
            else m1 |= 1ull << (KD - 64 - 1 - (k - 64));
        }
    }
#pragma unroll
    for (int o = TPR / 2; o >= 1; o >>= 1) {
        m0 |= __shfl_xor_sync(0xffffffffu, m0, o);
        m1 |= __shfl_xor_sync(0xffffffffu, m1, o);
    }
    __syncthreads();
    int* dst = os + (size_t)blockIdx.x * kQB * KD;
    for (int i = t; i < kQB * KD; i += kQB * TPR) __stcs(dst + i, tile[i]);
    if (sub == 0) {
        __stcs(masks + (size_t)row * words, m0);
        if (words == 2) __stcs(masks + (size_t)row * words + 1, m1);
    }
    for (int k = t; k < KD; k += kQB * TPR) blk_counts[(size_t)blockIdx.x * KD + k] = cnt[k];
}

// TPR threads per output row (offsets k = sub, sub+TPR, ...; up to
// ceil(KD/TPR) independent probes in flight per thread), 128 rows per block.
// Writes the OS entries + masks of the block (pad rows get -1 / 0) and the
// block's per-offset pair counts.
template <int KD>
struct KShape {  // K and D implied by K^D (1, 9, 25, 27, 125)
    static constexpr int dims = (KD == 27 || KD == 125) ? 3 : 2;
    static constexpr int K = KD == 1 ? 1 : (KD == 9 || KD == 27) ? 3 : 5;
};

template <int KD, int TPR>
__global__ void __launch_bounds__(kQB * TPR) k_kmap_query(
    const int4* __restrict__ out_coords, int n_out, const ulonglong2* __restrict__ table,
    uint64_t mask, int K, int dims, int sx, int sy, int sz,
    int transposed, int words, int* __restrict__ os, unsigned long long* __restrict__ masks,
    int* __restrict__ blk_counts) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ int q_sh[];
    int* tile = q_sh;            // kQB x KD
    int* cnt = q_sh + kQB * KD;  // KD
    constexpr int PER = (KD + TPR - 1) / TPR;
    const int t = threadIdx.x;
    const int rl = t / TPR, sub = t % TPR;
    const int row = blockIdx.x * kQB + rl;
    for (int k = t; k < KD; k += kQB * TPR) cnt[k] = 0;
    __syncthreads();
    const bool live = row < n_out;
    const int4 q = live ? out_coords[row] : make_int4(0, 0, 0, 0);
    unsigned long long key[PER];
    ulonglong2 first[PER];
    uint64_t slot[PER];
    bool ok[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int k = sub + u * TPR;
        ok[u] = live && k < KD;
        if (!ok[u]) continue;
        // lexicographic offset (kmap.cpp:58-71) with compile-time K (no divides)
        constexpr int KK = KShape<KD>::K, H = KK / 2;
        int a, b, c;
        if (KShape<KD>::dims == 3) {
            a = k / (KK * KK) - H;
            b = (k / KK) % KK - H;
            c = k % KK - H;
        } else {
            a = k / KK - H;
            b = k % KK - H;
            c = 0;
        }
        int px, py, pz;
        if (!transposed) {
            px = q.y * sx + a;
            py = q.z * sy + b;
            pz = q.w * sz + c;
        } else {
            // q_in = (p_out + delta) / s only when every axis divides
            // (C++ truncating %, kmap.cpp:124-129)
            const int nx = q.y + a, ny = q.z + b, nz = q.w + c;
            if (nx % sx != 0 || ny % sy != 0 || (dims == 3 && nz % sz != 0)) {
                ok[u] = false;
                continue;
            }
            px = nx / sx;
            py = ny / sy;
            pz = dims == 3 ? nz / sz : 0;
        }
        if (!packable(q.x, px, py, pz)) {
            ok[u] = false;
            continue;
        }
        key[u] = pack_key(q.x, px, py, pz);
        slot[u] = hash_slot(key[u], mask);
        first[u] = __ldg(&table[slot[u]]);  // PER independent 16 B loads in flight
    }
    unsigned long long m0 = 0, m1 = 0;
    // lanes sub, sub + TPR, ... of a warp share offset k: one ballot per u and
    // one shared add per (warp, k) instead of TPR-strided contended atomics
    constexpr unsigned kSubLanes = TPR == 1 ? 0xffffffffu : TPR == 2 ? 0x55555555u
                                   : TPR == 4 ? 0x11111111u : 0x01010101u;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int k = sub + u * TPR;
        const int j = (k < KD && ok[u]) ? probe(table, mask, key[u], slot[u], first[u]) : -1;
        if (k < KD) tile[rl * KD + k] = j;
        const unsigned hit = __ballot_sync(0xffffffffu, j >= 0);
        const int lane = t & 31;
        if (lane < TPR && k < KD) {
            const int c = __popc(hit & (kSubLanes << lane));
            if (c) atomicAdd(&cnt[k], c);
        }
        if (j >= 0) {
            // big-endian bit order (kmap.cpp:38-45)
            if (k < 64) m0 |= 1ull << ((KD < 64 ? KD : 64) - 1 - k);
            else m1 |= 1ull << (KD - 64 - 1 - (k - 64));
        }
    }
#pragma unroll
    for (int o = TPR / 2; o >= 1; o >>= 1) {
        m0 |= __shfl_xor_sync(0xffffffffu, m0, o);
        m1 |= __shfl_xor_sync(0xffffffffu, m1, o);
    }
    __syncthreads();
    // streaming (evict-first) stores: the OS matrix is the bulk of the traffic
    // and must not push the hash table out of L2 while other blocks probe it
    int* dst = os + (size_t)blockIdx.x * kQB * KD;
    for (int i = t; i < kQB * KD; i += kQB * TPR) __stcs(dst + i, tile[i]);
    if (sub == 0) {
        __stcs(masks + (size_t)row * words, m0);
        if (words == 2) __stcs(masks + (size_t)row * words + 1, m1);
    }
    for (int k = t; k < KD; k += kQB * TPR) blk_counts[(size_t)blockIdx.x * KD + k] = cnt[k];
}

// masks + per-block counts from an existing OS matrix (transposed maps).
__global__ void __launch_bounds__(kQB) k_finalize(const int* __restrict__ os, int kd, int words,
                                                  unsigned long long* __restrict__ masks,
                                                  int* __restrict__ blk_counts) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ int sh[];
    int* tile = sh;
    int* cnt = sh + kQB * kd;
    const int t = threadIdx.x;
    const int row = blockIdx.x * kQB + t;
    for (int k = t; k < kd; k += kQB) cnt[k] = 0;
    const int* src = os + (size_t)blockIdx.x * kQB * kd;
    for (int i = t; i < kQB * kd; i += kQB) tile[i] = src[i];
    __syncthreads();
    unsigned long long m0 = 0, m1 = 0;
    for (int k = 0; k < kd; ++k) {
        int j = tile[t * kd + k];
        unsigned hit = __ballot_sync(0xffffffffu, j >= 0);
        if ((t & 31) == 0 && hit) atomicAdd(&cnt[k], __popc(hit));
        if (j >= 0) {
            if (k < 64) m0 |= 1ull << ((kd < 64 ? kd : 64) - 1 - k);
            else m1 |= 1ull << (kd - 64 - 1 - (k - 64));
        }
    }
    __syncthreads();
    masks[(size_t)row * words] = m0;
    if (words == 2) masks[(size_t)row * words + 1] = m1;
    for (int k = t; k < kd; k += kQB) blk_counts[(size_t)blockIdx.x * kd + k] = cnt[k];
}

// Per-offset exclusive scan over blocks (one warp per offset), then the CSR
// pointer over offsets and the FOD/GGS tile schedule (128 pairs per tile).
__global__ void __launch_bounds__(1024) k_ws_scan(const int* __restrict__ blk_counts,
                                                  int n_blocks, int kd,
                                                  long long* __restrict__ blk_off,
                                                  long long* __restrict__ ptr,
                                                  int* __restrict__ tile_ptr) {
    pdl_wait();
    pdl_trigger();
    __shared__ long long tot[128];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int k = warp; k < kd; k += 32) {
        long long run = 0;
        for (int b0 = 0; b0 < n_blocks; b0 += 32) {
            int b = b0 + lane;
            long long v = b < n_blocks ? blk_counts[(size_t)b * kd + k] : 0;
            long long inc = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                long long u = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += u;
            }
            if (b < n_blocks) blk_off[(size_t)b * kd + k] = run + inc - v;
            run += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) tot[k] = run;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long acc = 0;
        int tacc = 0;
        for (int k = 0; k < kd; ++k) {
            ptr[k] = acc;
            tile_ptr[k] = tacc;
            acc += tot[k];
            tacc += (int)((tot[k] + kTileWS - 1) / kTileWS);
        }
        ptr[kd] = acc;
        tile_ptr[kd] = tacc;
    }
}

__global__ void __launch_bounds__(kQB) k_ws_scatter(const int* __restrict__ os, int kd,
                                                    const long long* __restrict__ blk_off,
                                                    const long long* __restrict__ ptr,
                                                    const int* __restrict__ tile_ptr,
                                                    int* __restrict__ ws_in,
                                                    int* __restrict__ ws_out,
                                                    int* __restrict__ in_pad,
                                                    int* __restrict__ out_pad) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ int sh[];
    int* tile = sh;
    __shared__ int wcnt[kQB / 32];
    const int t = threadIdx.x, warp = t / 32, lane = t % 32;
    const int row = blockIdx.x * kQB + t;
    const int* src = os + (size_t)blockIdx.x * kQB * kd;
    for (int i = t; i < kQB * kd; i += kQB) tile[i] = src[i];
    __syncthreads();
    for (int k = 0; k < kd; ++k) {
        int j = tile[t * kd + k];
        unsigned hit = __ballot_sync(0xffffffffu, j >= 0);
        if (lane == 0) wcnt[warp] = __popc(hit);
        __syncthreads();
        int before = 0;
        for (int w = 0; w < warp; ++w) before += wcnt[w];
        if (j >= 0) {
            long long rel = blk_off[(size_t)blockIdx.x * kd + k] + before +
                            __popc(hit & ((1u << lane) - 1));
            long long pos = ptr[k] + rel;
            ws_in[pos] = j;
            ws_out[pos] = row;
            // per-offset lists padded to 256-pair tiles (-1 pads) for FOD/GGS tiles
            long long pp = (long long)tile_ptr[k] * kTileWS + rel;
            in_pad[pp] = j;
            out_pad[pp] = row;
        }
        __syncthreads();
    }
}

__global__ void k_transpose(const int* __restrict__ os, int n_out, int kd, int* __restrict__ ost) {
    pdl_wait();
    pdl_trigger();
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)n_out * kd) return;
    int q = (int)(i / kd), k = (int)(i % kd);
    int j = os[i];
    if (j >= 0) ost[(size_t)j * kd + (kd - 1 - k)] = q;
}

// Sort keys for split_and_sort: key = (split << W) | (~local_mask & wmask) so
// one stable ascending radix sort orders every split by DESCENDING mask,
// stable (std::stable_sort with mask_greater, kmap.cpp:252-256).
__global__ void k_split_keys(const int* __restrict__ os, int n, int kd, int ns,
                             const int* __restrict__ begin, int W, int word,
                             const int* __restrict__ perm, unsigned long long* __restrict__ keys,
                             int* __restrict__ vals) {
    pdl_wait();
    pdl_trigger();
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)n * ns) return;
    int s = (int)(i / n), r = (int)(i % n);
    if (perm) r = perm[i];
    int b = begin[s], e = begin[s + 1], w = e - b;
    // split-local mask words (word 0 most significant); `word` selects which
    // 64-bit word is the key for wide (w > 64) single-split maps
    unsigned long long m = 0;
    const int* row = os + (size_t)r * kd;
    int words = (w + 63) / 64;
    int wi_lo = word * 64, bits = min(64, w - wi_lo);
    for (int j = 0; j < bits; ++j)
        if (row[b + wi_lo + j] >= 0) m |= 1ull << (bits - 1 - j);
    unsigned long long wm = bits == 64 ? ~0ull : ((1ull << bits) - 1);
    unsigned long long key = (~m) & wm;
    if (words == 1 && ns > 1) key |= (unsigned long long)s << W;
    keys[i] = key;
    vals[i] = r;
}

constexpr int kMaxSplitDesc = 128;  // splits <= K^D <= 125
// split bounds for the prepare kernels, passed by value (no host->device copy)
struct SplitDesc {
    int ns, kd, W, n;
    int begin[kMaxSplitDesc + 1];
    int woff[kMaxSplitDesc + 1];
};

// k_split_keys32 + the radix sort's digit histograms for every pass (warp-
// aggregated smem counters, one global atomic per nonzero bin per block) +
// the split bounds on the device: one launch ahead of the sort passes
__global__ void __launch_bounds__(256) k_split_keygen32(
    const unsigned long long* __restrict__ masks, const SplitDesc sd, int dbits, int passes,
    unsigned* __restrict__ keys, int* __restrict__ vals, uint32_t* __restrict__ ghist,
    int* __restrict__ d_begin, int* __restrict__ d_woff) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ uint32_t hsh[];  // [passes][1 << dbits]
    const int D = 1 << dbits;
    for (int i = threadIdx.x; i < passes * D; i += blockDim.x) hsh[i] = 0;
    if (blockIdx.x == 0)
        for (int i = threadIdx.x; i <= sd.ns; i += blockDim.x) {
            d_begin[i] = sd.begin[i];
            d_woff[i] = sd.woff[i];
        }
    __syncthreads();
    const long long tot = (long long)sd.n * sd.ns;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long lim = (tot + stride - 1) / stride * stride;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < lim; i += stride) {
        unsigned key = 0;
        const bool ok = i < tot;
        if (ok) {
            const int s = (int)(i / sd.n), r = (int)(i % sd.n);
            const int b = sd.begin[s], e = sd.begin[s + 1], w = e - b;
            const unsigned long long m = masks[r];  // column j <-> bit kd-1-j
            const unsigned local = (unsigned)((m >> (sd.kd - e)) & ((1ull << w) - 1));
            key = ~local & ((1u << w) - 1);
            if (sd.ns > 1) key |= (unsigned)s << sd.W;
            keys[i] = key;
            vals[i] = r;
        }
        for (int p = 0; p < passes; ++p)
            hist_add(hsh + p * D, ok ? (int)((key >> (p * dbits)) & (unsigned)(D - 1)) : -1);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * D; i += blockDim.x)
        if (hsh[i]) atomicAdd(&ghist[i], hsh[i]);
}

__global__ void k_split_desc(const SplitDesc sd, int* __restrict__ d_begin, int* __restrict__ d_woff) {
    pdl_wait();
    pdl_trigger();
    for (int i = threadIdx.x; i <= sd.ns; i += blockDim.x) {
        d_begin[i] = sd.begin[i];
        d_woff[i] = sd.woff[i];
    }
}

__device__ void row_reorder(const int* __restrict__ os, int n, int kd, int rows_pad,
                            const int* __restrict__ begin, const int* __restrict__ word_off,
                            const int* __restrict__ order, int* __restrict__ entries,
                            int* __restrict__ out_row, unsigned long long* __restrict__ masks,
                            int s, int p, unsigned long long (&mm)[2]) {
    int b = begin[s], w = begin[s + 1] - b, words = (w + 63) / 64;
    // tile-column-major: [tile][column][128 rows] so one column of one tile is a
    // contiguous, 512B-aligned vector (one bulk copy feeds a 128-row gather)
    int* dst = entries + (size_t)rows_pad * b + ((size_t)(p / kTileM) * w) * kTileM + (p % kTileM);
    unsigned long long* md = masks + (size_t)rows_pad * word_off[s] + (size_t)p * words;
    if (p >= n) {
        for (int j = 0; j < w; ++j) dst[(size_t)j * kTileM] = -1;
        out_row[(size_t)s * rows_pad + p] = -1;
        for (int u = 0; u < words; ++u) md[u] = 0;
        mm[0] = mm[1] = 0;
        return;
    }
    int src = order[(size_t)s * n + p];
    const int* row = os + (size_t)src * kd + b;
    unsigned long long m[2] = {0, 0};
    // 16 loads in flight per batch (a load -> store chain per column paid one
    // L2 latency per entry)
    for (int j0 = 0; j0 < w; j0 += 16) {
        int v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = j0 + u < w ? __ldg(row + j0 + u) : -1;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int j = j0 + u;
            if (j >= w) break;
            dst[(size_t)j * kTileM] = v[u];
            if (v[u] >= 0) {
                const int wi = j / 64, biw = min(64, w - wi * 64);
                m[wi] |= 1ull << (biw - 1 - (j - wi * 64));
            }
        }
    }
    out_row[(size_t)s * rows_pad + p] = src;
    for (int u = 0; u < words; ++u) md[u] = m[u];
    mm[0] = m[0];
    mm[1] = words == 2 ? m[1] : 0;
}

// one 128-thread block per (split, 128-row tile): reorders the rows and
// writes the tile's OR-mask (the implicit-GEMM offset skip list) in the same pass
__global__ void __launch_bounds__(kTileM) k_split_reorder(
    const int* __restrict__ os, int n, int kd, int ns, int rows_pad,
    const int* __restrict__ begin, const int* __restrict__ word_off, const int* __restrict__ order,
    int* __restrict__ entries, int* __restrict__ out_row, unsigned long long* __restrict__ masks,
    unsigned long long* __restrict__ tmask) {
    pdl_wait();
    pdl_trigger();
    __shared__ unsigned long long red[2][kTileM / 32];
    const long long i = (long long)blockIdx.x * kTileM + threadIdx.x;  // rows_pad % 128 == 0
    const int s = (int)(i / rows_pad), p = (int)(i % rows_pad);
    unsigned long long mm[2] = {0, 0};
    row_reorder(os, n, kd, rows_pad, begin, word_off, order, entries, out_row, masks, s, p, mm);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        mm[0] |= __shfl_xor_sync(0xffffffffu, mm[0], o);
        mm[1] |= __shfl_xor_sync(0xffffffffu, mm[1], o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x / 32] = mm[0];
        red[1][threadIdx.x / 32] = mm[1];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long a = 0, b = 0;
        for (int w = 0; w < kTileM / 32; ++w) {
            a |= red[0][w];
            b |= red[1][w];
        }
        tmask[(size_t)blockIdx.x * 2] = a;  // tile index = s * n_tiles + t = blockIdx.x
        tmask[(size_t)blockIdx.x * 2 + 1] = b;
    }
}


// K=1 stride-1 map on one coordinate set: entries[q][0] = q (identity)
__global__ void k_identity_map(int n_out, int rows_pad, int* __restrict__ os,
                               unsigned long long* __restrict__ masks,
                               int* __restrict__ blk_counts) {
    pdl_wait();
    pdl_trigger();
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= rows_pad) return;
    os[q] = q < n_out ? q : -1;
    masks[q] = q < n_out ? 1ull : 0ull;
    if (q % kQB == 0) blk_counts[q / kQB] = min(kQB, n_out - q) > 0 ? min(kQB, n_out - q) : 0;
}

__global__ void k_iota(int* __restrict__ v, int n) {
    pdl_wait();
    pdl_trigger();
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = i;
}

// load factor <= 1/4: short linear-probing chains keep warps convergent (a
// warp waits for its longest chain); 16 B slots -> 64 n..128 n bytes, L2-resident
int64_t pow2_cap(int64_t n) {
    constexpr int64_t m = 4;  // slots per key (load factor 1/4; 1/2 measured 1.6x slower, r02_kmap.md)
    int64_t c = 64;
    while (c < m * n) c <<= 1;
    return c;
}

void coords_build_blocks(sk_coords* c, cudaStream_t st) {
    std::lock_guard<std::mutex> lock(c->mu);
    if (c->has_blocks) {
        stream_after(c->blocks_on, st);
        return;
    }
    c->blocks_on.mark(st);
    int64_t cap = 64;
    while (cap < 2 * (int64_t)c->n) cap <<= 1;  // n_blocks <= n: load <= 1/2 worst case
    c->bcap = cap;
    c->btable.alloc((size_t)cap * 16, st);
    fill_async(c->btable.p, 0xFF, c->btable.bytes, st);
    c->bdense.alloc((size_t)std::max(c->n, 1) * 64 * 4, st);  // cells initialised per block
    c->bcount.alloc(4, st);
    fill_async(c->bcount.p, 0, 4, st);
    if (c->n > 0) {
        launch_pdl(k_block_claim, (int)ceil_div(c->n, 256), 256, 0, st, c->coords.as<int4>(), c->n,
                   c->btable.as<ulonglong2>(), (uint64_t)cap - 1, c->bdense.as<int>(), c->bcount.as<int>());
        launch_pdl(k_block_fill, (int)ceil_div(c->n, 256), 256, 0, st, c->coords.as<int4>(), c->n,
                   (const ulonglong2*)c->btable.as<ulonglong2>(), (uint64_t)cap - 1, c->bdense.as<int>());
    }
    c->has_blocks = true;
}

// stride-1, non-transposed, 3-D, K in {3, 5}, input sets >= 64k voxels: the
// block-index query (with z-row loads and the claim/fill build it is faster
// than the per-voxel probes from ~50k voxels: SECOND scan 2122 -> 2188 scans/s,
// 0.68 -> 0.61 ms per scan; 1M voxels 2x). The threshold is a context setting
// (sk_ctx_set_kmap_block_rows, default 1 << 16).
bool use_block_query(const sk_kmap* m, const sk_coords* in) {
    const bool shape = !m->transposed && m->dims == 3 && (m->kernel == 3 || m->kernel == 5) &&
                       m->stride[0] == 1 && m->stride[1] == 1 && m->stride[2] == 1;
    return shape && in->n > 0 && m->n_in >= in->ctx->kmap_block_rows;
}

void launch_query(sk_kmap* m, const int4* out_coords, sk_coords* in, cudaStream_t st) {
    if (use_block_query(m, in)) {
        coords_build_blocks(in, st);
        const int grid = m->rows_pad / kQB;
        const size_t smem = (size_t)(kQB * m->kd + m->kd) * 4;
        auto run = [&](auto kern) {
            ensure_smem(reinterpret_cast<const void*>(kern), smem);
            launch_pdl(kern, grid, kQB, smem, st, out_coords, m->n_out, in->btable.as<ulonglong2>(),
                                          (uint64_t)in->bcap - 1, in->bdense.as<int>(), m->words,
                                          m->os.as<int>(), m->masks.as<unsigned long long>(),
                                          m->blk_counts.as<int>());
        };
        if (m->kernel == 3) run(k_kmap_query_blk<3>);
        else run(k_kmap_query_blk<5>);
        return;
    }
    coords_build_table(in, st);  // first hash query on this set builds its table
    const int grid = m->rows_pad / kQB;
    const uint64_t mask = (uint64_t)in->cap - 1;
    const size_t smem = (size_t)(kQB * m->kd + m->kd) * 4;
#define SK_Q(KDV, TPRV)                                                                      \
    ensure_smem(reinterpret_cast<const void*>(k_kmap_query<KDV, TPRV>), smem);               \
    launch_pdl(k_kmap_query<KDV, TPRV>, grid, kQB * TPRV, smem, st, \
        out_coords, m->n_out, in->table.as<ulonglong2>(), mask,                              \
        m->kernel, m->dims, m->stride[0], m->stride[1], m->stride[2], m->transposed, m->words, \
        m->os.as<int>(), m->masks.as<unsigned long long>(), m->blk_counts.as<int>())
    switch (m->kd) {
        case 1: SK_Q(1, 1); break;
        case 9: SK_Q(9, 2); break;
        case 25: SK_Q(25, 4); break;
        case 27: SK_Q(27, 4); break;
        case 125: SK_Q(125, 8); break;
        default: fail(SK_ERR_VALIDATION, "unsupported kernel volume " + std::to_string(m->kd));
    }
#undef SK_Q
}

void alloc_map(sk_kmap* m, cudaStream_t st) {
    m->rows_pad = (int)ceil_div(std::max(m->n_out, 1), kTileM) * kTileM;
    m->words = (m->kd + 63) / 64;
    m->n_blocks = m->rows_pad / kQB;
    m->os.alloc((size_t)m->rows_pad * m->kd * 4, st);
    m->masks.alloc((size_t)m->rows_pad * m->words * 8, st);
    m->blk_counts.alloc((size_t)m->n_blocks * m->kd * 4, st);
}

}  // namespace

uint64_t next_coord_set_id() {
    static std::atomic<uint64_t> counter{1};
    return counter.fetch_add(1);
}

void coords_check_range(sk_ctx*, const int32_t*, int, cudaStream_t) {}

namespace {
void build_table_locked(sk_coords* c, cudaStream_t st, int* err) {
    c->table_on.mark(st);
    c->cap = pow2_cap(c->n);
    c->table.alloc((size_t)c->cap * 16, st);
    fill_async(c->table.p, 0xFF, c->table.bytes, st);  // empty key, row = UINT_MAX
    if (c->n > 0) {
        launch_pdl(k_hash_insert, (int)ceil_div(c->n, 256), 256, 0, st, c->coords.as<int4>(), c->n,
                   c->table.as<ulonglong2>(), (uint64_t)c->cap - 1, err);
    }
    c->has_table = true;
}
}  // namespace

// creation-time validation of a root set (the packable range; the reference
// throws at construction), one 4 B read-back. Sets below the block-query
// threshold get their hash table here (the insert checks the range; callers
// like the ScanPipeline build it on their copy stream, off the forward's
// path); larger sets run a check kernel only and build the table on first
// use (coords_build_table): their stride-1 maps read only the block index.
// below this many voxels the table is built at creation even when the set's
// stride-1 maps use the block index: its strided maps / down-sampling need it
// anyway, and building it with the creation keeps it off the forward's path
// (ScanPipeline: copy stream); measured e2e -2.5 % with it lazy at 125k voxels
constexpr int kLazyTableRows = 1 << 19;

void coords_validate(sk_coords* c, cudaStream_t st) {
    if (c->n == 0) return;
    DevBuf err;
    err.alloc(4, st);
    fill_async(err.p, 0, 4, st);
    if (c->n < std::max(c->ctx->kmap_block_rows, kLazyTableRows)) {
        std::lock_guard<std::mutex> lock(c->mu);
        build_table_locked(c, st, err.as<int>());
    } else {
        launch_pdl(k_coords_check, (int)ceil_div(c->n, 256), 256, 0, st, c->coords.as<int4>(), c->n,
                   err.as<int>());
    }
    int h_err = 0;
    read_back(st, {{err.p, 4}}, &h_err);
    validate(h_err == 0,
             "coordinate outside the packable range (batch [0,4096), xyz [-65536,65536))");
}

void coords_build_table(sk_coords* c, cudaStream_t st) {
    std::lock_guard<std::mutex> lock(c->mu);
    if (c->has_table) {
        stream_after(c->table_on, st);
        return;
    }
    build_table_locked(c, st, nullptr);
}

sk_coords* coords_downsample(sk_coords* in, const int32_t stride[3], cudaStream_t st) {
    const int n = in->n;
    auto* out = new sk_coords();
    out->ctx = in->ctx;
    out->dims = in->dims;
    out->id = next_coord_set_id();
    for (int d = 0; d < 3; ++d) out->stride_tag[d] = in->stride_tag[d] * (d < in->dims ? stride[d] : 1);
    out->cap = pow2_cap(n);
    out->table.alloc((size_t)out->cap * 16, st);
    fill_async(out->table.p, 0xFF, out->table.bytes, st);
    if (n == 0) {
        out->n = 0;
        out->has_table = true;
        return out;
    }
    DevBuf slot, q, flag, pos, tmp, total;
    slot.alloc((size_t)n * 4, st);
    q.alloc((size_t)n * 16, st);
    flag.alloc((size_t)n * 4, st);
    pos.alloc((size_t)n * 4 + 4, st);
    const int g = (int)ceil_div(n, 256);
    launch_pdl(k_down_insert, g, 256, 0, st, in->coords.as<int4>(), n, stride[0], stride[1],
                                     in->dims == 3 ? stride[2] : 1, in->dims,
                                     out->table.as<ulonglong2>(), (uint64_t)out->cap - 1,
                                     slot.as<int>(), q.as<int4>());
    launch_pdl(k_down_flag, g, 256, 0, st, slot.as<int>(), out->table.as<ulonglong2>(), n, flag.as<int>());
    scan_exclusive_i32(flag.as<int>(), pos.as<int>(), n, pos.as<int>() + n, st);
    // the output coordinates are sized by the upper bound (n_out <= n), so the
    // compaction is queued before the count read-back and runs while the host
    // waits, instead of after it on the map stream's critical path
    out->coords.alloc((size_t)n * 16, st);
    launch_pdl(k_down_compact, g, 256, 0, st, flag.as<int>(), pos.as<int>(), slot.as<int>(),
                                      q.as<int4>(), n, out->table.as<ulonglong2>(),
                                      out->coords.as<int4>());
    int h_count = 0;
    read_back(st, {{pos.as<int>() + n, 4}}, &h_count);
    out->n = h_count;
    out->has_table = true;
    return out;
}


sk_coords* coords_quantize(sk_ctx* ctx, int dims, int m, const double* raw, const int32_t* batch,
                           const double voxel[3], int32_t* point_rows, cudaStream_t st) {
    validate(dims == 2 || dims == 3, "dims must be 2 or 3");
    validate(m >= 0, "negative point count");
    for (int d = 0; d < dims; ++d)
        validate(voxel[d] > 0.0, "voxel size components must be positive");
    auto* out = new sk_coords();
    out->ctx = ctx;
    out->dims = dims;
    out->id = next_coord_set_id();
    out->cap = pow2_cap(m);
    out->table.alloc((size_t)out->cap * 16, st);
    fill_async(out->table.p, 0xFF, out->table.bytes, st);
    if (m == 0) {
        out->n = 0;
        out->coords.alloc(16, st);
        out->has_table = true;
        return out;
    }
    DevBuf slot, q, flag, pos, tmp, err;
    slot.alloc((size_t)m * 4, st);
    q.alloc((size_t)m * 16, st);
    flag.alloc((size_t)m * 4, st);
    pos.alloc((size_t)m * 4 + 4, st);
    err.alloc(4, st);
    fill_async(err.p, 0, 4, st);
    const int g = (int)ceil_div(m, 256);
    launch_pdl(k_quant_insert, g, 256, 0, st, raw, batch, m, dims, voxel[0], voxel[1],
                                      dims == 3 ? voxel[2] : 1.0, out->table.as<ulonglong2>(),
                                      (uint64_t)out->cap - 1, slot.as<int>(), q.as<int4>(),
                                      err.as<int>());
    int h_err = 0;
    read_back(st, {{err.p, 4}}, &h_err);
    if (h_err) {
        delete out;
        validate(!(h_err & 1), "non-finite input coordinate");
        validate(false, "quantized coordinate outside the packable range "
                        "(batch [0,4096), xyz [-65536,65536))");
    }
    launch_pdl(k_down_flag, g, 256, 0, st, slot.as<int>(), out->table.as<ulonglong2>(), m, flag.as<int>());
    scan_exclusive_i32(flag.as<int>(), pos.as<int>(), m, pos.as<int>() + m, st);
    int h_count = 0;
    read_back(st, {{pos.as<int>() + m, 4}}, &h_count);
    out->n = h_count;
    out->coords.alloc((size_t)std::max(out->n, 1) * 16, st);
    launch_pdl(k_down_compact, g, 256, 0, st, flag.as<int>(), pos.as<int>(), slot.as<int>(), q.as<int4>(),
                                      m, out->table.as<ulonglong2>(), out->coords.as<int4>());
    out->has_table = true;
    if (point_rows) {
        launch_pdl(k_point_rows, g, 256, 0, st, slot.as<int>(), out->table.as<ulonglong2>(), m, point_rows);
    }
    return out;
}

void quantize_features(int m, int channels, const double* feats, const int32_t* point_rows,
                       int n, int rule, sk_dtype dt, void* out, cudaStream_t st) {
    validate(rule == 0 || rule == 1, "unknown dedup rule");
    validate(channels >= 0, "negative channel count");
    if (n == 0) return;
    validate(m > 0 && point_rows, "point rows required");
    auto launch = [&](auto tag) {
        using T = decltype(tag);
        T* o = static_cast<T*>(out);
        if (channels == 0) {  // occupancy: one channel of ones
            launch_pdl(k_fill<T>, (int)ceil_div(n, 256), 256, 0, st, o, n, 1.0);
            return;
        }
        const long long tot = (long long)n * channels;
        const int g = (int)ceil_div(tot, 256);
        if (rule == 0) {
            DevBuf first;
            first.alloc((size_t)n * 4, st);
            fill_async(first.p, 0x7F, (size_t)n * 4, st);
            launch_pdl(k_first_point, (int)ceil_div(m, 256), 256, 0, st, point_rows, m, first.as<int>());
            launch_pdl(k_quant_feats_first<T>, g, 256, 0, st, feats, channels, first.as<int>(), n, o);
        } else {
            DevBuf sum, cnt;
            sum.alloc((size_t)tot * 8, st);
            cnt.alloc((size_t)n * 4, st);
            fill_async(sum.p, 0, sum.bytes, st);
            fill_async(cnt.p, 0, cnt.bytes, st);
            launch_pdl(k_quant_sum, (int)ceil_div((long long)m * channels, 256), 256, 0, st, feats, channels, point_rows, m, sum.as<double>(), cnt.as<int>());
            launch_pdl(k_quant_mean<T>, g, 256, 0, st, sum.as<double>(), cnt.as<int>(), channels, n, o);
        }
    };
    if (dt == SK_F32) launch(float());
    else if (dt == SK_F64) launch(double());
    else if (dt == SK_F16) launch(__half());
    else if (dt == SK_BF16) launch(__nv_bfloat16());
    else fail(SK_ERR_VALIDATION, "unknown feature dtype");
}


sk_kmap* kmap_from_edges(sk_ctx* ctx, const int32_t* d_edges, int E, int R, int n_in, int n_out,
                         cudaStream_t st) {
    validate(R >= 1, "need at least one relation");
    validate(E >= 0 && n_in >= 0 && n_out >= 0, "negative size");
    auto* m = new sk_kmap();
    m->ctx = ctx;
    m->graph = true;
    m->kernel = 0;
    m->kd = R;
    m->n_in = n_in;
    m->n_out = n_out;
    m->rows_pad = (int)ceil_div(std::max(n_out, 1), kTileM) * kTileM;
    m->words = (R + 63) / 64;
    m->ws_ptr.alloc((size_t)(R + 1) * 8, st);
    m->ws_tile_ptr.alloc((size_t)(R + 1) * 4, st);
    m->ws_in.alloc((size_t)std::max(E, 1) * 4, st);
    m->ws_out.alloc((size_t)std::max(E, 1) * 4, st);
    const size_t cap_pad = (size_t)E + (size_t)R * kTileWS;
    m->ws_in_pad.alloc(cap_pad * 4, st);
    m->ws_out_pad.alloc(cap_pad * 4, st);
    fill_async(m->ws_in_pad.p, 0xFF, m->ws_in_pad.bytes, st);
    fill_async(m->ws_out_pad.p, 0xFF, m->ws_out_pad.bytes, st);
    DevBuf counts, err, keys, keys2, vals, order, tmp;
    counts.alloc((size_t)R * 4, st);
    err.alloc(4, st);
    fill_async(counts.p, 0, counts.bytes, st);
    fill_async(err.p, 0, 4, st);
    if (E > 0) {
        keys.alloc((size_t)E * 8, st);
        keys2.alloc((size_t)E * 8, st);
        vals.alloc((size_t)E * 4, st);
        order.alloc((size_t)E * 4, st);
        const int g = (int)ceil_div(E, 256);
        launch_pdl(k_edge_keys, g, 256, 0, st, d_edges, E, R, n_in, n_out, keys.as<unsigned long long>(),
                                       vals.as<int>(), counts.as<int>(), err.as<int>());
        int h_err = 0;
        read_back(st, {{err.p, 4}}, &h_err);
        if (h_err) {
            delete m;
            validate(!(h_err & 1), "relation id out of range");
            validate(false, "edge node id out of range");
        }
        int rbits = 1;
        while ((1 << rbits) < R) ++rbits;
        // LSD radix sort is stable: equal (relation, dst) keep the edge order
        unsigned long long* kb[2] = {keys.as<unsigned long long>(), keys2.as<unsigned long long>()};
        int* vb[2] = {vals.as<int>(), order.as<int>()};
        const int res = radix_sort_pairs<unsigned long long>(kb, vb, E, 0, 32 + rbits, st);
        if (res == 0) {  // k_edge_scatter reads keys2 / order
            SK_CUDA(cudaMemcpyAsync(keys2.p, keys.p, (size_t)E * 8, cudaMemcpyDeviceToDevice, st));
            SK_CUDA(cudaMemcpyAsync(order.p, vals.p, (size_t)E * 4, cudaMemcpyDeviceToDevice, st));
        }
        launch_pdl(k_edge_scan, 1, 1, 0, st, counts.as<int>(), R, m->ws_ptr.as<long long>(),
                                     m->ws_tile_ptr.as<int>());
        launch_pdl(k_edge_scatter, g, 256, 0, st, d_edges, keys2.as<unsigned long long>(), order.as<int>(),
                                          E, m->ws_ptr.as<long long>(), m->ws_tile_ptr.as<int>(),
                                          m->ws_in.as<int>(), m->ws_out.as<int>(),
                                          m->ws_in_pad.as<int>(), m->ws_out_pad.as<int>());
    } else {
        launch_pdl(k_edge_scan, 1, 1, 0, st, counts.as<int>(), R, m->ws_ptr.as<long long>(),
                                     m->ws_tile_ptr.as<int>());
    }
    m->has_ws = true;
    m->ws_on.mark(st);
    m->built_on.mark(st);
    m->total_pairs_host = E;
    return m;
}

sk_kmap* kmap_build(sk_coords* in, sk_coords* out, int kernel, const int32_t stride[3],
                    int transposed, cudaStream_t st) {
    validate(in->dims == out->dims, "offset dims mismatch");
    validate(kernel >= 1 && kernel % 2 == 1, "kernel size must be odd (even kernels unsupported)");
    validate(kernel <= 5, "kernel size > 5 unsupported");
    for (int d = 0; d < in->dims; ++d) validate(stride[d] >= 1, "stride components must be >= 1");
    auto* m = new sk_kmap();
    m->ctx = in->ctx;
    m->dims = in->dims;
    m->kernel = kernel;
    m->kd = in->dims == 3 ? kernel * kernel * kernel : kernel * kernel;
    for (int d = 0; d < 3; ++d) m->stride[d] = d < in->dims ? stride[d] : 1;
    m->transposed = transposed;
    m->n_in = in->n;
    m->n_out = out->n;
    m->identity = kernel == 1 && in == out && m->stride[0] == 1 && m->stride[1] == 1 &&
                  m->stride[2] == 1;
    alloc_map(m, st);
    if (m->identity) {
        launch_pdl(k_identity_map, (int)ceil_div(m->rows_pad, 256), 256, 0, st, m->n_out, m->rows_pad, m->os.as<int>(), m->masks.as<unsigned long long>(),
            m->blk_counts.as<int>());
    } else {
        launch_query(m, out->coords.as<int4>(), in, st);
    }
    return m;
}

// build_kmap with per-axis kernel sizes and dilation (extension). Odd,
// symmetric kernels with dilation 1 take the standard path.
sk_kmap* kmap_build_ex(sk_coords* in, sk_coords* out, const int32_t kernel[3],
                       const int32_t stride[3], const int32_t dilation[3], int transposed,
                       cudaStream_t st) {
    validate(in->dims == out->dims, "offset dims mismatch");
    const int dims = in->dims;
    int k3[3] = {kernel[0], kernel[1], dims == 3 ? kernel[2] : 1};
    int d3[3] = {dilation[0], dilation[1], dims == 3 ? dilation[2] : 1};
    for (int d = 0; d < 3; ++d) {
        validate(k3[d] >= 1 && k3[d] <= 8, "kernel size per axis must be in [1, 8]");
        validate(d3[d] >= 1, "dilation components must be >= 1");
    }
    for (int d = 0; d < dims; ++d) validate(stride[d] >= 1, "stride components must be >= 1");
    const int KD = k3[0] * k3[1] * k3[2];
    validate(KD <= 128, "kernel volume > 128 unsupported");
    const bool standard = k3[0] == k3[1] && (dims == 2 || k3[1] == k3[2]) && k3[0] % 2 == 1 &&
                          k3[0] <= 5 && d3[0] == 1 && d3[1] == 1 && d3[2] == 1;
    if (standard) return kmap_build(in, out, k3[0], stride, transposed, st);
    coords_build_table(in, st);
    auto* m = new sk_kmap();
    m->ctx = in->ctx;
    m->dims = dims;
    m->kernel = -1;  // generalized offsets (see kmap_build_ex)
    m->kd = KD;
    for (int d = 0; d < 3; ++d) m->stride[d] = d < dims ? stride[d] : 1;
    m->transposed = transposed;
    m->n_in = in->n;
    m->n_out = out->n;
    alloc_map(m, st);
    std::vector<int4> h(KD);
    int n = 0;
    for (int a = 0; a < k3[0]; ++a)
        for (int b = 0; b < k3[1]; ++b)
            for (int c = 0; c < k3[2]; ++c)
                h[n++] = make_int4(d3[0] * (a - (k3[0] - 1) / 2), d3[1] * (b - (k3[1] - 1) / 2),
                                   dims == 3 ? d3[2] * (c - (k3[2] - 1) / 2) : 0, 0);
    DevBuf offs;
    offs.alloc((size_t)KD * 16, st);
    SK_CUDA(cudaMemcpyAsync(offs.p, h.data(), (size_t)KD * 16, cudaMemcpyHostToDevice, st));
    constexpr int TPR = 4;
    const size_t smem = (size_t)(kQB * KD + ((KD + 3) & ~3)) * 4 + (size_t)KD * 16;
    ensure_smem(reinterpret_cast<const void*>(k_kmap_query_gen<TPR>), smem);
    launch_pdl(k_kmap_query_gen<TPR>, m->rows_pad / kQB, kQB * TPR, smem, st, out->coords.as<int4>(), m->n_out, in->table.as<ulonglong2>(), (uint64_t)in->cap - 1,
        offs.as<int4>(), KD, dims, m->stride[0], m->stride[1], m->stride[2], transposed, m->words,
        m->os.as<int>(), m->masks.as<unsigned long long>(), m->blk_counts.as<int>());
    // the offsets table must outlive the kernel: a stream-ordered free
    return m;
}

sk_kmap* kmap_transpose(sk_kmap* src, cudaStream_t st) {
    // transpose_map rejects graph maps (kmap.cpp:290-295): so does conv_dgrad on them
    contract(!src->graph, "graph maps cannot be transposed");
    std::lock_guard<std::mutex> lock(src->mu);
    if (src->transpose_cache) {
        stream_after(src->transpose_cache->built_on, st);
        return src->transpose_cache;
    }
    auto* m = new sk_kmap();
    m->ctx = src->ctx;
    m->dims = src->dims;
    m->kernel = src->kernel;
    m->kd = src->kd;
    for (int d = 0; d < 3; ++d) m->stride[d] = src->stride[d];
    m->transposed = !src->transposed;
    m->n_in = src->n_out;
    m->n_out = src->n_in;
    m->identity = src->identity;
    alloc_map(m, st);
    fill_async(m->os.p, 0xFF, m->os.bytes, st);
    long long total = (long long)src->n_out * src->kd;
    if (total > 0) {
        launch_pdl(k_transpose, (int)ceil_div(total, 256), 256, 0, st, src->os.as<int>(), src->n_out,
                                                               src->kd, m->os.as<int>());
    }
    size_t smem = (size_t)(kQB * m->kd + m->kd) * 4;
    ensure_smem(reinterpret_cast<const void*>(k_finalize), smem);
    launch_pdl(k_finalize, m->n_blocks, kQB, smem, st, m->os.as<int>(), m->kd, m->words,
                                               m->masks.as<unsigned long long>(),
                                               m->blk_counts.as<int>());
    m->built_on.mark(st);
    src->transpose_cache = m;  // owned by src, released in ~sk_kmap
    return m;
}

void kmap_ensure_ws(sk_kmap* m, cudaStream_t st) {
    std::lock_guard<std::mutex> lock(m->mu);
    if (m->has_ws) {
        stream_after(m->ws_on, st);
        return;
    }
    m->ws_on.mark(st);
    m->ws_ptr.alloc((size_t)(m->kd + 1) * 8, st);
    m->ws_tile_ptr.alloc((size_t)(m->kd + 1) * 4, st);
    m->blk_off.alloc((size_t)m->n_blocks * m->kd * 8, st);
    size_t cap = (size_t)std::max<int64_t>(1, (int64_t)m->n_out * m->kd);
    m->ws_in.alloc(cap * 4, st);
    m->ws_out.alloc(cap * 4, st);
    const size_t cap_pad = cap + (size_t)m->kd * kTileWS;
    m->ws_in_pad.alloc(cap_pad * 4, st);
    m->ws_out_pad.alloc(cap_pad * 4, st);
    fill_async(m->ws_in_pad.p, 0xFF, m->ws_in_pad.bytes, st);
    fill_async(m->ws_out_pad.p, 0xFF, m->ws_out_pad.bytes, st);
    launch_pdl(k_ws_scan, 1, 1024, 0, st, m->blk_counts.as<int>(), m->n_blocks, m->kd,
                                  m->blk_off.as<long long>(), m->ws_ptr.as<long long>(),
                                  m->ws_tile_ptr.as<int>());
    size_t smem = (size_t)kQB * m->kd * 4;
    ensure_smem(reinterpret_cast<const void*>(k_ws_scatter), smem);
    launch_pdl(k_ws_scatter, m->n_blocks, kQB, smem, st, m->os.as<int>(), m->kd,
                                                 m->blk_off.as<long long>(),
                                                 m->ws_ptr.as<long long>(), m->ws_tile_ptr.as<int>(),
                                                 m->ws_in.as<int>(), m->ws_out.as<int>(),
                                                 m->ws_in_pad.as<int>(), m->ws_out_pad.as<int>());
    m->has_ws = true;
}

int64_t kmap_total_pairs(sk_kmap* m, cudaStream_t st) {
    kmap_ensure_ws(m, st);
    if (m->total_pairs_host >= 0) return m->total_pairs_host;
    long long v = 0;
    read_back(st, {{m->ws_ptr.as<long long>() + m->kd, 8}}, &v);
    m->total_pairs_host = v;
    return v;
}

Prepared* kmap_prepare(sk_kmap* m, int splits, int pad, cudaStream_t st) {
    contract(!m->graph, "graph maps have no OS form (pair-list dataflows only)");
    validate(splits >= 0, "split count must be >= 0");
    validate(splits <= m->kd, "split count exceeds number of kernel offsets");
    validate(pad >= 1, "pad multiple must be >= 1");
    std::lock_guard<std::mutex> lock(m->mu);
    auto key = std::make_pair(splits, pad);
    auto it = m->prepared.find(key);
    if (it != m->prepared.end()) {
        stream_after(it->second->built_on, st);
        return it->second.get();
    }

    auto p = std::make_unique<Prepared>();
    p->splits = splits;
    p->pad = pad;
    p->num_splits = std::max(splits, 1);
    // rows padded to lcm(pad, 128) so every prepared map also runs in 128-row tiles
    int64_t a = pad, b = kTileM;
    while (b) { int64_t t = a % b; a = b; b = t; }
    int64_t l = (int64_t)pad / a * kTileM;
    p->rows_pad = (int)(ceil_div(std::max(m->n_out, 1), l) * l);
    const int ns = p->num_splits, n = m->n_out, kd = m->kd;
    p->begin.resize(ns + 1);
    if (splits == 0) {
        p->begin = {0, kd};
    } else {
        int chunk = kd / splits, rem = kd % splits, bb = 0;
        for (int s = 0; s < splits; ++s) {  // kmap.cpp:227-236
            p->begin[s] = bb;
            bb += chunk + (s < rem ? 1 : 0);
        }
        p->begin[splits] = bb;
    }
    p->word_off.resize(ns + 1);
    int wacc = 0, W = 0;
    for (int s = 0; s < ns; ++s) {
        int w = p->begin[s + 1] - p->begin[s];
        p->word_off[s] = wacc;
        wacc += (w + 63) / 64;
        W = std::max(W, w);
    }
    p->word_off[ns] = wacc;
    p->mask_words_max = (W + 63) / 64;
    p->entries.alloc((size_t)p->rows_pad * kd * 4, st);
    p->out_row.alloc((size_t)p->rows_pad * ns * 4, st);
    p->masks.alloc((size_t)p->rows_pad * wacc * 8, st);
    DevBuf& d_begin = p->d_begin;
    DevBuf d_woff;
    d_begin.alloc((ns + 1) * 4, st);
    d_woff.alloc((ns + 1) * 4, st);
    validate(ns <= kMaxSplitDesc, "split count exceeds 128");
    SplitDesc sd;
    sd.ns = ns;
    sd.kd = kd;
    sd.W = W;
    sd.n = n;
    for (int i = 0; i <= ns; ++i) {
        sd.begin[i] = p->begin[i];
        sd.woff[i] = p->word_off[i];
    }
    int sbits = 0;
    while ((1 << sbits) < ns) ++sbits;
    // the fused key-generation path (32-bit keys from the query's masks) writes
    // the split bounds itself; every other path gets them from k_split_desc
    const bool fused32 = splits != 0 && n != 0 && kd <= 64 && W + (ns > 1 ? sbits : 0) <= 32;
    if (!fused32) {
        launch_pdl(k_split_desc, 1, 128, 0, st, sd, d_begin.as<int>(), d_woff.as<int>());
    }

    DevBuf order;
    order.alloc((size_t)std::max(n * ns, 1) * 4, st);
    if (splits == 0 || n == 0) {
        // unsorted: identity order (split_and_sort(0) leaves the map unchanged)
        if (n) {
            launch_pdl(k_iota, (int)ceil_div(n, 256), 256, 0, st, order.as<int>(), n);
        }
    } else {
        const long long tot = (long long)n * ns;
        DevBuf k_in, k_out, v_in, v_out, order1;
        k_in.alloc(tot * (fused32 ? 4 : 8), st);
        k_out.alloc(tot * (fused32 ? 4 : 8), st);
        v_in.alloc(tot * 4, st);
        if (!fused32) v_out.alloc(tot * 4, st);
        if (!fused32 && W > 64) order1.alloc(tot * 4, st);
        const int g = (int)ceil_div(tot, 256);
        // stable sort of (key, row) -> dst (hand-written radix sort, sort.cu)
        auto sort_to = [&](auto* kdummy, int end_bit, int* dst) {
            using KT = std::remove_pointer_t<decltype(kdummy)>;
            KT* kb[2] = {k_in.as<KT>(), k_out.as<KT>()};
            int* vb[2] = {v_in.as<int>(), v_out.as<int>()};
            const int r = radix_sort_pairs<KT>(kb, vb, (int)tot, 0, end_bit, st);
            SK_CUDA(cudaMemcpyAsync(dst, vb[r], (size_t)tot * 4, cudaMemcpyDeviceToDevice, st));
        };
        auto sort_pass = [&](int word, int end_bit, const int* perm, int* dst) {
            launch_pdl(k_split_keys, g, 256, 0, st, m->os.as<int>(), n, kd, ns, d_begin.as<int>(), W, word,
                                            perm, k_in.as<unsigned long long>(), v_in.as<int>());
            sort_to((unsigned long long*)nullptr, end_bit, dst);
        };
        if (fused32) {
            const int end_bit = W + (ns > 1 ? sbits : 0);
            const RadixPlan pl = radix_plan((int)tot, end_bit);
            DevBuf scratch;
            scratch.alloc(pl.scratch_words * 4, st);
            fill_async(scratch.p, 0, scratch.bytes, st);
            // values start in the buffer that makes the last pass land in order
            int* vb[2];
            vb[pl.passes % 2] = order.as<int>();
            vb[(pl.passes + 1) % 2] = v_in.as<int>();
            unsigned* kb[2] = {k_in.as<unsigned>(), k_out.as<unsigned>()};
            const size_t hsm = pl.hist_words * 4;
            ensure_smem(reinterpret_cast<const void*>(k_split_keygen32), hsm);
            const int kg = (int)std::min<long long>(ceil_div(tot, 256), 2 * 148);
            launch_pdl(k_split_keygen32, kg, 256, hsm, st, m->masks.as<unsigned long long>(), sd, pl.dbits,
                                                   pl.passes, kb[0], vb[0], scratch.as<uint32_t>(),
                                                   d_begin.as<int>(), d_woff.as<int>());
            const int r = radix_sort_run<unsigned>(kb, vb, (int)tot, 0, pl, scratch.as<uint32_t>(),
                                                   true, st);
            if (vb[r] != order.as<int>())  // fewer passes ran (n <= 1)
                SK_CUDA(cudaMemcpyAsync(order.p, vb[r], (size_t)tot * 4, cudaMemcpyDeviceToDevice, st));
        } else if (W <= 64) {
            sort_pass(0, std::min(64, W + (ns > 1 ? sbits : 0)), nullptr, order.as<int>());
        } else {
            // one split wider than 64 columns (K=5, s=1): stable LSD over the
            // two mask words -- low word first, then stably by the high word
            // over the pass-1 order (== big-endian word compare, kmap.cpp:49-54)
            sort_pass(1, W - 64, nullptr, order1.as<int>());
            sort_pass(0, 64, order1.as<int>(), order.as<int>());
        }
    }
    const long long tot_rows = (long long)p->rows_pad * ns;
    const int n_tiles = p->rows_pad / kTileM;
    p->tile_masks.alloc((size_t)n_tiles * ns * 16, st);
    launch_pdl(k_split_reorder, (int)(tot_rows / kTileM), kTileM, 0, st, m->os.as<int>(), n, kd, ns, p->rows_pad, d_begin.as<int>(), d_woff.as<int>(),
        order.as<int>(), p->entries.as<int>(), p->out_row.as<int>(),
        p->masks.as<unsigned long long>(), p->tile_masks.as<unsigned long long>());
    Prepared* raw = p.get();
    raw->built_on.mark(st);
    m->prepared[key] = std::move(p);
    return raw;
}

}  // namespace sk
