// Hand-written device primitives of the kernel-map pipeline (no CUB):
//
//  * scan_exclusive_i32: single-pass exclusive prefix sum with decoupled
//    look-back (one launch + one status memset): tiles of 4096 ints claim
//    their index from an atomic counter, publish their aggregate, look back
//    over the predecessors' (flag, value) words and publish their inclusive
//    prefix. Used by the first-appearance compactions (build_out_coords,
//    quantize; kmap.cpp:80-88, tensor.cpp:87-142).
//
//  * radix_sort_pairs: stable LSD radix sort of (key, int value) pairs with
//    up-to-10-bit digits (split_and_sort's stable mask sort, kmap.cpp:252-256;
//    the graph maps' stable (relation, dst) order, kmap.cpp:317-336). One
//    histogram launch computes every pass's global digit counts; then ONE
//    launch per pass ("onesweep"): each 2048-key tile ranks its keys stably
//    in shared memory (per-warp digit counters, __match_any_sync peers),
//    publishes its per-digit counts and looks back over the earlier tiles'
//    counts (decoupled look-back) to find its output offsets. A 27-bit split
//    mask key sorts in 3 passes (CUB's 8-bit onesweep: 4), a split-local key
//    of <= 11 bits (3+ splits at K=3) in two of <= 6 bits.
#include "sk_internal.hpp"

namespace sk {

namespace {

constexpr int kScanThreads = 1024, kScanIpt = 4, kScanTile = kScanThreads * kScanIpt;
constexpr uint32_t kFlagAgg = 1u << 30, kFlagPre = 2u << 30, kValMask = (1u << 30) - 1;

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// block-wide exclusive scan of one value per thread (blockDim multiple of 32)
template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, int* warp_sums, int& total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[w] = x;
    __syncthreads();
    if (w == 0) {
        int s = lane < NT / 32 ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < NT / 32) warp_sums[lane] = s;  // inclusive warp prefix
    }
    __syncthreads();
    total = warp_sums[NT / 32 - 1];
    const int base = w > 0 ? warp_sums[w - 1] : 0;
    __syncthreads();
    return base + x - v;
}

// status[0] = tile counter, status[1 + t] = (flag | value) of tile t
__global__ void __launch_bounds__(kScanThreads) k_scan_lookback(const int* __restrict__ in,
                                                                int* __restrict__ out, int n,
                                                                uint32_t* __restrict__ status,
                                                                int* __restrict__ total_out) {
    pdl_wait();
    pdl_trigger();
    __shared__ int warp_sums[32];
    __shared__ int s_tile, s_prefix;
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(status, 1u);
    __syncthreads();
    const int tile = s_tile;
    const long long base = (long long)tile * kScanTile + (long long)threadIdx.x * kScanIpt;
    int v[kScanIpt];
    int sum = 0;
#pragma unroll
    for (int i = 0; i < kScanIpt; ++i) {
        v[i] = base + i < n ? in[base + i] : 0;
        sum += v[i];
    }
    int agg = 0;
    const int excl = block_excl_scan<kScanThreads>(sum, warp_sums, agg);
    uint32_t* st = status + 1;
    if (threadIdx.x == 0) {
        if (tile == 0) {
            st_relaxed(st, kFlagPre | (uint32_t)agg);
            s_prefix = 0;
        } else {
            st_relaxed(st + tile, kFlagAgg | (uint32_t)agg);
        }
    }
    if (tile > 0 && threadIdx.x < 32) {
        // warp look-back: lanes read 32 predecessors at once, newest first
        int prefix = 0;
        int t = tile - 1 - (int)threadIdx.x;
        for (;;) {
            uint32_t s = t >= 0 ? ld_volatile(st + t) : kFlagPre;
            while (__any_sync(0xffffffffu, (s >> 30) == 0)) {
                if ((s >> 30) == 0) s = ld_volatile(st + t);
            }
            const uint32_t pre = __ballot_sync(0xffffffffu, (s >> 30) == 2);
            const int stop = pre ? __ffs(pre) - 1 : 32;  // first (newest) lane with a prefix
            int add = (int)threadIdx.x <= stop && t >= 0 ? (int)(s & kValMask) : 0;
#pragma unroll
            for (int o = 16; o; o >>= 1) add += __shfl_xor_sync(0xffffffffu, add, o);
            prefix += add;
            if (pre) break;
            t -= 32;
        }
        if (threadIdx.x == 0) {
            st_relaxed(st + tile, kFlagPre | (uint32_t)(prefix + agg));
            s_prefix = prefix;
        }
    }
    __syncthreads();
    int run = s_prefix + excl;
#pragma unroll
    for (int i = 0; i < kScanIpt; ++i) {
        if (base + i < n) out[base + i] = run;
        run += v[i];
    }
    if (total_out && base + kScanIpt >= n && base < n) *total_out = run;
}

// ---- radix sort ------------------------------------------------------------
constexpr int kRsThreads = 256, kRsWarps = 8, kRsIpt = 8, kRsTile = kRsThreads * kRsIpt;
// 10-bit digits: 27-bit masks in 3 passes, 3-4 split keys (<= 11 bits) in 2
// passes of <= 6 bits rather than one of 11 (measured, tools/prep_bench.py:
// 1024+-digit look-backs made the single pass the slowest: s=3 prepare 70.6
// -> 52.2 us, s=1 65.5 -> 64.5 us)
constexpr int kRsMaxBits = 10, kRsMaxPasses = 8;
constexpr int kLookBatch = 16;  // 32 / 64 measured slower (register pressure)

template <typename KT>
__global__ void __launch_bounds__(kRsThreads) k_radix_hist(const KT* __restrict__ keys, int n,
                                                            int begin_bit, int dbits, int passes,
                                                            uint32_t* __restrict__ ghist) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ uint32_t sh[];  // [passes][1 << dbits]
    const int D = 1 << dbits;
    for (int i = threadIdx.x; i < passes * D; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long lim = (n + stride - 1) / stride * stride;  // whole warps iterate together
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < lim; i += stride) {
        if (i >= n) {
            for (int p = 0; p < passes; ++p) hist_add(sh + p * D, -1);
            continue;
        }
        const KT k = keys[i];
        for (int p = 0; p < passes; ++p)
            hist_add(sh + p * D, (int)((k >> (begin_bit + p * dbits)) & (KT)(D - 1)));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * D; i += blockDim.x)
        if (sh[i]) atomicAdd(&ghist[i], sh[i]);
}

// one stable counting pass over digit (k >> shift) & (D-1)
template <typename KT>
__global__ void __launch_bounds__(kRsThreads) k_radix_pass(
    const KT* __restrict__ kin, const int* __restrict__ vin, KT* __restrict__ kout,
    int* __restrict__ vout, int n, int shift, int dbits, const uint32_t* __restrict__ ghist,
    uint32_t* __restrict__ status /* [0] counter, then [tiles][D] */) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ int rs[];
    const int D = 1 << dbits;
    int* whist = rs;                      // [warps][D]: per-warp counts -> warp offsets
    int* boff = whist + kRsWarps * D;     // [D] block's global start per digit
    __shared__ int s_tile;
    __shared__ int wsum[kRsWarps];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kRsWarps * D; i += kRsThreads) whist[i] = 0;
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(status, 1u);
    __syncthreads();
    const int tile = s_tile;
    uint32_t* st = status + 1;
    // blocked arrangement: warp w ranks keys [w*256, w*256+256) of the tile in
    // 8 steps of 32 (coalesced loads; warp order = key order -> stable)
    const long long t0 = (long long)tile * kRsTile + (long long)w * (32 * kRsIpt);
    KT k[kRsIpt];
    int v[kRsIpt], d[kRsIpt], r[kRsIpt];
#pragma unroll
    for (int j = 0; j < kRsIpt; ++j) {
        const long long i = t0 + j * 32 + lane;
        const bool ok = i < n;
        k[j] = ok ? kin[i] : (KT)0;
        v[j] = ok ? vin[i] : 0;
        d[j] = ok ? (int)((k[j] >> shift) & (KT)(D - 1)) : -1;
    }
    int* wh = whist + w * D;
#pragma unroll
    for (int j = 0; j < kRsIpt; ++j) {
        const unsigned peers = __match_any_sync(0xffffffffu, d[j]);
        const int below = __popc(peers & ((1u << lane) - 1));
        const int cur = d[j] >= 0 ? wh[d[j]] : 0;
        __syncwarp();
        r[j] = cur + below;
        if (d[j] >= 0 && below == 0) wh[d[j]] = cur + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // per digit: block count, then per-warp exclusive offsets (in place)
    for (int dd = threadIdx.x; dd < D; dd += kRsThreads) {
        int c = 0;
#pragma unroll
        for (int ww = 0; ww < kRsWarps; ++ww) {
            const int x = whist[ww * D + dd];
            whist[ww * D + dd] = c;
            c += x;
        }
        boff[dd] = c;  // block count for now
        // publish this tile's aggregate for digit dd
        st_relaxed(st + (size_t)tile * D + dd, (tile == 0 ? kFlagPre : kFlagAgg) | (uint32_t)c);
    }
    // global exclusive start of every digit (from the all-pass histogram)
    {
        const int per = D / kRsThreads > 0 ? D / kRsThreads : 1;  // digits per thread
        int loc = 0;
        const int d0 = threadIdx.x * per;
        for (int q = 0; q < per; ++q)
            if (d0 + q < D) loc += (int)ghist[d0 + q];
        int tot = 0;
        int excl = block_excl_scan<kRsThreads>(loc, wsum, tot);
        // look back per digit: thread handles digits d0..d0+per-1
        for (int q = 0; q < per; ++q) {
            const int dd = d0 + q;
            if (dd >= D) break;
            int pre = 0;
            if (tile > 0) {
                // batched look-back: 16 independent (relaxed) status loads per
                // round, summed newest-first until an inclusive prefix; the
                // flag and the count share one word, so no acquire is needed
                bool done = false;
                for (int t = tile - 1; !done; t -= kLookBatch) {
                    uint32_t sv[kLookBatch];
#pragma unroll
                    for (int u = 0; u < kLookBatch; ++u)
                        sv[u] = t - u >= 0 ? ld_volatile(st + (size_t)(t - u) * D + dd) : kFlagPre;
#pragma unroll
                    for (int u = 0; u < kLookBatch; ++u) {
                        if (done) break;
                        while ((sv[u] >> 30) == 0) sv[u] = ld_volatile(st + (size_t)(t - u) * D + dd);
                        pre += (int)(sv[u] & kValMask);
                        done = (sv[u] >> 30) == 2;
                    }
                }
                st_relaxed(st + (size_t)tile * D + dd, kFlagPre | (uint32_t)(pre + boff[dd]));
            }
            boff[dd] = excl + pre;
            excl += (int)ghist[dd];
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kRsIpt; ++j) {
        if (d[j] < 0) continue;
        const int pos = boff[d[j]] + whist[w * D + d[j]] + r[j];
        kout[pos] = k[j];
        vout[pos] = v[j];
    }
}

}  // namespace

void scan_exclusive_i32(const int* in, int* out, int n, int* total_dev, cudaStream_t st) {
    if (n <= 0) {
        if (total_dev) fill_async(total_dev, 0, 4, st);
        return;
    }
    const int tiles = (int)ceil_div(n, kScanTile);
    DevBuf status;
    status.alloc((size_t)(tiles + 1) * 4, st);
    fill_async(status.p, 0, status.bytes, st);
    launch_pdl(k_scan_lookback, tiles, kScanThreads, 0, st, in, out, n, status.as<uint32_t>(), total_dev);
}

RadixPlan radix_plan(int n, int bits) {
    RadixPlan r;
    r.bits = bits;
    r.passes = bits > 0 ? (int)ceil_div(bits, kRsMaxBits) : 0;
    if (r.passes > kRsMaxPasses) fail(SK_ERR_VALIDATION, "radix sort key wider than 80 bits");
    if ((long long)n >= (1ll << 30)) fail(SK_ERR_VALIDATION, "radix sort: too many keys");
    r.dbits = r.passes ? (int)ceil_div(bits, r.passes) : 0;
    r.digits = 1 << r.dbits;
    r.tiles = (int)ceil_div(std::max(n, 1), kRsTile);
    r.hist_words = (size_t)r.passes * r.digits;
    r.scratch_words = r.hist_words + (size_t)r.passes * ((size_t)r.tiles * r.digits + 1);
    return r;
}

template <typename KT>
int radix_sort_run(KT* keys[2], int* vals[2], int n, int begin_bit, const RadixPlan& pl,
                   uint32_t* scratch, bool have_hist, cudaStream_t st) {
    if (n <= 1 || pl.passes == 0) return 0;
    const int D = pl.digits;
    if (!have_hist) {
        const size_t hsm = pl.hist_words * 4;
        ensure_smem(reinterpret_cast<const void*>(k_radix_hist<KT>), hsm);
        const int hg = (int)std::min<int64_t>(ceil_div(n, kRsThreads * 8), 148 * 4);
        launch_pdl(k_radix_hist<KT>, hg, kRsThreads, hsm, st, keys[0], n, begin_bit, pl.dbits, pl.passes,
                                                       scratch);
    }
    const size_t psm = (size_t)(kRsWarps + 1) * D * 4;
    ensure_smem(reinterpret_cast<const void*>(k_radix_pass<KT>), psm);
    uint32_t* status = scratch + pl.hist_words;
    int cur = 0;
    for (int p = 0; p < pl.passes; ++p) {
        launch_pdl(k_radix_pass<KT>, pl.tiles, kRsThreads, psm, st, (const KT*)keys[cur],
                   (const int*)vals[cur], keys[cur ^ 1], vals[cur ^ 1], n, begin_bit + p * pl.dbits,
                   pl.dbits, (const uint32_t*)(scratch + (size_t)p * D),
                   status + (size_t)p * ((size_t)pl.tiles * D + 1));
        cur ^= 1;
    }
    return cur;
}

template <typename KT>
int radix_sort_pairs(KT* keys[2], int* vals[2], int n, int begin_bit, int end_bit, cudaStream_t st) {
    if (n <= 1 || end_bit <= begin_bit) return 0;
    const RadixPlan pl = radix_plan(n, end_bit - begin_bit);
    DevBuf scratch;
    scratch.alloc(pl.scratch_words * 4, st);
    fill_async(scratch.p, 0, scratch.bytes, st);
    return radix_sort_run<KT>(keys, vals, n, begin_bit, pl, scratch.as<uint32_t>(), false, st);
}

template int radix_sort_pairs<uint32_t>(uint32_t* keys[2], int* vals[2], int, int, int, cudaStream_t);
template int radix_sort_pairs<unsigned long long>(unsigned long long* keys[2], int* vals[2], int,
                                                  int, int, cudaStream_t);
template int radix_sort_run<uint32_t>(uint32_t* keys[2], int* vals[2], int, int, const RadixPlan&,
                                      uint32_t*, bool, cudaStream_t);
template int radix_sort_run<unsigned long long>(unsigned long long* keys[2], int* vals[2], int, int,
                                                const RadixPlan&, uint32_t*, bool, cudaStream_t);

}  // namespace sk
