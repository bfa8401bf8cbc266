// sk200 internal object model behind the C ABI (include/sk200.h).
#pragma once
#include <atomic>

#include "sk_common.cuh"

struct sk_ctx {
    int device = 0;
    int num_sms = 148;
    bool deterministic = false;
    int kmap_block_rows = 1 << 16;  // sk_ctx_set_kmap_block_rows
    size_t smem_optin = 227 * 1024;
    // dynamic work queues of the persistent conv kernels: kSchedSlots pairs
    // {next item, CTAs done}, zeroed once; a launch takes the next slot and
    // its last CTA re-zeroes it
    static constexpr uint32_t kSchedSlots = 16384;
    int* sched = nullptr;
    std::atomic<uint32_t> sched_seq{0};
    int* sched_slot() { return sched ? sched + 2 * (sched_seq.fetch_add(1) % kSchedSlots) : nullptr; }
};

namespace sk {

struct Refcounted {
    std::atomic<int> refs{1};
    virtual ~Refcounted() = default;
};

// Prepared (split + sorted + padded) OS map: prepare_os_map (exec.cpp:342-344).
struct Prepared {
    int splits = 0;       // requested (0 = unsorted single split)
    int pad = 1;          // pad multiple (TilePreset::cta_m)
    int num_splits = 1;   // max(splits, 1)
    int rows_pad = 0;     // per split
    int mask_words_max = 1;
    std::vector<int> begin;  // num_splits + 1 global offset bounds
    DevBuf d_begin;          // begin[] on device
    DevBuf entries;          // split s at rows_pad*begin[s]: [tile][col][128] (tile-column-major)
    DevBuf out_row;          // num_splits x rows_pad (-1 pad rows)
    DevBuf masks;            // split s at rows_pad*word_off[s]: rows_pad x words_s
    std::vector<int> word_off;
    DevBuf tile_masks;       // num_splits x n_tiles(of 128) x 2 u64 (OR of row masks)
    int tile_rows = 128;
    BuiltOn built_on;
};

}  // namespace sk

struct sk_coords : sk::Refcounted {
    sk_ctx* ctx = nullptr;
    int dims = 3;
    int n = 0;
    int32_t stride_tag[3] = {1, 1, 1};
    uint64_t id = 0;
    sk::DevBuf coords;  // int4 [n]
    // open-addressing hash: 16 B slots {u64 key, u32 row, pad} [cap]
    sk::DevBuf table;
    int64_t cap = 0;
    bool has_table = false;
    // 4x4x4 block index for stride-1 queries (built on first use): block hash
    // {u64 block key, u32 block id} [bcap] and per block the 64 rows of its
    // cells (INT_MAX = empty) -- one hash probe per neighbour BLOCK instead of
    // per neighbour voxel
    sk::DevBuf btable, bdense, bcount;
    int64_t bcap = 0;
    bool has_blocks = false;
    std::mutex mu;
    sk::BuiltOn built_on;   // stream of a lazily built (down-sampled / quantized) set
    sk::BuiltOn blocks_on;  // stream the block index was built on
    sk::BuiltOn table_on;   // stream a root set's hash table was built on (first use)
    // children: downsampled sets by stride (owned), maps by key (owned)
    std::map<std::tuple<int, int, int>, sk_coords*> down;
    // key: (out id, kernel code, stride xyz, transposed, dilation code)
    std::map<std::tuple<uint64_t, int, int, int, int, int, int>, sk_kmap*> maps;
    ~sk_coords() override;
};

struct sk_kmap : sk::Refcounted {
    sk_ctx* ctx = nullptr;
    int dims = 3, kernel = 3, kd = 27;
    int stride[3] = {1, 1, 1};
    int transposed = 0;
    int n_in = 0, n_out = 0;
    int rows_pad = 0;       // n_out rounded up to 128 (the raw OS is stored padded)
    bool identity = false;  // K=1, stride 1, in set == out set: entries[q][0] == q
    bool graph = false;     // kmap_from_edges (kmap.cpp:317-336): WS lists only, kd = relations
    int words = 1;          // mask words of the full-width map
    int n_blocks = 0;       // query blocks (for per-block pair counts)
    sk::DevBuf os;          // rows_pad x kd int32
    sk::DevBuf masks;       // rows_pad x words u64
    sk::DevBuf blk_counts;  // n_blocks x kd int32
    sk::DevBuf ws_ptr;      // kd+1 int64 (exclusive scan of per-offset counts)
    sk::DevBuf blk_off;     // n_blocks x kd int64 (write cursor per block/offset)
    sk::DevBuf ws_in, ws_out;  // total_pairs (allocated at n_out*kd upper bound)
    sk::DevBuf ws_in_pad, ws_out_pad;  // per offset padded to 128-pair tiles, -1 pads
    bool has_ws = false;
    int64_t total_pairs_host = -1;
    // FOD/GGS tile schedule over WS lists: per offset first tile index
    sk::DevBuf ws_tile_ptr;    // kd+1 int32
    std::map<std::pair<int, int>, std::unique_ptr<sk::Prepared>> prepared;
    sk_kmap* transpose_cache = nullptr;  // owned
    std::mutex mu;
    sk::BuiltOn built_on;  // stream the map was built on (stream_after)
    sk::BuiltOn ws_on;     // stream the pair lists were built on
    ~sk_kmap() override;
};

namespace sk {

constexpr int kTileM = 128;  // MMA M rows per tile = pad multiple
constexpr int kTileWS = 256; // pairs per FOD/GGS tile (padded per offset)

// kmap.cu
void coords_build_table(sk_coords* c, cudaStream_t st);
void coords_validate(sk_coords* c, cudaStream_t st);
void coords_check_range(sk_ctx* ctx, const int32_t* d, int n, cudaStream_t st);
sk_coords* coords_downsample(sk_coords* in, const int32_t stride[3], cudaStream_t st);
// quantize (tensor.cpp:87-142): coordinates in first-appearance order and the
// output row of every point (optional); features reduced by DedupRule
sk_coords* coords_quantize(sk_ctx* ctx, int dims, int m, const double* raw, const int32_t* batch,
                           const double voxel[3], int32_t* point_rows, cudaStream_t st);
void quantize_features(int m, int channels, const double* feats, const int32_t* point_rows,
                       int n, int rule, sk_dtype dt, void* out, cudaStream_t st);
sk_kmap* kmap_build(sk_coords* in, sk_coords* out, int kernel, const int32_t stride[3],
                    int transposed, cudaStream_t st);
sk_kmap* kmap_transpose(sk_kmap* m, cudaStream_t st);
// build_kmap with per-axis (odd or even) kernel sizes and dilation (extension,
// SURVEY §8(f) rank 3); standard shapes delegate to kmap_build
sk_kmap* kmap_build_ex(sk_coords* in, sk_coords* out, const int32_t kernel[3],
                       const int32_t stride[3], const int32_t dilation[3], int transposed,
                       cudaStream_t st);
// kmap_from_edges (kmap.cpp:317-336): edges int32 [E][3] = (src, dst, relation)
// on the device; per relation, pairs stably sorted by dst (WS only)
sk_kmap* kmap_from_edges(sk_ctx* ctx, const int32_t* d_edges, int E, int relations, int n_in,
                         int n_out, cudaStream_t st);
void kmap_ensure_ws(sk_kmap* m, cudaStream_t st);
Prepared* kmap_prepare(sk_kmap* m, int splits, int pad, cudaStream_t st);
int64_t kmap_total_pairs(sk_kmap* m, cudaStream_t st);

// conv.cu
// w_kmajor (optional, forward only): W already transposed to [kd][c_out][c_in]
// residual (optional): y = conv(x) + residual, same shape as y (fused skip add)
// Builds, on st, the prepared OS map or the WS pair lists a forward
// conv_forward(m, cfg, dt, c_in, c_out) will read (nothing for the paths that
// read the raw map): lets the network runner build them ahead on its map stream.
void conv_forward_prepare(sk_ctx* ctx, sk_kmap* m, const sk_dataflow_cfg& cfg, sk_dtype dt,
                          int c_in, int c_out, cudaStream_t st);
// identity-map (K=1, stride 1) layers as a dense tcgen05 GEMM (dense.cu);
// b = [n_total][k_total] K-major; false = shape not handled
bool dense_identity_tc(sk_ctx* ctx, sk_dtype dt, long long rows, int k_total, int n_total,
                       const void* x, const void* b, void* y, const void* residual,
                       float* y_accum, int cta_n, cudaStream_t st);
void conv_forward(sk_ctx* ctx, sk_kmap* m, const sk_dataflow_cfg& cfg, sk_dtype dt, int c_in,
                  int c_out, const void* x, const void* w, void* y, bool dgrad, cudaStream_t st,
                  const void* w_kmajor = nullptr, const void* residual = nullptr,
                  float* y_accum = nullptr);
// y_accum (optional): ADD the result into this fp32 [n_out][n] buffer instead
// of writing y (training: dgrad straight into the input's gradient sum)
// W [kd][c_in][c_out] -> W^T [kd][c_out][c_in]
void transpose_weights(sk_dtype dt, const void* w, int kd, int c_in, int c_out, void* wt,
                       cudaStream_t st);
// accumulate: dw += (instead of dw =) the weight gradient
void conv_wgrad(sk_ctx* ctx, sk_kmap* m, const sk_dataflow_cfg& cfg, sk_dtype dt, int c_in,
                int c_out, const void* x, const void* dy, float* dw, cudaStream_t st,
                bool accumulate = false);

// sort.cu: hand-written scan / stable radix sort (no CUB)
// out[i] = sum in[0..i); *total_dev (optional, device) = sum of all n
void scan_exclusive_i32(const int* in, int* out, int n, int* total_dev, cudaStream_t st);
// stable LSD sort of (key, value) pairs on bits [begin_bit, end_bit); keys[0]
// / vals[0] hold the input, keys[1] / vals[1] scratch of the same size;
// returns the index (0 / 1) of the buffers holding the sorted result
template <typename KT>
int radix_sort_pairs(KT* keys[2], int* vals[2], int n, int begin_bit, int end_bit, cudaStream_t st);
// the same in steps, for callers that fuse the digit histogram into their key
// generation: plan, a zeroed scratch of scratch_words u32 (digit histograms
// [passes][digits] first, then the look-back status), run
struct RadixPlan {
    int bits = 0, passes = 0, dbits = 0, digits = 1, tiles = 0;
    size_t hist_words = 0, scratch_words = 0;
};
RadixPlan radix_plan(int n, int bits);
template <typename KT>
int radix_sort_run(KT* keys[2], int* vals[2], int n, int begin_bit, const RadixPlan& pl,
                   uint32_t* scratch, bool have_hist, cudaStream_t st);

uint64_t next_coord_set_id();
void set_last_error(const std::string& m);

}  // namespace sk
