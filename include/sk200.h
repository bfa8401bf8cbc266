/* sk200 — B200-native sparse-convolution engine: the drop-in C ABI.
 *
 * This header is the boundary a sparsekit caller binds to replace the CPU
 * hot path of the reference (namespace sparsekit, /root/reference/proj).
 * Each entry point names the reference interface it replaces (file:line).
 * The reference itself has no extern "C"/FFI layer; its
 * boundary is the C++ header API, so INTEGRATION.md shows the C++ shim a
 * maintainer adds to route those calls here.
 *
 * Conventions
 *  - Every function returns sk_status; details via sk_last_error() (per
 *    thread). No C++ exception crosses this ABI. The reference's
 *    ValidationError maps to SK_ERR_VALIDATION, ContractError to
 *    SK_ERR_CONTRACT (common.hpp:19-27).
 *  - All device pointers are caller-owned unless stated; handles
 *    (sk_coords, sk_kmap) are library-owned, reference counted, immutable
 *    after construction and usable from any stream after event sync
 *    (SparseTensor immutability, tensor.hpp:84-85).
 *  - Every call is stream-ordered on the `stream` argument (a cudaStream_t;
 *    NULL = legacy default stream). Calls never synchronise the device except
 *    where documented (output-coordinate counts, host exports).
 *  - Coordinates are int32[n][4] = (batch, x, y, z), z = 0 for dims = 2
 *    (Coord, tensor.hpp:15-20). Packable range: batch in [0, 4096),
 *    x/y/z in [-65536, 65536); outside it SK_ERR_VALIDATION.
 *  - Features are row-major [n][C]; weights are [K^D][C_in][C_out]
 *    row-major in offset order of OffsetSet (WeightTensor, exec.hpp:11-39).
 */
#ifndef SK200_H
#define SK200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SK_OK = 0,
    SK_ERR_VALIDATION = 1, /* sparsekit::ValidationError (common.hpp:19-22) */
    SK_ERR_CONTRACT = 2,   /* sparsekit::ContractError   (common.hpp:24-27) */
    SK_ERR_CUDA = 3,
    SK_ERR_NCCL = 4,
    SK_ERR_INTERNAL = 5
} sk_status;

/* SK_F64: quantize features only (the reference's f64 Features); conv paths
 * take F32 / F16 / BF16. */
typedef enum { SK_F32 = 0, SK_F16 = 1, SK_BF16 = 2, SK_F64 = 3 } sk_dtype;

/* DataflowKind (exec.hpp:59) */
typedef enum {
    SK_GATHER_GEMM_SCATTER = 0,
    SK_FETCH_ON_DEMAND = 1,
    SK_IMPLICIT_GEMM = 2
} sk_dataflow_kind;

/* ReorderMode (exec.hpp:60) */
typedef enum { SK_REORDER_OFFLINE = 0, SK_REORDER_ONLINE = 1 } sk_reorder;

/* TilePreset (exec.hpp:46-54) re-read for the tcgen05 gathered GEMM
 * (SURVEY App. A.8); the tuner's space (sk_tune_space_entry) holds the
 * reference's two presets plus the B200 variants below:
 *   cta_m      128: 128-row MMA tiles in 256-row items, two CTAs per SM
 *              (8 gather warps each) when C_out <= 128 and stages fit;
 *              256: one CTA per SM (16 gather warps, ~200 KB of stages);
 *              64: implicit GEMM work items of ONE 128-row tile (twice the
 *              items: small layers spread over more SMs)
 *   cta_n      C_out tile (multiple of 16, <= 256; 0 = whole C_out)
 *   cta_k      channels per pipeline stage: 0 = auto (64/32/16 dividing
 *              C_in; C_in = 96 as three 32-channel slabs), 16 / 32 / 64 =
 *              that single-slab step when it divides C_in
 *   warp_rows  lockstep rows of the cost model (traffic_model)
 *   load_width 4 = cp.async row gathers (16 B per lane); 1 = TMA
 *              tile::gather4 (one tensor-map gather per 4 rows) */
typedef struct {
    int cta_m, cta_n, cta_k, warp_rows, load_width;
} sk_tile;

/* DataflowConfig (exec.hpp:65-73) */
typedef struct {
    int kind;    /* sk_dataflow_kind */
    int splits;  /* 0 = unsorted; implicit GEMM only */
    sk_tile tile;
    int reorder; /* sk_reorder */
} sk_dataflow_cfg;

typedef struct sk_ctx sk_ctx;
typedef struct sk_coords sk_coords;
typedef struct sk_kmap sk_kmap;

typedef struct {
    int dims, kernel_size, num_offsets, n_in, n_out, transposed;
    int stride[3];
    int64_t total_pairs; /* KernelMapWS::total_pairs (kmap.hpp:51-55); syncs */
} sk_kmap_info;

/* ---- errors / context ---------------------------------------------------- */
const char* sk_last_error(void);
const char* sk_version(void);
/* number of device kernels this library has launched (diagnostic) */
uint64_t sk_kernel_launches(void);
/* One context per device; owns the stream-ordered memory pool and the
 * kernel-map cache (MapCache, kmap.hpp:159-176). */
sk_status sk_ctx_create(int device, sk_ctx** out);
sk_status sk_ctx_destroy(sk_ctx* ctx);
/* Deterministic mode (ExecContext::deterministic, common.hpp:29-32): every
 * dataflow accumulates splits/offsets in a fixed order (no float atomics). */
sk_status sk_ctx_set_deterministic(sk_ctx* ctx, int on);
/* Stride-1 3-D K = 3 / 5 kernel maps over input sets of at least min_rows
 * voxels are queried through a 4x4x4 block index (default 1 << 16; a tuning
 * knob of the build, results are identical either way). */
sk_status sk_ctx_set_kmap_block_rows(sk_ctx* ctx, int min_rows);

/* ---- coordinate sets (SparseTensor coords + CoordLookup) ------------------ */
/* SparseTensor(dims, coords, ...) / coords_only (tensor.hpp:89-92) and the
 * CoordLookup hash (tensor.hpp:118-130, tensor.cpp:80-85): copies d_coords,
 * validates the packable range, assigns a process-unique id (coord_set_id,
 * tensor.cpp:26-29) and builds the device hash table once. */
sk_status sk_coords_create(sk_ctx* ctx, int dims, int n, const int32_t* d_coords,
                           const int32_t stride_tag[3], void* stream, sk_coords** out);
/* Same from host memory (copies H2D on `stream`). */
sk_status sk_coords_create_host(sk_ctx* ctx, int dims, int n, const int32_t* h_coords,
                                const int32_t stride_tag[3], void* stream, sk_coords** out);
sk_status sk_coords_retain(sk_coords* c);
/* Release (refcounted). Device buffers return to the stream-ordered pool on
 * the stream that built them; a set or map also used from OTHER streams must
 * be released after that work completes (the usual stream-ordered lifetime
 * rule; readers on other streams are ordered after the build automatically). */
sk_status sk_coords_release(sk_coords* c);
int sk_coords_n(const sk_coords* c);
int sk_coords_dims(const sk_coords* c);
uint64_t sk_coords_id(const sk_coords* c);
const int32_t* sk_coords_device_ptr(const sk_coords* c);
sk_status sk_coords_stride_tag(const sk_coords* c, int32_t out[3]);
/* D2H copy of the coordinates (syncs `stream`). */
sk_status sk_coords_export(const sk_coords* c, int32_t* h_coords, void* stream);

/* quantize (tensor.cpp:87-142, the step before the path): floor(raw / voxel)
 * per axis (toward -inf), first-appearance dedup (emplace order). d_raw:
 * device double[m][dims]; d_batch: device int32[m] or NULL (batch 0);
 * d_point_rows (optional, device int32[m]) receives each point's output row.
 * Non-finite input or a voxel outside the packable range -> SK_ERR_VALIDATION.
 * Reads back the output count (one sync). */
sk_status sk_quantize(sk_ctx* ctx, int dims, int m, const double* d_raw, const int32_t* d_batch,
                      const double voxel[3], void* stream, sk_coords** out,
                      int32_t* d_point_rows);
/* Features of a quantized set (DedupRule, tensor.hpp:45): rule 0 = first
 * (the first point's features), 1 = mean; channels 0 = one occupancy channel
 * of ones. d_feats: device double[m][channels]; d_out: device [n][max(1,
 * channels)] of dtype (caller-owned). */
sk_status sk_quantize_features(sk_ctx* ctx, int m, int channels, const double* d_feats,
                               const int32_t* d_point_rows, int n, int rule, sk_dtype dtype,
                               void* d_out, void* stream);

/* build_out_coords (kmap.cpp:73-94): stride 1 returns the same set
 * (retained); stride > 1 returns unique(floor_div(p, s)) in first-appearance
 * order, stride_tag *= s. Reads back the output count (one sync). Cached per
 * (input id, stride). */
sk_status sk_out_coords(sk_ctx* ctx, sk_coords* in, const int32_t stride[3], void* stream,
                        sk_coords** out);

/* ---- kernel maps ------------------------------------------------------------ */
/* build_kmap_os / build_kmap_ws (kmap.cpp:96-143) + compute_masks
 * (kmap.cpp:34-47): device OS matrix n_out x K^D (-1 sentinel), per-row
 * big-endian masks, per-offset pair counts; the WS pair lists (ascending
 * out row per offset) are derived on first use. transposed = 1 builds the
 * map of the transposed convolution directly (kmap.cpp:124-129). Cached in
 * the context by MapKey (kmap.hpp:99-107). Odd kernel only, K <= 5. */
sk_status sk_kmap_build(sk_ctx* ctx, sk_coords* in, sk_coords* out, int kernel_size,
                        const int32_t stride[3], int transposed, void* stream, sk_kmap** map);
/* EXTENSION beyond the reference (the reference accepts
 * odd symmetric K only and has no dilation): per-axis kernel sizes in [1, 8]
 * (odd or even; axis offsets dil * (lo .. lo+k-1), lo = -((k-1)/2), i.e.
 * {-1,0,1} for 3 and {0,1} for 2 as in MinkowskiEngine / TorchSparse) and
 * dilation per axis; kernel volume <= 128; lexicographic offset order.
 * Standard shapes return the same cached map as sk_kmap_build. */
sk_status sk_kmap_build_ex(sk_ctx* ctx, sk_coords* in, sk_coords* out, const int32_t kernel[3],
                           const int32_t stride[3], const int32_t dilation[3], int transposed,
                           void* stream, sk_kmap** map);
/* kmap_from_edges (kmap.cpp:317-336): a graph (R-GCN) map over relations.
 * d_edges: device int32[E][3] = (src, dst, relation); per relation the pairs
 * are stably sorted by dst. WS form only: forward through GGS / FOD and
 * wgrad; implicit GEMM, prepare, OS export, transpose and dgrad raise
 * SK_ERR_CONTRACT like the reference ("graph maps cannot be transposed"). Out-of-range ids ->
 * SK_ERR_VALIDATION (one sync). */
sk_status sk_kmap_from_edges(sk_ctx* ctx, const int32_t* d_edges, int num_edges,
                             int num_relations, int n_in, int n_out, void* stream, sk_kmap** out);
/* transpose_map (kmap.cpp:290-315): swap (in, out), mirror offsets. */
sk_status sk_kmap_transpose(sk_ctx* ctx, sk_kmap* map, void* stream, sk_kmap** out);
/* split_and_sort + pad_map (kmap.cpp:211-288), i.e. prepare_os_map
 * (exec.cpp:342-344). Cached on the map per (splits, pad_multiple). */
sk_status sk_kmap_prepare(sk_ctx* ctx, sk_kmap* map, int splits, int pad_multiple,
                          void* stream);
sk_status sk_kmap_retain(sk_kmap* map);
sk_status sk_kmap_release(sk_kmap* map);
sk_status sk_kmap_get_info(sk_kmap* map, void* stream, sk_kmap_info* info);

/* Host exports for parity (test-only, sync `stream`). */
sk_status sk_kmap_export_os(sk_kmap* map, int32_t* h_entries, uint64_t* h_masks, void* stream);
/* WS CSR: h_ptr[K^D+1], then pairs (in, out) per offset, ascending out. */
sk_status sk_kmap_export_ws(sk_kmap* map, int64_t* h_ptr, int32_t* h_in, int32_t* h_out,
                            void* stream);
/* One prepared split: begin/end offsets, padded row count, then
 * entries rows x (end-begin), out_row rows, masks rows x words. Pass NULL
 * data pointers to query sizes only. */
sk_status sk_kmap_export_split(sk_kmap* map, int splits, int pad_multiple, int s, int* begin,
                               int* end, int* n_rows, int* mask_words, int32_t* h_entries,
                               int32_t* h_out_row, uint64_t* h_masks, void* stream);

/* ---- dataflows (exec.hpp:86-124) ---------------------------------------------
 * dtype: SK_F16/SK_BF16 -> tcgen05 tensor cores (fp32 accumulate in TMEM);
 * SK_F32 -> fp32 SIMT path (the 1e-5 parity path). x: [n_in][c_in],
 * w: [K^D][c_in][c_out], y: [n_out][c_out], all `dtype`. Kernels are launched
 * with programmatic stream serialization (each waits for its predecessor on
 * the stream before touching memory; a runner turns this off with
 * sk_net_set_pdl, direct calls always use it): ordering and results are those
 * of plain stream order. */

/* conv_forward (exec.cpp:368-383) — dispatches on cfg->kind; implicit GEMM
 * with reorder=offline prepares (cached) the map for cfg->splits. */
sk_status sk_conv_forward(sk_ctx* ctx, sk_kmap* map, const sk_dataflow_cfg* cfg, sk_dtype dtype,
                          int c_in, int c_out, const void* d_x, const void* d_w, void* d_y,
                          void* stream);
/* conv_dgrad (exec.cpp:385-396): dx = dy through the transposed map with
 * mirrored, transposed weights. dy: [n_out][c_out] -> dx: [n_in][c_in]. */
sk_status sk_conv_dgrad(sk_ctx* ctx, sk_kmap* map, const sk_dataflow_cfg* cfg, sk_dtype dtype,
                        int c_in, int c_out, const void* d_dy, const void* d_w, void* d_dx,
                        void* stream);
/* conv_wgrad (exec.cpp:398-414): dW_k = sum over pairs x_j^T dy_q.
 * dw is fp32 [K^D][c_in][c_out] (master gradient), overwritten. */
sk_status sk_conv_wgrad(sk_ctx* ctx, sk_kmap* map, const sk_dataflow_cfg* cfg, sk_dtype dtype,
                        int c_in, int c_out, const void* d_x, const void* d_dy, float* d_dw,
                        void* stream);

/* ---- cost model (cost.hpp:31-62) ---------------------------------------------
 * count_macs over the map prepared for (splits, pad) with warp_rows rows in
 * lockstep (cost.cpp:7-30); syncs. */
sk_status sk_kmap_count_macs(sk_kmap* map, int splits, int pad_multiple, int warp_rows,
                             int c_in, int c_out, int64_t* effective, int64_t* redundant,
                             void* stream);

/* ---- NetworkRunner (network.hpp:81-119) + autotuner (tuner.hpp) ----------
 * Spec text: one layer per line "name kind c_in c_out kernel stride inputs
 * transpose_of" (kind conv|conv_transposed, inputs comma list or "-",
 * transpose_of name or "-"), the LayerSpec fields of network.hpp:20-33.
 * Weights live on the device in `dtype`, [K^D][c_in][c_out] per layer. */
typedef struct sk_net sk_net;
sk_status sk_net_create(sk_ctx* ctx, int dims, const char* spec_text, sk_dtype dtype,
                        sk_net** out);
sk_status sk_net_destroy(sk_net* net);
int sk_net_num_layers(const sk_net* net);
/* partition_groups (network.cpp:141-158): map-sharing groups */
int sk_net_num_groups(const sk_net* net);
int sk_net_group_of_layer(const sk_net* net, int layer);
sk_status sk_net_layer_info(const sk_net* net, int layer, int* num_offsets, int* c_in,
                            int* c_out, int64_t* wgrad_offset);
int64_t sk_net_num_params(const sk_net* net);
/* device weight buffer of a layer (write it with cudaMemcpy / kernels).
 * Calling this marks the runner's cached transposed weights stale. */
sk_status sk_net_weight_ptr(sk_net* net, int layer, void** ptr);
/* GroupConfig (network.hpp:54-58): phase 0 forward, 1 dgrad, 2 wgrad */
sk_status sk_net_set_config(sk_net* net, int group, int phase, const sk_dataflow_cfg* cfg);
sk_status sk_net_get_config(const sk_net* net, int group, int phase, sk_dataflow_cfg* cfg);
/* NetworkRunner::forward (network.cpp:392): maps are built once per input
 * coordinate set and group, then cached. d_out is library-owned (valid until
 * the next forward). mapping_ms / kernel_ms: per-group CUDA-event timing
 * (RunStats), NULL to skip (no sync). */
sk_status sk_net_forward(sk_net* net, sk_coords* in, const void* d_feats, int channels,
                         void* stream, const void** d_out, int* n_out, double* mapping_ms,
                         double* kernel_ms);
sk_status sk_net_layer_output(sk_net* net, int layer, const void** d_out, int* rows);
/* forward with per-layer GPU milliseconds (CUDA events, one sync at the end)
 * and the total map-building time */
sk_status sk_net_forward_profiled(sk_net* net, sk_coords* in, const void* d_feats, int channels,
                                  void* stream, double* layer_ms, double* mapping_ms_total);
/* NetworkRunner::measure_ms (network.cpp:398-438) */
sk_status sk_net_measure(sk_net* net, sk_coords* in, const void* d_feats, int channels,
                         int forward, int dgrad, int wgrad, void* stream, double* ms);
int64_t sk_net_map_builds(const sk_net* net);
/* Overlapped map build (default on): a forward on a new coordinate set builds
 * each layer's maps on a runner-owned stream from a helper host thread while
 * the convs run on the caller's stream (kernel-map readback syncs stall only
 * the helper). Turn off when several runners are already in flight on one GPU
 * (they fill each other's sync bubbles). No reference counterpart (sk200
 * runtime). */
sk_status sk_net_set_overlap(sk_net* net, int on);
/* Programmatic dependent launch (default on): every kernel of the runner's
 * calls is launched with programmatic stream serialization, so its launch
 * and prologue overlap the previous kernel's tail (griddepcontrol.wait
 * before it touches memory): -5 % single-scan latency on MinkUNet. Turn off
 * when several runners share the GPU: early-resident CTAs waiting on their
 * predecessor hold shared memory other streams' kernels could use (-7 %
 * scans/s at 6 in flight). No reference counterpart (sk200 runtime). */
sk_status sk_net_set_pdl(sk_net* net, int on);
/* Cold-map tuning (default off = the reference's tuner: every probe runs on
 * the tuning set's cached maps). On: every forward-only probe (inference
 * tuning, training = 0, and the forward pass of sparse_mapping) runs on a
 * fresh copy of the coordinate set, so a candidate's map preparation (split +
 * sort, pair lists) is timed with its convolutions -- the objective of a
 * workload whose maps are new every scan; probes that include dgrad / wgrad
 * keep the cached maps. Same call counts. No reference counterpart (sk200
 * runtime). */
sk_status sk_net_set_tune_cold(sk_net* net, int on);
/* modeled_group_traffic (network.cpp:453-471) */
sk_status sk_net_group_traffic(sk_net* net, int group, const sk_dataflow_cfg* cfg, void* stream,
                               double* bytes);
/* Chained backward of the last forward over layers [layer_lo, layer_hi]
 * (call with decreasing ranges to overlap gradient all-reduce buckets).
 * accumulate != 0 adds into d_wgrad_flat (several scans per rank). */
sk_status sk_net_backward(sk_net* net, const void* d_grad_out, float* d_wgrad_flat, int layer_hi,
                          int layer_lo, int accumulate, void* stream);
/* tune_inference / tune_training (tuner.cpp:134-220): training 0 =
 * inference, 1 = workload_pattern, 2 = sparse_mapping. Log entries are
 * {pass, group, space index, ms}. Leaves the winning configs set. */
sk_status sk_net_tune(sk_net* net, sk_coords* in, const void* d_feats, int channels,
                      int training, int warmup, int runs, void* stream, double* latency_ms,
                      double* log, int log_cap, int* log_len);
/* default_space (tuner.cpp:9-26): GGS, FOD, implicit GEMM x splits 0..4 x
 * {small, large} */
int sk_tune_space_size(void);
sk_status sk_tune_space_entry(int i, sk_dataflow_cfg* cfg);

#ifdef __cplusplus
}
#endif
#endif /* SK200_H */
