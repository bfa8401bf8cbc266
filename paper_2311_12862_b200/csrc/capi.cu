#include <functional>
// sk200 C ABI (include/sk200.h): handle lifetimes, error mapping, caches.
// No C++ exception crosses this boundary.
#include <cstring>

#include "sk_internal.hpp"

namespace {
thread_local std::string g_last_error;

template <class F>
sk_status guard(F&& f) {
    try {
        f();
        return SK_OK;
    } catch (const sk::Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return SK_ERR_INTERNAL;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return SK_ERR_INTERNAL;
    }
}

inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

}  // namespace

namespace sk {
void set_last_error(const std::string& m) { g_last_error = m; }
std::atomic<unsigned long long>& launch_counter() {
    static std::atomic<unsigned long long> c{0};
    return c;
}
bool& pdl_enabled() {
    thread_local bool on = true;
    return on;
}

namespace {
__global__ void k_fill_bytes(uint8_t* __restrict__ p, size_t bytes, uint32_t word) {
    pdl_wait();
    pdl_trigger();
    const size_t n16 = bytes / 16;
    const int4 v = make_int4((int)word, (int)word, (int)word, (int)word);
    const size_t i0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    int4* q = reinterpret_cast<int4*>(p);
    for (size_t i = i0; i < n16; i += (size_t)gridDim.x * blockDim.x) q[i] = v;
    if (i0 < bytes - n16 * 16) p[n16 * 16 + i0] = (uint8_t)word;
}
}  // namespace

void fill_async(void* p, int byte, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return;
    // the kernel only where PDL chains the launches (one scan at a time) and
    // the fill is small; replicated runners (no PDL) keep the memset, which
    // the copy engine runs without waiting for SM slots behind other
    // streams' persistent kernels (measured: kernels everywhere cost 2-3 %
    // scans/s at 8 in flight)
    if (!pdl_enabled() || bytes > (1u << 20) || reinterpret_cast<uintptr_t>(p) % 16 != 0) {
        SK_CUDA(cudaMemsetAsync(p, byte, bytes, st));
        return;
    }
    const uint32_t word = 0x01010101u * (uint32_t)(byte & 0xFF);
    const int64_t blocks = std::min<int64_t>(std::max<int64_t>(ceil_div((int64_t)(bytes / 16), 256), 1),
                                             148 * 8);
    launch_pdl(k_fill_bytes, (int)blocks, 256, 0, st, (uint8_t*)p, bytes, word);
}

void stream_after(const BuiltOn& on, cudaStream_t st) {
    if (!on.set || on.s == st) return;
    cudaEvent_t ev;
    SK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    SK_CUDA(cudaEventRecord(ev, on.s));
    SK_CUDA(cudaStreamWaitEvent(st, ev, 0));
    SK_CUDA(cudaEventDestroy(ev));  // released once the recorded work completes
}

void ensure_smem(const void* kern, size_t smem) {
    static std::mutex mu;
    static std::map<const void*, size_t> done;
    std::lock_guard<std::mutex> g(mu);
    size_t& have = done[kern];
    if (smem > have) {
        SK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        have = smem;
    }
}

namespace {
// 4 size classes per octave (<= 25% slack), 4 KB minimum
size_t size_class(size_t n) {
    if (n <= 4096) return 4096;
    const int b = 63 - __builtin_clzll((unsigned long long)(n - 1));
    const size_t q = (size_t)1 << (b - 2);
    return (n + q - 1) / q * q;
}
struct BlockCache {
    std::mutex mu;
    std::map<std::pair<cudaStream_t, size_t>, std::vector<void*>> free;
    size_t cached = 0;
    size_t cap = [] {
        const char* e = getenv("SK_CACHE_MB");
        return (size_t)(e ? atol(e) : 32768) << 20;
    }();
};
BlockCache& block_cache() {
    static BlockCache* c = new BlockCache();  // never destroyed: no frees after CUDA teardown
    return *c;
}
}  // namespace

void* cache_alloc(size_t n, cudaStream_t s) {
    const size_t c = size_class(n);
    BlockCache& bc = block_cache();
    {
        std::lock_guard<std::mutex> g(bc.mu);
        auto it = bc.free.find({s, c});
        if (it != bc.free.end() && !it->second.empty()) {
            void* p = it->second.back();
            it->second.pop_back();
            bc.cached -= c;
            return p;
        }
    }
    void* p = nullptr;
    if (cudaMallocAsync(&p, c, s) != cudaSuccess) {
        (void)cudaGetLastError();
        cache_trim();  // give the cached blocks back to the pool and retry once
        SK_CUDA(cudaDeviceSynchronize());
        SK_CUDA(cudaMallocAsync(&p, c, s));
    }
    return p;
}

void cache_free(void* p, size_t n, cudaStream_t s) {
    const size_t c = size_class(n);
    BlockCache& bc = block_cache();
    {
        std::lock_guard<std::mutex> g(bc.mu);
        if (bc.cached + c <= bc.cap) {
            bc.free[{s, c}].push_back(p);
            bc.cached += c;
            return;
        }
    }
    cudaFreeAsync(p, s);
}

void cache_trim() {
    BlockCache& bc = block_cache();
    std::lock_guard<std::mutex> g(bc.mu);
    for (auto& kv : bc.free)
        for (void* p : kv.second) cudaFreeAsync(p, kv.first.first);
    bc.free.clear();
    bc.cached = 0;
}

namespace {
struct RbArgs {
    const uint8_t* src[4];
    int bytes[4];
    int n;
};
__global__ void k_read_back(RbArgs a, volatile uint8_t* dst) {
    pdl_wait();
    pdl_trigger();
    int o = 0;
    for (int k = 0; k < a.n; ++k) {
        for (int i = threadIdx.x; i < a.bytes[k]; i += blockDim.x) dst[o + i] = a.src[k][i];
        o += a.bytes[k];
    }
}
struct Mapped {
    uint8_t* h = nullptr;
    uint8_t* d = nullptr;
    std::atomic<unsigned> next{0};
};
constexpr int kRbSlots = 256, kRbSlotBytes = 64;
Mapped& mapped() {
    static Mapped* m = [] {
        auto* r = new Mapped();
        SK_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&r->h), kRbSlots * kRbSlotBytes,
                              cudaHostAllocMapped));
        SK_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&r->d), r->h, 0));
        return r;
    }();
    return *m;
}
}  // namespace

void read_back(cudaStream_t st, std::initializer_list<RbSeg> segs, void* dst) {
    RbArgs a{};
    size_t total = 0;
    for (const RbSeg& g : segs) {
        validate(a.n < 4, "read_back: too many segments");
        a.src[a.n] = static_cast<const uint8_t*>(g.src);
        a.bytes[a.n++] = (int)g.bytes;
        total += g.bytes;
    }
    validate(total <= (size_t)kRbSlotBytes, "read_back: too many bytes");
    Mapped& m = mapped();
    const unsigned slot = m.next.fetch_add(1) % kRbSlots;
    launch_pdl(k_read_back, 1, 32, 0, st, a, m.d + slot * kRbSlotBytes);
    SK_CUDA(cudaStreamSynchronize(st));
    memcpy(dst, m.h + slot * kRbSlotBytes, total);
}
}  // namespace sk

namespace {

void release_coords(sk_coords* c);
void release_kmap(sk_kmap* m);

}  // namespace

sk_coords::~sk_coords() {
    for (auto& kv : maps) release_kmap(kv.second);
    for (auto& kv : down) release_coords(kv.second);
}

sk_kmap::~sk_kmap() {
    if (transpose_cache) release_kmap(transpose_cache);
}

namespace {
void release_coords(sk_coords* c) {
    if (c && c->refs.fetch_sub(1) == 1) delete c;
}
void release_kmap(sk_kmap* m) {
    if (m && m->refs.fetch_sub(1) == 1) delete m;
}

// One prepared split as row-major rows_pad x w on the host (the device keeps
// it tile-column-major, see kmap.cu k_split_reorder).
std::vector<int32_t> split_rows_host(sk::Prepared* p, int s, cudaStream_t st) {
    const int b = p->begin[s], w = p->begin[s + 1] - b;
    std::vector<int32_t> dev((size_t)p->rows_pad * w), rows((size_t)p->rows_pad * w);
    if (!dev.empty())
        SK_CUDA(cudaMemcpyAsync(dev.data(), p->entries.as<int32_t>() + (size_t)p->rows_pad * b,
                                dev.size() * 4, cudaMemcpyDeviceToHost, st));
    SK_CUDA(cudaStreamSynchronize(st));
    for (int r = 0; r < p->rows_pad; ++r)
        for (int j = 0; j < w; ++j)
            rows[(size_t)r * w + j] =
                dev[((size_t)(r / sk::kTileM) * w + j) * sk::kTileM + (r % sk::kTileM)];
    return rows;
}

sk_coords* make_coords(sk_ctx* ctx, int dims, int n, const int32_t* src, bool host,
                       const int32_t* stride_tag, cudaStream_t st) {
    sk::validate(ctx != nullptr, "null context");
    sk::validate(dims == 2 || dims == 3, "dims must be 2 or 3");
    sk::validate(n >= 0, "negative coordinate count");
    auto* c = new sk_coords();
    try {
        c->ctx = ctx;
        c->dims = dims;
        c->n = n;
        c->id = sk::next_coord_set_id();
        for (int d = 0; d < 3; ++d) c->stride_tag[d] = stride_tag ? stride_tag[d] : 1;
        c->coords.alloc((size_t)std::max(n, 1) * 16, st);
        if (n)
            SK_CUDA(cudaMemcpyAsync(c->coords.p, src, (size_t)n * 16,
                                    host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
        sk::coords_validate(c, st);  // the packable range; the hash table is built on first use
    } catch (...) {
        delete c;
        throw;
    }
    return c;
}
}  // namespace

extern "C" {

const char* sk_last_error(void) { return g_last_error.c_str(); }
const char* sk_version(void) { return "sk200 0.1 (sm_100a)"; }
uint64_t sk_kernel_launches(void) { return sk::launch_counter().load(); }

sk_status sk_ctx_create(int device, sk_ctx** out) {
    return guard([&] {
        sk::validate(out != nullptr, "null output pointer");
        SK_CUDA(cudaSetDevice(device));
        auto* c = new sk_ctx();
        c->device = device;
        cudaDeviceProp prop;
        SK_CUDA(cudaGetDeviceProperties(&prop, device));
        c->num_sms = prop.multiProcessorCount;
        c->smem_optin = prop.sharedMemPerBlockOptin;
        SK_CUDA(cudaMalloc(&c->sched, sk_ctx::kSchedSlots * 2 * sizeof(int)));
        SK_CUDA(cudaMemset(c->sched, 0, sk_ctx::kSchedSlots * 2 * sizeof(int)));
        // keep freed blocks in the stream-ordered pool (no cudaFree syncs)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t thr = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            // pre-grow the pool once so steady-state scans never map new
            // memory: growing it mid-run blocked the whole device for
            // 10-100 ms per cudaMallocAsync (several runners in flight)
            // (capped at a third of the free memory, so a shared GPU or a
            // second process still has room; a failed grow is harmless and
            // must not leave the runtime's sticky last error set)
            const char* pg = getenv("SK_POOL_MB");
            size_t grow = (size_t)(pg ? atol(pg) : 24576) << 20;
            size_t free_b = 0, total_b = 0;
            if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) grow = std::min(grow, free_b / 3);
            else (void)cudaGetLastError();
            void* p = nullptr;
            if (grow && cudaMallocAsync(&p, grow, nullptr) == cudaSuccess) cudaFreeAsync(p, nullptr);
            else (void)cudaGetLastError();
            cudaStreamSynchronize(nullptr);
            (void)cudaGetLastError();
        }
        *out = c;
    });
}

sk_status sk_ctx_destroy(sk_ctx* ctx) {
    return guard([&] {
        if (ctx && ctx->sched) {
            cudaDeviceSynchronize();
            cudaFree(ctx->sched);
        }
        delete ctx;
    });
}

sk_status sk_ctx_set_deterministic(sk_ctx* ctx, int on) {
    return guard([&] {
        sk::validate(ctx != nullptr, "null context");
        ctx->deterministic = on != 0;
    });
}

sk_status sk_ctx_set_kmap_block_rows(sk_ctx* ctx, int min_rows) {
    return guard([&] {
        sk::validate(ctx != nullptr, "null context");
        sk::validate(min_rows >= 0, "min_rows must be >= 0");
        ctx->kmap_block_rows = min_rows;
    });
}

sk_status sk_coords_create(sk_ctx* ctx, int dims, int n, const int32_t* d_coords,
                           const int32_t stride_tag[3], void* stream, sk_coords** out) {
    return guard([&] { *out = make_coords(ctx, dims, n, d_coords, false, stride_tag, S(stream)); });
}

sk_status sk_coords_create_host(sk_ctx* ctx, int dims, int n, const int32_t* h_coords,
                                const int32_t stride_tag[3], void* stream, sk_coords** out) {
    return guard([&] { *out = make_coords(ctx, dims, n, h_coords, true, stride_tag, S(stream)); });
}

sk_status sk_quantize(sk_ctx* ctx, int dims, int m, const double* d_raw, const int32_t* d_batch,
                      const double voxel[3], void* stream, sk_coords** out,
                      int32_t* d_point_rows) {
    return guard([&] {
        sk::validate(ctx && out && voxel, "null argument");
        sk::validate(m == 0 || d_raw, "null raw points");
        *out = sk::coords_quantize(ctx, dims, m, d_raw, d_batch, voxel, d_point_rows, S(stream));
        (*out)->built_on.mark(S(stream));
    });
}

sk_status sk_quantize_features(sk_ctx* ctx, int m, int channels, const double* d_feats,
                               const int32_t* d_point_rows, int n, int rule, sk_dtype dtype,
                               void* d_out, void* stream) {
    return guard([&] {
        sk::validate(ctx != nullptr, "null context");
        sk::validate(n == 0 || d_out, "null output");
        sk::validate(channels == 0 || n == 0 || d_feats, "null features");
        sk::quantize_features(m, channels, d_feats, d_point_rows, n, rule, dtype, d_out, S(stream));
    });
}

sk_status sk_coords_retain(sk_coords* c) {
    return guard([&] {
        sk::validate(c != nullptr, "null coords");
        c->refs.fetch_add(1);
    });
}

sk_status sk_coords_release(sk_coords* c) {
    return guard([&] { release_coords(c); });
}

int sk_coords_n(const sk_coords* c) { return c ? c->n : -1; }
int sk_coords_dims(const sk_coords* c) { return c ? c->dims : -1; }
uint64_t sk_coords_id(const sk_coords* c) { return c ? c->id : 0; }
const int32_t* sk_coords_device_ptr(const sk_coords* c) {
    return c ? c->coords.as<const int32_t>() : nullptr;
}

sk_status sk_coords_stride_tag(const sk_coords* c, int32_t out[3]) {
    return guard([&] {
        sk::validate(c != nullptr, "null coords");
        for (int d = 0; d < 3; ++d) out[d] = c->stride_tag[d];
    });
}

sk_status sk_coords_export(const sk_coords* c, int32_t* h, void* stream) {
    return guard([&] {
        if (c->n)
            SK_CUDA(cudaMemcpyAsync(h, c->coords.p, (size_t)c->n * 16, cudaMemcpyDeviceToHost,
                                    S(stream)));
        SK_CUDA(cudaStreamSynchronize(S(stream)));
    });
}

sk_status sk_out_coords(sk_ctx* ctx, sk_coords* in, const int32_t stride[3], void* stream,
                        sk_coords** out) {
    return guard([&] {
        sk::validate(ctx && in && out, "null argument");
        for (int d = 0; d < in->dims; ++d)
            sk::validate(stride[d] >= 1, "stride components must be >= 1");
        bool unit = true;
        for (int d = 0; d < in->dims; ++d) unit = unit && stride[d] == 1;
        if (unit) {  // submanifold: the same coordinate set (kmap.cpp:75-79)
            in->refs.fetch_add(1);
            *out = in;
            return;
        }
        auto key = std::make_tuple(stride[0], stride[1], in->dims == 3 ? stride[2] : 1);
        std::lock_guard<std::mutex> lock(in->mu);
        auto it = in->down.find(key);
        if (it == in->down.end()) {
            sk::stream_after(in->built_on, S(stream));
            sk_coords* c = sk::coords_downsample(in, stride, S(stream));
            c->built_on.mark(S(stream));
            it = in->down.emplace(key, c).first;
        }
        sk::stream_after(it->second->built_on, S(stream));
        it->second->refs.fetch_add(1);
        *out = it->second;
    });
}

namespace {
// MapCache (kmap.cpp:359-391): one build per key; kcode = K for the standard
// odd symmetric kernels, 256 + (kx | ky << 4 | kz << 8) for generalized ones
sk_kmap* cached_map(sk_coords* in, sk_coords* out, int kcode, const int32_t stride[3],
                    int transposed, int dcode, cudaStream_t st,
                    const std::function<sk_kmap*()>& build) {
    auto key = std::make_tuple(out->id, kcode, stride[0], stride[1],
                               in->dims == 3 ? stride[2] : 1, transposed ? 1 : 0, dcode);
    sk_kmap* m = nullptr;
    {
        std::lock_guard<std::mutex> lock(in->mu);
        auto it = in->maps.find(key);
        if (it != in->maps.end()) m = it->second;
    }
    if (!m) {
        sk::stream_after(in->built_on, st);  // sets built lazily on another stream
        sk::stream_after(out->built_on, st);
        sk_kmap* built = build();
        built->built_on.mark(st);
        std::lock_guard<std::mutex> lock(in->mu);
        auto ins = in->maps.emplace(key, built);
        if (!ins.second) release_kmap(built);  // lost a race: builds once per key
        m = ins.first->second;
    }
    sk::stream_after(m->built_on, st);
    m->refs.fetch_add(1);
    return m;
}
}  // namespace

sk_status sk_kmap_build(sk_ctx* ctx, sk_coords* in, sk_coords* out, int kernel_size,
                        const int32_t stride[3], int transposed, void* stream, sk_kmap** map) {
    return guard([&] {
        sk::validate(ctx && in && out && map, "null argument");
        *map = cached_map(in, out, kernel_size, stride, transposed, 0, S(stream), [&] {
            return sk::kmap_build(in, out, kernel_size, stride, transposed, S(stream));
        });
    });
}

sk_status sk_kmap_build_ex(sk_ctx* ctx, sk_coords* in, sk_coords* out, const int32_t kernel[3],
                           const int32_t stride[3], const int32_t dilation[3], int transposed,
                           void* stream, sk_kmap** map) {
    return guard([&] {
        sk::validate(ctx && in && out && map && kernel && stride && dilation, "null argument");
        const int dims = in->dims;
        const int kz = dims == 3 ? kernel[2] : 1, dz = dims == 3 ? dilation[2] : 1;
        for (int d = 0; d < dims; ++d)
            sk::validate(kernel[d] >= 1 && kernel[d] <= 8 && dilation[d] >= 1 && dilation[d] < 1024,
                         "kernel sizes must be in [1, 8] and dilations in [1, 1024)");
        const bool standard = kernel[0] == kernel[1] && kernel[1] == kz && kernel[0] % 2 == 1 &&
                              kernel[0] <= 5 && dilation[0] == 1 && dilation[1] == 1 && dz == 1;
        const int kcode = standard ? kernel[0] : 256 + (kernel[0] | kernel[1] << 4 | kz << 8);
        const int dcode = standard ? 0 : (dilation[0] | dilation[1] << 10 | dz << 20);
        *map = cached_map(in, out, kcode, stride, transposed, dcode, S(stream), [&] {
            return sk::kmap_build_ex(in, out, kernel, stride, dilation, transposed, S(stream));
        });
    });
}

sk_status sk_kmap_transpose(sk_ctx* ctx, sk_kmap* map, void* stream, sk_kmap** out) {
    return guard([&] {
        sk::validate(ctx && map && out, "null argument");
        sk_kmap* t = sk::kmap_transpose(map, S(stream));
        t->refs.fetch_add(1);
        *out = t;
    });
}

sk_status sk_kmap_prepare(sk_ctx* ctx, sk_kmap* map, int splits, int pad_multiple, void* stream) {
    return guard([&] {
        sk::validate(ctx && map, "null argument");
        sk::kmap_prepare(map, splits, pad_multiple, S(stream));
    });
}

sk_status sk_kmap_retain(sk_kmap* map) {
    return guard([&] { map->refs.fetch_add(1); });
}

sk_status sk_kmap_release(sk_kmap* map) {
    return guard([&] { release_kmap(map); });
}

sk_status sk_kmap_get_info(sk_kmap* m, void* stream, sk_kmap_info* info) {
    return guard([&] {
        info->dims = m->dims;
        info->kernel_size = m->kernel;
        info->num_offsets = m->kd;
        info->n_in = m->n_in;
        info->n_out = m->n_out;
        info->transposed = m->transposed;
        for (int d = 0; d < 3; ++d) info->stride[d] = m->stride[d];
        info->total_pairs = sk::kmap_total_pairs(m, S(stream));
    });
}

sk_status sk_kmap_from_edges(sk_ctx* ctx, const int32_t* d_edges, int num_edges,
                             int num_relations, int n_in, int n_out, void* stream, sk_kmap** out) {
    return guard([&] {
        sk::validate(ctx && out, "null argument");
        sk::validate(num_edges == 0 || d_edges, "null edges");
        *out = sk::kmap_from_edges(ctx, d_edges, num_edges, num_relations, n_in, n_out, S(stream));
    });
}

sk_status sk_kmap_export_os(sk_kmap* m, int32_t* h_entries, uint64_t* h_masks, void* stream) {
    return guard([&] {
        sk::contract(!m->graph, "graph maps have no OS form");
        cudaStream_t st = S(stream);
        if (m->n_out) {
            SK_CUDA(cudaMemcpyAsync(h_entries, m->os.p, (size_t)m->n_out * m->kd * 4,
                                    cudaMemcpyDeviceToHost, st));
            SK_CUDA(cudaMemcpyAsync(h_masks, m->masks.p, (size_t)m->n_out * m->words * 8,
                                    cudaMemcpyDeviceToHost, st));
        }
        SK_CUDA(cudaStreamSynchronize(st));
    });
}

sk_status sk_kmap_export_ws(sk_kmap* m, int64_t* h_ptr, int32_t* h_in, int32_t* h_out,
                            void* stream) {
    return guard([&] {
        cudaStream_t st = S(stream);
        sk::kmap_ensure_ws(m, st);
        SK_CUDA(cudaMemcpyAsync(h_ptr, m->ws_ptr.p, (size_t)(m->kd + 1) * 8,
                                cudaMemcpyDeviceToHost, st));
        SK_CUDA(cudaStreamSynchronize(st));
        const int64_t P = h_ptr[m->kd];
        if (P > 0 && h_in) {
            SK_CUDA(cudaMemcpyAsync(h_in, m->ws_in.p, (size_t)P * 4, cudaMemcpyDeviceToHost, st));
            SK_CUDA(cudaMemcpyAsync(h_out, m->ws_out.p, (size_t)P * 4, cudaMemcpyDeviceToHost, st));
        }
        SK_CUDA(cudaStreamSynchronize(st));
    });
}

sk_status sk_kmap_export_split(sk_kmap* m, int splits, int pad_multiple, int s, int* begin,
                               int* end, int* n_rows, int* mask_words, int32_t* h_entries,
                               int32_t* h_out_row, uint64_t* h_masks, void* stream) {
    return guard([&] {
        cudaStream_t st = S(stream);
        sk::Prepared* p = sk::kmap_prepare(m, splits, pad_multiple, st);
        sk::validate(s >= 0 && s < p->num_splits, "split index out of range");
        const int b = p->begin[s], e = p->begin[s + 1], w = e - b, words = (w + 63) / 64;
        // the reference pads to exactly `pad_multiple` (kmap.cpp:274-288)
        const int rows = (int)(sk::ceil_div(m->n_out, pad_multiple) * pad_multiple);
        *begin = b;
        *end = e;
        *n_rows = rows;
        *mask_words = words;
        if (h_entries) {
            std::vector<int32_t> e = split_rows_host(p, s, st);
            std::memcpy(h_entries, e.data(), (size_t)rows * w * 4);
            // device rows are padded to lcm(pad, 128) >= rows; the tail is pad rows
            SK_CUDA(cudaMemcpyAsync(h_out_row, p->out_row.as<int32_t>() + (size_t)s * p->rows_pad,
                                    (size_t)rows * 4, cudaMemcpyDeviceToHost, st));
            SK_CUDA(cudaMemcpyAsync(h_masks,
                                    p->masks.as<uint64_t>() + (size_t)p->rows_pad * p->word_off[s],
                                    (size_t)rows * words * 8, cudaMemcpyDeviceToHost, st));
        }
        SK_CUDA(cudaStreamSynchronize(st));
    });
}

sk_status sk_conv_forward(sk_ctx* ctx, sk_kmap* map, const sk_dataflow_cfg* cfg, sk_dtype dtype,
                          int c_in, int c_out, const void* d_x, const void* d_w, void* d_y,
                          void* stream) {
    return guard([&] {
        sk::validate(ctx && map && cfg, "null argument");
        sk::validate(dtype == SK_F32 || dtype == SK_F16 || dtype == SK_BF16,
                     "convolution dtype must be f32, f16 or bf16");
        sk::stream_after(map->built_on, S(stream));  // map fetched on another stream
        sk::conv_forward(ctx, map, *cfg, dtype, c_in, c_out, d_x, d_w, d_y, false, S(stream));
    });
}

sk_status sk_conv_dgrad(sk_ctx* ctx, sk_kmap* map, const sk_dataflow_cfg* cfg, sk_dtype dtype,
                        int c_in, int c_out, const void* d_dy, const void* d_w, void* d_dx,
                        void* stream) {
    return guard([&] {
        sk::validate(ctx && map && cfg, "null argument");
        sk::validate(dtype == SK_F32 || dtype == SK_F16 || dtype == SK_BF16,
                     "convolution dtype must be f32, f16 or bf16");
        sk::stream_after(map->built_on, S(stream));  // map fetched on another stream
        sk::conv_forward(ctx, map, *cfg, dtype, c_in, c_out, d_dy, d_w, d_dx, true, S(stream));
    });
}

sk_status sk_conv_wgrad(sk_ctx* ctx, sk_kmap* map, const sk_dataflow_cfg* cfg, sk_dtype dtype,
                        int c_in, int c_out, const void* d_x, const void* d_dy, float* d_dw,
                        void* stream) {
    return guard([&] {
        sk::validate(ctx && map && cfg, "null argument");
        sk::validate(dtype == SK_F32 || dtype == SK_F16 || dtype == SK_BF16,
                     "convolution dtype must be f32, f16 or bf16");
        sk::stream_after(map->built_on, S(stream));  // map fetched on another stream
        sk::conv_wgrad(ctx, map, *cfg, dtype, c_in, c_out, d_x, d_dy, d_dw, S(stream));
    });
}

sk_status sk_kmap_count_macs(sk_kmap* m, int splits, int pad_multiple, int warp_rows, int c_in,
                             int c_out, int64_t* effective, int64_t* redundant, void* stream) {
    return guard([&] {
        // count_macs (cost.cpp:7-30) over the exported prepared splits
        cudaStream_t st = S(stream);
        sk::Prepared* p = sk::kmap_prepare(m, splits, pad_multiple, st);
        const int rows = (int)(sk::ceil_div(m->n_out, pad_multiple) * pad_multiple);
        int64_t eff = 0, charged = 0;
        const int64_t unit = (int64_t)c_in * c_out;
        for (int s = 0; s < p->num_splits; ++s) {
            const int w = p->begin[s + 1] - p->begin[s];
            std::vector<int32_t> e = split_rows_host(p, s, st);
            e.resize((size_t)rows * w);
            for (int32_t v : e) eff += v != -1;
            for (int r0 = 0; r0 < rows; r0 += warp_rows)
                for (int j = 0; j < w; ++j) {
                    bool act = false;
                    for (int r = r0; r < std::min(rows, r0 + warp_rows) && !act; ++r)
                        act = e[(size_t)r * w + j] != -1;
                    if (act) charged += (int64_t)warp_rows * unit;
                }
        }
        *effective = eff * unit;
        *redundant = charged - eff * unit;
    });
}

}  // extern "C"
