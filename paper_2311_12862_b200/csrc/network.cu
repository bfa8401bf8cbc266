// sk200 NetworkRunner + group autotuner,
// native C++ over the device kmaps / dataflows.
//
//  * NetSpec / validate / propagate_syms / partition_groups restate
//    network.cpp:30-158 (same validation rules, same structural symbols, same
//    groups keyed by (in_sym, out_sym, K, stride); decoder layers join their
//    encoder's group).
//  * sk_net::forward restates run_forward (network.cpp:282-345): per layer,
//    resolve producers (<= 2, summed), take the group's maps (built once per
//    input coordinate set through the sk_coords map cache = GroupMaps cache,
//    network.cpp:183-275), run the group's forward config. Mapping and kernel
//    time are split per group with CUDA events (RunStats, network.hpp:62-70).
//  * measure (network.cpp:398-438): forward, then dgrad / wgrad sweeps with
//    all-ones dummy gradients, timed per phase (the tuner's probe).
//  * backward: a real chained backward (dgrad output of layer i feeds its
//    producers, skip fan-out summed), weight gradients in one flat fp32
//    buffer — the data-parallel training step's per-GPU half.
//  * tune: greedy_pass / tune_inference / tune_training (tuner.cpp:86-220)
//    with a CUDA-event RunnerProbe (warmup 2, median of 5, tuner.cpp:50-60);
//    ties break on the traffic model (cost.cpp:47-93) then space order.
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <atomic>
#include <mutex>
#include <cstring>
#include <exception>
#include <functional>
#include <thread>
#include <sstream>
#include <unordered_map>

#include "sk_internal.hpp"

namespace sk {

struct LayerSpec {
    std::string name;
    int kind = 0;  // 0 conv, 1 conv_transposed (LayerKind, network.hpp:15)
    int c_in = 1, c_out = 1, kernel = 3, stride = 1;
    std::vector<std::string> inputs;
    std::string transpose_of;
};

struct NetSpec {
    int dims = 3;
    std::vector<LayerSpec> layers;
    int index(const std::string& n) const {
        for (size_t i = 0; i < layers.size(); ++i)
            if (layers[i].name == n) return (int)i;
        return -1;
    }
    // NetworkSpec::validate (network.cpp:30-76)
    void validate() const {
        sk::validate(dims == 2 || dims == 3, "network dims must be 2 or 3");
        sk::validate(!layers.empty(), "network has no layers");
        std::map<std::string, int> seen;
        for (size_t i = 0; i < layers.size(); ++i) {
            const LayerSpec& l = layers[i];
            sk::validate(!l.name.empty(), "layer " + std::to_string(i) + " has no name");
            sk::validate(seen.emplace(l.name, (int)i).second, "duplicate layer name: " + l.name);
            sk::validate(l.c_in > 0 && l.c_out > 0, l.name + ": channel counts must be positive");
            sk::validate(l.kernel > 0 && l.kernel % 2 == 1,
                         l.name + ": kernel size must be odd and positive");
            sk::validate(l.stride > 0, l.name + ": stride must be positive");
            sk::validate(l.inputs.size() <= 2, l.name + ": at most two producers supported");
            for (const std::string& p : l.inputs) {
                int j = index(p);
                sk::validate(j >= 0 && j < (int)i,
                             l.name + ": producer '" + p + "' must be an earlier layer");
                sk::validate(layers[j].c_out == l.c_in,
                             l.name + ": c_in does not match producer '" + p + "' c_out");
            }
            if (l.kind == 1) {
                int j = index(l.transpose_of);
                sk::validate(j >= 0 && j < (int)i,
                             l.name + ": transpose_of must name an earlier layer");
                sk::validate(layers[j].kind == 0, l.name + ": transpose_of must be a conv layer");
                sk::validate(layers[j].kernel == l.kernel && layers[j].stride == l.stride,
                             l.name + ": kernel/stride must match '" + l.transpose_of + "'");
            } else {
                sk::validate(l.transpose_of.empty(),
                             l.name + ": transpose_of is only valid on conv_transposed");
            }
        }
    }
};

NetSpec parse_spec(int dims, const char* text) {
    NetSpec s;
    s.dims = dims;
    std::istringstream is(text ? text : "");
    std::string line;
    while (std::getline(is, line)) {
        if (line.empty() || line[0] == '#') continue;
        std::istringstream ls(line);
        LayerSpec l;
        std::string kind, inputs, tof;
        if (!(ls >> l.name >> kind >> l.c_in >> l.c_out >> l.kernel >> l.stride >> inputs >> tof))
            fail(SK_ERR_VALIDATION, "malformed layer line: " + line);
        if (kind == "conv") l.kind = 0;
        else if (kind == "conv_transposed") l.kind = 1;
        else fail(SK_ERR_VALIDATION, "unknown layer kind: " + kind);
        if (inputs != "-") {
            std::stringstream ss(inputs);
            std::string tok;
            while (std::getline(ss, tok, ',')) l.inputs.push_back(tok);
        }
        if (tof != "-") l.transpose_of = tof;
        s.layers.push_back(l);
    }
    s.validate();
    return s;
}

struct StructKey {
    int in_sym, out_sym, kernel, stride;
    bool operator==(const StructKey& o) const {
        return in_sym == o.in_sym && out_sym == o.out_sym && kernel == o.kernel &&
               stride == o.stride;
    }
};

// propagate_syms + partition_groups (network.cpp:98-158)
std::vector<std::vector<int>> partition_groups(const NetSpec& net) {
    const size_t L = net.layers.size();
    std::vector<std::pair<int, int>> syms(L);
    std::vector<StructKey> keys(L);
    int next_sym = 1;
    std::map<long long, int> derived;
    for (size_t i = 0; i < L; ++i) {
        const LayerSpec& l = net.layers[i];
        int in_sym = 0;
        if (!l.inputs.empty()) {
            in_sym = syms[net.index(l.inputs[0])].second;
            if (l.inputs.size() == 2)
                validate(syms[net.index(l.inputs[1])].second == in_sym,
                         l.name + ": skip producers live on different coordinate sets");
        }
        int out_sym;
        if (l.kind == 1) {
            int j = net.index(l.transpose_of);
            validate(syms[j].second == in_sym, l.name +
                                                   ": input coordinates do not match the output of '" +
                                                   l.transpose_of + "'");
            out_sym = syms[j].first;
            keys[i] = keys[j];
        } else if (l.stride == 1) {
            out_sym = in_sym;
            keys[i] = {in_sym, out_sym, l.kernel, 1};
        } else {
            long long dk = (long long)in_sym * 64 + l.stride;
            auto it = derived.find(dk);
            if (it == derived.end()) it = derived.emplace(dk, next_sym++).first;
            out_sym = it->second;
            keys[i] = {in_sym, out_sym, l.kernel, l.stride};
        }
        syms[i] = {in_sym, out_sym};
    }
    std::vector<std::vector<int>> groups;
    std::vector<int> head;
    for (size_t i = 0; i < L; ++i) {
        int gid = -1;
        for (size_t g = 0; g < groups.size(); ++g)
            if (keys[head[g]] == keys[i]) {
                gid = (int)g;
                break;
            }
        if (gid < 0) {
            groups.emplace_back();
            head.push_back((int)i);
            gid = (int)groups.size() - 1;
        }
        groups[gid].push_back((int)i);
    }
    return groups;
}

// Runner-owned streams live for the process: objects built on them (cached
// maps and coordinate sets, block-cache entries) can outlive the runner, and a
// destroyed handle could be reused by an unrelated stream.
namespace {
std::mutex g_stream_mu;
std::vector<std::pair<int, cudaStream_t>>& stream_pool() {
    static auto* v = new std::vector<std::pair<int, cudaStream_t>>();
    return *v;
}
}  // namespace
cudaStream_t acquire_runner_stream(int dev) {
    {
        std::lock_guard<std::mutex> g(g_stream_mu);
        auto& v = stream_pool();
        for (size_t i = 0; i < v.size(); ++i)
            if (v[i].first == dev) {
                cudaStream_t s = v[i].second;
                v.erase(v.begin() + (long)i);
                return s;
            }
    }
    int cur = 0;
    SK_CUDA(cudaGetDevice(&cur));
    SK_CUDA(cudaSetDevice(dev));
    cudaStream_t s = nullptr;
    SK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    SK_CUDA(cudaSetDevice(cur));
    return s;
}
void release_runner_stream(int dev, cudaStream_t s) {
    if (cudaStreamSynchronize(s) != cudaSuccess) {
        (void)cudaGetLastError();
        return;  // leaked, never reused
    }
    std::lock_guard<std::mutex> g(g_stream_mu);
    stream_pool().push_back({dev, s});
}

namespace {

template <typename T>
__device__ __forceinline__ float ld_f(const T* p, long long i);
template <>
__device__ __forceinline__ float ld_f<__half>(const __half* p, long long i) { return __half2float(p[i]); }
template <>
__device__ __forceinline__ float ld_f<__nv_bfloat16>(const __nv_bfloat16* p, long long i) { return __bfloat162float(p[i]); }
template <>
__device__ __forceinline__ float ld_f<float>(const float* p, long long i) { return p[i]; }
template <typename T>
__device__ __forceinline__ T cvt_f(float v);
template <>
__device__ __forceinline__ __half cvt_f<__half>(float v) { return __float2half_rn(v); }
template <>
__device__ __forceinline__ __nv_bfloat16 cvt_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }
template <>
__device__ __forceinline__ float cvt_f<float>(float v) { return v; }

// skip connection: y = a + b (network.cpp:174-181 sums producers)
template <typename T>
__global__ void k_add(const T* __restrict__ a, const T* __restrict__ b, long long n,
                      T* __restrict__ y) {
    pdl_wait();
    pdl_trigger();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        y[i] = cvt_f<T>(ld_f(a, i) + ld_f(b, i));
}
template <typename T>
__global__ void k_fill(T* __restrict__ y, long long n, float v) {
    pdl_wait();
    pdl_trigger();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        y[i] = cvt_f<T>(v);
}
// gradient accumulation: g (fp32) += dx
template <typename T>
__global__ void k_accum(float* __restrict__ g, const T* __restrict__ dx, long long n) {
    pdl_wait();
    pdl_trigger();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        g[i] += ld_f(dx, i);
}
// g1 += dx and g2 += dx (a two-input layer's gradient to both producers, dx
// read once); 4 elements per thread when n % 4 == 0
template <typename T>
__global__ void k_accum2(float* __restrict__ g1, float* __restrict__ g2, const T* __restrict__ dx,
                         long long n) {
    pdl_wait();
    pdl_trigger();
    const long long n4 = n / 4;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
         i += (long long)gridDim.x * blockDim.x) {
        const float a = ld_f(dx, 4 * i), b = ld_f(dx, 4 * i + 1), c = ld_f(dx, 4 * i + 2),
                    d = ld_f(dx, 4 * i + 3);
        float4 u = reinterpret_cast<float4*>(g1)[i];
        u.x += a; u.y += b; u.z += c; u.w += d;
        reinterpret_cast<float4*>(g1)[i] = u;
        float4 v = reinterpret_cast<float4*>(g2)[i];
        v.x += a; v.y += b; v.z += c; v.w += d;
        reinterpret_cast<float4*>(g2)[i] = v;
    }
    for (long long i = 4 * n4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const float a = ld_f(dx, i);
        g1[i] += a;
        g2[i] += a;
    }
}
template <typename T>
__global__ void k_cast_from_f32(const float* __restrict__ g, long long n, T* __restrict__ y) {
    pdl_wait();
    pdl_trigger();
    const long long n4 = n / 4;  // float4 in, 4 elements out per iteration
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
         i += (long long)gridDim.x * blockDim.x) {
        const float4 v = reinterpret_cast<const float4*>(g)[i];
        y[4 * i] = cvt_f<T>(v.x);
        y[4 * i + 1] = cvt_f<T>(v.y);
        y[4 * i + 2] = cvt_f<T>(v.z);
        y[4 * i + 3] = cvt_f<T>(v.w);
    }
    for (long long i = 4 * n4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        y[i] = cvt_f<T>(g[i]);
}

int grid_for(long long n) { return (int)std::min<long long>(std::max<long long>(1, ceil_div(n, 256)), 148 * 16); }

template <class F>
void by_dtype(sk_dtype dt, F&& f) {
    if (dt == SK_F16) f(__half{});
    else if (dt == SK_BF16) f(__nv_bfloat16{});
    else f(float{});
}

}  // namespace

}  // namespace sk

using namespace sk;

namespace sk {
// The runner's map-builder thread (overlapped forward), created on first use
// and kept for the runner's lifetime: one job per forward. After a job it
// polls (yielding) for the next one for 5 ms, so back-to-back scans hand over
// in microseconds (a condition-variable wake cost tens), then sleeps on a
// condition variable; spawning a thread per forward cost ~40 us of host
// latency before the first map kernel.
struct MapWorker {
    std::thread t;
    std::mutex mu;
    std::condition_variable cv, cv_done;
    std::function<void()> job;
    std::atomic<bool> pending{false};
    bool stop = false;
    void post(std::function<void()> j) {
        if (!t.joinable()) t = std::thread([this] { loop(); });
        {
            std::lock_guard<std::mutex> lk(mu);
            job = std::move(j);
            pending.store(true, std::memory_order_release);
        }
        cv.notify_one();
    }
    void wait() {
        std::unique_lock<std::mutex> lk(mu);
        cv_done.wait(lk, [&] { return !pending.load(std::memory_order_acquire); });
    }
    void loop() {
        for (;;) {
            const auto until = std::chrono::steady_clock::now() + std::chrono::milliseconds(5);
            while (!pending.load(std::memory_order_acquire) &&
                   std::chrono::steady_clock::now() < until)
                std::this_thread::yield();
            std::function<void()> j;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return stop || pending.load(std::memory_order_acquire); });
                if (!pending.load(std::memory_order_acquire)) return;  // stop
                j = std::move(job);
            }
            j();
            {
                std::lock_guard<std::mutex> lk(mu);
                pending.store(false, std::memory_order_release);
            }
            cv_done.notify_all();
        }
    }
    ~MapWorker() {
        if (!t.joinable()) return;
        {
            std::lock_guard<std::mutex> lk(mu);
            stop = true;
        }
        cv.notify_one();
        t.join();
    }
};
}  // namespace sk

struct sk_net {
    sk_ctx* ctx = nullptr;
    NetSpec spec;
    sk_dtype dt = SK_F16;
    std::vector<std::vector<int>> groups;
    std::vector<int> group_of;
    std::vector<int> kd;
    std::vector<DevBuf> w;
    std::vector<DevBuf> wt;    // W^T per layer for the forward B operand (K-major)
    bool wt_dirty = true;      // weights may have changed since the last transpose
    std::vector<sk_dataflow_cfg> cfg[3];  // per group: forward, dgrad, wgrad
    // state of the last forward
    uint64_t root_id = 0;
    std::vector<sk_coords*> in_set, out_set;  // retained
    std::vector<sk_kmap*> exec_map;           // retained, execution orientation
    std::vector<DevBuf> out, xsum;
    std::vector<void*> out_ptr;     // layer output (may alias the consumer's xsum)
    std::vector<const void*> x_ptr;
    // skip-add fusion: layer P (only consumer L = fuse_into[P]) writes
    // xsum[L] = conv_P(x) + out[residual_of[P]] in its epilogue
    std::vector<int> fuse_into, residual_of;
    std::vector<char> fused_input;  // L's xsum is produced by a fused producer
    std::vector<size_t> wgrad_off;
    size_t wgrad_total = 0;
    DevBuf gout_slab;              // fp32 output grads of every layer (backward), one slab
    std::vector<float*> gout;      // layer i's [n_out x c_out] view into gout_slab
    int64_t map_builds = 0;
    bool overlap = true;                      // overlapped map builds (sk_net_set_overlap)
    bool pdl = true;                          // programmatic dependent launch (sk_net_set_pdl)
    bool tune_cold = false;                   // tuner probes on fresh sets (sk_net_set_tune_cold)
    cudaStream_t map_stream = nullptr;        // overlapped map builds (run_forward)
    cudaStream_t cmp_stream = nullptr;        // overlapped forward's convs for legacy-stream callers
    std::vector<cudaEvent_t> map_ready;       // per layer: its maps are built on map_stream
    std::unique_ptr<sk::MapWorker> worker;    // overlapped map builder (run_forward)

    ~sk_net() {
        worker.reset();  // no job can be running: run_forward waits for its job
        clear_state();
        for (auto e : map_ready) cudaEventDestroy(e);
        // cached maps / sets built here still name these streams (BuiltOn
        // marks, block-cache keys): they go back to a process-lifetime pool
        // instead of being destroyed
        if (map_stream) sk::release_runner_stream(ctx->device, map_stream);
        if (cmp_stream) sk::release_runner_stream(ctx->device, cmp_stream);
    }
    void clear_state() {
        for (auto* c : in_set) if (c) sk_coords_release(c);
        for (auto* c : out_set) if (c) sk_coords_release(c);
        for (auto* m : exec_map) if (m) sk_kmap_release(m);
        in_set.clear();
        out_set.clear();
        exec_map.clear();
    }
    size_t es() const { return dt == SK_F32 ? 4 : 2; }
};

namespace {

// a group's config applied to one layer: implicit-GEMM splits are clamped to
// the layer's K^D (the K=1 projection layers of a group cannot split)
sk_dataflow_cfg layer_cfg(const sk_net* n, int phase, int layer) {
    sk_dataflow_cfg c = n->cfg[phase][n->group_of[layer]];
    if (c.splits > n->kd[layer]) c.splits = n->kd[layer];
    return c;
}

sk_dataflow_cfg default_cfg() {
    sk_dataflow_cfg c;
    memset(&c, 0, sizeof(c));
    c.kind = SK_GATHER_GEMM_SCATTER;  // default assignment (network.cpp:387-390)
    c.tile = {128, 64, 0, 128, 4};
    return c;
}

struct Timer {
    cudaEvent_t a, b;
    cudaStream_t st;
    explicit Timer(cudaStream_t s) : st(s) {
        SK_CUDA(cudaEventCreate(&a));
        SK_CUDA(cudaEventCreate(&b));
        SK_CUDA(cudaEventRecord(a, st));
    }
    float stop() {
        SK_CUDA(cudaEventRecord(b, st));
        SK_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        SK_CUDA(cudaEventElapsedTime(&ms, a, b));
        return ms;
    }
    ~Timer() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
};

// Maps of layer i for the network input `root` (layers before i done);
// reuses the sk_coords caches (one build per (coordinate set, K, stride,
// orientation) = per group).
void build_layer_maps(sk_net* n, sk_coords* root, size_t i, cudaStream_t st) {
    const LayerSpec& l = n->spec.layers[i];
    sk_coords* in = l.inputs.empty() ? root : n->out_set[n->spec.index(l.inputs[0])];
    sk_coords_retain(in);
    n->in_set[i] = in;
    int32_t s3[3] = {l.stride, l.stride, n->spec.dims == 3 ? l.stride : 1};
    if (l.kind == 0) {
        sk_coords* out = nullptr;
        sk_status rc0 = sk_out_coords(n->ctx, in, s3, st, &out);
        if (rc0) fail(rc0, sk_last_error());
        n->out_set[i] = out;
        sk_kmap* m = nullptr;
        sk_status rc = sk_kmap_build(n->ctx, in, out, l.kernel, s3, 0, st, &m);
        if (rc) fail(rc, sk_last_error());
        n->exec_map[i] = m;
    } else {
        const int j = n->spec.index(l.transpose_of);
        sk_coords* out = n->in_set[j];
        sk_coords_retain(out);
        n->out_set[i] = out;
        sk_kmap* t2 = nullptr;
        sk_status rc = sk_kmap_transpose(n->ctx, n->exec_map[j], st, &t2);
        if (rc) fail(rc, sk_last_error());
        n->exec_map[i] = t2;
    }
}

// a failed build leaves partial maps: root_id is cleared here and set only
// after every layer's maps are built, so a retry never takes them as cached
void reset_maps(sk_net* n) {
    n->root_id = 0;
    n->clear_state();
    const size_t L = n->spec.layers.size();
    n->in_set.assign(L, nullptr);
    n->out_set.assign(L, nullptr);
    n->exec_map.assign(L, nullptr);
}

bool maps_complete(const sk_net* n, const sk_coords* root) {
    return n->root_id != 0 && n->root_id == root->id && !n->exec_map.empty() &&
           n->exec_map.back() != nullptr;
}

void ensure_maps(sk_net* n, sk_coords* root, cudaStream_t st, std::vector<double>* map_ms) {
    if (maps_complete(n, root)) return;
    reset_maps(n);
    for (size_t i = 0; i < n->spec.layers.size(); ++i) {
        std::unique_ptr<Timer> t;
        if (map_ms) t = std::make_unique<Timer>(st);
        build_layer_maps(n, root, i, st);
        if (map_ms) (*map_ms)[n->group_of[i]] += t->stop();
    }
    n->root_id = root->id;
    ++n->map_builds;
}

// xsum[c] (the summed input of two-input layer c) sized from its first input's set
void ensure_xsum(sk_net* n, int c, cudaStream_t st) {
    const LayerSpec& l = n->spec.layers[c];
    const sk_coords* src = n->out_set[n->spec.index(l.inputs[0])];
    const size_t xb = (size_t)std::max(src->n, 1) * l.c_in * n->es();
    if (n->xsum[c].bytes != xb) n->xsum[c].alloc(xb, st);
}

// output buffer of layer i (or its alias into the fused consumer's xsum)
void alloc_layer_output(sk_net* n, size_t i, cudaStream_t st) {
    const LayerSpec& l = n->spec.layers[i];
    if (l.inputs.size() == 2 && !n->fused_input[i]) ensure_xsum(n, (int)i, st);
    if (n->fuse_into[i] >= 0) {
        ensure_xsum(n, n->fuse_into[i], st);
        n->out_ptr[i] = n->xsum[n->fuse_into[i]].p;
        return;
    }
    const size_t bytes = (size_t)std::max(n->out_set[i]->n, 1) * l.c_out * n->es();
    if (n->out[i].bytes != bytes) n->out[i].alloc(bytes, st);
    n->out_ptr[i] = n->out[i].p;
}

void alloc_outputs(sk_net* n, cudaStream_t st) {
    const size_t L = n->spec.layers.size();
    n->out.resize(L);
    n->xsum.resize(L);
    n->x_ptr.assign(L, nullptr);
    n->out_ptr.assign(L, nullptr);
    for (size_t i = 0; i < L; ++i) {
        const LayerSpec& l = n->spec.layers[i];
        if (l.inputs.size() == 2) {
            size_t xb = (size_t)std::max(n->in_set[i]->n, 1) * l.c_in * n->es();
            if (n->xsum[i].bytes != xb) n->xsum[i].alloc(xb, st);
        }
    }
    for (size_t i = 0; i < L; ++i) {
        const LayerSpec& l = n->spec.layers[i];
        if (n->fuse_into[i] >= 0) {
            n->out_ptr[i] = n->xsum[n->fuse_into[i]].p;
            continue;
        }
        size_t bytes = (size_t)std::max(n->out_set[i]->n, 1) * l.c_out * n->es();
        if (n->out[i].bytes != bytes) n->out[i].alloc(bytes, st);
        n->out_ptr[i] = n->out[i].p;
    }
}

// plan skip-add fusion: for L with producers {a, b}, the producer that runs
// later and whose only consumer is L adds the other one in its epilogue
void plan_fusion(sk_net* n) {
    const int L = (int)n->spec.layers.size();
    std::vector<int> consumers(L, 0);
    for (const LayerSpec& l : n->spec.layers)
        for (const std::string& p : l.inputs) ++consumers[n->spec.index(p)];
    n->fuse_into.assign(L, -1);
    n->residual_of.assign(L, -1);
    n->fused_input.assign(L, 0);
    for (int i = 0; i < L; ++i) {
        const LayerSpec& l = n->spec.layers[i];
        if (l.inputs.size() != 2) continue;
        const int a = n->spec.index(l.inputs[0]), b = n->spec.index(l.inputs[1]);
        int P = -1, Q = -1;
        if (consumers[a] == 1 && b < a) P = a, Q = b;
        else if (consumers[b] == 1 && a < b) P = b, Q = a;
        if (P < 0 || n->fuse_into[P] >= 0) continue;
        n->fuse_into[P] = i;
        n->residual_of[P] = Q;
        n->fused_input[i] = 1;
    }
}

// run_forward (network.cpp:282-345)
void refresh_wt(sk_net* n, cudaStream_t st) {
    if (!n->wt_dirty) return;
    n->wt.resize(n->w.size());
    for (size_t i = 0; i < n->w.size(); ++i) {
        const LayerSpec& l = n->spec.layers[i];
        if (n->wt[i].bytes != n->w[i].bytes) n->wt[i].alloc(n->w[i].bytes, st);
        transpose_weights(n->dt, n->w[i].p, n->kd[i], l.c_in, l.c_out, n->wt[i].p, st);
    }
    n->wt_dirty = false;
}

// per-layer CUDA events, read once at the end (no per-layer sync)
struct LayerEvents {
    std::vector<cudaEvent_t> ev;
    explicit LayerEvents(size_t n) : ev(2 * n) {
        for (auto& e : ev) SK_CUDA(cudaEventCreate(&e));
    }
    ~LayerEvents() {
        for (auto& e : ev) cudaEventDestroy(e);
    }
    float ms(size_t i) {
        float v = 0;
        SK_CUDA(cudaEventElapsedTime(&v, ev[2 * i], ev[2 * i + 1]));
        return v;
    }
};

void run_layers(sk_net* n, const void* feats, int channels, cudaStream_t st,
                std::vector<double>* ker_ms, std::vector<double>* layer_ms,
                const std::function<void(size_t)>& before) {
    const size_t L = n->spec.layers.size();
    std::unique_ptr<LayerEvents> evs;
    if (ker_ms || layer_ms) evs = std::make_unique<LayerEvents>(L);
    for (size_t i = 0; i < L; ++i) {
        const LayerSpec& l = n->spec.layers[i];
        if (before) before(i);
        if (evs) SK_CUDA(cudaEventRecord(evs->ev[2 * i], st));
        const void* x;
        if (l.inputs.empty()) {
            validate(channels == l.c_in, l.name + ": input channel mismatch");
            x = feats;
        } else if (l.inputs.size() == 1) {
            x = n->out_ptr[n->spec.index(l.inputs[0])];
        } else if (n->fused_input[i]) {
            x = n->xsum[i].p;  // written by the fused producer's epilogue
        } else {
            const long long cnt = (long long)n->in_set[i]->n * l.c_in;
            const void* a = n->out_ptr[n->spec.index(l.inputs[0])];
            const void* b = n->out_ptr[n->spec.index(l.inputs[1])];
            void* y = n->xsum[i].p;
            by_dtype(n->dt, [&](auto tag) {
                using T = decltype(tag);
                launch_pdl(k_add<T>, grid_for(cnt), 256, 0, st, (const T*)a, (const T*)b, cnt, (T*)y);
            });
            x = y;
        }
        n->x_ptr[i] = x;
        const void* res = n->fuse_into[i] >= 0 ? n->out_ptr[n->residual_of[i]] : nullptr;
        conv_forward(n->ctx, n->exec_map[i], layer_cfg(n, 0, (int)i), n->dt, l.c_in, l.c_out, x,
                     n->w[i].p, n->out_ptr[i], false, st, n->wt[i].p, res);
        if (evs) SK_CUDA(cudaEventRecord(evs->ev[2 * i + 1], st));
    }
    if (evs) {
        SK_CUDA(cudaEventSynchronize(evs->ev[2 * L - 1]));
        if (layer_ms) layer_ms->assign(L, 0.0);
        for (size_t i = 0; i < L; ++i) {
            const double v = evs->ms(i);
            if (ker_ms) (*ker_ms)[n->group_of[i]] += v;
            if (layer_ms) (*layer_ms)[i] = v;
        }
    }
}

void run_forward(sk_net* n, sk_coords* root, const void* feats, int channels, cudaStream_t st,
                 std::vector<double>* map_ms, std::vector<double>* ker_ms,
                 std::vector<double>* layer_ms = nullptr) {
    validate(channels == n->spec.layers[0].c_in || !n->spec.layers[0].inputs.empty(),
             "network input channel count does not match the first layer");
    const size_t L = n->spec.layers.size();
    const bool cached = maps_complete(n, root);
    if (cached || map_ms || !n->overlap) {
        ensure_maps(n, root, st, map_ms);
        alloc_outputs(n, st);
        refresh_wt(n, st);
        run_layers(n, feats, channels, st, ker_ms, layer_ms, nullptr);
        return;
    }
    // Overlapped map build: a host thread builds layer i's maps (down-sampled
    // sets with their count readbacks, queries, transposes, the prepared map
    // or pair lists the layer's dataflow reads) on the runner's map stream
    // and records map_ready[i]; this thread enqueues layer i's conv on st
    // behind that event. The readback syncs then stall only the builder, and
    // the device runs level l's convs while level l+1's maps are built.
    if (!n->map_stream) n->map_stream = acquire_runner_stream(n->ctx->device);
    // a caller on the legacy default stream gets the convs on a runner-owned
    // stream (measured: the overlap bought nothing with the convs on the
    // legacy stream), bracketed by events so the caller's order is unchanged
    const cudaStream_t caller = st;
    const bool legacy = st == nullptr || st == cudaStreamLegacy;
    if (legacy) {
        if (!n->cmp_stream) n->cmp_stream = acquire_runner_stream(n->ctx->device);
        st = n->cmp_stream;
    }
    while (n->map_ready.size() < L + 2) {
        cudaEvent_t e;
        SK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        n->map_ready.push_back(e);
    }
    cudaStream_t ms = n->map_stream;
    SK_CUDA(cudaEventRecord(n->map_ready[L], caller));  // the caller's prior work (root, feats)
    SK_CUDA(cudaStreamWaitEvent(ms, n->map_ready[L], 0));
    if (legacy) SK_CUDA(cudaStreamWaitEvent(st, n->map_ready[L], 0));
    // the previous scan's maps are released below, after the builder has its
    // job (dropping ~200 references took ~20 us of the critical path): their
    // buffers go back to the map stream's cache / pool behind the wait above,
    // i.e. after every conv of the previous scan that read them
    std::vector<sk_coords*> old_in, old_out;
    std::vector<sk_kmap*> old_maps;
    old_in.swap(n->in_set);
    old_out.swap(n->out_set);
    old_maps.swap(n->exec_map);
    reset_maps(n);
    // layer i's maps are ready once done > i; this thread spins (yielding) on
    // it: a condition-variable wake per layer added tens of microseconds
    std::atomic<size_t> done{0};
    std::atomic<bool> failed{false};
    std::exception_ptr err;
    const int dev = n->ctx->device;
    if (!n->worker) n->worker = std::make_unique<MapWorker>();
    MapWorker* builder = n->worker.get();
    const bool pdl = n->pdl;
    builder->post([&, pdl] {
        try {
            SK_CUDA(cudaSetDevice(dev));
            pdl_enabled() = pdl;
            for (size_t i = 0; i < L; ++i) {
                build_layer_maps(n, root, i, ms);
                const LayerSpec& l = n->spec.layers[i];
                conv_forward_prepare(n->ctx, n->exec_map[i], layer_cfg(n, 0, (int)i), n->dt,
                                     l.c_in, l.c_out, ms);
                SK_CUDA(cudaEventRecord(n->map_ready[i], ms));
                done.store(i + 1, std::memory_order_release);
            }
        } catch (...) {
            err = std::current_exception();
            failed.store(true, std::memory_order_release);
        }
    });
    struct Join {  // the job references this frame: wait for it on every exit path
        MapWorker* w;
        ~Join() { w->wait(); }
    } join{builder};
    for (auto* c : old_in) if (c) sk_coords_release(c);
    for (auto* c : old_out) if (c) sk_coords_release(c);
    for (auto* m : old_maps) if (m) sk_kmap_release(m);
    refresh_wt(n, st);
    n->out.resize(L);
    n->xsum.resize(L);
    n->x_ptr.assign(L, nullptr);
    n->out_ptr.assign(L, nullptr);
    run_layers(n, feats, channels, st, ker_ms, layer_ms, [&](size_t i) {
        while (done.load(std::memory_order_acquire) <= i) {
            if (failed.load(std::memory_order_acquire)) {
                builder->wait();
                std::rethrow_exception(err);
            }
            std::this_thread::yield();
        }
        SK_CUDA(cudaStreamWaitEvent(st, n->map_ready[i], 0));
        alloc_layer_output(n, i, st);
    });
    builder->wait();
    if (err) std::rethrow_exception(err);
    if (legacy) {  // the caller's stream continues after the convs
        SK_CUDA(cudaEventRecord(n->map_ready[L + 1], st));
        SK_CUDA(cudaStreamWaitEvent(caller, n->map_ready[L + 1], 0));
    }
    n->root_id = root->id;
    ++n->map_builds;
}

// measure_ms (network.cpp:398-438): forward always runs; dgrad / wgrad sweeps
// with all-ones dummy gradients when requested; only masked phases count.
double measure(sk_net* n, sk_coords* root, const void* feats, int channels, bool fwd, bool dg,
               bool wg, cudaStream_t st) {
    double total = 0;
    if (n->tune_cold && fwd && !dg && !wg) {
        // a fresh copy of the set: every map (and its split/sort or pair
        // lists for the candidate configs) is built inside the timed forward
        sk_coords* fresh = nullptr;
        const sk_status rc = sk_coords_create(n->ctx, root->dims, root->n,
                                              root->coords.as<int32_t>(), root->stride_tag, st, &fresh);
        if (rc) fail(rc, sk_last_error());
        Timer t(st);
        try {
            run_forward(n, fresh, feats, channels, st, nullptr, nullptr);
        } catch (...) {
            sk_coords_release(fresh);
            throw;
        }
        total += t.stop();
        sk_coords_release(fresh);
        return total;
    }
    {
        Timer t(st);
        run_forward(n, root, feats, channels, st, nullptr, nullptr);
        float ms = t.stop();
        if (fwd) total += ms;
    }
    if (!dg && !wg) return total;
    const size_t L = n->spec.layers.size();
    size_t max_out = 0, max_in = 0;
    for (size_t i = 0; i < L; ++i) {
        max_out = std::max(max_out, (size_t)n->out_set[i]->n * n->spec.layers[i].c_out);
        max_in = std::max(max_in, (size_t)n->in_set[i]->n * n->spec.layers[i].c_in);
    }
    DevBuf ones, dx, dw;
    ones.alloc(std::max<size_t>(max_out, 1) * n->es(), st);
    dx.alloc(std::max<size_t>(max_in, 1) * n->es(), st);
    size_t max_w = 0;
    for (size_t i = 0; i < L; ++i)
        max_w = std::max(max_w, (size_t)n->kd[i] * n->spec.layers[i].c_in * n->spec.layers[i].c_out);
    dw.alloc(max_w * 4, st);
    by_dtype(n->dt, [&](auto tag) {
        using T = decltype(tag);
        launch_pdl(k_fill<T>, grid_for((long long)max_out), 256, 0, st, (T*)ones.p, (long long)max_out, 1.f);
    });
    if (dg) {
        Timer t(st);
        for (size_t i = 0; i < L; ++i) {
            const LayerSpec& l = n->spec.layers[i];
            conv_forward(n->ctx, n->exec_map[i], layer_cfg(n, 1, (int)i), n->dt, l.c_in, l.c_out,
                         ones.p, n->w[i].p, dx.p, true, st);
        }
        total += t.stop();
    }
    if (wg) {
        Timer t(st);
        for (size_t i = 0; i < L; ++i) {
            const LayerSpec& l = n->spec.layers[i];
            conv_wgrad(n->ctx, n->exec_map[i], layer_cfg(n, 2, (int)i), n->dt, l.c_in, l.c_out,
                       n->x_ptr[i], ones.p, dw.as<float>(), st);
        }
        total += t.stop();
    }
    return total;
}

// Modeled DRAM bytes of a group under cfg (traffic_model, cost.cpp:47-93,
// elem_bytes of the run dtype); the tuner's tie-break.
double modeled_group_traffic(sk_net* n, int g, const sk_dataflow_cfg& cfg, cudaStream_t st) {
    double total = 0;
    for (int li : n->groups[g]) {
        const LayerSpec& l = n->spec.layers[li];
        sk_kmap* m = n->exec_map[li];
        if (!m) return 0;
        const double eb = (double)n->es();
        const double pairs = (double)kmap_total_pairs(m, st);
        const double n_out = m->n_out, kdv = m->kd, unit = (double)l.c_in * l.c_out;
        double rd = 0, wr = 0;
        if (cfg.kind == SK_GATHER_GEMM_SCATTER) {
            wr = pairs * l.c_in + pairs * l.c_out + n_out * l.c_out;
            rd = 2 * pairs * l.c_in + kdv * unit + pairs * l.c_out + n_out * l.c_out;
        } else if (cfg.kind == SK_FETCH_ON_DEMAND) {
            wr = pairs * l.c_out;
            rd = pairs * l.c_in + kdv * unit + pairs * l.c_out;
        } else {
            // prepare_os_map = pad_map(split_and_sort(raw, s), cta_m)
            // (exec.cpp:342-344): every split keeps all n_out rows padded to
            // the preset's cta_m and the split widths sum to K^D, so the A
            // loads are rows_padded * K^D * C_in whatever the split count
            const int pad = cfg.tile.cta_m > 0 ? cfg.tile.cta_m : kTileM;
            const double rows = (double)ceil_div((int64_t)m->n_out, pad) * pad;
            const double s_eff = std::max(1, std::min(cfg.splits, m->kd)), red = s_eff > 1 ? 1 : 0;
            const double a_loads = rows * kdv * l.c_in;
            wr = (s_eff * n_out + red * n_out) * l.c_out;
            rd = a_loads + kdv * unit + red * s_eff * n_out * l.c_out;
        }
        total += (rd + wr) * eb;
    }
    return total;
}

// chained backward over layers [lo, hi] in reverse order: gout[i] (fp32) holds
// dL/d out_i; writes dW_i into the flat buffer and pushes dL/dx into producers
void run_backward(sk_net* n, int hi, int lo, float* wgrad_flat, bool accumulate, cudaStream_t st) {
    const size_t L = n->spec.layers.size();
    size_t max_out = 0, max_in = 0;
    for (size_t i = 0; i < L; ++i) {
        max_out = std::max(max_out, (size_t)n->out_set[i]->n * n->spec.layers[i].c_out);
        max_in = std::max(max_in, (size_t)n->in_set[i]->n * n->spec.layers[i].c_in);
    }
    DevBuf dy, dx;
    dy.alloc(std::max<size_t>(max_out, 1) * n->es(), st);
    dx.alloc(std::max<size_t>(max_in, 1) * n->es(), st);
    if (!accumulate) {  // the range's weight gradients are contiguous: one fill, not one per layer
        const size_t a = n->wgrad_off[lo];
        const size_t b = n->wgrad_off[hi] + (size_t)n->kd[hi] * n->spec.layers[hi].c_in *
                                                n->spec.layers[hi].c_out;
        fill_async(wgrad_flat + a, 0, (b - a) * 4, st);
    }
    for (int i = hi; i >= lo; --i) {
        const LayerSpec& l = n->spec.layers[i];
        const long long no = (long long)n->out_set[i]->n * l.c_out;
        const long long ni = (long long)n->in_set[i]->n * l.c_in;
        by_dtype(n->dt, [&](auto tag) {
            using T = decltype(tag);
            launch_pdl(k_cast_from_f32<T>, grid_for((no + 3) / 4), 256, 0, st, n->gout[i], no, (T*)dy.p);
        });
        const int g = n->group_of[i];
        conv_wgrad(n->ctx, n->exec_map[i], layer_cfg(n, 2, i), n->dt, l.c_in, l.c_out, n->x_ptr[i],
                   dy.p, wgrad_flat + n->wgrad_off[i], st, true);  // range zeroed above
        if (l.inputs.empty()) continue;  // no gradient w.r.t. the network input
        if (l.inputs.size() == 1) {
            // single producer: dgrad accumulates straight into its fp32 gradient
            // sum in the conv epilogue (no dx round trip, no k_accum launch)
            const int j = n->spec.index(l.inputs[0]);
            conv_forward(n->ctx, n->exec_map[i], layer_cfg(n, 1, i), n->dt, l.c_in, l.c_out, dy.p,
                         n->w[i].p, nullptr, true, st, nullptr, nullptr, n->gout[j]);
            continue;
        }
        conv_forward(n->ctx, n->exec_map[i], layer_cfg(n, 1, i), n->dt, l.c_in, l.c_out, dy.p,
                     n->w[i].p, dx.p, true, st);
        if (l.inputs.size() == 2) {  // both producers in one pass over dx
            const int j1 = n->spec.index(l.inputs[0]), j2 = n->spec.index(l.inputs[1]);
            by_dtype(n->dt, [&](auto tag) {
                using T = decltype(tag);
                launch_pdl(k_accum2<T>, grid_for((ni + 3) / 4), 256, 0, st, n->gout[j1], n->gout[j2],
                           (const T*)dx.p, ni);
            });
            continue;
        }
        for (const std::string& pn : l.inputs) {
            const int j = n->spec.index(pn);
            by_dtype(n->dt, [&](auto tag) {
                using T = decltype(tag);
                launch_pdl(k_accum<T>, grid_for(ni), 256, 0, st, n->gout[j], (const T*)dx.p, ni);
            });
        }
    }
}

// ---- tuner (tuner.cpp) ----
// tuner.cpp:9-26's 12 entries, then the B200 kernel variants the reference's
// presets cannot name (include/sk200.h sk_tile): one CTA per SM (cta_m 256),
// TMA tile::gather4 producers (load_width 1) and single-slab 32-channel
// stages (cta_k 32) for the sorted implicit GEMM at 1-2 splits, and one
// 128-row tile per work item (cta_m 64) at 1-3 splits
std::vector<sk_dataflow_cfg> default_space() {
    std::vector<sk_dataflow_cfg> sp;
    sk_dataflow_cfg c = default_cfg();
    sp.push_back(c);
    c.kind = SK_FETCH_ON_DEMAND;
    sp.push_back(c);
    for (int s = 0; s <= 4; ++s)
        for (int large = 0; large < 2; ++large) {
            sk_dataflow_cfg ig = default_cfg();
            ig.kind = SK_IMPLICIT_GEMM;
            ig.splits = s;
            ig.tile.cta_n = large ? 0 : 64;  // tile_large = whole C_out per tile
            sp.push_back(ig);
        }
    for (int s = 1; s <= 2; ++s) {
        sk_dataflow_cfg ig = default_cfg();
        ig.kind = SK_IMPLICIT_GEMM;
        ig.splits = s;
        ig.tile.cta_n = 0;
        ig.tile.cta_m = 256;  // one CTA per SM, 16 gather warps
        sp.push_back(ig);
        ig.tile.cta_m = 128;
        ig.tile.load_width = 1;  // TMA tile::gather4
        sp.push_back(ig);
        ig.tile.load_width = 4;
        ig.tile.cta_k = 32;  // single-slab 32-channel stages
        sp.push_back(ig);
    }
    for (int s = 1; s <= 3; ++s) {  // one 128-row tile per work item: small layers fill more SMs
        sk_dataflow_cfg ig = default_cfg();
        ig.kind = SK_IMPLICIT_GEMM;
        ig.splits = s;
        ig.tile.cta_m = 64;
        ig.tile.cta_n = 64;
        sp.push_back(ig);
    }
    return sp;
}

}  // namespace

namespace {
template <class F>
sk_status nguard(F&& f) {
    try {
        f();
        return SK_OK;
    } catch (const sk::Error& e) {
        sk::set_last_error(e.what());
        return e.code;
    } catch (const std::exception& e) {
        sk::set_last_error(e.what());
        return SK_ERR_INTERNAL;
    }
}
inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
}  // namespace

extern "C" {

sk_status sk_net_create(sk_ctx* ctx, int dims, const char* spec_text, sk_dtype dtype, sk_net** out) {
    return nguard([&] {
        validate(dtype == SK_F32 || dtype == SK_F16 || dtype == SK_BF16,
                 "network dtype must be f32, f16 or bf16");
        validate(ctx && out, "null argument");
        auto n = std::make_unique<sk_net>();
        n->ctx = ctx;
        n->dt = dtype;
        n->spec = parse_spec(dims, spec_text);
        n->groups = partition_groups(n->spec);
        const size_t L = n->spec.layers.size();
        n->group_of.assign(L, 0);
        for (size_t g = 0; g < n->groups.size(); ++g)
            for (int li : n->groups[g]) n->group_of[li] = (int)g;
        n->kd.resize(L);
        n->w.resize(L);
        n->wgrad_off.resize(L);
        size_t off = 0;
        for (size_t i = 0; i < L; ++i) {
            const LayerSpec& l = n->spec.layers[i];
            n->kd[i] = dims == 3 ? l.kernel * l.kernel * l.kernel : l.kernel * l.kernel;
            n->w[i].alloc((size_t)n->kd[i] * l.c_in * l.c_out * n->es(), nullptr);
            n->wgrad_off[i] = off;
            off += (size_t)n->kd[i] * l.c_in * l.c_out;
        }
        n->wgrad_total = off;
        for (int ph = 0; ph < 3; ++ph) n->cfg[ph].assign(n->groups.size(), default_cfg());
        plan_fusion(n.get());
        SK_CUDA(cudaStreamSynchronize(nullptr));
        *out = n.release();
    });
}

sk_status sk_net_destroy(sk_net* n) {
    return nguard([&] { delete n; });
}

int sk_net_num_layers(const sk_net* n) { return n ? (int)n->spec.layers.size() : -1; }
int sk_net_num_groups(const sk_net* n) { return n ? (int)n->groups.size() : -1; }
int sk_net_group_of_layer(const sk_net* n, int layer) {
    return n && layer >= 0 && layer < (int)n->group_of.size() ? n->group_of[layer] : -1;
}

sk_status sk_net_layer_info(const sk_net* n, int layer, int* num_offsets, int* c_in, int* c_out,
                            int64_t* wgrad_offset) {
    return nguard([&] {
        validate(layer >= 0 && layer < (int)n->spec.layers.size(), "layer index out of range");
        *num_offsets = n->kd[layer];
        *c_in = n->spec.layers[layer].c_in;
        *c_out = n->spec.layers[layer].c_out;
        if (wgrad_offset) *wgrad_offset = (int64_t)n->wgrad_off[layer];
    });
}

int64_t sk_net_num_params(const sk_net* n) { return n ? (int64_t)n->wgrad_total : -1; }

sk_status sk_net_weight_ptr(sk_net* n, int layer, void** ptr) {
    return nguard([&] {
        validate(layer >= 0 && layer < (int)n->spec.layers.size(), "layer index out of range");
        *ptr = n->w[layer].p;
        n->wt_dirty = true;  // the caller may write through the pointer
    });
}

sk_status sk_net_set_config(sk_net* n, int group, int phase, const sk_dataflow_cfg* cfg) {
    return nguard([&] {
        validate(group >= 0 && group < (int)n->groups.size(), "group index out of range");
        validate(phase >= 0 && phase < 3, "phase must be 0 (forward), 1 (dgrad) or 2 (wgrad)");
        validate(cfg->splits >= 0 && cfg->kind >= 0 && cfg->kind <= 2, "invalid dataflow config");
        n->cfg[phase][group] = *cfg;
    });
}

sk_status sk_net_get_config(const sk_net* n, int group, int phase, sk_dataflow_cfg* cfg) {
    return nguard([&] {
        validate(group >= 0 && group < (int)n->groups.size(), "group index out of range");
        validate(phase >= 0 && phase < 3, "bad phase");
        *cfg = n->cfg[phase][group];
    });
}

// NetworkRunner::forward (network.cpp:392): returns the last layer's output
// (library-owned, valid until the next forward). mapping_ms / kernel_ms (per
// group, may be NULL) add CUDA-event timing (RunStats) and synchronise.
sk_status sk_net_forward(sk_net* n, sk_coords* in, const void* d_feats, int channels,
                         void* stream, const void** d_out, int* n_out, double* mapping_ms,
                         double* kernel_ms) {
    return nguard([&] {
        PdlScope pdl_scope(n && n->pdl);
        validate(n && in, "null argument");
        std::vector<double> mp(n->groups.size(), 0.0), kr(n->groups.size(), 0.0);
        const bool timed = mapping_ms || kernel_ms;
        run_forward(n, in, d_feats, channels, S(stream), timed ? &mp : nullptr,
                    timed ? &kr : nullptr);
        if (d_out) *d_out = n->out_ptr.back();
        if (n_out) *n_out = n->out_set.back()->n;
        for (size_t g = 0; g < n->groups.size(); ++g) {
            if (mapping_ms) mapping_ms[g] = mp[g];
            if (kernel_ms) kernel_ms[g] = kr[g];
        }
    });
}

// forward with per-layer GPU times (CUDA events, one sync at the end)
sk_status sk_net_forward_profiled(sk_net* n, sk_coords* in, const void* d_feats, int channels,
                                  void* stream, double* layer_ms, double* mapping_ms_total) {
    return nguard([&] {
        PdlScope pdl_scope(n && n->pdl);
        std::vector<double> mp(n->groups.size(), 0.0), lm;
        run_forward(n, in, d_feats, channels, S(stream), &mp, nullptr, &lm);
        for (size_t i = 0; i < lm.size(); ++i) layer_ms[i] = lm[i];
        double t = 0;
        for (double v : mp) t += v;
        if (mapping_ms_total) *mapping_ms_total = t;
    });
}

sk_status sk_net_layer_output(sk_net* n, int layer, const void** d_out, int* rows) {
    return nguard([&] {
        validate(layer >= 0 && layer < (int)n->out_ptr.size(), "no forward output for layer");
        validate(n->fuse_into[layer] < 0,
                 "layer output is fused into its consumer's skip sum (not materialised)");
        *d_out = n->out_ptr[layer];
        *rows = n->out_set[layer]->n;
    });
}

sk_status sk_net_measure(sk_net* n, sk_coords* in, const void* d_feats, int channels, int fwd,
                         int dgrad, int wgrad, void* stream, double* ms) {
    return nguard([&] {
        PdlScope pdl_scope(n && n->pdl);
        *ms = measure(n, in, d_feats, channels, fwd != 0, dgrad != 0, wgrad != 0, S(stream));
    });
}

int64_t sk_net_map_builds(const sk_net* n) { return n ? n->map_builds : -1; }

sk_status sk_net_set_overlap(sk_net* n, int on) {
    return nguard([&] {
        sk::validate(n != nullptr, "null network");
        n->overlap = on != 0;
    });
}

sk_status sk_net_set_pdl(sk_net* n, int on) {
    return nguard([&] {
        sk::validate(n != nullptr, "null network");
        n->pdl = on != 0;
    });
}

sk_status sk_net_set_tune_cold(sk_net* n, int on) {
    return nguard([&] {
        sk::validate(n != nullptr, "null network");
        n->tune_cold = on != 0;
    });
}

sk_status sk_net_group_traffic(sk_net* n, int group, const sk_dataflow_cfg* cfg, void* stream,
                               double* bytes) {
    return nguard([&] {
        validate(group >= 0 && group < (int)n->groups.size(), "group index out of range");
        *bytes = modeled_group_traffic(n, group, *cfg, S(stream));
    });
}

// Chained backward after sk_net_forward. d_grad_out: dL/d(last output) in the
// run dtype; layers [layer_lo, layer_hi] are processed (call with decreasing
// ranges to interleave gradient all-reduce buckets); the first call (layer_hi
// = last layer) seeds the gradient buffers. wgrad_flat: fp32, layout from
// sk_net_layer_info(... wgrad_offset).
sk_status sk_net_backward(sk_net* n, const void* d_grad_out, float* wgrad_flat, int layer_hi,
                          int layer_lo, int accumulate, void* stream) {
    return nguard([&] {
        PdlScope pdl_scope(n && n->pdl);
        const int L = (int)n->spec.layers.size();
        validate(layer_hi < L && layer_lo >= 0 && layer_lo <= layer_hi, "bad layer range");
        validate(n->root_id != 0 && !n->exec_map.empty() && n->exec_map.back() != nullptr,
                 "backward before a successful forward");
        cudaStream_t st = S(stream);
        if (layer_hi == L - 1) {
            // every layer's fp32 output gradient in one slab, zeroed by one fill
            std::vector<size_t> off(L + 1, 0);
            for (int i = 0; i < L; ++i)
                off[i + 1] = off[i] + ((size_t)std::max(n->out_set[i]->n, 1) *
                                           n->spec.layers[i].c_out + 3) / 4 * 4;  // 16 B aligned
            if (n->gout_slab.bytes < off[L] * 4) n->gout_slab.alloc(off[L] * 4, st);
            fill_async(n->gout_slab.p, 0, off[L] * 4, st);
            n->gout.assign(L, nullptr);
            for (int i = 0; i < L; ++i) n->gout[i] = n->gout_slab.as<float>() + off[i];
            const long long no = (long long)n->out_set[L - 1]->n * n->spec.layers[L - 1].c_out;
            by_dtype(n->dt, [&](auto tag) {
                using T = decltype(tag);
                launch_pdl(k_accum<T>, grid_for(no), 256, 0, st, n->gout[L - 1],
                                                         (const T*)d_grad_out, no);
            });
        }
        run_backward(n, layer_hi, layer_lo, wgrad_flat, accumulate != 0, st);
    });
}

// tune_inference / tune_training (tuner.cpp:134-220) over the default
// 12-entry space with a CUDA-event RunnerProbe (warmup, median of runs) on the
// given sample. training: 0 = inference, 1 = workload_pattern, 2 = sparse_mapping.
// log (optional, capacity log_cap entries of {pass, group, space_index, ms}).
sk_status sk_net_tune(sk_net* n, sk_coords* in, const void* d_feats, int channels, int training,
                      int warmup, int runs, void* stream, double* latency_ms, double* log,
                      int log_cap, int* log_len) {
    return nguard([&] {
        PdlScope pdl_scope(n && n->pdl);
        cudaStream_t st = S(stream);
        const std::vector<sk_dataflow_cfg> space = default_space();
        const int G = (int)n->groups.size();
        for (int ph = 0; ph < 3; ++ph) n->cfg[ph].assign(G, default_cfg());
        int nlog = 0;
        auto probe = [&](bool f, bool d, bool w) {
            for (int i = 0; i < warmup; ++i) measure(n, in, d_feats, channels, f, d, w, st);
            std::vector<double> t(std::max(runs, 1));
            for (auto& v : t) v = measure(n, in, d_feats, channels, f, d, w, st);
            std::nth_element(t.begin(), t.begin() + t.size() / 2, t.end());
            return t[t.size() / 2];
        };
        // greedy_pass (tuner.cpp:86-119): groups in first-appearance order,
        // later groups at the default, argmin with ties on (traffic, order)
        auto greedy = [&](int pass, bool f, bool d, bool w,
                          const std::function<void(int, const sk_dataflow_cfg&)>& bind) {
            double last = 0;
            for (int g = 0; g < G; ++g) {
                double best = 1e300, best_tr = 1e300;
                int best_i = -1;
                for (size_t si = 0; si < space.size(); ++si) {
                    bind(g, space[si]);
                    const double ms = probe(f, d, w);
                    const double tr = modeled_group_traffic(n, g, space[si], st);
                    if (log && nlog < log_cap) {
                        log[nlog * 4 + 0] = pass;
                        log[nlog * 4 + 1] = g;
                        log[nlog * 4 + 2] = (double)si;
                        log[nlog * 4 + 3] = ms;
                    }
                    ++nlog;
                    if (ms < best || (ms == best && tr < best_tr)) {
                        best = ms;
                        best_tr = tr;
                        best_i = (int)si;
                    }
                }
                bind(g, space[best_i]);
                last = best;
            }
            return last;
        };
        double lat = 0;
        if (training == 0) {
            lat = greedy(0, true, false, false,
                         [&](int g, const sk_dataflow_cfg& c) { n->cfg[0][g] = c; });
        } else if (training == 1) {  // workload_pattern: (fwd, dgrad) bound, then wgrad
            lat = greedy(0, true, true, false, [&](int g, const sk_dataflow_cfg& c) {
                n->cfg[0][g] = c;
                n->cfg[1][g] = c;
            });
            lat += greedy(1, false, false, true,
                          [&](int g, const sk_dataflow_cfg& c) { n->cfg[2][g] = c; });
        } else {  // sparse_mapping: forward alone, then (dgrad, wgrad) bound
            lat = greedy(0, true, false, false,
                         [&](int g, const sk_dataflow_cfg& c) { n->cfg[0][g] = c; });
            lat += greedy(1, false, true, true, [&](int g, const sk_dataflow_cfg& c) {
                n->cfg[1][g] = c;
                n->cfg[2][g] = c;
            });
        }
        if (latency_ms) *latency_ms = lat;
        if (log_len) *log_len = nlog;
    });
}

int sk_tune_space_size(void) { return (int)default_space().size(); }

sk_status sk_tune_space_entry(int i, sk_dataflow_cfg* cfg) {
    return nguard([&] {
        auto sp = default_space();
        validate(i >= 0 && i < (int)sp.size(), "space index out of range");
        *cfg = sp[i];
    });
}

}  // extern "C"
