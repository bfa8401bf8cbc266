// sparsekit_b200.hpp -- the sparsekit-side shim that routes the reference's
// hot path (kernel maps + the three dataflows, forward / dgrad / wgrad) to
// libsk200.so through its C ABI (include/sk200.h). Header-only: a maintainer
// adds it next to the sparsekit headers (/root/reference/proj/include) and
// links libsk200.so and libcudart. Compiled and exercised by
// integration/shim_check.cpp (oracle/Makefile target `shim`).
//
// Reference interfaces replaced (file:line under /root/reference/proj):
//   SparseTensor coords + CoordLookup      include/sparsekit/tensor.hpp:86-130
//   build_kmap_ws / build_kmap_os          include/sparsekit/kmap.hpp:126-131
//   MapCache::get_ws / get_os              include/sparsekit/kmap.hpp:159-176
//   conv_forward (+ the three executors)   include/sparsekit/exec.hpp:86-107
//   conv_dgrad / conv_wgrad                include/sparsekit/exec.hpp:117-124
//   ValidationError / ContractError        include/sparsekit/common.hpp:19-27
//   ExecContext::deterministic             include/sparsekit/common.hpp:29-32
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sk200.h"
#include "sparsekit/exec.hpp"
#include "sparsekit/kmap.hpp"
#include "sparsekit/tensor.hpp"

namespace sparsekit::b200 {

// sk_status -> the reference's exception types (common.hpp:19-27)
inline void check(sk_status s) {
    if (s == SK_OK) return;
    if (s == SK_ERR_VALIDATION) throw ValidationError(sk_last_error());
    if (s == SK_ERR_CONTRACT) throw ContractError(sk_last_error());
    throw std::runtime_error(std::string("sk200: ") + sk_last_error());
}
inline void cuda_check(cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("cuda: ") + cudaGetErrorString(e));
}

// ExecContext analogue: one per GPU; every call is ordered on its stream.
class Device {
public:
    explicit Device(int device = 0, bool deterministic = false) {
        cuda_check(cudaSetDevice(device));
        check(sk_ctx_create(device, &ctx_));
        check(sk_ctx_set_deterministic(ctx_, deterministic ? 1 : 0));
        cuda_check(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    }
    ~Device() {
        cudaStreamDestroy(st_);
        sk_ctx_destroy(ctx_);
    }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    sk_ctx* ctx() const { return ctx_; }
    cudaStream_t stream() const { return st_; }
    void sync() const { cuda_check(cudaStreamSynchronize(st_)); }

private:
    sk_ctx* ctx_ = nullptr;
    cudaStream_t st_ = nullptr;
};

// a device coordinate set (SparseTensor coords + its CoordLookup)
class Coords {
public:
    Coords() = default;
    explicit Coords(sk_coords* p) : p_(p) {}
    Coords(Coords&& o) noexcept : p_(std::exchange(o.p_, nullptr)) {}
    Coords& operator=(Coords&& o) noexcept {
        std::swap(p_, o.p_);
        return *this;
    }
    ~Coords() {
        if (p_) sk_coords_release(p_);
    }
    sk_coords* get() const { return p_; }

private:
    sk_coords* p_ = nullptr;
};

// a cached kernel map handle (the library owns the map; MapCache semantics)
class Map {
public:
    Map() = default;
    explicit Map(sk_kmap* p) : p_(p) {}
    Map(Map&& o) noexcept : p_(std::exchange(o.p_, nullptr)) {}
    Map& operator=(Map&& o) noexcept {
        std::swap(p_, o.p_);
        return *this;
    }
    ~Map() {
        if (p_) sk_kmap_release(p_);
    }
    sk_kmap* get() const { return p_; }

private:
    sk_kmap* p_ = nullptr;
};

// Coord is {int32 batch; int32 x[3]} = 16 B: a SparseTensor's coordinate
// vector already is the int4 layout sk200 reads.
inline Coords upload(Device& d, const SparseTensor& t) {
    static_assert(sizeof(Coord) == 16, "Coord must be 4 x int32");
    const int32_t tag[3] = {t.stride_tag()[0], t.stride_tag()[1], t.stride_tag()[2]};
    sk_coords* c = nullptr;
    check(sk_coords_create_host(d.ctx(), t.dims(), t.n(),
                                reinterpret_cast<const int32_t*>(t.coords().data()), tag,
                                d.stream(), &c));
    return Coords(c);
}

// build_kmap_ws / build_kmap_os(in, out, stride, OffsetSet(dims, kernel), transposed)
inline Map build_map(Device& d, const Coords& in, const Coords& out, int kernel,
                     const std::array<int, 3>& stride, bool transposed = false) {
    const int32_t s[3] = {stride[0], stride[1], stride[2]};
    sk_kmap* m = nullptr;
    check(sk_kmap_build(d.ctx(), in.get(), out.get(), kernel, s, transposed ? 1 : 0, d.stream(),
                        &m));
    return Map(m);
}

// DataflowConfig -> sk_dataflow_cfg. TilePreset keeps its field names; on
// B200 cta_m is the 128-row MMA tile, the pad multiple of
// prepared maps.
inline sk_dataflow_cfg to_c(const DataflowConfig& c) {
    sk_dataflow_cfg r;
    r.kind = c.kind == DataflowKind::gather_gemm_scatter ? SK_GATHER_GEMM_SCATTER
           : c.kind == DataflowKind::fetch_on_demand     ? SK_FETCH_ON_DEMAND
                                                         : SK_IMPLICIT_GEMM;
    r.splits = c.splits;
    r.tile.cta_m = c.tile.cta_m;
    r.tile.cta_n = c.tile.cta_n;
    r.tile.cta_k = c.tile.cta_k;
    r.tile.warp_rows = c.tile.warp_rows;
    r.tile.load_width = c.tile.load_width;
    r.reorder = c.reorder == ReorderMode::offline ? SK_REORDER_OFFLINE : SK_REORDER_ONLINE;
    return r;
}

namespace detail {
template <class T>
struct DeviceArray {
    T* p = nullptr;
    size_t n = 0;
    DeviceArray(size_t count, cudaStream_t st) : n(count) {
        cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&p), std::max<size_t>(n, 1) * sizeof(T), st));
    }
    ~DeviceArray() {
        if (p) cudaFree(p);
    }
    DeviceArray(const DeviceArray&) = delete;
    DeviceArray& operator=(const DeviceArray&) = delete;
};

// the GPU arithmetic type for a sparsekit precision: f32 rides the fp32 path
// (accumulated in fp64 on the device, rounded once); f64 inputs are rounded
// to f32 (the device has no f64 dataflow), results are widened back
inline std::vector<float> to_f32(const std::vector<double>& v) {
    return std::vector<float>(v.begin(), v.end());
}

template <class T>
inline void upload(DeviceArray<T>& d, const std::vector<T>& h, cudaStream_t st) {
    cuda_check(cudaMemcpyAsync(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, st));
}
}  // namespace detail

// sparsekit::conv_forward(in, w, ws, os, cfg, ctx) with the map given as a
// device handle (the WS/OS host objects never exist on this path)
inline Features conv_forward(Device& d, const Map& map, const Features& in, const WeightTensor& w,
                             const DataflowConfig& cfg) {
    sk_kmap_info info;
    check(sk_kmap_get_info(map.get(), d.stream(), &info));
    if (in.n() != info.n_in) throw ValidationError("feature rows do not match the map's input set");
    if (w.c_in() != in.channels()) throw ValidationError("weight C_in does not match features");
    const cudaStream_t st = d.stream();
    detail::DeviceArray<float> x(in.to_f64().size(), st), wd(w.as_f64().size(), st),
        y((size_t)info.n_out * w.c_out(), st);
    detail::upload(x, detail::to_f32(in.to_f64()), st);
    detail::upload(wd, detail::to_f32(w.as_f64()), st);
    const sk_dataflow_cfg c = to_c(cfg);
    check(sk_conv_forward(d.ctx(), map.get(), &c, SK_F32, w.c_in(), w.c_out(), x.p, wd.p, y.p, st));
    std::vector<float> h(y.n);
    cuda_check(cudaMemcpyAsync(h.data(), y.p, h.size() * sizeof(float), cudaMemcpyDeviceToHost, st));
    d.sync();
    return Features::from_f64(info.n_out, w.c_out(), std::vector<double>(h.begin(), h.end()),
                              in.precision());
}

// sparsekit::conv_dgrad(dy, w, map, cfg, ctx): dy [n_out][c_out] -> dx [n_in][c_in]
inline Features conv_dgrad(Device& d, const Map& map, const Features& dy, const WeightTensor& w,
                           const DataflowConfig& cfg) {
    sk_kmap_info info;
    check(sk_kmap_get_info(map.get(), d.stream(), &info));
    if (dy.n() != info.n_out || dy.channels() != w.c_out())
        throw ValidationError("gradient shape does not match the map / weights");
    const cudaStream_t st = d.stream();
    detail::DeviceArray<float> g(dy.to_f64().size(), st), wd(w.as_f64().size(), st),
        dx((size_t)info.n_in * w.c_in(), st);
    detail::upload(g, detail::to_f32(dy.to_f64()), st);
    detail::upload(wd, detail::to_f32(w.as_f64()), st);
    const sk_dataflow_cfg c = to_c(cfg);
    check(sk_conv_dgrad(d.ctx(), map.get(), &c, SK_F32, w.c_in(), w.c_out(), g.p, wd.p, dx.p, st));
    std::vector<float> h(dx.n);
    cuda_check(cudaMemcpyAsync(h.data(), dx.p, h.size() * sizeof(float), cudaMemcpyDeviceToHost, st));
    d.sync();
    return Features::from_f64(info.n_in, w.c_in(), std::vector<double>(h.begin(), h.end()),
                              dy.precision());
}

// sparsekit::conv_wgrad(x, dy, map, cfg, ctx) -> dW [K^D][c_in][c_out]
inline WeightTensor conv_wgrad(Device& d, const Map& map, const Features& x, const Features& dy,
                               const DataflowConfig& cfg) {
    sk_kmap_info info;
    check(sk_kmap_get_info(map.get(), d.stream(), &info));
    if (x.n() != info.n_in || dy.n() != info.n_out)
        throw ValidationError("feature rows do not match the map");
    const cudaStream_t st = d.stream();
    const size_t cells = (size_t)info.num_offsets * x.channels() * dy.channels();
    detail::DeviceArray<float> xd(x.to_f64().size(), st), g(dy.to_f64().size(), st), dw(cells, st);
    detail::upload(xd, detail::to_f32(x.to_f64()), st);
    detail::upload(g, detail::to_f32(dy.to_f64()), st);
    const sk_dataflow_cfg c = to_c(cfg);
    check(sk_conv_wgrad(d.ctx(), map.get(), &c, SK_F32, x.channels(), dy.channels(), xd.p, g.p,
                        dw.p, st));
    std::vector<float> h(cells);
    cuda_check(cudaMemcpyAsync(h.data(), dw.p, cells * sizeof(float), cudaMemcpyDeviceToHost, st));
    d.sync();
    return WeightTensor(info.num_offsets, x.channels(), dy.channels(),
                        std::vector<double>(h.begin(), h.end()), x.precision());
}

}  // namespace sparsekit::b200
