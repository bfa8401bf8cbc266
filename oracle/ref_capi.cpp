// TEST INFRASTRUCTURE — not product code.
//
// A thin extern "C" shim over the UNMODIFIED reference library (sparsekit,
// /root/reference/proj/src/*.cpp, compiled by oracle/Makefile into
// oracle/_ref/libsparsekit_ref.so). It exists so that the Python parity tests
// and bench.py's cpu_baseline / `--impl reference` leg can drive the
// reference's own C++ API (kmap.hpp, exec.hpp, network.hpp, tuner.hpp)
// through ctypes. Nothing in the product (paper_2311_12862_b200/) links or
// loads this file.
//
// Conventions: coordinates are int32[n][4] = (batch, x, y, z); features and
// weights cross the boundary as f64 and are converted to the requested
// reference Precision inside; every entry point returns 0 on success,
// 1 on sparsekit::ValidationError, 2 on sparsekit::ContractError, 5 other.

#include <array>
#include <chrono>
#include <cmath>
#include <random>
#include <cstdint>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "sparsekit/cost.hpp"
#include "sparsekit/exec.hpp"
#include "sparsekit/gen.hpp"
#ifdef SK_REF_IO
#include "sparsekit/io.hpp"
#endif
#include "sparsekit/kmap.hpp"
#include "sparsekit/network.hpp"
#include "sparsekit/tensor.hpp"
#include "sparsekit/tuner.hpp"

using namespace sparsekit;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return 1;
    } catch (const ContractError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}

std::vector<Coord> to_coords(int n, const int32_t* c) {
    std::vector<Coord> v(n);
    for (int i = 0; i < n; ++i) {
        v[i].batch = c[4 * i];
        v[i].x = {c[4 * i + 1], c[4 * i + 2], c[4 * i + 3]};
    }
    return v;
}

std::array<int, 3> to_stride(const int32_t* s) { return {s[0], s[1], s[2]}; }

Precision prec_of(int p) { return p == 1 ? Precision::f64 : Precision::f32; }

DataflowConfig make_cfg(int kind, int splits, int tile_large, int online) {
    DataflowConfig c;
    c.kind = static_cast<DataflowKind>(kind);
    c.splits = splits;
    c.tile = tile_large ? sparsekit::tile_large() : tile_small();
    c.reorder = online ? ReorderMode::online : ReorderMode::offline;
    return c;
}

}  // namespace

struct RefMap {
    KernelMapWS ws;
    KernelMapOS os;        // raw (unsplit) OS map
    KernelMapOS prepared;  // last prepare() result
    int dims = 3;
};

struct RefNet {
    NetworkSpec spec;
    std::unique_ptr<NetworkRunner> runner;
    SparseTensor input;
    GroupAssignment asg;
};

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_out_coords(int dims, int n, const int32_t* coords, const int32_t* stride,
                   int32_t* out, int* n_out) {
    return guard([&] {
        SparseTensor in = SparseTensor::coords_only(dims, to_coords(n, coords));
        SparseTensor o = build_out_coords(in, to_stride(stride));
        *n_out = o.n();
        for (int i = 0; i < o.n(); ++i) {
            const Coord& c = o.coords()[i];
            out[4 * i] = c.batch;
            out[4 * i + 1] = c.x[0];
            out[4 * i + 2] = c.x[1];
            out[4 * i + 3] = c.x[2];
        }
    });
}

int ref_map_build(int dims, int kernel, int n_in, const int32_t* in_coords, int n_out,
                  const int32_t* out_coords, const int32_t* stride, int transposed,
                  RefMap** out) {
    return guard([&] {
        auto m = std::make_unique<RefMap>();
        m->dims = dims;
        SparseTensor in = SparseTensor::coords_only(dims, to_coords(n_in, in_coords));
        SparseTensor o = SparseTensor::coords_only(dims, to_coords(n_out, out_coords));
        m->ws = build_kmap_ws(in, o, to_stride(stride), OffsetSet(dims, kernel),
                              transposed != 0);
        m->os = ws_to_os(m->ws);
        *out = m.release();
    });
}

int ref_map_from_edges(int E, const int32_t* edges, int relations, int n_in, int n_out,
                       RefMap** out) {
    return guard([&] {
        std::vector<std::array<int32_t, 3>> ev(E);
        for (int i = 0; i < E; ++i) ev[i] = {edges[3 * i], edges[3 * i + 1], edges[3 * i + 2]};
        auto* m = new RefMap();
        m->ws = kmap_from_edges(ev, relations, n_in, n_out);
        *out = m;
    });
}

int ref_map_transpose(const RefMap* m, RefMap** out) {
    return guard([&] {
        auto t = std::make_unique<RefMap>();
        t->dims = m->dims;
        t->ws = transpose_map(m->ws);
        if (!m->ws.graph) t->os = transpose_map(m->os);
        *out = t.release();
    });
}

void ref_map_free(RefMap* m) { delete m; }

int ref_map_num_offsets(const RefMap* m) { return m->ws.num_offsets; }
int ref_map_n_in(const RefMap* m) { return m->ws.n_in; }
int ref_map_n_out(const RefMap* m) { return m->ws.n_out; }

// Pair list of one offset: returns count; fills in/out when non-null.
int64_t ref_map_pairs(const RefMap* m, int k, int32_t* in_idx, int32_t* out_idx) {
    const auto& pl = m->ws.pairs[k];
    if (in_idx)
        for (size_t i = 0; i < pl.size(); ++i) {
            in_idx[i] = pl[i].first;
            out_idx[i] = pl[i].second;
        }
    return static_cast<int64_t>(pl.size());
}

// Raw OS map: entries n_out x K^D, masks n_out x mask_words.
int ref_map_os(const RefMap* m, int32_t* entries, uint64_t* masks, int* mask_words) {
    return guard([&] {
        const auto& sp = m->os.splits.at(0);
        std::memcpy(entries, sp.entries.data(), sp.entries.size() * sizeof(int32_t));
        std::memcpy(masks, sp.masks.data(), sp.masks.size() * sizeof(uint64_t));
        *mask_words = sp.mask_words;
    });
}

int ref_map_prepare(RefMap* m, int splits, int pad_multiple) {
    return guard([&] { m->prepared = pad_map(split_and_sort(m->os, splits), pad_multiple); });
}

int ref_prep_num_splits(const RefMap* m) { return static_cast<int>(m->prepared.splits.size()); }

int ref_prep_split_info(const RefMap* m, int s, int* begin, int* end, int* n_rows,
                        int* mask_words) {
    return guard([&] {
        const auto& sp = m->prepared.splits.at(s);
        *begin = sp.offset_begin;
        *end = sp.offset_end;
        *n_rows = sp.n_rows;
        *mask_words = sp.mask_words;
    });
}

int ref_prep_split_data(const RefMap* m, int s, int32_t* entries, int32_t* out_row,
                        uint64_t* masks) {
    return guard([&] {
        const auto& sp = m->prepared.splits.at(s);
        std::memcpy(entries, sp.entries.data(), sp.entries.size() * sizeof(int32_t));
        std::memcpy(out_row, sp.out_row.data(), sp.out_row.size() * sizeof(int32_t));
        std::memcpy(masks, sp.masks.data(), sp.masks.size() * sizeof(uint64_t));
    });
}

int ref_prep_count_macs(const RefMap* m, int warp_rows, int c_in, int c_out,
                        int64_t* effective, int64_t* redundant) {
    return guard([&] {
        TilePreset t = tile_small();
        t.cta_m = warp_rows;
        t.warp_rows = warp_rows;
        auto r = count_macs(m->prepared, t, c_in, c_out);
        *effective = r.first;
        *redundant = r.second;
    });
}

// Forward through conv_forward (exec.cpp:368-383) with a DataflowConfig built
// from (kind, splits, tile_large, online). prec: 0 = f32, 1 = f64.
int ref_conv_forward(const RefMap* m, int kind, int splits, int tile_large, int online,
                     int prec, int deterministic, int threads, int c_in, int c_out,
                     const double* x, const double* w, double* y) {
    return guard([&] {
        Precision p = prec_of(prec);
        Features fx = Features::from_f64(
            m->ws.n_in, c_in, std::vector<double>(x, x + size_t(m->ws.n_in) * c_in), p);
        WeightTensor wt(m->ws.num_offsets, c_in, c_out,
                        std::vector<double>(w, w + size_t(m->ws.num_offsets) * c_in * c_out),
                        p);
        DataflowConfig cfg = make_cfg(kind, splits, tile_large, online);
        ExecContext ctx;
        ctx.threads = threads;
        ctx.deterministic = deterministic != 0;
        KernelMapOS prepared;
        const KernelMapOS* osp = nullptr;
        if (cfg.kind == DataflowKind::implicit_gemm) {
            if (cfg.reorder == ReorderMode::offline) {
                prepared = prepare_os_map(m->os, cfg);
                osp = &prepared;
            } else {
                osp = &m->os;
            }
        }
        std::vector<double> r = conv_forward(fx, wt, &m->ws, osp, cfg, ctx).to_f64();
        std::memcpy(y, r.data(), r.size() * sizeof(double));
    });
}

int ref_conv_ref(const RefMap* m, int prec, int c_in, int c_out, const double* x,
                 const double* w, double* y) {
    return guard([&] {
        Precision p = prec_of(prec);
        Features fx = Features::from_f64(
            m->ws.n_in, c_in, std::vector<double>(x, x + size_t(m->ws.n_in) * c_in), p);
        WeightTensor wt(m->ws.num_offsets, c_in, c_out,
                        std::vector<double>(w, w + size_t(m->ws.num_offsets) * c_in * c_out),
                        p);
        std::vector<double> r = conv_ref(fx, wt, m->ws).to_f64();
        std::memcpy(y, r.data(), r.size() * sizeof(double));
    });
}

int ref_conv_dgrad(const RefMap* m, int kind, int splits, int tile_large, int prec,
                   int deterministic, int threads, int c_in, int c_out, const double* dy,
                   const double* w, double* dx) {
    return guard([&] {
        Precision p = prec_of(prec);
        Features fdy = Features::from_f64(
            m->ws.n_out, c_out, std::vector<double>(dy, dy + size_t(m->ws.n_out) * c_out), p);
        WeightTensor wt(m->ws.num_offsets, c_in, c_out,
                        std::vector<double>(w, w + size_t(m->ws.num_offsets) * c_in * c_out),
                        p);
        ExecContext ctx;
        ctx.threads = threads;
        ctx.deterministic = deterministic != 0;
        std::vector<double> r =
            conv_dgrad(fdy, wt, m->ws, make_cfg(kind, splits, tile_large, 0), ctx).to_f64();
        std::memcpy(dx, r.data(), r.size() * sizeof(double));
    });
}

int ref_conv_wgrad(const RefMap* m, int prec, int threads, int c_in, int c_out,
                   const double* x, const double* dy, double* dw) {
    return guard([&] {
        Precision p = prec_of(prec);
        Features fx = Features::from_f64(
            m->ws.n_in, c_in, std::vector<double>(x, x + size_t(m->ws.n_in) * c_in), p);
        Features fdy = Features::from_f64(
            m->ws.n_out, c_out, std::vector<double>(dy, dy + size_t(m->ws.n_out) * c_out), p);
        ExecContext ctx;
        ctx.threads = threads;
        std::vector<double> r = conv_wgrad(fx, fdy, m->ws, DataflowConfig{}, ctx).as_f64();
        std::memcpy(dw, r.data(), r.size() * sizeof(double));
    });
}

// gen_cloud (gen.cpp:32-85) + quantize (tensor.cpp:87-142), no features
// (occupancy). Two-phase: pass coords=nullptr to get the voxel count.
int ref_gen_voxels(int kind, int n, uint64_t seed, double extent, const double* voxel,
                   int32_t batch, int32_t* coords, int* n_vox) {
    return guard([&] {
        std::vector<double> raw = gen_cloud(static_cast<CloudKind>(kind), n, seed, extent);
        VoxelParams vp;
        vp.voxel_size = {voxel[0], voxel[1], voxel[2]};
        SparseTensor t = quantize(raw, 3, {}, 0, vp, DedupRule::first, Precision::f32);
        *n_vox = t.n();
        if (coords)
            for (int i = 0; i < t.n(); ++i) {
                coords[4 * i] = batch;
                coords[4 * i + 1] = t.coords()[i].x[0];
                coords[4 * i + 2] = t.coords()[i].x[1];
                coords[4 * i + 3] = t.coords()[i].x[2];
            }
    });
}

int ref_gen_cloud(int kind, int n, uint64_t seed, double extent, double* pts) {
    return guard([&] {
        std::vector<double> raw = gen_cloud(static_cast<CloudKind>(kind), n, seed, extent);
        std::memcpy(pts, raw.data(), raw.size() * sizeof(double));
    });
}

// quantize (tensor.cpp:87-142) with features; rule 0 = first, 1 = mean.
// Two-phase like ref_gen_voxels.
int ref_quantize(int dims, int m, const double* raw, int channels, const double* feats,
                 const double* voxel, int rule, const int32_t* batch, int32_t* coords,
                 double* out_feats, int* n_vox) {
    return guard([&] {
        std::vector<double> r(raw, raw + size_t(m) * dims);
        std::vector<double> f;
        if (channels > 0) f.assign(feats, feats + size_t(m) * channels);
        VoxelParams vp;
        vp.voxel_size = {voxel[0], voxel[1], voxel[2]};
        std::vector<int32_t> b;
        if (batch) b.assign(batch, batch + m);
        SparseTensor t = quantize(r, dims, f, channels, vp,
                                  rule ? DedupRule::mean : DedupRule::first, Precision::f64,
                                  batch ? &b : nullptr);
        *n_vox = t.n();
        if (coords) {
            for (int i = 0; i < t.n(); ++i) {
                coords[4 * i] = t.coords()[i].batch;
                coords[4 * i + 1] = t.coords()[i].x[0];
                coords[4 * i + 2] = t.coords()[i].x[1];
                coords[4 * i + 3] = t.coords()[i].x[2];
            }
            std::vector<double> fv = t.feats().to_f64();
            std::memcpy(out_feats, fv.data(), fv.size() * sizeof(double));
        }
    });
}

// --- network (network.cpp) ---------------------------------------------------
// Spec text: one layer per line, "name kind c_in c_out kernel stride inputs
// transpose_of" with inputs a comma list or "-", transpose_of a name or "-".
int ref_net_create(int dims, const char* spec_text, int prec, int threads,
                   uint64_t weight_seed, const double* weights, RefNet** out) {
    return guard([&] {
        auto net = std::make_unique<RefNet>();
        net->spec.dims = dims;
        std::istringstream is(spec_text);
        std::string line;
        while (std::getline(is, line)) {
            if (line.empty()) continue;
            std::istringstream ls(line);
            LayerSpec l;
            std::string kind, inputs, tof;
            ls >> l.name >> kind >> l.c_in >> l.c_out >> l.kernel >> l.stride >> inputs >> tof;
            l.kind = layer_kind_from_string(kind);
            if (inputs != "-") {
                std::stringstream ss(inputs);
                std::string tok;
                while (std::getline(ss, tok, ',')) l.inputs.push_back(tok);
            }
            if (tof != "-") l.transpose_of = tof;
            net->spec.layers.push_back(l);
        }
        net->spec.validate();
        // timing weights N(0, 1/sqrt(K^D c_in)), mt19937_64(seed)
        // weights: caller-provided (flat, layer order) or timing weights
        // N(0, 1/sqrt(K^D c_in)) from mt19937_64(seed)
        std::mt19937_64 rng(weight_seed);
        std::vector<WeightTensor> ws;
        size_t off = 0;
        for (const LayerSpec& l : net->spec.layers) {
            int kd = 1;
            for (int d = 0; d < dims; ++d) kd *= l.kernel;
            std::vector<double> v(size_t(kd) * l.c_in * l.c_out);
            if (weights) {
                std::copy(weights + off, weights + off + v.size(), v.begin());
            } else {
                std::normal_distribution<double> g(0.0, 1.0 / std::sqrt(double(kd) * l.c_in));
                for (double& x : v) x = g(rng);
            }
            off += v.size();
            ws.emplace_back(kd, l.c_in, l.c_out, std::move(v), prec_of(prec));
        }
        ExecContext ctx;
        ctx.threads = threads;
        net->runner = std::make_unique<NetworkRunner>(net->spec, std::move(ws), ctx);
        net->asg = net->runner->default_assignment();
        *out = net.release();
    });
}

void ref_net_free(RefNet* n) { delete n; }

int ref_net_num_groups(const RefNet* n) { return static_cast<int>(n->runner->groups().size()); }

int ref_net_group_of_layer(const RefNet* n, int layer) { return n->runner->group_of_layer(layer); }

int ref_net_set_input(RefNet* n, int n_vox, const int32_t* coords, int channels,
                      const double* feats, int prec) {
    return guard([&] {
        n->input = SparseTensor(
            n->spec.dims, to_coords(n_vox, coords),
            Features::from_f64(n_vox, channels,
                               std::vector<double>(feats, feats + size_t(n_vox) * channels),
                               prec_of(prec)));
    });
}

// One NetworkRunner::forward; *ms = wall time of the call, mapping/kernel
// split summed over groups.
int ref_net_forward(RefNet* n, double* ms, double* mapping_ms, double* kernel_ms) {
    return guard([&] {
        RunStats st;
        auto t0 = std::chrono::steady_clock::now();
        SparseTensor y = n->runner->forward(n->input, n->asg, &st);
        *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                  .count();
        double mp = 0, kr = 0;
        for (auto& g : st.groups) {
            mp += g.mapping_ms;
            kr += g.kernel_ms;
        }
        *mapping_ms = mp;
        *kernel_ms = kr;
    });
}

int ref_net_measure(RefNet* n, int fwd, int dgrad, int wgrad, double* ms) {
    return guard([&] {
        *ms = n->runner->measure_ms(n->input, n->asg, PhaseMask{fwd != 0, dgrad != 0, wgrad != 0});
    });
}

// Output of the last layer (features as f64), n_rows * c_out.
int ref_net_output(RefNet* n, double* y, int* n_rows, int* c_out) {
    return guard([&] {
        SparseTensor out = n->runner->forward(n->input, n->asg, nullptr);
        *n_rows = out.n();
        *c_out = out.channels();
        if (y) {
            std::vector<double> v = out.feats().to_f64();
            std::memcpy(y, v.data(), v.size() * sizeof(double));
        }
    });
}


// NetworkRunner::modeled_group_traffic (network.cpp:453-471) after a forward:
// traffic_model (cost.cpp:47-93) bytes of every layer of `group` under a
// default_space-style config (kind, splits, small/large preset).
int ref_net_group_traffic(RefNet* n, int group, int kind, int splits, int tile_large,
                          double* bytes) {
    return guard([&] {
        *bytes = n->runner->modeled_group_traffic(group, make_cfg(kind, splits, tile_large, 0));
    });
}

#ifdef SK_REF_IO
// ---- io.cpp (TSPW weights, DataflowConfig / TuneResult JSON) ----------------
int ref_tspw_write(const char* path, int n_layers, const int32_t* shapes, const double* vals) {
    return guard([&] {
        std::vector<WeightTensor> w;
        size_t off = 0;
        for (int i = 0; i < n_layers; ++i) {
            const int kd = shapes[3 * i], ci = shapes[3 * i + 1], co = shapes[3 * i + 2];
            const size_t cnt = (size_t)kd * ci * co;
            w.emplace_back(kd, ci, co, std::vector<double>(vals + off, vals + off + cnt),
                           Precision::f64);
            off += cnt;
        }
        write_tspw(path, w);
    });
}

// two calls: vals == nullptr returns the layer count and shapes (cap layers)
int ref_tspw_read(const char* path, int* n_layers, int32_t* shapes, int cap, double* vals) {
    return guard([&] {
        std::vector<WeightTensor> w = read_tspw(path, Precision::f64);
        *n_layers = static_cast<int>(w.size());
        size_t off = 0;
        for (int i = 0; i < (int)w.size() && i < cap; ++i) {
            shapes[3 * i] = w[i].num_offsets();
            shapes[3 * i + 1] = w[i].c_in();
            shapes[3 * i + 2] = w[i].c_out();
            if (vals) {
                std::vector<double> v = w[i].as_f64();
                std::memcpy(vals + off, v.data(), v.size() * sizeof(double));
                off += v.size();
            }
        }
    });
}

// parse a TuneResult JSON and dump it again (canonical form); out_len = bytes
int ref_tune_roundtrip(const char* text, char* out, int cap, int* out_len) {
    return guard([&] {
        const std::string t = tune_result_to_json(tune_result_from_json(text));
        *out_len = static_cast<int>(t.size());
        if (out && cap > (int)t.size()) std::memcpy(out, t.c_str(), t.size() + 1);
    });
}

// the test_net_io.cpp "tune result JSON round-trips" sample, dumped
int ref_tune_sample(char* out, int cap, int* out_len) {
    return guard([&] {
        TuneResult res;
        GroupChoice g;
        g.id = 0;
        g.layer_names = {"c1", "c2"};
        g.forward.kind = DataflowKind::implicit_gemm;
        g.forward.splits = 3;
        g.forward.tile = tile_large();
        DataflowConfig d;
        d.kind = DataflowKind::fetch_on_demand;
        g.dgrad = d;
        res.groups.push_back(g);
        res.latency_ms = 12.5;
        res.seed = 42;
        res.log.push_back({0, 0, g.forward, 3.25});
        const std::string t = tune_result_to_json(res);
        *out_len = static_cast<int>(t.size());
        if (out && cap > (int)t.size()) std::memcpy(out, t.c_str(), t.size() + 1);
    });
}
#endif
}  // extern "C"
