// Exercises integration/sparsekit_b200.hpp the way a sparsekit caller would:
// reference SparseTensor / Features / WeightTensor / DataflowConfig objects in,
// reference types out, checked against sparsekit::conv_ref / conv_dgrad /
// conv_wgrad of the UNMODIFIED reference library (oracle/_ref) on the frozen
// Fig. 2 instance (tests/golden.hpp:22-84) and seeded random instances
// (golden.hpp:95-125, the reference's own test_exec.cpp:88-116 recipe).
// Built by oracle/Makefile (target `shim`, needs /root/reference headers),
// run on the GPU box by tests/test_gpu_shim.py. Prints "shim ok" on success.
#include <cstdio>

#include "golden.hpp"
#include "sparsekit/exec.hpp"
#include "sparsekit/tuner.hpp"
#include "sparsekit_b200.hpp"

using namespace sparsekit;

namespace {
int failures = 0;
void expect(bool ok, const char* what, double err) {
    std::printf("%-58s max_rel_err %.3g %s\n", what, err, ok ? "ok" : "FAIL");
    if (!ok) ++failures;
}
}  // namespace

int main() {
    b200::Device dev(0);
    const double tol = 1e-5;  // the fp32 path (north_star)

    // Fig. 2 toy instance (D=2, K=3): every default_space config
    {
        SparseTensor in = golden::fig_in(), out = golden::fig_out();
        b200::Coords ci = b200::upload(dev, in), co = b200::upload(dev, out);
        b200::Map m = b200::build_map(dev, ci, co, 3, {1, 1, 1});
        Features x1 = Features::from_f64(5, 1, {1, 2, 3, 4, 5}, Precision::f32);
        WeightTensor w1(9, 1, 1, {1, 2, 3, 4, 5, 6, 7, 8, 9}, Precision::f32);
        auto want1 = golden::fig_conv_c1();
        std::vector<double> wv1(want1.begin(), want1.end());
        double worst = 0;
        for (const DataflowConfig& cfg : default_space())
            worst = std::max(worst, golden::max_rel_err(
                                        b200::conv_forward(dev, m, x1, w1, cfg).to_f64(), wv1));
        expect(worst <= tol, "fig2 C=1, 12 configs vs golden conv", worst);
        std::vector<double> x, w;
        for (int j = 0; j < 5; ++j) {
            x.push_back(j + 1.0);
            x.push_back(2.0 * j);
        }
        for (int k = 0; k < 9; ++k) {
            w.push_back(k + 1.0);
            w.push_back(0.5);
            w.push_back(-1.0);
            w.push_back(k);
        }
        std::vector<double> want2;
        for (const auto& r : golden::fig_conv_c2()) {
            want2.push_back(r[0]);
            want2.push_back(r[1]);
        }
        worst = 0;
        for (const DataflowConfig& cfg : default_space())
            worst = std::max(
                worst, golden::max_rel_err(b200::conv_forward(dev, m,
                                                              Features::from_f64(5, 2, x, Precision::f32),
                                                              WeightTensor(9, 2, 2, w, Precision::f32),
                                                              cfg).to_f64(),
                                           want2));
        expect(worst <= tol, "fig2 C=2, 12 configs vs golden conv", worst);
    }

    // random instances (test_exec.cpp:88-116 recipe) vs the reference
    ExecContext det;
    det.deterministic = true;
    int case_idx = 0;
    for (uint64_t seed : {11u, 12u, 13u}) {
        for (int stride : {1, 2}) {
            const int cin = (case_idx % 3 == 0) ? 1 : (case_idx % 3 == 1 ? 4 : 16);
            const int cout = (case_idx % 2) ? 4 : 16;
            ++case_idx;
            auto inst = golden::make_random_instance(seed, 300, cin, cout, stride, Precision::f64);
            // the GPU computes on f32-rounded inputs: the reference gets the same values
            std::vector<double> xr, wr;
            for (double v : inst.in.feats().to_f64()) xr.push_back((double)(float)v);
            for (double v : inst.w.as_f64()) wr.push_back((double)(float)v);
            Features xf = Features::from_f64(inst.in.n(), cin, xr, Precision::f64);
            WeightTensor wf(inst.w.num_offsets(), cin, cout, wr, Precision::f64);
            const std::vector<double> ref = conv_ref(xf, wf, inst.ws).to_f64();
            b200::Coords ci = b200::upload(dev, inst.in), co = b200::upload(dev, inst.out);
            b200::Map m = b200::build_map(dev, ci, co, 3, {stride, stride, stride});
            double worst = 0;
            for (const DataflowConfig& cfg : default_space())
                worst = std::max(worst, golden::max_rel_err(
                                            b200::conv_forward(dev, m, xf, wf, cfg).to_f64(), ref));
            char what[96];
            std::snprintf(what, sizeof what, "seed %llu s%d %d->%d fwd, 12 configs vs conv_ref",
                          (unsigned long long)seed, stride, cin, cout);
            expect(worst <= tol, what, worst);
            // backward vs the reference's own dgrad / wgrad (deterministic f64)
            std::vector<double> gv((size_t)inst.out.n() * cout);
            for (size_t i = 0; i < gv.size(); ++i) gv[i] = (double)(float)std::sin(0.37 * i + seed);
            Features dy = Features::from_f64(inst.out.n(), cout, gv, Precision::f64);
            DataflowConfig ggs;
            const std::vector<double> dx_ref = conv_dgrad(dy, wf, inst.ws, ggs, det).to_f64();
            const std::vector<double> dw_ref = conv_wgrad(xf, dy, inst.ws, ggs, det).as_f64();
            double e_dx = 0, e_dw = 0;
            for (const DataflowConfig& cfg : default_space()) {
                e_dx = std::max(e_dx, golden::max_rel_err(
                                          b200::conv_dgrad(dev, m, dy, wf, cfg).to_f64(), dx_ref));
                e_dw = std::max(e_dw, golden::max_rel_err(
                                          b200::conv_wgrad(dev, m, xf, dy, cfg).as_f64(), dw_ref));
            }
            std::snprintf(what, sizeof what, "seed %llu s%d dgrad vs conv_dgrad", (unsigned long long)seed,
                          stride);
            expect(e_dx <= tol, what, e_dx);
            std::snprintf(what, sizeof what, "seed %llu s%d wgrad vs conv_wgrad", (unsigned long long)seed,
                          stride);
            expect(e_dw <= tol, what, e_dw);
        }
    }

    // error conventions: ValidationError for bad input, as the reference throws
    {
        auto inst = golden::make_random_instance(5, 100, 4, 4, 1, Precision::f32);
        b200::Coords ci = b200::upload(dev, inst.in);
        bool threw = false;
        try {
            b200::build_map(dev, ci, ci, 4, {1, 1, 1});  // even kernel (kmap.cpp:60-61)
        } catch (const ValidationError&) {
            threw = true;
        }
        expect(threw, "even kernel size -> ValidationError", 0);
        b200::Map m = b200::build_map(dev, ci, ci, 3, {1, 1, 1});
        DataflowConfig bad;
        bad.kind = DataflowKind::implicit_gemm;
        bad.splits = 28;  // > K^D (kmap.cpp:214-216)
        threw = false;
        try {
            b200::conv_forward(dev, m, inst.in.feats(), inst.w, bad);
        } catch (const ValidationError&) {
            threw = true;
        }
        expect(threw, "splits > K^D -> ValidationError", 0);
    }
    if (failures) {
        std::printf("shim FAILED (%d)\n", failures);
        return 1;
    }
    std::printf("shim ok\n");
    return 0;
}
