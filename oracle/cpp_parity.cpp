// cpp_parity.cpp -- C++ parity driver (TEST INFRASTRUCTURE ONLY).
//
// Built by oracle/Makefile against the UNMODIFIED reference core and the
// product's C++ shim (include/ltlgrid_gpu.hpp -> libltlgrid_gpu.so).  For the
// reference's own test inputs (test_label.cpp:58-153) and seeded synthetic
// scenes it runs ltlgrid::label_all (CPU, reference) and
// ltlgrid::gpu::label_all (B200) and compares them with the reference's
// LabelMatrix::operator== (label.hpp:79).  Needs a GPU to run; exits 0 iff
// every case is bit-identical and the error behaviour matches.
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "ltlgrid/abstraction.hpp"
#include "ltlgrid/label.hpp"
#include "ltlgrid/rng.hpp"
#include "ltlgrid_gpu.hpp"

using namespace ltlgrid;

static std::vector<OccupancyBitset> random_rows(SplitMix64& rng, std::uint64_t rows, std::uint64_t cols,
                                                double density) {
    std::vector<OccupancyBitset> out;
    for (std::uint64_t i = 0; i < rows; ++i) {
        OccupancyBitset r(cols);
        for (std::uint64_t c = 0; c < cols; ++c)
            if (rng.uniform() < density) r.set(c);
        out.push_back(std::move(r));
    }
    return out;
}

static int failures = 0;
static void expect(bool ok, const std::string& what) {
    std::printf("%s %s\n", ok ? "ok  " : "FAIL", what.c_str());
    if (!ok) ++failures;
}

int main() {
    // Eq. 13 worked example (test_label.cpp:13-27, 87-99)
    {
        std::vector<OccupancyBitset> rows;
        for (auto cols : std::vector<std::vector<int>>{{4}, {1, 2}, {0}, {2, 3}, {3}}) {
            OccupancyBitset r(5);
            for (int c : cols) r.set(static_cast<std::uint64_t>(c));
            rows.push_back(r);
        }
        auto csr = to_csr(rows);
        OccupancyBitset col(5);
        col.set(4);
        DensePropMatrix p(5, {col});
        expect(gpu::label_all(csr, p) == label_all(csr, p), "eq13 x column{4}");
        DensePropMatrix pz(5, {OccupancyBitset(5), OccupancyBitset(5)});
        expect(gpu::label_all(csr, pz) == label_all(csr, pz), "eq13 x all-false");
        bool threw = false;
        try {
            gpu::label_all(csr, DensePropMatrix(8, {OccupancyBitset(8)}));
        } catch (const std::invalid_argument& e) {
            threw = std::string(e.what()) == "dimension mismatch: matrix cols 5 vs proposition rows 8";
        }
        expect(threw, "dimension mismatch -> std::invalid_argument, reference message");
    }
    // test_label.cpp:111-119 and :121-132
    {
        SplitMix64 rng(11);
        auto rows = random_rows(rng, 1000, 4096, 1e-3);
        auto cols = random_rows(rng, 3, 4096, 0.5);
        auto csr = to_csr(rows);
        DensePropMatrix p(4096, {cols[0], cols[1], cols[2]});
        expect(gpu::label_all(csr, p) == label_all(csr, p), "seed 11: 1000x4096 @1e-3 x 3 @0.5");
        SplitMix64 r2(77);
        auto rows2 = random_rows(r2, 333, 1024, 0.01);
        auto cols2 = random_rows(r2, 2, 1024, 0.4);
        auto csr2 = to_csr(rows2);
        DensePropMatrix p2(1024, {cols2[0], cols2[1]});
        const auto ref = label_all(csr2, p2, 1);
        for (int w : {1, 2, 5}) expect(gpu::label_all(csr2, p2, w) == ref, "seed 77 workers=" + std::to_string(w));
    }
    // resident engine across frames vs per-frame reference calls
    {
        SplitMix64 rng(2024);
        auto rows = random_rows(rng, 700, 16384, 0.002);
        auto csr = to_csr(rows);
        gpu::Engine eng;
        eng.load_abstraction(csr);
        for (int f = 0; f < 5; ++f) {
            auto cols = random_rows(rng, 20, 16384, 0.003 * (f + 1));
            DensePropMatrix p(16384, cols);
            eng.submit(p);
            expect(eng.labels<LabelMatrix>() == label_all(csr, p), "engine frame " + std::to_string(f));
        }
        // apply_labels (label.cpp:191-210): the EdgeLabeling hand-off
        std::vector<std::string> names;
        for (int j = 0; j < 20; ++j) names.push_back("p" + std::to_string(j));
        const Alphabet alphabet(names);
        TransitionSystem ts;
        ts.edges.resize(700);
        auto cols = random_rows(rng, 20, 16384, 0.004);
        DensePropMatrix p(16384, cols);
        eng.submit(p);
        const EdgeLabeling want = apply_labels(ts, label_all(csr, p), alphabet);
        const EdgeLabeling got = eng.apply_labels(ts, alphabet);
        expect(got.alphabet_size == want.alphabet_size && got.labels == want.labels, "apply_labels");
        for (int which = 0; which < 2; ++which) {  // row mismatch, then alphabet mismatch
            TransitionSystem t2;
            t2.edges.resize(which ? 700 : 699);
            const Alphabet a2(std::vector<std::string>(names.begin(), names.end() - 1));
            std::string ra, ga;
            try {
                apply_labels(t2, label_all(csr, p), a2);
            } catch (const std::invalid_argument& e) {
                ra = e.what();
            }
            try {
                eng.apply_labels(t2, a2);
            } catch (const std::invalid_argument& e) {
                ga = e.what();
            }
            expect(!ra.empty() && ra == ga, "apply_labels error: " + ra);
        }
    }
    // swept_volume_matrix (label.cpp:75-116) vs ltlgrid::gpu::swept_volume_matrix on the
    // reference's own build_abstraction output (test_label.cpp:212-235 configuration)
    {
        AbstractionConfig cfg;
        cfg.region = SampleRegion::Rect;
        cfg.x_min = 0;
        cfg.x_max = 64;
        cfg.y_min = 0;
        cfg.y_max = 64;
        cfg.speed_min = 4;
        cfg.speed_max = 8;
        cfg.tau_min = 0.2;
        cfg.tau_max = 2.5;
        cfg.tau_limit = 3.9;
        for (std::uint64_t target : {50ull, 1500ull}) {
            cfg.target_edges = target;
            auto ts = build_abstraction(cfg, 17);
            for (int depth : {9, 12, 18, 24}) {
                GridSpec g({{0.0, 64.0}, {0.0, 64.0}, {0.0, 4.0}}, depth);
                auto want = swept_volume_matrix(ts, cfg.footprint, g, 2);
                auto got = gpu::swept_volume_matrix(ts, cfg.footprint, g, 2);
                expect(got.rows == want.rows && got.cols == want.cols && got.row_offsets == want.row_offsets &&
                           got.col_indices == want.col_indices,
                       "swept_volume_matrix " + std::to_string(ts.num_edges()) + " edges, depth " +
                           std::to_string(depth));
            }
        }
        TransitionSystem bad;
        bad.trajectories.resize(1);
        bad.edges.resize(1);
        bad.trajectories[0].samples = {State5{9.8, 5, 0, 0, 0.5}};
        GridSpec g({{0.0, 10.0}, {0.0, 10.0}, {0.0, 1.0}}, 9);
        std::string a, b;
        try {
            swept_volume_matrix(bad, FootprintSpec{2.0, 1.0, 0.0}, g, 1);
        } catch (const std::domain_error& e) {
            a = e.what();
        }
        try {
            gpu::swept_volume_matrix(bad, FootprintSpec{2.0, 1.0, 0.0}, g, 1);
        } catch (const std::domain_error& e) {
            b = e.what();
        }
        expect(!a.empty() && a == b, "swept_volume_matrix leaving the workspace -> std::domain_error, same message");
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "PASSED", failures);
    return failures ? 1 : 0;
}
