// ref_shim.cpp -- extern "C" access to the UNMODIFIED reference core.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// reference sources where they lie under /root/reference/proj/core/src
// (nothing is copied into this repo) into oracle/_ref/libltlgrid_ref.so.
// Used to (a) generate tests/golden fixtures, (b) validate the C restatement
// in oracle/ltlg_oracle.c, and (c) time the reference CPU path
// (bench.py --impl reference, cpu_baseline kind "reference").
//
// Every entry point builds the reference's own value types and calls the
// reference's own functions: ltlgrid::label_all (label.cpp:150-189),
// CsrBoolMatrix::validate/save/load (label.cpp:16-40, 251-298),
// LabelMatrix::save/load (label.cpp:300-326), z_index (grid.cpp:108-117),
// save_bitset (grid.cpp:370-390).
#include <chrono>
#include <cstdint>
#include <algorithm>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include "ltlgrid/abstraction.hpp"
#include "ltlgrid/grid.hpp"
#include "ltlgrid/buchi.hpp"
#include "ltlgrid/label.hpp"
#include "ltlgrid/rng.hpp"
#include "ltlgrid/scenario.hpp"

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    return 1;
}

ltlgrid::DensePropMatrix make_props(std::uint64_t cells, int props, const std::uint64_t* colwords) {
    const std::uint64_t wpc = (cells + 63) / 64;
    std::vector<ltlgrid::OccupancyBitset> cols;
    cols.reserve(static_cast<std::size_t>(props));
    for (int j = 0; j < props; ++j) {
        std::vector<std::uint64_t> w(colwords + static_cast<std::uint64_t>(j) * wpc,
                                     colwords + static_cast<std::uint64_t>(j + 1) * wpc);
        cols.push_back(ltlgrid::OccupancyBitset::from_words(cells, std::move(w)));
    }
    return ltlgrid::DensePropMatrix(cells, std::move(cols));
}

void export_labels(const ltlgrid::LabelMatrix& l, std::uint64_t* out) {
    const int wpr = (l.props() + 63) / 64;
    std::memset(out, 0, l.rows() * static_cast<std::uint64_t>(wpr) * sizeof(std::uint64_t));
    for (std::uint64_t i = 0; i < l.rows(); ++i) {
        for (int j = 0; j < l.props(); ++j) {
            if (l.get(i, j)) {
                const std::uint64_t bit = i * static_cast<std::uint64_t>(wpr) * 64 + j;
                out[bit >> 6] |= std::uint64_t{1} << (bit & 63);
            }
        }
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// SplitMix64 stream straight from rng.hpp:10-29 (pins the numpy restatement).
void ref_splitmix_block(std::uint64_t seed, std::uint64_t n, std::uint64_t* out, double* uni) {
    ltlgrid::SplitMix64 a(seed), b(seed);
    for (std::uint64_t i = 0; i < n; ++i) {
        out[i] = a.next();
        uni[i] = b.uniform();
    }
}

std::uint64_t ref_mix_seed(std::uint64_t seed, std::uint64_t stream) { return ltlgrid::mix_seed(seed, stream); }

int ref_hardware_concurrency() { return static_cast<int>(std::thread::hardware_concurrency()); }

// Opaque reference CsrBoolMatrix, built once so timing excludes the copy.
void* ref_csr_create(std::uint64_t rows, std::uint64_t cols, const std::uint64_t* offsets,
                     const std::uint32_t* indices) {
    auto* m = new ltlgrid::CsrBoolMatrix;
    m->rows = rows;
    m->cols = cols;
    m->row_offsets.assign(offsets, offsets + rows + 1);
    m->col_indices.assign(indices, indices + offsets[rows]);
    return m;
}

void ref_csr_free(void* m) { delete static_cast<ltlgrid::CsrBoolMatrix*>(m); }

int ref_csr_validate(std::uint64_t rows, std::uint64_t cols, const std::uint64_t* offsets,
                     std::uint64_t n_offsets, const std::uint32_t* indices, std::uint64_t nnz) {
    try {
        ltlgrid::CsrBoolMatrix m;
        m.rows = rows;
        m.cols = cols;
        m.row_offsets.assign(offsets, offsets + n_offsets);
        m.col_indices.assign(indices, indices + nnz);
        m.validate();
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

void* ref_props_create(std::uint64_t cells, int props, const std::uint64_t* colwords) {
    try {
        return new ltlgrid::DensePropMatrix(make_props(cells, props, colwords));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void ref_props_free(void* p) { delete static_cast<ltlgrid::DensePropMatrix*>(p); }

// Mirrors time_label_ms (scenario.cpp:154-165): best of `repeats` timed
// label_all calls; labels of the last call exported into out (may be null).
double ref_time_label_ms(void* m, void* p, int workers, int repeats, std::uint64_t* out) {
    try {
        const auto& mm = *static_cast<ltlgrid::CsrBoolMatrix*>(m);
        const auto& pp = *static_cast<ltlgrid::DensePropMatrix*>(p);
        double best = std::numeric_limits<double>::infinity();
        ltlgrid::LabelMatrix l;
        for (int r = 0; r < (repeats < 1 ? 1 : repeats); ++r) {
            const auto t0 = std::chrono::steady_clock::now();
            l = ltlgrid::label_all(mm, pp, workers);
            const auto t1 = std::chrono::steady_clock::now();
            const double ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
            if (ms < best) best = ms;
        }
        if (out) export_labels(l, out);
        return best;
    } catch (const std::exception& e) {
        fail(e);
        return -1.0;
    }
}

// One-shot label_all over raw arrays (for goldens / small parity checks).
int ref_label_all(std::uint64_t rows, std::uint64_t cols, const std::uint64_t* offsets,
                  const std::uint32_t* indices, std::uint64_t cells, int props,
                  const std::uint64_t* colwords, int workers, std::uint64_t* out) {
    try {
        ltlgrid::CsrBoolMatrix m;
        m.rows = rows;
        m.cols = cols;
        m.row_offsets.assign(offsets, offsets + rows + 1);
        m.col_indices.assign(indices, indices + offsets[rows]);
        auto p = make_props(cells, props, colwords);
        auto l = ltlgrid::label_all(m, p, workers);
        export_labels(l, out);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_label_edge_counting(const std::uint32_t* row, std::uint64_t n, std::uint64_t cells,
                            const std::uint64_t* column, std::uint64_t* examined) {
    std::vector<std::uint64_t> w(column, column + (cells + 63) / 64);
    auto col = ltlgrid::OccupancyBitset::from_words(cells, std::move(w));
    auto [hit, e] = ltlgrid::label_edge_counting({row, n}, col);
    *examined = e;
    return hit ? 1 : 0;
}

int ref_csr_save(const char* path, std::uint64_t rows, std::uint64_t cols,
                 const std::uint64_t* offsets, const std::uint32_t* indices) {
    try {
        ltlgrid::CsrBoolMatrix m;
        m.rows = rows;
        m.cols = cols;
        m.row_offsets.assign(offsets, offsets + rows + 1);
        m.col_indices.assign(indices, indices + offsets[rows]);
        m.save(path);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Loads a CSB1 file; returns nnz (or -1) and fills the caller's buffers
// when they are non-null (call twice: sizes, then data).
std::int64_t ref_csr_load(const char* path, std::uint64_t* rows, std::uint64_t* cols,
                          std::uint64_t* offsets, std::uint32_t* indices) {
    try {
        auto m = ltlgrid::CsrBoolMatrix::load(path);
        *rows = m.rows;
        *cols = m.cols;
        if (offsets) std::memcpy(offsets, m.row_offsets.data(), m.row_offsets.size() * 8);
        if (indices) std::memcpy(indices, m.col_indices.data(), m.col_indices.size() * 4);
        return static_cast<std::int64_t>(m.nnz());
    } catch (const std::exception& e) {
        fail(e);
        return -1;
    }
}

int ref_label_save(const char* path, std::uint64_t rows, int props, const std::uint64_t* words) {
    try {
        ltlgrid::LabelMatrix l(rows, props);
        const int wpr = (props + 63) / 64;
        for (std::uint64_t i = 0; i < rows; ++i)
            for (int j = 0; j < props; ++j) {
                const std::uint64_t bit = i * static_cast<std::uint64_t>(wpr) * 64 + j;
                if ((words[bit >> 6] >> (bit & 63)) & 1u) l.set(i, j);
            }
        l.save(path);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// LabelMatrix::load (label.cpp:311-326): shape into rows/props; words into
// out when cap (u64 words) suffices. Returns 0 ok, 1 error (ref_last_error).
int ref_label_load(const char* path, std::uint64_t* rows, int* props, std::uint64_t* out, std::uint64_t cap) {
    try {
        const ltlgrid::LabelMatrix l = ltlgrid::LabelMatrix::load(path);
        *rows = l.rows();
        *props = l.props();
        const std::uint64_t n = l.rows() * static_cast<std::uint64_t>((l.props() + 63) / 64);
        if (out && n <= cap) export_labels(l, out);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// LabelMatrix::to_csv (label.cpp:328-344) with an Alphabet of `names`
// ('\n'-separated). Returns the CSV length (written to out if cap suffices),
// or -1 on error.
std::int64_t ref_label_to_csv(std::uint64_t rows, int props, const std::uint64_t* words, const char* names,
                              char* out, std::uint64_t cap) {
    try {
        ltlgrid::LabelMatrix l(rows, props);
        const int wpr = (props + 63) / 64;
        for (std::uint64_t i = 0; i < rows; ++i)
            for (int j = 0; j < props; ++j) {
                const std::uint64_t bit = i * static_cast<std::uint64_t>(wpr) * 64 + j;
                if ((words[bit >> 6] >> (bit & 63)) & 1u) l.set(i, j);
            }
        std::vector<std::string> nm;
        std::string cur;
        for (const char* c = names; *c; ++c) {
            if (*c == '\n') {
                nm.push_back(cur);
                cur.clear();
            } else {
                cur.push_back(*c);
            }
        }
        if (!cur.empty()) nm.push_back(cur);
        const ltlgrid::Alphabet a(nm);
        const std::string csv = l.to_csv(a);
        if (out && csv.size() <= cap) std::memcpy(out, csv.data(), csv.size());
        return static_cast<std::int64_t>(csv.size());
    } catch (const std::exception& e) {
        fail(e);
        return -1;
    }
}

// to_csr (label.cpp:42-57) of `rows` dense bitset rows of `cols` bits each
// (u64 words, ceil(cols/64) per row). Returns nnz, or -1 on error; offsets /
// indices written when nnz <= cap.
std::int64_t ref_to_csr(std::uint64_t rows, std::uint64_t cols, const std::uint64_t* words, std::uint64_t* offsets,
                        std::uint32_t* indices, std::uint64_t cap) {
    try {
        const std::uint64_t wpr = (cols + 63) / 64;
        std::vector<ltlgrid::OccupancyBitset> r;
        for (std::uint64_t i = 0; i < rows; ++i)
            r.push_back(ltlgrid::OccupancyBitset::from_words(
                cols, std::vector<std::uint64_t>(words + i * wpr, words + (i + 1) * wpr)));
        const ltlgrid::CsrBoolMatrix m = ltlgrid::to_csr(r);
        if (m.col_indices.size() <= cap) {
            std::copy(m.row_offsets.begin(), m.row_offsets.end(), offsets);
            std::copy(m.col_indices.begin(), m.col_indices.end(), indices);
        }
        return static_cast<std::int64_t>(m.col_indices.size());
    } catch (const std::exception& e) {
        fail(e);
        return -1;
    }
}

std::uint64_t ref_z_index(int k, int depth, const double* lo, const double* hi, const double* p) {
    try {
        std::vector<std::pair<double, double>> b;
        for (int i = 0; i < k; ++i) b.emplace_back(lo[i], hi[i]);
        ltlgrid::GridSpec g(std::move(b), depth);
        return ltlgrid::z_index({p, static_cast<std::size_t>(k)}, g);
    } catch (const std::exception& e) {
        fail(e);
        return ~std::uint64_t{0};
    }
}

int ref_save_bitset(const char* path, int k, int depth, const std::uint64_t* words) {
    try {
        std::vector<std::pair<double, double>> b;
        for (int i = 0; i < k; ++i) b.emplace_back(0.0, 1.0);
        ltlgrid::GridSpec g(std::move(b), depth);
        const std::uint64_t bits = std::uint64_t{1} << depth;
        std::vector<std::uint64_t> w(words, words + (bits + 63) / 64);
        ltlgrid::save_bitset(path, ltlgrid::OccupancyBitset::from_words(bits, std::move(w)), g);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Union of rasterize_box (grid.cpp:331-335) over nboxes boxes of a k-D grid
// (GridSpec(bounds, depth)) into out (ceil(2^depth / 64) u64 words).
int ref_rasterize_union(int k, int depth, const double* lo, const double* hi, std::uint64_t nboxes,
                        const double* blo, const double* bhi, std::uint64_t* out) {
    try {
        std::vector<std::pair<double, double>> bounds;
        for (int a = 0; a < k; ++a) bounds.emplace_back(lo[a], hi[a]);
        const ltlgrid::GridSpec g(bounds, depth);
        const std::uint64_t words = (g.cell_count() + 63) / 64;
        std::fill(out, out + words, 0);
        for (std::uint64_t b = 0; b < nboxes; ++b) {
            ltlgrid::Box box;
            for (int a = 0; a < k; ++a) {
                box.lo.push_back(blo[b * k + a]);
                box.hi.push_back(bhi[b * k + a]);
            }
            const auto bits = ltlgrid::rasterize_box(box, g);
            for (std::uint64_t w = 0; w < words; ++w) out[w] |= bits.words()[w];
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// TransitionGuard::admits (buchi.hpp:20-22) of every (label, guard):
// out[i] bit t = guard t admits labels[i].
void ref_guard_admits(std::uint64_t n, const std::uint64_t* labels, int n_guards, const std::uint64_t* pos,
                      const std::uint64_t* neg, std::uint64_t* out) {
    for (std::uint64_t i = 0; i < n; ++i) {
        ltlgrid::AlphabetSymbol sym;
        sym.bits = labels[i];
        std::uint64_t m = 0;
        for (int t = 0; t < n_guards; ++t) {
            ltlgrid::TransitionGuard g;
            g.positive = pos[t];
            g.negative = neg[t];
            if (g.admits(sym)) m |= std::uint64_t{1} << t;
        }
        out[i] = m;
    }
}

// build_abstraction (abstraction.cpp) with a Rect sampling region: the
// trajectories of its edges, flattened for the swept-volume parity tests.
// Returns a handle; ref_abstraction_sizes / _export read it out.
void* ref_abstraction_create(double x_min, double x_max, double y_min, double y_max, double speed_min,
                             double speed_max, double tau_min, double tau_max, double tau_limit,
                             std::uint64_t target_edges, std::uint64_t seed) {
    try {
        ltlgrid::AbstractionConfig cfg;
        cfg.region = ltlgrid::SampleRegion::Rect;
        cfg.x_min = x_min;
        cfg.x_max = x_max;
        cfg.y_min = y_min;
        cfg.y_max = y_max;
        cfg.speed_min = speed_min;
        cfg.speed_max = speed_max;
        cfg.tau_min = tau_min;
        cfg.tau_max = tau_max;
        cfg.tau_limit = tau_limit;
        cfg.target_edges = target_edges;
        return new ltlgrid::TransitionSystem(ltlgrid::build_abstraction(cfg, seed));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

// The reference benchmark's roadmap: build_abstraction(loop_abstraction_config(
// ScenarioConfig{}, default_bench_grid(depth), target_edges), seed)
// (scenario.cpp:20-46, abstraction.cpp:299).
void* ref_loop_abstraction_create(int depth, std::uint64_t target_edges, std::uint64_t seed) {
    try {
        const ltlgrid::ScenarioConfig cfg;
        const ltlgrid::GridSpec g = ltlgrid::default_bench_grid(depth);
        return new ltlgrid::TransitionSystem(
            ltlgrid::build_abstraction(ltlgrid::loop_abstraction_config(cfg, g, target_edges), seed));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void ref_abstraction_sizes(void* h, std::uint64_t* edges, std::uint64_t* samples) {
    const auto* ts = static_cast<const ltlgrid::TransitionSystem*>(h);
    *edges = ts->num_edges();
    std::uint64_t n = 0;
    for (const auto& tr : ts->trajectories) n += tr.samples.size();
    *samples = n;
}

// sample_off (edges + 1), samples (5 doubles per State5: px, py, heading, speed, tau)
void ref_abstraction_export(void* h, std::uint64_t* sample_off, double* samples) {
    const auto* ts = static_cast<const ltlgrid::TransitionSystem*>(h);
    std::uint64_t n = 0;
    sample_off[0] = 0;
    for (std::size_t e = 0; e < ts->num_edges(); ++e) {
        for (const auto& s : ts->trajectories[e].samples) {
            double* o = samples + 5 * n++;
            o[0] = s.px;
            o[1] = s.py;
            o[2] = s.heading;
            o[3] = s.speed;
            o[4] = s.tau;
        }
        sample_off[e + 1] = n;
    }
}

void ref_abstraction_free(void* h) { delete static_cast<ltlgrid::TransitionSystem*>(h); }

// swept_volume_matrix (label.cpp:75-116) over edges whose trajectories are
// the given samples, on a 3-d GridSpec(bounds, depth).  Writes row_offsets
// (edges + 1) and, when cols_cap >= nnz, cols.  Returns nnz, or -1 (error in
// ref_last_error, prefixed "invalid_argument: " / "domain_error: ").
std::int64_t ref_swept_volume(int depth, const double* lo, const double* hi, double length, double width,
                              double ref_offset, std::uint64_t edges, const std::uint64_t* sample_off,
                              const double* samples, int workers, std::uint64_t* row_offsets, std::uint32_t* cols,
                              std::uint64_t cols_cap) {
    try {
        ltlgrid::TransitionSystem ts;
        ts.trajectories.resize(edges);
        ts.edges.resize(edges);
        for (std::uint64_t e = 0; e < edges; ++e) {
            auto& tr = ts.trajectories[e];
            for (std::uint64_t i = sample_off[e]; i < sample_off[e + 1]; ++i) {
                const double* s = samples + 5 * i;
                tr.samples.push_back(ltlgrid::State5{s[0], s[1], s[2], s[3], s[4]});
            }
        }
        const ltlgrid::GridSpec g({{lo[0], hi[0]}, {lo[1], hi[1]}, {lo[2], hi[2]}}, depth);
        ltlgrid::FootprintSpec f{length, width, ref_offset};
        const auto csr = ltlgrid::swept_volume_matrix(ts, f, g, workers);
        std::copy(csr.row_offsets.begin(), csr.row_offsets.end(), row_offsets);
        if (cols && cols_cap >= csr.col_indices.size())
            std::copy(csr.col_indices.begin(), csr.col_indices.end(), cols);
        return static_cast<std::int64_t>(csr.col_indices.size());
    } catch (const std::domain_error& e) {
        g_err = std::string("domain_error: ") + e.what();
        return -1;
    } catch (const std::invalid_argument& e) {
        g_err = std::string("invalid_argument: ") + e.what();
        return -1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// generate_scenario (scenario.cpp:52-128) on GridSpec({{lo, hi} x 3}, depth):
// out = 2 x ceil(2^depth / 64) words, moving_vehicle then not_nominal_lane.
// cfg = {loop_cx, loop_cy, loop_radius, lane_width, agent_speed_min,
// agent_speed_max, agent_length, agent_width, lateral_spread, horizon}.
int ref_generate_scenario(const double* cfg, int agent_count, std::uint64_t seed, const double* lo, const double* hi,
                          int depth, std::uint64_t query_index, std::uint64_t* out) {
    try {
        ltlgrid::ScenarioConfig c;
        c.loop_cx = cfg[0];
        c.loop_cy = cfg[1];
        c.loop_radius = cfg[2];
        c.lane_width = cfg[3];
        c.agent_speed_min = cfg[4];
        c.agent_speed_max = cfg[5];
        c.agent_length = cfg[6];
        c.agent_width = cfg[7];
        c.lateral_spread = cfg[8];
        c.horizon = cfg[9];
        c.agent_count = agent_count;
        c.seed = seed;
        const ltlgrid::GridSpec g({{lo[0], hi[0]}, {lo[1], hi[1]}, {lo[2], hi[2]}}, depth);
        const auto v = ltlgrid::generate_scenario(c, g, query_index);
        const auto a = v.moving_vehicle.words(), b = v.not_nominal_lane.words();
        std::copy(a.begin(), a.end(), out);
        std::copy(b.begin(), b.end(), out + a.size());
        return 0;
    } catch (const std::domain_error& e) {
        g_err = std::string("domain_error: ") + e.what();
        return 1;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
