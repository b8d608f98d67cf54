// ltlgrid_gpu.hpp -- header-only C++ drop-in over the C ABI (ltlgrid_gpu.h).
//
// For code written against the reference core (proj/core/include/ltlgrid/
// label.hpp): include the reference header first, then this one, and switch
//     ltlgrid::label_all(m, p, workers)        (label.hpp:94-98)
// to
//     ltlgrid::gpu::label_all(m, p, workers)
// Same argument meaning, same exception types and messages
// (std::invalid_argument for LTLG_EINVAL -- dimension mismatch label.cpp:151-154,
// > 64 props label.cpp:124, malformed CSR label.cpp:16-40; std::runtime_error for
// file / CUDA failures).  `workers` is accepted and ignored: the result is
// identical for any value (test_label.cpp:121-132).
//
// ltlgrid::gpu::Engine keeps T resident in HBM across frames (the reference
// re-reads its CSR on every call): load once, then submit per frame.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "ltlgrid/abstraction.hpp"  // TransitionSystem / FootprintSpec (swept_volume_matrix, apply_labels)
#include "ltlgrid/alphabet.hpp"     // Alphabet / AlphabetSymbol (apply_labels)
#include "ltlgrid/grid.hpp"
#include "ltlgrid/label.hpp"  // the reference's CsrBoolMatrix / DensePropMatrix / LabelMatrix
#include "ltlgrid_gpu.h"

namespace ltlgrid {
namespace gpu {

[[noreturn]] inline void throw_status(ltlg_status s, const char* msg) {
    if (s == LTLG_EINVAL) throw std::invalid_argument(msg);
    if (s == LTLG_EDOMAIN) throw std::domain_error(msg);
    if (s == LTLG_ENOMEM) throw std::bad_alloc();
    throw std::runtime_error(msg);
}

inline void check(ltlg_status s, const ltlg_ctx* ctx) {
    if (s != LTLG_OK) throw_status(s, ltlg_last_error(ctx));
}

// DensePropMatrix columns -> contiguous column-major words (label.hpp:47-58).
template <class Dense>
std::vector<std::uint64_t> column_words(const Dense& p) {
    std::vector<std::uint64_t> w;
    const std::uint64_t per = (p.cells() + 63) / 64;
    w.reserve(per * static_cast<std::uint64_t>(p.num_props()));
    for (int j = 0; j < p.num_props(); ++j) {
        const auto col = p.column(j).words();
        w.insert(w.end(), col.begin(), col.end());
    }
    return w;
}

// Reference LabelMatrix from LabelMatrix-layout words (label.hpp:61-92).
template <class Labels>
Labels to_label_matrix(std::uint64_t rows, int props, const std::vector<std::uint64_t>& words) {
    Labels out(rows, props);
    const int wpr = (props + 63) / 64;
    for (std::uint64_t i = 0; i < rows; ++i)
        for (int w = 0; w < wpr; ++w) {
            std::uint64_t x = words[i * static_cast<std::uint64_t>(wpr) + static_cast<std::uint64_t>(w)];
            while (x) {
                const int b = __builtin_ctzll(x);
                out.set(i, w * 64 + b);
                x &= x - 1;
            }
        }
    return out;
}

class Engine {
public:
    explicit Engine(const std::vector<int>& devices = {0}) {
        check(ltlg_create(devices.data(), static_cast<int>(devices.size()), &ctx_), nullptr);
    }
    ~Engine() { ltlg_destroy(ctx_); }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    template <class Csr>
    void load_abstraction(const Csr& m) {
        check(ltlg_load_abstraction(ctx_, m.rows, m.cols, m.row_offsets.data(), m.col_indices.data()), ctx_);
    }
    void load_abstraction_file(const std::string& csb1_path) {
        check(ltlg_load_abstraction_file(ctx_, csb1_path.c_str()), ctx_);
    }
    template <class Dense>
    void submit(const Dense& p) {
        const auto w = column_words(p);
        check(ltlg_submit_grid(ctx_, p.cells(), p.num_props(), w.data(), 1), ctx_);
    }
    template <class Labels>
    Labels labels(int frame = 0) {
        ltlg_info info{};
        check(ltlg_get_info(ctx_, &info), ctx_);
        std::vector<std::uint64_t> words(info.rows * static_cast<std::uint64_t>(info.label_words));
        check(ltlg_get_labels(ctx_, frame, words.empty() ? nullptr : words.data()), ctx_);
        return to_label_matrix<Labels>(info.rows, info.props, words);
    }
    // Drop-in for ltlgrid::apply_labels (label.cpp:191-210) over this engine's
    // labels of `frame`: same checks, order, exception type and messages.
    EdgeLabeling apply_labels(const TransitionSystem& s, const Alphabet& alphabet, int frame = 0) {
        std::vector<std::uint64_t> sym(s.num_edges());
        check(ltlg_apply_labels(ctx_, frame, s.num_edges(), alphabet.size(), sym.empty() ? nullptr : sym.data()),
              ctx_);
        EdgeLabeling out;
        out.alphabet_size = alphabet.size();
        out.labels.resize(sym.size());
        for (std::size_t i = 0; i < sym.size(); ++i) out.labels[i].bits = sym[i];
        return out;
    }
    ltlg_ctx* handle() const { return ctx_; }

private:
    ltlg_ctx* ctx_ = nullptr;
};

// Drop-in for ltlgrid::label_all (label.cpp:150-189): same checks in the
// reference's order (DensePropMatrix already enforced <= 64 props; then the
// dimension check of label.cpp:151-154), same result bits.
inline LabelMatrix label_all(const CsrBoolMatrix& m, const DensePropMatrix& p, int workers = 0) {
    const auto w = column_words(p);
    const int wpr = (p.num_props() + 63) / 64;
    std::vector<std::uint64_t> words(m.rows * static_cast<std::uint64_t>(wpr));
    const ltlg_status s =
        ltlg_label_all(m.rows, m.cols, m.row_offsets.data(), m.col_indices.data(), p.cells(), p.num_props(),
                       w.empty() ? nullptr : w.data(), workers, words.empty() ? nullptr : words.data());
    if (s != LTLG_OK) throw_status(s, ltlg_last_error(nullptr));
    return to_label_matrix<LabelMatrix>(m.rows, p.num_props(), words);
}

// Drop-in for ltlgrid::swept_volume_matrix (label.hpp:42-43, label.cpp:75-116):
// the same CSR, built on the GPU; same exception types and messages.
inline CsrBoolMatrix swept_volume_matrix(const TransitionSystem& s, const FootprintSpec& f, const GridSpec& g,
                                         int workers = 0, int device = 0) {
    (void)workers;
    ltlg_gridk grid{};
    grid.dims = g.dims();
    grid.depth = g.depth();
    for (int a = 0; a < g.dims() && a < 4; ++a) {
        grid.lo[a] = g.lower(a);
        grid.hi[a] = g.upper(a);
    }
    std::vector<std::uint64_t> off(s.num_edges() + 1, 0);
    std::vector<double> samples;
    for (std::size_t e = 0; e < s.num_edges(); ++e) {
        for (const State5& x : s.trajectories[e].samples)
            samples.insert(samples.end(), {x.px, x.py, x.heading, x.speed, x.tau});
        off[e + 1] = samples.size() / 5;
    }
    const ltlg_footprint fp{f.length, f.width, f.ref_offset};
    ltlg_csr* m = nullptr;
    const ltlg_status st = ltlg_swept_volume(&grid, &fp, s.num_edges(), off.data(),
                                             samples.empty() ? nullptr : samples.data(), device, &m);
    if (st != LTLG_OK) throw_status(st, ltlg_last_error(nullptr));
    CsrBoolMatrix out;
    out.rows = ltlg_csr_rows(m);
    out.cols = ltlg_csr_cols(m);
    out.row_offsets.resize(out.rows + 1);
    out.col_indices.resize(ltlg_csr_nnz(m));
    const ltlg_status cs = ltlg_csr_copy(m, out.row_offsets.data(), out.col_indices.data());
    ltlg_csr_free(m);
    if (cs != LTLG_OK) throw_status(cs, ltlg_last_error(nullptr));
    return out;
}

}  // namespace gpu
}  // namespace ltlgrid
