// synth.cpp -- synthetic workloads for the labeling path (host, deterministic).
//
// Not part of the labeling engine: this library only manufactures inputs of
// the BASELINE configs so that the GPU engine, the CPU oracle and the
// reference core all consume the SAME T and P.
//
// T ("synthetic PRM", SURVEY App. B distributions).  A library of `nprim`
// motion primitives is drawn with SplitMix64(mix_seed(seed, p)) (rng.hpp:10-34):
// heading ~ U(-pi, pi), speed ~ U(8, 14) m/s, steer ~ U(+-0.25) rad,
// accel ~ U(+-1.5) m/s^2 (AbstractionConfig ranges, abstraction.hpp:130-135),
// plus a start offset inside one 32-cell z-word block.  Each primitive is the
// single-track bicycle model integrated with classical RK4 for 0.5 s at
// h = 0.0125 s (wheelbase 2.7 m, VehicleParams abstraction.hpp:36-41); at every
// sample the 4.6 x 2.0 m footprint (ref_offset -1.4 m, FootprintSpec
// abstraction.hpp:58-62) is voxelised with the strict separating-axis
// cell test of rect_cell_overlap (abstraction.cpp:156-169) over the
// overlap_cells candidate range (grid.cpp:49-61).  The swept cells are kept
// relative to the start block, so an edge = primitive id + start block:
// translating by whole z-word blocks leaves every 32-bit mask unchanged and
// only moves the word index (z-order scatter of grid.cpp:151-170), which makes
// row i a pure function of (seed, i) -- any row range can be generated
// independently, bit-identically, on any host.
//
// P (two archetypes of scenario.cpp:61-130, restated for a 2-D grid, SURVEY
// 8(d)): prop 0 "not_nominal_lane" = cells with |y - n/2| > 0.05 n (~90%);
// props 1.. "moving_vehicle" = union of 6 axis-aligned boxes of side n/20
// cells at SplitMix64(mix_seed(seed, frame)) positions (~1.5% each).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

struct Rng {
    uint64_t s;
    uint64_t next() {
        uint64_t z = (s += 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    uint64_t below(uint64_t n) { return n ? next() % n : 0; }
};

uint64_t mix_seed(uint64_t seed, uint64_t stream) {
    Rng r{seed ^ (stream * 0x9e3779b97f4a7c15ull + 0x2545f4914f6cdd1dull)};
    return r.next();
}

constexpr double kPi = 3.14159265358979323846;

// k = 2 z-order grid of 2^depth cells over [0, extent)^2.
struct Grid {
    int depth, bx, by;  // bits of axis 0 (x) and axis 1 (y)
    double extent;
    std::vector<uint64_t> sx, sy;  // ZScatter tables (grid.cpp:151-170)
    int blk_x, blk_y;              // cells per 32-bit word block along x / y
    Grid(int d, double e) : depth(d), extent(e) {
        bx = d / 2 + (d % 2);
        by = d / 2;
        sx.assign(1ull << bx, 0);
        sy.assign(1ull << by, 0);
        for (int a = 0; a < 2; ++a) {
            auto& t = a ? sy : sx;
            const int bits = a ? by : bx;
            for (uint64_t c = 0; c < t.size(); ++c) {
                uint64_t v = 0;
                for (int b = 0; b < bits; ++b)
                    if ((c >> b) & 1u) {
                        const int level = (bits - 1 - b) * 2 + a;
                        v |= 1ull << (depth - 1 - level);
                    }
                t[c] = v;
            }
        }
        // the low 5 z bits: count how many belong to each axis
        int nx = 0, ny = 0;
        for (int t = 0; t < 5 && t < depth; ++t) ((depth - 1 - t) % 2 == 0 ? nx : ny)++;
        blk_x = 1 << nx;
        blk_y = 1 << ny;
    }
    uint64_t nxc() const { return 1ull << bx; }
    uint64_t nyc() const { return 1ull << by; }
    double cw() const { return extent / static_cast<double>(nxc()); }
    double ch() const { return extent / static_cast<double>(nyc()); }
};

struct Entry {
    int32_t dbx, dby;  // block offset from the start block
    uint32_t mask;
};

struct Prim {
    std::vector<Entry> e;
    int32_t min_bx, max_bx, min_by, max_by;
};

struct State {
    double px, py, h, v;
};

State rhs(const State& x, double steer, double accel, double wb) {
    return {x.v * std::cos(x.h + steer), x.v * std::sin(x.h + steer), x.v / wb * std::sin(steer), accel};
}

Prim make_prim(const Grid& g, uint64_t seed, uint64_t p) {
    Rng r{mix_seed(seed, p)};
    State x{0, 0, r.uniform(-kPi, kPi), r.uniform(8, 14)};
    const double steer = r.uniform(-0.25, 0.25), accel = r.uniform(-1.5, 1.5);
    const double cw = g.cw(), ch = g.ch();
    x.px = r.uniform(0, g.blk_x * cw);  // start inside block (0, 0)
    x.py = r.uniform(0, g.blk_y * ch);
    const double h = 0.0125, wb = 2.7;
    const double L = 4.6, W = 2.0, ref = -1.4;
    std::vector<std::pair<int64_t, int64_t>> cells;
    for (int step = 0; step <= 40; ++step) {
        const double c = std::cos(x.h), s = std::sin(x.h);
        const double cx = x.px + ref * c, cy = x.py + ref * s;
        const double hl = L / 2, hw = W / 2, ac = std::fabs(c), as = std::fabs(s);
        const double ext_x = hl * ac + hw * as, ext_y = hl * as + hw * ac;
        const double half_x = cw / 2, half_y = ch / 2;
        const int64_t x0 = static_cast<int64_t>(std::floor((cx - ext_x) / cw));
        const int64_t x1 = static_cast<int64_t>(std::ceil((cx + ext_x) / cw)) - 1;
        const int64_t y0 = static_cast<int64_t>(std::floor((cy - ext_y) / ch));
        const int64_t y1 = static_cast<int64_t>(std::ceil((cy + ext_y) / ch)) - 1;
        for (int64_t i = x0; i <= x1; ++i) {
            const double ccx = (static_cast<double>(i) + 0.5) * cw;
            for (int64_t j = y0; j <= y1; ++j) {
                const double ccy = (static_cast<double>(j) + 0.5) * ch;
                const double dx = ccx - cx, dy = ccy - cy;
                if (std::fabs(dx) >= half_x + hl * ac + hw * as) continue;
                if (std::fabs(dy) >= half_y + hl * as + hw * ac) continue;
                if (std::fabs(dx * c + dy * s) >= hl + half_x * ac + half_y * as) continue;
                if (std::fabs(-dx * s + dy * c) >= hw + half_x * as + half_y * ac) continue;
                cells.emplace_back(i, j);
            }
        }
        if (step == 40) break;
        const State k1 = rhs(x, steer, accel, wb);
        const State k2 = rhs({x.px + h / 2 * k1.px, x.py + h / 2 * k1.py, x.h + h / 2 * k1.h, x.v + h / 2 * k1.v},
                             steer, accel, wb);
        const State k3 = rhs({x.px + h / 2 * k2.px, x.py + h / 2 * k2.py, x.h + h / 2 * k2.h, x.v + h / 2 * k2.v},
                             steer, accel, wb);
        const State k4 = rhs({x.px + h * k3.px, x.py + h * k3.py, x.h + h * k3.h, x.v + h * k3.v}, steer, accel, wb);
        x.px += h / 6 * (k1.px + 2 * k2.px + 2 * k3.px + k4.px);
        x.py += h / 6 * (k1.py + 2 * k2.py + 2 * k3.py + k4.py);
        x.h += h / 6 * (k1.h + 2 * k2.h + 2 * k3.h + k4.h);
        x.v += h / 6 * (k1.v + 2 * k2.v + 2 * k3.v + k4.v);
    }
    std::sort(cells.begin(), cells.end());
    cells.erase(std::unique(cells.begin(), cells.end()), cells.end());
    // group by block; mask bit = z-scatter of the in-block coordinates
    auto fdiv = [](int64_t a, int64_t b) { return a >= 0 ? a / b : -((-a + b - 1) / b); };
    std::vector<std::pair<std::pair<int32_t, int32_t>, uint32_t>> blocks;
    for (auto [i, j] : cells) {
        const int32_t bi = static_cast<int32_t>(fdiv(i, g.blk_x)), bj = static_cast<int32_t>(fdiv(j, g.blk_y));
        const uint64_t li = static_cast<uint64_t>(i - static_cast<int64_t>(bi) * g.blk_x);
        const uint64_t lj = static_cast<uint64_t>(j - static_cast<int64_t>(bj) * g.blk_y);
        const uint32_t bit = static_cast<uint32_t>((g.sx[li] | g.sy[lj]) & 31u);
        blocks.push_back({{bi, bj}, 1u << bit});
    }
    std::sort(blocks.begin(), blocks.end(),
              [](const auto& a, const auto& b) { return a.first < b.first; });
    Prim pr;
    pr.min_bx = pr.min_by = INT32_MAX;
    pr.max_bx = pr.max_by = INT32_MIN;
    for (size_t k = 0; k < blocks.size();) {
        uint32_t m = 0;
        size_t e = k;
        while (e < blocks.size() && blocks[e].first == blocks[k].first) m |= blocks[e++].second;
        pr.e.push_back({blocks[k].first.first, blocks[k].first.second, m});
        pr.min_bx = std::min(pr.min_bx, blocks[k].first.first);
        pr.max_bx = std::max(pr.max_bx, blocks[k].first.first);
        pr.min_by = std::min(pr.min_by, blocks[k].first.second);
        pr.max_by = std::max(pr.max_by, blocks[k].first.second);
        k = e;
    }
    return pr;
}

struct Prm {
    Grid g;
    uint64_t seed;
    std::vector<Prim> prims;
    Prm(uint64_t s, int depth, double extent, int nprim) : g(depth, extent), seed(s) {
        prims.resize(static_cast<size_t>(nprim));
        const unsigned T = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < T; ++t)
            pool.emplace_back([&, t] {
                for (size_t p = t; p < prims.size(); p += T) prims[p] = make_prim(g, seed, p);
            });
        for (auto& th : pool) th.join();
    }
    // Row i: primitive and start block.
    void edge(uint64_t i, const Prim** pr, int64_t* BX, int64_t* BY) const {
        Rng r{mix_seed(seed ^ 0x5eed0f7ab1e5ull, i)};
        const Prim& p = prims[r.below(prims.size())];
        const double sx = r.uniform(15.0 / 102.4 * g.extent, 87.4 / 102.4 * g.extent);
        const double sy = r.uniform(15.0 / 102.4 * g.extent, 87.4 / 102.4 * g.extent);
        const int64_t nbx = static_cast<int64_t>(g.nxc()) / g.blk_x, nby = static_cast<int64_t>(g.nyc()) / g.blk_y;
        int64_t bx = static_cast<int64_t>(std::floor(sx / (g.blk_x * g.cw())));
        int64_t by = static_cast<int64_t>(std::floor(sy / (g.blk_y * g.ch())));
        bx = std::min(std::max(bx, static_cast<int64_t>(-p.min_bx)), nbx - 1 - p.max_bx);
        by = std::min(std::max(by, static_cast<int64_t>(-p.min_by)), nby - 1 - p.max_by);
        *pr = &p;
        *BX = bx;
        *BY = by;
    }
    uint32_t word_of(int64_t bx, int64_t by) const {
        return static_cast<uint32_t>((g.sx[static_cast<uint64_t>(bx * g.blk_x)] | g.sy[static_cast<uint64_t>(by * g.blk_y)]) >> 5);
    }
};

template <typename F>
void parallel_rows(uint64_t n, F fn) {
    const unsigned T = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    if (n < 4096 || T == 1) {
        fn(uint64_t(0), n);
        return;
    }
    std::vector<std::thread> pool;
    const uint64_t step = (n + T - 1) / T;
    for (unsigned t = 0; t < T; ++t) {
        const uint64_t b = t * step, e = std::min(n, b + step);
        if (b < e) pool.emplace_back(fn, b, e);
    }
    for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

void* synth_prm_create(uint64_t seed, int depth, double extent, int nprim) {
    if (depth < 10 || depth > 30 || nprim < 1) return nullptr;
    return new Prm(seed, depth, extent, nprim);
}

void synth_prm_free(void* h) { delete static_cast<Prm*>(h); }

// Words per row for rows [b, e): out[0..e-b) (no prefix sum).
void synth_prm_row_words(void* h, uint64_t b, uint64_t e, uint64_t* out) {
    const Prm& P = *static_cast<Prm*>(h);
    parallel_rows(e - b, [&](uint64_t lo, uint64_t hi) {
        for (uint64_t k = lo; k < hi; ++k) {
            const Prim* p;
            int64_t bx, by;
            P.edge(b + k, &p, &bx, &by);
            out[k] = p->e.size();
        }
    });
}

// Cells per row for rows [b, e).
void synth_prm_row_cells(void* h, uint64_t b, uint64_t e, uint64_t* out) {
    const Prm& P = *static_cast<Prm*>(h);
    parallel_rows(e - b, [&](uint64_t lo, uint64_t hi) {
        for (uint64_t k = lo; k < hi; ++k) {
            const Prim* p;
            int64_t bx, by;
            P.edge(b + k, &p, &bx, &by);
            uint64_t n = 0;
            for (const Entry& en : p->e) n += static_cast<uint64_t>(__builtin_popcount(en.mask));
            out[k] = n;
        }
    });
}

// Word-CSR of rows [b, e) given offsets (e-b+1, relative, prefix-summed).
void synth_prm_fill_words(void* h, uint64_t b, uint64_t e, const uint64_t* offsets, uint32_t* words,
                          uint32_t* masks) {
    const Prm& P = *static_cast<Prm*>(h);
    parallel_rows(e - b, [&](uint64_t lo, uint64_t hi) {
        std::vector<std::pair<uint32_t, uint32_t>> tmp;
        for (uint64_t k = lo; k < hi; ++k) {
            const Prim* p;
            int64_t bx, by;
            P.edge(b + k, &p, &bx, &by);
            tmp.clear();
            for (const Entry& en : p->e) tmp.push_back({P.word_of(bx + en.dbx, by + en.dby), en.mask});
            std::sort(tmp.begin(), tmp.end());
            uint64_t o = offsets[k];
            for (auto& t : tmp) {
                words[o] = t.first;
                masks[o] = t.second;
                ++o;
            }
        }
    });
}

// Cell CSR (the reference CsrBoolMatrix) of rows [b, e) given cell offsets.
void synth_prm_fill_cells(void* h, uint64_t b, uint64_t e, const uint64_t* offsets, uint32_t* indices) {
    const Prm& P = *static_cast<Prm*>(h);
    parallel_rows(e - b, [&](uint64_t lo, uint64_t hi) {
        std::vector<std::pair<uint32_t, uint32_t>> tmp;
        for (uint64_t k = lo; k < hi; ++k) {
            const Prim* p;
            int64_t bx, by;
            P.edge(b + k, &p, &bx, &by);
            tmp.clear();
            for (const Entry& en : p->e) tmp.push_back({P.word_of(bx + en.dbx, by + en.dby), en.mask});
            std::sort(tmp.begin(), tmp.end());
            uint64_t o = offsets[k];
            for (auto& t : tmp)
                for (uint32_t m = t.second; m; m &= m - 1)
                    indices[o++] = (t.first << 5) | static_cast<uint32_t>(__builtin_ctz(m));
        }
    });
}

// Perception grid for `frames` frames starting at frame f0: out =
// frames x props x ceil(2^depth / 64) u64 words (DensePropMatrix columns).
void synth_props(uint64_t seed, int depth, int props, uint64_t f0, int frames, uint64_t* out) {
    const Grid g(depth, 1.0);
    const uint64_t nw = ((1ull << depth) + 63) / 64;
    const uint64_t nx = g.nxc(), ny = g.nyc();
    std::memset(out, 0, static_cast<size_t>(frames) * props * nw * 8);
    parallel_rows(static_cast<uint64_t>(frames), [&](uint64_t lo, uint64_t hi) {
        for (uint64_t f = lo; f < hi; ++f) {
            uint64_t* fr = out + f * props * nw;
            if (props >= 1) {
                // not_nominal_lane-like: |y - n/2| > 0.05 n  (cell coordinates)
                const double half = static_cast<double>(ny) / 2, band = 0.05 * static_cast<double>(ny);
                for (uint64_t y = 0; y < ny; ++y) {
                    if (std::fabs(static_cast<double>(y) + 0.5 - half) <= band) continue;
                    for (uint64_t x = 0; x < nx; ++x) {
                        const uint64_t z = g.sx[x] | g.sy[y];
                        fr[z >> 6] |= 1ull << (z & 63);
                    }
                }
            }
            Rng r{mix_seed(seed, f0 + f)};
            const uint64_t sx = std::max<uint64_t>(1, nx / 20), sy = std::max<uint64_t>(1, ny / 20);
            for (int j = 1; j < props; ++j) {
                uint64_t* col = fr + static_cast<uint64_t>(j) * nw;
                for (int b = 0; b < 6; ++b) {
                    const uint64_t x0 = r.below(nx - sx + 1), y0 = r.below(ny - sy + 1);
                    for (uint64_t x = x0; x < x0 + sx; ++x)
                        for (uint64_t y = y0; y < y0 + sy; ++y) {
                            const uint64_t z = g.sx[x] | g.sy[y];
                            col[z >> 6] |= 1ull << (z & 63);
                        }
                }
            }
        }
    });
}

}  // extern "C"
