// loader.cpp -- host side of "load abstraction": validate T exactly like the
// reference, bit-pack it into a word-CSR, order rows for z-locality, split it
// into device shards and warp tasks.
//
// Reference behaviour reproduced here:
//   CsrBoolMatrix::validate   proj/core/src/label.cpp:16-40   (checks, order, messages)
//   CsrBoolMatrix::load       proj/core/src/label.cpp:271-298 (CSB1 header, messages)
//   OccupancyBitset layout    proj/core/include/ltlgrid/grid.hpp:93-125 (cell c = word c>>5, bit c&31
//                             of the little-endian u32 view of the u64 words)
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <thread>

#include "engine.h"

#ifndef LTLG_AB_BUILD
#define LTLG_AB_BUILD 0
#endif


namespace ltlg {

int host_threads() {
    unsigned hw = std::thread::hardware_concurrency();
    if (hw == 0) hw = 1;
    return static_cast<int>(std::min(hw, 64u));
}

namespace {

// Run fn(begin, end, chunk_id) over [0, n) in contiguous chunks.
void parallel_chunks(uint64_t n, uint64_t min_chunk,
                     const std::function<void(uint64_t, uint64_t, int)>& fn) {
    int t = host_threads();
    if (n < min_chunk * 2 || t == 1) {
        fn(0, n, 0);
        return;
    }
    uint64_t chunks = std::min<uint64_t>(static_cast<uint64_t>(t), (n + min_chunk - 1) / min_chunk);
    uint64_t step = (n + chunks - 1) / chunks;
    std::vector<std::thread> pool;
    for (uint64_t c = 0; c < chunks; ++c) {
        uint64_t b = c * step, e = std::min(n, b + step);
        if (b >= e) break;
        pool.emplace_back(fn, b, e, static_cast<int>(c));
    }
    for (auto& th : pool) th.join();
}

bool fail(Error* err, Status code, const std::string& msg) {
    if (err) {
        err->code = code;
        err->msg = msg;
    }
    return false;
}

// Offsets checks of validate(), label.cpp:17-31, in the reference's order.
bool check_offsets(uint64_t rows, const uint64_t* offsets, uint64_t n_offsets, uint64_t nnz,
                   Error* err) {
    if (n_offsets != rows + 1) return fail(err, S_EINVAL, "row_offsets must have rows+1 entries");
    if (n_offsets && offsets[0] != 0) return fail(err, S_EINVAL, "row_offsets must start at 0");
    std::atomic<bool> bad{false};
    parallel_chunks(n_offsets ? n_offsets - 1 : 0, 1 << 20, [&](uint64_t b, uint64_t e, int) {
        for (uint64_t i = b; i < e; ++i)
            if (offsets[i] > offsets[i + 1]) {
                bad = true;
                return;
            }
    });
    if (bad) return fail(err, S_EINVAL, "row_offsets must be nondecreasing");
    if (n_offsets && offsets[n_offsets - 1] != nnz) return fail(err, S_EINVAL, "row_offsets must end at nnz");
    return true;
}

}  // namespace

bool validate_csr(uint64_t rows, uint64_t cols, const uint64_t* offsets, uint64_t n_offsets,
                  const uint32_t* indices, uint64_t nnz, Error* err) {
    if (!check_offsets(rows, offsets, n_offsets, nnz, err)) return false;
    // Per-row index checks, label.cpp:32-39: the first failing row (in row
    // order) decides the message; within a row, range before ascending.
    const int T = host_threads();
    std::vector<uint64_t> first_bad(static_cast<size_t>(T) + 1, UINT64_MAX);
    std::vector<int> kind(static_cast<size_t>(T) + 1, 0);
    parallel_chunks(rows, 1 << 14, [&](uint64_t b, uint64_t e, int c) {
        for (uint64_t i = b; i < e; ++i) {
            for (uint64_t k = offsets[i]; k < offsets[i + 1]; ++k) {
                int why = 0;
                if (static_cast<uint64_t>(indices[k]) >= cols) why = 1;
                else if (k > offsets[i] && indices[k - 1] >= indices[k]) why = 2;
                if (why) {
                    first_bad[static_cast<size_t>(c)] = i;
                    kind[static_cast<size_t>(c)] = why;
                    return;
                }
            }
        }
    });
    uint64_t best = UINT64_MAX;
    int why = 0;
    for (size_t c = 0; c < first_bad.size(); ++c)
        if (first_bad[c] < best) {
            best = first_bad[c];
            why = kind[c];
        }
    if (why == 1) return fail(err, S_EINVAL, "column index out of range");
    if (why == 2) return fail(err, S_EINVAL, "column indices must be strictly ascending per row");
    return true;
}

bool pack_csr(uint64_t rows, uint64_t cols, const uint64_t* offsets, const uint32_t* indices,
              WordCsr* out, Error* err) {
    (void)err;
    out->rows = rows;
    out->cols = cols;
    out->nnz = rows ? offsets[rows] : 0;
    out->offsets.assign(rows + 1, 0);
    // pass 1: distinct 32-bit words per row (indices are ascending)
    parallel_chunks(rows, 1 << 14, [&](uint64_t b, uint64_t e, int) {
        for (uint64_t i = b; i < e; ++i) {
            uint64_t n = 0;
            uint32_t last = UINT32_MAX;
            for (uint64_t k = offsets[i]; k < offsets[i + 1]; ++k) {
                const uint32_t w = indices[k] >> 5;
                n += (w != last);
                last = w;
            }
            out->offsets[i + 1] = n;
        }
    });
    for (uint64_t i = 0; i < rows; ++i) out->offsets[i + 1] += out->offsets[i];
    const uint64_t W = out->offsets[rows];
    out->word.assign(W, 0);
    out->mask.assign(W, 0);
    // pass 2: fill (word, mask)
    parallel_chunks(rows, 1 << 14, [&](uint64_t b, uint64_t e, int) {
        for (uint64_t i = b; i < e; ++i) {
            uint64_t o = out->offsets[i] - 1;
            uint32_t last = UINT32_MAX;
            for (uint64_t k = offsets[i]; k < offsets[i + 1]; ++k) {
                const uint32_t c = indices[k];
                const uint32_t w = c >> 5;
                if (w != last) {
                    ++o;
                    out->word[o] = w;
                    last = w;
                }
                out->mask[o] |= 1u << (c & 31);
            }
        }
    });
    return true;
}

bool take_words(uint64_t rows, uint64_t cols, const uint64_t* offsets, const uint32_t* word,
                const uint32_t* mask, WordCsr* out, Error* err) {
    const uint64_t W = rows ? offsets[rows] : 0;
    if (!check_offsets(rows, offsets, rows + 1, W, err)) return false;
    const uint64_t nwords = (cols + 31) / 32;
    const uint32_t tail_bits = static_cast<uint32_t>(cols & 31);
    const uint32_t tail_mask = tail_bits ? ((1u << tail_bits) - 1u) : 0xffffffffu;
    const int T = host_threads();
    std::vector<uint64_t> first_bad(static_cast<size_t>(T) + 1, UINT64_MAX);
    std::vector<int> kind(static_cast<size_t>(T) + 1, 0);
    std::vector<uint64_t> pop(static_cast<size_t>(T) + 1, 0);
    parallel_chunks(rows, 1 << 14, [&](uint64_t b, uint64_t e, int c) {
        uint64_t nnz = 0;
        for (uint64_t i = b; i < e; ++i) {
            for (uint64_t k = offsets[i]; k < offsets[i + 1]; ++k) {
                int why = 0;
                if (word[k] >= nwords || (word[k] == nwords - 1 && (mask[k] & ~tail_mask)))
                    why = 1;
                else if (mask[k] == 0)
                    why = 3;
                else if (k > offsets[i] && word[k - 1] >= word[k])
                    why = 2;
                if (why) {
                    first_bad[static_cast<size_t>(c)] = i;
                    kind[static_cast<size_t>(c)] = why;
                    return;
                }
                nnz += static_cast<uint64_t>(__builtin_popcount(mask[k]));
            }
        }
        pop[static_cast<size_t>(c)] = nnz;
    });
    uint64_t best = UINT64_MAX;
    int why = 0;
    for (size_t c = 0; c < first_bad.size(); ++c)
        if (first_bad[c] < best) {
            best = first_bad[c];
            why = kind[c];
        }
    if (why == 1) return fail(err, S_EINVAL, "column index out of range");
    if (why == 2) return fail(err, S_EINVAL, "column indices must be strictly ascending per row");
    if (why == 3) return fail(err, S_EINVAL, "word masks must be non-zero");
    out->rows = rows;
    out->cols = cols;
    out->nnz = 0;
    for (uint64_t p : pop) out->nnz += p;
    out->offsets.assign(offsets, offsets + rows + 1);
    out->word.assign(word, word + W);
    out->mask.assign(mask, mask + W);
    return true;
}

// CsrBoolMatrix::load, label.cpp:271-298.
bool read_csb1(const char* path, uint64_t* rows, uint64_t* cols, std::vector<uint64_t>* offsets,
               std::vector<uint32_t>* indices, Error* err) {
    const std::string p(path);
    FILE* f = std::fopen(path, "rb");
    if (!f) return fail(err, S_EIO, "cannot open: " + p);
    auto rd = [&](void* dst, size_t n) { return std::fread(dst, 1, n, f) == n; };
    char magic[4];
    if (!rd(magic, 4) || std::memcmp(magic, "CSB1", 4) != 0) {
        std::fclose(f);
        return fail(err, S_EFORMAT, "not a CSR file: " + p);
    }
    uint32_t flags = 0;
    uint64_t nnz = 0;
    bool ok = rd(&flags, 4) && rd(rows, 8) && rd(cols, 8) && rd(&nnz, 8);
    const bool wide = flags & 1u;
    if (ok && *cols > 0xffffffffull) {
        std::fclose(f);
        return fail(err, S_EFORMAT, "CSR column space too large for this build");
    }
    if (ok) {
        try {
            offsets->assign(*rows + 1, 0);
            indices->assign(nnz, 0);
        } catch (...) {
            std::fclose(f);
            return fail(err, S_ENOMEM, "cannot allocate CSR of the declared size: " + p);
        }
        if (wide) {
            ok = rd(offsets->data(), (*rows + 1) * 8);
            std::vector<uint64_t> tmp(1 << 20);
            for (uint64_t done = 0; ok && done < nnz;) {
                const uint64_t n = std::min<uint64_t>(tmp.size(), nnz - done);
                ok = rd(tmp.data(), n * 8);
                for (uint64_t i = 0; ok && i < n; ++i) (*indices)[done + i] = static_cast<uint32_t>(tmp[i]);
                done += n;
            }
        } else {
            std::vector<uint32_t> o32(*rows + 1);
            ok = rd(o32.data(), (*rows + 1) * 4) && rd(indices->data(), nnz * 4);
            for (uint64_t i = 0; i <= *rows; ++i) (*offsets)[i] = o32[i];
        }
    }
    std::fclose(f);
    if (!ok) return fail(err, S_EFORMAT, "truncated CSR file: " + p);
    return validate_csr(*rows, *cols, offsets->data(), offsets->size(), indices->data(), nnz, err);
}

bool read_csb1_words(const char* path, WordCsr* out, Error* err) {
    const std::string p(path);
    FILE* f = std::fopen(path, "rb");
    if (!f) return fail(err, S_EIO, "cannot open: " + p);
    struct Closer {
        FILE* f;
        ~Closer() { std::fclose(f); }
    } closer{f};
    auto rd = [&](void* dst, size_t n) { return std::fread(dst, 1, n, f) == n; };
    char magic[4];
    if (!rd(magic, 4) || std::memcmp(magic, "CSB1", 4) != 0) return fail(err, S_EFORMAT, "not a CSR file: " + p);
    uint32_t flags = 0;
    uint64_t rows = 0, cols = 0, nnz = 0;
    // a header cut short reads as zeros in the reference's get_u* and is then
    // reported as truncated (label.cpp:290)
    const bool hdr = rd(&flags, 4) && rd(&rows, 8) && rd(&cols, 8) && rd(&nnz, 8);
    const bool wide = flags & 1u;
    if (hdr && cols > 0xffffffffull) return fail(err, S_EFORMAT, "CSR column space too large for this build");
    const uint64_t isz = wide ? 8 : 4;
    // truncation is checked before validation (label.cpp:290 then :296): the
    // whole payload must be present
    std::fseek(f, 0, SEEK_END);
    const uint64_t fsize = static_cast<uint64_t>(std::ftell(f));
    const long long data0 = 4 + 4 + 24;
    if (!hdr || (rows + 1) > (UINT64_MAX / isz) ||
        fsize < static_cast<uint64_t>(data0) + (rows + 1) * isz + nnz * isz)
        return fail(err, S_EFORMAT, "truncated CSR file: " + p);
    std::fseek(f, data0, SEEK_SET);
    std::vector<uint64_t> offsets;
    try {
        offsets.assign(rows + 1, 0);
    } catch (...) {
        return fail(err, S_ENOMEM, "cannot allocate CSR of the declared size: " + p);
    }
    if (wide) {
        if (!rd(offsets.data(), (rows + 1) * 8)) return fail(err, S_EFORMAT, "truncated CSR file: " + p);
    } else {
        std::vector<uint32_t> o32(rows + 1);
        if (!rd(o32.data(), (rows + 1) * 4)) return fail(err, S_EFORMAT, "truncated CSR file: " + p);
        for (uint64_t i = 0; i <= rows; ++i) offsets[i] = o32[i];
    }
    if (!check_offsets(rows, offsets.data(), rows + 1, nnz, err)) return false;
    // stream the indices row range by row range: validate (first failing row
    // in row order decides the message, label.cpp:32-39) and pack
    out->rows = rows;
    out->cols = cols;
    out->nnz = nnz;
    out->offsets.assign(rows + 1, 0);
    out->word.clear();
    out->mask.clear();
    constexpr uint64_t kChunk = uint64_t(1) << 24;  // indices per read
    std::vector<uint32_t> idx;
    std::vector<uint64_t> tmp64;
    for (uint64_t r0 = 0; r0 < rows;) {
        uint64_t r1 = r0 + 1;
        while (r1 < rows && offsets[r1 + 1] - offsets[r0] <= kChunk) ++r1;
        const uint64_t k0 = offsets[r0], n = offsets[r1] - k0;
        idx.resize(n);
        if (wide) {
            tmp64.resize(n);
            if (n && !rd(tmp64.data(), n * 8)) return fail(err, S_EFORMAT, "truncated CSR file: " + p);
            for (uint64_t i = 0; i < n; ++i) idx[i] = static_cast<uint32_t>(tmp64[i]);
        } else if (n && !rd(idx.data(), n * 4)) {
            return fail(err, S_EFORMAT, "truncated CSR file: " + p);
        }
        // rows [r0, r1): validate + count words, then fill
        const uint64_t nr = r1 - r0;
        std::vector<uint64_t> cnt(nr + 1, 0);
        const int T = host_threads();
        std::vector<uint64_t> first_bad(static_cast<size_t>(T) + 1, UINT64_MAX);
        std::vector<int> kind(static_cast<size_t>(T) + 1, 0);
        parallel_chunks(nr, 1 << 12, [&](uint64_t b, uint64_t e, int c) {
            for (uint64_t i = b; i < e; ++i) {
                uint64_t words = 0;
                uint32_t last = UINT32_MAX;
                for (uint64_t k = offsets[r0 + i] - k0; k < offsets[r0 + i + 1] - k0; ++k) {
                    int why = 0;
                    if (static_cast<uint64_t>(idx[k]) >= cols) why = 1;
                    else if (k > offsets[r0 + i] - k0 && idx[k - 1] >= idx[k]) why = 2;
                    if (why) {
                        first_bad[static_cast<size_t>(c)] = i;
                        kind[static_cast<size_t>(c)] = why;
                        return;
                    }
                    const uint32_t w = idx[k] >> 5;
                    words += (w != last);
                    last = w;
                }
                cnt[i + 1] = words;
            }
        });
        uint64_t best = UINT64_MAX;
        int why = 0;
        for (size_t c = 0; c < first_bad.size(); ++c)
            if (first_bad[c] < best) {
                best = first_bad[c];
                why = kind[c];
            }
        if (why == 1) return fail(err, S_EINVAL, "column index out of range");
        if (why == 2) return fail(err, S_EINVAL, "column indices must be strictly ascending per row");
        for (uint64_t i = 0; i < nr; ++i) cnt[i + 1] += cnt[i];
        const uint64_t w0 = out->word.size();
        out->word.resize(w0 + cnt[nr], 0);
        out->mask.resize(w0 + cnt[nr], 0);
        for (uint64_t i = 0; i < nr; ++i) out->offsets[r0 + i + 1] = w0 + cnt[i + 1];
        parallel_chunks(nr, 1 << 12, [&](uint64_t b, uint64_t e, int) {
            for (uint64_t i = b; i < e; ++i) {
                uint64_t o = w0 + cnt[i] - 1;
                uint32_t last = UINT32_MAX;
                for (uint64_t k = offsets[r0 + i] - k0; k < offsets[r0 + i + 1] - k0; ++k) {
                    const uint32_t c = idx[k], w = c >> 5;
                    if (w != last) {
                        ++o;
                        out->word[o] = w;
                        last = w;
                    }
                    out->mask[o] |= 1u << (c & 31);
                }
            }
        });
        r0 = r1;
    }
    return true;
}

bool read_zobv(const char* path, uint64_t cells, uint64_t* dst, Error* err) {
    const std::string p(path);
    FILE* f = std::fopen(path, "rb");
    if (!f) return fail(err, S_EIO, "cannot open: " + p);
    struct Closer {
        FILE* f;
        ~Closer() { std::fclose(f); }
    } closer{f};
    unsigned char header[16];
    if (std::fread(header, 1, 16, f) != 16 || std::memcmp(header, "ZOBV", 4) != 0)
        return fail(err, S_EFORMAT, "not a bitset file: " + p);
    const int depth = header[5];
    if (depth < 1 || depth > 63) return fail(err, S_EFORMAT, "corrupt bitset header");
    const uint64_t size_bits = uint64_t(1) << depth, words = (size_bits + 63) / 64;
    // DensePropMatrix(cells, columns): every column is `cells` long (label.cpp:125-127)
    if (size_bits != cells) return fail(err, S_EINVAL, "column length mismatch");
    if (std::fread(dst, 8, words, f) != words) return fail(err, S_EFORMAT, "truncated bitset file: " + p);
    return true;  // 2^depth bits: no tail word to mask (from_words, grid.cpp:201-203)
}

bool write_lbm1(const char* path, uint64_t rows, int props, const uint64_t* words, Error* err) {
    const std::string p(path);
    FILE* f = std::fopen(path, "wb");
    if (!f) return fail(err, S_EIO, "cannot open for writing: " + p);
    const uint32_t version = 1, pr = static_cast<uint32_t>(props);
    const uint64_t n = rows * static_cast<uint64_t>((props + 63) / 64);
    bool ok = std::fwrite("LBM1", 1, 4, f) == 4 && std::fwrite(&version, 4, 1, f) == 1 &&
              std::fwrite(&rows, 8, 1, f) == 1 && std::fwrite(&pr, 4, 1, f) == 1 &&
              (n == 0 || std::fwrite(words, 8, n, f) == n);
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) return fail(err, S_EIO, "write failed: " + p);
    return true;
}

// CsrBoolMatrix::save (label.cpp:251-268): CSB1, little-endian, u32 fields
// unless cols or nnz exceed 32 bits.
bool write_csb1(const char* path, uint64_t rows, uint64_t cols, const uint64_t* offsets, const uint32_t* indices,
                Error* err) {
    const std::string p(path);
    FILE* f = std::fopen(path, "wb");
    if (!f) return fail(err, S_EIO, "cannot open for writing: " + p);
    const uint64_t nnz = offsets[rows];
    const bool wide = cols > 0xffffffffull || nnz > 0xffffffffull;
    const uint32_t flags = wide ? 1u : 0u;
    bool ok = std::fwrite("CSB1", 1, 4, f) == 4 && std::fwrite(&flags, 4, 1, f) == 1 &&
              std::fwrite(&rows, 8, 1, f) == 1 && std::fwrite(&cols, 8, 1, f) == 1 && std::fwrite(&nnz, 8, 1, f) == 1;
    std::vector<uint32_t> buf;
    if (ok && wide) {
        ok = std::fwrite(offsets, 8, rows + 1, f) == rows + 1;
        std::vector<uint64_t> w(1 << 16);
        for (uint64_t i = 0; ok && i < nnz; i += w.size()) {
            const uint64_t n = std::min<uint64_t>(w.size(), nnz - i);
            for (uint64_t k = 0; k < n; ++k) w[k] = indices[i + k];
            ok = std::fwrite(w.data(), 8, n, f) == n;
        }
    } else if (ok) {
        buf.resize(1 << 16);
        for (uint64_t i = 0; ok && i <= rows; i += buf.size()) {
            const uint64_t n = std::min<uint64_t>(buf.size(), rows + 1 - i);
            for (uint64_t k = 0; k < n; ++k) buf[k] = static_cast<uint32_t>(offsets[i + k]);
            ok = std::fwrite(buf.data(), 4, n, f) == n;
        }
        ok = ok && (nnz == 0 || std::fwrite(indices, 4, nnz, f) == nnz);
    }
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) return fail(err, S_EIO, "write failed: " + p);
    return true;
}

std::vector<uint64_t> shard_bounds(const WordCsr& t, int n) {
    std::vector<uint64_t> b(static_cast<size_t>(n) + 1, t.rows);
    b[0] = 0;
    if (n == 1 || t.rows == 0) return b;
    // pairs of row i = max(1, words) (empty rows carry one sentinel pair)
    const uint64_t total = t.offsets[t.rows] + t.rows;  // upper bound proxy: words + rows
    uint64_t acc = 0;
    int s = 1;
    for (uint64_t i = 0; i < t.rows && s < n; ++i) {
        acc += (t.offsets[i + 1] - t.offsets[i]) + 1;
        while (s < n && acc * static_cast<uint64_t>(n) >= total * static_cast<uint64_t>(s)) {
            b[static_cast<size_t>(s)] = i + 1;
            ++s;
        }
    }
    return b;
}

namespace {

// Tasks over rows [start, rows) appended to trow / tpair (no closing entry).
void make_tasks_range(const std::vector<uint64_t>& pair_off, uint64_t start, uint64_t rows, int target,
                      std::vector<uint32_t>* trow, std::vector<uint64_t>* tpair) {
    const uint64_t T = static_cast<uint64_t>(std::max(target, 1));
    while (start < rows) {
        trow->push_back(static_cast<uint32_t>(start));
        tpair->push_back(pair_off[start]);
        // first row whose end passes start_pairs + T (at least one row)
        const uint64_t goal = pair_off[start] + T;
        auto it = std::lower_bound(pair_off.begin() + static_cast<std::ptrdiff_t>(start) + 1,
                                   pair_off.begin() + static_cast<std::ptrdiff_t>(rows) + 1, goal);
        uint64_t end = static_cast<uint64_t>(it - pair_off.begin());
        if (end > rows) end = rows;
        if (end <= start) end = start + 1;
        start = end;
    }
}

// Tasks of every read-back block; block_task[c] = the block's first task.
void make_tasks(const std::vector<uint64_t>& pair_off, const std::vector<uint64_t>& block_row, int target,
                std::vector<uint32_t>* trow, std::vector<uint64_t>* tpair, std::vector<uint32_t>* block_task) {
    trow->clear();
    tpair->clear();
    block_task->clear();
    const size_t nb = block_row.size() - 1;
    for (size_t c = 0; c < nb; ++c) {
        block_task->push_back(static_cast<uint32_t>(trow->size()));
        make_tasks_range(pair_off, block_row[c], block_row[c + 1], target, trow, tpair);
    }
    block_task->push_back(static_cast<uint32_t>(trow->size()));
    const uint64_t rows = block_row[nb];
    trow->push_back(static_cast<uint32_t>(rows));
    tpair->push_back(pair_off[rows]);
}

}  // namespace

// The single-frame copy of the pairs (see kStreamK in engine.h): rows in
// their ORIGINAL order (the single-frame kernel reads the summary from shared
// memory, so it gains nothing from z-locality and stores label i at row i
// without a permutation gather), tasks re-based to even pair offsets, full
// chunks piece-transposed.
void build_stream_layout(const WordCsr& t, uint64_t row_begin, uint64_t row_end, uint32_t sentinel_word,
                         int stream_task_pairs, PackedShard* out) {
    const uint64_t R = row_end - row_begin;
    std::vector<uint64_t> pair_off(R + 1, 0);
    for (uint64_t r = 0; r < R; ++r) {
        const uint64_t n = t.offsets[row_begin + r + 1] - t.offsets[row_begin + r];
        pair_off[r + 1] = pair_off[r] + (n ? n : 1);
    }
    make_tasks(pair_off, out->block_row, stream_task_pairs, &out->task_row_stream, &out->task_pair_stream,
               &out->block_task_stream);
    const size_t nt = out->task_row_stream.size() - 1;
    std::vector<uint64_t> dst_off(nt + 1, 0);
    for (size_t k = 0; k < nt; ++k) {
        const uint64_t n = out->task_pair_stream[k + 1] - out->task_pair_stream[k];
        dst_off[k + 1] = dst_off[k] + n + (n & 1);
    }
    // The 32-cell single-frame copy is only streamed by the A/B knob
    // LTLG_STREAM64=0 (every prop count runs the 64-cell copy by default).
#if LTLG_AB_BUILD  // (the 32-cell single-frame kernels exist in the A/B build only)
    const char* knob = std::getenv("LTLG_STREAM64");
#else
    const char* knob = nullptr;
#endif
    if (!knob || std::atoi(knob) != 0) {
        out->pairs_stream.assign(kPairPad, Pair{0, sentinel_word | kHead});
        out->task_pair_stream = dst_off;
        return;
    }
    out->pairs_stream.assign(dst_off[nt] + kPairPad, Pair{0, sentinel_word | kHead});
    parallel_chunks(nt, 64, [&](uint64_t b, uint64_t e, int) {
        std::vector<Pair> src;
        for (uint64_t k = b; k < e; ++k) {
            // the task's rows in plain order
            src.clear();
            for (uint64_t r = out->task_row_stream[k]; r < out->task_row_stream[k + 1]; ++r) {
                const uint64_t o0 = t.offsets[row_begin + r], o1 = t.offsets[row_begin + r + 1];
                if (o1 == o0) {
                    src.push_back(Pair{0, sentinel_word | kHead});  // empty row: a no-op pair on the zero sentinel word
                    continue;
                }
                for (uint64_t q = o0; q < o1; ++q) src.push_back(Pair{t.mask[q], t.word[q] | (q == o0 ? kHead : 0u)});
            }
            Pair* dst = out->pairs_stream.data() + dst_off[k];
            const uint64_t n = src.size();
            uint64_t c = 0;
            for (; c + kStreamCH <= n; c += kStreamCH)  // full chunks: piece-transposed
                for (uint64_t l = 0; l < 32; ++l)
                    for (uint64_t h = 0; h < kStreamK / 2; ++h)
                        for (uint64_t e2 = 0; e2 < 2; ++e2)
                            dst[c + 2 * (h * 32 + l) + e2] = src[c + kStreamK * l + 2 * h + e2];
            for (; c < n; ++c) dst[c] = src[c];           // last partial chunk: plain
            if (n & 1) dst[n] = Pair{0, sentinel_word};   // no-op pair (no head) to an even count
        }
    });
    out->task_pair_stream = dst_off;
}

// The single-frame 64-cell-word copy (kChunk64Bytes, engine.h), over the
// same tasks (row ranges) as the 32-bit stream copy.
void build_stream64_layout(const WordCsr& t, uint64_t row_begin, uint32_t sentinel64, PackedShard* out) {
    const size_t nt = out->task_row_stream.size() - 1;
    std::vector<uint64_t> bytes(nt + 1, 0);
    out->task_n64.assign(nt, 0);
    // pass 1: pair counts
    parallel_chunks(nt, 64, [&](uint64_t b, uint64_t e, int) {
        for (uint64_t k = b; k < e; ++k) {
            uint64_t n = 0;
            for (uint64_t r = out->task_row_stream[k]; r < out->task_row_stream[k + 1]; ++r) {
                const uint64_t o0 = t.offsets[row_begin + r], o1 = t.offsets[row_begin + r + 1];
                uint64_t cnt = 0;
                for (uint64_t q = o0; q < o1; ++q)
                    if (q == o0 || (t.word[q] >> 1) != (t.word[q - 1] >> 1)) ++cnt;
                n += cnt ? cnt : 1;
            }
            out->task_n64[k] = static_cast<uint32_t>(n);
        }
    });
    for (size_t k = 0; k < nt; ++k) {
        const uint64_t n = out->task_n64[k], full = n / kStreamCH, part = n % kStreamCH;
        bytes[k + 1] = bytes[k] + full * kChunk64Bytes + ((8 * part + 15) & ~uint64_t(15)) + ((4 * part + 15) & ~uint64_t(15));
    }
    out->stream64.assign(bytes[nt] + kPad64Bytes, 0);
    out->task_byte64 = bytes;
    // pass 2: fill
    parallel_chunks(nt, 64, [&](uint64_t b, uint64_t e, int) {
        std::vector<uint64_t> mk;
        std::vector<uint32_t> wd;
        for (uint64_t k = b; k < e; ++k) {
            mk.clear();
            wd.clear();
            for (uint64_t r = out->task_row_stream[k]; r < out->task_row_stream[k + 1]; ++r) {
                const uint64_t o0 = t.offsets[row_begin + r], o1 = t.offsets[row_begin + r + 1];
                if (o1 == o0) {  // empty row: a no-op pair on the zero sentinel word
                    mk.push_back(0);
                    wd.push_back(sentinel64 | kHead);
                    continue;
                }
                for (uint64_t q = o0; q < o1; ++q) {
                    const uint32_t w64 = t.word[q] >> 1;
                    const uint64_t m = static_cast<uint64_t>(t.mask[q]) << (32 * (t.word[q] & 1));
                    if (q > o0 && w64 == (wd.back() & kWordMask)) {
                        mk.back() |= m;
                    } else {
                        mk.push_back(m);
                        wd.push_back(w64 | (q == o0 ? kHead : 0u));
                    }
                }
            }
            uint8_t* dst = out->stream64.data() + bytes[k];
            const uint64_t n = mk.size(), full = n / kStreamCH, part = n % kStreamCH;
            for (uint64_t c = 0; c < full; ++c) {
                uint64_t* dm = reinterpret_cast<uint64_t*>(dst + c * kChunk64Bytes);
                uint32_t* dw = reinterpret_cast<uint32_t*>(dst + c * kChunk64Bytes + 8 * kStreamCH);
                const uint64_t base = c * kStreamCH;
                for (uint64_t l = 0; l < 32; ++l) {
                    for (uint64_t h = 0; h < kStreamK / 2; ++h)
                        for (uint64_t e2 = 0; e2 < 2; ++e2)
                            dm[2 * (h * 32 + l) + e2] = mk[base + kStreamK * l + 2 * h + e2];
                    for (uint64_t h = 0; h < kStreamK / 4; ++h)
                        for (uint64_t e4 = 0; e4 < 4; ++e4)
                            dw[4 * (h * 32 + l) + e4] = wd[base + kStreamK * l + 4 * h + e4];
                }
            }
            if (part) {
                uint8_t* pm = dst + full * kChunk64Bytes;
                std::memcpy(pm, mk.data() + full * kStreamCH, 8 * part);
                std::memcpy(pm + ((8 * part + 15) & ~uint64_t(15)), wd.data() + full * kStreamCH, 4 * part);
            }
        }
    });
}

// The multi-frame 64-cell-word copy (SoA), rows in the batch layout's order.
void build_batch64_layout(const WordCsr& t, uint64_t row_begin, uint32_t sentinel64, PackedShard* out) {
    const uint64_t R = out->perm.size();
    std::vector<uint64_t> off(R + 1, 0);
    parallel_chunks(R, 1 << 14, [&](uint64_t b, uint64_t e, int) {
        for (uint64_t s = b; s < e; ++s) {
            const uint64_t r = row_begin + out->perm[s];
            uint64_t cnt = 0;
            for (uint64_t q = t.offsets[r]; q < t.offsets[r + 1]; ++q)
                if (q == t.offsets[r] || (t.word[q] >> 1) != (t.word[q - 1] >> 1)) ++cnt;
            off[s + 1] = cnt ? cnt : 1;
        }
    });
    for (uint64_t s = 0; s < R; ++s) off[s + 1] += off[s];
    constexpr uint64_t kPad = 64;  // lanes load up to 31 pairs past a task
    out->mask_b64.assign(off[R] + kPad, 0);
    out->word_b64.assign(off[R] + kPad, sentinel64 | kHead);
    parallel_chunks(R, 1 << 14, [&](uint64_t b, uint64_t e, int) {
        for (uint64_t s = b; s < e; ++s) {
            const uint64_t r = row_begin + out->perm[s];
            uint64_t o = off[s];
            if (t.offsets[r + 1] == t.offsets[r]) {  // empty row: a no-op pair on the zero sentinel word
                out->mask_b64[o] = 0;
                out->word_b64[o] = sentinel64 | kHead;
                continue;
            }
            for (uint64_t q = t.offsets[r]; q < t.offsets[r + 1]; ++q) {
                const uint32_t w64 = t.word[q] >> 1;
                const uint64_t m = static_cast<uint64_t>(t.mask[q]) << (32 * (t.word[q] & 1));
                if (q > t.offsets[r] && w64 == (out->word_b64[o - 1] & kWordMask)) {
                    out->mask_b64[o - 1] |= m;
                } else {
                    out->mask_b64[o] = m;
                    out->word_b64[o] = w64 | (q == t.offsets[r] ? kHead : 0u);
                    ++o;
                }
            }
        }
    });
    out->touched64.assign(sentinel64 / 32 + 1, 0u);
    for (const uint32_t wh : out->word_b64) {
        const uint32_t w = wh & kWordMask;
        if (w <= sentinel64) out->touched64[w >> 5] |= 1u << (w & 31);
    }
    const size_t nt = out->task_row_batch.size() - 1;
    out->task_pair_b64.resize(nt + 1);
    for (size_t k = 0; k <= nt; ++k) out->task_pair_b64[k] = off[out->task_row_batch[k]];
}

// The word-major copy (engine.h): per task of <= wm_rows batch rows, its
// 64-cell pairs sorted by (word, row).
void build_wm_layout(const WordCsr& t, uint64_t row_begin, int wm_rows, PackedShard* out) {
    const uint64_t R = out->perm.size();
    const uint64_t rows_per = static_cast<uint64_t>(std::max(1, std::min(wm_rows, 256)));
    out->wm_task_row.clear();
    out->block_task_wm.clear();
    const size_t nb = out->block_row.size() - 1;
    for (size_t c = 0; c < nb; ++c) {
        out->block_task_wm.push_back(static_cast<uint32_t>(out->wm_task_row.size()));
        for (uint64_t r = out->block_row[c]; r < out->block_row[c + 1]; r += rows_per)
            out->wm_task_row.push_back(static_cast<uint32_t>(r));
    }
    const size_t nt = out->wm_task_row.size();
    out->block_task_wm.push_back(static_cast<uint32_t>(nt));
    out->wm_task_row.push_back(static_cast<uint32_t>(R));
    // pass 1: 64-cell pairs per task and distinct words per task
    std::vector<uint64_t> n_ent(nt + 1, 0), n_grp(nt + 1, 0);
    auto task_entries = [&](size_t k, std::vector<uint64_t>* key, std::vector<uint64_t>* msk) {
        key->clear();
        msk->clear();
        const uint64_t r0 = out->wm_task_row[k], r1 = out->wm_task_row[k + 1];
        for (uint64_t s = r0; s < r1; ++s) {
            const uint64_t r = row_begin + out->perm[s];
            for (uint64_t q = t.offsets[r]; q < t.offsets[r + 1]; ++q) {
                const uint64_t w64 = t.word[q] >> 1;
                const uint64_t m = static_cast<uint64_t>(t.mask[q]) << (32 * (t.word[q] & 1));
                if (q > t.offsets[r] && !key->empty() && (key->back() >> 8) == w64 && (key->back() & 255) == s - r0) {
                    msk->back() |= m;  // the other 32-cell half of the same 64-cell word
                } else {
                    key->push_back((w64 << 8) | (s - r0));
                    msk->push_back(m);
                }
            }
        }
    };
    parallel_chunks(nt, 256, [&](uint64_t b, uint64_t e, int) {
        std::vector<uint64_t> key, msk;
        for (uint64_t k = b; k < e; ++k) {
            task_entries(k, &key, &msk);
            std::sort(key.begin(), key.end());
            uint64_t g = 0;
            for (size_t i = 0; i < key.size(); ++i) g += (i == 0 || (key[i] >> 8) != (key[i - 1] >> 8));
            n_ent[k + 1] = key.size();
            n_grp[k + 1] = g;
        }
    });
    for (size_t k = 0; k < nt; ++k) {
        n_ent[k + 1] += n_ent[k];
        n_grp[k + 1] += n_grp[k];
    }
    out->wm_mask.assign(n_ent[nt] + 32, 0);  // (+32: a warp loads whole 32-entry chunks)
    out->wm_row.assign(n_ent[nt] + 32, 0);
    out->wm_gword.assign(n_grp[nt], 0);
    out->wm_gstart.assign(n_grp[nt] + 1, static_cast<uint32_t>(n_ent[nt]));
    out->wm_task_grp.assign(nt + 1, 0);
    for (size_t k = 0; k <= nt; ++k) out->wm_task_grp[k] = static_cast<uint32_t>(n_grp[k]);
    // pass 2: fill, sorted by (word, row)
    parallel_chunks(nt, 256, [&](uint64_t b, uint64_t e, int) {
        std::vector<uint64_t> key, msk;
        std::vector<uint32_t> ord;
        std::vector<std::pair<size_t, size_t>> grp;  // (first in ord, entries)
        for (uint64_t k = b; k < e; ++k) {
            task_entries(k, &key, &msk);
            ord.resize(key.size());
            for (size_t i = 0; i < ord.size(); ++i) ord[i] = static_cast<uint32_t>(i);
            std::sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t c) { return key[a] < key[c]; });
            // the word groups, largest first: the CTA's warps take them in
            // this order, so the task ends on small groups (less waiting at
            // the task's barrier)
            grp.clear();
            for (size_t i = 0; i < ord.size(); ++i)
                if (i == 0 || (key[ord[i]] >> 8) != (key[ord[i - 1]] >> 8)) grp.push_back({i, 0});
            for (size_t g = 0; g < grp.size(); ++g)
                grp[g].second = (g + 1 < grp.size() ? grp[g + 1].first : ord.size()) - grp[g].first;
            std::stable_sort(grp.begin(), grp.end(), [](const auto& a, const auto& c) { return a.second > c.second; });
            uint64_t en = n_ent[k], gn = n_grp[k];
            for (const auto& gr : grp) {
                out->wm_gword[gn] = static_cast<uint32_t>(key[ord[gr.first]] >> 8);
                out->wm_gstart[gn] = static_cast<uint32_t>(en);
                ++gn;
                for (size_t i = gr.first; i < gr.first + gr.second; ++i) {
                    out->wm_mask[en] = msk[ord[i]];
                    out->wm_row[en] = static_cast<uint8_t>(key[ord[i]] & 255);
                    ++en;
                }
            }
        }
    });
}

void build_shard(const WordCsr& t, uint64_t row_begin, uint64_t row_end, bool sort_rows,
                 uint32_t sentinel_word, int stream_task_pairs, int batch_task_pairs, int blocks,
                 PackedShard* out, int wm_rows, bool need_pairs32, bool need_stream64) {
    const uint64_t R = row_end - row_begin;
    out->row_begin = row_begin;
    out->row_end = row_end;
    out->words = t.offsets[row_end] - t.offsets[row_begin];
    out->perm.resize(R);
    const uint64_t nb = static_cast<uint64_t>(std::max(1, blocks));
    out->block_row.resize(nb + 1);
    for (uint64_t c = 0; c <= nb; ++c) out->block_row[c] = R * c / nb;
    if (sort_rows) {
        // z-locality key: the row's median 32-bit word (rows are ascending in
        // z-order, so this is a point inside the swept volume's z-range);
        // rows are sorted within their read-back block only.
        std::vector<uint64_t> key(R);
        parallel_chunks(R, 1 << 16, [&](uint64_t b, uint64_t e, int) {
            for (uint64_t r = b; r < e; ++r) {
                const uint64_t o0 = t.offsets[row_begin + r], o1 = t.offsets[row_begin + r + 1];
                const uint64_t k = o1 > o0 ? t.word[o0 + (o1 - o0 - 1) / 2] : 0;
                key[r] = (k << 32) | r;
            }
        });
        for (uint64_t c = 0; c < nb; ++c)
            std::sort(key.begin() + static_cast<std::ptrdiff_t>(out->block_row[c]),
                      key.begin() + static_cast<std::ptrdiff_t>(out->block_row[c + 1]));
        for (uint64_t s = 0; s < R; ++s) out->perm[s] = static_cast<uint32_t>(key[s] & 0xffffffffu);
    } else {
        for (uint64_t s = 0; s < R; ++s) out->perm[s] = static_cast<uint32_t>(s);
    }
    std::vector<uint64_t> pair_off(R + 1, 0);
    for (uint64_t s = 0; s < R; ++s) {
        const uint64_t r = row_begin + out->perm[s];
        const uint64_t n = t.offsets[r + 1] - t.offsets[r];
        pair_off[s + 1] = pair_off[s] + (n ? n : 1);
    }
    out->n_pairs = pair_off[R];
    // The 32-cell multi-frame copy is read only by the 32-cell kernels: the
    // A/B knobs (LTLG_BATCH64=0, LTLG_PROPLANE=0) and grids too large for the
    // prop-lane / word-major summaries (33..64 props).  Otherwise only its
    // padding is kept (518 MB less HBM and host packing at config 4).
    // padding: no-op head pairs, so the pair after any task is a head (the
    // single-frame kernel closes a task's last row on it)
    if (!need_pairs32) {
        out->pairs.assign(kPairPad, Pair{0, sentinel_word | kHead});
    } else {
    out->pairs.assign(out->n_pairs + kPairPad, Pair{0, sentinel_word | kHead});
    parallel_chunks(R, 1 << 14, [&](uint64_t b, uint64_t e, int) {
        for (uint64_t s = b; s < e; ++s) {
            const uint64_t r = row_begin + out->perm[s];
            const uint64_t o0 = t.offsets[r], o1 = t.offsets[r + 1];
            Pair* dst = out->pairs.data() + pair_off[s];
            if (o1 == o0) {
                dst[0] = Pair{0, sentinel_word | kHead};  // empty row: a no-op pair on the zero sentinel word
                continue;
            }
            for (uint64_t k = o0; k < o1; ++k) dst[k - o0] = Pair{t.mask[k], t.word[k]};
            dst[0].word |= kHead;
        }
    });
    }
    make_tasks(pair_off, out->block_row, batch_task_pairs, &out->task_row_batch, &out->task_pair_batch,
               &out->block_task_batch);
    build_stream_layout(t, row_begin, row_end, sentinel_word, stream_task_pairs, out);
    if (need_stream64) {
        build_stream64_layout(t, row_begin, sentinel_word / 2, out);  // sentinel_word = nw32 = 2 * nw64
    } else {  // (no prop count takes the stream64 kernel on this grid: padding only)
        const size_t nt = out->task_row_stream.size() - 1;
        out->task_n64.assign(nt, 0);
        out->task_byte64.assign(nt + 1, 0);
        out->stream64.assign(kPad64Bytes, 0);
    }
    build_batch64_layout(t, row_begin, sentinel_word / 2, out);
    build_wm_layout(t, row_begin, wm_rows, out);
}

}  // namespace ltlg
