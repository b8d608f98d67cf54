// engine.h -- internal types of the B200 labeling engine (not part of the ABI).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace ltlg {

// Status codes mirror ltlg_status in include/ltlgrid_gpu.h.
enum Status : int { S_OK = 0, S_EINVAL = 1, S_EFORMAT = 2, S_EIO = 3, S_ECUDA = 4, S_ENCCL = 5, S_ENOMEM = 6, S_ESTATE = 7 };

struct Error {
    Status code;
    std::string msg;
};

// One T pair as stored in HBM: 8 bytes, AoS so a 16-byte load yields two.
//   mask : bit b = cell 32*word + b of the row's swept volume
//   word : bits 0..30 word index (z-order), bit 31 = first pair of its row
struct Pair {
    uint32_t mask;
    uint32_t word;
};
constexpr uint32_t kHead = 0x80000000u;
constexpr uint32_t kWordMask = 0x7fffffffu;

// Word-CSR of the whole abstraction in ORIGINAL row order (host).
struct WordCsr {
    uint64_t rows = 0, cols = 0, nnz = 0;
    std::vector<uint64_t> offsets;  // rows + 1
    std::vector<uint32_t> word;     // W32
    std::vector<uint32_t> mask;     // W32
};

// The device image of one shard (host staging copy).
struct PackedShard {
    uint64_t row_begin = 0, row_end = 0;  // original rows [row_begin, row_end)
    uint64_t words = 0;                   // W32 of the shard
    std::vector<Pair> pairs;              // sorted-row order, padded (see kPairPad)
    std::vector<Pair> pairs_stream;       // the same pairs in the single-frame layout (see kStreamK)
    // single-frame 64-cell-word copy (see kStreamK): per stream task, its bytes
    // start at task_byte64[t] and hold task_n64[t] (mask64, word64) pairs
    std::vector<uint8_t> stream64;
    std::vector<uint64_t> task_byte64;    // ntasks + 1
    std::vector<uint32_t> task_n64;       // ntasks
    // multi-frame 64-cell-word copy: SoA arrays in the batch layout's row
    // order; task t's pairs are [task_pair_b64[t], task_pair_b64[t+1])
    std::vector<uint64_t> mask_b64;
    std::vector<uint32_t> word_b64;
    std::vector<uint64_t> task_pair_b64;  // ntasks + 1
    // bit w: some pair of the multi-frame copy is on 64-cell word w (the
    // sentinel word included); the prop-lane summary skips the other words
    std::vector<uint32_t> touched64;
    // word-major multi-frame copy (the prop-lane path's default kernel,
    // label_wm_kernel): CTA tasks of <= wm_rows consecutive rows of the batch row
    // order (never crossing a read-back block); a task's 64-cell pairs are
    // grouped by word, so the word's per-frame summary and partial records
    // are read once per task and tested against every pair on it.
    //   task t: rows [wm_task_row[t], wm_task_row[t+1]) (batch positions),
    //           groups [wm_task_grp[t], wm_task_grp[t+1])
    //   group g: word wm_gword[g], entries [wm_gstart[g], wm_gstart[g+1])
    //   entry e: mask wm_mask[e] (64 cells), row wm_row[e] - task's first row
    std::vector<uint64_t> wm_mask;
    std::vector<uint8_t> wm_row;
    std::vector<uint32_t> wm_gword, wm_gstart;         // ngroups (+1 for gstart)
    std::vector<uint32_t> wm_task_row, wm_task_grp;    // ntasks + 1
    std::vector<uint32_t> block_task_wm;               // per read-back block (+1)
    uint64_t n_pairs = 0;                 // meaningful pairs (incl. sentinels)
    std::vector<uint32_t> perm;           // sorted position -> local original row
    // warp tasks: [row_begin, row_end) in sorted positions, pairs [pair_begin, pair_end)
    std::vector<uint32_t> task_row_stream, task_row_batch;    // ntasks + 1
    std::vector<uint64_t> task_pair_stream, task_pair_batch;  // ntasks + 1
    // read-back blocks: rows [block_row[c], block_row[c+1]) (local, original
    // order) are z-sorted only among themselves, so the tasks
    // [block_task_*[c], block_task_*[c+1]) write exactly that row range
    std::vector<uint64_t> block_row;
    std::vector<uint32_t> block_task_stream, block_task_batch;
};

constexpr uint64_t kPairPad = 512;  // tail padding so vector loads never leave the array
constexpr int kWmRows = 128;  // rows per word-major CTA task (label_wm_kernel: 256 B of shared memory per row and 32 props)

// Single-frame layout.  The stream kernel gives each lane kStreamK consecutive
// pairs of a warp chunk of 32*kStreamK pairs and reads them as 16-byte pieces.
// So that those reads are coalesced (one 512-byte run per warp instruction
// instead of 32 pieces at a 64-byte lane stride), every FULL chunk of a stream
// task is stored piece-transposed: the piece holding pairs (K*l + 2h,
// K*l + 2h + 1) of the chunk sits at piece h*32 + l.  A task's last, partial
// chunk stays in plain order.  Tasks start on 16-byte boundaries (a task with
// an odd pair count gets one no-op pair appended).
constexpr int kStreamK = 8;
constexpr uint64_t kStreamCH = 32 * kStreamK;
// The 64-cell-word single-frame copy uses the same chunking with 12-byte
// pairs stored SoA per chunk: a full chunk is 2 KB of u64 masks (piece h*32+l
// = masks of pairs K*l+2h, K*l+2h+1) then 1 KB of u32 word fields (piece
// h*32+l = words of pairs K*l+4h .. K*l+4h+3); a partial last chunk of n
// pairs is n masks then n words, each region padded to 16 bytes.
constexpr uint64_t kChunk64Bytes = kStreamCH * 12;
constexpr uint64_t kPad64Bytes = 4096;  // tail padding: lane-contiguous loads of a partial chunk stay inside

// Host-side loader (loader.cpp).
bool validate_csr(uint64_t rows, uint64_t cols, const uint64_t* offsets, uint64_t n_offsets,
                  const uint32_t* indices, uint64_t nnz, Error* err);
bool pack_csr(uint64_t rows, uint64_t cols, const uint64_t* offsets, const uint32_t* indices,
              WordCsr* out, Error* err);
bool take_words(uint64_t rows, uint64_t cols, const uint64_t* offsets, const uint32_t* word,
                const uint32_t* mask, WordCsr* out, Error* err);
bool read_csb1(const char* path, uint64_t* rows, uint64_t* cols, std::vector<uint64_t>* offsets,
               std::vector<uint32_t>* indices, Error* err);
// CsrBoolMatrix::load + validate + pack, streaming: the u32 index array is
// never held whole (peak host memory = offsets + one chunk + the word-CSR).
bool read_csb1_words(const char* path, WordCsr* out, Error* err);
// load_bitset (grid.cpp:375-405) of one proposition column into dst
// (ceil(cells/64) u64); the file's cell count must equal `cells`.
bool read_zobv(const char* path, uint64_t cells, uint64_t* dst, Error* err);
// LabelMatrix::save (label.cpp:300-309): LBM1 of rows x ceil(props/64) words.
bool write_lbm1(const char* path, uint64_t rows, int props, const uint64_t* words, Error* err);
// CsrBoolMatrix::save (label.cpp:251-268): CSB1 of rows x cols.
bool write_csb1(const char* path, uint64_t rows, uint64_t cols, const uint64_t* offsets, const uint32_t* indices,
                Error* err);
// Split rows into n contiguous shards balanced by stored pairs.
std::vector<uint64_t> shard_bounds(const WordCsr& t, int n);
void build_shard(const WordCsr& t, uint64_t row_begin, uint64_t row_end, bool sort_rows,
                 uint32_t sentinel_word, int stream_task_pairs, int batch_task_pairs, int blocks,
                 PackedShard* out, int wm_rows = kWmRows, bool need_pairs32 = true, bool need_stream64 = true);
int host_threads();

}  // namespace ltlg
