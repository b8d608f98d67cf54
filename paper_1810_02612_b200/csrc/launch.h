// launch.h -- host launchers of the sm_100a kernels (kernels.cu), used by api.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "engine.h"

namespace ltlg {

constexpr uint32_t kCtrStride = 256;  // task counters per launch (one per SM slice)

struct LaunchArgs {
    const Pair* pairs;
    const uint64_t* task_pair;
    const uint32_t* task_row;
    uint32_t task_begin;  // tasks [task_begin, ntasks) of this launch
    uint32_t ntasks;
    const void* sf;
    const uint32_t* P32;
    uint32_t nw32;
    int props;
    int frames;
    const uint32_t* perm;
    void* out;
    int label_bytes;
    uint32_t ostride;  // single-frame kernels: label of row r at out[r * ostride] (0 = 1)
    uint32_t* task_ctr;  // this launch's kCtrStride device counters, reset by the summary kernel
    const void* s_only;  // S mask per (word, frame): over-path probes, full-mask pairs
    // 64-cell-word single-frame copy (null: use the 32-bit stream copy)
    const uint8_t* t64;
    const uint64_t* task_byte64;
    const uint32_t* task_n64;
    uint32_t nw64;
    // 64-cell-word multi-frame copy (null: use the 32-bit pairs)
    const uint64_t* mask_b64;
    const uint32_t* word_b64;
    const uint64_t* task_pair_b64;
    const uint64_t* pb64;  // Pb table of summary_b64_kernel
    int prop_lane;         // multi-frame: the prop-lane kernel (sf = its launch_pl work buffer)
    int pdl;               // single frame: launch as a programmatic dependent of the summary kernel
    // word-major multi-frame copy (PackedShard::wm_*): label_wm_kernel
    int word_major;
    int tc;  // (word_major, multi-frame) the tcgen05 kind::i8 kernel (tc_i8.cu)
    const uint64_t* wm_mask;
    const uint8_t* wm_row;
    const uint32_t* wm_gword;
    const uint32_t* wm_gstart;
    const uint32_t* wm_task_row;
    const uint32_t* wm_task_grp;
    int wm_rows;
};

cudaError_t launch_summary(const uint32_t* P32, int props, int frames, uint32_t nw32, uint64_t cells,
                           void* tab, void* s_only, uint32_t* task_ctr, int nctr, cudaStream_t st);
int entry_format(int props);
size_t summary_entry_bytes(int props);
size_t s_only_bytes(int props);
size_t split_table_bytes(int props, uint32_t nw32);
size_t split64_table_bytes(int props, uint32_t nw64);
cudaError_t launch_summary_b64(const uint64_t* P64, int props, int frames, uint32_t nw64, uint64_t cells, void* tab,
                               uint64_t* pbt, void* s_only, uint32_t* task_ctr, int nctr, cudaStream_t st);
cudaError_t launch_pl(const uint64_t* P64, int props, int frames, uint32_t nw64, uint64_t cells, void* work,
                      size_t work_bytes, uint32_t* task_ctr, int nctr, cudaStream_t st,
                      const uint32_t* touched64 = nullptr);
size_t pl_work_bytes(int props, int frames, uint32_t nw64);
// the word-major kernel's summary (label_wm_kernel): frame-major masks + lane records
cudaError_t launch_wm_build(const uint64_t* P64, int props, int frames, uint32_t nw64, uint64_t cells, void* work,
                            size_t work_bytes, uint32_t* task_ctr, int nctr, cudaStream_t st,
                            const uint32_t* touched64 = nullptr);
size_t wm_work_bytes(int props, uint32_t nw64);
// the tcgen05 kind::i8 formulation (tc_i8.cu, dev knob LTLG_TC=1)
size_t tc_work_bytes(uint32_t nw64);
cudaError_t launch_tc_build(const uint64_t* P64, int props, int frames, uint32_t nw64, uint64_t cells, void* work,
                            uint32_t* task_ctr, int nctr, cudaStream_t st, const uint32_t* touched64);
cudaError_t launch_tc_label(const LaunchArgs& a, cudaStream_t st);
cudaError_t launch_summary64(const uint64_t* P64, int props, uint32_t nw64, uint64_t cells, void* tab, void* s_only,
                             uint32_t* task_ctr, int nctr, cudaStream_t st, uint64_t* P_copy,
                             const uint32_t* touched64 = nullptr);
bool stream_table_in_smem(int props, uint32_t nw32);
// where label_stream64_kernel keeps its split table: 1 = all in shared
// memory, 2 = M in shared memory / X through L1, 0 = all through L1
int stream64_table_loc(int props, uint32_t nw64);
cudaError_t launch_label(const LaunchArgs& a, cudaStream_t st);
cudaError_t launch_extract(const void* labels, int label_bytes, uint64_t rows, int frames, int frame,
                           uint64_t* out, cudaStream_t st);
cudaError_t launch_edge_count(const uint64_t* masks, const uint32_t* words, const uint64_t* task_pair,
                              const uint32_t* task_row, uint32_t ntasks, const uint32_t* perm, const uint64_t* col,
                              uint8_t* hit, uint64_t* examined, cudaStream_t st);
cudaError_t launch_guards(const void* labels, int label_bytes, uint64_t n, const uint64_t* lut, uint64_t always,
                          uint64_t all_guards, uint64_t* admitted, cudaStream_t st);
cudaError_t launch_lane(int depth, const uint64_t* flags, int ncols, int col0, int col_step, uint64_t* out,
                        cudaStream_t st);
cudaError_t launch_rasterize(int k, int depth, int cols_total, const uint64_t* box_off, const int64_t* ranges,
                             uint64_t* out, cudaStream_t st);
cudaError_t launch_resample(int vdepth, double vlo0, double vhi0, double vlo1, double vhi1, int wdepth,
                            double wlo0, double whi0, double wlo1, double whi1, const void* poses,
                            int frames, int props, const uint32_t* world32, uint32_t wnw32, int outside,
                            uint32_t vnw32, uint32_t* out32, cudaStream_t st);

// swept-volume matrix (sweep.cu): 3-axis grid of depth <= 32, so every
// z-order cell index fits in 32 bits
constexpr int kSweepThreads = 128;
constexpr uint32_t kSweepTable = 2048;             // shared-memory set slots per CTA
constexpr uint32_t kSweepCap = kSweepTable / 2;    // distinct cells per row before overflow
struct SweepParams {
    double lo[3], hi[3];
    double cells[3];  // cells per axis, as double (GridSpec::axis_cells)
    double w[3];      // GridSpec::cell_width
    int64_t ncell[3];
    int zoff[3];      // ZScatter shift per axis
    double length, width, ref_offset;  // FootprintSpec
    uint64_t edges;
    const uint64_t* sample_off;  // edges + 1
    const double* samples;       // 5 doubles per State5
    unsigned long long* err_key; // [0] min(sample * 4 + kind), [1] global-table overflows
};
struct SweepBufs {
    uint32_t* edge_ctr;
    uint32_t* row_cnt;
    const uint64_t* row_off;
    uint32_t* cols;
    uint32_t* over_list;
    uint32_t* n_over;
    unsigned long long* gtab;
    uint32_t* gkeys;
    uint32_t* stage;           // staged rows (MODE 2)
    uint64_t stage_cap;
    unsigned long long* bump;  // staging allocator
    uint64_t* stage_off;       // per edge
};
size_t sweep_smem_bytes();
cudaError_t launch_sweep(int mode, bool global, const SweepParams& p, const SweepBufs& b, uint32_t glog2,
                         int gblocks, cudaStream_t st);
cudaError_t launch_sweep_gather(uint64_t edges, const SweepBufs& b, cudaStream_t st);
cudaError_t launch_scan_counts(const uint32_t* cnt, uint64_t n, uint64_t* bsum, uint64_t* off, cudaStream_t st);

}  // namespace ltlg
