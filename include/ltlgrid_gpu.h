/*
 * ltlgrid_gpu.h -- C ABI of the B200 edge-labeling engine (libltlgrid_gpu.so).
 *
 * Drop-in for the reference labeling path L = T o P over the OR-AND semiring:
 *   ltlgrid::label_all(const CsrBoolMatrix&, const DensePropMatrix&, int)
 *   (reference: proj/core/include/ltlgrid/label.hpp:94-98, label.cpp:150-189)
 * split into the reference's own life cycle "load abstraction -> submit grid
 * -> get per-edge label bitsets".  Plain pointers and sizes only; no CUDA or
 * torch types cross this boundary.  All host buffers are owned by the caller
 * and never retained after a call returns (inputs are copied to the device,
 * label reads are synchronous).  A context is used by one host thread at a
 * time; distinct contexts are independent (reference: label_all is reentrant,
 * SPEC.md:424).
 *
 * Bit layouts are the reference's, verbatim:
 *   T  CSR, row i's set cells col_indices[row_offsets[i] .. row_offsets[i+1]),
 *      strictly ascending, each < cols            (label.hpp:18-35)
 *   P  props columns of ceil(cells/64) u64 words, little-endian, bit c of the
 *      column = cell c in z-order                 (label.hpp:47-58, grid.hpp:93-125)
 *   L  LabelMatrix: rows x ceil(props/64) u64 words, bit j of edge i = prop j
 *                                                 (label.hpp:61-92)
 *
 * Errors: every entry point returns an ltlg_status; the message of the last
 * failure is ltlg_last_error(ctx) (ltlg_last_error(NULL) for ltlg_create and
 * the one-shot ltlg_label_all).  LTLG_EINVAL messages are the reference's
 * std::invalid_argument texts (label.cpp:16-40, 124-132, 151-154), LTLG_EFORMAT /
 * LTLG_EIO the std::runtime_error texts of the file loaders (label.cpp:271-298).
 */
#ifndef LTLGRID_GPU_H
#define LTLGRID_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LTLG_ABI_VERSION 1

typedef enum ltlg_status {
    LTLG_OK = 0,
    LTLG_EINVAL = 1,  /* reference std::invalid_argument                 */
    LTLG_EFORMAT = 2, /* reference std::runtime_error (bad file content) */
    LTLG_EIO = 3,     /* reference std::runtime_error (open/read/write)  */
    LTLG_ECUDA = 4,   /* CUDA runtime error (no device, launch failure)  */
    LTLG_ENCCL = 5,   /* NCCL error (multi-device contexts)              */
    LTLG_ENOMEM = 6,  /* device or host allocation failed                */
    LTLG_ESTATE = 7,  /* call out of order (e.g. submit before load)     */
    LTLG_EDOMAIN = 8  /* reference std::domain_error                     */
} ltlg_status;

typedef struct ltlg_ctx ltlg_ctx;

/* Engine options (ltlg_create_ex).  Zero-initialise and set what you need. */
typedef struct ltlg_options {
    int sort_rows;        /* 1 (default via ltlg_create): store T rows in z-locality order, undo on output */
    int stream_task_pairs;/* target T pairs per warp task, single-frame kernel (0 = default 2048) */
    int batch_task_pairs; /* target T pairs per warp task, multi-frame kernel (0 = default 256)   */
    int profile;          /* 1: record CUDA events around each stage (ltlg_stage_times) */
    int readback_chunks;  /* >1: split each shard's rows into this many blocks (<= 64); multi-frame
                             submits of host-memory P label them with separate launches, so
                             ltlg_get_labels_packed copies block c to the host while later blocks
                             are still being labelled (0/1 = off) */
    int task_rows;        /* rows per CTA task of the word-major multi-frame kernel (0 = default 128,
                             at most 256); its shared memory per CTA grows with it */
    int reserved[5];
} ltlg_options;

/* Shape / layout facts about the loaded abstraction and the last submit. */
typedef struct ltlg_info {
    uint64_t rows;         /* edges E                                    */
    uint64_t cols;         /* cells of T's column space                  */
    uint64_t nnz;          /* stored cells of T                          */
    uint64_t words;        /* W32: distinct (row, 32-bit word) pairs     */
    uint64_t pairs;        /* stored T pairs incl. empty-row sentinels   */
    uint64_t t_bytes;      /* device bytes of the packed T (all shards)  */
    int n_devices;
    int props;             /* props of the last submit                   */
    int frames;            /* frames of the last submit                  */
    int label_bytes;       /* bytes per packed label word: 1, 2, 4 or 8  */
    int label_words;       /* LabelMatrix words per row, ceil(props/64)  */
    int reserved[7];
} ltlg_info;

/* Create an engine on the given CUDA devices (n >= 1; NULL = device 0).
 * T rows are sharded across the devices; each frame's P is uploaded to the
 * first device and broadcast to the others (NCCL when n > 1). */
ltlg_status ltlg_create(const int* devices, int n_devices, ltlg_ctx** out);
ltlg_status ltlg_create_ex(const int* devices, int n_devices, const ltlg_options* opts,
                           ltlg_ctx** out);
void ltlg_destroy(ltlg_ctx* ctx);
const char* ltlg_last_error(const ltlg_ctx* ctx);
int ltlg_abi_version(void);

/* Load T from a CSR (replaces CsrBoolMatrix + validate, label.hpp:18-35,
 * label.cpp:16-40).  Validated with the reference's rules and messages, then
 * bit-packed once into the device word-CSR; the host arrays are not retained. */
ltlg_status ltlg_load_abstraction(ltlg_ctx* ctx, uint64_t rows, uint64_t cols,
                                  const uint64_t* row_offsets, const uint32_t* col_indices);

/* Load T from a CSB1 file (replaces CsrBoolMatrix::load, label.cpp:271-298):
 * same header checks and messages, then validate, then pack -- streamed, so
 * the u32 index array (4 B per swept cell) is never held in host memory. */
ltlg_status ltlg_load_abstraction_file(ltlg_ctx* ctx, const char* csb1_path);

/* Load T already packed as a word-CSR: row i's 32-bit words are
 * word_index[row_word_offsets[i] .. row_word_offsets[i+1]) (strictly
 * ascending, < ceil(cols/32)) with non-zero word_mask (bit b = cell
 * 32*word + b, every such cell < cols).  Same semantics as the CSR form. */
ltlg_status ltlg_load_abstraction_words(ltlg_ctx* ctx, uint64_t rows, uint64_t cols,
                                        const uint64_t* row_word_offsets,
                                        const uint32_t* word_index, const uint32_t* word_mask);

/* Submit `frames` perception grids and label every edge for each of them
 * (replaces DensePropMatrix + label_all, label.hpp:47-58 / 94-98).
 * column_words: frames x num_props x ceil(cells/64) u64, i.e. `frames`
 * DensePropMatrix column sets back to back.  Requires cells == cols of T
 * (else LTLG_EINVAL "dimension mismatch: ..."), 0 <= num_props <= 64.
 * Asynchronous: returns after enqueueing the upload and the kernels.  A
 * pageable column_words may be reused at once; a pinned (page-locked) one
 * must stay unmodified until ltlg_wait, as with cudaMemcpyAsync (one frame
 * on one device reads it in place through the host mapping). */
ltlg_status ltlg_submit_grid(ltlg_ctx* ctx, uint64_t cells, int num_props,
                             const uint64_t* column_words, int frames);

/* Same, but column_words already lives on the context's first device
 * (e.g. written by a perception kernel, or received by an NCCL broadcast).
 * A single-device engine reads it in place: keep it alive and unmodified
 * until ltlg_wait / ltlg_get_labels* returns. */
ltlg_status ltlg_submit_grid_device(ltlg_ctx* ctx, uint64_t cells, int num_props,
                                    const uint64_t* device_column_words, int frames);

/* Same as ltlg_submit_grid_device; readback != 0 declares that the labels
 * will be copied to the host (ltlg_get_labels_packed), so a multi-frame
 * submit is labelled block by block (ltlg_options.readback_chunks) and the
 * copy of block c overlaps the labelling of later blocks -- what
 * ltlg_submit_grid does for host P. */
ltlg_status ltlg_submit_grid_device_ex(ltlg_ctx* ctx, uint64_t cells, int num_props,
                                       const uint64_t* device_column_words, int frames, int readback);

/* Same as ltlg_submit_grid_device_ex, for a pipelining caller: P (on the
 * first device) is ready when `ready_event` (a cudaEvent_t, as void*,
 * recorded by the caller) completes -- the engine orders its reads of P after
 * that event only, not after the engine's own earlier work.  The multi-frame
 * summary then runs on the shard's comm stream and overlaps the previous
 * submit's labelling; the labelling still follows the previous one.  P must
 * stay unmodified until the labels are ready, as for the device form. */
ltlg_status ltlg_submit_grid_device_async(ltlg_ctx* ctx, uint64_t cells, int num_props,
                                          const uint64_t* device_column_words, int frames, int readback,
                                          void* ready_event);

/* World-frame perception grid -> vehicle-frame P resample, then label
 * (north_star subsystem 2; transform convention of translate_system,
 * abstraction.cpp:396-404).  Grids are k=2 z-order grids; world_words is
 * num_props x ceil(2^world_depth/64) u64 (device or host, see flag).
 * Cells whose centre maps outside the world take `outside` (0 or 1). */
typedef struct ltlg_grid2 {
    int depth;
    double lo0, hi0, lo1, hi1;
} ltlg_grid2;
typedef struct ltlg_pose2 {
    double dx, dy, cos_t, sin_t;
} ltlg_pose2;
ltlg_status ltlg_submit_world_grid(ltlg_ctx* ctx, const ltlg_grid2* vehicle, const ltlg_grid2* world,
                                   int num_props, const uint64_t* world_words, int words_on_device,
                                   const ltlg_pose2* poses, int frames, int outside);

/* Submit `frames` x num_props ZOBV proposition columns (load_bitset,
 * grid.cpp:375-405; paths[f * num_props + j] = prop j of frame f), read
 * straight into pinned staging memory and labelled like ltlg_submit_grid.
 * Every column must be cols-of-T bits long (DensePropMatrix, label.cpp:125-127:
 * "column length mismatch").  File errors: "cannot open: <path>" (EIO),
 * "not a bitset file: <path>", "corrupt bitset header",
 * "truncated bitset file: <path>" (EFORMAT).  Returns when the labels are ready. */
ltlg_status ltlg_submit_grid_files(ltlg_ctx* ctx, const char* const* paths, int num_props, int frames);

/* Write one frame's labels as an LBM1 file (LabelMatrix::save, label.cpp:300-309). */
ltlg_status ltlg_save_labels(ltlg_ctx* ctx, int frame, const char* path);

/* Host-only: stream-read, validate and pack a CSB1 file exactly as
 * ltlg_load_abstraction_file does (CsrBoolMatrix::load + validate, label.cpp:
 * 271-298 / 16-40: same checks, same order, same messages), reporting its
 * shape.  The index array is never held whole.  No device needed. */
ltlg_status ltlg_read_csb1_words(const char* path, uint64_t* rows, uint64_t* cols, uint64_t* nnz, uint64_t* words);

/* Host-only: one ZOBV proposition column of `cells` bits into words_out
 * (ceil(cells/64) u64), with the ltlg_submit_grid_files checks. */
ltlg_status ltlg_read_zobv(const char* path, uint64_t cells, uint64_t* words_out);

/* k-D z-order grid (GridSpec, grid.hpp:22-57): axis a gets depth/k bits,
 * the first depth%k axes one extra; bounds lo[a] < hi[a].  dims <= 4. */
typedef struct ltlg_gridk {
    int dims;
    int depth;
    double lo[4], hi[4];
} ltlg_gridk;

/* Rasterize axis-aligned boxes into z-ordered proposition columns on the GPU
 * (rasterize_box, grid.cpp:260-344, one column = the union of its boxes):
 * column c (of num_cols) is the union of boxes [box_offsets[c],
 * box_offsets[c+1]); box b spans [box_lo[b*dims + a], box_hi[b*dims + a]] on
 * axis a, cell ranges by overlap_cells (grid.cpp:49-61).  out_words =
 * num_cols x ceil(2^depth/64) u64 (host).  Runs on `device`, synchronous.
 * Errors: the GridSpec messages ("grid needs at least one axis", "grid depth
 * must be in [k, 63]", "grid bounds must satisfy lo < hi"). */
ltlg_status ltlg_rasterize_boxes(const ltlg_gridk* grid, int num_cols, const uint64_t* box_offsets,
                                 const double* box_lo, const double* box_hi, int device, uint64_t* out_words);

/* The same rasterization straight into the context's P (frames x num_props
 * columns, column f*num_props + j), then labelling -- the frame's proposition
 * volumes never touch host bitsets.  2^depth must equal cols
 * of T.  Asynchronous like ltlg_submit_grid_device. */
ltlg_status ltlg_submit_boxes(ltlg_ctx* ctx, const ltlg_gridk* grid, int num_props, int frames,
                              const uint64_t* box_offsets, const double* box_lo, const double* box_hi);

/* The reference benchmark's perception volumes on the GPU:
 * generate_scenario (core/src/scenario.cpp:52-128, ScenarioConfig
 * scenario.hpp:18-31) on a 3-axis (x, y, tau) grid.  Column 0 =
 * moving_vehicle: the agents' anticipated swept boxes (SplitMix64 seeded by
 * mix_seed(seed, query_index), rasterize_box per agent per time slab);
 * column 1 = not_nominal_lane: every cell outside the circular lane tube.
 * The per-agent geometry and the per-(x, y) lane test run on the host with
 * the reference's own arithmetic (libm cos / sin / hypot); the cells are
 * written on the GPU.  Errors: the GridSpec messages; LTLG_EINVAL "scenario
 * needs a 3-d (x, y, tau) grid", "horizon exceeds the grid's tau extent";
 * LTLG_EDOMAIN "agent radius collapsed to the loop centre", "agent outside
 * workspace". */
typedef struct ltlg_scenario {
    double loop_cx, loop_cy, loop_radius, lane_width;
    int agent_count;
    double agent_speed_min, agent_speed_max, agent_length, agent_width, lateral_spread, horizon;
    uint64_t seed;
} ltlg_scenario;

/* out_words = 2 x ceil(2^depth/64) u64 (host): moving_vehicle, not_nominal_lane. */
ltlg_status ltlg_generate_scenario(const ltlg_scenario* cfg, const ltlg_gridk* grid, uint64_t query_index,
                                   int device, uint64_t* out_words);

/* `frames` scenario queries (query_index0 + f) straight into the context's P
 * (frames x 2 props: moving_vehicle = prop 0, not_nominal_lane = prop 1),
 * then labelling; 2^depth must equal cols of T.  Asynchronous. */
ltlg_status ltlg_submit_scenario(ltlg_ctx* ctx, const ltlg_scenario* cfg, const ltlg_gridk* grid,
                                 uint64_t query_index0, int frames);

/* Resident-label consumer: monitor transition guards
 * (TransitionGuard {positive, negative}, buchi.hpp:16-26; admits(s) =
 * (s & positive) == positive && (s & negative) == 0).  After every later
 * submit the engine also computes, per (edge, frame), the u64 mask of
 * admitted guards (bit t = guard t admits the edge's label) -- the edge test
 * of build_product (planner.cpp:53-64; AND it with the live-target mask).
 * n_guards in [0, 64]; 0 turns the consumer off. */
ltlg_status ltlg_set_guards(ltlg_ctx* ctx, int n_guards, const uint64_t* positive, const uint64_t* negative);

/* Copy one frame's admitted-guard masks (rows u64).  Synchronous. */
ltlg_status ltlg_get_admitted(ltlg_ctx* ctx, int frame, uint64_t* out);

/* Resident admitted-guard masks of shard s (rows x frames u64, edge-major). */
ltlg_status ltlg_device_admitted(ltlg_ctx* ctx, int shard, void** dev_ptr);

/* Block until every submitted frame is labelled. */
ltlg_status ltlg_wait(ltlg_ctx* ctx);

/* Copy one frame's labels in the reference LabelMatrix word layout
 * (rows x ceil(props/64) u64).  Synchronous. */
ltlg_status ltlg_get_labels(ltlg_ctx* ctx, int frame, uint64_t* out);

/* apply_labels (reference label.cpp:191-210, label.hpp:107-114): the labels of
 * one frame as per-edge AlphabetSymbol bits (alphabet.hpp:39-46) -- the
 * EdgeLabeling hand-off a planner / monitor consumes (planner.cpp:56).
 * num_edges is the TransitionSystem's num_edges(), alphabet_size the
 * Alphabet's size(); the reference's two checks run in its order with its
 * messages ("label matrix rows R vs edges E", "label matrix props P vs
 * alphabet size A"; LTLG_EINVAL).  symbols = num_edges u64 (zeros when
 * props == 0).  Synchronous. */
ltlg_status ltlg_apply_labels(ltlg_ctx* ctx, int frame, uint64_t num_edges, int alphabet_size,
                              uint64_t* symbols);

/* label_edge_counting (reference label.cpp:140-148, the Eq. 14 diagnostic of
 * bernoulli_experiment, scenario.cpp:232-255) for EVERY resident edge against
 * one (frame, prop) column of the last submit, on the device: hit[i] = label
 * bit, examined[i] = number of the row's stored indices a linear scan
 * examines (first witness position + 1, or the row's nnz).  hit: rows bytes,
 * examined: rows u64 (either may be NULL).  Synchronous. */
ltlg_status ltlg_edge_counting(ltlg_ctx* ctx, int frame, int prop, uint8_t* hit, uint64_t* examined);

/* Copy all frames' packed labels: edge-major rows x frames words of
 * ltlg_info.label_bytes each (bit j = prop j).  out_bytes must be >=
 * rows * frames * label_bytes.  Synchronous. */
ltlg_status ltlg_get_labels_packed(ltlg_ctx* ctx, void* out, size_t out_bytes);

/* Resident labels for downstream consumers: device pointer of shard s
 * (rows [row_begin, row_end) x frames packed words) -- stays valid until the
 * next submit / load / destroy. */
ltlg_status ltlg_device_labels(ltlg_ctx* ctx, int shard, void** dev_ptr, uint64_t* row_begin,
                               uint64_t* row_end, int* device);

ltlg_status ltlg_get_info(ltlg_ctx* ctx, ltlg_info* out);

/* The CUDA stream (as void*) the engine enqueues shard s's work on, so that
 * callers can time with events on the launching stream. */
ltlg_status ltlg_stream(ltlg_ctx* ctx, int shard, void** stream);

/* Turn the per-submit stage events (ltlg_stage_times) on or off.  Off, a
 * single-frame submit launches its labeling kernel as a programmatic
 * dependent of the summary kernel (no event between them). */
ltlg_status ltlg_set_profiling(ltlg_ctx* ctx, int on);

/* With ltlg_options.profile = 1: device time (CUDA events on the launching
 * stream) of the stages of the submit `back` submits ago (0 = the last one,
 * up to 255) on shard s -- P upload / broadcast, per-word summary build,
 * labeling kernel.  Waits for that submit only. */
ltlg_status ltlg_stage_times(ltlg_ctx* ctx, int shard, int back, float* upload_ms, float* summary_ms,
                             float* label_ms);

/* Host-only CsrBoolMatrix::validate (label.cpp:16-40): same checks, same
 * order, same messages (written to err, NUL-terminated).  No device needed. */
ltlg_status ltlg_validate_csr(uint64_t rows, uint64_t cols, const uint64_t* row_offsets,
                              uint64_t n_offsets, const uint32_t* col_indices, uint64_t nnz,
                              char* err, size_t err_len);

/* One-shot drop-in for ltlgrid::label_all (label.cpp:150-189) on device 0:
 * out = rows x ceil(num_props/64) u64 LabelMatrix words.  `workers` is
 * accepted for signature parity and ignored (the GPU partition is internal;
 * results are identical for any value, as test_label.cpp:121-132 requires). */
ltlg_status ltlg_label_all(uint64_t rows, uint64_t cols, const uint64_t* row_offsets,
                           const uint32_t* col_indices, uint64_t cells, int num_props,
                           const uint64_t* column_words, int workers, uint64_t* out);

/* ------------------------------------------------------------------------
 * Swept-volume matrix on the GPU: the abstraction T itself.
 * Replaces swept_volume_matrix (core/include/ltlgrid/label.hpp:42-43,
 * core/src/label.cpp:75-116) = sweep_voxelize_indices per edge
 * (abstraction.hpp:88-93, abstraction.cpp:172-221).
 *
 * grid: a 3-axis (x, y, tau) GridSpec, depth <= 32.  footprint: FootprintSpec
 * (abstraction.hpp:58-62).  Edge e's trajectory is samples
 * [sample_offsets[e], sample_offsets[e+1]), 5 doubles per sample in State5
 * order (px, py, heading, speed, tau; abstraction.hpp:16-22).  Synchronous on
 * `device`; the CSR stays resident there until copied out or loaded.
 * Errors, in the reference's order: the GridSpec messages; LTLG_EINVAL
 * "swept_volume_matrix supports depth <= 32"; LTLG_EINVAL "sweep_voxelize
 * requires a 3-d (x, y, tau) grid" (when there are edges); per sample in
 * (edge, sample) order: LTLG_EDOMAIN "trajectory exits workspace (time
 * axis)", LTLG_EINVAL "footprint must be positive", LTLG_EDOMAIN
 * "trajectory exits workspace (position)".
 * ---------------------------------------------------------------------- */
typedef struct ltlg_footprint {
    double length, width, ref_offset;
} ltlg_footprint;

typedef struct ltlg_csr ltlg_csr;

ltlg_status ltlg_swept_volume(const ltlg_gridk* grid, const ltlg_footprint* footprint, uint64_t num_edges,
                              const uint64_t* sample_offsets, const double* samples, int device, ltlg_csr** out);
uint64_t ltlg_csr_rows(const ltlg_csr* m);
uint64_t ltlg_csr_cols(const ltlg_csr* m);
uint64_t ltlg_csr_nnz(const ltlg_csr* m);
/* Kernel time of the last ltlg_swept_volume in ms (both passes, CUDA events). */
double ltlg_csr_build_ms(const ltlg_csr* m);
/* Host copies: row_offsets (rows + 1 u64), col_indices (nnz u32); either may be NULL. */
ltlg_status ltlg_csr_copy(const ltlg_csr* m, uint64_t* row_offsets, uint32_t* col_indices);
/* CsrBoolMatrix::save (label.cpp:251-268): the matrix as a CSB1 file,
 * byte-identical to the reference's.  LTLG_EIO "cannot open for writing:
 * <path>" / "write failed: <path>". */
ltlg_status ltlg_csr_save(const ltlg_csr* m, const char* path);
/* ltlg_load_abstraction of the swept-volume matrix into an engine. */
ltlg_status ltlg_load_csr(ltlg_ctx* ctx, const ltlg_csr* m);
void ltlg_csr_free(ltlg_csr* m);

#ifdef __cplusplus
}
#endif

#endif /* LTLGRID_GPU_H */
