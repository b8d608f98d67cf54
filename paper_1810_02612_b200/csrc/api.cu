// api.cu -- the C ABI of include/ltlgrid_gpu.h: engine context, device memory,
// P upload / broadcast, kernel sequencing and label read-back.
//
// Reference interface replaced (proj/core/include/ltlgrid/label.hpp):
//   CsrBoolMatrix (:18-35) + validate/load (label.cpp:16-40, 271-298) -> ltlg_load_abstraction*
//   DensePropMatrix (:47-58) + label_all (:94-98, label.cpp:150-189)   -> ltlg_submit_grid*
//   LabelMatrix (:61-92)                                               -> ltlg_get_labels*
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "../../include/ltlgrid_gpu.h"
#include "engine.h"
#include "launch.h"

// The dev knobs that select A/B-only kernels (kernels.cu LTLG_AB_BUILD) act
// in the A/B build only; the product library always takes the default path.
#ifndef LTLG_AB_BUILD
#define LTLG_AB_BUILD 0
#endif
#define AB_KNOB(expr, product_value) (LTLG_AB_BUILD ? (expr) : (product_value))


using namespace ltlg;

namespace {

thread_local std::string g_error;

// --- NCCL, loaded lazily so single-device engines never need it ------------
struct Nccl {
    bool tried = false, ok = false;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
Nccl& nccl() {
    static Nccl n;
    if (!n.tried) {
        n.tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            n.CommInitAll = reinterpret_cast<decltype(n.CommInitAll)>(dlsym(h, "ncclCommInitAll"));
            n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
            n.Broadcast = reinterpret_cast<decltype(n.Broadcast)>(dlsym(h, "ncclBroadcast"));
            n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(dlsym(h, "ncclGroupStart"));
            n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
            n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
            n.ok = n.CommInitAll && n.CommDestroy && n.Broadcast && n.GroupStart && n.GroupEnd;
        }
    }
    return n;
}

// Every entry point leaves the caller's current CUDA device as it found it
// (the engine switches devices per shard).
struct DeviceGuard {
    int dev = -1;
    DeviceGuard() {
        if (cudaGetDevice(&dev) != cudaSuccess) {
            dev = -1;
            cudaGetLastError();
        }
    }
    ~DeviceGuard() {
        int now = -1;
        if (dev >= 0 && cudaGetDevice(&now) == cudaSuccess && now != dev) cudaSetDevice(dev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};

template <typename T>
struct DevBuf {
    T* ptr = nullptr;
    size_t bytes = 0;
    int device = 0;
    cudaError_t reserve(size_t b) {
        if (b <= bytes) return cudaSuccess;
        release();
        if (b == 0) return cudaSuccess;
        cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&ptr), b);
        if (e != cudaSuccess) {
            ptr = nullptr;
            bytes = 0;
            return e;
        }
        bytes = b;
        return cudaSuccess;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
    }
};

struct Shard {
    int device = 0;
    cudaStream_t stream = nullptr;
    // profiling: a ring of kRing event quintuples (submit, summary start,
    // summary end, labelling start, end); the summary may run on the comm
    // stream (ltlg_submit_grid_device_async), so its end and the labelling's
    // start are separate events
    static constexpr int kRing = 256;
    static constexpr int kEv = 5;
    std::vector<cudaEvent_t> ring;  // kRing * kEv when profiling
    uint64_t submits = 0;           // profiled submits recorded so far
    cudaEvent_t* ev = nullptr;      // the quadruple of the current submit
    uint64_t row_begin = 0, row_end = 0, n_pairs = 0, words = 0;
    uint32_t ntask_stream = 0, ntask_batch = 0;
    std::vector<uint64_t> block_row;                           // read-back blocks (local rows)
    std::vector<uint32_t> block_task_s, block_task_b;          // their first task, per layout
    cudaStream_t copy_stream = nullptr;                        // label read-back
    std::vector<cudaEvent_t> block_done;                       // per block, recorded after its launch
    int blocks_last = 0;                                       // blocks labelled by the last submit
    DevBuf<Pair> pairs, pairs_s;  // plain (multi-frame) and single-frame layouts
    DevBuf<uint8_t> t64;          // single-frame 64-cell-word copy
    DevBuf<uint64_t> mask_b64, tpair_b64, pb64;  // multi-frame 64-cell-word copy, its Pb table
    DevBuf<uint32_t> word_b64;
    DevBuf<uint32_t> touched64;  // PackedShard::touched64
    // word-major multi-frame copy (PackedShard::wm_*)
    DevBuf<uint64_t> wm_mask;
    DevBuf<uint8_t> wm_row;
    DevBuf<uint32_t> wm_gword, wm_gstart, wm_task_row, wm_task_grp;
    std::vector<uint32_t> block_task_wm;
    int wm_rows = 0;
    DevBuf<uint64_t> tbyte64;
    DevBuf<uint32_t> tn64;
    DevBuf<uint32_t> perm, trow_s, trow_b;
    DevBuf<uint64_t> tpair_s, tpair_b;
    // P (frames x props x nw64) is double-buffered: each submit takes the
    // buffer the previous submit did not read (rotate_P), so the upload /
    // broadcast of submit k+1 on the comm stream overlaps the labelling of
    // submit k; a buffer's read_done event (recorded after the labelling that
    // read it) gates its refill.
    struct PBuf {
        DevBuf<uint64_t> b;
        DevBuf<uint8_t> sf;    // the submit's summary (work buffer of the summary kernels)
        DevBuf<uint32_t> ctr;  // its persistent-kernel task counters (reset by the summary kernels)
        cudaEvent_t read_done = nullptr;
    };
    PBuf pb, pb_alt;               // pb = this submit's P
    cudaStream_t comm = nullptr;   // P upload (shard 0) and broadcast
    cudaEvent_t src_ready = nullptr, p_ready = nullptr;
    cudaEvent_t sum_done = nullptr;  // a summary built on the comm stream (ltlg_submit_grid_device_async)
    const uint64_t* P_in = nullptr;  // caller's device P used in place (single device)
    // caller's pinned host P, device-mapped: the single-frame summary kernel
    // reads it over PCIe and writes the device copy as it goes (no separate H2D).
    // That copy is PARTIAL: only the words some pair of this shard is on are
    // written (touched64), which are the only words the labeling kernel reads.
    // Any other reader of s.P after a fused submit must not assume the rest.
    // Consumed (reset) by run_label on every path.
    const uint64_t* P_host = nullptr;
    bool P_resident = true;  // Pdev() holds the last submit's P (not after a fused word-major upload)
    const uint64_t* Pdev() const { return P_in ? P_in : pb.b.ptr; }
    DevBuf<uint8_t> labels;
    DevBuf<uint64_t> stage;
    DevBuf<uint8_t> stage_hit;  // ltlg_edge_counting
    DevBuf<uint64_t> world;
    DevBuf<uint8_t> poses;
    DevBuf<uint64_t> poses_off;  // box offsets of ltlg_submit_boxes
    DevBuf<uint64_t> admitted;   // guard consumer: rows x frames admitted-guard masks
    DevBuf<uint64_t> guard_lut;  // its byte lookup table (8 x 256)
    DevBuf<uint64_t> lane_flags;  // ltlg_submit_scenario: per-(x, y) not-nominal-lane flags
    uint64_t guard_lut_key = ~0ull;  // (guard epoch, props) the uploaded table is for
    DevBuf<uint8_t> box_rng;     // and their per-axis cell ranges
    DevBuf<uint8_t> s_only;  // S mask per (word, frame)
    bool have_times = false;
    uint64_t rows() const { return row_end - row_begin; }
};

}  // namespace

struct ltlg_ctx {
    std::vector<Shard> shards;
    std::vector<ncclComm_t> comms;
    ltlg_options opts{};
    std::string err;
    bool loaded = false, submitted = false;
    uint64_t rows = 0, cols = 0, nnz = 0, words = 0, pairs = 0, t_bytes = 0;
    int props = 0, frames = 0, label_bytes = 0;
    std::vector<uint64_t> guard_pos, guard_neg;  // monitor guards (ltlg_set_guards)
    uint64_t guard_epoch = 0;                    // bumped by every ltlg_set_guards
    uint64_t cells = 0;
    // this submit's P is ready when this caller event completes
    // (ltlg_submit_grid_device_async): the engine does not order P's reads
    // after its own earlier work, so the summary can overlap the previous
    // submit's labelling on the comm stream
    cudaEvent_t ready_ev = nullptr;
};

namespace {

ltlg_status set_err(ltlg_ctx* ctx, ltlg_status s, const std::string& msg) {
    if (ctx) ctx->err = msg;
    g_error = msg;
    return s;
}

ltlg_status cuda_fail(ltlg_ctx* ctx, cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation)
        return set_err(ctx, LTLG_ENOMEM, std::string(what) + ": " + cudaGetErrorString(e));
    return set_err(ctx, LTLG_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(call, what)                                  \
    do {                                                \
        cudaError_t e_ = (call);                        \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, what); \
    } while (0)

int label_bytes_for(int props) {
    if (props <= 8) return 1;
    if (props <= 16) return 2;
    if (props <= 32) return 4;
    return 8;
}

uint32_t nw32_of(uint64_t cells) { return static_cast<uint32_t>(2 * ((cells + 63) / 64)); }

ltlg_status upload_shard(ltlg_ctx* ctx, Shard& s, const PackedShard& p) {
    CK(cudaSetDevice(s.device), "cudaSetDevice");
    s.row_begin = p.row_begin;
    s.row_end = p.row_end;
    s.n_pairs = p.n_pairs;
    s.words = p.words;
    s.ntask_stream = static_cast<uint32_t>(p.task_row_stream.size() - 1);
    s.ntask_batch = static_cast<uint32_t>(p.task_row_batch.size() - 1);
    s.block_row = p.block_row;
    s.block_task_s = p.block_task_stream;
    s.block_task_b = p.block_task_batch;
    s.block_task_wm = p.block_task_wm;
    s.wm_rows = 0;
    for (size_t k = 0; k + 1 < p.wm_task_row.size(); ++k)
        s.wm_rows = std::max(s.wm_rows, static_cast<int>(p.wm_task_row[k + 1] - p.wm_task_row[k]));
    const size_t nb = p.block_row.size() - 1;
    while (s.block_done.size() < nb) {
        cudaEvent_t ev;
        CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
        s.block_done.push_back(ev);
    }
    if (!s.copy_stream) CK(cudaStreamCreateWithFlags(&s.copy_stream, cudaStreamNonBlocking), "stream");
    auto put = [&](auto& buf, const auto& vec, const char* what) -> ltlg_status {
        using T = typename std::decay_t<decltype(vec)>::value_type;
        const size_t b = vec.size() * sizeof(T);
        cudaError_t e = buf.reserve(b ? b : sizeof(T));
        if (e != cudaSuccess) return cuda_fail(ctx, e, what);
        if (b) {
            e = cudaMemcpy(buf.ptr, vec.data(), b, cudaMemcpyHostToDevice);
            if (e != cudaSuccess) return cuda_fail(ctx, e, what);
        }
        return LTLG_OK;
    };
    ltlg_status st;
    if ((st = put(s.pairs, p.pairs, "upload T pairs")) != LTLG_OK) return st;
    if ((st = put(s.pairs_s, p.pairs_stream, "upload T pairs")) != LTLG_OK) return st;
    if ((st = put(s.t64, p.stream64, "upload T pairs")) != LTLG_OK) return st;
    if ((st = put(s.tbyte64, p.task_byte64, "upload tasks")) != LTLG_OK) return st;
    if ((st = put(s.tn64, p.task_n64, "upload tasks")) != LTLG_OK) return st;
    if ((st = put(s.mask_b64, p.mask_b64, "upload T pairs")) != LTLG_OK) return st;
    if ((st = put(s.word_b64, p.word_b64, "upload T pairs")) != LTLG_OK) return st;
    if ((st = put(s.tpair_b64, p.task_pair_b64, "upload tasks")) != LTLG_OK) return st;
    if ((st = put(s.touched64, p.touched64, "upload word map")) != LTLG_OK) return st;
    if ((st = put(s.wm_mask, p.wm_mask, "upload T pairs")) != LTLG_OK) return st;
    if ((st = put(s.wm_row, p.wm_row, "upload T pairs")) != LTLG_OK) return st;
    if ((st = put(s.wm_gword, p.wm_gword, "upload T groups")) != LTLG_OK) return st;
    if ((st = put(s.wm_gstart, p.wm_gstart, "upload T groups")) != LTLG_OK) return st;
    if ((st = put(s.wm_task_row, p.wm_task_row, "upload tasks")) != LTLG_OK) return st;
    if ((st = put(s.wm_task_grp, p.wm_task_grp, "upload tasks")) != LTLG_OK) return st;
    if ((st = put(s.perm, p.perm, "upload row permutation")) != LTLG_OK) return st;
    if ((st = put(s.trow_s, p.task_row_stream, "upload tasks")) != LTLG_OK) return st;
    if ((st = put(s.tpair_s, p.task_pair_stream, "upload tasks")) != LTLG_OK) return st;
    if ((st = put(s.trow_b, p.task_row_batch, "upload tasks")) != LTLG_OK) return st;
    if ((st = put(s.tpair_b, p.task_pair_batch, "upload tasks")) != LTLG_OK) return st;
    ctx->t_bytes += (p.pairs.size() + p.pairs_stream.size()) * sizeof(Pair) + p.stream64.size() + p.perm.size() * 4 +
                    p.mask_b64.size() * 8 + p.word_b64.size() * 4 + p.wm_mask.size() * 9 +
                    (p.wm_gword.size() + p.wm_gstart.size()) * 4;
    return LTLG_OK;
}

// Whether a multi-frame submit may take a 32-cell kernel that reads the
// shard's 32-cell pair copy: the A/B knobs, or a grid whose worst-case
// prop-lane / word-major summary needs 32-bit+ record indices (run_label).
bool env_off(const char* k) { return getenv(k) && atoi(getenv(k)) == 0; }
bool need_pairs32(uint64_t cols) {
    const uint64_t nw64 = (cols + 63) / 64;
    return env_off("LTLG_BATCH64") || env_off("LTLG_PROPLANE") || (nw64 + 1) * 64 * 64 >= (uint64_t(1) << 31);
}

// One frame: the word-major single-frame kernel, or the stream64 kernel (see run_label).
bool use_wm1(int props, uint32_t nw64) {
    const char* k = getenv("LTLG_WM1");
    if (k) return atoi(k) != 0;
    return stream64_table_loc(props, nw64) != 1;
}

// The single-frame 64-cell copy is read only where some prop count takes the
// stream64 kernel: its smallest (1-prop) split table fits in shared memory,
// or a dev knob asks for it.
bool need_stream64(uint64_t cols) {
    const uint32_t nw64 = static_cast<uint32_t>((cols + 63) / 64);
    return getenv("LTLG_WM1") || AB_KNOB(env_off("LTLG_WORDMAJOR"), false) || !use_wm1(1, nw64);
}

ltlg_status load_words(ltlg_ctx* ctx, WordCsr& t) {
    ctx->loaded = false;
    ctx->submitted = false;
    ctx->t_bytes = 0;
    const int n = static_cast<int>(ctx->shards.size());
    const uint32_t sentinel = nw32_of(t.cols);
    if (static_cast<uint64_t>(sentinel) >= kWordMask)
        return set_err(ctx, LTLG_EINVAL, "CSR column space too large for this build");
    const std::vector<uint64_t> b = shard_bounds(t, n);
    uint64_t pairs = 0;
    for (int i = 0; i < n; ++i) {
        PackedShard p;
        if (b[i + 1] - b[i] > 0xffffffffull)
            return set_err(ctx, LTLG_EINVAL, "a device shard holds more than 2^32-1 rows");
        // single-frame task size: 2048 32-cell pairs, but small abstractions get
        // smaller tasks (down to one 256-pair chunk) so that every warp of the
        // persistent grid has a task -- a lone warp streaming 2048 pairs is
        // a ~20 us critical path (cfg 2: 200k edges)
        int stream_pairs = ctx->opts.stream_task_pairs;
        if (stream_pairs <= 0) {
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->shards[static_cast<size_t>(i)].device);
            const uint64_t words = t.offsets[b[i + 1]] - t.offsets[b[i]];
            const uint64_t want = words / (static_cast<uint64_t>(sms) * 32ull);
            stream_pairs = static_cast<int>(std::min<uint64_t>(2048, std::max<uint64_t>(256, want)));
        }
        build_shard(t, b[i], b[i + 1], ctx->opts.sort_rows != 0, sentinel, stream_pairs,
                    ctx->opts.batch_task_pairs > 0 ? ctx->opts.batch_task_pairs : 256,
                    ctx->opts.readback_chunks > 1 ? (ctx->opts.readback_chunks < 64 ? ctx->opts.readback_chunks : 64) : 1,
                    &p, ctx->opts.task_rows > 0 ? std::min(ctx->opts.task_rows, 256) : kWmRows, need_pairs32(t.cols),
                    need_stream64(t.cols));
        ltlg_status st = upload_shard(ctx, ctx->shards[static_cast<size_t>(i)], p);
        if (st != LTLG_OK) return st;
        pairs += p.n_pairs;
    }
    ctx->rows = t.rows;
    ctx->cols = t.cols;
    ctx->nnz = t.nnz;
    ctx->words = t.offsets.empty() ? 0 : t.offsets[t.rows];
    ctx->pairs = pairs;
    ctx->loaded = true;
    return LTLG_OK;
}

ltlg_status check_grid(ltlg_ctx* ctx, uint64_t cells, int num_props, int frames) {
    if (!ctx) return set_err(nullptr, LTLG_EINVAL, "null context");
    if (!ctx->loaded) return set_err(ctx, LTLG_ESTATE, "no abstraction loaded");
    // DensePropMatrix ctor (label.cpp:122-128) before label_all's check (:151-154)
    if (num_props > 64) return set_err(ctx, LTLG_EINVAL, "at most 64 propositions");
    if (num_props < 0) return set_err(ctx, LTLG_EINVAL, "props must be in [0, 64]");
    if (frames < 1) return set_err(ctx, LTLG_EINVAL, "frames must be >= 1");
    if (ctx->cols != cells)
        return set_err(ctx, LTLG_EINVAL,
                       "dimension mismatch: matrix cols " + std::to_string(ctx->cols) +
                           " vs proposition rows " + std::to_string(cells));
    return LTLG_OK;
}

// Every submit: take the P buffer the previous submit did not read, sized
// for `bytes` (the caller then fills shard 0's, and broadcast_P the others).
ltlg_status rotate_P(ltlg_ctx* ctx, size_t bytes) {
    for (Shard& s : ctx->shards) {
        CK(cudaSetDevice(s.device), "cudaSetDevice");
        std::swap(s.pb, s.pb_alt);
        if (bytes) CK(s.pb.b.reserve(bytes), "allocate P");
    }
    return LTLG_OK;
}

// Shard 0's P (written on stream `src` of device 0) to every shard's P
// buffer, on the comm streams: NCCL broadcast over NVLink when the devices
// are distinct, peer copies otherwise.  Each comm stream first waits for the
// labelling that last read its buffer (read_done); each shard's labelling
// stream then waits for its broadcast (p_ready).  So the broadcast of
// submit k+1 runs while submit k labels.
ltlg_status broadcast_P(ltlg_ctx* ctx, size_t words, cudaStream_t src) {
    const int n = static_cast<int>(ctx->shards.size());
    Shard& s0 = ctx->shards[0];
    if (words == 0 || (n == 1 && src == s0.stream)) return LTLG_OK;
    CK(cudaSetDevice(s0.device), "cudaSetDevice");
    CK(cudaEventRecord(s0.src_ready, src), "event");
    for (int i = 0; i < n; ++i) {
        Shard& s = ctx->shards[static_cast<size_t>(i)];
        CK(cudaSetDevice(s.device), "cudaSetDevice");
        if (src != s.comm) CK(cudaStreamWaitEvent(s.comm, s0.src_ready, 0), "stream wait");
        CK(cudaStreamWaitEvent(s.comm, s.pb.read_done, 0), "stream wait");
    }
    if (n > 1) {
        if (!ctx->comms.empty()) {
            Nccl& N = nccl();
            N.GroupStart();
            for (int i = 0; i < n; ++i) {
                Shard& s = ctx->shards[static_cast<size_t>(i)];
                cudaSetDevice(s.device);
                ncclResult_t r = N.Broadcast(s0.pb.b.ptr, s.pb.b.ptr, words, ncclUint64, 0,
                                             ctx->comms[static_cast<size_t>(i)], s.comm);
                if (r != ncclSuccess) {
                    N.GroupEnd();
                    return set_err(ctx, LTLG_ENCCL, std::string("ncclBroadcast: ") + N.GetErrorString(r));
                }
            }
            ncclResult_t r = N.GroupEnd();
            if (r != ncclSuccess) return set_err(ctx, LTLG_ENCCL, std::string("ncclGroupEnd: ") + N.GetErrorString(r));
        } else {
            for (int i = 1; i < n; ++i) {
                Shard& s = ctx->shards[static_cast<size_t>(i)];
                CK(cudaSetDevice(s.device), "cudaSetDevice");
                CK(cudaMemcpyPeerAsync(s.pb.b.ptr, s.device, s0.pb.b.ptr, s0.device, words * 8, s.comm), "peer copy");
            }
        }
    }
    for (int i = 0; i < n; ++i) {
        Shard& s = ctx->shards[static_cast<size_t>(i)];
        CK(cudaSetDevice(s.device), "cudaSetDevice");
        CK(cudaEventRecord(s.p_ready, s.comm), "event");
        CK(cudaStreamWaitEvent(s.stream, s.p_ready, 0), "stream wait");
    }
    cudaSetDevice(s0.device);
    return LTLG_OK;
}

// Summary + labeling on every shard for P already resident in shard.P.
// Resident-label consumer: admitted-guard masks of shard s for the current
// submit (labels already enqueued on s.stream).
ltlg_status run_guards(ltlg_ctx* ctx, Shard& s) {
    const int props = ctx->props, frames = ctx->frames;
    const int nbytes = ctx->label_bytes;
    std::vector<uint64_t> lut(static_cast<size_t>(nbytes) * 256, 0);
    uint64_t always = 0;
    const size_t ng = ctx->guard_pos.size();
    for (int j = 0; j < 64; ++j) {
        uint64_t needs = 0, forbids = 0;  // guards with prop j positive / negative
        for (size_t t = 0; t < ng; ++t) {
            needs |= (ctx->guard_pos[t] >> j & 1u) << t;
            forbids |= (ctx->guard_neg[t] >> j & 1u) << t;
        }
        if (j >= 8 * nbytes || j >= props) {  // the label never carries prop j
            always |= needs;
            continue;
        }
        for (int v = 0; v < 256; ++v) lut[static_cast<size_t>(j / 8) * 256 + v] |= (v >> (j % 8) & 1) ? forbids : needs;
    }
    const uint64_t all = ng >= 64 ? ~0ull : ((1ull << ng) - 1ull);
    const uint64_t n = s.rows() * static_cast<uint64_t>(frames);
    CK(s.admitted.reserve(n * 8), "allocate guards");
    if (s.guard_lut_key != ctx->guard_epoch * 128 + static_cast<uint64_t>(props)) {  // (re)upload on change only
        CK(s.guard_lut.reserve(8 * 256 * 8), "allocate guards");
        CK(cudaMemcpyAsync(s.guard_lut.ptr, lut.data(), lut.size() * 8, cudaMemcpyHostToDevice, s.stream), "guards");
        CK(cudaStreamSynchronize(s.stream), "guards");  // the pageable upload completes before lut goes away
        s.guard_lut_key = ctx->guard_epoch * 128 + static_cast<uint64_t>(props);
    }
    CK(launch_guards(s.labels.ptr, nbytes, n, s.guard_lut.ptr, always, all, s.admitted.ptr, s.stream),
       "guard kernel");
    return LTLG_OK;
}
// A/B knob LTLG_PL_TOUCHED=0: the summaries (prop-lane and single-frame) over
// every word of the grid instead of only the words the shard's pairs are on.
static bool pl_touched_on() {
    static const bool on = !getenv("LTLG_PL_TOUCHED") || atoi(getenv("LTLG_PL_TOUCHED")) != 0;
    return on;
}


constexpr int kSmallFrames = 16;  // sweep_frames: per-frame single-frame launches win up to ~16 frames (<= 16 props)

// Multi-frame submit of few frames: per frame, the 64-cell summary + one
// single-frame launch writing labels[row * frames + f].
ltlg_status run_label_per_frame(ltlg_ctx* ctx, Shard& s, uint32_t nw64) {
    const int props = ctx->props, frames = ctx->frames;
    CK(s.pb.sf.reserve(split64_table_bytes(props, nw64)), "allocate summary");
    CK(s.pb.ctr.reserve(64 * kCtrStride * sizeof(uint32_t)), "allocate task counters");
    CK(s.s_only.reserve(static_cast<size_t>(nw64 + 1) * s_only_bytes(props)), "allocate summary");
    const bool prof = ctx->opts.profile != 0;
    if (prof) CK(cudaEventRecord(s.ev[1], s.stream), "event");
    const size_t pw = static_cast<size_t>(props) * nw64;  // u64 words of one frame's P
    static const bool wm_ok = AB_KNOB(!env_off("LTLG_WORDMAJOR"), true);
    const bool wm1 = wm_ok && s.wm_rows > 0 && use_wm1(props, nw64);  // (as for one frame, frame by frame)
    if (wm1) CK(s.pb.sf.reserve(pl_work_bytes(props, 1, nw64)), "allocate summary");
    for (int f = 0; f < frames; ++f) {
        if (wm1)
            CK(launch_pl(s.Pdev() + f * pw, props, 1, nw64, ctx->cells, s.pb.sf.ptr, s.pb.sf.bytes, s.pb.ctr.ptr,
                         static_cast<int>(kCtrStride), s.stream, pl_touched_on() ? s.touched64.ptr : nullptr),
               "summary kernel");
        else
            CK(launch_summary64(s.Pdev() + f * pw, props, nw64, ctx->cells, s.pb.sf.ptr, s.s_only.ptr, s.pb.ctr.ptr,
                                static_cast<int>(kCtrStride), s.stream, nullptr,
                                pl_touched_on() ? s.touched64.ptr : nullptr),
               "summary kernel");
        if (prof && f == 0) {
            CK(cudaEventRecord(s.ev[2], s.stream), "event");
            CK(cudaEventRecord(s.ev[3], s.stream), "event");
        }
        LaunchArgs a{};
        a.sf = s.pb.sf.ptr;
        a.P32 = reinterpret_cast<const uint32_t*>(s.Pdev() + f * pw);
        a.nw32 = 2 * nw64;
        a.props = props;
        a.frames = 1;
        a.out = s.labels.ptr + static_cast<size_t>(f) * static_cast<size_t>(ctx->label_bytes);
        a.ostride = static_cast<uint32_t>(frames);
        a.label_bytes = ctx->label_bytes;
        a.s_only = s.s_only.ptr;
        a.t64 = s.t64.ptr;
        a.task_byte64 = s.tbyte64.ptr;
        a.task_n64 = s.tn64.ptr;
        a.nw64 = nw64;
        a.task_row = s.trow_s.ptr;
        a.task_begin = 0;
        a.ntasks = s.block_task_s.back();
        a.task_ctr = s.pb.ctr.ptr;
        if (wm1) {
            a.word_major = 1;
            a.wm_mask = s.wm_mask.ptr;
            a.wm_row = s.wm_row.ptr;
            a.wm_gword = s.wm_gword.ptr;
            a.wm_gstart = s.wm_gstart.ptr;
            a.wm_task_row = s.wm_task_row.ptr;
            a.wm_task_grp = s.wm_task_grp.ptr;
            a.wm_rows = s.wm_rows;
            a.perm = s.perm.ptr;
            a.ntasks = s.block_task_wm.back();
        }
        CK(launch_label(a, s.stream), "label kernel");
    }
    s.blocks_last = 1;
    if (!ctx->guard_pos.empty()) {
        const ltlg_status gst = run_guards(ctx, s);
        if (gst != LTLG_OK) return gst;
    }
    if (prof) CK(cudaEventRecord(s.ev[4], s.stream), "event");
    s.have_times = prof;
    return LTLG_OK;
}

// split: one launch per read-back block (submits whose labels are expected
// to go back to the host: host-memory P); otherwise one launch.
ltlg_status run_label(ltlg_ctx* ctx, bool split) {
    const uint32_t nw32 = nw32_of(ctx->cells);
    const int props = ctx->props, frames = ctx->frames;
    for (Shard& s : ctx->shards) {
        CK(cudaSetDevice(s.device), "cudaSetDevice");
        // the caller's pinned P mapping is good for this submit only: consume it
        // here on every path, so no later submit (world grid, boxes, scenario)
        // can read a stale host buffer
        const uint64_t* const P_host = s.P_host;
        s.P_host = nullptr;
        s.P_resident = true;
        const size_t lab = s.rows() * static_cast<size_t>(frames) * static_cast<size_t>(ctx->label_bytes);
        CK(s.labels.reserve(lab ? lab : 8), "allocate labels");
        if (props == 0 || s.rows() == 0) {
            s.have_times = false;
            s.blocks_last = 0;
            if (s.rows() && !ctx->guard_pos.empty()) {  // no props: every label is empty
                CK(cudaMemsetAsync(s.labels.ptr, 0, lab, s.stream), "labels");
                const ltlg_status gst = run_guards(ctx, s);
                if (gst != LTLG_OK) return gst;
            }
            CK(cudaEventRecord(s.pb.read_done, s.stream), "event");
            continue;
        }
        const uint32_t nw64 = nw32 / 2;
        // 64-cell-word single-frame path (dev knob LTLG_STREAM64=0 selects the 32-cell copy for A/B runs)
        static const bool wide_ok = AB_KNOB(!getenv("LTLG_STREAM64") || atoi(getenv("LTLG_STREAM64")) != 0, true);
        const bool wide = wide_ok && frames == 1;
        if (P_host && !wide)  // the fused upload only exists on the single-frame 64-cell path
            CK(cudaMemcpyAsync(s.pb.b.ptr, P_host, static_cast<size_t>(frames) * props * nw64 * 8,
                               cudaMemcpyHostToDevice, s.stream),
               "upload P");
        // Few frames: the frame-per-lane multi-frame kernel would leave most
        // lanes idle (its cost is ~flat for frames <= 32), so label frame by
        // frame with the single-frame kernel, each launch writing one column
        // of the edge-major labels.
        // The cut-over follows the measured per-frame cost (sweep_frames.py,
        // B200): ~0.09 ms/frame up to 16 props, 0.13 at 32, 0.28-0.31 at 33-64
        // props, against the prop-lane kernel's ~1.4-2.8 ms fixed cost per
        // pass.  (dev knob LTLG_SMALL_FRAMES: a fixed cut-over, for A/B runs)
        static const int small_frames_env = getenv("LTLG_SMALL_FRAMES") ? atoi(getenv("LTLG_SMALL_FRAMES")) : -1;
        const int small_frames = small_frames_env >= 0 ? small_frames_env
                                 : props <= 16       ? kSmallFrames
                                 : props <= 32       ? 14
                                                     : 9;
        if (wide_ok && frames > 1 && frames <= small_frames) {
            const ltlg_status fst = run_label_per_frame(ctx, s, nw64);
            if (fst != LTLG_OK) return fst;
            CK(cudaEventRecord(s.pb.read_done, s.stream), "event");  // (the labelling is done with this P buffer)
            continue;
        }
        static const bool wide_b_ok = !getenv("LTLG_BATCH64") || atoi(getenv("LTLG_BATCH64")) != 0;
        const bool wide_b = wide_b_ok && frames > 1 && props <= 32;  // 64-cell-word multi-frame path
        // prop-lane kernel, in slices of <= 64 frames (dev knob LTLG_PROPLANE=0:
        // the frame-per-lane kernels); <= 32 props: one prop per lane, 33..64: two
        static const bool pl_ok = !getenv("LTLG_PROPLANE") || atoi(getenv("LTLG_PROPLANE")) != 0;
        // (the record indices are 32-bit and the work buffer is sized for the
        // worst case -- every (word, prop, frame) partial: huge grids take the
        // frame-per-lane kernels instead)
        const uint64_t pl_worst = static_cast<uint64_t>(nw64 + 1) * (props > 32 ? 64u : 32u) *
                                  static_cast<uint64_t>(std::min(frames, 64));
        const bool pl = wide_b_ok && pl_ok && frames > 1 && props <= 64 && pl_worst < (uint64_t(1) << 31);
        // word-major kernel (label_wm_kernel) over the prop-lane summary; dev knob
        // LTLG_WORDMAJOR=0: the pair-major label_pl_kernel, for A/B runs
        static const bool wm_ok = AB_KNOB(!getenv("LTLG_WORDMAJOR") || atoi(getenv("LTLG_WORDMAJOR")) != 0, true);
        const bool wm = wm_ok && s.wm_rows > 0;
        // one frame: the word-major single-frame kernel (label_wm1_kernel) over
        // the one-frame prop-lane summary where the stream64 kernel's split
        // table outgrows shared memory (its per-pair gathers then go to L1 /
        // L2: cfg-5 shard 0.273 ms vs 0.226 ms); the stream64 kernel otherwise
        // (cfg 3: 0.094 ms vs 0.141 ms).  Dev knob LTLG_WM1=0/1 forces it.
        const bool wm1 = wide && wm && props <= 64 && use_wm1(props, nw64);
        // the fused upload (summary reading pinned P through the mapping) leaves
        // no device copy of P on the word-major path: the summary holds all the
        // labelling needs (ltlg_edge_counting then asks for a resubmit)
        s.P_resident = !(wm1 && P_host);
        const int nslice = pl ? (frames + 63) / 64 : 1;
        // dev knob LTLG_TC=1: the tcgen05 kind::i8 formulation (tc_i8.cu) on
        // the word-major copy instead of label_wm_kernel (measured, not kept)
        static const bool tc_on = AB_KNOB(getenv("LTLG_TC") && atoi(getenv("LTLG_TC")) != 0, false);
        const bool tc = pl && wm && tc_on && s.wm_rows <= 128;
#if LTLG_AB_BUILD
        const size_t tc_bytes = tc ? tc_work_bytes(nw64) : 0;
#else
        const size_t tc_bytes = 0;
#endif
        CK(s.pb.sf.reserve(tc ? tc_bytes
                        : pl && wm ? wm_work_bytes(props, nw64)
                        : wm1 ? pl_work_bytes(props, 1, nw64)
                        : pl ? pl_work_bytes(props, std::min(frames, 64), nw64)
                        : wide_b ? static_cast<size_t>(nw64 + 1) * frames * 32
                        : wide ? split64_table_bytes(props, nw64)
                             : frames == 1 && props <= 32
                                   ? split_table_bytes(props, nw32)
                                   : static_cast<size_t>(nw32 + 1) * frames * summary_entry_bytes(props)),
           "allocate summary");
        CK(s.pb.ctr.reserve(64 * kCtrStride * sizeof(uint32_t)), "allocate task counters");
        CK(s.s_only.reserve(static_cast<size_t>(nw32 + 1) * frames * s_only_bytes(props)), "allocate summary");
        const bool prof = ctx->opts.profile != 0;
        // the word-major summary of an async submit runs on the comm stream,
        // after the caller's ready event and the labelling that last used this
        // summary buffer, so it overlaps the previous submit's labelling
        const bool async_sum = ctx->ready_ev && pl && wm && !tc && nslice == 1;
        const cudaStream_t sst = async_sum ? s.comm : s.stream;
        if (async_sum) {
            if (&s == &ctx->shards[0] && ctx->shards.size() == 1)
                CK(cudaStreamWaitEvent(s.comm, ctx->ready_ev, 0), "stream wait");
            CK(cudaStreamWaitEvent(s.comm, s.pb.read_done, 0), "stream wait");
        } else if (ctx->ready_ev && ctx->shards.size() == 1) {
            CK(cudaStreamWaitEvent(s.stream, ctx->ready_ev, 0), "stream wait");
        }
        if (prof) CK(cudaEventRecord(s.ev[1], sst), "event");
        const int nctr = static_cast<int>((s.block_row.size() - 1) * kCtrStride);
        for (int sl = 0; sl < nslice; ++sl) {  // (frame slices: prop-lane path only)
        // balanced slices (65 frames -> 33 + 32, not 64 + 1)
        const int f0 = frames * sl / nslice, nf = pl ? frames * (sl + 1) / nslice - f0 : frames;
        if (wm1)
            CK(launch_pl(P_host ? P_host : s.Pdev(), props, 1, nw64, ctx->cells, s.pb.sf.ptr, s.pb.sf.bytes, s.pb.ctr.ptr, nctr,
                         s.stream, pl_touched_on() ? s.touched64.ptr : nullptr),
               "summary kernel");
        else if (wide)
            CK(launch_summary64(P_host ? P_host : s.Pdev(), props, nw64, ctx->cells, s.pb.sf.ptr, s.s_only.ptr,
                                s.pb.ctr.ptr, nctr, s.stream, P_host ? s.pb.b.ptr : nullptr,
                                pl_touched_on() ? s.touched64.ptr : nullptr),
               "summary kernel");
#if LTLG_AB_BUILD
        else if (tc)
            CK(launch_tc_build(s.Pdev() + static_cast<size_t>(f0) * props * nw64, props, nf, nw64, ctx->cells, s.pb.sf.ptr,
                               s.pb.ctr.ptr, nctr, s.stream, pl_touched_on() ? s.touched64.ptr : nullptr),
               "summary kernel");
#endif
        else if (pl && wm)
            CK(launch_wm_build(s.Pdev() + static_cast<size_t>(f0) * props * nw64, props, nf, nw64, ctx->cells, s.pb.sf.ptr,
                               s.pb.sf.bytes, s.pb.ctr.ptr, nctr, sst, pl_touched_on() ? s.touched64.ptr : nullptr),
               "summary kernel");
        else if (pl)
            CK(launch_pl(s.Pdev() + static_cast<size_t>(f0) * props * nw64, props, nf, nw64, ctx->cells, s.pb.sf.ptr,
                         s.pb.sf.bytes, s.pb.ctr.ptr, nctr, s.stream, pl_touched_on() ? s.touched64.ptr : nullptr),
               "summary kernel");
        else if (wide_b)
            CK(launch_summary_b64(s.Pdev(), props, frames, nw64, ctx->cells, s.pb.sf.ptr, nullptr, s.s_only.ptr,
                                  s.pb.ctr.ptr, nctr, s.stream),
               "summary kernel");
        else
            CK(launch_summary(reinterpret_cast<const uint32_t*>(s.Pdev()), props, frames, nw32, ctx->cells, s.pb.sf.ptr,
                              s.s_only.ptr, s.pb.ctr.ptr, nctr, s.stream),
               "summary kernel");
        if (prof && sl == 0) CK(cudaEventRecord(s.ev[2], sst), "event");
        if (async_sum) {  // the labelling waits for its summary
            CK(cudaEventRecord(s.sum_done, s.comm), "event");
            CK(cudaStreamWaitEvent(s.stream, s.sum_done, 0), "stream wait");
        }
        if (prof && sl == 0) CK(cudaEventRecord(s.ev[3], s.stream), "event");
        LaunchArgs a{};
        // single frame: the labeling kernel is a programmatic dependent of the
        // summary kernel (not when profiling: the event between them would
        // serialise the two anyway)
        a.pdl = wide && !prof ? 1 : 0;
        a.pairs = s.pairs.ptr;
        a.perm = s.perm.ptr;
        a.sf = s.pb.sf.ptr;
        a.P32 = reinterpret_cast<const uint32_t*>(s.Pdev());
        a.nw32 = nw32;
        a.props = props;
        a.frames = nf;
        a.out = static_cast<uint8_t*>(s.labels.ptr) + static_cast<size_t>(f0) * static_cast<size_t>(ctx->label_bytes);
        if (nslice > 1) a.ostride = static_cast<uint32_t>(frames);
        a.label_bytes = ctx->label_bytes;
        a.s_only = s.s_only.ptr;
        const bool single = frames == 1;
        if (single) a.pairs = s.pairs_s.ptr;
        if (wide_b || pl) {
            a.prop_lane = pl ? 1 : 0;
            a.mask_b64 = s.mask_b64.ptr;
            a.word_b64 = s.word_b64.ptr;
            a.task_pair_b64 = s.tpair_b64.ptr;
            a.nw64 = nw64;
        }
        if ((pl && wm) || wm1) {
            a.word_major = 1;
            a.tc = tc ? 1 : 0;
            a.wm_mask = s.wm_mask.ptr;
            a.wm_row = s.wm_row.ptr;
            a.wm_gword = s.wm_gword.ptr;
            a.wm_gstart = s.wm_gstart.ptr;
            a.wm_task_row = s.wm_task_row.ptr;
            a.wm_task_grp = s.wm_task_grp.ptr;
            a.wm_rows = s.wm_rows;
        }
        if (wide) {
            a.t64 = s.t64.ptr;
            a.task_byte64 = s.tbyte64.ptr;
            a.task_n64 = s.tn64.ptr;
            a.nw64 = nw64;
        }
        a.task_pair = single ? s.tpair_s.ptr : s.tpair_b.ptr;
        a.task_row = single ? s.trow_s.ptr : s.trow_b.ptr;
        // one launch per read-back block for multi-frame submits (their labels are
        // large: rows x frames words); a single frame's labels are small, so it
        // runs as one launch over all tasks (tasks are listed block by block)
        const std::vector<uint32_t>& bt = single ? (wm1 ? s.block_task_wm : s.block_task_s)
                                          : (pl && wm) ? s.block_task_wm : s.block_task_b;
        const int nb = single || !split ? 1 : static_cast<int>(bt.size() - 1);
        for (int c = 0; c < nb; ++c) {
            a.task_begin = bt[static_cast<size_t>(c)];
            a.ntasks = nb == 1 ? bt.back() : bt[static_cast<size_t>(c) + 1];
            a.task_ctr = s.pb.ctr.ptr + static_cast<size_t>(c) * kCtrStride;
            CK(launch_label(a, s.stream), "label kernel");
            if (nb > 1 && sl == nslice - 1) CK(cudaEventRecord(s.block_done[static_cast<size_t>(c)], s.stream), "event");
        }
        s.blocks_last = nb;
        }  // frame slices
        if (!ctx->guard_pos.empty()) {
            const ltlg_status gst = run_guards(ctx, s);
            if (gst != LTLG_OK) return gst;
        }
        if (prof) CK(cudaEventRecord(s.ev[4], s.stream), "event");
        s.have_times = prof;
        CK(cudaEventRecord(s.pb.read_done, s.stream), "event");  // (the labelling is done with this P buffer)
    }
    ctx->submitted = true;
    return LTLG_OK;
}

ltlg_status submit(ltlg_ctx* ctx, uint64_t cells, int num_props, const uint64_t* words, int frames,
                   bool on_device, bool readback, cudaEvent_t ready = nullptr) {
    ltlg_status st = check_grid(ctx, cells, num_props, frames);
    if (st != LTLG_OK) return st;
    ctx->cells = cells;
    ctx->props = num_props;
    ctx->frames = frames;
    ctx->label_bytes = label_bytes_for(num_props);
    const size_t nwords = static_cast<size_t>(frames) * num_props * ((cells + 63) / 64);
    if (nwords && !words) return set_err(ctx, LTLG_EINVAL, "null column_words");
    // A single-device engine reads a device-resident P in place (no copy);
    // the caller keeps it alive and unmodified until the labels are ready.
    const bool in_place = on_device && ctx->shards.size() == 1;
    if ((st = rotate_P(ctx, in_place ? 0 : nwords * 8 + 16)) != LTLG_OK) return st;
    if (ctx->opts.profile)
        for (Shard& s : ctx->shards) s.ev = &s.ring[static_cast<size_t>(s.submits++ % Shard::kRing) * Shard::kEv];
    Shard& s0 = ctx->shards[0];
    CK(cudaSetDevice(s0.device), "cudaSetDevice");
    if (ctx->opts.profile) CK(cudaEventRecord(s0.ev[0], s0.stream), "event");
    s0.P_in = in_place ? words : nullptr;
    s0.P_host = nullptr;
    // One frame from pinned host memory on one device: no copy-engine upload;
    // the summary kernel reads P through the mapping and writes the device
    // copy (dev knob LTLG_FUSED_UPLOAD=0 restores the cudaMemcpyAsync).
    static const bool fuse_ok = !getenv("LTLG_FUSED_UPLOAD") || atoi(getenv("LTLG_FUSED_UPLOAD")) != 0;
    if (fuse_ok && nwords && !on_device && frames == 1 && num_props <= 64 && ctx->shards.size() == 1) {
        cudaPointerAttributes pa{};
        if (cudaPointerGetAttributes(&pa, words) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer &&
            static_cast<const uint64_t*>(pa.hostPointer) == words)
            s0.P_host = static_cast<const uint64_t*>(pa.devicePointer);
        else
            cudaGetLastError();  // pageable memory: not an error, just no mapping
    }
    // The upload: on the comm stream when there are shards to broadcast to
    // (it and the broadcast then overlap the previous submit's labelling); on
    // the labelling stream for one shard -- measured steadier for the
    // two-engine host pipeline of bench.py (e2e 1.36-1.38e10 vs 1.17-1.37e10).
    cudaStream_t src = s0.stream;
    if (nwords && !in_place && !s0.P_host) {
        if (ctx->shards.size() > 1) src = s0.comm;
        CK(cudaStreamWaitEvent(src, s0.pb.read_done, 0), "stream wait");
        if (ready) CK(cudaStreamWaitEvent(src, ready, 0), "stream wait");
        CK(cudaMemcpyAsync(s0.pb.b.ptr, words, nwords * 8, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                           src),
           "upload P");
    }
    if ((st = broadcast_P(ctx, nwords, src)) != LTLG_OK) return st;
    if (ctx->opts.profile)
        for (size_t i = 1; i < ctx->shards.size(); ++i) {
            cudaSetDevice(ctx->shards[i].device);
            cudaEventRecord(ctx->shards[i].ev[0], ctx->shards[i].stream);
        }
    ctx->ready_ev = ready;
    st = run_label(ctx, readback);
    ctx->ready_ev = nullptr;
    return st;
}

ltlg_status sync_all(ltlg_ctx* ctx) {
    for (Shard& s : ctx->shards) {
        CK(cudaSetDevice(s.device), "cudaSetDevice");
        CK(cudaStreamSynchronize(s.stream), "labeling");
    }
    return LTLG_OK;
}

}  // namespace

extern "C" {

int ltlg_abi_version(void) { return LTLG_ABI_VERSION; }

const char* ltlg_last_error(const ltlg_ctx* ctx) { return ctx ? ctx->err.c_str() : g_error.c_str(); }

ltlg_status ltlg_create_ex(const int* devices, int n_devices, const ltlg_options* opts, ltlg_ctx** out) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!out) return set_err(nullptr, LTLG_EINVAL, "null output handle");
    *out = nullptr;
    if (n_devices < 1) n_devices = 1;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return set_err(nullptr, LTLG_ECUDA,
                       std::string("no CUDA device available: ") + (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices"));
    auto ctx = std::make_unique<ltlg_ctx>();
    if (opts) ctx->opts = *opts;
    else ctx->opts.sort_rows = 1;
    ctx->shards.resize(static_cast<size_t>(n_devices));
    std::vector<int> devs;
    for (int i = 0; i < n_devices; ++i) {
        const int d = devices ? devices[i] : i;
        if (d < 0 || d >= count) return set_err(nullptr, LTLG_EINVAL, "device index out of range: " + std::to_string(d));
        Shard& s = ctx->shards[static_cast<size_t>(i)];
        s.device = d;
        devs.push_back(d);
        if ((e = cudaSetDevice(d)) != cudaSuccess) return cuda_fail(nullptr, e, "cudaSetDevice");
        int major = 0;
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d);
        if (major != 10)
            return set_err(nullptr, LTLG_ECUDA, "device " + std::to_string(d) + " is not sm_100 (built for B200 only)");
        if ((e = cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking)) != cudaSuccess)
            return cuda_fail(nullptr, e, "stream");
        if ((e = cudaStreamCreateWithFlags(&s.comm, cudaStreamNonBlocking)) != cudaSuccess)
            return cuda_fail(nullptr, e, "stream");
        for (cudaEvent_t* ev : {&s.pb.read_done, &s.pb_alt.read_done, &s.src_ready, &s.p_ready, &s.sum_done})
            if ((e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming)) != cudaSuccess)
                return cuda_fail(nullptr, e, "event");
        if (ctx->opts.profile) {
            s.ring.assign(Shard::kRing * Shard::kEv, nullptr);
            for (auto& ev : s.ring)
                if ((e = cudaEventCreate(&ev)) != cudaSuccess) return cuda_fail(nullptr, e, "event");
        }
    }
    bool distinct = true;  // a device listed twice = several shards on one GPU (tests, MIG-like splits)
    for (int i = 0; i < n_devices; ++i)
        for (int j = 0; j < i; ++j) distinct = distinct && devs[static_cast<size_t>(i)] != devs[static_cast<size_t>(j)];
    if (n_devices > 1 && distinct) {
        Nccl& N = nccl();
        if (N.ok) {
            ctx->comms.resize(static_cast<size_t>(n_devices));
            ncclResult_t r = N.CommInitAll(ctx->comms.data(), n_devices, devs.data());
            if (r != ncclSuccess) {
                ctx->comms.clear();
                return set_err(nullptr, LTLG_ENCCL, std::string("ncclCommInitAll: ") + N.GetErrorString(r));
            }
        } else {
            for (int i = 0; i < n_devices; ++i)
                for (int j = 0; j < n_devices; ++j)
                    if (i != j) {
                        cudaSetDevice(devs[static_cast<size_t>(i)]);
                        cudaDeviceEnablePeerAccess(devs[static_cast<size_t>(j)], 0);
                        cudaGetLastError();
                    }
        }
    }
    *out = ctx.release();
    return LTLG_OK;
}

ltlg_status ltlg_create(const int* devices, int n_devices, ltlg_ctx** out) {
    ltlg_options o{};
    o.sort_rows = 1;
    return ltlg_create_ex(devices, n_devices, &o, out);
}

void ltlg_destroy(ltlg_ctx* ctx) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!ctx) return;
    for (ncclComm_t c : ctx->comms) nccl().CommDestroy(c);
    for (Shard& s : ctx->shards) {
        cudaSetDevice(s.device);
        if (s.stream) cudaStreamSynchronize(s.stream);
        s.pairs.release();
        s.pairs_s.release();
        s.t64.release();
        s.tbyte64.release();
        s.tn64.release();
        s.mask_b64.release();
        s.word_b64.release();
        s.touched64.release();
        s.tpair_b64.release();
        s.pb64.release();
        s.perm.release();
        s.trow_s.release();
        s.trow_b.release();
        s.tpair_s.release();
        s.tpair_b.release();
        for (Shard::PBuf* q : {&s.pb, &s.pb_alt}) {
            q->b.release();
            q->sf.release();
            q->ctr.release();
        }
        for (cudaEvent_t ev : {s.pb.read_done, s.pb_alt.read_done, s.src_ready, s.p_ready, s.sum_done})
            if (ev) cudaEventDestroy(ev);
        if (s.comm) cudaStreamDestroy(s.comm);
        s.pb.sf.release();
        s.labels.release();
        s.stage.release();
        s.world.release();
        s.poses.release();
        s.poses_off.release();
        s.admitted.release();
        s.guard_lut.release();
        s.lane_flags.release();
        s.box_rng.release();
        s.pb.ctr.release();
        s.s_only.release();
        for (auto& ev : s.ring)
            if (ev) cudaEventDestroy(ev);
        for (auto& ev : s.block_done) cudaEventDestroy(ev);
        if (s.copy_stream) cudaStreamDestroy(s.copy_stream);
        if (s.stream) cudaStreamDestroy(s.stream);
    }
    delete ctx;
}

ltlg_status ltlg_load_abstraction(ltlg_ctx* ctx, uint64_t rows, uint64_t cols, const uint64_t* row_offsets,
                                  const uint32_t* col_indices) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!ctx) return set_err(nullptr, LTLG_EINVAL, "null context");
    if (!row_offsets) return set_err(ctx, LTLG_EINVAL, "row_offsets must have rows+1 entries");
    Error err{S_OK, ""};
    const uint64_t nnz = row_offsets[rows];
    if (nnz && !col_indices) return set_err(ctx, LTLG_EINVAL, "null col_indices");
    if (!validate_csr(rows, cols, row_offsets, rows + 1, col_indices, nnz, &err))
        return set_err(ctx, static_cast<ltlg_status>(err.code), err.msg);
    if (cols > (1ull << 36)) return set_err(ctx, LTLG_EINVAL, "CSR column space too large for this build");
    WordCsr t;
    if (!pack_csr(rows, cols, row_offsets, col_indices, &t, &err))
        return set_err(ctx, static_cast<ltlg_status>(err.code), err.msg);
    return load_words(ctx, t);
}

ltlg_status ltlg_load_abstraction_file(ltlg_ctx* ctx, const char* path) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!ctx) return set_err(nullptr, LTLG_EINVAL, "null context");
    if (!path) return set_err(ctx, LTLG_EINVAL, "null path");
    Error err{S_OK, ""};
    WordCsr t;
    if (!read_csb1_words(path, &t, &err)) return set_err(ctx, static_cast<ltlg_status>(err.code), err.msg);
    return load_words(ctx, t);
}

ltlg_status ltlg_load_abstraction_words(ltlg_ctx* ctx, uint64_t rows, uint64_t cols, const uint64_t* row_word_offsets,
                                        const uint32_t* word_index, const uint32_t* word_mask) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!ctx) return set_err(nullptr, LTLG_EINVAL, "null context");
    if (!row_word_offsets) return set_err(ctx, LTLG_EINVAL, "row_offsets must have rows+1 entries");
    if (row_word_offsets[rows] && (!word_index || !word_mask))
        return set_err(ctx, LTLG_EINVAL, "null word arrays");
    if (cols > (1ull << 36)) return set_err(ctx, LTLG_EINVAL, "CSR column space too large for this build");
    Error err{S_OK, ""};
    WordCsr t;
    if (!take_words(rows, cols, row_word_offsets, word_index, word_mask, &t, &err))
        return set_err(ctx, static_cast<ltlg_status>(err.code), err.msg);
    return load_words(ctx, t);
}

ltlg_status ltlg_submit_grid(ltlg_ctx* ctx, uint64_t cells, int num_props, const uint64_t* column_words, int frames) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    return submit(ctx, cells, num_props, column_words, frames, false, true);
}

ltlg_status ltlg_submit_grid_device(ltlg_ctx* ctx, uint64_t cells, int num_props, const uint64_t* dev_words,
                                    int frames) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    return submit(ctx, cells, num_props, dev_words, frames, true, false);
}

ltlg_status ltlg_submit_grid_device_ex(ltlg_ctx* ctx, uint64_t cells, int num_props, const uint64_t* dev_words,
                                       int frames, int readback) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    return submit(ctx, cells, num_props, dev_words, frames, true, readback != 0);
}

ltlg_status ltlg_submit_grid_device_async(ltlg_ctx* ctx, uint64_t cells, int num_props, const uint64_t* dev_words,
                                          int frames, int readback, void* ready_event) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!ready_event) return set_err(ctx, LTLG_EINVAL, "null ready event");
    return submit(ctx, cells, num_props, dev_words, frames, true, readback != 0, static_cast<cudaEvent_t>(ready_event));
}

ltlg_status ltlg_submit_world_grid(ltlg_ctx* ctx, const ltlg_grid2* vehicle, const ltlg_grid2* world, int num_props,
                                   const uint64_t* world_words, int words_on_device, const ltlg_pose2* poses,
                                   int frames, int outside) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!ctx) return set_err(nullptr, LTLG_EINVAL, "null context");
    if (!vehicle || !world || !poses) return set_err(ctx, LTLG_EINVAL, "null grid or pose");
    if (vehicle->depth < 2 || vehicle->depth > 32 || world->depth < 2 || world->depth > 32)
        return set_err(ctx, LTLG_EINVAL, "grid depth must be in [2, 32]");
    if (!(vehicle->lo0 < vehicle->hi0 && vehicle->lo1 < vehicle->hi1 && world->lo0 < world->hi0 &&
          world->lo1 < world->hi1))
        return set_err(ctx, LTLG_EINVAL, "grid bounds must satisfy lo < hi");
    const uint64_t cells = 1ull << vehicle->depth;
    ltlg_status st = check_grid(ctx, cells, num_props, frames);
    if (st != LTLG_OK) return st;
    ctx->cells = cells;
    ctx->props = num_props;
    ctx->frames = frames;
    ctx->label_bytes = label_bytes_for(num_props);
    const uint64_t wcells = 1ull << world->depth;
    const size_t wwords = static_cast<size_t>(num_props) * ((wcells + 63) / 64);
    const size_t vwords = static_cast<size_t>(frames) * num_props * ((cells + 63) / 64);
    if (wwords && !world_words) return set_err(ctx, LTLG_EINVAL, "null world_words");
    if ((st = rotate_P(ctx, vwords * 8 + 16)) != LTLG_OK) return st;
    if (ctx->opts.profile)
        for (Shard& s : ctx->shards) s.ev = &s.ring[static_cast<size_t>(s.submits++ % Shard::kRing) * Shard::kEv];
    Shard& s0 = ctx->shards[0];
    CK(cudaSetDevice(s0.device), "cudaSetDevice");
    s0.P_in = nullptr;
    if (ctx->opts.profile) CK(cudaEventRecord(s0.ev[0], s0.stream), "event");
    const uint64_t* wsrc = world_words;
    if (!words_on_device && wwords) {
        CK(s0.world.reserve(wwords * 8), "allocate world grid");
        CK(cudaMemcpyAsync(s0.world.ptr, world_words, wwords * 8, cudaMemcpyHostToDevice, s0.stream), "upload world");
        wsrc = s0.world.ptr;
    }
    CK(s0.poses.reserve(sizeof(ltlg_pose2) * static_cast<size_t>(frames)), "allocate poses");
    CK(cudaMemcpyAsync(s0.poses.ptr, poses, sizeof(ltlg_pose2) * static_cast<size_t>(frames), cudaMemcpyHostToDevice,
                       s0.stream),
       "upload poses");
    CK(launch_resample(vehicle->depth, vehicle->lo0, vehicle->hi0, vehicle->lo1, vehicle->hi1, world->depth, world->lo0,
                       world->hi0, world->lo1, world->hi1, s0.poses.ptr, frames, num_props,
                       reinterpret_cast<const uint32_t*>(wsrc), nw32_of(wcells), outside ? 1 : 0, nw32_of(cells),
                       reinterpret_cast<uint32_t*>(s0.pb.b.ptr), s0.stream),
       "resample kernel");
    // pageable pose upload must complete before the caller's buffer may change
    CK(cudaStreamSynchronize(s0.stream), "resample");
    if ((st = broadcast_P(ctx, vwords, s0.stream)) != LTLG_OK) return st;
    return run_label(ctx, !words_on_device);
}

ltlg_status ltlg_submit_grid_files(ltlg_ctx* ctx, const char* const* paths, int num_props, int frames) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!ctx) return set_err(nullptr, LTLG_EINVAL, "null context");
    if (!ctx->loaded) return set_err(ctx, LTLG_ESTATE, "no abstraction loaded");
    if (num_props > 64) return set_err(ctx, LTLG_EINVAL, "at most 64 propositions");
    if (num_props < 0) return set_err(ctx, LTLG_EINVAL, "props must be in [0, 64]");
    if (frames < 1) return set_err(ctx, LTLG_EINVAL, "frames must be >= 1");
    const size_t nw = (ctx->cols + 63) / 64;
    const size_t n = static_cast<size_t>(frames) * static_cast<size_t>(num_props);
    if (n && !paths) return set_err(ctx, LTLG_EINVAL, "null paths");
    // read every column straight into one pinned staging buffer, then submit
    uint64_t* staging = nullptr;
    if (n) {
        Shard& s0 = ctx->shards[0];
        CK(cudaSetDevice(s0.device), "cudaSetDevice");
        CK(cudaHostAlloc(reinterpret_cast<void**>(&staging), n * nw * 8, cudaHostAllocDefault), "pinned staging");
    }
    std::unique_ptr<uint64_t, cudaError_t (*)(void*)> hold(staging, cudaFreeHost);
    for (size_t i = 0; i < n; ++i) {
        Error err{S_OK, ""};
        if (!paths[i]) return set_err(ctx, LTLG_EINVAL, "null path");
        if (!read_zobv(paths[i], ctx->cols, staging + i * nw, &err))
            return set_err(ctx, static_cast<ltlg_status>(err.code), err.msg);
    }
    ltlg_status st = submit(ctx, ctx->cols, num_props, staging, frames, false, true);
    if (st == LTLG_OK && n) st = sync_all(ctx);  // the staging buffer is freed on return
    return st;
}

ltlg_status ltlg_save_labels(ltlg_ctx* ctx, int frame, const char* path) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!ctx) return set_err(nullptr, LTLG_EINVAL, "null context");
    if (!path) return set_err(ctx, LTLG_EINVAL, "null path");
    if (!ctx->submitted) return set_err(ctx, LTLG_ESTATE, "no grid submitted");
    if (frame < 0 || frame >= ctx->frames) return set_err(ctx, LTLG_EINVAL, "frame out of range");
    const int wpr = (ctx->props + 63) / 64;
    std::vector<uint64_t> words(ctx->rows * static_cast<uint64_t>(wpr));
    if (!words.empty()) {
        ltlg_status st = ltlg_get_labels(ctx, frame, words.data());
        if (st != LTLG_OK) return st;
    } else {
        ltlg_status st = sync_all(ctx);
        if (st != LTLG_OK) return st;
    }
    Error err{S_OK, ""};
    if (!write_lbm1(path, ctx->rows, ctx->props, words.data(), &err))
        return set_err(ctx, static_cast<ltlg_status>(err.code), err.msg);
    return LTLG_OK;
}

ltlg_status ltlg_read_csb1_words(const char* path, uint64_t* rows, uint64_t* cols, uint64_t* nnz, uint64_t* words) {
    if (!path) return set_err(nullptr, LTLG_EINVAL, "null path");
    Error err{S_OK, ""};
    WordCsr t;
    if (!read_csb1_words(path, &t, &err)) return set_err(nullptr, static_cast<ltlg_status>(err.code), err.msg);
    if (rows) *rows = t.rows;
    if (cols) *cols = t.cols;
    if (nnz) *nnz = t.nnz;
    if (words) *words = t.offsets.empty() ? 0 : t.offsets[t.rows];
    return LTLG_OK;
}

ltlg_status ltlg_read_zobv(const char* path, uint64_t cells, uint64_t* words_out) {
    if (!path || (!words_out && cells)) return set_err(nullptr, LTLG_EINVAL, "null argument");
    Error err{S_OK, ""};
    if (!read_zobv(path, cells, words_out, &err)) return set_err(nullptr, static_cast<ltlg_status>(err.code), err.msg);
    return LTLG_OK;
}

}  // extern "C"

namespace {

// GridSpec ctor checks (grid.cpp:18-33) + this build's limits.
ltlg_status check_gridk(ltlg_ctx* ctx, const ltlg_gridk* g) {
    if (!g) return set_err(ctx, LTLG_EINVAL, "null grid");
    if (g->dims < 1) return set_err(ctx, LTLG_EINVAL, "grid needs at least one axis");
    if (g->depth < g->dims || g->depth > 63) return set_err(ctx, LTLG_EINVAL, "grid depth must be in [k, 63]");
    for (int a = 0; a < g->dims && a < 4; ++a)
        if (!(g->lo[a] < g->hi[a])) return set_err(ctx, LTLG_EINVAL, "grid bounds must satisfy lo < hi");
    if (g->dims > 4) return set_err(ctx, LTLG_EINVAL, "at most 4 grid axes in this build");
    if (g->depth > 36) return set_err(ctx, LTLG_EINVAL, "grid depth > 36 not supported by this build");
    return LTLG_OK;
}

// overlap_cells (grid.cpp:49-61) of every box on every axis -> int64 ranges
// (first, last) x 4 per box; an empty overlap on any axis empties the box.
std::vector<int64_t> box_ranges(const ltlg_gridk* g, uint64_t nboxes, const double* blo, const double* bhi) {
    std::vector<int64_t> r(nboxes * 8, 0);
    for (uint64_t b = 0; b < nboxes; ++b) {
        bool empty = false;
        for (int a = 0; a < 4; ++a) {
            int64_t first = 0, last = 0;
            if (a < g->dims) {
                const int bits = g->depth / g->dims + (a < g->depth % g->dims ? 1 : 0);
                const double lo = g->lo[a], hi = g->hi[a];
                const double cells = static_cast<double>(uint64_t(1) << bits);
                const double z_lo = (blo[b * g->dims + a] - lo) / (hi - lo) * cells;
                const double z_hi = (bhi[b * g->dims + a] - lo) / (hi - lo) * cells;
                first = static_cast<int64_t>(std::floor(z_lo));
                last = static_cast<int64_t>(std::ceil(z_hi)) - 1;
                first = std::max<int64_t>(first, 0);
                last = std::min<int64_t>(last, static_cast<int64_t>(uint64_t(1) << bits) - 1);
                if (first > last) empty = true;
            }
            r[b * 8 + 2 * a] = first;
            r[b * 8 + 2 * a + 1] = last;
        }
        if (empty) {  // rasterize_box_impl returns early: no cells
            r[b * 8] = 1;
            r[b * 8 + 1] = 0;
        }
    }
    return r;
}

// Upload ranges/offsets to `dev` scratch buffers and rasterize into out (device).
ltlg_status rasterize_on(ltlg_ctx* ctx, const ltlg_gridk* g, int cols, const uint64_t* box_off, const double* blo,
                         const double* bhi, DevBuf<uint64_t>& off_buf, DevBuf<uint8_t>& rng_buf, uint64_t* out,
                         cudaStream_t st) {
    const uint64_t nboxes = cols ? box_off[cols] : 0;
    for (int c = 0; c < cols; ++c)
        if (box_off[c] > box_off[c + 1]) return set_err(ctx, LTLG_EINVAL, "box_offsets must be nondecreasing");
    const std::vector<int64_t> r = box_ranges(g, nboxes, blo, bhi);
    CK(off_buf.reserve(static_cast<size_t>(cols + 1) * 8), "allocate boxes");
    CK(rng_buf.reserve(r.empty() ? 8 : r.size() * 8), "allocate boxes");
    CK(cudaMemcpyAsync(off_buf.ptr, box_off, static_cast<size_t>(cols + 1) * 8, cudaMemcpyHostToDevice, st), "upload boxes");
    if (!r.empty())
        CK(cudaMemcpyAsync(rng_buf.ptr, r.data(), r.size() * 8, cudaMemcpyHostToDevice, st), "upload boxes");
    CK(launch_rasterize(g->dims, g->depth, cols, off_buf.ptr, reinterpret_cast<const int64_t*>(rng_buf.ptr), out, st),
       "rasterize kernel");
    // the pageable range upload must complete before r goes out of scope
    CK(cudaStreamSynchronize(st), "rasterize");
    return LTLG_OK;
}

}  // namespace

extern "C" {

ltlg_status ltlg_rasterize_boxes(const ltlg_gridk* grid, int num_cols, const uint64_t* box_offsets,
                                 const double* box_lo, const double* box_hi, int device, uint64_t* out_words) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    ltlg_ctx* ctx = nullptr;
    ltlg_status st = check_gridk(nullptr, grid);
    if (st != LTLG_OK) return st;
    if (num_cols < 0 || (num_cols && (!box_offsets || !out_words)))
        return set_err(nullptr, LTLG_EINVAL, "null argument");
    if (num_cols && box_offsets[num_cols] && (!box_lo || !box_hi)) return set_err(nullptr, LTLG_EINVAL, "null boxes");
    const int devs[1] = {device};
    if ((st = ltlg_create(devs, 1, &ctx)) != LTLG_OK) return st;
    std::unique_ptr<ltlg_ctx, void (*)(ltlg_ctx*)> hold(ctx, ltlg_destroy);
    Shard& s0 = ctx->shards[0];
    const size_t nw = ((uint64_t(1) << grid->depth) + 63) / 64;
    CK(s0.world.reserve(static_cast<size_t>(num_cols) * nw * 8 + 8), "allocate P");  // (scratch: not a submit's P)
    st = rasterize_on(ctx, grid, num_cols, box_offsets, box_lo, box_hi, s0.poses_off, s0.box_rng, s0.world.ptr, s0.stream);
    if (st != LTLG_OK) {
        g_error = ctx->err;
        return st;
    }
    if (num_cols) {
        cudaError_t e = cudaMemcpy(out_words, s0.world.ptr, static_cast<size_t>(num_cols) * nw * 8, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return cuda_fail(nullptr, e, "download P");
    }
    return LTLG_OK;
}

ltlg_status ltlg_submit_boxes(ltlg_ctx* ctx, const ltlg_gridk* grid, int num_props, int frames,
                              const uint64_t* box_offsets, const double* box_lo, const double* box_hi) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!ctx) return set_err(nullptr, LTLG_EINVAL, "null context");
    ltlg_status st = check_gridk(ctx, grid);
    if (st != LTLG_OK) return st;
    const uint64_t cells = uint64_t(1) << grid->depth;
    if ((st = check_grid(ctx, cells, num_props, frames)) != LTLG_OK) return st;
    const int cols = frames * num_props;
    if (cols && !box_offsets) return set_err(ctx, LTLG_EINVAL, "null box_offsets");
    if (cols && box_offsets[cols] && (!box_lo || !box_hi)) return set_err(ctx, LTLG_EINVAL, "null boxes");
    ctx->cells = cells;
    ctx->props = num_props;
    ctx->frames = frames;
    ctx->label_bytes = label_bytes_for(num_props);
    const size_t nwords = static_cast<size_t>(cols) * ((cells + 63) / 64);
    if ((st = rotate_P(ctx, nwords * 8 + 16)) != LTLG_OK) return st;
    if (ctx->opts.profile)
        for (Shard& s : ctx->shards) s.ev = &s.ring[static_cast<size_t>(s.submits++ % Shard::kRing) * Shard::kEv];
    Shard& s0 = ctx->shards[0];
    CK(cudaSetDevice(s0.device), "cudaSetDevice");
    s0.P_in = nullptr;
    if (ctx->opts.profile) CK(cudaEventRecord(s0.ev[0], s0.stream), "event");
    if ((st = rasterize_on(ctx, grid, cols, box_offsets, box_lo, box_hi, s0.poses_off, s0.box_rng, s0.pb.b.ptr, s0.stream)) !=
        LTLG_OK)
        return st;
    if ((st = broadcast_P(ctx, nwords, s0.stream)) != LTLG_OK) return st;
    return run_label(ctx, false);
}

}  // extern "C"

namespace {

// SplitMix64 / mix_seed (rng.hpp:10-35)
struct Splitmix {
    uint64_t state;
    uint64_t next() {
        uint64_t z = (state += 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
};
uint64_t mix_seed(uint64_t seed, uint64_t stream) {
    Splitmix r{seed ^ (stream * 0x9e3779b97f4a7c15ull + 0x2545f4914f6cdd1dull)};
    return r.next();
}

// generate_scenario's host geometry (scenario.cpp:52-128), the same double
// operations in the same order: the agents' boxes of one query (3 lo + 3 hi
// doubles each) and, if lane != nullptr, the per-(cx, cy) not-nominal flags
// (bit cy * nx + cx).
ltlg_status scenario_geometry(ltlg_ctx* ctx, const ltlg_scenario* c, const ltlg_gridk* g, uint64_t query,
                              std::vector<double>* blo, std::vector<double>* bhi, std::vector<uint64_t>* lane) {
    constexpr double kPi = 3.14159265358979323846;
    if (g->dims != 3) return set_err(ctx, LTLG_EINVAL, "scenario needs a 3-d (x, y, tau) grid");
    if (c->horizon > g->hi[2] - g->lo[2] + 1e-9)
        return set_err(ctx, LTLG_EINVAL, "horizon exceeds the grid's tau extent");
    int bits[3];
    double w[3];
    for (int a = 0; a < 3; ++a) {
        bits[a] = g->depth / 3 + (a < g->depth % 3 ? 1 : 0);
        w[a] = (g->hi[a] - g->lo[a]) / static_cast<double>(uint64_t(1) << bits[a]);  // GridSpec::cell_width
    }
    const uint64_t nx = uint64_t(1) << bits[0], ny = uint64_t(1) << bits[1], nt = uint64_t(1) << bits[2];
    if (lane) {
        lane->assign((nx * ny + 63) / 64, 0);
        const double half_lane = c->lane_width / 2;
        for (uint64_t cx = 0; cx < nx; ++cx) {
            const double x = g->lo[0] + (static_cast<double>(cx) + 0.5) * w[0];
            for (uint64_t cy = 0; cy < ny; ++cy) {
                const double y = g->lo[1] + (static_cast<double>(cy) + 0.5) * w[1];
                const double r = std::hypot(x - c->loop_cx, y - c->loop_cy);
                if (std::abs(r - c->loop_radius) <= half_lane) continue;  // nominal lane
                const uint64_t f = cy * nx + cx;
                (*lane)[f >> 6] |= uint64_t(1) << (f & 63);
            }
        }
    }
    Splitmix rng{mix_seed(c->seed, query)};
    const double w_tau = w[2];
    for (int agent = 0; agent < c->agent_count; ++agent) {
        const double angle0 = rng.uniform(0, 2 * kPi);
        const double direction = rng.uniform() < 0.5 ? 1.0 : -1.0;
        const double speed = rng.uniform(c->agent_speed_min, c->agent_speed_max);
        const double radius = c->loop_radius + rng.uniform(-c->lateral_spread, c->lateral_spread);
        if (radius <= 1.0) return set_err(ctx, LTLG_EDOMAIN, "agent radius collapsed to the loop centre");
        const double omega = direction * speed / radius;
        auto extent = [&](double tau, double& x_lo, double& x_hi, double& y_lo, double& y_hi) {
            const double phi = angle0 + omega * tau;
            const double px = c->loop_cx + radius * std::cos(phi);
            const double py = c->loop_cy + radius * std::sin(phi);
            const double heading = phi + direction * kPi / 2;
            const double ext_x = c->agent_length / 2 * std::abs(std::cos(heading)) +
                                 c->agent_width / 2 * std::abs(std::sin(heading));
            const double ext_y = c->agent_length / 2 * std::abs(std::sin(heading)) +
                                 c->agent_width / 2 * std::abs(std::cos(heading));
            x_lo = px - ext_x;
            x_hi = px + ext_x;
            y_lo = py - ext_y;
            y_hi = py + ext_y;
        };
        const auto slabs = static_cast<uint64_t>(std::min<double>(static_cast<double>(nt), std::ceil(c->horizon / w_tau)));
        for (uint64_t ct = 0; ct < slabs; ++ct) {
            const double tau_a = static_cast<double>(ct) * w_tau;
            const double tau_b = tau_a + w_tau;
            double ax0, ax1, ay0, ay1, bx0, bx1, by0, by1;
            extent(tau_a, ax0, ax1, ay0, ay1);
            extent(tau_b, bx0, bx1, by0, by1);
            const double lo[3] = {std::min(ax0, bx0), std::min(ay0, by0),
                                  g->lo[2] + (static_cast<double>(ct) + 0.25) * w_tau};
            const double hi[3] = {std::max(ax1, bx1), std::max(ay1, by1),
                                  g->lo[2] + (static_cast<double>(ct) + 0.75) * w_tau};
            if (lo[0] < g->lo[0] || hi[0] > g->hi[0] || lo[1] < g->lo[1] || hi[1] > g->hi[1])
                return set_err(ctx, LTLG_EDOMAIN, "agent outside workspace");
            blo->insert(blo->end(), lo, lo + 3);
            bhi->insert(bhi->end(), hi, hi + 3);
        }
    }
    return LTLG_OK;
}

// frames scenario queries into P (device): column 2 f = moving_vehicle of
// query q0 + f, column 2 f + 1 = not_nominal_lane.
ltlg_status scenario_on(ltlg_ctx* ctx, const ltlg_scenario* c, const ltlg_gridk* g, uint64_t q0, int frames,
                        Shard& s, uint64_t* P) {
    std::vector<double> blo, bhi;
    std::vector<uint64_t> lane, off(static_cast<size_t>(2 * frames) + 1, 0);
    for (int f = 0; f < frames; ++f) {
        const ltlg_status st = scenario_geometry(ctx, c, g, q0 + static_cast<uint64_t>(f), &blo, &bhi,
                                                 f == 0 ? &lane : nullptr);
        if (st != LTLG_OK) return st;
        off[static_cast<size_t>(2 * f) + 1] = blo.size() / 3;  // moving_vehicle: this query's boxes
        off[static_cast<size_t>(2 * f) + 2] = blo.size() / 3;  // not_nominal_lane: no boxes (lane kernel)
    }
    ltlg_status st = rasterize_on(ctx, g, 2 * frames, off.data(), blo.data(), bhi.data(), s.poses_off, s.box_rng, P,
                                  s.stream);
    if (st != LTLG_OK) return st;
    CK(s.lane_flags.reserve(lane.size() * 8), "allocate lane flags");
    CK(cudaMemcpyAsync(s.lane_flags.ptr, lane.data(), lane.size() * 8, cudaMemcpyHostToDevice, s.stream), "upload lane");
    CK(launch_lane(g->depth, s.lane_flags.ptr, frames, 1, 2, P, s.stream), "lane kernel");
    CK(cudaStreamSynchronize(s.stream), "scenario");  // the pageable lane flags are read before they go away
    return LTLG_OK;
}

}  // namespace

extern "C" {

ltlg_status ltlg_generate_scenario(const ltlg_scenario* cfg, const ltlg_gridk* grid, uint64_t query_index,
                                   int device, uint64_t* out_words) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!cfg || !out_words) return set_err(nullptr, LTLG_EINVAL, "null argument");
    ltlg_status st = check_gridk(nullptr, grid);
    if (st != LTLG_OK) return st;
    ltlg_ctx* ctx = nullptr;
    const int devs[1] = {device};
    if ((st = ltlg_create(devs, 1, &ctx)) != LTLG_OK) return st;
    std::unique_ptr<ltlg_ctx, void (*)(ltlg_ctx*)> hold(ctx, ltlg_destroy);
    Shard& s0 = ctx->shards[0];
    const size_t nw = ((uint64_t(1) << grid->depth) + 63) / 64;
    CK(s0.world.reserve(2 * nw * 8 + 8), "allocate P");  // (scratch: not a submit's P)
    if ((st = scenario_on(ctx, cfg, grid, query_index, 1, s0, s0.world.ptr)) != LTLG_OK) {
        g_error = ctx->err;
        return st;
    }
    cudaError_t e = cudaMemcpy(out_words, s0.world.ptr, 2 * nw * 8, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(nullptr, e, "download P");
    return LTLG_OK;
}

ltlg_status ltlg_submit_scenario(ltlg_ctx* ctx, const ltlg_scenario* cfg, const ltlg_gridk* grid,
                                 uint64_t query_index0, int frames) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!ctx) return set_err(nullptr, LTLG_EINVAL, "null context");
    if (!cfg) return set_err(ctx, LTLG_EINVAL, "null argument");
    ltlg_status st = check_gridk(ctx, grid);
    if (st != LTLG_OK) return st;
    const uint64_t cells = uint64_t(1) << grid->depth;
    if ((st = check_grid(ctx, cells, 2, frames)) != LTLG_OK) return st;
    ctx->cells = cells;
    ctx->props = 2;
    ctx->frames = frames;
    ctx->label_bytes = label_bytes_for(2);
    const size_t nwords = static_cast<size_t>(frames) * 2 * ((cells + 63) / 64);
    if ((st = rotate_P(ctx, nwords * 8 + 16)) != LTLG_OK) return st;
    if (ctx->opts.profile)
        for (Shard& s : ctx->shards) s.ev = &s.ring[static_cast<size_t>(s.submits++ % Shard::kRing) * Shard::kEv];
    Shard& s0 = ctx->shards[0];
    CK(cudaSetDevice(s0.device), "cudaSetDevice");
    s0.P_in = nullptr;
    s0.P_host = nullptr;
    if (ctx->opts.profile) CK(cudaEventRecord(s0.ev[0], s0.stream), "event");
    if ((st = scenario_on(ctx, cfg, grid, query_index0, frames, s0, s0.pb.b.ptr)) != LTLG_OK) return st;
    if ((st = broadcast_P(ctx, nwords, s0.stream)) != LTLG_OK) return st;
    return run_label(ctx, false);
}

ltlg_status ltlg_set_guards(ltlg_ctx* ctx, int n_guards, const uint64_t* positive, const uint64_t* negative) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!ctx) return set_err(nullptr, LTLG_EINVAL, "null context");
    if (n_guards < 0 || n_guards > 64) return set_err(ctx, LTLG_EINVAL, "guards must be in [0, 64]");
    if (n_guards && (!positive || !negative)) return set_err(ctx, LTLG_EINVAL, "null guards");
    ctx->guard_pos.assign(positive, positive + n_guards);
    ctx->guard_neg.assign(negative, negative + n_guards);
    ++ctx->guard_epoch;
    return LTLG_OK;
}

ltlg_status ltlg_get_admitted(ltlg_ctx* ctx, int frame, uint64_t* out) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!ctx) return set_err(nullptr, LTLG_EINVAL, "null context");
    if (!ctx->submitted) return set_err(ctx, LTLG_ESTATE, "no grid submitted");
    if (ctx->guard_pos.empty()) return set_err(ctx, LTLG_ESTATE, "no guards set");
    if (frame < 0 || frame >= ctx->frames) return set_err(ctx, LTLG_EINVAL, "frame out of range");
    if (ctx->rows && !out) return set_err(ctx, LTLG_EINVAL, "null output");
    for (Shard& s : ctx->shards) {
        if (s.rows() == 0) continue;
        CK(cudaSetDevice(s.device), "cudaSetDevice");
        // strided copy: frame `frame` of every edge (edge-major rows x frames)
        CK(cudaMemcpy2DAsync(out + s.row_begin, 8, s.admitted.ptr + frame, static_cast<size_t>(ctx->frames) * 8, 8,
                             s.rows(), cudaMemcpyDeviceToHost, s.stream),
           "download admitted");
    }
    return sync_all(ctx);
}

ltlg_status ltlg_device_admitted(ltlg_ctx* ctx, int shard, void** dev_ptr) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!ctx || !dev_ptr) return set_err(ctx, LTLG_EINVAL, "null argument");
    if (shard < 0 || shard >= static_cast<int>(ctx->shards.size())) return set_err(ctx, LTLG_EINVAL, "shard out of range");
    if (!ctx->submitted || ctx->guard_pos.empty()) return set_err(ctx, LTLG_ESTATE, "no guarded submit");
    *dev_ptr = ctx->shards[static_cast<size_t>(shard)].admitted.ptr;
    return LTLG_OK;
}

ltlg_status ltlg_wait(ltlg_ctx* ctx) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!ctx) return set_err(nullptr, LTLG_EINVAL, "null context");
    return sync_all(ctx);
}

ltlg_status ltlg_apply_labels(ltlg_ctx* ctx, int frame, uint64_t num_edges, int alphabet_size, uint64_t* symbols) {
    if (!ctx) return set_err(nullptr, LTLG_EINVAL, "null context");
    if (!ctx->submitted) return set_err(ctx, LTLG_ESTATE, "no grid submitted");
    // label.cpp:193-200, in the reference's order and words
    if (ctx->rows != num_edges)
        return set_err(ctx, LTLG_EINVAL,
                       "label matrix rows " + std::to_string(ctx->rows) + " vs edges " + std::to_string(num_edges));
    if (ctx->props != alphabet_size)
        return set_err(ctx, LTLG_EINVAL,
                       "label matrix props " + std::to_string(ctx->props) + " vs alphabet size " +
                           std::to_string(alphabet_size));
    if (frame < 0 || frame >= ctx->frames) return set_err(ctx, LTLG_EINVAL, "frame out of range");
    if (num_edges && !symbols) return set_err(ctx, LTLG_EINVAL, "null output");
    if (ctx->props == 0) {  // every AlphabetSymbol is empty (label.cpp:205-208)
        if (num_edges) std::memset(symbols, 0, num_edges * 8);
        return sync_all(ctx);
    }
    // props <= 64: one LabelMatrix word per edge == AlphabetSymbol::bits
    return ltlg_get_labels(ctx, frame, symbols);
}

ltlg_status ltlg_edge_counting(ltlg_ctx* ctx, int frame, int prop, uint8_t* hit, uint64_t* examined) {
    DeviceGuard device_guard;
    if (!ctx) return set_err(nullptr, LTLG_EINVAL, "null context");
    if (!ctx->submitted) return set_err(ctx, LTLG_ESTATE, "no grid submitted");
    if (frame < 0 || frame >= ctx->frames) return set_err(ctx, LTLG_EINVAL, "frame out of range");
    if (prop < 0 || prop >= ctx->props) return set_err(ctx, LTLG_EINVAL, "prop out of range");
    const uint64_t nw64 = (ctx->cells + 63) / 64;
    const size_t colw = (static_cast<size_t>(frame) * ctx->props + static_cast<size_t>(prop)) * nw64;
    for (Shard& s : ctx->shards)
        if (!s.P_resident)
            return set_err(ctx, LTLG_ESTATE,
                           "the last submit read its pinned P in place and kept no device copy: resubmit the frame "
                           "from pageable or device memory for edge counting");
    for (Shard& s : ctx->shards) {
        if (s.rows() == 0) continue;
        CK(cudaSetDevice(s.device), "cudaSetDevice");
        CK(s.stage.reserve(s.rows() * 8), "allocate staging");
        CK(s.stage_hit.reserve(s.rows()), "allocate staging");
        CK(launch_edge_count(s.mask_b64.ptr, s.word_b64.ptr, s.tpair_b64.ptr, s.trow_b.ptr, s.ntask_batch, s.perm.ptr,
                             s.Pdev() + colw, s.stage_hit.ptr, s.stage.ptr, s.stream),
           "edge counting kernel");
        if (hit)
            CK(cudaMemcpyAsync(hit + s.row_begin, s.stage_hit.ptr, s.rows(), cudaMemcpyDeviceToHost, s.stream),
               "download");
        if (examined)
            CK(cudaMemcpyAsync(examined + s.row_begin, s.stage.ptr, s.rows() * 8, cudaMemcpyDeviceToHost, s.stream),
               "download");
    }
    return sync_all(ctx);
}

ltlg_status ltlg_get_labels(ltlg_ctx* ctx, int frame, uint64_t* out) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!ctx) return set_err(nullptr, LTLG_EINVAL, "null context");
    if (!ctx->submitted) return set_err(ctx, LTLG_ESTATE, "no grid submitted");
    if (frame < 0 || frame >= ctx->frames) return set_err(ctx, LTLG_EINVAL, "frame out of range");
    if (ctx->props == 0 || ctx->rows == 0) return sync_all(ctx);
    if (!out) return set_err(ctx, LTLG_EINVAL, "null output");
    for (Shard& s : ctx->shards) {
        if (s.rows() == 0) continue;
        CK(cudaSetDevice(s.device), "cudaSetDevice");
        CK(s.stage.reserve(s.rows() * 8), "allocate staging");
        CK(launch_extract(s.labels.ptr, ctx->label_bytes, s.rows(), ctx->frames, frame, s.stage.ptr, s.stream),
           "extract kernel");
        CK(cudaMemcpyAsync(out + s.row_begin, s.stage.ptr, s.rows() * 8, cudaMemcpyDeviceToHost, s.stream),
           "download labels");
    }
    return sync_all(ctx);
}

ltlg_status ltlg_get_labels_packed(ltlg_ctx* ctx, void* out, size_t out_bytes) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!ctx) return set_err(nullptr, LTLG_EINVAL, "null context");
    if (!ctx->submitted) return set_err(ctx, LTLG_ESTATE, "no grid submitted");
    const size_t per_row = static_cast<size_t>(ctx->frames) * static_cast<size_t>(ctx->label_bytes);
    if (ctx->props == 0) return sync_all(ctx);
    if (out_bytes < ctx->rows * per_row) return set_err(ctx, LTLG_EINVAL, "output buffer too small");
    for (Shard& s : ctx->shards) {
        if (s.rows() == 0) continue;
        CK(cudaSetDevice(s.device), "cudaSetDevice");
        uint8_t* dst = static_cast<uint8_t*>(out) + s.row_begin * per_row;
        if (s.blocks_last > 1) {
            // block c goes back on the copy stream as soon as its launch is done,
            // while the later blocks are still being labelled
            for (int c = 0; c < s.blocks_last; ++c) {
                const uint64_t r0 = s.block_row[static_cast<size_t>(c)], r1 = s.block_row[static_cast<size_t>(c) + 1];
                if (r1 == r0) continue;
                CK(cudaStreamWaitEvent(s.copy_stream, s.block_done[static_cast<size_t>(c)], 0), "stream wait");
                CK(cudaMemcpyAsync(dst + r0 * per_row, s.labels.ptr + r0 * per_row, (r1 - r0) * per_row,
                                   cudaMemcpyDeviceToHost, s.copy_stream),
                   "download labels");
            }
        } else {
            CK(cudaMemcpyAsync(dst, s.labels.ptr, s.rows() * per_row, cudaMemcpyDeviceToHost, s.stream),
               "download labels");
        }
    }
    for (Shard& s : ctx->shards) {
        if (s.blocks_last > 1) {
            CK(cudaSetDevice(s.device), "cudaSetDevice");
            CK(cudaStreamSynchronize(s.copy_stream), "download labels");
        }
    }
    return sync_all(ctx);
}

ltlg_status ltlg_device_labels(ltlg_ctx* ctx, int shard, void** dev_ptr, uint64_t* row_begin, uint64_t* row_end,
                               int* device) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!ctx) return set_err(nullptr, LTLG_EINVAL, "null context");
    if (shard < 0 || shard >= static_cast<int>(ctx->shards.size())) return set_err(ctx, LTLG_EINVAL, "shard out of range");
    if (!ctx->submitted) return set_err(ctx, LTLG_ESTATE, "no grid submitted");
    Shard& s = ctx->shards[static_cast<size_t>(shard)];
    if (dev_ptr) *dev_ptr = s.labels.ptr;
    if (row_begin) *row_begin = s.row_begin;
    if (row_end) *row_end = s.row_end;
    if (device) *device = s.device;
    return LTLG_OK;
}

ltlg_status ltlg_get_info(ltlg_ctx* ctx, ltlg_info* out) {
    if (!ctx || !out) return set_err(ctx, LTLG_EINVAL, "null argument");
    std::memset(out, 0, sizeof(*out));
    out->rows = ctx->rows;
    out->cols = ctx->cols;
    out->nnz = ctx->nnz;
    out->words = ctx->words;
    out->pairs = ctx->pairs;
    out->t_bytes = ctx->t_bytes;
    out->n_devices = static_cast<int>(ctx->shards.size());
    out->props = ctx->props;
    out->frames = ctx->frames;
    out->label_bytes = ctx->label_bytes;
    out->label_words = (ctx->props + 63) / 64;
    return LTLG_OK;
}

ltlg_status ltlg_stream(ltlg_ctx* ctx, int shard, void** stream) {
    if (!ctx || !stream) return set_err(ctx, LTLG_EINVAL, "null argument");
    if (shard < 0 || shard >= static_cast<int>(ctx->shards.size())) return set_err(ctx, LTLG_EINVAL, "shard out of range");
    *stream = ctx->shards[static_cast<size_t>(shard)].stream;
    return LTLG_OK;
}

ltlg_status ltlg_set_profiling(ltlg_ctx* ctx, int on) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!ctx) return set_err(nullptr, LTLG_EINVAL, "null context");
    if (on) {
        for (Shard& s : ctx->shards) {
            if (!s.ring.empty()) continue;
            CK(cudaSetDevice(s.device), "cudaSetDevice");
            s.ring.assign(Shard::kRing * Shard::kEv, nullptr);
            for (auto& ev : s.ring) CK(cudaEventCreate(&ev), "event");
        }
    } else {
        for (Shard& s : ctx->shards) s.have_times = false;
    }
    ctx->opts.profile = on ? 1 : 0;
    return LTLG_OK;
}

ltlg_status ltlg_stage_times(ltlg_ctx* ctx, int shard, int back, float* upload_ms, float* summary_ms,
                             float* label_ms) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!ctx) return set_err(nullptr, LTLG_EINVAL, "null context");
    if (shard < 0 || shard >= static_cast<int>(ctx->shards.size())) return set_err(ctx, LTLG_EINVAL, "shard out of range");
    Shard& s = ctx->shards[static_cast<size_t>(shard)];
    if (!ctx->opts.profile || !s.have_times) return set_err(ctx, LTLG_ESTATE, "no profiled submit on this shard");
    if (back < 0 || back >= Shard::kRing || static_cast<uint64_t>(back) >= s.submits)
        return set_err(ctx, LTLG_EINVAL, "profiled submit out of range");
    CK(cudaSetDevice(s.device), "cudaSetDevice");
    cudaEvent_t* q = &s.ring[static_cast<size_t>((s.submits - 1 - static_cast<uint64_t>(back)) % Shard::kRing) * Shard::kEv];
    CK(cudaEventSynchronize(q[4]), "sync");
    float a = 0, b = 0, c = 0;
    CK(cudaEventElapsedTime(&a, q[0], q[1]), "event time");
    CK(cudaEventElapsedTime(&b, q[1], q[2]), "event time");
    CK(cudaEventElapsedTime(&c, q[3], q[4]), "event time");
    if (upload_ms) *upload_ms = a;
    if (summary_ms) *summary_ms = b;
    if (label_ms) *label_ms = c;
    return LTLG_OK;
}

ltlg_status ltlg_validate_csr(uint64_t rows, uint64_t cols, const uint64_t* row_offsets, uint64_t n_offsets,
                              const uint32_t* col_indices, uint64_t nnz, char* err, size_t err_len) {
    Error e{S_OK, ""};
    if (!row_offsets && n_offsets) e = Error{S_EINVAL, "null row_offsets"};
    else if (!col_indices && nnz) e = Error{S_EINVAL, "null col_indices"};
    else validate_csr(rows, cols, row_offsets, n_offsets, col_indices, nnz, &e);
    if (err && err_len) {
        std::strncpy(err, e.msg.c_str(), err_len - 1);
        err[err_len - 1] = '\0';
    }
    if (e.code != S_OK) g_error = e.msg;
    return static_cast<ltlg_status>(e.code);
}

ltlg_status ltlg_label_all(uint64_t rows, uint64_t cols, const uint64_t* row_offsets, const uint32_t* col_indices,
                           uint64_t cells, int num_props, const uint64_t* column_words, int workers, uint64_t* out) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    (void)workers;
    if (num_props > 64) return set_err(nullptr, LTLG_EINVAL, "at most 64 propositions");
    if (num_props < 0) return set_err(nullptr, LTLG_EINVAL, "props must be in [0, 64]");
    if (cols != cells)
        return set_err(nullptr, LTLG_EINVAL,
                       "dimension mismatch: matrix cols " + std::to_string(cols) + " vs proposition rows " +
                           std::to_string(cells));
    ltlg_ctx* ctx = nullptr;
    ltlg_status st = ltlg_create(nullptr, 1, &ctx);
    if (st != LTLG_OK) return st;
    st = ltlg_load_abstraction(ctx, rows, cols, row_offsets, col_indices);
    if (st == LTLG_OK) st = ltlg_submit_grid(ctx, cells, num_props, column_words, 1);
    if (st == LTLG_OK && num_props > 0) st = ltlg_get_labels(ctx, 0, out);
    if (st != LTLG_OK) g_error = ctx->err;
    ltlg_destroy(ctx);
    return st;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Swept-volume matrix: swept_volume_matrix, label.cpp:75-116.
// ---------------------------------------------------------------------------
struct ltlg_csr {
    int device = 0;
    uint64_t rows = 0, cols = 0, nnz = 0;
    DevBuf<uint64_t> off;
    DevBuf<uint32_t> idx;
    double ms = 0;
    ~ltlg_csr() {
        off.release();
        idx.release();
    }
};

namespace {

struct SweepScratch {
    DevBuf<uint64_t> off_in, bsum, stage_off;
    DevBuf<double> samples;
    DevBuf<uint32_t> row_cnt, over, ctr, stage, gkeys;
    DevBuf<unsigned long long> err, gtab;
    ~SweepScratch() {
        off_in.release();
        bsum.release();
        stage_off.release();
        samples.release();
        row_cnt.release();
        over.release();
        ctr.release();
        stage.release();
        gkeys.release();
        err.release();
        gtab.release();
    }
};

// Pass 1 rasterizes every edge once into shared-memory sets and stages the
// sorted rows (bump allocator); the exclusive scan of the row sizes gives
// the offsets and a gather moves the rows into place.  Rows past kSweepCap
// distinct cells take global-memory sets (count, then fill after the scan).
// If the staging buffer runs out, the rows are rasterized again straight
// into place (MODE 1).
ltlg_status sweep_build(const ltlg_gridk* g, const ltlg_footprint* f, uint64_t edges, const uint64_t* sample_off,
                        const double* samples, ltlg_csr* m) {
    using namespace ltlg;
    ltlg_ctx* const ctx = nullptr;  // errors go to the thread's last-error slot
    const uint64_t nsamp = edges ? sample_off[edges] : 0;
    SweepScratch s;
    cudaStream_t st = nullptr;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    std::unique_ptr<CUstream_st, void (*)(cudaStream_t)> hold_st(st, [](cudaStream_t x) { cudaStreamDestroy(x); });
    cudaEvent_t ev[4];
    for (auto& e : ev) CK(cudaEventCreate(&e), "event");
    struct EvFree {
        cudaEvent_t* e;
        ~EvFree() {
            for (int i = 0; i < 4; ++i) cudaEventDestroy(e[i]);
        }
    } ev_free{ev};
    const uint64_t ne = std::max<uint64_t>(edges, 1);
    // staging: ~8 distinct cells per sample covers the driving configurations
    // with room to spare; a shortfall only costs the MODE 1 rerun
    // (test knob LTLG_SWEEP_STAGE: the staging capacity in cells)
    const char* stage_env = getenv("LTLG_SWEEP_STAGE");
    const uint64_t stage_cap = stage_env ? std::strtoull(stage_env, nullptr, 10) : nsamp * 8 + (uint64_t(1) << 20);
    CK(s.off_in.reserve((edges + 1) * 8), "allocate sweep inputs");
    CK(s.samples.reserve(std::max<uint64_t>(nsamp, 1) * 40), "allocate sweep inputs");
    CK(s.row_cnt.reserve(ne * 4), "allocate sweep scratch");
    CK(s.over.reserve(ne * 4), "allocate sweep scratch");
    CK(s.stage_off.reserve(ne * 8), "allocate sweep scratch");
    CK(s.stage.reserve(stage_cap * 4), "allocate sweep scratch");
    CK(s.ctr.reserve(16), "allocate sweep scratch");
    CK(s.err.reserve(24), "allocate sweep scratch");
    CK(s.bsum.reserve(((edges + 1023) / 1024 + 1) * 8), "allocate sweep scratch");
    CK(m->off.reserve((edges + 1) * 8), "allocate CSR");
    CK(cudaMemcpyAsync(s.off_in.ptr, sample_off, (edges + 1) * 8, cudaMemcpyHostToDevice, st), "upload trajectories");
    if (nsamp) CK(cudaMemcpyAsync(s.samples.ptr, samples, nsamp * 40, cudaMemcpyHostToDevice, st), "upload trajectories");
    const unsigned long long err_init[3] = {~0ull, 0ull, 0ull};
    CK(cudaMemcpyAsync(s.err.ptr, err_init, 24, cudaMemcpyHostToDevice, st), "upload");
    CK(cudaMemsetAsync(s.ctr.ptr, 0, 16, st), "memset");

    SweepParams p{};
    for (int a = 0; a < 3; ++a) {
        const int bits = g->depth / 3 + (a < g->depth % 3 ? 1 : 0);
        p.lo[a] = g->lo[a];
        p.hi[a] = g->hi[a];
        p.ncell[a] = int64_t(1) << bits;
        p.cells[a] = static_cast<double>(p.ncell[a]);
        p.w[a] = (g->hi[a] - g->lo[a]) / p.cells[a];  // GridSpec::cell_width
        p.zoff[a] = g->depth % 3 + 2 - a - 3 * (a < g->depth % 3 ? 1 : 0);
    }
    p.length = f->length;
    p.width = f->width;
    p.ref_offset = f->ref_offset;
    p.edges = edges;
    p.sample_off = s.off_in.ptr;
    p.samples = s.samples.ptr;
    p.err_key = s.err.ptr;
    SweepBufs b{};
    b.edge_ctr = s.ctr.ptr;
    b.n_over = s.ctr.ptr + 1;
    b.row_cnt = s.row_cnt.ptr;
    b.over_list = s.over.ptr;
    b.stage = s.stage.ptr;
    b.stage_cap = stage_cap;
    b.bump = s.err.ptr + 2;
    b.stage_off = s.stage_off.ptr;

    // pass 1: rasterize + stage every row
    CK(cudaEventRecord(ev[0], st), "event");
    if (edges) CK(launch_sweep(2, false, p, b, 0, 0, st), "sweep kernel");
    unsigned long long err[3];
    uint32_t nov = 0;
    CK(cudaMemcpyAsync(err, s.err.ptr, 24, cudaMemcpyDeviceToHost, st), "download");
    CK(cudaMemcpyAsync(&nov, b.n_over, 4, cudaMemcpyDeviceToHost, st), "download");
    CK(cudaEventRecord(ev[1], st), "event");
    CK(cudaStreamSynchronize(st), "sweep");
    if (err[0] != ~0ull) {
        static const char* const msg[3] = {"trajectory exits workspace (time axis)", "footprint must be positive",
                                           "trajectory exits workspace (position)"};
        const int kind = static_cast<int>(err[0] & 3);
        return set_err(nullptr, kind == 1 ? LTLG_EINVAL : LTLG_EDOMAIN, msg[kind]);
    }
    const bool staged = err[2] <= stage_cap;
    // rows past kSweepCap distinct cells: global-memory sets, grown until they fit
    CK(cudaEventRecord(ev[2], st), "event");
    uint32_t glog2 = 15;
    int gblocks = 0;
    while (nov) {
        gblocks = static_cast<int>(std::min<uint32_t>(nov, 148));
        CK(s.gtab.reserve((static_cast<size_t>(gblocks) << glog2) * 8), "allocate sweep overflow sets");
        CK(s.gkeys.reserve((static_cast<size_t>(gblocks) << (glog2 - 1)) * 4), "allocate sweep overflow sets");
        b.gtab = s.gtab.ptr;
        b.gkeys = s.gkeys.ptr;
        CK(cudaMemsetAsync(s.err.ptr + 1, 0, 8, st), "memset");
        CK(launch_sweep(0, true, p, b, glog2, gblocks, st), "sweep overflow count kernel");
        CK(cudaMemcpyAsync(err, s.err.ptr, 16, cudaMemcpyDeviceToHost, st), "download");
        CK(cudaStreamSynchronize(st), "sweep overflow count");
        if (!err[1]) break;
        if (glog2 >= 30) return set_err(nullptr, LTLG_ENOMEM, "swept-volume row too large");
        glog2 += 2;
    }
    // row offsets; rows into place
    CK(launch_scan_counts(s.row_cnt.ptr, edges, s.bsum.ptr, m->off.ptr, st), "scan kernel");
    uint64_t nnz = 0;
    CK(cudaMemcpyAsync(&nnz, m->off.ptr + edges, 8, cudaMemcpyDeviceToHost, st), "download");
    CK(cudaStreamSynchronize(st), "scan");
    CK(m->idx.reserve(std::max<uint64_t>(nnz, 1) * 4), "allocate CSR");
    b.row_off = m->off.ptr;
    b.cols = m->idx.ptr;
    if (edges) {
        if (staged) CK(launch_sweep_gather(edges, b, st), "sweep gather kernel");
        else CK(launch_sweep(1, false, p, b, 0, 0, st), "sweep fill kernel");
    }
    if (nov) CK(launch_sweep(1, true, p, b, glog2, gblocks, st), "sweep overflow fill kernel");
    CK(cudaEventRecord(ev[3], st), "event");
    CK(cudaStreamSynchronize(st), "sweep fill");
    float t01 = 0, t23 = 0;
    cudaEventElapsedTime(&t01, ev[0], ev[1]);
    cudaEventElapsedTime(&t23, ev[2], ev[3]);
    m->ms = static_cast<double>(t01) + t23;
    m->rows = edges;
    m->cols = uint64_t(1) << g->depth;
    m->nnz = nnz;
    return LTLG_OK;
}

}  // namespace

extern "C" {

ltlg_status ltlg_swept_volume(const ltlg_gridk* grid, const ltlg_footprint* footprint, uint64_t num_edges,
                              const uint64_t* sample_offsets, const double* samples, int device, ltlg_csr** out) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!out) return set_err(nullptr, LTLG_EINVAL, "null argument");
    *out = nullptr;
    if (!grid || !footprint || (num_edges && !sample_offsets)) return set_err(nullptr, LTLG_EINVAL, "null argument");
    // GridSpec ctor (grid.cpp:18-33), then swept_volume_matrix / sweep_collect
    if (grid->dims < 1) return set_err(nullptr, LTLG_EINVAL, "grid needs at least one axis");
    if (grid->depth < grid->dims || grid->depth > 63)
        return set_err(nullptr, LTLG_EINVAL, "grid depth must be in [k, 63]");
    if (grid->dims > 4) return set_err(nullptr, LTLG_EINVAL, "at most 4 grid axes in this build");
    for (int a = 0; a < grid->dims; ++a)
        if (!(grid->lo[a] < grid->hi[a])) return set_err(nullptr, LTLG_EINVAL, "grid bounds must satisfy lo < hi");
    if (grid->depth > 32) return set_err(nullptr, LTLG_EINVAL, "swept_volume_matrix supports depth <= 32");
    if (num_edges && grid->dims != 3)
        return set_err(nullptr, LTLG_EINVAL, "sweep_voxelize requires a 3-d (x, y, tau) grid");
    if (num_edges > 0xffffffffull) return set_err(nullptr, LTLG_EINVAL, "at most 2^32 - 1 edges in this build");
    for (uint64_t e = 0; e < num_edges; ++e)
        if (sample_offsets[e] > sample_offsets[e + 1])
            return set_err(nullptr, LTLG_EINVAL, "sample_offsets must be nondecreasing");
    if (num_edges && sample_offsets[num_edges] > sample_offsets[0] && !samples)
        return set_err(nullptr, LTLG_EINVAL, "null samples");
    if (num_edges && sample_offsets[0] != 0) return set_err(nullptr, LTLG_EINVAL, "sample_offsets[0] must be 0");
    ltlg_ctx* const ctx = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return set_err(nullptr, LTLG_ECUDA, "no CUDA device");
    if (device < 0 || device >= ndev) return set_err(nullptr, LTLG_EINVAL, "device out of range");
    CK(cudaSetDevice(device), "cudaSetDevice");
    std::unique_ptr<ltlg_csr> m(new (std::nothrow) ltlg_csr);
    if (!m) return set_err(nullptr, LTLG_ENOMEM, "out of host memory");
    m->device = device;
    const ltlg_status st = sweep_build(grid, footprint, num_edges, sample_offsets, samples, m.get());
    if (st != LTLG_OK) return st;
    *out = m.release();
    return LTLG_OK;
}

uint64_t ltlg_csr_rows(const ltlg_csr* m) { return m ? m->rows : 0; }
uint64_t ltlg_csr_cols(const ltlg_csr* m) { return m ? m->cols : 0; }
uint64_t ltlg_csr_nnz(const ltlg_csr* m) { return m ? m->nnz : 0; }
double ltlg_csr_build_ms(const ltlg_csr* m) { return m ? m->ms : 0.0; }

ltlg_status ltlg_csr_copy(const ltlg_csr* m, uint64_t* row_offsets, uint32_t* col_indices) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!m) return set_err(nullptr, LTLG_EINVAL, "null csr");
    ltlg_ctx* const ctx = nullptr;
    CK(cudaSetDevice(m->device), "cudaSetDevice");
    if (row_offsets) CK(cudaMemcpy(row_offsets, m->off.ptr, (m->rows + 1) * 8, cudaMemcpyDeviceToHost), "download CSR");
    if (col_indices && m->nnz)
        CK(cudaMemcpy(col_indices, m->idx.ptr, m->nnz * 4, cudaMemcpyDeviceToHost), "download CSR");
    return LTLG_OK;
}

ltlg_status ltlg_csr_save(const ltlg_csr* m, const char* path) {
    DeviceGuard device_guard;
    if (!m || !path) return set_err(nullptr, LTLG_EINVAL, "null argument");
    std::vector<uint64_t> off(m->rows + 1);
    std::vector<uint32_t> idx(std::max<uint64_t>(m->nnz, 1));
    const ltlg_status st = ltlg_csr_copy(m, off.data(), idx.data());
    if (st != LTLG_OK) return st;
    Error e{S_OK, ""};
    if (!write_csb1(path, m->rows, m->cols, off.data(), idx.data(), &e)) {
        g_error = e.msg;
        return static_cast<ltlg_status>(e.code);
    }
    return LTLG_OK;
}

ltlg_status ltlg_load_csr(ltlg_ctx* ctx, const ltlg_csr* m) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!ctx) return set_err(nullptr, LTLG_EINVAL, "null context");
    if (!m) return set_err(ctx, LTLG_EINVAL, "null csr");
    std::vector<uint64_t> off(m->rows + 1);
    std::vector<uint32_t> idx(std::max<uint64_t>(m->nnz, 1));
    const ltlg_status st = ltlg_csr_copy(m, off.data(), idx.data());
    if (st != LTLG_OK) return st;
    return ltlg_load_abstraction(ctx, m->rows, m->cols, off.data(), idx.data());
}

void ltlg_csr_free(ltlg_csr* m) {
    DeviceGuard device_guard;  // the caller's current device is restored on return
    if (!m) return;
    cudaSetDevice(m->device);
    delete m;
}

}  // extern "C"
