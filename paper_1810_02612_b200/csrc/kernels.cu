// kernels.cu -- sm_100a kernels of the labeling path L = T o P (OR-AND).
//
// Reference semantics (proj/core/src/label.cpp:150-189): L(i,j) = 1 iff some
// stored cell c of row i has P_j[c] = 1.  The reference scans each row once
// per proposition with a random bit probe per cell; here a row is a list of
// (32-bit z-word, mask) pairs and one pair answers every proposition at once:
//
//   hit_j(w, m) = (m & P_j[w]) != 0.
//
// A per-frame summary of P makes that test mostly table-driven:
//   S[w] bit j = P_j[w] != 0           (some cell of the word is set)
//   F[w] bit j = P_j[w] covers the word (every valid cell of the word is set)
// Since every stored mask is non-zero, F[w] props hit unconditionally, props
// outside S[w] never hit, and only the "partial" props S & ~F need the exact
// (m & P_j[w]) probe -- this is exact, not a heuristic.  For the bench
// archetypes (a 90%-occupancy lane complement and 1.5%-occupancy boxes) the
// partial set is empty for most (pair, frame) visits.
//
// Kernels:
//   summary_kernel       P columns -> {S, F} per (word, frame)
//   label_stream_kernel  single frame; lanes own 4 consecutive pairs each, rows
//                        are recovered with a warp-wide segmented OR scan over
//                        head flags (T is streamed once with 2x16-byte
//                        L1::no_allocate loads; HBM-bound)
//   label_batch_kernel   F frames; lanes own frames, pairs are broadcast by
//                        shuffle, each T pair is read from HBM once for all F
//   extract_kernel       one frame of the packed labels -> LabelMatrix u64 words
//   resample_kernel      world-frame grid + pose -> vehicle-frame P columns
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "engine.h"
#include "launch.h"

namespace ltlg {

// Summary entry of one (32-bit word, frame):
//   s, f  : the S / F prop masks above
//   pa, pb: the P words (valid bits only) of the two lowest "partial" props
//           (s & ~f), 0 when absent -- so the exact probe of up to two partial
//           props is branch-free and needs no dependent gather.  Partial
//           props beyond the second fall back to a gather of P (rare).
template <typename LW>
struct alignas(16) SF {
    LW s;
    LW f;
    uint32_t pa;
    uint32_t pb;
};

__device__ __forceinline__ uint4 ld_stream16(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ uint2 ld_stream8(const void* p) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}

template <typename LW>
__device__ __forceinline__ SF<LW> ld_sf(const SF<LW>* p);

template <>
__device__ __forceinline__ SF<uint32_t> ld_sf<uint32_t>(const SF<uint32_t>* p) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    return SF<uint32_t>{v.x, v.y, v.z, v.w};
}

template <>
__device__ __forceinline__ SF<uint64_t> ld_sf<uint64_t>(const SF<uint64_t>* p) {
    const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(p));
    const uint2 w = __ldg(reinterpret_cast<const uint2*>(p) + 2);
    return SF<uint64_t>{v.x, v.y, w.x, w.y};
}

__device__ __forceinline__ int lowest_bit(uint32_t x) { return __ffs(x) - 1; }
__device__ __forceinline__ int lowest_bit(uint64_t x) { return __ffsll(static_cast<long long>(x)) - 1; }

template <typename LW>
__device__ __forceinline__ LW shfl_up(LW v, int d) {
    return __shfl_up_sync(0xffffffffu, v, d);
}
template <typename LW>
__device__ __forceinline__ LW shfl_idx(LW v, int l) {
    return __shfl_sync(0xffffffffu, v, l);
}

// Label contribution of one stored pair (mask m of word w) for one frame.
//   e    : the frame's summary entry of word w
//   skip : props already known to hit (their probes are unnecessary)
//   col0 : the frame's P column 0 (u32 view); column j starts at col0 + j*nw32
template <typename LW>
__device__ __forceinline__ LW pair_hits(uint32_t m, uint32_t w, const SF<LW>& e, LW skip,
                                        const uint32_t* __restrict__ col0, uint32_t nw32) {
    const LW partial = e.s & ~e.f;
    const LW abit = partial & (~partial + 1);
    const LW rest = partial ^ abit;
    const LW bbit = rest & (~rest + 1);
    LW v = e.f;
    v |= (m & e.pa) ? abit : LW(0);
    v |= (m & e.pb) ? bbit : LW(0);
    LW over = (rest ^ bbit) & ~skip;
    while (over) {  // a third partial prop at this word/frame: exact probe
        const int j = lowest_bit(over);
        if (m & __ldg(col0 + static_cast<uint64_t>(j) * nw32 + w)) v |= LW(1) << j;
        over &= over - 1;
    }
    return v;
}

// ---------------------------------------------------------------------------
// Summary build: thread per (word, frame).  P32 = frames x props x nw32 u32.
// Output layout sf[w * frames + f]; entry nw32 of every frame is the all-zero
// sentinel that empty rows point at.
// ---------------------------------------------------------------------------
template <typename LW>
__global__ void __launch_bounds__(256) summary_kernel(const uint32_t* __restrict__ P32, int props, int frames,
                                                      uint32_t nw32, uint64_t cells,
                                                      SF<LW>* __restrict__ sf, LW* __restrict__ s_only,
                                                      uint32_t* __restrict__ task_ctr, uint8_t* __restrict__ split,
                                                      int split_mb) {
    const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
    const int f = blockIdx.y;
    if (w == 0 && f == 0) *task_ctr = 0;  // the labeling kernel that follows pulls tasks from 0
    if (w > nw32) return;
    LW s = 0, full = 0;
    uint32_t pa = 0, pb = 0;
    int np = 0;
    const uint64_t lo = static_cast<uint64_t>(w) * 32;
    if (w < nw32 && lo < cells) {
        const uint32_t valid = (cells - lo >= 32) ? 0xffffffffu : ((1u << (cells - lo)) - 1u);
        const uint32_t* base = P32 + static_cast<uint64_t>(f) * props * nw32 + w;
#pragma unroll 4
        for (int j = 0; j < props; ++j) {
            const uint32_t x = base[static_cast<uint64_t>(j) * nw32] & valid;
            s |= LW(x != 0) << j;
            full |= LW(x == valid) << j;
            if (x != 0 && x != valid) {
                if (np == 0) pa = x;
                else if (np == 1) pb = x;
                ++np;
            }
        }
    }
    sf[static_cast<uint64_t>(w) * frames + f] = SF<LW>{s, full, pa, pb};
    if (s_only) s_only[static_cast<uint64_t>(w) * frames + f] = s;
    if (split) {  // single frame, shared-memory split layout: M[w] then X[w] = {pa, pb}
        if (split_mb == 4) reinterpret_cast<uint32_t*>(split)[w] = static_cast<uint32_t>(s) | (static_cast<uint32_t>(full) << 16);
        else reinterpret_cast<uint2*>(split)[w] = make_uint2(static_cast<uint32_t>(s), static_cast<uint32_t>(full));
        const uint32_t xoff = (static_cast<uint32_t>(split_mb) * (nw32 + 1) + 15u) & ~15u;
        reinterpret_cast<uint2*>(split + xoff)[w] = make_uint2(pa, pb);
    }
}

// ---------------------------------------------------------------------------
// TMA bulk copy + mbarrier helpers (sm_90+ PTX, used on sm_100a)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    // bounded: a bulk copy that can never complete traps instead of hanging the GPU
    for (uint32_t spin = 0;; ++spin) {
        uint32_t done;
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
        if (done) return;
        if (spin > (1u << 22)) __trap();
    }
}

// ---------------------------------------------------------------------------
// Single frame.  Persistent: warps pull tasks (runs of whole rows, pairs
// [p0, p1)) from an atomic counter.  With TAB_SMEM the frame's summary table
// is TMA-bulk-copied once per CTA into shared memory (one CTA of 32 warps per
// SM), so the per-pair gathers hit shared-memory banks instead of L1 tags.
// ---------------------------------------------------------------------------
template <typename LW, typename SW, int TAB, int K>
__global__ void __launch_bounds__(TAB ? 1024 : 256)
    label_stream_kernel(const Pair* __restrict__ pairs, const uint64_t* __restrict__ task_pair,
                        const uint32_t* __restrict__ task_row, uint32_t ntasks, uint32_t* __restrict__ task_ctr,
                        const SF<LW>* __restrict__ sf, uint32_t tab_bytes, const uint32_t* __restrict__ P32,
                        uint32_t nw32, const uint32_t* __restrict__ perm, SW* __restrict__ out) {
    constexpr uint32_t CH = 32 * K;         // pairs per warp chunk
    extern __shared__ __align__(128) uint8_t smem_raw[];
    __shared__ uint64_t tab_bar;
    const int lane = threadIdx.x & 31;
    const SF<LW>* tab = sf;
    constexpr bool TAB_SMEM = TAB != 0;
    constexpr bool SPLIT = TAB == 4 || TAB == 8;
    const uint8_t* xtab = nullptr;  // split mode: {Pa, Pb} table after the M table
    if constexpr (TAB_SMEM) {
        if (threadIdx.x == 0) {
            mbar_init(&tab_bar, 1);
            mbar_expect_tx(&tab_bar, tab_bytes);
            for (uint32_t o = 0; o < tab_bytes; o += 32768u) {
                const uint32_t n = tab_bytes - o < 32768u ? tab_bytes - o : 32768u;
                bulk_g2s(smem_raw + o, reinterpret_cast<const uint8_t*>(sf) + o, n, &tab_bar);
            }
        }
        __syncthreads();
        tab = reinterpret_cast<const SF<LW>*>(smem_raw);
        if constexpr (SPLIT) xtab = smem_raw + ((static_cast<uint32_t>(TAB) * (nw32 + 1) + 15u) & ~15u);
    }
    bool tab_ready = TAB == 0;
    const uint32_t le = 0xffffffffu >> (31 - lane);

    for (;;) {
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(task_ctr, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= ntasks) break;
        const uint64_t p0 = task_pair[t];
        const uint32_t lead = static_cast<uint32_t>(p0 & 3);                        // pairs before p0
        const uint32_t end = lead + static_cast<uint32_t>(task_pair[t + 1] - p0);   // chunk-relative end
        const uint4* base = reinterpret_cast<const uint4*>(pairs + (p0 - lead));     // 32-byte aligned
        const int32_t r0 = static_cast<int32_t>(task_row[t]);
        int32_t open_row = r0 - 1;  // row owning `carry`
        LW carry = 0;

        uint4 cur[K / 2], nxt[K / 2];
#pragma unroll
        for (int h = 0; h < K / 2; ++h) cur[h] = ld_stream16(base + (K / 2) * lane + h);
        if constexpr (TAB_SMEM) {
            if (!tab_ready) {
                mbar_wait(&tab_bar, 0);
                tab_ready = true;
            }
        }
        for (uint32_t c = 0; c < end; c += CH) {
            // software prefetch of the next chunk (the pair array is padded by kPairPad)
            if (c + CH < end) {
#pragma unroll
                for (int h = 0; h < K / 2; ++h) nxt[h] = ld_stream16(base + (c + CH) / 2 + (K / 2) * lane + h);
            }
            const uint32_t q0 = c + K * lane;
            const bool interior = c >= lead && c + CH <= end;  // warp-uniform: every pair valid
            uint32_t heads = 0;  // bit k: pair k opens a row
            LW v[K];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const uint32_t mk = (k & 1) ? cur[k / 2].z : cur[k / 2].x;
                const uint32_t wh = (k & 1) ? cur[k / 2].w : cur[k / 2].y;
                const bool valid = interior || (q0 + k >= lead && q0 + k < end);
                heads |= static_cast<uint32_t>(valid && (wh & kHead)) << k;
                const uint32_t w = valid ? (wh & kWordMask) : nw32;  // invalid -> zero sentinel
                if constexpr (SPLIT) {
                    LW S, F;
                    if constexpr (TAB == 4) {
                        const uint32_t e = reinterpret_cast<const uint32_t*>(smem_raw)[w];
                        S = e & 0xffffu;
                        F = e >> 16;
                    } else {
                        const uint2 e = reinterpret_cast<const uint2*>(smem_raw)[w];
                        S = e.x;
                        F = e.y;
                    }
                    const LW partial = S & ~F;
                    LW vv = F;
                    if (partial) {
                        const uint2 x = reinterpret_cast<const uint2*>(xtab)[w];
                        vv = pair_hits<LW>(mk, w, SF<LW>{S, F, x.x, x.y}, LW(0), P32, nw32);
                    }
                    v[k] = vv;
                } else {
                    SF<LW> e;
                    if constexpr (TAB_SMEM) e = tab[w];
                    else e = ld_sf(tab + w);
                    v[k] = pair_hits<LW>(mk, w, e, LW(0), P32, nw32);
                }
            }
            // rows opened in lower lanes (exclusive prefix of head counts)
            const int nh = __popc(heads);
            int incl = nh;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += y;
            }
            const int hb = incl - nh;
            const int tot = __shfl_sync(0xffffffffu, incl, 31);
            // lane-local segmentation: rows that start and end inside this lane
            LW pre = 0, cur_or = 0;
            int seen = 0;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (heads >> k & 1u) {
                    if (seen) out[perm[open_row + hb + seen]] = static_cast<SW>(cur_or);
                    else pre = cur_or;
                    ++seen;
                    cur_or = 0;
                }
                cur_or |= v[k];
            }
            if (!nh) pre = cur_or;
            // warp-wide segmented inclusive OR scan; a segment starts at the last
            // lane <= this one holding a head (lane 0 otherwise, carrying the open row)
            const uint32_t hmask = __ballot_sync(0xffffffffu, nh > 0) & le;
            const int seg = hmask ? 31 - __clz(hmask) : 0;
            LW x = nh ? cur_or : pre;
            if (lane == 0 && !nh) x |= carry;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const LW y = shfl_up(x, d);
                if (lane - d >= seg) x |= y;
            }
            LW excl = shfl_up(x, 1);
            if (lane == 0) excl = carry;
            if (nh) {
                const int32_t row = open_row + hb;  // the row open before this lane's first head
                if (row >= r0) out[perm[row]] = static_cast<SW>(excl | pre);
            }
            carry = shfl_idx(x, 31);
            open_row += tot;
#pragma unroll
            for (int h = 0; h < K / 2; ++h) cur[h] = nxt[h];
        }
        if (lane == 0 && open_row >= r0) out[perm[open_row]] = static_cast<SW>(carry);
    }
    if constexpr (TAB_SMEM) {
        if (!tab_ready) mbar_wait(&tab_bar, 0);  // never leave with a bulk copy in flight
    }
}

// ---------------------------------------------------------------------------
// F frames.  Persistent warps pull tasks; lane l owns frames l, l+32, ...
// (FPL of them; FULL = every lane owns exactly FPL frames).  Each T pair is
// read from HBM once for all F frames and broadcast by shuffle.
//   sf[w * frames + f]  full summary entry (16 B for <= 32 props)
//   s_only[w * frames + f]  the S mask alone: a pair whose mask covers the
//                       whole word hits exactly the props set somewhere in
//                       the word (warp-uniform fast path, 4 B per lookup)
//   P32 frame f column j at (f*props + j) * nw32
//   out[perm[row] * frames + f] (edge-major)
// ---------------------------------------------------------------------------
template <typename LW, typename SW, int FPL, bool FULL>
__global__ void __launch_bounds__(256)
    label_batch_kernel(const Pair* __restrict__ pairs, const uint64_t* __restrict__ task_pair,
                       const uint32_t* __restrict__ task_row, uint32_t ntasks, uint32_t* __restrict__ task_ctr,
                       const SF<LW>* __restrict__ sf, const LW* __restrict__ s_only,
                       const uint32_t* __restrict__ P32, uint32_t nw32, int props, int frames,
                       const uint32_t* __restrict__ perm, SW* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const uint64_t frame_stride = static_cast<uint64_t>(props) * nw32;
    const SF<LW>* lane_sf = sf + lane;
    const LW* lane_s = s_only + lane;
    const uint32_t* lane_P = P32 + static_cast<uint64_t>(lane) * frame_stride;
    bool fv[FPL];
#pragma unroll
    for (int q = 0; q < FPL; ++q) fv[q] = FULL || lane + 32 * q < frames;

    for (;;) {
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(task_ctr, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= ntasks) break;
        const uint64_t p0 = task_pair[t], p1 = task_pair[t + 1];
        const int64_t r0 = task_row[t];
        int64_t row = r0 - 1;
        LW acc[FPL];
#pragma unroll
        for (int q = 0; q < FPL; ++q) acc[q] = 0;
        auto store = [&](int64_t r) {
            SW* o = out + static_cast<uint64_t>(perm[r]) * frames + lane;
#pragma unroll
            for (int q = 0; q < FPL; ++q)
                if (fv[q]) o[32 * q] = static_cast<SW>(acc[q]);
        };
        uint2 cur = ld_stream8(pairs + p0 + lane);
        for (uint64_t c = p0; c < p1; c += 32) {
            uint2 nxt = cur;
            if (c + 32 < p1) nxt = ld_stream8(pairs + c + 32 + lane);
            const int n = static_cast<int>(p1 - c < 32 ? p1 - c : 32);
            for (int i = 0; i < n; ++i) {
                const uint32_t m = __shfl_sync(0xffffffffu, cur.x, i);
                const uint32_t wh = __shfl_sync(0xffffffffu, cur.y, i);
                if (wh & kHead) {  // warp-uniform
                    if (row >= r0) store(row);
                    ++row;
#pragma unroll
                    for (int q = 0; q < FPL; ++q) acc[q] = 0;
                }
                const uint32_t w = wh & kWordMask;
                const uint32_t off = w * static_cast<uint32_t>(frames);
                if (m == 0xffffffffu) {  // warp-uniform: the whole word is swept
#pragma unroll
                    for (int q = 0; q < FPL; ++q)
                        if (fv[q]) acc[q] |= __ldg(lane_s + off + 32 * q);
                } else {
#pragma unroll
                    for (int q = 0; q < FPL; ++q)
                        if (fv[q]) {
                            const SF<LW> x = ld_sf(lane_sf + off + 32 * q);
                            acc[q] |= pair_hits<LW>(m, w, x, acc[q], lane_P + 32 * q * frame_stride, nw32);
                        }
                }
            }
            cur = nxt;
        }
        if (row >= r0) store(row);
    }
}

// One frame of packed edge-major labels -> LabelMatrix u64 words.
template <typename SW>
__global__ void extract_kernel(const SW* __restrict__ labels, uint64_t rows, int frames, int frame,
                               uint64_t* __restrict__ out) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i < rows) out[i] = static_cast<uint64_t>(labels[i * frames + frame]);
}

// ---------------------------------------------------------------------------
// World -> vehicle resample (north_star subsystem 2).  Thread per (vehicle
// 32-bit word, group of 8 props, frame).  fp64 with explicit round-to-nearest
// intrinsics in the order of oracle_resample (built with -ffp-contract=off),
// so results are bit-identical to the CPU restatement.
// ---------------------------------------------------------------------------
struct Grid2 {
    int depth;
    double lo0, hi0, lo1, hi1;
};
struct Pose2 {
    double dx, dy, c, s;
};

__device__ __forceinline__ int axis_bits2(int depth, int axis) { return depth / 2 + (axis < depth % 2 ? 1 : 0); }

__device__ __forceinline__ int64_t quantize_dev(double lo, double hi, int bits, double x) {
    if (!(x >= lo && x < hi)) return -1;
    const double z = __ddiv_rn(__dadd_rn(x, -lo), __dadd_rn(hi, -lo));
    const double scaled = floor(__dmul_rn(z, static_cast<double>(1ull << bits)));
    uint64_t c = static_cast<uint64_t>(scaled);
    if (c >= (1ull << bits)) c = (1ull << bits) - 1;
    return static_cast<int64_t>(c);
}

__global__ void resample_kernel(Grid2 vg, Grid2 wg, const Pose2* __restrict__ poses, int props,
                                const uint32_t* __restrict__ world32, uint32_t wnw32, int outside,
                                uint32_t vnw32, uint32_t* __restrict__ out32) {
    const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
    const int g0 = blockIdx.y * 8;
    const int f = blockIdx.z;
    if (w >= vnw32) return;
    const Pose2 ps = poses[f];
    const int bvx = axis_bits2(vg.depth, 0), bvy = axis_bits2(vg.depth, 1);
    const int bwx = axis_bits2(wg.depth, 0), bwy = axis_bits2(wg.depth, 1);
    const uint64_t vcells = 1ull << vg.depth;
    const double wxv = __ddiv_rn(__dadd_rn(vg.hi0, -vg.lo0), static_cast<double>(1ull << bvx));
    const double wyv = __ddiv_rn(__dadd_rn(vg.hi1, -vg.lo1), static_cast<double>(1ull << bvy));
    uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int ng = props - g0 < 8 ? props - g0 : 8;
    for (int b = 0; b < 32; ++b) {
        const uint64_t z = static_cast<uint64_t>(w) * 32 + b;
        if (z >= vcells) break;
        uint64_t cx = 0, cy = 0;
        for (int level = 0; level < vg.depth; ++level) {
            const uint64_t bit = (z >> (vg.depth - 1 - level)) & 1u;
            if ((level & 1) == 0) cx = (cx << 1) | bit;
            else cy = (cy << 1) | bit;
        }
        const double x = __dadd_rn(vg.lo0, __dmul_rn(__dadd_rn(static_cast<double>(cx), 0.5), wxv));
        const double y = __dadd_rn(vg.lo1, __dmul_rn(__dadd_rn(static_cast<double>(cy), 0.5), wyv));
        const double xw = __dadd_rn(__dadd_rn(__dmul_rn(ps.c, x), -__dmul_rn(ps.s, y)), ps.dx);
        const double yw = __dadd_rn(__dadd_rn(__dmul_rn(ps.s, x), __dmul_rn(ps.c, y)), ps.dy);
        const int64_t qx = quantize_dev(wg.lo0, wg.hi0, bwx, xw);
        const int64_t qy = quantize_dev(wg.lo1, wg.hi1, bwy, yw);
        if (qx < 0 || qy < 0) {
            if (outside)
                for (int j = 0; j < ng; ++j) acc[j] |= 1u << b;
            continue;
        }
        uint64_t zw = 0;
        for (int level = 0; level < wg.depth; ++level) {
            const int axis = level & 1;
            const int bit_pos = (axis ? bwy : bwx) - 1 - level / 2;
            zw = (zw << 1) | (((axis ? static_cast<uint64_t>(qy) : static_cast<uint64_t>(qx)) >> bit_pos) & 1u);
        }
        for (int j = 0; j < ng; ++j) {
            const uint32_t word = __ldg(world32 + static_cast<uint64_t>(g0 + j) * wnw32 + (zw >> 5));
            acc[j] |= ((word >> (zw & 31)) & 1u) << b;
        }
    }
    uint32_t* dst = out32 + static_cast<uint64_t>(f) * props * vnw32 + w;
    for (int j = 0; j < ng; ++j) dst[static_cast<uint64_t>(g0 + j) * vnw32] = acc[j];
}

// ---------------------------------------------------------------------------
// Host launchers
// ---------------------------------------------------------------------------

// Single-frame shared-memory "split" table: M[w] (S|F<<16 in 4 B for <= 16
// props, {S, F} in 8 B for <= 32) followed by X[w] = {pa, pb}; the wider M
// halves the bank-conflict wavefronts of the per-pair gathers and X is only
// read by lanes whose word has a partial prop.
int split_entry_bytes(int props) { return props <= 16 ? 4 : props <= 32 ? 8 : 0; }
size_t split_table_bytes(int props, uint32_t nw32) {
    const int mb = split_entry_bytes(props);
    if (!mb) return 0;
    // both parts 16-byte aligned: the whole table is one set of TMA bulk copies
    return ((static_cast<size_t>(mb) * (nw32 + 1) + 15u) & ~size_t(15)) + ((8u * (nw32 + 1) + 15u) & ~size_t(15));
}

cudaError_t launch_summary(const uint32_t* P32, int props, int frames, uint32_t nw32, uint64_t cells,
                           void* sf, void* s_only, uint32_t* task_ctr, void* split, cudaStream_t st) {
    dim3 grid((nw32 + 1 + 255) / 256, static_cast<unsigned>(frames));
    const int mb = split_entry_bytes(props);
    if (props <= 32)
        summary_kernel<uint32_t><<<grid, 256, 0, st>>>(P32, props, frames, nw32, cells,
                                                       static_cast<SF<uint32_t>*>(sf),
                                                       static_cast<uint32_t*>(s_only), task_ctr,
                                                       static_cast<uint8_t*>(split), mb);
    else
        summary_kernel<uint64_t><<<grid, 256, 0, st>>>(P32, props, frames, nw32, cells,
                                                       static_cast<SF<uint64_t>*>(sf),
                                                       static_cast<uint64_t*>(s_only), task_ctr, nullptr, 0);
    return cudaGetLastError();
}

size_t summary_entry_bytes(int props) { return props <= 32 ? sizeof(SF<uint32_t>) : sizeof(SF<uint64_t>); }

static int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

constexpr uint32_t kMaxSmemTable = 200u * 1024u;

// Dev knobs (A/B sweeps on the GPU box): LTLG_STREAM_TABLE=smem|global, LTLG_STREAM_K=4|8
static int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v && *v ? atoi(v) : dflt;
}

template <typename LW, typename SW, int TAB, int K>
static cudaError_t launch_stream_v(const LaunchArgs& a, uint32_t tab_bytes, const void* tab_src, cudaStream_t st) {
    const auto* tab = static_cast<const SF<LW>*>(tab_src);
    if constexpr (TAB != 0) {
        static uint64_t attr_set = 0;  // per device
        int dev = 0;
        cudaGetDevice(&dev);
        if (!(attr_set >> dev & 1u)) {
            cudaFuncSetAttribute(label_stream_kernel<LW, SW, TAB, K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kMaxSmemTable));
            attr_set |= 1ull << dev;
        }
        if (tab_bytes % 16u) return cudaErrorInvalidValue;  // never launch an uncompletable TMA copy
        label_stream_kernel<LW, SW, TAB, K><<<sm_count(), 1024, tab_bytes, st>>>(
            a.pairs, a.task_pair, a.task_row, a.ntasks, a.task_ctr, tab, tab_bytes, a.P32, a.nw32, a.perm,
            static_cast<SW*>(a.out));
    } else {
        static int per_sm = 0;
        if (!per_sm) {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, label_stream_kernel<LW, SW, 0, K>, 256, 0);
            if (per_sm <= 0) per_sm = 4;
        }
        label_stream_kernel<LW, SW, 0, K><<<sm_count() * per_sm, 256, 0, st>>>(
            a.pairs, a.task_pair, a.task_row, a.ntasks, a.task_ctr, tab, tab_bytes, a.P32, a.nw32, a.perm,
            static_cast<SW*>(a.out));
    }
    return cudaSuccess;
}

// Which single-frame table layout a submit uses (the summary kernel must
// write the split layout when this returns a split mode).
int stream_table_mode(int props, uint32_t nw32) {
    static const int want = env_int("LTLG_STREAM_TABLE", -1);  // dev knob: 0 global, 1 smem, 2 split
    const size_t comb = static_cast<size_t>(nw32 + 1) * summary_entry_bytes(props);
    const size_t split = split_table_bytes(props, nw32);
    if (want == 0) return 0;
    if (want == 1) return comb <= kMaxSmemTable ? 1 : 0;
    if (split && split <= kMaxSmemTable) return split_entry_bytes(props);
    return comb <= kMaxSmemTable ? 1 : 0;
}

template <typename LW, typename SW>
static cudaError_t launch_stream_t(const LaunchArgs& a, cudaStream_t st) {
    static const int k = env_int("LTLG_STREAM_K", 8);
    const int mode = stream_table_mode(a.props, a.nw32);
    const uint32_t comb = (a.nw32 + 1) * static_cast<uint32_t>(sizeof(SF<LW>));
    if (mode == 0) {
        if (k == 8) return launch_stream_v<LW, SW, 0, 8>(a, comb, a.sf, st);
        else return launch_stream_v<LW, SW, 0, 4>(a, comb, a.sf, st);
    } else if (mode == 1) {
        if (k == 8) return launch_stream_v<LW, SW, 1, 8>(a, comb, a.sf, st);
        else return launch_stream_v<LW, SW, 1, 4>(a, comb, a.sf, st);
    } else if constexpr (sizeof(LW) == 4) {
        const uint32_t sb = static_cast<uint32_t>(split_table_bytes(a.props, a.nw32));
        if (mode == 4) {
            if (k == 8) return launch_stream_v<LW, SW, 4, 8>(a, sb, a.split, st);
            else return launch_stream_v<LW, SW, 4, 4>(a, sb, a.split, st);
        } else {
            if (k == 8) return launch_stream_v<LW, SW, 8, 8>(a, sb, a.split, st);
            else return launch_stream_v<LW, SW, 8, 4>(a, sb, a.split, st);
        }
    }
    return cudaErrorInvalidValue;
}

template <typename LW, typename SW, int FPL, bool FULL>
static void launch_batch_t(const LaunchArgs& a, cudaStream_t st) {
    static int per_sm = 0;
    if (!per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, label_batch_kernel<LW, SW, FPL, FULL>, 256, 0);
        if (per_sm <= 0) per_sm = 4;
    }
    label_batch_kernel<LW, SW, FPL, FULL><<<sm_count() * per_sm, 256, 0, st>>>(
        a.pairs, a.task_pair, a.task_row, a.ntasks, a.task_ctr, static_cast<const SF<LW>*>(a.sf),
        static_cast<const LW*>(a.s_only), a.P32, a.nw32, a.props, a.frames, a.perm, static_cast<SW*>(a.out));
}

template <typename LW, typename SW>
static void launch_batch_fpl(const LaunchArgs& a, cudaStream_t st) {
    if (a.frames == 32) launch_batch_t<LW, SW, 1, true>(a, st);
    else if (a.frames == 64) launch_batch_t<LW, SW, 2, true>(a, st);
    else if (a.frames == 128) launch_batch_t<LW, SW, 4, true>(a, st);
    else if (a.frames < 32) launch_batch_t<LW, SW, 1, false>(a, st);
    else if (a.frames < 64) launch_batch_t<LW, SW, 2, false>(a, st);
    else if (a.frames < 128) launch_batch_t<LW, SW, 4, false>(a, st);
    else launch_batch_t<LW, SW, 8, false>(a, st);
}

cudaError_t launch_label(const LaunchArgs& a, cudaStream_t st) {
    if (a.ntasks == 0) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    if (a.frames == 1) {
        switch (a.label_bytes) {
            case 1: e = launch_stream_t<uint32_t, uint8_t>(a, st); break;
            case 2: e = launch_stream_t<uint32_t, uint16_t>(a, st); break;
            case 4: e = launch_stream_t<uint32_t, uint32_t>(a, st); break;
            default: e = launch_stream_t<uint64_t, uint64_t>(a, st); break;
        }
    } else {
        switch (a.label_bytes) {
            case 1: launch_batch_fpl<uint32_t, uint8_t>(a, st); break;
            case 2: launch_batch_fpl<uint32_t, uint16_t>(a, st); break;
            case 4: launch_batch_fpl<uint32_t, uint32_t>(a, st); break;
            default: launch_batch_fpl<uint64_t, uint64_t>(a, st); break;
        }
    }
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_extract(const void* labels, int label_bytes, uint64_t rows, int frames, int frame,
                           uint64_t* out, cudaStream_t st) {
    if (rows == 0) return cudaSuccess;
    const unsigned blocks = static_cast<unsigned>((rows + 255) / 256);
    switch (label_bytes) {
        case 1: extract_kernel<<<blocks, 256, 0, st>>>(static_cast<const uint8_t*>(labels), rows, frames, frame, out); break;
        case 2: extract_kernel<<<blocks, 256, 0, st>>>(static_cast<const uint16_t*>(labels), rows, frames, frame, out); break;
        case 4: extract_kernel<<<blocks, 256, 0, st>>>(static_cast<const uint32_t*>(labels), rows, frames, frame, out); break;
        default: extract_kernel<<<blocks, 256, 0, st>>>(static_cast<const uint64_t*>(labels), rows, frames, frame, out); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_resample(int vdepth, double vlo0, double vhi0, double vlo1, double vhi1, int wdepth,
                            double wlo0, double whi0, double wlo1, double whi1, const void* poses,
                            int frames, int props, const uint32_t* world32, uint32_t wnw32, int outside,
                            uint32_t vnw32, uint32_t* out32, cudaStream_t st) {
    if (props == 0) return cudaSuccess;
    Grid2 vg{vdepth, vlo0, vhi0, vlo1, vhi1};
    Grid2 wg{wdepth, wlo0, whi0, wlo1, whi1};
    dim3 grid((vnw32 + 127) / 128, static_cast<unsigned>((props + 7) / 8), static_cast<unsigned>(frames));
    resample_kernel<<<grid, 128, 0, st>>>(vg, wg, static_cast<const Pose2*>(poses), props, world32, wnw32,
                                          outside, vnw32, out32);
    return cudaGetLastError();
}

}  // namespace ltlg
