// kernels.cu -- sm_100a kernels of the labeling path L = T o P (OR-AND).
//
// Reference semantics (proj/core/src/label.cpp:150-189): L(i,j) = 1 iff some
// stored cell c of row i has P_j[c] = 1.  The reference scans each row once
// per proposition with a random bit probe per cell; here a row is a list of
// (32-bit z-word, mask) pairs and one pair answers every proposition at once:
//
//   hit_j(w, m) = (m & P_j[w]) != 0.
//
// A per-frame summary of P makes that test table-driven:
//   S[w] bit j = P_j[w] != 0           (some cell of the word is set)
//   F[w] bit j = P_j[w] covers the word (every valid cell of the word is set)
// Since every stored mask is non-zero, F[w] props hit unconditionally, props
// outside S[w] never hit, and only the "partial" props S & ~F need the exact
// (m & P_j[w]) probe -- this is exact, not a heuristic.
//
// Summary entry of one (word, frame), 16 bytes, branch-free to evaluate:
//   FMT 16 (props <= 16): {F | over<<31, Pa, Pb, Abit | Bbit<<16}
//   FMT 32 (props <= 32): {F,            Pa, Pb, ia | ib<<8 | over<<16}
//   (Pa, Pb = P words of the two lowest partial props a < b, 0 when absent;
//    Abit/Bbit = their prop bits, ia/ib their indices; over = a third
//    partial prop exists -> exact gather of P, rare)
//   FMT 64 (props <= 64): SF<u64> {S, F, Pa, Pb} (32 bytes, pair_hits).
// Evaluating an entry for mask m:  v = F | (m&Pa ? A : 0) | (m&Pb ? B : 0).
// FMT 16 leaves flag/Bbit garbage in bits 16..31 of v; labels of <= 16 props
// are stored as u8/u16, so the store truncates it away.
// The S masks are also written on their own (s_only): the over path needs S,
// and the multi-frame kernel uses it for full-mask pairs (hits == S).
//
// Kernels:
//   summary_kernel       P columns -> entries + S per (word, frame)
//   label_stream_kernel  single frame; lanes own K consecutive pairs each, rows
//                        are recovered with a warp-wide segmented OR scan over
//                        head flags (T is streamed once with coalesced 16-byte
//                        L1::no_allocate loads from its own row-order copy;
//                        HBM-bound)
//   label_batch_kernel   F frames; lanes own frames, pairs are broadcast by
//                        shuffle, each T pair is read from HBM once for all F
//   extract_kernel       one frame of the packed labels -> LabelMatrix u64 words
//   resample_kernel      world-frame grid + pose -> vehicle-frame P columns
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <vector>

#include "engine.h"
#include "launch.h"

namespace ltlg {

template <typename LW>
struct alignas(16) SF {
    LW s;
    LW f;
    uint32_t pa;
    uint32_t pb;
};

template <int FMT>
struct Fmt {
    using LW = uint32_t;
    using E = uint4;
};
template <>
struct Fmt<64> {
    using LW = uint64_t;
    using E = SF<uint64_t>;
};

// LTLG_AB_BUILD=1 (libltlgrid_gpu_ab.so, tests and dev tools only): also the
// A/B variants the dispatch reaches only through dev knobs -- the 32-cell
// single-frame kernels, the pair-major prop-lane kernel, the tcgen05 kind::i8
// formulation.  The product library leaves them out.
#ifndef LTLG_AB_BUILD
#define LTLG_AB_BUILD 0
#endif
constexpr uint32_t kOver16 = 0x80000000u;
constexpr uint32_t kOver32 = 0x10000u;

int entry_format(int props) { return props <= 16 ? 16 : props <= 32 ? 32 : 64; }
size_t summary_entry_bytes(int props) { return props <= 32 ? sizeof(uint4) : sizeof(SF<uint64_t>); }
size_t s_only_bytes(int props) { return props <= 32 ? 4 : 8; }

// Single-frame split table (FMT 16/32): M[w] (4 B: (16+ia) | (16+ib)<<5 |
// partial<<10 | over<<11 | F<<16 for <= 16 props -- the labels accumulate in
// the high half and are shifted down once per stored row; 8 B: {F, ia |
// ib<<8 | partial<<16 | over<<17} for <= 32) followed, 16-byte aligned, by
// X[w] = {Pa, Pb}.  Every
// pair reads M; only lanes whose word has a partial prop read X, so the
// random shared-memory gathers cost ~1.5 wavefronts per pair instead of the
// ~11 of a 16-byte entry.
__host__ __device__ __forceinline__ uint32_t split_x_offset(int fmt, uint32_t nw32) {
    return ((fmt == 16 ? 4u : 8u) * (nw32 + 1) + 15u) & ~15u;
}
// 64-cell-word split table: M[w64] as above (FMT 64: 16 B {F lo, F hi,
// ia | ib<<8 | partial<<16 | over<<17, 0}), then (16-byte aligned) X[w64] =
// {Pa lo, Pa hi, Pb lo, Pb hi}.
// FMT 64 (33..64 props, u64 labels) keeps M as two arrays, F[w] (u64) then
// meta[w] (u32: ia | ib<<6 | ic<<12 | id<<18 | partial<<24 | over<<25), and
// X[w] = the P words of the four lowest partial props (32 B): with 64
// props a 64-cell word has >= 3 partial props 1.7% of the time at 1024^2,
// >= 5 only 0.02%.  12 B of M per word fit 1024^2 (196 KB) in shared memory.
__host__ __device__ __forceinline__ uint32_t split64_m_bytes(int fmt) { return fmt == 16 ? 4u : fmt == 32 ? 8u : 12u; }
__host__ __device__ __forceinline__ uint32_t split64_x_offset(int fmt, uint32_t nw64) {
    return (split64_m_bytes(fmt) * (nw64 + 1) + 15u) & ~15u;
}
__host__ __device__ __forceinline__ uint32_t split64_meta_offset(uint32_t nw64) { return 8u * (nw64 + 1); }
__host__ __device__ __forceinline__ uint32_t split64_x_bytes(int fmt) { return fmt == 64 ? 32u : 16u; }
size_t split64_table_bytes(int props, uint32_t nw64) {
    const int fmt = entry_format(props);
    return split64_x_offset(fmt, nw64) + split64_x_bytes(fmt) * (nw64 + 1);
}
size_t split_table_bytes(int props, uint32_t nw32) {
    const int fmt = entry_format(props);
    if (fmt == 64) return 0;
    return split_x_offset(fmt, nw32) + ((8u * (nw32 + 1) + 15u) & ~15u);
}

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

__device__ __forceinline__ uint4 ld_entry(const uint4* p) { return __ldg(p); }

// base + idx elements as one IMAD.WIDE (FMA pipe) instead of 64-bit ALU adds
template <typename T>
__device__ __forceinline__ const T* index_wide(const T* base, uint32_t idx) {
    uint64_t r;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(idx), "n"(static_cast<int>(sizeof(T))), "l"(base));
    return reinterpret_cast<const T*>(r);
}
__device__ __forceinline__ SF<uint64_t> ld_entry(const SF<uint64_t>* p) {
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

// Exact probe of the props in `over` (bit j = prop j) for mask m of word w:
// gather P_j[w].  col0 = the frame's P column 0 (u32 view).
template <typename LW>
__device__ __forceinline__ LW probe_gather(uint32_t m, uint32_t w, LW over, const uint32_t* __restrict__ col0,
                                        uint32_t nw32) {
    LW v = 0;
    while (over) {
        const int j = lowest_bit(over);
        if (m & __ldg(col0 + static_cast<uint64_t>(j) * nw32 + w)) v |= LW(1) << j;
        over &= over - 1;
    }
    return v;
}

// Out-of-line copy for the multi-frame kernel's inner loop: inlining the
// rare gather loop there costs more (code size, scheduling) than the call.
template <typename LW>
__device__ __noinline__ LW probe_gather_call(uint32_t m, uint32_t w, LW over, const uint32_t* __restrict__ col0,
                                             uint32_t nw32) {
    return probe_gather<LW>(m, w, over, col0, nw32);
}

// Label contribution of one stored pair (mask m of word w) for one frame.
//   e    : the frame's summary entry of word w
//   sp   : base + index of the frame's S mask of word w (read only on the
//          rare over path, so its address is formed there)
//   skip : props already known to hit (their probes are unnecessary)
template <int FMT>
__device__ __forceinline__ typename Fmt<FMT>::LW probe(const typename Fmt<FMT>::E& e, uint32_t m, uint32_t w,
                                                       const typename Fmt<FMT>::LW* s_base, uint32_t s_idx,
                                                       typename Fmt<FMT>::LW skip,
                                                       const uint32_t* __restrict__ col0, uint32_t nw32) {
    if constexpr (FMT == 16) {
        uint32_t v = e.x;
        if (m & e.y) v |= e.w;
        if (m & e.z) v |= e.w >> 16;
        if (e.x & kOver16) {
            const uint32_t known = (e.x | e.w | (e.w >> 16)) & 0xffffu;
            v |= probe_gather_call<uint32_t>(m, w, __ldg(s_base + s_idx) & ~known & ~skip, col0, nw32);
        }
        return v;
    } else if constexpr (FMT == 32) {
        const uint32_t abit = __funnelshift_l(0u, 1u, e.w);
        const uint32_t bbit = __funnelshift_l(0u, 1u, e.w >> 8);
        uint32_t v = e.x;
        if (m & e.y) v |= abit;
        if (m & e.z) v |= bbit;
        if (e.w & kOver32)
            v |= probe_gather_call<uint32_t>(m, w, __ldg(s_base + s_idx) & ~(e.x | abit | bbit | skip), col0, nw32);
        return v;
    } else {
        (void)s_base;
        (void)s_idx;
        const uint64_t partial = e.s & ~e.f;
        const uint64_t abit = partial & (~partial + 1);
        const uint64_t rest = partial ^ abit;
        const uint64_t bbit = rest & (~rest + 1);
        uint64_t v = e.f;
        if (m & e.pa) v |= abit;
        if (m & e.pb) v |= bbit;
        const uint64_t over = (rest ^ bbit) & ~skip;
        if (over) v |= probe_gather_call<uint64_t>(m, w, over, col0, nw32);
        return v;
    }
}

// ---------------------------------------------------------------------------
// Summary build: thread per (word, frame).  P32 = frames x props x nw32 u32.
// Output index w * frames + f; entry nw32 of every frame is the all-zero
// sentinel that empty rows and neutralised pairs point at.
// ---------------------------------------------------------------------------
template <int FMT, bool SPLIT>
__global__ void __launch_bounds__(256) summary_kernel(const uint32_t* __restrict__ P32, int props, int frames,
                                                      uint32_t nw32, uint64_t cells, void* __restrict__ tab,
                                                      void* __restrict__ s_only, uint32_t* __restrict__ task_ctr,
                                                      int nctr) {
    using LW = typename Fmt<FMT>::LW;
    const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
    const int f = blockIdx.y;
    if (f == 0 && w < static_cast<uint32_t>(nctr)) task_ctr[w] = 0;  // the labeling launches that follow pull from 0
    if (w > nw32) return;
    LW s = 0, full = 0;
    uint32_t pa = 0, pb = 0, ia = 0, ib = 0;
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
                if (np == 0) {
                    pa = x;
                    ia = static_cast<uint32_t>(j);
                } else if (np == 1) {
                    pb = x;
                    ib = static_cast<uint32_t>(j);
                }
                ++np;
            }
        }
    }
    const uint64_t idx = static_cast<uint64_t>(w) * frames + f;
    const uint32_t over = np > 2 ? 1u : 0u;
    if constexpr (SPLIT) {  // single frame: the stream kernel's M / X tables (see split_table_bytes)
        static_assert(FMT != 64, "split tables hold <= 32 props");
        const uint32_t part = np > 0 ? 1u : 0u;
        uint8_t* base = static_cast<uint8_t*>(tab);
        if constexpr (FMT == 16)  // F in the high half: the probe bits are 1 << (16 + ia) straight from M
            reinterpret_cast<uint32_t*>(base)[w] =
                (static_cast<uint32_t>(full) << 16) | (16u + ia) | ((16u + ib) << 5) | (part << 10) | (over << 11);
        else
            reinterpret_cast<uint2*>(base)[w] =
                make_uint2(static_cast<uint32_t>(full), ia | (ib << 8) | (part << 16) | (over << 17));
        reinterpret_cast<uint2*>(base + split_x_offset(FMT, nw32))[w] = make_uint2(pa, pb);
    } else if constexpr (FMT == 16) {
        const uint32_t ab = (np > 0 ? 1u << ia : 0u) | (np > 1 ? (1u << ib) << 16 : 0u);
        static_cast<uint4*>(tab)[idx] = make_uint4(static_cast<uint32_t>(full) | (over << 31), pa, pb, ab);
    } else if constexpr (FMT == 32) {
        static_cast<uint4*>(tab)[idx] = make_uint4(static_cast<uint32_t>(full), pa, pb, ia | (ib << 8) | (over << 16));
    } else {
        static_cast<SF<uint64_t>*>(tab)[idx] = SF<uint64_t>{s, full, pa, pb};
    }
    static_cast<LW*>(s_only)[idx] = s;
}

// Single-frame summary over 64-cell words (P's own u64 column words): the
// split table of split64_x_offset + S per word.  Thread per word.
// P may be host memory read through the mapping: a plain global load (the
// read-only path is only a hint, but keep mapped reads on the ordinary path)
__device__ __forceinline__ uint64_t ld_nc_u64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

template <int FMT>
__global__ void __launch_bounds__(256) summary64_kernel(const uint64_t* __restrict__ P64, int props, uint32_t nw64,
                                                        uint64_t cells, uint8_t* __restrict__ tab,
                                                        void* __restrict__ s_only_g, uint32_t* __restrict__ task_ctr,
                                                        int nctr, uint64_t* __restrict__ P_copy,
                                                        const uint32_t* __restrict__ touched64) {
    // CTA = 32 consecutive words x 8 warps: warp g reads props g, g+8, ...
    // (coalesced 256-B rows of P), lane = word; the eight partial masks meet
    // in shared memory and warp 0 assembles the entries (first <= 2 / 4
    // partial props in prop order, as before)
    using LW = typename Fmt<FMT>::LW;
    // let a programmatically dependent labeling launch get its CTAs resident;
    // it waits for this grid's completion before touching our outputs
    asm volatile("griddepcontrol.launch_dependents;");
    __shared__ uint64_t s_pv[64][32];              // P value of (prop, word) when partial
    __shared__ uint64_t s_any[8][32], s_full[8][32], s_part[8][32];
    const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < static_cast<uint32_t>(nctr)) task_ctr[t] = 0;  // the labeling launches that follow pull from 0
    const uint32_t w = blockIdx.x * 32 + lane;
    uint64_t any = 0, full = 0, part = 0;
    const uint64_t lo = static_cast<uint64_t>(w) * 64;
    // words no pair of the shard is on are never looked up: no read of P
    // (over PCIe when P comes through the host mapping), a zero entry
    if (w < nw64 && lo < cells && !(touched64 && !(__ldg(touched64 + (w >> 5)) >> (w & 31) & 1u))) {
        const uint64_t valid = (cells - lo >= 64) ? ~0ull : ((1ull << (cells - lo)) - 1ull);
        uint64_t x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // all loads in flight before any use
            const int j = g + 8 * k;
            x[k] = j < props ? ld_nc_u64(P64 + static_cast<uint64_t>(j) * nw64 + w) : 0;
        }
        if (P_copy) {  // P arrived through the host mapping: keep the device copy
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (g + 8 * k < props) P_copy[static_cast<uint64_t>(g + 8 * k) * nw64 + w] = x[k];
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] &= valid;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int j = g + 8 * k;
            any |= static_cast<uint64_t>(x[k] != 0) << j;
            full |= static_cast<uint64_t>(j < props && x[k] == valid) << j;
            if (x[k] != 0 && x[k] != valid) {
                part |= 1ull << j;
                s_pv[j][lane] = x[k];
            }
        }
    }
    s_any[g][lane] = any;
    s_full[g][lane] = full;
    s_part[g][lane] = part;
    __syncthreads();
    if (g != 0 || w > nw64) return;
#pragma unroll
    for (int k = 1; k < 8; ++k) {
        any |= s_any[k][lane];
        full |= s_full[k][lane];
        part |= s_part[k][lane];
    }
    uint32_t ix[4] = {0, 0, 0, 0};
    uint64_t pv[4] = {0, 0, 0, 0};
    const int np = __popcll(part);
    uint64_t rest = part;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (rest) {
            ix[k] = static_cast<uint32_t>(__ffsll(static_cast<long long>(rest)) - 1);
            pv[k] = s_pv[ix[k]][lane];
            rest &= rest - 1;
        }
    }
    const uint32_t over = np > (FMT == 64 ? 4 : 2) ? 1u : 0u, haspart = np > 0 ? 1u : 0u;
    const LW sm = static_cast<LW>(any), fm = static_cast<LW>(full);
    if constexpr (FMT == 16)
        reinterpret_cast<uint32_t*>(tab)[w] = (static_cast<uint32_t>(fm) << 16) | (16u + ix[0]) | ((16u + ix[1]) << 5) |
                                              (haspart << 10) | (over << 11);
    else if constexpr (FMT == 32)
        reinterpret_cast<uint2*>(tab)[w] =
            make_uint2(static_cast<uint32_t>(fm), ix[0] | (ix[1] << 8) | (haspart << 16) | (over << 17));
    else {
        reinterpret_cast<uint64_t*>(tab)[w] = static_cast<uint64_t>(fm);
        reinterpret_cast<uint32_t*>(tab + split64_meta_offset(nw64))[w] =
            ix[0] | (ix[1] << 6) | (ix[2] << 12) | (ix[3] << 18) | (haspart << 24) | (over << 25);
    }
    uint4* xo = reinterpret_cast<uint4*>(tab + split64_x_offset(FMT, nw64));
    const uint32_t xs = split64_x_bytes(FMT) / 16;
    xo[xs * w] = make_uint4(static_cast<uint32_t>(pv[0]), static_cast<uint32_t>(pv[0] >> 32),
                            static_cast<uint32_t>(pv[1]), static_cast<uint32_t>(pv[1] >> 32));
    if (xs == 2)
        xo[xs * w + 1] = make_uint4(static_cast<uint32_t>(pv[2]), static_cast<uint32_t>(pv[2] >> 32),
                                    static_cast<uint32_t>(pv[3]), static_cast<uint32_t>(pv[3] >> 32));
    static_cast<LW*>(s_only_g)[w] = sm;
}

// Multi-frame summary over 64-cell words, thread per (word, frame), index
// w * frames + f:
//   tab  : 32-B entry {F, ia | ib<<8 | hasB<<16 | over<<17, Pa lo, Pa hi,
//          Pb lo, Pb hi, S, 0} -- one 256-bit load, branch-free probes
//   s_only: S (4 B; full-mask pairs read only this)
constexpr uint32_t kHasB64 = 0x10000u, kOver64 = 0x20000u;
__global__ void __launch_bounds__(256) summary_b64_kernel(const uint64_t* __restrict__ P64, int props, int frames,
                                                          uint32_t nw64, uint64_t cells, uint4* __restrict__ tab,
                                                          uint64_t* __restrict__ pbt, uint32_t* __restrict__ s_only,
                                                          uint32_t* __restrict__ task_ctr, int nctr) {
    const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
    const int f = blockIdx.y;
    if (f == 0 && w < static_cast<uint32_t>(nctr)) task_ctr[w] = 0;
    if (w > nw64) return;
    uint32_t s = 0, full = 0, ia = 0, ib = 0;
    uint64_t pa = 0, pb = 0;
    int np = 0;
    const uint64_t lo = static_cast<uint64_t>(w) * 64;
    if (w < nw64 && lo < cells) {
        const uint64_t valid = (cells - lo >= 64) ? ~0ull : ((1ull << (cells - lo)) - 1ull);
        const uint64_t* base = P64 + static_cast<uint64_t>(f) * props * nw64 + w;
#pragma unroll 4
        for (int j = 0; j < props; ++j) {
            const uint64_t x = base[static_cast<uint64_t>(j) * nw64] & valid;
            s |= static_cast<uint32_t>(x != 0) << j;
            full |= static_cast<uint32_t>(x == valid) << j;
            if (x != 0 && x != valid) {
                if (np == 0) {
                    pa = x;
                    ia = static_cast<uint32_t>(j);
                } else if (np == 1) {
                    pb = x;
                    ib = static_cast<uint32_t>(j);
                }
                ++np;
            }
        }
    }
    const uint64_t idx = static_cast<uint64_t>(w) * frames + f;
    (void)pbt;
    tab[2 * idx] = make_uint4(full, ia | (ib << 8) | (np > 1 ? kHasB64 : 0u) | (np > 2 ? kOver64 : 0u),
                              static_cast<uint32_t>(pa), static_cast<uint32_t>(pa >> 32));
    tab[2 * idx + 1] = make_uint4(static_cast<uint32_t>(pb), static_cast<uint32_t>(pb >> 32), s, 0u);
    s_only[idx] = s;
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
// HEAD flag (bit 31) of a pair's word field as 0/1, on the FMA pipe (the
// ALU pipe is the single-frame kernel's bottleneck): hi32(wh * 2).
__device__ __forceinline__ uint32_t head_bit(uint32_t wh) {
    uint32_t r;
    asm("mul.hi.u32 %0, %1, 2;" : "=r"(r) : "r"(wh));
    return r;
}
// acc + b * 2^k on the FMA pipe
__device__ __forceinline__ uint32_t mad_pow2(uint32_t b, uint32_t pow2, uint32_t acc) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(b), "r"(pow2), "r"(acc));
    return r;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
    uint2 v;
    asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
// x = smem[a] (16 B) if c != 0, else unchanged (callers pre-zero)
__device__ __forceinline__ void lds128_if(uint32_t c, uint32_t a, uint4& x) {
    asm("{\n .reg .pred p;\n setp.ne.u32 p, %4, 0;\n @p ld.shared.v4.u32 {%0, %1, %2, %3}, [%5];\n}\n"
        : "+r"(x.x), "+r"(x.y), "+r"(x.z), "+r"(x.w)
        : "r"(c), "r"(a));
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
// {x, y} = smem[a] if c != 0, else unchanged (callers pre-zero)
__device__ __forceinline__ void lds64_if(uint32_t c, uint32_t a, uint32_t& x, uint32_t& y) {
    asm("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p ld.shared.v2.u32 {%0, %1}, [%3];\n}\n"
        : "+r"(x), "+r"(y)
        : "r"(c), "r"(a));
}
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    if (bytes) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
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
// [p0, p1)) from an atomic counter.  The frame's split table (M / X) is
// TMA-bulk-copied once per CTA into shared memory when it fits (one CTA of
// 32 warps per SM), else read through L1.
//
// A warp chunk is 32*K consecutive pairs, lane l owning pairs [K*l, K*l+K).
// Row recovery: HEAD flags mark each row's first pair.  When every lane holds
// at most one head (rows longer than K pairs -- the common case), a lane's
// pairs split into `pre` (before its head: the row open from lower lanes)
// and `post` (from its head on), computed with predicated ORs; the head
// count prefix is one ballot, and the rows spanning lanes are closed by one
// warp-wide segmented OR scan.  Chunks where some lane holds several heads
// (short rows) take the general lane-local loop.
// ---------------------------------------------------------------------------

// Per-kernel constants of the single-frame chunk processing.
template <int FMT, typename SW, bool SMEM>
struct StreamCtx {
    using LW = typename Fmt<FMT>::LW;
    using E = typename Fmt<FMT>::E;
    static constexpr int kShift = FMT == 16 ? 16 : 0;  // label bits sit at [kShift, kShift + props) of v
    const uint8_t* tab;     // split table (smem or global) / SF<u64> entries (FMT 64)
    const uint8_t* xbytes;  // X part of the split table
    uint32_t tab_s, x_s;    // the same as shared-memory addresses (SMEM)
    const LW* s_only;
    const uint32_t* P32;
    uint32_t nw32;
    SW* out;       // label of row r at out[r * ostride] (ostride = frames of the
    uint32_t ostride;  // submit: one frame of an edge-major multi-frame buffer)
    int lane;
    uint32_t lt, le;
};

// The row being assembled across chunks of one task.
template <typename LW>
struct RowState {
    int32_t r0, r1;      // the task's rows [r0, r1): only these are stored
    int32_t open_row;    // row owning `carry`
    LW carry;
};

// Row recovery for one warp chunk: lane l's K consecutive pairs have label
// contributions v[0..K) and HEAD bits `heads`; closes every row that ends in
// the chunk (stores rows in [rs.r0, rs.r1) only) and carries the open row.
template <int FMT, typename SW, bool SMEM, int K>
__device__ __forceinline__ void segment_chunk(const StreamCtx<FMT, SW, SMEM>& sc,
                                              RowState<typename Fmt<FMT>::LW>& rs, uint32_t heads,
                                              const typename Fmt<FMT>::LW (&v)[K]) {
    using LW = typename Fmt<FMT>::LW;
    constexpr int kShift = StreamCtx<FMT, SW, SMEM>::kShift;
    const int lane = sc.lane;
    SW* out = sc.out;
    if (!__any_sync(0xffffffffu, (heads & (heads - 1)) != 0)) {
        // ---- fast path: every lane holds at most one head ----------
        const uint32_t hmask_all = __ballot_sync(0xffffffffu, heads != 0);
        const int hb = __popc(hmask_all & sc.lt);  // rows opened in lower lanes
        LW pre = 0, post = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if ((heads & ((2u << k) - 1u)) == 0) pre |= v[k];
            else post |= v[k];
        }
        const uint32_t hm = hmask_all & sc.le;
        const int seg = hm ? 31 - __clz(hm) : 0;
        LW x = heads ? post : pre;
        if (lane == 0 && !heads) x |= rs.carry;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const LW y = shfl_up(x, d);
            if (lane - d >= seg) x |= y;
        }
        LW excl = shfl_up(x, 1);
        if (lane == 0) excl = rs.carry;
        if (heads) {
            const int32_t row = rs.open_row + hb;  // the row open before this lane's head
            if (row >= rs.r0 && row < rs.r1) out[static_cast<uint64_t>(row) * sc.ostride] = static_cast<SW>((excl | pre) >> kShift);
        }
        rs.carry = shfl_idx(x, 31);
        rs.open_row += __popc(hmask_all);
    } else {
        // ---- general path: lanes may hold several heads -----------
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
                if (seen) {
                    const int32_t row = rs.open_row + hb + seen;
                    if (row < rs.r1) out[static_cast<uint64_t>(row) * sc.ostride] = static_cast<SW>(cur_or >> kShift);
                } else {
                    pre = cur_or;
                }
                ++seen;
                cur_or = 0;
            }
            cur_or |= v[k];
        }
        if (!nh) pre = cur_or;
        const uint32_t hmask = __ballot_sync(0xffffffffu, nh > 0) & sc.le;
        const int seg = hmask ? 31 - __clz(hmask) : 0;
        LW x = nh ? cur_or : pre;
        if (lane == 0 && !nh) x |= rs.carry;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const LW y = shfl_up(x, d);
            if (lane - d >= seg) x |= y;
        }
        LW excl = shfl_up(x, 1);
        if (lane == 0) excl = rs.carry;
        if (nh) {
            const int32_t row = rs.open_row + hb;  // the row open before this lane's first head
            if (row >= rs.r0 && row < rs.r1) out[static_cast<uint64_t>(row) * sc.ostride] = static_cast<SW>((excl | pre) >> kShift);
        }
        rs.carry = shfl_idx(x, 31);
        rs.open_row += tot;
    }
}

// One warp chunk held in cur (lane-contiguous K pairs).  `reload(h0, h1)` is
// called once pieces [h0, h1) of cur are no longer needed (after each half),
// so a caller can prefetch the next chunk in place.
template <int FMT, typename SW, bool SMEM, int K, typename Reload>
__device__ __forceinline__ void stream_chunk(const StreamCtx<FMT, SW, SMEM>& sc,
                                             RowState<typename Fmt<FMT>::LW>& rs, uint4 (&cur)[K / 2],
                                             Reload&& reload) {
    using LW = typename Fmt<FMT>::LW;
    using E = typename Fmt<FMT>::E;
    constexpr int kShift = StreamCtx<FMT, SW, SMEM>::kShift;
    const int lane = sc.lane;
    uint32_t heads = 0;  // bit k: pair k opens a row
    LW v[K];
    if constexpr (FMT == 64) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint32_t mk = (k & 1) ? cur[k / 2].z : cur[k / 2].x;
            const uint32_t wh = (k & 1) ? cur[k / 2].w : cur[k / 2].y;
            heads |= (wh >> 31) << k;
            const uint32_t w = wh & kWordMask;
            v[k] = probe<FMT>(ld_entry(reinterpret_cast<const E*>(sc.tab) + w), mk, w, sc.s_only, w, LW(0), sc.P32,
                              sc.nw32);
            if (k == K / 2 - 1) reload(0, K / 4);
        }
        reload(K / 4, K / 2);
    } else {
        const uint32_t* mtab16 = reinterpret_cast<const uint32_t*>(sc.tab);
        const uint2* mtab32 = reinterpret_cast<const uint2*>(sc.tab);
        const uint2* xtab = reinterpret_cast<const uint2*>(sc.xbytes);
        // straight-line per half: M gathers, predicated X gathers, probes;
        // the rare third-partial-prop fix-up runs after each half
        auto look = [&](int k, uint32_t& over) {
            const uint32_t mk = (k & 1) ? cur[k / 2].z : cur[k / 2].x;
            const uint32_t wh = (k & 1) ? cur[k / 2].w : cur[k / 2].y;
            heads = mad_pow2(head_bit(wh), 1u << k, heads);
            if constexpr (FMT == 16) {
                // byte offsets straight from the pair's word field: the HEAD
                // bit (31) shifts out (shared-memory tables are small); X is
                // gathered only by lanes whose word has a partial prop (an
                // unconditional gather saves ALU work but saturates the
                // shared-memory pipe)
                uint32_t mw;
                uint2 x = make_uint2(0u, 0u);
                if constexpr (SMEM) {
                    mw = lds32(sc.tab_s + (wh << 2));
                    lds64_if(mw & (1u << 10), sc.x_s + (wh << 3), x.x, x.y);
                } else {
                    mw = mtab16[wh & kWordMask];
                    if (mw & (1u << 10)) x = xtab[wh & kWordMask];
                }
                uint32_t vv = mw;  // F<<16; bits < 16 are index/flag garbage, shifted out at the store
                if (mk & x.x) vv |= __funnelshift_l(0u, 1u, mw);
                if (mk & x.y) vv |= __funnelshift_l(0u, 1u, mw >> 5);
                over |= mw & (1u << 11);
                v[k] = vv;
            } else {
                const uint32_t w = wh & kWordMask;
                const uint2 mw = mtab32[w];
                uint2 x = make_uint2(0u, 0u);
                if (mw.y & 0x10000u) x = xtab[w];
                uint32_t vv = mw.x;
                if (mk & x.x) vv |= __funnelshift_l(0u, 1u, mw.y);
                if (mk & x.y) vv |= __funnelshift_l(0u, 1u, mw.y >> 8);
                over |= mw.y & 0x20000u;
                v[k] = vv;
            }
        };
        auto fix = [&](int k) {  // a word with >= 3 partial props: exact gather of the rest
            const uint32_t mk = (k & 1) ? cur[k / 2].z : cur[k / 2].x;
            const uint32_t w = ((k & 1) ? cur[k / 2].w : cur[k / 2].y) & kWordMask;
            uint32_t known, ov;
            if constexpr (FMT == 16) {
                const uint32_t mw = mtab16[w];
                known = (mw >> 16) | (1u << ((mw & 31) - 16)) | (1u << ((mw >> 5 & 31) - 16));
                ov = mw >> 11 & 1u;
            } else {
                const uint2 mw = mtab32[w];
                known = mw.x | (1u << (mw.y & 31)) | (1u << (mw.y >> 8 & 31));
                ov = mw.y >> 17 & 1u;
            }
            if (ov) v[k] |= probe_gather<uint32_t>(mk, w, sc.s_only[w] & ~known, sc.P32, sc.nw32) << kShift;
        };
        uint32_t ov_lo = 0, ov_hi = 0;
#pragma unroll
        for (int k = 0; k < K / 2; ++k) look(k, ov_lo);
        if (ov_lo) {
#pragma unroll
            for (int k = 0; k < K / 2; ++k) fix(k);
        }
        reload(0, K / 4);
#pragma unroll
        for (int k = K / 2; k < K; ++k) look(k, ov_hi);
        if (ov_hi) {
#pragma unroll
            for (int k = K / 2; k < K; ++k) fix(k);
        }
        reload(K / 4, K / 2);
    }
    segment_chunk<FMT, SW, SMEM, K>(sc, rs, heads, v);
}

template <int FMT, typename SW, bool SMEM>
__device__ __forceinline__ void stream_close_task(const StreamCtx<FMT, SW, SMEM>& sc,
                                                  const RowState<typename Fmt<FMT>::LW>& rs) {
    if (sc.lane == 0 && rs.open_row >= rs.r0 && rs.open_row < rs.r1)
        sc.out[static_cast<uint64_t>(rs.open_row) * sc.ostride] =
            static_cast<SW>(rs.carry >> StreamCtx<FMT, SW, SMEM>::kShift);
}

// Copies the split table into shared memory (thread 0 issues, all wait later).
__device__ __forceinline__ void stage_table(uint8_t* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_expect_tx(bar, bytes);
        for (uint32_t o = 0; o < bytes; o += 32768u) {
            const uint32_t n = bytes - o < 32768u ? bytes - o : 32768u;
            bulk_g2s(dst + o, static_cast<const uint8_t*>(src) + o, n, bar);
        }
    }
    __syncthreads();
}

#if LTLG_AB_BUILD  // 32-cell single-frame kernel (A/B knob LTLG_STREAM64=0)
// Register-prefetch variant (tables in L1 / 64-prop entries, or A/B runs):
// the next chunk is loaded in place (IP) half by half, or double-buffered.
template <int FMT, typename SW, bool SMEM, int K, int NT, bool IP>
__global__ void __launch_bounds__(NT)
    label_stream_kernel(const Pair* __restrict__ pairs, const uint64_t* __restrict__ task_pair,
                        const uint32_t* __restrict__ task_row, uint32_t task_begin, uint32_t ntasks,
                        uint32_t* __restrict__ task_ctr, const void* __restrict__ tab_g, uint32_t tab_bytes,
                        const void* __restrict__ s_only_g, const uint32_t* __restrict__ P32, uint32_t nw32,
                        SW* __restrict__ out, uint32_t ostride) {
    using LW = typename Fmt<FMT>::LW;
    static_assert(!(SMEM && FMT == 64), "the 64-prop entry table is read through L1");
    static_assert(K == kStreamK, "the HBM chunk layout is built for kStreamK pairs per lane");
    constexpr uint32_t CH = 32 * K;  // pairs per warp chunk
    extern __shared__ __align__(128) uint8_t smem_raw[];
    __shared__ uint64_t tab_bar;
    const int lane = threadIdx.x & 31;
    const uint8_t* tab = static_cast<const uint8_t*>(tab_g);
    if constexpr (SMEM) {
        stage_table(smem_raw, tab_g, tab_bytes, &tab_bar);
        tab = smem_raw;
    }
    StreamCtx<FMT, SW, SMEM> sc{tab, tab + split_x_offset(FMT, nw32), SMEM ? smem_u32(tab) : 0u,
                               SMEM ? smem_u32(tab) + split_x_offset(FMT, nw32) : 0u, static_cast<const LW*>(s_only_g),
                               P32, nw32, out, ostride, lane, (1u << lane) - 1u, ((1u << lane) - 1u) | (1u << lane)};
    bool tab_ready = !SMEM;

    for (;;) {
        uint32_t t = 0;
        if (lane == 0) t = task_begin + atomicAdd(task_ctr, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= ntasks) break;
        const uint64_t p0 = task_pair[t];  // even: 16-byte aligned
        const uint32_t end = static_cast<uint32_t>(task_pair[t + 1] - p0);
        const uint4* base = reinterpret_cast<const uint4*>(pairs + p0);
        // Rows [r0, r1) are this task's.  Pairs loaded past `end` (last chunk)
        // belong to later rows: the pair at `end` is always a head (the next
        // task's first row, or the head padding after the last task), so they
        // are processed like any other pair and only the stores are
        // restricted to [r0, r1).
        RowState<LW> rs{static_cast<int32_t>(task_row[t]), static_cast<int32_t>(task_row[t + 1]),
                        static_cast<int32_t>(task_row[t]) - 1, LW(0)};
        // Full chunks are piece-transposed in HBM (kStreamK, engine.h), so
        // piece h of lane l is at h*32 + l: each load is one coalesced
        // 512-byte run.  The partial last chunk is in plain order.
        auto load_chunk = [&](uint4 (&cur)[K / 2], uint32_t c, int h0, int h1) {
            const uint4* q = base + c / 2;
            if (c + CH <= end) {
#pragma unroll
                for (int h = h0; h < h1; ++h) cur[h] = ld_stream16(q + h * 32 + lane);
            } else {
#pragma unroll
                for (int h = h0; h < h1; ++h) cur[h] = ld_stream16(q + (K / 2) * lane + h);
            }
        };
        uint4 bufA[K / 2];
        load_chunk(bufA, 0, 0, K / 2);
        if constexpr (SMEM) {
            if (!tab_ready) {
                mbar_wait(&tab_bar, 0);
                tab_ready = true;
            }
        }
        if constexpr (IP) {
            for (uint32_t c = 0; c < end; c += CH) {
                const bool more = c + CH < end;
                stream_chunk<FMT, SW, SMEM, K>(sc, rs, bufA, [&](int h0, int h1) {
                    if (more) load_chunk(bufA, c + CH, h0, h1);
                });
            }
        } else {  // double-buffered: chunk c is processed while chunk c + CH is in flight
            uint4 bufB[K / 2];
            auto none = [](int, int) {};
            for (uint32_t c = 0; c < end; c += 2 * CH) {
                if (c + CH < end) load_chunk(bufB, c + CH, 0, K / 2);
                stream_chunk<FMT, SW, SMEM, K>(sc, rs, bufA, none);
                if (c + CH >= end) break;
                if (c + 2 * CH < end) load_chunk(bufA, c + 2 * CH, 0, K / 2);
                stream_chunk<FMT, SW, SMEM, K>(sc, rs, bufB, none);
            }
        }
        stream_close_task(sc, rs);
    }
    if constexpr (SMEM) {
        if (!tab_ready) mbar_wait(&tab_bar, 0);  // never leave with a bulk copy in flight
    }
}

// 64-cell-word variant (<= 32 props): T from its 12-byte-pair SoA copy
// (kChunk64Bytes, engine.h), one (mask64, word64) pair per swept 64-cell word
// -- 41% fewer pairs per row than 32-cell words at 512^2 --
// against the 64-cell split summary (summary64_kernel).  Same lane
// ownership, in-place prefetch and row segmentation as label_stream_kernel.
#endif  // LTLG_AB_BUILD
// TABLOC: 0 = split table read through L1, 1 = all of it in shared memory,
// 2 = M (every pair) in shared memory and X (partial-prop lanes only) through
// L1 -- for grids whose full table exceeds shared memory.
template <int FMT, typename SW, int TABLOC, int NT>
__global__ void __launch_bounds__(NT)
    label_stream64_kernel(const uint8_t* __restrict__ t64, const uint64_t* __restrict__ task_byte,
                          const uint32_t* __restrict__ task_n, const uint32_t* __restrict__ task_row,
                          uint32_t task_begin, uint32_t ntasks, uint32_t* __restrict__ task_ctr,
                          const void* __restrict__ tab_g, uint32_t tab_bytes, const void* __restrict__ s_only_g,
                          const uint64_t* __restrict__ P64, uint32_t nw64, SW* __restrict__ out, uint32_t ostride) {
    constexpr bool SMEM = TABLOC != 0;   // M in shared memory
    constexpr bool XSMEM = TABLOC == 1;  // X in shared memory
    using LW = typename Fmt<FMT>::LW;
    constexpr int K = kStreamK;
    constexpr uint32_t CH = kStreamCH;
    constexpr int kShift = FMT == 16 ? 16 : 0;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    __shared__ uint64_t tab_bar;
    const int lane = threadIdx.x & 31;
    const uint32_t xoff = split64_x_offset(FMT, nw64);
    const uint8_t* tab = static_cast<const uint8_t*>(tab_g);
    const uint8_t* xg = static_cast<const uint8_t*>(tab_g) + xoff;  // X in global memory
    {  // the warp's static first task (below): its first chunk of T into L2
       // while the summary is still running
        const uint32_t t0 = task_begin + blockIdx.x * (NT / 32) + (threadIdx.x >> 5);
        if (t0 < ntasks && __ldg(task_n + t0) >= CH && static_cast<uint32_t>(lane) * 128u < kChunk64Bytes)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(t64 + __ldg(task_byte + t0) + lane * 128u));
    }
    // launched as a programmatic dependent of the summary kernel: its table,
    // S words and the reset task counter are ready after this
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if constexpr (SMEM) {
        stage_table(smem_raw, tab_g, XSMEM ? tab_bytes : xoff, &tab_bar);
        tab = smem_raw;
    }
    const LW* s_only = static_cast<const LW*>(s_only_g);
    StreamCtx<FMT, SW, SMEM> sc{tab, XSMEM ? tab + xoff : xg, SMEM ? smem_u32(tab) : 0u,
                               XSMEM ? smem_u32(tab) + xoff : 0u, s_only, reinterpret_cast<const uint32_t*>(P64), nw64,
                               out, ostride, lane, (1u << lane) - 1u, ((1u << lane) - 1u) | (1u << lane)};
    const uint32_t* mtab16 = reinterpret_cast<const uint32_t*>(tab);
    const uint2* mtab32 = reinterpret_cast<const uint2*>(tab);
    const uint4* xtab = reinterpret_cast<const uint4*>(XSMEM ? tab + xoff : xg);
    bool tab_ready = !SMEM;

    // a warp's first task is static (task_begin + its global warp index), so
    // its critical path starts without an atomic round trip; later tasks
    // come from the counter, after the static ones
    const uint32_t nwarps = gridDim.x * (NT / 32);
    uint32_t t_static = task_begin + blockIdx.x * (NT / 32) + (threadIdx.x >> 5);
    const bool dyn = task_begin + nwarps < ntasks;
    for (;;) {
        uint32_t t = t_static;
        if (t_static == ~0u) {
            // every task static (small abstractions: one task per warp): no
            // failing fetch, so no burst of same-address atomics at the end
            if (lane == 0) t = dyn ? task_begin + nwarps + atomicAdd(task_ctr, 1u) : ntasks;
            t = __shfl_sync(0xffffffffu, t, 0);
        }
        t_static = ~0u;
        if (t >= ntasks) break;
        const uint8_t* base = t64 + task_byte[t];
        const uint32_t n = task_n[t];
        const uint32_t nfull = n / CH;
        const uint32_t part = n - nfull * CH;
        const uint8_t* pm = base + static_cast<uint64_t>(nfull) * kChunk64Bytes;      // partial chunk masks
        const uint8_t* pw = pm + ((8u * part + 15u) & ~15u);                            // and words
        RowState<LW> rs{static_cast<int32_t>(task_row[t]), static_cast<int32_t>(task_row[t + 1]),
                        static_cast<int32_t>(task_row[t]) - 1, LW(0)};
        uint4 cm[K / 2], cw[K / 4];  // masks (2 per piece), word fields (4 per piece)
        // pieces [h0, h1) of masks and [h0/2, h1/2) of words of chunk c
        auto load = [&](uint32_t c, int h0, int h1) {
            if (c + CH <= n) {  // full chunk: piece-transposed, coalesced
                const uint8_t* q = base + static_cast<uint64_t>(c / CH) * kChunk64Bytes;
#pragma unroll
                for (int h = h0; h < h1; ++h) cm[h] = ld_stream16(q + (h * 32 + lane) * 16);
#pragma unroll
                for (int h = h0 / 2; h < h1 / 2; ++h) cw[h] = ld_stream16(q + 8 * CH + (h * 32 + lane) * 16);
            } else {  // partial chunk: plain, lane-contiguous
#pragma unroll
                for (int h = h0; h < h1; ++h) cm[h] = ld_stream16(pm + lane * 64 + h * 16);
#pragma unroll
                for (int h = h0 / 2; h < h1 / 2; ++h) cw[h] = ld_stream16(pw + lane * 32 + h * 16);
            }
        };
        load(0, 0, K / 2);
        if constexpr (SMEM) {
            if (!tab_ready) {
                mbar_wait(&tab_bar, 0);
                tab_ready = true;
            }
        }
        for (uint32_t c = 0; c < n; c += CH) {
            const bool more = c + CH < n;
            if (c + CH > n) {  // partial chunk: pairs past n become no-op heads
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    if (static_cast<uint32_t>(K * lane + k) >= part) {
                        if (k & 1) {
                            cm[k / 2].z = 0;
                            cm[k / 2].w = 0;
                        } else {
                            cm[k / 2].x = 0;
                            cm[k / 2].y = 0;
                        }
                        const uint32_t sw = nw64 | kHead;
                        switch (k & 3) {
                            case 0: cw[k / 4].x = sw; break;
                            case 1: cw[k / 4].y = sw; break;
                            case 2: cw[k / 4].z = sw; break;
                            default: cw[k / 4].w = sw; break;
                        }
                    }
                }
            }
            uint32_t heads = 0;
            LW v[K];
            auto mlo = [&](int k) { return (k & 1) ? cm[k / 2].z : cm[k / 2].x; };
            auto mhi = [&](int k) { return (k & 1) ? cm[k / 2].w : cm[k / 2].y; };
            auto wfield = [&](int k) {
                switch (k & 3) {
                    case 0: return cw[k / 4].x;
                    case 1: return cw[k / 4].y;
                    case 2: return cw[k / 4].z;
                    default: return cw[k / 4].w;
                }
            };
            auto look = [&](int k, uint32_t& over) {
                const uint32_t lo = mlo(k), hi = mhi(k), wh = wfield(k);
                heads = mad_pow2(head_bit(wh), 1u << k, heads);
                uint32_t meta, part;
                LW f;
                uint4 x = make_uint4(0u, 0u, 0u, 0u);
                if constexpr (FMT == 16) {
                    const uint32_t mw = SMEM ? lds32(sc.tab_s + (wh << 2)) : mtab16[wh & kWordMask];
                    meta = mw;
                    f = mw;
                    part = mw & (1u << 10);
                    over |= mw & (1u << 11);
                } else if constexpr (FMT == 32) {
                    const uint2 m2 = SMEM ? lds64(sc.tab_s + (wh << 3)) : mtab32[wh & kWordMask];
                    f = m2.x;
                    meta = m2.y;
                    part = m2.y & 0x10000u;
                    over |= (m2.y >> 1) & 0x10000u;
                } else {
                    const uint32_t wi = wh & kWordMask;
                    if constexpr (SMEM) {
                        const uint2 f2 = lds64(sc.tab_s + (wi << 3));
                        f = (static_cast<uint64_t>(f2.y) << 32) | f2.x;
                        meta = lds32(sc.tab_s + split64_meta_offset(nw64) + (wi << 2));
                    } else {
                        f = __ldg(reinterpret_cast<const uint64_t*>(tab) + wi);
                        meta = __ldg(reinterpret_cast<const uint32_t*>(tab + split64_meta_offset(nw64)) + wi);
                    }
                    part = meta & (1u << 24);
                    over |= (meta >> 9) & 0x10000u;  // bit 25 -> the shared over flag bit 16
                }
                uint4 x2 = make_uint4(0u, 0u, 0u, 0u);  // FMT 64: partial props c, d
                if constexpr (FMT == 64) {
                    const uint32_t wi = wh & kWordMask;
                    if constexpr (XSMEM) {
                        lds128_if(part, sc.x_s + (wi << 5), x);
                        lds128_if(part, sc.x_s + (wi << 5) + 16, x2);
                    } else if (part) {
                        x = __ldg(xtab + 2 * wi);
                        x2 = __ldg(xtab + 2 * wi + 1);
                    }
                } else if constexpr (XSMEM) {
                    lds128_if(part, sc.x_s + ((wh & kWordMask) << 4), x);
                } else {
                    if (part) x = __ldg(xtab + (wh & kWordMask));
                }
                LW vv = f;  // FMT 16: F<<16; bits < 16 are index/flag garbage, shifted out at the store
                if constexpr (FMT == 64) {
                    if ((lo & x.x) | (hi & x.y)) vv |= LW(1) << (meta & 63);
                    if ((lo & x.z) | (hi & x.w)) vv |= LW(1) << (meta >> 6 & 63);
                    if ((lo & x2.x) | (hi & x2.y)) vv |= LW(1) << (meta >> 12 & 63);
                    if ((lo & x2.z) | (hi & x2.w)) vv |= LW(1) << (meta >> 18 & 63);
                } else {
                    if ((lo & x.x) | (hi & x.y)) vv |= __funnelshift_l(0u, 1u, meta);
                    if ((lo & x.z) | (hi & x.w)) vv |= __funnelshift_l(0u, 1u, meta >> (FMT == 16 ? 5 : 8));
                }
                v[k] = vv;
            };
            auto fix = [&](int k) {  // a word with >= 3 partial props: exact gather of the rest
                const uint32_t w = wfield(k) & kWordMask;
                LW known;
                uint32_t ov;
                if constexpr (FMT == 16) {
                    const uint32_t mw = mtab16[w];
                    known = (mw >> 16) | (1u << ((mw & 31) - 16)) | (1u << ((mw >> 5 & 31) - 16));
                    ov = mw >> 11 & 1u;
                } else if constexpr (FMT == 32) {
                    const uint2 mw = mtab32[w];
                    known = mw.x | (1u << (mw.y & 31)) | (1u << (mw.y >> 8 & 31));
                    ov = mw.y >> 17 & 1u;
                } else {
                    const uint32_t mt = reinterpret_cast<const uint32_t*>(tab + split64_meta_offset(nw64))[w];
                    known = reinterpret_cast<const uint64_t*>(tab)[w] | (LW(1) << (mt & 63)) | (LW(1) << (mt >> 6 & 63)) |
                            (LW(1) << (mt >> 12 & 63)) | (LW(1) << (mt >> 18 & 63));
                    ov = mt >> 25 & 1u;
                }
                if (ov) {
                    const uint64_t m = (static_cast<uint64_t>(mhi(k)) << 32) | mlo(k);
                    LW rest = s_only[w] & ~known, hit = 0;
                    while (rest) {
                        const int j = lowest_bit(rest);
                        if (m & __ldg(P64 + static_cast<uint64_t>(j) * nw64 + w)) hit |= LW(1) << j;
                        rest &= rest - 1;
                    }
                    v[k] |= hit << kShift;
                }
            };
            uint32_t ov_lo = 0, ov_hi = 0;
#pragma unroll
            for (int k = 0; k < K / 2; ++k) look(k, ov_lo);
            if (ov_lo) {
#pragma unroll
                for (int k = 0; k < K / 2; ++k) fix(k);
            }
            if (more) load(c + CH, 0, K / 4);
#pragma unroll
            for (int k = K / 2; k < K; ++k) look(k, ov_hi);
            if (ov_hi) {
#pragma unroll
                for (int k = K / 2; k < K; ++k) fix(k);
            }
            if (more) load(c + CH, K / 4, K / 2);
            segment_chunk<FMT, SW, SMEM, K>(sc, rs, heads, v);
        }
        stream_close_task(sc, rs);
    }
    if constexpr (SMEM) {
        if (!tab_ready) mbar_wait(&tab_bar, 0);  // never leave with a bulk copy in flight
    }
}

#if LTLG_AB_BUILD  // 32-cell single-frame TMA-ring kernel (A/B knob LTLG_STREAM_CFG=4)
// TMA-ring variant (split table in shared memory): every warp streams its
// chunks through a 2-slot ring of 32*K-pair buffers filled by
// cp.async.bulk (TMA) with one mbarrier per slot.  A chunk is copied into
// registers (4 conflict-free LDS.128 per lane) as soon as its slot lands and
// the slot is refilled at once, so two chunks per warp (4 KB) are always in
// flight independent of registers.  The chunk sequence runs across task
// boundaries: the next task is claimed when the issue side reaches the end
// of the current one.
constexpr int kRingSlots = 2;
size_t stream_ring_bytes(int warps) {
    return static_cast<size_t>(warps) * kRingSlots * kStreamCH * sizeof(Pair) + static_cast<size_t>(warps) * kRingSlots * 8;
}

template <int FMT, typename SW, int NT>
__global__ void __launch_bounds__(NT)
    label_stream_tma_kernel(const Pair* __restrict__ pairs, const uint64_t* __restrict__ task_pair,
                            const uint32_t* __restrict__ task_row, uint32_t task_begin, uint32_t ntasks,
                            uint32_t* __restrict__ task_ctr, const void* __restrict__ tab_g, uint32_t tab_bytes,
                            const void* __restrict__ s_only_g, const uint32_t* __restrict__ P32, uint32_t nw32,
                            SW* __restrict__ out, uint32_t ostride) {
    static_assert(FMT != 64, "split tables only");
    using LW = typename Fmt<FMT>::LW;
    constexpr int K = kStreamK;
    constexpr uint32_t CH = kStreamCH;
    constexpr uint32_t kSlotBytes = CH * sizeof(Pair);
    constexpr int kWarps = NT / 32;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    __shared__ uint64_t tab_bar;
    __shared__ uint32_t sink;  // target of the never-relied-upon store that pins LDS completion
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    // layout: [table (tab_bytes, 16-aligned)] [rings: kWarps x kRingSlots x slot] [mbarriers]
    const uint32_t ring_off = (tab_bytes + 127u) & ~127u;
    uint8_t* ring = smem_raw + ring_off + static_cast<uint32_t>(warp) * kRingSlots * kSlotBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + ring_off + kWarps * kRingSlots * kSlotBytes) +
                     warp * kRingSlots;
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < kRingSlots; ++q) mbar_init(&bars[q], 1);
    }
    stage_table(smem_raw, tab_g, tab_bytes, &tab_bar);  // includes __syncthreads (barrier inits visible)
    const uint8_t* tab = smem_raw;
    StreamCtx<FMT, SW, true> sc{tab, tab + split_x_offset(FMT, nw32), smem_u32(tab), smem_u32(tab) + split_x_offset(FMT, nw32),
                               static_cast<const LW*>(s_only_g), P32, nw32, out, ostride, lane, (1u << lane) - 1u,
                               ((1u << lane) - 1u) | (1u << lane)};

    // ---- issue side (warp-uniform state; lane 0 issues the copies) --------
    uint32_t it = 0;     // task of the next chunk to issue (>= ntasks: none)
    uint64_t ip0 = 0;    // its first pair
    uint32_t iend = 0;   // its pair count
    uint32_t ic = 0;     // chunk offset of the next chunk to issue
    auto claim = [&]() {
        uint32_t tn = 0;
        if (lane == 0) tn = task_begin + atomicAdd(task_ctr, 1u);
        it = __shfl_sync(0xffffffffu, tn, 0);
        ic = 0;
        if (it < ntasks) {
            ip0 = task_pair[it];
            iend = static_cast<uint32_t>(task_pair[it + 1] - ip0);
        }
    };
    static_assert(kRingSlots == 2, "slot bookkeeping below is written for two slots");
    uint32_t st0 = 0, sc0 = 0, st1 = 0, sc1 = 0;  // (task, chunk offset) held by slot 0 / 1
    auto issue = [&](int q) {
        if (q) {
            st1 = it;
            sc1 = ic;
        } else {
            st0 = it;
            sc0 = ic;
        }
        if (it >= ntasks) return;
        if (lane == 0) {
            mbar_expect_tx(&bars[q], kSlotBytes);
            bulk_g2s(ring + q * kSlotBytes, pairs + ip0 + ic, kSlotBytes, &bars[q]);  // may read past the task: padded
        }
        ic += CH;
        if (ic >= iend) claim();
    };
    claim();
#pragma unroll
    for (int q = 0; q < kRingSlots; ++q) issue(q);
    mbar_wait(&tab_bar, 0);

    // ---- compute side -----------------------------------------------------
    uint32_t ph = 0;               // bit q: parity to wait for on slot q
    uint32_t ct = ~0u;             // task being assembled
    uint32_t cend = 0;
    RowState<LW> rs{0, 0, -1, LW(0)};
    for (int q = 0;; q ^= 1) {
        const uint32_t t = q ? st1 : st0;
        if (t >= ntasks) break;
        const uint32_t c = q ? sc1 : sc0;
        if (t != ct) {  // first chunk of a new task
            if (ct != ~0u) stream_close_task(sc, rs);
            ct = t;
            cend = static_cast<uint32_t>(task_pair[t + 1] - task_pair[t]);
            rs = RowState<LW>{static_cast<int32_t>(task_row[t]), static_cast<int32_t>(task_row[t + 1]),
                              static_cast<int32_t>(task_row[t]) - 1, LW(0)};
        }
        mbar_wait(&bars[q], ph >> q & 1u);
        ph ^= 1u << q;
        // piece-transposed full chunk: piece h of this lane at (h*32 + lane)*16,
        // lane-consecutive and conflict-free; the plain partial last chunk at
        // (K/2*lane + h)*16
        const bool full = c + CH <= cend;
        const uint8_t* lp = ring + q * kSlotBytes + lane * (full ? 16 : 8 * K);
        const uint32_t step = full ? 512u : 16u;
        uint4 cur[K / 2];
#pragma unroll
        for (int h = 0; h < K / 2; ++h) cur[h] = *reinterpret_cast<const uint4*>(lp + h * step);
        // the slot may be refilled only after every lane's LDS has returned:
        // consume the loaded registers (a compare the compiler cannot drop)
        // before the warp barrier that precedes the refill
        asm volatile("{\n .reg .pred p;\n setp.eq.u32 p, %0, %1;\n @p st.shared.u32 [%2], %0;\n}\n" ::"r"(cur[0].x),
                     "r"(cur[K / 2 - 1].w), "r"(smem_u32(&sink)));
        __syncwarp();
        issue(q);
        stream_chunk<FMT, SW, true, K>(sc, rs, cur, [](int, int) {});
    }
    if (ct != ~0u) stream_close_task(sc, rs);
}

#endif  // LTLG_AB_BUILD
// ---------------------------------------------------------------------------
// F frames.  Persistent warps pull tasks; lane l owns frames l, l+32, ...
// (FPL of them; FULL = every lane owns exactly FPL frames).  Each T pair is
// read from HBM once for all F frames and broadcast by shuffle.
//   tab[w * frames + f]     entry (16 B for <= 32 props)
//   s_only[w * frames + f]  the S mask alone: a pair whose mask covers the
//                           whole word hits exactly the props set somewhere in
//                           the word (warp-uniform fast path, 4 B per lookup)
//   P32 frame f column j at (f*props + j) * nw32
//   out[perm[row] * frames + f] (edge-major)
// ---------------------------------------------------------------------------
template <int FMT, typename SW, int FPL, bool FULL>
__global__ void __launch_bounds__(256)
    label_batch_kernel(const Pair* __restrict__ pairs, const uint64_t* __restrict__ task_pair,
                       const uint32_t* __restrict__ task_row, uint32_t task_begin, uint32_t ntasks,
                       uint32_t* __restrict__ task_ctr, const void* __restrict__ tab_g, const void* __restrict__ s_only_g,
                       const uint32_t* __restrict__ P32, uint32_t nw32, int props, int frames,
                       const uint32_t* __restrict__ perm, SW* __restrict__ out) {
    using LW = typename Fmt<FMT>::LW;
    using E = typename Fmt<FMT>::E;
    const int lane = threadIdx.x & 31;
    const uint64_t frame_stride = static_cast<uint64_t>(props) * nw32;
    const E* lane_tab = static_cast<const E*>(tab_g) + lane;
    const LW* lane_s = static_cast<const LW*>(s_only_g) + lane;
    const uint32_t* lane_P = P32 + static_cast<uint64_t>(lane) * frame_stride;
    bool fv[FPL];
#pragma unroll
    for (int q = 0; q < FPL; ++q) fv[q] = FULL || lane + 32 * q < frames;

    for (;;) {
        uint32_t t = 0;
        if (lane == 0) t = task_begin + atomicAdd(task_ctr, 1u);
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
        // one pair (mask m, word field wh), broadcast to every lane
        auto pair_step = [&](uint32_t m, uint32_t wh) {
            if (wh & kHead) {  // warp-uniform
                if (row >= r0) store(row);
                ++row;
#pragma unroll
                for (int q = 0; q < FPL; ++q) acc[q] = 0;
            }
            const uint32_t w = wh & kWordMask;
            const uint32_t off = w * static_cast<uint32_t>(frames);
            if (m == 0xffffffffu) {  // warp-uniform: the whole word is swept
                const LW* sp = index_wide(lane_s, off);
#pragma unroll
                for (int q = 0; q < FPL; ++q)
                    if (fv[q]) acc[q] |= __ldg(sp + 32 * q);
            } else {
                const E* ep = index_wide(lane_tab, off);
#pragma unroll
                for (int q = 0; q < FPL; ++q)
                    if (fv[q]) {
                        const E e = ld_entry(ep + 32 * q);
                        acc[q] |= probe<FMT>(e, m, w, lane_s, off + 32 * q, acc[q],
                                             lane_P + 32 * q * frame_stride, nw32);
                    }
            }
        };
        uint2 cur = ld_stream8(pairs + p0 + lane);
        for (uint64_t c = p0; c < p1; c += 32) {
            uint2 nxt = cur;
            if (c + 32 < p1) nxt = ld_stream8(pairs + c + 32 + lane);
            const int n = static_cast<int>(p1 - c < 32 ? p1 - c : 32);
            for (int i = 0; i < n; ++i)
                pair_step(__shfl_sync(0xffffffffu, cur.x, i), __shfl_sync(0xffffffffu, cur.y, i));
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

// 2-D z-order (de)interleave: bits of x at every second position
__device__ __forceinline__ uint64_t compact1by1(uint64_t x) {
    x &= 0x5555555555555555ull;
    x = (x | (x >> 1)) & 0x3333333333333333ull;
    x = (x | (x >> 2)) & 0x0f0f0f0f0f0f0f0full;
    x = (x | (x >> 4)) & 0x00ff00ff00ff00ffull;
    x = (x | (x >> 8)) & 0x0000ffff0000ffffull;
    x = (x | (x >> 16)) & 0x00000000ffffffffull;
    return x;
}
__device__ __forceinline__ uint64_t spread1by1(uint64_t x) {
    x &= 0x00000000ffffffffull;
    x = (x | (x << 16)) & 0x0000ffff0000ffffull;
    x = (x | (x << 8)) & 0x00ff00ff00ff00ffull;
    x = (x | (x << 4)) & 0x0f0f0f0f0f0f0f0full;
    x = (x | (x << 2)) & 0x3333333333333333ull;
    x = (x | (x << 1)) & 0x5555555555555555ull;
    return x;
}

// Thread per vehicle cell (blockIdx.y = frame): the cell's centre through
// the pose into world coordinates (the oracle's fp64 operations, in order),
// its world cell, then one ballot per proposition assembles the 32-cell word
// (lane j keeps props j and j + 32 and writes them).  Axis 0 takes the
// z-index bits from the top, round-robin (grid.cpp:108-126): x sits at the
// positions of parity (depth - 1) & 1.
__global__ void __launch_bounds__(256) resample_kernel(Grid2 vg, Grid2 wg, const Pose2* __restrict__ poses,
                                                       int props, const uint32_t* __restrict__ world32,
                                                       uint32_t wnw32, int outside, uint32_t vnw32,
                                                       uint32_t* __restrict__ out32) {
    const uint64_t z = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const int f = blockIdx.y, lane = threadIdx.x & 31;
    const uint32_t w = static_cast<uint32_t>(z >> 5);
    if (w >= vnw32) return;  // whole warps (vnw32 words of 32 cells)
    const Pose2 ps = poses[f];
    const int bvx = axis_bits2(vg.depth, 0), bvy = axis_bits2(vg.depth, 1);
    const int bwx = axis_bits2(wg.depth, 0), bwy = axis_bits2(wg.depth, 1);
    const bool valid = z < (1ull << vg.depth);
    bool in = false, out_all = false;
    uint64_t zw = 0;
    if (valid) {
        const double wxv = __ddiv_rn(__dadd_rn(vg.hi0, -vg.lo0), static_cast<double>(1ull << bvx));
        const double wyv = __ddiv_rn(__dadd_rn(vg.hi1, -vg.lo1), static_cast<double>(1ull << bvy));
        const uint64_t cx = compact1by1(z >> ((vg.depth - 1) & 1)) & ((1ull << bvx) - 1);
        const uint64_t cy = compact1by1(z >> (vg.depth & 1)) & ((1ull << bvy) - 1);
        const double x = __dadd_rn(vg.lo0, __dmul_rn(__dadd_rn(static_cast<double>(cx), 0.5), wxv));
        const double y = __dadd_rn(vg.lo1, __dmul_rn(__dadd_rn(static_cast<double>(cy), 0.5), wyv));
        const double xw = __dadd_rn(__dadd_rn(__dmul_rn(ps.c, x), -__dmul_rn(ps.s, y)), ps.dx);
        const double yw = __dadd_rn(__dadd_rn(__dmul_rn(ps.s, x), __dmul_rn(ps.c, y)), ps.dy);
        const int64_t qx = quantize_dev(wg.lo0, wg.hi0, bwx, xw);
        const int64_t qy = quantize_dev(wg.lo1, wg.hi1, bwy, yw);
        if (qx < 0 || qy < 0) {
            out_all = outside != 0;
        } else {
            in = true;
            zw = (spread1by1(static_cast<uint64_t>(qx)) << ((wg.depth - 1) & 1)) |
                 (spread1by1(static_cast<uint64_t>(qy)) << (wg.depth & 1));
        }
    }
    uint32_t mine0 = 0, mine1 = 0;
    const uint32_t* wsrc = world32 + (zw >> 5);
    for (int j = 0; j < props; ++j) {
        const bool bit = in ? ((__ldg(wsrc + static_cast<uint64_t>(j) * wnw32) >> (zw & 31)) & 1u) != 0 : out_all;
        const uint32_t word = __ballot_sync(0xffffffffu, bit);
        if ((j & 31) == lane) {
            if (j < 32) mine0 = word;
            else mine1 = word;
        }
    }
    uint32_t* dst = out32 + static_cast<uint64_t>(f) * props * vnw32 + w;
    if (lane < props) dst[static_cast<uint64_t>(lane) * vnw32] = mine0;
    if (lane + 32 < props) dst[static_cast<uint64_t>(lane + 32) * vnw32] = mine1;
}


// ---------------------------------------------------------------------------
// Resident-label consumer: monitor transition guards
// TransitionGuard::admits (buchi.hpp:20-22) evaluated over the resident
// labels, as the per-(edge, frame) mask of admitted transitions that
// build_product needs (planner.cpp:53-64).  Guard t is violated by a label L
// iff some prop of positive[t] is absent or some prop of negative[t] present;
// per label byte the violated set is a table lookup:
//   violated(L) = always | OR_b lut[b][(L >> 8b) & 255]
// (lut in shared memory: nbytes x 256 u64; `always` = guards needing a prop
// the labels do not carry).
// ---------------------------------------------------------------------------
template <typename SW>
__global__ void __launch_bounds__(256) guard_kernel(const SW* __restrict__ labels, uint64_t n,
                                                    const uint64_t* __restrict__ lut, uint64_t always,
                                                    uint64_t all_guards, uint64_t* __restrict__ admitted) {
    constexpr int kBytes = sizeof(SW);
    __shared__ uint64_t s_lut[kBytes * 256];
    for (int i = threadIdx.x; i < kBytes * 256; i += blockDim.x) s_lut[i] = lut[i];
    __syncthreads();
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t L = static_cast<uint64_t>(labels[i]);
        uint64_t v = always;
#pragma unroll
        for (int b = 0; b < kBytes; ++b) v |= s_lut[b * 256 + ((L >> (8 * b)) & 255u)];
        admitted[i] = ~v & all_guards;
    }
}

// ---------------------------------------------------------------------------
// Box rasterization into z-ordered P (rasterize_box,
// grid.cpp:260-344).  The host turns every box into integer per-axis cell
// ranges [first, last] with the reference's overlap_cells (grid.cpp:49-61);
// here a thread owns one 64-cell z-word of one (frame, prop) column and ORs
// the boxes' cell masks.  Within a word the low 6 z-bits give every cell a
// fixed per-axis offset, so the cells of axis a whose coordinate lies in
// [first, last] form OR_v PAT[a][v] over the in-range offsets v; a box's
// mask is the AND of its axes' masks.
// ---------------------------------------------------------------------------
struct RasterGeom {
    int k;                 // axes (<= kMaxRasterAxes)
    int depth;
    uint32_t nvals[4];     // distinct within-word offsets per axis
};
__constant__ uint64_t c_raster_pat[4][64];  // [axis][offset] -> cells of the word with that offset
__constant__ RasterGeom c_raster_geom;

__global__ void __launch_bounds__(256) rasterize_kernel(uint32_t nw64, int cols_total, const uint64_t* __restrict__ box_off,
                                                        const int64_t* __restrict__ ranges, uint64_t cells,
                                                        uint64_t* __restrict__ out) {
    const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
    const int col = blockIdx.y;  // frame * props + prop
    if (w >= nw64 || col >= cols_total) return;
    const RasterGeom& g = c_raster_geom;
    // base coordinates of the word's first cell (de-interleave z = 64 w,
    // level l = MSB first, axis l % k, axis bit bits_a - 1 - l / k)
    int64_t base[4] = {0, 0, 0, 0};
    const uint64_t z = static_cast<uint64_t>(w) << 6;
    for (int l = 0; l < g.depth; ++l) {
        const int a = l % g.k;
        base[a] = (base[a] << 1) | static_cast<int64_t>((z >> (g.depth - 1 - l)) & 1u);
    }
    uint64_t m = 0;
    for (uint64_t b = box_off[col]; b < box_off[col + 1]; ++b) {
        const int64_t* r = ranges + b * 8;  // first/last per axis
        uint64_t bm = ~0ull;
        for (int a = 0; a < g.k; ++a) {
            uint64_t am = 0;
            for (uint32_t v = 0; v < g.nvals[a]; ++v) {
                const int64_t c = base[a] + static_cast<int64_t>(v);
                if (c >= r[2 * a] && c <= r[2 * a + 1]) am |= c_raster_pat[a][v];
            }
            bm &= am;
        }
        m |= bm;
    }
    const uint64_t lo = static_cast<uint64_t>(w) * 64;
    if (cells - lo < 64) m &= (1ull << (cells - lo)) - 1ull;
    out[static_cast<uint64_t>(col) * nw64 + w] = m;
}

// ---------------------------------------------------------------------------
// Host launchers
// ---------------------------------------------------------------------------
cudaError_t launch_summary(const uint32_t* P32, int props, int frames, uint32_t nw32, uint64_t cells, void* tab,
                           void* s_only, uint32_t* task_ctr, int nctr, cudaStream_t st) {
    const uint32_t nthreads = nw32 + 1 > static_cast<uint32_t>(nctr) ? nw32 + 1 : static_cast<uint32_t>(nctr);
    dim3 grid((nthreads + 255) / 256, static_cast<unsigned>(frames));
    const int fmt = entry_format(props);
    if (frames == 1 && fmt == 16)
        summary_kernel<16, true><<<grid, 256, 0, st>>>(P32, props, frames, nw32, cells, tab, s_only, task_ctr, nctr);
    else if (frames == 1 && fmt == 32)
        summary_kernel<32, true><<<grid, 256, 0, st>>>(P32, props, frames, nw32, cells, tab, s_only, task_ctr, nctr);
    else if (fmt == 16)
        summary_kernel<16, false><<<grid, 256, 0, st>>>(P32, props, frames, nw32, cells, tab, s_only, task_ctr, nctr);
    else if (fmt == 32)
        summary_kernel<32, false><<<grid, 256, 0, st>>>(P32, props, frames, nw32, cells, tab, s_only, task_ctr, nctr);
    else
        summary_kernel<64, false><<<grid, 256, 0, st>>>(P32, props, frames, nw32, cells, tab, s_only, task_ctr, nctr);
    return cudaGetLastError();
}

cudaError_t launch_summary64(const uint64_t* P64, int props, uint32_t nw64, uint64_t cells, void* tab, void* s_only,
                             uint32_t* task_ctr, int nctr, cudaStream_t st, uint64_t* P_copy, const uint32_t* touched64) {
    // 32 words per CTA (word nw64 is the zero sentinel entry); enough CTAs to
    // reset the nctr task counters too
    const uint32_t nblk_w = (nw64 + 1 + 31) / 32, nblk_c = (static_cast<uint32_t>(nctr) + 255) / 256;
    const unsigned grid = nblk_w > nblk_c ? nblk_w : nblk_c;
    switch (entry_format(props)) {
        case 16: summary64_kernel<16><<<grid, 256, 0, st>>>(P64, props, nw64, cells, static_cast<uint8_t*>(tab), s_only, task_ctr, nctr, P_copy, touched64); break;
        case 32: summary64_kernel<32><<<grid, 256, 0, st>>>(P64, props, nw64, cells, static_cast<uint8_t*>(tab), s_only, task_ctr, nctr, P_copy, touched64); break;
        default: summary64_kernel<64><<<grid, 256, 0, st>>>(P64, props, nw64, cells, static_cast<uint8_t*>(tab), s_only, task_ctr, nctr, P_copy, touched64); break;
    }
    return cudaGetLastError();
}

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

// Dev knobs (A/B sweeps on the GPU box): LTLG_STREAM_TABLE=0 forces the global table
static int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v && *v ? atoi(v) : dflt;
}

#if LTLG_AB_BUILD  // launchers of the 32-cell single-frame kernels
bool stream_table_in_smem(int props, uint32_t nw32) {
    static const int want = env_int("LTLG_STREAM_TABLE", -1);
    if (want == 0 || entry_format(props) == 64) return false;
    return split_table_bytes(props, nw32) <= kMaxSmemTable;
}

template <int FMT, typename SW, bool SMEM, int K, int NT, bool IP = false>
static cudaError_t launch_stream_v(const LaunchArgs& a, cudaStream_t st) {
    const uint32_t tab_bytes = FMT == 64 ? (a.nw32 + 1) * static_cast<uint32_t>(summary_entry_bytes(a.props))
                                         : static_cast<uint32_t>(split_table_bytes(a.props, a.nw32));
    auto kern = label_stream_kernel<FMT, SW, SMEM, K, NT, IP>;
    if constexpr (SMEM) {
        static uint64_t attr_set = 0;  // per device
        int dev = 0;
        cudaGetDevice(&dev);
        if (!(attr_set >> dev & 1u)) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kMaxSmemTable));
            attr_set |= 1ull << dev;
        }
        if (tab_bytes % 16u || tab_bytes > kMaxSmemTable) return cudaErrorInvalidValue;  // never launch an uncompletable TMA copy
        kern<<<sm_count(), NT, tab_bytes, st>>>(a.pairs, a.task_pair, a.task_row, a.task_begin, a.ntasks, a.task_ctr, a.sf, tab_bytes,
                                                a.s_only, a.P32, a.nw32, static_cast<SW*>(a.out), a.ostride ? a.ostride : 1u);
    } else {
        static int per_sm = 0;
        if (!per_sm) {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, 0);
            if (per_sm <= 0) per_sm = 4;
        }
        kern<<<sm_count() * per_sm, NT, 0, st>>>(a.pairs, a.task_pair, a.task_row, a.task_begin, a.ntasks, a.task_ctr, a.sf, tab_bytes,
                                                 a.s_only, a.P32, a.nw32, static_cast<SW*>(a.out), a.ostride ? a.ostride : 1u);
    }
    return cudaSuccess;
}

// Single-frame variant: LTLG_STREAM_CFG (dev knob for A/B sweeps) picks the
// prefetch scheme of the shared-memory-table kernel:
//   2 = double-buffered registers, 3 = in-place prefetch (default; fastest,
//   ncu r02), 4 = TMA ring (needs table + rings in shared memory; it removes
//   the load-latency stalls but spends more ALU-pipe issue, the bottleneck)
constexpr uint32_t kMaxDynSmem = 227u * 1024u - 1024u;  // opt-in limit minus static shared memory
template <int FMT, typename SW>
static cudaError_t launch_stream_tma(const LaunchArgs& a, uint32_t tab_bytes, cudaStream_t st) {
    constexpr int NT = 1024;
    const uint32_t smem = ((tab_bytes + 127u) & ~127u) + static_cast<uint32_t>(stream_ring_bytes(NT / 32));
    auto kern = label_stream_tma_kernel<FMT, SW, NT>;
    static uint32_t attr_set[64] = {};  // per device: dynamic shared memory granted so far
    int dev = 0;
    cudaGetDevice(&dev);
    if (tab_bytes % 16u || smem > kMaxDynSmem || dev >= 64) return cudaErrorInvalidValue;
    if (attr_set[dev] < smem) {
        const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        attr_set[dev] = smem;
    }
    kern<<<sm_count(), NT, smem, st>>>(a.pairs, a.task_pair, a.task_row, a.task_begin, a.ntasks, a.task_ctr, a.sf, tab_bytes,
                                       a.s_only, a.P32, a.nw32, static_cast<SW*>(a.out), a.ostride ? a.ostride : 1u);
    return cudaSuccess;
}

template <int FMT, typename SW>
static cudaError_t launch_stream_t(const LaunchArgs& a, cudaStream_t st) {
    static const int cfg = env_int("LTLG_STREAM_CFG", 3);
    if constexpr (FMT != 64) {
        if (stream_table_in_smem(a.props, a.nw32)) {
            const uint32_t tab_bytes = static_cast<uint32_t>(split_table_bytes(a.props, a.nw32));
            const bool ring_fits = ((tab_bytes + 127u) & ~127u) + stream_ring_bytes(32) <= kMaxDynSmem;
            if (cfg == 4 && ring_fits) return launch_stream_tma<FMT, SW>(a, tab_bytes, st);
            if (cfg == 2) return launch_stream_v<FMT, SW, true, kStreamK, 1024>(a, st);
            return launch_stream_v<FMT, SW, true, kStreamK, 1024, true>(a, st);
        }
    }
    return launch_stream_v<FMT, SW, false, kStreamK, 256, true>(a, st);
}
#endif  // LTLG_AB_BUILD

// Where the 64-cell single-frame kernel keeps its split table (TABLOC).
int stream64_table_loc(int props, uint32_t nw64) {
    static const int want = env_int("LTLG_STREAM_TABLE", -1);
    if (want == 0) return 0;
    const int fmt = entry_format(props);
    if (split64_table_bytes(props, nw64) <= kMaxSmemTable) return 1;
    if (split64_x_offset(fmt, nw64) <= kMaxSmemTable) return 2;
    return 0;
}

template <int FMT, typename SW, int TABLOC, int NT>
static cudaError_t launch_stream64_v(const LaunchArgs& a, cudaStream_t st) {
    const uint32_t tab_bytes = static_cast<uint32_t>(split64_table_bytes(a.props, a.nw64));
    const uint32_t smem = TABLOC == 1 ? tab_bytes : TABLOC == 2 ? split64_x_offset(FMT, a.nw64) : 0u;
    auto kern = label_stream64_kernel<FMT, SW, TABLOC, NT>;
    const uint64_t* P64 = reinterpret_cast<const uint64_t*>(a.P32);
    if constexpr (TABLOC != 0) {
        static uint64_t attr_set = 0;  // per device
        int dev = 0;
        cudaGetDevice(&dev);
        if (!(attr_set >> dev & 1u)) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kMaxSmemTable));
            attr_set |= 1ull << dev;
        }
        if (smem % 16u || smem > kMaxSmemTable) return cudaErrorInvalidValue;
        // programmatic dependent launch: the CTAs get resident while the
        // summary kernel finishes; they wait on it (griddepcontrol.wait) first
        cudaLaunchConfig_t cfg{};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = a.pdl ? 1 : 0;
        cfg.gridDim = dim3(static_cast<unsigned>(sm_count()));
        cfg.blockDim = dim3(NT);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kern, a.t64, a.task_byte64, a.task_n64, a.task_row, a.task_begin, a.ntasks,
                                  a.task_ctr, a.sf, tab_bytes, a.s_only, P64, a.nw64, static_cast<SW*>(a.out),
                                  a.ostride ? a.ostride : 1u);
    } else {
        static int per_sm = 0;
        if (!per_sm) {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, 0);
            if (per_sm <= 0) per_sm = 4;
        }
        kern<<<sm_count() * per_sm, NT, 0, st>>>(a.t64, a.task_byte64, a.task_n64, a.task_row, a.task_begin, a.ntasks,
                                                 a.task_ctr, a.sf, tab_bytes, a.s_only, P64, a.nw64,
                                                 static_cast<SW*>(a.out), a.ostride ? a.ostride : 1u);
    }
    return cudaSuccess;
}

template <int FMT, typename SW>
static cudaError_t launch_stream64_t(const LaunchArgs& a, cudaStream_t st) {
    // u64 labels: 24 warps per SM at 75 registers (no spills); 32 warps would
    // need <= 64 and spill (cfg-5 shard: 512 threads 0.373 of HBM, 768 0.417,
    // 1024 0.380).  Dev knob LTLG_NT64 = 512 / 1024 for A/B runs.
    if constexpr (FMT == 64) {
        static const int nt64 = env_int("LTLG_NT64", 768);
        const int loc = stream64_table_loc(a.props, a.nw64);
        if (loc == 0) return launch_stream64_v<FMT, SW, 0, 256>(a, st);
        if (nt64 == 512) return loc == 1 ? launch_stream64_v<FMT, SW, 1, 512>(a, st) : launch_stream64_v<FMT, SW, 2, 512>(a, st);
        if (nt64 == 1024)
            return loc == 1 ? launch_stream64_v<FMT, SW, 1, 1024>(a, st) : launch_stream64_v<FMT, SW, 2, 1024>(a, st);
        return loc == 1 ? launch_stream64_v<FMT, SW, 1, 768>(a, st) : launch_stream64_v<FMT, SW, 2, 768>(a, st);
    } else {
        switch (stream64_table_loc(a.props, a.nw64)) {
            case 1: return launch_stream64_v<FMT, SW, 1, 1024>(a, st);
            case 2: return launch_stream64_v<FMT, SW, 2, 1024>(a, st);
            default: return launch_stream64_v<FMT, SW, 0, 256>(a, st);
        }
    }
}

struct E32 {
    uint32_t f, meta, pa_lo, pa_hi, pb_lo, pb_hi, s, pad;
};
__device__ __forceinline__ E32 ld_entry32(const E32* p) {
    E32 e;
    asm("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(e.f), "=r"(e.meta), "=r"(e.pa_lo), "=r"(e.pa_hi), "=r"(e.pb_lo), "=r"(e.pb_hi), "=r"(e.s), "=r"(e.pad)
        : "l"(p));
    return e;
}

template <typename SW, int FPL, bool FULL>
__global__ void __launch_bounds__(256)
    label_batch64_kernel(const uint64_t* __restrict__ masks, const uint32_t* __restrict__ words,
                         const uint64_t* __restrict__ task_pair, const uint32_t* __restrict__ task_row,
                         uint32_t task_begin, uint32_t ntasks, uint32_t* __restrict__ task_ctr,
                         const uint4* __restrict__ tab, const uint64_t* __restrict__ pbt,
                         const uint32_t* __restrict__ s_only, const uint64_t* __restrict__ P64, uint32_t nw64,
                         int props, int frames, const uint32_t* __restrict__ perm, SW* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const uint64_t frame_stride = static_cast<uint64_t>(props) * nw64;
    const E32* lane_tab = reinterpret_cast<const E32*>(tab) + lane;
    (void)pbt;
    const uint32_t* lane_s = s_only + lane;
    bool fv[FPL];
#pragma unroll
    for (int q = 0; q < FPL; ++q) fv[q] = FULL || lane + 32 * q < frames;

    for (;;) {
        uint32_t t = 0;
        if (lane == 0) t = task_begin + atomicAdd(task_ctr, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= ntasks) break;
        const uint64_t p0 = task_pair[t], p1 = task_pair[t + 1];
        const int64_t r0 = task_row[t];
        int64_t row = r0 - 1;
        uint32_t acc[FPL];
#pragma unroll
        for (int q = 0; q < FPL; ++q) acc[q] = 0;
        auto store = [&](int64_t r) {
            SW* o = out + static_cast<uint64_t>(perm[r]) * frames + lane;
#pragma unroll
            for (int q = 0; q < FPL; ++q)
                if (fv[q]) o[32 * q] = static_cast<SW>(acc[q]);
        };
        auto pair_step = [&](uint32_t mlo, uint32_t mhi, uint32_t wh) {
            if (wh & kHead) {  // warp-uniform
                if (row >= r0) store(row);
                ++row;
#pragma unroll
                for (int q = 0; q < FPL; ++q) acc[q] = 0;
            }
            const uint32_t w = wh & kWordMask;
            const uint32_t off = w * static_cast<uint32_t>(frames);
            if ((mlo & mhi) == 0xffffffffu) {  // warp-uniform: the whole 64-cell word is swept
                const uint32_t* sp = index_wide(lane_s, off);
#pragma unroll
                for (int q = 0; q < FPL; ++q)
                    if (fv[q]) acc[q] |= __ldg(sp + 32 * q);
                return;
            }
            const E32* ep = index_wide(lane_tab, off);
#pragma unroll
            for (int q = 0; q < FPL; ++q) {
                if (!fv[q]) continue;
                const E32 e = ld_entry32(ep + 32 * q);
                uint32_t v = e.f;
                if ((mlo & e.pa_lo) | (mhi & e.pa_hi)) v |= __funnelshift_l(0u, 1u, e.meta);
                if ((mlo & e.pb_lo) | (mhi & e.pb_hi)) v |= __funnelshift_l(0u, 1u, e.meta >> 8);
                {
                    if (e.meta & kOver64) {  // a third partial prop: exact gather of the rest
                        const uint32_t known = e.f | (1u << (e.meta & 31)) | (1u << (e.meta >> 8 & 31));
                        uint32_t rest = e.s & ~known & ~acc[q];
                        const uint64_t m = (static_cast<uint64_t>(mhi) << 32) | mlo;
                        const uint64_t* col0 = P64 + static_cast<uint64_t>(lane + 32 * q) * frame_stride + w;
                        while (rest) {
                            const int j = __ffs(rest) - 1;
                            if (m & __ldg(col0 + static_cast<uint64_t>(j) * nw64)) v |= 1u << j;
                            rest &= rest - 1;
                        }
                    }
                }
                acc[q] |= v;
            }
        };
        uint2 cm = __ldg(reinterpret_cast<const uint2*>(masks + p0 + lane));
        uint32_t cw = __ldg(words + p0 + lane);
        for (uint64_t c = p0; c < p1; c += 32) {
            uint2 nm = cm;
            uint32_t nwd = cw;
            if (c + 32 < p1) {
                nm = __ldg(reinterpret_cast<const uint2*>(masks + c + 32 + lane));
                nwd = __ldg(words + c + 32 + lane);
            }
            const int n = static_cast<int>(p1 - c < 32 ? p1 - c : 32);
            for (int i = 0; i < n; ++i)
                pair_step(__shfl_sync(0xffffffffu, cm.x, i), __shfl_sync(0xffffffffu, cm.y, i),
                          __shfl_sync(0xffffffffu, cw, i));
            cm = nm;
            cw = nwd;
        }
        if (row >= r0) store(row);
    }
}

template <typename SW, int FPL, bool FULL>
static void launch_batch64_t(const LaunchArgs& a, cudaStream_t st) {
    static int per_sm = 0;
    auto kern = label_batch64_kernel<SW, FPL, FULL>;
    if (!per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
        if (per_sm <= 0) per_sm = 4;
    }
    kern<<<sm_count() * per_sm, 256, 0, st>>>(a.mask_b64, a.word_b64, a.task_pair_b64, a.task_row, a.task_begin, a.ntasks,
                                              a.task_ctr, static_cast<const uint4*>(a.sf), a.pb64,
                                              static_cast<const uint32_t*>(a.s_only),
                                              reinterpret_cast<const uint64_t*>(a.P32), a.nw64, a.props, a.frames,
                                              a.perm, static_cast<SW*>(a.out));
}

template <typename SW>
static void launch_batch64_fpl(const LaunchArgs& a, cudaStream_t st) {
    if (a.frames == 32) launch_batch64_t<SW, 1, true>(a, st);
    else if (a.frames == 64) launch_batch64_t<SW, 2, true>(a, st);
    else if (a.frames == 128) launch_batch64_t<SW, 4, true>(a, st);
    else if (a.frames < 32) launch_batch64_t<SW, 1, false>(a, st);
    else if (a.frames < 64) launch_batch64_t<SW, 2, false>(a, st);
    else if (a.frames < 128) launch_batch64_t<SW, 4, false>(a, st);
    else launch_batch64_t<SW, 8, false>(a, st);
}

cudaError_t launch_summary_b64(const uint64_t* P64, int props, int frames, uint32_t nw64, uint64_t cells, void* tab,
                               uint64_t* pbt, void* s_only, uint32_t* task_ctr, int nctr, cudaStream_t st) {
    const uint32_t nthreads = nw64 + 1 > static_cast<uint32_t>(nctr) ? nw64 + 1 : static_cast<uint32_t>(nctr);
    dim3 grid((nthreads + 255) / 256, static_cast<unsigned>(frames));
    summary_b64_kernel<<<grid, 256, 0, st>>>(P64, props, frames, nw64, cells, static_cast<uint4*>(tab), pbt,
                                             static_cast<uint32_t*>(s_only), task_ctr, nctr);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Prop-lane multi-frame path (<= 64 props, <= 64 frames): lane l owns
// propositions l and (PW = 2, > 32 props) l + 32, each with a 64-bit mask
// over the frames.  Per 64-cell word w, with pw = 32 * PW prop slots:
//   ffr[w * pw + j]  frames where P_j[w] covers the word  (hit for any mask)
//   sfr[w * pw + j]  frames where P_j[w] != 0            (hit for a full mask)
//   rec[rec_se[w].x .. rec_se[w].y)  one record per partial (frame, prop):
//        {P_j^f[w] lo, hi, byte offset of accumulator word f + 64 (j / 32),
//         1 << (j % 32)}
//        grouped by prop, so the 32 records one probe round reads mostly
//        name distinct frames (distinct shared-memory words, no same-address
//        serialisation of the ORs)
// A pair (m, w) ORs ffr into its lanes and probes the word's records with
// all 32 lanes, OR-ing hits (j, f) into a per-warp shared-memory label
// accumulator acc[f] |= 1 << j; at each row end a 32x32 bit transpose turns
// the prop-major ffr masks into frame-major ones (lane f holds frame f and
// f + 32) and ORs in acc[f].
// ---------------------------------------------------------------------------
// The prop-lane summary in one kernel.  A CTA owns WPB consecutive words x
// all 1 << pshift prop slots (thread j * WPB + wl: consecutive threads read
// consecutive words of one prop, coalesced).  Per word, the partial-record
// counts of its props are prefix-summed in shared memory and the word's
// record segment is taken from one global cursor (segments land in any word
// order; records stay grouped by prop, in prop order).  Each thread then
// re-reads its P words (now in L1/L2) and writes its records.
template <int PSHIFT, int NT>
__global__ void __launch_bounds__(NT) pl_build_kernel(const uint64_t* __restrict__ P64, int props, int frames,
                                                        uint32_t nw64, uint64_t cells, uint64_t* __restrict__ ffr,
                                                        uint64_t* __restrict__ sfr, uint2* __restrict__ rec_se,
                                                        uint32_t* __restrict__ rec_cursor, uint4* __restrict__ rec,
                                                        uint32_t* __restrict__ task_ctr, int nctr,
                                                        const uint32_t* __restrict__ touched64,
                                                        uint4* __restrict__ wdat) {
    constexpr int NP = 1 << PSHIFT, WPB = NT / NP;
    // a programmatically dependent labeling launch may get resident now; it
    // waits for this grid's completion before reading our outputs
    asm volatile("griddepcontrol.launch_dependents;");
    __shared__ uint32_t s_cnt[NP][WPB];
    __shared__ uint32_t s_base[WPB];
    __shared__ uint32_t s_full[WPB][2];  // (wdat) props full in frame 0, per word
    if (threadIdx.x < 2 * WPB) (&s_full[0][0])[threadIdx.x] = 0;
    const uint32_t gt = blockIdx.x * static_cast<uint32_t>(NT) + threadIdx.x;
    if (gt < static_cast<uint32_t>(nctr)) task_ctr[gt] = 0;
    const uint32_t j = threadIdx.x / WPB, wl = threadIdx.x % WPB;
    const uint32_t w = blockIdx.x * WPB + wl;
    const bool in = w <= nw64;  // word nw64 is the zero sentinel
    const bool live = in && w < nw64 && static_cast<uint64_t>(w) * 64 < cells && j < static_cast<uint32_t>(props) &&
                      !(touched64 && !(__ldg(touched64 + (w >> 5)) >> (w & 31) & 1u));
    const uint64_t lo = static_cast<uint64_t>(w) * 64;
    const uint64_t valid = !live ? 0ull : (cells - lo >= 64) ? ~0ull : ((1ull << (cells - lo)) - 1ull);
    const uint64_t* base = P64 + static_cast<uint64_t>(j) * nw64 + w;
    const uint64_t fstride = static_cast<uint64_t>(props) * nw64;
    uint64_t full = 0, any = 0;
    uint32_t n = 0;
    if (live) {
        for (int f = 0; f < frames; ++f) {
            const uint64_t x = base[static_cast<uint64_t>(f) * fstride] & valid;
            any |= static_cast<uint64_t>(x != 0) << f;
            full |= static_cast<uint64_t>(x == valid) << f;
            n += (x != 0 && x != valid);
        }
    }
    if (in) {
        const uint64_t o = (static_cast<uint64_t>(w) << PSHIFT) | j;
        ffr[o] = full;
        sfr[o] = any;
    }
    s_cnt[j][wl] = n;
    __syncthreads();  // (also orders the s_full zeroing before the ORs)
    if (wdat) {  // one frame: the word's full-prop mask (label_wm1_kernel)
        if (full & 1u) atomicOr(&s_full[wl][j >> 5], 1u << (j & 31));
        __syncthreads();
    }
    if (j == 0 && in) {  // per word: exclusive prefix over props, then its segment
        uint32_t run = 0;
        for (int k = 0; k < NP; ++k) {
            const uint32_t c = s_cnt[k][wl];
            s_cnt[k][wl] = run;
            run += c;
        }
        const uint32_t b = run ? atomicAdd(rec_cursor, run) : 0u;
        s_base[wl] = b;
        rec_se[w] = make_uint2(b, b + run);
        if (wdat) {  // {full lo, full hi, record range}, then the first record (below; none: zero)
            wdat[2 * static_cast<uint64_t>(w)] = make_uint4(s_full[wl][0], s_full[wl][1], b, b + run);
            if (!run) wdat[2 * static_cast<uint64_t>(w) + 1] = make_uint4(0u, 0u, 0u, 0u);
        }
    }
    __syncthreads();
    if (!n) return;
    uint32_t pos = s_base[wl] + s_cnt[j][wl];
    for (int f = 0; f < frames; ++f) {
        const uint64_t x = base[static_cast<uint64_t>(f) * fstride] & valid;
        if (x != 0 && x != valid) {  // smem label accumulator word f + 64 (j / 32), bit j % 32
            const uint4 r = make_uint4(static_cast<uint32_t>(x), static_cast<uint32_t>(x >> 32),
                                       4u * (static_cast<uint32_t>(f) + 64u * (j >> 5)), 1u << (j & 31));
            if (wdat && pos == s_base[wl]) wdat[2 * static_cast<uint64_t>(w) + 1] = r;  // (one frame: the word's first)
            rec[pos++] = r;
        }
    }
}

// The word-major kernel's per-submit summary, one pass (label_wm_kernel).
// A CTA owns WPB consecutive grid words x all 1 << PSHIFT prop slots (thread
// j * WPB + wl: consecutive threads read consecutive words of one prop).  Per
// grid word w and prop half h (props 32 h .. 32 h + 31) it writes
//   ffrT[w][h][f]         bit j % 32 for every prop j of the half that is
//                         full on w in frame f (frame-major);
//   wpair[w][h][k]        the two frames lane k of the labelling warp owns,
//                         fa | fb << 8.  Frames f and f + 32 go to different
//                         lanes' (fa and fb) sides, so a warp's 32 fa (and 32
//                         fb) accumulator words are distinct banks; the sides
//                         are paired busiest-with-idlest by partial-record
//                         count, which evens the records per lane;
//   lane records          one 16-B record {P lo, P hi, wlo, whi} per partial
//                         (frame f, prop j), in the lane that owns f, at slot
//                         row (records of fa first, then of fb); wlo = 1 << j % 32
//                         if f = fa, whi if f = fb.  Half h fills ns[h] slot
//                         rows of 32 records (ns = the largest per-lane count;
//                         holes are zero records, which never hit);
//   whdr[w]               {first slot row, ns[0] | ns[1] << 16}.
template <int PSHIFT, int NT>
__global__ void __launch_bounds__(NT) wm_build_kernel(const uint64_t* __restrict__ P64, int props, int frames,
                                                        uint32_t nw64, uint64_t cells, uint32_t* __restrict__ ffrT,
                                                        uint2* __restrict__ whdr,
                                                        uint16_t* __restrict__ wpair, uint32_t* __restrict__ row_cursor,
                                                        uint4* __restrict__ lrec, uint32_t* __restrict__ task_ctr,
                                                        int nctr, const uint32_t* __restrict__ touched64) {
    constexpr int NP = 1 << PSHIFT, WPB = NT / NP, NH = NP / 32;
    constexpr int TW = 64 * NH;  // frame-major u32 words per grid word: [prop half][frame]
    __shared__ uint32_t s_fT[WPB][TW];
    __shared__ uint32_t s_cnt[WPB][NH][64];  // partial records per frame, then the frame's next slot
    __shared__ uint16_t s_own[WPB][NH][64];   // frame -> owning lane | first slot << 8
    __shared__ uint32_t s_row[WPB][NH];       // first slot row of each (word, half)
    __shared__ uint32_t s_nrows[WPB];         // slot rows of each word
    for (int k = threadIdx.x; k < WPB * TW; k += NT) {
        (&s_fT[0][0])[k] = 0;
        (&s_cnt[0][0][0])[k] = 0;
    }
    const uint32_t gt = blockIdx.x * static_cast<uint32_t>(NT) + threadIdx.x;
    if (gt < static_cast<uint32_t>(nctr)) task_ctr[gt] = 0;
    const uint32_t w0 = blockIdx.x * WPB;
    if (touched64 && w0 < nw64) {  // no pair of the shard is on any of this CTA's words: nothing reads them
        static_assert(32 % WPB == 0, "a CTA's words in one touched64 word");
        const uint32_t tw = __ldg(touched64 + (w0 >> 5)) >> (w0 & 31);
        if ((WPB == 32 ? tw : tw & ((1u << (WPB & 31)) - 1u)) == 0u) return;
    }
    const uint32_t j = threadIdx.x / WPB, wl = threadIdx.x % WPB, h = j >> 5;
    const uint32_t w = w0 + wl;
    const bool in = w <= nw64;  // word nw64 is the zero sentinel
    const bool live = in && w < nw64 && static_cast<uint64_t>(w) * 64 < cells && j < static_cast<uint32_t>(props) &&
                      !(touched64 && !(__ldg(touched64 + (w >> 5)) >> (w & 31) & 1u));
    const uint64_t lo = static_cast<uint64_t>(w) * 64;
    const uint64_t valid = !live ? 0ull : (cells - lo >= 64) ? ~0ull : ((1ull << (cells - lo)) - 1ull);
    const uint64_t* base = P64 + static_cast<uint64_t>(j) * nw64 + w;
    const uint64_t fstride = static_cast<uint64_t>(props) * nw64;
    __syncthreads();  // (the zeroing before the ORs)
    uint64_t part = 0;
    if (live) {
        const uint32_t bit = 1u << (j & 31);
        for (int f0 = 0; f0 < frames; f0 += 16) {  // 16 loads in flight, then their updates
            uint64_t xs[16];
#pragma unroll
            for (int u = 0; u < 16; ++u)
                xs[u] = f0 + u < frames ? __ldg(base + static_cast<uint64_t>(f0 + u) * fstride) & valid : 0ull;
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int f = f0 + u;
                if (f >= frames) break;
                if (xs[u] == valid) atomicOr(&s_fT[wl][64 * h + f], bit);
                if (xs[u] != 0 && xs[u] != valid) {
                    part |= 1ull << f;
                    atomicAdd(&s_cnt[wl][h][f], 1u);
                }
            }
        }
    }
    __syncthreads();
    static_assert(WPB * NH == NT / 32, "one warp per (word, prop half)");
    {  // warp q * NH + hh: the frame pairing of (word q, half hh); lane r holds residue r
        const uint32_t wq = threadIdx.x >> 5, r = threadIdx.x & 31;
        const uint32_t q = wq / NH, hh = wq % NH;
        uint32_t* c = s_cnt[q][hh];
        // side a = the busier of frames (r, r + 32), side b the other
        const uint32_t c0 = c[r], c1 = c[r + 32];
        const uint32_t fa = c1 > c0 ? r + 32 : r, fb = c1 > c0 ? r : r + 32;
        const uint32_t ca = max(c0, c1), cb = min(c0, c1);
        // ranks: a by count descending, b ascending (ties by residue)
        uint32_t ra = 0, rb = 0;
        for (int k = 0; k < 32; ++k) {
            const uint32_t xa = __shfl_sync(0xffffffffu, ca, k), xb = __shfl_sync(0xffffffffu, cb, k);
            ra += (xa > ca) || (xa == ca && static_cast<uint32_t>(k) < r);
            rb += (xb < cb) || (xb == cb && static_cast<uint32_t>(k) < r);
        }
        uint16_t* own = s_own[q][hh];  // (scratch first: own[rank] = a frame, own[32 + rank] = b frame)
        own[ra] = static_cast<uint16_t>(fa);
        own[32 + rb] = static_cast<uint16_t>(fb);
        __syncwarp();
        const uint32_t ka = own[r], kb = own[32 + r];  // lane r's pair: a of rank r, b of rank r
        const uint32_t na = c[ka], nb = c[kb];
        __syncwarp();
        own[ka] = static_cast<uint16_t>(r);                   // lane | side << 5 | first slot << 8
        own[kb] = static_cast<uint16_t>(r | 32u | na << 8);
        c[ka] = 0;  // the frame's next slot
        c[kb] = na;
        uint32_t ns = na + nb;
        for (int d = 16; d; d >>= 1) ns = max(ns, __shfl_xor_sync(0xffffffffu, ns, d));
        const uint32_t ww = blockIdx.x * WPB + q;
        if (ww <= nw64) wpair[(static_cast<uint64_t>(ww) * NH + hh) * 32 + r] = static_cast<uint16_t>(ka | kb << 8);
        if (r == 0) s_row[q][hh] = ns;  // (counts for now)
    }
    __syncthreads();
    if (threadIdx.x < WPB) {  // per word: its segment of slot rows
        const uint32_t ww = blockIdx.x * WPB + threadIdx.x;
        uint32_t ns[NH], run = 0;
#pragma unroll
        for (int hh = 0; hh < NH; ++hh) {
            ns[hh] = s_row[threadIdx.x][hh];
            run += ns[hh];
        }
        const uint32_t r0 = run ? atomicAdd(row_cursor, run) : 0u;
        s_nrows[threadIdx.x] = run;
        uint32_t acc = r0;
#pragma unroll
        for (int hh = 0; hh < NH; ++hh) {
            s_row[threadIdx.x][hh] = acc;
            acc += ns[hh];
        }
        if (ww <= nw64) whdr[ww] = make_uint2(r0, ns[0] | (NH > 1 ? ns[NH - 1] << 16 : 0u));
    }
    __syncthreads();
    // the frame-major summary (coalesced rows of TW words per grid word), and
    // zero records over every slot row of the CTA's words (the holes)
    for (int k = threadIdx.x; k < WPB * TW; k += NT) {
        const uint32_t ww = blockIdx.x * WPB + static_cast<uint32_t>(k / TW);
        if (ww <= nw64) ffrT[static_cast<uint64_t>(ww) * TW + k % TW] = (&s_fT[0][0])[k];
    }
    for (int q = 0; q < WPB; ++q) {
        if (blockIdx.x * WPB + q > nw64) break;
        for (uint32_t k = threadIdx.x; k < s_nrows[q] * 32; k += NT)
            lrec[static_cast<uint64_t>(s_row[q][0]) * 32 + k] = make_uint4(0u, 0u, 0u, 0u);
    }
    __syncthreads();
    const uint32_t bit = 1u << (j & 31);
    for (uint64_t x = part; x;) {  // the partial frames, 4 loads in flight at a time
        int fs[4];
        uint64_t ps[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            fs[u] = x ? __ffsll(static_cast<long long>(x)) - 1 : -1;
            x &= x - 1;
            ps[u] = fs[u] >= 0 ? __ldg(base + static_cast<uint64_t>(fs[u]) * fstride) & valid : 0ull;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (fs[u] < 0) break;
            const uint32_t o = s_own[wl][h][fs[u]], side_b = o & 32u;
            const uint32_t slot = atomicAdd(&s_cnt[wl][h][fs[u]], 1u);
            lrec[(static_cast<uint64_t>(s_row[wl][h]) + slot) * 32 + (o & 31u)] =
                make_uint4(static_cast<uint32_t>(ps[u]), static_cast<uint32_t>(ps[u] >> 32), side_b ? 0u : bit,
                           side_b ? bit : 0u);
        }
    }
}

#if LTLG_AB_BUILD  // pair-major prop-lane kernel (A/B knob LTLG_WORDMAJOR=0)
// 32x32 bit transpose across the warp: in, lane l holds row l; out, lane l
// holds column l (bit r = row r's bit l).
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
    const uint32_t masks[5] = {0x0000ffffu, 0x00ff00ffu, 0x0f0f0f0fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const int d = 16 >> i;
        const uint32_t m = masks[i];
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, d);
        x = (lane & d) ? ((x & ~m) | ((y >> d) & m)) : ((x & m) | ((y << d) & ~m));
    }
    return x;
}

template <typename SW, int PW>
__global__ void __launch_bounds__(256)
    label_pl_kernel(const uint64_t* __restrict__ masks, const uint32_t* __restrict__ words,
                    const uint64_t* __restrict__ task_pair, const uint32_t* __restrict__ task_row, uint32_t task_begin,
                    uint32_t ntasks, uint32_t* __restrict__ task_ctr, const uint64_t* __restrict__ ffr,
                    const uint64_t* __restrict__ sfr, const uint2* __restrict__ rec_se,
                    const uint4* __restrict__ rec, int frames, const uint32_t* __restrict__ perm,
                    SW* __restrict__ out, uint32_t ostride) {
    // per warp: partial-record hits, one 32-bit prop mask per frame (a native
    // shared-memory OR; 64-bit ones are CAS loops)
    // (PW = 2: words 64..127 hold props 32..63)
    __shared__ uint32_t s_acc[8][64 * PW];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint32_t* sacc = s_acc[wib];
    const uint32_t sacc_s = smem_u32(sacc);
#pragma unroll
    for (int k = 0; k < 2 * PW; ++k) sacc[lane + 32 * k] = 0;
    __syncwarp();
    const uint4* lane_rec = rec + lane;
    const uint64_t* lane_ffr = ffr + lane;
    const uint64_t* lane_sfr = sfr + lane;
    constexpr uint32_t kPw = 32u * PW;  // prop slots per word in ffr / sfr
    for (;;) {
        uint32_t t = 0;
        if (lane == 0) t = task_begin + atomicAdd(task_ctr, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= ntasks) break;
        const uint64_t p0 = task_pair[t], p1 = task_pair[t + 1];
        const int64_t r0 = task_row[t];
        int64_t row = r0 - 1;
        uint64_t acc = 0;   // frames where prop `lane` covers a swept word of the open row
        uint64_t acc2 = 0;  // (PW = 2) the same for prop lane + 32
        auto store = [&](int64_t r) {
            __syncwarp();
            const uint32_t lo = transpose32(static_cast<uint32_t>(acc), lane) | sacc[lane];  // frame lane
            const uint32_t hi = transpose32(static_cast<uint32_t>(acc >> 32), lane) | sacc[lane + 32];  // frame lane + 32
            SW* o = out + static_cast<uint64_t>(perm[r]) * ostride;
            if constexpr (PW == 2) {
                const uint32_t lo2 = transpose32(static_cast<uint32_t>(acc2), lane) | sacc[lane + 64];
                const uint32_t hi2 = transpose32(static_cast<uint32_t>(acc2 >> 32), lane) | sacc[lane + 96];
                if (lane < frames) o[lane] = static_cast<SW>((static_cast<uint64_t>(lo2) << 32) | lo);
                if (lane + 32 < frames) o[lane + 32] = static_cast<SW>((static_cast<uint64_t>(hi2) << 32) | hi);
            } else {
                if (lane < frames) o[lane] = static_cast<SW>(lo);
                if (lane + 32 < frames) o[lane + 32] = static_cast<SW>(hi);
            }
#pragma unroll
            for (int k = 0; k < 2 * PW; ++k) sacc[lane + 32 * k] = 0;
            __syncwarp();
        };
        uint2 cm = __ldg(reinterpret_cast<const uint2*>(masks + p0 + lane));
        uint32_t cw = __ldg(words + p0 + lane);
        for (uint64_t c = p0; c < p1; c += 32) {
            uint2 nm = cm;
            uint32_t nwd = cw;
            if (c + 32 < p1) {
                nm = __ldg(reinterpret_cast<const uint2*>(masks + c + 32 + lane));
                nwd = __ldg(words + c + 32 + lane);
            }
            const int n = static_cast<int>(p1 - c < 32 ? p1 - c : 32);
            // lane i fetches the record range of pair i once per chunk (the
            // words arrived with the previous chunk's prefetch)
            const uint2 cse = __ldg(rec_se + (lane < n ? (cw & kWordMask) : 0u));
            for (int i = 0; i < n; ++i) {
                const uint32_t mlo = __shfl_sync(0xffffffffu, cm.x, i), mhi = __shfl_sync(0xffffffffu, cm.y, i);
                const uint32_t wh = __shfl_sync(0xffffffffu, cw, i);
                if (wh & kHead) {  // warp-uniform
                    if (row >= r0) store(row);
                    ++row;
                    acc = 0;
                    acc2 = 0;
                }
                const uint32_t w = wh & kWordMask;
                if ((mlo & mhi) == 0xffffffffu) {  // the whole 64-cell word is swept: every nonzero frame hits
                    acc |= __ldg(index_wide(lane_sfr, w * kPw));
                    if constexpr (PW == 2) acc2 |= __ldg(index_wide(lane_sfr, w * kPw + 32u));
                    continue;
                }
                acc |= __ldg(index_wide(lane_ffr, w * kPw));
                if constexpr (PW == 2) acc2 |= __ldg(index_wide(lane_ffr, w * kPw + 32u));
                const uint2 se = make_uint2(__shfl_sync(0xffffffffu, cse.x, i), __shfl_sync(0xffffffffu, cse.y, i));
                // all lanes probe 32 records at a time (the array is padded, so
                // reading past the word's last record is harmless)
                for (uint32_t q = se.x; q < se.y; q += 32) {
                    const uint4 r = __ldg(index_wide(lane_rec, q));
                    const bool hit = (q + lane < se.y) && ((mlo & r.x) | (mhi & r.y));
                    if (hit) asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(sacc_s + r.z), "r"(r.w) : "memory");
                }
            }
            cm = nm;
            cw = nwd;
        }
        if (row >= r0) store(row);
    }
}

#endif  // LTLG_AB_BUILD

// ---------------------------------------------------------------------------
// Word-major multi-frame labelling (<= 64 frames per launch, <= 64 props).
//
// A CTA task is a run of <= R consecutive rows of the batch order (z-sorted,
// so they sweep a compact region of the grid), with the rows' 64-cell pairs
// grouped by word (PackedShard::wm_*).  The CTA's warps take the task's word
// groups from a shared-memory counter.  Lane k owns two frames of the word,
// fa and fb (wm_build_kernel's wpair), and two accumulator words per row and
// prop half.  Per group a warp reads, once, the word's full-prop masks of the
// lane's frames (ffrT) and the lane's partial records (slot rows of 32: each
// lane's own records of fa / fb, {P lo, P hi, bit if fa, bit if fb}), into
// registers, then streams the group's pairs (staged 32 at a time in the
// warp's shared-memory slice, one broadcast 16-B read each) past them:
// v_fa = full props | bits of the records with m & P != 0 (two LOP3s and a
// predicated add per record: see rec_test)
// (likewise v_fb), and one red.shared.or per accumulator word.  Every lane
// ORs into its own frame's word, so the 32 lanes hit 32 distinct banks.
// acc is the CTA's shared-memory label block, frame-major per row (several
// warps may OR into one row: the reductions are atomic), so the row-end
// stores are coalesced 4-byte words (lane f = frame f) with no bit transpose.
// The pair-major label_pl_kernel re-read each pair's word summary (256 B)
// and records (~600 B) from L1 for every pair and scattered its record hits
// with bank-conflicting atomics; here a word's data is read once per task and
// amortised over its pairs (~26 per group at R = 128 on config 4).
// ---------------------------------------------------------------------------
constexpr int kWmThreads = 256;
constexpr int kWmMaxRows = 256;  // rows per task at most (PackedShard::wm_row is a byte)
constexpr int kWmSlots = 4;  // slot rows (per prop half) held in registers per word; more are re-read per pair

// v0 |= z and v1 |= w if (mlo & x) | (mhi & y) != 0: a record test.  A
// lane's records of one frame are distinct props, none of them full, so the
// bit z (w) is never already in v0 (v1) and the OR is an ADD: predicated
// adds, which ptxas issues as IMAD.IADD on the FMA pipe, leaving the ALU pipe
// (the kernel's binding one) the two LOP3s of the test
__device__ __forceinline__ void rec_test(uint32_t mlo, uint32_t mhi, const uint4& r, uint32_t& v0, uint32_t& v1) {
    asm("{\n\t.reg .pred p;\n\t.reg .b32 t, u;\n\t"
        "and.b32 t, %2, %4;\n\tand.b32 u, %3, %5;\n\tor.b32 t, t, u;\n\t"
        "setp.ne.u32 p, t, 0;\n\t@p add.u32 %0, %0, %6;\n\t@p add.u32 %1, %1, %7;\n\t}"
        : "+r"(v0), "+r"(v1)
        : "r"(mlo), "r"(mhi), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w));
}

// The pairs [e0, e1) of one word group against the word's summary (fv / sv:
// lane's frames fa, fb of each prop half) and its lane records: NS slot rows
// per half in registers (r0: half 0, r1: half 1); MORE: more rows than that,
// re-read per pair from lrec (rows [m0, m0 + mn0) of half 0, [m1, m1 + mn1)
// of half 1).  One red.shared.or per accumulator word (oa / ob: the lane's
// frames' byte offsets in a row) and pair.
template <int PW, int NS, bool MORE>
__device__ __forceinline__ void wm_group(const uint64_t* __restrict__ emask, const uint8_t* __restrict__ erow,
                                         uint32_t e0, uint32_t e1, const uint32_t (&fv)[2 * PW],
                                         const uint32_t (&off)[2 * PW],
                                         const uint4 (&r0)[kWmSlots], const uint4 (&r1)[kWmSlots], uint32_t ns0,
                                         uint32_t ns1, const uint4* __restrict__ lrec, uint32_t m0, uint32_t mn0,
                                         uint32_t m1, uint32_t mn1, uint32_t acc_s, uint32_t sp,
                                         const uint4* spp, int lane) {
    constexpr uint32_t RB = 64 * PW * 4;  // accumulator bytes per row
    for (uint32_t c = e0; c < e1; c += 32) {
        const uint2 cm = __ldg(reinterpret_cast<const uint2*>(emask + c + lane));
        const uint32_t cr = __ldg(erow + c + lane);
        const int n = static_cast<int>(e1 - c < 32u ? e1 - c : 32u);
        // the chunk's pairs {mask lo, mask hi, row byte offset} through the
        // warp's shared-memory slice: one broadcast 16-B read per pair
        __syncwarp();
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(sp + 16u * lane), "r"(cm.x), "r"(cm.y),
                     "r"(cr * RB), "r"(0u)
                     : "memory");
        __syncwarp();
        for (int i = 0; i < n; ++i) {
            const uint4 pq = spp[i];
            const uint32_t mlo = pq.x, mhi = pq.y, rowb = pq.z;
            // full props hit any pair; a partial prop hits iff one of its
            // records does (for a pair sweeping the whole word every record
            // hits, so no special case for it)
            uint32_t v[2 * PW];
#pragma unroll
            for (int k = 0; k < 2 * PW; ++k) v[k] = fv[k];
            {
                // (slot rows past a half's count hold zero records: no hit)
#pragma unroll
                for (int k = 0; k < NS; ++k) rec_test(mlo, mhi, r0[k], v[0], v[1]);
                if constexpr (PW == 2) {
#pragma unroll
                    for (int k = 0; k < NS; ++k) rec_test(mlo, mhi, r1[k], v[2], v[3]);
                }
                if constexpr (MORE) {
                    for (uint32_t q = 0; q < mn0; ++q)
                        rec_test(mlo, mhi, __ldg(lrec + static_cast<uint64_t>(m0 + q) * 32 + lane), v[0], v[1]);
                    if constexpr (PW == 2)
                        for (uint32_t q = 0; q < mn1; ++q)
                            rec_test(mlo, mhi, __ldg(lrec + static_cast<uint64_t>(m1 + q) * 32 + lane), v[2], v[3]);
                }
            }
#pragma unroll
            for (int k = 0; k < 2 * PW; ++k)  // (an OR of 0 is a no-op: no branch around it; the
                // accumulator block and the pair slice are disjoint, and __syncthreads
                // orders the reductions against the row stores)
                asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(rowb + off[k]), "r"(v[k]));
        }
    }
}

template <typename SW, int PW>
__global__ void __launch_bounds__(kWmThreads)
    label_wm_kernel(const uint64_t* __restrict__ emask, const uint8_t* __restrict__ erow,
                    const uint32_t* __restrict__ gword, const uint32_t* __restrict__ gstart,
                    const uint32_t* __restrict__ task_row, const uint32_t* __restrict__ task_grp,
                    uint32_t task_begin, uint32_t ntasks, uint32_t* __restrict__ task_ctr,
                    const uint32_t* __restrict__ ffrT, const uint2* __restrict__ whdr, const uint16_t* __restrict__ wpair,
                    const uint4* __restrict__ lrec, int frames, const uint32_t* __restrict__ perm,
                    SW* __restrict__ out, uint32_t ostride, int rows_per_task) {
    extern __shared__ uint32_t wm_acc[];
    __shared__ uint32_t s_task, s_group;
    __shared__ uint32_t s_perm[kWmMaxRows];  // the task's output rows (cp.async during the task)
    constexpr int RW = 64 * PW;  // accumulator words per row: [prop half][frame]
    constexpr int NW = kWmThreads / 32;
    __shared__ uint4 s_pair[NW][32];  // each warp's current chunk of pairs
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint32_t acc_s = smem_u32(wm_acc), sp = smem_u32(&s_pair[wib][0]);
    for (int k = threadIdx.x; k < rows_per_task * RW; k += kWmThreads) wm_acc[k] = 0;
    for (;;) {
        if (threadIdx.x == 0) {
            s_task = task_begin + atomicAdd(task_ctr, 1u);
            s_group = 0;
        }
        __syncthreads();
        const uint32_t t = s_task;
        if (t >= ntasks) break;
        const uint32_t r0 = task_row[t], nr = task_row[t + 1] - r0;
        const uint32_t g0 = task_grp[t], ng = task_grp[t + 1] - g0;
        if (threadIdx.x < nr)  // the store's row ids, fetched in the background (no register held)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(s_perm + threadIdx.x)),
                         "l"(perm + r0 + threadIdx.x)
                         : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
        for (;;) {
            uint32_t gi = 0;
            if (lane == 0) gi = atomicAdd(&s_group, 1u);
            gi = __shfl_sync(0xffffffffu, gi, 0);
            if (gi >= ng) break;
            const uint32_t g = g0 + gi;
            const uint32_t w = gword[g];
            const uint32_t e0 = gstart[g], e1 = gstart[g + 1];
            uint32_t fv[2 * PW], off[2 * PW];
#pragma unroll
            for (int hh = 0; hh < PW; ++hh) {  // the lane's two frames of each prop half
                const uint32_t pr = __ldg(wpair + (static_cast<uint64_t>(w) * PW + hh) * 32 + lane);
                off[2 * hh] = acc_s + 4u * (64u * hh + (pr & 0xffu));  // (shared-memory addresses in row 0)
                off[2 * hh + 1] = acc_s + 4u * (64u * hh + (pr >> 8));
            }
#pragma unroll
            for (int k = 0; k < 2 * PW; ++k) fv[k] = __ldg(ffrT + static_cast<uint64_t>(w) * RW + (off[k] - acc_s) / 4);
            const uint2 hd = __ldg(whdr + w);
            const uint32_t ns0 = hd.y & 0xffffu, ns1 = hd.y >> 16;
            uint4 ra[kWmSlots], rb[kWmSlots];
            const uint4* l0 = lrec + static_cast<uint64_t>(hd.x) * 32 + lane;
            const uint4* l1 = l0 + static_cast<uint64_t>(ns0) * 32;
#pragma unroll
            for (int k = 0; k < kWmSlots; ++k) {
                ra[k] = k < ns0 ? __ldg(l0 + 32 * k) : make_uint4(0u, 0u, 0u, 0u);
                rb[k] = (PW == 2 && k < ns1) ? __ldg(l1 + 32 * k) : make_uint4(0u, 0u, 0u, 0u);
            }
            const uint32_t mn0 = ns0 > kWmSlots ? ns0 - kWmSlots : 0u, mn1 = ns1 > kWmSlots ? ns1 - kWmSlots : 0u;
            const uint32_t m0 = hd.x + kWmSlots, m1 = hd.x + ns0 + kWmSlots;
            if (mn0 | mn1)
                wm_group<PW, kWmSlots, true>(emask, erow, e0, e1, fv, off, ra, rb, ns0, ns1, lrec, m0, mn0, m1, mn1, acc_s, sp, s_pair[wib], lane);
            else
                switch (ns0 > ns1 ? ns0 : ns1) {  // warp-uniform: one specialised pair loop per slot-row count
                    case 0: wm_group<PW, 0, false>(emask, erow, e0, e1, fv, off, ra, rb, ns0, ns1, lrec, m0, 0, m1, 0, acc_s, sp, s_pair[wib], lane); break;
                    case 1: wm_group<PW, 1, false>(emask, erow, e0, e1, fv, off, ra, rb, ns0, ns1, lrec, m0, 0, m1, 0, acc_s, sp, s_pair[wib], lane); break;
                    case 2: wm_group<PW, 2, false>(emask, erow, e0, e1, fv, off, ra, rb, ns0, ns1, lrec, m0, 0, m1, 0, acc_s, sp, s_pair[wib], lane); break;
                    case 3: wm_group<PW, 3, false>(emask, erow, e0, e1, fv, off, ra, rb, ns0, ns1, lrec, m0, 0, m1, 0, acc_s, sp, s_pair[wib], lane); break;
                    default: wm_group<PW, 4, false>(emask, erow, e0, e1, fv, off, ra, rb, ns0, ns1, lrec, m0, 0, m1, 0, acc_s, sp, s_pair[wib], lane); break;
                }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        // the task's rows: warp wib stores rows wib, wib + NW, ...; lane f
        // frames f and f + 32; then clears them
        for (uint32_t r = wib; r < nr; r += NW) {
            SW* o = out + static_cast<uint64_t>(s_perm[r]) * ostride;
            uint32_t* a = wm_acc + r * RW;
            uint64_t lo = a[lane], hi = a[lane + 32];
            if constexpr (PW == 2) {
                lo |= static_cast<uint64_t>(a[lane + 64]) << 32;
                hi |= static_cast<uint64_t>(a[lane + 96]) << 32;
            }
            if (lane < frames) o[lane] = static_cast<SW>(lo);
            if (lane + 32 < frames) o[lane + 32] = static_cast<SW>(hi);
#pragma unroll
            for (int k = 0; k < 2 * PW; ++k) a[lane + 32 * k] = 0;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Word-major single-frame labelling (<= 64 props): the word-major copy of T
// (PackedShard::wm_*) against the one-frame prop-lane summary (pl_build_kernel
// with frames = 1: wdat[w] = {full-prop mask lo, hi, record range}, then the
// word's first partial record {P lo, P hi, 4 * 64 * (j / 32), 1 << j % 32} or
// zeros).  A warp owns a task (<= R rows; its label words in the warp's slice
// of shared memory, one plane per prop half) and takes the task's word groups
// 32 at a time.  The batches' group starts and word data come by cp.async into
// two shared-memory buffers, one batch ahead (the next batch's word ids two
// ahead), so no dependent load chain sits between batches.  A task's batches
// are consecutive ranges of T, streamed as a software pipeline of iterations
// of kWm1U chunks of 32 pairs: the next iteration's masks and row-byte window
// (8-byte loads, staged through shared memory) are in flight while this one
// is processed, across batch boundaries too.  Lane i of a chunk finds its
// pair's group from the group starts in the chunk (one redux.sync.or + popc)
// and reads the word data from the buffer: v = full | the bits of the records
// whose P word meets the pair's mask, ORed into the row's label word(s).
// ---------------------------------------------------------------------------
constexpr int kWm1Warps = 8;
#ifndef WM1_U
#define WM1_U 4
#endif
#ifdef WM1_MINB
#define WM1_BOUNDS __launch_bounds__(kWm1Warps * 32, WM1_MINB)
#else
#define WM1_BOUNDS __launch_bounds__(kWm1Warps * 32)
#endif
constexpr int kWm1U = WM1_U;  // 32-pair chunks per iteration (two iterations in flight per warp)
constexpr int kWm1Rw = 4 * kWm1U + 1;  // u64 words of an iteration's row-byte window

__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

// MAXR: rows per task at most (128 or 256: the label block's size)
template <typename SW, int PW, int MAXR>
__global__ void WM1_BOUNDS
    label_wm1_kernel(const uint64_t* __restrict__ emask, const uint8_t* __restrict__ erow,
                     const uint32_t* __restrict__ gword, const uint32_t* __restrict__ gstart,
                     const uint32_t* __restrict__ task_row, const uint32_t* __restrict__ task_grp,
                     uint32_t task_begin, uint32_t ntasks, uint32_t* __restrict__ task_ctr,
                     const uint4* __restrict__ wdat, const uint4* __restrict__ rec,
                     const uint32_t* __restrict__ perm, SW* __restrict__ out, uint32_t ostride) {
    __shared__ uint32_t s_acc[kWm1Warps][MAXR * PW];
    __shared__ uint32_t s_perm[kWm1Warps][MAXR];
    __shared__ __align__(16) uint4 s_grp[kWm1Warps][2][32][2];  // per batch buffer: word data, first record
    __shared__ uint32_t s_gw[kWm1Warps][2][32];                 // word ids
    __shared__ uint32_t s_ge[kWm1Warps][2][33];                 // group starts + the batch's end
    __shared__ uint64_t s_rows[kWm1Warps][kWm1Rw];              // the iteration's row bytes
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint32_t* acc = s_acc[wib];
    for (int k = lane; k < MAXR * PW; k += 32) acc[k] = 0;
    const uint32_t acc_s = smem_u32(acc);
    const uint32_t le = 0xffffffffu >> (31 - lane);  // lanes 0..lane
    // a warp's first task is static (task_begin + its grid-wide warp index), so
    // its T-side data (row ids, group starts and word ids) is fetched before
    // the summary this kernel depends on is complete (programmatic dependent
    // launch); later tasks come from the counter the summary resets
    const uint32_t nwarps = gridDim.x * kWm1Warps;
    uint32_t t = task_begin + blockIdx.x * kWm1Warps + wib;
    for (bool first = true;; first = false) {
        if (!first) {
            if (lane == 0) t = task_begin + nwarps + atomicAdd(task_ctr, 1u);
            t = __shfl_sync(0xffffffffu, t, 0);
        }
        if (t >= ntasks) break;
        const uint32_t r0 = __ldg(task_row + t), nr = __ldg(task_row + t + 1) - r0;
        const uint32_t g0 = __ldg(task_grp + t), ng = __ldg(task_grp + t + 1) - g0;
        for (uint32_t r = lane; r < nr; r += 32)  // the store's row ids, in the background
            cp_async4(smem_u32(s_perm[wib] + r), perm + r0 + r);
        // batch gb's word ids and group starts into buffer bf
        auto fetch_starts = [&](int bf, uint32_t gb) {
            const uint32_t n = ng - gb < 32u ? ng - gb : 32u;
            if (static_cast<uint32_t>(lane) < n) {
                cp_async4(smem_u32(&s_gw[wib][bf][lane]), gword + g0 + gb + lane);
                cp_async4(smem_u32(&s_ge[wib][bf][lane]), gstart + g0 + gb + lane);
            }
            if (lane == 0) cp_async4(smem_u32(&s_ge[wib][bf][n]), gstart + g0 + gb + n);
        };
        // batch gb's word data into buffer bf (its word ids have landed)
        auto fetch_words = [&](int bf, uint32_t gb) {
            const uint32_t n = ng - gb < 32u ? ng - gb : 32u;
            if (static_cast<uint32_t>(lane) < n) {
                const uint4* src = wdat + 2 * static_cast<uint64_t>(s_gw[wib][bf][lane]);
                cp_async16(smem_u32(&s_grp[wib][bf][lane][0]), src);
                cp_async16(smem_u32(&s_grp[wib][bf][lane][1]), src + 1);
            }
        };
        fetch_starts(0, 0);
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (first) asm volatile("griddepcontrol.wait;" ::: "memory");  // (the summary's outputs from here on)
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        fetch_words(0, 0);
        if (ng > 32) fetch_starts(1, 32);
        asm volatile("cp.async.commit_group;" ::: "memory");
        constexpr int RWL = (kWm1Rw + 31) / 32;  // row-window words per lane
        // an iteration's T: kWm1U chunks of masks, and its row bytes as
        // 8-byte loads over the 8-aligned window (kWm1Rw words)
        auto load_it = [&](uint32_t c, uint32_t E1, uint2 (&m)[kWm1U], uint64_t (&rwv)[RWL]) {
#pragma unroll
            for (int u = 0; u < kWm1U; ++u) {
                const uint32_t e = c + 32u * u + lane;
                m[u] = e < E1 ? __ldg(reinterpret_cast<const uint2*>(emask + e)) : make_uint2(0u, 0u);
            }
            const uint32_t cb = c & ~7u;
            const uint64_t* rw = reinterpret_cast<const uint64_t*>(erow + cb);
#pragma unroll
            for (int k = 0; k < RWL; ++k) {
                const uint32_t i = 32u * k + lane;
                rwv[k] = i < static_cast<uint32_t>(kWm1Rw) && cb + 8u * i < E1 ? __ldg(rw + i) : 0ull;
            }
        };
        // software pipeline: the next iteration's loads are in flight
        // during this one's processing (across batches too: a task's
        // batches are consecutive ranges of T)
        uint2 mn[kWm1U];
        uint64_t rn[RWL];
        int bf = 0;
        for (uint32_t gb = 0; gb < ng; gb += 32, bf ^= 1) {
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncwarp();  // batch gb's starts and word data, batch gb + 32's starts
            const uint32_t n = ng - gb < 32u ? ng - gb : 32u;
            const uint32_t ek0 = static_cast<uint32_t>(lane) < n ? s_ge[wib][bf][lane] : 0xffffffffu;
            const uint32_t E0 = s_ge[wib][bf][0], E1 = s_ge[wib][bf][n];
            const uint32_t F1 = gb + 32 < ng ? s_ge[wib][bf ^ 1][ng - gb - 32 < 32u ? ng - gb - 32 : 32u] : E1;  // next batch's end
            if (gb == 0) load_it(E0, E1, mn, rn);
            __syncwarp();  // (buffer bf's starts are in registers before batch gb + 64's land there)
            if (gb + 32 < ng) fetch_words(bf ^ 1, gb + 32);
            if (gb + 64 < ng) fetch_starts(bf, gb + 64);
            asm volatile("cp.async.commit_group;" ::: "memory");
            const uint4(*grp)[2] = s_grp[wib][bf];
            uint32_t gcount = 0;  // groups of the batch started before the chunk
            for (uint32_t c = E0; c < E1; c += 32 * kWm1U) {
                uint2 m[kWm1U];
                uint64_t rwv[RWL];
#pragma unroll
                for (int u = 0; u < kWm1U; ++u) m[u] = mn[u];
#pragma unroll
                for (int k = 0; k < RWL; ++k) rwv[k] = rn[k];
                {  // the next iteration: this batch's, else the next batch's first
                    const bool in = c + 32 * kWm1U < E1;
                    const uint32_t nc = in ? c + 32 * kWm1U : E1, nb = in ? E1 : F1;
                    if (nc < nb) load_it(nc, nb, mn, rn);
                }
                const uint32_t cb = c & ~7u;
                __syncwarp();  // (the previous iteration's row reads are done)
#pragma unroll
                for (int k = 0; k < RWL; ++k)
                    if (32 * k + lane < kWm1Rw) s_rows[wib][32 * k + lane] = rwv[k];
                __syncwarp();
                const uint8_t* rows_b = reinterpret_cast<const uint8_t*>(s_rows[wib]) + (c - cb) + lane;
#pragma unroll
                for (int u = 0; u < kWm1U; ++u) {
                    const uint32_t cu = c + 32u * u;
                    if (cu >= E1) break;  // (warp-uniform)
                    const uint32_t rowu = rows_b[32 * u];
                    const uint32_t d = ek0 - cu;  // lane k's group starts in this chunk iff d < 32
                    const uint32_t starts = __reduce_or_sync(0xffffffffu, d < 32u ? 1u << d : 0u);
                    const int gi = static_cast<int>(gcount + __popc(starts & le)) - 1;
                    gcount += __popc(starts);
                    // the pair's word data: two 16-byte shared-memory reads (broadcast within a group)
                    const uint4 ga = grp[gi][0], gr = grp[gi][1];
                    uint32_t v0 = ga.x;
                    uint32_t v1 = PW == 2 ? ga.y : 0u;
                    const uint32_t s0 = ga.z, s1 = ga.w;
                    if ((m[u].x & gr.x) | (m[u].y & gr.y)) {  // the group's first partial record (zero: none)
                        if (PW == 1 || gr.z == 0) v0 |= gr.w;
                        else v1 |= gr.w;
                    }
                    for (uint32_t q = s0 + 1; q < s1; ++q) {  // (rare) more partial props on the word
                        const uint4 r = __ldg(rec + q);
                        if ((m[u].x & r.x) | (m[u].y & r.y)) {
                            if (PW == 1 || r.z == 0) v0 |= r.w;
                            else v1 |= r.w;
                        }
                    }
                    if (cu + lane < E1) {  // (a task's rows are this warp's alone; rows of a group are distinct)
                        asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(acc_s + 4u * rowu), "r"(v0) : "memory");
                        if constexpr (PW == 2)
                            asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(acc_s + 4u * (MAXR + rowu)), "r"(v1)
                                         : "memory");
                    }
                }
            }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        for (uint32_t r = lane; r < nr; r += 32) {  // lane r stores row r's label
            uint64_t l = acc[r];  // (prop halves in two planes: a row's two words are the same bank)
            if constexpr (PW == 2) l |= static_cast<uint64_t>(acc[MAXR + r]) << 32;
            out[static_cast<uint64_t>(s_perm[wib][r]) * ostride] = static_cast<SW>(l);
#pragma unroll
            for (int h = 0; h < PW; ++h) acc[MAXR * h + r] = 0;
        }
        __syncwarp();
    }
}

// Byte layout of the word-major work buffer: frame-major summaries, word
// headers, the slot-row cursor, then the lane records (worst case: every
// (word, prop, frame) partial, one per slot row) + 1 row of padding.
struct WmLayout {
    uint64_t nt;  // (nw64 + 1) * prop slots
    size_t ffrT, whdr, wpair, cursor, lrec, total;
    WmLayout(int props, uint32_t nw64) {
        nt = static_cast<uint64_t>(nw64 + 1) * (props > 32 ? 64u : 32u);
        auto up = [](size_t x, size_t a) { return (x + a - 1) & ~(a - 1); };
        ffrT = 0;
        whdr = ffrT + nt * 8;  // ffrT: (nw64 + 1) x 64 frames x prop halves u32
        wpair = whdr + (nw64 + 1) * 8;  // (nw64 + 1) x prop halves x 32 lanes u16 = nt * 2 bytes
        cursor = up(wpair + nt * 2, 8);
        lrec = up(cursor + 4, 16);
        total = lrec + (nt * 64 + 32) * 16;
    }
};

size_t wm_work_bytes(int props, uint32_t nw64) { return WmLayout(props, nw64).total; }

cudaError_t launch_wm_build(const uint64_t* P64, int props, int frames, uint32_t nw64, uint64_t cells, void* work,
                            size_t work_bytes, uint32_t* task_ctr, int nctr, cudaStream_t st,
                            const uint32_t* touched64) {
    if (props > 64 || frames > 64) return cudaErrorInvalidValue;
    const WmLayout L(props, nw64);
    if (L.total > work_bytes) return cudaErrorInvalidValue;
    uint8_t* wb = static_cast<uint8_t*>(work);
    cudaError_t e = cudaMemsetAsync(wb + L.cursor, 0, 4, st);
    if (e != cudaSuccess) return e;
    // 8 (4) words x 32 (64) prop slots per CTA: many small CTAs (the kernel is
    // a chain of dependent phases), and CTAs whose words no pair is on exit
    constexpr int kNT = 256;
    const int pshift = props > 32 ? 6 : 5;
    const int wpb = kNT >> pshift;
    const uint64_t gw = (static_cast<uint64_t>(nw64) + 1 + wpb - 1) / wpb, gc = (static_cast<uint64_t>(nctr) + kNT - 1) / kNT;
    const unsigned grid = static_cast<unsigned>(gw > gc ? gw : gc);
    auto* ffrT = reinterpret_cast<uint32_t*>(wb + L.ffrT);
    auto* whdr = reinterpret_cast<uint2*>(wb + L.whdr);
    auto* cur = reinterpret_cast<uint32_t*>(wb + L.cursor);
    auto* lrec = reinterpret_cast<uint4*>(wb + L.lrec);
    auto* wpair = reinterpret_cast<uint16_t*>(wb + L.wpair);
    if (pshift == 5)
        wm_build_kernel<5, kNT><<<grid, kNT, 0, st>>>(P64, props, frames, nw64, cells, ffrT, whdr, wpair, cur,
                                                      lrec, task_ctr, nctr, touched64);
    else
        wm_build_kernel<6, kNT><<<grid, kNT, 0, st>>>(P64, props, frames, nw64, cells, ffrT, whdr, wpair, cur,
                                                      lrec, task_ctr, nctr, touched64);
    return cudaGetLastError();
}

// Byte layout of the prop-lane work buffer (label_pl_kernel): summary masks
// (pw prop slots per word), the record cursor and ranges, then the records
// (worst case: every (word, prop, frame) partial) + 32 records of padding for
// the last probe round.
struct PlLayout {
    uint64_t nt;  // (nw64 + 1) * pw
    size_t ffr, sfr, wdat, cursor, rec_se, rec, total;
    PlLayout(int props, int frames, uint32_t nw64) {
        nt = static_cast<uint64_t>(nw64 + 1) * (props > 32 ? 64u : 32u);
        auto up = [](size_t x, size_t a) { return (x + a - 1) & ~(a - 1); };
        ffr = 0;
        sfr = ffr + nt * 8;
        wdat = up(sfr + nt * 8, 16);  // one frame: (nw64 + 1) x 32 B word data (pl_build_kernel)
        cursor = wdat + (static_cast<size_t>(nw64) + 1) * 32;
        rec_se = up(cursor + 4, 8);
        rec = up(rec_se + (nw64 + 2) * 8, 16);
        total = rec + (nt * static_cast<uint64_t>(frames) + 32) * 16;
    }
};

cudaError_t launch_pl(const uint64_t* P64, int props, int frames, uint32_t nw64, uint64_t cells, void* work,
                      size_t work_bytes, uint32_t* task_ctr, int nctr, cudaStream_t st, const uint32_t* touched64) {
    if (props > 64 || frames > 64) return cudaErrorInvalidValue;
    const int pshift = props > 32 ? 6 : 5;
    const PlLayout L(props, frames, nw64);
    if (L.total > work_bytes) return cudaErrorInvalidValue;
    uint8_t* wb = static_cast<uint8_t*>(work);
    uint64_t* ffr = reinterpret_cast<uint64_t*>(wb + L.ffr);
    uint64_t* sfr = reinterpret_cast<uint64_t*>(wb + L.sfr);
    uint32_t* cursor = reinterpret_cast<uint32_t*>(wb + L.cursor);
    uint2* rec_se = reinterpret_cast<uint2*>(wb + L.rec_se);
    uint4* rec = reinterpret_cast<uint4*>(wb + L.rec);
    cudaError_t e = cudaMemsetAsync(cursor, 0, 4, st);
    if (e != cudaSuccess) return e;
    // 32 (16) words x 32 (64) prop slots per CTA.  256-thread CTAs fill the
    // GPU better (summary 40 -> 43 us anyway) but scatter the word segments
    // more, and the prop-lane labelling kernel lost 60 us to record locality.
    constexpr int kNT = 1024;
    const int wpb = kNT >> pshift;
    const uint64_t gw = (static_cast<uint64_t>(nw64) + 1 + wpb - 1) / wpb, gc = (static_cast<uint64_t>(nctr) + kNT - 1) / kNT;
    const unsigned grid = static_cast<unsigned>(gw > gc ? gw : gc);
    uint4* wdat = frames == 1 ? reinterpret_cast<uint4*>(wb + L.wdat) : nullptr;
    if (pshift == 5)
        pl_build_kernel<5, kNT><<<grid, kNT, 0, st>>>(P64, props, frames, nw64, cells, ffr, sfr, rec_se, cursor, rec,
                                                  task_ctr, nctr, touched64, wdat);
    else
        pl_build_kernel<6, kNT><<<grid, kNT, 0, st>>>(P64, props, frames, nw64, cells, ffr, sfr, rec_se, cursor, rec,
                                                  task_ctr, nctr, touched64, wdat);
    return cudaGetLastError();
}

size_t pl_work_bytes(int props, int frames, uint32_t nw64) { return PlLayout(props, frames, nw64).total; }

#if LTLG_AB_BUILD
template <typename SW, int PW>
static void launch_pl_label(const LaunchArgs& a, cudaStream_t st) {
    const PlLayout L(a.props, a.frames, a.nw64);
    const uint8_t* wb = static_cast<const uint8_t*>(a.sf);
    static int per_sm = 0;
    auto kern = label_pl_kernel<SW, PW>;
    if (!per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
        if (per_sm <= 0) per_sm = 4;
    }
    kern<<<sm_count() * per_sm, 256, 0, st>>>(a.mask_b64, a.word_b64, a.task_pair_b64, a.task_row, a.task_begin,
                                              a.ntasks, a.task_ctr, reinterpret_cast<const uint64_t*>(wb + L.ffr),
                                              reinterpret_cast<const uint64_t*>(wb + L.sfr),
                                              reinterpret_cast<const uint2*>(wb + L.rec_se),
                                              reinterpret_cast<const uint4*>(wb + L.rec), a.frames, a.perm,
                                              static_cast<SW*>(a.out), a.ostride ? a.ostride : static_cast<uint32_t>(a.frames));
}
#endif  // LTLG_AB_BUILD

template <typename SW, int PW>
static void launch_wm_label(const LaunchArgs& a, cudaStream_t st) {
    const WmLayout L(a.props, a.nw64);
    const uint8_t* wb = static_cast<const uint8_t*>(a.sf);
    auto kern = label_wm_kernel<SW, PW>;
    const size_t smem = static_cast<size_t>(a.wm_rows) * 64 * PW * 4;  // the CTA's label block
    static size_t smem_set = 0;
    static int per_sm = 0;
    static size_t per_sm_smem = ~size_t(0);
    if (smem > smem_set) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        smem_set = smem;
    }
    if (per_sm_smem != smem) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWmThreads, smem);
        if (per_sm <= 0) per_sm = 1;
        per_sm_smem = smem;
    }
    kern<<<sm_count() * per_sm, kWmThreads, smem, st>>>(
        a.wm_mask, a.wm_row, a.wm_gword, a.wm_gstart, a.wm_task_row, a.wm_task_grp, a.task_begin, a.ntasks,
        a.task_ctr, reinterpret_cast<const uint32_t*>(wb + L.ffrT),
        reinterpret_cast<const uint2*>(wb + L.whdr), reinterpret_cast<const uint16_t*>(wb + L.wpair),
        reinterpret_cast<const uint4*>(wb + L.lrec), a.frames, a.perm,
        static_cast<SW*>(a.out), a.ostride ? a.ostride : static_cast<uint32_t>(a.frames), a.wm_rows);
}

template <typename SW, int PW, int MAXR>
static cudaError_t launch_wm1_label_r(const LaunchArgs& a, cudaStream_t st) {
    const PlLayout L(a.props, 1, a.nw64);
    const uint8_t* wb = static_cast<const uint8_t*>(a.sf);
    auto kern = label_wm1_kernel<SW, PW, MAXR>;
    constexpr size_t smem = 0;
    static int per_sm = 0;
    if (!per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWm1Warps * 32, smem);
        if (per_sm <= 0) per_sm = 1;
    }
    // programmatic dependent launch: the CTAs get resident while the summary
    // kernel finishes (label_wm1_kernel waits on it first)
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = a.pdl ? 1 : 0;
    cfg.gridDim = dim3(static_cast<unsigned>(sm_count() * per_sm));
    cfg.blockDim = dim3(kWm1Warps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a.wm_mask, a.wm_row, a.wm_gword, a.wm_gstart, a.wm_task_row, a.wm_task_grp,
                              a.task_begin, a.ntasks, a.task_ctr, reinterpret_cast<const uint4*>(wb + L.wdat),
                              reinterpret_cast<const uint4*>(wb + L.rec),
                              a.perm, static_cast<SW*>(a.out), a.ostride ? a.ostride : 1u);
}

// (tasks of <= 128 rows -- the default -- take the smaller label block: more CTAs per SM)
template <typename SW, int PW>
static cudaError_t launch_wm1_label(const LaunchArgs& a, cudaStream_t st) {
    return a.wm_rows <= 128 ? launch_wm1_label_r<SW, PW, 128>(a, st) : launch_wm1_label_r<SW, PW, kWmMaxRows>(a, st);
}

template <int FMT, typename SW, int FPL, bool FULL>
static void launch_batch_t(const LaunchArgs& a, cudaStream_t st) {
    static int per_sm = 0;
    if (!per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, label_batch_kernel<FMT, SW, FPL, FULL>, 256, 0);
        if (per_sm <= 0) per_sm = 4;
    }
    label_batch_kernel<FMT, SW, FPL, FULL><<<sm_count() * per_sm, 256, 0, st>>>(
        a.pairs, a.task_pair, a.task_row, a.task_begin, a.ntasks, a.task_ctr, a.sf, a.s_only, a.P32, a.nw32, a.props, a.frames,
        a.perm, static_cast<SW*>(a.out));
}

template <int FMT, typename SW>
static void launch_batch_fpl(const LaunchArgs& a, cudaStream_t st) {
    if (a.frames == 32) launch_batch_t<FMT, SW, 1, true>(a, st);
    else if (a.frames == 64) launch_batch_t<FMT, SW, 2, true>(a, st);
    else if (a.frames == 128) launch_batch_t<FMT, SW, 4, true>(a, st);
    else if (a.frames < 32) launch_batch_t<FMT, SW, 1, false>(a, st);
    else if (a.frames < 64) launch_batch_t<FMT, SW, 2, false>(a, st);
    else if (a.frames < 128) launch_batch_t<FMT, SW, 4, false>(a, st);
    else launch_batch_t<FMT, SW, 8, false>(a, st);
}

cudaError_t launch_label(const LaunchArgs& a, cudaStream_t st) {
    if (a.ntasks <= a.task_begin) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    if (a.frames == 1 && a.word_major) {  // word-major single-frame path (<= 64 props)
        switch (a.label_bytes) {
            case 1: e = launch_wm1_label<uint8_t, 1>(a, st); break;
            case 2: e = launch_wm1_label<uint16_t, 1>(a, st); break;
            case 4: e = launch_wm1_label<uint32_t, 1>(a, st); break;
            default: e = launch_wm1_label<uint64_t, 2>(a, st); break;
        }
#if LTLG_AB_BUILD
    } else if (a.prop_lane && a.word_major && a.tc) {  // dev knob LTLG_TC=1: tcgen05 kind::i8
        e = launch_tc_label(a, st);
#endif
    } else if (a.prop_lane && a.word_major) {  // word-major multi-frame path (<= 64 props, a slice of <= 64 frames)
        switch (a.label_bytes) {
            case 1: launch_wm_label<uint8_t, 1>(a, st); break;
            case 2: launch_wm_label<uint16_t, 1>(a, st); break;
            case 4: launch_wm_label<uint32_t, 1>(a, st); break;
            default: launch_wm_label<uint64_t, 2>(a, st); break;
        }
#if LTLG_AB_BUILD
    } else if (a.mask_b64 && a.prop_lane) {  // pair-major prop-lane kernel (A/B: LTLG_WORDMAJOR=0)
        switch (a.label_bytes) {
            case 1: launch_pl_label<uint8_t, 1>(a, st); break;
            case 2: launch_pl_label<uint16_t, 1>(a, st); break;
            case 4: launch_pl_label<uint32_t, 1>(a, st); break;
            default: launch_pl_label<uint64_t, 2>(a, st); break;
        }
#endif
    } else if (a.frames == 1 && a.t64) {  // 64-cell-word single-frame path (<= 32 props)
        switch (a.label_bytes) {
            case 1: e = launch_stream64_t<16, uint8_t>(a, st); break;
            case 2: e = launch_stream64_t<16, uint16_t>(a, st); break;
            case 4: e = launch_stream64_t<32, uint32_t>(a, st); break;
            default: e = launch_stream64_t<64, uint64_t>(a, st); break;
        }
    } else if (a.frames == 1) {
#if LTLG_AB_BUILD
        switch (a.label_bytes) {
            case 1: e = launch_stream_t<16, uint8_t>(a, st); break;
            case 2: e = launch_stream_t<16, uint16_t>(a, st); break;
            case 4: e = launch_stream_t<32, uint32_t>(a, st); break;
            default: e = launch_stream_t<64, uint64_t>(a, st); break;
        }
#else
        e = cudaErrorNotSupported;  // (the 32-cell single-frame kernels are in the A/B build only)
#endif
    } else if (a.mask_b64) {  // 64-cell-word multi-frame path (<= 32 props)
        switch (a.label_bytes) {
            case 1: launch_batch64_fpl<uint8_t>(a, st); break;
            case 2: launch_batch64_fpl<uint16_t>(a, st); break;
            default: launch_batch64_fpl<uint32_t>(a, st); break;
        }
    } else {
        switch (a.label_bytes) {
            case 1: launch_batch_fpl<16, uint8_t>(a, st); break;
            case 2: launch_batch_fpl<16, uint16_t>(a, st); break;
            case 4: launch_batch_fpl<32, uint32_t>(a, st); break;
            default: launch_batch_fpl<64, uint64_t>(a, st); break;
        }
    }
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// label_edge_counting (label.cpp:140-148) for every row against one P column:
// a thread walks one batch task's 64-cell pairs in order.  Within a row the
// words ascend and a word's bit b is cell 64 w + b, so the reference's linear
// scan over ascending cell indices examines, for the first pair with a hit,
// the cells of the earlier pairs plus the mask bits below the lowest hit bit,
// plus the witness itself; with no hit it examines all of the row's cells.
__global__ void __launch_bounds__(256) edge_count_kernel(const uint64_t* __restrict__ masks,
                                                         const uint32_t* __restrict__ words,
                                                         const uint64_t* __restrict__ task_pair,
                                                         const uint32_t* __restrict__ task_row, uint32_t ntasks,
                                                         const uint32_t* __restrict__ perm,
                                                         const uint64_t* __restrict__ col, uint8_t* __restrict__ hit,
                                                         uint64_t* __restrict__ examined) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntasks) return;
    int64_t row = static_cast<int64_t>(task_row[t]) - 1;
    uint64_t before = 0, at = 0;
    bool found = false;
    auto close = [&]() {
        const uint32_t r = perm[row];
        if (hit) hit[r] = found ? 1 : 0;
        if (examined) examined[r] = found ? at : before;
    };
    for (uint64_t q = task_pair[t]; q < task_pair[t + 1]; ++q) {
        const uint32_t wh = words[q];
        const uint64_t m = masks[q];
        if (wh & kHead) {
            if (row >= static_cast<int64_t>(task_row[t])) close();
            ++row;
            before = 0;
            found = false;
        }
        if (found || !m) continue;  // (the empty row's sentinel pair has mask 0)
        const uint64_t x = m & __ldg(col + (wh & kWordMask));
        if (x) {
            at = before + __popcll(m & ((x & (~x + 1)) - 1)) + 1;
            found = true;
        } else {
            before += __popcll(m);
        }
    }
    if (row >= static_cast<int64_t>(task_row[t])) close();
}

cudaError_t launch_edge_count(const uint64_t* masks, const uint32_t* words, const uint64_t* task_pair,
                              const uint32_t* task_row, uint32_t ntasks, const uint32_t* perm, const uint64_t* col,
                              uint8_t* hit, uint64_t* examined, cudaStream_t st) {
    if (ntasks == 0) return cudaSuccess;
    edge_count_kernel<<<(ntasks + 255) / 256, 256, 0, st>>>(masks, words, task_pair, task_row, ntasks, perm, col, hit,
                                                            examined);
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

cudaError_t launch_guards(const void* labels, int label_bytes, uint64_t n, const uint64_t* lut, uint64_t always,
                          uint64_t all_guards, uint64_t* admitted, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 148ull * 16));
    switch (label_bytes) {
        case 1: guard_kernel<<<blocks, 256, 0, st>>>(static_cast<const uint8_t*>(labels), n, lut, always, all_guards, admitted); break;
        case 2: guard_kernel<<<blocks, 256, 0, st>>>(static_cast<const uint16_t*>(labels), n, lut, always, all_guards, admitted); break;
        case 4: guard_kernel<<<blocks, 256, 0, st>>>(static_cast<const uint32_t*>(labels), n, lut, always, all_guards, admitted); break;
        default: guard_kernel<<<blocks, 256, 0, st>>>(static_cast<const uint64_t*>(labels), n, lut, always, all_guards, admitted); break;
    }
    return cudaGetLastError();
}

// ranges: nboxes x (first, last) per axis (4 axes, int64), box_off: cols + 1
// generate_scenario's not_nominal_lane (scenario.cpp:59-76): a cell (cx, cy,
// ct) is set iff flag bit cy * nx + cx is set (the host evaluates the lane
// test per (cx, cy) with the reference's libm hypot); the same column goes to
// ncols columns out + (col0 + c * col_step) * nw64.
__device__ __forceinline__ uint64_t compact3(uint64_t x) {
    x &= 0x1249249249249249ull;
    x = (x ^ (x >> 2)) & 0x10c30c30c30c30c3ull;
    x = (x ^ (x >> 4)) & 0x100f00f00f00f00full;
    x = (x ^ (x >> 8)) & 0x1f0000ff0000ffull;
    x = (x ^ (x >> 16)) & 0x1f00000000ffffull;
    x = (x ^ (x >> 32)) & 0x1fffffull;
    return x;
}

__global__ void __launch_bounds__(256) lane_kernel(uint32_t nw64, uint64_t cells, int off0, int off1, int bits0,
                                                   const uint64_t* __restrict__ flags, int ncols, int col0,
                                                   int col_step, uint64_t* __restrict__ out) {
    const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= nw64) return;
    uint64_t v = 0;
    for (int b = 0; b < 64; ++b) {
        const uint64_t i = static_cast<uint64_t>(w) * 64 + b;
        if (i >= cells) break;
        const uint64_t cx = compact3(i >> off0), cy = compact3(i >> off1);
        const uint64_t f = (cy << bits0) | cx;
        v |= ((flags[f >> 6] >> (f & 63)) & 1ull) << b;
    }
    for (int c = 0; c < ncols; ++c) out[static_cast<uint64_t>(col0 + c * col_step) * nw64 + w] = v;
}

cudaError_t launch_lane(int depth, const uint64_t* flags, int ncols, int col0, int col_step, uint64_t* out,
                        cudaStream_t st) {
    const uint64_t cells = uint64_t(1) << depth;
    const uint32_t nw64 = static_cast<uint32_t>((cells + 63) / 64);
    const int r = depth % 3;
    auto off = [&](int a) { return r + 2 - a - 3 * (a < r ? 1 : 0); };
    const int bits0 = depth / 3 + (0 < r ? 1 : 0);
    lane_kernel<<<(nw64 + 255) / 256, 256, 0, st>>>(nw64, cells, off(0), off(1), bits0, flags, ncols, col0, col_step,
                                                    out);
    return cudaGetLastError();
}

cudaError_t launch_rasterize(int k, int depth, int cols_total, const uint64_t* box_off, const int64_t* ranges,
                             uint64_t* out, cudaStream_t st) {
    if (k < 1 || k > 4 || depth < k || depth > 36) return cudaErrorInvalidValue;
    RasterGeom g{};
    g.k = k;
    g.depth = depth;
    uint64_t pat[4][64] = {};
    const int low = depth < 6 ? depth : 6;  // z-bits inside one 64-cell word
    std::vector<int> bits(static_cast<size_t>(k));
    for (int a = 0; a < k; ++a) bits[static_cast<size_t>(a)] = depth / k + (a < depth % k ? 1 : 0);
    for (int a = 0; a < k; ++a) {
        uint32_t nv = 1;
        for (int p = 0; p < low; ++p)
            if ((depth - 1 - p) % k == a) nv <<= 1;
        g.nvals[a] = nv;
    }
    for (uint32_t b = 0; b < (1u << low); ++b) {
        uint32_t off[4] = {0, 0, 0, 0};
        for (int p = 0; p < low; ++p) {
            if (!(b >> p & 1u)) continue;
            const int l = depth - 1 - p, a = l % k, ab = bits[static_cast<size_t>(a)] - 1 - l / k;
            off[a] |= 1u << ab;
        }
        for (int a = 0; a < k; ++a) pat[a][off[a]] |= 1ull << b;
    }
    cudaError_t e = cudaMemcpyToSymbolAsync(c_raster_pat, pat, sizeof(pat), 0, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
    e = cudaMemcpyToSymbolAsync(c_raster_geom, &g, sizeof(g), 0, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
    const uint64_t cells = 1ull << depth;
    const uint32_t nw64 = static_cast<uint32_t>((cells + 63) / 64);
    if (cols_total == 0) return cudaSuccess;
    dim3 grid((nw64 + 255) / 256, static_cast<unsigned>(cols_total));
    rasterize_kernel<<<grid, 256, 0, st>>>(nw64, cols_total, box_off, ranges, cells, out);
    return cudaGetLastError();
}

cudaError_t launch_resample(int vdepth, double vlo0, double vhi0, double vlo1, double vhi1, int wdepth,
                            double wlo0, double whi0, double wlo1, double whi1, const void* poses,
                            int frames, int props, const uint32_t* world32, uint32_t wnw32, int outside,
                            uint32_t vnw32, uint32_t* out32, cudaStream_t st) {
    if (props == 0) return cudaSuccess;
    Grid2 vg{vdepth, vlo0, vhi0, vlo1, vhi1};
    Grid2 wg{wdepth, wlo0, whi0, wlo1, whi1};
    const uint64_t threads = static_cast<uint64_t>(vnw32) * 32;
    dim3 grid(static_cast<unsigned>((threads + 255) / 256), static_cast<unsigned>(frames));
    resample_kernel<<<grid, 256, 0, st>>>(vg, wg, static_cast<const Pose2*>(poses), props, world32, wnw32,
                                          outside, vnw32, out32);
    return cudaGetLastError();
}

}  // namespace ltlg
