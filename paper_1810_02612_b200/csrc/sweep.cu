// sweep.cu -- the swept-volume matrix T on the GPU.
//
// Reference: swept_volume_matrix (core/src/label.cpp:75-116) runs
// sweep_voxelize_indices (core/src/abstraction.cpp:172-221) per edge on CPU
// worker threads: every trajectory sample's oriented footprint rectangle
// (footprint_polygon, abstraction.cpp:136-146) is rasterized into the time
// slab of its tau by a strict separating-axis test per candidate cell
// (rect_cell_overlap, abstraction.cpp:156-170), the z-order indices
// (ZScatter, grid.cpp:151-168) are sorted and de-duplicated, and the rows
// are concatenated into a CsrBoolMatrix.
//
// B200 design: one CTA per edge, edges pulled from a counter (persistent
// grid).  A warp per trajectory sample, lanes over the sample's candidate
// cells; hits go into a shared-memory open-addressing set (32-bit z-index
// keys tagged with a per-edge epoch, so the table is never cleared); the
// set is compacted and bitonic-sorted in shared memory and written as the
// row.  Two passes over the edges: COUNT (row sizes -> exclusive scan ->
// row offsets) and FILL.  Rows with more than kSweepCap distinct cells
// overflow to a global-memory table of the same design.  The double
// arithmetic is the reference's, operation for operation (the library is
// built with --fmad=false, so nothing is contracted into FMAs).
#include <cstdint>

#include "launch.h"

namespace ltlg {

namespace {

// spread the low 21 bits of x to every third bit
__device__ __forceinline__ uint64_t spread3(uint64_t x) {
    x &= 0x1fffffull;
    x = (x | x << 32) & 0x1f00000000ffffull;
    x = (x | x << 16) & 0x1f0000ff0000ffull;
    x = (x | x << 8) & 0x100f00f00f00f00full;
    x = (x | x << 4) & 0x10c30c30c30c30c3ull;
    x = (x | x << 2) & 0x1249249249249249ull;
    return x;
}

// ZScatter::scatter for a 3-axis grid (grid.cpp:151-168): bit b of axis a's
// coordinate lands at index bit depth-1-((bits_a-1-b)*3 + a) = 3b + off_a.
__device__ __forceinline__ uint32_t scatter3(const SweepParams& p, int a, uint64_t c) {
    return static_cast<uint32_t>(spread3(c) << p.zoff[a]);
}

// GridSpec::overlap_cells (grid.cpp:49-61)
__device__ __forceinline__ void overlap_cells(const SweepParams& p, int a, double x_lo, double x_hi, int64_t& first,
                                              int64_t& last) {
    const double lo = p.lo[a], hi = p.hi[a], cells = p.cells[a];
    const double z_lo = (x_lo - lo) / (hi - lo) * cells;
    const double z_hi = (x_hi - lo) / (hi - lo) * cells;
    first = static_cast<int64_t>(floor(z_lo));
    last = static_cast<int64_t>(ceil(z_hi)) - 1;
    if (first < 0) first = 0;
    if (last > p.ncell[a] - 1) last = p.ncell[a] - 1;
}

// Insert a key into the epoch-tagged open-addressing set.  Returns false if
// the set is full or the distinct count passed `cap` (overflow).
__device__ __forceinline__ bool set_insert(unsigned long long* tab, uint32_t hmask, uint32_t epoch, uint32_t key,
                                           uint32_t* cnt, uint32_t cap) {
    const unsigned long long mine = (static_cast<unsigned long long>(epoch) << 32) | key;
    uint32_t h = (key * 0x9E3779B1u) & hmask;
    for (uint32_t probe = 0; probe <= hmask; ++probe) {
        unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(tab + h);
        if (cur == mine) return true;
        if (static_cast<uint32_t>(cur >> 32) != epoch) {  // free for this edge
            const unsigned long long old = atomicCAS(tab + h, cur, mine);
            if (old == cur) return atomicAdd(cnt, 1u) < cap;
            if (old == mine) return true;
            if (static_cast<uint32_t>(old >> 32) != epoch) {  // raced with a stale value: look again
                --probe;
                continue;
            }
        }
        h = (h + 1) & hmask;
    }
    return false;
}

// Bitonic sort of n2 (power of two) keys by the whole CTA.
__device__ void bitonic_sort(uint32_t* k, uint32_t n2) {
    for (uint32_t size = 2; size <= n2; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = threadIdx.x; i < n2 / 2; i += blockDim.x) {
                const uint32_t lo = 2 * i - (i & (stride - 1));
                const uint32_t hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint32_t a = k[lo], b = k[hi];
                if ((a > b) == up) {
                    k[lo] = b;
                    k[hi] = a;
                }
            }
            __syncthreads();
        }
    }
}

}  // namespace

// MODE 0: row sizes into row_cnt.  MODE 1: rows into cols at row_off.
// MODE 2: rows into the staging buffer at a bump-allocated position
// (stage_off[e]; ~0 if the row overflowed or the buffer ran out), sizes
// into row_cnt -- one rasterization pass instead of count + fill.
// GLOBAL = false: every edge, shared-memory sets (an overflowing edge is
// listed in over_list and skipped); true: the over_list edges, global-memory
// sets of 2^glog2 entries per CTA (an overflow there bumps err_key[1] and the
// host retries with a larger table).
template <int MODE, bool GLOBAL>
__global__ void __launch_bounds__(kSweepThreads) sweep_kernel(SweepParams p, SweepBufs b, uint32_t glog2) {
    extern __shared__ unsigned long long smem_tab[];
    __shared__ uint32_t s_edge, s_cnt, s_pos, s_bad;
    __shared__ unsigned long long s_stage;
    const uint32_t hsize = GLOBAL ? (1u << glog2) : kSweepTable;
    const uint32_t cap = GLOBAL ? hsize / 2 : kSweepCap;
    unsigned long long* tab = GLOBAL ? b.gtab + static_cast<size_t>(blockIdx.x) * hsize : smem_tab;
    uint32_t* keys = GLOBAL ? b.gkeys + static_cast<size_t>(blockIdx.x) * (hsize / 2)
                            : reinterpret_cast<uint32_t*>(smem_tab + kSweepTable);
    for (uint32_t i = threadIdx.x; i < hsize; i += blockDim.x) tab[i] = 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const double half_x = p.w[0] / 2, half_y = p.w[1] / 2;
    for (uint32_t epoch = 1;; ++epoch) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t k = atomicAdd(b.edge_ctr, 1u);
            s_edge = GLOBAL ? (k < *b.n_over ? b.over_list[k] : 0xffffffffu) : k;
            s_cnt = 0;
            s_pos = 0;
            s_bad = 0;
        }
        __syncthreads();
        const uint32_t e = s_edge;
        if (GLOBAL ? e == 0xffffffffu : e >= p.edges) break;
        const uint64_t sb = p.sample_off[e], se = p.sample_off[e + 1];
        const bool report = MODE == 2 || (MODE == 0 && !GLOBAL);
        // warp `warp` owns samples sb + warp + k * nwarps; lane k sets up the
        // k-th of a batch of 32 of them (footprint, checks, cell ranges), then
        // the warp walks the batch, lanes over each sample's candidate cells
        for (uint64_t base = sb + warp; base < se; base += 32ull * nwarps) {
            const uint64_t i = base + static_cast<uint64_t>(lane) * nwarps;
            const uint64_t left = (se - base + nwarps - 1) / nwarps;
            const uint32_t nb = left < 32 ? static_cast<uint32_t>(left) : 32u;
            uint32_t n = 0, ny = 1, ct_bits = 0;
            int64_t x0 = 0, y0 = 0;
            double rcx = 0, rcy = 0, cs = 0, sn = 0, sep_x = 0, sep_y = 0, sep_l = 0, sep_w = 0;
            if (i < se) {
                const double* s5 = p.samples + 5 * i;
                const double px = s5[0], py = s5[1], heading = s5[2], tau = s5[4];
                // sweep_collect (abstraction.cpp:180-199): the checks, in order
                if (!(tau >= p.lo[2] && tau < p.hi[2])) {
                    if (report) atomicMin(p.err_key, static_cast<unsigned long long>(i) * 4 + 0);
                } else if (p.length <= 0 || p.width <= 0) {  // footprint_polygon's check
                    if (report) atomicMin(p.err_key, static_cast<unsigned long long>(i) * 4 + 1);
                } else {
                    // GridSpec::quantize (grid.cpp:35-47) of tau
                    uint64_t ct = static_cast<uint64_t>(floor((tau - p.lo[2]) / (p.hi[2] - p.lo[2]) * p.cells[2]));
                    if (ct >= static_cast<uint64_t>(p.ncell[2])) ct = p.ncell[2] - 1;
                    ct_bits = scatter3(p, 2, ct);
                    sincos(heading, &sn, &cs);
                    rcx = px + p.ref_offset * cs;
                    rcy = py + p.ref_offset * sn;
                    const double hl = p.length / 2, hw = p.width / 2;
                    const double ac = fabs(cs), as = fabs(sn);
                    const double ext_x = hl * ac + hw * as;
                    const double ext_y = hl * as + hw * ac;
                    if (rcx - ext_x < p.lo[0] || rcx + ext_x > p.hi[0] || rcy - ext_y < p.lo[1] ||
                        rcy + ext_y > p.hi[1]) {
                        if (report) atomicMin(p.err_key, static_cast<unsigned long long>(i) * 4 + 2);
                    } else {
                        int64_t x1, y1;
                        overlap_cells(p, 0, rcx - ext_x, rcx + ext_x, x0, x1);
                        overlap_cells(p, 1, rcy - ext_y, rcy + ext_y, y0, y1);
                        if (x1 >= x0 && y1 >= y0) {
                            ny = static_cast<uint32_t>(y1 - y0 + 1);
                            n = static_cast<uint32_t>(x1 - x0 + 1) * ny;
                        }
                        // rect_cell_overlap's right-hand sides (abstraction.cpp:
                        // 163-168): functions of the sample only, hoisted
                        sep_x = half_x + hl * ac + hw * as;
                        sep_y = half_y + hl * as + hw * ac;
                        sep_l = hl + half_x * ac + half_y * as;
                        sep_w = hw + half_x * as + half_y * ac;
                    }
                }
            }
            for (uint32_t k = 0; k < nb; ++k) {
                const uint32_t nk = __shfl_sync(0xffffffffu, n, k);
                if (!nk) continue;
                const uint32_t nyk = __shfl_sync(0xffffffffu, ny, k);
                const uint32_t ctk = __shfl_sync(0xffffffffu, ct_bits, k);
                const int64_t x0k = __shfl_sync(0xffffffffu, x0, k), y0k = __shfl_sync(0xffffffffu, y0, k);
                const double rcxk = __shfl_sync(0xffffffffu, rcx, k), rcyk = __shfl_sync(0xffffffffu, rcy, k);
                const double csk = __shfl_sync(0xffffffffu, cs, k), snk = __shfl_sync(0xffffffffu, sn, k);
                const double sxk = __shfl_sync(0xffffffffu, sep_x, k), syk = __shfl_sync(0xffffffffu, sep_y, k);
                const double slk = __shfl_sync(0xffffffffu, sep_l, k), swk = __shfl_sync(0xffffffffu, sep_w, k);
                for (uint32_t t = lane; t < nk; t += 32) {
                    const int64_t cx = x0k + t / nyk, cy = y0k + t % nyk;
                    const double ccx = p.lo[0] + (static_cast<double>(cx) + 0.5) * p.w[0];
                    const double ccy = p.lo[1] + (static_cast<double>(cy) + 0.5) * p.w[1];
                    // rect_cell_overlap (abstraction.cpp:156-170)
                    const double dx = ccx - rcxk, dy = ccy - rcyk;
                    if (fabs(dx) >= sxk) continue;
                    if (fabs(dy) >= syk) continue;
                    if (fabs(dx * csk + dy * snk) >= slk) continue;
                    if (fabs(-dx * snk + dy * csk) >= swk) continue;
                    const uint32_t key = scatter3(p, 0, static_cast<uint64_t>(cx)) |
                                         scatter3(p, 1, static_cast<uint64_t>(cy)) | ctk;
                    if (!s_bad && !set_insert(tab, hsize - 1, epoch, key, &s_cnt, cap)) s_bad = 1;
                }
            }
        }
        __syncthreads();
        const uint32_t cnt = s_cnt;
        if (MODE == 0) {
            if (threadIdx.x == 0) {
                b.row_cnt[e] = s_bad ? 0u : cnt;
                if (s_bad) {
                    if (GLOBAL) atomicAdd(p.err_key + 1, 1ull);  // retry with a larger table
                    else b.over_list[atomicAdd(b.n_over, 1u)] = e;
                }
            }
            continue;
        }
        if (s_bad) {  // listed for the global-memory sets (MODE 2), or already listed (MODE 1)
            if (MODE == 2 && threadIdx.x == 0) {
                b.row_cnt[e] = 0;
                b.stage_off[e] = ~0ull;
                b.over_list[atomicAdd(b.n_over, 1u)] = e;
            }
            continue;
        }
        // compact this edge's keys, sort them, write the row (sweep_voxelize_indices'
        // sort + unique, abstraction.cpp:214-221)
        for (uint32_t i = threadIdx.x; i < hsize; i += blockDim.x) {
            const unsigned long long v = tab[i];
            if (static_cast<uint32_t>(v >> 32) == epoch) keys[atomicAdd(&s_pos, 1u)] = static_cast<uint32_t>(v);
        }
        uint32_t n2 = 1;
        while (n2 < cnt) n2 <<= 1;
        if (MODE == 2 && threadIdx.x == 0) {
            const unsigned long long pos = atomicAdd(b.bump, static_cast<unsigned long long>(cnt));
            s_stage = pos + cnt <= b.stage_cap ? pos : ~0ull;
            b.row_cnt[e] = cnt;
            b.stage_off[e] = s_stage;
        }
        __syncthreads();
        for (uint32_t i = cnt + threadIdx.x; i < n2; i += blockDim.x) keys[i] = 0xffffffffu;
        __syncthreads();
        if (cnt > 1) bitonic_sort(keys, n2);
        if (MODE == 2 && s_stage == ~0ull) continue;  // staging buffer full: the host reruns MODE 1
        uint32_t* out = MODE == 2 ? b.stage + s_stage : b.cols + b.row_off[e];
        for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) out[i] = keys[i];
    }
}

// staged rows -> their CSR positions (one warp per edge)
__global__ void __launch_bounds__(256) sweep_gather_kernel(uint64_t edges, const uint32_t* __restrict__ row_cnt,
                                                            const uint64_t* __restrict__ stage_off,
                                                            const uint32_t* __restrict__ stage,
                                                            const uint64_t* __restrict__ row_off,
                                                            uint32_t* __restrict__ cols) {
    const int lane = threadIdx.x & 31;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x >> 5) + (threadIdx.x >> 5); e < edges; e += nw) {
        const uint64_t so = stage_off[e];
        if (so == ~0ull) continue;  // an overflow row: written by the global-memory pass
        const uint32_t n = row_cnt[e];
        const uint32_t* src = stage + so;
        uint32_t* dst = cols + row_off[e];
        for (uint32_t i = lane; i < n; i += 32) dst[i] = src[i];
    }
}

// exclusive scan of u32 counts into u64 offsets [0, n]: per-block sums,
// one block scanning them, per-block scan + block base
__global__ void __launch_bounds__(1024) scan_block_sums(const uint32_t* __restrict__ cnt, uint64_t n,
                                                         uint64_t* __restrict__ bsum) {
    __shared__ uint64_t red[32];
    const uint64_t i = blockIdx.x * 1024ull + threadIdx.x;
    uint64_t v = i < n ? cnt[i] : 0;
    for (int d = 16; d; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = red[threadIdx.x];
        for (int d = 16; d; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
        if (threadIdx.x == 0) bsum[blockIdx.x] = v;
    }
}

__global__ void __launch_bounds__(1024) scan_sums(uint64_t* __restrict__ bsum, uint32_t nb) {
    __shared__ uint64_t part[1024];
    const uint32_t per = (nb + 1023) / 1024, b = threadIdx.x * per, e = b + per < nb ? b + per : nb;
    uint64_t s = 0;
    for (uint32_t i = b; i < e; ++i) s += bsum[i];
    part[threadIdx.x] = s;
    __syncthreads();
    for (uint32_t d = 1; d < 1024; d <<= 1) {
        const uint64_t v = threadIdx.x >= d ? part[threadIdx.x - d] : 0;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    uint64_t acc = part[threadIdx.x] - s;
    for (uint32_t i = b; i < e; ++i) {
        const uint64_t v = bsum[i];
        bsum[i] = acc;
        acc += v;
    }
}

__global__ void __launch_bounds__(1024) scan_apply(const uint32_t* __restrict__ cnt, uint64_t n,
                                                    const uint64_t* __restrict__ bbase, uint64_t* __restrict__ off) {
    __shared__ uint64_t warp_tot[32];
    const uint64_t i = blockIdx.x * 1024ull + threadIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t v = i < n ? cnt[i] : 0;
    uint64_t x = v;
    for (int d = 1; d < 32; d <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
        uint64_t t = warp_tot[lane];
        for (int d = 1; d < 32; d <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, t, d);
            if (lane >= d) t += y;
        }
        warp_tot[lane] = t;
    }
    __syncthreads();
    const uint64_t incl = x + (w ? warp_tot[w - 1] : 0) + bbase[blockIdx.x];
    if (i < n) off[i + 1] = incl;
    if (i == 0) off[0] = 0;
}

size_t sweep_smem_bytes() { return kSweepTable * sizeof(unsigned long long) + kSweepCap * sizeof(uint32_t); }

cudaError_t launch_sweep(int mode, bool global, const SweepParams& p, const SweepBufs& b, uint32_t glog2,
                         int gblocks, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(b.edge_ctr, 0, sizeof(uint32_t), st);
    if (e != cudaSuccess) return e;
    if (global) {
        auto gk = mode == 1 ? sweep_kernel<1, true> : sweep_kernel<0, true>;
        gk<<<gblocks, kSweepThreads, 0, st>>>(p, b, glog2);
        return cudaGetLastError();
    }
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = sweep_smem_bytes();
    auto kern = mode == 2 ? sweep_kernel<2, false> : mode == 1 ? sweep_kernel<1, false> : sweep_kernel<0, false>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSweepThreads, smem);
    if (per_sm <= 0) per_sm = 1;
    uint64_t blocks = static_cast<uint64_t>(sms) * per_sm;
    if (blocks > p.edges) blocks = p.edges ? p.edges : 1;
    kern<<<static_cast<unsigned>(blocks), kSweepThreads, smem, st>>>(p, b, glog2);
    return cudaGetLastError();
}

cudaError_t launch_sweep_gather(uint64_t edges, const SweepBufs& b, cudaStream_t st) {
    if (!edges) return cudaSuccess;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t want = (edges + 7) / 8;
    const unsigned blocks = static_cast<unsigned>(want < static_cast<uint64_t>(sms) * 8 ? want : sms * 8);
    sweep_gather_kernel<<<blocks, 256, 0, st>>>(edges, b.row_cnt, b.stage_off, b.stage, b.row_off, b.cols);
    return cudaGetLastError();
}

cudaError_t launch_scan_counts(const uint32_t* cnt, uint64_t n, uint64_t* bsum, uint64_t* off, cudaStream_t st) {
    const uint64_t nb = (n + 1023) / 1024;
    if (nb == 0) return cudaMemsetAsync(off, 0, sizeof(uint64_t), st);
    scan_block_sums<<<static_cast<unsigned>(nb), 1024, 0, st>>>(cnt, n, bsum);
    scan_sums<<<1, 1024, 0, st>>>(bsum, static_cast<uint32_t>(nb));
    scan_apply<<<static_cast<unsigned>(nb), 1024, 0, st>>>(cnt, n, bsum, off);
    return cudaGetLastError();
}

}  // namespace ltlg
