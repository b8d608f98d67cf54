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

// FILL = false: row sizes into row_cnt; true: rows into cols at row_off.
// GLOBAL = false: every edge, shared-memory sets (an overflowing edge is
// listed in over_list and skipped); true: the over_list edges, global-memory
// sets of 2^glog2 entries per CTA (an overflow there bumps err_key[1] and the
// host retries with a larger table).
template <bool FILL, bool GLOBAL>
__global__ void __launch_bounds__(kSweepThreads)
    sweep_kernel(SweepParams p, uint32_t* __restrict__ edge_ctr, uint32_t* __restrict__ row_cnt,
                 const uint64_t* __restrict__ row_off, uint32_t* __restrict__ cols, uint32_t* __restrict__ over_list,
                 uint32_t* __restrict__ n_over, unsigned long long* __restrict__ gtab, uint32_t* __restrict__ gkeys,
                 uint32_t glog2) {
    extern __shared__ unsigned long long smem_tab[];
    __shared__ uint32_t s_edge, s_cnt, s_pos, s_bad;
    constexpr bool kGlobal = GLOBAL;
    const uint32_t hsize = kGlobal ? (1u << glog2) : kSweepTable;
    const uint32_t cap = kGlobal ? hsize / 2 : kSweepCap;
    unsigned long long* tab = kGlobal ? gtab + static_cast<size_t>(blockIdx.x) * hsize : smem_tab;
    uint32_t* keys = kGlobal ? gkeys + static_cast<size_t>(blockIdx.x) * (hsize / 2)
                             : reinterpret_cast<uint32_t*>(smem_tab + kSweepTable);
    for (uint32_t i = threadIdx.x; i < hsize; i += blockDim.x) tab[i] = 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const double half_x = p.w[0] / 2, half_y = p.w[1] / 2;
    for (uint32_t epoch = 1;; ++epoch) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t k = atomicAdd(edge_ctr, 1u);
            s_edge = kGlobal ? (k < *n_over ? over_list[k] : 0xffffffffu) : k;
            s_cnt = 0;
            s_pos = 0;
            s_bad = 0;
        }
        __syncthreads();
        const uint32_t e = s_edge;
        if (kGlobal ? e == 0xffffffffu : e >= p.edges) break;
        const uint64_t sb = p.sample_off[e], se = p.sample_off[e + 1];
        for (uint64_t i = sb + warp; i < se; i += nwarps) {
            const double* s5 = p.samples + 5 * i;
            const double px = s5[0], py = s5[1], heading = s5[2], tau = s5[4];
            // sweep_collect (abstraction.cpp:180-199): the checks, in order
            if (!(tau >= p.lo[2] && tau < p.hi[2])) {
                if (lane == 0 && !FILL) atomicMin(p.err_key, static_cast<unsigned long long>(i) * 4 + 0);
                continue;
            }
            // GridSpec::quantize (grid.cpp:35-47) of tau
            uint64_t ct = static_cast<uint64_t>(floor((tau - p.lo[2]) / (p.hi[2] - p.lo[2]) * p.cells[2]));
            if (ct >= static_cast<uint64_t>(p.ncell[2])) ct = p.ncell[2] - 1;
            const uint32_t ct_bits = scatter3(p, 2, ct);
            if (p.length <= 0 || p.width <= 0) {  // footprint_polygon's check
                if (lane == 0 && !FILL) atomicMin(p.err_key, static_cast<unsigned long long>(i) * 4 + 1);
                continue;
            }
            double sn, cs;
            sincos(heading, &sn, &cs);
            const double rcx = px + p.ref_offset * cs, rcy = py + p.ref_offset * sn;
            const double hl = p.length / 2, hw = p.width / 2;
            const double ac = fabs(cs), as = fabs(sn);
            const double ext_x = hl * ac + hw * as;
            const double ext_y = hl * as + hw * ac;
            if (rcx - ext_x < p.lo[0] || rcx + ext_x > p.hi[0] || rcy - ext_y < p.lo[1] || rcy + ext_y > p.hi[1]) {
                if (lane == 0 && !FILL) atomicMin(p.err_key, static_cast<unsigned long long>(i) * 4 + 2);
                continue;
            }
            int64_t x0, x1, y0, y1;
            overlap_cells(p, 0, rcx - ext_x, rcx + ext_x, x0, x1);
            overlap_cells(p, 1, rcy - ext_y, rcy + ext_y, y0, y1);
            if (x1 < x0 || y1 < y0) continue;
            const uint32_t ny = static_cast<uint32_t>(y1 - y0 + 1);
            const uint32_t n = static_cast<uint32_t>(x1 - x0 + 1) * ny;
            for (uint32_t t = lane; t < n; t += 32) {
                const int64_t cx = x0 + t / ny, cy = y0 + t % ny;
                const double ccx = p.lo[0] + (static_cast<double>(cx) + 0.5) * p.w[0];
                const double ccy = p.lo[1] + (static_cast<double>(cy) + 0.5) * p.w[1];
                // rect_cell_overlap (abstraction.cpp:156-170)
                const double dx = ccx - rcx, dy = ccy - rcy;
                if (fabs(dx) >= half_x + hl * ac + hw * as) continue;
                if (fabs(dy) >= half_y + hl * as + hw * ac) continue;
                if (fabs(dx * cs + dy * sn) >= hl + half_x * ac + half_y * as) continue;
                if (fabs(-dx * sn + dy * cs) >= hw + half_x * as + half_y * ac) continue;
                const uint32_t key = scatter3(p, 0, static_cast<uint64_t>(cx)) |
                                     scatter3(p, 1, static_cast<uint64_t>(cy)) | ct_bits;
                if (!s_bad && !set_insert(tab, hsize - 1, epoch, key, &s_cnt, cap)) s_bad = 1;
            }
        }
        __syncthreads();
        const uint32_t cnt = s_cnt;
        if (!FILL) {
            if (threadIdx.x == 0) {
                row_cnt[e] = s_bad ? 0u : cnt;
                if (s_bad) {
                    if (GLOBAL) atomicAdd(p.err_key + 1, 1ull);  // retry with a larger table
                    else over_list[atomicAdd(n_over, 1u)] = e;
                }
            }
            continue;
        }
        if (s_bad) continue;  // shared-memory fill: a listed overflow edge
        // compact this edge's keys, sort them, write the row (sweep_voxelize_indices'
        // sort + unique, abstraction.cpp:214-221)
        for (uint32_t i = threadIdx.x; i < hsize; i += blockDim.x) {
            const unsigned long long v = tab[i];
            if (static_cast<uint32_t>(v >> 32) == epoch) keys[atomicAdd(&s_pos, 1u)] = static_cast<uint32_t>(v);
        }
        uint32_t n2 = 1;
        while (n2 < cnt) n2 <<= 1;
        __syncthreads();
        for (uint32_t i = cnt + threadIdx.x; i < n2; i += blockDim.x) keys[i] = 0xffffffffu;
        __syncthreads();
        if (cnt > 1) bitonic_sort(keys, n2);
        uint32_t* out = cols + row_off[e];
        for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) out[i] = keys[i];
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

cudaError_t launch_sweep(int mode, const SweepParams& p, uint32_t* edge_ctr, uint32_t* row_cnt, const uint64_t* row_off,
                         uint32_t* cols, uint32_t* over_list, uint32_t* n_over, unsigned long long* gtab,
                         uint32_t* gkeys, uint32_t glog2, int gblocks, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(edge_ctr, 0, sizeof(uint32_t), st);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // mode bit 0: fill, bit 1: global-memory sets over the overflow list
    if (mode & 2) {
        auto gk = (mode & 1) ? sweep_kernel<true, true> : sweep_kernel<false, true>;
        gk<<<gblocks, kSweepThreads, 0, st>>>(p, edge_ctr, row_cnt, row_off, cols, over_list, n_over, gtab, gkeys,
                                             glog2);
        return cudaGetLastError();
    }
    const size_t smem = sweep_smem_bytes();
    auto kern = (mode & 1) ? sweep_kernel<true, false> : sweep_kernel<false, false>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSweepThreads, smem);
    if (per_sm <= 0) per_sm = 1;
    uint64_t blocks = static_cast<uint64_t>(sms) * per_sm;
    if (blocks > p.edges) blocks = p.edges ? p.edges : 1;
    kern<<<static_cast<unsigned>(blocks), kSweepThreads, smem, st>>>(p, edge_ctr, row_cnt, row_off, cols, over_list,
                                                                     n_over, gtab, gkeys, glog2);
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
