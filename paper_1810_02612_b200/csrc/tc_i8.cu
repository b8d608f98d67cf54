// tc_i8.cu -- the tcgen05 kind::i8 formulation of the multi-frame labelling
// (north_star: "a tcgen05 kind::i8 dense-contraction variant (threshold > 0)
// is kept only if ncu shows it beating the bit-packed path").  In the A/B
// build only (libltlgrid_gpu_ab.so, dev knob LTLG_TC=1); measured against
// label_wm_kernel in DESIGN.md (N1).
//
// Per word group of the word-major copy (rows sharing 64-cell word w):
//   A (M = 128 rows x K = 64 cells, u8 0/1): the group's pair masks, expanded
//   B (N columns x K = 64 cells, u8 0/1):   every (frame f, prop j) whose
//     P_j[w] is non-zero in frame f (the word's column list, tc_build_kernel)
//   C = A . B^T (s32, in TMEM): swept cells the pair shares with P_j[w]
// and label bit j of (row, f) = C > 0 (threshold > 0): the OR-AND product as
// an integer contraction.  Columns with P_j[w] = 0 never hit and are left
// out, so N is the word's non-zero (frame, prop) count, not F x props.
// One CTA (4 warps) per group at a time: threads expand A and B into shared
// memory in the canonical no-swizzle K-major layout (8-row x 16-byte core
// matrices), one thread issues two tcgen05.mma (K = 32 each) per 256-column
// N tile and commits to an mbarrier, and each warp reads its 32 TMEM lanes
// (rows) back with tcgen05.ld.32x32b and ORs the hits into the CTA's
// frame-major label block (as label_wm_kernel does).  The operands are
// built from bits by the threads, not loaded by TMA: the bit -> byte
// expansion is the format change the contraction needs.
#include <cuda_runtime.h>

#include <cstdint>

#include "engine.h"
#include "launch.h"

namespace ltlg {

namespace {

constexpr int kTcThreads = 128;
constexpr uint32_t kTcCap = 1024;   // column capacity per word (the build flags overflow)
constexpr uint32_t kTcNTile = 256;  // N per MMA
constexpr uint32_t kTcRows = 128;   // rows per task at most (the default task size)

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// no-swizzle K-major shared-memory matrix descriptor (tcgen05): start, LBO
// (between the two 16-byte K halves of one MMA K step), SBO (between 8-row
// groups), version 1, layout SWIZZLE_NONE
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return static_cast<uint64_t>((addr >> 4) & 0x3fffu) | static_cast<uint64_t>((lbo >> 4) & 0x3fffu) << 16 |
           static_cast<uint64_t>((sbo >> 4) & 0x3fffu) << 32 | 1ull << 46;
}

// instruction descriptor, kind::i8: u8 x u8 -> s32, both K-major, M = 128
__device__ __forceinline__ uint32_t idesc_i8(uint32_t n) {
    return (2u << 4) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}

// the core-matrix offset of (row r, 16-byte K chunk q) in a tile of K = 64 bytes
__device__ __forceinline__ uint32_t core_off(uint32_t r, uint32_t q) {
    return (r >> 3) * 512u + q * 128u + (r & 7u) * 16u;  // SBO = 512, LBO = 128
}

// 64 bits -> 64 bytes of 0/1, written as four 16-byte chunks of one row
__device__ __forceinline__ void expand_row(uint8_t* tile, uint32_t r, uint64_t bits) {
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q) {
        uint32_t w[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const uint32_t nib = static_cast<uint32_t>(bits >> (16 * q + 4 * b)) & 0xfu;
            // spread 4 bits into 4 bytes
            w[b] = (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
        }
        *reinterpret_cast<uint4*>(tile + core_off(r, q)) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

}  // namespace

// Per grid word (warp per word): its non-zero (frame, prop) columns
// {P lo, P hi, 4 (f + 64 (j / 32)) | (j % 32) << 24} and their count.
__global__ void __launch_bounds__(256) tc_build_kernel(const uint64_t* __restrict__ P64, int props, int frames,
                                                       uint32_t nw64, uint64_t cells, uint4* __restrict__ cols,
                                                       uint32_t* __restrict__ ncol, uint32_t* __restrict__ task_ctr,
                                                       int nctr, const uint32_t* __restrict__ touched64,
                                                       uint32_t* __restrict__ overflow) {
    const uint32_t gt = blockIdx.x * blockDim.x + threadIdx.x;
    if (gt < static_cast<uint32_t>(nctr)) task_ctr[gt] = 0;
    const uint32_t w = gt >> 5, lane = threadIdx.x & 31;
    if (w > nw64) return;
    const bool live = w < nw64 && static_cast<uint64_t>(w) * 64 < cells &&
                      !(touched64 && !(__ldg(touched64 + (w >> 5)) >> (w & 31) & 1u));
    const uint64_t lo = static_cast<uint64_t>(w) * 64;
    const uint64_t valid = !live ? 0ull : (cells - lo >= 64) ? ~0ull : ((1ull << (cells - lo)) - 1ull);
    uint32_t n = 0;
    for (int f = 0; f < frames && live; ++f)
        for (int j0 = 0; j0 < props; j0 += 32) {
            const int j = j0 + static_cast<int>(lane);
            const uint64_t x = j < props ? __ldg(P64 + (static_cast<uint64_t>(f) * props + j) * nw64 + w) & valid : 0ull;
            const uint32_t nz = __ballot_sync(0xffffffffu, x != 0);
            const uint32_t pos = n + __popc(nz & ((1u << lane) - 1u));
            if (x != 0 && pos < kTcCap)
                cols[static_cast<uint64_t>(w) * kTcCap + pos] =
                    make_uint4(static_cast<uint32_t>(x), static_cast<uint32_t>(x >> 32),
                               4u * (static_cast<uint32_t>(f) + 64u * static_cast<uint32_t>(j >> 5)), 1u << (j & 31));
            n += __popc(nz);
        }
    if (lane == 0) {
        ncol[w] = n < kTcCap ? n : kTcCap;
        if (n > kTcCap) atomicAdd(overflow, 1u);
    }
}

template <typename SW, int PW>
__global__ void __launch_bounds__(kTcThreads)
    label_tc_kernel(const uint64_t* __restrict__ emask, const uint8_t* __restrict__ erow,
                    const uint32_t* __restrict__ gword, const uint32_t* __restrict__ gstart,
                    const uint32_t* __restrict__ task_row, const uint32_t* __restrict__ task_grp, uint32_t task_begin,
                    uint32_t ntasks, uint32_t* __restrict__ task_ctr, const uint4* __restrict__ cols,
                    const uint32_t* __restrict__ ncol, int frames, const uint32_t* __restrict__ perm,
                    SW* __restrict__ out, uint32_t ostride) {
    constexpr int RW = 64 * PW;
    extern __shared__ __align__(1024) uint8_t tc_raw[];
    uint8_t* sA = tc_raw;                                                  // 128 x 64 bytes
    uint8_t* sB = tc_raw + 128 * 64;                                       // kTcNTile x 64 bytes
    uint32_t* s_acc = reinterpret_cast<uint32_t*>(tc_raw + (128 + kTcNTile) * 64);  // kTcRows x RW
    __shared__ uint4 s_col[kTcNTile];  // the tile's column targets
    __shared__ uint32_t s_row[128];
    __shared__ uint64_t s_bar;
    __shared__ uint32_t s_tmem, s_task;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_addr(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&s_bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int k = tid; k < static_cast<int>(kTcRows) * RW; k += kTcThreads) s_acc[k] = 0;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    uint32_t phase = 0;
    const uint32_t idesc = idesc_i8(kTcNTile);
    for (;;) {
        if (tid == 0) s_task = task_begin + atomicAdd(task_ctr, 1u);
        __syncthreads();
        const uint32_t t = s_task;
        if (t >= ntasks) break;
        const uint32_t r0 = task_row[t], nr = task_row[t + 1] - r0;
        for (uint32_t g = task_grp[t]; g < task_grp[t + 1]; ++g) {
            const uint32_t w = __ldg(gword + g), e0 = __ldg(gstart + g), e1 = __ldg(gstart + g + 1);
            const uint32_t nc = __ldg(ncol + w);
            for (uint32_t eb = e0; eb < e1; eb += 128) {  // (groups of more than 128 pairs: several M tiles)
                const uint32_t e = eb + tid;
                const bool on = e < e1;
                expand_row(sA, tid, on ? __ldg(emask + e) : 0ull);
                s_row[tid] = on ? __ldg(erow + e) : 0xffffffffu;
                for (uint32_t nb = 0; nb < nc; nb += kTcNTile) {
                    for (uint32_t c = tid; c < kTcNTile; c += kTcThreads) {
                        const uint4 col = nb + c < nc ? __ldg(cols + static_cast<uint64_t>(w) * kTcCap + nb + c)
                                                      : make_uint4(0u, 0u, 0u, 0u);
                        expand_row(sB, c, (static_cast<uint64_t>(col.y) << 32) | col.x);
                        s_col[c] = col;
                    }
                    // the generic-proxy tile writes, visible to the tensor core
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncthreads();
                    if (tid == 0) {
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                        for (uint32_t k = 0; k < 2; ++k) {  // K = 64 cells = two K = 32 steps (two core-matrix columns each)
                            const uint64_t da = sdesc(smem_addr(sA) + 256u * k, 128u, 512u);
                            const uint64_t db = sdesc(smem_addr(sB) + 256u * k, 128u, 512u);
                            asm volatile(
                                "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %4, 0;\n\t"
                                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                                "l"(da), "l"(db), "r"(idesc), "r"(k));
                        }
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                         smem_addr(&s_bar))
                                     : "memory");
                    }
                    // wait for the MMA, then each warp reads its 32 rows (TMEM lanes)
                    {
                        uint32_t done = 0;
                        while (!done)
                            asm volatile(
                                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                                "selp.u32 %0, 1, 0, p;\n\t}"
                                : "=r"(done)
                                : "r"(smem_addr(&s_bar)), "r"(phase)
                                : "memory");
                        phase ^= 1u;
                    }
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t row = s_row[tid];
                    const uint32_t ntile = nc - nb < kTcNTile ? nc - nb : kTcNTile;
                    for (uint32_t c0 = 0; c0 < ntile; c0 += 16) {
                        uint32_t v[16];
                        asm volatile(
                            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                              "=r"(v[14]), "=r"(v[15])
                            : "r"(tmem + ((32u * warp) << 16) + c0));
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                        if (row != 0xffffffffu) {
#pragma unroll
                            for (int q = 0; q < 16; ++q) {
                                if (c0 + q < ntile && v[q] > 0u) {  // threshold > 0: the pair meets P_j[w] in frame f
                                    const uint4 col = s_col[c0 + q];
                                    atomicOr(&s_acc[row * RW + col.z / 4u], col.w);
                                }
                            }
                        }
                    }
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    __syncthreads();  // (the tiles are rewritten next)
                }
            }
        }
        __syncthreads();
        for (uint32_t r = tid; r < nr; r += kTcThreads) {  // thread r stores row r's frames
            SW* o = out + static_cast<uint64_t>(__ldg(perm + r0 + r)) * ostride;
            for (int f = 0; f < frames; ++f) {
                uint64_t l = s_acc[r * RW + f];
                if constexpr (PW == 2) l |= static_cast<uint64_t>(s_acc[r * RW + 64 + f]) << 32;
                o[f] = static_cast<SW>(l);
            }
            for (int k = 0; k < RW; ++k) s_acc[r * RW + k] = 0;
        }
        __syncthreads();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

// work buffer: columns (kTcCap per word), counts, overflow flag
size_t tc_work_bytes(uint32_t nw64) { return (static_cast<size_t>(nw64) + 1) * (kTcCap * 16 + 4) + 16; }

cudaError_t launch_tc_build(const uint64_t* P64, int props, int frames, uint32_t nw64, uint64_t cells, void* work,
                            uint32_t* task_ctr, int nctr, cudaStream_t st, const uint32_t* touched64) {
    uint8_t* wb = static_cast<uint8_t*>(work);
    uint4* cols = reinterpret_cast<uint4*>(wb);
    uint32_t* ncol = reinterpret_cast<uint32_t*>(wb + (static_cast<size_t>(nw64) + 1) * kTcCap * 16);
    uint32_t* over = ncol + nw64 + 1;
    cudaMemsetAsync(over, 0, 4, st);
    const uint64_t threads = (static_cast<uint64_t>(nw64) + 1) * 32;
    const uint64_t need = threads > static_cast<uint64_t>(nctr) ? threads : static_cast<uint64_t>(nctr);
    tc_build_kernel<<<static_cast<unsigned>((need + 255) / 256), 256, 0, st>>>(P64, props, frames, nw64, cells, cols,
                                                                              ncol, task_ctr, nctr, touched64, over);
    return cudaGetLastError();
}

template <typename SW, int PW>
static cudaError_t launch_tc_t(const LaunchArgs& a, cudaStream_t st) {
    const uint8_t* wb = static_cast<const uint8_t*>(a.sf);
    const uint4* cols = reinterpret_cast<const uint4*>(wb);
    const uint32_t* ncol = reinterpret_cast<const uint32_t*>(wb + (static_cast<size_t>(a.nw64) + 1) * kTcCap * 16);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t smem = (128 + kTcNTile) * 64 + static_cast<size_t>(kTcRows) * 64 * PW * 4;
    cudaFuncSetAttribute(label_tc_kernel<SW, PW>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    label_tc_kernel<SW, PW><<<sms * 2, kTcThreads, smem, st>>>(a.wm_mask, a.wm_row, a.wm_gword, a.wm_gstart, a.wm_task_row,
                                                          a.wm_task_grp, a.task_begin, a.ntasks, a.task_ctr, cols, ncol,
                                                          a.frames, a.perm, static_cast<SW*>(a.out),
                                                          a.ostride ? a.ostride : static_cast<uint32_t>(a.frames));
    return cudaGetLastError();
}

cudaError_t launch_tc_label(const LaunchArgs& a, cudaStream_t st) {
    if (a.wm_rows > static_cast<int>(kTcRows)) return cudaErrorInvalidValue;
    switch (a.label_bytes) {
        case 1: return launch_tc_t<uint8_t, 1>(a, st);
        case 2: return launch_tc_t<uint16_t, 1>(a, st);
        case 4: return launch_tc_t<uint32_t, 1>(a, st);
        default: return launch_tc_t<uint64_t, 2>(a, st);
    }
}

}  // namespace ltlg
