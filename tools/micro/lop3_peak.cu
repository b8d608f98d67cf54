// LOP3 throughput microbenchmark ("measure it on the box with a
// LOP3 microbench, as MEASURED_PEAKS does for HBM").  Every thread runs 8
// independent chains of `a = (a & b) | c` (one LOP3.LUT each) over many
// iterations; the grid fills every SM.  Prints LOP3/s and LOP3/clk/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lop3_peak lop3_peak.cu && ./lop3_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lop3_kernel(unsigned* out, unsigned iters, unsigned seed) {
    unsigned a[8], b = seed * 0x9E3779B9u + threadIdx.x, c = seed ^ 0x5bd1e995u;
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * (k + 1) + blockIdx.x;
    for (unsigned i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(a[k]) : "r"(b), "r"(c));
        b += 1;  // keep the operands live (one IADD per 8 LOP3)
    }
    unsigned x = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) x ^= a[k];
    if (x == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

int main() {
    int dev = 0, sms = 0, clk_khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    unsigned* out;
    cudaMalloc(&out, 1 << 24);
    const int threads = 512, blocks = sms * 4;
    const unsigned iters = 1 << 16;
    lop3_kernel<<<blocks, threads>>>(out, 1024, 1);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        lop3_kernel<<<blocks, threads>>>(out, iters, rep + 2);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double ops = double(blocks) * threads * iters * 8.0;
    const double per_s = ops / (best / 1e3);
    printf("{\"lop3_per_s\": %.6g, \"sms\": %d, \"max_clock_mhz\": %.1f, \"lop3_per_clk_per_sm_at_max_clock\": %.2f, "
           "\"kernel_ms\": %.4f}\n",
           per_s, sms, clk_khz / 1e3, per_s / sms / (clk_khz * 1e3), best);
    return 0;
}
