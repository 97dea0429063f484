// Microbenchmark: FP64 tensor (DMMA.8x8x4 via mma.sync.m8n8k4.f64) and FP64 FMA (DFMA)
// throughput on one B200. Sets the roofline denominator for the Θ contraction.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters) {
    double a = threadIdx.x * 1e-9, b = 1.0 + threadIdx.x * 1e-9;
    double c[CHAINS][2];
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0; c[i][1] = 0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.0) out[threadIdx.x] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters) {
    double a = threadIdx.x * 1e-9, b = 1.0 + threadIdx.x * 1e-9;
    double c[CHAINS];
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) c[i] = fma(a, c[i], b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) s += c[i];
    if (s == 12345.0) out[threadIdx.x] = s;
}

int main() {
    int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
    int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_per_block_optin\": %zu, \"clock_khz\": %d}\n",
           p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin, clk);
    double* out; CK(cudaMalloc(&out, 1 << 20));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int sms = p.multiProcessorCount;
    for (int wpb : {4, 8, 16}) for (int bps : {1, 2, 4}) {
        int iters = 20000;
        dim3 grid(sms * bps), block(32 * wpb);
        dmma_loop<8><<<grid, block>>>(out, 100);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        dmma_loop<8><<<grid, block>>>(out, iters);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 256.0 * 8 * iters * (double)grid.x * wpb;  // 256 FMA per DMMA per warp
        printf("{\"kind\": \"dmma_m8n8k4\", \"warps_per_block\": %d, \"blocks_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n",
               wpb, bps, ms, flops / ms / 1e9);
    }
    for (int wpb : {4, 8, 16}) for (int bps : {1, 2, 4}) {
        int iters = 20000;
        dim3 grid(sms * bps), block(32 * wpb);
        dfma_loop<8><<<grid, block>>>(out, 100);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        dfma_loop<8><<<grid, block>>>(out, iters);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * iters * (double)grid.x * block.x;
        printf("{\"kind\": \"dfma\", \"warps_per_block\": %d, \"blocks_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n",
               wpb, bps, ms, flops / ms / 1e9);
    }
    // sustained DMMA for ~3 s (clock/power behaviour under FP64 tensor load)
    {
        dim3 grid(sms * 2), block(256);
        int iters = 200000;
        cudaEventRecord(e0);
        for (int r = 0; r < 4; ++r) dmma_loop<8><<<grid, block>>>(out, iters);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 4 * 2.0 * 256.0 * 8 * iters * (double)grid.x * 8;
        printf("{\"kind\": \"dmma_sustained\", \"ms\": %.3f, \"tflops\": %.2f}\n", ms, flops / ms / 1e9);
    }
    return 0;
}
