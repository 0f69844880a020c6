// FP64 pipe throughput microbenchmark (B200, sm_100a).  Measures DFMA/DMUL rate
// with (a) three distinct register operands, (b) one constant-bank operand,
// (c) DMUL.  Independent accumulator chains per thread hide latency.
#include <cstdio>
#include <cuda_runtime.h>

__constant__ double cc[8] = {1.0000001, 0.9999999, 1.0000002, 0.9999998, 1.0000003, 0.9999997, 1.0000004, 0.9999996};

template <int MODE>
__global__ void __launch_bounds__(256) kern(double* out, int iters, double s) {
    constexpr int C = 8;
    double acc[C], x[C], y[C];
#pragma unroll
    for (int i = 0; i < C; ++i) { acc[i] = threadIdx.x * 1e-3 + i; x[i] = s + i * 1e-7; y[i] = 1e-9 * i - s * 1e-3; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < C; ++i) {
            if (MODE == 0) acc[i] = fma(acc[i], x[i], y[i]);          // 3 register operands
            if (MODE == 1) acc[i] = fma(acc[i], x[i], cc[i]);         // constant-bank addend
            if (MODE == 2) acc[i] = acc[i] * x[i];                    // DMUL
            if (MODE == 3) acc[i] = fma(acc[i], x[0], y[0]);          // shared operands (reuse)
        }
    }
    double r = 0;
#pragma unroll
    for (int i = 0; i < C; ++i) r += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int MODE>
void run(const char* name, int sms) {
    const int blocks = sms * 8, threads = 256, iters = 4096;
    double* out;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    kern<MODE><<<blocks, threads>>>(out, 16, 1.0);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<MODE><<<blocks, threads>>>(out, iters, 1.0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double ops = double(blocks) * threads * iters * 8;  // fp64 instructions (thread level)
    const double flop = ops * (MODE == 2 ? 1 : 2);
    printf("%-28s %8.3f ms  %7.2f T fp64-instr/s  %7.2f TFLOP/s\n", name, ms, ops / ms / 1e9, flop / ms / 1e9);
    cudaFree(out);
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("SMs %d, clock %.0f MHz, nominal 64 DFMA/clk/SM -> %.2f TFLOP/s\n", sms, clk / 1e3, sms * 64 * 2 * clk * 1e3 / 1e12);
    for (int rep = 0; rep < 2; ++rep) {
        run<0>("DFMA 3 reg operands", sms);
        run<1>("DFMA const addend", sms);
        run<2>("DMUL", sms);
        run<3>("DFMA shared operands", sms);
    }
    return 0;
}
