// Dependent-chain latency of DFMA / DMUL / DADD and of the rcp/exp helpers on B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double a, double b, int n) {
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a); }
    long long t1 = clock64();
    double y = a;
    for (int i = 0; i < n; ++i) { y = y * b; y = y * b; y = y * b; y = y * b; }
    long long t2 = clock64();
    double z = a;
    for (int i = 0; i < n; ++i) { z = z + b; z = z + b; z = z + b; z = z + b; }
    long long t3 = clock64();
    out[0] = x + y + z;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 64); cudaMalloc(&c, 64);
    lat<<<1, 1>>>(o, c, 1.0, 0.999999, 1024);
    lat<<<1, 1>>>(o, c, 1.0, 0.999999, 1024);
    long long h[3]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    printf("dependent latency (cycles): DFMA %.2f  DMUL %.2f  DADD %.2f\n", h[0] / 4096.0, h[1] / 4096.0, h[2] / 4096.0);
    return 0;
}
