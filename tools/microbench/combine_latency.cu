// Latency of chained filter / smoother aggregate combines (d = 3) and of the aggregate shuffles:
// one warp, 64 dependent operations, clock64 around them.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include "../../paper_2102_09964_b200/csrc/pssgp_kernels.cuh"
using namespace pssgp;

__global__ void k(const double* in, double* out, long long* cyc) {
    FAgg<3> a, b;
    for (int i = 0; i < 27; ++i) { reinterpret_cast<double*>(&a)[i] = in[i]; reinterpret_cast<double*>(&b)[i] = in[27 + i]; }
    long long t0 = clock64();
    for (int r = 0; r < 64; ++r) { FAgg<3> o; combine(a, b, o); a = o; }
    long long t1 = clock64();
    for (int r = 0; r < 64; ++r) { FAgg<3> o; shfl_down_all(o, a, 1); a = o; }
    long long t2 = clock64();
    SAgg<3> s, u;
    for (int i = 0; i < 18; ++i) { reinterpret_cast<double*>(&s)[i] = in[i]; reinterpret_cast<double*>(&u)[i] = in[20 + i]; }
    long long t3 = clock64();
    for (int r = 0; r < 64; ++r) { SAgg<3> o; combine(s, u, o); s = o; }
    long long t4 = clock64();
    Gauss<3> g;
    for (int i = 0; i < 9; ++i) reinterpret_cast<double*>(&g)[i] = in[i];
    long long t5 = clock64();
    for (int r = 0; r < 64; ++r) { Gauss<3> o; apply_prefix(g, b, o); g = o; }
    long long t6 = clock64();
    if (threadIdx.x == 0) {
        cyc[0] = (t1 - t0) / 64; cyc[1] = (t2 - t1) / 64; cyc[2] = (t4 - t3) / 64; cyc[3] = (t6 - t5) / 64;
        for (int i = 0; i < 27; ++i) out[i] = reinterpret_cast<double*>(&a)[i] + reinterpret_cast<double*>(&s)[i % 18] + reinterpret_cast<double*>(&g)[i % 9];
    }
}

int main() {
    double h[64];
    for (int i = 0; i < 64; ++i) h[i] = 0.01 * (i % 7) + ((i % 10) == 0 ? 1.0 : 0.0);
    double *din, *dout; long long* dc;
    cudaMalloc(&din, sizeof(h)); cudaMalloc(&dout, 64 * 8); cudaMalloc(&dc, 4 * 8);
    cudaMemcpy(din, h, sizeof(h), cudaMemcpyHostToDevice);
    k<<<1, 32>>>(din, dout, dc);
    k<<<1, 32>>>(din, dout, dc);
    long long c[4];
    cudaMemcpy(c, dc, sizeof(c), cudaMemcpyDeviceToHost);
    printf("cycles per op: filter combine %lld, FAgg shuffle %lld, smoother combine %lld, apply_prefix %lld\n", c[0], c[1], c[2], c[3]);
    return 0;
}
