// pssgp_f32.cu — the optional fp32 build of the thread-per-chain path (
// north_star: "An optional fp32 path must match to 1e-3"), for single Matern components
// (closed form, d <= 3; SURVEY.md §8(b) "scope fp32 to Matern configs").
//
// The same kernel source as the fp64 path (pssgp_kernels.cuh, pssgp_math.cuh), compiled a second
// time with real = float in namespace pssgp_f32: moments, aggregates, F, Q and the filtered state
// in HBM are fp32; times, observations, mean / var outputs and the NLL accumulation stay fp64
// (fp32 ulp at t ~ 2048 exceeds the step).
#define PSSGP_NS pssgp_f32
#define PSSGP_REAL float
#define PSSGP_MINB 4
#include "pssgp_kernels.cuh"
#include "pssgp_f32.h"

namespace pssgp_f32 {

namespace {

template <int D>
int occ() {
    int a = 0, b = 0, c = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_filter_reduce<D, kClosed>, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_filter_apply<D, kClosed>, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, k_smoother_apply<D, kClosed>, kThreads, 0);
    return a < b ? (a < c ? a : c) : (b < c ? b : c);
}

template <int D>
size_t ws_reals(int64_t K, int nb) {
    const size_t nchp = static_cast<size_t>(nb) * kThreads;
    return nchp * FN(D) + static_cast<size_t>(nb) * FN(D) + static_cast<size_t>(nb) * CN(D) +
           static_cast<size_t>(nb) * kWarps * K * CN(D) * 32 + nchp * SN(D) + static_cast<size_t>(nb) * SN(D) +
           static_cast<size_t>(nb) * CN(D) + 64;
}

template <int D>
cudaError_t launch_d(const Run& r, int phase) {
    KParams<D> p;
    memset(&p, 0, sizeof(p));
    p.m.r = static_cast<float>(r.r);
    p.m.lam = static_cast<float>(r.lam);
    p.m.s2 = static_cast<float>(r.s2);
    for (int i = 0; i < ns(D); ++i) p.m.Pinf[i] = static_cast<float>(r.Pinf[i]);
    for (int i = 0; i < D; ++i) p.m.H[i] = (i == 0) ? 1.0f : 0.0f;
    p.m.closed = 1;
    p.m.h_unit = 1;
    const size_t nchp = static_cast<size_t>(r.nb) * kThreads;
    // NLL partials first (fp64, 8-byte aligned), then the fp32 state buffers
    p.nll_block = reinterpret_cast<double*>(r.ws);
    float* w = reinterpret_cast<float*>(p.nll_block + r.nb + (r.nb & 1));
    p.chain_f = w; w += nchp * FN(D);
    p.block_f = w; w += static_cast<size_t>(r.nb) * FN(D);
    p.fcarry = w; w += static_cast<size_t>(r.nb) * CN(D);
    w += (reinterpret_cast<uintptr_t>(w) >> 2) & 1;   // 8-byte aligned records (paired state loads)
    p.xp = w; w += static_cast<size_t>(r.nb) * kWarps * r.K * CN(D) * 32;
    p.chain_s = w; w += nchp * SN(D);
    p.block_s = w; w += static_cast<size_t>(r.nb) * SN(D);
    p.scarry = w;
    p.t = r.t; p.y = r.y; p.mask = r.mask;
    p.n = r.n; p.k0 = 0; p.nglob = r.n;
    p.K = r.K; p.nb = r.nb;
    p.mean = r.mean; p.var = r.var;
    p.err = r.err; p.flag = r.flag;
    p.rank = 0; p.world = 1;
    const bool smooth = r.mean || r.var;
    p.store_state = smooth ? 1 : 0;
    switch (phase) {
        case 1: k_filter_reduce<D, kClosed><<<r.nb, kThreads, 0, r.stream>>>(p); break;
        case 2:
            if (smooth) k_filter_apply<D, kClosed><<<r.nb, kThreads, 0, r.stream>>>(p);
            else k_filter_apply<D, kClosed, false><<<r.nb, kThreads, 0, r.stream>>>(p);
            break;
        case 3:
            p.nll_out = r.nll;
            k_smoother_apply<D, kClosed><<<r.nb, kThreads, 0, r.stream>>>(p);
            break;
        case 4: k_nll_sum<<<1, kThreads, 0, r.stream>>>(p.nll_block, r.nb, r.nll, 1); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace

int occupancy(int d) {
    const int o = d == 1 ? occ<1>() : d == 2 ? occ<2>() : occ<3>();
    return o > 0 ? o : 1;
}

size_t ws_bytes(int d, int64_t K, int nb) {
    const size_t nr = d == 1 ? ws_reals<1>(K, nb) : d == 2 ? ws_reals<2>(K, nb) : ws_reals<3>(K, nb);
    return nr * sizeof(float) + (static_cast<size_t>(nb) + 2) * sizeof(double);
}

cudaError_t launch(const Run& r, int phase) {
    switch (r.d) {
        case 1: return launch_d<1>(r, phase);
        case 2: return launch_d<2>(r, phase);
        case 3: return launch_d<3>(r, phase);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace pssgp_f32
