// pssgp_f32.h — internal interface between the C ABI (pssgp_api.cu) and the optional fp32
// build of the thread-per-chain kernels (pssgp_f32.cu, north_star "an optional
// fp32 path must match to 1e-3").  Plain types only; not part of include/pssgp.h.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace pssgp_f32 {

struct Run {
    int d;                      // state dimension 1..3 (single Matern component, closed form)
    int64_t n, K;               // steps, chain length
    int nb;                     // CTAs (one wave)
    const double* t;            // times (fp64 in every build)
    const double* y;
    const uint8_t* mask;
    double* mean;               // nullable (NLL only when mean == var == nullptr)
    double* var;
    double* nll;                // nullable
    void* ws;                   // workspace of ws_bytes(d, K, nb) bytes
    unsigned long long* err;    // device error word
    unsigned long long* flag;   // K3 carry publication word
    double lam, s2, r;          // Matern lambda, sigma^2, noise variance
    double Pinf[6];             // P_inf in the Jordan basis (packed upper)
    cudaStream_t stream;
};

// resident CTAs per SM of the fp32 kernels (min over K1, K3, K5) for state dimension d
int occupancy(int d);
size_t ws_bytes(int d, int64_t K, int nb);
// phase 1 = K1 (fold), 2 = K3 (Kalman rescan; stores the filtered state when mean/var are
// requested), 3 = K5 (RTS rescan + NLL sum), 4 = NLL sum only.  Returns the launch error.
cudaError_t launch(const Run& r, int phase);

}  // namespace pssgp_f32
