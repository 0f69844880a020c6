// pssgp_wide.cuh — warp-per-chain kernels for larger state dimensions (4 <= D <= 32).
//
// Thread-per-chain (pssgp_kernels.cuh) keeps a whole filter aggregate in registers,
// which stops working past d = 3 (d = 6: 90 doubles, d = 16: 560).  Here one WARP
// owns one chain; every matrix of the chain lives in shared memory (full D x D,
// row stride D+1) and the 32 lanes split each matrix operation over its output
// elements.  Same three-pass structure as the d <= 3 path (PAPER.md:116-123 fold,
// 326-330 Kalman rescan, 431-435 RTS rescan), but the carries come from
// Kogge-Stone scans over the chain aggregates in which each general operator
// (x)_f / (x)_s is evaluated cooperatively by one warp (Gauss-Jordan with
// partial pivoting for (I + C_i J_j)^-1).
//
// Discretisation: uniform-dt models (F, Q precomputed on the host, copied once to
// device memory); dt == 0 -> (I, 0); any other dt -> PSSGP_E_UNSUPPORTED.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "pssgp_kernels.cuh"

namespace pssgp {
namespace wide {

constexpr int kWWarps = 4;                       // chains (warps) per CTA in the chain kernels
#ifndef PSSGP_WMINB
#define PSSGP_WMINB 1                            // min resident CTAs/SM the wide chain kernels are built for
#endif

PS_CX int LD(int D) { return D + 1; }            // padded row stride of a shared matrix
PS_CX int FNW(int D) { return 3 * D * D + 2 * D; } // full filter aggregate: A, b, C, eta, J
PS_CX int SNW(int D) { return 2 * D * D + D; }     // full smoother aggregate: E, g, L
PS_CX int CNW(int D) { return D + D * (D + 1) / 2; } // filtered (x, P packed upper)
PS_CX int MODW(int D) { return 5 * D * D + D + 2; }  // model: F, Q, Pinf, H, r, udt, G, W
PS_CX int FQW(int D) { return 2 * D * LD(D); }     // per-step F, Q (rows of stride LD) in kPade mode
// Taylor coefficient matrices of F(dt) = sum_k G^k / k! dt^k (k = 0..kPolyM) and Q(dt) = sum_k M_k dt^k
// (k = 1..kPolyM+1, M_1 = W, M_{k+1} = (G M_k + M_k G^T) / (k + 1): the Lyapunov ODE's series), host-
// computed in long double and appended to the model buffer after MODW doubles
constexpr int kPolyM = 12;
constexpr double kPolyNorm = 0.05;               // ||G dt||_1 up to which the polynomial path is used
PS_CX int MODP(int D) { return 2 * (kPolyM + 1) * D * D; }

struct WParams {
    const double* t;
    const double* y;
    const uint8_t* mask;
    int64_t n, k0, nglob, K;
    int nch;                    // chains (= warps) of this launch plan
    const double* model;        // MODW doubles
    double* fagg;               // [nch][FNW] chain filter aggregates, then their inclusive scan
    double* fbuf;               // [nch][FNW] ping-pong
    double* xp;                 // [nch][K][CNW] filtered moments
    double* sagg;               // [nch][SNW]
    double* sbuf;               // [nch][SNW]
    double* nll_chain;          // [nch]
    double* mean;
    double* var;
    double* nll_out;
    const double* in_filt;      // sharded inputs (nullable), D-specific packing = FNW / SNW
    const double* in_smooth;
    int rank, world;
    unsigned long long* err;
    int store_state;
    const double* fq;           // per-step (F, Q) [n(+1)][FQW] from kw_discretize (irregular dt), else NULL
    double* qagg;               // [nch][kQ-1][FNW] quarter prefix filter aggregates (lane-per-row fold, D <= 8)
    double* sqagg;              // [nch][kQ-1][SNW] smoother aggregates of quarters 1..3 (quarter Kalman rescan)
    double* qmom;               // [nch][2][QMW] half-chain rescan (9 <= D <= 16): each half's end moments
};
PS_CX int QMW(int D) { return 3 * D * D + 2 * D; }   // (P, Sg, P0 full; x, x0)

// ------------------------------------------------------------------ shared-memory model
template <int D>
struct SModel {
    double F[D][LD(D)];
    double Q[D][LD(D)];
    double Pinf[D][LD(D)];
    double H[D];
    double r, udt;
};

template <int D>
__device__ __forceinline__ void load_model(SModel<D>& sm, const double* __restrict__ g) {
    for (int e = threadIdx.x; e < D * D; e += blockDim.x) {
        const int i = e / D, j = e - (e / D) * D;
        sm.F[i][j] = g[e];
        sm.Q[i][j] = g[D * D + e];
        sm.Pinf[i][j] = g[2 * D * D + e];
    }
    for (int i = threadIdx.x; i < D; i += blockDim.x) sm.H[i] = g[3 * D * D + i];
    if (threadIdx.x == 0) {
        sm.r = g[3 * D * D + D];
        sm.udt = g[3 * D * D + D + 1];
    }
}

// ------------------------------------------------------------------ warp matrix primitives
// Out = A B (+ Cadd);  TA/TB: use A^T / B^T.  All D x D, shared, stride LD(D).
// D = 16 / 8: register-blocked, each lane owns an RB x CB output block (32 blocks),
// so per k it loads RB + CB operands for RB*CB FMAs; other D: one output per lane-step.
template <int D>
struct Blk {
    static constexpr bool ok = (D == 16 || D == 8);
    static constexpr int RB = (D == 16) ? 2 : 1;
    static constexpr int CB = (D == 16) ? 4 : 2;
};

#ifndef PSSGP_WMM_TILED
#define PSSGP_WMM_TILED 1
#endif
template <int D, bool TA = false, bool TB = false>
__device__ __forceinline__ void wmm(double (*Out)[LD(D)], const double (*A)[LD(D)], const double (*B)[LD(D)],
                                    const double (*Cadd)[LD(D)], int lane) {
    if constexpr (Blk<D>::ok) {
        constexpr int RB = Blk<D>::RB, CB = Blk<D>::CB, NCB = D / CB;
        const int i0 = (lane / NCB) * RB, j0 = (lane % NCB) * CB;
        double acc[RB][CB];
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int c = 0; c < CB; ++c) acc[r][c] = Cadd ? Cadd[i0 + r][j0 + c] : 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            double a[RB], b[CB];
#pragma unroll
            for (int r = 0; r < RB; ++r) a[r] = TA ? A[k][i0 + r] : A[i0 + r][k];
#pragma unroll
            for (int c = 0; c < CB; ++c) b[c] = TB ? B[j0 + c][k] : B[k][j0 + c];
#pragma unroll
            for (int r = 0; r < RB; ++r)
#pragma unroll
                for (int c = 0; c < CB; ++c) acc[r][c] = fma(a[r], b[c], acc[r][c]);
        }
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int c = 0; c < CB; ++c) Out[i0 + r][j0 + c] = acc[r][c];
    } else if constexpr (D * D <= 32 || !PSSGP_WMM_TILED) {
        for (int e = lane; e < D * D; e += 32) {
            const int i = e / D, j = e - (e / D) * D;
            double s = Cadd ? Cadd[i][j] : 0.0;
#pragma unroll 8
            for (int k = 0; k < D; ++k) s = fma(TA ? A[k][i] : A[i][k], TB ? B[j][k] : B[k][j], s);
            Out[i][j] = s;
        }
    } else {
        // other D: a 4 x 8 lane grid, each lane a register tile of RB = ceil(D / 4) contiguous rows x
        // CB = ceil(D / 8) columns strided by 8 (RB + CB shared loads per RB CB FMAs instead of 2 per
        // FMA); edge lanes clamp their loads and skip their stores.  No lane-dependent trip count.
        constexpr int PC = 8, RB = (D + 3) / 4, CB = (D + PC - 1) / PC;
        const int i0 = (lane / PC) * RB, pc = lane % PC;
        int ri[RB], cj[CB];
#pragma unroll
        for (int r = 0; r < RB; ++r) ri[r] = min(i0 + r, D - 1);
#pragma unroll
        for (int c = 0; c < CB; ++c) cj[c] = min(pc + c * PC, D - 1);
        double acc[RB][CB];
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int c = 0; c < CB; ++c) acc[r][c] = Cadd ? Cadd[ri[r]][cj[c]] : 0.0;
#pragma unroll 2
        for (int k = 0; k < D; ++k) {
            double a[RB], b[CB];
#pragma unroll
            for (int r = 0; r < RB; ++r) a[r] = TA ? A[k][ri[r]] : A[ri[r]][k];
#pragma unroll
            for (int c = 0; c < CB; ++c) b[c] = TB ? B[cj[c]][k] : B[k][cj[c]];
#pragma unroll
            for (int r = 0; r < RB; ++r)
#pragma unroll
                for (int c = 0; c < CB; ++c) acc[r][c] = fma(a[r], b[c], acc[r][c]);
        }
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int c = 0; c < CB; ++c)
                if (i0 + r < D && pc + c * PC < D) Out[i0 + r][pc + c * PC] = acc[r][c];
    }
}

// Cholesky factor of an SPD shared matrix (lower triangle of Lm, reciprocal of the
// diagonal in Li; left-looking Crout, lanes over the rows of each column, D
// warp-synchronous rounds; dot products split over two accumulators).
template <int D>
__device__ bool wcholesky(const double (*S)[LD(D)], double (*Lm)[LD(D)], double* Li, int lane) {
    bool ok = true;
    for (int j = 0; j < D; ++j) {
        double d0 = S[j][j], d1 = 0.0;
        int k = 0;
        for (; k + 1 < j; k += 2) {
            d0 = fma(-Lm[j][k], Lm[j][k], d0);
            d1 = fma(-Lm[j][k + 1], Lm[j][k + 1], d1);
        }
        if (k < j) d0 = fma(-Lm[j][k], Lm[j][k], d0);
        const double d = d0 + d1;
        ok = ok && (d > 0.0);
        const double il = rsqrt(d);
        for (int i = j + 1 + lane; i < D; i += 32) {
            double t0 = S[i][j], t1 = 0.0;
            int q = 0;
            for (; q + 1 < j; q += 2) {
                t0 = fma(-Lm[i][q], Lm[j][q], t0);
                t1 = fma(-Lm[i][q + 1], Lm[j][q + 1], t1);
            }
            if (q < j) t0 = fma(-Lm[i][q], Lm[j][q], t0);
            Lm[i][j] = (t0 + t1) * il;
        }
        if (lane == 0) {
            Lm[j][j] = d * il;
            Li[j] = il;
        }
        __syncwarp();
    }
    return ok;
}

// X[:, j] = S^-1 R[:, j] for j < D with S = Lm Lm^T: lane j solves column j
// (forward then backward substitution, vector in registers).  X may alias R.
template <int D>
__device__ __forceinline__ void wchol_solve(const double (*Lm)[LD(D)], const double* Li, const double (*R)[LD(D)],
                                            double (*X)[LD(D)], int lane) {
    if (lane < D) {
        double z[D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double s0 = R[i][lane], s1 = 0.0;
#pragma unroll
            for (int k = 0; k < i; ++k) {
                if (k & 1) s1 = fma(-Lm[i][k], z[k], s1);
                else s0 = fma(-Lm[i][k], z[k], s0);
            }
            z[i] = (s0 + s1) * Li[i];
        }
#pragma unroll
        for (int i = D - 1; i >= 0; --i) {
            double s0 = z[i], s1 = 0.0;
#pragma unroll
            for (int k = i + 1; k < D; ++k) {
                if (k & 1) s1 = fma(-Lm[k][i], z[k], s1);
                else s0 = fma(-Lm[k][i], z[k], s0);
            }
            z[i] = (s0 + s1) * Li[i];
        }
#pragma unroll
        for (int i = 0; i < D; ++i) X[i][lane] = z[i];
    }
    __syncwarp();
}

// X = S^-1 R for a symmetric positive-definite shared S (D x D) and shared R (D x D) by
// Gauss-Jordan elimination on [S | R] held in REGISTERS, one row per lane (lanes < D), the
// pivot row broadcast by warp shuffles: no shared-memory round trips or warp barriers inside
// the elimination, fully unrolled (compile-time register indices).  No pivoting: S is SPD
// (pivots are the Schur complements, positive).  Returns false on a non-positive pivot.
template <int D>
__device__ __forceinline__ bool wgj_solve(const double (*S)[LD(D)], const double (*R)[LD(D)], double (*X)[LD(D)],
                                          int lane) {
    static_assert(D <= 32, "one row per lane");
    const int r = lane < D ? lane : D - 1;
    double a[D], b[D];
#pragma unroll
    for (int j = 0; j < D; ++j) { a[j] = S[r][j]; b[j] = R[r][j]; }
    bool ok = true;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        const double piv = __shfl_sync(0xffffffffu, a[j], j);
        ok = ok && (piv > 0.0);
        const double ip = 1.0 / piv;
        const double f = (lane == j) ? 0.0 : a[j] * ip;       // multiplier of this lane's row
        // pivot row (entries right of the pivot, and the RHS), scaled row update
#pragma unroll
        for (int k = j + 1; k < D; ++k) {
            const double pk = __shfl_sync(0xffffffffu, a[k], j);
            a[k] = (lane == j) ? a[k] * ip : fma(-f, pk, a[k]);
        }
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const double pk = __shfl_sync(0xffffffffu, b[k], j);
            b[k] = (lane == j) ? b[k] * ip : fma(-f, pk, b[k]);
        }
    }
    if (lane < D) {
#pragma unroll
        for (int k = 0; k < D; ++k) X[lane][k] = b[k];
    }
    __syncwarp();
    return ok;
}

// out = A v (TA: A^T v)
template <int D, bool TA = false>
__device__ __forceinline__ void wmv(double* out, const double (*A)[LD(D)], const double* v, int lane) {
    for (int i = lane; i < D; i += 32) {
        double s = 0.0;
#pragma unroll 8
        for (int k = 0; k < D; ++k) s = fma(TA ? A[k][i] : A[i][k], v[k], s);
        out[i] = s;
    }
}

// warp sum of a per-lane partial
__device__ __forceinline__ double wsum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// dot(a, b) over D elements in shared memory, result in every lane
template <int D>
__device__ __forceinline__ double wdot(const double* a, const double* b, int lane) {
    double s = 0.0;
    for (int i = lane; i < D; i += 32) s = fma(a[i], b[i], s);
    return wsum(s);
}

// In-place inverse of a general D x D shared matrix by Gauss-Jordan with partial
// pivoting (W: D x 2D scratch, stride 2D+1).  Returns false on a zero pivot.
template <int D>
__device__ bool winverse(double (*M)[LD(D)], double (*W)[2 * D + 1], int lane) {
    for (int e = lane; e < D * 2 * D; e += 32) {
        const int i = e / (2 * D), j = e - (e / (2 * D)) * (2 * D);
        W[i][j] = (j < D) ? M[i][j] : ((j - D == i) ? 1.0 : 0.0);
    }
    __syncwarp();
    bool ok = true;
    for (int c = 0; c < D; ++c) {
        // pivot: argmax |W[r][c]|, r >= c
        double best = -1.0;
        int br = c;
        for (int r = c + lane; r < D; r += 32) {
            const double v = fabs(W[r][c]);
            if (v > best) { best = v; br = r; }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, off);
            const int orr = __shfl_xor_sync(0xffffffffu, br, off);
            if (ob > best || (ob == best && orr < br)) { best = ob; br = orr; }
        }
        ok = ok && (best > 0.0);
        if (br != c) {
            for (int j = lane; j < 2 * D; j += 32) {
                const double u = W[c][j];
                W[c][j] = W[br][j];
                W[br][j] = u;
            }
        }
        __syncwarp();
        const double ip = 1.0 / W[c][c];
        __syncwarp();
        for (int j = lane; j < 2 * D; j += 32) W[c][j] *= ip;
        __syncwarp();
        // eliminate column c from every other row (factors read before the row is updated)
        for (int e = lane; e < D * 2 * D; e += 32) {
            const int i = e / (2 * D), j = e - (e / (2 * D)) * (2 * D);
            if (i != c && j != c) W[i][j] = fma(-W[i][c], W[c][j], W[i][j]);
        }
        __syncwarp();
        for (int i = lane; i < D; i += 32)
            if (i != c) W[i][c] = 0.0;
        __syncwarp();
    }
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        M[i][j] = W[i][D + j];
    }
    __syncwarp();
    return ok;
}

// ------------------------------------------------------------------ shared aggregates
template <int D>
struct SF {   // filter aggregate in shared memory
    double A[D][LD(D)];
    double C[D][LD(D)];
    double J[D][LD(D)];
    double b[D];
    double eta[D];
};
template <int D>
struct SS {   // smoother aggregate
    double E[D][LD(D)];
    double L[D][LD(D)];
    double g[D];
};

// global (row-major, full) <-> shared
template <int D>
__device__ __forceinline__ void gload(SF<D>& a, const double* __restrict__ g, int lane) {
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        a.A[i][j] = g[e];
        a.C[i][j] = g[D * D + D + e];
        a.J[i][j] = g[2 * D * D + 2 * D + e];
    }
    for (int i = lane; i < D; i += 32) {
        a.b[i] = g[D * D + i];
        a.eta[i] = g[2 * D * D + D + i];
    }
    __syncwarp();
}
template <int D>
__device__ __forceinline__ void gstore(const SF<D>& a, double* __restrict__ g, int lane) {
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        g[e] = a.A[i][j];
        g[D * D + D + e] = a.C[i][j];
        g[2 * D * D + 2 * D + e] = a.J[i][j];
    }
    for (int i = lane; i < D; i += 32) {
        g[D * D + i] = a.b[i];
        g[2 * D * D + D + i] = a.eta[i];
    }
}
template <int D>
__device__ __forceinline__ void gload(SS<D>& a, const double* __restrict__ g, int lane) {
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        a.E[i][j] = g[e];
        a.L[i][j] = g[D * D + D + e];
    }
    for (int i = lane; i < D; i += 32) a.g[i] = g[D * D + i];
    __syncwarp();
}
template <int D>
__device__ __forceinline__ void gstore(const SS<D>& a, double* __restrict__ g, int lane) {
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        g[e] = a.E[i][j];
        g[D * D + D + e] = a.L[i][j];
    }
    for (int i = lane; i < D; i += 32) g[D * D + i] = a.g[i];
}
template <int D>
__device__ __forceinline__ void set_identity(SF<D>& a, int lane) {
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        a.A[i][j] = (i == j) ? 1.0 : 0.0;
        a.C[i][j] = 0.0;
        a.J[i][j] = 0.0;
    }
    for (int i = lane; i < D; i += 32) { a.b[i] = 0.0; a.eta[i] = 0.0; }
    __syncwarp();
}
template <int D>
__device__ __forceinline__ void set_identity(SS<D>& a, int lane) {
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        a.E[i][j] = (i == j) ? 1.0 : 0.0;
        a.L[i][j] = 0.0;
    }
    for (int i = lane; i < D; i += 32) a.g[i] = 0.0;
    __syncwarp();
}

// scratch for the general filtering operator
template <int D>
struct SCombF {
    double M[D][LD(D)];
    double T1[D][LD(D)];
    double T2[D][LD(D)];
    double W[D][2 * D + 1];
    double v1[D], v2[D];
};

// out = ei (x) ej, with Minv = (I + C_i J_j)^-1 and
// (I + J_j C_i)^-1 = Minv^T.  out may alias ej but not ei.
#ifndef PSSGP_WCOMBINE_GJ
#define PSSGP_WCOMBINE_GJ 1
#endif
// The filtering operator by one warp, solve form: X = (I + C_i J_j)^-1 [A_i | v1 |
// C_i] (v1 = b_i + C_i eta_j) by a register Gauss-Jordan elimination with partial pivoting, one row
// of the augmented system per lane and the pivot row broadcast by shuffles (no shared traffic, no
// explicit inverse); then A = A_j X_A, b = A_j X_v + b_j, C = A_j X_C A_j^T + C_j,
// eta = X_A^T (eta_j - J_j b_i) + eta_i, J = X_A^T J_j A_i + J_i (X_A^T = A_i^T (I + J_j C_i)^-1 by
// the symmetry of C and J) - five register-tiled products.  out may alias ej.
template <int D>
__device__ bool wcombine_gj(const SF<D>& ei, SF<D>& ej, SF<D>& out, SCombF<D>& s, int lane) {
    static_assert(D <= 32, "one row per lane");
    double (*Wm)[LD(D)] = reinterpret_cast<double (*)[LD(D)]>(&s.W[0][0]);   // D x LD fits in D x (2D + 1)
    wmm<D>(s.M, ei.C, ej.J, nullptr, lane);                                     // C_i J_j
    if (lane < D) {
        double a1 = ei.b[lane], a2 = ej.eta[lane];
#pragma unroll
        for (int k = 0; k < D; ++k) {
            a1 = fma(ei.C[lane][k], ej.eta[k], a1);
            a2 = fma(-ej.J[lane][k], ei.b[k], a2);
        }
        s.v1[lane] = a1;
        s.v2[lane] = a2;
    }
    __syncwarp();
    constexpr int NX = 2 * D + 1;
    const bool act = lane < D;
    const int r = act ? lane : D - 1;
    double a[D], x[NX];
#pragma unroll
    for (int j = 0; j < D; ++j) a[j] = s.M[r][j] + ((j == r) ? 1.0 : 0.0);
#pragma unroll
    for (int j = 0; j < D; ++j) {
        x[j] = ei.A[r][j];
        x[D + 1 + j] = ei.C[r][j];
    }
    x[D] = s.v1[r];
    bool ok = true;
    unsigned used = 0u;
    int myj = -1;                                   // the column this lane's row pivots
#pragma unroll
    for (int j = 0; j < D; ++j) {
        double v = (act && !((used >> lane) & 1u)) ? fabs(a[j]) : -1.0;
        int who = lane;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, v, off);
            const int ow = __shfl_xor_sync(0xffffffffu, who, off);
            if (ov > v || (ov == v && ow < who)) { v = ov; who = ow; }
        }
        ok = ok && (v > 0.0);
        used |= 1u << who;
        if (lane == who) myj = j;
        const double ip = 1.0 / __shfl_sync(0xffffffffu, a[j], who);
        const double f = (lane == who) ? 0.0 : a[j] * ip;
#pragma unroll
        for (int k = j + 1; k < D; ++k) {
            const double pk = __shfl_sync(0xffffffffu, a[k], who);
            a[k] = (lane == who) ? a[k] * ip : fma(-f, pk, a[k]);
        }
#pragma unroll
        for (int c = 0; c < NX; ++c) {
            const double pc = __shfl_sync(0xffffffffu, x[c], who);
            x[c] = (lane == who) ? x[c] * ip : fma(-f, pc, x[c]);
        }
    }
    __syncwarp();                                   // everyone is done reading s.v1 / s.M
    if (act) {                                      // solution row myj: X_A, X_v, X_C
#pragma unroll
        for (int j = 0; j < D; ++j) {
            s.T2[myj][j] = x[j];
            s.T1[myj][j] = x[D + 1 + j];
        }
        s.v1[myj] = x[D];
    }
    __syncwarp();
    wmm<D>(s.M, ej.A, s.T1, nullptr, lane);                                     // A_j X_C
    wmm<D>(Wm, ej.J, ei.A, nullptr, lane);                                      // J_j A_i
    double nb = 0.0, ne = 0.0;
    if (act) {
        nb = ej.b[lane];
        ne = ei.eta[lane];
#pragma unroll
        for (int k = 0; k < D; ++k) {
            nb = fma(ej.A[lane][k], s.v1[k], nb);
            ne = fma(s.T2[k][lane], s.v2[k], ne);
        }
    }
    __syncwarp();
    wmm<D, false, true>(s.T1, s.M, ej.A, ej.C, lane);                           // C = A_j X_C A_j^T + C_j
    __syncwarp();
    wmm<D>(s.M, ej.A, s.T2, nullptr, lane);                                     // A = A_j X_A
    __syncwarp();                                   // A_j, J_j, C_j are read for the last time above
    wmm<D, true, false>(out.A, s.T2, Wm, ei.J, lane);                           // X_A^T J_j A_i + J_i (in out.A)
    __syncwarp();
    for (int e0 = 0; e0 < D * D; e0 += 32) {        // J, C symmetrised (the same trip count in every lane)
        const int e = e0 + lane;
        if (e < D * D) {
            const int i = e / D, j = e - (e / D) * D;
            out.J[i][j] = 0.5 * (out.A[i][j] + out.A[j][i]);
            out.C[i][j] = 0.5 * (s.T1[i][j] + s.T1[j][i]);
        }
    }
    __syncwarp();
    for (int e0 = 0; e0 < D * D; e0 += 32) {
        const int e = e0 + lane;
        if (e < D * D) out.A[e / D][e % D] = s.M[e / D][e % D];
    }
    if (act) {
        out.b[lane] = nb;
        out.eta[lane] = ne;
    }
    __syncwarp();
    return ok;
}

template <int D>
__device__ bool wcombine(const SF<D>& ei, SF<D>& ej, SF<D>& out, SCombF<D>& s, int lane) {
    if constexpr (PSSGP_WCOMBINE_GJ && D <= 32) return wcombine_gj<D>(ei, ej, out, s, lane);
    // M = I + C_i J_j
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        double acc = (i == j) ? 1.0 : 0.0;
        for (int k = 0; k < D; ++k) acc = fma(ei.C[i][k], ej.J[k][j], acc);
        s.M[i][j] = acc;
    }
    __syncwarp();
    const bool ok = winverse<D>(s.M, s.W, lane);
    // v1 = b_i + C_i eta_j ; v2 = eta_j - J_j b_i
    for (int i = lane; i < D; i += 32) {
        double a1 = ei.b[i], a2 = ej.eta[i];
        for (int k = 0; k < D; ++k) {
            a1 = fma(ei.C[i][k], ej.eta[k], a1);
            a2 = fma(-ej.J[i][k], ei.b[k], a2);
        }
        s.v1[i] = a1;
        s.v2[i] = a2;
    }
    __syncwarp();
    // T1 = A_j Minv
    wmm<D>(s.T1, ej.A, s.M, nullptr, lane);
    __syncwarp();
    // b_out = T1 v1 + b_j ; eta_out = A_i^T Minv^T v2 + eta_i  (= (Minv A_i)^T v2)
    // T2 = Minv A_i (needed for J and eta)
    wmm<D>(s.T2, s.M, ei.A, nullptr, lane);
    __syncwarp();
    double nb[(D + 31) / 32], ne[(D + 31) / 32];
    for (int i = lane, q = 0; i < D; i += 32, ++q) {
        double a1 = ej.b[i], a2 = ei.eta[i];
        for (int k = 0; k < D; ++k) {
            a1 = fma(s.T1[i][k], s.v1[k], a1);
            a2 = fma(s.T2[k][i], s.v2[k], a2);
        }
        nb[q] = a1;
        ne[q] = a2;
    }
    __syncwarp();
    // J_out = A_i^T Minv^T J_j A_i + J_i = T2^T J_j A_i + J_i  -> M (free) = J_j A_i first
    wmm<D>(s.M, ej.J, ei.A, nullptr, lane);
    __syncwarp();
    double* ojv = &out.J[0][0];
    (void)ojv;
    // compute new J into W (as D x D block) to allow out aliasing ej
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        double acc = ei.J[i][j];
        for (int k = 0; k < D; ++k) acc = fma(s.T2[k][i], s.M[k][j], acc);
        s.W[i][j] = acc;
    }
    __syncwarp();
    // A_out = T1 A_i ; C_out = T1 C_i A_j^T + C_j   (M := T1 C_i)
    wmm<D>(s.M, s.T1, ei.C, nullptr, lane);
    __syncwarp();
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        double aa = 0.0, cc = ej.C[i][j];
        for (int k = 0; k < D; ++k) {
            aa = fma(s.T1[i][k], ei.A[k][j], aa);
            cc = fma(s.M[i][k], ej.A[j][k], cc);
        }
        s.T2[i][j] = aa;     // T2 no longer needed
        s.W[i][D + j] = cc;
    }
    __syncwarp();
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        out.A[i][j] = s.T2[i][j];
        out.J[i][j] = 0.5 * (s.W[i][j] + s.W[j][i]);
        out.C[i][j] = 0.5 * (s.W[i][D + j] + s.W[j][D + i]);
    }
    for (int i = lane, q = 0; i < D; i += 32, ++q) {
        out.b[i] = nb[q];
        out.eta[i] = ne[q];
    }
    __syncwarp();
    return ok;
}

// out = ei (x)_s ej = (E_i E_j, E_i g_j + g_i, E_i L_j E_i^T + L_i); out may alias ej.
template <int D>
__device__ void wcombine(const SS<D>& ei, SS<D>& ej, SS<D>& out, SCombF<D>& s, int lane) {
    wmm<D>(s.T1, ei.E, ej.L, nullptr, lane);        // E_i L_j
    wmm<D>(s.T2, ei.E, ej.E, nullptr, lane);        // E_i E_j
    for (int i = lane; i < D; i += 32) {
        double a = ei.g[i];
        for (int k = 0; k < D; ++k) a = fma(ei.E[i][k], ej.g[k], a);
        s.v1[i] = a;
    }
    __syncwarp();
    wmm<D, false, true>(s.M, s.T1, ei.E, ei.L, lane);   // E_i L_j E_i^T + L_i
    __syncwarp();
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        out.E[i][j] = s.T2[i][j];
        out.L[i][j] = 0.5 * (s.M[i][j] + s.M[j][i]);
    }
    for (int i = lane; i < D; i += 32) out.g[i] = s.v1[i];
    __syncwarp();
}

// collapsed prefix (0, x, P, 0, 0) (x) a  ->  (x', P') written into (x, P)
template <int D>
__device__ bool wapply_prefix(double* x, double (*P)[LD(D)], const SF<D>& a, SCombF<D>& s, int lane) {
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        double acc = (i == j) ? 1.0 : 0.0;
        for (int k = 0; k < D; ++k) acc = fma(P[i][k], a.J[k][j], acc);
        s.M[i][j] = acc;
    }
    __syncwarp();
    const bool ok = winverse<D>(s.M, s.W, lane);
    for (int i = lane; i < D; i += 32) {
        double acc = x[i];
        for (int k = 0; k < D; ++k) acc = fma(P[i][k], a.eta[k], acc);
        s.v1[i] = acc;
    }
    __syncwarp();
    wmm<D>(s.T1, a.A, s.M, nullptr, lane);          // A Minv
    __syncwarp();
    wmm<D>(s.T2, s.T1, P, nullptr, lane);           // A Minv P
    __syncwarp();
    for (int i = lane; i < D; i += 32) {
        double acc = a.b[i];
        for (int k = 0; k < D; ++k) acc = fma(s.T1[i][k], s.v1[k], acc);
        s.v2[i] = acc;
    }
    wmm<D, false, true>(s.M, s.T2, a.A, a.C, lane);      // A Minv P A^T + C
    __syncwarp();
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        P[i][j] = 0.5 * (s.M[i][j] + s.M[j][i]);
    }
    for (int i = lane; i < D; i += 32) x[i] = s.v2[i];
    __syncwarp();
    return ok;
}

// (x, P) <- (x, P) (x) a in solve form with caller scratch (three D x LD matrices, two D vectors):
// [X_P | X_x] = (I + P J)^-1 [P | x + P eta] by the register Gauss-Jordan of wcombine_gj, then
// P = A X_P A^T + C (symmetrised), x = A X_x + b.
template <int D>
__device__ bool wapply_prefix_gj(double* x, double (*P)[LD(D)], const SF<D>& a, double (*Mb)[LD(D)],
                                 double (*Xb)[LD(D)], double (*Tb)[LD(D)], double* v1, double* v2, int lane) {
    static_assert(D <= 32, "one row per lane");
    wmm<D>(Mb, P, a.J, nullptr, lane);                                          // P J
    if (lane < D) {
        double acc = x[lane];
#pragma unroll
        for (int k = 0; k < D; ++k) acc = fma(P[lane][k], a.eta[k], acc);
        v1[lane] = acc;
    }
    __syncwarp();
    constexpr int NX = D + 1;
    const bool act = lane < D;
    const int r = act ? lane : D - 1;
    double am[D], xr[NX];
#pragma unroll
    for (int j = 0; j < D; ++j) {
        am[j] = Mb[r][j] + ((j == r) ? 1.0 : 0.0);
        xr[j] = P[r][j];
    }
    xr[D] = v1[r];
    bool ok = true;
    unsigned used = 0u;
    int myj = -1;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        double v = (act && !((used >> lane) & 1u)) ? fabs(am[j]) : -1.0;
        int who = lane;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, v, off);
            const int ow = __shfl_xor_sync(0xffffffffu, who, off);
            if (ov > v || (ov == v && ow < who)) { v = ov; who = ow; }
        }
        ok = ok && (v > 0.0);
        used |= 1u << who;
        if (lane == who) myj = j;
        const double ip = 1.0 / __shfl_sync(0xffffffffu, am[j], who);
        const double f = (lane == who) ? 0.0 : am[j] * ip;
#pragma unroll
        for (int k = j + 1; k < D; ++k) {
            const double pk = __shfl_sync(0xffffffffu, am[k], who);
            am[k] = (lane == who) ? am[k] * ip : fma(-f, pk, am[k]);
        }
#pragma unroll
        for (int c = 0; c < NX; ++c) {
            const double pc = __shfl_sync(0xffffffffu, xr[c], who);
            xr[c] = (lane == who) ? xr[c] * ip : fma(-f, pc, xr[c]);
        }
    }
    __syncwarp();
    if (act) {
#pragma unroll
        for (int j = 0; j < D; ++j) Xb[myj][j] = xr[j];
        v2[myj] = xr[D];
    }
    __syncwarp();
    wmm<D>(Tb, a.A, Xb, nullptr, lane);                                         // A X_P
    double xn = 0.0;
    if (act) {
        xn = a.b[lane];
#pragma unroll
        for (int k = 0; k < D; ++k) xn = fma(a.A[lane][k], v2[k], xn);
    }
    __syncwarp();
    wmm<D, false, true>(Mb, Tb, a.A, a.C, lane);                                // A X_P A^T + C
    __syncwarp();
    for (int e0 = 0; e0 < D * D; e0 += 32) {
        const int e = e0 + lane;
        if (e < D * D) {
            const int i = e / D, j = e - (e / D) * D;
            P[i][j] = 0.5 * (Mb[i][j] + Mb[j][i]);
        }
    }
    if (act) x[lane] = xn;
    __syncwarp();
    return ok;
}

// E = S A^-1 for a symmetric A by one warp: rows of [A | S^T] per lane, the register Gauss-Jordan of
// wcombine_gj (partial pivoting); E must alias neither S nor A.
template <int D>
__device__ bool wright_div_sym_gj(double (*E)[LD(D)], const double (*S)[LD(D)], const double (*A)[LD(D)],
                                  int lane) {
    static_assert(D <= 32, "one row per lane");
    const bool act = lane < D;
    const int r = act ? lane : D - 1;
    double am[D], xr[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
        am[j] = A[r][j];
        xr[j] = S[j][r];
    }
    bool ok = true;
    unsigned used = 0u;
    int myj = -1;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        double v = (act && !((used >> lane) & 1u)) ? fabs(am[j]) : -1.0;
        int who = lane;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, v, off);
            const int ow = __shfl_xor_sync(0xffffffffu, who, off);
            if (ov > v || (ov == v && ow < who)) { v = ov; who = ow; }
        }
        ok = ok && (v > 0.0);
        used |= 1u << who;
        if (lane == who) myj = j;
        const double ip = 1.0 / __shfl_sync(0xffffffffu, am[j], who);
        const double f = (lane == who) ? 0.0 : am[j] * ip;
#pragma unroll
        for (int k = j + 1; k < D; ++k) {
            const double pk = __shfl_sync(0xffffffffu, am[k], who);
            am[k] = (lane == who) ? am[k] * ip : fma(-f, pk, am[k]);
        }
#pragma unroll
        for (int c = 0; c < D; ++c) {
            const double pc = __shfl_sync(0xffffffffu, xr[c], who);
            xr[c] = (lane == who) ? xr[c] * ip : fma(-f, pc, xr[c]);
        }
    }
    __syncwarp();
    if (act) {
#pragma unroll
        for (int i = 0; i < D; ++i) E[i][myj] = xr[i];
    }
    __syncwarp();
    return ok;
}

// scratch of the suffix application (no inverse needed)
template <int D>
struct SSufScratch {
    double M[D][LD(D)];
    double T1[D][LD(D)];
    double v1[D];
};

// a (x)_s collapsed suffix (0, m, P) -> (E m + g, E P E^T + L) written into (m, P)
template <int D, typename Scratch>
__device__ void wapply_suffix(const SS<D>& a, double* m, double (*P)[LD(D)], Scratch& s, int lane) {
    wmm<D>(s.T1, a.E, P, nullptr, lane);
    for (int i = lane; i < D; i += 32) {
        double acc = a.g[i];
        for (int k = 0; k < D; ++k) acc = fma(a.E[i][k], m[k], acc);
        s.v1[i] = acc;
    }
    __syncwarp();
    wmm<D, false, true>(s.M, s.T1, a.E, a.L, lane);     // E P E^T + L
    __syncwarp();
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        P[i][j] = 0.5 * (s.M[i][j] + s.M[j][i]);
    }
    for (int i = lane; i < D; i += 32) m[i] = s.v1[i];
    __syncwarp();
}

// ------------------------------------------------------------------ discretisation (table)
// returns 0 (F, Q valid in fz / via model), 1 = dt == 0 (identity), 2 = unsupported
__device__ __forceinline__ int wdisc_kind(double dt, double udt, bool stream = false) {
    if (stream) return dt == 0.0 ? 1 : 0;           // per-step (F, Q) from kw_discretize
    if (fabs(dt - udt) <= 1e-12 * udt) return 0;   // uniform step up to time-stamp rounding
    if (dt == 0.0) return 1;
    return 2;
}

// (F, Q) used for local step k: the model's table, or the per-step pair of kw_discretize
template <int D>
struct FQp {
    const double (*F)[LD(D)];
    const double (*Q)[LD(D)];
};
template <int D>
__device__ __forceinline__ FQp<D> wfq(const WParams& p, const SModel<D>& M, int64_t k) {
    if (p.fq) {
        const double (*b)[LD(D)] = reinterpret_cast<const double (*)[LD(D)]>(p.fq + k * FQW(D));
        return {b, b + D};
    }
    return {M.F, M.Q};
}

// ------------------------------------------------------------------ KDw: per-step discretisation
// One warp per step (grid-stride).  On the scaled step tau = dt / 2^s with ||G tau||_1 <= 1/8:
// F_tau by a truncated Taylor polynomial in Paterson-Stockmeyer form (no pivoted solve: a warp
// elimination costs D serial rounds; degree 6 for ||G dt|| <= 0.017, else 12) and
// Q_tau = sum_{k=1..m} Z_k, Z_1 = tau W, Z_{k+1} = (A Z_k + Z_k A^T)/(k+1) (Taylor series of the
// Lyapunov ODE, cancellation-free; m = 7 / 12), then s doublings Q <- Q + F Q F^T, F <- F^2.
// (The stationary shortcut P_inf - F P_inf F^T loses the small entries of Q on fine grids,
// SURVEY A.4.)  Writes fq[k] for local steps k in [0, nfq) with a predecessor and dt != 0.
template <int D>
struct KDSmem {
    double G[D][LD(D)];
    double Pinf[D][LD(D)];
    double Wd[D][LD(D)];
    double gnorm;
    struct PerWarp {
        double A[D][LD(D)], A2[D][LD(D)], A3[D][LD(D)], X[D][LD(D)], T[D][LD(D)], B[D][LD(D)];
    } w[kWWarps];
};

template <int D>
__device__ __forceinline__ void taylor_block(double (*B)[LD(D)], const double (*A)[LD(D)], const double (*A2)[LD(D)],
                                             const double (*A3)[LD(D)], double c0, double c1, double c2, double c3,
                                             int lane) {
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        double v = fma(c2, A2[i][j], c1 * A[i][j]);
        if (A3) v = fma(c3, A3[i][j], v);
        B[i][j] = v + ((i == j) ? c0 : 0.0);
    }
}

template <int D>
__global__ void __launch_bounds__(32 * kWWarps) kw_discretize(const double* __restrict__ t, int64_t nfq, int64_t k0,
                                                               const double* __restrict__ model, double* fq,
                                                               unsigned long long* err) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    KDSmem<D>& sh = *reinterpret_cast<KDSmem<D>*>(smem_raw);
    for (int e = threadIdx.x; e < D * D; e += blockDim.x) {
        const int i = e / D, j = e - (e / D) * D;
        sh.G[i][j] = model[3 * D * D + D + 2 + e];
        sh.Pinf[i][j] = model[2 * D * D + e];
        sh.Wd[i][j] = model[4 * D * D + D + 2 + e];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double nrm = 0.0;
        for (int j = 0; j < D; ++j) {
            double c = 0.0;
            for (int i = 0; i < D; ++i) c += fabs(sh.G[i][j]);
            nrm = fmax(nrm, c);
        }
        sh.gnorm = nrm;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    auto& W = sh.w[wid];
    // 1 / j!
    constexpr double c[13] = {1.0, 1.0, 1.0 / 2, 1.0 / 6, 1.0 / 24, 1.0 / 120, 1.0 / 720, 1.0 / 5040, 1.0 / 40320,
                              1.0 / 362880, 1.0 / 3628800, 1.0 / 39916800, 1.0 / 479001600};
    const int64_t nw = static_cast<int64_t>(gridDim.x) * kWWarps;
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * kWWarps + wid; k < nfq; k += nw) {
        if (k0 + k == 0) continue;
        const double dt = __ldg(t + k) - __ldg(t + k - 1);
        if (dt == 0.0 || !(dt == dt)) continue;
        const double nrm = sh.gnorm * fabs(dt);
        if (nrm <= kPolyNorm) {   // small step: Taylor polynomials in dt (as kw_discretize_lpr)
            double* o = fq + k * FQW(D);
            const double* fc = model + MODW(D);
            const double* qc = fc + (kPolyM + 1) * D * D;
            for (int e = lane; e < D * D; e += 32) {
                const int i = e / D, j = e - (e / D) * D;
                double f = __ldg(fc + kPolyM * D * D + e), q = __ldg(qc + kPolyM * D * D + e);
#pragma unroll
                for (int kk = kPolyM - 1; kk >= 0; --kk) {
                    f = fma(f, dt, __ldg(fc + kk * D * D + e));
                    q = fma(q, dt, __ldg(qc + kk * D * D + e));
                }
                o[i * LD(D) + j] = f;
                o[(D + i) * LD(D) + j] = q * dt;
            }
            continue;
        }
        int s = 0;
        if (nrm > 0.125) frexp(nrm / 0.125, &s);
        const bool low = (nrm <= 0.017);
        const double tau = ldexp(dt, -s);
        for (int e = lane; e < D * D; e += 32) W.A[e / D][e % D] = sh.G[e / D][e % D] * tau;
        __syncwarp();
        wmm<D>(W.A2, W.A, W.A, nullptr, lane);
        __syncwarp();
        wmm<D>(W.A3, W.A2, W.A, nullptr, lane);
        __syncwarp();
        if (low) {   // m = 6: F = B0 + A3 (c3 I + c4 A + c5 A2 + c6 A3)
            taylor_block<D>(W.X, W.A, W.A2, W.A3, c[3], c[4], c[5], c[6], lane);
            taylor_block<D>(W.B, W.A, W.A2, nullptr, c[0], c[1], c[2], 0.0, lane);
            __syncwarp();
            wmm<D>(W.T, W.A3, W.X, W.B, lane);
        } else {     // m = 12: Horner in A3 over degree-2 blocks, top block degree 3
            taylor_block<D>(W.X, W.A, W.A2, W.A3, c[9], c[10], c[11], c[12], lane);
            taylor_block<D>(W.B, W.A, W.A2, nullptr, c[6], c[7], c[8], 0.0, lane);
            __syncwarp();
            wmm<D>(W.T, W.A3, W.X, W.B, lane);
            __syncwarp();
            taylor_block<D>(W.B, W.A, W.A2, nullptr, c[3], c[4], c[5], 0.0, lane);
            __syncwarp();
            wmm<D>(W.X, W.A3, W.T, W.B, lane);
            __syncwarp();
            taylor_block<D>(W.B, W.A, W.A2, nullptr, c[0], c[1], c[2], 0.0, lane);
            __syncwarp();
            wmm<D>(W.T, W.A3, W.X, W.B, lane);
        }
        __syncwarp();
        double (*F)[LD(D)] = W.T;
        // Q_tau: Z = tau W (in A2), Q (in X) accumulates, Y = A Z (in A3)
        double (*Z)[LD(D)] = W.A2;
        double (*Qc)[LD(D)] = W.X;
        for (int e = lane; e < D * D; e += 32) {
            const int i = e / D, j = e - (e / D) * D;
            Z[i][j] = sh.Wd[i][j] * tau;
            Qc[i][j] = Z[i][j];
        }
        __syncwarp();
        const int mq = low ? 7 : 12;
        for (int kk = 1; kk < mq; ++kk) {
            wmm<D>(W.A3, W.A, Z, nullptr, lane);
            __syncwarp();
            const double ik = 1.0 / (kk + 1);
            for (int e = lane; e < D * D; e += 32) {
                const int i = e / D, j = e - (e / D) * D;
                const double zz = (W.A3[i][j] + W.A3[j][i]) * ik;
                Z[i][j] = zz;
                Qc[i][j] += zz;
            }
            __syncwarp();
        }
        // doublings: Q <- Q + F Q F^T, F <- F F   (buffers: B = F Q, A2 / X ping-pong for Q, A3 for F^2)
        double (*Qn)[LD(D)] = W.A2;
        double (*Fn)[LD(D)] = W.A3;
        for (int q = 0; q < s; ++q) {
            wmm<D>(W.B, F, Qc, nullptr, lane);
            __syncwarp();
            wmm<D, false, true>(Qn, W.B, F, Qc, lane);
            wmm<D>(Fn, F, F, nullptr, lane);
            __syncwarp();
            double (*t1)[LD(D)] = Qc; Qc = Qn; Qn = t1;
            double (*t2)[LD(D)] = F; F = Fn; Fn = t2;
        }
        double* o = fq + k * FQW(D);
        for (int e = lane; e < D * D; e += 32) {
            const int i = e / D, j = e - (e / D) * D;
            o[i * LD(D) + j] = F[i][j];
            o[(D + i) * LD(D) + j] = 0.5 * (Qc[i][j] + Qc[j][i]);
        }
        __syncwarp();
    }
    (void)err;
}

// Per-step (F, Q) of a model whose G and W are block diagonal with B x B blocks (pssgp_model::fblock:
// sums of components, periodic harmonics as 2 x 2 rotations, quasi-periodic products in blocks of 2m):
// expm and the Lyapunov integral act block by block, so one LANE per (step, block) runs
// kw_discretize's algorithm on its B x B block in registers — the Taylor series of degree 12 of
// F_tau = e^{G tau} and of Q_tau = sum_k Z_k (Z_1 = tau W, Z_{k+1} = sym(G tau Z_k) 2 / (k + 1)) at
// tau = dt / 2^s with ||G_b tau||_1 <= 1/8 for the block's own norm, then s doublings
// Q <- F Q F^T + Q, F <- F F.  A warp takes SPW <= 32 / NB consecutive steps at a time, assembles
// their records (zeros off the blocks) in shared memory and writes them out as one contiguous,
// coalesced run.  O(B^3) per block instead of O(D^3) warp products per step.
constexpr int kBlkWarps = 2;
template <int D, int B>
struct BlkDisc {
    static constexpr int NB = (D + B - 1) / B;   // the last block may be partial (d = 14 in blocks of 4)
    // steps per warp: one lane per block, staged records within 40 KB of static shared memory per CTA
    static constexpr int SPW0 = 32 / NB, SPWM = 40960 / (kBlkWarps * FQW(D) * 8);
    static constexpr int SPW = SPW0 < SPWM ? SPW0 : SPWM;
};
template <int D, int B>
__global__ void __launch_bounds__(32 * kBlkWarps) kw_discretize_blk(const double* __restrict__ t, int64_t nfq,
                                                                    int64_t k0, const double* __restrict__ model,
                                                                    double* fq) {
    constexpr int NB = BlkDisc<D, B>::NB, SPW = BlkDisc<D, B>::SPW;
    static_assert(NB <= 32, "one lane per block");
    __shared__ double rec[kBlkWarps][SPW * FQW(D)];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double* sr = rec[wid];
    const int js = lane / NB, bb = lane - js * NB, o0 = bb * B, bs = min(B, D - o0);
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kBlkWarps;
    for (int64_t kw = (static_cast<int64_t>(blockIdx.x) * kBlkWarps + wid) * SPW; kw < nfq; kw += nwarps * SPW) {
        const int nst = static_cast<int>(min(static_cast<int64_t>(SPW), nfq - kw));
        for (int e = lane; e < SPW * FQW(D); e += 32) sr[e] = 0.0;
        __syncwarp();
        const int64_t k = kw + js;
        bool act = js < nst && k0 + k != 0;
        const double dt = act ? __ldg(t + k) - __ldg(t + k - 1) : 0.0;
        act = act && dt != 0.0 && dt == dt;
        if (act) {
            double G[B][B], Wm[B][B];
            double nrm = 0.0;
#pragma unroll
            for (int j = 0; j < B; ++j) {
                double c = 0.0;
#pragma unroll
                for (int i = 0; i < B; ++i) {
                    const bool in = i < bs && j < bs;   // padding of a partial block: G = W = 0
                    G[i][j] = in ? __ldg(model + 3 * D * D + D + 2 + (o0 + i) * D + o0 + j) : 0.0;
                    Wm[i][j] = in ? __ldg(model + 4 * D * D + D + 2 + (o0 + i) * D + o0 + j) : 0.0;
                    c += fabs(G[i][j]);
                }
                nrm = fmax(nrm, c);
            }
            nrm *= fabs(dt);
            int s = 0;
            if (nrm > 0.125) frexp(nrm / 0.125, &s);
            const double tau = ldexp(dt, -s);
            double A[B][B], F[B][B], Z[B][B], Q[B][B];
#pragma unroll
            for (int i = 0; i < B; ++i)
#pragma unroll
                for (int j = 0; j < B; ++j) {
                    A[i][j] = G[i][j] * tau;
                    F[i][j] = (i == j) ? 1.0 : 0.0;
                    Z[i][j] = Wm[i][j] * tau;
                    Q[i][j] = Z[i][j];
                }
            // F_tau by Horner: F = I + A/m (I + A/(m-1) (...)), m = 12
#pragma unroll
            for (int kk = 12; kk >= 1; --kk) {
                double T[B][B];
                const double ik = 1.0 / kk;
#pragma unroll
                for (int i = 0; i < B; ++i)
#pragma unroll
                    for (int j = 0; j < B; ++j) {
                        double a = 0.0;
#pragma unroll
                        for (int l = 0; l < B; ++l) a = fma(A[i][l], F[l][j], a);
                        T[i][j] = fma(a, ik, (i == j) ? 1.0 : 0.0);
                    }
#pragma unroll
                for (int i = 0; i < B; ++i)
#pragma unroll
                    for (int j = 0; j < B; ++j) F[i][j] = T[i][j];
            }
            // Q_tau = sum_{k=1}^{12} Z_k
#pragma unroll
            for (int kk = 1; kk < 12; ++kk) {
                double Y[B][B];
#pragma unroll
                for (int i = 0; i < B; ++i)
#pragma unroll
                    for (int j = 0; j < B; ++j) {
                        double a = 0.0;
#pragma unroll
                        for (int l = 0; l < B; ++l) a = fma(A[i][l], Z[l][j], a);
                        Y[i][j] = a;
                    }
                const double ik = 1.0 / (kk + 1);
#pragma unroll
                for (int i = 0; i < B; ++i)
#pragma unroll
                    for (int j = 0; j < B; ++j) {
                        Z[i][j] = (Y[i][j] + Y[j][i]) * ik;
                        Q[i][j] += Z[i][j];
                    }
            }
            for (int q = 0; q < s; ++q) {   // doublings
                double FQ[B][B], Fn[B][B];
#pragma unroll
                for (int i = 0; i < B; ++i)
#pragma unroll
                    for (int j = 0; j < B; ++j) {
                        double a = 0.0, f = 0.0;
#pragma unroll
                        for (int l = 0; l < B; ++l) {
                            a = fma(F[i][l], Q[l][j], a);
                            f = fma(F[i][l], F[l][j], f);
                        }
                        FQ[i][j] = a;
                        Fn[i][j] = f;
                    }
#pragma unroll
                for (int i = 0; i < B; ++i)
#pragma unroll
                    for (int j = 0; j < B; ++j) {
                        double a = Q[i][j];
#pragma unroll
                        for (int l = 0; l < B; ++l) a = fma(FQ[i][l], F[j][l], a);
                        Z[i][j] = a;
                    }
#pragma unroll
                for (int i = 0; i < B; ++i)
#pragma unroll
                    for (int j = 0; j < B; ++j) {
                        Q[i][j] = Z[i][j];
                        F[i][j] = Fn[i][j];
                    }
            }
            double* o = sr + js * FQW(D);
#pragma unroll
            for (int i = 0; i < B; ++i)
#pragma unroll
                for (int jb = 0; jb < B; ++jb)
                    if (i < bs && jb < bs) {
                        o[(o0 + i) * LD(D) + o0 + jb] = F[i][jb];
                        o[(D + o0 + i) * LD(D) + o0 + jb] = 0.5 * (Q[i][jb] + Q[jb][i]);
                    }
        }
        __syncwarp();
        double* g = fq + kw * FQW(D);
        for (int e = lane; e < nst * FQW(D); e += 32) g[e] = sr[e];
        __syncwarp();
    }
}

// ------------------------------------------------------------------ K1w: fold
template <int D>
struct K1Smem {
    SModel<D> m;
    struct PerWarp {
        SF<D> a;
        double FA[D][LD(D)];
        double T[D][LD(D)];
        double Cm[D][LD(D)];
        double Fb[D], HC[D], w[D];
    } w[kWWarps];
};

template <int D>
__global__ void __launch_bounds__(32 * kWWarps, PSSGP_WMINB) kw_filter_fold(const WParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K1Smem<D>& sh = *reinterpret_cast<K1Smem<D>*>(smem_raw);
    load_model<D>(sh.m, p.model);
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = blockIdx.x * kWWarps + wid;
    if (c >= p.nch) return;
    auto& W = sh.w[wid];
    set_identity<D>(W.a, lane);
    const int64_t kb = static_cast<int64_t>(c) * p.K;
    const int64_t ke = min(kb + p.K, p.n);
    const SModel<D>& M = sh.m;
    double tprev = (kb < p.n && (kb > 0 || p.k0 > 0)) ? __ldg(p.t + kb - 1) : 0.0;
    // (t, mask, y) of the next step prefetched one step ahead (global latency off the step)
    double tn_ = 0.0, yn_ = 0.0;
    unsigned char mn_ = 0;
    if (kb < ke) { tn_ = __ldg(p.t + kb); mn_ = __ldg(p.mask + kb); yn_ = __ldg(p.y + kb); }
    for (int64_t k = kb; k < ke; ++k) {
        const double tk = tn_;
        const bool obs = mn_ != 0;
        const double yk = obs ? yn_ : 0.0;
        if (k + 1 < ke) { tn_ = __ldg(p.t + k + 1); mn_ = __ldg(p.mask + k + 1); yn_ = __ldg(p.y + k + 1); }
        const int64_t g = p.k0 + k;
        int kind = 0;
        if (g == 0) kind = 3;                                   // F = 0, Q = P_inf
        else kind = wdisc_kind(tk - tprev, M.udt, p.fq != nullptr);
        const FQp<D> fqp = wfq<D>(p, M, k);
        if (lane == 0) {
            if (g > 0 && !(tk - tprev >= 0.0)) raise_error(p.err, g, kErrInput);
            if (!isfinite(tk) || (obs && !isfinite(yk))) raise_error(p.err, g, kErrInput);
            if (kind == 2) raise_error(p.err, g, kErrUnsupported);
        }
        tprev = tk;
        // FA = F A, T = F C, Fb = F b, Cm = T F^T + Q   (kind 1: F = I, Q = 0; kind 3: F = 0, Q = P_inf)
        if (kind == 0) {
            wmm<D>(W.FA, fqp.F, W.a.A, nullptr, lane);
            wmm<D>(W.T, fqp.F, W.a.C, nullptr, lane);
            for (int i = lane; i < D; i += 32) {
                double s = 0.0;
                for (int q = 0; q < D; ++q) s = fma(fqp.F[i][q], W.a.b[q], s);
                W.Fb[i] = s;
            }
            __syncwarp();
            wmm<D, false, true>(W.Cm, W.T, fqp.F, fqp.Q, lane);
        } else {
            for (int e = lane; e < D * D; e += 32) {
                const int i = e / D, j = e - (e / D) * D;
                W.FA[i][j] = (kind == 1) ? W.a.A[i][j] : 0.0;
                W.Cm[i][j] = (kind == 1) ? W.a.C[i][j] : M.Pinf[i][j];
            }
            for (int i = lane; i < D; i += 32) W.Fb[i] = (kind == 1) ? W.a.b[i] : 0.0;
        }
        __syncwarp();
        // HC = Cm H^T ; w = (H FA)^T
        for (int i = lane; i < D; i += 32) {
            double hc = 0.0, ww = 0.0;
            for (int q = 0; q < D; ++q) {
                hc = fma(W.Cm[i][q], M.H[q], hc);
                ww = fma(M.H[q], W.FA[q][i], ww);
            }
            W.HC[i] = hc;
            W.w[i] = ww;
        }
        __syncwarp();
        const double S = wdot<D>(M.H, W.HC, lane) + M.r;
        const double hb = wdot<D>(M.H, W.Fb, lane);
        const double iS = obs ? 1.0 / S : 0.0;
        const double vs = obs ? (yk - hb) * iS : 0.0;
        for (int e = lane; e < D * D; e += 32) {
            const int i = e / D, j = e - (e / D) * D;
            const double Ki = W.HC[i] * iS;
            W.a.A[i][j] = fma(-Ki, W.w[j], W.FA[i][j]);
            W.a.C[i][j] = fma(-Ki, W.HC[j], W.Cm[i][j]);
            W.a.J[i][j] = fma(W.w[i] * iS, W.w[j], W.a.J[i][j]);
        }
        for (int i = lane; i < D; i += 32) {
            W.a.b[i] = fma(W.HC[i], vs, W.Fb[i]);
            W.a.eta[i] = fma(W.w[i], vs, W.a.eta[i]);
        }
        __syncwarp();
    }
    gstore<D>(W.a, p.fagg + static_cast<int64_t>(c) * FNW(D), lane);
}

// ------------------------------------------------------------------ K1w for D <= 8: lane-per-row fold
// Same grid and output as kw_filter_fold (one warp per chain, fagg[c]), but the chain is split
// into kQ = 4 consecutive quarters, each folded IN REGISTERS by one 8-lane group: lane r of a
// group holds column r of A, rows r of C and J (symmetric) and b_r, eta_r.  F and Q are read
// from shared memory (one address per group: broadcast); the full vectors a step needs (b, HC,
// w) are gathered by shuffles and F C is transposed through a per-group shared buffer.  The
// four quarter aggregates are then combined in order with the warp operator (
// any grouping).  Steps past a quarter's end are identity steps (F = I, Q = 0, y
// missing), which leave the aggregate unchanged exactly, so all lanes run the same trip count
// (full-warp shuffles).  Replaces one warp-cooperative shared-memory step per chain (36-64
// outputs over 32 lanes, ~4,400 cycles at d = 6) by four register steps in parallel.
constexpr int kQ = 4, kGL = 8;
// staging slot of one step's (F_k, Q_k) record: only the per-step (STREAM) kernels reserve it
PS_CX int FQS(int D, bool stream) { return stream ? FQW(D) : 1; }
template <int D, bool STREAM, int G = kGL, int WPC = kWWarps>
struct K1LSmem {
    static constexpr int NP = 32 / G;
    SModel<D> m;
    double I[D][LD(D)], Z[D][LD(D)];
    struct PerWarp {
        // 8-lane groups combine the quarter aggregates here; 16-lane groups write their halves to
        // global memory from registers (kw_combine_halves combines them)
        std::conditional_t<(G == kGL), SF<D>[NP], char> q;
        union {                                    // U in the step loop, s in the final combination
            std::conditional_t<(G == kGL), SCombF<D>, char> s;
            double U[NP][D][LD(D)];
        };
        double fqs[NP][2][FQS(D, STREAM)];         // STREAM: each quarter's (F_k, Q_k) staged one step ahead
    } w[WPC];
};

#ifndef PSSGP_WLPR_MINB
#define PSSGP_WLPR_MINB 4                        // resident CTAs/SM the lane-per-row fold is register-capped for
#endif
// lane-per-row kernels with G-lane groups: G = 8 (D <= 8, four quarter chains per warp, 4 warps per CTA)
// or G = 16 (9 <= D <= 16, two half chains per warp, 2 warps per CTA: the per-warp shared state of
// d = 16 would otherwise cap residency at one CTA per SM); register cap 168 / 255
PS_CX int lpr_minb(int G) { return G == kGL ? PSSGP_WLPR_MINB : 4; }
// F's block-diagonal structure (sum models: one block per component; periodic components: 2 x 2
// rotation blocks; quasi-periodic products: blocks of 2 m): FB = the aligned block size every
// nonzero of G and W lies within (the host checks it, pssgp_model::fblock; FB = D = dense), so
// products with F skip its structural zeros at compile time: row i of F is nonzero only in columns
// [fblo(i), fbhi(i)).
PS_CX int fblo(int i, int FB) { return (i / FB) * FB; }
PS_CX int fbhi(int i, int FB, int D) { return (i / FB) * FB + FB < D ? (i / FB) * FB + FB : D; }
PS_CX unsigned group_mask(int G, int gb) { return (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << gb; }

// ------------------------------------------------------------------ KDl: lane-per-row discretisation
// The same algorithm as kw_discretize (Taylor expm of G tau and the Van Loan series of Q_tau, then s
// squarings: supp. P:294-303) with one step per 8-lane group and row r of every matrix in lane r's
// registers; products take the other rows by group shuffles.  Four steps per warp, no shared
// memory, no __syncwarp phases.  The A Z + (A Z)^T symmetrisation is formed as A Z + Z A^T with
// the same products in the same order (Z symmetric), so it is exactly symmetric as before.
template <int D>
__device__ __forceinline__ void g_mm(double (&out)[D], const double (&x)[D], const double (&y)[D], unsigned gm) {
#pragma unroll
    for (int j = 0; j < D; ++j) out[j] = 0.0;
#pragma unroll
    for (int q = 0; q < D; ++q)
#pragma unroll
        for (int j = 0; j < D; ++j) out[j] = fma(x[q], __shfl_sync(gm, y[j], q, kGL), out[j]);
}
template <int D>   // row r of X Y^T (+ add)
__device__ __forceinline__ void g_mmt(double (&out)[D], const double (&x)[D], const double (&y)[D], const double* add,
                                      unsigned gm) {
#pragma unroll
    for (int i = 0; i < D; ++i) out[i] = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) out[i] = fma(x[j], __shfl_sync(gm, y[j], i, kGL), out[i]);
    if (add) {
#pragma unroll
        for (int i = 0; i < D; ++i) out[i] += add[i];
    }
}

#ifndef PSSGP_WDISC_MINB
#define PSSGP_WDISC_MINB 4                       // resident CTAs/SM kw_discretize_lpr is register-capped for (1: 5.31, 4: 5.04, 5: 5.31 ms at C3 irregular)
#endif
template <int D>
__global__ void __launch_bounds__(32 * kWWarps, PSSGP_WDISC_MINB) kw_discretize_lpr(const double* __restrict__ t, int64_t nfq, int64_t k0,
                                                                   const double* __restrict__ model, double* fq) {
    static_assert(D <= kGL, "one row per lane of an 8-lane group");
    const int lane = threadIdx.x & 31, grp = lane / kGL, r0 = lane % kGL;
    const bool act = (D == kGL) || r0 < D;
    const int r = act ? r0 : 0;
    const unsigned gm = 0xFFu << (grp * kGL);
    double Gr[D], Wr[D];
    double gnorm = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        Gr[j] = __ldg(model + 3 * D * D + D + 2 + r * D + j);
        Wr[j] = __ldg(model + 4 * D * D + D + 2 + r * D + j);
        double cs = 0.0;
        for (int i = 0; i < D; ++i) cs += fabs(__ldg(model + 3 * D * D + D + 2 + i * D + j));
        gnorm = fmax(gnorm, cs);
    }
    constexpr double c[13] = {1.0, 1.0, 1.0 / 2, 1.0 / 6, 1.0 / 24, 1.0 / 120, 1.0 / 720, 1.0 / 5040, 1.0 / 40320,
                              1.0 / 362880, 1.0 / 3628800, 1.0 / 39916800, 1.0 / 479001600};
    // the Taylor coefficient matrices (MODP) in shared memory for the polynomial path
    __shared__ double FCs[kPolyM + 1][D * D], QCs[kPolyM + 1][D * D];
    for (int e = threadIdx.x; e < (kPolyM + 1) * D * D; e += blockDim.x) {
        FCs[e / (D * D)][e % (D * D)] = __ldg(model + MODW(D) + e);
        QCs[e / (D * D)][e % (D * D)] = __ldg(model + MODW(D) + (kPolyM + 1) * D * D + e);
    }
    __syncthreads();
    const int64_t ng = static_cast<int64_t>(gridDim.x) * blockDim.x / kGL;
    for (int64_t k = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / kGL; k < nfq; k += ng) {
        if (k0 + k == 0) continue;
        const double dt = __ldg(t + k) - __ldg(t + k - 1);
        if (dt == 0.0 || !(dt == dt)) continue;
        const double nrm = gnorm * fabs(dt);
        if (nrm <= kPolyNorm) {
            // small step: F and Q are their Taylor polynomials in the scalar dt (Horner, row r of each
            // coefficient matrix; truncation <= (2 ||G dt||)^13 / 13! relative): no matrix products, no
            // shuffles.  The coefficients are exactly symmetric for Q, so lane j's (j, r) equals (r, j).
            if (act) {
                double* o = fq + k * FQW(D);
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    double f = FCs[kPolyM][r * D + j], q = QCs[kPolyM][r * D + j];
#pragma unroll
                    for (int kk = kPolyM - 1; kk >= 0; --kk) {
                        f = fma(f, dt, FCs[kk][r * D + j]);
                        q = fma(q, dt, QCs[kk][r * D + j]);
                    }
                    o[r * LD(D) + j] = f;
                    o[(D + r) * LD(D) + j] = q * dt;
                }
                o[r * LD(D) + D] = 0.0;
                o[(D + r) * LD(D) + D] = 0.0;
            }
            continue;
        }
        int s = 0;
        if (nrm > 0.125) frexp(nrm / 0.125, &s);
        const bool low = (nrm <= 0.017);
        const double tau = ldexp(dt, -s);
        double A[D], A2[D], A3[D], X[D], B[D], T[D];
#pragma unroll
        for (int j = 0; j < D; ++j) A[j] = Gr[j] * tau;
        g_mm<D>(A2, A, A, gm);
        g_mm<D>(A3, A2, A, gm);
        auto tblock = [&](double (&o)[D], double c0, double c1, double c2, double c3, bool use3) {
#pragma unroll
            for (int j = 0; j < D; ++j) {
                double v = fma(c2, A2[j], c1 * A[j]);
                if (use3) v = fma(c3, A3[j], v);
                o[j] = v + ((j == r) ? c0 : 0.0);
            }
        };
        if (low) {   // m = 6: F = B0 + A3 (c3 I + c4 A + c5 A2 + c6 A3)
            tblock(X, c[3], c[4], c[5], c[6], true);
            tblock(B, c[0], c[1], c[2], 0.0, false);
            g_mm<D>(T, A3, X, gm);
#pragma unroll
            for (int j = 0; j < D; ++j) T[j] += B[j];
        } else {     // m = 12: Horner in A3 over degree-2 blocks, top block degree 3
            tblock(X, c[9], c[10], c[11], c[12], true);
            tblock(B, c[6], c[7], c[8], 0.0, false);
            g_mm<D>(T, A3, X, gm);
#pragma unroll
            for (int j = 0; j < D; ++j) T[j] += B[j];
            tblock(B, c[3], c[4], c[5], 0.0, false);
            g_mm<D>(X, A3, T, gm);
#pragma unroll
            for (int j = 0; j < D; ++j) X[j] += B[j];
            tblock(B, c[0], c[1], c[2], 0.0, false);
            g_mm<D>(T, A3, X, gm);
#pragma unroll
            for (int j = 0; j < D; ++j) T[j] += B[j];
        }
        // Q_tau = sum_k tau^k ... : Z = tau W, Z <- (A Z + Z A^T) / (k + 1), Q += Z
        double Z[D], Qc[D];
#pragma unroll
        for (int j = 0; j < D; ++j) { Z[j] = Wr[j] * tau; Qc[j] = Z[j]; }
        const int mq = low ? 7 : 12;
        for (int kk = 1; kk < mq; ++kk) {
            g_mm<D>(A3, A, Z, gm);
            g_mmt<D>(X, Z, A, nullptr, gm);
            const double ik = 1.0 / (kk + 1);
#pragma unroll
            for (int j = 0; j < D; ++j) {
                Z[j] = (A3[j] + X[j]) * ik;
                Qc[j] += Z[j];
            }
        }
        // doublings: Q <- Q + F Q F^T, F <- F F   (F in T)
        for (int q = 0; q < s; ++q) {
            g_mm<D>(B, T, Qc, gm);
            g_mmt<D>(A2, B, T, Qc, gm);
            g_mm<D>(A3, T, T, gm);
#pragma unroll
            for (int j = 0; j < D; ++j) { Qc[j] = A2[j]; T[j] = A3[j]; }
        }
        // column r of Q (lane j's element r) for the symmetrised output
        double Qt[D];
#pragma unroll
        for (int cc = 0; cc < D; ++cc)
#pragma unroll
            for (int j = 0; j < D; ++j) {
                const double v = __shfl_sync(gm, Qc[cc], j, kGL);
                if (cc == r) Qt[j] = v;
            }
        if (act) {
            double* o = fq + k * FQW(D);
#pragma unroll
            for (int j = 0; j < D; ++j) {
                o[r * LD(D) + j] = T[j];
                o[(D + r) * LD(D) + j] = 0.5 * (Qc[j] + Qt[j]);
            }
            // the padding column too, so every sector of the record is written whole (no DRAM
            // fill reads for partially written sectors: 1.66 GB per launch at C3 without it)
            o[r * LD(D) + D] = 0.0;
            o[(D + r) * LD(D) + D] = 0.0;
        }
    }
}
// scratch of one general filtering operator on two loaded aggregates (scans, half combination)
template <int D>
struct ScanSmemF {
    SF<D> a, b;
    SCombF<D> s;
};

template <int D, bool STREAM, int G = kGL, int WPC = kWWarps, int FB = D>
__global__ void __launch_bounds__(32 * WPC, lpr_minb(G)) kw_filter_fold_lpr(const WParams p) {
    static_assert(D <= G, "lane-per-row fold holds one row per lane of a G-lane group");
    constexpr int NP = 32 / G;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K1LSmem<D, STREAM, G, WPC>& sh = *reinterpret_cast<K1LSmem<D, STREAM, G, WPC>*>(smem_raw);
    load_model<D>(sh.m, p.model);
    for (int e = threadIdx.x; e < D * D; e += blockDim.x) {
        const int i = e / D, j = e - (e / D) * D;
        sh.I[i][j] = (i == j) ? 1.0 : 0.0;
        sh.Z[i][j] = 0.0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = blockIdx.x * WPC + wid;
    if (c >= p.nch) return;                                     // warp-uniform
    const int q = lane / G, r = lane % G, gb = q * G;
    const bool act = (D == G) || r < D;                       // compile-time true when the group is full
    const int rr = act ? r : 0;                                 // row addressed by idle lanes
    auto& W = sh.w[wid];
    const SModel<D>& M = sh.m;
    const int64_t kb = static_cast<int64_t>(c) * p.K;
    const int64_t ke = min(kb + p.K, p.n);
    const int64_t Kq = (p.K + NP - 1) / NP;
    const int64_t qb = min(kb + q * Kq, ke), qe = min(qb + Kq, ke);

    double Ac[D], Cr[D], Jr[D], b = 0.0, eta = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) { Ac[i] = (i == r) ? 1.0 : 0.0; Cr[i] = 0.0; Jr[i] = 0.0; }
    double tprev = (qb < qe && (qb > 0 || p.k0 > 0)) ? __ldg(p.t + qb - 1) : 0.0;
    double tn_ = 0.0, yn_ = 0.0;
    unsigned char mn_ = 0;
    if (qb < qe) { tn_ = __ldg(p.t + qb); mn_ = __ldg(p.mask + qb); yn_ = __ldg(p.y + qb); }
    const double hr = act ? M.H[r] : 0.0;
    auto& fqs = W.fqs[q];
    if (STREAM) {
        if (qb < qe)
            for (int i = r; i < FQW(D); i += G) cp_async8(&fqs[0][i], p.fq + qb * FQW(D) + i, 8);
        cp_async_commit();
    }
    for (int64_t j = 0; j < Kq; ++j) {
        const int64_t k = qb + j;
        const int fb = static_cast<int>(j & 1);
        if (STREAM) {
            // slot fb holds (F_k, Q_k); slot fb^1 was last read in step j - 1, before this sync
            cp_async_wait<0>();
            __syncwarp();
            if (k + 1 < qe)
                for (int i = r; i < FQW(D); i += G) cp_async8(&fqs[fb ^ 1][i], p.fq + (k + 1) * FQW(D) + i, 8);
            cp_async_commit();
        }
        const bool valid = k < qe;
        const double tk = tn_;
        const bool obs = valid && mn_ != 0;
        const double yk = obs ? yn_ : 0.0;
        if (k + 1 < qe) { tn_ = __ldg(p.t + k + 1); mn_ = __ldg(p.mask + k + 1); yn_ = __ldg(p.y + k + 1); }
        const int64_t g = p.k0 + k;
        int kind = 1;                                            // identity step past the quarter's end
        if (valid) kind = (g == 0) ? 3 : wdisc_kind(tk - tprev, M.udt, STREAM);
        if (valid && r == 0) {
            if (g > 0 && !(tk - tprev >= 0.0)) raise_error(p.err, g, kErrInput);
            if (!isfinite(tk) || (obs && !isfinite(yk))) raise_error(p.err, g, kErrInput);
            if (kind == 2) raise_error(p.err, g, kErrUnsupported);
        }
        if (valid) tprev = tk;
        const double* Fp;
        const double* Qp;
        if (kind == 0) {
            if (STREAM) { Fp = &fqs[fb][0]; Qp = Fp + D * LD(D); }
            else { Fp = &M.F[0][0]; Qp = &M.Q[0][0]; }
        } else if (kind == 1) {
            Fp = &sh.I[0][0]; Qp = &sh.Z[0][0];
        } else {                                                 // 3 (and 2, reported): F = 0, Q = P_inf
            Fp = &sh.Z[0][0]; Qp = &M.Pinf[0][0];
        }
        // FA column r and U = F C column r (column r of C = row r)
        double FAc[D], Uc[D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double sa = 0.0, su = 0.0;
#pragma unroll
            for (int kk = fblo(i, FB); kk < fbhi(i, FB, D); ++kk) {
                const double f = Fp[i * LD(D) + kk];
                sa = fma(f, Ac[kk], sa);
                su = fma(f, Cr[kk], su);
            }
            FAc[i] = sa;
            Uc[i] = su;
        }
        // Fb_r = F[r,:] b
        double Fb = 0.0;
#pragma unroll
        for (int kk = 0; kk < D; ++kk) Fb = fma(Fp[rr * LD(D) + kk], __shfl_sync(0xffffffffu, b, gb + kk), Fb);
        // row r of U through shared; Cm row r = U[r,:] F^T + Q[r,:]
        if (act) {
#pragma unroll
            for (int i = 0; i < D; ++i) W.U[q][i][r] = Uc[i];
        }
        __syncwarp();
        double Ur[D];
#pragma unroll
        for (int kk = 0; kk < D; ++kk) Ur[kk] = W.U[q][rr][kk];
        __syncwarp();
        double Cm[D];
        double HC = 0.0, w = 0.0;
#pragma unroll
        for (int jj = 0; jj < D; ++jj) {
            double s = Qp[rr * LD(D) + jj];
#pragma unroll
            for (int kk = fblo(jj, FB); kk < fbhi(jj, FB, D); ++kk) s = fma(Ur[kk], Fp[jj * LD(D) + kk], s);
            Cm[jj] = s;
            HC = fma(s, M.H[jj], HC);
            w = fma(M.H[jj], FAc[jj], w);
        }
        if (!act) { HC = 0.0; w = 0.0; Fb = 0.0; }
        double S = hr * HC, hb = hr * Fb;
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) {
            S += __shfl_xor_sync(0xffffffffu, S, off);
            hb += __shfl_xor_sync(0xffffffffu, hb, off);
        }
        S += M.r;
        const double iS = obs ? 1.0 / S : 0.0;
        const double vs = obs ? (yk - hb) * iS : 0.0;
        const double HCs = HC * iS, ws = w * iS;
#pragma unroll
        for (int jj = 0; jj < D; ++jj) {
            const double HCj = __shfl_sync(0xffffffffu, HC, gb + jj);
            const double wj = __shfl_sync(0xffffffffu, w, gb + jj);
            Ac[jj] = fma(-HCj * iS, w, FAc[jj]);
            Cr[jj] = fma(-HCs, HCj, Cm[jj]);
            Jr[jj] = fma(ws, wj, Jr[jj]);
        }
        b = fma(HC, vs, Fb);
        eta = fma(w, vs, eta);
    }
    if constexpr (G > kGL) {
        // two half aggregates straight from registers to global memory (A by columns, C and J by rows,
        // the gstore layout): q0 -> qagg[c] (the prefix the second half's rescan starts from), q1 ->
        // fbuf[c]; kw_combine_halves forms fagg[c] = q0 (x) q1
        static_assert(NP == 2, "16-lane groups: two halves");
        if (act) {
            double* g = (q == 0) ? p.qagg + static_cast<int64_t>(c) * FNW(D) : p.fbuf + static_cast<int64_t>(c) * FNW(D);
#pragma unroll
            for (int i = 0; i < D; ++i) {
                g[i * D + r] = Ac[i];
                g[D * D + D + r * D + i] = Cr[i];
                g[2 * D * D + 2 * D + r * D + i] = Jr[i];
            }
            g[D * D + r] = b;
            g[2 * D * D + D + r] = eta;
        }
        return;
    } else {
    // quarter aggregates -> shared, ordered combination, store
    if (act) {
        SF<D>& o = W.q[q];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            o.A[i][r] = Ac[i];
            o.C[r][i] = Cr[i];
            o.J[r][i] = Jr[i];
        }
        o.b[r] = b;
        o.eta[r] = eta;
    }
    __syncwarp();
    bool ok = true;
#pragma unroll 1
    for (int i = 1; i < NP; ++i) {
        // W.q[i - 1] is the prefix q0 (x) ... (x) q_{i-1}: the quarter rescans start from the
        // chain carry applied to it (kw_filter_apply_q)
        if (p.qagg) gstore<D>(W.q[i - 1], p.qagg + (static_cast<int64_t>(c) * (NP - 1) + (i - 1)) * FNW(D), lane);
        ok = wcombine<D>(W.q[i - 1], W.q[i], W.q[i], W.s, lane) && ok;
        __syncwarp();
    }
    if (!ok && lane == 0) raise_error(p.err, p.k0 + kb, kErrNumeric);
    gstore<D>(W.q[NP - 1], p.fagg + static_cast<int64_t>(c) * FNW(D), lane);
    }
}

// fagg[c] = qagg[c] (x) fbuf[c]: the chain aggregate from the two half aggregates of the 16-lane fold
// (PAPER.md:116-121).  One warp per chain.
template <int D>
__global__ void __launch_bounds__(32) kw_combine_halves(const WParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ScanSmemF<D>& sh = *reinterpret_cast<ScanSmemF<D>*>(smem_raw);
    const int lane = threadIdx.x, c = blockIdx.x;
    gload<D>(sh.a, p.qagg + static_cast<int64_t>(c) * FNW(D), lane);
    gload<D>(sh.b, p.fbuf + static_cast<int64_t>(c) * FNW(D), lane);
    if (!wcombine<D>(sh.a, sh.b, sh.b, sh.s, lane) && lane == 0) raise_error(p.err, p.k0 + static_cast<int64_t>(c) * p.K, kErrNumeric);
    gstore<D>(sh.b, p.fagg + static_cast<int64_t>(c) * FNW(D), lane);
}

// ------------------------------------------------------------------ Kogge-Stone scan levels (1 warp per element)
template <int D>
__global__ void __launch_bounds__(32) kw_scan_filter(const double* __restrict__ in, double* __restrict__ out, int nch,
                                                     int off, unsigned long long* err) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ScanSmemF<D>& sh = *reinterpret_cast<ScanSmemF<D>*>(smem_raw);
    const int lane = threadIdx.x;
    const int c = blockIdx.x;
    if (c >= off) {
        gload<D>(sh.a, in + static_cast<int64_t>(c - off) * FNW(D), lane);
        gload<D>(sh.b, in + static_cast<int64_t>(c) * FNW(D), lane);
        if (!wcombine<D>(sh.a, sh.b, sh.b, sh.s, lane) && lane == 0) raise_error(err, c, kErrNumeric);
        gstore<D>(sh.b, out + static_cast<int64_t>(c) * FNW(D), lane);
    } else {
        for (int e = lane; e < FNW(D); e += 32) out[static_cast<int64_t>(c) * FNW(D) + e] = in[static_cast<int64_t>(c) * FNW(D) + e];
    }
}

template <int D>
struct ScanSmemS {
    SS<D> a, b;
    SCombF<D> s;
};
template <int D>
__global__ void __launch_bounds__(32) kw_scan_smoother(const double* __restrict__ in, double* __restrict__ out,
                                                       int nch, int off) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ScanSmemS<D>& sh = *reinterpret_cast<ScanSmemS<D>*>(smem_raw);
    const int lane = threadIdx.x;
    const int c = blockIdx.x;
    if (c + off < nch) {
        gload<D>(sh.a, in + static_cast<int64_t>(c) * SNW(D), lane);
        gload<D>(sh.b, in + static_cast<int64_t>(c + off) * SNW(D), lane);
        wcombine<D>(sh.a, sh.b, sh.b, sh.s, lane);
        gstore<D>(sh.b, out + static_cast<int64_t>(c) * SNW(D), lane);
    } else {
        for (int e = lane; e < SNW(D); e += 32) out[static_cast<int64_t>(c) * SNW(D) + e] = in[static_cast<int64_t>(c) * SNW(D) + e];
    }
}

// ------------------------------------------------------------------ K3w: Kalman rescan
template <int D>
struct K3Smem {
    SModel<D> m;
    struct PerWarp {
        double P[D][LD(D)];
        double x[D];
        union {
            struct {                  // carry phase (wapply_prefix_gj with its own scratch)
                SF<D> a;
                double Mb[D][LD(D)], Xb[D][LD(D)], Tb[D][LD(D)];
                double v1[D], v2[D];
            } c;
            struct {                  // step phase (+ chain smoother aggregate)
                double Sg[D][LD(D)], P0[D][LD(D)], Sm[D][LD(D)], Pm[D][LD(D)], FP[D][LD(D)];
                double xm[D], x0[D], HP[D], SH[D];
                SS<D> sagg;
            } st;
        } u;
    } w[kWWarps];
};

// chain smoother aggregate (E, g, L) of K3w from the chain's last filtered moments (W.P, W.x) and
// the propagated moments (W.u.st.Sg, P0, x0); shared by both K3w kernels
template <int D>
__device__ void k3w_chain_sagg(const WParams& p, typename K3Smem<D>::PerWarp& W, const SModel<D>& M, int c,
                               int64_t kb, int64_t ke, double tprev, int lane) {
    // ---- chain smoother aggregate (E, g, L), as in the d <= 3 path
    SS<D>* sagg = &W.u.st.sagg;
    if (ke <= kb) {
        set_identity<D>(*sagg, lane);
    } else if (p.k0 + ke == p.nglob) {
        for (int e = lane; e < D * D; e += 32) {
            const int i = e / D, j = e - (e / D) * D;
            sagg->E[i][j] = 0.0;
            sagg->L[i][j] = W.u.st.P0[i][j];
        }
        for (int i = lane; i < D; i += 32) sagg->g[i] = W.u.st.x0[i];
        __syncwarp();
    } else {
        const double tn = __ldg(p.t + ke);
        const int kind = wdisc_kind(tn - tprev, M.udt, p.fq != nullptr);
        const FQp<D> fqp = wfq<D>(p, M, ke);
        // Pm, xm of the next step; Sm = Sg F^T
        for (int e = lane; e < D * D; e += 32) {
            const int i = e / D, j = e - (e / D) * D;
            double fp = 0.0, sm = 0.0;
            if (kind == 0) {
                for (int q = 0; q < D; ++q) {
                    fp = fma(fqp.F[i][q], W.P[q][j], fp);
                    sm = fma(W.u.st.Sg[i][q], fqp.F[j][q], sm);
                }
            } else {
                fp = W.P[i][j];
                sm = W.u.st.Sg[i][j];
            }
            W.u.st.FP[i][j] = fp;
            W.u.st.Sm[i][j] = sm;
        }
        for (int i = lane; i < D; i += 32) {
            double s = 0.0;
            if (kind == 0)
                for (int q = 0; q < D; ++q) s = fma(fqp.F[i][q], W.x[q], s);
            else
                s = W.x[i];
            W.u.st.xm[i] = s;
        }
        __syncwarp();
        for (int e = lane; e < D * D; e += 32) {
            const int i = e / D, j = e - (e / D) * D;
            double s = (kind == 0) ? fqp.Q[i][j] : 0.0;
            if (kind == 0)
                for (int q = 0; q < D; ++q) s = fma(W.u.st.FP[i][q], fqp.F[j][q], s);
            else
                s = W.u.st.FP[i][j];
            W.u.st.Pm[i][j] = s;
        }
        __syncwarp();
        // E = Sm Pm^-1 (Pm symmetric): a register Gauss-Jordan solve, no explicit inverse
        if (!wright_div_sym_gj<D>(sagg->E, W.u.st.Sm, W.u.st.Pm, lane) && lane == 0)
            raise_error(p.err, p.k0 + ke, kErrNumeric);
        for (int i = lane; i < D; i += 32) {
            double a = W.u.st.x0[i];
            for (int q = 0; q < D; ++q) a = fma(-sagg->E[i][q], W.u.st.xm[q], a);
            sagg->g[i] = a;
        }
        for (int e = lane; e < D * D; e += 32) {
            const int i = e / D, j = e - (e / D) * D;
            double a = W.u.st.P0[i][j];
            for (int q = 0; q < D; ++q) a = fma(-sagg->E[i][q], W.u.st.Sm[j][q], a);
            W.u.st.Pm[i][j] = a;
        }
        __syncwarp();
        for (int e = lane; e < D * D; e += 32) {
            const int i = e / D, j = e - (e / D) * D;
            sagg->L[i][j] = 0.5 * (W.u.st.Pm[i][j] + W.u.st.Pm[j][i]);
        }
        __syncwarp();
    }
    gstore<D>(*sagg, p.sagg + static_cast<int64_t>(c) * SNW(D), lane);
}

template <int D>
__global__ void __launch_bounds__(32 * kWWarps, PSSGP_WMINB) kw_filter_apply(const WParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K3Smem<D>& sh = *reinterpret_cast<K3Smem<D>*>(smem_raw);
    load_model<D>(sh.m, p.model);
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = blockIdx.x * kWWarps + wid;
    if (c >= p.nch) return;
    auto& W = sh.w[wid];
    const SModel<D>& M = sh.m;
    // ---- carry (x, P) entering the chain: incoming (sharded) (x) inclusive scan up to chain c-1
    for (int e = lane; e < D * D; e += 32) W.P[e / D][e % D] = 0.0;
    for (int i = lane; i < D; i += 32) W.x[i] = 0.0;
    __syncwarp();
    for (int g = 0; g < p.rank && p.in_filt; ++g) {
        gload<D>(W.u.c.a, p.in_filt + static_cast<int64_t>(g) * FNW(D), lane);
        if (!wapply_prefix_gj<D>(W.x, W.P, W.u.c.a, W.u.c.Mb, W.u.c.Xb, W.u.c.Tb, W.u.c.v1, W.u.c.v2, lane) && lane == 0) raise_error(p.err, p.k0, kErrNumeric);
    }
    if (c > 0) {
        gload<D>(W.u.c.a, p.fagg + static_cast<int64_t>(c - 1) * FNW(D), lane);
        if (!wapply_prefix_gj<D>(W.x, W.P, W.u.c.a, W.u.c.Mb, W.u.c.Xb, W.u.c.Tb, W.u.c.v1, W.u.c.v2, lane) && lane == 0) raise_error(p.err, p.k0, kErrNumeric);
    }
    const int64_t kb = static_cast<int64_t>(c) * p.K;
    const int64_t ke = min(kb + p.K, p.n);
    double tprev = (kb < p.n && (kb > 0 || p.k0 > 0)) ? __ldg(p.t + kb - 1) : 0.0;
    double quad = 0.0, logs = 0.0;
    int nobs = 0;
    double* xpc = p.xp + static_cast<int64_t>(c) * p.K * CNW(D);
    double tn_ = 0.0, yn_ = 0.0;                        // next step's inputs, prefetched
    unsigned char mn_ = 0;
    if (kb < ke) { tn_ = __ldg(p.t + kb); mn_ = __ldg(p.mask + kb); yn_ = __ldg(p.y + kb); }
    for (int64_t k = kb; k < ke; ++k) {
        const double tk = tn_;
        const bool obs = mn_ != 0;
        const double yk = obs ? yn_ : 0.0;
        if (k + 1 < ke) { tn_ = __ldg(p.t + k + 1); mn_ = __ldg(p.mask + k + 1); yn_ = __ldg(p.y + k + 1); }
        const int64_t g = p.k0 + k;
        const int kind = (g == 0) ? 3 : wdisc_kind(tk - tprev, M.udt, p.fq != nullptr);
        const FQp<D> fqp = wfq<D>(p, M, k);
        const bool first = (k == kb);
        tprev = tk;
        // predict: xm = F x, FP = F P, Pm = FP F^T + Q ; Sm = Sg F^T
        if (kind == 0) {
            wmm<D>(W.u.st.FP, fqp.F, W.P, nullptr, lane);
            if (!first) wmm<D, false, true>(W.u.st.Sm, W.u.st.Sg, fqp.F, nullptr, lane);
            for (int i = lane; i < D; i += 32) {
                double s = 0.0;
                for (int q = 0; q < D; ++q) s = fma(fqp.F[i][q], W.x[q], s);
                W.u.st.xm[i] = s;
            }
            __syncwarp();
            wmm<D, false, true>(W.u.st.Pm, W.u.st.FP, fqp.F, fqp.Q, lane);
        } else {
            for (int e = lane; e < D * D; e += 32) {
                const int i = e / D, j = e - (e / D) * D;
                W.u.st.Sm[i][j] = (kind == 1) ? W.u.st.Sg[i][j] : 0.0;
                W.u.st.Pm[i][j] = (kind == 1) ? W.P[i][j] : M.Pinf[i][j];
            }
            for (int i = lane; i < D; i += 32) W.u.st.xm[i] = (kind == 1) ? W.x[i] : 0.0;
        }
        __syncwarp();
        for (int i = lane; i < D; i += 32) {
            double hp = 0.0, sh_ = 0.0;
            for (int q = 0; q < D; ++q) {
                hp = fma(W.u.st.Pm[i][q], M.H[q], hp);
                sh_ = fma(W.u.st.Sm[i][q], M.H[q], sh_);
            }
            W.u.st.HP[i] = hp;
            W.u.st.SH[i] = sh_;
        }
        __syncwarp();
        const double S = wdot<D>(M.H, W.u.st.HP, lane) + M.r;
        const double hx = wdot<D>(M.H, W.u.st.xm, lane);
        if (lane == 0 && obs && !(S > 0.0 && S < INFINITY)) raise_error(p.err, g, kErrNumeric);
        const double iS = obs ? 1.0 / S : 0.0;
        const double v = obs ? (yk - hx) : 0.0;
        const double vs = v * iS;
        for (int e = lane; e < D * D; e += 32) {
            const int i = e / D, j = e - (e / D) * D;
            const double Pn = fma(-W.u.st.HP[i] * iS, W.u.st.HP[j], W.u.st.Pm[i][j]);
            W.P[i][j] = Pn;
            if (first) {
                W.u.st.P0[i][j] = Pn;
                W.u.st.Sg[i][j] = Pn;
            } else {
                W.u.st.Sg[i][j] = fma(-W.u.st.SH[i] * iS, W.u.st.HP[j], W.u.st.Sm[i][j]);
                W.u.st.P0[i][j] = fma(-W.u.st.SH[i] * iS, W.u.st.SH[j], W.u.st.P0[i][j]);
            }
        }
        for (int i = lane; i < D; i += 32) {
            const double xn = fma(W.u.st.HP[i], vs, W.u.st.xm[i]);
            W.x[i] = xn;
            W.u.st.x0[i] = first ? xn : fma(W.u.st.SH[i], vs, W.u.st.x0[i]);
        }
        if (obs) {
            quad = fma(v, vs, quad);
            logs += log(S);
            ++nobs;
        }
        __syncwarp();
        if (p.store_state) {
            double* o = xpc + (k - kb) * CNW(D);
            for (int i = lane; i < D; i += 32) o[i] = W.x[i];
            for (int e = lane; e < D * D; e += 32) {
                const int i = e / D, j = e - (e / D) * D;
                if (j >= i) o[D + si(D, i, j)] = W.P[i][j];
            }
        }
    }
    if (lane == 0) {
        p.nll_chain[c] = nobs ? 0.5 * (quad + logs + nobs * 1.8378770664093453) : 0.0;
    }
    if (!p.store_state) return;
    k3w_chain_sagg<D>(p, W, M, c, kb, ke, tprev, lane);
}

// ------------------------------------------------------------------ K3w for D <= 8: lane-per-row Kalman rescan
// Same grid, carry, outputs and chain smoother aggregate as kw_filter_apply; the step recursion
// (PAPER.md:285-324 Kalman step from the collapsed carry, Prop. 1 order) runs in registers with
// lane r (< D) owning row r of P, Sg = Cov(x_k0, x_k), P0 and x_r, x0_r; F P is transposed
// through a per-warp shared buffer, the full x, HP, SH vectors are gathered by shuffles.  The
// moments are written back to the shared layout for the chain smoother aggregate.
template <int D, bool STREAM>
struct K3LSmem {
    K3Smem<D> b;
    double I[D][LD(D)], Z[D][LD(D)];
    double U[kWWarps][D][LD(D)];
    double fqs[kWWarps][2][FQS(D, STREAM)];         // STREAM: per-step (F_k, Q_k) staged one step ahead
};

template <int D, bool STREAM>
__global__ void __launch_bounds__(32 * kWWarps, PSSGP_WLPR_MINB) kw_filter_apply_lpr(const WParams p) {
    static_assert(D <= kGL, "lane-per-row rescan holds one row per lane");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K3LSmem<D, STREAM>& shl = *reinterpret_cast<K3LSmem<D, STREAM>*>(smem_raw);
    K3Smem<D>& sh = shl.b;
    load_model<D>(sh.m, p.model);
    for (int e = threadIdx.x; e < D * D; e += blockDim.x) {
        const int i = e / D, j = e - (e / D) * D;
        shl.I[i][j] = (i == j) ? 1.0 : 0.0;
        shl.Z[i][j] = 0.0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = blockIdx.x * kWWarps + wid;
    if (c >= p.nch) return;
    auto& W = sh.w[wid];
    auto& U = shl.U[wid];
    const SModel<D>& M = sh.m;
    // ---- carry (x, P) entering the chain (warp-cooperative, as kw_filter_apply)
    for (int e = lane; e < D * D; e += 32) W.P[e / D][e % D] = 0.0;
    for (int i = lane; i < D; i += 32) W.x[i] = 0.0;
    __syncwarp();
    for (int g = 0; g < p.rank && p.in_filt; ++g) {
        gload<D>(W.u.c.a, p.in_filt + static_cast<int64_t>(g) * FNW(D), lane);
        if (!wapply_prefix_gj<D>(W.x, W.P, W.u.c.a, W.u.c.Mb, W.u.c.Xb, W.u.c.Tb, W.u.c.v1, W.u.c.v2, lane) && lane == 0) raise_error(p.err, p.k0, kErrNumeric);
    }
    if (c > 0) {
        gload<D>(W.u.c.a, p.fagg + static_cast<int64_t>(c - 1) * FNW(D), lane);
        if (!wapply_prefix_gj<D>(W.x, W.P, W.u.c.a, W.u.c.Mb, W.u.c.Xb, W.u.c.Tb, W.u.c.v1, W.u.c.v2, lane) && lane == 0) raise_error(p.err, p.k0, kErrNumeric);
    }
    const bool act = lane < D;
    const int r = act ? lane : 0;
    double Pr[D], Sgr[D], P0r[D], xr = W.x[r], x0r = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) { Pr[j] = W.P[r][j]; Sgr[j] = 0.0; P0r[j] = 0.0; }
    const double hr = act ? M.H[r] : 0.0;
    __syncwarp();

    const int64_t kb = static_cast<int64_t>(c) * p.K;
    const int64_t ke = min(kb + p.K, p.n);
    double tprev = (kb < p.n && (kb > 0 || p.k0 > 0)) ? __ldg(p.t + kb - 1) : 0.0;
    double quad = 0.0, logs = 0.0;
    int nobs = 0;
    bool bad_s = false;
    int64_t bad_g = 0;
    double* xpc = p.xp + static_cast<int64_t>(c) * p.K * CNW(D);
    double tn_ = 0.0, yn_ = 0.0;
    unsigned char mn_ = 0;
    if (kb < ke) { tn_ = __ldg(p.t + kb); mn_ = __ldg(p.mask + kb); yn_ = __ldg(p.y + kb); }
    auto& fqs = shl.fqs[wid];
    if (STREAM && kb < ke) {
        const double* src = p.fq + kb * FQW(D);
        for (int i = lane; i < FQW(D); i += 32) cp_async8(&fqs[0][i], src + i, 8);
        cp_async_commit();
    }
    for (int64_t k = kb; k < ke; ++k) {
        const int fb = static_cast<int>((k - kb) & 1);
        if (STREAM) {
            // (F_k, Q_k) staged in slot fb; slot fb^1 was last read before the previous step's
            // closing __syncwarp, so the copy for k + 1 may start once this one is visible
            cp_async_wait<0>();
            __syncwarp();
            if (k + 1 < ke) {
                const double* src = p.fq + (k + 1) * FQW(D);
                for (int i = lane; i < FQW(D); i += 32) cp_async8(&fqs[fb ^ 1][i], src + i, 8);
                cp_async_commit();
            }
        }
        const double tk = tn_;
        const bool obs = mn_ != 0;
        const double yk = obs ? yn_ : 0.0;
        if (k + 1 < ke) { tn_ = __ldg(p.t + k + 1); mn_ = __ldg(p.mask + k + 1); yn_ = __ldg(p.y + k + 1); }
        const int64_t g = p.k0 + k;
        const int kind = (g == 0) ? 3 : wdisc_kind(tk - tprev, M.udt, STREAM);
        const bool first = (k == kb);
        tprev = tk;
        const double* Fp;
        const double* Qp;
        if (kind == 0) {
            if (STREAM) { Fp = &fqs[fb][0]; Qp = Fp + D * LD(D); }
            else { Fp = &M.F[0][0]; Qp = &M.Q[0][0]; }
        } else if (kind == 1) {
            Fp = &shl.I[0][0]; Qp = &shl.Z[0][0];
        } else {                                     // 3 (and 2, reported by the fold): F = 0, Q = P_inf
            Fp = &shl.Z[0][0]; Qp = &M.Pinf[0][0];
        }
        // column r of F P, xm_r = F[r,:] x, row r of Sm = Sg[r,:] F^T
        double Uc[D], xm = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double su = 0.0;
#pragma unroll
            for (int q = 0; q < D; ++q) su = fma(Fp[i * LD(D) + q], Pr[q], su);
            Uc[i] = su;
        }
#pragma unroll
        for (int q = 0; q < D; ++q) xm = fma(Fp[r * LD(D) + q], __shfl_sync(0xffffffffu, xr, q), xm);
        if (act) {
#pragma unroll
            for (int i = 0; i < D; ++i) U[i][r] = Uc[i];
        }
        __syncwarp();
        double Pm[D], Sm[D], HP = 0.0, SH = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            double s2 = Qp[r * LD(D) + j], s3 = 0.0;
#pragma unroll
            for (int q = 0; q < D; ++q) {
                const double f = Fp[j * LD(D) + q];
                s2 = fma(U[r][q], f, s2);
                s3 = fma(Sgr[q], f, s3);
            }
            Pm[j] = s2;
            Sm[j] = s3;
            HP = fma(s2, M.H[j], HP);
            SH = fma(s3, M.H[j], SH);
        }
        __syncwarp();                                 // U is rewritten by the next step
        if (!act) { HP = 0.0; SH = 0.0; }
        double S = hr * HP, hx = hr * xm;
#pragma unroll
        for (int off = kGL / 2; off > 0; off >>= 1) {
            S += __shfl_xor_sync(0xffffffffu, S, off);
            hx += __shfl_xor_sync(0xffffffffu, hx, off);
        }
        S += M.r;
        if (obs && !(S > 0.0 && S < INFINITY) && !bad_s) { bad_s = true; bad_g = g; }
        const double iS = obs ? 1.0 / S : 0.0;
        const double v = obs ? (yk - hx) : 0.0;
        const double vs = v * iS;
        const double HPs = HP * iS, SHs = SH * iS;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const double HPj = __shfl_sync(0xffffffffu, HP, j);
            const double SHj = __shfl_sync(0xffffffffu, SH, j);
            const double Pn = fma(-HPs, HPj, Pm[j]);
            Pr[j] = Pn;
            if (first) {
                P0r[j] = Pn;
                Sgr[j] = Pn;
            } else {
                Sgr[j] = fma(-SHs, HPj, Sm[j]);
                P0r[j] = fma(-SHs, SHj, P0r[j]);
            }
        }
        xr = fma(HP, vs, xm);
        x0r = first ? xr : fma(SH, vs, x0r);
        if (obs) {
            quad = fma(v, vs, quad);
            logs += log(S);
            ++nobs;
        }
        if (p.store_state && act) {
            double* o = xpc + (k - kb) * CNW(D);
            o[r] = xr;
#pragma unroll
            for (int j = 0; j < D; ++j)
                if (j >= r) o[D + si(D, r, j)] = Pr[j];
        }
    }
    if (bad_s && lane == 0) raise_error(p.err, bad_g, kErrNumeric);
    if (lane == 0) p.nll_chain[c] = nobs ? 0.5 * (quad + logs + nobs * 1.8378770664093453) : 0.0;
    if (!p.store_state) return;
    // moments back to the shared layout for the chain smoother aggregate
    if (act) {
#pragma unroll
        for (int j = 0; j < D; ++j) {
            W.P[r][j] = Pr[j];
            W.u.st.Sg[r][j] = Sgr[j];
            W.u.st.P0[r][j] = P0r[j];
        }
        W.x[r] = xr;
        W.u.st.x0[r] = x0r;
    }
    __syncwarp();
    k3w_chain_sagg<D>(p, W, M, c, kb, ke, tprev, lane);
}

// ------------------------------------------------------------------ K5w: RTS rescan
template <int D>
struct K5Smem {
    SModel<D> m;
    struct PerWarp {
        double Ps[D][LD(D)];
        double ms[D];
        double xst[2][CNW(D)];            // staged packed (xbar, P) records (cp.async)
        union {
            struct {                  // carry phase
                SS<D> a;
                SSufScratch<D> s;
            } c;
            struct {                  // step phase
                double P[D][LD(D)], Pm[D][LD(D)], FP[D][LD(D)], G[D][LD(D)], T[D][LD(D)];
                double x[D], xm[D], dm[D], Li[D];
            } st;
        } u;
    } w[kWWarps];
};

template <int D>
__global__ void __launch_bounds__(32 * kWWarps, PSSGP_WMINB) kw_smoother_apply(const WParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K5Smem<D>& sh = *reinterpret_cast<K5Smem<D>*>(smem_raw);
    load_model<D>(sh.m, p.model);
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = blockIdx.x * kWWarps + wid;
    // NLL: fixed-order sum of the chain partials (CTA 0, warp 0)
    if (blockIdx.x == 0 && wid == 0 && p.nll_out) {
        double s = 0.0;
        const int per = (p.nch + 31) / 32;
        for (int i = 0; i < per; ++i) {
            const int q = lane * per + i;
            if (q < p.nch) s += p.nll_chain[q];
        }
        for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
        if (lane == 0) *p.nll_out = s;
    }
    if (c >= p.nch) return;
    auto& W = sh.w[wid];
    const SModel<D>& M = sh.m;
    // ---- carry: collapsed suffix after the chain = incoming (sharded) then scanned suffix of c+1
    for (int e = lane; e < D * D; e += 32) W.Ps[e / D][e % D] = 0.0;
    for (int i = lane; i < D; i += 32) W.ms[i] = 0.0;
    __syncwarp();
    for (int g = p.world - 1; g > p.rank && p.in_smooth; --g) {
        gload<D>(W.u.c.a, p.in_smooth + static_cast<int64_t>(g) * (SNW(D) + 1), lane);   // blob = aggregate + NLL partial
        wapply_suffix<D>(W.u.c.a, W.ms, W.Ps, W.u.c.s, lane);
    }
    if (c + 1 < p.nch) {
        gload<D>(W.u.c.a, p.sagg + static_cast<int64_t>(c + 1) * SNW(D), lane);
        wapply_suffix<D>(W.u.c.a, W.ms, W.Ps, W.u.c.s, lane);
    }
    const int64_t kb = static_cast<int64_t>(c) * p.K;
    const int64_t ke = min(kb + p.K, p.n);
    const double* xpc = p.xp + static_cast<int64_t>(c) * p.K * CNW(D);
    double tnext = (ke > kb && p.k0 + ke < p.nglob) ? __ldg(p.t + ke) : 0.0;
    // the packed (xbar, P) record of the next step down is staged by cp.async one step ahead
    // (double buffer per warp), t one step ahead in a register
    double tk_next = 0.0;
    if (ke > kb) {
        const double* src = xpc + (ke - 1 - kb) * CNW(D);
        for (int i = lane; i < CNW(D); i += 32) cp_async8(&W.xst[0][i], src + i, 8);
        cp_async_commit();
        tk_next = __ldg(p.t + ke - 1);
    }
    int sb = 0;
    for (int64_t k = ke - 1; k >= kb; --k) {
        const double tk = tk_next;
        const int64_t g = p.k0 + k;
        cp_async_wait<0>();
        __syncwarp();
        if (k > kb) {
            const double* src = xpc + (k - 1 - kb) * CNW(D);
            for (int i = lane; i < CNW(D); i += 32) cp_async8(&W.xst[sb ^ 1][i], src + i, 8);
            cp_async_commit();
            tk_next = __ldg(p.t + k - 1);
        }
        {
            const double* src = W.xst[sb];
            for (int i = lane; i < D; i += 32) W.u.st.x[i] = src[i];
            for (int e = lane; e < D * D; e += 32) {
                const int i = e / D, j = e - (e / D) * D;
                W.u.st.P[i][j] = src[D + si(D, i, j)];
            }
        }
        sb ^= 1;
        __syncwarp();
        if (g == p.nglob - 1) {
            for (int e = lane; e < D * D; e += 32) W.Ps[e / D][e % D] = W.u.st.P[e / D][e % D];
            for (int i = lane; i < D; i += 32) W.ms[i] = W.u.st.x[i];
            __syncwarp();
        } else {
            const int kind = wdisc_kind(tnext - tk, M.udt, p.fq != nullptr);
            const FQp<D> fqp = wfq<D>(p, M, k + 1);
            if (kind == 0) {
                wmm<D>(W.u.st.FP, fqp.F, W.u.st.P, nullptr, lane);                     // F P
                for (int i = lane; i < D; i += 32) {
                    double s2 = 0.0;
                    for (int q = 0; q < D; ++q) s2 = fma(fqp.F[i][q], W.u.st.x[q], s2);
                    W.u.st.xm[i] = s2;
                }
                __syncwarp();
                wmm<D, false, true>(W.u.st.Pm, W.u.st.FP, fqp.F, fqp.Q, lane);         // F P F^T + Q
            } else {
                for (int e = lane; e < D * D; e += 32) {
                    const int i = e / D, j = e - (e / D) * D;
                    W.u.st.FP[i][j] = W.u.st.P[i][j];
                    W.u.st.Pm[i][j] = W.u.st.P[i][j];
                }
                for (int i = lane; i < D; i += 32) W.u.st.xm[i] = W.u.st.x[i];
            }
            __syncwarp();
            // X = Pm^-1 F P (so G = P F^T Pm^-1 = X^T) by Cholesky, lanes over right-hand sides
#if PSSGP_WIDE_CHOL
            if (!wcholesky<D>(W.u.st.Pm, W.u.st.T, W.u.st.Li, lane) && lane == 0) raise_error(p.err, g, kErrNumeric);
            wchol_solve<D>(W.u.st.T, W.u.st.Li, W.u.st.FP, W.u.st.G, lane);                  // W.u.st.G holds X (not G)
#else
            if (!wgj_solve<D>(W.u.st.Pm, W.u.st.FP, W.u.st.G, lane) && lane == 0) raise_error(p.err, g, kErrNumeric);
#endif
            // ms = x + X^T (ms - xm)
            for (int i = lane; i < D; i += 32) W.u.st.dm[i] = W.ms[i] - W.u.st.xm[i];
            __syncwarp();
            for (int i = lane; i < D; i += 32) {
                double s2 = W.u.st.x[i];
                for (int q = 0; q < D; ++q) s2 = fma(W.u.st.G[q][i], W.u.st.dm[q], s2);
                W.u.st.xm[i] = s2;
            }
            // Ps = P + X^T (Ps - Pm) X
            for (int e = lane; e < D * D; e += 32) {
                const int i = e / D, j = e - (e / D) * D;
                W.u.st.Pm[i][j] = W.Ps[i][j] - W.u.st.Pm[i][j];
            }
            __syncwarp();
            wmm<D>(W.u.st.T, W.u.st.Pm, W.u.st.G, nullptr, lane);                 // (Ps - Pm) X
            __syncwarp();
            wmm<D, true, false>(W.u.st.FP, W.u.st.G, W.u.st.T, W.u.st.P, lane);        // P + X^T (Ps - Pm) X
            __syncwarp();
            for (int e = lane; e < D * D; e += 32) {
                const int i = e / D, j = e - (e / D) * D;
                W.Ps[i][j] = 0.5 * (W.u.st.FP[i][j] + W.u.st.FP[j][i]);
            }
            for (int i = lane; i < D; i += 32) W.ms[i] = W.u.st.xm[i];
            __syncwarp();
        }
        tnext = tk;
        // projection mean = H m^s, var = H P^s H^T: lane i owns row i, warp sums
        double mo = 0.0, vo = 0.0;
        if (lane < D) {
            double s2 = 0.0;
#pragma unroll 4
            for (int j = 0; j < D; ++j) s2 = fma(W.Ps[lane][j], M.H[j], s2);
            mo = M.H[lane] * W.ms[lane];
            vo = M.H[lane] * s2;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            mo += __shfl_xor_sync(0xffffffffu, mo, off);
            vo += __shfl_xor_sync(0xffffffffu, vo, off);
        }
        if (lane == 0) {
            if (p.mean) p.mean[k] = mo;
            if (p.var) p.var[k] = vo;
        }
        __syncwarp();
    }
}


// ------------------------------------------------------------------ K5w for D <= 8: lane-per-row RTS
// Same grid, carries and outputs as kw_smoother_apply; the per-step RTS recursion (PAPER.md:
// 422-430 / Prop. 2 order) runs in registers with lane r (< D) owning row r of P, P^s
// and column r of F P and X = P^-_{k+1}^-1 F P (so the gain is X^T).  Matrices a lane needs in
// full (P^-, P^s, X) go through per-warp shared buffers; every lane factors P^- (Cholesky,
// upper triangle as the symmetric source of truth) in registers and solves for its own column.
template <int D, bool STREAM>
struct K5LSmem {
    K5Smem<D> b;
    double I[D][LD(D)], Z[D][LD(D)];
    struct G {
        double U[D][LD(D)], Pm[D][LD(D)], Ps[D][LD(D)] /* P^s_{k+1} - P^- */, X[D][LD(D)];
        double dm[D];
        double fqs[2][FQS(D, STREAM)];              // STREAM: (F_{k+1}, Q_{k+1}) staged with the record of k
    } g[kWWarps];
};

template <int D, bool STREAM>
__global__ void __launch_bounds__(32 * kWWarps, PSSGP_WLPR_MINB) kw_smoother_apply_lpr(const WParams p) {
    static_assert(D <= kGL, "lane-per-row RTS holds one row per lane");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K5LSmem<D, STREAM>& shl = *reinterpret_cast<K5LSmem<D, STREAM>*>(smem_raw);
    K5Smem<D>& sh = shl.b;
    load_model<D>(sh.m, p.model);
    for (int e = threadIdx.x; e < D * D; e += blockDim.x) {
        const int i = e / D, j = e - (e / D) * D;
        shl.I[i][j] = (i == j) ? 1.0 : 0.0;
        shl.Z[i][j] = 0.0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = blockIdx.x * kWWarps + wid;
    // NLL: fixed-order sum of the chain partials (CTA 0, warp 0) — as kw_smoother_apply
    if (blockIdx.x == 0 && wid == 0 && p.nll_out) {
        double s = 0.0;
        const int per = (p.nch + 31) / 32;
        for (int i = 0; i < per; ++i) {
            const int q = lane * per + i;
            if (q < p.nch) s += p.nll_chain[q];
        }
        for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
        if (lane == 0) *p.nll_out = s;
    }
    if (c >= p.nch) return;
    auto& W = sh.w[wid];
    auto& Gs = shl.g[wid];
    const SModel<D>& M = sh.m;
    // ---- carry (warp-cooperative, shared layout): collapsed suffix after the chain
    for (int e = lane; e < D * D; e += 32) W.Ps[e / D][e % D] = 0.0;
    for (int i = lane; i < D; i += 32) W.ms[i] = 0.0;
    __syncwarp();
    for (int g = p.world - 1; g > p.rank && p.in_smooth; --g) {
        gload<D>(W.u.c.a, p.in_smooth + static_cast<int64_t>(g) * (SNW(D) + 1), lane);   // blob = aggregate + NLL partial
        wapply_suffix<D>(W.u.c.a, W.ms, W.Ps, W.u.c.s, lane);
    }
    if (c + 1 < p.nch) {
        gload<D>(W.u.c.a, p.sagg + static_cast<int64_t>(c + 1) * SNW(D), lane);
        wapply_suffix<D>(W.u.c.a, W.ms, W.Ps, W.u.c.s, lane);
    }
    const bool act = lane < D;
    const int r = act ? lane : 0;
    double Psr[D], msr = W.ms[r];
#pragma unroll
    for (int j = 0; j < D; ++j) Psr[j] = W.Ps[r][j];
    const double hr = act ? M.H[r] : 0.0;
    __syncwarp();                                   // W.u (carry scratch) is reused by the staging below

    const int64_t kb = static_cast<int64_t>(c) * p.K;
    const int64_t ke = min(kb + p.K, p.n);
    const double* xpc = p.xp + static_cast<int64_t>(c) * p.K * CNW(D);
    double tnext = (ke > kb && p.k0 + ke < p.nglob) ? __ldg(p.t + ke) : 0.0;
    double tk_next = 0.0;
    if (ke > kb) {
        const double* src = xpc + (ke - 1 - kb) * CNW(D);
        for (int i = lane; i < CNW(D); i += 32) cp_async8(&W.xst[0][i], src + i, 8);
        if (STREAM && p.k0 + ke < p.nglob) {       // F, Q of the transition out of ke - 1 (record ke)
            const double* fsrc = p.fq + ke * FQW(D);
            for (int i = lane; i < FQW(D); i += 32) cp_async8(&Gs.fqs[0][i], fsrc + i, 8);
        }
        cp_async_commit();
        tk_next = __ldg(p.t + ke - 1);
    }
    int sb = 0;
    bool bad = false;
    for (int64_t k = ke - 1; k >= kb; --k) {
        const double tk = tk_next;
        const int64_t g = p.k0 + k;
        cp_async_wait<0>();
        __syncwarp();
        if (k > kb) {
            const double* src = xpc + (k - 1 - kb) * CNW(D);
            for (int i = lane; i < CNW(D); i += 32) cp_async8(&W.xst[sb ^ 1][i], src + i, 8);
            if (STREAM) {                           // record k: the transition out of k - 1
                const double* fsrc = p.fq + k * FQW(D);
                for (int i = lane; i < FQW(D); i += 32) cp_async8(&Gs.fqs[sb ^ 1][i], fsrc + i, 8);
            }
            cp_async_commit();
            tk_next = __ldg(p.t + k - 1);
        }
        const int fb = sb;
        // filtered (xbar_k, row r of P_k) from the staged packed record
        double xa[D], Pr[D];
        {
            const double* src = W.xst[sb];
#pragma unroll
            for (int i = 0; i < D; ++i) xa[i] = src[i];
#pragma unroll
            for (int j = 0; j < D; ++j) Pr[j] = src[D + si(D, r, j)];
        }
        sb ^= 1;
        if (g == p.nglob - 1) {                     // terminal element: smoothed = filtered
#pragma unroll
            for (int j = 0; j < D; ++j) Psr[j] = Pr[j];
            msr = xa[r];
        } else {
            const int kind = wdisc_kind(tnext - tk, M.udt, STREAM);
            const double* Fp;
            const double* Qp;
            if (kind == 0) {
                if (STREAM) { Fp = &Gs.fqs[fb][0]; Qp = Fp + D * LD(D); }
                else { Fp = &M.F[0][0]; Qp = &M.Q[0][0]; }
            } else {                                // dt == 0 (or unsupported, reported by the fold): F = I, Q = 0
                Fp = &shl.I[0][0]; Qp = &shl.Z[0][0];
            }
            // column r of F P (P symmetric: column r = row r); xm_r = F[r,:] xbar
            double Uc[D], xm = 0.0;
#pragma unroll
            for (int i = 0; i < D; ++i) {
                double su = 0.0;
#pragma unroll
                for (int q = 0; q < D; ++q) su = fma(Fp[i * LD(D) + q], Pr[q], su);
                Uc[i] = su;
            }
#pragma unroll
            for (int q = 0; q < D; ++q) xm = fma(Fp[r * LD(D) + q], xa[q], xm);
            if (act) {
#pragma unroll
                for (int i = 0; i < D; ++i) Gs.U[i][r] = Uc[i];
            }
            __syncwarp();
            // row r of P^- = (F P)[r,:] F^T + Q[r,:]
            double Ur[D];
#pragma unroll
            for (int q = 0; q < D; ++q) Ur[q] = Gs.U[r][q];
            if (act) {
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    double s2 = Qp[r * LD(D) + j];
#pragma unroll
                    for (int q = 0; q < D; ++q) s2 = fma(Ur[q], Fp[j * LD(D) + q], s2);
                    Gs.Pm[r][j] = s2;
                    Gs.Ps[r][j] = Psr[j] - s2;          // Delta = P^s_{k+1} - P^- (row r)
                }
                Gs.dm[r] = msr - xm;
            }
            __syncwarp();
            // Cholesky of P^- (upper triangle) in every lane: L lower, Li = 1 / L_jj
            double L[D][D], Li[D];
#pragma unroll
            for (int j = 0; j < D; ++j) {
                double sd = Gs.Pm[j][j];
#pragma unroll
                for (int q = 0; q < j; ++q) sd = fma(-L[j][q], L[j][q], sd);
                bad = bad || !(sd > 0.0);
                Li[j] = rsqrt(sd);
#pragma unroll
                for (int i = j + 1; i < D; ++i) {
                    double so = Gs.Pm[j][i];
#pragma unroll
                    for (int q = 0; q < j; ++q) so = fma(-L[i][q], L[j][q], so);
                    L[i][j] = so * Li[j];
                }
                L[j][j] = sd * Li[j];
            }
            // column r of X = P^-^{-1} (F P)
            double Xc[D];
#pragma unroll
            for (int i = 0; i < D; ++i) {
                double z = Uc[i];
#pragma unroll
                for (int q = 0; q < i; ++q) z = fma(-L[i][q], Xc[q], z);
                Xc[i] = z * Li[i];
            }
#pragma unroll
            for (int i = D - 1; i >= 0; --i) {
                double z = Xc[i];
#pragma unroll
                for (int q = i + 1; q < D; ++q) z = fma(-L[q][i], Xc[q], z);
                Xc[i] = z * Li[i];
            }
            // m^s_r = xbar_r + X[:,r] . (m^s_{k+1} - xm);  V = X[:,r]^T (P^s_{k+1} - P^-) (upper triangles)
            double ms_new = xa[r], V[D];
#pragma unroll
            for (int q = 0; q < D; ++q) ms_new = fma(Xc[q], Gs.dm[q], ms_new);
#pragma unroll
            for (int bb = 0; bb < D; ++bb) {
                double v = 0.0;
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    const int lo = a < bb ? a : bb, hi = a < bb ? bb : a;
                    v = fma(Xc[a], Gs.Ps[lo][hi], v);
                }
                V[bb] = v;
            }
            if (act) {
#pragma unroll
                for (int i = 0; i < D; ++i) Gs.X[i][r] = Xc[i];
            }
            __syncwarp();
            // row r of P^s_k = P[r,:] + V X
#pragma unroll
            for (int j = 0; j < D; ++j) {
                double s2 = Pr[j];
#pragma unroll
                for (int bb = 0; bb < D; ++bb) s2 = fma(V[bb], Gs.X[bb][j], s2);
                Psr[j] = s2;
            }
            msr = ms_new;
            __syncwarp();                           // Gs buffers are rewritten by the next step
        }
        tnext = tk;
        // projection mean = H m^s, var = H P^s H^T (rows summed over the lanes)
        double mo = hr * msr, vo = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) vo = fma(Psr[j], M.H[j], vo);
        vo *= hr;
#pragma unroll
        for (int off = kGL / 2; off > 0; off >>= 1) {
            mo += __shfl_xor_sync(0xffffffffu, mo, off);
            vo += __shfl_xor_sync(0xffffffffu, vo, off);
        }
        if (lane == 0) {
            if (p.mean) p.mean[k] = mo;
            if (p.var) p.var[k] = vo;
        }
    }
    if (bad && lane == 0) raise_error(p.err, p.k0 + kb, kErrNumeric);
}


// ================================================================== quarter-parallel rescans (D <= 8)
// The fold (kw_filter_fold_lpr) splits every chain into kQ = 4 quarters [qb, qe) (the split below,
// identical in all three kernels) and stores the quarter PREFIX aggregates q0, q0 (x) q1,
// q0 (x) q1 (x) q2 (p.qagg).  The rescans then run the four quarters of a chain at once, one per
// 8-lane group (lane r of a group owns row r of every matrix, as in the lane-per-row kernels),
// from per-quarter carries: the filtered state entering quarter q is the chain carry applied to
// the prefix aggregate of quarters < q (any grouping of the scan), and the
// smoothed state after quarter q is the chain's suffix carry applied through the smoother
// aggregates of the later quarters.  All four groups of a warp are busy (the
// lane-per-row rescans kept one group busy per chain).
__device__ __forceinline__ void quarter_bounds(int64_t kb, int64_t ke, int64_t K, int q, int64_t& qb, int64_t& qe,
                                               int np = kQ) {
    const int64_t Kq = (K + np - 1) / np;
    qb = min(kb + q * Kq, ke);
    qe = min(qb + Kq, ke);
}

// scratch of a quarter smoother aggregate (the k3w_chain_sagg computation on explicit operands)
template <int D>
struct SQScratch {
    double FP[D][LD(D)], Sm[D][LD(D)], Pm[D][LD(D)], W2[D][2 * D + 1];
    double xm[D];
};

// (E, g, L) of the quarter [qb, qe) from its moments at the quarter's last step: filtered (x, P),
// cross-covariance Sg = Cov(x_qb, x_{qe-1} | y_1:qe-1), entry moments (x0, P0) = E / Cov(x_qb | y_1:qe-1)
// (DESIGN.md §5 "chain smoother aggregates", reading N1), tprev = t[qe - 1].  Warp-cooperative.
template <int D>
__device__ void quarter_sagg(const WParams& p, const SModel<D>& M, const double (*P)[LD(D)], const double* x,
                             const double (*Sg)[LD(D)], const double (*P0)[LD(D)], const double* x0, int64_t qb,
                             int64_t qe, double tprev, SS<D>& out, SQScratch<D>& w, int lane) {
    if (qe <= qb) {
        set_identity<D>(out, lane);
        return;
    }
    if (p.k0 + qe == p.nglob) {                  // terminal element inside: (0, m^s_qb, P^s_qb) = (0, x0, P0)
        for (int e = lane; e < D * D; e += 32) {
            const int i = e / D, j = e - (e / D) * D;
            out.E[i][j] = 0.0;
            out.L[i][j] = P0[i][j];
        }
        for (int i = lane; i < D; i += 32) out.g[i] = x0[i];
        __syncwarp();
        return;
    }
    const double tn = __ldg(p.t + qe);
    const int kind = wdisc_kind(tn - tprev, M.udt, p.fq != nullptr);
    const FQp<D> fqp = wfq<D>(p, M, qe);
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        double fp = 0.0, sm = 0.0;
        if (kind == 0) {
            for (int q = 0; q < D; ++q) {
                fp = fma(fqp.F[i][q], P[q][j], fp);
                sm = fma(Sg[i][q], fqp.F[j][q], sm);
            }
        } else {
            fp = P[i][j];
            sm = Sg[i][j];
        }
        w.FP[i][j] = fp;
        w.Sm[i][j] = sm;
    }
    for (int i = lane; i < D; i += 32) {
        double s2 = 0.0;
        if (kind == 0)
            for (int q = 0; q < D; ++q) s2 = fma(fqp.F[i][q], x[q], s2);
        else
            s2 = x[i];
        w.xm[i] = s2;
    }
    __syncwarp();
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        double s2 = (kind == 0) ? fqp.Q[i][j] : 0.0;
        if (kind == 0)
            for (int q = 0; q < D; ++q) s2 = fma(w.FP[i][q], fqp.F[j][q], s2);
        else
            s2 = w.FP[i][j];
        w.Pm[i][j] = s2;
    }
    __syncwarp();
    for (int e = lane; e < D * D; e += 32) w.FP[e / D][e % D] = w.Pm[e / D][e % D];
    __syncwarp();
    if (!winverse<D>(w.FP, w.W2, lane) && lane == 0) raise_error(p.err, p.k0 + qe, kErrNumeric);
    wmm<D>(out.E, w.Sm, w.FP, nullptr, lane);           // E = Sm Pm^-1
    __syncwarp();
    for (int i = lane; i < D; i += 32) {
        double a = x0[i];
        for (int q = 0; q < D; ++q) a = fma(-out.E[i][q], w.xm[q], a);
        out.g[i] = a;
    }
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        double a = P0[i][j];
        for (int q = 0; q < D; ++q) a = fma(-out.E[i][q], w.Sm[j][q], a);
        w.Pm[i][j] = a;
    }
    __syncwarp();
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        out.L[i][j] = 0.5 * (w.Pm[i][j] + w.Pm[j][i]);
    }
    __syncwarp();
}

// ------------------------------------------------------------------ K3q: quarter-parallel Kalman rescan
template <int D>
struct QAgPhase {                                  // one quarter's moments and the running aggregate
    double P[D][LD(D)], Sg[D][LD(D)], P0[D][LD(D)];
    double x[D], x0[D];
    SS<D> acc, cur;
    union {                                        // used one after the other
        SQScratch<D> w;
        SCombF<D> s;
    };
};
template <int D, bool STREAM, int G = kGL, int WPC = kWWarps>
struct K3QSmem {
    static constexpr int NP = 32 / G;
    SModel<D> m;
    double I[D][LD(D)], Z[D][LD(D)];
    struct PerWarp {
        union {
            struct {                               // carry phase (the carries are read once, before the
                double cx[NP][D];                  // step phase reuses the space): filtered state
                double cP[NP][D][LD(D)];           // entering each quarter
                SF<D> a;
                SCombF<D> s;
            } c;
            struct {                               // step phase, one slot per group
                double U[NP][D][LD(D)];
                double fqs[NP][2][FQS(D, STREAM)];
            } st;
            // quarter smoother aggregates, one quarter at a time (8-lane groups; the half-chain kernel
            // hands its moments to kw_part_sagg instead)
            std::conditional_t<(G == kGL), QAgPhase<D>, char> ag;
        } u;
    } w[WPC];
};

template <int D, bool STREAM, int G = kGL, int WPC = kWWarps, int FB = D>
__global__ void __launch_bounds__(32 * WPC, lpr_minb(G)) kw_filter_apply_q(const WParams p) {
    static_assert(D <= G, "one row per lane of a G-lane group");
    constexpr int NP = 32 / G;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K3QSmem<D, STREAM, G, WPC>& sh = *reinterpret_cast<K3QSmem<D, STREAM, G, WPC>*>(smem_raw);
    load_model<D>(sh.m, p.model);
    for (int e = threadIdx.x; e < D * D; e += blockDim.x) {
        const int i = e / D, j = e - (e / D) * D;
        sh.I[i][j] = (i == j) ? 1.0 : 0.0;
        sh.Z[i][j] = 0.0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = blockIdx.x * WPC + wid;
    if (c >= p.nch) return;                                     // warp-uniform
    auto& W = sh.w[wid];
    const SModel<D>& M = sh.m;
    const int64_t kb = static_cast<int64_t>(c) * p.K;
    const int64_t ke = min(kb + p.K, p.n);
    // ---- carries: the chain's (incoming sharded (x) scanned chains < c), then through the quarter
    // prefix aggregates of the fold
    for (int e = lane; e < D * D; e += 32) W.u.c.cP[0][e / D][e % D] = 0.0;
    for (int i = lane; i < D; i += 32) W.u.c.cx[0][i] = 0.0;
    __syncwarp();
    bool ok = true;
    for (int g = 0; g < p.rank && p.in_filt; ++g) {
        gload<D>(W.u.c.a, p.in_filt + static_cast<int64_t>(g) * FNW(D), lane);
        ok = wapply_prefix<D>(W.u.c.cx[0], W.u.c.cP[0], W.u.c.a, W.u.c.s, lane) && ok;
    }
    if (c > 0) {
        gload<D>(W.u.c.a, p.fagg + static_cast<int64_t>(c - 1) * FNW(D), lane);
        ok = wapply_prefix<D>(W.u.c.cx[0], W.u.c.cP[0], W.u.c.a, W.u.c.s, lane) && ok;
    }
    for (int q = 1; q < NP; ++q) {
        for (int e = lane; e < D * D; e += 32) W.u.c.cP[q][e / D][e % D] = W.u.c.cP[0][e / D][e % D];
        for (int i = lane; i < D; i += 32) W.u.c.cx[q][i] = W.u.c.cx[0][i];
        __syncwarp();
        gload<D>(W.u.c.a, p.qagg + (static_cast<int64_t>(c) * (NP - 1) + (q - 1)) * FNW(D), lane);
        ok = wapply_prefix<D>(W.u.c.cx[q], W.u.c.cP[q], W.u.c.a, W.u.c.s, lane) && ok;
    }
    if (!ok && lane == 0) raise_error(p.err, p.k0 + kb, kErrNumeric);

    // ---- the four quarters, one per 8-lane group, in registers
    const int q = lane / G, r0 = lane % G, gb = q * G;
    const unsigned gm = group_mask(G, gb);
    const bool act = (D == G) || r0 < D;                      // compile-time true when the group is full
    const int r = act ? r0 : 0;
    int64_t qb, qe;
    quarter_bounds(kb, ke, p.K, q, qb, qe, NP);
    double Pr[D], Sgr[D], P0r[D], xr = W.u.c.cx[q][r], x0r = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) { Pr[j] = W.u.c.cP[q][r][j]; Sgr[j] = 0.0; P0r[j] = 0.0; }
    const double hr = act ? M.H[r] : 0.0;
    __syncwarp();                                               // W.u is reused by the step phase
    double tprev = (qb < qe && (qb > 0 || p.k0 > 0)) ? __ldg(p.t + qb - 1) : 0.0;
    double quad = 0.0, logs = 0.0;
    int nobs = 0;
    bool bad_s = false;
    int64_t bad_g = 0;
    double* xpc = p.xp + static_cast<int64_t>(c) * p.K * CNW(D);
    double tn_ = 0.0, yn_ = 0.0;
    unsigned char mn_ = 0;
    if (qb < qe) { tn_ = __ldg(p.t + qb); mn_ = __ldg(p.mask + qb); yn_ = __ldg(p.y + qb); }
    auto& U = W.u.st.U[q];
    auto& fqs = W.u.st.fqs[q];
    if (STREAM) {
        if (qb < qe)
            for (int i = r0; i < FQW(D); i += G) cp_async8(&fqs[0][i], p.fq + qb * FQW(D) + i, 8);
        cp_async_commit();
    }
    for (int64_t k = qb; k < qe; ++k) {
        const int fb = static_cast<int>((k - qb) & 1);
        if (STREAM) {
            // slot fb holds (F_k, Q_k); slot fb^1 was last read in step k - 1, before its closing sync
            cp_async_wait<0>();
            __syncwarp(gm);
            if (k + 1 < qe)
                for (int i = r0; i < FQW(D); i += G) cp_async8(&fqs[fb ^ 1][i], p.fq + (k + 1) * FQW(D) + i, 8);
            cp_async_commit();
        }
        const double tk = tn_;
        const bool obs = mn_ != 0;
        const double yk = obs ? yn_ : 0.0;
        if (k + 1 < qe) { tn_ = __ldg(p.t + k + 1); mn_ = __ldg(p.mask + k + 1); yn_ = __ldg(p.y + k + 1); }
        const int64_t g = p.k0 + k;
        const int kind = (g == 0) ? 3 : wdisc_kind(tk - tprev, M.udt, STREAM);
        const bool first = (k == qb);
        tprev = tk;
        const double* Fp;
        const double* Qp;
        if (kind == 0) {
            if (STREAM) { Fp = &fqs[fb][0]; Qp = Fp + D * LD(D); }
            else { Fp = &M.F[0][0]; Qp = &M.Q[0][0]; }
        } else if (kind == 1) {
            Fp = &sh.I[0][0]; Qp = &sh.Z[0][0];
        } else {                                     // 3 (and 2, reported by the fold): F = 0, Q = P_inf
            Fp = &sh.Z[0][0]; Qp = &M.Pinf[0][0];
        }
        // column r of F P, xm_r = F[r,:] x, row r of Sm = Sg[r,:] F^T
        double Uc[D], xm = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double su = 0.0;
#pragma unroll
            for (int qq = fblo(i, FB); qq < fbhi(i, FB, D); ++qq) su = fma(Fp[i * LD(D) + qq], Pr[qq], su);
            Uc[i] = su;
        }
#pragma unroll
        for (int qq = 0; qq < D; ++qq) xm = fma(Fp[r * LD(D) + qq], __shfl_sync(gm, xr, qq, G), xm);
        if (act) {
#pragma unroll
            for (int i = 0; i < D; ++i) U[i][r] = Uc[i];
        }
        __syncwarp(gm);
        double Pm[D], Sm[D], HP = 0.0, SH = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            double s2 = Qp[r * LD(D) + j], s3 = 0.0;
#pragma unroll
            for (int qq = fblo(j, FB); qq < fbhi(j, FB, D); ++qq) {
                const double f = Fp[j * LD(D) + qq];
                s2 = fma(U[r][qq], f, s2);
                s3 = fma(Sgr[qq], f, s3);
            }
            Pm[j] = s2;
            Sm[j] = s3;
            HP = fma(s2, M.H[j], HP);
            SH = fma(s3, M.H[j], SH);
        }
        __syncwarp(gm);                               // U is rewritten by the next step
        if (!act) { HP = 0.0; SH = 0.0; }
        double S = hr * HP, hx = hr * xm;
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) {
            S += __shfl_xor_sync(gm, S, off);
            hx += __shfl_xor_sync(gm, hx, off);
        }
        S += M.r;
        if (obs && !(S > 0.0 && S < INFINITY) && !bad_s) { bad_s = true; bad_g = g; }
        const double iS = obs ? 1.0 / S : 0.0;
        const double v = obs ? (yk - hx) : 0.0;
        const double vs = v * iS;
        const double HPs = HP * iS, SHs = SH * iS;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const double HPj = __shfl_sync(gm, HP, j, G);
            const double SHj = __shfl_sync(gm, SH, j, G);
            const double Pn = fma(-HPs, HPj, Pm[j]);
            Pr[j] = Pn;
            if (first) {
                P0r[j] = Pn;
                Sgr[j] = Pn;
            } else {
                Sgr[j] = fma(-SHs, HPj, Sm[j]);
                P0r[j] = fma(-SHs, SHj, P0r[j]);
            }
        }
        xr = fma(HP, vs, xm);
        x0r = first ? xr : fma(SH, vs, x0r);
        if (obs) {
            quad = fma(v, vs, quad);
            logs += log(S);
            ++nobs;
        }
        if (p.store_state && act) {
            double* o = xpc + (k - kb) * CNW(D);
            o[r] = xr;
#pragma unroll
            for (int j = 0; j < D; ++j)
                if (j >= r) o[D + si(D, r, j)] = Pr[j];
        }
    }
    __syncwarp();
    if (bad_s && r0 == 0) raise_error(p.err, bad_g, kErrNumeric);
    // NLL partial of the chain: the four groups' sums (identical in every lane of a group) in order
    {
        double nl = nobs ? 0.5 * (quad + logs + nobs * 1.8378770664093453) : 0.0;
        double tot = 0.0;
#pragma unroll
        for (int qq = 0; qq < NP; ++qq) tot += __shfl_sync(0xffffffffu, nl, qq * G);
        if (lane == 0) p.nll_chain[c] = tot;
    }
    if (!p.store_state) return;
    if constexpr (G > kGL) {
        // half chains: each group's end moments to global memory (kw_part_sagg forms the half smoother
        // aggregates and the chain's), keeping this kernel's shared memory small
        if (act) {
            double* o = p.qmom + (static_cast<int64_t>(c) * NP + q) * QMW(D);
#pragma unroll
            for (int j = 0; j < D; ++j) {
                o[r * D + j] = Pr[j];
                o[D * D + r * D + j] = Sgr[j];
                o[2 * D * D + r * D + j] = P0r[j];
            }
            o[3 * D * D + r] = xr;
            o[3 * D * D + D + r] = x0r;
        }
    } else {
    // ---- quarter smoother aggregates (E, g, L), combined in time order into the chain's
    const double tq = tprev;
    SS<D>* acc = &W.u.ag.acc;
    SS<D>* cur = &W.u.ag.cur;
#pragma unroll 1
    for (int qq = 0; qq < NP; ++qq) {
        if (q == qq && act) {
#pragma unroll
            for (int j = 0; j < D; ++j) {
                W.u.ag.P[r][j] = Pr[j];
                W.u.ag.Sg[r][j] = Sgr[j];
                W.u.ag.P0[r][j] = P0r[j];
            }
            W.u.ag.x[r] = xr;
            W.u.ag.x0[r] = x0r;
        }
        __syncwarp();
        int64_t sb, se;
        quarter_bounds(kb, ke, p.K, qq, sb, se, NP);
        const double tpq = __shfl_sync(0xffffffffu, tq, qq * G);
        quarter_sagg<D>(p, M, W.u.ag.P, W.u.ag.x, W.u.ag.Sg, W.u.ag.P0, W.u.ag.x0, sb, se, tpq, *cur, W.u.ag.w, lane);
        if (qq > 0) {
            gstore<D>(*cur, p.sqagg + (static_cast<int64_t>(c) * (NP - 1) + (qq - 1)) * SNW(D), lane);
            __syncwarp();
            wcombine<D>(*acc, *cur, *cur, W.u.ag.s, lane);   // acc (x) cur, earlier quarter on the left
        }
        SS<D>* t = acc; acc = cur; cur = t;
        __syncwarp();
    }
    gstore<D>(*acc, p.sagg + static_cast<int64_t>(c) * SNW(D), lane);
    }
}

// The half smoother aggregates and the chain's from the half-chain rescan's end moments (p.qmom):
// the quarter-aggregate phase of kw_filter_apply_q for 16-lane groups, one warp per chain.
template <int D, int NP>
__global__ void __launch_bounds__(32) kw_part_sagg(const WParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    QAgPhase<D>& A = *reinterpret_cast<QAgPhase<D>*>(smem_raw);
    __shared__ SModel<D> M;
    load_model<D>(M, p.model);
    __syncwarp();
    const int lane = threadIdx.x, c = blockIdx.x;
    const int64_t kb = static_cast<int64_t>(c) * p.K;
    const int64_t ke = min(kb + p.K, p.n);
    SS<D>* acc = &A.acc;
    SS<D>* cur = &A.cur;
#pragma unroll 1
    for (int qq = 0; qq < NP; ++qq) {
        const double* o = p.qmom + (static_cast<int64_t>(c) * NP + qq) * QMW(D);
        for (int e = lane; e < D * D; e += 32) {
            const int i = e / D, j = e - (e / D) * D;
            A.P[i][j] = o[e];
            A.Sg[i][j] = o[D * D + e];
            A.P0[i][j] = o[2 * D * D + e];
        }
        for (int i = lane; i < D; i += 32) {
            A.x[i] = o[3 * D * D + i];
            A.x0[i] = o[3 * D * D + D + i];
        }
        __syncwarp();
        int64_t sb, se;
        quarter_bounds(kb, ke, p.K, qq, sb, se, NP);
        const double tpq = (se > sb) ? __ldg(p.t + se - 1) : 0.0;
        quarter_sagg<D>(p, M, A.P, A.x, A.Sg, A.P0, A.x0, sb, se, tpq, *cur, A.w, lane);
        if (qq > 0) {
            gstore<D>(*cur, p.sqagg + (static_cast<int64_t>(c) * (NP - 1) + (qq - 1)) * SNW(D), lane);
            __syncwarp();
            wcombine<D>(*acc, *cur, *cur, A.s, lane);
        }
        SS<D>* t = acc; acc = cur; cur = t;
        __syncwarp();
    }
    gstore<D>(*acc, p.sagg + static_cast<int64_t>(c) * SNW(D), lane);
}

// ------------------------------------------------------------------ K5q: quarter-parallel RTS rescan
template <int D, bool STREAM, int G = kGL, int WPC = kWWarps>
struct K5QSmem {
    static constexpr int NP = 32 / G;
    SModel<D> m;
    double I[D][LD(D)], Z[D][LD(D)];
    struct PerWarp {
        union {
            struct {                               // carry phase (read once before the step phase)
                double cm[NP][D];                  // smoothed state after each quarter
                double cP[NP][D][LD(D)];
                SS<D> a;
                SSufScratch<D> s;
            } c;
            struct Grp {                           // step phase, one slot per group
                double xst[2][CNW(D)];             // staged packed (xbar, P) records (cp.async)
                double U[D][LD(D)], Pm[D][LD(D)], Ps[D][LD(D)] /* P^s_{k+1} - P^- */, X[D][LD(D)];
                double dm[D];
                double fqs[2][FQS(D, STREAM)];     // STREAM: (F_{k+1}, Q_{k+1}) staged with record k
            } g[NP];
        } u;
    } w[WPC];
};

template <int D, bool STREAM, int G = kGL, int WPC = kWWarps, int FB = D>
__global__ void __launch_bounds__(32 * WPC, lpr_minb(G)) kw_smoother_apply_q(const WParams p) {
    static_assert(D <= G, "one row per lane of a G-lane group");
    constexpr int NP = 32 / G;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K5QSmem<D, STREAM, G, WPC>& sh = *reinterpret_cast<K5QSmem<D, STREAM, G, WPC>*>(smem_raw);
    load_model<D>(sh.m, p.model);
    for (int e = threadIdx.x; e < D * D; e += blockDim.x) {
        const int i = e / D, j = e - (e / D) * D;
        sh.I[i][j] = (i == j) ? 1.0 : 0.0;
        sh.Z[i][j] = 0.0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = blockIdx.x * WPC + wid;
    if (c >= p.nch) return;
    auto& W = sh.w[wid];
    const SModel<D>& M = sh.m;
    const int64_t kb = static_cast<int64_t>(c) * p.K;
    const int64_t ke = min(kb + p.K, p.n);
    // ---- carries: collapsed suffix after the chain (incoming sharded, scanned chains > c), then
    // back through the smoother aggregates of quarters 3, 2, 1 (kw_filter_apply_q)
    auto& c3P = W.u.c.cP[NP - 1];
    for (int e = lane; e < D * D; e += 32) c3P[e / D][e % D] = 0.0;
    for (int i = lane; i < D; i += 32) W.u.c.cm[NP - 1][i] = 0.0;
    __syncwarp();
    for (int g = p.world - 1; g > p.rank && p.in_smooth; --g) {
        gload<D>(W.u.c.a, p.in_smooth + static_cast<int64_t>(g) * (SNW(D) + 1), lane);   // blob = aggregate + NLL partial
        wapply_suffix<D>(W.u.c.a, W.u.c.cm[NP - 1], c3P, W.u.c.s, lane);
    }
    if (c + 1 < p.nch) {
        gload<D>(W.u.c.a, p.sagg + static_cast<int64_t>(c + 1) * SNW(D), lane);
        wapply_suffix<D>(W.u.c.a, W.u.c.cm[NP - 1], c3P, W.u.c.s, lane);
    }
    for (int q = NP - 2; q >= 0; --q) {
        for (int e = lane; e < D * D; e += 32) W.u.c.cP[q][e / D][e % D] = W.u.c.cP[q + 1][e / D][e % D];
        for (int i = lane; i < D; i += 32) W.u.c.cm[q][i] = W.u.c.cm[q + 1][i];
        __syncwarp();
        gload<D>(W.u.c.a, p.sqagg + (static_cast<int64_t>(c) * (NP - 1) + q) * SNW(D), lane);   // quarter q + 1
        wapply_suffix<D>(W.u.c.a, W.u.c.cm[q], W.u.c.cP[q], W.u.c.s, lane);
    }
    const int q = lane / G, r0 = lane % G, gb = q * G;
    const unsigned gm = group_mask(G, gb);
    const bool act = (D == G) || r0 < D;                      // compile-time true when the group is full
    const int r = act ? r0 : 0;
    int64_t qb, qe;
    quarter_bounds(kb, ke, p.K, q, qb, qe, NP);
    double Psr[D], msr = W.u.c.cm[q][r];
#pragma unroll
    for (int j = 0; j < D; ++j) Psr[j] = W.u.c.cP[q][r][j];
    const double hr = act ? M.H[r] : 0.0;
    __syncwarp();                                   // W.u (carry scratch) is reused by the staging below
    auto& Gs = W.u.g[q];
    const double* xpc = p.xp + static_cast<int64_t>(c) * p.K * CNW(D);
    double tnext = (qe > qb && p.k0 + qe < p.nglob) ? __ldg(p.t + qe) : 0.0;
    double tk_next = 0.0;
    if (qe > qb) {
        const double* src = xpc + (qe - 1 - kb) * CNW(D);
        for (int i = r0; i < CNW(D); i += G) cp_async8(&Gs.xst[0][i], src + i, 8);
        if (STREAM && p.k0 + qe < p.nglob) {        // F, Q of the transition out of qe - 1 (record qe)
            const double* fsrc = p.fq + qe * FQW(D);
            for (int i = r0; i < FQW(D); i += G) cp_async8(&Gs.fqs[0][i], fsrc + i, 8);
        }
        cp_async_commit();
        tk_next = __ldg(p.t + qe - 1);
    }
    int sb = 0;
    bool bad = false;
    for (int64_t k = qe - 1; k >= qb; --k) {
        const double tk = tk_next;
        const int64_t g = p.k0 + k;
        cp_async_wait<0>();
        __syncwarp(gm);
        if (k > qb) {
            const double* src = xpc + (k - 1 - kb) * CNW(D);
            for (int i = r0; i < CNW(D); i += G) cp_async8(&Gs.xst[sb ^ 1][i], src + i, 8);
            if (STREAM) {                           // record k: the transition out of k - 1
                const double* fsrc = p.fq + k * FQW(D);
                for (int i = r0; i < FQW(D); i += G) cp_async8(&Gs.fqs[sb ^ 1][i], fsrc + i, 8);
            }
            cp_async_commit();
            tk_next = __ldg(p.t + k - 1);
        }
        const int fb = sb;
        // this step's filtered (xbar_k, row r of P_k): registers for 8-lane groups, read from the staged
        // record on use for 16-lane groups (register budget of d = 16)
        const double* rec = Gs.xst[sb];
        double xa_r[G == kGL ? D : 1], Pr_r[G == kGL ? D : 1];
        if constexpr (G == kGL) {
#pragma unroll
            for (int i = 0; i < D; ++i) xa_r[i] = rec[i];
#pragma unroll
            for (int j = 0; j < D; ++j) Pr_r[j] = rec[D + si(D, r, j)];
        }
        auto XA = [&](int i) -> double {
            if constexpr (G == kGL) return xa_r[i];
            else return rec[i];
        };
        auto PR = [&](int j) -> double {
            if constexpr (G == kGL) return Pr_r[j];
            else return rec[D + si(D, r, j)];
        };
        sb ^= 1;
        if (g == p.nglob - 1) {                     // terminal element: smoothed = filtered
#pragma unroll
            for (int j = 0; j < D; ++j) Psr[j] = PR(j);
            msr = XA(r);
        } else {
            const int kind = wdisc_kind(tnext - tk, M.udt, STREAM);
            const double* Fp;
            const double* Qp;
            if (kind == 0) {
                if (STREAM) { Fp = &Gs.fqs[fb][0]; Qp = Fp + D * LD(D); }
                else { Fp = &M.F[0][0]; Qp = &M.Q[0][0]; }
            } else {                                // dt == 0 (or unsupported, reported by the fold): F = I, Q = 0
                Fp = &sh.I[0][0]; Qp = &sh.Z[0][0];
            }
            double Uc[D], xm = 0.0;
#pragma unroll
            for (int i = 0; i < D; ++i) {
                double su = 0.0;
#pragma unroll
                for (int qq = fblo(i, FB); qq < fbhi(i, FB, D); ++qq) su = fma(Fp[i * LD(D) + qq], PR(qq), su);
                Uc[i] = su;
            }
#pragma unroll
            for (int qq = 0; qq < D; ++qq) xm = fma(Fp[r * LD(D) + qq], XA(qq), xm);
            if (act) {
#pragma unroll
                for (int i = 0; i < D; ++i) Gs.U[i][r] = Uc[i];
            }
            __syncwarp(gm);
            double Ur[D];
#pragma unroll
            for (int qq = 0; qq < D; ++qq) Ur[qq] = Gs.U[r][qq];
            if (act) {
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    double s2 = Qp[r * LD(D) + j];
#pragma unroll
                    for (int qq = fblo(j, FB); qq < fbhi(j, FB, D); ++qq) s2 = fma(Ur[qq], Fp[j * LD(D) + qq], s2);
                    Gs.Pm[r][j] = s2;
                    Gs.Ps[r][j] = Psr[j] - s2;          // Delta = P^s_{k+1} - P^- (row r)
                }
                Gs.dm[r] = msr - xm;
            }
            __syncwarp(gm);
            // column r of X = (P^-)^-1 F P: registers for 8-lane groups, the group's shared X (column r)
            // for 16-lane groups
            double Xc[G == kGL ? D : 1];
            if constexpr (G == kGL) {
                // D <= 8: every lane factors P^- itself (L in registers)
                double L[D][D], Li[D];
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    double sd = Gs.Pm[j][j];
#pragma unroll
                    for (int qq = 0; qq < j; ++qq) sd = fma(-L[j][qq], L[j][qq], sd);
                    bad = bad || !(sd > 0.0);
                    Li[j] = rsqrt(sd);
#pragma unroll
                    for (int i = j + 1; i < D; ++i) {
                        double so = Gs.Pm[j][i];
#pragma unroll
                        for (int qq = 0; qq < j; ++qq) so = fma(-L[i][qq], L[j][qq], so);
                        L[i][j] = so * Li[j];
                    }
                    L[j][j] = sd * Li[j];
                }
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    double z = Uc[i];
#pragma unroll
                    for (int qq = 0; qq < i; ++qq) z = fma(-L[i][qq], Xc[qq], z);
                    Xc[i] = z * Li[i];
                }
#pragma unroll
                for (int i = D - 1; i >= 0; --i) {
                    double z = Xc[i];
#pragma unroll
                    for (int qq = i + 1; qq < D; ++qq) z = fma(-L[qq][i], Xc[qq], z);
                    Xc[i] = z * Li[i];
                }
            } else {
                // 9 <= D <= 16: cooperative left-looking Cholesky, lane r building row r of L in
                // registers (row j of L from lane j by shuffles, column j's pivot from lane j), then
                // L through shared memory for each lane's two triangular solves on its column
                // (the diagonal slot of the shared factor holds 1 / L_jj: the solves never read L_jj)
                double Lr[D];
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    double sv = Gs.Pm[r][j];
#pragma unroll
                    for (int qq = 0; qq < j; ++qq) sv = fma(-Lr[qq], __shfl_sync(gm, Lr[qq], j, G), sv);
                    const double sj = __shfl_sync(gm, sv, j, G);
                    bad = bad || !(sj > 0.0);
                    const double lij = rsqrt(sj);
                    Lr[j] = (r == j) ? lij : sv * lij;    // row r: L_rj (j < r), 1 / L_rr; j > r unused
                }
                auto& Lm = Gs.Pm;                    // the factor overwrites P^-: lane r read only row r
                if (act) {
#pragma unroll
                    for (int qq = 0; qq < D; ++qq) Lm[r][qq] = Lr[qq];
                }
                __syncwarp(gm);
                // the two solves on column r, in place in the shared X (U still holds F P's columns)
                if (act) {
#pragma unroll 4
                    for (int i = 0; i < D; ++i) {
                        double z = Gs.U[i][r];
                        for (int qq = 0; qq < i; ++qq) z = fma(-Lm[i][qq], Gs.X[qq][r], z);
                        Gs.X[i][r] = z * Lm[i][i];
                    }
#pragma unroll 4
                    for (int i = D - 1; i >= 0; --i) {
                        double z = Gs.X[i][r];
                        for (int qq = i + 1; qq < D; ++qq) z = fma(-Lm[qq][i], Gs.X[qq][r], z);
                        Gs.X[i][r] = z * Lm[i][i];
                    }
                }
            }
            // 16-lane groups: column r of X back from its shared slot into registers for the two
            // products below (one shared load per element instead of one per use)
            double Xr[G == kGL ? 1 : D];
            if constexpr (G > kGL) {
                __syncwarp(gm);
#pragma unroll
                for (int i = 0; i < D; ++i) Xr[i] = Gs.X[i][r];
            }
            auto XC = [&](int i) -> double {
                if constexpr (G == kGL) return Xc[i];
                else return Xr[i];
            };
            double ms_new = XA(r), V[D];
#pragma unroll
            for (int qq = 0; qq < D; ++qq) ms_new = fma(XC(qq), Gs.dm[qq], ms_new);
#pragma unroll
            for (int bb = 0; bb < D; ++bb) {
                double v = 0.0;
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    const int lo = a < bb ? a : bb, hi = a < bb ? bb : a;
                    v = fma(XC(a), Gs.Ps[lo][hi], v);
                }
                V[bb] = v;
            }
            if constexpr (G == kGL) {
                if (act) {
#pragma unroll
                    for (int i = 0; i < D; ++i) Gs.X[i][r] = Xc[i];
                }
            }
            __syncwarp(gm);
#pragma unroll
            for (int j = 0; j < D; ++j) {
                double s2 = PR(j);
#pragma unroll
                for (int bb = 0; bb < D; ++bb) s2 = fma(V[bb], Gs.X[bb][j], s2);
                Psr[j] = s2;
            }
            msr = ms_new;
            __syncwarp(gm);                         // Gs buffers are rewritten by the next step
        }
        tnext = tk;
        double mo = hr * msr, vo = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) vo = fma(Psr[j], M.H[j], vo);
        vo *= hr;
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) {
            mo += __shfl_xor_sync(gm, mo, off);
            vo += __shfl_xor_sync(gm, vo, off);
        }
        if (r0 == 0) {
            if (p.mean) p.mean[k] = mo;
            if (p.var) p.var[k] = vo;
        }
    }
    if (bad && r0 == 0) raise_error(p.err, p.k0 + qb, kErrNumeric);
}


// ------------------------------------------------------------------ K5m: RTS rescan in adjoint form
// The modified Bryson-Frazier form of the RTS recursion (an exact rewriting of supplement
// PAPER.md:422-430): with the filtered (x_k, P_k), the smoothed moments are
//   m^s_k = x_k - P_k lh_k,   P^s_k = P_k - P_k Lh_k P_k,
// where (lh, Lh) run backwards without any solve:
//   lt_k = (I - K_k h)^T lh_k - h^T v_k / S_k,   Lt_k = (I - K_k h)^T Lh_k (I - K_k h) + h^T h / S_k
//   (a missing y_k: lt = lh, Lt = Lh),   lh_{k-1} = F_k^T lt_k,   Lh_{k-1} = F_k^T Lt_k F_k,
// K_k, S_k, v_k being the Kalman gain, innovation variance and innovation of step k, recomputed
// from the filtered record of k - 1 (only P^- h^T is needed, never P^-).  Only f = h x is output, so
//   mean_k = h x_k - (P_k h^T) . lh_k,   var_k = h P_k h^T - (P_k h^T)^T Lh_k (P_k h^T)
// and a step costs O(d^2) (O(d^2 FB) for the F products of a block-diagonal F) instead of the RTS
// step's Cholesky factor, two triangular solves and congruence (O(d^3)).  The group's carry (the
// smoothed moments at its end, from the chain scan and the quarter / half smoother aggregates as in
// kw_smoother_apply_q) enters once:  lh = X^T (x^- - m^s), Lh = X^T (P^- - P^s) X with
// X = (P^-)^-1 F of the transition out of the group's last step (one cooperative Cholesky factor and
// two triangular solves per group).  Lane r of a G-lane group holds row r of Lh and lh_r.
template <int D, bool STREAM, int G = kGL, int WPC = kWWarps>
struct K5MSmem {
    static constexpr int NP = 32 / G;
    SModel<D> m;
    double I[D][LD(D)], Z[D][LD(D)];
    struct PerWarp {
        union {
            struct {                               // carry phase
                double cm[NP][D];
                double cP[NP][D][LD(D)];
                SS<D> a;
                SSufScratch<D> s;
            } c;
            struct Grp {                           // step phase, one slot per group
                double xst[3][CNW(D)];             // filtered records k, k - 1 and k - 2 (cp.async ring)
                // boundary: P^- (then L), P^- - P^s, X; in the step loop Pm holds the rows of Lt F
                // (stride D) and Ps the exchanged vectors (P h^T, P_{k-1} g, K, Lh K) - 16-byte rows
                alignas(16) double Pm[D][LD(D)];
                alignas(16) double Ps[D][LD(D)];
                double X[D][LD(D)];
                double dm[D];
                double fqs[2][FQS(D, STREAM)];     // STREAM: (F_k, Q_k) of the transition into k
            } g[NP];
        } u;
    } w[WPC];
};

// sum_j a(j) b(j) with four interleaved accumulators (a dependent FMA chain of D / 4)
template <int N, typename FA, typename FB2>
__device__ __forceinline__ double dot4(FA&& a, FB2&& b) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int j = 0; j < N; j += 4) {
        s0 = fma(a(j), b(j), s0);
        if (j + 1 < N) s1 = fma(a(j + 1), b(j + 1), s1);
        if (j + 2 < N) s2 = fma(a(j + 2), b(j + 2), s2);
        if (j + 3 < N) s3 = fma(a(j + 3), b(j + 3), s3);
    }
    return (s0 + s1) + (s2 + s3);
}

// n doubles of a 16-byte aligned shared row into registers (128-bit loads when n is even)
template <int N>
__device__ __forceinline__ void ld_row(const double* src, double (&dst)[N]) {
    if constexpr (N % 2 == 0) {
#pragma unroll
        for (int i = 0; i < N / 2; ++i) {
            const double2 v = reinterpret_cast<const double2*>(src)[i];
            dst[2 * i] = v.x;
            dst[2 * i + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) dst[i] = src[i];
    }
}

template <int D, bool STREAM, int G = kGL, int WPC = kWWarps, int FB = D>
__global__ void __launch_bounds__(32 * WPC, lpr_minb(G)) kw_smoother_mbf_q(const WParams p) {
    static_assert(D <= G, "one row per lane of a G-lane group");
    constexpr int NP = 32 / G;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K5MSmem<D, STREAM, G, WPC>& sh = *reinterpret_cast<K5MSmem<D, STREAM, G, WPC>*>(smem_raw);
    load_model<D>(sh.m, p.model);
    for (int e = threadIdx.x; e < D * D; e += blockDim.x) {
        const int i = e / D, j = e - (e / D) * D;
        sh.I[i][j] = (i == j) ? 1.0 : 0.0;
        sh.Z[i][j] = 0.0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = blockIdx.x * WPC + wid;
    if (c >= p.nch) return;
    auto& W = sh.w[wid];
    const SModel<D>& M = sh.m;
    const int64_t kb = static_cast<int64_t>(c) * p.K;
    const int64_t ke = min(kb + p.K, p.n);
    // ---- carries (as kw_smoother_apply_q): smoothed moments after each group's last step
    auto& c3P = W.u.c.cP[NP - 1];
    for (int e = lane; e < D * D; e += 32) c3P[e / D][e % D] = 0.0;
    for (int i = lane; i < D; i += 32) W.u.c.cm[NP - 1][i] = 0.0;
    __syncwarp();
    for (int g = p.world - 1; g > p.rank && p.in_smooth; --g) {
        gload<D>(W.u.c.a, p.in_smooth + static_cast<int64_t>(g) * (SNW(D) + 1), lane);
        wapply_suffix<D>(W.u.c.a, W.u.c.cm[NP - 1], c3P, W.u.c.s, lane);
    }
    if (c + 1 < p.nch) {
        gload<D>(W.u.c.a, p.sagg + static_cast<int64_t>(c + 1) * SNW(D), lane);
        wapply_suffix<D>(W.u.c.a, W.u.c.cm[NP - 1], c3P, W.u.c.s, lane);
    }
    for (int q = NP - 2; q >= 0; --q) {
        for (int e = lane; e < D * D; e += 32) W.u.c.cP[q][e / D][e % D] = W.u.c.cP[q + 1][e / D][e % D];
        for (int i = lane; i < D; i += 32) W.u.c.cm[q][i] = W.u.c.cm[q + 1][i];
        __syncwarp();
        gload<D>(W.u.c.a, p.sqagg + (static_cast<int64_t>(c) * (NP - 1) + q) * SNW(D), lane);
        wapply_suffix<D>(W.u.c.a, W.u.c.cm[q], W.u.c.cP[q], W.u.c.s, lane);
    }
    const int q = lane / G, r0 = lane % G, gb = q * G;
    const unsigned gm = group_mask(G, gb);
    const bool act = (D == G) || r0 < D;
    const double af = act ? 1.0 : 0.0;
    const int r = act ? r0 : 0;
    int64_t qb, qe;
    quarter_bounds(kb, ke, p.K, q, qb, qe, NP);
    double Psr[D], msr = W.u.c.cm[q][r];
#pragma unroll
    for (int j = 0; j < D; ++j) Psr[j] = W.u.c.cP[q][r][j];
    const double hr = act ? M.H[r] : 0.0;
    __syncwarp();                                   // W.u (carry scratch) is reused below
    auto& Gs = W.u.g[q];
    const double* xp = p.xp;                        // record of local step k at xp + k CNW
    auto gsum = [&](double v) {
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) v += __shfl_xor_sync(gm, v, off);
        return v;
    };
    auto stage_rec = [&](int64_t k) {
        double* dst = Gs.xst[static_cast<int>(k % 3)];
        const double* src = xp + k * CNW(D);
        for (int i = r0; i < CNW(D); i += G) cp_async8(&dst[i], src + i, 8);
    };
    auto stage_fq = [&](int64_t k) {                // (F_k, Q_k): the transition into local step k
        if (STREAM) {
            const double* fsrc = p.fq + k * FQW(D);
            for (int i = r0; i < FQW(D); i += G) cp_async8(&Gs.fqs[static_cast<int>(k & 1)][i], fsrc + i, 8);
        }
    };
    // (F, Q) of the transition into local step k (shared pointers)
    auto fq_into = [&](int64_t k, const double*& Fp, const double*& Qp) {
        const int kind = wdisc_kind(__ldg(p.t + k) - __ldg(p.t + k - 1), M.udt, STREAM);
        if (kind == 0) {
            if (STREAM) { Fp = &Gs.fqs[static_cast<int>(k & 1)][0]; Qp = Fp + D * LD(D); }
            else { Fp = &M.F[0][0]; Qp = &M.Q[0][0]; }
        } else {
            Fp = &sh.I[0][0]; Qp = &sh.Z[0][0];
        }
    };
    double lh = 0.0, Lh[D];
#pragma unroll
    for (int j = 0; j < D; ++j) Lh[j] = 0.0;
    bool bad = false;
    if (qe > qb) {
        const bool carry = p.k0 + qe - 1 != p.nglob - 1;   // else the group ends the series: lh = Lh = 0
        stage_rec(qe - 1);
        if (qe - 1 > qb) stage_rec(qe - 2);
        if (carry) stage_fq(qe);
        if (qe - 1 > qb) stage_fq(qe - 1);
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp(gm);
        if (carry) {
            // ---- boundary: lh = X^T (x^- - m^s), Lh = X^T (P^- - P^s) X, X = (P^-)^-1 F (transition qe)
            const double* rec = Gs.xst[static_cast<int>((qe - 1) % 3)];
            const double* Fp;
            const double* Qp;
            fq_into(qe, Fp, Qp);
            double FPr[D], xm = 0.0;                // row r of F P_{qe-1}, (F x)_r
#pragma unroll
            for (int j = 0; j < D; ++j) {
                double s2 = 0.0;
#pragma unroll
                for (int t = 0; t < FB; ++t) {
                    const int qq = fblo(r, FB) + t;
                    if (qq < D) s2 = fma(Fp[r * LD(D) + qq], rec[D + si(D, qq, j)], s2);
                }
                FPr[j] = s2;
            }
#pragma unroll
            for (int t = 0; t < FB; ++t) {
                const int qq = fblo(r, FB) + t;
                if (qq < D) xm = fma(Fp[r * LD(D) + qq], rec[qq], xm);
            }
            if (act) {
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    double s2 = Qp[r * LD(D) + j];
#pragma unroll
                    for (int qq = fblo(j, FB); qq < fbhi(j, FB, D); ++qq) s2 = fma(FPr[qq], Fp[j * LD(D) + qq], s2);
                    Gs.Pm[r][j] = s2;
                    Gs.Ps[r][j] = s2 - Psr[j];       // P^- - P^s
                }
                Gs.dm[r] = xm - msr;                 // x^- - m^s
#pragma unroll
                for (int i = 0; i < D; ++i) Gs.X[i][r] = Fp[i * LD(D) + r];   // right-hand side: column r of F
            }
            __syncwarp(gm);
            // cooperative Cholesky of P^- (lane r builds row r of L; 1 / L_rr on the diagonal), then
            // the two triangular solves in place on column r of X
            double Lr[D];
#pragma unroll
            for (int j = 0; j < D; ++j) {
                double sv = Gs.Pm[r][j];
#pragma unroll
                for (int qq = 0; qq < j; ++qq) sv = fma(-Lr[qq], __shfl_sync(gm, Lr[qq], j, G), sv);
                const double sj = __shfl_sync(gm, sv, j, G);
                bad = bad || !(sj > 0.0);
                const double lij = rsqrt(sj);
                Lr[j] = (r == j) ? lij : sv * lij;
            }
            __syncwarp(gm);
            auto& Lm = Gs.Pm;
            if (act) {
#pragma unroll
                for (int qq = 0; qq < D; ++qq) Lm[r][qq] = Lr[qq];
            }
            __syncwarp(gm);
            if (act) {
#pragma unroll 4
                for (int i = 0; i < D; ++i) {
                    double z = Gs.X[i][r];
                    for (int qq = 0; qq < i; ++qq) z = fma(-Lm[i][qq], Gs.X[qq][r], z);
                    Gs.X[i][r] = z * Lm[i][i];
                }
#pragma unroll 4
                for (int i = D - 1; i >= 0; --i) {
                    double z = Gs.X[i][r];
                    for (int qq = i + 1; qq < D; ++qq) z = fma(-Lm[qq][i], Gs.X[qq][r], z);
                    Gs.X[i][r] = z * Lm[i][i];
                }
            }
            __syncwarp(gm);
            double Xr[D], V[D];
#pragma unroll
            for (int i = 0; i < D; ++i) Xr[i] = Gs.X[i][r];
#pragma unroll
            for (int i = 0; i < D; ++i) lh = fma(Xr[i], Gs.dm[i], lh);
#pragma unroll
            for (int bb = 0; bb < D; ++bb) {
                double v = 0.0;
#pragma unroll
                for (int a = 0; a < D; ++a) v = fma(Xr[a], Gs.Ps[a][bb], v);
                V[bb] = v;
            }
#pragma unroll
            for (int j = 0; j < D; ++j) {
                double s2 = 0.0;
#pragma unroll
                for (int bb = 0; bb < D; ++bb) s2 = fma(V[bb], Gs.X[bb][j], s2);
                Lh[j] = s2;
            }
            __syncwarp(gm);
        }
    }
    double hrow[D];
#pragma unroll
    for (int j = 0; j < D; ++j) hrow[j] = M.H[j];
    for (int64_t k = qe - 1; k >= qb; --k) {
        // prefetch the record of k - 2 and (F, Q) into k - 1 (the next step's update)
        if (k - 2 >= qb) stage_rec(k - 2);
        if (k - 1 > qb) stage_fq(k - 1);
        cp_async_commit();
        const double* rec = Gs.xst[static_cast<int>(k % 3)];
        // ---- output: mean = h x - (P h^T) . lh, var = h P h^T - (P h^T)^T Lh (P h^T)
        const double Ph = dot4<D>([&](int j) { return rec[D + si(D, r, j)]; }, [&](int j) { return hrow[j]; });
        const double hx = dot4<D>([&](int j) { return hrow[j]; }, [&](int j) { return rec[j]; });
        // row vectors are exchanged through the group's shared slots (one store, vector loads)
        double* vPh = &Gs.Ps[0][0];                 // [D]: P_k h^T
        double* vPg = vPh + 2 * ((D + 1) / 2);      // [D]: P_{k-1} g
        double* vK = vPg + 2 * ((D + 1) / 2);       // [D]: K_k
        double* vw = vK + 2 * ((D + 1) / 2);        // [D]: Lh K
        double (*LFs)[LD(D)] = Gs.Pm;               // rows of Lt F_k (padded stride: conflict-free columns)
        if (act) vPh[r] = Ph;
        __syncwarp(gm);
        double tmp[D];
        ld_row<D>(vPh, tmp);
        const double LPh = dot4<D>([&](int j) { return Lh[j]; }, [&](int j) { return tmp[j]; });
        const double s_quad = gsum(af * Ph * LPh), s_lph = gsum(af * Ph * lh), s_hph = gsum(hr * Ph);
        if (r0 == 0) {
            if (p.mean) p.mean[k] = hx - s_lph;
            if (p.var) p.var[k] = s_hph - s_quad;
        }
        if (k > qb) {
            // ---- update at k, then back through F_k to k - 1
            const double* prv = Gs.xst[static_cast<int>((k - 1) % 3)];
            const double* Fp;
            const double* Qp;
            fq_into(k, Fp, Qp);
            const bool obs = __ldg(p.mask + k) != 0;
            const double yk = obs ? __ldg(p.y + k) : 0.0;
            // g = F^T h^T (all of it), P_{k-1} g (row r), P^- h^T = F (P g) + Q h^T (row r), x^- = F x
            double gv[D];
#pragma unroll
            for (int i = 0; i < D; ++i) {
                double s2 = 0.0;
#pragma unroll
                for (int qq = fblo(i, FB); qq < fbhi(i, FB, D); ++qq) s2 = fma(Fp[qq * LD(D) + i], hrow[qq], s2);
                gv[i] = s2;
            }
            const double Pg = dot4<D>([&](int j) { return prv[D + si(D, r, j)]; }, [&](int j) { return gv[j]; });
            if (act) vPg[r] = Pg;
            __syncwarp(gm);
            double PmH = 0.0, xm = 0.0;
#pragma unroll
            for (int t = 0; t < FB; ++t) {
                const int qq = fblo(r, FB) + t;
                if (qq < D) {
                    const double f = Fp[r * LD(D) + qq];
                    PmH = fma(f, vPg[qq], PmH);
                    PmH = fma(Qp[r * LD(D) + qq], hrow[qq], PmH);
                    xm = fma(f, prv[qq], xm);
                }
            }
            double lt = lh, Lt[D];
#pragma unroll
            for (int j = 0; j < D; ++j) Lt[j] = Lh[j];
            const double S = gsum(hr * PmH) + M.r, hxm = gsum(hr * xm);
            if (obs) {
                bad = bad || !(S > 0.0);
                const double iS = 1.0 / S, vs = (yk - hxm) * iS;
                const double Kr = PmH * iS;
                if (act) vK[r] = Kr;
                __syncwarp(gm);
                ld_row<D>(vK, tmp);
                const double w = dot4<D>([&](int j) { return Lh[j]; }, [&](int j) { return tmp[j]; });
                if (act) vw[r] = w;
                const double cK = gsum(af * Kr * w), Kl = gsum(af * Kr * lh);   // (the reduction orders the store)
                __syncwarp(gm);
                ld_row<D>(vw, tmp);
#pragma unroll
                for (int j = 0; j < D; ++j)
                    Lt[j] = fma(-hr, tmp[j], fma(-w, hrow[j], fma((cK + iS) * hr, hrow[j], Lh[j])));
                lt = fma(-hr, Kl + vs, lh);
            }
            // lh <- F^T lt, Lh <- F^T Lt F: row r of Lt F in registers and shared, then the rows of
            // r's block
            double LF[D];
#pragma unroll
            for (int j = 0; j < D; ++j) {
                double s2 = 0.0;
#pragma unroll
                for (int qq = fblo(j, FB); qq < fbhi(j, FB, D); ++qq) s2 = fma(Lt[qq], Fp[qq * LD(D) + j], s2);
                LF[j] = s2;
            }
            __syncwarp(gm);                         // every lane is done with the previous LFs
            if (act) {
#pragma unroll
                for (int j = 0; j < D; ++j) LFs[r][j] = LF[j];
                vPh[r] = lt;                        // (vPh is free again: reused for lt)
            }
            __syncwarp(gm);
            double lhn = 0.0, Lhn[D];
#pragma unroll
            for (int j = 0; j < D; ++j) Lhn[j] = 0.0;
#pragma unroll
            for (int t = 0; t < FB; ++t) {
                const int qq = fblo(r, FB) + t;
                if (qq < D) {
                    const double fqr = Fp[qq * LD(D) + r];
                    lhn = fma(fqr, vPh[qq], lhn);
#pragma unroll
                    for (int j = 0; j < D; ++j) Lhn[j] = fma(fqr, LFs[qq][j], Lhn[j]);
                }
            }
            lh = lhn;
#pragma unroll
            for (int j = 0; j < D; ++j) Lh[j] = Lhn[j];
        }
        cp_async_wait<0>();
        __syncwarp(gm);
    }
    if (bad && r0 == 0) raise_error(p.err, p.k0 + qb, kErrNumeric);
}


// ================================================================== NLL gradient of any model (uniform dt)
// Reverse mode over the Kalman recursion (supplement PAPER.md:304-315; the paper differentiates the
// parallel filter by AD).  With the adjoint (b_k, C_k) = d NLL_{>k} / d (x_k, P_k) of
// the filtered moments, one step k maps it back as an affine map
//   b_{k-1} = M_k^T b_k + beta_k,  C_{k-1} = M_k^T C_k M_k + sym(M_k^T b_k u_k^T) + Gamma_k,
//   M_k = (I - K_k h^T) F,  g = F^T h,  u_k = (v/S) g,  beta_k = -u_k,  Gamma_k = c1 g g^T,
//   c1 = (1/S - v^2/S^2) / 2   (missing y: M_k = F, u = beta = Gamma = 0),
// and these maps compose in closed form: (M, U, Gamma) with beta = -U always,
//   Phi_1 o Phi_2 = (M_2 M_1, U_1 + M_1^T U_2, Gamma_1 - sym(M_1^T U_2 U_1^T) + M_1^T Gamma_2 M_1)
// (Phi_2 applied first, i.e. the later steps).  The forward rescan (kw_grad_forward) composes each
// chain's map step by step at O(d^2) + one F M product per step, a reverse Kogge-Stone scan
// (kw_scan_adjoint) gives the adjoint entering every chain from the right, and the backward rescan
// (kw_grad_backward) runs the adjoint recursion, accumulating with the adjoint before the update
// (b^-, C^-) of every uniform step
//   Z += b^- x_{k-1}^T + 2 C^- F P_{k-1},   Cs += C^-,   gr += c1 - (b_k . K)(v/S) + K^T C_k K,
// and C0 = C^- of the global first step; then d NLL / d theta_p = <dF_p, Z> + <dQ_p, Cs> +
// <dP_inf_p, C0> (+ r gr for log r) because dF_p, dQ_p are the same at every uniform step
// (k_grad_contract).  Steps with dt = 0 (F = I, Q = 0) carry the adjoint but have no theta
// dependence.  DESIGN.md §5c.
struct GradBufs {
    double* gagg;      // [nch][SNW]  chain adjoint maps (M, U, Gamma full) -> their reverse scan
    double* gbuf;      // [nch][SNW]  ping-pong of the scan
    double* gcar;      // [nch][CNW]  filtered state entering each chain
    double* gpart;     // [nch][2 D^2 + 1]  per-chain (Z, Cs, gr)
    double* gc0;       // [D^2]       C^- of the global first step
};
PS_CX int GPN(int D) { return 2 * D * D + 1; }

template <int D>
struct GFwdSmem {
    SModel<D> m;
    struct PerWarp {
        double P[D][LD(D)], M[D][LD(D)], Gam[D][LD(D)];
        double x[D], U[D];
        double FP[D][LD(D)], Pm[D][LD(D)], FM[D][LD(D)];   // step scratch (also the carry's)
        double xm[D], HP[D], w[D];
        SF<D> a;                                             // the scanned aggregate before the chain
    } w[kWWarps];
};

template <int D>
__global__ void __launch_bounds__(32 * kWWarps) kw_grad_forward(const WParams p, const GradBufs gb) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    GFwdSmem<D>& sh = *reinterpret_cast<GFwdSmem<D>*>(smem_raw);
    load_model<D>(sh.m, p.model);
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = blockIdx.x * kWWarps + wid;
    if (c >= p.nch) return;
    auto& W = sh.w[wid];
    const SModel<D>& M = sh.m;
    for (int e = lane; e < D * D; e += 32) W.P[e / D][e % D] = 0.0;
    for (int i = lane; i < D; i += 32) W.x[i] = 0.0;
    __syncwarp();
    if (c > 0) {
        gload<D>(W.a, p.fagg + static_cast<int64_t>(c - 1) * FNW(D), lane);
        if (!wapply_prefix_gj<D>(W.x, W.P, W.a, W.FP, W.Pm, W.FM, W.xm, W.HP, lane) && lane == 0)
            raise_error(p.err, p.k0, kErrNumeric);
    }
    {   // filtered state entering the chain (for the backward rescan's first step)
        double* o = gb.gcar + static_cast<int64_t>(c) * CNW(D);
        for (int i = lane; i < D; i += 32) o[i] = W.x[i];
        for (int e = lane; e < D * D; e += 32) {
            const int i = e / D, j = e - (e / D) * D;
            if (j >= i) o[D + si(D, i, j)] = W.P[i][j];
        }
    }
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        W.M[i][j] = (i == j) ? 1.0 : 0.0;
        W.Gam[i][j] = 0.0;
    }
    for (int i = lane; i < D; i += 32) W.U[i] = 0.0;
    __syncwarp();
    const int64_t kb = static_cast<int64_t>(c) * p.K;
    const int64_t ke = min(kb + p.K, p.n);
    double tprev = (kb < p.n && (kb > 0 || p.k0 > 0)) ? __ldg(p.t + kb - 1) : 0.0;
    double quad = 0.0, logs = 0.0;
    int nobs = 0;
    double* xpc = p.xp + static_cast<int64_t>(c) * p.K * CNW(D);
    // the step inputs are loaded one step ahead (their latency overlaps the previous step)
    double tn = 0.0, yn = 0.0;
    bool on = false;
    if (kb < ke) {
        tn = __ldg(p.t + kb);
        on = __ldg(p.mask + kb) != 0;
        yn = on ? __ldg(p.y + kb) : 0.0;
    }
    for (int64_t k = kb; k < ke; ++k) {
        const double tk = tn;
        const bool obs = on;
        const double yk = yn;
        if (k + 1 < ke) {
            tn = __ldg(p.t + k + 1);
            on = __ldg(p.mask + k + 1) != 0;
            yn = on ? __ldg(p.y + k + 1) : 0.0;
        }
        const int64_t g = p.k0 + k;
        const int kind = (g == 0) ? 3 : wdisc_kind(tk - tprev, M.udt, false);
        tprev = tk;
        if (kind == 0) {
            wmm<D>(W.FP, M.F, W.P, nullptr, lane);
            wmm<D>(W.FM, M.F, W.M, nullptr, lane);
            for (int i = lane; i < D; i += 32) {
                double s2 = 0.0;
                for (int q = 0; q < D; ++q) s2 = fma(M.F[i][q], W.x[q], s2);
                W.xm[i] = s2;
            }
            __syncwarp();
            wmm<D, false, true>(W.Pm, W.FP, M.F, M.Q, lane);
        } else {
            for (int e = lane; e < D * D; e += 32) {
                const int i = e / D, j = e - (e / D) * D;
                W.FM[i][j] = (kind == 1) ? W.M[i][j] : 0.0;
                W.Pm[i][j] = (kind == 1) ? W.P[i][j] : M.Pinf[i][j];
            }
            for (int i = lane; i < D; i += 32) W.xm[i] = (kind == 1) ? W.x[i] : 0.0;
        }
        __syncwarp();
        for (int i = lane; i < D; i += 32) {
            double hp = 0.0, ww = 0.0;
            for (int q = 0; q < D; ++q) {
                hp = fma(W.Pm[i][q], M.H[q], hp);
                ww = fma(W.FM[q][i], M.H[q], ww);
            }
            W.HP[i] = hp;
            W.w[i] = ww;
        }
        __syncwarp();
        const double S = wdot<D>(M.H, W.HP, lane) + M.r;
        const double hx = wdot<D>(M.H, W.xm, lane);
        if (lane == 0 && obs && !(S > 0.0 && S < INFINITY)) raise_error(p.err, g, kErrNumeric);
        const double iS = obs ? 1.0 / S : 0.0;
        const double v = obs ? (yk - hx) : 0.0;
        const double vs = v * iS;
        const double c1 = obs ? 0.5 * (iS - vs * vs) : 0.0;
        for (int e = lane; e < D * D; e += 32) {
            const int i = e / D, j = e - (e / D) * D;
            const double hpi = W.HP[i] * iS;
            W.P[i][j] = fma(-hpi, W.HP[j], W.Pm[i][j]);
            W.M[i][j] = fma(-hpi, W.w[j], W.FM[i][j]);
            const double wi = W.w[i], wj = W.w[j];
            W.Gam[i][j] += fma(c1 * wi, wj, -0.5 * vs * (wi * W.U[j] + W.U[i] * wj));
        }
        __syncwarp();
        for (int i = lane; i < D; i += 32) {
            W.x[i] = fma(W.HP[i], vs, W.xm[i]);
            W.U[i] = fma(vs, W.w[i], W.U[i]);
        }
        if (obs) {
            quad = fma(v, vs, quad);
            logs += log(S);
            ++nobs;
        }
        __syncwarp();
        double* o = xpc + (k - kb) * CNW(D);
        for (int i = lane; i < D; i += 32) o[i] = W.x[i];
        for (int e = lane; e < D * D; e += 32) {
            const int i = e / D, j = e - (e / D) * D;
            if (j >= i) o[D + si(D, i, j)] = W.P[i][j];
        }
    }
    if (lane == 0) p.nll_chain[c] = nobs ? 0.5 * (quad + logs + nobs * 1.8378770664093453) : 0.0;
    double* ga = gb.gagg + static_cast<int64_t>(c) * SNW(D);
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        ga[e] = W.M[i][j];
        ga[D * D + D + e] = W.Gam[i][j];
    }
    for (int i = lane; i < D; i += 32) ga[D * D + i] = W.U[i];
}

// One reverse Kogge-Stone level of the chain adjoint maps: out[c] = in[c] o in[c + off] (the later
// chain's map applied first), or in[c] when c + off >= nch.  One warp per element.
template <int D>
struct ScanSmemA {
    double M1[D][LD(D)], M2[D][LD(D)], G1[D][LD(D)], G2[D][LD(D)], T1[D][LD(D)], T2[D][LD(D)];
    double U1[D], U2[D], MU[D];
};
template <int D>
__global__ void __launch_bounds__(32) kw_scan_adjoint(const double* __restrict__ in, double* __restrict__ out,
                                                      int nch, int off) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ScanSmemA<D>& sh = *reinterpret_cast<ScanSmemA<D>*>(smem_raw);
    const int lane = threadIdx.x;
    const int c = blockIdx.x;
    const double* a = in + static_cast<int64_t>(c) * SNW(D);
    double* o = out + static_cast<int64_t>(c) * SNW(D);
    if (c + off >= nch) {
        for (int e = lane; e < SNW(D); e += 32) o[e] = a[e];
        return;
    }
    const double* b = in + static_cast<int64_t>(c + off) * SNW(D);
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        sh.M1[i][j] = a[e];
        sh.G1[i][j] = a[D * D + D + e];
        sh.M2[i][j] = b[e];
        sh.G2[i][j] = b[D * D + D + e];
    }
    for (int i = lane; i < D; i += 32) {
        sh.U1[i] = a[D * D + i];
        sh.U2[i] = b[D * D + i];
    }
    __syncwarp();
    wmm<D>(sh.T1, sh.G2, sh.M1, nullptr, lane);                 // Gamma_2 M_1
    wmm<D>(sh.T2, sh.M2, sh.M1, nullptr, lane);                 // M_2 M_1
    for (int i = lane; i < D; i += 32) {
        double s2 = 0.0;
        for (int q = 0; q < D; ++q) s2 = fma(sh.M1[q][i], sh.U2[q], s2);
        sh.MU[i] = s2;                                          // M_1^T U_2
    }
    __syncwarp();
    wmm<D, true, false>(sh.M2, sh.M1, sh.T1, sh.G1, lane);      // Gamma_1 + M_1^T Gamma_2 M_1 (into M2)
    __syncwarp();
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        o[e] = sh.T2[i][j];
        const double gsym = 0.5 * (sh.M2[i][j] + sh.M2[j][i]);
        o[D * D + D + e] = gsym - 0.5 * (sh.MU[i] * sh.U1[j] + sh.U1[i] * sh.MU[j]);
    }
    for (int i = lane; i < D; i += 32) o[D * D + i] = sh.U1[i] + sh.MU[i];
}

template <int D>
struct GBwdSmem {
    SModel<D> m;
    struct PerWarp {
        double C[D][LD(D)], Z[D][LD(D)], Cs[D][LD(D)], Pp[D][LD(D)], FP[D][LD(D)], Pm[D][LD(D)], T[D][LD(D)],
            Cm[D][LD(D)];
        double b[D], xp[D], xm[D], HP[D], K[D], CK[D], KT[D], Mb[D], bm[D];
        double rec[CNW(D)];                 // the packed filtered record of the previous step
    } w[kWWarps];
};

template <int D>
__global__ void __launch_bounds__(32 * kWWarps) kw_grad_backward(const WParams p, const GradBufs gb,
                                                                  const double* __restrict__ scanned) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    GBwdSmem<D>& sh = *reinterpret_cast<GBwdSmem<D>*>(smem_raw);
    load_model<D>(sh.m, p.model);
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = blockIdx.x * kWWarps + wid;
    if (c >= p.nch) return;
    auto& W = sh.w[wid];
    const SModel<D>& M = sh.m;
    // adjoint after the chain's last step: (beta, Gamma) = (-U, Gamma) of the scanned maps of c + 1 ...
    for (int e = lane; e < D * D; e += 32) {
        const int i = e / D, j = e - (e / D) * D;
        W.C[i][j] = (c + 1 < p.nch) ? scanned[static_cast<int64_t>(c + 1) * SNW(D) + D * D + D + e] : 0.0;
        W.Z[i][j] = 0.0;
        W.Cs[i][j] = 0.0;
    }
    for (int i = lane; i < D; i += 32)
        W.b[i] = (c + 1 < p.nch) ? -scanned[static_cast<int64_t>(c + 1) * SNW(D) + D * D + i] : 0.0;
    __syncwarp();
    const int64_t kb = static_cast<int64_t>(c) * p.K;
    const int64_t ke = min(kb + p.K, p.n);
    const double* xpc = p.xp + static_cast<int64_t>(c) * p.K * CNW(D);
    double gr = 0.0;
    // the filtered record of step k - 1 and the inputs of step k are loaded one step ahead into
    // registers (the global-load latency overlaps the previous step's work)
    constexpr int NPL = (CNW(D) + 31) / 32;
    double pre[NPL];
    auto load_rec = [&](int64_t k) {
        const double* src = (k > kb) ? xpc + (k - 1 - kb) * CNW(D) : gb.gcar + static_cast<int64_t>(c) * CNW(D);
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const int e = lane + 32 * q;
            pre[q] = (e < CNW(D)) ? src[e] : 0.0;
        }
    };
    double tn = 0.0, tpn = 0.0, yn = 0.0;
    bool on = false;
    auto load_in = [&](int64_t k) {
        tn = __ldg(p.t + k);
        tpn = (p.k0 + k > 0) ? __ldg(p.t + k - 1) : 0.0;
        on = __ldg(p.mask + k) != 0;
        yn = on ? __ldg(p.y + k) : 0.0;
    };
    if (ke > kb) {
        load_rec(ke - 1);
        load_in(ke - 1);
    }
    for (int64_t k = ke - 1; k >= kb; --k) {
        const int64_t g = p.k0 + k;
        const double tk = tn;
        const int kind = (g == 0) ? 3 : wdisc_kind(tk - tpn, M.udt, false);
        const bool obs = on;
        const double yk = yn;
        if (kind != 3) {   // filtered state of the previous step (prefetched)
#pragma unroll
            for (int q = 0; q < NPL; ++q) {
                const int e = lane + 32 * q;
                if (e < CNW(D)) W.rec[e] = pre[q];
            }
            __syncwarp();
            for (int i = lane; i < D; i += 32) W.xp[i] = W.rec[i];
            for (int e = lane; e < D * D; e += 32) {
                const int i = e / D, j = e - (e / D) * D;
                W.Pp[i][j] = W.rec[D + si(D, i, j)];
            }
            __syncwarp();
        }
        if (k - 1 >= kb) {
            load_rec(k - 1);
            load_in(k - 1);
        }
        // P^- h^T (W.HP) and x^- (W.xm); P^- itself is never formed
        if (kind == 0) {
            for (int i = lane; i < D; i += 32) {     // g = F^T h^T (in W.bm, rewritten below), x^- = F x
                double s2 = 0.0, xm = 0.0;
                for (int q = 0; q < D; ++q) {
                    s2 = fma(M.F[q][i], M.H[q], s2);
                    xm = fma(M.F[i][q], W.xp[q], xm);
                }
                W.bm[i] = s2;
                W.xm[i] = xm;
            }
            __syncwarp();
            for (int i = lane; i < D; i += 32) {     // P_{k-1} g (in W.Mb, rewritten below)
                double s2 = 0.0;
                for (int q = 0; q < D; ++q) s2 = fma(W.Pp[i][q], W.bm[q], s2);
                W.Mb[i] = s2;
            }
            __syncwarp();
            for (int i = lane; i < D; i += 32) {     // F (P g) + Q h^T
                double s2 = 0.0;
                for (int q = 0; q < D; ++q) s2 = fma(M.F[i][q], W.Mb[q], fma(M.Q[i][q], M.H[q], s2));
                W.HP[i] = s2;
            }
        } else {
            for (int i = lane; i < D; i += 32) {
                double hp = 0.0;
                for (int q = 0; q < D; ++q) hp = fma((kind == 1) ? W.Pp[i][q] : M.Pinf[i][q], M.H[q], hp);
                W.HP[i] = hp;
                W.xm[i] = (kind == 1) ? W.xp[i] : 0.0;
            }
        }
        __syncwarp();
        if (obs) {
            const double S = wdot<D>(M.H, W.HP, lane) + M.r;
            const double v = yk - wdot<D>(M.H, W.xm, lane);
            const double iS = 1.0 / S, vs = v * iS, c1 = 0.5 * (iS - vs * vs);
            for (int i = lane; i < D; i += 32) W.K[i] = W.HP[i] * iS;
            __syncwarp();
            for (int i = lane; i < D; i += 32) {
                double s2 = 0.0;
                for (int q = 0; q < D; ++q) s2 = fma(W.C[i][q], W.K[q], s2);
                W.CK[i] = s2;
            }
            __syncwarp();
            const double bK = wdot<D>(W.b, W.K, lane), KCK = wdot<D>(W.K, W.CK, lane);
            gr += c1 - bK * vs + KCK;
            // (I - K h^T)^T C (I - K h^T) + (v/S) sym(h Mb^T) + c1 h h^T, Mb = (I - K h^T)^T b
            for (int e = lane; e < D * D; e += 32) {
                const int i = e / D, j = e - (e / D) * D;
                W.T[i][j] = fma(-W.CK[i], M.H[j], W.C[i][j]);   // C (I - K h^T)
            }
            for (int i = lane; i < D; i += 32) W.Mb[i] = fma(-M.H[i], bK, W.b[i]);
            __syncwarp();
            for (int j = lane; j < D; j += 32) {
                double s2 = 0.0;
                for (int q = 0; q < D; ++q) s2 = fma(W.K[q], W.T[q][j], s2);
                W.KT[j] = s2;
            }
            __syncwarp();
            for (int e = lane; e < D * D; e += 32) {
                const int i = e / D, j = e - (e / D) * D;
                const double hi = M.H[i], hj = M.H[j];
                W.Cm[i][j] = fma(-hi, W.KT[j], W.T[i][j]) + 0.5 * vs * (hi * W.Mb[j] + W.Mb[i] * hj) + c1 * hi * hj;
            }
            for (int i = lane; i < D; i += 32) W.bm[i] = fma(-vs, M.H[i], W.Mb[i]);
        } else {
            for (int e = lane; e < D * D; e += 32) W.Cm[e / D][e % D] = W.C[e / D][e % D];
            for (int i = lane; i < D; i += 32) W.bm[i] = W.b[i];
        }
        __syncwarp();
        if (kind == 3) {   // the global first step: x^- = 0, P^- = P_inf
            for (int e = lane; e < D * D; e += 32) gb.gc0[e] = W.Cm[e / D][e % D];
            break;
        }
        if (kind == 0) {
            wmm<D>(W.FP, W.Cm, M.F, nullptr, lane);                  // C^- F
            for (int i = lane; i < D; i += 32) {
                double s2 = 0.0;
                for (int q = 0; q < D; ++q) s2 = fma(M.F[q][i], W.bm[q], s2);
                W.b[i] = s2;                                          // F^T b^-
            }
            __syncwarp();
            wmm<D>(W.T, W.FP, W.Pp, nullptr, lane);                  // C^- F P_{k-1}
            wmm<D, true, false>(W.Pm, M.F, W.FP, nullptr, lane);     // F^T C^- F
            __syncwarp();
            for (int e = lane; e < D * D; e += 32) {
                const int i = e / D, j = e - (e / D) * D;
                W.Z[i][j] += fma(W.bm[i], W.xp[j], 2.0 * W.T[i][j]);
                W.Cs[i][j] += W.Cm[i][j];
                W.C[i][j] = 0.5 * (W.Pm[i][j] + W.Pm[j][i]);
            }
        } else {
            for (int e = lane; e < D * D; e += 32) W.C[e / D][e % D] = W.Cm[e / D][e % D];
            for (int i = lane; i < D; i += 32) W.b[i] = W.bm[i];
        }
        __syncwarp();
    }
    double* o = gb.gpart + static_cast<int64_t>(c) * GPN(D);
    for (int e = lane; e < D * D; e += 32) {
        o[e] = W.Z[e / D][e % D];
        o[D * D + e] = W.Cs[e / D][e % D];
    }
    if (lane == 0) o[2 * D * D] = gr;
}

// d NLL / d theta_p = <dF_p, Z> + <dQ_p, Cs> + <dP_inf_p, C0>  (p < npar - 1), r gr (log noise):
// fixed-order sums of the chain partials, then one warp per parameter.  <<<1, 256>>>.
template <int D>
__global__ void __launch_bounds__(256) k_grad_contract(const double* __restrict__ gpart, int nch,
                                                       const double* __restrict__ gc0,
                                                       const double* __restrict__ gder, int npar, double r,
                                                       double* grad) {
    __shared__ double tot[GPN(D)];
    for (int e = threadIdx.x; e < GPN(D); e += blockDim.x) {
        double s2 = 0.0;
        for (int c = 0; c < nch; ++c) s2 += gpart[static_cast<int64_t>(c) * GPN(D) + e];
        tot[e] = s2;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int pp = wid; pp < npar; pp += blockDim.x / 32) {
        double acc = 0.0;
        if (pp < npar - 1) {
            const double* dd = gder + static_cast<int64_t>(pp) * 3 * D * D;
            for (int e = lane; e < D * D; e += 32)
                acc += dd[e] * tot[e] + dd[D * D + e] * tot[D * D + e] + dd[2 * D * D + e] * gc0[e];
        } else if (lane == 0) {
            acc = r * tot[2 * D * D];
        }
        acc = wsum(acc);
        if (lane == 0) grad[pp] = acc;
    }
}

}  // namespace wide
}  // namespace pssgp
