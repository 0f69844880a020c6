// pssgp_math.cuh — register-resident small-matrix math of the PSSGP hot path.
//
// Everything is fp64 (the optional fp32 build, pssgp_f32.cu, re-includes this file with
// real = float for the state algebra), fully unrolled at compile time for a state dimension D,
// with symmetric matrices (C, J, P, L, Q, P_inf) stored as PACKED UPPER
// TRIANGLES so that the symmetry the filtering operator needs for
// associativity (SURVEY.md finding 3) is structural.
// Functions are __host__ __device__ so the host introspection entry points
// (pssgp_debug_discretize) run exactly the code the kernels run.
//
// Paper map (PAPER.md = arXiv:2102.09964 text):
//   filter element + fold  : Eqs. (6)-(8) PAPER.md:94-112, observed case PAPER.md:359
//   filtering operator     : PAPER.md:116-121
//   Kalman step            : supplement PAPER.md:285-315
//   smoother operator      : PAPER.md:433, 446-449 (reading Z2)
//   RTS step               : PAPER.md:422-430
//   discretisation         : PAPER.md:294-303 (closed forms for Matern)
#pragma once
#include <type_traits>
#include <cstdint>
#include <cmath>

#ifndef PSSGP_ESTRIN
#define PSSGP_ESTRIN 1
#endif

#if defined(__CUDACC__)
#define PS_HD __host__ __device__ __forceinline__
#define PS_CX __host__ __device__ constexpr
#else
#define PS_HD inline
#define PS_CX constexpr
#endif

#ifndef PSSGP_NS
#define PSSGP_NS pssgp          // the fp64 build; pssgp_f32.cu re-includes with pssgp_f32 / float
#endif
#ifndef PSSGP_REAL
#define PSSGP_REAL double
#endif

namespace PSSGP_NS {

// scalar type of the state algebra (moments, aggregates, F, Q); times, observations, outputs and
// the NLL accumulation stay fp64 in every build (fp32 ulp at t ~ 2048 exceeds the step)
using real = PSSGP_REAL;

PS_CX int ns(int D) { return D * (D + 1) / 2; }
// packed-upper index of (i, j), any order
PS_CX int si(int D, int i, int j) {
    return i <= j ? i * (2 * D - i + 1) / 2 + (j - i) : j * (2 * D - j + 1) / 2 + (i - j);
}
PS_CX int FN(int D) { return D * D + 2 * D + 2 * ns(D); }  // filter aggregate reals
PS_CX int SN(int D) { return D * D + D + ns(D); }          // smoother aggregate reals
PS_CX int CN(int D) { return D + ns(D); }                  // (mean, cov) pair reals

// ------------------------------------------------------------------ branch-free scalar math
// Constants live in a table (device: __constant__, host: constexpr) so the
// kernels read them as constant-bank operands instead of re-materialising
// 64-bit literals with uniform-register moves.
struct MathConsts {
    real expc[28];   // 1/k!, k = 0..27 (Taylor of e^r on |r| <= ln2/2 uses k <= 13; R_m series)
    real inv[32];    // 1/n, n = 0..31 (inv[0] unused)
    real qw[4];      // Jordan-basis Q weights 2/3, 4/3, 8/3, 2 (constant-bank operands, not immediates)
};
#define PS_MATH_CONSTS                                                                         \
    {{1.0, 1.0, 0.5, 0.16666666666666666, 0.041666666666666664,  \
      0.008333333333333333, 0.001388888888888889, 0.0001984126984126984, 2.48015873015873e-05, 2.7557319223985893e-06,  \
      2.755731922398589e-07, 2.505210838544172e-08, 2.08767569878681e-09, 1.6059043836821613e-10, 1.1470745597729725e-11,  \
      7.647163731819816e-13, 4.779477332387385e-14, 2.8114572543455206e-15, 1.5619206968586225e-16, 8.22063524662433e-18,  \
      4.110317623312165e-19, 1.9572941063391263e-20, 8.896791392450574e-22, 3.868170170630684e-23, 1.6117375710961184e-24,  \
      6.446950284384474e-26, 2.4795962632247976e-27, 9.183689863795546e-29},  \
     {0.0, 1.0, 1.0 / 2, 1.0 / 3, 1.0 / 4, 1.0 / 5, 1.0 / 6, 1.0 / 7, 1.0 / 8, 1.0 / 9, 1.0 / 10, \
      1.0 / 11, 1.0 / 12, 1.0 / 13, 1.0 / 14, 1.0 / 15, 1.0 / 16, 1.0 / 17, 1.0 / 18, 1.0 / 19,   \
      1.0 / 20, 1.0 / 21, 1.0 / 22, 1.0 / 23, 1.0 / 24, 1.0 / 25, 1.0 / 26, 1.0 / 27, 1.0 / 28,   \
      1.0 / 29, 1.0 / 30, 1.0 / 31},                                                              \
     {2.0 / 3.0, 4.0 / 3.0, 8.0 / 3.0, 2.0}}
#if defined(__CUDACC__)
static __constant__ MathConsts d_mc = PS_MATH_CONSTS;
#endif
static constexpr MathConsts h_mc = PS_MATH_CONSTS;
PS_HD const MathConsts& mc() {
#if defined(__CUDA_ARCH__)
    return d_mc;
#else
    return h_mc;
#endif
}

// Reciprocal of a positive normal double, branch-free: scale into [1, 2) by
// exponent-field arithmetic, fp32 hardware reciprocal as the seed (~2^-23),
// two Newton steps in fp64 (error squared each: < 2^-90), scale back.
// Host: plain division.
PS_HD double rcp(double a) {
#if defined(__CUDA_ARCH__)
    const long long bits = __double_as_longlong(a);
    const long long ex = bits & 0x7ff0000000000000LL;
    const double m = __longlong_as_double((bits & ~0x7ff0000000000000LL) | 0x3ff0000000000000LL);  // [1, 2)
    float rf;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rf) : "f"(__double2float_rn(m)));
    double r = static_cast<double>(rf);
    double e = fma(-m, r, 1.0);
    r = fma(r, e, r);
    e = fma(-m, r, 1.0);
    r = fma(r, e, r);                                                     // 1/m in (0.5, 1]
    // 1/a = r * 2^-(E-1023): subtract the exponent field (result stays normal for normal a
    // with E in (1, 2046))
    return __longlong_as_double(__double_as_longlong(r) - (ex - 0x3ff0000000000000LL));
#else
    return 1.0 / a;
#endif
}

// e^{-z} for z >= 0, branch-free: n = rint(z / ln2), r = n ln2 - z (Cody-Waite),
// Taylor-13 of e^r, times 2^-n by exponent arithmetic.  z is clamped to 708
// (e^-708 ~ 3e-308: below every quantity the kernels combine it with).
template <bool FAST = false>
PS_HD double exp_neg(double z) {
#if defined(__CUDA_ARCH__)
    const MathConsts& C = mc();
    if (FAST || z < 0.015625) {   // FAST: caller guarantees 0 <= z < 2^-6
        // |z| < 2^-6: Taylor-9 of e^{-z} directly (truncation < 4e-22 relative), no range reduction
        double pz = C.expc[9];
#pragma unroll
        for (int k = 8; k >= 0; --k) pz = fma(pz, -z, C.expc[k]);
        return pz;
    }
    z = fmin(fmax(z, 0.0), 708.0);
    const double n = rint(z * 1.4426950408889634);
    const double r = fma(n, 1.9082149292705877e-10, fma(n, 0.6931471803691238, -z));
#if PSSGP_ESTRIN
    // Estrin scheme: dependency depth 5 instead of 13
    const double r2 = r * r, r4 = r2 * r2, r8 = r4 * r4;
    const double p01 = fma(C.expc[1], r, C.expc[0]), p23 = fma(C.expc[3], r, C.expc[2]);
    const double p45 = fma(C.expc[5], r, C.expc[4]), p67 = fma(C.expc[7], r, C.expc[6]);
    const double p89 = fma(C.expc[9], r, C.expc[8]), pab = fma(C.expc[11], r, C.expc[10]);
    const double pcd = fma(C.expc[13], r, C.expc[12]);
    const double q03 = fma(p23, r2, p01), q47 = fma(p67, r2, p45), q8b = fma(pab, r2, p89);
    const double q07 = fma(q47, r4, q03), q8d = fma(pcd, r4, q8b);
    const double pz = fma(q8d, r8, q07);
#else
    double pz = C.expc[13];
#pragma unroll
    for (int k = 12; k >= 0; --k) pz = fma(pz, r, C.expc[k]);
#endif
    const long long ni = static_cast<long long>(n);
    return __longlong_as_double(__double_as_longlong(pz) - (ni << 52));
#else
    return std::exp(-z);
#endif
}

// fp32 build (real = float): hardware reciprocal + one Newton step (~1 ulp), hardware exp.
PS_HD float rcp(float a) {
#if defined(__CUDA_ARCH__)
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
    return fmaf(r, fmaf(-a, r, 1.0f), r);
#else
    return 1.0f / a;
#endif
}
template <bool FAST = false>
PS_HD float exp_neg(float z) {
#if defined(__CUDA_ARCH__)
    return __expf(-z);
#else
    return std::exp(-z);
#endif
}

// Model constants the kernels need (kernel parameter, i.e. constant bank).
template <int D>
struct ModelParams {
    real Pinf[ns(D)];   // stationary covariance (balanced coordinates)
    real H[D];          // observation row (balanced coordinates)
    real r;             // observation noise variance sigma_n^2 > 0
    real lam;           // Matern lambda = sqrt(2 nu) / ell (closed form), else 0
    real s2;            // Matern variance sigma^2
    real udt;           // uniform dt (> 0) for which Fu, Qu are valid, else 0
    real Fu[D * D];     // F(udt)
    real Qu[ns(D)];     // Q(udt)
    real G[D * D];      // continuous drift (balanced coordinates), kPade mode
    real W[ns(D)];      // diffusion L q L^T (balanced coordinates), kPade mode
    int closed;           // 1: Matern closed form of order D available in the lambda-scaled basis
    int h_unit;           // 1: H == e_0
};

// ------------------------------------------------------------------ aggregates
template <int D>
struct FAgg {  // filter element / aggregate (A, b, C, eta, J)
    real A[D * D];
    real b[D];
    real C[ns(D)];
    real eta[D];
    real J[ns(D)];
};

template <int D>
struct SAgg {  // smoother element / aggregate (E, g, L)
    real E[D * D];
    real g[D];
    real L[ns(D)];
};

template <int D>
struct Gauss {  // (mean, covariance) — a collapsed global prefix (0, x, P, 0, 0) or suffix (0, m, P)
    real x[D];
    real P[ns(D)];
};

template <int D>
PS_HD void set_identity(FAgg<D>& a) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
#pragma unroll
        for (int j = 0; j < D; ++j) a.A[i * D + j] = (i == j) ? 1.0 : 0.0;
        a.b[i] = 0.0;
        a.eta[i] = 0.0;
    }
#pragma unroll
    for (int i = 0; i < ns(D); ++i) { a.C[i] = 0.0; a.J[i] = 0.0; }
}

template <int D>
PS_HD void set_identity(SAgg<D>& a) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
#pragma unroll
        for (int j = 0; j < D; ++j) a.E[i * D + j] = (i == j) ? 1.0 : 0.0;
        a.g[i] = 0.0;
    }
#pragma unroll
    for (int i = 0; i < ns(D); ++i) a.L[i] = 0.0;
}

template <int D>
PS_HD void set_zero(Gauss<D>& c) {
#pragma unroll
    for (int i = 0; i < D; ++i) c.x[i] = 0.0;
#pragma unroll
    for (int i = 0; i < ns(D); ++i) c.P[i] = 0.0;
}

// flat views for loads / stores / shuffles
template <int D> PS_HD real* flat(FAgg<D>& a) { return a.A; }
template <int D> PS_HD const real* flat(const FAgg<D>& a) { return a.A; }
template <int D> PS_HD real* flat(SAgg<D>& a) { return a.E; }
template <int D> PS_HD const real* flat(const SAgg<D>& a) { return a.E; }
template <int D> PS_HD real* flat(Gauss<D>& a) { return a.x; }
template <int D> PS_HD const real* flat(const Gauss<D>& a) { return a.x; }

// ------------------------------------------------------------------ small dense helpers
// Gaussian elimination with partial pivoting on [M | R] (M D x D row-major,
// R D x NR row-major), solving M X = R in place (X -> R).  Pivot rows are
// chosen by compare-and-swap with compile-time indices only (no dynamic
// register indexing).  Returns false on a zero pivot.
template <int D, int NR>
PS_HD bool gauss_solve(real (&M)[D * D], real (&R)[D * NR]) {
    bool ok = true;
#pragma unroll
    for (int c = 0; c < D; ++c) {
#pragma unroll
        for (int r = c + 1; r < D; ++r) {
            const bool sw = fabs(M[r * D + c]) > fabs(M[c * D + c]);
#pragma unroll
            for (int k = c; k < D; ++k) {
                const real u = M[c * D + k], v = M[r * D + k];
                M[c * D + k] = sw ? v : u;
                M[r * D + k] = sw ? u : v;
            }
#pragma unroll
            for (int k = 0; k < NR; ++k) {
                const real u = R[c * NR + k], v = R[r * NR + k];
                R[c * NR + k] = sw ? v : u;
                R[r * NR + k] = sw ? u : v;
            }
        }
        const real piv = M[c * D + c];
        ok = ok && (piv != 0.0);
        const real ip = rcp(piv);
#pragma unroll
        for (int r = c + 1; r < D; ++r) {
            const real f = M[r * D + c] * ip;
#pragma unroll
            for (int k = c + 1; k < D; ++k) M[r * D + k] = fma(-f, M[c * D + k], M[r * D + k]);
#pragma unroll
            for (int k = 0; k < NR; ++k) R[r * NR + k] = fma(-f, R[c * NR + k], R[r * NR + k]);
        }
        M[c * D + c] = ip;  // keep the reciprocal for back substitution
    }
#pragma unroll
    for (int c = D - 1; c >= 0; --c) {
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            real s = R[c * NR + k];
#pragma unroll
            for (int j = c + 1; j < D; ++j) s = fma(-M[c * D + j], R[j * NR + k], s);
            R[c * NR + k] = s * M[c * D + c];
        }
    }
    return ok;
}

// Inverse of a small D x D matrix (D <= 3) by the adjugate: cofactors in parallel, one
// reciprocal of the determinant — a short dependency chain (no pivot search, no
// compare-and-swap), for the (I + C J) and (I + P J) of the filtering operator, whose
// eigenvalues are >= 1 (C, J, P positive semi-definite).  Returns false
// for a zero or non-finite determinant.
template <int D>
PS_HD bool inv_small(const real (&M)[D * D], real (&Mi)[D * D]) {
    static_assert(D <= 3, "adjugate inverse for D <= 3");
    if constexpr (D == 1) {
        Mi[0] = rcp(M[0]);
        return M[0] != 0.0;
    } else if constexpr (D == 2) {
        const real det = fma(M[0], M[3], -M[1] * M[2]);
        const real id = rcp(det);
        Mi[0] = M[3] * id; Mi[1] = -M[1] * id; Mi[2] = -M[2] * id; Mi[3] = M[0] * id;
        return det != 0.0 && isfinite(id);
    } else {
        const real c00 = fma(M[4], M[8], -M[5] * M[7]);
        const real c01 = fma(M[5], M[6], -M[3] * M[8]);
        const real c02 = fma(M[3], M[7], -M[4] * M[6]);
        const real det = fma(M[0], c00, fma(M[1], c01, M[2] * c02));
        const real id = rcp(det);
        Mi[0] = c00 * id;
        Mi[3] = c01 * id;
        Mi[6] = c02 * id;
        Mi[1] = fma(M[2], M[7], -M[1] * M[8]) * id;
        Mi[4] = fma(M[0], M[8], -M[2] * M[6]) * id;
        Mi[7] = fma(M[1], M[6], -M[0] * M[7]) * id;
        Mi[2] = fma(M[1], M[5], -M[2] * M[4]) * id;
        Mi[5] = fma(M[2], M[3], -M[0] * M[5]) * id;
        Mi[8] = fma(M[0], M[4], -M[1] * M[3]) * id;
        return det != 0.0 && isfinite(id);
    }
}

// Solve M X = R (R: D x NR row-major, in place): adjugate for D <= 3, pivoted elimination above.
template <int D, int NR>
PS_HD bool small_solve(real (&M)[D * D], real (&R)[D * NR]) {
    if constexpr (D <= 3) {
        real Mi[D * D];
        const bool ok = inv_small<D>(M, Mi);
        real X[D * NR];
#pragma unroll
        for (int r = 0; r < D; ++r)
#pragma unroll
            for (int c = 0; c < NR; ++c) {
                real s = 0.0;
#pragma unroll
                for (int k = 0; k < D; ++k) s = fma(Mi[r * D + k], R[k * NR + c], s);
                X[r * NR + c] = s;
            }
#pragma unroll
        for (int i = 0; i < D * NR; ++i) R[i] = X[i];
        return ok;
    } else {
        return gauss_solve<D, NR>(M, R);
    }
}

// LDL^T factorisation of a symmetric positive-definite packed matrix.
// Lo: strictly-lower factor (row-major D x D, only i > j used), id: 1 / d.
template <int D>
PS_HD bool ldlt(const real (&S)[ns(D)], real (&Lo)[D * D], real (&id)[D]) {
    real dd[D];
    bool ok = true;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        real d = S[si(D, j, j)];
#pragma unroll
        for (int k = 0; k < j; ++k) d = fma(-Lo[j * D + k] * dd[k], Lo[j * D + k], d);
        ok = ok && (d > 0.0);
        dd[j] = d;
        id[j] = rcp(d);
#pragma unroll
        for (int i = j + 1; i < D; ++i) {
            real s = S[si(D, i, j)];
#pragma unroll
            for (int k = 0; k < j; ++k) s = fma(-Lo[i * D + k] * dd[k], Lo[j * D + k], s);
            Lo[i * D + j] = s * id[j];
        }
    }
    return ok;
}

// Solve S X = R with the LDL^T factors (R: D x NR row-major, in place).
template <int D, int NR>
PS_HD void ldlt_solve(const real (&Lo)[D * D], const real (&id)[D], real (&R)[D * NR]) {
#pragma unroll
    for (int k = 0; k < NR; ++k) {
#pragma unroll
        for (int i = 1; i < D; ++i) {
            real s = R[i * NR + k];
#pragma unroll
            for (int j = 0; j < i; ++j) s = fma(-Lo[i * D + j], R[j * NR + k], s);
            R[i * NR + k] = s;
        }
#pragma unroll
        for (int i = 0; i < D; ++i) R[i * NR + k] *= id[i];
#pragma unroll
        for (int i = D - 2; i >= 0; --i) {
            real s = R[i * NR + k];
#pragma unroll
            for (int j = i + 1; j < D; ++j) s = fma(-Lo[j * D + i], R[j * NR + k], s);
            R[i * NR + k] = s;
        }
    }
}

// ------------------------------------------------------------------ discretisation
// R_m(x) = e^{-x} sum_{n>=m} x^n / n!  (regularised lower incomplete gamma P(m, x)),
// evaluated without cancellation: truncated series for x <= 2, complement
// 1 - e^{-x} sum_{n<m} x^n/n! above (cancellation <= ~20x there).
template <int M, bool FAST = false>
PS_HD real inc_gamma_tail(real x, real emx) {
    const MathConsts& C = mc();
    real xm;                                    // x^M
    if constexpr (M == 5) {
        const real x2 = x * x;
        xm = x2 * x2 * x;
    } else {
        xm = x;
#pragma unroll
        for (int n = 1; n < M; ++n) xm *= x;
    }
    const real lead = emx * xm;                 // e^{-x} x^M; series coefficients 1/(M+j)!
    if (FAST || x <= real(0.015625)) {   // FAST: caller guarantees 0 <= x <= 2^-6
        real s = C.expc[M + 7];
#pragma unroll
        for (int j = 6; j >= 0; --j) s = fma(s, x, C.expc[M + j]);
        return lead * s;
    } else if (x <= real(0.5)) {
        real s = C.expc[M + 13];
#pragma unroll
        for (int j = 12; j >= 0; --j) s = fma(s, x, C.expc[M + j]);
        return lead * s;
    } else if (x <= real(2.0)) {
        real s = C.expc[M + 22];
#pragma unroll
        for (int j = 21; j >= 0; --j) s = fma(s, x, C.expc[M + j]);
        return lead * s;
    } else {
        real p = 1.0, term = 1.0;
#pragma unroll
        for (int n = 1; n < M; ++n) { term *= x * C.inv[n]; p += term; }
        return fma(-emx, p, real(1.0));
    }
}

// ------------------------------------------------------------------ transitions
// A transition matrix F is passed to the step kernels as one of two types with the same
// interface: F(i, j) reads an element, FT::nz(i, j) is a compile-time "may be nonzero" so
// the fully unrolled products skip structural zeros.
template <int D>
struct FMat {                        // general F (row-major)
    real a[D * D];
    PS_HD real operator()(int i, int j) const { return a[i * D + j]; }
    static PS_HD constexpr bool nz(int, int) { return true; }
};
// Closed-form Matern-(2D-1)/2 in the JORDAN basis of its drift: with x_hat_i = x_i / lambda^i
// the drift is lambda times the companion matrix of (s + 1)^D, which is similar to the single
// Jordan block J = -I + N (N = ones on the superdiagonal) through a unit lower-triangular P
// whose first row is e_0 (DESIGN.md §5 "Jordan basis").  In x~ = P^-1 x_hat the observation
// row stays H = e_0 and
//     F(z) = e^{-z} (I + z N + z^2/2 N^2 + ...),   z = lambda dt,
// an upper-triangular Toeplitz matrix: F(i, j) = ec[j - i] = e^{-z} z^(j-i) / (j-i)!.
template <int D>
struct FJor {
    real ec[D];      // e^{-z} z^k / k!
    real e;          // e^{-z}
    real u[D];       // z^k / k! (u[0] = 1 unused): F = e U
    PS_HD real operator()(int i, int j) const { return j >= i ? ec[j - i] : 0.0; }
    static PS_HD constexpr bool nz(int i, int j) { return j >= i; }
};
template <int D>
PS_HD void set_zero(FMat<D>& f) {
#pragma unroll
    for (int i = 0; i < D * D; ++i) f.a[i] = 0.0;
}
template <int D>
PS_HD void set_zero(FJor<D>& f) {
#pragma unroll
    for (int i = 0; i < D; ++i) { f.ec[i] = 0.0; f.u[i] = 0.0; }
    f.e = 0.0;
}

// F S F^T + Q for symmetric packed S (packed result).  General F: T = F S, then T F^T.
template <int D>
PS_HD void cong_plus(const FMat<D>& F, const real (&S)[ns(D)], const real (&Q)[ns(D)], real (&R)[ns(D)]) {
    real T[D * D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
            real t = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) t = fma(F(i, k), S[si(D, k, j)], t);
            T[i * D + j] = t;
        }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = i; j < D; ++j) {
            real r = Q[si(D, i, j)];
#pragma unroll
            for (int k = 0; k < D; ++k) r = fma(T[i * D + k], F(j, k), r);
            R[si(D, i, j)] = r;
        }
}
// Jordan F = e U (U unit upper-triangular Toeplitz): e^2 (U S U^T) + Q, the unit diagonal and
// the structural zeros of U skipped (D = 3: 13 FMA for U S U^T instead of 45).
template <int D>
PS_HD void cong_plus(const FJor<D>& F, const real (&S)[ns(D)], const real (&Q)[ns(D)], real (&R)[ns(D)]) {
    real X[D * D];   // X = U S
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
            real t = S[si(D, i, j)];
#pragma unroll
            for (int k = i + 1; k < D; ++k) t = fma(F.u[k - i], S[si(D, k, j)], t);
            X[i * D + j] = t;
        }
    const real e2 = F.e * F.e;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = i; j < D; ++j) {
            real y = X[i * D + j];
#pragma unroll
            for (int l = j + 1; l < D; ++l) y = fma(X[i * D + l], F.u[l - j], y);
            R[si(D, i, j)] = fma(e2, y, Q[si(D, i, j)]);
        }
}
template <int D, class FT>
PS_HD FMat<D> to_full(const FT& f) {
    FMat<D> o;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) o.a[i * D + j] = f(i, j);
    return o;
}

// R_m(x) = e^{-x} sum_{n >= m} x^n / n!, m = 1..M, from R_M by R_m = R_{m+1} + e^{-x} x^m / m!
// (every term positive: no cancellation at any x).  R[m] for m = 1..M (R[0] unused).
template <int M, bool FAST = false>
PS_HD void inc_gamma_tails(real x, real emx, real (&R)[M + 1]) {
    const MathConsts& C = mc();
    R[M] = inc_gamma_tail<M, FAST>(x, emx);
    real tm = emx * x;                         // e^{-x} x^1 / 1!
    real t[M + 1];
    t[1] = tm;
#pragma unroll
    for (int m = 2; m < M; ++m) { tm = tm * x * C.inv[m]; t[m] = tm; }
#pragma unroll
    for (int m = M - 1; m >= 1; --m) R[m] = R[m + 1] + t[m];
}

// Matern-(2D-1)/2 closed form in the Jordan basis (above).  With x = 2z and
// W = sigma^2 w e_{D-1} e_{D-1}^T (w = 2, 4, 16/3), Q(z) = sigma^2 w int_0^z e^{-2u} c(u) c(u)^T du,
// c(u) = (u^(D-1)/(D-1)!, ..., u, 1), and int_0^z e^{-2u} u^k du = k! / 2^(k+1) R_{k+1}(x), so
// every entry is a POSITIVE multiple of one R_m (derivation: DESIGN.md §5; pinned against the
// oracle's Van Loan in tests/test_library_host.py):
//   D = 1: Q = s2 R1
//   D = 2: Q00 = s2 R3, Q01 = s2 R2, Q11 = 2 s2 R1
//   D = 3: Q00 = s2 R5, Q01 = s2 R4, Q02 = 2/3 s2 R3, Q11 = 4/3 s2 R3, Q12 = 4/3 s2 R2, Q22 = 8/3 s2 R1
// P_inf = lim Q (R_m -> 1).  FAST: the caller guarantees 0 <= z <= 2^-7.
template <int D, bool FAST = false>
PS_HD void matern_closed(real lam, real s2, double dt, FJor<D>& F, real (&Q)[ns(D)]) {
    const real z = static_cast<real>(lam * dt);
    const real e = exp_neg<FAST>(z);
    const real x = real(2.0) * z;
    const real ex = e * e;  // e^{-x}
    F.e = e;
    F.u[0] = 1.0;
    F.ec[0] = e;
    if constexpr (D >= 2) { F.u[1] = z; F.ec[1] = e * z; }
    if constexpr (D >= 3) { F.u[2] = real(0.5) * z * z; F.ec[2] = e * F.u[2]; }
    if constexpr (D == 1) {
        Q[0] = s2 * inc_gamma_tail<1, FAST>(x, ex);
    } else if constexpr (D == 2) {
        real R[4];
        inc_gamma_tails<3, FAST>(x, ex, R);
        Q[si(2, 0, 0)] = s2 * R[3];
        Q[si(2, 0, 1)] = s2 * R[2];
        Q[si(2, 1, 1)] = (mc().qw[3] * s2) * R[1];
    } else if constexpr (D == 3) {
        real R[6];
        inc_gamma_tails<5, FAST>(x, ex, R);
        const MathConsts& C = mc();
        const real s43 = s2 * C.qw[1];
        Q[si(3, 0, 0)] = s2 * R[5];
        Q[si(3, 0, 1)] = s2 * R[4];
        Q[si(3, 0, 2)] = (s2 * C.qw[0]) * R[3];
        Q[si(3, 1, 1)] = s43 * R[3];
        Q[si(3, 1, 2)] = s43 * R[2];
        Q[si(3, 2, 2)] = (s2 * C.qw[2]) * R[1];
    }
}

// Discretise one step (transition into a step whose predecessor is dt earlier).
// Returns 0, or a nonzero code when the model has no device discretisation for dt.
// MODE (compile time): kClosed = Matern closed form only (dt = 0 gives F = I,
// Q = 0 exactly; any uniform_dt is ignored, the closed form is cheaper than a table
// lookup), kTable = the host-precomputed pair for dt == udt (dt = 0 -> I, 0; anything
// else unsupported), kMixed = retired (closed models always use kClosed),
// kPade = any model, any dt: F = expm(G dt) by scaling and squaring with the
// [7/7] Pade approximant and Q by the Taylor series of the Lyapunov ODE on the same scaled
// step, composed by doubling (taylor_fq; north_star "per-step small-matrix expm via
// scaling-and-squaring Pade").
enum DiscMode : int { kClosed = 0, kTable = 1, kMixed = 2, kPade = 3 };

// F = expm(G dt), D x D row-major.  Higham (2005): the [7/7] Pade approximant is
// accurate to unit roundoff for ||A||_1 <= theta_7 = 0.9504; A = G dt / 2^s with the
// smallest such s, then s squarings.  (V - U) F = V + U by pivoted elimination.
template <int D>
PS_HD void expm_pade7(const real (&G)[D * D], real dt, real (&F)[D * D]) {
    real nrm = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        real c = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) c += fabs(G[i * D + j]);
        nrm = fmax(nrm, c);
    }
    nrm *= fabs(dt);
    int s = 0;
    if (nrm > 0.9504) {
        int e;
        frexp(nrm / 0.9504, &e);   // nrm / theta = f 2^e, f in [0.5, 1)  ->  2^e >= nrm / theta
        s = e;
    }
    const real sc = ldexp(dt, -s);
    real A[D * D], A2[D * D], A4[D * D], A6[D * D];
#pragma unroll
    for (int i = 0; i < D * D; ++i) A[i] = G[i] * sc;
    auto mm = [](const real (&X)[D * D], const real (&Y)[D * D], real (&Z)[D * D]) {
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) {
                real acc = 0.0;
#pragma unroll
                for (int k = 0; k < D; ++k) acc = fma(X[i * D + k], Y[k * D + j], acc);
                Z[i * D + j] = acc;
            }
    };
    mm(A, A, A2);
    mm(A2, A2, A4);
    mm(A4, A2, A6);
    constexpr real b0 = 17297280.0, b1 = 8648640.0, b2 = 1995840.0, b3 = 277200.0, b4 = 25200.0,
                     b5 = 1512.0, b6 = 56.0, b7 = 1.0;
    real T[D * D], U[D * D], V[D * D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const int e = i * D + j;
            const real id = (i == j) ? 1.0 : 0.0;
            T[e] = fma(b7, A6[e], fma(b5, A4[e], fma(b3, A2[e], b1 * id)));
            V[e] = fma(b6, A6[e], fma(b4, A4[e], fma(b2, A2[e], b0 * id)));
        }
    mm(A, T, U);
#pragma unroll
    for (int e = 0; e < D * D; ++e) {
        T[e] = V[e] - U[e];
        F[e] = V[e] + U[e];
    }
    gauss_solve<D, D>(T, F);
    for (int q = 0; q < s; ++q) {
        real Fs[D * D];
        mm(F, F, Fs);
#pragma unroll
        for (int e = 0; e < D * D; ++e) F[e] = Fs[e];
    }
}

// F = e^{G dt} and Q = int_0^dt e^{Gs} W e^{G^T s} ds together, cancellation-free at every dt
// (the stationary shortcut P_inf - F P_inf F^T loses the small entries of Q when ||G dt|| << 1,
// SURVEY A.4): on the scaled step tau = dt / 2^s with ||G tau||_1 <= 1/8,
//   F_tau = [7/7] Pade of e^A,  Q_tau = sum_{k=1..m} Z_k,  A = G tau,
//   Z_1 = tau W,  Z_{k+1} = (A Z_k + Z_k A^T) / (k + 1)      (Taylor series of the Lyapunov ODE),
// m = 12 (truncation (2/8)^m / (m+1)! < 1e-17 relative; m = 7 when ||G dt|| <= 1/100), then s
// doublings Q <- Q + F Q F^T, F <- F F (the semigroup identity, as Van Loan composes sub-steps).
template <int D>
PS_HD void taylor_fq(const real (&G)[D * D], const real (&W)[ns(D)], real dt, real (&F)[D * D],
                     real (&Q)[ns(D)]) {
    real nrm = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        real c = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) c += fabs(G[i * D + j]);
        nrm = fmax(nrm, c);
    }
    nrm *= fabs(dt);
    int s = 0;
    if (nrm > 0.125) {
        int e;
        frexp(nrm / 0.125, &e);
        s = e;
    }
    const real tau = ldexp(dt, -s);
    const int m = (nrm <= 0.01) ? 7 : 12;
    real A[D * D];
#pragma unroll
    for (int i = 0; i < D * D; ++i) A[i] = G[i] * tau;
    // F on the scaled step: [7/7] Pade (||A||_1 <= 1/8 < theta_7: no further scaling)
    real T[D * D];
    expm_pade7<D>(G, tau, F);
    // Q: Z_1 = tau W, Z_{k+1} = (A Z_k + Z_k A^T) / (k + 1)
    real Z[ns(D)];
#pragma unroll
    for (int i = 0; i < ns(D); ++i) { Z[i] = W[i] * tau; Q[i] = Z[i]; }
    for (int k = 1; k < m; ++k) {
        const real ik = 1.0 / (k + 1);
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) {
                real acc = 0.0;
#pragma unroll
                for (int l = 0; l < D; ++l) acc = fma(A[i * D + l], Z[si(D, l, j)], acc);
                T[i * D + j] = acc;                         // Y = A Z
            }
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = i; j < D; ++j) {
                Z[si(D, i, j)] = (T[i * D + j] + T[j * D + i]) * ik;
                Q[si(D, i, j)] += Z[si(D, i, j)];
            }
    }
    // doublings: Q(2t) = Q(t) + F(t) Q(t) F(t)^T, F(2t) = F(t)^2
    for (int q = 0; q < s; ++q) {
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) {
                real acc = 0.0;
#pragma unroll
                for (int l = 0; l < D; ++l) acc = fma(F[i * D + l], Q[si(D, l, j)], acc);
                T[i * D + j] = acc;                         // F Q
            }
        real Qn[ns(D)];
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = i; j < D; ++j) {
                real acc = Q[si(D, i, j)];
#pragma unroll
                for (int l = 0; l < D; ++l) acc = fma(T[i * D + l], F[j * D + l], acc);
                Qn[si(D, i, j)] = acc;
            }
#pragma unroll
        for (int i = 0; i < ns(D); ++i) Q[i] = Qn[i];
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) {
                real acc = 0.0;
#pragma unroll
                for (int l = 0; l < D; ++l) acc = fma(F[i * D + l], F[l * D + j], acc);
                T[i * D + j] = acc;
            }
#pragma unroll
        for (int i = 0; i < D * D; ++i) F[i] = T[i];
    }
}

// transition type of each mode: Jordan-structured for the Matern closed form
template <int D, int MODE>
using FT_t = typename std::conditional<MODE == kClosed, FJor<D>, FMat<D>>::type;

template <int D, int MODE>
PS_HD int disc(const ModelParams<D>& p, double dt, FT_t<D, MODE>& Ft, real (&Q)[ns(D)]) {
    if constexpr (MODE == kClosed) {
        if constexpr (D <= 3) matern_closed<D>(p.lam, p.s2, dt, Ft, Q);
        return 0;
    } else {
        real (&F)[D * D] = Ft.a;
        if (fabs(dt - p.udt) <= 1e-12 * p.udt) {   // uniform step up to time-stamp rounding
#pragma unroll
            for (int i = 0; i < D * D; ++i) F[i] = p.Fu[i];
#pragma unroll
            for (int i = 0; i < ns(D); ++i) Q[i] = p.Qu[i];
            return 0;
        }
        if constexpr (MODE == kPade) {
            if (dt == 0.0) {   // exact I, 0 on ties (reading Z13)
#pragma unroll
                for (int i = 0; i < D; ++i)
#pragma unroll
                    for (int j = 0; j < D; ++j) F[i * D + j] = (i == j) ? 1.0 : 0.0;
#pragma unroll
                for (int i = 0; i < ns(D); ++i) Q[i] = 0.0;
                return 0;
            }
            taylor_fq<D>(p.G, p.W, dt, F, Q);
            return 0;
        } else {
            const bool zero = (dt == 0.0);
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = 0; j < D; ++j) F[i * D + j] = (zero && i == j) ? 1.0 : 0.0;
#pragma unroll
            for (int i = 0; i < ns(D); ++i) Q[i] = 0.0;
            return zero ? 0 : 1;
        }
    }
}

// Host-side dispatcher used by pssgp_debug_discretize.
template <int D>
PS_HD int discretize(const ModelParams<D>& p, double dt, real (&F)[D * D], real (&Q)[ns(D)]) {
    int rc;
    FMat<D> f;
    if (p.closed) {
        FJor<D> fj;
        rc = disc<D, kClosed>(p, dt, fj, Q);
        f = to_full<D>(fj);
    } else {
        rc = p.udt > 0.0 ? disc<D, kTable>(p, dt, f, Q) : disc<D, kPade>(p, dt, f, Q);
    }
#pragma unroll
    for (int i = 0; i < D * D; ++i) F[i] = f.a[i];
    return rc;
}

// ------------------------------------------------------------------ filter fold
// a <- a (x) e_k, where e_k is the raw filter element of step k built from
// (F, Q, y_k, mask_k) (Eqs. (6), (8) PAPER.md:97-112 for a missing y
// for an observed y).  Because J_k = u u^T / S_k has rank one, the operator
// reduces to a Kalman step conditioned on the chain's
// entry state: predict C- = F C F^T + Q, then a rank-one update (no solve).
// For the global first step pass F = 0, Q = P_inf (Eq. (7) PAPER.md:103-107 and
// reading Z1: the observed first element is the KF update of N(0, P_inf)).
template <int D, bool HU = false, class FT>
PS_HD void fold_step(FAgg<D>& a, const FT& F, const real (&Q)[ns(D)],
                     const ModelParams<D>& p, bool obs, real yk) {
    real FA[D * D], Fb[D], Cm[ns(D)];
#pragma unroll
    for (int i = 0; i < D; ++i) {
        real sb = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            real sa = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k)
                if (FT::nz(i, k)) sa = fma(F(i, k), a.A[k * D + j], sa);
            FA[i * D + j] = sa;
            if (FT::nz(i, j)) sb = fma(F(i, j), a.b[j], sb);
        }
        Fb[i] = sb;
    }
    cong_plus<D>(F, a.C, Q, Cm);
    // observation update; branchless: a missing y (Eqs. (6), (8)) is the same
    // formulas with 1/S and the innovation set to zero (A = F A, b = F b, C = C-)
    real HC[D], w[D], hb, S;
    if (HU || p.h_unit) {
#pragma unroll
        for (int i = 0; i < D; ++i) { HC[i] = Cm[si(D, i, 0)]; w[i] = FA[i]; }
        hb = Fb[0];
        S = Cm[0] + p.r;
    } else {
        hb = 0.0; S = p.r;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            real s = 0.0, ww = 0.0;
#pragma unroll
            for (int j = 0; j < D; ++j) {
                s = fma(Cm[si(D, i, j)], p.H[j], s);
                ww = fma(p.H[j], FA[j * D + i], ww);
            }
            HC[i] = s; w[i] = ww;
            hb = fma(p.H[i], Fb[i], hb);
        }
#pragma unroll
        for (int i = 0; i < D; ++i) S = fma(p.H[i], HC[i], S);
    }
    const real iS = obs ? rcp(S) : 0.0;
    const real v = obs ? (yk - hb) : 0.0;
    const real vs = v * iS;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        const real Kc = HC[i] * iS;
#pragma unroll
        for (int j = 0; j < D; ++j) a.A[i * D + j] = fma(-Kc, w[j], FA[i * D + j]);
        a.b[i] = fma(HC[i], vs, Fb[i]);
        a.eta[i] = fma(w[i], vs, a.eta[i]);
    }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = i; j < D; ++j) {
            a.C[si(D, i, j)] = fma(-HC[i] * iS, HC[j], Cm[si(D, i, j)]);
            a.J[si(D, i, j)] = fma(w[i] * iS, w[j], a.J[si(D, i, j)]);
        }
}

// ------------------------------------------------------------------ general filtering operator
// (A,b,C,eta,J)_i (x) (A,b,C,eta,J)_j, with solves against
// (I + C_i J_j) and (I + J_j C_i) (never explicit inverses).
template <int D>
PS_HD bool combine(const FAgg<D>& ei, const FAgg<D>& ej, FAgg<D>& out) {
    constexpr int NX = 2 * D + 1, NY = D + 1;
    real M[D * D], MT[D * D], X[D * NX], Y[D * NY];
#pragma unroll
    for (int r = 0; r < D; ++r) {
#pragma unroll
        for (int c = 0; c < D; ++c) {
            real s = (r == c) ? 1.0 : 0.0, st = s;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                s = fma(ei.C[si(D, r, k)], ej.J[si(D, k, c)], s);     // (I + C_i J_j)
                st = fma(ej.J[si(D, r, k)], ei.C[si(D, k, c)], st);   // (I + J_j C_i)
            }
            M[r * D + c] = s;
            MT[r * D + c] = st;
        }
        // X rhs = [A_i | b_i + C_i eta_j | C_i]
#pragma unroll
        for (int c = 0; c < D; ++c) X[r * NX + c] = ei.A[r * D + c];
        real s = ei.b[r];
#pragma unroll
        for (int k = 0; k < D; ++k) s = fma(ei.C[si(D, r, k)], ej.eta[k], s);
        X[r * NX + D] = s;
#pragma unroll
        for (int c = 0; c < D; ++c) X[r * NX + D + 1 + c] = ei.C[si(D, r, c)];
        // Y rhs = [J_j A_i | eta_j - J_j b_i]
#pragma unroll
        for (int c = 0; c < D; ++c) {
            real u = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) u = fma(ej.J[si(D, r, k)], ei.A[k * D + c], u);
            Y[r * NY + c] = u;
        }
        real e = ej.eta[r];
#pragma unroll
        for (int k = 0; k < D; ++k) e = fma(-ej.J[si(D, r, k)], ei.b[k], e);
        Y[r * NY + D] = e;
    }
#if PSSGP_PIVOTED_COMBINE
    bool ok = gauss_solve<D, NX>(M, X);
    ok = gauss_solve<D, NY>(MT, Y) && ok;
#else
    bool ok;
    if constexpr (D <= 3) {
        // (I + J_j C_i) = (I + C_i J_j)^T (C, J symmetric): one inverse serves both solves
        real Mi[D * D], Xo[D * NX], Yo[D * NY];
        ok = inv_small<D>(M, Mi);
#pragma unroll
        for (int r = 0; r < D; ++r) {
#pragma unroll
            for (int c = 0; c < NX; ++c) {
                real t = 0.0;
#pragma unroll
                for (int k = 0; k < D; ++k) t = fma(Mi[r * D + k], X[k * NX + c], t);
                Xo[r * NX + c] = t;
            }
#pragma unroll
            for (int c = 0; c < NY; ++c) {
                real t = 0.0;
#pragma unroll
                for (int k = 0; k < D; ++k) t = fma(Mi[k * D + r], Y[k * NY + c], t);
                Yo[r * NY + c] = t;
            }
        }
#pragma unroll
        for (int i = 0; i < D * NX; ++i) X[i] = Xo[i];
#pragma unroll
        for (int i = 0; i < D * NY; ++i) Y[i] = Yo[i];
    } else {
        ok = gauss_solve<D, NX>(M, X);
        ok = gauss_solve<D, NY>(MT, Y) && ok;
    }
#endif
    // A_ij = A_j X_A ; b_ij = A_j X_b + b_j ; C_ij = A_j X_C A_j^T + C_j
    real AX[D * D];
#pragma unroll
    for (int r = 0; r < D; ++r) {
        real sb = ej.b[r];
#pragma unroll
        for (int c = 0; c < D; ++c) {
            real sa = 0.0, sc = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                sa = fma(ej.A[r * D + k], X[k * NX + c], sa);
                sc = fma(ej.A[r * D + k], X[k * NX + D + 1 + c], sc);
            }
            out.A[r * D + c] = sa;
            AX[r * D + c] = sc;
        }
#pragma unroll
        for (int k = 0; k < D; ++k) sb = fma(ej.A[r * D + k], X[k * NX + D], sb);
        out.b[r] = sb;
    }
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = r; c < D; ++c) {
            real s = ej.C[si(D, r, c)];
#pragma unroll
            for (int k = 0; k < D; ++k) s = fma(AX[r * D + k], ej.A[c * D + k], s);
            out.C[si(D, r, c)] = s;
        }
    // eta_ij = A_i^T Y_eta + eta_i ; J_ij = A_i^T Y_J + J_i
#pragma unroll
    for (int r = 0; r < D; ++r) {
        real se = ei.eta[r];
#pragma unroll
        for (int k = 0; k < D; ++k) se = fma(ei.A[k * D + r], Y[k * NY + D], se);
        out.eta[r] = se;
#pragma unroll
        for (int c = r; c < D; ++c) {
            real s = ei.J[si(D, r, c)];
#pragma unroll
            for (int k = 0; k < D; ++k) s = fma(ei.A[k * D + r], Y[k * NY + c], s);
            out.J[si(D, r, c)] = s;
        }
    }
    return ok;
}

// Collapsed global prefix (0, x, P, 0, 0) (x) aggregate (A, b, C, eta, J):
// x' = A (I + P J)^-1 (x + P eta) + b,  P' = A (I + P J)^-1 P A^T + C.
template <int D>
PS_HD bool apply_prefix(const Gauss<D>& g, const FAgg<D>& a, Gauss<D>& out) {
    constexpr int NX = D + 1;
    real M[D * D], X[D * NX];
#pragma unroll
    for (int r = 0; r < D; ++r) {
        real s0 = g.x[r];
#pragma unroll
        for (int c = 0; c < D; ++c) {
            real s = (r == c) ? 1.0 : 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) s = fma(g.P[si(D, r, k)], a.J[si(D, k, c)], s);
            M[r * D + c] = s;
            X[r * NX + c] = g.P[si(D, r, c)];
            s0 = fma(g.P[si(D, r, c)], a.eta[c], s0);
        }
        X[r * NX + D] = s0;
    }
#if PSSGP_PIVOTED_COMBINE
    const bool ok = gauss_solve<D, NX>(M, X);
#else
    const bool ok = small_solve<D, NX>(M, X);
#endif
    real AX[D * D];
#pragma unroll
    for (int r = 0; r < D; ++r) {
        real sx = a.b[r];
#pragma unroll
        for (int c = 0; c < D; ++c) {
            real s = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) s = fma(a.A[r * D + k], X[k * NX + c], s);
            AX[r * D + c] = s;
        }
#pragma unroll
        for (int k = 0; k < D; ++k) sx = fma(a.A[r * D + k], X[k * NX + D], sx);
        out.x[r] = sx;
    }
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = r; c < D; ++c) {
            real s = a.C[si(D, r, c)];
#pragma unroll
            for (int k = 0; k < D; ++k) s = fma(AX[r * D + k], a.A[c * D + k], s);
            out.P[si(D, r, c)] = s;
        }
    return ok;
}

// ------------------------------------------------------------------ smoothing operator
// (E,g,L)_i (x) (E,g,L)_j = (E_i E_j, E_i g_j + g_i, E_i L_j E_i^T + L_i), i earlier.
template <int D>
PS_HD void combine(const SAgg<D>& ei, const SAgg<D>& ej, SAgg<D>& out) {
    real EL[D * D];
#pragma unroll
    for (int r = 0; r < D; ++r) {
        real sg = ei.g[r];
#pragma unroll
        for (int c = 0; c < D; ++c) {
            real se = 0.0, sl = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                se = fma(ei.E[r * D + k], ej.E[k * D + c], se);
                sl = fma(ei.E[r * D + k], ej.L[si(D, k, c)], sl);
            }
            out.E[r * D + c] = se;
            EL[r * D + c] = sl;
            sg = fma(ei.E[r * D + c], ej.g[c], sg);
        }
        out.g[r] = sg;
    }
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = r; c < D; ++c) {
            real s = ei.L[si(D, r, c)];
#pragma unroll
            for (int k = 0; k < D; ++k) s = fma(EL[r * D + k], ei.E[c * D + k], s);
            out.L[si(D, r, c)] = s;
        }
}

// Aggregate (E, g, L) (x) collapsed global suffix (0, m, P) = (0, E m + g, E P E^T + L).
template <int D>
PS_HD void apply_suffix(const SAgg<D>& a, const Gauss<D>& s, Gauss<D>& out) {
    real EP[D * D];
#pragma unroll
    for (int r = 0; r < D; ++r) {
        real sx = a.g[r];
#pragma unroll
        for (int c = 0; c < D; ++c) {
            real t = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) t = fma(a.E[r * D + k], s.P[si(D, k, c)], t);
            EP[r * D + c] = t;
            sx = fma(a.E[r * D + c], s.x[c], sx);
        }
        out.x[r] = sx;
    }
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = r; c < D; ++c) {
            real t = a.L[si(D, r, c)];
#pragma unroll
            for (int k = 0; k < D; ++k) t = fma(EP[r * D + k], a.E[c * D + k], t);
            out.P[si(D, r, c)] = t;
        }
}

// ------------------------------------------------------------------ Kalman step (supplement PAPER.md:304-315)
// Predict: xm = F x, FP = F P, Pm = FP F^T + Q.
template <int D, class FT>
PS_HD void kf_predict(const real (&x)[D], const real (&P)[ns(D)], const FT& F,
                      const real (&Q)[ns(D)], real (&xm)[D], real (&FP)[D * D], real (&Pm)[ns(D)]) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
        real sx = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            real s = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k)
                if (FT::nz(i, k)) s = fma(F(i, k), P[si(D, k, j)], s);
            FP[i * D + j] = s;
            if (FT::nz(i, j)) sx = fma(F(i, j), x[j], sx);
        }
        xm[i] = sx;
    }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = i; j < D; ++j) {
            real s = Q[si(D, i, j)];
#pragma unroll
            for (int k = 0; k < D; ++k)
                if (FT::nz(j, k)) s = fma(FP[i * D + k], F(j, k), s);
            Pm[si(D, i, j)] = s;
        }
}

// Predict without F P: xm = F x, Pm = F P F^T + Q (the structured congruence for Jordan F).
template <int D, class FT>
PS_HD void kf_predict_pm(const real (&x)[D], const real (&P)[ns(D)], const FT& F, const real (&Q)[ns(D)],
                         real (&xm)[D], real (&Pm)[ns(D)]) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
        real sx = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j)
            if (FT::nz(i, j)) sx = fma(F(i, j), x[j], sx);
        xm[i] = sx;
    }
    cong_plus<D>(F, P, Q, Pm);
}

// Sm = Sg F^T (general Sg)
template <int D, class FT>
PS_HD void mul_bt(const real (&Sg)[D * D], const FT& F, real (&Sm)[D * D]) {
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
            real s = 0.0;
#pragma unroll
            for (int l = 0; l < D; ++l)
                if (FT::nz(j, l)) s = fma(Sg[i * D + l], F(j, l), s);
            Sm[i * D + j] = s;
        }
}

// ------------------------------------------------------------------ SPD solve
// Solve S X = R for symmetric positive-definite packed S.  D <= 3: cofactor
// (adjugate) inverse with ONE reciprocal (short dependency chain; relative
// error ~ cond(S) eps, cond(P-) ~ 2e4 on the metric workload); larger D: LDL^T.
template <int D, int NR>
PS_HD bool spd_solve(const real (&S)[ns(D)], real (&R)[D * NR]) {
    if constexpr (D == 1) {
        const bool ok = S[0] > 0.0;
        const real i0 = rcp(S[0]);
#pragma unroll
        for (int k = 0; k < NR; ++k) R[k] *= i0;
        return ok;
    } else if constexpr (D == 2) {
        const real a = S[0], b = S[1], d = S[2];
        const real det = fma(a, d, -b * b);
        const bool ok = (a > 0.0) && (det > 0.0);
        const real id = rcp(det);
        const real i00 = d * id, i01 = -b * id, i11 = a * id;
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            const real r0 = R[k], r1 = R[NR + k];
            R[k] = fma(i00, r0, i01 * r1);
            R[NR + k] = fma(i01, r0, i11 * r1);
        }
        return ok;
    } else if constexpr (D == 3) {
        const real a = S[0], b = S[1], c = S[2], d = S[3], e = S[4], f = S[5];
        const real A00 = fma(d, f, -e * e), A01 = fma(c, e, -b * f), A02 = fma(b, e, -c * d);
        const real A11 = fma(a, f, -c * c), A12 = fma(b, c, -a * e), A22 = fma(a, d, -b * b);
        const real det = fma(a, A00, fma(b, A01, c * A02));
        const bool ok = (a > 0.0) && (A22 > 0.0) && (det > 0.0);
        const real id = rcp(det);
        const real i00 = A00 * id, i01 = A01 * id, i02 = A02 * id, i11 = A11 * id, i12 = A12 * id, i22 = A22 * id;
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            const real r0 = R[k], r1 = R[NR + k], r2 = R[2 * NR + k];
            R[k] = fma(i00, r0, fma(i01, r1, i02 * r2));
            R[NR + k] = fma(i01, r0, fma(i11, r1, i12 * r2));
            R[2 * NR + k] = fma(i02, r0, fma(i12, r1, i22 * r2));
        }
        return ok;
    } else {
        real Lo[D * D], id[D];
        const bool ok = ldlt<D>(S, Lo, id);
        ldlt_solve<D, NR>(Lo, id, R);
        return ok;
    }
}

// ------------------------------------------------------------------ chain smoother aggregate
// The ordered product (x)_s of the smoother elements of steps k0..k1 is the
// Gaussian conditional p(x_k0 | x_{k1+1}, y_1:k1) (each element is
// p(x_k | x_{k+1}, y_1:k), reading Z2; Markov property).  With the chain-entry
// moments conditioned on the whole chain, x0 = E[x_k0 | y_1:k1] and
// P0 = Cov(x_k0 | y_1:k1), the cross-covariance Sm = Cov(x_k0, x_{k1+1} | y_1:k1)
// and the predicted (xm, Pm) of step k1+1 it is
//   E = Sm Pm^-1,  g = x0 - E xm,  L = P0 - E Sm^T.
template <int D>
PS_HD bool chain_smoother_agg(const real (&x0)[D], const real (&P0)[ns(D)], const real (&Sm)[D * D],
                              const real (&xm)[D], const real (&Pm)[ns(D)], SAgg<D>& out) {
    real Et[D * D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) Et[i * D + j] = Sm[j * D + i];
    const bool ok = spd_solve<D, D>(Pm, Et);  // Et = Pm^-1 Sm^T = E^T
#pragma unroll
    for (int i = 0; i < D; ++i) {
        real s = x0[i];
#pragma unroll
        for (int j = 0; j < D; ++j) {
            out.E[i * D + j] = Et[j * D + i];
            s = fma(-Et[j * D + i], xm[j], s);
        }
        out.g[i] = s;
    }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = i; j < D; ++j) {
            real s = P0[si(D, i, j)];
#pragma unroll
            for (int k = 0; k < D; ++k) s = fma(-Et[k * D + i], Sm[j * D + k], s);
            out.L[si(D, i, j)] = s;
        }
    return ok;
}

// ------------------------------------------------------------------ RTS step
// Given the filtered (x, P) at k, the predicted (xm, Pm) at k+1, FP = F P, and the
// smoothed (ms, Ps) at k+1, overwrite (ms, Ps) with the smoothed moments at k.
// G_k = P F^T Pm^-1 via an LDL^T solve of Pm G_k^T = F P.
template <int D>
PS_HD bool rts_step(const real (&x)[D], const real (&P)[ns(D)], const real (&xm)[D],
                    const real (&Pm)[ns(D)], const real (&FP)[D * D], real (&ms)[D],
                    real (&Ps)[ns(D)]) {
    real Gt[D * D];
#pragma unroll
    for (int i = 0; i < D * D; ++i) Gt[i] = FP[i];
    const bool ok = spd_solve<D, D>(Pm, Gt);   // Gt = Pm^-1 F P = G^T, G[i][j] = Gt[j][i]
    real dm[D], T[D * D];
#pragma unroll
    for (int i = 0; i < D; ++i) dm[i] = ms[i] - xm[i];
#pragma unroll
    for (int i = 0; i < D; ++i) {
        real s = x[i];
#pragma unroll
        for (int j = 0; j < D; ++j) s = fma(Gt[j * D + i], dm[j], s);
        ms[i] = s;
    }
    // T = G (Ps - Pm)
    real dP[ns(D)];
#pragma unroll
    for (int i = 0; i < ns(D); ++i) dP[i] = Ps[i] - Pm[i];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
            real s = Gt[i] * dP[si(D, 0, j)];
#pragma unroll
            for (int k = 1; k < D; ++k) s = fma(Gt[k * D + i], dP[si(D, k, j)], s);
            T[i * D + j] = s;
        }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = i; j < D; ++j) {
            real s = P[si(D, i, j)];
#pragma unroll
            for (int k = 0; k < D; ++k) s = fma(T[i * D + k], Gt[k * D + j], s);
            Ps[si(D, i, j)] = s;
        }
    return ok;
}

}  // namespace PSSGP_NS
