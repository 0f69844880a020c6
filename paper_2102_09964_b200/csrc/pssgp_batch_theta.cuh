// pssgp_batch_theta.cuh — batched independent series, each with its OWN log hyper-parameters, for
// sums of Matern, periodic and quasi-periodic components on uniform grids (SURVEY.md §8(f) row 2
// widened: the paper's HMC chains / multi-start fits on the CO2 model C_Per x C_Mat + C_Mat,
// PAPER.md:206-209, 224-235).
//
// Per series b the model at theta_b and its derivatives are closed forms in the device basis of the
// base model (Matern blocks in the Jordan basis of the drift, periodic blocks as rotations), so no
// matrix exponential is needed:
//   Matern(nu, s2, ell), lambda = sqrt(2 nu) / ell:  F = e^{-z} U(z) (z = lambda dt), Q, P_inf = s2 P1
//     (pssgp_math.cuh matern_closed); G = lambda (-I + N), W = lambda s2 w e e^T
//   periodic(J, s2, ell, p): F_j = rotation by j w0 dt (w0 = 2 pi / p), Q = 0, P_inf_j = q_j^2 I,
//     q_j^2 = (2 - [j = 0]) s2 I_j(ell^-2) e^{-ell^-2}
//   quasi-periodic: F = F_p (x) F_m, Q = P_p (x) Q_m (rotations leave P_p = q_j^2 I invariant),
//     P_inf = P_p (x) P_m
// and with the basis held constant (reading Z27): d/dlog s2 scales (Q, P_inf) [W, P_inf]; a time
// scale tau (Matern ell, period, the product's Matern ell) gives dF = -(G_tau dt) F with G_tau the
// part of G it scales (commuting with F), dQ = -dt F W_tau F^T (Q(dt) = Q_0(dt tau_0 / tau)); the
// periodic lengthscale moves only the Bessel weights.  One warp per series then runs the sequential
// Kalman filter + RTS smoother (posterior) or the filter + reverse-mode adjoint (NLL gradient) of
// its series — series share nothing, so no scan is needed (supplement PAPER.md:285-324, 422-430).
#pragma once
#include "pssgp_wide.cuh"

namespace pssgp {
namespace wide {

// NW warps per series (NT = 32 NW threads).  Thread-strided loops with a trip count that is the
// same in every thread (the guard, not the loop, diverges): ptxas 12.9 dropped the end-of-step
// __syncwarp of a one-warp series loop whose last inner loop had lane-dependent trip counts (D * D
// > 32) without re-converging the warp, and lanes that finished early read half-updated shared
// state.  Loops over D (<= 20) elements run in warp 0 only.
#define BT_EACH(v, n) \
    for (int v##_0 = 0; v##_0 < (n); v##_0 += NT) \
        if (const int v = v##_0 + tid; v < (n))

template <int NW>
__device__ __forceinline__ void bsync() {
    if constexpr (NW == 1) __syncwarp();
    else __syncthreads();
}

// Out = op(A) op(B) (+ Cadd) by the series' NT threads, shared operands (Out aliases neither A nor
// B).  D * D > NT: the threads form an (NT / 8) x 8 grid and each holds a register tile of RB
// contiguous rows x CB columns strided by 8 (RB = ceil(D / (NT / 8)), CB = ceil(D / 8); 2 x 3 at
// D = 18, NW = 4): RB + CB shared loads per RB * CB FMAs instead of 2 per FMA; edge threads clamp
// their loads and skip their stores.
template <int D, int NW, bool TA = false, bool TB = false>
__device__ __forceinline__ void bmm(double (*Out)[LD(D)], const double (*A)[LD(D)], const double (*B)[LD(D)],
                                    const double (*Cadd)[LD(D)], int tid) {
    constexpr int NT = 32 * NW;
    if constexpr (D * D <= NT) {
        BT_EACH(e, D * D) {
            const int i = e / D, j = e - (e / D) * D;
            double s = Cadd ? Cadd[i][j] : 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) s = fma(TA ? A[k][i] : A[i][k], TB ? B[j][k] : B[k][j], s);
            Out[i][j] = s;
        }
    } else {
        constexpr int PC = 8, PR = NT / PC, RB = (D + PR - 1) / PR, CB = (D + PC - 1) / PC;
        const int i0 = (tid / PC) * RB, pc = tid % PC;
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

template <int D>
__device__ __forceinline__ double bdot(const double* a, const double* b, int lane) {   // in every warp
    static_assert(D <= 32, "one element per lane");
    const double s = lane < D ? a[lane] * b[lane] : 0.0;
    return wsum(s);
}

enum : int { kBcMatern = 1, kBcPeriodic = 2, kBcQuasi = 3 };
struct BComp {
    int kind, order, nu2, off, size, par;   // order: harmonics J; nu2: 2 nu of the Matern (factor)
};
constexpr int kBMaxComp = 16;
struct BModelDesc {
    int nc, npar, d;
    double udt;
    BComp c[kBMaxComp];
};
// per-series model record: F, Q, P_inf (d x d row-major), then (npar - 1) x (dF, dQ, dP_inf), then r
PS_CX int BREC(int D, int npar) { return (3 + 3 * (npar - 1)) * D * D + 1; }

__device__ inline double b_ive(int j, double a) {   // I_j(a) e^{-a}, power series
    double term = 1.0;
    for (int k = 1; k <= j; ++k) term *= (a / 2.0) / k;
    double sum = 0.0;
    const double q = a * a / 4.0;
    for (int m = 0; m < 2000; ++m) {
        sum += term;
        term *= q / ((m + 1.0) * (m + 1.0 + j));
        if (term < sum * 1e-18 && m > a) break;
    }
    return sum * exp(-a);
}
__device__ inline double b_ive_dloga(int j, double a) {   // d (I_j(a) e^{-a}) / d log a
    return a * (0.5 * (b_ive(j == 0 ? 1 : j - 1, a) + b_ive(j + 1, a)) - b_ive(j, a));
}

// one Matern block of size m in the Jordan basis: F, Q, P_inf, G, W (m x m row-major, local)
template <int M>
__device__ void b_matern(double lam, double s2, double dt, double* F, double* Q, double* P, double* G, double* W) {
    FJor<M> fj;
    double qp[ns(M)];
    matern_closed<M, false>(lam, s2, dt, fj, qp);
    const double P1[3][9] = {{1.0}, {1.0, 1.0, 1.0, 2.0},
                             {1.0, 1.0, 2.0 / 3.0, 1.0, 4.0 / 3.0, 4.0 / 3.0, 2.0 / 3.0, 4.0 / 3.0, 8.0 / 3.0}};
    const double w = (M == 1) ? 2.0 : (M == 2) ? 4.0 : 16.0 / 3.0;
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < M; ++j) {
            F[i * M + j] = fj(i, j);
            Q[i * M + j] = qp[si(M, i, j)];
            P[i * M + j] = s2 * P1[M - 1][i * M + j];
            G[i * M + j] = (i == j) ? -lam : ((j == i + 1) ? lam : 0.0);
            W[i * M + j] = (i == M - 1 && j == M - 1) ? lam * s2 * w : 0.0;
        }
}
__device__ inline void b_matern_any(int m, double lam, double s2, double dt, double* F, double* Q, double* P, double* G,
                                    double* W) {
    if (m == 1) b_matern<1>(lam, s2, dt, F, Q, P, G, W);
    else if (m == 2) b_matern<2>(lam, s2, dt, F, Q, P, G, W);
    else b_matern<3>(lam, s2, dt, F, Q, P, G, W);
}

// The series model record at log hyper-parameters th (one thread; model-build O(d^2) per parameter).
template <int D>
__device__ void b_build(const BModelDesc& md, const double* th, double* rec) {
    const int dd = D * D;
    double* F = rec;
    double* Q = rec + dd;
    double* P = rec + 2 * dd;
    double* der = rec + 3 * dd;
    for (int e = 0; e < (3 + 3 * (md.npar - 1)) * dd; ++e) rec[e] = 0.0;
    const double dt = md.udt;
    for (int ci = 0; ci < md.nc; ++ci) {
        const BComp& c = md.c[ci];
        const int o = c.off, n = c.size, p0 = c.par;
        const double s2 = exp(th[p0]), ell = exp(th[p0 + 1]);
        auto at = [&](double* base, int i, int j) -> double& { return base[(o + i) * D + o + j]; };
        auto dF = [&](int pp) { return der + (3 * pp) * dd; };
        auto dQ = [&](int pp) { return der + (3 * pp + 1) * dd; };
        auto dP = [&](int pp) { return der + (3 * pp + 2) * dd; };
        if (c.kind == kBcMatern) {
            double f[9], q[9], pp_[9], g[9], w[9];
            const double lam = sqrt(static_cast<double>(c.nu2)) / ell;
            b_matern_any(n, lam, s2, dt, f, q, pp_, g, w);
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j) {
                    at(F, i, j) = f[i * n + j];
                    at(Q, i, j) = q[i * n + j];
                    at(P, i, j) = pp_[i * n + j];
                    at(dQ(p0), i, j) = q[i * n + j];              // log variance
                    at(dP(p0), i, j) = pp_[i * n + j];
                    double gf = 0.0, fwf = 0.0;                   // log lengthscale: -(G dt) F, -dt F W F^T
                    for (int k = 0; k < n; ++k) gf += g[i * n + k] * f[k * n + j];
                    for (int k = 0; k < n; ++k)
                        for (int l = 0; l < n; ++l) fwf += f[i * n + k] * w[k * n + l] * f[j * n + l];
                    at(dF(p0 + 1), i, j) = -dt * gf;
                    at(dQ(p0 + 1), i, j) = -dt * fwf;
                }
        } else {
            // periodic part (harmonics j = 0..J, 2 x 2 blocks)
            const int J = c.order;
            const double per = exp(th[p0 + 2]);
            const double w0 = 2.0 * 3.14159265358979323846 / per, a = 1.0 / (ell * ell);
            const int m = (c.kind == kBcQuasi) ? (c.nu2 + 1) / 2 : 1;   // Kronecker factor size
            double fm[9] = {1.0}, qm[9] = {0.0}, pm[9] = {1.0}, gm[9] = {0.0}, wm[9] = {0.0};
            double mell = 1.0;
            if (c.kind == kBcQuasi) {
                mell = exp(th[p0 + 3]);
                b_matern_any(m, sqrt(static_cast<double>(c.nu2)) / mell, 1.0, dt, fm, qm, pm, gm, wm);
            }
            for (int jh = 0; jh <= J; ++jh) {
                const double q2 = (jh == 0 ? 1.0 : 2.0) * s2 * b_ive(jh, a);
                const double dq2 = (jh == 0 ? 1.0 : 2.0) * s2 * b_ive_dloga(jh, a) * (-2.0);   // d / dlog ell
                const double cs = cos(jh * w0 * dt), sn = sin(jh * w0 * dt);
                const double fp[4] = {cs, -sn, sn, cs};
                const double gp[4] = {0.0, -jh * w0, jh * w0, 0.0};
                for (int a1 = 0; a1 < 2; ++a1)
                    for (int b1 = 0; b1 < 2; ++b1) {
                        const double pp_ = (a1 == b1) ? q2 : 0.0, dpp = (a1 == b1) ? dq2 : 0.0;
                        double gfp = 0.0;
                        for (int k = 0; k < 2; ++k) gfp += gp[a1 * 2 + k] * fp[k * 2 + b1];
                        for (int i2 = 0; i2 < m; ++i2)
                            for (int j2 = 0; j2 < m; ++j2) {
                                const int i = (2 * jh + a1) * m + i2, j = (2 * jh + b1) * m + j2;
                                const double fmv = fm[i2 * m + j2];
                                at(F, i, j) = fp[a1 * 2 + b1] * fmv;
                                at(Q, i, j) = pp_ * qm[i2 * m + j2];
                                at(P, i, j) = pp_ * pm[i2 * m + j2];
                                at(dQ(p0), i, j) = pp_ * qm[i2 * m + j2];              // log variance
                                at(dP(p0), i, j) = pp_ * pm[i2 * m + j2];
                                at(dQ(p0 + 1), i, j) = dpp * qm[i2 * m + j2];           // log lengthscale
                                at(dP(p0 + 1), i, j) = dpp * pm[i2 * m + j2];
                                at(dF(p0 + 2), i, j) = -dt * gfp * fmv;                 // log period
                                if (c.kind == kBcQuasi) {                               // log Matern ell
                                    double gfm = 0.0, fwf = 0.0;
                                    for (int k = 0; k < m; ++k) gfm += gm[i2 * m + k] * fm[k * m + j2];
                                    for (int k = 0; k < m; ++k)
                                        for (int l = 0; l < m; ++l) fwf += fm[i2 * m + k] * wm[k * m + l] * fm[j2 * m + l];
                                    at(dF(p0 + 3), i, j) = -dt * fp[a1 * 2 + b1] * gfm;
                                    at(dQ(p0 + 3), i, j) = -dt * pp_ * fwf;
                                }
                            }
                    }
            }
        }
    }
    rec[(3 + 3 * (md.npar - 1)) * dd] = exp(th[md.npar - 1]);   // noise variance
}

template <int D>
__global__ void __launch_bounds__(128) kb_build(const BModelDesc md, int nseg, const double* __restrict__ theta,
                                                double* recs) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nseg) return;
    b_build<D>(md, theta + static_cast<int64_t>(b) * md.npar, recs + static_cast<int64_t>(b) * BREC(D, md.npar));
}

// ------------------------------------------------------------------ one warp per series
struct BParamsT {
    const int64_t* off;     // series b = steps [off[b], off[b+1])
    int nseg, npar;
    double udt;
    const double* recs;     // per-series model records (kb_build)
    const double* t;
    const double* y;
    const uint8_t* mask;
    double* xs;             // filtered (x, P packed) per step, CNW doubles (global scratch)
    double* mean;
    double* var;
    double* nll;            // [nseg]
    double* grad;           // [nseg][npar]
    unsigned long long* err;
};

template <int D>
struct BSmem {
    struct PerWarp {
        double F[D][LD(D)], Q[D][LD(D)], Pinf[D][LD(D)];
        double P[D][LD(D)], FP[D][LD(D)], Pm[D][LD(D)], T[D][LD(D)], C[D][LD(D)], Cm[D][LD(D)], Z[D][LD(D)],
            Cs[D][LD(D)];
        double x[D], xm[D], HP[D], K[D], b[D], bm[D], CK[D], KT[D], Mb[D], dm[D];
    } w[1];
};

// step kind inside a series: 3 = series start (x^- = 0, P^- = P_inf), 0 = uniform step, 1 = dt = 0
__device__ __forceinline__ int b_kind(const BParamsT& q, int64_t k, int64_t s0, double tk) {
    if (k == s0) return 3;
    const double dt = tk - __ldg(q.t + k - 1);
    if (dt == 0.0) return 1;
    if (fabs(dt - q.udt) <= 1e-12 * q.udt) return 0;
    return 2;
}

// Kalman filter over one series (warp-cooperative), storing the filtered moments; returns its NLL.
template <int D, int NW>
__device__ double b_filter(const BParamsT& q, typename BSmem<D>::PerWarp& W, const double* H, double r, int64_t s0,
                           int64_t s1, int tid) {
    constexpr int NT = 32 * NW;
    const int lane = tid & 31;
    double quad = 0.0, logs = 0.0;
    int nobs = 0;
    BT_EACH(i, D) W.x[i] = 0.0;
    BT_EACH(e, D * D) W.P[e / D][e % D] = 0.0;
    bsync<NW>();
    for (int64_t k = s0; k < s1; ++k) {
        const double tk = __ldg(q.t + k);
        const bool obs = __ldg(q.mask + k) != 0;
        const double yk = obs ? __ldg(q.y + k) : 0.0;
        const int kind = b_kind(q, k, s0, tk);
        if (tid == 0 && (kind == 2 || !isfinite(tk) || (obs && !isfinite(yk))))
            raise_error(q.err, k, kind == 2 ? kErrUnsupported : kErrInput);
        if (kind == 0) {
            bmm<D, NW>(W.FP, W.F, W.P, nullptr, tid);
            BT_EACH(i, D) {
                double s = 0.0;
                for (int j = 0; j < D; ++j) s = fma(W.F[i][j], W.x[j], s);
                W.xm[i] = s;
            }
            bsync<NW>();
            bmm<D, NW, false, true>(W.Pm, W.FP, W.F, W.Q, tid);
        } else {
            BT_EACH(e, D * D) {
                const int i = e / D, j = e - (e / D) * D;
                W.Pm[i][j] = (kind == 1) ? W.P[i][j] : W.Pinf[i][j];
            }
            BT_EACH(i, D) W.xm[i] = (kind == 1) ? W.x[i] : 0.0;
        }
        bsync<NW>();
        BT_EACH(i, D) {
            double s = 0.0;
            for (int j = 0; j < D; ++j) s = fma(W.Pm[i][j], H[j], s);
            W.HP[i] = s;
        }
        bsync<NW>();
        const double S = bdot<D>(H, W.HP, lane) + r;
        const double hx = bdot<D>(H, W.xm, lane);
        if (tid == 0 && obs && !(S > 0.0 && S < INFINITY)) raise_error(q.err, k, kErrNumeric);
        const double iS = obs ? 1.0 / S : 0.0;
        const double v = obs ? (yk - hx) : 0.0;
        BT_EACH(e, D * D) {
            const int i = e / D, j = e - (e / D) * D;
            W.P[i][j] = fma(-W.HP[i] * iS, W.HP[j], W.Pm[i][j]);
        }
        BT_EACH(i, D) W.x[i] = fma(W.HP[i], v * iS, W.xm[i]);
        if (obs) {
            quad = fma(v, v * iS, quad);
            logs += log(S);
            ++nobs;
        }
        bsync<NW>();
        double* o = q.xs + k * CNW(D);
        BT_EACH(i, D) o[i] = W.x[i];
        BT_EACH(e, D * D) {
            const int i = e / D, j = e - (e / D) * D;
            if (j >= i) o[D + si(D, i, j)] = W.P[i][j];
        }
        bsync<NW>();
    }
    return nobs ? 0.5 * (quad + logs + nobs * 1.8378770664093453) : 0.0;
}

template <int D, int NW>
__device__ void b_load_model(const double* rec, typename BSmem<D>::PerWarp& W, int tid) {
    constexpr int NT = 32 * NW;
    BT_EACH(e, D * D) {
        const int i = e / D, j = e - (e / D) * D;
        W.F[i][j] = rec[e];
        W.Q[i][j] = rec[D * D + e];
        W.Pinf[i][j] = rec[2 * D * D + e];
    }
    bsync<NW>();
}

// posterior: filter, then the RTS smoother from the series' terminal element; mean / var of f
template <int D, int NW>
__global__ void __launch_bounds__(32 * NW) kb_posterior(const BParamsT q, const double* __restrict__ Hg) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BSmem<D>& sh = *reinterpret_cast<BSmem<D>*>(smem_raw);
    auto& W = sh.w[0];
    constexpr int NT = 32 * NW;
    const int tid = threadIdx.x, lane = tid & 31, b = blockIdx.x;
    const int64_t s0 = __ldg(q.off + b), s1 = __ldg(q.off + b + 1);
    const double* rec = q.recs + static_cast<int64_t>(b) * BREC(D, q.npar);
    const double r = rec[(3 + 3 * (q.npar - 1)) * D * D];
    __shared__ double H[D];
    BT_EACH(i, D) H[i] = Hg[i];
    b_load_model<D, NW>(rec, W, tid);
    const double nl = b_filter<D, NW>(q, W, H, r, s0, s1, tid);
    if (tid == 0) q.nll[b] = nl;
    // RTS smoother (supplement PAPER.md:422-430) in its adjoint (modified Bryson-Frazier) form, as
    // kw_smoother_mbf_q: m^s_k = x_k - P_k lh_k, P^s_k = P_k - P_k Lh_k P_k with lh (W.b),
    // Lh (W.C) zero at the series end and, backwards, the rank-one update of step k and F_k^T . F_k;
    // only mean = h m^s and var = h P^s h^T are formed.
    bool bad = false;
    BT_EACH(i, D) W.b[i] = 0.0;
    BT_EACH(e, D * D) W.C[e / D][e % D] = 0.0;
    bsync<NW>();
    for (int64_t k = s1 - 1; k >= s0; --k) {
        const double* src = q.xs + k * CNW(D);
        BT_EACH(i, D) {                                  // P_k h^T
            double s = 0.0;
            for (int j = 0; j < D; ++j) s = fma(src[D + si(D, i, j)], H[j], s);
            W.HP[i] = s;
            W.x[i] = src[i];
        }
        bsync<NW>();
        BT_EACH(i, D) {                                  // Lh (P_k h^T)
            double s = 0.0;
            for (int j = 0; j < D; ++j) s = fma(W.C[i][j], W.HP[j], s);
            W.CK[i] = s;
        }
        bsync<NW>();
        const double hx = bdot<D>(H, W.x, lane), lph = bdot<D>(W.HP, W.b, lane);
        const double hph = bdot<D>(H, W.HP, lane), quad = bdot<D>(W.HP, W.CK, lane);
        if (tid == 0) {
            if (q.mean) q.mean[k] = hx - lph;
            if (q.var) q.var[k] = hph - quad;
        }
        if (k > s0) {
            const int kind = b_kind(q, k, s0, __ldg(q.t + k));   // transition into k: 0 uniform, 1 tie
            const double* prv = q.xs + (k - 1) * CNW(D);
            const bool obs = __ldg(q.mask + k) != 0;
            const double yk = obs ? __ldg(q.y + k) : 0.0;
            if (kind == 0) {
                BT_EACH(i, D) {                          // g = F^T h^T
                    double s = 0.0;
                    for (int j = 0; j < D; ++j) s = fma(W.F[j][i], H[j], s);
                    W.dm[i] = s;
                }
                bsync<NW>();
                BT_EACH(i, D) {                          // P_{k-1} g
                    double s = 0.0;
                    for (int j = 0; j < D; ++j) s = fma(prv[D + si(D, i, j)], W.dm[j], s);
                    W.bm[i] = s;
                }
                bsync<NW>();
                BT_EACH(i, D) {                          // P^- h^T = F (P g) + Q h^T, x^- = F x_{k-1}
                    double s = 0.0, xm = 0.0;
                    for (int j = 0; j < D; ++j) {
                        s = fma(W.F[i][j], W.bm[j], fma(W.Q[i][j], H[j], s));
                        xm = fma(W.F[i][j], prv[j], xm);
                    }
                    W.Mb[i] = s;
                    W.xm[i] = xm;
                }
            } else {                                     // a tie: F = I, Q = 0
                BT_EACH(i, D) {
                    double s = 0.0;
                    for (int j = 0; j < D; ++j) s = fma(prv[D + si(D, i, j)], H[j], s);
                    W.Mb[i] = s;
                    W.xm[i] = prv[i];
                }
            }
            bsync<NW>();
            const double S = bdot<D>(H, W.Mb, lane) + r, hxm = bdot<D>(H, W.xm, lane);
            if (obs) {
                bad = bad || !(S > 0.0);
                const double iS = 1.0 / S, vs = (yk - hxm) * iS;
                BT_EACH(i, D) W.K[i] = W.Mb[i] * iS;
                bsync<NW>();
                BT_EACH(i, D) {                          // w = Lh K
                    double s = 0.0;
                    for (int j = 0; j < D; ++j) s = fma(W.C[i][j], W.K[j], s);
                    W.KT[i] = s;
                }
                bsync<NW>();
                const double cK = bdot<D>(W.K, W.KT, lane), Kl = bdot<D>(W.K, W.b, lane);
                bsync<NW>();
                BT_EACH(e, D * D) {                      // Lt = (I - K h)^T Lh (I - K h) + h^T h / S
                    const int i = e / D, j = e - (e / D) * D;
                    W.C[i][j] = fma(-H[i], W.KT[j], fma(-W.KT[i], H[j], fma((cK + iS) * H[i], H[j], W.C[i][j])));
                }
                BT_EACH(i, D) W.b[i] = fma(-H[i], Kl + vs, W.b[i]);
                bsync<NW>();
            }
            if (kind == 0) {                             // lh <- F^T lt, Lh <- F^T Lt F
                bmm<D, NW>(W.T, W.C, W.F, nullptr, tid);
                BT_EACH(i, D) {
                    double s = 0.0;
                    for (int j = 0; j < D; ++j) s = fma(W.F[j][i], W.b[j], s);
                    W.x[i] = s;
                }
                bsync<NW>();
                bmm<D, NW, true, false>(W.C, W.F, W.T, nullptr, tid);
                BT_EACH(i, D) W.b[i] = W.x[i];
                bsync<NW>();
            }
        }
    }
    if (bad && tid == 0) raise_error(q.err, s0, kErrNumeric);
}

// NLL + gradient: filter, then the reverse-mode adjoint of the filter from the series end (b = C = 0)
// accumulating Z, Cs, gr, C0 and contracting them with the series' own dF, dQ, dP_inf.
template <int D, int NW>
__global__ void __launch_bounds__(32 * NW) kb_nll_grad(const BParamsT q, const double* __restrict__ Hg) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BSmem<D>& sh = *reinterpret_cast<BSmem<D>*>(smem_raw);
    auto& W = sh.w[0];
    constexpr int NT = 32 * NW;
    const int tid = threadIdx.x, lane = tid & 31, b = blockIdx.x;
    const int64_t s0 = __ldg(q.off + b), s1 = __ldg(q.off + b + 1);
    const double* rec = q.recs + static_cast<int64_t>(b) * BREC(D, q.npar);
    const double r = rec[(3 + 3 * (q.npar - 1)) * D * D];
    __shared__ double H[D];
    BT_EACH(i, D) H[i] = Hg[i];
    b_load_model<D, NW>(rec, W, tid);
    const double nl = b_filter<D, NW>(q, W, H, r, s0, s1, tid);
    BT_EACH(e, D * D) {
        W.C[e / D][e % D] = 0.0;
        W.Z[e / D][e % D] = 0.0;
        W.Cs[e / D][e % D] = 0.0;
        W.Pm[e / D][e % D] = 0.0;   // C0 stays here after the loop (series start)
    }
    BT_EACH(i, D) W.b[i] = 0.0;
    bsync<NW>();
    double gr = 0.0;
    bool have_c0 = false;
    for (int64_t k = s1 - 1; k >= s0; --k) {
        const double tk = __ldg(q.t + k);
        const int kind = b_kind(q, k, s0, tk);
        const bool obs = __ldg(q.mask + k) != 0;
        const double yk = obs ? __ldg(q.y + k) : 0.0;
        if (kind != 3) {   // filtered state of k - 1
            const double* src = q.xs + (k - 1) * CNW(D);
            BT_EACH(i, D) W.dm[i] = src[i];
            BT_EACH(e, D * D) W.T[e / D][e % D] = src[D + si(D, e / D, e % D)];
            bsync<NW>();
        }
        // P^- h^T (W.HP) and x^- (W.xm) of step k; P^- itself is never formed (only its product with h)
        if (kind == 0) {
            BT_EACH(i, D) {                              // g = F^T h^T (in W.x), x^- = F x_{k-1}
                double s = 0.0, xm = 0.0;
                for (int j = 0; j < D; ++j) {
                    s = fma(W.F[j][i], H[j], s);
                    xm = fma(W.F[i][j], W.dm[j], xm);
                }
                W.x[i] = s;
                W.xm[i] = xm;
            }
            bsync<NW>();
            BT_EACH(i, D) {                              // P_{k-1} g (in W.bm, rewritten below)
                double s = 0.0;
                for (int j = 0; j < D; ++j) s = fma(W.T[i][j], W.x[j], s);
                W.bm[i] = s;
            }
            bsync<NW>();
            BT_EACH(i, D) {                              // F (P g) + Q h^T
                double s = 0.0;
                for (int j = 0; j < D; ++j) s = fma(W.F[i][j], W.bm[j], fma(W.Q[i][j], H[j], s));
                W.HP[i] = s;
            }
        } else {
            BT_EACH(i, D) {
                double s = 0.0;
                for (int j = 0; j < D; ++j) s = fma((kind == 1) ? W.T[i][j] : W.Pinf[i][j], H[j], s);
                W.HP[i] = s;
                W.xm[i] = (kind == 1) ? W.dm[i] : 0.0;
            }
        }
        bsync<NW>();
        if (obs) {
            const double S = bdot<D>(H, W.HP, lane) + r;
            const double v = yk - bdot<D>(H, W.xm, lane);
            const double iS = 1.0 / S, vs = v * iS, c1 = 0.5 * (iS - vs * vs);
            BT_EACH(i, D) W.K[i] = W.HP[i] * iS;
            bsync<NW>();
            BT_EACH(i, D) {
                double s = 0.0;
                for (int j = 0; j < D; ++j) s = fma(W.C[i][j], W.K[j], s);
                W.CK[i] = s;
            }
            bsync<NW>();
            const double bK = bdot<D>(W.b, W.K, lane), KCK = bdot<D>(W.K, W.CK, lane);
            gr += c1 - bK * vs + KCK;
            BT_EACH(e, D * D) {
                const int i = e / D, j = e - (e / D) * D;
                W.Cm[i][j] = fma(-W.CK[i], H[j], W.C[i][j]);   // C (I - K h^T)
            }
            BT_EACH(i, D) W.Mb[i] = fma(-H[i], bK, W.b[i]);
            bsync<NW>();
            BT_EACH(j, D) {
                double s = 0.0;
                for (int i = 0; i < D; ++i) s = fma(W.K[i], W.Cm[i][j], s);
                W.KT[j] = s;
            }
            bsync<NW>();
            BT_EACH(e, D * D) {
                const int i = e / D, j = e - (e / D) * D;
                const double hi = H[i], hj = H[j];
                W.Cm[i][j] = fma(-hi, W.KT[j], W.Cm[i][j]) + 0.5 * vs * (hi * W.Mb[j] + W.Mb[i] * hj) + c1 * hi * hj;
            }
            BT_EACH(i, D) W.bm[i] = fma(-vs, H[i], W.Mb[i]);
        } else {
            BT_EACH(e, D * D) W.Cm[e / D][e % D] = W.C[e / D][e % D];
            BT_EACH(i, D) W.bm[i] = W.b[i];
        }
        bsync<NW>();
        if (kind == 3) {
            BT_EACH(e, D * D) W.Pm[e / D][e % D] = W.Cm[e / D][e % D];   // C0
            have_c0 = true;
            break;
        }
        if (kind == 0) {
            bmm<D, NW>(W.FP, W.Cm, W.F, nullptr, tid);                          // C^- F
            BT_EACH(i, D) {
                double s = 0.0;
                for (int j = 0; j < D; ++j) s = fma(W.F[j][i], W.bm[j], s);
                W.b[i] = s;
            }
            bsync<NW>();
            bmm<D, NW>(W.Pm, W.FP, W.T, nullptr, tid);                          // C^- F P_{k-1}
            bmm<D, NW, true, false>(W.P, W.F, W.FP, nullptr, tid);              // F^T C^- F
            bsync<NW>();
            BT_EACH(e, D * D) {
                const int i = e / D, j = e - (e / D) * D;
                W.Z[i][j] += fma(W.bm[i], W.dm[j], 2.0 * W.Pm[i][j]);
                W.Cs[i][j] += W.Cm[i][j];
                W.C[i][j] = 0.5 * (W.P[i][j] + W.P[j][i]);
            }
        } else {
            BT_EACH(e, D * D) W.C[e / D][e % D] = W.Cm[e / D][e % D];
            BT_EACH(i, D) W.b[i] = W.bm[i];
        }
        bsync<NW>();
    }
    (void)have_c0;
    // contraction with the series' derivative records (fixed order: deterministic): warp partials,
    // then the NW warp sums in order
    __shared__ double red[NW];
    const double* der = rec + 3 * D * D;
    for (int pp = 0; pp < q.npar; ++pp) {
        double acc = 0.0;
        if (pp < q.npar - 1) {
            const double* dd = der + static_cast<int64_t>(pp) * 3 * D * D;
            BT_EACH(e, D * D) {
                const int i = e / D, j = e - (e / D) * D;
                acc += dd[e] * W.Z[i][j] + dd[D * D + e] * W.Cs[i][j] + dd[2 * D * D + e] * W.Pm[i][j];
            }
        } else if (tid == 0) {
            acc = r * gr;
        }
        acc = wsum(acc);
        if (lane == 0) red[tid >> 5] = acc;
        bsync<NW>();
        if (tid == 0) {
            double g = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) g += red[w];
            q.grad[static_cast<int64_t>(b) * q.npar + pp] = g;
        }
        bsync<NW>();
    }
    if (tid == 0) q.nll[b] = nl;
}

}  // namespace wide
}  // namespace pssgp
