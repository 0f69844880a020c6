// pssgp_grad.cuh — NLL gradient d NLL / d theta (NEXT row f1, SURVEY.md §8(f);
// the hyper-parameter gradient the paper obtains by
// automatic differentiation through the parallel filter).
//
// theta = (log sigma^2, log ell, log sigma_n^2) of a single-component Matern model.
// Forward mode, exact: differentiating the Kalman step (supplement PAPER.md:304-315)
// in the direction of one parameter gives, with M = (I - K H) F, u = F^T H^T v / S,
//     dx_k = M dx_{k-1} + M dP_{k-1} u + e_k,     dP_k = M dP_{k-1} M^T + N_k,
//     e_k  = (I - K H)(dF x + B H^T v / S) - K dr v / S,
//     N_k  = (I - K H) B (I - K H)^T + K dr K^T,   B = dF P F^T + F P dF^T + dQ,
// and the NLL term's tangent is an affine functional of the incoming tangent state,
//     dnll_k = alpha_k + beta_k . dx_{k-1} + tr(Gamma_k dP_{k-1}),
//     alpha_k = c1 (H B H^T + dr) - (v/S) H dF x,  beta_k = -(v/S) g,  Gamma_k = c1 g g^T,
//     g = F^T H^T,  c1 = (1/S - v^2/S^2) / 2     (observed steps; zero when y is missing).
// Affine maps of this form are closed under composition, and the functional can be
// pulled back through them, so a chain of steps folds into one aggregate
// (M, u, e, N | a, b, C) — no solves — and d NLL / d theta is the `a` of the ORDERED
// product of all chain aggregates (the global first element has M = 0, so the
// incoming tangent is irrelevant).  The associativity that licenses the grouping is
// that of function composition (the same argument as PAPER.md:326).
// In the Jordan basis of the closed form (pssgp_math.cuh) F(z), Q(z) depend on z = lambda dt
// only and dF/dz = J F, dQ/dz = sigma^2 w f f^T (f = last column of F, W1 = w e_d e_d^T),
// so theta_ell = log ell gives dz = -z; P_inf = sigma^2 P1 does not depend on ell.
#pragma once
#include "pssgp_kernels.cuh"

namespace pssgp {

template <int D>
struct TAgg {
    double M[D * D];
    double u[D];
    double e[D];
    double N[ns(D)];
    double a;
    double b[D];
    double C[ns(D)];
};

template <int D>
PS_HD void set_identity(TAgg<D>& t) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
#pragma unroll
        for (int j = 0; j < D; ++j) t.M[i * D + j] = (i == j) ? 1.0 : 0.0;
        t.u[i] = 0.0; t.e[i] = 0.0; t.b[i] = 0.0;
    }
#pragma unroll
    for (int i = 0; i < ns(D); ++i) { t.N[i] = 0.0; t.C[i] = 0.0; }
    t.a = 0.0;
}

// out = t2 o t1 (t1 earlier in time): map composition + functional pull-back
template <int D>
PS_HD void combine(const TAgg<D>& t1, const TAgg<D>& t2, TAgg<D>& out) {
    double Nu[D], MN[D * D], Mb[D];
    // functional: a = a1 + a2 + b2.e1 + tr(C2 N1); b = b1 + M1^T b2; C = C1 + sym(w u1^T) + M1^T C2 M1, w = M1^T b2
    double a = t1.a + t2.a;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        a = fma(t2.b[i], t1.e[i], a);
#pragma unroll
        for (int j = 0; j < D; ++j) a = fma(t2.C[si(D, i, j)], t1.N[si(D, j, i)], a);
    }
    double C2M[D * D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) s = fma(t1.M[k * D + i], t2.b[k], s);
        Mb[i] = s;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            double c = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) c = fma(t2.C[si(D, i, k)], t1.M[k * D + j], c);
            C2M[i * D + j] = c;                                   // C2 M1
        }
    }
#pragma unroll
    for (int i = 0; i < D; ++i) {
        out.b[i] = t1.b[i] + Mb[i];
#pragma unroll
        for (int j = i; j < D; ++j) {
            double c = t1.C[si(D, i, j)] + 0.5 * (Mb[i] * t1.u[j] + t1.u[i] * Mb[j]);
#pragma unroll
            for (int k = 0; k < D; ++k) c = fma(t1.M[k * D + i], C2M[k * D + j], c);
            out.C[si(D, i, j)] = c;
        }
    }
    out.a = a;
    // map: M = M2 M1; u = u1 + M1^T u2; e = M2 e1 + M2 N1 u2 + e2; N = M2 N1 M2^T + N2
#pragma unroll
    for (int i = 0; i < D; ++i) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) s = fma(t1.N[si(D, i, k)], t2.u[k], s);
        Nu[i] = s;
    }
    double M[D * D], u[D], e[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
        double ue = t1.u[i], ee = t2.e[i];
#pragma unroll
        for (int k = 0; k < D; ++k) {
            ue = fma(t1.M[k * D + i], t2.u[k], ue);
            ee = fma(t2.M[i * D + k], t1.e[k] + Nu[k], ee);
        }
        u[i] = ue;
        e[i] = ee;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            double m = 0.0, mn = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                m = fma(t2.M[i * D + k], t1.M[k * D + j], m);
                mn = fma(t2.M[i * D + k], t1.N[si(D, k, j)], mn);
            }
            M[i * D + j] = m;
            MN[i * D + j] = mn;
        }
    }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = i; j < D; ++j) {
            double s = t2.N[si(D, i, j)];
#pragma unroll
            for (int k = 0; k < D; ++k) s = fma(MN[i * D + k], t2.M[j * D + k], s);
            out.N[si(D, i, j)] = s;
        }
#pragma unroll
    for (int i = 0; i < D * D; ++i) out.M[i] = M[i];
#pragma unroll
    for (int i = 0; i < D; ++i) { out.u[i] = u[i]; out.e[i] = e[i]; }
}

// Append one step (primal entering the step: x = xbar_{k-1}, P = P_{k-1}) to the aggregate.
// PAR: 0 = log sigma^2, 1 = log ell, 2 = log sigma_n^2.  first: global first element.
template <int D, int PAR>
PS_HD void grad_fold_step(TAgg<D>& A, const double (&x)[D], const double (&P)[ns(D)], const FMat<D>& Fm,
                          const double (&Q)[ns(D)], double z, const ModelParams<D>& m, bool first, bool obs,
                          double yk) {
    const double (&F)[D * D] = Fm.a;
    // primal predict + update quantities
    double FP[D * D], Pm[ns(D)], xm[D];
    kf_predict<D>(x, P, Fm, Q, xm, FP, Pm);
    const double S = Pm[0] + m.r;
    const double iS = obs ? rcp(S) : 0.0;
    const double v = obs ? (yk - xm[0]) : 0.0;
    const double vs = v * iS;
    double K[D];
#pragma unroll
    for (int i = 0; i < D; ++i) K[i] = Pm[si(D, i, 0)] * iS;
    // parameter derivatives dF, dQ, dr
    double dF[D * D], dQ[ns(D)];
    double dr = 0.0;
#pragma unroll
    for (int i = 0; i < D * D; ++i) dF[i] = 0.0;
#pragma unroll
    for (int i = 0; i < ns(D); ++i) dQ[i] = 0.0;
    if constexpr (PAR == 0) {
#pragma unroll
        for (int i = 0; i < ns(D); ++i) dQ[i] = Q[i];             // Q, P_inf proportional to sigma^2
    } else if constexpr (PAR == 1) {
        if (!first) {
            // dF = -z J F (Jordan basis: J = -I + N), dQ = -z sigma^2 w f f^T
            const double w = (D == 1) ? 2.0 : (D == 2) ? 4.0 : 16.0 / 3.0;
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = 0; j < D; ++j)
                    dF[i * D + j] = -z * ((i + 1 < D) ? F[(i + 1) * D + j] - F[i * D + j] : -F[i * D + j]);
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = i; j < D; ++j) dQ[si(D, i, j)] = -z * m.s2 * w * F[i * D + D - 1] * F[j * D + D - 1];
        }
    } else {
        dr = m.r;
    }
    // B = dF P F^T + F P dF^T + dQ = X + X^T + dQ, X = dF (F P)^T
    double B[ns(D)], dFx[D];
    {
        double X[D * D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) s = fma(dF[i * D + k], x[k], s);
            dFx[i] = s;
#pragma unroll
            for (int j = 0; j < D; ++j) {
                double t = 0.0;
#pragma unroll
                for (int k = 0; k < D; ++k) t = fma(dF[i * D + k], FP[j * D + k], t);
                X[i * D + j] = t;
            }
        }
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = i; j < D; ++j) B[si(D, i, j)] = X[i * D + j] + X[j * D + i] + dQ[si(D, i, j)];
    }
    // step element: Mk = (I - K H) F, uk = F^T H^T v/S, ek, Nk
    double Mk[D * D], uk[D], ek[D], Nk[ns(D)], IB[D * D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
#pragma unroll
        for (int j = 0; j < D; ++j) Mk[i * D + j] = fma(-K[i], F[j], F[i * D + j]);
        uk[i] = F[i] * vs;                                        // F[0][i]: g = F^T e0
    }
    // IB = (I - K H) B  (full), then Nk = IB (I - K H)^T + K dr K^T
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) IB[i * D + j] = fma(-K[i], B[si(D, 0, j)], B[si(D, i, j)]);
#pragma unroll
    for (int i = 0; i < D; ++i) {
        ek[i] = fma(-K[i], dFx[0] + B[si(D, 0, 0)] * vs, dFx[i] + B[si(D, i, 0)] * vs) - K[i] * dr * vs;
#pragma unroll
        for (int j = i; j < D; ++j) Nk[si(D, i, j)] = fma(-IB[i * D], K[j], IB[i * D + j]) + K[i] * dr * K[j];
    }
    // functional of this step, pulled back through A: alpha + beta.e + tr(Gamma N); b += M^T beta;
    // C += sym(M^T beta u^T) + c1 h h^T with g = F[0,:]^T, h = M^T g, beta = -(v/S) g
    if (obs) {
        const double c1 = 0.5 * (iS - vs * vs);
        double h[D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) s = fma(A.M[k * D + i], F[k], s);
            h[i] = s;
        }
        double ge = 0.0, gNg = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            ge = fma(F[i], A.e[i], ge);
#pragma unroll
            for (int j = 0; j < D; ++j) gNg = fma(F[i] * A.N[si(D, i, j)], F[j], gNg);
        }
        A.a += c1 * (B[0] + dr) - vs * dFx[0] - vs * ge + c1 * gNg;
#pragma unroll
        for (int i = 0; i < D; ++i) A.b[i] = fma(-vs, h[i], A.b[i]);
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = i; j < D; ++j)
                A.C[si(D, i, j)] += -0.5 * vs * (h[i] * A.u[j] + A.u[i] * h[j]) + c1 * h[i] * h[j];
    }
    // compose the map: M = Mk M, u = u + M^T uk, e = Mk e + Mk N uk + ek, N = Mk N Mk^T + Nk
    TAgg<D> step;
#pragma unroll
    for (int i = 0; i < D * D; ++i) step.M[i] = Mk[i];
#pragma unroll
    for (int i = 0; i < D; ++i) { step.u[i] = uk[i]; step.e[i] = ek[i]; step.b[i] = 0.0; }
#pragma unroll
    for (int i = 0; i < ns(D); ++i) { step.N[i] = Nk[i]; step.C[i] = 0.0; }
    step.a = 0.0;
    TAgg<D> r;
    combine(A, step, r);
    A = r;
}

// ------------------------------------------------------------------ KG: fold tangent aggregates per chain
// Reads the filtered moments (xbar_k, P_k) written by k_filter_apply (same launch plan).
template <int D, int PAR>
__global__ void __launch_bounds__(kThreads, PSSGP_MINB) k_grad_fold(const KParams<D> p, double* block_out) {
    __shared__ TAgg<D> wagg[kWarps];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t c = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
    const int64_t wg = static_cast<int64_t>(blockIdx.x) * kWarps + wid;
    const int64_t kb = c * p.K;
    const int64_t ke = min(kb + p.K, p.n);
    TAgg<D> A;
    set_identity(A);
    double x[D], P[ns(D)];
#pragma unroll
    for (int i = 0; i < D; ++i) x[i] = 0.0;
#pragma unroll
    for (int i = 0; i < ns(D); ++i) P[i] = 0.0;
    double tprev = 0.0;
    if (kb < ke && kb > 0) {
        // primal entering the chain = filtered moments of step kb-1 (last step of chain c-1)
        const int64_t cp = c - 1;
        const double* src = p.xp + (((cp / 32) * p.K + (p.K - 1)) * CN(D)) * 32 + (cp % 32);
#pragma unroll
        for (int i = 0; i < D; ++i) x[i] = src[i * 32];
#pragma unroll
        for (int i = 0; i < ns(D); ++i) P[i] = src[(D + i) * 32];
        tprev = __ldg(p.t + kb - 1);
    }
    const double* xpw = p.xp + (wg * p.K * CN(D)) * 32 + lane;
#pragma unroll 1
    for (int64_t k = kb; k < ke; ++k) {
        const double tk = __ldg(p.t + k);
        const bool obs = __ldg(p.mask + k) != 0;
        const double yk = obs ? __ldg(p.y + k) : 0.0;
        FJor<D> Fj;
        double Q[ns(D)];
        const bool first = (k == 0);
        double z = 0.0;
        if (first) {
            set_zero(Fj);
#pragma unroll
            for (int i = 0; i < ns(D); ++i) Q[i] = p.m.Pinf[i];
        } else {
            z = p.m.lam * (tk - tprev);
            matern_closed<D>(p.m.lam, p.m.s2, tk - tprev, Fj, Q);
        }
        grad_fold_step<D, PAR>(A, x, P, to_full<D>(Fj), Q, z, p.m, first, obs, yk);
        tprev = tk;
        const double* src = xpw + ((k - kb) * CN(D)) * 32;
#pragma unroll
        for (int i = 0; i < D; ++i) x[i] = src[i * 32];
#pragma unroll
        for (int i = 0; i < ns(D); ++i) P[i] = src[(D + i) * 32];
    }
    // ordered CTA reduction
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        TAgg<D> o;
        shfl_down_all(o, A, off);
        if ((lane & (2 * off - 1)) == 0) {
            TAgg<D> r;
            combine(A, o, r);
            A = r;
        }
    }
    if (lane == 0) wagg[wid] = A;
    __syncthreads();
    if (threadIdx.x == 0) {
        TAgg<D> acc = wagg[0];
        for (int w = 1; w < kWarps; ++w) {
            TAgg<D> r;
            combine(acc, wagg[w], r);
            acc = r;
        }
        store_aos(acc, block_out + static_cast<int64_t>(blockIdx.x) * (sizeof(TAgg<D>) / sizeof(double)));
    }
}

}  // namespace pssgp
