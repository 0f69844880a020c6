/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct fp64 CPU reference for the PSSGP hot path:
 * sequential Kalman filter + RTS smoother + negative log marginal likelihood
 * of a state-space GP.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code with the CUDA path (paper_2102_09964_b200/csrc) and never includes it.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md):
 *   - Discretisation, supplement Eq. "Above, we have":
 *       F = expm(dt G),  Q = int_0^dt e^{(dt-s)G} L q L^T e^{(dt-s)G}^T ds,
 *     evaluated with Van Loan's matrix fraction (the paper's "matrix
 *     fractions"): E = expm([[G, W],[0, -G^T]] dt),
 *     F = E11, Q = E12 E11^T.  expm is scaling-and-squaring Pade(13)
 *     (Higham 2005), a library-primitive-style step written out in C.
 *   - Kalman filter, supplement PAPER.md:285-315 (Eqs. nomeas / withmeas1):
 *       k = 1: prior (0, P_inf) ("p(x_1)", Eq. (7))
 *       k > 1: x- = F x,  P- = F P F^T + Q
 *       observed: S = H P- H^T + r, K = P- H^T / S, x = x- + K (y - H x-),
 *                 P = P- - K S K^T ; missing: x = x-, P = P-.
 *   - NLL (reading Z3): sum over observed k of
 *       0.5 * (log(2 pi S_k) + v_k^2 / S_k), v_k = y_k - H x-_k,
 *     accumulated with Neumaier compensated summation.
 *   - RTS smoother, supplement PAPER.md:422-430 (Eq. smoother), with the
 *     transition OUT of step k (F_k maps k -> k+1):
 *       G_k = P_k F^T (F P_k F^T + Q)^-1   (Cholesky solve)
 *       ms_k = x_k + G_k (ms_{k+1} - F x_k)
 *       Ps_k = P_k + G_k (Ps_{k+1} - F P_k F^T - Q) G_k^T
 *   - Outputs: mean_k = H ms_k, var_k = H Ps_k H^T (latent f).
 *
 * Pins (tests/test_oracle_*.py): dense O(N^3) GP regression (Lemma 1,
 * PAPER.md:262-283), closed-form Matern discretisation, stationarity and
 * semigroup of (F, Q), Simpson quadrature of the Q integral, SPEC hand
 * examples, interleaving / all-missing invariants.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_E_ARG 1
#define OR_E_INPUT 2
#define OR_E_NUMERIC 3
#define OR_E_NOMEM 5

/* ---------------------------------------------------------------- dense helpers (row-major) */
static void mat_mul(int n, const double *A, const double *B, double *C) {
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double s = 0.0;
            for (int k = 0; k < n; ++k) s += A[i * n + k] * B[k * n + j];
            C[i * n + j] = s;
        }
}

static double norm1(int n, const double *A) {
    double best = 0.0;
    for (int j = 0; j < n; ++j) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += fabs(A[i * n + j]);
        if (s > best) best = s;
    }
    return best;
}

/* Solve A X = B (A n x n, B n x m) by Gaussian elimination with partial pivoting.
 * A and B are overwritten; X is returned in B.  Returns 0 or OR_E_NUMERIC. */
static int lu_solve(int n, int m, double *A, double *B) {
    for (int c = 0; c < n; ++c) {
        int p = c;
        for (int r = c + 1; r < n; ++r)
            if (fabs(A[r * n + c]) > fabs(A[p * n + c])) p = r;
        if (A[p * n + c] == 0.0) return OR_E_NUMERIC;
        if (p != c) {
            for (int k = 0; k < n; ++k) { double t = A[c * n + k]; A[c * n + k] = A[p * n + k]; A[p * n + k] = t; }
            for (int k = 0; k < m; ++k) { double t = B[c * m + k]; B[c * m + k] = B[p * m + k]; B[p * m + k] = t; }
        }
        for (int r = c + 1; r < n; ++r) {
            double f = A[r * n + c] / A[c * n + c];
            if (f == 0.0) continue;
            for (int k = c; k < n; ++k) A[r * n + k] -= f * A[c * n + k];
            for (int k = 0; k < m; ++k) B[r * m + k] -= f * B[c * m + k];
        }
    }
    for (int c = n - 1; c >= 0; --c) {
        for (int k = 0; k < m; ++k) {
            double s = B[c * m + k];
            for (int j = c + 1; j < n; ++j) s -= A[c * n + j] * B[j * m + k];
            B[c * m + k] = s / A[c * n + c];
        }
    }
    return OR_OK;
}

/* ---------------------------------------------------------------- expm: Pade(13) scaling & squaring */
/* Higham, "The scaling and squaring method for the matrix exponential revisited" (2005). */
int oracle_expm(int n, const double *A, double *E) {
    static const double b[14] = {64764752532480000.0, 32382376266240000.0, 7771770303897600.0,
                                 1187353796428800.0, 129060195264000.0, 10559470521600.0,
                                 670442572800.0, 33522128640.0, 1323241920.0, 40840800.0,
                                 960960.0, 16380.0, 182.0, 1.0};
    const double theta13 = 5.371920351148152;
    size_t nn = (size_t)n * n;
    double *w = (double *)calloc(8 * nn, sizeof(double));
    if (!w) return OR_E_NOMEM;
    double *As = w, *A2 = w + nn, *A4 = w + 2 * nn, *A6 = w + 3 * nn, *U = w + 4 * nn, *V = w + 5 * nn,
           *T1 = w + 6 * nn, *T2 = w + 7 * nn;
    double nrm = norm1(n, A);
    int s = 0;
    if (nrm > theta13) s = (int)ceil(log2(nrm / theta13));
    if (s > 1000) { free(w); return OR_E_NUMERIC; }
    double scale = ldexp(1.0, -s);
    for (size_t i = 0; i < nn; ++i) As[i] = A[i] * scale;
    mat_mul(n, As, As, A2);
    mat_mul(n, A2, A2, A4);
    mat_mul(n, A4, A2, A6);
    /* U = A [A6 (b13 A6 + b11 A4 + b9 A2) + b7 A6 + b5 A4 + b3 A2 + b1 I] */
    for (size_t i = 0; i < nn; ++i) T1[i] = b[13] * A6[i] + b[11] * A4[i] + b[9] * A2[i];
    mat_mul(n, A6, T1, T2);
    for (size_t i = 0; i < nn; ++i) T2[i] += b[7] * A6[i] + b[5] * A4[i] + b[3] * A2[i];
    for (int i = 0; i < n; ++i) T2[i * n + i] += b[1];
    mat_mul(n, As, T2, U);
    /* V = A6 (b12 A6 + b10 A4 + b8 A2) + b6 A6 + b4 A4 + b2 A2 + b0 I */
    for (size_t i = 0; i < nn; ++i) T1[i] = b[12] * A6[i] + b[10] * A4[i] + b[8] * A2[i];
    mat_mul(n, A6, T1, V);
    for (size_t i = 0; i < nn; ++i) V[i] += b[6] * A6[i] + b[4] * A4[i] + b[2] * A2[i];
    for (int i = 0; i < n; ++i) V[i * n + i] += b[0];
    /* (V - U) R = (V + U) */
    for (size_t i = 0; i < nn; ++i) { T1[i] = V[i] - U[i]; E[i] = V[i] + U[i]; }
    if (lu_solve(n, n, T1, E) != OR_OK) { free(w); return OR_E_NUMERIC; }
    for (int k = 0; k < s; ++k) {
        mat_mul(n, E, E, T1);
        memcpy(E, T1, nn * sizeof(double));
    }
    for (size_t i = 0; i < nn; ++i)
        if (!isfinite(E[i])) { free(w); return OR_E_NUMERIC; }
    free(w);
    return OR_OK;
}

/* ---------------------------------------------------------------- discretisation (Van Loan) */
/* F = expm(G dt), Q = int_0^dt e^{Gs} W e^{G^T s} ds  (supplement PAPER.md:294-303).
 * Van Loan's block exponential loses accuracy once |G dt| is large (the
 * -G^T block grows like e^{+|G| dt}), so dt is first split into 2^s equal
 * sub-steps with |G dt/2^s|_1 <= 1, Van Loan is applied to one sub-step, and
 * the sub-steps are composed with the semigroup identity of the integral,
 *   F(2h) = F(h)^2,  Q(2h) = F(h) Q(h) F(h)^T + Q(h). */
static int van_loan(int n, const double *G, const double *W, double dt, double *F, double *Q) {
    int m = 2 * n;
    double *M = (double *)calloc((size_t)m * m * 2, sizeof(double));
    if (!M) return OR_E_NOMEM;
    double *E = M + (size_t)m * m;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            M[i * m + j] = G[i * n + j] * dt;              /* top-left:  G dt     */
            M[i * m + n + j] = W[i * n + j] * dt;          /* top-right: W dt     */
            M[(n + i) * m + n + j] = -G[j * n + i] * dt;   /* bottom-right: -G^T dt */
        }
    int st = oracle_expm(m, M, E);
    if (st != OR_OK) { free(M); return st; }
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) F[i * n + j] = E[i * m + j];
    /* Q = E12 E11^T */
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double s = 0.0;
            for (int k = 0; k < n; ++k) s += E[i * m + n + k] * E[j * m + k];
            Q[i * n + j] = s;
        }
    free(M);
    return OR_OK;
}

int oracle_discretize(int n, const double *G, const double *W, double dt, double *F, double *Q) {
    size_t nn = (size_t)n * n;
    double g = norm1(n, G) * fabs(dt);
    int s = 0;
    if (g > 1.0) s = (int)ceil(log2(g));
    if (s > 1000) return OR_E_NUMERIC;
    int st = van_loan(n, G, W, ldexp(dt, -s), F, Q);
    if (st != OR_OK) return st;
    if (s > 0) {
        double *T = (double *)malloc(2 * nn * sizeof(double));
        if (!T) return OR_E_NOMEM;
        double *T2 = T + nn;
        for (int r = 0; r < s; ++r) {
            /* Q <- F Q F^T + Q */
            mat_mul(n, F, Q, T);
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j) {
                    double acc = 0.0;
                    for (int k = 0; k < n; ++k) acc += T[i * n + k] * F[j * n + k];
                    T2[i * n + j] = acc + Q[i * n + j];
                }
            memcpy(Q, T2, nn * sizeof(double));
            /* F <- F F */
            mat_mul(n, F, F, T);
            memcpy(F, T, nn * sizeof(double));
        }
        free(T);
    }
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) {
            double a = 0.5 * (Q[i * n + j] + Q[j * n + i]);
            Q[i * n + j] = a; Q[j * n + i] = a;
        }
    for (size_t i = 0; i < nn; ++i)
        if (!isfinite(F[i]) || !isfinite(Q[i])) return OR_E_NUMERIC;
    return OR_OK;
}

/* ---------------------------------------------------------------- Cholesky solve */
/* Solve S X = B for symmetric positive-definite S (n x n), B (n x m); B <- X. */
static int chol_solve(int n, int m, const double *S, double *B, double *Lw) {
    for (int i = 0; i < n; ++i)
        for (int j = 0; j <= i; ++j) {
            double s = S[i * n + j];
            for (int k = 0; k < j; ++k) s -= Lw[i * n + k] * Lw[j * n + k];
            if (i == j) {
                if (!(s > 0.0)) return OR_E_NUMERIC;
                Lw[i * n + i] = sqrt(s);
            } else {
                Lw[i * n + j] = s / Lw[j * n + j];
            }
        }
    for (int k = 0; k < m; ++k) {
        for (int i = 0; i < n; ++i) {
            double s = B[i * m + k];
            for (int j = 0; j < i; ++j) s -= Lw[i * n + j] * B[j * m + k];
            B[i * m + k] = s / Lw[i * n + i];
        }
        for (int i = n - 1; i >= 0; --i) {
            double s = B[i * m + k];
            for (int j = i + 1; j < n; ++j) s -= Lw[j * n + i] * B[j * m + k];
            B[i * m + k] = s / Lw[i * n + i];
        }
    }
    return OR_OK;
}

/* ---------------------------------------------------------------- (F, Q) cache keyed by dt */
typedef struct {
    int n, valid;
    double dt;
    double *F, *Q;
} fq_cache;

static int fq_get(fq_cache *c, const double *G, const double *W, double dt) {
    if (c->valid && c->dt == dt) return OR_OK;  /* identical dt -> identical (F, Q) */
    int st = oracle_discretize(c->n, G, W, dt, c->F, c->Q);
    c->valid = (st == OR_OK);
    c->dt = dt;
    return st;
}

/* ---------------------------------------------------------------- KF + RTS + NLL */
/*
 * n: state dim; G, W = L q L^T, Pinf: n x n row-major; H: n; r > 0: noise variance.
 * t (N, non-decreasing), y (N; read only where mask != 0), mask (N).
 * Outputs: mean, var (N; nullable -> smoother skipped), nll (scalar, nullable),
 * xf (N x n), Pf (N x n x n) filtered moments (nullable; then an internal buffer is used),
 * xs (N x n), Ps (N x n x n) smoothed moments (nullable).
 * err_index (nullable): first failing step.
 */
int oracle_kf_rts(int n, const double *G, const double *W, const double *H, const double *Pinf,
                  double r, int64_t N, const double *t, const double *y, const uint8_t *mask,
                  double *mean, double *var, double *nll, double *xf, double *Pf, double *xs,
                  double *Ps, int64_t *err_index) {
    if (n < 1 || n > 64 || N < 0 || !(r > 0.0)) return OR_E_ARG;
    if (err_index) *err_index = -1;
    for (int64_t k = 0; k < N; ++k) {
        if (!isfinite(t[k]) || (k > 0 && t[k] < t[k - 1])) { if (err_index) *err_index = k; return OR_E_INPUT; }
        if (mask[k] && !isfinite(y[k])) { if (err_index) *err_index = k; return OR_E_INPUT; }
    }
    size_t nn = (size_t)n * n;
    int own_xf = (xf == NULL), own_Pf = (Pf == NULL);
    int want_smooth = (mean != NULL || var != NULL || xs != NULL || Ps != NULL);
    if (own_xf) xf = (double *)malloc((size_t)(N > 0 ? N : 1) * n * sizeof(double));
    if (own_Pf) Pf = (double *)malloc((size_t)(N > 0 ? N : 1) * nn * sizeof(double));
    double *wk = (double *)calloc(12 * nn + 8 * (size_t)n, sizeof(double));
    fq_cache cache = {n, 0, 0.0, NULL, NULL};
    cache.F = (double *)malloc(nn * sizeof(double));
    cache.Q = (double *)malloc(nn * sizeof(double));
    int st = OR_OK;
    if (!xf || !Pf || !wk || !cache.F || !cache.Q) { st = OR_E_NOMEM; goto done; }
    double *Pm = wk, *FP = wk + nn, *T1 = wk + 2 * nn, *Gk = wk + 3 * nn, *Lw = wk + 4 * nn,
           *D = wk + 5 * nn, *GD = wk + 6 * nn, *Pcur = wk + 7 * nn, *Psn = wk + 8 * nn;
    double *xm = wk + 12 * nn, *Kg = xm + n, *dm = Kg + n, *msn = dm + n;

    /* forward Kalman filter */
    double acc = 0.0, comp = 0.0;  /* Neumaier summation */
    for (int64_t k = 0; k < N; ++k) {
        double *xk = xf + (size_t)k * n, *Pk = Pf + (size_t)k * nn;
        if (k == 0) {
            for (int i = 0; i < n; ++i) xm[i] = 0.0;
            memcpy(Pm, Pinf, nn * sizeof(double));
        } else {
            const double *xp = xf + (size_t)(k - 1) * n, *Pp = Pf + (size_t)(k - 1) * nn;
            if ((st = fq_get(&cache, G, W, t[k] - t[k - 1])) != OR_OK) { if (err_index) *err_index = k; goto done; }
            const double *F = cache.F, *Q = cache.Q;
            for (int i = 0; i < n; ++i) {
                double s = 0.0;
                for (int j = 0; j < n; ++j) s += F[i * n + j] * xp[j];
                xm[i] = s;
            }
            mat_mul(n, F, Pp, FP);
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j) {
                    double s = 0.0;
                    for (int l = 0; l < n; ++l) s += FP[i * n + l] * F[j * n + l];
                    Pm[i * n + j] = s + Q[i * n + j];
                }
        }
        if (mask[k]) {
            double S = r, hx = 0.0;
            for (int i = 0; i < n; ++i) {
                hx += H[i] * xm[i];
                double s = 0.0;
                for (int j = 0; j < n; ++j) s += Pm[i * n + j] * H[j];
                Kg[i] = s;                       /* P- H^T */
                S += H[i] * s;
            }
            if (!(S > 0.0) || !isfinite(S)) { st = OR_E_NUMERIC; if (err_index) *err_index = k; goto done; }
            double v = y[k] - hx;
            for (int i = 0; i < n; ++i) xk[i] = xm[i] + Kg[i] / S * v;
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j) Pk[i * n + j] = Pm[i * n + j] - Kg[i] * Kg[j] / S;
            double term = 0.5 * (log(6.283185307179586476925 * S) + v * v / S);
            double sum = acc + term;
            if (fabs(acc) >= fabs(term)) comp += (acc - sum) + term; else comp += (term - sum) + acc;
            acc = sum;
        } else {
            memcpy(xk, xm, n * sizeof(double));
            memcpy(Pk, Pm, nn * sizeof(double));
        }
        for (int i = 0; i < n; ++i)
            for (int j = i + 1; j < n; ++j) {
                double a = 0.5 * (Pk[i * n + j] + Pk[j * n + i]);
                Pk[i * n + j] = a; Pk[j * n + i] = a;
            }
    }
    if (nll) *nll = acc + comp;

    if (!want_smooth || N == 0) goto done;
    /* backward RTS smoother */
    {
        const double *xl = xf + (size_t)(N - 1) * n, *Pl = Pf + (size_t)(N - 1) * nn;
        memcpy(msn, xl, n * sizeof(double));
        memcpy(Psn, Pl, nn * sizeof(double));
        if (xs) memcpy(xs + (size_t)(N - 1) * n, msn, n * sizeof(double));
        if (Ps) memcpy(Ps + (size_t)(N - 1) * nn, Psn, nn * sizeof(double));
        for (int64_t k = N - 1; k >= 0; --k) {
            const double *xk = xf + (size_t)k * n, *Pk = Pf + (size_t)k * nn;
            double *mcur = dm;  /* reuse: smoothed mean at k */
            double mk[64];
            if (k == N - 1) {
                memcpy(mk, msn, n * sizeof(double));
                memcpy(Pcur, Psn, nn * sizeof(double));
            } else {
                if ((st = fq_get(&cache, G, W, t[k + 1] - t[k])) != OR_OK) { if (err_index) *err_index = k + 1; goto done; }
                const double *F = cache.F, *Q = cache.Q;
                mat_mul(n, F, Pk, FP);                         /* F P_k */
                for (int i = 0; i < n; ++i)
                    for (int j = 0; j < n; ++j) {
                        double s = 0.0;
                        for (int l = 0; l < n; ++l) s += FP[i * n + l] * F[j * n + l];
                        Pm[i * n + j] = s + Q[i * n + j];       /* P-_{k+1} */
                    }
                for (int i = 0; i < n; ++i)
                    for (int j = i + 1; j < n; ++j) {
                        double a = 0.5 * (Pm[i * n + j] + Pm[j * n + i]);
                        Pm[i * n + j] = a; Pm[j * n + i] = a;
                    }
                /* P-_{k+1} Gk^T = F P_k  ->  Gk^T */
                memcpy(T1, FP, nn * sizeof(double));
                if ((st = chol_solve(n, n, Pm, T1, Lw)) != OR_OK) { if (err_index) *err_index = k; goto done; }
                for (int i = 0; i < n; ++i)
                    for (int j = 0; j < n; ++j) Gk[i * n + j] = T1[j * n + i];
                for (int i = 0; i < n; ++i) {
                    double s = 0.0;
                    for (int j = 0; j < n; ++j) s += F[i * n + j] * xk[j];
                    mcur[i] = msn[i] - s;                       /* ms_{k+1} - F x_k */
                }
                for (int i = 0; i < n; ++i) {
                    double s = 0.0;
                    for (int j = 0; j < n; ++j) s += Gk[i * n + j] * mcur[j];
                    mk[i] = xk[i] + s;
                }
                for (size_t i = 0; i < nn; ++i) D[i] = Psn[i] - Pm[i];
                mat_mul(n, Gk, D, GD);
                for (int i = 0; i < n; ++i)
                    for (int j = 0; j < n; ++j) {
                        double s = 0.0;
                        for (int l = 0; l < n; ++l) s += GD[i * n + l] * Gk[j * n + l];
                        Pcur[i * n + j] = Pk[i * n + j] + s;
                    }
                for (int i = 0; i < n; ++i)
                    for (int j = i + 1; j < n; ++j) {
                        double a = 0.5 * (Pcur[i * n + j] + Pcur[j * n + i]);
                        Pcur[i * n + j] = a; Pcur[j * n + i] = a;
                    }
            }
            if (xs) memcpy(xs + (size_t)k * n, mk, n * sizeof(double));
            if (Ps) memcpy(Ps + (size_t)k * nn, Pcur, nn * sizeof(double));
            if (mean) {
                double s = 0.0;
                for (int i = 0; i < n; ++i) s += H[i] * mk[i];
                mean[k] = s;
            }
            if (var) {
                double s = 0.0;
                for (int i = 0; i < n; ++i)
                    for (int j = 0; j < n; ++j) s += H[i] * Pcur[i * n + j] * H[j];
                var[k] = s;
            }
            memcpy(msn, mk, n * sizeof(double));
            memcpy(Psn, Pcur, nn * sizeof(double));
        }
    }
done:
    if (own_xf) free(xf);
    if (own_Pf) free(Pf);
    free(wk);
    free(cache.F);
    free(cache.Q);
    return st;
}
