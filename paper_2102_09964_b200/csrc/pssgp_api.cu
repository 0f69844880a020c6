// pssgp_api.cu — C ABI (include/pssgp.h): model construction, workspace,
// launch plan and kernel launches of the PSSGP hot path on sm_100a.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstddef>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "pssgp_internal.hpp"
#include "pssgp_kernels.cuh"
#include "pssgp_batch.cuh"
#include "pssgp_grad.cuh"
#include "pssgp_f32.h"

using namespace pssgp;
using namespace pssgp_internal;
namespace ph = pssgp_host;




namespace pssgp_internal {
pssgp_status ensure_device(pssgp_model* m) {
    if (m->sm_count > 0) return PSSGP_OK;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) return fail(m, PSSGP_E_CUDA, "no CUDA device available");
    int dev = m->device;
    if (dev < 0) cudaGetDevice(&dev);
    m->device = dev;
    e = cudaDeviceGetAttribute(&m->sm_count, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return cuda_fail(m, e, "cudaDeviceGetAttribute");
    // word 0: latched error; 1..4: K3 publication flag, tile ticket, published-block and finished-CTA
    // counters (pssgp_kernels.cuh KParams::flag); then 8 scratch doubles
    e = cudaMalloc(&m->d_err, 8 * sizeof(unsigned long long) + 8 * sizeof(double));
    if (e != cudaSuccess) return fail(m, PSSGP_E_NOMEM, "cudaMalloc(error word)");
    cudaMemset(m->d_err, 0xff, sizeof(unsigned long long));
    cudaMemset(m->d_err + 1, 0, 7 * sizeof(unsigned long long));
    m->d_scalar = reinterpret_cast<double*>(m->d_err + 8);
    return PSSGP_OK;
}

pssgp_status nll_sum(pssgp_model* m, const double* parts, int nb, double* out, cudaStream_t s, int stride) {
    ProfScope ps(m, S_K6, s);
    k_nll_sum<<<1, kThreads, 0, s>>>(parts, nb, out, stride);
    LAUNCH_CHECK(m, "k_nll_sum");
    return PSSGP_OK;
}
}  // namespace pssgp_internal

namespace {


template <int D>
void fill_params(const pssgp_model* m, ModelParams<D>& p) {
    std::memset(&p, 0, sizeof(p));
    for (int i = 0; i < D; ++i)
        for (int j = i; j < D; ++j) p.Pinf[si(D, i, j)] = static_cast<double>(m->ssm.Pinf[i * D + j]);
    bool hu = true;
    for (int i = 0; i < D; ++i) {
        p.H[i] = static_cast<double>(m->ssm.H[i]);
        if (p.H[i] != (i == 0 ? 1.0 : 0.0)) hu = false;
    }
    p.h_unit = hu ? 1 : 0;
    p.r = m->r;
    p.lam = m->lam;
    p.s2 = m->s2;
    p.closed = m->closed ? 1 : 0;
    p.udt = m->udt > 0.0 ? m->udt : -1.0;  // -1 never equals a valid dt >= 0
    for (int i = 0; i < D * D; ++i) p.G[i] = static_cast<double>(m->ssm.G[i]);
    for (int i = 0; i < D; ++i)
        for (int j = i; j < D; ++j) p.W[si(D, i, j)] = static_cast<double>(m->ssm.W[i * D + j]);
    if (m->udt > 0.0) {
        for (int i = 0; i < D * D; ++i) p.Fu[i] = m->Fu[i];
        for (int i = 0; i < D; ++i)
            for (int j = i; j < D; ++j) p.Qu[si(D, i, j)] = m->Qu[i * D + j];
    }
}

template <int D>
int occupancy() {
    int a = 0, b = 0, c = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_filter_reduce<D, kClosed>, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_filter_apply<D, kClosed>, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, k_smoother_apply<D, kClosed>, kThreads, 0);
    return std::max(1, std::min(a, std::min(b, c)));
}

struct Plan {
    int64_t K = 0, nch = 0;
    int nb = 0;
};

template <int D>
Plan make_plan(pssgp_model* m, int64_t n) {
    if (m->occ == 0) m->occ = occupancy<D>();
    const int bps = m->blocks_per_sm > 0 ? m->blocks_per_sm : m->occ;
    const int64_t target_chains = static_cast<int64_t>(m->sm_count) * bps * kThreads;
    Plan pl;
    // one wave of chains; K rounded up to whole staging windows, except below one window, where
    // short chains (down to one step) keep the wave full at small N (the paper's N = 1,200 / 3,200
    // problems run in ~40 instead of ~70 us: the latency is the scan span, tools/small_n_sweep.py)
    int64_t K = m->forced_K > 0 ? m->forced_K : std::max<int64_t>(1, (n + target_chains - 1) / target_chains);
    if (m->forced_K <= 0 && K > kWin / 4) K = ((K + kWin - 1) / kWin) * kWin;
    pl.K = K;
    pl.nch = std::max<int64_t>(1, (n + K - 1) / K);
    pl.nb = static_cast<int>((pl.nch + kThreads - 1) / kThreads);
    return pl;
}

template <int D>
size_t ws_doubles(const Plan& pl) {
    const size_t nchp = static_cast<size_t>(pl.nb) * kThreads;
    return nchp * FN(D) + static_cast<size_t>(pl.nb) * FN(D) + static_cast<size_t>(pl.nb) * CN(D) +
           static_cast<size_t>(pl.nb) * kWarps * pl.K * CN(D) * 32 + nchp * SN(D) +
           static_cast<size_t>(pl.nb) * SN(D) + static_cast<size_t>(pl.nb) * CN(D) + pl.nb + 64;
}

template <int D>
pssgp_status setup(pssgp_model* m, const Plan& pl, KParams<D>& p) {
    const size_t need = ws_doubles<D>(pl) * sizeof(double);
    if (need > m->ws_bytes) {
        if (m->ws) cudaFree(m->ws);
        m->ws = nullptr;
        m->ws_bytes = 0;
        cudaError_t e = cudaMalloc(&m->ws, need);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(m, PSSGP_E_NOMEM, "cudaMalloc(workspace) failed");
        }
        m->ws_bytes = need;
    }
    std::memset(&p, 0, sizeof(p));
    fill_params<D>(m, p.m);
    const size_t nchp = static_cast<size_t>(pl.nb) * kThreads;
    double* w = reinterpret_cast<double*>(m->ws);
    p.chain_f = w; w += nchp * FN(D);
    p.block_f = w; w += static_cast<size_t>(pl.nb) * FN(D);
    p.fcarry = w; w += static_cast<size_t>(pl.nb) * CN(D);
    w += (reinterpret_cast<uintptr_t>(w) >> 3) & 1;   // 16-byte aligned records (paired state loads)
    p.xp = w; w += static_cast<size_t>(pl.nb) * kWarps * pl.K * CN(D) * 32;
    p.chain_s = w; w += nchp * SN(D);
    p.block_s = w; w += static_cast<size_t>(pl.nb) * SN(D);
    p.scarry = w; w += static_cast<size_t>(pl.nb) * CN(D);
    p.nll_block = w;
    p.K = pl.K;
    p.nb = pl.nb;
    p.err = m->d_err;
    p.flag = m->d_err + 1;
    p.rank = 0;
    p.world = 1;
    p.store_state = 1;
    return PSSGP_OK;
}

// launch kernel template KERN<D, mode> with the model's discretisation mode
#define LAUNCH_MODE(m, KERN, grid, block, s, p)                                  \
    do {                                                                         \
        if ((m)->mode == kClosed) KERN<D, kClosed><<<grid, block, 0, s>>>(p);    \
        else if ((m)->mode == kPade) KERN<D, kPade><<<grid, block, 0, s>>>(p);   \
        else KERN<D, kTable><<<grid, block, 0, s>>>(p);                          \
    } while (0)

template <int D>
pssgp_status phase_filter_reduce(pssgp_model* m, KParams<D>& p, cudaStream_t s) {
    ProfScope ps(m, S_K1, s);
    LAUNCH_MODE(m, k_filter_reduce, p.nb, kThreads, s, p);
    LAUNCH_CHECK(m, "k_filter_reduce");
    return PSSGP_OK;
}

// sagg = false: filtered-state stores without the smoother-aggregate work (gradient primal pass)
template <int D>
pssgp_status phase_filter_apply(pssgp_model* m, KParams<D>& p, cudaStream_t s, bool sagg = true) {
    ProfScope ps(m, S_K3, s);
    if (p.store_state && !sagg && m->mode == kClosed)
        k_filter_apply<D, kClosed, true, false><<<p.nb, kThreads, 0, s>>>(p);
    else if (p.store_state) LAUNCH_MODE(m, k_filter_apply, p.nb, kThreads, s, p);
    else if (m->mode == kClosed) k_filter_apply<D, kClosed, false><<<p.nb, kThreads, 0, s>>>(p);
    else if (m->mode == kPade) k_filter_apply<D, kPade, false><<<p.nb, kThreads, 0, s>>>(p);
    else k_filter_apply<D, kTable, false><<<p.nb, kThreads, 0, s>>>(p);
    LAUNCH_CHECK(m, "k_filter_apply");
    return PSSGP_OK;
}

// single-pass K1 + K3 (k_filter_fused) instead of two launches: PSSGP_FUSED=1 (A/B)
bool fused_filter() {
    static const bool v = [] { const char* e = getenv("PSSGP_FUSED"); return e && *e == '1'; }();
    return v;
}

// the cooperative launch needs the whole grid resident (one-wave plans are, forced chain lengths
// may not be: those take the two-launch path)
template <int D>
bool fused_fits(pssgp_model* m, int nb) {
    int occ = 0;
    if (m->mode == kClosed) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_filter_fused<D, kClosed>, kThreads, 0);
    else if (m->mode == kPade) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_filter_fused<D, kPade>, kThreads, 0);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_filter_fused<D, kTable>, kThreads, 0);
    return nb <= occ * m->sm_count;
}

template <int D>
pssgp_status phase_filter_fused(pssgp_model* m, KParams<D>& p, cudaStream_t s) {
    ProfScope ps(m, S_K3, s);
    // flag[0..3] from zero whichever kernel ran last (K3 leaves its publication word and ticket set)
    cudaError_t e0 = cudaMemsetAsync(p.flag, 0, 4 * sizeof(unsigned long long), s);
    if (e0 != cudaSuccess) return cuda_fail(m, e0, "cudaMemsetAsync(flags)");
    void* args[] = {&p};
    const void* fn = (m->mode == kClosed) ? reinterpret_cast<const void*>(k_filter_fused<D, kClosed>)
                     : (m->mode == kPade) ? reinterpret_cast<const void*>(k_filter_fused<D, kPade>)
                                          : reinterpret_cast<const void*>(k_filter_fused<D, kTable>);
    const cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(p.nb), dim3(kThreads), args, 0, s);
    if (e != cudaSuccess) return cuda_fail(m, e, "k_filter_fused (cooperative launch)");
    return PSSGP_OK;
}

template <int D>
pssgp_status phase_smoother(pssgp_model* m, KParams<D>& p, cudaStream_t s) {
    ProfScope ps(m, S_K5, s);
    LAUNCH_MODE(m, k_smoother_apply, p.nb, kThreads, s, p);
    LAUNCH_CHECK(m, "k_smoother_apply");
    return PSSGP_OK;
}

pssgp_status check_args(pssgp_model* m, int64_t N, const double* t, const double* y, const uint8_t* mask) {
    if (!m) return PSSGP_E_ARG;
    if (N < 0) return fail(m, PSSGP_E_ARG, "N < 0");
    if (N > 0 && (!t || !y || !mask)) return fail(m, PSSGP_E_ARG, "NULL input array");
    if (N > (int64_t(1) << 40)) return fail(m, PSSGP_E_ARG, "N too large");
    return PSSGP_OK;
}

template <int D>
pssgp_status run_posterior(pssgp_model* m, int64_t N, const double* t, const double* y, const uint8_t* mask,
                           double* mean, double* var, double* nll, cudaStream_t s, bool smooth) {
    if (N == 0) {
        if (nll) {
            cudaError_t e = cudaMemsetAsync(nll, 0, sizeof(double), s);
            if (e != cudaSuccess) return cuda_fail(m, e, "cudaMemsetAsync");
        }
        return PSSGP_OK;
    }
    const Plan pl = make_plan<D>(m, N);
    KParams<D> p;
    pssgp_status st = setup<D>(m, pl, p);
    if (st) return st;
    p.t = t; p.y = y; p.mask = mask;
    p.n = N; p.k0 = 0; p.nglob = N;
    p.mean = mean; p.var = var;
    p.store_state = smooth ? 1 : 0;
    if (smooth && fused_filter() && fused_fits<D>(m, p.nb)) {
        if ((st = phase_filter_fused<D>(m, p, s))) return st;
    } else {
        if ((st = phase_filter_reduce<D>(m, p, s))) return st;
        if ((st = phase_filter_apply<D>(m, p, s))) return st;
    }
    if (smooth) {
        p.nll_out = nll;                       // K5's CTA 0 sums the NLL partials
        if ((st = phase_smoother<D>(m, p, s))) return st;
    } else if (nll && (st = nll_sum(m, p.nll_block, p.nb, nll, s))) {
        return st;
    }
    return PSSGP_OK;
}

// NLL gradient (f1): primal filter storing (xbar, P), then ONE tangent fold of all three
// parameter directions + an ordered block reduction (pssgp_grad.cuh).
template <int D>
pssgp_status run_grad(pssgp_model* m, int64_t N, const double* t, const double* y, const uint8_t* mask,
                      double* nll, double* grad, cudaStream_t s) {
    if (N == 0) {
        cudaError_t e = cudaMemsetAsync(grad, 0, 3 * sizeof(double), s);
        if (e == cudaSuccess && nll) e = cudaMemsetAsync(nll, 0, sizeof(double), s);
        if (e != cudaSuccess) return cuda_fail(m, e, "cudaMemsetAsync");
        return PSSGP_OK;
    }
    const Plan pl = make_plan<D>(m, N);
    KParams<D> p;
    pssgp_status st = setup<D>(m, pl, p);
    if (st) return st;
    p.t = t; p.y = y; p.mask = mask;
    p.n = N; p.k0 = 0; p.nglob = N;
    p.store_state = 1;
    if ((st = phase_filter_reduce<D>(m, p, s))) return st;
    if ((st = phase_filter_apply<D>(m, p, s, false))) return st;
    if (nll && (st = nll_sum(m, p.nll_block, p.nb, nll, s))) return st;
    // block tangent aggregates reuse the smoother-aggregate region (not read on this path)
    constexpr size_t NA = sizeof(TAgg3<D>) / sizeof(double);
    static_assert(NA <= kThreads * SN(D), "grad scratch");
    double* blocks = p.chain_s;
    double* out = p.chain_s + static_cast<size_t>(pl.nb) * NA;
    {
        ProfScope ps(m, S_GRAD, s);
        k_grad_fold<D><<<p.nb, kThreads, 0, s>>>(p, blocks);
        LAUNCH_CHECK(m, "k_grad_fold");
    }
    {
        ProfScope ps(m, S_RED, s);
        k_reduce_blocks<D, TAgg3<D>><<<1, kCarryThreads, 0, s>>>(blocks, p.nb, out, nullptr, 0);
        LAUNCH_CHECK(m, "k_reduce_blocks(grad)");
    }
    cudaError_t e = cudaMemcpyAsync(grad, out + offsetof(TAgg3<D>, a) / sizeof(double), 3 * sizeof(double),
                                    cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(m, e, "cudaMemcpyAsync(grad)");
    return PSSGP_OK;
}

template <int D>
pssgp_status debug_disc(const pssgp_model* m, double dt, double* F, double* Q) {
    ModelParams<D> p;
    fill_params<D>(m, p);
    double f[D * D], q[ns(D)];
    const int rc = discretize<D>(p, dt, f, q);
    for (int i = 0; i < D * D; ++i) F[i] = f[i];
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j) Q[i * D + j] = q[si(D, i, j)];
    return rc ? PSSGP_E_UNSUPPORTED : PSSGP_OK;
}

#define DISPATCH_D(m, CALL)                                         \
    switch ((m)->d) {                                               \
        case 1: { constexpr int D_ = 1; return CALL; }              \
        case 2: { constexpr int D_ = 2; return CALL; }              \
        case 3: { constexpr int D_ = 3; return CALL; }              \
        default: return fail((m), PSSGP_E_UNSUPPORTED, "state dimension not compiled"); \
    }

}  // namespace



// ========================================================================== C ABI
extern "C" {

pssgp_status pssgp_create(const pssgp_component* comps, int n_comps, double noise_var, const pssgp_options* opt,
                          pssgp_model** out) {
    if (!out) return PSSGP_E_ARG;
    *out = nullptr;
    if (!comps || n_comps < 1 || n_comps > 16) return PSSGP_E_ARG;
    if (!(noise_var > 0.0) || !std::isfinite(noise_var)) return PSSGP_E_ARG;
    pssgp_options o{1, -1, 0.0, 0, 0};
    if (opt) o = *opt;
    auto* m = new (std::nothrow) pssgp_model();
    if (!m) return PSSGP_E_NOMEM;
    m->r = noise_var;
    m->device = o.device;
    m->forced_K = o.chain_len;
    m->blocks_per_sm = o.blocks_per_sm;
    std::vector<ph::Ssm> parts;
    std::vector<std::vector<ph::ParamDeriv>> cder;   // per component: d(G, W, P_inf)/d theta_p, local basis
    // variance: W and P_inf scale; time-scale parameter: G, W scale as 1 / tau (host_model.hpp)
    auto vscale = [](const ph::Ssm& p) { return ph::ParamDeriv{ph::zeros(p.d), p.W, p.Pinf}; };
    auto tscale = [](const ph::Ssm& p) { return ph::ParamDeriv{ph::scaled(p.G, -1.0L), ph::scaled(p.W, -1.0L), ph::zeros(p.d)}; };
    int boff = 0, bpar = 0;
    m->bt_ok = true;
    for (int c = 0; c < n_comps; ++c) {
        const pssgp_component& k = comps[c];
        if (!(k.variance > 0.0) || !std::isfinite(k.variance) || !(k.lengthscale > 0.0) || !std::isfinite(k.lengthscale)) {
            delete m;
            return PSSGP_E_ARG;
        }
        ph::Ssm part;
        if (k.kind >= PSSGP_MATERN12 && k.kind <= PSSGP_MATERN52) {
            ph::ld lam;
            part = ph::matern(k.kind, k.variance, k.lengthscale, &lam);
            if (n_comps == 1) {
                m->closed = true;
                m->lam = static_cast<double>(lam);
                m->s2 = k.variance;
            }
        } else if (k.kind == PSSGP_RBF_TAYLOR) {
            if (k.order < 1 || k.order > 12) { delete m; return PSSGP_E_ARG; }
            std::string err;
            if (!ph::rbf_taylor(k.order, k.variance, k.lengthscale, part, err)) { delete m; return PSSGP_E_NUMERIC; }
            if (o.balance) ph::apply_balance(part, ph::osborne(part.G, part.d));
            if (!ph::lyapunov(part.G, part.W, part.d, part.Pinf)) { delete m; return PSSGP_E_NUMERIC; }
        } else if (k.kind == PSSGP_PERIODIC) {
            if (k.order < 0 || k.order > 32 || !(k.period > 0.0)) { delete m; return PSSGP_E_ARG; }
            part = ph::periodic(k.order, k.variance, k.lengthscale, k.period);
            cder.push_back({vscale(part),
                            ph::ParamDeriv{ph::zeros(part.d), ph::zeros(part.d),
                                           ph::periodic_dP_dlogell(k.order, k.variance, k.lengthscale)},
                            tscale(part)});
        } else if (k.kind == PSSGP_QUASIPERIODIC) {
            if (k.order < 0 || k.order > 16 || !(k.period > 0.0) || !(k.mat_lengthscale > 0.0) ||
                (k.mat_nu2 != 1 && k.mat_nu2 != 3 && k.mat_nu2 != 5)) {
                delete m;
                return PSSGP_E_ARG;
            }
            ph::ld lam;
            const ph::Ssm per = ph::periodic(k.order, k.variance, k.lengthscale, k.period);
            const ph::Ssm mat = ph::matern((k.mat_nu2 + 1) / 2, 1.0L, k.mat_lengthscale, &lam);
            part = ph::kron_product(per, mat);
            // log ell: P_p -> dP_p (Bessel weights); log period: -(G_p (x) I); log Matern ell: -(I (x) G_m), -W
            ph::Ssm per_l = per, per_t = per, mat_0 = mat, per_0 = per, mat_t = mat;
            per_l.G = ph::zeros(per.d);
            per_l.Pinf = ph::periodic_dP_dlogell(k.order, k.variance, k.lengthscale);
            per_t.G = ph::scaled(per.G, -1.0L);
            per_t.Pinf = ph::zeros(per.d);
            mat_0.G = ph::zeros(mat.d);
            per_0.G = ph::zeros(per.d);
            mat_t.G = ph::scaled(mat.G, -1.0L);
            const ph::Ssm kl = ph::kron_product(per_l, mat), kp = ph::kron_product(per_t, mat_0),
                          km = ph::kron_product(per_0, mat_t);
            cder.push_back({vscale(part), ph::ParamDeriv{ph::zeros(part.d), kl.W, kl.Pinf},
                            ph::ParamDeriv{kp.G, ph::zeros(part.d), ph::zeros(part.d)},
                            ph::ParamDeriv{km.G, ph::scaled(part.W, -1.0L), ph::zeros(part.d)}});
        } else {
            delete m;
            return PSSGP_E_UNSUPPORTED;
        }
        if (k.kind != PSSGP_PERIODIC && k.kind != PSSGP_QUASIPERIODIC) cder.push_back({vscale(part), tscale(part)});
        {   // structure for the batched per-series-theta path (closed-form models only, not RBF)
            const int bk = (k.kind <= PSSGP_MATERN52) ? 1 : (k.kind == PSSGP_PERIODIC ? 2 : (k.kind == PSSGP_QUASIPERIODIC ? 3 : 0));
            if (bk == 0) m->bt_ok = false;
            const int nu2 = (k.kind <= PSSGP_MATERN52) ? 2 * k.kind - 1 : k.mat_nu2;
            m->bdesc.insert(m->bdesc.end(), {bk, k.order, nu2, boff, part.d, bpar});
            boff += part.d;
            bpar += static_cast<int>(cder.back().size());
        }
        parts.push_back(part);
    }
    m->ssm = parts.size() == 1 ? parts[0] : ph::block_sum(parts);
    m->d = m->ssm.d;
    {   // F = e^{G dt} (and Q) are block diagonal wherever G and W are: the smallest aligned block
        // size 2 or 4 that contains every nonzero of both (else d), for the half-chain kernels
        auto blocked = [&](int B) {
            for (int i = 0; i < m->d; ++i)
                for (int j = 0; j < m->d; ++j)
                    if ((m->ssm.G[i * m->d + j] != 0.0L || m->ssm.W[i * m->d + j] != 0.0L) && i / B != j / B) return false;
            return true;
        };
        m->fblock = blocked(2) ? 2 : (blocked(4) ? 4 : m->d);
    }
    {   // embed the per-component derivatives into the d x d state (block-diagonal sum)
        int o = 0;
        for (size_t c = 0; c < parts.size(); ++c) {
            const int pd = parts[c].d;
            for (const auto& q : cder[c]) {
                ph::ParamDeriv g{ph::zeros(m->d), ph::zeros(m->d), ph::zeros(m->d)};
                for (int i = 0; i < pd; ++i)
                    for (int j = 0; j < pd; ++j) {
                        g.dG[(o + i) * m->d + o + j] = q.dG[i * pd + j];
                        g.dW[(o + i) * m->d + o + j] = q.dW[i * pd + j];
                        g.dP[(o + i) * m->d + o + j] = q.dP[i * pd + j];
                    }
                m->pder.push_back(g);
            }
            o += pd;
        }
    }
    if (m->d > kMaxD && !wide_ops_for(m->d)) {
        delete m;
        return PSSGP_E_UNSUPPORTED;
    }
    if (o.uniform_dt > 0.0 && std::isfinite(o.uniform_dt)) {
        m->udt = o.uniform_dt;
        ph::Mat F, Q;
        ph::van_loan(m->ssm.G, m->ssm.W, m->d, static_cast<ph::ld>(o.uniform_dt), F, Q);
        m->Fu.resize(F.size());
        m->Qu.resize(Q.size());
        for (size_t i = 0; i < F.size(); ++i) { m->Fu[i] = static_cast<double>(F[i]); m->Qu[i] = static_cast<double>(Q[i]); }
    }
    m->mode = m->closed ? kClosed : (m->udt > 0.0 ? kTable : kPade);
    *out = m;
    return PSSGP_OK;
}

void pssgp_destroy(pssgp_model* m) {
    if (!m) return;
    if (m->ws) cudaFree(m->ws);
    if (m->io) cudaFree(m->io);
    if (m->mg) cudaFree(m->mg);
    if (m->bt) cudaFree(m->bt);
    if (m->fq) cudaFree(m->fq);
    if (m->gb) cudaFree(m->gb);
    for (int i = 0; i < 2; ++i) {
        if (m->aio[i]) cudaFree(m->aio[i]);
        if (m->astream[i]) cudaStreamDestroy(m->astream[i]);
        if (m->aout[i]) cudaStreamDestroy(m->aout[i]);
        if (m->ev_in[i]) cudaEventDestroy(m->ev_in[i]);
        if (m->ev_comp[i]) cudaEventDestroy(m->ev_comp[i]);
        if (m->ev_out[i]) cudaEventDestroy(m->ev_out[i]);
    }
    if (m->acs) cudaStreamDestroy(m->acs);
    if (m->d_err) cudaFree(m->d_err);
    if (m->d_model) cudaFree(m->d_model);
    if (m->d_gder) cudaFree(m->d_gder);
    if (m->gw) cudaFree(m->gw);
    if (m->bw) cudaFree(m->bw);
    for (int s = 0; s < kSlots; ++s)
        for (auto& pr : m->ev[s]) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
    for (auto e : m->ev_pool) cudaEventDestroy(e);
    delete m;
}

int pssgp_state_dim(const pssgp_model* m) { return m ? m->d : -1; }

pssgp_status pssgp_posterior(pssgp_model* m, int64_t N, const double* t, const double* y, const uint8_t* mask,
                             double* mean, double* var, double* nll, void* stream) {
    NvtxCall nvtx_("pssgp_posterior");
    pssgp_status st = check_args(m, N, t, y, mask);
    if (st) return st;
    if ((st = ensure_device(m))) return st;
    auto s = static_cast<cudaStream_t>(stream);
    m->last_stream = s;
    const bool smooth = (mean != nullptr) || (var != nullptr);
    if (m->d > kMaxD) return wide_ops_for(m->d)->posterior(m, N, t, y, mask, mean, var, nll, s, smooth);
    DISPATCH_D(m, run_posterior<D_>(m, N, t, y, mask, mean, var, nll, s, smooth));
}

pssgp_status pssgp_nll(pssgp_model* m, int64_t N, const double* t, const double* y, const uint8_t* mask,
                       double* nll, void* stream) {
    NvtxCall nvtx_("pssgp_nll");
    pssgp_status st = check_args(m, N, t, y, mask);
    if (st) return st;
    if (!nll) return fail(m, PSSGP_E_ARG, "nll is NULL");
    if ((st = ensure_device(m))) return st;
    auto s = static_cast<cudaStream_t>(stream);
    m->last_stream = s;
    if (m->d > kMaxD) return wide_ops_for(m->d)->posterior(m, N, t, y, mask, nullptr, nullptr, nll, s, false);
    DISPATCH_D(m, run_posterior<D_>(m, N, t, y, mask, nullptr, nullptr, nll, s, false));
}

// Optional fp32 path: the thread-per-chain kernels compiled with fp32 state
// (pssgp_f32.cu); single Matern components only.  Same one-wave plan as make_plan with the fp32
// kernels' occupancy (fewer registers: 4 CTAs / SM at d = 3).
Plan make_plan_f32(pssgp_model* m, int64_t N) {
    if (m->occ32 == 0) m->occ32 = pssgp_f32::occupancy(m->d);
    const int bps = m->blocks_per_sm > 0 ? m->blocks_per_sm : m->occ32;
    const int64_t target_chains = static_cast<int64_t>(m->sm_count) * bps * kThreads;
    Plan pl;
    int64_t K = m->forced_K > 0 ? m->forced_K : std::max<int64_t>(1, (N + target_chains - 1) / target_chains);
    if (m->forced_K <= 0 && K > kWin / 4) K = ((K + kWin - 1) / kWin) * kWin;
    pl.K = K;
    pl.nch = std::max<int64_t>(1, (N + K - 1) / K);
    pl.nb = static_cast<int>((pl.nch + kThreads - 1) / kThreads);
    return pl;
}

pssgp_status pssgp_posterior_f32(pssgp_model* m, int64_t N, const double* t, const double* y, const uint8_t* mask,
                                 double* mean, double* var, double* nll, void* stream) {
    NvtxCall nvtx_("pssgp_posterior_f32");
    pssgp_status st = check_args(m, N, t, y, mask);
    if (st) return st;
    if (!m->closed || m->d > 3)
        return fail(m, PSSGP_E_UNSUPPORTED, "the fp32 path covers single Matern components (d <= 3)");
    if (!mean && !var && !nll) return fail(m, PSSGP_E_ARG, "no output requested");
    if ((st = ensure_device(m))) return st;
    auto s = static_cast<cudaStream_t>(stream);
    m->last_stream = s;
    if (N == 0) {
        if (nll) {
            cudaError_t e = cudaMemsetAsync(nll, 0, sizeof(double), s);
            if (e != cudaSuccess) return cuda_fail(m, e, "cudaMemsetAsync");
        }
        return PSSGP_OK;
    }
    const Plan pl = make_plan_f32(m, N);
    pssgp_f32::Run r;
    std::memset(&r, 0, sizeof(r));
    r.d = m->d;
    r.n = N;
    r.K = pl.K;
    r.nb = pl.nb;
    const size_t need = pssgp_f32::ws_bytes(m->d, pl.K, r.nb);
    if (need > m->ws_bytes) {
        if (m->ws) cudaFree(m->ws);
        m->ws = nullptr;
        m->ws_bytes = 0;
        if (cudaMalloc(&m->ws, need) != cudaSuccess) {
            cudaGetLastError();
            return fail(m, PSSGP_E_NOMEM, "cudaMalloc(workspace) failed");
        }
        m->ws_bytes = need;
    }
    r.t = t; r.y = y; r.mask = mask;
    r.mean = mean; r.var = var; r.nll = nll;
    r.ws = m->ws;
    r.err = m->d_err;
    r.flag = m->d_err + 1;
    r.lam = m->lam; r.s2 = m->s2; r.r = m->r;
    switch (m->d) {
#define F32_PINF(DD)                                              \
    case DD: {                                                    \
        ModelParams<DD> mp;                                       \
        fill_params<DD>(m, mp);                                   \
        for (int i = 0; i < ns(DD); ++i) r.Pinf[i] = mp.Pinf[i];  \
        break;                                                    \
    }
        F32_PINF(1) F32_PINF(2) F32_PINF(3)
#undef F32_PINF
    }
    r.stream = s;
    const bool smooth = mean || var;
    cudaError_t e;
    { ProfScope ps(m, S_K1, s); e = pssgp_f32::launch(r, 1); }
    if (e != cudaSuccess) return cuda_fail(m, e, "k_filter_reduce (fp32)");
    { ProfScope ps(m, S_K3, s); e = pssgp_f32::launch(r, 2); }
    if (e != cudaSuccess) return cuda_fail(m, e, "k_filter_apply (fp32)");
    if (smooth) {
        ProfScope ps(m, S_K5, s);
        e = pssgp_f32::launch(r, 3);
    } else {
        ProfScope ps(m, S_K6, s);
        e = pssgp_f32::launch(r, 4);
    }
    if (e != cudaSuccess) return cuda_fail(m, e, smooth ? "k_smoother_apply (fp32)" : "k_nll_sum (fp32)");
    return PSSGP_OK;
}

pssgp_status pssgp_nll_grad(pssgp_model* m, int64_t N, const double* t, const double* y, const uint8_t* mask,
                            double* nll, double* grad, void* stream) {
    NvtxCall nvtx_("pssgp_nll_grad");
    pssgp_status st = check_args(m, N, t, y, mask);
    if (st) return st;
    if (!grad) return fail(m, PSSGP_E_ARG, "grad is NULL");
    if (!m->closed && m->mode != kTable)
        return fail(m, PSSGP_E_UNSUPPORTED, "the gradient of this model needs a uniform grid (options.uniform_dt > 0)");
    if ((st = ensure_device(m))) return st;
    auto s = static_cast<cudaStream_t>(stream);
    m->last_stream = s;
    if (!m->closed) {   // any other model on a uniform grid: reverse mode on the warp-per-chain path
        const WideOps* ops = wide_ops_for(m->d);
        if (!ops) return fail(m, PSSGP_E_UNSUPPORTED, "state dimension not compiled");
        return ops->nll_grad(m, N, t, y, mask, nll, grad, s);
    }
    DISPATCH_D(m, run_grad<D_>(m, N, t, y, mask, nll, grad, s));
}

int pssgp_num_params(const pssgp_model* m) { return m ? static_cast<int>(m->pder.size()) + 1 : -1; }

pssgp_status pssgp_merge_grid(pssgp_model* m, int64_t n_train, const double* t_train, const double* y_train,
                              int64_t n_test, const double* t_test, double* t_out, double* y_out,
                              uint8_t* mask_out, int64_t* test_index, void* stream) {
    if (!m) return PSSGP_E_ARG;
    if (n_train < 0 || n_test < 0 || (n_train > 0 && (!t_train || !y_train)) || (n_test > 0 && (!t_test || !test_index)) ||
        (n_train + n_test > 0 && (!t_out || !y_out || !mask_out)))
        return fail(m, PSSGP_E_ARG, "bad merge arguments");
    pssgp_status st = ensure_device(m);
    if (st) return st;
    auto s = static_cast<cudaStream_t>(stream);
    m->last_stream = s;
    const int64_t tot = n_train + n_test;
    if (tot == 0) return PSSGP_OK;
    const int64_t blocks = (tot + 255) / 256;
    k_merge<<<static_cast<unsigned>(blocks), 256, 0, s>>>(n_train, t_train, y_train, n_test, t_test, t_out, y_out,
                                                         mask_out, test_index, m->d_err);
    LAUNCH_CHECK(m, "k_merge");
    return PSSGP_OK;
}

pssgp_status pssgp_gather(pssgp_model* m, int64_t n_test, const int64_t* test_index, const double* mean,
                          const double* var, double* mean_test, double* var_test, void* stream) {
    if (!m) return PSSGP_E_ARG;
    if (n_test < 0 || (n_test > 0 && !test_index)) return fail(m, PSSGP_E_ARG, "bad gather arguments");
    if (n_test == 0) return PSSGP_OK;
    auto s = static_cast<cudaStream_t>(stream);
    k_gather<<<static_cast<unsigned>((n_test + 255) / 256), 256, 0, s>>>(n_test, test_index, mean, var, mean_test,
                                                                          var_test);
    LAUNCH_CHECK(m, "k_gather");
    return PSSGP_OK;
}

pssgp_status pssgp_predict(pssgp_model* m, int64_t n_train, const double* t_train, const double* y_train,
                           int64_t n_test, const double* t_test, double* mean_test, double* var_test, double* nll,
                           void* stream) {
    NvtxCall nvtx_("pssgp_predict");
    if (!m) return PSSGP_E_ARG;
    if (n_train < 0 || n_test < 0) return fail(m, PSSGP_E_ARG, "negative size");
    if ((n_train > 0 && (!t_train || !y_train)) || (n_test > 0 && (!t_test || !mean_test || !var_test)))
        return fail(m, PSSGP_E_ARG, "NULL input/output array");
    pssgp_status st = ensure_device(m);
    if (st) return st;
    const size_t tot = static_cast<size_t>(n_train + n_test);
    const size_t need = tot * (8 + 8 + 8 + 8 + 1) + static_cast<size_t>(n_test) * 8 + 64;
    if (need > m->mg_bytes) {
        if (m->mg) cudaFree(m->mg);
        m->mg = nullptr;
        m->mg_bytes = 0;
        if (cudaMalloc(&m->mg, need) != cudaSuccess) {
            cudaGetLastError();
            return fail(m, PSSGP_E_NOMEM, "cudaMalloc(merge buffers)");
        }
        m->mg_bytes = need;
    }
    double* tg = reinterpret_cast<double*>(m->mg);
    double* yg = tg + tot;
    double* mean = yg + tot;
    double* var = mean + tot;
    int64_t* idx = reinterpret_cast<int64_t*>(var + tot);
    uint8_t* mk = reinterpret_cast<uint8_t*>(idx + n_test);
    if ((st = pssgp_merge_grid(m, n_train, t_train, y_train, n_test, t_test, tg, yg, mk, idx, stream))) return st;
    if ((st = pssgp_posterior(m, static_cast<int64_t>(tot), tg, yg, mk, mean, var, nll, stream))) return st;
    return pssgp_gather(m, n_test, idx, mean, var, mean_test, var_test, stream);
}

// the launch plan the batched kernels use (same as make_plan<D>; sizes the NLL piece buffers)
Plan batch_plan(pssgp_model* m, int64_t N) {
    switch (m->d) {
        case 1: return make_plan<1>(m, N);
        case 2: return make_plan<2>(m, N);
        default: return make_plan<3>(m, N);
    }
}

pssgp_status pssgp_posterior_batched(pssgp_model* m, int nseg, const int64_t* offsets, const double* variance,
                                     const double* lengthscale, const double* noise_var, int64_t N,
                                     const double* t, const double* y, const uint8_t* mask, double* mean,
                                     double* var, double* nll, void* stream) {
    NvtxCall nvtx_("pssgp_posterior_batched");
    pssgp_status st = check_args(m, N, t, y, mask);
    if (st) return st;
    if (nseg < 1 || !offsets || !nll) return fail(m, PSSGP_E_ARG, "bad batched arguments");
    if (!m->closed) return fail(m, PSSGP_E_UNSUPPORTED, "batched mode needs a single closed-form Matern model");
    if ((st = ensure_device(m))) return st;
    auto s = static_cast<cudaStream_t>(stream);
    m->last_stream = s;
    const Plan bpl = batch_plan(m, std::max<int64_t>(N, 1));
    const size_t nchp = static_cast<size_t>(bpl.nb) * kThreads;
    const size_t need = 2 * nchp * sizeof(double);   // NLL head / tail pieces per chain
    if (need > m->bt_bytes) {
        if (m->bt) cudaFree(m->bt);
        m->bt = nullptr;
        m->bt_bytes = 0;
        if (cudaMalloc(&m->bt, need) != cudaSuccess) {
            cudaGetLastError();
            return fail(m, PSSGP_E_NOMEM, "cudaMalloc(batched)");
        }
        m->bt_bytes = need;
    }
    pssgp::batch::BParams q;
    q.off = offsets;
    q.nseg = nseg;
    q.var = variance;
    q.ell = lengthscale;
    q.noise = noise_var;
    q.sqrt2nu = std::sqrt(2.0 * m->d - 1.0);
    q.nll_head = m->bt;
    q.nll_tail = m->bt + nchp;
    q.nll_seg = nll;
    pssgp::batch::k_batch_check_offsets<<<(nseg + 256) / 256, 256, 0, s>>>(offsets, nseg, N, m->d_err);
    LAUNCH_CHECK(m, "k_batch_check_offsets");
    if (N > 0) {
        switch (m->d) {
#define BATCH_RUN(DD)                                                                                   \
    case DD: {                                                                                          \
        const Plan pl = make_plan<DD>(m, N);                                                            \
        KParams<DD> p;                                                                                  \
        if ((st = setup<DD>(m, pl, p))) return st;                                                      \
        p.t = t; p.y = y; p.mask = mask; p.n = N; p.k0 = 0; p.nglob = N; p.mean = mean; p.var = var;    \
        { ProfScope ps(m, S_K1, s); pssgp::batch::k_batch_filter_reduce<DD><<<pl.nb, kThreads, 0, s>>>(p, q); } \
        LAUNCH_CHECK(m, "k_batch_filter_reduce");                                                       \
        { ProfScope ps(m, S_K3, s); pssgp::batch::k_batch_filter_apply<DD><<<pl.nb, kThreads, 0, s>>>(p, q); } \
        LAUNCH_CHECK(m, "k_batch_filter_apply");                                                        \
        { ProfScope ps(m, S_K5, s); pssgp::batch::k_batch_smoother_apply<DD><<<pl.nb, kThreads, 0, s>>>(p, q); } \
        LAUNCH_CHECK(m, "k_batch_smoother_apply");                                                      \
        break;                                                                                          \
    }
            BATCH_RUN(1) BATCH_RUN(2) BATCH_RUN(3)
#undef BATCH_RUN
            default: return fail(m, PSSGP_E_UNSUPPORTED, "state dimension");
        }
    }
    {
        ProfScope ps(m, S_K6, s);
        pssgp::batch::k_batch_nll<<<(nseg + 3) / 4, 128, 0, s>>>(q, bpl.K);
    }
    LAUNCH_CHECK(m, "k_batch_nll");
    return PSSGP_OK;
}

pssgp_status pssgp_nll_grad_batched(pssgp_model* m, int nseg, const int64_t* offsets, const double* variance,
                                    const double* lengthscale, const double* noise_var, int64_t N, const double* t,
                                    const double* y, const uint8_t* mask, double* nll, double* grad, void* stream) {
    NvtxCall nvtx_("pssgp_nll_grad_batched");
    pssgp_status st = check_args(m, N, t, y, mask);
    if (st) return st;
    if (nseg < 1 || !offsets || !nll || !grad) return fail(m, PSSGP_E_ARG, "bad batched-gradient arguments");
    if (!m->closed || m->d > kMaxD)
        return fail(m, PSSGP_E_UNSUPPORTED, "batched gradient needs a single closed-form Matern model");
    if ((st = ensure_device(m))) return st;
    auto s = static_cast<cudaStream_t>(stream);
    m->last_stream = s;
    const Plan bpl = batch_plan(m, std::max<int64_t>(N, 1));
    const size_t nchp = static_cast<size_t>(bpl.nb) * kThreads;
    const size_t need = 2 * nchp * sizeof(double);   // NLL head / tail pieces per chain
    if (need > m->bt_bytes) {
        if (m->bt) cudaFree(m->bt);
        m->bt = nullptr;
        m->bt_bytes = 0;
        if (cudaMalloc(&m->bt, need) != cudaSuccess) {
            cudaGetLastError();
            return fail(m, PSSGP_E_NOMEM, "cudaMalloc(batched)");
        }
        m->bt_bytes = need;
    }
    pssgp::batch::BParams q;
    q.off = offsets;
    q.nseg = nseg;
    q.var = variance;
    q.ell = lengthscale;
    q.noise = noise_var;
    q.sqrt2nu = std::sqrt(2.0 * m->d - 1.0);
    q.nll_head = m->bt;
    q.nll_tail = m->bt + nchp;
    q.nll_seg = nll;
    pssgp::batch::k_batch_check_offsets<<<(nseg + 256) / 256, 256, 0, s>>>(offsets, nseg, N, m->d_err);
    LAUNCH_CHECK(m, "k_batch_check_offsets");
    if (N == 0) {
        cudaError_t e = cudaMemsetAsync(nll, 0, nseg * sizeof(double), s);
        if (e == cudaSuccess) e = cudaMemsetAsync(grad, 0, 3 * nseg * sizeof(double), s);
        if (e != cudaSuccess) return cuda_fail(m, e, "cudaMemsetAsync");
        return PSSGP_OK;
    }
    switch (m->d) {
#define BGRAD_RUN(DD)                                                                                      \
    case DD: {                                                                                             \
        const Plan pl = make_plan<DD>(m, N);                                                               \
        KParams<DD> p;                                                                                     \
        if ((st = setup<DD>(m, pl, p))) return st;                                                         \
        p.t = t; p.y = y; p.mask = mask; p.n = N; p.k0 = 0; p.nglob = N;                                   \
        const size_t gnch = static_cast<size_t>(pl.nb) * kThreads;                                        \
        const size_t na = sizeof(TAgg3<DD>) / sizeof(double);                                             \
        const size_t gneed = 2 * gnch * na * sizeof(double);                                               \
        if (gneed > m->gb_bytes) {                                                                         \
            if (m->gb) cudaFree(m->gb);                                                                    \
            m->gb = nullptr;                                                                               \
            m->gb_bytes = 0;                                                                               \
            if (cudaMalloc(&m->gb, gneed) != cudaSuccess) {                                                \
                cudaGetLastError();                                                                        \
                return fail(m, PSSGP_E_NOMEM, "cudaMalloc(batched gradient)");                             \
            }                                                                                              \
            m->gb_bytes = gneed;                                                                           \
        }                                                                                                  \
        double* head = m->gb;                                                                              \
        double* tail = m->gb + gnch * na;                                                                  \
        { ProfScope ps(m, S_K1, s); pssgp::batch::k_batch_filter_reduce<DD><<<pl.nb, kThreads, 0, s>>>(p, q); } \
        LAUNCH_CHECK(m, "k_batch_filter_reduce");                                                          \
        { ProfScope ps(m, S_K3, s); pssgp::batch::k_batch_filter_apply<DD><<<pl.nb, kThreads, 0, s>>>(p, q); } \
        LAUNCH_CHECK(m, "k_batch_filter_apply");                                                           \
        { ProfScope ps(m, S_GRAD, s); k_batch_grad_fold<DD><<<pl.nb, kThreads, 0, s>>>(p, q, head, tail, grad); } \
        LAUNCH_CHECK(m, "k_batch_grad_fold");                                                              \
        { ProfScope ps(m, S_RED, s); k_batch_grad_combine<DD><<<(nseg + 127) / 128, 128, 0, s>>>(q, pl.K, head, tail, grad); } \
        LAUNCH_CHECK(m, "k_batch_grad_combine");                                                           \
        { ProfScope ps(m, S_RED, s); k_batch_grad_combine_long<DD><<<nseg, kThreads, 0, s>>>(q, pl.K, head, tail, grad); } \
        LAUNCH_CHECK(m, "k_batch_grad_combine_long");                                                      \
        break;                                                                                             \
    }
        BGRAD_RUN(1) BGRAD_RUN(2) BGRAD_RUN(3)
#undef BGRAD_RUN
        default: return fail(m, PSSGP_E_UNSUPPORTED, "state dimension");
    }
    {
        ProfScope ps(m, S_K6, s);
        pssgp::batch::k_batch_nll<<<(nseg + 3) / 4, 128, 0, s>>>(q, bpl.K);
    }
    LAUNCH_CHECK(m, "k_batch_nll");
    return PSSGP_OK;
}

}  // extern "C"

namespace {
// DFMA throughput probe (pssgp_measure_fp64_peak): 8 independent FMA chains per thread hide the
// pipe latency; MODE 0 three register operands, MODE 1 a constant-bank addend (the form the
// closed-form discretisation uses).
__constant__ double c_fp64_probe[8] = {1.0000001, 0.9999999, 1.0000002, 0.9999998,
                                       1.0000003, 0.9999997, 1.0000004, 0.9999996};
template <int MODE>
__global__ void __launch_bounds__(256) k_fp64_probe(double* out, int iters, double s) {
    double acc[8], x[8], y[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc[i] = threadIdx.x * 1e-3 + i; x[i] = s + i * 1e-7; y[i] = 1e-9 * i - s * 1e-3; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], x[i], MODE == 0 ? y[i] : c_fp64_probe[i]);
    }
    double r = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
}  // namespace

extern "C" {

pssgp_status pssgp_measure_fp64_peak(pssgp_model* m, double* tflops) {
    if (!m || !tflops) return PSSGP_E_ARG;
    pssgp_status st = ensure_device(m);
    if (st) return st;
    const int blocks = m->sm_count * 8, threads = 256, iters = 4096;
    double* out = nullptr;
    if (cudaMalloc(&out, sizeof(double) * blocks * threads) != cudaSuccess) {
        cudaGetLastError();
        return fail(m, PSSGP_E_NOMEM, "cudaMalloc(fp64 probe)");
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double best = 0.0;
    for (int rep = 0; rep < 6; ++rep) {
        const int mode = rep & 1;
        if (mode == 0) k_fp64_probe<0><<<blocks, threads>>>(out, 16, 1.0);
        else k_fp64_probe<1><<<blocks, threads>>>(out, 16, 1.0);
        cudaEventRecord(a);
        if (mode == 0) k_fp64_probe<0><<<blocks, threads>>>(out, iters, 1.0);
        else k_fp64_probe<1><<<blocks, threads>>>(out, iters, 1.0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        const double flop = 2.0 * blocks * threads * static_cast<double>(iters) * 8;
        if (ms > 0.f) best = std::max(best, flop / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(m, e, "fp64 probe");
    *tflops = best;
    return PSSGP_OK;
}

// batched series with per-series log hyper-parameters (pssgp_batch_theta.cuh)
static pssgp_status batched_theta(pssgp_model* m, int nseg, const int64_t* offsets, const double* theta, int64_t N,
                                  const double* t, const double* y, const uint8_t* mask, double* mean, double* var,
                                  double* nll, double* grad, void* stream) {
    pssgp_status st = check_args(m, N, t, y, mask);
    if (st) return st;
    if (nseg < 1 || !offsets || !theta || !nll) return fail(m, PSSGP_E_ARG, "bad batched-theta arguments");
    if (!m->bt_ok || !(m->udt > 0.0))
        return fail(m, PSSGP_E_UNSUPPORTED,
                    "batched per-series hyper-parameters need Matern / periodic / quasi-periodic components on a "
                    "uniform grid (options.uniform_dt > 0)");
    if ((st = ensure_device(m))) return st;
    auto s = static_cast<cudaStream_t>(stream);
    m->last_stream = s;
    pssgp::batch::k_batch_check_offsets<<<(nseg + 256) / 256, 256, 0, s>>>(offsets, nseg, N, m->d_err);
    LAUNCH_CHECK(m, "k_batch_check_offsets");
    const WideOps* ops = wide_ops_for(m->d);
    if (!ops) return fail(m, PSSGP_E_UNSUPPORTED, "state dimension not compiled");
    return ops->batched_theta(m, nseg, offsets, theta, N, t, y, mask, mean, var, nll, grad, s);
}

pssgp_status pssgp_posterior_batched_theta(pssgp_model* m, int nseg, const int64_t* offsets, const double* theta,
                                           int64_t N, const double* t, const double* y, const uint8_t* mask,
                                           double* mean, double* var, double* nll, void* stream) {
    NvtxCall nvtx_("pssgp_posterior_batched_theta");
    return batched_theta(m, nseg, offsets, theta, N, t, y, mask, mean, var, nll, nullptr, stream);
}

pssgp_status pssgp_nll_grad_batched_theta(pssgp_model* m, int nseg, const int64_t* offsets, const double* theta,
                                          int64_t N, const double* t, const double* y, const uint8_t* mask,
                                          double* nll, double* grad, void* stream) {
    NvtxCall nvtx_("pssgp_nll_grad_batched_theta");
    if (!grad) return fail(m, PSSGP_E_ARG, "grad is NULL");
    return batched_theta(m, nseg, offsets, theta, N, t, y, mask, nullptr, nullptr, nll, grad, stream);
}

pssgp_status pssgp_check(pssgp_model* m) {
    if (!m) return PSSGP_E_ARG;
    if (!m->d_err) return PSSGP_OK;
    cudaError_t e = cudaStreamSynchronize(m->last_stream);
    if (e != cudaSuccess) return cuda_fail(m, e, "cudaStreamSynchronize");
    unsigned long long w = 0;
    e = cudaMemcpy(&w, m->d_err, sizeof(w), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(m, e, "cudaMemcpy(error word)");
    if (w == ~0ULL) return PSSGP_OK;
    cudaMemset(m->d_err, 0xff, sizeof(unsigned long long));
    cudaMemset(m->d_err + 1, 0, 7 * sizeof(unsigned long long));   // K3 publication flag, ticket, counters
    const unsigned code = static_cast<unsigned>(w & 0xff);
    const int64_t idx = static_cast<int64_t>((w >> 8) & 0xffffffffffffULL);
    const char* what = code == kErrInput ? "invalid input (unsorted/non-finite t or non-finite observed y)"
                       : code == kErrNumeric ? "numerical failure (S <= 0 or non-PD predicted covariance)"
                                             : "dt differs from the declared uniform_dt (use uniform_dt = 0 for "
                                               "per-step device discretisation)";
    return fail(m, static_cast<pssgp_status>(code), std::string(what) + " at step " + std::to_string(idx), idx);
}

int64_t pssgp_error_index(const pssgp_model* m) { return m ? m->err_index : -1; }

const char* pssgp_last_error(const pssgp_model* m) { return m ? m->last_err.c_str() : "NULL handle"; }

pssgp_status pssgp_posterior_host(pssgp_model* m, int64_t N, const double* t, const double* y, const uint8_t* mask,
                                  double* mean, double* var, double* nll, void* stream) {
    pssgp_status st = check_args(m, N, t, y, mask);
    if (st) return st;
    if ((st = ensure_device(m))) return st;
    auto s = static_cast<cudaStream_t>(stream);
    const size_t nd = static_cast<size_t>(N);
    const size_t need = nd * (8 + 8 + 8 + 8) + nd + 64;
    if (need > m->io_bytes) {
        if (m->io) cudaFree(m->io);
        m->io = nullptr;
        m->io_bytes = 0;
        if (cudaMalloc(&m->io, need) != cudaSuccess) {
            cudaGetLastError();
            return fail(m, PSSGP_E_NOMEM, "cudaMalloc(io)");
        }
        m->io_bytes = need;
    }
    double* dt_ = reinterpret_cast<double*>(m->io);
    double* dy = dt_ + nd;
    double* dmean = dy + nd;
    double* dvar = dmean + nd;
    uint8_t* dmask = reinterpret_cast<uint8_t*>(dvar + nd);
    if (N > 0) {
        cudaMemcpyAsync(dt_, t, nd * 8, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(dy, y, nd * 8, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(dmask, mask, nd, cudaMemcpyHostToDevice, s);
    }
    st = pssgp_posterior(m, N, dt_, dy, dmask, mean ? dmean : nullptr, var ? dvar : nullptr,
                         nll ? m->d_scalar : nullptr, stream);
    if (st) return st;
    if (N > 0 && mean) cudaMemcpyAsync(mean, dmean, nd * 8, cudaMemcpyDeviceToHost, s);
    if (N > 0 && var) cudaMemcpyAsync(var, dvar, nd * 8, cudaMemcpyDeviceToHost, s);
    if (nll) cudaMemcpyAsync(nll, m->d_scalar, 8, cudaMemcpyDeviceToHost, s);
    m->last_stream = s;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(m, e, "pssgp_posterior_host copies");
    return pssgp_check(m);
}

pssgp_status pssgp_posterior_host_async(pssgp_model* m, int64_t N, const double* t, const double* y,
                                        const uint8_t* mask, double* mean, double* var, double* nll) {
    pssgp_status st = check_args(m, N, t, y, mask);
    if (st) return st;
    if ((st = ensure_device(m))) return st;
    if (!m->acs) {
        bool ok = cudaStreamCreateWithFlags(&m->acs, cudaStreamNonBlocking) == cudaSuccess;
        for (int i = 0; i < 2; ++i) {
            ok = ok && cudaStreamCreateWithFlags(&m->astream[i], cudaStreamNonBlocking) == cudaSuccess;
            ok = ok && cudaStreamCreateWithFlags(&m->aout[i], cudaStreamNonBlocking) == cudaSuccess;
            ok = ok && cudaEventCreateWithFlags(&m->ev_in[i], cudaEventDisableTiming) == cudaSuccess;
            ok = ok && cudaEventCreateWithFlags(&m->ev_comp[i], cudaEventDisableTiming) == cudaSuccess;
            ok = ok && cudaEventCreateWithFlags(&m->ev_out[i], cudaEventDisableTiming) == cudaSuccess;
        }
        if (!ok) return fail(m, PSSGP_E_CUDA, "cudaStreamCreate / cudaEventCreate");
    }
    const int slot = m->aslot;
    m->aslot ^= 1;
    cudaStream_t sin = m->astream[slot], sout = m->aout[slot], sc = m->acs;
    const size_t nd = static_cast<size_t>(N);
    const size_t need = nd * (8 + 8 + 8 + 8) + nd + 64;
    if (need > m->aio_bytes[slot]) {
        if (m->aio[slot]) cudaFree(m->aio[slot]);      // synchronising: the slot's last call is done
        m->aio[slot] = nullptr;
        m->aio_bytes[slot] = 0;
        if (cudaMalloc(&m->aio[slot], need) != cudaSuccess) {
            cudaGetLastError();
            return fail(m, PSSGP_E_NOMEM, "cudaMalloc(async io)");
        }
        m->aio_bytes[slot] = need;
    }
    double* dnll = reinterpret_cast<double*>(m->aio[slot]);
    double* dt_ = dnll + 8;
    double* dy = dt_ + nd;
    double* dmean = dy + nd;
    double* dvar = dmean + nd;
    uint8_t* dmask = reinterpret_cast<uint8_t*>(dvar + nd);
    // host -> device: the slot's input buffers are free once its previous compute has run; the copy
    // does not wait for that call's device -> host copies (separate stream), so consecutive calls'
    // inputs stream back to back while earlier outputs drain the other direction
    if (m->arec[slot]) cudaStreamWaitEvent(sin, m->ev_comp[slot], 0);
    if (N > 0) {
        cudaMemcpyAsync(dt_, t, nd * 8, cudaMemcpyHostToDevice, sin);
        cudaMemcpyAsync(dy, y, nd * 8, cudaMemcpyHostToDevice, sin);
        cudaMemcpyAsync(dmask, mask, nd, cudaMemcpyHostToDevice, sin);
    }
    cudaEventRecord(m->ev_in[slot], sin);
    // compute (one stream: calls in order, never sharing the GPU): after the inputs, and after the
    // slot's previous outputs have left (the compute overwrites them)
    cudaStreamWaitEvent(sc, m->ev_in[slot], 0);
    if (m->arec[slot]) cudaStreamWaitEvent(sc, m->ev_out[slot], 0);
    st = pssgp_posterior(m, N, dt_, dy, dmask, mean ? dmean : nullptr, var ? dvar : nullptr, nll ? dnll : nullptr,
                         sc);
    if (st) return st;
    cudaEventRecord(m->ev_comp[slot], sc);
    cudaStreamWaitEvent(sout, m->ev_comp[slot], 0);
    if (N > 0 && mean) cudaMemcpyAsync(mean, dmean, nd * 8, cudaMemcpyDeviceToHost, sout);
    if (N > 0 && var) cudaMemcpyAsync(var, dvar, nd * 8, cudaMemcpyDeviceToHost, sout);
    if (nll) cudaMemcpyAsync(nll, dnll, 8, cudaMemcpyDeviceToHost, sout);
    cudaEventRecord(m->ev_out[slot], sout);
    m->arec[slot] = true;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(m, e, "pssgp_posterior_host_async copies");
    return PSSGP_OK;
}

pssgp_status pssgp_sync(pssgp_model* m) {
    if (!m) return PSSGP_E_ARG;
    for (int i = 0; i < 2; ++i) {
        if (m->aout[i]) {
            cudaError_t e = cudaStreamSynchronize(m->aout[i]);
            if (e != cudaSuccess) return cuda_fail(m, e, "cudaStreamSynchronize(async)");
        }
        if (m->astream[i]) cudaStreamSynchronize(m->astream[i]);
    }
    if (m->acs) cudaStreamSynchronize(m->acs);
    return pssgp_check(m);
}

pssgp_status pssgp_get_ssm(const pssgp_model* m, double* G, double* W, double* H, double* Pinf, double* D) {
    if (!m) return PSSGP_E_ARG;
    const int n = m->d;
    for (int i = 0; i < n * n; ++i) {
        if (G) G[i] = static_cast<double>(m->ssm.G[i]);
        if (W) W[i] = static_cast<double>(m->ssm.W[i]);
        if (Pinf) Pinf[i] = static_cast<double>(m->ssm.Pinf[i]);
    }
    for (int i = 0; i < n; ++i) {
        if (H) H[i] = static_cast<double>(m->ssm.H[i]);
        if (D) D[i] = static_cast<double>(m->ssm.Dbal[i]);
    }
    return PSSGP_OK;
}

pssgp_status pssgp_debug_discretize(const pssgp_model* m, double dt, double* F, double* Q) {
    if (!m || !F || !Q) return PSSGP_E_ARG;
    pssgp_model* mm = const_cast<pssgp_model*>(m);
    if (m->d > kMaxD && m->mode == kPade && dt != 0.0) {
        // per-step device discretisation (kw_discretize): run it on the device for one step
        const WideOps* ops = wide_ops_for(m->d);
        if (!ops) return fail(mm, PSSGP_E_UNSUPPORTED, "state dimension not compiled");
        return ops->debug_disc(mm, dt, F, Q);
    }
    if (m->d > kMaxD) {   // mirrors wide::wdisc_kind
        const int d = m->d;
        const bool tab = (m->udt > 0.0 && std::fabs(dt - m->udt) <= 1e-12 * m->udt), zero = (dt == 0.0);
        for (int i = 0; i < d * d; ++i) {
            F[i] = tab ? m->Fu[i] : ((zero && i % (d + 1) == 0) ? 1.0 : 0.0);
            Q[i] = tab ? m->Qu[i] : 0.0;
        }
        return (tab || zero) ? PSSGP_OK : PSSGP_E_UNSUPPORTED;
    }
    DISPATCH_D(mm, debug_disc<D_>(m, dt, F, Q));
}

pssgp_status pssgp_plan_f32(pssgp_model* m, int64_t N, int64_t* chain_len, int64_t* n_chains, int* n_blocks,
                            int* threads_per_block) {
    if (!m || N < 0) return PSSGP_E_ARG;
    if (!m->closed || m->d > 3) return PSSGP_E_UNSUPPORTED;
    pssgp_status st = ensure_device(m);
    if (st) return st;
    const Plan pl = make_plan_f32(m, N);
    if (chain_len) *chain_len = pl.K;
    if (n_chains) *n_chains = pl.nch;
    if (n_blocks) *n_blocks = pl.nb;
    if (threads_per_block) *threads_per_block = kThreads;
    return PSSGP_OK;
}

pssgp_status pssgp_plan(pssgp_model* m, int64_t N, int64_t* chain_len, int64_t* n_chains, int* n_blocks,
                        int* threads_per_block) {
    if (!m || N < 0) return PSSGP_E_ARG;
    pssgp_status st = ensure_device(m);
    if (st) return st;
    Plan pl;
    switch (m->d) {
        case 1: pl = make_plan<1>(m, N); break;
        case 2: pl = make_plan<2>(m, N); break;
        case 3: pl = make_plan<3>(m, N); break;
        default: {
            const WideOps* ops = wide_ops_for(m->d);
            if (!ops) return PSSGP_E_UNSUPPORTED;
            ops->plan(m, N, chain_len, n_chains, n_blocks, threads_per_block);
            return PSSGP_OK;
        }
    }
    if (chain_len) *chain_len = pl.K;
    if (n_chains) *n_chains = pl.nch;
    if (n_blocks) *n_blocks = pl.nb;
    if (threads_per_block) *threads_per_block = kThreads;
    return PSSGP_OK;
}

void pssgp_profile_enable(pssgp_model* m, int on) {
    if (m) m->prof = (on != 0);
}

int pssgp_profile_read(pssgp_model* m, double* ms, int64_t* launches, int cap) {
    if (!m) return 0;
    const int n = std::min(cap, kSlots);
    for (int s = 0; s < kSlots; ++s) {
        double acc = 0.0;
        for (auto& pr : m->ev[s]) {
            cudaEventSynchronize(pr.second);
            float x = 0.f;
            cudaEventElapsedTime(&x, pr.first, pr.second);
            acc += x;
            m->ev_pool.push_back(pr.first);
            m->ev_pool.push_back(pr.second);
        }
        if (s < n) {
            if (ms) ms[s] = acc;
            if (launches) launches[s] = static_cast<int64_t>(m->ev[s].size());
        }
        m->ev[s].clear();
    }
    return n;
}

const char* pssgp_profile_name(int slot) { return slot_name(slot); }

// ---------------------------------------------------------------- sharded path
size_t pssgp_aggregate_bytes(const pssgp_model* m, int which) {
    if (!m) return 0;
    const int d = m->d;
    int fn = d * d + 2 * d + d * (d + 1);
    int sn = d * d + d + d * (d + 1) / 2;
    if (d > kMaxD) {                 // wide path stores full matrices
        fn = 3 * d * d + 2 * d;
        sn = 2 * d * d + d;
    }
    return static_cast<size_t>(which == 0 ? fn : sn + 1) * sizeof(double);   // smoother blob: + NLL partial
}

}  // extern "C"

namespace {

template <int D>
pssgp_status shard_setup(pssgp_model* m, int64_t k0, int64_t n, int64_t Ng, KParams<D>& p, Plan& pl) {
    pl = make_plan<D>(m, n);
    pssgp_status st = setup<D>(m, pl, p);
    if (st) return st;
    p.n = n; p.k0 = k0; p.nglob = Ng;
    return PSSGP_OK;
}

template <int D>
pssgp_status shard_reduce(pssgp_model* m, int64_t k0, int64_t n, int64_t Ng, const double* t, const double* y,
                          const uint8_t* mask, void* out, cudaStream_t s) {
    KParams<D> p;
    Plan pl;
    pssgp_status st = shard_setup<D>(m, k0, n, Ng, p, pl);
    if (st) return st;
    p.t = t; p.y = y; p.mask = mask;
    if ((st = phase_filter_reduce<D>(m, p, s))) return st;
    ProfScope ps(m, S_RED, s);
    k_reduce_blocks<D, FAgg<D>><<<1, kCarryThreads, 0, s>>>(p.block_f, p.nb, static_cast<double*>(out), p.err, k0);
    LAUNCH_CHECK(m, "k_reduce_blocks(filter)");
    return PSSGP_OK;
}

template <int D>
pssgp_status shard_fapply(pssgp_model* m, int64_t k0, int64_t n, int64_t Ng, const double* t, const double* y,
                          const uint8_t* mask, const void* all, int rank, int world, void* sout, double* nllp,
                          cudaStream_t s) {
    KParams<D> p;
    Plan pl;
    pssgp_status st = shard_setup<D>(m, k0, n, Ng, p, pl);
    if (st) return st;
    p.t = t; p.y = y; p.mask = mask;
    p.in_filt = static_cast<const double*>(all);
    p.rank = rank; p.world = world;
    if ((st = phase_filter_apply<D>(m, p, s))) return st;
    // the chunk's NLL partial travels in the smoother blob, after the aggregate
    if ((st = nll_sum(m, p.nll_block, p.nb, static_cast<double*>(sout) + SN(D), s))) return st;
    if (nllp && (st = nll_sum(m, p.nll_block, p.nb, nllp, s))) return st;
    ProfScope ps(m, S_RED, s);
    k_reduce_blocks<D, SAgg<D>><<<1, kCarryThreads, 0, s>>>(p.block_s, p.nb, static_cast<double*>(sout), nullptr, 0);
    LAUNCH_CHECK(m, "k_reduce_blocks(smoother)");
    return PSSGP_OK;
}

template <int D>
pssgp_status shard_sapply(pssgp_model* m, int64_t k0, int64_t n, int64_t Ng, const double* t, const void* all,
                          int rank, int world, double* mean, double* var, double* nll, cudaStream_t s) {
    KParams<D> p;
    Plan pl;
    pssgp_status st = shard_setup<D>(m, k0, n, Ng, p, pl);
    if (st) return st;
    p.t = t;
    p.in_smooth = static_cast<const double*>(all);
    p.rank = rank; p.world = world;
    p.mean = mean; p.var = var;
    if ((st = phase_smoother<D>(m, p, s))) return st;
    // total NLL: fixed-order sum over ranks of the partials carried in the gathered blobs
    if (nll) return nll_sum(m, static_cast<const double*>(all) + SN(D), world, nll, s, SN(D) + 1);
    return PSSGP_OK;
}

pssgp_status shard_args(pssgp_model* m, int64_t k0, int64_t n, int64_t Ng, const double* t) {
    if (!m) return PSSGP_E_ARG;
    if (k0 < 0 || n < 1 || Ng < 1 || k0 + n > Ng || !t) return fail(m, PSSGP_E_ARG, "bad shard arguments");
    return ensure_device(m);
}

}  // namespace

extern "C" {

pssgp_status pssgp_shard_filter_reduce(pssgp_model* m, int64_t k0, int64_t n, int64_t N_global, const double* t,
                                       const double* y, const uint8_t* mask, void* filt_agg_out, void* stream) {
    NvtxCall nvtx_("pssgp_shard_filter_reduce");
    pssgp_status st = shard_args(m, k0, n, N_global, t);
    if (st) return st;
    if (!y || !mask || !filt_agg_out) return fail(m, PSSGP_E_ARG, "NULL argument");
    auto s = static_cast<cudaStream_t>(stream);
    m->last_stream = s;
    m->sh_k0 = k0; m->sh_n = n; m->sh_N = N_global;
    if (m->d > kMaxD) return wide_ops_for(m->d)->shard_reduce(m, k0, n, N_global, t, y, mask, filt_agg_out, s);
    DISPATCH_D(m, shard_reduce<D_>(m, k0, n, N_global, t, y, mask, filt_agg_out, s));
}

pssgp_status pssgp_shard_filter_apply(pssgp_model* m, int64_t k0, int64_t n, int64_t N_global, const double* t,
                                      const double* y, const uint8_t* mask, const void* all_filt_aggs, int rank,
                                      int world, void* smooth_agg_out, double* nll_partial, void* stream) {
    NvtxCall nvtx_("pssgp_shard_filter_apply");
    pssgp_status st = shard_args(m, k0, n, N_global, t);
    if (st) return st;
    if (!y || !mask || !all_filt_aggs || !smooth_agg_out || rank < 0 || rank >= world)
        return fail(m, PSSGP_E_ARG, "bad argument");
    if (m->sh_k0 != k0 || m->sh_n != n || m->sh_N != N_global)
        return fail(m, PSSGP_E_ARG, "shard phases called with different chunk arguments");
    auto s = static_cast<cudaStream_t>(stream);
    m->last_stream = s;
    if (m->d > kMaxD) {
        return wide_ops_for(m->d)->shard_fapply(m, k0, n, N_global, t, y, mask, all_filt_aggs, rank, world,
                                                smooth_agg_out, nll_partial, s);
    }
    DISPATCH_D(m, shard_fapply<D_>(m, k0, n, N_global, t, y, mask, all_filt_aggs, rank, world, smooth_agg_out,
                                   nll_partial, s));
}

pssgp_status pssgp_shard_smoother_apply(pssgp_model* m, int64_t k0, int64_t n, int64_t N_global, const double* t,
                                        const void* all_smooth_aggs, int rank, int world, double* mean, double* var,
                                        double* nll, void* stream) {
    NvtxCall nvtx_("pssgp_shard_smoother_apply");
    pssgp_status st = shard_args(m, k0, n, N_global, t);
    if (st) return st;
    if (!all_smooth_aggs || rank < 0 || rank >= world) return fail(m, PSSGP_E_ARG, "bad argument");
    if (m->sh_k0 != k0 || m->sh_n != n || m->sh_N != N_global)
        return fail(m, PSSGP_E_ARG, "shard phases called with different chunk arguments");
    auto s = static_cast<cudaStream_t>(stream);
    m->last_stream = s;
    if (m->d > kMaxD) {
        return wide_ops_for(m->d)->shard_sapply(m, k0, n, N_global, t, all_smooth_aggs, rank, world, mean, var, nll, s);
    }
    DISPATCH_D(m, shard_sapply<D_>(m, k0, n, N_global, t, all_smooth_aggs, rank, world, mean, var, nll, s));
}

}  // extern "C"
