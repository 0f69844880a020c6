// pssgp_batch.cuh — batched independent problems (NEXT row f2).
//
// B independent series, concatenated along the time axis (offsets[b]..offsets[b+1]),
// each with its own Matern hyper-parameters (sigma_b^2, ell_b, sigma_n,b^2): the
// multi-start / HMC workloads of PAPER.md:206, 224 in one launch.  No new algebra
// is needed: the first element of every series has A = 0 (Eq. (7)), so the forward
// scan's carry cannot cross a series start, and the terminal element of every series
// has E = 0, so the reverse scan's carry cannot cross a series end — the three-pass
// kernels of pssgp_kernels.cuh apply unchanged to the concatenation, with
//   * series starts handled like the global first step (F = 0, Q = P_inf,b),
//   * series ends like the global terminal (chain smoother aggregate (0, m^s, P^s),
//     RTS reset m^s = xbar, P^s = P),
//   * per-series discretisation (lambda_b, sigma_b^2) and noise r_b,
//   * per-step NLL terms reduced per series in fixed order (deterministic).
// Closed-form Matern models (d <= 3) only; per-step work is the d <= 3 path's.
#pragma once
#include "pssgp_kernels.cuh"

namespace pssgp {
namespace batch {

struct BParams {
    const int64_t* off;     // [nseg + 1] series offsets (global step indices), off[0] = 0, off[nseg] = N
    int nseg;
    const double* var;      // [nseg] sigma_b^2 (nullable: model's)
    const double* ell;      // [nseg] lengthscale (nullable: model's)
    const double* noise;    // [nseg] sigma_n,b^2 (nullable: model's)
    double sqrt2nu;         // sqrt(2 nu) of the model's Matern order
    double* nll_head;       // [chains] NLL of chain start .. first series end in the chain (or the whole
                            //          chain) when that series started in an earlier chain
    double* nll_tail;       // [chains] NLL of the last series start in the chain .. chain end when that
                            //          series continues past the chain
    double* nll_seg;        // [nseg] per-series NLL
};

struct Seg {
    int b;
    int64_t start, end;     // [start, end)
    double lam, s2, r, pscale;
};

template <int D>
__device__ __forceinline__ void seg_load(Seg& s, const KParams<D>& p, const BParams& q, int b) {
    // out-of-range series (invalid offsets, reported by k_batch_check_offsets) degrade to an
    // empty/unbounded segment so the step loops always terminate
    const bool over = b > q.nseg - 1, under = b < 0;
    b = max(0, min(b, q.nseg - 1));
    s.b = b;
    s.start = under ? INT64_MIN : __ldg(q.off + b);
    s.end = over ? INT64_MAX : __ldg(q.off + b + 1);
    s.s2 = q.var ? __ldg(q.var + b) : p.m.s2;
    s.lam = q.ell ? q.sqrt2nu / __ldg(q.ell + b) : p.m.lam;
    s.r = q.noise ? __ldg(q.noise + b) : p.m.r;
    s.pscale = s.s2 / p.m.s2;           // P_inf is proportional to sigma^2 in the lambda basis
}

// series containing global step k (largest b with off[b] <= k)
__device__ __forceinline__ int seg_find(const BParams& q, int64_t k) {
    int lo = 0, hi = q.nseg - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(q.off + mid) <= k) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

template <int D>
__device__ __forceinline__ void seg_first(const KParams<D>& p, const Seg& s, FJor<D>& F, double (&Q)[ns(D)]) {
    set_zero(F);
#pragma unroll
    for (int i = 0; i < ns(D); ++i) Q[i] = p.m.Pinf[i] * s.pscale;
}

// ------------------------------------------------------------------ K1b: fold
// Inputs staged like K1 (cp.async windows of t, y in a transposed [step][chain] layout,
// the window's mask bytes as one word); series starts are global-first-like elements.
template <int D>
__global__ void __launch_bounds__(kThreads, PSSGP_MINB) k_batch_filter_reduce(const KParams<D> p, const BParams q) {
    __shared__ AsyncStage st[kWarps];
    __shared__ FAgg<D> wagg[kWarps];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t c = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
    const int64_t nch = static_cast<int64_t>(p.nb) * kThreads;
    const int64_t wbase = (static_cast<int64_t>(blockIdx.x) * kThreads + wid * 32) * p.K;
    const int64_t kb = c * p.K;
    const int64_t ke = min(kb + p.K, p.n);
    if (blockIdx.x == 0 && threadIdx.x == 0) { p.flag[0] = 0ull; p.flag[1] = 0ull; }   // K3b's publication word, ticket
    FAgg<D> a;
    set_identity(a);
    ModelParams<D> mp = p.m;
    Seg s;
    if (kb < ke) seg_load(s, p, q, seg_find(q, kb));
    double tprev = (kb > 0 && kb < ke) ? __ldg(p.t + kb - 1) : 0.0;
    int ferr = -1;
    const int64_t nwin = (p.K + kWinA - 1) / kWinA;
    issue_window(st[wid], 0, p.t, p.y, wbase, p.K, p.n, 0, lane);
    unsigned long long mnext = mask_word(p.mask, kb, ke);
    for (int64_t w = 0; w < nwin; ++w) {
        const int64_t j0 = w * kWinA;
        const int buf = static_cast<int>(w & 1);
        if (w + 1 < nwin) issue_window(st[wid], buf ^ 1, p.t, p.y, wbase, p.K, p.n, j0 + kWinA, lane);
        else cp_async_commit();
        const unsigned long long mwin = mnext;
        mnext = mask_word(p.mask, kb + j0 + kWinA, ke);
        cp_async_wait<1>();
        __syncwarp();
        const int jend = static_cast<int>(min(static_cast<int64_t>(kWinA), ke - (kb + j0)));
#pragma unroll 1
        for (int jj = 0; jj < jend; ++jj) {
            const int64_t k = kb + j0 + jj;
            while (k >= s.end) seg_load(s, p, q, s.b + 1);
            const double tk = st[wid].t[buf][jj][lane];
            const bool obs = ((mwin >> (8 * jj)) & 0xffull) != 0;
            const double yk = obs ? st[wid].y[buf][jj][lane] : 0.0;
            FJor<D> F;
            double Q[ns(D)];
            const bool start = (k == s.start);
            if (start) seg_first(p, s, F, Q);
            else matern_closed<D>(s.lam, s.s2, tk - tprev, F, Q);
            const bool bad = (!start && !(tk - tprev >= 0.0)) || !isfinite(tk) || (obs && !isfinite(yk));
            ferr = (bad && ferr < 0) ? static_cast<int>(k - kb) : ferr;
            mp.r = s.r;
            fold_step<D, true>(a, F, Q, mp, obs, yk);
            tprev = tk;
        }
        __syncwarp();
    }
    if (ferr >= 0) raise_error(p.err, kb + ferr, kErrInput);
    store_soa(a, p.chain_f, nch, c);
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        FAgg<D> o;
        shfl_down_all(o, a, off);
        if ((lane & (2 * off - 1)) == 0) {
            FAgg<D> r;
            if (!combine(a, o, r)) raise_error(p.err, kb, kErrNumeric);
            a = r;
        }
    }
    if (lane == 0) wagg[wid] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        FAgg<D> acc = wagg[0];
        bool ok = true;
        for (int w = 1; w < kWarps; ++w) {
            FAgg<D> r;
            ok = combine(acc, wagg[w], r) && ok;
            acc = r;
        }
        if (!ok) raise_error(p.err, kb, kErrNumeric);
        store_aos(acc, p.block_f + static_cast<int64_t>(blockIdx.x) * FN(D));
    }
}

// ------------------------------------------------------------------ K3b: Kalman rescan
// Staged inputs as in K3.  NLL per (chain, series) piece: a series inside the chain is written to
// nll_seg directly, the pieces of series crossing the chain's ends go to nll_head / nll_tail and
// are summed per series by k_batch_nll (as k_batch_grad_combine composes the gradient pieces).
template <int D>
__global__ void __launch_bounds__(kThreads, PSSGP_MINB) k_batch_filter_apply(const KParams<D> p, const BParams q) {
    __shared__ AsyncStage st[kWarps];
    __shared__ FAgg<D> tot[kWarps];
    __shared__ Gauss<D> wcar[kWarps];
    __shared__ SAgg<D> stot[kWarps];
    __shared__ int s_bid;
    const int bid = k3_ticket(p.flag, &s_bid);               // logical CTA index (arrival order)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t c = static_cast<int64_t>(bid) * kThreads + threadIdx.x;
    const int64_t nch = static_cast<int64_t>(p.nb) * kThreads;
    const int64_t wg = static_cast<int64_t>(bid) * kWarps + wid;
    const int64_t wbase = wg * 32 * p.K;
    const int64_t kb = c * p.K;
    const int64_t ke = min(kb + p.K, p.n);
    const Gauss<D> cur = filter_chain_carry<D>(p, tot, wcar, c, nch, lane, wid, bid);
    double x[D], P[ns(D)], x0[D], P0[ns(D)], Sg[D * D];
#pragma unroll
    for (int i = 0; i < D; ++i) x[i] = cur.x[i];
#pragma unroll
    for (int i = 0; i < ns(D); ++i) P[i] = cur.P[i];
    ModelParams<D> mp = p.m;
    Seg s;
    if (kb < ke) seg_load(s, p, q, seg_find(q, kb));
    double tprev = (kb > 0 && kb < ke) ? __ldg(p.t + kb - 1) : 0.0;
    bool sag_done = false, head_done = false;
    int ferr = -1;
    double quad = 0.0, prodm = 1.0;
    long long prode = 0;
    int nobs = 0;
    const int64_t nwin = (p.K + kWinA - 1) / kWinA;
    issue_window(st[wid], 0, p.t, p.y, wbase, p.K, p.n, 0, lane);
    unsigned long long mnext = mask_word(p.mask, kb, ke);
    for (int64_t w = 0; w < nwin; ++w) {
        const int64_t j0 = w * kWinA;
        const int buf = static_cast<int>(w & 1);
        if (w + 1 < nwin) issue_window(st[wid], buf ^ 1, p.t, p.y, wbase, p.K, p.n, j0 + kWinA, lane);
        else cp_async_commit();
        const unsigned long long mwin = mnext;
        mnext = mask_word(p.mask, kb + j0 + kWinA, ke);
        cp_async_wait<1>();
        __syncwarp();
        const int jend = static_cast<int>(min(static_cast<int64_t>(kWinA), ke - (kb + j0)));
#pragma unroll 1
        for (int jj = 0; jj < jend; ++jj) {
            const int64_t k = kb + j0 + jj;
            while (k >= s.end) seg_load(s, p, q, s.b + 1);
            const double tk = st[wid].t[buf][jj][lane];
            const bool obs = ((mwin >> (8 * jj)) & 0xffull) != 0;
            const double yk = obs ? st[wid].y[buf][jj][lane] : 0.0;
            const bool first = (k == kb);
            FJor<D> F;
            double Q[ns(D)], xm[D], Pm[ns(D)];
            if (k == s.start) seg_first(p, s, F, Q);
            else matern_closed<D>(s.lam, s.s2, tk - tprev, F, Q);
            kf_predict_pm<D>(x, P, F, Q, xm, Pm);
            tprev = tk;
            mp.r = s.r;
            double HP[D], S, hx;
            obs_terms<D>(mp, xm, Pm, HP, S, hx, true);
            const bool bad = obs && !(S > 0.0 && S < INFINITY);
            ferr = (bad && ferr < 0) ? static_cast<int>(k - kb) : ferr;
            const double iS = obs ? rcp(S) : 0.0;
            const double v = obs ? (yk - hx) : 0.0;
            const double vs = v * iS;
#pragma unroll
            for (int i = 0; i < D; ++i) x[i] = fma(HP[i], vs, xm[i]);
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = i; j < D; ++j) P[si(D, i, j)] = fma(-HP[i] * iS, HP[j], Pm[si(D, i, j)]);
            if (first) {
#pragma unroll
                for (int i = 0; i < D; ++i) x0[i] = x[i];
#pragma unroll
                for (int i = 0; i < ns(D); ++i) P0[i] = P[i];
#pragma unroll
                for (int i = 0; i < D; ++i)
#pragma unroll
                    for (int j = 0; j < D; ++j) Sg[i * D + j] = P[si(D, i, j)];
            } else {
                double Sm[D * D], SH[D];
                mul_bt<D>(Sg, F, Sm);
#pragma unroll
                for (int i = 0; i < D; ++i) SH[i] = Sm[i * D];          // H = e_0 (Jordan basis)
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    const double si_ = SH[i] * iS;
#pragma unroll
                    for (int j = 0; j < D; ++j) Sg[i * D + j] = fma(-si_, HP[j], Sm[i * D + j]);
                    x0[i] = fma(SH[i], vs, x0[i]);
#pragma unroll
                    for (int j = i; j < D; ++j) P0[si(D, i, j)] = fma(-si_, SH[j], P0[si(D, i, j)]);
                }
            }
            // NLL of the (chain, series) piece: running v^2/S sum and S product (one log per piece)
            nll_accumulate(obs, v, vs, S, quad, prodm, prode, nobs);
            if (k == s.end - 1) {
                const double term = nobs > 0 ? 0.5 * (quad + log(prodm) + static_cast<double>(prode) * 0.6931471805599453 +
                                                      nobs * 1.8378770664093453) : 0.0;
                if (s.start >= kb) q.nll_seg[s.b] = term;           // the whole series is in this chain
                else if (!head_done) { q.nll_head[c] = term; head_done = true; }
                quad = 0.0; prodm = 1.0; prode = 0; nobs = 0;
            }
            if (k == s.end - 1 && !sag_done) {
                // first series end in this chain: the chain's smoother aggregate is the collapsed
                // (0, m^s_k0, P^s_k0) of that series (terminal element), stored at
                // once (not held in registers across the loop)
                SAgg<D> sag;
#pragma unroll
                for (int i = 0; i < D * D; ++i) sag.E[i] = 0.0;
#pragma unroll
                for (int i = 0; i < D; ++i) sag.g[i] = x0[i];
#pragma unroll
                for (int i = 0; i < ns(D); ++i) sag.L[i] = P0[i];
                store_soa(sag, p.chain_s, nch, c);
                sag_done = true;
            }
            double* o = p.xp + ((wg * p.K + (k - kb)) * CN(D)) * 32 + lane;
            st_xP<D>(o, lane, x, P);
        }
        __syncwarp();
    }
    if (ferr >= 0) raise_error(p.err, kb + ferr, kErrNumeric);
    if (ke > kb && s.end > ke) {                  // a series continues past the chain end
        const double term = nobs > 0 ? 0.5 * (quad + log(prodm) + static_cast<double>(prode) * 0.6931471805599453 +
                                              nobs * 1.8378770664093453) : 0.0;
        if (s.start >= kb) q.nll_tail[c] = term;  // it started in this chain
        else q.nll_head[c] = term;                // it runs through the whole chain
    }
    SAgg<D> sag;
    if (sag_done) {
        load_soa(sag, p.chain_s, nch, c);
    } else {
        set_identity(sag);
        if (ke > kb) {
            // the next step exists and belongs to the same series (a series end would have set sag)
            const double tn = __ldg(p.t + ke);
            FJor<D> F;
            double Q[ns(D)], xm[D], Pm[ns(D)], Sm[D * D];
            matern_closed<D>(s.lam, s.s2, tn - tprev, F, Q);
            kf_predict_pm<D>(x, P, F, Q, xm, Pm);
            mul_bt<D>(Sg, F, Sm);
            if (!chain_smoother_agg<D>(x0, P0, Sm, xm, Pm, sag)) raise_error(p.err, ke, kErrNumeric);
        }
        store_soa(sag, p.chain_s, nch, c);
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        SAgg<D> o;
        shfl_down_all(o, sag, off);
        if ((lane & (2 * off - 1)) == 0) {
            SAgg<D> r;
            combine(sag, o, r);
            sag = r;
        }
    }
    if (lane == 0) stot[wid] = sag;
    __syncthreads();
    if (threadIdx.x == 0) {
        SAgg<D> acc = stot[0];
        for (int w = 1; w < kWarps; ++w) {
            SAgg<D> r;
            combine(acc, stot[w], r);
            acc = r;
        }
        store_aos(acc, p.block_s + static_cast<int64_t>(bid) * SN(D));
    }
}

// ------------------------------------------------------------------ K5b: RTS rescan
// t staged in windows and mean/var leaving through a transposed tile (coalesced), the
// filtered record of the next step down prefetched one step ahead, as in K5.
template <int D>
__global__ void __launch_bounds__(kThreads, PSSGP_MINB) k_batch_smoother_apply(const KParams<D> p, const BParams q) {
    __shared__ StageOut so[kWarps];
    __shared__ SAgg<D> tot[kWarps];
    __shared__ Gauss<D> wcar[kWarps + 1];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t c = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
    const int64_t nch = static_cast<int64_t>(p.nb) * kThreads;
    const int64_t wg = static_cast<int64_t>(blockIdx.x) * kWarps + wid;
    const int64_t wbase = wg * 32 * p.K;
    const int64_t kb = c * p.K;
    const int64_t ke = min(kb + p.K, p.n);
    const Gauss<D> cur = smoother_chain_carry<D>(p, tot, wcar, c, nch, lane, wid);
    double ms[D], Ps[ns(D)];
#pragma unroll
    for (int i = 0; i < D; ++i) ms[i] = cur.x[i];
#pragma unroll
    for (int i = 0; i < ns(D); ++i) Ps[i] = cur.P[i];
    Seg s;
    if (kb < ke) seg_load(s, p, q, seg_find(q, ke - 1));
    double tnext = (kb < ke && ke < p.n) ? __ldg(p.t + ke) : 0.0;
    const double* xpw = p.xp + (wg * p.K * CN(D)) * 32 + lane;
    double nx[CN(D)];
    if (kb < ke) {
        const double* s1 = xpw + ((ke - 1 - kb) * CN(D)) * 32;
        ld_state<D>(s1, lane, nx);
    }
    int ferr = -1;
    const int64_t nwin = (p.K + kWinA - 1) / kWinA;
    issue_copies<false>(so[wid].t[(nwin - 1) & 1], nullptr, p.t, nullptr, wbase, p.K, p.n, (nwin - 1) * kWinA, lane);
    for (int64_t w = nwin - 1; w >= 0; --w) {
        const int64_t j0 = w * kWinA;
        const int buf = static_cast<int>(w & 1);
        if (w > 0) issue_copies<false>(so[wid].t[buf ^ 1], nullptr, p.t, nullptr, wbase, p.K, p.n, j0 - kWinA, lane);
        else cp_async_commit();
        if (PSSGP_TY_PF > 0 && j0 - (1 + PSSGP_TY_PF) * kWinA >= 0)
            prefetch_ty_l2<false>(p.t, nullptr, kb, j0 - (1 + PSSGP_TY_PF) * kWinA, ke);
        cp_async_wait<1>();
        __syncwarp();
        const int jstart = static_cast<int>(min(static_cast<int64_t>(kWinA - 1), ke - 1 - (kb + j0)));
#pragma unroll 1
        for (int jj = jstart; jj >= 0; --jj) {
            const int64_t k = kb + j0 + jj;
            while (k < s.start) seg_load(s, p, q, s.b - 1);
            const double tk = so[wid].t[buf][jj][lane];
            double x[D], P[ns(D)];
#pragma unroll
            for (int i = 0; i < D; ++i) x[i] = nx[i];
#pragma unroll
            for (int i = 0; i < ns(D); ++i) P[i] = nx[D + i];
            if (k > kb) {
                const double* src = xpw + ((k - 1 - kb) * CN(D)) * 32;
                ld_state<D>(src, lane, nx);
            }
            if (PSSGP_K5_PF > 0 && k - PSSGP_K5_PF >= kb) prefetch_state_l2<D>(xpw, lane, k - PSSGP_K5_PF - kb);
            if (k == s.end - 1) {   // series end: terminal element
#pragma unroll
                for (int i = 0; i < D; ++i) ms[i] = x[i];
#pragma unroll
                for (int i = 0; i < ns(D); ++i) Ps[i] = P[i];
            } else {
                FJor<D> F;
                double Q[ns(D)], xm[D], Pm[ns(D)], FP[D * D];
                matern_closed<D>(s.lam, s.s2, tnext - tk, F, Q);
                kf_predict<D>(x, P, F, Q, xm, FP, Pm);
                const bool bad = !rts_step<D>(x, P, xm, Pm, FP, ms, Ps);
                ferr = bad ? static_cast<int>(k - kb) : ferr;   // backward: last hit = first index
            }
            tnext = tk;
            so[wid].m[jj][lane] = ms[0];
            so[wid].v[jj][lane] = Ps[0];
        }
        __syncwarp();
        {
            const int col = lane & (kWinA - 1), rb = lane / kWinA;
            const int64_t j = j0 + col;
#pragma unroll
            for (int i = 0; i < 32 / (32 / kWinA); ++i) {
                const int r = rb + (32 / kWinA) * i;
                const int64_t idx = wbase + r * p.K + j;
                const int64_t rend = min(wbase + (r + 1) * p.K, p.n);
                if (j < p.K && idx < rend) {
                    if (PSSGP_CS_HINTS & 4) {   // streaming stores of the outputs
                        if (p.mean) __stcs(p.mean + idx, so[wid].m[col][r]);
                        if (p.var) __stcs(p.var + idx, so[wid].v[col][r]);
                    } else {
                        if (p.mean) p.mean[idx] = so[wid].m[col][r];
                        if (p.var) p.var[idx] = so[wid].v[col][r];
                    }
                }
            }
        }
        __syncwarp();
    }
    if (ferr >= 0) raise_error(p.err, kb + ferr, kErrNumeric);
}

// ------------------------------------------------------------------ offsets validation
// off[0] = 0, off[nseg] = N, non-decreasing; the first violation is reported as an input
// error at the offending series index.
__global__ void __launch_bounds__(256) k_batch_check_offsets(const int64_t* __restrict__ off, int nseg, int64_t N,
                                                             unsigned long long* err) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b > nseg) return;
    const int64_t o = __ldg(off + b);
    bool bad = (b == 0 && o != 0) || (b == nseg && o != N) || o < 0 || o > N;
    if (b > 0) bad = bad || (__ldg(off + b - 1) > o);
    if (bad) raise_error(err, b, kErrInput);
}

// ------------------------------------------------------------------ per-series NLL (1 warp per series)
// Per-series NLL of series that cross chain boundaries: tail(c1) + head(c1+1) + ... + head(c2)
// (fixed order, one warp per series); series inside one chain were written by K3b, empty ones get 0.
__global__ void __launch_bounds__(128) k_batch_nll(const BParams q, int64_t K) {
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.x * 4 + (threadIdx.x >> 5);
    if (b >= q.nseg) return;
    const int64_t a0 = __ldg(q.off + b), a1 = __ldg(q.off + b + 1);
    if (a1 <= a0) {
        if (lane == 0) q.nll_seg[b] = 0.0;
        return;
    }
    const int64_t c1 = a0 / K, c2 = (a1 - 1) / K;
    if (c1 == c2) return;
    double s = lane == 0 ? q.nll_tail[c1] : 0.0;
    for (int64_t c = c1 + 1 + lane; c <= c2; c += 32) s += q.nll_head[c];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
    if (lane == 0) q.nll_seg[b] = s;
}

}  // namespace batch
}  // namespace pssgp
