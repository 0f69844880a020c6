// pssgp_wide_host.cuh — host side of the warp-per-chain path (d >= 4): launch plan, workspace,
// and the kernel sequences of pssgp_posterior / the sharded phases for one state dimension D.
// Included only by pssgp_wide_inst.cu (one object per D in pssgp_dims.h).
#pragma once
#include <algorithm>
#include <atomic>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "pssgp_internal.hpp"
#include "pssgp_wide.cuh"
#include "pssgp_batch_theta.cuh"

namespace pssgp_internal {
namespace widehost {
using namespace pssgp;
// 9 <= D <= 16: lane-per-row kernels in 16-lane groups, two half chains per warp, 2 warps per CTA
constexpr int kHalfG = 16, kHalfWPC = 2;
template <int D>
constexpr bool wide_halves() { return D > pssgp::wide::kGL && D <= kHalfG; }
// the F block size of the half-chain kernels (pssgp_model::fblock: 2, 4, or dense), compile time
template <int D, typename Fn>
void with_fblock(const pssgp_model* m, Fn&& fn) {
    if constexpr (D > 4) {
        if (m->fblock == 2) { fn(std::integral_constant<int, 2>{}); return; }
        if (m->fblock == 4) { fn(std::integral_constant<int, 4>{}); return; }
    }
    fn(std::integral_constant<int, D>{});
}
// ========================================================================== wide path (d >= 4)
constexpr int kMbfWPC = 2;   // d > 16: warps (chains) per CTA of the adjoint-form RTS rescan

// The >48 KB dynamic shared-memory opt-in is a per-device function attribute: set it once per
// device (bit `device` of a process-wide mask; setting it twice is harmless, so a race only repeats
// the calls).
template <int D>
void wide_set_smem_attrs(int device) {
    using namespace pssgp::wide;
    static std::atomic<unsigned long long> done{0ull};
    const unsigned long long bit = 1ull << (device & 63);
    if (done.load() & bit) return;
    cudaFuncSetAttribute(kw_filter_fold<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K1Smem<D>));
    if constexpr (D <= kGL) {
        cudaFuncSetAttribute(kw_filter_fold_lpr<D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K1LSmem<D, false>));
        cudaFuncSetAttribute(kw_filter_fold_lpr<D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K1LSmem<D, true>));
        cudaFuncSetAttribute(kw_filter_apply_lpr<D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K3LSmem<D, false>));
        cudaFuncSetAttribute(kw_filter_apply_lpr<D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K3LSmem<D, true>));
        cudaFuncSetAttribute(kw_smoother_apply_lpr<D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K5LSmem<D, false>));
        cudaFuncSetAttribute(kw_smoother_apply_lpr<D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K5LSmem<D, true>));
        cudaFuncSetAttribute(kw_filter_apply_q<D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K3QSmem<D, false>));
        cudaFuncSetAttribute(kw_filter_apply_q<D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K3QSmem<D, true>));
        cudaFuncSetAttribute(kw_smoother_apply_q<D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K5QSmem<D, false>));
        cudaFuncSetAttribute(kw_smoother_apply_q<D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K5QSmem<D, true>));
        cudaFuncSetAttribute(kw_smoother_mbf_q<D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K5MSmem<D, false>));
        cudaFuncSetAttribute(kw_smoother_mbf_q<D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K5MSmem<D, true>));
    } else if constexpr (wide_halves<D>()) {
        auto set = [](auto fbc) {
            constexpr int G = kHalfG, W = kHalfWPC, FB = decltype(fbc)::value;
            cudaFuncSetAttribute(kw_filter_fold_lpr<D, false, G, W, FB>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K1LSmem<D, false, G, W>));
            cudaFuncSetAttribute(kw_filter_fold_lpr<D, true, G, W, FB>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K1LSmem<D, true, G, W>));
            cudaFuncSetAttribute(kw_filter_apply_q<D, false, G, W, FB>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K3QSmem<D, false, G, W>));
            cudaFuncSetAttribute(kw_filter_apply_q<D, true, G, W, FB>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K3QSmem<D, true, G, W>));
            cudaFuncSetAttribute(kw_smoother_apply_q<D, false, G, W, FB>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K5QSmem<D, false, G, W>));
            cudaFuncSetAttribute(kw_smoother_apply_q<D, true, G, W, FB>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K5QSmem<D, true, G, W>));
            cudaFuncSetAttribute(kw_smoother_mbf_q<D, false, G, W, FB>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K5MSmem<D, false, G, W>));
            cudaFuncSetAttribute(kw_smoother_mbf_q<D, true, G, W, FB>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K5MSmem<D, true, G, W>));
        };
        set(std::integral_constant<int, D>{});
        cudaFuncSetAttribute(kw_combine_halves<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(ScanSmemF<D>));
        cudaFuncSetAttribute(kw_part_sagg<D, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(QAgPhase<D>));
        if constexpr (D > 4) {
            set(std::integral_constant<int, 2>{});
            set(std::integral_constant<int, 4>{});
        }
    }
    cudaFuncSetAttribute(kw_filter_apply<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K3Smem<D>));
    cudaFuncSetAttribute(kw_smoother_apply<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K5Smem<D>));
    if constexpr (D > 16) {   // adjoint-form RTS rescan, one 32-lane group (row per lane) per chain
        auto setm = [](auto fbc) {
            constexpr int FB = decltype(fbc)::value;
            cudaFuncSetAttribute(kw_smoother_mbf_q<D, false, 32, kMbfWPC, FB>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K5MSmem<D, false, 32, kMbfWPC>));
            cudaFuncSetAttribute(kw_smoother_mbf_q<D, true, 32, kMbfWPC, FB>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(K5MSmem<D, true, 32, kMbfWPC>));
        };
        setm(std::integral_constant<int, D>{});
        setm(std::integral_constant<int, 2>{});
        setm(std::integral_constant<int, 4>{});
    }
    cudaFuncSetAttribute(kw_scan_filter<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(ScanSmemF<D>));
    cudaFuncSetAttribute(kw_scan_smoother<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(ScanSmemS<D>));
    cudaFuncSetAttribute(kw_discretize<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(KDSmem<D>));
    cudaFuncSetAttribute(kw_grad_forward<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(GFwdSmem<D>));
    cudaFuncSetAttribute(kw_grad_backward<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(GBwdSmem<D>));
    cudaFuncSetAttribute(kw_scan_adjoint<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(ScanSmemA<D>));
    done.fetch_or(bit);
}

// lane-per-row kernels of the wide path for D <= 8 (bit 0: fold, bit 1: RTS rescan, bit 2: both
// rescans also with per-step (F, Q) staged in shared memory, bit 3: one-wave plan for them on the
// table path, bit 4: Kalman rescan, bit 5: the one-wave plan also on the per-step (F, Q) path, bit 6:
// lane-per-row discretisation, bit 7: quarter-parallel rescans (all four 8-lane groups of a warp
// busy; needs bit 0, whose fold stores the quarter prefix aggregates), bit 8: see below, bit 9:
// per-block discretisation of block-diagonal models (kw_discretize_blk) where the lane-per-row one
// does not run), bits 10, 11: see below); env PSSGP_WIDE_LPR overrides the default 2047 for A/B runs
// (0 = the shared-memory kernels)
inline int wide_lpr_mask() {
    static const int v = [] { const char* e = getenv("PSSGP_WIDE_LPR"); return e && *e ? atoi(e) : 2047; }();
    return v;
}
inline bool wide_quarter_rescans() { return (wide_lpr_mask() & 129) == 129; }
// bit 8: 9 <= D <= 16 on the lane-per-row fold and half-chain rescans (16-lane groups, two half
// chains per warp, 2 warps per CTA: kHalfG / kHalfWPC)
inline bool wide_half_rescans() { return (wide_lpr_mask() & 256) != 0; }
// bit 10: the half-chain RTS rescan (9 <= D <= 16) in adjoint (modified Bryson-Frazier) form,
// kw_smoother_mbf_q: O(d^2 FB) per step instead of a Cholesky solve per step (C4 K5w 75.3 -> 17.7
// ms); bit 11: the same for the quarter rescans of D <= 8 (dense F there: F^T Lt F costs 2 d^3,
// measured 1.42 -> 1.57 ms at C3, so off by default)
inline bool wide_mbf() { return (wide_lpr_mask() & 1024) != 0; }
inline bool wide_mbf_quarters() { return (wide_lpr_mask() & 3072) == 3072; }

struct WPlan {
    int64_t K = 0;
    int nch = 0, nb = 0;
};

template <int D>
WPlan make_wplan(pssgp_model* m, int64_t n, bool grad = false) {
    using namespace pssgp::wide;
    wide_set_smem_attrs<D>(m->device);
    if constexpr (D > 16) {
        // the gradient runs the fold and the two gradient rescans only: its own occupancy (the
        // posterior's RTS kernel holds fewer CTAs per SM)
        if (grad && m->wocc_grad == 0) {
            int a = 0, b = 0, c = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, kw_filter_fold<D>, 32 * kWWarps, sizeof(K1Smem<D>));
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kw_grad_forward<D>, 32 * kWWarps, sizeof(GFwdSmem<D>));
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, kw_grad_backward<D>, 32 * kWWarps, sizeof(GBwdSmem<D>));
            m->wocc_grad = std::max(1, std::min(a, std::min(b, c)));
            if (getenv("PSSGP_WIDE_DEBUG"))
                fprintf(stderr, "wide gradient plan D=%d occupancy: fold %d, forward %d, backward %d (smem %zu / %zu / %zu)\n",
                        D, a, b, c, sizeof(K1Smem<D>), sizeof(GFwdSmem<D>), sizeof(GBwdSmem<D>));
        }
    }
    if (m->wocc == 0) {
        int a = 0, b = 0, c = 0;
        // (the lane-per-row fold of D <= 8 is not part of the plan's occupancy: it is register-
        // capped at PSSGP_WLPR_MINB CTAs/SM and simply runs the same grid)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, kw_filter_fold<D>, 32 * kWWarps, sizeof(K1Smem<D>));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kw_filter_apply<D>, 32 * kWWarps, sizeof(K3Smem<D>));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, kw_smoother_apply<D>, 32 * kWWarps, sizeof(K5Smem<D>));
        m->wocc = std::max(1, std::min(a, std::min(b, c)));
        if constexpr (D > 16) {
            if (wide_mbf()) {   // the RTS rescan in adjoint form replaces kw_smoother_apply in the plan
                int l5 = 0;
                with_fblock<D>(m, [&](auto fbc) {
                    constexpr int FB = decltype(fbc)::value;
                    if (m->mode == kPade)
                        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l5, kw_smoother_mbf_q<D, true, 32, kMbfWPC, FB>, 32 * kMbfWPC, sizeof(K5MSmem<D, true, 32, kMbfWPC>));
                    else
                        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l5, kw_smoother_mbf_q<D, false, 32, kMbfWPC, FB>, 32 * kMbfWPC, sizeof(K5MSmem<D, false, 32, kMbfWPC>));
                });
                m->wchains = std::max(1, std::min(std::min(a, b) * kWWarps, l5 * kMbfWPC));
                if (getenv("PSSGP_WIDE_DEBUG"))
                    fprintf(stderr, "wide plan D=%d: fold %d, apply %d CTAs/SM of %d warps, adjoint RTS %d of %d -> %d chains/SM\n",
                            D, a, b, kWWarps, l5, kMbfWPC, m->wchains);
            }
        }
        if constexpr (D <= kGL) {
            int l1 = 0, l5 = 0, l3 = 0;
            if (wide_quarter_rescans()) {
                if (m->mode == kPade) {
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l1, kw_filter_fold_lpr<D, true>, 32 * kWWarps, sizeof(K1LSmem<D, true>));
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l3, kw_filter_apply_q<D, true>, 32 * kWWarps, sizeof(K3QSmem<D, true>));
                    if (wide_mbf_quarters()) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l5, kw_smoother_mbf_q<D, true>, 32 * kWWarps, sizeof(K5MSmem<D, true>));
                    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l5, kw_smoother_apply_q<D, true>, 32 * kWWarps, sizeof(K5QSmem<D, true>));
                } else {
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l1, kw_filter_fold_lpr<D, false>, 32 * kWWarps, sizeof(K1LSmem<D, false>));
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l3, kw_filter_apply_q<D, false>, 32 * kWWarps, sizeof(K3QSmem<D, false>));
                    if (wide_mbf_quarters()) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l5, kw_smoother_mbf_q<D, false>, 32 * kWWarps, sizeof(K5MSmem<D, false>));
                    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l5, kw_smoother_apply_q<D, false>, 32 * kWWarps, sizeof(K5QSmem<D, false>));
                }
            } else if (m->mode == kPade) {   // per-step (F, Q) variants (their staging buffers cost shared memory)
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l1, kw_filter_fold_lpr<D, true>, 32 * kWWarps, sizeof(K1LSmem<D, true>));
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l3, kw_filter_apply_lpr<D, true>, 32 * kWWarps, sizeof(K3LSmem<D, true>));
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l5, kw_smoother_apply_lpr<D, true>, 32 * kWWarps, sizeof(K5LSmem<D, true>));
            } else {
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l1, kw_filter_fold_lpr<D, false>, 32 * kWWarps, sizeof(K1LSmem<D, false>));
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l3, kw_filter_apply_lpr<D, false>, 32 * kWWarps, sizeof(K3LSmem<D, false>));
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l5, kw_smoother_apply_lpr<D, false>, 32 * kWWarps, sizeof(K5LSmem<D, false>));
            }
            if (wide_lpr_mask() & 16) l5 = std::min(l5, l3);
            if (getenv("PSSGP_WIDE_DEBUG"))
                fprintf(stderr, "wide plan D=%d occupancy: fold %d, apply %d, smoother %d, lpr fold %d, lpr/q apply %d, "
                        "lpr/q smoother %d\n", D, a, b, c, l1, l3, l5);
            // bit 3: on the table (uniform-dt) path, where both lane-per-row kernels run, size the
            // plan so they run in one wave (C3: 13.8 -> 11.7 ms; on the per-step (F, Q) path the
            // fewer, longer chains slow the shared-memory rescans: 26.2 -> 28.3 ms, so not there)
            if ((wide_lpr_mask() & 8) && (m->mode != kPade || (wide_lpr_mask() & 32))) m->wocc = std::max(1, std::min(m->wocc, std::min(l1, l5)));
            if (wide_quarter_rescans()) m->wocc = std::max(1, std::min(l1, std::min(l3, l5)));
        } else if constexpr (wide_halves<D>()) {
            if (wide_half_rescans()) {   // one wave of the half-chain kernels (2-warp CTAs)
                constexpr int G = kHalfG, W = kHalfWPC;
                int l1 = 0, l3 = 0, l5 = 0;
                with_fblock<D>(m, [&](auto fbc) {
                    constexpr int FB = decltype(fbc)::value;
                    if (m->mode == kPade) {
                        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l1, kw_filter_fold_lpr<D, true, G, W, FB>, 32 * W, sizeof(K1LSmem<D, true, G, W>));
                        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l3, kw_filter_apply_q<D, true, G, W, FB>, 32 * W, sizeof(K3QSmem<D, true, G, W>));
                        if (wide_mbf()) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l5, kw_smoother_mbf_q<D, true, G, W, FB>, 32 * W, sizeof(K5MSmem<D, true, G, W>));
                        else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l5, kw_smoother_apply_q<D, true, G, W, FB>, 32 * W, sizeof(K5QSmem<D, true, G, W>));
                    } else {
                        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l1, kw_filter_fold_lpr<D, false, G, W, FB>, 32 * W, sizeof(K1LSmem<D, false, G, W>));
                        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l3, kw_filter_apply_q<D, false, G, W, FB>, 32 * W, sizeof(K3QSmem<D, false, G, W>));
                        if (wide_mbf()) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l5, kw_smoother_mbf_q<D, false, G, W, FB>, 32 * W, sizeof(K5MSmem<D, false, G, W>));
                        else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l5, kw_smoother_apply_q<D, false, G, W, FB>, 32 * W, sizeof(K5QSmem<D, false, G, W>));
                    }
                });
                m->wchains = std::max(1, std::min(l1, std::min(l3, l5))) * W;
                if (getenv("PSSGP_WIDE_DEBUG"))
                    fprintf(stderr, "wide plan D=%d half-chain kernels: fold %d, apply %d, smoother %d CTAs/SM of %d warps\n",
                            D, l1, l3, l5, W);
            }
        }
    }
    int64_t per_sm = m->wchains > 0 ? m->wchains : static_cast<int64_t>(m->wocc) * kWWarps;   // chains per SM
    if (D > 16 && grad && m->wocc_grad > 0) per_sm = static_cast<int64_t>(m->wocc_grad) * kWWarps;
    const int64_t target = static_cast<int64_t>(m->sm_count) * per_sm;
    WPlan pl;
    // small N: chains of at least 16 steps (8 for the warp-cooperative kernels of d > 16, whose chain
    // steps cost more than an extra scan level: CO2 J = 3 gradient at N = 3,200: 0.74 -> 0.67 ms)
    const int64_t kmin = D > 16 ? 8 : 16;
    pl.K = m->forced_K > 0 ? m->forced_K : std::max<int64_t>(kmin, (n + target - 1) / target);
    pl.nch = static_cast<int>(std::max<int64_t>(1, (n + pl.K - 1) / pl.K));
    pl.nb = (pl.nch + kWWarps - 1) / kWWarps;
    return pl;
}

template <int D>
pssgp_status wide_setup(pssgp_model* m, const WPlan& pl, pssgp::wide::WParams& p) {
    using namespace pssgp::wide;
    const size_t nch = static_cast<size_t>(pl.nch);
    const bool quarters = (D <= kGL && wide_quarter_rescans()) || (wide_halves<D>() && wide_half_rescans());
    const bool halves = wide_halves<D>() && wide_half_rescans();
    // quarter prefix / smoother aggregates (+ the halves' end moments for kw_part_sagg)
    const size_t nq = quarters ? nch * (kQ - 1) * (FNW(D) + SNW(D)) + (halves ? nch * 2 * QMW(D) : 0) : 0;
    const size_t need = (2 * nch * FNW(D) + nch * pl.K * CNW(D) + 2 * nch * SNW(D) + nch + nq + 64) * sizeof(double);
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
    if (!m->d_model) {
        std::vector<double> h(MODW(D) + MODP(D), 0.0);
        for (int i = 0; i < D * D; ++i) {
            h[i] = m->udt > 0.0 ? m->Fu[i] : 0.0;
            h[D * D + i] = m->udt > 0.0 ? m->Qu[i] : 0.0;
            h[2 * D * D + i] = static_cast<double>(m->ssm.Pinf[i]);
        }
        for (int i = 0; i < D; ++i) h[3 * D * D + i] = static_cast<double>(m->ssm.H[i]);
        h[3 * D * D + D] = m->r;
        h[3 * D * D + D + 1] = m->udt > 0.0 ? m->udt : -1.0;
        for (int i = 0; i < D * D; ++i) h[3 * D * D + D + 2 + i] = static_cast<double>(m->ssm.G[i]);
        for (int i = 0; i < D * D; ++i) h[4 * D * D + D + 2 + i] = static_cast<double>(m->ssm.W[i]);
        {   // Taylor coefficients of F(dt), Q(dt) (kw_discretize_lpr's polynomial path), long double
            using pssgp_host::Mat;
            const Mat& G = m->ssm.G;
            Mat Fk = pssgp_host::eye(D), Mk = m->ssm.W;
            for (int k = 0; k <= kPolyM; ++k) {
                for (int i = 0; i < D * D; ++i) {
                    h[MODW(D) + k * D * D + i] = static_cast<double>(Fk[i]);
                    h[MODW(D) + (kPolyM + 1 + k) * D * D + i] = static_cast<double>(Mk[i]);   // M_{k+1}
                }
                Fk = pssgp_host::matmul(Fk, G, D);
                for (auto& v : Fk) v /= static_cast<pssgp_host::ld>(k + 1);
                const Mat GM = pssgp_host::matmul(G, Mk, D);
                Mat Mn = pssgp_host::zeros(D);
                for (int i = 0; i < D; ++i)
                    for (int j = 0; j < D; ++j)
                        Mn[i * D + j] = (GM[i * D + j] + GM[j * D + i]) / static_cast<pssgp_host::ld>(k + 2);
                Mk = Mn;
            }
        }
        if (cudaMalloc(&m->d_model, h.size() * sizeof(double)) != cudaSuccess) {
            cudaGetLastError();
            return fail(m, PSSGP_E_NOMEM, "cudaMalloc(model)");
        }
        cudaMemcpy(m->d_model, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice);
    }
    std::memset(&p, 0, sizeof(p));
    double* w = reinterpret_cast<double*>(m->ws);
    p.fagg = w; w += nch * FNW(D);
    p.fbuf = w; w += nch * FNW(D);
    p.xp = w; w += nch * pl.K * CNW(D);
    p.sagg = w; w += nch * SNW(D);
    p.sbuf = w; w += nch * SNW(D);
    p.nll_chain = w; w += nch;
    if (quarters) {
        p.qagg = w; w += nch * (kQ - 1) * FNW(D);
        p.sqagg = w; w += nch * (kQ - 1) * SNW(D);
        if (halves) p.qmom = w;
    }
    p.K = pl.K;
    p.nch = pl.nch;
    p.model = m->d_model;
    p.err = m->d_err;
    p.rank = 0;
    p.world = 1;
    p.store_state = 1;
    return PSSGP_OK;
}

// kPade mode (no closed form, no uniform step): per-step (F, Q) for local steps
// [0, n] (step n = the successor read by the smoother when it exists globally)
template <int D>
pssgp_status wide_prepare(pssgp_model* m, pssgp::wide::WParams& p, cudaStream_t s) {
    using namespace pssgp::wide;
    p.fq = nullptr;
    if (m->mode != kPade || p.n == 0) return PSSGP_OK;
    const int64_t nfq = p.n + ((p.k0 + p.n < p.nglob) ? 1 : 0);
    const size_t need = static_cast<size_t>(nfq) * FQW(D) * sizeof(double);
    if (need > m->fq_bytes) {
        if (m->fq) cudaFree(m->fq);
        m->fq = nullptr;
        m->fq_bytes = 0;
        if (cudaMalloc(&m->fq, need) != cudaSuccess) {
            cudaGetLastError();
            return fail(m, PSSGP_E_NOMEM, "cudaMalloc(per-step F, Q) failed");
        }
        m->fq_bytes = need;
    }
    if constexpr (D <= kGL) {
        if (wide_lpr_mask() & 64) {   // lane-per-row discretisation: one step per 8-lane group
            int occ = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kw_discretize_lpr<D>, 32 * kWWarps, 0);
            const int64_t want = (nfq * kGL + 32 * kWWarps - 1) / (32 * kWWarps);
            const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(m->sm_count) * std::max(1, occ))));
            {
                ProfScope ps(m, S_DISC, s);
                kw_discretize_lpr<D><<<grid, 32 * kWWarps, 0, s>>>(p.t, nfq, p.k0, m->d_model, m->fq);
                LAUNCH_CHECK(m, "kw_discretize_lpr");
            }
            p.fq = m->fq;
            return PSSGP_OK;
        }
    }
    if (m->fblock > 0 && m->fblock < D && (wide_lpr_mask() & 512)) {   // block-diagonal G, W: per-block threads
        bool done = false;
        with_fblock<D>(m, [&](auto fbc) {
            constexpr int FB = decltype(fbc)::value;
            if constexpr (FB < D) {
                constexpr int SPW = BlkDisc<D, FB>::SPW;
                int occ = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kw_discretize_blk<D, FB>, 32 * kBlkWarps, 0);
                const int64_t want = (nfq + SPW * kBlkWarps - 1) / (SPW * kBlkWarps);
                const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(m->sm_count) * std::max(1, occ))));
                ProfScope ps(m, S_DISC, s);
                kw_discretize_blk<D, FB><<<grid, 32 * kBlkWarps, 0, s>>>(p.t, nfq, p.k0, m->d_model, m->fq);
                done = true;
            }
        });
        if (done) {
            LAUNCH_CHECK(m, "kw_discretize_blk");
            p.fq = m->fq;
            return PSSGP_OK;
        }
    }
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kw_discretize<D>, 32 * kWWarps, sizeof(KDSmem<D>));
    const int64_t want = (nfq + kWWarps - 1) / kWWarps;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(m->sm_count) * std::max(1, occ))));
    {
        ProfScope ps(m, S_DISC, s);
        kw_discretize<D><<<grid, 32 * kWWarps, sizeof(KDSmem<D>), s>>>(p.t, nfq, p.k0, m->d_model, m->fq, p.err);
        LAUNCH_CHECK(m, "kw_discretize");
    }
    p.fq = m->fq;
    return PSSGP_OK;
}

// One step of kw_discretize on the device (pssgp_debug_discretize for kPade wide models).
template <int D>
pssgp_status wide_debug_discretize(pssgp_model* m, double dt, double* F, double* Q) {
    using namespace pssgp::wide;
    pssgp_status st = ensure_device(m);
    if (st) return st;
    WParams p;
    if ((st = wide_setup<D>(m, make_wplan<D>(m, 2), p))) return st;
    double* tbuf = nullptr;
    if (cudaMalloc(&tbuf, 2 * sizeof(double) + 2 * FQW(D) * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        return fail(m, PSSGP_E_NOMEM, "cudaMalloc(debug discretize)");
    }
    double* fq = tbuf + 2;
    const double th[2] = {0.0, dt};
    cudaMemcpy(tbuf, th, sizeof(th), cudaMemcpyHostToDevice);
    // the same kernel wide_prepare launches for this model (lane-per-row for D <= 8 by default)
    bool lpr = false;
    if constexpr (D <= kGL) lpr = (wide_lpr_mask() & 64) != 0;
    if constexpr (D <= kGL) {
        if (lpr) kw_discretize_lpr<D><<<1, 32 * kWWarps>>>(tbuf, 2, 0, m->d_model, fq);
    }
    bool blk = false;
    if (!lpr && m->fblock > 0 && m->fblock < D && (wide_lpr_mask() & 512)) {
        with_fblock<D>(m, [&](auto fbc) {
            constexpr int FB = decltype(fbc)::value;
            if constexpr (FB < D) {
                kw_discretize_blk<D, FB><<<1, 32 * kBlkWarps>>>(tbuf, 2, 0, m->d_model, fq);
                blk = true;
            }
        });
    }
    if (!lpr && !blk) {
        cudaFuncSetAttribute(kw_discretize<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(KDSmem<D>));
        kw_discretize<D><<<1, 32 * kWWarps, sizeof(KDSmem<D>)>>>(tbuf, 2, 0, m->d_model, fq, m->d_err);
    }
    std::vector<double> h(FQW(D));
    cudaError_t e = cudaMemcpy(h.data(), fq + FQW(D), FQW(D) * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(tbuf);
    if (e != cudaSuccess) return cuda_fail(m, e, "debug discretize");
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j) {
            F[i * D + j] = h[i * LD(D) + j];
            Q[i * D + j] = h[(D + i) * LD(D) + j];
        }
    return PSSGP_OK;
}

// Kogge-Stone levels with ping-pong buffers; returns the buffer holding the inclusive scan
template <int D>
double* wide_scan_f(pssgp_model* m, pssgp::wide::WParams& p, cudaStream_t s, pssgp_status& st) {
    using namespace pssgp::wide;
    ProfScope ps(m, S_K2, s);
    double* in = p.fagg;
    double* out = p.fbuf;
    for (int off = 1; off < p.nch; off <<= 1) {
        kw_scan_filter<D><<<p.nch, 32, sizeof(ScanSmemF<D>), s>>>(in, out, p.nch, off, p.err);
        std::swap(in, out);
    }
    cudaError_t e = cudaGetLastError();
    st = (e == cudaSuccess) ? PSSGP_OK : cuda_fail(m, e, "kw_scan_filter");
    return in;
}

template <int D>
double* wide_scan_s(pssgp_model* m, pssgp::wide::WParams& p, cudaStream_t s, pssgp_status& st) {
    using namespace pssgp::wide;
    ProfScope ps(m, S_K4, s);
    double* in = p.sagg;
    double* out = p.sbuf;
    for (int off = 1; off < p.nch; off <<= 1) {
        kw_scan_smoother<D><<<p.nch, 32, sizeof(ScanSmemS<D>), s>>>(in, out, p.nch, off);
        std::swap(in, out);
    }
    cudaError_t e = cudaGetLastError();
    st = (e == cudaSuccess) ? PSSGP_OK : cuda_fail(m, e, "kw_scan_smoother");
    return in;
}

template <int D>
pssgp_status wide_fold(pssgp_model* m, pssgp::wide::WParams& p, int nb, cudaStream_t s) {
    using namespace pssgp::wide;
    ProfScope ps(m, S_K1, s);
    if constexpr (D <= kGL) {
        // lane-per-row fold (D <= 8); PSSGP_WIDE_LPR=0 selects the shared-memory fold (A/B runs)
        if (wide_lpr_mask() & 1) {
            if (p.fq) kw_filter_fold_lpr<D, true><<<nb, 32 * kWWarps, sizeof(K1LSmem<D, true>), s>>>(p);
            else kw_filter_fold_lpr<D, false><<<nb, 32 * kWWarps, sizeof(K1LSmem<D, false>), s>>>(p);
            LAUNCH_CHECK(m, "kw_filter_fold_lpr");
            return PSSGP_OK;
        }
    } else if constexpr (wide_halves<D>()) {
        if (wide_half_rescans()) {   // lane-per-row fold in 16-lane groups (two half chains per warp)
            constexpr int G = kHalfG, W = kHalfWPC;
            const int nbh = (p.nch + W - 1) / W;
            with_fblock<D>(m, [&](auto fbc) {
                constexpr int FB = decltype(fbc)::value;
                if (p.fq) kw_filter_fold_lpr<D, true, G, W, FB><<<nbh, 32 * W, sizeof(K1LSmem<D, true, G, W>), s>>>(p);
                else kw_filter_fold_lpr<D, false, G, W, FB><<<nbh, 32 * W, sizeof(K1LSmem<D, false, G, W>), s>>>(p);
            });
            LAUNCH_CHECK(m, "kw_filter_fold_lpr (16-lane)");
            kw_combine_halves<D><<<p.nch, 32, sizeof(ScanSmemF<D>), s>>>(p);   // fagg = half 0 (x) half 1
            LAUNCH_CHECK(m, "kw_combine_halves");
            return PSSGP_OK;
        }
    }
    kw_filter_fold<D><<<nb, 32 * kWWarps, sizeof(K1Smem<D>), s>>>(p);
    LAUNCH_CHECK(m, "kw_filter_fold");
    return PSSGP_OK;
}

template <int D>
pssgp_status wide_fapply(pssgp_model* m, pssgp::wide::WParams& p, int nb, cudaStream_t s) {
    using namespace pssgp::wide;
    ProfScope ps(m, S_K3, s);
    if constexpr (D <= kGL) {
        if (p.qagg) {   // quarter-parallel Kalman rescan (the fold stored the quarter prefix aggregates)
            if (p.fq) kw_filter_apply_q<D, true><<<nb, 32 * kWWarps, sizeof(K3QSmem<D, true>), s>>>(p);
            else kw_filter_apply_q<D, false><<<nb, 32 * kWWarps, sizeof(K3QSmem<D, false>), s>>>(p);
            LAUNCH_CHECK(m, "kw_filter_apply_q");
            return PSSGP_OK;
        }
        // bit 4: lane-per-row Kalman rescan (uniform dt unless bit 2)
        if ((wide_lpr_mask() & 16) && (!p.fq || (wide_lpr_mask() & 4))) {
            if (p.fq) kw_filter_apply_lpr<D, true><<<nb, 32 * kWWarps, sizeof(K3LSmem<D, true>), s>>>(p);
            else kw_filter_apply_lpr<D, false><<<nb, 32 * kWWarps, sizeof(K3LSmem<D, false>), s>>>(p);
            LAUNCH_CHECK(m, "kw_filter_apply_lpr");
            return PSSGP_OK;
        }
    } else if constexpr (wide_halves<D>()) {
        if (p.qagg) {   // half-chain Kalman rescan (the fold stored the half prefix aggregates)
            constexpr int G = kHalfG, W = kHalfWPC;
            const int nbh = (p.nch + W - 1) / W;
            with_fblock<D>(m, [&](auto fbc) {
                constexpr int FB = decltype(fbc)::value;
                if (p.fq) kw_filter_apply_q<D, true, G, W, FB><<<nbh, 32 * W, sizeof(K3QSmem<D, true, G, W>), s>>>(p);
                else kw_filter_apply_q<D, false, G, W, FB><<<nbh, 32 * W, sizeof(K3QSmem<D, false, G, W>), s>>>(p);
            });
            LAUNCH_CHECK(m, "kw_filter_apply_q (16-lane)");
            if (p.store_state) {   // the half smoother aggregates and the chain's from the end moments
                kw_part_sagg<D, 2><<<p.nch, 32, sizeof(QAgPhase<D>), s>>>(p);
                LAUNCH_CHECK(m, "kw_part_sagg");
            }
            return PSSGP_OK;
        }
    }
    kw_filter_apply<D><<<nb, 32 * kWWarps, sizeof(K3Smem<D>), s>>>(p);
    LAUNCH_CHECK(m, "kw_filter_apply");
    return PSSGP_OK;
}

template <int D>
pssgp_status wide_sapply(pssgp_model* m, pssgp::wide::WParams& p, int nb, cudaStream_t s) {
    using namespace pssgp::wide;
    ProfScope ps(m, S_K5, s);
    if constexpr (D <= kGL) {
        if (p.sqagg) {  // quarter-parallel RTS rescan (kw_filter_apply_q stored the quarter smoother aggregates)
            if (wide_mbf_quarters() && p.y && p.mask) {   // the adjoint form needs y (the shard phase has none)
                if (p.fq) kw_smoother_mbf_q<D, true><<<nb, 32 * kWWarps, sizeof(K5MSmem<D, true>), s>>>(p);
                else kw_smoother_mbf_q<D, false><<<nb, 32 * kWWarps, sizeof(K5MSmem<D, false>), s>>>(p);
            } else {
                if (p.fq) kw_smoother_apply_q<D, true><<<nb, 32 * kWWarps, sizeof(K5QSmem<D, true>), s>>>(p);
                else kw_smoother_apply_q<D, false><<<nb, 32 * kWWarps, sizeof(K5QSmem<D, false>), s>>>(p);
            }
            LAUNCH_CHECK(m, "kw_smoother_apply_q");
            return PSSGP_OK;
        }
        // uniform dt only by default: with per-step (F, Q) read from global memory it measured
        // slower than the shared-memory kernel (C3 irregular K5w 8.4 -> 11.3 ms); bit 2 forces it
        if ((wide_lpr_mask() & 2) && (!p.fq || (wide_lpr_mask() & 4))) {
            if (p.fq) kw_smoother_apply_lpr<D, true><<<nb, 32 * kWWarps, sizeof(K5LSmem<D, true>), s>>>(p);
            else kw_smoother_apply_lpr<D, false><<<nb, 32 * kWWarps, sizeof(K5LSmem<D, false>), s>>>(p);
            LAUNCH_CHECK(m, "kw_smoother_apply_lpr");
            return PSSGP_OK;
        }
    } else if constexpr (wide_halves<D>()) {
        if (p.sqagg) {  // half-chain RTS rescan
            constexpr int G = kHalfG, W = kHalfWPC;
            const int nbh = (p.nch + W - 1) / W;
            with_fblock<D>(m, [&](auto fbc) {
                constexpr int FB = decltype(fbc)::value;
                if (wide_mbf() && p.y && p.mask) {   // the adjoint form needs y (the shard phase has none)
                    if (p.fq) kw_smoother_mbf_q<D, true, G, W, FB><<<nbh, 32 * W, sizeof(K5MSmem<D, true, G, W>), s>>>(p);
                    else kw_smoother_mbf_q<D, false, G, W, FB><<<nbh, 32 * W, sizeof(K5MSmem<D, false, G, W>), s>>>(p);
                } else {
                    if (p.fq) kw_smoother_apply_q<D, true, G, W, FB><<<nbh, 32 * W, sizeof(K5QSmem<D, true, G, W>), s>>>(p);
                    else kw_smoother_apply_q<D, false, G, W, FB><<<nbh, 32 * W, sizeof(K5QSmem<D, false, G, W>), s>>>(p);
                }
            });
            LAUNCH_CHECK(m, "kw_smoother_apply_q (16-lane)");
            return PSSGP_OK;
        }
    }
    if constexpr (D > 16) {
        if (wide_mbf() && p.y && p.mask && p.sagg) {   // adjoint form (needs y; the shard phase has none)
            const int nbm = (p.nch + kMbfWPC - 1) / kMbfWPC;
            with_fblock<D>(m, [&](auto fbc) {
                constexpr int FB = decltype(fbc)::value;
                if (p.fq) kw_smoother_mbf_q<D, true, 32, kMbfWPC, FB><<<nbm, 32 * kMbfWPC, sizeof(K5MSmem<D, true, 32, kMbfWPC>), s>>>(p);
                else kw_smoother_mbf_q<D, false, 32, kMbfWPC, FB><<<nbm, 32 * kMbfWPC, sizeof(K5MSmem<D, false, 32, kMbfWPC>), s>>>(p);
            });
            LAUNCH_CHECK(m, "kw_smoother_mbf_q (32-lane)");
            return PSSGP_OK;
        }
    }
    kw_smoother_apply<D><<<nb, 32 * kWWarps, sizeof(K5Smem<D>), s>>>(p);
    LAUNCH_CHECK(m, "kw_smoother_apply");
    return PSSGP_OK;
}

template <int D>
pssgp_status wide_posterior(pssgp_model* m, int64_t N, const double* t, const double* y, const uint8_t* mask,
                            double* mean, double* var, double* nll, cudaStream_t s, bool smooth) {
    if (N == 0) {
        if (nll && cudaMemsetAsync(nll, 0, sizeof(double), s) != cudaSuccess) return fail(m, PSSGP_E_CUDA, "memset");
        return PSSGP_OK;
    }
    const WPlan pl = make_wplan<D>(m, N);
    pssgp::wide::WParams p;
    pssgp_status st = wide_setup<D>(m, pl, p);
    if (st) return st;
    p.t = t; p.y = y; p.mask = mask;
    p.n = N; p.k0 = 0; p.nglob = N;
    p.mean = mean; p.var = var;
    p.store_state = smooth ? 1 : 0;
    if ((st = wide_prepare<D>(m, p, s))) return st;
    if ((st = wide_fold<D>(m, p, pl.nb, s))) return st;
    p.fagg = wide_scan_f<D>(m, p, s, st);
    if (st) return st;
    if ((st = wide_fapply<D>(m, p, pl.nb, s))) return st;
    if (smooth) {
        p.sagg = wide_scan_s<D>(m, p, s, st);
        if (st) return st;
        p.nll_out = nullptr;   // summed by k_nll_sum as on the NLL-only path: bit-identical NLL
        if ((st = wide_sapply<D>(m, p, pl.nb, s))) return st;
    }
    if (nll) return nll_sum(m, p.nll_chain, p.nch, nll, s);
    return PSSGP_OK;
}

// ---- sharded wide phases
template <int D>
pssgp_status wide_shard_reduce(pssgp_model* m, int64_t k0, int64_t n, int64_t Ng, const double* t, const double* y,
                               const uint8_t* mask, void* out, cudaStream_t s) {
    const WPlan pl = make_wplan<D>(m, n);
    pssgp::wide::WParams p;
    pssgp_status st = wide_setup<D>(m, pl, p);
    if (st) return st;
    p.t = t; p.y = y; p.mask = mask; p.n = n; p.k0 = k0; p.nglob = Ng;
    if ((st = wide_prepare<D>(m, p, s))) return st;
    if ((st = wide_fold<D>(m, p, pl.nb, s))) return st;
    double* inc = wide_scan_f<D>(m, p, s, st);
    if (st) return st;
    const cudaError_t e = cudaMemcpyAsync(out, inc + static_cast<int64_t>(pl.nch - 1) * pssgp::wide::FNW(D),
                                          pssgp::wide::FNW(D) * sizeof(double), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(m, e, "cudaMemcpyAsync(chunk aggregate)");
    return PSSGP_OK;
}

inline int ks_levels(int nch) {
    int l = 0;
    for (int off = 1; off < nch; off <<= 1) ++l;
    return l;
}

template <int D>
pssgp_status wide_shard_fapply(pssgp_model* m, int64_t k0, int64_t n, int64_t Ng, const double* t, const double* y,
                               const uint8_t* mask, const void* all, int rank, int world, void* sout, double* nllp,
                               cudaStream_t s) {
    const WPlan pl = make_wplan<D>(m, n);
    pssgp::wide::WParams p;
    pssgp_status st = wide_setup<D>(m, pl, p);
    if (st) return st;
    p.t = t; p.y = y; p.mask = mask; p.n = n; p.k0 = k0; p.nglob = Ng;
    p.in_filt = static_cast<const double*>(all);
    p.rank = rank; p.world = world;
    if (ks_levels(pl.nch) & 1) p.fagg = p.fbuf;          // where the reduce phase left the scan
    if ((st = wide_prepare<D>(m, p, s))) return st;
    if ((st = wide_fapply<D>(m, p, pl.nb, s))) return st;
    // the chunk's NLL partial travels in the smoother blob, after the aggregate
    double* blob = static_cast<double*>(sout);
    if ((st = nll_sum(m, p.nll_chain, p.nch, blob + pssgp::wide::SNW(D), s))) return st;
    if (nllp && (st = nll_sum(m, p.nll_chain, p.nch, nllp, s))) return st;
    double* inc = wide_scan_s<D>(m, p, s, st);
    if (st) return st;
    const cudaError_t e = cudaMemcpyAsync(sout, inc, pssgp::wide::SNW(D) * sizeof(double), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(m, e, "cudaMemcpyAsync(chunk smoother aggregate)");
    return PSSGP_OK;
}

template <int D>
pssgp_status wide_shard_sapply(pssgp_model* m, int64_t k0, int64_t n, int64_t Ng, const double* t, const void* all,
                               int rank, int world, double* mean, double* var, double* nll, cudaStream_t s) {
    const WPlan pl = make_wplan<D>(m, n);
    pssgp::wide::WParams p;
    pssgp_status st = wide_setup<D>(m, pl, p);
    if (st) return st;
    p.t = t; p.n = n; p.k0 = k0; p.nglob = Ng;
    p.in_smooth = static_cast<const double*>(all);
    p.rank = rank; p.world = world;
    p.mean = mean; p.var = var;
    if (ks_levels(pl.nch) & 1) p.sagg = p.sbuf;
    if ((st = wide_prepare<D>(m, p, s))) return st;
    if ((st = wide_sapply<D>(m, p, pl.nb, s))) return st;
    // total NLL: fixed-order sum over ranks of the partials carried in the gathered blobs
    if (nll) return nll_sum(m, static_cast<const double*>(all) + pssgp::wide::SNW(D), world, nll, s,
                            pssgp::wide::SNW(D) + 1);
    return PSSGP_OK;
}


// ---- NLL gradient of any model on a uniform grid (pssgp_nll_grad): primal fold +
// chain scan, forward rescan composing the chain adjoint maps, their reverse scan, backward
// rescan accumulating (Z, Cs, gr, C0), contraction with the per-parameter dF, dQ, dP_inf.
template <int D>
pssgp_status wide_nll_grad(pssgp_model* m, int64_t N, const double* t, const double* y, const uint8_t* mask,
                           double* nll, double* grad, cudaStream_t s) {
    using namespace pssgp::wide;
    const int npar = static_cast<int>(m->pder.size()) + 1;
    if (m->mode != kTable)
        return fail(m, PSSGP_E_UNSUPPORTED, "the gradient of this model needs a uniform grid (options.uniform_dt > 0)");
    if (N == 0) {
        cudaError_t e = cudaMemsetAsync(grad, 0, npar * sizeof(double), s);
        if (e == cudaSuccess && nll) e = cudaMemsetAsync(nll, 0, sizeof(double), s);
        return e == cudaSuccess ? PSSGP_OK : cuda_fail(m, e, "cudaMemsetAsync");
    }
    if (!m->d_gder) {   // dF_p, dQ_p at uniform_dt (Van Loan tangent, long double) and dP_inf_p
        const int d = m->d;
        std::vector<double> hbuf(static_cast<size_t>(npar - 1) * 3 * d * d);
        for (int pp = 0; pp + 1 < npar; ++pp) {
            pssgp_host::Mat F, Q, dF, dQ;
            pssgp_host::van_loan_tangent(m->ssm.G, m->ssm.W, m->pder[pp].dG, m->pder[pp].dW, d,
                                         static_cast<pssgp_host::ld>(m->udt), F, Q, dF, dQ);
            for (int e = 0; e < d * d; ++e) {
                hbuf[(static_cast<size_t>(pp) * 3 + 0) * d * d + e] = static_cast<double>(dF[e]);
                hbuf[(static_cast<size_t>(pp) * 3 + 1) * d * d + e] = static_cast<double>(dQ[e]);
                hbuf[(static_cast<size_t>(pp) * 3 + 2) * d * d + e] = static_cast<double>(m->pder[pp].dP[e]);
            }
        }
        if (cudaMalloc(&m->d_gder, std::max<size_t>(1, hbuf.size()) * sizeof(double)) != cudaSuccess) {
            cudaGetLastError();
            m->d_gder = nullptr;
            return fail(m, PSSGP_E_NOMEM, "cudaMalloc(gradient model)");
        }
        if (!hbuf.empty()) cudaMemcpy(m->d_gder, hbuf.data(), hbuf.size() * sizeof(double), cudaMemcpyHostToDevice);
    }
    const WPlan pl = make_wplan<D>(m, N, true);
    WParams p;
    pssgp_status st = wide_setup<D>(m, pl, p);
    if (st) return st;
    p.t = t; p.y = y; p.mask = mask;
    p.n = N; p.k0 = 0; p.nglob = N;
    p.store_state = 1;
    const size_t nch = static_cast<size_t>(pl.nch);
    const size_t need = (nch * CNW(D) + nch * GPN(D) + D * D + 8) * sizeof(double);
    if (need > m->gw_bytes) {
        if (m->gw) cudaFree(m->gw);
        m->gw = nullptr;
        m->gw_bytes = 0;
        if (cudaMalloc(&m->gw, need) != cudaSuccess) {
            cudaGetLastError();
            return fail(m, PSSGP_E_NOMEM, "cudaMalloc(gradient workspace)");
        }
        m->gw_bytes = need;
    }
    GradBufs gb;
    gb.gagg = p.sagg;
    gb.gbuf = p.sbuf;
    gb.gcar = reinterpret_cast<double*>(m->gw);
    gb.gpart = gb.gcar + nch * CNW(D);
    gb.gc0 = gb.gpart + nch * GPN(D);
    if ((st = wide_fold<D>(m, p, pl.nb, s))) return st;
    p.fagg = wide_scan_f<D>(m, p, s, st);
    if (st) return st;
    {
        ProfScope ps(m, S_K3, s);
        kw_grad_forward<D><<<pl.nb, 32 * kWWarps, sizeof(GFwdSmem<D>), s>>>(p, gb);
        LAUNCH_CHECK(m, "kw_grad_forward");
    }
    double* in = gb.gagg;
    double* out = gb.gbuf;
    {
        ProfScope ps(m, S_K4, s);
        for (int off = 1; off < p.nch; off <<= 1) {
            kw_scan_adjoint<D><<<p.nch, 32, sizeof(ScanSmemA<D>), s>>>(in, out, p.nch, off);
            std::swap(in, out);
        }
        LAUNCH_CHECK(m, "kw_scan_adjoint");
    }
    {
        ProfScope ps(m, S_GRAD, s);
        kw_grad_backward<D><<<pl.nb, 32 * kWWarps, sizeof(GBwdSmem<D>), s>>>(p, gb, in);
        LAUNCH_CHECK(m, "kw_grad_backward");
    }
    {
        ProfScope ps(m, S_RED, s);
        k_grad_contract<D><<<1, 256, 0, s>>>(gb.gpart, p.nch, gb.gc0, m->d_gder, npar, m->r, grad);
        LAUNCH_CHECK(m, "k_grad_contract");
    }
    if (nll) return nll_sum(m, p.nll_chain, p.nch, nll, s);
    return PSSGP_OK;
}


// ---- batched series with per-series log hyper-parameters (pssgp_batch_theta.cuh): the series
// models on the device, then one warp per series for the posterior or the NLL gradient
template <int D>
pssgp_status wide_batched_theta(pssgp_model* m, int nseg, const int64_t* off, const double* theta, int64_t N,
                                const double* t, const double* y, const uint8_t* mask, double* mean, double* var,
                                double* nll, double* grad, cudaStream_t s) {
    using namespace pssgp::wide;
    if (!m->bt_ok || !(m->udt > 0.0))
        return fail(m, PSSGP_E_UNSUPPORTED,
                    "batched per-series hyper-parameters need Matern / periodic / quasi-periodic components on a "
                    "uniform grid (options.uniform_dt > 0)");
    const int nc = static_cast<int>(m->bdesc.size() / 6);
    if (nc > kBMaxComp) return fail(m, PSSGP_E_UNSUPPORTED, "too many components");
    BModelDesc md;
    std::memset(&md, 0, sizeof(md));
    md.nc = nc;
    md.npar = static_cast<int>(m->pder.size()) + 1;
    md.d = D;
    md.udt = m->udt;
    for (int c = 0; c < nc; ++c) {
        const int* v = &m->bdesc[6 * c];
        md.c[c] = BComp{v[0], v[1], v[2], v[3], v[4], v[5]};
    }
    const size_t nrec = static_cast<size_t>(nseg) * BREC(D, md.npar);
    const size_t need = (nrec + static_cast<size_t>(N) * CNW(D) + D + 8) * sizeof(double);
    if (need > m->bw_bytes) {
        if (m->bw) cudaFree(m->bw);
        m->bw = nullptr;
        m->bw_bytes = 0;
        if (cudaMalloc(&m->bw, need) != cudaSuccess) {
            cudaGetLastError();
            return fail(m, PSSGP_E_NOMEM, "cudaMalloc(batched-theta workspace)");
        }
        m->bw_bytes = need;
    }
    double* recs = reinterpret_cast<double*>(m->bw);
    double* xs = recs + nrec;
    double* Hd = xs + static_cast<size_t>(N) * CNW(D);
    {
        double hh[D];
        for (int i = 0; i < D; ++i) hh[i] = static_cast<double>(m->ssm.H[i]);
        cudaMemcpyAsync(Hd, hh, sizeof(hh), cudaMemcpyHostToDevice, s);
        cudaStreamSynchronize(s);   // hh is a host stack buffer
    }
    {
        ProfScope ps(m, S_DISC, s);
        kb_build<D><<<(nseg + 127) / 128, 128, 0, s>>>(md, nseg, theta, recs);
        LAUNCH_CHECK(m, "kb_build");
    }
    BParamsT q;
    q.off = off; q.nseg = nseg; q.npar = md.npar; q.udt = m->udt; q.recs = recs;
    q.t = t; q.y = y; q.mask = mask; q.xs = xs;
    q.mean = mean; q.var = var; q.nll = nll; q.grad = grad; q.err = m->d_err;
    static_assert(sizeof(BSmem<D>) <= 48 * 1024, "per-series shared state");
    // warps per series: one by default.  2 or 4 (PSSGP_BT_NW, A/B) split the series' matrix products
    // over more threads but pay a CTA barrier per phase: measured on 1,024 CO2 J = 3 series (d = 18),
    // NLL + gradient 46.0 / 56.7 / 78.0 ms and posterior 70.3 / 86.7 / 140.9 ms for 1 / 2 / 4 warps
    // (profiles/r2/bt_nw_ab.txt)
    int nw = 1;
    if (const char* e = getenv("PSSGP_BT_NW")) {
        const int v = atoi(e);
        if (v == 1 || v == 2 || v == 4) nw = v;
    }
    auto launch = [&](auto nwc) {
        constexpr int NW = decltype(nwc)::value;
        if (grad) {
            ProfScope ps(m, S_GRAD, s);
            kb_nll_grad<D, NW><<<nseg, 32 * NW, sizeof(BSmem<D>), s>>>(q, Hd);
            LAUNCH_CHECK(m, "kb_nll_grad");
        } else {
            ProfScope ps(m, S_K3, s);
            kb_posterior<D, NW><<<nseg, 32 * NW, sizeof(BSmem<D>), s>>>(q, Hd);
            LAUNCH_CHECK(m, "kb_posterior");
        }
        return PSSGP_OK;
    };
    if (nw == 4) return launch(std::integral_constant<int, 4>{});
    if (nw == 2) return launch(std::integral_constant<int, 2>{});
    return launch(std::integral_constant<int, 1>{});
}

}  // namespace widehost
}  // namespace pssgp_internal
