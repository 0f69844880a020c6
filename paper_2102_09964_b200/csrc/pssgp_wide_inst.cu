// pssgp_wide_inst.cu — the warp-per-chain path (pssgp_wide.cuh kernels, pssgp_wide_host.cuh launch
// sequences) for ONE state dimension, compiled once per entry of pssgp_dims.h with -DPSSGP_WD=d so
// the dimensions build in parallel; pssgp_api.cu reaches them through wide_ops_for(d).
#ifndef PSSGP_WD
#error "compile with -DPSSGP_WD=<state dimension>"
#endif
#define PSSGP_NO_MISC_KERNELS 1   // k_nll_sum / k_merge / k_gather live in pssgp_api.cu
#include "pssgp_wide_host.cuh"

namespace pssgp_internal {
namespace {
constexpr int D = PSSGP_WD;

void wplan(pssgp_model* m, int64_t N, int64_t* K, int64_t* nch, int* nb, int* threads) {
    const widehost::WPlan wp = widehost::make_wplan<D>(m, N);
    if (K) *K = wp.K;
    if (nch) *nch = wp.nch;
    if (nb) *nb = wp.nb;
    if (threads) *threads = 32 * pssgp::wide::kWWarps;
}
}  // namespace

template <>
const WideOps* wide_ops<D>() {
    static const WideOps ops = {widehost::wide_posterior<D>, widehost::wide_shard_reduce<D>,
                                widehost::wide_shard_fapply<D>, widehost::wide_shard_sapply<D>,
                                widehost::wide_debug_discretize<D>, widehost::wide_nll_grad<D>,
                                widehost::wide_batched_theta<D>, wplan};
    return &ops;
}
}  // namespace pssgp_internal
