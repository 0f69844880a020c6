// pssgp_internal.hpp — library-internal state shared by the translation units of libpssgp.so
// (pssgp_api.cu: C ABI + the d <= 3 thread-per-chain path; pssgp_wide_inst.cu, compiled once per
// state dimension listed in pssgp_dims.h: the warp-per-chain path).  Not part of include/pssgp.h.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/pssgp.h"
#include "host_model.hpp"
#include "pssgp_dims.h"

namespace pssgp_internal {
namespace ph = pssgp_host;
constexpr int kMaxD = 3;              // thread-per-chain path: d = 1, 2, 3
constexpr int kSlots = 9;
enum Slot { S_K1 = 0, S_K2, S_K3, S_K4, S_K5, S_K6, S_RED, S_GRAD, S_DISC };
}  // namespace pssgp_internal

struct pssgp_model {
    int d = 0;
    pssgp_host::Ssm ssm;                 // balanced host model (long double)
    bool closed = false;         // standalone Matern closed form
    int mode = 1 /* kTable */;           // DiscMode of the kernels (kClosed / kTable / kPade)
    double lam = 0.0, s2 = 0.0, r = 0.0;
    double udt = 0.0;
    std::vector<double> Fu, Qu;  // F(udt), Q(udt) row-major d x d
    std::vector<pssgp_host::ParamDeriv> pder;   // d(G, W, P_inf) / d theta_p, p < npar - 1 (log noise last)
    std::vector<int> bdesc;      // per component: kind (1 Matern, 2 periodic, 3 quasi, 0 other), order,
                                 // 2 nu, state offset, block size, first parameter (batched-theta path)
    bool bt_ok = false;          // every component has a closed-form per-series model
    char* bw = nullptr;          // batched-theta workspace (series model records, filtered moments)
    size_t bw_bytes = 0;
    double* d_gder = nullptr;    // device: per parameter dF, dQ (at udt), dP_inf (d x d each)
    char* gw = nullptr;          // general-model gradient workspace
    size_t gw_bytes = 0;
    int device = 0;
    int64_t forced_K = 0;
    int blocks_per_sm = 0;
    int sm_count = 0;
    int occ = 0;
    int occ32 = 0;               // fp32 build (pssgp_posterior_f32): resident CTAs / SM
    // workspace
    char* ws = nullptr;
    size_t ws_bytes = 0;
    unsigned long long* d_err = nullptr;  // separate small allocation
    double* d_scalar = nullptr;           // scratch nll scalar
    double* d_model = nullptr;            // wide path: F, Q, Pinf, H, r, udt (device copy)
    int wocc = 0;                         // wide path: resident CTAs / SM
    int wchains = 0;                      // wide path: resident chains / SM when the kernels use other CTA shapes
    int wocc_grad = 0;                    // wide path, d > 16: resident CTAs / SM of the gradient kernels
    int fblock = 0;                       // aligned block size (2, 4 or d) containing every nonzero of G and W
    char* io = nullptr;                   // e2e device buffers
    size_t io_bytes = 0;
    char* mg = nullptr;                   // pssgp_predict merged-grid buffers
    size_t mg_bytes = 0;
    double* bt = nullptr;                 // batched: per-step NLL terms
    size_t bt_bytes = 0;
    double* gb = nullptr;                 // batched gradient: head / tail tangent pieces per chain
    size_t gb_bytes = 0;
    double* fq = nullptr;                 // wide path, kPade mode: per-step (F, Q)
    size_t fq_bytes = 0;
    // pipelined host API (pssgp_posterior_host_async): two slots, each with its own stream and
    // device I/O buffers; inputs, computes (one stream, call order) and outputs on separate streams
    char* aio[2] = {nullptr, nullptr};
    size_t aio_bytes[2] = {0, 0};
    cudaStream_t astream[2] = {nullptr, nullptr};   // per slot: host -> device copies
    cudaStream_t aout[2] = {nullptr, nullptr};      // per slot: device -> host copies
    cudaStream_t acs = nullptr;                      // computes, in call order
    cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_comp[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
    bool arec[2] = {false, false};                   // the slot has a previous call
    int aslot = 0;
    cudaStream_t last_stream = nullptr;
    int64_t err_index = -1;
    std::string last_err;
    // sharded plan state
    int64_t sh_k0 = -1, sh_n = -1, sh_N = -1;
    // profiling
    bool prof = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[pssgp_internal::kSlots];
    std::vector<cudaEvent_t> ev_pool;
};

namespace pssgp_internal {

inline pssgp_status fail(pssgp_model* m, pssgp_status st, const std::string& msg, int64_t idx = -1) {
    if (m) {
        m->last_err = msg;
        m->err_index = idx;
    }
    return st;
}

inline pssgp_status cuda_fail(pssgp_model* m, cudaError_t e, const char* where) {
    return fail(m, PSSGP_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

inline cudaEvent_t get_event(pssgp_model* m) {
    if (!m->ev_pool.empty()) {
        cudaEvent_t e = m->ev_pool.back();
        m->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

inline const char* slot_name(int slot) {
    static const char* names[kSlots] = {"k_filter_reduce", "k_filter_scan", "k_filter_apply",
                                        "k_smoother_scan", "k_smoother_apply", "k_nll_sum", "k_reduce_blocks",
                                        "k_grad_fold", "k_discretize"};
    return (slot >= 0 && slot < kSlots) ? names[slot] : "";
}

// One phase of a call: an NVTX range named after the profile slot (seen by nsys / ncu --nvtx; a no-op
// without a tool attached) and, when profiling is enabled, CUDA events on the launch stream.
struct ProfScope {
    pssgp_model* m;
    int slot;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    ProfScope(pssgp_model* m_, int slot_, cudaStream_t s_) : m(m_), slot(slot_), s(s_) {
        nvtxRangePushA(slot_name(slot));
        if (m->prof) {
            a = get_event(m);
            cudaEventRecord(a, s);
        }
    }
    ~ProfScope() {
        if (m->prof) {
            cudaEvent_t b = get_event(m);
            cudaEventRecord(b, s);
            m->ev[slot].emplace_back(a, b);
        }
        nvtxRangePop();
    }
};

// NVTX range around one C-ABI call (the pipeline stage of PAPER.md:168-172 it runs)
struct NvtxCall {
    explicit NvtxCall(const char* name) { nvtxRangePushA(name); }
    ~NvtxCall() { nvtxRangePop(); }
};

#define LAUNCH_CHECK(m, where)                                    \
    do {                                                          \
        cudaError_t e_ = cudaGetLastError();                      \
        if (e_ != cudaSuccess) return cuda_fail((m), e_, where);  \
    } while (0)

// defined in pssgp_api.cu
pssgp_status ensure_device(pssgp_model* m);
// fixed-order sum of parts[0], parts[stride], ..., parts[(nb - 1) stride] into *out (one CTA)
pssgp_status nll_sum(pssgp_model* m, const double* parts, int nb, double* out, cudaStream_t s, int stride = 1);

// The warp-per-chain path of one compiled state dimension D (pssgp_wide_inst.cu, -DPSSGP_WD=D).
struct WideOps {
    pssgp_status (*posterior)(pssgp_model*, int64_t N, const double* t, const double* y, const uint8_t* mask,
                              double* mean, double* var, double* nll, cudaStream_t s, bool smooth);
    pssgp_status (*shard_reduce)(pssgp_model*, int64_t k0, int64_t n, int64_t Ng, const double* t, const double* y,
                                 const uint8_t* mask, void* out, cudaStream_t s);
    pssgp_status (*shard_fapply)(pssgp_model*, int64_t k0, int64_t n, int64_t Ng, const double* t, const double* y,
                                 const uint8_t* mask, const void* all, int rank, int world, void* sout, double* nllp,
                                 cudaStream_t s);
    pssgp_status (*shard_sapply)(pssgp_model*, int64_t k0, int64_t n, int64_t Ng, const double* t, const void* all,
                                 int rank, int world, double* mean, double* var, double* nll,
                                 cudaStream_t s);
    pssgp_status (*debug_disc)(pssgp_model*, double dt, double* F, double* Q);
    pssgp_status (*nll_grad)(pssgp_model*, int64_t N, const double* t, const double* y, const uint8_t* mask,
                             double* nll, double* grad, cudaStream_t s);
    pssgp_status (*batched_theta)(pssgp_model*, int nseg, const int64_t* off, const double* theta, int64_t N,
                                  const double* t, const double* y, const uint8_t* mask, double* mean, double* var,
                                  double* nll, double* grad, cudaStream_t s);
    void (*plan)(pssgp_model*, int64_t N, int64_t* K, int64_t* nch, int* nb, int* threads);
};
template <int D>
const WideOps* wide_ops();
#define PSSGP_DECL_WIDE(DD) template <> const WideOps* wide_ops<DD>();
PSSGP_WIDE_DIMS(PSSGP_DECL_WIDE)
#undef PSSGP_DECL_WIDE

inline const WideOps* wide_ops_for(int d) {
    switch (d) {
#define PSSGP_CASE_WIDE(DD) case DD: return wide_ops<DD>();
        PSSGP_WIDE_DIMS(PSSGP_CASE_WIDE)
#undef PSSGP_CASE_WIDE
        default: return nullptr;
    }
}

}  // namespace pssgp_internal
