// pssgp_kernels.cuh — sm_100a kernels of the PSSGP hot path (one-wave, three-pass scan).
//
// Decomposition: the grid is ONE wave of CTAs (148 SMs x
// resident CTAs).  Thread c owns the contiguous chain [c K, (c+1) K) of K time
// steps; CTA b owns chains [128 b, 128 b + 128).
//
//   k_filter_reduce   (K1)  per chain: discretise + build + fold filter elements
//                           (rank-one fold, PAPER.md:116-121 with J_k = u u^T / S)
//                           -> chain aggregate; CTA tree-reduce -> block aggregate.
//   (K2)                    folded into K3's prologue: each CTA reduces the block
//                           aggregates of all earlier CTAs -> collapsed prefix (xbar, P).
//   k_filter_apply    (K3)  per CTA: scan of its chain aggregates, then per chain
//                           the Kalman recursion from the carry (Prop. 1 proof order,
//                           PAPER.md:326-330): writes (xbar_k, P_k), NLL partials,
//                           and the chain's smoother aggregate (E, g, L) from the
//                           cross-covariance Cov(x_k0, x_k1+1 | y_1:k1).
//   (K4)                    folded into K5's prologue (block smoother aggregates of
//                           all later CTAs), which also sums the NLL partials.
//   k_smoother_apply  (K5)  per CTA: reverse scan of chain smoother aggregates, then
//                           per chain the RTS recursion (Prop. 2 proof order,
//                           PAPER.md:431-435) -> mean = H m^s, var = H P^s H^T.
//   k_nll_sum         (K6)  fixed-order sum of per-CTA NLL partials (deterministic).
//
// Global prefixes collapse to (0, xbar, P, 0, 0) and global suffixes to
// (0, m^s, P^s) (A_1 = 0 by Eq. (7); E_N = 0), so applying a carry to a chain
// is one Kalman / RTS step per element: the general operator only combines
// chain / block aggregates.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "pssgp_math.cuh"

namespace PSSGP_NS {

#ifndef PSSGP_UNROLL
#define PSSGP_UNROLL 1                  // step-loop unroll (lets ptxas interleave consecutive steps)
#endif
#ifndef PSSGP_MINB
#define PSSGP_MINB 3                    // resident CTAs per SM the main kernels are register-capped for
#endif
constexpr int kUnroll = PSSGP_UNROLL;
#ifndef PSSGP_THREADS
#define PSSGP_THREADS 128               // threads per CTA of the thread-per-chain kernels
#endif
constexpr int kThreads = PSSGP_THREADS;
constexpr int kWarps = kThreads / 32;
constexpr int kWin = 16;                // staging window (steps) per chain
constexpr int kCarryThreads = 256;      // single-CTA scan kernels
#ifndef PSSGP_TY_PF
#define PSSGP_TY_PF 0                   // K5: L2 prefetch distance (staging windows) of t; 0 = off (measured: no gain)
#endif
#ifndef PSSGP_K5_PF
#define PSSGP_K5_PF 2                   // K5: L2 prefetch distance (steps) of the filtered state, 0 = off
#endif

// error word: (class << 56) | (index << 8) | code; atomicMin keeps data errors
// (input / unsupported dt, class 0) ahead of their numerical consequences
// (class 1), then the first failing index.
enum : unsigned { kErrInput = 2, kErrNumeric = 3, kErrUnsupported = 6 };

__device__ __forceinline__ void raise_error(unsigned long long* err, int64_t gidx, unsigned code) {
    const unsigned long long cls = (code == kErrNumeric) ? 1ULL : 0ULL;
    const unsigned long long w = (cls << 56) | ((static_cast<unsigned long long>(gidx) & 0xffffffffffffULL) << 8) | code;
    if (w < *reinterpret_cast<volatile unsigned long long*>(err)) atomicMin(err, w);
}

// combine() of the filtering operator reports a singular (I + C_i J_j) (false); the smoothing and
// tangent operators cannot fail.  Every operator tree ANDs the results into a per-thread flag and
// latches kErrNumeric once after the tree.
template <typename Agg>
__device__ __forceinline__ bool combine_chk(const Agg& a, const Agg& b, Agg& r) {
    if constexpr (std::is_same_v<decltype(combine(a, b, r)), bool>) {
        return combine(a, b, r);
    } else {
        combine(a, b, r);
        return true;
    }
}

template <int D>
struct KParams {
    ModelParams<D> m;
    const double* t;        // local step 0; t[-1], t[n] valid when they exist globally
    const double* y;
    const uint8_t* mask;
    int64_t n;              // local steps
    int64_t k0;             // global index of local step 0
    int64_t nglob;          // global number of steps
    int64_t K;              // chain length
    int nb;                 // CTAs of the apply kernels
    real* chain_f;        // [FN][nb*128]  chain filter aggregates (SoA)
    real* block_f;        // [nb][FN]
    real* fcarry;         // [nb][CN]      global prefix entering each CTA
    real* xp;             // filtered (xbar, P), lane-interleaved [warp][K][CN][32]
    real* chain_s;        // [SN][nb*128]
    real* block_s;        // [nb][SN]
    real* scarry;         // [nb][CN]      global suffix after each CTA
    double* nll_block;      // [nb]
    double* mean;
    double* var;
    const real* in_filt;  // sharded: all ranks' filter aggregates [world][FN] (nullable)
    const real* in_smooth;// sharded: all ranks' smoother aggregates [world][SN] (nullable)
    int rank, world;
    real* out_agg;        // sharded: chunk aggregate output (nullable)
    double* nll_out;        // nll scalar output (nullable)
    unsigned long long* err;
    int store_state;        // K3: write (xbar, P) and smoother aggregates (0 for NLL-only)
    unsigned long long* flag;   // flag[0]: K3 block-carry publication word (set to 1 by logical CTA 0);
                                // flag[1]: K3 tile ticket (logical CTA index = arrival order); both reset
                                // to 0 by K1 (stream-ordered, so CUDA-graph replays are safe).  Single-pass
                                // kernel: flag[2] counts published block aggregates, flag[3] finished
                                // CTAs; the last CTA to finish resets flag[0..3].
};

// The last CTA of a single-pass launch resets the publication word, ticket and counters (the host
// also zeroes them before each single-pass launch; K1 resets flag[0..1] before every K3).
__device__ __forceinline__ void k3_finish(unsigned long long* flag, int nb) {
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(flag + 3, 1ull) == static_cast<unsigned long long>(nb) - 1) {
        flag[0] = 0ull; flag[1] = 0ull; flag[2] = 0ull; flag[3] = 0ull;
        __threadfence();
    }
}

// K3's logical CTA index: the arrival order of the CTAs (an atomic ticket), so the CTA that scans
// the block aggregates and publishes every CTA's carry (logical 0) is the first one that ever ran.
// A CTA spins only after taking a later ticket, i.e. after logical 0 is resident, and logical 0
// waits on nobody: forward progress needs no co-residency or dispatch-order assumption (other
// streams, MPS, grids larger than one wave).
__device__ __forceinline__ int k3_ticket(unsigned long long* flag, int* s_bid) {
    if (threadIdx.x == 0) *s_bid = static_cast<int>(atomicAdd(flag + 1, 1ull));
    __syncthreads();
    return *s_bid;
}

// ------------------------------------------------------------------ warp shuffles of aggregates
template <typename T>
__device__ __forceinline__ void shfl_up_all(T& dst, const T& src, int off) {
    constexpr int n = sizeof(T) / sizeof(real);
    const real* s = reinterpret_cast<const real*>(&src);
    real* d = reinterpret_cast<real*>(&dst);
#pragma unroll
    for (int i = 0; i < n; ++i) d[i] = __shfl_up_sync(0xffffffffu, s[i], off);
}
template <typename T>
__device__ __forceinline__ void shfl_down_all(T& dst, const T& src, int off) {
    constexpr int n = sizeof(T) / sizeof(real);
    const real* s = reinterpret_cast<const real*>(&src);
    real* d = reinterpret_cast<real*>(&dst);
#pragma unroll
    for (int i = 0; i < n; ++i) d[i] = __shfl_down_sync(0xffffffffu, s[i], off);
}
template <typename T>
__device__ __forceinline__ void load_soa(T& a, const real* base, int64_t stride, int64_t idx) {
    constexpr int n = sizeof(T) / sizeof(real);
    real* d = reinterpret_cast<real*>(&a);
#pragma unroll
    for (int i = 0; i < n; ++i) d[i] = base[i * stride + idx];
}
template <typename T>
__device__ __forceinline__ void store_soa(const T& a, real* base, int64_t stride, int64_t idx) {
    constexpr int n = sizeof(T) / sizeof(real);
    const real* s = reinterpret_cast<const real*>(&a);
#pragma unroll
    for (int i = 0; i < n; ++i) base[i * stride + idx] = s[i];
}
template <typename T>
__device__ __forceinline__ void load_aos(T& a, const real* base) {
    constexpr int n = sizeof(T) / sizeof(real);
    real* d = reinterpret_cast<real*>(&a);
#pragma unroll
    for (int i = 0; i < n; ++i) d[i] = base[i];
}
template <typename T>
__device__ __forceinline__ void load_aos_cg(T& a, const real* base) {   // L2 (written by other CTAs)
    constexpr int n = sizeof(T) / sizeof(real);
    real* d = reinterpret_cast<real*>(&a);
#pragma unroll
    for (int i = 0; i < n; ++i) d[i] = __ldcg(base + i);
}
template <typename T>
__device__ __forceinline__ void store_aos(const T& a, real* base) {
    constexpr int n = sizeof(T) / sizeof(real);
    const real* s = reinterpret_cast<const real*>(&a);
#pragma unroll
    for (int i = 0; i < n; ++i) base[i] = s[i];
}

// ------------------------------------------------------------------ filtered-state record layout
// xp holds, per (warp, step), one block of CN * 32 reals (the warp's 32 chains).  PSSGP_VEC_STATE = 1:
// component pairs (2c, 2c+1) of lane l at block + 64 c + 2 l (one 16-byte access per lane for fp64),
// an odd last component at block + 64 (CN / 2) + l; 0: component i of lane l at block + 32 i + l.
// Every site passes `at` = block + lane (the lane's component-0 position of the plain layout).
#ifndef PSSGP_VEC_STATE
#define PSSGP_VEC_STATE 0
#endif
#ifndef PSSGP_CS_HINTS
#define PSSGP_CS_HINTS 1                // bit 0: streaming (evict-first) record stores; bit 1: streaming record loads; bit 2: output stores
#endif
template <typename T> struct Vec2;
template <> struct Vec2<double> { using type = double2; };
template <> struct Vec2<float> { using type = float2; };

template <int D>
__device__ __forceinline__ void ld_state(const real* at, int lane, real (&v)[CN(D)]) {
    if (PSSGP_VEC_STATE) {
        using V = typename Vec2<real>::type;
        const real* blk = at - lane;
#pragma unroll
        for (int c = 0; c < CN(D) / 2; ++c) {
            const V q = *reinterpret_cast<const V*>(blk + 64 * c + 2 * lane);
            v[2 * c] = q.x;
            v[2 * c + 1] = q.y;
        }
        if (CN(D) & 1) v[CN(D) - 1] = blk[64 * (CN(D) / 2) + lane];
    } else if (PSSGP_CS_HINTS & 2) {
#pragma unroll
        for (int i = 0; i < CN(D); ++i) v[i] = __ldcs(at + i * 32);
    } else {
#pragma unroll
        for (int i = 0; i < CN(D); ++i) v[i] = at[i * 32];
    }
}
template <int D>
__device__ __forceinline__ void ld_xP(const real* at, int lane, real (&x)[D], real (&P)[ns(D)]) {
    real v[CN(D)];
    ld_state<D>(at, lane, v);
#pragma unroll
    for (int i = 0; i < D; ++i) x[i] = v[i];
#pragma unroll
    for (int i = 0; i < ns(D); ++i) P[i] = v[D + i];
}
template <int D>
__device__ __forceinline__ void st_xP(real* at, int lane, const real (&x)[D], const real (&P)[ns(D)]) {
    real v[CN(D)];
#pragma unroll
    for (int i = 0; i < D; ++i) v[i] = x[i];
#pragma unroll
    for (int i = 0; i < ns(D); ++i) v[D + i] = P[i];
    if (PSSGP_VEC_STATE) {
        using V = typename Vec2<real>::type;
        real* blk = at - lane;
#pragma unroll
        for (int c = 0; c < CN(D) / 2; ++c) {
            V q;
            q.x = v[2 * c];
            q.y = v[2 * c + 1];
            *reinterpret_cast<V*>(blk + 64 * c + 2 * lane) = q;
        }
        if (CN(D) & 1) blk[64 * (CN(D) / 2) + lane] = v[CN(D) - 1];
    } else if (PSSGP_CS_HINTS & 1) {
#pragma unroll
        for (int i = 0; i < CN(D); ++i) __stcs(at + i * 32, v[i]);
    } else {
#pragma unroll
        for (int i = 0; i < CN(D); ++i) at[i * 32] = v[i];
    }
}

// ------------------------------------------------------------------ asynchronous staging
// A warp's 32 chains are 32 contiguous segments of K steps.  Windows of kWinA
// steps of t and y for all 32 chains are copied global -> shared with cp.async
// (8-byte copies, 8 lanes per 64-byte row segment) into a TRANSPOSED, padded
// layout [step][chain] so that each lane later reads its own chain
// conflict-free; two buffers per warp so the copy of window w+1 overlaps the
// arithmetic of window w.  Out-of-range elements are zero-filled (src-size 0).
// The observation mask is prefetched one step ahead into a register instead.
constexpr int kWinA = 8;
struct AsyncStage {
    double t[2][kWinA][33];
    double y[2][kWinA][33];
};

__device__ __forceinline__ void cp_async8(void* dst, const void* src, int src_bytes) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <bool WITH_Y = true>
__device__ __forceinline__ void issue_copies(double (*ts)[33], double (*ys)[33], const double* __restrict__ t,
                                             const double* __restrict__ y, int64_t wbase, int64_t K, int64_t n,
                                             int64_t j0, int lane) {
    const int col = lane & (kWinA - 1), rb = lane / kWinA;
    const int64_t j = j0 + col;
#pragma unroll
    for (int i = 0; i < 32 / (32 / kWinA); ++i) {
        const int r = rb + (32 / kWinA) * i;
        const int64_t idx = wbase + r * K + j;
        const bool ok = (j >= 0) && (j < K) && (idx < n);
        cp_async8(&ts[col][r], ok ? t + idx : t, ok ? 8 : 0);
        if (WITH_Y) cp_async8(&ys[col][r], ok ? y + idx : y, ok ? 8 : 0);
    }
    cp_async_commit();
}

__device__ __forceinline__ void issue_window(AsyncStage& s, int buf, const double* __restrict__ t,
                                             const double* __restrict__ y, int64_t wbase, int64_t K, int64_t n,
                                             int64_t j0, int lane) {
    issue_copies<true>(s.t[buf], s.y[buf], t, y, wbase, K, n, j0, lane);
}

// L2 prefetch of this lane's chain at chain-relative step j (t, and y when WITH_Y).
template <bool WITH_Y>
__device__ __forceinline__ void prefetch_ty_l2(const double* __restrict__ t, const double* __restrict__ y,
                                               int64_t kb, int64_t j, int64_t ke) {
    if (kb + j < ke) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(t + kb + j));
        if (WITH_Y) asm volatile("prefetch.global.L2 [%0];" ::"l"(y + kb + j));
    }
}

// ------------------------------------------------------------------ mask words
// The mask bytes of one staging window (kWinA = 8 steps) as one 64-bit word, loaded one
// window ahead (HBM latency exceeds one step of compute); byte jj = step j0 + jj.  Bytes at
// or past the chain end are 0.  Vector load when the 8 bytes are aligned and in range.
static_assert(kWinA == 8, "mask words hold 8 steps");
__device__ __forceinline__ unsigned long long mask_word(const uint8_t* __restrict__ mask, int64_t pos, int64_t ke) {
    if (pos >= ke) return 0ull;
    const uint8_t* a = mask + pos;
    if ((reinterpret_cast<uintptr_t>(a) & 7) == 0 && pos + 8 <= ke)
        return __ldg(reinterpret_cast<const unsigned long long*>(a));
    unsigned long long w = 0ull;
#pragma unroll
    for (int i = 0; i < 8; ++i)
        if (pos + i < ke) w |= static_cast<unsigned long long>(__ldg(a + i)) << (8 * i);
    return w;
}

// ------------------------------------------------------------------ K1: fold chains
// K1 body for logical CTA `bid` (the kernel below, and the fused single-pass k_filter_fused)
template <int D, int MODE>
__device__ __forceinline__ void k1_body(const KParams<D>& p, int bid, AsyncStage* st, FAgg<D>* wagg) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t c = static_cast<int64_t>(bid) * kThreads + threadIdx.x;
    const int64_t nch = static_cast<int64_t>(p.nb) * kThreads;
    const int64_t wbase = (static_cast<int64_t>(bid) * kThreads + wid * 32) * p.K;
    const int64_t kb = c * p.K;
    const int64_t ke = min(kb + p.K, p.n);

    FAgg<D> a;
    set_identity(a);
    double tprev = 0.0;
    // first step of the chain, peeled (the only place the global first element,
    // F = 0 / Q = P_inf (Eq. (7)), can occur)
    if (kb < ke) {
        if (kb > 0 || p.k0 > 0) tprev = __ldg(p.t + kb - 1);
        const double tk = __ldg(p.t + kb);
        const bool obs = __ldg(p.mask + kb) != 0;
        const double yk = obs ? __ldg(p.y + kb) : 0.0;
        const int64_t g = p.k0 + kb;
        FT_t<D, MODE> F;
        real Q[ns(D)];
        const double dt = tk - tprev;
        if (g == 0) {
set_zero(F);
#pragma unroll
            for (int i = 0; i < ns(D); ++i) Q[i] = p.m.Pinf[i];
        } else if (disc<D, MODE>(p.m, dt, F, Q)) {
            raise_error(p.err, g, kErrUnsupported);
        }
        if ((g > 0 && !(dt >= 0.0)) || !isfinite(tk) || (obs && !isfinite(yk))) raise_error(p.err, g, kErrInput);
        fold_step<D, MODE == kClosed>(a, F, Q, p.m, obs, yk);
        tprev = tk;
    }

    int ferr_u = -1, ferr_i = -1;
    const int64_t nwin = (p.K + kWinA - 1) / kWinA;
    issue_window(st[wid], 0, p.t, p.y, wbase, p.K, p.n, 0, lane);
    unsigned long long mnext = mask_word(p.mask, kb, ke);             // mask bytes of window 0
    unsigned long long mnext2 = mask_word(p.mask, kb + kWinA, ke);     // ... and of window 1 (2 ahead)
    for (int64_t w = 0; w < nwin; ++w) {
        const int64_t j0 = w * kWinA;
        const int buf = static_cast<int>(w & 1);
        if (w + 1 < nwin) issue_window(st[wid], buf ^ 1, p.t, p.y, wbase, p.K, p.n, j0 + kWinA, lane);
        else cp_async_commit();
        const unsigned long long mwin = mnext;
        mnext = mnext2;
        mnext2 = mask_word(p.mask, kb + j0 + 2 * kWinA, ke);
        cp_async_wait<1>();
        __syncwarp();
        const int jend = static_cast<int>(min(static_cast<int64_t>(kWinA), ke - (kb + j0)));
#pragma unroll kUnroll
        for (int jj = (w == 0) ? 1 : 0; jj < jend; ++jj) {
            const int jl = static_cast<int>(j0) + jj;          // step within the chain
            const double tk = st[wid].t[buf][jj][lane];
            const bool obs = ((mwin >> (8 * jj)) & 0xffull) != 0;
            const double yk = obs ? st[wid].y[buf][jj][lane] : 0.0;
            FT_t<D, MODE> F;
            real Q[ns(D)];
            const double dt = tk - tprev;
            const bool bad_u = disc<D, MODE>(p.m, dt, F, Q) != 0;
            const bool bad_i = !(dt >= 0.0) || !isfinite(tk) || (obs && !isfinite(yk));
            // first failing step of the chain, kept branch-free (reported after the loop)
            ferr_u = (bad_u && ferr_u < 0) ? jl : ferr_u;
            ferr_i = (bad_i && ferr_i < 0) ? jl : ferr_i;
            fold_step<D, MODE == kClosed>(a, F, Q, p.m, obs, yk);
            tprev = tk;
        }
        __syncwarp();
    }
    if (ferr_u >= 0) raise_error(p.err, p.k0 + kb + ferr_u, kErrUnsupported);
    if (ferr_i >= 0) raise_error(p.err, p.k0 + kb + ferr_i, kErrInput);
    store_soa(a, p.chain_f, nch, c);

    // CTA tree reduce (ordered): lane 0 of each warp, then warp 0
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        FAgg<D> o;
        shfl_down_all(o, a, off);
        if ((lane & (2 * off - 1)) == 0) {
            FAgg<D> r;
            if (!combine(a, o, r)) raise_error(p.err, p.k0 + kb, kErrNumeric);
            a = r;
        }
    }
    if (lane == 0) wagg[wid] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        FAgg<D> acc = wagg[0];
        bool ok = true;
#pragma unroll 1
        for (int w = 1; w < kWarps; ++w) {
            FAgg<D> r;
            ok = combine(acc, wagg[w], r) && ok;
            acc = r;
        }
        if (!ok) raise_error(p.err, p.k0 + kb, kErrNumeric);
        store_aos(acc, p.block_f + static_cast<int64_t>(bid) * FN(D));
    }
}

template <int D, int MODE>
__global__ void __launch_bounds__(kThreads, PSSGP_MINB) k_filter_reduce(const KParams<D> p) {
    __shared__ AsyncStage st[kWarps];
    __shared__ FAgg<D> wagg[kWarps];
    if (blockIdx.x == 0 && threadIdx.x == 0) { p.flag[0] = 0ull; p.flag[1] = 0ull; }   // K3 publication word, ticket
    k1_body<D, MODE>(p, blockIdx.x, st, wagg);
}

// ------------------------------------------------------------------ CTA-wide ordered reductions
// Ordered product blocks[lo] (x) ... (x) blocks[hi-1] of aggregates (AoS, NA
// reals each) by one CTA of kThreads: contiguous runs per thread, ordered
// warp trees, then the warp totals in order.  Result valid in thread 0.
// wred: shared scratch of kWarps aggregates.  Used by K3/K5 to build the
// collapsed carry entering the CTA from the block aggregates of all earlier
// (K3) / later (K5) CTAs: the block scan is thus spread over every SM instead
// of a separate single-CTA kernel.
template <typename Agg>
__device__ __forceinline__ Agg cta_reduce_range(const real* __restrict__ blocks, int lo, int hi, Agg* wred,
                                                bool* ok_out = nullptr) {
    constexpr int NA = sizeof(Agg) / sizeof(real);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int cnt = max(hi - lo, 0);
    const int per = (cnt + kThreads - 1) / kThreads;
    const int b0 = lo + min(static_cast<int>(threadIdx.x) * per, cnt), b1 = min(b0 + per, lo + cnt);
    Agg a;
    set_identity(a);
    bool ok = true;
    for (int b = b0; b < b1; ++b) {
        Agg e;
        load_aos(e, blocks + static_cast<int64_t>(b) * NA);
        if (b == b0) {
            a = e;
        } else {
            Agg r;
            ok = combine_chk(a, e, r) && ok;
            a = r;
        }
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        Agg o;
        shfl_down_all(o, a, off);
        if ((lane & (2 * off - 1)) == 0 && (threadIdx.x + off) * per < cnt) {
            Agg r;
            ok = combine_chk(a, o, r) && ok;
            a = r;
        }
    }
    if (lane == 0) wred[wid] = a;
    __syncthreads();
    Agg acc = wred[0];
    if (threadIdx.x == 0) {
        for (int w = 1; w < kWarps && w * 32 * per < cnt; ++w) {
            Agg r;
            ok = combine_chk(acc, wred[w], r) && ok;
            acc = r;
        }
    }
    if (ok_out) *ok_out = ok;
    __syncthreads();
    return acc;
}

// Deterministic fixed-order sum of parts[0, n) (element b at parts[b * stride]) by one CTA; result
// valid in thread 0.
__device__ __forceinline__ double cta_sum(const double* __restrict__ parts, int n, double* red, int stride = 1) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int per = (n + kThreads - 1) / kThreads;
    double s = 0.0;
    for (int i = 0; i < per; ++i) {
        const int b = threadIdx.x * per + i;
        if (b < n) s += parts[static_cast<int64_t>(b) * stride];
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
    if (lane == 0) red[wid] = s;
    __syncthreads();
    double tsum = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < kWarps; ++w) tsum += red[w];
    __syncthreads();
    return tsum;
}

// observation-row terms of a predicted (xm, Pm): HP = Pm H^T, S = H Pm H^T + r, hx = H xm
template <int D>
__device__ __forceinline__ void obs_terms(const ModelParams<D>& m, const real (&xm)[D], const real (&Pm)[ns(D)],
                                          real (&HP)[D], real& S, real& hx, bool hu_static = false) {
    if (hu_static || m.h_unit) {
#pragma unroll
        for (int i = 0; i < D; ++i) HP[i] = Pm[si(D, i, 0)];
        S = Pm[0] + m.r;
        hx = xm[0];
    } else {
        S = m.r; hx = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            real s2 = 0.0;
#pragma unroll
            for (int j = 0; j < D; ++j) s2 = fma(Pm[si(D, i, j)], m.H[j], s2);
            HP[i] = s2;
            hx = fma(m.H[i], xm[i], hx);
        }
#pragma unroll
        for (int i = 0; i < D; ++i) S = fma(m.H[i], HP[i], S);
    }
}

// NLL term 0.5 (log 2 pi S + v^2/S): v^2/S summed, S multiplied into a running
// product whose binary exponent is kept apart (one log per chain).
__device__ __forceinline__ void nll_accumulate(bool obs, double v, double vs, double S, double& quad, double& prodm,
                                               long long& prode, int& nobs) {
    quad = fma(v, vs, quad);
    prodm *= obs ? S : 1.0;
    long long bits = __double_as_longlong(prodm);
    prode += ((bits >> 52) & 0x7ff) - 1023;
    bits = (bits & ~(0x7ffLL << 52)) | (1023LL << 52);
    prodm = __longlong_as_double(bits);
    nobs += obs ? 1 : 0;
}

// Collapsed global prefix (xbar, P) entering chain c (the block scan spread over
// CTAs + the CTA's chain scan); shared scratch tot[kWarps], wcar[kWarps].
template <int D, bool FUSED = false>
__device__ __forceinline__ Gauss<D> filter_chain_carry(const KParams<D>& p, FAgg<D>* tot, Gauss<D>* wcar, int64_t c,
                                                       int64_t nch, int lane, int wid, int bid) {
    // ---- collapsed prefix entering this CTA.  Logical CTA 0 (the first to arrive, k3_ticket) alone
    // scans the block aggregates (an exclusive scan producing the collapsed carry (x, P) entering
    // every CTA, starting from the incoming carry of earlier ranks when sharded), writes them to
    // p.fcarry and publishes 1 in p.flag[0] (K1 of the same posterior reset it); the other CTAs run
    // their warps' chain scans below and then wait for the flag.  Logical CTA 0 waits on nobody and
    // has started before any CTA that waits, so the wait always ends.  One scan of depth ~15 in one
    // CTA replaces a redundant per-CTA reduction of all earlier blocks (~20 dependent operator
    // levels, throughput-bound across the wave).
    Gauss<D> cur;
    bool ok = true;
    if (bid == 0) {
        if (FUSED) {
            // single-pass kernel: every CTA of the (cooperative, co-resident) grid publishes its block
            // aggregate before counting itself in flag[2]; logical CTA 0 scans once all have
            if (threadIdx.x == 0)
                while (atomicAdd(p.flag + 2, 0ull) < static_cast<unsigned long long>(p.nb)) __nanosleep(32);
            __syncthreads();
            __threadfence();
        }
        const int per = (p.nb + kThreads - 1) / kThreads;
        const int b0 = min(static_cast<int>(threadIdx.x) * per, p.nb), b1 = min(b0 + per, p.nb);
        FAgg<D> a;
        set_identity(a);
        for (int b = b0; b < b1; ++b) {
            FAgg<D> e, r;
            if (FUSED) load_aos_cg(e, p.block_f + static_cast<int64_t>(b) * FN(D));   // written in this launch
            else load_aos(e, p.block_f + static_cast<int64_t>(b) * FN(D));
            ok = combine(a, e, r) && ok;
            a = r;
        }
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            FAgg<D> o;
            shfl_up_all(o, a, off);
            if (lane >= off) {
                FAgg<D> r;
                ok = combine(o, a, r) && ok;
                a = r;
            }
        }
        if (lane == 31) tot[wid] = a;
        FAgg<D> ex;
        shfl_up_all(ex, a, 1);
        __syncthreads();
        if (threadIdx.x == 0) {
            Gauss<D> R;
            set_zero(R);
            for (int g = 0; g < p.rank && p.in_filt; ++g) {
                FAgg<D> ag;
                load_aos(ag, p.in_filt + static_cast<int64_t>(g) * FN(D));
                Gauss<D> r2;
                ok = apply_prefix(R, ag, r2) && ok;
                R = r2;
            }
            for (int w = 0; w < kWarps; ++w) {
                wcar[w] = R;
                Gauss<D> r2;
                ok = apply_prefix(R, tot[w], r2) && ok;
                R = r2;
            }
        }
        __syncthreads();
        Gauss<D> C = wcar[wid];
        if (lane > 0) {
            Gauss<D> r2;
            ok = apply_prefix(C, ex, r2) && ok;
            C = r2;
        }
        for (int b = b0; b < b1; ++b) {
            store_aos(C, p.fcarry + static_cast<int64_t>(b) * CN(D));
            FAgg<D> e;
            if (FUSED) load_aos_cg(e, p.block_f + static_cast<int64_t>(b) * FN(D));
            else load_aos(e, p.block_f + static_cast<int64_t>(b) * FN(D));
            Gauss<D> r2;
            ok = apply_prefix(C, e, r2) && ok;
            C = r2;
        }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) atomicExch(p.flag, 1ull);
    }
    // ---- carry into this chain: CTA carry (x) exclusive scan of chain aggregates
    {
        FAgg<D> a;
        load_soa(a, p.chain_f, nch, c);
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            FAgg<D> o;
            shfl_up_all(o, a, off);
            if (lane >= off) {
                FAgg<D> r;
                ok = combine(o, a, r) && ok;
                a = r;
            }
        }
        FAgg<D> ex;
        shfl_up_all(ex, a, 1);
        __syncthreads();                        // CTA 0: its block scan is done with tot / wcar
        if (lane == 31) tot[wid] = a;
        __syncthreads();
        if (threadIdx.x == 0) {
            // wait for CTA 0's publication, then read this CTA's collapsed carry
            while (atomicAdd(p.flag, 0ull) == 0ull) __nanosleep(64);   // logical CTA 0 runs (k3_ticket)
            __threadfence();
            Gauss<D> acc;
            {   // L2 loads (the carry was written by another CTA in this launch)
                real* d = reinterpret_cast<real*>(&acc);
                const real* src = p.fcarry + static_cast<int64_t>(bid) * CN(D);
#pragma unroll
                for (int i = 0; i < CN(D); ++i) d[i] = __ldcg(src + i);
            }
            for (int w = 0; w < kWarps; ++w) {
                wcar[w] = acc;
                Gauss<D> r2;
                ok = apply_prefix(acc, tot[w], r2) && ok;
                acc = r2;
            }
        }
        __syncthreads();
        cur = wcar[wid];
        if (lane > 0) {
            Gauss<D> r2;
            ok = apply_prefix(cur, ex, r2) && ok;
            cur = r2;
        }
    }
    // a singular (I + C_i J_j) anywhere in the carry trees: latched at the CTA's first step
    if (!ok) raise_error(p.err, p.k0 + static_cast<int64_t>(bid) * kThreads * p.K, kErrNumeric);

    return cur;
}

// ------------------------------------------------------------------ K3: Kalman rescan
// STORE = false (NLL only): no filtered-state stores; SAGG = false: no smoother-aggregate
// moments / aggregates (NLL only, and the gradient's primal pass which needs only the stores).
template <int D, int MODE, bool STORE, bool SAGG, bool FUSED = false>
__device__ __forceinline__ void k3_body(const KParams<D>& p, int bid, AsyncStage* st, FAgg<D>* tot, Gauss<D>* wcar,
                                        SAgg<D>* stot, double* nred) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t c = static_cast<int64_t>(bid) * kThreads + threadIdx.x;
    const int64_t nch = static_cast<int64_t>(p.nb) * kThreads;
    const int64_t wg = static_cast<int64_t>(bid) * kWarps + wid;
    const int64_t wbase = wg * 32 * p.K;
    const int64_t kb = c * p.K;
    const int64_t ke = min(kb + p.K, p.n);

    const Gauss<D> cur = filter_chain_carry<D, FUSED>(p, tot, wcar, c, nch, lane, wid, bid);

    // ---- Kalman filter over the chain (supplement PAPER.md:285-315), carrying the
    // chain-entry moments E[x_k0 | y_1:k], Cov(x_k0 | y_1:k) and the cross-covariance
    // Cov(x_k0, x_k | y_1:k) for the chain's smoother aggregate.
    real x[D], P[ns(D)];
#pragma unroll
    for (int i = 0; i < D; ++i) x[i] = cur.x[i];
#pragma unroll
    for (int i = 0; i < ns(D); ++i) P[i] = cur.P[i];
    real x0[D], P0[ns(D)], Sg[D * D];
    double quad = 0.0, prodm = 1.0;
    long long prode = 0;
    int nobs = 0;
    double tprev = 0.0;
    // ---- first step of the chain (peeled: global first element, entry moments)
    if (kb < ke) {
        if (kb > 0 || p.k0 > 0) tprev = __ldg(p.t + kb - 1);
        const double tk = __ldg(p.t + kb);
        const bool obs = __ldg(p.mask + kb) != 0;
        const double yk = obs ? __ldg(p.y + kb) : 0.0;
        const int64_t g = p.k0 + kb;
        real xm[D], Pm[ns(D)];
        if (g == 0) {
#pragma unroll
            for (int i = 0; i < D; ++i) xm[i] = 0.0;
#pragma unroll
            for (int i = 0; i < ns(D); ++i) Pm[i] = p.m.Pinf[i];
        } else {
            FT_t<D, MODE> F;
            real Q[ns(D)];
            disc<D, MODE>(p.m, tk - tprev, F, Q);
            kf_predict_pm<D>(x, P, F, Q, xm, Pm);
        }
        tprev = tk;
        real HP[D], S, hx;
        obs_terms<D>(p.m, xm, Pm, HP, S, hx, MODE == kClosed);
        if (obs && !(S > 0.0 && S < INFINITY)) raise_error(p.err, g, kErrNumeric);
        const real iS = obs ? rcp(S) : 0.0;
        const real v = obs ? (static_cast<real>(yk) - hx) : real(0.0);
        const real vs = v * iS;
#pragma unroll
        for (int i = 0; i < D; ++i) x[i] = fma(HP[i], vs, xm[i]);
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = i; j < D; ++j) P[si(D, i, j)] = fma(-HP[i] * iS, HP[j], Pm[si(D, i, j)]);
#pragma unroll
        for (int i = 0; i < D; ++i) x0[i] = x[i];
#pragma unroll
        for (int i = 0; i < ns(D); ++i) P0[i] = P[i];
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) Sg[i * D + j] = P[si(D, i, j)];
        nll_accumulate(obs, v, vs, S, quad, prodm, prode, nobs);
        if (STORE) {
            real* o = p.xp + (wg * p.K * CN(D)) * 32 + lane;
            st_xP<D>(o, lane, x, P);
        }
    }

    int ferr_n = -1;
    const int64_t nwin = (p.K + kWinA - 1) / kWinA;
    issue_window(st[wid], 0, p.t, p.y, wbase, p.K, p.n, 0, lane);
    unsigned long long mnext = mask_word(p.mask, kb, ke);             // mask bytes of window 0
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
#pragma unroll kUnroll
        for (int jj = (w == 0) ? 1 : 0; jj < jend; ++jj) {
            const int64_t k = kb + j0 + jj;
            {
                const double tk = st[wid].t[buf][jj][lane];
                const bool obs = ((mwin >> (8 * jj)) & 0xffull) != 0;
                const double yk = obs ? st[wid].y[buf][jj][lane] : 0.0;
                FT_t<D, MODE> F;
                real xm[D], Pm[ns(D)], Q[ns(D)];
                disc<D, MODE>(p.m, tk - tprev, F, Q);
                kf_predict_pm<D>(x, P, F, Q, xm, Pm);
                tprev = tk;
                // observation update (branchless: missing y -> 1/S = 0, v = 0)
                real HP[D], S, hx;
                obs_terms<D>(p.m, xm, Pm, HP, S, hx, MODE == kClosed);
                const bool bad_n = obs && !(S > 0.0 && S < INFINITY);
                ferr_n = (bad_n && ferr_n < 0) ? static_cast<int>(k - kb) : ferr_n;
                const real iS = obs ? rcp(S) : 0.0;
                const real v = obs ? (static_cast<real>(yk) - hx) : real(0.0);
                const real vs = v * iS;
#pragma unroll
                for (int i = 0; i < D; ++i) x[i] = fma(HP[i], vs, xm[i]);
#pragma unroll
                for (int i = 0; i < D; ++i)
#pragma unroll
                    for (int j = i; j < D; ++j) P[si(D, i, j)] = fma(-HP[i] * iS, HP[j], Pm[si(D, i, j)]);
                // Sigma- = Sigma F^T, then the rank-one update by y_k of the
                // cross-covariance and of the chain-entry moments
                if (SAGG) {
                real Sm[D * D], SH[D];
                mul_bt<D>(Sg, F, Sm);
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    if (MODE == kClosed || p.m.h_unit) SH[i] = Sm[i * D];
                    else {
                        real s2 = 0.0;
#pragma unroll
                        for (int j = 0; j < D; ++j) s2 = fma(Sm[i * D + j], p.m.H[j], s2);
                        SH[i] = s2;
                    }
                }
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    const real si_ = SH[i] * iS;
#pragma unroll
                    for (int j = 0; j < D; ++j) Sg[i * D + j] = fma(-si_, HP[j], Sm[i * D + j]);
                    x0[i] = fma(SH[i], vs, x0[i]);
#pragma unroll
                    for (int j = i; j < D; ++j) P0[si(D, i, j)] = fma(-si_, SH[j], P0[si(D, i, j)]);
                }
                }
                nll_accumulate(obs, v, vs, S, quad, prodm, prode, nobs);
                if (STORE) {
                    real* o = p.xp + ((wg * p.K + (k - kb)) * CN(D)) * 32 + lane;
                    st_xP<D>(o, lane, x, P);
                }
            }
        }
        __syncwarp();
    }
    if (ferr_n >= 0) raise_error(p.err, p.k0 + kb + ferr_n, kErrNumeric);

    // ---- chain smoother aggregate
    if (SAGG) {
        SAgg<D> sag;
        set_identity(sag);
        if (ke > kb) {
            if (p.k0 + ke == p.nglob) {
                // chain ending with the terminal element (0, xbar_N, P_N): the entry
                // moments conditioned on all data are the smoothed moments -> (0, m^s_k0, P^s_k0)
#pragma unroll
                for (int i = 0; i < D * D; ++i) sag.E[i] = 0.0;
#pragma unroll
                for (int i = 0; i < D; ++i) sag.g[i] = x0[i];
#pragma unroll
                for (int i = 0; i < ns(D); ++i) sag.L[i] = P0[i];
            } else {
                // peek one step past the chain (prediction only)
                const int64_t g1 = p.k0 + ke;
                const double tn = __ldg(p.t + ke);
                FT_t<D, MODE> F;
                real Q[ns(D)], xm[D], Pm[ns(D)], Sm[D * D];
                disc<D, MODE>(p.m, tn - tprev, F, Q);
                kf_predict_pm<D>(x, P, F, Q, xm, Pm);
                mul_bt<D>(Sg, F, Sm);
                if (!chain_smoother_agg<D>(x0, P0, Sm, xm, Pm, sag)) raise_error(p.err, g1, kErrNumeric);
            }
        }
        store_soa(sag, p.chain_s, nch, c);
        // ordered CTA reduce of smoother aggregates -> block aggregate
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
    }

    // ---- NLL partial: 0.5 (sum v^2/S + log prod S + nobs log 2 pi)
    double nl = 0.0;
    if (nobs > 0) nl = 0.5 * (quad + log(prodm) + static_cast<double>(prode) * 0.6931471805599453 +
                              nobs * 1.8378770664093453);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) nl += __shfl_down_sync(0xffffffffu, nl, off);
    if (lane == 0) nred[wid] = nl;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s2 = 0.0;
        for (int w = 0; w < kWarps; ++w) s2 += nred[w];
        p.nll_block[bid] = s2;
        if (SAGG) {
            SAgg<D> acc = stot[0];
            for (int w = 1; w < kWarps; ++w) {
                SAgg<D> r;
                combine(acc, stot[w], r);
                acc = r;
            }
            store_aos(acc, p.block_s + static_cast<int64_t>(bid) * SN(D));
        }
    }
}

template <int D, int MODE, bool STORE = true, bool SAGG = STORE>
__global__ void __launch_bounds__(kThreads, PSSGP_MINB) k_filter_apply(const KParams<D> p) {
    __shared__ AsyncStage st[kWarps];
    __shared__ FAgg<D> tot[kWarps];
    __shared__ Gauss<D> wcar[kWarps];
    __shared__ SAgg<D> stot[kWarps];
    __shared__ double nred[kWarps];
    __shared__ int s_bid;
    const int bid = k3_ticket(p.flag, &s_bid);               // logical CTA index (arrival order)
    k3_body<D, MODE, STORE, SAGG>(p, bid, st, tot, wcar, stot, nred);
}

// ------------------------------------------------------------------ single-pass K1 + K3 (A/B variant)
// The fold and the Kalman rescan in ONE launch (north_star's single-pass scan): each CTA folds its
// chains and publishes its block aggregate (flag[2] counts them), logical CTA 0 scans all block
// aggregates once every CTA has published and publishes the collapsed carries (flag[0]), every CTA
// then rescans its chains - the inter-CTA exchange of the separate K1 / K3 launches done in place.
// A look-back in which CTA i combines the aggregates of its predecessors itself would serialise
// ~nb general operators (~1 us each at d = 3) on the last CTA, so the prefix scan stays with one CTA.
// Needs every CTA co-resident: launched cooperatively (the one-wave plan fits by construction).
template <int D, int MODE>
__global__ void __launch_bounds__(kThreads, PSSGP_MINB) k_filter_fused(const KParams<D> p) {
    __shared__ AsyncStage st[kWarps];
    __shared__ FAgg<D> tot[kWarps];
    __shared__ Gauss<D> wcar[kWarps];
    __shared__ SAgg<D> stot[kWarps];
    __shared__ double nred[kWarps];
    __shared__ int s_bid;
    const int bid = k3_ticket(p.flag, &s_bid);
    k1_body<D, MODE>(p, bid, st, tot);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(p.flag + 2, 1ull);                          // block aggregate published
    }
    k3_body<D, MODE, true, true, true>(p, bid, st, tot, wcar, stot, nred);
    k3_finish(p.flag, p.nb);
}

// Collapsed global suffix (m^s, P^s) after chain c (smoothed state at the first
// step of chain c+1); shared scratch tot[kWarps], wcar[kWarps + 1].
template <int D>
__device__ __forceinline__ Gauss<D> smoother_chain_carry(const KParams<D>& p, SAgg<D>* tot, Gauss<D>* wcar,
                                                         int64_t c, int64_t nch, int lane, int wid) {
    Gauss<D> res;
    // ---- collapsed suffix after this CTA: ordered product of the block aggregates of
    // CTAs blockIdx+1..nb-1 (x) incoming carry of later ranks (sharded)
    {
        const SAgg<D> after = cta_reduce_range<SAgg<D>>(p.block_s, blockIdx.x + 1, p.nb, tot);
        if (threadIdx.x == 0) {
            Gauss<D> R;
            set_zero(R);
            for (int g = p.world - 1; g > p.rank && p.in_smooth; --g) {
                SAgg<D> ag;
                load_aos(ag, p.in_smooth + static_cast<int64_t>(g) * (SN(D) + 1));   // blob = aggregate + NLL partial
                Gauss<D> r2;
                apply_suffix(ag, R, r2);
                R = r2;
            }
            if (blockIdx.x + 1 < p.nb) {
                Gauss<D> r2;
                apply_suffix(after, R, r2);
                R = r2;
            }
            wcar[kWarps] = R;
        }
        __syncthreads();
    }
    {
        SAgg<D> a;
        load_soa(a, p.chain_s, nch, c);
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            SAgg<D> o;
            shfl_down_all(o, a, off);
            if (lane + off < 32) {
                SAgg<D> r;
                combine(a, o, r);
                a = r;
            }
        }
        if (lane == 0) tot[wid] = a;
        SAgg<D> ex;
        shfl_down_all(ex, a, 1);
        __syncthreads();
        if (threadIdx.x == 0) {
            Gauss<D> acc = wcar[kWarps];
            for (int w = kWarps - 1; w >= 0; --w) {
                wcar[w + 1] = acc;
                Gauss<D> r2;
                apply_suffix(tot[w], acc, r2);
                acc = r2;
            }
        }
        __syncthreads();
        Gauss<D> cur = wcar[wid + 1];
        if (lane < 31) {
            Gauss<D> r2;
            apply_suffix(ex, cur, r2);
            cur = r2;
        }
        res = cur;
    }

    return res;
}

// L2 prefetch of a warp's filtered state at chain-relative step kp: the 32 chains' (xbar, P) of
// one step are one contiguous run of CN * 32 reals in the [warp][K][CN][32] layout, fetched as one
// 128-byte line per lane into L2 (no registers held, unlike a deeper register prefetch).
template <int D>
__device__ __forceinline__ void prefetch_state_l2(const real* xpw, int lane, int64_t kp) {
    constexpr int kLines = (CN(D) * 32 * static_cast<int>(sizeof(real)) + 127) / 128;
    if (lane < kLines) {
        const char* a = reinterpret_cast<const char*>(xpw - lane + (kp * CN(D)) * 32) + lane * 128;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
    }
}

// ------------------------------------------------------------------ K5: RTS rescan
// f-space projection: mean = H m^s, var = H P^s H^T
template <int D>
__device__ __forceinline__ void project(const ModelParams<D>& m, const real (&ms)[D], const real (&Ps)[ns(D)],
                                        real& mo, real& vo, bool hu_static = false) {
    if (hu_static || m.h_unit) {
        mo = ms[0];
        vo = Ps[0];
    } else {
        mo = 0.0; vo = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            mo = fma(m.H[i], ms[i], mo);
            real s2 = 0.0;
#pragma unroll
            for (int j = 0; j < D; ++j) s2 = fma(Ps[si(D, i, j)], m.H[j], s2);
            vo = fma(m.H[i], s2, vo);
        }
    }
}

struct StageOut {
    double t[2][kWinA][33];   // double-buffered t, transposed [step][chain]
    double m[kWinA][33];      // mean of the current window, transposed
    double v[kWinA][33];      // variance
};

template <int D, int MODE>
__global__ void __launch_bounds__(kThreads, PSSGP_MINB) k_smoother_apply(const KParams<D> p) {
    __shared__ StageOut so[kWarps];
    __shared__ __align__(8) SAgg<D> tot[kWarps];   // also the NLL sum scratch (doubles)
    __shared__ Gauss<D> wcar[kWarps + 1];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t c = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
    const int64_t nch = static_cast<int64_t>(p.nb) * kThreads;
    const int64_t wg = static_cast<int64_t>(blockIdx.x) * kWarps + wid;
    const int64_t wbase = wg * 32 * p.K;
    const int64_t kb = c * p.K;
    const int64_t ke = min(kb + p.K, p.n);

    // ---- NLL: fixed-order sum of the per-CTA partials written by K3 (CTA 0 only)
    if (blockIdx.x == 0 && p.nll_out) {
        const double v = cta_sum(p.nll_block, p.nb, reinterpret_cast<double*>(tot));
        if (threadIdx.x == 0) *p.nll_out = v;
    }
    real ms[D], Ps[ns(D)];
    {
        const Gauss<D> cur = smoother_chain_carry<D>(p, tot, wcar, c, nch, lane, wid);
#pragma unroll
        for (int i = 0; i < D; ++i) ms[i] = cur.x[i];
#pragma unroll
        for (int i = 0; i < ns(D); ++i) Ps[i] = cur.P[i];
    }

    // ---- RTS over the chain, last step first; the filtered
    // (xbar, P) of the next step down is prefetched one step ahead.
    const real* xpw = p.xp + (wg * p.K * CN(D)) * 32 + lane;
    real nx[CN(D)];
    double tnext = 0.0;
    // last step of the chain, peeled (the only place the terminal element can occur);
    // its outputs are stored directly (one scalar store per chain)
    if (ke > kb) {
        const int64_t k = ke - 1;
        const real* src = xpw + ((k - kb) * CN(D)) * 32;
        real x[D], P[ns(D)];
        ld_xP<D>(src, lane, x, P);
        if (k > kb) {
            const real* s1 = xpw + ((k - 1 - kb) * CN(D)) * 32;
            ld_state<D>(s1, lane, nx);
        }
        const double tk = __ldg(p.t + k);
        if (p.k0 + k == p.nglob - 1) {
#pragma unroll
            for (int i = 0; i < D; ++i) ms[i] = x[i];
#pragma unroll
            for (int i = 0; i < ns(D); ++i) Ps[i] = P[i];
        } else {
            const double tn = __ldg(p.t + ke);
            FT_t<D, MODE> F;
            real Q[ns(D)], xm[D], Pm[ns(D)], FP[D * D];
            disc<D, MODE>(p.m, tn - tk, F, Q);
            kf_predict<D>(x, P, F, Q, xm, FP, Pm);
            if (!rts_step<D>(x, P, xm, Pm, FP, ms, Ps)) raise_error(p.err, p.k0 + k, kErrNumeric);
        }
        tnext = tk;
        real mo, vo;
        project<D>(p.m, ms, Ps, mo, vo, MODE == kClosed);
        if (p.mean) p.mean[k] = mo;
        if (p.var) p.var[k] = vo;
    }
    int ferr_n = -1;
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
        const int jstart = static_cast<int>(min(static_cast<int64_t>(kWinA - 1), ke - 2 - (kb + j0)));
#pragma unroll kUnroll
        for (int jj = jstart; jj >= 0; --jj) {
            const int64_t k = kb + j0 + jj;
            {
                const double tk = so[wid].t[buf][jj][lane];
                real x[D], P[ns(D)];
#pragma unroll
                for (int i = 0; i < D; ++i) x[i] = nx[i];
#pragma unroll
                for (int i = 0; i < ns(D); ++i) P[i] = nx[D + i];
                if (k > kb) {
                    const real* src = xpw + ((k - 1 - kb) * CN(D)) * 32;
                    ld_state<D>(src, lane, nx);
                }
                if (PSSGP_K5_PF > 0 && k - PSSGP_K5_PF >= kb) prefetch_state_l2<D>(xpw, lane, k - PSSGP_K5_PF - kb);
                FT_t<D, MODE> F;
            real Q[ns(D)], xm[D], Pm[ns(D)], FP[D * D];
                disc<D, MODE>(p.m, tnext - tk, F, Q);
                kf_predict<D>(x, P, F, Q, xm, FP, Pm);
                const bool bad_n = !rts_step<D>(x, P, xm, Pm, FP, ms, Ps);
                ferr_n = bad_n ? static_cast<int>(k - kb) : ferr_n;   // backward: last hit = first index
                tnext = tk;
                real mo, vo;
                project<D>(p.m, ms, Ps, mo, vo, MODE == kClosed);
                so[wid].m[jj][lane] = mo;
                so[wid].v[jj][lane] = vo;
            }
        }
        __syncwarp();
        {
            const int col = lane & (kWinA - 1), rb = lane / kWinA;
            const int64_t j = j0 + col;
#pragma unroll
            for (int i = 0; i < 32 / (32 / kWinA); ++i) {
                const int r = rb + (32 / kWinA) * i;
                const int64_t idx = wbase + r * p.K + j;
                const int64_t last = min(wbase + (r + 1) * p.K, p.n) - 1;   // row r's peeled step
                if ((j < p.K) && (idx < last)) {
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
    if (ferr_n >= 0) raise_error(p.err, p.k0 + kb + ferr_n, kErrNumeric);
}

#ifndef PSSGP_NO_MISC_KERNELS
// ------------------------------------------------------------------ K6: deterministic NLL sum
// The same fixed-order CTA sum (cta_sum, kThreads threads) as K5's CTA 0 uses, so the NLL-only
// path returns bit-for-bit the NLL of the full posterior.  Launch <<<1, kThreads>>>.  stride > 1:
// the partials are spread over gathered per-rank blobs (sharded total NLL).
__global__ void __launch_bounds__(kThreads, 1) k_nll_sum(const double* __restrict__ parts, int nb, double* out,
                                                         int stride) {
    __shared__ double red[kWarps];
    const double v = cta_sum(parts, nb, red, stride);
    if (threadIdx.x == 0) *out = v;
}
#endif

// ------------------------------------------------------------------ chunk aggregate reducers (sharded path, 1 CTA)
template <int D, typename Agg>
__global__ void __launch_bounds__(kCarryThreads, 1) k_reduce_blocks(const real* __restrict__ blocks, int nb,
                                                                    real* out, unsigned long long* err,
                                                                    int64_t err_index) {
    constexpr int NW = kCarryThreads / 32;
    constexpr int NA = sizeof(Agg) / sizeof(real);
    __shared__ Agg wred[NW];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int per = (nb + kCarryThreads - 1) / kCarryThreads;
    Agg a;
    set_identity(a);
    bool ok = true;
    for (int i = 0; i < per; ++i) {
        const int b = threadIdx.x * per + i;
        if (b < nb) {
            Agg e, r;
            load_aos(e, blocks + static_cast<int64_t>(b) * NA);
            ok = combine_chk(a, e, r) && ok;
            a = r;
        }
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        Agg o;
        shfl_down_all(o, a, off);
        if ((lane & (2 * off - 1)) == 0) {
            Agg r;
            ok = combine_chk(a, o, r) && ok;
            a = r;
        }
    }
    if (lane == 0) wred[wid] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        Agg acc = wred[0];
        for (int w = 1; w < NW; ++w) {
            Agg r;
            ok = combine_chk(acc, wred[w], r) && ok;
            acc = r;
        }
        store_aos(acc, out);
    }
    if (!ok && err) raise_error(err, err_index, kErrNumeric);
}

}  // namespace PSSGP_NS

#ifndef PSSGP_NO_MISC_KERNELS
namespace PSSGP_NS {
// ------------------------------------------------------------------ test-time merge (stage 4)
// Rank-based parallel merge of sorted training times (observed) and sorted test
// times (missing): a training time goes to i + #{test < t_i}, a test time to
// j + #{train <= s_j} (training first on ties, reading Z12), each rank by binary
// search — span O(log(N + M)), work O((N + M) log).  Unsorted input -> error.
__device__ __forceinline__ int64_t count_less(const double* __restrict__ a, int64_t n, double v, bool or_equal) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        const double x = __ldg(a + mid);
        if (or_equal ? (x <= v) : (x < v)) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(256) k_merge(int64_t n_tr, const double* __restrict__ t_tr,
                                               const double* __restrict__ y_tr, int64_t n_te,
                                               const double* __restrict__ t_te, double* __restrict__ t_out,
                                               double* __restrict__ y_out, uint8_t* __restrict__ m_out,
                                               int64_t* __restrict__ test_index, unsigned long long* err) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n_tr) {
        const double v = __ldg(t_tr + i);
        if (!isfinite(v) || (i > 0 && !(__ldg(t_tr + i - 1) <= v))) raise_error(err, i, kErrInput);
        const int64_t dst = i + count_less(t_te, n_te, v, false);
        t_out[dst] = v;
        y_out[dst] = __ldg(y_tr + i);
        m_out[dst] = 1;
    } else if (i < n_tr + n_te) {
        const int64_t j = i - n_tr;
        const double v = __ldg(t_te + j);
        if (!isfinite(v) || (j > 0 && !(__ldg(t_te + j - 1) <= v))) raise_error(err, n_tr + j, kErrInput);
        const int64_t dst = j + count_less(t_tr, n_tr, v, true);
        t_out[dst] = v;
        y_out[dst] = 0.0;
        m_out[dst] = 0;
        test_index[j] = dst;
    }
}

__global__ void __launch_bounds__(256) k_gather(int64_t n_te, const int64_t* __restrict__ test_index,
                                                const double* __restrict__ mean, const double* __restrict__ var,
                                                double* __restrict__ mean_te, double* __restrict__ var_te) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < n_te) {
        const int64_t k = __ldg(test_index + j);
        if (mean_te) mean_te[j] = __ldg(mean + k);
        if (var_te) var_te[j] = __ldg(var + k);
    }
}
}  // namespace PSSGP_NS
#endif  // PSSGP_NO_MISC_KERNELS
