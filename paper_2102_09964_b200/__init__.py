"""B200-native parallel state-space GP (PSSGP) hot path — Python binding.

Thin marshalling layer over the C ABI in include/pssgp.h (libpssgp.so, CUDA
kernels for sm_100a).  Functions keep the C names; `Model` is a convenience
wrapper.  PyTorch is used only for device memory and streams.  There is no
CPU fallback: importing the compute functions without the built library
raises ImportError.

Paper: Corenflos, Zhao & Sarkka, "Temporal Gaussian Process Regression in
Logarithmic Time" (arXiv:2102.09964) — filter elements with missing
measurements (Eqs. (6)-(8)), filtering operator, parallel
RTS smoother (supplement Prop. 2), NLL.
"""
from __future__ import annotations

import ctypes
from typing import Iterable, Optional, Sequence

import numpy as np

from ._native import (KINDS, STATUS_NAMES, Component, Options, PssgpError, build, lib)  # noqa: F401

__all__ = ["Model", "PssgpError", "build", "lib", "pssgp_create", "pssgp_destroy", "pssgp_posterior",
           "pssgp_nll", "pssgp_nll_grad", "pssgp_posterior_host_async", "pssgp_sync", "pssgp_posterior_host", "pssgp_check", "pssgp_error_index", "pssgp_last_error",
           "pssgp_state_dim", "pssgp_get_ssm", "pssgp_debug_discretize", "pssgp_plan",
           "pssgp_aggregate_bytes", "pssgp_shard_filter_reduce", "pssgp_shard_filter_apply",
           "pssgp_shard_smoother_apply", "pssgp_profile_enable", "pssgp_profile_read", "pssgp_profile_name",
           "pssgp_merge_grid", "pssgp_gather", "pssgp_predict", "pssgp_posterior_batched", "pssgp_nll_grad_batched",
           "pssgp_posterior_f32", "pssgp_plan_f32", "pssgp_measure_fp64_peak", "pssgp_num_params",
           "pssgp_posterior_batched_theta", "pssgp_nll_grad_batched_theta"]


def _ptr(x) -> Optional[int]:
    """Device pointer of a torch tensor (or None)."""
    if x is None:
        return None
    return int(x.data_ptr())


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        import torch
        return int(torch.cuda.current_stream().cuda_stream) or None
    if isinstance(stream, int):
        return stream or None
    return int(stream.cuda_stream) or None


def _raise(handle, st: int):
    if st != 0:
        msg = lib().pssgp_last_error(handle).decode() if handle else ""
        idx = lib().pssgp_error_index(handle) if handle else -1
        raise PssgpError(st, msg, idx)


# ------------------------------------------------------------------------- C-named thin wrappers
def pssgp_create(components: Sequence, noise_var: float, uniform_dt: float = 0.0, balance: bool = True,
                 chain_len: int = 0, blocks_per_sm: int = 0, device: int = -1) -> int:
    """components: objects with .kind ('matern52', ...), .variance, .lengthscale, .period, .order."""
    n = len(components)
    arr = (Component * n)()
    for i, c in enumerate(components):
        kind = KINDS[c.kind] if isinstance(c.kind, str) else int(c.kind)
        arr[i] = Component(kind, float(c.variance), float(c.lengthscale), float(getattr(c, "period", 1.0)),
                           int(getattr(c, "order", 0)), float(getattr(c, "mat_lengthscale", 1.0)),
                           int(getattr(c, "mat_nu2", 3)))
    opt = Options(1 if balance else 0, int(device), float(uniform_dt), int(chain_len), int(blocks_per_sm))
    h = ctypes.c_void_p()
    st = lib().pssgp_create(arr, n, float(noise_var), ctypes.byref(opt), ctypes.byref(h))
    if st != 0:
        raise PssgpError(st, "pssgp_create failed")
    return h.value


def pssgp_destroy(h: int) -> None:
    lib().pssgp_destroy(h)


def pssgp_state_dim(h: int) -> int:
    return lib().pssgp_state_dim(h)


def pssgp_posterior(h, N, t, y, mask, mean, var, nll, stream=None) -> None:
    _raise(h, lib().pssgp_posterior(h, int(N), _ptr(t), _ptr(y), _ptr(mask), _ptr(mean), _ptr(var), _ptr(nll),
                                    _stream_ptr(stream)))


def pssgp_posterior_f32(h, N, t, y, mask, mean, var, nll, stream=None) -> None:
    _raise(h, lib().pssgp_posterior_f32(h, int(N), _ptr(t), _ptr(y), _ptr(mask), _ptr(mean), _ptr(var),
                                        _ptr(nll), _stream_ptr(stream)))


def pssgp_nll(h, N, t, y, mask, nll, stream=None) -> None:
    _raise(h, lib().pssgp_nll(h, int(N), _ptr(t), _ptr(y), _ptr(mask), _ptr(nll), _stream_ptr(stream)))


def pssgp_nll_grad(h, N, t, y, mask, nll, grad, stream=None) -> None:
    _raise(h, lib().pssgp_nll_grad(h, int(N), _ptr(t), _ptr(y), _ptr(mask), _ptr(nll), _ptr(grad),
                                   _stream_ptr(stream)))


def pssgp_posterior_host(h, N, t: np.ndarray, y: np.ndarray, mask: np.ndarray, mean: Optional[np.ndarray],
                         var: Optional[np.ndarray], nll: Optional[np.ndarray], stream=None) -> None:
    """Host (numpy / pinned torch CPU) arrays; synchronous."""
    def hp(a):
        if a is None:
            return None
        if hasattr(a, "data_ptr"):
            return int(a.data_ptr())
        return a.ctypes.data
    _raise(h, lib().pssgp_posterior_host(h, int(N), hp(t), hp(y), hp(mask), hp(mean), hp(var), hp(nll),
                                         _stream_ptr(stream)))


def pssgp_posterior_host_async(h, N, t, y, mask, mean, var, nll) -> None:
    """Pinned host arrays (torch pin_memory tensors or page-locked numpy); returns immediately."""
    def hp(a):
        if a is None:
            return None
        if hasattr(a, "data_ptr"):
            return int(a.data_ptr())
        return a.ctypes.data
    _raise(h, lib().pssgp_posterior_host_async(h, int(N), hp(t), hp(y), hp(mask), hp(mean), hp(var), hp(nll)))


def pssgp_sync(h) -> None:
    _raise(h, lib().pssgp_sync(h))


def pssgp_merge_grid(h, n_train, t_train, y_train, n_test, t_test, t_out, y_out, mask_out, test_index,
                     stream=None) -> None:
    _raise(h, lib().pssgp_merge_grid(h, int(n_train), _ptr(t_train), _ptr(y_train), int(n_test), _ptr(t_test),
                                     _ptr(t_out), _ptr(y_out), _ptr(mask_out), _ptr(test_index), _stream_ptr(stream)))


def pssgp_gather(h, n_test, test_index, mean, var, mean_test, var_test, stream=None) -> None:
    _raise(h, lib().pssgp_gather(h, int(n_test), _ptr(test_index), _ptr(mean), _ptr(var), _ptr(mean_test),
                                 _ptr(var_test), _stream_ptr(stream)))


def pssgp_predict(h, n_train, t_train, y_train, n_test, t_test, mean_test, var_test, nll, stream=None) -> None:
    _raise(h, lib().pssgp_predict(h, int(n_train), _ptr(t_train), _ptr(y_train), int(n_test), _ptr(t_test),
                                  _ptr(mean_test), _ptr(var_test), _ptr(nll), _stream_ptr(stream)))


def pssgp_posterior_batched(h, nseg, offsets, variance, lengthscale, noise_var, N, t, y, mask, mean, var, nll,
                            stream=None) -> None:
    _raise(h, lib().pssgp_posterior_batched(h, int(nseg), _ptr(offsets), _ptr(variance), _ptr(lengthscale),
                                            _ptr(noise_var), int(N), _ptr(t), _ptr(y), _ptr(mask), _ptr(mean),
                                            _ptr(var), _ptr(nll), _stream_ptr(stream)))


def pssgp_nll_grad_batched(h, nseg, offsets, variance, lengthscale, noise_var, N, t, y, mask, nll, grad,
                           stream=None) -> None:
    _raise(h, lib().pssgp_nll_grad_batched(h, int(nseg), _ptr(offsets), _ptr(variance), _ptr(lengthscale),
                                           _ptr(noise_var), int(N), _ptr(t), _ptr(y), _ptr(mask), _ptr(nll),
                                           _ptr(grad), _stream_ptr(stream)))


def pssgp_check(h) -> None:
    _raise(h, lib().pssgp_check(h))


def pssgp_error_index(h) -> int:
    return lib().pssgp_error_index(h)


def pssgp_last_error(h) -> str:
    return lib().pssgp_last_error(h).decode()


def pssgp_get_ssm(h):
    d = pssgp_state_dim(h)
    G = np.zeros((d, d)); W = np.zeros((d, d)); P = np.zeros((d, d)); H = np.zeros(d); D = np.zeros(d)
    dp = ctypes.POINTER(ctypes.c_double)
    _raise(h, lib().pssgp_get_ssm(h, G.ctypes.data_as(dp), W.ctypes.data_as(dp), H.ctypes.data_as(dp),
                                  P.ctypes.data_as(dp), D.ctypes.data_as(dp)))
    return dict(G=G, W=W, H=H, Pinf=P, D=D)


def pssgp_debug_discretize(h, dt: float):
    d = pssgp_state_dim(h)
    F = np.zeros((d, d)); Q = np.zeros((d, d))
    dp = ctypes.POINTER(ctypes.c_double)
    _raise(h, lib().pssgp_debug_discretize(h, float(dt), F.ctypes.data_as(dp), Q.ctypes.data_as(dp)))
    return F, Q


def pssgp_plan(h, N: int):
    K = ctypes.c_int64(); nch = ctypes.c_int64(); nb = ctypes.c_int(); thr = ctypes.c_int()
    _raise(h, lib().pssgp_plan(h, int(N), ctypes.byref(K), ctypes.byref(nch), ctypes.byref(nb), ctypes.byref(thr)))
    return dict(chain_len=K.value, n_chains=nch.value, n_blocks=nb.value, threads=thr.value)


def pssgp_plan_f32(h, N: int):
    K = ctypes.c_int64(); nch = ctypes.c_int64(); nb = ctypes.c_int(); thr = ctypes.c_int()
    _raise(h, lib().pssgp_plan_f32(h, int(N), ctypes.byref(K), ctypes.byref(nch), ctypes.byref(nb),
                                   ctypes.byref(thr)))
    return dict(chain_len=K.value, n_chains=nch.value, n_blocks=nb.value, threads=thr.value)


def pssgp_profile_enable(h, on: bool = True) -> None:
    lib().pssgp_profile_enable(h, 1 if on else 0)


def pssgp_profile_name(slot: int) -> str:
    return lib().pssgp_profile_name(slot).decode()


def pssgp_profile_read(h):
    ms = (ctypes.c_double * 16)()
    cnt = (ctypes.c_int64 * 16)()
    n = lib().pssgp_profile_read(h, ms, cnt, 16)
    return {pssgp_profile_name(i): (ms[i], cnt[i]) for i in range(n)}


def pssgp_aggregate_bytes(h, which: int) -> int:
    return int(lib().pssgp_aggregate_bytes(h, int(which)))


def pssgp_shard_filter_reduce(h, k0, n, N_global, t_ptr, y_ptr, mask_ptr, out_ptr, stream=None) -> None:
    _raise(h, lib().pssgp_shard_filter_reduce(h, int(k0), int(n), int(N_global), t_ptr, y_ptr, mask_ptr, out_ptr,
                                              _stream_ptr(stream)))


def pssgp_shard_filter_apply(h, k0, n, N_global, t_ptr, y_ptr, mask_ptr, all_ptr, rank, world, sout_ptr, nll_ptr,
                             stream=None) -> None:
    _raise(h, lib().pssgp_shard_filter_apply(h, int(k0), int(n), int(N_global), t_ptr, y_ptr, mask_ptr, all_ptr,
                                             int(rank), int(world), sout_ptr, nll_ptr, _stream_ptr(stream)))


def pssgp_shard_smoother_apply(h, k0, n, N_global, t_ptr, all_ptr, rank, world, mean_ptr, var_ptr, nll_ptr=None,
                               stream=None) -> None:
    _raise(h, lib().pssgp_shard_smoother_apply(h, int(k0), int(n), int(N_global), t_ptr, all_ptr, int(rank),
                                               int(world), mean_ptr, var_ptr, nll_ptr, _stream_ptr(stream)))


def pssgp_posterior_batched_theta(h, nseg, offsets, theta, N, t, y, mask, mean, var, nll, stream=None) -> None:
    _raise(h, lib().pssgp_posterior_batched_theta(h, int(nseg), _ptr(offsets), _ptr(theta), int(N), _ptr(t), _ptr(y),
                                                  _ptr(mask), _ptr(mean), _ptr(var), _ptr(nll), _stream_ptr(stream)))


def pssgp_nll_grad_batched_theta(h, nseg, offsets, theta, N, t, y, mask, nll, grad, stream=None) -> None:
    _raise(h, lib().pssgp_nll_grad_batched_theta(h, int(nseg), _ptr(offsets), _ptr(theta), int(N), _ptr(t), _ptr(y),
                                                 _ptr(mask), _ptr(nll), _ptr(grad), _stream_ptr(stream)))


def pssgp_num_params(h) -> int:
    """Number of log hyper-parameters (length of the pssgp_nll_grad gradient)."""
    return int(lib().pssgp_num_params(h))


def pssgp_measure_fp64_peak(h) -> float:
    """DFMA throughput of the handle's device in TFLOP/s (the fp64 roofline denominator)."""
    out = ctypes.c_double(0.0)
    _raise(h, lib().pssgp_measure_fp64_peak(h, ctypes.byref(out)))
    return out.value


# ------------------------------------------------------------------------- convenience wrapper
class Model:
    """Owns one pssgp_model handle.

    >>> m = Model([synth.Component('matern52', 1.0, 0.5)], noise_var=0.01)
    >>> mean, var, nll = m.posterior(t, y, mask)        # torch cuda tensors
    """

    def __init__(self, components: Iterable, noise_var: float, **kw):
        self.components = list(components)
        self.noise_var = float(noise_var)
        self.h = pssgp_create(self.components, noise_var, **kw)

    def close(self):
        if getattr(self, "h", None):
            pssgp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def state_dim(self) -> int:
        return pssgp_state_dim(self.h)

    def posterior(self, t, y, mask, out=None, stream=None, with_nll: bool = True):
        import torch
        N = int(t.shape[0])
        if out is None:
            mean = torch.empty(N, dtype=torch.float64, device=t.device)
            var = torch.empty_like(mean)
            nll = torch.zeros(1, dtype=torch.float64, device=t.device) if with_nll else None
        else:
            mean, var, nll = out
        pssgp_posterior(self.h, N, t, y, mask, mean, var, nll, stream)
        return mean, var, nll

    def posterior_f32(self, t, y, mask, out=None, stream=None, with_nll: bool = True):
        """The optional fp32-state path (single Matern components): same outputs as posterior()."""
        import torch
        N = int(t.shape[0])
        if out is None:
            mean = torch.empty(N, dtype=torch.float64, device=t.device)
            var = torch.empty_like(mean)
            nll = torch.zeros(1, dtype=torch.float64, device=t.device) if with_nll else None
        else:
            mean, var, nll = out
        pssgp_posterior_f32(self.h, N, t, y, mask, mean, var, nll, stream)
        return mean, var, nll

    def nll(self, t, y, mask, out=None, stream=None):
        import torch
        N = int(t.shape[0])
        nll = out if out is not None else torch.zeros(1, dtype=torch.float64, device=t.device)
        pssgp_nll(self.h, N, t, y, mask, nll, stream)
        return nll

    @property
    def num_params(self) -> int:
        return pssgp_num_params(self.h)

    def nll_grad(self, t, y, mask, stream=None):
        """(nll[1], grad[num_params]): d NLL / d log hyper-parameters in the order of
        include/pssgp.h (per component: log variance, log lengthscale[, log period[, log Matern
        lengthscale]]; then log noise variance)."""
        import torch
        N = int(t.shape[0])
        nll = torch.zeros(1, dtype=torch.float64, device=t.device)
        grad = torch.zeros(self.num_params, dtype=torch.float64, device=t.device)
        pssgp_nll_grad(self.h, N, t, y, mask, nll, grad, stream)
        return nll, grad

    @property
    def theta(self) -> np.ndarray:
        """The model's own log hyper-parameters in the order of nll_grad (host array)."""
        th = []
        for c in self.components:
            th += [np.log(c.variance), np.log(c.lengthscale)]
            if c.kind in ("periodic", "quasiperiodic"):
                th.append(np.log(c.period))
            if c.kind == "quasiperiodic":
                th.append(np.log(c.mat_lengthscale))
        return np.array(th + [np.log(self.noise_var)], dtype=np.float64)

    def nll_grad_batched_theta(self, offsets, theta, t, y, mask, stream=None):
        """Series b = [offsets[b], offsets[b+1]) with its own log hyper-parameters theta[b]
        (device [B, num_params]): (nll[B], grad[B, num_params])."""
        import torch
        B = int(offsets.shape[0]) - 1
        nll = torch.zeros(B, dtype=torch.float64, device=t.device)
        grad = torch.zeros((B, self.num_params), dtype=torch.float64, device=t.device)
        pssgp_nll_grad_batched_theta(self.h, B, offsets, theta, int(t.shape[0]), t, y, mask, nll, grad, stream)
        return nll, grad

    def posterior_batched_theta(self, offsets, theta, t, y, mask, stream=None):
        """(mean[N], var[N], nll[B]) of B series, each at its own log hyper-parameters theta[b]."""
        import torch
        B, N = int(offsets.shape[0]) - 1, int(t.shape[0])
        mean = torch.empty(N, dtype=torch.float64, device=t.device)
        var = torch.empty_like(mean)
        nll = torch.zeros(B, dtype=torch.float64, device=t.device)
        pssgp_posterior_batched_theta(self.h, B, offsets, theta, N, t, y, mask, mean, var, nll, stream)
        return mean, var, nll

    def posterior_host(self, t: np.ndarray, y: np.ndarray, mask: np.ndarray, mean=None, var=None, nll=None):
        N = int(t.shape[0])
        mean = np.empty(N) if mean is None else mean
        var = np.empty(N) if var is None else var
        nll = np.zeros(1) if nll is None else nll
        pssgp_posterior_host(self.h, N, t, y, mask, mean, var, nll)
        return mean, var, nll

    def predict(self, t_train, y_train, t_test, stream=None):
        """Merge test times (missing observations) into the training grid on the
        device, run filter + smoother + NLL, return (mean_test, var_test, nll)."""
        import torch
        mt = torch.empty(int(t_test.shape[0]), dtype=torch.float64, device=t_train.device)
        vt = torch.empty_like(mt)
        nll = torch.zeros(1, dtype=torch.float64, device=t_train.device)
        pssgp_predict(self.h, int(t_train.shape[0]), t_train, y_train, int(t_test.shape[0]), t_test, mt, vt, nll,
                      stream)
        return mt, vt, nll

    def check(self):
        pssgp_check(self.h)

    def ssm(self):
        return pssgp_get_ssm(self.h)

    def discretize(self, dt: float):
        return pssgp_debug_discretize(self.h, dt)

    def plan(self, N: int, f32: bool = False):
        return pssgp_plan_f32(self.h, N) if f32 else pssgp_plan(self.h, N)
