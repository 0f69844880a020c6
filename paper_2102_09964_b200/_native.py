"""ctypes binding of libpssgp.so (include/pssgp.h): argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module
only converts Python / torch arguments to the C ABI.  If the shared library
is missing the import fails loudly — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(_HERE)
LIB_PATH = os.path.abspath(os.environ.get("PSSGP_LIB") or os.path.join(_HERE, "libpssgp.so"))
CSRC = os.path.join(_HERE, "csrc")
HEADER = os.path.join(ROOT, "include", "pssgp.h")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]

PSSGP_OK, PSSGP_E_ARG, PSSGP_E_INPUT, PSSGP_E_NUMERIC, PSSGP_E_CUDA, PSSGP_E_NOMEM, PSSGP_E_UNSUPPORTED = range(7)
STATUS_NAMES = {0: "OK", 1: "E_ARG", 2: "E_INPUT", 3: "E_NUMERIC", 4: "E_CUDA", 5: "E_NOMEM", 6: "E_UNSUPPORTED"}
KINDS = {"matern12": 1, "matern32": 2, "matern52": 3, "rbf": 4, "periodic": 5, "quasiperiodic": 6}


def wide_dims():
    """State dimensions of the warp-per-chain path (csrc/pssgp_dims.h), one object each."""
    import re
    txt = open(os.path.join(CSRC, "pssgp_dims.h")).read()
    line = next(ln for ln in txt.splitlines() if ln.startswith("#define PSSGP_WIDE_DIMS"))
    return [int(x) for x in re.findall(r"X\((\d+)\)", line)]


def build(force: bool = False, verbose: bool = False, jobs: int = 0) -> str:
    """Compile libpssgp.so for sm_100a with nvcc, in-tree: pssgp_api.cu (C ABI, d <= 3 path),
    pssgp_f32.cu, and pssgp_wide_inst.cu once per wide state dimension, in parallel, then link."""
    from concurrent.futures import ThreadPoolExecutor
    srcs = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if not f.endswith(".o")]
    newest = max(os.path.getmtime(f) for f in srcs + [HEADER])
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= newest:
        return LIB_PATH
    objdir = os.path.join(_HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in NVCC_FLAGS if f != "-shared"] + ["-c"]
    units = [(os.path.join(CSRC, "pssgp_api.cu"), [], "pssgp_api.o"),
             (os.path.join(CSRC, "pssgp_f32.cu"), [], "pssgp_f32.o")]
    units += [(os.path.join(CSRC, "pssgp_wide_inst.cu"), [f"-DPSSGP_WD={d}"], f"pssgp_wide_{d}.o")
              for d in wide_dims()]

    def compile_one(u):
        src, defs, obj = u
        cmd = ["nvcc", *cflags, *defs, "-o", os.path.join(objdir, obj), src]
        return cmd, subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
        results = list(ex.map(compile_one, units))
    for cmd, res in results:
        if verbose or res.returncode != 0:
            print(" ".join(cmd), res.stdout, res.stderr)
        if res.returncode != 0:
            raise RuntimeError("nvcc failed building libpssgp.so")
    link = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
            "-o", LIB_PATH, *[os.path.join(objdir, u[2]) for u in units]]
    res = subprocess.run(link, capture_output=True, text=True)
    if verbose or res.returncode != 0:
        print(res.stdout, res.stderr)
    if res.returncode != 0:
        raise RuntimeError("nvcc link of libpssgp.so failed")
    return LIB_PATH


class PssgpError(RuntimeError):
    def __init__(self, status: int, msg: str = "", index: int = -1):
        super().__init__(f"pssgp status {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.index = index


class Component(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("variance", ctypes.c_double), ("lengthscale", ctypes.c_double),
                ("period", ctypes.c_double), ("order", ctypes.c_int), ("mat_lengthscale", ctypes.c_double),
                ("mat_nu2", ctypes.c_int)]


class Options(ctypes.Structure):
    _fields_ = [("balance", ctypes.c_int), ("device", ctypes.c_int), ("uniform_dt", ctypes.c_double),
                ("chain_len", ctypes.c_int64), ("blocks_per_sm", ctypes.c_int)]


_lib = None
_vp = ctypes.c_void_p
_dp = ctypes.POINTER(ctypes.c_double)
_i64 = ctypes.c_int64

# name -> (restype, argtypes); mirrors include/pssgp.h
SIGNATURES = {
    "pssgp_create": (ctypes.c_int, [ctypes.POINTER(Component), ctypes.c_int, ctypes.c_double,
                                    ctypes.POINTER(Options), ctypes.POINTER(_vp)]),
    "pssgp_destroy": (None, [_vp]),
    "pssgp_state_dim": (ctypes.c_int, [_vp]),
    "pssgp_posterior": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pssgp_nll": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, _vp, _vp]),
    "pssgp_nll_grad": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pssgp_num_params": (ctypes.c_int, [_vp]),
    "pssgp_posterior_f32": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pssgp_posterior_host": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pssgp_check": (ctypes.c_int, [_vp]),
    "pssgp_posterior_host_async": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pssgp_sync": (ctypes.c_int, [_vp]),
    "pssgp_merge_grid": (ctypes.c_int, [_vp, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pssgp_gather": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pssgp_predict": (ctypes.c_int, [_vp, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp]),
    "pssgp_posterior_batched": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp,
                                               _vp, _vp, _vp]),
    "pssgp_nll_grad_batched": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp,
                                              _vp, _vp]),
    "pssgp_posterior_batched_theta": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp,
                                                     _vp, _vp]),
    "pssgp_nll_grad_batched_theta": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp,
                                                    _vp]),
    "pssgp_error_index": (ctypes.c_int64, [_vp]),
    "pssgp_last_error": (ctypes.c_char_p, [_vp]),
    "pssgp_get_ssm": (ctypes.c_int, [_vp, _dp, _dp, _dp, _dp, _dp]),
    "pssgp_debug_discretize": (ctypes.c_int, [_vp, ctypes.c_double, _dp, _dp]),
    "pssgp_plan": (ctypes.c_int, [_vp, _i64, ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                                  ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    "pssgp_plan_f32": (ctypes.c_int, [_vp, _i64, ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                                  ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    "pssgp_profile_enable": (None, [_vp, ctypes.c_int]),
    "pssgp_profile_read": (ctypes.c_int, [_vp, _dp, ctypes.POINTER(_i64), ctypes.c_int]),
    "pssgp_profile_name": (ctypes.c_char_p, [ctypes.c_int]),
    "pssgp_aggregate_bytes": (ctypes.c_size_t, [_vp, ctypes.c_int]),
    "pssgp_measure_fp64_peak": (ctypes.c_int, [_vp, _dp]),
    "pssgp_shard_filter_reduce": (ctypes.c_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp]),
    "pssgp_shard_filter_apply": (ctypes.c_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, ctypes.c_int,
                                                ctypes.c_int, _vp, _vp, _vp]),
    "pssgp_shard_smoother_apply": (ctypes.c_int, [_vp, _i64, _i64, _i64, _vp, _vp, ctypes.c_int, ctypes.c_int,
                                                  _vp, _vp, _vp, _vp]),
}


def lib():
    """Load libpssgp.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib
