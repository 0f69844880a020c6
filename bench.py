"""bench.py — headline benchmark of the PSSGP hot path on B200.

Metric (BASELINE.json): time-steps/s of filter + smoother + NLL in fp64,
Matern-5/2, N = 2^24 grid points (irregular jittered times at the paper's
finest density h = 4/2^15, 1/16 of the points missing = test points).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (time-sharded, NCCL)

One JSON line on rank 0.  A "step" = one full pssgp_posterior over the whole
grid (all hot-path rows: discretisation, filter elements, forward scan,
smoother scan, NLL), inputs resident in HBM.  The working set (inputs 285 MB,
filtered state 1.2 GB, outputs 268 MB) is far larger than the 126 MB L2, so
no explicit L2 flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "time-steps/s (filter+smoother+NLL, fp64) Matern-5/2 N=2^24"
UNIT = "time-steps/s"
# fp64 pipe peak derived from the unit counts and clock: 148 SM x 64 DFMA/clk x 2 flop
# x 1.965 GHz; the roofline uses the DFMA throughput MEASURED live on this GPU (pssgp_measure_fp64_peak)
FP64_PEAK_DERIVED_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12
THROTTLE_BAD = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
SLOTS = ("k_filter_reduce", "k_filter_scan", "k_filter_apply", "k_smoother_scan", "k_smoother_apply",
         "k_nll_sum", "k_reduce_blocks", "k_grad_fold", "k_discretize")


def state_size(d: int) -> int:
    """S(d) = d + d(d+1)/2 reals per filtered-state record (x, P packed upper)."""
    return d + d * (d + 1) // 2


def path_alg_bytes(d: int, f32: bool = False) -> int:
    """Algorithmic bytes per time step of the whole path: t, y, mask in (17), the
    filtered state written and read once (2 x 8 S), t re-read (8), mean and var out (16)."""
    return 41 + (8 if f32 else 16) * state_size(d)


def alg_bytes(slot: str, d: int, wide_stream: bool = False, f32: bool = False) -> int:
    """Algorithmic bytes per time step moved by the kernel in profile slot `slot`:
    K1 reads t, y, mask; K3 reads them and writes the filtered state; K5 reads t and the filtered
    state and writes mean, var; the gradient fold reads the inputs and the filtered state.  On the
    wide path with per-step discretisation (irregular dt) each pass also reads the step's (F, Q)
    record of 2 d (d+1) doubles, which k_discretize writes.  Scans / sums: O(chains), 0 per step."""
    st = (4 if f32 else 8) * state_size(d)
    fq = 16 * d * (d + 1) if wide_stream else 0
    return {"k_filter_reduce": 17 + fq, "k_filter_apply": 17 + st + fq, "k_smoother_apply": 8 + st + 16 + fq,
            "k_grad_fold": 17 + st, "k_discretize": 8 + 16 * d * (d + 1)}.get(slot, 0)


# kernel families behind each profile slot (thread path d <= 3, wide path d >= 4)
_FAMILY = {"k_filter_reduce": ("k_filter_reduce", ("kw_filter_fold",)),
           "k_filter_apply": ("k_filter_apply", ("kw_filter_apply", "kw_grad_forward", "kb_posterior")),
           "k_smoother_apply": ("k_smoother_apply", ("kw_smoother_apply", "kw_smoother_mbf")),
           "k_grad_fold": ("k_grad_fold", ("k_grad_fold", "kw_grad_backward", "kb_nll_grad")),
           "k_discretize": ("k_discretize", ("kw_discretize", "kb_build")), "k_filter_scan": ("", ("kw_scan_filter",)),
           "k_smoother_scan": ("", ("kw_scan_smoother", "kw_scan_adjoint"))}


def _ncu_row(slot: str, d: int, cfg_key: str, f32: bool = False):
    """Row of the kernel behind `slot` at state dimension d in the newest committed ncu summary of
    this configuration (profiles/*/ncu_full_<tag>_summary.csv from tools/make_profile_summary.py;
    tags end in _<config key>, e.g. r2a_c3; untagged round-1 captures are the d = 3 metric
    workload; fp32 captures are tagged f32).  DRAM bytes in GB."""
    import csv
    import glob
    fam = _FAMILY.get(slot)
    if fam is None:
        return None, None
    fams = (fam[0],) if (d <= 3 and cfg_key != "gradco2") else fam[1]
    fams = [f for f in fams if f]
    if not fams:
        return None, None

    def tag_key(f):
        tag = os.path.basename(f)[len("ncu_full_"):-len("_summary.csv")]
        if "f32" in tag:
            return "f32"
        return tag.split("_", 1)[1] if "_" in tag else "metric"
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "ncu_full_*_summary.csv")))
    want = "f32" if f32 else cfg_key
    for f in reversed(files):
        if tag_key(f) != want:
            continue
        for row in csv.DictReader(open(f)):
            name = row["Kernel Name"]
            if any(fam + "<" in name or fam + "_lpr<" in name or fam + "_q<" in name for fam in fams):
                targs = name[name.index("<") + 1:]
                if targs.startswith(f"{d},") or targs.startswith(f"{d}>"):
                    return row, os.path.relpath(f, ROOT)
    return None, None


def ncu_traffic(slot: str, d: int, cfg_key: str, f32: bool = False):
    """dram read+write bytes per launch of the kernel behind `slot` from one `ncu --set full` capture."""
    row, src = _ncu_row(slot, d, cfg_key, f32)
    if row is None:
        return None, None
    return (float(row["dram__bytes_read.sum"]) + float(row["dram__bytes_write.sum"])) * 1e9, src


# warp-cooperative kernels whose d x d products (per step, per chain) run through the register-tiled
# wmm (pssgp_wide.cuh) for d outside {8, 16}: the padded tile rows / columns execute FMAs that are
# not algorithmic work
_TILED_PRODUCTS = {"kw_filter_fold<": 3, "kw_filter_apply<": 3, "kw_grad_forward<": 3, "kw_grad_backward<": 3}


def flops_per_step(slot: str, d: int, cfg_key: str):
    """Algorithmic fp64 flops per time step (DFMA = 2): the SASS counts of the committed capture, less
    the padded-tile FMAs of the register-tiled warp products (2 (32 RB CB d - d^3) each)."""
    row, _ = _ncu_row(slot, d, cfg_key)
    if row is not None and row.get("fp64_flops_per_step"):
        fl = float(row["fp64_flops_per_step"])
        name = row["Kernel Name"]
        if d * d > 32 and d not in (8, 16):
            rb, cb = (d + 3) // 4, (d + 7) // 8
            for k, n in _TILED_PRODUCTS.items():
                if k in name:
                    fl -= n * 2 * (32 * rb * cb * d - d ** 3)
        return fl
    return None


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--N", type=int, default=2 ** 24)
    ap.add_argument("--uniform", action="store_true", help="uniform dt (secondary row)")
    ap.add_argument("--kind", default="matern52")
    ap.add_argument("--config", default="metric", choices=["metric", "c2", "c3", "c4", "c5", "batched", "grad", "gradb", "gradco2", "gradbt",
                                                          "batchedbt", "co2post", "f32"],
                    help="workload (default: the BASELINE metric); c3/c4 are the d = 6 / d = 16 rows")
    ap.add_argument("--irregular", action="store_true", help="c3/c4 on a jittered grid (device Pade discretisation)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=2 ** 21)
    ap.add_argument("--chain-len", type=int, default=0)
    ap.add_argument("--blocks-per-sm", type=int, default=0)
    return ap.parse_args()


def config_key(args) -> str:
    """Key of the committed ncu summaries of this workload (profiles/*/ncu_full_<tag>_<key>_summary.csv)."""
    if args.config == "metric":
        return "metric_uniform" if args.uniform else "metric"
    return args.config + ("i" if args.irregular and args.config in ("c3", "c4") else "")


def ensure_ranks(args) -> None:
    """`--gpus N` means N ranks, one per GPU.  Under torchrun (WORLD_SIZE set) WORLD_SIZE must equal
    N; started directly with N > 1 the script re-launches itself through torch.distributed.run with
    N local ranks (NCCL), or exits with an error when fewer than N GPUs are visible.  It never
    falls back to fewer GPUs than asked for."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is not None:
        if int(ws) != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; launch one rank per GPU")
        return
    if args.gpus <= 1 or args.impl == "reference":
        return
    import socket
    import torch
    n = torch.cuda.device_count()
    if n < args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, {n} visible; refusing to run "
                 f"fewer ranks than asked for")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    print("bench.py: launching " + " ".join(cmd), file=sys.stderr, flush=True)
    os.execv(sys.executable, cmd)


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    REASONS = ["clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
               "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def start(self):
        q = "clocks.sm,clocks.max.sm,power.draw," + ",".join(self.REASONS)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 3:
                self.samples.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in self.samples:
            for name, v in zip(names, s[3:]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "_fallback": True}


# ------------------------------------------------------------------------------ cpu baseline (oracle)
_CPU_JOB = None


def _cpu_replica(_):
    import oracle
    comps, r, t, y, mask = _CPU_JOB
    m = oracle.ssm.build(comps)
    t0 = time.perf_counter()
    oracle.kf_rts(m, r, t, y, mask)
    return time.perf_counter() - t0


def cpu_baseline(w, sample: int):
    """The oracle as it stands on the host cores: one sequential run (the recurrence is serial), plus
    an all-cores row of os.cpu_count() concurrent independent replicas."""
    global _CPU_JOB
    import multiprocessing as mp
    import oracle
    n = min(sample, w.N)
    m = oracle.ssm.build(w.components)
    t0 = time.perf_counter()
    oracle.kf_rts(m, w.noise_var, w.t[:n], w.y[:n], w.mask[:n])
    dt = time.perf_counter() - t0
    ncpu = os.cpu_count() or 1
    nr = max(1, n // 4)
    _CPU_JOB = (w.components, w.noise_var, w.t[:nr], w.y[:nr], w.mask[:nr])
    allc = None
    try:
        with mp.get_context("fork").Pool(ncpu) as pool:
            dts = pool.map(_cpu_replica, range(ncpu), chunksize=1)
        allc = {"value": ncpu * nr / max(dts), "cores": ncpu,
                "sample": f"{ncpu} concurrent replicas x first {nr} steps, slowest {max(dts):.2f} s"}
    except OSError as e:   # no fork / too few resources: report the single-core row only
        allc = {"unavailable": str(e)}
    return {"value": n / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"first {n} steps of the same grid, sequential C oracle (KF+RTS+NLL, Van Loan per step), "
                      f"{dt:.2f} s on {ncpu} host cores (1 used)",
            "cpu_model": cpu_model(), "host_cores": ncpu, "all_cores": allc}


def make_workload(args):
    import synth
    if args.config == "c2":
        return synth.config2()
    if args.config == "c3":
        return synth.config3(n=args.N if args.N != 2 ** 24 else 2 ** 22, irregular=args.irregular)
    if args.config == "c4":
        return synth.config4(n=args.N, irregular=args.irregular)
    if args.config == "f32":
        return synth.metric_workload(args.N)
    if args.config == "c5":
        return synth.metric_workload(2 ** 27 if args.N == 2 ** 24 else args.N)
    if args.config in ("batched", "gradb"):
        return synth.metric_workload(3200 * 4, kind="matern52")
    if args.config == "grad":
        return synth.metric_workload(args.N)
    if args.config in ("gradbt", "batchedbt"):
        # B HMC chains / multi-start fits of the paper's CO2 model (J = 3, n_x = 18), one 3,200-week
        # series each
        return synth.co2_product(n=3200, order=3)
    if args.config == "co2post":
        # the posterior of the paper's CO2 model C_Per x C_Mat + C_Mat at n_x = 18 (J = 3), weekly grid
        return synth.co2_product(n=args.N if args.N != 2 ** 24 else 2 ** 20, order=3)
    if args.config == "gradco2":
        # the paper's HMC model C_Per x C_Mat + C_Mat at n_x = 18 (J = 3), weekly grid
        return synth.co2_product(n=args.N if args.N != 2 ** 24 else 2 ** 20, order=3)
    return synth.metric_workload(args.N, uniform=args.uniform, kind=args.kind)


def run_reference(args, rank: int):
    """--impl reference: the CPU oracle as the reference arm (rank 0 only)."""
    if rank != 0:
        return
    w = make_workload(args)
    import oracle
    m = oracle.ssm.build(w.components)
    n = min(2 ** 19, w.N)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.kf_rts(m, w.noise_var, w.t[:n], w.y[:n], w.mask[:n])
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    tot = sum(times)
    val = n * args.steps / tot
    metric = METRIC if (args.config == "metric" and not args.uniform) else \
        f"time-steps/s (filter+smoother+NLL, fp64) {w.name} N={w.N}"
    line = {"impl": "reference", "metric": metric, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": w.name, "N": w.N, "sample_steps": n},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"first {n} steps of {w.name} per step", "cpu_model": cpu_model(),
                             "host_cores": os.cpu_count()},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ ours
def main():
    args = parse()
    ensure_ranks(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    import torch
    import synth
    import paper_2102_09964_b200 as P
    from paper_2102_09964_b200 import sharded

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    nccl_info = None
    if world > 1:
        # NCCL's own INIT lines (communicator size, ring / NVLS setup) in the log, once at start-up
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        # communicator check: one all_reduce of ones over NCCL must equal the world size
        one = torch.ones(1, device=dev)
        dist.all_reduce(one)
        nccl_info = {"backend": dist.get_backend(), "comm_nranks": int(one.item()),
                     "world_size": dist.get_world_size(), "nccl_version": ".".join(map(str, torch.cuda.nccl.version()))}
        if rank == 0:
            print(f"bench.py: NCCL communicator of {nccl_info['comm_nranks']} ranks "
                  f"(NCCL {nccl_info['nccl_version']})", file=sys.stderr, flush=True)

    w = make_workload(args)
    model = P.Model(w.components, w.noise_var, uniform_dt=w.uniform_dt, chain_len=args.chain_len,
                    blocks_per_sm=args.blocks_per_sm, device=local)
    N = w.N
    stream = torch.cuda.current_stream()

    if args.config in ("batched", "gradb"):
        # f2: B series of 3,200 points (the sunspot N of PAPER.md:206), each with its own
        # hyper-parameters (multi-start / HMC shape), one launch
        # multi-GPU: every rank runs its own batch of independent series (replicas, no collective)
        B = max(1, args.N // 3200)
        rng = np.random.default_rng(rank)
        lens = np.full(B, 3200, np.int64)
        off = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)])).to(dev)
        VB = torch.from_numpy(rng.uniform(0.5, 2.0, B)).to(dev)
        EB = torch.from_numpy(rng.uniform(0.2, 1.0, B)).to(dev)
        RB = torch.from_numpy(rng.uniform(0.005, 0.05, B)).to(dev)
        N = int(lens.sum())
        tb = np.tile(w.t[:3200] - w.t[0], B); yb = np.tile(w.y[:3200], B); mb = np.tile(w.mask[:3200], B)
        t = torch.from_numpy(tb).to(dev); y = torch.from_numpy(yb).to(dev); mk = torch.from_numpy(mb).to(dev)
        mean = torch.empty(N, dtype=torch.float64, device=dev)
        var = torch.empty_like(mean)
        nllb = torch.empty(B, dtype=torch.float64, device=dev)
        gb = torch.empty(3 * B, dtype=torch.float64, device=dev)

        if args.config == "batched":
            def step():
                P.pssgp_posterior_batched(model.h, B, off, VB, EB, RB, N, t, y, mk, mean, var, nllb, stream)
        else:
            # f1 x f2: per-series NLL + gradient (one multi-start / HMC evaluation of B fits)
            def step():
                P.pssgp_nll_grad_batched(model.h, B, off, VB, EB, RB, N, t, y, mk, nllb, gb, stream)
        n_local = N
    elif args.config in ("gradbt", "batchedbt"):
        # f2 widened: B series of the CO2 grid, each at its own log hyper-parameters (theta_b drawn
        # around the model's own, +-0.25), one launch: the HMC-chain shape of PAPER.md:224-235
        B = max(1, args.N // 3200) if args.N != 2 ** 24 else 1024
        rng = np.random.default_rng(rank)
        lens = np.full(B, w.N, np.int64)
        off = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)])).to(dev)
        th = torch.from_numpy(model.theta[None, :] + rng.uniform(-0.25, 0.25, (B, model.num_params))).to(dev)
        N = int(lens.sum())
        t = torch.from_numpy(np.tile(w.t, B)).to(dev)
        y = torch.from_numpy(np.tile(w.y, B)).to(dev)
        mk = torch.from_numpy(np.tile(w.mask, B)).to(dev)
        nllb = torch.empty(B, dtype=torch.float64, device=dev)
        gb = torch.empty(B * model.num_params, dtype=torch.float64, device=dev)
        mean = torch.empty(N, dtype=torch.float64, device=dev)
        var = torch.empty_like(mean)
        if args.config == "gradbt":
            def step():
                P.pssgp_nll_grad_batched_theta(model.h, B, off, th, N, t, y, mk, nllb, gb, stream)
        else:
            def step():
                P.pssgp_posterior_batched_theta(model.h, B, off, th, N, t, y, mk, mean, var, nllb, stream)
        n_local = N
    elif args.config in ("grad", "gradco2"):
        # f1: NLL + its gradient in every log hyper-parameter (one L-BFGS / HMC evaluation): the metric
        # grid (one Matern component, 3 parameters) or the CO2 model (reverse mode, 8 parameters)
        t = torch.from_numpy(w.t).to(dev)
        y = torch.from_numpy(w.y).to(dev)
        mk = torch.from_numpy(w.mask).to(dev)
        nll = torch.zeros(1, dtype=torch.float64, device=dev)
        gr = torch.zeros(model.num_params, dtype=torch.float64, device=dev)

        def step():
            P.pssgp_nll_grad(model.h, N, t, y, mk, nll, gr, stream)
        n_local = N
    elif args.config == "f32" and world == 1:
        # the optional fp32-state path on the metric workload
        t = torch.from_numpy(w.t).to(dev)
        y = torch.from_numpy(w.y).to(dev)
        mk = torch.from_numpy(w.mask).to(dev)
        mean = torch.empty(N, dtype=torch.float64, device=dev)
        var = torch.empty_like(mean)
        nll = torch.zeros(1, dtype=torch.float64, device=dev)

        def step():
            P.pssgp_posterior_f32(model.h, N, t, y, mk, mean, var, nll, stream)
        n_local = N
    elif world == 1:
        t = torch.from_numpy(w.t).to(dev)
        y = torch.from_numpy(w.y).to(dev)
        mk = torch.from_numpy(w.mask).to(dev)
        mean = torch.empty(N, dtype=torch.float64, device=dev)
        var = torch.empty_like(mean)
        nll = torch.zeros(1, dtype=torch.float64, device=dev)

        def step():
            P.pssgp_posterior(model.h, N, t, y, mk, mean, var, nll, stream)
        n_local = N
    else:
        k0, n_local = sharded.split(N, world)[rank]
        tt, yy, mm = sharded.chunk_inputs(w.t, w.y, w.mask, k0, n_local, dev)
        shard = sharded.DeviceShard(model, tt, yy, mm, k0, n_local, N, rank, world, stream)

        def step():
            sharded.sharded_posterior(shard, sharded.nccl_exchange, rank, world)

    for _ in range(args.warmup):
        step()
    model.check()
    torch.cuda.synchronize()

    def timed_region():
        clocks = ClockSampler(local)
        clocks.start()
        P.pssgp_profile_enable(model.h, True)
        P.pssgp_profile_read(model.h)  # reset
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ms = ev0.elapsed_time(ev1)
        prof_ = P.pssgp_profile_read(model.h)
        P.pssgp_profile_enable(model.h, False)
        return ms, prof_, clocks.stop()

    ms_total, prof, clk = timed_region()
    if set(clk.get("reasons", [])) & THROTTLE_BAD:      # rejected run: measure once more
        ms_total, prof, clk = timed_region()
        clk["remeasured"] = True
    model.check()
    if dist:
        tt_ = torch.tensor([ms_total], dtype=torch.float64, device=dev)
        dist.all_reduce(tt_, op=dist.ReduceOp.MAX)
        ms_total = float(tt_.item())
    ms_step = ms_total / args.steps
    # independent problems per rank (batched series, gradient evaluations): weak scaling, the
    # job's units are all ranks' steps; the time-sharded posterior: strong scaling over one grid
    replicas = args.config in ("batched", "grad", "gradb", "gradco2", "gradbt", "batchedbt") and world > 1
    units = N * world if replicas else N
    value = units / (ms_step * 1e-3)

    # ---- e2e through the public host API (pinned buffers, copies inside the timed region)
    e2e = None
    if world == 1 and args.config not in ("batched", "grad", "gradb", "gradco2", "gradbt", "batchedbt", "f32"):
        th = torch.from_numpy(w.t).pin_memory()
        yh = torch.from_numpy(w.y).pin_memory()
        mh = torch.from_numpy(w.mask).pin_memory()
        meanh = torch.empty(N, dtype=torch.float64).pin_memory()
        varh = torch.empty(N, dtype=torch.float64).pin_memory()
        nllh = torch.zeros(1, dtype=torch.float64).pin_memory()

        # the pipelined host API: each call copies its inputs host -> device, runs the path and
        # copies mean, var, nll back; consecutive calls overlap one call's device -> host with
        # the next call's host -> device (two output sets alternate).  Wall clock around the
        # whole loop + pssgp_sync (every byte of every step is inside the timed region).
        meanh2 = torch.empty(N, dtype=torch.float64).pin_memory()
        varh2 = torch.empty(N, dtype=torch.float64).pin_memory()
        nllh2 = torch.zeros(1, dtype=torch.float64).pin_memory()
        outs = [(meanh, varh, nllh), (meanh2, varh2, nllh2)]

        def step_host(i):
            mo, vo, no = outs[i & 1]
            P.pssgp_posterior_host_async(model.h, N, th, yh, mh, mo, vo, no)
        for i in range(2):
            step_host(i)
        P.pssgp_sync(model.h)
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        for i in range(args.steps):
            step_host(i)
        P.pssgp_sync(model.h)
        e_ms = (time.perf_counter() - h0) * 1e3 / args.steps
        # the synchronous call (no overlap between calls), for reference
        s0 = time.perf_counter()
        for _ in range(max(2, args.steps // 2)):
            P.pssgp_posterior_host(model.h, N, th, yh, mh, meanh, varh, nllh, stream)
        sync_ms = (time.perf_counter() - s0) * 1e3 / max(2, args.steps // 2)
        e2e = {"value": N / (e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(N * 17),
               "d2h_bytes_per_step": int(N * 16 + 8), "ms_per_step": e_ms,
               "api": "pssgp_posterior_host_async (pipelined, wall clock)", "sync_api_ms_per_step": sync_ms}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    # ---- roofline for the dominant kernel: algorithmic bytes / HBM peak or executed
    # fp64 flops / fp64 peak, whichever floor is larger, from per-kernel CUDA-event times of the
    # timed region (events recorded by the library on the launch stream)
    pk = peaks()
    d = model.state_dim
    f32 = args.config == "f32"
    wide_stream = d > 3 and w.uniform_dt == 0.0
    ckey = config_key(args)
    fp64_peak = P.pssgp_measure_fp64_peak(model.h) if hasattr(P, "pssgp_measure_fp64_peak") else None
    fp64_src = "measured in this run: DFMA throughput kernel, all SMs (pssgp_measure_fp64_peak)"
    if not fp64_peak:
        fp64_peak, fp64_src = FP64_PEAK_DERIVED_TFLOPS, "derived: 148 SM x 64 DFMA/clk x 2 x 1.965 GHz"
    kern = {k: v for k, v in prof.items() if v[1] > 0}
    per_kernel = {}
    for k, (kms, kl) in kern.items():
        b = alg_bytes(k, d, wide_stream, f32) * n_local
        fl = flops_per_step(k, d, ckey)
        if args.config in ("gradbt", "batchedbt") and k in ("k_grad_fold", "k_filter_apply"):
            # one warp per series: the algorithmic count of its sequential filter + adjoint (10 d^3 +
            # 38 d^2) or filter + adjoint-form RTS (8 d^3 + 32 d^2) per step; the SASS
            # count of the register-tiled kernels includes the padded tile rows / columns
            fl = 10 * d ** 3 + 38 * d ** 2 if k == "k_grad_fold" else 8 * d ** 3 + 32 * d ** 2
        launch_ms = kms / kl
        e = {"ms_per_step": kms / args.steps, "launches_per_step": kl / args.steps, "alg_bytes_per_step": alg_bytes(k, d, wide_stream, f32)}
        if b:
            e["hbm_frac"] = b / (launch_ms * 1e-3) / 1e9 / pk.get("hbm_gbs")
        if fl and not f32:
            e["fp64_flops_per_step"] = fl
            e["fp64_frac"] = fl * n_local / (launch_ms * 1e-3) / 1e12 / fp64_peak
        per_kernel[k] = e
    dom = max(kern, key=lambda k: kern[k][0])
    dom_ms, dom_launches = kern[dom]
    per_launch_ms = dom_ms / dom_launches
    alg_b = alg_bytes(dom, d, wide_stream, f32) * n_local
    hbm_gbs = alg_b / (per_launch_ms * 1e-3) / 1e9
    fl = per_kernel[dom].get("fp64_flops_per_step")
    launches = int(sum(v[1] for v in kern.values()))
    traffic, traffic_src = ncu_traffic(dom, d, ckey, f32)
    hbm_frac = hbm_gbs / pk.get("hbm_gbs")
    alu = None
    if fl:
        achieved_tf = fl * n_local / (per_launch_ms * 1e-3) / 1e12
        alu = {"achieved_tflops": achieved_tf, "peak_tflops": fp64_peak, "frac": achieved_tf / fp64_peak,
               "flops_per_step": fl, "peak_source": fp64_src, "peak_derived_tflops": FP64_PEAK_DERIVED_TFLOPS}
    if alu and alu["frac"] > hbm_frac:
        roof = {"bound": "alu", "kernel": dom, "achieved": alu["achieved_tflops"], "peak": fp64_peak,
                "unit": "TFLOP/s", "frac": alu["frac"], "traffic": traffic}
    else:
        roof = {"bound": "hbm", "kernel": dom, "achieved": hbm_gbs, "peak": pk.get("hbm_gbs"), "unit": "GB/s",
                "frac": hbm_frac, "traffic": traffic}
    roof["alu"] = alu
    path_b = path_alg_bytes(d, f32)
    fl_all = [per_kernel[k].get("fp64_flops_per_step") for k in kern if alg_bytes(k, d) or k == "k_grad_fold"]
    plan = model.plan(n_local, f32=f32)
    roof.update({
        "traffic_source": traffic_src,
        "alg_bytes_per_launch": alg_b,
        "hbm": {"achieved_gbs": hbm_gbs, "peak_gbs": pk.get("hbm_gbs"), "frac": hbm_frac,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if not pk.get("_fallback") else "fallback"},
        "avg_launch_ms": per_launch_ms,
        "share_of_step": dom_ms / ms_total,
        "per_kernel": per_kernel,
        "per_kernel_ms_per_step": {k: v[0] / args.steps for k, v in kern.items()},
        "state_dim": d,
        "path_alg_bytes_per_step": path_b,
        "path_hbm_frac": path_b * N / (ms_step * 1e-3) / 1e9 / pk.get("hbm_gbs"),
        "path_fp64_frac": (sum(fl_all) * N / (ms_step * 1e-3) / 1e12 / fp64_peak)
        if fl_all and all(fl_all) and not f32 else None})
    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_baseline(w, args.cpu_sample)
    if args.config == "metric" and not args.uniform:
        metric = METRIC
    elif args.config in ("grad", "gradco2"):
        metric = f"time-steps/s (NLL + {model.num_params}-parameter gradient, fp64) {w.name} N={N}"
    elif args.config == "f32":
        metric = f"time-steps/s (filter+smoother+NLL, fp32 state) {w.name} N={N}"
    elif args.config == "gradb":
        metric = f"time-steps/s (per-series NLL + gradient, fp64) batched Matern-5/2 series of 3200 N={N}"
    elif args.config == "gradbt":
        metric = (f"time-steps/s (per-series NLL + {model.num_params}-parameter gradient at per-series theta, fp64) "
                  f"{w.name} x {N // w.N} series N={N}")
    elif args.config == "batchedbt":
        metric = f"time-steps/s (filter+smoother+NLL at per-series theta, fp64) {w.name} x {N // w.N} series N={N}"
    else:
        metric = (f"time-steps/s (filter+smoother+NLL, fp64) "
                  f"{w.name if args.config != 'batched' else 'batched Matern-5/2 series of 3200'} N={N}")
    extra = {}
    if args.config in ("grad", "gradco2"):
        # latency of one NLL+gradient evaluation at the sunspot size N = 3,200 (Table 1;
        # the CO2 series has ~3,200 weekly points)
        n1 = 3200
        t1, y1, m1 = t[:n1].contiguous(), y[:n1].contiguous(), mk[:n1].contiguous()
        for _ in range(5):
            P.pssgp_nll_grad(model.h, n1, t1, y1, m1, nll, gr, stream)
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(200):
            P.pssgp_nll_grad(model.h, n1, t1, y1, m1, nll, gr, stream)
        a1.record(stream)
        torch.cuda.synchronize()
        extra["latency_n3200_ms"] = a0.elapsed_time(a1) / 200
    line = {"metric": metric, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak" if replicas else "strong", "vs_baseline": None,
            "dtype": "f32 (state; f64 times, I/O, NLL sum)" if args.config == "f32" else "f64",
            "data": "synthetic",
            "config": {"workload": w.name, "N": N, "state_dim": model.state_dim, "chain_len": plan["chain_len"],
                       "ctas": plan["n_blocks"], "threads_per_cta": plan["threads"],
                       "l2": f"no flush: working set ({path_b * N / 1e9:.2f} GB per step) >> 126 MB L2",
                       "parallelism": f"time-sharded x{world}" if world > 1 else "single GPU", "nccl": nccl_info},
            "clocks": clk, "e2e": e2e, "gpu_launches": launches, "roofline": roof, "cpu_baseline": cpu, **extra}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
