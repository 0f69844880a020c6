"""Build the committed ncu summary for one profiling round from tools/profile_round.sh output.

usage: python tools/make_profile_summary.py gpurun_out/TAG profiles/ROUND N [TAG]
Writes profiles/TAG/ncu_full_TAG_summary.csv (per hot kernel: duration in us, DRAM bytes in GB, fp64 pipe
and issue utilisation, stall ratios, executed fp64 instructions and flops per time step from the
SASS source page), copies the launch list and the bench line."""
import csv
import glob
import os
import shutil
import sys

src, dst, N = sys.argv[1], sys.argv[2], float(sys.argv[3])
tag = sys.argv[4] if len(sys.argv) > 4 else os.path.basename(src.rstrip("/"))
os.makedirs(dst, exist_ok=True)
SCALE = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}
TSCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
           "launch__registers_per_thread", "sm__warps_active.avg.per_cycle_active",
           "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
           "sm__cycles_elapsed.avg.per_second"]


def fp64_per_step(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Source" in r)
    hdr = rows[hi]
    i_src, i_pt = hdr.index("Source"), hdr.index("Predicated-On Thread Instructions Executed")
    cnt = {"DFMA": 0.0, "DMUL": 0.0, "DADD": 0.0}
    for r in rows[hi + 1:]:
        if len(r) <= max(i_src, i_pt):
            continue
        toks = r[i_src].strip().split()
        if not toks:
            continue
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        if op in cnt:
            try:
                cnt[op] += float(r[i_pt])
            except ValueError:
                pass
    instr = sum(cnt.values()) / N
    flops = (2 * cnt["DFMA"] + cnt["DMUL"] + cnt["DADD"]) / N
    return instr, flops


out = []
for raw in sorted(glob.glob(os.path.join(src, "raw_*.csv"))):
    k = os.path.basename(raw)[4:-4]
    rows = list(csv.reader(open(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    rec = {"Kernel Name": v[h.index("Kernel Name")]}
    for m in METRICS:
        i = h.index(m)
        val = float(v[i])
        if m.startswith("dram__bytes"):
            val *= SCALE[u[i]]           # -> GB
        if m == "gpu__time_duration.sum":
            val *= TSCALE[u[i]]          # -> us
        rec[m] = val
    s = os.path.join(src, f"src_{k}.csv")
    if os.path.exists(s):
        rec["fp64_instr_per_step"], rec["fp64_flops_per_step"] = fp64_per_step(s)
    out.append(rec)
cols = ["Kernel Name"] + METRICS + ["fp64_instr_per_step", "fp64_flops_per_step"]
with open(os.path.join(dst, f"ncu_full_{tag}_summary.csv"), "w", newline="") as f:
    w = csv.DictWriter(f, fieldnames=cols)
    w.writeheader()
    for r in out:
        w.writerow(r)
for name in ("launches.csv", "bench.json"):
    if os.path.exists(os.path.join(src, name)):
        shutil.copy(os.path.join(src, name), os.path.join(dst, f"{name.split('.')[0]}_{tag}.{name.split('.')[1]}"))
for r in out:
    print(r["Kernel Name"][:40], round(r["gpu__time_duration.sum"], 1), "us",
          round(r["dram__bytes_read.sum"] + r["dram__bytes_write.sum"], 3), "GB",
          round(r.get("fp64_flops_per_step", 0), 1), "flop/step")
