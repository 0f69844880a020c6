"""Executed fp64 flops per time step from an ncu source-page CSV (thread-level,
predicated-on): DFMA = 2 flops, DMUL/DADD = 1.  usage: fp64_flops.py src.csv N"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
N = float(sys.argv[2])
hdr = rows[1]
i_src = hdr.index("Source"); i_pt = hdr.index("Predicated-On Thread Instructions Executed")
cnt = {"DFMA": 0, "DMUL": 0, "DADD": 0}
for r in rows[2:]:
    if len(r) <= max(i_src, i_pt): continue
    toks = r[i_src].strip().split()
    if not toks: continue
    op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
    if op in cnt:
        try: cnt[op] += float(r[i_pt])
        except ValueError: pass
fl = (2 * cnt["DFMA"] + cnt["DMUL"] + cnt["DADD"])
print({k: v / N for k, v in cnt.items()}, "flops/step", fl / N)
