"""Opcode mix (executed warp instructions) and stall samples from an ncu source-page CSV."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
i_src, i_ex, i_smp = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
mix = collections.Counter(); smp = collections.Counter(); tot = 0; tots = 0
for r in rows[2:]:
    try:
        n = int(float(r[i_ex])); s = int(float(r[i_smp]))
    except Exception:
        continue
    op = r[i_src].strip().split()[0] if r[i_src].strip() else "?"
    if op.startswith("@"):
        op = r[i_src].strip().split()[1]
    base = op.split(".")[0]
    mix[base] += n; smp[base] += s; tot += n; tots += s
print(f"total warp instrs {tot:.4g}, samples {tots}")
for k, v in mix.most_common(40):
    print(f"{k:12s} {v/tot*100:6.2f}% instr   {smp[k]/max(tots,1)*100:6.2f}% stall-samples")
