"""Summarise an ncu SASS source-page CSV: instruction-count blocks by execution count, opcode mix
and stall samples of the hottest block.  usage: python tools/hot_blocks.py src.csv [nblocks]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Source" in r)
hdr = rows[hi]
i_src, i_ex, i_s = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[hi + 1:]:
    try:
        data.append((r[i_src].strip(), int(float(r[i_ex])), int(float(r[i_s]))))
    except (ValueError, IndexError):
        continue
tot = sum(d[1] for d in data)
tots = sum(d[2] for d in data)
print(f"total warp instrs {tot:.4g}  stall samples {tots}")
by = collections.defaultdict(list)
for d in data:
    by[d[1]].append(d)
blocks = sorted(by.items(), key=lambda kv: -kv[0] * len(kv[1]))
for cnt, ds in blocks[: int(sys.argv[2]) if len(sys.argv) > 2 else 6]:
    mix = collections.Counter()
    st = collections.Counter()
    for src, n, s in ds:
        op = src.split()[1] if src.startswith("@") else (src.split()[0] if src else "?")
        op = op.split(".")[0]
        mix[op] += 1
        st[op] += s
    fp = mix["DFMA"] + mix["DMUL"] + mix["DADD"]
    print(f"\nexec {cnt} x {len(ds)} instrs = {cnt*len(ds)/tot*100:.1f}% of instrs, "
          f"{sum(d[2] for d in ds)/max(tots,1)*100:.1f}% of stalls; fp64 {fp} ({fp/len(ds)*100:.0f}%)")
    print("   " + ", ".join(f"{k} {v}" for k, v in mix.most_common(14)))
