"""Top stalled instructions of the hottest block of an ncu SASS source-page CSV.
usage: python tools/hot_stalls.py src.csv [min_frac]"""
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
cnt = collections.Counter(d[1] for d in data)
top = max(cnt, key=lambda c: c * cnt[c])
hot = [d for d in data if d[1] == top]
tot = sum(d[2] for d in hot)
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
print(f"hot block: {len(hot)} instrs x {top}, {tot} stall samples")
for i, (src, n, s) in enumerate(hot):
    if s > thr * tot:
        print(f"{i:4d} {s:6d} {s / tot * 100:5.1f}%  {src}")
