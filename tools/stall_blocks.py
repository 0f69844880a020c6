"""Group stall samples of an ncu source-page CSV by contiguous SASS regions with
the same execution count (~ basic blocks) and print the heaviest regions with
their dominant stall reasons.  usage: stall_blocks.py src.csv [top]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
hdr = rows[1]
i_src = hdr.index("Source"); i_ex = hdr.index("Instructions Executed"); i_s = hdr.index("Warp Stall Sampling (All Samples)")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ri = [hdr.index(h) for h in reasons]
lines = []
for r in rows[2:]:
    if len(r) <= max(i_s, i_ex, max(ri)): continue
    try: n = int(float(r[i_ex])); s = int(float(r[i_s]))
    except ValueError: continue
    st = []
    for j in ri:
        try: st.append(float(r[j]))
        except ValueError: st.append(0.0)
    lines.append((n, s, r[i_src].strip(), st))
# only the first copy (the source page lists the kernel twice)
half = len(lines) // 2
if half and all(lines[i][2] == lines[i + half][2] for i in range(0, half, max(1, half // 20))):
    lines = lines[:half]
tot = sum(l[1] for l in lines) or 1
blocks = []
cur = None
for i, (n, s, src, st) in enumerate(lines):
    if cur is None or n != cur["n"]:
        cur = {"n": n, "start": i, "samples": 0, "instr": [], "st": [0.0] * len(ri)}
        blocks.append(cur)
    cur["samples"] += s
    cur["instr"].append(src)
    cur["st"] = [a + b for a, b in zip(cur["st"], st)]
for b in sorted(blocks, key=lambda b: -b["samples"])[:top]:
    dom = sorted(zip(reasons, b["st"]), key=lambda x: -x[1])[:4]
    ops = collections.Counter(x.split()[0] if not x.startswith("@") else x.split()[1] for x in b["instr"] if x)
    print(f"{b['samples']/tot*100:5.1f}% exec={b['n']:8d} len={len(b['instr']):4d} start=#{b['start']} "
          f"{', '.join(f'{k[6:]}={v:.0f}' for k, v in dom)} | {', '.join(f'{k}:{v}' for k, v in ops.most_common(5))}")
