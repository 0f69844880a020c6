"""List lane-strided loops (a conditional backward branch whose body steps an index by 32) that no
BSSY/BSYNC re-convergence region encloses, in every kernel of the given objects.  Such a loop
followed by a shared-memory hand-off relies on the __syncwarp that ptxas may elide (DESIGN.md §5d,
"A compiler finding").  usage: python tools/sass_divergent_loops.py paper_2102_09964_b200/build/*.o"""
import re
import subprocess
import sys


def functions(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    name, body = None, []
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if name:
                yield name, body
            name, body = m.group(1), []
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            body.append((int(m.group(1), 16), m.group(2).strip()))
    if name:
        yield name, body


def scan(path):
    lines = []
    for name, body in functions(path):
        regions = [(pc, int(m.group(1), 16)) for pc, ins in body
                   for m in [re.match(r"BSSY(?:\.RECONVERGENT)?\s+B\d+,\s*0x([0-9a-f]+)", ins)] if m]
        for pc, ins in body:
            m = re.match(r"@!?P\d\s+BRA\s+0x([0-9a-f]+)", ins)
            if not m:
                continue
            tgt = int(m.group(1), 16)
            if tgt >= pc or any(b < tgt and r > pc for b, r in regions):
                continue
            loop = [i for p, i in body if tgt <= p <= pc]
            after = [i for p, i in body if p > pc][:3]
            if any(re.search(r"(VIADD|IADD3).*0x20 ?$", i) for i in loop) and len(loop) < 120:
                lines.append(f"{path.split('/')[-1]} {name[:80]} loop {hex(tgt)}-{hex(pc)} ({len(loop)} instr), "
                             "then: " + " | ".join(after))
    return lines


def main(paths):
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=16) as ex:
        found = [ln for lines in ex.map(scan, paths) for ln in lines]
    for ln in found:
        print(ln)
    print("unenclosed lane-strided loops:", len(found))


if __name__ == "__main__":
    main(sys.argv[1:])
