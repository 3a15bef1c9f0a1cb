"""Attribute ncu SASS stall samples (ncu --page source --csv) to CUDA source
lines through nvdisasm line info of the same build:
    cd /tmp/cubins && cuobjdump -xelf all .../libmdsx.so
    python tools/ncu_lines.py capture.csv /tmp/cubins/k_x.sm_100a.cubin kernel_substring [top]"""
import collections
import csv
import re
import subprocess
import sys

csv_path, cubin, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
sass = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
lines = sass.splitlines()
# the function's section
start = next(i for i, l in enumerate(lines) if l.startswith(".text.") and kname in l and l.endswith(":"))
off2line, cur = {}, None
for l in lines[start + 1:]:
    if l.startswith(".text.") and l.endswith(":"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        off2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csv_path)))
hdr = rows[1]
S = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
addrs = [int(r[0], 16) for r in data]
# first kernel instance only: addresses contiguous from the minimum
base = addrs[0]
seen, inst = set(), []
for a, r in zip(addrs, data):
    if a in seen:
        break
    seen.add(a)
    inst.append((a - base, r))
by = collections.defaultdict(lambda: [0.0, collections.Counter(), ""])
tot = 0.0
for off, r in inst:
    key = off2line.get(off, ("?", 0))
    v = float(r[S] or 0)
    tot += v
    e = by[key]
    e[0] += v
    for i in stall_cols:
        try:
            e[1][hdr[i][6:]] += float(r[i] or 0)
        except ValueError:
            pass
src = {}
print(f"{len(inst)} instructions, {tot:.0f} samples")
for key, (v, c, _) in sorted(by.items(), key=lambda t: -t[1][0])[:top]:
    reasons = ", ".join(f"{k}={x / max(v, 1):.0%}" for k, x in c.most_common(3))
    print(f"{v / tot:6.1%}  {key[0]}:{key[1]:<5d} {reasons}")
