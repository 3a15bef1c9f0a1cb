"""Summarise an `ncu --page source --csv` (SASS) export: stall samples by
opcode and the top stalled instructions with their dominant stall reasons.
    python tools/ncu_src_summary.py file.csv [top]"""
import csv, sys, collections

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(path)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
stall_cols = [h for h in hdr if h.startswith("stall_") or "Stall" in h and h not in
              ("Warp Stall Sampling (All Samples)", "Warp Stall Sampling (Not-issued Samples)")]
S = "Warp Stall Sampling (All Samples)"
tot = sum(float(d[S] or 0) for d in data)
byop = collections.Counter()
for d in data:
    op = d["Source"].split()[0] if d["Source"].split() else "?"
    if op.startswith("@"):
        op = d["Source"].split()[1]
    byop[op.split(".")[0]] += float(d[S] or 0)
print(f"total samples {tot:.0f}; instructions {len(data)}")
for op, v in byop.most_common(15):
    print(f"  {op:12s} {v / tot:6.1%}")
print("stall columns:", len(stall_cols))
agg = collections.Counter()
for d in data:
    for c in stall_cols:
        try:
            agg[c] += float(d[c] or 0)
        except ValueError:
            pass
for c, v in agg.most_common(12):
    print(f"  {c:50s} {v / max(tot, 1):6.1%}")
print("top instructions:")
for d in sorted(data, key=lambda d: -float(d[S] or 0))[:top]:
    rs = sorted(((float(d[c] or 0), c) for c in stall_cols if (d[c] or "0").replace(".", "").isdigit()), reverse=True)[:2]
    print(f"  {float(d[S]) / tot:6.2%} {d['Address'][-5:]} {d['Source'].strip()[:60]:60s} " +
          " ".join(f"{c.replace('stall_', '')}={v:.0f}" for v, c in rs))
