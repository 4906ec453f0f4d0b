"""Stall samples / instructions aggregated per CUDA source line (ncu source page, sass+cuda view).
usage: python tools/exp/ncu_lines.py REPORT [N] [metric]"""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
metric = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg, hdr, fn, cur = {}, None, None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fn = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    if r[0]:
        cur = (fn, r[0], r[1].strip()[:100])
    try:
        v = float(r[hdr.index(metric)] or 0)
        ie = float(r[hdr.index("Instructions Executed")] or 0)
    except ValueError:
        continue
    a = agg.setdefault(cur, [0.0, 0.0])
    a[0] += v
    a[1] += ie
tot = sum(a[0] for a in agg.values()) or 1
itot = sum(a[1] for a in agg.values()) or 1
print(f"total {metric}: {tot:.0f}; instructions {itot:.0f}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{a[0]:7.0f} {100 * a[0] / tot:5.1f}%  inst {100 * a[1] / itot:5.1f}%  {k[0]}:{k[1]} {k[2]}")
