"""Per-region instruction / stall breakdown of one kernel in an ncu report.
python sass_regions.py rep kernel_index [blocks_per_launch] [region_size]"""
import csv, subprocess, sys, collections
rep, ki = sys.argv[1], int(sys.argv[2])
nb = float(sys.argv[3]) if len(sys.argv) > 3 else 32768
rsz = int(sys.argv[4]) if len(sys.argv) > 4 else 100
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
ks = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
st = ks[ki]; en = ks[ki + 1] if ki + 1 < len(ks) else len(rows)
name = rows[st][1]; h = rows[st + 1]; body = rows[st + 2:en]
ci = h.index("Warp Stall Sampling (All Samples)"); ie = h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
print(name[:100])
tot = sum(float(r[ci] or 0) for r in body); inst = sum(float(r[ie] or 0) for r in body) / nb
print(f"samples {tot:.0f}  inst/block {inst:.0f}")
for lo in range(0, len(body), rsz):
    seg = body[lo:lo + rsz]
    s = sum(float(r[ci] or 0) for r in seg); n = sum(float(r[ie] or 0) for r in seg) / nb
    if s < 0.01 * tot and n < 5:
        continue
    rs = collections.Counter()
    for r in seg:
        for c in reasons:
            rs[c[6:]] += float(r[h.index(c)] or 0)
    print(f"{lo:5d} samples {s / tot * 100:5.1f}%  inst {n:6.1f}  " + " ".join(f"{k}:{v / max(s, 1) * 100:.0f}" for k, v in rs.most_common(4)))
with open(f"/tmp/sass_{ki}.txt", "w") as f:
    for i, r in enumerate(body):
        f.write(f"{i:5d} {r[ci]:>5} {float(r[ie] or 0) / nb:7.2f} {r[1].strip()[:100]}\n")
