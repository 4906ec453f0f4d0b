"""Top stall sites from an ncu report's source page: python ncu_src.py rep kernel_idx reason [n] [sass|cuda]"""
import csv, subprocess, sys
rep, kidx, reason = sys.argv[1], int(sys.argv[2]), sys.argv[3]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 25
mode = sys.argv[5] if len(sys.argv) > 5 else "sass"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", mode],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
ks = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
start = ks[kidx]
end = ks[kidx + 1] if kidx + 1 < len(ks) else len(rows)
h = rows[start + 1]
body = rows[start + 2:end]
ci = h.index(reason) if reason in h else h.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[ci] or 0) for r in body)
allc = h.index("Warp Stall Sampling (All Samples)")
totall = sum(float(r[allc] or 0) for r in body)
print(rows[start][1][:90], f"total {reason} {tot:.0f} of all {totall:.0f}")
src = h.index("Source")
addr = h.index("Address") if "Address" in h else 0
for r in sorted(body, key=lambda r: -float(r[ci] or 0))[:n]:
    print(f"{float(r[ci] or 0):8.0f} {float(r[allc] or 0):8.0f}  {r[addr][-5:]} {r[src].strip()[:110]}")
