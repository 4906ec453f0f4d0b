"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv)."""
import csv, sys, collections
allrows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(r for r in allrows if r[0] == "ID")
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
rows = [r for r in allrows if r[0].isdigit()]
agg = collections.OrderedDict()
for r in rows:
    name = r[ik]
    short = name.split('(')[0].replace('void ', '').replace('<unnamed>::', '')[:60]
    v = float(r[iv].replace(",", ""))
    a = agg.setdefault(short, [0, 0.0])
    a[0] += 1; a[1] += v
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':62s} {'n':>4s} {'mean us':>9s} {'share':>6s}")
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:62s} {n:4d} {v / n / 1000 if v > 1e4 else v / n:9.2f} {100 * v / tot:5.1f}%")
