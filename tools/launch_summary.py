"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv)."""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0].isdigit()]
agg = collections.OrderedDict()
for r in rows:
    name = r[4]
    short = name.split('(')[0].replace('void ', '').replace('<unnamed>::', '')[:60]
    v = float(r[14])
    a = agg.setdefault(short, [0, 0.0])
    a[0] += 1; a[1] += v
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':62s} {'n':>4s} {'mean us':>9s} {'share':>6s}")
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:62s} {n:4d} {v / n / 1000 if v > 1e4 else v / n:9.2f} {100 * v / tot:5.1f}%")
