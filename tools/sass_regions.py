"""Summarise an ncu source-page SASS csv: instructions per block grouped by
execution count (loop nesting) and the top stall instructions."""
import csv, collections, sys
path, nblocks = sys.argv[1], float(sys.argv[2])
rows = list(csv.reader(open(path)))
h = rows[1]
ai, si, ei, wi = h.index('Address'), h.index('Source'), h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)')
seen, data = set(), []
for r in rows[2:]:
    if len(r) <= ei or not r[ei].isdigit() or r[ai] in seen:
        continue
    seen.add(r[ai])
    data.append((r[ai], r[si].strip(), int(r[ei]), int(r[wi] or 0)))
tot = sum(d[2] for d in data)
print(f"total inst/block {tot / nblocks:.1f}   samples {sum(d[3] for d in data)}")
byc = collections.defaultdict(lambda: [0, 0, 0])
for a, s, e, w in data:
    b = byc[e]; b[0] += 1; b[1] += e; b[2] += w
for c, (n, v, w) in sorted(byc.items(), key=lambda x: -x[1][1])[:12]:
    print(f"exec {c:9d} ({c / nblocks:6.2f}/blk): {n:5d} instrs  {v / nblocks:7.1f} inst/blk  samples {w}")
# regions: consecutive instructions with the same exec count
print("--- regions (consecutive same-count runs >= 8 instrs)")
run = []
def flush():
    if len(run) >= 8:
        c = run[0][2]
        ops = collections.Counter((x[1].split()[1] if x[1].startswith('@') else x[1].split()[0]).split('.')[0] for x in run)
        print(f"  {len(run):4d} instrs x {c / nblocks:6.2f}/blk = {len(run) * c / nblocks:7.1f}  samples {sum(x[3] for x in run):5d}  {dict(ops.most_common(6))}")
for d in data:
    if run and d[2] != run[-1][2]:
        flush(); run = []
    run.append(d)
flush()
