"""Per-CUDA-source-line instruction counts and stall samples from an ncu
source page exported with --print-source cuda,sass."""
import csv, collections, sys
path, nblk = sys.argv[1], float(sys.argv[2])
rows = list(csv.reader(open(path)))
agg, inst, src = collections.Counter(), collections.Counter(), {}
for r in rows[3:]:
    if len(r) < 8 or not r[0].strip().isdigit():
        continue
    ln = int(r[0]); src[ln] = r[1]
    try:
        agg[ln] += int(r[4]); inst[ln] += int(r[7])
    except ValueError:
        pass
tot, ti = sum(agg.values()), sum(inst.values())
print(f"samples {tot}  inst/blk {ti / nblk:.1f}")
for ln, v in sorted(inst.items(), key=lambda x: -x[1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    print(f"{v / nblk:7.1f} {agg[ln]:5d}  L{ln}: {src.get(ln, '').strip()[:100]}")
