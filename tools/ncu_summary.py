"""Summarise an ncu report: key metrics per kernel + SASS opcode histogram (run here, no GPU)."""
import csv, subprocess, sys, io
from collections import Counter
rep = sys.argv[1]
blocks = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]; ix = {h: i for i, h in enumerate(hdr)}
want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Block Limit Shared Mem", "Block Limit Registers", "No Eligible", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "L2 Hit Rate", "L1/TEX Hit Rate"]
for r in rows[1:]:
    if r[ix["Metric Name"]] in want:
        print(r[ix["Kernel Name"]][:45], "|", r[ix["Metric Name"]], r[ix["Metric Value"]], r[ix["Metric Unit"]])
for k in sys.argv[3:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + k],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]; ii = h.index("Instructions Executed"); isrc = h.index("Source")
    st = h.index("Warp Stall Sampling (All Samples)")
    c = Counter(); s = Counter(); tot = 0; stot = 0
    seen = set()
    for r in rows[2:]:
        if r and r[0] in seen:  # the source page lists each SASS row twice
            continue
        if r: seen.add(r[0])
        if len(r) <= ii: continue
        try: n = int(r[ii])
        except ValueError: continue
        src = r[isrc].strip(); op = src.split()[0] if src else "?"
        if op.startswith("@"): op = src.split()[1]
        op = op.split(".")[0]
        c[op] += n; tot += n; sv = int(r[st] or 0); s[op] += sv; stot += sv
    print(f"== {k}: warp-instr total {tot}  per block {tot / blocks:.0f}")
    for op, n in c.most_common(22):
        print(f"  {op:10s} {n / blocks:9.1f}/blk {n / tot * 100:5.1f}%  stall {s[op] / max(stot,1) * 100:5.1f}%")
