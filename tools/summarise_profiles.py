"""Summarise the ncu artefacts gpurun brought back (gpurun_out/) into the
tracked profiles/ directory.  Usage: python tools/summarise_profiles.py r01"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import Counter, defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def ncu_csv(args):
    r = subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout
    lines = [l for l in r.splitlines() if l.startswith('"')]
    return list(csv.reader(io.StringIO("\n".join(lines))))


def short(name):
    return name.split("(")[0].replace("void ", "").replace("<unnamed>::", "")[:60]


def launches(tag):
    path = os.path.join(OUT, "launches.csv")
    if not os.path.exists(path):
        return None
    allrows = [r for r in csv.reader(open(path)) if r]
    hdr = next(r for r in allrows if r[0] == "ID")
    ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    rows = [r for r in allrows if r[0].isdigit()]
    per = defaultdict(list)
    for r in rows:
        if r[im] == "gpu__time_duration.sum":
            per[short(r[ik])].append(float(r[iv].replace(",", "")))
    tot = sum(sum(v) for v in per.values())
    lines = [f"# ncu launch list ({tag}): per-kernel device time, cold-cache and serialised",
             "", "Command: `ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include timed/ "
             "--nvtx-include cublas/ python bench.py --steps 2 --warmup 3 --no-cpu-baseline` (the 2 timed steps: "
             "fused K, fused V + finalize; and the cuBLAS fp16 GEMV comparison leg)", "",
             "| kernel | launches | mean us | share of listed time |", "|---|---|---|---|"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | {sum(v) / tot * 100:.1f}% |")
    open(os.path.join(PROF, f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")
    return per


def full(tag):
    rep = os.path.join(OUT, "prof_full.ncu-rep")
    if not os.path.exists(rep):
        return
    rows = ncu_csv(["-i", rep, "--page", "raw", "--csv"])
    h = rows[0]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active"]
    stalls = [i for i, x in enumerate(h) if "smsp__average_warps_issue_stalled" in x and "per_issue_active" in x]
    lines = [f"# ncu --set full summary ({tag})", "",
             "Command: `ncu --set full --clock-control none --import-source on -k regex:fast_kernel -s 4 -c 2 "
             "python bench.py --steps 1 --warmup 3 --no-cublas --no-cpu-baseline` (config B, one K and one V launch)", ""]
    traffic = {}
    for r in rows[2:]:
        name = short(r[h.index("Kernel Name")])
        lines += [f"## `{name}`", "", "| metric | value |", "|---|---|"]
        for m in want:
            if m in h:
                lines.append(f"| {m} | {r[h.index(m)]} |")
        top = sorted(((float(r[i] or 0), h[i]) for i in stalls), reverse=True)[:6]
        lines.append("")
        lines.append("Top warp stall reasons (warps per issue): " + ", ".join(
            f"{n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {v:.2f}"
            for v, n in top))
        lines.append("")
        kind = "k" if "fused_k" in name else "v"
        rd = float(r[h.index("dram__bytes_read.sum")] or 0)
        wr = float(r[h.index("dram__bytes_write.sum")] or 0)
        unit_r = r[h.index("dram__bytes_read.sum")]
        traffic[f"B_{kind}"] = {"read": rd, "write": wr}
    # SASS opcode mix per kernel
    for k in ("fused_k", "fused_v"):
        srows = ncu_csv(["-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + k])
        if len(srows) < 3:
            continue
        hh = srows[1]
        ii, isrc = hh.index("Instructions Executed"), hh.index("Source")
        c, seen = Counter(), set()
        for r in srows[2:]:
            if len(r) <= ii or r[0] in seen:
                continue
            seen.add(r[0])
            try:
                n = int(r[ii])
            except ValueError:
                continue
            op = r[isrc].split()[0] if r[isrc].split() else "?"
            if op.startswith("@"):
                op = r[isrc].split()[1]
            c[op.split(".")[0]] += n
        tot = sum(c.values())
        lines += [f"### SASS mix `{k}` ({tot} warp-instructions per launch)", "",
                  " ".join(f"{op} {n / tot * 100:.1f}%" for op, n in c.most_common(14)), ""]
    open(os.path.join(PROF, f"{tag}_ncu_full.md"), "w").write("\n".join(lines) + "\n")
    # dram traffic per launch (bytes), read by bench.py for roofline.traffic
    tpath = os.path.join(OUT, "traffic.csv")
    per = {}
    if os.path.exists(tpath):
        allrows = [r for r in csv.reader(open(tpath)) if r]
        hdr = next(r for r in allrows if r[0] == "ID")
        ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
        for r in allrows:
            if not r[0].isdigit():
                continue
            kind = "k" if "fused_k" in r[ik] else "v"
            per.setdefault(kind, {})[r[im]] = float(r[iv].replace(",", ""))
    js = {}
    for kind, m in per.items():
        js[f"B_{kind}"] = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    js["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch of the fused kernels on config B, "
                   f"from gpurun_out/traffic.csv ({tag}); units bytes")
    json.dump(js, open(os.path.join(PROF, "ncu_traffic.json"), "w"), indent=1)


def single(tag):
    """profiles/<tag>_single_pass.md: the single-pass attention kernel's ncu
    summary and the config C decode-step launch list (per layer)."""
    lines = [f"# Single-pass decode attention and the decode loop ({tag})", ""]
    rep = os.path.join(OUT, "prof_single.ncu-rep")
    if os.path.exists(rep):
        rows = ncu_csv(["-i", rep, "--page", "raw", "--csv"])
        h = rows[0]
        want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
                "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
                "launch__registers_per_thread", "smsp__cycles_active.avg", "sm__cycles_elapsed.avg"]
        stalls = [i for i, x in enumerate(h) if "smsp__average_warps_issue_stalled" in x and "per_issue_active" in x]
        lines += ["`ncu --set full` of attn_fused_kernel<1> on config B (tools/exp/kbench.py s)", ""]
        for r in rows[2:]:
            lines += [f"## `{short(r[h.index('Kernel Name')])}`", "", "| metric | value |", "|---|---|"]
            lines += [f"| {m} | {r[h.index(m)]} |" for m in want if m in h]
            top = sorted(((float(r[i] or 0), h[i]) for i in stalls), reverse=True)[:7]
            lines += ["", "Top warp stall reasons (warps per issue): " + ", ".join(
                f"{n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {v:.2f}"
                for v, n in top), ""]
    path = os.path.join(OUT, "launches_C.csv")
    if os.path.exists(path):
        allrows = [r for r in csv.reader(open(path)) if r]
        hdr = next(r for r in allrows if r[0] == "ID")
        ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
        ks = [(short(r[ik]), float(r[iv].replace(",", ""))) for r in allrows if r[0].isdigit()]
        tail = ks[-40 * 10 * 3:]
        per = defaultdict(list)
        for k, v in tail:
            per[k].append(v)
        lines += ["## Config C decode step: launch list (steady state, cold-cache, serialised)", "",
                  "`ncu --metrics gpu__time_duration.sum python bench.py --config C --stream-steps 200` (the last "
                  "launches: 40 layers per step)", "", "| kernel | launches | mean us |", "|---|---|---|"]
        for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.2f} |")
    open(os.path.join(PROF, f"{tag}_single_pass.md"), "w").write("\n".join(lines) + "\n")


def compressor(tag):
    """profiles/<tag>_compressor.md: prefill launch list (time, DRAM bytes) and
    the full-set summary of the warp-per-block compressor kernels."""
    path = os.path.join(OUT, "comp_launches.csv")
    if not os.path.exists(path):
        return
    allrows = [r for r in csv.reader(open(path)) if r]
    hdr = next(r for r in allrows if r[0] == "ID")
    ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    per = defaultdict(lambda: defaultdict(list))
    for r in allrows:
        if r[0].isdigit():
            per[short(r[ik])][r[im]].append(float(r[iv].replace(",", "")))
    lines = [f"# Compressor profile ({tag})", "",
             "Prefill of 4096 tokens x batch 8 x 8 kv-heads x 128 (K and V, repack none) in bench.py's compressor "
             "leg; `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --nvtx "
             "--nvtx-include prefill/` (cold cache, serialised; both prefill repetitions listed)", "",
             "| kernel | launches | mean us | DRAM read MB | DRAM write MB |", "|---|---|---|---|---|"]
    for k, m in per.items():
        t = m.get("gpu__time_duration.sum", [0])
        rd = m.get("dram__bytes_read.sum", [0])
        wr = m.get("dram__bytes_write.sum", [0])
        lines.append(f"| `{k}` | {len(t)} | {sum(t) / len(t) / 1e3:.1f} | {sum(rd) / len(rd) / 1e6:.1f} | "
                     f"{sum(wr) / len(wr) / 1e6:.1f} |")
    rep = os.path.join(OUT, "prof_comp.ncu-rep")
    if os.path.exists(rep):
        rows = ncu_csv(["-i", rep, "--page", "raw", "--csv"])
        h = rows[0]
        want = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
                "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
        lines += ["", "## ncu --set full (one launch each)", ""]
        for r in rows[2:]:
            lines += [f"### `{short(r[h.index('Kernel Name')])}`", "", "| metric | value |", "|---|---|"]
            lines += [f"| {m} | {r[h.index(m)]} |" for m in want if m in h]
            lines.append("")
    open(os.path.join(PROF, f"{tag}_compressor.md"), "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PROF, exist_ok=True)
    launches(tag)
    full(tag)
    single(tag)
    compressor(tag)
    print(open(os.path.join(PROF, "ncu_traffic.json")).read())
