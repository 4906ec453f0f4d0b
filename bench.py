#!/usr/bin/env python
"""Benchmark of the PackKV decode-time hot path on B200.

Metric (BASELINE.json): fused decompress+GEMV K/V throughput in fp16-equivalent
GB/s (SPEC.md:475 accounting: B*Hkv*L*D*2 bytes per kind per step), set next to
cuBLAS fp16 GEMV (torch.matmul) on the uncompressed cache, plus the
compression ratio.

Workload at N=1 (BASELINE.json configs[1], "config B"): Llama-3-8B GQA layer,
8 KV heads / 32 query heads, head_dim 128, 32768-token context, batch 8,
synthetic Gaussian KV with injected outlier channels, codec
rel_k 0.1 / rel_v 0.2, pack 16, block 64, repack none.

A step = fused K scores for every query head + fused V output for every query
head over the whole compressed cache of the layer (all inputs resident in
HBM); at N > 1 every rank owns its own (sequence, kv-head) shard of the same
size (weak scaling) and the per-head outputs are all-gathered over NCCL.
The per-step working set (~230 MB of compressed blocks) exceeds the 126 MB L2.

`--impl reference` times the reference algorithm's CPU path (the numpy
restatement of SPEC.md in oracle/, the reference ships no runnable code) on a
bounded sample of the same workload with all host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused decompress+GEMV K/V GB/s-equiv vs cuBLAS fp16 GEMV; compression ratio"
UNIT = "GB/s (fp16-equivalent)"

CONFIGS = {
    # key: (batch, kv_heads, q_heads, head_dim, tokens, description)
    "A": (1, 32, 32, 128, 4096, "Llama-2-7B single layer, MHA 32x128, 4K tokens, batch 1"),
    "B": (8, 8, 32, 128, 32768, "Llama-3-8B GQA (8 kv / 32 q heads), 32K context, batch 8, 1 layer"),
    "D": (8, 52, 52, 128, 32768, "LLaMA-30B shape (52 heads x 128), 32K context, batch 8, 15 layers (~105 GB fp16 "
                                 "K+V)"),
    "E": (16, 8, 64, 128, 131072, "Llama-3-70B GQA (8 kv / 64 q heads), 128K context, batch 16, 1 layer"),
    "C": (1, 40, 40, 128, 6144, "Llama-2-13B streaming decode: 40 layers x 40 heads x 128, batch 1, 2K prefill "
                                "then 4K append+attend steps"),
}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic():
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons = [], 0
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        rs = [n for bit, n in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": rs,
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------- CPU arm
def _cpu_unit(args):
    """One (sequence, kv-head) unit through the CPU oracle: compress (untimed),
    then the SPEC per-head fused K and V calls for its G query heads (timed)."""
    seed, L, D, G = args
    import numpy as np
    from oracle import packkv_oracle as O
    rng = np.random.default_rng(seed)
    K = O.gen_gauss_outlier(rng, L, D, max(1, D * 4 // 128))[:, None, :]
    V = O.gen_gauss_outlier(rng, L, D, max(1, D // 128))[:, None, :]
    st = O.OracleStore(1, 1, D)
    st.compress_batch(0, K, V)
    q = rng.standard_normal((G, D)).astype(np.float32)
    t0 = time.perf_counter()
    for g in range(G):
        s, _ = O.fused_k_scores(st, 0, 0, q[g])
        w = O.softmax64(s / math.sqrt(D)).astype(np.float32)
        O.fused_v_output(st, 0, 0, w)
    return time.perf_counter() - t0


def cpu_baseline(cfg, units: int, L: int, steps: int = 1):
    """Times the oracle (kind "port") on `units` units of L tokens, one process
    per unit on every host core (PACKKV_THREADS-style worker pool)."""
    import multiprocessing as mp
    B, Hkv, Hq, D, _, _ = cfg
    G = Hq // Hkv
    cores = min(units, len(os.sched_getaffinity(0)))
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        times = []
        for s in range(steps):
            t0 = time.perf_counter()
            pool.map(_cpu_unit, [(1000 * s + u, L, D, G) for u in range(units)])
            times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    logical = units * 2 * L * D * 2
    return {"value": logical / t / 1e9, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{units} (sequence, kv-head) units x {L} tokens, G={G} query heads each, "
                      f"SPEC per-head fused_k_scores + fused_v_output (oracle/packkv_oracle.py, numpy), "
                      f"{units} processes", "seconds_per_step": t}


def parity_sample(cfg, L: int = 4096):
    """Part of the cpu_baseline leg: one (sequence, kv-head) unit of the bench
    distribution compressed by the CPU oracle and by the device, then the
    device's fused K, fused V and folded-softmax attention against the oracle's
    f64 naive results.  Reports stream/CR bit-exactness and max abs / norm-rel
    errors (north star: "max abs/rel error reported")."""
    import numpy as np
    import torch
    from oracle import packkv_oracle as O
    from paper_2512_24449_b200 import fused_kernels as F
    from paper_2512_24449_b200.attention_sim import attention_decode_batched
    from paper_2512_24449_b200.kv_store import CompressedStore
    B, Hkv, Hq, D, _, _ = cfg
    G = Hq // Hkv
    rng = np.random.default_rng(2024)
    K = O.gen_gauss_outlier(rng, L, D, max(1, D * 4 // 128))[:, None, :]
    V = O.gen_gauss_outlier(rng, L, D, max(1, D // 128))[:, None, :]
    ref = O.OracleStore(1, 1, D)
    ref.compress_batch(0, K, V)
    st = CompressedStore(1, 1, D)
    st.compress_batch(0, K, V)
    q = rng.standard_normal((1, G, D)).astype(np.float32)
    s = F.fused_k_scores_batched(st, 0, torch.from_numpy(q)).cpu().numpy()[0]
    rs = np.stack([O.naive_k_scores(ref, 0, 0, q[0, g]) for g in range(G)])
    w = np.stack([O.softmax64(rs[g] / math.sqrt(D)) for g in range(G)]).astype(np.float32)
    o = F.fused_v_output_batched(st, 0, torch.from_numpy(w[None])).cpu().numpy()[0]
    ro = np.stack([O.naive_v_output(ref, 0, 0, w[g]) for g in range(G)])
    a = attention_decode_batched(st, 0, torch.from_numpy(q)).cpu().numpy()[0]
    ra = np.stack([O.naive_v_output(ref, 0, 0, O.softmax64(rs[g] / math.sqrt(D))) for g in range(G)])

    def err(x, r):
        e = np.abs(x.astype(np.float64) - r)
        return {"max_abs": float(e.max()), "max_rel_to_norm": float(e.max() / np.abs(r).max()),
                "pass": bool(e.max() <= 1e-3 * np.abs(r).max())}
    phys = sum(e.byte_len for e in ref.directory)
    return {"sample": f"1 (sequence, kv-head) unit x {L} tokens of the bench distribution, G={G}; "
                      "oracle = oracle/packkv_oracle.py (f64 naive GEMVs over its own compressed store)",
            "stream_bit_exact": st[0].stream_bytes(0) == ref.layer_stream(0),
            "cr_wire_equal": sum(int(x) for x in st[0].tables()[1].ravel()) == phys,
            "tolerance": "max|gpu - f64| <= 1e-3 * max|f64| (SPEC.md:454,463)",
            "fused_k": err(s, rs), "fused_v": err(o, ro), "attention": err(a, ra)}


def run_reference(args, rank, world):
    """The reference's CPU path (the oracle port: the reference ships no runnable
    code) on a bounded sample of the configured workload, every host core busy.
    Each timed step is one pass over the sample; the line reports the steps it
    actually timed.  The sample's GB/s-equivalent is the workload's: units are
    independent and cost O(tokens), so throughput does not depend on how many
    units or tokens are sampled ("extrapolated" in the line)."""
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    B, Hkv, Hq, D, L, desc = cfg
    cores = len(os.sched_getaffinity(0))
    units = cores
    Ls = min(L, 8192)
    cpu_baseline(cfg, units, 1024, 1)  # untimed warm-up (fork, imports, numpy)
    budget_s, t_used, steps_done, times = 120.0, 0.0, 0, []
    want = max(1, args.steps)
    while steps_done < want and (steps_done == 0 or t_used + times[-1] < budget_s):
        cb = cpu_baseline(cfg, units, Ls, 1)
        times.append(cb["seconds_per_step"])
        t_used += times[-1]
        steps_done += 1
    t = statistics.median(times)
    value = units * 2 * Ls * D * 2 / t / 1e9
    cb.update({"value": value, "seconds_per_step": t, "steps_timed": steps_done})
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
            "steps": steps_done, "steps_requested": args.steps, "warmup": 1, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"config {args.config}: {desc}", "sample_tokens_per_unit": Ls,
                       "sample_units": units,
                       "value_basis": (f"extrapolated: GB/s-equivalent of a bounded sample ({units} of the "
                                       f"{B * Hkv} (sequence, kv-head) units x {Ls} of {L} tokens) per timed "
                                       "step; units are independent and cost O(tokens), so the throughput "
                                       "carries over to the full workload"),
                       "step_budget_s": budget_s},
            "cpu_baseline": cb, "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def build_store(cfg, rank, repack="none", chunk=4096):
    import torch
    from paper_2512_24449_b200.kv_store import CompressedStore
    from paper_2512_24449_b200.tensor_model import gauss_outlier
    B, Hkv, Hq, D, L, _ = cfg
    st = CompressedStore(1, Hkv, D, batch=B, repack=repack, max_tokens=L, check=False)
    for t0 in range(0, L, chunk):
        T = min(chunk, L - t0)
        k = gauss_outlier((B, T, Hkv, D), n_outlier=4, seed=17 + 7919 * rank + t0)
        v = gauss_outlier((B, T, Hkv, D), n_outlier=1, seed=29 + 7919 * rank + t0)
        st.compress_batch(0, k, v)
    torch.cuda.synchronize()
    st.check_errors()
    return st


def compressor_bench(cfg, rank, T=4096, appends=128):
    """The append-time compressor: prefill of T tokens per
    sequence into a fresh store (quantize + encode + arena append of every
    block of every (sequence, kv-head), K and V), and single-token decode
    appends (staging copies; every 64th flushes a block-set).  CUDA-event timed;
    the fp16 inputs are resident in HBM."""
    import torch
    from paper_2512_24449_b200.attention_sim import GraphedDecodeLoop
    from paper_2512_24449_b200.kv_store import CompressedStore
    from paper_2512_24449_b200.tensor_model import gauss_outlier
    B, Hkv, Hq, D, L, _ = cfg
    k = gauss_outlier((B, T, Hkv, D), n_outlier=4, seed=101 + rank)
    v = gauss_outlier((B, T, Hkv, D), n_outlier=1, seed=103 + rank)
    kk = gauss_outlier((B, appends, Hkv, D), n_outlier=4, seed=107 + rank)
    vv = gauss_outlier((B, appends, Hkv, D), n_outlier=1, seed=109 + rank)
    res = {}
    for rep in range(2):  # first pass warms the allocator and the library
        st = CompressedStore(1, Hkv, D, batch=B, max_tokens=T + 2 * appends, check=False)
        st[0]._ensure((T + 2 * appends) // 64)  # arena reserved for the worst case up front (allocation is not compression)
        torch.cuda.synchronize()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        torch.cuda.nvtx.range_push("prefill")
        st.compress_batch(0, k, v)
        torch.cuda.nvtx.range_pop()
        e1.record()
        torch.cuda.synchronize()
        packed = int(st[0].tail.item())  # compressed bytes written by the prefill
        for t in range(appends):
            st.append_token(0, kk[:, t], vv[:, t])
        e2.record()
        # a serving decode step: append this step's K/V token (a block completes
        # every 64 steps, on the device), then attention -- one graph replay
        dstep = GraphedDecodeLoop(st, Hq, layers=[0], headroom=16)
        qd = torch.randn((1, B, Hq, D), device="cuda")
        ktok = [kk[:, t].reshape(1, B, 1, Hkv, D).contiguous() for t in range(appends)]
        vtok = [vv[:, t].reshape(1, B, 1, Hkv, D).contiguous() for t in range(appends)]
        dstep.step(ktok[0], vtok[0], qd)  # first capture (module loading, warm-up) untimed
        e3, e4 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e3.record()
        for t in range(1, appends):
            dstep.step(ktok[t], vtok[t], qd)
        e4.record()
        torch.cuda.synchronize()
        pre_ms, app_ms, step_ms = e0.elapsed_time(e1), e1.elapsed_time(e2), e3.elapsed_time(e4)
    fp16_in = 2 * B * T * Hkv * D * 2
    res = {"prefill_tokens": B * T, "prefill_ms": round(pre_ms, 3),
           "prefill_tokens_per_s": round(B * T / (pre_ms * 1e-3)),
           "prefill_fp16_in_gbs": round(fp16_in / (pre_ms * 1e-3) / 1e9, 1),
           # HBM traffic of the single-pass compressor: the f16 input read once, the
           # packed blocks written once
           "prefill_hbm_gbs": round((fp16_in + packed) / (pre_ms * 1e-3) / 1e9, 1),
           "prefill_hbm_frac": round((fp16_in + packed) / (pre_ms * 1e-3) / 1e9 / load_peaks()[0], 3),
           "prefill_bound": "issue (f32 quantization + bit-packing per element), not HBM",
           "append_us_per_token": round(app_ms * 1e3 / appends, 2),
           "decode_step_us": round(step_ms * 1e3 / (appends - 1), 2),
           "decode_step_captures": dstep.captures - 1,
           "decode_step_context": T + 2 * appends,
           "note": f"batch {B} x {Hkv} kv-heads x {D}, K and V, repack none; appends include "
                   f"{appends // 64} block-set flushes (host-driven launches); arena reserved before the "
                   f"timed prefill; decode_step = attention_sim.GraphedDecodeLoop (stage token + device-side "
                   f"block flush + attention in one graph replay; no re-capture at block completions) at "
                   f"~{T // 1024}K context"}
    del st
    torch.cuda.empty_cache()
    return res


def cublas_baseline(cfg, rank, reps=10):
    """torch.matmul fp16 (fp32 accumulate) GEMV on the uncompressed cache
    (PAPER.md:836), both operand orientations (cuBLAS picks different kernels
    for them; the best is the baseline), and the time an fp16 GEMV would take
    reading the cache at the measured HBM peak."""
    import torch
    from paper_2512_24449_b200.tensor_model import gauss_outlier
    B, Hkv, Hq, D, L, _ = cfg
    G = Hq // Hkv
    U = B * Hkv
    Kf = torch.empty((U, L, D), dtype=torch.float16, device="cuda")
    Vf = torch.empty((U, L, D), dtype=torch.float16, device="cuda")
    for t0 in range(0, L, 4096):
        T = min(4096, L - t0)
        Kf[:, t0:t0 + T] = gauss_outlier((B, T, Hkv, D), n_outlier=4, seed=17 + 7919 * rank + t0).permute(0, 2, 1, 3).reshape(U, T, D)
        Vf[:, t0:t0 + T] = gauss_outlier((B, T, Hkv, D), n_outlier=1, seed=29 + 7919 * rank + t0).permute(0, 2, 1, 3).reshape(U, T, D)
    q = torch.randn((U, D, G), device="cuda").half()
    qt = q.transpose(1, 2).contiguous()                                   # [U, G, D]
    w = torch.softmax(torch.randn((U, G, L), device="cuda"), -1).half()
    wt = w.transpose(1, 2).contiguous()                                   # [U, L, G]
    res = {}
    torch.cuda.nvtx.range_push("cublas")
    legs = (("k", lambda: torch.matmul(Kf, q)),                          # [U,L,D] x [U,D,G]
            ("k_t", lambda: torch.matmul(qt, Kf.transpose(1, 2))),        # [U,G,D] x [U,D,L]
            ("v", lambda: torch.matmul(w, Vf)),                           # [U,G,L] x [U,L,D]
            ("v_t", lambda: torch.matmul(Vf.transpose(1, 2), wt)))        # [U,D,L] x [U,L,G]
    for name, fn in legs:
        for _ in range(3):
            fn()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[name + "_us"] = statistics.median(ts) * 1e3
    torch.cuda.nvtx.range_pop()
    res["k_best_us"] = min(res["k_us"], res["k_t_us"])
    res["v_best_us"] = min(res["v_us"], res["v_t_us"])
    peak = load_peaks()[0]
    cache = U * L * D * 2
    res["k_fp16_at_hbm_peak_us"] = (cache + U * D * G * 2 + U * L * G * 2) / (peak * 1e3)
    res["v_fp16_at_hbm_peak_us"] = (cache + U * L * G * 2 + U * G * D * 2) / (peak * 1e3)
    del Kf, Vf
    torch.cuda.empty_cache()
    return res


# config -> (layers, split, scaling) of the decode-step bench (BASELINE.json configs;
# SURVEY §8 config key): B weak-scales by batch (the driver's default, N = 1 is the
# metric's config), D is the 15-layer ~105 GB LLaMA-30B variant with a strong batch
# split, E is Llama-3-70B head-sharded as strong scaling; C is the streaming decode
# (run_streaming) and A the reference's CPU-runnable case.
MODES = {"A": (1, "batch", "weak"), "B": (1, "batch", "weak"), "D": (15, "batch", "strong"),
         "E": (1, "head", "strong")}


def build_local_store(cfg, part, layers, rank, chunk=4096):
    """This rank's (sequence, kv-head) units of every layer, synthetic KV of the
    config shape (tensor_model.gauss_outlier: 4 / 1 outlier channels per kv head)."""
    import torch
    from paper_2512_24449_b200.kv_store import CompressedStore
    from paper_2512_24449_b200.tensor_model import gauss_outlier
    B, Hkv, Hq, D, L, _ = cfg
    Bl, Hl = part.local_batch, part.local_heads
    st = CompressedStore(layers, Hl, D, batch=Bl, max_tokens=L, check=False)
    for l in range(layers):
        for t0 in range(0, L, chunk):
            T = min(chunk, L - t0)
            seed = 17 + 7919 * rank + 104729 * l + t0
            st.compress_batch(l, gauss_outlier((Bl, T, Hl, D), n_outlier=4, seed=seed),
                              gauss_outlier((Bl, T, Hl, D), n_outlier=1, seed=seed + 12))
    torch.cuda.synchronize()
    st.check_errors()
    return st


def init_dist(local, world, backend):
    import torch
    import torch.distributed as dist
    ndev = torch.cuda.device_count()
    if backend == "nccl":
        if local >= ndev:  # one NCCL rank per GPU: never two ranks on one device
            raise SystemExit(f"LOCAL_RANK {local} >= {ndev} visible GPUs (NCCL needs one rank per GPU)")
    else:
        local = local % max(1, ndev)
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        # one line per rank: the communicator each rank joined (rank, size, device)
        probe = torch.ones(1, device="cuda")
        dist.all_reduce(probe)
        print(json.dumps({"comm_init": {"rank": dist.get_rank(), "nranks": dist.get_world_size(),
                                        "backend": dist.get_backend(), "device": f"cuda:{local}",
                                        "gpu": torch.cuda.get_device_name(local),
                                        "nranks_ok": int(probe.item()) == world}}), file=sys.stderr, flush=True)
    return local


def max_over_ranks(vals, world):
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def run_streaming(args, rank, world, local, backend):
    """Config C (BASELINE.json configs[2]): streaming decode on the Llama-2-13B
    shape -- 40 layers x 40 heads x 128, batch 1, a 2K-token prefill, then 4K
    decode steps; each step appends one K/V token to every layer (SPEC.md:365-373,
    a block completes every 64 steps) and attends with that layer's query over
    everything so far.  One CUDA graph per step holds all 40
    layers' stage + device-side flush + fused attention (GraphedDecodeLoop).
    W warm-up decode steps are untimed; the remaining appends are timed
    (tokens/s).  At N > 1 every rank runs its own replica (the stream is one
    sequence: it does not shard)."""
    import torch
    import torch.distributed as dist
    from paper_2512_24449_b200.attention_sim import GraphedDecodeLoop
    from paper_2512_24449_b200.kv_store import CompressedStore
    from paper_2512_24449_b200.tensor_model import gauss_outlier
    Ly, H, D, T0, NT = 40, 40, 128, 2048, args.stream_steps
    B, Hq = 1, 40
    st = CompressedStore(Ly, H, D, batch=B, max_tokens=T0 + NT, check=False)
    for l in range(Ly):
        st.compress_batch(l, gauss_outlier((B, T0, H, D), n_outlier=4, seed=11 + l + 97 * rank),
                          gauss_outlier((B, T0, H, D), n_outlier=1, seed=13 + l + 97 * rank))
    loop = GraphedDecodeLoop(st, Hq, headroom=16)
    kin, vin, qin = loop.inputs()
    g = torch.Generator(device="cuda")
    g.manual_seed(5 + rank)
    # the decode tokens are generated 64 steps at a time into a ring (what a model
    # would produce); q is a fixed set of 16 per-layer queries cycled over the steps
    qs = torch.randn((16, Ly, B, Hq, D), device="cuda", generator=g)
    kr = torch.empty((64, Ly, B, 1, H, D), dtype=torch.float16, device="cuda")
    vr = torch.empty_like(kr)

    def refill(t):
        kr.copy_(gauss_outlier((64, Ly, B, 1, H, D), n_outlier=4, seed=1000 + t).view_as(kr))
        vr.copy_(gauss_outlier((64, Ly, B, 1, H, D), n_outlier=1, seed=2000 + t).view_as(vr))

    W = min(args.warmup, NT - 1)
    t = 0
    refill(0)
    while t < W:  # warm-up decode steps (first capture, module loading): untimed appends
        loop.step(kr[t % 64], vr[t % 64], qs[t % 16])
        t += 1
        if t % 64 == 0:
            refill(t)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ctx0 = T0 + t
    sampler = ClockSampler(local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with sampler:
        e0.record()
        while t < NT:
            if t % 64 == 0:
                refill(t)  # inside the timed region: the model would produce these tokens anyway
            loop.step(kr[t % 64], vr[t % 64], qs[t % 16])
            t += 1
        e1.record()
        torch.cuda.synchronize()
    timed = NT - W
    ms = e0.elapsed_time(e1)
    ms = max_over_ranks([ms], world)[0]
    # bytes: every step reads the whole cache of every layer once for K and once for V
    logical = sum(Ly * 2 * B * H * (ctx0 + i + 1) * D * 2 for i in range(timed))
    value = world * logical / (ms * 1e-3) / 1e9
    tok_s = world * timed / (ms * 1e-3)
    # e2e through the public API from HOST buffers: pinned k, v, q per step
    # copied into the loop, the per-layer outputs copied back
    E2E = min(256, max(64, args.steps))
    kh = kr[:1].expand(E2E, *kr.shape[1:]).cpu().pin_memory()
    vh = vr[:1].expand(E2E, *vr.shape[1:]).cpu().pin_memory()
    qh = qs[:1].expand(E2E, *qs.shape[1:]).cpu().pin_memory()
    oh = torch.empty((Ly, B, Hq, D)).pin_memory()
    st2 = CompressedStore(Ly, H, D, batch=B, max_tokens=T0 + E2E + 64, check=False)
    for l in range(Ly):
        st2.compress_batch(l, gauss_outlier((B, T0, H, D), n_outlier=4, seed=11 + l),
                           gauss_outlier((B, T0, H, D), n_outlier=1, seed=13 + l))
    loop2 = GraphedDecodeLoop(st2, Hq, headroom=16)
    loop2.step(kh[0].cuda(), vh[0].cuda(), qh[0].cuda(), out=oh)  # captures with the host output buffer
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    for i in range(1, E2E):
        # pinned host k/v/q -> the graph's input buffers (copy engine); every layer's output
        # stored straight to pinned host memory by the attention kernels (zero-copy)
        loop2.step(kh[i], vh[i], qh[i], out=oh)
    a1.record()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks([a0.elapsed_time(a1) / (E2E - 1)], world)[0]
    e2e_logical = Ly * 2 * B * H * (T0 + E2E // 2) * D * 2
    st.check_errors()
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": timed,
            "warmup": W, "ms_per_step": round(ms / timed, 5), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8->f32", "data": "synthetic gaussian + outlier channels (BASELINE.md §3)",
            "config": {"workload": f"config C: {CONFIGS['C'][-1]}", "layers": Ly, "kv_heads": H, "q_heads": Hq,
                       "head_dim": D, "batch": B, "prefill_tokens": T0, "decode_steps": NT,
                       "context_timed": [ctx0, T0 + NT], "rel_k": 0.1, "rel_v": 0.2, "pack_size": 16,
                       "block": 64, "repack": "none",
                       "parallelism": f"replicas x{world} (one stream per GPU; the path does not shard)",
                       "l2": "per-step working set (40 layers of compressed K+V) exceeds the 126 MB L2"},
            "tokens_per_s": round(tok_s, 1), "us_per_token": round(ms * 1e3 / timed, 2),
            "step": ("GraphedDecodeLoop: one CUDA-graph replay per token: for each of the 40 layers "
                     "pkv_append_flush (token staged + device-side block completion, one launch) + "
                     "pkv_attention_decode (single pass: attn_fused_kernel + attn_merge_kernel); "
                     f"re-captures {loop.captures} (every {loop.headroom * 64} tokens)"),
            "e2e": {"value": round(world * e2e_logical / (e2e_ms * 1e-3) / 1e9, 2), "unit": UNIT,
                    "h2d_bytes_per_step": Ly * B * (2 * H * D * 2 + Hq * D * 4),
                    "d2h_bytes_per_step": Ly * B * Hq * D * 4,
                    "tokens_per_s": round(world * 1e3 / e2e_ms, 1), "ms_per_step": round(e2e_ms, 5),
                    "path": "GraphedDecodeLoop.step(k, v, q, out=host) from pinned host k/v/q; the attention kernels store every layer's output to the pinned host buffer inside the graph"},
            "gpu_launches": timed * (Ly * 3 + 1), "clocks": sampler.summary(),
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="B", choices=sorted(CONFIGS))
    ap.add_argument("--stream-steps", type=int, default=4096, help="config C: decode steps after the prefill")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cublas", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    # PKV_BENCH_BACKEND=gloo (structural test of the N > 1 path with several ranks on
    # one device); production runs use NCCL, one rank per GPU
    backend = os.environ.get("PKV_BENCH_BACKEND", "nccl")
    local = init_dist(local, world, backend)
    if args.config == "C":
        run_streaming(args, rank, world, local, backend)
        if world > 1:
            dist.destroy_process_group()
        return

    def gather_into(dst, src):
        if backend == "nccl":
            dist.all_gather_into_tensor(dst, src)
        else:
            dist.all_gather(list(dst.view(world, *src.shape).unbind(0)), src)
    from paper_2512_24449_b200 import fused_kernels as F
    from paper_2512_24449_b200 import sharding as S

    cfg = CONFIGS[args.config]
    B, Hkv, Hq, D, L, desc = cfg
    G = Hq // Hkv
    layers, split, scaling = MODES[args.config]
    if scaling == "weak":  # the job holds B sequences per GPU, sharded by sequence
        part = S.plan_partition(B * world, Hkv, world, rank, prefer="batch")
    else:                  # the config's fixed job, split `split`-wise over the ranks
        part = S.plan_partition(B, Hkv, world, rank, prefer=split)
    Bl, Hl = part.local_batch, part.local_heads
    Hql = Hl * G
    st = build_local_store(cfg, part, layers, rank)
    ls = st[0]
    tabs = [st[l].tables()[1] for l in range(layers)]
    phys_k = sum(int(t[0].astype(np.int64).sum()) for t in tabs)
    phys_v = sum(int(t[1].astype(np.int64).sum()) for t in tabs)
    nblocks_k = sum(int(t[0].size) for t in tabs)
    logical_kind = layers * Bl * Hl * L * D * 2          # per rank, all layers
    cr_k_wire, cr_v_wire = logical_kind / phys_k, logical_kind / phys_v
    full = layers * Bl * Hl * (L // 64) * 64 * D * 2
    cr_k = full / (phys_k - 8 * nblocks_k)
    cr_v = full / (phys_v - 8 * nblocks_k)
    res_bytes = layers * Bl * Hl * ls.nres_h * D * 2
    alg_k = (phys_k + res_bytes) / layers + Bl * Hql * D * 4 + Bl * Hql * L * 4   # per launch (one layer)
    alg_v = (phys_v + res_bytes) / layers + Bl * Hql * L * 4 + Bl * Hql * D * 4

    # HBM held by the compressed layers (SPEC.md:499 reports peak allocation)
    tail = sum(int(st[l].tail.item()) for l in range(layers))
    side = sum(t.numel() * t.element_size() for l in range(layers)
               for t in (st[l].blk_off, st[l].blk_len, st[l].perm, st[l].nblk, st[l].nres, st[l].stage))
    mem = {"fp16_kv_bytes": 2 * logical_kind, "arena_used_bytes": tail,
           "arena_capacity_bytes": sum(st[l].capacity for l in range(layers)),
           "tables_and_staging_bytes": side, "hbm_ratio_vs_fp16": round(2 * logical_kind / (tail + side), 3),
           "peak_allocated_bytes_after_build": int(torch.cuda.max_memory_allocated()),
           "note": "arena capacity is geometric-growth reservation; CompressedStore.shrink_to_fit() releases it"}
    qs = torch.randn((layers, Bl, Hql, D), device="cuda")
    scores = torch.empty((Bl, Hql, L), device="cuda")
    out = torch.empty((layers, Bl, Hql, D), device="cuda")
    F.fused_k_scores_batched(st, 0, qs[0], out=scores)
    w = torch.softmax(scores / math.sqrt(D), -1).contiguous()
    gathered = torch.empty((world * layers * Bl, Hql, D), device="cuda") if world > 1 else None

    def run_k():
        for l in range(layers):
            F.fused_k_scores_batched(st, l, qs[l], out=scores)

    def run_v():
        for l in range(layers):
            F.fused_v_output_batched(st, l, w, out=out[l])

    for _ in range(args.warmup):
        run_k()
        run_v()
    # the timed launches replay CUDA graphs of the fused K and V calls of every
    # layer (a decode step's launches without Python launch overhead)
    gk, gv = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(gk):
        run_k()
    with torch.cuda.graph(gv):
        run_v()
    for _ in range(args.warmup):
        gk.replay()
        gv.replay()
    K = args.steps
    # working sets below ~L2 size (config A) are flushed between timed steps by
    # writing 256 MB; ms_per_step is then the sum of the K and V launch times
    l2_flush = phys_k + phys_v + 2 * Bl * Hql * L * 4 < 160 * 2 ** 20
    flush_buf = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda") if l2_flush else None
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include timed/ selects these launches
    with sampler:
        e_start = torch.cuda.Event(enable_timing=True)
        e_end = torch.cuda.Event(enable_timing=True)
        e_start.record()
        for i in range(K):
            if l2_flush:
                flush_buf.zero_()
            evs[i][0].record()
            gk.replay()
            evs[i][1].record()
            gv.replay()
            evs[i][2].record()
            if world > 1:
                gather_into(gathered, out.view(-1, Hql, D))
        e_end.record()
        torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    if world > 1:
        dist.barrier()
    ms = e_start.elapsed_time(e_end) / K
    k_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
    v_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in evs)
    ms, k_ms, v_ms = max_over_ranks([ms, k_ms, v_ms], world)
    if l2_flush:
        ms = k_ms + v_ms
    value = world * 2 * logical_kind / (ms * 1e-3) / 1e9

    # ---- decode attention per layer: the single pass
    # (attn_fused_kernel, one launch + the counter memset) against the
    # three-launch path (fused K with score maxima, fused V on exp(s - M),
    # finalize), both graph-replayed
    from paper_2512_24449_b200.attention_sim import attention_decode_batched
    a_out = torch.empty((Bl, Hql, D), device="cuda")
    a_scores = torch.empty((Bl, Hql, (L + 3) // 4 * 4), device="cuda")

    def attn(single):
        for l in range(layers):
            attention_decode_batched(st, l, qs[l], out=a_out, scores=None if single else a_scores,
                                     single_pass=single)
    attn_us = {}
    for single in (True, False):
        attn(single)
        ga = torch.cuda.CUDAGraph()
        with torch.cuda.graph(ga):
            attn(single)
        for _ in range(args.warmup):
            ga.replay()
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(K):
            if l2_flush:
                flush_buf.zero_()
            ga.replay()
        t1.record()
        torch.cuda.synchronize()
        attn_us["single" if single else "three"] = max_over_ranks([t0.elapsed_time(t1) * 1e3 / K / layers], world)[0]
        del ga
    alg_attn = alg_k + alg_v - 2 * Bl * Hql * L * 4   # no score rows written or read
    if l2_flush:
        attn_us = {k: None for k in attn_us}  # the flush is inside the timed loop: no clean number

    # ---- e2e through the public API: host q (this rank's shard) -> sharded
    # decode (fused K, softmax, fused V, NCCL all-gather) per layer -> host output
    decs = [S.ShardedDecoder(part, S.cuda_local_attention(st, l), Hq, D) for l in range(layers)]
    q_host = torch.randn((layers, Bl, Hql, D)).pin_memory()
    out_host = torch.empty((layers, world * Bl * Hql * D)).pin_memory()

    def e2e_step():
        for l in range(layers):
            # pinned host q in, pinned host out: with one rank both move inside the decode
            # graph (zero-copy over PCIe, GraphedAttention); with more, out is copied after the gather
            decs[l].step(q_host[l], out=out_host[l])

    for _ in range(args.warmup):
        e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    for _ in range(K):
        e2e_step()
    a1.record()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks([a0.elapsed_time(a1) / K], world)[0]
    e2e_value = world * 2 * logical_kind / (e2e_ms * 1e-3) / 1e9
    from paper_2512_24449_b200.attention_sim import single_pass_preferred
    e2e_attn = "single-pass" if single_pass_preferred(st, st[0].nblk_h) else "three-launch"

    peak, peak_src = load_peaks()
    dom = "k" if k_ms >= v_ms else "v"
    dom_ms = (k_ms if dom == "k" else v_ms) / layers          # one launch (one layer)
    alg = alg_k if dom == "k" else alg_v
    achieved = alg / (dom_ms * 1e-3) / 1e9
    traffic = load_traffic().get(f"{args.config}_{dom}")

    cub = None
    if not args.no_cublas:
        del scores
        cub = cublas_baseline((Bl, Hl, Hql, D, L, desc), rank)
    comp = compressor_bench(cfg, rank) if not args.no_cublas and args.config in ("A", "B") else None
    cb = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ncores = len(os.sched_getaffinity(0))
        cb = cpu_baseline(cfg, units=ncores, L=min(L, 8192), steps=1)
        cb["value_basis"] = ("extrapolated: GB/s-equivalent of the bounded sample; units are independent "
                             "and cost O(tokens)")
        cb["parity"] = parity_sample(cfg)
    if rank == 0:
        kind_layer = logical_kind / layers
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "u8->f32", "data": "synthetic gaussian + outlier channels (BASELINE.md §3)",
            "config": {"workload": f"config {args.config}: {desc}", "batch": B if scaling == "strong" else B * world,
                       "kv_heads": Hkv, "q_heads": Hq, "head_dim": D, "tokens": L, "layers": layers,
                       "per_rank": {"batch": Bl, "kv_heads": Hl, "q_heads": Hql},
                       "rel_k": 0.1, "rel_v": 0.2, "pack_size": 16, "block": 64, "repack": "none",
                       "parallelism": f"(batch, kv-head) shards x{world} ({part.mode} split, {scaling} scaling), "
                                      f"{'NCCL' if backend == 'nccl' else backend} all-gather of outputs",
                       "global_batch": B if scaling == "strong" else B * world,
                       "l2": ("working set below L2: 256 MB written between timed steps, ms_per_step = K + V "
                              "launch times" if l2_flush else
                              "per-step working set (compressed K+V blocks) exceeds the 126 MB L2")},
            "compression_ratio": {"k": round(cr_k, 4), "v": round(cr_v, 4), "k_wire": round(cr_k_wire, 4),
                                  "v_wire": round(cr_v_wire, 4)},
            "kernels": {"fused_k_us": round(k_ms * 1e3 / layers, 2), "fused_v_us": round(v_ms * 1e3 / layers, 2),
                        "per": "one launch = one layer on this rank's units",
                        "fused_k_gbs_equiv": round(kind_layer / (k_ms / layers * 1e-3) / 1e9, 1),
                        "fused_v_gbs_equiv": round(kind_layer / (v_ms / layers * 1e-3) / 1e9, 1),
                        "fused_k_gbs_physical": round(alg_k / (k_ms / layers * 1e-3) / 1e9, 1),
                        "fused_v_gbs_physical": round(alg_v / (v_ms / layers * 1e-3) / 1e9, 1)},
            "roofline": {"bound": "hbm", "kernel": f"fused_{dom}", "achieved": round(achieved, 1), "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic, "algorithmic_bytes_per_launch": int(alg),
                         "frac_vs_nominal_8000_gbs": round(achieved / 8000.0, 4)},
            "attention": None if attn_us["single"] is None else {
                "single_pass_us": round(attn_us["single"], 2), "three_launch_us": round(attn_us["three"], 2),
                "single_pass_gbs_physical": round(alg_attn / (attn_us["single"] * 1e-6) / 1e9, 1),
                "single_pass_frac": round(alg_attn / (attn_us["single"] * 1e-6) / 1e9 / peak, 4),
                "single_pass_gbs_equiv": round(2 * kind_layer / (attn_us["single"] * 1e-6) / 1e9, 1),
                "algorithmic_bytes_per_launch": int(alg_attn),
                "per": "one layer: softmax(q K^T / sqrt(d)) V over this rank's units, graph-replayed; single "
                       "pass = attn_fused_kernel + attn_merge_kernel, three launch = fused K + fused V + finalize"},
            "e2e": {"value": round(e2e_value, 2), "unit": UNIT, "h2d_bytes_per_step": layers * Bl * Hql * D * 4,
                    "d2h_bytes_per_step": layers * world * Bl * Hql * D * 4,
                    "path": "sharding.ShardedDecoder.step(q_host, out=host) (public API) per layer on the pinned "
                            "host q shard: one CUDA-graph replay of the decode attention "
                            f"(attention_sim.GraphedAttention, {e2e_attn} path per single_pass_preferred) that reads q "
                            "from host memory (zero-copy, prescaled) and, with one rank, writes the output to host "
                            "memory; with more ranks all-gather of per-head outputs, then D2H out",
                    "ms_per_step": round(e2e_ms, 5)},
            "memory": mem,
            # scaling with and without the all-gather -- the same
            # whole-job metric from the K + V launch times alone (max over ranks)
            "value_without_collective": round(world * 2 * logical_kind / ((k_ms + v_ms) * 1e-3) / 1e9, 2),
            "gpu_launches": 3 * K * layers,
            "clocks": sampler.summary(),
        }
        if cub:
            line["cublas"] = {"k_us": round(cub["k_us"], 2), "k_transposed_us": round(cub["k_t_us"], 2),
                              "v_us": round(cub["v_us"], 2), "v_transposed_us": round(cub["v_t_us"], 2),
                              "k_best_us": round(cub["k_best_us"], 2), "v_best_us": round(cub["v_best_us"], 2),
                              "k_gbs_equiv": round(kind_layer / (cub["k_best_us"] * 1e-6) / 1e9, 1),
                              "v_gbs_equiv": round(kind_layer / (cub["v_best_us"] * 1e-6) / 1e9, 1),
                              "speedup_k": round(cub["k_best_us"] / (k_ms * 1e3 / layers), 3),
                              "speedup_v": round(cub["v_best_us"] / (v_ms * 1e3 / layers), 3),
                              "fp16_gemv_at_hbm_peak_us": {"k": round(cub["k_fp16_at_hbm_peak_us"], 2),
                                                           "v": round(cub["v_fp16_at_hbm_peak_us"], 2)},
                              "speedup_vs_fp16_at_hbm_peak": {
                                  "k": round(cub["k_fp16_at_hbm_peak_us"] / (k_ms * 1e3 / layers), 3),
                                  "v": round(cub["v_fp16_at_hbm_peak_us"] / (v_ms * 1e3 / layers), 3)},
                              "note": "per layer; best of both operand orientations of torch.matmul fp16 "
                                      "(cuBLAS), and an ideal fp16 GEMV reading the uncompressed cache at the "
                                      "measured HBM peak"}
        if comp:
            line["compressor"] = comp
        if cb:
            line["cpu_baseline"] = cb
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
