#!/usr/bin/env python
"""ReAttention decode-step benchmark (BASELINE.json metric: decode µs/token/layer at 1M ctx;
K-scan HBM GB/s vs ~8 TB/s).

A step is one single-layer ReAttention decode step (the reference's attend_step,
engine.hpp:43-114) for one new token: group-mean q·Kᵀ scan + top-k over the middle
(selection.hpp:168), vote + spans (selection.hpp:252-349), scope assembly (scope.hpp:37), RoPE at
compact positions and finite-scope attention (attend.hpp:25) — LLaMA-3.1-8B head geometry
(32 q / 8 kv heads, d=128), bf16 KV cache of 1,048,576 tokens, selection defaults
(k=4, k'=127, m=32, g=32, local=4096), batch 1.  Inputs are synthetic (splitmix64 uniform
[-1,1), the same generator on device and host) and resident in HBM; each step gets a fresh
query.  The 2.1 GB K scan is far larger than the 126 MB L2, and L2 is additionally flushed
before every timed step by reading a 256 MiB buffer (outside the timed intervals; a write
flush would leave ~126 MB of dirty lines whose write-back lands inside the next step).

--impl reference times the reference's own CPU attend_step (oracle/_ref: the reference
headers compiled in place) on the host cores, on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "ReAttention decode µs/token/layer at 1M ctx"
UNIT = "µs/token/layer"
CTX = 1 << 20
N_KV, N_HEAD, D = 8, 32, 128
ROPE_BASE = 500000.0
WINDOW = 8192
DTYPE = ("bf16 KV storage; scores fp32 in the reference's exact 8-lane order (bit-identical "
         "top-k); decode attention logits fp32 with ex2.approx.ftz softmax weights and f64 "
         "softmax state (A, B) across chunks -- the reference computes f64 logits "
         "(attend.hpp:50-69); outputs held to 1e-6 of it")

# The BASELINE.json decode configs, built identically by this bench, tools/bench_configs.py
# and the parity tests that pin the timed plans to the oracle (tests/test_timed_paths_gpu.py).
DECODE_CONFIGS = {
    1: dict(n_head=32, n_kv=8, total=32 * 1024, dtype="f32",
            workload="LLaMA-3.1-8B heads (32/8), 32K tokens, fp32 cache, batch 1, 1 layer"),
    2: dict(n_head=32, n_kv=8, total=128 * 1024, dtype="bf16",
            workload="LLaMA-3.1-8B heads (32/8), 128K tokens, bf16, batch 1, 1 layer"),
    4: dict(n_head=32, n_kv=8, total=1 << 20, dtype="bf16",
            workload="LLaMA-3.1-8B heads (32/8), 1M tokens, bf16, batch 1, 1 layer"),
    5: dict(n_head=24, n_kv=8, total=1 << 22, dtype="bf16",
            workload="LLaMA-3.2-3B heads (24/8), 4M tokens, bf16, batch 1, 1 layer"),
}


def config_seeds(cid: int) -> tuple[int, int, int]:
    """(K seed, V seed, query seed) of a decode config's synthetic inputs."""
    return 1000 + 10 * cid, 1001 + 10 * cid, 5000 + 10 * cid


def build_decode(ctx, cid: int, total: int | None = None, extra_rows: int = 0):
    """The decode workload of config `cid` on one GPU: a synthetic cache (splitmix64 uniform
    [-1, 1), bf16-rounded for bf16 caches), the rotary table and the CUDA-graph plan that
    bench.py times.  Returns (cache, rope, plan, cfg, meta)."""
    from paper_2407_15176_b200 import native as N
    c = DECODE_CONFIGS[cid]
    total = total or c["total"]
    cfg = N.SelectionConfig()
    dt = N.F32 if c["dtype"] == "f32" else N.BF16
    cache = N.Cache(ctx, c["n_kv"], D, cfg.l_global, cfg.l_local, total + extra_rows, dt)
    ks, vs, _ = config_seeds(cid)
    ctx.synth_uniform(cache.keys_tensor(), ks)
    ctx.synth_uniform(cache.values_tensor(), vs)
    cache.set_total(total)
    rope = N.Rope(ctx, D, ROPE_BASE, WINDOW)
    plan = N.Plan(ctx, cache, rope, 1, c["n_head"], cfg)
    return cache, rope, plan, cfg, dict(c, total=total, cid=cid)


def load_read_ceiling() -> dict | None:
    """The read-only bandwidth of K1's own access pattern without its arithmetic (TMA boxes,
    ring and CTA count of the scan; tools/micro/hbm_read.cu, committed measurement)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_hbm_read_ceiling.txt")) as f:
            for line in f:
                if line.startswith("tma 256r x 3 ef1 144 CTAs"):
                    return {"gbs": float(line.split()[7]),
                            "source": "profiles/r2_hbm_read_ceiling.txt (tools/micro/hbm_read.cu)"}
    except Exception:
        pass
    return None


def load_traffic() -> dict | None:
    """dram read+write bytes per scan launch from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_decode_1m.json")) as f:
            p = json.load(f)
        return {"bytes": int(p["traffic_bytes"]), "source": p["source"]}
    except Exception:
        return None


def load_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm_gbs": float(p["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------------
def _ref_cache(ctx_tokens: int, n_kv: int, keys_np, values_np):
    import numpy as np
    import oracle_bind as ob
    lib = ob.ref()
    if lib is None:
        raise RuntimeError("oracle/_ref not built (needs /root/reference at build time)")
    t0 = time.perf_counter()
    cache = lib.ref_cache_create(n_kv, D, 32, 4096, np.ascontiguousarray(keys_np).ravel(),
                                 np.ascontiguousarray(values_np).ravel(), ctx_tokens)
    return lib, cache, time.perf_counter() - t0


def _ref_step(lib, cache, q, n_head):
    import ctypes as C
    import numpy as np
    import oracle_bind as ob
    cfg = ob.SelectionConfig()
    out = np.zeros(n_head * D, np.float32)
    st = ob.StepStats()
    sb = np.zeros(cfg.k_prime, np.uint64)
    se = np.zeros(cfg.k_prime, np.uint64)
    rc = lib.ref_attend_step(cache, q, 1, n_head, cfg.k, cfg.k_prime, cfg.span_m,
                             cfg.tile_size, cfg.l_global, cfg.l_local, cfg.l_chunk,
                             cfg.span_mode, ROPE_BASE, WINDOW, 2, out, C.byref(st), sb, se)
    assert rc == 0


def reference_cpu(steps: int, warmup: int, threads: int, ctx_tokens: int, seed: int = 1000,
                  keys_np=None, values_np=None, single_reps: int = 5) -> dict:
    """The reference's own attend_step (oracle/_ref: its headers compiled in place) on the host
    cores, on the same workload (LLaMA-3.1-8B heads, the bf16-valued cache upcast to fp32):
      * latency: one thread pinned to one core (sched_setaffinity, as
        taskset), 1 warm-up + the median of `single_reps` single calls;
      * throughput: `threads` concurrent decode steps sharing the read-only cache
        (attend_step is pure and reentrant), `steps` rounds after `warmup`."""
    import numpy as np
    import synth
    if keys_np is None:
        n = N_KV * ctx_tokens * D
        keys_np = synth.uniform(seed, n, bf16=True).reshape(N_KV, ctx_tokens, D)
        values_np = synth.uniform(seed + 1, n, bf16=True).reshape(N_KV, ctx_tokens, D)
    lib, cache, build_s = _ref_cache(ctx_tokens, N_KV, keys_np, values_np)
    qs = [synth.uniform(seed + 100 + i, N_HEAD * D).reshape(1, -1) for i in range(max(threads, 1))]
    res = {"unit": UNIT, "kind": "reference", "cache_build_s": build_s}
    # ---- single-thread latency, pinned
    lat = None
    if single_reps > 0:
        try:
            old = os.sched_getaffinity(0)
            core = sorted(old)[-1]
            os.sched_setaffinity(0, {core})
        except (AttributeError, OSError):
            old, core = None, None
        try:
            _ref_step(lib, cache, qs[0], N_HEAD)  # warm-up
            ts = []
            for i in range(single_reps):
                t0 = time.perf_counter()
                _ref_step(lib, cache, qs[i % len(qs)], N_HEAD)
                ts.append(time.perf_counter() - t0)
        finally:
            if old is not None:
                os.sched_setaffinity(0, old)
        ts.sort()
        lat = ts[len(ts) // 2] * 1e6
        res["latency_1core"] = {"value": lat, "unit": UNIT, "cores": 1, "pinned_core": core,
                                "sample": f"1 warm-up + median of {single_reps} single attend_step "
                                          f"calls, one thread pinned to one core"}
    # ---- all-core throughput
    if steps > 0 and threads > 0:
        def one(i):
            _ref_step(lib, cache, qs[i], N_HEAD)

        def round_():
            ths = [threading.Thread(target=one, args=(i,)) for i in range(threads)]
            for t in ths:
                t.start()
            for t in ths:
                t.join()

        for _ in range(warmup):
            round_()
        t0 = time.perf_counter()
        for _ in range(steps):
            round_()
        wall = time.perf_counter() - t0
        res["throughput_all_cores"] = {
            "value": wall / (steps * threads) * 1e6, "unit": UNIT, "cores": threads,
            "sample": f"{steps} rounds x {threads} concurrent attend_step calls (1 token, 1 layer, "
                      f"{ctx_tokens} ctx, fp32 upcast of the bf16 cache) after {warmup} warm-up; "
                      f"cache build {build_s:.1f}s untimed",
            "steps_timed": steps * threads, "wall_s": wall}
    lib.ref_cache_destroy(cache)
    return res


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference_arm(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = args.cpu_threads or os.cpu_count() or 1
    # a step is one attend_step call (1 token, 1 layer, the BASELINE workload); K steps run as
    # ceil(K / threads) rounds of `threads` concurrent calls on the host cores, W likewise
    rounds = max(1, -(-args.steps // threads))
    warm_rounds = max(1, -(-args.warmup // threads))
    r = reference_cpu(rounds, warm_rounds, threads, CTX, single_reps=3)
    tp = r["throughput_all_cores"]
    line = {"impl": "reference", "metric": METRIC, "value": tp["value"], "unit": UNIT,
            "n_gpus": args.gpus, "steps": tp["steps_timed"], "warmup": warm_rounds * threads,
            "ms_per_step": tp["value"] / 1000.0, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32 (bf16-valued cache upcast)",
            "data": "synthetic (splitmix64 uniform, bf16-rounded)",
            "config": {"workload": "LLaMA-3.1-8B geometry decode, 1 layer, batch 1, 1M ctx",
                       "ctx": CTX, "n_head": N_HEAD, "n_kv": N_KV, "d": D,
                       "host_cpu": cpu_model()},
            "cpu_baseline": {"value": tp["value"], "unit": UNIT, "cores": threads,
                             "kind": "reference", "sample": tp["sample"],
                             "latency_1core": r.get("latency_1core")},
            "e2e": {"value": tp["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------
def _flush_buffer(torch, dev):
    """256 MiB of int64: `.sum()` READS it (an int64 reduction, no cast), evicting L2 with
    clean lines, so no write-back of the flush lands inside the next timed step."""
    return torch.empty(32 << 20, dtype=torch.int64, device=dev).fill_(1)


def time_plan(plan, qbank, stream, flush, steps: int, warmup: int, scan_too: bool = False):
    """Device time per replay (CUDA events on the plan's stream, L2 read-flushed before
    every timed step, a fresh resident query per step)."""
    import torch
    with torch.cuda.stream(stream):
        for i in range(warmup):
            plan.q.copy_(qbank[i % qbank.shape[0]:i % qbank.shape[0] + 1])
            plan.launch()
        plan.stats()
        torch.cuda.synchronize()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        for i in range(steps):
            flush.sum()
            j = (warmup + i) % qbank.shape[0]
            plan.q.copy_(qbank[j:j + 1])
            starts[i].record(stream)
            plan.launch()
            ends[i].record(stream)
        torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in zip(starts, ends)) / steps


def per_config_lines(ctx, stream, flush, peaks, cids, steps: int) -> list:
    """The other BASELINE decode configs on this GPU (step µs and fraction of HBM), so the
    driver's run records them beside the headline."""
    import torch
    out = []
    for cid in cids:
        try:
            cache, rope, plan, cfg, meta = build_decode(ctx, cid)
            _, _, qs = config_seeds(cid)
            qbank = torch.empty(steps + 5, meta["n_head"] * D, dtype=torch.float32,
                                device=f"cuda:{ctx.device}")
            ctx.synth_uniform(qbank, qs)
            ms = time_plan(plan, qbank, stream, flush, steps, 5)
            st = plan.stats()
            info = plan.info()
            esz = 4 if meta["dtype"] == "f32" else 2
            byts = info["scan_bytes"] + meta["n_kv"] * st.scope_len * 2 * D * esz
            gbs = byts / (ms * 1e-3) / 1e9
            out.append({"config": cid, "workload": meta["workload"], "us_per_token_layer": ms * 1e3,
                        "scope_len": st.scope_len, "algorithmic_bytes": byts, "step_gbs": gbs,
                        "frac_of_8tbs_nominal": gbs / 8000.0,
                        "frac_of_measured_copy_peak": gbs / peaks["hbm_gbs"],
                        "kernels_per_step": int(info["kernels_per_step"]), "steps": steps})
            del plan, cache, rope, qbank
            torch.cuda.empty_cache()
        except Exception as e:  # reported, never fatal for the headline
            out.append({"config": cid, "error": str(e)[:200]})
    return out


def batch_sweep_lines(ctx, stream, flush, batches, steps: int) -> list:
    """Config 5's batch dimension on this GPU (LLaMA-3.2-3B heads, 4M tokens per sequence,
    each sequence its own 17 GB cache): one BatchPlan graph per batch size, device time per
    replay over the batch (µs per token-layer per sequence)."""
    import torch
    from paper_2407_15176_b200 import native as N
    c = DECODE_CONFIGS[5]
    out = []
    cfg = N.SelectionConfig()
    rope = N.Rope(ctx, D, ROPE_BASE, WINDOW)
    caches = []
    try:
        for B in batches:
            while len(caches) < B:
                i = len(caches)
                cache = N.Cache(ctx, c["n_kv"], D, cfg.l_global, cfg.l_local, c["total"], N.BF16)
                ks, vs, _ = config_seeds(5)
                ctx.synth_uniform(cache.keys_tensor(), ks + 7919 * i)
                ctx.synth_uniform(cache.values_tensor(), vs + 7919 * i)
                cache.set_total(c["total"])
                caches.append(cache)
            bp = N.BatchPlan(ctx, caches[:B], rope, c["n_head"], cfg)
            qb = torch.empty(B, c["n_head"] * D, device=f"cuda:{ctx.device}")
            ctx.synth_uniform(qb, 5051)
            bp.q.copy_(qb)
            with torch.cuda.stream(stream):
                for _ in range(3):
                    bp.launch()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                tot = 0.0
                for _ in range(steps):
                    flush.sum()
                    e0.record(stream)
                    bp.launch()
                    e1.record(stream)
                    e1.synchronize()
                    tot += e0.elapsed_time(e1)
            ms = tot / steps
            info = bp.info()
            out.append({"config": 5, "batch": B, "ms_per_step": ms,
                        "us_per_token_layer_per_sequence": ms * 1e3 / B,
                        "scan_gbs": info["scan_bytes"] / (ms * 1e-3) / 1e9,
                        "kernels_per_step": int(info["kernels_per_step"])})
            del bp
    except Exception as e:  # (memory: 17 GB per sequence) reported, never fatal
        out.append({"config": 5, "error": str(e)[:200]})
    del caches
    torch.cuda.empty_cache()
    return out


def prefill_config3_line(ctx) -> dict:
    """Config 3: one layer's chunked prefill to 256K (tools/bench_prefill_layer.py)."""
    try:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import bench_prefill_layer as bpl
        a = argparse.Namespace(ctx=256 * 1024, chunk=4096, every=1, start=0, stop=1 << 30)
        r = bpl.run(ctx, a)
        r.pop("last_chunk", None)
        return r
    except Exception as e:
        return {"error": str(e)[:200]}


def run_ours(args) -> None:
    import torch

    from paper_2407_15176_b200 import native as N

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = f"cuda:{local}"
    ctx = N.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    cid = args.config
    n_e2e = max(10, args.steps // 4)
    # headroom for the end-to-end leg, whose steps append a row each (append + attend_step)
    cache, rope, plan, cfg, meta = build_decode(ctx, cid, total=args.ctx if cid == 4 else None,
                                                extra_rows=n_e2e + 8)
    info = plan.info()
    K, W = args.steps, args.warmup
    n_head = meta["n_head"]
    _, _, qseed = config_seeds(cid)
    qbank = torch.empty(K + W, n_head * D, dtype=torch.float32, device=dev)
    ctx.synth_uniform(qbank, qseed)
    flush = _flush_buffer(torch, dev)

    with ClockSampler(local) as clk:
        t_wall = time.perf_counter()
        ms_per_step = time_plan(plan, qbank, stream, flush, K, W)
        t_wall = time.perf_counter() - t_wall
    st = plan.stats()
    with torch.cuda.stream(stream):
        # dominant kernel alone (K scan), CUDA events on the launching stream
        n_scan = max(20, K // 4)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        scan_ms = 0.0
        for i in range(n_scan):
            flush.sum()
            s0.record(stream)
            plan.launch_scan()
            s1.record(stream)
            s1.synchronize()
            scan_ms += s0.elapsed_time(s1)
        scan_ms /= n_scan
        # end to end through the public C-ABI from pinned host memory, as a decoder calls it per
        # token and layer: this step's K/V rows appended to the cache (kv_cache.hpp:54-68)
        # inside the same graph, then the step (reattn_plan_step_host: H2D q, k, v; replay;
        # D2H out; synchronise).  The cache grows by one row per call.
        plan.set_append(True)
        qh = qbank[:1].cpu().pin_memory()
        oh = torch.empty_like(qh).pin_memory()
        kvw = meta["n_kv"] * D
        kh = torch.empty(kvw, dtype=torch.float32).pin_memory()
        vh = torch.empty(kvw, dtype=torch.float32).pin_memory()
        kh.copy_(torch.from_numpy(__import__("synth").uniform(77, kvw, bf16=True)))
        vh.copy_(torch.from_numpy(__import__("synth").uniform(78, kvw, bf16=True)))
        for _ in range(3):
            plan.step_host(qh, kh, vh, oh)
        t0 = time.perf_counter()
        for i in range(n_e2e):
            plan.step_host(qh, kh, vh, oh)
        e2e_us = (time.perf_counter() - t0) / n_e2e * 1e6

    peaks = load_peaks()
    scan_bytes = info["scan_bytes"]
    esz = 4 if meta["dtype"] == "f32" else 2
    scope_bytes = meta["n_kv"] * st.scope_len * 2 * D * esz
    achieved = scan_bytes / (scan_ms * 1e-3) / 1e9
    step_bytes = scan_bytes + scope_bytes
    line = {
        "metric": METRIC, "value": ms_per_step * 1000.0, "unit": UNIT, "n_gpus": 1,
        "steps": K, "warmup": W, "ms_per_step": ms_per_step, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": DTYPE,
        "data": "synthetic (splitmix64 uniform [-1,1), bf16), resident in HBM",
        "config": {"workload": meta["workload"] + (" (BASELINE.json metric; config 4 at 1 GPU)"
                                                   if cid == 4 else ""),
                   "config_id": cid, "ctx": meta["total"], "n_head": n_head, "n_kv": meta["n_kv"],
                   "d": D, "k": cfg.k, "k_prime": cfg.k_prime, "span_m": cfg.span_m,
                   "l_global": cfg.l_global, "l_local": cfg.l_local, "scope_len": st.scope_len,
                   "l2": "inputs >> L2 (2.1 GB scan at 1M); L2 flushed before each timed step by "
                         "READING a 256 MiB int64 buffer (outside the timed intervals; a read "
                         "flush leaves no dirty lines whose write-back would land in the step)",
                   "parallelism": "1 GPU"},
        "step_hbm_gbs": step_bytes / (ms_per_step * 1e-3) / 1e9,
        "step_frac_of_8tbs": step_bytes / (ms_per_step * 1e-3) / 1e9 / 8000.0,
        "step_frac_of_hbm": step_bytes / (ms_per_step * 1e-3) / 1e9 / peaks["hbm_gbs"],
        "roofline": {"bound": "hbm", "kernel": "scan_fast_kernel (K1)", "achieved": achieved,
                     "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                     "traffic": (load_traffic() or {}).get("bytes") if cid == 4 else None,
                     "traffic_source": (load_traffic() or {}).get("source") if cid == 4 else None,
                     "bytes_per_launch": scan_bytes,
                     "launch_us": scan_ms * 1000.0, "peak_source": peaks["source"],
                     "peak_note": "peak is the measured copy (read+write) bandwidth; the scan "
                                  "only reads, so frac can exceed 1",
                     "read_ceiling_gbs": (load_read_ceiling() or {}).get("gbs"),
                     "frac_of_read_ceiling": (achieved / load_read_ceiling()["gbs"]
                                              if load_read_ceiling() else None),
                     "read_ceiling_source": (load_read_ceiling() or {}).get("source"),
                     "share_of_step": scan_ms / ms_per_step},
        "e2e": {"value": e2e_us, "unit": UNIT,
                "h2d_bytes_per_step": n_head * D * 4 + 2 * meta["n_kv"] * D * 4,
                "d2h_bytes_per_step": n_head * D * 4,
                "path": "reattn_plan_step_host (C-ABI) on pinned host buffers: one graph launch "
                        "that reads q and the step's K/V rows from host memory (zero-copy kernel), "
                        "appends the rows, runs attend_step and writes the output back to host "
                        "memory; then synchronise.  The cache grows by one row per step"},
        "gpu_launches": int(info["kernels_per_step"]) * K,
        "kernels_per_step": int(info["kernels_per_step"]),
        "wall_s_timed_region": t_wall,
        "clocks": clk.summary(),
    }
    if not args.no_per_config:
        del plan, cache
        torch.cuda.empty_cache()
        others = [c for c in (1, 2, 4, 5) if c != cid]
        line["per_config"] = per_config_lines(ctx, stream, flush, peaks, others, args.per_config_steps)
        line["config5_batch_sweep_1gpu"] = batch_sweep_lines(ctx, stream, flush, (1, 2, 4, 8), 10)
        line["prefill_config3"] = prefill_config3_line(ctx)
    if not args.no_cpu_baseline and cid == 4:
        try:
            # the same synthetic cache, regenerated on the host in fp32 (bf16-rounded values)
            ks, vs, _ = config_seeds(cid)
            r = reference_cpu(args.cpu_steps, 1, args.cpu_threads or os.cpu_count() or 1,
                              meta["total"], seed=ks, single_reps=5)
            lat, tp = r["latency_1core"], r["throughput_all_cores"]
            line["cpu_baseline"] = {"value": lat["value"], "unit": UNIT, "cores": 1,
                                    "kind": "reference", "sample": lat["sample"],
                                    "throughput_all_cores": {k: tp[k] for k in ("value", "unit",
                                                                                 "cores", "sample")}}
        except Exception as e:  # the baseline is reported, never required
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    print(json.dumps(line), flush=True)


def run_sharded(args) -> None:
    """Configs 4 and 5 with the middle sequence-sharded over the ranks (one GPU each): local K
    scan, NCCL all-gather of (index, score) candidates, redundant exact merge + vote + spans,
    owned-row attention partials, NCCL all-gather of the partials, combine.  The library
    issues both collectives on its own NCCL communicator (reattn_shard_step, the C-ABI host
    path); the whole step replays as one CUDA graph.  --batch B runs B sequences per step."""
    import torch
    import torch.distributed as dist

    from paper_2407_15176_b200 import native as N
    from paper_2407_15176_b200 import sharded as S

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = f"cuda:{local}"
    stream = torch.cuda.Stream(device=dev)
    ctx = N.Context(local, stream=stream.cuda_stream)
    cid = args.config if args.config in (4, 5) else 4
    c = DECODE_CONFIGS[cid]
    n_head, n_kv = c["n_head"], c["n_kv"]
    cfg = N.SelectionConfig()
    total = args.ctx if cid == 4 else c["total"]
    segs = S.local_row_segments(total, cfg, world, rank)
    rows = sum(e - b for b, e in segs)
    comm = S.NcclComm(ctx, world, rank)
    rope = N.Rope(ctx, D, ROPE_BASE, WINDOW)
    steps_ = []
    keep = []
    for b_ in range(args.batch):
        cache = N.Cache(ctx, n_kv, D, cfg.l_global, cfg.l_local, rows, N.BF16)
        kt, vt = cache.keys_tensor(), cache.values_tensor()
        ks, vs, _ = config_seeds(cid)
        o = 0
        for b, e in segs:  # the rows of the global synthetic cache this rank holds
            for h in range(n_kv):
                ctx.synth_uniform(kt[h, o:o + e - b], ks + 7919 * b_, (h * total + b) * D)
                ctx.synth_uniform(vt[h, o:o + e - b], vs + 7919 * b_, (h * total + b) * D)
            o += e - b
        cache.set_total(rows)
        ops = S.NativeOps(ctx, cache, rope, n_head, cfg, total, world, rank)
        steps_.append(S.NcclDecodeStep(ops, comm))
        keep.append(cache)
    K, W = args.steps, args.warmup
    _, _, qs = config_seeds(cid)
    qbank = torch.empty(K + W, args.batch, n_head * D, dtype=torch.float32, device=dev)
    ctx.synth_uniform(qbank, qs)  # identical queries on every rank
    flush = _flush_buffer(torch, dev)
    g, ls = S.global_geometry(total, cfg.l_global, cfg.l_local)
    shard_len = S.shard_range(ls - g, cfg.span_m, world, rank)[1]

    def step(i):
        for b_, st_ in enumerate(steps_):
            st_.ops.q.copy_(qbank[i, b_:b_ + 1])
            st_.step()

    with torch.cuda.stream(stream):
        for i in range(W):
            step(i)
        st0, _ = steps_[0].ops.stats(cfg.k_prime)
        torch.cuda.synchronize()
        dist.barrier()
        for st_ in steps_:
            st_.capture()  # the whole step, NCCL all-gathers included, as one CUDA graph
        torch.cuda.synchronize()
        dist.barrier()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
        with ClockSampler(local) as clk:
            t_wall = time.perf_counter()
            for i in range(K):
                flush.sum()
                for b_, st_ in enumerate(steps_):
                    st_.ops.q.copy_(qbank[W + i, b_:b_ + 1])  # stage the resident queries
                starts[i].record(stream)
                for st_ in steps_:
                    st_.step()
                ends[i].record(stream)
            torch.cuda.synchronize()
            t_wall = time.perf_counter() - t_wall
        dist.barrier()
        ms = sum(a.elapsed_time(b) for a, b in zip(starts, ends)) / K
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_per_step = float(t.item())
        # this rank's K scan alone (events on the launching stream)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        scan_ms = 0.0
        n_scan = max(20, K // 4)
        for i in range(n_scan):
            flush.sum()
            s0.record(stream)
            steps_[0].ops.scan()
            s1.record(stream)
            s1.synchronize()
            scan_ms += s0.elapsed_time(s1)
        scan_ms /= n_scan
        t = torch.tensor([scan_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        scan_ms = float(t.item())
        # end to end through the C-ABI (reattn_shard_run_host: H2D q, graph, D2H out), per rank
        qh = qbank[0, 0:1].cpu().pin_memory()
        oh = torch.empty_like(qh).pin_memory()
        dist.barrier()
        n_e2e = max(10, K // 4)
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            for st_ in steps_:
                st_.run_host(qh, oh)
        e2e_us = (time.perf_counter() - t0) / n_e2e * 1e6
        t = torch.tensor([e2e_us], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_us = float(t.item())
    if rank == 0:
        peaks = load_peaks()
        scan_bytes = n_kv * shard_len * D * 2 * args.batch
        achieved = scan_bytes / (scan_ms * args.batch * 1e-3) / 1e9
        per_seq_us = ms_per_step * 1000.0 / args.batch
        line = {
            "metric": METRIC, "value": per_seq_us, "unit": UNIT, "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": ms_per_step, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": DTYPE,
            "data": "synthetic (splitmix64 uniform [-1,1), bf16), resident in HBM",
            "config": {"workload": c["workload"].replace("batch 1", f"batch {args.batch}") +
                                   ", middle sequence-sharded (config %d)" % cid,
                       "config_id": cid, "ctx": total, "n_head": n_head, "n_kv": n_kv, "d": D,
                       "batch": args.batch, "scope_len": st0.scope_len,
                       "shard_rows_rank0": shard_len,
                       "l2": "L2 read-flushed (256 MiB int64 sum) before each timed step",
                       "parallelism": f"sp{world} (library-owned NCCL communicator: all-gather "
                                      f"of candidates + partials, captured in the step graph)"},
            "roofline": {"bound": "hbm", "kernel": "scan_fast_kernel (K1, per-rank shard)",
                         "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / peaks["hbm_gbs"], "traffic": None,
                         "bytes_per_launch": scan_bytes // args.batch, "launch_us": scan_ms * 1000.0,
                         "peak_source": peaks["source"],
                         "share_of_step": scan_ms * args.batch / ms_per_step},
            "e2e": {"value": e2e_us / args.batch, "unit": UNIT,
                    "h2d_bytes_per_step": n_head * D * 4 * args.batch,
                    "d2h_bytes_per_step": n_head * D * 4 * args.batch,
                    "path": "reattn_shard_run_host (C-ABI + library NCCL) from pinned host"},
            "gpu_launches": 4 * K * args.batch, "kernels_per_step": 4 * args.batch,
            "collectives_per_step": 2 * args.batch,
            "wall_s_timed_region": t_wall, "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    del steps_, comm
    dist.destroy_process_group()


def spawn_ranks(args) -> int:
    """`--gpus N` without a launcher: start N ranks (one per GPU) through torch's launcher on
    127.0.0.1 and pass their output through."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main() -> None:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=4, choices=sorted(DECODE_CONFIGS),
                    help="BASELINE.json decode config (4 = the headline: 1M ctx)")
    ap.add_argument("--batch", type=int, default=1, help="sequences per step (sharded runs)")
    ap.add_argument("--ctx", type=int, default=CTX)
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-per-config", action="store_true")
    ap.add_argument("--per-config-steps", type=int, default=50)
    ap.add_argument("--sharded", action="store_true",
                    help="use the sequence-sharded path even on one rank (torchrun)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.impl == "reference":
        run_reference_arm(args)
    elif args.gpus > 1 and world == 0:
        sys.exit(spawn_ranks(args))
    elif args.sharded or world > 1:
        run_sharded(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
