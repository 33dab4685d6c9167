#!/usr/bin/env python
"""Config 3 (BASELINE.json), a whole layer: the chunked prefill of 262,144 tokens the way the
reference's Engine::prefill runs it (engine.hpp:147-160): a first block of l_global + l_local =
4,128 tokens, then 4,096-token chunks, each an attend_step (engine.hpp:43-114) over the cache
that already holds the chunk's K/V -- Mistral-v0.3 heads (32 q / 8 kv, d = 128), RoPE base 1e6,
bf16 cache, selection defaults with l_chunk = 4096.

Every chunk runs as a CUDA-graph plan on the tensor-core prefill path (K2 score GEMM with
exact re-scoring, the large-candidate vote, K6 attention); its replay is timed with CUDA events
(L2 read-flushed before each), and K2 alone (plan.launch_scan) is timed for the score-GEMM
share.  FLOP accounting: scan 2·n_q·d·middle·n_kv per chunk (69.25 TFLOP per
layer), attention 4·d·n_head·Σ visible prefix.  Prints one JSON line."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2407_15176_b200 import native as N  # noqa: E402


def run(ctx, args) -> dict:
    n_kv, nh, d = 8, 32, 128
    stream = torch.cuda.ExternalStream(ctx.stream)
    cfg = N.SelectionConfig(l_chunk=args.chunk)
    total = args.ctx
    cache = N.Cache(ctx, n_kv, d, cfg.l_global, cfg.l_local, total, N.BF16)
    ctx.synth_uniform(cache.keys_tensor(), 3100)
    ctx.synth_uniform(cache.values_tensor(), 3101)
    rope = N.Rope(ctx, d, 1.0e6, 8192)
    flush = bench._flush_buffer(torch, f"cuda:{ctx.device}")
    first = min(total, cfg.l_global + cfg.l_local)
    ends = [first]
    while ends[-1] < total:
        ends.append(min(total, ends[-1] + args.chunk))
    q_all = torch.empty(args.chunk if args.chunk > first else first, nh * d, device="cuda")
    ctx.synth_uniform(q_all, 3102)

    def time_launch(fn):
        flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            fn()
            e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1)

    ctx.set_prefill(N.PREFILL_TENSOR)
    start, stop = getattr(args, "start", 0), getattr(args, "stop", 1 << 30)
    rows = []
    prev = 0
    for ci, end in enumerate(ends):
        n_q = end - prev
        timed = ci == 0 or ci == len(ends) - 1 or ci % args.every == 0
        if timed and start <= ci <= stop:
            dbg = (lambda *m: print(ci, *m, file=sys.stderr, flush=True)) if os.environ.get("VERBOSE") else (lambda *m: None)
            cache.set_total(end)
            plan = N.Plan(ctx, cache, rope, n_q, nh, cfg)
            dbg("created")
            plan.q.copy_(q_all[:n_q])
            torch.cuda.synchronize()
            plan.launch()
            st = plan.stats()
            dbg("warm launch done")
            step_ms = time_launch(plan.launch)
            dbg("timed step")
            scan_ms = time_launch(plan.launch_scan) if st.n_spans else 0.0
            dbg("timed scan")
            L = st.scope_len
            middle = max(0, end - cfg.l_global - cfg.l_local)
            visible = sum(L - n_q + i + 1 for i in range(n_q))
            rows.append(dict(chunk=ci, end=end, n_q=n_q, L=L, step_ms=step_ms, scan_ms=scan_ms,
                             scan_tflop=2.0 * n_q * d * middle * n_kv / 1e12,
                             attn_tflop=4.0 * d * nh * visible / 1e12))
            if os.environ.get("VERBOSE"):
                print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
            del plan
        prev = end
    ctx.set_prefill(N.PREFILL_DEFAULT)
    if start or stop < len(ends) - 1:  # debugging / profiling a few chunks: no total
        return {"rows": rows}
    # interpolate untimed chunks linearly in the chunk index between timed neighbours
    timed_idx = [r["chunk"] for r in rows]
    by = {r["chunk"]: r for r in rows}
    total_ms = total_scan_ms = 0.0
    for ci in range(len(ends)):
        if ci in by:
            total_ms += by[ci]["step_ms"]
            total_scan_ms += by[ci]["scan_ms"]
            continue
        lo = max(t for t in timed_idx if t < ci)
        hi = min(t for t in timed_idx if t > ci)
        w = (ci - lo) / (hi - lo)
        total_ms += (1 - w) * by[lo]["step_ms"] + w * by[hi]["step_ms"]
        total_scan_ms += (1 - w) * by[lo]["scan_ms"] + w * by[hi]["scan_ms"]
    scan_tflop = sum(2.0 * (e - s) * d * max(0, e - cfg.l_global - cfg.l_local) * n_kv / 1e12
                     for s, e in zip([0] + ends[:-1], ends))
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    line = {"workload": "config 3: Mistral-v0.3 heads, chunked prefill of one layer to 256K "
                        "(first block 4128, then 4096-token chunks)",
            "chunks": len(ends), "chunks_timed": len(rows), "layer_ms": total_ms,
            "score_gemm_ms": total_scan_ms, "score_gemm_tflop": scan_tflop,
            "score_gemm_tflops": scan_tflop / (total_scan_ms * 1e-3) if total_scan_ms else None,
            "score_gemm_frac_of_bf16_burst": (scan_tflop / (total_scan_ms * 1e-3)) / peaks["bf16_tflops"]
            if total_scan_ms else None,
            "target_score_gemm_ms": 72.0, "last_chunk": rows[-1]}
    del cache
    torch.cuda.empty_cache()
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, default=256 * 1024)
    ap.add_argument("--chunk", type=int, default=4096)
    ap.add_argument("--every", type=int, default=1, help="time every n-th chunk, interpolate the rest")
    ap.add_argument("--start", type=int, default=0, help="debugging: skip the chunks before this one")
    ap.add_argument("--stop", type=int, default=1 << 30, help="debugging: skip the chunks after this one")
    args = ap.parse_args()
    print(json.dumps(run(N.Context(0), args)), flush=True)


if __name__ == "__main__":
    main()
