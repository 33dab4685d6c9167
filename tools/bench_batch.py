#!/usr/bin/env python
"""Batched decode sweep on one GPU (BASELINE config 5's batch dimension): n_seq sequences
with their own caches in one graph (reattn_batch_plan), L2 read-flushed before each timed
step.  Reports µs per token-layer (step time / n_seq) and aggregate tokens/s per layer.
  --config 4: LLaMA-3.1-8B heads, 1M tokens per sequence
  --config 5: LLaMA-3.2-3B heads (24/8), 4M tokens per sequence"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2407_15176_b200 import native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--batches", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    nh, total = (32, 1 << 20) if args.config == 4 else (24, 1 << 22)
    ctx = N.Context(0)
    stream = torch.cuda.ExternalStream(ctx.stream)
    cfg = N.SelectionConfig()
    rope = N.Rope(ctx, 128, 500000.0, 8192)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    bmax = max(int(x) for x in args.batches.split(","))
    caches = []
    for i in range(bmax):
        c = N.Cache(ctx, 8, 128, cfg.l_global, cfg.l_local, total, N.BF16)
        ctx.synth_uniform(c.keys_tensor(), 100 + 2 * i)
        ctx.synth_uniform(c.values_tensor(), 101 + 2 * i)
        c.set_total(total)
        caches.append(c)
    for B in [int(x) for x in args.batches.split(",")]:
        bp = N.BatchPlan(ctx, caches[:B], rope, nh, cfg)
        q = torch.empty(B, nh * 128, device="cuda")
        ctx.synth_uniform(q, 7 + B)
        ts = []
        with torch.cuda.stream(stream):
            for i in range(args.steps + 2):
                bp.q.copy_(q)
                flush.sum()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                bp.launch()
                b.record(stream)
                b.synchronize()
                if i >= 2:
                    ts.append(a.elapsed_time(b) * 1000.0)
        us = sum(ts) / len(ts)
        info = bp.info()
        print(json.dumps({"config": args.config, "batch": B, "ctx_per_seq": total, "n_head": nh,
                          "step_us": round(us, 1), "us_per_token_layer": round(us / B, 1),
                          "tokens_per_s_per_layer": round(B / (us * 1e-6), 1),
                          "scan_gbs": round(info["scan_bytes"] / (us * 1e-6) / 1e9, 1),
                          "side_sms": info["side_sms"], "kernels_per_step": info["kernels_per_step"]}),
              flush=True)
        del bp


if __name__ == "__main__":
    main()
