#!/usr/bin/env python
"""One JSON line per BASELINE.json decode config on one GPU (batch 1, one layer, selection
defaults): the CUDA-graph decode step timed with CUDA events on the plan stream, L2 flushed
by a 256 MiB read before every timed step.

  config 1: LLaMA-3.1-8B heads (32/8), 32K tokens, fp32 cache (the CPU-reference config,
            here on the GPU)
  config 2: LLaMA-3.1-8B heads, 128K tokens, bf16
  config 4: LLaMA-3.1-8B heads, 1M tokens, bf16 (bench.py's headline, 1 GPU)
  config 5: LLaMA-3.2-3B heads (24/8, group 3), 4M tokens, bf16, batch 1 on 1 GPU

Algorithmic bytes per step = scan (n_kv x middle x d x esz) + scope (n_kv x L' x 2 x d x esz)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2407_15176_b200 import native as N  # noqa: E402

CONFIGS = {
    1: dict(n_head=32, n_kv=8, total=32 * 1024, dtype=N.F32, model="LLaMA-3.1-8B heads, fp32 cache"),
    2: dict(n_head=32, n_kv=8, total=128 * 1024, dtype=N.BF16, model="LLaMA-3.1-8B heads"),
    4: dict(n_head=32, n_kv=8, total=1 << 20, dtype=N.BF16, model="LLaMA-3.1-8B heads"),
    5: dict(n_head=24, n_kv=8, total=1 << 22, dtype=N.BF16, model="LLaMA-3.2-3B heads"),
}


def run(cid, steps, warmup):
    c = CONFIGS[cid]
    d = 128
    ctx = N.Context(0)
    stream = torch.cuda.ExternalStream(ctx.stream)
    cfg = N.SelectionConfig()
    cache = N.Cache(ctx, c["n_kv"], d, cfg.l_global, cfg.l_local, c["total"], c["dtype"])
    ctx.synth_uniform(cache.keys_tensor(), 1000 + cid)
    ctx.synth_uniform(cache.values_tensor(), 2000 + cid)
    cache.set_total(c["total"])
    rope = N.Rope(ctx, d, 500000.0, 8192)
    plan = N.Plan(ctx, cache, rope, 1, c["n_head"], cfg)
    qbank = torch.empty(steps + warmup, c["n_head"] * d, device="cuda")
    ctx.synth_uniform(qbank, 3000 + cid)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    with torch.cuda.stream(stream):
        for i in range(steps + warmup):
            plan.q.copy_(qbank[i:i + 1])
            flush.sum()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            plan.launch()
            b.record(stream)
            b.synchronize()
            if i >= warmup:
                ts.append(a.elapsed_time(b) * 1000.0)
    st = plan.stats()
    info = plan.info()
    esz = 4 if c["dtype"] == N.F32 else 2
    scope_bytes = c["n_kv"] * st.scope_len * 2 * d * esz
    us = sum(ts) / len(ts)
    gbs = (info["scan_bytes"] + scope_bytes) / (us * 1e-6) / 1e9
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    return {"config": cid, "workload": f"{c['model']}, {c['total']} tokens, batch 1, 1 layer",
            "us_per_token_layer": round(us, 2), "scan_bytes": info["scan_bytes"],
            "scope_len": st.scope_len, "step_gbs": round(gbs, 1),
            "frac_of_measured_copy_peak": round(gbs / peak, 3),
            "frac_of_8tbs_nominal": round(gbs / 8000.0, 3),
            "kernels_per_step": int(info["kernels_per_step"]), "steps": steps}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,4,5")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    args = ap.parse_args()
    for cid in [int(x) for x in args.configs.split(",")]:
        print(json.dumps(run(cid, args.steps, args.warmup)), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
