#!/usr/bin/env python
"""Decode step in context: one token through L layers of attention, each layer its own
cache (L x config bytes, far larger than L2), the plans replayed back to back on one stream
with no flush between them -- what a multi-layer model's decode sees (the kernels' code and
the rotary table stay warm across layers; every layer's keys come from HBM).  Printed beside
the single-layer numbers with and without the L2 read-flush.

  python tools/bench_layers.py --config 2 --layers 16 --steps 10
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2407_15176_b200 import native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--layers", type=int, default=16)
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    ctx = N.Context(0)
    stream = torch.cuda.ExternalStream(ctx.stream)
    flush = bench._flush_buffer(torch, "cuda:0")
    layers = [bench.build_decode(ctx, args.config) for _ in range(args.layers)]
    meta = layers[0][4]
    qbank = torch.empty(args.steps + 8, meta["n_head"] * bench.D, device="cuda:0")
    ctx.synth_uniform(qbank, 77)
    plan0 = layers[0][2]
    single_flush = bench.time_plan(plan0, qbank, stream, flush, args.steps, 5)
    with torch.cuda.stream(stream):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # single layer, no flush
        for i in range(5):
            plan0.launch()
        torch.cuda.synchronize()
        tot = 0.0
        for i in range(args.steps):
            plan0.q.copy_(qbank[i:i + 1])
            e0.record(stream)
            plan0.launch()
            e1.record(stream)
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        single_noflush = tot / args.steps
        # L layers back to back
        for (_, _, p, _, _) in layers:
            p.q.copy_(qbank[0:1])
            p.launch()
        torch.cuda.synchronize()
        tot = 0.0
        for i in range(args.steps):
            flush.sum()
            e0.record(stream)
            for (_, _, p, _, _) in layers:
                p.launch()
            e1.record(stream)
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        multi = tot / args.steps / args.layers
    print(json.dumps({"config": args.config, "workload": meta["workload"], "layers": args.layers,
                      "single_layer_flushed_us": single_flush * 1e3,
                      "single_layer_unflushed_us": single_noflush * 1e3,
                      "per_layer_in_stack_us": multi * 1e3,
                      "kernels_per_step": int(plan0.info()["kernels_per_step"]),
                      "env": {k: v for k, v in os.environ.items() if k.startswith("REATTN_")}}),
          flush=True)


if __name__ == "__main__":
    main()
