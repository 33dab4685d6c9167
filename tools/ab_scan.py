#!/usr/bin/env python
"""A/B helper: time the 1M-context K scan graph (plan.launch_scan) and the full decode step
(plan.launch) with and without a 256 MiB L2 flush before each launch.  Run with
REATTN_LIB=<path> to compare builds on the same box.  Prints one JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2407_15176_b200 import native as N  # noqa: E402


def main():
    ctx = N.Context(0)
    stream = torch.cuda.ExternalStream(ctx.stream)
    cfg = N.SelectionConfig()
    total = 1 << 20
    cache = N.Cache(ctx, 8, 128, cfg.l_global, cfg.l_local, total, N.BF16)
    ctx.synth_uniform(cache.keys_tensor(), 1000)
    ctx.synth_uniform(cache.values_tensor(), 1001)
    cache.set_total(total)
    rope = N.Rope(ctx, 128, 500000.0, 8192)
    plan = N.Plan(ctx, cache, rope, 1, 32, cfg)
    q = torch.empty(1, 32 * 128, device="cuda")
    ctx.synth_uniform(q, 5)
    plan.q.copy_(q)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = {"lib": os.environ.get("REATTN_LIB", "default")}
    with torch.cuda.stream(stream):
        for name, fn in (("scan", plan.launch_scan), ("step", plan.launch)):
            for fl in ("flush", "readflush", "warm"):
                for _ in range(3):
                    fn()
                ts = []
                for _ in range(20):
                    if fl == "flush":
                        flush.zero_()
                    elif fl == "readflush":
                        flush.sum()  # evicts L2 with clean lines: no write-back charged later
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    fn()
                    b.record(stream)
                    b.synchronize()
                    ts.append(a.elapsed_time(b) * 1000)
                ts.sort()
                out[f"{name}_{fl}_us"] = round(ts[len(ts) // 2], 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
