#!/usr/bin/env python
"""Per-rank device time of the sequence-sharded decode step (config 4: 1M context,
LLaMA-3.1-8B heads) for world = 2, 4, 8, emulated on ONE GPU: every rank's local cache
([global | middle shard | local]) is built on this GPU and each rank's stages are timed
alone with CUDA events (L2 read-flushed before each), the all-gathers replaced by device
copies.  The per-stage max over ranks approximates the N-GPU step minus the two NCCL
all-gathers (256 B and n_head x 544 B per rank).  Prints one JSON line per world size."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from paper_2407_15176_b200 import native as N  # noqa: E402
from paper_2407_15176_b200 import sharded as S  # noqa: E402


def build_local_cache(ctx, gk, gv, total, cfg, world, rank):
    segs = S.local_row_segments(total, cfg, world, rank)
    rows = sum(e - b for b, e in segs)
    n_kv, _, d = gk.shape
    c = N.Cache(ctx, n_kv, d, cfg.l_global, cfg.l_local, rows, N.BF16)
    kt, vt = c.keys_tensor(), c.values_tensor()
    o = 0
    for b, e in segs:
        kt[:, o:o + e - b].copy_(gk[:, b:e])
        vt[:, o:o + e - b].copy_(gv[:, b:e])
        o += e - b
    torch.cuda.synchronize()
    c.set_total(rows)
    return c


def timed(fn, stream, flush, reps=10):
    ts = []
    for _ in range(reps):
        flush.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1000.0)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ctx = N.Context(0)
    stream = torch.cuda.ExternalStream(ctx.stream)
    cfg = N.SelectionConfig()
    n_kv, nh, d, total = 8, 32, 128, 1 << 20
    g = N.Cache(ctx, n_kv, d, cfg.l_global, cfg.l_local, total, N.BF16)
    ctx.synth_uniform(g.keys_tensor(), 1000)
    ctx.synth_uniform(g.values_tensor(), 1001)
    g.set_total(total)
    rope = N.Rope(ctx, d, 500000.0, 8192)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    q = torch.empty(1, nh * d, device="cuda")
    ctx.synth_uniform(q, 5000)
    with torch.cuda.stream(stream):
        for world in (2, 4, 8):
            ops = [S.NativeOps(ctx, build_local_cache(ctx, g.keys_tensor(), g.values_tensor(), total,
                                                      cfg, world, r), rope, nh, cfg, total, world, r)
                   for r in range(world)]
            for o in ops:
                o.q.copy_(q)
            stages = {"scan": [], "select": [], "attend": [], "combine": []}
            for o in ops:
                stages["scan"].append(timed(o.scan, stream, flush))
            torch.cuda.synchronize()
            cand = torch.cat([o.cand_send for o in ops])
            for o in ops:
                o.cand_recv.copy_(cand)
            torch.cuda.synchronize()
            for o in ops:
                stages["select"].append(timed(o.select, stream, flush))
                stages["attend"].append(timed(o.attend, stream, flush))
            torch.cuda.synchronize()
            part = torch.cat([o.part_send for o in ops])
            for o in ops:
                o.part_recv.copy_(part)
            torch.cuda.synchronize()
            for o in ops:
                stages["combine"].append(timed(o.combine, stream, flush))
            # each rank's whole step as one CUDA graph, the two all-gathers replaced by
            # device copies from the buffers gathered above (what NCCL would deliver)
            cand_all, part_all = cand.clone(), part.clone()
            graph_us = []
            for o in ops:
                def body(o=o):
                    o.scan()
                    o.cand_recv.copy_(cand_all)
                    o.select()
                    o.attend()
                    o.part_recv.copy_(part_all)
                    o.combine()
                body()
                torch.cuda.synchronize()
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr, stream=stream):
                    body()
                graph_us.append(timed(gr.replay, stream, flush))
                del gr
            stages["graph_step"] = graph_us
            mx = {k: round(max(v), 1) for k, v in stages.items()}
            line = {"world": world, "ctx": total, "per_stage_max_over_ranks_us": mx,
                    "per_rank_us": {k: [round(x, 1) for x in v] for k, v in stages.items()},
                    "device_sum_us": round(sum(v for k, v in mx.items() if k != "graph_step"), 1),
                    "exchange_bytes_per_rank": [int(ops[0].cand_send.numel() * ops[0].cand_send.element_size()),
                                                int(ops[0].part_send.numel() * ops[0].part_send.element_size())],
                    "note": "one GPU, ranks timed one at a time; excludes the two NCCL all-gathers"}
            print(json.dumps(line), flush=True)
            del ops
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
