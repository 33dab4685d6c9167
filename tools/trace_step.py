#!/usr/bin/env python
"""Device timeline of one decode step (diagnostics): REATTN_TRACE=1 makes K1 and K5 stamp
%globaltimer; this prints, relative to the first K1 CTA start, when the scan's CTAs start and
finish their tiles, when the last CTA's merge and select end, and when the decode attention's
CTAs start / finish.  Usage: REATTN_TRACE=1 python tools/trace_step.py --ctx 131072"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2407_15176_b200 import native as N  # noqa: E402


def summarize(v):
    v = sorted(v)
    return (f"min {v[0] / 1e3:8.2f}  med {statistics.median(v) / 1e3:8.2f}  "
            f"p90 {v[int(0.9 * (len(v) - 1))] / 1e3:8.2f}  max {v[-1] / 1e3:8.2f} us")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, default=131072)
    ap.add_argument("--n-head", type=int, default=32)
    ap.add_argument("--n-kv", type=int, default=8)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--no-flush", action="store_true", help="keep L2 warm between steps")
    ap.add_argument("--slow", action="store_true", help="list the slowest scan CTAs")
    args = ap.parse_args()
    assert os.environ.get("REATTN_TRACE") == "1", "set REATTN_TRACE=1"
    ctx = N.Context(0)
    cfg = N.SelectionConfig()
    dt = N.BF16 if args.dtype == "bf16" else N.F32
    cache = N.Cache(ctx, args.n_kv, 128, cfg.l_global, cfg.l_local, args.ctx, dt)
    ctx.synth_uniform(cache.keys_tensor(), 11)
    ctx.synth_uniform(cache.values_tensor(), 12)
    cache.set_total(args.ctx)
    rope = N.Rope(ctx, 128, 500000.0, 8192)
    plan = N.Plan(ctx, cache, rope, 1, args.n_head, cfg)
    ctx.synth_uniform(plan.q, 13)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for rep in range(args.reps):
        if not args.no_flush:
            flush.sum()
        torch.cuda.synchronize()
        N.debug_trace()  # clear by reading (stamps are overwritten by the next replay)
        plan.launch()
        t = N.debug_trace()
        G = sum(1 for x in t[:512] if x)
        t0 = min(x for x in t[:G])
        rel = lambda xs: [x - t0 for x in xs if x]  # noqa: E731
        print(f"--- rep {rep}  ctx {args.ctx}  scan CTAs {G}")
        print("K1 CTA start      ", summarize(rel(t[:G])))
        print("K1 CTA loop done  ", summarize(rel(t[512:512 + G])))
        if any(t[1200:1200 + G]):
            fl = [t[512 + c] - t[1200 + c] for c in range(G) if t[1200 + c]]
            print("K1 final flush    ", summarize(fl))
        if args.slow:
            order = sorted(range(G), key=lambda c: -(t[512 + c] - t0))
            print("   slowest CTAs (cta, sm, done us):",
                  [(c, t[1100 + c], round((t[512 + c] - t0) / 1e3, 1)) for c in order[:12]])
            print("   fastest CTAs:", [(c, t[1100 + c], round((t[512 + c] - t0) / 1e3, 1))
                                      for c in order[-6:]])
        print(f"K1 last ticket {(t[1024] - t0) / 1e3:8.2f}  merge done {(t[1025] - t0) / 1e3:8.2f}"
              f"  select done {(t[1026] - t0) / 1e3:8.2f} us")
        print(f"   K1 detail: warp0 slots read {(t[1027] - t0) / 1e3:8.2f}  pre-select {(t[1028] - t0) / 1e3:8.2f}"
              f"  warp part done {(t[1029] - t0) / 1e3:8.2f} us")
        print(f"   select warp part: {t[1041] - t[1040]} SM cycles over {(t[1029] - t[1028])} ns")
        print(f"   select phases: tally {(t[1030] - t0) / 1e3:8.2f}  rank/spans {(t[1031] - t0) / 1e3:8.2f}"
              f"  sort {(t[1032] - t0) / 1e3:8.2f} us")
        s5 = rel(t[1536:2048])
        if s5:
            print("K5 CTA start      ", summarize(s5))
            print("K5 CTA compute end", summarize(rel(t[2560:3072])))
        sl = rel(t[2048:2560])
        if sl:
            print("K5 local start    ", summarize(sl))
            print("K5 local end      ", summarize(rel(t[3072:3584])))
        if t[3700]:
            print(f"   K5 part0/kv0: q rotated {(t[3700] - t0) / 1e3:8.2f}  first copy issued "
                  f"{(t[3704] - t0) / 1e3:8.2f}  first chunk landed {(t[3701] - t0) / 1e3:8.2f}  "
                  f"warps merged {(t[3703] - t0) / 1e3:8.2f} us")
        if t[3904]:
            iss = [(c, t[3712 + c], t[3776 + c], t[3840 + c]) for c in range(64) if t[3712 + c]]
            print(f"   K5 CTA(0,0) resident {(t[3904] - t0) / 1e3:8.2f} us; per chunk: issued / landed / consumed")
            for c, a_, b_, c_ in iss:
                f = lambda x: f"{(x - t0) / 1e3:8.2f}" if x else "     -  "  # noqa: E731
                print(f"      chunk {c:2d}: {f(a_)} {f(b_)} {f(c_)}")
        if any(t[3600:3600 + args.n_kv]):
            print("K5 last ticket    ", summarize(rel(t[3600:3600 + args.n_kv])))
            print("K5 M/w loops done ", summarize(rel(t[3664:3664 + args.n_kv])))
        hm = rel(t[3584:3584 + args.n_kv])
        if hm:
            print("K5 head merge done", summarize(hm))
        # clear
        torch.cuda.synchronize()
    del plan


if __name__ == "__main__":
    main()
