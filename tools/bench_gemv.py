#!/usr/bin/env python
"""The decoder's fp32 GEMV alone (reattn_debug_gemv), at the LLaMA3-8B decode shapes: per
launch time with CUDA events over a rotation of weight matrices larger than L2 (every launch
streams its weights from HBM), back to back on one stream, and the achieved GB/s."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2407_15176_b200 import native as N  # noqa: E402

SHAPES = {"wq/wo": (4096, 4096), "wk": (4096, 1024), "gate": (4096, 14336), "down": (14336, 4096),
          "lm_head": (4096, 128256)}


def main():
    ctx = N.Context(0)
    lib = ctx.lib
    stream = torch.cuda.ExternalStream(ctx.stream)
    res = {}
    for name, (k, n) in SHAPES.items():
        per = k * n * 4
        count = max(2, int((600 << 20) // per) + 1)  # > 4 x L2 of weights in rotation
        ws_ = [torch.empty(k, n, device="cuda").uniform_(-0.02, 0.02) for _ in range(count)]
        x = torch.randn(k, device="cuda")
        y = torch.zeros(n, device="cuda")
        wsb = torch.zeros(lib.reattn_debug_gemv_workspace(n), dtype=torch.uint8, device="cuda")
        torch.cuda.synchronize()

        def go(i):
            ctx.check(lib.reattn_debug_gemv(ctx.h, x.data_ptr(), ws_[i % count].data_ptr(), n, n, k,
                                            y.data_ptr(), 0.0, wsb.data_ptr()))
        for i in range(3 * count):
            go(i)
        reps = max(20, 3 * count)
        with torch.cuda.stream(stream):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for i in range(reps):
                go(i)
            b.record(stream)
        b.synchronize()
        us = a.elapsed_time(b) * 1000.0 / reps
        ref = x @ ws_[(reps - 1) % count]
        err = float((y - ref).abs().max() / ref.abs().max())
        res[name] = {"k": k, "n": n, "us": round(us, 2), "gbs": round(per / us / 1e3, 1), "rel_err": err}
        del ws_
        torch.cuda.empty_cache()
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
