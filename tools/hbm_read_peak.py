#!/usr/bin/env python
"""Read-only HBM bandwidth probes on this GPU (the roofline denominator question for the
K scan, which only reads): torch reductions over a 2.1 GB bf16 tensor (same size as the
1M-context K scan), CUDA events, best of N.  Prints one JSON line."""
import json

import torch


def best(fn, n=10):
    ts = []
    for _ in range(n):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    return min(ts)


def main():
    n = 8 * 1044448 * 128  # K scan elements at 1M context
    x = torch.empty(n, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    y = torch.empty(n // 2, dtype=torch.float32, device="cuda").uniform_(-1, 1)
    b = x.numel() * 2
    out = {}
    for name, fn, nbytes in (("bf16_sum", lambda: x.sum(), b), ("bf16_amax", lambda: x.amax(), b),
                             ("f32_sum", lambda: y.sum(), b),
                             ("copy_rw", lambda: x.clone(), 2 * b)):
        fn()
        ms = best(fn)
        out[name] = round(nbytes / (ms * 1e-3) / 1e9, 1)
    print(json.dumps({"read_gbs": out, "bytes": b}))


if __name__ == "__main__":
    main()
