#!/usr/bin/env python
"""Config 3 (BASELINE.json): Mistral-v0.3 geometry (32 q / 8 kv heads, d=128) chunked
prefill at 256K — the prefill score scan + fused top-k on tcgen05 (K2, ε-tie parity) vs
the exact CUDA-core path, timed with CUDA events on the launching stream.

Per chunk the reference's score GEMM is 2·n_q·d·middle·n_kv FLOP; K2
executes it twice (bf16 hi + lo split of the fp32 query).  Prints one JSON line."""
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
    ap.add_argument("--ctx", type=int, default=256 * 1024)
    ap.add_argument("--n-q", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--exact", action="store_true", help="also time the exact CUDA-core path")
    args = ap.parse_args()
    n_kv, nh, d, k = 8, 32, 128, 4
    ctx = N.Context(0)
    stream = torch.cuda.ExternalStream(ctx.stream)
    g, loc = 32, 4096
    total = args.ctx
    middle = total - g - loc
    keys = torch.empty(n_kv, total, d, dtype=torch.bfloat16, device="cuda")
    ctx.synth_uniform(keys, 3000)
    q = torch.empty(args.n_q, nh * d, dtype=torch.float32, device="cuda")
    ctx.synth_uniform(q, 3001)
    idx = torch.zeros(n_kv * args.n_q * k, dtype=torch.int32, device="cuda")
    sc = torch.zeros(n_kv * args.n_q * k, dtype=torch.float32, device="cuda")
    flops = 2.0 * args.n_q * d * middle * n_kv

    def timed(mode):
        ctx.set_prefill(mode)
        for _ in range(2):
            ctx.fused_topk(q, nh, keys, n_kv, total, g, middle, d, k, idx, sc, N.BF16)
        ts = []
        for _ in range(args.reps):
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            ctx.fused_topk(q, nh, keys, n_kv, total, g, middle, d, k, idx, sc, N.BF16)
            s1.record(stream)
            s1.synchronize()
            ts.append(s0.elapsed_time(s1))
        ctx.set_prefill(N.PREFILL_EXACT)
        ts.sort()
        return ts[len(ts) // 2]

    ms = timed(N.PREFILL_TENSOR)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    line = {"workload": "config 3: Mistral-v0.3 geometry prefill chunk score scan + top-k",
            "ctx": total, "n_q": args.n_q, "middle": middle, "n_kv": n_kv, "d": d, "k": k,
            "tc_ms": ms, "algorithmic_tflop": flops / 1e12,
            "algorithmic_tflops": flops / (ms * 1e-3) / 1e12,
            "executed_tflops": flops / (ms * 1e-3) / 1e12,  # one bf16 pass
            "peak_tflops_burst": peaks["bf16_tflops"],
            "executed_frac_of_burst": flops / (ms * 1e-3) / 1e12 / peaks["bf16_tflops"]}
    if args.exact:
        ex = timed(N.PREFILL_EXACT)
        line["exact_ms"] = ex
        line["speedup_vs_exact_cuda_cores"] = ex / ms
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
