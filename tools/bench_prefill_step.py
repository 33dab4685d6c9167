#!/usr/bin/env python
"""Config 3 (BASELINE.json) end to end: one ReAttention prefill step (engine.hpp:43
attend_step) for the last 4096-query chunk at 256K context, Mistral-v0.3 head geometry
(32 q / 8 kv heads, d = 128, rope base 1e6), bf16 cache, default selection
(k = 4, k' = 127, m = 32, g = 32, local = 4096).

Times the CUDA-graph step plan with CUDA events on the plan's stream for the tensor-core
prefill paths (K2 scan + K6 attention) and, with --exact, the bit-exact CUDA-core paths.
Flop accounting: scan 2·n_q·d·middle·n_kv; scope attention
2·2·d·n_head·Σ_i visible_i (QK^T and PV over each query's causal prefix of the scope).
Prints one JSON line."""
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
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--exact", action="store_true", help="also time the exact CUDA-core paths")
    args = ap.parse_args()
    n_kv, nh, d = 8, 32, 128
    ctx = N.Context(0)
    stream = torch.cuda.ExternalStream(ctx.stream)
    cfg = N.SelectionConfig()
    total, n_q = args.ctx, args.n_q
    cache = N.Cache(ctx, n_kv, d, cfg.l_global, cfg.l_local, total, N.BF16)
    ctx.synth_uniform(cache.keys_tensor(), 3100)
    ctx.synth_uniform(cache.values_tensor(), 3101)
    cache.set_total(total)
    rope = N.Rope(ctx, d, 1.0e6, 32768)
    q = torch.empty(n_q, nh * d, dtype=torch.float32, device="cuda")
    ctx.synth_uniform(q, 3102)
    middle = total - cfg.l_global - cfg.l_local

    def run(mode, reps):
        ctx.set_prefill(mode)
        plan = N.Plan(ctx, cache, rope, n_q, nh, cfg)
        ctx.set_prefill(N.PREFILL_EXACT)
        plan.q.copy_(q)
        torch.cuda.synchronize()
        plan.launch()
        st = plan.stats()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            plan.launch()
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        out = plan.out.clone()
        del plan
        return ts[len(ts) // 2], st, out

    tc_ms, st, out_tc = run(N.PREFILL_TENSOR, args.reps)
    L = st.scope_len
    boundary = L - n_q
    visible = sum(boundary + i + 1 for i in range(n_q))
    scan_flop = 2.0 * n_q * d * middle * n_kv
    attn_flop = 4.0 * d * nh * visible
    line = {"workload": "config 3: Mistral-v0.3 geometry prefill step, last 4K chunk at 256K",
            "ctx": total, "n_q": n_q, "scope_len": L, "middle": middle,
            "tensor_ms": tc_ms,
            "scan_tflop": scan_flop / 1e12, "attn_tflop": attn_flop / 1e12,
            "algorithmic_tflops": (scan_flop + attn_flop) / (tc_ms * 1e-3) / 1e12}
    if args.exact:
        ex_ms, st_ex, out_ex = run(N.PREFILL_EXACT, 1)
        line["exact_ms"] = ex_ms
        line["speedup_vs_exact"] = ex_ms / tc_ms
        line["same_scope_len"] = st_ex.scope_len == L
        line["max_abs_vs_exact"] = (out_tc - out_ex).abs().max().item()
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
