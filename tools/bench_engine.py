#!/usr/bin/env python
"""Decode throughput of the drop-in Engine (engine.hpp:163-174 decode_step) at the shape of the
paper's decode-throughput table (LLaMA3-8B, 1×A800, tokens/s at 32K-256K):
32 layers, d_model 4096, 32 q / 8 kv heads of 128, d_ff 14336, vocab 128256, window 8192,
RoPE base 5e5, selection defaults, bf16 KV cache, batch 1.  Weights are synthetic (the
reference's architecture, values filled on the device: reattn_weights_synth; fp32, as the
reference's DenseMatrix), and every layer's cache is filled with `ctx` synthetic rows as if a
prompt of that length had been prefilled (reattn_engine_synth_context).  Each decode step is
the full token: embedding, per layer RMSNorm + fp32 projections (cuBLAS) + the append + the
graph-captured ReAttention step, FFN, final norm, lm_head, argmax.  Wall clock per step (the
engine synchronises once per step).  Prints one JSON line."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2407_15176_b200 import native as N  # noqa: E402


def run(ctx, contexts, steps=16, warmup=4) -> dict:
    cfg = N.ModelConfig(n_layer=32, n_head=32, n_kv_head=8, d_model=4096, d_head=128, d_ff=14336,
                        vocab_size=128256, pretrain_window=8192, rope_base=500000.0,
                        attention_mode=N.MODE_REATTENTION)
    w = N.Weights.synth(ctx, cfg, 7)
    sel = N.SelectionConfig()
    res = {"model": "LLaMA3-8B shape (32 x 4096, 32/8 heads, d_ff 14336, vocab 128256), fp32 weights, "
                    "bf16 KV cache, batch 1", "per_context": []}
    for total in contexts:
        eng = N.Engine(ctx, w, sel, N.MODE_REATTENTION, N.BF16)
        eng.synth_context(total, 3)
        tok = 11
        for _ in range(warmup):
            tok = eng.decode_step(tok)
        t0 = time.perf_counter()
        for _ in range(steps):
            tok = eng.decode_step(tok)
        dt = (time.perf_counter() - t0) / steps
        res["per_context"].append({"ctx": total, "ms_per_token": dt * 1e3, "tokens_per_s": 1.0 / dt})
        del eng
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--contexts", default="32768,131072")
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--warmup", type=int, default=4)
    args = ap.parse_args()
    print(json.dumps(run(N.Context(0), [int(x) for x in args.contexts.split(",")], args.steps,
              args.warmup)),
          flush=True)


if __name__ == "__main__":
    main()
