#!/usr/bin/env python
"""One JSON line per BASELINE.json decode config on one GPU (batch 1, one layer, selection
defaults): the CUDA-graph decode step timed with CUDA events on the plan stream, L2
read-flushed before every timed step.  The workloads are bench.py's (build_decode):

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

import bench  # noqa: E402
from paper_2407_15176_b200 import native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,4,5")
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    ctx = N.Context(0)
    stream = torch.cuda.ExternalStream(ctx.stream)
    flush = bench._flush_buffer(torch, "cuda:0")
    peaks = bench.load_peaks()
    for line in bench.per_config_lines(ctx, stream, flush, peaks,
                                       [int(x) for x in args.configs.split(",")], args.steps):
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
