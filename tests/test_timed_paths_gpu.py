"""The TIMED paths pinned to the CPU oracle at their full sizes.

bench.py times `Plan` replays built by bench.build_decode (configs 1, 2, 4 and 5 of
BASELINE.json, one GPU, exactly the plans and inputs of the bench line and its per_config
object: the 1M plan with the default local-window fork, the 144-SM scan and the select fused
into the scan's merger CTA).  Each test replays that plan twice on fresh queries and compares
every attend_step output with the oracle's attend_step (engine.hpp:43-114) run on the
device cache's own bytes (bf16 words widened exactly, or the fp32 rows):
  spans / L' / coverage   identical
  outputs                 max-abs <= 1e-6 (north_star fp32 bar 1e-5)
  row entropies           max-abs <= 1e-6 (every head, not only the max)
The prefill test runs config 3 at its full last-chunk shape (Mistral-v0.3 heads, 4096 queries
against a 262,144-token cache, middle 258,016 rows, RoPE base 1e6) through the default
prefill path (K2 tcgen05 scan + exact re-scoring, K3 large vote, K6 tcgen05 attention):
the per-head top-k lists bit-identical (indices and score bits), spans identical, outputs
within 2e-4 (north_star bf16 bar 1e-2).
"""
import numpy as np
import pytest

import bench
import oracle_bind as ob

torch = pytest.importorskip("torch")
from paper_2407_15176_b200 import native as N  # noqa: E402

pytestmark = pytest.mark.gpu

OUT_TOL = 1e-6
ENT_TOL = 1e-6


def host_cache(cache, dtype):
    """The device cache as host arrays: fp32 rows or bf16 words (no widening copy)."""
    if dtype == "f32":
        return cache.keys_tensor().cpu().numpy(), cache.values_tensor().cpu().numpy()
    return ob.bf16_words(cache.keys_tensor()), ob.bf16_words(cache.values_tensor())


@pytest.mark.parametrize("cid", [1, 2, 4, 5])
def test_bench_plan_matches_oracle(ctx, cid):
    cache, rope, plan, cfg, meta = bench.build_decode(ctx, cid)
    n_head, total = meta["n_head"], meta["total"]
    hk, hv = host_cache(cache, meta["dtype"])
    _, _, qseed = bench.config_seeds(cid)
    qbank = torch.empty(2, n_head * bench.D, dtype=torch.float32, device="cuda")
    ctx.synth_uniform(qbank, qseed)
    ocfg = ob.SelectionConfig()
    for rep in range(2):
        plan.q.copy_(qbank[rep:rep + 1])
        torch.cuda.synchronize()
        plan.launch()
        res = plan.result(cfg.k_prime)
        got = res.out.cpu().numpy()
        q = qbank[rep:rep + 1].cpu().numpy()
        out, ent, st, (sb, se), _ = ob.attend_step_ex(q, n_head, hk, hv, total, ocfg,
                                                      bench.ROPE_BASE, bench.WINDOW)
        label = f"config {cid} replay {rep}"
        assert res.stats.scope_len == st.scope_len, label
        assert res.stats.n_spans == st.n_spans and res.stats.coverage == st.coverage, label
        assert np.array_equal(res.spans[0], sb) and np.array_equal(res.spans[1], se), label
        assert res.stats.max_position_used == st.max_position_used, label
        err = float(np.abs(got - out).max())
        assert err <= OUT_TOL, (label, err)
        eerr = float(np.abs(res.entropy - ent).max())
        assert eerr <= ENT_TOL, (label, eerr)
        assert abs(res.stats.entropy_max - st.entropy_max) <= ENT_TOL, label


@pytest.mark.slow
def test_config3_prefill_chunk_full_shape(ctx):
    """BASELINE config 3's last chunk at full size through the default prefill path."""
    n_kv, nh, d, total, n_q = 8, 32, 128, 262144, 4096
    base, window = 1e6, 8192
    cfg = N.SelectionConfig(l_chunk=4096)
    cache = N.Cache(ctx, n_kv, d, cfg.l_global, cfg.l_local, total, N.BF16)
    ctx.synth_uniform(cache.keys_tensor(), 3001)
    ctx.synth_uniform(cache.values_tensor(), 3002)
    cache.set_total(total)
    rope = N.Rope(ctx, d, base, window)
    q = torch.empty(n_q, nh * d, dtype=torch.float32, device="cuda")
    ctx.synth_uniform(q, 3003)
    ctx.set_prefill(N.PREFILL_TENSOR)
    try:
        res = N.attend_step(ctx, cache, rope, q, nh, cfg)
        # the K2 score lists on their own (reattn_fused_topk routes n_q > 1 to K2 as well)
        info = cache.info()
        g, ls = info["global_end"], info["local_start"]
        idx = torch.zeros(n_kv * n_q * cfg.k, dtype=torch.int32, device="cuda")
        sc = torch.zeros(n_kv * n_q * cfg.k, dtype=torch.float32, device="cuda")
        ctx.fused_topk(q, nh, cache.keys_tensor(), n_kv, info["capacity"], g, ls - g, d, cfg.k,
                       idx, sc, N.BF16)
    finally:
        ctx.set_prefill(N.PREFILL_DEFAULT)
    hk, hv = host_cache(cache, "bf16")
    ocfg = ob.SelectionConfig(l_chunk=4096)
    out, ent, st, (sb, se), _, (ci, cs) = ob.attend_step_ex(q.cpu().numpy(), nh, hk, hv, total,
                                                            ocfg, base, window, candidates=True)
    gi = idx.cpu().numpy().view(np.uint32).reshape(n_kv, n_q, cfg.k).astype(np.uint64)
    gs = sc.cpu().numpy().reshape(n_kv, n_q, cfg.k)
    assert np.array_equal(gi, ci), "K2 top-k indices differ from the oracle"
    nz = gs != 0
    assert np.array_equal(gs, cs) and np.array_equal(gs[nz].view(np.uint32), cs[nz].view(np.uint32))
    assert res.stats.scope_len == st.scope_len
    assert np.array_equal(res.spans[0], sb) and np.array_equal(res.spans[1], se)
    err = float(np.abs(res.out.cpu().numpy() - out).max())
    assert err <= 2e-4, err
    assert float(np.abs(res.entropy - ent).max()) <= 2e-3


def test_reference_lane_mode_on_this_host():
    """The compiled reference (oracle/_ref, loaded for this host's ISA level) must score d=128
    keys with the lane arithmetic the library uses by default (unfused): checked
    on the GPU box's own CPU, where the bench's reference arm and the CPU baseline run."""
    mode = ob.ref_lane_mode(128)
    if ob.ref() is None:
        pytest.skip("oracle/_ref not shipped to this host")
    assert mode == N.LANES_UNFUSED == ob.LANES_UNFUSED, mode
