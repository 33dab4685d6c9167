"""K6 (prefill finite-scope attention on tcgen05) — attend_step parity with the tensor
attention enabled (PREFILL_TENSOR_ATTN; the scan stays exact so the scope is identical).

Reference: attend_step (engine.hpp:43-114) -> attend (attend.hpp:25-77).  K6 computes
S with bf16 hi+lo split operands and fp32 TMEM accumulation, so the bar is the north_star
bf16 tolerance (max-abs 1e-2); the measured error is orders of magnitude below it and the
tighter bound below pins that."""
import numpy as np
import pytest

import oracle_bind as ob
import synth

torch = pytest.importorskip("torch")
from paper_2407_15176_b200 import native as N  # noqa: E402

pytestmark = pytest.mark.gpu

BF16_TOL = 1e-2      # north_star attention tolerance at bf16
MEASURED_TOL = 2e-4  # what the hi+lo split actually achieves (kept as a regression bound)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def make_cache(ctx, n_kv, d, total, cfg, seed):
    cache = N.Cache(ctx, n_kv, d, cfg.l_global, cfg.l_local, total, N.BF16)
    kt, vt = cache.keys_tensor(), cache.values_tensor()
    ctx.synth_uniform(kt, seed)
    ctx.synth_uniform(vt, seed + 1)
    cache.set_total(total)
    return cache, kt.float().cpu().numpy(), vt.float().cpu().numpy()


def step(ctx, cache, rope, q, nh, cfg, mode_bits):
    ctx.set_prefill(mode_bits)
    try:
        return N.attend_step(ctx, cache, rope, q, nh, cfg)
    finally:
        ctx.set_prefill(N.PREFILL_DEFAULT)


@pytest.mark.parametrize("n_q,total", [(128, 5000), (200, 6000), (37, 4500)])
def test_prefill_attention_tc_vs_oracle(ctx, n_q, total):
    """LLaMA-3.1-8B head geometry, bf16 cache, default selection; ragged query blocks."""
    cfg = N.SelectionConfig()
    cache, hk, hv = make_cache(ctx, 8, 128, total, cfg, 700 + n_q)
    base, window = 500000.0, 8192
    rope = N.Rope(ctx, 128, base, window)
    q = synth.uniform(701 + n_q, n_q * 32 * 128).reshape(n_q, 32 * 128)
    res = step(ctx, cache, rope, dev(q), 32, cfg, N.PREFILL_TENSOR_ATTN)
    ocfg = ob.SelectionConfig(cfg.k, cfg.k_prime, cfg.span_m, cfg.tile_size, cfg.l_global,
                              cfg.l_local, cfg.l_chunk, cfg.span_mode)
    out, st, spans = ob.attend_step(q, 32, hk, hv, total, ocfg, base, window, N.MODE_REATTENTION)
    assert res.stats.scope_len == st.scope_len
    assert np.array_equal(res.spans[0], spans[0]) and np.array_equal(res.spans[1], spans[1])
    err = np.abs(res.out.cpu().numpy() - out).max()
    assert err <= BF16_TOL
    assert err <= MEASURED_TOL, err
    assert abs(res.stats.entropy_max - st.entropy_max) <= 1e-4
    assert abs(res.stats.entropy_sum - st.entropy_sum) <= 1e-4 * n_q * 32


@pytest.mark.parametrize("n_q,total", [(1024, 40000), (4096, 65536)])
def test_prefill_attention_tc_vs_exact_gpu(ctx, n_q, total):
    """Larger prefill chunks: K6 against the f64 CUDA-core attention (itself oracle-pinned
    by test_gpu_parity), same scope."""
    cfg = N.SelectionConfig()
    cache, _, _ = make_cache(ctx, 8, 128, total, cfg, 800 + n_q)
    rope = N.Rope(ctx, 128, 500000.0, 16384)
    q = torch.empty(n_q, 32 * 128, dtype=torch.float32, device="cuda")
    ctx.synth_uniform(q, 801 + n_q)
    exact = step(ctx, cache, rope, q, 32, cfg, N.PREFILL_EXACT)
    tc = step(ctx, cache, rope, q, 32, cfg, N.PREFILL_TENSOR_ATTN)
    assert tc.stats.scope_len == exact.stats.scope_len
    err = (tc.out - exact.out).abs().max().item()
    assert err <= MEASURED_TOL, err
    assert abs(tc.stats.entropy_max - exact.stats.entropy_max) <= 1e-4


def test_prefill_attention_tc_window_mode(ctx):
    """AttentionMode::Window (no selection): scope = global ++ local, causal tail block."""
    cfg = N.SelectionConfig()
    cache, _, _ = make_cache(ctx, 8, 128, 9000, cfg, 900)
    rope = N.Rope(ctx, 128, 500000.0, 8192)
    q = torch.empty(300, 32 * 128, dtype=torch.float32, device="cuda")
    ctx.synth_uniform(q, 901)
    ctx.set_prefill(N.PREFILL_EXACT)
    exact = N.attend_step(ctx, cache, rope, q, 32, cfg, N.MODE_WINDOW)
    ctx.set_prefill(N.PREFILL_TENSOR_ATTN)
    try:
        tc = N.attend_step(ctx, cache, rope, q, 32, cfg, N.MODE_WINDOW)
    finally:
        ctx.set_prefill(N.PREFILL_DEFAULT)
    assert (tc.out - exact.out).abs().max().item() <= MEASURED_TOL
