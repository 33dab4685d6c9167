"""Batched decode (reattn_batch_plan_*): n_seq independent sequences with their own caches
in one graph.  Each sequence's output must equal the CPU oracle's attend_step (engine.hpp:
43-114) on that sequence's cache -- spans and L' identical, outputs and entropies within
1e-6 -- and the GPU's own single-sequence step (the pipelined path attends sequence b on a
few SMs beside scan b+1, so only the order of the fp32/f64 partial merges differs)."""
import numpy as np
import pytest

import oracle_bind as ob
import synth

torch = pytest.importorskip("torch")
from paper_2407_15176_b200 import native as N  # noqa: E402

pytestmark = pytest.mark.gpu
ATTN_TOL = 1e-6


def make(ctx, total, seed, dtype, cfg, n_kv=8, d=128):
    c = N.Cache(ctx, n_kv, d, cfg.l_global, cfg.l_local, total, dtype)
    ctx.synth_uniform(c.keys_tensor(), seed)
    ctx.synth_uniform(c.values_tensor(), seed + 1)
    c.set_total(total)
    return c


@pytest.mark.parametrize("dtype,totals,nh", [(N.BF16, [9000, 60000, 300000], 32),
                                             (N.BF16, [131072], 32),
                                             (N.BF16, [200000, 200000, 50000, 5000], 24),
                                             (N.F32, [7000, 20000], 32)])
def test_batch_plan_equals_single_steps(ctx, dtype, totals, nh):
    cfg = N.SelectionConfig()
    caches = [make(ctx, t, 40 + i, dtype, cfg) for i, t in enumerate(totals)]
    rope = N.Rope(ctx, 128, 500000.0, 8192)
    bp = N.BatchPlan(ctx, caches, rope, nh, cfg)
    info = bp.info()
    assert info["side_sms"] == (8 if dtype == N.BF16 and len(totals) > 1 else 0) or info["side_sms"] % 8 == 0
    for rep in range(2):
        q = torch.from_numpy(synth.uniform(90 + rep, len(totals) * nh * 128)
                             .reshape(len(totals), -1)).cuda()
        bp.q.copy_(q)
        torch.cuda.synchronize()
        bp.launch()
        torch.cuda.synchronize()
        for i, c in enumerate(caches):
            ref = N.attend_step(ctx, c, rope, q[i:i + 1], nh, cfg)
            st = bp.stats(i)
            assert st.scope_len == ref.stats.scope_len
            err = (bp.out[i:i + 1] - ref.out).abs().max().item()
            assert err <= ATTN_TOL, (i, err)
            assert abs(st.entropy_max - ref.stats.entropy_max) <= 1e-6
            if rep == 0:  # the oracle, on the cache's own bytes
                hk = c.keys_tensor().cpu().numpy() if dtype == N.F32 else ob.bf16_words(c.keys_tensor())
                hv = c.values_tensor().cpu().numpy() if dtype == N.F32 else ob.bf16_words(c.values_tensor())
                out, ent, ost, (sb, se), _ = ob.attend_step_ex(q[i:i + 1].cpu().numpy(), nh, hk, hv,
                                                               totals[i], ob.SelectionConfig(),
                                                               500000.0, 8192)
                assert st.scope_len == ost.scope_len, i
                assert np.array_equal(ref.spans[0], sb) and np.array_equal(ref.spans[1], se), i
                oerr = float(np.abs(bp.out[i:i + 1].cpu().numpy() - out).max())
                assert oerr <= ATTN_TOL, (i, oerr)
                assert abs(st.entropy_max - ost.entropy_max) <= 1e-6, i
    qh = q.cpu().pin_memory()
    oh = torch.empty_like(qh).pin_memory()
    bp.run_host(qh, oh)
    assert torch.equal(oh, bp.out.cpu())
