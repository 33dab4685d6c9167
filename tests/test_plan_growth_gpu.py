"""One decode plan across a growing cache (engine.hpp:163-198 appends a row every decode step,
kv_cache.hpp:54-68 promotes the oldest local row into the middle).

A decode plan reads the cache length from the device, so the SAME graph is replayed after
every append -- through reattn_cache_append or through the plan's own append node -- and each
replay must equal the oracle's attend_step on the cache as it is then (spans, L', outputs
<= 1e-6).  Frozen plan shapes and reallocated storage are refused instead of silently
attending a stale scope."""
import numpy as np
import pytest

import oracle_bind as ob
import synth

torch = pytest.importorskip("torch")
from paper_2407_15176_b200 import native as N  # noqa: E402

pytestmark = pytest.mark.gpu

TOL = 1e-6


def host_words(cache, dtype):
    if dtype == N.F32:
        return cache.keys_tensor().cpu().numpy(), cache.values_tensor().cpu().numpy()
    return ob.bf16_words(cache.keys_tensor()), ob.bf16_words(cache.values_tensor())


def check_vs_oracle(plan, cache, dtype, q, total, nh=32, label=""):
    res = plan.result(127)
    hk, hv = host_words(cache, dtype)
    out, ent, st, (sb, se), _ = ob.attend_step_ex(q.cpu().numpy(), nh, hk, hv, total,
                                                  ob.SelectionConfig(), 500000.0, 8192)
    assert res.stats.scope_len == st.scope_len, label
    assert np.array_equal(res.spans[0], sb) and np.array_equal(res.spans[1], se), label
    err = float(np.abs(res.out.cpu().numpy() - out).max())
    assert err <= TOL, (label, err)
    assert float(np.abs(res.entropy - ent).max()) <= TOL, label


def kv_rows(seed, rows, n_kv=8, d=128, bf16=True):
    k = synth.uniform(seed, rows * n_kv * d, bf16=bf16).reshape(rows, n_kv * d)
    v = synth.uniform(seed + 1, rows * n_kv * d, bf16=bf16).reshape(rows, n_kv * d)
    return k, v


@pytest.mark.parametrize("dtype,fork", [(N.BF16, "0"), (N.BF16, "1"), (N.F32, "0")])
def test_one_plan_follows_appends(ctx, dtype, fork, monkeypatch):
    monkeypatch.setenv("REATTN_FORK", fork)
    cfg = N.SelectionConfig()
    total = 50000
    cache = N.Cache(ctx, 8, 128, cfg.l_global, cfg.l_local, total + 64, dtype)
    ctx.synth_uniform(cache.keys_tensor(), 71)
    ctx.synth_uniform(cache.values_tensor(), 72)
    cache.set_total(total)
    rope = N.Rope(ctx, 128, 500000.0, 8192)
    plan = N.Plan(ctx, cache, rope, 1, 32, cfg)
    q = torch.empty(1, 32 * 128, device="cuda")
    for step, rows in enumerate([0, 1, 3, 1, 29]):
        if rows:
            k, v = kv_rows(900 + step, rows, bf16=dtype == N.BF16)
            cache.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
            total += rows
        ctx.synth_uniform(q, 500 + step)
        plan.q.copy_(q)
        torch.cuda.synchronize()
        plan.launch()
        plan.stage_result()  # the engine's per-layer path: copies behind the replay, one sync
        torch.cuda.synchronize()
        staged = plan.result(127, staged=True)
        check_vs_oracle(plan, cache, dtype, q, total, label=f"step {step} total {total}")
        direct = plan.result(127)
        assert staged.stats.scope_len == direct.stats.scope_len
        assert staged.stats.entropy_max == direct.stats.entropy_max
        assert np.array_equal(staged.spans[0], direct.spans[0])
        assert np.array_equal(staged.spans[1], direct.spans[1])
        assert np.array_equal(staged.entropy, direct.entropy)


@pytest.mark.parametrize("fork", ["0", "1"])
def test_append_node_in_the_graph(ctx, fork, monkeypatch):
    """Append mode: each replay appends the step's K/V rows, then attends (forward_block's
    order, engine.hpp:196-198); the cache grows by one row per replay."""
    monkeypatch.setenv("REATTN_FORK", fork)
    cfg = N.SelectionConfig()
    total = 40000
    cache = N.Cache(ctx, 8, 128, cfg.l_global, cfg.l_local, total + 5, N.BF16)
    ctx.synth_uniform(cache.keys_tensor(), 81)
    ctx.synth_uniform(cache.values_tensor(), 82)
    cache.set_total(total)
    rope = N.Rope(ctx, 128, 500000.0, 8192)
    plan = N.Plan(ctx, cache, rope, 1, 32, cfg)
    plan.set_append(True)
    for step in range(4):
        k, v = kv_rows(1000 + step, 1)
        plan.k_in.copy_(torch.from_numpy(k.ravel()))
        plan.v_in.copy_(torch.from_numpy(v.ravel()))
        ctx.synth_uniform(plan.q, 600 + step)
        q = plan.q.clone()
        torch.cuda.synchronize()
        plan.launch()
        total += 1
        assert cache.info()["total"] == total
        check_vs_oracle(plan, cache, N.BF16, q, total, label=f"append step {step}")
    # the end-to-end host entry point appends too
    k, v = kv_rows(2000, 1)
    qh = torch.from_numpy(synth.uniform(700, 32 * 128).reshape(1, -1)).pin_memory()
    oh = torch.zeros_like(qh).pin_memory()
    kh = torch.from_numpy(np.ascontiguousarray(k.ravel())).pin_memory()
    vh = torch.from_numpy(np.ascontiguousarray(v.ravel())).pin_memory()
    plan.step_host(qh, kh, vh, oh)
    total += 1
    res = plan.result(127)
    assert torch.equal(oh, res.out.cpu())
    check_vs_oracle(plan, cache, N.BF16, qh, total, label="step_host")
    # capacity: 5 rows were reserved
    with pytest.raises(N.ReattnError, match="capacity exceeded"):
        plan.launch()


def test_frozen_and_reallocated_plans_are_refused(ctx):
    cfg = N.SelectionConfig()
    cache = N.Cache(ctx, 8, 128, cfg.l_global, cfg.l_local, 30000, N.BF16)
    ctx.synth_uniform(cache.keys_tensor(), 91)
    ctx.synth_uniform(cache.values_tensor(), 92)
    cache.set_total(20000)
    rope = N.Rope(ctx, 128, 500000.0, 8192)
    frozen = N.Plan(ctx, cache, rope, 2, 32, cfg)  # a 2-query block: frozen shape
    decode = N.Plan(ctx, cache, rope, 1, 32, cfg)
    with pytest.raises(N.InvalidArgument, match="append"):
        frozen.set_append(True)
    frozen.launch()
    cache.set_total(20001)
    with pytest.raises(N.ReattnError, match="length changed"):
        frozen.launch()
    decode.launch()  # follows the length
    decode.stats()
    ctx.check(ctx.lib.reattn_cache_reserve(ctx.h, cache.h, 60000))
    with pytest.raises(N.ReattnError, match="reallocated"):
        decode.launch()
