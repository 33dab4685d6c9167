"""Sequence-sharded decode on one GPU: W ranks' device stages run one after another in one
process (no kernel waits on another rank), the two all-gathers replaced by device copies.
The result must equal the unsharded attend_step: same spans and L', outputs within 1e-6
(the ranks attend disjoint scope rows with fp32 logits; only the merge order differs)."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
from paper_2407_15176_b200 import native as N  # noqa: E402
from paper_2407_15176_b200 import sharded as S  # noqa: E402

pytestmark = pytest.mark.gpu


def build_local_cache(ctx, gk, gv, total, cfg, world, rank, dtype):
    segs = S.local_row_segments(total, cfg, world, rank)
    rows = sum(e - b for b, e in segs)
    n_kv, _, d = gk.shape
    c = N.Cache(ctx, n_kv, d, cfg.l_global, cfg.l_local, rows, dtype)
    kt, vt = c.keys_tensor(), c.values_tensor()
    o = 0
    for b, e in segs:
        kt[:, o:o + e - b].copy_(gk[:, b:e])
        vt[:, o:o + e - b].copy_(gv[:, b:e])
        o += e - b
    torch.cuda.synchronize()
    c.set_total(rows)
    return c


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("total", [40000, 300000])
def test_sharded_equals_unsharded(ctx, world, total):
    cfg = N.SelectionConfig()
    n_kv, nh, d = 8, 32, 128
    gcache = N.Cache(ctx, n_kv, d, cfg.l_global, cfg.l_local, total, N.BF16)
    ctx.synth_uniform(gcache.keys_tensor(), 77)
    ctx.synth_uniform(gcache.values_tensor(), 78)
    gcache.set_total(total)
    rope = N.Rope(ctx, d, 500000.0, 8192)
    gk, gv = gcache.keys_tensor(), gcache.values_tensor()
    ops = [S.NativeOps(ctx, build_local_cache(ctx, gk, gv, total, cfg, world, r, N.BF16), rope,
                       nh, cfg, total, world, r) for r in range(world)]
    for step in range(2):
        q = torch.from_numpy(synth.uniform(500 + step, nh * d).reshape(1, -1)).cuda()
        ref = N.attend_step(ctx, gcache, rope, q, nh, cfg)
        for o in ops:
            o.q.copy_(q)
        torch.cuda.synchronize()
        for o in ops:
            o.scan()
        ctx.synchronize()
        cand = torch.cat([o.cand_send for o in ops])
        for o in ops:
            o.cand_recv.copy_(cand)
        torch.cuda.synchronize()
        for o in ops:
            o.select()
            o.attend()
        ctx.synchronize()
        part = torch.cat([o.part_send for o in ops])
        for o in ops:
            o.part_recv.copy_(part)
        torch.cuda.synchronize()
        for o in ops:
            o.combine()
        ctx.synchronize()
        for r, o in enumerate(ops):
            st, (sb, se) = o.stats(cfg.k_prime)
            assert st.scope_len == ref.stats.scope_len, (world, r)
            assert np.array_equal(sb, ref.spans[0]) and np.array_equal(se, ref.spans[1]), (world, r)
            err = (o.out - ref.out).abs().max().item()
            assert err <= 1e-6, (world, r, err)
            assert abs(st.entropy_max - ref.stats.entropy_max) <= 1e-6


def test_shard_range_matches_c_rule(ctx):
    for M in (0, 1, 31, 32, 1000, 1044448, 4190176):
        for world in (1, 2, 3, 4, 7, 8):
            prev = 0
            for r in range(world):
                b, n = N.u64(), N.u64()
                assert ctx.lib.reattn_shard_range(M, 32, world, r, N.C.byref(b), N.C.byref(n)) == 0
                assert (b.value, n.value) == S.shard_range(M, 32, world, r)
                assert b.value == prev and (b.value % 32 == 0 or b.value == M)
                prev = b.value + n.value
            assert prev == M


def test_library_nccl_step_world1(ctx):
    """The product host path (sharded.NcclDecodeStep over reattn_shard_step / _capture: the
    library's own NCCL communicator issues both all-gathers) at world size 1 on this GPU,
    eager and graph-captured, equals the unsharded step; end to end through
    reattn_shard_run_host as well."""
    cfg = N.SelectionConfig()
    n_kv, nh, d, total = 8, 32, 128, 60000
    cache = N.Cache(ctx, n_kv, d, cfg.l_global, cfg.l_local, total, N.BF16)
    ctx.synth_uniform(cache.keys_tensor(), 81)
    ctx.synth_uniform(cache.values_tensor(), 82)
    cache.set_total(total)
    rope = N.Rope(ctx, d, 500000.0, 8192)
    ops = S.NativeOps(ctx, cache, rope, nh, cfg, total, 1, 0)
    step = S.NcclDecodeStep(ops, S.NcclComm(ctx, 1, 0))
    for rep in range(3):
        if rep == 1:
            step.capture()
        q = torch.from_numpy(synth.uniform(900 + rep, nh * d).reshape(1, -1)).cuda()
        ref = N.attend_step(ctx, cache, rope, q, nh, cfg)
        out = step.step(q)
        torch.cuda.synchronize()
        assert (out - ref.out).abs().max().item() <= 1e-6, rep
        st, spans = ops.stats(cfg.k_prime)
        assert st.scope_len == ref.stats.scope_len and np.array_equal(spans[0], ref.spans[0])
    qh = q.cpu().pin_memory()
    oh = torch.empty_like(qh).pin_memory()
    step.run_host(qh, oh)
    assert (oh - ref.out.cpu()).abs().max().item() <= 1e-6
