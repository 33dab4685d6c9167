"""GPU parity: the sm_100a kernels (through the C-ABI) vs the CPU oracle (oracle/).

Bars (north_star): selected indices and fp32 scores bit-identical (eps = 0 — the kernels
emulate the reference's exact lane arithmetic); attention outputs max-abs <= 1e-5 (we hold
them to 1e-6, the reference's own attend-vs-long-double bar, test_numerics.cpp:295),
entropies <= 1e-9.  Mirrors the reference's tests: test_selection.cpp, test_scope.cpp,
test_numerics.cpp, test_engine.cpp, acceptance_test.cpp C01/C04/C05/C09.
"""
import numpy as np
import pytest

import oracle_bind as ob
import synth

torch = pytest.importorskip("torch")
from paper_2407_15176_b200 import native as N  # noqa: E402

pytestmark = pytest.mark.gpu

ATTN_TOL = 1e-6
ENT_TOL = 1e-9
# decode attention (n_q == 1, d == 128) computes logits in fp32 (f64 state across chunks):
# outputs stay within ATTN_TOL, row entropies within 1e-6 of the f64 reference
DEC_ENT_TOL = 1e-6


def dev(x, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return t if dtype is None else t.to(dtype)


def gpu_topk(ctx, q, n_heads, keys_hm, k, dtype=N.F32, head_stride=None, row0=0, count=None):
    """keys_hm: numpy [n_kv, rows, d] fp32 (bf16-representable when dtype == BF16)."""
    n_kv, rows, d = keys_hm.shape
    count = rows - row0 if count is None else count
    kt = dev(keys_hm, torch.bfloat16 if dtype == N.BF16 else torch.float32)
    qt = dev(q.astype(np.float32))
    n_q = q.shape[0]
    idx = torch.zeros(n_kv * n_q * k, dtype=torch.int32, device="cuda")
    sc = torch.zeros(n_kv * n_q * k, dtype=torch.float32, device="cuda")
    n_out, scratch = ctx.fused_topk(qt, n_heads, kt, n_kv, head_stride or rows, row0, count, d, k,
                                    idx, sc, dtype)
    i = idx.cpu().numpy().view(np.uint32).reshape(n_kv, n_q, k)[:, :, :n_out].astype(np.uint64)
    s = sc.cpu().numpy().reshape(n_kv, n_q, k)[:, :, :n_out]
    return i, s, scratch


def oracle_topk(q, n_heads, keys_hm, k, lanes, row0=0, count=None):
    n_kv, rows, d = keys_hm.shape
    count = rows - row0 if count is None else count
    heads = [np.ascontiguousarray(keys_hm[h, row0:row0 + count]) for h in range(n_kv)]
    with ob.lane_mode(lanes):
        return ob.topk(q, n_heads, heads, k)


def assert_topk_equal(got, want, label=""):
    gi, gs = got[0], got[1]
    wi, ws = want
    assert gi.shape == wi.shape, label
    assert np.array_equal(gi, wi), f"{label}: index mismatch\n{gi}\n{wi}"
    # bit-identical scores (a zero score may differ only in its sign: == treats them equal)
    assert np.array_equal(gs, ws), f"{label}: scores differ\n{gs}\n{ws}"
    nz = gs != 0
    assert np.array_equal(gs[nz].view(np.uint32), ws[nz].view(np.uint32)), label


# ---------------------------------------------------------------------------------------
def test_synth_generator_matches_host(ctx):
    for dt in (torch.float32, torch.bfloat16):
        t = torch.empty(100003, dtype=dt, device="cuda")
        ctx.synth_uniform(t, seed=77, offset=5)
        want = synth.uniform(77, 100003, offset=5)
        if dt == torch.bfloat16:
            want = synth.bf16_round(want)
        assert np.array_equal(t.float().cpu().numpy(), want)


@pytest.mark.parametrize("lanes", [N.LANES_UNFUSED, N.LANES_FMA])
@pytest.mark.parametrize("dtype", [N.BF16, N.F32])
def test_fast_scan_decode_geometry(ctx, lanes, dtype):
    """K1 fast path: LLaMA-3.1-8B heads (32 q / 8 kv, d=128), n_q=1, k in 1..8, sizes that
    straddle the 224/128-row TMA tiles and the per-CTA split."""
    ctx.set_lanes(lanes)
    try:
        for count, k, seed in [(1, 4, 1), (3, 4, 2), (4, 4, 3), (5, 8, 4), (223, 4, 5), (224, 4, 6),
                               (225, 1, 7), (4097, 8, 8), (28640, 4, 9), (126944, 4, 10)]:
            n_kv, d, nh = 8, 128, 32
            rows = count + 37
            keys = synth.uniform(seed, n_kv * rows * d).reshape(n_kv, rows, d)
            if dtype == N.BF16:
                keys = synth.bf16_round(keys)
            q = synth.uniform(seed + 1000, nh * d).reshape(1, nh * d)
            got = gpu_topk(ctx, q, nh, keys, k, dtype, row0=32, count=count)
            want = oracle_topk(q, nh, keys, k, lanes, row0=32, count=count)
            assert_topk_equal(got, want, f"count={count} k={k}")
    finally:
        ctx.set_lanes(N.LANES_UNFUSED)


@pytest.mark.parametrize("lanes", [N.LANES_UNFUSED, N.LANES_FMA])
def test_generic_scan_matches_oracle(ctx, lanes):
    """Generic path: test_selection.cpp:105-131 sizes x k (incl. large k), several d / n_q /
    GQA groups, fp32 keys."""
    ctx.set_lanes(lanes)
    rng = np.random.default_rng(31)
    try:
        for count in [0, 1, 3, 4, 5, 127, 1000, 2047, 2048, 2049, 10000]:
            for k in (1, 4, 8, 100):
                n_kv = 1 + count % 2
                nh = n_kv * (1 + (count + k) % 3)
                d = [32, 16, 8, 24, 128][(count + k) % 5]
                n_q = 1 + (count + k) % 5
                keys = rng.uniform(-1, 1, (n_kv, count, d)).astype(np.float32)
                q = rng.uniform(-1, 1, (n_q, nh * d)).astype(np.float32)
                got = gpu_topk(ctx, q, nh, keys, k)
                want = oracle_topk(q, nh, keys, k, lanes)
                assert_topk_equal(got, want, f"count={count} k={k} d={d} n_q={n_q}")
    finally:
        ctx.set_lanes(N.LANES_UNFUSED)


def test_topk_ties_keep_lower_index(ctx):
    """test_selection.cpp:168-191 known answer: ten equal keys -> {0, 7, 15, 16}."""
    d, L = 8, 64
    data = np.zeros((1, L, d), np.float32)
    for i in (0, 7, 15, 16, 17, 31, 32, 49, 62, 63):
        data[0, i] = 0.5
    q = np.ones((1, d), np.float32)
    i, s, _ = gpu_topk(ctx, q, 1, data, 4)
    assert list(i[0, 0]) == [0, 7, 15, 16]
    # same on the fast path (d=128, bf16)
    d = 128
    data = np.zeros((8, 3000, d), np.float32)
    for h in range(8):
        for r in (0, 7, 15, 16, 17, 31, 32, 49, 62, 63, 1500, 2999):
            data[h, r] = 0.5
    q = np.ones((1, 32 * d), np.float32)
    i, s, _ = gpu_topk(ctx, q, 32, data, 4, N.BF16)
    assert all(list(i[h, 0]) == [0, 7, 15, 16] for h in range(8))


def test_scratch_independent_of_middle_length(ctx):
    """test_selection.cpp:210-231 / acceptance C06: device workspace is flat in middle len."""
    scr = []
    for count in (4096, 262144):
        keys = synth.uniform(5, count * 32).reshape(1, count, 32)
        q = synth.uniform(6, 4 * 32).reshape(4, 32)
        scr.append(gpu_topk(ctx, q, 1, keys, 4)[2])
    assert scr[0] == scr[1]


def test_vote_and_tally_match_oracle(ctx):
    """test_selection.cpp:233-298 (map oracle) via the reference-restating oracle."""
    rng = np.random.default_rng(53)
    for it in range(300):
        n = int(rng.integers(1, 200))
        idx = rng.integers(0, 50, n).astype(np.uint64)
        score = (rng.integers(0, 1000, n) / 500.0 - 1.0).astype(np.float32)
        kp = int(rng.integers(1, 25))
        want = ob.vote(idx, score, kp)
        w = torch.zeros(kp, dtype=torch.int32, device="cuda")
        nw = ctx.vote(dev(idx.astype(np.int32)), dev(score), kp, w)
        got = w.cpu().numpy()[:nw].astype(np.uint64)
        assert np.array_equal(got, want), it
    # known answers (test_selection.cpp:272-292)
    for idx, sc, kp, want in [([9, 2, 7], [5.0, 3.0, 1.0], 2, [9, 2]),
                              ([7, 3, 7, 5], [0.1, 9.0, 0.2, 0.05], 3, [7, 3, 5])]:
        w = torch.zeros(kp, dtype=torch.int32, device="cuda")
        nw = ctx.vote(dev(np.array(idx, np.int32)), dev(np.array(sc, np.float32)), kp, w)
        assert list(w.cpu().numpy()[:nw]) == want


def test_expand_spans_match_oracle(ctx):
    rng = np.random.default_rng(59)
    for it in range(200):
        mode = it % 2
        m = 1 + it % 64 if mode == 0 else 2 + it % 63
        L = int(rng.integers(m, 100000))
        wn = rng.integers(0, L, int(rng.integers(1, 128))).astype(np.uint64)
        want = ob.expand_spans(wn, m, L, mode)
        b = torch.zeros(len(wn), dtype=torch.int32, device="cuda")
        e = torch.zeros_like(b)
        ns = ctx.expand_spans(dev(wn.astype(np.int32)), m, L, mode, b, e)
        assert np.array_equal(b.cpu().numpy()[:ns].astype(np.uint64), want[0]), it
        assert np.array_equal(e.cpu().numpy()[:ns].astype(np.uint64), want[1]), it
    # known answers (test_selection.cpp:325-337) and the range error (:373-376)
    b = torch.zeros(2, dtype=torch.int32, device="cuda")
    e = torch.zeros_like(b)
    assert ctx.expand_spans(dev(np.array([5, 20], np.int32)), 32, 100, 0, b, e) == 1
    assert (b[0].item(), e[0].item()) == (0, 32)
    assert ctx.expand_spans(dev(np.array([98], np.int32)), 32, 100, 0, b, e) == 1
    assert (b[0].item(), e[0].item()) == (96, 100)
    with pytest.raises(N.OutOfRange, match="expand_spans: winner outside middle"):
        ctx.expand_spans(dev(np.array([100], np.int32)), 32, 100, 0, b, e)


def test_attend_matches_oracle(ctx):
    """test_numerics.cpp:281-302: 1000-instance style fuzz (fewer here), f64 state."""
    rng = np.random.default_rng(23)
    for it in range(200):
        n_q, L, d = int(rng.integers(1, 9)), int(rng.integers(1, 513)), int(rng.integers(4, 65)) & ~1
        dv = d if it % 3 else max(2, d // 2)
        q = rng.uniform(-1, 1, (n_q, d)).astype(np.float32)
        k = rng.uniform(-1, 1, (L, d)).astype(np.float32)
        v = rng.uniform(-1, 1, (L, dv)).astype(np.float32)
        bd = L - n_q if (it % 2 == 0 and L >= n_q) else None
        out = torch.zeros(n_q, dv, device="cuda")
        ent = torch.zeros(n_q, dtype=torch.float64, device="cuda")
        ctx.attend(dev(q), dev(k), dev(v), bd, out, ent)
        wo, we = ob.attend(q, k, v, bd)
        assert np.abs(out.cpu().numpy() - wo).max() <= ATTN_TOL, it
        assert np.abs(ent.cpu().numpy() - we).max() <= ENT_TOL, it
    with pytest.raises(N.InvalidArgument, match="empty key set"):
        ctx.attend(dev(np.zeros((1, 8), np.float32)), dev(np.zeros((0, 8), np.float32)),
                   dev(np.zeros((0, 8), np.float32)), None, out, ent)


def test_rope_tables_and_rotation(ctx):
    r = N.Rope(ctx, 128, 500000.0, 8192)
    c, s = r.tables()
    wc, ws = ob.rope_table(128, 500000.0, 8192)
    assert np.array_equal(c, wc) and np.array_equal(s, ws)
    rows = synth.uniform(3, 16 * 128).reshape(16, 128)
    pos = np.array([0, 1, 5, 100, 4095, 8191] + list(range(10)), np.uint64)
    t = dev(rows)
    r.rotate(t, pos)
    want = rows.copy()
    for i in range(16):
        row = want[i].copy()
        ob.oracle().oracle_rotate_row(row, 128, wc[pos[i]].copy(), ws[pos[i]].copy())
        want[i] = row
    assert np.array_equal(t.cpu().numpy(), want)
    with pytest.raises(N.OutOfRange, match="position out of pretrained range"):
        r.rotate(t[:1], [8192])


# ---------------------------------------------------------------------------------------
def make_cache(ctx, n_kv, d, total, cfg, dtype, seed, extra=0):
    """Device cache filled with synthetic rows; returns (cache, host fp32 K, host fp32 V)."""
    cap = total + extra
    cache = N.Cache(ctx, n_kv, d, cfg.l_global, cfg.l_local, cap, dtype)
    kt, vt = cache.keys_tensor(), cache.values_tensor()
    ctx.synth_uniform(kt, seed)
    ctx.synth_uniform(vt, seed + 1)
    cache.set_total(total)
    return cache, kt.float().cpu().numpy(), vt.float().cpu().numpy()


def step_vs_oracle(ctx, n_kv, nh, d, total, cfg, dtype, seed, window, base=500000.0, n_q=1,
                   mode=N.MODE_REATTENTION):
    cache, hk, hv = make_cache(ctx, n_kv, d, total, cfg, dtype, seed)
    rope = N.Rope(ctx, d, base, window)
    q = synth.uniform(seed + 7, n_q * nh * d).reshape(n_q, nh * d)
    res = N.attend_step(ctx, cache, rope, dev(q), nh, cfg, mode)
    ocfg = ob.SelectionConfig(cfg.k, cfg.k_prime, cfg.span_m, cfg.tile_size, cfg.l_global,
                              cfg.l_local, cfg.l_chunk, cfg.span_mode)
    out, st, spans = ob.attend_step(q, nh, hk, hv, total, ocfg, base, window, mode)
    return res, out, st, spans


@pytest.mark.parametrize("total", [100, 4128, 4200, 9000, 40000, 131072])
def test_attend_step_llama_geometry_bf16(ctx, total):
    """engine.hpp:43 attend_step at LLaMA-3.1-8B head geometry, bf16 cache, defaults."""
    cfg = N.SelectionConfig()
    res, out, st, spans = step_vs_oracle(ctx, 8, 32, 128, total, cfg, N.BF16, 11 + total, 8192)
    assert res.stats.scope_len == st.scope_len
    assert np.array_equal(res.spans[0], spans[0]) and np.array_equal(res.spans[1], spans[1])
    assert np.abs(res.out.cpu().numpy() - out).max() <= ATTN_TOL
    assert abs(res.stats.entropy_max - st.entropy_max) <= DEC_ENT_TOL
    assert abs(res.stats.entropy_sum - st.entropy_sum) <= 32 * DEC_ENT_TOL
    assert res.stats.max_position_used == st.max_position_used
    assert bool(res.stats.coverage_total) == bool(st.coverage_total)


@pytest.mark.parametrize("n_kv,nh,d,dtype,total", [(96, 96, 128, N.BF16, 20000),  # > 64 kv heads
                                                    (8, 32, 64, N.BF16, 30000),     # d = 64
                                                    (4, 16, 256, N.F32, 12000),     # d = 256
                                                    (2, 14, 128, N.BF16, 50000)])   # group 7
def test_attend_step_decode_geometries(ctx, n_kv, nh, d, dtype, total):
    """Decode steps away from the LLaMA geometry: more than 64 kv heads (the decode
    attention's per-head tickets), head dims 64 / 256 (the generic scan and
    attention), group 7 -- spans, L' and outputs against the oracle; then a plan replayed
    twice on the same cache."""
    cfg = N.SelectionConfig()
    res, out, st, spans = step_vs_oracle(ctx, n_kv, nh, d, total, cfg, dtype, 333 + d, 8192)
    assert res.stats.scope_len == st.scope_len
    assert np.array_equal(res.spans[0], spans[0]) and np.array_equal(res.spans[1], spans[1])
    assert np.abs(res.out.cpu().numpy() - out).max() <= ATTN_TOL
    cache, _, _ = make_cache(ctx, n_kv, d, total, cfg, dtype, 333 + d)
    rope = N.Rope(ctx, d, 500000.0, 8192)
    plan = N.Plan(ctx, cache, rope, 1, nh, cfg)
    plan.q.copy_(dev(synth.uniform(333 + d + 7, nh * d).reshape(1, nh * d)))
    for _ in range(2):
        plan.launch()
        r = plan.result(cfg.k_prime)
        assert r.stats.scope_len == st.scope_len
        assert np.abs(r.out.cpu().numpy() - out).max() <= ATTN_TOL


@pytest.mark.parametrize("k,n_q,total", [(4, 160, 16000), (16, 96, 12000), (4, 129, 5000), (4, 256, 4200)])
def test_attend_step_prefill_default_mode(ctx, k, n_q, total):
    """A fresh context's prefill path (REATTN_PREFILL_TENSOR: the tcgen05 score GEMM where
    k <= 8, the exact scan otherwise; tcgen05 scope attention) against the oracle: spans and
    L' exactly, outputs within 2e-4 (north_star bf16 bar 1e-2); a middle that is empty or
    shorter than k' spans included."""
    c = N.Context(0)  # default prefill mode
    cfg = N.SelectionConfig(k=k)
    res, out, st, spans = step_vs_oracle(c, 8, 32, 128, total, cfg, N.BF16, 900 + k + n_q, 8192,
                                         base=1e6, n_q=n_q)
    assert res.stats.scope_len == st.scope_len
    assert np.array_equal(res.spans[0], spans[0]) and np.array_equal(res.spans[1], spans[1])
    assert np.abs(res.out.cpu().numpy() - out).max() <= 2e-4


@pytest.mark.parametrize("seed", range(64))
def test_attend_step_randomized_vs_oracle(ctx, seed):
    """Random geometries and selection settings (kv heads, group, head dim, dtype, cache
    length, k, k', span_m, both span modes, l_global, l_local, decode or a prefill block),
    each against the oracle: spans and L' exactly, stats, outputs within 1e-6 (exact paths)
    or 2e-4 (the tcgen05 prefill attention on bf16 d=128).  Errors must match too: when the
    oracle raises (e.g. the query block longer than the scope) the device raises the same."""
    rng = np.random.default_rng(1000 + seed)
    n_kv = int(rng.choice([1, 2, 4, 8]))
    group = int(rng.choice([1, 2, 3, 4]))
    d = int(rng.choice([16, 32, 64, 128]))
    dtype = N.BF16 if rng.random() < 0.6 else N.F32
    l_local = int(rng.choice([16, 64, 256, 512]))
    l_global = int(rng.integers(0, 65))
    span_m = int(rng.choice([1, 4, 16, 32, 64]))
    k = int(rng.integers(1, 9))
    k_prime = int(rng.integers(0, 65))
    window = 8192
    while l_global + k_prime * span_m + l_local > window:
        k_prime //= 2
    n_q = 1 if rng.random() < 0.6 else int(rng.integers(2, min(64, l_local) + 1))
    cfg = N.SelectionConfig(k=k, k_prime=k_prime, span_m=span_m, l_global=l_global, l_local=l_local,
                            l_chunk=max(1, min(l_local, 128)), span_mode=int(rng.integers(0, 2)))
    total = int(rng.integers(n_q, 20000))
    nh = n_kv * group
    label = (n_kv, nh, d, dtype, total, n_q, k, k_prime, span_m, l_global, l_local, cfg.span_mode)
    ocfg = ob.SelectionConfig(cfg.k, cfg.k_prime, cfg.span_m, cfg.tile_size, cfg.l_global,
                              cfg.l_local, cfg.l_chunk, cfg.span_mode)
    cache, hk, hv = make_cache(ctx, n_kv, d, total, cfg, dtype, 2000 + seed)
    rope = N.Rope(ctx, d, 10000.0, window)
    q = synth.uniform(2100 + seed, n_q * nh * d).reshape(n_q, nh * d)
    try:
        out, st, spans = ob.attend_step(q, nh, hk, hv, total, ocfg, 10000.0, window)
    except Exception as e:  # the reference's error: the device must raise it too
        with pytest.raises(N.ReattnError):
            N.attend_step(ctx, cache, rope, dev(q), nh, cfg)
        return
    res = N.attend_step(ctx, cache, rope, dev(q), nh, cfg)
    assert res.stats.scope_len == st.scope_len, label
    assert np.array_equal(res.spans[0], spans[0]) and np.array_equal(res.spans[1], spans[1]), label
    tol = 2e-4 if (n_q > 1 and dtype == N.BF16 and d == 128) else ATTN_TOL
    assert np.abs(res.out.cpu().numpy() - out).max() <= tol, label
    # the same step as a plan (decode plans follow the device cache length), replayed twice
    plan = N.Plan(ctx, cache, rope, n_q, nh, cfg)
    plan.q.copy_(dev(q))
    for _ in range(2):
        plan.launch()
        r = plan.result(max(1, k_prime))
        assert r.stats.scope_len == st.scope_len, label
        assert np.array_equal(r.spans[0], spans[0]) and np.array_equal(r.spans[1], spans[1]), label
        assert np.abs(r.out.cpu().numpy() - out).max() <= tol, label


@pytest.mark.parametrize("case", range(8))
def test_attend_step_toy_geometries(ctx, case):
    """test_engine.cpp toy_selection-like configs, fp32 caches, prefill-sized n_q, both span
    modes and the window mode (k'=0 / AttentionMode::Window)."""
    rng = np.random.default_rng(case)
    cfg = N.SelectionConfig(k=4, k_prime=64, span_m=16, l_global=16, l_local=256, l_chunk=128)
    cfg.span_mode = case % 2
    if case == 5:
        cfg.k_prime = 0
    n_q = [1, 4, 128, 1, 32, 7, 40, 16][case]
    total = [300, 1000, 2000, 5000, 777, 4200, 3000, 20000][case]
    mode = N.MODE_WINDOW if case == 7 else N.MODE_REATTENTION
    if case == 6:
        cfg.k, cfg.k_prime = 100, 100
    res, out, st, spans = step_vs_oracle(ctx, 2, 4, 16, total, cfg, N.F32, 100 + case, 2048,
                                         base=10000.0, n_q=n_q, mode=mode)
    assert res.stats.scope_len == st.scope_len
    assert np.array_equal(res.spans[0], spans[0])
    assert np.abs(res.out.cpu().numpy() - out).max() <= ATTN_TOL
    assert abs(res.stats.entropy_max - st.entropy_max) <= ENT_TOL


def test_attend_step_errors(ctx):
    cfg = N.SelectionConfig(l_global=4, l_local=8, k_prime=2, span_m=4)
    cache, _, _ = make_cache(ctx, 1, 4, 12, cfg, N.F32, 3)
    rope = N.Rope(ctx, 4, 10000.0, 11)
    q = dev(np.zeros((1, 4), np.float32))
    with pytest.raises(N.InvalidArgument, match="scope exceeds pretrain window"):
        N.attend_step(ctx, cache, rope, q, 1, cfg)
    rope = N.Rope(ctx, 4, 10000.0, 64)
    with pytest.raises(N.LogicError, match="query block longer than scope"):
        N.attend_step(ctx, cache, rope, dev(np.zeros((13, 4), np.float32)), 1, cfg)
    with pytest.raises(N.InvalidArgument, match="multiple of kv heads"):
        cache2, _, _ = make_cache(ctx, 3, 4, 12, cfg, N.F32, 3)
        N.attend_step(ctx, cache2, rope, dev(np.zeros((1, 16), np.float32)), 4, cfg)


def test_plan_graph_replay_matches_step(ctx):
    """The CUDA-graph plan replays exactly the synchronous attend_step (bitwise)."""
    cfg = N.SelectionConfig()
    cache, _, _ = make_cache(ctx, 8, 128, 60000, cfg, N.BF16, 21)
    rope = N.Rope(ctx, 128, 500000.0, 8192)
    plan = N.Plan(ctx, cache, rope, 1, 32, cfg)
    for s in range(3):
        q = dev(synth.uniform(300 + s, 32 * 128).reshape(1, -1))
        ref = N.attend_step(ctx, cache, rope, q, 32, cfg)
        plan.q.copy_(q)
        torch.cuda.synchronize()
        plan.launch()
        st = plan.stats()
        assert torch.equal(plan.out, ref.out), \
            (s, (plan.out - ref.out).abs().max().item(), st.scope_len, ref.stats.scope_len)
        assert st.scope_len == ref.stats.scope_len
        qh = q.cpu().pin_memory()
        oh = torch.empty_like(qh).pin_memory()
        plan.run_host(qh, oh)
        assert torch.equal(oh, ref.out.cpu())


def test_plan_adaptive_partition_replays(ctx, monkeypatch):
    """The adaptive scan partition (forced on at this size) changes the CTAs' tile ranges
    between replays; the selection is exact under any partition, so every replay must equal the
    synchronous step bitwise."""
    monkeypatch.setenv("REATTN_BALANCE_MIN_TILES", "1")
    cfg = N.SelectionConfig()
    cache, _, _ = make_cache(ctx, 8, 128, 90000, cfg, N.BF16, 23)
    rope = N.Rope(ctx, 128, 500000.0, 8192)
    plan = N.Plan(ctx, cache, rope, 1, 32, cfg)
    for s in range(8):
        q = dev(synth.uniform(400 + s % 3, 32 * 128).reshape(1, -1))
        ref = N.attend_step(ctx, cache, rope, q, 32, cfg)
        plan.q.copy_(q)
        torch.cuda.synchronize()
        plan.launch()
        st = plan.stats()
        assert torch.equal(plan.out, ref.out), (s, (plan.out - ref.out).abs().max().item())
        assert st.scope_len == ref.stats.scope_len


def test_vote_large_candidate_sets(ctx):
    """> 8192 candidates (prefill): device radix-sort vote vs the oracle."""
    rng = np.random.default_rng(7)
    for n, span, kp in ((8193, 3000, 127), (20000, 500, 64), (131072, 100000, 127),
                        (131072, 200, 512)):
        idx = rng.integers(0, span, n).astype(np.uint64)
        score = (rng.integers(0, 4000, n) / 2000.0 - 1.0).astype(np.float32)
        want = ob.vote(idx, score, kp)
        w = torch.zeros(kp, dtype=torch.int32, device="cuda")
        nw = ctx.vote(dev(idx.astype(np.int32)), dev(score), kp, w)
        assert np.array_equal(w.cpu().numpy()[:nw].astype(np.uint64), want), n


def test_vote_small_path_large_k_prime(ctx):
    """<= 8192 candidates (the shared-memory select) with k' up to the candidate count."""
    rng = np.random.default_rng(17)
    for n, span, kp in ((8192, 9000, 8192), (5000, 300, 4000), (3000, 3000, 2999)):
        idx = rng.integers(0, span, n).astype(np.uint64)
        score = (rng.integers(0, 5000, n) / 2500.0 - 1.0).astype(np.float32)
        want = ob.vote(idx, score, kp)
        w = torch.zeros(kp, dtype=torch.int32, device="cuda")
        nw = ctx.vote(dev(idx.astype(np.int32)), dev(score), kp, w)
        assert np.array_equal(w.cpu().numpy()[:nw].astype(np.uint64), want), (n, kp)


def test_tally_large_unbounded_indices(ctx):
    """reattn_tally over > 8192 candidates with indices spread over the whole u32 range (the
    standalone path: hand-written radix sorts): every distinct index once, ranked by (votes
    desc, max score desc, index asc) as the oracle's vote with k' = n, with its vote count and
    max score (selection.hpp:252-286)."""
    rng = np.random.default_rng(91)
    for n, span in ((9000, 2500), (40000, 40000)):
        base = rng.integers(0, 1 << 31, span).astype(np.uint64)
        idx = base[rng.integers(0, span, n)]
        score = (rng.integers(0, 3000, n) / 1500.0 - 1.0).astype(np.float32)
        want = ob.vote(idx, score, n)
        io = torch.zeros(n, dtype=torch.int32, device="cuda")
        vo = torch.zeros(n, dtype=torch.int32, device="cuda")
        so = torch.zeros(n, dtype=torch.float32, device="cuda")
        nu = ctx.tally(dev(idx.astype(np.uint32).view(np.int32)), dev(score), io, vo, so)
        got = io.cpu().numpy()[:nu].view(np.uint32).astype(np.uint64)
        assert np.array_equal(got, want), n
        uniq, counts = np.unique(idx, return_counts=True)
        cnt = dict(zip(uniq.tolist(), counts.tolist()))
        mx = {}
        for i, sc in zip(idx.tolist(), score.tolist()):
            mx[i] = max(mx.get(i, -np.inf), sc)
        v = vo.cpu().numpy()[:nu]
        sv = so.cpu().numpy()[:nu]
        for j in range(0, nu, max(1, nu // 500)):
            assert v[j] == cnt[int(got[j])] and sv[j] == np.float32(mx[int(got[j])]), (n, j)


def test_attend_step_prefill_chunk_large_vote(ctx):
    """test_engine.cpp-style k = k' = 100 prefill chunk: 2 x 100 x 100 = 20,000 candidates."""
    cfg = N.SelectionConfig(k=100, k_prime=100, span_m=16, l_global=16, l_local=256, l_chunk=128)
    res, out, st, spans = step_vs_oracle(ctx, 2, 4, 16, 3000, cfg, N.F32, 600, 2048,
                                         base=10000.0, n_q=100)
    assert res.stats.scope_len == st.scope_len
    assert np.array_equal(res.spans[0], spans[0])
    assert np.abs(res.out.cpu().numpy() - out).max() <= ATTN_TOL


@pytest.mark.parametrize("kp,total", [(600, 20000), (127, 150000), (1000, 60000)])
def test_attend_step_prefill_bounded_vote(ctx, kp, total):
    """The plans' large vote (histogram tally, per-CTA bitonic rank of 2048 middle rows, 4-ary
    merge tree): k' up to 1024 kept rows, several tree levels, against the oracle -- through
    the synchronous step (fresh workspace) and a plan replayed twice (its tallies must come
    back clean)."""
    cfg = N.SelectionConfig(k=8, k_prime=kp, span_m=2, l_global=16, l_local=256, l_chunk=512)
    n_kv, nh, d, n_q, window, base = 4, 8, 32, 300, 4096, 10000.0
    res, out, st, spans = step_vs_oracle(ctx, n_kv, nh, d, total, cfg, N.BF16, 1700 + kp, window,
                                         base=base, n_q=n_q)
    assert res.stats.scope_len == st.scope_len
    assert np.array_equal(res.spans[0], spans[0]) and np.array_equal(res.spans[1], spans[1])
    assert np.abs(res.out.cpu().numpy() - out).max() <= ATTN_TOL
    cache, _, _ = make_cache(ctx, n_kv, d, total, cfg, N.BF16, 1700 + kp)
    rope = N.Rope(ctx, d, base, window)
    plan = N.Plan(ctx, cache, rope, n_q, nh, cfg)
    plan.q.copy_(dev(synth.uniform(1700 + kp + 7, n_q * nh * d).reshape(n_q, nh * d)))
    for _ in range(2):
        plan.launch()
        r = plan.result(kp)
        assert r.stats.scope_len == st.scope_len
        assert np.array_equal(r.spans[0], spans[0]) and np.array_equal(r.spans[1], spans[1])
        assert np.abs(r.out.cpu().numpy() - out).max() <= ATTN_TOL


@pytest.mark.parametrize("total", [9000, 40000, 131072])
def test_attend_step_decode_local_fork(ctx, total, monkeypatch):
    """Decode with the local-window attention forked beside the scan (REATTN_FORK=1): the
    local segment is attended at shifted RoPE positions on its own SMs and merged with the
    post-selection part.  Same parity bar as the unforked step."""
    monkeypatch.setenv("REATTN_FORK", "1")
    cfg = N.SelectionConfig()
    res, out, st, spans = step_vs_oracle(ctx, 8, 32, 128, total, cfg, N.BF16, 71 + total, 8192)
    assert res.stats.scope_len == st.scope_len
    assert np.array_equal(res.spans[0], spans[0]) and np.array_equal(res.spans[1], spans[1])
    assert np.abs(res.out.cpu().numpy() - out).max() <= ATTN_TOL
    assert abs(res.stats.entropy_max - st.entropy_max) <= DEC_ENT_TOL
    monkeypatch.setenv("REATTN_FORK", "0")
    plain = step_vs_oracle(ctx, 8, 32, 128, total, cfg, N.BF16, 71 + total, 8192)[0]
    assert (plain.out - res.out).abs().max().item() <= ATTN_TOL


def test_attend_step_decode_local_after_scan(ctx, monkeypatch):
    """REATTN_FORK=2: the local window launched after the scan on every SM (a programmatic
    dependent that completes only after the scan), then the head launch; plan and synchronous
    step both match the oracle."""
    monkeypatch.setenv("REATTN_FORK", "2")
    cfg = N.SelectionConfig()
    res, out, st, spans = step_vs_oracle(ctx, 8, 32, 128, 131072, cfg, N.BF16, 97, 8192)
    assert res.stats.scope_len == st.scope_len
    assert np.array_equal(res.spans[0], spans[0]) and np.array_equal(res.spans[1], spans[1])
    assert np.abs(res.out.cpu().numpy() - out).max() <= ATTN_TOL
    cache, _, _ = make_cache(ctx, 8, 128, 131072, cfg, N.BF16, 98)
    rope = N.Rope(ctx, 128, 500000.0, 8192)
    plan = N.Plan(ctx, cache, rope, 1, 32, cfg)
    for s in range(3):
        q = dev(synth.uniform(700 + s, 32 * 128).reshape(1, -1))
        ref = N.attend_step(ctx, cache, rope, q, 32, cfg)
        plan.q.copy_(q)
        torch.cuda.synchronize()
        plan.launch()
        plan.stats()
        assert torch.equal(plan.out, ref.out), s


@pytest.mark.parametrize("hpc", [2, 4, 8])
def test_attend_step_decode_local_fork_heads_per_cta(ctx, hpc, monkeypatch):
    """The planner's default at long contexts gives each local-window CTA several kv heads in
    turn (1M: two); forced here at 131072 tokens for 2, 4 and 8 heads per CTA."""
    monkeypatch.setenv("REATTN_FORK", "1")
    monkeypatch.setenv("REATTN_FORK_HPC", str(hpc))
    cfg = N.SelectionConfig()
    res, out, st, spans = step_vs_oracle(ctx, 8, 32, 128, 131072, cfg, N.BF16, 90 + hpc, 8192)
    assert res.stats.scope_len == st.scope_len
    assert np.array_equal(res.spans[0], spans[0]) and np.array_equal(res.spans[1], spans[1])
    assert np.abs(res.out.cpu().numpy() - out).max() <= ATTN_TOL
    assert abs(res.stats.entropy_max - st.entropy_max) <= DEC_ENT_TOL
