"""The device Engine (capi_engine.cpp) against the reference's own Engine, forward_full and
WindowReference, compiled in place (oracle/_ref).  Mirrors test_engine.cpp and the
acceptance criteria C02/C03 (acceptance_test.cpp:100-190): same model configs, seeds and
token streams (the reference build's own random_tokens).

Parity bars:
* weights: init_random and the RATW file are bit-identical to the reference's;
* logits: max-abs <= 1e-4 against the quadratic forward_full on full-coverage runs (the
  reference's own bar, test_engine.cpp:104 / acceptance C02); the GEMMs are fp32 on both
  sides, with different summation orders;
* greedy tokens: equal to the reference's greedy decoder;
* device-internal identities are bitwise (single-token prefill == decode on an empty
  cache; window mode == reattention with k' = 0; two identical runs)."""
import math
import os

import numpy as np
import pytest

import oracle_bind as ob

torch = pytest.importorskip("torch")
from paper_2407_15176_b200 import native as N  # noqa: E402

pytestmark = pytest.mark.gpu

if ob.ref() is None:  # the compiled reference is the checker here
    pytest.skip("oracle/_ref not built", allow_module_level=True)


def toy_config(**kw):  # test_engine.cpp:23-33
    c = dict(n_layer=2, n_head=4, n_kv_head=2, d_model=64, d_head=16, d_ff=128, vocab_size=128,
             pretrain_window=2048)
    c.update(kw)
    return N.ModelConfig(**c)


def toy_selection(**kw):  # test_engine.cpp:37-47
    s = dict(k=4, k_prime=64, span_m=16, tile_size=512, l_global=16, l_local=256, l_chunk=128)
    s.update(kw)
    return N.SelectionConfig(**s)


def pair(ctx, cfg, seed):
    return N.Weights.init_random(ctx, cfg, seed), ob.RefModel(cfg, seed)


SHAPE_KINDS = [(N.W_EMBEDDING, False), (N.W_WQ, True), (N.W_WK, True), (N.W_WV, True),
               (N.W_WO, True), (N.W_GATE, True), (N.W_UP, True), (N.W_DOWN, True),
               (N.W_NORM_ATTN, True), (N.W_NORM_FFN, True), (N.W_NORM_FINAL, False),
               (N.W_LM_HEAD, False)]


def assert_same_weights(w, ref_model, cfg):
    for kind, per_layer in SHAPE_KINDS:
        for layer in range(cfg.n_layer if per_layer else 1):
            mine = w.tensor(kind, layer)
            theirs = ref_model.tensor(kind, layer, mine.shape)
            assert np.array_equal(mine.view(np.uint32), theirs.view(np.uint32)), (kind, layer)


def test_init_random_is_the_reference_stream(ctx):
    cfg = N.ModelConfig()  # the reference's default toy model
    w, r = pair(ctx, cfg, 7)
    assert_same_weights(w, r, cfg)


def test_weights_file_round_trip_both_ways(ctx, tmp_path):
    cfg = toy_config(n_layer=3)
    w, r = pair(ctx, cfg, 11)
    mine, theirs = str(tmp_path / "mine.ratw"), str(tmp_path / "theirs.ratw")
    w.save(mine)
    r.save(theirs)
    assert open(mine, "rb").read() == open(theirs, "rb").read()  # byte-identical files
    assert_same_weights(N.Weights.load(ctx, theirs), ob.RefModel(path=mine), cfg)


def _ref_load_error(path):
    with pytest.raises(RuntimeError) as e:
        ob.RefModel(path=path)
    return str(e.value)


def test_weights_file_errors_match_reference(ctx, tmp_path):
    cfg = toy_config()
    w = N.Weights.init_random(ctx, cfg, 3)
    good = str(tmp_path / "good.ratw")
    w.save(good)
    data = open(good, "rb").read()
    cases = {
        "magic": b"XXXX" + data[4:],
        "version": data[:4] + (9).to_bytes(4, "little") + data[8:],
        "trunc_cfg": data[:20],
        "trunc_tensor": data[: len(data) // 2],
        "trailing": data + b"\0",
        "mode": data[:52] + (7).to_bytes(4, "little") + data[56:],
        "shape": data[:56] + (5).to_bytes(8, "little") + data[64:],
        "config": data[:8] + (0).to_bytes(4, "little") + data[12:],
    }
    for name, blob in cases.items():
        p = str(tmp_path / f"{name}.ratw")
        open(p, "wb").write(blob)
        want = _ref_load_error(p)
        with pytest.raises(N.ReattnError) as got:
            N.Weights.load(ctx, p)
        assert str(got.value) == want, name
    with pytest.raises(N.ReattnError, match="cannot open weights file"):
        N.Weights.load(ctx, str(tmp_path / "missing.ratw"))


def test_rejects_full_mode_and_over_budget_selection(ctx):  # test_engine.cpp:57-66
    w = N.Weights.init_random(ctx, toy_config(), 20)
    with pytest.raises(N.InvalidArgument, match="full attention is the reference path"):
        N.Engine(ctx, w, toy_selection(), N.MODE_FULL)
    with pytest.raises(N.InvalidArgument, match="exceeds pretrain window 2048"):
        N.Engine(ctx, w, toy_selection(k_prime=1000))
    with pytest.raises(N.InvalidArgument, match="l_chunk must not exceed l_local"):
        N.Engine(ctx, w, toy_selection(l_chunk=257))
    with pytest.raises(N.InvalidArgument, match="d_model != n_head"):
        N.Weights.init_random(ctx, toy_config(d_model=60), 1)


def test_single_token_prefill_equals_decode_on_empty_cache(ctx):  # test_engine.cpp:68-78
    w = N.Weights.init_random(ctx, toy_config(), 21)
    a = N.Engine(ctx, w, toy_selection())
    b = N.Engine(ctx, w, toy_selection())
    la = a.logits(a.prefill([42]))
    b.decode_step(42)
    assert np.array_equal(la[0], b.last_logits())


def test_full_coverage_prefill_matches_quadratic_reference(ctx):  # test_engine.cpp:80-110
    cfg = toy_config()
    w, r = pair(ctx, cfg, 22)
    tokens = ob.random_tokens(372, 128, 220)
    eng = N.Engine(ctx, w, toy_selection(k=100, k_prime=100))
    hidden = eng.prefill(tokens)
    assert eng.stats().coverage_total
    got = eng.logits(hidden)
    full = r.forward_full(tokens, cfg.vocab_size)
    assert got.shape[0] == 100
    md = np.abs(got.astype(np.float64) - full[-100:].astype(np.float64)).max()
    assert md <= 1e-4, md
    assert int(got[-1].argmax()) == int(full[-1].argmax())


def test_c02_full_attention_equivalence_10_seeds(ctx):  # acceptance_test.cpp:102-150
    cfg = N.ModelConfig(pretrain_window=16544)
    sel = N.SelectionConfig(k=512, k_prime=512, span_m=32, l_global=32, l_local=128, l_chunk=64)
    assert sel.budget() == 16544
    ties = 0
    for seed in range(10):
        w, r = pair(ctx, cfg, seed)
        tokens = ob.random_tokens(512, cfg.vocab_size, 900 + seed)
        eng = N.Engine(ctx, w, sel)
        got = eng.logits(eng.prefill(tokens))
        st = eng.stats()
        assert st.coverage_total and st.ood_positions == 0
        oracle = r.forward_full(tokens, cfg.vocab_size)
        tail = got.shape[0]
        md = np.abs(got.astype(np.float64) - oracle[512 - tail:].astype(np.float64)).max()
        assert md <= 1e-4, (seed, md)
        if int(got[-1].argmax()) != int(oracle[-1].argmax()):
            top = np.sort(oracle[-1])[::-1]
            assert top[0] - top[1] <= 2e-4, seed
            ties += 1
    assert ties <= 1


def test_selection_off_matches_window_reference(ctx):  # test_engine.cpp:112-131, C03
    cfg = toy_config()
    w, r = pair(ctx, cfg, 23)
    tokens = ob.random_tokens(900, 128, 230)
    sel = toy_selection(k_prime=0)
    eng = N.Engine(ctx, w, sel)
    ref = ob.RefEngine(r, sel, kind=1, d_model=cfg.d_model, vocab=cfg.vocab_size)
    gh, rh = eng.prefill(tokens), ref.prefill(tokens)
    assert np.abs(gh - rh).max() <= 1e-4
    for s in range(4):
        ta = eng.decode_step(s)
        tb, lb = ref.decode_step(s)
        assert ta == tb
        assert np.abs(eng.last_logits() - lb).max() <= 1e-4


def test_window_mode_ignores_selection_parameters(ctx):  # test_engine.cpp:133-145 (bitwise)
    w = N.Weights.init_random(ctx, toy_config(), 24)
    tokens = ob.random_tokens(700, 128, 240)
    a = N.Engine(ctx, w, toy_selection(), N.MODE_WINDOW).prefill(tokens)
    b = N.Engine(ctx, w, toy_selection(k_prime=0), N.MODE_REATTENTION).prefill(tokens)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_greedy_decode_agrees_with_reference_decoder(ctx):  # test_engine.cpp:147-171
    cfg = toy_config()
    w, r = pair(ctx, cfg, 25)
    prompt = ob.random_tokens(300, 128, 250)
    want = ob.greedy_decode_full(r, prompt, 6)
    eng = N.Engine(ctx, w, toy_selection(k=64, k_prime=64))
    eng.prefill(prompt[:-1])
    got, feed = [], int(prompt[-1])
    for _ in range(6):
        feed = eng.decode_step(feed)
        got.append(feed)
    assert eng.stats().coverage_total
    assert got == want


def test_selection_active_matches_reference_engine(ctx):
    """ReAttention with a real selection (the middle outgrows k' spans): the device engine
    and the reference Engine choose the same spans in every layer and agree on the hidden
    states and the greedy continuation."""
    cfg = toy_config()
    w, r = pair(ctx, cfg, 31)
    tokens = ob.random_tokens(1400, 128, 310)
    sel = toy_selection(k_prime=8)
    eng = N.Engine(ctx, w, sel)
    ref = ob.RefEngine(r, sel, d_model=cfg.d_model, vocab=cfg.vocab_size)
    gh, rh = eng.prefill(tokens), ref.prefill(tokens)
    assert not eng.stats().coverage_total
    assert np.abs(gh - rh).max() <= 1e-4
    feed = int(tokens[-1])
    for _ in range(4):
        a = eng.decode_step(feed)
        b, _ = ref.decode_step(feed)
        assert a == b
        feed = a
    rs, gs = ref.stats(), eng.stats()
    assert gs.scope_len_max == rs["scope_len_max"]
    assert gs.max_position_used == rs["max_position_used"]
    assert gs.chunks_processed == rs["chunks_processed"]
    assert gs.decode_steps == rs["decode_steps"]
    assert abs(gs.entropy_max - rs["entropy_max"]) <= 1e-4


@pytest.mark.parametrize("cache_dtype", [N.F32, N.BF16])
def test_decode_projection_shapes_match_reference_engine(ctx, cache_dtype):
    """Decode tokens at widths that are not multiples of the GEMV's 128-column tiles or
    64-row units (d_model 260 = 5 heads x 52, d_ff 1000, vocab 1032, one kv head): the
    fused q/k/v GEMV with the K/V rows written into the cache from its epilogue, the
    gate/up pair with silu in the epilogue, the stream-K fix-up across tile boundaries --
    logits within 1e-4 of the reference Engine (fp32 cache) and the same greedy tokens."""
    cfg = toy_config(d_model=260, n_head=5, n_kv_head=1, d_head=52, d_ff=1000, vocab_size=1032)
    w, r = pair(ctx, cfg, 41)
    tokens = ob.random_tokens(600, cfg.vocab_size, 410)
    sel = toy_selection(k_prime=8)
    eng = N.Engine(ctx, w, sel, cache_dtype=cache_dtype)
    ref = ob.RefEngine(r, sel, d_model=cfg.d_model, vocab=cfg.vocab_size)
    gh, rh = eng.prefill(tokens), ref.prefill(tokens)
    tol = 1e-4 if cache_dtype == N.F32 else 2e-2
    assert np.abs(gh - rh).max() <= tol
    feed = int(tokens[-1])
    for _ in range(5):
        a = eng.decode_step(feed)
        b, lb = ref.decode_step(feed)
        assert np.abs(eng.last_logits() - lb).max() <= tol
        if cache_dtype == N.F32:
            assert a == b
        feed = b


def test_long_context_never_leaves_pretrain_range(ctx):  # test_engine.cpp:173-195
    cfg = toy_config()
    w = N.Weights.init_random(ctx, cfg, 26)
    sel = toy_selection()
    tokens = ob.random_tokens(5000, 128, 260)
    eng = N.Engine(ctx, w, sel)
    hidden = eng.prefill(tokens)
    assert np.isfinite(hidden).all()
    st = eng.stats()
    assert st.ood_positions == 0
    assert st.max_position_used < cfg.pretrain_window
    assert st.scope_len_max <= min(cfg.pretrain_window, sel.budget())
    assert st.entropy_max <= math.log(cfg.pretrain_window) + 1e-9
    assert not st.coverage_total
    tok = int(tokens[-1])
    for _ in range(8):
        tok = eng.decode_step(tok)
        assert tok < cfg.vocab_size
    assert eng.stats().ood_positions == 0


def test_deterministic_across_identical_runs(ctx):  # test_engine.cpp:197-217
    w = N.Weights.init_random(ctx, toy_config(), 27)
    tokens = ob.random_tokens(1500, 128, 270)
    runs = []
    for _ in range(2):
        eng = N.Engine(ctx, w, toy_selection())
        eng.prefill(tokens)
        toks, tok = [], int(tokens[-1])
        for _ in range(16):
            tok = eng.decode_step(tok)
            toks.append(tok)
        runs.append((toks, eng.last_logits().copy()))
    assert runs[0][0] == runs[1][0]
    assert np.array_equal(runs[0][1], runs[1][1])


def test_stats_count_chunks_and_steps(ctx):  # test_engine.cpp:219-231
    cfg = toy_config()
    w = N.Weights.init_random(ctx, cfg, 28)
    eng = N.Engine(ctx, w, toy_selection())
    eng.prefill(ob.random_tokens(700, 128, 280))
    assert eng.stats().chunks_processed == 1 + 4
    eng.decode_step(1)
    eng.decode_step(2)
    assert eng.stats().decode_steps == 2
    assert len(eng.decode_latencies()) == 2
    assert all(isinstance(eng.last_spans(l), list) for l in range(cfg.n_layer))


def test_bf16_cache_engine_tracks_fp32(ctx):
    """bf16 cache storage (the GEMM output rounded into the cache) stays close to fp32."""
    cfg = toy_config()
    w = N.Weights.init_random(ctx, cfg, 33)
    tokens = ob.random_tokens(800, 128, 330)
    a = N.Engine(ctx, w, toy_selection(k=100, k_prime=100), cache_dtype=N.F32)
    b = N.Engine(ctx, w, toy_selection(k=100, k_prime=100), cache_dtype=N.BF16)
    la = a.logits(a.prefill(tokens))
    lb = b.logits(b.prefill(tokens))
    assert np.abs(la - lb).max() <= 1e-2


def test_token_outside_vocabulary(ctx):
    w = N.Weights.init_random(ctx, toy_config(), 5)
    eng = N.Engine(ctx, w, toy_selection())
    with pytest.raises(N.OutOfRange, match="token id outside vocabulary"):
        eng.prefill([1, 2, 128])
    with pytest.raises(N.InvalidArgument, match="empty input"):
        eng.prefill([])
