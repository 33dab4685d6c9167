"""K2 (prefill score scan on tcgen05) vs the oracle: bit-identical indices and scores.

K2 runs the score GEMM once with the bf16 rounding of the fp32 group-mean query, bounds the
error of those scores (2^-8 * ||mq||_1 * max|k|), and recomputes the reference's exact fp32
dot_f32 (dense_matrix.hpp:41-56) for every key that could still enter a row's top-k -- so
the selected indices AND scores must equal fused_topk_scores (selection.hpp:168-248) bit for
bit, in both lane arithmetics (unfused mul+add, or FMA: SURVEY §8(c))."""
import numpy as np
import pytest

import oracle_bind as ob
import synth

torch = pytest.importorskip("torch")
from paper_2407_15176_b200 import native as N  # noqa: E402

pytestmark = pytest.mark.gpu


def run(ctx, q, n_heads, keys_bf16, k):
    n_kv, count, d = keys_bf16.shape
    n_q = q.shape[0]
    kt = torch.from_numpy(keys_bf16).cuda().to(torch.bfloat16)
    qt = torch.from_numpy(q).cuda()
    idx = torch.zeros(n_kv * n_q * k, dtype=torch.int32, device="cuda")
    sc = torch.zeros(n_kv * n_q * k, dtype=torch.float32, device="cuda")
    ctx.set_prefill(N.PREFILL_TENSOR_SCAN)
    try:
        n_out, _ = ctx.fused_topk(qt, n_heads, kt, n_kv, count, 0, count, d, k, idx, sc, N.BF16)
    finally:
        ctx.set_prefill(N.PREFILL_DEFAULT)
    i = idx.cpu().numpy().view(np.uint32).reshape(n_kv, n_q, k)[:, :, :n_out]
    s = sc.cpu().numpy().reshape(n_kv, n_q, k)[:, :, :n_out]
    return i, s


@pytest.mark.parametrize("n_q,count,k", [(2, 1, 1), (64, 255, 4), (128, 256, 4), (200, 1000, 8),
                                         (512, 28640, 4), (300, 5000, 2),
                                         # key-range splits > 1 with k below the list length
                                         (256, 40000, 3), (128, 40000, 5)])
def test_prefill_tc_bit_exact(ctx, n_q, count, k):
    n_kv, nh, d = 8, 32, 128
    keys = synth.uniform(900 + count, n_kv * count * d, bf16=True).reshape(n_kv, count, d)
    q = synth.uniform(901 + n_q, n_q * nh * d).reshape(n_q, nh * d)
    gi, gs = run(ctx, q, nh, keys, k)
    oi, osc = ob.topk(q, nh, [np.ascontiguousarray(keys[h]) for h in range(n_kv)], k)
    assert gi.shape == oi.shape
    assert np.array_equal(gi.astype(np.uint64), oi), "indices differ"
    assert np.array_equal(gs.view(np.uint32), osc.view(np.uint32)), "scores differ"


@pytest.mark.parametrize("lanes", [N.LANES_UNFUSED, N.LANES_FMA])
def test_prefill_tc_lane_modes_and_ties(ctx, lanes):
    """Both lane arithmetics, with planted exact ties (duplicate key rows: equal scores, the
    lower index must win) and a shifted key distribution."""
    n_kv, nh, d, count, n_q, k = 8, 32, 128, 9000, 160, 4
    keys = synth.uniform(77, n_kv * count * d, bf16=True).reshape(n_kv, count, d) + 0.25
    keys = synth.bf16_round(keys)
    keys[:, 5000:5100] = keys[:, 100:200]  # exact duplicates -> ties by index
    q = synth.uniform(78, n_q * nh * d).reshape(n_q, nh * d)
    ctx.set_lanes(lanes)
    try:
        gi, gs = run(ctx, q, nh, keys, k)
    finally:
        ctx.set_lanes(N.LANES_UNFUSED)
    with ob.lane_mode(lanes):
        oi, osc = ob.topk(q, nh, [np.ascontiguousarray(keys[h]) for h in range(n_kv)], k)
    assert np.array_equal(gi.astype(np.uint64), oi)
    assert np.array_equal(gs.view(np.uint32), osc.view(np.uint32))


def test_prefill_tc_window_overflow_rescan(ctx):
    """64 copies of one scaled key row: for every query that ranks it highly the 2-delta window
    holds far more than the L = KT + 4 list slots, so the part's dropped S_hi reaches the window
    and the merge re-scans that key range exactly -- the result must still be the reference's
    (equal scores: the lowest indices).  Zero query rows (delta == 0, all scores 0) too."""
    n_kv, nh, d, count, n_q, k = 8, 32, 128, 20000, 96, 4
    keys = synth.uniform(91, n_kv * count * d, bf16=True).reshape(n_kv, count, d)
    keys[:, 7000:7064] = synth.bf16_round(keys[:, 123:124] * 3.0)
    q = synth.uniform(92, n_q * nh * d).reshape(n_q, nh * d)
    q[5] = 0.0
    q[40] = 0.0
    gi, gs = run(ctx, q, nh, keys, k)
    oi, osc = ob.topk(q, nh, [np.ascontiguousarray(keys[h]) for h in range(n_kv)], k)
    assert np.array_equal(gi.astype(np.uint64), oi)
    assert np.array_equal(gs.view(np.uint32), osc.view(np.uint32))
    # the planted copies really were selected somewhere (the rescan path ran)
    assert ((oi >= 7000) & (oi < 7064)).any()
