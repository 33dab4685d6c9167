"""CPU-only tests (no GPU): pin the oracle (oracle/reattn_oracle.c) against the golden
fixtures produced by the reference itself (tests/golden/, from oracle/_ref) and against the
live compiled reference when it is present; check the synthetic-input twins and the
reference's known-answer cases; check that the C-ABI library loads and exports every
symbol include/reattn_cuda.h declares (no compute calls without a GPU).
"""
import hashlib
import json
import os
import re
import subprocess

import numpy as np
import pytest

import oracle_bind as ob
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLD, "manifest.json")) as f:
        man = json.load(f)
    arrs = np.load(os.path.join(GOLD, "ref_golden.npz"))
    return man["cases"], arrs


def _keys(seed, n_kv, count, d, bf16=False):
    return synth.uniform(seed, n_kv * count * d, bf16=bf16).reshape(n_kv, count, d)


# ---- oracle vs golden fixtures (reference outputs) -------------------------------------
def test_golden_topk_bit_exact(golden):
    cases, A = golden
    for c in cases["topk"]:
        K = _keys(c["seed"], c["n_kv"], c["count"], c["d"])
        q = synth.uniform(c["seed"] + 50000, c["n_q"] * c["n_heads"] * c["d"]).reshape(c["n_q"], -1)
        with ob.lane_mode(c["lanes"]):
            idx, sc = ob.topk(q, c["n_heads"], [np.ascontiguousarray(K[h]) for h in range(c["n_kv"])],
                              c["k"])
        assert np.array_equal(idx.astype(np.uint32), A[c["name"] + "_idx"]), c
        assert np.array_equal(sc.view(np.uint32), A[c["name"] + "_score"].view(np.uint32)), c


def test_golden_vote_and_spans(golden):
    cases, A = golden
    for c in cases["vote"]:
        n = c["name"]
        w = ob.vote(A[n + "_in_idx"].astype(np.uint64), A[n + "_in_score"], c["k_prime"])
        assert np.array_equal(w.astype(np.uint32), A[n + "_out"]), c
    for c in cases["spans"]:
        n = c["name"]
        b, e = ob.expand_spans(A[n + "_in"].astype(np.uint64), c["span_m"], c["middle_len"], c["mode"])
        assert np.array_equal(b.astype(np.uint32), A[n + "_b"]), c
        assert np.array_equal(e.astype(np.uint32), A[n + "_e"]), c


def test_golden_attend(golden):
    cases, A = golden
    for c in cases["attend"]:
        s = c["seed"]
        q = synth.uniform(s, c["n_q"] * c["d"]).reshape(c["n_q"], c["d"])
        k = synth.uniform(s + 1, c["L"] * c["d"]).reshape(c["L"], c["d"])
        v = synth.uniform(s + 2, c["L"] * c["dv"]).reshape(c["L"], c["dv"])
        o, e = ob.attend(q, k, v, c["boundary"])
        assert np.abs(o - A[c["name"] + "_out"]).max() <= 1e-7, c
        assert np.abs(e - A[c["name"] + "_ent"]).max() <= 1e-12, c


def test_golden_rope_tables(golden):
    cases, _ = golden
    for c in cases["rope"]:
        cs, sn = ob.rope_table(c["d"], c["base"], c["max_position"])
        assert hashlib.sha256(cs.tobytes() + sn.tobytes()).hexdigest() == c["sha256"], c


def test_golden_attend_step(golden):
    cases, A = golden
    for c in cases["attend_step"]:
        K = _keys(c["seed"], c["n_kv"], c["total"], c["d"], c["bf16"])
        V = _keys(c["seed"] + 1, c["n_kv"], c["total"], c["d"], c["bf16"])
        q = synth.uniform(c["seed"] + 2, c["n_q"] * c["nh"] * c["d"]).reshape(c["n_q"], -1)
        cfg = ob.SelectionConfig(**c["cfg"])
        with ob.lane_mode(c["lanes"]):
            o, st, (sb, se) = ob.attend_step(q, c["nh"], K, V, c["total"], cfg, c["base"],
                                             c["window"], 2)
        assert st.scope_len == c["scope_len"], c["name"]
        assert np.array_equal(sb.astype(np.uint32), A[c["name"] + "_sb"]), c["name"]
        assert np.array_equal(se.astype(np.uint32), A[c["name"] + "_se"]), c["name"]
        # RoPE float ops may be contracted differently by the reference build: ulp-level
        assert np.abs(o - A[c["name"] + "_out"]).max() <= 1e-7, c["name"]
        assert abs(st.entropy_max - c["entropy_max"]) <= 1e-8, c["name"]


def test_golden_attend_step_ex_bf16_words(golden):
    """The storage-generic, multi-threaded oracle (used by the full-size GPU parity tests on
    bf16 caches held as words) reproduces the golden attend_step cases bit for bit in the
    selection and within the same tolerance in the outputs."""
    cases, A = golden
    for c in cases["attend_step"]:
        if not c["bf16"]:
            continue
        K = _keys(c["seed"], c["n_kv"], c["total"], c["d"], True)
        V = _keys(c["seed"] + 1, c["n_kv"], c["total"], c["d"], True)
        kw = np.ascontiguousarray(K).view(np.uint32) >> 16
        vw = np.ascontiguousarray(V).view(np.uint32) >> 16
        q = synth.uniform(c["seed"] + 2, c["n_q"] * c["nh"] * c["d"]).reshape(c["n_q"], -1)
        cfg = ob.SelectionConfig(**c["cfg"])
        with ob.lane_mode(c["lanes"]):
            o, ent, st, (sb, se), _ = ob.attend_step_ex(q, c["nh"], kw.astype(np.uint16),
                                                        vw.astype(np.uint16), c["total"], cfg,
                                                        c["base"], c["window"], 2, threads=5)
        assert st.scope_len == c["scope_len"], c["name"]
        assert np.array_equal(sb.astype(np.uint32), A[c["name"] + "_sb"]), c["name"]
        assert np.array_equal(se.astype(np.uint32), A[c["name"] + "_se"]), c["name"]
        assert np.abs(o - A[c["name"] + "_out"]).max() <= 1e-7, c["name"]
        assert abs(st.entropy_max - c["entropy_max"]) <= 1e-8, c["name"]
        assert abs(ent.max() - c["entropy_max"]) <= 1e-8, c["name"]


def test_topk_ex_matches_sequential_oracle():
    """Range-split, multi-threaded top-k == the sequential TopkBuffer restatement, including
    planted exact ties across range boundaries (ties keep the lower index)."""
    rng = np.random.default_rng(5)
    for it, (count, n_kv, nh, d, k, nq) in enumerate([(5000, 2, 8, 128, 4, 1), (9000, 1, 3, 64, 8, 3),
                                                      (2049, 3, 3, 16, 1, 2), (20000, 2, 4, 128, 5, 1)]):
        K = rng.uniform(-1, 1, (n_kv, count, d)).astype(np.float32)
        K[:, 100] = K[:, 4000 % count] = K[:, count - 1] = K[:, 7]  # exact score ties
        q = rng.uniform(-1, 1, (nq, nh * d)).astype(np.float32)
        want = ob.topk(q, nh, [np.ascontiguousarray(K[h]) for h in range(n_kv)], k)
        for threads in (1, 4, 13):
            got = ob.topk_ex(q, nh, K, 0, count, k, threads=threads)
            assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1]), (it, threads)
        # bf16 words
        Kb = ob.round_bf16(K)
        want = ob.topk(q, nh, [np.ascontiguousarray(Kb[h]) for h in range(n_kv)], k)
        got = ob.topk_ex(q, nh, (Kb.view(np.uint32) >> 16).astype(np.uint16), 0, count, k, threads=6)
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1]), it


# ---- oracle vs the live compiled reference (this container only) ------------------------
needs_ref = pytest.mark.skipif(ob.ref() is None, reason="oracle/_ref not built here")


@needs_ref
def test_live_reference_fuzz_topk():
    rng = np.random.default_rng(37)
    r = ob.ref()
    for it in range(150):
        count = int(rng.integers(0, 4500))
        n_kv = 1 + it % 2
        nh = n_kv * (1 + (3 if it % 4 == 0 else 1))
        d = [16, 32, 8, 128, 64][it % 5]
        keys = [rng.uniform(-1, 1, (count, d)).astype(np.float32) for _ in range(n_kv)]
        q = rng.uniform(-1, 1, (int(rng.integers(1, 6)), nh * d)).astype(np.float32)
        k = 1 + it % 8
        lanes = ob.ref_lane_mode(d)
        if lanes is None:
            continue
        with ob.lane_mode(lanes):
            a = ob.topk(q, nh, keys, k)
        b = ob.topk(q, nh, keys, k, lib=r, tile=1 + (it * 97) % 3000)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), it


@needs_ref
def test_live_reference_attend_step():
    r = ob.ref()
    for total, seed in ((6000, 1), (12000, 2)):
        K = _keys(seed, 8, total, 128, True)
        V = _keys(seed + 1, 8, total, 128, True)
        q = synth.uniform(seed + 2, 32 * 128).reshape(1, -1)
        cfg = ob.SelectionConfig()
        a = ob.attend_step(q, 32, K, V, total, cfg, 500000.0, 8192)
        b = ob.attend_step(q, 32, K, V, total, cfg, 500000.0, 8192, lib=r)
        assert a[1].scope_len == b[1].scope_len
        assert np.array_equal(a[2][0], b[2][0])
        assert np.abs(a[0] - b[0]).max() <= 1e-7


# ---- known answers of the reference's own tests, through the oracle ---------------------
def test_known_answers():
    # test_selection.cpp:168-191 ties keep the lower index
    data = np.zeros((64, 8), np.float32)
    for i in (0, 7, 15, 16, 17, 31, 32, 49, 62, 63):
        data[i] = 0.5
    idx, _ = ob.topk(np.ones((1, 8), np.float32), 1, [data], 4)
    assert list(idx[0, 0]) == [0, 7, 15, 16]
    # :272-292 vote order
    assert list(ob.vote(np.array([9, 2, 7], np.uint64), np.array([5, 3, 1], np.float32), 2)) == [9, 2]
    assert list(ob.vote(np.array([7, 3, 7, 5], np.uint64),
                        np.array([0.1, 9.0, 0.2, 0.05], np.float32), 3)) == [7, 3, 5]
    assert len(ob.vote(np.array([1], np.uint64), np.array([1.0], np.float32), 0)) == 0
    # :325-337 spans
    b, e = ob.expand_spans([5, 20], 32, 100)
    assert (list(b), list(e)) == ([0], [32])
    b, e = ob.expand_spans([98], 32, 100)
    assert (list(b), list(e)) == ([96], [100])
    with pytest.raises(IndexError):
        ob.expand_spans([100], 32, 100)
    # test_scope.cpp:117-132 / acceptance C01: 32 + 127*32 + 4096 = 8192
    wn = np.arange(127, dtype=np.uint64) * 32
    b, e = ob.expand_spans(wn, 32, 9000 - 32 - 4096)
    n = int((e - b).sum())
    assert 32 + n + 4096 == 8192
    # test_numerics.cpp:257-266 single key returns its value row, entropy 0
    o, h = ob.attend(np.ones((3, 8), np.float32), np.ones((1, 8), np.float32),
                     np.arange(8, dtype=np.float32)[None])
    assert np.array_equal(o, np.tile(np.arange(8, dtype=np.float32), (3, 1))) and h.max() == 0.0


def test_synth_twins_agree():
    for seed, n, off in ((1, 1000, 0), (77, 100003, 5), (2**40 + 3, 4097, 123456789)):
        assert np.array_equal(synth.uniform(seed, n, off), synth.uniform_np(seed, n, off))
        assert np.array_equal(synth.uniform(seed, n, off, bf16=True),
                              synth.bf16_round(synth.uniform_np(seed, n, off)))


def test_group_mean_multiplies_by_reciprocal():
    """selection.hpp:143-151: x float(1/group), not /group (differs at group 3)."""
    q = synth.uniform(5, 3 * 128).reshape(1, 3 * 128)
    mq = np.zeros((1, 128), np.float32)
    ob.oracle().oracle_group_mean(q, 1, 3, 1, 128, mq)
    acc = (q[0, :128] + q[0, 128:256]) + q[0, 256:]
    assert np.array_equal(mq[0], acc * np.float32(1.0 / 3.0))


# ---- the C-ABI library: loads on a GPU-less host and exports the whole header -----------
def header_functions():
    text = open(os.path.join(ROOT, "include", "reattn_cuda.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(reattn_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2407_15176_b200 import native
    lib = native.load_library()
    names = header_functions()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", native.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (reattn_[a-z0-9_]+)", out))
    assert set(names) <= exported
    assert lib.reattn_version().decode().startswith("reattn-b200")


def test_binding_covers_header():
    from paper_2407_15176_b200 import native
    bound = {n for n, _, _ in native.SIGNATURES}
    assert set(header_functions()) == bound


def test_library_is_sm100a():
    from paper_2407_15176_b200 import native
    out = subprocess.run(["cuobjdump", "--list-elf", native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", native.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "UTMALDG" in sass  # TMA tensor loads in the K scan
    assert "FMUL2" in sass and "FADD2" in sass  # packed fp32 lanes (unfused emulation)


def test_selection_config_budget():
    from paper_2407_15176_b200 import native
    cfg = native.SelectionConfig()
    assert (cfg.k, cfg.k_prime, cfg.span_m, cfg.l_global, cfg.l_local) == (4, 127, 32, 32, 4096)
    assert cfg.budget() == 8192
