#!/usr/bin/env python
"""Generate tests/golden/ref_golden.npz from the REFERENCE itself (oracle/_ref: the
unmodified /root/reference headers compiled in place).  Run in the build container, where
/root/reference exists:  python tests/golden/make_golden.py

Inputs are regenerated deterministically from (seed, shape) with the splitmix64 generator
(tests/synth.py, identical to the library's reattn_synth_uniform), so only small inputs and
the reference's outputs are stored.  Each case records the lane arithmetic the compiled
reference used for its head dim; the oracle is checked against the
fixtures under that arithmetic.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle_bind as ob  # noqa: E402
import synth  # noqa: E402


def keys(seed, n_kv, count, d, bf16=False):
    return synth.uniform(seed, n_kv * count * d, bf16=bf16).reshape(n_kv, count, d)


def main():
    r = ob.ref()
    if r is None:
        sys.exit("oracle/_ref not built (make -C oracle ref)")
    out = {}
    manifest = {"generator": "oracle/_ref (reference headers compiled in place)",
                "ref_library": os.path.basename(ob._ref_path()), "cases": {}}

    # ---- fused_topk_scores: test_selection.cpp:105-149 style sizes / tiles / k / d ----
    topk_cases = []
    cid = 0
    for count in (0, 1, 3, 4, 5, 127, 1000, 2047, 2048, 2049, 5000):
        for k in (1, 4, 8):
            for d in (8, 16, 32, 128):
                n_kv = 1 + count % 2
                nh = n_kv * (1 + (count + k) % 3)
                n_q = 1 + (count + k + d) % 5
                seed = 100 + cid
                K = keys(seed, n_kv, count, d)
                q = synth.uniform(seed + 50000, n_q * nh * d).reshape(n_q, nh * d)
                idx, sc = ob.topk(q, nh, [np.ascontiguousarray(K[h]) for h in range(n_kv)], k,
                                  lib=r, tile=[16, 100, 2048][cid % 3])
                name = f"topk_{cid}"
                out[name + "_idx"] = idx.astype(np.uint32)
                out[name + "_score"] = sc
                topk_cases.append({"name": name, "seed": seed, "n_kv": n_kv, "n_heads": nh,
                                   "count": count, "d": d, "n_q": n_q, "k": k,
                                   "lanes": ob.ref_lane_mode(d)})
                cid += 1
    manifest["cases"]["topk"] = topk_cases

    # ---- vote (selection.hpp:278) and spans (:318) on random lists ----
    rng = np.random.default_rng(53)
    vote_cases = []
    for i in range(200):
        n = int(rng.integers(1, 120))
        idx = rng.integers(0, 50, n).astype(np.uint64)
        sc = (rng.integers(0, 1000, n) / 500.0 - 1.0).astype(np.float32)
        kp = int(rng.integers(0, 25))
        w = ob.vote(idx, sc, kp, lib=r)
        out[f"vote_{i}_in_idx"] = idx.astype(np.uint32)
        out[f"vote_{i}_in_score"] = sc
        out[f"vote_{i}_out"] = w.astype(np.uint32)
        vote_cases.append({"name": f"vote_{i}", "k_prime": kp})
    manifest["cases"]["vote"] = vote_cases
    span_cases = []
    for i in range(200):
        mode = i % 2
        m = 1 + i % 64 if mode == 0 else 2 + i % 63
        L = int(rng.integers(m, 100000))
        w = rng.integers(0, L, int(rng.integers(1, 128))).astype(np.uint64)
        b, e = ob.expand_spans(w, m, L, mode, lib=r)
        out[f"spans_{i}_in"] = w.astype(np.uint32)
        out[f"spans_{i}_b"] = b.astype(np.uint32)
        out[f"spans_{i}_e"] = e.astype(np.uint32)
        span_cases.append({"name": f"spans_{i}", "span_m": m, "middle_len": L, "mode": mode})
    manifest["cases"]["spans"] = span_cases

    # ---- attend (attend.hpp:25) ----
    att_cases = []
    for i in range(60):
        n_q, L, d = 1 + i % 8, 1 + (i * 37) % 512, max(4, (8 + (i * 11) % 60) & ~1)
        dv = d if i % 3 else max(2, d // 2)
        seed = 7000 + i
        q = synth.uniform(seed, n_q * d).reshape(n_q, d)
        k = synth.uniform(seed + 1, L * d).reshape(L, d)
        v = synth.uniform(seed + 2, L * dv).reshape(L, dv)
        bd = L - n_q if (i % 2 == 0 and L >= n_q) else None
        o, e = ob.attend(q, k, v, bd, lib=r)
        out[f"attend_{i}_out"] = o
        out[f"attend_{i}_ent"] = e
        att_cases.append({"name": f"attend_{i}", "seed": seed, "n_q": n_q, "L": L, "d": d,
                          "dv": dv, "boundary": bd})
    manifest["cases"]["attend"] = att_cases

    # ---- rotary tables (rope.hpp:21): sha of the exact bytes ----
    import hashlib
    ropes = []
    for d, base, mp in ((128, 500000.0, 8192), (128, 1e6, 8192), (16, 10000.0, 2048),
                        (32, 10000.0, 4096)):
        c, s = ob.rope_table(d, base, mp, lib=r)
        ropes.append({"d": d, "base": base, "max_position": mp,
                      "sha256": hashlib.sha256(c.tobytes() + s.tobytes()).hexdigest()})
    manifest["cases"]["rope"] = ropes

    # ---- attend_step (engine.hpp:43) ----
    step_cases = []
    specs = [
        # LLaMA-3.1-8B heads, bf16-valued cache, defaults
        dict(n_kv=8, nh=32, d=128, total=9000, n_q=1, base=500000.0, window=8192, cfg={}),
        dict(n_kv=8, nh=32, d=128, total=40000, n_q=1, base=500000.0, window=8192, cfg={}),
        # LLaMA-3.2-3B heads (group 3)
        dict(n_kv=8, nh=24, d=128, total=20000, n_q=1, base=500000.0, window=8192, cfg={}),
        # toy geometries (test_engine.cpp toy_selection)
        dict(n_kv=2, nh=4, d=16, total=2000, n_q=1, base=10000.0, window=2048,
             cfg=dict(l_global=16, l_local=256, l_chunk=128, span_m=16, k=4, k_prime=64)),
        dict(n_kv=2, nh=4, d=16, total=3000, n_q=64, base=10000.0, window=2048,
             cfg=dict(l_global=16, l_local=256, l_chunk=128, span_m=16, k=4, k_prime=64,
                      span_mode=1)),
        dict(n_kv=2, nh=4, d=16, total=900, n_q=128, base=10000.0, window=2048,
             cfg=dict(l_global=16, l_local=256, l_chunk=128, span_m=16, k=4, k_prime=0)),
    ]
    for i, sp in enumerate(specs):
        seed = 9000 + 10 * i
        bf = sp["d"] == 128
        K = keys(seed, sp["n_kv"], sp["total"], sp["d"], bf16=bf)
        V = keys(seed + 1, sp["n_kv"], sp["total"], sp["d"], bf16=bf)
        q = synth.uniform(seed + 2, sp["n_q"] * sp["nh"] * sp["d"]).reshape(sp["n_q"], -1)
        cfg = ob.SelectionConfig(**sp["cfg"])
        o, st, (sb, se) = ob.attend_step(q, sp["nh"], K, V, sp["total"], cfg, sp["base"],
                                         sp["window"], 2, lib=r)
        name = f"step_{i}"
        out[name + "_out"] = o
        out[name + "_sb"] = sb.astype(np.uint32)
        out[name + "_se"] = se.astype(np.uint32)
        case = dict(name=name, seed=seed, bf16=bf, lanes=ob.ref_lane_mode(sp["d"]),
                    scope_len=int(st.scope_len), entropy_max=st.entropy_max,
                    entropy_sum=st.entropy_sum, coverage_total=int(st.coverage_total))
        case.update({k: v for k, v in sp.items()})
        step_cases.append(case)
    manifest["cases"]["attend_step"] = step_cases

    np.savez_compressed(os.path.join(HERE, "ref_golden.npz"), **out)
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1)
    print("wrote", len(out), "arrays;", sum(len(v) for v in manifest["cases"].values()), "cases")


if __name__ == "__main__":
    main()
