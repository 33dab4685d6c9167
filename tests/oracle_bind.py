"""ctypes bindings for the TEST-ONLY parity oracle (oracle/liboracle.so) and the
in-place reference shim (oracle/_ref/libreattn_ref_v{3,4}.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference leg import
this module; it is the checker, never the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "liboracle.so")
REF_DIR = os.path.join(ORACLE_DIR, "_ref")

u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
sz = C.c_size_t


class SelectionConfig(C.Structure):
    """Mirror of oracle_selection_config / reattn::SelectionConfig (selection.hpp:20-45)."""

    _fields_ = [("k", sz), ("k_prime", sz), ("span_m", sz), ("tile_size", sz),
                ("l_global", sz), ("l_local", sz), ("l_chunk", sz), ("span_mode", C.c_int)]

    def __init__(self, k=4, k_prime=127, span_m=32, tile_size=2048, l_global=32, l_local=4096,
                 l_chunk=512, span_mode=0):
        super().__init__(k, k_prime, span_m, tile_size, l_global, l_local, l_chunk, span_mode)


class StepStats(C.Structure):
    _fields_ = [("max_position_used", sz), ("ood_positions", sz), ("coverage_total", C.c_int),
                ("entropy_max", C.c_double), ("entropy_sum", C.c_double),
                ("entropy_rows", sz), ("scope_len_max", sz), ("scope_len", sz),
                ("n_spans", sz), ("coverage", sz)]


def ensure_oracle_built() -> None:
    if not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-C", ORACLE_DIR, "liboracle.so"], check=True,
                       stdout=subprocess.DEVNULL)


_oracle = None


def oracle() -> C.CDLL:
    global _oracle
    if _oracle is None:
        ensure_oracle_built()
        lib = C.CDLL(ORACLE_SO)
        lib.oracle_dot_f32.restype = C.c_float
        lib.oracle_dot_f32.argtypes = [f32p, f32p, sz]
        lib.oracle_dot_f64.restype = C.c_double
        lib.oracle_dot_f64.argtypes = [f32p, f32p, sz]
        lib.oracle_group_mean.argtypes = [f32p, sz, sz, sz, sz, f32p]
        lib.oracle_topk.argtypes = [f32p, sz, sz, C.POINTER(C.c_void_p), sz, sz, sz, sz, sz,
                                    u64p, f32p, C.POINTER(sz)]
        lib.oracle_vote.argtypes = [u64p, f32p, sz, sz, u64p, C.POINTER(sz)]
        lib.oracle_expand_spans.argtypes = [u64p, sz, sz, sz, C.c_int, u64p, u64p, C.POINTER(sz)]
        lib.oracle_rope_table.argtypes = [sz, C.c_double, sz, f32p, f32p]
        lib.oracle_attend.argtypes = [f32p, sz, f32p, f32p, sz, sz, sz, C.c_int, sz, f32p, f64p]
        lib.oracle_rotate_row.argtypes = [f32p, sz, f32p, f32p]
        lib.oracle_scope_indices.argtypes = [sz, sz, sz, u64p, u64p, sz, sz, u64p, C.POINTER(sz)]
        lib.oracle_attend_step.argtypes = [f32p, sz, sz, f32p, f32p, sz, sz, sz, sz,
                                           C.POINTER(SelectionConfig), f32p, f32p, sz, C.c_int,
                                           f32p, C.POINTER(StepStats), u64p, u64p]
        lib.oracle_set_lane_mode.argtypes = [C.c_int]
        lib.oracle_get_lane_mode.restype = C.c_int
        lib.oracle_synth_uniform.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, f32p, C.c_int]
        vp = C.c_void_p
        lib.oracle_topk_ex.argtypes = [f32p, sz, sz, C.POINTER(C.c_void_p), C.c_int, sz, sz, sz,
                                       sz, sz, C.c_int, u64p, f32p, C.POINTER(sz)]
        lib.oracle_attend_step_ex.argtypes = [f32p, sz, sz, vp, vp, C.c_int, sz, sz, sz, sz,
                                              C.POINTER(SelectionConfig), f32p, f32p, sz, C.c_int,
                                              C.c_int, f32p, f64p, C.POINTER(StepStats), u64p,
                                              u64p, u64p, C.POINTER(sz), vp, vp]
        lib.oracle_round_bf16.restype = C.c_float
        lib.oracle_round_bf16.argtypes = [C.c_float]
        _oracle = lib
    return _oracle


LANES_UNFUSED, LANES_FMA = 0, 1


class lane_mode:
    """Context manager: run the oracle's dot_f32 with the given lane arithmetic."""

    def __init__(self, mode: int):
        self.mode = mode

    def __enter__(self):
        self.prev = oracle().oracle_get_lane_mode()
        oracle().oracle_set_lane_mode(self.mode)
        return self

    def __exit__(self, *exc):
        oracle().oracle_set_lane_mode(self.prev)


def ref_lane_mode(d: int, trials: int = 512) -> int | None:
    """Which lane arithmetic the compiled reference uses for head dim d:
    LANES_UNFUSED, LANES_FMA, or None if it matches neither."""
    r = ref()
    if r is None:
        return None
    un, fm = sz(0), sz(0)
    v = r.ref_fma_selfcheck(d, trials, C.byref(un), C.byref(fm))
    return {0: LANES_UNFUSED, 1: LANES_FMA}.get(v)


def _ref_path() -> str | None:
    flags = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    flags = line
                    break
    except OSError:
        pass
    for name in (["libreattn_ref_v4.so"] if " avx512f" in flags else []) + ["libreattn_ref_v3.so"]:
        p = os.path.join(REF_DIR, name)
        if os.path.exists(p):
            return p
    return None


_ref = None


def ref() -> C.CDLL | None:
    """The reference headers compiled in place, or None when oracle/_ref was not built."""
    global _ref
    if _ref is None:
        p = _ref_path()
        if p is None:
            return None
        lib = C.CDLL(p)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_fused_topk.argtypes = [f32p, sz, sz, C.POINTER(C.c_void_p), sz, sz, sz, sz, sz,
                                       u64p, f32p, C.POINTER(sz), C.POINTER(sz)]
        lib.ref_naive_topk.argtypes = [f32p, sz, sz, C.POINTER(C.c_void_p), sz, sz, sz, sz,
                                       u64p, f32p, C.POINTER(sz), C.POINTER(sz)]
        lib.ref_vote.argtypes = [u64p, f32p, sz, sz, u64p, C.POINTER(sz)]
        lib.ref_expand_spans.argtypes = [u64p, sz, sz, sz, C.c_int, u64p, u64p, C.POINTER(sz)]
        lib.ref_rope_table.argtypes = [sz, C.c_double, sz, f32p, f32p]
        lib.ref_attend.argtypes = [f32p, sz, f32p, f32p, sz, sz, sz, C.c_int, sz, f32p, f64p]
        lib.ref_scope_indices.argtypes = [sz, sz, sz, u64p, u64p, sz, sz, u64p, C.POINTER(sz)]
        lib.ref_cache_create.restype = C.c_void_p
        lib.ref_cache_create.argtypes = [sz, sz, sz, sz, f32p, f32p, sz]
        lib.ref_cache_destroy.argtypes = [C.c_void_p]
        lib.ref_attend_step.argtypes = [C.c_void_p, f32p, sz, sz, sz, sz, sz, sz, sz, sz, sz,
                                        C.c_int, C.c_double, sz, C.c_int, f32p,
                                        C.POINTER(StepStats), u64p, u64p]
        lib.ref_fma_selfcheck.argtypes = [sz, sz, C.POINTER(sz), C.POINTER(sz)]
        lib.ref_snapshot_write.argtypes = [C.c_char_p, C.POINTER(C.c_void_p), sz]
        lib.ref_snapshot_read.argtypes = [C.c_char_p, sz, C.POINTER(sz), u64p, f32p, f32p, sz]
        vpp = C.c_void_p
        lib.ref_model_init.restype = vpp
        lib.ref_model_init.argtypes = [u64p, C.c_double, C.c_int, C.c_uint64]
        lib.ref_model_load.restype = vpp
        lib.ref_model_load.argtypes = [C.c_char_p]
        lib.ref_model_save.argtypes = [vpp, C.c_char_p]
        lib.ref_model_destroy.argtypes = [vpp]
        lib.ref_model_tensor.argtypes = [vpp, C.c_int, sz, f32p, sz]
        lib.ref_forward_full.argtypes = [vpp, C.POINTER(C.c_uint32), sz, f32p]
        lib.ref_engine_create.restype = vpp
        lib.ref_engine_create.argtypes = [vpp, u64p, C.c_int, C.c_int, C.c_int]
        lib.ref_engine_destroy.argtypes = [vpp]
        lib.ref_engine_prefill.argtypes = [vpp, C.POINTER(C.c_uint32), sz, f32p, sz, C.POINTER(sz)]
        lib.ref_engine_logits.argtypes = [vpp, f32p, sz, sz, f32p]
        lib.ref_engine_decode.argtypes = [vpp, C.c_uint32, C.POINTER(C.c_uint32), f32p, sz]
        lib.ref_engine_stats.argtypes = [vpp, f64p]
        lib.ref_random_tokens.argtypes = [sz, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32)]
        lib.ref_random_tokens.restype = None
        lib.ref_greedy_decode_full.argtypes = [vpp, C.POINTER(C.c_uint32), sz, sz,
                                               C.POINTER(C.c_uint32)]
        _ref = lib
    return _ref


# ---------------------------------------------------------------------------------------
# numpy-level helpers shared by both libraries (lib = oracle() or ref())

def _head_ptrs(keys_heads):
    arr = (C.c_void_p * len(keys_heads))(*[k.ctypes.data for k in keys_heads])
    return C.cast(arr, C.POINTER(C.c_void_p))


def topk(q: np.ndarray, n_heads: int, keys_heads: list[np.ndarray], k: int, lib=None,
         tile: int = 2048):
    """q: [n_q, n_heads*d] f32; keys_heads: n_kv arrays [count, d] f32 (contiguous).
    Returns (idx [n_kv, n_q, kk] u64, score [n_kv, n_q, kk] f32)."""
    lib = lib or oracle()
    q = np.ascontiguousarray(q, np.float32)
    n_q = q.shape[0]
    n_kv = len(keys_heads)
    count, d = keys_heads[0].shape
    idx = np.zeros(max(1, n_kv * n_q * k), np.uint64)
    sc = np.zeros(max(1, n_kv * n_q * k), np.float32)
    n_out = sz(0)
    ptrs = _head_ptrs(keys_heads)
    if lib is _oracle:
        rc = lib.oracle_topk(q, n_q, n_heads, ptrs, n_kv, count, d, d, k, idx, sc,
                             C.byref(n_out))
    else:
        rc = lib.ref_fused_topk(q, n_q, n_heads, ptrs, n_kv, count, d, k, tile, idx, sc,
                                C.byref(n_out), None)
    if rc != 0:
        raise ValueError(f"topk rc={rc}")
    kk = n_out.value
    idx = idx[: n_kv * n_q * k].reshape(n_kv, n_q, k)[:, :, :kk]
    sc = sc[: n_kv * n_q * k].reshape(n_kv, n_q, k)[:, :, :kk]
    return idx, sc


def vote(idx: np.ndarray, score: np.ndarray, k_prime: int, lib=None) -> np.ndarray:
    lib = lib or oracle()
    idx = np.ascontiguousarray(idx.ravel(), np.uint64)
    score = np.ascontiguousarray(score.ravel(), np.float32)
    out = np.zeros(max(1, min(k_prime, idx.size)), np.uint64)
    n = sz(0)
    fn = lib.oracle_vote if lib is _oracle else lib.ref_vote
    rc = fn(idx if idx.size else np.zeros(1, np.uint64),
            score if score.size else np.zeros(1, np.float32), idx.size, k_prime, out, C.byref(n))
    if rc != 0:
        raise ValueError(f"vote rc={rc}")
    return out[: n.value].copy()


def expand_spans(winners, span_m: int, middle_len: int, mode: int = 0, lib=None):
    lib = lib or oracle()
    w = np.ascontiguousarray(np.asarray(winners, np.uint64).ravel())
    b = np.zeros(max(1, w.size), np.uint64)
    e = np.zeros(max(1, w.size), np.uint64)
    n = sz(0)
    fn = lib.oracle_expand_spans if lib is _oracle else lib.ref_expand_spans
    rc = fn(w if w.size else np.zeros(1, np.uint64), w.size, span_m, middle_len, mode, b, e,
            C.byref(n))
    if rc == 2:
        raise IndexError("expand_spans: winner outside middle")
    if rc != 0:
        raise ValueError(f"expand_spans rc={rc}")
    return b[: n.value].copy(), e[: n.value].copy()


def rope_table(d: int, base: float, max_position: int, lib=None):
    lib = lib or oracle()
    c = np.zeros(max_position * (d // 2), np.float32)
    s = np.zeros(max_position * (d // 2), np.float32)
    fn = lib.oracle_rope_table if lib is _oracle else lib.ref_rope_table
    fn(d, base, max_position, c, s)
    return c.reshape(max_position, d // 2), s.reshape(max_position, d // 2)


def attend(q, k, v, boundary=None, lib=None):
    lib = lib or oracle()
    q = np.ascontiguousarray(q, np.float32)
    k = np.ascontiguousarray(k, np.float32)
    v = np.ascontiguousarray(v, np.float32)
    n_q, d = q.shape
    L, dv = v.shape
    out = np.zeros(max(1, n_q * dv), np.float32)
    ent = np.zeros(max(1, n_q), np.float64)
    fn = lib.oracle_attend if lib is _oracle else lib.ref_attend
    rc = fn(q, n_q, k, v, L, d, dv, int(boundary is not None), boundary or 0, out, ent)
    if rc != 0:
        raise ValueError("empty key set")
    return out[: n_q * dv].reshape(n_q, dv), ent[:n_q]


def cache_bounds(total: int, l_global: int, l_local: int):
    g = min(total, l_global)
    return g, total - min(total - g, l_local)


def attend_step(q_pre, n_head, cache_k, cache_v, total, cfg: SelectionConfig, rope_base,
                max_position, mode=2, lib=None, ref_cache=None):
    """cache_k/v: [n_kv, cap, d] f32 head-major.  Returns (out [n_q, n_head*d], stats,
    (span_begin, span_end))."""
    lib = lib or oracle()
    q_pre = np.ascontiguousarray(q_pre, np.float32)
    n_q = q_pre.shape[0]
    n_kv, cap, d = cache_k.shape
    out = np.zeros(max(1, n_q * n_head * d), np.float32)
    st = StepStats()
    st.coverage_total = 1
    sb = np.zeros(max(1, cfg.k_prime), np.uint64)
    se = np.zeros(max(1, cfg.k_prime), np.uint64)
    if lib is _oracle:
        ck = np.ascontiguousarray(cache_k, np.float32).ravel()
        cv = np.ascontiguousarray(cache_v, np.float32).ravel()
        cs, sn = rope_table(d, rope_base, max_position)
        rc = lib.oracle_attend_step(q_pre, n_q, n_head, ck, cv, n_kv, d, cap, total,
                                    C.byref(cfg), cs.ravel(), sn.ravel(), max_position, mode,
                                    out, C.byref(st), sb, se)
    else:
        own = ref_cache is None
        if own:
            ck = np.ascontiguousarray(cache_k[:, :total], np.float32)
            cv = np.ascontiguousarray(cache_v[:, :total], np.float32)
            ref_cache = lib.ref_cache_create(n_kv, d, cfg.l_global, cfg.l_local, ck.ravel(),
                                             cv.ravel(), total)
        rc = lib.ref_attend_step(ref_cache, q_pre, n_q, n_head, cfg.k, cfg.k_prime, cfg.span_m,
                                 cfg.tile_size, cfg.l_global, cfg.l_local, cfg.l_chunk,
                                 cfg.span_mode, rope_base, max_position, mode, out,
                                 C.byref(st), sb, se)
        if own:
            lib.ref_cache_destroy(ref_cache)
    if rc != 0:
        raise RuntimeError(f"attend_step rc={rc}")
    return out[: n_q * n_head * d].reshape(n_q, n_head * d), st, (sb[: st.n_spans].copy(),
                                                                   se[: st.n_spans].copy())


def host_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return max(1, os.cpu_count() or 1)


def _dtype_code(a: np.ndarray) -> int:
    if a.dtype == np.float32:
        return 0
    if a.dtype in (np.uint16, np.int16):
        return 1  # bf16 words
    raise TypeError(f"cache storage must be float32 or bf16 words (uint16), got {a.dtype}")


def topk_ex(q, n_heads: int, keys_hm: np.ndarray, row0: int, count: int, k: int,
            threads: int | None = None):
    """Multi-threaded oracle top-k over a head-major [n_kv, cap, d] fp32 or bf16-word array
    (middle rows [row0, row0 + count)).  Returns (idx [n_kv, n_q, kk], score)."""
    lib = oracle()
    q = np.ascontiguousarray(q, np.float32)
    n_q = q.shape[0]
    n_kv, cap, d = keys_hm.shape
    assert keys_hm.flags.c_contiguous
    dt = _dtype_code(keys_hm)
    esz = keys_hm.itemsize
    base = keys_hm.ctypes.data
    ptrs = (C.c_void_p * n_kv)(*[base + (h * cap + row0) * d * esz for h in range(n_kv)])
    idx = np.zeros(max(1, n_kv * n_q * k), np.uint64)
    sc = np.zeros(max(1, n_kv * n_q * k), np.float32)
    n_out = sz(0)
    rc = lib.oracle_topk_ex(q, n_q, n_heads, C.cast(ptrs, C.POINTER(C.c_void_p)), dt, n_kv, count,
                            d, d, k, threads or host_threads(), idx, sc, C.byref(n_out))
    if rc != 0:
        raise ValueError(f"topk_ex rc={rc}")
    kk = n_out.value
    return (idx[: n_kv * n_q * k].reshape(n_kv, n_q, k)[:, :, :kk],
            sc[: n_kv * n_q * k].reshape(n_kv, n_q, k)[:, :, :kk])


def attend_step_ex(q_pre, n_head, cache_k, cache_v, total, cfg: SelectionConfig, rope_base,
                   max_position, mode=2, threads: int | None = None, candidates: bool = False):
    """Multi-threaded oracle attend_step over a head-major [n_kv, cap, d] cache held as fp32
    or as bf16 words (uint16; widened exactly).  Returns (out [n_q, n_head*d],
    entropy [n_q, n_head], stats, (span_begin, span_end), winners), plus the per-head top-k
    lists (idx [n_kv, n_q, k], score) when candidates=True."""
    lib = oracle()
    q_pre = np.ascontiguousarray(q_pre, np.float32)
    n_q = q_pre.shape[0]
    n_kv, cap, d = cache_k.shape
    assert cache_k.flags.c_contiguous and cache_v.flags.c_contiguous
    assert cache_k.dtype == cache_v.dtype
    out = np.zeros(max(1, n_q * n_head * d), np.float32)
    ent = np.zeros(max(1, n_q * n_head), np.float64)
    st = StepStats()
    st.coverage_total = 1
    sb = np.zeros(max(1, cfg.k_prime), np.uint64)
    se = np.zeros(max(1, cfg.k_prime), np.uint64)
    wn = np.zeros(max(1, cfg.k_prime), np.uint64)
    nw = sz(0)
    cs, sn = rope_table(d, rope_base, max_position)
    ci = np.zeros(n_kv * n_q * cfg.k if candidates else 1, np.uint64)
    cf = np.zeros(n_kv * n_q * cfg.k if candidates else 1, np.float32)
    rc = lib.oracle_attend_step_ex(q_pre, n_q, n_head, cache_k.ctypes.data, cache_v.ctypes.data,
                                   _dtype_code(cache_k), n_kv, d, cap, total, C.byref(cfg),
                                   cs.ravel(), sn.ravel(), max_position, mode,
                                   threads or host_threads(), out, ent, C.byref(st), sb, se, wn,
                                   C.byref(nw), ci.ctypes.data if candidates else None,
                                   cf.ctypes.data if candidates else None)
    if rc != 0:
        raise RuntimeError(f"attend_step_ex rc={rc}")
    res = (out[: n_q * n_head * d].reshape(n_q, n_head * d), ent[: n_q * n_head].reshape(n_q, n_head),
           st, (sb[: st.n_spans].copy(), se[: st.n_spans].copy()), wn[: nw.value].copy())
    if candidates:
        res = res + ((ci.reshape(n_kv, n_q, cfg.k), cf.reshape(n_kv, n_q, cfg.k)),)
    return res


def bf16_words(t) -> np.ndarray:
    """A torch bf16 tensor (any device) as host uint16 words (no widening copy)."""
    import torch
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 (round to nearest even) -> fp32, vectorised like oracle_round_bf16."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


# ---------------------------------------------------------------------------------------
# the reference's decoder model and Engine (model.hpp, engine.hpp:119-216), run in place

def _u32(tokens):
    t = np.ascontiguousarray(np.asarray(tokens, dtype=np.uint32))
    return t, t.ctypes.data_as(C.POINTER(C.c_uint32))


class RefModel:
    """reattn::ModelWeights from init_random(cfg, seed) or load_weights(path)."""

    def __init__(self, cfg=None, seed=0, path=None):
        lib = ref()
        if lib is None:
            raise RuntimeError("oracle/_ref not built")
        self.lib = lib
        if path is not None:
            self.h = lib.ref_model_load(os.fsencode(path))
        else:
            c8 = np.array([cfg.n_layer, cfg.n_head, cfg.n_kv_head, cfg.d_model, cfg.d_head,
                           cfg.d_ff, cfg.vocab_size, cfg.pretrain_window], np.uint64)
            self.h = lib.ref_model_init(c8, cfg.rope_base, cfg.attention_mode, seed)
        if not self.h:
            raise RuntimeError(lib.ref_last_error().decode())
        self.cfg = cfg

    def tensor(self, kind, layer, shape):
        out = np.zeros(shape, np.float32)
        rc = self.lib.ref_model_tensor(self.h, kind, layer, out, out.size)
        if rc:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return out

    def save(self, path):
        rc = self.lib.ref_model_save(self.h, os.fsencode(path))
        if rc:
            raise RuntimeError(self.lib.ref_last_error().decode())

    def forward_full(self, tokens, vocab):
        t, tp = _u32(tokens)
        out = np.zeros((t.size, vocab), np.float32)
        rc = self.lib.ref_forward_full(self.h, tp, t.size, out)
        if rc:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return out

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_model_destroy(self.h)
            self.h = None


class RefEngine:
    """reattn::Engine (kind 0) or reattn::WindowReference (kind 1) over a RefModel."""

    def __init__(self, model: RefModel, sel, mode=2, kind=0, d_model=None, vocab=None):
        self.model, self.lib = model, model.lib
        s7 = np.array([sel.k, sel.k_prime, sel.span_m, sel.tile_size, sel.l_global, sel.l_local,
                       sel.l_chunk], np.uint64)
        self.h = self.lib.ref_engine_create(model.h, s7, sel.span_mode, mode, kind)
        if not self.h:
            raise RuntimeError(self.lib.ref_last_error().decode())
        self.d_model, self.vocab = d_model, vocab

    def _chk(self, rc):
        if rc:
            raise RuntimeError(self.lib.ref_last_error().decode())

    def prefill(self, tokens):
        t, tp = _u32(tokens)
        buf = np.zeros(t.size * self.d_model + 1, np.float32)
        rows = sz(0)
        self._chk(self.lib.ref_engine_prefill(self.h, tp, t.size, buf, buf.size, C.byref(rows)))
        return buf[: rows.value * self.d_model].reshape(rows.value, self.d_model).copy()

    def logits(self, hidden):
        h = np.ascontiguousarray(hidden, np.float32)
        out = np.zeros((h.shape[0], self.vocab), np.float32)
        self._chk(self.lib.ref_engine_logits(self.h, h, h.shape[0], self.d_model, out))
        return out

    def decode_step(self, tok):
        nt = C.c_uint32()
        lg = np.zeros(self.vocab, np.float32)
        self._chk(self.lib.ref_engine_decode(self.h, tok, C.byref(nt), lg, self.vocab))
        return nt.value, lg

    def stats(self):
        out = np.zeros(10, np.float64)
        self._chk(self.lib.ref_engine_stats(self.h, out))
        keys = ["max_position_used", "ood_positions", "coverage_total", "entropy_max",
                "entropy_sum", "entropy_rows", "scope_len_max", "peak_scratch_bytes",
                "chunks_processed", "decode_steps"]
        return dict(zip(keys, out.tolist()))

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_engine_destroy(self.h)
            self.h = None


def random_tokens(n: int, vocab: int, seed: int) -> np.ndarray:
    """test_engine.cpp:50-56 random_tokens, generated by the reference build itself."""
    out = np.zeros(n, np.uint32)
    ref().ref_random_tokens(n, vocab, seed, out.ctypes.data_as(C.POINTER(C.c_uint32)))
    return out


def greedy_decode_full(model: "RefModel", prompt, steps: int) -> list:
    t, tp = _u32(prompt)
    out = np.zeros(steps, np.uint32)
    rc = model.lib.ref_greedy_decode_full(model.h, tp, t.size, steps,
                                          out.ctypes.data_as(C.POINTER(C.c_uint32)))
    if rc:
        raise RuntimeError(model.lib.ref_last_error().decode())
    return out.tolist()
