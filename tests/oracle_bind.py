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
    """Mirror of oracle_selection_config / reattn::SelectionConfig (selection.hpp:127-152)."""

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


def round_bf16(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 (round to nearest even) -> fp32, vectorised like oracle_round_bf16."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)
