"""ctypes binding of libreattn_cuda.so (the C-ABI in include/reattn_cuda.h).

This is the Python host mirror of the reference's hot-path interface
(/root/reference/proj/include/reattn: fused_topk_scores, vote, expand_spans,
assemble_scope, attend, attend_step).  Device memory and streams come from PyTorch
(plumbing only); every computation runs in the sm_100a kernels of the library.  There is
no CPU fallback: if the library is missing or no GPU is present, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("REATTN_LIB", os.path.join(PKG_DIR, "libreattn_cuda.so"))
HEADER = os.path.join(os.path.dirname(PKG_DIR), "include", "reattn_cuda.h")

OK, EINVAL, ERANGE, ELOGIC, ECUDA, ERUNTIME = range(6)
F32, BF16 = 0, 1
SPAN_ALIGNED, SPAN_CENTERED = 0, 1
MODE_FULL, MODE_WINDOW, MODE_REATTENTION = 0, 1, 2
LANES_UNFUSED, LANES_FMA = 0, 1
PREFILL_EXACT, PREFILL_TENSOR_SCAN, PREFILL_TENSOR_ATTN, PREFILL_TENSOR = 0, 1, 2, 3
PREFILL_DEFAULT = PREFILL_TENSOR  # a new context's mode

u64 = C.c_uint64
vp = C.c_void_p


class SelectionConfig(C.Structure):
    """reattn::SelectionConfig (selection.hpp:20-45); defaults are the reference's."""

    _fields_ = [("k", u64), ("k_prime", u64), ("span_m", u64), ("tile_size", u64),
                ("l_global", u64), ("l_local", u64), ("l_chunk", u64), ("span_mode", C.c_int32),
                ("reserved", C.c_int32)]

    def __init__(self, k=4, k_prime=127, span_m=32, tile_size=2048, l_global=32, l_local=4096,
                 l_chunk=512, span_mode=SPAN_ALIGNED):
        super().__init__(k, k_prime, span_m, tile_size, l_global, l_local, l_chunk, span_mode, 0)

    def budget(self) -> int:
        return self.l_global + self.k_prime * self.span_m + self.l_local


class StepStats(C.Structure):
    _fields_ = [("max_position_used", u64), ("ood_positions", u64), ("coverage_total", C.c_int32),
                ("reserved", C.c_int32), ("entropy_max", C.c_double), ("entropy_sum", C.c_double),
                ("entropy_rows", u64), ("scope_len", u64), ("n_spans", u64), ("coverage", u64),
                ("peak_scratch_bytes", u64)]


class ModelConfig(C.Structure):
    """reattn::ModelConfig (model.hpp:39-61); defaults are the reference's toy model."""

    _fields_ = [("n_layer", u64), ("n_head", u64), ("n_kv_head", u64), ("d_model", u64),
                ("d_head", u64), ("d_ff", u64), ("vocab_size", u64), ("pretrain_window", u64),
                ("rope_base", C.c_double), ("attention_mode", C.c_int32), ("reserved", C.c_int32)]

    def __init__(self, n_layer=2, n_head=4, n_kv_head=2, d_model=128, d_head=32, d_ff=512,
                 vocab_size=512, pretrain_window=4096, rope_base=10000.0,
                 attention_mode=MODE_REATTENTION):
        super().__init__(n_layer, n_head, n_kv_head, d_model, d_head, d_ff, vocab_size,
                         pretrain_window, rope_base, attention_mode, 0)


class RunStats(C.Structure):
    """reattn::RunStats (engine.hpp:23-37) accumulated by an Engine."""

    _fields_ = [("max_position_used", u64), ("ood_positions", u64), ("coverage_total", C.c_int32),
                ("reserved", C.c_int32), ("entropy_max", C.c_double), ("entropy_sum", C.c_double),
                ("entropy_rows", u64), ("scope_len_max", u64), ("peak_scratch_bytes", u64),
                ("chunks_processed", u64), ("decode_steps", u64)]


# reattn_weight_kind
(W_EMBEDDING, W_WQ, W_WK, W_WV, W_WO, W_GATE, W_UP, W_DOWN, W_NORM_ATTN, W_NORM_FFN,
 W_NORM_FINAL, W_LM_HEAD) = range(12)


class ReattnError(RuntimeError):
    pass


class InvalidArgument(ReattnError, ValueError):
    """std::invalid_argument"""


class OutOfRange(ReattnError, IndexError):
    """std::out_of_range"""


class LogicError(ReattnError):
    """std::logic_error"""


class CudaError(ReattnError):
    pass


_EXC = {EINVAL: InvalidArgument, ERANGE: OutOfRange, ELOGIC: LogicError, ECUDA: CudaError,
        ERUNTIME: ReattnError}

# (name, restype, argtypes) for every exported symbol; tests check this list against the
# header so the binding and include/reattn_cuda.h cannot drift.
SIGNATURES = [
    ("reattn_version", C.c_char_p, []),
    ("reattn_ctx_create", C.c_int, [C.c_int, C.POINTER(vp)]),
    ("reattn_ctx_destroy", None, [vp]),
    ("reattn_last_error", C.c_char_p, [vp]),
    ("reattn_ctx_set_stream", C.c_int, [vp, vp]),
    ("reattn_ctx_stream", vp, [vp]),
    ("reattn_ctx_set_lanes", C.c_int, [vp, C.c_int]),
    ("reattn_ctx_set_prefill", C.c_int, [vp, C.c_int]),
    ("reattn_ctx_synchronize", C.c_int, [vp]),
    ("reattn_ctx_num_sms", C.c_int, [vp]),
    ("reattn_malloc", C.c_int, [vp, u64, C.POINTER(vp)]),
    ("reattn_free", C.c_int, [vp, vp]),
    ("reattn_memcpy_h2d", C.c_int, [vp, vp, vp, u64]),
    ("reattn_memcpy_d2h", C.c_int, [vp, vp, vp, u64]),
    ("reattn_cache_create", C.c_int, [vp, u64, u64, u64, u64, u64, C.c_int, C.POINTER(vp)]),
    ("reattn_cache_destroy", None, [vp]),
    ("reattn_cache_reserve", C.c_int, [vp, vp, u64]),
    ("reattn_cache_append", C.c_int, [vp, vp, vp, vp, u64, C.c_int]),
    ("reattn_cache_set_total", C.c_int, [vp, vp, u64]),
    ("reattn_snapshot_open", C.c_int, [vp, C.c_char_p, C.POINTER(vp)]),
    ("reattn_snapshot_info", C.c_int, [vp] + [C.POINTER(C.c_uint32)] * 3),
    ("reattn_snapshot_layer_info", C.c_int, [vp, C.c_uint32] + [C.POINTER(u64)] * 3),
    ("reattn_snapshot_load_layer", C.c_int, [vp, vp, C.c_uint32, C.c_int, u64, C.POINTER(vp)]),
    ("reattn_snapshot_close", None, [vp]),
    ("reattn_snapshot_write", C.c_int, [vp, C.c_char_p, C.POINTER(vp), C.c_uint32]),
    ("reattn_cache_info", C.c_int, [vp] + [C.POINTER(u64)] * 8 + [C.POINTER(C.c_int)]),
    ("reattn_cache_keys", vp, [vp]),
    ("reattn_cache_values", vp, [vp]),
    ("reattn_rope_create", C.c_int, [vp, u64, C.c_double, u64, C.POINTER(vp)]),
    ("reattn_rope_destroy", None, [vp]),
    ("reattn_rope_tables_host", C.c_int, [vp, vp, vp]),
    ("reattn_rope_rotate", C.c_int, [vp, vp, vp, vp, u64]),
    ("reattn_fused_topk", C.c_int, [vp, vp, u64, u64, vp, C.c_int, u64, u64, u64, u64, u64, u64,
                                    vp, vp, C.POINTER(u64), C.POINTER(u64)]),
    ("reattn_naive_topk", C.c_int, [vp, vp, u64, u64, vp, C.c_int, u64, u64, u64, u64, u64, u64,
                                    vp, vp, C.POINTER(u64), C.POINTER(u64)]),
    ("reattn_group_mean", C.c_int, [vp, vp, u64, u64, u64, u64, vp]),
    ("reattn_dot_f32", C.c_int, [vp, vp, vp, u64, u64, vp]),
    ("reattn_dot_f64", C.c_int, [vp, vp, vp, u64, u64, vp]),
    ("reattn_matmul", C.c_int, [vp, vp, vp, u64, u64, u64, vp]),
    ("reattn_vote", C.c_int, [vp, vp, vp, u64, u64, vp, C.POINTER(u64)]),
    ("reattn_tally", C.c_int, [vp, vp, vp, u64, vp, vp, vp, C.POINTER(u64)]),
    ("reattn_expand_spans", C.c_int, [vp, vp, u64, u64, u64, C.c_int, vp, vp, C.POINTER(u64)]),
    ("reattn_assemble_scope", C.c_int, [vp, vp, vp, vp, u64, u64, vp, vp, vp, C.POINTER(u64)]),
    ("reattn_attend", C.c_int, [vp, vp, u64, vp, vp, u64, u64, u64, C.c_int, u64, vp, vp]),
    ("reattn_attend_step", C.c_int, [vp, vp, vp, vp, u64, u64, C.POINTER(SelectionConfig),
                                     C.c_int, vp, C.POINTER(StepStats), vp, vp, vp]),
    ("reattn_plan_create", C.c_int, [vp, vp, vp, u64, u64, C.POINTER(SelectionConfig), C.c_int,
                                     C.POINTER(vp)]),
    ("reattn_plan_destroy", None, [vp]),
    ("reattn_plan_q", vp, [vp]),
    ("reattn_plan_out", vp, [vp]),
    ("reattn_plan_launch", C.c_int, [vp]),
    ("reattn_plan_launch_scan", C.c_int, [vp]),
    ("reattn_debug_trace", C.c_int, [C.POINTER(u64), u64]),
    ("reattn_rmsnorm", C.c_int, [vp, vp, u64, u64, vp, vp]),
    ("reattn_silu_mul", C.c_int, [vp, vp, vp, u64]),
    ("reattn_stable_softmax", C.c_int, [vp, vp, u64, vp]),
    ("reattn_attention_entropy", C.c_int, [vp, vp, u64, vp]),
    ("reattn_debug_gemv_workspace", C.c_size_t, [u64]),
    ("reattn_debug_gemv", C.c_int, [vp, vp, vp, u64, u64, u64, vp, C.c_float, vp]),
    ("reattn_plan_run_host", C.c_int, [vp, vp, vp]),
    ("reattn_plan_stats", C.c_int, [vp, C.POINTER(StepStats)]),
    ("reattn_plan_info", C.c_int, [vp, C.POINTER(u64), C.POINTER(u64), C.POINTER(u64)]),
    ("reattn_plan_result", C.c_int, [vp, C.POINTER(StepStats), vp, vp, vp]),
    ("reattn_plan_stage_result", C.c_int, [vp]),
    ("reattn_plan_staged_result", C.c_int, [vp, C.POINTER(StepStats), vp, vp, vp]),
    ("reattn_plan_set_append", C.c_int, [vp, C.c_int]),
    ("reattn_plan_follows_cache", C.c_int, [vp]),
    ("reattn_plan_cache_generation", u64, [vp]),
    ("reattn_plan_k_in", vp, [vp]),
    ("reattn_plan_v_in", vp, [vp]),
    ("reattn_plan_step_host", C.c_int, [vp, vp, vp, vp, vp]),
    ("reattn_batch_plan_create", C.c_int, [vp, C.POINTER(vp), C.c_uint32, vp, u64, vp, C.c_int,
                                           C.POINTER(vp)]),
    ("reattn_batch_plan_destroy", None, [vp]),
    ("reattn_batch_plan_q", vp, [vp]),
    ("reattn_batch_plan_out", vp, [vp]),
    ("reattn_batch_plan_launch", C.c_int, [vp]),
    ("reattn_batch_plan_run_host", C.c_int, [vp, vp, vp]),
    ("reattn_batch_plan_stats", C.c_int, [vp, C.c_uint32, vp]),
    ("reattn_batch_plan_info", C.c_int, [vp, C.POINTER(u64), C.POINTER(u64), C.POINTER(C.c_int)]),
    ("reattn_synth_uniform", C.c_int, [vp, vp, u64, C.c_int, u64, u64]),
    ("reattn_model_config_validate", C.c_int, [vp, C.POINTER(ModelConfig)]),
    ("reattn_weights_create", C.c_int, [vp, C.POINTER(ModelConfig), C.POINTER(vp)]),
    ("reattn_weights_init_random", C.c_int, [vp, C.POINTER(ModelConfig), u64, C.POINTER(vp)]),
    ("reattn_weights_load", C.c_int, [vp, C.c_char_p, C.POINTER(vp)]),
    ("reattn_weights_save", C.c_int, [vp, vp, C.c_char_p]),
    ("reattn_weights_config", C.c_int, [vp, C.POINTER(ModelConfig)]),
    ("reattn_weights_shape", C.c_int, [vp, C.c_int, C.POINTER(u64), C.POINTER(u64)]),
    ("reattn_weights_upload", C.c_int, [vp, vp, C.c_int, u64, vp, u64]),
    ("reattn_weights_download", C.c_int, [vp, vp, C.c_int, u64, vp, u64]),
    ("reattn_weights_destroy", None, [vp]),
    ("reattn_weights_synth", C.c_int, [vp, C.POINTER(ModelConfig), u64, C.POINTER(vp)]),
    ("reattn_engine_synth_context", C.c_int, [vp, u64, u64]),
    ("reattn_engine_create", C.c_int, [vp, vp, C.POINTER(SelectionConfig), C.c_int, C.c_int,
                                       C.POINTER(vp)]),
    ("reattn_engine_reset", C.c_int, [vp]),
    ("reattn_engine_prefill", C.c_int, [vp, vp, u64, C.POINTER(u64)]),
    ("reattn_engine_hidden", C.c_int, [vp, vp, u64]),
    ("reattn_engine_logits", C.c_int, [vp, vp, u64, vp]),
    ("reattn_engine_decode_step", C.c_int, [vp, C.c_uint32, C.POINTER(C.c_uint32)]),
    ("reattn_engine_last_logits", C.c_int, [vp, vp, u64]),
    ("reattn_engine_stats", C.c_int, [vp, C.POINTER(RunStats)]),
    ("reattn_engine_decode_latencies", C.c_int, [vp, vp, u64, C.POINTER(u64)]),
    ("reattn_engine_last_spans", C.c_int, [vp, u64, vp, vp, u64, C.POINTER(u64)]),
    ("reattn_engine_cache", vp, [vp, u64]),
    ("reattn_engine_destroy", None, [vp]),
    ("reattn_shard_plan_create", C.c_int, [vp, vp, vp, u64, C.POINTER(SelectionConfig), u64,
                                           C.c_int, C.c_int, C.POINTER(vp)]),
    ("reattn_shard_plan_destroy", None, [vp]),
    ("reattn_shard_range", C.c_int, [u64, u64, C.c_int, C.c_int, C.POINTER(u64), C.POINTER(u64)]),
    ("reattn_shard_plan_q", vp, [vp]),
    ("reattn_shard_plan_out", vp, [vp]),
    ("reattn_shard_buffers", C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(u64),
                                       C.POINTER(vp), C.POINTER(vp), C.POINTER(u64)]),
    ("reattn_shard_scan", C.c_int, [vp]),
    ("reattn_shard_select", C.c_int, [vp]),
    ("reattn_shard_attend", C.c_int, [vp]),
    ("reattn_shard_combine", C.c_int, [vp]),
    ("reattn_shard_stats", C.c_int, [vp, C.POINTER(StepStats), vp, vp]),
    ("reattn_comm_unique_id", C.c_int, [vp]),
    ("reattn_comm_create", C.c_int, [vp, C.c_int, C.c_int, vp, C.POINTER(vp)]),
    ("reattn_comm_destroy", None, [vp]),
    ("reattn_shard_step", C.c_int, [vp, vp]),
    ("reattn_shard_capture", C.c_int, [vp, vp]),
    ("reattn_shard_run_host", C.c_int, [vp, vp, vp, vp]),
]

_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load libreattn_cuda.so.  Raises if it has not been built (no silent fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built; run __graft_entry__.build() "
                          "(make -C paper_2407_15176_b200/csrc)")
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _ptr(t) -> int:
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


class Context:
    """One device context (reattn_ctx): stream, lane arithmetic, scratch arena."""

    def __init__(self, device: int = 0, stream=None, lanes: int = LANES_UNFUSED):
        self.lib = load_library()
        h = vp()
        rc = self.lib.reattn_ctx_create(device, C.byref(h))
        if rc != OK:
            raise CudaError(f"reattn_ctx_create failed (rc={rc}); is a GPU visible?")
        self.h = h
        self.device = device
        if stream is not None:
            self.check(self.lib.reattn_ctx_set_stream(self.h, stream))
        self.set_lanes(lanes)

    def check(self, rc: int) -> None:
        if rc != OK:
            msg = self.lib.reattn_last_error(self.h).decode()
            raise _EXC.get(rc, ReattnError)(msg)

    def set_lanes(self, lanes: int) -> None:
        self.check(self.lib.reattn_ctx_set_lanes(self.h, lanes))

    def set_prefill(self, mode: int) -> None:
        """Bit mask: PREFILL_TENSOR_SCAN (tcgen05 scan, bit-exact; the default),
        PREFILL_TENSOR_ATTN (tcgen05 attention, bf16 tolerance), PREFILL_TENSOR (both);
        PREFILL_EXACT (0) = CUDA-core scan and f64 attention."""
        self.check(self.lib.reattn_ctx_set_prefill(self.h, mode))

    @property
    def stream(self) -> int:
        return self.lib.reattn_ctx_stream(self.h)

    def synchronize(self) -> None:
        self.check(self.lib.reattn_ctx_synchronize(self.h))

    def close(self) -> None:
        if self.h:
            self.lib.reattn_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- selection (device tensors) ----
    def fused_topk(self, q, n_heads: int, keys, n_kv: int, head_stride: int, row0: int,
                   count: int, d: int, k: int, idx_out, score_out, key_dtype: int) -> tuple:
        n_out, scratch = u64(), u64()
        self.check(self.lib.reattn_fused_topk(self.h, _ptr(q), q.shape[0], n_heads, _ptr(keys),
                                              key_dtype, n_kv, head_stride, row0, count, d, k,
                                              _ptr(idx_out), _ptr(score_out), C.byref(n_out),
                                              C.byref(scratch)))
        return n_out.value, scratch.value

    def naive_topk(self, q, n_heads: int, keys, n_kv: int, head_stride: int, row0: int,
                   count: int, d: int, k: int, idx_out, score_out, key_dtype: int) -> tuple:
        n_out, scratch = u64(), u64()
        self.check(self.lib.reattn_naive_topk(self.h, _ptr(q), q.shape[0], n_heads, _ptr(keys),
                                              key_dtype, n_kv, head_stride, row0, count, d, k,
                                              _ptr(idx_out), _ptr(score_out), C.byref(n_out),
                                              C.byref(scratch)))
        return n_out.value, scratch.value

    def group_mean(self, q, n_heads: int, n_kv: int, d: int, out) -> None:
        self.check(self.lib.reattn_group_mean(self.h, _ptr(q), q.shape[0], n_heads, n_kv, d, _ptr(out)))

    def dot_f32(self, a, b, out) -> None:
        self.check(self.lib.reattn_dot_f32(self.h, _ptr(a), _ptr(b), a.shape[0], a.shape[1], _ptr(out)))

    def dot_f64(self, a, b, out) -> None:
        self.check(self.lib.reattn_dot_f64(self.h, _ptr(a), _ptr(b), a.shape[0], a.shape[1], _ptr(out)))

    def matmul(self, a, b, out) -> None:
        self.check(self.lib.reattn_matmul(self.h, _ptr(a), _ptr(b), a.shape[0], a.shape[1],
                                          b.shape[1], _ptr(out)))

    def vote(self, idx, score, k_prime: int, winners_out) -> int:
        n = u64()
        self.check(self.lib.reattn_vote(self.h, _ptr(idx), _ptr(score), idx.numel(), k_prime,
                                        _ptr(winners_out), C.byref(n)))
        return n.value

    def tally(self, idx, score, idx_out, votes_out, score_out) -> int:
        n = u64()
        self.check(self.lib.reattn_tally(self.h, _ptr(idx), _ptr(score), idx.numel(),
                                         _ptr(idx_out), _ptr(votes_out), _ptr(score_out),
                                         C.byref(n)))
        return n.value

    def expand_spans(self, winners, span_m: int, middle_len: int, mode: int, b_out, e_out) -> int:
        n = u64()
        self.check(self.lib.reattn_expand_spans(self.h, _ptr(winners), winners.numel(), span_m,
                                                middle_len, mode, _ptr(b_out), _ptr(e_out),
                                                C.byref(n)))
        return n.value

    def attend(self, q, k, v, boundary, out, entropy) -> None:
        n_q, d = q.shape
        L, dv = v.shape
        self.check(self.lib.reattn_attend(self.h, _ptr(q), n_q, _ptr(k), _ptr(v), L, d, dv,
                                          int(boundary is not None), boundary or 0, _ptr(out),
                                          _ptr(entropy)))

    def synth_uniform(self, t, seed: int, offset: int = 0) -> None:
        import torch
        dt = BF16 if t.dtype == torch.bfloat16 else F32
        self.check(self.lib.reattn_synth_uniform(self.h, _ptr(t), t.numel(), dt, seed, offset))


class Snapshot:
    """RKVC cache snapshot (kv_cache.hpp:120-209) read into device caches."""

    def __init__(self, ctx: Context, path: str):
        self.ctx = ctx
        h = vp()
        ctx.check(ctx.lib.reattn_snapshot_open(ctx.h, os.fsencode(path), C.byref(h)))
        self.h = h
        a, b, c = C.c_uint32(), C.c_uint32(), C.c_uint32()
        ctx.lib.reattn_snapshot_info(h, C.byref(a), C.byref(b), C.byref(c))
        self.n_layers, self.n_kv, self.d = a.value, b.value, c.value

    def layer_info(self, layer: int) -> dict:
        t, g, l = u64(), u64(), u64()
        self.ctx.check(self.ctx.lib.reattn_snapshot_layer_info(self.h, layer, C.byref(t),
                                                               C.byref(g), C.byref(l)))
        return {"total": t.value, "l_global": g.value, "l_local_max": l.value}

    def load_layer(self, layer: int, dtype: int = F32, capacity: int = 0) -> "Cache":
        h = vp()
        self.ctx.check(self.ctx.lib.reattn_snapshot_load_layer(self.ctx.h, self.h, layer, dtype,
                                                               capacity, C.byref(h)))
        return Cache._adopt(self.ctx, h)

    def close(self) -> None:
        if getattr(self, "h", None):
            self.ctx.lib.reattn_snapshot_close(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def write_snapshot(ctx: Context, path: str, caches) -> None:
    """write_cache_snapshot (kv_cache.hpp:143-166) from device caches."""
    arr = (vp * max(1, len(caches)))(*[c.h for c in caches])
    ctx.check(ctx.lib.reattn_snapshot_write(ctx.h, os.fsencode(path), arr, len(caches)))


class Rope:
    """reattn::RotaryTable (rope.hpp:19-68) with its tables resident on the device."""

    def __init__(self, ctx: Context, head_dim: int, base: float, max_position: int):
        self.ctx = ctx
        h = vp()
        ctx.check(ctx.lib.reattn_rope_create(ctx.h, head_dim, base, max_position, C.byref(h)))
        self.h = h
        self.head_dim, self.base, self.max_position = head_dim, base, max_position

    def rotate(self, rows, positions) -> None:
        import numpy as np
        pos = np.ascontiguousarray(np.asarray(positions, dtype=np.uint64))
        self.ctx.check(self.ctx.lib.reattn_rope_rotate(self.ctx.h, self.h, _ptr(rows),
                                                       pos.ctypes.data, rows.shape[0]))

    def tables(self):
        import numpy as np
        c = np.zeros((self.max_position, self.head_dim // 2), np.float32)
        s = np.zeros_like(c)
        self.ctx.check(self.ctx.lib.reattn_rope_tables_host(self.h, c.ctypes.data, s.ctypes.data))
        return c, s

    def __del__(self):
        # dependents keep their Context alive; skip if it was closed explicitly
        if getattr(self, "h", None) and self.ctx.h:
            self.ctx.lib.reattn_rope_destroy(self.h)
            self.h = None


class Cache:
    """Device SegmentedKvCache (kv_cache.hpp:38-118): head-major [n_kv][capacity][d]."""

    def __init__(self, ctx: Context, n_kv: int, d: int, l_global: int, l_local_max: int,
                 capacity: int, dtype: int = BF16):
        self.ctx = ctx
        h = vp()
        ctx.check(ctx.lib.reattn_cache_create(ctx.h, n_kv, d, l_global, l_local_max, capacity,
                                              dtype, C.byref(h)))
        self.h = h
        self.n_kv, self.d, self.l_global, self.l_local_max = n_kv, d, l_global, l_local_max
        self.capacity, self.dtype = capacity, dtype

    @classmethod
    def _adopt(cls, ctx: Context, h) -> "Cache":
        self = cls.__new__(cls)
        self.ctx, self.h = ctx, h
        i = self.info()
        self.n_kv, self.d, self.l_global, self.l_local_max = i["n_kv"], i["d"], i["l_global"], i["l_local_max"]
        self.capacity, self.dtype = i["capacity"], i["dtype"]
        return self

    def append(self, keys, values) -> None:
        """keys/values: torch [rows, n_kv*d] fp32 (device) or numpy fp32 (host)."""
        on_dev = hasattr(keys, "data_ptr")
        kp = keys.data_ptr() if on_dev else keys.ctypes.data
        vpp = values.data_ptr() if on_dev else values.ctypes.data
        self.ctx.check(self.ctx.lib.reattn_cache_append(self.ctx.h, self.h, kp, vpp,
                                                        keys.shape[0], int(on_dev)))

    def set_total(self, total: int) -> None:
        self.ctx.check(self.ctx.lib.reattn_cache_set_total(self.ctx.h, self.h, total))

    def info(self) -> dict:
        vals = [u64() for _ in range(8)]
        dt = C.c_int()
        self.ctx.lib.reattn_cache_info(self.h, *[C.byref(v) for v in vals], C.byref(dt))
        keys = ["n_kv", "d", "l_global", "l_local_max", "capacity", "total", "global_end",
                "local_start"]
        out = {k: v.value for k, v in zip(keys, vals)}
        out["dtype"] = dt.value
        return out

    def keys_tensor(self):
        return self._view(self.ctx.lib.reattn_cache_keys(self.h))

    def values_tensor(self):
        return self._view(self.ctx.lib.reattn_cache_values(self.h))

    def _view(self, ptr):
        import torch
        dt = torch.bfloat16 if self.dtype == BF16 else torch.float32
        n = self.n_kv * self.capacity * self.d
        return _wrap_device(ptr, n, dt, self.ctx.device).view(self.n_kv, self.capacity, self.d)

    def __del__(self):
        # dependents keep their Context alive; skip if it was closed explicitly
        if getattr(self, "h", None) and self.ctx.h:
            self.ctx.lib.reattn_cache_destroy(self.h)
            self.h = None


def _wrap_device(ptr: int, numel: int, dtype, device: int):
    """Zero-copy torch view of library-owned device memory (via __cuda_array_interface__)."""
    import torch

    class _CAI:
        pass

    typestr = {torch.float32: "<f4", torch.bfloat16: "<V2", torch.float64: "<f8",
               torch.int32: "<i4"}[dtype]
    holder = _CAI()
    holder.__cuda_array_interface__ = {"shape": (numel,), "typestr": typestr if dtype != torch.bfloat16 else "<i2",
                                       "data": (ptr, False), "version": 3}
    t = torch.as_tensor(holder, device=f"cuda:{device}")
    if dtype == torch.bfloat16:
        t = t.view(torch.bfloat16)
    return t


@dataclass
class StepResult:
    out: object
    stats: StepStats
    spans: tuple
    entropy: object


def attend_step(ctx: Context, cache: Cache, rope: Rope, q, n_head: int, cfg: SelectionConfig,
                mode: int = MODE_REATTENTION, out=None) -> StepResult:
    """engine.hpp:43 attend_step on device tensors.  q: [n_q, n_head*d] fp32 (cuda)."""
    import numpy as np
    import torch
    n_q = q.shape[0]
    if out is None:
        out = torch.empty_like(q)
    st = StepStats()
    kp = max(1, cfg.k_prime)
    sb = np.zeros(kp, np.uint64)
    se = np.zeros(kp, np.uint64)
    ent = np.zeros(max(1, n_q * n_head), np.float64)
    ctx.check(ctx.lib.reattn_attend_step(ctx.h, cache.h, rope.h, _ptr(q), n_q, n_head,
                                         C.byref(cfg), mode, _ptr(out), C.byref(st),
                                         sb.ctypes.data, se.ctypes.data, ent.ctypes.data))
    n = st.n_spans
    return StepResult(out, st, (sb[:n].copy(), se[:n].copy()), ent[: n_q * n_head].reshape(n_q, n_head))


def debug_trace(n: int = 4096):
    """Device timeline stamps (REATTN_TRACE=1 at plan build; layout in csrc/misc.cu)."""
    lib = load_library()
    buf = (u64 * n)()
    rc = lib.reattn_debug_trace(buf, n)
    if rc:
        raise ReattnError(f"reattn_debug_trace: status {rc} (REATTN_TRACE unset?)")
    return list(buf)


class Plan:
    """One attend_step shape captured as a CUDA graph (reattn_plan_*)."""

    def __init__(self, ctx: Context, cache: Cache, rope: Rope, n_q: int, n_head: int,
                 cfg: SelectionConfig, mode: int = MODE_REATTENTION):
        self.ctx, self.cache, self.rope = ctx, cache, rope
        h = vp()
        ctx.check(ctx.lib.reattn_plan_create(ctx.h, cache.h, rope.h, n_q, n_head, C.byref(cfg),
                                             mode, C.byref(h)))
        self.h = h
        self.n_q, self.n_head = n_q, n_head
        numel = n_q * n_head * cache.d
        import torch
        self.q = _wrap_device(ctx.lib.reattn_plan_q(h), numel, torch.float32, ctx.device).view(n_q, -1)
        self.out = _wrap_device(ctx.lib.reattn_plan_out(h), numel, torch.float32, ctx.device).view(n_q, -1)

    def launch(self) -> None:
        self.ctx.check(self.ctx.lib.reattn_plan_launch(self.h))

    def set_append(self, enable: bool = True) -> None:
        """Append mode: each launch first appends the step's K/V rows (self.k_in / self.v_in,
        [n_kv * d] fp32 in DenseMatrix layout) to the cache, then runs the step."""
        import torch
        self.ctx.check(self.ctx.lib.reattn_plan_set_append(self.h, int(enable)))
        n = self.cache.n_kv * self.cache.d
        self.k_in = _wrap_device(self.ctx.lib.reattn_plan_k_in(self.h), n, torch.float32, self.ctx.device)
        self.v_in = _wrap_device(self.ctx.lib.reattn_plan_v_in(self.h), n, torch.float32, self.ctx.device)

    def step_host(self, q_host, k_host, v_host, out_host) -> None:
        self.ctx.check(self.ctx.lib.reattn_plan_step_host(self.h, _ptr(q_host), _ptr(k_host),
                                                          _ptr(v_host), _ptr(out_host)))

    def launch_scan(self) -> None:
        self.ctx.check(self.ctx.lib.reattn_plan_launch_scan(self.h))

    def run_host(self, q_host, out_host) -> None:
        self.ctx.check(self.ctx.lib.reattn_plan_run_host(self.h, _ptr(q_host), _ptr(out_host)))

    def stats(self) -> StepStats:
        st = StepStats()
        self.ctx.check(self.ctx.lib.reattn_plan_stats(self.h, C.byref(st)))
        return st

    def result(self, k_prime: int, staged: bool = False) -> "StepResult":
        """The last replay's attend_step outputs: out (device tensor), stats, spans and the
        row entropies [n_q, n_head] (reattn_plan_result; staged=True: the copies enqueued by
        stage_result, read after the caller synchronised -- reattn_plan_staged_result)."""
        import numpy as np
        st = StepStats()
        sb = np.zeros(max(1, k_prime), np.uint64)
        se = np.zeros(max(1, k_prime), np.uint64)
        ent = np.zeros(max(1, self.n_q * self.n_head), np.float64)
        fn = self.ctx.lib.reattn_plan_staged_result if staged else self.ctx.lib.reattn_plan_result
        self.ctx.check(fn(self.h, C.byref(st), sb.ctypes.data, se.ctypes.data, ent.ctypes.data))
        n = st.n_spans
        return StepResult(self.out, st, (sb[:n].copy(), se[:n].copy()),
                          ent[: self.n_q * self.n_head].reshape(self.n_q, self.n_head))

    def stage_result(self) -> None:
        self.ctx.check(self.ctx.lib.reattn_plan_stage_result(self.h))

    def info(self) -> dict:
        a, b, c = u64(), u64(), u64()
        self.ctx.check(self.ctx.lib.reattn_plan_info(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return {"kernels_per_step": a.value, "scan_bytes": b.value, "scope_bytes_upper": c.value}

    def __del__(self):
        # dependents keep their Context alive; skip if it was closed explicitly
        if getattr(self, "h", None) and self.ctx.h:
            self.ctx.lib.reattn_plan_destroy(self.h)
            self.h = None


class BatchPlan:
    """Batched decode: one CUDA graph over n_seq sequences, each with its own cache
    (reattn_batch_plan_*).  q / out: [n_seq, n_head*d] fp32 device tensors."""

    def __init__(self, ctx: Context, caches, rope: Rope, n_head: int, cfg: SelectionConfig,
                 mode: int = MODE_REATTENTION):
        import torch
        self.ctx, self.caches, self.rope = ctx, list(caches), rope
        arr = (vp * len(self.caches))(*[c.h for c in self.caches])
        h = vp()
        ctx.check(ctx.lib.reattn_batch_plan_create(ctx.h, arr, len(self.caches), rope.h, n_head,
                                                   C.byref(cfg), mode, C.byref(h)))
        self.h = h
        n, d = len(self.caches), self.caches[0].d
        numel = n * n_head * d
        self.q = _wrap_device(ctx.lib.reattn_batch_plan_q(h), numel, torch.float32,
                              ctx.device).view(n, -1)
        self.out = _wrap_device(ctx.lib.reattn_batch_plan_out(h), numel, torch.float32,
                                ctx.device).view(n, -1)

    def launch(self) -> None:
        self.ctx.check(self.ctx.lib.reattn_batch_plan_launch(self.h))

    def run_host(self, q_host, out_host) -> None:
        self.ctx.check(self.ctx.lib.reattn_batch_plan_run_host(self.h, _ptr(q_host), _ptr(out_host)))

    def stats(self, seq: int) -> StepStats:
        st = StepStats()
        self.ctx.check(self.ctx.lib.reattn_batch_plan_stats(self.h, seq, C.byref(st)))
        return st

    def info(self) -> dict:
        a, b, c = u64(), u64(), C.c_int()
        self.ctx.check(self.ctx.lib.reattn_batch_plan_info(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return {"kernels_per_step": a.value, "scan_bytes": b.value, "side_sms": c.value}

    def __del__(self):
        if getattr(self, "h", None) and self.ctx.h:
            self.ctx.lib.reattn_batch_plan_destroy(self.h)
            self.h = None


class Weights:
    """reattn::ModelWeights (model.hpp:66-84) resident on the device (fp32)."""

    def __init__(self, ctx: Context, h):
        self.ctx, self.h = ctx, h
        cfg = ModelConfig()
        ctx.check(ctx.lib.reattn_weights_config(h, C.byref(cfg)))
        self.config = cfg

    @classmethod
    def init_random(cls, ctx: Context, cfg: ModelConfig, seed: int) -> "Weights":
        """init_random (model.hpp:120-152): the reference's pinned Gaussian stream."""
        h = vp()
        ctx.check(ctx.lib.reattn_weights_init_random(ctx.h, C.byref(cfg), seed, C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def synth(cls, ctx: Context, cfg: ModelConfig, seed: int) -> "Weights":
        """Benchmarking weights filled on the device (reattn_weights_synth)."""
        h = vp()
        ctx.check(ctx.lib.reattn_weights_synth(ctx.h, C.byref(cfg), seed, C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def zeros(cls, ctx: Context, cfg: ModelConfig) -> "Weights":
        h = vp()
        ctx.check(ctx.lib.reattn_weights_create(ctx.h, C.byref(cfg), C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def load(cls, ctx: Context, path: str) -> "Weights":
        """load_weights (model.hpp:292-339), RATW file."""
        h = vp()
        ctx.check(ctx.lib.reattn_weights_load(ctx.h, os.fsencode(path), C.byref(h)))
        return cls(ctx, h)

    def save(self, path: str) -> None:
        self.ctx.check(self.ctx.lib.reattn_weights_save(self.ctx.h, self.h, os.fsencode(path)))

    def shape(self, kind: int):
        r, c = u64(), u64()
        self.ctx.check(self.ctx.lib.reattn_weights_shape(self.h, kind, C.byref(r), C.byref(c)))
        return r.value, c.value

    def tensor(self, kind: int, layer: int = 0):
        import numpy as np
        r, c = self.shape(kind)
        out = np.zeros((r, c), np.float32)
        self.ctx.check(self.ctx.lib.reattn_weights_download(self.ctx.h, self.h, kind, layer,
                                                            out.ctypes.data, out.size))
        return out

    def set_tensor(self, kind: int, layer: int, values) -> None:
        import numpy as np
        v = np.ascontiguousarray(values, dtype=np.float32)
        self.ctx.check(self.ctx.lib.reattn_weights_upload(self.ctx.h, self.h, kind, layer,
                                                          v.ctypes.data, v.size))

    def __del__(self):
        if getattr(self, "h", None) and self.ctx.h:
            self.ctx.lib.reattn_weights_destroy(self.h)
            self.h = None


class Engine:
    """reattn::Engine (engine.hpp:119-216) on the device: per-layer caches, chunked
    prefill, greedy decode.  `weights` must outlive the engine (held here)."""

    def __init__(self, ctx: Context, weights: Weights, sel: SelectionConfig,
                 mode: int = MODE_REATTENTION, cache_dtype: int = F32):
        self.ctx, self.weights, self.sel = ctx, weights, sel
        h = vp()
        ctx.check(ctx.lib.reattn_engine_create(ctx.h, weights.h, C.byref(sel), mode, cache_dtype,
                                               C.byref(h)))
        self.h = h
        self.config = weights.config

    def reset(self) -> None:
        self.ctx.check(self.ctx.lib.reattn_engine_reset(self.h))

    def synth_context(self, total: int, seed: int = 1) -> None:
        """Benchmarking: every layer's cache holds `total` synthetic rows."""
        self.ctx.check(self.ctx.lib.reattn_engine_synth_context(self.h, total, seed))

    def prefill(self, tokens):
        """Returns the final chunk's hidden states (rows x d_model, numpy)."""
        import numpy as np
        t = np.ascontiguousarray(np.asarray(tokens, dtype=np.uint32))
        rows = u64()
        self.ctx.check(self.ctx.lib.reattn_engine_prefill(self.h, t.ctypes.data if t.size else None,
                                                          t.size, C.byref(rows)))
        out = np.zeros((rows.value, self.config.d_model), np.float32)
        self.ctx.check(self.ctx.lib.reattn_engine_hidden(self.h, out.ctypes.data, out.size))
        return out

    def logits(self, hidden):
        import numpy as np
        hid = np.ascontiguousarray(hidden, dtype=np.float32)
        out = np.zeros((hid.shape[0], self.config.vocab_size), np.float32)
        self.ctx.check(self.ctx.lib.reattn_engine_logits(self.h, hid.ctypes.data, hid.shape[0],
                                                         out.ctypes.data))
        return out

    def decode_step(self, last_token: int) -> int:
        nt = C.c_uint32()
        self.ctx.check(self.ctx.lib.reattn_engine_decode_step(self.h, last_token, C.byref(nt)))
        return nt.value

    def last_logits(self):
        import numpy as np
        out = np.zeros(self.config.vocab_size, np.float32)
        self.ctx.check(self.ctx.lib.reattn_engine_last_logits(self.h, out.ctypes.data, out.size))
        return out

    def stats(self) -> RunStats:
        st = RunStats()
        self.ctx.check(self.ctx.lib.reattn_engine_stats(self.h, C.byref(st)))
        return st

    def decode_latencies(self):
        import numpy as np
        n = u64()
        self.ctx.lib.reattn_engine_decode_latencies(self.h, None, 0, C.byref(n))
        out = np.zeros(n.value, np.float64)
        self.ctx.lib.reattn_engine_decode_latencies(self.h, out.ctypes.data, n.value, C.byref(n))
        return out

    def last_spans(self, layer: int):
        import numpy as np
        n = u64()
        self.ctx.check(self.ctx.lib.reattn_engine_last_spans(self.h, layer, None, None, 0, C.byref(n)))
        b = np.zeros(n.value, np.uint64)
        e = np.zeros(n.value, np.uint64)
        self.ctx.check(self.ctx.lib.reattn_engine_last_spans(self.h, layer, b.ctypes.data,
                                                             e.ctypes.data, n.value, C.byref(n)))
        return list(zip(b.tolist(), e.tolist()))

    def __del__(self):
        if getattr(self, "h", None) and self.ctx.h:
            self.ctx.lib.reattn_engine_destroy(self.h)
            self.h = None
