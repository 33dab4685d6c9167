"""Sequence-sharded ReAttention decode over several GPUs.

The middle segment of the KV cache (kv_cache.hpp:65-67) is split into `world` contiguous
ranges whose boundaries are multiples of span_m, so an aligned span never straddles
ranks; the global and local blocks are replicated.  One decode step per rank:

    scan      K1 on the rank's shard            -> per (kv head) top-k, shard-local indices
    gather 1  all_gather of (index, score)      (n_kv * k * 8 B per rank: 128 B at decode)
    select    merge (exact: top-k of the union under (score desc, index asc) is the global
              top-k), vote, spans, global scope — redundantly and identically on every
              rank — then map scope rows to this rank's rows (others masked)
    attend    f64 partial softmax states over the rows this rank owns
    gather 2  all_gather of the partial states
    combine   fixed-order merge -> the full output on every rank

Two hosts of the same protocol:
  * NcclDecodeStep (the product path): the library owns an NCCL communicator
    (reattn_comm_*) and issues both all-gathers itself -- reattn_shard_step /
    reattn_shard_capture, exactly what a C++ host calls (include/reattn/sharded.hpp);
    torch.distributed only ships the 128-byte NCCL id from rank 0 and times the run.
  * ShardedDecodeStep: the collectives through torch.distributed; `ops` is pluggable so
    the identical protocol code runs under gloo on CPU in the tests
    (tests/test_sharded_cpu.py).
"""
from __future__ import annotations

import ctypes as C

from . import native as N


def shard_range(middle_len: int, span_m: int, world: int, rank: int) -> tuple[int, int]:
    """Rank's [begin, begin+len) of the middle: floor(r*M/world/m)*m boundaries (the rule
    implemented by reattn_shard_range)."""
    b = [((r * middle_len) // world) // span_m * span_m for r in range(world)] + [middle_len]
    for r in range(world - 1, -1, -1):
        b[r] = min(b[r], b[r + 1])
    return b[rank], b[rank + 1] - b[rank]


def global_geometry(total: int, l_global: int, l_local: int) -> tuple[int, int]:
    """(global_end, local_start) of a cache with `total` rows (kv_cache.hpp:65-67)."""
    g = min(total, l_global)
    return g, total - min(total - g, l_local)


def local_row_segments(total: int, cfg: N.SelectionConfig, world: int, rank: int):
    """Global cache row ranges that make up rank's local cache: [global | shard | local]."""
    g, ls = global_geometry(total, cfg.l_global, cfg.l_local)
    b, n = shard_range(ls - g, cfg.span_m, world, rank)
    return [(0, g), (g + b, g + b + n), (ls, total)]


class NativeOps:
    """Device stages through the C-ABI (reattn_shard_*)."""

    def __init__(self, ctx: N.Context, local_cache: N.Cache, rope: N.Rope, n_head: int,
                 cfg: N.SelectionConfig, global_total: int, world: int, rank: int):
        import torch
        self.ctx, self.lib = ctx, ctx.lib
        h = N.vp()
        ctx.check(self.lib.reattn_shard_plan_create(ctx.h, local_cache.h, rope.h, n_head,
                                                    C.byref(cfg), global_total, world, rank,
                                                    C.byref(h)))
        self.h = h
        self._keep = (local_cache, rope)
        dev = ctx.device
        cs, cr, ps, pr = N.vp(), N.vp(), N.vp(), N.vp()
        cb, pb = N.u64(), N.u64()
        self.lib.reattn_shard_buffers(h, C.byref(cs), C.byref(cr), C.byref(cb), C.byref(ps),
                                      C.byref(pr), C.byref(pb))
        u8 = torch.uint8
        self.cand_send = N._wrap_device(cs.value, cb.value // 4, torch.int32, dev).view(u8)
        self.cand_recv = N._wrap_device(cr.value, cb.value * world // 4, torch.int32, dev).view(u8)
        self.part_send = N._wrap_device(ps.value, pb.value // 8, torch.float64, dev).view(u8)
        self.part_recv = N._wrap_device(pr.value, pb.value * world // 8, torch.float64, dev).view(u8)
        d = local_cache.d
        self.q = N._wrap_device(self.lib.reattn_shard_plan_q(h), n_head * d, torch.float32, dev).view(1, -1)
        self.out = N._wrap_device(self.lib.reattn_shard_plan_out(h), n_head * d, torch.float32, dev).view(1, -1)

    def scan(self):
        self.ctx.check(self.lib.reattn_shard_scan(self.h))

    def select(self):
        self.ctx.check(self.lib.reattn_shard_select(self.h))

    def attend(self):
        self.ctx.check(self.lib.reattn_shard_attend(self.h))

    def combine(self):
        self.ctx.check(self.lib.reattn_shard_combine(self.h))

    def stats(self, k_prime: int):
        import numpy as np
        st = N.StepStats()
        sb = np.zeros(max(1, k_prime), np.uint64)
        se = np.zeros(max(1, k_prime), np.uint64)
        self.ctx.check(self.lib.reattn_shard_stats(self.h, C.byref(st), sb.ctypes.data,
                                                   se.ctypes.data))
        return st, (sb[:st.n_spans].copy(), se[:st.n_spans].copy())

    def __del__(self):
        if getattr(self, "h", None) and self.ctx.h:
            self.lib.reattn_shard_plan_destroy(self.h)
            self.h = None


class ShardedDecodeStep:
    """One rank's sequence-sharded decode step.  All ranks call step() collectively.

    capture() records the whole step -- K scan, candidate all-gather (NCCL), merge + vote +
    spans + scope, attention over this rank's scope rows, partial-state all-gather (NCCL),
    combine -- as ONE CUDA graph on the context stream (NCCL collectives are captured like
    kernels), so a step costs one graph launch instead of six host launches."""

    def __init__(self, ops, group=None):
        self.ops = ops
        self.group = group
        self.graph = None

    def _body(self):
        import torch.distributed as dist
        o = self.ops
        o.scan()
        dist.all_gather_into_tensor(o.cand_recv, o.cand_send, group=self.group)
        o.select()
        o.attend()
        dist.all_gather_into_tensor(o.part_recv, o.part_send, group=self.group)
        o.combine()

    def step(self, q):
        o = self.ops
        o.q.copy_(q)
        if self.graph is not None:
            self.graph.replay()
        else:
            self._body()
        return o.out

    def capture(self):
        """Capture the step for the query buffer ops.q (call collectively on every rank, on
        the stream the context launches on)."""
        import torch
        s = torch.cuda.current_stream()
        self._body()  # warm-up outside capture: communicator and kernel attribute set-up
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            self._body()
        torch.cuda.synchronize()
        self.graph = g
        return self


class NcclComm:
    """The library's own NCCL communicator (reattn_comm_*).  Rank 0's unique id is shipped to
    the other ranks through torch.distributed (plumbing only: 128 bytes, once)."""

    def __init__(self, ctx: N.Context, world: int, rank: int, group=None):
        import torch
        import torch.distributed as dist
        self.ctx, self.lib = ctx, ctx.lib
        idb = (C.c_uint8 * 128)()
        if rank == 0:
            ctx.check(self.lib.reattn_comm_unique_id(idb))
        if world > 1:
            t = torch.tensor(list(idb), dtype=torch.uint8,
                             device=f"cuda:{ctx.device}" if dist.get_backend(group) == "nccl" else "cpu")
            dist.broadcast(t, src=0, group=group)
            for i, v in enumerate(t.cpu().tolist()):
                idb[i] = v
        h = N.vp()
        ctx.check(self.lib.reattn_comm_create(ctx.h, world, rank, idb, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.reattn_comm_destroy(self.h)
            self.h = None


class NcclDecodeStep:
    """One rank's sharded decode step with the collectives issued by the library
    (reattn_shard_step): the C-ABI host path.  capture() records the step, both NCCL
    all-gathers included, as one CUDA graph (reattn_shard_capture; collective)."""

    def __init__(self, ops: NativeOps, comm: NcclComm):
        self.ops, self.comm = ops, comm
        self.captured = False

    def step(self, q=None):
        o = self.ops
        if q is not None:
            o.q.copy_(q)
        o.ctx.check(o.lib.reattn_shard_step(o.h, self.comm.h))
        return o.out

    def capture(self):
        o = self.ops
        o.ctx.check(o.lib.reattn_shard_capture(o.h, self.comm.h))
        self.captured = True
        return self

    def run_host(self, q_host, out_host):
        o = self.ops
        o.ctx.check(o.lib.reattn_shard_run_host(o.h, self.comm.h, N._ptr(q_host), N._ptr(out_host)))
