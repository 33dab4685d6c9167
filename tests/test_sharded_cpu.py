"""CPU, world size 2 over gloo: the product's sharded-decode protocol
(paper_2407_15176_b200/sharded.py: shard ranges, local cache layout, the two all-gathers,
buffer layouts) driven with oracle-backed stages, checked against the unsharded oracle
attend_step.  The device stages themselves are covered by tests/test_sharded_gpu.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_bind as ob
import synth
from paper_2407_15176_b200 import native as N
from paper_2407_15176_b200 import sharded as S

NO = 0xFFFFFFFF


class OracleOps:
    """Stage semantics of reattn_shard_* restated on the CPU with the test oracle."""

    def __init__(self, K, V, total, cfg, n_head, world, rank, base, window):
        self.cfg, self.world, self.rank, self.n_head = cfg, world, rank, n_head
        self.n_kv, _, self.d = K.shape
        self.total, self.base, self.window = total, base, window
        self.g, self.ls = S.global_geometry(total, cfg.l_global, cfg.l_local)
        self.M = self.ls - self.g
        segs = S.local_row_segments(total, cfg, world, rank)
        self.local_K = np.concatenate([K[:, b:e] for b, e in segs], axis=1)
        self.local_V = np.concatenate([V[:, b:e] for b, e in segs], axis=1)
        self.begin, self.slen = S.shard_range(self.M, cfg.span_m, world, rank)
        k = cfg.k
        self.cb = ((self.n_kv * k * 8 + 255) // 256) * 256
        self.cand_send = torch.zeros(self.cb, dtype=torch.uint8)
        self.cand_recv = torch.zeros(self.cb * world, dtype=torch.uint8)
        self.pb = n_head * (4 + self.d) * 8
        self.part_send = torch.zeros(self.pb, dtype=torch.uint8)
        self.part_recv = torch.zeros(self.pb * world, dtype=torch.uint8)
        self.q = torch.zeros(1, n_head * self.d)
        self.out = torch.zeros(1, n_head * self.d)
        self.cos, self.sin = ob.rope_table(self.d, base, window)

    def scan(self):
        k, n = self.cfg.k, self.n_kv * self.cfg.k
        idx = np.full(n, NO, np.uint32)
        sc = np.zeros(n, np.float32)
        if self.slen:
            heads = [np.ascontiguousarray(self.local_K[h, self.g:self.g + self.slen])
                     for h in range(self.n_kv)]
            i, s = ob.topk(self.q.numpy(), self.n_head, heads, k)
            for h in range(self.n_kv):
                idx[h * k:h * k + i.shape[2]] = i[h, 0]
                sc[h * k:h * k + i.shape[2]] = s[h, 0]
        buf = np.zeros(self.cb, np.uint8)
        buf[:n * 4] = idx.view(np.uint8)
        buf[n * 4:n * 8] = sc.view(np.uint8)
        self.cand_send.copy_(torch.from_numpy(buf))

    def select(self):
        k, n = self.cfg.k, self.n_kv * self.cfg.k
        kk = min(k, self.M)
        recv = self.cand_recv.numpy()
        merged_i, merged_s = [], []
        for h in range(self.n_kv):
            cands = []
            for r in range(self.world):
                blk = recv[r * self.cb:(r + 1) * self.cb]
                idx = blk[:n * 4].view(np.uint32)[h * k:(h + 1) * k]
                sc = blk[n * 4:n * 8].view(np.float32)[h * k:(h + 1) * k]
                off = S.shard_range(self.M, self.cfg.span_m, self.world, r)[0]
                cands += [(-float(s), int(i) + off) for i, s in zip(idx, sc) if i != NO]
            cands.sort()
            for s, i in cands[:kk]:
                merged_i.append(i)
                merged_s.append(-s)
        w = ob.vote(np.array(merged_i, np.uint64), np.array(merged_s, np.float32), self.cfg.k_prime)
        b, e = ob.expand_spans(w, self.cfg.span_m, self.M, self.cfg.span_mode)
        src = np.zeros(self.window + 1, np.uint64)
        L = ob.sz(0)
        ob.oracle().oracle_scope_indices(self.total, self.cfg.l_global, self.cfg.l_local,
                                         b if len(b) else np.zeros(1, np.uint64),
                                         e if len(e) else np.zeros(1, np.uint64), len(b),
                                         self.window, src, ob.C.byref(L))
        self.L = L.value
        self.local_src = []
        for s in src[:self.L]:
            s = int(s)
            if s < self.g:
                self.local_src.append(s if self.rank == 0 else None)
            elif s >= self.ls:
                self.local_src.append(self.g + self.slen + s - self.ls if self.rank == 0 else None)
            else:
                m = s - self.g
                own = self.begin <= m < self.begin + self.slen
                self.local_src.append(self.g + m - self.begin if own else None)

    def attend(self):
        d, L, G = self.d, self.L, self.n_head // self.n_kv
        half = d // 2
        part = np.zeros((self.n_head, 4 + d), np.float64)
        for h in range(self.n_head):
            kv = h // G
            q = self.q.numpy()[0, h * d:(h + 1) * d].copy()
            ob.oracle().oracle_rotate_row(q, d, self.cos[L - 1].copy(), self.sin[L - 1].copy())
            m, A, B, acc = -np.inf, 0.0, 0.0, np.zeros(d)
            ls, vs = [], []
            for r, row in enumerate(self.local_src):
                if row is None:
                    continue
                kr = self.local_K[kv, row].copy()
                ob.oracle().oracle_rotate_row(kr, d, self.cos[r].copy(), self.sin[r].copy())
                ls.append(ob.oracle().oracle_dot_f64(q, kr, d) / np.sqrt(d))
                vs.append(self.local_V[kv, row].astype(np.float64))
            if ls:
                ls = np.array(ls)
                m = ls.max()
                w = np.exp(ls - m)
                A, B = w.sum(), ((ls - m) * w).sum()
                acc = (w[:, None] * np.array(vs)).sum(0)
            part[h, :4] = (m, A, B, 0.0)
            part[h, 4:] = acc
        self.part_send.copy_(torch.from_numpy(part.view(np.uint8).ravel()))

    def combine(self):
        d = self.d
        parts = self.part_recv.numpy().view(np.float64).reshape(self.world, self.n_head, 4 + d)
        out = np.zeros(self.n_head * d, np.float32)
        self.entropy = np.zeros(self.n_head)
        for h in range(self.n_head):
            p = parts[:, h]
            live = p[:, 1] > 0
            M = p[live, 0].max()
            w = np.where(live, np.exp(np.where(live, p[:, 0] - M, 0.0)), 0.0)
            A = (p[live, 1] * w[live]).sum()
            B = (w[live] * (p[live, 2] + (p[live, 0] - M) * p[live, 1])).sum()
            out[h * d:(h + 1) * d] = ((w[:, None] * p[:, 4:]).sum(0) / A).astype(np.float32)
            self.entropy[h] = max(0.0, np.log(A) - B / A)
        self.out.copy_(torch.from_numpy(out).view(1, -1))


def _worker(rank, world, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = N.SelectionConfig(k=4, k_prime=16, span_m=16, l_global=16, l_local=256)
        n_kv, nh, d, total = 2, 4, 16, 3000
        K = synth.uniform(11, n_kv * total * d).reshape(n_kv, total, d)
        V = synth.uniform(12, n_kv * total * d).reshape(n_kv, total, d)
        ops = OracleOps(K, V, total, cfg, nh, world, rank, 10000.0, 2048)
        step = S.ShardedDecodeStep(ops)
        outs = []
        for s in range(2):
            q = torch.from_numpy(synth.uniform(40 + s, nh * d).reshape(1, -1))
            outs.append((step.step(q).numpy().copy(), ops.L, ops.entropy.max()))
        result_q.put((rank, outs))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2])
def test_sharded_protocol_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # unsharded oracle
    cfg = ob.SelectionConfig(k=4, k_prime=16, span_m=16, l_global=16, l_local=256)
    n_kv, nh, d, total = 2, 4, 16, 3000
    K = synth.uniform(11, n_kv * total * d).reshape(n_kv, total, d)
    V = synth.uniform(12, n_kv * total * d).reshape(n_kv, total, d)
    for s in range(2):
        qv = synth.uniform(40 + s, nh * d).reshape(1, -1)
        want, st, _ = ob.attend_step(qv, nh, K, V, total, cfg, 10000.0, 2048)
        for r in range(world):
            out, L, emax = res[r][s]
            assert L == st.scope_len
            assert np.abs(out - want).max() <= 1e-6, (r, s, np.abs(out - want).max())
            assert abs(emax - st.entropy_max) <= 1e-9


def test_shard_ranges_cover_and_align():
    for M in (0, 5, 100, 1044448, 4190176):
        for world in (1, 2, 4, 8):
            prev = 0
            for r in range(world):
                b, n = S.shard_range(M, 32, world, r)
                assert b == prev and (b % 32 == 0 or b == M)
                prev = b + n
            assert prev == M
