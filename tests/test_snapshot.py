"""RKVC cache snapshots (reference kv_cache.hpp:120-209) to and from device caches.

Files written by the reference's own write_cache_snapshot (oracle/_ref) are read by
reattn_snapshot_*; files written by reattn_snapshot_write are read back by the reference's
read_cache_snapshot.  Corrupt files must fail the same way (exception kind and message,
kv_cache.hpp:168-209 read order)."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle_bind as ob
import synth

from paper_2407_15176_b200 import native as N

ref = ob.ref()
needs_ref = pytest.mark.skipif(ref is None, reason="oracle/_ref not built")


def make_layers(seed, geoms, d=8, n_kv=2):
    """[(total, l_global, l_local)] -> list of (keys, values) head-major fp32 + geometry."""
    out = []
    for i, (total, g, loc) in enumerate(geoms):
        k = synth.uniform(seed + 2 * i, n_kv * total * d).reshape(n_kv, total, d)
        v = synth.uniform(seed + 2 * i + 1, n_kv * total * d).reshape(n_kv, total, d)
        out.append((k, v, total, g, loc))
    return out


def ref_write(path, layers, d=8, n_kv=2):
    caches = []
    for k, v, total, g, loc in layers:
        h = ref.ref_cache_create(n_kv, d, g, loc, np.ascontiguousarray(k).ravel(),
                                 np.ascontiguousarray(v).ravel(), total)
        assert h, ref.ref_last_error()
        caches.append(h)
    arr = (C.c_void_p * len(caches))(*caches)
    rc = ref.ref_snapshot_write(os.fsencode(path), arr, len(caches))
    for h in caches:
        ref.ref_cache_destroy(h)
    assert rc == 0, ref.ref_last_error()


def ref_read(path, layer=0, cap=0):
    n = C.c_size_t()
    info = np.zeros(5, np.uint64)
    keys = np.zeros(max(cap, 1), np.float32)
    vals = np.zeros(max(cap, 1), np.float32)
    rc = ref.ref_snapshot_read(os.fsencode(path), layer, C.byref(n), info, keys, vals, cap)
    msg = ref.ref_last_error().decode() if rc else ""
    return rc, msg, n.value, info, keys, vals


def our_open(lib, path):
    h = C.c_void_p()
    rc = lib.reattn_snapshot_open(None, os.fsencode(path), C.byref(h))
    return rc, h


GEOMS = [(50, 4, 16), (0, 4, 16), (7, 32, 64), (33, 0, 1)]


@needs_ref
def test_snapshot_header_parse_cpu(tmp_path):
    """No GPU: our parser reads the reference's files (layer geometry, per-layer offsets)."""
    lib = N.load_library()
    path = str(tmp_path / "ref.rkvc")
    layers = make_layers(10, GEOMS)
    ref_write(path, layers)
    rc, h = our_open(lib, path)
    assert rc == N.OK
    a, b, c = C.c_uint32(), C.c_uint32(), C.c_uint32()
    lib.reattn_snapshot_info(h, C.byref(a), C.byref(b), C.byref(c))
    assert (a.value, b.value, c.value) == (len(GEOMS), 2, 8)
    for i, (total, g, loc) in enumerate(GEOMS):
        t, gg, ll = C.c_uint64(), C.c_uint64(), C.c_uint64()
        assert lib.reattn_snapshot_layer_info(h, i, C.byref(t), C.byref(gg), C.byref(ll)) == N.OK
        assert (t.value, gg.value, ll.value) == (total, g, loc)
    assert lib.reattn_snapshot_layer_info(h, len(GEOMS), None, None, None) == N.ERANGE
    lib.reattn_snapshot_close(h)


def corruptions(raw):
    """(name, bytes) variants of a valid snapshot exercising every failure in read order."""
    bad_magic = b"RKVX" + raw[4:]
    bad_version = raw[:4] + (2).to_bytes(4, "little") + raw[8:]
    zero_local = bytearray(raw)
    zero_local[20 + 16:20 + 24] = (0).to_bytes(8, "little")  # layer 0 l_local_max
    zero_heads = bytearray(raw)
    zero_heads[12:16] = (0).to_bytes(4, "little")            # n_kv_heads = 0
    return [("bad_magic", bad_magic), ("bad_version", bad_version),
            ("trunc_version", raw[:6]), ("trunc_nlayers", raw[:10]), ("trunc_nkv", raw[:14]),
            ("trunc_d", raw[:18]), ("trunc_total", raw[:24]), ("trunc_lglobal", raw[:32]),
            ("trunc_llocal", raw[:40]), ("trunc_keys", raw[:44 + 100]),
            ("trunc_values", raw[:44 + 2 * 50 * 8 * 4 + 8]), ("zero_local", bytes(zero_local)),
            ("zero_heads", bytes(zero_heads)), ("empty", b"")]


@needs_ref
def test_snapshot_corrupt_files_fail_like_reference_cpu(tmp_path):
    lib = N.load_library()
    good = str(tmp_path / "good.rkvc")
    ref_write(good, make_layers(20, GEOMS[:2]))
    raw = open(good, "rb").read()
    for name, data in corruptions(raw):
        p = str(tmp_path / f"{name}.rkvc")
        open(p, "wb").write(data)
        rc_ref, msg, _, _, _, _ = ref_read(p)
        rc, h = our_open(lib, p)
        assert rc_ref != 0, name
        assert rc == rc_ref, (name, rc, rc_ref, msg)
    rc_ref, _, _, _, _, _ = ref_read(str(tmp_path / "missing.rkvc"))
    assert our_open(lib, str(tmp_path / "missing.rkvc"))[0] == rc_ref == N.ERUNTIME


# ---------------------------------------------------------------------------------------
torch = pytest.importorskip("torch")


@pytest.mark.gpu
@needs_ref
def test_snapshot_messages_match_reference(ctx, tmp_path):
    good = str(tmp_path / "good.rkvc")
    ref_write(good, make_layers(30, GEOMS[:2]))
    raw = open(good, "rb").read()
    for name, data in corruptions(raw) + [("missing", None)]:
        p = str(tmp_path / f"{name}.rkvc")
        if data is not None:
            open(p, "wb").write(data)
        rc_ref, msg, _, _, _, _ = ref_read(p)
        with pytest.raises(N.ReattnError) as ei:
            N.Snapshot(ctx, p)
        assert str(ei.value) == msg, name


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("dtype", [N.F32, N.BF16])
def test_snapshot_reference_file_loads_into_device_caches(ctx, tmp_path, dtype):
    path = str(tmp_path / "ref.rkvc")
    layers = make_layers(40, GEOMS)
    ref_write(path, layers)
    snap = N.Snapshot(ctx, path)
    assert snap.n_layers == len(GEOMS)
    for i, (k, v, total, g, loc) in enumerate(layers):
        cache = snap.load_layer(i, dtype, capacity=total + 5)
        info = cache.info()
        assert (info["total"], info["l_global"], info["l_local_max"]) == (total, g, loc)
        assert info["capacity"] >= total + 5
        if total == 0:
            continue
        kt = cache.keys_tensor()[:, :total].float().cpu().numpy()
        vt = cache.values_tensor()[:, :total].float().cpu().numpy()
        if dtype == N.F32:
            assert np.array_equal(kt, k) and np.array_equal(vt, v)
        else:
            assert np.array_equal(kt, synth.bf16_round(k)) and np.array_equal(vt, synth.bf16_round(v))
    snap.close()


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("dtype", [N.F32, N.BF16])
def test_snapshot_write_read_by_reference(ctx, tmp_path, dtype):
    """reattn_snapshot_write -> the reference's read_cache_snapshot: same rows, bit for bit
    (bf16 caches are widened exactly)."""
    caches, want = [], []
    for i, (total, g, loc) in enumerate([(300, 32, 100), (1, 4, 16), (0, 4, 16)]):
        c = N.Cache(ctx, 2, 8, g, loc, total + 3, dtype)
        k = synth.uniform(50 + i, total * 16).reshape(total, 16)
        v = synth.uniform(60 + i, total * 16).reshape(total, 16)
        if total:
            c.append(k, v)
        caches.append(c)
        kh = k.reshape(total, 2, 8).transpose(1, 0, 2)
        vh = v.reshape(total, 2, 8).transpose(1, 0, 2)
        if dtype == N.BF16:
            kh, vh = synth.bf16_round(kh), synth.bf16_round(vh)
        want.append((kh, vh, total, g, loc))
    path = str(tmp_path / "ours.rkvc")
    N.write_snapshot(ctx, path, caches)
    for li, (kh, vh, total, g, loc) in enumerate(want):
        rc, msg, n, info, keys, vals = ref_read(path, li, cap=2 * 8 * max(total, 1))
        assert rc == 0, msg
        assert n == 3
        assert list(info) == [2, 8, total, g, loc]
        if total:
            assert np.array_equal(keys[:2 * total * 8].reshape(2, total, 8), kh)
            assert np.array_equal(vals[:2 * total * 8].reshape(2, total, 8), vh)
    with pytest.raises(N.InvalidArgument, match="cache snapshot: no layers"):
        N.write_snapshot(ctx, path, [])
    with pytest.raises(N.ReattnError, match="for writing"):
        N.write_snapshot(ctx, str(tmp_path / "no_such_dir" / "x.rkvc"), caches)


@pytest.mark.gpu
@needs_ref
def test_attend_step_on_snapshot_cache(ctx, tmp_path):
    """A cache loaded from a reference snapshot drives attend_step exactly like the same rows
    appended directly (decode geometry, bf16)."""
    cfg = N.SelectionConfig()
    total, d, n_kv = 6000, 128, 8
    k = synth.uniform(70, n_kv * total * d).reshape(n_kv, total, d)
    v = synth.uniform(71, n_kv * total * d).reshape(n_kv, total, d)
    path = str(tmp_path / "big.rkvc")
    ref_write(path, [(k, v, total, cfg.l_global, cfg.l_local)], d=d, n_kv=n_kv)
    snap = N.Snapshot(ctx, path)
    c1 = snap.load_layer(0, N.BF16)
    c2 = N.Cache(ctx, n_kv, d, cfg.l_global, cfg.l_local, total, N.BF16)
    c2.append(np.ascontiguousarray(k.transpose(1, 0, 2).reshape(total, n_kv * d)),
              np.ascontiguousarray(v.transpose(1, 0, 2).reshape(total, n_kv * d)))
    rope = N.Rope(ctx, d, 500000.0, 8192)
    q = torch.from_numpy(synth.uniform(72, 32 * d).reshape(1, -1)).cuda()
    a = N.attend_step(ctx, c1, rope, q, 32, cfg)
    b = N.attend_step(ctx, c2, rope, q, 32, cfg)
    assert torch.equal(a.out, b.out)
    assert np.array_equal(a.spans[0], b.spans[0])
