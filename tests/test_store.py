"""Pinned-host chunk store through the C ABI: ports of
proj/tests/test_storage.cpp and acceptance criterion 9, plus bit-exact chunk
placement/payload checks (north star: chunk indexing must match exactly)."""
import time

import numpy as np
import pytest

from hc_testutil import golden
from paper_2410_05004_b200 import capi
from paper_2410_05004_b200 import hcache as H

K = H.StateKind


def pattern(rows, cols, scale=1e-3, shift=0.0):
    # test_storage.cpp:29-34
    i = np.arange(rows * cols)
    return (scale * ((i % 2001) - 1000).astype(np.float32) + np.float32(shift)).astype(
        np.float32).reshape(rows, cols)


def seed(sid, d, n_layers, elem_bytes=4, tokens=(1, 2, 3)):
    return H.SessionSeed(sid, 99, n_layers, d, elem_bytes,
                         H.RestorationPlan.make(n_layers, n_layers, H.Complement.NONE), list(tokens))


def test_duplicate_session_rejected():
    s = H.StorageManager(H.DevicePool(2))
    s.create_session(seed("a", 16, 1))
    with pytest.raises(capi.HCacheError):
        s.create_session(seed("a", 16, 1))


def test_130_tokens_three_chunks():
    s = H.StorageManager(H.DevicePool(3))
    s.create_session(seed("s", 32, 1))
    s.snapshot("s", 0, K.HIDDEN, pattern(130, 32))
    s.finalize("s")
    m = s.open("s")
    lc = m.find(0, K.HIDDEN)
    assert (lc.n_tokens, lc.n_chunks, m.n_tokens) == (130, 3, 130)
    assert sum(s.device_chunk_counts()) == 3


def test_chunks_stripe_evenly():
    s = H.StorageManager(H.DevicePool(4))
    s.create_session(seed("s", 64, 2))
    for L in range(2):
        s.snapshot("s", L, K.HIDDEN, pattern(1024, 64))
    s.finalize("s")
    assert s.device_chunk_counts() == [8, 8, 8, 8]


def test_hidden_and_kv_roundtrip_bitwise_fp32():
    s = H.StorageManager(H.DevicePool(2))
    s.create_session(seed("s", 48, 2))
    h = pattern(200, 48)
    k, v = pattern(200, 48, 2e-3), pattern(200, 48, -1e-3)
    s.snapshot("s", 0, K.HIDDEN, h)
    s.snapshot("s", 1, K.KV, H.interleave_kv(k, v))
    s.finalize("s")
    m = s.open("s")
    assert np.array_equal(s.read_layer(m, 0, K.HIDDEN), h)
    k2, v2 = H.split_kv(s.read_layer(m, 1, K.KV))
    assert np.array_equal(k2, k) and np.array_equal(v2, v)
    assert m.tokens == [1, 2, 3]


def test_fp16_persistence_quantization_error():
    s = H.StorageManager(H.DevicePool(2))
    sd = seed("s", 32, 1, 2)
    sd.dtype = capi.HC_DTYPE_F16
    s.create_session(sd)
    h = pattern(100, 32)
    s.snapshot("s", 0, K.HIDDEN, h)
    s.finalize("s")
    bits = s.read_layer(s.open("s"), 0, K.HIDDEN)
    back = bits.view(np.float16).astype(np.float32)
    err = np.max(np.abs(back - h))
    assert 0 < err < 1e-3


def test_bf16_persistence_is_rne(oracle):
    from oracle import bf16_bits
    s = H.StorageManager(H.DevicePool(1))
    s.create_session(seed("s", 32, 1, 2))
    h = pattern(100, 32, 1.37e-3, 0.1)
    s.snapshot("s", 0, K.HIDDEN, h)
    s.finalize("s")
    assert np.array_equal(s.read_layer(s.open("s"), 0, K.HIDDEN), bf16_bits(h))


def test_interleaved_sessions_do_not_bleed():
    s = H.StorageManager(H.DevicePool(2))
    s.create_session(seed("x", 16, 1))
    s.create_session(seed("y", 16, 1))
    hx, hy = pattern(70, 16, 1e-3, 0.5), pattern(70, 16, 1e-3, -0.5)
    for i in range(7):
        s.snapshot("x", 0, K.HIDDEN, hx[10 * i:10 * (i + 1)])
        s.snapshot("y", 0, K.HIDDEN, hy[10 * i:10 * (i + 1)])
    s.finalize("x")
    s.finalize("y")
    assert np.array_equal(s.read_layer(s.open("x"), 0, K.HIDDEN), hx)
    assert np.array_equal(s.read_layer(s.open("y"), 0, K.HIDDEN), hy)


def test_finalize_idempotent_open_before_finalize_throws():
    s = H.StorageManager(H.DevicePool(1))
    s.create_session(seed("s", 16, 1))
    s.snapshot("s", 0, K.HIDDEN, pattern(10, 16))
    s.drain_all()
    with pytest.raises(capi.Incomplete):
        s.open("s")
    s.finalize("s")
    s.finalize("s")
    assert s.open("s").finalized and s.open("s").n_tokens == 10
    with pytest.raises(capi.NotFound):
        s.open("never")


def test_absent_layers_read_back_none():
    s = H.StorageManager(H.DevicePool(1))
    s.create_session(seed("s", 16, 3))
    s.snapshot("s", 1, K.HIDDEN, pattern(5, 16))
    s.finalize("s")
    m = s.open("s")
    assert s.read_layer(m, 0, K.HIDDEN) is None
    assert s.read_layer(m, 1, K.KV) is None
    assert s.read_layer(m, 1, K.HIDDEN) is not None


def test_simulated_read_time():
    # test_storage.cpp:179-197
    bw, lat = 1e9, 1e-4
    s = H.StorageManager(H.DevicePool(4, bw, lat))
    chunk_b = 64.0 * 64.0 * 4.0
    want = 4 * (lat + chunk_b / bw)
    assert s.simulated_read_seconds_tokens(1024, 64, 4) == pytest.approx(want, rel=1e-12)
    assert s.simulated_read_seconds_tokens(1024, 128, 4) == pytest.approx(4 * (lat + 2 * chunk_b / bw), rel=1e-12)


def test_reopen_for_append_extends_seamlessly():
    s = H.StorageManager(H.DevicePool(2))
    allrows = pattern(150, 32)
    s.create_session(seed("s", 32, 1))
    s.snapshot("s", 0, K.HIDDEN, allrows[:90])
    s.finalize("s")
    s.reopen_for_append("s", [7, 8])
    with pytest.raises(capi.Incomplete):
        s.open("s")
    s.snapshot("s", 0, K.HIDDEN, allrows[90:])
    s.finalize("s")
    m = s.open("s")
    assert m.n_tokens == 150 and m.tokens == [1, 2, 3, 7, 8]
    assert np.array_equal(s.read_layer(m, 0, K.HIDDEN), allrows)


def test_full_buffer_pushes_back():
    s = H.StorageManager(H.DevicePool(1), buffer_capacity_bytes=4 * 1024)
    s.create_session(seed("s", 16, 1))
    h = pattern(80, 16)
    assert s.snapshot("s", 0, K.HIDDEN, h[:40])
    assert not s.snapshot("s", 0, K.HIDDEN, h[40:])
    assert s.backpressure_events() == 1
    s.drain()
    assert s.snapshot("s", 0, K.HIDDEN, h[40:])
    s.finalize("s")
    assert np.array_equal(s.read_layer(s.open("s"), 0, K.HIDDEN), h)


def test_daemon_drains():
    s = H.StorageManager(H.DevicePool(2))
    s.start_daemon()
    s.create_session(seed("s", 32, 1))
    h = pattern(256, 32)
    for i in range(4):
        s.snapshot("s", 0, K.HIDDEN, h[64 * i:64 * (i + 1)])
    for _ in range(200):
        if s.buffer_bytes() == 0:
            break
        time.sleep(0.002)
    assert s.buffer_bytes() == 0
    s.stop_daemon()
    s.finalize("s")
    assert np.array_equal(s.read_layer(s.open("s"), 0, K.HIDDEN), h)


def test_snapshot_validation():
    s = H.StorageManager(H.DevicePool(1))
    s.create_session(seed("s", 16, 1))
    with pytest.raises(capi.HCacheError):
        s.snapshot("nope", 0, K.HIDDEN, pattern(4, 16))
    with pytest.raises(ValueError):
        s.snapshot("s", 0, K.HIDDEN, pattern(4, 8))
    with pytest.raises(ValueError):
        s.snapshot("s", 0, K.KV, pattern(4, 16))
    s.finalize("s")
    with pytest.raises(capi.HCacheError):
        s.snapshot("s", 0, K.HIDDEN, pattern(4, 16))


def test_randomized_roundtrip_criterion9():
    """acceptance.cpp:384-429 + placement/payload bit-exactness vs goldens."""
    rng = np.random.default_rng(99)
    for trial in range(25):
        n, devices, layers, d = int(rng.integers(1, 2049)), int(rng.integers(1, 5)), \
            int(rng.integers(1, 4)), 32
        s = H.StorageManager(H.DevicePool(devices))
        s.create_session(seed("s", d, layers))
        data = []
        for L in range(layers):
            m = (rng.integers(0, 65536, (n, d)).astype(np.float32) - 32768) / 16384
            at = 0
            while at < n:
                take = min(int(rng.integers(1, 201)), n - at)
                while not s.snapshot("s", L, K.HIDDEN, m[at:at + take]):
                    s.drain()
                at += take
            data.append(m.astype(np.float32))
        s.finalize("s")
        man = s.open("s")
        want_chunks = (n + 63) // 64
        for L in range(layers):
            assert np.array_equal(s.read_layer(man, L, K.HIDDEN), data[L])
            assert man.find(L, K.HIDDEN).n_chunks == want_chunks
            per_dev = [0] * devices
            for c in range(want_chunks):
                dev, ptr, nbytes = s.chunk_info("s", L, K.HIDDEN, c)
                assert dev == H.device_for_chunk(L, c, devices) == (L + c) % devices
                per_dev[dev] += 1
                # payload layout: tokens consecutive, d fp32 elements each
                rows = min(64, n - 64 * c)
                assert nbytes == rows * d * 4
                payload = np.ctypeslib.as_array((np.ctypeslib.ctypes.c_float * (rows * d)).from_address(ptr))
                assert np.array_equal(payload.reshape(rows, d), data[L][64 * c: 64 * c + rows])
            assert max(per_dev) - min(per_dev) <= 1


def test_placement_matches_reference_goldens():
    for c in golden("storage.json"):
        for L, row in enumerate(c["placement"]):
            assert [H.device_for_chunk(L, ci, c["devices"]) for ci in range(len(row))] == row


def test_read_layer_range_sharded_fetch():
    """Head-sharded fetch: chunk-aligned token ranges reassemble."""
    s = H.StorageManager(H.DevicePool(3))
    s.create_session(seed("s", 16, 2))
    h = pattern(1000, 16)
    s.snapshot("s", 1, K.HIDDEN, h)
    s.finalize("s")
    import ctypes as Cc
    out = np.zeros((1000, 16), np.float32)
    for b, e in ((0, 320), (320, 640), (640, 1000)):
        buf = np.zeros((e - b, 16), np.float32)
        capi.check(capi.lib().hc_store_read_layer_range(s._h, b"s", 1, 0, b, e, buf.ctypes.data,
                                                        buf.nbytes, 0, None))
        out[b:e] = buf
    assert np.array_equal(out, h)
    buf = np.zeros((10, 16), np.float32)
    st = capi.lib().hc_store_read_layer_range(s._h, b"s", 1, 0, 10, 20, buf.ctypes.data,
                                              buf.nbytes, 0, None)
    assert st == capi.HC_EINVAL  # begin must be chunk aligned
    del Cc


def test_range_snapshot_keeps_chunk_indexing():
    """hc_store_snapshot_range (the head-sharded save path): a rank stores
    tokens [128, 300) of a layer; chunk c keeps its reference index, device
    (layer + c) % ndev and payload; chunks below the range are not held here."""
    import ctypes as C
    st = H.StorageManager(H.DevicePool(3))
    st.create_session(seed("r", 64, 2, tokens=range(300)))
    rows = pattern(172, 64)
    assert st.snapshot("r", 1, K.HIDDEN, rows, tok_begin=128)
    with pytest.raises(ValueError):  # not chunk aligned
        st.snapshot("r", 0, K.HIDDEN, rows, tok_begin=100)
    st.finalize("r")
    lc = st.open("r").find(1, K.HIDDEN)
    assert (lc.n_chunks, lc.n_tokens) == (5, 300)
    for c in (2, 3, 4):
        dev, ptr, nb = st.chunk_info("r", 1, K.HIDDEN, c)
        assert dev == (1 + c) % 3
        want = rows[(c - 2) * 64:(c - 1) * 64]
        got = np.frombuffer((C.c_char * nb).from_address(ptr), dtype=np.float32)
        assert np.array_equal(got, want.ravel())
    with pytest.raises(capi.NotFound):  # held by another rank
        st.chunk_info("r", 1, K.HIDDEN, 1)
    out = np.empty((172, 64), np.float32)
    capi.check(capi.lib().hc_store_read_layer_range(st._h, b"r", 1, int(K.HIDDEN), 128, 300,
                                                    out.ctypes.data, out.nbytes, 0, None))
    assert np.array_equal(out, rows)
    bad = np.empty((300, 64), np.float32)
    with pytest.raises(capi.NotFound):
        capi.check(capi.lib().hc_store_read_layer_range(st._h, b"r", 1, int(K.HIDDEN), 0, 300,
                                                        bad.ctypes.data, bad.nbytes, 0, None))
    assert sum(st.device_chunk_counts()) == 3


def test_shard_geometry():
    for n, world in ((700, 2), (1000, 4), (100, 4), (4096, 8), (32768, 8)):
        rs = [H.shard_range(n, world, r) for r in range(world)]
        assert rs[0][0] == 0 and rs[-1][1] == n
        for (a, b), (c, _) in zip(rs, rs[1:]):
            assert b == c and (b % 128 == 0 or b == n)
    assert H.shard_heads(8, 4, 3) == (6, 2)
    with pytest.raises(ValueError):
        H.shard_heads(8, 3, 0)
