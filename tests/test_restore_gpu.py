"""End-to-end restore on the GPU: pinned chunk store -> H2D copy engine ->
K1 / K4 -> paged KV, checked against the oracle (reference algorithm) and
the reference's restore test contracts (proj/tests/test_restore.cpp)."""
import numpy as np
import pytest

from hc_testutil import REL_TOL, cpu_hidden, cpu_wkv, dev_hidden, dev_wkv, max_rel_err

pytestmark = pytest.mark.gpu


def _setup(n_layers=4, d=512, heads=8, n=1024, page=64, kvh=None, rope=True):
    import torch
    from paper_2410_05004_b200 import hcache as H
    cfg = H.ModelConfig(n_layers=n_layers, d_hidden=d, n_heads=heads, n_kv_heads=kvh or heads,
                        d_ffn=4 * d, max_seq=max(n, 1024), rope_enabled=rope)
    w = H.Weights(cfg)
    for L in range(n_layers):
        w.set_layer_kv(L, dev_wkv(d, cfg.kv_heads() * cfg.d_head(), L))
    n_pages = (n + page - 1) // page + 3
    kv = H.KvCache(n_layers, n_pages, page, w.d_kv)
    table = torch.randperm(n_pages, generator=torch.Generator().manual_seed(1))[
        : (n + page - 1) // page].to(torch.int32).cuda()
    return cfg, w, kv, table


def _store_hidden(H, store, sid, cfg, n, plan, hidden_rows_fn, kv_rows_fn=None, tokens=None):
    store.create_session(H.SessionSeed(sid, cfg.hash(), cfg.n_layers, cfg.d_hidden, 2, plan,
                                       tokens if tokens is not None else list(range(n)),
                                       d_kv=cfg.kv_heads() * cfg.d_head()))
    for L, m in enumerate(plan.layer_assignment):
        if m == H.LayerMethod.HIDDEN:
            assert store.snapshot(sid, L, H.StateKind.HIDDEN, hidden_rows_fn(L))
        elif m == H.LayerMethod.KV_OFFLOAD:
            assert store.snapshot(sid, L, H.StateKind.KV, kv_rows_fn(L))
    store.finalize(sid)


@pytest.mark.parametrize("devices", [1, 2, 4])
def test_restore_all_hidden_matches_oracle(cuda, oracle, devices):
    """Config 1 shape: 4 layers, d=512, 8 heads, 1K tokens, paged cache."""
    import torch
    from paper_2410_05004_b200 import hcache as H
    n = 1024 + 64 * 9  # > 8 chunk slots per extent: runs span several pinned extents
    cfg, w, kv, table = _setup(n=n)
    store = H.StorageManager(H.DevicePool(devices))
    plan = H.RestorationPlan.make(4, 4, H.Complement.NONE)
    # layer L's hidden states: synthetic rows with seed 7 + L, saved D2H from the GPU
    _store_hidden(H, store, "s", cfg, n, plan, lambda L: dev_hidden(n, 512, seed=7 + L))
    res = H.restore(store, "s", w, plan, H.ThrottleConfig(), kv, table)
    torch.cuda.synchronize()
    for L in range(4):
        kr, vr = oracle.project(cpu_hidden(oracle, n, 512, seed=7 + L),
                                *cpu_wkv(oracle, 512, 512, L), 8)
        k, v = kv.gather(L, table, n)
        assert max_rel_err(k.float().cpu().numpy(), kr) < REL_TOL
        assert max_rel_err(v.float().cpu().numpy(), vr) < REL_TOL
    tl = res.timeline
    assert tl.total_s > 0 and tl.fill_s > 0
    kinds = sorted({e.kind for e in tl.events})
    assert kinds == ["fetch_hidden", "project"]
    assert sum(e.kind == "project" for e in tl.events) == 4
    # each projection starts after its own fetch finished
    fetch_end = {e.layer: e.end_s for e in tl.events if e.kind == "fetch_hidden"}
    for e in tl.events:
        if e.kind == "project":
            assert e.start_s >= fetch_end[e.layer] - 1e-6


@pytest.mark.parametrize("offset", [8.0, -40.0])
def test_restore_layernorm_large_mean(cuda, oracle, offset):
    """Hidden rows whose mean dwarfs their spread, restored through the store:
    the restore centres them in their staging slot (side stream) before K1;
    odd layers are ordinary rows, so flagged and unflagged layers alternate
    on the two K1 lanes."""
    import torch
    from oracle import bf16_round
    from paper_2410_05004_b200 import hcache as H
    n = 640
    cfg, w, kv, table = _setup(n=n)
    store = H.StorageManager(H.DevicePool(2))
    plan = H.RestorationPlan.make(4, 4, H.Complement.NONE)

    def rows(L):
        base = cpu_hidden(oracle, n, 512, seed=7 + L)
        return bf16_round(np.float32(offset) + np.float32(0.1) * base) if L % 2 == 0 else base
    _store_hidden(H, store, "s", cfg, n, plan,
                  lambda L: torch.from_numpy(rows(L)).cuda().bfloat16())
    H.restore(store, "s", w, plan, H.ThrottleConfig(), kv, table)
    torch.cuda.synchronize()
    for L in range(4):
        kr, vr = oracle.project(rows(L), *cpu_wkv(oracle, 512, 512, L), 8)
        k, v = kv.gather(L, table, n)
        assert max_rel_err(k.float().cpu().numpy(), kr) < REL_TOL
        assert max_rel_err(v.float().cpu().numpy(), vr) < REL_TOL


def test_restore_is_deterministic_and_equals_resident_path(cuda):
    import ctypes as C

    import torch
    from paper_2410_05004_b200 import hcache as H
    from paper_2410_05004_b200.capi import check, lib
    n = 700
    cfg, w, kv, table = _setup(n=n)
    store = H.StorageManager(H.DevicePool(3))
    plan = H.RestorationPlan.make(4, 4, H.Complement.NONE)
    hid = [dev_hidden(n, 512, seed=70 + L) for L in range(4)]
    _store_hidden(H, store, "s", cfg, n, plan, lambda L: hid[L])
    H.restore(store, "s", w, plan, H.ThrottleConfig(prefetch_depth=1), kv, table)
    torch.cuda.synchronize()
    a = [(kv.k[L].clone(), kv.v[L].clone()) for L in range(4)]
    _, w2, kv2, _ = _setup(n=n)
    ptrs = (C.c_void_p * 4)(*[h.data_ptr() for h in hid])
    check(lib().hc_restore_resident(w2._h, ptrs, n, None, 1, C.byref(kv2.desc), table.data_ptr(),
                                    0, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    for L in range(4):
        k2, v2 = kv2.gather(L, table, n)
        k1, v1 = kv.gather(L, table, n)
        assert torch.equal(k1, k2) and torch.equal(v1, v2)


def test_kv_offload_layers_restore_bit_exact(cuda):
    """Hybrid 2H+2KV plan (test_restore.cpp:128-135): KV layers come back
    bit-exact through H2D + K4 scatter."""
    import torch
    from paper_2410_05004_b200 import hcache as H
    n = 333
    cfg, w, kv, table = _setup(n=n)
    store = H.StorageManager(H.DevicePool(2))
    plan = H.RestorationPlan.make(4, 2, H.Complement.KV_OFFLOAD)
    kvrows = {L: dev_hidden(n, 1024, seed=500 + L) for L in range(4)}  # [K_row | V_row]
    _store_hidden(H, store, "s", cfg, n, plan, lambda L: dev_hidden(n, 512, seed=7 + L),
                  lambda L: kvrows[L])
    res = H.restore(store, "s", w, plan, H.ThrottleConfig(), kv, table)
    torch.cuda.synchronize()
    for L in (2, 3):
        k, v = kv.gather(L, table, n)
        assert torch.equal(k, kvrows[L][:, :512]) and torch.equal(v, kvrows[L][:, 512:])
    for L in (0, 1):
        kd, vd = H.project_hidden_to_kv(w, L, dev_hidden(n, 512, seed=7 + L), 0)
        k, v = kv.gather(L, table, n)
        torch.cuda.synchronize()
        assert torch.equal(k, kd) and torch.equal(v, vd)
    assert sum(e.kind == "fetch_kv" for e in res.timeline.events) == 2
    assert sum(e.kind == "scatter" for e in res.timeline.events) == 2


def test_restore_error_contract(cuda):
    """test_restore.cpp:199-207 (plan mismatch -> invalid_argument) and the
    storage errors (missing / unfinalized session)."""
    import torch  # noqa: F401
    from paper_2410_05004_b200 import capi
    from paper_2410_05004_b200 import hcache as H
    n = 64
    cfg, w, kv, table = _setup(n=n)
    store = H.StorageManager(H.DevicePool(1))
    stored = H.RestorationPlan.make(4, 4, H.Complement.NONE)
    _store_hidden(H, store, "s", cfg, n, stored, lambda L: dev_hidden(n, 512, seed=L))
    other = H.RestorationPlan.make(4, 2, H.Complement.KV_OFFLOAD)
    with pytest.raises(ValueError):
        H.restore(store, "s", w, other, H.ThrottleConfig(), kv, table)
    with pytest.raises(capi.NotFound):
        H.restore(store, "nope", w, stored, H.ThrottleConfig(), kv, table)
    store.create_session(H.SessionSeed("open", 0, 4, 512, 2, stored, [], d_kv=512))
    with pytest.raises(capi.Incomplete):
        H.restore(store, "open", w, stored, H.ThrottleConfig(), kv, table)
    # an empty session has no chunks (restore.cpp:70-71: runtime_error)
    store.finalize("open")
    with pytest.raises(capi.NotFound):
        H.restore(store, "open", w, stored, H.ThrottleConfig(), kv, table)


def test_device_snapshot_roundtrip_bitexact(cuda):
    """Stage-1 D2H snapshot on a side stream -> chunks -> read_layer H2D."""
    import torch
    from paper_2410_05004_b200 import hcache as H
    store = H.StorageManager(H.DevicePool(3), buffer_capacity_bytes=64 << 20)
    plan = H.RestorationPlan.make(2, 2, H.Complement.NONE)
    store.create_session(H.SessionSeed("s", 1, 2, 256, 2, plan, [1, 2]))
    rows = dev_hidden(1000, 256, seed=3)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for a, b in ((0, 100), (100, 163), (163, 1000)):  # ragged pieces
            assert store.snapshot("s", 0, H.StateKind.HIDDEN, rows[a:b], stream=side.cuda_stream)
    store.finalize("s")
    back = torch.empty_like(rows)
    store.read_layer_device("s", 0, H.StateKind.HIDDEN, back)
    torch.cuda.synchronize()
    assert torch.equal(back, rows)
    man = store.open("s")
    host = store.read_layer(man, 0, H.StateKind.HIDDEN)
    assert np.array_equal(host, rows.view(torch.int16).cpu().numpy().view(np.uint16))
    assert store.read_layer(man, 1, H.StateKind.HIDDEN) is None


@pytest.mark.parametrize("b,pieces", [(0, [(0, 384)]), (128, [(128, 300), (300, 333)]),
                                      (192, [(192, 256), (256, 1000)])])
def test_device_range_snapshot_roundtrip_bitexact(cuda, b, pieces):
    """A head-sharded rank's save (snapshot_range from device rows): the
    direct D2H path starts a fresh stream at tok_begin; a continuation at the
    stored end keeps it, a ragged one falls back to stage 1. The rank's token
    range reads back bit-exact; tokens below it are not held."""
    import torch
    from paper_2410_05004_b200 import capi
    from paper_2410_05004_b200 import hcache as H
    store = H.StorageManager(H.DevicePool(3), buffer_capacity_bytes=64 << 20)
    plan = H.RestorationPlan.make(2, 2, H.Complement.NONE)
    n = 1000
    store.create_session(H.SessionSeed("s", 1, 2, 256, 2, plan, list(range(n))))
    rows = dev_hidden(n, 256, seed=5)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for x, y in pieces:
            tb = x if x % 64 == 0 else None
            assert store.snapshot("s", 0, H.StateKind.HIDDEN, rows[x:y].contiguous(),
                                  tok_begin=tb, stream=side.cuda_stream)
    side.synchronize()
    store.finalize("s")
    e = pieces[-1][1]
    back = torch.empty((e - b, 256), dtype=rows.dtype, device="cuda")

    def read(x, y, dst):
        return capi.lib().hc_store_read_layer_range(
            store._h, b"s", 0, int(H.StateKind.HIDDEN), x, y, dst.data_ptr(),
            dst.numel() * dst.element_size(), 1, torch.cuda.current_stream().cuda_stream)
    capi.check(read(b, e, back))
    torch.cuda.synchronize()
    assert torch.equal(back, rows[b:e])
    if b:
        assert read(0, 64, back[:64]) == capi.HC_ENOENT  # held by another rank


def test_restore_batch_ragged_equals_single(cuda):
    """Config 4 layout: several sessions restored by one grouped K1 per layer."""
    import torch
    from paper_2410_05004_b200 import hcache as H
    d, page = 512, 64
    lens = [130, 1, 64, 517]
    cfg, w, _, _ = _setup(n=max(lens))
    store = H.StorageManager(H.DevicePool(2))
    plan = H.RestorationPlan.make(4, 4, H.Complement.NONE)
    for s, n in enumerate(lens):
        _store_hidden(H, store, f"s{s}", cfg, n, plan,
                      lambda L, s=s, n=n: dev_hidden(n, d, seed=1000 * s + L))
    stride = max((n + page - 1) // page for n in lens)
    tables = torch.arange(len(lens) * stride, dtype=torch.int32).view(len(lens), stride).cuda()
    kv = H.KvCache(4, len(lens) * stride, page, 512)
    res = H.restore_batch(store, [f"s{s}" for s in range(len(lens))], w, H.ThrottleConfig(), kv,
                          tables)
    torch.cuda.synchronize()
    assert sum(e.kind == "project" for e in res.timeline.events) == 4
    for s, n in enumerate(lens):
        for L in range(4):
            kd, vd = H.project_hidden_to_kv(w, L, dev_hidden(n, d, seed=1000 * s + L), 0)
            k, v = kv.gather(L, tables[s], n)
            torch.cuda.synchronize()
            assert torch.equal(k, kd) and torch.equal(v, vd), (s, L)


def test_profile_and_three_way_plan(cuda):
    from paper_2410_05004_b200 import hcache as H
    cfg, w, _, _ = _setup(n=1024)
    t = H.profile_hardware(w, 1024)
    assert t.io_h > 0 and t.io_kv > 0 and t.c_h > 0 and t.c_token > 0
    assert 1.5 < t.io_kv / t.io_h < 2.5  # MHA: KV rows are twice the hidden bytes
    p, ms = H.plan_three_way(t, 4)
    assert p.n_layers() == 4 and ms > 0


def test_h2d_bandwidth_is_pcie_class(cuda):
    from paper_2410_05004_b200 import hcache as H
    bw = H.measure_h2d(64 << 20)
    assert 5e9 < bw < 400e9


def _store_everything(n, sid="tw"):
    """test_restore.cpp:209-244 setup: every layer stored as HIDDEN and KV,
    KV rows = the K1 projection of the hidden rows (a consistent session)."""
    import torch
    from paper_2410_05004_b200 import hcache as H
    cfg, w, kv, table = _setup(n=n)
    store = H.StorageManager(H.DevicePool(2))
    plan = H.RestorationPlan.make(4, 4, H.Complement.NONE)
    store.create_session(H.SessionSeed(sid, cfg.hash(), 4, 512, 2, plan, list(range(n)), d_kv=512))
    want = []
    for L in range(4):
        h = dev_hidden(n, 512, seed=600 + L)
        k, v = H.project_hidden_to_kv(w, L, h, 0)
        want.append((k, v))
        assert store.snapshot(sid, L, H.StateKind.HIDDEN, h)
        assert store.snapshot(sid, L, H.StateKind.KV, torch.cat([k, v], 1).contiguous())
    store.finalize(sid)
    return cfg, w, kv, table, store, want


@pytest.mark.parametrize("split", [0, 130, 192, 256, 320])
def test_token_wise_split_restores_correctly(cuda, split):
    import torch
    from paper_2410_05004_b200 import hcache as H
    n = 320
    cfg, w, kv, table, store, want = _store_everything(n)
    res = H.restore_token_wise(store, "tw", w, split, kv, table)
    torch.cuda.synchronize()
    for L in range(4):
        k, v = kv.gather(L, table, n)
        assert torch.equal(k, want[L][0]) and torch.equal(v, want[L][1]), (split, L)
    assert sum(e.kind == "fetch" for e in res.timeline.events) == 4


def test_token_wise_rejects_bad_splits(cuda):
    from paper_2410_05004_b200 import hcache as H
    cfg, w, kv, table, store, want = _store_everything(100, "tw2")
    for bad in (-1, 101):
        with pytest.raises(ValueError):
            H.restore_token_wise(store, "tw2", w, bad, kv, table)


@pytest.mark.parametrize("fmt", ["f32", "f16"])
def test_restore_reference_element_formats(cuda, oracle, fmt):
    """Sessions persisted in the reference's own formats -- fp32
    (ModelConfig::elem_bytes = 4, its default) and the fp16 codec
    (fp16.hpp) -- restore through the same device path: rows travel as stored
    and are rounded to bf16 on the device. HIDDEN layers vs the oracle
    projection of the bf16-rounded rows (REL_TOL); KV-offload layers equal the
    bf16 rounding of the stored rows exactly."""
    import torch
    from oracle import bf16_round
    from paper_2410_05004_b200 import capi
    from paper_2410_05004_b200 import hcache as H
    n = 450
    cfg, w, kv, table = _setup(n=n)
    store = H.StorageManager(H.DevicePool(2))
    plan = H.RestorationPlan.make(4, 3, H.Complement.KV_OFFLOAD)
    eb, dt = (4, capi.HC_DTYPE_F32) if fmt == "f32" else (2, capi.HC_DTYPE_F16)
    store.create_session(H.SessionSeed("r", cfg.hash(), 4, 512, eb, plan, list(range(n)), d_kv=512,
                                       dtype=dt))
    rng = np.random.default_rng(5)
    hid = [rng.standard_normal((n, 512)).astype(np.float32) for _ in range(3)]
    kvrows = rng.standard_normal((n, 1024)).astype(np.float32)
    for L in range(3):
        assert store.snapshot("r", L, H.StateKind.HIDDEN, hid[L])  # host fp32 -> session codec
    assert store.snapshot("r", 3, H.StateKind.KV, kvrows)
    store.finalize("r")
    H.restore(store, "r", w, plan, H.ThrottleConfig(), kv, table)
    torch.cuda.synchronize()

    def stored(x):  # what the session holds, as fp32
        return x if fmt == "f32" else x.astype(np.float16).astype(np.float32)
    for L in range(3):
        kr, vr = oracle.project(bf16_round(stored(hid[L])), *cpu_wkv(oracle, 512, 512, L), 8)
        k, v = kv.gather(L, table, n)
        assert max_rel_err(k.float().cpu().numpy(), kr) < REL_TOL, L
        assert max_rel_err(v.float().cpu().numpy(), vr) < REL_TOL, L
    k, v = kv.gather(3, table, n)
    want = torch.from_numpy(stored(kvrows)).bfloat16()
    assert torch.equal(k.cpu(), want[:, :512]) and torch.equal(v.cpu(), want[:, 512:])
