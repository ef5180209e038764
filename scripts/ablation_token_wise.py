"""Token-wise vs layer-wise partition ablation (reference
restore_token_wise, proj/src/restore.cpp:237-301; PAPER Fig. 11).

Llama-2-7B shape, 4096-token context, restored from the pinned store on one
B200. For each hidden fraction f the layer-wise partition restores f*L layers
from hidden states and the rest from stored KV (hc_restore with
Complement::KV_OFFLOAD); the token-wise partition restores the first f*n tokens
of EVERY layer from hidden states and splices KV for the rest
(hc_restore_token_wise). Both move the same hidden/KV byte mix (token-wise
re-reads the KV chunk straddling the split). Timed with CUDA events over
`steps` restores after warm-up; prints one JSON object and writes it to
profiles/r1_ablation_token_wise.json when --out is given."""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2410_05004_b200 import capi
from paper_2410_05004_b200 import hcache as H
from paper_2410_05004_b200.capi import check, lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    L, d, n = a.layers, a.d, a.n
    heads = d // 128
    stream = torch.cuda.current_stream().cuda_stream
    mc = H.ModelConfig(n_layers=L, d_hidden=d, n_heads=heads, d_ffn=4 * d, max_seq=n)
    w = H.Weights(mc)
    bound = float(np.float32(1) / np.sqrt(np.float32(d)))
    for layer in range(L):
        t = torch.empty((2 * d, d), dtype=torch.bfloat16, device="cuda")
        check(lib().hc_fill_symmetric(t.data_ptr(), t.numel(), 1234 + layer, 0, bound, 1, stream))
        w.set_layer_kv(layer, t)
    hid = torch.empty((n, d), dtype=torch.bfloat16, device="cuda")
    check(lib().hc_fill_symmetric(hid.data_ptr(), hid.numel(), 7, 0, 1.7320508, 1, stream))
    kvrows = torch.empty((n, 2 * d), dtype=torch.bfloat16, device="cuda")
    check(lib().hc_fill_symmetric(kvrows.data_ptr(), kvrows.numel(), 8, 0, 1.0, 1, stream))
    page = 64
    kv = H.KvCache(L, n // page, page, d)
    table = torch.arange(n // page, dtype=torch.int32, device="cuda")
    tokens = list(range(n))

    def timed(fn):
        for _ in range(a.warmup):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.steps

    rows = []
    opts = capi.RestoreOptsC(0, 0)
    for f in (0.0, 0.25, 0.5, 0.75, 1.0):
        lh, s = int(round(f * L)), int(round(f * n))
        store = H.StorageManager(H.DevicePool(1), buffer_capacity_bytes=4 << 30)
        p = H.RestorationPlan.make(L, lh, H.Complement.KV_OFFLOAD if lh < L else H.Complement.NONE)
        store.create_session(H.SessionSeed("lw", mc.hash(), L, d, 2, p, tokens))
        for layer, m in enumerate(p.layer_assignment):
            src = hid if m == H.LayerMethod.HIDDEN else kvrows
            kind = H.StateKind.HIDDEN if m == H.LayerMethod.HIDDEN else H.StateKind.KV
            while not store.snapshot("lw", layer, kind, src):
                store.drain()
        store.finalize("lw")
        t_lw = timed(lambda: check(lib().hc_restore(store._h, b"lw", w._h, C.byref(p._c),
                                                    C.byref(opts), C.byref(kv.desc),
                                                    table.data_ptr(), stream, None)))
        store.close()
        store = H.StorageManager(H.DevicePool(1), buffer_capacity_bytes=4 << 30)
        store.create_session(H.SessionSeed("tw", mc.hash(), L, d, 2,
                                           H.RestorationPlan.make(L, L, H.Complement.NONE), tokens))
        for layer in range(L):
            for kind, src in ((H.StateKind.HIDDEN, hid), (H.StateKind.KV, kvrows)):
                while not store.snapshot("tw", layer, kind, src):
                    store.drain()
        store.finalize("tw")
        t_tw = timed(lambda: check(lib().hc_restore_token_wise(store._h, b"tw", w._h, s,
                                                               C.byref(kv.desc), table.data_ptr(),
                                                               stream, None)))
        store.close()
        kv_b = (s // 64) * 64
        bytes_lw = lh * n * d * 2 + (L - lh) * n * 2 * d * 2
        bytes_tw = L * (s * d * 2 + (n - kv_b) * 2 * d * 2)
        rows.append({"hidden_fraction": f, "layer_wise": {"hidden_layers": lh, "ms": t_lw,
                                                         "h2d_bytes": bytes_lw},
                     "token_wise": {"hidden_tokens": s, "ms": t_tw, "h2d_bytes": bytes_tw},
                     "token_wise_slowdown": t_tw / t_lw})
        print(json.dumps(rows[-1]), flush=True)
    out = {"config": {"layers": L, "d_hidden": d, "n_tokens": n, "gpu": torch.cuda.get_device_name()},
           "rows": rows}
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
