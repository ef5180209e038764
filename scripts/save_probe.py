"""Save-path probe (north star (1)): a 7B prefill's 32 layer inputs (4096
tokens x 4096, bf16, on the device) snapshotted into the pinned chunk store --
device rows at a chunk boundary go D2H on a side stream straight into their
chunk slots, stage 1 keeps the copy's event -- then drained and finalized; and,
for scale, one device->host copy of the same bytes. Cold runs pin the arena on
the way (cudaHostAlloc), reserved runs page-lock it first (hc_store_reserve)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2410_05004_b200 import hcache as H


def main():
    L, n, d = 32, 4096, 4096
    torch.cuda.set_device(0)
    rows = [torch.randn(n, d, device="cuda").bfloat16() for _ in range(L)]
    side = torch.cuda.Stream()
    nbytes = L * n * d * 2
    cfg = H.ModelConfig(n_layers=L, d_hidden=d, n_heads=32, d_ffn=11008, max_seq=4096)
    plan = H.RestorationPlan.make(L, L, H.Complement.NONE)
    for it in range(4):
        store = H.StorageManager(H.DevicePool(1), buffer_capacity_bytes=2 << 30)
        warm = it >= 2
        if warm:  # the arena page-locked up front (hc_store_reserve), as a serving host does
            store.reserve(2 * nbytes + (64 << 20))
        store.create_session(H.SessionSeed("s", cfg.hash(), L, d, 2, plan, list(range(n))))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        stalls = 0
        for layer in range(L):
            while not store.snapshot("s", layer, H.StateKind.HIDDEN, rows[layer],
                                     stream=side.cuda_stream):
                stalls += 1
                store.drain()
        t1 = time.perf_counter()
        store.drain_all()
        store.finalize("s")
        t2 = time.perf_counter()
        print(f"run {it} ({'reserved arena' if warm else 'cold: pins on the way'}): snapshot calls {nbytes / (t1 - t0) / 1e9:6.1f} GB/s "
              f"({(t1 - t0) * 1e3:7.1f} ms, {stalls} backpressure drains), "
              f"to finalized {nbytes / (t2 - t0) / 1e9:6.1f} GB/s ({(t2 - t0) * 1e3:7.1f} ms)")
        store.close()
    host = torch.empty(n * d, dtype=torch.bfloat16, pin_memory=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for layer in range(L):
        host.copy_(rows[layer].view(-1), non_blocking=True)
    torch.cuda.synchronize()
    print(f"plain pinned D2H of the same bytes: {nbytes / (time.perf_counter() - t0) / 1e9:6.1f} GB/s")


if __name__ == "__main__":
    main()
