"""Serving benchmark (PAPER Fig. 7-9 TTFT/TBT metrics):
the device serving loop (hc_serve_run) over a conversation trace on a
Llama-2-7B-shaped model (random-init bf16 weights, 32 layers, d=4096), one
B200, for the four strategies (harness.cpp:14-31), plus the saving-mode
comparison of acceptance criterion 8 (proj/tests/acceptance.cpp:340-381):
TBT with two-stage saving vs IDEAL (no saving) vs direct saving.

Prints one JSON object (and writes it with --out)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2410_05004_b200 import hcache as H
from paper_2410_05004_b200.capi import check, lib


def build_weights(L, d, heads, dffn, vocab, max_seq, stream):
    mc = H.ModelConfig(n_layers=L, d_hidden=d, n_heads=heads, d_ffn=dffn, vocab_size=vocab,
                       max_seq=max_seq)
    w = H.Weights(mc)
    bound = float(np.float32(1) / np.sqrt(np.float32(d)))
    keep = []

    def fill(shape, seed):
        t = shape if torch.is_tensor(shape) else torch.empty(shape, dtype=torch.bfloat16,
                                                              device="cuda")
        check(lib().hc_fill_symmetric(t.data_ptr(), t.numel(), seed, 0, bound, 1, stream))
        keep.append(t)
        return t
    w.set_embedding(fill((vocab, d), 99))
    for layer in range(L):
        qkv = fill((3 * d, d), 0)  # [W_q ; W_k ; W_v]: the fused Q/K/V GEMM
        wq, wkv = fill(qkv[:d], 5000 + layer), fill(qkv[d:], 1234 + layer)
        w.set_layer_kv(layer, wkv)
        w.set_layer_full(layer, wq, wkv, fill((d, d), 6000 + layer),
                         fill((dffn, d), 7000 + layer), fill((d, dffn), 8000 + layer))
    torch.cuda.synchronize()
    return mc, w, keep


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--sessions", type=int, default=16)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--mean-input", type=float, default=66.8)
    ap.add_argument("--mean-output", type=float, default=64.0)
    ap.add_argument("--rate", type=float, default=2.0)
    ap.add_argument("--gap", type=float, default=30.0)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--strategies", default="IDEAL,HCACHE,KV_OFFLOAD,RECOMPUTE")
    ap.add_argument("--long-sessions", type=int, default=6)
    ap.add_argument("--arenas", type=int, default=4)
    ap.add_argument("--skip-conv", action="store_true")
    ap.add_argument("--skip-saving", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    stream = torch.cuda.current_stream().cuda_stream
    L, d = a.layers, a.d
    heads, dffn, vocab = d // 128, int(d * 11008 / 4096) // 32 * 32, 32000
    mc, w, keep = build_weights(L, d, heads, dffn, vocab, 8192, stream)
    p = H.TraceParams(n_sessions=a.sessions, rounds=a.rounds, mean_input=a.mean_input,
                      mean_output=a.mean_output, arrival_rate_per_s=a.rate, round_gap_s=a.gap,
                      vocab=vocab)
    tr = H.gen_trace(H.TraceKind.CONVERSATION, p, a.seed)
    # bubble-free plan from the measured timings at the trace's mean history
    hist = [r.history_tokens for r in tr.requests if r.history_tokens > 0]
    n_prof = int(np.clip(np.mean(hist) if hist else 1024, 256, 4096))
    prof = H.profile_hardware(w, n_prof)
    prof.n_layers = L
    plan, plan_ms = H.plan_three_way(prof, L)
    out = {"config": {"model": "llama2-7b-shape (random-init bf16)", "layers": L, "d_hidden": d,
                      "d_ffn": dffn, "trace": vars(p), "trace_seed": a.seed,
                      "requests": len(tr.requests),
                      "history_tokens": int(sum(r.history_tokens for r in tr.requests)),
                      "generated_tokens": int(sum(r.output_budget for r in tr.requests)),
                      "gpu": torch.cuda.get_device_name()},
           "plan": plan.serialize(), "profiled_at_tokens": n_prof,
           "profiled": {"io_h_ms": prof.io_h * 1e3, "io_kv_ms": prof.io_kv * 1e3,
                        "c_h_ms": prof.c_h * 1e3, "c_token_ms": prof.c_token * 1e3},
           "strategies": {}, "saving": {}}

    def one(trace, strategy, saving=H.SavingMode.TWO_STAGE, plan_=None):
        store = H.StorageManager(H.DevicePool(a.arenas), buffer_capacity_bytes=1 << 30)
        t0 = time.perf_counter()
        m = H.run(trace, w, store, H.RunOptions(strategy=strategy, saving=saving,
                                                hcache_plan=plan_ or plan))
        wall = time.perf_counter() - t0
        store.close()
        return {"ttft_p50_s": m.ttft_p50, "ttft_p95_s": m.ttft_p95, "tbt_mean_s": m.tbt_mean,
                "tbt_p50_s": m.tbt_p50, "tbt_p95_s": m.tbt_p95,
                "restore_tokens_per_s": m.restore_tokens_per_s,
                "storage_bytes_per_token": m.storage_bytes_per_token,
                "busy_s": m.busy_s, "save_stall_s": m.save_stall_s,
                "persist_wait_s": m.persist_wait_s, "decode_steps": m.decode_steps,
                "backpressure_stalls": m.backpressure_stalls, "wall_s": wall,
                "per_request": [[r.history_tokens, round(r.restore_s * 1e3, 3), round(r.ttft_s * 1e3, 3)]
                                for r in m.per_request]}, m

    # warm-up (first-use costs: pools, tensor maps, attributes) outside the numbers
    warm = [H.Request(f"w{i}", 1, 0, [], list(range(1, 40)), 8, 0.0) for i in range(4)]
    one(warm, H.Strategy.HCACHE)
    ms = {}
    for name in ([] if a.skip_conv else a.strategies.split(",")):
        s = H.Strategy[name]
        out["strategies"][name], ms[s] = one(tr, s)
        print(name, json.dumps(out["strategies"][name]), flush=True)
    if H.Strategy.HCACHE in ms:
        print(H.report(list(ms.values())), flush=True)
        hc = out["strategies"]["HCACHE"]
        for name, r in out["strategies"].items():
            r["ttft_p50_vs_hcache"] = r["ttft_p50_s"] / hc["ttft_p50_s"] if hc["ttft_p50_s"] else None
    # long-context trace (PAPER L-Eval setting): every request restores a
    # 2K-6K-token context, so TTFT = restore + prompt prefill
    if a.long_sessions > 0:
        lp = H.TraceParams(n_sessions=a.long_sessions, ctx_min=2048, ctx_max=6144,
                           arrival_rate_per_s=0.5, vocab=vocab)
        ltr = H.gen_trace(H.TraceKind.LONG_CONTEXT, lp, a.seed)
        out["long_context"] = {"trace": vars(lp), "requests": len(ltr.requests),
                               "context_tokens": sum(len(r.context) for r in ltr.requests),
                               "strategies": {}}
        # plan for the long contexts: profiled at their mean length
        lprof = H.profile_hardware(w, int(np.mean([len(r.context) for r in ltr.requests])))
        lprof.n_layers = L
        lplan, _ = H.plan_three_way(lprof, L)
        out["long_context"]["plan"] = lplan.serialize()
        lms = {}
        for name in a.strategies.split(","):
            s = H.Strategy[name]
            out["long_context"]["strategies"][name], lms[s] = one(ltr, s, plan_=lplan)
            print("long", name, json.dumps(out["long_context"]["strategies"][name]), flush=True)
        if H.Strategy.HCACHE in lms:
            print(H.report(list(lms.values())), flush=True)
            hc = out["long_context"]["strategies"]["HCACHE"]
            for name, r in out["long_context"]["strategies"].items():
                r["ttft_p50_vs_hcache"] = r["ttft_p50_s"] / hc["ttft_p50_s"]
    if a.skip_saving:
        print(json.dumps(out))
        if a.out:
            with open(a.out, "w") as f:
                json.dump(out, f, indent=1)
        return
    # criterion 8 on the device (acceptance.cpp:340-381): decode batch of 16
    # first-round requests arriving together, no restores, so TBT differs only
    # by how the states are saved
    rng = np.random.default_rng(a.seed)
    sav = [H.Request(f"b{i}", 1, 0, [], [int(x) for x in rng.integers(0, vocab, 66)], 128, 0.0)
           for i in range(16)]
    out["saving"]["trace"] = "16 requests at t=0, prompt 66, budget 128, round 1"
    out["saving"]["IDEAL"], _ = one(sav, H.Strategy.IDEAL)
    for mode in (H.SavingMode.TWO_STAGE, H.SavingMode.DIRECT, H.SavingMode.OFF):
        out["saving"][mode.name], _ = one(sav, H.Strategy.HCACHE, mode)
    ideal = out["saving"]["IDEAL"]["tbt_mean_s"]
    out["saving"]["tbt_vs_ideal"] = {k: out["saving"][k]["tbt_mean_s"] / ideal
                                     for k in ("TWO_STAGE", "DIRECT", "OFF")}
    print("saving", json.dumps(out["saving"]["tbt_vs_ideal"]), flush=True)
    print(json.dumps(out))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
