"""Generates tests/golden/*.json from the reference compiled from source
(oracle/_ref/libhcache_ref.so). TEST INFRASTRUCTURE.

The reference ships no golden files; every golden value here
is produced by the unmodified reference routines on seeded inputs, so the
oracle restatement can be pinned on hosts where the reference is absent.

    python oracle/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import Oracle, Reference, bf16_round  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def fnv(arr) -> str:
    a = np.ascontiguousarray(arr)
    h = 1469598103934665603
    # vectorised FNV-1a would reorder; use the oracle's C routine for speed
    return format(Oracle().fnv1a(a), "016x") if a.nbytes else format(h, "016x")


def samples(arr, k=8, seed=0):
    a = np.asarray(arr).reshape(-1)
    idx = np.random.default_rng(seed).choice(a.size, size=min(k, a.size), replace=False)
    return {"idx": [int(i) for i in idx], "val_bits": [int(a[i].view(np.uint32)) for i in idx]}


def model_goldens(ref: Reference):
    cases = []
    for cfg, seed, n, stride in (
        (dict(n_layers=2, d_hidden=64, n_heads=4, d_ffn=256, vocab_size=128), 3, 33, 7),
        (dict(n_layers=1, d_hidden=64, n_heads=4, d_ffn=256, vocab_size=128, norm=0, rope=0), 5, 12, 7),
        (dict(n_layers=4, d_hidden=256, n_heads=8, d_ffn=1024, vocab_size=1024), 1234, 128, 11),
    ):
        toks = np.array([(i * stride + (3 if stride == 7 else 1)) % cfg["vocab_size"]
                         for i in range(n)], np.int32)
        w = ref.init_model(cfg["n_layers"], cfg["d_hidden"], cfg["n_heads"], cfg["d_ffn"],
                           cfg["vocab_size"], seed)
        pr = ref.prefill(cfg, seed, toks)
        cases.append({
            "cfg": cfg, "seed": seed, "tokens": toks.tolist(),
            "weights_fnv": fnv(w), "weights_samples": samples(w),
            "inputs_fnv": fnv(pr["inputs"]), "k_fnv": fnv(pr["k"]), "v_fnv": fnv(pr["v"]),
            "final_fnv": fnv(pr["final"]), "next_token": int(pr["next_token"]),
            "k_samples": samples(pr["k"]), "v_samples": samples(pr["v"]),
        })
    # prefill_layers prefix (the RECOMPUTE method, restore.cpp:96-99)
    cfg = dict(n_layers=4, d_hidden=64, n_heads=4, d_ffn=256, vocab_size=128)
    toks = np.array([(i * 13 + 5) % 128 for i in range(100)], np.int32)
    k, v = ref.prefill_layers(cfg, 10, toks, 0, 3)
    pl = {"cfg": cfg, "seed": 10, "tokens": toks.tolist(), "lb": 0, "le": 3,
          "k_fnv": fnv(k[:3]), "v_fnv": fnv(v[:3])}
    return {"prefill": cases, "prefill_layers": pl}


def project_goldens(ref: Reference, o: Oracle):
    cases = []
    for (n, d, d_kv, heads, start, norm, rope, seed) in (
        (50, 256, 64, 2, 17, 1, 1, 0),      # GQA-shaped (n_heads := n_kv_heads)
        (64, 128, 128, 4, 0, 1, 1, 1),
        (7, 96, 96, 3, 5, 0, 1, 2),
        (33, 64, 64, 4, 100, 1, 0, 3),
        (130, 512, 256, 2, 4000, 1, 1, 4),  # large positions
    ):
        h = bf16_round(o.symmetric(n * d, 100 + seed, 0, 1.7320508).reshape(n, d))
        wk = bf16_round(o.symmetric(d_kv * d, 1234 + seed, 0, 1 / np.sqrt(d)).reshape(d_kv, d))
        wv = bf16_round(o.symmetric(d_kv * d, 1234 + seed, d_kv * d, 1 / np.sqrt(d)).reshape(d_kv, d))
        kr, vr = ref.project(h, wk, wv, heads, start, bool(norm), bool(rope))
        cases.append({"n": n, "d": d, "d_kv": d_kv, "heads": heads, "start": start, "norm": norm,
                      "rope": rope, "seed": seed, "k_fnv": fnv(kr), "v_fnv": fnv(vr),
                      "k_samples": samples(kr), "v_samples": samples(vr)})
    return cases


def rope_goldens(ref: Reference):
    out = []
    for n_pos, d_head in ((4096, 128), (1024, 64), (32768, 128)):
        # coefficient table through the reference apply_rope: rotate e0 pairs
        # (a=1, b=0) -> (c, s) at every position
        rows = n_pos
        x = np.zeros((rows, d_head), np.float32)
        x[:, 0::2] = 1.0
        y = ref.apply_rope(x, 1, 0)
        cos, sin = y[:, 0::2], y[:, 1::2]
        out.append({"n_pos": n_pos, "d_head": d_head, "cos_fnv": fnv(np.ascontiguousarray(cos)),
                    "sin_fnv": fnv(np.ascontiguousarray(sin))})
    return out


def planner_goldens(ref: Reference):
    rng = np.random.default_rng(12345)
    cases = []
    for _ in range(300):
        io_h = float(rng.uniform(0.05, 2.0))
        io_kv = float(rng.choice([2 * io_h, rng.uniform(0.05, 2.0)]))
        c_h = float(rng.uniform(0.05, 2.0))
        c_tok = max(float(rng.uniform(0.05, 2.0)), c_h)
        L = int(rng.integers(1, 81))
        (lh, lo, comp), ms = ref.plan(io_h, io_kv, c_h, c_tok, L)
        (blh, blo, bcomp), bms = ref.plan(io_h, io_kv, c_h, c_tok, L, brute=True)
        cases.append({"t": [io_h, io_kv, c_h, c_tok, L], "plan": [lh, lo, comp], "makespan": ms,
                      "brute": [blh, blo, bcomp], "brute_makespan": bms,
                      "serialized": ref.plan_serialize(L, lh, comp)})
    return cases


def pipeline_goldens(ref: Reference):
    rng = np.random.default_rng(7)
    cases = []
    for _ in range(60):
        n = int(rng.integers(1, 24))
        jobs = []
        for j in range(n):
            kind = int(rng.integers(0, 3))  # 0 hidden, 1 kv, 2 recompute
            jobs.append((j, float(rng.uniform(0.1, 2.0)) if kind != 2 else 0.0,
                         float(rng.uniform(0.1, 2.0)) if kind != 1 else 0.0,
                         int(kind != 2), int(kind != 1)))
        depth = int(rng.integers(1, 5))
        ev, total, fill = ref.simulate_pipeline(jobs, depth)
        cases.append({"jobs": jobs, "depth": depth, "events": ev, "total": total, "fill": fill})
    return cases


def storage_goldens(ref: Reference):
    # criterion 9 style (acceptance.cpp:384-429): chunk counts / placement
    rng = np.random.default_rng(99)
    cases = []
    for _ in range(40):
        n = int(rng.integers(1, 2049))
        devs = int(rng.integers(1, 5))
        layers = int(rng.integers(1, 4))
        cases.append({"n": n, "devices": devs, "layers": layers,
                      "placement": [[ref.lib.ref_device_for_chunk(L, c, devs)
                                     for c in range((n + 63) // 64)] for L in range(layers)]})
    return cases


def trace_goldens(ref: Reference):
    out = {"n_sessions": 32, "rounds": 4, "seed": 7,
           "history": ref.conversation_history(32, 4, 7).tolist(), "full": []}
    # full gen_trace outputs (arrival order) for conversation and long-context
    for kind, n_s, rounds, seed in ((0, 32, 4, 7), (0, 5, 3, 11), (1, 6, 1, 3)):
        meta, arr, hsh = ref.gen_trace(kind, n_s, rounds, seed)
        out["full"].append({"kind": kind, "n_sessions": n_s, "rounds": rounds, "seed": seed,
                            "meta": meta.tolist(), "arrival": arr.tolist(),
                            "token_fnv": [str(int(h)) for h in hsh]})
    return out


def fp16_goldens(ref: Reference):
    vals = [0.0, -0.0, 1.0, -2.5, 65504.0, 65520.0, 1e-8, 6.1e-5, 5.96e-8, 3.0e-8, 1e5,
            0.333333, float("inf"), -float("inf"), 1.0009765625, 1.00048828125, 2.0 ** -24,
            2.0 ** -25, 1.5 * 2.0 ** -25]
    enc = [int(ref.lib.ref_float_to_half(v)) for v in vals]
    dec = [float(ref.lib.ref_half_to_float(h)) for h in range(0, 65536, 97)]
    return {"values": vals, "encoded": enc, "decode_every_97": dec}


def main():
    ref, o = Reference(), Oracle()
    os.makedirs(OUT, exist_ok=True)
    goldens = {
        "model.json": model_goldens(ref),
        "project.json": project_goldens(ref, o),
        "rope.json": rope_goldens(ref),
        "planner.json": planner_goldens(ref),
        "pipeline.json": pipeline_goldens(ref),
        "storage.json": storage_goldens(ref),
        "trace.json": trace_goldens(ref),
        "fp16.json": fp16_goldens(ref),
    }
    for name, data in goldens.items():
        with open(os.path.join(OUT, name), "w") as f:
            json.dump({"generator": "oracle/make_golden.py (reference built from source)",
                       "data": data}, f, indent=None, separators=(",", ":"))
        print("wrote", name, os.path.getsize(os.path.join(OUT, name)), "bytes")


if __name__ == "__main__":
    main()
