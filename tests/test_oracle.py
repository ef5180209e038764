"""Pins the oracle restatement (oracle/hc_oracle.c) to the reference: against
the committed golden vectors (generated from the reference built from
source, oracle/make_golden.py) and, where oracle/_ref exists, directly."""
import numpy as np
import pytest

from hc_testutil import golden
from oracle import bf16_round


def hexfnv(oracle, a):
    return format(oracle.fnv1a(np.ascontiguousarray(a)), "016x")


def test_init_model_and_prefill_match_golden(oracle):
    for case in golden("model.json")["prefill"]:
        cfg = dict(case["cfg"])
        w = oracle.init_model(cfg["n_layers"], cfg["d_hidden"], cfg["d_ffn"], cfg["vocab_size"],
                              case["seed"])
        assert hexfnv(oracle, w) == case["weights_fnv"]
        pr = oracle.prefill(cfg, w, np.array(case["tokens"], np.int32), nthreads=4)
        assert hexfnv(oracle, pr["inputs"]) == case["inputs_fnv"]
        assert hexfnv(oracle, pr["k"]) == case["k_fnv"]
        assert hexfnv(oracle, pr["v"]) == case["v_fnv"]
        assert hexfnv(oracle, pr["final"]) == case["final_fnv"]
        assert pr["next_token"] == case["next_token"]


def test_prefill_layers_prefix_matches_golden(oracle):
    g = golden("model.json")["prefill_layers"]
    cfg = g["cfg"]
    w = oracle.init_model(cfg["n_layers"], cfg["d_hidden"], cfg["d_ffn"], cfg["vocab_size"],
                          g["seed"])
    k, v = oracle.prefill_layers(cfg, w, np.array(g["tokens"], np.int32), g["lb"], g["le"])
    assert hexfnv(oracle, k[: g["le"]]) == g["k_fnv"]
    assert hexfnv(oracle, v[: g["le"]]) == g["v_fnv"]


def test_projection_matches_golden(oracle):
    for c in golden("project.json"):
        n, d, dkv = c["n"], c["d"], c["d_kv"]
        h = bf16_round(oracle.symmetric(n * d, 100 + c["seed"], 0, 1.7320508).reshape(n, d))
        wk = bf16_round(oracle.symmetric(dkv * d, 1234 + c["seed"], 0, 1 / np.sqrt(d))).reshape(dkv, d)
        wv = bf16_round(oracle.symmetric(dkv * d, 1234 + c["seed"], dkv * d, 1 / np.sqrt(d))).reshape(dkv, d)
        k, v = oracle.project(h, wk, wv, c["heads"], c["start"], bool(c["norm"]), bool(c["rope"]))
        assert hexfnv(oracle, k) == c["k_fnv"], c
        assert hexfnv(oracle, v) == c["v_fnv"], c


def test_rope_table_matches_reference_coefficients(oracle):
    for c in golden("rope.json"):
        cos, sin = oracle.rope_table(c["n_pos"], c["d_head"])
        assert hexfnv(oracle, cos) == c["cos_fnv"]
        assert hexfnv(oracle, sin) == c["sin_fnv"]


def test_planner_matches_golden(oracle):
    for c in golden("planner.json"):
        io_h, io_kv, c_h, c_tok, L = c["t"]
        (lh, lo, comp), ms = oracle.plan(io_h, io_kv, c_h, c_tok, int(L))
        assert [lh, lo, comp] == c["plan"] and ms == c["makespan"]
        (lh, lo, comp), ms = oracle.plan(io_h, io_kv, c_h, c_tok, int(L), brute=True)
        assert [lh, lo, comp] == c["brute"] and ms == c["brute_makespan"]


def test_pipeline_matches_golden(oracle):
    for c in golden("pipeline.json"):
        jobs = [tuple(j) for j in c["jobs"]]
        ev, total, fill = oracle.simulate_pipeline(jobs, c["depth"])
        assert [list(e) for e in ev] == c["events"]
        assert total == c["total"] and fill == c["fill"]


def test_chunk_placement_matches_golden(oracle):
    for c in golden("storage.json"):
        for L, row in enumerate(c["placement"]):
            assert [oracle.device_for_chunk(L, ci, c["devices"]) for ci in range(len(row))] == row
            assert oracle.num_chunks(c["n"]) == len(row)


def test_trace_lengths_match_golden(oracle):
    g = golden("trace.json")
    hist = oracle.conversation_history(g["n_sessions"], g["rounds"], g["seed"])
    assert hist.tolist() == g["history"]
    # config 4: the 32 round-4 requests restore sum(n) = 44,145 tokens
    assert int(hist[3::4].sum()) == 44145


def test_fp16_codec_matches_golden(oracle):
    g = golden("fp16.json")
    assert [int(oracle.lib.hco_float_to_half(v)) for v in g["values"]] == g["encoded"]
    dec = [oracle.lib.hco_half_to_float(h) for h in range(0, 65536, 97)]
    np.testing.assert_array_equal(np.array(dec, np.float32), np.array(g["decode_every_97"], np.float32))


# ---------------------------------------------------- direct vs the reference
def test_oracle_equals_reference_random(oracle, reference):
    rng = np.random.default_rng(5)
    for _ in range(6):
        n, heads = int(rng.integers(1, 80)), int(rng.choice([1, 2, 4]))
        dh = int(rng.choice([2, 16, 64]))
        d = int(rng.choice([32, 96, 128]))
        h = rng.standard_normal((n, d)).astype(np.float32)
        wk = rng.uniform(-.1, .1, (heads * dh, d)).astype(np.float32)
        wv = rng.uniform(-.1, .1, (heads * dh, d)).astype(np.float32)
        start = int(rng.integers(0, 5000))
        for norm in (True, False):
            for rope in (True, False):
                ko, vo = oracle.project(h, wk, wv, heads, start, norm, rope)
                kr, vr = reference.project(h, wk, wv, heads, start, norm, rope)
                np.testing.assert_array_equal(ko, kr)
                np.testing.assert_array_equal(vo, vr)


def test_bf16_round_is_rne(oracle):
    x = np.array([1.0, 1.00390625, 1.005859375, -3.3e38, 1e-40, np.inf, 3.14159], np.float32)
    got = bf16_round(x)
    want = np.array([oracle.lib.hco_bf16_to_float(oracle.lib.hco_float_to_bf16(float(v)))
                     for v in x], np.float32)
    np.testing.assert_array_equal(got, want)
    assert got[1] == np.float32(1.0)          # tie -> even
    assert got[2] == np.float32(1.0078125)    # above half -> up


@pytest.mark.parametrize("n", [1, 7, 64, 128])
def test_projection_is_lossless_vs_prefill(oracle, n):
    """test_model.cpp:162-178: restore from H_L == prefill KV exactly."""
    cfg = dict(n_layers=2, d_hidden=64, n_heads=4, d_ffn=256, vocab_size=128)
    w = oracle.init_model(2, 64, 256, 128, 11)
    toks = np.array([(i * 7 + 3) % 128 for i in range(n)], np.int32)
    pr = oracle.prefill(cfg, w, toks)
    _, layers = oracle.split_weights(w, 2, 64, 256, 128)
    for L in range(2):
        k, v = oracle.project(pr["inputs"][L], layers[L]["wk"], layers[L]["wv"], 4)
        np.testing.assert_array_equal(k, pr["k"][L])
        np.testing.assert_array_equal(v, pr["v"][L])
