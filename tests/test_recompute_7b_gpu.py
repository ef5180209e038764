"""RECOMPUTE layers at the benchmarked shape (Llama-2-7B, d=4096,
d_ffn=11008, 32 heads): the GPU prefill (K6) of all 32 layers -- the bench
plan recomputes the first 8 -- against the oracle's fp32 prefill_layers
(model.cpp:349-356), layer by layer, elementwise.

The GPU runs a 1024-token context; by causality rows [0, m) of every layer's
K/V depend only on the first m tokens, so the oracle runs just those (its
fp32 prefill of 32 such layers takes seconds, the whole context would take
hours). The weights are the bench's synthetic model (oracle/parity.py seeds).

Stated tolerance for recomputed K/V: K6 computes with
bf16 operands (the layer input, attention P and output, FFN hidden state are
rounded to bf16 before each GEMM, fp32 accumulate, fp32 residual stream), so
its error is absolute-scale: max |g - r| / rms(r) <= RECOMPUTE_NORM_TOL.
Measured on B200: 1.4 % at layer 0 (K/V output rounding only) and 2.0-2.9 %
at every deeper layer -- flat with depth (no compounding over 32 layers), so
the planner needs no recompute-depth cap. The north-star elementwise metric
(|g - r| / max(|r|, 1e-2 rms(r)) <= 1e-2) holds for K/V projected from
hidden states, whose operands are the stored bf16 rows themselves; for
recomputed rows it is reported, not asserted (~1.5: bf16 rounding of a layer
input perturbs near-zero outputs by ~1 % of rms)."""
import os

import pytest

from hc_testutil import max_rel_err, norm_err

pytestmark = pytest.mark.gpu

RECOMPUTE_NORM_TOL = 5e-2
L_RE = int(os.environ.get("HC_TEST_RE_LAYERS", "32"))
D, HEADS, DFFN, VOCAB = 4096, 32, 11008, 32000


def dev_bench_model(n_layers, d, heads, d_ffn, vocab, max_seq=4096):
    """The bench's synthetic model on the GPU (hc_fill_symmetric, bf16)."""
    import torch
    from hc_testutil import dev_symmetric
    from oracle import parity as P
    from paper_2410_05004_b200 import hcache as H
    cfg = H.ModelConfig(n_layers=n_layers, d_hidden=d, n_heads=heads, d_ffn=d_ffn,
                        vocab_size=vocab, max_seq=max_seq)
    w = H.Weights(cfg)
    b = P.w_bound(d)
    keep = [dev_symmetric(vocab * d, P.SEED_EMB, 0, b).view(vocab, d)]
    w.set_embedding(keep[0])
    for layer in range(n_layers):
        # [W_q ; W_k ; W_v] in one allocation, as bench.py lays it out (fused Q/K/V GEMM)
        qkv = torch.empty((3 * d, d), dtype=torch.bfloat16, device="cuda")
        qkv[:d] = dev_symmetric(d * d, P.SEED_WQ + layer, 0, b).view(d, d)
        qkv[d:] = dev_symmetric(2 * d * d, P.SEED_WKV + layer, 0, b).view(2 * d, d)
        wq, wkv = qkv[:d], qkv[d:]
        wo = dev_symmetric(d * d, P.SEED_WO + layer, 0, b).view(d, d)
        fc1 = dev_symmetric(d_ffn * d, P.SEED_FC1 + layer, 0, b).view(d_ffn, d)
        fc2 = dev_symmetric(d * d_ffn, P.SEED_FC2 + layer, 0, b).view(d, d_ffn)
        w.set_layer_kv(layer, wkv)
        w.set_layer_full(layer, wq, wkv, wo, fc1, fc2)
        keep += [wkv, wq, wo, fc1, fc2]
    torch.cuda.synchronize()
    w._keep = keep
    return cfg, w


@pytest.mark.slow
def test_recompute_all_layers_7b_shape(cuda, oracle):
    import ctypes as C

    import torch
    from oracle import parity as P
    from paper_2410_05004_b200 import hcache as H
    from paper_2410_05004_b200.capi import check, lib
    n, m, page = 1024, 48, 64
    tokens = [(i * 11 + 1) % VOCAB for i in range(n)]
    cfg, w = dev_bench_model(L_RE, D, HEADS, DFFN, VOCAB)
    kv = H.KvCache(L_RE, n // page, page, D)
    table = torch.arange(n // page, dtype=torch.int32, device="cuda")
    toks = torch.tensor(tokens, dtype=torch.int32, device="cuda")
    check(lib().hc_prefill_layers(w._h, toks.data_ptr(), n, 0, L_RE, C.byref(kv.desc),
                                  table.data_ptr(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    ref = P.recompute_kv(oracle, D, HEADS, DFFN, tokens[:m], L_RE)
    rows = []
    for layer in range(L_RE):
        k, v = kv.gather(layer, table, m)
        k, v = k.float().cpu().numpy(), v.float().cpu().numpy()
        kr, vr = ref[layer]
        rows.append((layer, max_rel_err(k, kr), max_rel_err(v, vr), norm_err(k, kr),
                     norm_err(v, vr)))
    for r in rows:
        print("layer %d  K max_rel %.3e  V max_rel %.3e  (normwise K %.2e V %.2e)" % r)
    worst = max(max(r[3], r[4]) for r in rows)
    assert worst <= RECOMPUTE_NORM_TOL, rows
    # layer 0 reads the exact (bf16) embedding: only the K/V output rounding
    assert max(rows[0][1], rows[0][2]) <= 1e-2, rows[0]
