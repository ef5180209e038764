"""Batched continuation forward (forward_tokens / decode_step,
proj/src/model.cpp:305-347) on the GPU: sequences that already hold a paged
cache append new tokens — a prompt after a restore, or one decode token per
sequence — in one hc_forward_batch call.

Oracle: in the reference, continuing from a cache is the same arithmetic as a
one-shot prefill of the whole sequence (causal attention reads only keys
<= position; every GEMM is row-independent), so the reference prefill of the
full token sequence is the expected K/V, layer inputs and next token of the
continuation. Tolerance: the recompute path's normwise bound
(test_recompute_gpu.RECOMPUTE_TOL); the next token must be a maximiser of the
oracle's logits up to that tolerance (bf16 weights can swap near-ties)."""
import numpy as np
import pytest

from hc_testutil import norm_err
from test_recompute_gpu import RECOMPUTE_TOL, build, oracle_prefill

pytestmark = pytest.mark.gpu

CFG = dict(n_layers=4, d_hidden=512, n_heads=8, d_ffn=2048, vocab_size=1024, max_seq=1024)
SEED = 1234


def _tokens(n, salt):
    return [(i * 11 + 1 + 7 * salt) % 1024 for i in range(n)]


def _logit_ok(oracle, cfg, ref_final_row, tok):
    from oracle import bf16_round
    flat = bf16_round(oracle.init_model(cfg.n_layers, cfg.d_hidden, cfg.d_ffn, cfg.vocab_size, SEED))
    emb = flat[: cfg.vocab_size * cfg.d_hidden].reshape(cfg.vocab_size, cfg.d_hidden)
    logits = emb.astype(np.float64) @ ref_final_row.astype(np.float64)
    scale = np.sqrt(np.mean(logits ** 2))
    return logits[tok] >= logits.max() - RECOMPUTE_TOL * scale


def _run(oracle, prefix_lens, new_lens, page=64):
    """Prefill each sequence's prefix (hc_prefill), then append new_lens[s]
    tokens to every sequence in ONE batched forward; compare with the oracle
    prefill of prefix+new."""
    import ctypes as C

    import torch
    from paper_2410_05004_b200 import hcache as H
    from paper_2410_05004_b200.capi import check, lib
    cfg, w = build(CFG, SEED)
    B = len(prefix_lens)
    stride = max((a + b + page - 1) // page for a, b in zip(prefix_lens, new_lens))
    n_pages = B * stride
    kv = H.KvCache(cfg.n_layers, n_pages, page, w.d_kv)
    tables = torch.randperm(n_pages, generator=torch.Generator().manual_seed(5)).to(
        torch.int32).view(B, stride).cuda()
    full = [_tokens(a + b, s) for s, (a, b) in enumerate(zip(prefix_lens, new_lens))]
    stream = torch.cuda.current_stream().cuda_stream
    for s, a in enumerate(prefix_lens):
        toks = torch.tensor(full[s][:a], dtype=torch.int32, device="cuda")
        nxt = C.c_int32(-1)
        check(lib().hc_prefill(w._h, toks.data_ptr(), a, C.byref(kv.desc), tables[s].data_ptr(),
                               None, C.byref(nxt), stream))
    new_toks = torch.tensor(sum((full[s][a:] for s, a in enumerate(prefix_lens)), []),
                            dtype=torch.int32, device="cuda")
    T = int(new_toks.numel())
    inputs = torch.empty((cfg.n_layers, T, cfg.d_hidden), dtype=torch.bfloat16, device="cuda")
    nxt = H.forward_batch(w, new_toks, new_lens, prefix_lens, kv, tables, inputs)
    torch.cuda.synchronize()
    off = np.concatenate([[0], np.cumsum(new_lens)])
    for s, (a, b) in enumerate(zip(prefix_lens, new_lens)):
        ref = oracle_prefill(oracle, cfg, SEED, full[s])
        for L in range(cfg.n_layers):
            k, v = kv.gather(L, tables[s], a + b)
            assert norm_err(k.float().cpu().numpy(), ref["k"][L]) < RECOMPUTE_TOL, (s, L)
            assert norm_err(v.float().cpu().numpy(), ref["v"][L]) < RECOMPUTE_TOL, (s, L)
            got = inputs[L, off[s]:off[s + 1]].float().cpu().numpy()
            assert norm_err(got, ref["inputs"][L][a:]) < RECOMPUTE_TOL, (s, L)
        tok = int(nxt[s].item())
        assert tok == ref["next_token"] or _logit_ok(oracle, cfg, ref["final"][-1], tok), s


def test_prompt_after_history_matches_oracle(cuda, oracle):
    """One sequence: 200 cached tokens, a 70-token prompt (admit's prefill)."""
    _run(oracle, [200], [70])


def test_decode_step_batch_matches_oracle(cuda, oracle):
    """Continuous-batching decode: one token for each of 5 sequences with
    ragged cache lengths (page-boundary cases 63, 64, 65 included)."""
    _run(oracle, [63, 64, 65, 130, 7], [1, 1, 1, 1, 1])


def test_mixed_ragged_continuation(cuda, oracle):
    """Ragged prompts of several query tiles over ragged histories."""
    _run(oracle, [1, 100, 257], [130, 3, 64])


def test_forward_batch_rejects_overflow(cuda):
    import torch
    from paper_2410_05004_b200 import hcache as H
    cfg, w = build(CFG, SEED)
    kv = H.KvCache(cfg.n_layers, 4, 64, w.d_kv)
    tables = torch.arange(4, dtype=torch.int32, device="cuda").view(1, 4)
    toks = torch.zeros(2, dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError):  # beyond the page-table row
        H.forward_batch(w, toks, [2], [255], kv, tables)
    with pytest.raises(ValueError):  # beyond max_seq
        H.forward_batch(w, toks, [2], [1023], kv, torch.zeros((1, 16), dtype=torch.int32,
                                                                device="cuda"))


def test_kv_gather_rows_roundtrip(cuda):
    """hc_kv_gather_rows is the inverse of hc_kv_scatter_to_pages (bit-exact)."""
    import torch
    from paper_2410_05004_b200 import hcache as H
    kv = H.KvCache(2, 6, 64, 256)
    table = torch.tensor([4, 1, 5, 0, 2, 3], dtype=torch.int32, device="cuda")
    for L in range(2):
        kv.k[L].copy_(torch.randn_like(kv.k[L], dtype=torch.float32).bfloat16())
        kv.v[L].copy_(torch.randn_like(kv.v[L], dtype=torch.float32).bfloat16())
    rows = H.kv_gather_rows(kv, 1, table, 37, 200)
    k, v = kv.gather(1, table, 237)
    torch.cuda.synchronize()
    assert torch.equal(rows[:, :256], k[37:]) and torch.equal(rows[:, 256:], v[37:])
