"""CPU reference values for the benchmarked restore -- TEST INFRASTRUCTURE.

The bench (``bench.py``) and the GPU tests build their synthetic model with
``hc_fill_symmetric`` (the reference ``Rng::symmetric`` stream,
model.cpp:17-31) under fixed seeds; this module regenerates the same values
on the CPU (bf16-rounded, as the device stores them) and runs the oracle on
them, so a restore executed on the GPU can be checked after the fact:

* HIDDEN layers: ``project_hidden_to_kv`` (model.cpp:219-235) on a token
  slice ``[s, s+m)`` at ``start_pos = s`` (rows are independent);
* RECOMPUTE layers: ``prefill_layers`` (model.cpp:349-356) of the first m
  tokens -- causal, so rows ``[0, m)`` of a longer context's recomputed K/V
  depend on those tokens only -- walked layer by layer with
  ``Oracle.block_forward`` (the full weight set never materialises).

Only tests/ and bench.py's parity check import this; the product path never
does.
"""
from __future__ import annotations

import numpy as np

from . import Oracle

# seeds of the bench's synthetic model (bench.py run_ours): weights are
# symmetric(bound = 1/sqrt(d)) draws from offset 0 of seed BASE + layer
SEED_EMB = 99
SEED_WKV = 1234
SEED_WQ = 5000
SEED_WO = 6000
SEED_FC1 = 7000
SEED_FC2 = 8000
SEED_HIDDEN = 7
HIDDEN_BOUND = 1.7320508


def w_bound(d):
    return float(np.float32(1) / np.sqrt(np.float32(d)))


def sym(o: Oracle, n, seed, offset, bound):
    return o.symmetric_bf16(n, seed, offset, bound)


def layer_wkv(o: Oracle, layer, d, d_kv):
    full = sym(o, 2 * d_kv * d, SEED_WKV + layer, 0, w_bound(d)).reshape(2 * d_kv, d)
    return full[:d_kv], full[d_kv:]


def layer_full(o: Oracle, layer, d, d_ffn):
    b = w_bound(d)
    wk, wv = layer_wkv(o, layer, d, d)
    return dict(wq=sym(o, d * d, SEED_WQ + layer, 0, b).reshape(d, d), wk=wk, wv=wv,
                wo=sym(o, d * d, SEED_WO + layer, 0, b).reshape(d, d),
                fc1=sym(o, d_ffn * d, SEED_FC1 + layer, 0, b).reshape(d_ffn, d),
                fc2=sym(o, d * d_ffn, SEED_FC2 + layer, 0, b).reshape(d, d_ffn))


def embedding_rows(o: Oracle, tokens, d):
    """Rows of the (vocab x d) embedding for `tokens` (bf16 values)."""
    b = w_bound(d)
    return np.stack([sym(o, d, SEED_EMB, int(t) * d, b) for t in tokens]).astype(np.float32)


def hidden_rows(o: Oracle, layer, n, d, s, m):
    """Rows [s, s+m) of layer `layer` of the bench's (L, n, d) hidden tensor."""
    return sym(o, m * d, SEED_HIDDEN, (layer * n + s) * d, HIDDEN_BOUND).reshape(m, d)


def hidden_kv(o: Oracle, layer, n, d, d_kv, n_kv_heads, s, m, rope=True, nthreads=None):
    """Reference K/V of the HIDDEN layer's token slice [s, s+m)."""
    wk, wv = layer_wkv(o, layer, d, d_kv)
    return o.project(hidden_rows(o, layer, n, d, s, m), wk, wv, n_kv_heads, s, True, rope,
                     nthreads=nthreads)


def max_rel_err(g, r, tau_frac=1e-2):
    """North-star metric: max |g - r| / max(|r|, tau), tau = tau_frac rms(r)."""
    g = np.asarray(g, np.float64)
    r = np.asarray(r, np.float64)
    if not r.size:
        return 0.0
    tau = tau_frac * np.sqrt(np.mean(r * r))
    return float(np.max(np.abs(g - r) / np.maximum(np.abs(r), tau)))


def norm_err(g, r):
    """max |g - r| / rms(r) (the stated recompute metric)."""
    g = np.asarray(g, np.float64)
    r = np.asarray(r, np.float64)
    if not r.size:
        return 0.0
    return float(np.max(np.abs(g - r)) / max(np.sqrt(np.mean(r * r)), 1e-30))


def recompute_kv(o: Oracle, d, heads, d_ffn, tokens, n_layers, rope=True, nthreads=None):
    """Reference K/V of layers [0, n_layers) recomputed from `tokens`
    (prefill_layers at positions 0..m-1); a list of (K, V) float32."""
    cfg = dict(d_hidden=d, n_heads=heads, d_ffn=d_ffn, rope=int(rope))
    x = np.ascontiguousarray(embedding_rows(o, tokens, d))
    out = []
    for layer in range(n_layers):
        out.append(o.block_forward(cfg, layer_full(o, layer, d, d_ffn), x, nthreads=nthreads))
    return out
