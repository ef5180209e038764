"""Shared helpers for the parity tests: seeded synthetic data generated on
the GPU by the library (hc_fill_symmetric) and element-for-element on the CPU
by the oracle, plus the tolerance metrics the north star states."""
from __future__ import annotations

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# North star: bf16 inputs, fp32 accumulate, max relative error <= 1e-2, with
# relative error |g - r| / max(|r|, tau), tau = TAU_FRAC * rms(r).
REL_TOL = 1e-2
TAU_FRAC = 1e-2
# fp32-output projection: normwise max|g - r| / rms(r) (accumulation order only)
F32_NORM_TOL = 2e-4

H_SEED = 7
H_BOUND = float(np.float32(np.sqrt(3.0)))  # unit variance hidden states
W_SEED = 1234


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)["data"]


def max_rel_err(g, r, tau_frac=TAU_FRAC):
    g = np.asarray(g, np.float64)
    r = np.asarray(r, np.float64)
    tau = tau_frac * np.sqrt(np.mean(r * r)) if r.size else 0.0
    return float(np.max(np.abs(g - r) / np.maximum(np.abs(r), tau))) if r.size else 0.0


def norm_err(g, r):
    g = np.asarray(g, np.float64)
    r = np.asarray(r, np.float64)
    return float(np.max(np.abs(g - r)) / max(np.sqrt(np.mean(r * r)), 1e-30)) if r.size else 0.0


def w_bound(d):
    return float(np.float32(1.0) / np.sqrt(np.float32(d)))


# ---------------------------------------------------------------- CPU side
def cpu_hidden(oracle, n_rows, d, seed=H_SEED, row0=0):
    """Rows [row0, row0+n_rows) of the synthetic bf16 hidden matrix."""
    from oracle import bf16_round
    return bf16_round(oracle.symmetric(n_rows * d, seed, row0 * d, H_BOUND)).reshape(n_rows, d)


def cpu_wkv(oracle, d, d_kv_all, layer, head_begin=0, head_count=None, d_head=None):
    """(W_k, W_v) rows of the synthetic layer weights: [W_k(all); W_v(all)]
    = symmetric(2*d_kv_all*d, seed W_SEED+layer); slice local heads."""
    from oracle import bf16_round
    full = bf16_round(oracle.symmetric(2 * d_kv_all * d, W_SEED + layer, 0, w_bound(d)))
    full = full.reshape(2 * d_kv_all, d)
    wk, wv = full[:d_kv_all], full[d_kv_all:]
    if head_count is not None:
        a, b = head_begin * d_head, (head_begin + head_count) * d_head
        wk, wv = wk[a:b], wv[a:b]
    return np.ascontiguousarray(wk), np.ascontiguousarray(wv)


# ---------------------------------------------------------------- GPU side
def dev_symmetric(n, seed, offset, bound, dtype=None):
    import ctypes as C

    import torch
    from paper_2410_05004_b200 import capi
    dtype = dtype or torch.bfloat16
    t = torch.empty(n, dtype=dtype, device="cuda")
    code = {torch.float32: 0, torch.bfloat16: 1, torch.float16: 2}[dtype]
    capi.check(capi.lib().hc_fill_symmetric(C.c_void_p(t.data_ptr()), n, seed, offset, bound,
                                            code, torch.cuda.current_stream().cuda_stream))
    return t


def dev_hidden(n_rows, d, seed=H_SEED, row0=0):
    return dev_symmetric(n_rows * d, seed, row0 * d, H_BOUND).view(n_rows, d)


def dev_wkv(d, d_kv_all, layer, head_begin=0, head_count=None, d_head=None):
    import torch
    full = dev_symmetric(2 * d_kv_all * d, W_SEED + layer, 0, w_bound(d)).view(2 * d_kv_all, d)
    if head_count is None:
        return full
    a, b = head_begin * d_head, (head_begin + head_count) * d_head
    return torch.cat([full[a:b], full[d_kv_all + a: d_kv_all + b]]).contiguous()
