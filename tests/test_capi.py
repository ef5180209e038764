"""The C-ABI library: loads on a GPU-less host, exports every symbol the
header declares, and its compute entry points fail loudly without a B200
(no CPU fallback)."""
import ctypes as C

import pytest

from paper_2410_05004_b200 import capi
from paper_2410_05004_b200 import hcache as H


def test_library_exports_every_header_symbol():
    lib = capi.lib()
    syms = capi.header_symbols()
    assert len(syms) >= 50
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # every declared symbol has a ctypes prototype in the binding
    assert set(syms) <= set(capi._PROTOS), set(syms) - set(capi._PROTOS)


def test_abi_version_and_chunk_constants():
    assert capi.lib().hc_abi_version() == 1
    assert capi.lib().hc_chunk_tokens() == 64 == H.kChunkTokens
    assert capi.lib().hc_device_for_chunk(3, 5, 4) == (3 + 5) % 4


def test_struct_layouts_match_header_sizes():
    # plain-C layouts (x86-64 SysV): guards the ctypes mirror
    assert C.sizeof(capi.PlanC) == 6 * 4 + 256
    assert C.sizeof(capi.EventC) == 32
    assert C.sizeof(capi.TimelineC) == 24 + 32 * capi.HC_MAX_EVENTS
    assert C.sizeof(capi.KvPagesC) == 40
    assert C.sizeof(capi.PipelineJobC) == 40


def test_config_validation_and_hash_match_reference():
    cfg = H.ModelConfig(n_layers=2, d_hidden=64, n_heads=4, d_ffn=256, vocab_size=128,
                        elem_bytes=4)
    cfg.validate()
    for bad in (dict(n_heads=3), dict(elem_bytes=3), dict(n_layers=0)):
        c = H.ModelConfig(**{**cfg.__dict__, **bad})
        with pytest.raises(ValueError):
            c.validate()
    # FNV-1a over the reference's fields (model.cpp:152-168)
    h = 1469598103934665603
    for x in (2, 64, 4, 256, 128, 4096, 4, 1, 1):
        h = ((h ^ x) * 1099511628211) & (2 ** 64 - 1)
    assert cfg.hash() == h


def test_compute_entry_points_fail_loudly_without_gpu():
    if capi.lib().hc_device_count() > 0:
        pytest.skip("a GPU is present")
    cfg = H.ModelConfig(n_layers=1, d_hidden=64, n_heads=2, d_ffn=128)
    with pytest.raises(capi.CudaError):
        H.Weights(cfg)
    out = C.c_double()
    assert capi.lib().hc_measure_h2d(0, 1 << 20, 1, C.byref(out)) == capi.HC_ECUDA
    assert b"no CUDA device" in capi.lib().hc_last_error()
