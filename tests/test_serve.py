"""Serving-loop host logic on CPU: the trace generator (trace.cpp:55-100)
against the reference's own outputs (golden vectors from the reference built
from source, oracle/make_golden.py), the report format (harness.cpp:492-525)
and argument validation of hc_serve_run (no GPU work)."""
import ctypes as C

import numpy as np
import pytest

from hc_testutil import golden


def _fnv(tokens):
    h = 1469598103934665603
    for b in np.asarray(tokens, np.int32).tobytes():
        h ^= b
        h = (h * 1099511628211) & ((1 << 64) - 1)
    return h


@pytest.mark.parametrize("case", range(3))
def test_gen_trace_matches_reference(case):
    from paper_2410_05004_b200 import hcache as H
    g = golden("trace.json")["full"][case]
    params = H.TraceParams(n_sessions=g["n_sessions"], rounds=g["rounds"])
    tr = H.gen_trace(H.TraceKind(g["kind"]), params, g["seed"])
    assert len(tr.requests) == len(g["meta"])
    for r, meta, arr, fnv in zip(tr.requests, g["meta"], g["arrival"], g["token_fnv"]):
        assert [int(r.session_id[4:]), r.round, r.history_tokens, len(r.context), len(r.prompt),
                r.output_budget] == meta
        assert r.arrival_s == arr  # bit-exact double
        assert _fnv(list(r.context) + list(r.prompt)) == int(fnv)


def test_gen_trace_history_golden():
    """Config 4's request lengths: sum of round-4 histories = 44,145."""
    from paper_2410_05004_b200 import hcache as H
    g = golden("trace.json")
    tr = H.gen_trace(H.TraceKind.CONVERSATION, H.TraceParams(n_sessions=32, rounds=4), 7)
    by = {(r.session_id, r.round): r.history_tokens for r in tr.requests}
    hist = [by[(f"sess{s}", rd)] for s in range(32) for rd in range(1, 5)]
    assert hist == g["history"]
    assert sum(hist[3::4]) == 44145


def test_gen_trace_live_reference(reference):
    from paper_2410_05004_b200 import hcache as H
    meta, arr, hsh = reference.gen_trace(0, 9, 2, 1234)
    tr = H.gen_trace(H.TraceKind.CONVERSATION, H.TraceParams(n_sessions=9, rounds=2), 1234)
    assert [r.arrival_s for r in tr.requests] == arr.tolist()
    assert [_fnv(r.prompt) for r in tr.requests] == [int(h) for h in hsh]


def test_trace_params_validate():
    from paper_2410_05004_b200 import hcache as H
    for bad in (dict(n_sessions=0), dict(mean_input=0.5), dict(arrival_rate_per_s=0),
                dict(ctx_min=10, ctx_max=5), dict(round_gap_s=-1)):
        with pytest.raises(ValueError):
            H.TraceParams(**bad).validate()


def test_report_layout():
    from paper_2410_05004_b200 import hcache as H
    m1 = H.Metrics(H.Strategy.HCACHE, [], [], ttft_p50=0.5)
    m2 = H.Metrics(H.Strategy.RECOMPUTE, [], [], ttft_p50=1.5)
    txt = H.report([m1, m2])
    assert txt.splitlines()[0].startswith("strategy")
    assert txt.splitlines()[2].rstrip().endswith("3.00")
    csv = H.report([m1, m2], csv=True).splitlines()
    assert csv[0].split(",")[-1] == "ttft_vs_hcache" and csv[2].split(",")[-1] == "3.0"


def test_serve_run_rejects_null_arguments():
    from paper_2410_05004_b200 import capi
    from paper_2410_05004_b200.capi import lib
    m = capi.ServeMetricsC()
    per = (capi.RequestMetricsC * 1)()
    o = capi.ServeOptsC()
    assert lib().hc_serve_run(None, None, None, 0, C.byref(o), per, None, C.byref(m), None) == 1


def test_metrics_csv_roundtrip_and_aggregates():
    """Metrics::to_csv / from_csv (harness.cpp:153-187) and the aggregates of
    finalize_aggregates (harness.cpp:133-151)."""
    from paper_2410_05004_b200 import hcache as H
    per = [H.RequestMetrics("s0", 1, 0.5, 0, 0.0, 0.25, 0.01, 5),
           H.RequestMetrics("s1", 2, 1.0, 300, 0.02, 0.125, 0.03, 3),
           H.RequestMetrics("s2", 1, 1.5, 100, 0.01, 0.5, 0.0, 1)]
    m = H.Metrics(H.Strategy.HCACHE, per, [])
    back = H.metrics_from_csv(H.metrics_to_csv(m))
    assert back.strategy == H.Strategy.HCACHE and back.per_request == per
    assert back.ttft_p50 == 0.25 and back.ttft_p95 == 0.25 + 0.9 * 0.25
    assert back.tbt_mean == 0.02  # the generated == 1 request is excluded
    assert back.restore_tokens_per_s == 400 / 0.03
    with pytest.raises(RuntimeError):
        H.metrics_from_csv("a,b,c\n")
