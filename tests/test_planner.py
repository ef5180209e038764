"""Scheduler + timeline through the C ABI: ports of proj/tests/test_planner.cpp,
the timeline arithmetic of proj/tests/test_restore.cpp (simulated clock),
acceptance criteria 4-7, and golden vectors from the reference."""
import math

import numpy as np
import pytest

from hc_testutil import golden
from paper_2410_05004_b200 import hcache as H

C, M = H.Complement, H.LayerMethod


def T(io_h, io_kv, c_h, c_token, n):
    return H.ProfiledTimings(io_h, io_kv, c_h, c_token, n)


def test_compute_heavy_takes_kv_offload():
    # test_planner.cpp:24-36
    t = T(0.26, 0.52, 0.28, 1.9, 32)
    p = H.plan(t)
    assert (p.l_h, p.l_o, p.complement) == (31, 1, C.KV_OFFLOAD)
    assert H.makespan(p, t) == pytest.approx(8.68, rel=1e-12)
    assert p.layer_assignment[0] == M.HIDDEN and p.layer_assignment[-1] == M.KV_OFFLOAD


def test_io_heavy_takes_recompute_prefix():
    # test_planner.cpp:38-49
    t = T(0.5, 1.0, 0.3, 1.0, 48)
    p = H.plan(t)
    assert (p.l_h, p.l_o, p.complement) == (40, 8, C.RECOMPUTE)
    assert p.layer_assignment[0] == M.RECOMPUTE and p.layer_assignment[8] == M.HIDDEN
    assert H.makespan(p, t) == pytest.approx(20.0, rel=1e-12)


def test_balanced_needs_no_complement():
    t = T(0.4, 0.8, 0.4, 2.0, 16)
    p = H.plan(t)
    assert (p.l_h, p.l_o, p.complement) == (16, 0, C.NONE)
    assert H.makespan(p, t) == pytest.approx(16 * 0.4)


@pytest.mark.parametrize("seed,lo,hi,maxl", [(12345, 0.05, 2.0, 60), (777, 0.02, 3.0, 80)])
def test_closed_form_within_one_stage_of_brute_force(seed, lo, hi, maxl):
    # test_planner.cpp:60-79 and acceptance criterion 4
    rng = np.random.default_rng(seed)
    for _ in range(1000):
        io_h = float(rng.uniform(lo, hi))
        t = T(io_h, 2 * io_h, float(rng.uniform(lo, hi)), float(rng.uniform(lo, hi)),
              int(rng.integers(1, maxl + 1)))
        t.c_token = max(t.c_token, t.c_h)
        mc = H.makespan(H.plan(t), t)
        mb = H.makespan(H.brute_force_plan(t), t)
        assert mb <= mc + 1e-12
        assert mc <= mb + max(t.io_h, t.io_kv, t.c_h, t.c_token) + 1e-9


def test_more_expensive_kv_shifts_layers_to_hidden():
    prev = 0
    for io_kv in (0.3, 0.5, 0.8, 1.2, 2.0):
        p = H.plan(T(0.25, io_kv, 0.6, 2.0, 40))
        assert p.l_h >= prev
        prev = p.l_h


def test_serialize_parse_roundtrip():
    p = H.RestorationPlan.make(48, 40, C.RECOMPUTE)
    q = H.RestorationPlan.parse(p.serialize())
    assert (q.l_h, q.l_o, q.complement, q.layer_assignment) == \
        (p.l_h, p.l_o, p.complement, p.layer_assignment)
    with pytest.raises(H.capi.HCacheError):
        H.RestorationPlan.parse("garbage")
    m = H.RestorationPlan.make_mixed(3, 20, 5)
    assert H.RestorationPlan.parse(m.serialize()) == m
    assert m.layer_assignment[:3] == [M.RECOMPUTE] * 3 and m.layer_assignment[-5:] == [M.KV_OFFLOAD] * 5


def test_timings_validation_and_make_errors():
    with pytest.raises(ValueError):
        T(0, 1, 1, 1, 4).validate()
    with pytest.raises(ValueError):
        T(1, 1, 1, 1, 0).validate()
    T(1, 2, 1, 4, 4).validate()
    with pytest.raises(ValueError):
        H.RestorationPlan.make(4, 5, C.NONE)
    with pytest.raises(ValueError):
        H.RestorationPlan.make(4, 2, C.NONE)


def test_extreme_timings_clamp():
    assert H.plan(T(1e-6, 2e-6, 1e-6, 1.0, 32)).l_h == 32
    q = H.plan(T(1e-6, 2e-6, 10.0, 20.0, 32))
    assert q.complement == C.KV_OFFLOAD and q.l_h <= 1


def test_planner_equals_reference_goldens():
    for c in golden("planner.json"):
        io_h, io_kv, c_h, c_tok, L = c["t"]
        t = T(io_h, io_kv, c_h, c_tok, int(L))
        p = H.plan(t)
        assert [p.l_h, p.l_o, int(p.complement)] == c["plan"]
        assert H.makespan(p, t) == c["makespan"]
        assert p.serialize() == c["serialized"]
        b = H.brute_force_plan(t)
        assert [b.l_h, b.l_o, int(b.complement)] == c["brute"]
        assert H.makespan(b, t) == c["brute_makespan"]


def test_schedule_reproduction_criterion5():
    # acceptance.cpp:227-258: 31H+1KV and 40H+8RE, storage ratios
    p32 = H.plan(T(0.26, 0.52, 0.28, 1.9, 32))
    p48 = H.plan(T(0.5, 1.0, 0.3, 1.0, 48))
    assert (p32.l_h, p32.complement) == (31, C.KV_OFFLOAD)
    assert (p48.l_h, p48.complement) == (40, C.RECOMPUTE)

    def ratio(p):  # offload bytes / hcache bytes (cost_model.cpp:66-81)
        hc = sum({M.HIDDEN: 1, M.KV_OFFLOAD: 2, M.RECOMPUTE: 0}[m] for m in p.layer_assignment)
        return 2 * p.n_layers() / hc
    assert ratio(p32) == pytest.approx(256 / 132, rel=0.05)
    assert ratio(p48) == pytest.approx(672 / 280, rel=0.05)


# -------------------------------------------------------------- pipeline
def _jobs(plan, io_h, io_kv, c_h, c_tok, kv_only_last=False):
    """restore_simulated job list (restore.cpp:89-131) in compute order.
    kv_only_last: the B200 executor's prefix, whose last layer stops after
    its K/V projection (costed c_h, as hc_plan_three_way does)."""
    jobs = []
    last_re = max([L for L, m in enumerate(plan.layer_assignment) if m == M.RECOMPUTE],
                  default=-1)
    for method in (M.RECOMPUTE, M.HIDDEN, M.KV_OFFLOAD):
        for L, m in enumerate(plan.layer_assignment):
            if m != method:
                continue
            if m == M.HIDDEN:
                jobs.append(H.PipelineJob(L, io_h, c_h, True, True, "fetch_hidden", "project"))
            elif m == M.KV_OFFLOAD:
                jobs.append(H.PipelineJob(L, io_kv, 0, True, False, "fetch_kv", "project"))
            else:
                c = c_h if (kv_only_last and L == last_re) else c_tok
                jobs.append(H.PipelineJob(L, 0, c, False, True, "fetch", "recompute"))
    return jobs


KIO = 256.0 * 64 * 4 / 1e9  # test_restore.cpp:86


def test_balanced_all_hidden_finishes_in_n_plus_1_stages():
    # test_restore.cpp:90-102
    tl = H.simulate_pipeline(_jobs(H.RestorationPlan.make(4, 4, C.NONE), KIO, 2 * KIO, KIO, 0), 1)
    assert tl.total_s == pytest.approx(5 * KIO, rel=1e-9)
    assert tl.fill_s == pytest.approx(KIO, rel=1e-9)
    assert tl.bubble_fraction() < 0.25


def test_pure_kv_is_io_serial():
    # test_restore.cpp:104-114
    tl = H.simulate_pipeline(_jobs(H.RestorationPlan.make(4, 0, C.KV_OFFLOAD), KIO, 2 * KIO, KIO, 0), 1)
    assert tl.total_s == pytest.approx(8 * KIO, rel=1e-9)
    assert tl.bubble_fraction() == pytest.approx(1.0)


def test_io_twice_compute_leaves_predicted_bubble():
    # test_restore.cpp:116-126
    tl = H.simulate_pipeline(_jobs(H.RestorationPlan.make(4, 4, C.NONE), KIO, 2 * KIO, KIO / 2, 0), 1)
    assert tl.total_s == pytest.approx(4.5 * KIO, rel=1e-9)
    assert tl.bubble_fraction() == pytest.approx(4 / 9, rel=1e-9)


def test_recompute_prefix_events():
    tl = H.simulate_pipeline(_jobs(H.RestorationPlan.make(4, 1, C.RECOMPUTE), KIO, 2 * KIO, KIO, 5 * KIO), 1)
    assert sum(e.kind == "recompute" for e in tl.events) == 3


def test_pipeline_equals_reference_goldens():
    for c in golden("pipeline.json"):
        jobs = [H.PipelineJob(j[0], j[1], j[2], bool(j[3]), bool(j[4])) for j in c["jobs"]]
        tl = H.simulate_pipeline(jobs, c["depth"])
        assert [[int(e.lane), e.layer, e.start_s, e.end_s] for e in tl.events] == c["events"]
        assert tl.total_s == c["total"] and tl.fill_s == c["fill"]


def test_staging_depth_finding8():
    """the closed form's 25H+7RE plan for B200-like 7B timings is
    worse than all-hidden at depth 1; the three-way planner, costing the
    bounded pipeline, never returns a plan worse than all-hidden."""
    t = T(0.61e-3, 1.22e-3, 0.20e-3, 1.27e-3, 32)
    closed = H.plan(t)
    assert closed.complement == C.RECOMPUTE
    jobs = _jobs(closed, t.io_h, t.io_kv, t.c_h, t.c_token)
    at1 = H.simulate_pipeline(jobs, 1).total_s
    all_h = H.simulate_pipeline(_jobs(H.RestorationPlan.make(32, 32, C.NONE), t.io_h, t.io_kv,
                                      t.c_h, t.c_token), 1).total_s
    assert at1 > all_h
    for depth in (1, 4, 16, 32):
        p, ms = H.plan_three_way(t, depth)
        assert ms <= all_h + 1e-12
        assert ms == pytest.approx(H.simulate_pipeline(_jobs(p, t.io_h, t.io_kv, t.c_h, t.c_token,
                                                             True), depth).total_s)
    p32, ms32 = H.plan_three_way(t, 32)
    assert ms32 == pytest.approx(H.makespan(closed, t), rel=0.05) or ms32 < H.makespan(closed, t)


def test_three_way_considers_pure_kv_offload_for_gqa():
    """with GQA io_kv < io_h; the closed form never picks pure KV
    offload, the three-way planner does when it is faster."""
    t = T(1.0, 0.25, 0.05, 5.0, 80)
    closed = H.plan(t)
    p, ms = H.plan_three_way(t, 80)
    assert ms <= H.makespan(closed, t) + 1e-12
    # KV offload carries most layers; recomputing a few while the IO lane
    # streams KV balances the lanes (3 x 5.0 <= 77 x 0.25)
    assert p.l_kv >= 75 and ms <= 80 * 0.25 + 1e-12
    assert ms < H.makespan(closed, t)


def test_three_way_is_exhaustive_optimum():
    rng = np.random.default_rng(3)
    for _ in range(30):
        n = int(rng.integers(1, 12))
        t = T(*[float(x) for x in rng.uniform(0.1, 2.0, 4)], n)
        depth = int(rng.integers(1, 4))
        p, ms = H.plan_three_way(t, depth)
        best = math.inf
        for l_re in range(n + 1):
            for l_kv in range(n + 1 - l_re):
                q = H.RestorationPlan.make_mixed(l_re, n - l_re - l_kv, l_kv)
                best = min(best, H.simulate_pipeline(_jobs(q, t.io_h, t.io_kv, t.c_h, t.c_token,
                                                           True), depth).total_s)
        assert ms == pytest.approx(best, rel=1e-12)


def test_end_to_end_ratio_criterion6():
    # acceptance.cpp:260-291: A100-like profile, 1-4 devices, n=1024, d=4096
    n, d, eb, eff, L = 1024, 4096, 2, 312e12 * 0.5, 32
    for devices in range(1, 5):
        io_h = n * d * eb / (6.9e9 * devices)
        t = T(io_h, 2 * io_h, 4 * n * d * d / eff, (24 * n * d * d + n * n * d) / eff, L)
        r = L * t.io_kv / H.makespan(H.plan(t), t)
        assert 1.33 <= r <= 2.66
        if devices == 4:
            assert L * t.c_token / H.makespan(H.plan(t), t) >= 5.0


def test_token_split_balances_the_lanes():
    """B200 extension: splitting the first hidden layer between the recompute
    prefix and the IO lane never loses and, at a lane imbalance smaller than
    one layer, wins (7B-like timings)."""
    t = T(0.61e-3, 1.21e-3, 0.20e-3, 1.31e-3, 32)
    for l_re in (0, 6, 7, 8):
        p = H.RestorationPlan.make(32, 32 - l_re, C.RECOMPUTE if l_re else C.NONE)
        base = H.simulate_pipeline(_jobs(p, t.io_h, t.io_kv, t.c_h, t.c_token, True), 32).total_s
        s, ms = H.plan_token_split(t, p, 4096, 32)
        assert s % 64 == 0 and 0 <= s < 4096
        assert ms <= base + 1e-12
    pw, _ = H.plan_three_way(t, 32)  # the best whole-layer plan (8RE+24H)
    s, ms = H.plan_token_split(t, pw, 4096, 32)
    best_whole = min(H.simulate_pipeline(_jobs(H.RestorationPlan.make(32, 32 - r, C.RECOMPUTE if r
                                                                       else C.NONE),
                                               t.io_h, t.io_kv, t.c_h, t.c_token, True),
                                         32).total_s
                     for r in range(0, 12))
    assert s > 0 and ms < best_whole
    # no HIDDEN layer right after the prefix (KV-offload-only plan): no split
    pk = H.RestorationPlan.make(32, 0, C.KV_OFFLOAD)
    assert H.plan_token_split(t, pk, 4096, 32)[0] == 0


def _timeline(events, total):
    from paper_2410_05004_b200 import capi
    tc = capi.TimelineC()
    tc.n_events = len(events)
    tc.total_s = total
    for i, (lane, a, b) in enumerate(events):
        tc.events[i].lane, tc.events[i].layer = int(lane), i
        tc.events[i].start_s, tc.events[i].end_s = a, b
    return H.Timeline.from_c(tc)


def test_device_timeline_counts_overlapping_lanes_once():
    """The device executor overlaps compute events (K1 launches alternate two
    streams, statistics on a side stream): busy time is the union of the
    intervals, so it can never exceed the timeline's total."""
    ev = [(H.Lane.IO, 0.0, 4.0), (H.Lane.IO, 4.0, 8.0),
          (H.Lane.COMPUTE, 1.0, 3.0), (H.Lane.COMPUTE, 2.5, 5.0),  # overlap 0.5
          (H.Lane.COMPUTE, 4.5, 6.0), (H.Lane.COMPUTE, 7.0, 9.0)]
    tl = _timeline(ev, 9.0)
    assert tl.lane_busy(H.Lane.IO) == pytest.approx(8.0)
    assert tl.lane_busy(H.Lane.COMPUTE) == pytest.approx(7.0)  # [1,6] + [7,9]
    assert tl.bubble_fraction() == pytest.approx(1.0 / 9.0)
    py = H.Timeline(tl.events, tl.total_s, tl.fill_s)  # the Python-side union
    assert py.lane_busy(H.Lane.COMPUTE) == pytest.approx(7.0)
    assert tl.lane_busy(H.Lane.COMPUTE) <= tl.total_s


def test_serial_lanes_keep_the_reference_sum():
    ev = [(H.Lane.COMPUTE, 0.1, 0.3), (H.Lane.COMPUTE, 0.3, 0.7), (H.Lane.COMPUTE, 0.9, 1.0)]
    tl = _timeline(ev, 1.0)
    assert tl.lane_busy(H.Lane.COMPUTE) == (0.3 - 0.1) + (0.7 - 0.3) + (1.0 - 0.9)


def test_three_way_prices_the_prefix_last_layer_as_a_projection():
    """The executor stops the RECOMPUTE prefix's last layer after its K/V
    projection, so a one-layer prefix (layer 0 = embedding + K1, no fetch)
    costs c_h and the planner takes it whenever the IO lane is the longer
    one; c_token >= RECOMPUTE_UNAVAILABLE forbids any prefix."""
    t = T(0.61e-3, 1.21e-3, 0.20e-3, 1.31e-3, 32)
    p, ms = H.plan_three_way(t, 32)
    assert p.l_re >= 1
    one = H.RestorationPlan.make(32, 31, C.RECOMPUTE)
    assert H.simulate_pipeline(_jobs(one, t.io_h, t.io_kv, t.c_h, t.c_token, True), 32).total_s \
        < H.simulate_pipeline(_jobs(H.RestorationPlan.make(32, 32, C.NONE), t.io_h, t.io_kv,
                                    t.c_h, t.c_token), 32).total_s
    t.c_token = H.RECOMPUTE_UNAVAILABLE
    p, _ = H.plan_three_way(t, 32)
    assert p.l_re == 0


def test_timings_from_timeline_per_kind_busy_time():
    """hc_timings_from_timeline: per-kind union / count; the prefix's last
    (projection-only) recompute layer is left out of c_token; kinds without
    events keep the base value."""
    tl = _timeline([(H.Lane.COMPUTE, 0.0, 1.0), (H.Lane.COMPUTE, 1.0, 2.0),
                    (H.Lane.COMPUTE, 2.0, 2.2), (H.Lane.IO, 0.0, 0.5), (H.Lane.IO, 0.5, 1.1),
                    (H.Lane.COMPUTE, 2.2, 2.5), (H.Lane.COMPUTE, 2.4, 2.7)], 2.7)
    kinds = [3, 3, 3, 0, 0, 2, 2]  # recompute x3 (layers 0-2), fetch_hidden x2, project x2
    for i, k in enumerate(kinds):
        tl._c.events[i].kind = k
    base = T(9.0, 8.0, 7.0, 6.0, 7)
    t = H.timings_from_timeline(tl, base)
    assert t.c_token == pytest.approx(1.0)    # layers 0, 1 (layer 2 is the last)
    assert t.io_h == pytest.approx(0.55)
    assert t.c_h == pytest.approx(0.25)       # union 0.5 over two overlapping launches
    assert t.io_kv == 8.0 and t.n_layers == 7
