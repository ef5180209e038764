// planner.cpp -- the bubble-free restoration scheduler and the two-lane
// timeline (host C++; negligible cost).
//
// plan / makespan / brute_force_plan keep the reference's closed form and tie
// rules exactly (proj/src/planner.cpp:75-128) so its pinned schedules
// (31H+1KV, 40H+8RE) reproduce. The B200 extension hc_plan_three_way searches
// every (recompute prefix, hidden, KV suffix) split and costs each candidate
// with the bounded-staging pipeline the executor really runs
// (simulate_pipeline at prefetch_depth), fixing the unbounded-prefetch
// assumption the closed form makes and considering pure KV
// offload, which the closed form never picks when io_kv < io_h (GQA).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "common.h"

namespace hc {

namespace {

void check_timings(const hc_timings* t) {
  // ProfiledTimings::validate (planner.cpp:28-33)
  if (!t) fail(HC_EINVAL, "ProfiledTimings: null");
  if (t->io_h <= 0 || t->io_kv <= 0 || t->c_h <= 0 || t->c_token <= 0)
    fail(HC_EINVAL, "ProfiledTimings: nonpositive timing");
  if (t->n_layers < 1) fail(HC_EINVAL, "ProfiledTimings: n_layers < 1");
  if (t->n_layers > HC_MAX_LAYERS) fail(HC_EINVAL, "ProfiledTimings: too many layers");
}

void make_plan(int n_layers, int l_h, int complement, hc_plan* p) {
  // RestorationPlan::make (planner.cpp:34-51)
  if (n_layers < 1 || n_layers > HC_MAX_LAYERS) fail(HC_EINVAL, "plan: bad layer count");
  if (l_h < 0 || l_h > n_layers) fail(HC_EINVAL, "plan: l_h out of range");
  std::memset(p, 0, sizeof(*p));
  p->n_layers = n_layers;
  p->l_h = l_h;
  p->l_o = n_layers - l_h;
  if (p->l_o > 0 && complement == HC_COMPLEMENT_NONE)
    fail(HC_EINVAL, "plan: l_o > 0 needs a complement method");
  if (complement == HC_COMPLEMENT_MIXED) fail(HC_EINVAL, "plan: use hc_plan_make_mixed");
  p->complement = p->l_o == 0 ? HC_COMPLEMENT_NONE : complement;
  for (int i = 0; i < n_layers; ++i) p->layer_assignment[i] = HC_METHOD_HIDDEN;
  if (p->complement == HC_COMPLEMENT_RECOMPUTE) {
    p->l_re = p->l_o;
    for (int i = 0; i < p->l_o; ++i) p->layer_assignment[i] = HC_METHOD_RECOMPUTE;  // prefix
  } else if (p->complement == HC_COMPLEMENT_KV_OFFLOAD) {
    p->l_kv = p->l_o;
    for (int i = n_layers - p->l_o; i < n_layers; ++i)
      p->layer_assignment[i] = HC_METHOD_KV_OFFLOAD;  // suffix
  }
}

void make_mixed(int l_re, int l_h, int l_kv, hc_plan* p) {
  const int n = l_re + l_h + l_kv;
  if (l_re < 0 || l_h < 0 || l_kv < 0 || n < 1 || n > HC_MAX_LAYERS)
    fail(HC_EINVAL, "plan: bad three-way split");
  if (l_re == 0 || l_kv == 0) {
    // single complement: identical to the reference's representation
    make_plan(n, l_h, l_re ? HC_COMPLEMENT_RECOMPUTE
                           : (l_kv ? HC_COMPLEMENT_KV_OFFLOAD : HC_COMPLEMENT_NONE),
              p);
    return;
  }
  std::memset(p, 0, sizeof(*p));
  p->n_layers = n;
  p->l_h = l_h;
  p->l_o = l_re + l_kv;
  p->l_re = l_re;
  p->l_kv = l_kv;
  p->complement = HC_COMPLEMENT_MIXED;
  for (int i = 0; i < n; ++i)
    p->layer_assignment[i] = i < l_re ? HC_METHOD_RECOMPUTE
                                      : (i < l_re + l_h ? HC_METHOD_HIDDEN : HC_METHOD_KV_OFFLOAD);
}

double makespan_of(const hc_plan* p, const hc_timings* t) {
  // planner.cpp:92-107 (two lanes, unbounded prefetch)
  const double lh = p->l_h, lo = p->l_o;
  switch (p->complement) {
    case HC_COMPLEMENT_NONE:
      return std::max(t->c_h * lh, t->io_h * lh);
    case HC_COMPLEMENT_KV_OFFLOAD:
      return std::max(t->c_h * lh, t->io_h * lh + t->io_kv * lo);
    case HC_COMPLEMENT_RECOMPUTE:
      return std::max(t->io_h * lh, t->c_token * lo + t->c_h * lh);
    default:
      return std::max(t->io_h * lh + t->io_kv * double(p->l_kv),
                      t->c_token * double(p->l_re) + t->c_h * lh);
  }
}

const char* comp_name(int c) {
  switch (c) {
    case HC_COMPLEMENT_NONE: return "NONE";
    case HC_COMPLEMENT_KV_OFFLOAD: return "KV_OFFLOAD";
    case HC_COMPLEMENT_RECOMPUTE: return "RECOMPUTE";
    default: return "MIXED";
  }
}

}  // namespace

// simulate_pipeline (pipeline.cpp:33-104): one job per restored layer in
// compute order; fetches issue in job order on the IO lane; a fetch feeding a
// compute stage waits for a staging buffer (prefetch_depth+1 of them).
void simulate(const hc_pipeline_job* jobs, int n, int depth, hc_timeline* tl) {
  if (depth < 1) fail(HC_EINVAL, "prefetch_depth < 1");
  if (n < 0 || 2 * n > HC_MAX_EVENTS) fail(HC_EINVAL, "simulate_pipeline: too many jobs");
  std::memset(tl, 0, sizeof(*tl));
  std::vector<int> io_order, staged_order, staged_rank(size_t(n), -1);
  for (int j = 0; j < n; ++j)
    if (jobs[j].has_io) io_order.push_back(j);
  for (int j : io_order)
    if (jobs[j].has_compute) staged_order.push_back(j);
  for (size_t r = 0; r < staged_order.size(); ++r) staged_rank[size_t(staged_order[r])] = int(r);
  std::vector<double> fetch_end(size_t(n), 0), compute_end(size_t(n), 0);
  std::vector<char> computed(size_t(n), 0);
  double io_free = 0, compute_free = 0;
  size_t next_io = 0;
  std::vector<hc_event> ev;
  auto issue_ready = [&] {
    while (next_io < io_order.size()) {
      const int j = io_order[next_io];
      double dep = 0;
      if (jobs[j].has_compute) {
        const int r = staged_rank[size_t(j)];
        if (r >= depth + 1) {
          const int blocker = staged_order[size_t(r - depth - 1)];
          if (!computed[size_t(blocker)]) return;
          dep = compute_end[size_t(blocker)];
        }
      }
      const double start = std::max(io_free, dep), end = start + jobs[j].io_s;
      ev.push_back(hc_event{HC_LANE_IO, jobs[j].layer, jobs[j].io_kind, 0, start, end});
      fetch_end[size_t(j)] = end;
      io_free = end;
      if (ev.size() == 1) tl->fill_s = end;
      ++next_io;
    }
  };
  issue_ready();
  for (int j = 0; j < n; ++j) {
    if (!jobs[j].has_compute) continue;
    const double start = std::max(compute_free, jobs[j].has_io ? fetch_end[size_t(j)] : 0.0);
    const double end = start + jobs[j].compute_s;
    ev.push_back(hc_event{HC_LANE_COMPUTE, jobs[j].layer, jobs[j].compute_kind, 0, start, end});
    compute_end[size_t(j)] = end;
    computed[size_t(j)] = 1;
    compute_free = end;
    issue_ready();
  }
  if (next_io != io_order.size()) fail(HC_ERUNTIME, "pipeline: unresolved fetch dependency");
  for (const auto& e : ev) tl->total_s = std::max(tl->total_s, e.end_s);
  std::stable_sort(ev.begin(), ev.end(),
                   [](const hc_event& a, const hc_event& b) { return a.start_s < b.start_s; });
  tl->n_events = int32_t(ev.size());
  std::copy(ev.begin(), ev.end(), tl->events);
}

// Jobs of a plan in the executor's compute order (restore.cpp:50-63):
// recompute prefix, hidden layers, KV suffix. The prefix's last layer costs
// a projection (c_h), not a block: the executor stops that layer after its
// K/V (the next layer is restored from its stored input), where the
// reference's prefill_layers runs the whole block (model.cpp:349-356).
std::vector<hc_pipeline_job> plan_jobs(const hc_plan* p, const hc_timings* t) {
  std::vector<hc_pipeline_job> jobs;
  int last_re = -1;
  for (int L = 0; L < p->n_layers; ++L)
    if (p->layer_assignment[L] == HC_METHOD_RECOMPUTE) last_re = L;
  auto add = [&](int method) {
    for (int L = 0; L < p->n_layers; ++L) {
      if (p->layer_assignment[L] != method) continue;
      hc_pipeline_job j{};
      j.layer = L;
      if (method == HC_METHOD_RECOMPUTE) {
        j.has_compute = 1;
        j.compute_s = L == last_re ? t->c_h : t->c_token;
        j.compute_kind = HC_EV_RECOMPUTE;
      } else if (method == HC_METHOD_HIDDEN) {
        j.has_io = j.has_compute = 1;
        j.io_s = t->io_h;
        j.io_kind = HC_EV_FETCH_HIDDEN;
        j.compute_s = t->c_h;
        j.compute_kind = HC_EV_PROJECT;
      } else {
        j.has_io = 1;
        j.io_s = t->io_kv;
        j.io_kind = HC_EV_FETCH_KV;
      }
      jobs.push_back(j);
    }
  };
  add(HC_METHOD_RECOMPUTE);
  add(HC_METHOD_HIDDEN);
  add(HC_METHOD_KV_OFFLOAD);
  return jobs;
}

std::string plan_serialize(const hc_plan* p) {
  char buf[160];
  if (p->complement == HC_COMPLEMENT_MIXED)
    std::snprintf(buf, sizeof buf, "l_h=%d l_o=%d complement=MIXED l_re=%d l_kv=%d", p->l_h,
                  p->l_o, p->l_re, p->l_kv);
  else
    std::snprintf(buf, sizeof buf, "l_h=%d l_o=%d complement=%s", p->l_h, p->l_o,
                  comp_name(p->complement));
  return buf;
}

void plan_parse(const char* rec, hc_plan* out) {
  // RestorationPlan::parse (planner.cpp:53-73)
  if (!rec) fail(HC_EINVAL, "RestorationPlan: null record");
  int lh = -1, lo = -1;
  char comp[32] = {0};
  if (std::sscanf(rec, "l_h=%d l_o=%d complement=%31s", &lh, &lo, comp) != 3)
    fail(HC_ERUNTIME, std::string("RestorationPlan: bad record: ") + rec);
  std::string c(comp);
  if (c == "MIXED") {
    int lre = -1, lkv = -1;
    const char* tail = std::strstr(rec, "l_re=");
    if (!tail || std::sscanf(tail, "l_re=%d l_kv=%d", &lre, &lkv) != 2 || lre + lkv != lo)
      fail(HC_ERUNTIME, std::string("RestorationPlan: bad record: ") + rec);
    make_mixed(lre, lh, lkv, out);
    return;
  }
  int cm;
  if (c == "NONE") cm = HC_COMPLEMENT_NONE;
  else if (c == "KV_OFFLOAD") cm = HC_COMPLEMENT_KV_OFFLOAD;
  else if (c == "RECOMPUTE") cm = HC_COMPLEMENT_RECOMPUTE;
  else fail(HC_ERUNTIME, "RestorationPlan: bad complement: " + c);
  if (lo > 0 && cm == HC_COMPLEMENT_NONE)
    fail(HC_ERUNTIME, "RestorationPlan: l_o > 0 with complement NONE");
  make_plan(lh + lo, lh, cm, out);
}

}  // namespace hc

using namespace hc;

extern "C" {

hc_status hc_timings_validate(const hc_timings* t) {
  return guard([&] { check_timings(t); });
}

hc_status hc_plan_make(int32_t n_layers, int32_t l_h, int32_t complement, hc_plan* out) {
  return guard([&] {
    if (!out) fail(HC_EINVAL, "plan: null out");
    make_plan(n_layers, l_h, complement, out);
  });
}

hc_status hc_plan_make_mixed(int32_t l_re, int32_t l_h, int32_t l_kv, hc_plan* out) {
  return guard([&] {
    if (!out) fail(HC_EINVAL, "plan: null out");
    make_mixed(l_re, l_h, l_kv, out);
  });
}

hc_status hc_plan_serialize(const hc_plan* p, char* buf, int32_t cap) {
  return guard([&] {
    if (!p || !buf || cap < 1) fail(HC_EINVAL, "plan_serialize: bad buffer");
    std::string s = plan_serialize(p);
    if (int32_t(s.size()) >= cap) fail(HC_EINVAL, "plan_serialize: buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

hc_status hc_plan_parse(const char* record, hc_plan* out) {
  return guard([&] {
    if (!out) fail(HC_EINVAL, "plan_parse: null out");
    plan_parse(record, out);
  });
}

hc_status hc_plan_closed_form(const hc_timings* t, hc_plan* out) {
  return guard([&] {
    // plan (planner.cpp:75-90)
    check_timings(t);
    if (!out) fail(HC_EINVAL, "plan: null out");
    const int n = t->n_layers;
    double lh_real;
    int comp;
    if (t->c_h > t->io_h) {
      comp = HC_COMPLEMENT_KV_OFFLOAD;
      lh_real = double(n) * t->io_kv / (t->io_kv + t->c_h - t->io_h);
    } else {
      comp = HC_COMPLEMENT_RECOMPUTE;
      lh_real = double(n) * t->c_token / (t->c_token + t->io_h - t->c_h);
    }
    int l_h = int(std::ceil(lh_real - 1e-12));
    l_h = std::max(0, std::min(n, l_h));
    make_plan(n, l_h, comp, out);
  });
}

hc_status hc_makespan(const hc_plan* p, const hc_timings* t, double* out) {
  return guard([&] {
    if (!p || !t || !out) fail(HC_EINVAL, "makespan: null argument");
    if (p->n_layers != t->n_layers)
      fail(HC_EINVAL, "makespan: plan/timings layer count mismatch");
    *out = makespan_of(p, t);
  });
}

hc_status hc_brute_force_plan(const hc_timings* t, hc_plan* out) {
  return guard([&] {
    // brute_force_plan (planner.cpp:109-128): strict improvement, or equal
    // cost with larger l_h
    check_timings(t);
    if (!out) fail(HC_EINVAL, "plan: null out");
    bool have = false;
    double best_cost = 0;
    hc_plan best{}, cand{};
    for (int lh = 0; lh <= t->n_layers; ++lh)
      for (int c : {HC_COMPLEMENT_KV_OFFLOAD, HC_COMPLEMENT_RECOMPUTE}) {
        make_plan(t->n_layers, lh, c, &cand);
        const double cost = makespan_of(&cand, t);
        if (!have || cost < best_cost || (cost == best_cost && cand.l_h > best.l_h)) {
          best = cand;
          best_cost = cost;
          have = true;
        }
      }
    *out = best;
  });
}

hc_status hc_plan_three_way(const hc_timings* t, int32_t prefetch_depth, hc_plan* out,
                            double* makespan_out) {
  return guard([&] {
    check_timings(t);
    if (!out) fail(HC_EINVAL, "plan: null out");
    if (prefetch_depth < 1) fail(HC_EINVAL, "prefetch_depth < 1");
    const int n = t->n_layers;
    bool have = false;
    double best_cost = 0;
    hc_plan best{}, cand{};
    hc_timeline* tl = new hc_timeline;
    // c_token >= HC_RECOMPUTE_UNAVAILABLE: no full block weights (or no
    // whole model on this GPU) -- no RECOMPUTE layers, not even the
    // projection-only first layer the cost model would otherwise price at c_h
    const int max_re = t->c_token >= HC_RECOMPUTE_UNAVAILABLE ? 0 : n;
    try {
      for (int l_re = 0; l_re <= max_re; ++l_re)
        for (int l_kv = 0; l_kv + l_re <= n; ++l_kv) {
          const int l_h = n - l_re - l_kv;
          make_mixed(l_re, l_h, l_kv, &cand);
          auto jobs = plan_jobs(&cand, t);
          simulate(jobs.data(), int(jobs.size()), prefetch_depth, tl);
          const double cost = tl->total_s;
          // ties: more hidden layers (less storage), then fewer recomputed
          const bool better =
              !have || cost < best_cost * (1 - 1e-12) ||
              (cost <= best_cost * (1 + 1e-12) &&
               (cand.l_h > best.l_h || (cand.l_h == best.l_h && cand.l_re < best.l_re)));
          if (better) {
            best = cand;
            best_cost = cost;
            have = true;
          }
        }
    } catch (...) {
      delete tl;
      throw;
    }
    delete tl;
    *out = best;
    if (makespan_out) *makespan_out = best_cost;
  });
}

hc_status hc_plan_token_split(const hc_timings* t, int32_t prefetch_depth, const hc_plan* plan,
                              int32_t n_tokens, int32_t* split_out, double* makespan_out) {
  return guard([&] {
    check_timings(t);
    if (!plan || !split_out) fail(HC_EINVAL, "plan_token_split: null argument");
    if (prefetch_depth < 1) fail(HC_EINVAL, "prefetch_depth < 1");
    if (n_tokens < 1) fail(HC_EINVAL, "plan_token_split: n_tokens < 1");
    if (plan->n_layers != t->n_layers) fail(HC_EINVAL, "plan_token_split: layer count mismatch");
    const auto base = plan_jobs(plan, t);
    // the first job after the recompute prefix, if it is the HIDDEN layer l_re
    size_t at = 0;
    while (at < base.size() && base[at].compute_kind == HC_EV_RECOMPUTE && !base[at].has_io) ++at;
    const bool ok = at < base.size() && base[at].io_kind == HC_EV_FETCH_HIDDEN &&
                    base[at].layer == int(at);
    hc_timeline* tl = new hc_timeline;
    int best_s = 0;
    double best = 0;
    try {
      simulate(base.data(), int(base.size()), prefetch_depth, tl);
      best = tl->total_s;
      // split s: the layer's first s tokens join the prefix (recompute cost
      // linear in s -- the attention part is sub-linear, so this errs high:
      // the previous layer's block for s rows + this layer's projection of
      // them), the rest is fetched and projected
      for (int sp = HC_CHUNK_TOKENS; ok && sp < n_tokens; sp += HC_CHUNK_TOKENS) {
        const double x = double(sp) / double(n_tokens);
        std::vector<hc_pipeline_job> jobs(base.begin(), base.begin() + long(at));
        hc_pipeline_job re{};
        re.layer = base[at].layer;
        re.has_compute = 1;
        re.compute_s = t->c_token * x;
        re.compute_kind = HC_EV_RECOMPUTE;
        jobs.push_back(re);
        hc_pipeline_job h = base[at];
        h.io_s *= 1.0 - x;
        h.compute_s *= 1.0 - x;
        jobs.push_back(h);
        jobs.insert(jobs.end(), base.begin() + long(at) + 1, base.end());
        simulate(jobs.data(), int(jobs.size()), prefetch_depth, tl);
        if (tl->total_s < best * (1 - 1e-9)) {
          best = tl->total_s;
          best_s = sp;
        }
      }
    } catch (...) {
      delete tl;
      throw;
    }
    delete tl;
    *split_out = best_s;
    if (makespan_out) *makespan_out = best;
  });
}

double hc_timeline_lane_busy(const hc_timeline* tl, int32_t lane) {
  // Timeline::lane_busy (pipeline.cpp:9-14) sums event durations: the
  // reference's lanes are strictly serial, so that is the time the lane was
  // busy. The device executor's compute lane is not (consecutive K1 launches
  // alternate two streams, row statistics run on a side stream), so busy time
  // is the length of the union of the lane's intervals -- identical to the
  // sum whenever events do not overlap (every simulated timeline).
  if (!tl) return 0;
  std::vector<std::pair<double, double>> iv;
  iv.reserve(size_t(std::max(0, tl->n_events)));
  for (int i = 0; i < tl->n_events; ++i)
    if (tl->events[i].lane == lane && tl->events[i].end_s > tl->events[i].start_s)
      iv.emplace_back(tl->events[i].start_s, tl->events[i].end_s);
  std::sort(iv.begin(), iv.end());
  double b = 0, cur_s = 0, cur_e = 0;
  bool open = false;
  for (const auto& [s, e] : iv) {
    if (open && s < cur_e) {
      cur_e = std::max(cur_e, e);
      continue;
    }
    if (open) b += cur_e - cur_s;
    cur_s = s;
    cur_e = e;
    open = true;
  }
  if (open) b += cur_e - cur_s;
  return b;
}

hc_status hc_timings_from_timeline(const hc_timeline* tl, hc_timings* io) {
  return guard([&] {
    if (!tl || !io) fail(HC_EINVAL, "timings_from_timeline: null argument");
    // the prefix's last layer stops after its K/V projection: not a block
    int last_re = -1, n_re = 0;
    for (int i = 0; i < tl->n_events; ++i)
      if (tl->events[i].kind == HC_EV_RECOMPUTE) {
        last_re = std::max(last_re, tl->events[i].layer);
        ++n_re;
      }
    // per kind: the union of its intervals / its event count -- the lane's
    // throughput for that kind (K1 launches on two streams overlap)
    auto per_event = [&](int kind, double* out) {
      std::vector<std::pair<double, double>> iv;
      for (int i = 0; i < tl->n_events; ++i) {
        const hc_event& e = tl->events[i];
        if (e.kind != kind || e.end_s <= e.start_s) continue;
        if (kind == HC_EV_RECOMPUTE && n_re > 1 && e.layer == last_re) continue;
        iv.emplace_back(e.start_s, e.end_s);
      }
      if (iv.empty()) return;
      std::sort(iv.begin(), iv.end());
      double b = 0, cs = iv[0].first, ce = iv[0].second;
      for (size_t k = 1; k < iv.size(); ++k) {
        if (iv[k].first < ce) {
          ce = std::max(ce, iv[k].second);
          continue;
        }
        b += ce - cs;
        cs = iv[k].first;
        ce = iv[k].second;
      }
      b += ce - cs;
      *out = b / double(iv.size());
    };
    per_event(HC_EV_FETCH_HIDDEN, &io->io_h);
    per_event(HC_EV_FETCH_KV, &io->io_kv);
    per_event(HC_EV_PROJECT, &io->c_h);
    if (n_re > 1) per_event(HC_EV_RECOMPUTE, &io->c_token);
  });
}

hc_status hc_timeline_bubble_fraction(const hc_timeline* tl, double* out) {
  return guard([&] {
    // Timeline::bubble_fraction (pipeline.cpp:16-22)
    if (!tl || !out) fail(HC_EINVAL, "bubble_fraction: null argument");
    if (tl->n_events == 0) fail(HC_EINVAL, "bubble_fraction: empty timeline");
    if (tl->total_s <= 0) {
      *out = 0;
      return;
    }
    const double io = hc_timeline_lane_busy(tl, HC_LANE_IO);
    const double comp = hc_timeline_lane_busy(tl, HC_LANE_COMPUTE);
    const double f = (std::max(io, comp) - std::min(io, comp)) / tl->total_s;
    *out = std::min(1.0, std::max(0.0, f));
  });
}

hc_status hc_simulate_pipeline(const hc_pipeline_job* jobs, int32_t n_jobs,
                               int32_t prefetch_depth, hc_timeline* out) {
  return guard([&] {
    if (!out || (n_jobs > 0 && !jobs)) fail(HC_EINVAL, "simulate_pipeline: null argument");
    simulate(jobs, n_jobs, prefetch_depth, out);
  });
}

}  // extern "C"
