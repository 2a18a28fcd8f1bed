// Niyama per-replica QoS scheduler core: hybrid priority
// (Eq. 4-5), violation checker, eager relegation, selective preemption, relegated
// service, dynamic chunking with multi-fill, completion bookkeeping.  Follows
// PAPER.md §3 (P:205 steps ①-⑦) with the readings R21-R29 of DESIGN.md.
// The cost model is a niyama_predictor (a8); the batch it emits is a
// niyama_batch_desc ready for niyama_plan_create (a2).  C ABI: include/niyama.h.
#include <algorithm>
#include <cmath>
#include <limits>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "internal.h"
#include "niyama.h"

namespace {

enum State : int32_t { kPrefill = 0, kDecode = 1, kRelegated = 2, kDone = 3 };

struct Req {
  int64_t id;
  double t_arrival;
  int32_t prompt;
  niyama_qos_spec qos;
  int32_t low, app, tier;
  int32_t prefill_done = 0, decoded = 0;
  State state = kPrefill;
  int32_t relegated = 0;
  // cache of Prefill_rem (R24): valid while prefill_done == rem_at
  int32_t rem_at = -1;
  double rem_s = 0.0;
};

struct Hist {
  int64_t n = 0;
  double mean = 0.0, m2 = 0.0;
};

bool feasible(double t, double slack) { return t <= slack + 1e-12 * std::max(1.0, std::fabs(slack)); }

}  // namespace

struct niyama_sched {
  niyama_sched_config cfg;
  const niyama_predictor* model;
  std::unordered_map<int64_t, Req> reqs;
  std::vector<int64_t> order;  // submission order (stable iteration)
  std::unordered_map<int32_t, Hist> hist;
  int64_t inflight = -1;
  bool has_inflight = false;
  bool outstanding = false;  // a non-empty batch awaits complete()
  // the last batch (arrays handed out through niyama_sched_batch)
  std::vector<int64_t> slice_id, dec_id, relegated_now;
  std::vector<int32_t> slice_off, slice_len, dec_ctx;
  std::vector<uint8_t> tier;
  // scratch for model calls
  mutable std::vector<int64_t> s_seq;
  mutable std::vector<int32_t> s_off, s_len;

  double iter_time(const std::vector<int32_t>& off, const std::vector<int32_t>& len, const int32_t* ctx,
                   int32_t nctx) const {
    niyama_batch_desc d{};
    d.num_prefill = static_cast<int32_t>(off.size());
    s_seq.assign(off.size(), 0);
    d.prefill_seq = s_seq.data();
    d.prefill_offset = off.data();
    d.prefill_len = len.data();
    d.num_decode = nctx;
    d.decode_seq = nullptr;
    d.decode_ctx = ctx;
    return cfg.fixed_s + cfg.layers * niyama_predict_iter_time(model, &d);  // R30
  }
  double one_slice(int32_t off, int32_t len, const int32_t* ctx, int32_t nctx) const {
    s_off.assign(1, off);
    s_len.assign(1, len);
    if (len <= 0) {
      s_off.clear();
      s_len.clear();
    }
    return iter_time(s_off, s_len, ctx, nctx);
  }

  // R24: remaining prefill alone, max_chunk-sized chunks from the current offset
  double prefill_rem(Req& r) {
    if (r.rem_at == r.prefill_done) return r.rem_s;
    double t = 0.0;
    int32_t off = r.prefill_done;
    while (off < r.prompt) {
      const int32_t c = std::min(cfg.max_chunk, r.prompt - off);
      t += one_slice(off, c, nullptr, 0);
      off += c;
    }
    r.rem_at = r.prefill_done;
    r.rem_s = t;
    return t;
  }
  // P:276 mean + 2 std of the app's completed decode lengths (prior before min_samples)
  double estimate(int32_t app) const {
    auto it = hist.find(app);
    const int64_t n = it == hist.end() ? 0 : it->second.n;
    if (n < std::max<int64_t>(1, cfg.history_min_samples)) return cfg.prior_mean + 2.0 * cfg.prior_std;
    const double sd = std::sqrt(it->second.m2 / static_cast<double>(n));
    return it->second.mean + 2.0 * sd;
  }
  double decode_rem(const Req& r) const {  // R25
    return std::max(0.0, estimate(r.app) - r.decoded) * cfg.decode_token_s;
  }
  double deadline(const Req& r) const {  // Eq. 1 / Eq. 3
    return r.qos.interactive ? r.t_arrival + r.qos.slo_ttft : r.t_arrival + r.qos.slo_ttlt;
  }
  double key(Req& r) {
    switch (cfg.policy) {
      case NIYAMA_POLICY_FCFS: return r.t_arrival;
      case NIYAMA_POLICY_EDF: return deadline(r);
      case NIYAMA_POLICY_SJF: return static_cast<double>(r.prompt);
      case NIYAMA_POLICY_SRPF: return static_cast<double>(r.prompt - r.prefill_done);
      default: {
        double work = prefill_rem(r);
        if (!r.qos.interactive) work += decode_rem(r);   // Eq. 5
        return deadline(r) + cfg.alpha * work;           // Eq. 4
      }
    }
  }
  int32_t status(Req& r, double now) {  // violation checker (P:205 ②; R23)
    const double d = deadline(r);
    if (d < now) return NIYAMA_VIOLATED;
    double horizon = prefill_rem(r);
    if (!r.qos.interactive)
      horizon += decode_rem(r);
    else
      horizon += cfg.decode_token_s;  // R23: the first token needs one decode iteration
    return d < now + horizon ? NIYAMA_WILL_VIOLATE : NIYAMA_QOS_OK;
  }
  double decode_slack(const Req& r, double now) const {
    if (r.qos.interactive) {  // Eq. 2 at n = decoded + 1 (R21); a late token is paced at TBT (R31)
      const double s = r.t_arrival + r.qos.slo_ttft + static_cast<double>(r.decoded) * r.qos.slo_tbt - now;
      return s >= 0.0 ? s : r.qos.slo_tbt;
    }
    const double est = std::max(1.0, estimate(r.app) - r.decoded);
    return (r.t_arrival + r.qos.slo_ttlt - now) / est;  // R17
  }
};

namespace {

struct Keyed {
  double k, t;
  int64_t id;
  Req* r;
};
bool operator<(const Keyed& a, const Keyed& b) {
  if (a.k != b.k) return a.k < b.k;
  if (a.t != b.t) return a.t < b.t;
  return a.id < b.id;
}

niyama_status check_cfg(const niyama_sched_config* c) {
  if (c->policy < NIYAMA_POLICY_NIYAMA || c->policy > NIYAMA_POLICY_SRPF)
    return niyama::set_error(NIYAMA_EINVAL, "sched config: policy");
  if (c->preemption < NIYAMA_PREEMPT_NEVER || c->preemption > NIYAMA_PREEMPT_ALWAYS)
    return niyama::set_error(NIYAMA_EINVAL, "sched config: preemption");
  if (!(c->alpha >= 0.0) || std::isinf(c->alpha)) return niyama::set_error(NIYAMA_EINVAL, "sched config: alpha < 0");
  if (c->max_chunk < 1 || c->fixed_chunk < 0) return niyama::set_error(NIYAMA_EINVAL, "sched config: chunk sizes");
  if (!(c->decode_token_s >= 0.0) || !(c->prior_mean >= 0.0) || !(c->prior_std >= 0.0) ||
      c->history_min_samples < 0)
    return niyama::set_error(NIYAMA_EINVAL, "sched config: history / decode_token_s");
  if (!(c->layers > 0.0) || !(c->fixed_s >= 0.0) || std::isinf(c->layers) || std::isinf(c->fixed_s))
    return niyama::set_error(NIYAMA_EINVAL, "sched config: layers > 0, fixed_s >= 0");
  if (c->kv_token_budget < 0) return niyama::set_error(NIYAMA_EINVAL, "sched config: kv_token_budget < 0");
  return NIYAMA_OK;
}

}  // namespace

extern "C" void niyama_sched_config_default(niyama_sched_config* c) {
  if (!c) return;
  *c = niyama_sched_config{};
  c->policy = NIYAMA_POLICY_NIYAMA;
  c->preemption = NIYAMA_PREEMPT_SELECTIVE;
  c->dynamic_chunk = 1;
  c->fixed_chunk = 256;
  c->max_chunk = 2048;
  c->relegation = 1;
  c->multi_fill = 1;
  c->history_min_samples = 30;
  c->alpha = 0.0;
  c->prior_mean = 415.0;
  c->prior_std = 300.0;
  c->decode_token_s = 0.05;
  c->layers = 1.0;
  c->fixed_s = 0.0;
  c->kv_token_budget = 0;
}

extern "C" niyama_status niyama_sched_create(const niyama_sched_config* cfg, const niyama_predictor* model,
                                            niyama_sched** out) {
  if (!cfg || !model || !out) return niyama::set_error(NIYAMA_EINVAL, "NULL argument");
  const niyama_status s = check_cfg(cfg);
  if (s != NIYAMA_OK) return s;
  auto* p = new niyama_sched();
  p->cfg = *cfg;
  p->model = model;
  *out = p;
  return NIYAMA_OK;
}

extern "C" void niyama_sched_destroy(niyama_sched* s) { delete s; }

extern "C" niyama_status niyama_sched_submit(niyama_sched* s, int64_t id, double t_arrival, int32_t prompt_tokens,
                                            const niyama_qos_spec* qos, int32_t low_priority, int32_t app_id,
                                            int32_t tier) {
  if (!s || !qos) return niyama::set_error(NIYAMA_EINVAL, "NULL argument");
  if (prompt_tokens < 1) return niyama::set_error(NIYAMA_EINVAL, "prompt_tokens < 1");
  if (std::isnan(t_arrival)) return niyama::set_error(NIYAMA_EINVAL, "t_arrival is NaN");
  if (qos->interactive ? !(qos->slo_ttft >= 0.0 && qos->slo_tbt >= 0.0) : !(qos->slo_ttlt >= 0.0))
    return niyama::set_error(NIYAMA_EINVAL, "qos: negative or NaN SLO");
  if (tier < 0 || tier > 255) return niyama::set_error(NIYAMA_EINVAL, "tier outside [0, 255]");
  if (s->reqs.count(id)) return niyama::set_error(NIYAMA_EINVAL, "request id already submitted");
  Req r;
  r.id = id;
  r.t_arrival = t_arrival;
  r.prompt = prompt_tokens;
  r.qos = *qos;
  r.low = low_priority ? 1 : 0;
  r.app = app_id;
  r.tier = tier;
  s->reqs.emplace(id, r);
  s->order.push_back(id);
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_sched_next_batch(niyama_sched* s, double now, niyama_sched_batch* out) {
  if (!s || !out) return niyama::set_error(NIYAMA_EINVAL, "NULL argument");
  if (std::isnan(now)) return niyama::set_error(NIYAMA_EINVAL, "now is NaN");
  if (s->outstanding) return niyama::set_error(NIYAMA_ESTATE, "complete() the outstanding batch first");
  const niyama_sched_config& c = s->cfg;

  // running decodes, (arrival, id) order; their slack, relegated ones excluded (R29)
  std::vector<Keyed> dec;
  std::vector<Keyed> pre, rel;
  for (int64_t id : s->order) {
    Req& r = s->reqs.at(id);
    if (r.state == kDecode) dec.push_back(Keyed{r.t_arrival, r.t_arrival, r.id, &r});
  }
  std::sort(dec.begin(), dec.end());
  s->dec_id.clear();
  s->dec_ctx.clear();
  double slack = std::numeric_limits<double>::infinity();
  for (const Keyed& k : dec) {
    s->dec_id.push_back(k.id);
    s->dec_ctx.push_back(k.r->prompt + k.r->decoded + 1);  // R4: keys visible after the new token
    if (!k.r->relegated) slack = std::min(slack, s->decode_slack(*k.r, now));
  }
  const int32_t nd = static_cast<int32_t>(s->dec_ctx.size());
  const int32_t* ctx = s->dec_ctx.data();

  // ① prefill queue by priority; ②-③ relegation (R22)
  for (int64_t id : s->order) {
    Req& r = s->reqs.at(id);
    if (r.state == kPrefill) pre.push_back(Keyed{s->key(r), r.t_arrival, r.id, &r});
  }
  std::sort(pre.begin(), pre.end());
  s->relegated_now.clear();
  if (c.relegation) {
    std::vector<int32_t> st(pre.size());
    bool any_low = false;
    for (size_t i = 0; i < pre.size(); ++i) {
      st[i] = s->status(*pre[i].r, now);
      if (pre[i].r->low && st[i] != NIYAMA_QOS_OK) any_low = true;
    }
    std::vector<Keyed> keep;
    for (size_t i = 0; i < pre.size(); ++i) {
      Req& r = *pre[i].r;
      const bool go = st[i] != NIYAMA_QOS_OK && (any_low ? r.low != 0 : r.low == 0);
      if (go) {
        r.state = kRelegated;
        r.relegated = 1;
        s->relegated_now.push_back(r.id);
      } else {
        keep.push_back(pre[i]);
      }
    }
    pre.swap(keep);
  }
  std::vector<Req*> queue;
  for (const Keyed& k : pre) queue.push_back(k.r);
  if (queue.empty()) {  // R28: relegated service, earliest original deadline first
    for (int64_t id : s->order) {
      Req& r = s->reqs.at(id);
      if (r.state == kRelegated) rel.push_back(Keyed{s->deadline(r), r.t_arrival, r.id, &r});
    }
    std::sort(rel.begin(), rel.end());
    for (const Keyed& k : rel) {
      queue.push_back(k.r);
      if (!c.multi_fill) break;
    }
  }

  // selective preemption (R26)
  if (s->has_inflight && !queue.empty() && queue[0]->id != s->inflight && c.preemption != NIYAMA_PREEMPT_ALWAYS) {
    auto it = std::find_if(queue.begin(), queue.end(), [&](Req* r) { return r->id == s->inflight; });
    if (it != queue.end() && (*it)->prefill_done > 0) {
      Req* cur = *it;
      bool keep = true;
      if (c.preemption == NIYAMA_PREEMPT_SELECTIVE) {
        Req* head = queue[0];
        const double delay =
            s->one_slice(head->prefill_done, std::min(c.max_chunk, head->prompt - head->prefill_done), ctx, nd);
        keep = s->status(*cur, now + delay) != NIYAMA_QOS_OK;
      }
      if (keep) {
        queue.erase(it);
        queue.insert(queue.begin(), cur);
      }
    }
  }

  // ④ chunk budget (S:116-124 by bisection)
  int32_t budget = 0, infeasible = 0;
  if (!queue.empty()) {
    if (!c.dynamic_chunk) {
      budget = c.fixed_chunk;
    } else {
      const int32_t off = queue[0]->prefill_done;
      auto ok = [&](int32_t C) { return feasible(s->one_slice(off, C, ctx, nd), slack); };
      if (!ok(0)) {
        infeasible = 1;
      } else if (ok(c.max_chunk)) {
        budget = c.max_chunk;
      } else {
        int32_t lo = 0, hi = c.max_chunk;
        while (hi - lo > 1) {
          const int32_t mid = lo + (hi - lo) / 2;
          if (ok(mid))
            lo = mid;
          else
            hi = mid;
        }
        budget = lo;
      }
    }
  }

  // ⑤ greedy fill (R27), within the KV token budget (R32)
  s->slice_id.clear();
  s->slice_off.clear();
  s->slice_len.clear();
  int32_t left = budget;
  if (c.kv_token_budget > 0) {
    int64_t held = nd;  // the decodes' new tokens
    for (const auto& kvp : s->reqs) {
      const Req& r = kvp.second;
      if (r.state != kDone) held += r.prefill_done + r.decoded;
    }
    left = static_cast<int32_t>(std::max<int64_t>(0, std::min<int64_t>(left, c.kv_token_budget - held)));
  }
  for (Req* r : queue) {
    if (left <= 0) break;
    const int32_t n = std::min(r->prompt - r->prefill_done, left);
    s->slice_id.push_back(r->id);
    s->slice_off.push_back(r->prefill_done);
    s->slice_len.push_back(n);
    left -= n;
    if (!c.multi_fill) break;
  }
  double pred = s->iter_time(s->slice_off, s->slice_len, ctx, nd);
  if (c.dynamic_chunk && !s->slice_len.empty() && !feasible(pred, slack)) {
    const int32_t n = s->slice_len.back();
    int32_t lo = 0, hi = n;
    while (hi - lo > 1) {
      const int32_t mid = lo + (hi - lo) / 2;
      s->slice_len.back() = mid;
      if (feasible(s->iter_time(s->slice_off, s->slice_len, ctx, nd), slack))
        lo = mid;
      else
        hi = mid;
    }
    if (lo > 0) {
      s->slice_len.back() = lo;
    } else {
      s->slice_id.pop_back();
      s->slice_off.pop_back();
      s->slice_len.pop_back();
    }
    pred = s->iter_time(s->slice_off, s->slice_len, ctx, nd);
  }

  s->tier.clear();
  for (int64_t id : s->slice_id) s->tier.push_back(static_cast<uint8_t>(s->reqs.at(id).tier));
  for (int64_t id : s->dec_id) s->tier.push_back(static_cast<uint8_t>(s->reqs.at(id).tier));
  s->outstanding = !s->slice_id.empty() || !s->dec_id.empty();

  *out = niyama_sched_batch{};
  out->desc.num_prefill = static_cast<int32_t>(s->slice_id.size());
  out->desc.prefill_seq = s->slice_id.data();
  out->desc.prefill_offset = s->slice_off.data();
  out->desc.prefill_len = s->slice_len.data();
  out->desc.num_decode = nd;
  out->desc.decode_seq = s->dec_id.data();
  out->desc.decode_ctx = s->dec_ctx.data();
  out->desc.tier = s->tier.data();
  out->chunk_budget = budget;
  out->infeasible = infeasible;
  out->predicted_s = pred;
  out->min_slack_s = slack;
  out->num_relegated = static_cast<int32_t>(s->relegated_now.size());
  out->relegated = s->relegated_now.data();
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_sched_complete(niyama_sched* s, double now, const int64_t* finished,
                                              int32_t n_finished) {
  if (!s || n_finished < 0 || (n_finished > 0 && !finished)) return niyama::set_error(NIYAMA_EINVAL, "NULL argument");
  if (!s->outstanding) return niyama::set_error(NIYAMA_ESTATE, "no batch outstanding");
  std::unordered_set<int64_t> fin;
  {
    std::unordered_set<int64_t> in_batch(s->dec_id.begin(), s->dec_id.end());
    for (int32_t i = 0; i < n_finished; ++i) {
      if (!in_batch.count(finished[i])) return niyama::set_error(NIYAMA_EINVAL, "finished id not among the batch's decodes");
      fin.insert(finished[i]);
    }
  }
  s->outstanding = false;
  for (int64_t id : s->dec_id) {  // ⑦ one token per running decode
    Req& r = s->reqs.at(id);
    r.decoded += 1;
    if (fin.count(id)) {
      r.state = kDone;
      Hist& h = s->hist[r.app];  // Welford
      h.n += 1;
      const double x = r.decoded;
      const double d = x - h.mean;
      h.mean += d / static_cast<double>(h.n);
      h.m2 += d * (x - h.mean);
    }
  }
  int64_t last = -1;
  bool any = false;
  for (size_t i = 0; i < s->slice_id.size(); ++i) {
    Req& r = s->reqs.at(s->slice_id[i]);
    r.prefill_done += s->slice_len[i];
    last = r.id;
    any = true;
    if (r.prefill_done == r.prompt) r.state = kDecode;
  }
  s->has_inflight = false;
  if (any) {
    const Req& r = s->reqs.at(last);
    if (r.state == kPrefill || r.state == kRelegated) {
      s->has_inflight = true;
      s->inflight = last;
    }
  }
  (void)now;
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_sched_request(const niyama_sched* s, int64_t id, niyama_request_info* out) {
  if (!s || !out) return niyama::set_error(NIYAMA_EINVAL, "NULL argument");
  auto it = s->reqs.find(id);
  if (it == s->reqs.end()) return niyama::set_error(NIYAMA_ENOSEQ, "unknown request id");
  const Req& r = it->second;
  out->state = r.state;
  out->relegated = r.relegated;
  out->prefill_done = r.prefill_done;
  out->decoded = r.decoded;
  out->prompt = r.prompt;
  out->low = r.low;
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_sched_counts(const niyama_sched* s, int32_t* counts4) {
  if (!s || !counts4) return niyama::set_error(NIYAMA_EINVAL, "NULL argument");
  for (int i = 0; i < 4; ++i) counts4[i] = 0;
  for (const auto& kv : s->reqs) counts4[kv.second.state] += 1;
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_sched_priority(niyama_sched* s, int64_t id, double now, double* key_out,
                                              int32_t* status_out) {
  if (!s || !key_out || !status_out) return niyama::set_error(NIYAMA_EINVAL, "NULL argument");
  auto it = s->reqs.find(id);
  if (it == s->reqs.end()) return niyama::set_error(NIYAMA_ENOSEQ, "unknown request id");
  *key_out = s->key(it->second);
  *status_out = s->status(it->second, now);
  return NIYAMA_OK;
}
