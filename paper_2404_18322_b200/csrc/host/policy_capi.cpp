// C ABI of the routing / marking / placement policy (include/blockpolicy.h).
#include <cstring>
#include <stdexcept>
#include <string>

#include "../../../include/blockpolicy.h"
#include "policy.hpp"

struct bh_policy {
  explicit bh_policy(const bh::PolicyConfig& c) : p(c) {}
  bh::Policy p;
  bh::Interception tint;
  std::string err;
};

namespace {
template <class F>
int guard(bh_policy* h, F&& f) {
  if (h == nullptr) return BE_ERR_INVALID;
  try {
    f();
    return BE_OK;
  } catch (const std::invalid_argument& e) {
    h->err = e.what();
    return BE_ERR_INVALID;
  } catch (const std::logic_error& e) {
    h->err = e.what();
    return BE_ERR_STATE;
  } catch (const std::exception& e) {
    h->err = e.what();
    return BE_ERR_RUNTIME;
  }
}
std::string str(const char* s) { return s ? std::string(s) : std::string(); }
bh::Grid grid(const bh_grid* g) {
  if (g == nullptr || g->nx <= 0 || g->ny <= 0 || !g->xs || !g->ys || !g->v)
    throw bh::PolicyError("empty interpolation axis");
  bh::Grid out;
  out.xs.assign(g->xs, g->xs + g->nx);
  out.ys.assign(g->ys, g->ys + g->ny);
  out.v.assign(g->v, g->v + static_cast<std::size_t>(g->nx) * g->ny);
  return out;
}
bh::Query query(const bh_binding_query* q) {
  if (q == nullptr || q->chain_block == nullptr) throw bh::PolicyError("null query");
  bh::Query x;
  x.request_id = q->request_id;
  x.chain_block = q->chain_block;
  x.decode = q->phase == BE_PHASE_DECODE;
  x.tokens = q->tokens;
  x.context_tokens = q->context_tokens;
  x.from_device = q->from_device;
  x.now = q->now;
  return x;
}
void copy_id(char* dst, std::size_t cap, const std::string& s) {
  if (s.size() >= cap) throw bh::PolicyError("id longer than the output field: " + s);
  std::memcpy(dst, s.c_str(), s.size() + 1);
}
// '\n'-joined ids into ids[cap] (+ optional parallel int array)
template <class V, class IdOf, class DevOf>
void put_list(const V& v, char* ids, int cap, int* devs, int dev_cap, int* n, IdOf id_of,
              DevOf dev_of) {
  std::string joined;
  for (std::size_t i = 0; i < v.size(); ++i) {
    if (i) joined += '\n';
    joined += id_of(v[i]);
  }
  if (ids == nullptr || cap <= static_cast<int>(joined.size()))
    throw bh::PolicyError("id buffer too small");
  std::memcpy(ids, joined.c_str(), joined.size() + 1);
  if (devs != nullptr) {
    if (dev_cap < static_cast<int>(v.size())) throw bh::PolicyError("device buffer too small");
    for (std::size_t i = 0; i < v.size(); ++i) devs[i] = dev_of(v[i]);
  }
  *n = static_cast<int>(v.size());
}
}  // namespace

extern "C" {

bh_policy* bh_policy_new(const bh_policy_config* c) {
  bh::PolicyConfig cfg;
  if (c != nullptr) {
    cfg.adaptive = c->adaptive != 0;
    cfg.least_busy = c->least_busy != 0;
    cfg.frag_min = c->frag_min != 0;
    cfg.speculation = c->speculation != 0;
    cfg.spec_fraction = c->spec_fraction;
    cfg.scale_queue_us = c->scale_queue_us;
    cfg.expected_tokens = c->expected_tokens;
    cfg.sur_attention_only = c->sur_attention_only;
    cfg.sur_ffn_only = c->sur_ffn_only;
    cfg.sur_one_layer = c->sur_one_layer;
    cfg.sur_multi_layer = c->sur_multi_layer;
    cfg.sur_allow_adapter_blocks = c->sur_allow_adapter_blocks != 0;
  }
  return new bh_policy(cfg);
}
void bh_policy_free(bh_policy* p) { delete p; }
const char* bh_policy_last_error(const bh_policy* p) { return p ? p->err.c_str() : "null policy"; }

int bh_policy_add_cost_class(bh_policy* p, const char* key, const bh_grid* pre, const bh_grid* dec,
                             int64_t kv) {
  return guard(p, [&] { p->p.add_cost_class(str(key), grid(pre), grid(dec), kv); });
}
int bh_policy_add_stitch_class(bh_policy* p, const char* key, const bh_grid* g) {
  return guard(p, [&] { p->p.add_stitch_class(str(key), grid(g)); });
}
int bh_policy_set_device_class(bh_policy* p, const char* name, double speed) {
  return guard(p, [&] { p->p.set_device_class(str(name), speed); });
}
int bh_policy_add_component(bh_policy* p, const char* id, int kind, int dim, int layer, int n,
                            const char* const* pids, const int64_t* pbytes) {
  return guard(p, [&] {
    if (kind < 0 || kind > 4) throw bh::PolicyError("unknown component kind");
    std::vector<std::pair<std::string, std::int64_t>> pieces;
    for (int i = 0; i < n; ++i) pieces.emplace_back(str(pids[i]), pbytes[i]);
    p->p.add_component(str(id), static_cast<bh::Kind>(kind), dim, layer, std::move(pieces));
  });
}
int bh_policy_add_block(bh_policy* p, const char* id, int n, const char* const* comps, int dout) {
  return guard(p, [&] {
    std::vector<std::string> v;
    for (int i = 0; i < n; ++i) v.push_back(str(comps[i]));
    p->p.add_block(str(id), std::move(v), dout);
  });
}
int bh_policy_add_chain(bh_policy* p, const char* model, int n, const char* const* blocks) {
  return guard(p, [&] {
    std::vector<std::string> v;
    for (int i = 0; i < n; ++i) v.push_back(str(blocks[i]));
    p->p.add_chain(str(model), std::move(v));
  });
}
int bh_policy_add_candidate(bh_policy* p, const char* b, const char* c, const char* st, double s) {
  return guard(p, [&] { p->p.add_candidate(str(b), str(c), str(st), s); });
}
int bh_policy_add_server(bh_policy* p, int id, double bps) {
  return guard(p, [&] { p->p.add_server(id, bps); });
}
int bh_policy_set_inter_bandwidth(bh_policy* p, int a, int b, double bps) {
  return guard(p, [&] { p->p.set_inter_bandwidth(a, b, bps); });
}
int bh_policy_set_inter_default(bh_policy* p, double bps) {
  return guard(p, [&] { p->p.set_inter_default(bps); });
}
int bh_policy_add_device(bh_policy* p, int id, int server, const char* cls, int64_t cap,
                         double mem_bps, double load_bps) {
  return guard(p, [&] { p->p.add_device(id, server, str(cls), cap, mem_bps, load_bps); });
}

int bh_policy_clear_state(bh_policy* p) {
  return guard(p, [&] { p->p.clear_state(); });
}
int bh_policy_put_instance(bh_policy* p, const bh_policy_instance* in) {
  return guard(p, [&] {
    if (in == nullptr || in->id == nullptr) throw bh::PolicyError("null instance");
    bh::PolicyInstance x;
    x.id = in->id;
    x.block_id = str(in->block_id);
    x.device = in->device;
    x.ready = in->ready != 0;
    x.ready_at = in->ready_at;
    x.last_used = in->last_used;
    x.created_seq = in->created_seq;
    x.executing = in->executing != 0;
    x.queue_len = in->queue_len;
    x.queued_cost_us = in->queued_cost_us;
    x.queued_cost_hwm = in->queued_cost_hwm;
    p->p.put_instance(x);
  });
}
int bh_policy_remove_instance(bh_policy* p, const char* id) {
  return guard(p, [&] { p->p.remove_instance(str(id)); });
}
int bh_policy_set_ledger(bh_policy* p, int dev, int64_t params, int64_t kv, int64_t act) {
  return guard(p, [&] { p->p.set_ledger(dev, params, kv, act); });
}
int bh_policy_set_lane(bh_policy* p, int dev, int64_t busy_until) {
  return guard(p, [&] { p->p.set_lane(dev, busy_until); });
}
int bh_policy_set_kv(bh_policy* p, uint64_t req, const char* b, int owner, int pages) {
  return guard(p, [&] { p->p.set_kv(req, str(b), owner, pages); });
}
int bh_policy_set_adjacency(bh_policy* p, const char* from, const char* to, int64_t n) {
  return guard(p, [&] { p->p.set_adjacency(str(from), str(to), n); });
}
int bh_policy_note_adjacency(bh_policy* p, const char* from, const char* to) {
  return guard(p, [&] { p->p.note_adjacency(str(from), str(to)); });
}

int bh_policy_choose_binding(bh_policy* p, const bh_binding_query* q, bh_binding_choice* out,
                             int* found) {
  return guard(p, [&] {
    if (out == nullptr || found == nullptr) throw bh::PolicyError("null output");
    auto c = p->p.choose_binding(query(q));
    *found = c.has_value() ? 1 : 0;
    std::memset(out, 0, sizeof(*out));
    out->device = -1;
    if (!c) return;
    copy_id(out->block_id, sizeof(out->block_id), c->block_id);
    copy_id(out->stitch_class, sizeof(out->stitch_class), c->stitch_class);
    copy_id(out->instance_id, sizeof(out->instance_id), c->instance_id);
    out->device = c->device;
    out->adaptive = c->adaptive ? 1 : 0;
    out->evict_bytes = c->evict_bytes;
    out->queue_us = c->est.queue_us;
    out->compute_us = c->est.compute_us;
    out->transfer_us = c->est.transfer_us;
    out->load_us = c->est.load_us;
  });
}
int bh_policy_estimate(bh_policy* p, const bh_binding_query* q, const char* b, const char* st,
                       const char* inst, int dev, double* out4, int64_t* evict) {
  return guard(p, [&] {
    const bh::PolicyInstance* in = nullptr;
    if (inst != nullptr) {
      in = p->p.find(inst);
      if (in == nullptr) throw bh::PolicyError(std::string("unknown instance ") + inst);
    }
    std::int64_t ev = 0;
    const bh::Estimate e = p->p.estimate(query(q), str(b), str(st), in, dev, &ev);
    out4[0] = e.queue_us;
    out4[1] = e.compute_us;
    out4[2] = e.transfer_us;
    out4[3] = e.load_us;
    if (evict) *evict = ev;
  });
}
int bh_policy_speculation_marks(bh_policy* p, char* ids, int cap, int* n) {
  return guard(p, [&] {
    const auto v = p->p.speculation_marks();
    put_list(v, ids, cap, nullptr, 0, n, [](const std::string& s) { return s; },
             [](const std::string&) { return 0; });
  });
}
int bh_policy_scale_decisions(bh_policy* p, char* ids, int cap, int* devs, int dev_cap, int* n) {
  return guard(p, [&] {
    const auto v = p->p.scale_decisions();
    put_list(v, ids, cap, devs, dev_cap, n, [](const auto& x) { return x.first; },
             [](const auto& x) { return x.second; });
  });
}
int bh_policy_choose_device(bh_policy* p, const char* b, int pref, const int* excl, int n_excl,
                            int* dev) {
  return guard(p, [&] {
    if (pref < 0 || pref > 2) throw bh::PolicyError("unknown device preference");
    std::set<int> ex;
    for (int i = 0; i < n_excl; ++i) ex.insert(excl[i]);
    *dev = p->p.choose_device(str(b), static_cast<bh::DevicePref>(pref), ex);
  });
}
int bh_policy_placement_moves(bh_policy* p, char* ids, int cap, int* devs, int dev_cap, int* n) {
  return guard(p, [&] {
    const auto v = p->p.placement_moves();
    put_list(v, ids, cap, devs, dev_cap, n, [](const auto& x) { return x.first; },
             [](const auto& x) { return x.second; });
  });
}
int bh_policy_migration_rates(bh_policy* p, const char* b, int src, int dst, int64_t* rec,
                              int64_t* cp) {
  return guard(p, [&] {
    const auto r = p->p.migration_rates(str(b), src, dst);
    *rec = r.first;
    *cp = r.second;
  });
}
int bh_policy_param_bytes_needed(bh_policy* p, const char* b, int dev, int64_t* out) {
  return guard(p, [&] { *out = p->p.param_bytes_needed(str(b), dev); });
}

int bh_policy_interception_record(bh_policy* p, const char* key, int64_t sample) {
  return guard(p, [&] { p->tint.record(str(key), sample); });
}
int bh_policy_interception_set(bh_policy* p, const char* key, double sum, uint64_t n) {
  return guard(p, [&] {
    if (key == nullptr)
      p->tint.set_global(sum, n);
    else
      p->tint.set(key, sum, n);
  });
}
int bh_policy_interception_predict(bh_policy* p, const char* key, int64_t t_call, int64_t now,
                                   int64_t* out, int* found) {
  return guard(p, [&] {
    const auto r = p->tint.predicted_remaining(str(key), t_call, now);
    *found = r.has_value() ? 1 : 0;
    *out = r.value_or(0);
  });
}
int bh_policy_kv_review(bh_policy* p, const bh_queued_decode* q, int n, int64_t now,
                        int recalc_only, int* order, int cap, int* n_out) {
  return guard(p, [&] {
    std::vector<bh::QueuedDecode> v;
    for (int i = 0; i < n; ++i) {
      bh::QueuedDecode e;
      e.instance = str(q[i].instance);
      e.inst_block = str(q[i].inst_block);
      e.device = q[i].device;
      e.request_id = q[i].request_id;
      e.chain_block = str(q[i].chain_block);
      e.owner = q[i].owner;
      e.pages = q[i].pages;
      e.shared_pages = q[i].shared_pages;
      e.pending = q[i].pending != 0;
      e.pending_key = str(q[i].pending_key);
      e.t_call = q[i].t_call;
      v.push_back(std::move(e));
    }
    const auto out = p->p.kv_review(v, p->tint, now, recalc_only != 0);
    if ((int)out.size() > cap) throw bh::PolicyError("order buffer too small");
    for (std::size_t i = 0; i < out.size(); ++i) order[i] = out[i];
    *n_out = (int)out.size();
  });
}

int bh_plan_migration(int pages, int64_t rec, int64_t cp, int64_t* out6) {
  try {
    const bh::Migration m = bh::plan_migration(pages, rec, cp);
    out6[0] = m.pages;
    out6[1] = m.recompute_pages;
    out6[2] = m.copy_pages;
    out6[3] = m.completion_us;
    out6[4] = rec;
    out6[5] = cp;
    return BE_OK;
  } catch (const std::invalid_argument&) {
    return BE_ERR_INVALID;
  }
}

}  // extern "C"
