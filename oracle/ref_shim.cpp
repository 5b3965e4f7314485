// TEST INFRASTRUCTURE: a C ABI over the reference's own blocksim classes, compiled together with
// the unmodified reference sources under /root/reference/proj/core into oracle/_ref/ (see
// oracle/Makefile). Only tests/ load it, as the parity checker for the host control plane of
// paper_2404_18322_b200 (csrc/host/*): queue/batch formation (InstancePool, agent.cpp:132-224),
// paged KV bookkeeping (KvStore, kv.cpp:105-237), the cosine (signature_similarity,
// zoo.cpp:78-88), migration planning (plan_migration, kv.cpp:16-58), percentiles
// (metrics.cpp:30-38) and whole-simulation batch traces (Simulation::pump/on_batch_finish,
// scenario.cpp:465-578).
#include <dlfcn.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <queue>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <tuple>
#include <unordered_set>
#include <utility>
#include <vector>

#include "json.hpp"
// Page ids and the running batch are private in the reference; the checker reads them.
#define private public
#include "blocksim/agent.hpp"
#include "blocksim/config.hpp"
#include "blocksim/costmodel.hpp"
#include "blocksim/kv.hpp"
#include "blocksim/metrics.hpp"
#include "blocksim/scenario.hpp"
#include "blocksim/scheduler.hpp"
#include "blocksim/cluster.hpp"
#include "blocksim/zoo.hpp"
#undef private

using namespace blocksim;

namespace {
int code_of(const std::exception& e) {
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
  if (dynamic_cast<const std::logic_error*>(&e)) return 2;
  return 5;
}
template <class F>
int guard(std::string& err, F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    err = e.what();
    return code_of(e);
  }
}
}  // namespace

// Same layout as bh_entry (include/blockhost.h)
struct rs_entry {
  int32_t request_id, chain_step, phase, tokens, context_tokens, kv_resident;
  double est_cost_us;
  uint64_t enqueue_seq;
};

static rs_entry to_rs(const QueueEntry& e) {
  rs_entry r;
  r.request_id = e.request_id;
  r.chain_step = e.chain_step;
  r.phase = e.phase == Phase::kDecode ? 1 : 0;
  r.tokens = e.tokens;
  r.context_tokens = e.context_tokens;
  r.kv_resident = e.kv_resident ? 1 : 0;
  r.est_cost_us = e.est_cost_us;
  r.enqueue_seq = e.enqueue_seq;
  return r;
}

static Cluster big_cluster(int n_devices) {
  Cluster c;
  c.add_server({0, 1e12});
  for (int d = 0; d < n_devices; ++d) c.add_device({d, 0, "std", (std::int64_t)1 << 50, 1e15, 1e15});
  c.set_inter_default(1e12);
  return c;
}

// ---------------------------------------------------------------- InstancePool
struct rs_pool {
  Zoo zoo;
  Cluster cluster;
  std::unique_ptr<MemoryLedger> ledger;
  std::unique_ptr<InstancePool> pool;
  std::string err;
};

extern "C" {

// n_blocks one-component foundations "m<i>" give blocks "b0".."b<n-1>"
rs_pool* rs_pool_new(int n_blocks, int n_devices) {
  auto* h = new rs_pool();
  for (int i = 0; i < n_blocks; ++i) {
    ComponentDescriptor c;
    c.id = "m" + std::to_string(i) + ".att0";
    c.kind = ComponentKind::kAttention;
    c.embed_dim = 256;
    c.model_id = "m" + std::to_string(i);
    c.contents = {{c.id + ".w", 1000}};
    h->zoo.add_foundation("m" + std::to_string(i), {c});
  }
  h->cluster = big_cluster(n_devices);
  h->ledger = std::make_unique<MemoryLedger>(h->cluster);
  h->pool = std::make_unique<InstancePool>(h->zoo, h->cluster, *h->ledger);
  return h;
}
void rs_pool_free(rs_pool* h) { delete h; }
const char* rs_pool_last_error(const rs_pool* h) { return h->err.c_str(); }

int rs_pool_create_instance(rs_pool* h, const char* block, int device, int64_t now,
                            int64_t ready_at, char* id_out, int cap) {
  std::string id;
  int rc = guard(h->err, [&] { id = h->pool->create(block, device, now, ready_at).id; });
  if (rc) return rc;
  if ((int)id.size() >= cap) return 1;
  std::memcpy(id_out, id.c_str(), id.size() + 1);
  return 0;
}
int rs_pool_mark_ready(rs_pool* h, const char* inst, int64_t now) {
  return guard(h->err, [&] { h->pool->mark_ready(inst, now); });
}
int rs_pool_enqueue(rs_pool* h, const char* inst, const rs_entry* e) {
  QueueEntry q;
  q.request_id = e->request_id;
  q.chain_step = e->chain_step;
  q.phase = e->phase ? Phase::kDecode : Phase::kPrefill;
  q.tokens = e->tokens;
  q.context_tokens = e->context_tokens;
  q.kv_resident = e->kv_resident != 0;
  q.est_cost_us = e->est_cost_us;
  return guard(h->err, [&] { h->pool->enqueue(inst, q); });
}
static int put(const std::vector<QueueEntry>& v, rs_entry* out, int cap, int* n) {
  if (n) *n = (int)v.size();
  if ((int)v.size() > cap) return 1;
  for (size_t i = 0; i < v.size(); ++i) out[i] = to_rs(v[i]);
  return 0;
}
int rs_pool_pop_batch(rs_pool* h, const char* inst, int budget, int64_t now, rs_entry* out, int cap,
                      int* n, int* phase) {
  ExecBatch b;
  int rc = guard(h->err, [&] { b = h->pool->pop_batch(inst, budget, now); });
  if (rc) return rc;
  if (phase) *phase = b.phase == Phase::kDecode ? 1 : 0;
  return put(b.members, out, cap, n);
}
int rs_pool_finish_batch(rs_pool* h, const char* inst, int64_t now) {
  return guard(h->err, [&] { h->pool->finish_batch(inst, now); });
}
int rs_pool_next_runnable(rs_pool* h, int device, int64_t now, char* id_out, int cap) {
  Instance* in = h->pool->next_runnable(device, now);
  if (!in) return 0;
  if ((int)in->id.size() >= cap) return -1;
  std::memcpy(id_out, in->id.c_str(), in->id.size() + 1);
  return 1;
}
int rs_pool_remove_queued(rs_pool* h, const char* inst, int req, rs_entry* out, int cap, int* n) {
  std::vector<QueueEntry> v;
  int rc = guard(h->err, [&] { v = h->pool->remove_queued(inst, req); });
  return rc ? rc : put(v, out, cap, n);
}
int rs_pool_take_tail(rs_pool* h, const char* inst, int count, rs_entry* out, int cap, int* n) {
  std::vector<QueueEntry> v;
  int rc = guard(h->err, [&] { v = h->pool->take_tail(inst, (size_t)count); });
  return rc ? rc : put(v, out, cap, n);
}
int rs_pool_queue(rs_pool* h, const char* inst, rs_entry* out, int cap, int* n, double* cost,
                  int* executing) {
  Instance* in = h->pool->find(inst);
  if (!in) {
    h->err = std::string("pool: unknown instance ") + inst;
    return 2;
  }
  if (cost) *cost = in->queued_cost_us;
  if (executing) *executing = in->executing ? 1 : 0;
  std::vector<QueueEntry> v(in->queue.begin(), in->queue.end());
  return put(v, out, cap, n);
}

// ---------------------------------------------------------------- KvStore
struct rs_kv {
  Cluster cluster;
  std::unique_ptr<MemoryLedger> ledger;
  std::unique_ptr<KvStore> kv;
  std::string err;
};

rs_kv* rs_kv_new(int n_devices) {
  auto* h = new rs_kv();
  h->cluster = big_cluster(n_devices);
  h->ledger = std::make_unique<MemoryLedger>(h->cluster);
  h->kv = std::make_unique<KvStore>(*h->ledger);
  return h;
}
void rs_kv_free(rs_kv* h) { delete h; }
const char* rs_kv_last_error(const rs_kv* h) { return h->err.c_str(); }
int rs_kv_create_segment(rs_kv* h, uint64_t r, const char* b, int dev, int64_t bpt) {
  return guard(h->err, [&] { h->kv->create_segment(r, b, dev, bpt); });
}
int rs_kv_append_tokens(rs_kv* h, uint64_t r, const char* b, int n, int* added) {
  return guard(h->err, [&] {
    int a = h->kv->append_tokens(r, b, n);
    if (added) *added = a;
  });
}
int rs_kv_share_prefix(rs_kv* h, uint64_t r, uint64_t from, const char* b, int t, int* covered) {
  return guard(h->err, [&] {
    int c = h->kv->share_prefix(r, from, b, t);
    if (covered) *covered = c;
  });
}
int rs_kv_release(rs_kv* h, uint64_t r, const char* b) {
  return guard(h->err, [&] { h->kv->release(r, b); });
}
int rs_kv_release_request(rs_kv* h, uint64_t r) {
  return guard(h->err, [&] { h->kv->release_request(r); });
}
int rs_kv_move_segment(rs_kv* h, uint64_t r, const char* b, int dst) {
  return guard(h->err, [&] { h->kv->move_segment(r, b, dst); });
}
int64_t rs_kv_query(const rs_kv* h, uint64_t r, const char* b, int what) {
  switch (what) {
    case 0: return h->kv->device_of(r, b);
    case 1: return h->kv->tokens(r, b);
    case 2: return h->kv->pages(r, b);
    case 3: return h->kv->shared_pages(r, b);
    case 4: return h->kv->segment_bytes(r, b);
    case 5: return h->kv->has_segment(r, b) ? 1 : 0;
    default: return -1;
  }
}
int64_t rs_kv_bytes_saved(const rs_kv* h) { return h->kv->bytes_saved_by_sharing(); }
int64_t rs_kv_used(const rs_kv* h, int dev) {
  return h->ledger->used(dev, MemoryLedger::Category::kKv);
}
int rs_kv_page_ids(const rs_kv* h, uint64_t r, const char* b, uint64_t* out, int cap, int* n) {
  auto it = h->kv->segments_.find({r, std::string(b)});
  if (it == h->kv->segments_.end()) {
    if (n) *n = 0;
    return 0;
  }
  const auto& ids = it->second.page_ids;
  if (n) *n = (int)ids.size();
  if ((int)ids.size() > cap) return 1;
  for (size_t i = 0; i < ids.size(); ++i) out[i] = ids[i];
  return 0;
}

// ---------------------------------------------------------------- scalar functions
double rs_cosine(const double* a, int na, const double* b, int nb, int* err) {
  std::vector<double> va(a, a + na), vb(b, b + nb);
  try {
    *err = 0;
    return signature_similarity(va, vb);
  } catch (const std::exception& e) {
    *err = code_of(e);
    return 0.0;
  }
}
int rs_plan_migration(int pages, int64_t rec, int64_t cp, int64_t* out /*[6]*/) {
  try {
    MigrationPlan p = plan_migration(pages, rec, cp);
    out[0] = p.pages;
    out[1] = p.rec_us_per_page;
    out[2] = p.cp_us_per_page;
    out[3] = p.recompute_pages;
    out[4] = p.copy_pages;
    out[5] = p.completion_us;
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}
int rs_percentile(const double* v, int n, double q, double* out) {
  try {
    *out = percentile(std::vector<double>(v, v + n), q);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// ---------------------------------------------------------------- whole simulation trace
// Zoo: foundation "base" of n_layers (attention, ffn) layers at `dim`, plus n_lora LoRA variants
// whose attention is fused (attach "fuse") from layer `first_adapted` upward; served models are
// the LoRAs. One device, instant parameter loads, no speculation/adaptivity/scaling, reviews
// beyond the horizon: on one lane the batch sequence is independent of the cost tables.
struct rs_sim {
  std::vector<std::string> blocks;                 // block ids in zoo order
  std::vector<std::string> block_kinds;            // per block: "a"/"f" per component
  std::vector<std::vector<int>> chains;            // served model -> block indices
  std::vector<int> req_model;                      // per request: served model index
  // trace: per batch (instance, block, phase, members...)
  std::vector<std::tuple<int, int, int>> recs;     // (instance index, block index, phase)
  std::vector<std::vector<std::tuple<int, int, int>>> members;  // (req, step, ctx)
  std::string err;
  std::string report;
};

// The drop-in run (rs_sim_run_gpu): the same Simulation drives the product's batch executor
// (bh_executor_run_batch, include/blockhost.h - the call that replaces batch_duration_us at
// scenario.cpp:493) through the Engine's trace hook, which sees every kBatchFinish event before
// its handler: each batch the reference formed runs on the GPU, in the reference's order, with
// the reference's members. The product library is opened by path (dlopen), so this checker
// carries no link dependency on it.
struct GpuHook {
  void* lib = nullptr;
  void* ctx = nullptr;
  void* exec = nullptr;
  int (*run)(void*, const char*, const char*, int, int, const void*) = nullptr;
  const char* (*err)(const void*) = nullptr;
  std::vector<char> rows;  // decode rows read back at the end
  int64_t batches = 0;
};

static void run_sim(rs_sim* h, int n_layers, int dim, int n_lora, int first_adapted,
                    int n_requests, const int32_t* prompts, const int32_t* outputs,
                    int max_batch_tokens, int64_t arrival_gap_us, GpuHook* gpu,
                    const int32_t* prefix_group = nullptr, const int32_t* prefix_tokens = nullptr);

// The same run with prefix groups (Request::prefix_group / prefix_tokens, workload.hpp:19-20):
// the report's kv.shared_bytes is the high-water mark of bytes saved by sharing.
rs_sim* rs_sim_run_prefix(int n_layers, int dim, int n_lora, int first_adapted, int n_requests,
                          const int32_t* prompts, const int32_t* outputs, int max_batch_tokens,
                          const int32_t* prefix_group, const int32_t* prefix_tokens) {
  auto* h = new rs_sim();
  run_sim(h, n_layers, dim, n_lora, first_adapted, n_requests, prompts, outputs,
          max_batch_tokens, 0, nullptr, prefix_group, prefix_tokens);
  return h;
}

rs_sim* rs_sim_run(int n_layers, int dim, int n_lora, int first_adapted, int n_requests,
                   const int32_t* prompts, const int32_t* outputs, int max_batch_tokens,
                   int64_t arrival_gap_us) {
  auto* h = new rs_sim();
  run_sim(h, n_layers, dim, n_lora, first_adapted, n_requests, prompts, outputs,
          max_batch_tokens, arrival_gap_us, nullptr);
  return h;
}

// bh_executor_desc / bh_member of include/blockhost.h (same layout)
struct rs_exec_desc {
  int d_model, n_heads, d_ff, max_pos, max_batch_tokens;
  float init_scale;
  uint64_t seed;
};
struct rs_member {
  int32_t request_id, chain_step, tokens, context_tokens, chain_final;
};

rs_sim* rs_sim_run_gpu(const char* product_lib, int device, int n_layers, int dim, int n_heads,
                       int n_lora, int first_adapted, int n_requests, const int32_t* prompts,
                       const int32_t* outputs, int max_batch_tokens, int64_t arrival_gap_us,
                       uint64_t seed, float init_scale, void* decode_rows_out) {
  auto* h = new rs_sim();
  GpuHook g;
  try {
    g.lib = dlopen(product_lib, RTLD_NOW | RTLD_LOCAL);
    if (g.lib == nullptr) throw std::runtime_error(std::string("dlopen: ") + dlerror());
    auto sym = [&](const char* n) {
      void* f = dlsym(g.lib, n);
      if (f == nullptr) throw std::runtime_error(std::string("missing symbol ") + n);
      return f;
    };
    auto ctx_create = reinterpret_cast<int (*)(int, void**)>(sym("be_ctx_create"));
    auto ctx_destroy = reinterpret_cast<int (*)(void*)>(sym("be_ctx_destroy"));
    auto ex_create = reinterpret_cast<int (*)(void*, const rs_exec_desc*, int, const int32_t*,
                                              const int32_t*, void**)>(sym("bh_executor_create"));
    auto ex_free = reinterpret_cast<int (*)(void*)>(sym("bh_executor_free"));
    auto ex_read = reinterpret_cast<int (*)(void*, int, void*)>(sym("bh_executor_read_rows"));
    g.run = reinterpret_cast<int (*)(void*, const char*, const char*, int, int, const void*)>(
        sym("bh_executor_run_batch"));
    g.err = reinterpret_cast<const char* (*)(const void*)>(sym("bh_executor_last_error"));
    if (ctx_create(device, &g.ctx) != 0) throw std::runtime_error("be_ctx_create failed");
    int max_ctx = 0;
    for (int i = 0; i < n_requests; ++i) max_ctx = std::max(max_ctx, prompts[i] + outputs[i]);
    rs_exec_desc d{dim, n_heads, 3 * dim, max_ctx + 16, max_batch_tokens, init_scale, seed};
    if (ex_create(g.ctx, &d, n_requests, prompts, outputs, &g.exec) != 0)
      throw std::runtime_error("bh_executor_create failed");
    run_sim(h, n_layers, dim, n_lora, first_adapted, n_requests, prompts, outputs,
            max_batch_tokens, arrival_gap_us, &g);
    if (h->err.empty() && decode_rows_out != nullptr && ex_read(g.exec, 1, decode_rows_out) != 0)
      h->err = std::string("read rows: ") + g.err(g.exec);
    ex_free(g.exec);
    ctx_destroy(g.ctx);
  } catch (const std::exception& e) {
    h->err = e.what();
  }
  return h;
}

static void run_sim(rs_sim* h, int n_layers, int dim, int n_lora, int first_adapted,
                    int n_requests, const int32_t* prompts, const int32_t* outputs,
                    int max_batch_tokens, int64_t arrival_gap_us, GpuHook* gpu,
                    const int32_t* prefix_group, const int32_t* prefix_tokens) {
  try {
    Zoo zoo;
    std::vector<ComponentDescriptor> base;
    for (int l = 0; l < n_layers; ++l) {
      for (int k = 0; k < 2; ++k) {
        ComponentDescriptor c;
        c.id = "base." + std::string(k ? "ffn" : "att") + std::to_string(l);
        c.kind = k ? ComponentKind::kFfn : ComponentKind::kAttention;
        c.embed_dim = dim;
        c.model_id = "base";
        c.layer = l;
        c.slot = k;
        c.contents = {{c.id + ".w", k ? 3000 : 1000}};
        base.push_back(c);
      }
    }
    zoo.add_foundation("base", base);
    for (int v = 0; v < n_lora; ++v) {
      const std::string m = "lora" + std::to_string(v);
      std::vector<ComponentDescriptor> comps;
      for (int l = 0; l < n_layers; ++l) {
        if (l >= first_adapted) {
          ComponentDescriptor att;
          att.id = m + ".att" + std::to_string(l);
          att.kind = ComponentKind::kAttention;
          att.embed_dim = dim;
          att.model_id = m;
          att.layer = l;
          att.slot = 0;
          att.attach = "fuse";
          att.contents = {{"base.att" + std::to_string(l) + ".w", 1000}, {m + ".delta" + std::to_string(l), 8}};
          comps.push_back(att);
        } else {
          comps.push_back(zoo.component("base.att" + std::to_string(l)));
        }
        comps.push_back(zoo.component("base.ffn" + std::to_string(l)));
      }
      zoo.add_model_pe(m, TuningKind::kLora, "base", comps);
    }
    Cluster cl;
    cl.add_server({0, 1e12});
    cl.add_device({0, 0, "std", (std::int64_t)1 << 50, 1e15, 1e18});
    CostModel cost;
    cost.set_device_class("std", 1.0);
    auto grid = [](double coef) {
      Interp2D g;
      g.xs = {1, 64};
      g.ys = {1, 4096};
      g.v = {{coef, coef * 4096}, {coef * 64, coef * 64 * 4096}};
      return g;
    };
    ComponentClassProfile att;
    att.prefill = grid(3.0);
    att.decode = grid(0.5);
    cost.add_class(CostModel::class_key(ComponentKind::kAttention, dim), att);
    ComponentClassProfile ffn;
    ffn.prefill = grid(5.0);
    ffn.decode = grid(0.7);
    cost.add_class(CostModel::class_key(ComponentKind::kFfn, dim), ffn);
    std::vector<Request> reqs;
    for (int i = 0; i < n_requests; ++i) {
      Request r;
      r.id = (std::uint64_t)(i + 1);
      r.app_id = i;
      r.arrival_us = arrival_gap_us * i;
      r.prompt_tokens = prompts[i];
      r.output_tokens = outputs[i];
      if (prefix_group != nullptr) {
        r.prefix_group = prefix_group[i];
        r.prefix_tokens = prefix_tokens[i];
      }
      reqs.push_back(r);
    }
    ScenarioConfig cfg;
    cfg.name = "parity";
    cfg.speculation = false;
    cfg.adaptive = false;
    cfg.scaling = false;
    cfg.max_batch_tokens = max_batch_tokens;
    cfg.review_period_us = us_from_s(1e6);
    cfg.kv_review_period_us = us_from_s(1e6);
    cfg.metrics_tick_us = us_from_s(1e6);
    Simulation sim(cfg, zoo, cl, cost, reqs);
    // export zoo structure
    const auto& pz = sim.plan().zoo;
    std::map<std::string, int> bidx;
    for (const auto& b : pz.block_ids()) {
      bidx[b] = (int)h->blocks.size();
      h->blocks.push_back(b);
      std::string kinds;
      for (const auto& c : pz.block_components(b))
        kinds += c.kind == ComponentKind::kAttention ? "a" : "f";
      h->block_kinds.push_back(kinds);
    }
    for (const auto& mid : sim.plan().served_models) {
      std::vector<int> ch;
      for (const auto& b : sim.plan().chains.at(mid)) ch.push_back(bidx.at(b));
      h->chains.push_back(ch);
    }
    for (const auto& r : reqs)
      h->req_model.push_back((int)(r.app_id % sim.plan().served_models.size()));
    Simulation* sp = &sim;
    std::map<std::string, int> inst_index;
    sim.engine().set_trace_hook([h, sp, &bidx, &inst_index, gpu, &pz](SimTime, std::uint64_t,
                                                                      EventKind kind) {
      if (kind != EventKind::kBatchFinish) return;
      for (const auto& [dev, rb] : sp->running_) {
        const Instance* in = sp->pool().find(rb.instance_id);
        if (gpu != nullptr) {
          // the batch runs on the GPU now, before the reference advances its members
          std::string comps;
          for (const auto& c : pz.block_components(in->block_id))
            comps += c.kind == ComponentKind::kAttention ? "a" : "f";
          std::vector<rs_member> mem;
          for (const auto& m : rb.batch.members) {
            const auto& r = sp->live_.at(static_cast<std::uint64_t>(m.request_id));
            mem.push_back({(int32_t)m.request_id, m.chain_step, m.tokens, m.context_tokens,
                           m.chain_step + 1 == (int)r.chain->size() ? 1 : 0});
          }
          if (gpu->run(gpu->exec, in->block_id.c_str(), comps.c_str(),
                       rb.batch.phase == Phase::kDecode ? 1 : 0, (int)mem.size(), mem.data()) != 0)
            throw std::runtime_error(std::string("bh_executor_run_batch: ") + gpu->err(gpu->exec));
          ++gpu->batches;
        }
        auto it = inst_index.find(rb.instance_id);
        if (it == inst_index.end())
          it = inst_index.emplace(rb.instance_id, std::stoi(rb.instance_id.substr(1)) - 1).first;
        h->recs.emplace_back(it->second, bidx.at(in->block_id),
                             rb.batch.phase == Phase::kDecode ? 1 : 0);
        std::vector<std::tuple<int, int, int>> mem;
        for (const auto& m : rb.batch.members)
          mem.emplace_back(m.request_id, m.chain_step, m.context_tokens);
        h->members.push_back(mem);
      }
    });
    auto rep = sim.run();
    h->report = rep.dump();
  } catch (const std::exception& e) {
    h->err = e.what();
  }
}
void rs_sim_free(rs_sim* h) { delete h; }
const char* rs_sim_error(const rs_sim* h) { return h->err.c_str(); }
const char* rs_sim_report(const rs_sim* h) { return h->report.c_str(); }
int rs_sim_n_blocks(const rs_sim* h) { return (int)h->blocks.size(); }
const char* rs_sim_block_id(const rs_sim* h, int i) { return h->blocks[i].c_str(); }
const char* rs_sim_block_kinds(const rs_sim* h, int i) { return h->block_kinds[i].c_str(); }
int rs_sim_n_chains(const rs_sim* h) { return (int)h->chains.size(); }
int rs_sim_chain(const rs_sim* h, int m, int32_t* out, int cap) {
  const auto& c = h->chains[m];
  for (size_t i = 0; i < c.size() && (int)i < cap; ++i) out[i] = c[i];
  return (int)c.size();
}
int rs_sim_req_model(const rs_sim* h, int r) { return h->req_model[r]; }
int rs_sim_n_batches(const rs_sim* h) { return (int)h->recs.size(); }
// rec: [instance, block, phase, n_members]; members: (req, step, ctx) triples
int rs_sim_batch(const rs_sim* h, int i, int32_t* rec, int32_t* members, int cap) {
  rec[0] = std::get<0>(h->recs[i]);
  rec[1] = std::get<1>(h->recs[i]);
  rec[2] = std::get<2>(h->recs[i]);
  const auto& m = h->members[i];
  rec[3] = (int)m.size();
  for (size_t j = 0; j < m.size() && (int)j < cap; ++j) {
    members[3 * j] = std::get<0>(m[j]);
    members[3 * j + 1] = std::get<1>(m[j]);
    members[3 * j + 2] = std::get<2>(m[j]);
  }
  return 0;
}

// The reference's own profiles loader (config.cpp load_profiles) on a profiles.json, and its
// CostModel::component_us lookup at (class, phase, batch, tokens): checks that measured B200
// profiles (scripts/make_profiles.py) are accepted and read back as written.
int rs_profile_component_us(const char* path, const char* cls, int prefill, double batch,
                            double tokens, double* out, char* err, int err_cap) {
  try {
    blocksim::CostModel cm = blocksim::load_profiles(path);
    *out = cm.component_us(cls, prefill ? blocksim::Phase::kPrefill : blocksim::Phase::kDecode,
                           batch, tokens);
    return 0;
  } catch (const std::exception& e) {
    std::snprintf(err, err_cap, "%s", e.what());
    return 1;
  }
}


// ---------------------------------------------------------------- scheduler decisions in flight
// Runs a multi-device Simulation (LoRA + fully fine-tuned models with equivalence edges, memory
// tight enough to evict, speculation / scaling / placement reviews on) and, every `every`-th
// engine event, records the complete state the Scheduler reads plus its answers: choose_binding
// for every live request's current step, speculation_marks, scale_decisions, placement_moves,
// choose_device per block and preference, migration_rates, param_bytes_needed. Output is JSON;
// tests/test_policy.py replays each snapshot into bh_policy (include/blockpolicy.h).
struct rs_policy_trace {
  std::string out;
  std::string err;
};

namespace {
nlohmann::json grid_json(const Interp2D& g) {
  nlohmann::json v = nlohmann::json::array();
  for (const auto& row : g.v) v.push_back(row);
  return {{"xs", g.xs}, {"ys", g.ys}, {"v", v}};
}
nlohmann::json choice_json(const std::optional<BindingChoice>& c) {
  if (!c) return nullptr;
  return {{"block", c->block_id}, {"stitch", c->stitch_class}, {"instance", c->instance_id},
          {"device", c->device}, {"adaptive", c->adaptive}, {"evict", c->evict_bytes},
          {"est", {c->est.queue_us, c->est.compute_us, c->est.transfer_us, c->est.load_us}}};
}
}  // namespace

rs_policy_trace* rs_policy_trace_run(const char* spec_json) {
  auto* h = new rs_policy_trace();
  try {
    const auto spec = nlohmann::json::parse(spec_json);
    const int n_layers = spec.value("n_layers", 4), dim = spec.value("dim", 64);
    const int n_lora = spec.value("n_lora", 2), n_ff = spec.value("n_ff", 2);
    const int n_servers = spec.value("n_servers", 2), per_server = spec.value("per_server", 2);
    const std::int64_t capacity = spec.value("capacity", (std::int64_t)64 << 20);
    const std::int64_t att_bytes = spec.value("att_bytes", (std::int64_t)4 << 20);
    const std::int64_t ffn_bytes = spec.value("ffn_bytes", (std::int64_t)8 << 20);
    const int every = spec.value("every", 7), max_snaps = spec.value("max_snapshots", 60);
    std::uint64_t rng = spec.value("seed", 1);
    auto next = [&rng]() {  // splitmix64
      std::uint64_t z = (rng += 0x9E3779B97F4A7C15ull);
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      return z ^ (z >> 31);
    };
    auto unif = [&next]() { return (next() >> 11) * (1.0 / 9007199254740992.0); };

    Zoo zoo(0.98);
    std::vector<ComponentDescriptor> base;
    std::vector<LayerSignature> base_sigs;
    for (int l = 0; l < n_layers; ++l) {
      for (int k = 0; k < 2; ++k) {
        ComponentDescriptor c;
        c.id = "base." + std::string(k ? "ffn" : "att") + std::to_string(l);
        c.kind = k ? ComponentKind::kFfn : ComponentKind::kAttention;
        c.embed_dim = dim;
        c.model_id = "base";
        c.layer = l;
        c.slot = k;
        c.contents = {{c.id + ".w", k ? ffn_bytes : att_bytes}};
        base.push_back(c);
      }
      LayerSignature s{"base", l, {}};
      for (int i = 0; i < 8; ++i) s.probs.push_back(1.0 + i + 0.1 * l);
      base_sigs.push_back(s);
    }
    zoo.add_foundation("base", base);
    for (int v = 0; v < n_lora; ++v) {
      const std::string m = "lora" + std::to_string(v);
      const int first = 1 + v % std::max(1, n_layers - 1);
      std::vector<ComponentDescriptor> comps;
      for (int l = 0; l < n_layers; ++l) {
        if (l >= first) {
          ComponentDescriptor att;
          att.id = m + ".att" + std::to_string(l);
          att.kind = ComponentKind::kAttention;
          att.embed_dim = dim;
          att.model_id = m;
          att.layer = l;
          att.slot = 0;
          att.attach = "fuse";
          att.contents = {{"base.att" + std::to_string(l) + ".w", att_bytes},
                          {m + ".delta" + std::to_string(l), att_bytes / 64}};
          comps.push_back(att);
        } else {
          comps.push_back(zoo.component("base.att" + std::to_string(l)));
        }
        comps.push_back(zoo.component("base.ffn" + std::to_string(l)));
      }
      zoo.add_model_pe(m, TuningKind::kLora, "base", comps);
    }
    for (int v = 0; v < n_ff; ++v) {
      const std::string m = "ft" + std::to_string(v);
      std::vector<ComponentDescriptor> comps;
      std::vector<LayerSignature> sigs;
      for (int l = 0; l < n_layers; ++l) {
        for (int k = 0; k < 2; ++k) {
          ComponentDescriptor c;
          c.id = m + "." + std::string(k ? "ffn" : "att") + std::to_string(l);
          c.kind = k ? ComponentKind::kFfn : ComponentKind::kAttention;
          c.embed_dim = dim;
          c.model_id = m;
          c.layer = l;
          c.slot = k;
          c.contents = {{c.id + ".w", k ? ffn_bytes : att_bytes}};
          comps.push_back(c);
        }
        // the first (v+1) layers track the foundation (equivalent), the rest diverge
        LayerSignature s{m, l, base_sigs[l].probs};
        if (l > v) std::reverse(s.probs.begin(), s.probs.end());
        sigs.push_back(s);
      }
      zoo.add_model_ff(m, "base", comps, sigs, base_sigs);
    }

    Cluster cl;
    for (int s = 0; s < n_servers; ++s) cl.add_server({s, spec.value("intra_bps", 300e9)});
    cl.set_inter_default(spec.value("inter_bps", 25e9));
    if (n_servers >= 2) cl.set_inter_bandwidth(0, 1, spec.value("inter01_bps", 50e9));
    for (int s = 0; s < n_servers; ++s)
      for (int d = 0; d < per_server; ++d)
        cl.add_device({s * per_server + d, s, d % 2 ? "slow" : "fast",
                       capacity + (std::int64_t)(d * 3) * (1 << 20), 1e12,
                       spec.value("load_bps", 16e9)});
    CostModel cost;
    cost.set_device_class("fast", 1.0);
    cost.set_device_class("slow", 0.625);
    auto grid = [&](double coef, bool prefill) {
      Interp2D g;
      g.xs = {1, 4, 16, 64};
      g.ys = prefill ? std::vector<double>{1, 64, 512, 4096} : std::vector<double>{1, 256, 2048, 8192};
      for (double x : g.xs) {
        std::vector<double> row;
        for (double y : g.ys)
          row.push_back(coef * (prefill ? 0.5 * x * y : 20.0 + x + y / 64.0) * (0.9 + 0.2 * unif()));
        g.v.push_back(row);
      }
      return g;
    };
    ComponentClassProfile att{grid(3.0, true), grid(4.0, false), -1};
    ComponentClassProfile ffn{grid(5.0, true), grid(6.0, false), 0};
    cost.add_class(CostModel::class_key(ComponentKind::kAttention, dim), att);
    cost.add_class(CostModel::class_key(ComponentKind::kFfn, dim), ffn);

    std::vector<Request> reqs;
    const auto prompts = spec.at("prompts").get<std::vector<int>>();
    const auto outputs = spec.at("outputs").get<std::vector<int>>();
    const auto gaps = spec.at("gaps").get<std::vector<std::int64_t>>();
    SimTime t = 0;
    for (std::size_t i = 0; i < prompts.size(); ++i) {
      Request r;
      r.id = i + 1;
      r.app_id = (int)i;
      t += gaps[i];
      r.arrival_us = t;
      r.prompt_tokens = prompts[i];
      r.output_tokens = outputs[i];
      reqs.push_back(r);
    }
    ScenarioConfig cfg;
    cfg.name = "policy-parity";
    cfg.seed = spec.value("seed", 1);
    cfg.speculation = spec.value("speculation", true);
    cfg.spec_fraction = spec.value("spec_fraction", 0.25);
    cfg.adaptive = spec.value("adaptive", true);
    cfg.least_busy = spec.value("least_busy", false);
    cfg.placement = spec.value("frag_min", false) ? PlacementPolicy::kFragMin : PlacementPolicy::kLocality;
    cfg.scaling = spec.value("scaling", true);
    cfg.scale_queue_us = spec.value("scale_queue_us", (std::int64_t)3000);
    cfg.expected_tokens = spec.value("expected_tokens", 64);
    cfg.max_batch_tokens = spec.value("max_batch_tokens", 512);
    cfg.review_period_us = spec.value("review_period_us", (std::int64_t)5000);
    cfg.kv_review_period_us = spec.value("kv_review_period_us", (std::int64_t)2000);
    cfg.metrics_tick_us = us_from_s(1e6);

    Simulation sim(cfg, zoo, cl, cost, reqs);
    const Zoo& pz = sim.plan_.zoo;
    const CostModel& cm = sim.cost_;
    nlohmann::json st;
    st["config"] = {{"adaptive", cfg.adaptive}, {"least_busy", cfg.least_busy},
                    {"frag_min", cfg.placement == PlacementPolicy::kFragMin},
                    {"speculation", cfg.speculation}, {"spec_fraction", cfg.spec_fraction},
                    {"scale_queue_us", cfg.scale_queue_us}, {"expected_tokens", cfg.expected_tokens}};
    const auto& sr = cm.surrogate_;
    st["surrogate"] = {sr.attention_only, sr.ffn_only, sr.one_layer, sr.multi_layer,
                       sr.allow_adapter_blocks};
    for (const auto& [k, c] : cm.classes_)
      st["classes"][k] = {{"prefill", grid_json(c.prefill)}, {"decode", grid_json(c.decode)},
                          {"kv", c.kv_bytes_per_token}};
    st["stitches"] = nlohmann::json::object();
    for (const auto& [k, g] : cm.stitch_classes_) st["stitches"][k] = grid_json(g);
    for (const auto& [k, s] : cm.device_classes_) st["device_classes"][k] = s;
    std::set<std::string> comp_ids;
    for (const auto& b : pz.block_ids()) {
      const auto& bd = pz.block(b);
      nlohmann::json cands = nlohmann::json::array();
      auto cs = pz.candidate_instances(b);
      for (std::size_t i = 1; i < cs.size(); ++i)
        cands.push_back({cs[i].block_id,
                         cs[i].stitch_id.empty() ? "" : pz.stitch(cs[i].stitch_id).cost_class,
                         cs[i].score});
      st["blocks"].push_back({{"id", b}, {"comps", bd.component_ids},
                              {"dim_out", bd.embed_dim_out}, {"candidates", cands}});
      for (const auto& c : bd.component_ids) comp_ids.insert(c);
    }
    for (const auto& cid : comp_ids) {
      const auto& c = pz.component(cid);
      nlohmann::json pieces = nlohmann::json::array();
      for (const auto& p : c.contents) pieces.push_back({p.content_id, p.bytes});
      st["components"].push_back({{"id", cid}, {"kind", (int)c.kind}, {"dim", c.embed_dim},
                                  {"layer", c.layer}, {"pieces", pieces}});
    }
    for (const auto& mid : pz.model_ids()) st["chains"].push_back({mid, pz.model(mid).chain});
    for (const auto& [id, s] : sim.cluster_.servers_) st["servers"].push_back({id, s.intra_bandwidth_bps});
    st["inter_default"] = sim.cluster_.inter_default_;
    st["inter"] = nlohmann::json::array();
    for (const auto& [pr, b] : sim.cluster_.inter_) st["inter"].push_back({pr.first, pr.second, b});
    for (const auto& [id, d] : sim.cluster_.devices_)
      st["devices"].push_back({id, d.server, d.device_class, d.mem_capacity_bytes,
                               d.mem_bandwidth_bps, d.load_bandwidth_bps});

    nlohmann::json snaps = nlohmann::json::array();
    Simulation* sp = &sim;
    std::uint64_t n_events = 0;
    sim.engine().set_trace_hook([&](SimTime now, std::uint64_t, EventKind) {
      if (++n_events % (std::uint64_t)every != 0 || (int)snaps.size() >= max_snaps) return;
      const Simulation& s = *sp;
      nlohmann::json sn;
      sn["now"] = now;
      for (const auto& [id, in] : s.pool_.all())
        sn["instances"].push_back({{"id", id}, {"block", in.block_id}, {"device", in.device},
                                   {"ready", in.state == InstanceState::kReady},
                                   {"ready_at", in.ready_at}, {"last_used", in.last_used},
                                   {"created_seq", in.created_seq}, {"executing", in.executing},
                                   {"queue_len", (int)in.queue.size()},
                                   {"queued_cost", in.queued_cost_us},
                                   {"queued_hwm", in.queued_cost_hwm}});
      if (!sn.contains("instances")) sn["instances"] = nlohmann::json::array();
      for (const auto& [dev, res] : s.pool_.residency_)
        for (const auto& [cid, rc] : res)
          if (rc.first > 0) sn["residency"].push_back({dev, cid, rc.first});
      for (int dev : s.cluster_.device_ids()) {
        using C = MemoryLedger::Category;
        sn["ledger"].push_back({dev, s.ledger_.used(dev, C::kParams), s.ledger_.used(dev, C::kKv),
                                s.ledger_.used(dev, C::kActivation)});
        sn["lanes"].push_back({dev, s.pool_.lane(dev).busy_until});
      }
      sn["adjacency"] = nlohmann::json::array();
      for (const auto& [pr, n] : s.sched_.adjacency_) sn["adjacency"].push_back({pr.first, pr.second, n});
      sn["queries"] = nlohmann::json::array();
      for (const auto& [rid, r] : s.live_) {
        if (r.done || r.step < 0 || r.step >= (int)r.chain->size()) continue;
        BindingQuery q;
        q.request_id = rid;
        q.chain_block = (*r.chain)[(std::size_t)r.step];
        q.phase = r.phase;
        q.tokens = r.phase == Phase::kPrefill ? r.req.prompt_tokens : 1;
        q.context_tokens = r.context_tokens;
        q.from_device = r.from_device;
        q.now = now;
        const int owner = s.kv_.device_of(rid, q.chain_block);
        const int pages = owner >= 0 ? s.kv_.pages(rid, q.chain_block) : 0;
        nlohmann::json qj = {{"request", rid}, {"block", q.chain_block},
                             {"decode", q.phase == Phase::kDecode}, {"tokens", q.tokens},
                             {"context", q.context_tokens}, {"from", q.from_device},
                             {"kv_owner", owner}, {"kv_pages", pages}};
        try {
          qj["choice"] = choice_json(s.sched_.choose_binding(q));
        } catch (const std::exception& e) {
          qj["error"] = e.what();
        }
        sn["queries"].push_back(qj);
      }
      // synthetic steps for every block: a fresh prefill at chain entry and a decode hop from
      // device 1 (no cache yet) - these reach the new-instance / eviction paths
      std::uint64_t fresh = 1000000;
      for (const auto& b : s.plan_.zoo.block_ids()) {
        for (int k = 0; k < 2; ++k) {
          BindingQuery q;
          q.request_id = ++fresh;
          q.chain_block = b;
          q.phase = k ? Phase::kDecode : Phase::kPrefill;
          q.tokens = k ? 1 : 96;
          q.context_tokens = k ? 300 : 96;
          q.from_device = k ? 1 : -1;
          q.now = now;
          nlohmann::json qj = {{"request", q.request_id}, {"block", b}, {"decode", k == 1},
                               {"tokens", q.tokens}, {"context", q.context_tokens},
                               {"from", q.from_device}, {"kv_owner", -1}, {"kv_pages", 0}};
          try {
            qj["choice"] = choice_json(s.sched_.choose_binding(q));
          } catch (const std::exception& e) {
            qj["error"] = e.what();
          }
          sn["queries"].push_back(qj);
        }
      }
      // proactive KV review inputs (scenario.cpp:844-900) and the reference primitives' answers:
      // queued decode entries with remote caches, the interception tracker, and the migration
      // order kv_review's loop produces from them (order_migrations, predicted_remaining)
      sn["kvq"] = nlohmann::json::array();
      std::vector<MigrationCandidate> mcs;
      std::vector<int> picked;
      int qi = 0;
      for (const auto& [iid, inst] : s.pool_.all()) {
        for (const auto& e : inst.queue) {
          if (e.phase != Phase::kDecode) continue;
          const auto& r = s.live_.at((std::uint64_t)e.request_id);
          const std::string& cb = (*r.chain)[(std::size_t)e.chain_step];
          const int owner = s.kv_.device_of(r.req.id, cb);
          auto pend = s.tint_pending_.find({r.req.id, e.chain_step});
          const bool pending = pend != s.tint_pending_.end();
          nlohmann::json ej = {{"instance", iid}, {"inst_block", inst.block_id},
                               {"device", inst.device}, {"request", r.req.id}, {"chain_block", cb},
                               {"owner", owner},
                               {"pages", owner >= 0 ? s.kv_.pages(r.req.id, cb) : 0},
                               {"shared", owner >= 0 ? s.kv_.shared_pages(r.req.id, cb) : 0},
                               {"pending", pending},
                               {"pending_key", pending ? pend->second.first : std::string()},
                               {"t_call", pending ? pend->second.second : (SimTime)0}};
          sn["kvq"].push_back(ej);
          if (owner >= 0 && owner != inst.device) {
            auto [rec, cp] = s.sched_.migration_rates(inst.block_id, owner, inst.device);
            if (s.cfg_.kv_recalc_only) cp = 0;
            MigrationPlan plan = plan_migration(s.kv_.pages(r.req.id, cb), rec, cp);
            const std::string key = pending ? pend->second.first : inst.id;
            const SimTime t_call = pending ? pend->second.second : now;
            auto pred = s.tint_.predicted_remaining(key, t_call, now);
            if (pred.has_value() && *pred >= plan.completion_us) {
              MigrationCandidate mc;
              mc.request_id = r.req.id;
              mc.block_id = cb;
              mc.shared_pages = s.kv_.shared_pages(r.req.id, cb);
              mc.resume_time = t_call + *pred;
              mcs.push_back(mc);
              picked.push_back(qi);
            }
          }
          ++qi;
        }
      }
      std::vector<MigrationCandidate> ord = mcs;
      order_migrations(ord);
      sn["kv_review"] = nlohmann::json::array();
      for (const auto& mc : ord)
        for (std::size_t k = 0; k < mcs.size(); ++k)
          if (mcs[k].request_id == mc.request_id && mcs[k].block_id == mc.block_id) {
            sn["kv_review"].push_back(picked[k]);
            break;
          }
      sn["tint"] = {{"keys", nlohmann::json::array()},
                    {"global", {s.tint_.global_sum_, s.tint_.global_n_}}};
      for (const auto& [k, v] : s.tint_.per_key_) {
        sn["tint"]["keys"].push_back({k, v.first, v.second});
        for (SimTime dt : {(SimTime)0, (SimTime)500, (SimTime)5000}) {
          auto pr = s.tint_.predicted_remaining(k, now - dt, now);
          sn["tint_predict"].push_back({k, now - dt, pr.has_value() ? *pr : (SimTime)-1});
        }
      }
      sn["marks"] = s.sched_.speculation_marks();
      sn["scale"] = nlohmann::json::array();
      for (const auto& d : s.sched_.scale_decisions(now)) sn["scale"].push_back({d.instance_id, d.device});
      sn["moves"] = nlohmann::json::array();
      for (const auto& m : s.sched_.placement_moves()) sn["moves"].push_back({m.instance_id, m.dst_device});
      for (const auto& b : s.plan_.zoo.block_ids()) {
        for (int pref = 0; pref < 3; ++pref) {
          sn["devices"].push_back({b, pref, std::vector<int>{},
                                   s.sched_.choose_device(b, (DevicePreference)pref, {})});
          sn["devices"].push_back({b, pref, std::vector<int>{0},
                                   s.sched_.choose_device(b, (DevicePreference)pref, {0})});
        }
        for (int dev : s.cluster_.device_ids())
          sn["need"].push_back({b, dev, s.pool_.param_bytes_needed(b, dev)});
        const auto ids = s.cluster_.device_ids();
        for (std::size_t a = 0; a < ids.size(); ++a)
          for (std::size_t c = 0; c < ids.size(); ++c)
            if (a != c) {
              auto [rec, cp] = s.sched_.migration_rates(b, ids[a], ids[c]);
              sn["rates"].push_back({b, ids[a], ids[c], rec, cp});
            }
      }
      snaps.push_back(std::move(sn));
    });
    auto rep = sim.run();
    nlohmann::json out = {{"static", st}, {"snapshots", snaps}, {"events", n_events},
                          {"completed", rep.value("completed", nlohmann::json())}};
    h->out = out.dump();
  } catch (const std::exception& e) {
    h->err = e.what();
  }
  return h;
}
const char* rs_policy_trace_json(const rs_policy_trace* h) { return h->out.c_str(); }
const char* rs_policy_trace_error(const rs_policy_trace* h) { return h->err.c_str(); }
void rs_policy_trace_free(rs_policy_trace* h) { delete h; }

}  // extern "C"
