// Routing / speculation-marking / placement policy (see policy.hpp for the reference map).
#include "policy.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <tuple>

namespace bh {

namespace {
constexpr double kInf = std::numeric_limits<double>::infinity();
constexpr int kPageTokens = 16;  // kv.hpp:16

const char* kind_name(Kind k) {
  switch (k) {
    case Kind::kAttention: return "attention";
    case Kind::kFfn: return "ffn";
    case Kind::kEmbedding: return "embedding";
    case Kind::kLmHead: return "lm_head";
    case Kind::kAdapter: return "adapter";
  }
  return "unknown";
}

// cell: the largest i with axis[i] <= x, kept inside [0, n-2]; t: position inside the cell,
// clamped to [0, 1] (costmodel.cpp:15-32).
std::size_t cell(const std::vector<double>& a, double x) {
  if (a.size() < 2) return 0;
  const std::size_t hi = static_cast<std::size_t>(std::upper_bound(a.begin(), a.end(), x) - a.begin());
  if (hi == 0) return 0;
  return std::min(hi - 1, a.size() - 2);
}
double frac(const std::vector<double>& a, std::size_t i, double x) {
  if (a.size() < 2) return 0.0;
  if (x <= a[i]) return 0.0;
  if (x >= a[i + 1]) return 1.0;
  return (x - a[i]) / (a[i + 1] - a[i]);
}
}  // namespace

void Grid::check() const {
  if (xs.empty() || ys.empty()) throw PolicyError("empty interpolation axis");
  for (std::size_t i = 1; i < xs.size(); ++i)
    if (!(xs[i - 1] < xs[i])) throw PolicyError("interpolation axes must be strictly increasing");
  for (std::size_t i = 1; i < ys.size(); ++i)
    if (!(ys[i - 1] < ys[i])) throw PolicyError("interpolation axes must be strictly increasing");
  if (v.size() != xs.size() * ys.size()) throw PolicyError("interpolation grid size mismatch");
}

double Grid::at(double x, double y) const {
  const std::size_t i = cell(xs, x), j = cell(ys, y);
  const double tx = frac(xs, i, x), ty = frac(ys, j, y);
  const std::size_t i1 = xs.size() < 2 ? i : i + 1, j1 = ys.size() < 2 ? j : j + 1;
  const std::size_t ny = ys.size();
  const double a = v[i * ny + j], b = v[i * ny + j1], c = v[i1 * ny + j], d = v[i1 * ny + j1];
  // same association order as the reference's sum of the four weighted corners
  return a * (1 - tx) * (1 - ty) + b * (1 - tx) * ty + c * tx * (1 - ty) + d * tx * ty;
}

Migration plan_migration(int pages, std::int64_t rec, std::int64_t cp) {
  if (pages < 0) throw PolicyError("negative page count");
  if (rec < 0 || cp < 0) throw PolicyError("negative per-page cost");
  Migration m;
  m.pages = pages;
  if (pages == 0) return m;
  if (rec == 0 && cp == 0) throw PolicyError("both migration paths disabled");
  if (rec == 0) {
    m.copy_pages = pages;
    m.completion_us = static_cast<std::int64_t>(pages) * cp;
    return m;
  }
  if (cp == 0) {
    m.recompute_pages = pages;
    m.completion_us = static_cast<std::int64_t>(pages) * rec;
    return m;
  }
  // each page goes to the path that frees first; on a tie the cheaper path, then the copy path
  std::int64_t rfree = 0, cfree = 0;
  for (int k = 0; k < pages; ++k) {
    const bool to_rec = rfree != cfree ? rfree < cfree : (rec != cp && rec < cp);
    if (to_rec) {
      rfree += rec;
      ++m.recompute_pages;
    } else {
      cfree += cp;
      ++m.copy_pages;
    }
  }
  m.completion_us = std::max(rfree, cfree);
  return m;
}

// ------------------------------------------------------------------ static description
void Policy::add_cost_class(const std::string& key, Grid prefill, Grid decode, std::int64_t kv) {
  prefill.check();
  decode.check();
  if (!classes_.emplace(key, CostClass{std::move(prefill), std::move(decode), kv}).second)
    throw PolicyError("duplicate class: " + key);
}
void Policy::add_stitch_class(const std::string& key, Grid g) {
  g.check();
  if (!stitches_.emplace(key, std::move(g)).second) throw PolicyError("duplicate stitch class");
}
void Policy::set_device_class(const std::string& name, double speed) {
  if (speed <= 0.0) throw PolicyError("speed factor must be positive");
  dev_classes_[name] = speed;
}
void Policy::add_component(const std::string& id, Kind kind, int dim, int layer,
                           std::vector<std::pair<std::string, std::int64_t>> pieces) {
  Component c;
  c.kind = kind;
  c.embed_dim = dim;
  c.layer = layer;
  c.class_key = std::string(kind_name(kind)) + ":" + std::to_string(dim);
  c.pieces = std::move(pieces);
  comps_[id] = std::move(c);
}
void Policy::add_block(const std::string& id, std::vector<std::string> comps, int dim_out) {
  for (const auto& c : comps)
    if (!comps_.count(c)) throw PolicyError("unknown component " + c);
  Block b;
  b.comps = std::move(comps);
  b.embed_dim_out = dim_out;
  blocks_[id] = std::move(b);
}
void Policy::add_chain(const std::string& model, std::vector<std::string> chain) {
  for (const auto& b : chain) block(b);
  chains_.emplace_back(model, std::move(chain));
}
void Policy::add_candidate(const std::string& b, const std::string& cand, const std::string& st,
                           double score) {
  block(cand);
  blocks_.at(b).candidates.emplace_back(cand, st, score);
}
void Policy::add_server(int id, double bps) { servers_[id] = bps; }
void Policy::set_inter_bandwidth(int a, int b, double bps) {
  inter_[{std::min(a, b), std::max(a, b)}] = bps;
}
void Policy::add_device(int id, int server, const std::string& cls, std::int64_t cap,
                        double mem_bps, double load_bps) {
  if (!servers_.count(server)) throw PolicyError("unknown server " + std::to_string(server));
  devices_[id] = Device{server, cls, cap, mem_bps, load_bps};
  ledger_[id];
  lanes_[id];
}

// ------------------------------------------------------------------ dynamic state
void Policy::clear_state() {
  insts_.clear();
  for (auto& [d, l] : ledger_) l = Ledger{};
  for (auto& [d, t] : lanes_) t = 0;
  kv_.clear();
  adjacency_.clear();
}
void Policy::put_instance(const PolicyInstance& inst) {
  block(inst.block_id);
  device(inst.device);
  insts_[inst.id] = inst;
}
void Policy::remove_instance(const std::string& id) { insts_.erase(id); }
void Policy::set_ledger(int dev, std::int64_t params, std::int64_t kv, std::int64_t act) {
  device(dev);
  ledger_[dev] = Ledger{params, kv, act};
}
void Policy::set_lane(int dev, std::int64_t busy_until) {
  device(dev);
  lanes_[dev] = busy_until;
}
void Policy::set_kv(std::uint64_t req, const std::string& b, int owner, int pages) {
  if (owner < 0)
    kv_.erase({req, b});
  else
    kv_[{req, b}] = {owner, pages};
}
void Policy::set_adjacency(const std::string& from, const std::string& to, std::int64_t n) {
  adjacency_[{from, to}] = n;
}
void Policy::note_adjacency(const std::string& from, const std::string& to) {
  // scheduler.cpp:316-319: self and empty hops carry no locality signal
  if (from.empty() || to.empty() || from == to) return;
  adjacency_[{from, to}] += 1;
}

// ------------------------------------------------------------------ model queries
const Policy::Block& Policy::block(const std::string& id) const {
  auto it = blocks_.find(id);
  if (it == blocks_.end()) throw PolicyError("unknown block " + id);
  return it->second;
}
const Policy::Device& Policy::device(int id) const {
  auto it = devices_.find(id);
  if (it == devices_.end()) throw PolicyError("unknown device " + std::to_string(id));
  return it->second;
}
double Policy::speed(int dev) const {
  auto it = dev_classes_.find(device(dev).cls);
  if (it == dev_classes_.end()) throw PolicyError("unknown device class " + device(dev).cls);
  return it->second;
}
double Policy::path_bandwidth(int a, int b) const {
  if (a == b) return kInf;
  const Device &da = device(a), &db = device(b);
  const double ia = servers_.at(da.server);
  if (da.server == db.server) return ia;
  auto it = inter_.find({std::min(da.server, db.server), std::max(da.server, db.server)});
  const double inter = it != inter_.end() ? it->second : inter_default_;
  if (inter <= 0.0) throw PolicyError("no inter-server bandwidth configured");
  return std::min({ia, inter, servers_.at(db.server)});
}
double Policy::block_us(const std::string& b, bool decode, double batch, double tokens,
                        double sp) const {
  if (sp <= 0.0) throw PolicyError("speed factor must be positive");
  double sum = 0.0;
  for (const auto& cid : block(b).comps) {
    const Component& c = comps_.at(cid);
    auto it = classes_.find(c.class_key);
    if (it == classes_.end()) throw PolicyError("unknown component class: " + c.class_key);
    sum += (decode ? it->second.decode : it->second.prefill).at(batch, tokens);
  }
  return sum / sp;
}
std::int64_t Policy::kv_bytes_per_token(const std::string& b) const {
  std::int64_t n = 0;
  for (const auto& cid : block(b).comps) {
    const Component& c = comps_.at(cid);
    auto it = classes_.find(c.class_key);
    if (it != classes_.end() && it->second.kv_bpt >= 0)
      n += it->second.kv_bpt;
    else if (c.kind == Kind::kAttention)
      n += 4LL * c.embed_dim;  // K and V, 2 bytes each
  }
  return n;
}
std::optional<double> Policy::surrogate_speedup(const std::string& b) const {
  bool att = false, ffn = false, other = false, adapter = false;
  std::set<int> layers;
  for (const auto& cid : block(b).comps) {
    const Component& c = comps_.at(cid);
    layers.insert(c.layer);
    if (c.kind == Kind::kAttention) att = true;
    else if (c.kind == Kind::kFfn) ffn = true;
    else if (c.kind == Kind::kAdapter) adapter = true;
    else other = true;
  }
  if (adapter && !cfg_.sur_allow_adapter_blocks) return std::nullopt;
  if (att && !ffn && !other) return cfg_.sur_attention_only;
  if (ffn && !att && !other) return cfg_.sur_ffn_only;
  return layers.size() <= 1 ? cfg_.sur_one_layer : cfg_.sur_multi_layer;
}
std::int64_t Policy::free_bytes(int dev) const {
  const Ledger& l = ledger_.at(dev);
  return device(dev).capacity - (l.params + l.kv + l.act);
}
std::map<std::string, int> Policy::residency_refs(int dev) const {
  std::map<std::string, int> refs;
  for (const auto& [id, in] : insts_) {
    if (in.device != dev) continue;
    for (const auto& cid : block(in.block_id).comps)
      for (const auto& p : comps_.at(cid).pieces) refs[p.first] += 1;
  }
  return refs;
}
std::int64_t Policy::param_bytes_needed(const std::string& b, int dev) const {
  const auto refs = residency_refs(dev);
  std::int64_t need = 0;
  for (const auto& cid : block(b).comps)
    for (const auto& [content, bytes] : comps_.at(cid).pieces) {
      auto it = refs.find(content);
      if (it == refs.end() || it->second <= 0) need += bytes;
    }
  return need;
}
Policy::Eviction Policy::eviction_plan(int dev, std::int64_t bytes) const {
  Eviction e;
  if (bytes <= 0) return e;
  std::vector<const PolicyInstance*> idle;
  for (const auto& [id, in] : insts_)
    if (in.device == dev && !in.executing && in.queue_len == 0 && in.ready) idle.push_back(&in);
  std::sort(idle.begin(), idle.end(), [](const PolicyInstance* a, const PolicyInstance* b) {
    return std::tie(a->last_used, a->created_seq) < std::tie(b->last_used, b->created_seq);
  });
  auto refs = residency_refs(dev);
  // least recently used first; shared content frees only with its last holder
  for (const PolicyInstance* in : idle) {
    if (e.freed >= bytes) break;
    for (const auto& cid : block(in->block_id).comps)
      for (const auto& [content, sz] : comps_.at(cid).pieces)
        if (--refs[content] == 0) e.freed += sz;
  }
  e.ok = e.freed >= bytes;
  return e;
}
const PolicyInstance* Policy::find(const std::string& id) const {
  auto it = insts_.find(id);
  return it == insts_.end() ? nullptr : &it->second;
}
const PolicyInstance* Policy::instance_of(const std::string& b, int dev) const {
  for (const auto& [id, in] : insts_)
    if (in.block_id == b && in.device == dev) return &in;
  return nullptr;
}
bool Policy::chain_final(const std::string& b) const {
  for (const auto& [m, ch] : chains_)
    if (!ch.empty() && ch.back() == b) return true;
  return false;
}

std::pair<std::int64_t, std::int64_t> Policy::migration_rates(const std::string& b, int src,
                                                              int dst) const {
  // recompute: one 16-page prefill chunk on the destination, per page; copy: one page over the
  // path. Both at least 1 us.
  const double chunk = block_us(b, false, 1.0, 16.0 * kPageTokens, speed(dst));
  const std::int64_t rec = std::max<std::int64_t>(1, std::llround(chunk / 16.0));
  const std::int64_t page = kv_bytes_per_token(b) * kPageTokens;
  const double bw = path_bandwidth(src, dst);
  std::int64_t cp = 1;
  if (std::isfinite(bw) && bw > 0.0)
    cp = std::max<std::int64_t>(1, std::llround(static_cast<double>(page) / bw * 1e6));
  return {rec, cp};
}

// ------------------------------------------------------------------ decisions
Estimate Policy::estimate(const Query& q, const std::string& b, const std::string& stitch,
                          const PolicyInstance* inst, int dev, std::int64_t* evict_out) const {
  Estimate e;
  const double sp = speed(dev);
  e.compute_us = block_us(b, q.decode, 1.0, q.context_tokens, sp);
  if (!stitch.empty()) {
    auto it = stitches_.find(stitch);
    if (it == stitches_.end()) throw PolicyError("unknown stitch class: " + stitch);
    e.compute_us += it->second.at(1.0, q.context_tokens) / sp;
  }
  auto lane = lanes_.find(dev);
  const std::int64_t busy = lane == lanes_.end() ? 0 : lane->second;
  const double lane_rem = std::max(0.0, static_cast<double>(busy - q.now));
  e.queue_us = lane_rem + (inst ? inst->queued_cost_us : 0.0);

  double tx = 0.0;
  if (q.from_device >= 0 && q.from_device != dev) {
    const std::int64_t act = act_bytes_per_token(b) * (q.decode ? 1 : q.context_tokens);
    tx = static_cast<double>(act) / path_bandwidth(q.from_device, dev) * 1e6;
  }
  if (q.decode) {
    auto it = kv_.find({q.request_id, q.chain_block});
    if (it != kv_.end() && it->second.first >= 0 && it->second.first != dev) {
      const auto [rec, cp] = migration_rates(b, it->second.first, dev);
      tx += static_cast<double>(plan_migration(it->second.second, rec, cp).completion_us);
    }
  }
  e.transfer_us = tx;

  if (inst) {
    if (!inst->ready) {
      const double rem = std::max(0.0, static_cast<double>(inst->ready_at - q.now));
      e.load_us = lane_rem > 0.0 ? rem : std::max(0.0, rem - e.transfer_us);  // idle load path overlaps the hop
    }
    return e;
  }
  const std::int64_t need = param_bytes_needed(b, dev);
  std::int64_t evict = 0;
  const std::int64_t free = free_bytes(dev);
  if (need > free) {
    const Eviction ev = eviction_plan(dev, need - free);
    if (!ev.ok) {
      e.load_us = kInf;
      return e;
    }
    evict = ev.freed;
  }
  if (evict_out) *evict_out = evict;
  const Device& d = device(dev);
  const double swap = (static_cast<double>(evict) / d.mem_bps +
                       static_cast<double>(need) / d.load_bps) * 1e6;
  e.load_us = lane_rem > 0.0 ? swap : std::max(0.0, swap - e.transfer_us);
  return e;
}

std::optional<Choice> Policy::choose_binding(const Query& q) const {
  // candidates: self first, then the equivalents (adaptive only)
  std::vector<std::tuple<std::string, std::string, double>> cands;
  cands.emplace_back(q.chain_block, "", 1.0);
  if (cfg_.adaptive)
    for (const auto& c : block(q.chain_block).candidates) cands.push_back(c);

  struct Opt {
    Choice c;
    double score;
  };
  std::vector<Opt> opts;
  auto consider = [&](const std::string& b, const std::string& st, const PolicyInstance* in,
                      int dev) {
    std::int64_t evict = 0;
    const Estimate e = estimate(q, b, st, in, dev, &evict);
    if (!std::isfinite(e.total())) return;
    Opt o;
    o.c.block_id = b;
    o.c.stitch_class = st;
    o.c.instance_id = in ? in->id : "";
    o.c.device = dev;
    o.c.adaptive = b != q.chain_block;
    o.c.evict_bytes = evict;
    o.c.est = e;
    o.score = cfg_.least_busy ? e.queue_us : e.total();
    opts.push_back(std::move(o));
  };
  for (const auto& [b, st, score] : cands)
    for (const auto& [id, in] : insts_)
      if (in.block_id == b) consider(b, st, &in, in.device);

  // a decode step whose cache lives on a device with a ready candidate stays there
  if (q.decode && !cfg_.least_busy) {
    auto it = kv_.find({q.request_id, q.chain_block});
    if (it != kv_.end() && it->second.first >= 0) {
      std::vector<Opt> home;
      for (const auto& o : opts) {
        const PolicyInstance* in = find(o.c.instance_id);
        if (o.c.device == it->second.first && in && in->ready) home.push_back(o);
      }
      if (!home.empty()) opts.swap(home);
    }
  }
  if (opts.empty()) {
    // nothing serves any candidate yet: a new instance per candidate on its preferred device
    const DevicePref pref = cfg_.frag_min ? DevicePref::kTightestFit : DevicePref::kLocality;
    for (const auto& [b, st, score] : cands) {
      const int dev = choose_device(b, pref, {});
      if (dev >= 0) consider(b, st, nullptr, dev);
    }
  }
  if (opts.empty()) return std::nullopt;
  const Opt* best = &opts.front();
  auto key = [](const Opt& o) {
    return std::make_tuple(o.score, o.c.est.transfer_us, o.c.device, o.c.instance_id);
  };
  for (const auto& o : opts)
    if (key(o) < key(*best)) best = &o;
  return best->c;
}

std::vector<std::string> Policy::speculation_marks() const {
  if (!cfg_.speculation || cfg_.spec_fraction <= 0.0 || insts_.empty()) return {};
  std::vector<const PolicyInstance*> ranked;
  for (const auto& [id, in] : insts_) ranked.push_back(&in);
  std::sort(ranked.begin(), ranked.end(), [](const PolicyInstance* a, const PolicyInstance* b) {
    if (a->queued_cost_us != b->queued_cost_us) return a->queued_cost_us > b->queued_cost_us;
    return a->id < b->id;
  });
  const std::size_t want =
      static_cast<std::size_t>(std::ceil(cfg_.spec_fraction * static_cast<double>(ranked.size())));
  std::set<std::string> marked_blocks;
  std::vector<std::string> out;
  for (const PolicyInstance* in : ranked) {
    if (out.size() >= want) break;
    const std::string& b = in->block_id;
    if (!surrogate_speedup(b) || chain_final(b)) continue;
    bool next_to_marked = false;
    for (const auto& [m, ch] : chains_) {
      for (std::size_t i = 0; i + 1 < ch.size() && !next_to_marked; ++i)
        next_to_marked = (ch[i] == b && marked_blocks.count(ch[i + 1])) ||
                         (ch[i + 1] == b && marked_blocks.count(ch[i]));
      if (next_to_marked) break;
    }
    if (next_to_marked) continue;
    marked_blocks.insert(b);
    out.push_back(in->id);
  }
  return out;
}

std::int64_t Policy::max_queue_len(const PolicyInstance& in) const {
  const std::int64_t per_token = kv_bytes_per_token(in.block_id) + act_bytes_per_token(in.block_id);
  if (per_token <= 0) return std::numeric_limits<std::int64_t>::max();
  const std::int64_t request_mem = device(in.device).capacity - ledger_.at(in.device).params;
  if (request_mem <= 0) return 0;
  return request_mem / (static_cast<std::int64_t>(cfg_.expected_tokens) * per_token);
}

std::vector<std::pair<std::string, int>> Policy::scale_decisions() const {
  auto pressure = [](const PolicyInstance* in) {
    return std::max(in->queued_cost_us, in->queued_cost_hwm);
  };
  std::vector<const PolicyInstance*> hot;
  for (const auto& [id, in] : insts_) {
    const std::int64_t maxq = max_queue_len(in);
    const bool by_len = maxq != std::numeric_limits<std::int64_t>::max() &&
                        static_cast<double>(in.queue_len) > 0.8 * static_cast<double>(maxq);
    const bool by_delay =
        cfg_.scale_queue_us > 0 && pressure(&in) > static_cast<double>(cfg_.scale_queue_us);
    if (by_len || by_delay) hot.push_back(&in);
  }
  std::sort(hot.begin(), hot.end(), [&](const PolicyInstance* a, const PolicyInstance* b) {
    if (pressure(a) != pressure(b)) return pressure(a) > pressure(b);
    return a->id < b->id;
  });
  std::vector<std::pair<std::string, int>> out;
  std::map<std::string, std::set<int>> claimed;
  for (const PolicyInstance* in : hot) {
    const int dev = choose_device(in->block_id, DevicePref::kMostFree, claimed[in->block_id]);
    if (dev < 0) continue;
    out.emplace_back(in->id, dev);
    claimed[in->block_id].insert(dev);
  }
  return out;
}

int Policy::choose_device(const std::string& b, DevicePref pref, const std::set<int>& excl) const {
  std::vector<std::pair<int, std::int64_t>> ok;  // (device, free bytes), device order
  for (const auto& [dev, d] : devices_) {
    if (excl.count(dev) || instance_of(b, dev)) continue;
    const std::int64_t need = param_bytes_needed(b, dev), free = free_bytes(dev);
    if (need > free && !eviction_plan(dev, need - free).ok) continue;
    ok.emplace_back(dev, free);
  }
  if (ok.empty()) return -1;
  auto most_free = [&] {
    auto best = ok.begin();
    for (auto it = ok.begin(); it != ok.end(); ++it)
      if (it->second > best->second) best = it;
    return best->first;
  };
  if (pref == DevicePref::kTightestFit) {
    auto best = ok.begin();
    for (auto it = ok.begin(); it != ok.end(); ++it)
      if (it->second < best->second) best = it;
    return best->first;
  }
  if (pref == DevicePref::kLocality) {
    // observed hop counts plus one per static chain neighbour pair
    auto weight = adjacency_;
    for (const auto& [m, ch] : chains_)
      for (std::size_t i = 0; i + 1 < ch.size(); ++i) weight[{ch[i], ch[i + 1]}] += 1;
    int best = -1;
    std::int64_t best_score = -1, best_free = 0;
    for (const auto& [dev, free] : ok) {
      std::int64_t s = 0;
      for (const auto& [id, in] : insts_) {
        if (in.device != dev) continue;
        auto w = weight.find({in.block_id, b});
        if (w != weight.end()) s += w->second;
        w = weight.find({b, in.block_id});
        if (w != weight.end()) s += w->second;
      }
      if (best < 0 || s > best_score || (s == best_score && free > best_free)) {
        best = dev;
        best_score = s;
        best_free = free;
      }
    }
    if (best_score > 0) return best;
  }
  return most_free();
}

std::vector<std::pair<std::string, int>> Policy::placement_moves() const {
  if (cfg_.frag_min) return {};
  std::vector<std::pair<std::int64_t, std::pair<std::string, std::string>>> hot;
  for (const auto& [pr, n] : adjacency_) hot.push_back({n, pr});
  std::sort(hot.begin(), hot.end(), [](const auto& a, const auto& b) {
    if (a.first != b.first) return a.first > b.first;
    return a.second < b.second;
  });
  std::vector<std::pair<std::string, int>> moves;
  std::set<std::string> moved;
  std::set<int> targeted;
  auto idle = [&](const PolicyInstance* i) {
    return !i->executing && i->queue_len == 0 && i->ready && !moved.count(i->id);
  };
  auto fits = [&](const std::string& blk, int dev) {
    if (instance_of(blk, dev)) return false;
    const std::int64_t need = param_bytes_needed(blk, dev), free = free_bytes(dev);
    return need <= free || eviction_plan(dev, need - free).ok;
  };
  auto of_block = [&](const std::string& blk) {
    std::vector<const PolicyInstance*> v;
    for (const auto& [id, in] : insts_)
      if (in.block_id == blk) v.push_back(&in);
    return v;
  };
  // co-locate the hottest cross-server adjacent pair: move whichever side is idle and fits
  for (const auto& [n, pr] : hot) {
    if (moves.size() >= 2 || n <= 0) break;
    for (const PolicyInstance* a : of_block(pr.first)) {
      if (moves.size() >= 2) break;
      for (const PolicyInstance* b : of_block(pr.second)) {
        if (moves.size() >= 2) break;
        if (same_server(a->device, b->device)) continue;
        if (targeted.count(a->device) + targeted.count(b->device) > 0) continue;
        if (idle(b) && fits(b->block_id, a->device)) {
          moves.emplace_back(b->id, a->device);
          moved.insert(b->id);
          targeted.insert(a->device);
        } else if (idle(a) && fits(a->block_id, b->device)) {
          moves.emplace_back(a->id, b->device);
          moved.insert(a->id);
          targeted.insert(b->device);
        }
      }
    }
  }
  return moves;
}

// ------------------------------------------------------------------ proactive KV review
void Interception::record(const std::string& key, std::int64_t sample) {
  if (sample < 0) throw PolicyError("negative interception sample");
  auto& [sum, n] = per_key_[key];
  sum += static_cast<double>(sample);
  ++n;
  global_sum_ += static_cast<double>(sample);
  ++global_n_;
}
std::optional<double> Interception::mean(const std::string& key) const {
  auto it = per_key_.find(key);
  if (it == per_key_.end() || it->second.second == 0) return std::nullopt;
  return it->second.first / static_cast<double>(it->second.second);
}
std::optional<double> Interception::global_mean() const {
  if (global_n_ == 0) return std::nullopt;
  return global_sum_ / static_cast<double>(global_n_);
}
std::optional<std::int64_t> Interception::predicted_remaining(const std::string& key,
                                                              std::int64_t t_call,
                                                              std::int64_t now) const {
  auto m = mean(key);
  if (!m) m = global_mean();
  if (!m) return std::nullopt;
  const double left = std::max(0.0, *m - static_cast<double>(now - t_call));
  return static_cast<std::int64_t>(std::llround(left));  // round_us, time.hpp:22-25
}

void order_migrations(std::vector<MigrationCandidate>& c) {
  std::sort(c.begin(), c.end(), [](const MigrationCandidate& a, const MigrationCandidate& b) {
    return std::tie(a.shared_pages, a.resume_time, a.request_id, a.block_id) <
           std::tie(b.shared_pages, b.resume_time, b.request_id, b.block_id);
  });
}

std::vector<int> Policy::kv_review(const std::vector<QueuedDecode>& q, const Interception& tint,
                                   std::int64_t now, bool recalc_only) const {
  std::vector<int> picked;
  std::vector<MigrationCandidate> cands;
  for (int i = 0; i < (int)q.size(); ++i) {
    const QueuedDecode& e = q[i];
    if (e.owner < 0 || e.owner == e.device) continue;
    auto [rec, cp] = migration_rates(e.inst_block, e.owner, e.device);
    if (recalc_only) cp = 0;
    const Migration plan = plan_migration(e.pages, rec, cp);
    const std::string& key = e.pending ? e.pending_key : e.instance;
    const std::int64_t t_call = e.pending ? e.t_call : now;
    const auto left = tint.predicted_remaining(key, t_call, now);
    if (!left || *left < plan.completion_us) continue;  // would not finish before it is needed
    picked.push_back(i);
    cands.push_back({e.request_id, e.chain_block, e.shared_pages, t_call + *left});
  }
  std::vector<MigrationCandidate> order = cands;
  order_migrations(order);
  std::vector<int> out;
  for (const auto& mc : order)
    for (std::size_t k = 0; k < cands.size(); ++k)
      if (cands[k].request_id == mc.request_id && cands[k].block_id == mc.block_id) {
        out.push_back(picked[k]);  // the first queued entry of that (request, block)
        break;
      }
  return out;
}

}  // namespace bh
