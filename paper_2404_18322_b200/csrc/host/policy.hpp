// Host control plane, part 3: the routing / speculation-marking / placement policy (§8 rows
// a10, a14, a15). Decides, over a snapshot of the serving state, which block instance a chain
// step binds to, which instances get a draft surrogate, and where new or moved instances go.
//
// Mirrors blocksim's Scheduler decision functions with identical arithmetic and tie-breaks:
//   estimate          scheduler.cpp:23-78   (queue + compute + transfer + load, in us)
//   choose_binding    scheduler.cpp:80-160  (argmin (score, transfer, device, instance id);
//                                            decode sticks to the KV owner's ready instances)
//   speculation_marks scheduler.cpp:180-215 (top ceil(f*N) by queued cost, skip chain-final /
//                                            surrogate-less / chain-adjacent-to-marked blocks)
//   scale_decisions   scheduler.cpp:217-260; choose_device :262-314; placement_moves :321-366;
//   migration_rates   scheduler.cpp:368-381; plan_migration kv.cpp:16-58;
//   block_us / stitch_us / surrogate_speedup / Interp2D  costmodel.cpp:50-151;
//   path_bandwidth    cluster.cpp:65-75; param_bytes_needed / eviction_plan agent.cpp:29-109.
//
// The state is a plain snapshot (instances, ledger, lanes, KV owners, adjacency) the host
// updates as it runs; every decision is a pure function of it. Parity: tests/test_policy.py
// replays snapshots taken inside the reference's own running Simulation (oracle/ref_shim.cpp)
// and requires every decision to match exactly.
#pragma once
#include <cstdint>
#include <map>
#include <optional>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace bh {

struct PolicyError : std::invalid_argument {
  explicit PolicyError(const std::string& w) : std::invalid_argument("policy: " + w) {}
};

// Bilinear table over (batch, tokens), clamped to the grid (costmodel.cpp:15-59).
struct Grid {
  std::vector<double> xs, ys;
  std::vector<double> v;  // row-major [xs.size()][ys.size()]
  double at(double x, double y) const;
  void check() const;
};

enum class Kind : int { kAttention = 0, kFfn = 1, kEmbedding = 2, kLmHead = 3, kAdapter = 4 };

struct PolicyConfig {
  bool adaptive = true;
  bool least_busy = false;
  bool frag_min = false;  // placement policy: false = locality, true = tightest fit
  bool speculation = true;
  double spec_fraction = 0.10;
  std::int64_t scale_queue_us = 0;
  int expected_tokens = 256;
  double sur_attention_only = 37.43, sur_ffn_only = 1.71, sur_one_layer = 22.91,
         sur_multi_layer = 18.55;
  bool sur_allow_adapter_blocks = false;
};

struct Query {
  std::uint64_t request_id = 0;
  std::string chain_block;
  bool decode = false;
  int tokens = 0;
  int context_tokens = 0;
  int from_device = -1;
  std::int64_t now = 0;
};

struct Estimate {
  double queue_us = 0, compute_us = 0, transfer_us = 0, load_us = 0;
  double total() const { return queue_us + compute_us + transfer_us + load_us; }
};

struct Choice {
  std::string block_id, stitch_class, instance_id;  // instance empty: create on `device`
  int device = -1;
  bool adaptive = false;
  std::int64_t evict_bytes = 0;
  Estimate est;
};

struct PolicyInstance {
  std::string id, block_id;
  int device = -1;
  bool ready = false;
  std::int64_t ready_at = 0, last_used = 0;
  std::uint64_t created_seq = 0;
  bool executing = false;
  int queue_len = 0;
  double queued_cost_us = 0, queued_cost_hwm = 0;
};

enum class DevicePref : int { kLocality = 0, kTightestFit = 1, kMostFree = 2 };

struct Migration {
  int pages = 0, recompute_pages = 0, copy_pages = 0;
  std::int64_t completion_us = 0;
};
// Two-path page migration (recompute on the destination vs copy over the path), greedy
// earliest-free claim per page (kv.cpp:16-58).
Migration plan_migration(int pages, std::int64_t rec_us_per_page, std::int64_t cp_us_per_page);

// Idle-time predictor for parked KV (InterceptionTracker, kv.cpp:70-103): mean of the observed
// gaps per key (instance id), the global mean as the fallback.
class Interception {
 public:
  void record(const std::string& key, std::int64_t sample);
  void set(const std::string& key, double sum, std::uint64_t n) { per_key_[key] = {sum, n}; }
  void set_global(double sum, std::uint64_t n) {
    global_sum_ = sum;
    global_n_ = n;
  }
  std::optional<double> mean(const std::string& key) const;
  std::optional<double> global_mean() const;
  std::optional<std::int64_t> predicted_remaining(const std::string& key, std::int64_t t_call,
                                                  std::int64_t now) const;

 private:
  std::map<std::string, std::pair<double, std::uint64_t>> per_key_;
  double global_sum_ = 0.0;
  std::uint64_t global_n_ = 0;
};

struct MigrationCandidate {
  std::uint64_t request_id = 0;
  std::string block_id;
  int shared_pages = 0;
  std::int64_t resume_time = 0;
};
// fewest shared pages first, then earliest resumption, then ids (kv.cpp:60-68)
void order_migrations(std::vector<MigrationCandidate>& c);

// A queued decode entry seen by the proactive KV review (scenario.cpp:844-900)
struct QueuedDecode {
  std::string instance, inst_block;  // the instance holding the entry, its serving block
  int device = -1;                   // that instance's device
  std::uint64_t request_id = 0;
  std::string chain_block;           // the request chain's block at this step
  int owner = -1, pages = 0, shared_pages = 0;  // the cache segment of (request, chain block)
  bool pending = false;              // an interception sample is open for this step
  std::string pending_key;
  std::int64_t t_call = 0;
};

class Policy {
 public:
  explicit Policy(PolicyConfig cfg) : cfg_(cfg) {}

  // ---- static description: cost model, zoo structure, cluster
  void add_cost_class(const std::string& key, Grid prefill, Grid decode, std::int64_t kv_bpt);
  void add_stitch_class(const std::string& key, Grid g);
  void set_device_class(const std::string& name, double speed);
  void add_component(const std::string& id, Kind kind, int embed_dim, int layer,
                     std::vector<std::pair<std::string, std::int64_t>> pieces);
  void add_block(const std::string& id, std::vector<std::string> components, int embed_dim_out);
  void add_chain(const std::string& model, std::vector<std::string> blocks);
  // Serving candidates of a chain block after itself (Zoo::candidate_instances, zoo.cpp:568-589,
  // resolved by the host: equivalents, with the stitch cost class when dims differ).
  void add_candidate(const std::string& block, const std::string& cand,
                     const std::string& stitch_class, double score);
  void add_server(int id, double intra_bps);
  void set_inter_bandwidth(int a, int b, double bps);
  void set_inter_default(double bps) { inter_default_ = bps; }
  void add_device(int id, int server, const std::string& cls, std::int64_t capacity,
                  double mem_bps, double load_bps);

  // ---- dynamic state
  void clear_state();
  void put_instance(const PolicyInstance& inst);
  void remove_instance(const std::string& id);
  void set_ledger(int dev, std::int64_t params, std::int64_t kv, std::int64_t act);
  void set_lane(int dev, std::int64_t busy_until);
  void set_kv(std::uint64_t request, const std::string& block, int owner, int pages);
  void set_adjacency(const std::string& from, const std::string& to, std::int64_t count);
  void note_adjacency(const std::string& from, const std::string& to);

  // ---- decisions
  Estimate estimate(const Query& q, const std::string& block, const std::string& stitch_class,
                    const PolicyInstance* inst, int device, std::int64_t* evict_out) const;
  std::optional<Choice> choose_binding(const Query& q) const;
  std::vector<std::string> speculation_marks() const;
  std::vector<std::pair<std::string, int>> scale_decisions() const;
  int choose_device(const std::string& block, DevicePref pref, const std::set<int>& excl) const;
  std::vector<std::pair<std::string, int>> placement_moves() const;
  std::pair<std::int64_t, std::int64_t> migration_rates(const std::string& block, int src,
                                                        int dst) const;
  std::int64_t max_queue_len(const PolicyInstance& inst) const;
  // Proactive migrations (Simulation::kv_review, scenario.cpp:844-900): entries whose cache is
  // remote and predicted to stay idle long enough for the planned move; returned as indices
  // into `q`, in migration order.
  std::vector<int> kv_review(const std::vector<QueuedDecode>& q, const Interception& tint,
                             std::int64_t now, bool recalc_only) const;

  // ---- model queries (costmodel.cpp)
  double block_us(const std::string& block, bool decode, double batch, double tokens,
                  double speed) const;
  std::optional<double> surrogate_speedup(const std::string& block) const;
  std::int64_t param_bytes_needed(const std::string& block, int device) const;
  std::int64_t free_bytes(int dev) const;
  const PolicyInstance* find(const std::string& id) const;
  const std::map<std::string, PolicyInstance>& instances() const { return insts_; }

 private:
  struct Component {
    Kind kind = Kind::kAttention;
    int embed_dim = 0, layer = 0;
    std::string class_key;
    std::vector<std::pair<std::string, std::int64_t>> pieces;
  };
  struct Block {
    std::vector<std::string> comps;
    int embed_dim_out = 0;
    std::vector<std::tuple<std::string, std::string, double>> candidates;  // (block, stitch, score)
  };
  struct CostClass {
    Grid prefill, decode;
    std::int64_t kv_bpt = -1;
  };
  struct Device {
    int server = 0;
    std::string cls;
    std::int64_t capacity = 0;
    double mem_bps = 0, load_bps = 0;
  };
  struct Ledger {
    std::int64_t params = 0, kv = 0, act = 0;
  };
  struct Eviction {
    bool ok = true;
    std::int64_t freed = 0;
  };

  const Block& block(const std::string& id) const;
  const Device& device(int id) const;
  double speed(int dev) const;
  double path_bandwidth(int a, int b) const;
  bool same_server(int a, int b) const { return device(a).server == device(b).server; }
  std::int64_t kv_bytes_per_token(const std::string& block) const;
  std::int64_t act_bytes_per_token(const std::string& b) const { return 2LL * block(b).embed_dim_out; }
  Eviction eviction_plan(int dev, std::int64_t bytes) const;
  bool chain_final(const std::string& block) const;
  const PolicyInstance* instance_of(const std::string& block, int dev) const;
  std::map<std::string, int> residency_refs(int dev) const;

  PolicyConfig cfg_;
  std::map<std::string, CostClass> classes_;
  std::map<std::string, Grid> stitches_;
  std::map<std::string, double> dev_classes_;
  std::map<std::string, Component> comps_;
  std::map<std::string, Block> blocks_;
  std::vector<std::pair<std::string, std::vector<std::string>>> chains_;  // registration order
  std::map<int, double> servers_;
  std::map<std::pair<int, int>, double> inter_;
  double inter_default_ = 0.0;
  std::map<int, Device> devices_;

  std::map<std::string, PolicyInstance> insts_;
  std::map<int, Ledger> ledger_;
  std::map<int, std::int64_t> lanes_;
  std::map<std::pair<std::uint64_t, std::string>, std::pair<int, int>> kv_;  // owner, pages
  std::map<std::pair<std::string, std::string>, std::int64_t> adjacency_;
};

}  // namespace bh
