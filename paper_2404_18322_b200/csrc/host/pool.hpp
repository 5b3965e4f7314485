// Host control plane, part 1: block instances and their queues — the gather rule that forms
// per-block batches. Mirrors the semantics of blocksim's InstancePool queue mechanics
// (proj/core/include/blocksim/agent.hpp:20-140, src/agent.cpp:132-224) so batch membership,
// order and arbitration are bit-identical to the reference; parameter residency / LRU eviction
// (agent.cpp:29-130) is not on the execution path and is not mirrored here.
#pragma once
#include <cstdint>
#include <deque>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace bh {

enum class Phase : int { kPrefill = 0, kDecode = 1 };

// One queued (request, chain-step) row (agent.hpp:20-30).
struct Entry {
  int request_id = -1;
  int chain_step = -1;
  Phase phase = Phase::kPrefill;
  int tokens = 0;          // batch-budget weight: prompt length (prefill) or 1 (decode)
  int context_tokens = 0;  // sequence length seen by the block
  double est_cost_us = 0.0;
  std::uint64_t enqueue_seq = 0;
  bool kv_resident = false;  // priority segment
  int stitch_class = -1;
};

struct Batch {
  std::vector<Entry> members;
  Phase phase = Phase::kPrefill;
  int max_context_tokens() const {
    int m = 0;
    for (const auto& e : members) m = e.context_tokens > m ? e.context_tokens : m;
    return m;
  }
};

struct Instance {
  std::string id;        // "i<N>" (agent.cpp:61)
  std::string block_id;
  int device = -1;
  bool ready = false;
  std::int64_t ready_at = 0;
  std::int64_t last_used = 0;
  bool executing = false;
  std::deque<Entry> queue;
  double queued_cost_us = 0.0;
  double queued_cost_hwm = 0.0;
  std::uint64_t created_seq = 0;
};

// std::logic_error in the reference (agent.cpp:9)
struct PoolError : std::logic_error {
  explicit PoolError(const std::string& w) : std::logic_error("pool: " + w) {}
};

class Pool {
 public:
  Instance& create(const std::string& block_id, int device, std::int64_t now,
                   std::int64_t ready_at);
  void mark_ready(const std::string& id, std::int64_t now);
  void enqueue(const std::string& id, Entry e);
  std::vector<Entry> remove_queued(const std::string& id, int request_id);
  std::vector<Entry> take_tail(const std::string& id, std::size_t count);
  Batch pop_batch(const std::string& id, int max_batch_tokens, std::int64_t now);
  void finish_batch(const std::string& id, std::int64_t now);
  // Continuous batching: every queued decode entry of `id` boards `running` (the batch the
  // instance is executing) in queue order (scenario.cpp:438-463, try_join_running).
  std::vector<Entry> join_running(const std::string& id, Batch& running);
  Instance* next_runnable(int device, std::int64_t now);
  Instance* find(const std::string& id);
  Instance& get(const std::string& id);
  Instance* instance_of(const std::string& block_id, int device);
  const std::map<std::string, Instance>& all() const { return instances_; }
  std::uint64_t next_enqueue_seq() { return ++enqueue_seq_; }

 private:
  std::map<std::string, Instance> instances_;  // lexicographic id order, as the reference
  std::uint64_t next_instance_ = 0;
  std::uint64_t enqueue_seq_ = 0;
  std::uint64_t created_seq_ = 0;
};

}  // namespace bh
