// Queue mechanics of block instances; see pool.hpp for the reference mapping.
#include "pool.hpp"

#include <algorithm>

namespace bh {

Instance& Pool::create(const std::string& block_id, int device, std::int64_t now,
                       std::int64_t ready_at) {
  if (instance_of(block_id, device) != nullptr)
    throw PoolError("device " + std::to_string(device) + " already serves " + block_id);
  Instance inst;
  inst.id = "i" + std::to_string(++next_instance_);
  inst.block_id = block_id;
  inst.device = device;
  inst.ready = !(ready_at > now);
  inst.ready_at = ready_at;
  inst.last_used = now;
  inst.created_seq = ++created_seq_;
  auto res = instances_.emplace(inst.id, std::move(inst));
  if (!res.second) throw PoolError("duplicate instance id");
  return res.first->second;
}

Instance* Pool::find(const std::string& id) {
  auto it = instances_.find(id);
  return it == instances_.end() ? nullptr : &it->second;
}

Instance& Pool::get(const std::string& id) {
  Instance* p = find(id);
  if (p == nullptr) throw PoolError("unknown instance " + id);
  return *p;
}

Instance* Pool::instance_of(const std::string& block_id, int device) {
  for (auto& kv : instances_)
    if (kv.second.block_id == block_id && kv.second.device == device) return &kv.second;
  return nullptr;
}

void Pool::mark_ready(const std::string& id, std::int64_t now) {
  Instance& in = get(id);
  in.ready = true;
  in.ready_at = std::min(in.ready_at, now);
}

void Pool::enqueue(const std::string& id, Entry e) {
  Instance& in = get(id);
  e.enqueue_seq = next_enqueue_seq();
  in.queued_cost_us += e.est_cost_us;
  in.queued_cost_hwm = std::max(in.queued_cost_hwm, in.queued_cost_us);
  if (e.kv_resident) {
    // resident decode work forms a stable priority segment ahead of everything else
    auto pos = in.queue.begin();
    while (pos != in.queue.end() && pos->kv_resident) ++pos;
    in.queue.insert(pos, e);
  } else {
    in.queue.push_back(e);
  }
}

std::vector<Entry> Pool::remove_queued(const std::string& id, int request_id) {
  Instance& in = get(id);
  std::vector<Entry> out;
  std::deque<Entry> keep;
  for (auto& e : in.queue) {
    if (e.request_id == request_id) {
      in.queued_cost_us -= e.est_cost_us;
      out.push_back(e);
    } else {
      keep.push_back(e);
    }
  }
  in.queue.swap(keep);
  return out;
}

std::vector<Entry> Pool::take_tail(const std::string& id, std::size_t count) {
  Instance& in = get(id);
  count = std::min(count, in.queue.size());
  std::vector<Entry> out(in.queue.end() - static_cast<std::ptrdiff_t>(count), in.queue.end());
  for (std::size_t i = 0; i < count; ++i) {
    in.queued_cost_us -= in.queue.back().est_cost_us;
    in.queue.pop_back();
  }
  if (in.queue.empty()) in.queued_cost_us = 0.0;
  return out;
}

Batch Pool::pop_batch(const std::string& id, int max_batch_tokens, std::int64_t now) {
  Instance& in = get(id);
  if (in.queue.empty()) throw PoolError(id + ": pop from empty queue");
  if (in.executing) throw PoolError(id + " is already executing");
  // Longest queue prefix in the head's phase whose budget tokens fit; an oversized head still
  // runs alone (agent.cpp:182-204).
  Batch b;
  b.phase = in.queue.front().phase;
  long long used = 0;
  while (!in.queue.empty()) {
    const Entry& head = in.queue.front();
    if (head.phase != b.phase) break;
    if (!b.members.empty() && used + head.tokens > max_batch_tokens) break;
    used += head.tokens;
    in.queued_cost_us -= head.est_cost_us;
    b.members.push_back(head);
    in.queue.pop_front();
  }
  if (in.queue.empty()) in.queued_cost_us = 0.0;
  in.executing = true;
  in.last_used = now;
  return b;
}

void Pool::finish_batch(const std::string& id, std::int64_t now) {
  Instance& in = get(id);
  if (!in.executing) throw PoolError(id + " is not executing");
  in.executing = false;
  in.last_used = now;
}

std::vector<Entry> Pool::join_running(const std::string& id, Batch& running) {
  Instance& in = get(id);
  std::vector<Entry> joined;
  if (running.phase != Phase::kDecode) return joined;
  for (auto it = in.queue.begin(); it != in.queue.end();) {
    if (it->phase != Phase::kDecode) {
      ++it;
      continue;
    }
    Entry e = *it;
    it = in.queue.erase(it);
    in.queued_cost_us = std::max(0.0, in.queued_cost_us - e.est_cost_us);
    running.members.push_back(e);
    joined.push_back(e);
  }
  return joined;
}

Instance* Pool::next_runnable(int device, std::int64_t now) {
  // among ready idle instances of the device, the one whose head entered earliest
  Instance* best = nullptr;
  for (auto& kv : instances_) {
    Instance& in = kv.second;
    if (in.device != device || in.executing || in.queue.empty()) continue;
    if (!in.ready || in.ready_at > now) continue;
    if (best == nullptr || in.queue.front().enqueue_seq < best->queue.front().enqueue_seq)
      best = &in;
  }
  return best;
}

}  // namespace bh
