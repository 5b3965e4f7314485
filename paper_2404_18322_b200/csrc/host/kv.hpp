// Host control plane, part 2: the block-local paged KV store and its GPU page tables.
// Mirrors blocksim's KvStore (proj/core/include/blocksim/kv.hpp:72-128, src/kv.cpp:105-237):
// one segment per (request, chain block) on one device, ceil(tokens/16) pages, global page ids
// from 1 (kv.hpp:126), prefix pages shared by reference count, shared pages duplicated when a
// segment moves. On top of the reference's bookkeeping every page id is bound to a physical
// slot of the (block, device) KV pool on the GPU, so a segment's page ids become the page-table
// row the attention kernel walks.
#pragma once
#include <cstdint>
#include <map>
#include <unordered_map>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace bh {

constexpr int kPageTokens = 16;

struct KvError : std::invalid_argument {
  explicit KvError(const std::string& w) : std::invalid_argument("kv: " + w) {}
};
// over-capacity / negative release (MemoryLedger, cluster.cpp:135-152, std::logic_error)
struct LedgerError : std::logic_error {
  explicit LedgerError(const std::string& w) : std::logic_error("ledger: " + w) {}
};

// Physical slot allocator of one (block, device) KV pool: lowest free slot first.
class SlotPool {
 public:
  explicit SlotPool(int n = 0) {
    for (int i = 0; i < n; ++i) free_.insert(i);
    size_ = n;
  }
  int alloc() {
    if (free_.empty()) return -1;
    const int s = *free_.begin();
    free_.erase(free_.begin());
    return s;
  }
  void release(int s) {
    if (s >= 0) free_.insert(s);
  }
  int size() const { return size_; }
  int free_count() const { return static_cast<int>(free_.size()); }

 private:
  std::set<int> free_;
  int size_ = 0;
};

class KvStore {
 public:
  // Registers the GPU pool backing segments of `pool_key` (the serving block) on `device`.
  void attach_pool(const std::string& pool_key, int device, int n_pages);
  // Optional per-device KV capacity in bytes (ledger guard); unlimited when unset.
  void set_capacity(int device, std::int64_t bytes) { capacity_[device] = bytes; }

  void create_segment(std::uint64_t request, const std::string& block, int device,
                      std::int64_t bytes_per_token, const std::string& pool_key = "");
  bool has_segment(std::uint64_t request, const std::string& block) const;
  int append_tokens(std::uint64_t request, const std::string& block, int n);
  // append_tokens on the segment if it exists (one lookup); false when there is none
  bool append_if_present(std::uint64_t request, const std::string& block, int n);
  int share_prefix(std::uint64_t request, std::uint64_t from, const std::string& block,
                   int tokens);
  void release(std::uint64_t request, const std::string& block);
  void release_request(std::uint64_t request);
  // Re-homes a segment; returns (src_slot, dst_slot) pairs of the pages whose bytes must be
  // copied to the destination pool (private pages move, shared pages are duplicated).
  std::vector<std::pair<int, int>> move_segment(std::uint64_t request, const std::string& block,
                                                int dst_device);

  int device_of(std::uint64_t request, const std::string& block) const;
  int tokens(std::uint64_t request, const std::string& block) const;
  int pages(std::uint64_t request, const std::string& block) const;
  int shared_pages(std::uint64_t request, const std::string& block) const;
  std::int64_t segment_bytes(std::uint64_t request, const std::string& block) const;
  std::int64_t bytes_saved_by_sharing() const { return saved_by_sharing_; }
  std::int64_t used(int device) const;
  std::vector<std::uint64_t> page_ids(std::uint64_t request, const std::string& block) const;
  // Physical slots of the segment's pages, in token order (the GPU page-table row).
  std::vector<int> page_slots(std::uint64_t request, const std::string& block) const;

  // The GPU writes a token's K/V while the block runs, but the reference creates the page that
  // holds it later: prompt pages after the prefill step (scenario.cpp:671-695), decode pages at
  // chain end (append_decode_kv, scenario.cpp:697-719). To keep page ids bit-identical, physical
  // slots are reserved ahead of the bookkeeping and bound when the page id is created.
  // Returns the page-table row covering `total_pages` pages (existing, then reserved).
  // Frees the first n slots reserved for (request, block): pages a prefix share supplied
  // after the slots were reserved (their content was written, identical, into both).
  void drop_reserved_front(std::uint64_t request, const std::string& block, int n);
  std::vector<int> reserve_slots(std::uint64_t request, const std::string& block,
                                 const std::string& pool_key, int device, int total_pages);

 private:
  struct Page {
    std::int64_t bytes = 0;
    int ref = 0;
    int device = -1;
    std::string pool_key;
    int slot = -1;
  };
  struct Segment {
    int device = -1;
    std::int64_t bytes_per_page = 0;
    int tokens = 0;
    std::string pool_key;
    std::vector<std::uint64_t> page_ids;
  };
  Segment& seg(std::uint64_t request, const std::string& block);
  const Segment* find(std::uint64_t request, const std::string& block) const;
  void reserve(int device, std::int64_t bytes);
  void unreserve(int device, std::int64_t bytes);
  std::uint64_t new_page(std::uint64_t request, const std::string& block, const Segment& s, int device);
  void deref(std::uint64_t id);
  int alloc_slot(const std::string& pool_key, int device);
  void free_slot(const std::string& pool_key, int device, int slot);

  struct Reserved {
    std::string pool_key;
    int device = -1;
    std::vector<int> slots;
  };
  std::map<std::pair<std::uint64_t, std::string>, Reserved> reserved_;
  std::map<std::pair<std::uint64_t, std::string>, Segment> segments_;
  std::unordered_map<std::uint64_t, Page> pages_;  // looked up by id only (never iterated)
  std::map<std::pair<std::string, int>, SlotPool> pools_;
  std::map<int, std::int64_t> used_;
  std::map<int, std::int64_t> capacity_;
  std::uint64_t next_page_ = 1;
  std::int64_t saved_by_sharing_ = 0;
};

}  // namespace bh
