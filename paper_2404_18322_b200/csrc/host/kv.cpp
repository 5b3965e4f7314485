// Paged KV bookkeeping + physical page-slot binding; see kv.hpp for the reference mapping.
#include "kv.hpp"

#include <algorithm>

namespace bh {

namespace {
int pages_for(int tokens) { return (tokens + kPageTokens - 1) / kPageTokens; }
}  // namespace

void KvStore::attach_pool(const std::string& pool_key, int device, int n_pages) {
  pools_[{pool_key, device}] = SlotPool(n_pages);
}

void KvStore::reserve(int device, std::int64_t bytes) {
  auto cap = capacity_.find(device);
  if (cap != capacity_.end() && used_[device] + bytes > cap->second)
    throw LedgerError("device " + std::to_string(device) + " kv over capacity");
  used_[device] += bytes;
}

void KvStore::unreserve(int device, std::int64_t bytes) {
  auto& u = used_[device];
  if (u < bytes) throw LedgerError("release below zero");
  u -= bytes;
}

int KvStore::alloc_slot(const std::string& pool_key, int device) {
  auto it = pools_.find({pool_key, device});
  if (it == pools_.end()) return -1;  // pure bookkeeping (no GPU pool attached)
  const int s = it->second.alloc();
  if (s < 0) throw LedgerError("kv pool " + pool_key + "@" + std::to_string(device) + " full");
  return s;
}

void KvStore::free_slot(const std::string& pool_key, int device, int slot) {
  if (slot < 0) return;
  auto it = pools_.find({pool_key, device});
  if (it != pools_.end()) it->second.release(slot);
}

std::uint64_t KvStore::new_page(std::uint64_t request, const std::string& block,
                                const Segment& s, int device) {
  reserve(device, s.bytes_per_page);
  const std::uint64_t id = next_page_++;
  Page p;
  p.bytes = s.bytes_per_page;
  p.ref = 1;
  p.device = device;
  p.pool_key = s.pool_key;
  auto rit = reserved_.find({request, block});
  if (rit != reserved_.end() && !rit->second.slots.empty() && rit->second.device == device &&
      rit->second.pool_key == s.pool_key) {
    p.slot = rit->second.slots.front();
    rit->second.slots.erase(rit->second.slots.begin());
    if (rit->second.slots.empty()) reserved_.erase(rit);
  } else {
    try {
      p.slot = alloc_slot(s.pool_key, device);
    } catch (...) {
      unreserve(device, s.bytes_per_page);
      --next_page_;
      throw;
    }
  }
  pages_[id] = p;
  return id;
}

void KvStore::drop_reserved_front(std::uint64_t request, const std::string& block, int n) {
  auto rit = reserved_.find({request, block});
  if (rit == reserved_.end() || n <= 0) return;
  auto& v = rit->second.slots;
  const int k = std::min<int>(n, static_cast<int>(v.size()));
  for (int i = 0; i < k; ++i) free_slot(rit->second.pool_key, rit->second.device, v[i]);
  v.erase(v.begin(), v.begin() + k);
  if (v.empty()) reserved_.erase(rit);
}

std::vector<int> KvStore::reserve_slots(std::uint64_t request, const std::string& block,
                                        const std::string& pool_key, int device,
                                        int total_pages) {
  std::vector<int> row = page_slots(request, block);
  auto rit = reserved_.find({request, block});
  if (rit == reserved_.end() && static_cast<int>(row.size()) >= total_pages)
    return row;  // nothing reserved and nothing to reserve (the common decode step)
  auto& r = rit != reserved_.end() ? rit->second : reserved_[{request, block}];
  if (r.slots.empty()) {
    r.pool_key = pool_key;
    r.device = device;
  } else if (r.pool_key != pool_key || r.device != device) {
    throw KvError("slot reservation moved between pools");
  }
  while (static_cast<int>(row.size() + r.slots.size()) < total_pages)
    r.slots.push_back(alloc_slot(pool_key, device));
  row.insert(row.end(), r.slots.begin(), r.slots.end());
  if (r.slots.empty()) reserved_.erase({request, block});
  return row;
}

void KvStore::create_segment(std::uint64_t request, const std::string& block, int device,
                             std::int64_t bytes_per_token, const std::string& pool_key) {
  if (bytes_per_token <= 0) throw KvError("bytes_per_token must be positive");
  if (find(request, block)) throw KvError("segment already exists");
  Segment s;
  s.device = device;
  s.bytes_per_page = bytes_per_token * kPageTokens;
  s.pool_key = pool_key.empty() ? block : pool_key;
  segments_.emplace(std::make_pair(request, block), std::move(s));
}

bool KvStore::has_segment(std::uint64_t request, const std::string& block) const {
  return find(request, block) != nullptr;
}

int KvStore::append_tokens(std::uint64_t request, const std::string& block, int n) {
  if (n < 0) throw KvError("negative token append");
  Segment& s = seg(request, block);
  s.tokens += n;
  const int need = pages_for(s.tokens);
  int added = 0;
  while (static_cast<int>(s.page_ids.size()) < need) {
    s.page_ids.push_back(new_page(request, block, s, s.device));
    ++added;
  }
  return added;
}

bool KvStore::append_if_present(std::uint64_t request, const std::string& block, int n) {
  if (n < 0) throw KvError("negative token append");
  auto it = segments_.find({request, block});
  if (it == segments_.end()) return false;
  Segment& s = it->second;
  s.tokens += n;
  const int need = pages_for(s.tokens);
  while (static_cast<int>(s.page_ids.size()) < need)
    s.page_ids.push_back(new_page(request, block, s, s.device));
  return true;
}

int KvStore::share_prefix(std::uint64_t request, std::uint64_t from, const std::string& block,
                          int tokens) {
  Segment& dst = seg(request, block);
  Segment& src = seg(from, block);
  if (!dst.page_ids.empty() || dst.tokens != 0) throw KvError("share_prefix into non-empty segment");
  if (dst.device != src.device) throw KvError("share_prefix across devices");
  if (dst.bytes_per_page != src.bytes_per_page) throw KvError("share_prefix page size mismatch");
  // only whole pages are shareable
  const int full = std::min(tokens, src.tokens) / kPageTokens;
  const int usable = std::min(full, static_cast<int>(src.page_ids.size()));
  for (int i = 0; i < usable; ++i) {
    Page& p = pages_.at(src.page_ids[static_cast<std::size_t>(i)]);
    ++p.ref;
    dst.page_ids.push_back(src.page_ids[static_cast<std::size_t>(i)]);
    saved_by_sharing_ += p.bytes;
  }
  dst.tokens = usable * kPageTokens;
  return dst.tokens;
}

void KvStore::deref(std::uint64_t id) {
  Page& p = pages_.at(id);
  if (--p.ref == 0) {
    unreserve(p.device, p.bytes);
    free_slot(p.pool_key, p.device, p.slot);
    pages_.erase(id);
  }
}

void KvStore::release(std::uint64_t request, const std::string& block) {
  auto rit = reserved_.find({request, block});
  if (rit != reserved_.end()) {
    for (int s : rit->second.slots) free_slot(rit->second.pool_key, rit->second.device, s);
    reserved_.erase(rit);
  }
  auto it = segments_.find({request, block});
  if (it == segments_.end()) return;
  for (std::uint64_t id : it->second.page_ids) deref(id);
  segments_.erase(it);
}

void KvStore::release_request(std::uint64_t request) {
  for (auto rit = reserved_.lower_bound({request, std::string()});
       rit != reserved_.end() && rit->first.first == request;) {
    for (int s : rit->second.slots) free_slot(rit->second.pool_key, rit->second.device, s);
    rit = reserved_.erase(rit);
  }
  auto it = segments_.lower_bound({request, std::string()});
  while (it != segments_.end() && it->first.first == request) {
    for (std::uint64_t id : it->second.page_ids) deref(id);
    it = segments_.erase(it);
  }
}

std::vector<std::pair<int, int>> KvStore::move_segment(std::uint64_t request,
                                                       const std::string& block, int dst) {
  Segment& s = seg(request, block);
  std::vector<std::pair<int, int>> copies;
  if (s.device == dst) return copies;
  for (auto& id : s.page_ids) {
    Page& p = pages_.at(id);
    if (p.ref == 1) {
      // private page: its bytes move to the destination pool (slot first: a full pool throws
      // before the ledger has changed; a ledger failure hands the slot back)
      const int nslot = alloc_slot(p.pool_key, dst);
      try {
        reserve(dst, p.bytes);
      } catch (...) {
        free_slot(p.pool_key, dst, nslot);
        throw;
      }
      unreserve(p.device, p.bytes);
      copies.emplace_back(p.slot, nslot);
      free_slot(p.pool_key, p.device, p.slot);
      p.slot = nslot;
      p.device = dst;
    } else {
      // shared page stays for its other readers; this segment gets a fresh private copy
      const int nslot = alloc_slot(p.pool_key, dst);
      try {
        reserve(dst, p.bytes);
      } catch (...) {
        free_slot(p.pool_key, dst, nslot);
        throw;
      }
      --p.ref;
      const std::uint64_t cid = next_page_++;
      Page c;
      c.bytes = p.bytes;
      c.ref = 1;
      c.device = dst;
      c.pool_key = p.pool_key;
      c.slot = nslot;
      copies.emplace_back(p.slot, c.slot);
      pages_[cid] = c;
      id = cid;
    }
  }
  s.device = dst;
  return copies;
}

int KvStore::device_of(std::uint64_t request, const std::string& block) const {
  const Segment* s = find(request, block);
  return s ? s->device : -1;
}
int KvStore::tokens(std::uint64_t request, const std::string& block) const {
  const Segment* s = find(request, block);
  return s ? s->tokens : 0;
}
int KvStore::pages(std::uint64_t request, const std::string& block) const {
  const Segment* s = find(request, block);
  return s ? static_cast<int>(s->page_ids.size()) : 0;
}
int KvStore::shared_pages(std::uint64_t request, const std::string& block) const {
  const Segment* s = find(request, block);
  if (!s) return 0;
  int n = 0;
  for (std::uint64_t id : s->page_ids)
    if (pages_.at(id).ref > 1) ++n;
  return n;
}
std::int64_t KvStore::segment_bytes(std::uint64_t request, const std::string& block) const {
  const Segment* s = find(request, block);
  return s ? static_cast<std::int64_t>(s->page_ids.size()) * s->bytes_per_page : 0;
}
std::int64_t KvStore::used(int device) const {
  auto it = used_.find(device);
  return it == used_.end() ? 0 : it->second;
}
std::vector<std::uint64_t> KvStore::page_ids(std::uint64_t request, const std::string& block) const {
  const Segment* s = find(request, block);
  return s ? s->page_ids : std::vector<std::uint64_t>{};
}
std::vector<int> KvStore::page_slots(std::uint64_t request, const std::string& block) const {
  std::vector<int> out;
  const Segment* s = find(request, block);
  if (!s) return out;
  out.reserve(s->page_ids.size());
  for (std::uint64_t id : s->page_ids) out.push_back(pages_.at(id).slot);
  return out;
}

KvStore::Segment& KvStore::seg(std::uint64_t request, const std::string& block) {
  auto it = segments_.find({request, block});
  if (it == segments_.end())
    throw KvError("unknown segment: request " + std::to_string(request) + " block " + block);
  return it->second;
}
const KvStore::Segment* KvStore::find(std::uint64_t request, const std::string& block) const {
  auto it = segments_.find({request, block});
  return it == segments_.end() ? nullptr : &it->second;
}

}  // namespace bh
