// C ABI of the host control plane pieces (include/blockhost.h: bh_pool_*, bh_kv_*).
#include <cstring>
#include <stdexcept>
#include <string>

#include "../../../include/blockhost.h"
#include "kv.hpp"
#include "pool.hpp"

struct bh_pool {
  bh::Pool p;
  std::string err;
};
struct bh_kv {
  bh::KvStore k;
  std::string err;
};

namespace {
template <class H, class F>
int guard(H* h, F&& f) {
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
int put_id(const std::string& id, char* out, int cap) {
  if (out == nullptr || cap <= static_cast<int>(id.size())) return BE_ERR_INVALID;
  std::memcpy(out, id.c_str(), id.size() + 1);
  return BE_OK;
}
bh::Entry to_entry(const bh_entry& e) {
  bh::Entry x;
  x.request_id = e.request_id;
  x.chain_step = e.chain_step;
  x.phase = e.phase == BE_PHASE_DECODE ? bh::Phase::kDecode : bh::Phase::kPrefill;
  x.tokens = e.tokens;
  x.context_tokens = e.context_tokens;
  x.kv_resident = e.kv_resident != 0;
  x.est_cost_us = e.est_cost_us;
  return x;
}
bh_entry from_entry(const bh::Entry& x) {
  bh_entry e;
  e.request_id = x.request_id;
  e.chain_step = x.chain_step;
  e.phase = x.phase == bh::Phase::kDecode ? BE_PHASE_DECODE : BE_PHASE_PREFILL;
  e.tokens = x.tokens;
  e.context_tokens = x.context_tokens;
  e.kv_resident = x.kv_resident ? 1 : 0;
  e.est_cost_us = x.est_cost_us;
  e.enqueue_seq = x.enqueue_seq;
  return e;
}
template <class V>
int put_entries(const V& v, bh_entry* out, int cap, int* n_out) {
  if (n_out) *n_out = static_cast<int>(v.size());
  if (static_cast<int>(v.size()) > cap) return BE_ERR_INVALID;
  int i = 0;
  for (const auto& x : v) out[i++] = from_entry(x);
  return BE_OK;
}
}  // namespace

extern "C" {

bh_pool* bh_pool_new(void) { return new bh_pool(); }
void bh_pool_free(bh_pool* p) { delete p; }
const char* bh_pool_last_error(const bh_pool* p) { return p ? p->err.c_str() : "null"; }

int bh_pool_create_instance(bh_pool* p, const char* block, int device, int64_t now,
                            int64_t ready_at, char* id_out, int cap) {
  if (!p || !block) return BE_ERR_INVALID;
  std::string id;
  const int rc = guard(p, [&] { id = p->p.create(block, device, now, ready_at).id; });
  return rc != BE_OK ? rc : put_id(id, id_out, cap);
}
int bh_pool_mark_ready(bh_pool* p, const char* inst, int64_t now) {
  if (!p || !inst) return BE_ERR_INVALID;
  return guard(p, [&] { p->p.mark_ready(inst, now); });
}
int bh_pool_enqueue(bh_pool* p, const char* inst, const bh_entry* e) {
  if (!p || !inst || !e) return BE_ERR_INVALID;
  return guard(p, [&] { p->p.enqueue(inst, to_entry(*e)); });
}
int bh_pool_pop_batch(bh_pool* p, const char* inst, int budget, int64_t now, bh_entry* out,
                      int cap, int* n_out, int* phase_out) {
  if (!p || !inst || !out) return BE_ERR_INVALID;
  bh::Batch b;
  const int rc = guard(p, [&] { b = p->p.pop_batch(inst, budget, now); });
  if (rc != BE_OK) return rc;
  if (phase_out) *phase_out = b.phase == bh::Phase::kDecode ? BE_PHASE_DECODE : BE_PHASE_PREFILL;
  return put_entries(b.members, out, cap, n_out);
}
int bh_pool_finish_batch(bh_pool* p, const char* inst, int64_t now) {
  if (!p || !inst) return BE_ERR_INVALID;
  return guard(p, [&] { p->p.finish_batch(inst, now); });
}
int bh_pool_next_runnable(bh_pool* p, int device, int64_t now, char* id_out, int cap) {
  if (!p) return -BE_ERR_INVALID;
  bh::Instance* in = p->p.next_runnable(device, now);
  if (in == nullptr) return 0;
  return put_id(in->id, id_out, cap) == BE_OK ? 1 : -BE_ERR_INVALID;
}
int bh_pool_remove_queued(bh_pool* p, const char* inst, int req, bh_entry* out, int cap, int* n) {
  if (!p || !inst) return BE_ERR_INVALID;
  std::vector<bh::Entry> v;
  const int rc = guard(p, [&] { v = p->p.remove_queued(inst, req); });
  return rc != BE_OK ? rc : put_entries(v, out, cap, n);
}
int bh_pool_take_tail(bh_pool* p, const char* inst, int count, bh_entry* out, int cap, int* n) {
  if (!p || !inst || count < 0) return BE_ERR_INVALID;
  std::vector<bh::Entry> v;
  const int rc = guard(p, [&] { v = p->p.take_tail(inst, static_cast<std::size_t>(count)); });
  return rc != BE_OK ? rc : put_entries(v, out, cap, n);
}
int bh_pool_queue(bh_pool* p, const char* inst, bh_entry* out, int cap, int* n, double* cost,
                  int* executing) {
  if (!p || !inst) return BE_ERR_INVALID;
  bh::Instance* in = p->p.find(inst);
  if (in == nullptr) {
    p->err = std::string("pool: unknown instance ") + inst;
    return BE_ERR_STATE;
  }
  if (cost) *cost = in->queued_cost_us;
  if (executing) *executing = in->executing ? 1 : 0;
  return put_entries(in->queue, out, cap, n);
}

bh_kv* bh_kv_new(void) { return new bh_kv(); }
void bh_kv_free(bh_kv* k) { delete k; }
const char* bh_kv_last_error(const bh_kv* k) { return k ? k->err.c_str() : "null"; }
int bh_kv_attach_pool(bh_kv* k, const char* key, int device, int n_pages) {
  if (!k || !key || n_pages < 0) return BE_ERR_INVALID;
  return guard(k, [&] { k->k.attach_pool(key, device, n_pages); });
}
int bh_kv_set_capacity(bh_kv* k, int device, int64_t bytes) {
  if (!k) return BE_ERR_INVALID;
  return guard(k, [&] { k->k.set_capacity(device, bytes); });
}
int bh_kv_create_segment(bh_kv* k, uint64_t req, const char* block, int device, int64_t bpt) {
  if (!k || !block) return BE_ERR_INVALID;
  return guard(k, [&] { k->k.create_segment(req, block, device, bpt); });
}
int bh_kv_append_tokens(bh_kv* k, uint64_t req, const char* block, int n, int* added) {
  if (!k || !block) return BE_ERR_INVALID;
  return guard(k, [&] {
    const int a = k->k.append_tokens(req, block, n);
    if (added) *added = a;
  });
}
int bh_kv_share_prefix(bh_kv* k, uint64_t req, uint64_t from, const char* block, int tokens,
                       int* covered) {
  if (!k || !block) return BE_ERR_INVALID;
  return guard(k, [&] {
    const int c = k->k.share_prefix(req, from, block, tokens);
    if (covered) *covered = c;
  });
}
int bh_kv_release(bh_kv* k, uint64_t req, const char* block) {
  if (!k || !block) return BE_ERR_INVALID;
  return guard(k, [&] { k->k.release(req, block); });
}
int bh_kv_release_request(bh_kv* k, uint64_t req) {
  if (!k) return BE_ERR_INVALID;
  return guard(k, [&] { k->k.release_request(req); });
}
int bh_kv_move_segment(bh_kv* k, uint64_t req, const char* block, int dst) {
  if (!k || !block) return BE_ERR_INVALID;
  return guard(k, [&] { k->k.move_segment(req, block, dst); });
}
int bh_kv_move_segment_slots(bh_kv* k, uint64_t req, const char* block, int dst,
                             int32_t* src_slots, int32_t* dst_slots, int cap, int* n_out) {
  if (!k || !block || !n_out || (cap > 0 && (!src_slots || !dst_slots))) return BE_ERR_INVALID;
  return guard(k, [&] {
    const auto copies = k->k.move_segment(req, block, dst);
    if ((int)copies.size() > cap) throw std::invalid_argument("move_segment: slot buffer too small");
    for (size_t i = 0; i < copies.size(); ++i) {
      src_slots[i] = copies[i].first;
      dst_slots[i] = copies[i].second;
    }
    *n_out = static_cast<int>(copies.size());
  });
}
int64_t bh_kv_query(const bh_kv* k, uint64_t req, const char* block, int what) {
  if (!k || !block) return -1;
  switch (what) {
    case 0: return k->k.device_of(req, block);
    case 1: return k->k.tokens(req, block);
    case 2: return k->k.pages(req, block);
    case 3: return k->k.shared_pages(req, block);
    case 4: return k->k.segment_bytes(req, block);
    case 5: return k->k.has_segment(req, block) ? 1 : 0;
    default: return -1;
  }
}
int64_t bh_kv_bytes_saved(const bh_kv* k) { return k ? k->k.bytes_saved_by_sharing() : 0; }
int64_t bh_kv_used(const bh_kv* k, int device) { return k ? k->k.used(device) : 0; }
int bh_kv_page_ids(const bh_kv* k, uint64_t req, const char* block, uint64_t* out, int cap, int* n) {
  if (!k || !block) return BE_ERR_INVALID;
  const auto v = k->k.page_ids(req, block);
  if (n) *n = static_cast<int>(v.size());
  if (static_cast<int>(v.size()) > cap) return BE_ERR_INVALID;
  for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
  return BE_OK;
}
int bh_kv_page_slots(const bh_kv* k, uint64_t req, const char* block, int32_t* out, int cap, int* n) {
  if (!k || !block) return BE_ERR_INVALID;
  const auto v = k->k.page_slots(req, block);
  if (n) *n = static_cast<int>(v.size());
  if (static_cast<int>(v.size()) > cap) return BE_ERR_INVALID;
  for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
  return BE_OK;
}

}  // extern "C"
