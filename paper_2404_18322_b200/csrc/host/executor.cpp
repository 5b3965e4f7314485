// bh_executor: the drop-in for Simulation::batch_duration_us (proj/core/src/scenario.cpp:493).
//
// A host that already forms batches - the reference Simulation itself - hands each batch it pops
// to bh_executor_run_batch instead of (or beside) pricing it: the batch's block runs on the
// B200 over the members' activation rows and block-local paged KV, exactly as the bh_runner
// loop runs it (Runner::plan / execute_direct, runner.cpp), but with the caller deciding what
// runs when. The executor owns the device side the reference does not have: block weights
// (loaded on first use from the block id and its component kinds), one KV pool per block with
// page slots bound per (request, block) segment (the KvStore mirror, kv.cpp), the prompt rows
// of every request and one decode row per request.
//
// Data flow follows the chain: a prefill batch updates its members' prompt rows in place; at a
// request's chain-final step the last prompt row becomes its decode row (the first token,
// advance_from, scenario.cpp:635-647); decode batches update decode rows in place.
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/blockhost.h"
#include "kv.hpp"

namespace {
int pages_for(int tokens) { return (tokens + bh::kPageTokens - 1) / bh::kPageTokens; }

struct ExecError : std::runtime_error {
  int code;
  ExecError(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};
void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw ExecError(BE_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace

struct bh_executor {
  be_ctx* ctx = nullptr;
  cudaStream_t st = nullptr;
  bh_executor_desc desc{};
  std::vector<int> prompt, output, poff;
  struct Blk {
    std::string comps;
    be_block* blk = nullptr;
    be_kv_pool* pool = nullptr;
    bool attn = false;
  };
  std::map<std::string, Blk> blocks;
  bh::KvStore kv;
  be_workspace* ws = nullptr;
  void* prefill_rows = nullptr;  // [sum prompts][d]
  void* decode_rows = nullptr;   // [n_requests][d]
  int64_t batches = 0, tokens = 0;
  std::string err;

  ~bh_executor() {
    if (st) cudaStreamSynchronize(st);
    if (ws) be_workspace_free(ws);
    for (auto& [id, b] : blocks) {
      if (b.pool) be_kv_pool_free(b.pool);
      if (b.blk) be_block_free(b.blk);
    }
    if (prefill_rows) cudaFree(prefill_rows);
    if (decode_rows) cudaFree(decode_rows);
  }

  Blk& block(const std::string& id, const char* comps) {
    auto it = blocks.find(id);
    if (it != blocks.end()) return it->second;
    if (comps == nullptr || *comps == 0)
      throw ExecError(BE_ERR_INVALID, "block " + id + ": first use needs its component kinds");
    Blk b;
    b.comps = comps;
    b.attn = b.comps.find('a') != std::string::npos;
    be_block_desc d{};
    d.n_layers = (int)b.comps.size();
    d.d_model = desc.d_model;
    d.n_heads = desc.n_heads;
    d.head_dim = desc.d_model / desc.n_heads;
    d.d_ff = desc.d_ff;
    d.max_pos = desc.max_pos;
    d.norm_eps = 1e-5f;
    d.rope_theta = 10000.f;
    d.init_scale = desc.init_scale;
    d.seed = desc.seed;
    d.name = id.c_str();
    d.components = b.comps.c_str();
    int rc = be_block_load(ctx, &d, &b.blk);
    if (rc != BE_OK) throw ExecError(rc, std::string("block load: ") + be_last_error(ctx));
    // every request may hold a full-length segment in every block
    int pages = 1;
    for (size_t r = 0; r < prompt.size(); ++r) pages += pages_for(prompt[r] + output[r]) + 1;
    rc = be_kv_pool_create(ctx, b.blk, pages, &b.pool);
    if (rc != BE_OK) throw ExecError(rc, std::string("kv pool: ") + be_last_error(ctx));
    kv.attach_pool(id, 0, pages);
    return blocks.emplace(id, std::move(b)).first->second;
  }

  void run(const char* block_id, const char* comps, int phase, int n, const bh_member* m) {
    Blk& b = block(block_id, comps);
    const std::string bn = block_id;
    const int stride = pages_for(desc.max_pos) + 1;
    std::vector<int32_t> pt((size_t)n * stride, -1);
    std::vector<be_token> toks;
    for (int i = 0; i < n; ++i) {
      const int r = m[i].request_id - 1;
      if (r < 0 || r >= (int)prompt.size()) throw ExecError(BE_ERR_INVALID, "unknown request");
      const bool pre = phase == BE_PHASE_PREFILL;
      const int first = pre ? 0 : m[i].context_tokens - 1;  // the decode token's position
      const int count = pre ? prompt[r] : 1;
      if (first + count > desc.max_pos) throw ExecError(BE_ERR_INVALID, "context beyond max_pos");
      std::vector<int> row;
      if (b.attn) {
        if (!pre && kv.tokens(r + 1, bn) != first)
          throw ExecError(BE_ERR_STATE, "kv segment of request " + std::to_string(r + 1) +
                                            " at block " + bn + " out of step with its context");
        row = kv.reserve_slots(r + 1, bn, bn, 0, pages_for(first + count));
        std::copy(row.begin(), row.end(), pt.begin() + (size_t)i * stride);
      } else {
        row.assign(pages_for(first + count), 0);  // no attention: no KV page is touched
        for (size_t p = 0; p < row.size(); ++p) pt[(size_t)i * stride + p] = 0;
      }
      for (int t = 0; t < count; ++t) {
        const int pos = first + t;
        be_token k;
        k.src_row = pre ? poff[r] + t : r;
        k.dst_row = k.src_row;
        k.kv_slot = row[pos / bh::kPageTokens] * bh::kPageTokens + pos % bh::kPageTokens;
        k.pos = pos;
        k.pt_row = i;
        toks.push_back(k);
      }
    }
    void* arena = phase == BE_PHASE_PREFILL ? prefill_rows : decode_rows;
    int rc = be_exec_batch(ctx, b.blk, b.pool, ws, phase, (int)toks.size(), toks.data(), n, stride,
                           pt.data(), arena, arena, st);
    if (rc != BE_OK) throw ExecError(rc, std::string("exec: ") + be_last_error(ctx));
    // host metadata was staged from pageable memory: keep the host in step with the device
    ck(cudaStreamSynchronize(st), "batch");
    ++batches;
    tokens += (int64_t)toks.size();
    // KV bookkeeping and the chain's data flow
    for (int i = 0; i < n; ++i) {
      const int r = m[i].request_id - 1;
      if (phase == BE_PHASE_PREFILL) {
        if (b.attn && !kv.has_segment(r + 1, bn)) {
          kv.create_segment(r + 1, bn, 0, 1);
          kv.append_tokens(r + 1, bn, prompt[r]);
        }
        if (m[i].chain_final)
          ck(cudaMemcpyAsync(static_cast<char*>(decode_rows) + (size_t)r * desc.d_model * 2,
                             static_cast<char*>(prefill_rows) +
                                 (size_t)(poff[r] + prompt[r] - 1) * desc.d_model * 2,
                             (size_t)desc.d_model * 2, cudaMemcpyDeviceToDevice, st),
             "first token row");
      } else if (b.attn) {
        kv.append_tokens(r + 1, bn, 1);
      }
    }
  }
};

namespace {
template <class F>
int guard(bh_executor* x, F&& f) {
  try {
    f();
    return BE_OK;
  } catch (const ExecError& e) {
    if (x) x->err = e.what();
    return e.code;
  } catch (const std::invalid_argument& e) {
    if (x) x->err = e.what();
    return BE_ERR_INVALID;
  } catch (const std::logic_error& e) {
    if (x) x->err = e.what();
    return BE_ERR_STATE;
  } catch (const std::exception& e) {
    if (x) x->err = e.what();
    return BE_ERR_RUNTIME;
  }
}
}  // namespace

extern "C" int bh_executor_create(be_ctx* ctx, const bh_executor_desc* d, int n_requests,
                                  const int32_t* req_prompt, const int32_t* req_output,
                                  bh_executor** out) {
  if (ctx == nullptr || d == nullptr || out == nullptr || n_requests <= 0 ||
      req_prompt == nullptr || req_output == nullptr || d->d_model <= 0 || d->n_heads <= 0 ||
      d->d_model % d->n_heads != 0 || d->max_pos <= 0)
    return BE_ERR_INVALID;
  *out = nullptr;
  auto* x = new bh_executor();
  const int rc = guard(x, [&] {
    x->ctx = ctx;
    x->st = static_cast<cudaStream_t>(be_ctx_stream(ctx));
    x->desc = *d;
    int total = 0, max_prompt = 0;
    for (int r = 0; r < n_requests; ++r) {
      if (req_prompt[r] <= 0 || req_output[r] <= 0) throw ExecError(BE_ERR_INVALID, "bad request");
      x->prompt.push_back(req_prompt[r]);
      x->output.push_back(req_output[r]);
      x->poff.push_back(total);
      total += req_prompt[r];
      max_prompt = std::max(max_prompt, req_prompt[r]);
    }
    const int max_tok = std::max({std::min(total, std::max(d->max_batch_tokens, max_prompt)),
                                  n_requests, 1});
    int e = be_workspace_create(ctx, d->d_model, d->d_ff, d->n_heads, max_tok, n_requests,
                                pages_for(d->max_pos) + 1, &x->ws);
    if (e != BE_OK) throw ExecError(e, std::string("workspace: ") + be_last_error(ctx));
    ck(cudaMalloc(&x->prefill_rows, (size_t)total * d->d_model * 2), "prompt rows");
    ck(cudaMalloc(&x->decode_rows, (size_t)n_requests * d->d_model * 2), "decode rows");
    ck(cudaMemsetAsync(x->decode_rows, 0, (size_t)n_requests * d->d_model * 2, x->st), "rows");
    // the requests' synthetic prompt embeddings (the runner's stream "inputs:req<id>")
    for (int r = 0; r < n_requests; ++r) {
      const std::string sid = "inputs:req" + std::to_string(r + 1);
      e = be_synth_rows(ctx, static_cast<char*>(x->prefill_rows) + (size_t)x->poff[r] * d->d_model * 2,
                        (int64_t)x->prompt[r] * d->d_model, d->seed, sid.c_str(), 1.7320508f, x->st);
      if (e != BE_OK) throw ExecError(e, "synthetic prompts");
    }
    ck(cudaStreamSynchronize(x->st), "init");
  });
  if (rc != BE_OK) {
    delete x;
    return rc;
  }
  *out = x;
  return BE_OK;
}

extern "C" int bh_executor_free(bh_executor* x) {
  if (x == nullptr) return BE_ERR_INVALID;
  delete x;
  return BE_OK;
}

extern "C" const char* bh_executor_last_error(const bh_executor* x) {
  return x == nullptr ? "null executor" : x->err.c_str();
}

extern "C" int bh_executor_run_batch(bh_executor* x, const char* block_id, const char* components,
                                     int phase, int n_members, const bh_member* members) {
  if (x == nullptr || block_id == nullptr || n_members <= 0 || members == nullptr ||
      (phase != BE_PHASE_PREFILL && phase != BE_PHASE_DECODE))
    return BE_ERR_INVALID;
  return guard(x, [&] { x->run(block_id, components, phase, n_members, members); });
}

extern "C" int bh_executor_read_rows(bh_executor* x, int decode, void* host_out) {
  if (x == nullptr || host_out == nullptr) return BE_ERR_INVALID;
  return guard(x, [&] {
    const size_t rows = decode ? x->prompt.size() : (size_t)(x->poff.back() + x->prompt.back());
    ck(cudaMemcpyAsync(host_out, decode ? x->decode_rows : x->prefill_rows,
                       rows * x->desc.d_model * 2, cudaMemcpyDeviceToHost, x->st), "read rows");
    ck(cudaStreamSynchronize(x->st), "read rows");
  });
}

extern "C" int bh_executor_stats(const bh_executor* x, int64_t* batches, int64_t* tokens) {
  if (x == nullptr) return BE_ERR_INVALID;
  if (batches) *batches = x->batches;
  if (tokens) *tokens = x->tokens;
  return BE_OK;
}
