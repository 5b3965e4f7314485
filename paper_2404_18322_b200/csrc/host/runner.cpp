// The executor loop on one device: requests walk their block chains; at every block instance
// queued (request, step) rows are gathered into a batch (Pool::pop_batch), the batch runs on the
// GPU (be_exec_batch: gather -> decoder layers -> scatter), and each member advances to its next
// chain step, its first decode token, or its next token.
//
// Reference mapping (proj/core/src/scenario.cpp): on_arrival :194-208, dispatch_step :210-242
// (instances created lazily at first use, ids "i<N>"), enqueue_step :310-334 (decode entries
// whose cache sits on the instance's device are kv-resident), pump :465-557 (one lane per
// device: next_runnable -> pop_batch -> run), on_batch_finish :559-578 (members advance with
// pumps deferred until all advanced), advance_after_step / advance_from :595-669,
// create_kv_for_step :671-695 (prompt pages after the prefill step), append_decode_kv :697-719
// (one token on every chain segment at chain end). The cost-table duration of pump is replaced by
// the real block run; speculation, scale-out, migration and reviews are outside this loop.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/blockhost.h"
#include "kv.hpp"
#include "pool.hpp"

namespace bh {

namespace {
int pages_for(int tokens) { return (tokens + kPageTokens - 1) / kPageTokens; }

struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};
void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
struct BeError : std::runtime_error {
  int code;
  BeError(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};
}  // namespace

struct Request {
  int idx = 0;       // 0-based
  int id = 0;        // reference request id (1-based, workload.cpp:89-96)
  int tenant = 0;
  int prompt = 0;
  int output = 0;
  int step = 0;
  Phase phase = Phase::kPrefill;
  int generated = 0;
  int ctx = 0;       // context tokens (QueueEntry::context_tokens)
  bool done = false;
  int poff = 0;      // first row of its prompt in the prefill arena
  int prefix_group = -1;
  int prefix_tokens = 0;
};

struct PlannedBatch {
  int inst = 0;
  int block = 0;
  Phase phase = Phase::kDecode;
  std::vector<be_token> toks;
  std::vector<int32_t> pt;  // [n_rows][stride]
  int n_rows = 0;
  int stride = 1;
  std::vector<int> shared_pages;  // prefill: per member, prefix pages taken from a donor
};

class Runner {
 public:
  Runner(be_ctx* ctx, const bh_workload& w);
  ~Runner();
  Runner(const Runner&) = delete;
  Runner& operator=(const Runner&) = delete;
  void run(int max_batches);
  // group -1 / members null: every live request; else one micro-batch (own CUDA graph)
  void decode_step(const void* host_in, void* host_out, int* n_batches, int group = -1,
                   const std::vector<int>* members = nullptr);
  void serve(const std::int64_t* arrival_us, std::int64_t* first_us, std::int64_t* done_us);
  // KV migration: requests taken over mid-decode (their KV pages are copied in by the caller)
  void adopt(int n, const int32_t* idx, const int32_t* ctx, const int32_t* generated);
  void request_state(int idx, int32_t* ctx, int32_t* generated, int32_t* done) const;
  std::vector<int> kv_segment(int idx, int block, int* tokens) const;
  be_kv_pool* kv_pool(int block) const { return pools_[block]; }
  int n_blocks() const { return static_cast<int>(names_.size()); }
  int live() const;
  std::int64_t generated() const { return tokens_generated_; }
  void* arena() { return arena_; }
  std::int64_t kv_used() const { return kv_.used(0); }
  std::int64_t kv_saved() const { return kv_.bytes_saved_by_sharing(); }
  int requests() const { return static_cast<int>(reqs_.size()); }
  void* prefill_arena() { return parena_; }
  std::int64_t prefill_rows() const { return prefill_rows_; }

  std::vector<bh_batch_rec> recs;
  std::vector<int32_t> m_req, m_step, m_ctx;
  bh_step_stats stats{};
  const bh_spec_stats& spec_stats() const { return spec_stats_; }

 private:
  // --- executor loop pieces (scenario.cpp)
  void dispatch(Request& r);
  void pump();
  void finish_running();
  void advance_after_step(Request& r, int step, int planned_shared = 0);
  void advance_from(Request& r, int step);
  std::string instance_for(int block);
  PlannedBatch plan(const std::string& inst_id, const Batch& b);
  void launch(const PlannedBatch& pb, const be_token* d_tok, const int32_t* d_pt);
  void execute_direct(const PlannedBatch& pb);
  void record(const PlannedBatch& pb, const Batch& b);
  void account(const PlannedBatch& pb);
  int chain_len(const Request& r) const { return chain_ptr_[r.tenant + 1] - chain_ptr_[r.tenant]; }
  int chain_block(const Request& r, int step) const { return chain_blocks_[chain_ptr_[r.tenant] + step]; }

  be_ctx* ctx_;
  cudaStream_t st_ = nullptr;
  bool dry_ = false;  // control plane only
  std::vector<std::string> comps_;
  std::vector<std::int64_t> kv_bpt_;  // per block
  int n_created_ = 0;
  int mode_ = 0;
  bool use_graphs_ = false;
  bool group_ = true;  // decode: run independent same-shape batches as one grouped launch
  int max_batch_tokens_ = 4096;
  int d_ = 0;
  int max_ctx_ = 0;
  std::vector<be_block_desc> descs_;
  std::vector<std::string> names_;
  std::vector<be_block*> blocks_;
  // LoRA variants: base block index (-1: own weights), adapters, which blocks_ entries we own
  std::vector<int> lora_base_;
  std::vector<be_lora*> loras_;
  std::vector<char> own_block_;
  void init(const bh_workload& w);  // the constructor's body
  void release();                    // frees every device / host resource held so far
  int32_t* d_zero_idx_ = nullptr;  // adapter index 0 for every row of a single-variant launch
  int wbase(int b) const { return lora_base_[b] >= 0 ? lora_base_[b] : b; }
  // a LoRA launch adds two shrink kernels per attention component
  int lora_launches(int b) const {
    return lora_base_[b] >= 0 ? 2 * (int)(kv_bpt_[b] / (4LL * d_)) : 0;  // n_att from KV bytes
  }
  std::vector<be_kv_pool*> pools_;
  // speculation: surrogate block and its KV pool per marked block, the verify lane's workspace,
  // [n_requests][d] scratch rows (draft, true, next) and the next block's row indices
  std::vector<char> spec_;
  std::vector<be_block*> sur_;
  std::vector<be_kv_pool*> sur_pool_;
  be_workspace* ws_verify_ = nullptr;
  void* spec_buf_ = nullptr;
  int32_t* spec_dst_ = nullptr;
  float spec_thr_ = 0.95f;
  bh_spec_stats spec_stats_{0, 0, 0, 0.0, 1.0};
  std::vector<int> chain_ptr_, chain_blocks_;
  std::vector<Request> reqs_;
  std::vector<std::string> inst_of_block_;
  std::vector<int> inst_index_;  // block -> instance creation index
  Pool pool_;
  KvStore kv_;
  std::map<std::pair<int, int>, int> prefix_donors_;  // (prefix group, block) -> request id
  bool prefix_share_ = true;
  int prefix_donor(const Request& r, int block, int* want) const;
  be_workspace* ws_ = nullptr;
  void* arena_ = nullptr;   // decode rows [n_req][d]
  void* parena_ = nullptr;  // prefill rows [sum prompt][d]
  std::int64_t prefill_rows_ = 0;
  bool has_running_ = false;
  std::string running_inst_;
  Batch running_;
  PlannedBatch running_plan_;
  std::vector<int> step_done_order_;  // lockstep: completion order of the last step
  // live serving: requests whose first token / last token the bookkeeping just produced
  bool serving_ = false;
  std::vector<int> just_first_, just_done_;
  bool in_lockstep_step_ = false;
  std::int64_t tokens_generated_ = 0;
  int batches_run_ = 0;
  // graph replay of a steady-state lockstep decode step, one per request group
  // one launch of a decode step: a batch, or several independent same-shape batches grouped
  struct LaunchEntry {
    std::vector<int> plans;
    std::vector<be_token> toks;  // grouped: concatenated, page-table rows renumbered
    std::vector<int32_t> pt;
    int stride = 1;
    bool lora = false;           // LoRA variants of one base: one weight stream, per-row adapters
    std::vector<int32_t> lidx;   // lora: adapter slot per token (group index, -1 = the base)
  };
  std::vector<LaunchEntry> group_plans(const std::vector<PlannedBatch>& plans) const;
  bool spec_pair(const std::vector<PlannedBatch>& plans, const LaunchEntry& a,
                 const LaunchEntry& b) const;
  void run_speculative(const PlannedBatch& pv, const PlannedBatch& pn);
  // one planned decode step: host bookkeeping done, metadata laid out, nothing on the device yet
  struct StepPlan {
    bool valid = false;
    int group = -1;
    std::vector<int> rows;  // live requests of the step, request order (host row order)
    std::vector<PlannedBatch> plans;
    std::vector<LaunchEntry> entries;
    std::vector<size_t> off_tok, off_pt, off_idx;
    size_t total = 0;
    std::vector<std::tuple<int, int, int>> sig;
    bh_step_stats stats{};
  };
  StepPlan plan_step(int group, const std::vector<int>* members);
  void stage_and_launch(StepPlan& sp, const void* host_in);
  bool plan_ahead_ = false;  // plan step k+1 while step k runs (decode_step without a group)
  StepPlan pending_;
  void copy_host_rows(const std::vector<int>& rows, bool to_dev, void* host);
  void launch_entry(const std::vector<PlannedBatch>& plans, const LaunchEntry& le,
                    const be_token* d_tok, const int32_t* d_pt, const int32_t* d_idx);
  struct GraphSlot {
    std::vector<std::tuple<int, int, int>> sig;  // (block, n_tokens, stride*16+n) per launch
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t graph = nullptr;
    void reset() {
      if (exec) cudaGraphExecDestroy(exec);
      if (graph) cudaGraphDestroy(graph);
      exec = nullptr;
      graph = nullptr;
    }
  };
  std::map<int, GraphSlot> graphs_;
  // pinned staging ring: the host plans step s+1 while step s still runs; slot k is rewritten
  // only after its previous upload (two steps back) has executed
  char* meta_host_[2] = {nullptr, nullptr};
  cudaEvent_t meta_ev_[2] = {nullptr, nullptr};
  int meta_slot_ = 0;
  char* meta_dev_ = nullptr;
  size_t meta_cap_ = 0;
};

// A construction that fails part-way (e.g. out of device memory for the next pool) frees what
// it allocated before rethrowing: the destructor does not run for a throwing constructor.
Runner::Runner(be_ctx* ctx, const bh_workload& w) : ctx_(ctx) {
  try {
    init(w);
  } catch (...) {
    release();
    throw;
  }
}

void Runner::init(const bh_workload& w) {
  be_ctx* ctx = ctx_;
  if (w.n_blocks <= 0 || w.n_tenants <= 0 || w.n_requests <= 0 || !w.blocks || !w.chain_ptr ||
      !w.chain_blocks || !w.req_tenant || !w.req_prompt || !w.req_output)
    throw BeError(BE_ERR_INVALID, "runner: incomplete workload");
  dry_ = w.dry_run != 0;
  if (!dry_ && ctx == nullptr) throw BeError(BE_ERR_INVALID, "runner: no device context");
  st_ = dry_ ? nullptr : static_cast<cudaStream_t>(be_ctx_stream(ctx));
  mode_ = w.mode;
  use_graphs_ = w.use_graphs != 0;
  plan_ahead_ = w.plan_ahead != 0;
  if (const char* g = std::getenv("BH_GROUP")) group_ = std::atoi(g) != 0;
  // experiments / tests: prefix inputs without page sharing (every request its own donor)
  if (const char* g = std::getenv("BH_PREFIX_SHARE")) prefix_share_ = std::atoi(g) != 0;
  max_batch_tokens_ = w.max_batch_tokens > 0 ? w.max_batch_tokens : 4096;
  d_ = w.blocks[0].d_model;
  for (int b = 0; b < w.n_blocks; ++b) {
    if (w.blocks[b].d_model != d_) throw BeError(BE_ERR_INVALID, "runner: blocks differ in d_model");
    descs_.push_back(w.blocks[b]);
    names_.push_back(w.blocks[b].name ? w.blocks[b].name : ("b" + std::to_string(b)));
    descs_.back().name = nullptr;
  }
  chain_ptr_.assign(w.chain_ptr, w.chain_ptr + w.n_tenants + 1);
  chain_blocks_.assign(w.chain_blocks, w.chain_blocks + chain_ptr_.back());
  for (int t = 0; t < w.n_tenants; ++t) {
    if (chain_ptr_[t + 1] <= chain_ptr_[t]) throw BeError(BE_ERR_INVALID, "runner: empty chain");
    for (int s = chain_ptr_[t]; s < chain_ptr_[t + 1]; ++s)
      if (chain_blocks_[s] < 0 || chain_blocks_[s] >= w.n_blocks)
        throw BeError(BE_ERR_INVALID, "runner: chain names an unknown block");
  }
  // requests; per-block KV page demand
  std::vector<long long> pages_needed(w.n_blocks, 0);
  int poff = 0, max_prompt = 0;
  for (int i = 0; i < w.n_requests; ++i) {
    Request r;
    r.idx = i;
    r.id = i + 1;
    r.tenant = w.req_tenant[i];
    r.prompt = w.req_prompt[i];
    r.output = w.req_output[i];
    if (r.tenant < 0 || r.tenant >= w.n_tenants || r.prompt <= 0 || r.output <= 0)
      throw BeError(BE_ERR_INVALID, "runner: bad request");
    r.ctx = r.prompt;
    r.poff = poff;
    if (w.req_prefix_group != nullptr && w.req_prefix_tokens != nullptr &&
        w.req_prefix_group[i] >= 0 && w.req_prefix_tokens[i] > 0) {
      r.prefix_group = w.req_prefix_group[i];
      r.prefix_tokens = std::min(w.req_prefix_tokens[i], r.prompt);
    }
    poff += r.prompt;
    max_prompt = std::max(max_prompt, r.prompt);
    const int total = r.prompt + r.output;
    max_ctx_ = std::max(max_ctx_, total);
    for (int s = chain_ptr_[r.tenant]; s < chain_ptr_[r.tenant + 1]; ++s)
      pages_needed[chain_blocks_[s]] += pages_for(total) + 1;
    reqs_.push_back(r);
  }
  lora_base_.assign(w.n_blocks, -1);
  if (w.block_lora_base != nullptr) {
    for (int b = 0; b < w.n_blocks; ++b) {
      const int base = w.block_lora_base[b];
      if (base < -1 || base >= w.n_blocks || base == b ||
          (base >= 0 && (w.block_lora_base[base] >= 0 || w.block_lora_name == nullptr ||
                         w.block_lora_name[b] == nullptr)))
        throw BeError(BE_ERR_INVALID, "runner: bad LoRA base for block " + std::to_string(b));
      lora_base_[b] = base;
    }
  }
  blocks_.assign(w.n_blocks, nullptr);
  pools_.assign(w.n_blocks, nullptr);
  loras_.assign(w.n_blocks, nullptr);
  own_block_.assign(w.n_blocks, 0);
  std::vector<int> np_of(w.n_blocks, 1);
  int dff = 0, H = 0;
  for (int b = 0; b < w.n_blocks; ++b) {
    // component sequence -> KV bytes per token (4 * d per attention component,
    // CostModel::kv_bytes_per_token, costmodel.cpp:114-127)
    int n_att = 0;
    if (w.blocks[b].components != nullptr) {
      for (const char* c = w.blocks[b].components; *c; ++c) n_att += *c == 'a' ? 1 : 0;
      comps_.push_back(w.blocks[b].components);
    } else {
      n_att = w.blocks[b].n_layers;
      comps_.push_back(std::string());
    }
    kv_bpt_.push_back(4LL * d_ * n_att);
    descs_[b].components = nullptr;  // re-pointed at comps_ when loading
    if (descs_[b].max_pos < max_ctx_) descs_[b].max_pos = max_ctx_ + 16;
    const int np = static_cast<int>(std::max<long long>(1, pages_needed[b]));
    if (kv_bpt_[b] > 0) kv_.attach_pool(names_[b], 0, np);
    if (dff == 0) {
      dff = descs_[b].d_ff;
      H = descs_[b].n_heads;
    } else if (dff != descs_[b].d_ff || H != descs_[b].n_heads) {
      throw BeError(BE_ERR_INVALID, "runner: blocks differ in d_ff / heads");
    }
    np_of[b] = np;
    if (dry_ || lora_base_[b] >= 0) continue;  // LoRA variants: after their base is loaded
    be_block_desc d = descs_[b];
    d.name = names_[b].c_str();
    d.components = comps_[b].empty() ? nullptr : comps_[b].c_str();
    be_block* blk = nullptr;
    int rc = be_block_load(ctx, &d, &blk);
    if (rc != BE_OK) throw BeError(rc, std::string("block load: ") + be_last_error(ctx));
    blocks_[b] = blk;
    own_block_[b] = 1;
    be_kv_pool* kp = nullptr;
    rc = be_kv_pool_create(ctx, blk, np, &kp);
    if (rc != BE_OK) throw BeError(rc, std::string("kv pool: ") + be_last_error(ctx));
    pools_[b] = kp;
  }
  // LoRA variants: the base's weights, their own adapter and KV pool
  for (int b = 0; b < w.n_blocks && !dry_; ++b) {
    const int base = lora_base_[b];
    if (base < 0) continue;
    if (comps_[b] != comps_[base] || descs_[b].d_ff != descs_[base].d_ff)
      throw BeError(BE_ERR_INVALID, "runner: a LoRA variant must have its base's shape");
    blocks_[b] = blocks_[base];
    int rc = be_lora_load(ctx, blocks_[base], w.block_lora_name[b], w.seed, descs_[b].init_scale,
                          descs_[b].init_scale, &loras_[b]);
    if (rc != BE_OK) throw BeError(rc, std::string("lora load: ") + be_last_error(ctx));
    rc = be_kv_pool_create(ctx, blocks_[base], np_of[b], &pools_[b]);
    if (rc != BE_OK) throw BeError(rc, std::string("kv pool: ") + be_last_error(ctx));
  }
  inst_of_block_.assign(w.n_blocks, "");
  inst_index_.assign(w.n_blocks, -1);
  n_created_ = 0;
  if (dry_) return;
  const int max_tok = std::max(std::min(poff, std::max(max_batch_tokens_, max_prompt)), w.n_requests);
  int rc = be_workspace_create(ctx, d_, dff, H, max_tok, w.n_requests, pages_for(max_ctx_) + 1, &ws_);
  if (rc != BE_OK) throw BeError(rc, std::string("workspace: ") + be_last_error(ctx));
  if (std::any_of(lora_base_.begin(), lora_base_.end(), [](int x) { return x >= 0; })) {
    ck(cudaMalloc(&d_zero_idx_, (size_t)max_tok * sizeof(int32_t)), "lora idx");
    ck(cudaMemsetAsync(d_zero_idx_, 0, (size_t)max_tok * sizeof(int32_t), st_), "lora idx");
  }
  spec_.assign(w.n_blocks, 0);
  sur_.assign(w.n_blocks, nullptr);
  sur_pool_.assign(w.n_blocks, nullptr);
  if (w.n_spec_blocks > 0 && w.spec_blocks != nullptr) {
    spec_thr_ = w.spec_threshold;
    const float keep = w.spec_keep > 0.f && w.spec_keep < 1.f ? w.spec_keep : 0.5f;
    for (int i = 0; i < w.n_spec_blocks; ++i) {
      const int b = w.spec_blocks[i];
      if (b < 0 || b >= w.n_blocks || lora_base_[b] >= 0 || kv_bpt_[b] == 0)
        throw BeError(BE_ERR_INVALID, "runner: block " + std::to_string(b) + " cannot speculate");
      if (spec_[b]) continue;
      spec_[b] = 1;
      // the surrogate: the block's own weights with the FFN cut to a channel prefix
      be_block_desc sd = descs_[b];
      sd.name = names_[b].c_str();
      sd.components = comps_[b].empty() ? nullptr : comps_[b].c_str();
      sd.ffn_src = descs_[b].d_ff;
      sd.d_ff = std::max(64, (int)(descs_[b].d_ff * keep) / 64 * 64);
      rc = be_block_load(ctx, &sd, &sur_[b]);
      if (rc != BE_OK) throw BeError(rc, std::string("surrogate load: ") + be_last_error(ctx));
      rc = be_kv_pool_create(ctx, sur_[b], np_of[b], &sur_pool_[b]);
      if (rc != BE_OK) throw BeError(rc, std::string("surrogate kv pool: ") + be_last_error(ctx));
    }
    rc = be_workspace_create(ctx, d_, dff, H, max_tok, w.n_requests, pages_for(max_ctx_) + 1,
                             &ws_verify_);
    if (rc != BE_OK) throw BeError(rc, std::string("verify workspace: ") + be_last_error(ctx));
    ck(cudaMalloc(&spec_buf_, (size_t)3 * w.n_requests * d_ * 2), "speculation rows");
    ck(cudaMalloc(&spec_dst_, (size_t)w.n_requests * sizeof(int32_t)), "speculation rows");
  }
  ck(cudaMalloc(&arena_, (size_t)w.n_requests * d_ * 2), "arena");
  ck(cudaMalloc(&parena_, (size_t)poff * d_ * 2), "prefill arena");
  prefill_rows_ = poff;
  for (const auto& r : reqs_) {
    const std::string sid = "inputs:req" + std::to_string(r.id);
    rc = be_synth_rows(ctx, static_cast<char*>(parena_) + (size_t)r.poff * d_ * 2,
                       (int64_t)r.prompt * d_, w.seed, sid.c_str(), 1.7320508f, st_);
    if (rc != BE_OK) throw BeError(rc, "synthetic prompts");
    if (r.prefix_group >= 0) {  // the group's common prefix
      const std::string pid = "inputs:prefix" + std::to_string(r.prefix_group);
      rc = be_synth_rows(ctx, static_cast<char*>(parena_) + (size_t)r.poff * d_ * 2,
                         (int64_t)r.prefix_tokens * d_, w.seed, pid.c_str(), 1.7320508f, st_);
      if (rc != BE_OK) throw BeError(rc, "synthetic prefixes");
    }
  }
  ck(cudaStreamSynchronize(st_), "init");
}

Runner::~Runner() { release(); }

void Runner::release() {
  for (auto& kv : graphs_) kv.second.reset();
  if (!dry_ && st_ != nullptr) cudaStreamSynchronize(st_);
  for (int k = 0; k < 2; ++k) {
    if (meta_host_[k]) cudaFreeHost(meta_host_[k]);
    if (meta_ev_[k]) cudaEventDestroy(meta_ev_[k]);
  }
  if (meta_dev_) cudaFree(meta_dev_);
  if (arena_) cudaFree(arena_);
  if (parena_) cudaFree(parena_);
  if (ws_) be_workspace_free(ws_);
  for (auto* p : pools_)
    if (p) be_kv_pool_free(p);
  for (size_t b = 0; b < blocks_.size(); ++b)
    if (own_block_[b] && blocks_[b]) be_block_free(blocks_[b]);
  for (auto* l : loras_)
    if (l) be_lora_free(l);
  if (d_zero_idx_) cudaFree(d_zero_idx_);
  for (auto* p : sur_pool_)
    if (p) be_kv_pool_free(p);
  for (auto* b : sur_)
    if (b) be_block_free(b);
  if (ws_verify_) be_workspace_free(ws_verify_);
  if (spec_buf_) cudaFree(spec_buf_);
  if (spec_dst_) cudaFree(spec_dst_);
}

int Runner::live() const {
  int n = 0;
  for (const auto& r : reqs_) n += r.done ? 0 : 1;
  return n;
}

std::string Runner::instance_for(int block) {
  if (inst_of_block_[block].empty()) {
    // created on first dispatch, ready at once (parameters resident: no load time here)
    Instance& in = pool_.create(names_[block], 0, 0, 0);
    inst_of_block_[block] = in.id;
    inst_index_[block] = n_created_++;
  }
  return inst_of_block_[block];
}

void Runner::dispatch(Request& r) {
  const int block = chain_block(r, r.step);
  const std::string inst = instance_for(block);
  Entry e;
  e.request_id = r.id;
  e.chain_step = r.step;
  e.phase = r.phase;
  e.tokens = r.phase == Phase::kPrefill ? r.prompt : 1;
  e.context_tokens = r.ctx;
  e.kv_resident = r.phase == Phase::kDecode && kv_.device_of(r.id, names_[block]) == 0;
  pool_.enqueue(inst, e);
}

PlannedBatch Runner::plan(const std::string& inst_id, const Batch& b) {
  PlannedBatch pb;
  const Instance& in = pool_.get(inst_id);
  int block = 0;
  while (names_[block] != in.block_id) ++block;
  pb.block = block;
  pb.inst = inst_index_[block];
  pb.phase = b.phase;
  pb.n_rows = static_cast<int>(b.members.size());
  pb.stride = pages_for(max_ctx_) + 1;
  pb.pt.assign((size_t)pb.n_rows * pb.stride, -1);
  for (int m = 0; m < pb.n_rows; ++m) {
    const Entry& e = b.members[m];
    Request& r = reqs_[e.request_id - 1];
    const std::string& bn = names_[block];
    // the decode token sits at position context - 1 (the segment holds the tokens before it)
    const int first = b.phase == Phase::kPrefill ? 0 : r.ctx - 1;
    const int count = b.phase == Phase::kPrefill ? r.prompt : 1;
    std::vector<int> row;
    int shared = 0;
    if (kv_bpt_[block] > 0) {
      if (b.phase == Phase::kDecode && kv_.tokens(r.id, bn) != first)
        throw BeError(BE_ERR_STATE, "runner: kv segment out of step with the context");
      int want = 0;
      const int donor = b.phase == Phase::kPrefill && !kv_.has_segment(r.id, bn)
                            ? prefix_donor(r, block, &want) : -1;
      if (donor > 0) {
        // the donor's whole prefix pages (share_prefix, kv.cpp): the prefill reads them and
        // rewrites the same K/V into them (identical prefix tokens, identical bits)
        const std::vector<int> ds = kv_.page_slots(donor, bn);
        shared = std::min(std::min(want, kv_.tokens(donor, bn)) / kPageTokens, (int)ds.size());
        row.assign(ds.begin(), ds.begin() + shared);
        const std::vector<int> own =
            kv_.reserve_slots(r.id, bn, bn, 0, pages_for(first + count) - shared);
        row.insert(row.end(), own.begin(), own.end());
      } else {
        row = kv_.reserve_slots(r.id, bn, bn, 0, pages_for(first + count));
      }
      std::copy(row.begin(), row.end(), pb.pt.begin() + (size_t)m * pb.stride);
    } else {
      row.assign(pages_for(first + count), 0);  // ffn-only block: no KV is written or read
    }
    for (int i = 0; i < count; ++i) {
      const int pos = first + i;
      be_token t;
      if (b.phase == Phase::kPrefill) {
        t.src_row = r.poff + i;
        t.dst_row = r.poff + i;
      } else {
        t.src_row = r.idx;
        t.dst_row = r.idx;
      }
      t.kv_slot = row[pos / kPageTokens] * kPageTokens + pos % kPageTokens;
      t.pos = pos;
      t.pt_row = m;
      pb.toks.push_back(t);
    }
    pb.shared_pages.push_back(shared);
  }
  return pb;
}

// create_kv_for_step's donor rule (scenario.cpp:679-692): the group's recorded donor at this
// block, if it is another request whose segment already holds the prefix; -1 otherwise.
int Runner::prefix_donor(const Request& r, int block, int* want) const {
  if (r.prefix_group < 0 || r.prefix_tokens <= 0 || !prefix_share_) return -1;
  *want = std::min(r.prefix_tokens, r.prompt);
  auto it = prefix_donors_.find({r.prefix_group, block});
  if (it == prefix_donors_.end() || it->second == r.id) return -1;
  const std::string& bn = names_[block];
  if (!kv_.has_segment(it->second, bn) || kv_.tokens(it->second, bn) < *want) return -1;
  return it->second;
}

void Runner::launch(const PlannedBatch& pb, const be_token* d_tok, const int32_t* d_pt) {
  void* arena = pb.phase == Phase::kPrefill ? parena_ : arena_;
  if (loras_[pb.block] != nullptr) {
    const be_lora* l = loras_[pb.block];
    const int rc = be_exec_lora_batch_dev(
        ctx_, blocks_[pb.block], pools_[pb.block], ws_,
        pb.phase == Phase::kPrefill ? BE_PHASE_PREFILL : BE_PHASE_DECODE,
        static_cast<int>(pb.toks.size()), d_tok, pb.stride, d_pt, 1, &l, d_zero_idx_, arena, arena,
        st_);
    if (rc != BE_OK) throw BeError(rc, std::string("exec lora: ") + be_last_error(ctx_));
    return;
  }
  const int rc = be_exec_batch_dev(ctx_, blocks_[pb.block], pools_[pb.block], ws_,
                                   pb.phase == Phase::kPrefill ? BE_PHASE_PREFILL : BE_PHASE_DECODE,
                                   static_cast<int>(pb.toks.size()), d_tok, pb.stride, d_pt, arena,
                                   arena, st_);
  if (rc != BE_OK) throw BeError(rc, std::string("exec: ") + be_last_error(ctx_));
}

void Runner::execute_direct(const PlannedBatch& pb) {
  if (dry_) return;
  void* arena = pb.phase == Phase::kPrefill ? parena_ : arena_;
  if (loras_[pb.block] != nullptr) {
    const be_lora* l = loras_[pb.block];
    const std::vector<int32_t> zeros(pb.toks.size(), 0);
    const int rc = be_exec_lora_batch(ctx_, blocks_[pb.block], pools_[pb.block], ws_,
                                      pb.phase == Phase::kPrefill ? BE_PHASE_PREFILL : BE_PHASE_DECODE,
                                      static_cast<int>(pb.toks.size()), pb.toks.data(), pb.n_rows,
                                      pb.stride, pb.pt.data(), 1, &l, zeros.data(), arena, arena, st_);
    if (rc != BE_OK) throw BeError(rc, std::string("exec lora: ") + be_last_error(ctx_));
    ck(cudaStreamSynchronize(st_), "batch");
    return;
  }
  const int rc = be_exec_batch(ctx_, blocks_[pb.block], pools_[pb.block], ws_,
                               pb.phase == Phase::kPrefill ? BE_PHASE_PREFILL : BE_PHASE_DECODE,
                               static_cast<int>(pb.toks.size()), pb.toks.data(), pb.n_rows,
                               pb.stride, pb.pt.data(), arena, arena, st_);
  if (rc != BE_OK) throw BeError(rc, std::string("exec: ") + be_last_error(ctx_));
  // be_exec_batch stages metadata from pageable memory: keep the host side in step
  ck(cudaStreamSynchronize(st_), "batch");
}

void Runner::record(const PlannedBatch& pb, const Batch& b) {
  bh_batch_rec rec;
  rec.instance = pb.inst;
  rec.block = pb.block;
  rec.phase = b.phase == Phase::kPrefill ? BE_PHASE_PREFILL : BE_PHASE_DECODE;
  rec.n_members = static_cast<int32_t>(b.members.size());
  rec.first_member = static_cast<int32_t>(m_req.size());
  for (const auto& e : b.members) {
    m_req.push_back(e.request_id);
    m_step.push_back(e.chain_step);
    m_ctx.push_back(e.context_tokens);
  }
  recs.push_back(rec);
}

void Runner::account(const PlannedBatch& pb) {
  const be_block_desc& D = descs_[pb.block];
  const double d = D.d_model, F = D.d_ff;
  const double La = static_cast<double>(kv_bpt_[pb.block]) / (4.0 * d);  // attention components
  const std::string& cs = comps_[pb.block];
  const double Lf = cs.empty() ? D.n_layers : static_cast<double>(cs.size()) - La;
  const double n = static_cast<double>(pb.toks.size());
  stats.weight_bytes += 2.0 * (La * 4.0 * d * d + Lf * 3.0 * d * F);
  double ctx_sum = 0.0;
  for (const auto& t : pb.toks) ctx_sum += t.pos + 1;
  stats.kv_bytes += ctx_sum * La * 2.0 * d * 2.0;
  stats.act_bytes += 2.0 * n * d * 2.0;
  stats.flops += 2.0 * n * (La * 4.0 * d * d + Lf * 3.0 * d * F) + 4.0 * ctx_sum * d * La;
  if (!dry_)
    stats.launches += be_exec_batch_launches(ctx_, blocks_[pb.block],
                                             static_cast<int>(pb.toks.size()), pb.stride) +
                      lora_launches(pb.block);
}

void Runner::pump() {
  if (has_running_) return;  // decode joins only happen on multi-lane timelines
  Instance* in = pool_.next_runnable(0, 0);
  if (in == nullptr) return;
  running_inst_ = in->id;
  running_ = pool_.pop_batch(in->id, max_batch_tokens_, 0);
  running_plan_ = plan(running_inst_, running_);
  record(running_plan_, running_);
  has_running_ = true;
}

void Runner::finish_running() {
  // the block run (replaces the cost-table duration of pump)
  execute_direct(running_plan_);
  account(running_plan_);
  ++batches_run_;
  has_running_ = false;
  pool_.finish_batch(running_inst_, 0);
  const Batch b = running_;
  for (size_t i = 0; i < b.members.size(); ++i)
    advance_after_step(reqs_[b.members[i].request_id - 1], b.members[i].chain_step,
                       running_plan_.shared_pages[i]);
  pump();
}

void Runner::advance_after_step(Request& r, int step, int planned_shared) {
  if (r.phase == Phase::kPrefill) {
    const int block = chain_block(r, step);
    const std::string& bn = names_[block];
    if (kv_bpt_[block] > 0 && !kv_.has_segment(r.id, bn)) {
      // create_kv_for_step (scenario.cpp:671-695): share the donor's prefix or become the donor
      int want = 0;
      const int donor = prefix_donor(r, block, &want);
      kv_.create_segment(r.id, bn, 0, kv_bpt_[block]);
      int covered = 0;
      if (donor > 0) {
        covered = kv_.share_prefix(r.id, donor, bn, want);
      } else if (r.prefix_group >= 0) {
        prefix_donors_[{r.prefix_group, block}] = r.id;
      }
      // a donor that finished in the same batch: the request wrote its own prefix pages too;
      // the shared ones replace them
      kv_.drop_reserved_front(r.id, bn, covered / kPageTokens - planned_shared);
      kv_.append_tokens(r.id, bn, r.prompt - covered);
    }
  }
  advance_from(r, step);
}

void Runner::advance_from(Request& r, int step) {
  if (step + 1 < chain_len(r)) {
    r.step = step + 1;
    dispatch(r);
    return;
  }
  if (r.phase == Phase::kPrefill) {
    // first token: the last prompt row's output becomes the first decode input
    if (!dry_)
      ck(cudaMemcpyAsync(static_cast<char*>(arena_) + (size_t)r.idx * d_ * 2,
                         static_cast<char*>(parena_) + (size_t)(r.poff + r.prompt - 1) * d_ * 2,
                         (size_t)d_ * 2, cudaMemcpyDeviceToDevice, st_),
         "first token row");
    r.generated = 1;
    ++tokens_generated_;
    r.ctx = r.prompt + 1;
    if (serving_) just_first_.push_back(r.idx);
    if (r.generated >= r.output) {
      r.done = true;
      if (serving_) just_done_.push_back(r.idx);
      kv_.release_request(r.id);
      return;
    }
    r.phase = Phase::kDecode;
    r.step = 0;
    if (mode_ == 0) dispatch(r);
    return;
  }
  // decode token done: one more token on every segment of the chain
  for (int s = 0; s < chain_len(r); ++s) kv_.append_if_present(r.id, names_[chain_block(r, s)], 1);
  r.generated += 1;
  ++tokens_generated_;
  r.ctx += 1;
  if (r.generated >= r.output) {
    r.done = true;
    if (serving_) just_done_.push_back(r.idx);
    kv_.release_request(r.id);
    return;
  }
  r.step = 0;
  if (mode_ == 0) {
    dispatch(r);
  } else {
    step_done_order_.push_back(r.idx);
  }
}

void Runner::run(int max_batches) {
  if (batches_run_ == 0 && !has_running_) {
    // arrivals at t = 0 in request order; the first one starts the lane at once
    for (auto& r : reqs_) {
      dispatch(r);
      pump();
    }
  }
  int n = 0;
  while (has_running_ && (max_batches <= 0 || n < max_batches)) {
    finish_running();
    ++n;
  }
  if (!dry_) ck(cudaStreamSynchronize(st_), "run");
  if (mode_ == 1 && !has_running_) {
    // lockstep: decode starts for everyone together, in request order
    step_done_order_.clear();
    for (const auto& r : reqs_)
      if (!r.done && r.phase == Phase::kDecode) step_done_order_.push_back(r.idx);
  }
}

// Consecutive decode batches at blocks of one shape and component sequence whose members are
// disjoint (no request is in two of them, so none consumes another's output) form one grouped
// launch (be_exec_group_dev) - e.g. the tenants' private blocks at one chain position. Groups
// need equal member counts of 16/32/64 (the GEMM n-tile of each block).
std::vector<Runner::LaunchEntry> Runner::group_plans(const std::vector<PlannedBatch>& plans) const {
  std::vector<LaunchEntry> out;
  size_t i = 0;
  while (i < plans.size()) {
    LaunchEntry le;
    le.plans.push_back(static_cast<int>(i));
    const PlannedBatch& a = plans[i];
    const bool groupable = group_ && a.phase == Phase::kDecode && a.toks.size() <= 64;
    std::vector<int> seen;
    for (const auto& t : a.toks) seen.push_back(t.src_row);
    size_t j = i + 1;
    size_t rmax = a.toks.size();
    while (groupable && j < plans.size() && le.plans.size() < 8) {
      const PlannedBatch& b = plans[j];
      if (b.phase != Phase::kDecode || b.toks.size() > 64 || comps_[b.block] != comps_[a.block] ||
          descs_[b.block].d_ff != descs_[a.block].d_ff || b.block == a.block)
        break;
      // LoRA variants group only with variants of the same base (one shared weight stream)
      const bool la = lora_base_[a.block] >= 0, lb = lora_base_[b.block] >= 0;
      if ((la || lb) && wbase(a.block) != wbase(b.block)) break;
      bool disjoint = true;
      for (const auto& t : b.toks)
        if (std::find(seen.begin(), seen.end(), t.src_row) != seen.end()) disjoint = false;
      if (!disjoint) break;
      for (const auto& t : b.toks) seen.push_back(t.src_row);
      le.plans.push_back(static_cast<int>(j));
      rmax = std::max(rmax, b.toks.size());
      ++j;
    }
    if (le.plans.size() > 1) {
      // rows per block: the GEMM n-tile (16/32/64); shorter batches get padding rows that are
      // computed but never stored (dst -1, no KV slot, empty context)
      const size_t R = rmax <= 16 ? 16 : rmax <= 32 ? 32 : 64;
      for (int k : le.plans) le.stride = std::max(le.stride, plans[k].stride);
      int row0 = 0;
      for (int k : le.plans) {
        const PlannedBatch& pb = plans[k];
        for (be_token t : pb.toks) {
          t.pt_row += row0;
          le.toks.push_back(t);
        }
        for (size_t p = pb.toks.size(); p < R; ++p) {
          be_token pad;
          pad.src_row = pb.toks[0].src_row;
          pad.dst_row = -1;
          pad.kv_slot = -1;
          pad.pos = -1;
          pad.pt_row = row0;
          le.toks.push_back(pad);
        }
        for (int r = 0; r < pb.n_rows; ++r)
          for (int c = 0; c < le.stride; ++c)
            le.pt.push_back(c < pb.stride ? pb.pt[(size_t)r * pb.stride + c] : -1);
        row0 += pb.n_rows;
      }
      for (int k : le.plans) le.lora = le.lora || lora_base_[plans[k].block] >= 0;
      if (le.lora)
        for (size_t g = 0; g < le.plans.size(); ++g)
          for (size_t p = 0; p < R; ++p)
            le.lidx.push_back(lora_base_[plans[le.plans[g]].block] >= 0 && p < plans[le.plans[g]].toks.size()
                                  ? static_cast<int32_t>(g) : -1);
    }
    out.push_back(std::move(le));
    i = j;
  }
  return out;
}

void Runner::launch_entry(const std::vector<PlannedBatch>& plans, const LaunchEntry& le,
                          const be_token* d_tok, const int32_t* d_pt, const int32_t* d_idx) {
  if (le.plans.size() == 1) {
    launch(plans[le.plans[0]], d_tok, d_pt);
    return;
  }
  be_block* blks[8];
  be_kv_pool* pls[8];
  for (size_t g = 0; g < le.plans.size(); ++g) {
    blks[g] = blocks_[plans[le.plans[g]].block];
    pls[g] = pools_[plans[le.plans[g]].block];
  }
  if (le.lora) {
    // adapter slot g = group g's variant (a group of the base itself keeps index -1)
    const be_lora* ls[8];
    const be_lora* any = nullptr;
    for (size_t g = 0; g < le.plans.size(); ++g)
      if (loras_[plans[le.plans[g]].block]) any = loras_[plans[le.plans[g]].block];
    for (size_t g = 0; g < le.plans.size(); ++g) {
      const be_lora* l = loras_[plans[le.plans[g]].block];
      ls[g] = l ? l : any;
    }
    const int rc = be_exec_lora_group_dev(
        ctx_, static_cast<int>(le.plans.size()), blks, pls, ws_, BE_PHASE_DECODE,
        static_cast<int>(le.toks.size()), d_tok, le.stride, d_pt,
        static_cast<int>(le.plans.size()), ls, d_idx, arena_, arena_, st_);
    if (rc != BE_OK) throw BeError(rc, std::string("exec lora group: ") + be_last_error(ctx_));
    return;
  }
  const int rc = be_exec_group_dev(ctx_, static_cast<int>(le.plans.size()), blks, pls, ws_,
                                   BE_PHASE_DECODE, static_cast<int>(le.toks.size()), d_tok,
                                   le.stride, d_pt, arena_, arena_, st_);
  if (rc != BE_OK) throw BeError(rc, std::string("exec group: ") + be_last_error(ctx_));
}

Runner::StepPlan Runner::plan_step(int group, const std::vector<int>* members) {
  StepPlan sp;
  sp.valid = true;
  sp.group = group;
  std::vector<int> order;
  if (members == nullptr) {
    order = step_done_order_;
    step_done_order_.clear();
  } else {
    // one micro-batch of the pipeline: its requests step, the others keep waiting
    std::vector<char> in(reqs_.size(), 0);
    for (int idx : *members) {
      if (idx < 0 || idx >= (int)reqs_.size()) throw BeError(BE_ERR_INVALID, "bad request index");
      in[idx] = 1;
    }
    std::vector<int> rest;
    for (int idx : step_done_order_) (in[idx] ? order : rest).push_back(idx);
    step_done_order_.swap(rest);
  }
  // host rows are the live requests in request order
  sp.rows = order;
  std::sort(sp.rows.begin(), sp.rows.end());
  for (int idx : order) dispatch(reqs_[idx]);
  // plan the whole step on the host (bookkeeping does not depend on GPU results)
  const bh_step_stats saved = stats;
  stats = bh_step_stats{};
  for (;;) {
    pump();
    if (!has_running_) break;
    sp.plans.push_back(running_plan_);
    has_running_ = false;
    pool_.finish_batch(running_inst_, 0);
    account(running_plan_);
    ++batches_run_;
    for (size_t i = 0; i < running_.members.size(); ++i)
      advance_after_step(reqs_[running_.members[i].request_id - 1], running_.members[i].chain_step,
                         running_plan_.shared_pages[i]);
  }
  sp.stats = stats;
  stats = saved;
  if (dry_) return sp;
  // launches: single batches, and groups of independent same-shape batches
  sp.entries = group_plans(sp.plans);
  const auto& plans = sp.plans;
  auto ent_toks = [&](const LaunchEntry& le) -> const std::vector<be_token>& {
    return le.plans.size() == 1 ? plans[le.plans[0]].toks : le.toks;
  };
  if (sp.entries.size() != plans.size()) {  // launch accounting per grouped launch
    sp.stats.launches = 0;
    for (const auto& le : sp.entries) {
      const PlannedBatch& p0 = plans[le.plans[0]];
      int lora_extra = 0;
      for (int k : le.plans) lora_extra = std::max(lora_extra, lora_launches(plans[k].block));
      sp.stats.launches += be_exec_batch_launches(ctx_, blocks_[p0.block],
                                                  static_cast<int>(ent_toks(le).size()),
                                                  le.plans.size() == 1 ? p0.stride : le.stride) +
                           lora_extra;
    }
  }
  // LoRA groups stream the shared base weights once (account() charged every variant), plus
  // each variant's adapter factors (8 r d bf16 per attention component)
  for (const auto& le : sp.entries) {
    if (!le.lora) continue;
    const PlannedBatch& p0 = plans[le.plans[0]];
    const be_block_desc& D = descs_[p0.block];
    const double d = D.d_model, F = D.d_ff;
    const double La = static_cast<double>(kv_bpt_[p0.block]) / (4.0 * d);
    const double Lf = comps_[p0.block].empty() ? D.n_layers
                                               : static_cast<double>(comps_[p0.block].size()) - La;
    const double w = 2.0 * (La * 4.0 * d * d + Lf * 3.0 * d * F);
    const double g = static_cast<double>(le.plans.size());
    sp.stats.weight_bytes -= (g - 1.0) * w;
    sp.stats.weight_bytes += g * La * 8.0 * 16.0 * d * 2.0;
  }
  // metadata layout: per launch [tokens][page table], 256-byte aligned
  sp.off_tok.resize(sp.entries.size());
  sp.off_pt.resize(sp.entries.size());
  sp.off_idx.resize(sp.entries.size());
  for (size_t i = 0; i < sp.entries.size(); ++i) {
    const LaunchEntry& le = sp.entries[i];
    const auto& tk = ent_toks(le);
    const auto& pt = le.plans.size() == 1 ? plans[le.plans[0]].pt : le.pt;
    sp.off_tok[i] = sp.total;
    sp.total += (tk.size() * sizeof(be_token) + 255) & ~size_t(255);
    sp.off_pt[i] = sp.total;
    sp.total += (pt.size() * sizeof(int32_t) + 255) & ~size_t(255);
    sp.off_idx[i] = sp.total;  // LoRA groups: adapter slot per token
    sp.total += (le.lidx.size() * sizeof(int32_t) + 255) & ~size_t(255);
    const int stride = le.plans.size() == 1 ? plans[le.plans[0]].stride : le.stride;
    sp.sig.emplace_back(plans[le.plans[0]].block, static_cast<int>(tk.size()),
                        stride * 16 + static_cast<int>(le.plans.size()));
  }
  return sp;
}

void Runner::stage_and_launch(StepPlan& sp, const void* host_in) {
  const auto& plans = sp.plans;
  const auto& entries = sp.entries;
  const size_t row_bytes = (size_t)d_ * 2;
  if (host_in != nullptr) copy_host_rows(sp.rows, true, const_cast<void*>(host_in));
  if (sp.total > meta_cap_) {
    ck(cudaStreamSynchronize(st_), "meta grow");
    for (int k = 0; k < 2; ++k) {
      if (meta_host_[k]) cudaFreeHost(meta_host_[k]);
      if (!meta_ev_[k]) ck(cudaEventCreateWithFlags(&meta_ev_[k], cudaEventDisableTiming), "meta ev");
    }
    if (meta_dev_) cudaFree(meta_dev_);
    meta_cap_ = sp.total * 2;
    for (int k = 0; k < 2; ++k) ck(cudaMallocHost(&meta_host_[k], meta_cap_), "meta host");
    ck(cudaMalloc(&meta_dev_, meta_cap_), "meta dev");
    for (auto& kv : graphs_) kv.second.reset();  // captured graphs point into the old buffer
  }
  (void)row_bytes;
  GraphSlot& gs = graphs_[sp.group];
  // the device copy of the metadata is stream-ordered after the previous step's kernels; only
  // the host staging slot needs its earlier upload to have executed
  const int slot = meta_slot_;
  meta_slot_ ^= 1;
  ck(cudaEventSynchronize(meta_ev_[slot]), "meta reuse");
  char* stage = meta_host_[slot];
  for (size_t i = 0; i < entries.size(); ++i) {
    const LaunchEntry& le = entries[i];
    const auto& tk = le.plans.size() == 1 ? plans[le.plans[0]].toks : le.toks;
    const auto& pt = le.plans.size() == 1 ? plans[le.plans[0]].pt : le.pt;
    std::memcpy(stage + sp.off_tok[i], tk.data(), tk.size() * sizeof(be_token));
    std::memcpy(stage + sp.off_pt[i], pt.data(), pt.size() * sizeof(int32_t));
    if (!le.lidx.empty())
      std::memcpy(stage + sp.off_idx[i], le.lidx.data(), le.lidx.size() * sizeof(int32_t));
  }
  ck(cudaMemcpyAsync(meta_dev_, stage, sp.total, cudaMemcpyHostToDevice, st_), "meta h2d");
  ck(cudaEventRecord(meta_ev_[slot], st_), "meta ev record");
  auto launch_all = [&]() {
    for (size_t i = 0; i < entries.size(); ++i)
      launch_entry(plans, entries[i], reinterpret_cast<const be_token*>(meta_dev_ + sp.off_tok[i]),
                   reinterpret_cast<const int32_t*>(meta_dev_ + sp.off_pt[i]),
                   reinterpret_cast<const int32_t*>(meta_dev_ + sp.off_idx[i]));
  };
  stats = sp.stats;
  stats.graph_replayed = 0;
  bool any_spec = false;
  for (size_t i = 0; i + 1 < entries.size() && !any_spec; ++i)
    any_spec = spec_pair(plans, entries[i], entries[i + 1]);
  if (any_spec) {
    // speculative pairs are host-synchronous (the K7 verdict is read back): no graph
    for (size_t i = 0; i < entries.size(); ++i) {
      if (i + 1 < entries.size() && spec_pair(plans, entries[i], entries[i + 1])) {
        run_speculative(plans[entries[i].plans[0]], plans[entries[i + 1].plans[0]]);
        ++i;
        continue;
      }
      launch_entry(plans, entries[i], reinterpret_cast<const be_token*>(meta_dev_ + sp.off_tok[i]),
                   reinterpret_cast<const int32_t*>(meta_dev_ + sp.off_pt[i]),
                   reinterpret_cast<const int32_t*>(meta_dev_ + sp.off_idx[i]));
    }
    gs.reset();
    gs.sig.clear();
    return;
  }
  if (be_prof_active(ctx_)) {
    launch_all();  // per-launch event timing: plain launches, the captured graph is kept
    if (sp.sig != gs.sig) gs.reset();
  } else if (use_graphs_ && sp.sig == gs.sig && gs.exec != nullptr) {
    ck(cudaGraphLaunch(gs.exec, st_), "graph launch");
    stats.graph_replayed = 1;
  } else if (use_graphs_ && sp.sig == gs.sig) {
    // second step with this structure: capture it
    ck(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal), "capture begin");
    try {
      launch_all();
    } catch (...) {
      cudaGraph_t g;
      cudaStreamEndCapture(st_, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    gs.reset();
    ck(cudaStreamEndCapture(st_, &gs.graph), "capture end");
    ck(cudaGraphInstantiate(&gs.exec, gs.graph, 0), "graph instantiate");
    ck(cudaGraphLaunch(gs.exec, st_), "graph launch");
    stats.graph_replayed = 1;
  } else {
    launch_all();
    gs.reset();
  }
  gs.sig = sp.sig;
}

// host rows <-> arena rows of a step's live requests; contiguous runs move in one copy
void Runner::copy_host_rows(const std::vector<int>& rows, bool to_dev, void* host) {
  const size_t row_bytes = (size_t)d_ * 2;
  size_t i = 0;
  while (i < rows.size()) {
    size_t j = i + 1;
    while (j < rows.size() && rows[j] == rows[j - 1] + 1) ++j;
    char* dev = static_cast<char*>(arena_) + (size_t)rows[i] * row_bytes;
    char* hp = static_cast<char*>(host) + i * row_bytes;
    ck(cudaMemcpyAsync(to_dev ? (void*)dev : (void*)hp, to_dev ? (void*)hp : (void*)dev,
                       (j - i) * row_bytes, to_dev ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost,
                       st_),
       "host rows");
    i = j;
  }
}

void Runner::decode_step(const void* host_in, void* host_out, int* n_batches, int group,
                         const std::vector<int>* members) {
  if (mode_ != 1) throw BeError(BE_ERR_STATE, "decode_step needs lockstep mode");
  if (has_running_) throw BeError(BE_ERR_STATE, "prefill still running");
  const bool whole = group < 0 && members == nullptr;
  StepPlan sp;
  if (pending_.valid) {
    if (!whole) throw BeError(BE_ERR_STATE, "a planned-ahead whole step is pending");
    sp = std::move(pending_);
    pending_ = StepPlan{};
  } else {
    sp = plan_step(group, members);
  }
  if (n_batches) *n_batches = static_cast<int>(sp.plans.size());
  if (dry_) {
    stats = sp.stats;
    return;
  }
  stage_and_launch(sp, host_in);
  // plan step k+1 on the host while step k runs on the device (its inputs arrive next call)
  if (plan_ahead_ && whole && !step_done_order_.empty()) pending_ = plan_step(-1, nullptr);
  if (host_out != nullptr) {
    copy_host_rows(sp.rows, false, host_out);
    ck(cudaStreamSynchronize(st_), "d2h sync");
  }
}

// A speculative pair: a marked block's batch followed by a batch of one other block holding the
// same rows in the same order (every member continues to that block), both plain launches.
bool Runner::spec_pair(const std::vector<PlannedBatch>& plans, const LaunchEntry& a,
                       const LaunchEntry& b) const {
  if (a.plans.size() != 1 || b.plans.size() != 1) return false;
  const PlannedBatch& pa = plans[a.plans[0]];
  const PlannedBatch& pb = plans[b.plans[0]];
  if (!spec_[pa.block] || pa.phase != Phase::kDecode || pb.phase != Phase::kDecode ||
      loras_[pb.block] != nullptr || pa.toks.size() != pb.toks.size())
    return false;
  for (size_t i = 0; i < pa.toks.size(); ++i)
    if (pa.toks[i].src_row != pb.toks[i].src_row) return false;
  return true;
}

// be_exec_speculative over the pair (scenario.cpp:502-548 draft + early forward, 740-807
// verification): rows go arena -> [draft | true] scratch rows 0..n-1 -> next -> scratch z ->
// scattered back to their arena rows. The draft keeps its own KV pool (same slots).
void Runner::run_speculative(const PlannedBatch& pv, const PlannedBatch& pn) {
  const int n = static_cast<int>(pv.toks.size());
  const size_t rows_bytes = (size_t)reqs_.size() * d_ * 2;
  char* ydraft = static_cast<char*>(spec_buf_);
  char* ytrue = ydraft + rows_bytes;
  char* z = ytrue + rows_bytes;
  std::vector<be_token> tv(pv.toks), tn(pn.toks);
  std::vector<int32_t> dst(n);
  for (int i = 0; i < n; ++i) {
    dst[i] = tv[i].dst_row;
    tv[i].dst_row = i;  // y rows 0..n-1: K7 compares row i of draft and true
    tn[i].src_row = i;
    tn[i].dst_row = i;
  }
  be_spec_stage verify{blocks_[pv.block], pools_[pv.block], ws_verify_, tv.data(), pv.n_rows,
                       pv.stride, pv.pt.data()};
  be_spec_stage draft{sur_[pv.block], sur_pool_[pv.block], ws_, tv.data(), pv.n_rows, pv.stride,
                      pv.pt.data()};
  be_spec_stage next{blocks_[pn.block], pools_[pn.block], ws_, tn.data(), pn.n_rows, pn.stride,
                     pn.pt.data()};
  std::vector<float> cosv(n);
  std::vector<int32_t> acc(n);
  int n_acc = 0;
  int rc = be_exec_speculative(ctx_, &verify, &draft, &next, n, arena_, ydraft, ytrue, z,
                               spec_thr_, cosv.data(), acc.data(), &n_acc);
  if (rc != BE_OK) throw BeError(rc, std::string("speculative step: ") + be_last_error(ctx_));
  ck(cudaMemcpyAsync(spec_dst_, dst.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, st_),
     "speculation rows");
  rc = be_scatter_rows(ctx_, z, spec_dst_, n, d_, arena_, st_);
  if (rc != BE_OK) throw BeError(rc, std::string("speculative scatter: ") + be_last_error(ctx_));
  ck(cudaStreamSynchronize(st_), "speculation rows");  // dst staged from pageable memory
  spec_stats_.runs += 1;
  spec_stats_.rows += n;
  spec_stats_.accepted += n_acc;
  for (float c : cosv) {
    spec_stats_.cos_sum += c;
    spec_stats_.cos_min = std::min(spec_stats_.cos_min, (double)c);
  }
}

// Taking over requests mid-decode (lockstep mode, a fresh runner): request idx[k] continues at
// context ctx[k] with generated[k] tokens out; on every KV block of its chain a segment holding
// ctx - 1 tokens is created on fresh page slots (kv_segment returns them) for the caller to fill
// with the pages it migrates - the destination side of start_kv_migration
// (scenario.cpp:361-431) when a request's chain steps are rebound to this device.
void Runner::adopt(int n, const int32_t* idx, const int32_t* ctx, const int32_t* generated) {
  if (mode_ != 1) throw BeError(BE_ERR_STATE, "adopt needs lockstep mode");
  if (batches_run_ != 0 || has_running_) throw BeError(BE_ERR_STATE, "adopt on a used runner");
  std::vector<char> seen(reqs_.size(), 0);
  for (int k = 0; k < n; ++k) {
    if (idx[k] < 0 || idx[k] >= (int)reqs_.size() || seen[idx[k]])
      throw BeError(BE_ERR_INVALID, "adopt: bad request index");
    seen[idx[k]] = 1;
    Request& r = reqs_[idx[k]];
    if (ctx[k] <= r.prompt || ctx[k] > r.prompt + r.output || generated[k] < 1 ||
        generated[k] >= r.output || ctx[k] != r.prompt + generated[k])
      throw BeError(BE_ERR_INVALID, "adopt: inconsistent request state");
    r.phase = Phase::kDecode;
    r.step = 0;
    r.ctx = ctx[k];
    r.generated = generated[k];
    for (int s = 0; s < chain_len(r); ++s) {
      const int b = chain_block(r, s);
      if (kv_bpt_[b] == 0) continue;
      const std::string& bn = names_[b];
      kv_.create_segment(r.id, bn, 0, kv_bpt_[b]);
      kv_.append_tokens(r.id, bn, r.ctx - 1);
    }
    tokens_generated_ += generated[k];
  }
  for (int i = 0; i < (int)reqs_.size(); ++i)
    if (seen[i]) step_done_order_.push_back(i);
  batches_run_ = 1;  // the runner is live: run() must not prefill these requests again
}

void Runner::request_state(int idx, int32_t* ctx, int32_t* generated, int32_t* done) const {
  if (idx < 0 || idx >= (int)reqs_.size()) throw BeError(BE_ERR_INVALID, "bad request index");
  const Request& r = reqs_[idx];
  if (ctx) *ctx = r.ctx;
  if (generated) *generated = r.generated;
  if (done) *done = r.done ? 1 : 0;
}

std::vector<int> Runner::kv_segment(int idx, int block, int* tokens) const {
  if (idx < 0 || idx >= (int)reqs_.size() || block < 0 || block >= (int)names_.size())
    throw BeError(BE_ERR_INVALID, "bad request / block index");
  const Request& r = reqs_[idx];
  if (tokens) *tokens = kv_.tokens(r.id, names_[block]);
  return kv_.page_slots(r.id, names_[block]);
}

// Live serving (lockstep mode). Requests arrive at arrival_us (relative to the call) and are
// admitted in arrival order; every admission round prefills the new arrivals through their
// chains (pop_batch under the token budget, batches run as they form, as one device lane does:
// Simulation::pump, scenario.cpp:465-557) and the new decoders board the next lockstep decode
// iteration with everyone already decoding - continuous batching at the iteration boundary, the
// rule try_join_running applies to decode arrivals (scenario.cpp:432-463). Time stamps are taken
// on the host after the stream has drained the batch or step that produced the token.
void Runner::serve(const std::int64_t* arrival_us, std::int64_t* first_us, std::int64_t* done_us) {
  if (mode_ != 1) throw BeError(BE_ERR_STATE, "serve needs lockstep mode");
  if (batches_run_ != 0 || has_running_) throw BeError(BE_ERR_STATE, "serve on a used runner");
  const int n = static_cast<int>(reqs_.size());
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) {
    if (arrival_us[i] < 0) throw BeError(BE_ERR_INVALID, "negative arrival time");
    order[i] = i;
    first_us[i] = done_us[i] = -1;
  }
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return arrival_us[a] < arrival_us[b]; });
  const bool saved_plan_ahead = plan_ahead_;
  plan_ahead_ = false;  // admissions change the next step's membership
  serving_ = true;
  const auto t0 = std::chrono::steady_clock::now();
  auto now_us = [&] {
    return std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() -
                                                                  t0).count();
  };
  auto stamp = [&](std::vector<int>& v, std::int64_t* out) {
    const std::int64_t t = now_us();
    for (int idx : v) out[idx] = t;
    v.clear();
  };
  size_t next = 0;
  int completed = 0;
  try {
    while (completed < n) {
      bool admitted = false;
      while (next < order.size() && arrival_us[order[next]] <= now_us()) {
        dispatch(reqs_[order[next++]]);
        admitted = true;
      }
      if (admitted) {
        // prefill the arrivals: batches run one at a time (execute_direct drains the stream)
        // new decoders board the next decode iteration after everyone already decoding
        auto boarded = [&] {
          for (int idx : just_first_)
            if (!reqs_[idx].done) step_done_order_.push_back(idx);
          stamp(just_first_, first_us);
        };
        pump();
        while (has_running_) {
          finish_running();
          boarded();
        }
        if (!dry_) ck(cudaStreamSynchronize(st_), "serve prefill");
        boarded();
        completed += static_cast<int>(just_done_.size());
        stamp(just_done_, done_us);
        continue;  // arrivals that came during the prefill board before the next step
      }
      if (!step_done_order_.empty()) {
        int nb = 0;
        decode_step(nullptr, nullptr, &nb);
        if (!dry_) ck(cudaStreamSynchronize(st_), "serve step");
        completed += static_cast<int>(just_done_.size());
        stamp(just_done_, done_us);
        continue;
      }
      if (next < order.size()) {
        // idle until the next arrival
        const std::int64_t wait = arrival_us[order[next]] - now_us();
        if (wait > 200) std::this_thread::sleep_for(std::chrono::microseconds(wait - 100));
      } else {
        throw BeError(BE_ERR_STATE, "serve: requests left but nothing to run");
      }
    }
  } catch (...) {
    serving_ = false;
    plan_ahead_ = saved_plan_ahead;
    throw;
  }
  serving_ = false;
  plan_ahead_ = saved_plan_ahead;
}

}  // namespace bh

// ------------------------------------------------------------------------------ C ABI
struct bh_runner {
  std::unique_ptr<bh::Runner> r;
  std::string err;
};

namespace {
template <class F>
int guard(bh_runner* h, F&& f) {
  try {
    f();
    return BE_OK;
  } catch (const bh::BeError& e) {
    if (h) h->err = e.what();
    return e.code;
  } catch (const std::invalid_argument& e) {
    if (h) h->err = e.what();
    return BE_ERR_INVALID;
  } catch (const std::logic_error& e) {
    if (h) h->err = e.what();
    return BE_ERR_STATE;
  } catch (const std::exception& e) {
    if (h) h->err = e.what();
    return BE_ERR_RUNTIME;
  }
}
}  // namespace

extern "C" int bh_runner_create(be_ctx* ctx, const bh_workload* w, bh_runner** out) {
  if (w == nullptr || out == nullptr || (ctx == nullptr && !w->dry_run)) return BE_ERR_INVALID;
  *out = nullptr;
  auto* h = new bh_runner();
  const int rc = guard(h, [&] { h->r = std::make_unique<bh::Runner>(ctx, *w); });
  if (rc != BE_OK) {
    std::fprintf(stderr, "bh_runner_create: %s\n", h->err.c_str());
    delete h;
    return rc;
  }
  *out = h;
  return BE_OK;
}
extern "C" int bh_runner_free(bh_runner* h) {
  if (h == nullptr) return BE_ERR_INVALID;
  delete h;
  return BE_OK;
}
extern "C" const char* bh_runner_last_error(const bh_runner* h) { return h ? h->err.c_str() : "null"; }
extern "C" int bh_runner_run(bh_runner* h, int max_batches) {
  if (h == nullptr) return BE_ERR_INVALID;
  return guard(h, [&] { h->r->run(max_batches); });
}
extern "C" int bh_runner_decode_step(bh_runner* h, const void* in, void* out, int* n_batches) {
  if (h == nullptr) return BE_ERR_INVALID;
  return guard(h, [&] { h->r->decode_step(in, out, n_batches); });
}
extern "C" int bh_runner_decode_group(bh_runner* h, int group, const int32_t* reqs, int n,
                                      const void* in, void* out, int* n_batches) {
  if (h == nullptr || group < 0 || (n > 0 && reqs == nullptr)) return BE_ERR_INVALID;
  std::vector<int> members(reqs, reqs + n);
  return guard(h, [&] { h->r->decode_step(in, out, n_batches, group, &members); });
}
extern "C" int bh_runner_serve(bh_runner* h, const int64_t* arrival_us, int64_t* first_token_us,
                               int64_t* completion_us) {
  if (h == nullptr || arrival_us == nullptr || first_token_us == nullptr || completion_us == nullptr)
    return BE_ERR_INVALID;
  return guard(h, [&] { h->r->serve(arrival_us, first_token_us, completion_us); });
}
extern "C" int bh_runner_adopt(bh_runner* h, int n, const int32_t* idx, const int32_t* ctx,
                               const int32_t* generated) {
  if (h == nullptr || n < 0 || (n > 0 && (idx == nullptr || ctx == nullptr || generated == nullptr)))
    return BE_ERR_INVALID;
  return guard(h, [&] { h->r->adopt(n, idx, ctx, generated); });
}
extern "C" int bh_runner_request_state(const bh_runner* h, int idx, int32_t* ctx,
                                       int32_t* generated, int32_t* done) {
  if (h == nullptr) return BE_ERR_INVALID;
  return guard(const_cast<bh_runner*>(h), [&] { h->r->request_state(idx, ctx, generated, done); });
}
extern "C" int bh_runner_kv_segment(const bh_runner* h, int idx, int block, int32_t* slots, int cap,
                                    int* n_pages, int* tokens) {
  if (h == nullptr || n_pages == nullptr) return BE_ERR_INVALID;
  return guard(const_cast<bh_runner*>(h), [&] {
    const std::vector<int> v = h->r->kv_segment(idx, block, tokens);
    *n_pages = static_cast<int>(v.size());
    for (int i = 0; i < std::min(cap, *n_pages) && slots != nullptr; ++i) slots[i] = v[i];
  });
}
extern "C" be_kv_pool* bh_runner_kv_pool(const bh_runner* h, int block) {
  if (h == nullptr || block < 0 || block >= h->r->n_blocks()) return nullptr;
  return h->r->kv_pool(block);
}
extern "C" int bh_runner_kv_bytes(const bh_runner* h, int64_t* used, int64_t* saved) {
  if (h == nullptr) return BE_ERR_INVALID;
  if (used) *used = h->r->kv_used();
  if (saved) *saved = h->r->kv_saved();
  return BE_OK;
}
extern "C" int bh_runner_live_requests(const bh_runner* h) { return h ? h->r->live() : 0; }
extern "C" int64_t bh_runner_tokens_generated(const bh_runner* h) { return h ? h->r->generated() : 0; }
extern "C" void* bh_runner_arena(bh_runner* h) { return h ? h->r->arena() : nullptr; }
extern "C" int bh_runner_requests(const bh_runner* h) { return h ? h->r->requests() : 0; }
extern "C" void* bh_runner_prefill_arena(bh_runner* h, int64_t* rows) {
  if (h == nullptr) return nullptr;
  if (rows) *rows = h->r->prefill_rows();
  return h->r->prefill_arena();
}
extern "C" int bh_runner_trace(const bh_runner* h, bh_batch_rec* recs, int cap, int* n_out,
                               int32_t* mreq, int32_t* mstep, int32_t* mctx, int mcap, int* m_out) {
  if (h == nullptr || n_out == nullptr) return BE_ERR_INVALID;
  const auto& R = *h->r;
  *n_out = static_cast<int>(R.recs.size());
  if (m_out) *m_out = static_cast<int>(R.m_req.size());
  if (recs != nullptr)
    for (int i = 0; i < std::min(cap, *n_out); ++i) recs[i] = R.recs[i];
  const int nm = std::min<int>(mcap, static_cast<int>(R.m_req.size()));
  for (int i = 0; i < nm; ++i) {
    if (mreq) mreq[i] = R.m_req[i];
    if (mstep) mstep[i] = R.m_step[i];
    if (mctx) mctx[i] = R.m_ctx[i];
  }
  return BE_OK;
}
extern "C" int bh_runner_clear_trace(bh_runner* h) {
  if (h == nullptr) return BE_ERR_INVALID;
  h->r->recs.clear();
  h->r->m_req.clear();
  h->r->m_step.clear();
  h->r->m_ctx.clear();
  return BE_OK;
}
extern "C" int bh_runner_spec_stats(const bh_runner* h, bh_spec_stats* out) {
  if (h == nullptr || out == nullptr) return BE_ERR_INVALID;
  *out = h->r->spec_stats();
  return BE_OK;
}
extern "C" int bh_runner_step_stats(const bh_runner* h, bh_step_stats* out) {
  if (h == nullptr || out == nullptr) return BE_ERR_INVALID;
  *out = h->r->stats;
  return BE_OK;
}
