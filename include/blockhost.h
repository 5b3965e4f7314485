/*
 * blockhost.h — C ABI of the host control plane that forms per-block batches and drives
 * be_exec_batch (include/blockexec.h).
 *
 * Two layers, both mirroring blocksim semantics bit-for-bit where the reference defines them:
 *  - bh_pool_* : block instances and queues — enqueue with the kv-resident priority segment,
 *                greedy prefix pop_batch under a token budget, earliest-head arbitration
 *                (InstancePool, proj/core/src/agent.cpp:132-224).
 *  - bh_kv_*   : block-local paged KV bookkeeping with global page ids and the physical page
 *                slots the GPU page tables hold (KvStore, proj/core/src/kv.cpp:105-237).
 *  - bh_runner_* : the executor loop on one device (Simulation::pump / on_batch_finish /
 *                advance_from, proj/core/src/scenario.cpp:465-669) with the GPU block run in
 *                place of batch_duration_us (scenario.cpp:493).
 * Status codes as in blockexec.h (0 ok, 1 invalid_argument, 2 logic_error, 5 runtime_error).
 */
#ifndef BLOCKHOST_H
#define BLOCKHOST_H

#include <stdint.h>

#include "blockexec.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bh_pool bh_pool;
typedef struct bh_kv bh_kv;
typedef struct bh_runner bh_runner;

/* QueueEntry (proj/core/include/blocksim/agent.hpp:20-30) */
typedef struct {
  int32_t request_id;
  int32_t chain_step;
  int32_t phase; /* BE_PHASE_* */
  int32_t tokens;
  int32_t context_tokens;
  int32_t kv_resident;
  double est_cost_us;
  uint64_t enqueue_seq; /* assigned by enqueue */
} bh_entry;

/* ---- pool ---- */
bh_pool* bh_pool_new(void);
void bh_pool_free(bh_pool* p);
const char* bh_pool_last_error(const bh_pool* p);
int bh_pool_create_instance(bh_pool* p, const char* block_id, int device, int64_t now,
                            int64_t ready_at, char* id_out, int id_cap);
int bh_pool_mark_ready(bh_pool* p, const char* inst, int64_t now);
int bh_pool_enqueue(bh_pool* p, const char* inst, const bh_entry* e);
int bh_pool_pop_batch(bh_pool* p, const char* inst, int max_batch_tokens, int64_t now,
                      bh_entry* out, int cap, int* n_out, int* phase_out);
int bh_pool_finish_batch(bh_pool* p, const char* inst, int64_t now);
/* 1 = found (id written), 0 = none */
int bh_pool_next_runnable(bh_pool* p, int device, int64_t now, char* id_out, int id_cap);
int bh_pool_remove_queued(bh_pool* p, const char* inst, int request_id, bh_entry* out, int cap,
                          int* n_out);
int bh_pool_take_tail(bh_pool* p, const char* inst, int count, bh_entry* out, int cap, int* n_out);
int bh_pool_queue(bh_pool* p, const char* inst, bh_entry* out, int cap, int* n_out,
                  double* queued_cost_us, int* executing);

/* ---- kv ---- */
bh_kv* bh_kv_new(void);
void bh_kv_free(bh_kv* k);
const char* bh_kv_last_error(const bh_kv* k);
int bh_kv_attach_pool(bh_kv* k, const char* pool_key, int device, int n_pages);
int bh_kv_set_capacity(bh_kv* k, int device, int64_t bytes);
int bh_kv_create_segment(bh_kv* k, uint64_t request, const char* block, int device,
                         int64_t bytes_per_token);
int bh_kv_append_tokens(bh_kv* k, uint64_t request, const char* block, int n, int* added);
int bh_kv_share_prefix(bh_kv* k, uint64_t request, uint64_t from, const char* block, int tokens,
                       int* covered);
int bh_kv_release(bh_kv* k, uint64_t request, const char* block);
int bh_kv_release_request(bh_kv* k, uint64_t request);
int bh_kv_move_segment(bh_kv* k, uint64_t request, const char* block, int dst_device);
/* Same, returning the page copies the move implies: (source slot on the old device, slot on
 * dst_device) per page in token order - private pages move, shared ones are copied
 * (KvStore::move_segment, kv.cpp:165-200). Feed them to be_kv_copy_pages. The bookkeeping is
 * updated only if all copies fit in cap. */
int bh_kv_move_segment_slots(bh_kv* k, uint64_t request, const char* block, int dst_device,
                             int32_t* src_slots, int32_t* dst_slots, int cap, int* n_out);
/* query: what = 0 device_of, 1 tokens, 2 pages, 3 shared_pages, 4 segment_bytes, 5 has_segment */
int64_t bh_kv_query(const bh_kv* k, uint64_t request, const char* block, int what);
int64_t bh_kv_bytes_saved(const bh_kv* k);
int64_t bh_kv_used(const bh_kv* k, int device);
int bh_kv_page_ids(const bh_kv* k, uint64_t request, const char* block, uint64_t* out, int cap,
                   int* n_out);
int bh_kv_page_slots(const bh_kv* k, uint64_t request, const char* block, int32_t* out, int cap,
                     int* n_out);

/* ---- runner: the multi-tenant block-chain workload on one device ---- */
typedef struct {
  int n_blocks;
  const be_block_desc* blocks; /* distinct blocks of the zoo; all share d_model */
  int n_tenants;
  const int32_t* chain_ptr;    /* [n_tenants + 1] CSR offsets into chain_blocks */
  const int32_t* chain_blocks; /* block indices, the tenant's chain in order */
  int n_requests;
  const int32_t* req_tenant;   /* [n_requests] */
  const int32_t* req_prompt;   /* [n_requests] prompt tokens */
  const int32_t* req_output;   /* [n_requests] tokens to generate (first token comes from prefill) */
  int max_batch_tokens;        /* pop_batch budget (ScenarioConfig::max_batch_tokens) */
  int mode;                    /* 0 = reference event order (arrivals at t=0, interleaved
                                  prefill/decode); 1 = lockstep (all prefill, then decode) */
  int use_graphs;              /* capture steady-state decode steps in CUDA graphs */
  uint64_t seed;               /* synthetic prompt embeddings: stream "inputs:req<r>" */
  int dry_run;                 /* 1: control plane only (no device work; ctx may be NULL) */
  int plan_ahead;              /* 1: bh_runner_decode_step plans step k+1 on the host while step
                                  k runs on the device (hides host bookkeeping behind the GPU);
                                  the request counters then run one step ahead */
  const int32_t* block_lora_base;     /* NULL, or [n_blocks]: the block whose weights a LoRA
                                         variant shares (-1: a block with its own weights) */
  const char* const* block_lora_name; /* [n_blocks] adapter names of the LoRA variants
                                         (be_lora_load); LoRA variants of one base at a chain
                                         position decode in one launch (be_exec_lora_group_dev) */
  /* speculation (§8 a14; scenario.cpp:502-548, 740-807): blocks marked for speculative
   * execution (e.g. by bh_policy_speculation_marks). In a lockstep decode step, a marked block
   * whose rows all continue to one next block runs as be_exec_speculative: its surrogate (the
   * block with its FFN pruned to the first spec_keep fraction of channels)
   * feeds the next block early on a second stream while the block itself verifies; K7 accepts
   * a row when cos(draft, true) >= spec_threshold, rejected rows re-run the next block. Steps
   * with speculation run without CUDA graphs (the verdict is read back on the host). */
  int n_spec_blocks;
  const int32_t* spec_blocks;
  float spec_threshold; /* 0.95 in the paper */
  float spec_keep;      /* surrogate FFN fraction, e.g. 0.5 */
  /* prefix groups (Request::prefix_group / prefix_tokens, workload.hpp:19-20; NULL = none):
   * requests of a group share the first prefix_tokens prompt tokens (synthetic stream
   * "inputs:prefix<group>"); at each block the first member to finish prefill donates its
   * prefix pages and later members share them (create_kv_for_step, scenario.cpp:671-695). */
  const int32_t* req_prefix_group;
  const int32_t* req_prefix_tokens;
} bh_workload;

typedef struct {
  int32_t instance; /* instance index (creation order, "i<instance+1>") */
  int32_t block;
  int32_t phase;
  int32_t n_members;
  int32_t first_member; /* offset into the member arrays of bh_runner_trace */
} bh_batch_rec;

int bh_runner_create(be_ctx* ctx, const bh_workload* w, bh_runner** out);
int bh_runner_free(bh_runner* r);
const char* bh_runner_last_error(const bh_runner* r);
/* Runs until every request finished prefill (lockstep) or `max_batches` batches ran (mode 0,
 * <= 0 = until all requests complete). */
int bh_runner_run(bh_runner* r, int max_batches);
/* Lockstep decode: one token for every live request (one pass over all chains). host_in /
 * host_out optional pinned or pageable [n_live][d] bf16 rows (request order) copied in before
 * and out after the step; *n_batches receives the batches executed. */
int bh_runner_decode_step(bh_runner* r, const void* host_in, void* host_out, int* n_batches);
/* Lockstep decode of one request group (a pipeline micro-batch): only requests reqs[0..n) step;
 * host_in/host_out rows are the group's live requests in request order. Each group keeps its
 * own CUDA graph. */
int bh_runner_decode_group(bh_runner* r, int group, const int32_t* reqs, int n,
                           const void* host_in, void* host_out, int* n_batches);
/* Live serving (lockstep mode, on a fresh runner): request i arrives arrival_us[i] after the
 * call starts; arrivals are prefilled in arrival order as they come and then board the next
 * lockstep decode iteration (continuous batching at the iteration boundary, the decode-join rule
 * of Simulation::try_join_running, scenario.cpp:432-463). Returns when every request finished;
 * first_token_us[i] / completion_us[i] receive host times (us since the call) taken after the
 * device finished the batch / step producing the token (MetricsCollector's first_token_us /
 * completion_us, metrics.cpp:159-190). */
int bh_runner_serve(bh_runner* r, const int64_t* arrival_us, int64_t* first_token_us,
                    int64_t* completion_us);
int bh_runner_live_requests(const bh_runner* r);
/* KV migration between runners (§8 f rank 1; start_kv_migration, scenario.cpp:361-431):
 * bh_runner_adopt takes over requests mid-decode on a fresh lockstep runner (request idx[k]
 * continues at context ctx[k] with generated[k] tokens out; KV segments of ctx - 1 tokens are
 * created on fresh page slots); bh_runner_kv_segment returns a segment's page slots in token
 * order (and its token count) and bh_runner_kv_pool the block's pool, so the caller moves the
 * pages (be_kv_copy_pages in a process, be_hop_* across) before the next decode step. */
int bh_runner_adopt(bh_runner* r, int n, const int32_t* idx, const int32_t* ctx,
                    const int32_t* generated);
int bh_runner_request_state(const bh_runner* r, int idx, int32_t* ctx, int32_t* generated,
                            int32_t* done);
int bh_runner_kv_segment(const bh_runner* r, int idx, int block, int32_t* slots, int cap,
                         int* n_pages, int* tokens);
be_kv_pool* bh_runner_kv_pool(const bh_runner* r, int block);
/* KV bookkeeping: bytes of pages in use and bytes saved by prefix sharing (KvStore). */
int bh_runner_kv_bytes(const bh_runner* r, int64_t* used, int64_t* saved_by_sharing);
int64_t bh_runner_tokens_generated(const bh_runner* r);
/* Batch trace since creation. members: request ids, steps, context tokens (may be NULL). */
int bh_runner_trace(const bh_runner* r, bh_batch_rec* recs, int cap, int* n_out,
                    int32_t* member_req, int32_t* member_step, int32_t* member_ctx, int mcap,
                    int* m_out);
int bh_runner_clear_trace(bh_runner* r);
/* Device pointer of the decode activation arena ([n_requests][d] bf16, row = request). */
void* bh_runner_arena(bh_runner* r);
int bh_runner_requests(const bh_runner* r); /* n_requests: rows of the decode arena */
/* Device pointer of the prefill arena ([sum of prompts][d] bf16, requests in order) and its
 * row count; a pipeline stage receives its prompts' hidden states here before bh_runner_run. */
void* bh_runner_prefill_arena(bh_runner* r, int64_t* rows);
/* Per-step accounting of the last decode step for roofline reporting. */
typedef struct {
  double weight_bytes;   /* bytes of block weights streamed */
  double kv_bytes;       /* bytes of K/V read by attention */
  double act_bytes;      /* gather + scatter bytes */
  double flops;          /* 2*M*N*K over all GEMMs + 4*ctx*d attention */
  int launches;          /* kernel launches of the step */
  int graph_replayed;    /* 1 when the step ran as a CUDA graph replay */
} bh_step_stats;
int bh_runner_step_stats(const bh_runner* r, bh_step_stats* out);
/* Speculation counters since creation: speculative block runs, rows verified, rows accepted,
 * and the sum / minimum of the K7 cosines. */
typedef struct {
  int64_t runs, rows, accepted;
  double cos_sum, cos_min;
} bh_spec_stats;
int bh_runner_spec_stats(const bh_runner* r, bh_spec_stats* out);

/* ---- executor: the drop-in for Simulation::batch_duration_us (scenario.cpp:493) ----
 * A host that forms batches itself (the reference Simulation) passes each popped ExecBatch to
 * bh_executor_run_batch: the batch's block (loaded on first use from its id and component kinds,
 * 'a' / 'f' per ComponentKind, zoo.hpp:12) runs on the GPU over the members' rows and
 * block-local paged KV (page slots per (request, block) segment). Prefill members update their
 * prompt rows in place; a chain-final prefill member's last prompt row becomes its decode row
 * (the first token); decode members update their decode row in place (position =
 * context_tokens - 1). Synchronous (the caller's event loop continues after the block ran). */
typedef struct bh_executor bh_executor;
typedef struct {
  int d_model, n_heads, d_ff, max_pos;
  int max_batch_tokens;
  float init_scale;
  uint64_t seed; /* weights "weights:<block>:...", prompts "inputs:req<id>" as bh_runner */
} bh_executor_desc;
typedef struct {
  int32_t request_id;     /* QueueEntry::request_id, 1-based */
  int32_t chain_step;
  int32_t tokens;         /* prefill: prompt tokens; decode: 1 */
  int32_t context_tokens; /* QueueEntry::context_tokens */
  int32_t chain_final;    /* 1: the step is the request's last block */
} bh_member;
int bh_executor_create(be_ctx* ctx, const bh_executor_desc* d, int n_requests,
                       const int32_t* req_prompt, const int32_t* req_output, bh_executor** out);
int bh_executor_free(bh_executor* x);
const char* bh_executor_last_error(const bh_executor* x);
int bh_executor_run_batch(bh_executor* x, const char* block_id, const char* components, int phase,
                          int n_members, const bh_member* members);
/* decode = 1: the decode rows [n_requests][d]; 0: the prompt rows; bf16 to host. */
int bh_executor_read_rows(bh_executor* x, int decode, void* host_out);
int bh_executor_stats(const bh_executor* x, int64_t* batches, int64_t* tokens);

/* ---- cluster: the executor loop over several GPUs with block placement (§8 a11 / a15 / e) ----
 * Blocks are placed on ranks (one GPU each); a token step is a fixed list of phases. In phase k
 * every rank steps the runner that holds its rows' k-th leg (a leg = consecutive chain blocks on
 * one device), then the phase's hops move row ranges between runners: be_hop_send / be_hop_recv
 * across processes (NCCL over NVLink), a device copy between runners of this process (the
 * reference's deliver, scenario.cpp:282-308; same-device hops cost nothing there either). The
 * plan is identical on every rank; each process executes the runs and hops touching its own
 * ranks, in plan order, on its context's stream (no host synchronisation inside a step).
 * comm NULL: ranks rank0 .. rank0+n_local-1 all live in this process (e.g. several ranks on one
 * GPU for tests); with a communicator: one local rank, = be_comm_rank(comm). */
typedef struct bh_cluster bh_cluster;
#define BH_ARENA_DECODE 0  /* one row per request (bh_runner_arena) */
#define BH_ARENA_PREFILL 1 /* prompt rows (bh_runner_prefill_arena) */
typedef struct {
  int32_t src_rank, src_runner; /* global rank, runner slot on it */
  int32_t dst_rank, dst_runner;
  int32_t arena;                /* BH_ARENA_* (the same on both sides) */
  int32_t pad_;
  int64_t src_row, dst_row, rows;
} bh_hop;
typedef struct {
  int64_t steps, batches;
  int64_t sent_bytes, recv_bytes; /* NCCL P2P payload of this rank */
  int64_t local_bytes;            /* device copies between runners of this process */
} bh_cluster_stats;
int bh_cluster_create(be_comm* comm, int rank0, int n_local, be_ctx* const* ctxs, int d_model,
                      bh_cluster** out);
int bh_cluster_free(bh_cluster* c);
const char* bh_cluster_last_error(const bh_cluster* c);
int bh_cluster_add_runner(bh_cluster* c, int rank, int slot, bh_runner* r);
/* kind BE_PHASE_PREFILL (runs bh_runner_run) or BE_PHASE_DECODE (bh_runner_decode_step);
 * runs = n_runs (rank, slot) pairs. */
int bh_cluster_add_phase(bh_cluster* c, int kind, int n_runs, const int32_t* runs, int n_hops,
                         const bh_hop* hops);
int bh_cluster_prefill(bh_cluster* c);
/* One token for every request of every rank. host_in / host_out (one local rank only): the
 * home runner's (slot home_slot, first decode phase) rows in before / out after the step. */
int bh_cluster_decode_step(bh_cluster* c, int home_slot, const void* host_in, void* host_out);
int bh_cluster_get_stats(const bh_cluster* c, bh_cluster_stats* out);

#ifdef __cplusplus
}
#endif
#endif /* BLOCKHOST_H */
