/* C ABI of the routing / speculation-marking / placement policy.
 *
 * The reference makes these decisions in blocksim's Scheduler (proj/core/include/blocksim/
 * scheduler.hpp:62-118, src/scheduler.cpp); this library makes the same decisions, with the same
 * arithmetic and tie-breaks, over a snapshot of the serving state the host maintains
 * (paper_2404_18322_b200/csrc/host/policy.{hpp,cpp}):
 *
 *   bh_policy_choose_binding     Scheduler::choose_binding   scheduler.cpp:80-160
 *   bh_policy_estimate           Scheduler::estimate         scheduler.cpp:23-78
 *   bh_policy_speculation_marks  Scheduler::speculation_marks scheduler.cpp:180-215
 *   bh_policy_scale_decisions    Scheduler::scale_decisions  scheduler.cpp:227-260
 *   bh_policy_choose_device      Scheduler::choose_device    scheduler.cpp:262-314
 *   bh_policy_placement_moves    Scheduler::placement_moves  scheduler.cpp:321-366
 *   bh_policy_migration_rates    Scheduler::migration_rates  scheduler.cpp:368-381
 *   bh_plan_migration            plan_migration              kv.cpp:16-58
 *   bh_policy_kv_review          Simulation::kv_review       scenario.cpp:844-900
 *
 * Ids are NUL-terminated strings (the reference's instance / block / model ids). List outputs
 * are written as '\n'-separated ids into a caller buffer. Every call returns a be_status code
 * (include/blockexec.h): BE_ERR_INVALID for std::invalid_argument in the reference. */
#ifndef BLOCKPOLICY_H
#define BLOCKPOLICY_H

#include <stdint.h>

#include "blockexec.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bh_policy bh_policy;

/* ScenarioConfig knobs the decisions read (config.hpp:33-69) + SurrogateRules (costmodel.hpp:39-48) */
typedef struct {
  int adaptive;          /* candidates include equivalents */
  int least_busy;        /* score = queue only; no stick-to-cache */
  int frag_min;          /* placement policy: 0 locality, 1 tightest fit */
  int speculation;
  double spec_fraction;
  int64_t scale_queue_us;
  int expected_tokens;
  double sur_attention_only, sur_ffn_only, sur_one_layer, sur_multi_layer;
  int sur_allow_adapter_blocks;
} bh_policy_config;

/* Interp2D (costmodel.hpp): v row-major [nx][ny] */
typedef struct {
  const double* xs;
  int nx;
  const double* ys;
  int ny;
  const double* v;
} bh_grid;

typedef struct {
  const char* id;
  const char* block_id;
  int device;
  int ready;             /* InstanceState::kReady (else kLoading) */
  int64_t ready_at;
  int64_t last_used;
  uint64_t created_seq;
  int executing;
  int queue_len;
  double queued_cost_us;
  double queued_cost_hwm;
} bh_policy_instance;

typedef struct {               /* BindingQuery (scheduler.hpp) */
  uint64_t request_id;
  const char* chain_block;
  int phase;                   /* BE_PHASE_PREFILL / BE_PHASE_DECODE */
  int tokens;
  int context_tokens;
  int from_device;             /* -1 at chain entry */
  int64_t now;
} bh_binding_query;

typedef struct {               /* BindingChoice (scheduler.hpp) */
  char block_id[96];
  char stitch_class[96];
  char instance_id[32];        /* "" -> create a new instance on `device` */
  int device;
  int adaptive;
  int64_t evict_bytes;
  double queue_us, compute_us, transfer_us, load_us;
} bh_binding_choice;

enum { BH_PREF_LOCALITY = 0, BH_PREF_TIGHTEST_FIT = 1, BH_PREF_MOST_FREE = 2 };
/* ComponentKind order (zoo.hpp:12) */
enum { BH_KIND_ATTENTION = 0, BH_KIND_FFN = 1, BH_KIND_EMBEDDING = 2, BH_KIND_LM_HEAD = 3,
       BH_KIND_ADAPTER = 4 };

bh_policy* bh_policy_new(const bh_policy_config* cfg);
void bh_policy_free(bh_policy* p);
const char* bh_policy_last_error(const bh_policy* p);

/* static description: cost model, zoo structure, cluster */
int bh_policy_add_cost_class(bh_policy* p, const char* key, const bh_grid* prefill,
                             const bh_grid* decode, int64_t kv_bytes_per_token /* -1: derive */);
int bh_policy_add_stitch_class(bh_policy* p, const char* key, const bh_grid* g);
int bh_policy_set_device_class(bh_policy* p, const char* name, double speed_factor);
int bh_policy_add_component(bh_policy* p, const char* id, int kind, int embed_dim, int layer,
                            int n_pieces, const char* const* piece_ids, const int64_t* piece_bytes);
int bh_policy_add_block(bh_policy* p, const char* id, int n_comps, const char* const* comp_ids,
                        int embed_dim_out);
int bh_policy_add_chain(bh_policy* p, const char* model_id, int n, const char* const* blocks);
int bh_policy_add_candidate(bh_policy* p, const char* block, const char* candidate,
                            const char* stitch_class /* "" when dims match */, double score);
int bh_policy_add_server(bh_policy* p, int id, double intra_bps);
int bh_policy_set_inter_bandwidth(bh_policy* p, int server_a, int server_b, double bps);
int bh_policy_set_inter_default(bh_policy* p, double bps);
int bh_policy_add_device(bh_policy* p, int id, int server, const char* device_class,
                         int64_t capacity, double mem_bps, double load_bps);

/* dynamic state */
int bh_policy_clear_state(bh_policy* p);
int bh_policy_put_instance(bh_policy* p, const bh_policy_instance* inst);
int bh_policy_remove_instance(bh_policy* p, const char* id);
int bh_policy_set_ledger(bh_policy* p, int device, int64_t params, int64_t kv, int64_t act);
int bh_policy_set_lane(bh_policy* p, int device, int64_t busy_until);
int bh_policy_set_kv(bh_policy* p, uint64_t request, const char* block, int owner, int pages);
int bh_policy_set_adjacency(bh_policy* p, const char* from, const char* to, int64_t count);
int bh_policy_note_adjacency(bh_policy* p, const char* from, const char* to);

/* decisions */
int bh_policy_choose_binding(bh_policy* p, const bh_binding_query* q, bh_binding_choice* out,
                             int* found);
int bh_policy_estimate(bh_policy* p, const bh_binding_query* q, const char* block,
                       const char* stitch_class, const char* instance_id /* NULL: new */,
                       int device, double* out4 /* queue, compute, transfer, load */,
                       int64_t* evict_bytes);
int bh_policy_speculation_marks(bh_policy* p, char* ids, int cap, int* n_out);
int bh_policy_scale_decisions(bh_policy* p, char* ids, int cap, int* devices, int dev_cap,
                              int* n_out);
int bh_policy_choose_device(bh_policy* p, const char* block, int pref, const int* exclude,
                            int n_exclude, int* device_out);
int bh_policy_placement_moves(bh_policy* p, char* ids, int cap, int* devices, int dev_cap,
                              int* n_out);
int bh_policy_migration_rates(bh_policy* p, const char* block, int src, int dst,
                              int64_t* rec_us_per_page, int64_t* cp_us_per_page);
int bh_policy_param_bytes_needed(bh_policy* p, const char* block, int device, int64_t* out);

/* Proactive KV review (Simulation::kv_review, scenario.cpp:844-900): the interception tracker
 * (InterceptionTracker, kv.cpp:70-103) and the queued decode entries whose cache is remote;
 * order_out receives indices into q of the entries to migrate now, in order_migrations order
 * (kv.cpp:60-68). */
typedef struct {
  const char* instance;     /* the instance holding the queued entry */
  const char* inst_block;   /* its serving block */
  int device;               /* its device */
  uint64_t request_id;
  const char* chain_block;  /* the request chain's block at the entry's step */
  int owner;                /* device of the (request, chain block) cache segment, -1 none */
  int pages, shared_pages;
  int pending;              /* an interception sample is open for this step */
  const char* pending_key;
  int64_t t_call;
} bh_queued_decode;

int bh_policy_interception_record(bh_policy* p, const char* key, int64_t sample);
/* key NULL: the global accumulator */
int bh_policy_interception_set(bh_policy* p, const char* key, double sum, uint64_t n);
int bh_policy_interception_predict(bh_policy* p, const char* key, int64_t t_call, int64_t now,
                                   int64_t* out, int* found);
int bh_policy_kv_review(bh_policy* p, const bh_queued_decode* q, int n, int64_t now,
                        int recalc_only, int* order_out, int cap, int* n_out);

/* out6 = pages, recompute_pages, copy_pages, completion_us, rec_us_per_page, cp_us_per_page */
int bh_plan_migration(int pages, int64_t rec_us_per_page, int64_t cp_us_per_page, int64_t* out6);

#ifdef __cplusplus
}
#endif
#endif
