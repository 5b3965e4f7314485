/*
 * blockexec.h — C ABI of the B200 per-block batched execution path (BlockLLM, arXiv 2404.18322).
 *
 * The reference (blocksim, /root/reference/proj/core) has no GPU and no FFI: "running a block"
 * is Simulation::batch_duration_us(const Instance&, const ExecBatch&) -> double µs
 * (proj/core/include/blocksim/scenario.hpp:94, called only from pump, src/scenario.cpp:493),
 * a cost-table lookup (CostModel::block_us, src/costmodel.cpp:96-105). This header is the seam a
 * maintainer drops in at that call site: the host keeps its Instance/ExecBatch/KvStore state and
 * hands the batch to be_exec_batch, which gathers the members' activation rows, runs the block's
 * decoder layers on the GPU and scatters the outputs to their next-hop rows.
 *
 * Conventions: plain C types, device pointers where marked d_*, int status codes (BE_OK = 0),
 * never throws; be_last_error() describes the last failure of a context. One host thread per
 * context (the reference Engine is single-threaded). Work is asynchronous on the
 * stream passed in (NULL = the context's stream).
 */
#ifndef BLOCKEXEC_H
#define BLOCKEXEC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  BE_OK = 0,
  BE_ERR_INVALID = 1,  /* bad argument: std::invalid_argument in the reference */
  BE_ERR_STATE = 2,    /* misuse of an object: std::logic_error in the reference */
  BE_ERR_CUDA = 3,     /* CUDA runtime/driver failure */
  BE_ERR_NOMEM = 4,    /* device allocation failed (MemoryLedger over capacity) */
  BE_ERR_RUNTIME = 5   /* std::runtime_error class ("run: ...") */
};

enum { BE_PHASE_PREFILL = 0, BE_PHASE_DECODE = 1 }; /* blocksim::Phase, costmodel.hpp:12 */

typedef struct be_ctx be_ctx;
typedef struct be_block be_block;
typedef struct be_kv_pool be_kv_pool;
typedef struct be_workspace be_workspace;

/* A block = a contiguous run of Llama decoder layers (attention + ffn components of the zoo,
 * zoo.hpp:29-54). Weights are synthetic (random init), generated on the device from
 * (seed, name) by the counter-mode generator of oracle/synth.h. */
typedef struct {
  int n_layers;
  int d_model;     /* embed_dim_in == embed_dim_out */
  int n_heads;
  int head_dim;
  int d_ff;
  int max_pos;     /* RoPE table length */
  float norm_eps;
  float rope_theta;
  float init_scale; /* weights uniform in [-s, s] */
  uint64_t seed;
  const char* name; /* stream prefix, e.g. "b0" */
  /* Component sequence of the block, one char per zoo component (ComponentKind, zoo.hpp:12):
   * 'a' attention (RMSNorm, QKV, RoPE, paged attention, O, residual), 'f' ffn (RMSNorm, SwiGLU
   * MLP, residual). NULL = n_layers decoder layers "afaf...". Blocks split by the zoo's
   * partitioner may start or end mid-layer ("fa", "a", "f"). */
  const char* components;
  /* Structured-pruned surrogate: when > d_ff, this block's FFN is the first
   * d_ff channels of the FFN of a block with ffn_src channels and the same (seed, name) - the
   * draft model of speculation (be_exec_speculative). 0 = d_ff. */
  int ffn_src;
} be_block_desc;

/* One token row of an execution batch (decode: one per request; prefill: one per prompt token). */
typedef struct {
  int32_t src_row;   /* activation-arena row holding this token's block input */
  int32_t dst_row;   /* arena row receiving this token's block output (-1: not stored) */
  int32_t kv_slot;   /* physical KV token slot = page_slot * 16 + pos % 16 */
  int32_t pos;       /* absolute position in its sequence (RoPE, causal extent) */
  int32_t pt_row;    /* row of the page table naming this token's segment pages */
} be_token;

/* Context / device ------------------------------------------------------------------------ */
int be_ctx_create(int device, be_ctx** out);
int be_ctx_destroy(be_ctx* ctx);
const char* be_last_error(const be_ctx* ctx);
int be_ctx_num_sms(const be_ctx* ctx);
void* be_ctx_stream(be_ctx* ctx); /* cudaStream_t */
int be_synchronize(be_ctx* ctx);

/* Blocks (weights) ------------------------------------------------------------------------- */
int be_block_load(be_ctx* ctx, const be_block_desc* desc, be_block** out);
int be_block_free(be_block* blk);
int64_t be_block_param_bytes(const be_block* blk);
/* bytes of K+V per token for the whole block: sum over its attention layers of 4*d
 * (CostModel::kv_bytes_per_token, costmodel.cpp:114-127) */
int64_t be_block_kv_bytes_per_token(const be_block* blk);

/* Block-local paged KV pool: n_pages pages of 16 tokens (kv.hpp:16) x all layers ------------ */
int be_kv_pool_create(be_ctx* ctx, const be_block* blk, int n_pages, be_kv_pool** out);
int be_kv_pool_free(be_kv_pool* pool);
void* be_kv_pool_data(be_kv_pool* pool); /* device base pointer: [page][layer][K|V][head][16][hd] */
int64_t be_kv_pool_page_bytes(const be_kv_pool* pool);
/* Synchronous copy of pool bytes [offset, offset+bytes) to host memory (tests / migration). */
int be_kv_pool_read(be_kv_pool* pool, int64_t offset, int64_t bytes, void* host_dst);

/* Scratch for one executing batch (sized for max_tokens tokens) ----------------------------- */
int be_workspace_create(be_ctx* ctx, int d_model, int d_ff, int n_heads, int max_tokens,
                        int max_rows, int max_pages_per_row, be_workspace** out);
int be_workspace_free(be_workspace* ws);

/* Execute one batch of one block instance (replaces Simulation::batch_duration_us).
 * tokens: host array of n_tokens be_token; page_table: host [n_pt_rows][pt_stride] int32 of
 * physical page slots; d_arena_in/out: device bf16 [rows][d_model] activation arenas (may alias).
 * The metadata is staged into the workspace and uploaded on `stream`. */
int be_exec_batch(be_ctx* ctx, be_block* blk, be_kv_pool* pool, be_workspace* ws, int phase,
                  int n_tokens, const be_token* tokens, int n_pt_rows, int pt_stride,
                  const int32_t* page_table, const void* d_arena_in, void* d_arena_out,
                  void* stream);

/* Same, with all metadata already on the device (CUDA-graph friendly: no host work besides
 * launches). d_tokens: device be_token[n_tokens]; d_page_table: device int32. */
int be_exec_batch_dev(be_ctx* ctx, be_block* blk, be_kv_pool* pool, be_workspace* ws, int phase,
                      int n_tokens, const be_token* d_tokens, int pt_stride,
                      const int32_t* d_page_table, const void* d_arena_in, void* d_arena_out,
                      void* stream);

/* One speculative decode step (§8 a14, K6 + K7). The draft block (a surrogate of verify->blk,
 * e.g. its 50%-pruned FFN, be_block_desc.ffn_src) runs on a second stream and
 * its output is forwarded at once to next->blk - the early forward of scenario.cpp:521-537 -
 * while verify->blk computes the true output on the context stream. K7 then compares the
 * draft and true rows (cos >= threshold accepts; PAPER.md:637 uses 0.95, the reference's
 * stand-in is a Bernoulli verdict, config.hpp:60) and `next` is re-run from the true rows for
 * the rejected ones (finish_verified, scenario.cpp:740-807), overwriting their KV slots.
 * d_x_in / d_y_draft / d_y_true / d_z_out: device bf16 [n_tokens][d] rows; each stage's host
 * token records index them (src_row/dst_row). verify->ws must differ from draft/next's (the
 * two lanes run concurrently). cos_out / accept_out: host [n_tokens]. Synchronous. */
typedef struct {
  be_block* blk;
  be_kv_pool* pool;
  be_workspace* ws;
  const be_token* tokens; /* host, n_tokens */
  int n_pt_rows, pt_stride;
  const int32_t* page_table; /* host */
} be_spec_stage;
int be_exec_speculative(be_ctx* ctx, const be_spec_stage* verify, const be_spec_stage* draft,
                        const be_spec_stage* next, int n_tokens, const void* d_x_in,
                        void* d_y_draft, void* d_y_true, void* d_z_out, float threshold,
                        float* cos_out, int32_t* accept_out, int* n_accepted);

/* A grouped batch: n_blocks independent batches of blocks with identical shape and component
 * sequence (e.g. the tenants' private blocks at one chain position, which share no request)
 * executed as one batch - one launch per kernel instead of n_blocks. Token rows
 * [g*R, (g+1)*R) (R = n_tokens / n_blocks, one of 16/32/64) belong to blks[g] / pools[g]; a
 * group with fewer members is padded with rows {src 0, dst -1, kv_slot -1, pos -1} (computed,
 * never stored). Each batch's semantics are unchanged (its own weights, KV pool, page rows). */
int be_exec_group_dev(be_ctx* ctx, int n_blocks, be_block* const* blks, be_kv_pool* const* pools,
                      be_workspace* ws, int phase, int n_tokens, const be_token* d_tokens,
                      int pt_stride, const int32_t* d_page_table, const void* d_arena_in,
                      void* d_arena_out, void* stream);

/* Kernel launches one be_exec_batch of n_tokens performs (for launch accounting). */
int be_exec_batch_launches(be_ctx* ctx, const be_block* blk, int n_tokens, int pt_stride);

/* Per-launch timing of exec_batch kernels: while enabled, every launch is bracketed by CUDA
 * events on its stream (graph replay is bypassed by the runner). be_prof_read synchronises the
 * context stream and returns (and clears) the records; with cap < n only *n_out is written. */
enum {
  BE_K_GATHER = 0,
  BE_K_RMS = 1, /* reserved: the RMSNorm statistics are fused into gather / residual epilogues */
  BE_K_GEMM_QKV = 2,
  BE_K_ATTENTION = 3, /* decode/prefill attention (+ split combine); n = heads, k = head_dim */
  BE_K_GEMM_O = 4,
  BE_K_GEMM_GATE_UP = 5,
  BE_K_GEMM_DOWN = 6,
  BE_K_SCATTER = 7
};
typedef struct {
  int32_t cls;  /* BE_K_* */
  int32_t ntok; /* rows of the batch */
  int32_t n;    /* GEMM output features (rows of W), d_model for row kernels */
  int32_t k;    /* GEMM reduction dim */
  float ms;     /* event-timed duration */
  double bytes; /* algorithmic bytes (GEMM: 2(NK + MK + MN) per GEMM); 0 = caller computes */
  double flops; /* algorithmic flops (2 MNK per GEMM) */
} be_prof_rec;
int be_prof_enable(be_ctx* ctx, int on);
int be_prof_active(const be_ctx* ctx);
int be_prof_read(be_ctx* ctx, be_prof_rec* out, int cap, int* n_out);

/* Kernel timeline inside graph replays (PDL overlap included): while enabled (cap slots), every
 * exec_batch kernel records globaltimer ns of its first/last CTA start, first dependency release
 * (griddepcontrol.wait return) and last CTA end into its slot. be_timeline_begin resets the
 * window and restarts slot numbering at the next launch (graphs captured in a window keep their
 * slots); be_timeline_read synchronises and returns the written slots in slot order. */
typedef struct {
  int32_t slot;
  int32_t cls; /* BE_K_* */
  uint64_t start_first, start_last, go_first, end_last;
} be_timeline_rec;
int be_timeline_enable(be_ctx* ctx, int cap);
int be_timeline_begin(be_ctx* ctx);
int be_timeline_read(be_ctx* ctx, be_timeline_rec* out, int cap, int* n_out);

/* KV migration data path (§8 f: the P2P page copy of start_kv_migration, scenario.cpp:361-431):
 * copies whole pages src_slots[i] of src_pool to dst_slots[i] of dst_pool (host arrays) on the
 * destination context's stream; contiguous slot runs move as one copy. The pools may live on
 * different GPUs (peer copy over NVLink; peer access is enabled on first use). Async; the copy
 * is ordered after all work queued so far on the source context's stream. The source slots must
 * not be rewritten (e.g. reallocated after bh_kv_move_segment_slots freed them) before the copy
 * has executed: order such writes after `stream` (or synchronize it). */
int be_kv_copy_pages(be_ctx* dst_ctx, const be_kv_pool* src_pool, be_kv_pool* dst_pool,
                     const int32_t* src_slots, const int32_t* dst_slots, int n, void* stream);

/* LoRA adapters on a block's attention components (multi-tenant adapter
 * deltas by segmented GEMM). A fused-attention LoRA variant (the reference's attach "fuse",
 * gen_configs.py lora_components; its own block in the zoo, with the base weights as shared
 * content) runs as the BASE block plus a rank-16 delta per attention projection:
 * W'_x = W_x + B_x A_x for x in q, k, v, o. Synthetic factors: stream "lora:<name>:<l>:<t>"
 * (t in aq ak av ao: [16][d], scale_a; bq bk bv bo: [d][16], scale_b), splitmix counter mode as
 * the weights. One launch serves tokens of up to BE_MAX_LORA adapters (lora_idx per token, -1 =
 * the base block): the base GEMM streams the shared weights once, a shrink kernel forms
 * u = A x per token and the GEMM epilogue adds B u before RoPE / the residual add. */
#define BE_LORA_RANK 16
#define BE_MAX_LORA 8
typedef struct be_lora be_lora;
int be_lora_load(be_ctx* ctx, const be_block* base, const char* name, uint64_t seed,
                 float scale_a, float scale_b, be_lora** out);
int be_lora_free(be_lora* lora);
/* be_exec_batch with adapters: lora_idx (host, n_tokens) picks loras[idx] per token. */
int be_exec_lora_batch(be_ctx* ctx, be_block* blk, be_kv_pool* pool, be_workspace* ws, int phase,
                       int n_tokens, const be_token* tokens, int n_pt_rows, int pt_stride,
                       const int32_t* page_table, int n_lora, const be_lora* const* loras,
                       const int32_t* lora_idx, const void* d_arena_in, void* d_arena_out,
                       void* stream);
/* LoRA variants of ONE base block at a chain position in one launch: group g's rows (n_tokens /
 * n_blocks, padded as be_exec_group_dev) keep their own KV pool pools[g]; blks[g] must all be
 * the base block (its weights stream once for every row); d_lora_idx picks each row's adapter. */
int be_exec_lora_group_dev(be_ctx* ctx, int n_blocks, be_block* const* blks,
                           be_kv_pool* const* pools, be_workspace* ws, int phase, int n_tokens,
                           const be_token* d_tokens, int pt_stride, const int32_t* d_page_table,
                           int n_lora, const be_lora* const* loras, const int32_t* d_lora_idx,
                           const void* d_arena_in, void* d_arena_out, void* stream);
/* Same with every per-token array already on the device (graph-capturable). */
int be_exec_lora_batch_dev(be_ctx* ctx, be_block* blk, be_kv_pool* pool, be_workspace* ws,
                           int phase, int n_tokens, const be_token* d_tokens, int pt_stride,
                           const int32_t* d_page_table, int n_lora, const be_lora* const* loras,
                           const int32_t* d_lora_idx, const void* d_arena_in, void* d_arena_out,
                           void* stream);

/* Stitches: the linear map that lets a chain step of width dim_in enter an
 * equivalent block of width dim_out (Zoo::candidate_instances, zoo.cpp:568-589; its cost is
 * CostModel::stitch_us). y = x W^T with W [dim_out][dim_in] synthetic from stream
 * "stitch:<name>" (scale as block weights); rows are bf16 [rows][dim]. dim_in % 64 == 0,
 * dim_out % 128 == 0. */
typedef struct be_stitch be_stitch;
int be_stitch_load(be_ctx* ctx, int dim_in, int dim_out, const char* name, uint64_t seed,
                   float scale, be_stitch** out);
int be_stitch_free(be_stitch* s);
int be_stitch_rows(be_ctx* ctx, const be_stitch* s, const void* d_in, int rows, void* d_out,
                   void* stream);

/* KV migration with overlapped recompute / copy (the plan is
 * plan_migration, kv.cpp:16-58, bh_plan_migration; the move is start_kv_migration,
 * scenario.cpp:361-431). A segment's n_pages pages (src_slots -> dst_slots, token order, from
 * bh_kv_move_segment_slots) move to dst_pool: the first n_recompute pages are rebuilt on the
 * destination by a chunked prefill of `blk` over the head tokens' block-input rows
 * (d_head_rows, head_tokens rows, (n_recompute-1)*16 < head_tokens <= n_recompute*16, and
 * head_tokens == n_recompute*16 when tail pages are copied, so no token is left out), while the
 * other pages are copied from src_pool (peer GPU over NVLink, or the same GPU) on a side stream;
 * the call's stream waits for both. `blk`, dst_pool and ws belong to ctx. Async. */
int be_kv_migrate(be_ctx* ctx, be_block* blk, const be_kv_pool* src_pool, be_kv_pool* dst_pool,
                  be_workspace* ws, const int32_t* src_slots, const int32_t* dst_slots,
                  int n_pages, int n_recompute, int head_tokens, const void* d_head_rows,
                  void* stream);

/* K1 / K2 standalone: routing-table gather and scatter of bf16 rows. */
int be_gather_rows(be_ctx* ctx, const void* d_arena, const int32_t* d_src, int rows, int d,
                   void* d_out, void* stream);
int be_scatter_rows(be_ctx* ctx, const void* d_rows, const int32_t* d_dst, int rows, int d,
                    void* d_arena, void* stream);

/* K7: per-row cosine(pred, actual) in fp32 and accept = cos >= threshold (PAPER.md:637 uses
 * 0.95); the reference's scalar definition is signature_similarity, zoo.cpp:78-88. */
int be_cosine(be_ctx* ctx, const void* d_pred, const void* d_actual, int rows, int d,
              float threshold, float* d_cos, int32_t* d_accept, void* stream);

/* Synthetic data: counter-mode generator shared with oracle/synth.h. */
int be_synth_rows(be_ctx* ctx, void* d_dst, int64_t n_elems, uint64_t seed, const char* stream_id,
                  float scale, void* stream);
/* Copies one weight tensor of a block back in its LOGICAL layout (rows x cols, fp32 host array).
 * tensor: "wq","wk","wv","wo","wg","wu","wd". For parity tests. */
int be_block_read_weight(be_block* blk, int layer, const char* tensor, float* host_out);

/* Low-level kernels exported for tests and the roofline bench ------------------------------ */
/* Row-major [N][K] bf16 -> the packed GEMM weight layout (128x64 tiles, tile-major, each tile in
 * its 128B-swizzled shared-memory image; see csrc/ptx.cuh packed_index). Block weights are
 * generated directly in this layout. */
int be_pack_weight(be_ctx* ctx, const void* d_src, void* d_dst, int N, int K, void* stream);
/* out[t][f] = bf16(sum_k W[f][k] X[t][k]) with W packed (be_pack_weight), X [ntok][K] bf16
 * row-major. grid_cap bounds the persistent CTAs (0 = one per SM). */
int be_gemm_bf16(be_ctx* ctx, const void* d_w_packed, const void* d_x, void* d_out, int N, int K,
                 int ntok, int grid_cap, void* stream);
/* Roofline timing: device microseconds per GEMM launch from one CUDA-graph replay of `reps`
 * launches cycling over n_w packed weight copies. */
int be_bench_gemm(be_ctx* ctx, const void* const* d_w_packed, int n_w, const void* d_x,
                  void* d_out, int N, int K, int ntok, int reps, float* us_per_launch);
/* Paged attention over a pool (decode rows / causal prefill rows). */
int be_attention(be_ctx* ctx, const void* d_q, const void* d_pool, int n_layers, int n_heads,
                 int head_dim, int layer, const int32_t* d_page_table, int pt_stride,
                 const int32_t* d_row_pt, const int32_t* d_row_ctx, int rows, int splits,
                 void* d_out, void* stream);

/* ---- inter-block hop (§8 a11; replaces LinkManager::transfer, proj/core/src/cluster.cpp:170-192,
 * at the Simulation::deliver call, proj/core/src/scenario.cpp:282-308): the bf16 rows of a chain
 * crossing GPUs move by NCCL point-to-point over NVLink. One communicator per process (one
 * process per GPU, `rank` = its global rank); every rank passes the same unique id (made by
 * be_comm_unique_id on one rank and broadcast by the caller). The sends/recvs of one executor
 * phase go between be_hop_begin / be_hop_end (one NCCL group: no ordering deadlock between
 * peers) and are enqueued on `stream` (NULL = the context's stream) after the work that
 * produced the rows. Async; bytes are counted per communicator (be_comm_bytes). */
typedef struct be_comm be_comm;
#define BE_COMM_ID_BYTES 128
int be_comm_unique_id(void* id_out);
int be_comm_init(be_ctx* ctx, int n_ranks, int rank, const void* id, be_comm** out);
int be_comm_destroy(be_comm* comm);
const char* be_comm_last_error(const be_comm* comm);
int be_comm_rank(const be_comm* comm);
int be_comm_size(const be_comm* comm);
int64_t be_comm_bytes(const be_comm* comm, int sent);
int be_hop_begin(be_comm* comm);
int be_hop_send(be_comm* comm, int peer, const void* d_rows, int64_t bytes, void* stream);
int be_hop_recv(be_comm* comm, int peer, void* d_rows, int64_t bytes, void* stream);
int be_hop_end(be_comm* comm);

#ifdef __cplusplus
}
#endif
#endif /* BLOCKEXEC_H */
