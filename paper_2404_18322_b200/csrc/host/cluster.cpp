// The multi-GPU executor loop with block placement (SURVEY §8 a11 / a15 / e).
//
// The unit of placement is a block instance on a device (Instance, agent.hpp:44-56); a chain
// that crosses devices has one activation hop per crossing (Simulation::deliver,
// scenario.cpp:282-308). Here each rank (one GPU) runs single-device executor loops (bh_runner)
// over the blocks it holds, and a token step is a fixed sequence of phases:
//
//   phase k: every rank steps the runner holding its requests' k-th leg (a leg = consecutive
//            chain blocks on one device), then the rows whose chain continues elsewhere hop to
//            the runner of their next leg (NCCL send/recv across GPUs, a device copy between
//            runners of one process), the last leg's rows back to the request's home runner.
//
// The plan (which runner holds which blocks and rows, which row ranges hop where) is made by the
// caller from the placement (paper_2404_18322_b200/cluster.py); it is the same on every rank, and
// each process executes the runs and hops that touch its own ranks. All work of a rank is
// enqueued on its context's stream in phase order, so a hop waits for the block that produced
// its rows and the next leg waits for the hop, with no host synchronisation inside a step.
#include <cuda_runtime.h>

#include <cstdio>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/blockhost.h"

struct bh_cluster {
  be_comm* comm = nullptr;  // null: every rank of the plan lives in this process
  int rank0 = 0;
  std::vector<be_ctx*> ctxs;  // local ranks rank0 .. rank0 + n_local - 1
  int row_bytes = 0;
  std::map<std::pair<int, int>, bh_runner*> runners;  // (rank, slot) -> runner
  struct Phase {
    int kind = BE_PHASE_DECODE;
    std::vector<std::pair<int, int>> runs;
    std::vector<bh_hop> hops;
  };
  std::vector<Phase> phases;
  std::vector<cudaEvent_t> evs;  // per local rank: cross-context copies wait on the source
  bh_cluster_stats stats{};
  std::string err;

  bool local(int rank) const { return rank >= rank0 && rank < rank0 + (int)ctxs.size(); }
  be_ctx* ctx_of(int rank) const { return ctxs[rank - rank0]; }
  cudaStream_t stream_of(int rank) const {
    return static_cast<cudaStream_t>(be_ctx_stream(ctx_of(rank)));
  }
};

namespace {
struct ClusterError : std::runtime_error {
  int code;
  ClusterError(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw ClusterError(BE_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guard(bh_cluster* c, F&& f) {
  try {
    f();
    return BE_OK;
  } catch (const ClusterError& e) {
    if (c) c->err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    if (c) c->err = e.what();
    return BE_ERR_RUNTIME;
  }
}

bh_runner* runner_at(bh_cluster* c, int rank, int slot) {
  auto it = c->runners.find({rank, slot});
  if (it == c->runners.end())
    throw ClusterError(BE_ERR_STATE, "no runner at rank " + std::to_string(rank) + " slot " +
                                         std::to_string(slot));
  return it->second;
}

char* rows_of(bh_cluster* c, int rank, int slot, int arena, int64_t row, int64_t rows) {
  bh_runner* r = runner_at(c, rank, slot);
  char* base;
  int64_t cap;
  if (arena == BH_ARENA_PREFILL) {
    base = static_cast<char*>(bh_runner_prefill_arena(r, &cap));
  } else {
    base = static_cast<char*>(bh_runner_arena(r));
    cap = bh_runner_requests(r);
  }
  if (base == nullptr || row < 0 || rows < 0 || row + rows > cap)
    throw ClusterError(BE_ERR_INVALID, "hop rows out of the runner's arena");
  return base + row * c->row_bytes;
}

// one phase's hops: device copies between local runners, NCCL for the rest (one group)
void do_hops(bh_cluster* c, const bh_cluster::Phase& ph) {
  const bool any_remote = [&] {
    for (const auto& h : ph.hops)
      if (c->local(h.src_rank) != c->local(h.dst_rank)) return true;
    return false;
  }();
  if (any_remote) {
    if (c->comm == nullptr) throw ClusterError(BE_ERR_STATE, "remote hop without a communicator");
    if (be_hop_begin(c->comm) != BE_OK) throw ClusterError(BE_ERR_RUNTIME, be_comm_last_error(c->comm));
  }
  for (const auto& h : ph.hops) {
    const bool sl = c->local(h.src_rank), dl = c->local(h.dst_rank);
    if (!sl && !dl) continue;
    const int64_t bytes = h.rows * c->row_bytes;
    if (sl && dl) {
      const char* src = rows_of(c, h.src_rank, h.src_runner, h.arena, h.src_row, h.rows);
      char* dst = rows_of(c, h.dst_rank, h.dst_runner, h.arena, h.dst_row, h.rows);
      cudaStream_t st = c->stream_of(h.dst_rank);
      if (c->ctx_of(h.src_rank) != c->ctx_of(h.dst_rank)) {
        cudaEvent_t ev = c->evs[h.src_rank - c->rank0];
        ck(cudaEventRecord(ev, c->stream_of(h.src_rank)), "hop event");
        ck(cudaStreamWaitEvent(st, ev, 0), "hop wait");
      }
      ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st), "hop copy");
      c->stats.local_bytes += bytes;
    } else if (sl) {
      const char* src = rows_of(c, h.src_rank, h.src_runner, h.arena, h.src_row, h.rows);
      if (be_hop_send(c->comm, h.dst_rank, src, bytes, c->stream_of(h.src_rank)) != BE_OK)
        throw ClusterError(BE_ERR_RUNTIME, be_comm_last_error(c->comm));
      c->stats.sent_bytes += bytes;
    } else {
      char* dst = rows_of(c, h.dst_rank, h.dst_runner, h.arena, h.dst_row, h.rows);
      if (be_hop_recv(c->comm, h.src_rank, dst, bytes, c->stream_of(h.dst_rank)) != BE_OK)
        throw ClusterError(BE_ERR_RUNTIME, be_comm_last_error(c->comm));
      c->stats.recv_bytes += bytes;
    }
  }
  if (any_remote && be_hop_end(c->comm) != BE_OK)
    throw ClusterError(BE_ERR_RUNTIME, be_comm_last_error(c->comm));
}

void run_phases(bh_cluster* c, int kind, const void* host_in, void* host_out, int home_slot) {
  bool first = true;
  for (const auto& ph : c->phases) {
    if (ph.kind != kind) continue;
    for (const auto& [rank, slot] : ph.runs) {
      if (!c->local(rank)) continue;
      bh_runner* r = runner_at(c, rank, slot);
      int rc;
      if (kind == BE_PHASE_PREFILL) {
        rc = bh_runner_run(r, 0);
      } else {
        int nb = 0;
        const bool in_here = first && slot == home_slot && host_in != nullptr;
        rc = bh_runner_decode_step(r, in_here ? host_in : nullptr, nullptr, &nb);
        c->stats.batches += nb;
      }
      if (rc != BE_OK) throw ClusterError(rc, bh_runner_last_error(r));
    }
    do_hops(c, ph);
    first = false;
  }
  if (kind == BE_PHASE_DECODE) {
    ++c->stats.steps;
    if (host_out != nullptr) {
      // end to end: the home runner's rows (every request of this rank) back to the host
      bh_runner* home = runner_at(c, c->rank0, home_slot);
      const int64_t rows = bh_runner_requests(home);
      cudaStream_t st = c->stream_of(c->rank0);
      ck(cudaMemcpyAsync(host_out, bh_runner_arena(home), rows * c->row_bytes,
                         cudaMemcpyDeviceToHost, st), "host rows");
      ck(cudaStreamSynchronize(st), "host rows sync");
    }
  }
}
}  // namespace

extern "C" int bh_cluster_create(be_comm* comm, int rank0, int n_local, be_ctx* const* ctxs,
                                 int d_model, bh_cluster** out) {
  if (out == nullptr || n_local < 1 || ctxs == nullptr || d_model <= 0 || rank0 < 0)
    return BE_ERR_INVALID;
  *out = nullptr;
  auto* c = new bh_cluster();
  c->comm = comm;
  c->rank0 = rank0;
  c->row_bytes = d_model * 2;
  for (int i = 0; i < n_local; ++i) {
    if (ctxs[i] == nullptr) {
      delete c;
      return BE_ERR_INVALID;
    }
    c->ctxs.push_back(ctxs[i]);
    cudaEvent_t ev;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
      for (auto e : c->evs) cudaEventDestroy(e);
      delete c;
      return BE_ERR_CUDA;
    }
    c->evs.push_back(ev);
  }
  if (comm != nullptr && (be_comm_rank(comm) != rank0 || n_local != 1)) {
    for (auto e : c->evs) cudaEventDestroy(e);
    delete c;
    return BE_ERR_INVALID;  // with a communicator: one rank per process
  }
  *out = c;
  return BE_OK;
}

extern "C" int bh_cluster_free(bh_cluster* c) {
  if (c == nullptr) return BE_ERR_INVALID;
  for (auto e : c->evs) cudaEventDestroy(e);
  delete c;
  return BE_OK;
}

extern "C" const char* bh_cluster_last_error(const bh_cluster* c) {
  return c == nullptr ? "null cluster" : c->err.c_str();
}

extern "C" int bh_cluster_add_runner(bh_cluster* c, int rank, int slot, bh_runner* r) {
  if (c == nullptr || r == nullptr || !c->local(rank) || slot < 0) return BE_ERR_INVALID;
  c->runners[{rank, slot}] = r;
  return BE_OK;
}

extern "C" int bh_cluster_add_phase(bh_cluster* c, int kind, int n_runs, const int32_t* runs,
                                    int n_hops, const bh_hop* hops) {
  if (c == nullptr || (kind != BE_PHASE_PREFILL && kind != BE_PHASE_DECODE) || n_runs < 0 ||
      n_hops < 0 || (n_runs > 0 && runs == nullptr) || (n_hops > 0 && hops == nullptr))
    return BE_ERR_INVALID;
  bh_cluster::Phase ph;
  ph.kind = kind;
  for (int i = 0; i < n_runs; ++i) ph.runs.emplace_back(runs[2 * i], runs[2 * i + 1]);
  for (int i = 0; i < n_hops; ++i) {
    const bh_hop& h = hops[i];
    if (h.rows < 0 || h.src_row < 0 || h.dst_row < 0 ||
        (h.arena != BH_ARENA_DECODE && h.arena != BH_ARENA_PREFILL)) {
      c->err = "bad hop " + std::to_string(i);
      return BE_ERR_INVALID;
    }
    if (h.src_rank == h.dst_rank && h.src_runner == h.dst_runner) continue;  // rows stay put
    ph.hops.push_back(h);
  }
  c->phases.push_back(std::move(ph));
  return BE_OK;
}

extern "C" int bh_cluster_prefill(bh_cluster* c) {
  if (c == nullptr) return BE_ERR_INVALID;
  return guard(c, [&] {
    run_phases(c, BE_PHASE_PREFILL, nullptr, nullptr, 0);
    for (size_t i = 0; i < c->ctxs.size(); ++i)
      ck(cudaStreamSynchronize(c->stream_of(c->rank0 + (int)i)), "prefill sync");
  });
}

extern "C" int bh_cluster_decode_step(bh_cluster* c, int home_slot, const void* host_in,
                                      void* host_out) {
  if (c == nullptr || ((host_in != nullptr || host_out != nullptr) && c->ctxs.size() != 1))
    return BE_ERR_INVALID;
  return guard(c, [&] { run_phases(c, BE_PHASE_DECODE, host_in, host_out, home_slot); });
}

extern "C" int bh_cluster_get_stats(const bh_cluster* c, bh_cluster_stats* out) {
  if (c == nullptr || out == nullptr) return BE_ERR_INVALID;
  *out = c->stats;
  return BE_OK;
}
