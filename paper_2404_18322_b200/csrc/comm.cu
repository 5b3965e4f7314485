// The inter-block hop on the GPU: when a chain crosses GPUs, the [rows x d] bf16
// activation slab of the crossing moves by NCCL point-to-point send/recv over NVLink / NVSwitch
// (Simulation::deliver, proj/core/src/scenario.cpp:282-308; LinkManager::transfer,
// proj/core/src/cluster.cpp:170-192; payload 2*d_out bytes per token, costmodel.cpp:129-131).
// One communicator per process (one process per GPU); the hops of one executor phase are issued
// as one NCCL group on the compute stream, so they are ordered after the block that produced the
// rows and before the block that consumes them without any host synchronisation.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/blockexec.h"

struct be_comm {
  be_ctx* ctx = nullptr;
  ncclComm_t comm = nullptr;
  int n_ranks = 0, rank = 0, device = 0;
  int depth = 0;  // open be_hop_begin groups
  int64_t bytes_sent = 0, bytes_recv = 0;
  std::string err;
};

namespace {
int comm_fail(be_comm* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c != nullptr) c->err = buf;
  return code;
}
#define BE_NCCL(c, call)                                                                       \
  do {                                                                                         \
    const ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess) return comm_fail((c), BE_ERR_RUNTIME, "%s: %s", #call,              \
                                            ncclGetErrorString(r_));                           \
  } while (0)
}  // namespace

static_assert(sizeof(ncclUniqueId) == BE_COMM_ID_BYTES, "NCCL unique id size");

extern "C" int be_comm_unique_id(void* id_out) {
  if (id_out == nullptr) return BE_ERR_INVALID;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return BE_ERR_RUNTIME;
  std::memcpy(id_out, &id, sizeof(id));
  return BE_OK;
}

extern "C" int be_comm_init(be_ctx* ctx, int n_ranks, int rank, const void* id, be_comm** out) {
  if (ctx == nullptr || id == nullptr || out == nullptr || n_ranks < 1 || rank < 0 ||
      rank >= n_ranks)
    return BE_ERR_INVALID;
  *out = nullptr;
  auto* c = new be_comm();
  c->ctx = ctx;
  c->n_ranks = n_ranks;
  c->rank = rank;
  cudaGetDevice(&c->device);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  const ncclResult_t r = ncclCommInitRank(&c->comm, n_ranks, uid, rank);
  if (r != ncclSuccess) {
    std::fprintf(stderr, "be_comm_init: ncclCommInitRank: %s\n", ncclGetErrorString(r));
    delete c;
    return BE_ERR_RUNTIME;
  }
  *out = c;
  return BE_OK;
}

extern "C" int be_comm_destroy(be_comm* c) {
  if (c == nullptr) return BE_ERR_INVALID;
  if (c->comm) ncclCommDestroy(c->comm);
  delete c;
  return BE_OK;
}

extern "C" const char* be_comm_last_error(const be_comm* c) {
  return c == nullptr ? "null communicator" : c->err.c_str();
}
extern "C" int be_comm_rank(const be_comm* c) { return c ? c->rank : -1; }
extern "C" int be_comm_size(const be_comm* c) { return c ? c->n_ranks : 0; }
extern "C" int64_t be_comm_bytes(const be_comm* c, int sent) {
  return c == nullptr ? 0 : sent ? c->bytes_sent : c->bytes_recv;
}

extern "C" int be_hop_begin(be_comm* c) {
  if (c == nullptr) return BE_ERR_INVALID;
  BE_NCCL(c, ncclGroupStart());
  ++c->depth;
  return BE_OK;
}

extern "C" int be_hop_end(be_comm* c) {
  if (c == nullptr || c->depth <= 0) return BE_ERR_INVALID;
  --c->depth;
  BE_NCCL(c, ncclGroupEnd());
  return BE_OK;
}

namespace {
int hop(be_comm* c, int peer, void* rows, int64_t bytes, void* stream, bool send) {
  if (c == nullptr || peer < 0 || peer >= c->n_ranks || peer == c->rank || bytes < 0 ||
      (bytes > 0 && rows == nullptr))
    return comm_fail(c, BE_ERR_INVALID, "be_hop_%s: bad arguments (peer %d)", send ? "send" : "recv",
                     peer);
  if (bytes == 0) return BE_OK;
  cudaStream_t st = stream != nullptr ? static_cast<cudaStream_t>(stream)
                                      : static_cast<cudaStream_t>(be_ctx_stream(c->ctx));
  // bf16 rows travel as bytes: no reduction, so the element type does not matter to NCCL
  if (send) {
    BE_NCCL(c, ncclSend(rows, (size_t)bytes, ncclUint8, peer, c->comm, st));
    c->bytes_sent += bytes;
  } else {
    BE_NCCL(c, ncclRecv(rows, (size_t)bytes, ncclUint8, peer, c->comm, st));
    c->bytes_recv += bytes;
  }
  return BE_OK;
}
}  // namespace

extern "C" int be_hop_send(be_comm* c, int peer, const void* d_rows, int64_t bytes, void* stream) {
  return hop(c, peer, const_cast<void*>(d_rows), bytes, stream, true);
}

extern "C" int be_hop_recv(be_comm* c, int peer, void* d_rows, int64_t bytes, void* stream) {
  return hop(c, peer, d_rows, bytes, stream, false);
}
