// comm.cu -- multi-GPU plumbing: one process per GPU,
// destination-range partition.  The owned Y rows of every rank are gathered
// with grouped NCCL broadcasts (ranks own unequal row counts, so no padding
// is needed); dW / dA / dW0 are summed with an in-place NCCL all-reduce.
// NCCL runs over NVLink 5 / NVSwitch on the B200 box.
#include <nccl.h>

#include "common.cuh"
#include "kernels.cuh"

struct rgnn_comm {
  ncclComm_t nccl;              // caller-stream collectives (dW / dA all-reduce, dX reduce-scatter, sync gather)
  ncclComm_t gcomm;             // the asynchronous Y gather (its own stream; split from nccl)
  int nranks, rank;
  int flags;                    // RGNN_COMM_GATHER_ASYNC | RGNN_COMM_GATHER_BF16
  cudaStream_t side;            // stream of the asynchronous gather
  cudaEvent_t ev_ready, ev_done;  // owned rows written / gather finished
  bool pending;                 // an asynchronous gather was issued and not yet joined
  std::vector<int64_t> bounds;  // [nranks+1] dst ranges
};

namespace rgnn {

#define RGNN_NCCL_TRY(expr)                                                                       \
  do {                                                                                            \
    ncclResult_t _r = (expr);                                                                     \
    if (_r != ncclSuccess)                                                                        \
      return ::rgnn::set_error(RGNN_E_NCCL, "%s:%d %s: %s", __FILE__, __LINE__, #expr,             \
                               ncclGetErrorString(_r));                                           \
  } while (0)

rgnn_status comm_check_range(const rgnn_comm* c, int64_t v0, int64_t v1) {
  if (c->bounds[c->rank] != v0 || c->bounds[c->rank + 1] != v1)
    return set_error(RGNN_E_INVALID_ARG, "graph dst range [%lld,%lld) != comm bounds of rank %d", (long long)v0,
                     (long long)v1, c->rank);
  return RGNN_OK;
}

// Y_full[bounds[k]:bounds[k+1]] <- rank k's owned rows, for every k (grouped broadcasts: ranks own
// unequal row counts, so nothing is padded).  RGNN_COMM_GATHER_BF16: Y_full is bf16; the owned rows
// are rounded (RNE) into Y_full's own slice and broadcast from there (in place at the root).
// RGNN_COMM_GATHER_ASYNC: the broadcasts run on the communicator's stream (second NCCL
// communicator) after an event on `s`; `s` continues at once and rgnn_comm_join orders a later
// reader of Y_full after them.
rgnn_status comm_gather_rows(rgnn_comm* c, const float* Y_own, int64_t N, void* Y_full, cudaStream_t s) {
  const bool bf = (c->flags & RGNN_COMM_GATHER_BF16) != 0, async = (c->flags & RGNN_COMM_GATHER_ASYNC) != 0;
  const size_t esz = bf ? 2 : 4;
  char* base = static_cast<char*>(Y_full);
  const int64_t v0 = c->bounds[c->rank], v1 = c->bounds[c->rank + 1];
  const void* send = Y_own;
  if (bf) {
    RGNN_TRY(launch_f32_to_bf16((v1 - v0) * N, Y_own, base + (size_t)v0 * N * esz, s));
    send = base + (size_t)v0 * N * esz;
  }
  cudaStream_t gs = s;
  ncclComm_t comm = c->nccl;
  if (async) {
    RGNN_CUDA_TRY(cudaEventRecord(c->ev_ready, s));
    RGNN_CUDA_TRY(cudaStreamWaitEvent(c->side, c->ev_ready, 0));
    gs = c->side;
    comm = c->gcomm;
  }
  RGNN_NCCL_TRY(ncclGroupStart());
  for (int k = 0; k < c->nranks; ++k) {
    size_t cnt = (size_t)(c->bounds[k + 1] - c->bounds[k]) * (size_t)N;
    if (cnt == 0) continue;
    RGNN_NCCL_TRY(ncclBroadcast(k == c->rank ? send : nullptr, base + (size_t)c->bounds[k] * N * esz, cnt,
                                bf ? ncclBfloat16 : ncclFloat, k, comm, gs));
  }
  RGNN_NCCL_TRY(ncclGroupEnd());
  if (async) {
    RGNN_CUDA_TRY(cudaEventRecord(c->ev_done, gs));
    c->pending = true;
  }
  return RGNN_OK;
}

// dX over the dst partition: rank k receives the sum over all ranks of rows [bounds[k], bounds[k+1])
// (grouped in-place reduces, one root per slice: a reduce-scatter with unequal slices, half the
// volume of an all-reduce); the other rows keep this rank's partial sums.
rgnn_status comm_reduce_rows(rgnn_comm* c, float* buf, int64_t K, cudaStream_t s) {
  RGNN_NCCL_TRY(ncclGroupStart());
  for (int k = 0; k < c->nranks; ++k) {
    size_t cnt = (size_t)(c->bounds[k + 1] - c->bounds[k]) * (size_t)K;
    if (cnt == 0) continue;
    float* p = buf + (size_t)c->bounds[k] * K;
    RGNN_NCCL_TRY(ncclReduce(p, p, cnt, ncclFloat, ncclSum, k, c->nccl, s));
  }
  RGNN_NCCL_TRY(ncclGroupEnd());
  return RGNN_OK;
}

rgnn_status comm_allreduce_sum(rgnn_comm* c, float* const* bufs, const size_t* counts, int n, cudaStream_t s) {
  RGNN_NCCL_TRY(ncclGroupStart());
  for (int i = 0; i < n; ++i)
    if (bufs[i] && counts[i]) RGNN_NCCL_TRY(ncclAllReduce(bufs[i], bufs[i], counts[i], ncclFloat, ncclSum, c->nccl, s));
  RGNN_NCCL_TRY(ncclGroupEnd());
  return RGNN_OK;
}

}  // namespace rgnn

using namespace rgnn;

extern "C" {

rgnn_status rgnn_comm_unique_id(void* id) {
  if (!id) return set_error(RGNN_E_INVALID_ARG, "id is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "nccl id size");
  RGNN_NCCL_TRY(ncclGetUniqueId(static_cast<ncclUniqueId*>(id)));
  return RGNN_OK;
}

rgnn_status rgnn_comm_create(const void* id, int nranks, int rank, const int64_t* bounds, rgnn_comm** out) {
  if (!id || !out || !bounds || nranks < 1 || rank < 0 || rank >= nranks)
    return set_error(RGNN_E_INVALID_ARG, "rgnn_comm_create: bad arguments");
  for (int k = 0; k < nranks; ++k)
    if (bounds[k] > bounds[k + 1] || bounds[0] != 0) return set_error(RGNN_E_INVALID_ARG, "bounds not monotone from 0");
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm, gcomm;
  RGNN_NCCL_TRY(ncclCommInitRank(&comm, nranks, uid, rank));
  RGNN_NCCL_TRY(ncclCommSplit(comm, 0, rank, &gcomm, nullptr));  // the asynchronous gather's communicator
  rgnn_comm* c = new rgnn_comm();
  c->nccl = comm;
  c->gcomm = gcomm;
  c->nranks = nranks;
  c->rank = rank;
  c->flags = 0;
  c->pending = false;
  c->bounds.assign(bounds, bounds + nranks + 1);
  RGNN_CUDA_TRY(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
  RGNN_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming));
  RGNN_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming));
  *out = c;
  return RGNN_OK;
}

rgnn_status rgnn_comm_set_options(rgnn_comm* c, int flags) {
  if (!c) return set_error(RGNN_E_INVALID_ARG, "comm is NULL");
  if (flags & ~(RGNN_COMM_GATHER_ASYNC | RGNN_COMM_GATHER_BF16))
    return set_error(RGNN_E_INVALID_ARG, "unknown comm flags 0x%x", flags);
  c->flags = flags;
  return RGNN_OK;
}

rgnn_status rgnn_comm_join(rgnn_comm* c, void* stream) {
  if (!c) return set_error(RGNN_E_INVALID_ARG, "comm is NULL");
  if (c->pending) {
    RGNN_CUDA_TRY(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), c->ev_done, 0));
    c->pending = false;
  }
  return RGNN_OK;
}

void rgnn_comm_destroy(rgnn_comm* c) {
  if (!c) return;
  cudaStreamSynchronize(c->side);
  ncclCommDestroy(c->gcomm);
  ncclCommDestroy(c->nccl);
  cudaEventDestroy(c->ev_ready);
  cudaEventDestroy(c->ev_done);
  cudaStreamDestroy(c->side);
  delete c;
}

}  // extern "C"
