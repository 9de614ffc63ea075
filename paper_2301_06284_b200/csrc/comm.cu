// comm.cu -- multi-GPU plumbing: one process per GPU,
// destination-range partition.  The owned Y rows of every rank are gathered
// with grouped NCCL broadcasts (ranks own unequal row counts, so no padding
// is needed); dW / dA / dW0 are summed with an in-place NCCL all-reduce.
// NCCL runs over NVLink 5 / NVSwitch on the B200 box.
#include <nccl.h>

#include "common.cuh"

struct rgnn_comm {
  ncclComm_t nccl;
  int nranks, rank;
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

// Y_full[bounds[k]:bounds[k+1]] <- rank k's owned rows, for every k.
rgnn_status comm_gather_rows(rgnn_comm* c, const float* Y_own, int64_t N, float* Y_full, cudaStream_t s) {
  RGNN_NCCL_TRY(ncclGroupStart());
  for (int k = 0; k < c->nranks; ++k) {
    size_t cnt = (size_t)(c->bounds[k + 1] - c->bounds[k]) * (size_t)N;
    if (cnt == 0) continue;
    RGNN_NCCL_TRY(ncclBroadcast(k == c->rank ? (const void*)Y_own : nullptr, Y_full + c->bounds[k] * N, cnt,
                                ncclFloat, k, c->nccl, s));
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
  ncclComm_t comm;
  RGNN_NCCL_TRY(ncclCommInitRank(&comm, nranks, uid, rank));
  rgnn_comm* c = new rgnn_comm();
  c->nccl = comm;
  c->nranks = nranks;
  c->rank = rank;
  c->bounds.assign(bounds, bounds + nranks + 1);
  *out = c;
  return RGNN_OK;
}

void rgnn_comm_destroy(rgnn_comm* c) {
  if (!c) return;
  ncclCommDestroy(c->nccl);
  delete c;
}

}  // extern "C"
