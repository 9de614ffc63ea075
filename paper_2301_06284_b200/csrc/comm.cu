// comm.cu -- multi-GPU plumbing: one process per GPU,
// destination-range partition.  The owned Y rows of every rank are gathered
// with grouped NCCL broadcasts (ranks own unequal row counts, so no padding
// is needed); dW / dA / dW0 are summed with an in-place NCCL all-reduce.
// NCCL runs over NVLink 5 / NVSwitch on the B200 box.
#include <cuda.h>
#include <nccl.h>

#include <cstring>

#include "common.cuh"
#include "kernels.cuh"

struct rgnn_comm {
  // peer-memory mode (rgnn_comm_create_local + rgnn_comm_attach_peers; no NCCL): every rank's Y_full,
  // signal and staging buffers mapped into this process through CUDA IPC
  bool ipc = false;
  float* peer_y[rgnn::kMaxPeers] = {};      // other ranks' Y_full (index = peer slot, see peer_rank)
  int peer_rank[rgnn::kMaxPeers] = {};
  int npeer = 0;
  uint32_t* sig = nullptr;                  // this rank's signal words [nranks] + epoch counter
  uint32_t* peer_sig[rgnn::kMaxRanks] = {};  // every rank's signal words (own included)
  float* stage = nullptr;                   // this rank's staging buffer (gradient partials)
  float* peer_stage[rgnn::kMaxRanks] = {};  // every rank's staging buffer (own included)
  size_t stage_floats = 0;
  std::vector<void*> mapped;                // IPC mappings to close
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

rgnn_status comm_peer_gather(rgnn_comm* c, const float* Y_own, int64_t N, float* Y_full, bool fused, cudaStream_t s);

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
  if (c->ipc) return comm_peer_gather(c, Y_own, N, static_cast<float*>(Y_full), false, s);
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
  if (c->ipc) return set_error(RGNN_E_UNSUPPORTED, "dX with a peer-memory communicator (use NCCL)");
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

// ---------------------------------------------------------------- peer-memory (CUDA IPC) mode
// Device-side barrier over the ranks: each rank bumps its epoch, publishes it into every peer's
// signal word for this rank (release, system scope, after a system fence that orders the stores its
// earlier kernels made into peer memory -- each writing thread also fenced before exiting) and waits
// until every peer has published the same epoch into its own words (acquire).  Every rank runs the
// same sequence of barriers, so the epochs stay in step; the counter lives in device memory, so a
// captured CUDA graph replays correctly.
struct PeerSigs {
  uint32_t* p[kMaxRanks];
};
__global__ void k_peer_barrier(int nranks, int rank, PeerSigs peers, uint32_t* my_sig) {
  __shared__ uint32_t e;
  const int t = threadIdx.x;
  if (t == 0) { e = my_sig[kMaxRanks] + 1; my_sig[kMaxRanks] = e; }
  __syncthreads();
  __threadfence_system();
  if (t < nranks && t != rank)
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(peers.p[t] + rank), "r"(e) : "memory");
  if (t < nranks && t != rank) {
    uint32_t v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(my_sig + t) : "memory");
      if ((int32_t)(v - e) < 0) __nanosleep(256);
    } while ((int32_t)(v - e) < 0);
  }
  __syncthreads();
}
// dst = sum over ranks (in rank order) of stage_k[off .. off+n): the deterministic all-reduce.
struct PeerStages {
  const float* p[kMaxRanks];
};
__global__ void k_peer_sum(int nranks, PeerStages st, size_t off, size_t n, float* __restrict__ dst) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float v = 0.f;
    for (int k = 0; k < nranks; ++k) v += st.p[k][off + i];
    dst[i] = v;
  }
}
// owned Y rows pushed into every peer's Y_full (the models whose walk does not store to peers itself)
struct PeerRows {
  float* p[kMaxPeers];
};
__global__ void k_peer_push(int npeer, PeerRows peers, const float* __restrict__ Y, int64_t n, int64_t ofs) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = reinterpret_cast<const float4*>(Y)[i];
    for (int p = 0; p < npeer; ++p) reinterpret_cast<float4*>(peers.p[p] + ofs)[i] = v;
  }
  __threadfence_system();
}

int comm_peer_rows(const rgnn_comm* c, float** out) {
  if (!c || !c->ipc) return 0;
  for (int i = 0; i < c->npeer; ++i) out[i] = c->peer_y[i];
  return c->npeer;
}
bool comm_is_ipc(const rgnn_comm* c) { return c && c->ipc; }

rgnn_status comm_peer_barrier(rgnn_comm* c, cudaStream_t s) {
  PeerSigs ps{};
  for (int k = 0; k < c->nranks; ++k) ps.p[k] = c->peer_sig[k];
  RGNN_LAUNCH(k_peer_barrier, 1, 32, 0, s, c->nranks, c->rank, ps, c->sig);
  return RGNN_OK;
}

// Y_full of every rank gets this rank's owned rows: the walk has already stored them (fused) when
// `fused`; otherwise they are pushed here.  Then the barrier: after it, every rank's Y_full is complete.
rgnn_status comm_peer_gather(rgnn_comm* c, const float* Y_own, int64_t N, float* Y_full, bool fused, cudaStream_t s) {
  const int64_t v0 = c->bounds[c->rank], v1 = c->bounds[c->rank + 1];
  if (Y_full + v0 * N != Y_own && v1 > v0)
    RGNN_CUDA_TRY(cudaMemcpyAsync(Y_full + v0 * N, Y_own, sizeof(float) * (size_t)(v1 - v0) * N,
                                  cudaMemcpyDeviceToDevice, s));
  if (!fused) RGNN_TRY(comm_peer_barrier(c, s));  // entry barrier (the fused path had it before its walk)
  if (!fused && v1 > v0 && c->npeer > 0) {
    PeerRows pr{};
    for (int i = 0; i < c->npeer; ++i) pr.p[i] = c->peer_y[i];
    const int64_t n = (v1 - v0) * N;
    RGNN_LAUNCH(k_peer_push, (unsigned)std::min<int64_t>((n / 4 + 255) / 256, 148 * 8), 256, 0, s, c->npeer, pr,
                Y_own, n, v0 * N);
  }
  return comm_peer_barrier(c, s);
}

// In-place sums over the ranks through the staging buffers: partials -> own stage, barrier, every rank
// sums all stages in rank order (bit-identical results on every rank), barrier (no rank refills its
// stage before the others have read it).
rgnn_status comm_peer_allreduce(rgnn_comm* c, float* const* bufs, const size_t* counts, int n, cudaStream_t s) {
  size_t off = 0;
  for (int i = 0; i < n; ++i) {
    if (!bufs[i] || !counts[i]) continue;
    if (off + counts[i] > c->stage_floats)
      return set_error(RGNN_E_WORKSPACE, "peer staging buffer too small (%zu floats needed)", off + counts[i]);
    RGNN_CUDA_TRY(cudaMemcpyAsync(c->stage + off, bufs[i], sizeof(float) * counts[i], cudaMemcpyDeviceToDevice, s));
    off += counts[i];
  }
  RGNN_TRY(comm_peer_barrier(c, s));
  PeerStages st{};
  for (int k = 0; k < c->nranks; ++k) st.p[k] = c->peer_stage[k];
  off = 0;
  for (int i = 0; i < n; ++i) {
    if (!bufs[i] || !counts[i]) continue;
    RGNN_LAUNCH(k_peer_sum, (unsigned)std::min<size_t>((counts[i] + 255) / 256, 148 * 8), 256, 0, s, c->nranks, st,
                off, counts[i], bufs[i]);
    off += counts[i];
  }
  return comm_peer_barrier(c, s);
}

rgnn_status comm_allreduce_sum(rgnn_comm* c, float* const* bufs, const size_t* counts, int n, cudaStream_t s) {
  if (c->ipc) return comm_peer_allreduce(c, bufs, counts, n, s);
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

rgnn_status rgnn_comm_create_local(int nranks, int rank, const int64_t* bounds, rgnn_comm** out) {
  if (!out || !bounds || nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks)
    return set_error(RGNN_E_INVALID_ARG, "rgnn_comm_create_local: bad arguments (nranks <= %d)", kMaxRanks);
  for (int k = 0; k < nranks; ++k)
    if (bounds[k] > bounds[k + 1] || bounds[0] != 0) return set_error(RGNN_E_INVALID_ARG, "bounds not monotone from 0");
  rgnn_comm* c = new rgnn_comm();
  c->ipc = true;
  c->nccl = nullptr;
  c->gcomm = nullptr;
  c->nranks = nranks;
  c->rank = rank;
  c->flags = 0;
  c->pending = false;
  c->side = nullptr;
  c->bounds.assign(bounds, bounds + nranks + 1);
  *out = c;
  return RGNN_OK;
}

using PFN_memGetAddressRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

rgnn_status rgnn_ipc_export(const void* ptr, void* handle, int64_t* offset) {
  if (!ptr || !handle || !offset) return set_error(RGNN_E_INVALID_ARG, "NULL argument");
  static PFN_memGetAddressRange range = nullptr;
  if (!range) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
      return set_error(RGNN_E_CUDA, "cuMemGetAddressRange unavailable");
    range = reinterpret_cast<PFN_memGetAddressRange>(p);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
    return set_error(RGNN_E_INVALID_ARG, "pointer is not device memory");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
  RGNN_CUDA_TRY(cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t*>(handle), reinterpret_cast<void*>(base)));
  *offset = (int64_t)(reinterpret_cast<CUdeviceptr>(ptr) - base);
  return RGNN_OK;
}

rgnn_status rgnn_comm_attach_peers(rgnn_comm* c, const void* handles, const int64_t* offsets, float* Y_full,
                                   uint32_t* sig, float* stage, size_t stage_floats) {
  if (!c || !c->ipc) return set_error(RGNN_E_INVALID_ARG, "not a peer-memory communicator (rgnn_comm_create_local)");
  if (!handles || !offsets || !Y_full || !sig || !stage) return set_error(RGNN_E_INVALID_ARG, "NULL argument");
  const int P = c->nranks;
  auto open = [&](int k, int which, void** out) -> rgnn_status {
    cudaIpcMemHandle_t h;
    memcpy(&h, static_cast<const char*>(handles) + ((size_t)k * 3 + which) * 64, 64);
    void* base = nullptr;
    RGNN_CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    c->mapped.push_back(base);
    *out = static_cast<char*>(base) + offsets[(size_t)k * 3 + which];
    return RGNN_OK;
  };
  c->npeer = 0;
  for (int k = 0; k < P; ++k) {
    if (k == c->rank) {
      c->peer_sig[k] = sig;
      c->peer_stage[k] = stage;
      continue;
    }
    void *y, *sg, *st;
    RGNN_TRY(open(k, 0, &y));
    RGNN_TRY(open(k, 1, &sg));
    RGNN_TRY(open(k, 2, &st));
    c->peer_y[c->npeer] = static_cast<float*>(y);
    c->peer_rank[c->npeer] = k;
    ++c->npeer;
    c->peer_sig[k] = static_cast<uint32_t*>(sg);
    c->peer_stage[k] = static_cast<float*>(st);
  }
  c->sig = sig;
  c->stage = stage;
  c->stage_floats = stage_floats;
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
  if (c->ipc) {  // unmap the peers' buffers (the bases cudaIpcOpenMemHandle returned)
    for (void* b : c->mapped) cudaIpcCloseMemHandle(b);
    delete c;
    return;
  }
  cudaStreamSynchronize(c->side);
  ncclCommDestroy(c->gcomm);
  ncclCommDestroy(c->nccl);
  cudaEventDestroy(c->ev_ready);
  cudaEventDestroy(c->ev_done);
  cudaStreamDestroy(c->side);
  delete c;
}

}  // extern "C"
