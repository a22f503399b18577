// Tensor-parallel collectives of qs_forward_tp2 (config 4): NCCL all-reduce
// of the row-split partial sums and the vocab-split argmax (all-gather of per-rank
// (max, index) records, reduced in rank order -- lowest index wins ties, as
// numerics.py:81-86's first occurrence).  Everything is enqueued on the caller's
// stream: no host callback, no synchronisation, CUDA-graph capturable.
#include <nccl.h>

#include <cstring>

#include "../../include/qspec_b200.h"
#include "qs_common.cuh"

namespace qs {

constexpr int kTpMaxT = 64;  // tokens per forward (qs_linear_max_tokens)

int tp_allreduce_nccl(float* p, int64_t count, void* comm, cudaStream_t st) {
  return ncclAllReduce(p, p, (size_t)count, ncclFloat32, ncclSum, (ncclComm_t)comm, st) == ncclSuccess ? 0 : 1;
}

__global__ void tp_argmax_kernel(const int2* __restrict__ all, int world, int T, int32_t* __restrict__ argmax) {
  const int t = threadIdx.x;
  if (t >= T) return;
  int2 best = all[t];
  for (int r = 1; r < world; ++r) {
    const int2 c = all[(size_t)r * kTpMaxT + t];
    const float bv = __int_as_float(best.x), cv = __int_as_float(c.x);
    if (cv > bv || (cv == bv && c.y < best.y)) best = c;
  }
  argmax[t] = best.y;
}

int tp_argmax_reduce(const qs_tp_t* tp, int T, int32_t* argmax, cudaStream_t st) {
  if (T > kTpMaxT) return QS_ERR_SHAPE;
  int2* local = reinterpret_cast<int2*>(tp->scratch);
  int2* all = local + kTpMaxT;
  const size_t bytes = (size_t)kTpMaxT * sizeof(int2);
  if (tp->nccl_comm) {
    if (ncclAllGather(local, all, bytes / 4, ncclInt32, (ncclComm_t)tp->nccl_comm, st) != ncclSuccess)
      return QS_ERR_CUDA;
  } else if (tp->allgather(local, all, (int64_t)bytes, st, tp->user) != 0) {
    return QS_ERR_CUDA;
  }
  tp_argmax_kernel<<<1, kTpMaxT, 0, st>>>(all, tp->world, T, argmax);
  return cudaGetLastError() == cudaSuccess ? QS_OK : QS_ERR_CUDA;
}

}  // namespace qs

extern "C" {

size_t qs_tp_scratch_bytes(int32_t world) { return (size_t)(1 + world) * qs::kTpMaxT * sizeof(int2); }

int qs_tp_nccl_unique_id(uint8_t* id128) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return QS_ERR_CUDA;
  memcpy(id128, &id, sizeof(id));
  return QS_OK;
}

int qs_tp_nccl_init(int32_t world, int32_t rank, const uint8_t* id128, void** comm) {
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclComm_t c;
  if (ncclCommInitRank(&c, world, id, rank) != ncclSuccess) return QS_ERR_CUDA;
  *comm = c;
  return QS_OK;
}

int qs_tp_nccl_destroy(void* comm) {
  return (comm == nullptr || ncclCommDestroy((ncclComm_t)comm) == ncclSuccess) ? QS_OK : QS_ERR_CUDA;
}

}  // extern "C"
