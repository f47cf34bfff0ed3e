// shard.cu -- exchange kernels for particle-sharded runs whose shards live on
// one device (the protocol check of SURVEY.md 8e-3 on a single GPU).  Across
// GPUs the same exchanges are NCCL collectives (host.cu, NcclExchange).
#include "launch.h"

namespace smc {

__device__ __forceinline__ double xinf() { return __longlong_as_double(0x7ff0000000000000LL); }
__device__ __forceinline__ double* xfield(const GroupDesc& g, int buf) { return buf == 0 ? g.xbuf : g.stat_acc; }

// element-wise reduction over the n shards in shard-list order (deterministic),
// result written back to every shard
__global__ void k_xreduce(const GroupDesc* __restrict__ gds, const int* __restrict__ list, int n, int buf, int count,
                          int op) {
  for (int e = threadIdx.x; e < count; e += blockDim.x) {
    double v = op == XOP_SUM ? 0.0 : (op == XOP_MIN ? xinf() : -xinf());
    for (int r = 0; r < n; ++r) {
      const double x = xfield(gds[list[r]], buf)[e];
      v = op == XOP_SUM ? v + x : (op == XOP_MIN ? (x < v ? x : v) : (x > v ? x : v));
    }
    for (int r = 0; r < n; ++r) xfield(gds[list[r]], buf)[e] = v;
  }
}

// every shard's (xbuf[0], xbuf[1]) into slot g.shard of every shard's xgat
__global__ void k_xgather(const GroupDesc* __restrict__ gds, const int* __restrict__ list, int n) {
  for (int t = threadIdx.x; t < n * n; t += blockDim.x) {
    const GroupDesc& dst = gds[list[t / n]];
    const GroupDesc& src = gds[list[t % n]];
    dst.xgat[2 * src.shard] = src.xbuf[0];
    dst.xgat[2 * src.shard + 1] = src.xbuf[1];
  }
}

cudaError_t launch_xreduce(const GroupDesc* gds, const int* list, int n, int buf, int count, int op, cudaStream_t st) {
  k_xreduce<<<1, 256, 0, st>>>(gds, list, n, buf, count, op);
  return cudaGetLastError();
}

cudaError_t launch_xgather(const GroupDesc* gds, const int* list, int n, cudaStream_t st) {
  k_xgather<<<1, 256, 0, st>>>(gds, list, n);
  return cudaGetLastError();
}

}  // namespace smc
