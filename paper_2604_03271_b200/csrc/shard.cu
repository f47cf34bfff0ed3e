// shard.cu -- exchange kernels for particle-sharded runs whose shards live on
// one device (the protocol check of SURVEY.md 8e-3 on a single GPU).  Across
// GPUs the same exchanges are NCCL collectives (host.cu, NcclExchange).
#include "launch.h"

namespace smc {

__device__ __forceinline__ double xinf() { return __longlong_as_double(0x7ff0000000000000LL); }
__device__ __forceinline__ double* xfield(const GroupDesc& g, int buf) { return buf == 0 ? g.xbuf : g.stat_acc; }

// element-wise reduction over the nsh shards of each run (block = run; the
// list holds the runs' shards run-major, shard order), in shard order
// (deterministic); the result is written back to every shard
__global__ void k_xreduce(const GroupDesc* __restrict__ gds, const int* __restrict__ list, int nsh, int buf,
                          int count, int op) {
  const int* l = list + (size_t)blockIdx.x * nsh;
  if (count < 0) count = 2 * gds[l[0]].d;  // step statistics: 2d of this run
  for (int e = threadIdx.x; e < count; e += blockDim.x) {
    double v = op == XOP_SUM ? 0.0 : (op == XOP_MIN ? xinf() : -xinf());
    for (int r = 0; r < nsh; ++r) {
      const double x = xfield(gds[l[r]], buf)[e];
      v = op == XOP_SUM ? v + x : (op == XOP_MIN ? (x < v ? x : v) : (x > v ? x : v));
    }
    for (int r = 0; r < nsh; ++r) xfield(gds[l[r]], buf)[e] = v;
  }
}

// every shard's (xbuf[0], xbuf[1]) into slot g.shard of every shard's xgat (block = run)
__global__ void k_xgather(const GroupDesc* __restrict__ gds, const int* __restrict__ list, int nsh) {
  const int* l = list + (size_t)blockIdx.x * nsh;
  for (int t = threadIdx.x; t < nsh * nsh; t += blockDim.x) {
    const GroupDesc& dst = gds[l[t / nsh]];
    const GroupDesc& src = gds[l[t % nsh]];
    dst.xgat[2 * src.shard] = src.xbuf[0];
    dst.xgat[2 * src.shard + 1] = src.xbuf[1];
  }
}

cudaError_t launch_xreduce(const GroupDesc* gds, const int* list, int nruns, int nsh, int buf, int count, int op,
                           cudaStream_t st) {
  k_xreduce<<<nruns, 256, 0, st>>>(gds, list, nsh, buf, count, op);
  return cudaGetLastError();
}

cudaError_t launch_xgather(const GroupDesc* gds, const int* list, int nruns, int nsh, cudaStream_t st) {
  k_xgather<<<nruns, 256, 0, st>>>(gds, list, nsh);
  return cudaGetLastError();
}

}  // namespace smc
