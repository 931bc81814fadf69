// hmgpu_dist.cuh -- multi-GPU block-row sharding: NCCL loaded at run time
// and the device kernels of the distributed matvec (hmgpu_matvec_dist).
//
// each rank owns the blocks whose row cluster lies in its
// contiguous range of permuted rows [rb, re); its matvec writes those rows
// (internal order) into a segment of length maxseg per component and RHS;
// the segments of all ranks are all-gathered and every rank scatters them to
// external order, y[q][r][perm[rb_k + i]] = recv[k][q][r][i].
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>

namespace hmgpu {

// NCCL entry points resolved from libnccl.so.2 (the copy already mapped
// into the process -- e.g. torch's -- if there is one, else the system's),
// so the library loads and runs single-GPU on machines without NCCL.
struct NcclApi {
  bool ok = false;
  std::string why;
  int version = 0;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

inline NcclApi& nccl_api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      a.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) a.why = std::string("libnccl lacks ") + name;
      return fn != nullptr;
    };
    if (!(sym(a.GetVersion, "ncclGetVersion") && sym(a.GetUniqueId, "ncclGetUniqueId") &&
          sym(a.CommInitRank, "ncclCommInitRank") && sym(a.CommDestroy, "ncclCommDestroy") &&
          sym(a.Broadcast, "ncclBroadcast") && sym(a.AllGather, "ncclAllGather") &&
          sym(a.GetErrorString, "ncclGetErrorString")))
      return;
    a.GetVersion(&a.version);
    a.ok = true;
  });
  return a;
}

// internal row p of this shard -> its position in the segment (p - rb)
__global__ void dist_segperm_kernel(int* __restrict__ segperm, int n_rows, int rb, int re) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n_rows; p += gridDim.x * blockDim.x)
    segperm[p] = (p >= rb && p < re) ? p - rb : 0;
}

// recv: [world][nrhs][NOUT][maxseg] -> y: [nrhs][NOUT][n_rows] external
template <int NOUT>
__global__ void dist_scatter_kernel(const double* __restrict__ recv, int world, int nrhs,
                                    int maxseg, const int* __restrict__ rb,
                                    const int* __restrict__ len,
                                    const int* __restrict__ rperm, int n_rows,
                                    double* __restrict__ y) {
  const long long per_rank = (long long)nrhs * NOUT * maxseg;
  const long long total = per_rank * world;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % maxseg);
    const int k = (int)(t / per_rank);
    if (i >= len[k]) continue;
    const long long qr = (t % per_rank) / maxseg;  // q * NOUT + r
    y[qr * n_rows + rperm[rb[k] + i]] = recv[t];
  }
}

}  // namespace hmgpu
