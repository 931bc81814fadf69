// hmgpu.cu -- host side of the C ABI declared in include/hmgpu.h.
//
// One hmgpu_ctx owns every device buffer of one H-matrix problem on one
// device: geometry in cluster-tree (internal) order, the ACA work items
// (one per admissible block and component) with their resumable state,
// the packed U/V arena, the near-field arena and the matvec work lists.
// All work runs on the ctx's own stream.  No exceptions cross the ABI.

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <array>
#include <unordered_map>
#include <map>
#include <mutex>
#include <thread>
#include <exception>
#include <new>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "hmgpu.h"
#include "hmgpu_device.cuh"
#include "hmgpu_stream.cuh"
#include "hmgpu_mrhs.cuh"
#include "hmgpu_amvm.cuh"
#include "hmgpu_dist.cuh"

using namespace hmgpu;

namespace {

struct Fail {
  int code;
  std::string msg;
};

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) {                                               \
      const int code_ = e_ == cudaErrorMemoryAllocation ? HMGPU_ERR_OOM    \
                                                        : HMGPU_ERR_CUDA;  \
      throw Fail{code_, std::string(#x) + ": " + cudaGetErrorString(e_)};  \
    }                                                                      \
  } while (0)

[[noreturn]] void fail(int code, const std::string& msg) { throw Fail{code, msg}; }

// Device buffers are stream-ordered allocations from the context's own
// memory pool (release threshold: never), so re-assembly reuses the HBM of
// the previous one instead of paying cudaMalloc / cudaFree of gigabytes.
// guard() points these at the calling context.
thread_local cudaMemPool_t g_pool = nullptr;
thread_local cudaStream_t g_stream = nullptr;

// every live context's pool and stream: on an out-of-memory the idle memory
// of all of them goes back to the device (trim is safe against in-use blocks)
std::mutex g_pools_mu;
std::vector<std::pair<cudaMemPool_t, cudaStream_t>> g_pools;

void reclaim_idle_memory() {
  std::lock_guard<std::mutex> lk(g_pools_mu);
  for (auto& ps : g_pools) {
    cudaStreamSynchronize(ps.second);
    cudaMemPoolTrimTo(ps.first, 0);
  }
}

void* pool_alloc(size_t bytes) {
  void* p = nullptr;
  if (!g_pool) {
    CK(cudaMalloc(&p, bytes));
    return p;
  }
  cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, g_pool, g_stream);
  if (e == cudaErrorMemoryAllocation) {  // give the pools' idle memory back, retry
    (void)cudaGetLastError();
    CK(cudaStreamSynchronize(g_stream));
    reclaim_idle_memory();
    e = cudaMallocFromPoolAsync(&p, bytes, g_pool, g_stream);
  }
  CK(e);
  return p;
}

void pool_free(void* p) {
  if (!p) return;
  if (g_pool) cudaFreeAsync(p, g_stream);
  else cudaFree(p);
}

// device memory still obtainable: free HBM plus the pool's idle reserve
size_t avail_bytes() {
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  if (g_pool) {
    unsigned long long reserved = 0, used = 0;
    CK(cudaMemPoolGetAttribute(g_pool, cudaMemPoolAttrReservedMemCurrent, &reserved));
    CK(cudaMemPoolGetAttribute(g_pool, cudaMemPoolAttrUsedMemCurrent, &used));
    free_b += (size_t)(reserved - used);
  }
  return free_b;
}

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;  // elements
  void free() {
    pool_free(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    free();
    if (count == 0) count = 1;
    p = (T*)pool_alloc(count * sizeof(T));
    n = count;
  }
  void ensure(size_t count) {
    if (count > n || !p) alloc(count);
  }
  void upload(const std::vector<T>& h, cudaStream_t s) {
    ensure(h.size());
    if (!h.empty())
      CK(cudaMemcpyAsync(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void upload(const T* h, size_t count, cudaStream_t s) {
    ensure(count);
    if (count) CK(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
};

// host vector in page-locked memory (fast D2H/H2D of the item mirror)
template <class T>
struct PinnedVec {
  T* p = nullptr;
  size_t n = 0, cap = 0;
  PinnedVec() = default;
  PinnedVec(const PinnedVec&) = delete;
  PinnedVec& operator=(const PinnedVec&) = delete;
  ~PinnedVec() {
    if (p) cudaFreeHost(p);
  }
  void reserve(size_t c) {
    if (c <= cap) return;
    T* q = nullptr;
    CK(cudaMallocHost(&q, c * sizeof(T)));
    if (p) {
      std::memcpy(q, p, n * sizeof(T));
      cudaFreeHost(p);
    }
    p = q;
    cap = c;
  }
  void push_back(const T& v) {
    if (n == cap) reserve(std::max<size_t>(1024, cap * 2));
    p[n++] = v;
  }
  void clear() { n = 0; }
  void resize(size_t c) {  // contents unspecified (filled by a download)
    reserve(c);
    n = c;
  }
  size_t size() const { return n; }
  bool empty() const { return n == 0; }
  T* data() { return p; }
  const T* data() const { return p; }
  T& operator[](size_t i) { return p[i]; }
  const T& operator[](size_t i) const { return p[i]; }
  T* begin() { return p; }
  T* end() { return p + n; }
  const T* begin() const { return p; }
  const T* end() const { return p + n; }
};

// The ACA factor arena: a virtual-address range reserved once (as large as
// the device memory) into which physical memory is mapped on demand
// (cuMemCreate / cuMemMap), so capacity regrow and AMVM refinement extend it
// in place -- no copy of the arena and no old + new peak.  Driver entry
// points come from cudaGetDriverEntryPoint (no link-time libcuda).
struct VmmApi {
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) addr_free = nullptr;
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) set_access = nullptr;
  decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
  bool ok = false;
};
const VmmApi& vmm_api() {
  static const VmmApi api = [] {
    VmmApi a;
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess && *fn;
    };
    a.ok = get("cuMemAddressReserve", (void**)&a.reserve) &&
           get("cuMemAddressFree", (void**)&a.addr_free) &&
           get("cuMemCreate", (void**)&a.create) && get("cuMemRelease", (void**)&a.release) &&
           get("cuMemMap", (void**)&a.map) && get("cuMemUnmap", (void**)&a.unmap) &&
           get("cuMemSetAccess", (void**)&a.set_access) &&
           get("cuMemGetAllocationGranularity", (void**)&a.granularity);
    return a;
  }();
  return api;
}

#define CU(x)                                                                  \
  do {                                                                         \
    CUresult r_ = (x);                                                         \
    if (r_ != CUDA_SUCCESS)                                                    \
      throw Fail{r_ == CUDA_ERROR_OUT_OF_MEMORY ? HMGPU_ERR_OOM : HMGPU_ERR_CUDA, \
                 std::string(#x) + ": CUresult " + std::to_string((int)r_)};  \
  } while (0)

struct VArena {
  double* p = nullptr;
  size_t n = 0;  // mapped capacity in doubles
  CUdeviceptr base = 0;
  size_t va = 0, mapped = 0, gran = 0;
  int device = -1;
  std::vector<std::pair<CUmemGenericAllocationHandle, size_t>> chunks;

  VArena() = default;
  VArena(VArena&& o) noexcept { *this = std::move(o); }
  VArena(const VArena&) = delete;
  VArena& operator=(const VArena&) = delete;
  VArena& operator=(VArena&& o) noexcept {
    std::swap(p, o.p);
    std::swap(n, o.n);
    std::swap(base, o.base);
    std::swap(va, o.va);
    std::swap(mapped, o.mapped);
    std::swap(gran, o.gran);
    std::swap(device, o.device);
    std::swap(chunks, o.chunks);
    return *this;
  }
  ~VArena() { free(); }

  CUmemAllocationProp prop() const {
    CUmemAllocationProp pr{};
    pr.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    pr.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    pr.location.id = device;
    return pr;
  }
  // capacity for `count` doubles: maps more physical memory at the end
  void ensure(size_t count, int dev) {
    const VmmApi& api = vmm_api();
    if (!api.ok) fail(HMGPU_ERR_CUDA, "virtual memory management entry points unavailable");
    if (count == 0) count = 1;
    if (count <= n) return;
    if (!base) {
      device = dev;
      const CUmemAllocationProp pr = prop();
      CU(api.granularity(&gran, &pr, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
      size_t free_b = 0, total_b = 0;
      CK(cudaMemGetInfo(&free_b, &total_b));
      va = (total_b + gran - 1) / gran * gran;
      CU(api.reserve(&base, va, 0, 0, 0));
      p = reinterpret_cast<double*>(base);
    }
    const size_t want = count * sizeof(double);
    if (want > va) fail(HMGPU_ERR_OOM, "arena larger than the device memory");
    // grow by at least 1/8 of the mapped size (fewer, larger chunks)
    size_t delta = std::max(want - mapped, mapped / 8);
    delta = std::min((delta + gran - 1) / gran * gran, va - mapped);
    const CUmemAllocationProp pr = prop();
    CUmemGenericAllocationHandle hnd;
    const auto tg0 = std::chrono::steady_clock::now();
    CUresult rc = api.create(&hnd, delta, &pr, 0);
    if (rc == CUDA_ERROR_OUT_OF_MEMORY) {  // idle pool memory back to the device, retry
      reclaim_idle_memory();
      rc = api.create(&hnd, delta, &pr, 0);
    }
    const size_t need = (want - mapped + gran - 1) / gran * gran;
    if (rc == CUDA_ERROR_OUT_OF_MEMORY && need < delta) {  // the 1/8 headroom does not fit
      delta = need;
      rc = api.create(&hnd, delta, &pr, 0);
    }
    CU(rc);
    CUresult r = api.map(base + mapped, delta, 0, hnd, 0);
    if (r != CUDA_SUCCESS) {
      api.release(hnd);
      CU(r);
    }
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    r = api.set_access(base + mapped, delta, &acc, 1);
    if (r != CUDA_SUCCESS) {
      api.unmap(base + mapped, delta);
      api.release(hnd);
      CU(r);
    }
    chunks.push_back({hnd, delta});
    mapped += delta;
    n = mapped / sizeof(double);
    if (std::getenv("HMGPU_VERBOSE"))
      std::fprintf(stderr, "[hmgpu] arena grow +%.2f GB -> %.2f GB, %.1f ms\n", delta / 1e9,
                   mapped / 1e9,
                   std::chrono::duration<double, std::milli>(
                       std::chrono::steady_clock::now() - tg0).count());
  }
  // releases everything (callers synchronise the stream first)
  void free() {
    if (!base) return;
    const VmmApi& api = vmm_api();
    size_t off = 0;
    for (auto& ch : chunks) {
      api.unmap(base + off, ch.second);
      api.release(ch.first);
      off += ch.second;
    }
    chunks.clear();
    api.addr_free(base, va);
    base = 0;
    p = nullptr;
    n = 0;
    mapped = va = 0;
  }
};

struct KTime {
  double ms = 0.0;
  long long launches = 0;
};

struct PendingEv {
  std::string name;
  cudaEvent_t a, b;
};

long long align2(long long v) { return (v + 1) & ~1LL; }

// vector allocator whose resize() leaves trivial elements uninitialized (the
// plan tables are filled right after, in parallel: no serial zero-fill and
// the first-touch page faults spread over the filling threads)
template <class T>
struct NoInitAlloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = NoInitAlloc<U>;
  };
  NoInitAlloc() = default;
  template <class U>
  NoInitAlloc(const NoInitAlloc<U>&) {}
  template <class U>
  void construct(U* p) noexcept {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... A>
  void construct(U* p, A&&... a) {
    ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
  }
};
template <class T>
using fast_vector = std::vector<T, NoInitAlloc<T>>;
inline int c_comp_host_r(int q) {
  static const int r[6] = {0, 0, 0, 1, 1, 2};
  return r[q];
}
inline int c_comp_host_c(int q) {
  static const int c[6] = {0, 1, 2, 1, 2, 2};
  return c[q];
}
long long align16(long long v) { return (v + 15) & ~15LL; }

}  // namespace

struct hmgpu_ctx {
  int device = -1;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  std::string err;

  // ---- problem definition (host copies) ----
  int kind = -1;
  int NC = 1;  // components: 6 for the Kelvin grid, 1 otherwise
  std::vector<double> verts, centroid, area, diam, pts, amat;
  std::vector<int> tris;
  int n_vert = 0, n_tri = 0, n_pts = 0, am = 0, an = 0;
  double E = 1.0, nu = 0.3, diag = 2.0;
  RuleTable rules{};
  bool rules_set[3] = {false, false, false};
  int gal_which = 0;                   // galerkin: 0 V_kl grid, 1 V_Delta
  std::vector<double> normals;         // K_Delta: unit normals per triangle
  std::vector<double> eval_pts;        // Kelvin: evaluation points (empty: centroids)
  int dl_r = 0, dl_c = 0;              // double layer: grid cell
  std::vector<double> prule[4];        // galerkin singular pair rules, SoA per case
  int prule_n[4] = {0, 0, 0, 0};

  // ---- partition ----
  bool have_partition = false;
  int n_rows = 0, n_cols = 0;
  std::vector<int> rperm, cperm;
  std::vector<int> rnodes, cnodes;  // 4 ints per node
  std::vector<int> blocks;          // 4 ints per block
  int n_blocks = 0;
  int row_begin = 0, row_end = 0;
  bool same_tree = false;

  // ---- device geometry ----
  DBuf<double4> d_rowpt, d_colpt;
  DBuf<double> d_tri, d_A, d_prule;
  DBuf<double4> d_vtx;
  DBuf<int4> d_tvid, d_tvx;
  DBuf<double4> d_tce, d_tna;
  DBuf<int> d_vtptr;
  DBuf<int2> d_vttri;
  DBuf<int> d_rperm, d_cperm;
  Geom geom{};

  // ---- assembly state ----
  bool assembled = false;
  double eps = 0, beta = 0;
  int initial_rank = -1, lookahead = 2;
  long long max_rank = 1LL << 30;
  PinnedVec<Item> items;          // host mirror (sizes, offsets, ranks), pinned
  std::vector<int> item_of_block; // first item of block b (-1: dense/not owned)
  std::vector<int> dense_of_block;
  std::vector<DenseBlock> dblocks;
  DBuf<Item> d_items;
  VArena d_arena;                 // U/V factors (growable in place)
  VArena spare_arena;             // the other arena of the compaction, kept mapped
  long long arena_used = 0;
  DBuf<int2> d_piv;
  long long piv_used = 0;
  DBuf<uint8_t> d_cons;
  DBuf<double> d_dense;
  long long dense_used = 0;
  DBuf<DenseBlock> d_dblocks;
  DBuf<int> d_counter, d_overflow, d_list;
  DBuf<unsigned long long> d_nq;  // near-field quadrature points (counted flops)

  // ---- matvec structures ----
  std::vector<MvBlock> mvb;
  DBuf<MvBlock> d_mvb;
  DBuf<int> d_mvorder;
  int n_mv = 0;
  long long part_rows = 0;
  std::vector<int> leaf_begin, leaf_end, leaf_ptr;
  std::vector<long long> leaf_prow;
  std::vector<int2> leaf_blk;     // per leaf entry: (matvec block, row offset in block)
  DBuf<int> d_leaf_begin, d_leaf_end, d_leaf_ptr;
  DBuf<long long> d_leaf_prow;
  DBuf<int2> d_leaf_blk;
  int kmax = 0;
  DBuf<double> d_x, d_y, d_xi, d_ypart;

  // ---- streamed matvec plan (packed current-rank arena, task list) ----
  bool plan_valid = false;
  int plan_mode = -1, plan_nrhs = -1;
  int p_ntasks = 0, p_nz = 0;
  long long p_slots = 0, p_zslots = 0, p_arena_len = 0;
  size_t p_smem = 0;
  DBuf<WJob> d_pjobs;
  DBuf<WChunk> d_pchunks;
  DBuf<int> d_pwoff;
  int p_woff_base[2] = {0, 0}, p_chunk_base[2] = {0, 0};
  int p_nwarps = 0, p_njb = 0;
  int p_nwarps_pass[2] = {0, 0};
  int p_ngroups_pass[2] = {0, 0};  // pooled groups of small chain units per pass (dynamic tail)
  DBuf<int> d_mvctr;               // their counters (zeroed by the gather kernel)
  size_t p_smem_pass[2] = {0, 0};
  DBuf<double> d_zpart;
  DBuf<LeafEntry> d_pentries;

  // ---- device-resident AMVM estimator (hmgpu_amvm.cuh) ----
  bool am_geom_valid = false;
  // transposed matvec tables (column leaves), built on first use
  // parallel marking walk: chunk buffers (hmgpu_amvm_mark)
  DBuf<unsigned long long> w_keys, w_skeys;
  DBuf<int> w_slots, w_sslots;
  DBuf<long long> w_gslot;
  DBuf<double> w_rb, w_dots;
  bool t_valid = false;
  int t_nleaves = 0;
  long long t_rows = 0;
  DBuf<long long> d_tprow, d_tleaf_prow;
  DBuf<int> d_tleaf_begin, d_tleaf_end, d_tleaf_ptr;
  DBuf<double> d_tpart, d_xr;
  bool am_have_mark = false;  // hmgpu_amvm_mark ran since the last refine
  // hmgpu_set_matvec_policy: 0 the packed stream plan, 1 1-RHS matvecs sweep the
  // blocks in place, 2 automatic: the first 1-RHS product after a rank change
  // (assembly, promote, extend) runs in place, the plan is built for the second
  int mv_policy = 0;
  bool mv_auto_used = false;  // policy 2: the in-place product of these ranks is spent
  DBuf<int> d_row_leaf, d_sortp, d_tix, d_term_bi, d_cnt, d_ptr, d_lists, d_order, d_idx,
      d_marked, d_nm, d_mids;
  DBuf<long long> d_spoff, d_eptr, d_eidx, d_ecnt;
  DBuf<double> d_eval;
  DBuf<TailTerm> d_aterms;
  DBuf<double> d_aout, d_diff, d_resid, d_nsq, d_sc;
  DBuf<unsigned long long> d_keys, d_keys2;
  DBuf<unsigned char> d_inset, d_cub;
  int am_nterms = 0;
  long long am_nvals = 0;
  bool am_have_estimate = false;
  std::vector<int> marked_ids;

  // ---- multi-RHS (16 per pass, fp64 tensor cores) plan (hmgpu_mrhs.cuh) ----
  bool p16_valid = false;
  int p16_mode = -1;
  int p16_ns = 2, p16_stage = 0, p16_ncta = 0;
  int p16_zns = 3, p16_zstage = 0, p16_nctaz = 0, p16_znw = 8, p16_ynw = 8;
  int p16_zunits = 0, p16_yunits = 0;  // dynamically scheduled work units per pass
  DBuf<int> d_m16ctr;                  // their hand-out counters (phase 1, phase 2)
  int p16_nparts = 1;                  // parts per leaf in phase 2 (> 1: partial slices + reduce)
  bool p16_ypair = false;              // phase 2 over pairs of leaves (hmv16_y2_kernel)
  int p16_row0 = 0, p16_row1 = 0;      // internal row positions covered by the leaves
  DBuf<double> d_y16part;              // [part][16 RHS][3][rows] partial slices
  long long p16_zsize = 0, p16_alen = 0;
  int n_zch16 = 0, n_yst16 = 0;
  DBuf<ZChunk16> d_zch16;
  DBuf<ZTask16> d_ztask16;
  DBuf<M16Stage> d_yst16;
  DBuf<YItem16> d_yitem16;
  DBuf<M16Copy> d_ycopy16;
  DBuf<int> d_zcoff16, d_ycoff16;
  DBuf<double> d_z16buf, d_xp16;
  DBuf<AdmBlock> d_ablocks;
  DBuf<int> d_pleaf_ptr;
  std::vector<int> p_leaf_ptr;

  // ---- multi-GPU block-row sharding (hmgpu_comm_*, hmgpu_matvec_dist) ----
  int comm_kind = 0;  // 0 none, 1 NCCL (own), 2 NCCL (borrowed), 3 host callbacks
  int comm_n = 1, comm_rank = 0;
  ncclComm_t nccl = nullptr;
  hmgpu_comm_ops comm_ops{};
  std::vector<int> dist_rb, dist_len;  // row range of every rank
  int dist_maxseg = 0;
  DBuf<int> d_segperm, d_dist_rb, d_dist_len;
  DBuf<double> d_ysend, d_yrecv;
  PinnedVec<char> h_stage_a, h_stage_b;  // host-callback staging
  // where the matvec writes its rows: (rperm, n_rows) = external y; the
  // distributed product points this at the shard's segment map instead
  const int* out_perm = nullptr;
  int out_nrows = 0;

  // ---- profiling ----
  bool prof = false;
  std::map<std::string, KTime> times;
  std::vector<PendingEv> pending;
  std::vector<cudaEvent_t> ev_pool;

  cudaMemPool_t pool = nullptr;

  ~hmgpu_ctx() {
    if (device >= 0) cudaSetDevice(device);
    g_pool = pool;
    g_stream = stream;
    for (auto& p : pending) {
      ev_pool.push_back(p.a);
      ev_pool.push_back(p.b);
    }
    for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
    d_rowpt.free(); d_colpt.free(); d_tri.free(); d_A.free();
    if (stream) cudaStreamSynchronize(stream);
    d_rperm.free(); d_cperm.free(); d_items.free(); d_arena.free(); spare_arena.free();
    d_piv.free(); d_cons.free(); d_dense.free(); d_dblocks.free();
    d_counter.free(); d_overflow.free(); d_list.free(); d_mvb.free();
    d_mvorder.free(); d_leaf_begin.free(); d_leaf_end.free();
    d_leaf_ptr.free(); d_leaf_prow.free(); d_leaf_blk.free(); d_x.free(); d_y.free();
    d_xi.free(); d_ypart.free();
    d_pjobs.free(); d_pchunks.free(); d_pwoff.free(); d_zpart.free(); d_mvctr.free();
    d_pentries.free(); d_pleaf_ptr.free();
    d_zch16.free(); d_ztask16.free(); d_yst16.free(); d_zcoff16.free(); d_ycoff16.free(); d_m16ctr.free(); d_y16part.free();
    d_yitem16.free(); d_ycopy16.free();
    d_z16buf.free(); d_xp16.free(); d_ablocks.free();
    d_row_leaf.free(); d_sortp.free(); d_tix.free(); d_term_bi.free(); d_cnt.free();
    d_ptr.free(); d_lists.free(); d_order.free(); d_idx.free(); d_marked.free(); d_nm.free();
    d_mids.free(); d_spoff.free(); d_aterms.free(); d_aout.free(); d_diff.free();
    d_resid.free(); d_nsq.free(); d_sc.free(); d_keys.free(); d_keys2.free();
    d_inset.free(); d_cub.free(); d_eptr.free(); d_eidx.free(); d_eval.free(); d_ecnt.free();
    d_prule.free(); d_vtx.free(); d_tvid.free(); d_tvx.free(); d_tce.free(); d_tna.free();
    d_vtptr.free(); d_vttri.free(); d_tprow.free(); d_tleaf_prow.free(); d_tleaf_begin.free();
    d_tleaf_end.free(); d_tleaf_ptr.free(); d_tpart.free(); d_xr.free();
    w_keys.free(); w_skeys.free(); w_slots.free(); w_sslots.free(); w_gslot.free();
    w_rb.free(); w_dots.free();
    d_segperm.free(); d_dist_rb.free(); d_dist_len.free(); d_ysend.free(); d_yrecv.free();
    if (stream) cudaStreamSynchronize(stream);
    if (comm_kind == 1 && nccl) nccl_api().CommDestroy(nccl);
    if (pool) {
      std::lock_guard<std::mutex> lk(g_pools_mu);
      for (size_t i = 0; i < g_pools.size(); ++i)
        if (g_pools[i].first == pool) {
          g_pools.erase(g_pools.begin() + i);
          break;
        }
    }
    if (pool) cudaMemPoolDestroy(pool);
    g_pool = nullptr;
    g_stream = nullptr;
    if (stream) cudaStreamDestroy(stream);
  }

  const int* yperm() const { return out_perm ? out_perm : d_rperm.p; }
  int ynrows() const { return out_perm ? out_nrows : n_rows; }
  int ndof_rows() const { return n_rows * (NC == 6 ? 3 : 1); }
  int ndof_cols() const { return n_cols * (NC == 6 ? 3 : 1); }

  cudaEvent_t ev() {
    if (!ev_pool.empty()) {
      cudaEvent_t e = ev_pool.back();
      ev_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    return e;
  }
  // brackets a launch with events when profiling is on
  template <class F>
  void timed(const char* name, F&& launch) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (prof) {
      a = ev();
      b = ev();
      CK(cudaEventRecord(a, stream));
    }
    launch();
    CK(cudaGetLastError());
    if (prof) {
      CK(cudaEventRecord(b, stream));
      pending.push_back({name, a, b});
    }
  }
  void resolve_times() {
    for (auto& p : pending) {
      CK(cudaEventSynchronize(p.b));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, p.a, p.b));
      KTime& t = times[p.name];
      t.ms += ms;
      t.launches += 1;
      ev_pool.push_back(p.a);
      ev_pool.push_back(p.b);
    }
    pending.clear();
  }
  void sync() { CK(cudaStreamSynchronize(stream)); }
};

namespace {

template <class F>
int guard(hmgpu_ctx* c, F&& f) {
  if (!c) return HMGPU_ERR_INVALID;
  try {
    if (c->device >= 0) CK(cudaSetDevice(c->device));
    g_pool = c->pool;
    g_stream = c->stream;
    f();
    return HMGPU_OK;
  } catch (const Fail& e) {
    c->err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    c->err = "host allocation failed";
    return HMGPU_ERR_OOM;
  } catch (const std::exception& e) {
    c->err = e.what();
    return HMGPU_ERR_INVALID;
  }
}

bool verbose() {
  static const bool v = std::getenv("HMGPU_VERBOSE") != nullptr;
  return v;
}

int grid_for(hmgpu_ctx* c, long long work, int per_sm = 8) {
  const long long g = std::min<long long>(work, (long long)c->sm_count * per_sm);
  return (int)std::max<long long>(1, g);
}

// ---- device geometry in internal order ------------------------------------
void build_geometry(hmgpu_ctx* c) {
  Geom g{};
  g.kind = c->kind;
  // evaluation points are never the column triangles' centroids (no self term)
  g.same_tree = c->same_tree && c->eval_pts.empty() ? 1 : 0;
  c->d_rperm.upload(c->rperm, c->stream);
  c->d_cperm.upload(c->cperm, c->stream);
  g.rperm = c->d_rperm.p;
  g.cperm = c->d_cperm.p;
  if (c->kind == KIND_KELVIN || c->kind == KIND_GALERKIN) {
    const bool pts = c->kind == KIND_KELVIN && !c->eval_pts.empty();
    const long long nrow_geo = pts ? (long long)c->eval_pts.size() / 3 : c->n_tri;
    if (nrow_geo != c->n_rows || c->n_tri != c->n_cols)
      fail(HMGPU_ERR_DIMENSION, "triangle geometry does not match the partition");
    const double* rsrc = pts ? c->eval_pts.data() : c->centroid.data();
    std::vector<double4> rp(c->n_rows);
    for (int i = 0; i < c->n_rows; ++i) {
      const int t = c->rperm[i];
      rp[i] = make_double4(rsrc[3LL * t], rsrc[3LL * t + 1], rsrc[3LL * t + 2], 0.0);
    }
    // tiles of 32 triangles x 16 field slots (TriRef in hmgpu_device.cuh)
    const long long ntile = (c->n_cols + 31) / 32;
    std::vector<double> tr(ntile * 512, 0.0);
    for (int j = 0; j < c->n_cols; ++j) {
      const int t = c->cperm[j];
      const double* v0 = &c->verts[3LL * c->tris[3 * t]];
      const double* v1 = &c->verts[3LL * c->tris[3 * t + 1]];
      const double* v2 = &c->verts[3LL * c->tris[3 * t + 2]];
      double* T = &tr[(long long)(j >> 5) * 512 + (j & 31)];
      for (int d = 0; d < 3; ++d) {
        T[32 * d] = v0[d];
        T[32 * (3 + d)] = v1[d] - v0[d];
        T[32 * (6 + d)] = v2[d] - v0[d];
        T[32 * (9 + d)] = c->centroid[3 * t + d];
      }
      T[32 * 12] = c->area[t];
      T[32 * 13] = c->diam[t];
    }
    c->d_rowpt.upload(rp, c->stream);
    c->d_tri.upload(tr, c->stream);
    g.rowpt = c->d_rowpt.p;
    g.tri = c->d_tri.p;
    // c = (1+nu) / (8 pi E (1-nu)) in the reference's evaluation order
    g.cst = (1.0 + c->nu) / (8.0 * M_PI * c->E * (1.0 - c->nu));
    g.c34 = 3.0 - 4.0 * c->nu;
    if (c->kind == KIND_GALERKIN) {
      if (!c->same_tree) fail(HMGPU_ERR_DIMENSION, "galerkin needs one triangle tree");
      std::vector<double4> vx(c->n_vert);
      for (int v = 0; v < c->n_vert; ++v)
        vx[v] = make_double4(c->verts[3LL * v], c->verts[3LL * v + 1], c->verts[3LL * v + 2], 0);
      std::vector<int4> tv(c->n_rows);
      for (int i = 0; i < c->n_rows; ++i) {
        const int t = c->rperm[i];
        tv[i] = make_int4(c->tris[3 * t], c->tris[3 * t + 1], c->tris[3 * t + 2], t);
      }
      long long total = 0;
      for (int pc = 1; pc < 4; ++pc) {
        if (c->prule_n[pc] == 0) fail(HMGPU_ERR_STATE, "galerkin pair rule missing");
        g.pr_off[pc] = (int)total;
        g.pr_n[pc] = c->prule_n[pc];
        total += c->prule_n[pc];
      }
      std::vector<double> pr(5 * total);
      for (int pc = 1; pc < 4; ++pc)
        for (int f = 0; f < 5; ++f)
          std::copy(c->prule[pc].begin() + (long long)f * c->prule_n[pc],
                    c->prule[pc].begin() + (long long)(f + 1) * c->prule_n[pc],
                    pr.begin() + f * total + g.pr_off[pc]);
      c->d_vtx.upload(vx, c->stream);
      c->d_tvid.upload(tv, c->stream);
      c->d_prule.upload(pr, c->stream);
      g.vtx = c->d_vtx.p;
      g.tvid = c->d_tvid.p;
      g.prule = c->d_prule.p;
      g.prule_total = total;
      g.gal_delta = c->gal_which;
    }
  } else if (c->kind == KIND_KDELTA || c->kind == KIND_KDOUBLE) {
    const bool dbl = c->kind == KIND_KDOUBLE;
    const long long nrow_geo = dbl ? (long long)c->eval_pts.size() / 3 : c->n_tri;
    if (nrow_geo != c->n_rows || c->n_vert != c->n_cols)
      fail(HMGPU_ERR_DIMENSION, "node geometry does not match the partition");
    std::vector<double4> vx(c->n_vert), tce(c->n_tri), tna(c->n_tri);
    for (int v = 0; v < c->n_vert; ++v)
      vx[v] = make_double4(c->verts[3LL * v], c->verts[3LL * v + 1], c->verts[3LL * v + 2], 0);
    std::vector<int4> tvx(c->n_tri), tv(c->n_rows);
    for (int t = 0; t < c->n_tri; ++t) {
      tvx[t] = make_int4(c->tris[3 * t], c->tris[3 * t + 1], c->tris[3 * t + 2], t);
      tce[t] = make_double4(c->centroid[3 * t], c->centroid[3 * t + 1], c->centroid[3 * t + 2],
                            c->diam[t]);
      tna[t] = make_double4(c->normals[3 * t], c->normals[3 * t + 1], c->normals[3 * t + 2],
                            c->area[t]);
    }
    if (!dbl)
      for (int i = 0; i < c->n_rows; ++i) tv[i] = tvx[c->rperm[i]];
    // vertex_triangles (mesh.cpp:245-247) per internal column, ascending ids
    std::vector<std::vector<int2>> inc(c->n_vert);
    for (int t = 0; t < c->n_tri; ++t)
      for (int k = 0; k < 3; ++k) inc[c->tris[3 * t + k]].push_back(make_int2(t, k));
    std::vector<int> ptr(c->n_cols + 1, 0);
    std::vector<int2> lst;
    for (int j = 0; j < c->n_cols; ++j) {
      const auto& l = inc[c->cperm[j]];
      lst.insert(lst.end(), l.begin(), l.end());
      ptr[j + 1] = (int)lst.size();
    }
    long long total = 0;
    std::vector<double> pr;
    if (!dbl) {
      for (int pc = 1; pc < 4; ++pc) {
        if (c->prule_n[pc] == 0) fail(HMGPU_ERR_STATE, "galerkin pair rule missing");
        g.pr_off[pc] = (int)total;
        g.pr_n[pc] = c->prule_n[pc];
        total += c->prule_n[pc];
      }
      pr.resize(5 * total);
      for (int pc = 1; pc < 4; ++pc)
        for (int f = 0; f < 5; ++f)
          std::copy(c->prule[pc].begin() + (long long)f * c->prule_n[pc],
                    c->prule[pc].begin() + (long long)(f + 1) * c->prule_n[pc],
                    pr.begin() + f * total + g.pr_off[pc]);
    } else {
      std::vector<double4> rp(c->n_rows);
      for (int i = 0; i < c->n_rows; ++i) {
        const long long t = c->rperm[i];
        rp[i] = make_double4(c->eval_pts[3 * t], c->eval_pts[3 * t + 1],
                             c->eval_pts[3 * t + 2], 0.0);
      }
      c->d_rowpt.upload(rp, c->stream);
      g.rowpt = c->d_rowpt.p;
      // lame_constants (kernels.cpp:7-14) and the traction constants
      const double lam = c->E * c->nu / ((1.0 + c->nu) * (1.0 - 2.0 * c->nu));
      const double mu = c->E / (2.0 * (1.0 + c->nu));
      g.cst = (1.0 + c->nu) / (8.0 * M_PI * c->E * (1.0 - c->nu));
      g.c34 = 3.0 - 4.0 * c->nu;
      g.dl_b1 = 2.0 * mu - 2.0 * lam * (1.0 - 2.0 * c->nu);
      g.dl_a2 = mu * (1.0 - g.c34);
      g.dl_a6 = 6.0 * mu;
      g.dl_r = c->dl_r;
      g.dl_c = c->dl_c;
      tv.assign(1, make_int4(0, 0, 0, 0));
      pr.assign(5, 0.0);
    }
    c->d_vtx.upload(vx, c->stream);
    c->d_tvid.upload(tv, c->stream);
    c->d_tvx.upload(tvx, c->stream);
    c->d_tce.upload(tce, c->stream);
    c->d_tna.upload(tna, c->stream);
    c->d_vtptr.upload(ptr, c->stream);
    c->d_vttri.upload(lst, c->stream);
    c->d_prule.upload(pr, c->stream);
    g.vtx = c->d_vtx.p;
    g.tvid = c->d_tvid.p;
    g.tvx = c->d_tvx.p;
    g.tce = c->d_tce.p;
    g.tna = c->d_tna.p;
    g.vt_ptr = c->d_vtptr.p;
    g.vt_tri = c->d_vttri.p;
    g.prule = c->d_prule.p;
    g.prule_total = total;
  } else if (c->kind == KIND_NEWTON) {
    if (c->n_pts != c->n_rows || c->n_pts != c->n_cols)
      fail(HMGPU_ERR_DIMENSION, "points do not match the partition");
    std::vector<double4> rp(c->n_rows), cp(c->n_cols);
    for (int i = 0; i < c->n_rows; ++i) {
      const int t = c->rperm[i];
      rp[i] = make_double4(c->pts[3 * t], c->pts[3 * t + 1], c->pts[3 * t + 2], 0);
    }
    for (int j = 0; j < c->n_cols; ++j) {
      const int t = c->cperm[j];
      cp[j] = make_double4(c->pts[3 * t], c->pts[3 * t + 1], c->pts[3 * t + 2], 0);
    }
    c->d_rowpt.upload(rp, c->stream);
    c->d_colpt.upload(cp, c->stream);
    g.rowpt = c->d_rowpt.p;
    g.colpt = c->d_colpt.p;
    g.diag = c->diag;
  } else if (c->kind == KIND_DENSE) {
    if (c->am != c->n_rows || c->an != c->n_cols)
      fail(HMGPU_ERR_DIMENSION, "matrix does not match the partition");
    c->d_A.upload(c->amat, c->stream);
    g.A = c->d_A.p;
    g.lda = c->am;
  } else {
    fail(HMGPU_ERR_STATE, "no entry provider set");
  }
  c->geom = g;
}

void upload_rules(hmgpu_ctx* c) {
  for (int t = 0; t < 3; ++t)
    if (!c->rules_set[t]) fail(HMGPU_ERR_STATE, "quadrature rule tier missing");
  CK(cudaMemcpyToSymbolAsync(c_rules, &c->rules, sizeof(RuleTable), 0,
                             cudaMemcpyHostToDevice, c->stream));
}

// ---- ACA launch with capacity regrow ---------------------------------------
// Grows the U/V arena so that `extra` more doubles fit at its end.
void arena_reserve(hmgpu_ctx* c, long long extra_doubles, long long extra_piv) {
  const long long need = c->arena_used + extra_doubles;
  if (need > (long long)c->d_arena.n) {
    c->sync();  // mapping is synchronous with the host
    try {
      c->d_arena.ensure((size_t)need, c->device);
    } catch (const Fail& f) {
      // out of memory with the idle compaction arena still mapped (it only
      // hosts the stream / 16-RHS plans, rebuilt on the next matvec): give
      // it back and retry
      if (f.code != HMGPU_ERR_OOM || c->spare_arena.mapped == 0) throw;
      c->spare_arena.free();
      c->plan_valid = false;
      c->p16_valid = false;
      if (verbose()) std::fprintf(stderr, "[hmgpu] arena: idle spare arena released\n");
      c->d_arena.ensure((size_t)need, c->device);
    }
  }
  const long long needp = c->piv_used + extra_piv;
  if (needp > (long long)c->d_piv.n) {
    DBuf<int2> nb;
    nb.alloc((size_t)std::max<long long>(needp, (long long)(c->d_piv.n * 3 / 2)));
    if (c->piv_used)
      CK(cudaMemcpyAsync(nb.p, c->d_piv.p, c->piv_used * sizeof(int2),
                         cudaMemcpyDeviceToDevice, c->stream));
    c->sync();
    c->d_piv.free();
    c->d_piv = nb;
  }
}

void download_items(hmgpu_ctx* c) {
  if (c->items.empty()) return;
  CK(cudaMemcpyAsync(c->items.data(), c->d_items.p, c->items.size() * sizeof(Item),
                     cudaMemcpyDeviceToHost, c->stream));
  c->sync();
}

// refreshes the host mirror of the items in `ids` only
void download_items_subset(hmgpu_ctx* c, const std::vector<int>& ids) {
  if (ids.empty()) return;
  if (ids.size() * 4 > c->items.size()) {
    download_items(c);
    return;
  }
  DBuf<int> d_ids;
  DBuf<Item> d_out;
  d_ids.upload(ids, c->stream);
  d_out.alloc(ids.size());
  gather_items_kernel<<<(int)((ids.size() + 255) / 256), 256, 0, c->stream>>>(
      c->d_items.p, d_ids.p, (int)ids.size(), d_out.p);
  CK(cudaGetLastError());
  std::vector<Item> h(ids.size());
  CK(cudaMemcpyAsync(h.data(), d_out.p, ids.size() * sizeof(Item), cudaMemcpyDeviceToHost,
                     c->stream));
  c->sync();
  for (size_t t = 0; t < ids.size(); ++t) c->items[ids[t]] = h[t];
  d_ids.free();
  d_out.free();
}

// moves `ids` to fresh storage at the arena end with `caps` columns
void relocate(hmgpu_ctx* c, const std::vector<int>& ids, const std::vector<int>& caps) {
  if (ids.empty()) return;
  auto w0 = std::chrono::steady_clock::now();
  auto phase = [&](const char* what) {
    if (!verbose()) return;
    c->sync();
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[hmgpu] relocate %-8s %9.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - w0).count());
    w0 = now;
  };
  long long extra = 0, extrap = 0;
  std::vector<long long> nu(ids.size()), nv(ids.size()), np(ids.size());
  for (size_t t = 0; t < ids.size(); ++t) {
    const Item& it = c->items[ids[t]];
    nu[t] = c->arena_used + extra;
    extra += align2((long long)it.m * caps[t]);
    nv[t] = c->arena_used + extra;
    extra += align2((long long)it.n * caps[t]);
    np[t] = c->piv_used + extrap;
    extrap += caps[t];
  }
  phase("host");
  arena_reserve(c, extra, extrap);
  phase("reserve");
  DBuf<int> d_ids, d_caps;
  DBuf<long long> d_nu, d_nv, d_np;
  d_ids.upload(ids, c->stream);
  d_caps.upload(caps, c->stream);
  d_nu.upload(nu, c->stream);
  d_nv.upload(nv, c->stream);
  d_np.upload(np, c->stream);
  phase("upload");
  c->timed("relocate", [&] {
    relocate_kernel<<<grid_for(c, (long long)ids.size() / 8 + 1), 256, 0, c->stream>>>(
        c->d_items.p, d_ids.p, d_nu.p, d_nv.p, d_np.p, d_caps.p, (int)ids.size(),
        c->d_arena.p, c->d_arena.p, c->d_piv.p, c->d_piv.p);
  });
  c->arena_used += extra;
  c->piv_used += extrap;
  c->sync();
  phase("kernel");
  d_ids.free(); d_caps.free(); d_nu.free(); d_nv.free(); d_np.free();
}

// runs the ACA state machines of `list` to completion, regrowing the column
// capacity of items that run out of it (resume is exact: same state)
// items with m + n at or above this run CTA-cooperatively (aca_kernel)
int aca_cta_min() {
  static const int v = [] {
    const char* e = std::getenv("HMGPU_ACA_CTA_MIN");
    return e ? std::atoi(e) : 1024;
  }();
  return v;
}

// CTAs that take the CTA-cooperative items: all (default) or
// HMGPU_ACA_BIG_CTAS per SM
int aca_big_ctas(hmgpu_ctx* c, int grid) {
  static const int per_sm = [] {
    const char* e = std::getenv("HMGPU_ACA_BIG_CTAS");
    return e ? std::atoi(e) : 0;
  }();
  return per_sm > 0 ? std::min(grid, per_sm * c->sm_count) : grid;
}

// `list` is ordered by m + n (largest first); mn(idx) gives an item's m + n
template <class MN>
void run_aca(hmgpu_ctx* c, std::vector<int> list, int* relaunches, MN&& mn) {
  const double sf = c->eps * (1.0 - c->beta) / (1.0 + c->eps);  // aca.cpp:114
  int passes = 0;
  while (!list.empty()) {
    c->d_list.upload(list, c->stream);
    CK(cudaMemsetAsync(c->d_counter.p, 0, 2 * sizeof(int), c->stream));
    CK(cudaMemsetAsync(c->d_overflow.p, 0, sizeof(int), c->stream));
    int nbig = 0;
    while (nbig < (int)list.size() && mn(list[nbig]) >= aca_cta_min()) ++nbig;
    const int nwarps = (int)list.size();
    const int grid = grid_for(c, std::max(nbig, (nwarps + 7) / 8), 16);
    // HMGPU_ACA_TRACE=<file>: per-item completion times of this launch
    // (diagnostics: item size, mode and end time relative to the first)
    static const char* trace = std::getenv("HMGPU_ACA_TRACE");
    DBuf<unsigned long long> d_trace;
    if (trace) {
      d_trace.alloc(c->items.size());
      CK(cudaMemsetAsync(d_trace.p, 0, c->items.size() * 8, c->stream));
      unsigned long long* pt = d_trace.p;
      CK(cudaMemcpyToSymbolAsync(g_aca_trace, &pt, sizeof(pt), 0, cudaMemcpyHostToDevice,
                                 c->stream));
    }
    c->timed("aca", [&] {
      auto go = [&](auto kernel) {
        kernel<<<grid, ACA_NT, 0, c->stream>>>(
            c->geom, c->d_items.p, c->d_list.p, (int)list.size(), nbig, c->d_counter.p,
            c->d_arena.p, c->d_piv.p, c->d_cons.p, sf, c->max_rank, c->lookahead,
            c->d_overflow.p, aca_big_ctas(c, grid));
      };
      if (c->kind == KIND_KELVIN) go(aca_kernel<KIND_KELVIN>);
      else if (c->kind == KIND_GALERKIN) go(aca_kernel<KIND_GALERKIN>);
      else if (c->kind == KIND_KDELTA) go(aca_kernel<KIND_KDELTA>);
      else if (c->kind == KIND_KDOUBLE) go(aca_kernel<KIND_KDOUBLE>);
      else if (c->kind == KIND_NEWTON) go(aca_kernel<KIND_NEWTON>);
      else go(aca_kernel<KIND_DENSE>);
    });
    int over = 0;
    CK(cudaMemcpyAsync(&over, c->d_overflow.p, sizeof(int), cudaMemcpyDeviceToHost,
                       c->stream));
    c->sync();
    if (trace) {
      std::vector<unsigned long long> tt(c->items.size());
      CK(cudaMemcpy(tt.data(), d_trace.p, tt.size() * 8, cudaMemcpyDeviceToHost));
      unsigned long long* nullp = nullptr;
      CK(cudaMemcpyToSymbol(g_aca_trace, &nullp, sizeof(nullp)));
      unsigned long long t0 = ~0ull;
      for (int idx : list)
        if (tt[idx]) t0 = std::min(t0, tt[idx]);
      if (FILE* f = std::fopen(trace, passes == 0 ? "w" : "a")) {
        std::fprintf(f, "# pass %d nbig %d grid %d\n", passes, nbig, grid);
        for (size_t q = 0; q < list.size(); ++q) {
          const int idx = list[q];
          std::fprintf(f, "%d %d %d %d %.3f\n", (int)q, c->items[idx].m, c->items[idx].n,
                       (int)(q < (size_t)nbig), tt[idx] ? (tt[idx] - t0) * 1e-6 : -1.0);
        }
        std::fclose(f);
      }
      d_trace.free();
    }
    if (over == 0) break;
    ++passes;
    if (verbose())
      std::fprintf(stderr, "[hmgpu] aca overflow: pass %d, %zu items in the launch\n", passes,
                   list.size());
    download_items_subset(c, list);
    std::vector<int> ids, caps;
    for (int idx : list) {
      const Item& it = c->items[idx];
      if (it.status != ST_OVERFLOW) continue;
      const long long capr = std::min<long long>(c->max_rank, std::min(it.m, it.n));
      ids.push_back(idx);
      caps.push_back((int)std::min<long long>(capr, std::max(2 * it.cap, it.cap + 8)));
    }
    relocate(c, ids, caps);
    list = ids;
  }
  if (relaunches) *relaunches += passes;
}

// packs the arena: every item gets exactly K (+ slack) columns.  Sizes, a
// CUB exclusive scan for the new offsets and the copies all run on the
// device; the item mirror comes back once (pinned).
void compact(hmgpu_ctx* c, int slack) {
  const int ni = (int)c->items.size();
  if (ni == 0) return;
  DBuf<long long> usz, psz, uoff, poff;
  DBuf<int> caps;
  usz.alloc(ni);
  psz.alloc(ni);
  uoff.alloc(ni + 1);
  poff.alloc(ni + 1);
  caps.alloc(ni);
  const int grid = (ni + 255) / 256;
  compact_sizes_kernel<<<grid, 256, 0, c->stream>>>(c->d_items.p, ni, c->max_rank, slack,
                                                    usz.p, psz.p, caps.p);
  CK(cudaGetLastError());
  size_t tmp_bytes = 0, t2 = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, usz.p, uoff.p, ni + 0, c->stream));
  CK(cub::DeviceScan::ExclusiveSum(nullptr, t2, psz.p, poff.p, ni + 0, c->stream));
  DBuf<uint8_t> tmp;
  tmp.alloc(std::max(tmp_bytes, t2));
  CK(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, usz.p, uoff.p, ni, c->stream));
  CK(cub::DeviceScan::ExclusiveSum(tmp.p, t2, psz.p, poff.p, ni, c->stream));
  long long last[4];
  CK(cudaMemcpyAsync(&last[0], uoff.p + ni - 1, sizeof(long long), cudaMemcpyDeviceToHost,
                     c->stream));
  CK(cudaMemcpyAsync(&last[1], usz.p + ni - 1, sizeof(long long), cudaMemcpyDeviceToHost,
                     c->stream));
  CK(cudaMemcpyAsync(&last[2], poff.p + ni - 1, sizeof(long long), cudaMemcpyDeviceToHost,
                     c->stream));
  CK(cudaMemcpyAsync(&last[3], psz.p + ni - 1, sizeof(long long), cudaMemcpyDeviceToHost,
                     c->stream));
  c->sync();
  tmp.free();
  usz.free();
  psz.free();
  const long long used = last[0] + last[1], usedp = last[2] + last[3];
  const size_t free_b = avail_bytes() + c->spare_arena.mapped;
  if (8.0 * (double)used + 8.0 * (double)usedp > 0.9 * (double)free_b) {
    uoff.free();
    poff.free();
    caps.free();
    download_items(c);  // not enough room for the packed copy: keep the loose arena
    return;
  }
  VArena na = std::move(c->spare_arena);  // reuse the previous mapping
  na.ensure((size_t)used + 2, c->device);
  DBuf<int2> npv;
  npv.alloc((size_t)usedp + 1);
  c->timed("compact", [&] {
    compact_kernel<<<grid_for(c, (long long)ni / 8 + 1), 256, 0, c->stream>>>(
        c->d_items.p, ni, uoff.p, poff.p, caps.p, c->d_arena.p, na.p, c->d_piv.p, npv.p);
  });
  c->sync();
  uoff.free();
  poff.free();
  caps.free();
  c->d_arena = std::move(na);       // `na` now holds the loose arena: kept
  c->spare_arena = std::move(na);   // mapped, it hosts the matvec stream arena
  c->arena_used = used;
  c->d_piv.free();
  c->d_piv = npv;
  c->piv_used = usedp;
  download_items(c);
}

// block-row matvec work lists and the leaf reduction CSR
// Host tables of the matvec that depend on the partition only (owned blocks,
// partial-row offsets, leaves of the row tree and their covering blocks): no
// CUDA call and no rank in here, so hmgpu_assemble runs it on a host thread
// while the ACA kernel works (it was 12 of the assembly call's 45 ms of wall
// time at config 2).
void build_matvec_tables(hmgpu_ctx* c) {
  c->mvb.clear();
  long long prow = 0;
  for (int b = 0; b < c->n_blocks; ++b) {
    const int* B = &c->blocks[4 * b];
    const int* rn = &c->rnodes[4 * B[0]];
    const int* cn = &c->cnodes[4 * B[1]];
    if (rn[0] < c->row_begin || rn[1] > c->row_end) continue;
    MvBlock mb{};
    mb.m = rn[1] - rn[0];
    mb.n = cn[1] - cn[0];
    mb.row0 = rn[0];
    mb.col0 = cn[0];
    mb.dense = B[2] ? 0 : 1;
    mb.item0 = c->item_of_block[b];
    mb.dense_off = mb.dense ? c->dblocks[c->dense_of_block[b]].off : 0;
    mb.prow = prow;
    prow += mb.m;
    c->mvb.push_back(mb);
  }
  c->part_rows = prow;
  c->n_mv = (int)c->mvb.size();

  // leaves of the row tree inside the shard, in index order
  c->leaf_begin.clear();
  c->leaf_end.clear();
  const int nrn = (int)c->rnodes.size() / 4;
  for (int t = 0; t < nrn; ++t) {
    const int* nd = &c->rnodes[4 * t];
    if (nd[2] >= 0) continue;
    if (nd[0] < c->row_begin || nd[1] > c->row_end) continue;
    c->leaf_begin.push_back(nd[0]);
    c->leaf_end.push_back(nd[1]);
  }
  std::vector<int> lorder(c->leaf_begin.size());
  std::iota(lorder.begin(), lorder.end(), 0);
  std::sort(lorder.begin(), lorder.end(),
            [&](int a, int b) { return c->leaf_begin[a] < c->leaf_begin[b]; });
  std::vector<int> lb(lorder.size()), le(lorder.size());
  for (size_t i = 0; i < lorder.size(); ++i) {
    lb[i] = c->leaf_begin[lorder[i]];
    le[i] = c->leaf_end[lorder[i]];
  }
  c->leaf_begin = lb;
  c->leaf_end = le;
  const int nl = (int)lb.size();
  // two passes over the blocks (count, fill) instead of a vector per leaf
  std::vector<int> cnt(nl + 1, 0);
  auto leaves_of = [&](const MvBlock& mb, auto&& f) {
    int l0 = (int)(std::lower_bound(lb.begin(), lb.end(), mb.row0) - lb.begin());
    for (int l = l0; l < nl && lb[l] < mb.row0 + mb.m; ++l) {
      if (le[l] > mb.row0 + mb.m)
        fail(HMGPU_ERR_INVALID, "block rows do not align with row-tree leaves");
      f(l);
    }
  };
  for (const MvBlock& mb : c->mvb) leaves_of(mb, [&](int l) { ++cnt[l + 1]; });
  c->leaf_ptr.assign(nl + 1, 0);
  for (int l = 0; l < nl; ++l) c->leaf_ptr[l + 1] = c->leaf_ptr[l] + cnt[l + 1];
  c->leaf_prow.assign((size_t)c->leaf_ptr[nl], 0);
  c->leaf_blk.assign((size_t)c->leaf_ptr[nl], make_int2(0, 0));
  std::vector<int> fill(c->leaf_ptr.begin(), c->leaf_ptr.end() - 1);
  for (int bi = 0; bi < (int)c->mvb.size(); ++bi) {
    const MvBlock& mb = c->mvb[bi];
    leaves_of(mb, [&](int l) {
      const int o = fill[l]++;
      c->leaf_prow[o] = mb.prow + (lb[l] - mb.row0);
      c->leaf_blk[o] = make_int2(bi, lb[l] - mb.row0);
    });
  }
}

// The rank-dependent part (block order by bytes, kmax) and the uploads.
void build_matvec_finish(hmgpu_ctx* c) {
  c->kmax = 1;
  std::vector<long long> bytes(c->mvb.size());
  for (size_t b = 0; b < c->mvb.size(); ++b) {
    const MvBlock& mb = c->mvb[b];
    long long by = 0;
    if (mb.dense) {
      by = (long long)c->NC * mb.m * mb.n;
    } else {
      for (int q = 0; q < c->NC; ++q) {
        const Item& it = c->items[mb.item0 + q];
        by += (long long)it.k * (mb.m + mb.n);
        c->kmax = std::max(c->kmax, it.k);
      }
    }
    bytes[b] = by;
  }
  std::vector<int> order(c->n_mv);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return bytes[a] > bytes[b]; });
  c->d_mvb.upload(c->mvb, c->stream);
  c->d_mvorder.upload(order, c->stream);
  c->d_leaf_begin.upload(c->leaf_begin, c->stream);
  c->d_leaf_end.upload(c->leaf_end, c->stream);
  c->d_leaf_ptr.upload(c->leaf_ptr, c->stream);
  c->d_leaf_blk.upload(c->leaf_blk, c->stream);
  c->am_geom_valid = false;
  c->am_have_estimate = false;
  c->t_valid = false;
  c->d_leaf_prow.upload(c->leaf_prow, c->stream);
  c->sync();
}

// tables of the transposed matvec: a partial-row range per owned block over
// its column cluster, and per column-tree leaf the covering blocks in block
// order (deterministic reduction)
void build_matvec_t(hmgpu_ctx* c) {
  std::vector<long long> tprow(c->mvb.size());
  long long t = 0;
  for (size_t b = 0; b < c->mvb.size(); ++b) {
    tprow[b] = t;
    t += c->mvb[b].n;
  }
  c->t_rows = t;
  std::vector<int> lb, le;
  const int ncn = (int)c->cnodes.size() / 4;
  for (int q = 0; q < ncn; ++q) {
    const int* nd = &c->cnodes[4 * q];
    if (nd[2] >= 0) continue;
    lb.push_back(nd[0]);
    le.push_back(nd[1]);
  }
  std::vector<int> ord(lb.size());
  std::iota(ord.begin(), ord.end(), 0);
  std::sort(ord.begin(), ord.end(), [&](int a, int b) { return lb[a] < lb[b]; });
  std::vector<int> b2(lb.size()), e2(lb.size());
  for (size_t i = 0; i < ord.size(); ++i) {
    b2[i] = lb[ord[i]];
    e2[i] = le[ord[i]];
  }
  const int nl = (int)b2.size();
  std::vector<std::vector<long long>> lists(nl);
  for (size_t bi = 0; bi < c->mvb.size(); ++bi) {
    const MvBlock& mb = c->mvb[bi];
    int l0 = (int)(std::lower_bound(b2.begin(), b2.end(), mb.col0) - b2.begin());
    for (int l = l0; l < nl && b2[l] < mb.col0 + mb.n; ++l) {
      if (e2[l] > mb.col0 + mb.n)
        fail(HMGPU_ERR_INVALID, "block columns do not align with column-tree leaves");
      lists[l].push_back(tprow[bi] + (b2[l] - mb.col0));
    }
  }
  std::vector<int> ptr(nl + 1, 0);
  std::vector<long long> prow;
  for (int l = 0; l < nl; ++l) {
    ptr[l + 1] = ptr[l] + (int)lists[l].size();
    prow.insert(prow.end(), lists[l].begin(), lists[l].end());
  }
  c->t_nleaves = nl;
  c->d_tprow.upload(tprow, c->stream);
  c->d_tleaf_begin.upload(b2, c->stream);
  c->d_tleaf_end.upload(e2, c->stream);
  c->d_tleaf_ptr.upload(ptr, c->stream);
  c->d_tleaf_prow.upload(prow, c->stream);
  c->sync();
  c->t_valid = true;
}

// refresh kmax after rank changes (promote / extend)

// ---- streamed matvec plan (warp-private jobs, hmgpu_stream.cuh) -------------
// Default geometry of the warp pipelines (tuned on B200 with
// scripts/mv_sweep.sh: 12 warps per SM, two 7 KB stages each, 4.7 KB of job
// scratch -- more warps hide the FMA/shared-memory latency of the FUSED jobs;
// deeper rings and scratch below ~4.5 KB lost).  HMGPU_MV_CFG=
// "warps,stages,stage_doubles,scratch_doubles" overrides it for tuning.
struct MvCfg {
  int warps = 12, ns = 2, stage = 896, scratch = 600;
};
// pass 0 (FUSED / DENSE / VSPLIT jobs) and pass 1 (USPLIT); HMGPU_MV_CFG sets
// both, HMGPU_MV_CFG_A / HMGPU_MV_CFG_B one pass
MvCfg parse_mv_cfg(const char* e, MvCfg c) {
  int w, n, s, k;
  if (e && std::sscanf(e, "%d,%d,%d,%d", &w, &n, &s, &k) == 4) {
    c.warps = w;
    c.ns = n;
    c.stage = s;
    c.scratch = k;
  }
  return c;
}
MvCfg mv_cfg(int pass) {
  static const MvCfg both = parse_mv_cfg(std::getenv("HMGPU_MV_CFG"), MvCfg{});
  static const MvCfg a = parse_mv_cfg(std::getenv("HMGPU_MV_CFG_A"), both);
  static const MvCfg b = parse_mv_cfg(std::getenv("HMGPU_MV_CFG_B"), both);
  return pass == 0 ? a : b;
}

// HMGPU_MV_VROWS=0: FUSED V parts in column chunks only (A/B switch)
bool vrows_off() {
  static const bool off = [] {
    const char* e = std::getenv("HMGPU_MV_VROWS");
    return e && e[0] == '0';
  }();
  return off;
}

// streamed bytes (doubles) per chain unit of the matvec plan; 0 = automatic
// (HMGPU_MV_UNIT overrides, for tuning)
// HMGPU_MV_LAYOUT (both passes), HMGPU_MV_LAYOUT_A / _B (one pass):
// 0 automatic, 1 contiguous runs, 2 round-robin units
int mv_layout(int pass) {
  static const int both = [] {
    const char* e = std::getenv("HMGPU_MV_LAYOUT");
    return e ? std::atoi(e) : 0;
  }();
  static const int a = [] {
    const char* e = std::getenv("HMGPU_MV_LAYOUT_A");
    return e ? std::atoi(e) : both;
  }();
  static const int b = [] {
    const char* e = std::getenv("HMGPU_MV_LAYOUT_B");
    return e ? std::atoi(e) : both;
  }();
  return pass == 0 ? a : b;
}
// share of a pass's bytes (its smallest chain units) handed out dynamically
// after the static shares (HMGPU_MV_POOL, per cent; 0 = all static)
double mv_pool_frac() {
  static const double v = [] {
    const char* e = std::getenv("HMGPU_MV_POOL");
    const double pc = e ? std::atof(e) : 12.5;
    return pc < 0.0 || pc > 90.0 ? 0.125 : pc / 100.0;
  }();
  return v;
}
long long mv_unit_cap() {
  static const long long v = [] {
    const char* e = std::getenv("HMGPU_MV_UNIT");
    return e ? std::max(0LL, std::atoll(e)) : 0LL;
  }();
  return v;
}

void build_plan(hmgpu_ctx* c, int mode, int nrhs) {
  if (nrhs != 1) fail(HMGPU_ERR_INVALID, "streamed matvec: single right-hand side");
  c->p16_valid = false;  // the stream arena takes the spare arena the p16 plan used
  auto tp0 = std::chrono::steady_clock::now();
  auto pphase = [&](const char* what) {
    if (!verbose()) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[hmgpu] plan %-10s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - tp0).count());
    tp0 = now;
  };
  const MvCfg cfg = mv_cfg(0), cfgB = mv_cfg(1);
  const int kStageData = cfg.stage - 16;  // data + aux after the descriptor header
  const int kStageDataB = cfgB.stage - 16;
  const int kMaxKFused = (cfg.scratch - 256) / 4;  // scratch: x (256) + W (4 K)
  const int NC = c->NC;
  fast_vector<WJob> ja, jb;
  // chunks per job, flat (CSR over the pass's jobs)
  struct ChunkCSR {
    fast_vector<WChunk> flat;
    fast_vector<long long> ptr{0};
    fast_vector<long long> size;  // streamed doubles per job
    void add(const std::vector<WChunk>& chs) {
      long long s = 0;
      for (const WChunk& ch : chs) s += ch.len + 4LL * ch.aux_len;
      flat.insert(flat.end(), chs.begin(), chs.end());
      ptr.push_back((long long)flat.size());
      size.push_back(s);
    }
  } ca, cb;
  std::vector<WChunk> chs;  // the current job's chunks (reused)
  fast_vector<PackDesc> packs;
  ja.reserve(c->mvb.size() * 2);
  ca.flat.reserve(c->mvb.size() * 6);
  ca.ptr.reserve(c->mvb.size() * 2);
  ca.size.reserve(c->mvb.size() * 2);
  packs.reserve(c->mvb.size() * 12);
  long long alen = 0, slots = 0, wslots = 0;
  const int nl = (int)c->leaf_begin.size();
  std::vector<std::vector<LeafEntry>> lists(nl);
  auto add_rows = [&](int r_lo, int nrows, long long slot) {
    const int r_hi = r_lo + nrows;
    int l = (int)(std::upper_bound(c->leaf_begin.begin(), c->leaf_begin.end(), r_lo) -
                  c->leaf_begin.begin()) - 1;
    for (l = std::max(l, 0); l < nl && c->leaf_begin[l] < r_hi; ++l) {
      const int lb = c->leaf_begin[l], le = c->leaf_end[l];
      const int lo = std::max(lb, r_lo), hi = std::min(le, r_hi);
      if (lo >= hi) continue;
      lists[l].push_back(LeafEntry{slot + (lo - r_lo), lo - lb, hi - lb});
    }
  };
  auto chunk = [](long long src, int len, int src_kind, int aux_kind, long long aux,
                  int aux_len, int g0, int g1, int part) {
    WChunk ch{};
    ch.src = src;
    ch.len = (int)align2(len);
    ch.src_kind = src_kind;
    ch.aux_kind = aux_kind;
    ch.aux = aux;
    ch.aux_len = aux_len;
    ch.g0 = g0;
    ch.g1 = g1;
    ch.part = part;
    return ch;
  };
  // the blocks' jobs, chunks and pack descriptors, built by host threads over
  // contiguous block ranges with local arena / W-slot offsets, then
  // concatenated in range order with the offsets shifted (the same tables as
  // one sequential pass)
  struct Local {
    fast_vector<WJob> ja, jb;
    ChunkCSR ca, cb;
    fast_vector<PackDesc> packs;
    std::vector<WChunk> chs;
    long long alen = 0, wslots = 0;
    std::exception_ptr err;
  };
  auto run_range = [&](Local& Lc, size_t b0, size_t b1) {
    auto& ja = Lc.ja;
    auto& jb = Lc.jb;
    auto& ca = Lc.ca;
    auto& cb = Lc.cb;
    auto& packs = Lc.packs;
    auto& chs = Lc.chs;
    long long& alen = Lc.alen;
    long long& wslots = Lc.wslots;
    for (size_t bi = b0; bi < b1; ++bi) {
      const MvBlock& mb = c->mvb[bi];
    const int m = mb.m, n = mb.n;
    if (mb.dense) {
      if (m > 64 || n > 64)
        fail(HMGPU_ERR_INVALID, "near-field block larger than 64 for the streamed matvec");
      const int cp = (int)align2((long long)NC * m);
      const int cpc = std::max(1, (kStageData - 4 * n) / cp);
      WJob j{};
      j.kind = WJ_DENSE;
      j.m = m;
      j.n = n;
      j.ncols = n;
      j.row0 = mb.row0;
      chs.clear();
      for (int g0 = 0; g0 < n; g0 += cpc) {
        const int g1 = std::min(n, g0 + cpc);
        chs.push_back(chunk(mb.dense_off + (long long)g0 * cp, (g1 - g0) * cp, 1,
                            g0 == 0 ? WA_X : WA_NONE, mb.col0, g0 == 0 ? n : 0, g0, g1, 0));
      }
      ja.push_back(j);
      ca.add(chs);
      continue;
    }
    int k[6] = {0, 0, 0, 0, 0, 0};
    int K = 0;
    for (int q = 0; q < NC; ++q) {
      const Item& it = c->items[mb.item0 + q];
      k[q] = mode ? it.k : it.kcur;
      K += k[q];
    }
    if (K == 0) continue;
    int kp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int q = 0; q < 6; ++q) kp[q + 1] = kp[q] + (q < NC ? k[q] : 0);
    kp[7] = kp[6];
    if (m <= 64 && n <= 64 && K <= kMaxKFused) {
      WJob j{};
      j.kind = WJ_FUSED;
      j.m = m;
      j.n = n;
      j.ncols = K;
      j.row0 = mb.row0;
      std::copy(kp, kp + 8, j.kp);
      chs.clear();
      // V part, K <= 64: row chunks over all K columns (row-major [j][g]),
      // x rows with each chunk -- every lane busy (two columns per lane
      // above 32) instead of column chunks of the stage width
      if (K <= 64 && !vrows_off()) {
        j.vrows = 1;
        const int rpc = std::max(1, kStageData / (K + 4));
        for (int r0 = 0; r0 < n; r0 += rpc) {
          const int r1 = std::min(n, r0 + rpc);
          const long long off = alen;
          for (int q = 0; q < NC; ++q) {
            const int a = kp[q], b = kp[q + 1];
            if (a >= b) continue;
            packs.push_back(PackDesc{c->items[mb.item0 + q].v_off + r0, off + a, n, K, r1 - r0,
                                     b - a, 1, 0});
          }
          alen += align2((long long)(r1 - r0) * K);
          chs.push_back(chunk(off, (r1 - r0) * K, 0, WA_X, mb.col0 + r0, r1 - r0, r0, r1, 0));
        }
      }
      // V part, K > 64: row-major [j][g] chunks over whole columns, x rides along
      const int vcpc = std::max(1, (kStageData - 4 * n) / n);
      for (int g0 = 0; g0 < K && !j.vrows; g0 += vcpc) {
        const int g1 = std::min(K, g0 + vcpc);
        // the chunk's columns may span components: pack per component piece
        const long long off = alen;
        const int w = g1 - g0;  // row length of the row-major [j][g] tile
        for (int q = 0; q < NC; ++q) {
          const int a = std::max(g0, kp[q]), b = std::min(g1, kp[q + 1]);
          if (a >= b) continue;
          packs.push_back(PackDesc{c->items[mb.item0 + q].v_off + (long long)(a - kp[q]) * n,
                                   off + (a - g0), n, w, n, b - a, 1, 0});
        }
        alen += align2((long long)n * w);
        chs.push_back(chunk(off, n * w, 0, g0 == 0 ? WA_X : WA_NONE, mb.col0, g0 == 0 ? n : 0,
                            g0, g1, 0));
      }
      // U part: column-major [g][i] chunks
      const int ucpc = std::max(1, kStageData / m);
      for (int g0 = 0; g0 < K; g0 += ucpc) {
        const int g1 = std::min(K, g0 + ucpc);
        const long long off = alen;
        for (int q = 0; q < NC; ++q) {
          const int a = std::max(g0, kp[q]), b = std::min(g1, kp[q + 1]);
          if (a >= b) continue;
          packs.push_back(PackDesc{c->items[mb.item0 + q].u_off + (long long)(a - kp[q]) * m,
                                   off + (long long)(a - g0) * m, m, m, m, b - a, 0, 0});
        }
        alen += align2((long long)m * (g1 - g0));
        chs.push_back(chunk(off, m * (g1 - g0), 0, WA_NONE, 0, 0, g0, g1, 1));
      }
      ja.push_back(j);
      ca.add(chs);
      continue;
    }
    // split block: VSPLIT groups of <= 64 consecutive columns of the K
    // (component-major, balanced) -> W (global, the same slot order)
    const long long wbase = wslots;
    wslots += K;
    const int ngr = (K + 63) / 64, per = (K + ngr - 1) / ngr;
    for (int g0 = 0; g0 < K; g0 += per) {
      const int g1 = std::min(K, g0 + per), nc = g1 - g0;
      const int rpc = std::max(1, kStageData / (nc + 4));
      WJob j{};
      j.kind = WJ_VSPLIT;
      j.n = n;
      j.ncols = nc;
      j.comp = g0;
      std::copy(kp, kp + 8, j.kp);
      j.out = wbase + g0;
      j.row0 = -1;
      chs.clear();
      for (int r0 = 0; r0 < n; r0 += rpc) {
        const int r1 = std::min(n, r0 + rpc);
        const long long off = alen;  // row-major [j][g] tile, per component piece
        for (int q = 0; q < NC; ++q) {
          const int a = std::max(g0, kp[q]), b = std::min(g1, kp[q + 1]);
          if (a >= b) continue;
          packs.push_back(PackDesc{c->items[mb.item0 + q].v_off + r0 +
                                       (long long)(a - kp[q]) * n,
                                   off + (a - g0), n, nc, r1 - r0, b - a, 1, 0});
        }
        alen += align2((long long)(r1 - r0) * nc);
        chs.push_back(chunk(off, (r1 - r0) * nc, 0, WA_X, mb.col0 + r0, r1 - r0, r0, r1, 0));
      }
      ja.push_back(j);
      ca.add(chs);
    }
    // USPLIT row tiles over component groups whose W fits the warp scratch
    for (int q0 = 0; q0 < NC;) {
      int q1 = q0, kg = 0;
      while (q1 < NC && 4 * (kg + k[q1]) <= cfgB.scratch &&
             4 * (kg + k[q1]) <= kStageDataB / 2)
        kg += k[q1++];
      if (q1 == q0) fail(HMGPU_ERR_INVALID, "rank too large for the streamed matvec");
      if (kg == 0) {
        q0 = q1;
        continue;
      }
      int gkp[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // prefix sums restricted to the group
      for (int q = 0; q < 6; ++q) gkp[q + 1] = gkp[q] + (q >= q0 && q < q1 ? k[q] : 0);
      gkp[7] = gkp[6];
      for (int i0 = 0; i0 < m; i0 += 64) {
        const int rt = std::min(64, m - i0);
        WJob j{};
        j.kind = WJ_USPLIT;
        j.m = rt;
        j.ncols = kg;
        j.row0 = mb.row0 + i0;
        std::copy(gkp, gkp + 8, j.kp);
        chs.clear();
        const int first_cols = std::max(1, (kStageDataB - 4 * kg) / rt);
        const int cols = std::max(1, kStageDataB / rt);
        for (int g0 = 0; g0 < kg;) {
          const int g1 = std::min(kg, g0 + (g0 == 0 ? first_cols : cols));
          const long long off = alen;
          for (int q = q0; q < q1; ++q) {
            const int a = std::max(g0, gkp[q]), b = std::min(g1, gkp[q + 1]);
            if (a >= b) continue;
            packs.push_back(PackDesc{c->items[mb.item0 + q].u_off + i0 +
                                         (long long)(a - gkp[q]) * m,
                                     off + (long long)(a - g0) * rt, m, rt, rt, b - a, 0, 0});
          }
          alen += align2((long long)rt * (g1 - g0));
          chs.push_back(chunk(off, rt * (g1 - g0), 0, g0 == 0 ? WA_W : WA_NONE,
                              wbase + kp[q0], g0 == 0 ? kg : 0, g0, g1, 1));
          g0 = g1;
        }
        jb.push_back(j);
        cb.add(chs);
      }
      q0 = q1;
    }
      }
  };
  {
    const size_t nb = c->mvb.size();
    const int nthr = (int)std::max<size_t>(
        1, std::min<size_t>({(size_t)std::max(1u, std::thread::hardware_concurrency()),
                             (size_t)16, nb / 2048 + 1}));
    std::vector<Local> loc(nthr);
    std::vector<std::thread> pool;
    for (int t = 0; t < nthr; ++t) {
      const size_t b0 = nb * t / nthr, b1 = nb * (t + 1) / nthr;
      auto work = [&, t, b0, b1] {
        try {
          run_range(loc[t], b0, b1);
        } catch (...) {
          loc[t].err = std::current_exception();
        }
      };
      if (t + 1 < nthr) pool.emplace_back(work);
      else work();
    }
    for (auto& th : pool) th.join();
    for (auto& Lc : loc)
      if (Lc.err) std::rethrow_exception(Lc.err);
    // offsets of every thread's part in the concatenated tables, then each
    // thread shifts and copies its own part (in parallel)
    struct Off {
      size_t ja, jb, caf, cap, cbf, cbp, pk;
      long long alen, wslots;
    };
    std::vector<Off> off(nthr + 1);
    off[0] = Off{0, 0, 0, 1, 0, 1, 0, 0, 0};
    for (int t = 0; t < nthr; ++t) {
      const Local& Lc = loc[t];
      off[t + 1] = Off{off[t].ja + Lc.ja.size(), off[t].jb + Lc.jb.size(),
                       off[t].caf + Lc.ca.flat.size(), off[t].cap + Lc.ca.ptr.size() - 1,
                       off[t].cbf + Lc.cb.flat.size(), off[t].cbp + Lc.cb.ptr.size() - 1,
                       off[t].pk + Lc.packs.size(), off[t].alen + Lc.alen,
                       off[t].wslots + Lc.wslots};
    }
    const Off& tot = off[nthr];
    ja.resize(tot.ja);
    jb.resize(tot.jb);
    ca.flat.resize(tot.caf);
    ca.ptr.resize(tot.cap);
    ca.size.resize(tot.cap - 1);
    cb.flat.resize(tot.cbf);
    cb.ptr.resize(tot.cbp);
    cb.size.resize(tot.cbp - 1);
    packs.resize(tot.pk);
    ca.ptr[0] = 0;
    cb.ptr[0] = 0;
    auto place = [&](int t) {
      Local& Lc = loc[t];
      const Off& o = off[t];
      for (size_t i = 0; i < Lc.ja.size(); ++i) {
        WJob j = Lc.ja[i];
        if (j.kind == WJ_VSPLIT) j.out += o.wslots;
        ja[o.ja + i] = j;
      }
      std::copy(Lc.jb.begin(), Lc.jb.end(), jb.begin() + o.jb);
      auto put = [&](ChunkCSR& dst, const ChunkCSR& src, size_t fo, size_t po) {
        for (size_t i = 0; i < src.flat.size(); ++i) {
          WChunk ch = src.flat[i];
          if (ch.src_kind == 0) ch.src += o.alen;
          if (ch.aux_kind == WA_W) ch.aux += o.wslots;
          dst.flat[fo + i] = ch;
        }
        for (size_t i = 1; i < src.ptr.size(); ++i) dst.ptr[po + i - 1] = (long long)fo + src.ptr[i];
        std::copy(src.size.begin(), src.size.end(), dst.size.begin() + (po - 1));
      };
      put(ca, Lc.ca, o.caf, o.cap);
      put(cb, Lc.cb, o.cbf, o.cbp);
      for (size_t i = 0; i < Lc.packs.size(); ++i) {
        PackDesc pd = Lc.packs[i];
        pd.dst += o.alen;
        packs[o.pk + i] = pd;
      }
      Lc = Local{};
    };
    pool.clear();
    for (int t = 0; t + 1 < nthr; ++t) pool.emplace_back(place, t);
    place(nthr - 1);
    for (auto& th : pool) th.join();
    alen = tot.alen;
    wslots = tot.wslots;
  }
  pphase("blocks");
  // Job order per pass: the row jobs by (first row, rows) -- stable LSD
  // counting sorts, so a block row's jobs are adjacent -- then the VSPLIT
  // jobs.  Consecutive jobs on the same rows form chain units that one warp
  // runs back to back, accumulating in registers and writing ONE partial
  // row (the leaf pass then sums a few units per leaf instead of one partial
  // row per block).
  auto order = [&](const fast_vector<WJob>& J) {
    const size_t nj = J.size();
    std::vector<int> a(nj), b(nj);
    std::vector<int> cnt(66, 0);
    for (size_t i = 0; i < nj; ++i) ++cnt[J[i].row0 < 0 ? 0 : 1 + std::min(J[i].m, 64)];
    for (int k = 0, run = 0; k < 66; ++k) {
      const int t = cnt[k];
      cnt[k] = run;
      run += t;
    }
    for (size_t i = 0; i < nj; ++i) a[cnt[J[i].row0 < 0 ? 0 : 1 + std::min(J[i].m, 64)]++] = (int)i;
    std::vector<int> cr((size_t)c->n_rows + 2, 0);
    for (int i : a) ++cr[J[i].row0 < 0 ? (size_t)c->n_rows + 1 : (size_t)J[i].row0];
    for (size_t k = 0, run = 0; k < cr.size(); ++k) {
      const int t = cr[k];
      cr[k] = (int)run;
      run += t;
    }
    for (int i : a) b[cr[J[i].row0 < 0 ? (size_t)c->n_rows + 1 : (size_t)J[i].row0]++] = i;
    return b;
  };
  std::vector<WJob> jobs;
  std::vector<int> woff;
  const size_t nchunks_total = ca.flat.size() + cb.flat.size();
  fast_vector<WChunk> chunk_table(nchunks_total);
  WChunk* chunks = chunk_table.data();
  size_t nch = 0;
  for (int pass = 0; pass < 2; ++pass) {
    const int NWARPS = c->sm_count * (pass == 0 ? cfg.warps : cfgB.warps);
    auto& J = pass == 0 ? ja : jb;
    const ChunkCSR& C = pass == 0 ? ca : cb;
    const std::vector<int> ord = order(J);
    const size_t nj = ord.size();
    long long total = 0;
    for (int idx : ord) total += C.size[idx];
    // Chain units: runs of row jobs on the same rows (VSPLIT jobs: one unit
    // each).  Two layouts (measured):
    //  * a warp's share of the pass >= 2 MB (C3, C4): each warp streams one
    //    contiguous run of the order (1/NWARPS of the bytes, sequential
    //    pages), units cut at run ends;
    //  * smaller shares (C2: 1.6 MB, where one job is a sizeable part of a
    //    share): units cut at ~1/16 of a share, dealt round-robin largest
    //    first over the warps (the balance of a size-sorted round-robin).
    const bool contiguous =
        mv_layout(pass) == 1 || (mv_layout(pass) == 0 && total / NWARPS >= (2LL << 20) / 8);
    const long long cap = contiguous ? (1LL << 62)
                          : mv_unit_cap() > 0 ? mv_unit_cap()
                                              : std::max<long long>(4096, total / NWARPS / 16);
    std::vector<int> owner(nj, 0);
    if (contiguous) {
      const double share = std::max(1.0, (double)total / NWARPS);
      long long cum = 0;
      for (size_t t = 0; t < nj; ++t) {
        const long long sz = C.size[ord[t]];
        owner[t] = (int)std::min<double>(NWARPS - 1, std::floor((cum + 0.5 * sz) / share));
        cum += sz;
      }
    }
    std::vector<size_t> ubeg;  // unit u = ord positions [ubeg[u], ubeg[u + 1])
    std::vector<long long> usize;
    for (size_t t = 0; t < nj; ++t) {
      const WJob& q = J[ord[t]];
      const bool open = !ubeg.empty() && q.row0 >= 0 && usize.back() < cap &&
                        owner[t] == owner[t - 1] && J[ord[t - 1]].row0 == q.row0 &&
                        J[ord[t - 1]].m == q.m;
      if (!open) {
        ubeg.push_back(t);
        usize.push_back(0);
      }
      usize.back() += C.size[ord[t]];
    }
    const size_t nu = ubeg.size();
    ubeg.push_back(nj);
    std::vector<int> uord(nu);  // units in emission order
    std::iota(uord.begin(), uord.end(), 0);
    std::vector<int> uwarp(nu);
    if (contiguous) {
      for (size_t u = 0; u < nu; ++u) uwarp[u] = owner[ubeg[u]];
    } else {
      std::stable_sort(uord.begin(), uord.end(),
                       [&](int x, int y) { return usize[x] > usize[y]; });
      for (size_t i = 0; i < nu; ++i) uwarp[uord[i]] = (int)(i % NWARPS);
    }
    // Static shares leave the warps 86-90 % busy at config 2 (a warp's pace
    // depends on its SM neighbours, not only on its bytes), and handing
    // everything out dynamically loses the locality of a warp's run.  So the
    // round-robin layout keeps the SMALLEST units -- the last ~1/8 of the
    // bytes in the size-sorted order -- out of the static deal: they form a
    // pool of groups the warps pull from a global counter once their own
    // share is done.  ipool = first pooled position of uord.
    size_t ipool = nu;
    if (!contiguous && mv_pool_frac() > 0.0) {
      long long tail = 0;
      while (ipool > 0 && (double)(tail + usize[uord[ipool - 1]]) <= mv_pool_frac() * (double)total)
        tail += usize[uord[--ipool]];
      ipool -= ipool % (size_t)NWARPS;  // whole rounds of the static deal
    }
    std::vector<int> jpos(nj);  // ord position -> job table index
    for (size_t i = 0; i < nu; ++i) {
      const int u = uord[i];
      for (size_t t = ubeg[u]; t < ubeg[u + 1]; ++t) {
        jpos[t] = (int)jobs.size();
        WJob jt = J[ord[t]];
        if (jt.row0 >= 0) {
          if (t == ubeg[u]) {  // the unit's partial row
            add_rows(jt.row0, jt.m, slots);
            slots += jt.m;
          }
          jt.out = slots - jt.m;
          jt.chain = t + 1 < ubeg[u + 1];
        }
        jobs.push_back(jt);
      }
    }
    // per warp, its units in emission order (CSR over warps)
    std::vector<int> wptr(NWARPS + 1, 0), wunits(nu);
    for (size_t i = 0; i < ipool; ++i) ++wptr[uwarp[uord[i]] + 1];
    for (int w = 0; w < NWARPS; ++w) wptr[w + 1] += wptr[w];
    {
      std::vector<int> fill(wptr.begin(), wptr.end() - 1);
      for (size_t i = 0; i < ipool; ++i) wunits[fill[uwarp[uord[i]]]++] = uord[i];
    }
    pphase(pass == 0 ? "layout A/u" : "layout B/u");
    c->p_woff_base[pass] = (int)woff.size();
    c->p_chunk_base[pass] = (int)nch;
    // per warp its chunk count, the offsets, then the copies by host
    // threads over warp ranges (the table is the sequential one)
    std::vector<long long> wstart(NWARPS + 1, 0);
    for (int w = 0; w < NWARPS; ++w) {
      long long cnt = 0;
      for (int k = wptr[w]; k < wptr[w + 1]; ++k) {
        const int u = wunits[k];
        for (size_t t = ubeg[u]; t < ubeg[u + 1]; ++t) cnt += C.ptr[ord[t] + 1] - C.ptr[ord[t]];
      }
      wstart[w + 1] = wstart[w] + cnt;
      woff.push_back((int)wstart[w]);
    }
    {
      const int nthr = std::max(1, std::min<int>((int)std::max(1u, std::thread::hardware_concurrency()),
                                                 std::min(16, NWARPS)));
      auto fill = [&](int w0, int w1) {
        for (int w = w0; w < w1; ++w) {
          long long o = (long long)nch + wstart[w];
          for (int k = wptr[w]; k < wptr[w + 1]; ++k) {
            const int u = wunits[k];
            for (size_t t = ubeg[u]; t < ubeg[u + 1]; ++t) {
              for (long long q = C.ptr[ord[t]]; q < C.ptr[ord[t] + 1]; ++q) {
                WChunk ch = C.flat[q];
                ch.job = jpos[t];
                chunks[o++] = ch;
              }
            }
          }
        }
      };
      std::vector<std::thread> th;
      for (int t = 0; t + 1 < nthr; ++t)
        th.emplace_back(fill, NWARPS * t / nthr, NWARPS * (t + 1) / nthr);
      fill(NWARPS * (nthr - 1) / nthr, NWARPS);
      for (auto& x : th) x.join();
    }
    woff.push_back((int)wstart[NWARPS]);
    // the pool: its units in size order after the static part, in groups of
    // >= 1/64 of a share (offsets relative to the pass's chunks)
    {
      long long o = wstart[NWARPS];
      const long long gsize = std::max<long long>(2048, total / NWARPS / 64);
      long long acc = 0;
      int ngroups = 0;
      for (size_t i = ipool; i < nu; ++i) {
        if (i == ipool || acc >= gsize) {
          woff.push_back((int)o);
          ++ngroups;
          acc = 0;
        }
        const int u = uord[i];
        acc += usize[u];
        for (size_t t = ubeg[u]; t < ubeg[u + 1]; ++t)
          for (long long q = C.ptr[ord[t]]; q < C.ptr[ord[t] + 1]; ++q) {
            WChunk ch = C.flat[q];
            ch.job = jpos[t];
            chunks[nch + o++] = ch;
          }
      }
      woff.push_back((int)o);
      c->p_ngroups_pass[pass] = ngroups;
      nch += (size_t)o;
    }
    c->p_nwarps_pass[pass] = NWARPS;
  }
  c->p_nwarps = c->p_nwarps_pass[0];
  pphase("layout");
  std::vector<LeafEntry> entries;
  c->p_leaf_ptr.assign(nl + 1, 0);
  for (int l = 0; l < nl; ++l) {
    entries.insert(entries.end(), lists[l].begin(), lists[l].end());
    c->p_leaf_ptr[l + 1] = (int)entries.size();
  }
  pphase("entries");
  // the stream arena lives in the idle arena of the last compaction (the
  // loose ACA layout): no new device memory is mapped for it in steady state
  c->sync();
  c->spare_arena.ensure((size_t)alen + 2, c->device);
  if (!packs.empty()) {
    DBuf<PackDesc> d_packs;
    d_packs.upload(packs.data(), packs.size(), c->stream);
    c->timed("pack", [&] {
      pack_kernel<<<grid_for(c, ((long long)packs.size() + 7) / 8, 16), 256, 0, c->stream>>>(
          d_packs.p, (int)packs.size(), c->d_arena.p, c->spare_arena.p);
    });
    c->sync();
    d_packs.free();
  }
  pphase("pack");
  c->d_pjobs.upload(jobs, c->stream);
  c->d_pchunks.upload(chunks, nch, c->stream);
  c->d_pwoff.upload(woff, c->stream);
  c->d_pentries.upload(entries, c->stream);
  c->d_pleaf_ptr.upload(c->p_leaf_ptr, c->stream);
  c->p_ntasks = (int)jobs.size();
  c->p_nz = (int)ja.size();  // pass A = [0, p_nz), pass B = USPLIT
  c->p_njb = (int)jb.size();
  c->p_slots = slots;
  c->p_zslots = wslots;
  c->p_arena_len = alen;
  c->p_smem = sizeof(double) * (size_t)cfg.warps * (cfg.ns * cfg.stage + cfg.scratch);
  c->p_smem_pass[0] = c->p_smem;
  c->p_smem_pass[1] = sizeof(double) * (size_t)cfgB.warps * (cfgB.ns * cfgB.stage + cfgB.scratch);
  c->plan_mode = mode;
  c->plan_nrhs = nrhs;
  c->plan_valid = true;
  c->sync();
  pphase("upload");
  if (verbose())
    std::fprintf(stderr, "[hmgpu] plan: jobs=%d (pass A %zu, USPLIT %zu) chunks=%zu "
                         "arena=%.3f GB slots=%lld wslots=%lld entries=%zu smem=%zu B\n",
                 c->p_ntasks, ja.size(), jb.size(), nch, 8.0 * alen / 1e9, slots,
                 wslots, entries.size(), c->p_smem);
}

// ---- multi-RHS plan (hmgpu_mrhs.cuh) ----------------------------------------
// HMGPU_M16_CFG="ns,stage": ring depth (3, 4, 6 or 9) and doubles per stage
struct M16Cfg {  // measured on config 3: 3 x 3072 (3 CTAs / SM) best
  int ns = 3, stage = 0;  // stage 0: 3072 doubles at 3 CTAs per SM, 2304 at 4
  // phase 1 (HMGPU_M16_ZCFG="ns,stage,warps"): its own ring and consumer
  // warps (6, 8 or 12; 6 runs 4 CTAs per SM)
  int zns = 3, zstage = 0, znw = 8;
  // phase-2 consumer warps (HMGPU_M16_YNW: 5, 6, 8 or 16; 0 = from the
  // leaves' row tiles, so that no warp idles through a leaf)
  int ynw = 0;
};
M16Cfg m16_cfg() {
  static const M16Cfg cfg = [] {
    M16Cfg r;
    int a, b, w;
    const char* e = std::getenv("HMGPU_M16_CFG");
    if (e && std::sscanf(e, "%d,%d", &a, &b) == 2) {
      r.ns = a;
      r.stage = b;
      r.zns = a;
      r.zstage = b;
    }
    const char* yw = std::getenv("HMGPU_M16_YNW");
    if (yw) {
      const int v = std::atoi(yw);
      r.ynw = (v == 5 || v == 6 || v == 16) ? v : 8;
    }
    const char* z = std::getenv("HMGPU_M16_ZCFG");
    if (z && std::sscanf(z, "%d,%d,%d", &a, &b, &w) == 3) {
      r.zns = a;
      r.zstage = b;
      r.znw = w;
    }
    return r;
  }();
  return cfg;
}

// Multi-RHS plan: phase-1 tasks (block, <= 64 l of its components) with
// their column chunks, phase-2 stages per leaf, the p16 arena (current-rank
// factors re-packed in stage order, zero padded to the conflict-free
// pitches), the Z layout and the per-CTA runs of both passes.
void build_plan16(hmgpu_ctx* c, int mode) {
  M16Cfg cfg = m16_cfg();
  if (cfg.ynw == 0) {  // consumer warps = row tiles of the tallest leaf
    int rmax = 1;
    for (size_t L = 0; L < c->leaf_begin.size(); ++L)
      rmax = std::max(rmax, c->leaf_end[L] - c->leaf_begin[L]);
    const int rt = (rmax + 7) / 8;
    cfg.ynw = (rt == 6 || rt == 3) ? 6 : (rt == 5 ? 5 : 8);
  }
  // phase 2 over pairs of neighbouring leaves (hmv16_y2_kernel): when the
  // leaves fill their row tiles (rows = 8 warps, so the second leaf's tiles
  // start at a tile boundary) and the warps are not split over RHS halves;
  // HMGPU_M16_PAIR=0 keeps one leaf per unit
  bool ypair = false;
  {
    const char* e = std::getenv("HMGPU_M16_PAIR");
    int rmax = 1;
    for (size_t L = 0; L < c->leaf_begin.size(); ++L)
      rmax = std::max(rmax, c->leaf_end[L] - c->leaf_begin[L]);
    ypair = !(e && std::atoi(e) == 0) && cfg.ynw != 16 && (cfg.ns == 3 || cfg.ns == 4) &&
            rmax == 8 * cfg.ynw &&
            c->leaf_begin.size() >= 2;
  }
  const bool y4 = !ypair && (cfg.ynw == 5 || cfg.ynw == 6);  // 4 CTAs per SM
  if (cfg.stage == 0) {
    cfg.stage = y4 ? 2304 : 3072;
    // phase 1: 8 consumer warps and 3 CTAs per SM (6 warps x 4 CTAs with
    // 2304-double stages was ahead until the loops lost their branches; now
    // 2 % behind, profiles/ab_r02_mrhs_session4.txt)
    if (cfg.zstage == 0) cfg.zstage = cfg.znw == 6 ? 2304 : 3072;
  }
  if ((cfg.ns != 3 && cfg.ns != 4 && cfg.ns != 6 && cfg.ns != 9) || cfg.stage < 2048 || (cfg.stage & 3))
    fail(HMGPU_ERR_INVALID, "bad HMGPU_M16_CFG");
  if ((cfg.zns != 3 && cfg.zns != 4) || (cfg.znw != 6 && cfg.znw != 8 && cfg.znw != 12) || cfg.zstage < 2048 ||
      (cfg.zstage & 3))
    fail(HMGPU_ERR_INVALID, "bad HMGPU_M16_ZCFG");
  const int SD = cfg.zstage - M16_HDR;  // phase-1 data doubles per stage
  const int nb = c->n_mv;
  std::vector<std::array<int, 6>> rk(std::max(nb, 1)), zo(std::max(nb, 1));
  std::vector<long long> zb(std::max(nb, 1), -1);
  long long zsize = 0;
  for (int bi = 0; bi < nb; ++bi) {
    const MvBlock& mb = c->mvb[bi];
    rk[bi].fill(0);
    zo[bi].fill(0);
    if (mb.dense) continue;
    int K = 0, z4 = 0;
    for (int q = 0; q < 6; ++q) {
      const Item& it = c->items[mb.item0 + q];
      const int k = mode ? it.k : it.kcur;
      if (k > 255) fail(HMGPU_ERR_INVALID, "rank above 255 for the multi-RHS sweep");
      rk[bi][q] = k;
      zo[bi][q] = z4;
      z4 += (k + 3) & ~3;
      K += k;
    }
    if (K == 0) continue;
    zb[bi] = zsize;
    zsize += (long long)z4 * ZP;
  }
  std::vector<PackDesc> packs;
  long long alen = 0;

  // ---- phase 1: tasks and their chunks
  std::vector<ZTask16> tasks;
  std::vector<ZChunk16> zch;
  std::vector<long long> tbytes;
  std::vector<int> tptr{0};
  struct Seg {
    int c, lo, hi;
  };
  std::vector<Seg> segs, grp;
  for (int bi = 0; bi < nb; ++bi) {
    if (zb[bi] < 0) continue;
    const MvBlock& mb = c->mvb[bi];
    const int n = mb.n;
    segs.clear();
    for (int q = 0; q < 6; ++q)
      for (int lo = 0; lo < rk[bi][q]; lo += 64)
        segs.push_back({q, lo, std::min(rk[bi][q], lo + 64)});
    size_t si = 0;
    while (si < segs.size()) {
      grp.clear();
      int L = 0;
      while (si < segs.size() && grp.size() < 6 && L + (segs[si].hi - segs[si].lo) <= 64) {
        L += segs[si].hi - segs[si].lo;
        grp.push_back(segs[si++]);
      }
      ZTask16 tk{};
      tk.zdst = zb[bi];
      int vr = 0, grows[3] = {0, 0, 0}, gn[3] = {0, 0, 0};
      static const int kR[6] = {0, 0, 0, 1, 1, 2}, kC[6] = {0, 1, 2, 1, 2, 2};
      for (size_t e = 0; e < grp.size(); ++e) {
        const Seg& sg = grp[e];
        const int len = sg.hi - sg.lo, cr = kR[sg.c], cc = kC[sg.c];
        tk.len[e] = (unsigned char)len;
        tk.vrow[e] = (unsigned char)vr;
        tk.zrow[e] = (short)(zo[bi][sg.c] + sg.lo);
        vr += len;
        // Z_c = V_c^T x_C (part 0); W_c = V_c^T x_R (part 1, off-diagonal)
        tk.gent[cc][gn[cc]++] = (unsigned char)(e << 1);
        grows[cc] += len;
        if (cr != cc) {
          tk.gent[cr][gn[cr]++] = (unsigned char)((e << 1) | 1);
          grows[cr] += len;
        }
      }
      tk.gtile[0] = 0;
      for (int r = 0; r < 3; ++r) {
        tk.gn[r] = (unsigned char)gn[r];
        tk.grows[r] = (unsigned char)grows[r];
        tk.gtile[r + 1] = (unsigned char)(tk.gtile[r] + (grows[r] + 7) / 8);
      }
      tk.ntiles = tk.gtile[3];
      tk.pad0 = L;  // the zero row of the staged V^T
      if (tk.ntiles > 3 * cfg.znw) fail(HMGPU_ERR_INVALID, "multi-RHS task above 3 m-tiles per warp");
      // widest chunk whose V^T and X rows fit one stage
      int jc = std::min(n, 252);
      // (+ 1: a zero row after the V^T rows, read by the padding rows of the m-tiles)
      while (jc > 4 && (long long)(L + 1 + XP) * cf_pitch(jc) > SD) jc -= 4;
      if ((long long)(L + 1 + XP) * cf_pitch(jc) > SD)
        fail(HMGPU_ERR_INVALID, "multi-RHS stage too small");
      const int ti = (int)tasks.size();
      tasks.push_back(tk);
      long long by = 0;
      const int nch = (n + jc - 1) / jc;
      for (int q = 0; q < nch; ++q) {
        const int j0 = q * jc, jj = std::min(jc, n - j0), Pp = cf_pitch(jj);
        ZChunk16 ch{};
        ch.vsrc = alen;
        ch.vlen = (L + 1) * Pp;
        ch.xcol = mb.col0 + j0;
        ch.P = Pp;
        ch.task = ti;
        ch.flags = (q == 0 ? 1 : 0) | (q == nch - 1 ? 2 : 0);
        for (size_t e = 0; e < grp.size(); ++e) {
          const Seg& sg = grp[e];
          packs.push_back(PackDesc{c->items[mb.item0 + sg.c].v_off + (long long)sg.lo * n + j0,
                                   alen + M16_HDR + (long long)tk.vrow[e] * Pp, n, Pp, jj,
                                   sg.hi - sg.lo, 0, 0});
        }
        alen += M16_HDR + (long long)(L + 1) * Pp;  // records, V^T rows, the zero row
        by += (long long)(L + 1) * Pp + (long long)Pp * XP;
        zch.push_back(ch);
      }
      tbytes.push_back(by);
      tptr.push_back((int)zch.size());
    }
  }

  // ---- phase 2: pieces per leaf, the covering blocks in leaf_blk order (each
  // piece fits a stage after the item records)
  const int SDY = cfg.stage - Y16_HDR;
  // A/B switch (timing experiments): HMGPU_M16_SKIP=1 / 2 leaves out the
  // near-field / low-rank pieces (wrong products)
  static const int skip = [] {
    const char* e = std::getenv("HMGPU_M16_SKIP");
    return e ? std::atoi(e) : 0;
  }();
  std::vector<YStage16> yst;
  std::vector<long long> lbytes;
  std::vector<int> lptr{0};
  const int nl = (int)c->leaf_begin.size();
  // groups: one leaf, or (ypair) two neighbouring leaves whose first fills its tiles
  std::vector<int2> groups;  // (first leaf, second leaf or -1)
  for (int L = 0; L < nl;) {
    const int R = c->leaf_end[L] - c->leaf_begin[L];
    if (R > 64) fail(HMGPU_ERR_INVALID, "leaf above 64 rows for the multi-RHS sweep");
    if (ypair && L + 1 < nl && R == 8 * cfg.ynw && c->leaf_end[L] == c->leaf_begin[L + 1] &&
        c->leaf_end[L + 1] - c->leaf_begin[L + 1] <= 8 * cfg.ynw) {
      groups.push_back(make_int2(L, L + 1));
      L += 2;
    } else {
      groups.push_back(make_int2(L, -1));
      L += 1;
    }
  }
  const int ng = (int)groups.size();
  std::vector<int> grows(ng), gb0(ng);
  for (int G = 0; G < ng; ++G) {
    const int LA = groups[G].x, LB = groups[G].y;
    const int RA = c->leaf_end[LA] - c->leaf_begin[LA];
    const int RB = LB >= 0 ? c->leaf_end[LB] - c->leaf_begin[LB] : 0;
    const int rg = RA + RB;
    grows[G] = rg;
    gb0[G] = c->leaf_begin[LA];
    const size_t first = yst.size();
    long long by = 0;
    // the pieces of one block for R rows from row roff of the block: tile
    // slot tsel (0 first leaf, 1 second, 2 both: R = both leaves' rows)
    auto add_block = [&](int bi, int roff, int R, int tsel) {
      const int PR = cf_pitch(R);
      const MvBlock& mb = c->mvb[bi];
      if (mb.dense) {
        if (skip == 1) return;
        const long long cp = align2(6LL * mb.m);
        const int PD = cf_pitch(6 * mb.m);
        // as many columns as fit with their x rows (ceil4 of them); any
        // count: the last k-step is predicated
        int jd = SDY / (PD + XP) + 1;
        while (jd > 0 && (long long)jd * PD + (long long)((jd + 3) & ~3) * XP > SDY) --jd;
        if (jd < 1) fail(HMGPU_ERR_INVALID, "near-field block too tall for the multi-RHS stage");
        // whole k-steps of 4 columns (the last one of a block is predicated);
        // HMGPU_M16_JD4=0: as many columns as fit (A/B)
        static const bool jd4 = [] {
          const char* e = std::getenv("HMGPU_M16_JD4");
          return !(e && std::atoi(e) == 0);
        }();
        if (jd4 && jd > 4) jd &= ~3;
        for (int j0 = 0; j0 < mb.n; j0 += jd) {
          const int jj = std::min(jd, mb.n - j0);
          YStage16 d{};
          d.kind = Y16_DENSE;
          d.leaf = G;
          d.tsel = tsel;
          d.rg = rg;
          d.R = R;
          d.src = mb.dense_off + (long long)j0 * cp;
          d.len = 6 * mb.m;
          d.spitch = (int)cp;
          d.PR = PD;
          d.jd = jj;
          d.src2 = mb.col0 + j0;
          d.len2 = ((jj + 3) & ~3) * XP;
          d.m = mb.m;
          d.roff = roff;
          yst.push_back(d);
          by += (long long)jj * 6 * mb.m + d.len2;
        }
        return;
      }
      if (zb[bi] < 0 || skip == 2) return;
      YStage16 d{};
      bool open = false;
      int used = 0;
      auto flush = [&]() {
        // leaf pairs: a tile's last l-step may load U rows up to 3 PR + 127
        // doubles past the piece (dropped: their A is zero); at least 16 Z rows
        // after the U rows keep those loads inside the item, whatever follows it
        if (ypair && d.len2 < 16 * ZP) d.len2 = 16 * ZP;
        yst.push_back(d);
        by += d.len + d.len2;
        open = false;
      };
      for (int q = 0; q < 6; ++q) {
        const int k = rk[bi][q], k4 = (k + 3) & ~3;
        int lo = 0;
        while (lo < k) {
          if (!open) {
            d = YStage16{};
            d.kind = Y16_ADM;
            d.leaf = G;
          d.tsel = tsel;
          d.rg = rg;
            d.R = R;
            d.PR = PR;
            d.m = RA;  // rows of the first leaf (tsel 2: offset of the second's)
            d.src = alen;
            d.src2 = zb[bi] + (long long)(zo[bi][q] + lo) * ZP;
            used = 0;
            open = true;
          }
          const int left = SDY - used, rest = k - lo;
          int take = rest;
          if ((long long)rest * PR + (long long)(k4 - lo) * ZP > left)
            take = std::min(rest - 1, left / (PR + ZP)) & ~3;
          if (take <= 0) {
            if (used == 0) fail(HMGPU_ERR_INVALID, "multi-RHS stage too small");
            flush();
            continue;
          }
          const int hi = lo + take;
          d.lo[q] = (unsigned char)lo;
          d.hi[q] = (unsigned char)hi;
          packs.push_back(PackDesc{c->items[mb.item0 + q].u_off + (long long)lo * mb.m + roff,
                                   alen, mb.m, PR, R, take, 0, 0});
          alen += (long long)take * PR;
          const int zrows = ((hi + 3) & ~3) - lo;
          d.len += take * PR;
          d.len2 += zrows * ZP;
          used += take * PR + zrows * ZP;
          lo = hi;
          if (hi < k) flush();  // the component continues in the next stage
        }
      }
      if (open) flush();
        };
    if (LB < 0) {
      for (int e = c->leaf_ptr[LA]; e < c->leaf_ptr[LA + 1]; ++e)
        add_block(c->leaf_blk[e].x, c->leaf_blk[e].y, RA, 0);
    } else {
      // blocks covering both leaves (the second's rows follow the first's in
      // the block) take both tile slots; the rest one
      std::unordered_map<int, int> inb;  // block -> row offset of the second leaf
      for (int e = c->leaf_ptr[LB]; e < c->leaf_ptr[LB + 1]; ++e)
        inb[c->leaf_blk[e].x] = c->leaf_blk[e].y;
      for (int e = c->leaf_ptr[LA]; e < c->leaf_ptr[LA + 1]; ++e) {
        const int bi = c->leaf_blk[e].x, roff = c->leaf_blk[e].y;
        auto it = inb.find(bi);
        if (it != inb.end() && it->second == roff + RA && !c->mvb[bi].dense) {
          add_block(bi, roff, RA + RB, 2);
          inb.erase(it);
        } else {
          add_block(bi, roff, RA, 0);
        }
      }
      for (int e = c->leaf_ptr[LB]; e < c->leaf_ptr[LB + 1]; ++e)
        if (inb.count(c->leaf_blk[e].x)) add_block(c->leaf_blk[e].x, c->leaf_blk[e].y, RB, 1);
    }
    if (yst.size() == first) {  // no contribution: the leaf's rows are written as 0
      YStage16 d{};
      d.kind = Y16_ADM;
      d.leaf = G;
      d.R = RA;
      d.PR = cf_pitch(RA);
      d.rg = rg;
      yst.push_back(d);
    }
    lbytes.push_back(std::max<long long>(by, 1));
    lptr.push_back((int)yst.size());
  }
  // A leaf is the unit of the dynamic hand-out, and a pass over few leaves
  // per CTA ends with CTAs idling for up to a leaf's time (config 3: 6.9
  // leaves per CTA, the CTAs 93 % busy; config 2: 1.7 and 73 %).  Below 16
  // units per CTA every leaf's piece list is therefore cut into P parts of
  // about equal bytes; part p accumulates its own rows into slice p of a
  // partial buffer and y16_reduce_kernel adds the slices in part order
  // (deterministic).  P = 1: the leaves write y directly.
  const size_t ring_bytes = ((size_t)cfg.ns * cfg.stage + M16_SLACK) * sizeof(double);
  if (ring_bytes + 1024 > 227 * 1024) fail(HMGPU_ERR_INVALID, "HMGPU_M16_CFG ring too large");
  const int per_sm = cfg.ynw == 16 ? 1
                     : std::max(1, std::min(y4 ? 4 : 3, (int)((227 * 1024) / (ring_bytes + 1024))));
  const int ncta = c->sm_count * per_sm;
  int nparts = 1;
  {
    // HMGPU_M16_PARTS=1..8 forces the count (read per plan: tests and A/B runs)
    const char* fe = std::getenv("HMGPU_M16_PARTS");
    const int forced = fe ? std::atoi(fe) : 0;
    long long total = 0;
    for (long long b : lbytes) total += b;
    nparts = (int)std::min<long long>(8, (16LL * ncta + ng - 1) / std::max(ng, 1));
    // parts of at least 128 KB on average
    nparts = (int)std::min<long long>(nparts, total / std::max(ng, 1) / (128 * 1024 / 8));
    nparts = std::max(nparts, 1);
    if (forced >= 1 && forced <= 8) nparts = forced;
  }
  {
    std::vector<YStage16> parts;
    std::vector<long long> sbytes;
    std::vector<int> sptr{0};
    parts.reserve(yst.size() + (size_t)ng * nparts);
    auto plen0 = [](const YStage16& d) -> long long {
      return d.kind == Y16_ADM ? (long long)d.len + d.len2 : (long long)d.jd * d.PR + d.len2;
    };
    for (int L = 0; L < ng; ++L) {
      long long total = 0;
      for (int q = lptr[L]; q < lptr[L + 1]; ++q) total += plen0(yst[q]);
      long long cum = 0;
      int q = lptr[L];
      for (int pt = 0; pt < nparts; ++pt) {
        const size_t first = parts.size();
        long long by = 0;
        // pieces up to the part's share of the bytes (the last part takes the rest)
        const long long upto = pt == nparts - 1 ? total + 1 : (total * (pt + 1)) / nparts;
        while (q < lptr[L + 1] && (pt == nparts - 1 || cum + plen0(yst[q]) / 2 < upto)) {
          cum += plen0(yst[q]);
          by += plen0(yst[q]);
          parts.push_back(yst[q++]);
        }
        if (parts.size() == first) {  // nothing for this part: its rows are written as 0
          YStage16 d{};
          d.kind = Y16_ADM;
          d.leaf = L;
          d.R = std::min(grows[L], 8 * cfg.ynw);
          d.PR = cf_pitch(d.R);
          d.rg = grows[L];
          parts.push_back(d);
        }
        for (size_t e = first; e < parts.size(); ++e) parts[e].part = pt;
        parts[first].flags |= 1;
        parts.back().flags |= 2;
        sbytes.push_back(std::max<long long>(by, 1));
        sptr.push_back((int)parts.size());
      }
    }
    yst.swap(parts);
    lbytes.swap(sbytes);  // from here on per (leaf, part) segment
    lptr.swap(sptr);
  }
  const int nseg = (int)lbytes.size();

  // ---- per-CTA runs (up to 3 CTAs per SM, as many as their rings fit):
  // phase 1 by tasks, phase 2 by leaves (a leaf's accumulators live in one
  // CTA); within a CTA's leaves, consecutive pieces are packed into stages
  // of up to Y16_MAXIT items, their records and bulk copies
  const size_t zring_bytes = (size_t)cfg.zns * cfg.zstage * sizeof(double);
  if (zring_bytes + 1024 > 227 * 1024) fail(HMGPU_ERR_INVALID, "HMGPU_M16_ZCFG ring too large");
  const int zcta_sm = std::max(1, std::min(cfg.znw == 8 ? 3 : (cfg.znw == 6 ? 4 : 2),
                                           (int)((227 * 1024) / (zring_bytes + 1024))));
  const int nctaz = c->sm_count * zcta_sm;
  // work units handed out dynamically (hmgpu_mrhs.cuh UnitCursor): phase 1 a
  // run of consecutive tasks of >= M16_UNIT_BYTES, phase 2 a run of
  // consecutive leaves of >= M16_UNIT_BYTES (a leaf's accumulators live in
  // one CTA); the units go out in order, so the CTAs work on a window of
  // neighbouring leaves at any time and the Z of the blocks above them is
  // read from L2 by all of them.  zcoff / ycoff: first stage of each unit;
  // the entry after the last unit is the END stage both passes append.
  constexpr long long M16_UNIT_BYTES = 96 * 1024 / 8;  // doubles
  std::vector<int> zcoff, ycoff;
  std::vector<M16Stage> ystages;
  std::vector<YItem16> yitems;
  std::vector<M16Copy> ycopies;
  std::vector<unsigned char> ckind;  // copy source: 0 items, 1 p16 arena, 2 Z, 3 dense, 4 x
  {
    {
      long long acc = 0;
      for (size_t ti = 0; ti < tbytes.size(); ++ti) {
        if (ti == 0 || acc >= M16_UNIT_BYTES) {
          zcoff.push_back(tptr[ti]);
          acc = 0;
        }
        acc += tbytes[ti];
      }
      zcoff.push_back((int)zch.size());  // = END chunk
      ZChunk16 end{};
      end.flags = 4;
      end.vsrc = alen;  // records only
      alen += M16_HDR;
      zch.push_back(end);
    }
    const int SD2 = cfg.stage - Y16_HDR;
    auto plen = [](const YStage16& d) -> long long {
      return d.kind == Y16_ADM ? (long long)d.len + d.len2 : (long long)d.jd * d.PR + d.len2;
    };
    auto copy = [&](int kind, long long src_bytes, long long dst, long long bytes) {
      // Z (2) and x (4) are re-read by many stages: kept in L2 (evict last)
      const int keep = (kind == 2 || kind == 4) ? M16_KEEP : 0;
      ycopies.push_back(M16Copy{(unsigned long long)src_bytes, (int)dst | keep, (int)bytes});
      ckind.push_back((unsigned char)kind);
    };
    std::vector<std::vector<int>> cleaves;  // (leaf, part) segments of each unit
    {
      long long acc = 0;
      for (int L = 0; L < nseg; ++L) {
        if (L == 0 || acc >= M16_UNIT_BYTES) {
          cleaves.emplace_back();
          acc = 0;
        }
        cleaves.back().push_back(L);
        acc += lbytes[L];
      }
    }
    const int nunits = (int)cleaves.size();
    std::vector<int> cpieces;
    for (int k = 0; k < nunits; ++k) {
      ycoff.push_back((int)ystages.size());
      cpieces.clear();
      for (int L : cleaves[k])
        for (int q = lptr[L]; q < lptr[L + 1]; ++q) cpieces.push_back(q);
      const int p1 = (int)cpieces.size();
      for (int pi = 0; pi < p1;) {
        int pe = pi;
        long long used = 0;
        while (pe < p1 && pe - pi < Y16_MAXIT && used + plen(yst[cpieces[pe]]) <= SD2)
          used += plen(yst[cpieces[pe++]]);
        if (pe == pi) fail(HMGPU_ERR_INVALID, "multi-RHS piece larger than a stage");
        M16Stage st{};
        st.cbeg = (int)ycopies.size();
        st.nitems = pe - pi;
        const size_t rec = yitems.size();
        YItem16 cnt{};
        cnt.kind = st.nitems;  // the count record (first int of the stage)
        yitems.push_back(cnt);
        copy(0, (long long)rec * (long long)sizeof(YItem16), 0,
             (long long)sizeof(YItem16) * (1 + st.nitems));
        long long off = Y16_HDR, bytes = (long long)sizeof(YItem16) * (1 + st.nitems);
        for (int q = pi; q < pe; ++q) {
          const YStage16& d = yst[cpieces[q]];
          YItem16 it{};
          it.kind = d.kind;
          it.leaf = gb0[d.leaf];  // first internal row position of the leaf (pair)
          it.tsel = d.tsel;
          it.rg = d.rg;
          it.flags = d.flags;
          it.R = d.R;
          it.PR = d.PR;
          it.jd = d.jd;
          it.m = d.m;
          it.roff = d.roff;
          it.part = d.part;
          std::copy(d.lo, d.lo + 6, it.lo);
          std::copy(d.hi, d.hi + 6, it.hi);
          it.off1 = (int)off;
          if (d.kind == Y16_ADM) {
            it.off2 = (int)(off + d.len);
            if (d.len) copy(1, 8 * d.src, off, 8LL * d.len);
            if (d.len2) copy(2, 8 * d.src2, off + d.len, 8LL * d.len2);
          } else {
            it.off2 = (int)(off + (long long)d.jd * d.PR);
            for (int j = 0; j < d.jd; ++j)
              copy(3, 8 * (d.src + (long long)j * d.spitch), off + (long long)j * d.PR,
                   8LL * d.len);
            copy(4, 8 * d.src2 * XP, it.off2, 8LL * d.len2);
          }
          bytes += d.kind == Y16_ADM ? 8LL * (d.len + d.len2)
                                     : 8LL * ((long long)d.jd * d.len + d.len2);
          off += plen(d);
          yitems.push_back(it);
        }
        st.ncopies = (int)ycopies.size() - st.cbeg;
        st.bytes = (int)bytes;
        ystages.push_back(st);
        pi = pe;
      }
    }
    ycoff.push_back((int)ystages.size());  // = END stage: a count record of -1
    {
      M16Stage st{};
      st.cbeg = (int)ycopies.size();
      st.ncopies = 1;
      st.bytes = (int)sizeof(YItem16);
      YItem16 cnt{};
      cnt.kind = -1;
      copy(0, (long long)yitems.size() * (long long)sizeof(YItem16), 0,
           (long long)sizeof(YItem16));
      yitems.push_back(cnt);
      ystages.push_back(st);
    }
  }
  c->d_zch16.upload(zch, c->stream);
  if (tasks.empty()) tasks.push_back(ZTask16{});  // the END chunk's header names task 0
  c->d_ztask16.upload(tasks, c->stream);
  c->d_zcoff16.upload(zcoff, c->stream);
  c->d_ycoff16.upload(ycoff, c->stream);
  c->d_yst16.upload(ystages, c->stream);
  c->d_yitem16.upload(yitems, c->stream);
  // (+ 16 rows: a small piece of a leaf pair stages that many, see flush())
  c->d_z16buf.ensure((size_t)zsize + 16 * ZP);
  // rows past k_c of a component's last l-step stay zero (A is zero there)
  CK(cudaMemsetAsync(c->d_z16buf.p, 0, ((size_t)zsize + 16 * ZP) * sizeof(double), c->stream));
  c->d_xp16.ensure(((size_t)c->n_cols + M16_XPAD) * XP);
  CK(cudaMemsetAsync(c->d_xp16.p, 0, c->d_xp16.n * sizeof(double), c->stream));
  // the packed factors live in the idle compaction arena, like the 1-RHS
  // stream arena (no new device memory in steady state; at most one of the
  // two plans is valid at a time)
  c->sync();
  c->plan_valid = false;
  c->spare_arena.ensure((size_t)alen + 2, c->device);
  CK(cudaMemsetAsync(c->spare_arena.p, 0, ((size_t)alen + 2) * sizeof(double), c->stream));
  {
    const unsigned long long base[5] = {
        (unsigned long long)c->d_yitem16.p, (unsigned long long)c->spare_arena.p,
        (unsigned long long)c->d_z16buf.p, (unsigned long long)c->d_dense.p,
        (unsigned long long)c->d_xp16.p};
    for (size_t q = 0; q < ycopies.size(); ++q) ycopies[q].src += base[ckind[q]];
    c->d_ycopy16.upload(ycopies, c->stream);
  }
  if (!packs.empty()) {
    DBuf<PackDesc> d_packs;
    d_packs.upload(packs, c->stream);
    c->timed("pack16", [&] {
      pack_kernel<<<grid_for(c, ((long long)packs.size() + 7) / 8, 16), 256, 0, c->stream>>>(
          d_packs.p, (int)packs.size(), c->d_arena.p, c->spare_arena.p);
    });
    c->sync();
    d_packs.free();
  }
  // phase-1 stage headers into the arena, in front of each chunk's V^T
  z16_hdr_kernel<<<grid_for(c, ((long long)zch.size() + 255) / 256, 16), 256, 0, c->stream>>>(
      c->d_zch16.p, c->d_ztask16.p, (int)zch.size(), c->spare_arena.p);
  CK(cudaGetLastError());
  c->n_zch16 = (int)zch.size() - 1;  // without the END records
  c->n_yst16 = (int)ystages.size() - 1;
  c->p16_zunits = (int)zcoff.size() - 1;
  c->p16_yunits = (int)ycoff.size() - 1;
  c->d_m16ctr.ensure(2);
  c->p16_nparts = nparts;
  c->p16_ypair = ypair;
  c->p16_row0 = c->p16_row1 = 0;  // internal row positions the leaves cover
  if (nl > 0) {
    c->p16_row0 = c->leaf_begin[0];
    c->p16_row1 = c->leaf_end[0];
    for (int L = 1; L < nl; ++L) {
      c->p16_row0 = std::min(c->p16_row0, c->leaf_begin[L]);
      c->p16_row1 = std::max(c->p16_row1, c->leaf_end[L]);
    }
  }

  c->p16_ns = cfg.ns;
  c->p16_stage = cfg.stage;
  c->p16_ncta = ncta;
  c->p16_nctaz = nctaz;
  c->p16_zns = cfg.zns;
  c->p16_zstage = cfg.zstage;
  c->p16_znw = cfg.znw;
  c->p16_ynw = cfg.ynw;
  c->p16_zsize = zsize;
  c->p16_alen = alen;
  c->p16_mode = mode;
  c->p16_valid = true;
  c->sync();
  if (verbose()) {
    long long kb[5] = {0, 0, 0, 0, 0};  // staged bytes of phase 2 by source
    for (size_t q = 0; q < ycopies.size(); ++q) kb[ckind[q]] += ycopies[q].bytes;
    std::fprintf(stderr, "[hmgpu] plan16 phase-2 bytes per product: records %.3f GB, U %.3f GB, "
                         "Z %.3f GB, near field %.3f GB, x rows %.3f GB (parts %d)\n",
                 kb[0] / 1e9, kb[1] / 1e9, kb[2] / 1e9, kb[3] / 1e9, kb[4] / 1e9, nparts);
  }
  if (verbose())
    std::fprintf(stderr, "[hmgpu] plan16: tasks=%zu chunks=%zu (units %d) stages=%zu (units %d) "
                         "arena=%.3f GB Z=%.3f GB ctas=%d/%d warps=%d/%d%s ring=%zu B\n",
                 tasks.size(), zch.size(), c->p16_zunits, ystages.size(), c->p16_yunits,
                 8.0 * alen / 1e9, 8.0 * zsize / 1e9, nctaz, ncta, cfg.znw, cfg.ynw,
                 ypair ? " (leaf pairs)" : "", ring_bytes);
}

template <int NS, int NW = 8>
void launch_m16(hmgpu_ctx* c, M16Params P) {  // phase 2
  const size_t smem = ((size_t)NS * c->p16_stage + M16_SLACK) * sizeof(double);
  CK(cudaFuncSetAttribute(hmv16_y_kernel<NS, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)smem));
  P.coff = c->d_ycoff16.p;
  P.nunits = c->p16_yunits;
  P.ctr = c->d_m16ctr.p + 1;
  hmv16_y_kernel<NS, NW><<<std::max(1, std::min(c->p16_ncta, c->p16_yunits)), 32 * (NW + 1), smem,
                           c->stream>>>(P);
  CK(cudaGetLastError());
}
template <int NS, int NW>
void launch_m16y2(hmgpu_ctx* c, M16Params P) {  // phase 2 over pairs of leaves
  const size_t smem = ((size_t)NS * c->p16_stage + M16_SLACK) * sizeof(double);
  CK(cudaFuncSetAttribute(hmv16_y2_kernel<NS, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)smem));
  P.coff = c->d_ycoff16.p;
  P.nunits = c->p16_yunits;
  P.ctr = c->d_m16ctr.p + 1;
  hmv16_y2_kernel<NS, NW><<<std::max(1, std::min(c->p16_ncta, c->p16_yunits)), 32 * (NW + 1), smem,
                            c->stream>>>(P);
  CK(cudaGetLastError());
}
template <int NS, int NW>
void launch_m16z(hmgpu_ctx* c, M16Params P) {  // phase 1
  const size_t smem = (size_t)NS * c->p16_zstage * sizeof(double);
  CK(cudaFuncSetAttribute(hmv16_z_kernel<NS, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)smem));
  P.stage = c->p16_zstage;
  P.coff = c->d_zcoff16.p;
  P.nunits = c->p16_zunits;
  P.ctr = c->d_m16ctr.p;
  hmv16_z_kernel<NS, NW><<<std::max(1, std::min(c->p16_nctaz, c->p16_zunits)), 32 * (NW + 1), smem,
                           c->stream>>>(P);
  CK(cudaGetLastError());
}

void launch_mrhs(hmgpu_ctx* c, const double* dx, double* dy, int nrhs, int mode) {
  (void)mode;  // the plan carries the mode's ranks
  M16Params P{};
  P.tasks = c->d_ztask16.p;
  P.arena = c->spare_arena.p;  // the packed p16 arena
  P.dense = c->d_dense.p;
  P.xp = c->d_xp16.p;
  P.z = c->d_z16buf.p;
  P.leaf_begin = c->d_leaf_begin.p;
  P.rperm = c->yperm();
  P.y = dy;
  // slices sized for the rows of this product (a shard's segment or all rows)
  if (c->p16_nparts > 1) c->d_y16part.ensure((size_t)c->p16_nparts * MR * 3 * (size_t)c->ynrows());
  P.ypart = c->d_y16part.p;
  P.nparts = c->p16_nparts;
  P.nrows = c->ynrows();
  P.stage = c->p16_stage;
  static const int dbg = [] {
    const char* e = std::getenv("HMGPU_M16_DBG");
    return e ? std::atoi(e) : 0;
  }();
  P.dbg = dbg;
  static DBuf<unsigned long long> prof;
  if (dbg == 3) {
    prof.ensure(16 + 2 * M16_PROF_CTAS);
    CK(cudaMemsetAsync(prof.p, 0, (16 + 2 * M16_PROF_CTAS) * 8, c->stream));
    P.prof = prof.p;
  }
  for (int s0 = 0; s0 < nrhs; s0 += MR) {
    const int nr = std::min(MR, nrhs - s0);
    P.s0 = s0;
    P.nr = nr;
    CK(cudaMemsetAsync(c->d_m16ctr.p, 0, 2 * sizeof(int), c->stream));
    c->timed("gather", [&] {
      const long long total = 48LL * c->n_cols;
      gather16_kernel<<<grid_for(c, (total + 255) / 256, 16), 256, 0, c->stream>>>(
          dx, c->d_xp16.p, c->d_cperm.p, c->n_cols, s0, nr);
    });
    if (c->n_zch16 > 0)
      c->timed("hmv16_z", [&] {
        P.desc = c->d_zch16.p;
        P.coff = c->d_zcoff16.p;
        const int key = c->p16_zns * 100 + c->p16_znw;
        if (key == 306) launch_m16z<3, 6>(c, P);
        else if (key == 406) launch_m16z<4, 6>(c, P);
        else if (key == 412) launch_m16z<4, 12>(c, P);
        else if (key == 408) launch_m16z<4, 8>(c, P);
        else if (key == 312) launch_m16z<3, 12>(c, P);
        else launch_m16z<3, 8>(c, P);
      });
    c->timed("hmv16_leaf", [&] {
      P.desc = c->d_yst16.p;
      P.copies = c->d_ycopy16.p;
      P.coff = c->d_ycoff16.p;
      P.stage = c->p16_stage;
      if (c->p16_ypair) {
        if (c->p16_ns == 4) {
          if (c->p16_ynw == 5) launch_m16y2<4, 5>(c, P);
          else if (c->p16_ynw == 6) launch_m16y2<4, 6>(c, P);
          else launch_m16y2<4, 8>(c, P);
        } else if (c->p16_ynw == 5) launch_m16y2<3, 5>(c, P);
        else if (c->p16_ynw == 6) launch_m16y2<3, 6>(c, P);
        else launch_m16y2<3, 8>(c, P);
      } else if (c->p16_ynw == 16) {
        if (c->p16_ns == 6) launch_m16<6, 16>(c, P);
        else if (c->p16_ns == 9) launch_m16<9, 16>(c, P);
        else launch_m16<4, 16>(c, P);
      } else if (c->p16_ynw == 6) {
        if (c->p16_ns == 4) launch_m16<4, 6>(c, P);
        else launch_m16<3, 6>(c, P);
      } else if (c->p16_ynw == 5) {
        if (c->p16_ns == 4) launch_m16<4, 5>(c, P);
        else launch_m16<3, 5>(c, P);
      } else {
        switch (c->p16_ns) {
          case 4: launch_m16<4>(c, P); break;
          case 6: launch_m16<6>(c, P); break;
          case 9: launch_m16<9>(c, P); break;
          default: launch_m16<3>(c, P);
        }
      }
      if (c->p16_nparts > 1) {  // the leaf parts' slices -> y, in part order
        const int nint = c->p16_row1 - c->p16_row0;
        const long long total = (long long)nint * 3 * nr;
        if (total > 0)
          y16_reduce_kernel<<<grid_for(c, (total + 255) / 256, 16), 256, 0, c->stream>>>(
              c->d_y16part.p, dy, c->yperm() + c->p16_row0, nint, c->ynrows(), c->p16_nparts, s0,
              nr);
        CK(cudaGetLastError());
      }
    });
  }
  if (dbg == 3) {
    std::vector<unsigned long long> hv(16 + 2 * M16_PROF_CTAS);
    CK(cudaMemcpyAsync(hv.data(), prof.p, hv.size() * 8, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    const unsigned long long* h = hv.data();
    if (h[9])
      std::fprintf(stderr, "[hmgpu] m16 phase 2, CTA 0: %.4g cycles in %.4g ms -> SM clock %.0f MHz\n",
                   (double)h[8], h[9] * 1e-6, (double)h[8] / (double)h[9] * 1e3);
    // per-CTA loop cycles (HMGPU_M16_PROF_FILE): pass (0 phase 2, 1 phase 1), CTA, cycles
    if (const char* pf = std::getenv("HMGPU_M16_PROF_FILE")) {
      if (FILE* f = std::fopen(pf, "w")) {
        for (int pass = 0; pass < 2; ++pass) {
          const int n = std::min(M16_PROF_CTAS, pass ? c->p16_nctaz : c->p16_ncta);
          for (int b = 0; b < n; ++b)
            std::fprintf(f, "%d %d %llu\n", pass, b, h[16 + pass * M16_PROF_CTAS + b]);
        }
        std::fclose(f);
      }
    }
    std::fprintf(stderr, "[hmgpu] m16 cycles (sum over warps): z consumer wait %.3g work %.3g, "
                 "producer wait %.3g issue %.3g; y consumer wait %.3g work %.3g, producer "
                 "wait %.3g issue %.3g\n", (double)h[0], (double)h[1], (double)h[2], (double)h[3],
                 (double)h[4], (double)h[5], (double)h[6], (double)h[7]);
  }
}

void launch_stream(hmgpu_ctx* c, const double* dx, double* dy, int nrhs) {
  (void)nrhs;
  const int NOUT = c->NC == 6 ? 3 : 1;
  c->d_xi.ensure((size_t)c->n_cols * 4 + 2);
  c->d_mvctr.ensure(2);
  c->timed("gather", [&] {
    const long long total = 4LL * c->n_cols;
    const int grid = grid_for(c, (total + 255) / 256, 16);
    if (NOUT == 3)
      gather4_kernel<3><<<grid, 256, 0, c->stream>>>(dx, c->d_xi.p, c->d_cperm.p, c->n_cols,
                                                     c->d_mvctr.p);
    else
      gather4_kernel<1><<<grid, 256, 0, c->stream>>>(dx, c->d_xi.p, c->d_cperm.p, c->n_cols,
                                                     c->d_mvctr.p);
  });
  c->d_ypart.ensure((size_t)std::max<long long>(1, c->p_slots * NOUT));
  c->d_zpart.ensure((size_t)std::max<long long>(1, c->p_zslots * 4));
  WarpStreamParams P{};
  P.chunks = c->d_pchunks.p;
  P.arena = c->spare_arena.p;  // the packed stream arena
  P.dense = c->d_dense.p;
  P.xi = c->d_xi.p;
  P.wout = c->d_zpart.p;
  P.win = c->d_zpart.p;
  P.ypart = c->d_ypart.p;
  P.jobs = c->d_pjobs.p;
  auto run = [&](int pass, int count, const char* name) {
    if (count <= 0) return;
    const MvCfg cfg = mv_cfg(pass);
    P.stage = cfg.stage;
    P.scratch = cfg.scratch;
    P.nwarps = c->p_nwarps_pass[pass];
    P.chunks = c->d_pchunks.p + c->p_chunk_base[pass];
    P.woff = c->d_pwoff.p + c->p_woff_base[pass];
    P.goff = P.woff + P.nwarps + 1;  // the pool's group bounds follow the warps' offsets
    P.ngroups = c->p_ngroups_pass[pass];
    P.ctr = c->d_mvctr.p + pass;
    const int g = P.nwarps / cfg.warps;  // the layout's grid: one CTA per SM
    const size_t smem = c->p_smem_pass[pass];
#ifdef HMGPU_MV_PROF  // per-warp loop cycles -> HMGPU_MV_PROF_FILE.<pass> (balance of the plan)
    static DBuf<unsigned long long> mvprof;
    mvprof.ensure((size_t)P.nwarps);
    CK(cudaMemsetAsync(mvprof.p, 0, (size_t)P.nwarps * 8, c->stream));
    P.prof = mvprof.p;
#endif
    auto go = [&](auto kernel) {
      CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kernel<<<g, cfg.warps * 32, smem, c->stream>>>(P);
#ifdef HMGPU_MV_PROF
      if (const char* pf = std::getenv("HMGPU_MV_PROF_FILE")) {
        std::vector<unsigned long long> h((size_t)P.nwarps);
        CK(cudaMemcpyAsync(h.data(), mvprof.p, h.size() * 8, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        if (FILE* f = std::fopen((std::string(pf) + "." + std::to_string(pass)).c_str(), "w")) {
          for (size_t q = 0; q < h.size(); ++q) std::fprintf(f, "%zu %llu\n", q, h[q]);
          std::fclose(f);
        }
      }
#endif
    };
#define HMV_CASE(W, S)                                        \
  if (cfg.warps == W && cfg.ns == S) {                        \
    if (P.ngroups > 0) {                                      \
      if (c->NC == 6) go(hmv_warp_kernel<6, S, W, true>);     \
      else go(hmv_warp_kernel<1, S, W, true>);                \
    } else {                                                  \
      if (c->NC == 6) go(hmv_warp_kernel<6, S, W, false>);    \
      else go(hmv_warp_kernel<1, S, W, false>);               \
    }                                                         \
    return;                                                   \
  }
    c->timed(name, [&] {
      HMV_CASE(12, 2) HMV_CASE(8, 2) HMV_CASE(10, 2) HMV_CASE(14, 2) HMV_CASE(16, 2)
      HMV_CASE(7, 2)
      fail(HMGPU_ERR_INVALID, "HMGPU_MV_CFG: unsupported (warps, stages)");
    });
#undef HMV_CASE
  };
  run(0, c->p_nz, "hmv_stream");
  run(1, c->p_njb, "hmv_ypart");
  c->timed("hmv_reduce", [&] {
    const int nl = (int)c->leaf_begin.size();
    const int g = grid_for(c, nl, 16);
    if (NOUT == 3)
      hmv_leaf_reduce_kernel<3><<<g, LR_THREADS, 0, c->stream>>>(
          c->d_leaf_begin.p, c->d_leaf_end.p, c->d_pleaf_ptr.p, c->d_pentries.p, nl,
          c->d_ypart.p, c->yperm(), c->ynrows(), dy);
    else
      hmv_leaf_reduce_kernel<1><<<g, LR_THREADS, 0, c->stream>>>(
          c->d_leaf_begin.p, c->d_leaf_end.p, c->d_pleaf_ptr.p, c->d_pentries.p, nl,
          c->d_ypart.p, c->yperm(), c->ynrows(), dy);
  });
}

void check_ptr_kind(int ptr_kind) {
  if (ptr_kind != HMGPU_PTR_HOST && ptr_kind != HMGPU_PTR_DEVICE)
    fail(HMGPU_ERR_INVALID, "ptr_kind must be HMGPU_PTR_HOST or HMGPU_PTR_DEVICE");
}

void gather_x(hmgpu_ctx* c, const double* dx, int nrhs) {
  const long long total = (long long)c->ndof_cols() * nrhs;
  c->d_xi.ensure((size_t)total);
  c->timed("gather", [&] {
    const int grid = grid_for(c, (total + 255) / 256, 16);
    if (c->NC == 6)
      gather_kernel<3><<<grid, 256, 0, c->stream>>>(dx, c->d_xi.p, c->d_cperm.p,
                                                   c->n_cols, nrhs);
    else
      gather_kernel<1><<<grid, 256, 0, c->stream>>>(dx, c->d_xi.p, c->d_cperm.p,
                                                   c->n_cols, nrhs);
  });
}

std::vector<int> items_from_pairs(hmgpu_ctx* c, int n, const int* cb) {
  std::vector<int> out;
  for (int t = 0; t < n; ++t) {
    const int comp = cb[2 * t], b = cb[2 * t + 1];
    if (comp < 0 || comp >= c->NC || b < 0 || b >= c->n_blocks)
      fail(HMGPU_ERR_INVALID, "bad (component, block) pair");
    const int i0 = c->item_of_block[b];
    if (i0 < 0) continue;  // dense or not owned: no-op like the reference
    out.push_back(i0 + comp);
  }
  return out;
}

}  // namespace

// ===========================================================================
extern "C" {

int hmgpu_device_count(int* n) {
  if (!n) return HMGPU_ERR_INVALID;
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) c = 0;
  *n = c;
  return HMGPU_OK;
}

int hmgpu_create(int device, hmgpu_ctx** out) {
  if (!out) return HMGPU_ERR_INVALID;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    return HMGPU_ERR_NODEVICE;
  if (device < 0 || device >= count) return HMGPU_ERR_INVALID;
  hmgpu_ctx* c = new (std::nothrow) hmgpu_ctx();
  if (!c) return HMGPU_ERR_OOM;
  c->device = device;
  const int st = guard(c, [&] {
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    CK(cudaMemPoolCreate(&c->pool, &props));
    unsigned long long keep = ~0ULL;
    CK(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &keep));
    {
      std::lock_guard<std::mutex> lk(g_pools_mu);
      g_pools.push_back({c->pool, c->stream});
    }
    g_pool = c->pool;
    g_stream = c->stream;
    CK(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
    c->d_counter.alloc(2);
    c->d_overflow.alloc(1);
    c->d_nq.alloc(1);
    c->rules.far_ratio = 4.0;
    c->rules.mid_ratio = 1.5;
  });
  if (st != HMGPU_OK) {
    delete c;
    return st;
  }
  *out = c;
  return HMGPU_OK;
}

int hmgpu_destroy(hmgpu_ctx* ctx) {
  if (!ctx) return HMGPU_ERR_INVALID;
  delete ctx;
  return HMGPU_OK;
}

const char* hmgpu_last_error(const hmgpu_ctx* ctx) {
  return ctx ? ctx->err.c_str() : "null context";
}

int hmgpu_get_stream(hmgpu_ctx* ctx, void** s) {
  return guard(ctx, [&] {
    if (!s) fail(HMGPU_ERR_INVALID, "null output");
    *s = (void*)ctx->stream;
  });
}

int hmgpu_set_rule(hmgpu_ctx* ctx, int tier, int npts, const double* a,
                   const double* b, const double* w) {
  return guard(ctx, [&] {
    if (tier < 0 || tier > 2) fail(HMGPU_ERR_INVALID, "tier must be 0, 1 or 2");
    if (npts < 1 || npts > 12 || !a || !b || !w)
      fail(HMGPU_ERR_INVALID, "rule must have 1..12 points");
    ctx->rules.n[tier] = npts;
    for (int q = 0; q < npts; ++q) {
      ctx->rules.a[tier][q] = a[q];
      ctx->rules.b[tier][q] = b[q];
      ctx->rules.w[tier][q] = w[q];
    }
    ctx->rules_set[tier] = true;
  });
}

int hmgpu_set_tier_ratios(hmgpu_ctx* ctx, double far_ratio, double mid_ratio) {
  return guard(ctx, [&] {
    if (!(far_ratio > 0) || !(mid_ratio > 0))
      fail(HMGPU_ERR_INVALID, "ratios must be positive");
    ctx->rules.far_ratio = far_ratio;
    ctx->rules.mid_ratio = mid_ratio;
  });
}

int hmgpu_set_kelvin_geometry(hmgpu_ctx* ctx, int n_vert, const double* verts,
                              int n_tri, const int* tris, const double* centroid,
                              const double* area, const double* diam, double E,
                              double nu) {
  return guard(ctx, [&] {
    if (n_vert < 3 || n_tri < 1 || !verts || !tris || !centroid || !area || !diam)
      fail(HMGPU_ERR_INVALID, "bad kelvin geometry");
    if (E <= 0.0) fail(HMGPU_ERR_INVALID, "lame_constants: E must be positive");
    if (nu <= 0.0 || nu >= 0.5)
      fail(HMGPU_ERR_INVALID, "lame_constants: nu must lie in (0, 1/2)");
    for (long long t = 0; t < 3LL * n_tri; ++t)
      if (tris[t] < 0 || tris[t] >= n_vert)
        fail(HMGPU_ERR_INVALID, "vertex index out of range");
    ctx->kind = KIND_KELVIN;
    ctx->NC = 6;
    ctx->n_vert = n_vert;
    ctx->n_tri = n_tri;
    ctx->verts.assign(verts, verts + 3LL * n_vert);
    ctx->tris.assign(tris, tris + 3LL * n_tri);
    ctx->centroid.assign(centroid, centroid + 3LL * n_tri);
    ctx->area.assign(area, area + n_tri);
    ctx->diam.assign(diam, diam + n_tri);
    ctx->E = E;
    ctx->nu = nu;
    ctx->assembled = false;
  });
}

int hmgpu_set_galerkin_geometry(hmgpu_ctx* ctx, int n_vert, const double* verts,
                                int n_tri, const int* tris, const double* centroid,
                                const double* area, const double* diam, int which) {
  return guard(ctx, [&] {
    if (n_vert < 3 || n_tri < 1 || !verts || !tris || !centroid || !area || !diam)
      fail(HMGPU_ERR_INVALID, "bad galerkin geometry");
    if (which != 0 && which != 1) fail(HMGPU_ERR_INVALID, "which must be 0 (V_kl) or 1 (V_Delta)");
    for (long long t = 0; t < 3LL * n_tri; ++t)
      if (tris[t] < 0 || tris[t] >= n_vert)
        fail(HMGPU_ERR_INVALID, "vertex index out of range");
    ctx->kind = KIND_GALERKIN;
    ctx->NC = which == 0 ? 6 : 1;
    ctx->gal_which = which;
    ctx->n_vert = n_vert;
    ctx->n_tri = n_tri;
    ctx->verts.assign(verts, verts + 3LL * n_vert);
    ctx->tris.assign(tris, tris + 3LL * n_tri);
    ctx->centroid.assign(centroid, centroid + 3LL * n_tri);
    ctx->area.assign(area, area + n_tri);
    ctx->diam.assign(diam, diam + n_tri);
    ctx->assembled = false;
  });
}

int hmgpu_set_kdelta_geometry(hmgpu_ctx* ctx, int n_vert, const double* verts, int n_tri,
                              const int* tris, const double* centroid, const double* area,
                              const double* diam, const double* normals) {
  return guard(ctx, [&] {
    if (n_vert < 3 || n_tri < 1 || !verts || !tris || !centroid || !area || !diam || !normals)
      fail(HMGPU_ERR_INVALID, "bad K_Delta geometry");
    for (long long t = 0; t < 3LL * n_tri; ++t)
      if (tris[t] < 0 || tris[t] >= n_vert)
        fail(HMGPU_ERR_INVALID, "vertex index out of range");
    ctx->kind = KIND_KDELTA;
    ctx->NC = 1;
    ctx->n_vert = n_vert;
    ctx->n_tri = n_tri;
    ctx->verts.assign(verts, verts + 3LL * n_vert);
    ctx->tris.assign(tris, tris + 3LL * n_tri);
    ctx->centroid.assign(centroid, centroid + 3LL * n_tri);
    ctx->area.assign(area, area + n_tri);
    ctx->diam.assign(diam, diam + n_tri);
    ctx->normals.assign(normals, normals + 3LL * n_tri);
    ctx->assembled = false;
  });
}

int hmgpu_set_pair_rule(hmgpu_ctx* ctx, int pair_case, int n, const double* xr1,
                        const double* xr2, const double* yr1, const double* yr2,
                        const double* w) {
  return guard(ctx, [&] {
    if (pair_case < 1 || pair_case > 3) fail(HMGPU_ERR_INVALID, "pair_case must be 1..3");
    if (n < 1 || !xr1 || !xr2 || !yr1 || !yr2 || !w) fail(HMGPU_ERR_INVALID, "bad pair rule");
    std::vector<double>& r = ctx->prule[pair_case];
    r.resize(5LL * n);
    const double* src[5] = {xr1, xr2, yr1, yr2, w};
    for (int f = 0; f < 5; ++f) std::copy(src[f], src[f] + n, r.begin() + (long long)f * n);
    ctx->prule_n[pair_case] = n;
    ctx->assembled = false;
  });
}

// ---- sparse transforms of the operator algebra (build_sparse_ops, ---------
// operators.cpp:7-95): ELL with 3 slots per triangle row; the transpose
// gathers per vertex over the inverse index (ascending triangles), so both
// directions are deterministic (no atomics).
namespace {
__global__ void ell3_spmv_kernel(int rows, const int* __restrict__ col,
                                 const double* __restrict__ val, const double* __restrict__ x,
                                 double* __restrict__ y, double alpha, double beta) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) s = fma(val[3 * r + a], x[col[3 * r + a]], s);
    y[r] = beta == 0.0 ? alpha * s : fma(alpha, s, beta * y[r]);
  }
}
__global__ void ell3_spmv_t_kernel(int cols, const int* __restrict__ tptr,
                                   const int* __restrict__ tslot, const double* __restrict__ val,
                                   const double* __restrict__ x, double* __restrict__ y,
                                   double alpha, double beta) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < cols; v += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int p = tptr[v]; p < tptr[v + 1]; ++p) {
      const int e = tslot[p];
      s = fma(val[e], x[e / 3], s);
    }
    y[v] = beta == 0.0 ? alpha * s : fma(alpha, s, beta * y[v]);
  }
}
}  // namespace

int hmgpu_ell3_spmv(hmgpu_ctx* ctx, int rows, const int* col3, const double* val3,
                    const double* x, double* y, double alpha, double beta) {
  return guard(ctx, [&] {
    if (rows < 0 || (rows > 0 && (!col3 || !val3 || !x || !y)))
      fail(HMGPU_ERR_INVALID, "bad ell3 spmv arguments");
    if (rows == 0) return;
    ell3_spmv_kernel<<<grid_for(ctx, (rows + 255) / 256), 256, 0, ctx->stream>>>(
        rows, col3, val3, x, y, alpha, beta);
    CK(cudaGetLastError());
  });
}

int hmgpu_ell3_spmv_t(hmgpu_ctx* ctx, int cols, const int* tptr, const int* tslot,
                      const double* val3, const double* x, double* y, double alpha,
                      double beta) {
  return guard(ctx, [&] {
    if (cols < 0 || (cols > 0 && (!tptr || !tslot || !val3 || !x || !y)))
      fail(HMGPU_ERR_INVALID, "bad ell3 transposed spmv arguments");
    if (cols == 0) return;
    ell3_spmv_t_kernel<<<grid_for(ctx, (cols + 255) / 256), 256, 0, ctx->stream>>>(
        cols, tptr, tslot, val3, x, y, alpha, beta);
    CK(cudaGetLastError());
  });
}

int hmgpu_set_kdouble_geometry(hmgpu_ctx* ctx, int n_vert, const double* verts, int n_tri,
                               const int* tris, const double* centroid, const double* area,
                               const double* diam, const double* normals, double E,
                               double nu, int r, int c) {
  const int st = hmgpu_set_kdelta_geometry(ctx, n_vert, verts, n_tri, tris, centroid, area,
                                           diam, normals);
  if (st != HMGPU_OK) return st;
  return guard(ctx, [&] {
    if (E <= 0.0) fail(HMGPU_ERR_INVALID, "lame_constants: E must be positive");
    if (nu <= 0.0 || nu >= 0.5)
      fail(HMGPU_ERR_INVALID, "lame_constants: nu must lie in (0, 1/2)");
    if (r < 0 || r > 2 || c < 0 || c > 2) fail(HMGPU_ERR_INVALID, "cell (r, c) in 0..2");
    ctx->kind = KIND_KDOUBLE;
    ctx->E = E;
    ctx->nu = nu;
    ctx->dl_r = r;
    ctx->dl_c = c;
  });
}

int hmgpu_set_eval_points(hmgpu_ctx* ctx, int n, const double* pts) {
  return guard(ctx, [&] {
    if (ctx->kind != KIND_KELVIN && ctx->kind != KIND_KDOUBLE)
      fail(HMGPU_ERR_STATE, "set the Kelvin / double-layer geometry first");
    if (n < 0 || (n > 0 && !pts)) fail(HMGPU_ERR_INVALID, "bad evaluation points");
    ctx->eval_pts.assign(pts, pts + 3LL * n);
    ctx->assembled = false;
  });
}

int hmgpu_set_points(hmgpu_ctx* ctx, int n, const double* pts, double diag) {
  return guard(ctx, [&] {
    if (n < 1 || !pts) fail(HMGPU_ERR_INVALID, "bad points");
    ctx->kind = KIND_NEWTON;
    ctx->NC = 1;
    ctx->n_pts = n;
    ctx->pts.assign(pts, pts + 3LL * n);
    ctx->diag = diag;
    ctx->assembled = false;
  });
}

int hmgpu_set_dense_matrix(hmgpu_ctx* ctx, int m, int n, const double* a) {
  return guard(ctx, [&] {
    if (m < 1 || n < 1 || !a) fail(HMGPU_ERR_INVALID, "bad matrix");
    ctx->kind = KIND_DENSE;
    ctx->NC = 1;
    ctx->am = m;
    ctx->an = n;
    ctx->amat.assign(a, a + (long long)m * n);
    ctx->assembled = false;
  });
}

int hmgpu_set_partition(hmgpu_ctx* ctx, int n_rows, const int* row_perm,
                        int n_row_nodes, const int* row_nodes4, int n_cols,
                        const int* col_perm, int n_col_nodes, const int* col_nodes4,
                        int n_blocks, const int* blocks4, int row_begin,
                        int row_end) {
  return guard(ctx, [&] {
    if (n_rows < 1 || n_cols < 1 || !row_perm || !col_perm || !row_nodes4 ||
        !col_nodes4 || !blocks4 || n_blocks < 1 || n_row_nodes < 1 ||
        n_col_nodes < 1)
      fail(HMGPU_ERR_INVALID, "bad partition arguments");
    if (row_begin < 0 || row_end > n_rows || row_begin >= row_end)
      fail(HMGPU_ERR_INVALID, "bad row shard range");
    ctx->n_rows = n_rows;
    ctx->n_cols = n_cols;
    ctx->rperm.assign(row_perm, row_perm + n_rows);
    ctx->cperm.assign(col_perm, col_perm + n_cols);
    ctx->rnodes.assign(row_nodes4, row_nodes4 + 4LL * n_row_nodes);
    ctx->cnodes.assign(col_nodes4, col_nodes4 + 4LL * n_col_nodes);
    ctx->blocks.assign(blocks4, blocks4 + 4LL * n_blocks);
    ctx->n_blocks = n_blocks;
    ctx->row_begin = row_begin;
    ctx->row_end = row_end;
    for (int b = 0; b < n_blocks; ++b)
      if (blocks4[4 * b] < 0 || blocks4[4 * b] >= n_row_nodes ||
          blocks4[4 * b + 1] < 0 || blocks4[4 * b + 1] >= n_col_nodes)
        fail(HMGPU_ERR_INVALID, "block references a missing node");
    ctx->same_tree = n_rows == n_cols && ctx->rperm == ctx->cperm &&
                     ctx->rnodes == ctx->cnodes;
    ctx->have_partition = true;
    ctx->assembled = false;
  });
}

int hmgpu_assemble(hmgpu_ctx* c, double eps, double beta_stop, int initial_rank,
                   int lookahead, long long max_rank, hmgpu_assembly_stats* stats) {
  return guard(c, [&] {
    if (!c->have_partition) fail(HMGPU_ERR_STATE, "set_partition first");
    if (c->kind < 0) fail(HMGPU_ERR_STATE, "set an entry provider first");
    if (initial_rank < 0) {  // aca_run argument checks (aca.cpp:108-110)
      if (eps <= 0.0) fail(HMGPU_ERR_INVALID, "aca_run: eps must be positive");
      if (beta_stop <= 0.0 || beta_stop >= 1.0)
        fail(HMGPU_ERR_INVALID, "aca_run: beta must be in (0,1)");
    }
    if (lookahead < 0 || max_rank < 1) fail(HMGPU_ERR_INVALID, "bad lookahead/max_rank");
    if (c->kind == KIND_KELVIN || c->kind == KIND_GALERKIN || c->kind == KIND_KDELTA ||
        c->kind == KIND_KDOUBLE)
      upload_rules(c);
    build_geometry(c);
    c->eps = eps;
    c->beta = beta_stop;
    c->initial_rank = initial_rank;
    c->lookahead = lookahead;
    c->max_rank = max_rank;
    for (auto& p : c->pending) {
      c->ev_pool.push_back(p.a);
      c->ev_pool.push_back(p.b);
    }
    c->pending.clear();

    auto wall0 = std::chrono::steady_clock::now();
    auto phase = [&](const char* what) {
      if (!verbose()) return;
      c->sync();
      const auto now = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[hmgpu] %-12s %9.2f ms\n", what,
                   std::chrono::duration<double, std::milli>(now - wall0).count());
      wall0 = now;
    };
    cudaEvent_t t0, t1, tn0, tn1;
    CK(cudaEventCreate(&t0));
    CK(cudaEventCreate(&t1));
    CK(cudaEventCreate(&tn0));
    CK(cudaEventCreate(&tn1));
    CK(cudaEventRecord(t0, c->stream));

    // work items and dense blocks of the owned block rows
    c->items.clear();
    c->dblocks.clear();
    c->item_of_block.assign(c->n_blocks, -1);
    c->dense_of_block.assign(c->n_blocks, -1);
    c->arena_used = 0;
    c->piv_used = 0;
    c->dense_used = 0;
    long long cons_used = 0;
    const int NCq = c->NC;
    std::vector<AdmBlock> ablocks;
    // release the previous assembly before sizing this one
    c->sync();
    // both arenas stay mapped across assemblies; the larger one takes the
    // loose layout (the other is the compaction target)
    if (c->spare_arena.n > c->d_arena.n) std::swap(c->spare_arena, c->d_arena);
    c->d_dense.free();
    c->d_piv.free();
    c->d_cons.free();
    c->d_ypart.free();
    // Initial column capacity per item: the coarse mode knows its final
    // rank; full mode starts at 24 + lookahead columns, lowered when the
    // device memory would not hold it (items that outgrow their capacity
    // are relocated and resumed, see run_aca).
    long long sum_mn = 0, dense_total = 0;
    for (int b = 0; b < c->n_blocks; ++b) {
      const int* B = &c->blocks[4 * b];
      const int* rn = &c->rnodes[4 * B[0]];
      const int* cn = &c->cnodes[4 * B[1]];
      if (rn[0] < c->row_begin || rn[1] > c->row_end) continue;
      const long long m = rn[1] - rn[0], n = cn[1] - cn[0];
      if (B[2]) sum_mn += (m + n) * c->NC;
      else dense_total += n * align2((long long)c->NC * m);
    }
    c->sync();
    // mapped arenas are reused by this assembly
    const size_t free_b = avail_bytes() + c->d_arena.mapped + c->spare_arena.mapped;
    const double avail =
        (double)free_b - 8.0 * (double)dense_total - 4.0 * (1 << 30);
    // full mode: 24 columns before the look-ahead unless HMGPU_ACA_CAP0 says
    // otherwise (items that need more are relocated and resumed)
    static const int cap0 = [] {
      const char* e = std::getenv("HMGPU_ACA_CAP0");
      return e ? std::max(1, std::atoi(e)) : 24;
    }();
    int cap_init = (initial_rank >= 0 ? initial_rank : cap0) + lookahead;
    if (initial_rank < 0 && sum_mn > 0) {
      const long long fit = (long long)(0.55 * avail / (8.0 * (double)sum_mn));
      cap_init = (int)std::max<long long>(lookahead + 6, std::min<long long>(cap_init, fit));
    }
    // the largest blocks carry the highest ranks: they start with extra
    // columns when memory allows, so they rarely overflow into the
    // relocation pass (a second launch over a few large items, poorly
    // parallel: 11.5 ms of config 3's 287 ms ACA before this)
    static const int big_mn = [] {
      const char* e = std::getenv("HMGPU_ACA_BIG_MN");
      return e ? std::atoi(e) : 8192;
    }();
    static const int big_extra = [] {
      const char* e = std::getenv("HMGPU_ACA_BIG_EXTRA");
      return e ? std::max(0, std::atoi(e)) : 24;
    }();
    int cap_big = cap_init;
    if (initial_rank < 0 && big_extra > 0) {
      long long sum_mn_big = 0;
      for (int b = 0; b < c->n_blocks; ++b) {
        const int* B = &c->blocks[4 * b];
        const int* rn = &c->rnodes[4 * B[0]];
        const int* cn = &c->cnodes[4 * B[1]];
        if (!B[2] || rn[0] < c->row_begin || rn[1] > c->row_end) continue;
        const long long mn = (rn[1] - rn[0]) + (cn[1] - cn[0]);
        if (mn >= big_mn) sum_mn_big += mn * c->NC;
      }
      if (8.0 * ((double)sum_mn * cap_init + (double)sum_mn_big * big_extra) <= 0.55 * avail)
        cap_big = cap_init + big_extra;
    }
    for (int b = 0; b < c->n_blocks; ++b) {
      const int* B = &c->blocks[4 * b];
      const int* rn = &c->rnodes[4 * B[0]];
      const int* cn = &c->cnodes[4 * B[1]];
      if (rn[0] < c->row_begin || rn[1] > c->row_end) continue;
      const int m = rn[1] - rn[0], n = cn[1] - cn[0];
      if (B[2]) {
        // the NC items of this block are generated on the device from one
        // record (items_init_kernel); offsets assigned here in item order
        c->item_of_block[b] = (int)(NCq * ablocks.size());
        const long long capr = std::min<long long>(max_rank, std::min(m, n));
        const int cap = (int)std::min<long long>(capr, m + n >= big_mn ? cap_big : cap_init);
        AdmBlock ab{};
        ab.m = m;
        ab.n = n;
        ab.row0 = rn[0];
        ab.col0 = cn[0];
        ab.block = b;
        ab.cap = cap;
        ab.u_base = c->arena_used;
        ab.p_base = c->piv_used;
        ab.z_base = cons_used;
        c->arena_used += (long long)NCq * (align2((long long)m * cap) + align2((long long)n * cap));
        c->piv_used += (long long)NCq * std::max(cap, 1);
        cons_used += (long long)NCq * align16(m);
        ablocks.push_back(ab);
      } else {
        c->dense_of_block[b] = (int)c->dblocks.size();
        DenseBlock db{m, n, rn[0], cn[0], c->dense_used};
        c->dense_used += (long long)n * align2((long long)c->NC * m);
        c->dblocks.push_back(db);
      }
    }
    // small headroom at the arena end for relocated (regrown) items; the
    // arena grows in place beyond it (VArena)
    const size_t arena_cap = (size_t)(c->arena_used * 1.02) + 1024;
    c->items.resize((size_t)NCq * ablocks.size());  // mirror filled by download_items
    phase("items");
    c->d_items.ensure(std::max<size_t>(c->items.size(), 1));
    if (!ablocks.empty()) {
      c->d_ablocks.upload(ablocks, c->stream);
      items_init_kernel<<<(int)((ablocks.size() * NCq + 255) / 256), 256, 0, c->stream>>>(
          c->d_ablocks.p, (int)ablocks.size(), NCq,
          initial_rank >= 0 ? PH_INIT : PH_RUN, initial_rank >= 0 ? initial_rank : 0,
          c->d_items.p);
      CK(cudaGetLastError());
    }
    c->d_arena.ensure(arena_cap + 2, c->device);
    c->d_piv.alloc((size_t)(c->piv_used * 1.3) + 1);
    c->d_cons.alloc((size_t)cons_used + 16);
    CK(cudaMemsetAsync(c->d_cons.p, 0, cons_used + 16, c->stream));
    c->d_dense.alloc((size_t)c->dense_used + 2);
    c->d_dblocks.upload(c->dblocks, c->stream);

    phase("alloc+upload");
    // the partition-only tables of the matvec on a host thread, beside the
    // near-field and ACA kernels (joined before build_matvec_finish)
    std::exception_ptr tables_err;
    std::thread tables([&] {
      try {
        build_matvec_tables(c);
      } catch (...) {
        tables_err = std::current_exception();
      }
    });
    struct Joiner {
      std::thread& t;
      ~Joiner() {
        if (t.joinable()) t.join();
      }
    } tables_join{tables};
    // near-field fill
    CK(cudaMemsetAsync(c->d_nq.p, 0, sizeof(unsigned long long), c->stream));
    CK(cudaEventRecord(tn0, c->stream));
    if (!c->dblocks.empty()) {
      c->timed("nearfield", [&] {
        const int grid = grid_for(c, (long long)c->dblocks.size(), 8);
        const bool gal = c->kind == KIND_GALERKIN || c->kind == KIND_KDELTA;
        if (gal && c->NC == 6)
          nearfield_gal_kernel<6><<<grid, 256, 0, c->stream>>>(
              c->geom, c->d_dblocks.p, (int)c->dblocks.size(), c->d_dense.p, c->d_nq.p);
        else if (gal)
          nearfield_gal_kernel<1><<<grid, 256, 0, c->stream>>>(
              c->geom, c->d_dblocks.p, (int)c->dblocks.size(), c->d_dense.p, c->d_nq.p);
        else if (c->NC == 6)
          nearfield_kernel<6><<<grid, 256, 0, c->stream>>>(
              c->geom, c->d_dblocks.p, (int)c->dblocks.size(), c->d_dense.p, c->d_nq.p);
        else
          nearfield_kernel<1><<<grid, 256, 0, c->stream>>>(
              c->geom, c->d_dblocks.p, (int)c->dblocks.size(), c->d_dense.p, c->d_nq.p);
      });
    }
    CK(cudaEventRecord(tn1, c->stream));

    phase("nearfield");
    // ACA, largest blocks first (stable counting sort of the blocks on m + n;
    // a block's items stay in component order)
    std::vector<int> list(c->items.size());
    {
      int kmax_mn = 0;
      for (const AdmBlock& ab : ablocks) kmax_mn = std::max(kmax_mn, ab.m + ab.n);
      std::vector<int> cnt(kmax_mn + 2, 0);
      for (const AdmBlock& ab : ablocks) ++cnt[kmax_mn - (ab.m + ab.n) + 1];
      for (int k = 1; k <= kmax_mn + 1; ++k) cnt[k] += cnt[k - 1];
      for (size_t a = 0; a < ablocks.size(); ++a) {
        const int pos = cnt[kmax_mn - (ablocks[a].m + ablocks[a].n)]++;
        for (int q = 0; q < NCq; ++q) list[(size_t)pos * NCq + q] = (int)(a * NCq + q);
      }
    }
    int relaunch = 0;
    auto mn_of = [&](int idx) { return ablocks[idx / NCq].m + ablocks[idx / NCq].n; };
    static const bool split = std::getenv("HMGPU_ACA_CLASSES") != nullptr;
    if (split && !list.empty()) {
      // diagnostic: the ACA run class by class (m + n ranges, largest first)
      // with one event pair per class; the results are the same
      size_t s0 = 0;
      while (s0 < list.size()) {
        const AdmBlock& a0 = ablocks[list[s0] / NCq];
        int lo = 1;
        while (2 * lo <= a0.m + a0.n) lo *= 2;
        size_t s1 = s0;
        while (s1 < list.size()) {
          const AdmBlock& a1 = ablocks[list[s1] / NCq];
          if (a1.m + a1.n < lo) break;
          ++s1;
        }
        std::vector<int> sub(list.begin() + s0, list.begin() + s1);
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, c->stream));
        run_aca(c, sub, &relaunch, mn_of);
        CK(cudaEventRecord(e1, c->stream));
        c->sync();
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        std::fprintf(stderr, "[hmgpu] aca class m+n in [%d,%d): items=%zu ms=%.3f\n", lo,
                     2 * lo, sub.size(), ms);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        s0 = s1;
      }
    } else {
      run_aca(c, list, &relaunch, mn_of);
    }
    phase("aca");
    compact(c, 0);
    phase("compact");
    if (verbose()) {
      const size_t f2 = avail_bytes();
      std::fprintf(stderr, "[hmgpu] items=%zu cap_init=%d arena=%.2f GB dense=%.2f GB "
                           "free_after=%.2f GB relaunches=%d\n",
                   c->items.size(), cap_init, 8.0 * c->arena_used / 1e9,
                   8.0 * c->dense_used / 1e9, f2 / 1e9, relaunch);
    }
    CK(cudaEventRecord(t1, c->stream));
    c->sync();
    float ms_total = 0, ms_near = 0;
    CK(cudaEventElapsedTime(&ms_total, t0, t1));
    CK(cudaEventElapsedTime(&ms_near, tn0, tn1));
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    cudaEventDestroy(tn0);
    cudaEventDestroy(tn1);
    tables.join();
    if (tables_err) std::rethrow_exception(tables_err);
    build_matvec_finish(c);
    c->plan_valid = false;
    c->p16_valid = false;
    c->mv_auto_used = false;
    phase("build_matvec");
    c->assembled = true;
    if (stats) {
      hmgpu_assembly_stats s{};
      unsigned long long nq_dense = 0;
      CK(cudaMemcpy(&nq_dense, c->d_nq.p, sizeof(nq_dense), cudaMemcpyDeviceToHost));
      double flops = 0.0;
      for (const Item& it : c->items) {
        s.aca_entries += it.entries;
        s.aca_steps += it.steps;
        s.pivots += it.k;
        flops += 30.0 * (double)it.nq_sum + (double)it.entries;
      }
      // near-field: one rule per pair, six component entries of 30 n_q + 1
      flops += 6.0 * 30.0 * (double)nq_dense;
      for (const DenseBlock& d : c->dblocks)
        s.dense_entries += (long long)c->NC * d.m * d.n;
      s.ms_total = ms_total;
      s.ms_nearfield = ms_near;
      s.ms_aca = ms_total - ms_near;
      s.aca_relaunches = relaunch;
      for (const DenseBlock& d : c->dblocks) flops += (double)c->NC * d.m * d.n;
      s.counted_flops = c->kind == KIND_KELVIN ? flops : 0.0;
      *stats = s;
    }
  });
}

int hmgpu_matvec_transposed(hmgpu_ctx* c, const double* x, double* y, int nrhs, int mode,
                            int ptr_kind) {
  return guard(c, [&] {
    if (!c->assembled) fail(HMGPU_ERR_STATE, "assemble first");
    if (!x || !y || nrhs < 1) fail(HMGPU_ERR_INVALID, "bad matvec arguments");
    if (mode != HMGPU_MODE_CURRENT && mode != HMGPU_MODE_LOOKAHEAD)
      fail(HMGPU_ERR_INVALID, "bad mode");
    check_ptr_kind(ptr_kind);
    if (!c->t_valid) build_matvec_t(c);
    const int NOUT = c->NC == 6 ? 3 : 1;
    const long long nxr = (long long)c->n_rows * NOUT, nyc = (long long)c->n_cols * NOUT;
    const double* dx = x;
    double* dy = y;
    DBuf<double> hx, hy;
    if (ptr_kind == HMGPU_PTR_HOST) {
      hx.alloc((size_t)(nxr * nrhs));
      hy.alloc((size_t)(nyc * nrhs));
      CK(cudaMemcpyAsync(hx.p, x, nxr * nrhs * sizeof(double), cudaMemcpyHostToDevice,
                         c->stream));
      dx = hx.p;
      dy = hy.p;
    }
    c->d_xr.ensure((size_t)nxr);
    c->d_tpart.ensure((size_t)std::max<long long>(c->t_rows * NOUT, 1));
    const size_t smem = 2 * (size_t)std::max(c->kmax, 1) * sizeof(double);
    for (int q = 0; q < nrhs; ++q) {
      const int gg = grid_for(c, (nxr + 255) / 256);
      if (NOUT == 3)
        gather_kernel<3><<<gg, 256, 0, c->stream>>>(dx + q * nxr, c->d_xr.p, c->d_rperm.p,
                                                     c->n_rows, 1);
      else
        gather_kernel<1><<<gg, 256, 0, c->stream>>>(dx + q * nxr, c->d_xr.p, c->d_rperm.p,
                                                     c->n_rows, 1);
      const int grid = grid_for(c, c->n_mv, 4);
      if (c->NC == 6) {
        if (smem > 48 * 1024)
          CK(cudaFuncSetAttribute(hmvt_blocks_kernel<6>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        hmvt_blocks_kernel<6><<<grid, 256, smem, c->stream>>>(
            c->d_mvb.p, c->n_mv, c->d_tprow.p, c->d_items.p, c->d_arena.p, c->d_dense.p,
            c->d_xr.p, c->d_tpart.p, mode);
      } else {
        if (smem > 48 * 1024)
          CK(cudaFuncSetAttribute(hmvt_blocks_kernel<1>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        hmvt_blocks_kernel<1><<<grid, 256, smem, c->stream>>>(
            c->d_mvb.p, c->n_mv, c->d_tprow.p, c->d_items.p, c->d_arena.p, c->d_dense.p,
            c->d_xr.p, c->d_tpart.p, mode);
      }
      CK(cudaGetLastError());
      const int gr = grid_for(c, c->t_nleaves, 8);
      if (NOUT == 3)
        hmv_reduce_kernel<3><<<gr, 128, 0, c->stream>>>(
            c->d_tleaf_begin.p, c->d_tleaf_end.p, c->d_tleaf_ptr.p, c->d_tleaf_prow.p,
            c->t_nleaves, c->d_tpart.p, c->d_cperm.p, c->n_cols, dy + q * nyc, 1);
      else
        hmv_reduce_kernel<1><<<gr, 128, 0, c->stream>>>(
            c->d_tleaf_begin.p, c->d_tleaf_end.p, c->d_tleaf_ptr.p, c->d_tleaf_prow.p,
            c->t_nleaves, c->d_tpart.p, c->d_cperm.p, c->n_cols, dy + q * nyc, 1);
      CK(cudaGetLastError());
    }
    if (ptr_kind == HMGPU_PTR_HOST) {
      CK(cudaMemcpyAsync(y, hy.p, nyc * nrhs * sizeof(double), cudaMemcpyDeviceToHost,
                         c->stream));
      c->sync();
      hx.free();
      hy.free();
    }
  });
}

int hmgpu_ranks(hmgpu_ctx* c, int* k_cur, int* k_look, int* consumed, int* last_stop) {
  return guard(c, [&] {
    if (!c->assembled) fail(HMGPU_ERR_STATE, "assemble first");
    for (int q = 0; q < c->NC; ++q)
      for (int b = 0; b < c->n_blocks; ++b) {
        const long long o = (long long)q * c->n_blocks + b;
        const int i0 = c->item_of_block[b];
        const Item* it = i0 >= 0 ? &c->items[i0 + q] : nullptr;
        if (k_cur) k_cur[o] = it ? it->kcur : -1;
        if (k_look) k_look[o] = it ? it->k : -1;
        if (consumed) consumed[o] = it ? it->nconsumed : -1;
        if (last_stop) last_stop[o] = it ? it->last_stop : -1;
      }
  });
}

namespace {
// y = A x over the owned block rows, DEVICE pointers; the rows are written
// through (c->yperm(), c->ynrows()): external order by default (non-owned
// rows zeroed), the shard's segment for the distributed product
void matvec_local(hmgpu_ctx* c, const double* dx, double* dy, int nrhs, int mode) {
  const int NOUT = c->NC == 6 ? 3 : 1;
  if (!c->out_perm && (c->row_begin != 0 || c->row_end != c->n_rows))
    CK(cudaMemsetAsync(dy, 0, (size_t)c->ndof_rows() * nrhs * sizeof(double), c->stream));
  static const bool force_v1 = std::getenv("HMGPU_MATVEC_V1") != nullptr;
  if (nrhs > 1 && c->NC == 6 && !force_v1) {
    bool ok = true;
    if (!c->p16_valid || c->p16_mode != mode) {
      try {
        build_plan16(c, mode);
      } catch (const Fail& f) {
        if (f.code != HMGPU_ERR_INVALID) throw;
        ok = false;  // ranks beyond the shared-memory Z: block sweep below
        c->p16_valid = false;
      }
    }
    if (ok) {
      launch_mrhs(c, dx, dy, nrhs, mode);
      return;
    }
  }
  bool direct_now = c->mv_policy == 1;
  if (c->mv_policy == 2 && nrhs == 1 && !c->mv_auto_used &&
      !(c->plan_valid && c->plan_mode == mode && c->plan_nrhs == nrhs)) {
    direct_now = true;
    c->mv_auto_used = true;
  }
  bool streamed = !force_v1 && !(direct_now && nrhs == 1);
  if (streamed && (!c->plan_valid || c->plan_mode != mode || c->plan_nrhs != nrhs)) {
    try {
      const auto tp = std::chrono::steady_clock::now();
      build_plan(c, mode, nrhs);
      if (verbose())
        std::fprintf(stderr, "[hmgpu] build_plan %9.2f ms\n",
                     std::chrono::duration<double, std::milli>(
                         std::chrono::steady_clock::now() - tp).count());
    } catch (const Fail& f) {
      if (f.code != HMGPU_ERR_INVALID) throw;
      streamed = false;  // ranks / widths beyond the stream layout: block sweep
      c->plan_valid = false;
    }
  }
  if (streamed) {
    launch_stream(c, dx, dy, nrhs);
    return;
  }
  gather_x(c, dx, nrhs);
  c->d_ypart.ensure((size_t)std::max<long long>(1, c->part_rows * NOUT * nrhs));
  const size_t smem = sizeof(double) * 2 * (size_t)c->kmax * nrhs;
  if (smem > 200 * 1024) fail(HMGPU_ERR_INVALID, "rank x nrhs too large for matvec");
  c->timed("hmv_blocks", [&] {
    const int grid = grid_for(c, c->n_mv, 8);
    // always opt in: the kernel's static dred[] shares the 48 KB default
    // window, so any dynamic size needs the attribute
    if (c->NC == 6) {
      CK(cudaFuncSetAttribute(hmv_blocks_kernel<6>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      hmv_blocks_kernel<6><<<grid, 256, smem, c->stream>>>(
          c->d_mvb.p, c->d_mvorder.p, c->n_mv, c->d_items.p, c->d_arena.p,
          c->d_dense.p, c->d_xi.p, c->d_ypart.p, nrhs, mode);
    } else {
      CK(cudaFuncSetAttribute(hmv_blocks_kernel<1>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      hmv_blocks_kernel<1><<<grid, 256, smem, c->stream>>>(
          c->d_mvb.p, c->d_mvorder.p, c->n_mv, c->d_items.p, c->d_arena.p,
          c->d_dense.p, c->d_xi.p, c->d_ypart.p, nrhs, mode);
    }
  });
  c->timed("hmv_reduce", [&] {
    const int nl = (int)c->leaf_begin.size();
    const int grid = grid_for(c, nl, 16);
    if (c->NC == 6)
      hmv_reduce_kernel<3><<<grid, 128, 0, c->stream>>>(
          c->d_leaf_begin.p, c->d_leaf_end.p, c->d_leaf_ptr.p, c->d_leaf_prow.p,
          nl, c->d_ypart.p, c->yperm(), c->ynrows(), dy, nrhs);
    else
      hmv_reduce_kernel<1><<<grid, 128, 0, c->stream>>>(
          c->d_leaf_begin.p, c->d_leaf_end.p, c->d_leaf_ptr.p, c->d_leaf_prow.p,
          nl, c->d_ypart.p, c->yperm(), c->ynrows(), dy, nrhs);
  });
}

void check_matvec_args(hmgpu_ctx* c, int nrhs, int mode, int ptr_kind) {
  if (!c->assembled) fail(HMGPU_ERR_STATE, "assemble first");
  if (nrhs < 1) fail(HMGPU_ERR_INVALID, "bad matvec arguments");
  if (mode != HMGPU_MODE_CURRENT && mode != HMGPU_MODE_LOOKAHEAD)
    fail(HMGPU_ERR_INVALID, "bad mode");
  check_ptr_kind(ptr_kind);
}
}  // namespace

int hmgpu_matvec(hmgpu_ctx* c, const double* x, double* y, int nrhs, int mode,
                 int ptr_kind) {
  return guard(c, [&] {
    check_matvec_args(c, nrhs, mode, ptr_kind);
    if (!x || !y) fail(HMGPU_ERR_INVALID, "bad matvec arguments");
    const long long nx = (long long)c->ndof_cols() * nrhs;
    const long long ny = (long long)c->ndof_rows() * nrhs;
    const double* dx = x;
    double* dy = y;
    if (ptr_kind == HMGPU_PTR_HOST) {
      c->d_x.ensure((size_t)nx);
      c->d_y.ensure((size_t)ny);
      CK(cudaMemcpyAsync(c->d_x.p, x, nx * sizeof(double), cudaMemcpyHostToDevice,
                         c->stream));
      dx = c->d_x.p;
      dy = c->d_y.p;
    }
    matvec_local(c, dx, dy, nrhs, mode);
    if (ptr_kind == HMGPU_PTR_HOST) {
      CK(cudaMemcpyAsync(y, dy, ny * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      c->sync();
    }
  });
}

// ---- multi-GPU block-row sharding ------------------------------------------
namespace {
#define NK(x)                                                                     \
  do {                                                                            \
    ncclResult_t r_ = (x);                                                        \
    if (r_ != ncclSuccess)                                                        \
      throw Fail{HMGPU_ERR_COMM, std::string(#x) + ": " + nccl_api().GetErrorString(r_)}; \
  } while (0)

NcclApi& need_nccl() {
  NcclApi& a = nccl_api();
  if (!a.ok) fail(HMGPU_ERR_COMM, a.why);
  return a;
}

// in-place broadcast of a device buffer from `root`
void comm_bcast(hmgpu_ctx* c, const void* send, void* dbuf, size_t bytes, int root) {
  if (bytes == 0) return;
  if (c->comm_kind == 1 || c->comm_kind == 2) {
    NK(nccl_api().Broadcast(send ? send : dbuf, dbuf, bytes, ncclChar, root, c->nccl,
                            c->stream));
    return;
  }
  c->h_stage_a.resize(bytes);
  if (c->comm_rank == root)
    CK(cudaMemcpyAsync(c->h_stage_a.data(), send ? send : dbuf, bytes,
                       cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  if (c->comm_ops.broadcast(c->comm_ops.user, c->h_stage_a.data(), (long long)bytes, root))
    fail(HMGPU_ERR_COMM, "host broadcast callback failed");
  CK(cudaMemcpyAsync(dbuf, c->h_stage_a.data(), bytes, cudaMemcpyHostToDevice, c->stream));
}

// recv[r * bytes ...] = send of rank r (device buffers)
void comm_allgather(hmgpu_ctx* c, const void* dsend, void* drecv, size_t bytes) {
  if (c->comm_kind == 1 || c->comm_kind == 2) {
    NK(nccl_api().AllGather(dsend, drecv, bytes, ncclChar, c->nccl, c->stream));
    return;
  }
  c->h_stage_a.resize(bytes);
  c->h_stage_b.resize(bytes * c->comm_n);
  CK(cudaMemcpyAsync(c->h_stage_a.data(), dsend, bytes, cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  if (c->comm_ops.allgather(c->comm_ops.user, c->h_stage_a.data(), c->h_stage_b.data(),
                            (long long)bytes))
    fail(HMGPU_ERR_COMM, "host allgather callback failed");
  CK(cudaMemcpyAsync(drecv, c->h_stage_b.data(), bytes * c->comm_n, cudaMemcpyHostToDevice,
                     c->stream));
}

// after a transport is attached: exchange the row ranges, check that they
// tile the rows in rank order, build the segment map
void comm_setup(hmgpu_ctx* c) {
  const int n = c->comm_n;
  DBuf<int> mine, all;
  const int rr[2] = {c->row_begin, c->row_end};
  mine.upload(rr, 2, c->stream);
  all.ensure(2 * (size_t)n);
  comm_allgather(c, mine.p, all.p, 2 * sizeof(int));
  std::vector<int> h(2 * (size_t)n);
  CK(cudaMemcpyAsync(h.data(), all.p, h.size() * sizeof(int), cudaMemcpyDeviceToHost,
                     c->stream));
  c->sync();
  mine.free();
  all.free();
  c->dist_rb.assign(n, 0);
  c->dist_len.assign(n, 0);
  int expect = 0, maxseg = 1;
  for (int k = 0; k < n; ++k) {
    if (h[2 * k] != expect || h[2 * k + 1] < h[2 * k])
      fail(HMGPU_ERR_INVALID, "shard row ranges do not tile the rows in rank order");
    c->dist_rb[k] = h[2 * k];
    c->dist_len[k] = h[2 * k + 1] - h[2 * k];
    maxseg = std::max(maxseg, c->dist_len[k]);
    expect = h[2 * k + 1];
  }
  if (expect != c->n_rows) fail(HMGPU_ERR_INVALID, "shard row ranges do not cover the rows");
  c->dist_maxseg = maxseg;
  c->d_dist_rb.upload(c->dist_rb, c->stream);
  c->d_dist_len.upload(c->dist_len, c->stream);
  c->d_segperm.ensure((size_t)c->n_rows);
  dist_segperm_kernel<<<grid_for(c, (c->n_rows + 255) / 256, 8), 256, 0, c->stream>>>(
      c->d_segperm.p, c->n_rows, c->row_begin, c->row_end);
  CK(cudaGetLastError());
  c->sync();
}

void comm_reset(hmgpu_ctx* c) {
  if (c->comm_kind == 1 && c->nccl) nccl_api().CommDestroy(c->nccl);
  c->nccl = nullptr;
  c->comm_kind = 0;
  c->comm_n = 1;
  c->comm_rank = 0;
  c->comm_ops = hmgpu_comm_ops{};
}

void comm_args(hmgpu_ctx* c, int nranks, int rank) {
  if (!c->have_partition) fail(HMGPU_ERR_STATE, "set the partition (with the shard) first");
  if (nranks < 1 || rank < 0 || rank >= nranks) fail(HMGPU_ERR_INVALID, "bad nranks / rank");
}
}  // namespace

int hmgpu_nccl_available(int* available, int* version) {
  NcclApi& a = nccl_api();
  if (available) *available = a.ok ? 1 : 0;
  if (version) *version = a.version;
  return HMGPU_OK;
}

int hmgpu_nccl_unique_id(void* id128) {
  if (!id128) return HMGPU_ERR_INVALID;
  NcclApi& a = nccl_api();
  if (!a.ok) return HMGPU_ERR_COMM;
  ncclUniqueId id;
  if (a.GetUniqueId(&id) != ncclSuccess) return HMGPU_ERR_COMM;
  std::memcpy(id128, &id, sizeof(id));
  return HMGPU_OK;
}

int hmgpu_comm_init_nccl(hmgpu_ctx* c, int nranks, int rank, const void* id128) {
  return guard(c, [&] {
    comm_args(c, nranks, rank);
    if (!id128) fail(HMGPU_ERR_INVALID, "null unique id");
    NcclApi& a = need_nccl();
    comm_reset(c);
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t comm = nullptr;
    NK(a.CommInitRank(&comm, nranks, id, rank));
    c->nccl = comm;
    c->comm_kind = 1;
    c->comm_n = nranks;
    c->comm_rank = rank;
    comm_setup(c);
  });
}

int hmgpu_comm_set_nccl(hmgpu_ctx* c, void* nccl_comm, int nranks, int rank) {
  return guard(c, [&] {
    comm_args(c, nranks, rank);
    if (!nccl_comm) fail(HMGPU_ERR_INVALID, "null ncclComm_t");
    need_nccl();
    comm_reset(c);
    c->nccl = static_cast<ncclComm_t>(nccl_comm);
    c->comm_kind = 2;
    c->comm_n = nranks;
    c->comm_rank = rank;
    comm_setup(c);
  });
}

int hmgpu_comm_set_ops(hmgpu_ctx* c, int nranks, int rank, const hmgpu_comm_ops* ops) {
  return guard(c, [&] {
    comm_args(c, nranks, rank);
    if (!ops || !ops->broadcast || !ops->allgather)
      fail(HMGPU_ERR_INVALID, "comm ops need broadcast and allgather");
    comm_reset(c);
    c->comm_ops = *ops;
    c->comm_kind = 3;
    c->comm_n = nranks;
    c->comm_rank = rank;
    comm_setup(c);
  });
}

int hmgpu_comm_clear(hmgpu_ctx* c) {
  return guard(c, [&] { comm_reset(c); });
}

int hmgpu_comm_info(hmgpu_ctx* c, int* nranks, int* rank, int* kind, int* row_begin,
                    int* row_end) {
  return guard(c, [&] {
    if (nranks) *nranks = c->comm_n;
    if (rank) *rank = c->comm_rank;
    if (kind) *kind = c->comm_kind;
    if (c->comm_kind)
      for (int k = 0; k < c->comm_n; ++k) {
        if (row_begin) row_begin[k] = c->dist_rb[k];
        if (row_end) row_end[k] = c->dist_rb[k] + c->dist_len[k];
      }
  });
}

int hmgpu_comm_allgather(hmgpu_ctx* c, const void* send, void* recv,
                         long long bytes_per_rank) {
  return guard(c, [&] {
    if (!c->comm_kind) fail(HMGPU_ERR_STATE, "no communicator attached (hmgpu_comm_*)");
    if (bytes_per_rank < 0 || (bytes_per_rank > 0 && (!send || !recv)))
      fail(HMGPU_ERR_INVALID, "bad all-gather arguments");
    if (bytes_per_rank == 0) return;
    const size_t b = (size_t)bytes_per_rank;
    if (c->comm_kind == 3) {  // host callbacks work on host buffers directly
      if (c->comm_ops.allgather(c->comm_ops.user, send, recv, bytes_per_rank))
        fail(HMGPU_ERR_COMM, "allgather callback failed");
      return;
    }
    DBuf<char> ds, dr;
    ds.alloc(b);
    dr.alloc(b * c->comm_n);
    CK(cudaMemcpyAsync(ds.p, send, b, cudaMemcpyHostToDevice, c->stream));
    comm_allgather(c, ds.p, dr.p, b);
    CK(cudaMemcpyAsync(recv, dr.p, b * c->comm_n, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    ds.free();
    dr.free();
  });
}

int hmgpu_matvec_dist(hmgpu_ctx* c, const double* x, double* y, int nrhs, int mode,
                      int ptr_kind) {
  return guard(c, [&] {
    if (!c->comm_kind) fail(HMGPU_ERR_STATE, "no communicator attached (hmgpu_comm_*)");
    check_matvec_args(c, nrhs, mode, ptr_kind);
    if (!y || (c->comm_rank == 0 && !x)) fail(HMGPU_ERR_INVALID, "bad matvec arguments");
    const int NOUT = c->NC == 6 ? 3 : 1;
    const long long nx = (long long)c->ndof_cols() * nrhs;
    const long long ny = (long long)c->ndof_rows() * nrhs;
    // x from rank 0 into every rank's d_x (NCCL reads the root's x in place)
    c->d_x.ensure((size_t)nx);
    const double* root_src = nullptr;
    if (c->comm_rank == 0) {
      if (ptr_kind == HMGPU_PTR_HOST)
        CK(cudaMemcpyAsync(c->d_x.p, x, nx * sizeof(double), cudaMemcpyHostToDevice,
                           c->stream));
      else
        root_src = x;
    }
    c->timed("dist_bcast", [&] {
      comm_bcast(c, root_src, c->d_x.p, (size_t)nx * sizeof(double), 0);
    });
    // the shard's rows into its segment [nrhs][NOUT][maxseg]
    const long long seg = (long long)nrhs * NOUT * c->dist_maxseg;
    c->d_ysend.ensure((size_t)seg);
    c->d_yrecv.ensure((size_t)seg * c->comm_n);
    c->out_perm = c->d_segperm.p;
    c->out_nrows = c->dist_maxseg;
    try {
      matvec_local(c, c->d_x.p, c->d_ysend.p, nrhs, mode);
    } catch (...) {
      c->out_perm = nullptr;
      throw;
    }
    c->out_perm = nullptr;
    c->timed("dist_allgather", [&] {
      comm_allgather(c, c->d_ysend.p, c->d_yrecv.p, (size_t)seg * sizeof(double));
    });
    double* dy = y;
    if (ptr_kind == HMGPU_PTR_HOST) {
      c->d_y.ensure((size_t)ny);
      dy = c->d_y.p;
    }
    c->timed("dist_scatter", [&] {
      const long long total = seg * c->comm_n;
      const int g = grid_for(c, (total + 255) / 256, 16);
      if (NOUT == 3)
        dist_scatter_kernel<3><<<g, 256, 0, c->stream>>>(
            c->d_yrecv.p, c->comm_n, nrhs, c->dist_maxseg, c->d_dist_rb.p, c->d_dist_len.p,
            c->d_rperm.p, c->n_rows, dy);
      else
        dist_scatter_kernel<1><<<g, 256, 0, c->stream>>>(
            c->d_yrecv.p, c->comm_n, nrhs, c->dist_maxseg, c->d_dist_rb.p, c->d_dist_len.p,
            c->d_rperm.p, c->n_rows, dy);
    });
    if (ptr_kind == HMGPU_PTR_HOST) {
      CK(cudaMemcpyAsync(y, dy, ny * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      c->sync();
    }
  });
}

namespace {
void promote_ids(hmgpu_ctx* c, const std::vector<int>& ids) {
  if (ids.empty()) return;
  c->d_list.upload(ids, c->stream);
  c->timed("promote", [&] {
    promote_kernel<<<(int)(ids.size() + 255) / 256, 256, 0, c->stream>>>(
        c->d_items.p, c->d_list.p, (int)ids.size());
  });
  for (int i : ids) c->items[i].kcur = c->items[i].k;
  c->plan_valid = false;
  c->p16_valid = false;
  c->mv_auto_used = false;
  c->sync();
}

void extend_ids(hmgpu_ctx* c, std::vector<int> ids, int steps) {
  std::sort(ids.begin(), ids.end());
  ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
  if (ids.empty() || steps == 0) return;
  auto w0 = std::chrono::steady_clock::now();
  auto phase = [&](const char* what) {
    if (!verbose()) return;
    c->sync();
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[hmgpu] extend %-9s %9.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - w0).count());
    w0 = now;
  };
  if (c->kind == KIND_KELVIN || c->kind == KIND_GALERKIN || c->kind == KIND_KDELTA ||
      c->kind == KIND_KDOUBLE)
    upload_rules(c);
  {
    // items that cannot take `steps` more columns move to a larger slot up
    // front (growth as in run_aca's overflow path); the overflow path would
    // spend a launch, a mirror download and then the same relocation
    std::vector<int> rid, rcap;
    for (int idx : ids) {
      const Item& it = c->items[idx];
      const long long capr = std::min<long long>(c->max_rank, std::min(it.m, it.n));
      const long long need = std::min<long long>(capr, (long long)it.k + steps);
      if (need <= it.cap) continue;
      rid.push_back(idx);
      rcap.push_back((int)std::min<long long>(
          capr, std::max<long long>(need, std::max(2 * it.cap, it.cap + 8))));
    }
    relocate(c, rid, rcap);  // the mirror catches up with the download below
  }
  phase("relocate");
  c->d_list.upload(ids, c->stream);
  c->timed("prep_extend", [&] {
    prep_extend_kernel<<<(int)(ids.size() + 255) / 256, 256, 0, c->stream>>>(
        c->d_items.p, c->d_list.p, (int)ids.size(), steps);
  });
  c->sync();
  {  // largest m + n first, stable: keys gathered once (the comparator's
     // random reads of the 128-byte item table cost ~10 ms per sweep)
    std::vector<std::pair<int, int>> kv(ids.size());
    for (size_t t = 0; t < ids.size(); ++t)
      kv[t] = {-(c->items[ids[t]].m + c->items[ids[t]].n), ids[t]};
    std::stable_sort(kv.begin(), kv.end(),
                     [](const std::pair<int, int>& a, const std::pair<int, int>& b) {
                       return a.first < b.first;
                     });
    for (size_t t = 0; t < ids.size(); ++t) ids[t] = kv[t].second;
  }
  phase("prep");
  run_aca(c, ids, nullptr, [&](int idx) { return c->items[idx].m + c->items[idx].n; });
  phase("aca");
  download_items_subset(c, ids);
  phase("download");
  for (int idx : ids) c->kmax = std::max(c->kmax, c->items[idx].k);  // k only grows here
  phase("ranks");
  c->plan_valid = false;
  c->p16_valid = false;
  c->mv_auto_used = false;
}

// per-partition tables of the estimator: leaf of every internal row, and per
// matvec block its local rows in ascending external order
void build_amvm_geometry(hmgpu_ctx* c) {
  if (c->am_geom_valid) return;
  std::vector<int> row_leaf(std::max(c->n_rows, 1), 0);
  for (size_t l = 0; l < c->leaf_begin.size(); ++l)
    for (int p = c->leaf_begin[l]; p < c->leaf_end[l]; ++p) row_leaf[p] = (int)l;
  std::vector<long long> spoff(std::max(c->n_mv, 1), 0);
  std::vector<int> sortp;
  std::map<std::pair<int, int>, long long> seen;  // (row0, m) -> offset
  for (int bi = 0; bi < c->n_mv; ++bi) {
    const MvBlock& mb = c->mvb[bi];
    if (mb.dense) continue;
    auto key = std::make_pair(mb.row0, mb.m);
    auto f = seen.find(key);
    if (f != seen.end()) {
      spoff[bi] = f->second;
      continue;
    }
    const long long off = (long long)sortp.size();
    std::vector<int> loc(mb.m);
    std::iota(loc.begin(), loc.end(), 0);
    std::sort(loc.begin(), loc.end(), [&](int a, int b) {
      return c->rperm[mb.row0 + a] < c->rperm[mb.row0 + b];
    });
    sortp.insert(sortp.end(), loc.begin(), loc.end());
    seen[key] = off;
    spoff[bi] = off;
  }
  if (sortp.empty()) sortp.push_back(0);
  c->d_row_leaf.upload(row_leaf, c->stream);
  c->d_spoff.upload(spoff, c->stream);
  c->d_sortp.upload(sortp, c->stream);
  c->sync();
  c->am_geom_valid = true;
}

AmvmGeom amvm_geom(hmgpu_ctx* c) {
  AmvmGeom a{};
  a.row_leaf = c->d_row_leaf.p;
  a.leaf_begin = c->d_leaf_begin.p;
  a.leaf_ptr = c->d_leaf_ptr.p;
  a.leaf_blk = c->d_leaf_blk.p;
  a.blocks = c->d_mvb.p;
  a.rperm = c->d_rperm.p;
  a.tix = c->d_tix.p;
  a.terms = c->d_aterms.p;
  a.term_bi = c->d_term_bi.p;
  a.sortp = c->d_sortp.p;
  a.spoff = c->d_spoff.p;
  a.out = c->d_aout.p;
  a.N = c->n_rows;
  a.grid = c->NC == 6 ? 1 : 0;
  return a;
}
}  // namespace

int hmgpu_promote(hmgpu_ctx* c, int n, const int* comp_block) {
  return guard(c, [&] {
    if (!c->assembled) fail(HMGPU_ERR_STATE, "assemble first");
    if (n < 0 || (n > 0 && !comp_block)) fail(HMGPU_ERR_INVALID, "bad pairs");
    promote_ids(c, items_from_pairs(c, n, comp_block));
  });
}

int hmgpu_extend(hmgpu_ctx* c, int n, const int* comp_block, int steps) {
  return guard(c, [&] {
    if (!c->assembled) fail(HMGPU_ERR_STATE, "assemble first");
    if (n < 0 || (n > 0 && !comp_block) || steps < 0)
      fail(HMGPU_ERR_INVALID, "bad extend arguments");
    extend_ids(c, items_from_pairs(c, n, comp_block), steps);
  });
}

int hmgpu_set_matvec_policy(hmgpu_ctx* c, int direct) {
  return guard(c, [&] {
    if (direct < 0 || direct > 2) fail(HMGPU_ERR_INVALID, "matvec policy must be 0, 1 or 2");
    c->mv_policy = direct;
  });
}

int hmgpu_get_matvec_policy(hmgpu_ctx* c, int* direct) {
  return guard(c, [&] {
    if (!direct) fail(HMGPU_ERR_INVALID, "null direct");
    *direct = c->mv_policy;
  });
}

int hmgpu_amvm_estimate(hmgpu_ctx* c, const double* x, double* gamma, double* difference) {
  return guard(c, [&] {
    if (!c->assembled) fail(HMGPU_ERR_STATE, "assemble first");
    if (!x || !gamma) fail(HMGPU_ERR_INVALID, "null x / gamma");
    if (c->row_begin != 0 || c->row_end != c->n_rows)
      fail(HMGPU_ERR_INVALID, "the estimator needs the whole operator (no shard)");
    auto wall0 = std::chrono::steady_clock::now();
    auto phase = [&](const char* what) {
      if (!verbose()) return;
      c->sync();
      const auto now = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[hmgpu] est  %-10s %9.2f ms\n", what,
                   std::chrono::duration<double, std::milli>(now - wall0).count());
      wall0 = now;
    };
    build_amvm_geometry(c);
    phase("geometry");
    // terms: (comp, block) with a look-ahead tail, component-major, blocks
    // ascending (amvm.cpp:135-150) -- generated on the device (flags, two
    // CUB scans for the term index and the value offset)
    const int nslot = c->NC * c->n_mv;
    long long off = 0;
    int nterms = 0;
    {
      DBuf<int> flag, pos;
      DBuf<long long> size, offs;
      flag.alloc(nslot + 1);
      pos.alloc(nslot + 1);
      size.alloc(nslot + 1);
      offs.alloc(nslot + 1);
      CK(cudaMemsetAsync(flag.p + nslot, 0, sizeof(int), c->stream));
      CK(cudaMemsetAsync(size.p + nslot, 0, sizeof(long long), c->stream));
      if (nslot > 0)
        amvm_term_flags_kernel<<<(nslot + 255) / 256, 256, 0, c->stream>>>(
            c->d_mvb.p, c->n_mv, c->NC, c->d_items.p, flag.p, size.p);
      size_t t1 = 0, t2 = 0;
      CK(cub::DeviceScan::ExclusiveSum(nullptr, t1, flag.p, pos.p, nslot + 1, c->stream));
      CK(cub::DeviceScan::ExclusiveSum(nullptr, t2, size.p, offs.p, nslot + 1, c->stream));
      c->d_cub.ensure(std::max(t1, t2));
      CK(cub::DeviceScan::ExclusiveSum(c->d_cub.p, t1, flag.p, pos.p, nslot + 1, c->stream));
      CK(cub::DeviceScan::ExclusiveSum(c->d_cub.p, t2, size.p, offs.p, nslot + 1, c->stream));
      CK(cudaMemcpyAsync(&nterms, pos.p + nslot, sizeof(int), cudaMemcpyDeviceToHost,
                         c->stream));
      CK(cudaMemcpyAsync(&off, offs.p + nslot, sizeof(long long), cudaMemcpyDeviceToHost,
                         c->stream));
      c->sync();
      c->d_aterms.ensure((size_t)std::max(nterms, 1));
      c->d_term_bi.ensure((size_t)std::max(nterms, 1));
      c->d_tix.ensure(std::max<size_t>(c->items.size(), 1));
      CK(cudaMemsetAsync(c->d_tix.p, 0xff, std::max<size_t>(c->items.size(), 1) * sizeof(int),
                         c->stream));
      if (nterms > 0)
        amvm_term_write_kernel<<<(nslot + 255) / 256, 256, 0, c->stream>>>(
            c->d_mvb.p, c->n_mv, c->NC, flag.p, pos.p, offs.p, c->d_aterms.p, c->d_term_bi.p,
            c->d_tix.p);
      CK(cudaGetLastError());
      flag.free();
      pos.free();
      size.free();
      offs.free();
    }
    c->am_nterms = nterms;
    c->am_nvals = off;
    const long long M = (long long)c->ndof_rows();
    c->d_diff.ensure((size_t)M);
    c->d_sc.ensure(8);
    c->d_aout.ensure((size_t)std::max<long long>(off, 1));
    const long long nx = c->ndof_cols();
    c->d_x.ensure((size_t)nx);
    CK(cudaMemcpyAsync(c->d_x.p, x, nx * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    gather_x(c, c->d_x.p, 1);
    phase("terms");
    if (nterms > 0)
      c->timed("tail", [&] {
        const int grid = grid_for(c, ((long long)nterms + 7) / 8, 8);
        if (c->NC == 6)
          tail_kernel<3><<<grid, 256, 0, c->stream>>>(c->d_aterms.p, nterms, c->d_items.p,
                                                     c->d_arena.p, c->d_xi.p, c->d_aout.p, 1);
        else
          tail_kernel<1><<<grid, 256, 0, c->stream>>>(c->d_aterms.p, nterms, c->d_items.p,
                                                     c->d_arena.p, c->d_xi.p, c->d_aout.p, 0);
      });
    phase("tail");
    const AmvmGeom a = amvm_geom(c);
    c->timed("amvm_diff", [&] {
      amvm_diff_kernel<<<(c->n_rows + 127) / 128, 128, 0, c->stream>>>(a, c->d_diff.p);
    });
    amvm_sumsq_kernel<<<1, 32, 0, c->stream>>>(c->d_diff.p, M, c->d_sc.p);
    CK(cudaGetLastError());
    double sc[2];
    CK(cudaMemcpyAsync(sc, c->d_sc.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (difference)
      CK(cudaMemcpyAsync(difference, c->d_diff.p, M * sizeof(double), cudaMemcpyDeviceToHost,
                         c->stream));
    c->sync();
    phase("diff+dl");
    *gamma = sc[1];
    c->am_have_estimate = true;
  });
}

namespace {
// the greedy marking walk, parallel and bit-identical (hmgpu_amvm.cuh,
// walk_*_kernel): term sequence S by first appearance, then chunks of S
// with per-row residual-before values, per-term dots, the sequential
// res_sq scan and the residual update.  Writes d_marked / d_nm and
// d_sc[2] = gamma(P_k) like amvm_walk_kernel.
void parallel_walk(hmgpu_ctx* c, double theta, long long M, int nt) {
  double sc2[2];
  CK(cudaMemcpyAsync(sc2, c->d_sc.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  const double target = (1.0 - theta) * sc2[1];
  const double target_sq = target * target;
  int nm = 0;
  DBuf<long long> cnt, pre;
  DBuf<unsigned long long> first, fsorted;
  DBuf<int> tid, tS, count;
  if (sc2[0] > target_sq && nt > 0 && M > 0) {
    c->timed("amvm_walk", [&] {
      cnt.alloc(M + 1);
      pre.alloc(M + 1);
      walk_cnt_kernel<<<(int)((M + 256) / 256), 256, 0, c->stream>>>(c->d_order.p, M,
                                                                      c->d_ptr.p, cnt.p);
      size_t tb = 0;
      CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, pre.p, (int)(M + 1), c->stream));
      c->d_cub.ensure(tb);
      CK(cub::DeviceScan::ExclusiveSum(c->d_cub.p, tb, cnt.p, pre.p, (int)(M + 1), c->stream));
      first.alloc(nt);
      fsorted.alloc(nt);
      tid.alloc(nt);
      tS.alloc(nt);
      count.alloc(1);
      CK(cudaMemsetAsync(first.p, 0xff, nt * sizeof(unsigned long long), c->stream));
      CK(cudaMemsetAsync(count.p, 0, sizeof(int), c->stream));
      walk_first_kernel<<<(int)((M + 255) / 256), 256, 0, c->stream>>>(
          c->d_order.p, M, c->d_ptr.p, c->d_lists.p, pre.p, first.p);
      walk_tids_kernel<<<(nt + 255) / 256, 256, 0, c->stream>>>(nt, tid.p, first.p, count.p);
      tb = 0;
      CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, first.p, fsorted.p, tid.p, tS.p, nt, 0, 64,
                                         c->stream));
      c->d_cub.ensure(tb);
      CK(cub::DeviceRadixSort::SortPairs(c->d_cub.p, tb, first.p, fsorted.p, tid.p, tS.p, nt, 0,
                                         64, c->stream));
    });
    int L = 0;
    CK(cudaMemcpyAsync(&L, count.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    DBuf<long long> sz, cumE;
    sz.alloc(L + 1);
    cumE.alloc(L + 1);
    walk_sizes_kernel<<<(L + 256) / 256, 256, 0, c->stream>>>(tS.p, L, c->d_eptr.p, sz.p);
    size_t tb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, sz.p, cumE.p, L + 1, c->stream));
    c->d_cub.ensure(tb);
    CK(cub::DeviceScan::ExclusiveSum(c->d_cub.p, tb, sz.p, cumE.p, L + 1, c->stream));
    std::vector<long long> hcum(L + 1);
    CK(cudaMemcpyAsync(hcum.data(), cumE.p, (L + 1) * sizeof(long long),
                       cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    int row_bits = 1;
    while ((1LL << row_bits) <= M) ++row_bits;
    const long long kEmax = 1LL << 24;
    const int kTmax = 1 << 20;
    // chunk buffers live in the context (sized once for the largest chunk:
    // re-growing the pool on every sweep cost up to 0.3 s)
    DBuf<unsigned long long>& keys = c->w_keys;
    DBuf<unsigned long long>& skeys = c->w_skeys;
    DBuf<int>& slots = c->w_slots;
    DBuf<int>& sslots = c->w_sslots;
    DBuf<long long>& gslot = c->w_gslot;
    DBuf<double>& rb = c->w_rb;
    DBuf<double>& dots = c->w_dots;
    DBuf<double> st;
    st.alloc(2);
    {
      const long long emax = std::min<long long>(hcum[L], kEmax);
      long long e1max = 0;
      for (int a = 0, b = 0; a < L; a = b) {  // the largest chunk of this walk
        b = a + 1;
        while (b < L && b - a < kTmax && hcum[b + 1] - hcum[a] <= kEmax) ++b;
        e1max = std::max(e1max, hcum[b] - hcum[a]);
        if (e1max >= emax) break;
      }
      const size_t need = (size_t)std::max(e1max, 1LL);
      keys.ensure(need);
      skeys.ensure(need);
      slots.ensure(need);
      sslots.ensure(need);
      gslot.ensure(need);
      rb.ensure(need);
      dots.ensure((size_t)std::min(L, kTmax) + 1);
    }
    CK(cudaMemcpyAsync(st.p, c->d_sc.p, sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    int k0 = 0;
    bool stopped = false;
    while (k0 < L && !stopped) {
      int k1 = k0 + 1;
      while (k1 < L && k1 - k0 < kTmax && hcum[k1 + 1] - hcum[k0] <= kEmax) ++k1;
      const long long E = hcum[k1] - hcum[k0];
      const int nk = k1 - k0;
      c->timed("amvm_walk", [&] {
        keys.ensure(E);
        skeys.ensure(E);
        slots.ensure(E);
        sslots.ensure(E);
        gslot.ensure(E);
        rb.ensure(E);
        dots.ensure(nk);
        walk_build_kernel<<<(nk + 127) / 128, 128, 0, c->stream>>>(
            tS.p, k0, k1, cumE.p, c->d_eptr.p, c->d_eidx.p, keys.p, slots.p, gslot.p);
        size_t tbs = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tbs, keys.p, skeys.p, slots.p, sslots.p,
                                           (int)E, 0, 22 + row_bits, c->stream));
        c->d_cub.ensure(tbs);
        CK(cub::DeviceRadixSort::SortPairs(c->d_cub.p, tbs, keys.p, skeys.p, slots.p,
                                           sslots.p, (int)E, 0, 22 + row_bits, c->stream));
        const int ge = (int)((E + 255) / 256);
        walk_before_kernel<<<ge, 256, 0, c->stream>>>(skeys.p, sslots.p, E, gslot.p,
                                                       c->d_eval.p, c->d_resid.p, rb.p);
        walk_dot_kernel<<<(nk + 127) / 128, 128, 0, c->stream>>>(k0, k1, cumE.p, gslot.p,
                                                                 c->d_eval.p, rb.p, dots.p);
        walk_incr_kernel<<<(nk + 255) / 256, 256, 0, c->stream>>>(tS.p, k0, k1, c->d_nsq.p,
                                                                  dots.p);
        walk_scan_kernel<<<1, 1, 0, c->stream>>>(dots.p, nk, target_sq, st.p);
        walk_apply_kernel<<<ge, 256, 0, c->stream>>>(skeys.p, sslots.p, E, gslot.p,
                                                      c->d_eval.p, rb.p, st.p, nk,
                                                      c->d_resid.p);
      });
      double hst[2];
      CK(cudaMemcpyAsync(hst, st.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      c->sync();
      const int stop = (int)hst[1];
      if (stop >= 0) {
        nm = k0 + stop + 1;
        stopped = true;
      } else {
        nm = k1;
      }
      k0 = k1;
    }
    CK(cudaMemcpyAsync(c->d_marked.p, tS.p, (size_t)nm * sizeof(int), cudaMemcpyDeviceToDevice,
                       c->stream));
    st.free(); sz.free(); cumE.free();
  }
  CK(cudaMemcpyAsync(c->d_nm.p, &nm, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  // gamma(P_k): exact recomputation over the residual (amvm.cpp:181)
  amvm_sumsq_kernel<<<1, 1, 0, c->stream>>>(c->d_resid.p, M, c->d_sc.p + 4);
  CK(cudaMemcpyAsync(c->d_sc.p + 2, c->d_sc.p + 5, sizeof(double), cudaMemcpyDeviceToDevice,
                     c->stream));
  c->sync();
  cnt.free(); pre.free(); first.free(); fsorted.free(); tid.free(); tS.free(); count.free();
}
}  // namespace

int hmgpu_amvm_mark(hmgpu_ctx* c, double theta, int c_sp, long long m_rows, long long n_cols,
                    double* gamma_pk, int* n_marked) {
  return guard(c, [&] {
    if (!c->am_have_estimate) fail(HMGPU_ERR_STATE, "hmgpu_amvm_estimate first");
    if (!gamma_pk || !n_marked) fail(HMGPU_ERR_INVALID, "null outputs");
    const long long M = (long long)c->ndof_rows();
    const int nt = c->am_nterms;
    c->marked_ids.clear();
    c->am_have_mark = false;
    const AmvmGeom a = amvm_geom(c);
    const double csp_mn = (double)c_sp * (double)m_rows * (double)n_cols;
    auto wall0 = std::chrono::steady_clock::now();
    auto phase = [&](const char* what) {
      if (!verbose()) return;
      c->sync();
      const auto now = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[hmgpu] mark %-10s %9.2f ms\n", what,
                   std::chrono::duration<double, std::milli>(now - wall0).count());
      wall0 = now;
    };
    c->d_nsq.ensure((size_t)std::max(nt, 1));
    c->d_cnt.ensure((size_t)M + 1);
    c->d_ptr.ensure((size_t)M + 1);
    c->d_lists.ensure((size_t)std::max<long long>(c->am_nvals, 1));
    c->d_keys.ensure((size_t)M);
    c->d_keys2.ensure((size_t)M);
    c->d_idx.ensure((size_t)M);
    c->d_order.ensure((size_t)M);
    c->d_resid.ensure((size_t)M);
    c->d_inset.ensure((size_t)std::max(nt, 1));
    c->d_marked.ensure((size_t)std::max(nt, 1));
    c->d_mids.ensure((size_t)std::max(nt, 1));
    c->d_nm.ensure(1);
    // term entries (ascending output index) and |term|^2
    c->d_eptr.ensure((size_t)nt + 1);
    c->d_eidx.ensure((size_t)std::max<long long>(c->am_nvals, 1));
    c->d_eval.ensure((size_t)std::max<long long>(c->am_nvals, 1));
    if (nt > 0) {
      c->d_ecnt.ensure((size_t)nt + 1);
      CK(cudaMemsetAsync(c->d_ecnt.p + nt, 0, sizeof(long long), c->stream));
      amvm_entries_kernel<<<(nt + 127) / 128, 128, 0, c->stream>>>(
          a, c->d_items.p, nt, 0, c->d_ecnt.p, nullptr, nullptr, nullptr, nullptr);
      size_t tbe = 0;
      CK(cub::DeviceScan::ExclusiveSum(nullptr, tbe, c->d_ecnt.p, c->d_eptr.p, nt + 1,
                                       c->stream));
      c->d_cub.ensure(tbe);
      CK(cub::DeviceScan::ExclusiveSum(c->d_cub.p, tbe, c->d_ecnt.p, c->d_eptr.p, nt + 1,
                                       c->stream));
      amvm_entries_kernel<<<(nt + 127) / 128, 128, 0, c->stream>>>(
          a, c->d_items.p, nt, 1, nullptr, c->d_eptr.p, c->d_eidx.p, c->d_eval.p, c->d_nsq.p);
    }
    phase("entries");
    const int gr = (c->n_rows + 127) / 128;
    CK(cudaMemsetAsync(c->d_cnt.p, 0, (M + 1) * sizeof(int), c->stream));
    amvm_cand_kernel<<<gr, 128, 0, c->stream>>>(a, c->d_sc.p, theta, csp_mn, 0, c->d_cnt.p,
                                                nullptr, nullptr);
    size_t tb1 = 0, tb2 = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tb1, c->d_cnt.p, c->d_ptr.p, (int)(M + 1),
                                     c->stream));
    CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb2, c->d_keys.p, c->d_keys2.p,
                                                 c->d_idx.p, c->d_order.p, (int)M, 0, 64,
                                                 c->stream));
    c->d_cub.ensure(std::max(tb1, tb2));
    CK(cub::DeviceScan::ExclusiveSum(c->d_cub.p, tb1, c->d_cnt.p, c->d_ptr.p, (int)(M + 1),
                                     c->stream));
    amvm_cand_kernel<<<gr, 128, 0, c->stream>>>(a, c->d_sc.p, theta, csp_mn, 1, c->d_cnt.p,
                                                c->d_ptr.p, c->d_lists.p);
    amvm_keys_kernel<<<(int)((M + 255) / 256), 256, 0, c->stream>>>(c->d_diff.p, M,
                                                                     c->d_keys.p, c->d_idx.p);
    CK(cub::DeviceRadixSort::SortPairsDescending(c->d_cub.p, tb2, c->d_keys.p, c->d_keys2.p,
                                                 c->d_idx.p, c->d_order.p, (int)M, 0, 64,
                                                 c->stream));
    phase("cand+sort");
    CK(cudaMemcpyAsync(c->d_resid.p, c->d_diff.p, M * sizeof(double),
                       cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemsetAsync(c->d_inset.p, 0, (size_t)std::max(nt, 1), c->stream));
    static const bool seq_walk = [] {
      const char* e = std::getenv("HMGPU_AMVM_WALK");
      return e && std::string(e) == "seq";
    }();
    if (seq_walk) {
      c->timed("amvm_walk", [&] {
        const int wsmem = 4 * kWalkSmem * (int)sizeof(double);
        CK(cudaFuncSetAttribute(amvm_walk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                wsmem));
        amvm_walk_kernel<<<1, 32, wsmem, c->stream>>>(
            c->d_sc.p, theta, c->d_order.p, M, c->d_ptr.p, c->d_lists.p, c->d_eptr.p,
            c->d_eidx.p, c->d_eval.p, c->d_nsq.p, c->d_resid.p, c->d_inset.p, c->d_marked.p,
            c->d_nm.p, c->d_sc.p + 2);
      });
    } else {
      parallel_walk(c, theta, M, nt);
    }
    phase("walk");
    if (verbose() && seq_walk) {
      double st[2];
      CK(cudaMemcpy(st, c->d_sc.p + 3, 2 * sizeof(double), cudaMemcpyDeviceToHost));
      std::fprintf(stderr, "[hmgpu] walk rows %.0f candidates %.0f\n", st[0], st[1]);
    }
    if (nt > 0)
      amvm_items_kernel<<<(nt + 255) / 256, 256, 0, c->stream>>>(c->d_aterms.p, c->d_marked.p,
                                                                 c->d_nm.p, c->d_mids.p);
    CK(cudaGetLastError());
    int nm = 0;
    double pk = 0.0;
    CK(cudaMemcpyAsync(&nm, c->d_nm.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(&pk, c->d_sc.p + 2, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    c->marked_ids.resize(nm);
    if (nm > 0)
      CK(cudaMemcpyAsync(c->marked_ids.data(), c->d_mids.p, nm * sizeof(int),
                         cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    phase("items");
    *n_marked = nm;
    *gamma_pk = pk;
    c->am_have_mark = true;
  });
}

int hmgpu_amvm_refine(hmgpu_ctx* c, int steps, int* comp_block) {
  return guard(c, [&] {
    if (!c->assembled) fail(HMGPU_ERR_STATE, "assemble first");
    if (steps < 0) fail(HMGPU_ERR_INVALID, "bad steps");
    // one refinement per marking: a second call would promote and extend
    // the same items again (2*steps pivots instead of steps)
    if (!c->am_have_mark) fail(HMGPU_ERR_STATE, "hmgpu_amvm_mark first");
    if (comp_block)
      for (size_t q = 0; q < c->marked_ids.size(); ++q) {
        comp_block[2 * q] = c->items[c->marked_ids[q]].comp;
        comp_block[2 * q + 1] = c->items[c->marked_ids[q]].block;
      }
    promote_ids(c, c->marked_ids);
    extend_ids(c, c->marked_ids, steps);
    c->am_have_estimate = false;
    c->am_have_mark = false;
    c->marked_ids.clear();
  });
}

namespace {
int tail_terms_impl(hmgpu_ctx* c, const double* x, int* n_terms, long long* n_vals,
                    long long* meta4, double* vals, bool transposed);
}
int hmgpu_tail_terms(hmgpu_ctx* c, const double* x, int* n_terms, long long* n_vals,
                     long long* meta4, double* vals) {
  return tail_terms_impl(c, x, n_terms, n_vals, meta4, vals, false);
}
int hmgpu_tail_terms_t(hmgpu_ctx* c, const double* x, int* n_terms, long long* n_vals,
                       long long* meta4, double* vals) {
  return tail_terms_impl(c, x, n_terms, n_vals, meta4, vals, true);
}
namespace {
int tail_terms_impl(hmgpu_ctx* c, const double* x, int* n_terms, long long* n_vals,
                    long long* meta4, double* vals, bool transposed) {
  return guard(c, [&] {
    if (!c->assembled) fail(HMGPU_ERR_STATE, "assemble first");
    if (!n_terms || !n_vals) fail(HMGPU_ERR_INVALID, "null outputs");
    std::vector<TailTerm> terms;
    long long off = 0;
    for (int b = 0; b < c->n_blocks; ++b) {
      const int i0 = c->item_of_block[b];
      if (i0 < 0) continue;
      for (int q = 0; q < c->NC; ++q) {
        const Item& it = c->items[i0 + q];
        if (it.k <= it.kcur) continue;
        const int nocc = (c->NC == 6 && c_comp_host_r(q) != c_comp_host_c(q)) ? 2 : 1;
        terms.push_back({i0 + q, nocc, off});
        off += (long long)nocc * (transposed ? it.n : it.m);
      }
    }
    // terms in component-major order (the by-H-matrix grouping of
    // gamma_contributions, amvm.cpp:135-150)
    std::stable_sort(terms.begin(), terms.end(), [&](const TailTerm& a, const TailTerm& b) {
      return c->items[a.item].comp < c->items[b.item].comp;
    });
    off = 0;
    for (TailTerm& t : terms) {
      t.off = off;
      off += (long long)t.nocc * (transposed ? c->items[t.item].n : c->items[t.item].m);
    }
    *n_terms = (int)terms.size();
    *n_vals = off;
    if (!meta4) return;
    if (!x || !vals) fail(HMGPU_ERR_INVALID, "null x/vals");
    for (size_t t = 0; t < terms.size(); ++t) {
      const Item& it = c->items[terms[t].item];
      meta4[4 * t] = it.comp;
      meta4[4 * t + 1] = it.block;
      meta4[4 * t + 2] = terms[t].nocc;
      meta4[4 * t + 3] = terms[t].off;
    }
    if (terms.empty()) return;
    const int NOUT = c->NC == 6 ? 3 : 1;
    const long long nx = transposed ? (long long)c->n_rows * NOUT : c->ndof_cols();
    c->d_x.ensure((size_t)nx);
    CK(cudaMemcpyAsync(c->d_x.p, x, nx * sizeof(double), cudaMemcpyHostToDevice,
                       c->stream));
    if (transposed) {
      c->d_xr.ensure((size_t)nx);
      const int gg = grid_for(c, (nx + 255) / 256);
      if (NOUT == 3)
        gather_kernel<3><<<gg, 256, 0, c->stream>>>(c->d_x.p, c->d_xr.p, c->d_rperm.p,
                                                     c->n_rows, 1);
      else
        gather_kernel<1><<<gg, 256, 0, c->stream>>>(c->d_x.p, c->d_xr.p, c->d_rperm.p,
                                                     c->n_rows, 1);
    } else {
      gather_x(c, c->d_x.p, 1);
    }
    DBuf<TailTerm> d_terms;
    d_terms.upload(terms, c->stream);
    DBuf<double> d_out;
    d_out.alloc((size_t)off);
    c->timed("tail", [&] {
      const int grid = grid_for(c, ((long long)terms.size() + 7) / 8, 8);
      if (transposed && c->NC == 6)
        tail_t_kernel<3><<<grid, 256, 0, c->stream>>>(d_terms.p, (int)terms.size(),
                                                     c->d_items.p, c->d_arena.p, c->d_xr.p,
                                                     d_out.p, 1);
      else if (transposed)
        tail_t_kernel<1><<<grid, 256, 0, c->stream>>>(d_terms.p, (int)terms.size(),
                                                     c->d_items.p, c->d_arena.p, c->d_xr.p,
                                                     d_out.p, 0);
      else if (c->NC == 6)
        tail_kernel<3><<<grid, 256, 0, c->stream>>>(d_terms.p, (int)terms.size(),
                                                   c->d_items.p, c->d_arena.p,
                                                   c->d_xi.p, d_out.p, 1);
      else
        tail_kernel<1><<<grid, 256, 0, c->stream>>>(d_terms.p, (int)terms.size(),
                                                   c->d_items.p, c->d_arena.p,
                                                   c->d_xi.p, d_out.p, 0);
    });
    CK(cudaMemcpyAsync(vals, d_out.p, off * sizeof(double), cudaMemcpyDeviceToHost,
                       c->stream));
    c->sync();
    d_terms.free();
    d_out.free();
  });
}
}  // namespace

int hmgpu_download_factor(hmgpu_ctx* c, int comp, int block, int* m, int* n, int* K,
                          int* k_cur, double* U, double* V, int* piv, double* frob_sq) {
  return guard(c, [&] {
    if (!c->assembled) fail(HMGPU_ERR_STATE, "assemble first");
    if (comp < 0 || comp >= c->NC || block < 0 || block >= c->n_blocks)
      fail(HMGPU_ERR_INVALID, "bad (comp, block)");
    const int i0 = c->item_of_block[block];
    if (i0 < 0) fail(HMGPU_ERR_INVALID, "block is dense or not owned");
    Item it;
    CK(cudaMemcpyAsync(&it, c->d_items.p + i0 + comp, sizeof(Item),
                       cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    if (m) *m = it.m;
    if (n) *n = it.n;
    if (K) *K = it.k;
    if (k_cur) *k_cur = it.kcur;
    if (frob_sq) *frob_sq = it.frob_sq;
    if (!U) return;
    if (!V || !piv) fail(HMGPU_ERR_INVALID, "null V/piv");
    CK(cudaMemcpyAsync(U, c->d_arena.p + it.u_off, sizeof(double) * it.m * it.k,
                       cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(V, c->d_arena.p + it.v_off, sizeof(double) * it.n * it.k,
                       cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(piv, c->d_piv.p + it.p_off, sizeof(int2) * it.k,
                       cudaMemcpyDeviceToHost, c->stream));
    c->sync();
  });
}

int hmgpu_download_dense(hmgpu_ctx* c, int comp, int block, double* out) {
  return guard(c, [&] {
    if (!c->assembled) fail(HMGPU_ERR_STATE, "assemble first");
    if (comp < 0 || comp >= c->NC || block < 0 || block >= c->n_blocks || !out)
      fail(HMGPU_ERR_INVALID, "bad (comp, block)");
    const int d = c->dense_of_block[block];
    if (d < 0) fail(HMGPU_ERR_INVALID, "block is low-rank or not owned");
    const DenseBlock& db = c->dblocks[d];
    const long long cp = align2((long long)db.m * c->NC);
    std::vector<double> tmp(db.n * cp);
    CK(cudaMemcpyAsync(tmp.data(), c->d_dense.p + db.off, sizeof(double) * tmp.size(),
                       cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    for (int j = 0; j < db.n; ++j)  // [j][comp][i] -> column-major m x n
      for (int i = 0; i < db.m; ++i)
        out[(long long)j * db.m + i] = tmp[j * cp + (long long)comp * db.m + i];
    c->sync();
  });
}

// per-item sums of hmgpu_storage on the device (the item table is 128 B per
// (component, block): ~180 MB at config 4, a host scan took 16 ms per AMVM
// sweep): current / tail entries, matvec flops, pivots; integer sums, so
// the atomics are exact and order independent
__global__ void storage_sums_kernel(const Item* __restrict__ items, int n, int nc,
                                    unsigned long long* __restrict__ acc) {
  unsigned long long cur = 0, tail = 0, fl = 0, piv = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const Item& it = items[i];
    const unsigned long long mn = (unsigned long long)(it.m + it.n);
    const unsigned long long kc = it.kcur > 0 ? it.kcur : 0, k = it.k > 0 ? it.k : 0;
    const unsigned long long w = (nc == 6 && c_comp_r[it.comp] != c_comp_c[it.comp]) ? 2 : 1;
    cur += kc * mn;
    tail += (k > kc ? k - kc : 0) * mn;
    fl += 2 * w * kc * mn;
    piv += k;
  }
  for (int o = 16; o > 0; o >>= 1) {
    cur += __shfl_xor_sync(0xffffffffu, cur, o);
    tail += __shfl_xor_sync(0xffffffffu, tail, o);
    fl += __shfl_xor_sync(0xffffffffu, fl, o);
    piv += __shfl_xor_sync(0xffffffffu, piv, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(acc, cur);
    atomicAdd(acc + 1, tail);
    atomicAdd(acc + 2, fl);
    atomicAdd(acc + 3, piv);
  }
}

int hmgpu_storage(hmgpu_ctx* c, hmgpu_storage_info* info) {
  return guard(c, [&] {
    if (!c->assembled) fail(HMGPU_ERR_STATE, "assemble first");
    if (!info) fail(HMGPU_ERR_INVALID, "null info");
    double cur = 0, tail = 0, dense = 0;
    long long flops = 0, pivots = 0;
    const int ni = (int)c->items.size();
    if (ni > 0) {
      DBuf<unsigned long long> acc;
      acc.alloc(4);
      CK(cudaMemsetAsync(acc.p, 0, 4 * sizeof(unsigned long long), c->stream));
      storage_sums_kernel<<<grid_for(c, (ni + 255) / 256, 4), 256, 0, c->stream>>>(
          c->d_items.p, ni, c->NC, acc.p);
      unsigned long long h[4];
      CK(cudaMemcpyAsync(h, acc.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
      c->sync();
      acc.free();
      cur = (double)h[0];
      tail = (double)h[1];
      flops = (long long)h[2];
      pivots = (long long)h[3];
    }
    for (const DenseBlock& d : c->dblocks) {
      for (int q = 0; q < c->NC; ++q) {
        const int w = (c->NC == 6 && c_comp_host_r(q) != c_comp_host_c(q)) ? 2 : 1;
        flops += 2LL * w * d.m * d.n;
      }
      dense += (double)c->NC * d.m * d.n;
    }
    info->mb_current = (cur + dense) * 8.0 / (1 << 20);
    info->mb_tail = tail * 8.0 / (1 << 20);
    info->mb_dense = dense * 8.0 / (1 << 20);
    info->mb_arena_allocated = (double)c->d_arena.n * 8.0 / (1 << 20);
    // compulsory traffic: every stored entry once + x read + y written
    info->matvec_bytes = (long long)(8.0 * (cur + dense)) +
                         8LL * (c->ndof_cols() + c->ndof_rows());
    info->matvec_flops = flops;
    info->pivots = pivots;
  });
}

int hmgpu_fp64_peak(int device, double* tflops) {
  if (!tflops) return HMGPU_ERR_INVALID;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return HMGPU_ERR_NODEVICE;
  if (device < 0 || device >= count) return HMGPU_ERR_INVALID;
  if (cudaSetDevice(device) != cudaSuccess) return HMGPU_ERR_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return HMGPU_ERR_OOM;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grid = sms * 8, iters = 1 << 14;
  dfma_peak_kernel<<<grid, 256>>>(out, 64, 1.0000001, 1e-9);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    dfma_peak_kernel<<<grid, 256>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    best = std::min(best, ms);
  }
  const cudaError_t e = cudaGetLastError();
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  if (e != cudaSuccess) return HMGPU_ERR_CUDA;
  const double flops = 2.0 * 8.0 * iters * (double)grid * 256.0;
  *tflops = flops / (best * 1e-3) / 1e12;
  return HMGPU_OK;
}

int hmgpu_dmma_peak(int device, double* tflops) {
  if (!tflops) return HMGPU_ERR_INVALID;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return HMGPU_ERR_NODEVICE;
  if (device < 0 || device >= count) return HMGPU_ERR_INVALID;
  if (cudaSetDevice(device) != cudaSuccess) return HMGPU_ERR_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return HMGPU_ERR_OOM;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grid = sms * 8, iters = 1 << 12;
  dmma_peak_kernel<<<grid, 256>>>(out, 64);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    dmma_peak_kernel<<<grid, 256>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    best = std::min(best, ms);
  }
  const cudaError_t e = cudaGetLastError();
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  if (e != cudaSuccess) return HMGPU_ERR_CUDA;
  const double flops = 512.0 * 8.0 * iters * (double)grid * 8.0;  // 8 warps per CTA
  *tflops = flops / (best * 1e-3) / 1e12;
  return HMGPU_OK;
}

int hmgpu_dmma_peak_sustained(int device, double seconds, double* tflops) {
  if (!tflops || !(seconds >= 0.2 && seconds <= 10.0)) return HMGPU_ERR_INVALID;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return HMGPU_ERR_NODEVICE;
  if (device < 0 || device >= count) return HMGPU_ERR_INVALID;
  if (cudaSetDevice(device) != cudaSuccess) return HMGPU_ERR_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return HMGPU_ERR_OOM;
  const int grid = sms * 8, iters = 1 << 12, batch = 8;
  const double flops = 512.0 * 8.0 * iters * (double)grid * 8.0;  // per launch
  cudaEvent_t ev[3];
  for (auto& e : ev) cudaEventCreate(&e);
  dmma_peak_kernel<<<grid, 256>>>(out, 64);  // warm-up
  // batches of launches until `seconds` have passed; the rate of the second half
  std::vector<float> ms;
  double total = 0.0;
  while (total < seconds * 1e3 && ms.size() < 100000) {
    cudaEventRecord(ev[0]);
    for (int r = 0; r < batch; ++r) dmma_peak_kernel<<<grid, 256>>>(out, iters);
    cudaEventRecord(ev[1]);
    if (cudaEventSynchronize(ev[1]) != cudaSuccess) break;
    float t = 0.f;
    cudaEventElapsedTime(&t, ev[0], ev[1]);
    ms.push_back(t);
    total += t;
  }
  const cudaError_t e = cudaGetLastError();
  for (auto& v : ev) cudaEventDestroy(v);
  cudaFree(out);
  if (e != cudaSuccess || ms.empty()) return HMGPU_ERR_CUDA;
  double t2 = 0.0;
  const size_t h = ms.size() / 2;
  for (size_t q = h; q < ms.size(); ++q) t2 += ms[q];
  *tflops = flops * batch * (double)(ms.size() - h) / (t2 * 1e-3) / 1e12;
  return HMGPU_OK;
}

int hmgpu_set_profiling(hmgpu_ctx* c, int on) {
  return guard(c, [&] { c->prof = on != 0; });
}

int hmgpu_kernel_times(hmgpu_ctx* c, const char* name, double* ms, long long* launches,
                       int reset) {
  return guard(c, [&] {
    if (!name) fail(HMGPU_ERR_INVALID, "null name");
    c->resolve_times();
    auto it = c->times.find(name);
    if (ms) *ms = it == c->times.end() ? 0.0 : it->second.ms;
    if (launches) *launches = it == c->times.end() ? 0 : it->second.launches;
    if (reset && it != c->times.end()) it->second = KTime{};
  });
}

}  // extern "C"
