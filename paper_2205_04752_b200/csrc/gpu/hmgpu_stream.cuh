// Streamed H-matvec (the bandwidth-bound sweep).
//
// The host packs the current-rank factors into a "stream arena" laid out in
// task order: every task's data (the V and/or U factors of a block and a
// group of Kelvin components, or a row tile of a dense near-field block) is
// ONE contiguous, 16-byte aligned run.  A persistent CTA double-buffers
// tasks in shared memory: one elected thread issues a TMA bulk copy
// (cp.async.bulk + mbarrier complete_tx) of task t+1 and of its x segment
// while all warps compute task t from shared memory.  Every task writes a
// partial result for its rows; a per-leaf pass sums the partials of all
// tasks covering a leaf in a fixed order (deterministic, no atomics) and
// scatters to external order.
//
// Reference: HMatrix::matvec (proj/src/hmatrix.cpp:22-45) over the six
// component H-matrices of the 3x3 Kelvin grid (BlockGrid matvec,
// proj/src/expr.cpp:197-215); an off-diagonal component factor is read once
// and applied to both x_c and x_r (cells (r,c) and (c,r)).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace hmgpu {

enum { TK_FUSED = 0, TK_VCOLS = 1, TK_YPART = 2, TK_DENSE = 3 };

// One streamed task: its data is one contiguous run of the stream arena
// (FUSED, VCOLS, YPART) or a row tile of a dense block (DENSE).
//   FUSED  [V_c (n x k_c) | U_c (m x k_c)] for c in [c0,c1): z in shared
//          memory, then the block rows of y (one partial row slot each)
//   VCOLS  columns [l0, l1) of V_c restricted to a row tile: z slots
//          (final, or per-tile partials summed by zreduce_kernel)
//   YPART  a row tile of [U_c (rows x k_c)] for all c, z from global
//   DENSE  a row tile of the [i][j][comp] near-field block
struct __align__(16) MvTask {
  int kind;
  int c0, c1;          // component range [c0, c1)
  int rows;            // FUSED: m; VCOLS: V tile rows; YPART/DENSE: tile rows
  int cols;            // FUSED/DENSE: n (block columns); VCOLS: l1 - l0
  int src;             // 0: stream arena, 1: dense arena
  int x_rows;          // rows of the x segment (0: none); YPART: z slots
  int x_col0;          // first internal column of the x segment
  long long data_off;  // doubles into the source arena
  long long out_off;   // FUSED/YPART/DENSE: partial-row slot; VCOLS: z slot
  long long z_off;     // YPART: first z slot of the block (comp-major)
  int data_len;        // doubles (even)
  int l0;              // VCOLS: first column
  int k[6];            // rank per component (0 outside [c0, c1))
  int pad[2];
};
static_assert(sizeof(MvTask) % 16 == 0, "MvTask layout");

struct ZReduce {  // zfinal[dst + e] = sum_t zpart[src + t*stride + e], e < len
  long long dst, src;
  int len, tiles, stride, pad;
};

struct LeafEntry {
  long long slot;  // partial-row slot of the task row that maps to leaf row `lo`
  int lo, hi;      // covered leaf rows [lo, hi) (relative to the leaf begin)
};

struct PackDesc {  // dst[l*rows + i] = src[l*ld + i], i < rows, l < cols
  long long src, dst;
  int ld, rows, cols, pad;
};

// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// TMA bulk copy global -> shared, completion signalled on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------------------
// Launch-wide constants of one streamed matvec.
struct StreamParams {
  const MvTask* tasks;
  int ntasks;
  int* counter;
  const double* arena;    // stream arena (packed current-rank factors)
  const double* dense;    // near-field arena ([i][j][comp] per block)
  const double* xi;       // gathered x, XS doubles per internal column
  double* ypart;          // partial rows: NOUT * nrhs doubles per slot
  double* zpart;          // z slots written by VCOLS (2 * nrhs doubles each)
  const double* zfinal;   // z slots read by YPART
  int nrhs;
  int xs;                 // doubles per x column (4*nrhs or 2*nrhs)
  int stage_doubles;      // data capacity of one stage
  int xbuf_doubles;       // x capacity of one stage
  int zbuf_doubles;       // z buffer (FUSED / YPART)
  int part_doubles;       // segment partial sums (<= blockDim)
};

template <int NC>
__device__ __forceinline__ int comp_r(int c) {
  return NC == 6 ? c_comp_r[c] : 0;
}
template <int NC>
__device__ __forceinline__ int comp_c(int c) {
  return NC == 6 ? c_comp_c[c] : 0;
}

// component index of the symmetric pair (r, s)
template <int NC>
__device__ __forceinline__ int comp_of(int r, int s) {
  if (NC == 1) return 0;
  const int lo = r < s ? r : s, hi = r < s ? s : r;
  return lo == 0 ? hi : (lo == 1 ? 2 + hi : 5);
}

// lanes per unit: a power of two T = 2^lg <= 32 with units * T <= blockDim
__device__ __forceinline__ int lanes_log2(int units, int max_len) {
  const int a = (int)blockDim.x / max(units, 1);
  const int m = min(min(a, max_len >> 2), 32);
  return m >= 1 ? 31 - __clz(m) : 0;
}
// sum over T = 2^lg adjacent lanes; uniform control flow (all lanes shuffle)
__device__ __forceinline__ double group_sum(double v, int T) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double other = __shfl_xor_sync(0xffffffffu, v, o);
    if (o < T) v += other;
  }
  return v;
}

// z[p*2*NR + o*NR + q] = sum_j V_c[j,l] x_{o ? R : C}[j][q] for the (c, l)
// pairs p of the task in component order.  T = 2^lg adjacent lanes share one
// (p, o, q) unit over strided j and combine with shuffles.  NR = nrhs when
// known at compile time (1), else 0 and `nrhs` is used.
template <int NC, int NR>
__device__ void stream_zdots(const MvTask& t, const double* V, int vrows, int ld,
                             const double* xs, int XS, int nrhs_rt, double* zout) {
  const int nrhs = NR > 0 ? NR : nrhs_rt;
  // component prefix sums in registers (no local-memory array)
  const int k0 = NC == 6 && t.c0 <= 0 && t.c1 > 0 ? t.k[0] : (NC == 1 ? t.k[0] : 0);
  const int k1 = NC == 6 && t.c0 <= 1 && t.c1 > 1 ? t.k[1] : 0;
  const int k2 = NC == 6 && t.c0 <= 2 && t.c1 > 2 ? t.k[2] : 0;
  const int k3 = NC == 6 && t.c0 <= 3 && t.c1 > 3 ? t.k[3] : 0;
  const int k4 = NC == 6 && t.c0 <= 4 && t.c1 > 4 ? t.k[4] : 0;
  const int k5 = NC == 6 && t.c0 <= 5 && t.c1 > 5 ? t.k[5] : 0;
  const int p1 = k0, p2 = p1 + k1, p3 = p2 + k2, p4 = p3 + k3, p5 = p4 + k4;
  const int npairs = p5 + k5;
  const int units = npairs * 2 * nrhs;
  const int lg = lanes_log2(units, vrows);
  const int T = 1 << lg;
  const int Wr = ((units << lg) + 31) & ~31;  // whole warps (shuffles)
  for (int w = threadIdx.x; w < Wr; w += blockDim.x) {
    const int seg = w & (T - 1);
    const int u = w >> lg;
    double s = 0.0;
    if (u < units) {
      const int q = NR == 1 ? 0 : u % nrhs;
      const int uq = NR == 1 ? u : u / nrhs;
      const int o = uq & 1;
      const int p = uq >> 1;
      const int c = NC == 1 ? 0
                            : (p >= p1) + (p >= p2) + (p >= p3) + (p >= p4) + (p >= p5);
      const int base = c == 0 ? 0 : c == 1 ? p1 : c == 2 ? p2 : c == 3 ? p3 : c == 4 ? p4 : p5;
      const int l = p - base;
      const int rr = comp_r<NC>(c), cc = comp_c<NC>(c);
      if (o == 0 || rr != cc) {
        const double* vl = V + (long long)ld * base + (long long)l * ld;
        const double* xb = xs + (o == 0 ? cc : rr) * nrhs + q;
#pragma unroll 4
        for (int j = seg; j < vrows; j += T) s = fma(vl[j], xb[j * XS], s);
      }
    }
    s = group_sum(s, T);
    if (seg == 0 && u < units) zout[u] = s;
  }
}

// y[i][r][q] = sum over components (r,s) of U_(r,s)[i,:] z_(r,s)[:, r > s]
template <int NC, int NR>
__device__ void stream_urows(const MvTask& t, const double* U, int urows, const double* z,
                             int nrhs_rt, double* yout) {
  constexpr int NOUT = NC == 6 ? 3 : 1;
  const int nrhs = NR > 0 ? NR : nrhs_rt;
  int kmax = 1;
  for (int c = t.c0; c < t.c1; ++c) kmax = max(kmax, t.k[c]);
  const int units = urows * NOUT * nrhs;
  const int lg = lanes_log2(units, 3 * kmax);
  const int T = 1 << lg;
  const int Wr = ((units << lg) + 31) & ~31;
  for (int w = threadIdx.x; w < Wr; w += blockDim.x) {
    const int seg = w & (T - 1);
    const int u = w >> lg;
    double acc = 0.0;
    if (u < units) {
      const int q = NR == 1 ? 0 : u % nrhs;
      const int ur = NR == 1 ? u : u / nrhs;
      const int r = NOUT == 1 ? 0 : ur % NOUT;
      const int i = NOUT == 1 ? ur : ur / NOUT;
      long long uoff = 0;
      int slot = 0, e = 0;
      for (int c = t.c0; c < t.c1; ++c) {
        const int k = t.k[c];
        const int rr = comp_r<NC>(c), cc = comp_c<NC>(c);
        const int o = rr == r ? 0 : (cc == r ? 1 : -1);
        if (o >= 0) {
          const double* uu = U + uoff + i;
          const double* zz = z + slot * 2 * nrhs + o * nrhs + q;
          // term e runs over the (c, l) pairs touching r; lane seg takes e = seg mod T
          const int l0 = (seg - e) & (T - 1);
#pragma unroll 4
          for (int l = l0; l < k; l += T) acc = fma(uu[l * urows], zz[l * 2 * nrhs], acc);
          e += k;
        }
        uoff += (long long)urows * k;
        slot += k;
      }
    }
    acc = group_sum(acc, T);
    if (seg == 0 && u < units) yout[u] = acc;
  }
}

// dense row tile: y[i][r][q] = sum_j sum_s A_(r,s)[i][j] x_s[j][q]
template <int NC, int NR>
__device__ void stream_dense(const MvTask& t, const double* D, const double* xs, int XS,
                             int nrhs_rt, double* yout) {
  constexpr int NOUT = NC == 6 ? 3 : 1;
  const int nrhs = NR > 0 ? NR : nrhs_rt;
  const int pitch = (t.cols * NC + 1) & ~1;  // rows padded to 16 bytes
  const int units = t.rows * NOUT * nrhs;
  const int lg = lanes_log2(units, t.cols);
  const int T = 1 << lg;
  const int Wr = ((units << lg) + 31) & ~31;
  for (int w = threadIdx.x; w < Wr; w += blockDim.x) {
    const int seg = w & (T - 1);
    const int u = w >> lg;
    double acc = 0.0;
    if (u < units) {
      const int q = NR == 1 ? 0 : u % nrhs;
      const int ur = NR == 1 ? u : u / nrhs;
      const int r = NOUT == 1 ? 0 : ur % NOUT;
      const int i = NOUT == 1 ? ur : ur / NOUT;
      const double* d = D + i * pitch;
      const int c0 = comp_of<NC>(r, 0), c1 = comp_of<NC>(r, 1), c2 = comp_of<NC>(r, 2);
#pragma unroll 2
      for (int j = seg; j < t.cols; j += T) {
        const double* xj = xs + j * XS + q;
        const double* dj = d + j * NC;
        acc = fma(dj[c0], xj[0], acc);
        if (NOUT == 3) {
          acc = fma(dj[c1], xj[nrhs], acc);
          acc = fma(dj[c2], xj[2 * nrhs], acc);
        }
      }
    }
    acc = group_sum(acc, T);
    if (seg == 0 && u < units) yout[u] = acc;
  }
}

// Persistent CTAs, static round-robin task assignment (tasks sorted by
// size), NSTAGE-deep TMA pipeline: the task descriptor, its data and its x
// segment arrive as one mbarrier transaction; after consuming task k the
// elected thread refills the stage with task k + NSTAGE.
template <int NC, int NSTAGE, int NR>
__global__ void __launch_bounds__(256, 1)
hmv_stream_kernel(StreamParams P) {
  constexpr int NOUT = NC == 6 ? 3 : 1;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar[NSTAGE];
  __shared__ __align__(16) MvTask tdesc[NSTAGE];
  const int stage_total = P.stage_doubles + P.xbuf_doubles;
  double* zbuf = sm + (long long)NSTAGE * stage_total;
  const int G = gridDim.x;

  auto issue = [&](int ti, int s) {
    const MvTask& t = P.tasks[ti];
    const uint32_t dbytes = (uint32_t)t.data_len * 8u;
    // x segment, or (YPART) the task's z slots, into the stage's x area
    const bool ztask = t.kind == TK_YPART;
    const uint32_t xbytes = ztask ? (uint32_t)t.x_rows * 2u * (uint32_t)P.nrhs * 8u
                                  : (uint32_t)t.x_rows * (uint32_t)P.xs * 8u;
    mbar_expect_tx(&bar[s], dbytes + xbytes + (uint32_t)sizeof(MvTask));
    bulk_g2s(&tdesc[s], &P.tasks[ti], (uint32_t)sizeof(MvTask), &bar[s]);
    double* dst = sm + (long long)s * stage_total;
    if (dbytes)
      bulk_g2s(dst, (t.src == 0 ? P.arena : P.dense) + t.data_off, dbytes, &bar[s]);
    if (xbytes)
      bulk_g2s(dst + P.stage_doubles,
               ztask ? P.zfinal + t.z_off * 2 * P.nrhs : P.xi + (long long)t.x_col0 * P.xs,
               xbytes, &bar[s]);
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int s = 0; s < NSTAGE; ++s) {
      const int t = blockIdx.x + s * G;
      if (t < P.ntasks) issue(t, s);
    }
  const int nrhs = P.nrhs;
  for (int kk = 0;; ++kk) {
    const int ti = blockIdx.x + kk * G;
    if (ti >= P.ntasks) break;
    const int s = kk % NSTAGE;
    mbar_wait(&bar[s], (uint32_t)((kk / NSTAGE) & 1));
    const MvTask& t = tdesc[s];
    const double* data = sm + (long long)s * stage_total;
    const double* xs = data + P.stage_doubles;
    if (t.kind == TK_DENSE) {
      stream_dense<NC, NR>(t, data, xs, P.xs, nrhs, P.ypart + t.out_off * NOUT * nrhs);
    } else if (t.kind == TK_VCOLS) {
      stream_zdots<NC, NR>(t, data, t.rows, t.rows, xs, P.xs, nrhs,
                           P.zpart + t.out_off * 2 * nrhs);
    } else if (t.kind == TK_FUSED) {
      int ksum = 0;
      for (int c = t.c0; c < t.c1; ++c) ksum += t.k[c];
      stream_zdots<NC, NR>(t, data, t.cols, t.cols, xs, P.xs, nrhs, zbuf);
      __syncthreads();
      stream_urows<NC, NR>(t, data + (long long)t.cols * ksum, t.rows, zbuf, nrhs,
                           P.ypart + t.out_off * NOUT * nrhs);
    } else {  // TK_YPART: z slots arrived in the x area (x_rows = slot count)
      stream_urows<NC, NR>(t, data, t.rows, xs, nrhs, P.ypart + t.out_off * NOUT * nrhs);
    }
    __syncthreads();  // stage s consumed
    if (threadIdx.x == 0) {
      const int tn = ti + NSTAGE * G;
      if (tn < P.ntasks) {
        fence_proxy_async();
        issue(tn, s);
      }
    }
  }
}

// zfinal = sum of per-row-tile z partials, fixed order
__global__ void zreduce_kernel(const ZReduce* __restrict__ d, int n,
                               const double* __restrict__ zpart,
                               double* __restrict__ zfinal, int unit) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = gw; t < n; t += nw) {
    const ZReduce r = d[t];
    const long long len = (long long)r.len * unit;
    for (long long e = lane; e < len; e += 32) {
      double s = 0.0;
      for (int k = 0; k < r.tiles; ++k) s += zpart[(r.src + (long long)k * r.stride) * unit + e];
      zfinal[r.dst * unit + e] = s;
    }
  }
}


// per leaf: y(p) = sum over covering task rows (fixed order)
template <int NOUT>
__global__ void hmv_leaf_reduce_kernel(const int* __restrict__ leaf_begin,
                                       const int* __restrict__ leaf_end,
                                       const int* __restrict__ leaf_ptr,
                                       const LeafEntry* __restrict__ entries, int nleaves,
                                       const double* __restrict__ ypart,
                                       const int* __restrict__ rperm, int nrows,
                                       double* __restrict__ y, int nrhs) {
  const long long ndof = (long long)nrows * NOUT;
  for (int L = blockIdx.x; L < nleaves; L += gridDim.x) {
    const int b0 = leaf_begin[L], b1 = leaf_end[L];
    const int e0 = leaf_ptr[L], e1 = leaf_ptr[L + 1];
    const int cnt = (b1 - b0) * NOUT * nrhs;
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
      const int q = t % nrhs;
      const int r = (t / nrhs) % NOUT;
      const int i = t / (nrhs * NOUT);
      double s = 0.0;
      for (int e = e0; e < e1; ++e) {
        const LeafEntry en = entries[e];
        if (i >= en.lo && i < en.hi)
          s += ypart[((en.slot + (i - en.lo)) * NOUT + r) * nrhs + q];
      }
      y[q * ndof + (long long)r * nrows + rperm[b0 + i]] = s;
    }
  }
}

// gather x into the stream layout: XS doubles per internal column
template <int NOUT>
__global__ void gather_stream_kernel(const double* __restrict__ x, double* __restrict__ xi,
                                     const int* __restrict__ cperm, int ncols, int nrhs,
                                     int xs) {
  const long long total = (long long)ncols * xs;
  const long long ndof = (long long)ncols * NOUT;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int p = (int)(t / xs);
    const int w = (int)(t % xs);
    const int r = w / nrhs, q = w % nrhs;
    xi[t] = r < NOUT ? x[q * ndof + (long long)r * ncols + cperm[p]] : 0.0;
  }
}

// pack current-rank factor columns into the stream arena
__global__ void pack_kernel(const PackDesc* __restrict__ d, int n,
                            const double* __restrict__ src, double* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = gw; t < n; t += nw) {
    const PackDesc p = d[t];
    const long long tot = (long long)p.rows * p.cols;
    for (long long e = lane; e < tot; e += 32) {
      const long long l = e / p.rows, i = e % p.rows;
      dst[p.dst + e] = src[p.src + l * p.ld + i];
    }
  }
}

}  // namespace hmgpu
