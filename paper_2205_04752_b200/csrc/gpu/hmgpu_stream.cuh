// Streamed H-matvec (the bandwidth-bound sweep), warp-private pipelines.
//
// The host packs the current-rank factors into a "stream arena" in job
// order.  A job is processed by ONE warp; its data is a sequence of chunks,
// each one contiguous, 16-byte aligned run that a lane-0 TMA bulk copy
// (cp.async.bulk + mbarrier complete_tx) brings into the warp's private
// NS-deep ring in shared memory while the warp computes the previous chunk.
// No block-level barriers: warps only __syncwarp.
//
// Job kinds (one partial output row slot per block row):
//   FUSED  low-rank block with m, n <= 64: V part packed row-major
//          [j][g] (lane = column g: conflict-free), x with the first chunk;
//          per column the three dot products f_s = V_g . x_s give the
//          weights W[g][r] = (R==r) f_C + (C==r, R!=C) f_R; U part packed
//          column-major [g][i] (lane = row i): y_r += U[i,g] W[g][r]
//   VSPLIT up to 64 consecutive columns of the K = sum k_c columns of a
//          large block (across components, packed row-major [j][g] like
//          FUSED; lane = column, a second column at lane + 32), all rows
//          streamed in row chunks (x rows with each chunk); W to global
//   USPLIT a <= 64-row tile of all components' U of a large block; W of
//          the block from global with the first chunk
//   DENSE  a near-field block ([j][c][i] layout), m <= 64, x with chunk 0
// A per-leaf pass sums the partial rows of all blocks covering a leaf in a
// fixed order (deterministic, no atomics) and scatters to external order.
//
// Reference: HMatrix::matvec (proj/src/hmatrix.cpp:22-45) over the six
// component H-matrices of the 3x3 Kelvin grid (BlockGrid matvec,
// proj/src/expr.cpp:197-215); each off-diagonal component factor is read
// once and applied to both x_c and x_r.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace hmgpu {

enum { WJ_FUSED = 0, WJ_VSPLIT = 1, WJ_USPLIT = 2, WJ_DENSE = 3 };

struct __align__(16) WJob {
  int kind;
  int m;           // rows of the output tile (FUSED/USPLIT/DENSE); VSPLIT: 0
  int n;           // FUSED/DENSE: block columns; VSPLIT: rows of V
  int ncols;       // FUSED/USPLIT: K = sum k_c; VSPLIT: columns (<= 32); DENSE: n
  int chain;       // row jobs: the warp's next job adds to the same rows (keep y)
  int row0;        // row jobs: first internal row (host bookkeeping); VSPLIT: -1
  int comp;        // VSPLIT: first column (of the block's K) of the job
  int vrows;       // FUSED: V part streamed in row chunks (K <= 64), x with each
  long long out;   // FUSED/USPLIT/DENSE: partial row slot of its chain; VSPLIT: W slot of column 0
  int kp[8];       // FUSED/USPLIT: component prefix sums of the K columns
};
static_assert(sizeof(WJob) == 80, "WJob layout");

enum { WA_NONE = 0, WA_X = 1, WA_W = 2 };

struct __align__(16) WChunk {
  long long src;   // doubles into the arena (src_kind 0) or the dense arena (1)
  long long aux;   // WA_X: internal column of x; WA_W: W slot
  int len;         // doubles of data (even)
  int src_kind;
  int aux_kind;
  int aux_len;     // rows (WA_X) or columns (WA_W), 4 doubles each
  int g0, g1;      // column range (FUSED V/U part, USPLIT, DENSE) or row range (VSPLIT)
  int part;        // FUSED: 0 = V part, 1 = U part
  int job;         // index of the chunk's job in the job table
};
static_assert(sizeof(WChunk) == 48, "WChunk layout");

struct LeafEntry {
  long long slot;  // partial-row slot of the job row that maps to leaf row `lo`
  int lo, hi;      // covered leaf rows [lo, hi) (relative to the leaf begin)
};

// dst = pack of src (column-major, leading dimension ld) rows x cols:
// trans = 0: column-major dst[l*dld + i]; trans = 1: row-major dst[i*dld + l]
struct PackDesc {
  long long src, dst;
  int ld, dld, rows, cols, trans, pad;
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
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------------------
struct WarpStreamParams {
  const WJob* jobs;
  const WChunk* chunks;   // warp-major: warp w's static share at [woff[w], woff[w+1]),
  const int* woff;        // then the pool: group g at [goff[g], goff[g+1])
  const int* goff;
  int ngroups;            // pooled groups (the pass's smallest chain units), pulled from
  int* ctr;               // *ctr by warps that finished their share (zeroed by the gather)
  int nwarps;             // warps the chunk table was laid out for
  const double* arena;   // packed factors
  const double* dense;   // near-field blocks, [j][c][i] per block
  const double* xi;      // gathered x, 4 doubles per internal column (x, y, z, 0)
  double* wout;          // W slots written by VSPLIT (4 doubles each)
  const double* win;     // W slots read by USPLIT
  double* ypart;         // partial rows, 3 doubles each (1 for scalar kernels)
  int stage;             // doubles per stage (data + aux)
  int scratch;           // doubles of per-warp job scratch
  unsigned long long* prof;  // -DHMGPU_MV_PROF: cycles of every warp's chunk loop (balance)
};

template <int NC>
struct Comp {  // (R, C) of component c of the symmetric 3x3 grid
  __device__ static __forceinline__ int r(int c) { return NC == 6 ? c_comp_r[c] : 0; }
  __device__ static __forceinline__ int col(int c) { return NC == 6 ? c_comp_c[c] : 0; }
};

// component of column g from the prefix sums kp[0..6]
__device__ __forceinline__ int comp_of_col(const int* kp, int g) {
  return (g >= kp[1]) + (g >= kp[2]) + (g >= kp[3]) + (g >= kp[4]) + (g >= kp[5]);
}

// W[g][r] from the three dot products f_s of a column of component c
template <int NC>
__device__ __forceinline__ void weights(int c, double f0, double f1, double f2, double* w) {
  if (NC == 1) {
    w[0] = f0;
    w[1] = w[2] = w[3] = 0.0;
    return;
  }
  const int R = Comp<NC>::r(c), C = Comp<NC>::col(c);
  const double fC = C == 0 ? f0 : (C == 1 ? f1 : f2);
  const double fR = R == 0 ? f0 : (R == 1 ? f1 : f2);
  const bool off = R != C;
  w[0] = (R == 0 ? fC : 0.0) + (off && C == 0 ? fR : 0.0);
  w[1] = (R == 1 ? fC : 0.0) + (off && C == 1 ? fR : 0.0);
  w[2] = (R == 2 ? fC : 0.0) + (off && C == 2 ? fR : 0.0);
  w[3] = 0.0;
}

// f_s += sum_j V[j][col] x_s[j] over rows [0, nrows) of a row-major chunk
// (row length rl); x rows at xs (4 doubles per row)
template <int NC>
__device__ __forceinline__ void vdots(const double* V, int rl, int nrows, const double* xs,
                                      int col, double& f0, double& f1, double& f2) {
  // four independent accumulator sets (rows j mod 4) for ILP
  double a0[4] = {0, 0, 0, 0}, a1[4] = {0, 0, 0, 0}, a2[4] = {0, 0, 0, 0};
  int j = 0;
  for (; j + 3 < nrows; j += 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double v = V[(j + u) * rl + col];
      const double2 x01 = *reinterpret_cast<const double2*>(xs + 4 * (j + u));
      a0[u] = fma(v, x01.x, a0[u]);
      if (NC == 6) {
        a1[u] = fma(v, x01.y, a1[u]);
        a2[u] = fma(v, xs[4 * (j + u) + 2], a2[u]);
      }
    }
  }
  for (; j < nrows; ++j) {
    const double v = V[j * rl + col];
    a0[0] = fma(v, xs[4 * j], a0[0]);
    if (NC == 6) {
      a1[0] = fma(v, xs[4 * j + 1], a1[0]);
      a2[0] = fma(v, xs[4 * j + 2], a2[0]);
    }
  }
  f0 += (a0[0] + a0[1]) + (a0[2] + a0[3]);
  f1 += (a1[0] + a1[1]) + (a1[2] + a1[3]);
  f2 += (a2[0] + a2[1]) + (a2[2] + a2[3]);
}

// vdots for the two columns col and col + 32 of one lane in a single sweep
// over the rows (the x row loads shared); each column's arithmetic is that
// of vdots (same accumulators, same order).  Used when a chunk has more
// than 32 columns: one pass instead of two with the second mostly idle.
template <int NC>
__device__ __forceinline__ void vdots2(const double* V, int rl, int nrows, const double* xs,
                                       int col, bool two, double* f) {
  double a0[4] = {0, 0, 0, 0}, a1[4] = {0, 0, 0, 0}, a2[4] = {0, 0, 0, 0};
  double b0[4] = {0, 0, 0, 0}, b1[4] = {0, 0, 0, 0}, b2[4] = {0, 0, 0, 0};
  const int col2 = two ? col + 32 : col;
  int j = 0;
  for (; j + 3 < nrows; j += 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double v = V[(j + u) * rl + col];
      const double w = V[(j + u) * rl + col2];
      const double2 x01 = *reinterpret_cast<const double2*>(xs + 4 * (j + u));
      a0[u] = fma(v, x01.x, a0[u]);
      b0[u] = fma(w, x01.x, b0[u]);
      if (NC == 6) {
        const double x2 = xs[4 * (j + u) + 2];
        a1[u] = fma(v, x01.y, a1[u]);
        a2[u] = fma(v, x2, a2[u]);
        b1[u] = fma(w, x01.y, b1[u]);
        b2[u] = fma(w, x2, b2[u]);
      }
    }
  }
  for (; j < nrows; ++j) {
    const double v = V[j * rl + col];
    const double w = V[j * rl + col2];
    a0[0] = fma(v, xs[4 * j], a0[0]);
    b0[0] = fma(w, xs[4 * j], b0[0]);
    if (NC == 6) {
      a1[0] = fma(v, xs[4 * j + 1], a1[0]);
      a2[0] = fma(v, xs[4 * j + 2], a2[0]);
      b1[0] = fma(w, xs[4 * j + 1], b1[0]);
      b2[0] = fma(w, xs[4 * j + 2], b2[0]);
    }
  }
  f[0] = 0.0 + ((a0[0] + a0[1]) + (a0[2] + a0[3]));
  f[1] = 0.0 + ((a1[0] + a1[1]) + (a1[2] + a1[3]));
  f[2] = 0.0 + ((a2[0] + a2[1]) + (a2[2] + a2[3]));
  f[3] = 0.0 + ((b0[0] + b0[1]) + (b0[2] + b0[3]));
  f[4] = 0.0 + ((b1[0] + b1[1]) + (b1[2] + b1[3]));
  f[5] = 0.0 + ((b2[0] + b2[1]) + (b2[2] + b2[3]));
}

// y rows (lane, lane + 32) += sum_g U[g][i] W[g][:] over columns [0, ncol)
// of a column-major chunk with m rows
template <int NC>
__device__ __forceinline__ void urows1(const double* U, int m, int ncol, const double* W,
                                       int lane, double* y) {
  // m <= 32: one row per lane, four column accumulator sets
  double a[4][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  const int i = lane < m ? lane : 0;
  int g = 0;
  for (; g + 3 < ncol; g += 4) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const double2 w01 = *reinterpret_cast<const double2*>(W + 4 * (g + e));
      const double u = U[(g + e) * m + i];
      a[e][0] = fma(u, w01.x, a[e][0]);
      if (NC == 6) {
        a[e][1] = fma(u, w01.y, a[e][1]);
        a[e][2] = fma(u, W[4 * (g + e) + 2], a[e][2]);
      }
    }
  }
  for (; g < ncol; ++g) {
    const double u = U[g * m + i];
    a[0][0] = fma(u, W[4 * g], a[0][0]);
    if (NC == 6) {
      a[0][1] = fma(u, W[4 * g + 1], a[0][1]);
      a[0][2] = fma(u, W[4 * g + 2], a[0][2]);
    }
  }
  if (lane < m) {
    y[0] += (a[0][0] + a[1][0]) + (a[2][0] + a[3][0]);
    y[1] += (a[0][1] + a[1][1]) + (a[2][1] + a[3][1]);
    y[2] += (a[0][2] + a[1][2]) + (a[2][2] + a[3][2]);
  }
}

template <int NC>
__device__ __forceinline__ void urows(const double* U, int m, int ncol, const double* W,
                                      int lane, double* y) {
  if (m <= 32) {
    urows1<NC>(U, m, ncol, W, lane, y);
    return;
  }
  const bool r0 = lane < m, r1 = lane + 32 < m;
  const int i1 = r1 ? lane + 32 : lane;  // keeps the second load in bounds
  double a[2][3] = {{0, 0, 0}, {0, 0, 0}}, c[2][3] = {{0, 0, 0}, {0, 0, 0}};
  int g = 0;
  for (; g + 1 < ncol; g += 2) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const double2 w01 = *reinterpret_cast<const double2*>(W + 4 * (g + e));
      const double w2 = W[4 * (g + e) + 2];
      const double u = U[(g + e) * m + lane];
      const double v = U[(g + e) * m + i1];
      a[e][0] = fma(u, w01.x, a[e][0]);
      c[e][0] = fma(v, w01.x, c[e][0]);
      if (NC == 6) {
        a[e][1] = fma(u, w01.y, a[e][1]);
        a[e][2] = fma(u, w2, a[e][2]);
        c[e][1] = fma(v, w01.y, c[e][1]);
        c[e][2] = fma(v, w2, c[e][2]);
      }
    }
  }
  if (g < ncol) {
    const double2 w01 = *reinterpret_cast<const double2*>(W + 4 * g);
    const double w2 = W[4 * g + 2];
    const double u = U[g * m + lane];
    const double v = U[g * m + i1];
    a[0][0] = fma(u, w01.x, a[0][0]);
    c[0][0] = fma(v, w01.x, c[0][0]);
    if (NC == 6) {
      a[0][1] = fma(u, w01.y, a[0][1]);
      a[0][2] = fma(u, w2, a[0][2]);
      c[0][1] = fma(v, w01.y, c[0][1]);
      c[0][2] = fma(v, w2, c[0][2]);
    }
  }
  if (r0) {
    y[0] += a[0][0] + a[1][0];
    y[1] += a[0][1] + a[1][1];
    y[2] += a[0][2] + a[1][2];
  }
  if (r1) {
    y[3] += c[0][0] + c[1][0];
    y[4] += c[0][1] + c[1][1];
    y[5] += c[0][2] + c[1][2];
  }
}

// dense chunk columns [0, ncol): D[j][c][i] (column stride cp), x rows xs.
// Two accumulator sets (even / odd columns) so that the three-deep FMA
// chains of consecutive columns overlap.
template <int NC>
__device__ __forceinline__ void drows(const double* D, int m, int cp, int ncol,
                                      const double* xs, int lane, double* y) {
  const bool r0 = lane < m, r1 = lane + 32 < m;
  double a[2][3] = {{0, 0, 0}, {0, 0, 0}}, c[2][3] = {{0, 0, 0}, {0, 0, 0}};
  int j = 0;
  for (; j + 1 < ncol; j += 2) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const double* d = D + (j + h) * cp;
      const double2 x01 = *reinterpret_cast<const double2*>(xs + 4 * (j + h));
      const double x2 = xs[4 * (j + h) + 2];
      if (NC == 6) {
        const double p00 = r0 ? d[lane] : 0.0, p01 = r0 ? d[m + lane] : 0.0,
                     p02 = r0 ? d[2 * m + lane] : 0.0, p11 = r0 ? d[3 * m + lane] : 0.0,
                     p12 = r0 ? d[4 * m + lane] : 0.0, p22 = r0 ? d[5 * m + lane] : 0.0;
        a[h][0] = fma(p00, x01.x, fma(p01, x01.y, fma(p02, x2, a[h][0])));
        a[h][1] = fma(p01, x01.x, fma(p11, x01.y, fma(p12, x2, a[h][1])));
        a[h][2] = fma(p02, x01.x, fma(p12, x01.y, fma(p22, x2, a[h][2])));
        if (r1) {
          const int i = lane + 32;
          const double q00 = d[i], q01 = d[m + i], q02 = d[2 * m + i], q11 = d[3 * m + i],
                       q12 = d[4 * m + i], q22 = d[5 * m + i];
          c[h][0] = fma(q00, x01.x, fma(q01, x01.y, fma(q02, x2, c[h][0])));
          c[h][1] = fma(q01, x01.x, fma(q11, x01.y, fma(q12, x2, c[h][1])));
          c[h][2] = fma(q02, x01.x, fma(q12, x01.y, fma(q22, x2, c[h][2])));
        }
      } else {
        a[h][0] = fma(r0 ? d[lane] : 0.0, x01.x, a[h][0]);
        c[h][0] = fma(r1 ? d[lane + 32] : 0.0, x01.x, c[h][0]);
      }
    }
  }
  if (j < ncol) {
    const double* d = D + j * cp;
    const double2 x01 = *reinterpret_cast<const double2*>(xs + 4 * j);
    const double x2 = xs[4 * j + 2];
    if (NC == 6) {
      const double p00 = r0 ? d[lane] : 0.0, p01 = r0 ? d[m + lane] : 0.0,
                   p02 = r0 ? d[2 * m + lane] : 0.0, p11 = r0 ? d[3 * m + lane] : 0.0,
                   p12 = r0 ? d[4 * m + lane] : 0.0, p22 = r0 ? d[5 * m + lane] : 0.0;
      a[0][0] = fma(p00, x01.x, fma(p01, x01.y, fma(p02, x2, a[0][0])));
      a[0][1] = fma(p01, x01.x, fma(p11, x01.y, fma(p12, x2, a[0][1])));
      a[0][2] = fma(p02, x01.x, fma(p12, x01.y, fma(p22, x2, a[0][2])));
      if (r1) {
        const int i = lane + 32;
        const double q00 = d[i], q01 = d[m + i], q02 = d[2 * m + i], q11 = d[3 * m + i],
                     q12 = d[4 * m + i], q22 = d[5 * m + i];
        c[0][0] = fma(q00, x01.x, fma(q01, x01.y, fma(q02, x2, c[0][0])));
        c[0][1] = fma(q01, x01.x, fma(q11, x01.y, fma(q12, x2, c[0][1])));
        c[0][2] = fma(q02, x01.x, fma(q12, x01.y, fma(q22, x2, c[0][2])));
      }
    } else {
      a[0][0] = fma(r0 ? d[lane] : 0.0, x01.x, a[0][0]);
      c[0][0] = fma(r1 ? d[lane + 32] : 0.0, x01.x, c[0][0]);
    }
  }
  y[0] += a[0][0] + a[1][0];
  y[1] += a[0][1] + a[1][1];
  y[2] += a[0][2] + a[1][2];
  y[3] += c[0][0] + c[1][0];
  y[4] += c[0][1] + c[1][1];
  y[5] += c[0][2] + c[1][2];
}

// Warp-private pipelines: WARPS warps per CTA, each with NS stages of
// P.stage doubles and P.scratch doubles of job scratch.  Jobs are assigned
// round-robin over all warps of the grid (the host sorts them by size).
// Stage layout: [WChunk | WJob] header (128 B), data, aux -- descriptors
// arrive in the same mbarrier transaction as the data.
constexpr int kHdr = 16;  // doubles of stage header

// POOL: the warp goes on with groups from the pass's pool after its static
// share (layouts with a pool only: the cursor costs ~2 % where there is none)
template <int NC, int NS, int WARPS, bool POOL>
__global__ void __launch_bounds__(WARPS * 32, 1)
hmv_warp_kernel(WarpStreamParams P) {
  constexpr int NOUT = NC == 6 ? 3 : 1;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bars[WARPS * NS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * WARPS + warp;
  double* ring = sm + (long long)warp * (NS * P.stage + P.scratch);
  double* scratch = ring + NS * P.stage;
  uint64_t* bar = bars + warp * NS;

  if (lane == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
  }
  __syncwarp();

  // This warp's chunk sequence: its static share, then groups pulled from
  // the pool's counter, one after the other without draining the ring (the
  // next group is fetched while the current range streams).  Descriptors are
  // fetched 32 at a time (one coalesced load, lane l holds chunk win_base +
  // l) and handed to lane 0 by shuffles when it issues, so no global latency
  // sits on the issue path.
  int gq = gw < P.nwarps ? P.woff[gw] : 0;        // current range: next chunk, end
  int gend = gw < P.nwarps ? P.woff[gw + 1] : 0;
  int nq = -1, nend = -1;                          // prefetched pool group (-1: pool empty)
  int issued = POOL ? 0 : gend - gq;
  auto fetch_group = [&]() {
    int g = 0;
    if (lane == 0) g = atomicAdd(P.ctr, 1);
    g = __shfl_sync(0xffffffffu, g, 0);
    if (g < P.ngroups) {
      nq = P.goff[g];
      nend = P.goff[g + 1];
    } else {
      nq = nend = -1;
    }
  };
  if (POOL) fetch_group();
  const int ntotal = POOL ? P.goff[P.ngroups] : gend;
  WChunk win{};
  int win_base = -64;
  auto load_window = [&](int base) {
    win_base = base;
    if (base + lane < ntotal) win = P.chunks[base + lane];
  };
  auto issue = [&](int s) {  // all lanes call (shuffles), lane 0 issues the next chunk
    if (POOL) {
      while (gq >= 0 && gq >= gend) {  // range used up: on to the prefetched pool group
        gq = nq;
        gend = nend;
        if (gq >= 0) fetch_group();
      }
      if (gq < 0) return;
      ++issued;
    } else if (gq >= gend) {
      return;
    }
    const int idx = gq++;
    if (idx < win_base || idx >= win_base + 32) load_window(idx);
    const int src_l = idx - win_base;
    const long long src = __shfl_sync(0xffffffffu, win.src, src_l);
    const long long aux = __shfl_sync(0xffffffffu, win.aux, src_l);
    const int len = __shfl_sync(0xffffffffu, win.len, src_l);
    const int kinds = __shfl_sync(0xffffffffu, win.src_kind | (win.aux_kind << 4), src_l);
    const int aux_len = __shfl_sync(0xffffffffu, win.aux_len, src_l);
    const int job = __shfl_sync(0xffffffffu, win.job, src_l);
    if (lane == 0) {
      double* st = ring + s * P.stage;
      const int src_kind = kinds & 15, aux_kind = kinds >> 4;
      const uint32_t bytes = (uint32_t)len * 8u;
      const uint32_t abytes = aux_kind == WA_NONE ? 0u : (uint32_t)aux_len * 32u;
      fence_proxy_async();
      mbar_expect_tx(&bar[s], 128u + bytes + abytes);
      bulk_g2s(st, &P.chunks[idx], 48u, &bar[s]);
      bulk_g2s(st + 6, &P.jobs[job], 80u, &bar[s]);
      if (bytes) bulk_g2s(st + kHdr, (src_kind == 0 ? P.arena : P.dense) + src, bytes, &bar[s]);
      if (abytes)
        bulk_g2s(st + kHdr + len, (aux_kind == WA_X ? P.xi : P.win) + aux * 4, abytes, &bar[s]);
    }
  };
#ifdef HMGPU_MV_PROF
  const long long ck0 = clock64();
#endif
  for (int s = 0; s < NS; ++s) issue(s);

  // rows lane, lane+32 x 3 outputs; VSPLIT: f_s of columns lane, lane+32
  double y[6] = {0, 0, 0, 0, 0, 0};
  for (int consumed = 0; consumed < issued; ++consumed) {
    const int s = consumed % NS;
    mbar_wait(&bar[s], (uint32_t)((consumed / NS) & 1));
    const double* st = ring + s * P.stage;
    const WChunk& ch = *reinterpret_cast<const WChunk*>(st);
    const WJob& job = *reinterpret_cast<const WJob*>(st + 6);
    const double* data = st + kHdr;
    const double* aux = data + ch.len;
    const int kind = job.kind;
    const bool first = ch.part == 0 && ch.g0 == 0 && kind != WJ_VSPLIT && !job.vrows
                           ? true
                           : (kind == WJ_USPLIT && ch.g0 == 0);
    if (first) {  // keep the job's x / W for its later chunks
      for (int e = lane; e < 4 * ch.aux_len; e += 32) scratch[e] = aux[e];
      __syncwarp();
    }
    bool last;
    if (kind == WJ_FUSED) {
      double* W = scratch + 256;
      if (ch.part == 0 && job.vrows) {
        // rows [g0, g1) of V over all K <= 64 columns (as VSPLIT); the f_s
        // of columns lane, lane + 32 add up in the lane's own W slots (y may
        // hold the rows of a job chain) until the last row chunk gives W
        const int ncol = job.ncols;
        double f[6] = {0, 0, 0, 0, 0, 0};
        if (ncol > 32) {
          vdots2<NC>(data, ncol, ch.g1 - ch.g0, aux, lane, lane + 32 < ncol, f);
        } else if (lane < ncol) {
          vdots<NC>(data, ncol, ch.g1 - ch.g0, aux, lane, f[0], f[1], f[2]);
        }
        const bool vlast = ch.g1 == job.n;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int l = lane + 32 * h;
          if (l < ncol) {
            double* o = W + 4 * l;
            double a0 = f[3 * h], a1 = f[3 * h + 1], a2 = f[3 * h + 2];
            if (ch.g0 != 0) {
              a0 = o[0] + a0;
              a1 = o[1] + a1;
              a2 = o[2] + a2;
            }
            if (vlast) {
              double w[4];
              weights<NC>(comp_of_col(job.kp, l), a0, a1, a2, w);
              *reinterpret_cast<double2*>(o) = make_double2(w[0], w[1]);
              *reinterpret_cast<double2*>(o + 2) = make_double2(w[2], w[3]);
            } else {
              o[0] = a0;
              o[1] = a1;
              o[2] = a2;
            }
          }
        }
        if (vlast) __syncwarp();
      } else if (ch.part == 0) {
        const int ncol = ch.g1 - ch.g0;
        if (ncol > 32 && ncol <= 64) {
          // one sweep: lane takes columns lane and lane + 32
          if (lane < ncol) {
            const bool two = lane + 32 < ncol;
            double f[6];
            vdots2<NC>(data, ncol, job.n, scratch, lane, two, f);
            double w[4];
            weights<NC>(comp_of_col(job.kp, ch.g0 + lane), f[0], f[1], f[2], w);
            *reinterpret_cast<double2*>(W + 4 * (ch.g0 + lane)) = make_double2(w[0], w[1]);
            *reinterpret_cast<double2*>(W + 4 * (ch.g0 + lane) + 2) = make_double2(w[2], w[3]);
            if (two) {
              const int g = lane + 32;
              weights<NC>(comp_of_col(job.kp, ch.g0 + g), f[3], f[4], f[5], w);
              *reinterpret_cast<double2*>(W + 4 * (ch.g0 + g)) = make_double2(w[0], w[1]);
              *reinterpret_cast<double2*>(W + 4 * (ch.g0 + g) + 2) = make_double2(w[2], w[3]);
            }
          }
        } else {
          for (int g = lane; g < ncol; g += 32) {
            double a = 0.0, b = 0.0, c = 0.0;
            vdots<NC>(data, ncol, job.n, scratch, g, a, b, c);
            double w[4];
            weights<NC>(comp_of_col(job.kp, ch.g0 + g), a, b, c, w);
            *reinterpret_cast<double2*>(W + 4 * (ch.g0 + g)) = make_double2(w[0], w[1]);
            *reinterpret_cast<double2*>(W + 4 * (ch.g0 + g) + 2) = make_double2(w[2], w[3]);
          }
        }
        __syncwarp();
      } else {
        urows<NC>(data, job.m, ch.g1 - ch.g0, W + 4 * ch.g0, lane, y);
      }
      last = ch.part == 1 && ch.g1 == job.ncols;
    } else if (kind == WJ_USPLIT) {
      urows<NC>(data, job.m, ch.g1 - ch.g0, scratch + 4 * ch.g0, lane, y);
      last = ch.g1 == job.ncols;
    } else if (kind == WJ_DENSE) {
      const int cp = (NC * job.m + 1) & ~1;
      drows<NC>(data, job.m, cp, ch.g1 - ch.g0, scratch + 4 * ch.g0, lane, y);
      last = ch.g1 == job.n;
    } else {  // WJ_VSPLIT: rows [g0, g1) of V for this job's columns
      const int ncol = job.ncols;
      if (ncol > 32) {
        double f[6];
        vdots2<NC>(data, ncol, ch.g1 - ch.g0, aux, lane, lane + 32 < ncol, f);
#pragma unroll
        for (int r = 0; r < 6; ++r) y[r] += f[r];
      } else if (lane < ncol) {
        vdots<NC>(data, ncol, ch.g1 - ch.g0, aux, lane, y[0], y[1], y[2]);
      }
      last = ch.g1 == job.n;
    }
    // job epilogue (descriptor fields read before the stage is recycled)
    if (last) {
      if (kind == WJ_VSPLIT) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int l = lane + 32 * h;
          if (l < job.ncols) {
            double w[4];
            weights<NC>(comp_of_col(job.kp, job.comp + l), y[3 * h], y[3 * h + 1],
                        y[3 * h + 2], w);
            double* o = P.wout + (job.out + l) * 4;
            *reinterpret_cast<double2*>(o) = make_double2(w[0], w[1]);
            *reinterpret_cast<double2*>(o + 2) = make_double2(w[2], w[3]);
          }
        }
#pragma unroll
        for (int r = 0; r < 6; ++r) y[r] = 0.0;
      } else if (!job.chain) {
        double* yo = P.ypart + job.out * NOUT;
        if (lane < job.m)
          for (int r = 0; r < NOUT; ++r) yo[lane * NOUT + r] = y[r];
        if (lane + 32 < job.m)
          for (int r = 0; r < NOUT; ++r) yo[(lane + 32) * NOUT + r] = y[3 + r];
#pragma unroll
        for (int r = 0; r < 6; ++r) y[r] = 0.0;
      }
    }
    __syncwarp();  // all lanes done with stage s
    issue(s);
  }
#ifdef HMGPU_MV_PROF
  if (P.prof && lane == 0 && gw < P.nwarps) P.prof[gw] = (unsigned long long)(clock64() - ck0);
#endif
}

// per leaf: y(p) = sum over covering job rows (fixed order).  The leaf's
// entries are staged in shared memory; its (row, r) pairs are padded to a
// power of two P2 and the CTA's LR_THREADS / P2 thread groups take the
// entries round-robin (group h: entries h, h + G, ...; 8 partial-row loads
// in flight per thread), then the group partials are added in group order
// (deterministic).  The critical path is the entry count of the fullest
// leaf divided by G.  Leaves wider than LR_THREADS pairs: one thread per pair.
#ifndef HMV_LR_THREADS
#define HMV_LR_THREADS 256
#endif
#ifndef HMV_LR_UNROLL
#define HMV_LR_UNROLL 8
#endif
constexpr int LR_THREADS = HMV_LR_THREADS;
template <int NOUT>
__global__ void __launch_bounds__(LR_THREADS)
hmv_leaf_reduce_kernel(const int* __restrict__ leaf_begin, const int* __restrict__ leaf_end,
                       const int* __restrict__ leaf_ptr,
                       const LeafEntry* __restrict__ entries, int nleaves,
                       const double* __restrict__ ypart, const int* __restrict__ rperm,
                       int nrows, double* __restrict__ y) {
  constexpr int EC = 512;  // entries staged per round
  constexpr int U = HMV_LR_UNROLL;
  __shared__ LeafEntry se[EC];
  __shared__ double red[LR_THREADS];
  for (int L = blockIdx.x; L < nleaves; L += gridDim.x) {
    const int b0 = leaf_begin[L], b1 = leaf_end[L];
    const int e0 = leaf_ptr[L], e1 = leaf_ptr[L + 1];
    const int cnt = (b1 - b0) * NOUT;
    if (cnt > LR_THREADS) {
      for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
        const int r = t % NOUT, i = t / NOUT;
        double s = 0.0;
        for (int e = e0; e < e1; ++e) {
          const LeafEntry en = entries[e];
          if (i >= en.lo && i < en.hi) s += ypart[(en.slot + (i - en.lo)) * NOUT + r];
        }
        y[(long long)r * nrows + rperm[b0 + i]] = s;
      }
      continue;
    }
    int P2 = 1;
    while (P2 < cnt) P2 <<= 1;
    const int G = LR_THREADS / P2;
    const int p = threadIdx.x & (P2 - 1), h = threadIdx.x / P2;
    const bool act = p < cnt;
    const int r = p % NOUT, i = p / NOUT;
    double s = 0.0;
    for (int c0 = e0; c0 < e1; c0 += EC) {
      const int ne = min(EC, e1 - c0);
      __syncthreads();
      for (int q = threadIdx.x; q < ne; q += blockDim.x) se[q] = entries[c0 + q];
      __syncthreads();
      int e = h;
      for (; e + (U - 1) * G < ne; e += U * G) {
        double v[U];
        bool in[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {  // unconditional loads (clamped index): U in flight
          const LeafEntry en = se[e + u * G];
          in[u] = act && i >= en.lo && i < en.hi;
          v[u] = __ldg(ypart + (in[u] ? (en.slot + (i - en.lo)) * NOUT + r : 0));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) s += in[u] ? v[u] : 0.0;
      }
      for (; e < ne; e += G) {
        const LeafEntry en = se[e];
        if (act && i >= en.lo && i < en.hi) s += ypart[(en.slot + (i - en.lo)) * NOUT + r];
      }
    }
    red[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x < cnt) {
      double acc = red[threadIdx.x];
      for (int g = 1; g < G; ++g) acc += red[g * P2 + threadIdx.x];
      y[(long long)r * nrows + rperm[b0 + i]] = acc;
    }
    __syncthreads();
  }
}

// gather x into the stream layout: 4 doubles per internal column
template <int NOUT>
__global__ void gather4_kernel(const double* __restrict__ x, double* __restrict__ xi,
                               const int* __restrict__ cperm, int ncols, int* ctr) {
  // the pool counters of the two stream passes that follow
  if (blockIdx.x == 0 && threadIdx.x < 2) ctr[threadIdx.x] = 0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < 4LL * ncols;
       t += (long long)gridDim.x * blockDim.x) {
    const int p = (int)(t >> 2), r = (int)(t & 3);
    xi[t] = r < NOUT ? x[(long long)r * ncols + cperm[p]] : 0.0;
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
      if (p.trans) {  // row-major destination
        const long long i = e / p.cols, l = e % p.cols;
        dst[p.dst + i * p.dld + l] = src[p.src + l * p.ld + i];
      } else {
        const long long l = e / p.rows, i = e % p.rows;
        dst[p.dst + l * p.dld + i] = src[p.src + l * p.ld + i];
      }
    }
  }
}

}  // namespace hmgpu
