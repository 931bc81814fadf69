// Multi-right-hand-side H-matvec Y += A X for the 3x3 Kelvin grid, 16
// right-hand sides per pass, on the fp64 tensor cores (DMMA,
// mma.sync.m8n8k4.f64).  At 16 RHS every stored factor value feeds 32 (16
// for the diagonal components) multiply-adds, so the sweep is no longer
// HBM-bound: these are the "batched fp64 factor products" of the north star.
//
//   phase 1 (hmv16_z_kernel)  per admissible block and 128-column chunk:
//            Z_c = V_c^T X_C and W_c = V_c^T X_R for the six components
//            (one warp each)
//   phase 1b (hmv16_zsum_kernel) chunks of wide blocks summed in order
//   phase 2 (hmv16_leaf_kernel) per leaf of the row tree, over the blocks
//            covering it in a fixed order: Y_R += U_c Z_c, Y_C += U_c W_c
//            and, for near-field blocks,
//            Y_R += D_c X_C, Y_C += D_c X_R; y written once per row
//            (deterministic, no atomics, no partial rows).
//
// Layouts: x gathered to xi16[(col * 3 + comp) * 16 + s] (internal column
// order, zero-padded past nrhs).
// Factors are read in place from the ACA arena (U: m x cap and V: n x cap,
// column-major), near-field blocks from the dense arena ([j][c][i]).
//
// Reference: HMatrix::matvec with a multi-column Vec (proj/src/hmatrix.cpp:
// 22-45) over the BlockGrid (proj/src/expr.cpp:197-215).
#pragma once

#include <cuda_runtime.h>

namespace hmgpu {

constexpr int MR = 16;   // right-hand sides per pass
constexpr int JC = 128;  // columns per phase-1 task
#ifndef HMV16_ZK
#define HMV16_ZK 4
#endif
constexpr int ZK = HMV16_ZK;  // phase-1 k-steps of fragments in flight

struct Z16Task {
  int blk, j0, jlen, zi;
  long long zbase;  // doubles: the block's Z region [nz][K][32]
};
struct Z16Sum {
  long long zbase;
  int len, nz;  // len = K * 32
};

// D = A B + D, A 8x4 (row), B 4x8 (col), fp64; lane (g = lane/4, t = lane%4)
// holds A[g][t], B[t][g] and D[g][2t], D[g][2t+1]
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// xi16[(p * 3 + r) * 16 + s] = x[(s0 + s) * ndof + r * ncols + cperm[p]]
__global__ void gather16_kernel(const double* __restrict__ x, double* __restrict__ xi,
                                const int* __restrict__ cperm, int ncols, int s0, int nr) {
  const long long ndof = 3LL * ncols;
  const long long total = ndof * MR;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(t & (MR - 1));
    const long long pr = t >> 4;
    const int r = (int)(pr % 3);
    const long long p = pr / 3;
    xi[t] = s < nr ? x[(long long)(s0 + s) * ndof + r * (long long)ncols + cperm[p]] : 0.0;
  }
}

// Rank table of the plan: rk[8 * bi + c] = rank of component c of matvec
// block bi in the plan's mode, rk[8 * bi + 6] = their sum.

// phase 1: one warp per (task, component) pair; no shared memory, no block
// barriers.  NMT = 8-row m-tiles of V^T held in registers: the pairs with
// rank <= 16 (almost all) run the NMT = 2 instance, which needs half the
// registers and so keeps twice as many warps (loads) in flight.  Pairs are
// ordered by task, so neighbouring warps share the chunk's x rows in L1.
template <int NMT>
__global__ void __launch_bounds__(256)
hmv16_z_kernel(const int2* __restrict__ pairs, int npairs, const Z16Task* __restrict__ tasks,
               const MvBlock* __restrict__ blocks, const Item* __restrict__ items,
               const int* __restrict__ rk, const double* __restrict__ arena,
               const double* __restrict__ xi, double* __restrict__ zpart) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  constexpr int Rs[6] = {0, 0, 0, 1, 1, 2}, Cs[6] = {0, 1, 2, 1, 2, 2};
  for (int w = gw; w < npairs; w += nw) {
    const int2 pc = pairs[w];
    const Z16Task tk = tasks[pc.x];
    const int c = pc.y;
    const int* r8 = rk + 8 * tk.blk;
    const int k = r8[c];
    int kpre = 0;
    for (int q = 0; q < c; ++q) kpre += r8[q];
    const int K = r8[6];
    const MvBlock b = blocks[tk.blk];
    const int R = Rs[c], C = Cs[c];
    const bool two = R != C;
    const double* V = arena + items[b.item0 + c].v_off + tk.j0;
    const double* xb = xi + (long long)(b.col0 + tk.j0) * 48 + g;
    double* zp = zpart + tk.zbase + (long long)tk.zi * K * 32;
    for (int lg = 0; lg < k; lg += 8 * NMT) {
      double acc[NMT][2][2][2];
#pragma unroll
      for (int a = 0; a < NMT; ++a)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int xr = 0; xr < 2; ++xr) acc[a][nt][xr][0] = acc[a][nt][xr][1] = 0.0;
      const int nmt = min(NMT, (k - lg + 7) >> 3);  // warp-uniform
      // ZK k-steps (4 ZK columns) of A and B fragments issued before the MMAs
      for (int j16 = 0; j16 < tk.jlen; j16 += 4 * ZK) {
        double a[ZK][NMT], bc[ZK][2], br[ZK][2];
#pragma unroll
        for (int st = 0; st < ZK; ++st) {
          const int j = j16 + 4 * st + t;
          const bool jok = j < tk.jlen;
#pragma unroll
          for (int mt = 0; mt < NMT; ++mt) {
            const int l = lg + mt * 8 + g;
            a[st][mt] = (mt < nmt && l < k && jok) ? V[(long long)l * b.n + j] : 0.0;
          }
          const double* xr = xb + (long long)j * 48;
          bc[st][0] = jok ? xr[C * 16] : 0.0;
          bc[st][1] = jok ? xr[C * 16 + 8] : 0.0;
          br[st][0] = (jok && two) ? xr[R * 16] : 0.0;
          br[st][1] = (jok && two) ? xr[R * 16 + 8] : 0.0;
        }
#pragma unroll
        for (int st = 0; st < ZK; ++st) {
          if (j16 + 4 * st >= tk.jlen) break;  // warp-uniform
#pragma unroll
          for (int mt = 0; mt < NMT; ++mt) {
            if (mt < nmt) {
              dmma(acc[mt][0][0][0], acc[mt][0][0][1], a[st][mt], bc[st][0]);
              dmma(acc[mt][1][0][0], acc[mt][1][0][1], a[st][mt], bc[st][1]);
              if (two) {
                dmma(acc[mt][0][1][0], acc[mt][0][1][1], a[st][mt], br[st][0]);
                dmma(acc[mt][1][1][0], acc[mt][1][1][1], a[st][mt], br[st][1]);
              }
            }
          }
        }
      }
#pragma unroll
      for (int mt = 0; mt < NMT; ++mt) {
        const int l = lg + mt * 8 + g;
        if (mt < nmt && l < k) {
          double* row = zp + (long long)(kpre + l) * 32 + 2 * t;
#pragma unroll
          for (int xr = 0; xr < 2; ++xr)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
              *reinterpret_cast<double2*>(row + xr * 16 + nt * 8) =
                  make_double2(acc[mt][nt][xr][0], acc[mt][nt][xr][1]);
        }
      }
    }
  }
}

// phase 1b: Z of blocks wider than one chunk = sum of its chunks, in order
__global__ void hmv16_zsum_kernel(const Z16Sum* __restrict__ sums, int nsums,
                                  double* __restrict__ zpart) {
  for (int si = blockIdx.x; si < nsums; si += gridDim.x) {
    const Z16Sum s = sums[si];
    double* z = zpart + s.zbase;
    for (int e = threadIdx.x; e < s.len; e += blockDim.x) {
      double v = z[e];
      for (int q = 1; q < s.nz; ++q) v += z[(long long)q * s.len + e];
      z[e] = v;
    }
  }
}

// phase 2, per group of TR 8-row tiles of a leaf of the row tree
// (tiles[w] = (leaf, group)): one warp visits the blocks covering the leaf in
// a fixed order (leaf_blk) and accumulates in registers, so y is written once
// per row: no partial rows, no reduction pass, no atomics, no block barriers.
// Each Z / x fragment loaded feeds TR row tiles.
#ifndef HMV16_TR
#define HMV16_TR 2
#endif
#ifndef HMV16_KS
#define HMV16_KS 4
#endif
constexpr int TR = HMV16_TR;  // row tiles per warp
constexpr int KS = HMV16_KS;  // k-steps of fragments in flight

__global__ void __launch_bounds__(256)
hmv16_leaf_kernel(const int2* __restrict__ tiles, int ntiles,
                  const int* __restrict__ leaf_begin, const int* __restrict__ leaf_end,
                  const int* __restrict__ leaf_ptr, const int2* __restrict__ leaf_blk,
                  const MvBlock* __restrict__ blocks, const Item* __restrict__ items,
                  const int* __restrict__ rk, const long long* __restrict__ zbase,
                  const double* __restrict__ arena, const double* __restrict__ dense,
                  const double* __restrict__ xi, const double* __restrict__ zpart,
                  const int* __restrict__ rperm, int nrows, double* __restrict__ y, int s0,
                  int nr) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  constexpr int Rs[6] = {0, 0, 0, 1, 1, 2}, Cs[6] = {0, 1, 2, 1, 2, 2};
  for (int w = gw; w < ntiles; w += nw) {
    const int2 lt = tiles[w];
    const int b0 = leaf_begin[lt.x];
    const int rows = leaf_end[lt.x] - b0;
    const int r0 = lt.y * 8 * TR;  // first row of the group within the leaf
    const int ntr = min(TR, (rows - r0 + 7) >> 3);  // warp-uniform
    bool iok[TR];
#pragma unroll
    for (int q = 0; q < TR; ++q) iok[q] = q < ntr && r0 + 8 * q + g < rows;
    double acc[TR][3][2][2];
#pragma unroll
    for (int q = 0; q < TR; ++q)
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) acc[q][r][nt][0] = acc[q][r][nt][1] = 0.0;
    const int e1 = leaf_ptr[lt.x + 1];
    for (int e = leaf_ptr[lt.x]; e < e1; ++e) {
      const int2 be = leaf_blk[e];
      const MvBlock b = blocks[be.x];
      const int i = be.y + r0 + g;  // row of tile 0 within the block
      if (!b.dense) {
        const int* r8 = rk + 8 * be.x;
        const double* z = zpart + zbase[be.x] + g;
        int kp = 0;
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          const int k = r8[c];
          const int R = Rs[c], C = Cs[c];
          const double* U = arena + items[b.item0 + c].u_off + i;
          const double* zc = z + (long long)kp * 32;
          kp += k;
          for (int l0 = 0; l0 < k; l0 += 4 * KS) {  // KS k-steps in flight
            double a[KS][TR], zz[KS][4];
#pragma unroll
            for (int st = 0; st < KS; ++st) {
              const int l = l0 + 4 * st + t;
              const bool lok = l < k;
#pragma unroll
              for (int q = 0; q < TR; ++q)
                a[st][q] = (lok && iok[q]) ? U[(long long)l * b.m + 8 * q] : 0.0;
              const double* zr = zc + (long long)l * 32;
              zz[st][0] = lok ? zr[0] : 0.0;
              zz[st][1] = lok ? zr[8] : 0.0;
              zz[st][2] = (lok && R != C) ? zr[16] : 0.0;
              zz[st][3] = (lok && R != C) ? zr[24] : 0.0;
            }
#pragma unroll
            for (int st = 0; st < KS; ++st) {
              if (l0 + 4 * st >= k) break;  // warp-uniform
#pragma unroll
              for (int q = 0; q < TR; ++q) {
                if (q >= ntr) break;
                dmma(acc[q][R][0][0], acc[q][R][0][1], a[st][q], zz[st][0]);
                dmma(acc[q][R][1][0], acc[q][R][1][1], a[st][q], zz[st][1]);
                if (R != C) {
                  dmma(acc[q][C][0][0], acc[q][C][0][1], a[st][q], zz[st][2]);
                  dmma(acc[q][C][1][0], acc[q][C][1][1], a[st][q], zz[st][3]);
                }
              }
            }
          }
        }
      } else {
        const long long cp = (6LL * b.m + 1) & ~1LL;
        const double* D = dense + b.dense_off + i;
        const double* xb = xi + (long long)b.col0 * 48 + g;
        for (int j0 = 0; j0 < b.n; j0 += 4) {
          const int j = j0 + t;
          const bool jok = j < b.n;
          double bx[3][2];
          const double* xr = xb + (long long)j * 48;
#pragma unroll
          for (int xc = 0; xc < 3; ++xc) {
            bx[xc][0] = jok ? xr[xc * 16] : 0.0;
            bx[xc][1] = jok ? xr[xc * 16 + 8] : 0.0;
          }
#pragma unroll
          for (int q = 0; q < TR; ++q) {
            if (q >= ntr) break;
            double a[6];
#pragma unroll
            for (int c = 0; c < 6; ++c)
              a[c] = (jok && iok[q]) ? D[(long long)j * cp + (long long)c * b.m + 8 * q] : 0.0;
#pragma unroll
            for (int c = 0; c < 6; ++c) {
              const int R = Rs[c], C = Cs[c];
              dmma(acc[q][R][0][0], acc[q][R][0][1], a[c], bx[C][0]);
              dmma(acc[q][R][1][0], acc[q][R][1][1], a[c], bx[C][1]);
              if (R != C) {
                dmma(acc[q][C][0][0], acc[q][C][0][1], a[c], bx[R][0]);
                dmma(acc[q][C][1][0], acc[q][C][1][1], a[c], bx[R][1]);
              }
            }
          }
        }
      }
    }
    const long long ndof = 3LL * nrows;
#pragma unroll
    for (int q = 0; q < TR; ++q) {
      if (!iok[q]) continue;
      const long long row = rperm[b0 + r0 + 8 * q + g];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int s = nt * 8 + 2 * t + hh;
            if (s < nr)
              y[(long long)(s0 + s) * ndof + r * (long long)nrows + row] = acc[q][r][nt][hh];
          }
    }
  }
}

// fp64 tensor-core peak probe: eight independent DMMA chains per warp
__global__ void __launch_bounds__(256) dmma_peak_kernel(double* out, int iters) {
  const int lane = threadIdx.x & 31;
  const double a = 1.0 + lane * 1e-9, b = 1e-9;
  double d[8][2];
#pragma unroll
  for (int q = 0; q < 8; ++q) d[q][0] = d[q][1] = q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) dmma(d[q][0], d[q][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += d[q][0] + d[q][1];
  if (s == 12345.678) out[0] = s;  // practically never; keeps the chains live
}

}  // namespace hmgpu
