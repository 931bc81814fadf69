// Device-resident error estimator and marking of the adaptive H-matvec
// (Algorithm 2 of the paper).  One sweep of
// amvm_multiply keeps everything on the device except a handful of scalars:
//
//   tail_kernel          t_b = U[:, k:K] (V[:, k:K]^T x_s) per (comp, block)
//                        with a look-ahead tail (apply_range, aca.cpp:7-11)
//   amvm_diff_kernel     difference(r) = sum of the terms at output row r, in
//                        term order (gamma_contributions, amvm.cpp:46-125)
//   amvm_entries_kernel  each term's entries in ascending output index and
//                        |term|^2 (the sorted sparse terms of amvm.cpp:105-122)
//   amvm_cand_kernel     per output row the terms with |value| >= tau, in
//                        term order (the marking CSR, amvm.cpp:131-160)
//   (CUB)                rows stably sorted by |difference| descending
//   amvm_walk_kernel     the greedy walk until ||residual|| <= (1-theta) gamma
//                        (amvm.cpp:160-184), gamma(P_k)
//
// Every floating-point reduction is restated in the oracle's order (term
// order per row; ascending output index inside a term; sequential sums over
// rows), so gamma, the marked set and gamma(P_k) are bit-identical to the
// CPU oracle (tests/test_gpu_parity.py, tests/test_gpu_fullsize.py).
//
// Terms are (component, block) pairs with K > k, in component-major, block-
// ascending order; an output row is (rb, p): block-row rb of the 3x3 grid and
// internal row p, external index rb * N + rperm[p].  The blocks covering p
// are the leaf entries of p's leaf (leaf_blk, ascending block order).
#pragma once

#include <cuda_runtime.h>

namespace hmgpu {

struct AmvmGeom {
  const int* row_leaf;     // internal row -> leaf
  const int* leaf_begin;
  const int* leaf_ptr;
  const int2* leaf_blk;    // (matvec block, row offset of the leaf in the block)
  const MvBlock* blocks;
  const int* rperm;
  const int* tix;          // item -> term index or -1
  const TailTerm* terms;
  const int* term_bi;      // term -> matvec block
  const int* sortp;        // per matvec block: local rows in ascending rperm order
  const long long* spoff;  // matvec block -> offset into sortp
  const double* out;       // tail values [off + o * m + i]
  int N;                   // rows of one component block (internal rows)
  int grid;                // 1: 3x3 Kelvin grid (6 components), 0: scalar
};

// occurrence of component c in block-row rb: 0 (rows R, x_C), 1 (rows C, x_R)
__device__ __forceinline__ int amvm_occ(int grid, int c, int rb) {
  if (!grid) return 0;
  const int R = c_comp_r[c], C = c_comp_c[c];
  if (R == rb) return 0;
  if (C == rb && R != C) return 1;
  return -1;
}

// visits the terms at output row (rb, p) in term order: f(term, value)
template <class F>
__device__ __forceinline__ void amvm_row_terms(const AmvmGeom& a, int rb, int p, F&& f) {
  const int L = a.row_leaf[p];
  const int e0 = a.leaf_ptr[L], e1 = a.leaf_ptr[L + 1];
  const int ncomp = a.grid ? 6 : 1;
  for (int c = 0; c < ncomp; ++c) {
    const int o = amvm_occ(a.grid, c, rb);
    if (o < 0) continue;
    for (int e = e0; e < e1; ++e) {
      const int2 be = a.leaf_blk[e];
      const MvBlock& b = a.blocks[be.x];
      if (b.dense) continue;
      const int t = a.tix[b.item0 + c];
      if (t < 0) continue;
      const int i = p - b.row0;
      const double v = a.out[a.terms[t].off + (long long)o * b.m + i];
      f(t, v);
    }
  }
}

// the estimator's terms on the device: every (comp, block) with a
// look-ahead tail, component-major, blocks ascending (amvm.cpp:135-150)
__global__ void amvm_term_flags_kernel(const MvBlock* __restrict__ mvb, int n_mv, int nc,
                                       const Item* __restrict__ items, int* __restrict__ flag,
                                       long long* __restrict__ size) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nc * n_mv) return;
  const int q = t / n_mv, bi = t - q * n_mv;
  const MvBlock mb = mvb[bi];
  int f = 0;
  long long sz = 0;
  if (!mb.dense) {
    const Item& it = items[mb.item0 + q];
    if (it.k > it.kcur) {
      f = 1;
      const int nocc = (nc == 6 && c_comp_r[q] != c_comp_c[q]) ? 2 : 1;
      sz = (long long)nocc * it.m;
    }
  }
  flag[t] = f;
  size[t] = sz;
}
__global__ void amvm_term_write_kernel(const MvBlock* __restrict__ mvb, int n_mv, int nc,
                                       const int* __restrict__ flag,
                                       const int* __restrict__ pos,
                                       const long long* __restrict__ off,
                                       TailTerm* __restrict__ terms, int* __restrict__ term_bi,
                                       int* __restrict__ tix) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nc * n_mv || !flag[t]) return;
  const int q = t / n_mv, bi = t - q * n_mv;
  const int item = mvb[bi].item0 + q;
  const int k = pos[t];
  terms[k] = TailTerm{item, (nc == 6 && c_comp_r[q] != c_comp_c[q]) ? 2 : 1, off[t]};
  term_bi[k] = bi;
  tix[item] = k;
}

__global__ void amvm_diff_kernel(AmvmGeom a, double* __restrict__ diff) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= a.N) return;
  const int nrb = a.grid ? 3 : 1;
  for (int rb = 0; rb < nrb; ++rb) {
    double s = 0.0;
    amvm_row_terms(a, rb, p, [&](int, double v) {
      if (a.grid && v == 0.0) return;  // the occurrence scatter skips zeros
      s += v;
    });
    diff[(long long)rb * a.N + a.rperm[p]] = s;
  }
}

// s = sum_i d_i^2 in index order (one thread adds; loads 16 ahead)
__device__ __forceinline__ double seq_sumsq(const double* __restrict__ d, long long n) {
  double s = 0.0;
  long long i = 0;
  for (; i + 16 <= n; i += 16) {
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = d[i + u];
#pragma unroll
    for (int u = 0; u < 16; ++u) s += v[u] * v[u];
  }
  for (; i < n; ++i) s += d[i] * d[i];
  return s;
}

// one thread: out[0] = sum_i d_i^2 (index order), out[1] = sqrt
__global__ void amvm_sumsq_kernel(const double* __restrict__ d, long long n,
                                  double* __restrict__ out) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const double s = seq_sumsq(d, n);
  out[0] = s;
  out[1] = sqrt(s);
}

// calls f(ext_index, value) over a term's entries in ascending output index
template <class F>
__device__ __forceinline__ void amvm_term_entries(const AmvmGeom& a, const Item* items,
                                                  int t, F&& f) {
  const TailTerm tt = a.terms[t];
  const MvBlock& b = a.blocks[a.term_bi[t]];
  const int comp = items[tt.item].comp;
  const int* sp = a.sortp + a.spoff[a.term_bi[t]];
  for (int o = 0; o < tt.nocc; ++o) {
    const int rb = a.grid ? (o == 0 ? c_comp_r[comp] : c_comp_c[comp]) : 0;
    const double* v = a.out + tt.off + (long long)o * b.m;
    for (int q = 0; q < b.m; ++q) {
      const int i = sp[q];
      const double x = v[i];
      if (a.grid && x == 0.0) continue;
      f((long long)rb * a.N + a.rperm[b.row0 + i], x);
    }
  }
}

// pass 0: nnz[t] = entries of term t (zeros skipped on the grid);
// pass 1: the entries (ascending output index) at eptr[t] and |term|^2
__global__ void amvm_entries_kernel(AmvmGeom a, const Item* __restrict__ items, int nterms,
                                    int pass, long long* __restrict__ nnz,
                                    const long long* __restrict__ eptr,
                                    long long* __restrict__ eidx, double* __restrict__ eval,
                                    double* __restrict__ nsq) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nterms) return;
  if (pass == 0) {
    long long n = 0;
    amvm_term_entries(a, items, t, [&](long long, double) { ++n; });
    nnz[t] = n;
    return;
  }
  long long e = eptr[t];
  double s = 0.0;
  amvm_term_entries(a, items, t, [&](long long i, double v) {
    eidx[e] = i;
    eval[e] = v;
    ++e;
    s += v * v;
  });
  nsq[t] = s;
}

// tau = (1 - theta) gamma / sqrt(c_sp M N) (amvm.cpp:138-140), from the device gamma
__device__ __forceinline__ double amvm_tau(const double* sc, double theta, double csp_mn) {
  return (1.0 - theta) * sc[1] / sqrt(csp_mn);
}

// pass 0: cnt[r] = number of terms with |value| >= tau at output row r;
// pass 1: their term indices in term order at lists[ptr[r] ...]
__global__ void amvm_cand_kernel(AmvmGeom a, const double* __restrict__ sc, double theta,
                                 double csp_mn, int pass, int* __restrict__ cnt,
                                 const int* __restrict__ ptr, int* __restrict__ lists) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= a.N) return;
  const double tau = amvm_tau(sc, theta, csp_mn);
  const int nrb = a.grid ? 3 : 1;
  for (int rb = 0; rb < nrb; ++rb) {
    const long long r = (long long)rb * a.N + a.rperm[p];
    int n = 0;
    int* dst = pass ? lists + ptr[r] : nullptr;
    amvm_row_terms(a, rb, p, [&](int t, double v) {
      if (a.grid && v == 0.0) return;
      if (fabs(v) >= tau) {
        if (pass) dst[n] = t;
        ++n;
      }
    });
    if (!pass) cnt[r] = n;
  }
}

// sort keys: |difference| bit patterns (monotonic for x >= 0)
__global__ void amvm_keys_kernel(const double* __restrict__ d, long long n,
                                 unsigned long long* __restrict__ keys, int* __restrict__ idx) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = (unsigned long long)__double_as_longlong(fabs(d[i]));
  idx[i] = (int)i;
}

// The greedy walk (amvm.cpp:160-184), one warp: rows in order, their
// candidate terms in order; each new term updates ||residual||^2 by
// |term|^2 - 2 (residual . term) -- the dot product summed sequentially in
// entry order like the reference's loop (products formed 32 at a time in
// parallel, then added in order by shuffles) -- and the residual itself.
// Software-pipelined: the next new term is found and its entries loaded
// while the current one is applied (only its residual gather must wait).

// the walk's term sequence: rows 32 at a time, each row's candidates 32 at
// a time, terms already in the set skipped (warp-uniform control flow)
struct WalkGen {
  const int* order;
  long long nrows;
  const int* ptr;
  const int* lists;
  const unsigned char* in_set;
  int lane;
  long long q0, rows_seen, cands;
  int rc0, rc1, nrow, j, c1, cb, t_l;
  unsigned todo;

  __device__ __forceinline__ void init() {
    q0 = -32;
    rows_seen = cands = 0;
    rc0 = rc1 = nrow = 0;
    j = -1;
    c1 = cb = 0;
    t_l = -1;
    todo = 0u;
  }
  __device__ __forceinline__ int next() {
    for (;;) {
      if (todo) {
        const int src = __ffs(todo) - 1;
        todo &= todo - 1;
        return __shfl_sync(0xffffffffu, t_l, src);
      }
      if (cb < c1) {  // next candidate chunk of the current row
        t_l = -1;
        if (cb + lane < c1) {
          t_l = lists[cb + lane];
          if (in_set[t_l]) t_l = -1;
        }
        todo = __ballot_sync(0xffffffffu, t_l >= 0);
        cb += 32;
        continue;
      }
      if (++j >= nrow) {  // next chunk of rows
        q0 += 32;
        if (q0 >= nrows) return -1;
        rc0 = rc1 = 0;
        if (q0 + lane < nrows) {
          const int r = order[q0 + lane];
          rc0 = ptr[r];
          rc1 = ptr[r + 1];
        }
        nrow = (int)min(32LL, nrows - q0);
        j = 0;
      }
      cb = __shfl_sync(0xffffffffu, rc0, j);
      c1 = __shfl_sync(0xffffffffu, rc1, j);
      ++rows_seen;
      cands += c1 - cb;
    }
  }
};

// a term's entries, held in registers when it has at most 64
struct WalkTerm {
  long long e0, i0, i1;
  int n;
  double nsq, v0, v1;
};

__device__ __forceinline__ WalkTerm walk_load(int t, int lane, const long long* eptr,
                                              const long long* eidx, const double* eval,
                                              const double* nsq) {
  WalkTerm w{};
  if (t < 0) return w;
  w.e0 = eptr[t];
  w.n = (int)(eptr[t + 1] - w.e0);
  w.nsq = nsq[t];
  if (w.n <= 64) {
    if (lane < w.n) {
      w.i0 = eidx[w.e0 + lane];
      w.v0 = eval[w.e0 + lane];
    }
    if (lane + 32 < w.n) {
      w.i1 = eidx[w.e0 + lane + 32];
      w.v1 = eval[w.e0 + lane + 32];
    }
  }
  return w;
}

constexpr int kWalkSmem = 4096;  // entries of a term staged in shared memory
__global__ void __launch_bounds__(32)
amvm_walk_kernel(const double* __restrict__ sc, double theta, const int* __restrict__ order,
                 long long nrows, const int* __restrict__ ptr, const int* __restrict__ lists,
                 const long long* __restrict__ eptr, const long long* __restrict__ eidx,
                 const double* __restrict__ eval, const double* __restrict__ nsq,
                 double* __restrict__ residual, unsigned char* __restrict__ in_set,
                 int* __restrict__ marked, int* __restrict__ n_marked,
                 double* __restrict__ out_pk) {
  extern __shared__ double wsm[];  // [4][kWalkSmem]: indices, values, residuals, products
  const int lane = threadIdx.x & 31;
  const double target = (1.0 - theta) * sc[1];
  const double target_sq = target * target;
  double res_sq = sc[0];
  int nm = 0;
  WalkGen G{order, nrows, ptr, lists, in_set, lane};
  G.init();
  int t = res_sq <= target_sq ? -1 : G.next();
  WalkTerm w = walk_load(t, lane, eptr, eidx, eval, nsq);
  while (t >= 0) {
    __syncwarp();
    if (lane == 0) {
      in_set[t] = 1;
      marked[nm] = t;
    }
    ++nm;
    __syncwarp();
    const int tn = G.next();  // look ahead (t is in the set already)
    const WalkTerm wn = walk_load(tn, lane, eptr, eidx, eval, nsq);
    double dot = 0.0;
    if (w.n <= 64) {
      const bool a0 = lane < w.n, a1 = lane + 32 < w.n;
      const double r0 = a0 ? residual[w.i0] : 0.0;
      const double r1 = a1 ? residual[w.i1] : 0.0;
      const double p0 = r0 * w.v0, p1 = r1 * w.v1;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const double s = __shfl_sync(0xffffffffu, p0, k);
        if (k < w.n) dot += s;
      }
      if (w.n > 32) {
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const double s = __shfl_sync(0xffffffffu, p1, k);
          if (32 + k < w.n) dot += s;
        }
      }
      res_sq += w.nsq - 2.0 * dot;
      if (a0) residual[w.i0] = r0 - w.v0;
      if (a1) residual[w.i1] = r1 - w.v1;
    } else if (w.n <= kWalkSmem) {
      // staged in shared memory: every load of the term in flight at once;
      // the products are formed in parallel and lane 0 adds them in order
      long long* si = reinterpret_cast<long long*>(wsm);
      double* sv = wsm + kWalkSmem;
      double* sr = wsm + 2 * kWalkSmem;
      double* sp = wsm + 3 * kWalkSmem;
#pragma unroll 4
      for (int e = lane; e < w.n; e += 32) {
        si[e] = eidx[w.e0 + e];
        sv[e] = eval[w.e0 + e];
      }
      __syncwarp();
#pragma unroll 4
      for (int e = lane; e < w.n; e += 32) {
        const double r = residual[si[e]];
        sr[e] = r;
        sp[e] = r * sv[e];
      }
      __syncwarp();
      if (lane == 0) {
        double d = 0.0;
        int e = 0;
        for (; e + 8 <= w.n; e += 8) {
          double p[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) p[u] = sp[e + u];
#pragma unroll
          for (int u = 0; u < 8; ++u) d += p[u];
        }
        for (; e < w.n; ++e) d += sp[e];
        dot = d;
      }
      dot = __shfl_sync(0xffffffffu, dot, 0);
      res_sq += w.nsq - 2.0 * dot;
#pragma unroll 4
      for (int e = lane; e < w.n; e += 32) residual[si[e]] = sr[e] - sv[e];
    } else {
      const long long e1 = w.e0 + w.n;
      for (long long b = w.e0; b < e1; b += 32) {
        const long long e = b + lane;
        double pr = 0.0;
        if (e < e1) pr = residual[eidx[e]] * eval[e];
        const int cnt = (int)min(32LL, e1 - b);
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const double s = __shfl_sync(0xffffffffu, pr, k);
          if (k < cnt) dot += s;
        }
      }
      res_sq += w.nsq - 2.0 * dot;
      __syncwarp();
      for (long long e = w.e0 + lane; e < e1; e += 32) residual[eidx[e]] -= eval[e];
    }
    __syncwarp();
    if (res_sq <= target_sq) break;
    t = tn;
    w = wn;
  }
  __syncwarp();
  if (lane == 0) {
    *n_marked = nm;
    out_pk[0] = sqrt(seq_sumsq(residual, nrows));
    out_pk[1] = (double)G.rows_seen;  // walk statistics (verbose runs)
    out_pk[2] = (double)G.cands;
  }
}

// ---------------------------------------------------------------------------
// The same greedy walk, parallel and bit-identical.  The walk's term
// sequence S (rows in order, their candidates in order, each term at its
// first appearance) does not depend on the residual; only the stopping
// point does.  So: (1) S from the first-appearance position of every term
// (atomicMin over the concatenated candidate lists, then a radix sort);
// (2) per chunk of S, every entry's residual value BEFORE its term is
// applied -- per output row the entries of the chunk's terms in S order,
// subtracted sequentially from the carried residual (one thread per row
// run of the (row, rank)-sorted entries: the reference's per-row order of
// subtractions); (3) each term's dot = sum over its entries, in entry
// order, of residual_before * value (the reference's loop, one thread per
// term); (4) one thread scans res_sq += |term|^2 - 2 dot in S order and
// stops at the first res_sq <= target; (5) the residual of every row takes
// its value after the last applied entry.  Same operations, same order,
// per row and per term as the sequential walk.
__global__ void walk_cnt_kernel(const int* __restrict__ order, long long M,
                                const int* __restrict__ ptr, long long* __restrict__ cnt) {
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q > M) return;
  cnt[q] = q < M ? ptr[order[q] + 1] - ptr[order[q]] : 0;
}
__global__ void walk_first_kernel(const int* __restrict__ order, long long M,
                                  const int* __restrict__ ptr, const int* __restrict__ lists,
                                  const long long* __restrict__ pre,
                                  unsigned long long* __restrict__ first) {
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q >= M) return;
  const int r = order[q];
  const int s0 = ptr[r], s1 = ptr[r + 1];
  for (int s = s0; s < s1; ++s)
    atomicMin(first + lists[s], (unsigned long long)(pre[q] + (s - s0)));
}
__global__ void walk_tids_kernel(int nt, int* __restrict__ tid, unsigned long long* __restrict__ first,
                                 int* __restrict__ count) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  tid[t] = t;
  if (first[t] != ~0ull) atomicAdd(count, 1);
}
// entries of S's terms: sizes in S order (for the chunk offsets)
__global__ void walk_sizes_kernel(const int* __restrict__ tS, int L,
                                  const long long* __restrict__ eptr, long long* __restrict__ sz) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > L) return;
  sz[k] = k < L ? eptr[tS[k] + 1] - eptr[tS[k]] : 0;
}
// chunk [k0, k1): one key (row << 22 | rank) per entry, the entry's global
// position by chunk slot
__global__ void walk_build_kernel(const int* __restrict__ tS, int k0, int k1,
                                  const long long* __restrict__ cumE,
                                  const long long* __restrict__ eptr,
                                  const long long* __restrict__ eidx,
                                  unsigned long long* __restrict__ keys, int* __restrict__ slots,
                                  long long* __restrict__ gslot) {
  const int k = k0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= k1) return;
  const int t = tS[k];
  const long long base = cumE[k] - cumE[k0], e0 = eptr[t], n = eptr[t + 1] - e0;
  for (long long e = 0; e < n; ++e) {
    const long long sl = base + e;
    keys[sl] = ((unsigned long long)eidx[e0 + e] << 22) | (unsigned long long)(k - k0);
    slots[sl] = (int)sl;
    gslot[sl] = e0 + e;
  }
}
// (2): per row run of the sorted entries, the residual before each entry
__global__ void walk_before_kernel(const unsigned long long* __restrict__ skeys,
                                   const int* __restrict__ sslots, long long E,
                                   const long long* __restrict__ gslot,
                                   const double* __restrict__ eval,
                                   const double* __restrict__ resid, double* __restrict__ rb) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= E) return;
  const unsigned long long row = skeys[i] >> 22;
  if (i > 0 && (skeys[i - 1] >> 22) == row) return;
  double r = resid[row];
  for (long long j = i; j < E && (skeys[j] >> 22) == row; ++j) {
    const int sl = sslots[j];
    rb[sl] = r;
    r = r - eval[gslot[sl]];
  }
}
// (3): dot of every chunk term, entry order
__global__ void walk_dot_kernel(int k0, int k1, const long long* __restrict__ cumE,
                                const long long* __restrict__ gslot,
                                const double* __restrict__ eval, const double* __restrict__ rb,
                                double* __restrict__ dots) {
  const int k = k0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= k1) return;
  const long long b0 = cumE[k] - cumE[k0], b1 = cumE[k + 1] - cumE[k0];
  double d = 0.0;
  for (long long sl = b0; sl < b1; ++sl) d += rb[sl] * eval[gslot[sl]];
  dots[k - k0] = d;
}
// (4): the sequential res_sq scan; st[0] = res_sq (in/out), st[1] = stop
// rank within the chunk or -1
// the chunk's |term|^2 - 2 dot in S order, contiguous (parallel)
__global__ void walk_incr_kernel(const int* __restrict__ tS, int k0, int k1,
                                 const double* __restrict__ nsq, double* __restrict__ dots) {
  const int k = k0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= k1) return;
  dots[k - k0] = nsq[tS[k]] - 2.0 * dots[k - k0];
}
__global__ void walk_scan_kernel(const double* __restrict__ incr, int n, double target_sq,
                                 double* __restrict__ st) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double res = st[0];
  int stop = -1;
  int k = 0;
  // the increments are loaded 16 at a time ahead of the dependent adds
  for (; k + 16 <= n && stop < 0; k += 16) {
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = incr[k + u];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (stop < 0) {
        res += v[u];
        if (res <= target_sq) stop = k + u;
      }
    }
  }
  for (; k < n && stop < 0; ++k) {
    res += incr[k];
    if (res <= target_sq) stop = k;
  }
  st[0] = res;
  st[1] = (double)stop;
}
// (5): rows take their value after the last applied entry (rank <= lim)
__global__ void walk_apply_kernel(const unsigned long long* __restrict__ skeys,
                                  const int* __restrict__ sslots, long long E,
                                  const long long* __restrict__ gslot,
                                  const double* __restrict__ eval, const double* __restrict__ rb,
                                  const double* __restrict__ st, int nchunk,
                                  double* __restrict__ resid) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= E) return;
  const unsigned long long row = skeys[i] >> 22;
  if (i > 0 && (skeys[i - 1] >> 22) == row) return;
  const int stop = (int)st[1];
  const unsigned long long lim = stop >= 0 ? (unsigned long long)stop : (unsigned long long)(nchunk - 1);
  long long last = -1;
  for (long long j = i; j < E && (skeys[j] >> 22) == row; ++j)
    if ((skeys[j] & ((1ull << 22) - 1)) <= lim) last = j;
  if (last >= 0) {
    const int sl = sslots[last];
    resid[row] = rb[sl] - eval[gslot[sl]];
  }
}

// marked term -> work item
__global__ void amvm_items_kernel(const TailTerm* __restrict__ terms,
                                  const int* __restrict__ marked, const int* __restrict__ n,
                                  int* __restrict__ ids) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < *n) ids[q] = terms[marked[q]].item;
}

}  // namespace hmgpu
