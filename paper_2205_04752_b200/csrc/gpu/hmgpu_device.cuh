// Device side of the B200 H-matrix hot path: fused Kelvin / Newton / dense
// entry providers, batched ACA (warp or CTA per item), near-field fill, H-matvec
// sweep and look-ahead tail products.  fp64 throughout (sm_100a).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#ifndef HMGPU_RUNROLL
#define HMGPU_RUNROLL 2
#endif
#define HM_PRAGMA(x) _Pragma(#x)
#define HM_UNROLL(n) HM_PRAGMA(unroll n)

namespace hmgpu {

// ---------------------------------------------------------------------------
// quadrature tiers in constant memory: tier 0 far (order 2, 3 points),
// 1 mid (order 4, 6 points), 2 near (order 5, 7 points)
// (point_order, proj/src/kernels.cpp:87-93; gauss_rule, quadrature.cpp:55-95)
struct RuleTable {
  int n[3];
  int pad;
  double a[3][12], b[3][12], w[3][12];
  double far_ratio, mid_ratio;
};
__constant__ RuleTable c_rules;

// component (r,c) of the symmetric 3x3 grid, row-major upper triangle
__constant__ int c_comp_r[6] = {0, 0, 0, 1, 1, 2};
__constant__ int c_comp_c[6] = {0, 1, 2, 1, 2, 2};

enum { KIND_KELVIN = 0, KIND_NEWTON = 1, KIND_DENSE = 2, KIND_GALERKIN = 3, KIND_KDELTA = 4,
       KIND_KDOUBLE = 5 };

// Per-problem geometry, passed by value to every kernel.
struct Geom {
  int kind;
  int same_tree;            // row internal index == col internal index <=> same DOF
  const double4* rowpt;     // evaluation points, internal row order (x,y,z,-)
  const double* tri;        // kelvin: 14 fields per column triangle, internal order,
                            //   tiles of 32 (TriRef): v0[3] e1[3] e2[3] cen[3] area diam
  const double4* colpt;     // newton: column points, internal column order
  const double* A;          // dense: column-major matrix, external ids
  long long lda;
  const int* rperm;         // internal -> external (rows)
  const int* cperm;         // internal -> external (cols)
  double cst;               // (1+nu) / (8 pi E (1-nu))      (kernels.cpp:24)
  double c34;               // 3 - 4 nu
  double diag;              // newton diagonal value
  // galerkin (V_Delta / V_kl, kernels.cpp:95-149)
  const double4* vtx;       // mesh vertices, global ids
  const int4* tvid;         // per internal triangle: global vertex ids, w = external id
  const double* prule;      // singular pair rules, SoA [5][total] (xr1 xr2 yr1 yr2 w)
  long long prule_total;
  int pr_off[4], pr_n[4];   // per PairCase (1 vertex, 2 edge, 3 identical)
  int gal_delta;            // 1: the context holds V_Delta (one component)
  // K_Delta (triangles x nodes, kernels.cpp:151-167): per external triangle
  const int4* tvx;          // vertex ids, w = external id
  const double4* tce;       // centroid, diameter
  const double4* tna;       // unit normal, area
  const int* vt_ptr;        // per internal column (node): its triangles in vt_tri
  const int2* vt_tri;       // (triangle, local index of the node), ascending triangles
  // double layer (colloc_double, kernels.cpp:189-210): cell (dl_r, dl_c)
  int dl_r, dl_c;
  double dl_b1, dl_a2, dl_a6;  // 2mu - 2lambda(1-2nu), mu(1-(3-4nu)), 6mu
};

// ---------------------------------------------------------------------------
// one column triangle's fields (structure-of-arrays view)
// tiles of 32 triangles x 16 field slots: field f of triangle j at
// tri[(j / 32) * 512 + f * 32 + j % 32] -- consecutive j coalesce, and every
// field is a constant offset from one base pointer
struct TriRef {
  const double* p;
  __device__ __forceinline__ double operator[](int f) const { return p[f * 32]; }
};
__device__ __forceinline__ TriRef tri_ref(const Geom& g, int j) {
  return TriRef{g.tri + ((long long)(j >> 5) << 9) + (j & 31)};
}

// Kelvin collocation: quadrature tier decided with IEEE round-to-nearest
// operations in the reference's order so that it is bit-identical to the
// host/oracle decision: gap = |p - c_j| - 0.5 d_j (kernels.cpp:88-92).
__device__ __forceinline__ int kelvin_tier_exact(double d2, double dj) {
  const double gap = __dsub_rn(__dsqrt_rn(d2), __dmul_rn(0.5, dj));
  if (gap >= __dmul_rn(c_rules.far_ratio, dj)) return 0;
  if (gap >= __dmul_rn(c_rules.mid_ratio, dj)) return 1;
  return 2;
}
// The decision compares squared distances against the thresholds first and
// takes the exact IEEE path only inside a 1e-12 relative band around them,
// where the rounding of sqrt / subtract could matter; outside the band both
// give the same tier.
__device__ __forceinline__ int kelvin_tier(double px, double py, double pz,
                                           const TriRef& T) {
  const double dx = __dsub_rn(px, T[9]);
  const double dy = __dsub_rn(py, T[10]);
  const double dz = __dsub_rn(pz, T[11]);
  const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                              __dmul_rn(dz, dz));
  const double dj = T[13];
  const double t0 = (c_rules.far_ratio + 0.5) * dj, t1 = (c_rules.mid_ratio + 0.5) * dj;
  const double s0 = t0 * t0, s1 = t1 * t1;
  if (d2 > s0 * (1.0 + 1e-12)) return 0;
  if (d2 < s0 * (1.0 - 1e-12)) {
    if (d2 > s1 * (1.0 + 1e-12)) return 1;
    if (d2 < s1 * (1.0 - 1e-12)) return 2;
  }
  return kelvin_tier_exact(d2, dj);
}

// 1/sqrt(x) for x > 0: bit-level seed and four Newton steps written with
// explicit IEEE operations, y <- y (1.5 - (x/2) y y).  Deterministic, ~1 ulp,
// and restated operation for operation by the oracle (oracle/hmbem_oracle.cpp
// rsqrt_canon), so entries stay bit-identical; about 4x cheaper than the
// IEEE division of an IEEE square root.
// HMGPU_FAST_ENTRY (measurement builds only, scripts/aca_fast_ab.py): the
// CUDA math library's rsqrt instead (hardware seed + Newton), to price the
// bit-exact contract; its results are not bit-identical to the oracle.
__device__ __forceinline__ double rsqrt_canon(double x) {
#ifdef HMGPU_FAST_ENTRY
  return rsqrt(x);
#endif
  const long long i = 0x5fe6eb50c7b537a9LL - (__double_as_longlong(x) >> 1);
  double y = __longlong_as_double(i);
  const double h = 0.5 * x;
#pragma unroll
  for (int it = 0; it < 4; ++it) y = y * fma(-(h * y), y, 1.5);
  return y;
}

__device__ __forceinline__ double sel3(int r, double x, double y, double z) {
  return r == 0 ? x : (r == 1 ? y : z);
}

// Exact integral of the Kelvin tensor over the flat triangle for a point p
// in its plane (builder-defined self term, closed form; see
// oracle/hmbem_oracle.cpp Kelvin::self_term for the derivation).
__device__ __noinline__ void kelvin_self6(const Geom& g, double px, double py, double pz,
                             const TriRef T, double* out6) {
  const double v[3][3] = {{T[0], T[1], T[2]},
                          {T[0] + T[3], T[1] + T[4], T[2] + T[5]},
                          {T[0] + T[6], T[1] + T[7], T[2] + T[8]}};
  double nx = T[4] * T[8] - T[5] * T[7];
  double ny = T[5] * T[6] - T[3] * T[8];
  double nz = T[3] * T[7] - T[4] * T[6];
  const double nn = sqrt(nx * nx + ny * ny + nz * nz);
  nx /= nn;
  ny /= nn;
  nz /= nn;
  double i1 = 0.0;
  double irc[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll 1
  for (int e = 0; e < 3; ++e) {
    const double* a = v[e];
    const double* b = v[(e + 1) % 3];
    double tx = b[0] - a[0], ty = b[1] - a[1], tz = b[2] - a[2];
    const double len = sqrt(tx * tx + ty * ty + tz * tz);
    tx /= len;
    ty /= len;
    tz /= len;
    const double mx = ty * nz - tz * ny, my = tz * nx - tx * nz,
                 mz = tx * ny - ty * nx;
    const double pax = a[0] - px, pay = a[1] - py, paz = a[2] - pz;
    const double pbx = b[0] - px, pby = b[1] - py, pbz = b[2] - pz;
    const double h = pax * mx + pay * my + paz * mz;
    const double s1 = pax * tx + pay * ty + paz * tz;
    const double s2 = pbx * tx + pby * ty + pbz * tz;
    const double r1 = sqrt(pax * pax + pay * pay + paz * paz);
    const double r2 = sqrt(pbx * pbx + pby * pby + pbz * pbz);
    const double lg = log((r2 + s2) / (r1 + s1));
    const double dsin = s2 / r2 - s1 / r1;
    const double dcos = h / r1 - h / r2;
    i1 += h * lg;
    const double m[3] = {mx, my, mz}, t[3] = {tx, ty, tz};
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const int r = c_comp_r[k], c = c_comp_c[k];
      irc[k] += h * (m[r] * m[c] * dsin + (m[r] * t[c] + t[r] * m[c]) * dcos +
                     t[r] * t[c] * (lg - dsin));
    }
  }
#pragma unroll
  for (int k = 0; k < 6; ++k)
    out6[k] = g.cst * ((c_comp_r[k] == c_comp_c[k] ? g.c34 * i1 : 0.0) + irc[k]);
}

// A_rc[i, j] = 2 area_j sum_q w_q S(p_i - y_q)_rc for one component
// (colloc_single, kernels.cpp:176-187), S from kelvin_tensor (:21-28).
// Canonical evaluation order (the parity contract with the CPU oracle,
// oracle/hmbem_oracle.cpp Kelvin::colloc_single): c factored out of the
// sum, 1/|x| by rsqrt_canon (deterministic Newton), explicit fma
// (the library is compiled with --fmad=false so nothing else contracts).
// With it ACA pivots, ranks and factors are bit-identical to the oracle.
// SELF = false: the caller guarantees i != j (admissible blocks: the row and
// column clusters are disjoint), so the self-term path is not compiled in.
// quadrature sum of one component (R, C) fixed at compile time (no selects)
template <int R, int C>
__device__ __forceinline__ double kelvin_quad(const Geom& g, const double4& p,
                                              const TriRef& T, int tier) {
  const double v0x = T[0], v0y = T[1], v0z = T[2];
  const double e1x = T[3], e1y = T[4], e1z = T[5];
  const double e2x = T[6], e2y = T[7], e2z = T[8];
  double acc_d = 0.0, acc_x = 0.0;
  const int nq = c_rules.n[tier];
#pragma unroll 1
  for (int q = 0; q < nq; ++q) {
    const double a = c_rules.a[tier][q], b = c_rules.b[tier][q],
                 w = c_rules.w[tier][q];
    const double dx = p.x - fma(b, e2x, fma(a, e1x, v0x));
    const double dy = p.y - fma(b, e2y, fma(a, e1y, v0y));
    const double dz = p.z - fma(b, e2z, fma(a, e1z, v0z));
    const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
    const double ri = rsqrt_canon(r2);
    const double wr = w * ri;
    if (R == C) acc_d = acc_d + wr;
    const double dr = R == 0 ? dx : (R == 1 ? dy : dz);
    const double dc = C == 0 ? dx : (C == 1 ? dy : dz);
    acc_x = fma(wr * ri * ri, dr * dc, acc_x);
  }
  const double s = (R == C) ? fma(g.c34, acc_d, acc_x) : acc_x;
  return 2.0 * T[12] * g.cst * s;
}

template <bool SELF = true>
__device__ __forceinline__ double kelvin_entry1(const Geom& g, int i, int j,
                                                int comp, int& nq_acc) {
  const double4 p = g.rowpt[i];
  const TriRef T = tri_ref(g, j);
  if (SELF && g.same_tree && i == j) {
    double s6[6];
    kelvin_self6(g, p.x, p.y, p.z, T, s6);
    return s6[comp];
  }
  const int tier = kelvin_tier(p.x, p.y, p.z, T);
  nq_acc += c_rules.n[tier];
  switch (comp) {  // warp-uniform
    case 0: return kelvin_quad<0, 0>(g, p, T, tier);
    case 1: return kelvin_quad<0, 1>(g, p, T, tier);
    case 2: return kelvin_quad<0, 2>(g, p, T, tier);
    case 3: return kelvin_quad<1, 1>(g, p, T, tier);
    case 4: return kelvin_quad<1, 2>(g, p, T, tier);
    default: return kelvin_quad<2, 2>(g, p, T, tier);
  }
}

// all six components of one (point, triangle) pair (near-field fill), each
// in the same canonical order as kelvin_entry1
__device__ __forceinline__ void kelvin_entry6(const Geom& g, int i, int j,
                                              double* out6, int& nq_acc) {
  const double4 p = g.rowpt[i];
  const TriRef T = tri_ref(g, j);
  if (g.same_tree && i == j) {
    kelvin_self6(g, p.x, p.y, p.z, T, out6);
    return;
  }
  const int tier = kelvin_tier(p.x, p.y, p.z, T);
  const double v0x = T[0], v0y = T[1], v0z = T[2];
  const double e1x = T[3], e1y = T[4], e1z = T[5];
  const double e2x = T[6], e2y = T[7], e2z = T[8];
  double ad = 0.0, a00 = 0.0, a01 = 0.0, a02 = 0.0, a11 = 0.0, a12 = 0.0,
         a22 = 0.0;
  const int nq = c_rules.n[tier];
  nq_acc += nq;
  for (int q = 0; q < nq; ++q) {
    const double a = c_rules.a[tier][q], b = c_rules.b[tier][q],
                 w = c_rules.w[tier][q];
    const double dx = p.x - fma(b, e2x, fma(a, e1x, v0x));
    const double dy = p.y - fma(b, e2y, fma(a, e1y, v0y));
    const double dz = p.z - fma(b, e2z, fma(a, e1z, v0z));
    const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
    const double ri = rsqrt_canon(r2);
    const double wr = w * ri;
    const double w3 = wr * ri * ri;
    ad = ad + wr;
    a00 = fma(w3, dx * dx, a00);
    a01 = fma(w3, dx * dy, a01);
    a02 = fma(w3, dx * dz, a02);
    a11 = fma(w3, dy * dy, a11);
    a12 = fma(w3, dy * dz, a12);
    a22 = fma(w3, dz * dz, a22);
  }
  const double f = 2.0 * T[12] * g.cst;
  out6[0] = f * fma(g.c34, ad, a00);
  out6[1] = f * a01;
  out6[2] = f * a02;
  out6[3] = f * fma(g.c34, ad, a11);
  out6[4] = f * a12;
  out6[5] = f * fma(g.c34, ad, a22);
}

// ---------------------------------------------------------------------------
// Galerkin scalar kernels: V_Delta = (1/4pi) int int
// 1/|x-y| and V_kl = (1/4pi) int int (x_k-y_k)(x_l-y_l)/|x-y|^3 over pairs of
// triangles (integrate_pair, proj/src/kernels.cpp:95-149) with the pair
// rules of quadrature.cpp:127-338: disjoint pairs a tensor product of two
// triangle rules (order 2 / 4 / 5 by distance, disjoint_order kernels.cpp:
// 75-85; the tiers of c_rules), touching pairs the Sauter-Schwab tables.
// Canonical order shared bit for bit with oracle/hmbem_oracle.cpp Galerkin
// (points by explicit fma from the rotated corners, rsqrt_canon, 4 area_i
// area_j / (4 pi) factored out).  Components: 0..5 V_kl (c_comp_r/c_comp_c),
// 6 V_Delta.

__device__ __forceinline__ double warp_sum(double v);

// classify_pair (quadrature.cpp:127-156) on global vertex ids; returns the
// case and the rotations
__device__ __forceinline__ int gal_classify(const int4& a, const int4& b, int& ra, int& rb) {
  const int A[3] = {a.x, a.y, a.z}, B[3] = {b.x, b.y, b.z};
  ra = rb = 0;
  if (A[0] == B[0] && A[1] == B[1] && A[2] == B[2]) return 3;
#pragma unroll
  for (int rt = 0; rt < 3; ++rt)
#pragma unroll
    for (int rs = 0; rs < 3; ++rs)
      if (B[rs] == A[(rt + 1) % 3] && B[(rs + 1) % 3] == A[rt]) {
        ra = rt;
        rb = rs;
        return 2;
      }
#pragma unroll
  for (int rt = 0; rt < 3; ++rt)
#pragma unroll
    for (int rs = 0; rs < 3; ++rs)
      if (A[rt] == B[rs]) {
        ra = rt;
        rb = rs;
        return 1;
      }
  return 0;
}

// disjoint_order (kernels.cpp:75-85) as a tier of c_rules: 0 (order 2) if
// gap >= 4 dmax, 1 (order 4) if gap >= 0.75 dmax (the mid and near tiers
// share order 4), else 2 (order 5); IEEE operations in the oracle's order
__device__ __forceinline__ int gal_tier(double cix, double ciy, double ciz, double di,
                                        double cjx, double cjy, double cjz, double dj) {
  const double dmax = fmax(di, dj);
  const double dx = __dsub_rn(cix, cjx), dy = __dsub_rn(ciy, cjy), dz = __dsub_rn(ciz, cjz);
  const double nrm = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                          __dmul_rn(dz, dz)));
  const double gap = __dsub_rn(nrm, __dmul_rn(0.5, __dadd_rn(di, dj)));
  if (gap >= __dmul_rn(4.0, dmax)) return 0;
  if (gap >= __dmul_rn(0.75, dmax)) return 1;
  return 2;
}

struct GalPair {
  double x0[3], ex1[3], ex2[3], y0[3], ey1[3], ey2[3];
  double scale;  // 4 area_i area_j (1 / (4 pi))
  int pc, tier;
};

// the canonical pair setup: orientation by external triangle id
// (kernels.cpp:132-133, 141), classification, rotated corners.  TOUCH =
// false: the caller guarantees a disjoint pair (admissible blocks).
template <bool TOUCH>
__device__ __forceinline__ GalPair gal_setup(const Geom& g, int i, int j) {
  int4 a = g.tvid[i], b = g.tvid[j];
  int ii = i, jj = j;
  if (a.w > b.w) {
    const int4 t = a;
    a = b;
    b = t;
    ii = j;
    jj = i;
  }
  GalPair P;
  int ra = 0, rb = 0;
  P.pc = TOUCH ? gal_classify(a, b, ra, rb) : 0;
  const TriRef Ti = tri_ref(g, ii), Tj = tri_ref(g, jj);
  P.tier = P.pc == 0 ? gal_tier(Ti[9], Ti[10], Ti[11], Ti[13], Tj[9], Tj[10], Tj[11], Tj[13])
                     : 0;
  const int A[3] = {a.x, a.y, a.z}, B[3] = {b.x, b.y, b.z};
  // test_vertex_perm(ra) / trial_vertex_perm(pc, rb) (quadrature.cpp:158-166)
  const int xp0 = ra, xp1 = (ra + 1) % 3, xp2 = (ra + 2) % 3;
  int yp0 = rb, yp1 = (rb + 1) % 3;
  const int yp2 = (rb + 2) % 3;
  if (P.pc == 2) {
    const int t = yp0;
    yp0 = yp1;
    yp1 = t;
  }
  const double4 X0 = g.vtx[A[xp0]], X1 = g.vtx[A[xp1]], X2 = g.vtx[A[xp2]];
  const double4 Y0 = g.vtx[B[yp0]], Y1 = g.vtx[B[yp1]], Y2 = g.vtx[B[yp2]];
  P.x0[0] = X0.x; P.x0[1] = X0.y; P.x0[2] = X0.z;
  P.y0[0] = Y0.x; P.y0[1] = Y0.y; P.y0[2] = Y0.z;
  P.ex1[0] = X1.x - X0.x; P.ex1[1] = X1.y - X0.y; P.ex1[2] = X1.z - X0.z;
  P.ex2[0] = X2.x - X0.x; P.ex2[1] = X2.y - X0.y; P.ex2[2] = X2.z - X0.z;
  P.ey1[0] = Y1.x - Y0.x; P.ey1[1] = Y1.y - Y0.y; P.ey1[2] = Y1.z - Y0.z;
  P.ey2[0] = Y2.x - Y0.x; P.ey2[1] = Y2.y - Y0.y; P.ey2[2] = Y2.z - Y0.z;
  P.scale = 4.0 * Ti[12] * Tj[12] * (1.0 / (4.0 * M_PI));
  return P;
}

// one quadrature point of component COMP (0..5 V_kl, 6 V_Delta, -1 all)
template <int COMP>
__device__ __forceinline__ void gal_point(const GalPair& P, double a1, double a2, double b1,
                                          double b2, double w, double& ad, double* akl) {
  double d[3];
#pragma unroll
  for (int c = 0; c < 3; ++c)
    d[c] = fma(a2, P.ex2[c], fma(a1, P.ex1[c], P.x0[c])) -
           fma(b2, P.ey2[c], fma(b1, P.ey1[c], P.y0[c]));
  const double ri = rsqrt_canon(fma(d[2], d[2], fma(d[1], d[1], d[0] * d[0])));
  const double wr = w * ri;
  if (COMP == 6 || COMP < 0) ad = ad + wr;
  if (COMP != 6) {
    const double w3 = wr * ri * ri;
    if (COMP >= 0) {
      akl[0] = fma(w3, d[COMP == 0 || COMP == 1 || COMP == 2 ? 0 : (COMP == 5 ? 2 : 1)] *
                           d[COMP == 0 ? 0 : (COMP == 1 || COMP == 3 ? 1 : 2)],
                   akl[0]);
    } else {
      akl[0] = fma(w3, d[0] * d[0], akl[0]);
      akl[1] = fma(w3, d[0] * d[1], akl[1]);
      akl[2] = fma(w3, d[0] * d[2], akl[2]);
      akl[3] = fma(w3, d[1] * d[1], akl[3]);
      akl[4] = fma(w3, d[1] * d[2], akl[4]);
      akl[5] = fma(w3, d[2] * d[2], akl[5]);
    }
  }
}

// pair sum in rule order (disjoint: test point outer, trial inner, weight
// w_i w_j, one sequential sum; touching: the table in the canonical warp
// order -- lane l accumulates points l, l + 32, ... and the 32 partials are
// combined by the xor butterfly -- run by a whole warp, WARP = true)
template <int COMP, bool WARP = false>
__device__ __forceinline__ void gal_sum(const Geom& g, const GalPair& P, double& ad,
                                        double* akl, int& nq_acc, int lane = 0) {
  if (P.pc == 0) {
    const int t = P.tier;
    const int n = c_rules.n[t];
    nq_acc += n * n;
#pragma unroll 1
    for (int qi = 0; qi < n; ++qi) {
      const double a1 = c_rules.a[t][qi], a2 = c_rules.b[t][qi], wi = c_rules.w[t][qi];
#pragma unroll 1
      for (int qj = 0; qj < n; ++qj)
        gal_point<COMP>(P, a1, a2, c_rules.a[t][qj], c_rules.b[t][qj], wi * c_rules.w[t][qj],
                        ad, akl);
    }
  } else if (WARP) {
    const int n = g.pr_n[P.pc];
    const double* r = g.prule + g.pr_off[P.pc];
    const long long T = g.prule_total;
    if (lane == 0) nq_acc += n;
#pragma unroll 1
    for (int q = lane; q < n; q += 32)
      gal_point<COMP>(P, r[q], r[T + q], r[2 * T + q], r[3 * T + q], r[4 * T + q], ad, akl);
    if (COMP == 6 || COMP < 0) ad = warp_sum(ad);
    if (COMP < 0) {
#pragma unroll
      for (int k = 0; k < 6; ++k) akl[k] = warp_sum(akl[k]);
    } else if (COMP != 6) {
      akl[0] = warp_sum(akl[0]);
    }
  }
}

// one component of a disjoint pair (ACA rows / columns of admissible
// blocks); comp 0..5 = V_kl, 6 = V_Delta
__device__ __forceinline__ double galerkin_entry1(const Geom& g, int i, int j, int comp,
                                                  int& nq_acc) {
  const GalPair P = gal_setup<false>(g, i, j);
  double ad = 0.0, akl[1] = {0.0};
  switch (comp) {  // group-uniform
    case 0: gal_sum<0>(g, P, ad, akl, nq_acc); break;
    case 1: gal_sum<1>(g, P, ad, akl, nq_acc); break;
    case 2: gal_sum<2>(g, P, ad, akl, nq_acc); break;
    case 3: gal_sum<3>(g, P, ad, akl, nq_acc); break;
    case 4: gal_sum<4>(g, P, ad, akl, nq_acc); break;
    case 5: gal_sum<5>(g, P, ad, akl, nq_acc); break;
    default: gal_sum<6>(g, P, ad, akl, nq_acc); return P.scale * ad;
  }
  return P.scale * akl[0];
}

// all seven components of a pair (near-field fill): out7[0..5] V_kl, [6]
// V_Delta.  WARP = false: a disjoint pair by one thread; true: any pair by a
// whole warp (touching pairs in the warp order; every lane gets the result)
template <bool WARP>
__device__ __forceinline__ void galerkin_entry7(const Geom& g, int i, int j, double* out7,
                                                int& nq_acc, int lane) {
  const GalPair P = gal_setup<WARP>(g, i, j);
  double ad = 0.0, akl[6] = {0, 0, 0, 0, 0, 0};
  if (WARP && P.pc == 0) {
    int dummy = 0;
    gal_sum<-1>(g, P, ad, akl, lane == 0 ? nq_acc : dummy);
  } else {
    gal_sum<-1, WARP>(g, P, ad, akl, nq_acc, lane);
  }
#pragma unroll
  for (int k = 0; k < 6; ++k) out7[k] = P.scale * akl[k];
  out7[6] = P.scale * ad;
}

// K_Delta(i, node) = sum over the node's triangles tau != i (ascending) of
// integrate_pair(i, tau) of (x-y).n(tau) / (4 pi |x-y|^3) psi_node(y)
// (kernels.cpp:151-167, no orientation swap), in the oracle's canonical
// order (Galerkin::kdelta): per pair sum_q fma(w / r^3, ((x-y).n) bary, .),
// scaled by 4 area_i area_tau / (4 pi), pairs summed in tau order.
// WARP = false: no triangle of the node touches i (admissible blocks, and
// the near field's thread pass), one thread; true: a whole warp, touching
// pairs summed in the canonical warp order (every lane gets the result).
template <int WARP>
__device__ __forceinline__ double kdelta_entry(const Geom& g, int i, int j, int& nq_acc,
                                               int lane) {
  const int4 a = g.tvid[i];
  const double4 ca = g.tce[a.w], na = g.tna[a.w];
  const int A[3] = {a.x, a.y, a.z};
  double total = 0.0;
  const int p1 = g.vt_ptr[j + 1];
#pragma unroll 1
  for (int p = g.vt_ptr[j]; p < p1; ++p) {
    const int2 tl = g.vt_tri[p];
    const int tau = tl.x, local = tl.y;
    if (tau == a.w) continue;
    const int4 b = g.tvx[tau];
    int ra = 0, rb = 0;
    const int pc = WARP ? gal_classify(a, b, ra, rb) : 0;
    const double4 cb = g.tce[tau], nb = g.tna[tau];
    const int B[3] = {b.x, b.y, b.z};
    const int xp0 = ra, xp1 = (ra + 1) % 3, xp2 = (ra + 2) % 3;
    int yp0 = rb, yp1 = (rb + 1) % 3;
    const int yp2 = (rb + 2) % 3;
    if (pc == 2) {
      const int t = yp0;
      yp0 = yp1;
      yp1 = t;
    }
    const double4 X0 = g.vtx[A[xp0]], X1 = g.vtx[A[xp1]], X2 = g.vtx[A[xp2]];
    const double4 Y0 = g.vtx[B[yp0]], Y1 = g.vtx[B[yp1]], Y2 = g.vtx[B[yp2]];
    const double x0[3] = {X0.x, X0.y, X0.z}, y0[3] = {Y0.x, Y0.y, Y0.z};
    const double ex1[3] = {X1.x - X0.x, X1.y - X0.y, X1.z - X0.z};
    const double ex2[3] = {X2.x - X0.x, X2.y - X0.y, X2.z - X0.z};
    const double ey1[3] = {Y1.x - Y0.x, Y1.y - Y0.y, Y1.z - Y0.z};
    const double ey2[3] = {Y2.x - Y0.x, Y2.y - Y0.y, Y2.z - Y0.z};
    // which rotated coordinate carries psi_node (kernels.cpp:119-123)
    const int role = local == yp0 ? 0 : (local == yp1 ? 1 : 2);
    double acc = 0.0;
    auto point = [&](double a1, double a2, double b1, double b2, double w) {
      double d[3];
#pragma unroll
      for (int c = 0; c < 3; ++c)
        d[c] = fma(a2, ex2[c], fma(a1, ex1[c], x0[c])) - fma(b2, ey2[c], fma(b1, ey1[c], y0[c]));
      const double ri = rsqrt_canon(fma(d[2], d[2], fma(d[1], d[1], d[0] * d[0])));
      const double w3 = w * ri * ri * ri;
      const double dn = fma(d[2], nb.z, fma(d[1], nb.y, d[0] * nb.x));
      const double bv = role == 0 ? (1.0 - b1) - b2 : (role == 1 ? b1 : b2);
      acc = fma(w3, dn * bv, acc);
    };
    if (pc == 0) {
      const int t = gal_tier(ca.x, ca.y, ca.z, ca.w, cb.x, cb.y, cb.z, cb.w);
      const int n = c_rules.n[t];
      if (!WARP || lane == 0) nq_acc += n * n;
#pragma unroll 1
      for (int qi = 0; qi < n; ++qi) {
        const double a1 = c_rules.a[t][qi], a2 = c_rules.b[t][qi], wi = c_rules.w[t][qi];
#pragma unroll 1
        for (int qj = 0; qj < n; ++qj)
          point(a1, a2, c_rules.a[t][qj], c_rules.b[t][qj], wi * c_rules.w[t][qj]);
      }
    } else {
      const int n = g.pr_n[pc];
      const double* r = g.prule + g.pr_off[pc];
      const long long T = g.prule_total;
      if (lane == 0) nq_acc += n;
#pragma unroll 1
      for (int q = lane; q < n; q += 32)
        point(r[q], r[T + q], r[2 * T + q], r[3 * T + q], r[4 * T + q]);
      acc = warp_sum(acc);
    }
    total += 4.0 * na.w * nb.w * (1.0 / (4.0 * M_PI)) * acc;
  }
  return total;
}

// does the pair (row i, column j) need the touching-pair rules?
__device__ __forceinline__ bool gal_touching(const Geom& g, int i, int j) {
  int ra, rb;
  return gal_classify(g.tvid[i], g.tvid[j], ra, rb) != 0;
}
__device__ __forceinline__ bool kd_touching(const Geom& g, int i, int j) {
  const int4 a = g.tvid[i];
  for (int p = g.vt_ptr[j]; p < g.vt_ptr[j + 1]; ++p) {
    const int tau = g.vt_tri[p].x;
    int ra, rb;
    if (tau != a.w && gal_classify(a, g.tvx[tau], ra, rb) != 0) return true;
  }
  return false;
}

// ---------------------------------------------------------------------------
// Double-layer collocation (CollocDoubleOracle / colloc_double, kernels.cpp:
// 189-210): evaluation point i (rows) x node j (columns), the traction of
// the Kelvin columns (kelvin_traction, kernels.cpp:30-55) in the closed form
//   T_rc = c [ (b1 n_r x_c + a2 n_c x_r + delta_rc a2 (n.x)) / r^3
//              - a6 x_r x_c (n.x) / r^5 ],  x = y - p,
// times the hat function of the node, over the node's triangles in
// ascending order; point_order tiers as colloc_single.  Canonical order
// shared with oracle/hmbem_oracle.cpp Kelvin::colloc_double.
__device__ __forceinline__ int kelvin_tier_c(double px, double py, double pz, double cx,
                                             double cy, double cz, double dj) {
  const double dx = __dsub_rn(px, cx), dy = __dsub_rn(py, cy), dz = __dsub_rn(pz, cz);
  const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                              __dmul_rn(dz, dz));
  const double t0 = (c_rules.far_ratio + 0.5) * dj, t1 = (c_rules.mid_ratio + 0.5) * dj;
  const double s0 = t0 * t0, s1 = t1 * t1;
  if (d2 > s0 * (1.0 + 1e-12)) return 0;
  if (d2 < s0 * (1.0 - 1e-12)) {
    if (d2 > s1 * (1.0 + 1e-12)) return 1;
    if (d2 < s1 * (1.0 - 1e-12)) return 2;
  }
  return kelvin_tier_exact(d2, dj);
}

__device__ __forceinline__ double kdouble_entry(const Geom& g, int i, int j, int& nq_acc) {
  const double4 p = g.rowpt[i];
  const int R = g.dl_r, Cc = g.dl_c;
  double acc = 0.0;
  const int p1 = g.vt_ptr[j + 1];
#pragma unroll 1
  for (int pp = g.vt_ptr[j]; pp < p1; ++pp) {
    const int2 tl = g.vt_tri[pp];
    const int tau = tl.x, local = tl.y;
    const int4 tv = g.tvx[tau];
    const double4 ce = g.tce[tau], na = g.tna[tau];
    const int tier = kelvin_tier_c(p.x, p.y, p.z, ce.x, ce.y, ce.z, ce.w);
    const double4 Y0 = g.vtx[tv.x], Y1 = g.vtx[tv.y], Y2 = g.vtx[tv.z];
    const double y0[3] = {Y0.x, Y0.y, Y0.z};
    const double e1[3] = {Y1.x - Y0.x, Y1.y - Y0.y, Y1.z - Y0.z};
    const double e2[3] = {Y2.x - Y0.x, Y2.y - Y0.y, Y2.z - Y0.z};
    const double pv[3] = {p.x, p.y, p.z};
    const double nn[3] = {na.x, na.y, na.z};
    const double nr = sel3(R, na.x, na.y, na.z), nc = sel3(Cc, na.x, na.y, na.z);
    const int n = c_rules.n[tier];
    nq_acc += n;
    double part = 0.0;
#pragma unroll 1
    for (int q = 0; q < n; ++q) {
      const double a = c_rules.a[tier][q], b = c_rules.b[tier][q], w = c_rules.w[tier][q];
      double x[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) x[d] = fma(b, e2[d], fma(a, e1[d], y0[d])) - pv[d];
      const double ri = rsqrt_canon(fma(x[2], x[2], fma(x[1], x[1], x[0] * x[0])));
      const double ri2 = ri * ri, ri3 = ri2 * ri, ri5 = ri3 * ri2;
      const double nx = fma(x[2], nn[2], fma(x[1], nn[1], x[0] * nn[0]));
      const double xr = sel3(R, x[0], x[1], x[2]), xc = sel3(Cc, x[0], x[1], x[2]);
      double sv = fma(g.dl_b1, nr * xc, g.dl_a2 * (nc * xr));
      if (R == Cc) sv = fma(g.dl_a2, nx, sv);
      const double v = fma(-(g.dl_a6 * ri5), (xr * xc) * nx, ri3 * sv);
      const double psi = local == 0 ? (1.0 - a) - b : (local == 1 ? a : b);
      part = fma(w * psi, v, part);
    }
    acc = acc + (2.0 * na.w * g.cst) * part;
  }
  return acc;
}

// Newton kernel: IEEE ops in the oracle's order, so entries are bit-exact
__device__ __forceinline__ double newton_entry(const Geom& g, int i, int j) {
  const double4 a = g.rowpt[i];
  const double4 b = g.colpt[j];
  const double dx = __dsub_rn(a.x, b.x), dy = __dsub_rn(a.y, b.y),
               dz = __dsub_rn(a.z, b.z);
  const double r = __dsqrt_rn(__dadd_rn(
      __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
  return r == 0.0 ? g.diag : __ddiv_rn(1.0, r);
}

__device__ __forceinline__ double dense_entry(const Geom& g, int i, int j) {
  return g.A[(long long)g.rperm[i] + g.lda * (long long)g.cperm[j]];
}

// single entry of component `comp` at internal (row i, col j)
__device__ __forceinline__ double entry1(const Geom& g, int i, int j,
                                         int comp) {
  int nq = 0;
  if (g.kind == KIND_KELVIN) return kelvin_entry1(g, i, j, comp, nq);
  if (g.kind == KIND_KDOUBLE) return kdouble_entry(g, i, j, nq);
  if (g.kind == KIND_NEWTON) return newton_entry(g, i, j);
  return dense_entry(g, i, j);
}
// the same with the provider fixed at compile time, for admissible blocks
// only (no diagonal entries; ACA kernel instances); nq_acc accumulates the
// quadrature points used (counted-flop bookkeeping)
template <int KIND>
__device__ __forceinline__ double entry_k(const Geom& g, int i, int j, int comp,
                                          int& nq_acc) {
  if (KIND == KIND_KELVIN) return kelvin_entry1<false>(g, i, j, comp, nq_acc);
  if (KIND == KIND_GALERKIN)
    return galerkin_entry1(g, i, j, g.gal_delta ? 6 : comp, nq_acc);
  if (KIND == KIND_KDELTA) return kdelta_entry<0>(g, i, j, nq_acc, 0);
  if (KIND == KIND_KDOUBLE) return kdouble_entry(g, i, j, nq_acc);
  if (KIND == KIND_NEWTON) return newton_entry(g, i, j);
  return dense_entry(g, i, j);
}

// ---------------------------------------------------------------------------
// ACA work item: one (admissible block, component).  State persists in
// device memory so that assembly, capacity regrow and AMVM extension all
// resume the same partial-pivoting sequence (aca.hpp:76-94, aca.cpp:106-143).
enum { PH_RUN = 0, PH_INIT = 1, PH_EXT = 2, PH_DONE = 3 };
enum { ST_OK = 0, ST_OVERFLOW = 1 };
enum { STOP_NONE = 0, STOP_INEQ = 1, STOP_EXH = 2, STOP_RANKCAP = 3,
       STOP_STEPS = 4 };

struct __align__(16) Item {
  int m, n, row0, col0;
  int comp, cap, k, kcur;
  int phase, steps_left, nconsumed, last_stop;
  int status, block, pad0, pad1;
  long long u_off, v_off;   // doubles; U is m x cap, V is n x cap, column-major
  long long z_off, p_off;   // consumed-mask bytes; pivot (int2) slots
  double frob_sq;
  long long entries;        // kernel entries evaluated
  long long steps;          // cross attempts (incl. vanishing rows)
  long long nq_sum;         // quadrature points over all evaluated entries
};
static_assert(sizeof(Item) == 128, "Item layout");

// one admissible block's record from which its NC work items are generated
// on the device (offsets of item q: U at u_base + q (align2(m cap) +
// align2(n cap)), V right after its U, pivots p_base + q max(cap, 1),
// consumed mask z_base + q align16(m))
struct AdmBlock {
  int m, n, row0, col0;
  int block, cap, pad0, pad1;
  long long u_base, p_base, z_base;
};

__global__ void items_init_kernel(const AdmBlock* __restrict__ ab, int nab, int nc,
                                  int phase, int steps_left, Item* __restrict__ items) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nab * nc) return;
  const int a = t / nc, q = t - a * nc;
  const AdmBlock b = ab[a];
  const long long su = ((long long)b.m * b.cap + 1) & ~1LL;
  const long long sv = ((long long)b.n * b.cap + 1) & ~1LL;
  Item it{};
  it.m = b.m;
  it.n = b.n;
  it.row0 = b.row0;
  it.col0 = b.col0;
  it.comp = q;
  it.cap = b.cap;
  it.block = b.block;
  it.phase = phase;
  it.steps_left = steps_left;
  it.last_stop = 0;  // STOP_NONE
  it.u_off = b.u_base + (long long)q * (su + sv);
  it.v_off = it.u_off + su;
  it.p_off = b.p_base + (long long)q * max(b.cap, 1);
  it.z_off = b.z_base + (long long)q * ((b.m + 15) & ~15);
  items[t] = it;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// Max / arg-max of non-negative doubles with the integer reduction unit
// (redux.sync): for x >= 0 the IEEE bit pattern is monotonic, so the max is
// found on the high then the low 32 bits.  Exact (no arithmetic on values).
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long k) {
  const unsigned hi = __reduce_max_sync(0xffffffffu, (unsigned)(k >> 32));
  const unsigned lo = __reduce_max_sync(0xffffffffu, (unsigned)(k >> 32) == hi ? (unsigned)k : 0u);
  return ((unsigned long long)hi << 32) | lo;
}
// max of v >= 0 over the warp
__device__ __forceinline__ double warp_max(double v) {
  return __longlong_as_double((long long)warp_max_u64((unsigned long long)__double_as_longlong(v)));
}
// first-max arg-max: larger val wins, ties go to the smaller index; lanes
// without a candidate carry val < 0 (and idx -1).  val >= 0 otherwise.
__device__ __forceinline__ void warp_argmax(double& val, int& idx, double& aux) {
  const unsigned long long key =
      val >= 0.0 ? (unsigned long long)__double_as_longlong(val) + 1ull : 0ull;
  const unsigned long long mk = warp_max_u64(key);
  const bool win = key == mk;
  const int mi = __reduce_min_sync(0xffffffffu, win ? idx : 0x7fffffff);
  const unsigned bal = __ballot_sync(0xffffffffu, win && idx == mi);
  const int src = __ffs(bal) - 1;
  aux = __shfl_sync(0xffffffffu, aux, src);
  val = __shfl_sync(0xffffffffu, val, src);
  idx = mi;
}
__device__ __forceinline__ int warp_min_int(int v) {
  return __reduce_min_sync(0xffffffffu, v);
}

// Residual of one row (is_row) or one column of the block, one warp:
//   row i:  out[c] = A(i, c) - sum_l U(i, l) V(c, l)      (W = U, X = V)
//   col j:  out[r] = A(r, j) - sum_l V(j, l) U(r, l)      (W = V, X = U)
// l ascending with fma, exactly as aca.cpp:61-64 / :79-82 restated by the
// oracle.  Per lane: max |A| (row scale), first-max |out| and sum out^2.
// The only call site of the entry provider inside the ACA (one copy of the
// quadrature code: the ACA kernel is instruction-cache bound otherwise).
struct LineStats {
  double rs, pm, pv, sq;
  int pj, nq;
};

// Entry source of the ACA: evaluates the kernel from the geometry in HBM.
// (A variant that evaluated small blocks whole into shared memory first,
// all six components together, was measured slower: the per-step chain of
// small blocks is dominated by the factor loads and warp reductions, and the
// CTA-per-block occupancy was lower.)
template <int KIND>
struct EvalSrc {
  const Geom& g;
  int row0, col0, comp;
  __device__ __forceinline__ double operator()(bool is_row, int fix, int t, int& nq) const {
    const int i = is_row ? row0 + fix : row0 + t;
    const int j = is_row ? col0 + t : col0 + fix;
    return entry_k<KIND>(g, i, j, comp, nq);
  }
};

template <int NT, class SRC>
__device__ __forceinline__ LineStats residual_line(const SRC& src, bool is_row, int fix,
                                                   const double* __restrict__ W, int ldw,
                                                   const double* __restrict__ X, int ldx,
                                                   int len, int k, double* __restrict__ out,
                                                   double* __restrict__ ebuf, int lane) {
  constexpr int nt = NT;
  // nt threads (one warp, or the CTA for the largest items); element t is
  // handled by thread t % nt, the lane-strided order of the canonical sums
  LineStats st{0.0, -1.0, 0.0, 0.0, -1, 0};
  for (int base = 0; base < len; base += 4 * nt) {
    const int rem = len - base;  // group-uniform; nb = min(4, ceil(rem / nt))
    const int nb = rem > 3 * nt ? 4 : rem > 2 * nt ? 3 : rem > nt ? 2 : 1;
    double v[4];
    bool ok[4];
    // phase A: the kernel entries of up to 4 columns per lane (arithmetic
    // only; parked in this lane's shared-memory slots)
#pragma unroll 1
    for (int s = 0; s < nb; ++s) {
      const int t = base + nt * s + lane;
      ebuf[nt * s + lane] = t < len ? src(is_row, fix, t, st.nq) : 0.0;
    }
    // phase B: the low-rank correction, four independent columns per lane so
    // that eight panel loads are in flight per lane
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int t = base + nt * s + lane;
      ok[s] = s < nb && t < len;
      v[s] = ok[s] ? ebuf[nt * s + lane] : 0.0;
      if (ok[s]) st.rs = fmax(st.rs, fabs(v[s]));
    }
    const double* xb = X + base + lane;
HM_UNROLL(HMGPU_RUNROLL)
    for (int l = 0; l < k; ++l) {
      const double w = -W[(long long)l * ldw + fix];
      const double* xl = xb + (long long)l * ldx;
#pragma unroll
      for (int s = 0; s < 4; ++s)
        if (ok[s]) v[s] = fma(w, xl[nt * s], v[s]);
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (!ok[s]) continue;
      const int t = base + nt * s + lane;
      out[t] = v[s];
      st.sq = fma(v[s], v[s], st.sq);
      if (fabs(v[s]) > st.pm) {
        st.pm = fabs(v[s]);
        st.pj = t;
        st.pv = v[s];
      }
    }
  }
  return st;
}

// sum_l du_l dv_l (fma, l ascending) with du_l = warp-order dot(u, U(:,l)),
// dv_l = warp-order dot(v, V(:,l)).  Eight l at a time: lane-strided fma
// partials, then a reduce-scatter butterfly (bits 4, 3, 2 exchange halves,
// bits 1, 0 all-reduce).  Every node of that tree adds the same two operands
// as warp_sum's xor butterfly, so each du_l is bit-identical to
// warp_sum(partial) (the oracle's warp_dot), at 9 instead of 40 shuffles.
__device__ __forceinline__ double rs8(double (&p)[8], int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
  double a[4];
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const double send = b4 ? p[h] : p[h + 4];
    const double keep = b4 ? p[h + 4] : p[h];
    a[h] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  double b[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const double send = b3 ? a[h] : a[h + 2];
    const double keep = b3 ? a[h + 2] : a[h];
    b[h] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  const double send = b2 ? b[0] : b[1];
  const double keep = b2 ? b[1] : b[0];
  double v = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v;  // the full sum for index q = (lane >> 2) & 7
}

__device__ __forceinline__ double cross_terms(const double* __restrict__ uk,
                                           const double* __restrict__ U, int m,
                                           const double* __restrict__ vk,
                                           const double* __restrict__ V, int n, int k,
                                           int lane) {
  double cross = 0.0;
  for (int l0 = 0; l0 < k; l0 += 8) {
    const int nl = min(8, k - l0);
    double pu[8], pv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) pu[q] = pv[q] = 0.0;
    for (int r = lane; r < m; r += 64) {
      const bool two = r + 32 < m;
      const double a0 = uk[r], a1 = two ? uk[r + 32] : 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (q < nl) {
          const double* ul = U + (long long)(l0 + q) * m + r;
          const double x0 = ul[0];
          const double x1 = two ? ul[32] : 0.0;
          pu[q] = fma(a0, x0, pu[q]);
          if (two) pu[q] = fma(a1, x1, pu[q]);
        }
      }
    }
    for (int c = lane; c < n; c += 64) {
      const bool two = c + 32 < n;
      const double a0 = vk[c], a1 = two ? vk[c + 32] : 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (q < nl) {
          const double* vl = V + (long long)(l0 + q) * n + c;
          const double x0 = vl[0];
          const double x1 = two ? vl[32] : 0.0;
          pv[q] = fma(a0, x0, pv[q]);
          if (two) pv[q] = fma(a1, x1, pv[q]);
        }
      }
    }
    const double du = rs8(pu, lane);
    const double dv = rs8(pv, lane);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (q < nl) {
        const double a = __shfl_sync(0xffffffffu, du, 4 * q);
        const double b = __shfl_sync(0xffffffffu, dv, 4 * q);
        cross = fma(a, b, cross);
      }
    }
  }
  return cross;
}

// ---------------------------------------------------------------------------
// Work groups of the ACA.  An item (block, component) is run either by one
// warp (gsize 32, gtid = lane) or, for the largest blocks, by the whole CTA
// (gsize ACA_NT, gtid = threadIdx.x): a single warp on a block with m + n in
// the thousands was latency-bound on its panel loads and made the largest
// items the critical path of the assembly (config 3: 196 ms for the 192
// items with m + n >= 16384 run alone).  CTA of 128 threads, items with
// m + n >= 1024 (HMGPU_ACA_CTA_MIN; measured against 256 / 512 threads and
// 512 / 2048 / 4096).  Both modes give the same bits: the
// max / arg-max reductions are exact, and the CTA mode forms the canonical
// lane-strided sums (||u||^2, ||v||^2, u.U(:,l), v.V(:,l)) with one warp per
// sum from the stored line, in the warp mode's order.
#ifndef HMGPU_ACA_NT
#define HMGPU_ACA_NT 128
#endif
constexpr int ACA_NT = HMGPU_ACA_NT;
constexpr int ACA_NW = ACA_NT / 32;

struct AcaShared {
  double ebuf[4 * ACA_NT];   // entry slots: warp mode [warp][4][32], CTA mode [4][ACA_NT]
  double du[ACA_NT], dv[ACA_NT];  // CTA mode: per-l dots of the cross terms
  double rd[ACA_NW], ra[ACA_NW];
  long long rl[ACA_NW];
  int ri[ACA_NW];
  double uu, vv;
  int t;
};

template <int NT>
struct Grp {
  int tid;
  static constexpr int size = NT;
  __host__ __device__ static constexpr bool cta() { return NT > 32; }
  __device__ __forceinline__ int lane() const { return tid & 31; }
  __device__ __forceinline__ int warp() const { return tid >> 5; }
};

template <int NT>
__device__ __forceinline__ void gsync(const Grp<NT>& g) {
  if (g.cta()) __syncthreads();
  else __syncwarp();
}

template <int NT>
__device__ __forceinline__ double cta_max(double v, const Grp<NT>& g, AcaShared& sh) {
  if (g.lane() == 0) sh.rd[g.warp()] = v;
  __syncthreads();
  double r = sh.rd[0];
#pragma unroll
  for (int w = 1; w < ACA_NW; ++w) r = fmax(r, sh.rd[w]);
  __syncthreads();
  return r;
}
template <int NT>
__device__ __forceinline__ double grp_max(double v, const Grp<NT>& g, AcaShared& sh) {
  v = warp_max(v);
  return g.cta() ? cta_max(v, g, sh) : v;
}

template <int NT>
__device__ __forceinline__ int cta_min_int(int v, const Grp<NT>& g, AcaShared& sh) {
  if (g.lane() == 0) sh.ri[g.warp()] = v;
  __syncthreads();
  int r = sh.ri[0];
#pragma unroll
  for (int w = 1; w < ACA_NW; ++w) r = min(r, sh.ri[w]);
  __syncthreads();
  return r;
}
template <int NT>
__device__ __forceinline__ int grp_min_int(int v, const Grp<NT>& g, AcaShared& sh) {
  v = warp_min_int(v);
  return g.cta() ? cta_min_int(v, g, sh) : v;
}

template <int NT>
__device__ __forceinline__ long long grp_sum_ll(long long t, const Grp<NT>& g, AcaShared& sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (!g.cta()) return t;
  if (g.lane() == 0) sh.rl[g.warp()] = t;
  __syncthreads();
  long long r = 0;
#pragma unroll
  for (int w = 0; w < ACA_NW; ++w) r += sh.rl[w];
  __syncthreads();
  return r;
}

// first-max arg-max over the group (larger value, then smaller index)
template <int NT>
__device__ __forceinline__ void cta_argmax(double& val, int& idx, double& aux, const Grp<NT>& g,
                                        AcaShared& sh) {
  if (g.lane() == 0) {
    sh.rd[g.warp()] = val;
    sh.ri[g.warp()] = idx;
    sh.ra[g.warp()] = aux;
  }
  __syncthreads();
  double bv = sh.rd[0], ba = sh.ra[0];
  int bi = sh.ri[0];
#pragma unroll
  for (int w = 1; w < ACA_NW; ++w) {
    const double v = sh.rd[w];
    const int i = sh.ri[w];
    if (v > bv || (v == bv && i >= 0 && (bi < 0 || i < bi))) {
      bv = v;
      bi = i;
      ba = sh.ra[w];
    }
  }
  __syncthreads();
  val = bv;
  idx = bi;
  aux = ba;
}
template <int NT>
__device__ __forceinline__ void grp_argmax(double& val, int& idx, double& aux, const Grp<NT>& g,
                                           AcaShared& sh) {
  warp_argmax(val, idx, aux);
  if (g.cta()) cta_argmax(val, idx, aux, g, sh);
}

// canonical lane-strided dot (warp order, as warp_sum of fma partials)
__device__ __forceinline__ double warp_dot(const double* __restrict__ a,
                                           const double* __restrict__ b, int len, int lane) {
  double p = 0.0;
  for (int r = lane; r < len; r += 32) p = fma(a[r], b[r], p);
  return warp_sum(p);
}

// CTA mode: ||u||^2 and ||v||^2 (warps 0 and 1) and the dots u.U(:,l),
// v.V(:,l) of the cross terms (l spread over the warps), each a canonical
// warp-order sum of the stored line; cross = sum_l du_l dv_l in l order.
template <int NT>
__device__ __forceinline__ double cta_norms_cross(const double* __restrict__ uk, const double* __restrict__ U,
                                  int m, const double* __restrict__ vk,
                                  const double* __restrict__ V, int n, int k, const Grp<NT>& g,
                                  AcaShared& sh, double& uu, double& vv) {
  const int lane = g.lane(), w = g.warp();
  __syncthreads();  // the line is complete
  if (w == 0) {
    const double t = warp_dot(uk, uk, m, lane);
    if (lane == 0) sh.uu = t;
  } else if (w == 1) {
    const double t = warp_dot(vk, vk, n, lane);
    if (lane == 0) sh.vv = t;
  }
  double cross = 0.0;
  for (int l0 = 0; l0 < k; l0 += ACA_NT) {
    const int l1 = min(k, l0 + ACA_NT);
    // two l per pass share the loads of the line
    for (int l = l0 + w; l < l1; l += 2 * ACA_NW) {
      const int la = l, lb = l + ACA_NW;
      const bool hb = lb < l1;
      const double* Ua = U + (long long)la * m;
      const double* Ub = U + (long long)(hb ? lb : la) * m;
      const double* Va = V + (long long)la * n;
      const double* Vb = V + (long long)(hb ? lb : la) * n;
      double pa = 0.0, pb = 0.0, qa = 0.0, qb = 0.0;
      for (int r = lane; r < m; r += 32) {
        const double x = uk[r];
        pa = fma(x, Ua[r], pa);
        pb = fma(x, Ub[r], pb);
      }
      for (int c = lane; c < n; c += 32) {
        const double x = vk[c];
        qa = fma(x, Va[c], qa);
        qb = fma(x, Vb[c], qb);
      }
      pa = warp_sum(pa);
      qa = warp_sum(qa);
      pb = warp_sum(pb);
      qb = warp_sum(qb);
      if (lane == 0) {
        sh.du[la - l0] = pa;
        sh.dv[la - l0] = qa;
        if (hb) {
          sh.du[lb - l0] = pb;
          sh.dv[lb - l0] = qb;
        }
      }
    }
    __syncthreads();
    for (int l = l0; l < l1; ++l) cross = fma(sh.du[l - l0], sh.dv[l - l0], cross);
    __syncthreads();
  }
  if (k == 0) __syncthreads();
  uu = sh.uu;
  vv = sh.vv;
  return cross;
}

// One ACA step of aca_step (aca.cpp:41-102) executed by one group.
// sf < 0 disables the accuracy test (extension mode).  The candidate row
// residual is built in V(:,k) and the column residual in U(:,k); both are
// only committed (k += 1) when the step is accepted.
template <int NT, class SRC>
__device__ __forceinline__ int aca_step(const SRC& src, Item& s, double* __restrict__ U,
                        double* __restrict__ V, int2* __restrict__ piv,
                        uint8_t* __restrict__ Z, double sf, const Grp<NT>& g, int& nq_acc,
                        double* __restrict__ ebuf, AcaShared& sh) {
  const int m = s.m, n = s.n, k = s.k;
  const int tid = g.tid;
  constexpr int gs = NT;
  for (;;) {
    if (s.nconsumed == m) return STOP_EXH;
    s.steps++;
    // --- row pivot: first unconsumed row (k = 0) or first max |U(r,k-1)|
    int i;
    if (k == 0) {
      int first = 0x7fffffff;
      for (int r = tid; r < m; r += gs)
        if (!Z[r]) {
          first = r;
          break;
        }
      i = grp_min_int(first, g, sh);
    } else {
      const double* ul = U + (long long)(k - 1) * m;
      double best = -1.0, aux = 0.0;
      int bi = -1;
      for (int r = tid; r < m; r += gs) {
        if (Z[r]) continue;
        const double mag = fabs(ul[r]);
        if (mag > best) {
          best = mag;
          bi = r;
        }
      }
      grp_argmax(best, bi, aux, g, sh);
      i = bi;
    }
    // --- row of the residual: v = A(i,:) - sum_l U(i,l) V(:,l), then the
    // column u = A(:,j) - sum_l V(j,l) U(:,l); one loop so that the entry
    // provider is instantiated once (instruction cache)
    double* vk = V + (long long)k * n;
    double* uk = U + (long long)k * m;
    int fix = i, j = -1;
    double vv = 0.0, uu = 0.0;
    bool vanished = false;
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
      const bool is_row = pass == 0;
      const LineStats ls = residual_line<NT>(
          src, is_row, fix, is_row ? U : V, is_row ? m : n,
          is_row ? V : U, is_row ? n : m, is_row ? n : m, k, is_row ? vk : uk, ebuf, tid);
      nq_acc += ls.nq;
      s.entries += is_row ? n : m;
      if (!is_row) {
        if (!g.cta()) uu = warp_sum(ls.sq);
        break;
      }
      const double row_scale = grp_max(ls.rs, g, sh);
      double pm = ls.pm, pv = ls.pv;
      int pj = ls.pj;
      grp_argmax(pm, pj, pv, g, sh);
      if (tid == 0) Z[i] = 1;
      s.nconsumed++;
      gsync(g);
      if (pm <= 1e-14 * row_scale || row_scale == 0.0) {  // vanishing
        vanished = true;
        break;
      }
      j = pj;
      // thread t owns elements t mod gs of the line (as in residual_line)
      for (int c = tid; c < n; c += gs) {
        const double t = vk[c] / pv;
        vk[c] = t;
        vv = fma(t, t, vv);
      }
      fix = j;
    }
    if (vanished) continue;
    double cross = 0.0;
    if (g.cta()) {
      cross = cta_norms_cross(uk, U, m, vk, V, n, k, g, sh, uu, vv);
    } else {
      vv = warp_sum(vv);
    }
    if (sf >= 0.0 && sqrt(uu) * sqrt(vv) <= sf * sqrt(fmax(s.frob_sq, 0.0))) {
      gsync(g);
      return STOP_INEQ;
    }
    // ||S_k||^2 = ||S_{k-1}||^2 + 2 sum_l (u.u_l)(v.v_l) + ||u||^2 ||v||^2
    if (!g.cta()) cross = cross_terms(uk, U, m, vk, V, n, k, g.lane());
    s.frob_sq += 2.0 * cross + uu * vv;
    if (tid == 0) piv[k] = make_int2(i, j);
    s.k = k + 1;
    gsync(g);
    return STOP_NONE;
  }
}

// per-item completion times of the last ACA launch (null = off)
__device__ unsigned long long* g_aca_trace = nullptr;

// Runs one item's state machine until done or out of column capacity:
//   PH_RUN  aca_run to the stopping rule (aca.cpp:106-124)
//   PH_INIT coarse mode: aca_extend(initial_rank) (hmatrix.cpp:156-158)
//   PH_EXT  aca_extend(steps_left) (aca.cpp:126-143)
// One call site of the step for all phases and both group modes (code size).
template <int NT, class SRC>
__device__ __forceinline__ void aca_item(const SRC& src, Item& s, Item* __restrict__ items, int idx,
                         double* __restrict__ arena, int2* __restrict__ pivots,
                         uint8_t* __restrict__ cons, double sf_run, long long max_rank,
                         int lookahead, int* __restrict__ overflow, const Grp<NT>& g,
                         double* __restrict__ ebuf, AcaShared& sh) {
  double* U = arena + s.u_off;
  double* V = arena + s.v_off;
  int2* piv = pivots + s.p_off;
  uint8_t* Z = cons + s.z_off;
  const long long capr_ll = min(max_rank, (long long)min(s.m, s.n));
  const int capr = (int)capr_ll;
  s.status = ST_OK;
  int nq_acc = 0;
  while (s.phase != PH_DONE) {
    const bool run = s.phase == PH_RUN;
    const bool more = run ? s.k < capr : (s.steps_left > 0 && s.k < capr);
    int st = STOP_NONE;
    if (more) {
      if (s.k >= s.cap) {
        s.status = ST_OVERFLOW;
        break;
      }
      st = aca_step(src, s, U, V, piv, Z, run ? sf_run : -1.0, g, nq_acc, ebuf, sh);
      if (st == STOP_NONE) {
        if (!run) s.steps_left--;
        continue;
      }
    }
    if (run) {
      s.last_stop = st != STOP_NONE ? st : (s.nconsumed == s.m ? STOP_EXH : STOP_RANKCAP);
      s.kcur = s.k;
      s.phase = PH_EXT;
      s.steps_left = lookahead;
    } else {
      s.last_stop = st != STOP_NONE                      ? st
                    : (s.nconsumed == s.m)               ? STOP_EXH
                    : (s.k >= capr && s.steps_left > 0) ? STOP_RANKCAP
                                                        : STOP_STEPS;
      if (s.phase == PH_INIT) {
        s.kcur = s.k;
        s.phase = PH_EXT;
        s.steps_left = lookahead;
      } else {
        s.phase = PH_DONE;
        s.steps_left = 0;
      }
    }
  }
  gsync(g);
  s.nq_sum += grp_sum_ll(nq_acc, g, sh);
  if (g.tid == 0) {
    items[idx] = s;
    if (g_aca_trace) {  // diagnostics (HMGPU_ACA_TRACE): item end time, ns
      unsigned long long ns;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
      g_aca_trace[idx] = ns;
    }
    if (s.status == ST_OVERFLOW) atomicAdd(overflow, 1);
  }
}

// Persistent kernel.  list[0, nbig) (the largest items; the list is sorted
// by m + n, largest first) is run CTA by CTA through counter[0]; then every
// warp pulls single items from list[nbig, nlist) through counter[1].  One
// item machine instance per mode.
#ifndef HMGPU_ACA_MINB
#define HMGPU_ACA_MINB (512 / ACA_NT)
#endif
template <int KIND, int MINB = HMGPU_ACA_MINB>
__global__ void __launch_bounds__(ACA_NT, MINB)
aca_kernel(Geom g, Item* __restrict__ items, const int* __restrict__ list, int nlist,
           int nbig, int* __restrict__ counter, double* __restrict__ arena,
           int2* __restrict__ pivots, uint8_t* __restrict__ cons, double sf_run,
           long long max_rank, int lookahead, int* __restrict__ overflow, int big_ctas) {
  __shared__ AcaShared sh;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // only the first big_ctas CTAs take the CTA-cooperative items (fewer of
  // them in flight keeps their factor panels in L2); the others start with
  // the single-warp items
  bool cta_mode = nbig > 0 && (int)blockIdx.x < big_ctas;
  for (;;) {
    int t;
    if (cta_mode) {
      if (threadIdx.x == 0) sh.t = atomicAdd(counter, 1);
      __syncthreads();
      t = sh.t;
      __syncthreads();
      if (t >= nbig) {
        cta_mode = false;
        continue;
      }
    } else {
      t = 0;
      if (lane == 0) t = nbig + atomicAdd(counter + 1, 1);
      t = __shfl_sync(0xffffffffu, t, 0);
      if (t >= nlist) return;
    }
    const int idx = list[t];
    Item s = items[idx];
    const EvalSrc<KIND> src{g, s.row0, s.col0, s.comp};
    // the group size is a compile-time constant of each instance (a runtime
    // stride cost the warp mode 13 % on config 2)
    if (cta_mode)
      aca_item(src, s, items, idx, arena, pivots, cons, sf_run, max_rank, lookahead, overflow,
               Grp<ACA_NT>{(int)threadIdx.x}, sh.ebuf, sh);
    else
      aca_item(src, s, items, idx, arena, pivots, cons, sf_run, max_rank, lookahead, overflow,
               Grp<32>{lane}, sh.ebuf + 128 * warp, sh);  // [4][32] per warp
  }
}

// ---------------------------------------------------------------------------
// near-field fill: one CTA per non-admissible block, all NC components of a
// pair computed together (they share r and 1/r); layout per block
// [j][comp][i] with column pitch align2(NC*m): a column range of the block
// is one contiguous run (the unit the matvec streams) and rows are the
// fastest index (lane = row, conflict-free in shared memory)
struct DenseBlock {
  int m, n, row0, col0;
  long long off;  // doubles into the dense arena
};

template <int NC>
__global__ void __launch_bounds__(256)
nearfield_kernel(Geom g, const DenseBlock* __restrict__ blocks, int nblocks,
                 double* __restrict__ dense, unsigned long long* __restrict__ nq_total) {
  int nq_acc = 0;
  for (int bi = blockIdx.x; bi < nblocks; bi += gridDim.x) {
    const DenseBlock b = blocks[bi];
    const int mn = b.m * b.n;
    const int cp = (b.m * NC + 1) & ~1;  // column pitch, 16-byte multiple
    double* D = dense + b.off;
    for (int p = threadIdx.x; p < mn; p += blockDim.x) {
      const int i = p % b.m, j = p / b.m;
      if (NC == 6) {
        double e[6];
        if (g.kind == KIND_KELVIN) {
          kelvin_entry6(g, b.row0 + i, b.col0 + j, e, nq_acc);
        } else {
          const double v = entry1(g, b.row0 + i, b.col0 + j, 0);
#pragma unroll
          for (int c = 0; c < 6; ++c) e[c] = v;
        }
#pragma unroll
        for (int c = 0; c < 6; ++c) D[(long long)j * cp + c * b.m + i] = e[c];
      } else {
        D[(long long)j * cp + i] = entry1(g, b.row0 + i, b.col0 + j, 0);
      }
    }
  }
  unsigned long long t = (unsigned long long)nq_acc;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0 && t) atomicAdd(nq_total, t);
}

// Galerkin near field (V_kl grid: NC = 6, V_Delta / K_Delta: NC = 1): a
// thread per disjoint pair (sequential sum), then a warp per touching pair
// (the Sauter-Schwab tables, up to 39366 points, in the canonical warp
// order).  Pairs are taken in chunks of GAL_CHUNK; the touching ones of a
// chunk are listed in shared memory for the warp pass.
constexpr int GAL_CHUNK = 1024;
template <int NC>
__global__ void __launch_bounds__(256)
nearfield_gal_kernel(Geom g, const DenseBlock* __restrict__ blocks, int nblocks,
                     double* __restrict__ dense, unsigned long long* __restrict__ nq_total) {
  __shared__ int tlist[GAL_CHUNK];
  __shared__ int tcount;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool kd = g.kind == KIND_KDELTA;
  int nq_acc = 0;
  for (int bi = blockIdx.x; bi < nblocks; bi += gridDim.x) {
    const DenseBlock b = blocks[bi];
    const int mn = b.m * b.n;
    const int cp = (b.m * NC + 1) & ~1;  // column pitch, 16-byte multiple
    double* D = dense + b.off;
    auto store = [&](int i, int j, const double* e7) {
      if (NC == 6) {
#pragma unroll
        for (int c = 0; c < 6; ++c) D[(long long)j * cp + c * b.m + i] = e7[c];
      } else {
        D[(long long)j * cp + i] = e7[6];
      }
    };
    for (int c0 = 0; c0 < mn; c0 += GAL_CHUNK) {
      const int c1 = min(mn, c0 + GAL_CHUNK);
      if (threadIdx.x == 0) tcount = 0;
      __syncthreads();
      for (int p = c0 + threadIdx.x; p < c1; p += blockDim.x) {
        const int i = p % b.m, j = p / b.m;
        const bool touch = kd ? kd_touching(g, b.row0 + i, b.col0 + j)
                              : gal_touching(g, b.row0 + i, b.col0 + j);
        if (touch) {
          tlist[atomicAdd(&tcount, 1)] = p;
          continue;
        }
        double e7[7];
        if (kd) e7[6] = kdelta_entry<0>(g, b.row0 + i, b.col0 + j, nq_acc, lane);
        else galerkin_entry7<false>(g, b.row0 + i, b.col0 + j, e7, nq_acc, lane);
        store(i, j, e7);
      }
      __syncthreads();
      const int nt = tcount;
      for (int t = warp; t < nt; t += blockDim.x >> 5) {
        const int p = tlist[t];
        const int i = p % b.m, j = p / b.m;
        double e7[7];
        if (kd) e7[6] = kdelta_entry<1>(g, b.row0 + i, b.col0 + j, nq_acc, lane);
        else galerkin_entry7<true>(g, b.row0 + i, b.col0 + j, e7, nq_acc, lane);
        if (lane == 0) store(i, j, e7);
      }
      __syncthreads();
    }
  }
  unsigned long long t = (unsigned long long)nq_acc;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0 && t) atomicAdd(nq_total, t);
}

// ---------------------------------------------------------------------------
// H-matvec.  x is gathered into internal order xi[(p*NOUT + r)*nrhs + q];
// every owned block writes a partial ypart[(prow + i)*NOUT*nrhs + r*nrhs + q]
// for its rows; a per-leaf pass sums the partials of all blocks covering
// the leaf in a fixed order (deterministic) and scatters to external order.
struct MvBlock {
  int m, n, row0, col0;
  int dense, item0, pad0, pad1;
  long long dense_off;
  long long prow;  // partial row offset
};

template <int NOUT>
__global__ void gather_kernel(const double* __restrict__ x, double* __restrict__ xi,
                              const int* __restrict__ cperm, int ncols, int nrhs) {
  const long long total = (long long)ncols * NOUT * nrhs;
  const long long ndof = (long long)ncols * NOUT;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int q = (int)(t % nrhs);
    const long long pr = t / nrhs;
    const int r = (int)(pr % NOUT);
    const int p = (int)(pr / NOUT);
    xi[t] = x[q * ndof + (long long)r * ncols + cperm[p]];
  }
}

template <int NC>
__global__ void __launch_bounds__(256)
hmv_blocks_kernel(const MvBlock* __restrict__ blocks, const int* __restrict__ order,
                  int nblocks, const Item* __restrict__ items,
                  const double* __restrict__ arena,
                  const double* __restrict__ dense, const double* __restrict__ xi,
                  double* __restrict__ ypart, int nrhs, int mode) {
  constexpr int NOUT = NC == 6 ? 3 : 1;
  extern __shared__ double zsm[];  // [2][kmax][nrhs]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  for (int oi = blockIdx.x; oi < nblocks; oi += gridDim.x) {
    const MvBlock b = blocks[order[oi]];
    double* yp = ypart + b.prow * NOUT * nrhs;
    if (b.dense && b.m > (int)blockDim.x) {  // wide near-field block: a thread per row
      for (int i = threadIdx.x; i < b.m; i += blockDim.x) {
        for (int q = 0; q < nrhs; ++q) {
          double acc[NOUT];
#pragma unroll
          for (int r = 0; r < NOUT; ++r) acc[r] = 0.0;
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            const int rr = NC == 6 ? c_comp_r[c] : 0;
            const int cc = NC == 6 ? c_comp_c[c] : 0;
            const long long cp = (b.m * NC + 1) & ~1;
            const double* D = dense + b.dense_off + (long long)c * b.m + i;
            double s1 = 0.0, s2 = 0.0;
            for (int j = 0; j < b.n; ++j) {
              const double d = D[j * cp];
              const double* xj = xi + ((long long)(b.col0 + j) * NOUT) * nrhs + q;
              s1 = fma(d, xj[cc * nrhs], s1);
              if (rr != cc) s2 = fma(d, xj[rr * nrhs], s2);
            }
            acc[rr] += s1;
            if (rr != cc) acc[cc] += s2;
          }
#pragma unroll
          for (int r = 0; r < NOUT; ++r) yp[((long long)i * NOUT + r) * nrhs + q] = acc[r];
        }
      }
      __syncthreads();
      continue;
    }
    if (b.dense) {
      // thread (i, part): rows i < m, the P = blockDim / m parts take the
      // column range in contiguous slices; the part sums are added in part
      // order (deterministic) -- a near-field block has m <= 64 rows, so one
      // thread per row would leave most of the CTA idle
      __shared__ double dred[256 * NOUT];
      const int P = max(1, min((int)blockDim.x / b.m, b.n));
      const int per = (b.n + P - 1) / P;
      const int i = threadIdx.x % b.m, part = threadIdx.x / b.m;
      const bool act = part < P;
      const int j0 = act ? part * per : 0, j1 = act ? min(b.n, j0 + per) : 0;
      const long long cp = (b.m * NC + 1) & ~1;
      for (int q = 0; q < nrhs; ++q) {
        double acc[NOUT];
#pragma unroll
        for (int r = 0; r < NOUT; ++r) acc[r] = 0.0;
        if (act) {
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            const int rr = NC == 6 ? c_comp_r[c] : 0;
            const int cc = NC == 6 ? c_comp_c[c] : 0;
            const double* D = dense + b.dense_off + (long long)c * b.m + i;
            double s1 = 0.0, s2 = 0.0;
            for (int j = j0; j < j1; ++j) {
              const double d = D[j * cp];
              const double* xj = xi + ((long long)(b.col0 + j) * NOUT) * nrhs + q;
              s1 = fma(d, xj[cc * nrhs], s1);
              if (rr != cc) s2 = fma(d, xj[rr * nrhs], s2);
            }
            acc[rr] += s1;
            if (rr != cc) acc[cc] += s2;
          }
#pragma unroll
          for (int r = 0; r < NOUT; ++r) dred[(part * b.m + i) * NOUT + r] = acc[r];
        }
        __syncthreads();
        for (int t = threadIdx.x; t < b.m * NOUT; t += blockDim.x) {
          double s = dred[t];
          for (int h = 1; h < P; ++h) s += dred[h * b.m * NOUT + t];
          const int ii = t / NOUT, r = t % NOUT;
          yp[((long long)ii * NOUT + r) * nrhs + q] = s;
        }
        __syncthreads();
      }
      continue;
    }
    // low rank: per component z = V^T x_c (and w = V^T x_r), then U z
    for (int c = 0; c < NC; ++c) {
      const Item it = items[b.item0 + c];
      const int k = mode ? it.k : it.kcur;
      const int rr = NC == 6 ? c_comp_r[c] : 0;
      const int cc = NC == 6 ? c_comp_c[c] : 0;
      const bool two = rr != cc;
      const double* V = arena + it.v_off;
      const double* U = arena + it.u_off;
      for (int l = warp; l < k; l += nwarps) {
        const double* vl = V + (long long)l * b.n;
        for (int q = 0; q < nrhs; ++q) {
          double s1 = 0.0, s2 = 0.0;
          for (int j = lane; j < b.n; j += 32) {
            const double v = vl[j];
            const double* xj = xi + ((long long)(b.col0 + j) * NOUT) * nrhs + q;
            s1 = fma(v, xj[cc * nrhs], s1);
            if (two) s2 = fma(v, xj[rr * nrhs], s2);
          }
          s1 = warp_sum(s1);
          if (two) s2 = warp_sum(s2);
          if (lane == 0) {
            zsm[l * nrhs + q] = s1;
            zsm[(k + l) * nrhs + q] = s2;
          }
        }
      }
      __syncthreads();
      for (int i = threadIdx.x; i < b.m; i += blockDim.x) {
        for (int q = 0; q < nrhs; ++q) {
          double s1 = 0.0, s2 = 0.0;
          for (int l = 0; l < k; ++l) {
            const double u = U[(long long)l * b.m + i];
            s1 = fma(u, zsm[l * nrhs + q], s1);
            if (two) s2 = fma(u, zsm[(k + l) * nrhs + q], s2);
          }
          double* y = yp + (long long)i * NOUT * nrhs + q;
          if (c == 0) {
#pragma unroll
            for (int r = 0; r < NOUT; ++r) y[r * nrhs] = 0.0;
          }
          y[rr * nrhs] += s1;
          if (two) y[cc * nrhs] += s2;
        }
      }
      __syncthreads();
    }
  }
}

// Transposed H-matvec (HMatrix::matvec_transposed, proj/src/hmatrix.cpp:
// 47-72) over the owned blocks: a CTA per block writes the partial rows of
// its COLUMN range, tpart[(tprow + j) * NOUT + r]; the per-column-leaf pass
// (hmv_reduce_kernel on the column tables) sums them in a fixed order.  In
// the 3x3 grid the cell (R, C) transposed maps x_R to y_C and, for R != C,
// its alias (C, R) maps x_C to y_R.  xr: x gathered to internal row order.
template <int NC>
__global__ void __launch_bounds__(256)
hmvt_blocks_kernel(const MvBlock* __restrict__ blocks, int nblocks,
                   const long long* __restrict__ tprow, const Item* __restrict__ items,
                   const double* __restrict__ arena, const double* __restrict__ dense,
                   const double* __restrict__ xr, double* __restrict__ tpart, int mode) {
  constexpr int NOUT = NC == 6 ? 3 : 1;
  extern __shared__ double zsm[];  // [2][kmax]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  for (int bi = blockIdx.x; bi < nblocks; bi += gridDim.x) {
    const MvBlock b = blocks[bi];
    double* out = tpart + tprow[bi] * NOUT;
    const double* xs = xr + (long long)b.row0 * NOUT;
    if (b.dense) {
      const long long cp = (b.m * NC + 1) & ~1;
      for (int j = threadIdx.x; j < b.n; j += blockDim.x) {
        double acc[NOUT];
#pragma unroll
        for (int r = 0; r < NOUT; ++r) acc[r] = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const int R = NC == 6 ? c_comp_r[c] : 0, C = NC == 6 ? c_comp_c[c] : 0;
          const double* D = dense + b.dense_off + j * cp + (long long)c * b.m;
          double s1 = 0.0, s2 = 0.0;
          for (int i = 0; i < b.m; ++i) {
            s1 = fma(D[i], xs[i * NOUT + R], s1);
            if (R != C) s2 = fma(D[i], xs[i * NOUT + C], s2);
          }
          acc[C] += s1;
          if (R != C) acc[R] += s2;
        }
#pragma unroll
        for (int r = 0; r < NOUT; ++r) out[(long long)j * NOUT + r] = acc[r];
      }
      __syncthreads();
      continue;
    }
    for (int c = 0; c < NC; ++c) {
      const Item it = items[b.item0 + c];
      const int k = mode ? it.k : it.kcur;
      const int R = NC == 6 ? c_comp_r[c] : 0, C = NC == 6 ? c_comp_c[c] : 0;
      const double* U = arena + it.u_off;
      const double* V = arena + it.v_off;
      // z_l = U(:,l) . x_R (and w_l = U(:,l) . x_C for the alias)
      for (int l = warp; l < k; l += nwarps) {
        double s1 = 0.0, s2 = 0.0;
        for (int i = lane; i < b.m; i += 32) {
          const double u = U[(long long)l * b.m + i];
          s1 = fma(u, xs[i * NOUT + R], s1);
          if (R != C) s2 = fma(u, xs[i * NOUT + C], s2);
        }
        s1 = warp_sum(s1);
        s2 = warp_sum(s2);
        if (lane == 0) {
          zsm[l] = s1;
          zsm[k + l] = s2;
        }
      }
      __syncthreads();
      for (int j = threadIdx.x; j < b.n; j += blockDim.x) {
        double s1 = 0.0, s2 = 0.0;
        for (int l = 0; l < k; ++l) {
          const double v = V[(long long)l * b.n + j];
          s1 = fma(v, zsm[l], s1);
          if (R != C) s2 = fma(v, zsm[k + l], s2);
        }
        double* o = out + (long long)j * NOUT;
        if (c == 0) {
#pragma unroll
          for (int r = 0; r < NOUT; ++r) o[r] = 0.0;
        }
        o[C] += s1;
        if (R != C) o[R] += s2;
      }
      __syncthreads();
    }
  }
}

// per leaf: y(p) = sum over covering blocks (fixed order) of the partials
template <int NOUT>
__global__ void hmv_reduce_kernel(const int* __restrict__ leaf_begin,
                                  const int* __restrict__ leaf_end,
                                  const int* __restrict__ leaf_ptr,
                                  const long long* __restrict__ leaf_prow,
                                  int nleaves, const double* __restrict__ ypart,
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
      for (int e = e0; e < e1; ++e)
        s += ypart[((leaf_prow[e] + i) * NOUT + r) * nrhs + q];
      y[q * ndof + (long long)r * nrows + rperm[b0 + i]] = s;
    }
  }
}

// ---------------------------------------------------------------------------
// look-ahead tail products for AMVM (apply_range(k_cur, k_look), aca.cpp:7-11
// as used by gamma_contributions, amvm.cpp:72-122): one warp per item
struct TailTerm {
  int item, nocc;
  long long off;
};

template <int NOUT>
__global__ void tail_kernel(const TailTerm* __restrict__ terms, int nterms,
                            const Item* __restrict__ items,
                            const double* __restrict__ arena,
                            const double* __restrict__ xi, double* __restrict__ out,
                            int is_grid) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = gw; t < nterms; t += nw) {
    const TailTerm tt = terms[t];
    const Item it = items[tt.item];
    const int rr = is_grid ? c_comp_r[it.comp] : 0;
    const int cc = is_grid ? c_comp_c[it.comp] : 0;
    const double* U = arena + it.u_off;
    const double* V = arena + it.v_off;
    double* o = out + tt.off;
    for (int i = lane; i < tt.nocc * it.m; i += 32) o[i] = 0.0;
    __syncwarp();
    for (int l = it.kcur; l < it.k; ++l) {
      double s1 = 0.0, s2 = 0.0;
      for (int j = lane; j < it.n; j += 32) {
        const double v = V[(long long)l * it.n + j];
        const double* xj = xi + (long long)(it.col0 + j) * NOUT;
        s1 = fma(v, xj[cc], s1);
        if (tt.nocc == 2) s2 = fma(v, xj[rr], s2);
      }
      s1 = warp_sum(s1);
      s2 = warp_sum(s2);
      for (int i = lane; i < it.m; i += 32) {
        const double u = U[(long long)l * it.m + i];
        o[i] = fma(u, s1, o[i]);
        if (tt.nocc == 2) o[it.m + i] = fma(u, s2, o[it.m + i]);
      }
    }
  }
}

// transposed tails V[:,k:K](U[:,k:K]^T x) over the block columns (the
// transposed occurrences of gamma_contributions, amvm.cpp:100-106): in the
// grid the cell (R, C) maps x_R to columns of component C and its alias
// (C, R) maps x_C to component R.  xr: x gathered to internal row order.
template <int NOUT>
__global__ void tail_t_kernel(const TailTerm* __restrict__ terms, int nterms,
                              const Item* __restrict__ items,
                              const double* __restrict__ arena,
                              const double* __restrict__ xr, double* __restrict__ out,
                              int is_grid) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = gw; t < nterms; t += nw) {
    const TailTerm tt = terms[t];
    const Item it = items[tt.item];
    const int rr = is_grid ? c_comp_r[it.comp] : 0;
    const int cc = is_grid ? c_comp_c[it.comp] : 0;
    const double* U = arena + it.u_off;
    const double* V = arena + it.v_off;
    double* o = out + tt.off;
    for (int j = lane; j < tt.nocc * it.n; j += 32) o[j] = 0.0;
    __syncwarp();
    for (int l = it.kcur; l < it.k; ++l) {
      double s1 = 0.0, s2 = 0.0;
      for (int i = lane; i < it.m; i += 32) {
        const double u = U[(long long)l * it.m + i];
        const double* xi = xr + (long long)(it.row0 + i) * NOUT;
        s1 = fma(u, xi[rr], s1);
        if (tt.nocc == 2) s2 = fma(u, xi[cc], s2);
      }
      s1 = warp_sum(s1);
      s2 = warp_sum(s2);
      for (int j = lane; j < it.n; j += 32) {
        const double v = V[(long long)l * it.n + j];
        o[j] = fma(v, s1, o[j]);
        if (tt.nocc == 2) o[it.n + j] = fma(v, s2, o[it.n + j]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// DFMA throughput probe (roofline denominator for the fp64 kernels): 8
// independent FMA chains per thread, the result kept live.
__global__ void __launch_bounds__(256) dfma_peak_kernel(double* out, int iters, double a,
                                                        double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;  // practically never; keeps the chains live
}

// ---------------------------------------------------------------------------
// a subset of the item table (partial host-mirror refresh)
__global__ void gather_items_kernel(const Item* __restrict__ items, const int* __restrict__ ids,
                                    int n, Item* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) out[t] = items[ids[t]];
}

// ---------------------------------------------------------------------------
// small state kernels
__global__ void promote_kernel(Item* items, const int* idx, int n) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) items[idx[t]].kcur = items[idx[t]].k;
}

__global__ void prep_extend_kernel(Item* items, const int* idx, int n, int steps) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) {
    Item& it = items[idx[t]];
    it.phase = PH_EXT;
    it.steps_left = steps;
  }
}

// compaction: per item the packed size of U and V with cap = max(min(capr,
// k + slack), k) columns, and its pivot slots
__global__ void compact_sizes_kernel(const Item* __restrict__ items, int n,
                                     long long max_rank, int slack,
                                     long long* __restrict__ usz, long long* __restrict__ psz,
                                     int* __restrict__ caps) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const Item it = items[t];
  const long long capr = min(max_rank, (long long)min(it.m, it.n));
  const int cap = max((int)min(capr, (long long)it.k + slack), it.k);
  caps[t] = cap;
  usz[t] = (((long long)it.m * cap + 1) & ~1LL) + (((long long)it.n * cap + 1) & ~1LL);
  psz[t] = max(cap, 1);
}

// copies every item's U (m x K), V (n x K) and pivots to the scanned offsets
__global__ void compact_kernel(Item* __restrict__ items, int n,
                               const long long* __restrict__ uoff,
                               const long long* __restrict__ poff,
                               const int* __restrict__ caps,
                               const double* __restrict__ src, double* __restrict__ dst,
                               const int2* __restrict__ spiv, int2* __restrict__ dpiv) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = gw; t < n; t += nw) {
    Item it = items[t];
    const long long nu = (long long)it.m * it.k, nv = (long long)it.n * it.k;
    const long long u0 = uoff[t];
    const long long v0 = u0 + (((long long)it.m * caps[t] + 1) & ~1LL);
    const double* su = src + it.u_off;
    const double* sv = src + it.v_off;
    // every U / V region starts 16-byte aligned (align2 offsets): copy
    // double2 pairs, then the odd tail element
    auto copy2 = [&](double* d, const double* s_, long long len) {
      const double2* s2 = reinterpret_cast<const double2*>(s_);
      double2* d2 = reinterpret_cast<double2*>(d);
      // four 16-byte loads in flight per lane before their stores
      const long long h = len / 2;
      long long e = lane;
      for (; e + 96 < h; e += 128) {
        const double2 a = s2[e], b = s2[e + 32], c = s2[e + 64], f = s2[e + 96];
        d2[e] = a;
        d2[e + 32] = b;
        d2[e + 64] = c;
        d2[e + 96] = f;
      }
      for (; e < h; e += 32) d2[e] = s2[e];
      if ((len & 1) && lane == 0) d[len - 1] = s_[len - 1];
    };
    copy2(dst + u0, su, nu);
    copy2(dst + v0, sv, nv);
    for (int e = lane; e < it.k; e += 32) dpiv[poff[t] + e] = spiv[it.p_off + e];
    __syncwarp();
    if (lane == 0) {
      it.u_off = u0;
      it.v_off = v0;
      it.p_off = poff[t];
      it.cap = caps[t];
      items[t] = it;
    }
  }
}

// relocate item factors into new storage: copies U (m x K), V (n x K) prefix
// columns and K pivots to the offsets in `dst` (same item order)
__global__ void relocate_kernel(Item* __restrict__ items, const int* __restrict__ idx,
                                const long long* __restrict__ new_u,
                                const long long* __restrict__ new_v,
                                const long long* __restrict__ new_p,
                                const int* __restrict__ new_cap, int n,
                                const double* __restrict__ src_arena,
                                double* __restrict__ dst_arena,
                                const int2* __restrict__ src_piv,
                                int2* __restrict__ dst_piv) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = gw; t < n; t += nw) {
    Item it = items[idx[t]];
    const long long nu = (long long)it.m * it.k, nv = (long long)it.n * it.k;
    const double* su = src_arena + it.u_off;
    const double* sv = src_arena + it.v_off;
    double* du = dst_arena + new_u[t];
    double* dv = dst_arena + new_v[t];
    for (long long e = lane; e < nu; e += 32) du[e] = su[e];
    for (long long e = lane; e < nv; e += 32) dv[e] = sv[e];
    for (int e = lane; e < it.k; e += 32) dst_piv[new_p[t] + e] = src_piv[it.p_off + e];
    __syncwarp();
    if (lane == 0) {
      it.u_off = new_u[t];
      it.v_off = new_v[t];
      it.p_off = new_p[t];
      it.cap = new_cap[t];
      items[idx[t]] = it;
    }
  }
}

}  // namespace hmgpu
