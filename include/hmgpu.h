/*
 * hmgpu.h -- C ABI of the B200 hot path of the adaptive H-matrix BEM
 * (ACA assembly of Kelvin collocation blocks, near-field fill, H-matvec,
 * look-ahead tail terms for the adaptive matvec).
 *
 * This is the drop-in boundary under the reference's L4 "low-rank core"
 * (SURVEY.md section 8b).  Each entry point replaces one reference interface:
 *
 *   hmgpu_set_kelvin_geometry  CollocSingleOracle / GalerkinKernels::
 *                              colloc_single + point_order + kelvin_tensor
 *                              (proj/include/hmbem/kernels.hpp:107-126,
 *                               proj/src/kernels.cpp:21-28,87-93,176-187),
 *                              fused into the kernels instead of a callback
 *   hmgpu_set_kdouble_geometry CollocDoubleOracle (colloc_double + kelvin_traction,
 *                              proj/src/kernels.cpp:30-55,189-210), points x nodes
 *   hmgpu_set_eval_points      CollocSingleOracle at evaluate_interior's points
 *                              (proj/src/baca.cpp:645-687)
 *   hmgpu_set_rule             gauss_rule(order) tables (proj/src/quadrature.cpp:55-95)
 *   hmgpu_set_galerkin_geometry  KernelOracle over V_Delta / V_kl: GalerkinKernels::
 *                              vdelta / vkl / integrate_pair / disjoint_order
 *                              (proj/include/hmbem/kernels.hpp:95-105,
 *                               proj/src/kernels.cpp:75-149), fused into the kernels
 *   hmgpu_set_kdelta_geometry  KernelOracle over K_Delta: GalerkinKernels::kdelta
 *                              (proj/src/kernels.cpp:151-167), triangles x nodes
 *   hmgpu_ell3_spmv(_t)        SpMat products of the operator algebra (T12/T13/T23,
 *                              mass; build_sparse_ops, proj/src/operators.cpp:7-95)
 *   hmgpu_set_pair_rule        pair_rule(PairCase, order) Sauter-Schwab tables
 *                              (proj/src/quadrature.cpp:290-338)
 *   hmgpu_set_points           test fixtures CentroidKernelOracle / PointKernelOracle
 *                              (proj/tests/test_hmatrix.cpp:12-28, test_amvm.cpp:9-22)
 *   hmgpu_set_dense_matrix     DenseOracle (proj/include/hmbem/aca.hpp:34-44)
 *   hmgpu_set_partition        BlockPartition / ClusterTree handed to assemble()
 *                              (proj/include/hmbem/cluster.hpp:35-89, hmatrix.hpp:88-90)
 *   hmgpu_assemble             assemble() -> aca_run / aca_extend / dense fill
 *                              (proj/src/hmatrix.cpp:147-186, proj/src/aca.cpp:41-143)
 *   hmgpu_ranks                HBlock::current_rank / factor.rank() (hmatrix.hpp:31-39)
 *   hmgpu_matvec               HMatrix::matvec (hmatrix.cpp:22-45) composed by the
 *                              BlockGrid matvec (proj/src/expr.cpp:197-215)
 *   hmgpu_matvec_transposed    HMatrix::matvec_transposed (hmatrix.cpp:47-72)
 *   hmgpu_promote              HMatrix::promote (hmatrix.cpp:95-97)
 *   hmgpu_extend               HMatrix::extend_lookahead (hmatrix.cpp:104-111)
 *   hmgpu_tail_terms           the apply_range(k_cur, k_look) products of
 *                              gamma_contributions (proj/src/amvm.cpp:72-122)
 *   hmgpu_download_factor      LowRankFactor state (aca.hpp:76-94), parity dumps
 *   hmgpu_storage              storage_mb_current / storage_mb_tail (hmatrix.cpp:113-138)
 *
 * Conventions: plain pointers and sizes only; no exceptions cross the ABI.
 * Every call returns an int status (HMGPU_OK = 0); hmgpu_last_error(ctx)
 * returns a message for the last failure.  Reference errors map as:
 * DimensionError -> HMGPU_ERR_DIMENSION, Error (eps/beta range, state)
 * -> HMGPU_ERR_INVALID / HMGPU_ERR_STATE.
 * Threading: one ctx per device, not re-entrant; all work is issued on the
 * ctx's own CUDA stream (hmgpu_get_stream).  Host arrays are borrowed for
 * the duration of a call.  Index spaces: "external" ids are the reference's
 * DOF ids; "internal" positions are cluster-tree permuted positions
 * (perm[internal] = external, cluster.hpp:51-52).
 */
#ifndef HMGPU_H
#define HMGPU_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hmgpu_ctx hmgpu_ctx;

enum {
  HMGPU_OK = 0,
  HMGPU_ERR_INVALID = 1,   /* bad argument (reference: hmbem::Error) */
  HMGPU_ERR_OOM = 2,       /* device allocation failed */
  HMGPU_ERR_CUDA = 3,      /* CUDA runtime / launch error */
  HMGPU_ERR_NODEVICE = 4,  /* no CUDA device visible */
  HMGPU_ERR_STATE = 5,     /* call out of order (e.g. matvec before assemble) */
  HMGPU_ERR_DIMENSION = 6, /* size mismatch (reference: DimensionError) */
  HMGPU_ERR_COMM = 7       /* NCCL / transport failure (multi-GPU) */
};

enum {
  HMGPU_KERNEL_KELVIN = 0, /* 6-component Kelvin collocation (3x3 grid) */
  HMGPU_KERNEL_NEWTON = 1, /* scalar 1/|x-y| over points, bounded diagonal */
  HMGPU_KERNEL_DENSE = 2   /* scalar entries of an explicit matrix */
};

enum { HMGPU_MODE_CURRENT = 0, HMGPU_MODE_LOOKAHEAD = 1 };
enum { HMGPU_PTR_HOST = 0, HMGPU_PTR_DEVICE = 1 };

/* ACA stop reasons, as AcaStop (proj/include/hmbem/aca.hpp:66-72) */
enum {
  HMGPU_STOP_NONE = 0,
  HMGPU_STOP_INEQUALITY = 1,
  HMGPU_STOP_EXHAUSTED = 2,
  HMGPU_STOP_RANKCAP = 3,
  HMGPU_STOP_STEPSDONE = 4
};

typedef struct hmgpu_assembly_stats {
  long long aca_entries;      /* kernel entries evaluated by ACA (rows+cols) */
  long long dense_entries;    /* near-field component entries */
  long long aca_steps;        /* accepted + rejected cross attempts */
  long long pivots;           /* sum of look-ahead ranks */
  double ms_total;            /* device time of the whole assembly */
  double ms_nearfield;        /* device time of the near-field fill */
  double ms_aca;              /* device time of the ACA launches */
  int aca_relaunches;         /* capacity regrow passes */
  double counted_flops;       /* Kelvin only: sum of 30 n_q + 1 per component entry
                                 (SURVEY.md 8d convention, n_q = rule points) */
} hmgpu_assembly_stats;

typedef struct hmgpu_storage_info {
  double mb_current;          /* U,V of the current factors + dense (MB, 2^20) */
  double mb_tail;             /* look-ahead tails */
  double mb_dense;            /* dense near-field part */
  double mb_arena_allocated;  /* device bytes reserved for U,V */
  long long matvec_bytes;     /* algorithmic bytes of one MODE_CURRENT matvec, nrhs=1 */
  long long matvec_flops;     /* flops of one MODE_CURRENT matvec, nrhs=1 */
  long long pivots;           /* sum of the look-ahead ranks k over the low-rank
                               * (component, block) items: the reference's
                               * cumulative pivot count (HMatrix::total_pivots) */
} hmgpu_storage_info;

int hmgpu_device_count(int* n);
int hmgpu_create(int device, hmgpu_ctx** out);
int hmgpu_destroy(hmgpu_ctx* ctx);
const char* hmgpu_last_error(const hmgpu_ctx* ctx);
int hmgpu_get_stream(hmgpu_ctx* ctx, void** cuda_stream);

/* quadrature tier t (0: far, order-2 rule; 1: mid, order-4; 2: near, order-5)
 * with reference coordinates (a,b) and weights summing to 1/2.  far_ratio /
 * mid_ratio are QuadratureConfig::far_ratio / mid_ratio (kernels.hpp:44-52). */
int hmgpu_set_rule(hmgpu_ctx* ctx, int tier, int npts, const double* a,
                   const double* b, const double* w);
int hmgpu_set_tier_ratios(hmgpu_ctx* ctx, double far_ratio, double mid_ratio);

/* Kelvin collocation at triangle centroids, external triangle order.
 * verts: n_vert x 3, tris: n_tri x 3, centroid/area/diam as load_mesh
 * computes them (mesh.cpp:235-244, 105-109); material E, nu. */
int hmgpu_set_kelvin_geometry(hmgpu_ctx* ctx, int n_vert, const double* verts,
                              int n_tri, const int* tris,
                              const double* centroid, const double* area,
                              const double* diam, double E, double nu);
/* Galerkin scalar kernels on the triangle x triangle partition of
 * assemble_operators (operators.cpp:186-200): which = 0 -> the six V_kl as
 * the symmetric 3x3 grid (components (k,l) = 00 01 02 11 12 22; V_lk
 * aliases V_kl, operators.cpp:226-233), which = 1 -> V_Delta (one
 * component).  Arrays as hmgpu_set_kelvin_geometry.  Disjoint pairs use the
 * rule tiers of hmgpu_set_rule (0: order 2, 1: order 4, 2: order 5); touching
 * pairs the tables of hmgpu_set_pair_rule. */
int hmgpu_set_galerkin_geometry(hmgpu_ctx* ctx, int n_vert, const double* verts,
                                int n_tri, const int* tris, const double* centroid,
                                const double* area, const double* diam, int which);
/* K_Delta (kernels.cpp:151-167): triangles x vertices on the triangle x
 * node partition (node boxes = union of the incident triangles' boxes,
 * operators.cpp:190-200); normals n_tri x 3 as load_mesh computes them.
 * Uses the rule tiers and pair rules like hmgpu_set_galerkin_geometry. */
int hmgpu_set_kdelta_geometry(hmgpu_ctx* ctx, int n_vert, const double* verts, int n_tri,
                              const int* tris, const double* centroid, const double* area,
                              const double* diam, const double* normals);
/* singular pair rule of PairCase pair_case (1 vertex, 2 edge, 3 identical):
 * n points, reference coordinates on the rotated test (xr) and trial (yr)
 * triangles and weights (PairRule, quadrature.hpp:44-52) */
int hmgpu_set_pair_rule(hmgpu_ctx* ctx, int pair_case, int n, const double* xr1,
                        const double* xr2, const double* yr1, const double* yr2,
                        const double* w);
/* Sparse transforms of the operator algebra (build_sparse_ops,
 * operators.cpp:7-95) on the ctx's stream, DEVICE
 * pointers: an ELL matrix with 3 slots per row (col3 / val3, rows x 3).
 *   hmgpu_ell3_spmv:   y = alpha A x + beta y            (y: rows)
 *   hmgpu_ell3_spmv_t: y = alpha A^T x + beta y          (y: cols), gathered
 *                      per column over the inverse index tptr (cols + 1) /
 *                      tslot (flat slot ids 3 r + a, ascending rows)
 * beta == 0 does not read y. */
int hmgpu_ell3_spmv(hmgpu_ctx* ctx, int rows, const int* col3, const double* val3,
                    const double* x, double* y, double alpha, double beta);
int hmgpu_ell3_spmv_t(hmgpu_ctx* ctx, int cols, const int* tptr, const int* tslot,
                      const double* val3, const double* x, double* y, double alpha,
                      double beta);
/* One cell (r, c) of evaluate_interior's double-layer grid W~
 * (CollocDoubleOracle / colloc_double, kernels.cpp:189-210, with
 * kelvin_traction, kernels.cpp:30-55): rows = the evaluation points of
 * hmgpu_set_eval_points, columns = the vertices (node patches); arrays as
 * hmgpu_set_kdelta_geometry; rule tiers as the single layer. */
int hmgpu_set_kdouble_geometry(hmgpu_ctx* ctx, int n_vert, const double* verts, int n_tri,
                               const int* tris, const double* centroid, const double* area,
                               const double* diam, const double* normals, double E,
                               double nu, int r, int c);
/* Kelvin context only: collocation at n arbitrary evaluation points (the
 * rows; CollocSingleOracle with evaluate_interior's points, kernels.hpp:
 * 107-126, baca.cpp:645-687) instead of the triangle centroids; n = 0
 * restores the centroids.  The partition's rows are then the points. */
int hmgpu_set_eval_points(hmgpu_ctx* ctx, int n, const double* pts);
/* scalar Newton kernel 1/|x_i - x_j| with entry `diag` where x_i == x_j */
int hmgpu_set_points(hmgpu_ctx* ctx, int n, const double* pts, double diag);
/* scalar explicit matrix, column-major m x n, external ids */
int hmgpu_set_dense_matrix(hmgpu_ctx* ctx, int m, int n, const double* a);

/* Cluster trees (nodes as rows [begin, end, child0, child1]) with their
 * permutations, and the block partition (rows [row_node, col_node,
 * admissible, level]).  The ctx owns the blocks whose row node lies inside
 * the internal row range [row_begin, row_end) -- the block-row shard of
 * this device (pass 0, n_rows for a single device). */
int hmgpu_set_partition(hmgpu_ctx* ctx, int n_rows, const int* row_perm,
                        int n_row_nodes, const int* row_nodes4, int n_cols,
                        const int* col_perm, int n_col_nodes,
                        const int* col_nodes4, int n_blocks,
                        const int* blocks4, int row_begin, int row_end);

/* assemble(): full mode (initial_rank < 0: ACA to the stopping rule at eps
 * with beta_stop) or coarse mode (initial_rank pivots), then `lookahead`
 * further pivots; dense fill of non-admissible blocks.  stats may be NULL. */
int hmgpu_assemble(hmgpu_ctx* ctx, double eps, double beta_stop,
                   int initial_rank, int lookahead, long long max_rank,
                   hmgpu_assembly_stats* stats);

/* per (component, block): current and look-ahead rank (-1 = dense or not
 * owned), consumed rows, last stop rule; arrays of ncomp * n_blocks,
 * component-major.  Any pointer may be NULL. */
int hmgpu_ranks(hmgpu_ctx* ctx, int* k_cur, int* k_look, int* consumed,
                int* last_stop);

/* y = A x over the owned block rows (other rows of y are written 0).
 * x, y: dofs x nrhs column-major in external component-major order
 * (dofs = 3 * n for Kelvin, n otherwise).  ptr_kind: host or device
 * pointers; host calls stage through pinned buffers. */
int hmgpu_matvec(hmgpu_ctx* ctx, const double* x, double* y, int nrhs,
                 int mode, int ptr_kind);
/* y = A^T x (HMatrix::matvec_transposed, proj/src/hmatrix.cpp:47-72; in the
 * 3x3 grid the transpose of every cell): x over the rows (n_rows * 3 or
 * n_rows dofs per RHS), y over the columns; nrhs columns back to back;
 * deterministic (partial rows per block column range, fixed-order
 * reduction per column leaf).  Block-row shards give partial products. */
int hmgpu_matvec_transposed(hmgpu_ctx* ctx, const double* x, double* y, int nrhs,
                            int mode, int ptr_kind);

/* promote / extend work items given as (component, block) pairs */
int hmgpu_promote(hmgpu_ctx* ctx, int n, const int* comp_block);
int hmgpu_extend(hmgpu_ctx* ctx, int n, const int* comp_block, int steps);

/* Look-ahead tail products for every owned (component, block) with
 * k_look > k_cur: for occurrence o of the block in the operator (1 for
 * scalar kernels and diagonal Kelvin components, 2 for off-diagonal ones:
 * o = 0 is cell (r,c) applied to x_c, o = 1 is cell (c,r) applied to x_r),
 * vals[off + o*m + i] = (U[:,kc:kl] V[:,kc:kl]^T x_seg)[i], i over the block
 * rows in internal order.  Two-call protocol: with meta == NULL returns the
 * number of terms and total values; then fills meta rows
 * [comp, block, n_occ, off] and vals.  x is a host pointer. */
/* Device-resident estimator of the adaptive matvec (Algorithm 2; replaces
   gamma_contributions + mark_blocks, amvm.cpp:46-184, and the promote /
   extend_lookahead calls of amvm_multiply, amvm.cpp:255-266):
   hmgpu_amvm_estimate   tail terms, difference (optional host copy, rows in
                         external component-major order) and gamma = ||difference||
   hmgpu_amvm_mark       theta-marking walk on the device; gamma(P_k), count
   hmgpu_amvm_refine     promote + extend_lookahead(steps) of the marked
                         (comp, block) pairs (optional host copy of the pairs)
   Whole (unsharded) operators only; a block-row shard with a communicator
   runs the adaptive loop through the term-level API (hmb_amvm, operator.cpp
   amvm_multiply_sharded). */
int hmgpu_amvm_estimate(hmgpu_ctx* ctx, const double* x, double* gamma, double* difference);
/* direct = 1: 1-RHS matvecs sweep the blocks in place instead of building the
   packed stream plan (for one matvec per rank change, as in the adaptive loop;
   the plan pays off from the second matvec on the same ranks); 2: automatic --
   the first 1-RHS product after a rank change (assembly, promote, extend) runs
   in place and the plan is built when a second one follows (the two differ
   in the order of their sums, ~1e-16 relative); 0 (default): always the plan */
int hmgpu_set_matvec_policy(hmgpu_ctx* ctx, int direct);
int hmgpu_get_matvec_policy(hmgpu_ctx* ctx, int* direct);
int hmgpu_amvm_mark(hmgpu_ctx* ctx, double theta, int c_sp, long long m_rows,
                    long long n_cols, double* gamma_pk, int* n_marked);
int hmgpu_amvm_refine(hmgpu_ctx* ctx, int steps, int* comp_block);

int hmgpu_tail_terms(hmgpu_ctx* ctx, const double* x, int* n_terms,
                     long long* n_vals, long long* meta4, double* vals);
/* the transposed tails V[:,k:K](U[:,k:K]^T x) of the transposed occurrences
 * (gamma_contributions, amvm.cpp:100-106): x over the rows, per term nocc x n
 * values over the block columns (internal order); grid occurrence 0 is the
 * cell (R, C) (x_R -> component C), occurrence 1 its alias (x_C -> R) */
int hmgpu_tail_terms_t(hmgpu_ctx* ctx, const double* x, int* n_terms,
                       long long* n_vals, long long* meta4, double* vals);

/* factor of (comp, block): U (m x K) and V (n x K) column-major, pivots
 * (K x 2, local), frob_sq; with U == NULL only the sizes are returned */
int hmgpu_download_factor(hmgpu_ctx* ctx, int comp, int block, int* m, int* n,
                          int* K, int* k_cur, double* U, double* V, int* piv,
                          double* frob_sq);
/* dense payload of a non-admissible block for one component, m x n
 * column-major (rows/cols in internal order) */
int hmgpu_download_dense(hmgpu_ctx* ctx, int comp, int block, double* out);

int hmgpu_storage(hmgpu_ctx* ctx, hmgpu_storage_info* info);

/* ---- multi-GPU block-row sharding --------------------
 * One ctx per rank and device, each created with its shard's row range
 * (hmgpu_set_partition row_begin / row_end; the ranges of all ranks must
 * tile [0, n_rows) in rank order).  A communicator attached to the ctx makes
 * hmgpu_matvec_dist the whole sharded product: x is broadcast from rank 0,
 * every rank sweeps the blocks of its rows and writes its rows in internal
 * order into a segment buffer, the segments (padded to the longest shard)
 * are all-gathered, and every rank un-permutes the full y.  The reference
 * runs the same product on one process (HMatrix::matvec, hmatrix.cpp:22-45,
 * over the blocks assembled in parallel, hmatrix.cpp:147-186).
 *
 * Transports: NCCL (the library's own communicator from a unique id, or a
 * caller's ncclComm_t borrowed), loaded at run time from libnccl.so.2 (the
 * copy already in the process if there is one); or host callbacks on HOST
 * buffers (any other transport, e.g. a test harness), which the library
 * stages through pinned memory.  All collective calls of one product are
 * issued on the ctx's stream; every rank must call hmgpu_matvec_dist with
 * the same nrhs and mode. */
typedef struct hmgpu_comm_ops {
  /* in-place broadcast of `bytes` from rank `root`; returns 0 on success */
  int (*broadcast)(void* user, void* buf, long long bytes, int root);
  /* recv[r * bytes_per_rank ...] = send of rank r, for every rank r */
  int (*allgather)(void* user, const void* send, void* recv, long long bytes_per_rank);
  void* user;
} hmgpu_comm_ops;

/* 1 if libnccl.so.2 can be loaded (NCCL version in *version), else 0 */
int hmgpu_nccl_available(int* available, int* version);
/* ncclGetUniqueId: 128 bytes that rank 0 hands to every rank out of band */
int hmgpu_nccl_unique_id(void* id128);
/* create the ctx's own NCCL communicator (ncclCommInitRank; collective) */
int hmgpu_comm_init_nccl(hmgpu_ctx* ctx, int nranks, int rank, const void* id128);
/* borrow an existing ncclComm_t (not destroyed by the library) */
int hmgpu_comm_set_nccl(hmgpu_ctx* ctx, void* nccl_comm, int nranks, int rank);
/* host-callback transport (ops copied; ops->user must outlive the ctx) */
int hmgpu_comm_set_ops(hmgpu_ctx* ctx, int nranks, int rank, const hmgpu_comm_ops* ops);
int hmgpu_comm_clear(hmgpu_ctx* ctx);
/* kind: 0 none, 1 NCCL (own), 2 NCCL (borrowed), 3 host callbacks; row
 * ranges of all ranks (row_begin[nranks], row_end[nranks], may be NULL) */
int hmgpu_comm_info(hmgpu_ctx* ctx, int* nranks, int* rank, int* kind, int* row_begin,
                    int* row_end);
/* all-gather of HOST buffers over the ctx's communicator (collective):
 * recv[r * bytes_per_rank ...] = send of rank r (the sharded adaptive
 * matvec exchanges its estimator and marking events with it) */
int hmgpu_comm_allgather(hmgpu_ctx* ctx, const void* send, void* recv,
                         long long bytes_per_rank);
/* y = A x on all ranks (see above).  x is read on rank 0 only (other ranks
 * may pass NULL); y (dofs x nrhs, column-major, external order) is written
 * on every rank.  ptr_kind as hmgpu_matvec. */
int hmgpu_matvec_dist(hmgpu_ctx* ctx, const double* x, double* y, int nrhs, int mode,
                      int ptr_kind);

/* measured DFMA throughput of the device (TFLOP/s, 2 flops per FMA): the
 * fp64 roofline denominator of the assembly kernels */
int hmgpu_fp64_peak(int device, double* tflops);
/* measured fp64 tensor-core (DMMA m8n8k4) throughput of `device` in TFLOP/s:
   the peak the multi-RHS sweep is reported against */
int hmgpu_dmma_peak(int device, double* tflops);
/* the same chains launched back to back for `seconds` (0.2 .. 10): the mean
   rate over the second half of the run, i.e. at the clocks the power limit
   settles on under a long fp64 tensor load (burst: hmgpu_dmma_peak) */
int hmgpu_dmma_peak_sustained(int device, double seconds, double* tflops);

/* CUDA-event timing of every kernel launch (off by default).  names are
 * "gather", "nearfield", "aca", "hmv_blocks", "hmv_reduce", "tail", ...
 * hmgpu_kernel_times returns accumulated milliseconds and launch counts for
 * the kernel name and resets them when reset != 0. */
int hmgpu_set_profiling(hmgpu_ctx* ctx, int on);
int hmgpu_kernel_times(hmgpu_ctx* ctx, const char* name, double* ms,
                       long long* launches, int reset);

#ifdef __cplusplus
}
#endif

#endif /* HMGPU_H */
