/*
 * hmbem.h -- flat C API of the host layer (libhmbem.so): meshes, cluster
 * tree / block partition, the GPU-backed H-operator and the adaptive
 * matvec.  It is the binding surface of the Python package
 * paper_2205_04752_b200 (ctypes) and mirrors the reference's operator API:
 *
 *   hmb_mesh_*          SurfaceMesh / load_mesh / meshgen  (mesh.hpp:15-78,
 *                       proj/tools/meshgen.cpp:27-83)
 *   hmb_op_kelvin       evaluate_interior's 3x3 grid of CollocSingleOracle
 *                       H-matrices at triangle centroids (baca.cpp:645-687)
 *   hmb_op_galerkin     GalerkinKernels V_kl grid / V_Delta KernelOracle
 *                       H-matrices (kernels.cpp:95-149, operators.cpp:218-235)
 *   hmb_op_kdelta       K_Delta KernelOracle H-matrix, triangles x nodes
 *   hmb_op_newton/dense test fixtures (test_hmatrix.cpp:12-53, aca.hpp:34-44)
 *   hmb_tree_*, hmb_partition_*   ClusterTree / BlockPartition /
 *                       sparsity_constant / partition_to_json (cluster.hpp)
 *   hmb_assemble        assemble()                 (hmatrix.hpp:88-90)
 *   hmb_matvec          matvec(BlockGrid, x, Mode)  (expr.cpp:197-215)
 *   hmb_promote/extend  HMatrix::promote / extend_lookahead
 *   hmb_gamma/hmb_mark  gamma_contributions / mark_blocks (amvm.hpp:36-48)
 *   hmb_amvm            amvm_multiply               (amvm.hpp:67-71); on a block-row
 *                       shard with a communicator: the sharded loop
 *   hmb_mark_sharded    mark_blocks across block-row shards (amvm.cpp:131-184)
 *
 * Status convention: 0 = ok, otherwise an hmbem error class
 * (1 Error, 2 MeshError, 3 ConfigError, 4 DimensionError, 5 DeviceError);
 * hmb_last_error() returns the message (thread-local).
 */
#ifndef HMBEM_H
#define HMBEM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hmb_mesh hmb_mesh;
typedef struct hmb_op hmb_op;

enum {
  HMB_OK = 0,
  HMB_ERROR = 1,
  HMB_MESH_ERROR = 2,
  HMB_CONFIG_ERROR = 3,
  HMB_DIMENSION_ERROR = 4,
  HMB_DEVICE_ERROR = 5
};

const char* hmb_last_error(void);
int hmb_device_status(void); /* last DeviceError's hmgpu status */

/* ---- meshes ---- */
int hmb_mesh_icosphere(int level, hmb_mesh** out);
int hmb_mesh_ellipsoid(int level, double ax, double ay, double az, hmb_mesh** out);
int hmb_mesh_voxel_cube(int n, double lo, double hi, hmb_mesh** out);
int hmb_mesh_from_arrays(int nv, const double* verts, int nt, const int* tris,
                         hmb_mesh** out);
int hmb_mesh_load_off(const char* path, hmb_mesh** out);
int hmb_mesh_save_off(const hmb_mesh* m, const char* path);
int hmb_mesh_validate(const hmb_mesh* m);
int hmb_mesh_label(hmb_mesh* m, const char* dirichlet_predicate);
int hmb_mesh_sizes(const hmb_mesh* m, int* nv, int* nt);
/* any output may be NULL; dirichlet as 0/1 per triangle (0s if unlabeled) */
int hmb_mesh_get(const hmb_mesh* m, double* verts, int* tris, double* centroids,
                 double* areas, double* normals, double* diam, int* dirichlet);
void hmb_mesh_free(hmb_mesh* m);

/* the touching-pair (Sauter-Schwab) rule uploaded to the device:
 * pair_case 1 vertex, 2 edge, 3 identical; order = points per dimension
 * (quadrature.cpp:168-338); NULL arrays query n */
int hmb_pair_rule(int pair_case, int order, int* n, double* xr1, double* xr2, double* yr1,
                  double* yr2, double* w);
/* sparse transforms of build_sparse_ops (operators.cpp:7-95) in ELL form:
 * n_tri rows x 3 slots (slot a = local vertex a, value 0 where the reference
 * drops the entry).  which: 0 T12, 1 T13, 2 T23, 3 mass (area / 3). */
int hmb_sparse_op(const hmb_mesh* m, int which, int* cols3, double* vals3);

/* seeded synthetic input: kind 0 = uniform [-1,1) (mt19937_64, the
 * reference's random_vector, oracles.cpp:415-421), 1 = standard normal */
int hmb_random_vector(long long n, unsigned long long seed, int kind, double* out);

/* gauss_rule(order) tables as uploaded to the device (quadrature.cpp:55-95);
 * a/b/w may be NULL to query npts */
int hmb_gauss_rule(int order, int* npts, double* a, double* b, double* w);

/* admissibility of boxes [lo(3), hi(3)]: min diam < eta * dist (cluster.cpp:21-24) */
int hmb_admissible(const double* box_a6, const double* box_b6, double eta, int* out);

/* ---- operators (device < 0: host-only, tree and partition) ---- */
int hmb_op_kelvin(const hmb_mesh* m, double E, double nu, int b_min, double eta,
                  int device, int shard_rank, int shard_count, hmb_op** out);
/* the single-layer grid of evaluate_interior (baca.cpp:625-687): Kelvin
 * collocation at npts points (rows, a tree over the point boxes) against the
 * triangles (columns); points within min_distance_factor x the largest
 * triangle diameter of the surface are rejected (baca.cpp:632-643) */
int hmb_op_kelvin_points(const hmb_mesh* m, int npts, const double* pts, double E,
                         double nu, int b_min, double eta, double min_distance_factor,
                         int disjoint_order, int device, int shard_rank, int shard_count,
                         hmb_op** out);
/* one cell (r, c) of evaluate_interior's double-layer grid W~
 * (CollocDoubleOracle, kernels.cpp:189-210): points x vertices, partition
 * point tree x node tree (baca.cpp:650-651) */
int hmb_op_kelvin_double(const hmb_mesh* m, int npts, const double* pts, int r, int c,
                         double E, double nu, int b_min, double eta,
                         double min_distance_factor, int disjoint_order, int device,
                         int shard_rank, int shard_count, hmb_op** out);
/* Galerkin scalar kernels on the triangle partition (assemble_operators,
 * operators.cpp:186-235): which = 0 -> the six V_kl as the 3x3 grid,
 * 1 -> V_Delta (kernels.cpp:130-149) */
int hmb_op_galerkin(const hmb_mesh* m, int which, int b_min, double eta, int device,
                    int shard_rank, int shard_count, hmb_op** out);
/* K_Delta on the triangle x node partition (kernels.cpp:151-167): rows
 * triangles, columns vertices */
int hmb_op_kdelta(const hmb_mesh* m, int b_min, double eta, int device, int shard_rank,
                  int shard_count, hmb_op** out);
int hmb_op_newton(int n, const double* pts, const double* boxes6, double diag,
                  int b_min, double eta, int device, hmb_op** out);
int hmb_op_dense(int m, int n, const double* a_colmajor, const double* row_pts,
                 const double* col_pts, int b_min, double eta, int device,
                 hmb_op** out);
void hmb_op_free(hmb_op* op);
/* rows/cols in DOFs, ncomp (6 Kelvin, 1 scalar), owned row range */
int hmb_op_info(const hmb_op* op, long long* rows, long long* cols, int* ncomp,
                int* row_begin, int* row_end);
/* underlying hmgpu_ctx* (NULL for host-only operators) */
void* hmb_op_gpu(const hmb_op* op);

/* which = 0 row tree, 1 column tree */
int hmb_tree_info(const hmb_op* op, int which, int* n_nodes, int* depth, int* size);
/* nodes as [begin, end, child0, child1, level], boxes [lo, hi], perm */
int hmb_tree_nodes(const hmb_op* op, int which, int* nodes5, double* boxes6, int* perm);
int hmb_partition_info(const hmb_op* op, int* n_blocks, int* n_admissible, int* c_sp);
int hmb_partition_blocks(const hmb_op* op, int* blocks4);
int hmb_partition_json(const hmb_op* op, char* buf, long long* len);

/* stats8: aca_entries, dense_entries, aca_steps, pivots, ms_total,
 * ms_nearfield, relaunches, counted_flops (NULL allowed) */
int hmb_assemble(hmb_op* op, double eps, double beta, int initial_rank,
                 int lookahead, long long max_rank, double* stats8);
int hmb_matvec(const hmb_op* op, const double* x, double* y, int nrhs, int mode,
               int device_ptrs);
/* y = A^T x (HMatrix::matvec_transposed, hmatrix.cpp:47-72) */
int hmb_matvec_transposed(const hmb_op* op, const double* x, double* y, int nrhs, int mode,
                          int device_ptrs);
int hmb_ranks(const hmb_op* op, int* k_cur, int* k_look, int* consumed, int* last_stop);
int hmb_promote(hmb_op* op, int n, const int* comp_block);
int hmb_extend(hmb_op* op, int n, const int* comp_block, int steps);
/* mb_current, mb_tail, mb_dense, mb_arena, matvec_bytes, matvec_flops, pivots */
int hmb_storage(const hmb_op* op, double* out7);
int hmb_factor(const hmb_op* op, int comp, int block, int* m, int* n, int* K,
               int* k_cur, double* U, double* V, int* piv, double* frob_sq);
int hmb_dense_block(const hmb_op* op, int comp, int block, double* out);

/* ---- adaptive matvec ---- */
/* computes the estimator and keeps it in the operator for hmb_gamma_* */
int hmb_gamma(hmb_op* op, const double* x, double* gamma, double* difference,
              int* n_terms);
/* the same for the transposed occurrence: x over the rows, terms and
 * difference over the columns (amvm.cpp:100-106); kept like hmb_gamma's */
int hmb_gamma_t(hmb_op* op, const double* x, double* gamma, double* difference, int* n_terms);
/* per term: comp, block, nnz, norm_sq */
int hmb_gamma_terms(const hmb_op* op, int* comp, int* block, int* nnz, double* norm_sq);
int hmb_gamma_term_data(const hmb_op* op, int t, long long* idx, double* val);
int hmb_mark(const hmb_op* op, double theta, int c_sp, long long m_rows,
             long long n_cols, int* marked, int* n_marked, double* gamma_pk);
/* mark_blocks (amvm.cpp:131-184) over block-row shards: every rank passes its
 * own terms (CSR: term t's rows idx[term_ptr[t] .. term_ptr[t+1]), values
 * val), the WHOLE difference vector and the flags of its rows; the ranks
 * exchange their marking events through `allgather` (recv[r * bytes ...] =
 * send of rank r; returns 0 on success) and each gets its marked terms
 * (indices into its own list), the count over all ranks and gamma(P_k) --
 * the unsharded walk's result, bit for bit.  A sharded hmb_amvm runs this
 * between its ranks (the library's communicator). */
typedef int (*hmb_allgather_fn)(void* user, const void* send, void* recv,
                                long long bytes_per_rank);
int hmb_mark_sharded(int n_terms, const long long* term_ptr, const long long* idx,
                     const double* val, const double* difference,
                     const unsigned char* own_rows, long long m_rows, long long n_cols,
                     double theta, int c_sp, int nranks, int rank,
                     hmb_allgather_fn allgather, void* user, int* marked, int* n_marked,
                     int* n_marked_total, double* gamma_pk);
/* iterations as rows of 8 doubles [k, gamma, gamma_pk, marked,
 * cumulative_pivots, storage_mb, e_hat, ms]; iters8 holds max_iterations+1 rows */
int hmb_amvm(hmb_op* op, const double* x, double theta, double eps_amvm,
             int lookahead_steps, int max_iterations, double* b, double* iters8,
             int* n_iters, int* converged);

#ifdef __cplusplus
}
#endif

#endif /* HMBEM_H */
