"""Python mirror of the reference's operator API for the hot path.

Names, argument meaning and error behaviour follow the reference library
(/root/reference/proj/include/hmbem): ``build_cluster_tree`` /
``build_block_partition`` / ``sparsity_constant`` / ``partition_to_json``
(cluster.hpp), ``AssemblyConfig`` + ``assemble`` + ``HMatrix.matvec(x, Mode)``
+ ``promote`` / ``extend_lookahead`` + storage accounting (hmatrix.hpp),
``gamma_contributions`` / ``mark_blocks`` / ``amvm_multiply`` (amvm.hpp).
Every call goes through the native C API (include/hmbem.h) and the CUDA
C ABI (include/hmgpu.h); there is no Python compute path.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import host as _h


# ---- errors: the reference's exception hierarchy (types.hpp:20-38) -------
class Error(RuntimeError):
    pass


class MeshError(Error):
    pass


class ConfigError(Error):
    pass


class DimensionError(Error):
    pass


class DeviceError(Error):
    def __init__(self, msg: str, status: int = 0):
        super().__init__(msg)
        self.status = status


_ERRORS = {1: Error, 2: MeshError, 3: ConfigError, 4: DimensionError}


def _check(st: int) -> None:
    if st == 0:
        return
    msg = _h.hmb_last_error().decode(errors="replace")
    if st == 5:
        raise DeviceError(msg, _h.hmb_device_status())
    raise _ERRORS.get(st, Error)(msg)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def device_count() -> int:
    n = C.c_int(0)
    _lib.gpu.hmgpu_device_count(C.byref(n))
    return n.value


class Mode(enum.IntEnum):  # hmatrix.hpp:18
    Current = 0
    Lookahead = 1


class AcaStop(enum.IntEnum):  # aca.hpp:66-72
    NONE = 0
    Inequality = 1
    Exhausted = 2
    RankCap = 3
    StepsDone = 4


# ---------------------------------------------------------------------------
class Mesh:
    """Closed triangulated surface (SurfaceMesh, mesh.hpp:15-40)."""

    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        if getattr(self, "_h", None):
            _h.hmb_mesh_free(self._h)
            self._h = None

    @staticmethod
    def _make(fn, *args) -> "Mesh":
        out = C.c_void_p()
        _check(fn(*args, C.byref(out)))
        return Mesh(out)

    @classmethod
    def icosphere(cls, level: int) -> "Mesh":
        return cls._make(_h.hmb_mesh_icosphere, level)

    @classmethod
    def ellipsoid(cls, level: int, ax: float, ay: float, az: float) -> "Mesh":
        return cls._make(_h.hmb_mesh_ellipsoid, level, ax, ay, az)

    @classmethod
    def voxel_cube(cls, n: int, lo: float = 0.0, hi: float = 1.0) -> "Mesh":
        return cls._make(_h.hmb_mesh_voxel_cube, n, lo, hi)

    @classmethod
    def from_arrays(cls, verts, tris) -> "Mesh":
        v = _f64(verts).reshape(-1, 3)
        t = np.ascontiguousarray(tris, dtype=np.int32).reshape(-1, 3)
        return cls._make(_h.hmb_mesh_from_arrays, len(v), _ptr(v), len(t), _ptr(t))

    @classmethod
    def load_off(cls, path: str) -> "Mesh":
        return cls._make(_h.hmb_mesh_load_off, path.encode())

    def save_off(self, path: str) -> None:
        _check(_h.hmb_mesh_save_off(self._h, path.encode()))

    def validate(self) -> None:
        _check(_h.hmb_mesh_validate(self._h))

    def label_dirichlet(self, predicate: str) -> None:
        _check(_h.hmb_mesh_label(self._h, predicate.encode()))

    @property
    def sizes(self):
        nv, nt = C.c_int(), C.c_int()
        _check(_h.hmb_mesh_sizes(self._h, C.byref(nv), C.byref(nt)))
        return nv.value, nt.value

    def arrays(self) -> dict:
        nv, nt = self.sizes
        out = dict(vertices=np.zeros((nv, 3)), triangles=np.zeros((nt, 3), np.int32),
                   centroids=np.zeros((nt, 3)), areas=np.zeros(nt),
                   normals=np.zeros((nt, 3)), diam=np.zeros(nt),
                   dirichlet=np.zeros(nt, np.int32))
        _check(_h.hmb_mesh_get(self._h, *[_ptr(out[k]) for k in (
            "vertices", "triangles", "centroids", "areas", "normals", "diam",
            "dirichlet")]))
        return out

    @property
    def num_triangles(self) -> int:
        return self.sizes[1]

    @property
    def num_vertices(self) -> int:
        return self.sizes[0]


# ---------------------------------------------------------------------------
@dataclasses.dataclass
class AssemblyConfig:  # hmatrix.hpp:20-27
    eps: float = 1e-6
    beta: float = 0.8
    initial_rank: int = -1
    lookahead: int = 2
    max_rank: int = 1 << 30


@dataclasses.dataclass
class AssemblyStats:
    aca_entries: int
    dense_entries: int
    aca_steps: int
    pivots: int
    ms_total: float
    ms_nearfield: float
    relaunches: int
    counted_flops: float = 0.0

    @property
    def entries(self) -> int:
        return self.aca_entries + self.dense_entries


@dataclasses.dataclass
class ClusterTree:  # cluster.hpp:35-61 (a host-side snapshot)
    nodes: np.ndarray  # rows [begin, end, child0, child1, level]
    boxes: np.ndarray  # rows [lo(3), hi(3)]
    perm: np.ndarray
    depth: int

    @property
    def inv_perm(self) -> np.ndarray:
        inv = np.empty_like(self.perm)
        inv[self.perm] = np.arange(len(self.perm), dtype=self.perm.dtype)
        return inv

    def leaves(self) -> np.ndarray:
        return np.nonzero(self.nodes[:, 2] < 0)[0]


@dataclasses.dataclass
class BlockTerm:  # amvm.hpp:19-25
    comp: int
    block: int
    idx: np.ndarray
    val: np.ndarray
    norm_sq: float


@dataclasses.dataclass
class GammaContributions:  # amvm.hpp:27-31
    gamma: float
    difference: np.ndarray
    terms: list


@dataclasses.dataclass
class AmvmConfig:  # amvm.hpp:10-15
    theta: float = 0.7
    eps_amvm: float = 1e-6
    lookahead_steps: int = 2
    max_iterations: int = 100


@dataclasses.dataclass
class AmvmIteration:
    k: int
    gamma: float
    gamma_pk: float
    marked: int
    cumulative_pivots: int
    storage_mb: float
    e_hat: float
    ms: float


@dataclasses.dataclass
class AmvmReport:
    iterations: list
    termination: str
    converged: bool
    c_sp: int


class HMatrix:
    """GPU-resident H-matrix (scalar) or 3x3 Kelvin block grid of six
    component H-matrices sharing one partition (baca.cpp:669-687)."""

    def __init__(self, handle):
        self._h = handle
        rows, cols = C.c_longlong(), C.c_longlong()
        nc, rb, re = C.c_int(), C.c_int(), C.c_int()
        _check(_h.hmb_op_info(handle, C.byref(rows), C.byref(cols), C.byref(nc),
                              C.byref(rb), C.byref(re)))
        self.rows, self.cols, self.ncomp = rows.value, cols.value, nc.value
        self.row_range = (rb.value, re.value)
        self.config: Optional[AssemblyConfig] = None
        self.last_stats: Optional[AssemblyStats] = None

    def __del__(self):
        if getattr(self, "_h", None):
            _h.hmb_op_free(self._h)
            self._h = None

    # ---- construction ----
    @classmethod
    def kelvin(cls, mesh: Mesh, E: float = 1.0, nu: float = 0.3, b_min: int = 32,
               eta: float = 1.0, device: int = 0, shard: tuple = (0, 1)) -> "HMatrix":
        out = C.c_void_p()
        _check(_h.hmb_op_kelvin(mesh._h, E, nu, b_min, eta, device, shard[0], shard[1],
                                C.byref(out)))
        return cls(out)

    @classmethod
    def kelvin_points(cls, mesh: Mesh, points, E: float = 1.0, nu: float = 0.3,
                      b_min: int = 32, eta: float = 1.0, min_distance_factor: float = 0.5,
                      device: int = 0, shard: tuple = (0, 1),
                      disjoint_order: int = 4) -> "HMatrix":
        """The single-layer grid V~ of evaluate_interior (baca.cpp:625-687):
        CollocSingleOracle(r, c) at arbitrary points (rows) against the
        triangles (columns); 3 n_points x 3 N_t."""
        p = _f64(points).reshape(-1, 3)
        out = C.c_void_p()
        _check(_h.hmb_op_kelvin_points(mesh._h, len(p), _ptr(p), E, nu, b_min, eta,
                                       min_distance_factor, disjoint_order, device, shard[0],
                                       shard[1], C.byref(out)))
        return cls(out)

    @classmethod
    def kelvin_double(cls, mesh: Mesh, points, r: int, c: int, E: float = 1.0,
                      nu: float = 0.3, b_min: int = 32, eta: float = 1.0,
                      min_distance_factor: float = 0.5, device: int = 0,
                      shard: tuple = (0, 1), disjoint_order: int = 4) -> "HMatrix":
        """Cell (r, c) of evaluate_interior's double-layer grid W~
        (CollocDoubleOracle, kernels.cpp:189-210): n_points x N_v."""
        p = _f64(points).reshape(-1, 3)
        out = C.c_void_p()
        _check(_h.hmb_op_kelvin_double(mesh._h, len(p), _ptr(p), int(r), int(c), E, nu, b_min,
                                       eta, min_distance_factor, disjoint_order, device,
                                       shard[0], shard[1], C.byref(out)))
        return cls(out)

    @classmethod
    def galerkin(cls, mesh: Mesh, which: int = 0, b_min: int = 32, eta: float = 1.0,
                 device: int = 0, shard: tuple = (0, 1)) -> "HMatrix":
        """Galerkin scalar kernels over triangle pairs (GalerkinKernels,
        kernels.cpp:95-149) on the triangle partition of assemble_operators
        (operators.cpp:186-235): which = 0 -> the six V_kl as the symmetric
        3x3 grid (3 N_t dofs), 1 -> V_Delta (N_t dofs)."""
        out = C.c_void_p()
        _check(_h.hmb_op_galerkin(mesh._h, int(which), b_min, eta, device, shard[0],
                                  shard[1], C.byref(out)))
        return cls(out)

    @classmethod
    def kdelta(cls, mesh: Mesh, b_min: int = 32, eta: float = 1.0, device: int = 0,
               shard: tuple = (0, 1)) -> "HMatrix":
        """K_Delta (GalerkinKernels::kdelta, kernels.cpp:151-167) on the
        triangle x node partition (operators.cpp:186-200): N_t x N_v."""
        out = C.c_void_p()
        _check(_h.hmb_op_kdelta(mesh._h, b_min, eta, device, shard[0], shard[1],
                                C.byref(out)))
        return cls(out)

    @classmethod
    def newton(cls, points, boxes=None, diag: float = 2.0, b_min: int = 10,
               eta: float = 0.8, device: int = 0) -> "HMatrix":
        p = _f64(points).reshape(-1, 3)
        b = None if boxes is None else _f64(boxes).reshape(-1, 6)
        out = C.c_void_p()
        _check(_h.hmb_op_newton(len(p), _ptr(p), _ptr(b), diag, b_min, eta, device,
                                C.byref(out)))
        return cls(out)

    @classmethod
    def dense(cls, a, row_points, col_points, b_min: int = 10, eta: float = 0.8,
              device: int = 0) -> "HMatrix":
        a = np.asfortranarray(a, dtype=np.float64)
        m, n = a.shape
        rp = _f64(row_points).reshape(-1, 3)
        cp = _f64(col_points).reshape(-1, 3)
        out = C.c_void_p()
        _check(_h.hmb_op_dense(m, n, a.ctypes.data_as(C.c_void_p), _ptr(rp), _ptr(cp),
                               b_min, eta, device, C.byref(out)))
        return cls(out)

    @property
    def gpu_ctx(self):
        return _h.hmb_op_gpu(self._h)

    def set_matvec_policy(self, direct) -> None:
        """direct=True (1): 1-RHS matvecs sweep the blocks in place (no stream
        plan; for one matvec per rank change), False (0): the packed stream
        plan, "auto" (2): the first product after a rank change in place, the
        plan from the second on."""
        pol = 2 if direct == "auto" or direct == 2 else (1 if direct else 0)
        st = _lib.gpu.hmgpu_set_matvec_policy(self.gpu_ctx, pol)
        if st:
            raise DeviceError("hmgpu_set_matvec_policy failed", st)

    # ---- multi-GPU block-row shards ----
    def _gpu_check(self, st: int) -> None:
        if st:
            raise DeviceError(_lib.gpu.hmgpu_last_error(self.gpu_ctx).decode(), st)

    def attach_nccl(self, nranks: int, rank: int, unique_id: bytes) -> None:
        """The library's own NCCL communicator over the shards (collective:
        every rank calls it with rank 0's nccl_unique_id())."""
        uid = C.create_string_buffer(bytes(unique_id), 128)
        self._gpu_check(_lib.gpu.hmgpu_comm_init_nccl(self.gpu_ctx, nranks, rank, uid))

    def attach_comm(self, nranks: int, rank: int, broadcast, allgather) -> None:
        """Host-callback transport: broadcast(buf: np.uint8 array, root) in
        place, allgather(send: np.uint8 array, recv: np.uint8 array) with
        recv = concatenation over ranks (e.g. torch.distributed gloo,
        paper_2205_04752_b200.dist.torch_transport)."""
        def bc(_user, buf, nbytes, root):
            try:
                broadcast(np.ctypeslib.as_array(C.cast(buf, C.POINTER(C.c_uint8)),
                                                (int(nbytes),)), int(root))
                return 0
            except Exception:  # reported as HMGPU_ERR_COMM
                return 1

        def ag(_user, send, recv, nbytes):
            try:
                s = np.ctypeslib.as_array(C.cast(send, C.POINTER(C.c_uint8)), (int(nbytes),))
                r = np.ctypeslib.as_array(C.cast(recv, C.POINTER(C.c_uint8)),
                                          (int(nbytes) * nranks,))
                allgather(s, r)
                return 0
            except Exception:
                return 1

        ops = _lib.CommOps(_lib.BCAST_FN(bc), _lib.ALLGATHER_FN(ag), None)
        self._comm_keep = ops  # the callbacks must outlive the communicator
        self._gpu_check(_lib.gpu.hmgpu_comm_set_ops(self.gpu_ctx, nranks, rank, C.byref(ops)))

    def comm_info(self) -> dict:
        n, r, k = C.c_int(), C.c_int(), C.c_int()
        self._gpu_check(_lib.gpu.hmgpu_comm_info(self.gpu_ctx, C.byref(n), C.byref(r),
                                                 C.byref(k), None, None))
        rb = np.zeros(n.value, np.int32)
        re = np.zeros(n.value, np.int32)
        self._gpu_check(_lib.gpu.hmgpu_comm_info(self.gpu_ctx, None, None, None, _ptr(rb),
                                                 _ptr(re)))
        return dict(nranks=n.value, rank=r.value,
                    kind={0: "none", 1: "nccl", 2: "nccl (borrowed)", 3: "host"}[k.value],
                    row_begin=rb, row_end=re)

    def matvec_dist(self, x=None, mode: Mode = Mode.Current, nrhs: int = 1) -> np.ndarray:
        """The whole product A x on every rank: x (read on rank 0 only) is
        broadcast, each rank sweeps its block rows, the row segments are
        all-gathered (hmgpu_matvec_dist)."""
        y = np.zeros((self.rows, nrhs), order="F")
        xp = None
        if x is not None:
            xf = np.asfortranarray(np.asarray(x, dtype=np.float64).reshape(self.cols, -1))
            if xf.shape[1] != nrhs:
                raise DimensionError("matvec_dist: nrhs")
            xp = xf.ctypes.data_as(C.c_void_p)
        self._gpu_check(_lib.gpu.hmgpu_matvec_dist(self.gpu_ctx, xp,
                                                   y.ctypes.data_as(C.c_void_p), nrhs,
                                                   int(mode), 0))
        return y[:, 0].copy() if nrhs == 1 else y

    def matvec_dist_ptr(self, x_ptr: int, y_ptr: int, nrhs: int = 1,
                        mode: Mode = Mode.Current, device: bool = True) -> None:
        self._gpu_check(_lib.gpu.hmgpu_matvec_dist(self.gpu_ctx, C.c_void_p(x_ptr or None),
                                                   C.c_void_p(y_ptr), nrhs, int(mode),
                                                   1 if device else 0))

    # ---- tree / partition ----
    def tree(self, which: int = 0) -> ClusterTree:
        nn, dep, sz = C.c_int(), C.c_int(), C.c_int()
        _check(_h.hmb_tree_info(self._h, which, C.byref(nn), C.byref(dep), C.byref(sz)))
        nodes = np.zeros((nn.value, 5), np.int32)
        boxes = np.zeros((nn.value, 6))
        perm = np.zeros(sz.value, np.int32)
        _check(_h.hmb_tree_nodes(self._h, which, _ptr(nodes), _ptr(boxes), _ptr(perm)))
        return ClusterTree(nodes, boxes, perm, dep.value)

    def partition_info(self):
        nb, na, csp = C.c_int(), C.c_int(), C.c_int()
        _check(_h.hmb_partition_info(self._h, C.byref(nb), C.byref(na), C.byref(csp)))
        return nb.value, na.value, csp.value

    @property
    def num_blocks(self) -> int:
        return self.partition_info()[0]

    @property
    def sparsity_constant(self) -> int:
        return self.partition_info()[2]

    def partition_blocks(self) -> np.ndarray:
        out = np.zeros((self.num_blocks, 4), np.int32)
        _check(_h.hmb_partition_blocks(self._h, _ptr(out)))
        return out

    def partition_json(self) -> str:
        n = C.c_longlong()
        _check(_h.hmb_partition_json(self._h, None, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        _check(_h.hmb_partition_json(self._h, buf, C.byref(n)))
        return buf.value.decode()

    # ---- assembly / products ----
    def assemble(self, cfg: Optional[AssemblyConfig] = None, **kw) -> AssemblyStats:
        cfg = cfg or AssemblyConfig(**kw)
        st = np.zeros(8)
        _check(_h.hmb_assemble(self._h, cfg.eps, cfg.beta, cfg.initial_rank,
                               cfg.lookahead, cfg.max_rank, _ptr(st)))
        self.config = cfg
        self.last_stats = AssemblyStats(int(st[0]), int(st[1]), int(st[2]), int(st[3]),
                                        float(st[4]), float(st[5]), int(st[6]), float(st[7]))
        return self.last_stats

    def matvec(self, x, mode: Mode = Mode.Current) -> np.ndarray:
        x = np.asarray(x, dtype=np.float64)
        vec = x.ndim == 1
        xm = x.reshape(x.shape[0], -1)
        if xm.shape[0] != self.cols:
            raise DimensionError("HMatrix::matvec: size")
        nrhs = xm.shape[1]
        xf = np.asfortranarray(xm)
        y = np.zeros((self.rows, nrhs), order="F")
        _check(_h.hmb_matvec(self._h, xf.ctypes.data_as(C.c_void_p),
                             y.ctypes.data_as(C.c_void_p), nrhs, int(mode), 0))
        return y[:, 0].copy() if vec else y

    def matvec_transposed(self, x, mode: Mode = Mode.Current) -> np.ndarray:
        """y = A^T x (HMatrix::matvec_transposed, hmatrix.cpp:47-72)."""
        x = np.asarray(x, dtype=np.float64)
        vec = x.ndim == 1
        xm = x.reshape(x.shape[0], -1)
        if xm.shape[0] != self.rows:
            raise DimensionError("HMatrix::matvec_transposed: size")
        nrhs = xm.shape[1]
        xf = np.asfortranarray(xm)
        y = np.zeros((self.cols, nrhs), order="F")
        _check(_h.hmb_matvec_transposed(self._h, xf.ctypes.data_as(C.c_void_p),
                                        y.ctypes.data_as(C.c_void_p), nrhs, int(mode), 0))
        return y[:, 0].copy() if vec else y

    def matvec_ptr(self, x_ptr: int, y_ptr: int, nrhs: int = 1,
                   mode: Mode = Mode.Current, device: bool = True) -> None:
        """y = A x on raw pointers (device pointers by default, e.g. torch
        tensors' data_ptr(); host pointers should be pinned)."""
        _check(_h.hmb_matvec(self._h, C.c_void_p(x_ptr), C.c_void_p(y_ptr), nrhs,
                             int(mode), 1 if device else 0))

    def _pairs(self, pairs) -> np.ndarray:
        return np.ascontiguousarray(np.asarray(pairs, dtype=np.int32).reshape(-1, 2))

    def promote(self, pairs) -> None:
        p = self._pairs(pairs)
        _check(_h.hmb_promote(self._h, len(p), _ptr(p)))

    def extend_lookahead(self, pairs, steps: int) -> None:
        p = self._pairs(pairs)
        _check(_h.hmb_extend(self._h, len(p), _ptr(p), steps))

    def ranks(self):
        n = self.ncomp * self.num_blocks
        kc, kl, co, ls = (np.zeros(n, np.int32) for _ in range(4))
        _check(_h.hmb_ranks(self._h, _ptr(kc), _ptr(kl), _ptr(co), _ptr(ls)))
        shape = (self.ncomp, self.num_blocks)
        return kc.reshape(shape), kl.reshape(shape), co.reshape(shape), ls.reshape(shape)

    def storage(self) -> dict:
        out = np.zeros(7)
        _check(_h.hmb_storage(self._h, _ptr(out)))
        return dict(mb_current=out[0], mb_tail=out[1], mb_dense=out[2],
                    mb_arena=out[3], matvec_bytes=int(out[4]), matvec_flops=int(out[5]),
                    total_pivots=int(out[6]))

    def storage_mb_current(self) -> float:
        return self.storage()["mb_current"]

    def storage_mb_tail(self) -> float:
        return self.storage()["mb_tail"]

    def total_pivots(self) -> int:
        return self.storage()["total_pivots"]

    def factor(self, comp: int, block: int):
        m, n, K, kc = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        fs = C.c_double()
        _check(_h.hmb_factor(self._h, comp, block, C.byref(m), C.byref(n), C.byref(K),
                             C.byref(kc), None, None, None, C.byref(fs)))
        U = np.zeros((m.value, K.value), order="F")
        V = np.zeros((n.value, K.value), order="F")
        piv = np.zeros((K.value, 2), np.int32)
        _check(_h.hmb_factor(self._h, comp, block, C.byref(m), C.byref(n), C.byref(K),
                             C.byref(kc), U.ctypes.data_as(C.c_void_p),
                             V.ctypes.data_as(C.c_void_p), _ptr(piv), C.byref(fs)))
        return dict(U=U, V=V, pivots=piv, frob_sq=fs.value, k_cur=kc.value)

    def dense_block(self, comp: int, block: int) -> np.ndarray:
        nodes_r = self.tree(0).nodes
        nodes_c = self.tree(1).nodes
        b = self.partition_blocks()[block]
        m = nodes_r[b[0], 1] - nodes_r[b[0], 0]
        n = nodes_c[b[1], 1] - nodes_c[b[1], 0]
        out = np.zeros((m, n), order="F")
        _check(_h.hmb_dense_block(self._h, comp, block, out.ctypes.data_as(C.c_void_p)))
        return out

    # ---- adaptive matvec ----
    def gamma_contributions(self, x, term_data: bool = True,
                            transposed: bool = False) -> GammaContributions:
        """term_data = False skips the per-term index/value downloads (the
        terms then carry empty idx / val; gamma, difference and norm_sq are
        complete).  transposed: the transposed occurrence (x over the rows,
        terms over the columns)."""
        x = _f64(x)
        if x.shape != ((self.rows if transposed else self.cols),):
            raise DimensionError("gamma_contributions: size")
        g = C.c_double()
        diff = np.zeros(self.cols if transposed else self.rows)
        nt = C.c_int()
        fn = _h.hmb_gamma_t if transposed else _h.hmb_gamma
        _check(fn(self._h, _ptr(x), C.byref(g), _ptr(diff), C.byref(nt)))
        n = nt.value
        self._last_nterms = n
        comp, block, nnz = (np.zeros(n, np.int32) for _ in range(3))
        nsq = np.zeros(n)
        _check(_h.hmb_gamma_terms(self._h, _ptr(comp), _ptr(block), _ptr(nnz), _ptr(nsq)))
        terms = []
        for t in range(n):
            idx = np.zeros(nnz[t] if term_data else 0, np.int64)
            val = np.zeros(nnz[t] if term_data else 0)
            if term_data:
                _check(_h.hmb_gamma_term_data(self._h, t, _ptr(idx), _ptr(val)))
            terms.append(BlockTerm(int(comp[t]), int(block[t]), idx, val, float(nsq[t])))
        return GammaContributions(g.value, diff, terms)

    def mark_blocks(self, theta: float, c_sp: int, m_rows: int, n_cols: int):
        """Marks on the estimator of the last gamma_contributions call."""
        cap = max(1, getattr(self, "_last_nterms", 0))
        marked = np.zeros(cap, np.int32)
        nm = C.c_int()
        gpk = C.c_double()
        _check(_h.hmb_mark(self._h, theta, c_sp, m_rows, n_cols, _ptr(marked),
                           C.byref(nm), C.byref(gpk)))
        return marked[: nm.value].copy(), gpk.value

    def amvm_multiply(self, x, cfg: Optional[AmvmConfig] = None, **kw):
        cfg = cfg or AmvmConfig(**kw)
        x = _f64(x)
        if x.shape != (self.cols,):
            raise DimensionError("amvm_multiply: size")
        if cfg.max_iterations < 0:
            raise ConfigError("amvm_multiply: max_iterations must be >= 0")
        b = np.zeros(self.rows)
        iters = np.zeros((cfg.max_iterations + 1, 8))
        ni, conv = C.c_int(), C.c_int()
        _check(_h.hmb_amvm(self._h, _ptr(x), cfg.theta, cfg.eps_amvm, cfg.lookahead_steps,
                           cfg.max_iterations, _ptr(b), _ptr(iters), C.byref(ni),
                           C.byref(conv)))
        its = [AmvmIteration(int(r[0]), r[1], r[2], int(r[3]), int(r[4]), r[5], r[6], r[7])
               for r in iters[: ni.value]]
        term = "tolerance" if conv.value else "max_iterations"
        return b, AmvmReport(its, term, bool(conv.value), self.sparsity_constant)

    # ---- device-level helpers ----
    def stream(self) -> int:
        s = C.c_void_p()
        st = _lib.gpu.hmgpu_get_stream(self.gpu_ctx, C.byref(s))
        if st:
            raise DeviceError(_lib.gpu.hmgpu_last_error(self.gpu_ctx).decode(), st)
        return s.value or 0

    def set_profiling(self, on: bool) -> None:
        _lib.gpu.hmgpu_set_profiling(self.gpu_ctx, 1 if on else 0)

    def kernel_times(self, name: str, reset: bool = False):
        ms = C.c_double()
        n = C.c_longlong()
        st = _lib.gpu.hmgpu_kernel_times(self.gpu_ctx, name.encode(), C.byref(ms),
                                         C.byref(n), 1 if reset else 0)
        if st:
            raise DeviceError(_lib.gpu.hmgpu_last_error(self.gpu_ctx).decode(), st)
        return ms.value, n.value


def mark_blocks_sharded(terms, difference, own_rows, theta: float, c_sp: int, m_rows: int,
                        n_cols: int, nranks: int, rank: int, allgather):
    """mark_blocks (amvm.cpp:131-184) across block-row shards (hmb_mark_sharded).
    terms: this rank's BlockTerms (rows of its shard); difference: the whole
    difference vector; own_rows: bool flags of this rank's rows; allgather as
    HMatrix.attach_comm's (np.uint8 send / recv arrays, recv = concatenation
    over ranks).  Returns (this rank's marked term indices, marked count over
    all ranks, gamma(P_k)) -- the unsharded walk's result bit for bit."""
    diff = _f64(difference)
    if diff.shape != (m_rows,):
        raise DimensionError("mark_blocks: difference size")
    own = np.ascontiguousarray(np.asarray(own_rows, dtype=np.uint8))
    if own.shape != (m_rows,):
        raise DimensionError("mark_blocks: own_rows size")
    ptr = np.zeros(len(terms) + 1, np.int64)
    for t, term in enumerate(terms):
        ptr[t + 1] = ptr[t] + len(term.idx)
    idx = np.ascontiguousarray(np.concatenate([np.asarray(t.idx, np.int64) for t in terms])
                               if terms else np.zeros(1, np.int64))
    val = np.ascontiguousarray(np.concatenate([np.asarray(t.val, np.float64) for t in terms])
                               if terms else np.zeros(1))

    def ag(_user, send, recv, nbytes):
        try:
            s = np.ctypeslib.as_array(C.cast(send, C.POINTER(C.c_uint8)), (int(nbytes),))
            r = np.ctypeslib.as_array(C.cast(recv, C.POINTER(C.c_uint8)),
                                      (int(nbytes) * nranks,))
            allgather(s, r)
            return 0
        except Exception:
            return 1

    cb = _lib.ALLGATHER_FN(ag)
    marked = np.zeros(max(1, len(terms)), np.int32)
    nm, nt, gpk = C.c_int(), C.c_int(), C.c_double()
    _check(_h.hmb_mark_sharded(len(terms), _ptr(ptr), _ptr(idx), _ptr(val), _ptr(diff),
                               _ptr(own), m_rows, n_cols, theta, c_sp, nranks, rank, cb,
                               None, _ptr(marked), C.byref(nm), C.byref(nt), C.byref(gpk)))
    return marked[: nm.value].copy(), nt.value, gpk.value


def nccl_available():
    """(available, version) of the NCCL the library loads at run time."""
    a, v = C.c_int(), C.c_int()
    _lib.gpu.hmgpu_nccl_available(C.byref(a), C.byref(v))
    return bool(a.value), v.value


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    st = _lib.gpu.hmgpu_nccl_unique_id(buf)
    if st:
        raise DeviceError("ncclGetUniqueId failed (" + ("NCCL not loadable" if st == 7
                                                        else "error") + ")", st)
    return buf.raw


# ---- reference-style free functions ----------------------------------------
class InteriorEvaluator:
    """evaluate_interior (baca.cpp:625-696): displacements at interior
    points from the full Cauchy data, v = V~ t - W~ u, with the single-layer
    grid V~ (one Kelvin context at the points) and the nine double-layer
    cells W~_rc (points x nodes) as GPU H-matrices."""

    def __init__(self, mesh: Mesh, points, E: float = 1.0, nu: float = 0.3, b_min: int = 32,
                 eta: float = 1.0, min_distance_factor: float = 0.5, device: int = 0,
                 disjoint_order: int = 4):
        self.npts = len(_f64(points).reshape(-1, 3))
        self.nt, self.nv = mesh.num_triangles, mesh.num_vertices
        self.vt = HMatrix.kelvin_points(mesh, points, E, nu, b_min, eta, min_distance_factor,
                                        device, disjoint_order=disjoint_order)
        self.wt = [[HMatrix.kelvin_double(mesh, points, r, c, E, nu, b_min, eta,
                                          min_distance_factor, device,
                                          disjoint_order=disjoint_order)
                    for c in range(3)] for r in range(3)]

    def assemble(self, eps: float = 1e-6, lookahead: int = 2, beta: float = 0.8):
        self.vt.assemble(eps=eps, beta=beta, lookahead=lookahead)
        for row in self.wt:
            for h in row:
                h.assemble(eps=eps, beta=beta, lookahead=lookahead)

    def evaluate(self, t_total, u_total) -> np.ndarray:
        t = np.asarray(t_total, dtype=np.float64)
        u = np.asarray(u_total, dtype=np.float64)
        if t.shape != (3 * self.nt,) or u.shape != (3 * self.nv,):
            raise DimensionError("evaluate_interior: Cauchy data size")
        v = self.vt.matvec(t)
        n = self.npts
        for r in range(3):
            for c in range(3):
                v[r * n:(r + 1) * n] -= self.wt[r][c].matvec(u[c * self.nv:(c + 1) * self.nv])
        return v


class LameSingleLayer:
    """V_h = (1+nu) / (2E (1-nu)) [ (3-4nu) diag3(V_Delta) + grid(V_kl) ]
    (compose_Vh, proj/src/operators.cpp:97-105): the Galerkin single-layer
    operator of the Lame equations from the two GPU H-matrices (the V_kl
    grid and V_Delta, assembled with one partition), 3 N_t dofs
    component-major."""

    def __init__(self, mesh: Mesh, E: float = 1.0, nu: float = 0.3, b_min: int = 32,
                 eta: float = 1.0, device: int = 0, shard: tuple = (0, 1)):
        if E <= 0.0:
            raise Error("lame_constants: E must be positive")
        if not 0.0 < nu < 0.5:
            raise Error("lame_constants: nu must lie in (0, 1/2)")
        self.E, self.nu = E, nu
        self.vkl = HMatrix.galerkin(mesh, 0, b_min, eta, device, shard)
        self.vdelta = HMatrix.galerkin(mesh, 1, b_min, eta, device, shard)
        self.nt = self.vdelta.rows

    @property
    def rows(self) -> int:
        return 3 * self.nt

    @property
    def cols(self) -> int:
        return 3 * self.nt

    def assemble(self, cfg: Optional[AssemblyConfig] = None, **kw):
        return self.vkl.assemble(cfg, **kw), self.vdelta.assemble(cfg, **kw)

    def matvec(self, x, mode: Mode = Mode.Current) -> np.ndarray:
        x = np.asarray(x, dtype=np.float64)
        if x.shape != (self.cols,):
            raise DimensionError("V_h matvec: size")
        s = 0.5 / self.E * (1.0 + self.nu) / (1.0 - self.nu)
        yg = self.vkl.matvec(x, mode)
        # diag3(V_Delta): the three component blocks as three right-hand sides
        yd = self.vdelta.matvec(x.reshape(3, self.nt).T, mode).T.reshape(-1)
        return s * ((3.0 - 4.0 * self.nu) * yd + yg)


def pair_rule(pair_case: int, order: int):
    """The touching-pair rule the device uses (Sauter-Schwab, quadrature.cpp:
    168-338): (xr1, xr2, yr1, yr2, w)."""
    n = C.c_int()
    _check(_h.hmb_pair_rule(int(pair_case), int(order), C.byref(n), None, None, None, None,
                            None))
    arr = [np.zeros(n.value) for _ in range(5)]
    _check(_h.hmb_pair_rule(int(pair_case), int(order), C.byref(n), *[_ptr(a) for a in arr]))
    return tuple(arr)


def sparse_op(mesh: Mesh, which: int):
    """build_sparse_ops in ELL form (operators.cpp:7-95): which 0 T12, 1 T13,
    2 T23, 3 mass; returns (cols, vals), n_tri x 3 each."""
    m = mesh.num_triangles
    cols = np.zeros(3 * m, np.int32)
    vals = np.zeros(3 * m)
    _check(_h.hmb_sparse_op(mesh._h, int(which), _ptr(cols), _ptr(vals)))
    return cols.reshape(m, 3), vals.reshape(m, 3)


def lame_constants(E: float, nu: float):
    """lambda = E nu / ((1+nu)(1-2nu)), mu = E / (2(1+nu)) (kernels.cpp:7-14)."""
    if E <= 0.0:
        raise Error("lame_constants: E must be positive")
    if not 0.0 < nu < 0.5:
        raise Error("lame_constants: nu must lie in (0, 1/2)")
    return E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), E / (2.0 * (1.0 + nu))


class OperatorSet:
    """assemble_operators / OperatorSet (operators.hpp:62-96, SURVEY.md 8f
    ranks 2-3) on the device: the Galerkin H-matrices V_Delta, V_kl (3x3
    grid) and K_Delta, the sparse transforms T12 / T13 / T23 / mass of
    build_sparse_ops (ELL on the device, hmgpu_ell3_spmv), and the composed
    discrete operators

      V_h = (1+nu)/(2E(1-nu)) [(3-4nu) diag3(V_Delta) + grid(V_kl)]      3M x 3M
      K_h = diag3(K_Delta) - diag3(V_Delta) T_h + 2 mu V_h T_h           3M x 3N
      D_h = mu sum_k S_k' diag3(V_Delta) S_k + 2 mu T_h' diag3(V_Delta) T_h
            - 4 mu^2 T_h' V_h T_h + mu [sum_k T_kj' V_Delta T_ki]_ij      3N x 3N

    (compose_Vh / compose_Kh / compose_Dh, operators.cpp:97-158), evaluated
    on device vectors (torch) through the H-matrix and SpMV entry points.
    M = triangles, N = vertices, component-major."""

    def __init__(self, mesh: Mesh, E: float = 1.0, nu: float = 0.3, b_min: int = 32,
                 eta: float = 1.0, device: int = 0):
        import torch
        self._torch = torch
        self.E, self.nu = E, nu
        self.lam, self.mu = lame_constants(E, nu)
        self.device = device
        self.dev = torch.device("cuda", device)
        self._mesh = mesh
        self.vkl = HMatrix.galerkin(mesh, 0, b_min, eta, device)
        self.vdelta = HMatrix.galerkin(mesh, 1, b_min, eta, device)
        self.kdelta = HMatrix.kdelta(mesh, b_min, eta, device)
        self.m, self.n = mesh.num_triangles, mesh.num_vertices
        self._ctx = self.vdelta.gpu_ctx
        self._ell = []
        for which in range(4):  # T12, T13, T23, mass
            cols = np.zeros(3 * self.m, np.int32)
            vals = np.zeros(3 * self.m)
            _check(_h.hmb_sparse_op(mesh._h, which, _ptr(cols), _ptr(vals)))
            # inverse index for the transpose: slots by vertex, ascending rows
            order = np.argsort(cols, kind="stable").astype(np.int32)
            tptr = np.zeros(self.n + 1, np.int32)
            np.cumsum(np.bincount(cols, minlength=self.n), out=tptr[1:])
            self._ell.append(tuple(torch.tensor(a, device=self.dev)
                                   for a in (cols, vals, tptr, order)))

    def assemble(self, cfg: Optional[AssemblyConfig] = None, **kw):
        return (self.vkl.assemble(cfg, **kw), self.vdelta.assemble(cfg, **kw),
                self.kdelta.assemble(cfg, **kw))

    # ---- device building blocks (torch float64 tensors on self.dev) ----
    def _sync(self):
        self._torch.cuda.synchronize(self.dev)

    def _lib_stream(self, handle: int):
        """torch view of a context's stream (cached)."""
        cache = self.__dict__.setdefault("_streams", {})
        if handle not in cache:
            cache[handle] = self._torch.cuda.ExternalStream(handle, device=self.dev)
        return cache[handle]

    def _on_lib(self, handle: int, fn, *tensors):
        """Run a library call on the context's stream, ordered after torch's
        current stream and before its later work by events (no host
        synchronisation).  The tensors are not record_stream'ed on the
        library stream: torch's stream waits for the call, so any reuse of
        their memory on it comes after the library's work -- and a recorded
        event would outlive the context's stream at interpreter exit."""
        torch = self._torch
        ls = self._lib_stream(handle)
        cur = torch.cuda.current_stream(self.dev)
        ls.wait_stream(cur)
        st = fn()
        cur.wait_stream(ls)
        return st

    def _spmv(self, which: int, x, transpose: bool = False, alpha: float = 1.0):
        cols, vals, tptr, slot = self._ell[which]
        x = x.contiguous()
        if transpose:
            y = self._torch.empty(self.n, dtype=self._torch.float64, device=self.dev)
            fn = lambda: _lib.gpu.hmgpu_ell3_spmv_t(
                self._ctx, self.n, tptr.data_ptr(), slot.data_ptr(), vals.data_ptr(),
                x.data_ptr(), y.data_ptr(), alpha, 0.0)
        else:
            y = self._torch.empty(self.m, dtype=self._torch.float64, device=self.dev)
            fn = lambda: _lib.gpu.hmgpu_ell3_spmv(
                self._ctx, self.m, cols.data_ptr(), vals.data_ptr(), x.data_ptr(),
                y.data_ptr(), alpha, 0.0)
        st = self._on_lib(self.vdelta.stream(), fn, x, y)
        if st != 0:
            raise DeviceError(_lib.gpu.hmgpu_last_error(self._ctx).decode(), st)
        return y

    def _hmv(self, h: HMatrix, x, nrhs: int = 1):
        """y = H x for nrhs columns stored back to back (column-major)."""
        x = x.contiguous()
        y = self._torch.empty(h.rows * nrhs, dtype=self._torch.float64, device=self.dev)
        self._on_lib(h.stream(), lambda: h.matvec_ptr(
            x.data_ptr(), y.data_ptr(), nrhs, getattr(self, "mode", Mode.Current)), x, y)
        return y

    def _hmv_t(self, h: HMatrix, x, nrhs: int = 1):
        """y = H^T x (HMatrix::matvec_transposed) for nrhs columns."""
        x = x.contiguous()
        y = self._torch.empty(h.cols * nrhs, dtype=self._torch.float64, device=self.dev)
        st = self._on_lib(h.stream(), lambda: _h.hmb_matvec_transposed(
            h._h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), nrhs,
            int(getattr(self, "mode", Mode.Current)), 1), x, y)
        _check(st)
        return y

    # T_h = [0, T12, T13; -T12, 0, T23; -T13, -T23, 0] (operators.cpp:56-70)
    _TH = ((None, (0, 1.0), (1, 1.0)), ((0, -1.0), None, (2, 1.0)),
           ((1, -1.0), (2, -1.0), None))

    def t_h(self, x):
        """T_h x: 3N -> 3M."""
        n = self.n
        out = []
        for i in range(3):
            acc = None
            for j in range(3):
                e = self._TH[i][j]
                if e is None:
                    continue
                y = self._spmv(e[0], x[j * n:(j + 1) * n], alpha=e[1])
                acc = y if acc is None else acc + y
            out.append(acc)
        return self._torch.cat(out)

    def t_h_t(self, z):
        """T_h' z: 3M -> 3N."""
        m = self.m
        out = []
        for j in range(3):
            acc = None
            for i in range(3):
                e = self._TH[i][j]
                if e is None:
                    continue
                y = self._spmv(e[0], z[i * m:(i + 1) * m], transpose=True, alpha=e[1])
                acc = y if acc is None else acc + y
            out.append(acc)
        return self._torch.cat(out)

    # S_1 = diag3(-T23), S_2 = diag3(T13), S_3 = diag3(T12) (operators.cpp:72-77)
    _S = ((2, -1.0), (1, 1.0), (0, 1.0))

    def s_k(self, k: int, x, transpose: bool = False):
        w, a = self._S[k]
        blk = self.m if transpose else self.n
        return self._torch.cat([self._spmv(w, x[c * blk:(c + 1) * blk], transpose, a)
                                for c in range(3)])

    def vh_dev(self, x):
        """V_h x on a device vector (3M)."""
        s = 0.5 / self.E * (1.0 + self.nu) / (1.0 - self.nu)
        yg = self._hmv(self.vkl, x)
        yd = self._hmv(self.vdelta, x, 3)  # diag3(V_Delta): 3 RHS
        return s * ((3.0 - 4.0 * self.nu) * yd + yg)

    def vh_t_dev(self, z):
        """V_h^T z (the transpose of every leaf H-matrix; V_h^T = V_h up to
        the ACA approximation)."""
        s = 0.5 / self.E * (1.0 + self.nu) / (1.0 - self.nu)
        yg = self._hmv_t(self.vkl, z)
        yd = self._hmv_t(self.vdelta, z, 3)
        return s * ((3.0 - 4.0 * self.nu) * yd + yg)

    def kh_t_dev(self, z):
        """K_h^T z (3M -> 3N) = diag3(K_Delta)^T z - T_h^T diag3(V_Delta)^T z
        + 2 mu T_h^T V_h^T z (the transposed compose_Kh, as the reference's
        transpose(K_ND) in the saddle system, baca.cpp:12-40)."""
        return (self._hmv_t(self.kdelta, z, 3) - self.t_h_t(self._hmv_t(self.vdelta, z, 3))
                + 2.0 * self.mu * self.t_h_t(self.vh_t_dev(z)))

    def kh_dev(self, x):
        """K_h x (3N -> 3M) = diag3(K_Delta) x - diag3(V_Delta) T_h x + 2 mu V_h T_h x."""
        t = self.t_h(x)
        return (self._hmv(self.kdelta, x, 3) - self._hmv(self.vdelta, t, 3)
                + 2.0 * self.mu * self.vh_dev(t))

    def dh_dev(self, x):
        """D_h x (3N -> 3N), compose_Dh (operators.cpp:114-158).  All 24
        V_Delta products of the sandwiches go through ONE multi-RHS H-matvec
        (S_k x blocks, T_h x blocks -- shared with the diag3 part of V_h --
        and the T_ki x_j of the D' grid)."""
        torch = self._torch
        mu, n, m = self.mu, self.n, self.m
        # inputs of the V_Delta products, in order
        ins = []
        for k in range(3):  # S_k x: blocks c of diag3(+-T_w)
            w, a = self._S[k]
            ins += [self._spmv(w, x[c * n:(c + 1) * n], alpha=a) for c in range(3)]
        t = self.t_h(x)
        ins += [t[c * m:(c + 1) * m] for c in range(3)]

        def t_signed(k, l):
            if k == l:
                return None
            return ({(0, 1): 0, (0, 2): 1, (1, 2): 2}[(min(k, l), max(k, l))],
                    1.0 if k < l else -1.0)
        grid = []  # (i, w_kj, sign) per D' product
        for i in range(3):
            for j in range(3):
                for k in range(3):
                    tkj, tki = t_signed(k, j), t_signed(k, i)
                    if tkj is None or tki is None:
                        continue
                    ins.append(self._spmv(tki[0], x[j * n:(j + 1) * n]))
                    grid.append((i, tkj[0], tkj[1] * tki[1]))
        Y = self._hmv(self.vdelta, torch.cat(ins), len(ins)).view(len(ins), m)
        # sum_k mu S_k' diag3(V_Delta) S_k x
        y = None
        for k in range(3):
            w, a = self._S[k]
            z = torch.cat([self._spmv(w, Y[3 * k + c], transpose=True, alpha=a)
                           for c in range(3)])
            y = mu * z if y is None else y + mu * z
        vd_t = Y[9:12].reshape(-1)  # diag3(V_Delta) T_h x
        y = y + 2.0 * mu * self.t_h_t(vd_t)
        s = 0.5 / self.E * (1.0 + self.nu) / (1.0 - self.nu)
        vh_t = s * ((3.0 - 4.0 * self.nu) * vd_t + self._hmv(self.vkl, t))
        y = y - 4.0 * mu * mu * self.t_h_t(vh_t)
        dg = [None, None, None]
        for q, (i, w, sg) in enumerate(grid):
            r = self._spmv(w, Y[12 + q], transpose=True, alpha=sg)
            dg[i] = r if dg[i] is None else dg[i] + r
        return y + mu * torch.cat(dg)

    # ---- host-vector API (numpy in / out) ----
    def _run(self, f, x, n_in):
        x = np.asarray(x, dtype=np.float64)
        if x.shape != (n_in,):
            raise DimensionError("operator matvec: size")
        xd = self._torch.tensor(x, device=self.dev)
        y = f(xd)
        self._sync()
        return y.cpu().numpy()

    def vh(self, x):
        return self._run(self.vh_dev, x, 3 * self.m)

    def kh(self, x):
        return self._run(self.kh_dev, x, 3 * self.n)

    def dh(self, x):
        return self._run(self.dh_dev, x, 3 * self.n)

    def kh_t(self, z):
        return self._run(self.kh_t_dev, z, 3 * self.m)


@dataclasses.dataclass
class BacaConfig:  # baca.hpp:11-23
    theta: float = 0.8
    alpha: float = 10.0
    eps_baca: float = 1e-4
    inner_tol0: float = 1e-1
    inner_floor: float = 1e-12
    lookahead_steps: int = 2
    max_outer: int = 60
    max_inner: int = 10000


@dataclasses.dataclass
class BacaIteration:  # baca.hpp:124-139 (reduced mode: V marks only)
    k: int
    ek: float
    tail_norm: float
    residual: float
    inner_tol: float
    inner_iterations: int
    marked_v: int
    storage_mb: float
    wall_time_s: float


@dataclasses.dataclass
class BacaReport:
    iterations: list
    converged: bool
    termination: str


class VddPreconditioner:
    """build_vdd_preconditioner (baca.cpp:104-192) for the all-Dirichlet
    (reduced) system: the dense leaf-cluster diagonal blocks of V_h (all
    three components, taken from the near-field blocks of the V_kl and
    V_Delta contexts), Cholesky-factored on the device (batched), scaled by
    eta = half the smallest Ritz value of C0^{-1} V_h from a 10-step
    preconditioned Lanczos run, so that eta C0 stays spectrally below V_h."""

    def __init__(self, ops: "OperatorSet", dirichlet=None, vdd=None):
        """dirichlet: sorted Dirichlet triangle ids (None: all triangles);
        vdd: the V_DD matvec on device vectors (default V_h)."""
        torch = ops._torch
        self.ops = ops
        self._vdd = vdd or ops.vh_dev
        m = ops.m
        rank = np.arange(m) if dirichlet is None else np.full(m, -1)
        if dirichlet is not None:
            rank[np.asarray(dirichlet)] = np.arange(len(dirichlet))
        md = m if dirichlet is None else len(dirichlet)
        self.n = 3 * md
        pref = 0.5 / ops.E * (1.0 + ops.nu) / (1.0 - ops.nu)
        c34 = 3.0 - 4.0 * ops.nu
        tree = ops.vdelta.tree(0)
        blocks = ops.vdelta.partition_blocks()
        diag = {int(r): b for b, (r, c, adm, _) in enumerate(blocks) if r == c and not adm}
        idx = {(0, 0): 0, (0, 1): 1, (0, 2): 2, (1, 1): 3, (1, 2): 4, (2, 2): 5}
        groups, mats = [], []
        for leaf in tree.leaves():
            b0, b1 = tree.nodes[leaf, 0], tree.nodes[leaf, 1]
            # the Dirichlet members of the leaf (baca.cpp:113-127)
            sel = np.nonzero(rank[tree.perm[b0:b1]] >= 0)[0]
            if len(sel) == 0:
                continue
            members = tree.perm[b0:b1][sel]
            nm = len(members)
            b = diag[int(leaf)]
            dd = ops.vdelta.dense_block(0, b)[np.ix_(sel, sel)]
            blk = np.zeros((3 * nm, 3 * nm))
            for c1 in range(3):
                for c2 in range(3):
                    d = ops.vkl.dense_block(idx[(min(c1, c2), max(c1, c2))], b)[np.ix_(sel, sel)]
                    if c1 == c2:
                        d = d + c34 * dd
                    blk[c1 * nm:(c1 + 1) * nm, c2 * nm:(c2 + 1) * nm] = pref * d
            groups.append(np.concatenate([c * md + rank[members] for c in range(3)]))
            mats.append(blk)
        # batch by block size (leaves of one tree level share it)
        self.batches = []
        for size in sorted({len(g) for g in groups}):
            sel = [i for i, g in enumerate(groups) if len(g) == size]
            G = torch.tensor(np.stack([groups[i] for i in sel]), device=ops.dev)
            A = torch.tensor(np.stack([mats[i] for i in sel]), device=ops.dev)
            L = torch.linalg.cholesky(A)  # raises if a block is not SPD
            self.batches.append((G, A, L))
        self.eta = 1.0
        self.eta = self._ritz_eta()

    def solve(self, r):
        torch = self.ops._torch
        z = torch.zeros_like(r)
        for G, _, L in self.batches:
            z[G] = torch.cholesky_solve(r[G].unsqueeze(-1), L).squeeze(-1) / self.eta
        return z

    def apply(self, r):
        torch = self.ops._torch
        z = torch.zeros_like(r)
        for G, A, _ in self.batches:
            z[G] = self.eta * (A @ r[G].unsqueeze(-1)).squeeze(-1)
        return z

    def _ritz_eta(self) -> float:
        torch = self.ops._torch
        n = self.n
        i = torch.arange(n, dtype=torch.float64, device=self.ops.dev)
        r = 0.5 + 0.5 * torch.cos(3 * i + 1)
        z = self.solve(r)
        p = z.clone()
        rz = float(r @ z)
        alphas, betas = [], []
        for _ in range(10):
            ap = self._vdd(p)
            pap = float(p @ ap)
            if pap <= 0.0 or rz <= 0.0:
                break
            alpha = rz / pap
            r = r - alpha * ap
            z = self.solve(r)
            rz_new = float(r @ z)
            alphas.append(alpha)
            betas.append(rz_new / rz)
            rz = rz_new
            p = z + betas[-1] * p
            if np.sqrt(abs(rz)) < 1e-14:
                break
        if not alphas:
            return 1.0
        k = len(alphas)
        tri = np.zeros((k, k))
        for j in range(k):
            tri[j, j] = 1.0 / alphas[j] + (betas[j - 1] / alphas[j - 1] if j > 0 else 0.0)
            if j + 1 < k:
                off = np.sqrt(max(betas[j], 0.0)) / alphas[j]
                tri[j, j + 1] = tri[j + 1, j] = off
        lam = float(np.linalg.eigvalsh(tri).min())
        return 0.5 * lam if lam > 0 else 1.0


class DofLayout:
    """classify_dofs (mesh.cpp:278-293): the Dirichlet triangles (sorted)
    and the Neumann interior nodes (vertices none of whose triangles is
    Dirichlet), component-major DOF index sets (operators.cpp:160-176)."""

    def __init__(self, mesh: Mesh):
        a = mesh.arrays()
        T = a["triangles"]
        d = a["dirichlet"].astype(bool)
        self.num_triangles, self.num_nodes = len(T), len(a["vertices"])
        self.dirichlet_triangle_ids = np.nonzero(d)[0]
        touched = np.zeros(self.num_nodes, bool)
        touched[T.reshape(-1)] = True
        bad = np.zeros(self.num_nodes, bool)
        bad[T[d].reshape(-1)] = True
        self.neumann_interior_nodes = np.nonzero(touched & ~bad)[0]
        m, n = self.num_triangles, self.num_nodes
        self.t_dofs = np.concatenate([c * m + self.dirichlet_triangle_ids for c in range(3)])
        self.u_dofs = np.concatenate([c * n + self.neumann_interior_nodes for c in range(3)])


class SaddleSystem:
    """assemble_saddle (baca.cpp:12-40): the Lame saddle system
    [V_DD, -K_ND; K_ND^T, D_NN] over the Dirichlet-triangle and
    Neumann-node DOFs, as restrictions of the device compositions of
    OperatorSet (reduced to V_DD t = f_D when there is no Neumann node)."""

    def __init__(self, ops: "OperatorSet", layout: DofLayout):
        if len(layout.dirichlet_triangle_ids) == 0:
            raise Error("assemble_saddle: empty Dirichlet part")
        torch = ops._torch
        self.ops, self.layout = ops, layout
        self.t_idx = torch.tensor(layout.t_dofs, device=ops.dev)
        self.u_idx = torch.tensor(layout.u_dofs, device=ops.dev)
        self.nt, self.nu_ = len(layout.t_dofs), len(layout.u_dofs)
        self.reduced = self.nu_ == 0

    @property
    def dim(self) -> int:
        return self.nt + (0 if self.reduced else self.nu_)

    def _embed(self, v, idx, n):
        z = self.ops._torch.zeros(n, dtype=self.ops._torch.float64, device=self.ops.dev)
        z[idx] = v
        return z

    def vdd(self, xt):
        return self.ops.vh_dev(self._embed(xt, self.t_idx, 3 * self.ops.m))[self.t_idx]

    def knd(self, xu):
        return self.ops.kh_dev(self._embed(xu, self.u_idx, 3 * self.ops.n))[self.t_idx]

    def knd_t(self, zt):
        return self.ops.kh_t_dev(self._embed(zt, self.t_idx, 3 * self.ops.m))[self.u_idx]

    def dnn(self, xu):
        return self.ops.dh_dev(self._embed(xu, self.u_idx, 3 * self.ops.n))[self.u_idx]

    def a(self, x):
        """block2x2(vdd, knd, knd', dnn; 1, -1, 1, 1) applied to x = [t; u]."""
        if self.reduced:
            return self.vdd(x)
        xt, xu = x[:self.nt], x[self.nt:]
        return self.ops._torch.cat([self.vdd(xt) - self.knd(xu), self.knd_t(xt) + self.dnn(xu)])

    def preconditioner(self) -> VddPreconditioner:
        return VddPreconditioner(self.ops, self.layout.dirichlet_triangle_ids, self.vdd)

    def rhs(self, g_neumann, g_dirichlet):
        """assemble_rhs without AMVM (baca.cpp:42-76): the rows
        [Dirichlet triangles; Neumann nodes] of
        [-V_h, M/2 + K_h; M'/2 - K_h', -D_h] [g_N; g_D]."""
        ops, torch = self.ops, self.ops._torch
        gn = torch.tensor(np.asarray(g_neumann, dtype=np.float64), device=ops.dev)
        gd = torch.tensor(np.asarray(g_dirichlet, dtype=np.float64), device=ops.dev)
        if gn.shape[0] != 3 * ops.m or gd.shape[0] != 3 * ops.n:
            raise DimensionError("assemble_rhs: boundary data size")
        m, n = ops.m, ops.n
        mass_gd = torch.cat([ops._spmv(3, gd[c * n:(c + 1) * n]) for c in range(3)])
        mass_t_gn = torch.cat([ops._spmv(3, gn[c * m:(c + 1) * m], transpose=True)
                               for c in range(3)])
        top = -ops.vh_dev(gn) + (0.5 * mass_gd + ops.kh_dev(gd))
        bottom = (0.5 * mass_t_gn - ops.kh_t_dev(gn)) - ops.dh_dev(gd)
        f = torch.cat([top[self.t_idx], bottom[self.u_idx]])
        return f.cpu().numpy()


class SaddleEstimator:
    """estimator_Ek of the mixed system (baca.cpp:401-456) over the
    flattened leaf occurrences of V_DD, -K_ND, K_ND^T and D_NN
    (flatten_occurrences, expr.cpp:424-498): per occurrence the device
    computes every block's look-ahead tail (hmgpu_tail_terms / _t) on the
    occurrence's input (suffix x), the host maps it through the prefix (the
    restrictions, embeddings and T_h^T / S_k^T sandwiches, sparse) and sums
    it per (H-matrix, block) within each occurrence list
    (gamma_contributions, amvm.cpp:46-125); the K family merges the terms of
    -K_ND and K_ND^T by adding their norms (add_terms, baca.cpp:406-432)."""

    FAMILY = ("V", "K", "D")

    def __init__(self, sys: "SaddleSystem"):
        import scipy.sparse as sp
        self.sys = sys
        ops = sys.ops
        m, n = ops.m, ops.n
        L = sys.layout
        self.nt, self.nu = sys.nt, sys.nu_
        sel = lambda idx, N: sp.csr_matrix((np.ones(len(idx)), (np.arange(len(idx)), idx)),
                                           shape=(len(idx), N))
        self.St = sel(L.t_dofs, 3 * m)
        self.Su = sel(L.u_dofs, 3 * n)
        Tw = []
        for which in range(3):
            cols = np.zeros(3 * m, np.int32)
            vals = np.zeros(3 * m)
            _check(_h.hmb_sparse_op(ops._mesh._h, which, _ptr(cols), _ptr(vals)))
            Tw.append(sp.csr_matrix((vals, (np.repeat(np.arange(m), 3), cols)), shape=(m, n)))
        self.Tw = Tw
        Z = None
        blk = [[Z, Tw[0], Tw[1]], [-Tw[0], Z, Tw[2]], [-Tw[1], -Tw[2], Z]]
        self.Th = sp.bmat(blk, format="csr")
        self.Em = [sel(np.arange(m) + c * m, 3 * m).T.tocsr() for c in range(3)]  # 3m x m
        self.En = [sel(np.arange(n) + c * n, 3 * n).T.tocsr() for c in range(3)]  # 3n x n
        self.s = 0.5 / ops.E * (1.0 + ops.nu) / (1.0 - ops.nu)
        self.c34 = 3.0 - 4.0 * ops.nu
        self.mu = ops.mu

    # occurrence lists: (h, transposed, coeff, suffix, prefix); suffix /
    # prefix are sparse matrices (None = identity), h one of the contexts
    def _vh_occ(self, coeff, suffix, prefix):
        """the leaves of coeff * prefix V_h suffix (compose_Vh)."""
        o = [(self.sys.ops.vkl, False, coeff * self.s, suffix, prefix)]
        for c in range(3):
            sf = self.Em[c].T @ suffix
            pf = prefix @ self.Em[c]
            o.append((self.sys.ops.vdelta, False, coeff * self.s * self.c34, sf, pf))
        return o

    def _kh_occ(self, coeff, suffix, prefix):
        """the leaves of coeff * prefix K_h suffix (compose_Kh)."""
        ops = self.sys.ops
        o = []
        for c in range(3):
            o.append((ops.kdelta, False, coeff, self.En[c].T @ suffix, prefix @ self.Em[c]))
        for c in range(3):
            o.append((ops.vdelta, False, -coeff, self.Em[c].T @ self.Th @ suffix,
                      prefix @ self.Em[c]))
        o += self._vh_occ(2.0 * self.mu * coeff, self.Th @ suffix, prefix)
        return o

    def _dh_occ(self, suffix, prefix):
        ops, mu = self.sys.ops, self.mu
        o = []
        S = ((2, -1.0), (1, 1.0), (0, 1.0))
        for (w, a) in S:
            for c in range(3):
                o.append((ops.vdelta, False, mu, a * self.Tw[w] @ self.En[c].T @ suffix,
                          prefix @ self.En[c] @ (a * self.Tw[w].T)))
        for c in range(3):
            o.append((ops.vdelta, False, 2.0 * mu, self.Em[c].T @ self.Th @ suffix,
                      prefix @ self.Th.T @ self.Em[c]))
        o += self._vh_occ(-4.0 * mu * mu, self.Th @ suffix, prefix @ self.Th.T)
        ts = lambda k, l: None if k == l else ({(0, 1): 0, (0, 2): 1, (1, 2): 2}[
            (min(k, l), max(k, l))], 1.0 if k < l else -1.0)
        for i in range(3):
            for j in range(3):
                for k in range(3):
                    tkj, tki = ts(k, j), ts(k, i)
                    if tkj is None or tki is None:
                        continue
                    o.append((ops.vdelta, False, mu * tkj[1] * tki[1],
                              self.Tw[tki[0]] @ self.En[j].T @ suffix,
                              prefix @ self.En[i] @ self.Tw[tkj[0]].T))
        return o

    @staticmethod
    def _transpose(occ):
        return [(h, not tr, c, pf.T.tocsr(), sf.T.tocsr()) for (h, tr, c, sf, pf) in occ]

    def _gamma(self, occ, x, out_dim):
        """gamma_contributions over an occurrence list: {(h, comp, block):
        dense vector over out_dim}, grouped by H-matrix (first appearance)."""
        acc = {}
        for (h, tr, coeff, suffix, prefix) in occ:
            xin = suffix @ x
            g = h.gamma_contributions(xin, term_data=True, transposed=tr)
            for t in g.terms:
                v = prefix[:, t.idx] @ (coeff * t.val)
                key = (id(h), t.comp, t.block)
                if key not in acc:
                    acc[key] = (h, np.zeros(out_dim))
                acc[key][1][:] += v
        return acc

    def estimate(self, x):
        """(E_k, terms [(family, h, comp, block, norm_sq)], diff over [t; u])."""
        import scipy.sparse as sp
        nt, nu = self.nt, self.nu
        x = np.asarray(x, dtype=np.float64)
        xt, xu = x[:nt], x[nt:]
        diff = np.zeros(nt + nu)
        terms = []
        vdd = self._vh_occ(1.0, self.St.T.tocsr(), self.St)
        for key, (h, v) in self._gamma(vdd, xt, nt).items():
            terms.append(("V", h, key[1], key[2], float(v @ v)))
            diff[:nt] += v
        if nu:
            knd = self._kh_occ(1.0, self.Su.T.tocsr(), self.St)
            k12 = [(h, tr, -c, sf, pf) for (h, tr, c, sf, pf) in knd]
            k21 = self._transpose(knd)
            kt = {}
            for key, (h, v) in self._gamma(k12, xu, nt).items():
                kt[key] = ["K", h, key[1], key[2], float(v @ v)]
                diff[:nt] += v
            for key, (h, v) in self._gamma(k21, xt, nu).items():
                if key in kt:
                    kt[key][4] += float(v @ v)
                else:
                    kt[key] = ["K", h, key[1], key[2], float(v @ v)]
                diff[nt:] += v
            terms += [tuple(t) for t in kt.values()]
            dnn = self._dh_occ(self.Su.T.tocsr(), self.Su)
            for key, (h, v) in self._gamma(dnn, xu, nu).items():
                terms.append(("D", h, key[1], key[2], float(v @ v)))
                diff[nt:] += v
        ek = float(np.sqrt(sum(t[4] for t in terms)))
        return ek, terms, diff


def amvm_multiply_occurrences(occurrences, matvec, x, out_dim: int, n_cols: int,
                              cfg: Optional[AmvmConfig] = None, h_order=None, **kw):
    """amvm_multiply (amvm.cpp:199-268) over an operator EXPRESSION given by
    its flattened H-leaf occurrences (flatten_occurrences, expr.cpp:424-510):
    occurrences = [(h, transposed, coeff, suffix, prefix)] with h an HMatrix
    context (every component of a grid context is one H-matrix of the
    reference), suffix / prefix sparse (None = identity); matvec(x) the
    expression's product at the current ranks (numpy in / out).  Per sweep:
    gamma_contributions over the occurrences (amvm.cpp:46-125: every
    occurrence's device look-ahead tail on suffix x, mapped through prefix and
    coeff, summed per (H-matrix, block), terms grouped by H-matrix in
    h_order (the expression's first-appearance order, (context, comp) pairs;
    default: the order of the occurrence list) then block), the marking walk
    (mark_blocks, amvm.cpp:131-184, on the library's host walk), promotion +
    look-ahead extension of the marked blocks on the device, and the
    product again.  Returns (b, AmvmReport)."""
    import time as _time
    cfg = cfg or AmvmConfig(**kw)
    if not 0.0 < cfg.theta < 1.0:
        raise ConfigError("amvm_multiply: theta must lie in (0,1)")
    if cfg.eps_amvm <= 0.0:
        raise ConfigError("amvm_multiply: eps_amvm must be positive")
    if cfg.max_iterations < 0:
        raise ConfigError("amvm_multiply: max_iterations must be >= 0")
    x = _f64(x)
    if x.shape != (n_cols,):
        raise DimensionError("amvm_multiply: size")
    ctxs = []
    for o in occurrences:
        if all(o[0] is not h for h in ctxs):
            ctxs.append(o[0])
    if h_order is None:
        h_order = [(h, q) for h in ctxs for q in range(6 if h.ncomp == 6 else 1)]
    rank_of = {(id(h), q): i for i, (h, q) in enumerate(h_order)}
    # operator_sparsity_constant: the largest c_sp over the distinct partitions
    c_sp = max([1] + [h.sparsity_constant for h in ctxs])

    def one_world(send, recv):
        recv[:] = send

    def estimate():
        # per (H-matrix, block): the contributions of its occurrences in
        # occurrence order, (output index, value) pairs -- the Accum of
        # amvm.cpp:14-41, summed per index in that order (np.add.at is
        # unbuffered and runs in input order)
        acc = {}
        for (h, tr, coeff, suffix, prefix) in occurrences:
            xin = x if suffix is None else suffix @ x
            g = h.gamma_contributions(xin, term_data=True, transposed=tr)
            for t in g.terms:
                w = coeff * np.asarray(t.val)
                if prefix is None:
                    idx, val = np.asarray(t.idx, np.int64), w
                else:
                    # prefix column by column (block rows ascending), each
                    # column's nonzeros in row order: value * (coeff * y_r)
                    sub = prefix[:, t.idx].tocoo()
                    o = np.lexsort((sub.row, sub.col))
                    idx = sub.row[o].astype(np.int64)
                    val = sub.data[o] * w[sub.col[o]]
                    keep = w[sub.col[o]] != 0.0
                    idx, val = idx[keep], val[keep]
                key = (rank_of[(id(h), t.comp)], t.block)
                if key not in acc:
                    acc[key] = (h, t.comp, t.block, [], [])
                acc[key][3].append(idx)
                acc[key][4].append(val)
        terms = []
        diff = np.zeros(out_dim)
        for key in sorted(acc):
            h, comp, block, il, vl = acc[key]
            ci, cv = np.concatenate(il), np.concatenate(vl)
            if len(ci) == 0:
                continue
            uniq, inv = np.unique(ci, return_inverse=True)
            v = np.zeros(len(uniq))
            np.add.at(v, inv, cv)
            terms.append(BlockTerm(comp, block, uniq.astype(np.int64), v,
                                   float(np.cumsum(v * v)[-1])))
            terms[-1].ctx = h
            diff[uniq] += v  # term by term, as amvm.cpp:111-115
        return terms, diff
    t_start = _time.perf_counter()
    b = _f64(matvec(x))
    b_hat_prev = None
    its = []
    for k in range(cfg.max_iterations + 1):
        t0 = _time.perf_counter()
        terms, diff = estimate()
        # sequential sum in row order (difference.norm(), amvm.cpp:124);
        # numpy's sum is pairwise
        gamma = float(np.sqrt(np.cumsum(diff * diff)[-1])) if out_dim else 0.0
        if b_hat_prev is not None:
            its[-1].e_hat = float(np.linalg.norm(b + diff - b_hat_prev))
        pivots = sum(h.total_pivots() for h in ctxs)
        storage = sum(h.storage_mb_current() for h in ctxs)
        it = AmvmIteration(k, gamma, 0.0, 0, pivots, storage, -1.0, 0.0)
        if gamma <= cfg.eps_amvm or k >= cfg.max_iterations:
            it.ms = 1e3 * (_time.perf_counter() - t0)
            its.append(it)
            conv = gamma <= cfg.eps_amvm
            return b, AmvmReport(its, "tolerance" if conv else "max_iterations", conv, c_sp)
        marked, n_marked, gpk = mark_blocks_sharded(terms, diff, np.ones(out_dim, bool),
                                                    cfg.theta, c_sp, out_dim, n_cols, 1, 0,
                                                    one_world)
        it.gamma_pk, it.marked = gpk, n_marked
        b_hat_prev = b + diff
        by_ctx = {}
        for t in marked:
            by_ctx.setdefault(id(terms[t].ctx), (terms[t].ctx, []))[1].append(
                (terms[t].comp, terms[t].block))
        for h, pairs in by_ctx.values():
            h.promote(pairs)
            h.extend_lookahead(pairs, cfg.lookahead_steps)
        b = _f64(matvec(x))
        it.ms = 1e3 * (_time.perf_counter() - t0)
        its.append(it)
    raise AssertionError("unreachable")


def rhs_occurrences(sys: "SaddleSystem"):
    """The flattened H-leaf occurrences of rhs_operator (baca.cpp:42-55):
    rows [Dirichlet-triangle dofs; Neumann-node dofs] of
    [-V_h, M/2 + K_h; M'/2 - K_h', -D_h] over x = [g_N; g_D] (the mass
    matrix is sparse and carries no H-leaf), and the H-matrices in the
    expression's first-appearance order: V_Delta (in -V_h's diag3), the six
    V_kl components, K_Delta."""
    import scipy.sparse as sp
    est = SaddleEstimator(sys)
    ops = sys.ops
    m3, n3 = 3 * ops.m, 3 * ops.n
    nt, nu = sys.nt, sys.nu_
    out = nt + nu
    P0 = sp.vstack([est.St, sp.csr_matrix((nu, m3))]).tocsr()        # top rows
    P1 = sp.vstack([sp.csr_matrix((nt, n3)), est.Su]).tocsr()        # bottom rows
    Rn = sp.hstack([sp.identity(m3), sp.csr_matrix((m3, n3))]).tocsr()  # g_N
    Rd = sp.hstack([sp.csr_matrix((n3, m3)), sp.identity(n3)]).tocsr()  # g_D
    neg = lambda occ: [(h, tr, -c, sf, pf) for (h, tr, c, sf, pf) in occ]
    occ = neg(est._vh_occ(1.0, Rn, P0))                                # -V_h g_N
    occ += est._kh_occ(1.0, Rd, P0)                                    # +K_h g_D
    occ += est._transpose(neg(est._kh_occ(1.0, P1.T.tocsr(), Rn.T.tocsr())))  # -K_h' g_N
    occ += neg(est._dh_occ(Rd, P1))                                    # -D_h g_D
    order = [(ops.vdelta, 0)] + [(ops.vkl, q) for q in range(6)] + [(ops.kdelta, 0)]
    return occ, order, out, m3 + n3


def assemble_rhs(sys: "SaddleSystem", g_neumann, g_dirichlet, amvm: bool = False,
                 amvm_cfg: Optional[AmvmConfig] = None):
    """assemble_rhs (baca.cpp:57-76): f = rhs_operator [g_N; g_D], through the
    adaptive matvec over the composite operator when amvm is set (the paper's
    Table 3 workload).  Returns (f, AmvmReport or None)."""
    gn = _f64(g_neumann)
    gd = _f64(g_dirichlet)
    if gn.shape != (3 * sys.ops.m,) or gd.shape != (3 * sys.ops.n,):
        raise DimensionError("assemble_rhs: boundary data size")
    if not amvm:
        return sys.rhs(gn, gd), None
    occ, order, out, ncols = rhs_occurrences(sys)
    m3 = 3 * sys.ops.m
    return amvm_multiply_occurrences(occ, lambda v: sys.rhs(v[:m3], v[m3:]),
                                     np.concatenate([gn, gd]), out, ncols,
                                     amvm_cfg or AmvmConfig(), h_order=order)


def baca_solve_saddle(sys: "SaddleSystem", f, cfg: Optional[BacaConfig] = None):
    """baca_solve (baca.cpp:488-600) for the mixed system: BPCG under the
    adaptive accuracy condition, E_k over the V / K / D families, Doerfler
    marking, and the refinement in the operator order -- (1) D_NN wholly,
    (2) V_DD wholly plus the marked K blocks, (3) else the marked V blocks --
    by promotion + look-ahead extension on the device.  Returns (x, report)
    with per-sweep records (k, ek, tail_norm, residual, inner_tol,
    inner_iterations, marked per family, phases)."""
    import time as _time
    cfg = cfg or BacaConfig()
    if not 0.0 < cfg.theta < 1.0:
        raise Error("baca_solve: theta must lie in (0,1)")
    f = np.asarray(f, dtype=np.float64)
    if f.shape != (sys.dim,):
        raise DimensionError("baca_solve: rhs size")
    ops = sys.ops
    est = SaddleEstimator(sys)
    prec = sys.preconditioner()
    fnorm = float(np.linalg.norm(f))
    floor_abs = cfg.inner_floor * max(fnorm, 1e-300)
    x = np.zeros(sys.dim)
    tol_abs = max(cfg.inner_tol0 * fnorm, floor_abs)
    t0 = _time.perf_counter()
    its = []

    def all_blocks(h):  # every low-rank (comp, block) of a context
        kc = h.ranks()[0]
        return [(q, b) for q in range(kc.shape[0]) for b in range(kc.shape[1]) if kc[q, b] >= 0]

    for k in range(cfg.max_outer + 1):
        inner, used_fb = 0, False
        for _ in range(6):
            x, st = bpcg_solve(sys, prec, f, tol_abs, x)
            inner += st.iterations
            used_fb = used_fb or st.used_fallback
            ek, terms, diff = est.estimate(x)
            tail = float(np.linalg.norm(diff))
            cond = cfg.alpha * tail
            if st.residual <= max(cond, floor_abs):
                break
            tol_abs = max(cond, floor_abs)
        it = dict(k=k, ek=ek, tail_norm=tail, residual=st.residual, inner_tol=tol_abs,
                  inner_iterations=inner, used_fallback=used_fb, marked_v=0, marked_k=0,
                  marked_d=0, phases=[], wall_time_s=_time.perf_counter() - t0)
        if ek <= cfg.eps_baca:
            its.append(it)
            return x, BacaReport(its, True, "tolerance")
        if k >= cfg.max_outer:
            its.append(it)
            return x, BacaReport(its, False, "max_outer")
        order = sorted(range(len(terms)), key=lambda i: -terms[i][4])
        target = cfg.theta * cfg.theta * ek * ek
        marked, acc = [], 0.0
        for i in order:
            if acc >= target:
                break
            marked.append(i)
            acc += terms[i][4]
        fams = [terms[i][0] for i in marked]
        it["marked_v"], it["marked_k"], it["marked_d"] = (fams.count("V"), fams.count("K"),
                                                          fams.count("D"))
        promo = {}
        def add(h, comp, block):
            promo.setdefault(id(h), (h, set()))[1].add((comp, block))
        def add_all(hs):
            for h in hs:
                for (q, b) in all_blocks(h):
                    add(h, q, b)
        if it["marked_d"]:
            it["phases"].append(1)
            add_all([ops.vdelta, ops.vkl])  # the leaves of D_NN
        if it["marked_k"]:
            it["phases"].append(2)
            add_all([ops.vdelta, ops.vkl])  # V_DD wholly
            for i in marked:
                if terms[i][0] == "K":
                    add(terms[i][1], terms[i][2], terms[i][3])
        if not it["marked_d"] and not it["marked_k"]:
            it["phases"].append(3)
            for i in marked:
                add(terms[i][1], terms[i][2], terms[i][3])
        for (h, pairs) in promo.values():
            pairs = sorted(pairs)
            h.promote(pairs)
            h.extend_lookahead(pairs, cfg.lookahead_steps)
        its.append(it)
        tol_abs = max(tol_abs, floor_abs)
    return x, BacaReport(its, False, "max_outer")


@dataclasses.dataclass
class SolveStats:  # baca.hpp:91-96
    iterations: int = 0
    converged: bool = False
    used_fallback: bool = False
    residual: float = 0.0


def _bpcg_core(sys: SaddleSystem, prec: VddPreconditioner, f, tol_abs, x0, max_iter):
    """Bramble-Pasciak CG (baca.cpp:294-366) on [V, -K; -K', -D] with the
    left transform P^{-1} = [C^{-1}, 0; -K' C^{-1}, -I] and the inner
    product <x, y> = ((V - C) x_1, y_1) + x_2 . y_2."""
    nt = sys.nt
    torch = sys.ops._torch

    def abar(v):
        s = sys.a(v)
        return torch.cat([s[:nt], -s[nt:]])

    def ptrans(r):
        z1 = prec.solve(r[:nt])
        return torch.cat([z1, -sys.knd_t(z1) - r[nt:]])

    def h_dot(a, b, v_a1):
        return float(v_a1 @ b[:nt]) - float(prec.apply(a[:nt]) @ b[:nt]) + float(a[nt:] @ b[nt:])

    bbar = torch.cat([f[:nt], -f[nt:]])
    x = x0.clone()
    r_orig = bbar - abar(x)
    rhat = ptrans(r_orig)
    p = rhat.clone()
    v_rhat1 = sys.vdd(rhat[:nt])
    rho = h_dot(rhat, rhat, v_rhat1)
    st = SolveStats()
    if rho < 0:
        return x, st, True
    while float(r_orig.norm()) > tol_abs and st.iterations < max_iter:
        ap = abar(p)
        q = ptrans(ap)
        v_q1 = sys.vdd(q[:nt])
        denom = h_dot(q, p, v_q1)
        if denom <= 0:
            return x, st, True
        alpha = rho / denom
        x = x + alpha * p
        r_orig = r_orig - alpha * ap
        rhat = rhat - alpha * q
        v_rhat1 = v_rhat1 - alpha * v_q1
        rho_new = h_dot(rhat, rhat, v_rhat1)
        if rho_new < 0:
            return x, st, True
        p = rhat + (rho_new / rho) * p
        rho = rho_new
        st.iterations += 1
    st.residual = float(r_orig.norm())
    st.converged = st.residual <= tol_abs
    return x, st, False


def _minres(sys: SaddleSystem, prec: VddPreconditioner, f, tol_abs, x0, max_iter):
    """Preconditioned MINRES on the symmetric form [-V, K; K', D]
    (baca.cpp:227-292), the fallback solver."""
    nt = sys.nt
    torch = sys.ops._torch

    def sym(v):
        s = sys.a(v)
        return torch.cat([-s[:nt], s[nt:]])

    def pre(v):
        return torch.cat([prec.solve(v[:nt]), v[nt:]])

    b = torch.cat([-f[:nt], f[nt:]])
    x = x0.clone()
    r1 = b - sym(x)
    y = pre(r1)
    beta1 = float(r1 @ y)
    st = SolveStats()
    if beta1 < 0:
        raise Error("minres: preconditioner not positive definite")
    if beta1 == 0:
        st.converged = True
        return x, st
    beta1 = np.sqrt(beta1)
    eps_ln = dbar = oldb = 0.0
    beta = phibar = beta1
    cs, sn = -1.0, 0.0
    r2 = r1.clone()
    w = torch.zeros_like(x)
    w2 = torch.zeros_like(x)
    it = 0
    while it < max_iter and phibar > tol_abs:
        v = y / beta
        y = sym(v)
        if it > 0:
            y = y - (beta / oldb) * r1
        alfa = float(v @ y)
        y = y - (alfa / beta) * r2
        r1, r2 = r2, y
        y = pre(r2)
        oldb = beta
        beta_sq = float(r2 @ y)
        if beta_sq < 0:
            raise Error("minres: preconditioner breakdown")
        beta = np.sqrt(beta_sq)
        oldeps = eps_ln
        delta = cs * dbar + sn * alfa
        gbar = sn * dbar - cs * alfa
        eps_ln = sn * beta
        dbar = -cs * beta
        gamma = max(np.sqrt(gbar * gbar + beta * beta), 1e-30)
        cs, sn = gbar / gamma, beta / gamma
        phi = cs * phibar
        phibar = sn * phibar
        w1, w2 = w2, w
        w = (v - oldeps * w1 - delta * w2) / gamma
        x = x + phi * w
        it += 1
    st.iterations = it
    st.residual = float((f - sys.a(x)).norm())
    st.converged = st.residual <= tol_abs * 1.5
    return x, st


def bpcg_solve(sys: SaddleSystem, prec: VddPreconditioner, f, tol_abs: float, x0=None,
               use_bpcg: bool = True, max_iter: int = 10000):
    """bpcg_solve (baca.cpp:368-399): PCG in reduced mode, else
    Bramble-Pasciak CG with the MINRES fallback on breakdown.  Device
    vectors inside; f / x0 / result as numpy arrays.  Returns (x, stats)."""
    torch = sys.ops._torch
    f = np.asarray(f, dtype=np.float64)
    if f.shape != (sys.dim,):
        raise DimensionError("bpcg_solve: rhs size")
    if np.linalg.norm(f) == 0.0:
        return np.zeros(sys.dim), SolveStats(0, True, False, 0.0)
    fd = torch.tensor(f, device=sys.ops.dev)
    xd = torch.zeros_like(fd) if x0 is None else torch.tensor(np.asarray(x0, dtype=np.float64),
                                                               device=sys.ops.dev)
    if sys.reduced:
        x, it, res = _pcg(sys.vdd, prec, fd, tol_abs, xd, max_iter)
        return x.cpu().numpy(), SolveStats(it, res <= tol_abs, False, res)
    if use_bpcg:
        x, st, breakdown = _bpcg_core(sys, prec, fd, tol_abs, xd, max_iter)
        if not breakdown:
            return x.cpu().numpy(), st
        y, st2 = _minres(sys, prec, fd, tol_abs, x, max_iter)
        st2.iterations += st.iterations
        st2.used_fallback = True
        return y.cpu().numpy(), st2
    x, st = _minres(sys, prec, fd, tol_abs, xd, max_iter)
    return x.cpu().numpy(), st


def _pcg(apply_a, prec: VddPreconditioner, f, tol_abs: float, x0, max_iter: int):
    x = x0.clone()
    r = f - apply_a(x)
    z = prec.solve(r)
    p = z.clone()
    rz = float(r @ z)
    it = 0
    while float(r.norm()) > tol_abs and it < max_iter:
        ap = apply_a(p)
        alpha = rz / float(p @ ap)
        x = x + alpha * p
        r = r - alpha * ap
        z = prec.solve(r)
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
        it += 1
    return x, it, float(r.norm())


def pcg_spd(ops: "OperatorSet", prec: VddPreconditioner, f, tol_abs: float, x0, max_iter: int):
    """Preconditioned CG on V_h x = f (pcg_spd, baca.cpp:200-225); device vectors."""
    x = x0.clone()
    r = f - ops.vh_dev(x)
    z = prec.solve(r)
    p = z.clone()
    rz = float(r @ z)
    it = 0
    while float(r.norm()) > tol_abs and it < max_iter:
        ap = ops.vh_dev(p)
        alpha = rz / float(p @ ap)
        x = x + alpha * p
        r = r - alpha * ap
        z = prec.solve(r)
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
        it += 1
    res = float(r.norm())
    return x, it, res


def estimator_vh(ops: "OperatorSet", x):
    """estimator_Ek of the reduced system (baca.cpp:401-456): the look-ahead
    tail terms of V_h's leaf occurrences -- each V_kl block (grid embedding)
    scaled by (1+nu)/(2E(1-nu)), each V_Delta block over its three diag3
    occurrences scaled by that times (3-4nu) -- one term per (H-matrix,
    block); E_k = sqrt(sum of the terms' norm_sq), diff = sum of the terms."""
    m = ops.m
    pref = 0.5 / ops.E * (1.0 + ops.nu) / (1.0 - ops.nu)
    sd = pref * (3.0 - 4.0 * ops.nu)
    xh = x.detach().cpu().numpy() if hasattr(x, "detach") else np.asarray(x)
    # the scales enter linearly (diff) and squared (norm_sq), so only the
    # per-context difference vectors and term norms are downloaded
    terms = []  # (h, comp, block, norm_sq)
    g = ops.vkl.gamma_contributions(xh, term_data=False)
    diff = pref * g.difference
    for t in g.terms:
        terms.append((ops.vkl, t.comp, t.block, pref * pref * t.norm_sq))
    per_block = {}
    for c in range(3):
        gd = ops.vdelta.gamma_contributions(xh[c * m:(c + 1) * m], term_data=False)
        diff[c * m:(c + 1) * m] += sd * gd.difference
        for t in gd.terms:
            per_block[t.block] = per_block.get(t.block, 0.0) + sd * sd * t.norm_sq
    for b in sorted(per_block):
        terms.append((ops.vdelta, 0, b, per_block[b]))
    ek = float(np.sqrt(sum(t[3] for t in terms)))
    return ek, terms, diff


def doerfler_mark(terms, ek: float, theta: float):
    """Minimal greedy Doerfler set (baca.cpp:458-476)."""
    order = sorted(range(len(terms)), key=lambda i: -terms[i][3])  # stable
    target = theta * theta * ek * ek
    marked, acc = [], 0.0
    for i in order:
        if acc >= target:
            break
        marked.append(i)
        acc += terms[i][3]
    return marked


def baca_solve(ops: "OperatorSet", f, cfg: Optional[BacaConfig] = None):
    """baca_solve (baca.cpp:488-600) for the reduced all-Dirichlet system
    V_h t = f: inner PCG under ||f - A_k x|| <= alpha ||(A_k - A_hat_k) x||,
    estimator E_k, Doerfler marking (theta), promotion + look-ahead
    extension of the marked blocks (phase 3 of the reference).  All
    H-matrix work runs on the device.  Returns (x, BacaReport)."""
    import time as _time
    torch = ops._torch
    cfg = cfg or BacaConfig()
    if not 0.0 < cfg.theta < 1.0:
        raise Error("baca_solve: theta must lie in (0,1)")
    f = np.asarray(f, dtype=np.float64)
    if f.shape != (3 * ops.m,):
        raise DimensionError("baca_solve: rhs size")
    fd = torch.tensor(f, device=ops.dev)
    prec = VddPreconditioner(ops)
    fnorm = float(np.linalg.norm(f))
    floor_abs = cfg.inner_floor * max(fnorm, 1e-300)
    x = torch.zeros_like(fd)
    tol_abs = max(cfg.inner_tol0 * fnorm, floor_abs)
    t0 = _time.perf_counter()
    its = []
    for k in range(cfg.max_outer + 1):
        inner = 0
        for _ in range(6):
            x, n_it, res = pcg_spd(ops, prec, fd, tol_abs, x, cfg.max_inner)
            inner += n_it
            ek, terms, diff = estimator_vh(ops, x)
            tail = float(np.linalg.norm(diff))
            cond = cfg.alpha * tail
            if res <= max(cond, floor_abs):
                break
            tol_abs = max(cond, floor_abs)
        storage = (ops.vkl.storage_mb_current() + ops.vdelta.storage_mb_current())
        it = BacaIteration(k, ek, tail, res, tol_abs, inner, 0, storage,
                           _time.perf_counter() - t0)
        if ek <= cfg.eps_baca:
            its.append(it)
            return x.cpu().numpy(), BacaReport(its, True, "tolerance")
        if k >= cfg.max_outer:
            its.append(it)
            return x.cpu().numpy(), BacaReport(its, False, "max_outer")
        marked = doerfler_mark(terms, ek, cfg.theta)
        it.marked_v = len(marked)
        for h in (ops.vkl, ops.vdelta):
            pairs = [(terms[i][1], terms[i][2]) for i in marked if terms[i][0] is h]
            if pairs:
                h.promote(pairs)
                h.extend_lookahead(pairs, cfg.lookahead_steps)
        its.append(it)
        tol_abs = max(tol_abs, floor_abs)
    return x.cpu().numpy(), BacaReport(its, False, "max_outer")


def random_vector(n: int, seed: int, kind: str = "uniform") -> np.ndarray:
    """Seeded synthetic input: mt19937_64 + uniform [-1,1) (the reference's
    random_vector) or standard normal."""
    out = np.zeros(n)
    _check(_h.hmb_random_vector(n, seed, 0 if kind == "uniform" else 1, _ptr(out)))
    return out


def dmma_peak_tflops(device: int = 0) -> float:
    """Measured fp64 tensor-core (DMMA) throughput of the device: the roofline
    denominator of the multi-RHS sweep."""
    v = C.c_double()
    st = _lib.gpu.hmgpu_dmma_peak(device, C.byref(v))
    if st:
        raise DeviceError("hmgpu_dmma_peak failed", st)
    return v.value


def dmma_peak_sustained_tflops(device: int = 0, seconds: float = 1.0) -> float:
    """DMMA throughput over the second half of `seconds` of back-to-back
    launches: the rate at the clocks the power limit settles on."""
    v = C.c_double()
    st = _lib.gpu.hmgpu_dmma_peak_sustained(device, float(seconds), C.byref(v))
    if st:
        raise DeviceError("hmgpu_dmma_peak_sustained failed", st)
    return v.value


def fp64_peak_tflops(device: int = 0) -> float:
    """Measured DFMA throughput of the device (fp64 roofline denominator)."""
    v = C.c_double()
    st = _lib.gpu.hmgpu_fp64_peak(device, C.byref(v))
    if st:
        raise DeviceError("hmgpu_fp64_peak failed", st)
    return v.value


def gauss_rule(order: int):
    """(a, b, w) of the symmetric triangle rule (quadrature.cpp:55-95)."""
    n = C.c_int()
    _check(_h.hmb_gauss_rule(order, C.byref(n), None, None, None))
    a, b, w = np.zeros(n.value), np.zeros(n.value), np.zeros(n.value)
    _check(_h.hmb_gauss_rule(order, C.byref(n), _ptr(a), _ptr(b), _ptr(w)))
    return a, b, w


def admissible(box_t, box_s, eta: float) -> bool:
    """min(diam t, diam s) < eta * dist(t, s) on [lo, hi] boxes (cluster.cpp:21-24)."""
    a = _f64(box_t).reshape(6)
    b = _f64(box_s).reshape(6)
    out = C.c_int()
    _check(_h.hmb_admissible(_ptr(a), _ptr(b), eta, C.byref(out)))
    return bool(out.value)


def assemble(h: HMatrix, cfg: AssemblyConfig) -> HMatrix:
    h.assemble(cfg)
    return h


def gamma_contributions(h: HMatrix, x) -> GammaContributions:
    return h.gamma_contributions(x)


def amvm_multiply(h: HMatrix, x, cfg: AmvmConfig):
    return h.amvm_multiply(x, cfg)


def host_tree_and_partition(mesh: Mesh, b_min: int, eta: float):
    """Cluster tree + partition without touching a GPU (device = -1)."""
    return HMatrix.kelvin(mesh, b_min=b_min, eta=eta, device=-1)
