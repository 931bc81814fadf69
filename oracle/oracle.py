"""ctypes wrapper of the CPU oracle (oracle/build/libhmbem_oracle.so).

TEST INFRASTRUCTURE ONLY: used by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py as the checker and the
timed CPU baseline.  The product package never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "libhmbem_oracle.so")


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "hmbem_oracle.cpp")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(src) > os.path.getmtime(LIB_PATH):
        subprocess.run(["make", "-C", HERE, "-B" if force else "-s"], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.or_last_error.restype = C.c_char_p
        L.or_set_threads.argtypes = [C.c_int]
        L.or_problem_free.argtypes = [C.c_void_p]
        L.or_aca_dense_free.argtypes = [C.c_void_p]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def _ck(st: int) -> None:
    if st != 0:
        raise OracleError(lib().or_last_error().decode())


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


D = C.c_double


def set_threads(n: int) -> None:
    lib().or_set_threads(n)


def gauss_rule(order: int):
    n = C.c_int()
    _ck(lib().or_gauss_rule(order, C.byref(n), None, None, None))
    a, b, w = np.zeros(n.value), np.zeros(n.value), np.zeros(n.value)
    _ck(lib().or_gauss_rule(order, C.byref(n), _p(a), _p(b), _p(w)))
    return a, b, w


def gauss_legendre_01(n: int):
    x, w = np.zeros(n), np.zeros(n)
    _ck(lib().or_gauss_legendre_01(n, _p(x), _p(w)))
    return x, w


def lame_constants(E: float, nu: float):
    lam, mu = D(), D()
    _ck(lib().or_lame_constants(D(E), D(nu), C.byref(lam), C.byref(mu)))
    return lam.value, mu.value


def kelvin_tensor(x, E=1.0, nu=0.3) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros(9)
    _ck(lib().or_kelvin_tensor(_p(x), D(E), D(nu), _p(out)))
    return out.reshape(3, 3)


def voxel_surface(n: int, lo: float, hi: float):
    nv, nt = C.c_int(), C.c_int()
    _ck(lib().or_voxel_surface(n, D(lo), D(hi), C.byref(nv), C.byref(nt), None, None))
    v = np.zeros((nv.value, 3))
    t = np.zeros((nt.value, 3), np.int32)
    _ck(lib().or_voxel_surface(n, D(lo), D(hi), C.byref(nv), C.byref(nt), _p(v), _p(t)))
    return v, t


def ellipsoid(level: int, ax: float = 1.0, ay: float = 1.0, az: float = 1.0):
    """icosphere (semi-axes 1) or ellipsoid mesh: (vertices, triangles)"""
    nv, nt = C.c_int(), C.c_int()
    _ck(lib().or_ellipsoid(level, D(ax), D(ay), D(az), C.byref(nv), C.byref(nt), None, None))
    v = np.zeros((nv.value, 3))
    t = np.zeros((nt.value, 3), np.int32)
    _ck(lib().or_ellipsoid(level, D(ax), D(ay), D(az), C.byref(nv), C.byref(nt), _p(v), _p(t)))
    return v, t


def icosphere(level: int):
    return ellipsoid(level)


def mesh_geometry(verts, tris):
    v = np.ascontiguousarray(verts, dtype=np.float64)
    t = np.ascontiguousarray(tris, dtype=np.int32)
    nt = len(t)
    cen, nrm = np.zeros((nt, 3)), np.zeros((nt, 3))
    area, diam = np.zeros(nt), np.zeros(nt)
    _ck(lib().or_mesh_geometry(len(v), _p(v), nt, _p(t), _p(cen), _p(area), _p(nrm), _p(diam)))
    return dict(centroids=cen, areas=area, normals=nrm, diam=diam)


def random_vector(n: int, seed: int) -> np.ndarray:
    out = np.zeros(n)
    _ck(lib().or_random_vector(C.c_long(n), C.c_uint(seed), _p(out)))
    return out


def normal_vector(n: int, seed: int) -> np.ndarray:
    out = np.zeros(n)
    _ck(lib().or_normal_vector(C.c_long(n), C.c_ulong(seed), _p(out)))
    return out


def self_term_i1(v9, p) -> float:
    v9 = np.ascontiguousarray(v9, dtype=np.float64).reshape(9)
    p = np.ascontiguousarray(p, dtype=np.float64)
    out = D()
    _ck(lib().or_analytic_potential_self(_p(v9), _p(p), C.byref(out)))
    return out.value


def pair_rule(case: int, order: int):
    """pair_rule(PairCase, order) (quadrature.cpp:290-338); case 0 disjoint,
    1 vertex, 2 edge, 3 identical.  Returns xr1, xr2, yr1, yr2, w."""
    n = C.c_int()
    _ck(lib().or_pair_rule(case, order, C.byref(n), None, None, None, None, None))
    arr = [np.zeros(n.value) for _ in range(5)]
    _ck(lib().or_pair_rule(case, order, C.byref(n), *[_p(a) for a in arr]))
    return tuple(arr)


def sparse_op(verts, tris, which: int) -> np.ndarray:
    """build_sparse_ops (operators.cpp:7-95) as a dense n_tri x n_vert
    matrix: which 0 T12, 1 T13, 2 T23, 3 mass."""
    v = np.ascontiguousarray(verts, dtype=np.float64)
    t = np.ascontiguousarray(tris, dtype=np.int32)
    out = np.zeros((len(t), len(v)))
    _ck(lib().or_sparse_op(len(v), _p(v), len(t), _p(t), int(which), _p(out)))
    return out


def classify_pair(a, b):
    """classify_pair + test/trial vertex perms (quadrature.cpp:127-166)."""
    a = np.ascontiguousarray(a, dtype=np.int32)
    b = np.ascontiguousarray(b, dtype=np.int32)
    ra, rb = C.c_int(), C.c_int()
    pa, pb = np.zeros(3, np.int32), np.zeros(3, np.int32)
    _ck(lib().or_classify_pair(_p(a), _p(b), C.byref(ra), C.byref(rb), _p(pa), _p(pb)))
    return ra.value >> 4, ra.value & 15, rb.value, pa, pb


def admissible(box_a, box_b, eta) -> bool:
    a = np.ascontiguousarray(box_a, dtype=np.float64).reshape(6)
    b = np.ascontiguousarray(box_b, dtype=np.float64).reshape(6)
    out = C.c_int()
    _ck(lib().or_admissible(_p(a), _p(b), D(eta), C.byref(out)))
    return bool(out.value)


class Problem:
    """An oracle problem: tree + partition + (after assemble) the component
    H-matrices of the reference semantics."""

    def __init__(self, handle, ncomp: int, n: int, ncols: int = -1):
        self._h = handle
        self.ncomp = ncomp
        self.n = n
        self.ncols = n if ncols < 0 else ncols

    def __del__(self):
        if getattr(self, "_h", None):
            lib().or_problem_free(self._h)
            self._h = None

    @classmethod
    def kelvin(cls, verts, tris, E=1.0, nu=0.3, b_min=32, eta=1.0):
        v = np.ascontiguousarray(verts, dtype=np.float64)
        t = np.ascontiguousarray(tris, dtype=np.int32)
        h = C.c_void_p()
        _ck(lib().or_problem_kelvin(len(v), _p(v), len(t), _p(t), D(E), D(nu), b_min,
                                    D(eta), C.byref(h)))
        return cls(h, 6, len(t))

    @classmethod
    def galerkin(cls, verts, tris, which=0, b_min=32, eta=1.0):
        """Galerkin scalar kernels on the triangle partition: which = 0 the
        six V_kl as the symmetric 3x3 grid, 1 V_Delta (kernels.cpp:130-149)."""
        v = np.ascontiguousarray(verts, dtype=np.float64)
        t = np.ascontiguousarray(tris, dtype=np.int32)
        h = C.c_void_p()
        _ck(lib().or_problem_galerkin(len(v), _p(v), len(t), _p(t), int(which), b_min,
                                      D(eta), C.byref(h)))
        return cls(h, 6 if which == 0 else 1, len(t))

    @classmethod
    def kelvin_points(cls, verts, tris, pts, E=1.0, nu=0.3, b_min=32, eta=1.0):
        """evaluate_interior's single-layer grid: Kelvin collocation at
        arbitrary points (baca.cpp:645-687)."""
        v = np.ascontiguousarray(verts, dtype=np.float64)
        t = np.ascontiguousarray(tris, dtype=np.int32)
        p = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        h = C.c_void_p()
        _ck(lib().or_problem_kelvin_points(len(v), _p(v), len(t), _p(t), len(p), _p(p), D(E),
                                           D(nu), b_min, D(eta), C.byref(h)))
        return cls(h, 6, len(p), len(t))

    @classmethod
    def kelvin_double(cls, verts, tris, pts, r, c, E=1.0, nu=0.3, b_min=32, eta=1.0,
                      disjoint_order=4):
        """One cell (r, c) of evaluate_interior's double-layer grid W~
        (CollocDoubleOracle, kernels.cpp:189-210): points x nodes."""
        v = np.ascontiguousarray(verts, dtype=np.float64)
        t = np.ascontiguousarray(tris, dtype=np.int32)
        p = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        h = C.c_void_p()
        _ck(lib().or_problem_kelvin_double(len(v), _p(v), len(t), _p(t), len(p), _p(p), r, c,
                                           D(E), D(nu), b_min, D(eta), disjoint_order,
                                           C.byref(h)))
        return cls(h, 1, len(p), len(v))

    @classmethod
    def kdelta(cls, verts, tris, b_min=32, eta=1.0):
        """K_Delta on the triangle x node partition (kernels.cpp:151-167,
        operators.cpp:186-200): rows triangles, columns vertices."""
        v = np.ascontiguousarray(verts, dtype=np.float64)
        t = np.ascontiguousarray(tris, dtype=np.int32)
        h = C.c_void_p()
        _ck(lib().or_problem_kdelta(len(v), _p(v), len(t), _p(t), b_min, D(eta),
                                    C.byref(h)))
        return cls(h, 1, len(t), len(v))

    @classmethod
    def newton(cls, pts, boxes=None, diag=2.0, b_min=10, eta=0.8):
        p = np.ascontiguousarray(pts, dtype=np.float64)
        b = None if boxes is None else np.ascontiguousarray(boxes, dtype=np.float64)
        h = C.c_void_p()
        _ck(lib().or_problem_newton(len(p), _p(p), _p(b), D(diag), b_min, D(eta),
                                    C.byref(h)))
        return cls(h, 1, len(p))

    @classmethod
    def dense_matrix(cls, a, row_pts, col_pts, b_min=10, eta=0.8):
        a = np.asfortranarray(a, dtype=np.float64)
        rp = np.ascontiguousarray(row_pts, dtype=np.float64)
        cp = np.ascontiguousarray(col_pts, dtype=np.float64)
        h = C.c_void_p()
        _ck(lib().or_problem_dense(a.shape[0], a.shape[1], a.ctypes.data_as(C.c_void_p),
                                   _p(rp), _p(cp), b_min, D(eta), C.byref(h)))
        return cls(h, 1, a.shape[0], a.shape[1])

    @property
    def rows(self) -> int:
        return self.n * (3 if self.ncomp == 6 else 1)

    def tree(self, which=0):
        nn, dep, sz = C.c_int(), C.c_int(), C.c_int()
        _ck(lib().or_tree_info(self._h, which, C.byref(nn), C.byref(dep), C.byref(sz)))
        nodes = np.zeros((nn.value, 5), np.int32)
        boxes = np.zeros((nn.value, 6))
        perm = np.zeros(sz.value, np.int32)
        _ck(lib().or_tree_nodes(self._h, which, _p(nodes), _p(boxes), _p(perm)))
        return nodes, boxes, perm, dep.value

    def partition_info(self):
        nb, na, cs = C.c_int(), C.c_int(), C.c_int()
        _ck(lib().or_partition_info(self._h, C.byref(nb), C.byref(na), C.byref(cs)))
        return nb.value, na.value, cs.value

    def blocks(self) -> np.ndarray:
        out = np.zeros((self.partition_info()[0], 4), np.int32)
        _ck(lib().or_partition_blocks(self._h, _p(out)))
        return out

    def partition_json(self) -> str:
        n = C.c_long()
        _ck(lib().or_partition_json(self._h, None, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        _ck(lib().or_partition_json(self._h, buf, C.byref(n)))
        return buf.value.decode()

    def entry(self, comp: int, i: int, j: int) -> float:
        out = D()
        _ck(lib().or_entry(self._h, int(comp), C.c_long(i), C.c_long(j), C.byref(out)))
        return out.value

    def entry_literal(self, comp: int, i: int, j: int) -> float:
        out = D()
        _ck(lib().or_entry_literal(self._h, int(comp), C.c_long(i), C.c_long(j), C.byref(out)))
        return out.value

    def rows_dot(self, out_dofs, x):
        """(exact, mag) of the requested rows of A x from oracle entries
        (Kelvin grid; output dof r*N + i)."""
        d = np.ascontiguousarray(out_dofs, dtype=np.int64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        ex, mg = np.zeros(len(d)), np.zeros(len(d))
        _ck(lib().or_rows_dot(self._h, len(d), _p(d), _p(x), _p(ex), _p(mg)))
        return ex, mg

    def dense(self, comp: int = 0) -> np.ndarray:
        out = np.zeros((self.n, self.ncols))
        _ck(lib().or_dense(self._h, int(comp), _p(out)))
        return out

    def dense_grid(self) -> np.ndarray:
        """Full 3N x 3N matrix of the 6-component grid (Kelvin collocation or
        the Galerkin V_kl grid), component-major."""
        if self.ncomp == 1:
            return self.dense(0)
        n, nc = self.n, self.ncols
        A = np.zeros((3 * n, 3 * nc))
        idx = {(0, 0): 0, (0, 1): 1, (0, 2): 2, (1, 1): 3, (1, 2): 4, (2, 2): 5}
        for (r, c), k in idx.items():
            blk = self.dense(k)
            A[r * n:(r + 1) * n, c * nc:(c + 1) * nc] = blk
            A[c * n:(c + 1) * n, r * nc:(r + 1) * nc] = blk
        return A

    def assemble(self, eps=1e-6, beta=0.8, initial_rank=-1, lookahead=2, max_rank=1 << 30):
        _ck(lib().or_assemble(self._h, D(eps), D(beta), initial_rank, lookahead,
                              C.c_long(max_rank)))

    def assemble_time(self):
        s, e = D(), C.c_long()
        _ck(lib().or_assemble_time(self._h, C.byref(s), C.byref(e)))
        return s.value, e.value

    def ranks(self):
        nb = self.partition_info()[0]
        n = self.ncomp * nb
        kc, kl, co, st = (np.zeros(n, np.int32) for _ in range(4))
        _ck(lib().or_ranks(self._h, _p(kc), _p(kl), _p(co), _p(st)))
        sh = (self.ncomp, nb)
        return kc.reshape(sh), kl.reshape(sh), co.reshape(sh), st.reshape(sh)

    def factor(self, comp: int, b: int):
        m, n, K = C.c_int(), C.c_int(), C.c_int()
        fs = D()
        _ck(lib().or_factor(self._h, int(comp), int(b), C.byref(m), C.byref(n), C.byref(K),
                            None, None, None, C.byref(fs)))
        U = np.zeros((m.value, K.value), order="F")
        V = np.zeros((n.value, K.value), order="F")
        piv = np.zeros((K.value, 2), np.int32)
        _ck(lib().or_factor(self._h, int(comp), int(b), C.byref(m), C.byref(n), C.byref(K),
                            U.ctypes.data_as(C.c_void_p), V.ctypes.data_as(C.c_void_p),
                            _p(piv), C.byref(fs)))
        return dict(U=U, V=V, pivots=piv, frob_sq=fs.value)

    def aca_block(self, comp, b, eps=1e-6, beta=0.8, initial_rank=-1, lookahead=2):
        kc, K = C.c_int(), C.c_int()
        fs = D()
        ent = C.c_long()
        _ck(lib().or_aca_block(self._h, int(comp), int(b), D(eps), D(beta), initial_rank, lookahead,
                               C.byref(kc), C.byref(K), C.byref(fs), C.byref(ent)))
        return kc.value, K.value, fs.value, ent.value

    def dense_block(self, comp: int, b: int, m: int, n: int) -> np.ndarray:
        out = np.zeros((m, n), order="F")
        _ck(lib().or_dense_block(self._h, int(comp), int(b), out.ctypes.data_as(C.c_void_p)))
        return out

    def matvec(self, x, mode=0) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.rows)
        _ck(lib().or_matvec(self._h, _p(x), _p(y), mode))
        return y

    def matvec_transposed(self, x, mode=0) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.ncols * (3 if self.ncomp == 6 else 1))
        _ck(lib().or_matvec_transposed(self._h, _p(x), _p(y), mode))
        return y

    def matvec_time(self, x, reps=3) -> float:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.rows)
        best = D()
        _ck(lib().or_matvec_time(self._h, _p(x), _p(y), reps, C.byref(best)))
        return best.value

    def storage(self):
        a, b, p = D(), D(), C.c_long()
        _ck(lib().or_storage(self._h, C.byref(a), C.byref(b), C.byref(p)))
        return dict(mb_current=a.value, mb_tail=b.value, total_pivots=p.value)

    def promote(self, comp, b):
        _ck(lib().or_promote(self._h, int(comp), int(b)))

    def extend(self, comp, b, steps):
        _ck(lib().or_extend(self._h, int(comp), int(b), int(steps)))

    def gamma(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        g = D()
        diff = np.zeros(self.rows)
        nt = C.c_int()
        _ck(lib().or_gamma(self._h, _p(x), C.byref(g), _p(diff), C.byref(nt)))
        n = nt.value
        comp, block, nnz = (np.zeros(n, np.int32) for _ in range(3))
        nsq = np.zeros(n)
        _ck(lib().or_gamma_terms(_p(comp), _p(block), _p(nnz), _p(nsq)))
        terms = []
        for t in range(n):
            idx = np.zeros(nnz[t], np.int64)
            val = np.zeros(nnz[t])
            _ck(lib().or_gamma_term_data(t, _p(idx), _p(val)))
            terms.append(dict(comp=int(comp[t]), block=int(block[t]), idx=idx, val=val,
                              norm_sq=float(nsq[t])))
        return g.value, diff, terms

    def mark(self, theta, c_sp, m_rows, n_cols, n_terms):
        marked = np.zeros(max(1, n_terms), np.int32)
        nm = C.c_int()
        gpk = D()
        _ck(lib().or_mark(D(theta), c_sp, C.c_long(m_rows), C.c_long(n_cols), _p(marked),
                          C.byref(nm), C.byref(gpk)))
        return marked[: nm.value].copy(), gpk.value

    def amvm(self, x, theta=0.7, eps_amvm=1e-6, lookahead_steps=2, max_iterations=100):
        x = np.ascontiguousarray(x, dtype=np.float64)
        b = np.zeros(self.rows)
        it = np.zeros((max_iterations + 1, 7))
        ni, conv = C.c_int(), C.c_int()
        _ck(lib().or_amvm(self._h, _p(x), D(theta), D(eps_amvm), lookahead_steps,
                          max_iterations, _p(b), _p(it), C.byref(ni), C.byref(conv)))
        return b, it[: ni.value], bool(conv.value)


class AcaDense:
    """Single-block ACA on a dense matrix (test_aca.cpp ports)."""

    def __init__(self, a):
        a = np.asfortranarray(a, dtype=np.float64)
        self.m, self.n = a.shape
        h = C.c_void_p()
        _ck(lib().or_aca_dense_new(self.m, self.n, a.ctypes.data_as(C.c_void_p), C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib().or_aca_dense_free(self._h)
            self._h = None

    def run(self, eps, beta, max_rank):
        _ck(lib().or_aca_dense_step(self._h, 0, D(eps), D(beta), 0, C.c_long(max_rank)))
        return self

    def extend(self, steps, max_rank):
        _ck(lib().or_aca_dense_step(self._h, 1, D(0.0), D(0.0), steps, C.c_long(max_rank)))
        return self

    def state(self):
        K, nc, ls = C.c_int(), C.c_int(), C.c_int()
        fs = D()
        _ck(lib().or_aca_dense_state(self._h, C.byref(K), C.byref(nc), C.byref(ls),
                                     C.byref(fs), None, None, None))
        U = np.zeros((self.m, K.value), order="F")
        V = np.zeros((self.n, K.value), order="F")
        piv = np.zeros((K.value, 2), np.int32)
        _ck(lib().or_aca_dense_state(self._h, C.byref(K), C.byref(nc), C.byref(ls),
                                     C.byref(fs), U.ctypes.data_as(C.c_void_p),
                                     V.ctypes.data_as(C.c_void_p), _p(piv)))
        return dict(rank=K.value, num_consumed=nc.value, last_stop=ls.value, frob_sq=fs.value,
                    U=U, V=V, pivots=piv)
