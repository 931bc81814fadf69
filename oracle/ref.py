"""ctypes wrapper of oracle/_ref/libhmbem_ref.so: the reference's own
hot-path code (proj/src/{quadrature,mesh,cluster,kernels,aca,hmatrix,expr,
amvm}.cpp, compiled unmodified against oracle/ref_shim/) behind the C ABI of
oracle/ref_driver.cpp.

TEST INFRASTRUCTURE ONLY: used by tests/ (to pin oracle/hmbem_oracle.cpp and
the GPU path against the reference's code) and by bench.py's reference arm.
The library is built in the container that has /root/reference
(``make -C oracle ref``, called by __graft_entry__.build()); it travels to the
GPU box as a built file.  available() is False where it was never built.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libhmbem_ref.so")
REF_SRC = "/root/reference/proj/src"

_lib = None


def build() -> bool:
    """Compiles _ref from the reference sources when they are present."""
    import subprocess
    if not os.path.isdir(REF_SRC):
        return os.path.exists(LIB_PATH)
    subprocess.run(["make", "-C", HERE, "-s", "ref"], check=True)
    return True


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        L.hmr_last_error.restype = C.c_char_p
        L.hmr_destroy.argtypes = [C.c_void_p]
        L.hmr_create.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_double,
                                 C.c_double, C.c_int, C.c_double, C.c_void_p]
        L.hmr_assemble.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_int, C.c_int,
                                   C.c_longlong]
        L.hmr_entry.argtypes = [C.c_void_p, C.c_int, C.c_longlong, C.c_longlong, C.c_void_p]
        L.hmr_amvm.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_int, C.c_int,
                               C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.hmr_mark.argtypes = [C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_void_p]
        _lib = L
    return _lib


class RefError(RuntimeError):
    pass


def _ck(st: int) -> None:
    if st != 0:
        raise RefError(lib().hmr_last_error().decode())


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def set_threads(n: int) -> None:
    lib().hmr_set_threads(int(n))


class RefProblem:
    """One operator built by the reference's code: kind "kelvin" (the 3x3
    Kelvin centroid-collocation grid, 6 component H-matrices) or "newton"
    (the reference test suite's CentroidKernelOracle fixture)."""

    def __init__(self, verts, tris, kind: str = "kelvin", E: float = 1.0, nu: float = 0.3,
                 b_min: int = 32, eta: float = 1.0):
        v = np.ascontiguousarray(verts, dtype=np.float64)
        t = np.ascontiguousarray(tris, dtype=np.int32)
        h = C.c_void_p()
        _ck(lib().hmr_create({"kelvin": 0, "newton": 1}[kind], len(v), _p(v), len(t), _p(t),
                             E, nu, b_min, eta, C.byref(h)))
        self._h = h
        n, nb, nc, csp, nn = (C.c_int() for _ in range(5))
        _ck(lib().hmr_info(self._h, C.byref(n), C.byref(nb), C.byref(nc), C.byref(csp),
                           C.byref(nn)))
        self.nt, self.num_blocks, self.ncomp = n.value, nb.value, nc.value
        self.c_sp, self.n_nodes = csp.value, nn.value
        self.n = self.nt * (3 if self.ncomp == 6 else 1)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.hmr_destroy(self._h)
            self._h = None

    def partition_json(self) -> str:
        n = C.c_longlong()
        _ck(lib().hmr_partition_json(self._h, None, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        _ck(lib().hmr_partition_json(self._h, buf, C.byref(n)))
        return buf.value.decode()

    def tree(self):
        perm = np.zeros(self.nt, np.int32)
        nodes = np.zeros((self.n_nodes, 4), np.int32)
        blocks = np.zeros((self.num_blocks, 4), np.int32)
        _ck(lib().hmr_tree(self._h, _p(perm), _p(nodes), _p(blocks)))
        return perm, nodes, blocks

    def restrict_rows(self, row_begin: int, row_end: int) -> None:
        """Keep only the block rows inside [row_begin, row_end) (internal
        positions): a bounded sample of the operator for CPU timing."""
        _ck(lib().hmr_restrict_rows(self._h, int(row_begin), int(row_end)))
        nb = C.c_int()
        _ck(lib().hmr_info(self._h, None, C.byref(nb), None, None, None))
        self.num_blocks = nb.value

    def subtree_rows(self, depth: int):
        """[begin, end) of the row-tree node reached from the root by
        `depth` first-child steps (a 2^-depth sample of the rows)."""
        _, nodes, _ = self.tree()
        nd = 0
        for _ in range(depth):
            if nodes[nd, 2] < 0:
                break
            nd = nodes[nd, 2]
        return int(nodes[nd, 0]), int(nodes[nd, 1])

    def entry(self, comp: int, i: int, j: int) -> float:
        out = C.c_double()
        _ck(lib().hmr_entry(self._h, int(comp), int(i), int(j), C.byref(out)))
        return out.value

    def assemble(self, eps=1e-6, beta=0.8, initial_rank=-1, lookahead=2, max_rank=1 << 30):
        _ck(lib().hmr_assemble(self._h, eps, beta, initial_rank, lookahead, max_rank))

    def ranks(self):
        kc = np.zeros(self.ncomp * self.num_blocks, np.int32)
        kl = np.zeros_like(kc)
        _ck(lib().hmr_ranks(self._h, _p(kc), _p(kl)))
        return kc.reshape(self.ncomp, -1), kl.reshape(self.ncomp, -1)

    def storage(self):
        mb = C.c_double()
        piv = C.c_longlong()
        _ck(lib().hmr_storage(self._h, C.byref(mb), C.byref(piv)))
        return mb.value, piv.value

    def factor(self, comp: int, block: int):
        m, n, K, kc = (C.c_int() for _ in range(4))
        _ck(lib().hmr_factor(self._h, int(comp), int(block), C.byref(m), C.byref(n), C.byref(K),
                             C.byref(kc), None, None, None))
        U = np.zeros((m.value, K.value), order="F")
        V = np.zeros((n.value, K.value), order="F")
        piv = np.zeros((K.value, 2), np.int32)
        _ck(lib().hmr_factor(self._h, int(comp), int(block), C.byref(m), C.byref(n), C.byref(K),
                             C.byref(kc), _p(U), _p(V), _p(piv)))
        return dict(U=U, V=V, pivots=piv, k_cur=kc.value)

    def matvec(self, x, mode: int = 0) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.n)
        _ck(lib().hmr_matvec(self._h, _p(x), _p(y), mode))
        return y

    def gamma(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        g = C.c_double()
        diff = np.zeros(self.n)
        nt = C.c_int()
        _ck(lib().hmr_gamma(self._h, _p(x), C.byref(g), _p(diff), C.byref(nt)))
        self._nterms = nt.value
        return g.value, diff, nt.value

    def mark(self, theta: float):
        n = max(1, self._nterms)
        marked = np.zeros(n, np.int32)
        nm = C.c_int()
        gpk = C.c_double()
        cb = np.zeros((n, 2), np.int32)
        _ck(lib().hmr_mark(self._h, theta, _p(marked), C.byref(nm), C.byref(gpk), _p(cb)))
        return marked[: nm.value].copy(), gpk.value, cb[: self._nterms].copy()

    def amvm(self, x, theta=0.7, eps_amvm=1e-6, lookahead_steps=2, max_iterations=100):
        x = np.ascontiguousarray(x, dtype=np.float64)
        b = np.zeros(self.n)
        iters = np.zeros((max_iterations + 1, 8))
        ni, conv = C.c_int(), C.c_int()
        _ck(lib().hmr_amvm(self._h, _p(x), theta, eps_amvm, lookahead_steps, max_iterations,
                           _p(b), _p(iters), C.byref(ni), C.byref(conv)))
        return b, iters[: ni.value].copy(), bool(conv.value)


class RefOperatorSet:
    """assemble_operators (operators.cpp:187-245) by the reference's code on
    a labelled mesh (load_mesh with a centroid predicate), and the
    right-hand-side operator of assemble_rhs (baca.cpp:42-76): its product
    at the current ranks and its adaptive matvec (amvm_multiply over the
    flattened expression)."""

    def __init__(self, verts, tris, predicate: str, E=1.0, nu=0.3, b_min=8, eta=1.0,
                 eps=1e-6, beta_stop=0.8, lookahead=2):
        L = lib()
        L.hmr_ops_create.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_char_p,
                                     C.c_double, C.c_double, C.c_int, C.c_double, C.c_double,
                                     C.c_double, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        L.hmr_ops_destroy.argtypes = [C.c_void_p]
        L.hmr_ops_rhs.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.hmr_ops_rhs_amvm.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_double,
                                       C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p]
        v = np.ascontiguousarray(verts, dtype=np.float64)
        t = np.ascontiguousarray(tris, dtype=np.int32)
        h = C.c_void_p()
        rows, cols = C.c_longlong(), C.c_longlong()
        _ck(L.hmr_ops_create(len(v), _p(v), len(t), _p(t), predicate.encode(), E, nu, b_min,
                             eta, eps, beta_stop, lookahead, C.byref(h), C.byref(rows),
                             C.byref(cols)))
        self._h = h
        self.rows, self.cols = rows.value, cols.value

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.hmr_ops_destroy(self._h)
            self._h = None

    def rhs(self, g_neumann, g_dirichlet) -> np.ndarray:
        x = np.ascontiguousarray(np.concatenate([g_neumann, g_dirichlet]), dtype=np.float64)
        f = np.zeros(self.rows)
        _ck(lib().hmr_ops_rhs(self._h, _p(x), _p(f)))
        return f

    def rhs_amvm(self, g_neumann, g_dirichlet, theta=0.7, eps_amvm=1e-6, lookahead_steps=2,
                 max_iterations=100):
        x = np.ascontiguousarray(np.concatenate([g_neumann, g_dirichlet]), dtype=np.float64)
        f = np.zeros(self.rows)
        iters = np.zeros((max_iterations + 1, 8))
        ni, conv = C.c_int(), C.c_int()
        _ck(lib().hmr_ops_rhs_amvm(self._h, _p(x), theta, eps_amvm, lookahead_steps,
                                   max_iterations, _p(f), _p(iters), C.byref(ni),
                                   C.byref(conv)))
        return f, iters[: ni.value].copy(), bool(conv.value)
