"""The C ABI's error behaviour on a device (include/hmgpu.h status codes):
arguments the reference rejects with hmbem::Error / DimensionError
(aca.cpp:108-110, hmatrix.cpp:22-30) come back as HMGPU_ERR_INVALID /
HMGPU_ERR_DIMENSION, calls out of order as HMGPU_ERR_STATE, and a context
stays usable after a rejected call (the next valid matvec is unchanged)."""
import ctypes as C

import numpy as np
import pytest

import paper_2205_04752_b200 as hm
from paper_2205_04752_b200 import _lib
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

OK, INVALID, STATE = 0, 1, 5
HOST, DEVICE = 0, 1
g = _lib.gpu
DP = C.POINTER(C.c_double)


def _sig(name, *args):
    f = getattr(g, name)
    f.restype = C.c_int
    f.argtypes = list(args)
    return f


create = _sig("hmgpu_create", C.c_int, C.POINTER(C.c_void_p))
destroy = _sig("hmgpu_destroy", C.c_void_p)
set_points = _sig("hmgpu_set_points", C.c_void_p, C.c_int, DP, C.c_double)
assemble = _sig("hmgpu_assemble", C.c_void_p, C.c_double, C.c_double, C.c_int, C.c_int,
                C.c_longlong, C.c_void_p)
matvec = _sig("hmgpu_matvec", C.c_void_p, DP, DP, C.c_int, C.c_int, C.c_int)


def _dp(a):
    return a.ctypes.data_as(DP)


def test_create_and_destroy_arguments():
    ctx = C.c_void_p()
    assert create(-1, C.byref(ctx)) == INVALID
    assert create(1 << 20, C.byref(ctx)) == INVALID
    assert create(0, None) == INVALID
    assert destroy(None) == INVALID
    assert create(0, C.byref(ctx)) == OK and ctx.value
    assert destroy(ctx) == OK


def test_calls_out_of_order_and_bad_points():
    ctx = C.c_void_p()
    assert create(0, C.byref(ctx)) == OK
    try:
        x = np.ones(8)
        y = np.zeros(8)
        assert matvec(ctx, _dp(x), _dp(y), 1, 0, HOST) == STATE
        assert b"assemble" in g.hmgpu_last_error(ctx)
        assert assemble(ctx, 1e-6, 0.8, -1, 0, 1 << 30, None) == STATE
        assert set_points(ctx, 0, _dp(x), 0.0) == INVALID
        assert set_points(ctx, 4, None, 0.0) == INVALID
    finally:
        destroy(ctx)


def test_rejected_calls_leave_the_context_usable():
    mesh = hm.Mesh.icosphere(2)
    h = hm.HMatrix.kelvin(mesh, b_min=16, eta=1.0, device=0)
    h.assemble(eps=1e-4, beta=0.8)
    ctx = h.gpu_ctx
    n = h.cols
    x = orc.random_vector(n, 3)
    y0 = np.zeros(h.rows)
    assert matvec(ctx, _dp(x), _dp(y0), 1, 0, HOST) == OK
    y = np.zeros(h.rows)
    assert matvec(ctx, None, _dp(y), 1, 0, HOST) == INVALID
    assert matvec(ctx, _dp(x), _dp(y), 0, 0, HOST) == INVALID
    assert matvec(ctx, _dp(x), _dp(y), 1, 7, HOST) == INVALID
    assert matvec(ctx, _dp(x), _dp(y), 1, 0, 9) == INVALID
    assert assemble(ctx, 0.0, 0.8, -1, 0, 1 << 30, None) == INVALID  # aca.cpp:108-110
    assert assemble(ctx, 1e-4, 1.0, -1, 0, 1 << 30, None) == INVALID
    assert assemble(ctx, 1e-4, 0.8, -1, -1, 1 << 30, None) == INVALID
    assert matvec(ctx, _dp(x), _dp(y), 1, 0, HOST) == OK
    assert (y == y0).all()
    np.testing.assert_allclose(y0, h.matvec(x), rtol=0, atol=0)
