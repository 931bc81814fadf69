"""ctypes binding of the native libraries (lib/libhmbem.so -> lib/libhmgpu.so).

The product path is native only: if the libraries are missing the import
fails loudly -- there is no Python or CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# HMGPU_LIB_DIR: an alternate build of the same sources (development A/B runs)
LIB_DIR = os.environ.get("HMGPU_LIB_DIR") or os.path.join(_PKG, "lib")
HMBEM_PATH = os.path.join(LIB_DIR, "libhmbem.so")
HMGPU_PATH = os.path.join(LIB_DIR, "libhmgpu.so")

if not os.path.exists(HMBEM_PATH) or not os.path.exists(HMGPU_PATH):
    raise ImportError(
        "paper_2205_04752_b200 native libraries are not built; run "
        "`python paper_2205_04752_b200/build.py` (or __graft_entry__.build())")

gpu = C.CDLL(HMGPU_PATH, mode=C.RTLD_GLOBAL)
host = C.CDLL(HMBEM_PATH)

P = C.c_void_p
I = C.c_int
LL = C.c_longlong
D = C.c_double
IP = C.POINTER(C.c_int)
DP = C.POINTER(C.c_double)
LLP = C.POINTER(C.c_longlong)


def _sig(lib, name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


# ---- hmbem.h ----
_sig(host, "hmb_last_error", C.c_char_p)
_sig(host, "hmb_device_status", I)
_sig(host, "hmb_mesh_icosphere", I, I, C.POINTER(P))
_sig(host, "hmb_mesh_ellipsoid", I, I, D, D, D, C.POINTER(P))
_sig(host, "hmb_mesh_voxel_cube", I, I, D, D, C.POINTER(P))
_sig(host, "hmb_mesh_from_arrays", I, I, P, I, P, C.POINTER(P))
_sig(host, "hmb_mesh_load_off", I, C.c_char_p, C.POINTER(P))
_sig(host, "hmb_mesh_save_off", I, P, C.c_char_p)
_sig(host, "hmb_mesh_validate", I, P)
_sig(host, "hmb_mesh_label", I, P, C.c_char_p)
_sig(host, "hmb_mesh_sizes", I, P, IP, IP)
_sig(host, "hmb_mesh_get", I, P, P, P, P, P, P, P, P)
_sig(host, "hmb_mesh_free", None, P)
_sig(host, "hmb_admissible", I, P, P, D, IP)
_sig(host, "hmb_gauss_rule", I, I, IP, P, P, P)
_sig(host, "hmb_random_vector", I, LL, C.c_ulonglong, I, P)
_sig(host, "hmb_op_kelvin", I, P, D, D, I, D, I, I, I, C.POINTER(P))
_sig(host, "hmb_op_galerkin", I, P, I, I, D, I, I, I, C.POINTER(P))
_sig(host, "hmb_op_kelvin_points", I, P, I, P, D, D, I, D, D, I, I, I, I, C.POINTER(P))
_sig(host, "hmb_op_kelvin_double", I, P, I, P, I, I, D, D, I, D, D, I, I, I, I, C.POINTER(P))
_sig(host, "hmb_op_kdelta", I, P, I, D, I, I, I, C.POINTER(P))
_sig(host, "hmb_sparse_op", I, P, I, P, P)
_sig(host, "hmb_pair_rule", I, I, I, IP, P, P, P, P, P)
_sig(gpu, "hmgpu_ell3_spmv", I, P, I, P, P, P, P, D, D)
_sig(gpu, "hmgpu_ell3_spmv_t", I, P, I, P, P, P, P, P, D, D)
_sig(host, "hmb_op_newton", I, I, P, P, D, I, D, I, C.POINTER(P))
_sig(host, "hmb_op_dense", I, I, I, P, P, P, I, D, I, C.POINTER(P))
_sig(host, "hmb_op_free", None, P)
_sig(host, "hmb_op_info", I, P, LLP, LLP, IP, IP, IP)
_sig(host, "hmb_op_gpu", P, P)
_sig(host, "hmb_tree_info", I, P, I, IP, IP, IP)
_sig(host, "hmb_tree_nodes", I, P, I, P, P, P)
_sig(host, "hmb_partition_info", I, P, IP, IP, IP)
_sig(host, "hmb_partition_blocks", I, P, P)
_sig(host, "hmb_partition_json", I, P, C.c_char_p, LLP)
_sig(host, "hmb_assemble", I, P, D, D, I, I, LL, P)
_sig(host, "hmb_matvec", I, P, P, P, I, I, I)
_sig(host, "hmb_matvec_transposed", I, P, P, P, I, I, I)
_sig(host, "hmb_ranks", I, P, P, P, P, P)
_sig(host, "hmb_promote", I, P, I, P)
_sig(host, "hmb_extend", I, P, I, P, I)
_sig(host, "hmb_storage", I, P, P)
_sig(host, "hmb_factor", I, P, I, I, IP, IP, IP, IP, P, P, P, DP)
_sig(host, "hmb_dense_block", I, P, I, I, P)
_sig(host, "hmb_gamma", I, P, P, DP, P, IP)
_sig(host, "hmb_gamma_t", I, P, P, DP, P, IP)
_sig(host, "hmb_gamma_terms", I, P, P, P, P, P)
_sig(host, "hmb_gamma_term_data", I, P, I, P, P)
_sig(host, "hmb_mark", I, P, D, I, LL, LL, P, IP, DP)
_sig(host, "hmb_amvm", I, P, P, D, D, I, I, P, P, IP, IP)

# ---- hmgpu.h (direct device-level calls: stream, profiling) ----
_sig(gpu, "hmgpu_device_count", I, IP)
_sig(gpu, "hmgpu_last_error", C.c_char_p, P)
_sig(gpu, "hmgpu_get_stream", I, P, C.POINTER(P))
_sig(gpu, "hmgpu_set_profiling", I, P, I)
_sig(gpu, "hmgpu_kernel_times", I, P, C.c_char_p, DP, LLP, I)
_sig(gpu, "hmgpu_storage", I, P, P)
_sig(gpu, "hmgpu_fp64_peak", I, I, DP)
_sig(gpu, "hmgpu_dmma_peak", I, I, DP)
_sig(gpu, "hmgpu_dmma_peak_sustained", I, I, D, DP)
_sig(gpu, "hmgpu_set_matvec_policy", I, P, I)
_sig(gpu, "hmgpu_get_matvec_policy", I, P, IP)
# multi-GPU block-row shards
_sig(gpu, "hmgpu_nccl_available", I, IP, IP)
_sig(gpu, "hmgpu_nccl_unique_id", I, P)
_sig(gpu, "hmgpu_comm_init_nccl", I, P, I, I, P)
_sig(gpu, "hmgpu_comm_set_nccl", I, P, P, I, I)
_sig(gpu, "hmgpu_comm_clear", I, P)
_sig(gpu, "hmgpu_comm_info", I, P, IP, IP, IP, P, P)
_sig(gpu, "hmgpu_matvec_dist", I, P, P, P, I, I, I)

# hmgpu_comm_ops: host-callback transport
BCAST_FN = C.CFUNCTYPE(C.c_int, P, P, C.c_longlong, C.c_int)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, P, P, P, C.c_longlong)


_sig(host, "hmb_mark_sharded", I, I, P, P, P, P, P, LL, LL, D, I, I, I, ALLGATHER_FN, P, P,
     IP, IP, DP)
_sig(gpu, "hmgpu_comm_allgather", I, P, P, P, LL)


class CommOps(C.Structure):
    _fields_ = [("broadcast", BCAST_FN), ("allgather", ALLGATHER_FN), ("user", P)]


_sig(gpu, "hmgpu_comm_set_ops", I, P, I, I, C.POINTER(CommOps))

HMGPU_SYMBOLS = [
    "hmgpu_device_count", "hmgpu_create", "hmgpu_destroy", "hmgpu_last_error",
    "hmgpu_get_stream", "hmgpu_set_rule", "hmgpu_set_tier_ratios",
    "hmgpu_set_kelvin_geometry", "hmgpu_set_points", "hmgpu_set_dense_matrix",
    "hmgpu_set_partition", "hmgpu_assemble", "hmgpu_ranks", "hmgpu_matvec",
    "hmgpu_promote", "hmgpu_extend", "hmgpu_tail_terms", "hmgpu_download_factor",
    "hmgpu_download_dense", "hmgpu_storage", "hmgpu_set_profiling",
    "hmgpu_kernel_times", "hmgpu_fp64_peak", "hmgpu_dmma_peak", "hmgpu_amvm_estimate",
    "hmgpu_amvm_mark", "hmgpu_amvm_refine", "hmgpu_set_matvec_policy",
]
