"""ctypes binding of libsimopt_b200.so (the C ABI in include/simopt_b200.h).

There is no CPU fallback: if the shared library is missing or no CUDA device
is visible, every product entry point raises :class:`DeviceError`.
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

from .errors import STATUS_TO_ERROR, DeviceError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SIMOPT_LIB_PATH") or os.path.join(_HERE, "libsimopt_b200.so")  # override: experiments

_lock = threading.Lock()
_lib = None
_device_ok = False

_u64, _i64, _i32, _d, _vp = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p

# name -> argtypes (all return int status)
SIGNATURES = {
    "simopt_uniform01": [_vp, _u64, _u64, _u64, _u64, _i64, _vp],
    "simopt_standard_normal": [_vp, _u64, _u64, _u64, _u64, _i64, _vp],
    "simopt_sample_returns_diag": [_vp, _u64, _u64, _u64, _u64, _i64, _i64, _vp, _vp, _vp],
    "simopt_bernoulli_half": [_vp, _u64, _u64, _u64, _u64, _i64, _vp],
    "simopt_threshold": [_vp, _vp, _d, _i64, _vp],
    "simopt_dot": [_vp, _vp, _vp, _i64, _i64, _vp],
    "simopt_dot_fast": [_vp, _vp, _vp, _i64, _vp],
    "simopt_col_sums_fast": [_vp, _vp, _i64, _i64, _vp],
    "simopt_vec_sum": [_vp, _vp, _i64, _i64, _vp],
    "simopt_tree_sums2": [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _i64, _vp, _i64],
    "simopt_matvec": [_vp, _vp, _i64, _i64, _vp, _i64, _vp, _vp, _i64, _vp],
    "simopt_matvec_t": [_vp, _vp, _i64, _i64, _vp, _i64, _vp, _vp, _i64, _vp],
    "simopt_axpy": [_vp, _d, _vp, _vp, _i64, _vp],
    "simopt_axpy_ptr": [_vp, _vp, _vp, _vp, _i64, _vp],
    "simopt_map_kernel": [_vp, _i32, _vp, _i64, _vp],
    "simopt_timestamp": [_vp, _vp],
    "simopt_philox_floor": [_vp, _u64, _u64, _u64, _i64, _vp, _i64],
    "simopt_scale_sub": [_vp, _vp, _d, _vp, _i64, _vp],
    "simopt_min_value": [_vp, _vp, _i64, _vp],
    "simopt_lmo_simplex_slack": [_vp, _vp, _i64, _vp, _vp],
    "simopt_lmo_single_budget": [_vp, _vp, _vp, _d, _i64, _vp, _vp],
    "simopt_nv_layout": [_i64, _i64, _vp, _vp, _vp],
    "simopt_nv_geometry": [_vp, _vp],
    "simopt_nv_resample": [_vp, _u64, _u64, _u64, _u64, _i64, _i64, _vp, _vp],
    "simopt_nv_counts": [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _u64, _u64, _u64, _u64, _vp, _vp],
    "simopt_nv_approx_error": [_vp, _u64, _u64, _u64, _u64, _i64, _vp, _vp],
    "simopt_nv_decode": [_vp, _vp, _vp, _vp, _i64, _i64, _u64, _u64, _u64, _u64, _vp],
    "simopt_nv_iter": [_vp, _vp],
    "simopt_ecdf_count_sorted": [_vp, _vp, _i64, _i64, _vp, _vp],
    "simopt_nv_grad_from_counts": [_vp, _vp, _i64, _vp, _vp, _vp, _i64, _vp],
    "simopt_nv_grad_exact": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp],
    "simopt_nv_cost_terms": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp],
    "simopt_nv_epoch_records": [_vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64,
                                _vp, _vp],
    "simopt_logistic_resid": [_vp, _vp, _vp, _vp, _i64, _vp],
    "simopt_logistic_hvp_weights": [_vp, _vp, _vp, _i64, _vp],
    "simopt_logistic_loss_terms": [_vp, _vp, _vp, _vp, _i64, _vp],
    "simopt_bfgs_rank2": [_vp, _vp, _vp, _vp, _d, _d, _i64],
    "simopt_diag_fill": [_vp, _vp, _i64, _d],
    "simopt_vec_op": [_vp, _i32, _d, _vp, _vp, _i64, _vp],
    "simopt_sample_indices": [_vp, _u64, _u64, _u64, _u64, _i64, _i64, _vp],
    "simopt_fisher_yates_host": [_i64, _i64, _vp, _vp],
    "simopt_logistic_xtdx": [_vp, _vp, _vp, _i64, _i64, _vp],
    "simopt_cg_step1": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64],
    "simopt_cg_step2": [_vp, _vp, _vp, _vp, _vp, _i64],
    "simopt_fused_rows": [_vp, _i32, _vp, _i64, _i64, _vp, _vp, _vp, _d, _i32, _i32, _vp, _vp, _vp,
                          _vp, _vp],
    "simopt_fused_geometry": [_i32, _i64, _i32, _vp, _vp, _vp],
    "simopt_peer_reduce_bytes": [_i64, _i64],
    "simopt_sample_returns_diag_rows": [_vp, _u64, _u64, _u64, _u64, _i64, _i64, _i64, _vp, _vp, _vp],
    "simopt_bernoulli_half_range": [_vp, _u64, _u64, _u64, _u64, _i64, _i64, _vp],
    "simopt_matvec_t_partials": [_vp, _vp, _i64, _i64, _vp, _vp, _i64, _vp],
    "simopt_fold_partials": [_vp, _vp, _i64, _i64, _vp],
    "simopt_nv_lmo_pack": [_vp, _vp, _i64, _vp],
    "simopt_peer_alloc": [_i64, _vp, _vp],
    "simopt_peer_open": [_vp, _vp],
    "simopt_peer_close": [_vp],
    "simopt_peer_free": [_vp],
    "simopt_bernoulli_bits": [_vp, _u64, _u64, _u64, _u64, _i64, _i64, _i64, _vp],
    "simopt_matvec_bits": [_vp, _vp, _i64, _i64, _vp, _i64, _vp],
    "simopt_sample_indices_dev": [_vp, _vp, _i64, _i64, _vp],
    "simopt_bfgs_rank2_dev": [_vp, _vp, _vp, _vp, _d, _vp, _i64],
    "simopt_lmo_general": [_vp, _vp, _vp, _i64, _i64, _vp, _i64, _vp, _vp],
    "simopt_sqn_step": [_vp, _vp, _vp, _vp, _i64, _vp],
    "simopt_sqn_record": [_vp, _vp, _vp, _vp, _vp],
    "simopt_matvec_bits_idx": [_vp, _vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp],
    "simopt_matvec_t_bits": [_vp, _vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp],
    "simopt_unpack_bits": [_vp, _vp, _i64, _i64, _vp],
    "simopt_fused_rows_bits": [_vp, _i32, _vp, _i64, _i64, _vp, _vp, _d, _i32, _i32, _vp, _vp, _vp,
                               _vp, _vp],
    "simopt_logistic_xtdx_bits": [_vp, _vp, _vp, _i64, _i64, _vp],
    "simopt_u8t_geometry": [_i64, _vp, _vp],
    "simopt_bits_to_u8t": [_vp, _vp, _i64, _i64, _i64, _vp],
    "simopt_logistic_xtdx_i8": [_vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp],
    "simopt_logistic_xtdx_tc": [_vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp],
    "simopt_logistic_xtdx_tma": [_vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp],
    "simopt_logistic_xtdx_pair": [_vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp],
    "simopt_xtdx_last_passes": [],
    "simopt_comm_version": [_vp],
    "simopt_comm_unique_id": [_vp],
    "simopt_comm_init": [_vp, _i32, _i32, _vp],
    "simopt_comm_destroy": [_vp],
    "simopt_comm_allreduce_f64": [_vp, _vp, _vp, _vp, _i64],
    "simopt_comm_allreduce_min_f64": [_vp, _vp, _vp, _vp, _i64],
    "simopt_comm_allgather": [_vp, _vp, _vp, _vp, _i64],
    "simopt_comm_broadcast": [_vp, _vp, _vp, _vp, _i64, _i32],
    "simopt_mv_fw_tail": [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _i32],
    "simopt_mv_fw_epoch": [_vp, _vp, _i64, _i64, _vp, _d, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "simopt_project_budget": [_vp, _vp, _vp, _d, _i64, _vp, _vp],
    "simopt_project_box": [_vp, _vp, _d, _d, _i64, _vp],
    "simopt_philox4x32": [_vp, ctypes.c_uint32, ctypes.c_uint32, _vp, _i64, _vp],
    "simopt_sfc64": [_vp, _vp, _i64, _i64, _i32, _vp],
    "simopt_xoshiro256pp": [_vp, _vp, _i64, _i64, _i32, _vp],
    "simopt_xoshiro256pp_streams": [_vp, _i64, _vp],
    "simopt_nv_lmo_apply": [_vp, _vp, _i64, _i64, _i64, _vp],
}


# value-returning queries; every other entry point returns a status
INT64_RESULT = {"simopt_peer_reduce_bytes", "simopt_xtdx_last_passes"}


ABI_VERSION = 4  # csrc/capi.cu simopt_abi_version; bumped when an entry point's signature changes


def load(require_device: bool = True):
    """Load the library (idempotent).  Raises DeviceError when unusable."""
    global _lib, _device_ok
    if _lib is not None and (_device_ok or not require_device):
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise DeviceError(
                    f"{LIB_PATH} not built; run `python -m paper_2404_11631_b200.build` "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            lib.simopt_last_error.restype = ctypes.c_char_p
            lib.simopt_abi_version.restype = ctypes.c_int
            if lib.simopt_abi_version() != ABI_VERSION:
                raise DeviceError(
                    f"{LIB_PATH} has ABI {lib.simopt_abi_version()}, this package expects "
                    f"{ABI_VERSION}: rebuild with `python -m paper_2404_11631_b200.build`")
            for name, argt in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = argt
                fn.restype = ctypes.c_int64 if name in INT64_RESULT else ctypes.c_int
            _lib = lib
    if require_device:
        if not torch.cuda.is_available():
            raise DeviceError("no CUDA device visible: the sm_100a kernels have no CPU fallback")
        _device_ok = True
    return _lib


def exported_symbols():
    return ["simopt_last_error", "simopt_abi_version", *SIGNATURES]


def check(status: int):
    if status != 0:
        msg = _lib.simopt_last_error().decode(errors="replace") if _lib else ""
        raise STATUS_TO_ERROR.get(status, DeviceError)(msg)


def call(name: str, *args):
    lib = _lib if _device_ok else load()
    check(getattr(lib, name)(*args))


def stream_ptr(stream=None):
    if stream is None:
        return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(torch.cuda.current_device()))
    return ctypes.c_void_p(stream.cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)
