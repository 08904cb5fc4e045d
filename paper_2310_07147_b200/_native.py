"""ctypes binding of the C-ABI (``include/qft_b200.h``) exported by the in-tree
``_lib/libqft_b200.so``.

There is no fallback: if the library is missing the import fails loudly, and on
a host without a CUDA device every compute entry point returns ``QFTC_ECUDA``,
which :func:`check` raises as ``RuntimeError``.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QFT_B200_LIB") or os.path.join(_HERE, "_lib", "libqft_b200.so")

QFTC_OK, QFTC_EINVAL, QFTC_ERANGE, QFTC_ECUDA, QFTC_EOVERFLOW, QFTC_ENOTSUP = 0, -1, -2, -3, -4, -5
GRAD_U8, GRAD_F32, GRAD_BF16 = 0, 1, 2
PERCENTILE, RANGE_FRACTION = 0, 1


class CsrOverflow(RuntimeError):
    """The new nnz exceeded the CSR arena capacity (QFTC_EOVERFLOW)."""


class LionHyperC(C.Structure):
    """``qftc_lion_hyper`` == ``LionHyper<float>`` (optimizer.hpp:15-21)."""
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float),
                ("weight_decay", C.c_float)]


class LionTensorC(C.Structure):
    """``qftc_lion_tensor``: one layer of a grouped quantized Lion step."""
    _fields_ = [
        ("rows", C.c_int32), ("cols", C.c_int32),
        ("w_codes", C.c_void_p * 2), ("row_start", C.c_void_p * 2),
        ("row_count", C.c_void_p * 2),
        ("w_scale", C.c_void_p), ("w_zero_point", C.c_void_p),
        ("t_min", C.c_void_p), ("t_max", C.c_void_p),
        ("m_codes", C.c_void_p * 2), ("m_scale", C.c_void_p * 2),
        ("m_zero_point", C.c_void_p * 2),
        ("g_codes", C.c_void_p), ("g_scale", C.c_void_p), ("g_zero_point", C.c_void_p),
        ("g_raw", C.c_void_p),
    ]


class ExpandTensorC(C.Structure):
    """``qftc_expand_tensor``: one tensor of a grouped weight expansion."""
    _fields_ = [
        ("rows", C.c_int32), ("cols", C.c_int32),
        ("codes", C.c_void_p), ("scale", C.c_void_p), ("zero_point", C.c_void_p),
        ("row_start", C.c_void_p), ("row_count", C.c_void_p),
        ("col_idx", C.c_void_p), ("values", C.c_void_p), ("out", C.c_void_p),
    ]


class PackSegmentC(C.Structure):
    """``qftc_pack_segment``: one slotted segment of a ZeRO-1 packed CSR gather."""
    _fields_ = [("rows", C.c_int32), ("width", C.c_int32), ("rs_off", C.c_int64),
                ("cnt_off", C.c_int64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the sm_100a library first "
            "(python -m paper_2310_07147_b200.build or __graft_entry__.build())")
    return C.CDLL(LIB_PATH)


lib = _load()

_vp, _i, _i64, _d, _u64 = C.c_void_p, C.c_int, C.c_int64, C.c_double, C.c_uint64

_SIGS = {
    "qftc_last_error": (C.c_char_p, []),
    "qftc_version": (_i, []),
    "qftc_max_cols": (_i, []),
    "qftc_channel_minmax": (_i, [_vp, _i, _i, _vp, _vp, _vp]),
    "qftc_affine_params_from_bounds": (_i, [_vp, _vp, _i64, _i, _vp, _vp, _vp]),
    "qftc_quantize": (_i, [_vp, _i, _i, _vp, _vp, _i, _i, _vp, _vp]),
    "qftc_quantize_state": (_i, [_vp, _i, _i, _i, _vp, _vp, _vp, _i, _vp]),
    "qftc_dequantize": (_i, [_vp, _i, _i, _vp, _vp, _i, _vp, _vp]),
    "qftc_dequantize_bf16": (_i, [_vp, _i, _i, _vp, _vp, _i, _vp, _vp]),
    "qftc_outlier_thresholds": (_i, [_vp, _i, _i, _d, _i, _vp, _vp, _vp]),
    "qftc_decompose_dense_sparse": (_i, [_vp, _i, _i, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp,
                                         _vp, _i64, C.POINTER(_i64), _vp]),
    "qftc_reconstruct": (_i, [_vp, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "qftc_reconstruct_bf16": (_i, [_vp, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "qftc_plan_create": (_i, [C.POINTER(_vp), C.POINTER(LionTensorC), _i, _i, _i,
                              C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_i64), _vp]),
    "qftc_plan_set_arena": (_i, [_vp, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_i64)]),
    "qftc_plan_step": (_i, [_vp, _i, LionHyperC, _vp]),
    "qftc_plans_step": (_i, [C.POINTER(_vp), _i, _i, LionHyperC, _vp]),
    "qftc_pack_codes": (_i, [_vp, _i, _i, _i, _vp, _vp]),
    "qftc_unpack_codes": (_i, [_vp, _i, _i, _i, _vp, _vp]),
    "qftc_momentum_to_blocks": (_i, [_vp, _vp, _vp, _i, _i, _i, _i, _vp, _vp, _vp, _vp]),
    "qftc_momentum_from_blocks": (_i, [_vp, _vp, _vp, _i, _i, _i, _i, _vp, _vp, _vp, _vp]),
    "qftc_dequant_gemm_workspace_bytes": (_i64, [_i, _i]),
    "qftc_dequant_gemm_index": (_i, [_vp, _vp, _vp, _i, _i, _vp, _vp]),
    "qftc_dequant_gemm_prebuilt": (_i, [_vp, _i, _i, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "qftc_dequant_gemm_t_prebuilt": (_i, [_vp, _i, _i, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "qftc_dequant_gemm": (_i, [_vp, _i, _i, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "qftc_wgrad_workspace_bytes": (_i64, [_i]),
    "qftc_dequant_gemm_t_workspace_bytes": (_i64, [_i, _i]),
    "qftc_dequant_gemm_t": (_i, [_vp, _i, _i, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "qftc_wgrad_quant": (_i, [_vp, _vp, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _i, _vp]),
    "qftc_expand_plan_create": (_i, [C.POINTER(_vp), C.POINTER(ExpandTensorC), _i, _i, _vp]),
    "qftc_expand_plan_run": (_i, [_vp, _vp]),
    "qftc_expand_plan_destroy": (_i, [_vp]),
    "qftc_plan_set_ctas_per_sm": (_i, [_vp, _i]),
    "qftc_plan_set_peer_gradients": (_i, [_vp, C.POINTER(_i64), _i]),
    "qftc_ipc_handle": (_i, [_vp, C.c_char_p, C.POINTER(_i64)]),
    "qftc_ipc_open": (_i, [C.c_char_p, C.POINTER(_vp)]),
    "qftc_ipc_close": (_i, [_vp]),
    "qftc_copy_peer": (_i, [_vp, _vp, C.c_size_t, _vp]),
    "qftc_plan_result": (_i, [_vp, C.POINTER(_i64), _vp]),
    "qftc_plan_launches": (_i, [_vp]),
    "qftc_plan_kernel_name": (C.c_char_p, [_vp]),
    "qftc_plan_pending_overflow": (_i, [_vp]),
    "qftc_plan_tier_rows": (_i, [_vp, C.POINTER(_i64), C.POINTER(_i64), _vp]),
    "qftc_plan_tiers": (_i, [_vp, C.POINTER(_i64), _vp]),
    "qftc_crc32": (_i, [_vp, _vp, _i, _vp, _vp]),
    "qftc_accumulate_state": (_i, [_vp, _vp, _vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp]),
    "qftc_plan_destroy": (_i, [_vp]),
    "qftc_lion_step": (_i, [_i, _i, _i] + [_vp] * 21 + [_i64, LionHyperC, C.POINTER(_i64), _vp]),
    "qftc_lion_apply": (_i, [_vp, _vp, _vp, _i64, LionHyperC, _vp]),
    "qftc_synth": (_i, [_vp, _i64, _u64, _d, _d, _vp]),
    "qftc_csr_replan_caps": (_i, [_vp, _i, _i, _i, _vp, _vp, _i, _i, _vp, _vp]),
    "qftc_csr_plan_slots": (_i, [_vp, _vp, _i, _i, _vp, C.POINTER(_i64), _vp]),
    "qftc_csr_copy_rows": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp]),
    "qftc_csr_compact": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, C.POINTER(_i64),
                              _vp]),
    "qftc_csr_pack_plan_create": (_i, [C.POINTER(_vp), C.POINTER(PackSegmentC), _i, _i, _vp]),
    "qftc_csr_pack_run": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, C.POINTER(_i64), _vp, _vp]),
    "qftc_csr_pack_plan_destroy": (_i, [_vp]),
    "qftc_reconstruct_slots": (_i, [_vp, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _vp]),
    "qftc_expand": (_i, [_vp, _i, _i, _vp]),
    "qftc_device_alloc": (_i, [C.POINTER(_vp), C.c_size_t]),
    "qftc_device_free": (_i, [_vp]),
    "qftc_copy_to_device": (_i, [_vp, _vp, C.c_size_t, _vp]),
    "qftc_copy_to_host": (_i, [_vp, _vp, C.c_size_t, _vp]),
    "qftc_memset": (_i, [_vp, _i, C.c_size_t, _vp]),
    "qftc_stream_synchronize": (_i, [_vp]),
}

EXPORTS = tuple(_SIGS)

for _name, (_res, _args) in _SIGS.items():
    if os.environ.get("QFT_B200_LIB") and not hasattr(lib, _name):
        continue  # an older library build loaded for an A/B (tools/build_variant.py)
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def last_error() -> str:
    return lib.qftc_last_error().decode()


def check(rc: int) -> int:
    """Map a status code onto the reference's exception types
    (std::invalid_argument -> ValueError, std::out_of_range -> IndexError)."""
    if rc == QFTC_OK:
        return rc
    msg = last_error()
    if rc == QFTC_EINVAL:
        raise ValueError(msg)
    if rc == QFTC_ERANGE:
        raise IndexError(msg)
    if rc == QFTC_EOVERFLOW:
        raise CsrOverflow(msg)
    if rc == QFTC_ENOTSUP:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


def hyper(lr=1e-4, beta1=0.9, beta2=0.99, weight_decay=0.0) -> LionHyperC:
    return LionHyperC(lr, beta1, beta2, weight_decay)
