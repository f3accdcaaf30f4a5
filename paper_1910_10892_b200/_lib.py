"""ctypes binding of libmrf_cuda.so (the C-ABI in include/mrf_cuda.h).

The shared library is built in-tree by ``paper_1910_10892_b200.build`` (or
``__graft_entry__.build()``). There is no fallback: if it is missing, every
entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MRF_LIB_PATH") or os.path.join(HERE, "libmrf_cuda.so")  # override: A/B builds

MRF_OK, MRF_EINVAL, MRF_ECUDA, MRF_ENOMEM = 0, 1, 2, 3
ENGINE_ISGMR, ENGINE_TRWP = 0, 1


class MrfError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[mrf code {code}] {msg}")
        self.code = code


class MrfInvalidArgument(MrfError, ValueError):
    """Raised for MRF_EINVAL (the reference's std::invalid_argument cases)."""


class Problem(C.Structure):
    _fields_ = [("batch", C.c_int), ("height", C.c_int), ("width", C.c_int), ("labels", C.c_int),
                ("unary", C.c_void_p), ("pairwise", C.c_void_p), ("weight", C.c_float),
                ("weight_planes", C.c_void_p), ("rho", C.c_float), ("rho_planes", C.c_void_p),
                ("assume_finite", C.c_int), ("diag_gap", C.c_void_p)]


class ForwardOut(C.Structure):
    _fields_ = [("cost", C.c_void_p), ("labels", C.c_void_p), ("messages", C.c_void_p), ("p", C.c_void_p),
                ("q", C.c_void_p)]


class Grads(C.Structure):
    _fields_ = [("unary", C.c_void_p), ("pairwise", C.c_void_p), ("weight_planes", C.c_void_p)]


# Every symbol include/mrf_cuda.h declares, with its ctypes signature.
_vp, _i, _sz, _i64p = C.c_void_p, C.c_int, C.c_size_t, C.POINTER(C.c_int64)
_PP, _FO, _GR = C.POINTER(Problem), C.POINTER(ForwardOut), C.POINTER(Grads)
SIGNATURES = {
    "mrf_last_error": (C.c_char_p, []),
    "mrf_version": (_i, []),
    "mrf_topology_create": (_i, [_i, _i, _i, C.POINTER(_vp)]),
    "mrf_topology_destroy": (_i, [_vp]),
    "mrf_topology_info": (_i, [_vp, C.POINTER(_i), _i64p, _i64p, _i64p]),
    "mrf_topology_edge_index": (_i, [_vp, _vp]),
    "mrf_topology_scanlines": (_i, [_vp, _i, _vp, _vp, C.POINTER(C.c_int32), _i]),
    "mrf_check_finite_f32": (_i, [_vp, _sz, C.POINTER(_i), _vp]),
    "mrf_forward_workspace_bytes": (_sz, [_vp, _PP, _i, _i]),
    "mrf_isgmr_forward_f32": (_i, [_vp, _PP, _i, _FO, _vp, _sz, _vp]),
    "mrf_trwp_forward_f32": (_i, [_vp, _PP, _i, _FO, _vp, _sz, _vp]),
    "mrf_isgmr_step_f32": (_i, [_vp, _PP, _i, _i, _vp, _vp, _vp, _vp, _vp]),
    "mrf_trwp_step_f32": (_i, [_vp, _PP, _i, _i, _vp, _vp, _vp, _vp]),
    "mrf_aggregate_f32": (_i, [_vp, _PP, _vp, _vp, _vp, _vp]),
    "mrf_backward_workspace_bytes": (_sz, [_vp, _PP, _i, _i]),
    "mrf_isgmr_backward_f32": (_i, [_vp, _PP, _i, _vp, _vp, _vp, _GR, _vp, _sz, _vp]),
    "mrf_trwp_backward_f32": (_i, [_vp, _PP, _i, _vp, _vp, _vp, _GR, _vp, _sz, _vp]),
    "mrf_pack_shared_grads_f32": (_i, [_PP, _i, _GR, _vp, _vp]),
    "mrf_allreduce_grads_f32": (_i, [_vp, _vp, _sz, _vp]),
    "mrf_nccl_unique_id": (_i, [_vp, _sz]),
    "mrf_nccl_comm_init": (_i, [C.POINTER(_vp), _i, _vp, _i]),
    "mrf_nccl_comm_destroy": (_i, [_vp]),
    "mrf_soft_head_f32": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "mrf_energy_f32": (_i, [_vp, _PP, _vp, C.POINTER(C.c_double), _vp]),
    "mrf_sgm_f32": (_i, [_vp, _PP, _i, _vp, _vp, _vp, _vp]),
    "mrf_sgm_next_unary_f32": (_i, [_vp, _PP, _vp, _vp, _vp]),
    "mrf_profiler_enable": (_i, [_i]),
    "mrf_profiler_read": (_i, [_i, C.POINTER(C.c_double), _i64p]),
    "mrf_launch_count": (_i, [_i64p]),
}
KCLASS_FWD_SWEEP, KCLASS_BWD_SWEEP, KCLASS_AGGREGATE, KCLASS_AUX = 0, 1, 2, 3

_lib = None


def lib():
    """Load libmrf_cuda.so (once). Raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run paper_1910_10892_b200.build.build() "
                               "(or __graft_entry__.build()); there is no CPU fallback")
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(rc: int) -> None:
    if rc != MRF_OK:
        msg = lib().mrf_last_error().decode(errors="replace")
        if rc == MRF_EINVAL:
            raise MrfInvalidArgument(rc, msg)
        raise MrfError(rc, msg)
