"""ctypes binding of the C-ABI library ``libdlrsn.so`` (include/dlrsn.h).

The library is built in-tree (``paper_2601_18705_b200/build.py``) and loaded
from the package directory; there is no fallback: if the library is missing
or no CUDA device is visible, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import ContractViolation, InterpolationError, SolverError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DLRSN_LIB") or os.path.join(HERE, "libdlrsn.so")  # DLRSN_LIB: A/B builds

MAX_DW = 8

c_int = ctypes.c_int
c_i64 = ctypes.c_int64
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p


class CellOps(ctypes.Structure):
    _fields_ = [
        ("nx", c_int), ("ny", c_int),
        ("x0", c_dbl), ("y0", c_dbl), ("dx", c_dbl), ("dy", c_dbl),
        ("mass", c_dbl * 16), ("gx", c_dbl * 16), ("gy", c_dbl * 16),
        ("e2x", c_dbl * 4), ("e2y", c_dbl * 4), ("src_row", c_dbl * 4),
    ]


MAX_RANK = 128


class Advance(ctypes.Structure):  # struct dlrsn_advance
    _fields_ = [("n", c_int), ("T_in", c_vp), ("sigma_a_in", c_vp), ("denom_in", c_vp),
                ("sigma_a0", c_vp), ("opacity_power", c_dbl), ("rho_cv", c_vp), ("dt", c_dbl),
                ("c", c_dbl), ("a_r", c_dbl), ("t_floor", c_dbl), ("ss_phys", c_vp),
                ("q_ext", c_vp), ("T_out", c_vp), ("sigma_a", c_vp), ("sigma_t", c_vp),
                ("sigma_s", c_vp), ("q", c_vp), ("denom", c_vp)]


class StepParams(ctypes.Structure):
    _fields_ = [("rank", c_int), ("n_omega", c_int), ("omegas_host", c_vp), ("omegas_dev", c_vp),
                ("weights_dev", c_vp), ("inv_cdt", c_dbl), ("si_tol", c_dbl),
                ("si_max_iters", c_int), ("check_state", c_int), ("gs_method", c_int),
                ("sweep_dw", c_int), ("advance", c_vp), ("inflow", c_dbl * 4),
                ("x_check_in", c_vp), ("x_check_out", c_vp), ("si_batch_hint", c_int),
                ("angle_override", c_int), ("angle_indices_in", c_vp), ("x_new_host", c_vp),
                ("use_dsa", c_int), ("dsa_penalty", c_int), ("dsa_tol", c_dbl),
                ("dsa_max_iters", c_int), ("dsa_history", c_vp), ("dsa_hist_cap", c_int)]


class StepInfo(ctypes.Structure):
    _fields_ = [("iterations", c_int), ("spatial_deficiency", c_int),
                ("angular_deficiency", c_int), ("error_index", c_int), ("gs_fallback", c_int),
                ("residual", c_dbl), ("check_in", c_dbl * 2), ("check_out", c_dbl * 2),
                ("angle_indices", c_i64 * MAX_RANK), ("closure", c_dbl * MAX_RANK),
                ("si_batch_hint", c_int), ("sweep_status", c_int), ("deim_gap", c_dbl * MAX_RANK),
                ("dsa_iterations", c_int), ("dsa_solves", c_int)]


COMM_FN = ctypes.CFUNCTYPE(c_int, c_vp)


class Comm(ctypes.Structure):
    _fields_ = [("rank", c_int), ("world_size", c_int), ("user", c_vp),
                ("allreduce_sum", COMM_FN), ("allgather", COMM_FN), ("reduce_buf", c_vp),
                ("gather_send", c_vp), ("gather_recv", c_vp), ("gather_width", c_int)]


# numpy mirror of struct dlrsn_group (include/dlrsn.h)
GROUP_DTYPE = np.dtype([
    ("quad", np.int32), ("ndir", np.int32), ("slot", np.int32, (MAX_DW,)),
    ("ox", np.float64, (MAX_DW,)), ("oy", np.float64, (MAX_DW,)), ("cw", np.float64, (MAX_DW,)),
], align=True)

# name -> (restype, argtypes); keep in sync with include/dlrsn.h
_SIGNATURES = {
    "dlrsn_version": (c_int, []),
    "dlrsn_launch_count": (c_i64, []),
    "dlrsn_last_error": (ctypes.c_char_p, []),
    "dlrsn_device_sm_count": (c_int, [c_vp]),
    "dlrsn_sk_vec_len": (c_i64, [c_int, c_int]),
    "dlrsn_sk_scalar_len": (c_i64, [c_int, c_int]),
    "dlrsn_sweep_workspace_bytes": (c_i64, [c_int, c_int, c_int, c_int]),
    "dlrsn_sweep_workspace_init": (c_int, [c_vp, c_i64, c_vp]),
    "dlrsn_debug_trace": (c_int, [c_vp, c_int]),
    "dlrsn_debug_flags": (c_int, [c_int]),
    "dlrsn_linearize": (c_int, [c_int, c_vp, c_vp, c_vp, c_dbl, c_dbl, c_dbl, c_vp, c_vp,
                                c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "dlrsn_update_temperature": (c_int, [c_int, c_vp, c_int, c_vp, c_vp, c_vp, c_dbl, c_dbl,
                                         c_dbl, c_dbl, c_vp, c_vp]),
    "dlrsn_advance_relinearize": (c_int, [c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_dbl,
                                          c_vp, c_dbl, c_dbl, c_dbl, c_dbl, c_vp, c_vp, c_vp,
                                          c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "dlrsn_rhs_build": (c_int, [c_vp, c_int, c_vp, c_vp, c_dbl, c_vp, c_int, c_vp, c_int, c_vp,
                                c_vp]),
    "dlrsn_inflow_add": (c_int, [c_vp, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "dlrsn_inflow_project": (c_int, [c_vp, c_int, c_vp, c_int, c_vp, c_vp, c_vp]),
    "dlrsn_dsa_workspace_len": (c_i64, [c_int, c_int]),
    "dlrsn_dsa_correct": (c_int, [c_vp, c_vp, c_vp, c_dbl, c_dbl, c_vp, c_vp, c_vp, c_dbl, c_int,
                                  c_vp, c_i64, c_vp, c_vp, c_int, c_vp]),
    "dlrsn_cells_to_sk4": (c_int, [c_vp, c_vp, c_vp, c_vp]),
    "dlrsn_scatter_source": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "dlrsn_phi_combine": (c_int, [c_vp, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                  c_vp, c_vp]),
    "dlrsn_phi_finish": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "dlrsn_sk_to_canonical": (c_int, [c_vp, c_int, c_vp, c_vp, c_vp, c_int, c_vp]),
    "dlrsn_sweep": (c_int, [c_vp, c_int, c_vp, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64,
                            c_int, c_vp]),
    "dlrsn_sweep_closure": (c_int, [c_vp, c_int, c_vp, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64,
                                    c_int, c_vp]),
    "dlrsn_rowmix": (c_int, [c_i64, c_int, c_int, c_vp, c_int, c_vp, c_int, c_dbl, c_vp, c_int,
                             c_vp]),
    "dlrsn_rowmix_upper": (c_int, [c_i64, c_int, c_vp, c_int, c_vp, c_int, c_vp, c_int, c_vp]),
    "dlrsn_partials_len": (c_i64, [c_int, c_int, c_int, c_int]),
    "dlrsn_mgram": (c_int, [c_vp, c_int, c_int, c_vp, c_int, c_vp, c_int, c_vp, c_vp, c_vp, c_vp]),
    "dlrsn_project": (c_int, [c_vp, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "dlrsn_chol_upper": (c_int, [c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "dlrsn_small_matmul": (c_int, [c_int, c_int, c_int, c_vp, c_vp, c_vp, c_int, c_vp]),
    "dlrsn_row_inverse": (c_int, [c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "dlrsn_row_combine": (c_int, [c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "dlrsn_deim": (c_int, [c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_vp]),
    "dlrsn_dmma_probe": (c_int, [c_int, c_int, c_int, c_vp, c_vp]),
    "dlrsn_project_slab": (c_int, [c_vp, c_int, c_vp, c_vp, c_vp, c_int, c_vp, c_vp, c_vp, c_vp,
                                   c_vp, c_vp]),
    "dlrsn_project_timing": (c_int, [c_int]),
    "dlrsn_project_timing_read": (c_int, [c_int, c_vp, c_vp]),
    "dlrsn_deim_forced": (c_int, [c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "dlrsn_what_solve": (c_int, [c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_int, c_vp]),
    "dlrsn_cgs2_workspace_len": (c_i64, [c_int]),
    "dlrsn_cholqr2_small_smem": (c_i64, [c_int, c_int]),
    "dlrsn_cholqr2_small": (c_int, [c_int, c_int, c_vp, c_int, c_vp, c_vp, c_int, c_vp, c_vp, c_vp,
                                    c_vp, c_vp]),
    "dlrsn_sweep_timing": (c_int, [c_int]),
    "dlrsn_sweep_timing_read": (c_int, [c_int, c_vp, c_vp, c_vp, c_vp]),
    "dlrsn_step_workspace_bytes": (c_i64, [c_int, c_int, c_int, c_int, c_int]),
    "dlrsn_step_collocation": (c_int, [c_vp] * 16 + [c_i64, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "dlrsn_cgs2": (c_int, [c_int, c_int, c_vp, c_int, c_vp, c_int, c_vp, c_vp, c_int, c_vp, c_vp,
                           c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_int, c_vp]),
}

_lib = None


def exported_symbols():
    return sorted(_SIGNATURES)


def load(path=LIB_PATH):
    """Load (once) and type the library; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (the B200 path has no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status, what=""):
    if status == 0:
        return
    msg = load().dlrsn_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status == -1 or status == -6:
        raise ContractViolation(text)
    if status == -5:
        raise InterpolationError(text, column=-1)
    if status == -7:
        raise SolverError(text)
    if status in (-2, -3):
        raise SolverError(text)
    raise RuntimeError(f"dlrsn CUDA failure ({status}): {text}")




def call(name, *args):
    nargs = len(_SIGNATURES[name][1])
    if len(args) != nargs:  # ctypes would pass surplus arguments through
        raise TypeError(f"{name} takes {nargs} arguments ({len(args)} given)")
    check(getattr(load(), name)(*args), name)


def ptr(t):
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else c_vp(t.data_ptr())


def stream_handle(device=None):
    import torch

    return c_vp(torch.cuda.current_stream(device).cuda_stream)


def launch_count():
    """Kernels the library has launched since it was loaded (counted in C++
    at every launch site, csrc/common.cuh DLRSN_CHECK_LAUNCH)."""
    return int(load().dlrsn_launch_count())
