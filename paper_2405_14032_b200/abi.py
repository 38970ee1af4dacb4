"""ctypes binding of the C-ABI in include/gridnlp_b200.h.

The product path is the CUDA library `libgridnlp_b200.so` built in-tree by
`__graft_entry__.build()`.  There is no CPU fallback: importing this module
without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libgridnlp_b200.so"
# GRIDNLP_B200_LIB: load another build of the library (tuning variants, scripts/gpu_variants*.sh)
# instead of overwriting the in-tree one
LIB_ENV = "GRIDNLP_B200_LIB"

GN_OK, GN_ERR_INVALID, GN_ERR_EVAL, GN_ERR_CUDA, GN_ERR_UNSUPPORTED = 0, 1, 2, 3, 4
GN_MEM_HOST, GN_MEM_DEVICE, GN_MEM_DEVICE_ASYNC, GN_IN_FULL = 0, 1, 2, 16

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p


class GnError(C.Structure):
    _fields_ = [("code", C.c_int32), ("pattern", C.c_int32), ("record", C.c_int32),
                ("message", C.c_char * 244)]


class GnNetwork(C.Structure):
    """gn_network / or_network (identical layout)."""
    _fields_ = [
        ("n_bus", C.c_int32), ("n_line", C.c_int32), ("n_gen", C.c_int32),
        ("n_load", C.c_int32), ("reference_bus", C.c_int32),
        ("bus_vmin", f64p), ("bus_vmax", f64p), ("vm_start", f64p), ("va_start", f64p),
        ("line_from", i32p), ("line_to", i32p),
        ("line_g", f64p), ("line_b", f64p), ("line_smax", f64p), ("line_amin", f64p),
        ("line_amax", f64p),
        ("gen_bus", i32p),
        ("gen_pmin", f64p), ("gen_pmax", f64p), ("gen_qmin", f64p), ("gen_qmax", f64p),
        ("gen_ramp", f64p),
        ("gen_c2", f64p), ("gen_c1", f64p), ("gen_c0", f64p), ("gen_pstart", f64p),
        ("gen_qstart", f64p),
        ("load_bus", i32p),
        ("load_p", f64p), ("load_q", f64p),
    ]


class GnSizes(C.Structure):
    _fields_ = [(k, C.c_int64) for k in (
        "n_vars", "n_cons", "jac_nnz", "hess_nnz", "n_thermal", "n_ramp_gens", "periods",
        "n_free", "jac_nnz_lifted", "hess_nnz_lifted")]


class GnIterate(C.Structure):
    """gn_iterate: device pointers of an ipm::Iterate (iterate.hpp:16-19)."""
    _fields_ = [(k, vp) for k in ("x", "s", "y", "zlx", "zux", "zls", "zus")]


class GnResiduals(C.Structure):
    _fields_ = [(k, vp) for k in ("px", "ps", "py", "pzlx", "pzux", "pzls", "pzus")]


class GnDirection(C.Structure):
    _fields_ = [(k, vp) for k in ("dx", "ds", "dy", "dzlx", "dzux", "dzls", "dzus")]


_SIGS = {
    "gn_abi_version": (C.c_int, []),
    "gn_launch_count": (C.c_int64, []),
    "gn_device_count": (C.c_int, [i32p]),
    "gn_profile_enable": (None, [C.c_int]),
    "gn_profile_reset": (None, []),
    "gn_profile_count": (C.c_int, []),
    "gn_profile_get": (C.c_char_p, [C.c_int, f64p, i64p]),
    "gn_load_profile": (C.c_int, [C.c_int32, C.c_int32, C.c_double, C.c_uint64, C.c_double,
                                  C.c_double, f64p, C.POINTER(GnError)]),
    "gn_ctx_create": (C.c_int, [C.POINTER(GnNetwork), C.c_int32, f64p, C.c_int32,
                                C.POINTER(vp), C.POINTER(GnError)]),
    "gn_ctx_create_shard": (C.c_int, [C.POINTER(GnNetwork), C.c_int32, C.c_int32, C.c_int32, f64p,
                                      C.c_int32, C.POINTER(vp), C.POINTER(GnError)]),
    "gn_ctx_shard_info": (C.c_int, [vp, i64p, i32p]),
    "gn_ctx_destroy": (C.c_int, [vp]),
    "gn_ctx_publish": (C.c_int, [vp, C.c_int]),
    "gn_debug_kkt_guard": (C.c_int, [vp, C.c_int, C.c_uint64, i64p]),
    "gn_kkt_values_ptr": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp)]),
    "gn_kkt_values_start": (C.c_int, [vp, f64p, f64p]),
    "gn_kkt_values_wait": (C.c_int, [vp]),
    "gn_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(vp)]),
    "gn_host_free": (C.c_int, [vp]),
    "gn_halo_create": (C.c_int, [vp, C.c_int32, C.c_int32, C.POINTER(vp), C.POINTER(GnError)]),
    "gn_halo_ipc_handle": (C.c_int, [vp, vp]),
    "gn_halo_open": (C.c_int, [vp, vp]),
    "gn_halo_link": (C.c_int, [C.POINTER(vp), C.c_int32]),
    "gn_halo_exchange": (C.c_int, [vp, f64p, f64p, C.c_int, vp]),
    "gn_halo_objective": (C.c_int, [vp, f64p, f64p, C.c_int, vp]),
    "gn_halo_exchange_emulated": (C.c_int, [C.POINTER(vp), C.c_int32, C.POINTER(f64p),
                                            C.POINTER(f64p), vp]),
    "gn_halo_destroy": (C.c_int, [vp]),
    "gn_ctx_set_stream": (C.c_int, [vp, vp]),
    "gn_ctx_get_stream": (C.c_int, [vp, C.POINTER(vp)]),
    "gn_ctx_status": (C.c_int, [vp, C.POINTER(GnError)]),
    "gn_ctx_sizes": (C.c_int, [vp, C.POINTER(GnSizes)]),
    "gn_ctx_bounds": (C.c_int, [vp, f64p, f64p, f64p, f64p, f64p]),
    "gn_jac_structure": (C.c_int, [vp, i32p, i32p, C.c_int]),
    "gn_hess_structure": (C.c_int, [vp, i32p, i32p, C.c_int]),
    "gn_eval_f": (C.c_int, [vp, f64p, f64p, C.c_int, C.POINTER(GnError)]),
    "gn_eval_grad": (C.c_int, [vp, f64p, f64p, C.c_int, C.POINTER(GnError)]),
    "gn_eval_g": (C.c_int, [vp, f64p, f64p, C.c_int, C.POINTER(GnError)]),
    "gn_eval_jac": (C.c_int, [vp, f64p, f64p, C.c_int, C.POINTER(GnError)]),
    "gn_eval_hess": (C.c_int, [vp, f64p, f64p, C.c_double, f64p, C.c_int,
                               C.POINTER(GnError)]),
    "gn_eval_fg": (C.c_int, [vp, f64p, f64p, f64p, C.c_int, C.POINTER(GnError)]),
    "gn_eval_all": (C.c_int, [vp, f64p, f64p, C.c_double, f64p, f64p, f64p, f64p, f64p, C.c_int,
                              C.POINTER(GnError)]),
    "gn_ipm_create": (C.c_int, [vp, vp, vp, vp, vp, C.c_int, C.POINTER(vp), C.POINTER(GnError)]),
    "gn_ipm_destroy": (C.c_int, [vp]),
    "gn_ipm_jac_transpose_multiply": (C.c_int, [vp, vp, vp, vp, C.c_int]),
    "gn_ipm_jac_multiply": (C.c_int, [vp, vp, vp, vp, C.c_int]),
    "gn_ipm_residuals": (C.c_int, [vp, C.POINTER(GnIterate), vp, vp, vp, C.c_double,
                                   C.POINTER(GnResiduals), C.c_int]),
    "gn_ipm_bound_condensation": (C.c_int, [vp, C.POINTER(GnIterate), C.POINTER(GnResiduals),
                                            vp, vp, vp, vp, C.c_int]),
    "gn_ipm_fraction_to_boundary": (C.c_int, [vp, C.POINTER(GnIterate), C.POINTER(GnDirection),
                                              C.c_double, vp, C.c_int]),
    "gn_ipm_barrier_value": (C.c_int, [vp, C.c_double, vp, vp, C.c_double, vp, C.c_int]),
    "gn_ipm_barrier_slope": (C.c_int, [vp, vp, C.POINTER(GnIterate), C.POINTER(GnDirection),
                                       C.c_double, vp, C.c_int]),
    "gn_ipm_constraint_violation": (C.c_int, [vp, vp, vp, vp, C.c_int]),
    "gn_ipm_kkt_error": (C.c_int, [vp, C.POINTER(GnIterate), C.POINTER(GnResiduals), C.c_double,
                                   vp, C.c_int]),
    "gn_ipm_recover_bound_steps": (C.c_int, [vp, C.POINTER(GnIterate), C.POINTER(GnResiduals),
                                             C.POINTER(GnDirection), C.c_int]),
    "gn_kkt_solve_rhs": (C.c_int, [vp, vp, vp, vp, vp, C.c_double, C.c_double, vp, C.c_int]),
    "gn_kkt_solve_finish": (C.c_int, [vp, vp, vp, vp, vp, C.c_double, C.c_double, vp, vp,
                                      C.c_int]),
    "gn_lifted_create": (C.c_int, [vp, C.c_double, C.POINTER(GnError)]),
    "gn_lifted_structure": (C.c_int, [vp, i32p, i32p, i32p, i32p, i32p, i32p, i32p, f64p,
                                      f64p, C.c_int]),
    "gn_lifted_gather_jac": (C.c_int, [vp, f64p, f64p, C.c_int]),
    "gn_lifted_gather_hess": (C.c_int, [vp, f64p, f64p, C.c_int]),
    "gn_lifted_eval_f": (C.c_int, [vp, f64p, f64p, C.c_int, C.POINTER(GnError)]),
    "gn_lifted_eval_grad": (C.c_int, [vp, f64p, f64p, C.c_int, C.POINTER(GnError)]),
    "gn_lifted_eval_g": (C.c_int, [vp, f64p, f64p, C.c_int, C.POINTER(GnError)]),
    "gn_lifted_eval_jac": (C.c_int, [vp, f64p, f64p, C.c_int, C.POINTER(GnError)]),
    "gn_lifted_eval_hess": (C.c_int, [vp, f64p, f64p, C.c_double, f64p, C.c_int,
                                      C.POINTER(GnError)]),
    "gn_lifted_eval_fg": (C.c_int, [vp, f64p, f64p, f64p, C.c_int, C.POINTER(GnError)]),
    "gn_kkt_create": (C.c_int, [C.c_int32, C.c_int32, C.c_int64, i32p, i32p, C.c_int64, i32p,
                                i32p, C.c_int32, C.POINTER(vp), C.POINTER(GnError)]),
    "gn_kkt_create_lifted": (C.c_int, [vp, C.POINTER(vp), C.POINTER(GnError)]),
    "gn_kkt_destroy": (C.c_int, [vp]),
    "gn_kkt_set_stream": (C.c_int, [vp, vp]),
    "gn_kkt_dims": (C.c_int, [vp, i64p]),
    "gn_kkt_structure": (C.c_int, [vp, i32p, i32p, i32p, i32p, C.c_int]),
    "gn_kkt_slots": (C.c_int, [vp, i32p, i32p, i32p, i32p, C.c_int]),
    "gn_kkt_set_jacobian": (C.c_int, [vp, f64p, C.c_int]),
    "gn_kkt_assemble": (C.c_int, [vp, f64p, f64p, f64p, C.c_double, C.c_double, C.c_int]),
    "gn_kkt_values": (C.c_int, [vp, f64p, f64p, C.c_int]),
    "gn_kkt_set_jacobian_x": (C.c_int, [vp, f64p, C.c_int]),
    "gn_kkt_assemble_x": (C.c_int, [vp, f64p, f64p, C.c_double, f64p, f64p, C.c_double,
                                    C.c_double, C.c_int]),
    "gn_kkt_update_x": (C.c_int, [vp, f64p, f64p, C.c_double, f64p, f64p, C.c_double,
                                    C.c_double, C.c_int]),
    "gn_kkt_set_algorithm": (C.c_int, [vp, C.c_int]),
    "gn_kkt_set_grid_cap": (C.c_int, [vp, C.c_int]),
    "gn_compress_to_csc": (C.c_int, [C.c_int32, C.c_int32, C.c_int64, i32p, i32p, i32p, i32p,
                                     i32p, i32p, C.POINTER(GnError)]),
}

EXPORTED = tuple(_SIGS)


def load(path: Path | str | None = None) -> C.CDLL:
    path = Path(path or os.environ.get(LIB_ENV) or LIB_PATH)
    if not path.exists():
        raise ImportError(
            f"{path} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback.")
    lib = C.CDLL(str(path))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib: C.CDLL | None = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = load()
    return _lib
