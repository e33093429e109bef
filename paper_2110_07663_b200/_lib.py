"""ctypes binding of libsemlab_b200.so (the C-ABI of include/semlab_b200.h).

The library is built in-tree (`make`, or __graft_entry__.build()). There is no fallback: if the
shared object is missing or stale, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SEMLAB_LIB selects another in-tree build of the same C-ABI (A/B timing of kernel variants)
LIB_PATH = os.path.join(_HERE, os.environ.get("SEMLAB_LIB", "libsemlab_b200.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA extension first (`make` at the repo root or "
        "`python -c 'import __graft_entry__ as g; g.build()'`). There is no CPU fallback.")

lib = C.CDLL(LIB_PATH)

p = C.c_void_p
i32, i64, u64, f64 = C.c_int, C.c_int64, C.c_uint64, C.c_double
pf64 = C.POINTER(C.c_double)
pi64 = C.POINTER(C.c_int64)
pi32 = C.POINTER(C.c_int)


class ChebyParams(C.Structure):
    """ChebyParams, chebyshev.hpp:9-14."""
    _fields_ = [("order", i32), ("lambda_min_mult", f64), ("lambda_max_mult", f64), ("lambda_max_est", f64)]


class LambdaEstimateC(C.Structure):
    """LambdaEstimate, chebyshev.hpp:16-20."""
    _fields_ = [("value", f64), ("breakdown", i32), ("rounds_used", i32)]


class GmresConfigC(C.Structure):
    """GmresConfig, krylov.hpp:9-15."""
    _fields_ = [("restart", i32), ("tol", f64), ("max_iters", i32), ("use_abs_tol", i32), ("abs_tol", f64)]


class GmresStatsC(C.Structure):
    """GmresStats, krylov.hpp:17-25."""
    _fields_ = [("iterations", i32), ("converged", i32), ("breakdown", i32), ("initial_residual", f64),
                ("abs_residual", f64), ("rel_residual", f64), ("history", pf64), ("history_capacity", i32),
                ("history_len", i32)]


class PmgOptionsC(C.Structure):
    """semlab_pmg_options."""
    _fields_ = [("smoother", i32), ("cheb_order", i32), ("lambda_min_mult", f64), ("lambda_max_mult", f64),
                ("precision", i32), ("coarse", i32), ("bc", i32), ("cycle", i32)]


MAP_FN = C.CFUNCTYPE(None, p, f64, f64, f64, pf64)
APPLY_FN = C.CFUNCTYPE(None, p, p, p)

# name: (restype, argtypes)
SIGNATURES = {
    "semlab_last_error": (C.c_char_p, []),
    "semlab_version": (C.c_char_p, []),
    "semlab_debug_set_grid_cap": (i32, [i32]),
    "semlab_debug_set_gmres_form": (i32, [i32]),
    "semlab_ctx_create": (i32, [i32, p, C.POINTER(p)]),
    "semlab_ctx_create_dist": (i32, [i32, p, i32, i32, p, C.POINTER(p)]),
    "semlab_nccl_get_unique_id": (i32, [p]),
    "semlab_ctx_set_exchange": (i32, [p, i32]),
    "semlab_ctx_destroy": (i32, [p]),
    "semlab_ctx_synchronize": (i32, [p]),
    "semlab_ctx_launch_count": (i64, [p]),
    "semlab_mesh_kershaw": (i32, [p, f64, i32, C.POINTER(p)]),
    "semlab_mesh_box": (i32, [p, pi32, pf64, pf64, C.POINTER(p)]),
    "semlab_mesh_from_map": (i32, [p, pi32, MAP_FN, p, C.POINTER(p)]),
    "semlab_mesh_destroy": (i32, [p]),
    "semlab_mesh_lattice_coords": (i32, [p, i32, pf64, i64]),
    "semlab_space_create": (i32, [p, i32, i32, C.POINTER(p)]),
    "semlab_space_destroy": (i32, [p]),
    "semlab_space_sizes": (i32, [p, pi64]),
    "semlab_space_apply_A": (i32, [p, p, p]),
    "semlab_space_apply_A_geom32": (i32, [p, p, p]),
    "semlab_space_apply_local_stiffness": (i32, [p, p, p]),
    "semlab_space_gather": (i32, [p, p, p]),
    "semlab_space_scatter": (i32, [p, p, p]),
    "semlab_space_gather_scatter": (i32, [p, p, p]),
    "semlab_space_mask": (i32, [p, p]),
    "semlab_space_stiffness_diag": (i32, [p, p]),
    "semlab_space_mass_diag": (i32, [p, p]),
    "semlab_space_metric": (i32, [p, i32, pf64]),
    "semlab_space_build_rhs": (i32, [p, u64, p]),
    "semlab_space_dot": (i32, [p, p, p, pf64]),
    "semlab_op_A": (i32, [p, C.POINTER(p)]),
    "semlab_op_A_geom32": (i32, [p, C.POINTER(p)]),
    "semlab_op_jacobi": (i32, [p, C.POINTER(p)]),
    "semlab_op_schwarz": (i32, [p, C.POINTER(p)]),
    "semlab_op_pmg": (i32, [p, C.POINTER(p)]),
    "semlab_op_callback": (i32, [p, i64, APPLY_FN, p, C.POINTER(p)]),
    "semlab_op_apply": (i32, [p, p, p]),
    "semlab_op_destroy": (i32, [p]),
    "semlab_schwarz_create": (i32, [p, i32, i32, C.POINTER(p)]),
    "semlab_schwarz_destroy": (i32, [p]),
    "semlab_schwarz_apply": (i32, [p, p, p]),
    "semlab_schwarz_fdm_solve_all": (i32, [p, p, p]),
    "semlab_schwarz_element_info": (i32, [p, i32, pf64, pi32, pf64]),
    "semlab_estimate_lambda_max": (i32, [p, p, i64, i32, u64, C.POINTER(LambdaEstimateC)]),
    "semlab_cheby_create": (i32, [p, p, C.POINTER(ChebyParams), C.POINTER(p)]),
    "semlab_cheby_destroy": (i32, [p]),
    "semlab_cheby_smooth": (i32, [p, p, p]),
    "semlab_pmg_create": (i32, [p, i32, pi32, i32, i32, f64, f64, i32, i32, C.POINTER(p)]),
    "semlab_pmg_create_ex": (i32, [p, i32, pi32, C.POINTER(PmgOptionsC), C.POINTER(p)]),
    "semlab_pmg_destroy": (i32, [p]),
    "semlab_pmg_vcycle": (i32, [p, p, p]),
    "semlab_pmg_space": (i32, [p, i32, C.POINTER(p)]),
    "semlab_pmg_lambda": (i32, [p, i32, pf64]),
    "semlab_pmg_coarse_info": (i32, [p, pi32, pi64, i32]),
    "semlab_pmg_prolong": (i32, [p, i32, p, p]),
    "semlab_pmg_restrict": (i32, [p, i32, p, p]),
    "semlab_semfem_create": (i32, [p, C.POINTER(p)]),
    "semlab_semfem_destroy": (i32, [p]),
    "semlab_semfem_apply": (i32, [p, p, p]),
    "semlab_semfem_levels": (i32, [p, pi32, pi64, i32]),
    "semlab_op_semfem": (i32, [p, C.POINTER(p)]),
    "semlab_gmres_solve": (i32, [p, p, p, p, C.POINTER(GmresConfigC), C.POINTER(GmresStatsC)]),
    "semlab_pcg_solve": (i32, [p, p, p, p, C.POINTER(GmresConfigC), C.POINTER(GmresStatsC)]),
    "semlab_proj_create": (i32, [p, i64, i32, C.POINTER(p)]),
    "semlab_proj_destroy": (i32, [p]),
    "semlab_proj_initial_guess": (i32, [p, p, p]),
    "semlab_proj_insert": (i32, [p, p, p]),
    "semlab_proj_size": (i32, [p, C.POINTER(i32)]),
    "semlab_proj_clear": (i32, [p]),
    "semlab_proj_vector": (i32, [p, i32, p]),
    "semlab_host_gll": (i32, [i32, pf64, pf64, pf64]),
    "semlab_host_kershaw_map": (i32, [f64, f64, f64, f64, pf64]),
    "semlab_host_uniform_pm1": (i32, [u64, i64, pf64]),
    "semlab_host_gen_eig": (i32, [i32, pf64, pf64, pf64, pf64]),
    "semlab_host_max_abs_eig": (i32, [i32, pf64, pf64]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _f = getattr(lib, _name)  # AttributeError here = the .so does not export a declared symbol
    _f.restype = _res
    _f.argtypes = _args

SEMLAB_OK, SEMLAB_EINVAL, SEMLAB_ENUMERIC, SEMLAB_ECUDA, SEMLAB_ENCCL = 0, 1, 2, 3, 4


class SemlabCudaError(RuntimeError):
    pass


class SemlabNcclError(RuntimeError):
    pass


def check(code: int):
    """Re-raise the reference's exception type for a non-zero status."""
    if code == SEMLAB_OK:
        return
    msg = lib.semlab_last_error().decode()
    if code == SEMLAB_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if code == SEMLAB_ENUMERIC:
        raise RuntimeError(msg)  # std::runtime_error
    if code == SEMLAB_ECUDA:
        raise SemlabCudaError(msg)
    if code == SEMLAB_ENCCL:
        raise SemlabNcclError(msg)
    raise RuntimeError(f"semlab status {code}: {msg}")
