// TEMPORARY: entry points whose implementation lands next (Schwarz, pMG). Each returns EINVAL.
#include "capi_util.hpp"

extern "C" {
#define SB_PENDING(name, ...) \
  int name(__VA_ARGS__) { return guard([&] { sb::invalid(#name ": not built yet"); }); }
SB_PENDING(semlab_op_schwarz, semlab_schwarz, semlab_op*)
SB_PENDING(semlab_op_pmg, semlab_pmg, semlab_op*)
SB_PENDING(semlab_schwarz_create, semlab_space, int, int, semlab_schwarz*)
SB_PENDING(semlab_schwarz_destroy, semlab_schwarz)
SB_PENDING(semlab_schwarz_apply, semlab_schwarz, const double*, double*)
SB_PENDING(semlab_schwarz_fdm_solve_all, semlab_schwarz, const double*, double*)
SB_PENDING(semlab_schwarz_element_info, semlab_schwarz, int, double*, int*, double*)
SB_PENDING(semlab_pmg_create, semlab_mesh, int, const int*, int, int, double, double, int, int, semlab_pmg*)
SB_PENDING(semlab_pmg_destroy, semlab_pmg)
SB_PENDING(semlab_pmg_vcycle, semlab_pmg, const double*, double*)
SB_PENDING(semlab_pmg_space, semlab_pmg, int, semlab_space*)
SB_PENDING(semlab_pmg_lambda, semlab_pmg, int, double*)
SB_PENDING(semlab_pmg_prolong, semlab_pmg, int, const double*, double*)
SB_PENDING(semlab_pmg_restrict, semlab_pmg, int, const double*, double*)
}
