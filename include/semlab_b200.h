/*
 * semlab_b200 — C-ABI of the B200-native spectral-element pressure-Poisson hot path.
 *
 * Drop-in boundary for the reference library semlab (/root/reference/proj/core). The
 * reference passes every operator across layers as
 *     using LinOp = std::function<void(const Eigen::VectorXd&, Eigen::VectorXd&)>;   (types.hpp:13)
 * over host Eigen vectors. Here every object is an opaque handle, every vector is a DEVICE
 * pointer (double*, length = the object's n) that stays resident for the whole solve, and
 * every call is stream-ordered on the context's CUDA stream. No exception crosses this
 * boundary: calls return a status code and semlab_last_error() holds the message, using the
 * reference's exception texts (std::invalid_argument -> SEMLAB_EINVAL, std::runtime_error ->
 * SEMLAB_ENUMERIC). Non-convergence is NOT an error (GmresStats::converged, krylov.cpp:126-128).
 *
 * Each entry point names the reference interface it replaces (file:line under proj/core).
 */
#ifndef SEMLAB_B200_H
#define SEMLAB_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status ------------------------------------------------------------------------------ */
#define SEMLAB_OK 0
#define SEMLAB_EINVAL 1   /* std::invalid_argument in the reference                        */
#define SEMLAB_ENUMERIC 2 /* std::runtime_error in the reference (bad Jacobian, eigensolve) */
#define SEMLAB_ECUDA 3    /* CUDA runtime error (no reference analogue)                    */
#define SEMLAB_ENCCL 4    /* NCCL error (no reference analogue)                            */

/* Message of the last failed call on this thread ("" if none). */
const char* semlab_last_error(void);
/* Library version string. */
const char* semlab_version(void);
/* Test/debug knob (no reference analogue): cap the grid of the persistent grid-stride kernels
   (fused Ax, warp-per-element RAS) at max_ctas CTAs so every warp runs many elements even on a
   small mesh; results must not change. 0 restores the occupancy-sized grid. Process-wide. */
int semlab_debug_set_grid_cap(int max_ctas);
/* GMRES form (process-wide): 1 (default) keeps the preconditioned directions Z and updates
   x += Z y when device memory allows (flexible GMRES: equal to the reference's x += M (V y) for a
   linear M, one M fewer per cycle, and robust to the FP32 smoother); 0 always uses the
   reference's x += M (V y) (krylov.cpp:108-114), as the solver does when Z does not fit. */
int semlab_debug_set_gmres_form(int flexible);

/* ---- opaque handles ---------------------------------------------------------------------- */
typedef struct semlab_ctx_s* semlab_ctx;         /* device + stream (+ NCCL communicator)  */
typedef struct semlab_mesh_s* semlab_mesh;       /* HexMesh, mesh.hpp:44-100               */
typedef struct semlab_space_s* semlab_space;     /* SemSpace, sem_space.hpp:26-129         */
typedef struct semlab_schwarz_s* semlab_schwarz; /* SchwarzSmoother, schwarz.hpp:31-86     */
typedef struct semlab_op_s* semlab_op;           /* LinOp, types.hpp:13                    */
typedef struct semlab_cheby_s* semlab_cheby;     /* ChebyshevSmoother, chebyshev.hpp:36-46 */
typedef struct semlab_proj_s* semlab_proj;       /* ProjectionBasis, krylov.hpp:39-59      */
typedef struct semlab_pmg_s* semlab_pmg;         /* pMG hierarchy (pmg.cpp is MISSING in the
                                                    reference; API of SPEC.md:313-349)     */
typedef struct semlab_semfem_s* semlab_semfem;   /* SemfemPreconditioner, semfem.hpp:36-54 */

/* ---- enums (values mirror the reference enums) -------------------------------------------- */
#define SEMLAB_BC_DIRICHLET 0 /* BcMode::Dirichlet, sem_space.hpp:12 */
#define SEMLAB_BC_NEUMANN 1   /* BcMode::Neumann                      */
#define SEMLAB_SCHWARZ_ASM 0  /* SchwarzMode::Asm, schwarz.hpp:10     */
#define SEMLAB_SCHWARZ_RAS 1  /* SchwarzMode::Ras                     */
#define SEMLAB_SMOOTHER_JACOBI 0
#define SEMLAB_SMOOTHER_RAS 1
#define SEMLAB_SMOOTHER_ASM 2
#define SEMLAB_SMOOTHER_RAS_PLAIN 3 /* un-accelerated RAS: x = S b pre, x += S (b - A x) post  */
#define SEMLAB_SMOOTHER_ASM_PLAIN 4 /* un-accelerated ASM (MgLevel smoother kinds) */
#define SEMLAB_CYCLE_STANDARD 0 /* Alg. 1: pre-smooth, coarse correction, post-smooth          */
#define SEMLAB_CYCLE_ADDITIVE 1 /* additive V-cycle, no post-smoothing (PAPER §2.2.2) */
#define SEMLAB_COARSE_DIRECT 0 /* exact solve of the p=1 system (SPEC.md:341-344 default) */
#define SEMLAB_COARSE_AMG 1    /* one AmgHierarchy V-cycle (amg.hpp:34-37)   */

/* ---- plain-data structs (field-for-field the reference structs) -------------------------- */
typedef struct { /* ChebyParams, chebyshev.hpp:9-14 */
  int order;
  double lambda_min_mult;
  double lambda_max_mult;
  double lambda_max_est;
} semlab_cheby_params;

typedef struct { /* LambdaEstimate, chebyshev.hpp:16-20 */
  double value;
  int breakdown;
  int rounds_used;
} semlab_lambda_estimate;

typedef struct { /* GmresConfig, krylov.hpp:9-15 */
  int restart;
  double tol;
  int max_iters;
  int use_abs_tol;
  double abs_tol;
} semlab_gmres_config;

typedef struct { /* GmresStats, krylov.hpp:17-25 (history copied into a caller buffer) */
  int iterations;
  int converged;
  int breakdown;
  double initial_residual;
  double abs_residual;
  double rel_residual;
  double* history;      /* caller-owned, may be NULL */
  int history_capacity; /* entries available in history */
  int history_len;      /* entries written (<= capacity) */
} semlab_gmres_stats;

/* ---- context ------------------------------------------------------------------------------ */
/* One GPU per process: all contexts alive in a process must use the same device (a second
   device is refused with SEMLAB_EINVAL). All work is ordered on cuda_stream (a cudaStream_t;
   NULL = the device's default stream, as in the CUDA runtime). */
int semlab_ctx_create(int device, void* cuda_stream, semlab_ctx* out);
/* Multi-GPU: rank/nranks over NCCL; nccl_id is the 128-byte ncclUniqueId from rank 0. */
int semlab_ctx_create_dist(int device, void* cuda_stream, int rank, int nranks,
                           const void* nccl_id, semlab_ctx* out);
int semlab_nccl_get_unique_id(void* out128);
/* z-slab neighbour exchanges (interface sums, Schwarz halos, owner copy-ups): 0 (default) NCCL
   send/recv; 1 NVLink peer memory (CUDA IPC mail slots + flag/ack protocol) when every rank can
   map its neighbours, else NCCL. Set on every rank, in the same order, before the exchanges. */
int semlab_ctx_set_exchange(semlab_ctx ctx, int mode);
int semlab_ctx_destroy(semlab_ctx ctx);
int semlab_ctx_synchronize(semlab_ctx ctx);
/* Number of kernels this library launched on ctx since creation (bench gpu_launches). */
int64_t semlab_ctx_launch_count(semlab_ctx ctx);

/* ---- mesh (mesh.hpp:44-108) ------------------------------------------------------------- */
/* generate_kershaw(KershawParams{eps, elements_per_axis}, p), mesh.cpp:138-171 */
int semlab_mesh_kershaw(semlab_ctx ctx, double eps, int elements_per_axis, semlab_mesh* out);
/* HexMesh::box(dims, lo, hi), mesh.cpp:82-89 */
int semlab_mesh_box(semlab_ctx ctx, const int dims[3], const double lo[3], const double hi[3],
                    semlab_mesh* out);
/* HexMesh::from_map(dims, map), mesh.cpp:91-93: the std::function map becomes a C callback
   unit-cube (x,y,z) -> physical out[3]. */
typedef void (*semlab_map_fn)(void* user, double x, double y, double z, double out[3]);
int semlab_mesh_from_map(semlab_ctx ctx, const int dims[3], semlab_map_fn fn, void* user,
                         semlab_mesh* out);
int semlab_mesh_destroy(semlab_mesh mesh);
/* HexMesh::lattice_coords(order), mesh.cpp:104-136, into a HOST buffer of 3*n doubles. */
int semlab_mesh_lattice_coords(semlab_mesh mesh, int order, double* host_out, int64_t capacity);

/* ---- space (sem_space.hpp:26-129) ---------------------------------------------------------- */
/* SemSpace(mesh, order, bc), sem_space.cpp:10-102. Geometry is built on the device. Under a
   distributed context the space owns this rank's z-slab of elements. */
int semlab_space_create(semlab_mesh mesh, int order, int bc, semlab_space* out);
int semlab_space_destroy(semlab_space s);
/* sizes: [0]=n (local vector length), [1]=n_free (global), [2]=n_local_total (E-vector length),
   [3..5]=lattice nx,ny,nz (global), [6]=n (global), [7]=elements on this rank,
   [8]=z of local plane 0, [9]=first element layer, [10]=last element layer + 1 */
int semlab_space_sizes(semlab_space s, int64_t out[11]);
/* apply_A, sem_space.cpp:195-209: out = mask o Q^T A_L Q o mask (in). */
int semlab_space_apply_A(semlab_space s, const double* d_in, double* d_out);
/* Extension (no reference analogue): apply_A with the geometric factors rounded to FP32 and FP64
   arithmetic, the operator of the FP32 smoother (orders 7 and <= 5; EINVAL otherwise). */
int semlab_space_apply_A_geom32(semlab_space s, const double* d_in, double* d_out);
/* apply_local_stiffness on every element (E-vector in/out), sem_space.cpp:127-180. */
int semlab_space_apply_local_stiffness(semlab_space s, const double* d_local_in, double* d_local_out);
/* gather (Q^T) / scatter (Q) / gather_scatter (QQ^T), sem_space.cpp:110-125, hpp:86-88. */
int semlab_space_gather(semlab_space s, const double* d_local, double* d_global);
int semlab_space_scatter(semlab_space s, const double* d_global, double* d_local);
int semlab_space_gather_scatter(semlab_space s, const double* d_local_in, double* d_local_out);
/* mask_inplace, sem_space.cpp:104-108. */
int semlab_space_mask(semlab_space s, double* d_v);
/* stiffness_diag (sem_space.cpp:211-236) and mass_diag (hpp:74) into a device vector. */
int semlab_space_stiffness_diag(semlab_space s, double* d_out);
int semlab_space_mass_diag(semlab_space s, double* d_out);
/* Geometric factors of element e (6 per node, packed rr,rs,rt,ss,st,tt like metric_at,
   sem_space.hpp:93-98) into a HOST buffer of 6*(order+1)^3 doubles. */
int semlab_space_metric(semlab_space s, int e, double* host_out);
/* RESTATED build_rhs (bench.cpp missing) into a device vector. */
int semlab_space_build_rhs(semlab_space s, uint64_t seed, double* d_out);

/* ---- vector utilities on a space's layout (owned-plane aware under a slab partition) ----- */
int semlab_space_dot(semlab_space s, const double* d_a, const double* d_b, double* host_out);

/* ---- operators (LinOp, types.hpp:13) ------------------------------------------------------ */
int semlab_op_A(semlab_space s, semlab_op* out);          /* SemSpace::apply_A                */
int semlab_op_A_geom32(semlab_space s, semlab_op* out); /* extension: apply_A_geom32 as a LinOp
                                                              (the FP32 smoother's operator)  */
int semlab_op_jacobi(semlab_space s, semlab_op* out);     /* S = diag(A)^-1     */
int semlab_op_schwarz(semlab_schwarz sch, semlab_op* out); /* SchwarzSmoother::as_linop        */
int semlab_op_pmg(semlab_pmg pmg, semlab_op* out);        /* pMG V-cycle as a preconditioner  */
/* User operator on device vectors: fn(user, d_in, d_out) is called stream-ordered. */
typedef void (*semlab_apply_fn)(void* user, const double* d_in, double* d_out);
int semlab_op_callback(semlab_ctx ctx, int64_t n, semlab_apply_fn fn, void* user, semlab_op* out);
int semlab_op_apply(semlab_op op, const double* d_in, double* d_out);
int semlab_op_destroy(semlab_op op);

/* ---- Schwarz (schwarz.hpp:31-86) ------------------------------------------------------------ */
/* SchwarzSmoother(space, mode), schwarz.cpp:46-131; precision 32 (FP32 FDM, the paper's
   smoother) or 64 (FP64, bit-for-bit the reference's arithmetic type). */
int semlab_schwarz_create(semlab_space s, int mode, int precision, semlab_schwarz* out);
int semlab_schwarz_destroy(semlab_schwarz sch);
/* SchwarzSmoother::apply, schwarz.cpp:242-289. */
int semlab_schwarz_apply(semlab_schwarz sch, const double* d_r, double* d_z);
/* fdm_solve for every element on padded (order+3)^3 boxes, x fastest, schwarz.cpp:228-240. */
int semlab_schwarz_fdm_solve_all(semlab_schwarz sch, const double* d_boxes_in, double* d_boxes_out);
/* Box lengths / 1-D eigen data of element e (host): lengths[3]; n[3]; lambda[3*(order+3)]. */
int semlab_schwarz_element_info(semlab_schwarz sch, int e, double lengths[3], int n[3], double* lambda);

/* ---- Chebyshev (chebyshev.hpp:9-46) -------------------------------------------------------- */
/* estimate_lambda_max(S, A, n, rounds, seed), chebyshev.cpp:9-56. */
int semlab_estimate_lambda_max(semlab_op S, semlab_op A, int64_t n, int rounds, uint64_t seed,
                               semlab_lambda_estimate* out);
/* ChebyshevSmoother(S, A, params), chebyshev.cpp:58-74. */
int semlab_cheby_create(semlab_op S, semlab_op A, const semlab_cheby_params* params, semlab_cheby* out);
int semlab_cheby_destroy(semlab_cheby c);
/* ChebyshevSmoother::smooth(b, x), chebyshev.cpp:76-96 (x updated in place). */
int semlab_cheby_smooth(semlab_cheby c, const double* d_b, double* d_x);

/* ---- p-multigrid (RESTATED: pmg.cpp missing, Alg. 1) ------------ */
typedef struct { /* hierarchy options */
  int smoother;           /* SEMLAB_SMOOTHER_* */
  int cheb_order;         /* Chebyshev order eta (Chebyshev smoothers) */
  double lambda_min_mult; /* Chebyshev bounds (0.1, 1.1) lambda~ */
  double lambda_max_mult;
  int precision;          /* Schwarz FDM precision: 32 (paper) or 64 */
  int coarse;             /* SEMLAB_COARSE_* */
  int bc;                 /* SEMLAB_BC_*: Neumann builds every level in Neumann mode and solves the
                             singular coarse problem on the zero-mean subspace (direct coarse only) */
  int cycle;              /* SEMLAB_CYCLE_* */
} semlab_pmg_options;
int semlab_pmg_create_ex(semlab_mesh mesh, int nlevels, const int* orders, const semlab_pmg_options* opts,
                         semlab_pmg* out);
/* orders: strictly decreasing schedule ending at 1, e.g. {7,3,1}. smoother: SEMLAB_SMOOTHER_*;
   precision applies to Schwarz smoothers (32 or 64). coarse: SEMLAB_COARSE_*. */
int semlab_pmg_create(semlab_mesh mesh, int nlevels, const int* orders, int smoother,
                      int cheb_order, double lmin_mult, double lmax_mult, int precision,
                      int coarse, semlab_pmg* out);
int semlab_pmg_destroy(semlab_pmg p);
/* z = V-cycle(b) with x0 = 0. */
int semlab_pmg_vcycle(semlab_pmg p, const double* d_b, double* d_z);
/* fine-level space handle (owned by the hierarchy) */
int semlab_pmg_space(semlab_pmg p, int level, semlab_space* out);
/* Coarse AMG hierarchy (SEMLAB_COARSE_AMG): number of levels and the row count of each (up to
   cap), like AmgHierarchy::n_levels / level_size (amg.hpp:39-40); 0 levels for the direct solve. */
int semlab_pmg_coarse_info(semlab_pmg p, int* nlevels, int64_t* sizes, int cap);
/* lambda estimate used at a level */
int semlab_pmg_lambda(semlab_pmg p, int level, double* out);
/* P (coarse level+1 -> level) and P^T, device vectors of the two levels' spaces. */
int semlab_pmg_prolong(semlab_pmg p, int level, const double* d_coarse, double* d_fine);
int semlab_pmg_restrict(semlab_pmg p, int level, const double* d_fine, double* d_coarse);

/* ---- SEMFEM preconditioner (semfem.hpp:14-54) ----------------------------------------------- */
/* SemfemPreconditioner(space, SemfemInner::Amg), semfem.cpp:112-124: the linear-tetrahedral
   lattice matrix (assemble_semfem, semfem.cpp:12-98, bitwise the reference's) and its AMG
   hierarchy (amg.cpp:69-129; host setup, device cycle). Single-rank (whole-mesh) spaces. */
int semlab_semfem_create(semlab_space s, semlab_semfem* out);
int semlab_semfem_destroy(semlab_semfem p);
/* apply, semfem.cpp:127-134: z = mask(one AMG V-cycle of r). */
int semlab_semfem_apply(semlab_semfem p, const double* d_r, double* d_z);
/* AMG level sizes (AmgHierarchy::n_levels / level_size) */
int semlab_semfem_levels(semlab_semfem p, int* nlevels, int64_t* sizes, int cap);
int semlab_op_semfem(semlab_semfem p, semlab_op* out); /* SemfemPreconditioner::as_linop */

/* ---- Krylov (krylov.hpp:9-33) -------------------------------------------------------------- */
/* gmres_solve(A, M, b, x, config), krylov.cpp:20-129. M may be NULL (identity). */
int semlab_gmres_solve(semlab_op A, semlab_op M, const double* d_b, double* d_x,
                       const semlab_gmres_config* config, semlab_gmres_stats* stats);
/* RESTATED PCG (not in the reference): same config/stats types, restart
   ignored; converges on ||r|| <= tol ||b - A x0||. */
int semlab_pcg_solve(semlab_op A, semlab_op M, const double* d_b, double* d_x,
                     const semlab_gmres_config* config, semlab_gmres_stats* stats);

/* ---- ProjectionBasis (krylov.hpp:35-59, krylov.cpp:131-152) ------------------------------
   A-orthonormal basis of prior solutions kept on the device (vectors of length n of the
   operator's space). capacity in [1, 24]. */
int semlab_proj_create(semlab_ctx ctx, int64_t n, int capacity, semlab_proj* out);
int semlab_proj_destroy(semlab_proj p);
/* u = sum_i (x_i . b) x_i, zero for an empty basis (ProjectionBasis::initial_guess). */
int semlab_proj_initial_guess(semlab_proj p, const double* d_b, double* d_u);
/* A-orthonormalise x into the basis, two classical passes, skip if dependent, evict the oldest
   beyond capacity (ProjectionBasis::insert). A must act on vectors of length n. */
int semlab_proj_insert(semlab_proj p, const double* d_x, semlab_op A);
int semlab_proj_size(semlab_proj p, int* out);
int semlab_proj_clear(semlab_proj p);
/* basis vector i (0 = oldest) copied to d_out */
int semlab_proj_vector(semlab_proj p, int i, double* d_out);

/* ---- host-only helpers (no GPU needed; used by the CPU test suite) ------------------------ */
/* gll(order), gll.cpp:80-91: nodes, weights (order+1) and diff (column-major (order+1)^2). */
int semlab_host_gll(int order, double* nodes, double* weights, double* diff);
/* kershaw_map(eps, x, y, z), mesh.cpp:52-55 */
int semlab_host_kershaw_map(double eps, double x, double y, double z, double out[3]);
/* std::uniform_real_distribution<double>(-1,1) over std::mt19937_64(seed), n draws
   (the lambda-estimate start vector, chebyshev.cpp:12-15). */
int semlab_host_uniform_pm1(uint64_t seed, int64_t n, double* out);
/* Generalised symmetric-definite eigenproblem A s = lambda B s (n <= 16): lambda ascending,
   S column-major with S^T B S = I (GeneralizedSelfAdjointEigenSolver, schwarz.cpp:207). */
int semlab_host_gen_eig(int n, const double* A, const double* B, double* lambda, double* S);
/* Eigenvalue moduli max of a small real matrix (EigenSolver, chebyshev.cpp:53-54). */
int semlab_host_max_abs_eig(int n, const double* H_colmajor, double* out);

#ifdef __cplusplus
}
#endif
#endif /* SEMLAB_B200_H */
