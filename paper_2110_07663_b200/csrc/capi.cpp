// extern "C" boundary: every entry point of include/semlab_b200.h outside Schwarz and pMG.
// No exception crosses it: sb::Error / std::exception become status codes + semlab_last_error().
#include <nccl.h>

#include <atomic>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <new>

#include "capi_util.hpp"
#include "host_math.hpp"
#include "solvers.hpp"

using namespace sb;

namespace {
thread_local std::string g_err;
}

void sb_set_error(const std::string& msg) { g_err = msg; }

namespace {
std::atomic<int> g_grid_cap{0};
std::mutex g_dev_mu;
int g_ctx_device = -1;  // the one device this process's contexts use
int g_ctx_live = 0;
}  // namespace

namespace {
std::atomic<int> g_gmres_flexible{1};
}
namespace sb {
int grid_cap() { return g_grid_cap.load(std::memory_order_relaxed); }
bool gmres_flexible_allowed() { return g_gmres_flexible.load(std::memory_order_relaxed) != 0; }

int per_device_once(const void* key, const std::function<int()>& init) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> cache;
  int dev = 0;
  SB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({dev, key});
  if (it != cache.end()) return it->second;
  const int v = init();
  cache[{dev, key}] = v;
  return v;
}
}  // namespace sb

int sb_guard_impl(const std::function<void()>& f) {
  try {
    f();
    return SEMLAB_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return SEMLAB_ENUMERIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SEMLAB_ENUMERIC;
  }
}

extern "C" {

const char* semlab_last_error(void) { return g_err.c_str(); }
const char* semlab_version(void) { return "semlab_b200 0.2 (sm_100a)"; }

int semlab_debug_set_gmres_form(int flexible) {
  return guard([&] { g_gmres_flexible.store(flexible ? 1 : 0); });
}

int semlab_debug_set_grid_cap(int max_ctas) {
  return guard([&] {
    if (max_ctas < 0) invalid("semlab_debug_set_grid_cap: max_ctas must be >= 0");
    g_grid_cap.store(max_ctas);
  });
}

// ---------------------------------------------------------------- context
static void register_ctx(int device) {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  g_ctx_device = device;
  ++g_ctx_live;
}

static void ctx_init(semlab_ctx c, int device, void* stream) {
  int ndev = 0;
  SB_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) invalid("semlab_ctx_create: no CUDA device " + std::to_string(device));
  {
    // One GPU per process (one rank per GPU): entry points run on the calling thread's current
    // device, which the context sets here. A second device in the same process is refused.
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (g_ctx_live > 0 && g_ctx_device != device)
      invalid("semlab_ctx_create: contexts of one process must share a device (live contexts use device " +
              std::to_string(g_ctx_device) + ")");
  }
  SB_CUDA(cudaSetDevice(device));
  c->device = device;
  c->stream = static_cast<cudaStream_t>(stream);  // NULL = default stream (shared with the caller)
  c->dot_partial.alloc(size_t(kMaxDotBlocks) * 32);
  c->dot_counter.alloc(1);
  c->dot_counter.zero(c->stream);
  c->dot_out.alloc(64);
  SB_CUDA(cudaMallocHost(&c->host_pinned, 128 * sizeof(double)));
  c->sync();
}

int semlab_ctx_create(int device, void* stream, semlab_ctx* out) {
  return guard([&] {
    need(out, "semlab_ctx_create: out");
    auto c = std::make_unique<semlab_ctx_s>();
    ctx_init(c.get(), device, stream);
    register_ctx(device);
    *out = c.release();
  });
}

int semlab_nccl_get_unique_id(void* out128) {
  return guard([&] {
    need(out128, "semlab_nccl_get_unique_id: out");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) fail(kNccl, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    std::memcpy(out128, &id, sizeof(id));
  });
}

int semlab_ctx_create_dist(int device, void* stream, int rank, int nranks, const void* nccl_id, semlab_ctx* out) {
  return guard([&] {
    need(out, "semlab_ctx_create_dist: out");
    if (nranks < 1 || rank < 0 || rank >= nranks) invalid("semlab_ctx_create_dist: bad rank/nranks");
    auto c = std::make_unique<semlab_ctx_s>();
    ctx_init(c.get(), device, stream);
    c->rank = rank;
    c->nranks = nranks;
    if (nranks > 1) {
      need(nccl_id, "semlab_ctx_create_dist: nccl_id");
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof(id));
      ncclComm_t comm;
      ncclResult_t r = ncclCommInitRank(&comm, nranks, id, rank);
      if (r != ncclSuccess) fail(kNccl, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
      c->nccl = comm;
    }
    register_ctx(device);
    *out = c.release();
  });
}

int semlab_ctx_set_exchange(semlab_ctx c, int mode) {
  return guard([&] {
    need(c, "semlab_ctx_set_exchange: ctx");
    if (mode != 0 && mode != 1) invalid("semlab_ctx_set_exchange: mode must be 0 (NCCL) or 1 (peer)");
    c->exchange_mode = mode;
  });
}

int semlab_ctx_destroy(semlab_ctx c) {
  return guard([&] {
    if (!c) return;
    cudaStreamSynchronize(c->stream);
    c->peer.release();
    if (c->nccl) ncclCommDestroy(static_cast<ncclComm_t>(c->nccl));
    if (c->host_pinned) cudaFreeHost(c->host_pinned);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (g_ctx_live > 0) --g_ctx_live;
  });
}

int semlab_ctx_synchronize(semlab_ctx c) {
  return guard([&] {
    need(c, "semlab_ctx_synchronize: ctx");
    c->sync();
    if (c->peer_state == 1) c->peer.check(c);
  });
}

int64_t semlab_ctx_launch_count(semlab_ctx c) { return c ? c->launches : -1; }

// ---------------------------------------------------------------- mesh
int semlab_mesh_kershaw(semlab_ctx ctx, double eps, int epa, semlab_mesh* out) {
  return guard([&] {
    need(ctx, "semlab_mesh_kershaw: ctx");
    need(out, "semlab_mesh_kershaw: out");
    if (!(eps > 0.0) || eps > 1.0) invalid("generate_kershaw: eps must lie in (0,1]");
    if (epa < 2 || epa % 2 != 0) invalid("generate_kershaw: elements_per_axis must be even and >= 2");
    auto m = std::make_unique<semlab_mesh_s>();
    m->ctx = ctx;
    m->dims = {epa, epa, epa};
    m->kershaw_eps = eps;
    m->map = [eps](double x, double y, double z) { return kershaw_map(eps, x, y, z); };
    *out = m.release();
  });
}

int semlab_mesh_box(semlab_ctx ctx, const int dims[3], const double lo[3], const double hi[3], semlab_mesh* out) {
  return guard([&] {
    need(ctx, "semlab_mesh_box: ctx");
    need(out, "semlab_mesh_box: out");
    if (dims[0] < 1 || dims[1] < 1 || dims[2] < 1) invalid("HexMesh: element counts must be positive");
    auto m = std::make_unique<semlab_mesh_s>();
    m->ctx = ctx;
    m->dims = {dims[0], dims[1], dims[2]};
    const std::array<double, 3> l{lo[0], lo[1], lo[2]}, h{hi[0], hi[1], hi[2]};
    m->kershaw_eps = -1.0;  // pure C++ map (parallel evaluation allowed)
    m->map = [l, h](double x, double y, double z) {
      return std::array<double, 3>{l[0] + (h[0] - l[0]) * x, l[1] + (h[1] - l[1]) * y, l[2] + (h[2] - l[2]) * z};
    };
    *out = m.release();
  });
}

int semlab_mesh_from_map(semlab_ctx ctx, const int dims[3], semlab_map_fn fn, void* user, semlab_mesh* out) {
  return guard([&] {
    need(ctx, "semlab_mesh_from_map: ctx");
    need(out, "semlab_mesh_from_map: out");
    need(reinterpret_cast<void*>(fn), "semlab_mesh_from_map: fn");
    if (dims[0] < 1 || dims[1] < 1 || dims[2] < 1) invalid("HexMesh: element counts must be positive");
    auto m = std::make_unique<semlab_mesh_s>();
    m->ctx = ctx;
    m->dims = {dims[0], dims[1], dims[2]};
    m->kershaw_eps = 0.0;  // user callback: evaluated serially
    m->map = [fn, user](double x, double y, double z) {
      std::array<double, 3> o{};
      fn(user, x, y, z, o.data());
      return o;
    };
    *out = m.release();
  });
}

int semlab_mesh_destroy(semlab_mesh m) {
  return guard([&] { delete m; });
}

int semlab_mesh_lattice_coords(semlab_mesh m, int order, double* host_out, int64_t capacity) {
  return guard([&] {
    need(m, "semlab_mesh_lattice_coords: mesh");
    const int64_t nz = int64_t(m->dims[2]) * order + 1;
    auto c = m->lattice_planes(order, 0, nz);
    if (capacity < int64_t(c.size())) invalid("semlab_mesh_lattice_coords: buffer too small");
    std::memcpy(host_out, c.data(), c.size() * sizeof(double));
  });
}

// ---------------------------------------------------------------- space
int semlab_space_create(semlab_mesh mesh, int order, int bc, semlab_space* out) {
  return guard([&] {
    need(mesh, "semlab_space_create: mesh");
    need(out, "semlab_space_create: out");
    if (bc != SEMLAB_BC_DIRICHLET && bc != SEMLAB_BC_NEUMANN) invalid("SemSpace: unknown BcMode");
    auto s = std::make_unique<semlab_space_s>();
    s->ctx = mesh->ctx;
    s->mesh = mesh;
    s->order = order;
    s->bc = bc;
    SB_CUDA(cudaSetDevice(s->ctx->device));
    s->build();
    *out = s.release();
  });
}

int semlab_space_destroy(semlab_space s) {
  return guard([&] {
    if (s) cudaStreamSynchronize(s->ctx->stream);
    delete s;
  });
}

int semlab_space_sizes(semlab_space s, int64_t out[11]) {
  return guard([&] {
    need(s, "semlab_space_sizes: space");
    const Slab& sl = s->sl;
    const int64_t ng = sl.Nx * sl.Ny * sl.Nz;
    const int64_t nfree = s->bc == SEMLAB_BC_DIRICHLET ? (sl.Nx - 2) * (sl.Ny - 2) * (sl.Nz - 2) : ng;
    out[0] = s->n;
    out[1] = nfree;
    out[2] = s->E * s->nloc;
    out[3] = sl.Nx;
    out[4] = sl.Ny;
    out[5] = sl.Nz;
    out[6] = ng;
    out[7] = s->E;
    out[8] = sl.zlo;
    out[9] = sl.ez0;
    out[10] = sl.ez1;
  });
}

int semlab_space_apply_A(semlab_space s, const double* in, double* out) {
  return guard([&] {
    need(s, "apply_A: space");
    s->apply_A(in, out);
  });
}

int semlab_space_apply_A_geom32(semlab_space s, const double* in, double* out) {
  return guard([&] {
    need(s, "apply_A_geom32: space");
    if (!s->enable_geom32()) invalid("apply_A_geom32: FP32 geometric factors exist for orders 7 and <= 5 only");
    s->apply_A(in, out, true);
  });
}

int semlab_space_apply_local_stiffness(semlab_space s, const double* in, double* out) {
  return guard([&] {
    need(s, "apply_local_stiffness: space");
    s->ctx->count(launch_ax_local(s->sl, in, s->geom.p, out, s->ctx->stream));
  });
}

int semlab_space_gather(semlab_space s, const double* loc, double* glob) {
  return guard([&] {
    need(s, "gather: space");
    s->ctx->count(launch_gather(s->sl, loc, glob, s->ctx->stream));
    s->interface_sum(glob);
  });
}

int semlab_space_scatter(semlab_space s, const double* glob, double* loc) {
  return guard([&] {
    need(s, "scatter: space");
    s->ctx->count(launch_scatter(s->sl, glob, loc, s->ctx->stream));
  });
}

int semlab_space_gather_scatter(semlab_space s, const double* in, double* out) {
  return guard([&] {
    need(s, "gather_scatter: space");
    if (s->ctx->nranks > 1) {  // Q^T, cross-rank interface sum, then Q
      DevBuf<double> g(static_cast<size_t>(s->n));
      s->ctx->count(launch_gather(s->sl, in, g.p, s->ctx->stream));
      s->interface_sum(g.p);
      s->ctx->count(launch_scatter(s->sl, g.p, out, s->ctx->stream));
      s->ctx->sync();
    } else {
      s->ctx->count(launch_qqt(s->sl, in, out, s->ctx->stream));
    }
  });
}

int semlab_space_mask(semlab_space s, double* v) {
  return guard([&] {
    need(s, "mask: space");
    s->ctx->count(launch_mask(s->sl, v, s->ctx->stream));
  });
}

int semlab_space_stiffness_diag(semlab_space s, double* out) {
  return guard([&] {
    need(s, "stiffness_diag: space");
    s->stiffness_diag(out);
  });
}

int semlab_space_mass_diag(semlab_space s, double* out) {
  return guard([&] {
    need(s, "mass_diag: space");
    s->ctx->count(launch_copy(out, s->mass_diag.p, s->n, s->ctx->stream));
  });
}

int semlab_space_metric(semlab_space s, int e, double* host_out) {
  return guard([&] {
    need(s, "metric: space");
    if (e < 0 || e >= s->E) invalid("metric: element out of range");
    std::vector<double> soa(static_cast<size_t>(6 * s->nloc));
    SB_CUDA(cudaMemcpyAsync(soa.data(), s->geom.p + size_t(e) * 6 * s->nloc, soa.size() * sizeof(double),
                            cudaMemcpyDeviceToHost, s->ctx->stream));
    s->ctx->sync();
    for (int64_t node = 0; node < s->nloc; ++node)
      for (int c = 0; c < 6; ++c) host_out[node * 6 + c] = soa[size_t(c * s->nloc + node)];
  });
}

int semlab_space_build_rhs(semlab_space s, uint64_t seed, double* out) {
  return guard([&] {
    need(s, "build_rhs: space");
    const Slab& sl = s->sl;
    const int64_t n = s->n;
    std::vector<double> f(static_cast<size_t>(n)), g(static_cast<size_t>(n));
    uniform_pm1_range(seed, sl.zlo * sl.Nx * sl.Ny, n, g.data());
    const double pi = M_PI;
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < n; ++t) {
      const double X = s->coords[size_t(3 * t)], Y = s->coords[size_t(3 * t + 1)], Z = s->coords[size_t(3 * t + 2)];
      const double smooth = 3.0 * pi * pi * std::sin(pi * (X + 0.5)) * std::sin(pi * (Y + 0.5)) * std::sin(pi * (Z + 0.5));
      const double bubble = 64.0 * (0.25 - X * X) * (0.25 - Y * Y) * (0.25 - Z * Z);
      f[size_t(t)] = smooth + g[size_t(t)] * bubble;
    }
    DevBuf<double> df(static_cast<size_t>(n));
    df.upload(f.data(), size_t(n), s->ctx->stream);
    s->ctx->count(launch_mul(out, s->mass_diag.p, df.p, n, s->ctx->stream));
    s->ctx->count(launch_mask(sl, out, s->ctx->stream));
    s->ctx->sync();
  });
}

int semlab_space_dot(semlab_space s, const double* a, const double* b, double* host_out) {
  return guard([&] {
    need(s, "dot: space");
    *host_out = s->dot(a, b);
  });
}

// ---------------------------------------------------------------- operators
int semlab_op_A(semlab_space s, semlab_op* out) {
  return guard([&] {
    need(s, "semlab_op_A: space");
    auto o = std::make_unique<semlab_op_s>();
    o->kind = semlab_op_s::kA;
    o->ctx = s->ctx;
    o->n = s->n;
    o->space = s;
    *out = o.release();
  });
}

int semlab_op_A_geom32(semlab_space s, semlab_op* out) {
  return guard([&] {
    need(s, "semlab_op_A_geom32: space");
    if (!s->enable_geom32()) invalid("semlab_op_A_geom32: FP32 geometric factors exist for orders 7 and <= 5 only");
    auto o = std::make_unique<semlab_op_s>();
    o->kind = semlab_op_s::kA;
    o->ctx = s->ctx;
    o->n = s->n;
    o->space = s;
    o->geom32 = true;
    *out = o.release();
  });
}

int semlab_op_jacobi(semlab_space s, semlab_op* out) {
  return guard([&] {
    need(s, "semlab_op_jacobi: space");
    auto o = std::make_unique<semlab_op_s>();
    o->kind = semlab_op_s::kJacobi;
    o->ctx = s->ctx;
    o->n = s->n;
    o->space = s;
    s->jacobi_inv();
    *out = o.release();
  });
}

int semlab_op_callback(semlab_ctx ctx, int64_t n, semlab_apply_fn fn, void* user, semlab_op* out) {
  return guard([&] {
    need(ctx, "semlab_op_callback: ctx");
    need(reinterpret_cast<void*>(fn), "semlab_op_callback: fn");
    auto o = std::make_unique<semlab_op_s>();
    o->kind = semlab_op_s::kCallback;
    o->ctx = ctx;
    o->n = n;
    o->fn = fn;
    o->user = user;
    *out = o.release();
  });
}

int semlab_op_apply(semlab_op op, const double* in, double* out) {
  return guard([&] {
    need(op, "semlab_op_apply: op");
    op->apply(in, out);
  });
}

int semlab_op_destroy(semlab_op op) {
  return guard([&] { delete op; });
}

// ---------------------------------------------------------------- Chebyshev / lambda
int semlab_estimate_lambda_max(semlab_op S, semlab_op A, int64_t n, int rounds, uint64_t seed,
                               semlab_lambda_estimate* out) {
  return guard([&] {
    need(out, "estimate_lambda_max: out");
    *out = estimate_lambda_max(S, A, n, rounds, seed);
  });
}

int semlab_cheby_create(semlab_op S, semlab_op A, const semlab_cheby_params* p, semlab_cheby* out) {
  return guard([&] {
    need(p, "ChebyshevSmoother: params");
    auto c = std::make_unique<semlab_cheby_s>();
    c->init(S, A, *p);
    *out = c.release();
  });
}

int semlab_cheby_destroy(semlab_cheby c) {
  return guard([&] { delete c; });
}

int semlab_cheby_smooth(semlab_cheby c, const double* b, double* x) {
  return guard([&] {
    need(c, "ChebyshevSmoother::smooth: smoother");
    c->smooth(b, x, false);
  });
}

// ---------------------------------------------------------------- Krylov
static void copy_stats(const KrylovResult& r, semlab_gmres_stats* st) {
  if (!st) return;
  st->iterations = r.iterations;
  st->converged = r.converged ? 1 : 0;
  st->breakdown = r.breakdown ? 1 : 0;
  st->initial_residual = r.initial_residual;
  st->abs_residual = r.abs_residual;
  st->rel_residual = r.rel_residual;
  st->history_len = 0;
  if (st->history && st->history_capacity > 0) {
    const int k = std::min<int>(st->history_capacity, int(r.history.size()));
    for (int i = 0; i < k; ++i) st->history[i] = r.history[size_t(i)];
    st->history_len = k;
  }
}

int semlab_gmres_solve(semlab_op A, semlab_op M, const double* b, double* x, const semlab_gmres_config* cfg,
                       semlab_gmres_stats* stats) {
  return guard([&] {
    need(cfg, "gmres: config");
    copy_stats(gmres_solve(A, M, b, x, *cfg), stats);
  });
}

int semlab_pcg_solve(semlab_op A, semlab_op M, const double* b, double* x, const semlab_gmres_config* cfg,
                     semlab_gmres_stats* stats) {
  return guard([&] {
    need(cfg, "pcg: config");
    copy_stats(pcg_solve(A, M, b, x, *cfg), stats);
  });
}

// ---------------------------------------------------------------- host-only helpers
int semlab_host_gll(int order, double* nodes, double* weights, double* diff) {
  return guard([&] {
    const Gll& g = gll(order);
    if (nodes) std::memcpy(nodes, g.nodes.data(), g.nodes.size() * sizeof(double));
    if (weights) std::memcpy(weights, g.weights.data(), g.weights.size() * sizeof(double));
    if (diff) std::memcpy(diff, g.diff.data(), g.diff.size() * sizeof(double));
  });
}

int semlab_host_kershaw_map(double eps, double x, double y, double z, double out[3]) {
  return guard([&] {
    const auto p = kershaw_map(eps, x, y, z);
    out[0] = p[0];
    out[1] = p[1];
    out[2] = p[2];
  });
}

int semlab_host_uniform_pm1(uint64_t seed, int64_t n, double* out) {
  return guard([&] { uniform_pm1(seed, n, out); });
}

int semlab_host_gen_eig(int n, const double* A, const double* B, double* lambda, double* S) {
  return guard([&] {
    if (n < 1 || n > 16) invalid("gen_eig: n must be in [1,16]");
    if (!gen_sym_eig(n, A, B, lambda, S)) numeric("gen_eig: B is not positive definite");
  });
}

int semlab_host_max_abs_eig(int n, const double* H, double* out) {
  return guard([&] {
    if (n < 1 || n > 64) invalid("max_abs_eig: n must be in [1,64]");
    *out = max_abs_eig(n, H);
  });
}

}  // extern "C"
