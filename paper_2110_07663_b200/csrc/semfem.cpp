// SEMFEM preconditioner (the paper's low-order competitor, §2.2.1; reference
// semfem.cpp:12-134): the linear-tetrahedral stiffness matrix on the GLL lattice of a space,
// every hexahedral GLL sub-cell covered by its eight corner tetrahedra with an overall 1/2,
// Dirichlet dofs eliminated symmetrically (unit diagonal), exact zeros pruned; one AMG V-cycle
// (amg.cpp, setup on the host, cycle on the device) as the inner solve; z = mask(AMG(r)).
//
// The matrix is assembled on the host in the reference's arithmetic order (triplets in element,
// sub-cell, tetrahedron, (a, b) order; 3x3 determinant and cofactor inverse as the reference
// builds them; duplicates summed in insertion order), so it is bitwise the reference's matrix
// and the aggregation, which breaks ties on exact comparisons, builds the reference's hierarchy.
#include <algorithm>
#include <array>

#include "capi_util.hpp"
#include "pmg.hpp"

using namespace sb;

struct semlab_semfem_s {
  semlab_space sp = nullptr;
  sb::CoarseSolver amg;
  void apply(const double* r, double* z);
};

namespace {

HostCsr assemble_semfem(semlab_space sp) {
  if (sp->distributed()) invalid("SemfemPreconditioner: needs a whole-mesh space (single rank)");
  const Slab& sl = sp->sl;
  const int p = sp->order;
  const int64_t n = sp->n;
  const std::vector<double>& X = sp->coords;  // 3 per lattice point, x fastest
  struct V3 {
    double x, y, z;
  };
  auto point = [&](int64_t g) { return V3{X[size_t(3 * g)], X[size_t(3 * g + 1)], X[size_t(3 * g + 2)]}; };
  // corner tetrahedra of a sub-cell: the corner and its three edge-adjacent vertices, reordered
  // for a positive reference volume (semfem.cpp:25-41)
  std::array<std::array<int, 4>, 8> tets;
  {
    int t = 0;
    for (int cz = 0; cz <= 1; ++cz)
      for (int cy = 0; cy <= 1; ++cy)
        for (int cx = 0; cx <= 1; ++cx) {
          auto corner = [](int x, int y, int z) { return x + 2 * y + 4 * z; };
          std::array<int, 4> tet = {corner(cx, cy, cz), corner(1 - cx, cy, cz), corner(cx, 1 - cy, cz),
                                    corner(cx, cy, 1 - cz)};
          if ((cx + cy + cz) % 2) std::swap(tet[1], tet[2]);
          tets[size_t(t++)] = tet;
        }
  }
  auto masked = [&](int64_t g) {
    const int64_t x = g % sl.Nx, y = (g / sl.Nx) % sl.Ny, z = g / (sl.Nx * sl.Ny);
    return sl.masked(x, y, z);
  };
  std::vector<std::vector<std::pair<int64_t, double>>> rows(static_cast<size_t>(n));
  const int64_t E = sp->E;
  for (int64_t e = 0; e < E; ++e) {
    const int ex = int(e % sl.Ex), ey = int((e / sl.Ex) % sl.Ey), ez = int(e / (int64_t(sl.Ex) * sl.Ey));
    for (int k = 0; k < p; ++k)
      for (int j = 0; j < p; ++j)
        for (int i = 0; i < p; ++i) {
          std::array<int64_t, 8> cell;
          int c = 0;
          for (int cz = 0; cz <= 1; ++cz)
            for (int cy = 0; cy <= 1; ++cy)
              for (int cx = 0; cx <= 1; ++cx)
                cell[size_t(c++)] = sl.lidx(int64_t(ex) * p + i + cx, int64_t(ey) * p + j + cy, int64_t(ez) * p + k + cz);
          for (const auto& tet : tets) {
            const V3 p0 = point(cell[size_t(tet[0])]);
            double T[3][3];  // columns: vertex 1..3 minus vertex 0
            for (int col = 0; col < 3; ++col) {
              const V3 q = point(cell[size_t(tet[size_t(col + 1)])]);
              T[0][col] = q.x - p0.x;
              T[1][col] = q.y - p0.y;
              T[2][col] = q.z - p0.z;
            }
            const double det = T[0][0] * (T[1][1] * T[2][2] - T[2][1] * T[1][2]) -
                               T[1][0] * (T[0][1] * T[2][2] - T[2][1] * T[0][2]) +
                               T[2][0] * (T[0][1] * T[1][2] - T[1][1] * T[0][2]);
            if (det <= 0.0)
              numeric("assemble_semfem: inverted tetrahedron in element " + std::to_string(e) + ", sub-cell (" +
                      std::to_string(i) + "," + std::to_string(j) + "," + std::to_string(k) + ")");
            const double vol = det / 6.0;
            const double c00 = T[1][1] * T[2][2] - T[1][2] * T[2][1], c10 = T[1][2] * T[2][0] - T[1][0] * T[2][2],
                         c20 = T[1][0] * T[2][1] - T[1][1] * T[2][0];
            const double id = 1.0 / (T[0][0] * c00 + T[0][1] * c10 + T[0][2] * c20);
            double Ti[3][3];
            Ti[0][0] = c00 * id;
            Ti[1][0] = c10 * id;
            Ti[2][0] = c20 * id;
            Ti[0][1] = (T[0][2] * T[2][1] - T[0][1] * T[2][2]) * id;
            Ti[1][1] = (T[0][0] * T[2][2] - T[0][2] * T[2][0]) * id;
            Ti[2][1] = (T[0][1] * T[2][0] - T[0][0] * T[2][1]) * id;
            Ti[0][2] = (T[0][1] * T[1][2] - T[0][2] * T[1][1]) * id;
            Ti[1][2] = (T[0][2] * T[1][0] - T[0][0] * T[1][2]) * id;
            Ti[2][2] = (T[0][0] * T[1][1] - T[0][1] * T[1][0]) * id;
            double grad[4][3];  // barycentric gradients: rows of T^-1, grad0 = -(g1 + g2 + g3)
            for (int r = 0; r < 3; ++r)
              for (int d = 0; d < 3; ++d) grad[r + 1][d] = Ti[r][d];
            for (int d = 0; d < 3; ++d) grad[0][d] = -((grad[1][d] + grad[2][d]) + grad[3][d]);
            for (int a = 0; a < 4; ++a)
              for (int b = 0; b < 4; ++b) {
                const int64_t ga = cell[size_t(tet[size_t(a)])], gb = cell[size_t(tet[size_t(b)])];
                if (masked(ga) || masked(gb)) continue;
                double dot = 0.0;
                for (int d = 0; d < 3; ++d) dot += grad[a][d] * grad[b][d];
                rows[size_t(ga)].push_back({gb, 0.5 * vol * dot});
              }
          }
        }
  }
  for (int64_t g = 0; g < n; ++g)
    if (masked(g)) rows[size_t(g)].push_back({g, 1.0});
  HostCsr A;  // setFromTriplets (duplicates summed in insertion order), then prune(0, 0)
  A.n = A.m = n;
  A.ptr.assign(size_t(n) + 1, 0);
  for (int64_t i = 0; i < n; ++i) {
    auto& row = rows[size_t(i)];
    std::stable_sort(row.begin(), row.end(), [](auto& u, auto& v) { return u.first < v.first; });
    std::vector<std::pair<int64_t, double>> merged;
    for (auto& kv : row) {
      if (!merged.empty() && merged.back().first == kv.first)
        merged.back().second += kv.second;
      else
        merged.push_back(kv);
    }
    for (auto& kv : merged)
      if (kv.second != 0.0) {
        A.idx.push_back(int(kv.first));
        A.val.push_back(kv.second);
      }
    A.ptr[size_t(i) + 1] = int64_t(A.idx.size());
    std::vector<std::pair<int64_t, double>>().swap(row);
  }
  return A;
}

}  // namespace

void semlab_semfem_s::apply(const double* r, double* z) {
  amg.amg_cycle(0, r, z);  // AmgHierarchy::vcycle (amg.cpp:140-165) over all lattice dofs
  sp->ctx->count(launch_mask(sp->sl, z, sp->ctx->stream));  // space_->mask_inplace(z)
}

extern "C" {

int semlab_semfem_create(semlab_space s, semlab_semfem* out) {
  return guard([&] {
    need(s, "SemfemPreconditioner: space");
    need(out, "SemfemPreconditioner: out");
    auto p = std::make_unique<semlab_semfem_s>();
    p->sp = s;
    if (s->n >= (int64_t(1) << 31)) invalid("SemfemPreconditioner: needs < 2^31 dofs");
    const HostCsr A = assemble_semfem(s);
    p->amg.build_amg(s, A);
    *out = p.release();
  });
}

int semlab_semfem_destroy(semlab_semfem p) {
  return guard([&] {
    if (p && p->sp) cudaStreamSynchronize(p->sp->ctx->stream);
    delete p;
  });
}

int semlab_semfem_apply(semlab_semfem p, const double* r, double* z) {
  return guard([&] {
    need(p, "SemfemPreconditioner: handle");
    p->apply(r, z);
  });
}

int semlab_semfem_levels(semlab_semfem p, int* nlevels, int64_t* sizes, int cap) {
  return guard([&] {
    need(p, "SemfemPreconditioner: handle");
    need(nlevels, "semfem_levels: nlevels");
    *nlevels = int(p->amg.lev.size());
    for (int l = 0; l < *nlevels && l < cap; ++l) sizes[l] = p->amg.lev[size_t(l)].n;
  });
}

int semlab_op_semfem(semlab_semfem p, semlab_op* out) {
  return guard([&] {
    need(p, "semlab_op_semfem: handle");
    auto o = std::make_unique<semlab_op_s>();
    o->kind = semlab_op_s::kSemfem;
    o->ctx = p->sp->ctx;
    o->n = p->sp->n;
    o->space = p->sp;
    o->semfem = p;
    *out = o.release();
  });
}

}  // extern "C"

void semfem_apply(semlab_semfem p, const double* r, double* z) { p->apply(r, z); }
