// Drop-in check: the reference's own C++ objects (FeSpace, BilinearForm,
// form_linear_system, cg_solve -- the unmodified library from
// /root/reference/proj/src, namespace-renamed to tfem_ref at build time) next
// to the same problem routed through tensorfem_b200.hpp -> libtfem_cuda.so.
// Prints one PASS/FAIL line per check (acceptance_main.cpp style); exit code
// = number of failures.  Built by integration/Makefile; run by
// tests/test_integration.py on the GPU box.
#include "tensorfem_b200.hpp"

#include "tensorfem/driver.hpp"
#include "tensorfem/ncmesh.hpp"

#include <cmath>
#include <cstdio>
#include <random>
#include <set>

using namespace tensorfem;

namespace {

int failures = 0;

void report(const char *what, bool ok, const std::string &detail = "")
{
   std::printf("[%s] %s %s\n", ok ? "PASS" : "FAIL", what, detail.c_str());
   if (!ok) failures++;
}

Vector random_vector(int n, unsigned seed)
{
   std::mt19937 gen(seed); // test_forms.cpp:17-26
   std::uniform_real_distribution<double> dist(-1.0, 1.0);
   Vector x(n);
   for (int i = 0; i < n; i++) x[i] = dist(gen);
   return x;
}

bool equal(const Vector &a, const Vector &b)
{
   if (a.size() != b.size()) return false;
   for (int i = 0; i < a.size(); i++)
      if (a[i] != b[i]) return false;
   return true;
}

double varying(Vec2 p) { return 1.0 + p.x + 2.0 * p.y; }

std::vector<int> all_attrs(const Mesh &m)
{
   std::set<int> s;
   for (const auto &b : m.boundary_segments()) s.insert(b.attribute);
   return {s.begin(), s.end()};
}

void check_space(const b200::Device &dev, const FeSpace &space, const char *name)
{
   const int p = space.collection().order();
   b200::DeviceSpace ds(dev, space);
   for (IntegratorKind kind : {IntegratorKind::Diffusion, IntegratorKind::Mass}) {
      BilinearForm ref(space, AssemblyMode::Partial);
      if (kind == IntegratorKind::Diffusion) ref.add_diffusion(varying);
      else ref.add_mass(varying);
      ref.assemble();
      b200::DevicePa pa(ds, kind, varying);
      b200::DeviceOperator op(ds, {&pa});
      const Vector x = random_vector(space.n_true_dofs(), 100 * p);
      Vector yr(space.n_true_dofs()), yd(space.n_true_dofs());
      ref.mult_true(x, yr);
      op.mult(x, yd);
      char what[160];
      std::snprintf(what, sizeof what, "%s p=%d %s: mult_true bit-identical", name, p,
                    kind == IntegratorKind::Mass ? "mass" : "diffusion");
      report(what, equal(yr, yd));
      std::snprintf(what, sizeof what, "%s p=%d %s: diagonal_true bit-identical", name, p,
                    kind == IntegratorKind::Mass ? "mass" : "diffusion");
      report(what, equal(ref.diagonal_true(), op.diagonal()));
      std::snprintf(what, sizeof what, "%s p=%d %s: stored_reals", name, p,
                    kind == IntegratorKind::Mass ? "mass" : "diffusion");
      report(what, pa.stored_reals() == ref.stored_reals());
   }
}

} // namespace

int main()
{
   b200::Device dev(0, TFEM_NUMERICS_REFERENCE); // bit-identical mode for the == checks
   for (int p : {1, 2, 3, 4}) {
      check_space(dev, FeSpace(make_cartesian(8, 8), FeCollection(FeFamily::H1, p)), "cartesian");
      check_space(dev,
                  FeSpace(curve_mesh(make_cartesian(4, 4), 2,
                                     [](Vec2 q) {
                                        return Vec2{q.x * (1.0 + 0.2 * q.y),
                                                    q.y * (1.0 + 0.1 * q.x)};
                                     }),
                          FeCollection(FeFamily::H1, p)),
                  "curved");
   }

   // The driver's system (driver.cpp:129-164) solved both ways.
   for (int p : {2, 3}) {
      const FeSpace space(make_cartesian(16, 16), FeCollection(FeFamily::H1, p));
      const ManufacturedSolution sol = manufactured_solution(SolutionId::Front);
      BilinearForm a(space, AssemblyMode::Partial);
      a.add_diffusion([](Vec2) { return 1.0; });
      a.assemble();
      const LinearForm b(space, sol.f);
      const std::vector<int> ess = space.essential_true_dofs(all_attrs(space.mesh()));
      const GridFunction interp = project_coefficient(space, sol.u);
      const LinearSystem sys = form_linear_system(a, b, ess, space.local_to_true(interp.values()));
      Vector rhs = sys.rhs;
      for (int e : ess) rhs[e] = 0.0;
      Vector diag = a.diagonal_true();
      for (int e : ess) diag[e] = 1.0;

      b200::DeviceSpace ds(dev, space);
      b200::DevicePa pa(ds, IntegratorKind::Diffusion, [](Vec2) { return 1.0; });
      b200::DeviceOperator op(ds, {&pa}, ess);
      const Vector x = random_vector(space.n_true_dofs(), 9);
      Vector yr(x.size()), yd(x.size());
      sys.op->mult(x, yr);
      op.mult(x, yd);
      char what[160];
      std::snprintf(what, sizeof what, "front p=%d: ConstrainedOperator bit-identical", p);
      report(what, equal(yr, yd));
      Vector dd = op.diagonal();
      std::snprintf(what, sizeof what, "front p=%d: Jacobi diagonal bit-identical", p);
      report(what, equal(dd, diag));

      const CgResult cr = cg_solve(*sys.op, rhs, 1e-12, 2000, &diag);
      const CgResult cd = b200::cg_solve(op, rhs, 1e-12, 2000, &diag);
      double err = 0.0, scale = 0.0;
      for (int i = 0; i < rhs.size(); i++) {
         err = std::max(err, std::abs(cr.x[i] - cd.x[i]));
         scale = std::max(scale, std::abs(cr.x[i]));
      }
      char detail[96];
      std::snprintf(detail, sizeof detail, "(ref %d, device %d iterations; max diff %.1e)",
                    cr.iterations, cd.iterations, err / scale);
      std::snprintf(what, sizeof what, "front p=%d: cg_solve same iterations, x to 1e-10", p);
      report(what, cr.iterations == cd.iterations && cr.converged == cd.converged &&
                      err <= 1e-10 * scale,
             detail);
   }

   // Non-conforming forests (acceptance_main.cpp:58-68 refinement draw): the
   // device P, operator, diagonal and the constrained solve.
   for (int p : {1, 2, 3}) {
      NcForest forest(make_cartesian(4, 4));
      std::mt19937 gen(21 + p);
      for (int i = 0; i < 10; i++) {
         const int leaf = std::uniform_int_distribution<int>(0, forest.n_leaves() - 1)(gen);
         const int kind = std::uniform_int_distribution<int>(0, 2)(gen);
         forest.refine({{leaf, kind == 0   ? SplitKind::Iso
                               : kind == 1 ? SplitKind::X
                                           : SplitKind::Y}});
      }
      const FeSpace space(forest, FeCollection(FeFamily::H1, p));
      char what[160];
      check_space(dev, space, "forest");
      const ManufacturedSolution sol = manufactured_solution(SolutionId::Front);
      BilinearForm a(space, AssemblyMode::Partial);
      a.add_diffusion([](Vec2) { return 1.0; });
      a.assemble();
      const LinearForm b(space, sol.f);
      const std::vector<int> ess = space.essential_true_dofs(all_attrs(space.mesh()));
      const GridFunction interp = project_coefficient(space, sol.u);
      const LinearSystem sys = form_linear_system(a, b, ess, space.local_to_true(interp.values()));
      Vector rhs = sys.rhs;
      for (int e : ess) rhs[e] = 0.0;
      Vector diag = a.diagonal_true();
      for (int e : ess) diag[e] = 1.0;
      b200::DeviceSpace ds(dev, space);
      b200::DevicePa pa(ds, IntegratorKind::Diffusion, [](Vec2) { return 1.0; });
      b200::DeviceOperator op(ds, {&pa}, ess);
      const Vector x = random_vector(space.n_true_dofs(), 10 + p);
      Vector yr(x.size()), yd(x.size());
      sys.op->mult(x, yr);
      op.mult(x, yd);
      std::snprintf(what, sizeof what, "forest p=%d: ConstrainedOperator bit-identical", p);
      report(what, equal(yr, yd));
      std::snprintf(what, sizeof what, "forest p=%d: Jacobi diagonal bit-identical", p);
      report(what, equal(op.diagonal(), diag));
      const CgResult cr = cg_solve(*sys.op, rhs, 1e-12, 3000, &diag);
      const CgResult cd = b200::cg_solve(op, rhs, 1e-12, 3000, &diag);
      double err = 0.0, scale = 0.0;
      for (int i = 0; i < rhs.size(); i++) {
         err = std::max(err, std::abs(cr.x[i] - cd.x[i]));
         scale = std::max(scale, std::abs(cr.x[i]));
      }
      char detail[96];
      std::snprintf(detail, sizeof detail, "(ref %d, device %d iterations; max diff %.1e)",
                    cr.iterations, cd.iterations, err / scale);
      // dots are tree-reduced on the device: the stop may move by one
      // iteration when ||r|| lands on the threshold (tests/test_gpu_nc.py)
      std::snprintf(what, sizeof what, "forest p=%d: cg_solve iterations +-1, x to 1e-10", p);
      report(what, std::abs(cr.iterations - cd.iterations) <= 1 && cr.converged == cd.converged &&
                      err <= 1e-10 * scale,
             detail);
   }

   // The driver: the reference's solve_poisson /
   // convergence_study / amr_loop next to the same loops with every numeric
   // step on the device.  Rows: same DOF counts and stored reals, CG
   // iterations equal (+-1 on forests), L2 errors to 1e-9.
   auto compare_rows = [&](const char *name, const RunResult &r, const RunResult &d, int slack) {
      bool ok = r.rows.size() == d.rows.size() && r.converged == d.converged;
      double worst = 0.0;
      for (size_t i = 0; ok && i < r.rows.size(); i++) {
         const ConvergenceRow &a = r.rows[i], &b = d.rows[i];
         ok = a.n_true_dofs == b.n_true_dofs && a.pa_stored_reals == b.pa_stored_reals &&
              std::abs(a.cg_iterations - b.cg_iterations) <= slack && a.h == b.h;
         const double rel = std::abs(a.l2_error - b.l2_error) / a.l2_error;
         worst = std::max(worst, rel);
         ok = ok && rel <= 1e-9;
      }
      char detail[160];
      std::snprintf(detail, sizeof detail, "(%zu rows; last: ref %d / device %d iterations, "
                    "l2 %.6e / %.6e; worst l2 rel diff %.1e)", r.rows.size(),
                    r.rows.empty() ? 0 : r.rows.back().cg_iterations,
                    d.rows.empty() ? 0 : d.rows.back().cg_iterations,
                    r.rows.empty() ? 0.0 : r.rows.back().l2_error,
                    d.rows.empty() ? 0.0 : d.rows.back().l2_error, worst);
      report(name, ok, detail);
   };
   for (int p : {2, 3}) {
      RunConfig c;
      c.cartesian_n = 16;
      c.order = p;
      c.solution = SolutionId::Front;
      char what[96];
      std::snprintf(what, sizeof what, "driver solve_poisson front n=16 p=%d", p);
      compare_rows(what, solve_poisson(c), b200::solve_poisson(dev, c), 0);
   }
   {
      RunConfig c;
      c.cartesian_n = 4;
      c.order = 2;
      c.solution = SolutionId::Sine;
      c.convergence_levels = 4;
      compare_rows("driver convergence_study sine n=4 p=2, 4 levels", convergence_study(c),
                   b200::convergence_study(dev, c), 1);
   }
   {
      RunConfig c;
      c.cartesian_n = 4;
      c.order = 2;
      c.solution = SolutionId::Front;
      c.amr.iters = 4;
      c.amr.theta = 0.5;
      compare_rows("driver amr_loop front n=4 p=2, 4 rounds", amr_loop(c), b200::amr_loop(dev, c),
                   1);
      c.amr.anisotropic = true;
      compare_rows("driver amr_loop front anisotropic", amr_loop(c), b200::amr_loop(dev, c), 1);
   }

   // Error mapping: the reference's exception classes come back.
   {
      const FeSpace space(make_cartesian(2, 2), FeCollection(FeFamily::H1, 1));
      b200::DeviceSpace ds(dev, space);
      bool thrown = false;
      try {
         b200::DevicePa pa(ds, IntegratorKind::Diffusion, [](Vec2) { return 0.0; });
      } catch (const std::invalid_argument &e) {
         thrown = std::string(e.what()).find("coefficient must be positive") != std::string::npos;
      }
      report("non-positive coefficient -> std::invalid_argument", thrown);
   }
   std::printf("%d failure(s)\n", failures);
   return failures;
}
