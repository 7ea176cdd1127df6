// ORACLE INFRASTRUCTURE -- test/benchmark checker only, never on the product
// path.  A thin extern "C" shim over the UNMODIFIED reference library
// (tensorfem, /root/reference/proj/src), compiled in place by
// oracle/Makefile with -Dtensorfem=tfem_ref into oracle/_ref/libtfem_ref.so.
// Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu
// baseline legs load it.
//
// Every entry point returns a status code that mirrors the reference's
// exception classes (0 ok, 1 std::invalid_argument, 2 std::runtime_error,
// 3 std::logic_error, 9 anything else); the message is in ref_last_error().

#include "tensorfem/driver.hpp"
#include "tensorfem/forms.hpp"
#include "tensorfem/ncmesh.hpp"
#include "tensorfem/quadrature.hpp"

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

using namespace tensorfem; // expands to tfem_ref under -Dtensorfem=tfem_ref

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F &&f)
{
   try {
      f();
      return 0;
   } catch (const std::invalid_argument &e) {
      g_err = e.what();
      return 1;
   } catch (const std::logic_error &e) { // before runtime_error: unrelated
      g_err = e.what();
      return 3;
   } catch (const std::runtime_error &e) {
      g_err = e.what();
      return 2;
   } catch (const std::exception &e) {
      g_err = e.what();
      return 9;
   }
}

// Coefficient catalogue shared with the tests (ids are the ABI):
//   0: constant `value`  1: 1 + x + 2y  (test_forms.cpp:31, acceptance:50)
Coefficient make_coeff(int id, double value)
{
   if (id == 0) {
      return [value](Vec2) { return value; };
   }
   if (id == 1) {
      return [](Vec2 p) { return 1.0 + p.x + 2.0 * p.y; };
   }
   throw std::invalid_argument("ref_shim: unknown coefficient id");
}

// The curving map of test_forms.cpp:33-38 / acceptance_main.cpp:52-57.
Vec2 test_curve_map(Vec2 p)
{
   return Vec2{p.x * (1.0 + 0.2 * p.y), p.y * (1.0 + 0.1 * p.x)};
}

struct Space {
   std::shared_ptr<const FeSpace> fes;
};

struct Form {
   Space *space;
   std::unique_ptr<BilinearForm> form;
};

struct System {
   Form *form;
   std::vector<int> ess;
   Vector values;
   Vector rhs;  // homogenised (rhs[ess] = 0), driver.cpp:147-150
   Vector diag; // diag[ess] = 1, driver.cpp:151-159
   Vector x0;
   std::unique_ptr<LinearOperator> op;
   ManufacturedSolution sol;
};

std::vector<int> all_boundary_attrs(const Mesh &mesh)
{
   std::set<int> attrs;
   for (const BoundarySegment &s : mesh.boundary_segments()) {
      attrs.insert(s.attribute);
   }
   return {attrs.begin(), attrs.end()};
}

} // namespace

extern "C" {

const char *ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- 1D rules
int ref_gauss_legendre(int n, double *pts, double *wts)
{
   return guarded([&] {
      const QuadratureRule1D r = gauss_legendre(n);
      std::memcpy(pts, r.points.data(), sizeof(double) * n);
      std::memcpy(wts, r.weights.data(), sizeof(double) * n);
   });
}

int ref_gauss_lobatto(int n, double *pts, double *wts)
{
   return guarded([&] {
      const QuadratureRule1D r = gauss_lobatto(n);
      std::memcpy(pts, r.points.data(), sizeof(double) * n);
      std::memcpy(wts, r.weights.data(), sizeof(double) * n);
   });
}

// B1d/G1d (nq x (p+1), row-major) of the order-p basis on `node_kind`
// (0 GLL, 1 GL, 2 uniform) at the nq-point rule `rule_kind` (0 GL, 1 GLL).
int ref_eval_matrices(int p, int node_kind, int nq, int rule_kind, double *B,
                      double *G)
{
   return guarded([&] {
      const Basis1D basis(p, static_cast<NodeKind>(node_kind));
      const QuadratureRule1D rule =
         rule_kind == 0 ? gauss_legendre(nq) : gauss_lobatto(nq);
      const EvalMatrices em = eval_matrices(basis, rule);
      std::memcpy(B, em.B1d.data(), sizeof(double) * nq * (p + 1));
      std::memcpy(G, em.G1d.data(), sizeof(double) * nq * (p + 1));
   });
}

// ------------------------------------------------------------------ spaces
void *ref_space_cartesian(int nx, int ny, int p, double w, double h)
{
   Space *s = nullptr;
   const int rc = guarded([&] {
      s = new Space{std::make_shared<const FeSpace>(
         make_cartesian(nx, ny, w, h), FeCollection(FeFamily::H1, p))};
   });
   return rc == 0 ? s : nullptr;
}

// curve_mesh(make_cartesian(n, n), m, test map) -- acceptance_main.cpp:52-57
void *ref_space_curved(int n, int p, int m)
{
   Space *s = nullptr;
   const int rc = guarded([&] {
      s = new Space{std::make_shared<const FeSpace>(
         curve_mesh(make_cartesian(n, n), m, test_curve_map),
         FeCollection(FeFamily::H1, p))};
   });
   return rc == 0 ? s : nullptr;
}

// Forest over make_cartesian(n, n) refined `count` times by the seeded
// random leaf/kind draw of acceptance_main.cpp:58-68.
void *ref_space_random_forest(int n, int p, int count, unsigned seed)
{
   Space *s = nullptr;
   const int rc = guarded([&] {
      NcForest forest(make_cartesian(n, n));
      std::mt19937 gen(seed);
      for (int i = 0; i < count; i++) {
         const int leaf = std::uniform_int_distribution<int>(
            0, forest.n_leaves() - 1)(gen);
         const int kind = std::uniform_int_distribution<int>(0, 2)(gen);
         forest.refine({{leaf, kind == 0   ? SplitKind::Iso
                               : kind == 1 ? SplitKind::X
                                           : SplitKind::Y}});
      }
      s = new Space{std::make_shared<const FeSpace>(
         forest, FeCollection(FeFamily::H1, p))};
   });
   return rc == 0 ? s : nullptr;
}

void ref_space_free(void *s) { delete static_cast<Space *>(s); }

void ref_space_info(void *sp, int *n_dofs, int *n_true, int *n_elem,
                    int *order, int *conforming, int *geom_order)
{
   const FeSpace &f = *static_cast<Space *>(sp)->fes;
   *n_dofs = f.n_dofs();
   *n_true = f.n_true_dofs();
   *n_elem = f.mesh().n_elements();
   *order = f.collection().order();
   *conforming = f.conforming() ? 1 : 0;
   *geom_order = f.mesh().geometry_order();
}

void ref_space_element_dofs(void *sp, int *out)
{
   const FeSpace &f = *static_cast<Space *>(sp)->fes;
   const int nd2 = (f.collection().order() + 1) * (f.collection().order() + 1);
   for (int k = 0; k < f.mesh().n_elements(); k++) {
      const auto d = f.element_dofs(k);
      std::memcpy(out + static_cast<size_t>(k) * nd2, d.data(),
                  sizeof(int) * nd2);
   }
}

void ref_space_true_index(void *sp, int *out)
{
   const FeSpace &f = *static_cast<Space *>(sp)->fes;
   for (int d = 0; d < f.n_dofs(); d++) {
      out[d] = f.true_index(d);
   }
}

// Sorted essential true DOFs over every boundary attribute (driver.cpp:36-46).
int ref_space_essential(void *sp, int *out, int *count)
{
   return guarded([&] {
      const FeSpace &f = *static_cast<Space *>(sp)->fes;
      const std::vector<int> ess =
         f.essential_true_dofs(all_boundary_attrs(f.mesh()));
      if (out) {
         std::memcpy(out, ess.data(), sizeof(int) * ess.size());
      }
      *count = static_cast<int>(ess.size());
   });
}

// Prolongation P (n_dofs x n_true) as CSR; pass null arrays to get nnz.
int ref_space_prolongation(void *sp, int *rowptr, int *cols, double *vals,
                           long long *nnz)
{
   return guarded([&] {
      const FeSpace &f = *static_cast<Space *>(sp)->fes;
      const SparseMatrix &P = f.prolongation();
      *nnz = P.nnz();
      if (!rowptr) {
         return;
      }
      long long at = 0;
      rowptr[0] = 0;
      for (int i = 0; i < P.rows(); i++) {
         const auto c = P.row_cols(i);
         const auto v = P.row_vals(i);
         for (size_t j = 0; j < c.size(); j++) {
            cols[at] = c[j];
            vals[at] = v[j];
            at++;
         }
         rowptr[i + 1] = static_cast<int>(at);
      }
   });
}

// Element vertex coordinates, corner order v0..v3 (counterclockwise), as
// E x 4 x {x, y}.
void ref_space_element_vertices(void *sp, double *out)
{
   const Mesh &m = static_cast<Space *>(sp)->fes->mesh();
   for (int k = 0; k < m.n_elements(); k++) {
      for (int c = 0; c < 4; c++) {
         const Vec2 &v = m.vertex(m.element(k).v[c]);
         out[(static_cast<size_t>(k) * 4 + c) * 2 + 0] = v.x;
         out[(static_cast<size_t>(k) * 4 + c) * 2 + 1] = v.y;
      }
   }
}

// Geometry control points of a curved mesh: E x (m+1)^2 x {x, y}, lattice
// order x fastest (mesh.cpp:228-237).
int ref_space_geometry_nodes(void *sp, double *out)
{
   return guarded([&] {
      const Mesh &m = static_cast<Space *>(sp)->fes->mesh();
      const NodalField *nodes = m.nodes();
      if (!nodes) {
         throw std::invalid_argument("ref_space_geometry_nodes: straight mesh");
      }
      const int n2 = (nodes->order + 1) * (nodes->order + 1);
      for (int k = 0; k < m.n_elements(); k++) {
         const auto dofs = nodes->layout.dofs(k);
         for (int i = 0; i < n2; i++) {
            const Vec2 &c = nodes->coords[dofs[i]];
            out[(static_cast<size_t>(k) * n2 + i) * 2 + 0] = c.x;
            out[(static_cast<size_t>(k) * n2 + i) * 2 + 1] = c.y;
         }
      }
   });
}

// ------------------------------------------------------------------- forms
// mode 0 Full, 1 Partial; kinds 0 diffusion, 1 mass (forms.hpp:18-19).
void *ref_form_create(void *sp, int mode, int n_integ, const int *kinds,
                      const int *coeff_ids, const double *coeff_vals,
                      int threads)
{
   Form *f = nullptr;
   const int rc = guarded([&] {
      auto *space = static_cast<Space *>(sp);
      auto form = std::make_unique<BilinearForm>(
         *space->fes, mode == 0 ? AssemblyMode::Full : AssemblyMode::Partial);
      for (int i = 0; i < n_integ; i++) {
         Coefficient c = make_coeff(coeff_ids[i], coeff_vals[i]);
         if (kinds[i] == 0) {
            form->add_diffusion(c);
         } else {
            form->add_mass(c);
         }
      }
      form->assemble(threads);
      f = new Form{space, std::move(form)};
   });
   return rc == 0 ? f : nullptr;
}

void ref_form_free(void *f) { delete static_cast<Form *>(f); }

int ref_form_mult(void *fp, const double *x, double *y)
{
   return guarded([&] {
      const BilinearForm &a = *static_cast<Form *>(fp)->form;
      const int n = a.true_size();
      Vector xv(n), yv(n);
      std::memcpy(xv.data(), x, sizeof(double) * n);
      a.mult_true(xv, yv);
      std::memcpy(y, yv.data(), sizeof(double) * n);
   });
}

// Multiplies counted by the instrumented kernels during one mult_true
// (tensor_kernels.hpp:20-26).
int ref_form_mult_count(void *fp, const double *x, double *y,
                        unsigned long long *count)
{
   return guarded([&] {
      const BilinearForm &a = *static_cast<Form *>(fp)->form;
      const int n = a.true_size();
      Vector xv(n), yv(n);
      std::memcpy(xv.data(), x, sizeof(double) * n);
      reset_multiply_count();
      a.mult_true(xv, yv);
      *count = multiply_count();
      std::memcpy(y, yv.data(), sizeof(double) * n);
   });
}

int ref_form_diag(void *fp, double *out)
{
   return guarded([&] {
      const BilinearForm &a = *static_cast<Form *>(fp)->form;
      const Vector d = a.diagonal_true();
      std::memcpy(out, d.data(), sizeof(double) * d.size());
   });
}

long long ref_form_stored_reals(void *fp)
{
   return static_cast<Form *>(fp)->form->stored_reals();
}

// Point factors of integrator `integ`, reference layout [e][qy][qx][c].
int ref_form_qdata(void *fp, int integ, double *out, int *nq, int *nc)
{
   return guarded([&] {
      const auto &pa = static_cast<Form *>(fp)->form->pa_data().at(integ);
      *nq = pa.quad_1d();
      *nc = pa.kind() == IntegratorKind::Mass ? 1 : 3;
      if (!out) {
         return;
      }
      const size_t per = static_cast<size_t>(*nq) * *nq * *nc;
      for (int k = 0; k < pa.n_elements(); k++) {
         const auto d = pa.d(k);
         std::memcpy(out + per * k, d.data(), sizeof(double) * per);
      }
   });
}

// pa_setup on its own (forms.cpp:201-229), for error-path parity.
int ref_pa_setup(void *sp, int kind, int coeff_id, double coeff_val)
{
   return guarded([&] {
      const FeSpace &f = *static_cast<Space *>(sp)->fes;
      (void)pa_setup(f,
                     kind == 0 ? IntegratorKind::Diffusion
                               : IntegratorKind::Mass,
                     make_coeff(coeff_id, coeff_val));
   });
}

// Full-mode global true matrix as CSR (null arrays -> nnz only).
int ref_form_matrix(void *fp, int *rowptr, int *cols, double *vals,
                    long long *nnz)
{
   return guarded([&] {
      const SparseMatrix &A = static_cast<Form *>(fp)->form->matrix();
      *nnz = A.nnz();
      if (!rowptr) {
         return;
      }
      long long at = 0;
      rowptr[0] = 0;
      for (int i = 0; i < A.rows(); i++) {
         const auto c = A.row_cols(i);
         const auto v = A.row_vals(i);
         for (size_t j = 0; j < c.size(); j++) {
            cols[at] = c[j];
            vals[at] = v[j];
            at++;
         }
         rowptr[i + 1] = static_cast<int>(at);
      }
   });
}

// ----------------------------------------------------- driver-style system
// The Poisson system of solve_on_space (driver.cpp:129-159): manufactured
// solution `solution` (0 sine, 1 front), Dirichlet on every boundary
// attribute, homogenised rhs, Jacobi diagonal with ones on essential DOFs.
void *ref_system_create(void *fp, int solution)
{
   System *s = nullptr;
   const int rc = guarded([&] {
      auto *form = static_cast<Form *>(fp);
      const FeSpace &space = *form->space->fes;
      auto sys = std::make_unique<System>();
      sys->form = form;
      sys->sol = manufactured_solution(solution == 0 ? SolutionId::Sine
                                                     : SolutionId::Front);
      const LinearForm b(space, sys->sol.f);
      sys->ess = space.essential_true_dofs(all_boundary_attrs(space.mesh()));
      const GridFunction interp = project_coefficient(space, sys->sol.u);
      sys->values = space.local_to_true(interp.values());
      LinearSystem ls =
         form_linear_system(*form->form, b, sys->ess, sys->values);
      sys->rhs = ls.rhs;
      for (int e : sys->ess) {
         sys->rhs[e] = 0.0;
      }
      sys->x0 = ls.x0;
      sys->op = std::move(ls.op);
      sys->diag = form->form->diagonal_true();
      for (int e : sys->ess) {
         sys->diag[e] = 1.0;
      }
      s = sys.release();
   });
   return rc == 0 ? s : nullptr;
}

void ref_system_free(void *s) { delete static_cast<System *>(s); }

void ref_system_vectors(void *sp, double *rhs, double *diag, double *x0)
{
   const System &s = *static_cast<System *>(sp);
   const int n = s.rhs.size();
   if (rhs) std::memcpy(rhs, s.rhs.data(), sizeof(double) * n);
   if (diag) std::memcpy(diag, s.diag.data(), sizeof(double) * n);
   if (x0) std::memcpy(x0, s.x0.data(), sizeof(double) * n);
}

int ref_system_ess(void *sp, int *out)
{
   const System &s = *static_cast<System *>(sp);
   if (out) std::memcpy(out, s.ess.data(), sizeof(int) * s.ess.size());
   return static_cast<int>(s.ess.size());
}

// The constrained operator of form_linear_system (forms.cpp:164-190).
int ref_system_op_mult(void *sp, const double *x, double *y)
{
   return guarded([&] {
      const System &s = *static_cast<System *>(sp);
      const int n = s.rhs.size();
      Vector xv(n), yv(n);
      std::memcpy(xv.data(), x, sizeof(double) * n);
      s.op->mult(xv, yv);
      std::memcpy(y, yv.data(), sizeof(double) * n);
   });
}

// cg_solve on the constrained operator with an arbitrary rhs (null -> the
// system rhs); jacobi selects the system diagonal.  seconds = wall time of
// cg_solve alone (driver.cpp:160-164).
int ref_system_cg(void *sp, const double *rhs, double tol, int max_iters,
                  int jacobi, double *x_out, int *iters, int *converged,
                  double *seconds)
{
   return guarded([&] {
      const System &s = *static_cast<System *>(sp);
      const int n = s.rhs.size();
      Vector b = s.rhs;
      if (rhs) std::memcpy(b.data(), rhs, sizeof(double) * n);
      const auto t0 = std::chrono::steady_clock::now();
      const CgResult r =
         cg_solve(*s.op, b, tol, max_iters, jacobi ? &s.diag : nullptr);
      const std::chrono::duration<double> dt =
         std::chrono::steady_clock::now() - t0;
      if (seconds) *seconds = dt.count();
      if (x_out) std::memcpy(x_out, r.x.data(), sizeof(double) * n);
      *iters = r.iterations;
      *converged = r.converged ? 1 : 0;
   });
}

// L2 error of x_cg + x0 against the exact solution (driver.cpp:166-178).
int ref_system_l2_error(void *sp, const double *x_cg, double *err)
{
   return guarded([&] {
      const System &s = *static_cast<System *>(sp);
      const FeSpace &space = *s.form->space->fes;
      Vector x(s.rhs.size());
      for (int i = 0; i < x.size(); i++) {
         x[i] = x_cg[i] + s.x0[i];
      }
      const GridFunction u = recover_fem_solution(space, x);
      *err = compute_l2_error(u, s.sol.u);
   });
}

// LinearForm(space, f) (forms.cpp:400-431) for the manufactured source of
// `solution` (0 sine, 1 front): the L-vector b.
int ref_linear_form(void *sp, int solution, double *out)
{
   return guarded([&] {
      const FeSpace &space = *static_cast<Space *>(sp)->fes;
      const ManufacturedSolution sol =
         manufactured_solution(solution == 0 ? SolutionId::Sine : SolutionId::Front);
      const LinearForm b(space, sol.f);
      for (int i = 0; i < b.values().size(); i++) out[i] = b.values()[i];
   });
}

// project_coefficient(space, u) of the manufactured solution, L-vector.
int ref_project(void *sp, int solution, double *out)
{
   return guarded([&] {
      const FeSpace &space = *static_cast<Space *>(sp)->fes;
      const ManufacturedSolution sol =
         manufactured_solution(solution == 0 ? SolutionId::Sine : SolutionId::Front);
      const GridFunction g = project_coefficient(space, sol.u);
      for (int i = 0; i < g.values().size(); i++) out[i] = g.values()[i];
   });
}

// compute_l2_error of the L-vector x against the manufactured solution.
int ref_l2_error(void *sp, int solution, const double *x, double *err)
{
   return guarded([&] {
      const FeSpace &space = *static_cast<Space *>(sp)->fes;
      const ManufacturedSolution sol =
         manufactured_solution(solution == 0 ? SolutionId::Sine : SolutionId::Front);
      GridFunction g(space);
      for (int i = 0; i < g.values().size(); i++) g.values()[i] = x[i];
      *err = compute_l2_error(g, sol.u);
   });
}

// The manufactured solution u of `solution` at n points xy[2n].
int ref_solution_u(int solution, const double *xy, int n, double *out)
{
   return guarded([&] {
      const ManufacturedSolution sol =
         manufactured_solution(solution == 0 ? SolutionId::Sine : SolutionId::Front);
      for (int i = 0; i < n; i++) out[i] = sol.u(Vec2{xy[2 * i], xy[2 * i + 1]});
   });
}

// The manufactured source f of `solution` at n points xy[2n].
int ref_solution_f(int solution, const double *xy, int n, double *out)
{
   return guarded([&] {
      const ManufacturedSolution sol =
         manufactured_solution(solution == 0 ? SolutionId::Sine : SolutionId::Front);
      for (int i = 0; i < n; i++) out[i] = sol.f(Vec2{xy[2 * i], xy[2 * i + 1]});
   });
}

// Whole reference driver (driver.cpp:187-194) for table-level parity.
int ref_solve_poisson(int n, int p, int solution, int jacobi, double tol,
                      int max_iters, int threads, int *iters, int *converged,
                      double *l2, double *seconds, long long *pa_reals)
{
   return guarded([&] {
      RunConfig c;
      c.cartesian_n = n;
      c.order = p;
      c.solution = solution == 0 ? SolutionId::Sine : SolutionId::Front;
      c.prec = jacobi ? Preconditioner::Jacobi : Preconditioner::None;
      c.tol = tol;
      c.max_iters = max_iters;
      c.threads = threads;
      const RunResult r = solve_poisson(c);
      *iters = r.rows[0].cg_iterations;
      *converged = r.converged ? 1 : 0;
      *l2 = r.rows[0].l2_error;
      *seconds = r.rows[0].solve_seconds;
      *pa_reals = r.rows[0].pa_stored_reals;
   });
}

// ------------------------------------------------------ generic CG on CSR
int ref_cg_csr(int n, const int *rowptr, const int *cols, const double *vals,
               const double *b, double tol, int max_iters, const double *diag,
               double *x_out, int *iters, int *converged)
{
   return guarded([&] {
      SparseMatrix::Builder bld(n, n);
      for (int i = 0; i < n; i++) {
         for (int k = rowptr[i]; k < rowptr[i + 1]; k++) {
            bld.add(i, cols[k], vals[k]);
         }
      }
      const SparseMatrix A = bld.build();
      const SparseOperator op(A);
      Vector bv(n), dv(n);
      std::memcpy(bv.data(), b, sizeof(double) * n);
      if (diag) std::memcpy(dv.data(), diag, sizeof(double) * n);
      const CgResult r = cg_solve(op, bv, tol, max_iters, diag ? &dv : nullptr);
      std::memcpy(x_out, r.x.data(), sizeof(double) * n);
      *iters = r.iterations;
      *converged = r.converged ? 1 : 0;
   });
}

} // extern "C"
