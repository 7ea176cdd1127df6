// tensorfem_b200.hpp -- the reference-side binding of the B200 PA path.
//
// Header-only adaptor written against the reference's own public API
// (tensorfem::FeSpace, Coefficient, Vector, LinearOperator, CgResult;
// /root/reference/proj/include/tensorfem) that routes the hot path through
// the C ABI of libtfem_cuda.so (include/tfem_cuda.h).  This is what a
// maintainer adds to the reference (INTEGRATION.md shows the three call
// sites in forms.cpp / solvers.cpp); nothing else in the reference changes.
//
//   reference call                         routed to
//   pa_setup(space, kind, coeff)           tfem_pa_setup (coefficient
//                                          evaluated on the host at
//                                          tfem_geometry_points)
//   pa_apply_local(pa, space, x, y)        tfem_pa_apply_local
//   pa_diagonal(pa, space)                 tfem_pa_diagonal
//   BilinearForm::mult_true                tfem_operator_mult
//   ConstrainedOperator                    tfem_operator_create_p(..., ess)
//   FeSpace::prolongation() (NC forests)   tfem_prolongation_create
//   cg_solve(op, b, tol, it, diag)         tfem_cg_solve (device loop)
//   LinearForm(space, f)                   tfem_linear_form
//   project_coefficient / compute_l2_error tfem_project / tfem_l2_error
//   solve_on_space / convergence_study /   b200::solve_on_space & co. below:
//   amr_loop (driver.cpp:129-258)          every numeric step on the device,
//                                          forest refinement and marking on
//                                          the host (reference code)
#pragma once

#include "tensorfem/driver.hpp"
#include "tensorfem/forms.hpp"
#include "tensorfem/mesh_io.hpp"
#include "tensorfem/ncmesh.hpp"
#include "tfem_cuda.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <limits>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

namespace tensorfem {
namespace b200 {

// Status code -> the reference's exception classes.
inline void check(int rc)
{
   if (rc == TFEM_OK) return;
   const std::string msg = tfem_last_error();
   switch (rc) {
   case TFEM_INVALID_ARGUMENT: throw std::invalid_argument(msg);
   case TFEM_LOGIC_ERROR: throw std::logic_error(msg);
   default: throw std::runtime_error(msg);
   }
}

class Device {
public:
   /// numerics: TFEM_NUMERICS_FMA (default) or TFEM_NUMERICS_REFERENCE
   /// (the reference's operation order, bit-identical results).
   explicit Device(int device = 0, int numerics = TFEM_NUMERICS_FMA)
   {
      check(tfem_ctx_create(device, &ctx_));
      check(tfem_ctx_set_numerics(ctx_, numerics));
   }
   ~Device() { tfem_ctx_destroy(ctx_); }
   Device(const Device &) = delete;
   Device &operator=(const Device &) = delete;
   tfem_ctx *get() const { return ctx_; }

private:
   tfem_ctx *ctx_ = nullptr;
};

// Device vector with host Vector copies in / out.
class DVec {
public:
   DVec(const Device &d, int n) { check(tfem_vec_create(d.get(), n, &v_)); }
   DVec(const Device &d, const Vector &x) : DVec(d, x.size()) { upload(x); }
   ~DVec() { tfem_vec_destroy(v_); }
   DVec(const DVec &) = delete;
   DVec &operator=(const DVec &) = delete;
   void upload(const Vector &x) { check(tfem_vec_upload(v_, x.data(), x.size())); }
   void download(Vector &x) const { check(tfem_vec_download(v_, x.data(), x.size())); }
   tfem_vec *get() const { return v_; }

private:
   tfem_vec *v_ = nullptr;
};

// G, the element geometry and (non-conforming forests) P of a reference
// FeSpace.
class DeviceSpace {
public:
   DeviceSpace(const Device &dev, const FeSpace &space) : dev_(&dev), space_(&space)
   {
      const Mesh &mesh = space.mesh();
      const int ne = mesh.n_elements();
      const int p = space.collection().order();
      const int nd = (p + 1) * (p + 1);
      std::vector<int32_t> dofs(static_cast<size_t>(ne) * nd);
      for (int k = 0; k < ne; k++) {
         const auto d = space.element_dofs(k);
         for (int i = 0; i < nd; i++) dofs[static_cast<size_t>(k) * nd + i] = d[i];
      }
      check(tfem_restriction_create(dev.get(), 2, p, ne, space.n_dofs(), dofs.data(), &r_));
      // Control points in lattice order (mesh.cpp:228-241).
      const int m = mesh.geometry_order();
      const int nc = (m + 1) * (m + 1);
      std::vector<double> ctrl(static_cast<size_t>(ne) * nc * 2);
      for (int k = 0; k < ne; k++) {
         if (const NodalField *nodes = mesh.nodes()) {
            const auto gd = nodes->layout.dofs(k);
            for (int i = 0; i < nc; i++) {
               ctrl[(static_cast<size_t>(k) * nc + i) * 2] = nodes->coords[gd[i]].x;
               ctrl[(static_cast<size_t>(k) * nc + i) * 2 + 1] = nodes->coords[gd[i]].y;
            }
         } else {
            const auto &v = mesh.element(k).v;
            const int lat[4] = {v[0], v[1], v[3], v[2]};
            for (int i = 0; i < 4; i++) {
               ctrl[(static_cast<size_t>(k) * 4 + i) * 2] = mesh.vertex(lat[i]).x;
               ctrl[(static_cast<size_t>(k) * 4 + i) * 2 + 1] = mesh.vertex(lat[i]).y;
            }
         }
      }
      check(tfem_geometry_create(dev.get(), 2, m, ne, ctrl.data(), &g_));
      if (!space.conforming()) {
         // P = [I; W] (fespace.cpp:166-203) and true_index
         const SparseMatrix &P = space.prolongation();
         std::vector<int32_t> rp(1, 0), cols, tix(space.n_dofs());
         std::vector<double> vals;
         for (int l = 0; l < P.rows(); l++) {
            const auto c = P.row_cols(l);
            const auto v = P.row_vals(l);
            cols.insert(cols.end(), c.begin(), c.end());
            vals.insert(vals.end(), v.begin(), v.end());
            rp.push_back(static_cast<int32_t>(cols.size()));
            tix[l] = space.true_index(l);
         }
         check(tfem_prolongation_create(dev.get(), P.rows(), P.cols(), rp.data(), cols.data(),
                                        vals.data(), tix.data(), &p_));
      }
   }
   ~DeviceSpace()
   {
      tfem_restriction_destroy(r_);
      tfem_geometry_destroy(g_);
      tfem_prolongation_destroy(p_);
   }
   DeviceSpace(const DeviceSpace &) = delete;
   DeviceSpace &operator=(const DeviceSpace &) = delete;
   const Device &device() const { return *dev_; }
   const FeSpace &space() const { return *space_; }
   tfem_restriction *restriction() const { return r_; }
   tfem_geometry *geometry() const { return g_; }
   tfem_prolongation *prolongation() const { return p_; } // NULL: conforming

private:
   const Device *dev_;
   const FeSpace *space_;
   tfem_restriction *r_ = nullptr;
   tfem_geometry *g_ = nullptr;
   tfem_prolongation *p_ = nullptr;
};

// PaData on the device (forms.hpp:29-58).
class DevicePa {
public:
   DevicePa(const DeviceSpace &s, IntegratorKind kind, const Coefficient &coeff) : s_(&s)
   {
      if (!coeff) throw std::invalid_argument("pa_setup: coefficient is empty");
      const int p = s.space().collection().order();
      const int nq = p + 2; // forms.cpp:211
      const int ne = s.space().mesh().n_elements();
      std::vector<double> xy(static_cast<size_t>(ne) * nq * nq * 2);
      check(tfem_geometry_points(s.device().get(), s.geometry(), nq, TFEM_GAUSS_LEGENDRE,
                                 xy.data()));
      std::vector<double> c(static_cast<size_t>(ne) * nq * nq);
      for (size_t i = 0; i < c.size(); i++) c[i] = coeff(Vec2{xy[2 * i], xy[2 * i + 1]});
      check(tfem_pa_setup(s.device().get(),
                          kind == IntegratorKind::Mass ? TFEM_MASS : TFEM_DIFFUSION,
                          s.geometry(), p, nq, TFEM_GAUSS_LEGENDRE, c.data(), 0.0, &pa_,
                          nullptr));
   }
   ~DevicePa() { tfem_pa_destroy(pa_); }
   DevicePa(const DevicePa &) = delete;
   DevicePa &operator=(const DevicePa &) = delete;
   tfem_pa *get() const { return pa_; }
   std::int64_t stored_reals() const { return tfem_pa_stored_reals(pa_); }

   /// pa_apply_local: y += G^T B^T D B G x (forms.cpp:231-296)
   void apply_local(const Vector &x, Vector &y) const
   {
      const Device &d = s_->device();
      DVec dx(d, x), dy(d, y);
      check(tfem_pa_apply_local(d.get(), pa_, s_->restriction(), dx.get(), dy.get()));
      dy.download(y);
      count_multiplies(tfem_pa_multiply_count(pa_));
   }

   /// pa_diagonal (forms.cpp:311-382), on the true DOFs
   Vector diagonal() const
   {
      const Device &d = s_->device();
      const int n = s_->space().n_true_dofs();
      DVec dd(d, n);
      if (s_->prolongation())
         check(tfem_pa_diagonal_p(d.get(), pa_, s_->restriction(), s_->prolongation(), dd.get()));
      else
         check(tfem_pa_diagonal(d.get(), pa_, s_->restriction(), dd.get()));
      Vector out(n);
      dd.download(out);
      return out;
   }

private:
   const DeviceSpace *s_;
   tfem_pa *pa_ = nullptr;
};

// mult_true / ConstrainedOperator as a reference LinearOperator
// (forms.cpp:164-190, 527-543): the virtual seam cg_solve drives.
class DeviceOperator : public LinearOperator {
public:
   DeviceOperator(const DeviceSpace &s, const std::vector<const DevicePa *> &pa,
                  const std::vector<int> &essential = {})
      : s_(&s)
   {
      std::vector<tfem_pa *> h;
      for (const DevicePa *x : pa) h.push_back(x->get());
      check(tfem_operator_create_p(s.device().get(), static_cast<int>(h.size()), h.data(),
                                   s.restriction(), s.prolongation(),
                                   static_cast<int64_t>(essential.size()),
                                   essential.empty() ? nullptr : essential.data(), &op_));
   }
   ~DeviceOperator() override { tfem_operator_destroy(op_); }
   int rows() const override { return static_cast<int>(tfem_operator_size(op_)); }
   int cols() const override { return rows(); }
   void mult(const Vector &x, Vector &y) const override
   {
      const Device &d = s_->device();
      DVec dx(d, x), dy(d, y.size());
      check(tfem_operator_mult(d.get(), op_, dx.get(), dy.get()));
      dy.download(y);
   }
   Vector diagonal() const
   {
      const Device &d = s_->device();
      DVec dd(d, rows());
      check(tfem_operator_diagonal(d.get(), op_, dd.get()));
      Vector out(rows());
      dd.download(out);
      return out;
   }
   tfem_operator *get() const { return op_; }
   const DeviceSpace &space() const { return *s_; }

private:
   const DeviceSpace *s_;
   tfem_operator *op_ = nullptr;
};

// ----------------------------------------------------------- rhs / post
// Host values of a point function at device-computed physical points.
inline std::vector<double> eval_at(const std::vector<double> &xy,
                                   const std::function<double(Vec2)> &f)
{
   std::vector<double> v(xy.size() / 2);
   for (size_t i = 0; i < v.size(); i++) v[i] = f(Vec2{xy[2 * i], xy[2 * i + 1]});
   return v;
}

/// LinearForm(space, f) (forms.cpp:400-431) as a device L-vector.
inline void linear_form(const DeviceSpace &s, const std::function<double(Vec2)> &f, DVec &b)
{
   const int p = s.space().collection().order(), nq = p + 2;
   std::vector<double> xy(static_cast<size_t>(s.space().mesh().n_elements()) * nq * nq * 2);
   check(tfem_geometry_points(s.device().get(), s.geometry(), nq, TFEM_GAUSS_LEGENDRE, xy.data()));
   const std::vector<double> fv = eval_at(xy, f);
   check(tfem_linear_form(s.device().get(), s.geometry(), s.restriction(), p, fv.data(), b.get()));
}

/// project_coefficient (fespace.cpp:334-356) as a device L-vector.
inline void project(const DeviceSpace &s, const std::function<double(Vec2)> &f, DVec &g)
{
   const int p = s.space().collection().order(), nd = p + 1;
   std::vector<double> xy(static_cast<size_t>(s.space().mesh().n_elements()) * nd * nd * 2);
   check(tfem_geometry_node_points(s.device().get(), s.geometry(), p, xy.data()));
   const std::vector<double> fv = eval_at(xy, f);
   check(tfem_project(s.device().get(), s.restriction(), fv.data(), g.get()));
}

/// compute_l2_error (fespace.cpp:358-394) of a device L-vector.
inline double l2_error(const DeviceSpace &s, const DVec &x, const std::function<double(Vec2)> &u)
{
   const int p = s.space().collection().order(), nq = p + 3;
   std::vector<double> xy(static_cast<size_t>(s.space().mesh().n_elements()) * nq * nq * 2);
   check(tfem_geometry_points(s.device().get(), s.geometry(), nq, TFEM_GAUSS_LEGENDRE, xy.data()));
   const std::vector<double> uv = eval_at(xy, u);
   double err = 0.0;
   check(tfem_l2_error(s.device().get(), s.geometry(), s.restriction(), p, x.get(), uv.data(),
                       &err));
   return err;
}

/// cg_solve (solvers.cpp:11-97) with the whole loop on the device when the
/// operator is a DeviceOperator.
inline CgResult cg_solve(const DeviceOperator &a, const Vector &b, double rel_tol,
                         int max_iters, const Vector *jacobi_diag = nullptr)
{
   if (b.size() != a.rows()) throw std::invalid_argument("cg_solve: operator/vector size mismatch");
   if (jacobi_diag && jacobi_diag->size() != b.size())
      throw std::invalid_argument("cg_solve: preconditioner size mismatch");
   CgResult res;
   res.x = Vector(b.size());
   tfem_cg_result r{};
   check(tfem_cg_solve_host(a.space().device().get(), a.get(), b.data(), rel_tol, max_iters,
                            jacobi_diag ? jacobi_diag->data() : nullptr, res.x.data(), &r));
   res.iterations = r.iterations;
   res.converged = r.converged != 0;
   return res;
}

// ------------------------------------------------------------- driver
// driver.cpp's file-local helpers (driver.cpp:28-67), restated.
inline Mesh build_mesh(const RunConfig &c)
{
   return c.mesh_path.empty() ? make_cartesian(c.cartesian_n, c.cartesian_n)
                              : load_native_file(c.mesh_path);
}

inline std::vector<int> boundary_attributes(const Mesh &mesh)
{
   std::set<int> attrs;
   for (const BoundarySegment &s : mesh.boundary_segments()) attrs.insert(s.attribute);
   if (attrs.empty()) throw std::runtime_error("driver: mesh has no boundary to constrain");
   return {attrs.begin(), attrs.end()};
}

inline double max_diameter(const Mesh &mesh)
{
   double h = 0.0;
   for (int k = 0; k < mesh.n_elements(); k++) h = std::max(h, mesh.element_diameter(k));
   return h;
}

inline void fill_orders(std::vector<ConvergenceRow> &rows)
{
   for (size_t i = 1; i < rows.size(); i++) {
      const double prev = rows[i - 1].l2_error, cur = rows[i].l2_error;
      if (prev > 0.0 && cur > 0.0 && std::isfinite(prev) && std::isfinite(cur))
         rows[i].order = std::log2(prev / cur);
   }
}

/// solve_on_space (driver.cpp:129-185) on the device: PA assembly, the rhs,
/// the projection of the boundary data, form_linear_system (forms.cpp:
/// 591-630: P^T b - A x0, rhs[ess] = values[ess]), the Jacobi diagonal, CG,
/// recover_fem_solution (P x) and the L2 error all run on the device; the
/// driver's bookkeeping stays on the host.  Partial assembly only.
inline RunResult solve_on_space(const Device &dev, std::shared_ptr<const FeSpace> space,
                                const ManufacturedSolution &sol, const RunConfig &config)
{
   if (config.assembly != AssemblyMode::Partial)
      throw std::invalid_argument("b200: the device driver runs partial assembly");
   const FeSpace &fes = *space;
   const int n = fes.n_true_dofs(), nl = fes.n_dofs();
   DeviceSpace ds(dev, fes);
   DevicePa pa(ds, IntegratorKind::Diffusion, [](Vec2) { return 1.0; });
   DVec b(dev, nl);
   linear_form(ds, sol.f, b);
   const std::vector<int> ess = fes.essential_true_dofs(boundary_attributes(fes.mesh()));
   DVec interp(dev, nl), values(dev, n);
   project(ds, sol.u, interp);
   if (ds.prolongation())
      check(tfem_prolongation_local_to_true(dev.get(), ds.prolongation(), interp.get(), values.get()));
   else
      check(tfem_vec_axpy(dev.get(), 1.0, interp.get(), values.get()));
   // form_linear_system: rhs = P^T b; x0 = values on ess; rhs -= A x0;
   // rhs[ess] = values[ess] -- then the driver zeroes rhs[ess]
   DVec rhs(dev, n);
   if (ds.prolongation())
      check(tfem_prolongation_mult_transpose(dev.get(), ds.prolongation(), b.get(), rhs.get()));
   else
      check(tfem_vec_axpy(dev.get(), 1.0, b.get(), rhs.get()));
   Vector hval(n), x0(n);
   values.download(hval);
   for (int e : ess) x0[e] = hval[e];
   if (!ess.empty()) {
      const DeviceOperator a(ds, {&pa});
      DVec dx0(dev, x0), ax(dev, n);
      check(tfem_operator_mult(dev.get(), a.get(), dx0.get(), ax.get()));
      check(tfem_vec_axpy(dev.get(), -1.0, ax.get(), rhs.get()));
   }
   Vector hrhs(n);
   rhs.download(hrhs);
   for (int e : ess) hrhs[e] = 0.0;
   const DeviceOperator op(ds, {&pa}, ess);
   Vector diag;
   const Vector *precond = nullptr;
   if (config.prec == Preconditioner::Jacobi) {
      diag = op.diagonal(); // diagonal_true with diag[ess] = 1
      precond = &diag;
   }
   const auto t0 = std::chrono::steady_clock::now();
   const CgResult cg = b200::cg_solve(op, hrhs, config.tol, config.max_iters, precond);
   const std::chrono::duration<double> elapsed = std::chrono::steady_clock::now() - t0;
   Vector x = cg.x;
   for (int i = 0; i < x.size(); i++) x[i] += x0[i];
   // recover_fem_solution: u = P x
   DVec dxt(dev, x), ul(dev, nl);
   if (ds.prolongation())
      check(tfem_prolongation_mult(dev.get(), ds.prolongation(), dxt.get(), ul.get()));
   else
      check(tfem_vec_axpy(dev.get(), 1.0, dxt.get(), ul.get()));
   RunResult out;
   out.space = space;
   GridFunction g(fes);
   ul.download(g.values());
   out.converged = cg.converged;
   ConvergenceRow row;
   row.n_true_dofs = n;
   row.h = max_diameter(fes.mesh());
   row.l2_error = l2_error(ds, ul, sol.u);
   row.order = std::numeric_limits<double>::quiet_NaN();
   row.cg_iterations = cg.iterations;
   row.solve_seconds = elapsed.count();
   row.pa_stored_reals = pa.stored_reals();
   out.rows.push_back(row);
   out.u = std::move(g);
   return out;
}

/// solve_poisson (driver.cpp:187-194) on the device.
inline RunResult solve_poisson(const Device &dev, const RunConfig &config)
{
   validate(config);
   const auto space =
      std::make_shared<const FeSpace>(build_mesh(config), FeCollection(FeFamily::H1, config.order));
   return solve_on_space(dev, space, manufactured_solution(config.solution), config);
}

/// convergence_study (driver.cpp:196-228): uniform forest refinement on the
/// host, every level solved on the device.
inline RunResult convergence_study(const Device &dev, const RunConfig &config)
{
   validate(config);
   if (config.convergence_levels < 1)
      throw std::invalid_argument("driver: study needs at least one level");
   const ManufacturedSolution sol = manufactured_solution(config.solution);
   const auto forest = std::make_shared<NcForest>(build_mesh(config));
   RunResult out;
   out.forest = forest;
   for (int level = 0;; level++) {
      const auto space = std::make_shared<const FeSpace>(*forest, FeCollection(FeFamily::H1, config.order));
      RunResult solve = solve_on_space(dev, space, sol, config);
      out.rows.push_back(solve.rows[0]);
      out.converged = out.converged && solve.converged;
      out.space = solve.space;
      out.u = std::move(solve.u);
      if (level == config.convergence_levels - 1 || !out.converged) break;
      std::vector<std::pair<int, SplitKind>> marks;
      marks.reserve(forest->n_leaves());
      for (int leaf = 0; leaf < forest->n_leaves(); leaf++) marks.emplace_back(leaf, SplitKind::Iso);
      forest->refine(marks);
   }
   fill_orders(out.rows);
   return out;
}

/// amr_loop (driver.cpp:230-258): solve on the device, estimate / mark /
/// refine on the host with the reference's element_errors and
/// select_refinements.
inline RunResult amr_loop(const Device &dev, const RunConfig &config)
{
   validate(config);
   const ManufacturedSolution sol = manufactured_solution(config.solution);
   const auto forest = std::make_shared<NcForest>(build_mesh(config), config.amr.irregularity_limit);
   RunResult out;
   out.forest = forest;
   for (int iter = 0;; iter++) {
      const auto space = std::make_shared<const FeSpace>(*forest, FeCollection(FeFamily::H1, config.order));
      RunResult solve = solve_on_space(dev, space, sol, config);
      out.rows.push_back(solve.rows[0]);
      out.converged = out.converged && solve.converged;
      out.space = solve.space;
      out.u = std::move(solve.u);
      if (iter == config.amr.iters || !out.converged) break;
      const ElementErrors err = element_errors(*out.u, sol, config.amr.anisotropic);
      const std::vector<std::pair<int, SplitKind>> marks =
         select_refinements(err.l2, err.directional, config.amr.theta);
      if (marks.empty()) break;
      forest->refine(marks);
   }
   fill_orders(out.rows);
   return out;
}

} // namespace b200
} // namespace tensorfem
