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
#pragma once

#include "tensorfem/forms.hpp"
#include "tfem_cuda.h"

#include <memory>
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

} // namespace b200
} // namespace tensorfem
