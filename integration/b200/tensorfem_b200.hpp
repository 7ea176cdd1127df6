// tensorfem_b200.hpp -- the reference-side binding of libtfem_cuda.so.
//
// Compiled into the reference library when it is built with -DTENSORFEM_B200
// (integration/Makefile applies integration/patch/tensorfem_b200.patch to a
// build-time copy of forms.hpp / forms.cpp / solvers.cpp / vector.hpp /
// vector.cpp).  The patched call sites route the PA / CG hot path through the
// C ABI (include/tfem_cuda.h); every other line of the reference -- mesh,
// forest, FeSpace, LinearForm, full assembly, driver, I/O -- is unchanged and
// runs as before.
//
//   reference call (file:line, /root/reference/proj)    routed to
//   pa_setup                  forms.cpp:201-229          b200::pa_setup -> tfem_pa_setup
//   PaData::d                 forms.cpp:194-199          tfem_pa_qdata (lazy, once)
//   pa_apply_local            forms.cpp:231-296          tfem_pa_apply_local
//   pa_diagonal               forms.cpp:311-382          tfem_pa_diagonal(_p)
//   BilinearForm::assemble    forms.cpp:460-475          + tfem_operator_create_p
//   BilinearForm::mult_true   forms.cpp:527-543          tfem_operator_mult
//   BilinearForm::diagonal_true forms.cpp:545-557        tfem_operator_diagonal
//   ConstrainedOperator       forms.cpp:164-190, 635-638 DeviceOperator (ess)
//   cg_solve                  solvers.cpp:11-97          tfem_cg_solve (device loop)
//   Vector                    vector.hpp:14-48           + device mirror
//                                                        (tensorfem_b200_memory.hpp)
//
// Errors come back as the reference's exception classes with the reference's
// messages (tfem_last_error).  The instrumentation contracts hold: mult_true
// and the operators count multiplies exactly as the reference's tensor
// kernels would (tfem_pa_multiply_count), stored_reals = E q^2 nc.
#pragma once

#include "tensorfem/forms.hpp"
#include "tensorfem/solvers.hpp"
#include "tfem_cuda.h"

#include <functional>
#include <memory>
#include <vector>

namespace tensorfem {
namespace b200 {

/// Status code -> the reference's exception class.
void check(int rc);

/// Select the device / the numerics of the process context before its first
/// use.  Numerics: TFEM_NUMERICS_FMA (default; <= 1e-15 relative of the
/// reference) or TFEM_NUMERICS_REFERENCE (the reference's operation order:
/// bit-identical 2D operator, diagonal and point factors).
void set_device(int device);
void set_numerics(int mode);

/// G (element restriction), the element geometry and, on non-conforming
/// spaces, P of one FeSpace on the device.  make_cartesian meshes use the
/// device-generated Cartesian restriction (warp-patch element order: shared
/// DOFs summed in-warp) after checking that the mesh is exactly the one
/// make_cartesian builds; any other mesh uploads its element map.
struct SpaceHandle;
std::shared_ptr<SpaceHandle> device_space(const FeSpace &space);
/// True when `space` runs on the Cartesian restriction (diagnostics, tests).
bool is_cartesian(const SpaceHandle &s);

/// Device point factors of one integrator (PaData's device half).
struct PaHandle {
   std::shared_ptr<SpaceHandle> space;
   tfem_pa *pa = nullptr;
   ~PaHandle();
};

std::shared_ptr<PaHandle> pa_setup(const FeSpace &space, IntegratorKind kind,
                                   const Coefficient &coeff, const EvalMatrices &em);
/// PaData::d's host copy in the reference layout [e][q][c].
void pa_qdata(const PaHandle &h, std::vector<double> &d);
void pa_apply_local(const PaHandle &h, const FeSpace &space, const Vector &x, Vector &y);
Vector pa_diagonal(const PaHandle &h, const FeSpace &space);

/// mult_true / ConstrainedOperator on the device: the LinearOperator seam
/// cg_solve drives (solvers.hpp:16-23).
class DeviceOperator : public LinearOperator {
public:
   DeviceOperator(std::shared_ptr<SpaceHandle> space,
                  std::vector<std::shared_ptr<PaHandle>> pa,
                  const std::vector<int> &essential);
   ~DeviceOperator() override;
   DeviceOperator(const DeviceOperator &) = delete;
   DeviceOperator &operator=(const DeviceOperator &) = delete;
   int rows() const override { return n_; }
   int cols() const override { return n_; }
   void mult(const Vector &x, Vector &y) const override;
   Vector diagonal() const;
   tfem_operator *get() const { return op_; }
   /// Multiplies one application counts (tensor_kernels.cpp:10-16).
   std::uint64_t multiplies() const { return mults_; }

private:
   std::shared_ptr<SpaceHandle> space_;
   std::vector<std::shared_ptr<PaHandle>> pa_;
   tfem_operator *op_ = nullptr;
   int n_ = 0;
   std::uint64_t mults_ = 0;
};

/// The device half of a Partial BilinearForm: its integrators' PaHandles and
/// the unconstrained operator of mult_true.
struct FormHandle {
   std::unique_ptr<DeviceOperator> op;
   std::shared_ptr<SpaceHandle> space;
   std::vector<std::shared_ptr<PaHandle>> pa;
};
std::shared_ptr<FormHandle> form_operator(const FeSpace &space,
                                          const std::vector<PaData> &pa);
/// BilinearForm::mult_true / diagonal_true of a Partial form.
void form_mult(const FormHandle &f, const Vector &x, Vector &y);
Vector form_diagonal(const FormHandle &f);
std::unique_ptr<LinearOperator> constrained_operator(const FormHandle &f,
                                                     const std::vector<int> &essential);

/// RHS and post-processing on the device for H1 spaces;
/// each returns false (the reference's host code then runs) for spaces the
/// device tables do not cover (L2 families, orders > 16).
///   LinearForm (forms.cpp:400-431): b = G^T B^T (w detJ f)
///   project_coefficient (fespace.cpp:334-356): nodal values, last element wins
///   compute_l2_error (fespace.cpp:358-394): q = p+3 Gauss, the host's sequential sum
bool linear_form(const FeSpace &space, const Coefficient &f, Vector &b);
bool project(const FeSpace &space, const std::function<double(Vec2)> &f, Vector &values);
bool l2_error(const FeSpace &space, const Vector &values, const std::function<double(Vec2)> &u,
              double &err);

/// cg_solve with the whole loop on the device; only a 4-byte state word
/// crosses per batch of iterations (plus x per iteration when on_iterate is
/// set, as the callback needs it on the host).
const DeviceOperator *device_operator(const LinearOperator &a);
CgResult cg_solve(const DeviceOperator &a, const Vector &b, double rel_tol, int max_iters,
                  const Vector *jacobi_diag,
                  const std::function<void(int, const Vector &)> &on_iterate);

} // namespace b200
} // namespace tensorfem
