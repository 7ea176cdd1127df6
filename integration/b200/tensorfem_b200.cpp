// tensorfem_b200.cpp -- implementation of the reference-side binding
// (tensorfem_b200.hpp, tensorfem_b200_memory.hpp) over the C ABI of
// libtfem_cuda.so.  Compiled into the reference library by
// integration/Makefile together with the patched forms / solvers / vector.
#include "tensorfem_b200.hpp"

#include "tensorfem/mesh.hpp"

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>

namespace tensorfem {
namespace b200 {

void check(int rc)
{
   if (rc == TFEM_OK) return;
   const std::string msg = tfem_last_error();
   switch (rc) {
   case TFEM_INVALID_ARGUMENT: throw std::invalid_argument(msg);
   case TFEM_LOGIC_ERROR: throw std::logic_error(msg);
   default: throw std::runtime_error(msg);
   }
}

// --------------------------------------------------------------- context
namespace {
struct ProcessContext {
   std::once_flag once;
   tfem_ctx *ctx = nullptr;
   int device = 0;
   int numerics = TFEM_NUMERICS_FMA;
};
ProcessContext &pc()
{
   static ProcessContext *p = new ProcessContext; // lives to process exit
   return *p;
}
} // namespace

tfem_ctx *context()
{
   ProcessContext &p = pc();
   std::call_once(p.once, [&] {
      check(tfem_ctx_create(p.device, &p.ctx));
      check(tfem_ctx_set_numerics(p.ctx, p.numerics));
   });
   return p.ctx;
}

void set_device(int device)
{
   if (pc().ctx) throw std::logic_error("b200::set_device: the context already exists");
   pc().device = device;
}

void set_numerics(int mode)
{
   pc().numerics = mode;
   if (pc().ctx) check(tfem_ctx_set_numerics(pc().ctx, mode));
}

// ---------------------------------------------------------------- memory
void *host_alloc_pinned(std::size_t bytes)
{
   void *p = nullptr;
   if (tfem_host_alloc(bytes, &p) != TFEM_OK) throw std::bad_alloc();
   return p;
}

void host_free_pinned(void *p) noexcept { tfem_host_free(p); }

void Mirror::ensure(std::size_t n) const
{
   if (d_ && n_ == n) return;
   const_cast<Mirror *>(this)->release();
   void *p = nullptr;
   check(tfem_mem_alloc(context(), sizeof(double) * (n ? n : 1), &p));
   d_ = static_cast<double *>(p);
   n_ = n;
}

void Mirror::release() noexcept
{
   if (d_) tfem_mem_free(context(), d_);
   d_ = nullptr;
   n_ = 0;
}

void Mirror::download(double *host, std::size_t n) const
{
   if (n) check(tfem_copy(context(), host, d_, sizeof(double) * n));
   host_valid_ = true;
}

const double *Mirror::device_read(const double *host, std::size_t n) const
{
   ensure(n);
   if (!dev_valid_) {
      if (n) check(tfem_copy(context(), d_, host, sizeof(double) * n));
      dev_valid_ = true;
   }
   return d_;
}

double *Mirror::device_write(std::size_t n)
{
   ensure(n);
   dev_valid_ = true;
   host_valid_ = false;
   return d_;
}

double *Mirror::device_readwrite(const double *host, std::size_t n)
{
   device_read(host, n);
   host_valid_ = false;
   return d_;
}

void Mirror::init(double *host, std::size_t n, double value)
{
   if (value != 0.0 || n * sizeof(double) < kPinnedBytes) {
      std::fill(host, host + n, value);
      return;
   }
   double *d = device_write(n);
   tfem_vec *v = nullptr;
   check(tfem_vec_wrap(context(), d, static_cast<int64_t>(n), &v));
   const int rc = tfem_vec_fill(v, 0.0);
   tfem_vec_destroy(v);
   check(rc);
}

Mirror::Mirror(const Mirror &o) { *this = o; }

Mirror &Mirror::operator=(const Mirror &o)
{
   if (this == &o) return *this;
   if (!o.host_valid_) {
      // the device holds the only current copy: copy it device to device
      ensure(o.n_);
      if (o.n_) check(tfem_copy(context(), d_, o.d_, sizeof(double) * o.n_));
      dev_valid_ = true;
      host_valid_ = false;
   } else {
      // the host copy (copied by Vector itself) is current; ours re-uploads
      host_valid_ = true;
      dev_valid_ = false;
   }
   return *this;
}

Mirror::Mirror(Mirror &&o) noexcept
   : d_(o.d_), n_(o.n_), host_valid_(o.host_valid_), dev_valid_(o.dev_valid_)
{
   o.d_ = nullptr;
   o.n_ = 0;
   o.host_valid_ = true;
   o.dev_valid_ = false;
}

Mirror &Mirror::operator=(Mirror &&o) noexcept
{
   if (this == &o) return *this;
   release();
   d_ = o.d_;
   n_ = o.n_;
   host_valid_ = o.host_valid_;
   dev_valid_ = o.dev_valid_;
   o.d_ = nullptr;
   o.n_ = 0;
   o.host_valid_ = true;
   o.dev_valid_ = false;
   return *this;
}

Mirror::~Mirror() { release(); }

namespace {

// Non-owning tfem_vec view of a Vector's device half.
class Wrap {
public:
   Wrap(const double *p, std::int64_t n)
   {
      check(tfem_vec_wrap(context(), const_cast<double *>(p), n, &v_));
   }
   ~Wrap() { tfem_vec_destroy(v_); }
   Wrap(const Wrap &) = delete;
   Wrap &operator=(const Wrap &) = delete;
   operator tfem_vec *() const { return v_; }

private:
   tfem_vec *v_ = nullptr;
};

} // namespace

// ----------------------------------------------------------------- space
struct SpaceHandle {
   tfem_restriction *r = nullptr;
   tfem_geometry *g = nullptr;
   tfem_prolongation *P = nullptr;
   bool cartesian = false;
   int order = 1, n_dofs = 0, n_true = 0, n_elem = 0;
   // identity of the FeSpace this was built from (the registry's check
   // against a destroyed space whose address was reused)
   std::vector<int> first_dofs, last_dofs;
   std::vector<double> probe;
   ~SpaceHandle()
   {
      tfem_prolongation_destroy(P);
      tfem_geometry_destroy(g);
      tfem_restriction_destroy(r);
   }
};

bool is_cartesian(const SpaceHandle &s) { return s.cartesian; }

namespace {

// Mesh::element_control_points (mesh.cpp:228-241, private there): nodal
// geometry in its layout's order, else the corners in lattice order
// v0, v1, v3, v2.
std::vector<Vec2> control_points(const Mesh &m, int k)
{
   if (const NodalField *nodes = m.nodes()) {
      const auto d = nodes->layout.dofs(k);
      std::vector<Vec2> c(d.size());
      for (size_t i = 0; i < d.size(); i++) c[i] = nodes->coords[d[i]];
      return c;
   }
   const auto &v = m.element(k).v;
   return {m.vertex(v[0]), m.vertex(v[1]), m.vertex(v[3]), m.vertex(v[2])};
}

std::vector<double> probe_of(const FeSpace &space)
{
   const Mesh &m = space.mesh();
   std::vector<double> v;
   for (int k : {0, m.n_elements() - 1}) {
      for (const Vec2 &c : control_points(m, k)) {
         v.push_back(c.x);
         v.push_back(c.y);
      }
   }
   v.push_back(m.geometry_order());
   v.push_back(space.conforming() ? 1.0 : 0.0);
   v.push_back(static_cast<double>(space.collection().node_kind()));
   return v;
}

bool same_space(const SpaceHandle &h, const FeSpace &space)
{
   const int ne = space.mesh().n_elements();
   if (h.order != space.collection().order() || h.n_dofs != space.n_dofs() ||
       h.n_true != space.n_true_dofs() || h.n_elem != ne)
      return false;
   const auto f = space.element_dofs(0), l = space.element_dofs(ne - 1);
   return std::equal(f.begin(), f.end(), h.first_dofs.begin(), h.first_dofs.end()) &&
          std::equal(l.begin(), l.end(), h.last_dofs.begin(), h.last_dofs.end()) &&
          probe_of(space) == h.probe;
}

// make_cartesian(nx, ny, w, h) exactly (mesh.cpp:283-321): lattice vertices
// i fastest at (w i / nx, h j / ny), elements (i, j) i fastest with vertices
// (i,j) (i+1,j) (i+1,j+1) (i,j+1), straight geometry.
bool cartesian_of(const FeSpace &space, int &nx, int &ny, double &w, double &h)
{
   const Mesh &m = space.mesh();
   if (m.nodes() || !space.conforming() || space.collection().family() != FeFamily::H1)
      return false;
   const int nv = m.n_vertices();
   int c = 0;
   while (c < nv && m.vertex(c).y == 0.0) c++;
   nx = c - 1;
   if (nx < 1 || nv % (nx + 1) != 0) return false;
   ny = nv / (nx + 1) - 1;
   if (ny < 1 || static_cast<long>(m.n_elements()) != static_cast<long>(nx) * ny) return false;
   w = m.vertex(nx).x;
   h = m.vertex(nv - 1).y;
   for (int j = 0; j <= ny; j++)
      for (int i = 0; i <= nx; i++) {
         const Vec2 &v = m.vertex(i + j * (nx + 1));
         if (v.x != w * i / nx || v.y != h * j / ny) return false;
      }
   auto vid = [nx](int i, int j) { return i + j * (nx + 1); };
   for (int j = 0; j < ny; j++)
      for (int i = 0; i < nx; i++) {
         const auto &v = m.element(i + j * nx).v;
         if (v[0] != vid(i, j) || v[1] != vid(i + 1, j) || v[2] != vid(i + 1, j + 1) ||
             v[3] != vid(i, j + 1))
            return false;
      }
   return true;
}

std::shared_ptr<SpaceHandle> build_space(const FeSpace &space)
{
   tfem_ctx *ctx = context();
   auto h = std::make_shared<SpaceHandle>();
   const Mesh &mesh = space.mesh();
   const int ne = mesh.n_elements();
   const int p = space.collection().order();
   const int nd = (p + 1) * (p + 1);
   h->order = p;
   h->n_dofs = space.n_dofs();
   h->n_true = space.n_true_dofs();
   h->n_elem = ne;
   {
      const auto f = space.element_dofs(0), l = space.element_dofs(ne - 1);
      h->first_dofs.assign(f.begin(), f.end());
      h->last_dofs.assign(l.begin(), l.end());
      h->probe = probe_of(space);
   }
   std::vector<int32_t> dofs(static_cast<size_t>(ne) * nd);
   for (int k = 0; k < ne; k++) {
      const auto d = space.element_dofs(k);
      std::copy(d.begin(), d.end(), dofs.begin() + static_cast<size_t>(k) * nd);
   }
   int nx = 0, ny = 0;
   double w = 0, hh = 0;
   if (p >= 1 && cartesian_of(space, nx, ny, w, hh)) {
      // the device generator reproduces build_h1_layout on make_cartesian
      // (mesh.cpp:65-115); confirm it on this space before relying on it
      const int n[2] = {nx, ny};
      const double ext[2] = {w, hh};
      tfem_restriction *r = nullptr;
      check(tfem_restriction_cartesian(ctx, 2, n, p, &r));
      std::vector<int32_t> gen(dofs.size());
      const int rc = tfem_restriction_elem_dofs(r, gen.data());
      if (rc == TFEM_OK && gen == dofs && tfem_restriction_n_dofs(r) == space.n_dofs()) {
         h->r = r;
         check(tfem_geometry_cartesian(ctx, 2, n, ext, &h->g));
         h->cartesian = true;
         return h;
      }
      tfem_restriction_destroy(r);
   }
   check(tfem_restriction_create(ctx, 2, p, ne, space.n_dofs(), dofs.data(), &h->r));
   // control points in lattice order (mesh.cpp:228-241)
   const int m = mesh.geometry_order();
   const int nc = (m + 1) * (m + 1);
   std::vector<double> ctrl(static_cast<size_t>(ne) * nc * 2);
   for (int k = 0; k < ne; k++) {
      const std::vector<Vec2> c = control_points(mesh, k);
      for (int i = 0; i < nc; i++) {
         ctrl[(static_cast<size_t>(k) * nc + i) * 2] = c[i].x;
         ctrl[(static_cast<size_t>(k) * nc + i) * 2 + 1] = c[i].y;
      }
   }
   check(tfem_geometry_create(ctx, 2, m, ne, ctrl.data(), &h->g));
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
      check(tfem_prolongation_create(ctx, P.rows(), P.cols(), rp.data(), cols.data(),
                                     vals.data(), tix.data(), &h->P));
   }
   return h;
}

} // namespace

std::shared_ptr<SpaceHandle> device_space(const FeSpace &space)
{
   static std::mutex mu;
   static std::map<const FeSpace *, std::weak_ptr<SpaceHandle>> registry;
   std::lock_guard<std::mutex> lock(mu);
   for (auto it = registry.begin(); it != registry.end();)
      it = it->second.expired() ? registry.erase(it) : std::next(it);
   auto it = registry.find(&space);
   if (it != registry.end()) {
      std::shared_ptr<SpaceHandle> h = it->second.lock();
      if (h && same_space(*h, space)) return h;
   }
   std::shared_ptr<SpaceHandle> h = build_space(space);
   registry[&space] = h;
   return h;
}

// -------------------------------------------------------------------- PA
PaHandle::~PaHandle() { tfem_pa_destroy(pa); }

std::shared_ptr<PaHandle> pa_setup(const FeSpace &space, IntegratorKind kind,
                                   const Coefficient &coeff, const EvalMatrices &em)
{
   tfem_ctx *ctx = context();
   auto h = std::make_shared<PaHandle>();
   h->space = device_space(space);
   const int p = space.collection().order();
   const int nq = em.B1d.rows(); // order + 2 (forms.cpp:211)
   const int ne = space.mesh().n_elements();
   // the Coefficient is a host std::function: evaluate it at the device's
   // physical points (ElementTransformation::point, reference point order)
   std::vector<double> xy(static_cast<size_t>(ne) * nq * nq * 2);
   check(tfem_geometry_points(ctx, h->space->g, nq, TFEM_GAUSS_LEGENDRE, xy.data()));
   std::vector<double> c(static_cast<size_t>(ne) * nq * nq);
   for (size_t i = 0; i < c.size(); i++) c[i] = coeff(Vec2{xy[2 * i], xy[2 * i + 1]});
   check(tfem_pa_setup(ctx, kind == IntegratorKind::Mass ? TFEM_MASS : TFEM_DIFFUSION,
                       h->space->g, p, nq, TFEM_GAUSS_LEGENDRE, c.data(), 0.0, &h->pa, nullptr));
   if (space.collection().node_kind() != NodeKind::GaussLobatto)
      check(tfem_pa_set_basis(h->pa, em.B1d.data(), em.G1d.data()));
   return h;
}

void pa_qdata(const PaHandle &h, std::vector<double> &d)
{
   static std::mutex mu;
   std::lock_guard<std::mutex> lock(mu);
   if (!d.empty()) return;
   d.resize(static_cast<size_t>(tfem_pa_stored_reals(h.pa)));
   check(tfem_pa_qdata(h.pa, d.data()));
}

void pa_apply_local(const PaHandle &h, const FeSpace &space, const Vector &x, Vector &y)
{
   if (&x == &y) { // y += A y: the kernels need distinct buffers
      const Vector xc = x;
      pa_apply_local(h, space, xc, y);
      return;
   }
   (void)space; // check_space_match ran in forms.cpp
   tfem_ctx *ctx = context();
   const Wrap wx(x.device_read(), x.size());
   const Wrap wy(y.device_readwrite(), y.size());
   check(tfem_pa_apply_local(ctx, h.pa, h.space->r, wx, wy));
   count_multiplies(tfem_pa_multiply_count(h.pa));
}

Vector pa_diagonal(const PaHandle &h, const FeSpace &space)
{
   tfem_ctx *ctx = context();
   Vector diag(space.n_true_dofs());
   const Wrap wd(diag.device_write(), diag.size());
   check(tfem_vec_fill(wd, 0.0));
   if (h.space->P) check(tfem_pa_diagonal_p(ctx, h.pa, h.space->r, h.space->P, wd));
   else check(tfem_pa_diagonal(ctx, h.pa, h.space->r, wd));
   return diag;
}

// -------------------------------------------------------------- operator
DeviceOperator::DeviceOperator(std::shared_ptr<SpaceHandle> space,
                               std::vector<std::shared_ptr<PaHandle>> pa,
                               const std::vector<int> &essential)
   : space_(std::move(space)), pa_(std::move(pa))
{
   std::vector<tfem_pa *> h;
   for (const auto &x : pa_) {
      h.push_back(x->pa);
      mults_ += tfem_pa_multiply_count(x->pa);
   }
   check(tfem_operator_create_p(context(), static_cast<int>(h.size()), h.data(), space_->r,
                                space_->P, static_cast<int64_t>(essential.size()),
                                essential.empty() ? nullptr : essential.data(), &op_));
   n_ = static_cast<int>(tfem_operator_size(op_));
}

DeviceOperator::~DeviceOperator() { tfem_operator_destroy(op_); }

void DeviceOperator::mult(const Vector &x, Vector &y) const
{
   if (x.size() != n_ || y.size() != n_)
      throw std::invalid_argument("BilinearForm::mult_true: size mismatch");
   if (&x == &y) {
      const Vector xc = x;
      mult(xc, y);
      return;
   }
   const Wrap wx(x.device_read(), n_);
   const Wrap wy(y.device_write(), n_);
   check(tfem_operator_mult(context(), op_, wx, wy));
   count_multiplies(mults_);
}

Vector DeviceOperator::diagonal() const
{
   Vector d(n_);
   const Wrap wd(d.device_write(), n_);
   check(tfem_operator_diagonal(context(), op_, wd));
   return d;
}

namespace {
// A form without integrators: A = 0 (the reference's ConstrainedOperator
// then copies x on the essential DOFs).  No device work to do.
class ZeroConstrained : public LinearOperator {
public:
   ZeroConstrained(int n, std::vector<int> ess) : n_(n), ess_(std::move(ess)) {}
   int rows() const override { return n_; }
   int cols() const override { return n_; }
   void mult(const Vector &x, Vector &y) const override
   {
      Vector out(n_);
      for (int e : ess_) out[e] = x[e];
      y = out;
   }

private:
   int n_;
   std::vector<int> ess_;
};
} // namespace

std::shared_ptr<FormHandle> form_operator(const FeSpace &space, const std::vector<PaData> &pa)
{
   auto f = std::make_shared<FormHandle>();
   f->space = device_space(space);
   for (const PaData &d : pa) f->pa.push_back(d.device_handle());
   if (!f->pa.empty()) f->op = std::make_unique<DeviceOperator>(f->space, f->pa, std::vector<int>{});
   return f;
}

void form_mult(const FormHandle &f, const Vector &x, Vector &y)
{
   if (f.op) {
      f.op->mult(x, y);
      return;
   }
   y.set_zero(); // no integrators: A = 0
}

Vector form_diagonal(const FormHandle &f)
{
   return f.op ? f.op->diagonal() : Vector(f.space->n_true);
}

std::unique_ptr<LinearOperator> constrained_operator(const FormHandle &f,
                                                     const std::vector<int> &essential)
{
   if (f.pa.empty())
      return std::make_unique<ZeroConstrained>(f.space->n_true, essential);
   return std::make_unique<DeviceOperator>(f.space, f.pa, essential);
}

// ------------------------------------------------------ RHS / projection
namespace {
bool device_h1(const FeSpace &space)
{
   return space.collection().family() == FeFamily::H1 &&
          space.collection().map_type() == MapType::Value && space.collection().order() <= 16;
}

std::vector<double> eval_at(const std::vector<double> &xy, const std::function<double(Vec2)> &f)
{
   std::vector<double> v(xy.size() / 2);
   for (size_t i = 0; i < v.size(); i++) v[i] = f(Vec2{xy[2 * i], xy[2 * i + 1]});
   return v;
}
} // namespace

bool linear_form(const FeSpace &space, const Coefficient &f, Vector &b)
{
   if (!device_h1(space)) return false;
   tfem_ctx *ctx = context();
   const auto h = device_space(space);
   const int p = space.collection().order(), nq = p + 2;
   std::vector<double> xy(static_cast<size_t>(h->n_elem) * nq * nq * 2);
   check(tfem_geometry_points(ctx, h->g, nq, TFEM_GAUSS_LEGENDRE, xy.data()));
   const std::vector<double> fv = eval_at(xy, f);
   const Wrap wb(b.device_write(), b.size());
   check(tfem_linear_form(ctx, h->g, h->r, p, fv.data(), wb));
   return true;
}

bool project(const FeSpace &space, const std::function<double(Vec2)> &f, Vector &values)
{
   if (!device_h1(space)) return false;
   tfem_ctx *ctx = context();
   const auto h = device_space(space);
   const int p = space.collection().order(), nd = p + 1;
   std::vector<double> xy(static_cast<size_t>(h->n_elem) * nd * nd * 2);
   check(tfem_geometry_node_points(ctx, h->g, p, xy.data()));
   const std::vector<double> fv = eval_at(xy, f);
   // GridFunction(space) starts at zero; DOFs no element touches keep it
   const Wrap wv(values.device_readwrite(), values.size());
   check(tfem_project(ctx, h->r, fv.data(), wv));
   return true;
}

bool l2_error(const FeSpace &space, const Vector &values, const std::function<double(Vec2)> &u,
              double &err)
{
   if (!device_h1(space)) return false;
   tfem_ctx *ctx = context();
   const auto h = device_space(space);
   const int p = space.collection().order(), nq = p + 3;
   std::vector<double> xy(static_cast<size_t>(h->n_elem) * nq * nq * 2);
   check(tfem_geometry_points(ctx, h->g, nq, TFEM_GAUSS_LEGENDRE, xy.data()));
   const std::vector<double> uv = eval_at(xy, u);
   const Wrap wx(values.device_read(), values.size());
   check(tfem_l2_error(ctx, h->g, h->r, p, wx, uv.data(), &err));
   return true;
}

// -------------------------------------------------------------------- CG
const DeviceOperator *device_operator(const LinearOperator &a)
{
   return dynamic_cast<const DeviceOperator *>(&a);
}

namespace {
void iterate_trampoline(int it, const double *x, int64_t n, void *user)
{
   const auto &f = *static_cast<const std::function<void(int, const Vector &)> *>(user);
   Vector xv(static_cast<int>(n));
   std::memcpy(xv.data(), x, sizeof(double) * static_cast<size_t>(n));
   f(it, xv);
}
} // namespace

CgResult cg_solve(const DeviceOperator &a, const Vector &b, double rel_tol, int max_iters,
                  const Vector *jacobi_diag,
                  const std::function<void(int, const Vector &)> &on_iterate)
{
   const int n = b.size();
   if (a.rows() != n || a.cols() != n)
      throw std::invalid_argument("cg_solve: operator/vector size mismatch");
   if (jacobi_diag && jacobi_diag->size() != n)
      throw std::invalid_argument("cg_solve: preconditioner size mismatch");
   CgResult res;
   res.x = Vector(n);
   const Wrap wb(b.device_read(), n);
   std::unique_ptr<Wrap> wd;
   if (jacobi_diag) wd = std::make_unique<Wrap>(jacobi_diag->device_read(), n);
   const Wrap wx(res.x.device_write(), n);
   tfem_cg_result r{};
   check(tfem_cg_solve(context(), a.get(), wb, rel_tol, max_iters, wd ? static_cast<tfem_vec *>(*wd) : nullptr, wx, &r,
                       on_iterate ? iterate_trampoline : nullptr,
                       const_cast<void *>(static_cast<const void *>(&on_iterate))));
   res.iterations = r.iterations;
   res.converged = r.converged != 0;
   // one operator application per iteration run (solvers.cpp:60-66)
   count_multiplies(a.multiplies() * static_cast<std::uint64_t>(r.iterations > 0 ? r.iterations : 0));
   return res;
}

} // namespace b200
} // namespace tensorfem
