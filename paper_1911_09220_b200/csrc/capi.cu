// The C ABI of libtfem_cuda.so (include/tfem_cuda.h).  Every entry point runs
// its body under guard(): library exceptions become the status code of the
// reference's exception class with the message in tfem_last_error().
#include "common.cuh"

#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <set>
#include <string>

namespace tfem {
tfem_restriction *restriction_cartesian(tfem_ctx *ctx, int dim, const int *n, int p);
tfem_restriction *restriction_create(tfem_ctx *ctx, int dim, int p, int64_t ne, int64_t ndofs,
                                     const int32_t *elem_dofs);
void restriction_destroy(tfem_restriction *r);
void restriction_elem_dofs(const tfem_restriction *r, int32_t *host);
int64_t restriction_boundary_dofs(const tfem_restriction *r, int32_t *host);
void restriction_mult(tfem_ctx *ctx, const tfem_restriction *r, const double *l, double *e);
void vec_axpy(tfem_ctx *ctx, double a, const double *x, double *y, int64_t n);
void operator_set_ess(tfem_ctx *ctx, tfem_operator *op, int64_t n_ess, const int32_t *ess);
void operator_set_comm(tfem_ctx *ctx, tfem_operator *op, const tfem_comm &comm,
                       const tfem_halo &halo, int64_t n_not_owned, const int32_t *not_owned);
tfem_operator *operator_csr(tfem_ctx *ctx, int64_t n, const int32_t *rowptr, const int32_t *cols,
                            const double *vals);
void operator_release(tfem_operator *op);
tfem_prolongation *prolongation_create(tfem_ctx *ctx, int64_t n_local, int64_t n_true,
                                       const int32_t *rowptr, const int32_t *cols,
                                       const double *vals, const int32_t *true_index);
void prolongation_destroy(tfem_prolongation *P);
void operator_diagonal(tfem_ctx *ctx, const tfem_operator *op, double *diag);
void operator_set_nccl(tfem_ctx *ctx, tfem_operator *op, tfem_nccl *comm, int n_peers,
                       const int *peer, const int64_t *n_send, const int32_t *const *send_idx,
                       const int64_t *n_recv, const int32_t *const *recv_idx,
                       int64_t n_not_owned, const int32_t *not_owned);
} // namespace tfem

using namespace tfem;

namespace {

thread_local std::string g_last_error;

template <typename F>
int guard(F &&f)
{
   try {
      f();
      return TFEM_OK;
   } catch (const Error &e) {
      g_last_error = e.what();
      if (e.code == TFEM_CUDA_ERROR) (void)cudaGetLastError(); // don't leak into later calls
      return e.code;
   } catch (const std::bad_alloc &) {
      g_last_error = "out of host memory";
      return TFEM_RUNTIME_ERROR;
   } catch (const std::exception &e) {
      g_last_error = e.what();
      return TFEM_RUNTIME_ERROR;
   }
}

void need(const void *p, const char *what)
{
   if (!p) invalid(std::string(what) + ": null argument");
}

// Every entry point runs on its context's device, whatever the calling
// thread's current device is (one thread may drive several contexts).
void bind(const tfem_ctx *ctx)
{
   int cur = -1;
   TFEM_CUDA(cudaGetDevice(&cur));
   if (cur != ctx->device) TFEM_CUDA(cudaSetDevice(ctx->device));
}

void need(const tfem_ctx *ctx, const char *what)
{
   if (!ctx) invalid(std::string(what) + ": null argument");
   bind(ctx);
}

// Objects created through a context carry it.
template <typename T>
void need_obj(const T *o, const char *what)
{
   if (!o) invalid(std::string(what) + ": null argument");
   bind(o->ctx);
}

void check_vec(const tfem_vec *v, int64_t n, const char *what)
{
   need_obj(v, what);
   if (v->n != n) invalid(std::string(what) + ": size mismatch");
}

} // namespace

namespace tfem {
void max_dynamic_smem(const void *kernel, size_t bytes)
{
   static std::mutex mu;
   static std::set<std::pair<const void *, int>> done;
   int dev = 0;
   TFEM_CUDA(cudaGetDevice(&dev));
   std::lock_guard<std::mutex> lock(mu);
   if (done.count({kernel, dev})) return;
   TFEM_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(bytes)));
   done.insert({kernel, dev});
}
} // namespace tfem

void tfem_ctx::ensure_partials(int64_t n)
{
   if (n <= red.cap) return;
   cudaFree(red.partials);
   TFEM_CUDA(cudaMalloc(&red.partials, sizeof(double) * n));
   red.cap = n;
}

namespace tfem {
namespace {
std::mutex &refs_mu()
{
   static std::mutex mu;
   return mu;
}
} // namespace

void ctx_retain(tfem_ctx *ctx)
{
   std::lock_guard<std::mutex> lock(refs_mu());
   ctx->refs++;
}

void ctx_release(tfem_ctx *ctx)
{
   {
      std::lock_guard<std::mutex> lock(refs_mu());
      if (--ctx->refs > 0) return;
   }
   int cur = -1;
   cudaGetDevice(&cur);
   if (cur != ctx->device) cudaSetDevice(ctx->device);
   cudaStreamSynchronize(ctx->stream);
   for (auto &d : ctx->dot_sinks) {
      cudaFree(d.second.partials);
      cudaFree(d.second.chunks);
      cudaFree(d.second.tickets);
   }
   for (double *b : ctx->stage) cudaFree(b);
   for (auto &f : ctx->pool_free) cudaFree(f.second);
   for (auto &l : ctx->pool_live) cudaFree(l.first);
   cudaFree(ctx->red.partials);
   cudaFree(ctx->scalars);
   cudaFreeHost(ctx->host_scalars);
   cudaStreamDestroy(ctx->stream);
   delete ctx;
}
} // namespace tfem

extern "C" {

const char *tfem_last_error(void) { return g_last_error.c_str(); }
const char *tfem_version(void) { return "tfem_cuda 0.1 (sm_100a)"; }

// ------------------------------------------------------------------ context
int tfem_ctx_create(int device, tfem_ctx **out)
{
   return guard([&] {
      need(out, "tfem_ctx_create");
      int count = 0;
      TFEM_CUDA(cudaGetDeviceCount(&count));
      if (device >= count) invalid("tfem_ctx_create: no such device");
      if (device >= 0) TFEM_CUDA(cudaSetDevice(device));
      auto *c = new tfem_ctx;
      TFEM_CUDA(cudaGetDevice(&c->device));
      TFEM_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, c->device));
      TFEM_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      TFEM_CUDA(cudaMalloc(&c->scalars, sizeof(double) * 16));
      TFEM_CUDA(cudaMallocHost(&c->host_scalars, sizeof(double) * 16));
      *out = c;
   });
}

// The handle goes; the context itself lives until its last object does.
int tfem_ctx_destroy(tfem_ctx *ctx)
{
   return guard([&] {
      if (!ctx) return;
      bind(ctx);
      TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
      ctx_release(ctx);
   });
}

int tfem_ctx_sync(tfem_ctx *ctx)
{
   return guard([&] {
      need(ctx, "tfem_ctx_sync");
      TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   });
}

void *tfem_ctx_stream(tfem_ctx *ctx) { return ctx ? static_cast<void *>(ctx->stream) : nullptr; }

int tfem_ctx_set_numerics(tfem_ctx *ctx, int mode)
{
   return guard([&] {
      need(ctx, "tfem_ctx_set_numerics");
      if (mode != TFEM_NUMERICS_REFERENCE && mode != TFEM_NUMERICS_FMA)
         invalid("tfem_ctx_set_numerics: unknown mode");
      ctx->numerics = mode;
   });
}

int64_t tfem_ctx_launch_count(const tfem_ctx *ctx) { return ctx ? ctx->launches : 0; }

int tfem_ctx_set_max_blocks(tfem_ctx *ctx, int max_blocks)
{
   return guard([&] {
      need(ctx, "tfem_ctx_set_max_blocks");
      if (max_blocks < 0) invalid("tfem_ctx_set_max_blocks: negative cap");
      ctx->max_blocks = max_blocks;
   });
}

// ------------------------------------------------------------------ memory
namespace {
// Pool granularity: 512 B below 1 MiB, 2 MiB above (a vector of a given
// length always maps to the same class, so solves reuse their blocks).
size_t pool_class(size_t bytes)
{
   constexpr size_t kSmall = 512, kLarge = size_t(2) << 20;
   if (bytes == 0) bytes = 1;
   return bytes < (size_t(1) << 20) ? (bytes + kSmall - 1) / kSmall * kSmall
                                     : (bytes + kLarge - 1) / kLarge * kLarge;
}

struct HostPool {
   std::mutex mu;
   std::multimap<size_t, void *> free;
   std::unordered_map<void *, std::pair<size_t, bool>> live; // class, pinned
};
HostPool &host_pool()
{
   static HostPool *p = new HostPool; // never destroyed: frees may come late
   return *p;
}
} // namespace

int tfem_mem_alloc(tfem_ctx *ctx, size_t bytes, void **out)
{
   return guard([&] {
      need(ctx, "tfem_mem_alloc");
      need(out, "tfem_mem_alloc");
      const size_t cls = pool_class(bytes);
      std::lock_guard<std::mutex> lock(ctx->pool_mu);
      void *p = nullptr;
      auto it = ctx->pool_free.find(cls);
      if (it != ctx->pool_free.end()) {
         p = it->second;
         ctx->pool_free.erase(it);
      } else {
         cudaError_t e = cudaMalloc(&p, cls);
         if (e != cudaSuccess) {
            // release the cache and retry once before failing
            (void)cudaGetLastError();
            TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
            for (auto &f : ctx->pool_free) cudaFree(f.second);
            ctx->pool_free.clear();
            TFEM_CUDA(cudaMalloc(&p, cls));
         }
      }
      ctx->pool_live[p] = cls;
      *out = p;
   });
}

int tfem_mem_free(tfem_ctx *ctx, void *p)
{
   return guard([&] {
      need(ctx, "tfem_mem_free");
      if (!p) return;
      std::lock_guard<std::mutex> lock(ctx->pool_mu);
      auto it = ctx->pool_live.find(p);
      if (it == ctx->pool_live.end()) invalid("tfem_mem_free: not a pool block of this context");
      ctx->pool_free.emplace(it->second, p);
      ctx->pool_live.erase(it);
   });
}

int tfem_mem_trim(tfem_ctx *ctx)
{
   return guard([&] {
      need(ctx, "tfem_mem_trim");
      std::lock_guard<std::mutex> lock(ctx->pool_mu);
      TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
      for (auto &f : ctx->pool_free) cudaFree(f.second);
      ctx->pool_free.clear();
   });
}

int tfem_host_alloc(size_t bytes, void **out)
{
   return guard([&] {
      need(out, "tfem_host_alloc");
      const size_t cls = pool_class(bytes);
      HostPool &hp = host_pool();
      std::lock_guard<std::mutex> lock(hp.mu);
      void *p = nullptr;
      bool pinned = true;
      auto it = hp.free.find(cls); // cached blocks are all pinned
      if (it != hp.free.end()) {
         p = it->second;
         hp.free.erase(it);
      } else if (cudaHostAlloc(&p, cls, cudaHostAllocPortable) != cudaSuccess) {
         (void)cudaGetLastError(); // no device: pageable memory still works
         p = std::malloc(cls);
         pinned = false;
         if (!p) throw std::bad_alloc();
      }
      hp.live[p] = {cls, pinned};
      *out = p;
   });
}

int tfem_host_free(void *p)
{
   return guard([&] {
      if (!p) return;
      HostPool &hp = host_pool();
      std::lock_guard<std::mutex> lock(hp.mu);
      auto it = hp.live.find(p);
      if (it == hp.live.end()) invalid("tfem_host_free: not a pool block");
      if (it->second.second) hp.free.emplace(it->second.first, p);
      else std::free(p);
      hp.live.erase(it);
   });
}

int tfem_copy(tfem_ctx *ctx, void *dst, const void *src, size_t bytes)
{
   return guard([&] {
      need(ctx, "tfem_copy");
      if (!bytes) return;
      need(dst, "tfem_copy");
      need(src, "tfem_copy");
      TFEM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream));
      TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   });
}

// ------------------------------------------------------------------ tables
int tfem_quadrature(int rule, int n, double *points, double *weights)
{
   return guard([&] {
      need(points, "tfem_quadrature");
      std::vector<double> w;
      const std::vector<double> x = gauss_points(rule, n, &w);
      std::memcpy(points, x.data(), sizeof(double) * n);
      if (weights) std::memcpy(weights, w.data(), sizeof(double) * n);
   });
}

int tfem_eval_matrices(int p, int node_kind, int nq, int rule, double *B, double *G)
{
   return guard([&] {
      need(B, "tfem_eval_matrices");
      need(G, "tfem_eval_matrices");
      if (nq < 1) invalid("tfem_eval_matrices: need nq >= 1");
      eval_matrices(p, node_kind, nq, rule, B, G);
   });
}

// ------------------------------------------------------------------ vectors
int tfem_vec_create(tfem_ctx *ctx, int64_t n, tfem_vec **out)
{
   return guard([&] {
      need(ctx, "tfem_vec_create");
      need(out, "tfem_vec_create");
      if (n < 0) invalid("tfem_vec_create: negative size");
      auto *v = new tfem_vec;
      v->ctx = ctx;
      v->n = n;
      cudaError_t e = cudaMalloc(&v->d, sizeof(double) * static_cast<size_t>(n > 0 ? n : 1));
      if (e != cudaSuccess) {
         delete v;
         cuda_check(e, "tfem_vec_create");
      }
      TFEM_CUDA(cudaMemsetAsync(v->d, 0, sizeof(double) * n, ctx->stream));
      TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
      *out = v;
      ctx_retain(ctx);
   });
}

int tfem_vec_wrap(tfem_ctx *ctx, double *device_ptr, int64_t n, tfem_vec **out)
{
   return guard([&] {
      need(ctx, "tfem_vec_wrap");
      need(out, "tfem_vec_wrap");
      auto *v = new tfem_vec;
      v->ctx = ctx;
      v->d = device_ptr;
      v->n = n;
      v->owns = false;
      *out = v;
      ctx_retain(ctx);
   });
}

int tfem_vec_destroy(tfem_vec *v)
{
   return guard([&] {
      if (!v) return;
      bind(v->ctx);
      tfem_ctx *ctx = v->ctx;
      if (v->owns) cudaFree(v->d);
      delete v;
      ctx_release(ctx);
   });
}

int64_t tfem_vec_size(const tfem_vec *v) { return v ? v->n : 0; }
double *tfem_vec_data(tfem_vec *v) { return v ? v->d : nullptr; }

int tfem_vec_upload(tfem_vec *v, const double *host, int64_t n)
{
   return guard([&] {
      check_vec(v, n, "tfem_vec_upload");
      TFEM_CUDA(cudaMemcpyAsync(v->d, host, sizeof(double) * n, cudaMemcpyHostToDevice,
                                v->ctx->stream));
      TFEM_CUDA(cudaStreamSynchronize(v->ctx->stream));
   });
}

int tfem_vec_download(const tfem_vec *v, double *host, int64_t n)
{
   return guard([&] {
      check_vec(v, n, "tfem_vec_download");
      TFEM_CUDA(cudaMemcpyAsync(host, v->d, sizeof(double) * n, cudaMemcpyDeviceToHost,
                                v->ctx->stream));
      TFEM_CUDA(cudaStreamSynchronize(v->ctx->stream));
   });
}

int tfem_vec_fill(tfem_vec *v, double value)
{
   return guard([&] {
      need_obj(v, "tfem_vec_fill");
      vec_fill(v->ctx, v->d, v->n, value);
      TFEM_CUDA(cudaStreamSynchronize(v->ctx->stream));
   });
}

int tfem_vec_dot(tfem_ctx *ctx, const tfem_vec *a, const tfem_vec *b, double *out)
{
   return guard([&] {
      need(ctx, "Vector::dot");
      need(a, "Vector::dot");
      check_vec(b, a->n, "Vector::dot");
      *out = vec_dot(ctx, a->d, b->d, a->n);
   });
}

int tfem_vec_axpy(tfem_ctx *ctx, double a, const tfem_vec *x, tfem_vec *y)
{
   return guard([&] {
      need(ctx, "Vector::axpy");
      need(x, "Vector::axpy");
      check_vec(y, x->n, "Vector::axpy");
      vec_axpy(ctx, a, x->d, y->d, x->n);
      TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   });
}

// ------------------------------------------------------------- restriction
int tfem_restriction_create(tfem_ctx *ctx, int dim, int p, int64_t n_elem, int64_t n_dofs,
                            const int32_t *elem_dofs, tfem_restriction **out)
{
   return guard([&] {
      need(ctx, "tfem_restriction_create");
      need(elem_dofs, "tfem_restriction_create");
      need(out, "tfem_restriction_create");
      *out = restriction_create(ctx, dim, p, n_elem, n_dofs, elem_dofs);
      ctx_retain(ctx);
   });
}

int tfem_restriction_cartesian(tfem_ctx *ctx, int dim, const int *n, int p,
                               tfem_restriction **out)
{
   return guard([&] {
      need(ctx, "tfem_restriction_cartesian");
      need(n, "tfem_restriction_cartesian");
      need(out, "tfem_restriction_cartesian");
      *out = restriction_cartesian(ctx, dim, n, p);
      ctx_retain(ctx);
   });
}

int tfem_restriction_destroy(tfem_restriction *r)
{
   return guard([&] {
      if (!r) return;
      bind(r->ctx);
      tfem_ctx *ctx = r->ctx;
      restriction_destroy(r);
      ctx_release(ctx);
   });
}

int64_t tfem_restriction_n_dofs(const tfem_restriction *r) { return r ? r->ndofs : 0; }
int64_t tfem_restriction_n_elem(const tfem_restriction *r) { return r ? r->ne : 0; }

int tfem_restriction_elem_dofs(const tfem_restriction *r, int32_t *host)
{
   return guard([&] {
      need_obj(r, "tfem_restriction_elem_dofs");
      need(host, "tfem_restriction_elem_dofs");
      restriction_elem_dofs(r, host);
   });
}

int tfem_restriction_boundary_dofs(const tfem_restriction *r, int32_t *host, int64_t *count)
{
   return guard([&] {
      need_obj(r, "tfem_restriction_boundary_dofs");
      need(count, "tfem_restriction_boundary_dofs");
      *count = restriction_boundary_dofs(r, host);
   });
}

int tfem_restriction_mult(tfem_ctx *ctx, const tfem_restriction *r, const tfem_vec *l,
                          tfem_vec *e)
{
   return guard([&] {
      need(ctx, "ElementRestriction::Mult");
      need(r, "ElementRestriction::Mult");
      check_vec(l, r->ndofs, "ElementRestriction::Mult");
      check_vec(e, r->ne * r->nd, "ElementRestriction::Mult");
      restriction_mult(ctx, r, l->d, e->d);
      TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   });
}

int tfem_restriction_mult_transpose(tfem_ctx *ctx, const tfem_restriction *r, const tfem_vec *e,
                                    tfem_vec *l)
{
   return guard([&] {
      need(ctx, "ElementRestriction::MultTranspose");
      need(r, "ElementRestriction::MultTranspose");
      check_vec(l, r->ndofs, "ElementRestriction::MultTranspose");
      check_vec(e, r->ne * r->nd, "ElementRestriction::MultTranspose");
      restriction_mult_transpose(ctx, r, e->d, l->d);
      TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   });
}

// ---------------------------------------------------------------- geometry
int tfem_geometry_create(tfem_ctx *ctx, int dim, int order, int64_t n_elem, const double *ctrl,
                         tfem_geometry **out)
{
   return guard([&] {
      need(ctx, "tfem_geometry_create");
      need(ctrl, "tfem_geometry_create");
      need(out, "tfem_geometry_create");
      if (dim != 2 && dim != 3) invalid("tfem_geometry_create: dim must be 2 or 3");
      if (order < 1) invalid("curve_mesh: order must be >= 1");
      if (n_elem < 1) invalid("tfem_geometry_create: empty mesh");
      auto *g = new tfem_geometry;
      g->ctx = ctx;
      g->dim = dim;
      g->order = order;
      g->ne = n_elem;
      int64_t nc = 1;
      for (int d = 0; d < dim; d++) nc *= order + 1;
      const size_t bytes = sizeof(double) * static_cast<size_t>(n_elem * nc * dim);
      TFEM_CUDA(cudaMalloc(&g->ctrl, bytes));
      h2d(ctx->stream, g->ctrl, ctrl, bytes);
      *out = g;
      ctx_retain(ctx);
   });
}

int tfem_geometry_cartesian_box(tfem_ctx *ctx, int dim, const int *n_local, const int *origin,
                                const int *n_global, const double *ext, tfem_geometry **out)
{
   return guard([&] {
      need(ctx, "tfem_geometry_cartesian");
      need(n_local, "tfem_geometry_cartesian");
      need(out, "tfem_geometry_cartesian");
      if (dim != 2 && dim != 3) invalid("tfem_geometry_cartesian: dim must be 2 or 3");
      auto g = std::make_unique<tfem_geometry>();
      g->ctx = ctx;
      g->dim = dim;
      g->order = 1;
      g->cartesian = true;
      g->ne = 1;
      for (int d = 0; d < dim; d++) {
         if (n_local[d] < 1) invalid("make_cartesian: need nx, ny >= 1");
         const double e = ext ? ext[d] : 1.0;
         if (!(e > 0.0)) invalid("make_cartesian: need positive extents");
         g->n[d] = n_local[d];
         g->origin[d] = origin ? origin[d] : 0;
         g->n_global[d] = n_global ? n_global[d] : n_local[d];
         if (g->origin[d] < 0 || g->origin[d] + g->n[d] > g->n_global[d])
            invalid("tfem_geometry_cartesian_box: block outside the global mesh");
         g->ext[d] = e;
         g->ne *= n_local[d];
      }
      *out = g.release();
      ctx_retain(ctx);
   });
}

int tfem_geometry_cartesian(tfem_ctx *ctx, int dim, const int *n, const double *ext,
                            tfem_geometry **out)
{
   return tfem_geometry_cartesian_box(ctx, dim, n, nullptr, nullptr, ext, out);
}

int tfem_geometry_destroy(tfem_geometry *g)
{
   return guard([&] {
      if (!g) return;
      bind(g->ctx);
      tfem_ctx *ctx = g->ctx;
      cudaFree(g->ctrl);
      delete g;
      ctx_release(ctx);
   });
}

int tfem_geometry_points(tfem_ctx *ctx, const tfem_geometry *g, int nq, int rule,
                         double *host_xyz)
{
   return guard([&] {
      need(ctx, "tfem_geometry_points");
      need(g, "tfem_geometry_points");
      need(host_xyz, "tfem_geometry_points");
      geometry_points(ctx, g, nq, rule, host_xyz);
   });
}

// ---------------------------------------------------------------------- PA
int tfem_pa_setup(tfem_ctx *ctx, int kind, const tfem_geometry *g, int p, int nq, int rule,
                  const double *coeff, double coeff_const, tfem_pa **out, int64_t *bad_elem)
{
   return guard([&] {
      need(ctx, "pa_setup");
      need(g, "pa_setup");
      need(out, "pa_setup");
      *out = pa_setup(ctx, kind, g, p, nq, rule, coeff, coeff_const, bad_elem);
      ctx_retain(ctx);
   });
}

int tfem_pa_destroy(tfem_pa *pa)
{
   return guard([&] {
      if (!pa) return;
      bind(pa->ctx);
      tfem_ctx *ctx = pa->ctx;
      cudaFree(pa->qdata);
      delete pa;
      ctx_release(ctx);
   });
}

int tfem_pa_info(const tfem_pa *pa, int *kind, int *dim, int *p, int *nq, int64_t *n_elem)
{
   return guard([&] {
      need(pa, "tfem_pa_info");
      if (kind) *kind = pa->kind;
      if (dim) *dim = pa->dim;
      if (p) *p = pa->p;
      if (nq) *nq = pa->nq;
      if (n_elem) *n_elem = pa->ne;
   });
}

int64_t tfem_pa_stored_reals(const tfem_pa *pa)
{
   return pa ? pa->ne * pa->nqd * pa->ncomp : 0;
}

uint64_t tfem_pa_multiply_count(const tfem_pa *pa)
{
   if (!pa) return 0;
   const uint64_t a = pa->p + 1, q = pa->nq, e = pa->ne;
   uint64_t per;
   if (pa->dim == 2)
      per = pa->kind == TFEM_MASS ? 2 * (q * a * a + q * q * a) + q * q
                                  : 4 * (q * a * a + q * q * a) + 4 * q * q;
   else
      per = pa->kind == TFEM_MASS
               ? 2 * (q * a * a * a + q * q * a * a + q * q * q * a) + q * q * q
               : 2 * (2 * q * a * a * a + 3 * q * q * a * a + 3 * q * q * q * a) + 9 * q * q * q;
   return per * e;
}

int tfem_pa_qdata(const tfem_pa *pa, double *host)
{
   return guard([&] {
      need_obj(pa, "PaData::d");
      need(host, "PaData::d");
      const size_t n = static_cast<size_t>(pa->ncomp) * pa->nqd * pa->ne_pad;
      std::vector<double> dev(n);
      d2h(pa->ctx->stream, dev.data(), pa->qdata, sizeof(double) * n);
      for (int64_t e = 0; e < pa->ne; e++) {
         const int64_t pos = pa->order.pos_of(e);
         for (int q = 0; q < pa->nqd; q++)
            for (int c = 0; c < pa->ncomp; c++) {
               const double v = dev[qdata_index(pa->qlayout, pos, c, q, pa->ncomp, pa->nqd,
                                                pa->nq, pa->ne_pad)];
               host[(e * pa->nqd + q) * pa->ncomp + c] = v;
            }
      }
   });
}

int tfem_pa_basis(const tfem_pa *pa, double *B, double *G)
{
   return guard([&] {
      need(pa, "tfem_pa_basis");
      if (B) std::memcpy(B, pa->B.data(), sizeof(double) * pa->B.size());
      if (G) std::memcpy(G, pa->G.data(), sizeof(double) * pa->G.size());
   });
}

int tfem_pa_set_basis(tfem_pa *pa, const double *B, const double *G)
{
   return guard([&] {
      need_obj(pa, "tfem_pa_set_basis");
      need(B, "tfem_pa_set_basis");
      need(G, "tfem_pa_set_basis");
      std::memcpy(pa->B.data(), B, sizeof(double) * pa->B.size());
      std::memcpy(pa->G.data(), G, sizeof(double) * pa->G.size());
      pa->colloc = false; // tables of another basis: the general kernels
   });
}

int tfem_pa_apply_local(tfem_ctx *ctx, const tfem_pa *pa, const tfem_restriction *r,
                        const tfem_vec *x, tfem_vec *y)
{
   return guard([&] {
      need(ctx, "pa_apply_local");
      need(pa, "pa_apply_local");
      need(r, "pa_apply_local");
      if (!x || !y || x->n != r->ndofs || y->n != r->ndofs)
         invalid("pa_apply_local: size mismatch");
      if (x->d == y->d) invalid("pa_apply_local: x and y must not alias");
      ApplyFlags f;
      pa_apply(ctx, pa, r, x->d, y->d, f);
      TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   });
}

int tfem_pa_diagonal(tfem_ctx *ctx, const tfem_pa *pa, const tfem_restriction *r, tfem_vec *diag)
{
   return guard([&] {
      need(ctx, "pa_diagonal");
      need(pa, "pa_diagonal");
      need(r, "pa_diagonal");
      check_vec(diag, r->ndofs, "pa_diagonal");
      pa_diagonal(ctx, pa, r, diag->d);
      TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   });
}

// ---------------------------------------------------------------- operator
int tfem_operator_create(tfem_ctx *ctx, int n_pa, tfem_pa *const *pa, const tfem_restriction *r,
                         int64_t n_ess, const int32_t *ess, tfem_operator **out)
{
   return tfem_operator_create_p(ctx, n_pa, pa, r, nullptr, n_ess, ess, out);
}

int tfem_operator_create_p(tfem_ctx *ctx, int n_pa, tfem_pa *const *pa,
                           const tfem_restriction *r, const tfem_prolongation *P,
                           int64_t n_ess, const int32_t *ess, tfem_operator **out)
{
   return guard([&] {
      need(ctx, "tfem_operator_create");
      need(r, "tfem_operator_create");
      need(out, "tfem_operator_create");
      if (n_pa < 1) invalid("tfem_operator_create: need at least one integrator");
      if (P && P->n_local != r->ndofs)
         invalid("tfem_operator_create: prolongation / space size mismatch");
      auto *op = new tfem_operator;
      op->ctx = ctx;
      op->n = P ? P->n_true : r->ndofs;
      op->r = r;
      op->P = P;
      if (P) {
         TFEM_CUDA(cudaMalloc(&op->xl, sizeof(double) * static_cast<size_t>(r->ndofs)));
         TFEM_CUDA(cudaMalloc(&op->yl, sizeof(double) * static_cast<size_t>(r->ndofs)));
      }
      for (int k = 0; k < n_pa; k++) {
         if (!pa[k] || pa[k]->dim != r->dim || pa[k]->p != r->p || pa[k]->ne != r->ne) {
            delete op;
            invalid("forms: point factors were built for a different space");
         }
         op->pa.push_back(pa[k]);
      }
      try {
         operator_set_ess(ctx, op, n_ess, ess);
      } catch (...) {
         operator_release(op);
         throw;
      }
      *out = op;
      ctx_retain(ctx);
   });
}

int tfem_linear_form(tfem_ctx *ctx, const tfem_geometry *g, const tfem_restriction *r, int p,
                     const double *f_host, tfem_vec *b)
{
   return guard([&] {
      need(ctx, "LinearForm");
      need(g, "LinearForm");
      need(r, "LinearForm");
      need(f_host, "LinearForm: load function is empty");
      if (!b || b->n != r->ndofs) invalid("LinearForm: size mismatch");
      linear_form(ctx, g, r, p, f_host, b->d);
   });
}

int tfem_geometry_node_points(tfem_ctx *ctx, const tfem_geometry *g, int p, double *host_xy)
{
   return guard([&] {
      need(ctx, "project_coefficient");
      need(g, "project_coefficient");
      need(host_xy, "project_coefficient");
      geometry_node_points(ctx, g, p, host_xy);
   });
}

int tfem_project(tfem_ctx *ctx, const tfem_restriction *r, const double *f_nodes, tfem_vec *out)
{
   return guard([&] {
      need(ctx, "project_coefficient");
      need(r, "project_coefficient");
      need(f_nodes, "project_coefficient: function is empty");
      if (!out || out->n != r->ndofs) invalid("project_coefficient: size mismatch");
      double *e = nullptr;
      const size_t bytes = sizeof(double) * static_cast<size_t>(r->ne) * r->nd;
      TFEM_CUDA(cudaMalloc(&e, bytes));
      h2d(ctx->stream, e, f_nodes, bytes);
      restriction_assign_last(ctx, r, e, out->d);
      TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
      cudaFree(e);
   });
}

int tfem_l2_error(tfem_ctx *ctx, const tfem_geometry *g, const tfem_restriction *r, int p,
                  const tfem_vec *x, const double *u_exact_host, double *err)
{
   return guard([&] {
      need(ctx, "compute_l2_error");
      need(g, "compute_l2_error");
      need(r, "compute_l2_error");
      need(u_exact_host, "compute_l2_error: exact solution is empty");
      need(err, "compute_l2_error");
      if (!x || x->n != r->ndofs) invalid("compute_l2_error: size mismatch");
      *err = l2_error(ctx, g, r, p, x->d, u_exact_host);
   });
}

// ------------------------------------------------------------ prolongation
int tfem_prolongation_create(tfem_ctx *ctx, int64_t n_local, int64_t n_true, const int32_t *rowptr,
                             const int32_t *cols, const double *vals, const int32_t *true_index,
                             tfem_prolongation **out)
{
   return guard([&] {
      need(ctx, "tfem_prolongation_create");
      need(rowptr, "tfem_prolongation_create");
      need(true_index, "tfem_prolongation_create");
      need(out, "tfem_prolongation_create");
      if (rowptr[n_local] > 0 && (!cols || !vals)) invalid("tfem_prolongation_create: null CSR");
      *out = prolongation_create(ctx, n_local, n_true, rowptr, cols, vals, true_index);
      ctx_retain(ctx);
   });
}

int tfem_prolongation_destroy(tfem_prolongation *P)
{
   return guard([&] {
      if (!P) return;
      bind(P->ctx);
      tfem_ctx *ctx = P->ctx;
      prolongation_destroy(P);
      ctx_release(ctx);
   });
}

int tfem_prolongation_mult(tfem_ctx *ctx, const tfem_prolongation *P, const tfem_vec *x_true,
                           tfem_vec *y_local)
{
   return guard([&] {
      need(ctx, "SparseMatrix::mult");
      need(P, "SparseMatrix::mult");
      if (!x_true || !y_local || x_true->n != P->n_true || y_local->n != P->n_local)
         invalid("SparseMatrix::mult: size mismatch");
      prolongation_mult(ctx, P, x_true->d, nullptr, y_local->d, nullptr);
      TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   });
}

int tfem_prolongation_mult_transpose(tfem_ctx *ctx, const tfem_prolongation *P,
                                     const tfem_vec *x_local, tfem_vec *y_true)
{
   return guard([&] {
      need(ctx, "SparseMatrix::mult_transpose");
      need(P, "SparseMatrix::mult_transpose");
      if (!x_local || !y_true || x_local->n != P->n_local || y_true->n != P->n_true)
         invalid("SparseMatrix::mult_transpose: size mismatch");
      prolongation_mult_transpose(ctx, P, x_local->d, y_true->d, nullptr, nullptr, nullptr,
                                  nullptr);
      TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   });
}

int tfem_prolongation_local_to_true(tfem_ctx *ctx, const tfem_prolongation *P,
                                    const tfem_vec *x_local, tfem_vec *x_true)
{
   return guard([&] {
      need(ctx, "local_to_true");
      need(P, "local_to_true");
      if (!x_local || !x_true || x_local->n != P->n_local || x_true->n != P->n_true)
         invalid("local_to_true: size mismatch");
      prolongation_local_to_true(ctx, P, x_local->d, x_true->d);
      TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   });
}

int tfem_pa_diagonal_p(tfem_ctx *ctx, const tfem_pa *pa, const tfem_restriction *r,
                       const tfem_prolongation *P, tfem_vec *diag_true)
{
   return guard([&] {
      need(ctx, "pa_diagonal");
      need(pa, "pa_diagonal");
      need(r, "pa_diagonal");
      need(P, "pa_diagonal");
      if (!diag_true || diag_true->n != P->n_true) invalid("pa_diagonal: size mismatch");
      pa_diagonal_p(ctx, pa, r, P, diag_true->d);
   });
}

int tfem_operator_set_comm(tfem_operator *op, const tfem_comm *comm, const tfem_halo *halo,
                           int64_t n_not_owned, const int32_t *not_owned)
{
   return guard([&] {
      need_obj(op, "tfem_operator_set_comm");
      need(comm, "tfem_operator_set_comm");
      need(halo, "tfem_operator_set_comm");
      if (!comm->exchange || !comm->allreduce) invalid("tfem_operator_set_comm: null hook");
      operator_set_comm(op->ctx, op, *comm, *halo, n_not_owned, not_owned);
   });
}

int tfem_nccl_unique_id(unsigned char id[TFEM_NCCL_ID_BYTES])
{
   return guard([&] {
      need(id, "tfem_nccl_unique_id");
      nccl_unique_id(id);
   });
}

int tfem_nccl_create(tfem_ctx *ctx, int nranks, int rank, const unsigned char id[TFEM_NCCL_ID_BYTES],
                     tfem_nccl **out)
{
   return guard([&] {
      need(ctx, "tfem_nccl_create");
      need(id, "tfem_nccl_create");
      need(out, "tfem_nccl_create");
      *out = nccl_create(ctx, nranks, rank, id);
      ctx_retain(ctx);
   });
}

int tfem_nccl_destroy(tfem_nccl *comm)
{
   return guard([&] {
      if (!comm) return;
      bind(comm->ctx);
      tfem_ctx *ctx = comm->ctx;
      nccl_destroy(comm);
      ctx_release(ctx);
   });
}

int tfem_nccl_allreduce(tfem_ctx *ctx, tfem_nccl *comm, double *device_buf, int64_t k)
{
   return guard([&] {
      need(ctx, "tfem_nccl_allreduce");
      need(comm, "tfem_nccl_allreduce");
      if (k > 0) need(device_buf, "tfem_nccl_allreduce");
      if (k > 0) nccl_allreduce(ctx, comm, device_buf, k);
      TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   });
}

int tfem_operator_set_nccl(tfem_operator *op, tfem_nccl *comm, int n_peers, const int *peer,
                           const int64_t *n_send, const int32_t *const *send_idx,
                           const int64_t *n_recv, const int32_t *const *recv_idx,
                           int64_t n_not_owned, const int32_t *not_owned)
{
   return guard([&] {
      need_obj(op, "tfem_operator_set_nccl");
      need(comm, "tfem_operator_set_nccl");
      if (comm->ctx != op->ctx) invalid("tfem_operator_set_nccl: communicator of another context");
      if (n_peers > 0 && (!peer || !n_send || !send_idx || !n_recv || !recv_idx))
         invalid("tfem_operator_set_nccl: null halo list");
      operator_set_nccl(op->ctx, op, comm, n_peers, peer, n_send, send_idx, n_recv, recv_idx,
                        n_not_owned, not_owned);
   });
}

int tfem_operator_create_csr(tfem_ctx *ctx, int64_t n, const int32_t *rowptr, const int32_t *cols,
                             const double *vals, tfem_operator **out)
{
   return guard([&] {
      need(ctx, "tfem_operator_create_csr");
      need(rowptr, "tfem_operator_create_csr");
      need(out, "tfem_operator_create_csr");
      *out = operator_csr(ctx, n, rowptr, cols, vals);
      ctx_retain(ctx);
   });
}

int tfem_operator_destroy(tfem_operator *op)
{
   return guard([&] {
      if (!op) return;
      bind(op->ctx);
      tfem_ctx *ctx = op->ctx;
      operator_release(op);
      ctx_release(ctx);
   });
}

int64_t tfem_operator_size(const tfem_operator *op) { return op ? op->n : 0; }

int tfem_operator_mult(tfem_ctx *ctx, const tfem_operator *op, const tfem_vec *x, tfem_vec *y)
{
   return guard([&] {
      need(ctx, "BilinearForm::mult_true");
      need(op, "BilinearForm::mult_true");
      if (!x || !y || x->n != op->n || y->n != op->n)
         invalid("BilinearForm::mult_true: size mismatch");
      if (x->d == y->d) invalid("BilinearForm::mult_true: x and y must not alias");
      operator_mult(ctx, op, x->d, y->d, nullptr, nullptr, nullptr);
      TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   });
}

int tfem_operator_mult_async(tfem_ctx *ctx, const tfem_operator *op, const tfem_vec *x,
                             tfem_vec *y)
{
   return guard([&] {
      need(ctx, "BilinearForm::mult_true");
      need(op, "BilinearForm::mult_true");
      if (!x || !y || x->n != op->n || y->n != op->n)
         invalid("BilinearForm::mult_true: size mismatch");
      if (x->d == y->d) invalid("BilinearForm::mult_true: x and y must not alias");
      operator_mult(ctx, op, x->d, y->d, nullptr, nullptr, nullptr);
   });
}

int tfem_operator_diagonal(tfem_ctx *ctx, const tfem_operator *op, tfem_vec *diag)
{
   return guard([&] {
      need(ctx, "BilinearForm::diagonal_true");
      need(op, "BilinearForm::diagonal_true");
      check_vec(diag, op->n, "BilinearForm::diagonal_true");
      operator_diagonal(ctx, op, diag->d);
   });
}

// ---------------------------------------------------------------------- CG
int tfem_cg_solve(tfem_ctx *ctx, const tfem_operator *op, const tfem_vec *b, double rel_tol,
                  int max_iters, const tfem_vec *jacobi_diag, tfem_vec *x, tfem_cg_result *res,
                  tfem_cg_callback cb, void *user)
{
   return guard([&] {
      need(ctx, "cg_solve");
      need(op, "cg_solve");
      need(res, "cg_solve");
      if (!b || b->n != op->n) invalid("cg_solve: operator/vector size mismatch");
      if (!x || x->n != op->n) invalid("cg_solve: operator/vector size mismatch");
      if (jacobi_diag && jacobi_diag->n != op->n)
         invalid("cg_solve: preconditioner size mismatch");
      if (x->d == b->d) invalid("cg_solve: x and b must not alias");
      cg_solve(ctx, op, b->d, rel_tol, max_iters, jacobi_diag ? jacobi_diag->d : nullptr, x->d,
               res, cb, user);
   });
}

int tfem_cg_profile(tfem_ctx *ctx, const tfem_operator *op, const tfem_vec *b, int iters,
                    const tfem_vec *jacobi_diag, tfem_vec *x, double *seg_us)
{
   return guard([&] {
      need(ctx, "cg_profile");
      need(op, "cg_profile");
      need(seg_us, "cg_profile");
      if (op->has_comm) invalid("cg_profile: single-device operators only");
      if (iters < 1) invalid("cg_profile: iters must be >= 1");
      if (!b || b->n != op->n || !x || x->n != op->n)
         invalid("cg_profile: operator/vector size mismatch");
      if (jacobi_diag && jacobi_diag->n != op->n)
         invalid("cg_profile: preconditioner size mismatch");
      if (x->d == b->d) invalid("cg_profile: x and b must not alias");
      tfem_cg_result res{};
      cg_solve(ctx, op, b->d, 0.0, iters, jacobi_diag ? jacobi_diag->d : nullptr, x->d, &res,
               nullptr, nullptr, seg_us);
   });
}

int tfem_fp64_peak(tfem_ctx *ctx, double *tflops)
{
   return guard([&] {
      need(ctx, "fp64_peak");
      need(tflops, "fp64_peak");
      *tflops = fp64_peak_tflops(ctx);
   });
}

int tfem_dmma_peak(tfem_ctx *ctx, double *tflops)
{
   return guard([&] {
      need(ctx, "dmma_peak");
      need(tflops, "dmma_peak");
      *tflops = dmma_peak_tflops(ctx);
   });
}

int tfem_contraction_ab(tfem_ctx *ctx, int p, double *res)
{
   return guard([&] {
      need(ctx, "contraction_ab");
      need(res, "contraction_ab");
      bind(ctx);
      contraction_ab(ctx, p, res);
   });
}

int tfem_cg_solve_host(tfem_ctx *ctx, const tfem_operator *op, const double *b, double rel_tol,
                       int max_iters, const double *jacobi_diag, double *x, tfem_cg_result *res)
{
   return guard([&] {
      need(ctx, "cg_solve");
      need(op, "cg_solve");
      need(b, "cg_solve");
      need(x, "cg_solve");
      need(res, "cg_solve");
      const int64_t n = op->n;
      // Device staging buffers cached per context (and size).
      auto buf = [&](int slot) -> double * {
         if (ctx->stage_n[slot] != n) {
            TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
            cudaFree(ctx->stage[slot]);
            ctx->stage[slot] = nullptr;
            ctx->stage_n[slot] = 0;
            TFEM_CUDA(cudaMalloc(&ctx->stage[slot], sizeof(double) * n));
            ctx->stage_n[slot] = n;
         }
         return ctx->stage[slot];
      };
      double *db = buf(0), *dx = buf(1), *dd = jacobi_diag ? buf(2) : nullptr;
      TFEM_CUDA(cudaMemcpyAsync(db, b, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
      if (dd)
         TFEM_CUDA(cudaMemcpyAsync(dd, jacobi_diag, sizeof(double) * n, cudaMemcpyHostToDevice,
                                   ctx->stream));
      cg_solve(ctx, op, db, rel_tol, max_iters, dd, dx, res, nullptr, nullptr);
      TFEM_CUDA(cudaMemcpyAsync(x, dx, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
      TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   });
}

} // extern "C"
