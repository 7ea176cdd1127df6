// K5 / K6: operators and the device-resident Jacobi-PCG of cg_solve
// (solvers.cpp:11-97).
//
// Per iteration (all on the device, batches of 16 iterations replayed as one
// CUDA graph, only the CG state read back per batch), four launches:
//   1-2. q = A p          element kernel + shared-DOF scatter, fused p.q
//                         partials; the last block to finish folds them and
//                         takes alpha = rz / pq (emit, common.cuh)
//   3.   update kernel    r -= alpha q, z = r / d, partials of r.r and r.z;
//                         its last block takes ||r||, the best-iterate
//                         bookkeeping, beta and the stop test
//   4.   direction kernel x' = x + alpha p and p = r / d + beta p (p read once)
// Vector updates use unfused multiply + add in the reference's order
// (vector.cpp:20-23, solvers.cpp:84-87), so only the dot products differ from
// the CPU (tree vs sequential sum).  The best iterate (solvers.cpp:78-81) costs
// no copies: x rotates through three buffers and "best" is an index.
#include "common.cuh"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <unordered_map>

namespace tfem {

void vec_axpy(tfem_ctx *ctx, double a, const double *x, double *y, int64_t n);
void comm_allreduce(tfem_ctx *ctx, const tfem_operator *op, int k);

namespace {

constexpr int kVecThreads = 256;

inline unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

// Fixed grid for vector kernels: deterministic partial count for a given n.
// 4 blocks of 256 per SM (measured against 2-32: +2 % CG at 10M DOFs over 8,
// same at 100M).
inline unsigned vec_blocks(const tfem_ctx *ctx, int64_t n)
{
   constexpr int64_t per_sm = 4;
   const int64_t cap = static_cast<int64_t>(ctx->sm_count) * per_sm;
   const int64_t need = (n + kVecThreads - 1) / kVecThreads;
   return static_cast<unsigned>(need < cap ? (need > 0 ? need : 1) : cap);
}

__global__ void fill_kernel(double *d, int64_t n, double v)
{
   for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
        i += (int64_t)gridDim.x * blockDim.x)
      d[i] = v;
}

__global__ void __launch_bounds__(kVecThreads)
dot_kernel(const double *__restrict__ a, const double *__restrict__ b, int64_t n, DotSink sink,
           const uint32_t *notown)
{
   double s = 0.0;
   for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
        i += (int64_t)gridDim.x * blockDim.x)
      if (!(notown && bit_set(notown, static_cast<uint32_t>(i))))
         s = __dadd_rn(s, __dmul_rn(a[i], b[i]));
   const double v[1] = {s};
   emit<kVecThreads, 1>(sink, v);
}

// Fixed-order fold of `n` chunk sums by one block (valid in thread 0).
__device__ double fold(const double *p, int64_t n)
{
   double s = 0.0;
   for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += __ldcg(p + i);
   return block_sum<kVecThreads>(s);
}

__global__ void __launch_bounds__(kVecThreads)
fold_kernel(const double *chunks, int64_t n, double *out)
{
   const double s = fold(chunks, n);
   if (threadIdx.x == 0) out[0] = s;
}

__global__ void axpy_kernel(double a, const double *x, double *y, int64_t n)
{
   for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
        i += (int64_t)gridDim.x * blockDim.x)
      y[i] = __dadd_rn(y[i], __dmul_rn(a, x[i]));
}

__global__ void set_bits_kernel(const int32_t *list, int64_t n, uint32_t *mask)
{
   const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (i < n) atomicOr(mask + (list[i] >> 5), 1u << (list[i] & 31));
}

// tfem_operator::elem_ess: word[pos] bit i = slot i's DOF is in the mask.
__global__ void elem_ess_kernel(const uint32_t *gmap, int nd, int64_t npos, int64_t ne_pad,
                                const uint32_t *mask, uint32_t *words)
{
   const int64_t pos = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (pos >= npos) return;
   uint32_t w = 0;
   for (int i = 0; i < nd; i++)
      w |= static_cast<uint32_t>(bit_set(mask, gmap[i * ne_pad + pos] & kDofMask)) << i;
   words[pos] = w;
}

__global__ void set_values_kernel(const int32_t *list, int64_t n, double v, double *y)
{
   const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (i < n) y[list[i]] = v;
}

// SparseMatrix::mult (sparse.cpp:75-87), thread per row, optional x.y partial.
__global__ void __launch_bounds__(kVecThreads)
csr_kernel(const int32_t *rowptr, const int32_t *cols, const double *vals, int64_t n,
           const double *x, double *y, DotSink sink, const int *done)
{
   if (done && *done) return;
   const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   double dot = 0.0;
   if (i < n) {
      double s = 0.0;
      for (int k = rowptr[i]; k < rowptr[i + 1]; k++) s = __dadd_rn(s, __dmul_rn(vals[k], x[cols[k]]));
      y[i] = s;
      dot = __dmul_rn(x[i], s);
   }
   if (sink) {
      const double v[1] = {dot};
      emit<kVecThreads, 1>(sink, v);
   }
}

// ----------------------------------------------------------------- CG
// r = b, z = M r, p = z, x0 = 0; partials of r.r and r.z (solvers.cpp:43-58)
__global__ void __launch_bounds__(kVecThreads)
cg_init_kernel(const double *__restrict__ b, const double *__restrict__ diag, int64_t n,
               double *__restrict__ r, double *__restrict__ p, double *__restrict__ x,
               DotSink sink, const uint32_t *notown)
{
   double rr = 0.0, rz = 0.0;
   for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
        i += (int64_t)gridDim.x * blockDim.x) {
      const double ri = b[i];
      const double zi = diag ? __ddiv_rn(ri, diag[i]) : ri;
      r[i] = ri;
      p[i] = zi;
      x[i] = 0.0;
      if (notown && bit_set(notown, static_cast<uint32_t>(i))) continue;
      rr = __dadd_rn(rr, __dmul_rn(ri, ri));
      rz = __dadd_rn(rz, __dmul_rn(ri, zi));
   }
   const double v[2] = {rr, rz};
   emit<kVecThreads, 2>(sink, v);
}

__device__ void init_step(CgState *st, double rr, double rz)
{
   st->rz = rz;
   st->rnorm = sqrt(rr);
   st->best_rnorm = st->rnorm;
   st->it = 0;
   st->done = 0;
   st->converged = 0;
   st->iterations = 0;
   st->status = 0;
   st->cur = 0;
   st->best = 0;
   st->prev = 0;
   st->xpend = 0;
   if (st->rnorm <= st->target) { // top of iteration 1 (solvers.cpp:61-65)
      st->done = 1;
      st->converged = 1;
      st->iterations = 0;
   }
}

__global__ void __launch_bounds__(kVecThreads)
cg_init_finish_kernel(const double *chunks, int64_t nch, CgState *st)
{
   const double rr = fold(chunks, nch);
   const double rz = fold(chunks + nch, nch);
   if (threadIdx.x == 0) init_step(st, rr, rz);
}

// Distributed variants: the rank-local fold lands in red[] (device), the
// host hook sums red[] over ranks in place, then the step kernel reads it.
__global__ void __launch_bounds__(kVecThreads)
fold_to_kernel(const double *ch_a, int64_t na, const double *ch_b, int64_t nb, int k,
               double *out)
{
   for (int j = 0; j < k; j++) {
      double s = 0.0;
      for (int64_t i = threadIdx.x; i < na + nb; i += blockDim.x)
         s += __ldcg(i < na ? ch_a + j * na + i : ch_b + j * nb + (i - na));
      const double t = block_sum<kVecThreads>(s);
      if (threadIdx.x == 0) out[j] = t;
   }
}

__global__ void red_init_kernel(const double *red, CgState *st) { init_step(st, red[0], red[1]); }

__global__ void red_alpha_kernel(const double *red, CgState *st)
{
   if (!st->done) alpha_step(st, red[0]);
}

__global__ void red_beta_kernel(const double *red, CgState *st)
{
   if (!st->done) beta_step(st, red[0], red[1]);
}

struct XBufs {
   double *x[3];
};

constexpr int kUnroll = 4;

// r -= alpha q, z = r / d; partials of r.r, r.z.  Four independent
// elements per trip keep ~16 loads in flight per thread.  (x' = x + alpha p
// is taken by the direction kernel, which streams p anyway.)
__global__ void __launch_bounds__(kVecThreads)
cg_update_kernel(const CgState *st, const double *__restrict__ q, double *__restrict__ r,
                 const double *__restrict__ diag, int64_t n, DotSink sink,
                 const uint32_t *notown)
{
   if (st->done) return;
   const double nalpha = -st->alpha;
   double rr = 0.0, rz = 0.0;
   const int64_t stride = (int64_t)gridDim.x * blockDim.x;
   int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   for (; i + (kUnroll - 1) * stride < n; i += kUnroll * stride) {
      double rv[kUnroll], qv[kUnroll], dv[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; u++) {
         const int64_t j = i + u * stride;
         rv[u] = r[j];
         qv[u] = q[j];
         dv[u] = diag ? diag[j] : 1.0;
      }
#pragma unroll
      for (int u = 0; u < kUnroll; u++) {
         const int64_t j = i + u * stride;
         const double ri = __dadd_rn(rv[u], __dmul_rn(nalpha, qv[u]));
         r[j] = ri;
         const double zi = diag ? __ddiv_rn(ri, dv[u]) : ri;
         if (notown && bit_set(notown, static_cast<uint32_t>(j))) continue;
         rr = __dadd_rn(rr, __dmul_rn(ri, ri));
         rz = __dadd_rn(rz, __dmul_rn(ri, zi));
      }
   }
   for (; i < n; i += stride) {
      const double ri = __dadd_rn(r[i], __dmul_rn(nalpha, q[i]));
      r[i] = ri;
      const double zi = diag ? __ddiv_rn(ri, diag[i]) : ri;
      if (notown && bit_set(notown, static_cast<uint32_t>(i))) continue;
      rr = __dadd_rn(rr, __dmul_rn(ri, ri));
      rz = __dadd_rn(rz, __dmul_rn(ri, zi));
   }
   const double v[2] = {rr, rz};
   emit<kVecThreads, 2>(sink, v);
}

// x[cur] = x[prev] + alpha p (the iteration's pending x update, solvers.cpp:
// 66-67) and, unless the solve just ended, p = z + beta p with z = r / d
// (solvers.cpp:84-87): p is read once for both.  The last block clears the
// pending flag, so the no-op iterations after convergence skip it.
__global__ void __launch_bounds__(kVecThreads)
cg_direction_kernel(CgState *st, XBufs xb, const double *__restrict__ r,
                    const double *__restrict__ diag, double *__restrict__ p, int64_t n,
                    unsigned *ticket)
{
   const bool xu = st->xpend != 0, pu = !st->done;
   if (!xu && !pu) return;
   const double beta = st->beta, alpha = st->alpha;
   const double *__restrict__ xo = xb.x[st->prev];
   double *__restrict__ xn = xb.x[st->cur];
   const int64_t stride = (int64_t)gridDim.x * blockDim.x;
   int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   for (; i + (kUnroll - 1) * stride < n; i += kUnroll * stride) {
      double rv[kUnroll], dv[kUnroll], pv[kUnroll], xv[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; u++) {
         const int64_t j = i + u * stride;
         pv[u] = p[j];
         if (xu) xv[u] = xo[j];
         if (pu) {
            rv[u] = r[j];
            dv[u] = diag ? diag[j] : 1.0;
         }
      }
#pragma unroll
      for (int u = 0; u < kUnroll; u++) {
         const int64_t j = i + u * stride;
         if (xu) xn[j] = __dadd_rn(xv[u], __dmul_rn(alpha, pv[u]));
         if (pu) {
            const double zi = diag ? __ddiv_rn(rv[u], dv[u]) : rv[u];
            p[j] = __dadd_rn(zi, __dmul_rn(beta, pv[u]));
         }
      }
   }
   for (; i < n; i += stride) {
      const double pv = p[i];
      if (xu) xn[i] = __dadd_rn(xo[i], __dmul_rn(alpha, pv));
      if (pu) {
         const double zi = diag ? __ddiv_rn(r[i], diag[i]) : r[i];
         p[i] = __dadd_rn(zi, __dmul_rn(beta, pv));
      }
   }
   if (xu) {
      __shared__ bool last;
      __syncthreads();
      if (threadIdx.x == 0) {
         __threadfence();
         last = atomicAdd(ticket, 1u) == gridDim.x - 1;
      }
      __syncthreads();
      if (last && threadIdx.x == 0) {
         st->xpend = 0;
         *ticket = 0u;
      }
   }
}

__global__ void diag_check_kernel(const double *d, int64_t n, int *bad)
{
   for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
        i += (int64_t)gridDim.x * blockDim.x)
      if (!(d[i] > 0.0)) *bad = 1;
}

template <typename T>
T *dalloc(int64_t n)
{
   T *p = nullptr;
   TFEM_CUDA(cudaMalloc(&p, sizeof(T) * static_cast<size_t>(n > 0 ? n : 1)));
   return p;
}

// Device storage of a DotSink for `grid` blocks and `nv` values per block.
struct SinkStore {
   DotSink s;
   int64_t grid = 0, nch = 0;
   void alloc(cudaStream_t stream, int64_t g, int nv)
   {
      grid = g;
      nch = n_chunks(g);
      s.partials = dalloc<double>(nv * g);
      s.chunks = dalloc<double>(nv * nch);
      s.tickets = dalloc<unsigned>(nch + 1);
      TFEM_CUDA(cudaMemsetAsync(s.tickets, 0, sizeof(unsigned) * (nch + 1), stream));
   }
   void release()
   {
      cudaFree(s.partials);
      cudaFree(s.chunks);
      cudaFree(s.tickets);
      s = DotSink{};
      grid = nch = 0;
   }
};

// Per-operator CG workspace, reused across solves (vectors + graph).
struct Workspace {
   int64_t n = 0;
   double *r = nullptr, *p = nullptr, *q = nullptr, *xa = nullptr, *xb = nullptr;
   SinkStore s_elem, s_scatter, s_vec;
   CgState *st = nullptr;
   unsigned *dir_ticket = nullptr; // last-block ticket of the direction kernel
   CgState *host_st = nullptr; // pinned
   cudaGraphExec_t graph = nullptr;
   const double *g_diag = nullptr, *g_x = nullptr;
   int g_batch = 0, g_numerics = -1;
   int64_t g_launches = 0;
   int64_t ge = -1, gs = -1; // element / scatter grids the PA sinks are sized for
   ~Workspace()
   {
      cudaFree(r);
      cudaFree(p);
      cudaFree(q);
      cudaFree(xa);
      cudaFree(xb);
      s_elem.release();
      s_scatter.release();
      s_vec.release();
      cudaFree(st);
      cudaFree(dir_ticket);
      if (host_st) cudaFreeHost(host_st);
      if (graph) cudaGraphExecDestroy(graph);
   }
};

std::unordered_map<const tfem_operator *, std::unique_ptr<Workspace>> &workspaces()
{
   static std::unordered_map<const tfem_operator *, std::unique_ptr<Workspace>> w;
   return w;
}
std::mutex &workspaces_mu()
{
   static std::mutex mu;
   return mu;
}

// The element kernel's grid depends on the context's numerics (kernel
// variants differ in warps per block) and on its grid cap: the PA dot sinks
// follow it, and the captured graph is dropped when it changes.
void fit_pa_sinks(tfem_ctx *ctx, const tfem_operator *op, Workspace &w)
{
   if (op->csr || op->P) return;
   int64_t ge = 0, gs = 0;
   pa_apply_grids(op->pa.back(), op->r, &ge, &gs);
   if (ge == w.ge && gs == w.gs) return;
   TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   w.s_elem.release();
   w.s_scatter.release();
   w.s_elem.alloc(ctx->stream, ge, 1);
   if (gs > 0) w.s_scatter.alloc(ctx->stream, gs, 1);
   w.ge = ge;
   w.gs = gs;
   if (w.graph) {
      cudaGraphExecDestroy(w.graph);
      w.graph = nullptr;
   }
}

Workspace &workspace_for(tfem_ctx *ctx, const tfem_operator *op)
{
   std::lock_guard<std::mutex> lock(workspaces_mu());
   auto &m = workspaces();
   auto it = m.find(op);
   if (it != m.end()) {
      fit_pa_sinks(ctx, op, *it->second);
      return *it->second;
   }
   auto w = std::make_unique<Workspace>();
   w->n = op->n;
   w->r = dalloc<double>(op->n);
   w->p = dalloc<double>(op->n);
   w->q = dalloc<double>(op->n);
   w->xa = dalloc<double>(op->n);
   w->xb = dalloc<double>(op->n);
   if (op->csr) {
      w->s_elem.alloc(ctx->stream, blocks_for(op->n, kVecThreads), 1);
   } else if (op->P) {
      if (op->r->needs_evec()) const_cast<tfem_restriction *>(op->r)->ensure_evec();
      w->s_elem.alloc(ctx->stream, prolongation_grid(op->P), 1); // the P^T kernel's p . q
   } else {
      // everything the iteration touches must exist before graph capture
      if (op->r->needs_evec()) const_cast<tfem_restriction *>(op->r)->ensure_evec();
      fit_pa_sinks(ctx, op, *w);
   }
   w->s_vec.alloc(ctx->stream, vec_blocks(ctx, op->n), 2);
   w->st = dalloc<CgState>(1);
   w->dir_ticket = dalloc<unsigned>(1);
   TFEM_CUDA(cudaMemsetAsync(w->dir_ticket, 0, sizeof(unsigned), ctx->stream));
   TFEM_CUDA(cudaMallocHost(&w->host_st, sizeof(CgState)));
   auto &ref = *w;
   m.emplace(op, std::move(w));
   return ref;
}

// One CG iteration's launches (used eagerly and under stream capture).
void enqueue_iteration(tfem_ctx *ctx, const tfem_operator *op, Workspace &w, XBufs xb,
                       const double *diag, cudaEvent_t *ev = nullptr)
{

   const int64_t n = op->n;
   // alpha is taken by the last block of the operator's final launch, beta by
   // the last block of the update: four launches per iteration.
   DotSink se = w.s_elem.s, ss = w.s_scatter.s, sv = w.s_vec.s;
   DotSink &fin = w.s_scatter.grid ? ss : se;
   if (w.s_scatter.grid) {
      ss.pre = w.s_elem.s.chunks;
      ss.n_pre = w.s_elem.nch;
   }
   fin.state = w.st;
   fin.finish = kFinishAlpha;
   sv.state = w.st;
   sv.finish = kFinishBeta;
   operator_mult(ctx, op, w.p, w.q, &se, w.s_scatter.grid ? &ss : nullptr, &w.st->done);
   if (ev) TFEM_CUDA(cudaEventRecord(ev[1], ctx->stream));
   const unsigned vb = vec_blocks(ctx, n);
   cg_update_kernel<<<vb, kVecThreads, 0, ctx->stream>>>(w.st, w.q, w.r, diag, n, sv, nullptr);
   if (ev) TFEM_CUDA(cudaEventRecord(ev[2], ctx->stream));
   cg_direction_kernel<<<vb, kVecThreads, 0, ctx->stream>>>(w.st, xb, w.r, diag, w.p, n,
                                                            w.dir_ticket);
   if (ev) TFEM_CUDA(cudaEventRecord(ev[3], ctx->stream));
   ctx->launched(2);
   TFEM_CUDA(cudaGetLastError());
}

// The halo part of the direction update, packed for the send: out[i] = the
// new p at DOF idx[i], with cg_direction_kernel's arithmetic (same bits), so
// the exchange can run while that kernel updates all of p.
__global__ void pack_direction_kernel(const CgState *st, const double *__restrict__ r,
                                      const double *__restrict__ diag,
                                      const double *__restrict__ p, const int32_t *idx, int64_t n,
                                      double *out)
{
   if (st->done) return;
   const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (i >= n) return;
   const int32_t j = idx[i];
   const double zi = diag ? __ddiv_rn(r[j], diag[j]) : r[j];
   out[i] = __dadd_rn(zi, __dmul_rn(st->beta, p[j]));
}

__global__ void gather_idx_kernel(const double *v, const int32_t *idx, int64_t n, double *out)
{
   const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (i < n) out[i] = v[idx[i]];
}

__global__ void scatter_idx_kernel(const double *in, const int32_t *idx, int64_t n, double *v)
{
   const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (i < n) v[idx[i]] = in[i];
}

__global__ void copy_scalar_kernel(const double *src, double *dst) { *dst = *src; }

} // namespace

void vec_fill(tfem_ctx *ctx, double *d, int64_t n, double v)
{
   fill_kernel<<<vec_blocks(ctx, n), kVecThreads, 0, ctx->stream>>>(d, n, v);
   ctx->launched();
   TFEM_CUDA(cudaGetLastError());
}

double vec_dot(tfem_ctx *ctx, const double *a, const double *b, int64_t n,
               const tfem_operator *dist)
{
   const uint32_t *notown = dist ? dist->notown : nullptr;
   // dot sinks cached on the context, by grid size
   const unsigned nb = vec_blocks(ctx, n);
   DotSink sink;
   for (auto &d : ctx->dot_sinks)
      if (d.first == nb) {
         sink.partials = d.second.partials;
         sink.chunks = d.second.chunks;
         sink.tickets = d.second.tickets;
      }
   if (!sink) {
      SinkStore st;
      st.alloc(ctx->stream, nb, 1);
      sink = st.s;
      ctx->dot_sinks.push_back({nb, {sink.partials, sink.chunks, sink.tickets}});
   }
   const int64_t nch = n_chunks(nb);
   dot_kernel<<<nb, kVecThreads, 0, ctx->stream>>>(a, b, n, sink, notown);
   fold_kernel<<<1, kVecThreads, 0, ctx->stream>>>(sink.chunks, nch, ctx->scalars);
   ctx->launched(2);
   TFEM_CUDA(cudaGetLastError());
   if (dist) {
      copy_scalar_kernel<<<1, 1, 0, ctx->stream>>>(ctx->scalars, dist->red);
      comm_allreduce(ctx, dist, 1);
      copy_scalar_kernel<<<1, 1, 0, ctx->stream>>>(dist->red, ctx->scalars);
      ctx->launched(2);
   }
   TFEM_CUDA(cudaMemcpyAsync(ctx->host_scalars, ctx->scalars, sizeof(double),
                             cudaMemcpyDeviceToHost, ctx->stream));
   TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   return ctx->host_scalars[0];
}

void vec_axpy(tfem_ctx *ctx, double a, const double *x, double *y, int64_t n)
{
   axpy_kernel<<<vec_blocks(ctx, n), kVecThreads, 0, ctx->stream>>>(a, x, y, n);
   ctx->launched();
   TFEM_CUDA(cudaGetLastError());
}

void operator_set_ess(tfem_ctx *ctx, tfem_operator *op, int64_t n_ess, const int32_t *ess)
{
   op->n_ess = n_ess;
   if (n_ess == 0) return;
   for (int64_t i = 0; i < n_ess; i++) {
      if (ess[i] < 0 || ess[i] >= op->n) invalid("form_linear_system: essential DOF out of range");
      if (i > 0 && ess[i] <= ess[i - 1])
         invalid("form_linear_system: essential list must be sorted and unique");
   }
   op->ess = dalloc<int32_t>(n_ess);
   const int64_t words = (op->n + 31) / 32;
   op->ess_mask = dalloc<uint32_t>(words);
   h2d(ctx->stream, op->ess, ess, sizeof(int32_t) * n_ess);
   TFEM_CUDA(cudaMemsetAsync(op->ess_mask, 0, sizeof(uint32_t) * words, ctx->stream));
   set_bits_kernel<<<blocks_for(n_ess, 256), 256, 0, ctx->stream>>>(op->ess, n_ess,
                                                                   op->ess_mask);
   ctx->launched();
   TFEM_CUDA(cudaGetLastError());
   const tfem_restriction *r = op->r;
   if (r && !op->P && !r->elem_major && r->nd <= 32 && r->npos > 0) {
      op->elem_ess = dalloc<uint32_t>(r->ne_pad);
      TFEM_CUDA(cudaMemsetAsync(op->elem_ess, 0, sizeof(uint32_t) * r->ne_pad, ctx->stream));
      elem_ess_kernel<<<blocks_for(r->npos, 256), 256, 0, ctx->stream>>>(
         r->gmap, r->nd, r->npos, r->ne_pad, op->ess_mask, op->elem_ess);
      ctx->launched();
      TFEM_CUDA(cudaGetLastError());
   }
   TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
}

namespace {
// The owned halo buffers of an NCCL operator (and its reduction slots).
void free_nccl_buffers(tfem_operator *op)
{
   if (!op->nccl) return;
   for (int k = 0; k < op->n_peers; k++) {
      cudaFree(op->send_buf[k]);
      cudaFree(op->recv_buf[k]);
      op->send_buf[k] = op->recv_buf[k] = nullptr;
   }
   cudaFree(op->red);
   op->red = nullptr;
   if (op->side) cudaStreamDestroy(op->side);
   if (op->ev_fork) cudaEventDestroy(op->ev_fork);
   if (op->ev_join) cudaEventDestroy(op->ev_join);
   op->side = nullptr;
   op->ev_fork = op->ev_join = nullptr;
   nccl_destroy(op->nccl); // the operator's reference
   op->nccl = nullptr;
}

// Halo lists, ownership bitmap and buffers of a distributed operator
// (DESIGN.md 6), shared by the hook (set_comm) and NCCL (set_nccl) paths.
void set_plan(tfem_ctx *ctx, tfem_operator *op, int n_peers, const int64_t *n_send,
              const int32_t *const *send_idx, const int64_t *n_recv,
              const int32_t *const *recv_idx, int64_t n_not_owned, const int32_t *not_owned)
{
   if (op->csr) invalid("tfem_operator_set_comm: needs a PA operator");
   if (op->P) invalid("tfem_operator_set_comm: prolongated (non-conforming) operators run on one device");
   if (n_peers < 0 || n_peers > TFEM_MAX_PEERS) invalid("tfem_operator_set_comm: bad peer count");
   auto upload = [&](const int32_t *idx, int64_t n) -> int32_t * {
      for (int64_t i = 0; i < n; i++)
         if (idx[i] < 0 || idx[i] >= op->n) invalid("tfem_operator_set_comm: DOF out of range");
      int32_t *d = dalloc<int32_t>(n);
      h2d(ctx->stream, d, idx, sizeof(int32_t) * n);
      return d;
   };
   free_nccl_buffers(op);
   for (int k = 0; k < op->n_peers; k++) {
      cudaFree(op->send_idx[k]);
      cudaFree(op->recv_idx[k]);
   }
   op->n_peers = n_peers;
   for (int k = 0; k < n_peers; k++) {
      op->n_send[k] = n_send[k];
      op->n_recv[k] = n_recv[k];
      op->send_idx[k] = upload(send_idx[k], n_send[k]);
      op->recv_idx[k] = upload(recv_idx[k], n_recv[k]);
   }
   cudaFree(op->notown);
   op->notown = nullptr;
   if (n_not_owned > 0) {
      int32_t *d = upload(not_owned, n_not_owned);
      const int64_t words = (op->n + 31) / 32;
      op->notown = dalloc<uint32_t>(words);
      TFEM_CUDA(cudaMemsetAsync(op->notown, 0, sizeof(uint32_t) * words, ctx->stream));
      set_bits_kernel<<<blocks_for(n_not_owned, 256), 256, 0, ctx->stream>>>(d, n_not_owned,
                                                                              op->notown);
      ctx->launched();
      TFEM_CUDA(cudaGetLastError());
      TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
      cudaFree(d);
   }
   op->has_comm = true;
}
} // namespace

void operator_set_comm(tfem_ctx *ctx, tfem_operator *op, const tfem_comm &comm,
                       const tfem_halo &halo, int64_t n_not_owned, const int32_t *not_owned)
{
   if (!halo.red) invalid("tfem_operator_set_comm: null reduction buffer");
   set_plan(ctx, op, halo.n_peers, halo.n_send, halo.send_idx, halo.n_recv, halo.recv_idx,
            n_not_owned, not_owned);
   for (int k = 0; k < halo.n_peers; k++) {
      op->send_buf[k] = halo.send_buf[k];
      op->recv_buf[k] = halo.recv_buf[k];
   }
   op->red = halo.red;
   op->comm = comm;
}

void operator_set_nccl(tfem_ctx *ctx, tfem_operator *op, tfem_nccl *comm, int n_peers,
                       const int *peer, const int64_t *n_send, const int32_t *const *send_idx,
                       const int64_t *n_recv, const int32_t *const *recv_idx,
                       int64_t n_not_owned, const int32_t *not_owned)
{
   // a rank may list itself (a self send / receive pair: NCCL supports it;
   // periodic plans and the overlap test use it)
   for (int k = 0; k < n_peers; k++)
      if (peer[k] < 0 || peer[k] >= comm->nranks)
         invalid("tfem_operator_set_nccl: bad peer rank");
   set_plan(ctx, op, n_peers, n_send, send_idx, n_recv, recv_idx, n_not_owned, not_owned);
   for (int k = 0; k < n_peers; k++) {
      op->peer_rank[k] = peer[k];
      op->send_buf[k] = dalloc<double>(n_send[k]);
      op->recv_buf[k] = dalloc<double>(n_recv[k]);
   }
   op->red = dalloc<double>(4);
   op->comm = tfem_comm{};
   op->nccl = comm;
   nccl_retain(comm);
   if (n_peers > 0) {
      TFEM_CUDA(cudaStreamCreateWithFlags(&op->side, cudaStreamNonBlocking));
      TFEM_CUDA(cudaEventCreateWithFlags(&op->ev_fork, cudaEventDisableTiming));
      TFEM_CUDA(cudaEventCreateWithFlags(&op->ev_join, cudaEventDisableTiming));
   }
}

// Sum red[0..k) over the ranks, in stream order.
void comm_allreduce(tfem_ctx *ctx, const tfem_operator *op, int k)
{
   if (op->nccl) nccl_allreduce(ctx, op->nccl, op->red, k);
   else op->comm.allreduce(k, op->comm.user);
}

// Halo update of a device vector: pack, transfer, unpack (all on the stream).
void halo_exchange(tfem_ctx *ctx, const tfem_operator *op, double *v)
{
   for (int k = 0; k < op->n_peers; k++)
      if (op->n_send[k] > 0) {
         gather_idx_kernel<<<blocks_for(op->n_send[k], 256), 256, 0, ctx->stream>>>(
            v, op->send_idx[k], op->n_send[k], op->send_buf[k]);
         ctx->launched();
      }
   if (op->nccl) nccl_exchange(ctx, op, ctx->stream);
   else op->comm.exchange(op->comm.user);
   for (int k = 0; k < op->n_peers; k++)
      if (op->n_recv[k] > 0) {
         scatter_idx_kernel<<<blocks_for(op->n_recv[k], 256), 256, 0, ctx->stream>>>(
            op->recv_buf[k], op->recv_idx[k], op->n_recv[k], v);
         ctx->launched();
      }
   TFEM_CUDA(cudaGetLastError());
}

// The direction step of a distributed iteration with the next operator's
// halo update folded in: the send planes of the new p are packed straight
// from r, diag and the old p; with NCCL the exchange then runs on the side
// stream while cg_direction_kernel updates p and x on the context stream,
// and the received planes land after both (the direction kernel's values
// there -- not-owned DOFs -- are overwritten, as the halo update at the
// start of the iteration used to do).  The host-hook path runs the same
// data flow synchronously.
void halo_direction(tfem_ctx *ctx, const tfem_operator *op, CgState *st, const XBufs &xb,
                    const double *r, const double *diag, double *p, int64_t n, unsigned *ticket)
{
   for (int k = 0; k < op->n_peers; k++)
      if (op->n_send[k] > 0) {
         pack_direction_kernel<<<blocks_for(op->n_send[k], 256), 256, 0, ctx->stream>>>(
            st, r, diag, p, op->send_idx[k], op->n_send[k], op->send_buf[k]);
         ctx->launched();
      }
   const bool overlap = op->nccl && op->side;
   if (overlap) {
      TFEM_CUDA(cudaEventRecord(op->ev_fork, ctx->stream));
      TFEM_CUDA(cudaStreamWaitEvent(op->side, op->ev_fork, 0));
      nccl_exchange(ctx, op, op->side);
      TFEM_CUDA(cudaEventRecord(op->ev_join, op->side));
   } else if (op->nccl) {
      nccl_exchange(ctx, op, ctx->stream);
   } else {
      op->comm.exchange(op->comm.user);
   }
   cg_direction_kernel<<<vec_blocks(ctx, n), kVecThreads, 0, ctx->stream>>>(st, xb, r, diag, p, n,
                                                                           ticket);
   ctx->launched();
   if (overlap) TFEM_CUDA(cudaStreamWaitEvent(ctx->stream, op->ev_join, 0));
   for (int k = 0; k < op->n_peers; k++)
      if (op->n_recv[k] > 0) {
         scatter_idx_kernel<<<blocks_for(op->n_recv[k], 256), 256, 0, ctx->stream>>>(
            op->recv_buf[k], op->recv_idx[k], op->n_recv[k], p);
         ctx->launched();
      }
   TFEM_CUDA(cudaGetLastError());
}

tfem_operator *operator_csr(tfem_ctx *ctx, int64_t n, const int32_t *rowptr, const int32_t *cols,
                            const double *vals)
{
   if (n < 1) invalid("operator_create_csr: empty matrix");
   auto *op = new tfem_operator;
   op->ctx = ctx;
   op->csr = true;
   op->n = n;
   const int64_t nnz = rowptr[n];
   op->rowptr = dalloc<int32_t>(n + 1);
   op->cols = dalloc<int32_t>(nnz);
   op->vals = dalloc<double>(nnz);
   h2d(ctx->stream, op->rowptr, rowptr, sizeof(int32_t) * (n + 1));
   h2d(ctx->stream, op->cols, cols, sizeof(int32_t) * nnz);
   h2d(ctx->stream, op->vals, vals, sizeof(double) * nnz);
   return op;
}

void operator_release(tfem_operator *op)
{
   {
      std::lock_guard<std::mutex> lock(workspaces_mu());
      workspaces().erase(op);
   }
   free_nccl_buffers(op);
   for (int k = 0; k < op->n_peers; k++) {
      cudaFree(op->send_idx[k]);
      cudaFree(op->recv_idx[k]);
   }
   cudaFree(op->ess);
   cudaFree(op->ess_mask);
   cudaFree(op->elem_ess);
   cudaFree(op->notown);
   cudaFree(op->rowptr);
   cudaFree(op->cols);
   cudaFree(op->vals);
   cudaFree(op->xl);
   cudaFree(op->yl);
   delete op;
}

// mult_true / ConstrainedOperator::mult (forms.cpp:173-184, 527-543): the
// integrators in insertion order, the first overwriting y, later ones
// accumulating; essential DOFs masked on input for all and overwritten on
// output by the last (which also produces the fused x . y partials).
void operator_mult(tfem_ctx *ctx, const tfem_operator *op, const double *x, double *y,
                   const DotSink *dot_elem, const DotSink *dot_scatter, const int *done)
{
   if (op->csr) {
      csr_kernel<<<blocks_for(op->n, kVecThreads), kVecThreads, 0, ctx->stream>>>(
         op->rowptr, op->cols, op->vals, op->n, x, y, dot_elem ? *dot_elem : DotSink{}, done);
      ctx->launched();
      TFEM_CUDA(cudaGetLastError());
      return;
   }
   if (op->P) {
      // y_T = P^T (sum_i A_i) P x_T with the constraints on the true level:
      // x_L = P (x with x[ess] = 0), y_L = the integrators' sum, then
      // y_T = P^T y_L, y[ess] = x[ess] and the x . y partials
      // (forms.cpp:164-190, 534-542)
      prolongation_mult(ctx, op->P, x, op->ess_mask, op->xl, done);
      for (size_t k = 0; k < op->pa.size(); k++) {
         ApplyFlags f;
         f.overwrite = (k == 0);
         f.done = done;
         pa_apply(ctx, op->pa[k], op->r, op->xl, op->yl, f);
      }
      prolongation_mult_transpose(ctx, op->P, op->yl, y, x, op->ess_mask, dot_elem, done);
      return;
   }
   for (size_t k = 0; k < op->pa.size(); k++) {
      ApplyFlags f;
      f.overwrite = (k == 0);
      f.mask_in = op->ess_mask;
      f.elem_ess = op->elem_ess;
      const bool last = (k + 1 == op->pa.size());
      f.ess_out = last ? op->ess_mask : nullptr;
      f.notown = op->notown;
      if (last && dot_elem) f.dot = *dot_elem;
      if (last && dot_scatter) f.dot_scatter = *dot_scatter;
      f.done = done;
      pa_apply(ctx, op->pa[k], op->r, x, y, f);
   }
}

void operator_diagonal(tfem_ctx *ctx, const tfem_operator *op, double *diag)
{
   if (op->csr) invalid("operator_diagonal: not available for CSR operators");
   // diagonal_true (forms.cpp:545-557): each integrator's diagonal from zero,
   // then d.axpy(1.0, one) in insertion order.
   vec_fill(ctx, diag, op->n, 0.0);
   auto one_diag = [&](const tfem_pa *pa, double *d) {
      if (op->P) pa_diagonal_p(ctx, pa, op->r, op->P, d);
      else pa_diagonal(ctx, pa, op->r, d);
   };
   if (op->pa.size() == 1) {
      one_diag(op->pa[0], diag);
   } else {
      double *one = dalloc<double>(op->n);
      for (const tfem_pa *pa : op->pa) {
         vec_fill(ctx, one, op->n, 0.0);
         one_diag(pa, one);
         vec_axpy(ctx, 1.0, one, diag, op->n);
      }
      TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
      cudaFree(one);
   }
   if (op->n_ess > 0) {
      set_values_kernel<<<blocks_for(op->n_ess, 256), 256, 0, ctx->stream>>>(op->ess, op->n_ess,
                                                                            1.0, diag);
      ctx->launched();
   }
   TFEM_CUDA(cudaGetLastError());
   TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
}

void cg_solve(tfem_ctx *ctx, const tfem_operator *op, const double *b, double rel_tol,
              int max_iters, const double *diag, double *x, tfem_cg_result *res,
              tfem_cg_callback cb, void *user, double *seg_us)
{
   const int64_t n = op->n;
   res->iterations = 0;
   res->converged = 0;
   res->final_norm = 0.0;
   res->initial_norm = 0.0;
   res->x_norm = 0.0;
   if (diag) { // solvers.cpp:19-29
      int *bad = dalloc<int>(1);
      TFEM_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
      diag_check_kernel<<<vec_blocks(ctx, n), kVecThreads, 0, ctx->stream>>>(diag, n, bad);
      ctx->launched();
      int hb = 0;
      TFEM_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
      cudaFree(bad);
      if (hb) invalid("cg_solve: Jacobi diagonal must be strictly positive");
   }
   Workspace &w = workspace_for(ctx, op);
   const bool comm = op->has_comm;
   const double bnorm = std::sqrt(vec_dot(ctx, b, b, n, comm ? op : nullptr));
   res->initial_norm = bnorm;
   if (!std::isfinite(bnorm)) runtime("cg_solve: right-hand side is not finite");
   if (bnorm == 0.0) { // solvers.cpp:37-41
      vec_fill(ctx, x, n, 0.0);
      TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
      res->converged = 1;
      return;
   }
   CgState init{};
   init.target = rel_tol * bnorm;
   init.max_iters = max_iters;
   TFEM_CUDA(cudaMemcpyAsync(w.st, &init, sizeof(CgState), cudaMemcpyHostToDevice, ctx->stream));
   const unsigned vb = vec_blocks(ctx, n);
   cg_init_kernel<<<vb, kVecThreads, 0, ctx->stream>>>(b, diag, n, w.r, w.p, x, w.s_vec.s,
                                                       op->notown);
   if (comm) {
      fold_to_kernel<<<1, kVecThreads, 0, ctx->stream>>>(w.s_vec.s.chunks, w.s_vec.nch, nullptr,
                                                         0, 2, op->red);
      comm_allreduce(ctx, op, 2);
      red_init_kernel<<<1, 1, 0, ctx->stream>>>(op->red, w.st);
   } else {
      cg_init_finish_kernel<<<1, kVecThreads, 0, ctx->stream>>>(w.s_vec.s.chunks, w.s_vec.nch,
                                                                w.st);
   }
   ctx->launched(comm ? 3 : 2);
   TFEM_CUDA(cudaGetLastError());
   const XBufs xb{{x, w.xa, w.xb}};

   // Distributed iteration: the same kernels with the rank-local folds
   // summed over ranks (NCCL allreduce or the hook); p's halo is valid on
   // entry (the initial update below, then halo_direction at the end of
   // every iteration).
   if (comm) halo_exchange(ctx, op, w.p);
   auto dist_iteration = [&]() {
      operator_mult(ctx, op, w.p, w.q, &w.s_elem.s, w.s_scatter.grid ? &w.s_scatter.s : nullptr,
                    &w.st->done);
      fold_to_kernel<<<1, kVecThreads, 0, ctx->stream>>>(w.s_elem.s.chunks, w.s_elem.nch,
                                                         w.s_scatter.s.chunks, w.s_scatter.nch,
                                                         1, op->red);
      comm_allreduce(ctx, op, 1);
      red_alpha_kernel<<<1, 1, 0, ctx->stream>>>(op->red, w.st);
      cg_update_kernel<<<vb, kVecThreads, 0, ctx->stream>>>(w.st, w.q, w.r, diag, n, w.s_vec.s,
                                                            op->notown);
      fold_to_kernel<<<1, kVecThreads, 0, ctx->stream>>>(w.s_vec.s.chunks, w.s_vec.nch, nullptr,
                                                         0, 2, op->red);
      comm_allreduce(ctx, op, 2);
      red_beta_kernel<<<1, 1, 0, ctx->stream>>>(op->red, w.st);
      ctx->launched(5);
      halo_direction(ctx, op, w.st, xb, w.r, diag, w.p, n, w.dir_ticket);
   };

   auto read_state = [&]() {
      TFEM_CUDA(cudaMemcpyAsync(w.host_st, w.st, sizeof(CgState), cudaMemcpyDeviceToHost,
                                ctx->stream));
      TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
      return *w.host_st;
   };

   CgState hs = read_state();
   if (max_iters <= 0 && !hs.done) {
      // for-loop never runs (solvers.cpp:60, 89-96): x = best = 0
      res->iterations = max_iters;
      res->final_norm = res->x_norm = hs.rnorm;
      return;
   }
   if (cb) {
      std::vector<double> hx(n);
      while (!hs.done) {
         if (comm) dist_iteration();
         else enqueue_iteration(ctx, op, w, xb, diag);
         hs = read_state();
         if (hs.status == 0 && hs.it > 0) {
            d2h(ctx->stream, hx.data(), xb.x[hs.cur], sizeof(double) * n);
            cb(hs.it, hx.data(), n, user);
         }
      }
   } else if (comm && !op->nccl) {
      // Host hooks (e.g. gloo tests): eager, the hooks enqueue communication
      // on the stream.  All ranks see the same scalars, hence the same stop
      // decision at the same batch.
      while (!hs.done) {
         for (int k = 0; k < 8; k++) dist_iteration();
         hs = read_state();
      }
   } else if (seg_us) {
      // Diagnostics: eager iterations with events between the launches.
      cudaEvent_t ev[4];
      for (auto &e : ev) TFEM_CUDA(cudaEventCreate(&e));
      double acc[3] = {0, 0, 0};
      int nit = 0;
      constexpr int kSkip = 4; // warm-up iterations left out of the averages
      while (!hs.done) {
         for (int k = 0; k < 16 && nit < max_iters; k++) {
            TFEM_CUDA(cudaEventRecord(ev[0], ctx->stream));
            enqueue_iteration(ctx, op, w, xb, diag, ev);
            TFEM_CUDA(cudaEventSynchronize(ev[3]));
            float t[3];
            for (int j = 0; j < 3; j++) TFEM_CUDA(cudaEventElapsedTime(&t[j], ev[j], ev[j + 1]));
            if (nit >= kSkip)
               for (int j = 0; j < 3; j++) acc[j] += t[j];
            nit++;
         }
         hs = read_state();
      }
      const int n = nit > kSkip ? nit - kSkip : 1;
      for (int j = 0; j < 3; j++) seg_us[j] = 1e3 * acc[j] / n;
      for (auto &e : ev) cudaEventDestroy(e);
   } else {
      // Batches of iterations as one graph; the batch length keeps the
      // per-batch host round trip small against the work it covers.  A
      // distributed (NCCL) iteration is captured the same way -- its
      // collectives are stream-ordered NCCL calls; its first batch runs
      // eagerly so NCCL's lazy connection setup never happens under capture.
      // Every rank reads the same scalars, so all replay the same batches.
      const int batch = 16;
      auto iteration = [&]() {
         if (comm) dist_iteration();
         else enqueue_iteration(ctx, op, w, xb, diag);
      };
      if (comm && !w.graph && !hs.done) {
         for (int k = 0; k < batch; k++) iteration();
         hs = read_state();
      }
      if (!w.graph || w.g_diag != diag || w.g_x != x || w.g_batch != batch ||
          w.g_numerics != ctx->numerics) {
         if (w.graph) {
            cudaGraphExecDestroy(w.graph);
            w.graph = nullptr;
         }
         cudaGraph_t g;
         const int64_t before = ctx->launches;
         TFEM_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
         for (int k = 0; k < batch; k++) iteration();
         TFEM_CUDA(cudaStreamEndCapture(ctx->stream, &g));
         w.g_launches = ctx->launches - before;
         ctx->launches = before;
         TFEM_CUDA(cudaGraphInstantiate(&w.graph, g, 0));
         cudaGraphDestroy(g);
         w.g_diag = diag;
         w.g_x = x;
         w.g_batch = batch;
         w.g_numerics = ctx->numerics;
      }
      while (!hs.done) {
         TFEM_CUDA(cudaGraphLaunch(w.graph, ctx->stream));
         ctx->launched(w.g_launches);
         hs = read_state();
      }
   }
   if (hs.status == 1) runtime("cg_solve: breakdown (non-finite step)");
   if (hs.status == 2) runtime("cg_solve: breakdown (non-finite residual)");
   res->iterations = hs.iterations;
   res->converged = hs.converged;
   res->final_norm = hs.rnorm;
   res->x_norm = hs.converged ? hs.rnorm : hs.best_rnorm;
   const int pick = hs.converged ? hs.cur : hs.best; // solvers.cpp:89-96
   if (xb.x[pick] != x) {
      TFEM_CUDA(cudaMemcpyAsync(x, xb.x[pick], sizeof(double) * n, cudaMemcpyDeviceToDevice,
                                ctx->stream));
      TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   }
}

} // namespace tfem
