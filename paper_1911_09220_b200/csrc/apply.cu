// K3 / K4 and the K2 dispatch: the deterministic shared-DOF scatter, the
// exact diagonal, and pa_apply / pa_diagonal (forms.cpp:231-382).
//
// Element kernels (apply2d_reg.cu, apply_grp.cu) write DOFs owned by one
// element ("exclusive") straight to y and the others to the E-vector;
// scatter_kernel then sums each shared DOF's slots in ascending element order
// (forms.cpp:289-295) -- deterministic, no atomics.
#include "kernels.cuh"

namespace tfem {

namespace {

constexpr int kScatterThreads = 256;

inline unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

// --------------------------------------------------------------- scatter
// Shared DOFs: y[d] (+)= sum of E-vector slots in ascending element order,
// essential overwrite and the fused x . y partial.
template <bool EXACT>
__global__ void __launch_bounds__(kScatterThreads)
scatter_kernel(const int32_t *__restrict__ dofs, const int32_t *__restrict__ off,
               const uint32_t *__restrict__ slots, int64_t n_shared,
               const double *__restrict__ evec, const double *__restrict__ x, double *y,
               int overwrite, const uint32_t *ess_out, double *partials, const int *done)
{
   if (done && *done) return;
   const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   double dot = 0.0;
   if (s < n_shared) {
      const int32_t d = __ldg(dofs + s);
      const int beg = __ldg(off + s), end = __ldg(off + s + 1);
      double acc = __ldg(evec + __ldg(slots + beg));
      if (!overwrite) acc = add<EXACT>(y[d], acc);
      for (int k = beg + 1; k < end; k++) acc = add<EXACT>(acc, __ldg(evec + __ldg(slots + k)));
      if (ess_out && bit_set(ess_out, d)) acc = __ldg(x + d);
      y[d] = acc;
      if (partials) dot = mul<EXACT>(__ldg(x + d), acc);
   }
   if (partials) {
      const double t = block_sum<kScatterThreads>(dot);
      if (threadIdx.x == 0) partials[blockIdx.x] = t;
   }
}

// -------------------------------------------------------------- diagonal
// Exact diagonal with the dense tabulated tables of pa_diagonal
// (forms.cpp:22-42, 334-347): per (element, local DOF i) sum over the points
// in order.  i is uniform per block row (blockIdx.y) so the 1D-table reads
// are warp-uniform constant-bank loads.
template <int DIM>
__global__ void diag_kernel(const Tables t, int p, int nq, int kind, int64_t ne, int64_t ne_pad,
                            const double *__restrict__ qdata, const uint32_t *gmap,
                            int elem_major, double *evec, double *y)
{
   const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   const int i = blockIdx.y;
   if (e >= ne) return;
   const int D1 = p + 1;
   const int nd = DIM == 2 ? D1 * D1 : D1 * D1 * D1;
   const int nqd = DIM == 2 ? nq * nq : nq * nq * nq;
   const int ncomp = kind == TFEM_MASS ? 1 : (DIM == 2 ? 3 : 6);
   const int ia = i % D1, ib = (i / D1) % D1, ic = i / (D1 * D1);
   // qdata addressing follows the map layout (elem_major_layout)
   auto D = [&](int c, int q) -> double {
      return elem_major ? __ldg(qdata + (e * ncomp + c) * (int64_t)nqd + q)
                        : __ldg(qdata + (int64_t)(c * nqd + q) * ne_pad + e);
   };
   double s = 0.0;
   for (int q = 0; q < nqd; q++) {
      const int qx = q % nq, qy = (q / nq) % nq, qz = q / (nq * nq);
      if (DIM == 2) {
         if (kind == TFEM_MASS) {
            const double b = __dmul_rn(t.B[qx][ia], t.B[qy][ib]);
            s = __dadd_rn(s, __dmul_rn(__dmul_rn(b, b), D(0, q)));
         } else {
            const double gx = __dmul_rn(t.G[qx][ia], t.B[qy][ib]);
            const double gy = __dmul_rn(t.B[qx][ia], t.G[qy][ib]);
            const double term =
               __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(gx, gx), D(0, q)),
                                   __dmul_rn(__dmul_rn(__dmul_rn(2.0, gx), gy), D(1, q))),
                         __dmul_rn(__dmul_rn(gy, gy), D(2, q)));
            s = __dadd_rn(s, term);
         }
      } else {
         const double Bx = t.B[qx][ia], By = t.B[qy][ib], Bz = t.B[qz][ic];
         const double Gx = t.G[qx][ia], Gy = t.G[qy][ib], Gz = t.G[qz][ic];
         if (kind == TFEM_MASS) {
            const double b = __dmul_rn(__dmul_rn(Bx, By), Bz);
            s = __dadd_rn(s, __dmul_rn(__dmul_rn(b, b), D(0, q)));
         } else {
            const double g0 = __dmul_rn(__dmul_rn(Gx, By), Bz);
            const double g1 = __dmul_rn(__dmul_rn(Bx, Gy), Bz);
            const double g2 = __dmul_rn(__dmul_rn(Bx, By), Gz);
            double term = __dmul_rn(__dmul_rn(g0, g0), D(0, q));
            term = __dadd_rn(term, __dmul_rn(__dmul_rn(__dmul_rn(2.0, g0), g1), D(1, q)));
            term = __dadd_rn(term, __dmul_rn(__dmul_rn(__dmul_rn(2.0, g0), g2), D(2, q)));
            term = __dadd_rn(term, __dmul_rn(__dmul_rn(g1, g1), D(3, q)));
            term = __dadd_rn(term, __dmul_rn(__dmul_rn(__dmul_rn(2.0, g1), g2), D(4, q)));
            term = __dadd_rn(term, __dmul_rn(__dmul_rn(g2, g2), D(5, q)));
            s = __dadd_rn(s, term);
         }
      }
   }
   const int64_t slot = elem_major ? e * nd + i : (int64_t)i * ne_pad + e;
   const uint32_t g = gmap[slot];
   if (g & kExclusive) {
      const uint32_t d = g & kDofMask;
      y[d] = __dadd_rn(y[d], s);
   } else {
      evec[slot] = s;
   }
}

Tables tables_of(const tfem_pa *pa)
{
   Tables t{};
   const int D1 = pa->p + 1;
   for (int q = 0; q < pa->nq; q++)
      for (int i = 0; i < D1; i++) {
         t.B[q][i] = pa->B[q * D1 + i];
         t.G[q][i] = pa->G[q * D1 + i];
      }
   return t;
}

KernelPick pick(const tfem_ctx *ctx, const tfem_pa *pa)
{
   const bool exact = pa->dim == 2 && ctx->numerics == TFEM_NUMERICS_REFERENCE;
   KernelPick k = (pa->dim == 2 && pa->p <= 3) ? pick_apply2d_reg(pa->p, pa->nq, pa->kind, exact)
                                               : pick_apply_grp(pa->dim, pa->p, pa->nq, pa->kind, exact);
   if (!k.launch) invalid("pa_apply: unsupported (order, points) pair on the device");
   return k;
}

unsigned elem_blocks(const KernelPick &k, int64_t ne) { return blocks_for(ne, k.elems_per_block); }

} // namespace

int64_t pa_apply_partials(const tfem_pa *pa, const tfem_restriction *r)
{
   return elem_blocks(pick(pa->ctx, pa), pa->ne) + blocks_for(r->n_shared, kScatterThreads);
}

int64_t pa_apply(tfem_ctx *ctx, const tfem_pa *pa, const tfem_restriction *r, const double *x,
                 double *y, const ApplyFlags &f)
{
   if (pa->dim != r->dim || pa->p != r->p || pa->ne != r->ne)
      invalid("forms: point factors were built for a different space");
   const bool exact = pa->dim == 2 && ctx->numerics == TFEM_NUMERICS_REFERENCE;
   const KernelPick k = pick(ctx, pa);
   ApplyArgs a{};
   a.t = tables_of(pa);
   a.ne = pa->ne;
   a.ne_pad = pa->ne_pad;
   a.nd = r->nd;
   a.gmap = r->gmap;
   a.qdata = pa->qdata;
   a.x = x;
   a.y = y;
   a.evec = r->n_shared > 0 ? const_cast<tfem_restriction *>(r)->ensure_evec() : nullptr;
   a.overwrite = f.overwrite ? 1 : 0;
   a.mask_in = f.mask_in;
   a.ess_out = f.ess_out;
   a.partials = f.dot_partials;
   a.done = f.done;
   const unsigned nb = elem_blocks(k, pa->ne);
   k.launch(a, ctx->stream, nb);
   ctx->launched();
   TFEM_CUDA(cudaGetLastError());
   int64_t n_part = nb;
   if (r->n_shared > 0) {
      const unsigned sb = blocks_for(r->n_shared, kScatterThreads);
      double *sp = f.dot_partials ? f.dot_partials + nb : nullptr;
      if (exact)
         scatter_kernel<true><<<sb, kScatterThreads, 0, ctx->stream>>>(
            r->shared_dofs, r->shared_off, r->shared_slots, r->n_shared, a.evec, x, y,
            a.overwrite, f.ess_out, sp, f.done);
      else
         scatter_kernel<false><<<sb, kScatterThreads, 0, ctx->stream>>>(
            r->shared_dofs, r->shared_off, r->shared_slots, r->n_shared, a.evec, x, y,
            a.overwrite, f.ess_out, sp, f.done);
      ctx->launched();
      TFEM_CUDA(cudaGetLastError());
      n_part += sb;
   }
   return n_part;
}

void pa_diagonal(tfem_ctx *ctx, const tfem_pa *pa, const tfem_restriction *r, double *diag)
{
   if (pa->dim != r->dim || pa->p != r->p || pa->ne != r->ne)
      invalid("forms: point factors were built for a different space");
   const Tables t = tables_of(pa);
   double *evec = r->n_shared > 0 ? const_cast<tfem_restriction *>(r)->ensure_evec() : nullptr;
   const int T = 128;
   dim3 grid(blocks_for(pa->ne, T), r->nd);
   const int elem_major = pa->elem_major() ? 1 : 0;
   if (pa->dim == 2)
      diag_kernel<2><<<grid, T, 0, ctx->stream>>>(t, pa->p, pa->nq, pa->kind, pa->ne, pa->ne_pad,
                                                 pa->qdata, r->gmap, elem_major, evec, diag);
   else
      diag_kernel<3><<<grid, T, 0, ctx->stream>>>(t, pa->p, pa->nq, pa->kind, pa->ne, pa->ne_pad,
                                                 pa->qdata, r->gmap, elem_major, evec, diag);
   ctx->launched();
   TFEM_CUDA(cudaGetLastError());
   if (r->n_shared > 0) {
      const unsigned sb = blocks_for(r->n_shared, kScatterThreads);
      scatter_kernel<true><<<sb, kScatterThreads, 0, ctx->stream>>>(
         r->shared_dofs, r->shared_off, r->shared_slots, r->n_shared, evec, nullptr, diag, 0,
         nullptr, nullptr, nullptr);
      ctx->launched();
      TFEM_CUDA(cudaGetLastError());
   }
}

} // namespace tfem
