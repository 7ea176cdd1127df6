// K3 / K4 and the K2 dispatch: the deterministic shared-DOF scatter, the
// exact diagonal, and pa_apply / pa_diagonal (forms.cpp:231-382).
//
// Element kernels (apply2d_tma.cu 2D p<=3, apply2d_hi.cu 2D p>=4,
// apply3d_tma.cu 3D q<=7, apply_grp.cu otherwise; apply2d_reg.cu for A/B)
// write DOFs owned by one element ("exclusive") straight to y -- the 2D p<=3
// kernel also sums warp-local shared DOFs itself -- and the others to the
// E-vector; scatter_kernel then sums each remaining shared DOF's slots in
// ascending element order (forms.cpp:289-295) -- deterministic, no atomics.
#include "kernels.cuh"

#include <algorithm>
#include <cstdlib>
#include <string>

namespace tfem {

namespace {

constexpr int kScatterThreads = 256;
constexpr int kScatterRows = 4;      // rows per thread: all their loads in flight together
constexpr int kScatterMinBlocks = 4; // <= 64 registers: occupancy for the gathers (+1-2 %)

inline unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

// --------------------------------------------------------------- scatter
// Shared DOFs, one thread per DOF, bucketed by slot count c (ELL rows, one
// vector load for the row): y[d] (+)= sum of its E-vector slots in ascending
// element order, y[ess] = x[ess], fused x . y partial.  One launch covers all
// buckets; each block belongs to one bucket (uniform switch).
struct BucketArgs {
   int nb;
   int c[tfem_restriction::kMaxBuckets];
   int64_t n[tfem_restriction::kMaxBuckets];
   const int32_t *dofs[tfem_restriction::kMaxBuckets];
   const uint32_t *slots[tfem_restriction::kMaxBuckets];
   int64_t start[tfem_restriction::kMaxBuckets + 1]; // first block of each bucket
};

template <int C>
__device__ __forceinline__ void load_row(const uint32_t *__restrict__ row, uint32_t (&sl)[C])
{
   if constexpr (C == 2) {
      const uint2 v = __ldg(reinterpret_cast<const uint2 *>(row));
      sl[0] = v.x;
      sl[1] = v.y;
   } else if constexpr (C == 4 || C == 8) {
#pragma unroll
      for (int k = 0; k < C; k += 4) {
         const uint4 v = __ldg(reinterpret_cast<const uint4 *>(row) + k / 4);
         sl[k] = v.x;
         sl[k + 1] = v.y;
         sl[k + 2] = v.z;
         sl[k + 3] = v.w;
      }
   } else {
#pragma unroll
      for (int k = 0; k < C; k++) sl[k] = __ldg(row + k);
   }
}

// Rows s0 + k * kScatterThreads (k < kScatterRows) of bucket b: every load
// of the rows is issued before the first sum.
template <bool EXACT, int C>
__device__ __forceinline__ double scatter_rows(const BucketArgs &B, int b, int64_t s0,
                                               const double *__restrict__ evec,
                                               const double *__restrict__ x, double *y,
                                               int overwrite, const uint32_t *ess_out,
                                               bool want_dot, const uint32_t *notown, bool ess_only)
{
   constexpr int R = kScatterRows;
   const int64_t n = B.n[b];
   int32_t d[R];
   uint32_t sl[R][C];
   double v[R][C];
   uint32_t ew[R];
#pragma unroll
   for (int k = 0; k < R; k++) {
      const int64_t s = s0 + k * kScatterThreads;
      if (s < n) {
         d[k] = __ldg(B.dofs[b] + s);
         load_row<C>(B.slots[b] + s * C, sl[k]);
      }
   }
#pragma unroll
   for (int k = 0; k < R; k++) {
      if (s0 + k * kScatterThreads >= n) continue;
#pragma unroll
      for (int c = 0; c < C; c++) v[k][c] = __ldg(evec + sl[k][c]);
      ew[k] = ess_out ? __ldg(ess_out + (static_cast<uint32_t>(d[k]) >> 5)) : 0u;
   }
   double dv = 0.0;
#pragma unroll
   for (int k = 0; k < R; k++) {
      if (s0 + k * kScatterThreads >= n) continue;
      double acc = overwrite ? v[k][0] : add<EXACT>(y[d[k]], v[k][0]);
#pragma unroll
      for (int c = 1; c < C; c++) acc = add<EXACT>(acc, v[k][c]);
      const bool es = (ew[k] >> (d[k] & 31)) & 1u;
      if (es) acc = __ldg(x + d[k]);
      y[d[k]] = acc;
      // ess_only: the element kernel took x . y as element energies; only
      // the essential DOFs' x_d^2 is missing
      if (ess_only) {
         if (want_dot && es) dv = add<EXACT>(dv, mul<EXACT>(acc, acc));
      } else if (want_dot && !(notown && bit_set(notown, d[k]))) {
         dv = add<EXACT>(dv, mul<EXACT>(__ldg(x + d[k]), acc));
      }
   }
   return dv;
}

template <bool EXACT>
__global__ void __launch_bounds__(kScatterThreads, kScatterMinBlocks)
scatter_kernel(const BucketArgs B, const double *__restrict__ evec, const double *__restrict__ x,
               double *y, int overwrite, const uint32_t *ess_out, DotSink dot, const int *done,
               const uint32_t *notown, int ess_only)
{
   if (done && *done) return;
   int b = 0;
   while (b + 1 < B.nb && (int64_t)blockIdx.x >= B.start[b + 1]) b++;
   const int64_t s = ((int64_t)blockIdx.x - B.start[b]) * (kScatterThreads * kScatterRows) +
                     threadIdx.x;
   double dv = 0.0;
   if (s < B.n[b]) {
      const bool wd = static_cast<bool>(dot), eo = ess_only != 0;
      switch (B.c[b]) {
      case 2: dv = scatter_rows<EXACT, 2>(B, b, s, evec, x, y, overwrite, ess_out, wd, notown, eo); break;
      case 3: dv = scatter_rows<EXACT, 3>(B, b, s, evec, x, y, overwrite, ess_out, wd, notown, eo); break;
      case 4: dv = scatter_rows<EXACT, 4>(B, b, s, evec, x, y, overwrite, ess_out, wd, notown, eo); break;
      case 5: dv = scatter_rows<EXACT, 5>(B, b, s, evec, x, y, overwrite, ess_out, wd, notown, eo); break;
      case 6: dv = scatter_rows<EXACT, 6>(B, b, s, evec, x, y, overwrite, ess_out, wd, notown, eo); break;
      case 7: dv = scatter_rows<EXACT, 7>(B, b, s, evec, x, y, overwrite, ess_out, wd, notown, eo); break;
      case 8: dv = scatter_rows<EXACT, 8>(B, b, s, evec, x, y, overwrite, ess_out, wd, notown, eo); break;
      }
   }
   if (dot) {
      const double v[1] = {dv};
      emit<kScatterThreads, 1>(dot, v);
   }
}

BucketArgs bucket_args(const tfem_restriction *r, bool global_only)
{
   const int nb = global_only ? r->n_gbuckets : r->n_buckets;
   const tfem_restriction::Bucket *bk = global_only ? r->gbuckets : r->buckets;
   BucketArgs B{};
   B.nb = nb;
   int64_t blk = 0;
   for (int b = 0; b < nb; b++) {
      B.c[b] = bk[b].c;
      B.n[b] = bk[b].n;
      B.dofs[b] = bk[b].dofs;
      B.slots[b] = bk[b].slots;
      B.start[b] = blk;
      blk += blocks_for(bk[b].n, kScatterThreads * kScatterRows);
   }
   B.start[nb] = blk;
   return B;
}

// -------------------------------------------------------------- diagonal
// Exact diagonal with the dense tabulated tables of pa_diagonal
// (forms.cpp:22-42, 334-347): per (element, local DOF i) sum over the points
// in order.  i is uniform per block row (blockIdx.y) so the 1D-table reads
// are warp-uniform constant-bank loads.
template <int DIM>
__global__ void diag_kernel(const Tables t, int p, int nq, int kind, int64_t ne, int64_t ne_pad,
                            const double *__restrict__ qdata, int qlayout, const uint32_t *gmap,
                            int elem_major, const uint16_t *evperm, double *evec, double *y)
{
   const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; // position
   const int i = blockIdx.y;
   if (e >= ne) return;
   const int D1 = p + 1;
   const int nd = DIM == 2 ? D1 * D1 : D1 * D1 * D1;
   const int nqd = DIM == 2 ? nq * nq : nq * nq * nq;
   const int ncomp = kind == TFEM_MASS ? 1 : (DIM == 2 ? 3 : 6);
   const int ia = i % D1, ib = (i / D1) % D1, ic = i / (D1 * D1);
   // qdata addressing follows the map layout (elem_major_layout)
   auto D = [&](int c, int q) -> double {
      return __ldg(qdata + qdata_index(qlayout, e, c, q, ncomp, nqd, nq, ne_pad));
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
   if (is_exclusive(g)) {
      const uint32_t d = g & kDofMask;
      y[d] = __dadd_rn(y[d], s);
   } else {
      evec[elem_major ? ev_em_p(evperm, nd, e, i) : (int64_t)i * ne_pad + e] = s;
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
   KernelPick k;
   if (pa->dim == 2 && pa->p <= 3)
      k = pick_apply2d_tma(pa->p, pa->nq, pa->kind, exact, ctx->sm_count);
   else if (pa->dim == 3 &&
            (k = pick_apply3d_tma(pa->p, pa->nq, pa->kind, ctx->sm_count, pa->colloc)).launch)
      ;
   else if (pa->dim == 2 &&
            (k = pick_apply2d_hi(pa->p, pa->nq, pa->kind, exact, ctx->sm_count, pa->colloc)).launch)
      ;
   else
      k = pick_apply_grp(pa->dim, pa->p, pa->nq, pa->kind, exact);
   if (!k.launch) invalid("pa_apply: unsupported (order, points) pair on the device");
   return k;
}

// Persistent kernels: min(work, one block per SM); ctx->max_blocks (a test
// hook, tfem_ctx_set_max_blocks) caps them further so small meshes run many
// laps of every block's pipeline ring.
unsigned elem_blocks(const tfem_ctx *ctx, const KernelPick &k, int64_t ne)
{
   int64_t b = blocks_for(ne, k.elems_per_block);
   if (k.persistent_blocks > 0) {
      b = std::min<int64_t>(b, k.persistent_blocks);
      if (ctx->max_blocks > 0) b = std::min<int64_t>(b, ctx->max_blocks);
   }
   return static_cast<unsigned>(b > 0 ? b : 1);
}

} // namespace

int64_t scatter_grid(const tfem_restriction *r, bool global_only)
{
   const BucketArgs B = bucket_args(r, global_only);
   return B.start[B.nb];
}

int64_t scatter_shared(tfem_ctx *ctx, const tfem_restriction *r, const double *evec,
                       const double *x, double *y, bool overwrite, const uint32_t *ess_out,
                       const DotSink *dot, const int *done, bool exact,
                       const uint32_t *notown, bool global_only, bool ess_only)
{
   const BucketArgs B = bucket_args(r, global_only);
   const int64_t grid = B.start[B.nb];
   if (grid == 0) return 0;
   const DotSink sink = dot ? *dot : DotSink{};
   if (exact)
      scatter_kernel<true><<<(unsigned)grid, kScatterThreads, 0, ctx->stream>>>(
         B, evec, x, y, overwrite ? 1 : 0, ess_out, sink, done, notown, ess_only ? 1 : 0);
   else
      scatter_kernel<false><<<(unsigned)grid, kScatterThreads, 0, ctx->stream>>>(
         B, evec, x, y, overwrite ? 1 : 0, ess_out, sink, done, notown, ess_only ? 1 : 0);
   ctx->launched();
   TFEM_CUDA(cudaGetLastError());
   return grid;
}

// The bulk-copy kernel sums warp-local DOFs itself on ordered spaces.
bool tiled(const KernelPick &k, const tfem_restriction *r) { return k.warp_reduce && r->warp_local; }

void check_pair(const tfem_pa *pa, const tfem_restriction *r)
{
   if (pa->dim != r->dim || pa->p != r->p || pa->ne != r->ne)
      invalid("forms: point factors were built for a different space");
   if (!(pa->order == r->order))
      invalid("forms: point factors and restriction use different element orders (a Cartesian "
              "restriction needs a Cartesian geometry and vice versa)");
}

void pa_apply_grids(const tfem_pa *pa, const tfem_restriction *r, int64_t *g_elem,
                    int64_t *g_scatter)
{
   const KernelPick k = pick(pa->ctx, pa);
   *g_elem = elem_blocks(pa->ctx, k, pa->npos);
   *g_scatter = scatter_grid(r, tiled(k, r));
}

void pa_apply(tfem_ctx *ctx, const tfem_pa *pa, const tfem_restriction *r, const double *x,
              double *y, const ApplyFlags &f)
{
   check_pair(pa, r);
   const bool exact = pa->dim == 2 && ctx->numerics == TFEM_NUMERICS_REFERENCE;
   const KernelPick k = pick(ctx, pa);
   const bool tl = tiled(k, r);
   ApplyArgs a{};
   a.t = tables_of(pa);
   a.ne = pa->npos; // element kernels run over positions (padding included)
   a.ne_pad = pa->ne_pad;
   a.nd = r->nd;
   a.gmap = r->gmap;
   a.qdata = pa->qdata;
   a.x = x;
   a.y = y;
   a.evec = r->needs_evec() ? const_cast<tfem_restriction *>(r)->ensure_evec() : nullptr;
   a.evperm = r->evperm;
   a.overwrite = f.overwrite ? 1 : 0;
   a.mask_in = f.mask_in;
   a.ess_out = f.ess_out;
   a.elem_ess = f.mask_in ? f.elem_ess : nullptr;
   a.notown = f.notown;
   a.warp_local = tl ? 1 : 0;
   const bool edot = k.energy_dot && static_cast<bool>(f.dot) && f.overwrite &&
                     f.mask_in == f.ess_out && !f.notown;
   a.energy_dot = edot ? 1 : 0;
   a.dot = f.dot;
   a.done = f.done;
   k.launch(a, ctx->stream, elem_blocks(ctx, k, pa->npos));
   ctx->launched();
   TFEM_CUDA(cudaGetLastError());
   if (r->n_shared > 0)
      scatter_shared(ctx, r, a.evec, x, y, f.overwrite, f.ess_out,
                     f.dot_scatter ? &f.dot_scatter : nullptr, f.done, exact, f.notown, tl, edot);
}

void pa_diagonal(tfem_ctx *ctx, const tfem_pa *pa, const tfem_restriction *r, double *diag)
{
   check_pair(pa, r);
   const Tables t = tables_of(pa);
   double *evec = r->needs_evec() ? const_cast<tfem_restriction *>(r)->ensure_evec() : nullptr;
   const int T = 128;
   dim3 grid(blocks_for(pa->npos, T), r->nd);
   const int elem_major = pa->elem_major() ? 1 : 0;
   if (pa->dim == 2)
      diag_kernel<2><<<grid, T, 0, ctx->stream>>>(t, pa->p, pa->nq, pa->kind, pa->npos, pa->ne_pad,
                                                 pa->qdata, pa->qlayout, r->gmap, elem_major, r->evperm, evec, diag);
   else
      diag_kernel<3><<<grid, T, 0, ctx->stream>>>(t, pa->p, pa->nq, pa->kind, pa->npos, pa->ne_pad,
                                                 pa->qdata, pa->qlayout, r->gmap, elem_major, r->evperm, evec, diag);
   ctx->launched();
   TFEM_CUDA(cudaGetLastError());
   if (r->n_shared > 0)
      scatter_shared(ctx, r, evec, nullptr, diag, false, nullptr, nullptr, nullptr, true);
}

} // namespace tfem
