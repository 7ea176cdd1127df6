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
// in order.  Bt(q, i) / Gt(q, i) are the 1D tables, D(c, q) the element's
// point factors; both kernels below run this one expression.
template <int DIM, class TB, class TG, class TD>
__device__ __forceinline__ double diag_sum(int kind, int nq, int nqd, int ia, int ib, int ic,
                                           TB Bt, TG Gt, TD D)
{
   double s = 0.0;
   for (int q = 0; q < nqd; q++) {
      const int qx = q % nq, qy = (q / nq) % nq, qz = q / (nq * nq);
      if (DIM == 2) {
         if (kind == TFEM_MASS) {
            const double b = __dmul_rn(Bt(qx, ia), Bt(qy, ib));
            s = __dadd_rn(s, __dmul_rn(__dmul_rn(b, b), D(0, q)));
         } else {
            const double gx = __dmul_rn(Gt(qx, ia), Bt(qy, ib));
            const double gy = __dmul_rn(Bt(qx, ia), Gt(qy, ib));
            const double term =
               __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(gx, gx), D(0, q)),
                                   __dmul_rn(__dmul_rn(__dmul_rn(2.0, gx), gy), D(1, q))),
                         __dmul_rn(__dmul_rn(gy, gy), D(2, q)));
            s = __dadd_rn(s, term);
         }
      } else {
         const double Bx = Bt(qx, ia), By = Bt(qy, ib), Bz = Bt(qz, ic);
         const double Gx = Gt(qx, ia), Gy = Gt(qy, ib), Gz = Gt(qz, ic);
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
   return s;
}

__device__ __forceinline__ void diag_out(double s, int64_t slot, int64_t ev, const uint32_t *gmap,
                                         double *evec, double *y)
{
   const uint32_t g = gmap[slot];
   if (is_exclusive(g)) {
      const uint32_t d = g & kDofMask;
      y[d] = __dadd_rn(y[d], s);
   } else {
      evec[ev] = s;
   }
}

// Planes layout (2D p <= 3): a thread per element position, i uniform per
// block row (blockIdx.y) so the 1D-table reads are warp-uniform constant-bank
// loads and the point-factor reads are coalesced across elements.
__global__ void diag_planes_kernel(const Tables t, int p, int nq, int kind, int64_t ne,
                                   int64_t ne_pad, const double *__restrict__ qdata,
                                   const uint32_t *gmap, double *evec, double *y)
{
   const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; // position
   const int i = blockIdx.y;
   if (e >= ne) return;
   const int D1 = p + 1, nqd = nq * nq;
   const int ncomp = kind == TFEM_MASS ? 1 : 3;
   const double s = diag_sum<2>(
      kind, nq, nqd, i % D1, i / D1, 0, [&](int q, int k) { return t.B[q][k]; },
      [&](int q, int k) { return t.G[q][k]; },
      [&](int c, int q) { return __ldg(qdata + qdata_index(0, e, c, q, ncomp, nqd, nq, ne_pad)); });
   const int64_t slot = (int64_t)i * ne_pad + e;
   diag_out(s, slot, slot, gmap, evec, y);
}

// Element-major layout (3D, 2D p >= 4): a block per epb elements stages
// their point factors ([e][c][q], contiguous) in shared memory with coalesced
// loads -- each factor is read from HBM once, not once per local DOF -- and
// a thread per (element, i) sums over the points from there.  Elements whose
// factors exceed the budget (3D q >= 13) read them from global memory
// (staged = 0, one element per block: the block's loads of a factor coincide).
constexpr int kDiagThreads = 256;
constexpr size_t kDiagSmemMax = 96 * 1024;

template <int DIM>
__global__ void __launch_bounds__(kDiagThreads)
diag_em_kernel(const Tables t, int p, int nq, int kind, int64_t ne, int epb, int staged,
               const double *__restrict__ qdata, const uint32_t *gmap, const uint16_t *evperm,
               double *evec, double *y)
{
   extern __shared__ double sq[]; // [epb][ncomp][nqd]
   __shared__ double sB[kMaxQ * (kMaxP + 1)], sG[kMaxQ * (kMaxP + 1)];
   const int D1 = p + 1;
   const int nd = DIM == 2 ? D1 * D1 : D1 * D1 * D1;
   const int nqd = DIM == 2 ? nq * nq : nq * nq * nq;
   const int ncomp = kind == TFEM_MASS ? 1 : (DIM == 2 ? 3 : 6);
   const int per = ncomp * nqd;
   for (int j = threadIdx.x; j < nq * D1; j += blockDim.x) {
      sB[j] = t.B[j / D1][j % D1];
      sG[j] = t.G[j / D1][j % D1];
   }
   const int64_t e0 = blockIdx.x * (int64_t)epb;
   const int cnt = static_cast<int>(ne - e0 < epb ? ne - e0 : epb);
   const double *src = qdata + e0 * per;
   if (staged)
      for (int j = threadIdx.x; j < cnt * per; j += blockDim.x) sq[j] = __ldg(src + j);
   __syncthreads();
   for (int w = threadIdx.x; w < cnt * nd; w += blockDim.x) {
      const int el = w / nd, i = w % nd;
      const double *qd = (staged ? sq : src) + el * per;
      const double s = diag_sum<DIM>(
         kind, nq, nqd, i % D1, (i / D1) % D1, i / (D1 * D1),
         [&](int q, int k) { return sB[q * D1 + k]; }, [&](int q, int k) { return sG[q * D1 + k]; },
         [&](int c, int q) { return qd[c * nqd + q]; });
      const int64_t e = e0 + el;
      diag_out(s, e * nd + i, ev_em_p(evperm, nd, e, i), gmap, evec, y);
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
   if (!pa->elem_major()) {
      const int T = 128;
      const dim3 grid(blocks_for(pa->npos, T), r->nd);
      diag_planes_kernel<<<grid, T, 0, ctx->stream>>>(t, pa->p, pa->nq, pa->kind, pa->npos,
                                                      pa->ne_pad, pa->qdata, r->gmap, evec, diag);
   } else {
      const size_t per = sizeof(double) * pa->ncomp * pa->nqd;
      const int staged = per <= kDiagSmemMax ? 1 : 0;
      int epb = std::max(1, kDiagThreads / r->nd);
      epb = staged ? static_cast<int>(std::min<size_t>(epb, kDiagSmemMax / per)) : 1;
      const size_t smem = staged ? per * epb : 0;
      const unsigned grid = blocks_for(pa->npos, epb);
      if (pa->dim == 2) {
         max_dynamic_smem((const void *)diag_em_kernel<2>, kDiagSmemMax);
         diag_em_kernel<2><<<grid, kDiagThreads, smem, ctx->stream>>>(
            t, pa->p, pa->nq, pa->kind, pa->npos, epb, staged, pa->qdata, r->gmap, r->evperm, evec, diag);
      } else {
         max_dynamic_smem((const void *)diag_em_kernel<3>, kDiagSmemMax);
         diag_em_kernel<3><<<grid, kDiagThreads, smem, ctx->stream>>>(
            t, pa->p, pa->nq, pa->kind, pa->npos, epb, staged, pa->qdata, r->gmap, r->evperm, evec, diag);
      }
   }
   ctx->launched();
   TFEM_CUDA(cudaGetLastError());
   if (r->n_shared > 0)
      scatter_shared(ctx, r, evec, nullptr, diag, false, nullptr, nullptr, nullptr, true);
}

} // namespace tfem
