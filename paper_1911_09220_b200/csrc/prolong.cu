// Non-conforming spaces on the device: the prolongation P and its transpose
// (FeSpace::prolongation, fespace.cpp:62-72, 166-203; SparseMatrix::mult /
// mult_transpose, sparse.cpp:75-102) and pa_diagonal's constrained-element
// path (forms.cpp:311-382).
//
// P x: one thread per local row, the row's terms in CSR order.  P^T x: the
// transpose CSR built on the host by the reference's own traversal
// (SparseMatrix::transpose, sparse.cpp:104-124), so every true DOF sums its
// local rows in ascending order -- mult_transpose's accumulation order.
//
// Diagonal: every (target, value) contribution of pa_diagonal is generated
// in the reference's order (elements ascending; unconstrained: i ascending;
// constrained: i, j, a, b), stably sorted by target, and each target's run
// summed in sequence -- bit-identical to the serial loop, no atomics.
#include "kernels.cuh"

#include <cub/cub.cuh>

#include <algorithm>
#include <numeric>
#include <vector>

namespace tfem {

namespace {

constexpr int kT = 256;

inline unsigned blocks_for(int64_t n, int t = kT) { return static_cast<unsigned>((n + t - 1) / t); }

template <typename T>
T *dalloc(int64_t n)
{
   T *p = nullptr;
   TFEM_CUDA(cudaMalloc(&p, sizeof(T) * static_cast<size_t>(n > 0 ? n : 1)));
   return p;
}

// y_L = P (x_T with masked entries read as 0)   (SparseMatrix::mult)
template <bool EXACT>
__global__ void __launch_bounds__(kT)
p_mult_kernel(const int32_t *__restrict__ rowptr, const int32_t *__restrict__ cols,
              const double *__restrict__ vals, int64_t n, const double *__restrict__ x,
              const uint32_t *mask, double *__restrict__ y, const int *done)
{
   if (done && *done) return;
   const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (i >= n) return;
   double s = 0.0;
   for (int k = rowptr[i]; k < rowptr[i + 1]; k++) {
      const int32_t c = cols[k];
      const double xv = mask && bit_set(mask, static_cast<uint32_t>(c)) ? 0.0 : x[c];
      s = mac<EXACT>(s, vals[k], xv);
   }
   y[i] = s;
}

// y_T = P^T x_L (SparseMatrix::mult_transpose); optionally y[ess] = xt[ess]
// and the xt . y partials of CG's p . q.
template <bool EXACT>
__global__ void __launch_bounds__(kT)
pt_kernel(const int32_t *__restrict__ trowptr, const int32_t *__restrict__ trows,
          const double *__restrict__ tvals, int64_t n, const double *__restrict__ xl,
          double *__restrict__ y, const double *__restrict__ xt, const uint32_t *ess,
          DotSink sink, const int *done)
{
   if (done && *done) return;
   const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   double dv = 0.0;
   if (j < n) {
      double s = 0.0;
      for (int k = trowptr[j]; k < trowptr[j + 1]; k++) s = mac<EXACT>(s, tvals[k], xl[trows[k]]);
      if (ess && bit_set(ess, static_cast<uint32_t>(j))) s = xt[j];
      y[j] = s;
      if (sink) dv = mul<EXACT>(xt[j], s);
   }
   if (sink) {
      const double v[1] = {dv};
      emit<kT, 1>(sink, v);
   }
}

__global__ void l2t_kernel(const int32_t *true_dofs, int64_t n, const double *x, double *X)
{
   const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (t < n) X[t] = x[true_dofs[t]];
}

// ----------------------------------------------------- diagonal with P
struct DiagP {
   Tables t;
   int p, nq, kind, elem_major;
   int64_t ne, ne_pad;
   const double *qdata;
   const uint32_t *gmap;
   ElemOrder order;
   const int32_t *prow, *pcol;
   const double *pval;
   const int32_t *true_index;
};

__device__ __forceinline__ uint32_t dof_of(const DiagP &A, int nd, int i, int64_t pos)
{
   return A.gmap[A.elem_major ? pos * nd + i : (int64_t)i * A.ne_pad + pos] & kDofMask;
}

__device__ __forceinline__ double qd(const DiagP &A, int ncomp, int nqd, int64_t pos, int c, int q)
{
   return A.elem_major ? __ldg(A.qdata + (pos * ncomp + c) * (int64_t)nqd + q)
                       : __ldg(A.qdata + (int64_t)(c * nqd + q) * A.ne_pad + pos);
}

// Tabulated 2D basis values of local DOF i at point q (forms.cpp:22-42).
__device__ __forceinline__ void tab(const DiagP &A, int q, int i, double &b, double &gx, double &gy)
{
   const int D1 = A.p + 1, qx = q % A.nq, qy = q / A.nq, ia = i % D1, ib = i / D1;
   b = __dmul_rn(A.t.B[qx][ia], A.t.B[qy][ib]);
   gx = __dmul_rn(A.t.G[qx][ia], A.t.B[qy][ib]);
   gy = __dmul_rn(A.t.B[qx][ia], A.t.G[qy][ib]);
}

__device__ bool constrained(const DiagP &A, int nd, int64_t pos)
{
   for (int i = 0; i < nd; i++)
      if (A.true_index[dof_of(A, nd, i, pos)] < 0) return true;
   return false;
}

__global__ void diagp_count_kernel(DiagP A, int32_t *count)
{
   const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (e >= A.ne) return;
   const int nd = (A.p + 1) * (A.p + 1);
   const int64_t pos = A.order.pos_of(e);
   if (!constrained(A, nd, pos)) {
      count[e] = nd;
      return;
   }
   int c = 0;
   for (int i = 0; i < nd; i++) {
      const uint32_t di = dof_of(A, nd, i, pos);
      for (int j = 0; j < nd; j++) {
         const uint32_t dj = dof_of(A, nd, j, pos);
         for (int a = A.prow[di]; a < A.prow[di + 1]; a++)
            for (int b = A.prow[dj]; b < A.prow[dj + 1]; b++) c += A.pcol[a] == A.pcol[b];
      }
   }
   count[e] = c;
}

// Contributions of element e at off[e].., in the reference's loop order.
__global__ void diagp_fill_kernel(DiagP A, const int32_t *off, int32_t *tgt, double *val)
{
   const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (e >= A.ne) return;
   const int nd = (A.p + 1) * (A.p + 1), nqd = A.nq * A.nq;
   const bool mass = A.kind == TFEM_MASS;
   const int ncomp = mass ? 1 : 3;
   const int64_t pos = A.order.pos_of(e);
   int64_t o = off[e];
   if (!constrained(A, nd, pos)) {
      for (int i = 0; i < nd; i++) {
         double s = 0.0;
         for (int q = 0; q < nqd; q++) {
            double b, gx, gy;
            tab(A, q, i, b, gx, gy);
            if (mass) {
               s = __dadd_rn(s, __dmul_rn(__dmul_rn(b, b), qd(A, ncomp, nqd, pos, 0, q)));
            } else {
               const double term =
                  __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(gx, gx), qd(A, ncomp, nqd, pos, 0, q)),
                                      __dmul_rn(__dmul_rn(__dmul_rn(2.0, gx), gy),
                                                qd(A, ncomp, nqd, pos, 1, q))),
                            __dmul_rn(__dmul_rn(gy, gy), qd(A, ncomp, nqd, pos, 2, q)));
               s = __dadd_rn(s, term);
            }
         }
         tgt[o] = A.true_index[dof_of(A, nd, i, pos)];
         val[o] = s;
         o++;
      }
      return;
   }
   for (int i = 0; i < nd; i++) {
      const uint32_t di = dof_of(A, nd, i, pos);
      for (int j = 0; j < nd; j++) {
         const uint32_t dj = dof_of(A, nd, j, pos);
         double lij = 0.0;
         for (int q = 0; q < nqd; q++) {
            double bi, gxi, gyi, bj, gxj, gyj;
            tab(A, q, i, bi, gxi, gyi);
            tab(A, q, j, bj, gxj, gyj);
            if (mass) {
               lij = __dadd_rn(lij, __dmul_rn(__dmul_rn(bi, bj), qd(A, ncomp, nqd, pos, 0, q)));
            } else {
               const double t0 = __dmul_rn(__dmul_rn(gxi, gxj), qd(A, ncomp, nqd, pos, 0, q));
               const double t1 = __dmul_rn(__dadd_rn(__dmul_rn(gxi, gyj), __dmul_rn(gyi, gxj)),
                                           qd(A, ncomp, nqd, pos, 1, q));
               const double t2 = __dmul_rn(__dmul_rn(gyi, gyj), qd(A, ncomp, nqd, pos, 2, q));
               lij = __dadd_rn(lij, __dadd_rn(__dadd_rn(t0, t1), t2));
            }
         }
         for (int a = A.prow[di]; a < A.prow[di + 1]; a++)
            for (int b = A.prow[dj]; b < A.prow[dj + 1]; b++)
               if (A.pcol[a] == A.pcol[b]) {
                  tgt[o] = A.pcol[a];
                  val[o] = __dmul_rn(__dmul_rn(A.pval[a], A.pval[b]), lij);
                  o++;
               }
      }
   }
}

// diag[k] += the run of target k, summed in sorted (= reference) order.
__global__ void diagp_sum_kernel(const int32_t *key, const int32_t *perm, const double *val,
                                 int64_t n, double *diag)
{
   const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (i >= n || (i > 0 && key[i] == key[i - 1])) return;
   double acc = 0.0;
   for (int64_t m = i; m < n && key[m] == key[i]; m++) acc = __dadd_rn(acc, val[perm[m]]);
   diag[key[i]] = __dadd_rn(diag[key[i]], acc);
}

__global__ void iota_kernel(int32_t *a, int64_t n)
{
   const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (i < n) a[i] = static_cast<int32_t>(i);
}

Tables tables_of_pa(const tfem_pa *pa)
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

} // namespace

tfem_prolongation *prolongation_create(tfem_ctx *ctx, int64_t n_local, int64_t n_true,
                                       const int32_t *rowptr, const int32_t *cols,
                                       const double *vals, const int32_t *true_index)
{
   if (n_local < 1 || n_true < 1 || n_true > n_local)
      invalid("prolongation: need 1 <= n_true <= n_local");
   if (rowptr[0] != 0) invalid("prolongation: rowptr[0] must be 0");
   for (int64_t i = 0; i < n_local; i++)
      if (rowptr[i + 1] < rowptr[i]) invalid("prolongation: rowptr must be non-decreasing");
   const int64_t nnz = rowptr[n_local];
   for (int64_t k = 0; k < nnz; k++)
      if (cols[k] < 0 || cols[k] >= n_true) invalid("prolongation: column index out of range");
   std::vector<int32_t> true_dofs(static_cast<size_t>(n_true), -1);
   for (int64_t l = 0; l < n_local; l++) {
      const int32_t t = true_index[l];
      if (t < -1 || t >= n_true) invalid("prolongation: true_index out of range");
      if (t >= 0) {
         if (true_dofs[t] >= 0) invalid("prolongation: true_index is not injective");
         true_dofs[t] = static_cast<int32_t>(l);
      }
   }
   for (int32_t l : true_dofs)
      if (l < 0) invalid("prolongation: a true DOF has no local DOF");
   // transpose by the reference's traversal (sparse.cpp:104-124)
   std::vector<int32_t> trp(static_cast<size_t>(n_true) + 1, 0), trows(static_cast<size_t>(nnz));
   std::vector<double> tvals(static_cast<size_t>(nnz));
   for (int64_t k = 0; k < nnz; k++) trp[cols[k] + 1]++;
   for (int64_t j = 0; j < n_true; j++) trp[j + 1] += trp[j];
   std::vector<int32_t> next(trp.begin(), trp.end() - 1);
   for (int64_t i = 0; i < n_local; i++)
      for (int32_t k = rowptr[i]; k < rowptr[i + 1]; k++) {
         const int32_t pos = next[cols[k]]++;
         trows[pos] = static_cast<int32_t>(i);
         tvals[pos] = vals[k];
      }
   auto *P = new tfem_prolongation;
   P->ctx = ctx;
   P->n_local = n_local;
   P->n_true = n_true;
   P->nnz = nnz;
   cudaStream_t s = ctx->stream;
   P->rowptr = dalloc<int32_t>(n_local + 1);
   P->cols = dalloc<int32_t>(nnz);
   P->vals = dalloc<double>(nnz);
   P->trowptr = dalloc<int32_t>(n_true + 1);
   P->trows = dalloc<int32_t>(nnz);
   P->tvals = dalloc<double>(nnz);
   P->true_index = dalloc<int32_t>(n_local);
   P->true_dofs = dalloc<int32_t>(n_true);
   h2d(s, P->rowptr, rowptr, sizeof(int32_t) * (n_local + 1));
   h2d(s, P->cols, cols, sizeof(int32_t) * nnz);
   h2d(s, P->vals, vals, sizeof(double) * nnz);
   h2d(s, P->trowptr, trp.data(), sizeof(int32_t) * trp.size());
   h2d(s, P->trows, trows.data(), sizeof(int32_t) * nnz);
   h2d(s, P->tvals, tvals.data(), sizeof(double) * nnz);
   h2d(s, P->true_index, true_index, sizeof(int32_t) * n_local);
   h2d(s, P->true_dofs, true_dofs.data(), sizeof(int32_t) * n_true);
   return P;
}

void prolongation_destroy(tfem_prolongation *P)
{
   if (!P) return;
   for (void *p : {static_cast<void *>(P->rowptr), static_cast<void *>(P->cols),
                   static_cast<void *>(P->vals), static_cast<void *>(P->trowptr),
                   static_cast<void *>(P->trows), static_cast<void *>(P->tvals),
                   static_cast<void *>(P->true_index), static_cast<void *>(P->true_dofs)})
      cudaFree(p);
   delete P;
}

int64_t prolongation_grid(const tfem_prolongation *P) { return blocks_for(P->n_true); }

void prolongation_mult(tfem_ctx *ctx, const tfem_prolongation *P, const double *x_true,
                       const uint32_t *mask_true, double *y_local, const int *done)
{
   const bool exact = ctx->numerics == TFEM_NUMERICS_REFERENCE;
   if (exact)
      p_mult_kernel<true><<<blocks_for(P->n_local), kT, 0, ctx->stream>>>(
         P->rowptr, P->cols, P->vals, P->n_local, x_true, mask_true, y_local, done);
   else
      p_mult_kernel<false><<<blocks_for(P->n_local), kT, 0, ctx->stream>>>(
         P->rowptr, P->cols, P->vals, P->n_local, x_true, mask_true, y_local, done);
   ctx->launched();
   TFEM_CUDA(cudaGetLastError());
}

void prolongation_mult_transpose(tfem_ctx *ctx, const tfem_prolongation *P, const double *x_local,
                                 double *y_true, const double *x_true_ess,
                                 const uint32_t *ess_true, const DotSink *dot, const int *done)
{
   const bool exact = ctx->numerics == TFEM_NUMERICS_REFERENCE;
   const DotSink sink = dot ? *dot : DotSink{};
   if (exact)
      pt_kernel<true><<<blocks_for(P->n_true), kT, 0, ctx->stream>>>(
         P->trowptr, P->trows, P->tvals, P->n_true, x_local, y_true, x_true_ess, ess_true, sink,
         done);
   else
      pt_kernel<false><<<blocks_for(P->n_true), kT, 0, ctx->stream>>>(
         P->trowptr, P->trows, P->tvals, P->n_true, x_local, y_true, x_true_ess, ess_true, sink,
         done);
   ctx->launched();
   TFEM_CUDA(cudaGetLastError());
}

void prolongation_local_to_true(tfem_ctx *ctx, const tfem_prolongation *P, const double *x_local,
                                double *x_true)
{
   l2t_kernel<<<blocks_for(P->n_true), kT, 0, ctx->stream>>>(P->true_dofs, P->n_true, x_local,
                                                            x_true);
   ctx->launched();
   TFEM_CUDA(cudaGetLastError());
}

void pa_diagonal_p(tfem_ctx *ctx, const tfem_pa *pa, const tfem_restriction *r,
                   const tfem_prolongation *P, double *diag_true)
{
   if (pa->dim != 2) invalid("pa_diagonal: prolongated spaces are 2D (NcForest)");
   if (pa->dim != r->dim || pa->p != r->p || pa->ne != r->ne || !(pa->order == r->order))
      invalid("forms: point factors were built for a different space");
   if (P->n_local != r->ndofs) invalid("pa_diagonal: prolongation / space size mismatch");
   cudaStream_t s = ctx->stream;
   DiagP A{};
   A.t = tables_of_pa(pa);
   A.p = pa->p;
   A.nq = pa->nq;
   A.kind = pa->kind;
   A.elem_major = pa->elem_major() ? 1 : 0;
   A.ne = pa->ne;
   A.ne_pad = pa->ne_pad;
   A.qdata = pa->qdata;
   A.gmap = r->gmap;
   A.order = r->order;
   A.prow = P->rowptr;
   A.pcol = P->cols;
   A.pval = P->vals;
   A.true_index = P->true_index;
   const int64_t ne = pa->ne;
   int32_t *count = dalloc<int32_t>(ne + 1), *off = dalloc<int32_t>(ne + 1);
   TFEM_CUDA(cudaMemsetAsync(count + ne, 0, sizeof(int32_t), s));
   diagp_count_kernel<<<blocks_for(ne), kT, 0, s>>>(A, count);
   size_t tmp_bytes = 0;
   TFEM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, count, off, ne + 1, s));
   void *tmp = dalloc<char>(static_cast<int64_t>(tmp_bytes));
   TFEM_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, count, off, ne + 1, s));
   int32_t total = 0;
   d2h(s, &total, off + ne, sizeof(int32_t));
   cudaFree(tmp);
   int32_t *tgt = dalloc<int32_t>(total), *key = dalloc<int32_t>(total);
   int32_t *idx = dalloc<int32_t>(total), *perm = dalloc<int32_t>(total);
   double *val = dalloc<double>(total);
   diagp_fill_kernel<<<blocks_for(ne), kT, 0, s>>>(A, off, tgt, val);
   iota_kernel<<<blocks_for(total), kT, 0, s>>>(idx, total);
   tmp_bytes = 0;
   TFEM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, tgt, key, idx, perm, total, 0,
                                             32, s));
   tmp = dalloc<char>(static_cast<int64_t>(tmp_bytes));
   // radix sort is stable: runs keep the generation (= reference) order
   TFEM_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, tgt, key, idx, perm, total, 0, 32, s));
   diagp_sum_kernel<<<blocks_for(total), kT, 0, s>>>(key, perm, val, total, diag_true);
   ctx->launched(6);
   TFEM_CUDA(cudaGetLastError());
   TFEM_CUDA(cudaStreamSynchronize(s));
   for (void *p : {static_cast<void *>(count), static_cast<void *>(off), tmp,
                   static_cast<void *>(tgt), static_cast<void *>(key), static_cast<void *>(idx),
                   static_cast<void *>(perm), static_cast<void *>(val)})
      cudaFree(p);
}

} // namespace tfem
