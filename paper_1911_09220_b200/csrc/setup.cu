// K1: PA quadrature-data setup on the device (forms.cpp:46-68, 201-229;
// mesh.cpp:142-179, 243-260).
//
// One thread per (point, element), element fastest, so the qdata planes
// [(c * nqd + q)][ne_pad] are written coalesced.  Every multiply / add / divide
// is an explicit round-to-nearest intrinsic in the reference's order (no FMA
// contraction), so 2D qdata is bit-identical to pa_setup.  The geometry basis
// tables (Gauss-Lobatto order m at the rule points and at the m+2 Gauss check
// points) come from the host (host_basis.cpp).
#include "common.cuh"

namespace tfem {

namespace {

constexpr int kMaxGeo = 9;          // geometry order m <= 8 on the device
constexpr int kMaxPts = kMaxQ + 2;  // rule points or m+2 check points

struct GeoTables {
   int m, npts;                     // order, points per axis
   double l[kMaxPts][kMaxGeo];      // values at the points
   double d[kMaxPts][kMaxGeo];      // derivatives at the points
   double w[kMaxPts];               // rule weights
};

struct GeoSource {
   int dim;
   int64_t ne;
   const double *ctrl; // [e][l][dim] or null (Cartesian)
   int n[3];           // local cells per axis
   int origin[3];      // cell offset in the global mesh
   int ng[3];          // global cells per axis
   double ext[3];
};

__device__ __forceinline__ double M(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double A(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double S(double a, double b) { return __dsub_rn(a, b); }

// Control point `l` (lattice order) of element e, component r.
__device__ __forceinline__ double ctrl_at(const GeoSource &g, int64_t e, int l, int r, int n1)
{
   if (g.ctrl) return g.ctrl[(e * (g.dim == 2 ? n1 * n1 : n1 * n1 * n1) + l) * g.dim + r];
   // make_cartesian vertex coordinate width * i / nx (mesh.cpp:296), i global
   int64_t idx;
   if (r == 0) idx = e % g.n[0] + (l & 1);
   else if (r == 1) idx = (e / g.n[0]) % g.n[1] + ((l >> 1) & 1);
   else idx = e / ((int64_t)g.n[0] * g.n[1]) + ((l >> 2) & 1);
   idx += g.origin[r];
   return __ddiv_rn(M(g.ext[r], static_cast<double>(idx)), static_cast<double>(g.ng[r]));
}

// J[r][s] = d x_r / d xh_s at the lattice point (px, py, pz) of the tables
// (ElementTransformation::jacobian, mesh.cpp:159-179; 3D extends the loops
// c, b, a outer to inner with weights (d * l) * l).
template <int DIM>
__device__ void jacobian(const GeoSource &g, const GeoTables &t, int64_t e, int px, int py,
                         int pz, double J[3][3])
{
   const int n1 = t.m + 1;
   for (int r = 0; r < 3; r++)
      for (int s = 0; s < 3; s++) J[r][s] = 0.0;
   if (DIM == 2) {
      for (int b = 0; b < n1; b++)
         for (int a = 0; a < n1; a++) {
            const int l = a + b * n1;
            const double cx = ctrl_at(g, e, l, 0, n1), cy = ctrl_at(g, e, l, 1, n1);
            const double wx = M(t.d[px][a], t.l[py][b]);
            const double wy = M(t.l[px][a], t.d[py][b]);
            J[0][0] = A(J[0][0], M(wx, cx));
            J[1][0] = A(J[1][0], M(wx, cy));
            J[0][1] = A(J[0][1], M(wy, cx));
            J[1][1] = A(J[1][1], M(wy, cy));
         }
      return;
   }
   for (int c = 0; c < n1; c++)
      for (int b = 0; b < n1; b++)
         for (int a = 0; a < n1; a++) {
            const int l = a + n1 * (b + n1 * c);
            const double w0 = M(M(t.d[px][a], t.l[py][b]), t.l[pz][c]);
            const double w1 = M(M(t.l[px][a], t.d[py][b]), t.l[pz][c]);
            const double w2 = M(M(t.l[px][a], t.l[py][b]), t.d[pz][c]);
            for (int r = 0; r < 3; r++) {
               const double cr = ctrl_at(g, e, l, r, n1);
               J[r][0] = A(J[r][0], M(w0, cr));
               J[r][1] = A(J[r][1], M(w1, cr));
               J[r][2] = A(J[r][2], M(w2, cr));
            }
         }
}

template <int DIM>
__device__ __forceinline__ double det_of(const double J[3][3])
{
   if (DIM == 2) return S(M(J[0][0], J[1][1]), M(J[0][1], J[1][0]));
   return A(S(M(J[0][0], S(M(J[1][1], J[2][2]), M(J[1][2], J[2][1]))),
              M(J[0][1], S(M(J[1][0], J[2][2]), M(J[1][2], J[2][0])))),
            M(J[0][2], S(M(J[1][0], J[2][1]), M(J[1][1], J[2][0]))));
}

// Mesh::transformation's det J > 0 audit at the (m+2)^dim Gauss points.
template <int DIM>
__global__ void check_kernel(GeoSource g, GeoTables t, unsigned long long *err)
{
   const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   const int np = t.npts, npd = DIM == 2 ? np * np : np * np * np;
   if (idx >= npd * g.ne) return;
   const int q = static_cast<int>(idx / g.ne);
   const int64_t e = idx % g.ne;
   double J[3][3];
   jacobian<DIM>(g, t, e, q % np, (q / np) % np, q / (np * np), J);
   if (!(det_of<DIM>(J) > 0.0)) atomicMin(err, static_cast<unsigned long long>(e) << 24);
}

template <int DIM>
__global__ void setup_kernel(GeoSource g, GeoTables t, int kind, const double *coeff,
                             double coeff_const, int64_t ne_pad, int layout, ElemOrder order,
                             double *qdata, unsigned long long *err)
{
   const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   const int nq = t.npts, nqd = DIM == 2 ? nq * nq : nq * nq * nq;
   if (idx >= nqd * g.ne) return;
   // Planes [(c*nqd+q)][ne_pad]: element fastest; element-major [e][c][q]:
   // point fastest.  Either way the stores are coalesced.
   // e: reference element number; pos: its position in the device order
   const bool emaj = layout != 0;
   const int q = static_cast<int>(emaj ? idx % nqd : idx / g.ne);
   const int64_t e = emaj ? idx / nqd : idx % g.ne;
   const int64_t pos = order.pos_of(e);
   const int qx = q % nq, qy = (q / nq) % nq, qz = q / (nq * nq);
   const int ncomp = kind == TFEM_MASS ? 1 : (DIM == 2 ? 3 : 6);
   auto out = [&](int c) -> double & {
      return qdata[qdata_index(layout, pos, c, q, ncomp, nqd, nq, ne_pad)];
   };
   double J[3][3];
   jacobian<DIM>(g, t, e, qx, qy, qz, J);
   const double det = det_of<DIM>(J);
   // point_factors (forms.cpp:50-59): det check, then the coefficient.
   if (det <= 0.0) {
      atomicMin(err, (static_cast<unsigned long long>(e) << 24) | (1u + 2u * q));
      return;
   }
   const double c = coeff ? coeff[e * nqd + q] : coeff_const;
   if (!(c > 0.0)) {
      atomicMin(err, (static_cast<unsigned long long>(e) << 24) | (2u + 2u * q));
      return;
   }
   double wq = M(t.w[qx], t.w[qy]);
   if (DIM == 3) wq = M(wq, t.w[qz]);
   if (kind == TFEM_MASS) {
      out(0) = M(M(wq, det), c);
      return;
   }
   const double s = __ddiv_rn(M(wq, c), det);
   if (DIM == 2) {
      const double dxdx = J[0][0], dxdy = J[0][1], dydx = J[1][0], dydy = J[1][1];
      out(0) = M(s, A(M(dxdy, dxdy), M(dydy, dydy)));
      out(1) = M(-s, A(M(dxdy, dxdx), M(dydy, dydx)));
      out(2) = M(s, A(M(dxdx, dxdx), M(dydx, dydx)));
      return;
   }
   double adj[3][3]; // adj(J)[s][r] = det J^{-1}
   adj[0][0] = S(M(J[1][1], J[2][2]), M(J[1][2], J[2][1]));
   adj[0][1] = S(M(J[0][2], J[2][1]), M(J[0][1], J[2][2]));
   adj[0][2] = S(M(J[0][1], J[1][2]), M(J[0][2], J[1][1]));
   adj[1][0] = S(M(J[1][2], J[2][0]), M(J[1][0], J[2][2]));
   adj[1][1] = S(M(J[0][0], J[2][2]), M(J[0][2], J[2][0]));
   adj[1][2] = S(M(J[0][2], J[1][0]), M(J[0][0], J[1][2]));
   adj[2][0] = S(M(J[1][0], J[2][1]), M(J[1][1], J[2][0]));
   adj[2][1] = S(M(J[0][1], J[2][0]), M(J[0][0], J[2][1]));
   adj[2][2] = S(M(J[0][0], J[1][1]), M(J[0][1], J[1][0]));
   const int si[6] = {0, 0, 0, 1, 1, 2}, sj[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
   for (int k = 0; k < 6; k++) {
      const double *u = adj[si[k]], *v = adj[sj[k]];
      out(k) = M(s, A(A(M(u[0], v[0]), M(u[1], v[1])), M(u[2], v[2])));
   }
}

// ElementTransformation::point (mesh.cpp:142-157) at every rule point.
template <int DIM>
__global__ void points_kernel(GeoSource g, GeoTables t, double *xyz /* [e][q][dim] */)
{
   const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   const int nq = t.npts, nqd = DIM == 2 ? nq * nq : nq * nq * nq;
   if (idx >= nqd * g.ne) return;
   const int64_t e = idx / nqd;
   const int q = static_cast<int>(idx % nqd);
   const int qx = q % nq, qy = (q / nq) % nq, qz = q / (nq * nq);
   const int n1 = t.m + 1;
   double X[3] = {0.0, 0.0, 0.0};
   if (DIM == 2) {
      for (int b = 0; b < n1; b++)
         for (int a = 0; a < n1; a++) {
            const double w = M(t.l[qx][a], t.l[qy][b]);
            for (int r = 0; r < 2; r++) X[r] = A(X[r], M(w, ctrl_at(g, e, a + b * n1, r, n1)));
         }
   } else {
      for (int c = 0; c < n1; c++)
         for (int b = 0; b < n1; b++)
            for (int a = 0; a < n1; a++) {
               const double w = M(M(t.l[qx][a], t.l[qy][b]), t.l[qz][c]);
               for (int r = 0; r < 3; r++)
                  X[r] = A(X[r], M(w, ctrl_at(g, e, a + n1 * (b + n1 * c), r, n1)));
            }
   }
   for (int r = 0; r < DIM; r++) xyz[idx * DIM + r] = X[r];
}

// LinearForm (forms.cpp:400-431), 2D: per element q(qx, qy) =
// ((w_x w_y) detJ) f at the Gauss points, then tensor_interp_2d_transpose =
// mat_mult(mat_mult_tn(B, q), B) (tensor_kernels.cpp:18-65, 89-97) -- every
// sum from 0.0 in ascending index -- into the element vector [e][b D1 + a].
struct Basis1D {
   double B[kMaxQ][kMaxP + 1];
};

__global__ void linear_form_kernel(GeoSource g, GeoTables t, Basis1D bt, int p, const double *f,
                                   double *evec)
{
   const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (e >= g.ne) return;
   const int nq = t.npts, nd = p + 1;
   double q[kMaxQ][kMaxQ]; // q[qx][qy]
   for (int qy = 0; qy < nq; qy++)
      for (int qx = 0; qx < nq; qx++) {
         double J[3][3];
         jacobian<2>(g, t, e, qx, qy, 0, J);
         const double det = det_of<2>(J);
         q[qx][qy] = M(M(M(t.w[qx], t.w[qy]), det), f[e * nq * nq + qy * nq + qx]);
      }
   double T[kMaxP + 1][kMaxQ]; // mat_mult_tn(B, q): k (= qx) outermost
   for (int a = 0; a < nd; a++)
      for (int qy = 0; qy < nq; qy++) T[a][qy] = 0.0;
   for (int k = 0; k < nq; k++)
      for (int a = 0; a < nd; a++)
         for (int qy = 0; qy < nq; qy++) T[a][qy] = A(T[a][qy], M(bt.B[k][a], q[k][qy]));
   for (int a = 0; a < nd; a++)
      for (int b = 0; b < nd; b++) {
         double s = 0.0; // mat_mult: k (= qy) ascending
         for (int k = 0; k < nq; k++) s = A(s, M(T[a][k], bt.B[k][b]));
         evec[e * nd * nd + b * nd + a] = s;
      }
}

// compute_l2_error's per-point terms (fespace.cpp:358-394), 2D: u_h at the
// point from the element values [e][b D1 + a] (s over a, then u over b, each
// from 0.0), det J, d = u_h - u_exact, term ((((w_x w_y) det) d) d).
__global__ void l2_terms_kernel(GeoSource g, GeoTables t, Basis1D bt, int p, const double *ev,
                                const double *uex, double *terms)
{
   const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (e >= g.ne) return;
   const int nq = t.npts, nd = p + 1;
   for (int qy = 0; qy < nq; qy++)
      for (int qx = 0; qx < nq; qx++) {
         double u = 0.0;
         for (int b = 0; b < nd; b++) {
            double s = 0.0;
            for (int a = 0; a < nd; a++) s = A(s, M(bt.B[qx][a], ev[e * nd * nd + b * nd + a]));
            u = A(u, M(bt.B[qy][b], s));
         }
         double J[3][3];
         jacobian<2>(g, t, e, qx, qy, 0, J);
         const double det = det_of<2>(J);
         const int64_t q = e * nq * nq + qy * nq + qx;
         const double d = S(u, uex[q]);
         terms[q] = M(M(M(M(t.w[qx], t.w[qy]), det), d), d);
      }
}

GeoTables tables_at(int m, const std::vector<double> &pts, const std::vector<double> *w)
{
   GeoTables t{};
   t.m = m;
   t.npts = static_cast<int>(pts.size());
   std::vector<double> nodes, bary;
   basis_nodes(m, TFEM_NODES_GAUSS_LOBATTO, nodes, bary);
   for (int k = 0; k < t.npts; k++) {
      basis_eval(nodes, bary, pts[k], t.l[k], t.d[k]);
      t.w[k] = w ? (*w)[k] : 0.0;
   }
   return t;
}

GeoSource source_of(const tfem_geometry *g)
{
   GeoSource s{};
   s.dim = g->dim;
   s.ne = g->ne;
   s.ctrl = g->ctrl;
   for (int d = 0; d < 3; d++) {
      s.n[d] = g->n[d];
      s.origin[d] = g->origin[d];
      s.ng[d] = g->n_global[d];
      s.ext[d] = g->ext[d];
   }
   return s;
}

inline unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

} // namespace

// Mesh::transformation's audit (mesh.cpp:243-260) ahead of the functions
// that call it per element in the reference (LinearForm, project_coefficient,
// compute_l2_error, and the coefficient points of pa_setup): the first
// inverted element throws the reference's runtime_error.  Cartesian
// geometries with positive extents cannot invert.
void audit_geometry(tfem_ctx *ctx, const tfem_geometry *g)
{
   if (g->cartesian) return;
   const GeoTables tc = tables_at(g->order, gauss_points(TFEM_GAUSS_LEGENDRE, g->order + 2, nullptr),
                                  nullptr);
   const GeoSource src = source_of(g);
   unsigned long long *d_err = nullptr;
   TFEM_CUDA(cudaMalloc(&d_err, sizeof(unsigned long long)));
   TFEM_CUDA(cudaMemsetAsync(d_err, 0xff, sizeof(unsigned long long), ctx->stream));
   const int T = 256;
   const int ncd = g->dim == 2 ? tc.npts * tc.npts : tc.npts * tc.npts * tc.npts;
   if (g->dim == 2)
      check_kernel<2><<<blocks_for(ncd * g->ne, T), T, 0, ctx->stream>>>(src, tc, d_err);
   else
      check_kernel<3><<<blocks_for(ncd * g->ne, T), T, 0, ctx->stream>>>(src, tc, d_err);
   ctx->launched();
   TFEM_CUDA(cudaGetLastError());
   unsigned long long herr = 0;
   TFEM_CUDA(cudaMemcpyAsync(&herr, d_err, sizeof(herr), cudaMemcpyDeviceToHost, ctx->stream));
   TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   cudaFree(d_err);
   if (herr != ~0ull)
      runtime("Mesh::transformation: inverted element " + std::to_string(herr >> 24));
}

tfem_pa *pa_setup(tfem_ctx *ctx, int kind, const tfem_geometry *g, int p, int nq, int rule,
                  const double *coeff_host, double coeff_const, int64_t *bad_elem)
{
   if (kind != TFEM_DIFFUSION && kind != TFEM_MASS) invalid("pa_setup: unknown integrator kind");
   if (p < 1 || p > (g->dim == 3 ? kMaxP3D : kMaxP))
      invalid("pa_setup: order must be in [1, 16] (2D) / [1, 8] (3D) on the device");
   if (nq < 1 || nq > kMaxQ) invalid("pa_setup: quadrature points per axis must be in [1, 19]");
   if (g->order + 1 > kMaxGeo) invalid("pa_setup: geometry order must be <= 8 on the device");
   const int dim = g->dim;
   const int nqd = dim == 2 ? nq * nq : nq * nq * nq;
   auto *pa = new tfem_pa;
   pa->ctx = ctx;
   pa->kind = kind;
   pa->dim = dim;
   pa->p = p;
   pa->nq = nq;
   pa->rule = rule;
   pa->ncomp = kind == TFEM_MASS ? 1 : (dim == 2 ? 3 : 6);
   pa->nqd = nqd;
   pa->ne = g->ne;
   pa->order = elem_order_for(dim, p, g->cartesian, g->n);
   pa->npos = pa->order.n_pos(g->ne);
   pa->ne_pad = round_up(pa->npos, 64);
   pa->B.resize(static_cast<size_t>(nq) * (p + 1));
   pa->G.resize(pa->B.size());
   eval_matrices(p, TFEM_NODES_GAUSS_LOBATTO, nq, rule, pa->B.data(), pa->G.data());
   pa->qlayout = qdata_layout(dim, p, nq, kind);
   pa->colloc = nq == p + 1;
   for (int q = 0; q < nq && pa->colloc; q++)
      for (int i = 0; i <= p; i++)
         if (pa->B[q * (p + 1) + i] != (q == i ? 1.0 : 0.0)) pa->colloc = false;

   std::vector<double> w;
   const std::vector<double> pts = gauss_points(rule, nq, &w);
   const GeoTables tq = tables_at(g->order, pts, &w);
   const GeoTables tc = tables_at(g->order, gauss_points(TFEM_GAUSS_LEGENDRE, g->order + 2, nullptr),
                                  nullptr);
   const GeoSource src = source_of(g);

   const size_t qbytes = sizeof(double) * static_cast<size_t>(pa->ncomp) * nqd * pa->ne_pad;
   cudaError_t ce = cudaMalloc(&pa->qdata, qbytes);
   if (ce != cudaSuccess) {
      delete pa;
      cuda_check(ce, "pa_setup: qdata allocation");
   }
   TFEM_CUDA(cudaMemsetAsync(pa->qdata, 0, qbytes, ctx->stream));
   double *d_coeff = nullptr;
   if (coeff_host) {
      TFEM_CUDA(cudaMalloc(&d_coeff, sizeof(double) * nqd * g->ne));
      TFEM_CUDA(cudaMemcpyAsync(d_coeff, coeff_host, sizeof(double) * nqd * g->ne,
                                cudaMemcpyHostToDevice, ctx->stream));
   }
   unsigned long long *d_err = nullptr;
   TFEM_CUDA(cudaMalloc(&d_err, sizeof(unsigned long long)));
   TFEM_CUDA(cudaMemsetAsync(d_err, 0xff, sizeof(unsigned long long), ctx->stream));
   const int T = 256;
   const int ncd = dim == 2 ? tc.npts * tc.npts : tc.npts * tc.npts * tc.npts;
   if (dim == 2) {
      check_kernel<2><<<blocks_for(ncd * g->ne, T), T, 0, ctx->stream>>>(src, tc, d_err);
      setup_kernel<2><<<blocks_for(nqd * g->ne, T), T, 0, ctx->stream>>>(
         src, tq, kind, d_coeff, coeff_const, pa->ne_pad, pa->qlayout, pa->order, pa->qdata, d_err);
   } else {
      check_kernel<3><<<blocks_for(ncd * g->ne, T), T, 0, ctx->stream>>>(src, tc, d_err);
      setup_kernel<3><<<blocks_for(nqd * g->ne, T), T, 0, ctx->stream>>>(
         src, tq, kind, d_coeff, coeff_const, pa->ne_pad, pa->qlayout, pa->order, pa->qdata, d_err);
   }
   ctx->launched(2);
   TFEM_CUDA(cudaGetLastError());
   unsigned long long herr = 0;
   TFEM_CUDA(cudaMemcpyAsync(&herr, d_err, sizeof(herr), cudaMemcpyDeviceToHost, ctx->stream));
   TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   cudaFree(d_err);
   if (d_coeff) cudaFree(d_coeff);
   if (herr != ~0ull) {
      cudaFree(pa->qdata);
      delete pa;
      const int64_t e = static_cast<int64_t>(herr >> 24);
      const unsigned code = static_cast<unsigned>(herr & 0xffffffu);
      if (bad_elem) *bad_elem = e;
      if (code == 0) runtime("Mesh::transformation: inverted element " + std::to_string(e));
      if (code & 1u) runtime("forms: inverted element at a quadrature point");
      invalid("forms: coefficient must be positive");
   }
   return pa;
}

void geometry_points(tfem_ctx *ctx, const tfem_geometry *g, int nq, int rule, double *host_xyz)
{
   if (nq < 1 || nq > kMaxQ) invalid("geometry_points: points per axis must be in [1, 19]");
   audit_geometry(ctx, g);
   const int dim = g->dim;
   const int nqd = dim == 2 ? nq * nq : nq * nq * nq;
   const GeoTables t = tables_at(g->order, gauss_points(rule, nq, nullptr), nullptr);
   const GeoSource src = source_of(g);
   double *d = nullptr;
   const size_t bytes = sizeof(double) * static_cast<size_t>(g->ne) * nqd * dim;
   TFEM_CUDA(cudaMalloc(&d, bytes));
   const int T = 256;
   if (dim == 2)
      points_kernel<2><<<blocks_for(nqd * g->ne, T), T, 0, ctx->stream>>>(src, t, d);
   else
      points_kernel<3><<<blocks_for(nqd * g->ne, T), T, 0, ctx->stream>>>(src, t, d);
   ctx->launched();
   TFEM_CUDA(cudaGetLastError());
   TFEM_CUDA(cudaMemcpyAsync(host_xyz, d, bytes, cudaMemcpyDeviceToHost, ctx->stream));
   TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   cudaFree(d);
}

void linear_form(tfem_ctx *ctx, const tfem_geometry *g, const tfem_restriction *r, int p,
                 const double *f_host, double *b)
{
   if (g->dim != 2 || r->dim != 2) invalid("LinearForm: 2D spaces (forms.cpp:400-431)");
   if (r->p != p || r->ne != g->ne) invalid("LinearForm: geometry / space mismatch");
   if (p < 1 || p > kMaxP || p + 2 > kMaxQ) invalid("LinearForm: order must be in [1, 16]");
   const int nq = p + 2, nd = p + 1;
   std::vector<double> w;
   const std::vector<double> pts = gauss_points(TFEM_GAUSS_LEGENDRE, nq, &w);
   const GeoTables t = tables_at(g->order, pts, &w);
   Basis1D bt{};
   std::vector<double> B(static_cast<size_t>(nq) * nd), G(B.size());
   eval_matrices(p, TFEM_NODES_GAUSS_LOBATTO, nq, TFEM_GAUSS_LEGENDRE, B.data(), G.data());
   for (int q = 0; q < nq; q++)
      for (int i = 0; i < nd; i++) bt.B[q][i] = B[q * nd + i];
   const GeoSource src = source_of(g);
   const int64_t ne = g->ne;
   double *d_f = nullptr, *d_e = nullptr;
   TFEM_CUDA(cudaMalloc(&d_f, sizeof(double) * static_cast<size_t>(ne) * nq * nq));
   TFEM_CUDA(cudaMalloc(&d_e, sizeof(double) * static_cast<size_t>(ne) * nd * nd));
   TFEM_CUDA(cudaMemcpyAsync(d_f, f_host, sizeof(double) * static_cast<size_t>(ne) * nq * nq,
                             cudaMemcpyHostToDevice, ctx->stream));
   const int T = 128;
   linear_form_kernel<<<blocks_for(ne, T), T, 0, ctx->stream>>>(src, t, bt, p, d_f, d_e);
   ctx->launched();
   TFEM_CUDA(cudaGetLastError());
   // b = 0, then b[dofs[b D1 + a]] += bl(a, b) in element order (forms.cpp:424-428)
   vec_fill(ctx, b, r->ndofs, 0.0);
   restriction_mult_transpose(ctx, r, d_e, b);
   TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   cudaFree(d_f);
   cudaFree(d_e);
}

// ElementTransformation::point at the basis nodes (the GLL lattice),
// [e][b D1 + a][2] (project_coefficient, fespace.cpp:334-356).
void geometry_node_points(tfem_ctx *ctx, const tfem_geometry *g, int p, double *host_xy)
{
   if (g->dim != 2) invalid("project_coefficient: 2D spaces");
   if (p < 1 || p > kMaxP) invalid("project_coefficient: order must be in [1, 16]");
   audit_geometry(ctx, g);
   std::vector<double> nodes, bary;
   basis_nodes(p, TFEM_NODES_GAUSS_LOBATTO, nodes, bary);
   const GeoTables t = tables_at(g->order, nodes, nullptr);
   const GeoSource src = source_of(g);
   const int nd = p + 1;
   double *d = nullptr;
   const size_t bytes = sizeof(double) * static_cast<size_t>(g->ne) * nd * nd * 2;
   TFEM_CUDA(cudaMalloc(&d, bytes));
   const int T = 256;
   points_kernel<2><<<blocks_for(static_cast<int64_t>(nd) * nd * g->ne, T), T, 0, ctx->stream>>>(
      src, t, d);
   ctx->launched();
   TFEM_CUDA(cudaGetLastError());
   TFEM_CUDA(cudaMemcpyAsync(host_xy, d, bytes, cudaMemcpyDeviceToHost, ctx->stream));
   TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   cudaFree(d);
}

void restriction_mult(tfem_ctx *ctx, const tfem_restriction *r, const double *l, double *e);

// compute_l2_error (fespace.cpp:358-394): per-point terms on the device, the
// reference's sequential sum over elements and points on the host.
double l2_error(tfem_ctx *ctx, const tfem_geometry *g, const tfem_restriction *r, int p,
                const double *x, const double *u_exact_host)
{
   if (g->dim != 2 || r->dim != 2) invalid("compute_l2_error: 2D spaces");
   if (r->p != p || r->ne != g->ne) invalid("compute_l2_error: geometry / space mismatch");
   const int nq = p + 3, nd = p + 1;
   if (nq > kMaxQ) invalid("compute_l2_error: order must be <= 16 on the device");
   std::vector<double> w;
   const std::vector<double> pts = gauss_points(TFEM_GAUSS_LEGENDRE, nq, &w);
   const GeoTables t = tables_at(g->order, pts, &w);
   Basis1D bt{};
   std::vector<double> B(static_cast<size_t>(nq) * nd), G(B.size());
   eval_matrices(p, TFEM_NODES_GAUSS_LOBATTO, nq, TFEM_GAUSS_LEGENDRE, B.data(), G.data());
   for (int q = 0; q < nq; q++)
      for (int i = 0; i < nd; i++) bt.B[q][i] = B[q * nd + i];
   const int64_t ne = g->ne, npts = ne * nq * nq;
   double *ev = nullptr, *uex = nullptr, *terms = nullptr;
   TFEM_CUDA(cudaMalloc(&ev, sizeof(double) * static_cast<size_t>(ne) * nd * nd));
   TFEM_CUDA(cudaMalloc(&uex, sizeof(double) * static_cast<size_t>(npts)));
   TFEM_CUDA(cudaMalloc(&terms, sizeof(double) * static_cast<size_t>(npts)));
   restriction_mult(ctx, r, x, ev); // element values [e][b D1 + a]
   TFEM_CUDA(cudaMemcpyAsync(uex, u_exact_host, sizeof(double) * npts, cudaMemcpyHostToDevice,
                             ctx->stream));
   const int T = 128;
   l2_terms_kernel<<<blocks_for(ne, T), T, 0, ctx->stream>>>(source_of(g), t, bt, p, ev, uex,
                                                            terms);
   ctx->launched();
   TFEM_CUDA(cudaGetLastError());
   std::vector<double> h(static_cast<size_t>(npts));
   TFEM_CUDA(cudaMemcpyAsync(h.data(), terms, sizeof(double) * npts, cudaMemcpyDeviceToHost,
                             ctx->stream));
   TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   cudaFree(ev);
   cudaFree(uex);
   cudaFree(terms);
   volatile double err2 = 0.0; // the reference's left-to-right sum
   for (double v : h) err2 = err2 + v;
   return std::sqrt(static_cast<double>(err2));
}

} // namespace tfem
