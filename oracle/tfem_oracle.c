/*
 * ORACLE INFRASTRUCTURE -- CPU restatement of the reference algorithm for the
 * PA operator + Jacobi-CG hot path (test / bench checker only; see
 * tfem_oracle.h for the parity status of each part).
 *
 * Every function cites the reference file:line it restates.  Arithmetic is
 * written operation-for-operation in the reference's order (separate
 * multiplies and adds, sequential ascending sums) so the 2D results are
 * bit-identical to the reference built with -ffp-contract=off; 3D extends the
 * same contraction order axis by axis.
 */
#include "tfem_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORC_PI 3.14159265358979323846 /* glibc M_PI */

static _Thread_local char g_err[256];

static int fail(int code, const char *msg)
{
   snprintf(g_err, sizeof g_err, "%s", msg);
   return code;
}

const char *orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------ quadrature */

/* Legendre P_n and P'_n by the three-term recurrence (quadrature.cpp:20-31). */
static void legendre(int n, double x, double *p, double *dp)
{
   double p0 = 1.0, p1 = x;
   if (n == 0) {
      *p = p0;
      *dp = 0.0;
      return;
   }
   for (int k = 1; k < n; k++) {
      double p2 = ((2 * k + 1) * x * p1 - k * p0) / (k + 1);
      p0 = p1;
      p1 = p2;
   }
   *p = p1;
   *dp = n * (x * p1 - p0) / (x * x - 1.0);
}

/* Newton on f = P_n (gl=1) or f = P'_m (gl=0) (quadrature.cpp:34-45,101-106). */
static int newton_root(int gl, int n, double x, double *root)
{
   for (int it = 0; it < 100; it++) {
      double v, dv;
      if (gl) {
         legendre(n, x, &v, &dv);
      } else {
         double p, dp;
         legendre(n, x, &p, &dp);
         v = dp;
         dv = (2.0 * x * dp - n * (n + 1) * p) / (1.0 - x * x);
      }
      double dx = v / dv;
      x -= dx;
      if (fabs(dx) < 1e-15) {
         *root = x;
         return 0;
      }
   }
   return fail(2, "quadrature: Newton iteration did not converge");
}

/* quadrature.cpp:64-89 */
int orc_gauss_legendre(int n, double *pts, double *wts)
{
   if (n < 1) return fail(1, "gauss_legendre: need n >= 1");
   double x[ORC_MAX_Q * 4], w[ORC_MAX_Q * 4];
   if (n > ORC_MAX_Q * 4) return fail(1, "gauss_legendre: n too large");
   for (int i = 0; i < n / 2 + n % 2; i++) {
      double guess = -cos(ORC_PI * (i + 0.75) / (n + 0.5));
      double xi = 0.0;
      if (2 * i + 1 != n) {
         int rc = newton_root(1, n, guess, &xi);
         if (rc) return rc;
      }
      double p, dp;
      legendre(n, xi, &p, &dp);
      double wi = (2 * i + 1 == n) ? 2.0 / (dp * dp)
                                   : 2.0 / ((1.0 - xi * xi) * dp * dp);
      x[i] = xi;
      w[i] = wi;
      x[n - 1 - i] = -xi;
      w[n - 1 - i] = wi;
   }
   for (int i = 0; i < n; i++) { /* map_to_unit, quadrature.cpp:48-60 */
      pts[i] = 0.5 * (x[i] + 1.0);
      wts[i] = 0.5 * w[i];
   }
   return 0;
}

/* quadrature.cpp:91-125 */
int orc_gauss_lobatto(int n, double *pts, double *wts)
{
   if (n < 2) return fail(1, "gauss_lobatto: need n >= 2");
   if (n > ORC_MAX_Q * 4) return fail(1, "gauss_lobatto: n too large");
   double x[ORC_MAX_Q * 4], w[ORC_MAX_Q * 4];
   const int m = n - 1;
   x[0] = -1.0;
   x[n - 1] = 1.0;
   for (int i = 1; i <= (n - 1) / 2; i++) {
      double guess = -cos(ORC_PI * i / m);
      double xi = 0.0;
      if (2 * i != n - 1) {
         int rc = newton_root(0, m, guess, &xi);
         if (rc) return rc;
      }
      x[i] = xi;
      x[n - 1 - i] = -xi;
   }
   for (int i = 0; i < n; i++) {
      double p, dp;
      legendre(m, x[i], &p, &dp);
      w[i] = 2.0 / (n * m * p * p);
   }
   for (int i = 0; i < n / 2; i++) {
      double wi = 0.5 * (w[i] + w[n - 1 - i]);
      w[i] = w[n - 1 - i] = wi;
   }
   for (int i = 0; i < n; i++) {
      pts[i] = 0.5 * (x[i] + 1.0);
      wts[i] = 0.5 * w[i];
   }
   return 0;
}

/* ----------------------------------------------------------------- basis */

/* Basis1D::Basis1D (basis.cpp:12-46). */
int orc_basis_nodes(int p, int node_kind, double *nodes, double *bary)
{
   const int n = p + 1;
   double wts[ORC_MAX_Q * 4];
   if (p < 0) return fail(1, "Basis1D: order must be >= 0");
   if (n > ORC_MAX_Q * 4) return fail(1, "Basis1D: order too large");
   int rc = 0;
   if (node_kind == 0) {
      if (p < 1) return fail(1, "Basis1D: Gauss-Lobatto nodes need order >= 1");
      rc = orc_gauss_lobatto(n, nodes, wts);
   } else if (node_kind == 1) {
      rc = orc_gauss_legendre(n, nodes, wts);
   } else {
      if (p == 0) {
         nodes[0] = 0.5;
      } else {
         for (int i = 0; i < n; i++) nodes[i] = (double)i / p;
      }
   }
   if (rc) return rc;
   for (int j = 0; j < n; j++) {
      bary[j] = 1.0;
      for (int k = 0; k < n; k++) {
         if (k != j) bary[j] /= nodes[j] - nodes[k];
      }
   }
   return 0;
}

/* Basis1D::eval, both overloads (basis.cpp:48-93). */
void orc_basis_eval(int p, const double *nodes, const double *bary, double x,
                    double *values, double *derivs)
{
   const int n = p + 1;
   for (int i = 0; i < n; i++) {
      if (x == nodes[i]) {
         if (!derivs) {
            for (int k = 0; k < n; k++) values[k] = (k == i) ? 1.0 : 0.0;
            return;
         }
         double dii = 0.0;
         for (int j = 0; j < n; j++) {
            values[j] = (j == i) ? 1.0 : 0.0;
            if (j != i) {
               derivs[j] = (bary[j] / bary[i]) / (nodes[i] - nodes[j]);
               dii -= derivs[j];
            }
         }
         derivs[i] = dii;
         return;
      }
   }
   double denom = 0.0;
   for (int j = 0; j < n; j++) {
      values[j] = bary[j] / (x - nodes[j]);
      denom += values[j];
   }
   for (int j = 0; j < n; j++) values[j] /= denom;
   if (!derivs) return;
   double all = 0.0;
   for (int k = 0; k < n; k++) all += 1.0 / (x - nodes[k]);
   for (int j = 0; j < n; j++) derivs[j] = values[j] * (all - 1.0 / (x - nodes[j]));
}

static int rule_points(int nq, int rule_kind, double *pts, double *wts)
{
   return rule_kind == 0 ? orc_gauss_legendre(nq, pts, wts)
                         : orc_gauss_lobatto(nq, pts, wts);
}

/* eval_matrices (basis.cpp:95-109). */
int orc_eval_matrices(int p, int node_kind, int nq, int rule_kind, double *B,
                      double *G)
{
   double nodes[ORC_MAX_Q * 4], bary[ORC_MAX_Q * 4];
   double pts[ORC_MAX_Q * 4], wts[ORC_MAX_Q * 4];
   int rc = orc_basis_nodes(p, node_kind, nodes, bary);
   if (rc) return rc;
   rc = rule_points(nq, rule_kind, pts, wts);
   if (rc) return rc;
   for (int k = 0; k < nq; k++) {
      orc_basis_eval(p, nodes, bary, pts[k], B + k * (p + 1), G + k * (p + 1));
   }
   return 0;
}

/* ------------------------------------------------------------------ mesh */

int64_t orc_cartesian_nv(int dim, const int *n)
{
   int64_t v = 1;
   for (int d = 0; d < dim; d++) v *= (n[d] + 1);
   return v;
}

int64_t orc_cartesian_ne(int dim, const int *n)
{
   int64_t v = 1;
   for (int d = 0; d < dim; d++) v *= n[d];
   return v;
}

/* make_cartesian (mesh.cpp:283-306); 3D adds k outermost. */
void orc_cartesian_vertices(int dim, const int *n, const double *ext,
                            double *coords)
{
   const int nz = dim == 3 ? n[2] : 0;
   int64_t at = 0;
   for (int k = 0; k <= nz; k++)
      for (int j = 0; j <= n[1]; j++)
         for (int i = 0; i <= n[0]; i++) {
            coords[at * dim + 0] = ext[0] * i / n[0];
            coords[at * dim + 1] = ext[1] * j / n[1];
            if (dim == 3) coords[at * dim + 2] = ext[2] * k / n[2];
            at++;
         }
}

void orc_cartesian_elements(int dim, const int *n, int *ev)
{
   const int nx = n[0], ny = n[1], nz = dim == 3 ? n[2] : 1;
#define VID(i, j, k) ((i) + (nx + 1) * ((j) + (ny + 1) * (k)))
   int64_t e = 0;
   for (int k = 0; k < nz; k++)
      for (int j = 0; j < ny; j++)
         for (int i = 0; i < nx; i++) {
            if (dim == 2) {
               int *v = ev + 4 * e;
               v[0] = VID(i, j, 0);
               v[1] = VID(i + 1, j, 0);
               v[2] = VID(i + 1, j + 1, 0);
               v[3] = VID(i, j + 1, 0);
            } else {
               int *v = ev + 8 * e;
               v[0] = VID(i, j, k);
               v[1] = VID(i + 1, j, k);
               v[2] = VID(i + 1, j + 1, k);
               v[3] = VID(i, j + 1, k);
               v[4] = VID(i, j, k + 1);
               v[5] = VID(i + 1, j, k + 1);
               v[6] = VID(i + 1, j + 1, k + 1);
               v[7] = VID(i, j + 1, k + 1);
            }
            e++;
         }
#undef VID
}

/* Lattice-ordered straight-element control points (mesh.cpp:238-240). */
void orc_cartesian_ctrl(int dim, const int *n, const double *ext, double *ctrl)
{
   const int nx = n[0], ny = n[1], nz = dim == 3 ? n[2] : 1;
   const int nc = 1 << dim;
   int64_t e = 0;
   for (int k = 0; k < nz; k++)
      for (int j = 0; j < ny; j++)
         for (int i = 0; i < nx; i++) {
            for (int l = 0; l < nc; l++) {
               const int a = l & 1, b = (l >> 1) & 1, c = (l >> 2) & 1;
               double *o = ctrl + (e * nc + l) * dim;
               o[0] = ext[0] * (i + a) / nx;
               o[1] = ext[1] * (j + b) / ny;
               if (dim == 3) o[2] = ext[2] * (k + c) / nz;
            }
            e++;
         }
}

/* ---------------------------------------------------------------- layout */

/* MeshTopology (mesh.cpp:26-57) with an open-addressing map from the sorted
 * vertex pair to the discovery-order edge id, then build_h1_layout
 * (mesh.cpp:65-115). */
int64_t orc_h1_layout_quads(int nv, int ne, const int *ev, int p,
                            int *elem_dofs)
{
   static const int from[4] = {0, 1, 2, 3}, to[4] = {1, 2, 3, 0};
   if (p < 1) return -fail(1, "build_h1_layout: order must be >= 1");
   int64_t cap = 1;
   while (cap < 8 * (int64_t)ne + 16) cap <<= 1;
   int64_t *keys = malloc(sizeof(int64_t) * cap);
   int *vals = malloc(sizeof(int) * cap);
   int *eedge = malloc(sizeof(int) * 4 * (size_t)ne);
   if (!keys || !vals || !eedge) {
      free(keys); free(vals); free(eedge);
      return -fail(2, "layout: out of memory");
   }
   for (int64_t i = 0; i < cap; i++) keys[i] = -1;
   int n_edges = 0;
   for (int k = 0; k < ne; k++) {
      for (int le = 0; le < 4; le++) {
         int a = ev[4 * k + from[le]], b = ev[4 * k + to[le]];
         int lo = a < b ? a : b, hi = a < b ? b : a;
         int64_t key = (int64_t)lo * nv + hi;
         uint64_t h = ((uint64_t)key * 0x9E3779B97F4A7C15ull) & (cap - 1);
         while (keys[h] != -1 && keys[h] != key) h = (h + 1) & (cap - 1);
         if (keys[h] == -1) {
            keys[h] = key;
            vals[h] = n_edges++;
         }
         eedge[4 * k + le] = vals[h];
      }
   }
   const int pe = p - 1, pi = (p - 1) * (p - 1), D1 = p + 1;
   const int64_t edge_base = nv, interior_base = nv + (int64_t)n_edges * pe;
   for (int k = 0; k < ne; k++) {
      const int *v = ev + 4 * k;
      int *d = elem_dofs + (int64_t)k * D1 * D1;
#define AT(a, b) d[(a) + (b) * D1]
      AT(0, 0) = v[0];
      AT(p, 0) = v[1];
      AT(p, p) = v[2];
      AT(0, p) = v[3];
#define EDOF(le, f, t, n) \
   (int)(edge_base + (int64_t)eedge[4 * k + (le)] * pe + (((f) < (t)) ? (n) - 1 : pe - (n)))
      for (int n = 1; n < p; n++) {
         AT(n, 0) = EDOF(0, v[0], v[1], n);
         AT(p, n) = EDOF(1, v[1], v[2], n);
         AT(n, p) = EDOF(2, v[3], v[2], n);
         AT(0, n) = EDOF(3, v[0], v[3], n);
      }
      for (int b = 1; b < p; b++)
         for (int a = 1; a < p; a++)
            AT(a, b) = (int)(interior_base + (int64_t)k * pi + (a - 1) + (b - 1) * (p - 1));
#undef EDOF
#undef AT
   }
   free(keys);
   free(vals);
   free(eedge);
   return interior_base + (int64_t)ne * pi;
}

/* Closed forms.  2D reproduces the discovery order of MeshTopology on
 * make_cartesian (elements i-fastest, local edges bottom/right/top/left): row
 * 0 creates 4 edges at i = 0 and 3 per later element, rows j >= 1 create 3 at
 * i = 0 and 2 per later element.  3D: canonical structured numbering. */
static int64_t edge_right(int nx, int i, int j)
{
   if (j == 0) return i == 0 ? 1 : 3 * (int64_t)i + 2;
   const int64_t base = (3 * (int64_t)nx + 1) + (int64_t)(j - 1) * (2 * nx + 1);
   return i == 0 ? base : base + 2 * (int64_t)i + 1;
}

static int64_t edge_top(int nx, int i, int j)
{
   if (j == 0) return i == 0 ? 2 : 3 * (int64_t)i + 3;
   const int64_t base = (3 * (int64_t)nx + 1) + (int64_t)(j - 1) * (2 * nx + 1);
   return i == 0 ? base + 1 : base + 2 * (int64_t)i + 2;
}

static int64_t edge_bottom(int nx, int i, int j)
{
   if (j == 0) return i == 0 ? 0 : 3 * (int64_t)i + 1;
   return edge_top(nx, i, j - 1);
}

static int64_t edge_left(int nx, int i, int j)
{
   if (i > 0) return edge_right(nx, i - 1, j);
   if (j == 0) return 3;
   const int64_t base = (3 * (int64_t)nx + 1) + (int64_t)(j - 1) * (2 * nx + 1);
   return base + 2;
}

int64_t orc_h1_layout_cartesian(int dim, const int *n, int p, int *elem_dofs)
{
   if (p < 1) return -fail(1, "build_h1_layout: order must be >= 1");
   const int D1 = p + 1, pe = p - 1;
   if (dim == 2) {
      const int nx = n[0], ny = n[1];
      const int64_t nv = (int64_t)(nx + 1) * (ny + 1);
      const int64_t n_edges = (int64_t)nx * (ny + 1) + (int64_t)ny * (nx + 1);
      const int64_t ib = nv + n_edges * pe;
      for (int j = 0; j < ny; j++)
         for (int i = 0; i < nx; i++) {
            const int64_t e = i + (int64_t)nx * j;
            int *d = elem_dofs + e * D1 * D1;
            const int64_t v0 = i + (int64_t)(nx + 1) * j;
            d[0] = (int)v0;
            d[p] = (int)(v0 + 1);
            d[p * D1 + p] = (int)(v0 + nx + 2);
            d[p * D1] = (int)(v0 + nx + 1);
            const int64_t eb = nv + edge_bottom(nx, i, j) * pe;
            const int64_t er = nv + edge_right(nx, i, j) * pe;
            const int64_t et = nv + edge_top(nx, i, j) * pe;
            const int64_t el = nv + edge_left(nx, i, j) * pe;
            for (int m = 1; m < p; m++) {
               d[m] = (int)(eb + m - 1);
               d[p + m * D1] = (int)(er + m - 1);
               d[m + p * D1] = (int)(et + m - 1);
               d[m * D1] = (int)(el + m - 1);
            }
            for (int b = 1; b < p; b++)
               for (int a = 1; a < p; a++)
                  d[a + b * D1] = (int)(ib + e * pe * pe + (a - 1) + (b - 1) * pe);
         }
      return ib + (int64_t)nx * ny * pe * pe;
   }
   const int nx = n[0], ny = n[1], nz = n[2];
   const int64_t nvx = nx + 1, nvy = ny + 1, nvz = nz + 1;
   const int64_t pf = (int64_t)pe * pe, pin = pf * pe;
   const int64_t NV = nvx * nvy * nvz;
   const int64_t EX = nx * nvy * nvz, EY = nvx * ny * nvz, EZ = nvx * nvy * nz;
   const int64_t FX = nvx * ny * nz, FY = nx * nvy * nz;
   const int64_t FZ = (int64_t)nx * ny * nvz;
   const int64_t exb = NV, eyb = exb + EX * pe, ezb = eyb + EY * pe;
   const int64_t fxb = ezb + EZ * pe, fyb = fxb + FX * pf, fzb = fyb + FY * pf;
   const int64_t ib = fzb + FZ * pf;
   for (int k = 0; k < nz; k++)
      for (int j = 0; j < ny; j++)
         for (int i = 0; i < nx; i++) {
            const int64_t e = i + nx * ((int64_t)j + ny * k);
            int *d = elem_dofs + e * D1 * D1 * D1;
            for (int c = 0; c <= p; c++)
               for (int b = 0; b <= p; b++)
                  for (int a = 0; a <= p; a++) {
                     const int ea = (a == 0 || a == p), eb = (b == 0 || b == p),
                               ec = (c == 0 || c == p);
                     const int ia = i + (a == p), jb = j + (b == p), kc = k + (c == p);
                     int64_t dof;
                     if (ea && eb && ec) {
                        dof = ia + nvx * (jb + nvy * kc);
                     } else if (!ea && eb && ec) {
                        dof = exb + (i + nx * (jb + nvy * kc)) * pe + (a - 1);
                     } else if (ea && !eb && ec) {
                        dof = eyb + (ia + nvx * (j + ny * kc)) * pe + (b - 1);
                     } else if (ea && eb && !ec) {
                        dof = ezb + (ia + nvx * (jb + nvy * k)) * pe + (c - 1);
                     } else if (ea && !eb && !ec) {
                        dof = fxb + (ia + nvx * (j + ny * (int64_t)k)) * pf + (b - 1) + pe * (c - 1);
                     } else if (!ea && eb && !ec) {
                        dof = fyb + (i + nx * (jb + nvy * k)) * pf + (a - 1) + pe * (c - 1);
                     } else if (!ea && !eb && ec) {
                        dof = fzb + (i + nx * (j + (int64_t)ny * kc)) * pf + (a - 1) + pe * (b - 1);
                     } else {
                        dof = ib + e * pin + (a - 1) + pe * ((b - 1) + (int64_t)pe * (c - 1));
                     }
                     d[a + D1 * (b + D1 * c)] = (int)dof;
                  }
         }
   return ib + (int64_t)nx * ny * nz * pin;
}

/* Boundary DOFs: every DOF at a lattice position on the domain boundary.  In
 * 2D this is the set essential_true_dofs builds from the boundary segments
 * (fespace.cpp:218-241), returned sorted. */
int64_t orc_boundary_dofs_cartesian(int dim, const int *n, int p, int *out)
{
   const int D1 = p + 1;
   const int nd = dim == 2 ? D1 * D1 : D1 * D1 * D1;
   const int64_t ne = orc_cartesian_ne(dim, n);
   int *dofs = malloc(sizeof(int) * (size_t)(ne * nd));
   const int64_t ndofs = orc_h1_layout_cartesian(dim, n, p, dofs);
   char *mark = calloc((size_t)ndofs, 1);
   const int nz = dim == 3 ? n[2] : 1;
   for (int k = 0; k < nz; k++)
      for (int j = 0; j < n[1]; j++)
         for (int i = 0; i < n[0]; i++) {
            const int64_t e = i + (int64_t)n[0] * (j + (int64_t)n[1] * k);
            for (int l = 0; l < nd; l++) {
               const int a = l % D1, b = (l / D1) % D1, c = l / (D1 * D1);
               const int64_t gi = (int64_t)i * p + a, gj = (int64_t)j * p + b;
               const int64_t gk = (int64_t)k * p + c;
               int on = gi == 0 || gi == (int64_t)n[0] * p || gj == 0 ||
                        gj == (int64_t)n[1] * p;
               if (dim == 3) on = on || gk == 0 || gk == (int64_t)n[2] * p;
               if (on) mark[dofs[e * nd + l]] = 1;
            }
         }
   int64_t cnt = 0;
   for (int64_t d = 0; d < ndofs; d++)
      if (mark[d]) {
         if (out) out[cnt] = (int)d;
         cnt++;
      }
   free(mark);
   free(dofs);
   return cnt;
}

/* ------------------------------------------------------------- geometry */

typedef struct {
   int m; /* geometry order */
   double nodes[ORC_MAX_Q], bary[ORC_MAX_Q];
} geom_basis;

static int geom_init(geom_basis *g, int m)
{
   g->m = m;
   return orc_basis_nodes(m, 0, g->nodes, g->bary);
}

/* ElementTransformation::jacobian and ::point (mesh.cpp:142-179); 3D loops
 * c, b, a outermost to innermost with weights (d * l) * l.  J[r][s] =
 * d x_r / d xh_s. */
static void geom_eval(const geom_basis *g, int dim, const double *ctrl,
                      const double *xh, double J[3][3], double *X)
{
   const int n = g->m + 1;
   double l[3][ORC_MAX_Q], dl[3][ORC_MAX_Q];
   for (int s = 0; s < dim; s++) orc_basis_eval(g->m, g->nodes, g->bary, xh[s], l[s], dl[s]);
   for (int r = 0; r < 3; r++) {
      for (int s = 0; s < 3; s++) J[r][s] = 0.0;
      if (X) X[r] = 0.0;
   }
   if (dim == 2) {
      for (int b = 0; b < n; b++)
         for (int a = 0; a < n; a++) {
            const double *c = ctrl + 2 * (a + b * n);
            const double wx = dl[0][a] * l[1][b];
            const double wy = l[0][a] * dl[1][b];
            J[0][0] += wx * c[0];
            J[1][0] += wx * c[1];
            J[0][1] += wy * c[0];
            J[1][1] += wy * c[1];
         }
      if (X) {
         /* point() recomputes values only (basis.cpp:48-60 overload). */
         double lv[2][ORC_MAX_Q];
         for (int s = 0; s < 2; s++) orc_basis_eval(g->m, g->nodes, g->bary, xh[s], lv[s], NULL);
         for (int b = 0; b < n; b++)
            for (int a = 0; a < n; a++) {
               const double *c = ctrl + 2 * (a + b * n);
               const double w = lv[0][a] * lv[1][b];
               X[0] += w * c[0];
               X[1] += w * c[1];
            }
      }
      return;
   }
   for (int cc = 0; cc < n; cc++)
      for (int b = 0; b < n; b++)
         for (int a = 0; a < n; a++) {
            const double *c = ctrl + 3 * (a + n * (b + n * cc));
            const double w0 = dl[0][a] * l[1][b] * l[2][cc];
            const double w1 = l[0][a] * dl[1][b] * l[2][cc];
            const double w2 = l[0][a] * l[1][b] * dl[2][cc];
            for (int r = 0; r < 3; r++) {
               J[r][0] += w0 * c[r];
               J[r][1] += w1 * c[r];
               J[r][2] += w2 * c[r];
            }
         }
   if (X) {
      double lv[3][ORC_MAX_Q];
      for (int s = 0; s < 3; s++) orc_basis_eval(g->m, g->nodes, g->bary, xh[s], lv[s], NULL);
      for (int cc = 0; cc < n; cc++)
         for (int b = 0; b < n; b++)
            for (int a = 0; a < n; a++) {
               const double *c = ctrl + 3 * (a + n * (b + n * cc));
               const double w = lv[0][a] * lv[1][b] * lv[2][cc];
               for (int r = 0; r < 3; r++) X[r] += w * c[r];
            }
   }
}

static double det_of(int dim, double J[3][3])
{
   if (dim == 2) return J[0][0] * J[1][1] - J[0][1] * J[1][0];
   return J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
          J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
          J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
}

int orc_physical_points(int dim, int geom_order, int64_t ne, const double *ctrl,
                        int nq, int rule_kind, double *xyz)
{
   geom_basis g;
   double pts[ORC_MAX_Q * 4], wts[ORC_MAX_Q * 4];
   int rc = geom_init(&g, geom_order);
   if (rc) return rc;
   rc = rule_points(nq, rule_kind, pts, wts);
   if (rc) return rc;
   const int nc = dim == 2 ? (geom_order + 1) * (geom_order + 1)
                           : (geom_order + 1) * (geom_order + 1) * (geom_order + 1);
   const int nqd = dim == 2 ? nq * nq : nq * nq * nq;
   for (int64_t e = 0; e < ne; e++) {
      for (int q = 0; q < nqd; q++) {
         double xh[3] = {pts[q % nq], pts[(q / nq) % nq], pts[q / (nq * nq)]};
         double J[3][3], X[3];
         geom_eval(&g, dim, ctrl + e * nc * dim, xh, J, X);
         for (int r = 0; r < dim; r++) xyz[(e * nqd + q) * dim + r] = X[r];
      }
   }
   return 0;
}

/* ----------------------------------------------------------------- setup */

/* pa_setup + point_factors + the Mesh::transformation det check
 * (forms.cpp:46-68, 201-229; mesh.cpp:243-260).  3D: D = (w c / det)
 * adj(J) adj(J)^T with adj(J) = det J^{-1}. */
int orc_pa_setup(int dim, int kind, int nq, int rule_kind, int geom_order,
                 int64_t ne, const double *ctrl, const double *coeff,
                 double coeff_const, double *qdata, int64_t *bad_elem)
{
   geom_basis g;
   double pts[ORC_MAX_Q * 4], wts[ORC_MAX_Q * 4];
   double cpts[ORC_MAX_Q * 4], cwts[ORC_MAX_Q * 4];
   int rc = geom_init(&g, geom_order);
   if (rc) return rc;
   if ((rc = rule_points(nq, rule_kind, pts, wts))) return rc;
   /* transformation() checks det J at the geometry_order + 2 Gauss points */
   const int nchk = geom_order + 2;
   if ((rc = orc_gauss_legendre(nchk, cpts, cwts))) return rc;
   const int nc = dim == 2 ? (geom_order + 1) * (geom_order + 1)
                           : (geom_order + 1) * (geom_order + 1) * (geom_order + 1);
   const int nqd = dim == 2 ? nq * nq : nq * nq * nq;
   const int ncomp = kind == 1 ? 1 : (dim == 2 ? 3 : 6);
   const int nchkd = dim == 2 ? nchk * nchk : nchk * nchk * nchk;
   for (int64_t e = 0; e < ne; e++) {
      const double *ce = ctrl + e * nc * dim;
      for (int q = 0; q < nchkd; q++) {
         double xh[3] = {cpts[q % nchk], cpts[(q / nchk) % nchk], cpts[q / (nchk * nchk)]};
         double J[3][3];
         geom_eval(&g, dim, ce, xh, J, NULL);
         if (!(det_of(dim, J) > 0.0)) {
            if (bad_elem) *bad_elem = e;
            char msg[96];
            snprintf(msg, sizeof msg, "Mesh::transformation: inverted element %lld",
                     (long long)e);
            return fail(2, msg);
         }
      }
      for (int q = 0; q < nqd; q++) {
         const int qx = q % nq, qy = (q / nq) % nq, qz = q / (nq * nq);
         double xh[3] = {pts[qx], pts[qy], pts[qz]};
         double J[3][3];
         geom_eval(&g, dim, ce, xh, J, NULL);
         const double det = det_of(dim, J);
         if (det <= 0.0) {
            if (bad_elem) *bad_elem = e;
            return fail(2, "forms: inverted element at a quadrature point");
         }
         const double c = coeff ? coeff[e * nqd + q] : coeff_const;
         if (!(c > 0.0)) {
            if (bad_elem) *bad_elem = e;
            return fail(1, "forms: coefficient must be positive");
         }
         const double wq = dim == 2 ? wts[qx] * wts[qy] : wts[qx] * wts[qy] * wts[qz];
         double *out = qdata + (e * nqd + q) * ncomp;
         if (kind == 1) {
            out[0] = wq * det * c;
            continue;
         }
         const double s = wq * c / det;
         if (dim == 2) {
            const double dxdx = J[0][0], dxdy = J[0][1], dydx = J[1][0], dydy = J[1][1];
            out[0] = s * (dxdy * dxdy + dydy * dydy);
            out[1] = -s * (dxdy * dxdx + dydy * dydx);
            out[2] = s * (dxdx * dxdx + dydx * dydx);
            continue;
         }
         double A[3][3]; /* adj(J)[s][r] */
         A[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
         A[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
         A[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
         A[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
         A[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
         A[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
         A[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
         A[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
         A[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
         static const int si[6] = {0, 0, 0, 1, 1, 2}, sj[6] = {0, 1, 2, 1, 2, 2};
         for (int t = 0; t < 6; t++) {
            const double *u = A[si[t]], *v = A[sj[t]];
            out[t] = s * ((u[0] * v[0] + u[1] * v[1]) + u[2] * v[2]);
         }
      }
   }
   return 0;
}

/* ----------------------------------------------------------------- apply */

/* One element of pa_apply_local, 2D (forms.cpp:248-286) with the exact
 * operation order of tensor_grad_2d / tensor_interp_2d and their transposes
 * (tensor_kernels.cpp:18-110). */
static void apply_elem_2d(int kind, int nd, int nq, const double *B,
                          const double *G, const double *d, const double *V,
                          double *out)
{
#define Bm(i, j) B[(i) * nd + (j)]
#define Gm(i, j) G[(i) * nd + (j)]
   double T1[ORC_MAX_Q][ORC_MAX_Q], T2[ORC_MAX_Q][ORC_MAX_Q];
   double ux[ORC_MAX_Q][ORC_MAX_Q], uy[ORC_MAX_Q][ORC_MAX_Q];
   double S1[ORC_MAX_Q][ORC_MAX_Q], S2[ORC_MAX_Q][ORC_MAX_Q];
   double vx[ORC_MAX_Q][ORC_MAX_Q], vy[ORC_MAX_Q][ORC_MAX_Q];
   if (kind == 1) {
      /* q = B V B^t: mat_mult then mat_mult_nt */
      for (int i = 0; i < nq; i++)
         for (int j = 0; j < nd; j++) T1[i][j] = 0.0;
      for (int i = 0; i < nq; i++)
         for (int k = 0; k < nd; k++) {
            const double aik = Bm(i, k);
            for (int j = 0; j < nd; j++) T1[i][j] += aik * V[k * nd + j];
         }
      for (int i = 0; i < nq; i++)
         for (int j = 0; j < nq; j++) {
            double s = 0.0;
            for (int k = 0; k < nd; k++) s += T1[i][k] * Bm(j, k);
            ux[i][j] = s;
         }
      for (int qy = 0; qy < nq; qy++)
         for (int qx = 0; qx < nq; qx++) ux[qx][qy] *= d[qy * nq + qx];
      /* B^t Q B: mat_mult_tn then mat_mult */
      for (int i = 0; i < nd; i++)
         for (int j = 0; j < nq; j++) S1[i][j] = 0.0;
      for (int k = 0; k < nq; k++)
         for (int i = 0; i < nd; i++) {
            const double aki = Bm(k, i);
            for (int j = 0; j < nq; j++) S1[i][j] += aki * ux[k][j];
         }
      for (int i = 0; i < nd; i++)
         for (int j = 0; j < nd; j++) vx[i][j] = 0.0;
      for (int i = 0; i < nd; i++)
         for (int k = 0; k < nq; k++) {
            const double aik = S1[i][k];
            for (int j = 0; j < nd; j++) vx[i][j] += aik * Bm(k, j);
         }
      for (int b = 0; b < nd; b++)
         for (int a = 0; a < nd; a++) out[b * nd + a] = vx[a][b];
      return;
   }
   for (int i = 0; i < nq; i++)
      for (int j = 0; j < nd; j++) T1[i][j] = T2[i][j] = 0.0;
   for (int i = 0; i < nq; i++)
      for (int k = 0; k < nd; k++) {
         const double gik = Gm(i, k);
         for (int j = 0; j < nd; j++) T1[i][j] += gik * V[k * nd + j];
      }
   for (int i = 0; i < nq; i++)
      for (int j = 0; j < nq; j++) {
         double s = 0.0;
         for (int k = 0; k < nd; k++) s += T1[i][k] * Bm(j, k);
         ux[i][j] = s;
      }
   for (int i = 0; i < nq; i++)
      for (int k = 0; k < nd; k++) {
         const double bik = Bm(i, k);
         for (int j = 0; j < nd; j++) T2[i][j] += bik * V[k * nd + j];
      }
   for (int i = 0; i < nq; i++)
      for (int j = 0; j < nq; j++) {
         double s = 0.0;
         for (int k = 0; k < nd; k++) s += T2[i][k] * Gm(j, k);
         uy[i][j] = s;
      }
   for (int qy = 0; qy < nq; qy++)
      for (int qx = 0; qx < nq; qx++) {
         const double *dq = d + (qy * nq + qx) * 3;
         const double gx = ux[qx][qy], gy = uy[qx][qy];
         ux[qx][qy] = dq[0] * gx + dq[1] * gy;
         uy[qx][qy] = dq[1] * gx + dq[2] * gy;
      }
   for (int i = 0; i < nd; i++)
      for (int j = 0; j < nq; j++) S1[i][j] = S2[i][j] = 0.0;
   for (int k = 0; k < nq; k++)
      for (int i = 0; i < nd; i++) {
         const double gki = Gm(k, i);
         for (int j = 0; j < nq; j++) S1[i][j] += gki * ux[k][j];
      }
   for (int i = 0; i < nd; i++)
      for (int j = 0; j < nd; j++) vx[i][j] = vy[i][j] = 0.0;
   for (int i = 0; i < nd; i++)
      for (int k = 0; k < nq; k++) {
         const double aik = S1[i][k];
         for (int j = 0; j < nd; j++) vx[i][j] += aik * Bm(k, j);
      }
   for (int k = 0; k < nq; k++)
      for (int i = 0; i < nd; i++) {
         const double bki = Bm(k, i);
         for (int j = 0; j < nq; j++) S2[i][j] += bki * uy[k][j];
      }
   for (int i = 0; i < nd; i++)
      for (int k = 0; k < nq; k++) {
         const double aik = S2[i][k];
         for (int j = 0; j < nd; j++) vy[i][j] += aik * Gm(k, j);
      }
   for (int i = 0; i < nd; i++)
      for (int j = 0; j < nd; j++) vx[i][j] += vy[i][j];
   for (int b = 0; b < nd; b++)
      for (int a = 0; a < nd; a++) out[b * nd + a] = vx[a][b];
#undef Bm
#undef Gm
}

/* 3D element: the 2D order extended axis by axis -- in: contract x, then y,
 * then z; out: contract qx, then qy, then qz; r = (vx + vy) + vz.  All sums
 * ascending and sequential. */
#define Q3 (ORC_MAX_Q * ORC_MAX_Q * ORC_MAX_Q)
static void apply_elem_3d(int kind, int nd, int nq, const double *B,
                          const double *G, const double *d, const double *V,
                          double *out)
{
   static _Thread_local double TB[Q3], TG[Q3], UBB[Q3], UBG[Q3], UGB[Q3];
   static _Thread_local double ux[Q3], uy[Q3], uz[Q3];
   static _Thread_local double Xx[Q3], Xy[Q3], Xz[Q3], Yx[Q3], Yy[Q3], Yz[Q3];
   static _Thread_local double vx[Q3], vy[Q3], vz[Q3];
#define Bm(i, j) B[(i) * nd + (j)]
#define Gm(i, j) G[(i) * nd + (j)]
   const int n1 = nd, q1 = nq;
   /* stage 1: [qx][b][c] = sum_a M(qx,a) V[a][b][c]; V index a + nd(b + nd c) */
   for (int c = 0; c < n1; c++)
      for (int b = 0; b < n1; b++)
         for (int qx = 0; qx < q1; qx++) {
            double sb = 0.0, sg = 0.0;
            for (int a = 0; a < n1; a++) {
               const double v = V[a + n1 * (b + n1 * c)];
               sb += Bm(qx, a) * v;
               sg += Gm(qx, a) * v;
            }
            TB[qx + q1 * (b + n1 * c)] = sb;
            TG[qx + q1 * (b + n1 * c)] = sg;
         }
   /* stage 2: [qx][qy][c] */
   for (int c = 0; c < n1; c++)
      for (int qy = 0; qy < q1; qy++)
         for (int qx = 0; qx < q1; qx++) {
            double bb = 0.0, bg = 0.0, gb = 0.0;
            for (int b = 0; b < n1; b++) {
               const double tb = TB[qx + q1 * (b + n1 * c)];
               const double tg = TG[qx + q1 * (b + n1 * c)];
               bb += Bm(qy, b) * tb;
               bg += Gm(qy, b) * tb;
               gb += Bm(qy, b) * tg;
            }
            UBB[qx + q1 * (qy + q1 * c)] = bb;
            UBG[qx + q1 * (qy + q1 * c)] = bg;
            UGB[qx + q1 * (qy + q1 * c)] = gb;
         }
   /* stage 3: [qx][qy][qz] */
   for (int qz = 0; qz < q1; qz++)
      for (int qy = 0; qy < q1; qy++)
         for (int qx = 0; qx < q1; qx++) {
            double sx = 0.0, sy = 0.0, sz = 0.0;
            for (int c = 0; c < n1; c++) {
               const int i = qx + q1 * (qy + q1 * c);
               if (kind == 1) {
                  sx += Bm(qz, c) * UBB[i];
               } else {
                  sx += Bm(qz, c) * UGB[i];
                  sy += Bm(qz, c) * UBG[i];
                  sz += Gm(qz, c) * UBB[i];
               }
            }
            const int q = qx + q1 * (qy + q1 * qz);
            if (kind == 1) {
               ux[q] = sx * d[q];
            } else {
               const double *D = d + 6 * q;
               ux[q] = (D[0] * sx + D[1] * sy) + D[2] * sz;
               uy[q] = (D[1] * sx + D[3] * sy) + D[4] * sz;
               uz[q] = (D[2] * sx + D[4] * sy) + D[5] * sz;
            }
         }
   /* transpose stage 1: [a][qy][qz] = sum_qx M(qx,a) w[qx][qy][qz] */
   for (int qz = 0; qz < q1; qz++)
      for (int qy = 0; qy < q1; qy++)
         for (int a = 0; a < n1; a++) {
            double sx = 0.0, sy = 0.0, sz = 0.0;
            for (int qx = 0; qx < q1; qx++) {
               const int q = qx + q1 * (qy + q1 * qz);
               if (kind == 1) {
                  sx += Bm(qx, a) * ux[q];
               } else {
                  sx += Gm(qx, a) * ux[q];
                  sy += Bm(qx, a) * uy[q];
                  sz += Bm(qx, a) * uz[q];
               }
            }
            const int o = a + n1 * (qy + q1 * qz);
            Xx[o] = sx;
            Xy[o] = sy;
            Xz[o] = sz;
         }
   /* transpose stage 2: [a][b][qz] */
   for (int qz = 0; qz < q1; qz++)
      for (int b = 0; b < n1; b++)
         for (int a = 0; a < n1; a++) {
            double sx = 0.0, sy = 0.0, sz = 0.0;
            for (int qy = 0; qy < q1; qy++) {
               const int i = a + n1 * (qy + q1 * qz);
               if (kind == 1) {
                  sx += Bm(qy, b) * Xx[i];
               } else {
                  sx += Bm(qy, b) * Xx[i];
                  sy += Gm(qy, b) * Xy[i];
                  sz += Bm(qy, b) * Xz[i];
               }
            }
            const int o = a + n1 * (b + n1 * qz);
            Yx[o] = sx;
            Yy[o] = sy;
            Yz[o] = sz;
         }
   /* transpose stage 3: [a][b][c] */
   for (int c = 0; c < n1; c++)
      for (int b = 0; b < n1; b++)
         for (int a = 0; a < n1; a++) {
            double sx = 0.0, sy = 0.0, sz = 0.0;
            for (int qz = 0; qz < q1; qz++) {
               const int i = a + n1 * (b + n1 * qz);
               if (kind == 1) {
                  sx += Bm(qz, c) * Yx[i];
               } else {
                  sx += Bm(qz, c) * Yx[i];
                  sy += Bm(qz, c) * Yy[i];
                  sz += Gm(qz, c) * Yz[i];
               }
            }
            const int o = a + n1 * (b + n1 * c);
            vx[o] = sx;
            vy[o] = sy;
            vz[o] = sz;
         }
   const int nd3 = n1 * n1 * n1;
   for (int i = 0; i < nd3; i++) out[i] = kind == 1 ? vx[i] : (vx[i] + vy[i]) + vz[i];
#undef Bm
#undef Gm
}

/* pa_apply_local (forms.cpp:231-296): element results, then the
 * element-ordered scatter y[dofs[i]] += out[i]. */
void orc_pa_apply_local(int dim, int kind, int p, int nq, int64_t ne,
                        const double *B, const double *G, const double *qdata,
                        const int *elem_dofs, const double *x, double *y,
                        uint64_t *mults)
{
   const int nd = p + 1;
   const int ndd = dim == 2 ? nd * nd : nd * nd * nd;
   const int nqd = dim == 2 ? nq * nq : nq * nq * nq;
   const int ncomp = kind == 1 ? 1 : (dim == 2 ? 3 : 6);
   double V[Q3], out[Q3];
   for (int64_t e = 0; e < ne; e++) {
      const int *dofs = elem_dofs + e * ndd;
      const double *d = qdata + e * nqd * ncomp;
      if (dim == 2) {
         /* V stored [a][b] (x node, y node): v(a,b) = x[dofs[b*nd+a]] */
         for (int b = 0; b < nd; b++)
            for (int a = 0; a < nd; a++) V[a * nd + b] = x[dofs[b * nd + a]];
         apply_elem_2d(kind, nd, nq, B, G, d, V, out);
      } else {
         for (int i = 0; i < ndd; i++) V[i] = x[dofs[i]];
         apply_elem_3d(kind, nd, nq, B, G, d, V, out);
      }
      for (int i = 0; i < ndd; i++) y[dofs[i]] += out[i];
   }
   if (mults) {
      const uint64_t a = nd, q = nq;
      uint64_t per;
      if (dim == 2)
         per = kind == 1 ? 2 * (q * a * a + q * q * a) + q * q
                         : 4 * (q * a * a + q * q * a) + 4 * q * q;
      else
         per = kind == 1 ? 2 * (q * a * a * a + q * q * a * a + q * q * q * a) + q * q * q
                         : 2 * (2 * q * a * a * a + 3 * q * q * a * a + 3 * q * q * q * a) +
                              9 * q * q * q;
      *mults += per * (uint64_t)ne;
   }
}

/* Dense tabulated basis at the point lattice (forms.cpp:22-42): rows points,
 * columns DOFs, both x fastest. */
static void tab_entry(int dim, int nd, int nq, const double *B, const double *G,
                      int q, int i, double *b, double *g)
{
   const int qx = q % nq, qy = (q / nq) % nq, qz = q / (nq * nq);
   const int a = i % nd, bb = (i / nd) % nd, c = i / (nd * nd);
   const double Bx = B[qx * nd + a], By = B[qy * nd + bb];
   const double Gx = G[qx * nd + a], Gy = G[qy * nd + bb];
   if (dim == 2) {
      *b = Bx * By;
      g[0] = Gx * By;
      g[1] = Bx * Gy;
      return;
   }
   const double Bz = B[qz * nd + c], Gz = G[qz * nd + c];
   *b = Bx * By * Bz;
   g[0] = Gx * By * Bz;
   g[1] = Bx * Gy * Bz;
   g[2] = Bx * By * Gz;
}

/* pa_diagonal, unconstrained elements (forms.cpp:311-348). */
void orc_pa_diagonal(int dim, int kind, int p, int nq, int64_t ne,
                     const double *B, const double *G, const double *qdata,
                     const int *elem_dofs, double *diag)
{
   const int nd = p + 1;
   const int ndd = dim == 2 ? nd * nd : nd * nd * nd;
   const int nqd = dim == 2 ? nq * nq : nq * nq * nq;
   const int ncomp = kind == 1 ? 1 : (dim == 2 ? 3 : 6);
   for (int64_t e = 0; e < ne; e++) {
      const int *dofs = elem_dofs + e * ndd;
      const double *d = qdata + e * nqd * ncomp;
      for (int i = 0; i < ndd; i++) {
         double s = 0.0;
         for (int q = 0; q < nqd; q++) {
            double b, g[3];
            tab_entry(dim, nd, nq, B, G, q, i, &b, g);
            if (kind == 1) {
               s += b * b * d[q];
            } else if (dim == 2) {
               const double gx = g[0], gy = g[1];
               s += gx * gx * d[3 * q] + 2.0 * gx * gy * d[3 * q + 1] +
                    gy * gy * d[3 * q + 2];
            } else {
               const double *D = d + 6 * q;
               s += g[0] * g[0] * D[0] + 2.0 * g[0] * g[1] * D[1] +
                    2.0 * g[0] * g[2] * D[2] + g[1] * g[1] * D[3] +
                    2.0 * g[1] * g[2] * D[4] + g[2] * g[2] * D[5];
            }
         }
         diag[dofs[i]] += s;
      }
   }
}

/* local_matrix_tabulated on stored point factors (forms.cpp:70-104). */
void orc_element_matrix(int dim, int kind, int p, int nq, const double *B,
                        const double *G, const double *d, double *mat)
{
   const int nd = p + 1;
   const int ndd = dim == 2 ? nd * nd : nd * nd * nd;
   const int nqd = dim == 2 ? nq * nq : nq * nq * nq;
   memset(mat, 0, sizeof(double) * ndd * ndd);
   for (int q = 0; q < nqd; q++) {
      for (int i = 0; i < ndd; i++) {
         double bi, gi[3];
         tab_entry(dim, nd, nq, B, G, q, i, &bi, gi);
         if (kind == 1) {
            const double fb = d[q] * bi;
            for (int j = 0; j < ndd; j++) {
               double bj, gj[3];
               tab_entry(dim, nd, nq, B, G, q, j, &bj, gj);
               mat[i * ndd + j] += fb * bj;
            }
            continue;
         }
         double a[3];
         if (dim == 2) {
            const double *f = d + 3 * q;
            a[0] = f[0] * gi[0] + f[1] * gi[1];
            a[1] = f[1] * gi[0] + f[2] * gi[1];
         } else {
            const double *f = d + 6 * q;
            a[0] = (f[0] * gi[0] + f[1] * gi[1]) + f[2] * gi[2];
            a[1] = (f[1] * gi[0] + f[3] * gi[1]) + f[4] * gi[2];
            a[2] = (f[2] * gi[0] + f[4] * gi[1]) + f[5] * gi[2];
         }
         for (int j = 0; j < ndd; j++) {
            double bj, gj[3];
            tab_entry(dim, nd, nq, B, G, q, j, &bj, gj);
            double v = a[0] * gj[0] + a[1] * gj[1];
            if (dim == 3) v += a[2] * gj[2];
            mat[i * ndd + j] += v;
         }
      }
   }
}

/* -------------------------------------------------------------- operator */

/* ConstrainedOperator::mult over BilinearForm::mult_true with P = I
 * (forms.cpp:173-184, 527-543). */
void orc_op_mult(const orc_pa_operator *op, const double *x, double *y)
{
   const int64_t n = op->ndofs;
   double *z = malloc(sizeof(double) * n);
   memcpy(z, x, sizeof(double) * n);
   for (int64_t i = 0; i < op->n_ess; i++) z[op->ess[i]] = 0.0;
   memset(y, 0, sizeof(double) * n);
   for (int k = 0; k < op->n_integ; k++)
      orc_pa_apply_local(op->dim, op->kinds[k], op->p, op->nq, op->ne, op->B,
                         op->G, op->qdata[k], op->elem_dofs, z, y, NULL);
   for (int64_t i = 0; i < op->n_ess; i++) y[op->ess[i]] = x[op->ess[i]];
   free(z);
}

static double vdot(int64_t n, const double *a, const double *b)
{
   double s = 0.0;
   for (int64_t i = 0; i < n; i++) s += a[i] * b[i];
   return s;
}

typedef void (*mult_fn)(const void *ctx, const double *x, double *y);

/* cg_solve (solvers.cpp:11-97), Vector ops as in vector.cpp:13-36. */
static int cg_generic(mult_fn mult, const void *ctx, int64_t n, const double *b,
                      double rel_tol, int max_iters, const double *diag,
                      double *x, int *iters, int *converged)
{
   if (diag) {
      for (int64_t i = 0; i < n; i++)
         if (!(diag[i] > 0.0))
            return fail(1, "cg_solve: Jacobi diagonal must be strictly positive");
   }
   memset(x, 0, sizeof(double) * n);
   *iters = 0;
   *converged = 0;
   const double bnorm = sqrt(vdot(n, b, b));
   if (!isfinite(bnorm)) return fail(2, "cg_solve: right-hand side is not finite");
   const double target = rel_tol * bnorm;
   if (bnorm == 0.0) {
      *converged = 1;
      return 0;
   }
   double *r = malloc(sizeof(double) * n), *z = malloc(sizeof(double) * n);
   double *q = malloc(sizeof(double) * n), *p = malloc(sizeof(double) * n);
   double *best = calloc((size_t)n, sizeof(double));
   int rc = 0;
   memcpy(r, b, sizeof(double) * n);
   for (int64_t i = 0; i < n; i++) z[i] = diag ? r[i] / diag[i] : r[i];
   memcpy(p, z, sizeof(double) * n);
   double rz = vdot(n, r, z);
   double rnorm = sqrt(vdot(n, r, r));
   double best_rnorm = rnorm;
   int done = 0;
   for (int it = 1; it <= max_iters; it++) {
      if (rnorm <= target) {
         *converged = 1;
         *iters = it - 1;
         done = 1;
         break;
      }
      mult(ctx, p, q);
      const double pq = vdot(n, p, q);
      const double alpha = rz / pq;
      if (!isfinite(alpha)) {
         rc = fail(2, "cg_solve: breakdown (non-finite step)");
         goto out;
      }
      for (int64_t i = 0; i < n; i++) x[i] += alpha * p[i];
      const double nalpha = -alpha;
      for (int64_t i = 0; i < n; i++) r[i] += nalpha * q[i];
      rnorm = sqrt(vdot(n, r, r));
      if (!isfinite(rnorm)) {
         rc = fail(2, "cg_solve: breakdown (non-finite residual)");
         goto out;
      }
      if (rnorm < best_rnorm) {
         best_rnorm = rnorm;
         memcpy(best, x, sizeof(double) * n);
      }
      for (int64_t i = 0; i < n; i++) z[i] = diag ? r[i] / diag[i] : r[i];
      const double rz_next = vdot(n, r, z);
      const double beta = rz_next / rz;
      rz = rz_next;
      for (int64_t i = 0; i < n; i++) p[i] = z[i] + beta * p[i];
   }
   if (!done) {
      *iters = max_iters;
      if (rnorm <= target) {
         *converged = 1;
      } else {
         memcpy(x, best, sizeof(double) * n);
      }
   }
out:
   free(r);
   free(z);
   free(q);
   free(p);
   free(best);
   return rc;
}

static void pa_mult_cb(const void *ctx, const double *x, double *y)
{
   orc_op_mult((const orc_pa_operator *)ctx, x, y);
}

int orc_cg_pa(const orc_pa_operator *op, const double *b, double rel_tol,
              int max_iters, const double *diag, double *x, int *iters,
              int *converged)
{
   return cg_generic(pa_mult_cb, op, op->ndofs, b, rel_tol, max_iters, diag, x,
                     iters, converged);
}

typedef struct {
   int n;
   const int *rowptr, *cols;
   const double *vals;
} csr_ctx;

/* SparseMatrix::mult (sparse.cpp:75-87). */
static void csr_mult_cb(const void *ctx, const double *x, double *y)
{
   const csr_ctx *c = ctx;
   for (int i = 0; i < c->n; i++) {
      double s = 0.0;
      for (int k = c->rowptr[i]; k < c->rowptr[i + 1]; k++) s += c->vals[k] * x[c->cols[k]];
      y[i] = s;
   }
}

int orc_cg_csr(int n, const int *rowptr, const int *cols, const double *vals,
               const double *b, double rel_tol, int max_iters,
               const double *diag, double *x, int *iters, int *converged)
{
   csr_ctx c = {n, rowptr, cols, vals};
   return cg_generic(csr_mult_cb, &c, n, b, rel_tol, max_iters, diag, x, iters,
                     converged);
}
