/*
 * ORACLE INFRASTRUCTURE -- CPU restatement of the reference algorithm for
 * the PA operator / Jacobi-CG hot path.  Test / benchmark checker only:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load liboracle.so.  Never linked into the product.
 *
 * Parity status:
 *   - 2D (quads): pinned bit-for-bit against the reference itself
 *     (oracle/_ref/libtfem_ref.so, tests/test_oracle_ref.py) and against the
 *     committed goldens in tests/golden/ made from it.
 *   - 3D (hexes) and BP5 (q = p+1 Gauss-Lobatto): NOT expressible through the
 *     reference API -- parity unpinned at the reference
 *     level; pinned by the restatement's own checks (dense element matrix vs
 *     PA, volume / constant / patch tests, 2D-slab cross checks), see
 *     tests/test_oracle_3d.py.
 *
 * Conventions (all arrays row-major, C doubles / int32):
 *   dim in {2,3}; p = order; D1 = p+1; nq = points per axis;
 *   element DOFs: D1^dim entries, x fastest (mesh.hpp:85-95);
 *   qdata: reference layout [e][q][c], q x fastest (forms.cpp:219-225);
 *   diffusion components: 2D {00,01,11}; 3D {00,01,02,11,12,22}.
 * Status codes: 0 ok, 1 invalid_argument, 2 runtime_error, 3 logic_error.
 */
#ifndef TFEM_ORACLE_H
#define TFEM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_P 8
#define ORC_MAX_Q 12

/* 1D rules on [0,1] (quadrature.cpp:64-125). */
int orc_gauss_legendre(int n, double *pts, double *wts);
int orc_gauss_lobatto(int n, double *pts, double *wts);

/* Basis1D nodes + barycentric weights; node_kind 0 GLL, 1 GL, 2 uniform
 * (basis.cpp:12-46). */
int orc_basis_nodes(int p, int node_kind, double *nodes, double *bary);
/* values (and derivs if non-null) of the p+1 Lagrange polynomials at x
 * (basis.cpp:48-93). */
void orc_basis_eval(int p, const double *nodes, const double *bary, double x,
                    double *values, double *derivs);
/* B1d/G1d, nq x (p+1) (basis.cpp:95-109); rule_kind 0 GL, 1 GLL. */
int orc_eval_matrices(int p, int node_kind, int nq, int rule_kind, double *B,
                      double *G);

/* Cartesian meshes (mesh.cpp:283-321 and its 3D analogue): n[dim] cells,
 * ext[dim] extents.  Vertices i-fastest; elements i-fastest with corner order
 * 2D: CCW (v0..v3); 3D: bottom CCW then top CCW (v0..v7). */
int64_t orc_cartesian_nv(int dim, const int *n);
int64_t orc_cartesian_ne(int dim, const int *n);
void orc_cartesian_vertices(int dim, const int *n, const double *ext,
                            double *coords);
void orc_cartesian_elements(int dim, const int *n, int *elem_vertices);
/* Straight-element geometry control points in lattice order (x fastest),
 * E x 2^dim x dim (mesh.cpp:238-240). */
void orc_cartesian_ctrl(int dim, const int *n, const double *ext,
                        double *ctrl);

/* H1 DOF layouts.  2D: the reference numbering (vertices, edges in
 * discovery order, interiors; mesh.cpp:26-115) for an arbitrary conforming
 * quad mesh.  Returns n_dofs (<0 on error). */
int64_t orc_h1_layout_quads(int nv, int ne, const int *elem_vertices, int p,
                            int *elem_dofs);
/* Cartesian layouts: 2D identical to orc_h1_layout_quads on
 * orc_cartesian_elements (closed form); 3D the canonical structured
 * numbering documented in DESIGN.md (vertices, x/y/z edges, x/y/z-normal
 * faces, interiors). */
int64_t orc_h1_layout_cartesian(int dim, const int *n, int p, int *elem_dofs);
/* Sorted DOFs on the whole boundary of a Cartesian mesh (2D: identical to
 * FeSpace::essential_true_dofs over all attributes, fespace.cpp:205-242). */
int64_t orc_boundary_dofs_cartesian(int dim, const int *n, int p, int *out);

/* Physical quadrature points E x nq^dim x dim (mesh.cpp:142-157). */
int orc_physical_points(int dim, int geom_order, int64_t ne,
                        const double *ctrl, int nq, int rule_kind,
                        double *xyz);

/* PA setup (forms.cpp:46-68, 201-229; mesh.cpp:243-260): kind 0 diffusion,
 * 1 mass; coefficient per point (E x nq^dim, may be null) else coeff_const.
 * rule_kind 0: Gauss-Legendre nq (reference: nq = p+2); 1: Gauss-Lobatto.
 * On error *bad_elem holds the element. */
int orc_pa_setup(int dim, int kind, int nq, int rule_kind, int geom_order,
                 int64_t ne, const double *ctrl, const double *coeff,
                 double coeff_const, double *qdata, int64_t *bad_elem);

/* y += G^T B^T D B G x over all elements in element order
 * (forms.cpp:231-296; tensor_kernels.cpp:18-110).  `mults` (nullable) gets
 * the multiply count the instrumented reference would report. */
void orc_pa_apply_local(int dim, int kind, int p, int nq, int64_t ne,
                        const double *B, const double *G, const double *qdata,
                        const int *elem_dofs, const double *x, double *y,
                        uint64_t *mults);

/* diag += exact diagonal, dense tabulated tables (forms.cpp:311-348). */
void orc_pa_diagonal(int dim, int kind, int p, int nq, int64_t ne,
                     const double *B, const double *G, const double *qdata,
                     const int *elem_dofs, double *diag);

/* Dense element matrix by direct quadrature (forms.cpp:70-104, 384-398). */
void orc_element_matrix(int dim, int kind, int p, int nq, const double *B,
                        const double *G, const double *qdata_e, double *mat);

/* A conforming PA operator (P = I) with an optional essential set -- the
 * ConstrainedOperator of forms.cpp:164-190 when n_ess > 0. */
typedef struct {
   int dim, p, nq;
   int64_t ne, ndofs;
   const double *B, *G;
   int n_integ;
   const int *kinds;
   const double *const *qdata;
   const int *elem_dofs;
   int64_t n_ess;
   const int *ess;
} orc_pa_operator;

void orc_op_mult(const orc_pa_operator *op, const double *x, double *y);

/* cg_solve (solvers.cpp:11-97) on the PA operator.  diag nullable. */
int orc_cg_pa(const orc_pa_operator *op, const double *b, double rel_tol,
              int max_iters, const double *diag, double *x, int *iters,
              int *converged);
/* cg_solve on a CSR matrix. */
int orc_cg_csr(int n, const int *rowptr, const int *cols, const double *vals,
               const double *b, double rel_tol, int max_iters,
               const double *diag, double *x, int *iters, int *converged);

const char *orc_last_error(void);

#ifdef __cplusplus
}
#endif

#endif
