/*
 * tfem_cuda.h -- C ABI of libtfem_cuda.so, the B200 (sm_100a) partial-
 * assembly (PA) operator + Jacobi-CG path of tensorfem.
 *
 * This is the drop-in boundary of the reference's hot path
 * (/root/reference/proj, "tensorfem").  Plain C types only:
 * pointers, sizes, int status codes.  Every entry point names the reference
 * interface it replaces (file:line relative to /root/reference/proj).  The
 * reference-side binding (the lines a maintainer adds to forms.cpp /
 * solvers.cpp) is shown in INTEGRATION.md.
 *
 * Conventions
 *  - Status: TFEM_OK (0) or the reference's exception class:
 *      TFEM_INVALID_ARGUMENT  <-> std::invalid_argument
 *      TFEM_RUNTIME_ERROR     <-> std::runtime_error
 *      TFEM_LOGIC_ERROR       <-> std::logic_error
 *      TFEM_CUDA_ERROR        device / driver failure
 *    with the message text (same prefix as the reference's exception) in the
 *    calling thread's tfem_last_error().
 *  - Synchronous: every call has completed on the device when it returns
 *    (SPEC.md:517), unless its name ends in _async.
 *  - Device data: vectors live in HBM (tfem_vec); host arrays are copied in
 *    by the create/upload calls.  A context owns one CUDA stream.
 *  - DOF orders follow the reference: element DOFs x fastest
 *    (mesh.hpp:85-95); quadrature points x fastest; qdata host layout
 *    [e][q][c] (forms.cpp:219-225).  Device layouts are internal.
 *  - Numerics: the default TFEM_NUMERICS_FMA fuses multiply-adds (results
 *    within 1e-15 relative of the reference; the north-star bar is 1e-12);
 *    TFEM_NUMERICS_REFERENCE evaluates the 2D operator in the reference's
 *    exact operation order (no FMA), bit-identical to the CPU reference, at
 *    ~15 % lower throughput.  3D (no reference) always fuses.
 */
#ifndef TFEM_CUDA_H
#define TFEM_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TFEM_OK 0
#define TFEM_INVALID_ARGUMENT 1
#define TFEM_RUNTIME_ERROR 2
#define TFEM_LOGIC_ERROR 3
#define TFEM_CUDA_ERROR 4

/* IntegratorKind (forms.hpp:18) */
#define TFEM_DIFFUSION 0
#define TFEM_MASS 1

/* Quadrature rule families (quadrature.hpp:22,26) */
#define TFEM_GAUSS_LEGENDRE 0
#define TFEM_GAUSS_LOBATTO 1

/* Node families of Basis1D (basis.hpp:15) */
#define TFEM_NODES_GAUSS_LOBATTO 0
#define TFEM_NODES_GAUSS_LEGENDRE 1
#define TFEM_NODES_UNIFORM 2

#define TFEM_NUMERICS_REFERENCE 0
#define TFEM_NUMERICS_FMA 1

typedef struct tfem_ctx tfem_ctx;
typedef struct tfem_vec tfem_vec;
typedef struct tfem_restriction tfem_restriction;
typedef struct tfem_geometry tfem_geometry;
typedef struct tfem_pa tfem_pa;
typedef struct tfem_operator tfem_operator;
typedef struct tfem_prolongation tfem_prolongation;
typedef struct tfem_nccl tfem_nccl;

/* ------------------------------------------------------------- errors */
const char *tfem_last_error(void);
const char *tfem_version(void);

/* ------------------------------------------------------------ context */
/* One device + one stream.  `device` < 0 selects the current device. */
int tfem_ctx_create(int device, tfem_ctx **out);
int tfem_ctx_destroy(tfem_ctx *ctx);
int tfem_ctx_sync(tfem_ctx *ctx);
/* The context's cudaStream_t, for interop (e.g. torch.cuda.ExternalStream). */
void *tfem_ctx_stream(tfem_ctx *ctx);
int tfem_ctx_set_numerics(tfem_ctx *ctx, int mode);
/* Kernel launches issued through this context since creation. */
int64_t tfem_ctx_launch_count(const tfem_ctx *ctx);
/* Test hook (no reference counterpart): cap the persistent element kernels'
 * grids at max_blocks blocks (0 = one per SM, the default), so a small mesh
 * runs many laps of every block's pipeline ring -- the steady state the
 * parity tests must reach without the CPU oracle timing out. */
int tfem_ctx_set_max_blocks(tfem_ctx *ctx, int max_blocks);

/* -------------------------------------------------------------- memory */
/* Caching allocators behind the device-resident Vector of the reference-side
 * binding (the Memory / Read-Write mirror of PAPER.md:1664-1689; vector.hpp:
 * 14-48 is host-only).  Device blocks are per context and reused in stream
 * order; host blocks are pinned (cudaHostAllocPortable) and cached, with a
 * pageable fallback when no device exists.  Sizes are rounded to 512 B
 * below 1 MiB and 2 MiB above. */
int tfem_mem_alloc(tfem_ctx *ctx, size_t bytes, void **out);
int tfem_mem_free(tfem_ctx *ctx, void *p);
int tfem_mem_trim(tfem_ctx *ctx); /* cudaFree the cached device blocks */
int tfem_host_alloc(size_t bytes, void **out);
int tfem_host_free(void *p);
/* Any-direction copy (cudaMemcpyDefault) on the context stream, synchronous. */
int tfem_copy(tfem_ctx *ctx, void *dst, const void *src, size_t bytes);

/* -------------------------------------------- 1D rules and basis tables */
/* gauss_legendre / gauss_lobatto on [0,1] (quadrature.cpp:64-125). */
int tfem_quadrature(int rule, int n, double *points, double *weights);
/* eval_matrices(Basis1D(p, node_kind), rule(nq)) -> B1d, G1d, nq x (p+1)
 * row-major (basis.cpp:95-109). */
int tfem_eval_matrices(int p, int node_kind, int nq, int rule, double *B,
                       double *G);

/* ------------------------------------------------------------ vectors */
/* Vector (vector.hpp:14-48) resident in HBM. */
int tfem_vec_create(tfem_ctx *ctx, int64_t n, tfem_vec **out);
/* Non-owning view of existing device memory (e.g. a torch tensor). */
int tfem_vec_wrap(tfem_ctx *ctx, double *device_ptr, int64_t n, tfem_vec **out);
int tfem_vec_destroy(tfem_vec *v);
int64_t tfem_vec_size(const tfem_vec *v);
double *tfem_vec_data(tfem_vec *v);
int tfem_vec_upload(tfem_vec *v, const double *host, int64_t n);
int tfem_vec_download(const tfem_vec *v, double *host, int64_t n);
int tfem_vec_fill(tfem_vec *v, double value);
/* Vector::dot / axpy / norm2 (vector.cpp:13-36).  Deterministic (fixed-shape
 * tree reduction), not sequential: results differ from the CPU by round-off. */
int tfem_vec_dot(tfem_ctx *ctx, const tfem_vec *a, const tfem_vec *b,
                 double *out);
int tfem_vec_axpy(tfem_ctx *ctx, double a, const tfem_vec *x, tfem_vec *y);

/* ------------------------------------------- element restriction (G, G^T) */
/* The element -> DOF map of FeSpace::element_dofs (fespace.hpp:64), host
 * array [e][i] with D1^dim entries per element.  Builds the deterministic
 * transpose (DOF -> element slots sorted by element) on the device. */
int tfem_restriction_create(tfem_ctx *ctx, int dim, int p, int64_t n_elem,
                            int64_t n_dofs, const int32_t *elem_dofs,
                            tfem_restriction **out);
/* The same map generated on the device for an n[0] x ... Cartesian mesh:
 * 2D reproduces build_h1_layout on make_cartesian bit for bit
 * (mesh.cpp:65-115, 283-321); 3D uses the canonical numbering of DESIGN.md. */
int tfem_restriction_cartesian(tfem_ctx *ctx, int dim, const int *n, int p,
                               tfem_restriction **out);
int tfem_restriction_destroy(tfem_restriction *r);
int64_t tfem_restriction_n_dofs(const tfem_restriction *r);
int64_t tfem_restriction_n_elem(const tfem_restriction *r);
/* Download the map in the reference layout [e][i]. */
int tfem_restriction_elem_dofs(const tfem_restriction *r, int32_t *host);
/* Sorted DOFs on the boundary of a Cartesian restriction; count only when
 * host == NULL (FeSpace::essential_true_dofs, fespace.cpp:205-242). */
int tfem_restriction_boundary_dofs(const tfem_restriction *r, int32_t *host,
                                   int64_t *count);
/* ElementRestriction::Mult (L -> E, e-vector [e][i]) and MultTranspose
 * (E -> L, y += in element order) (forms.cpp:250-255, 289-295). */
int tfem_restriction_mult(tfem_ctx *ctx, const tfem_restriction *r,
                          const tfem_vec *l, tfem_vec *e);
int tfem_restriction_mult_transpose(tfem_ctx *ctx, const tfem_restriction *r,
                                    const tfem_vec *e, tfem_vec *l);

/* ----------------------------------------------------------- geometry */
/* Element maps of Mesh::transformation (mesh.cpp:131-179, 228-260): order-m
 * Gauss-Lobatto nodal geometry; control points E x (m+1)^dim x dim in
 * lattice order (x fastest).  Straight quads: m = 1, corners v0, v1, v3, v2
 * (mesh.cpp:238-240). */
int tfem_geometry_create(tfem_ctx *ctx, int dim, int order, int64_t n_elem,
                         const double *ctrl, tfem_geometry **out);
/* make_cartesian(n, ext) generated on the device (mesh.cpp:283-321). */
int tfem_geometry_cartesian(tfem_ctx *ctx, int dim, const int *n,
                            const double *ext, tfem_geometry **out);
/* The n_local block at cell offset `origin` of make_cartesian(n_global, ext):
 * vertex coordinates are ext * (origin + i) / n_global, bit-identical to the
 * global mesh (one rank's slab in an element-partitioned run). */
int tfem_geometry_cartesian_box(tfem_ctx *ctx, int dim, const int *n_local,
                                const int *origin, const int *n_global,
                                const double *ext, tfem_geometry **out);
int tfem_geometry_destroy(tfem_geometry *g);
/* Physical coordinates of the nq^dim points of `rule` in every element,
 * E x nq^dim x dim, so the host can evaluate a Coefficient
 * (ElementTransformation::point, mesh.cpp:142-157). */
int tfem_geometry_points(tfem_ctx *ctx, const tfem_geometry *g, int nq,
                         int rule, double *host_xyz);

/* ------------------------------------------------- partial assembly (D) */
/* pa_setup (forms.cpp:201-229, point_factors :46-68): geometric factors
 * times the coefficient at the nq^dim points of `rule` (reference: q = p+2
 * Gauss-Legendre; BP5: q = p+1 Gauss-Lobatto).  coeff == NULL -> constant
 * coeff_const, else per point E x nq^dim (reference point order).  Errors
 * as the reference: inverted element (runtime_error), non-positive
 * coefficient (invalid_argument); *bad_elem (nullable) gets the element. */
int tfem_pa_setup(tfem_ctx *ctx, int kind, const tfem_geometry *g, int p,
                  int nq, int rule, const double *coeff, double coeff_const,
                  tfem_pa **out, int64_t *bad_elem);
int tfem_pa_destroy(tfem_pa *pa);
int tfem_pa_info(const tfem_pa *pa, int *kind, int *dim, int *p, int *nq,
                 int64_t *n_elem);
/* PaData::stored_reals (forms.hpp:43-46) = E * nq^dim * ncomp. */
int64_t tfem_pa_stored_reals(const tfem_pa *pa);
/* Multiplies the instrumented reference kernels would count for one
 * application (tensor_kernels.hpp:20-26; test_forms.cpp:397-412). */
uint64_t tfem_pa_multiply_count(const tfem_pa *pa);
/* PaData::d in the reference layout [e][q][c] (forms.cpp:194-199). */
int tfem_pa_qdata(const tfem_pa *pa, double *host);
/* PaData::b1d / g1d (forms.hpp:36-37), nq x (p+1). */
int tfem_pa_basis(const tfem_pa *pa, double *B, double *G);
/* Replace the 1D tables with the caller's (nq x (p+1), row-major): PaData::
 * b1d / g1d of a basis other than the H1 Gauss-Lobatto one tfem_pa_setup
 * tabulates (an L2 space's Gauss-Legendre nodes, forms.cpp:213). */
int tfem_pa_set_basis(tfem_pa *pa, const double *B, const double *G);
/* pa_apply_local: y += G^T B^T D B G x on L-vectors (forms.cpp:231-296). */
int tfem_pa_apply_local(tfem_ctx *ctx, const tfem_pa *pa,
                        const tfem_restriction *r, const tfem_vec *x,
                        tfem_vec *y);
/* pa_diagonal: diag += exact diagonal (forms.cpp:311-382). */
int tfem_pa_diagonal(tfem_ctx *ctx, const tfem_pa *pa,
                     const tfem_restriction *r, tfem_vec *diag);

/* --------------------------------------------------------- prolongation */
/* FeSpace::prolongation() P (fespace.cpp:62-72, 166-203): N_L x N_T CSR with
 * unit rows for true DOFs and constraint weights for hanging DOFs on
 * non-conforming (forest) spaces; true_index[l] = FeSpace::true_index(l)
 * (-1 for a constrained DOF).  Host arrays are copied. */
int tfem_prolongation_create(tfem_ctx *ctx, int64_t n_local, int64_t n_true,
                             const int32_t *rowptr, const int32_t *cols,
                             const double *vals, const int32_t *true_index,
                             tfem_prolongation **out);
int tfem_prolongation_destroy(tfem_prolongation *P);
/* true_to_local: y_L = P x_T (SparseMatrix::mult, sparse.cpp:75-87). */
int tfem_prolongation_mult(tfem_ctx *ctx, const tfem_prolongation *P,
                           const tfem_vec *x_true, tfem_vec *y_local);
/* y_T = P^T x_L (SparseMatrix::mult_transpose, sparse.cpp:89-102: every
 * y_T[j] sums its rows in ascending order). */
int tfem_prolongation_mult_transpose(tfem_ctx *ctx, const tfem_prolongation *P,
                                     const tfem_vec *x_local, tfem_vec *y_true);
/* local_to_true: X[t] = x[true_dofs[t]] (fespace.cpp:252-262). */
int tfem_prolongation_local_to_true(tfem_ctx *ctx, const tfem_prolongation *P,
                                    const tfem_vec *x_local, tfem_vec *x_true);
/* pa_diagonal on a space with P (forms.cpp:311-382): unconstrained elements
 * add their exact local diagonal at true_index, constrained elements add the
 * P-weighted couplings of every local pair that lands on one true DOF, all
 * in the reference's element / pair order; diag_true += the result. */
int tfem_pa_diagonal_p(tfem_ctx *ctx, const tfem_pa *pa, const tfem_restriction *r,
                       const tfem_prolongation *P, tfem_vec *diag_true);

/* ----------------------------------------------------------- linear form */
/* LinearForm(space, f) (forms.cpp:400-431), 2D: b = G^T B^T (w detJ f) with
 * q = p + 2 Gauss-Legendre points; f_host[e][qy * nq + qx] holds f at the
 * physical points tfem_geometry_points(nq, TFEM_GAUSS_LEGENDRE) returns.
 * b is overwritten (L-vector of the restriction). */
int tfem_linear_form(tfem_ctx *ctx, const tfem_geometry *g, const tfem_restriction *r, int p,
                     const double *f_host, tfem_vec *b);

/* project_coefficient (fespace.cpp:334-356), 2D H1: the physical points of
 * every element's basis nodes, host_xy[e][b * (p+1) + a][2]; the caller
 * evaluates f there and tfem_project assigns out[dofs[i]] = f_nodes[e][i]
 * with the last element winning on shared DOFs (the reference's loop). */
int tfem_geometry_node_points(tfem_ctx *ctx, const tfem_geometry *g, int p, double *host_xy);
int tfem_project(tfem_ctx *ctx, const tfem_restriction *r, const double *f_nodes,
                 tfem_vec *out);
/* compute_l2_error (fespace.cpp:358-394), 2D H1, q = p + 3 Gauss-Legendre:
 * u_exact_host[e][qy * nq + qx] at tfem_geometry_points(p + 3, GL).  Per-point
 * terms on the device, the reference's sequential sum on the host. */
int tfem_l2_error(tfem_ctx *ctx, const tfem_geometry *g, const tfem_restriction *r, int p,
                  const tfem_vec *x, const double *u_exact_host, double *err);

/* ------------------------------------------------------------- operator */
/* BilinearForm::mult_true (forms.cpp:527-543) over n_pa integrators applied
 * in insertion order; with n_ess > 0 the ConstrainedOperator of
 * form_linear_system (forms.cpp:164-190): y = A(x with x[ess] = 0),
 * y[ess] = x[ess].  ess is sorted and unique. */
int tfem_operator_create(tfem_ctx *ctx, int n_pa, tfem_pa *const *pa,
                         const tfem_restriction *r, int64_t n_ess,
                         const int32_t *ess, tfem_operator **out);
/* The same on a space with prolongation P (non-conforming meshes):
 * y_T = P^T (sum_i A_i) P x_T (forms.cpp:534-542), essential DOFs and sizes
 * on the true level.  P = NULL is tfem_operator_create. */
int tfem_operator_create_p(tfem_ctx *ctx, int n_pa, tfem_pa *const *pa,
                           const tfem_restriction *r, const tfem_prolongation *P,
                           int64_t n_ess, const int32_t *ess,
                           tfem_operator **out);
/* SparseOperator over a CSR matrix (solvers.hpp:26-35). */
int tfem_operator_create_csr(tfem_ctx *ctx, int64_t n, const int32_t *rowptr,
                             const int32_t *cols, const double *vals,
                             tfem_operator **out);
int tfem_operator_destroy(tfem_operator *op);
int64_t tfem_operator_size(const tfem_operator *op);
int tfem_operator_mult(tfem_ctx *ctx, const tfem_operator *op,
                       const tfem_vec *x, tfem_vec *y);
/* Same, enqueued on the context stream without waiting (for timing loops). */
int tfem_operator_mult_async(tfem_ctx *ctx, const tfem_operator *op,
                             const tfem_vec *x, tfem_vec *y);
/* BilinearForm::diagonal_true (forms.cpp:545-557); with essential DOFs the
 * driver's diag[ess] = 1 (driver.cpp:151-159). */
int tfem_operator_diagonal(tfem_ctx *ctx, const tfem_operator *op,
                           tfem_vec *diag);

/* --------------------------------------------------- distributed operator */
/* Element-partitioned runs: each rank holds its elements plus
 * one ghost element layer, so every owned DOF gets all its contributions
 * locally, in global element order.  Per CG iteration the library packs
 * p[send_idx[k]] into send_buf[k], calls exchange(), unpacks recv_buf[k]
 * into p[recv_idx[k]]; reductions land in red[0..k) and allreduce(k) sums
 * them over ranks in place.  Hooks run on the host in stream order and must
 * only enqueue work on the context's stream (e.g. NCCL through
 * torch.distributed with that stream current); buffers are device memory
 * owned by the caller.  `not_owned` DOFs are left out of every dot. */
#define TFEM_MAX_PEERS 8
typedef struct {
   void (*exchange)(void *user);
   void (*allreduce)(int k, void *user);
   void *user;
} tfem_comm;

typedef struct {
   int n_peers;
   int64_t n_send[TFEM_MAX_PEERS], n_recv[TFEM_MAX_PEERS];
   const int32_t *send_idx[TFEM_MAX_PEERS], *recv_idx[TFEM_MAX_PEERS]; /* host */
   double *send_buf[TFEM_MAX_PEERS], *recv_buf[TFEM_MAX_PEERS];         /* device */
   double *red;                                                         /* device, >= 4 */
} tfem_halo;

int tfem_operator_set_comm(tfem_operator *op, const tfem_comm *comm, const tfem_halo *halo,
                           int64_t n_not_owned, const int32_t *not_owned);

/* The same plan with the communication inside the library over NCCL
 * (NVLink / NVSwitch): the halo update is one ncclSend / ncclRecv group per
 * iteration and the dots ncclAllReduce, all on the context's stream, so the
 * distributed CG iteration is captured into the same CUDA graphs as the
 * single-device one and no host code runs per iteration.  One communicator
 * per rank (one process -- or one context -- per GPU): rank 0 makes the id,
 * the caller ships it to the other ranks (any channel), every rank creates
 * its communicator.  peer[k] is the rank the k-th send / receive list pairs
 * with (a rank may list itself); send / receive buffers are allocated by the
 * library.  In CG the send planes of the new direction are packed first and
 * exchanged on a side stream while the direction update of the whole vector
 * runs (halo / compute overlap, graph-captured). */
#define TFEM_NCCL_ID_BYTES 128
int tfem_nccl_unique_id(unsigned char id[TFEM_NCCL_ID_BYTES]);
int tfem_nccl_create(tfem_ctx *ctx, int nranks, int rank,
                     const unsigned char id[TFEM_NCCL_ID_BYTES], tfem_nccl **out);
/* Operators keep their communicator alive: destroying the handle first is
 * safe (the last operator using it releases it). */
int tfem_nccl_destroy(tfem_nccl *comm);
/* Sum k doubles of device memory over the ranks, in place (synchronous). */
int tfem_nccl_allreduce(tfem_ctx *ctx, tfem_nccl *comm, double *device_buf, int64_t k);
int tfem_operator_set_nccl(tfem_operator *op, tfem_nccl *comm, int n_peers, const int *peer,
                           const int64_t *n_send, const int32_t *const *send_idx,
                           const int64_t *n_recv, const int32_t *const *recv_idx,
                           int64_t n_not_owned, const int32_t *not_owned);

/* ------------------------------------------------------------------- CG */
typedef struct {
   int iterations;      /* CgResult::iterations (solvers.hpp:37-41) */
   int converged;       /* CgResult::converged */
   double final_norm;   /* ||r|| of the recursive residual at exit */
   double initial_norm; /* ||b|| */
   double x_norm;       /* recursive ||r|| of the returned x (the best iterate
                           when not converged, solvers.cpp:89-96) */
} tfem_cg_result;

/* on_iterate(it, x_host, user) after every iteration (solvers.cpp:82);
 * forces a per-iteration device->host copy of x. */
typedef void (*tfem_cg_callback)(int it, const double *x, int64_t n,
                                 void *user);

/* cg_solve (solvers.cpp:11-97): Jacobi-PCG from x = 0; stop when
 * ||r|| <= rel_tol ||b|| (checked at the top of each iteration); on
 * exhaustion x is the best iterate and converged = 0; breakdown ->
 * TFEM_RUNTIME_ERROR with the reference message.  The whole loop runs on the
 * device; only a 4-byte status crosses per batch of iterations. */
int tfem_cg_solve(tfem_ctx *ctx, const tfem_operator *op, const tfem_vec *b,
                  double rel_tol, int max_iters, const tfem_vec *jacobi_diag,
                  tfem_vec *x, tfem_cg_result *res, tfem_cg_callback cb,
                  void *user);
/* Same with host buffers (copies in b / diag, copies out x): the call a
 * host-memory caller of cg_solve makes.  jacobi_diag may be NULL. */
int tfem_cg_solve_host(tfem_ctx *ctx, const tfem_operator *op,
                       const double *b, double rel_tol, int max_iters,
                       const double *jacobi_diag, double *x,
                       tfem_cg_result *res);

/* Diagnostics (no reference counterpart): `iters` iterations of the same
 * Jacobi-PCG (tolerance 0) run eagerly with CUDA events on the context's
 * stream between the launches; seg_us[0..2] = average time per iteration of
 * the operator (element kernel + scatter), the update and the direction
 * kernels, in microseconds -- the operator timed as it runs inside the
 * solve (p was just written, so partly L2-resident). */
int tfem_cg_profile(tfem_ctx *ctx, const tfem_operator *op, const tfem_vec *b,
                    int iters, const tfem_vec *jacobi_diag, tfem_vec *x,
                    double *seg_us);

/* Diagnostics (no reference counterpart): the measured CUDA-core FP64 (DFMA)
 * peak of the context's device in TFLOP/s -- the FP64 roofline bench.py
 * reports the element kernels against. */
int tfem_fp64_peak(tfem_ctx *ctx, double *tflops);
/* Diagnostics: the measured FP64 tensor-core (DMMA, mma.sync m8n8k4) peak in
 * TFLOP/s -- the ceiling a DMMA contraction would have (north_star: DMMA only
 * where it beats CUDA-core DFMA). */
int tfem_dmma_peak(tfem_ctx *ctx, double *tflops);
/* Diagnostics: DFMA vs DMMA A/B of the sum-factorisation contraction stage
 * (per element X[p+1][(p+1)^2] -> B X, G X with q = p+2 points) on shared-
 * memory-resident elements, order p in [2, 8]: res[0] DFMA and res[1] DMMA
 * useful TFLOP/s, res[2] max relative difference of the two results, res[3]
 * the DMMA tile padding factor (padded / useful multiply-adds). */
int tfem_contraction_ab(tfem_ctx *ctx, int p, double *res);

#ifdef __cplusplus
}
#endif

#endif
