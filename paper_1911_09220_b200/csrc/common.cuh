// Internal types and helpers of libtfem_cuda.so (not part of the C ABI).
#pragma once

#include "tfem_cuda.h"

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

namespace tfem {

// ----------------------------------------------------------------- errors
// Exceptions inside the library map 1:1 onto the reference's exception
// classes and are converted to status codes at the C boundary (capi.cu).
struct Error : std::runtime_error {
   int code;
   Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void invalid(const std::string &m) { throw Error(TFEM_INVALID_ARGUMENT, m); }
[[noreturn]] inline void runtime(const std::string &m) { throw Error(TFEM_RUNTIME_ERROR, m); }
[[noreturn]] inline void logic(const std::string &m) { throw Error(TFEM_LOGIC_ERROR, m); }

inline void cuda_check(cudaError_t e, const char *what)
{
   if (e != cudaSuccess) {
      throw Error(TFEM_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
   }
}
#define TFEM_CUDA(call) ::tfem::cuda_check((call), #call)

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) holds per device: the
// launch helpers call this before each launch; (kernel, device) pairs already
// set are remembered (capi.cu).
void max_dynamic_smem(const void *kernel, size_t bytes);

// Copies / fills ordered on a context's (non-blocking) stream.  Never use the
// legacy-stream cudaMemcpy / cudaMemset next to kernels on ctx->stream: the
// non-blocking stream does not wait for the legacy one.
inline void h2d(cudaStream_t s, void *dst, const void *src, size_t bytes)
{
   if (!bytes) return;
   TFEM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
   TFEM_CUDA(cudaStreamSynchronize(s));
}
inline void d2h(cudaStream_t s, void *dst, const void *src, size_t bytes)
{
   if (!bytes) return;
   TFEM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
   TFEM_CUDA(cudaStreamSynchronize(s));
}

// Flag bits (31:30) on an element-map entry:
//   10 kExclusive   the DOF has exactly one element slot: the element kernel
//                   owns it and writes it directly (no E-vector round trip)
//   00 shared       several slots; summed from the E-vector by the scatter
//   11 kWarpOwner / 01 kWarpMember
//                   several slots, all in one warp patch of an ordered space
//                   (ElemOrder): the 2D bulk-copy kernel sums them with warp
//                   shuffles into the owner slot (the highest element); every
//                   other kernel treats them as shared
constexpr uint32_t kFlagMask = 0xc0000000u;
constexpr uint32_t kExclusive = 0x80000000u;
constexpr uint32_t kWarpMember = 0x40000000u;
constexpr uint32_t kWarpOwner = 0xc0000000u;
constexpr uint32_t kDofMask = 0x3fffffffu;

// E-vector index of slot (element position e, local i) of an element-major
// map: [e][nd] like the map, with the slots of an element in the order
// tfem_restriction::evperm (interior, then each face's and edge's interior
// slots contiguous, so the scatter's reads of one face / edge share 32-byte
// sectors; null = natural order).  Slot-major maps use i * ne_pad + e.
// (A [i][ne_pad] E-vector for element-major maps was measured: +3 % at 3D
// p <= 2, -3 % at p = 3 and BP5 p = 4.)
__device__ __forceinline__ int64_t ev_em_p(const uint16_t *perm, int nd, int64_t e, int i)
{
   return e * nd + (perm ? static_cast<int>(__ldg(perm + i)) : i);
}

__host__ __device__ constexpr bool is_exclusive(uint32_t g) { return (g & kFlagMask) == kExclusive; }

// Device element order (positions of the element map / qdata / E-vector).
// pw == 0: position = element.  Otherwise (2D Cartesian, p <= 3) the mesh is
// cut into pw x ph = 8 x 4 patches, one per warp (32 positions, row-major
// inside: lane = 8 r + c), patches row-major: DOFs shared only inside a patch
// are summed by warp shuffles, and a warp's x gathers stay coalesced along
// its rows.  Partial patches at the mesh edge leave padding positions: zero
// qdata, map entries DOF 0 without flags (their E-vector slots are written
// but never read).
struct ElemOrder {
   int pw = 0, ph = 0;
   int64_t nx = 0, ny = 0, px = 0, py = 0; // cells, patches per axis
   __host__ __device__ int64_t n_pos(int64_t ne) const { return pw ? px * py * pw * ph : ne; }
   __host__ __device__ int64_t pos_of(int64_t e) const
   {
      if (!pw) return e;
      const int64_t i = e % nx, j = e / nx;
      return ((j / ph) * px + i / pw) * (pw * ph) + (j % ph) * pw + i % pw;
   }
   // reference element at a position, -1 for padding
   __host__ __device__ int64_t elem_at(int64_t pos) const
   {
      if (!pw) return pos;
      const int64_t t = pos / (pw * ph), r = pos % (pw * ph);
      const int64_t i = (t % px) * pw + r % pw, j = (t / px) * ph + r / pw;
      return i < nx && j < ny ? j * nx + i : -1;
   }
   bool operator==(const ElemOrder &o) const
   {
      return pw == o.pw && ph == o.ph && (pw == 0 || (nx == o.nx && ny == o.ny));
   }
};

// The order a (dim, p) space on a Cartesian mesh of n cells uses; the
// restriction and every PaData of the space derive it independently.
inline ElemOrder elem_order_for(int dim, int p, bool cartesian, const int *n)
{
   ElemOrder o;
   if (dim == 2 && p <= 3 && cartesian) {
      o.pw = 8;
      o.ph = 4;
      o.nx = n[0];
      o.ny = n[1];
      o.px = (o.nx + o.pw - 1) / o.pw;
      o.py = (o.ny + o.ph - 1) / o.ph;
   }
   return o;
}

// Orders: 2D up to p = 16 (the reference's target range), with
// up to q = p + 3 points (compute_l2_error's rule); 3D up to p = 8.
constexpr int kMaxP = 16;
constexpr int kMaxQ = 19;
constexpr int kMaxP3D = 8;

inline int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

// Device data layout of an (dim, p) space.  Low-order 2D runs one element per
// thread: slot-major element map [nd][ne_pad] and point-major qdata planes
// [(c*nqd+q)][ne_pad] (element fastest, coalesced).  3D and 2D p >= 4 run one
// element per thread group: element-major map [e][nd] and qdata [e][c][q].
inline bool elem_major_layout(int dim, int p) { return dim == 3 || p >= 4; }

// qdata layouts: 0 planes [(c*nqd + q)][ne_pad] (element fastest); 1
// element-major [e][c][q].  (A slab-major [e][qz][c][q2] layout streamed one
// qz plane at a time was measured for 3D q = 6, 7: slower at BP3 p = 4, 5
// -- the column stage's second lane pass re-waits on every slab -- and
// removed.)
inline int qdata_layout(int dim, int p, int nq, int kind)
{
   (void)nq;
   (void)kind;
   return elem_major_layout(dim, p) ? 1 : 0;
}
__host__ __device__ inline int64_t qdata_index(int layout, int64_t pos, int c, int q, int ncomp,
                                               int nqd, int nq, int64_t ne_pad)
{
   (void)nq;
   if (layout == 0) return (int64_t)(c * nqd + q) * ne_pad + pos;
   return (pos * ncomp + c) * (int64_t)nqd + q;
}

// Scratch for block partials of fused dot products and the last-block
// ticket.  One per context; every reduction uses a fixed grid so the result
// is deterministic run to run.
struct Reducer {
   double *partials = nullptr; // [cap]
   int64_t cap = 0;
   unsigned int *ticket = nullptr;
};

} // namespace tfem

struct tfem_ctx {
   // Reference count: the context handle plus every object created through
   // it (vectors, restrictions, geometries, PaData, operators, prolongations);
   // tfem_ctx_destroy drops the handle's count, the last object frees it.
   int refs = 1;
   int device = 0;
   cudaStream_t stream = nullptr;
   int numerics = TFEM_NUMERICS_FMA;
   int sm_count = 148;
   int max_blocks = 0; // test hook: cap on persistent grids (0 = none)
   int64_t launches = 0;
   tfem::Reducer red;
   double *scalars = nullptr;      // device scratch for small results
   double *host_scalars = nullptr; // pinned mirror
   // Device-side state cached per context (never per thread or process, so
   // contexts on different devices never share memory): the dot sinks of
   // vec_dot by grid size, the staging buffers of tfem_cg_solve_host.
   struct DotStore {
      double *partials = nullptr, *chunks = nullptr;
      unsigned *tickets = nullptr;
   };
   std::vector<std::pair<int64_t, DotStore>> dot_sinks;
   double *stage[3] = {nullptr, nullptr, nullptr};
   int64_t stage_n[3] = {0, 0, 0};
   // Caching device allocator (tfem_mem_alloc / tfem_mem_free): freed blocks
   // return to a size-keyed free list and are reused in stream order (the
   // context has one stream), so host-side objects that come and go -- the
   // device mirrors of the reference's Vector -- never cudaMalloc per call.
   std::mutex pool_mu;
   std::multimap<size_t, void *> pool_free;
   std::unordered_map<void *, size_t> pool_live;
   void ensure_partials(int64_t n);
   void launched(int64_t n = 1) { launches += n; }
};

struct tfem_nccl {
   tfem_ctx *ctx = nullptr;
   void *comm = nullptr; // ncclComm_t
   int rank = 0, nranks = 1;
   // the handle plus every operator using the communicator: destroying the
   // handle before its operators leaves the communicator to the last one
   int refs = 1;
};

struct tfem_vec {
   tfem_ctx *ctx = nullptr;
   double *d = nullptr;
   int64_t n = 0;
   bool owns = true;
};

struct tfem_restriction {
   tfem_ctx *ctx = nullptr;
   int dim = 2, p = 1, nd = 4; // nd = (p+1)^dim
   int64_t ne = 0, npos = 0, ne_pad = 0, ndofs = 0; // npos: positions (order.n_pos)
   // Element map with the kExclusive flag, layout elem_major_layout(dim, p):
   // slot-major [nd][ne_pad] or element-major [ne_pad][nd]; a `slot` indexes
   // both gmap and the E-vector.
   bool elem_major = false;
   uint32_t *gmap = nullptr;
   // DOFs with >= 2 element slots, bucketed by slot count c (ELL per
   // bucket): dofs[n] ascending, slots[n][c] sorted by element.
   struct Bucket {
      int c = 0;
      int64_t n = 0;
      int32_t *dofs = nullptr;
      uint32_t *slots = nullptr; // E-vector slots (= gmap slots unless evperm)
   };
   static constexpr int kMaxBuckets = 7; // c = 2..8
   int n_buckets = 0;
   Bucket buckets[kMaxBuckets];
   int64_t n_shared = 0;
   tfem::ElemOrder order;
   // Ordered spaces: the warp-local DOFs are flagged in gmap and the other
   // shared DOFs form the global buckets (the bulk-copy kernel's scatter).
   bool warp_local = false;
   int n_gbuckets = 0;
   Bucket gbuckets[kMaxBuckets];
   int64_t n_gshared = 0;
   // E-vector scratch (lazy) in the map's layout: slot-major [i][ne_pad],
   // element-major [e][nd] with the element's slots in evperm order (ev_em_p)
   double *evec = nullptr;
   uint16_t *evperm = nullptr; // element-major maps: E-vector slot order (ev_em_p)
   bool cartesian = false;
   int n[3] = {0, 0, 0};
   double *ensure_evec();
   // element kernels write E-vector slots (shared DOFs; padding positions)
   bool needs_evec() const { return n_shared > 0 || npos > ne; }
};

struct tfem_geometry {
   tfem_ctx *ctx = nullptr;
   int dim = 2, order = 1;
   int64_t ne = 0;
   double *ctrl = nullptr; // [e][l][dim] (null for Cartesian)
   bool cartesian = false;
   int n[3] = {0, 0, 0};        // local cells per axis
   int origin[3] = {0, 0, 0};   // cell offset inside the global mesh
   int n_global[3] = {0, 0, 0}; // global cells per axis
   double ext[3] = {1.0, 1.0, 1.0};
};

struct tfem_pa {
   tfem_ctx *ctx = nullptr;
   int kind = TFEM_DIFFUSION, dim = 2, p = 1, nq = 3, rule = TFEM_GAUSS_LEGENDRE;
   int ncomp = 3, nqd = 9;
   int64_t ne = 0, npos = 0, ne_pad = 0; // npos: element positions (order.n_pos)
   // elem_major_layout(dim, p) ? [e][c][q] : planes [(c * nqd + q)][ne_pad]
   double *qdata = nullptr;
   int qlayout = 0;       // tfem::qdata_layout(dim, p, nq, kind)
   tfem::ElemOrder order; // element positions of qdata (== the restriction's)
   bool elem_major() const { return tfem::elem_major_layout(dim, p); }
   std::vector<double> B, G; // nq x (p+1)
   // B == I exactly (q = p+1 Gauss-Lobatto points on the basis nodes, BP5):
   // the kernels skip the B contractions (collocated variants)
   bool colloc = false;
};

struct tfem_prolongation {
   tfem_ctx *ctx = nullptr;
   int64_t n_local = 0, n_true = 0, nnz = 0;
   int32_t *rowptr = nullptr, *cols = nullptr; // P, N_L rows
   double *vals = nullptr;
   int32_t *trowptr = nullptr, *trows = nullptr; // P^T, N_T rows, ascending P rows
   double *tvals = nullptr;
   int32_t *true_index = nullptr; // [N_L], -1: constrained
   int32_t *true_dofs = nullptr;  // [N_T]
};

struct tfem_operator {
   tfem_ctx *ctx = nullptr;
   bool csr = false;
   int64_t n = 0;
   std::vector<tfem_pa *> pa;
   const tfem_restriction *r = nullptr;
   const tfem_prolongation *P = nullptr; // non-conforming: y = P^T A_L P x
   double *xl = nullptr, *yl = nullptr;  // L-vector scratch (with P)
   int64_t n_ess = 0;
   int32_t *ess = nullptr;      // sorted list
   uint32_t *ess_mask = nullptr; // bitmap over DOFs
   // per element position: the slots whose DOF is in ess_mask (slot-major
   // maps with nd <= 32; read by the 2D bulk-copy kernel instead of one
   // bitmap load per slot)
   uint32_t *elem_ess = nullptr;
   uint32_t *notown = nullptr;   // bitmap: DOFs owned by another rank (dist)
   bool has_comm = false;        // distributed: NCCL (nccl) or the host hooks (comm)
   tfem_comm comm{};
   tfem_nccl *nccl = nullptr;    // library-side NCCL: buffers below owned here
   int peer_rank[TFEM_MAX_PEERS] = {};
   int n_peers = 0;
   int64_t n_send[TFEM_MAX_PEERS] = {}, n_recv[TFEM_MAX_PEERS] = {};
   int32_t *send_idx[TFEM_MAX_PEERS] = {}, *recv_idx[TFEM_MAX_PEERS] = {}; // device
   double *send_buf[TFEM_MAX_PEERS] = {}, *recv_buf[TFEM_MAX_PEERS] = {}; // caller's
   double *red = nullptr;                                                // caller's
   // NCCL halo overlap: the exchange runs on `side` while the direction
   // kernel runs on the context stream (fork / join events; graph-capturable)
   cudaStream_t side = nullptr;
   cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
   int32_t *rowptr = nullptr, *cols = nullptr;
   double *vals = nullptr;
};

namespace tfem {

void ctx_retain(tfem_ctx *ctx);
void ctx_release(tfem_ctx *ctx);

// NCCL (comm.cu)
void nccl_unique_id(unsigned char *id);
tfem_nccl *nccl_create(tfem_ctx *ctx, int nranks, int rank, const unsigned char *id);
void nccl_destroy(tfem_nccl *c); // drops one reference (handle or operator)
void nccl_retain(tfem_nccl *c);
void nccl_allreduce(tfem_ctx *ctx, const tfem_nccl *c, double *d, int64_t k);
void nccl_exchange(tfem_ctx *ctx, const tfem_operator *op, cudaStream_t s);

constexpr int kChunk = 32;

// Device-resident CG scalars (solvers.cpp:43-96), advanced by the last block
// of the kernels whose dot products they need (see emit).
struct CgState {
   double rz, alpha, beta, rnorm, best_rnorm, target;
   int it, max_iters, done, converged, iterations, status;
   int cur, best;
   // x' = x + alpha p is taken by the direction kernel (which reads p
   // anyway): x buffer `prev` -> `cur`, pending while xpend != 0
   int prev, xpend;
};

enum SinkFinish : int { kFinishNone = 0, kFinishAlpha = 1, kFinishBeta = 2 };

struct DotSink {
   double *partials = nullptr;   // [nv][grid]
   double *chunks = nullptr;     // [nv][n_chunks]
   unsigned *tickets = nullptr;  // [n_chunks + 1], zero between launches
   // Optional finish: the last chunk to complete folds `pre` (chunk sums of
   // an earlier kernel, e.g. the element kernel's share of p.q) and this
   // launch's chunks in a fixed order and advances the CG state.
   const double *pre = nullptr;  // [nv][n_pre]
   int64_t n_pre = 0;
   CgState *state = nullptr;
   int finish = kFinishNone;
   __host__ __device__ explicit operator bool() const { return partials != nullptr; }
};

__host__ __device__ inline int64_t n_chunks(int64_t grid) { return (grid + kChunk - 1) / kChunk; }

// Host-side 1D tables (host_basis.cpp).
std::vector<double> gauss_points(int rule, int n, std::vector<double> *weights);
void basis_nodes(int p, int node_kind, std::vector<double> &nodes, std::vector<double> &bary);
void basis_eval(const std::vector<double> &nodes, const std::vector<double> &bary, double x,
                double *values, double *derivs);
void eval_matrices(int p, int node_kind, int nq, int rule, double *B, double *G);

// Launch helpers implemented per translation unit.
void vec_fill(tfem_ctx *ctx, double *d, int64_t n, double v);
// Optional: skip DOFs in `notown`, then sum over ranks with the comm hook.
double vec_dot(tfem_ctx *ctx, const double *a, const double *b, int64_t n,
               const tfem_operator *dist = nullptr);

// Restriction / layout (restriction.cu)
tfem_restriction *restriction_from_map(tfem_ctx *ctx, int dim, int p, int64_t ne, int64_t ndofs,
                                       bool elem_major, uint32_t *d_gmap_raw /* owned */,
                                       ElemOrder order);
void restriction_mult_transpose(tfem_ctx *ctx, const tfem_restriction *r, const double *e,
                                double *l);

// Shared-DOF scatter over the buckets (apply.cu): y[d] (+)= sum of the
// E-vector slots of d in ascending element order; y[ess] = x[ess]; fused
// x . y partials.  `global_only`: just the DOFs that are not tile-local (the
// tile kernel summed the others).  Returns the grid size (for the dot sink).
int64_t scatter_shared(tfem_ctx *ctx, const tfem_restriction *r, const double *evec,
                       const double *x, double *y, bool overwrite, const uint32_t *ess_out,
                       const DotSink *dot, const int *done, bool exact,
                       const uint32_t *notown = nullptr, bool global_only = false,
                       bool ess_only = false);
int64_t scatter_grid(const tfem_restriction *r, bool global_only = false);

// PA kernels (apply.cu)
struct ApplyFlags {
   bool overwrite = false;   // y = (else y +=)
   const uint32_t *mask_in = nullptr;  // zero gathered essential DOFs
   const uint32_t *ess_out = nullptr;  // y[ess] = x[ess]
   const uint32_t *elem_ess = nullptr; // mask_in per position (tfem_operator::elem_ess)
   const uint32_t *notown = nullptr;   // excluded from the dot (other rank's DOFs)
   DotSink dot;                        // element-kernel x . y partials
   DotSink dot_scatter;                // scatter-kernel x . y partials
   const int *done = nullptr;          // device flag: skip when set (CG)
};
// Launches the element kernel and (if needed) the shared-DOF scatter.
void pa_apply(tfem_ctx *ctx, const tfem_pa *pa, const tfem_restriction *r, const double *x,
              double *y, const ApplyFlags &f);
// Grid sizes of the two launches of pa_apply (element kernel, scatter).
void pa_apply_grids(const tfem_pa *pa, const tfem_restriction *r, int64_t *g_elem,
                    int64_t *g_scatter);
void pa_diagonal(tfem_ctx *ctx, const tfem_pa *pa, const tfem_restriction *r, double *diag);

// Setup (setup.cu)
tfem_pa *pa_setup(tfem_ctx *ctx, int kind, const tfem_geometry *g, int p, int nq, int rule,
                  const double *coeff_host, double coeff_const, int64_t *bad_elem);
void geometry_points(tfem_ctx *ctx, const tfem_geometry *g, int nq, int rule, double *host_xyz);
void linear_form(tfem_ctx *ctx, const tfem_geometry *g, const tfem_restriction *r, int p,
                 const double *f_host, double *b);
void geometry_node_points(tfem_ctx *ctx, const tfem_geometry *g, int p, double *host_xy);
double l2_error(tfem_ctx *ctx, const tfem_geometry *g, const tfem_restriction *r, int p,
                const double *x, const double *u_exact_host);
void restriction_assign_last(tfem_ctx *ctx, const tfem_restriction *r, const double *e, double *l);

// Prolongation (prolong.cu)
void prolongation_mult(tfem_ctx *ctx, const tfem_prolongation *P, const double *x_true,
                       const uint32_t *mask_true, double *y_local, const int *done);
void prolongation_mult_transpose(tfem_ctx *ctx, const tfem_prolongation *P, const double *x_local,
                                 double *y_true, const double *x_true_ess,
                                 const uint32_t *ess_true, const DotSink *dot, const int *done);
void prolongation_local_to_true(tfem_ctx *ctx, const tfem_prolongation *P, const double *x_local,
                                double *x_true);
void pa_diagonal_p(tfem_ctx *ctx, const tfem_pa *pa, const tfem_restriction *r,
                   const tfem_prolongation *P, double *diag_true);
int64_t prolongation_grid(const tfem_prolongation *P);

// Operators / CG (cg.cu)
// With dot sinks set, the last integrator's launches emit x . y partials.
void operator_mult(tfem_ctx *ctx, const tfem_operator *op, const double *x, double *y,
                   const DotSink *dot_elem, const DotSink *dot_scatter, const int *done);
// Measured CUDA-core FP64 (DFMA) peak in TFLOP/s (probe.cu; diagnostics).
double fp64_peak_tflops(tfem_ctx *ctx);
// Measured FP64 tensor-core (DMMA m8n8k4) peak in TFLOP/s (probe.cu).
double dmma_peak_tflops(tfem_ctx *ctx);
// res[4]: DFMA / DMMA useful TFLOP/s of the x-stage contraction at order p,
// max relative difference of their results, DMMA padding factor
void contraction_ab(tfem_ctx *ctx, int p, double *res);

void cg_solve(tfem_ctx *ctx, const tfem_operator *op, const double *b, double rel_tol,
              int max_iters, const double *diag, double *x, tfem_cg_result *res,
              tfem_cg_callback cb, void *user, double *seg_us = nullptr);

} // namespace tfem

// ------------------------------------------------------------ device side
#ifdef __CUDACC__
namespace tfem {

__device__ __forceinline__ bool bit_set(const uint32_t *mask, uint32_t d)
{
   return (__ldg(mask + (d >> 5)) >> (d & 31)) & 1u;
}

// Block-wide sum with a fixed shape: warp shuffles, then warp 0.  Valid in
// thread 0 only.  Deterministic for a fixed blockDim.
template <int NT>
__device__ __forceinline__ double block_sum(double v)
{
   static_assert(NT % 32 == 0 && NT <= 1024, "block size");
   __shared__ double warp_part[NT / 32];
#pragma unroll
   for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
   if ((threadIdx.x & 31) == 0) warp_part[threadIdx.x >> 5] = v;
   __syncthreads();
   double s = 0.0;
   if (threadIdx.x < 32) {
      s = threadIdx.x < NT / 32 ? warp_part[threadIdx.x] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
   }
   __syncthreads(); // warp_part may be reused by the next call
   return s;
}

__device__ __forceinline__ int next_buffer(int cur, int best)
{
   for (int k = 0; k < 3; k++)
      if (k != cur && k != best) return k;
   return 0;
}

__device__ inline void alpha_step(CgState *st, double pq)
{
   const double alpha = st->rz / pq;
   st->alpha = alpha;
   if (!isfinite(alpha)) { // solvers.cpp:69-71
      st->status = 1;
      st->done = 1;
   }
}

__device__ inline void beta_step(CgState *st, double rr, double rz_next)
{
   const double rnorm = sqrt(rr);
   st->rnorm = rnorm;
   if (!isfinite(rnorm)) { // solvers.cpp:74-77
      st->status = 2;
      st->done = 1;
      return;
   }
   st->it += 1;
   const int nxt = next_buffer(st->cur, st->best);
   st->prev = st->cur;
   st->cur = nxt;
   st->xpend = 1;
   if (rnorm < st->best_rnorm) { // solvers.cpp:78-81
      st->best_rnorm = rnorm;
      st->best = nxt;
   }
   st->beta = rz_next / st->rz;
   st->rz = rz_next;
   if (rnorm <= st->target) { // checked at the top of the next iteration
      st->done = 1;
      st->converged = 1;
      st->iterations = st->it;
   } else if (st->it >= st->max_iters) {
      st->done = 1;
      st->converged = 0;
      st->iterations = st->max_iters;
   }
}

// Deterministic two-level reduction of per-block values.  Every block writes
// its block sums to partials[k][blockIdx]; the last block to finish in each
// chunk of kChunk consecutive blocks (atomic ticket) folds the chunk's
// partials in block order into chunks[k][chunk] and re-arms the ticket.  The
// consumer then folds the few hundred chunk sums in a fixed order.  No
// floating-point atomics anywhere, so results are bit-reproducible.
template <int NT, int NV>
__device__ __forceinline__ void emit(const DotSink &s, const double (&v)[NV])
{
   double tot[NV];
#pragma unroll
   for (int k = 0; k < NV; k++) tot[k] = block_sum<NT>(v[k]);
   __shared__ int is_last;
   const unsigned G = gridDim.x, chunk = blockIdx.x / kChunk;
   if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < NV; k++) s.partials[k * (int64_t)G + blockIdx.x] = tot[k];
      __threadfence();
      const unsigned nb = min((unsigned)kChunk, G - chunk * kChunk);
      is_last = atomicAdd(s.tickets + chunk, 1u) == nb - 1;
   }
   __syncthreads();
   if (!is_last) return; // block-uniform
   __shared__ int is_final;
   const int64_t nch = n_chunks(G);
   if (threadIdx.x == 0) {
      __threadfence();
      const unsigned nb = min((unsigned)kChunk, G - chunk * kChunk);
#pragma unroll
      for (int k = 0; k < NV; k++) {
         double a = 0.0;
         for (unsigned j = 0; j < nb; j++) a += __ldcg(s.partials + k * (int64_t)G + chunk * kChunk + j);
         s.chunks[k * nch + chunk] = a;
      }
      s.tickets[chunk] = 0u;
      is_final = 0;
      if (s.finish != kFinishNone) {
         __threadfence();
         is_final = atomicAdd(s.tickets + nch, 1u) == nch - 1;
      }
   }
   __syncthreads();
   if (!is_final) return;
   __threadfence();
   double f[NV];
#pragma unroll
   for (int k = 0; k < NV; k++) {
      double a = 0.0;
      for (int64_t i = threadIdx.x; i < s.n_pre + nch; i += NT)
         a += __ldcg(i < s.n_pre ? s.pre + k * s.n_pre + i : s.chunks + k * nch + (i - s.n_pre));
      f[k] = block_sum<NT>(a);
   }
   if (threadIdx.x == 0) {
      s.tickets[nch] = 0u;
      if (s.finish == kFinishAlpha) alpha_step(s.state, f[0]);
      else beta_step(s.state, f[0], f[NV - 1]);
   }
}

// Exact (reference-order, unfused) or fused arithmetic.
template <bool EXACT>
__device__ __forceinline__ double mul(double a, double b)
{
   return EXACT ? __dmul_rn(a, b) : a * b;
}
template <bool EXACT>
__device__ __forceinline__ double add(double a, double b)
{
   return EXACT ? __dadd_rn(a, b) : a + b;
}
template <bool EXACT>
__device__ __forceinline__ double mac(double acc, double a, double b)
{
   return EXACT ? __dadd_rn(acc, __dmul_rn(a, b)) : fma(a, b, acc);
}

} // namespace tfem
#endif
