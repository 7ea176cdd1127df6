// Element restriction G / G^T on the device.
//
// Device layout: the element map is stored slot-major,
// gmap[i * ne_pad + e] (thread-per-element gathers are coalesced), with bit 31
// set when DOF has a single element slot ("exclusive": written straight from
// the element kernel).  DOFs with >= 2 slots get a transpose CSR whose slot
// lists are sorted by element -- the reference's ascending-element
// accumulation (forms.cpp:289-295) without atomics.
#include "common.cuh"

#include <cub/cub.cuh>

namespace tfem {

namespace {

constexpr int kThreads = 256;

inline unsigned blocks_for(int64_t n, int t = kThreads)
{
   return static_cast<unsigned>((n + t - 1) / t);
}

// Map layout: slot of (local i, element e), and the element of a slot.
struct Layout {
   bool elem_major;
   int nd;
   int64_t ne, ne_pad;
   __host__ __device__ int64_t slot(int i, int64_t e) const
   {
      return elem_major ? e * nd + i : (int64_t)i * ne_pad + e;
   }
   __host__ __device__ int64_t elem_of(int64_t s) const { return elem_major ? s / nd : s % ne_pad; }
   __host__ __device__ int local_of(int64_t s) const
   {
      return static_cast<int>(elem_major ? s % nd : s / ne_pad);
   }
   // t in [0, ne*nd) enumerates every live slot
   __host__ __device__ int64_t live(int64_t t) const
   {
      return elem_major ? t : (t / ne) * ne_pad + t % ne;
   }
};

// ---------------------------------------------------------------- layouts
// 2D: build_h1_layout on make_cartesian (mesh.cpp:65-115, 283-321).  Edge ids
// follow MeshTopology's discovery order (mesh.cpp:26-57): row 0 discovers
// bottom/right/top(/left at i = 0) per element, rows j >= 1 right/top(/left).
__device__ int64_t edge_base_row(int nx, int j)
{
   return (3 * (int64_t)nx + 1) + (int64_t)(j - 1) * (2 * nx + 1);
}
__device__ int64_t edge_right(int nx, int i, int j)
{
   if (j == 0) return i == 0 ? 1 : 3 * (int64_t)i + 2;
   return i == 0 ? edge_base_row(nx, j) : edge_base_row(nx, j) + 2 * (int64_t)i + 1;
}
__device__ int64_t edge_top(int nx, int i, int j)
{
   if (j == 0) return i == 0 ? 2 : 3 * (int64_t)i + 3;
   return i == 0 ? edge_base_row(nx, j) + 1 : edge_base_row(nx, j) + 2 * (int64_t)i + 2;
}
__device__ int64_t edge_bottom(int nx, int i, int j)
{
   if (j == 0) return i == 0 ? 0 : 3 * (int64_t)i + 1;
   return edge_top(nx, i, j - 1);
}
__device__ int64_t edge_left(int nx, int i, int j)
{
   if (i > 0) return edge_right(nx, i - 1, j);
   return j == 0 ? 3 : edge_base_row(nx, j) + 2;
}

__global__ void layout2d_kernel(int nx, int ny, int p, Layout L, uint32_t *gmap)
{
   const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (e >= (int64_t)nx * ny) return;
   const int i = static_cast<int>(e % nx), j = static_cast<int>(e / nx);
   const int D1 = p + 1, pe = p - 1;
   const int64_t nv = (int64_t)(nx + 1) * (ny + 1);
   const int64_t n_edges = (int64_t)nx * (ny + 1) + (int64_t)ny * (nx + 1);
   const int64_t ib = nv + n_edges * pe;
   const int64_t v0 = i + (int64_t)(nx + 1) * j;
   auto put = [&](int a, int b, int64_t dof) {
      gmap[L.slot(a + b * D1, e)] = static_cast<uint32_t>(dof);
   };
   put(0, 0, v0);
   put(p, 0, v0 + 1);
   put(p, p, v0 + nx + 2);
   put(0, p, v0 + nx + 1);
   const int64_t eb = nv + edge_bottom(nx, i, j) * pe, er = nv + edge_right(nx, i, j) * pe;
   const int64_t et = nv + edge_top(nx, i, j) * pe, el = nv + edge_left(nx, i, j) * pe;
   for (int m = 1; m < p; m++) {
      put(m, 0, eb + m - 1);
      put(p, m, er + m - 1);
      put(m, p, et + m - 1);
      put(0, m, el + m - 1);
   }
   for (int b = 1; b < p; b++)
      for (int a = 1; a < p; a++) put(a, b, ib + e * pe * pe + (a - 1) + (b - 1) * pe);
}

// 3D canonical numbering: vertices, x/y/z edges, x/y/z-normal
// faces, interiors; every entity oriented along increasing coordinates.
__global__ void layout3d_kernel(int nx, int ny, int nz, int p, uint32_t *gmap)
{
   const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (e >= (int64_t)nx * ny * nz) return;
   const int i = static_cast<int>(e % nx);
   const int j = static_cast<int>((e / nx) % ny);
   const int k = static_cast<int>(e / ((int64_t)nx * ny));
   const int D1 = p + 1;
   const int64_t pe = p - 1, pf = pe * pe, pin = pf * pe;
   const int64_t nvx = nx + 1, nvy = ny + 1, nvz = nz + 1;
   const int64_t NV = nvx * nvy * nvz;
   const int64_t EX = nx * nvy * nvz, EY = nvx * ny * nvz, EZ = nvx * nvy * nz;
   const int64_t FX = nvx * ny * nz, FY = nx * nvy * nz, FZ = (int64_t)nx * ny * nvz;
   const int64_t exb = NV, eyb = exb + EX * pe, ezb = eyb + EY * pe;
   const int64_t fxb = ezb + EZ * pe, fyb = fxb + FX * pf, fzb = fyb + FY * pf;
   const int64_t ib = fzb + FZ * pf;
   for (int c = 0; c <= p; c++)
      for (int b = 0; b <= p; b++)
         for (int a = 0; a <= p; a++) {
            const bool ea = (a == 0 || a == p), eb = (b == 0 || b == p), ec = (c == 0 || c == p);
            const int64_t ia = i + (a == p), jb = j + (b == p), kc = k + (c == p);
            int64_t dof;
            if (ea && eb && ec) dof = ia + nvx * (jb + nvy * kc);
            else if (!ea && eb && ec) dof = exb + (i + nx * (jb + nvy * kc)) * pe + (a - 1);
            else if (ea && !eb && ec) dof = eyb + (ia + nvx * (j + ny * kc)) * pe + (b - 1);
            else if (ea && eb && !ec) dof = ezb + (ia + nvx * (jb + nvy * k)) * pe + (c - 1);
            else if (ea) dof = fxb + (ia + nvx * (j + (int64_t)ny * k)) * pf + (b - 1) + pe * (c - 1);
            else if (eb) dof = fyb + (i + nx * (jb + nvy * k)) * pf + (a - 1) + pe * (c - 1);
            else if (ec) dof = fzb + (i + nx * (j + (int64_t)ny * kc)) * pf + (a - 1) + pe * (b - 1);
            else dof = ib + e * pin + (a - 1) + pe * ((b - 1) + pe * (c - 1));
            gmap[e * (D1 * D1 * D1) + a + D1 * (b + D1 * c)] = static_cast<uint32_t>(dof);
         }
}

__global__ void transpose_in_kernel(const int32_t *emap, Layout L, int64_t ndofs,
                                    uint32_t *gmap, int *bad)
{
   const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (t >= L.ne * L.nd) return;
   const int32_t d = emap[t];
   if (d < 0 || d >= ndofs) atomicExch(bad, 1);
   gmap[L.slot(static_cast<int>(t % L.nd), t / L.nd)] = static_cast<uint32_t>(d);
}

__global__ void count_kernel(const uint32_t *gmap, Layout L, int32_t *counts)
{
   const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (t >= L.ne * L.nd) return;
   atomicAdd(counts + (gmap[L.live(t)] & kDofMask), 1);
}

__global__ void flag_kernel(const int32_t *counts, int64_t ndofs, int32_t *is_shared,
                            int32_t *shared_count)
{
   const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (d >= ndofs) return;
   const int c = counts[d];
   is_shared[d] = c >= 2 ? 1 : 0;
   shared_count[d] = c >= 2 ? c : 0;
}

__global__ void mark_exclusive_kernel(uint32_t *gmap, Layout L, const int32_t *counts)
{
   const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (t >= L.ne * L.nd) return;
   const int64_t s = L.live(t);
   const uint32_t g = gmap[s];
   if (counts[g & kDofMask] == 1) gmap[s] = g | kExclusive;
}

// rank[d] = position of shared DOF d in the compact list (from the scan of
// is_shared), slot_base[d] = offset of its slot list.
__global__ void fill_slots_kernel(const uint32_t *gmap, Layout L, const int32_t *rank,
                                  const int32_t *is_shared, const int32_t *off, int32_t *fill,
                                  uint32_t *slots)
{
   const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (t >= L.ne * L.nd) return;
   const int64_t s = L.live(t);
   const uint32_t d = gmap[s] & kDofMask;
   if (!is_shared[d]) return;
   const int r = rank[d];
   const int pos = off[r] + atomicAdd(fill + r, 1);
   slots[pos] = static_cast<uint32_t>(s);
}

__global__ void compact_shared_kernel(const int32_t *is_shared, const int32_t *rank,
                                      int64_t ndofs, int32_t *shared_dofs)
{
   const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (d >= ndofs || !is_shared[d]) return;
   shared_dofs[rank[d]] = static_cast<int32_t>(d);
}

__global__ void gather_off_kernel(const int32_t *sd, const int32_t *full, int64_t ns,
                                  int32_t *out)
{
   const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (s < ns) out[s] = full[sd[s]];
}

// Slot lists are tiny (<= 2^dim); insertion-sort each by element so the
// scatter adds contributions in ascending element order.
__global__ void sort_slots_kernel(const int32_t *off, int64_t n_shared, Layout L,
                                  uint32_t *slots)
{
   const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (s >= n_shared) return;
   const int beg = off[s], end = off[s + 1];
   for (int a = beg + 1; a < end; a++) {
      const uint32_t v = slots[a];
      const int64_t key = L.elem_of(v);
      int b = a - 1;
      while (b >= beg && L.elem_of(slots[b]) > key) {
         slots[b + 1] = slots[b];
         b--;
      }
      slots[b + 1] = v;
   }
}

__global__ void gather_kernel(const uint32_t *gmap, Layout L, const double *l,
                              double *evec /* [e][i] */)
{
   const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (t >= L.ne * L.nd) return;
   evec[t] = l[gmap[L.slot(static_cast<int>(t % L.nd), t / L.nd)] & kDofMask];
}

// Transpose of gather in element order, y += (forms.cpp:289-295).  Exclusive
// DOFs: one slot.  Shared DOFs: their sorted slot list.
__global__ void exclusive_add_kernel(const uint32_t *gmap, Layout L,
                                     const double *evec /* [e][i] */, double *l)
{
   const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (t >= L.ne * L.nd) return;
   const uint32_t g = gmap[L.slot(static_cast<int>(t % L.nd), t / L.nd)];
   if (g & kExclusive) l[g & kDofMask] += evec[t];
}

__global__ void shared_add_kernel(const int32_t *shared_dofs, const int32_t *off,
                                  const uint32_t *slots, int64_t n_shared, Layout L,
                                  const double *evec /* [e][i] */, double *l)
{
   const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (s >= n_shared) return;
   const int32_t d = shared_dofs[s];
   double acc = l[d];
   for (int k = off[s]; k < off[s + 1]; k++) {
      const uint32_t slot = slots[k];
      acc += evec[L.elem_of(slot) * L.nd + L.local_of(slot)];
   }
   l[d] = acc;
}

// Boundary of a Cartesian mesh: DOFs at lattice positions on the domain
// boundary (the set essential_true_dofs collects over all attributes).
__global__ void boundary_mark_kernel(const uint32_t *gmap, Layout L, int dim, int nx, int ny,
                                     int nz, int p, int32_t *mark)
{
   const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (e >= L.ne) return;
   const int i = static_cast<int>(e % nx);
   const int j = static_cast<int>((e / nx) % ny);
   const int k = dim == 3 ? static_cast<int>(e / ((int64_t)nx * ny)) : 0;
   const bool touches = i == 0 || i == nx - 1 || j == 0 || j == ny - 1 ||
                        (dim == 3 && (k == 0 || k == nz - 1));
   if (!touches) return;
   const int D1 = p + 1;
   const int nd = dim == 2 ? D1 * D1 : D1 * D1 * D1;
   for (int l = 0; l < nd; l++) {
      const int a = l % D1, b = (l / D1) % D1, c = l / (D1 * D1);
      bool on = (i == 0 && a == 0) || (i == nx - 1 && a == p) || (j == 0 && b == 0) ||
                (j == ny - 1 && b == p);
      if (dim == 3) on = on || (k == 0 && c == 0) || (k == nz - 1 && c == p);
      if (on) mark[gmap[L.slot(l, e)] & kDofMask] = 1;
   }
}

template <typename T>
T *dalloc(int64_t n)
{
   T *p = nullptr;
   TFEM_CUDA(cudaMalloc(&p, sizeof(T) * static_cast<size_t>(n > 0 ? n : 1)));
   return p;
}

void exclusive_scan(tfem_ctx *ctx, const int32_t *in, int32_t *out, int64_t n)
{
   size_t bytes = 0;
   TFEM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, ctx->stream));
   void *tmp = dalloc<char>(static_cast<int64_t>(bytes));
   TFEM_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, n, ctx->stream));
   TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   cudaFree(tmp);
   ctx->launched();
}

} // namespace

tfem_restriction *restriction_from_map(tfem_ctx *ctx, int dim, int p, int64_t ne, int64_t ndofs,
                                       bool elem_major, uint32_t *gmap)
{
   auto *r = new tfem_restriction;
   r->ctx = ctx;
   r->dim = dim;
   r->p = p;
   r->nd = dim == 2 ? (p + 1) * (p + 1) : (p + 1) * (p + 1) * (p + 1);
   r->ne = ne;
   r->ne_pad = round_up(ne, 64);
   r->ndofs = ndofs;
   r->elem_major = elem_major;
   r->gmap = gmap;
   const int64_t nslots = ne * r->nd;
   if (nslots >= (int64_t)INT32_MAX) invalid("restriction: more than 2^31-1 element slots on one device");
   const Layout L{elem_major, r->nd, ne, r->ne_pad};
   cudaStream_t s = ctx->stream;

   int32_t *counts = dalloc<int32_t>(ndofs), *is_shared = dalloc<int32_t>(ndofs);
   int32_t *shared_count = dalloc<int32_t>(ndofs), *rank = dalloc<int32_t>(ndofs + 1);
   int32_t *slot_off_full = dalloc<int32_t>(ndofs + 1);
   TFEM_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * ndofs, s));
   count_kernel<<<blocks_for(nslots), kThreads, 0, s>>>(gmap, L, counts);
   flag_kernel<<<blocks_for(ndofs), kThreads, 0, s>>>(counts, ndofs, is_shared, shared_count);
   mark_exclusive_kernel<<<blocks_for(nslots), kThreads, 0, s>>>(gmap, L, counts);
   ctx->launched(3);
   TFEM_CUDA(cudaGetLastError());
   exclusive_scan(ctx, is_shared, rank, ndofs);
   exclusive_scan(ctx, shared_count, slot_off_full, ndofs);
   int32_t last_rank = 0, last_flag = 0, last_off = 0, last_cnt = 0;
   TFEM_CUDA(cudaMemcpy(&last_rank, rank + ndofs - 1, 4, cudaMemcpyDeviceToHost));
   TFEM_CUDA(cudaMemcpy(&last_flag, is_shared + ndofs - 1, 4, cudaMemcpyDeviceToHost));
   TFEM_CUDA(cudaMemcpy(&last_off, slot_off_full + ndofs - 1, 4, cudaMemcpyDeviceToHost));
   TFEM_CUDA(cudaMemcpy(&last_cnt, shared_count + ndofs - 1, 4, cudaMemcpyDeviceToHost));
   r->n_shared = last_rank + last_flag;
   const int64_t n_shared_slots = static_cast<int64_t>(last_off) + last_cnt;

   r->shared_dofs = dalloc<int32_t>(r->n_shared);
   r->shared_off = dalloc<int32_t>(r->n_shared + 1);
   r->shared_slots = dalloc<uint32_t>(n_shared_slots);
   compact_shared_kernel<<<blocks_for(ndofs), kThreads, 0, s>>>(is_shared, rank, ndofs,
                                                               r->shared_dofs);
   // shared_off[rank[d]] = slot_off_full[d]; the last entry is the total.
   if (r->n_shared > 0) {
      gather_off_kernel<<<blocks_for(r->n_shared), kThreads, 0, s>>>(
         r->shared_dofs, slot_off_full, r->n_shared, r->shared_off);
      ctx->launched();
   }
   {
      const int32_t total = static_cast<int32_t>(n_shared_slots);
      TFEM_CUDA(cudaMemcpyAsync(r->shared_off + r->n_shared, &total, 4, cudaMemcpyHostToDevice, s));
      TFEM_CUDA(cudaStreamSynchronize(s));
   }
   TFEM_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * (r->n_shared > 0 ? r->n_shared : 1), s));
   fill_slots_kernel<<<blocks_for(nslots), kThreads, 0, s>>>(gmap, L, rank, is_shared,
                                                            r->shared_off, counts,
                                                            r->shared_slots);
   if (r->n_shared > 0) {
      sort_slots_kernel<<<blocks_for(r->n_shared), kThreads, 0, s>>>(r->shared_off, r->n_shared,
                                                                     L, r->shared_slots);
      ctx->launched();
   }
   ctx->launched(2);
   TFEM_CUDA(cudaGetLastError());
   TFEM_CUDA(cudaStreamSynchronize(s));
   cudaFree(counts);
   cudaFree(is_shared);
   cudaFree(shared_count);
   cudaFree(rank);
   cudaFree(slot_off_full);
   return r;
}

void restriction_mult_transpose(tfem_ctx *ctx, const tfem_restriction *r, const double *e,
                                double *l)
{
   const int64_t nslots = r->ne * r->nd;
   const Layout L{r->elem_major, r->nd, r->ne, r->ne_pad};
   exclusive_add_kernel<<<blocks_for(nslots), kThreads, 0, ctx->stream>>>(r->gmap, L, e, l);
   if (r->n_shared > 0)
      shared_add_kernel<<<blocks_for(r->n_shared), kThreads, 0, ctx->stream>>>(
         r->shared_dofs, r->shared_off, r->shared_slots, r->n_shared, L, e, l);
   ctx->launched(2);
   TFEM_CUDA(cudaGetLastError());
}

} // namespace tfem

using namespace tfem;

// Entry points used by capi.cu
namespace tfem {

tfem_restriction *restriction_cartesian(tfem_ctx *ctx, int dim, const int *n, int p)
{
   if (dim != 2 && dim != 3) invalid("restriction: dim must be 2 or 3");
   if (p < 1 || p > kMaxP) invalid("build_h1_layout: order must be >= 1 (and <= 8 on device)");
   for (int d = 0; d < dim; d++)
      if (n[d] < 1) invalid("make_cartesian: need nx, ny >= 1");
   int64_t ne = 1, nv = 1;
   for (int d = 0; d < dim; d++) {
      ne *= n[d];
      nv *= n[d] + 1;
   }
   const int64_t pe = p - 1;
   int64_t ndofs;
   if (dim == 2) {
      const int64_t n_edges = (int64_t)n[0] * (n[1] + 1) + (int64_t)n[1] * (n[0] + 1);
      ndofs = nv + n_edges * pe + ne * pe * pe;
   } else {
      const int64_t nvx = n[0] + 1, nvy = n[1] + 1, nvz = n[2] + 1;
      const int64_t edges = (int64_t)n[0] * nvy * nvz + nvx * n[1] * nvz + nvx * nvy * n[2];
      const int64_t faces = nvx * n[1] * n[2] + (int64_t)n[0] * nvy * n[2] +
                            (int64_t)n[0] * n[1] * nvz;
      ndofs = nv + edges * pe + faces * pe * pe + ne * pe * pe * pe;
   }
   if (ndofs >= (int64_t)kDofMask) invalid("restriction: more than 2^31-1 DOFs on one device");
   const int nd = dim == 2 ? (p + 1) * (p + 1) : (p + 1) * (p + 1) * (p + 1);
   const int64_t ne_pad = round_up(ne, 64);
   if ((int64_t)nd * ne_pad >= (int64_t)UINT32_MAX) invalid("restriction: too many element slots");
   uint32_t *gmap = dalloc<uint32_t>(nd * ne_pad);
   TFEM_CUDA(cudaMemsetAsync(gmap, 0, sizeof(uint32_t) * nd * ne_pad, ctx->stream));
   const bool em = elem_major_layout(dim, p);
   if (dim == 2)
      layout2d_kernel<<<blocks_for(ne), kThreads, 0, ctx->stream>>>(n[0], n[1], p,
                                                                   Layout{em, nd, ne, ne_pad}, gmap);
   else
      layout3d_kernel<<<blocks_for(ne), kThreads, 0, ctx->stream>>>(n[0], n[1], n[2], p, gmap);
   ctx->launched();
   TFEM_CUDA(cudaGetLastError());
   tfem_restriction *r = restriction_from_map(ctx, dim, p, ne, ndofs, em, gmap);
   r->cartesian = true;
   for (int d = 0; d < dim; d++) r->n[d] = n[d];
   return r;
}

tfem_restriction *restriction_create(tfem_ctx *ctx, int dim, int p, int64_t ne, int64_t ndofs,
                                     const int32_t *elem_dofs)
{
   if (dim != 2 && dim != 3) invalid("restriction: dim must be 2 or 3");
   if (p < 1 || p > kMaxP) invalid("restriction: order must be in [1, 8]");
   if (ne < 1 || ndofs < 1) invalid("restriction: empty mesh");
   if (ndofs >= (int64_t)kDofMask) invalid("restriction: more than 2^31-1 DOFs on one device");
   const int nd = dim == 2 ? (p + 1) * (p + 1) : (p + 1) * (p + 1) * (p + 1);
   const int64_t ne_pad = round_up(ne, 64);
   int32_t *emap = dalloc<int32_t>(ne * nd);
   int *bad = dalloc<int>(1);
   TFEM_CUDA(cudaMemcpy(emap, elem_dofs, sizeof(int32_t) * ne * nd, cudaMemcpyHostToDevice));
   TFEM_CUDA(cudaMemset(bad, 0, sizeof(int)));
   uint32_t *gmap = dalloc<uint32_t>(nd * ne_pad);
   TFEM_CUDA(cudaMemsetAsync(gmap, 0, sizeof(uint32_t) * nd * ne_pad, ctx->stream));
   const Layout L{elem_major_layout(dim, p), nd, ne, ne_pad};
   transpose_in_kernel<<<blocks_for(ne * nd), kThreads, 0, ctx->stream>>>(emap, L, ndofs, gmap,
                                                                         bad);
   ctx->launched();
   int hbad = 0;
   TFEM_CUDA(cudaMemcpy(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost));
   cudaFree(emap);
   cudaFree(bad);
   if (hbad) {
      cudaFree(gmap);
      invalid("restriction: element DOF index out of range");
   }
   return restriction_from_map(ctx, dim, p, ne, ndofs, elem_major_layout(dim, p), gmap);
}

void restriction_destroy(tfem_restriction *r)
{
   if (!r) return;
   cudaFree(r->gmap);
   cudaFree(r->shared_dofs);
   cudaFree(r->shared_off);
   cudaFree(r->shared_slots);
   cudaFree(r->evec);
   delete r;
}

void restriction_elem_dofs(const tfem_restriction *r, int32_t *host)
{
   std::vector<uint32_t> g(static_cast<size_t>(r->nd) * r->ne_pad);
   TFEM_CUDA(cudaMemcpy(g.data(), r->gmap, sizeof(uint32_t) * g.size(), cudaMemcpyDeviceToHost));
   const Layout L{r->elem_major, r->nd, r->ne, r->ne_pad};
   for (int64_t e = 0; e < r->ne; e++)
      for (int i = 0; i < r->nd; i++)
         host[e * r->nd + i] = static_cast<int32_t>(g[L.slot(i, e)] & kDofMask);
}

int64_t restriction_boundary_dofs(const tfem_restriction *r, int32_t *host)
{
   if (!r->cartesian) invalid("restriction_boundary_dofs: needs a Cartesian restriction");
   tfem_ctx *ctx = r->ctx;
   int32_t *mark = dalloc<int32_t>(r->ndofs);
   TFEM_CUDA(cudaMemsetAsync(mark, 0, sizeof(int32_t) * r->ndofs, ctx->stream));
   const Layout L{r->elem_major, r->nd, r->ne, r->ne_pad};
   boundary_mark_kernel<<<blocks_for(r->ne), kThreads, 0, ctx->stream>>>(
      r->gmap, L, r->dim, r->n[0], r->n[1], r->n[2], r->p, mark);
   ctx->launched();
   std::vector<int32_t> h(r->ndofs);
   TFEM_CUDA(cudaMemcpyAsync(h.data(), mark, sizeof(int32_t) * r->ndofs, cudaMemcpyDeviceToHost,
                             ctx->stream));
   TFEM_CUDA(cudaStreamSynchronize(ctx->stream));
   cudaFree(mark);
   int64_t cnt = 0;
   for (int64_t d = 0; d < r->ndofs; d++)
      if (h[d]) {
         if (host) host[cnt] = static_cast<int32_t>(d);
         cnt++;
      }
   return cnt;
}

void restriction_mult(tfem_ctx *ctx, const tfem_restriction *r, const double *l, double *e)
{
   const Layout L{r->elem_major, r->nd, r->ne, r->ne_pad};
   gather_kernel<<<blocks_for(r->ne * r->nd), kThreads, 0, ctx->stream>>>(r->gmap, L, l, e);
   ctx->launched();
   TFEM_CUDA(cudaGetLastError());
}

} // namespace tfem

double *tfem_restriction::ensure_evec()
{
   if (!evec) TFEM_CUDA(cudaMalloc(&evec, sizeof(double) * static_cast<size_t>(nd) * ne_pad));
   return evec;
}

