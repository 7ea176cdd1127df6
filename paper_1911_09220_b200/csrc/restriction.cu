// Element restriction G / G^T on the device.
//
// Device layout: the element map is stored slot-major,
// gmap[i * ne_pad + pos] (thread-per-element gathers are coalesced; pos is
// the element's position in ElemOrder), with bit 31 set when DOF has a single
// element slot ("exclusive": written straight from the element kernel).  DOFs
// with >= 2 slots get a transpose CSR whose slot lists are sorted by element
// -- the reference's ascending-element accumulation (forms.cpp:289-295)
// without atomics.  Ordered spaces (ElemOrder) also flag the DOFs whose slots
// all fall in one warp patch (kWarpOwner / kWarpMember).
#include "common.cuh"

#include <cub/cub.cuh>

#include <algorithm>

namespace tfem {

void restriction_destroy(tfem_restriction *r);

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
   ElemOrder order;
   // slot of (local i, element e) for an element in reference numbering
   __host__ __device__ int64_t slot_e(int i, int64_t e) const { return slot(i, order.pos_of(e)); }
   // reference element of a slot (the accumulation-order key)
   __host__ __device__ int64_t elem_key(int64_t s) const { return order.elem_at(elem_of(s)); }
   __host__ __device__ int64_t slot(int i, int64_t e) const
   {
      return elem_major ? e * nd + i : (int64_t)i * ne_pad + e;
   }
   __host__ __device__ int64_t elem_of(int64_t s) const { return elem_major ? s / nd : s % ne_pad; }
   __host__ __device__ int local_of(int64_t s) const
   {
      return static_cast<int>(elem_major ? s % nd : s / ne_pad);
   }
   // t in [0, ne*nd) enumerates every live slot (padding positions excluded)
   __host__ __device__ int64_t live(int64_t t) const
   {
      return elem_major ? t : slot_e(static_cast<int>(t / ne), t % ne);
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
      gmap[L.slot_e(a + b * D1, e)] = static_cast<uint32_t>(dof);
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

__global__ void mark_exclusive_kernel(uint32_t *gmap, Layout L, const int32_t *counts)
{
   const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (t >= L.ne * L.nd) return;
   const int64_t s = L.live(t);
   const uint32_t g = gmap[s];
   if (counts[g & kDofMask] == 1) gmap[s] = g | kExclusive;
}

__global__ void flag_count_kernel(const int32_t *counts, int64_t ndofs, int c, int32_t *flag)
{
   const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (d < ndofs) flag[d] = counts[d] == c ? 1 : 0;
}

// Position of every shared DOF inside its bucket: bucket_of[d] / rank[d].
__global__ void rank_kernel(const int32_t *flag, const int32_t *scan, int64_t ndofs, int b,
                            int8_t *bucket_of, int32_t *rank, int32_t *dofs)
{
   const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (d >= ndofs || !flag[d]) return;
   bucket_of[d] = static_cast<int8_t>(b);
   rank[d] = scan[d];
   dofs[scan[d]] = static_cast<int32_t>(d);
}

struct BucketPtrs {
   int c[tfem_restriction::kMaxBuckets];
   uint32_t *slots[tfem_restriction::kMaxBuckets];
};

__global__ void fill_slots_kernel(const uint32_t *gmap, Layout L, const int8_t *bucket_of,
                                  const int32_t *rank, int32_t *fill, BucketPtrs bp)
{
   const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (t >= L.ne * L.nd) return;
   const int64_t s = L.live(t);
   const uint32_t d = gmap[s] & kDofMask;
   const int b = bucket_of[d];
   if (b < 0) return;
   const int c = bp.c[b];
   const int pos = atomicAdd(fill + d, 1);
   bp.slots[b][(int64_t)rank[d] * c + pos] = static_cast<uint32_t>(s);
}

// Rows are tiny (c <= 8): insertion-sort each by element so the scatter adds
// contributions in ascending element order (forms.cpp:289-295).
__global__ void sort_rows_kernel(uint32_t *slots, int64_t n, int c, Layout L)
{
   const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (s >= n) return;
   uint32_t *row = slots + s * c;
   for (int a = 1; a < c; a++) {
      const uint32_t v = row[a];
      const int64_t key = L.elem_key(v);
      int b = a - 1;
      while (b >= 0 && L.elem_key(row[b]) > key) {
         row[b + 1] = row[b];
         b--;
      }
      row[b + 1] = v;
   }
}

__global__ void gather_kernel(const uint32_t *gmap, Layout L, const double *l,
                              double *evec /* [e][i] */)
{
   const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (t >= L.ne * L.nd) return;
   evec[t] = l[gmap[L.slot_e(static_cast<int>(t % L.nd), t / L.nd)] & kDofMask];
}

// Transpose of gather in element order, y += (forms.cpp:289-295).  Exclusive
// DOFs: one slot.  Shared DOFs: their sorted slot list.
__global__ void exclusive_add_kernel(const uint32_t *gmap, Layout L,
                                     const double *evec /* [e][i] */, double *l)
{
   const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (t >= L.ne * L.nd) return;
   const uint32_t g = gmap[L.slot_e(static_cast<int>(t % L.nd), t / L.nd)];
   if (is_exclusive(g)) l[g & kDofMask] += evec[t];
}

// API E-vector [e][i] -> internal gmap layout.
__global__ void to_internal_kernel(Layout L, const uint16_t *perm, const double *api, double *evec)
{
   const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (t >= L.ne * L.nd) return;
   const int i = static_cast<int>(t % L.nd);
   const int64_t pos = L.order.pos_of(t / L.nd);
   evec[L.elem_major ? ev_em_p(perm, L.nd, pos, i) : (int64_t)i * L.ne_pad + pos] = api[t];
}

// Bucket slots (map indices e nd + i) -> E-vector indices e nd + perm[i].
__global__ void remap_slots_kernel(uint32_t *slots, int64_t n, int nd, const uint16_t *perm)
{
   const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (k >= n) return;
   const uint32_t s = slots[k];
   slots[k] = (s / nd) * nd + perm[s % nd];
}

// E-vector slot order inside an element: the interior slots, then (3D) each
// face's (p-1)^2, each edge's p-1, the vertices -- sub-entities in (c, b, a)
// class order (0 / interior / p), slots in natural order inside.
std::vector<uint16_t> ev_perm(int dim, int p)
{
   const int D1 = p + 1, C1 = dim == 3 ? D1 : 1, K3 = dim == 3 ? 3 : 1;
   auto cls = [p](int x) { return x == 0 ? 0 : (x == p ? 2 : 1); };
   std::vector<uint16_t> perm(D1 * D1 * C1);
   int next = 0;
   for (int m = dim; m >= 0; m--) // interior coordinates of the sub-entity
      for (int kc = 0; kc < K3; kc++)
         for (int kb = 0; kb < 3; kb++)
            for (int ka = 0; ka < 3; ka++) {
               const int kcc = dim == 3 ? kc : -1;
               if ((ka == 1) + (kb == 1) + (kcc == 1) != m) continue;
               for (int c = 0; c < C1; c++)
                  for (int b = 0; b < D1; b++)
                     for (int a = 0; a < D1; a++)
                        if (cls(a) == ka && cls(b) == kb && (dim == 2 || cls(c) == kc))
                           perm[a + D1 * (b + D1 * c)] = static_cast<uint16_t>(next++);
            }
   return perm;
}


// project_coefficient's `g.values()[dofs[...]] = v` (fespace.cpp:334-356):
// every DOF takes the value of its last element.  Exclusive slots directly,
// shared DOFs from the last slot of their (element-sorted) bucket row.
__global__ void assign_exclusive_kernel(const uint32_t *gmap, Layout L,
                                        const double *evec /* [e][i] */, double *l)
{
   const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (t >= L.ne * L.nd) return;
   const uint32_t g = gmap[L.slot_e(static_cast<int>(t % L.nd), t / L.nd)];
   if (is_exclusive(g)) l[g & kDofMask] = evec[t];
}

__global__ void assign_last_kernel(const int32_t *dofs, const uint32_t *slots, int64_t n, int c,
                                   const double *evec_internal, double *l)
{
   const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (k < n) l[dofs[k]] = evec_internal[slots[k * c + c - 1]];
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
      if (on) mark[gmap[L.slot_e(l, e)] & kDofMask] = 1;
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

__global__ void first_slot_kernel(const uint32_t *slots, int64_t n, int c, uint32_t *key,
                                  int32_t *idx)
{
   const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (k >= n) return;
   key[k] = slots[k * c];
   idx[k] = static_cast<int32_t>(k);
}

__global__ void permute_rows_kernel(const int32_t *perm, int64_t n, int c, const int32_t *dofs,
                                    const uint32_t *slots, int32_t *dofs2, uint32_t *slots2)
{
   const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (k >= n) return;
   const int64_t src = perm[k];
   dofs2[k] = dofs[src];
   for (int j = 0; j < c; j++) slots2[k * c + j] = slots[src * c + j];
}

// Reorder a bucket's rows by their first slot (stable radix sort).
void sort_rows_by_first_slot(tfem_ctx *ctx, tfem_restriction::Bucket &bk)
{
   cudaStream_t s = ctx->stream;
   const int64_t n = bk.n;
   uint32_t *key = dalloc<uint32_t>(n), *key2 = dalloc<uint32_t>(n);
   int32_t *idx = dalloc<int32_t>(n), *perm = dalloc<int32_t>(n), *dofs2 = dalloc<int32_t>(n);
   uint32_t *slots2 = dalloc<uint32_t>(n * bk.c);
   first_slot_kernel<<<blocks_for(n), kThreads, 0, s>>>(bk.slots, n, bk.c, key, idx);
   size_t bytes = 0;
   TFEM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key, key2, idx, perm, n, 0, 32, s));
   void *tmp = dalloc<char>(static_cast<int64_t>(bytes));
   TFEM_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, key, key2, idx, perm, n, 0, 32, s));
   permute_rows_kernel<<<blocks_for(n), kThreads, 0, s>>>(perm, n, bk.c, bk.dofs, bk.slots, dofs2,
                                                         slots2);
   ctx->launched(3);
   TFEM_CUDA(cudaGetLastError());
   TFEM_CUDA(cudaStreamSynchronize(s));
   cudaFree(bk.dofs);
   cudaFree(bk.slots);
   bk.dofs = dofs2;
   bk.slots = slots2;
   for (void *p : {static_cast<void *>(key), static_cast<void *>(key2), static_cast<void *>(idx),
                   static_cast<void *>(perm), tmp})
      cudaFree(p);
}

// Warp-local DOFs of an ordered space (on the device, once per space).  A
// shared DOF is warp-local when all its slots lie in one warp patch (32
// positions, lane = 8 r + c); its slot of the highest element is the owner
// (kWarpOwner), the others members.  The kernel finds an owner's members by
// position alone (warp_partners below: left / lower neighbours inside the
// patch, in ascending element order) -- checked here against the sorted slot
// list, so a DOF is only flagged when the rule reproduces it exactly.  All
// other shared DOFs form the global buckets.
struct Partner {
   int lane_off, i; // member lane = owner lane - lane_off, local index i
};
__host__ __device__ int warp_partners(int p, int a, int b, int c, int r, Partner *out)
{
   const int D1 = p + 1;
   int n = 0;
   if (a == 0 && b == 0) {
      if (c >= 1 && r >= 1) out[n++] = {9, p + p * D1};
      if (r >= 1) out[n++] = {8, 0 + p * D1};
      if (c >= 1) out[n++] = {1, p + 0 * D1};
   } else if (a == 0 && b == p) {
      if (c >= 1) out[n++] = {1, p + p * D1};
   } else if (a == p && b == 0) {
      if (r >= 1) out[n++] = {8, p + p * D1};
   } else if (a == 0) {
      if (c >= 1) out[n++] = {1, p + b * D1};
   } else if (b == 0) {
      if (r >= 1) out[n++] = {8, a + p * D1};
   } else {
      return -1; // never an owner
   }
   return n;
}

// One thread per bucket row (sorted by element): flag a warp-local DOF's
// slots in place (members, owner = the last slot) when its slots share one
// patch and the owner's partner rule lists exactly the others; global[k] = 1
// for every other row (it stays with the scatter).
__global__ void warp_local_kernel(uint32_t *gmap, Layout L, int p, const uint32_t *slots,
                                  int64_t n, int c, int32_t *global)
{
   const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (k >= n) return;
   constexpr int W = 32;
   const int D1 = p + 1;
   const uint32_t *row = slots + k * c;
   const int64_t w0 = L.elem_of(row[0]) / W;
   bool local = true;
   for (int j = 1; j < c && local; j++) local = L.elem_of(row[j]) / W == w0;
   if (local) {
      const uint32_t os = row[c - 1];
      const int64_t opos = L.elem_of(os);
      const int oi = L.local_of(os), lane = static_cast<int>(opos % W);
      Partner pt[4];
      const int m = warp_partners(p, oi % D1, oi / D1, lane % 8, lane / 8, pt);
      local = m == c - 1;
      for (int j = 0; j < m && local; j++)
         local = row[j] == static_cast<uint32_t>(L.slot(pt[j].i, opos - pt[j].lane_off));
   }
   if (local) {
      for (int j = 0; j + 1 < c; j++) gmap[row[j]] |= kWarpMember;
      gmap[row[c - 1]] |= kWarpOwner;
   }
   global[k] = local ? 0 : 1;
}

// Copy the flagged rows (dofs + c slots) to their scanned positions.
__global__ void compact_rows_kernel(const int32_t *global, const int32_t *at, int64_t n, int c,
                                    const int32_t *dofs, const uint32_t *slots, int32_t *gdofs,
                                    uint32_t *gslots)
{
   const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   if (k >= n || !global[k]) return;
   const int64_t to = at[k];
   gdofs[to] = dofs[k];
   for (int j = 0; j < c; j++) gslots[to * c + j] = slots[k * c + j];
}

void build_warp_local(tfem_restriction *r, const Layout &L)
{
   tfem_ctx *ctx = r->ctx;
   cudaStream_t s = ctx->stream;
   for (int b = 0; b < r->n_buckets; b++) {
      const auto &bk = r->buckets[b];
      if (bk.n == 0) continue;
      int32_t *global = dalloc<int32_t>(bk.n), *at = dalloc<int32_t>(bk.n);
      warp_local_kernel<<<blocks_for(bk.n), kThreads, 0, s>>>(r->gmap, L, r->p, bk.slots, bk.n,
                                                             bk.c, global);
      ctx->launched();
      exclusive_scan(ctx, global, at, bk.n);
      int32_t last_at = 0, last_g = 0;
      d2h(s, &last_at, at + bk.n - 1, 4);
      d2h(s, &last_g, global + bk.n - 1, 4);
      const int64_t m = static_cast<int64_t>(last_at) + last_g;
      if (m > 0) {
         auto &g = r->gbuckets[r->n_gbuckets++];
         g.c = bk.c;
         g.n = m;
         g.dofs = dalloc<int32_t>(m);
         g.slots = dalloc<uint32_t>(m * g.c);
         compact_rows_kernel<<<blocks_for(bk.n), kThreads, 0, s>>>(global, at, bk.n, bk.c, bk.dofs,
                                                                  bk.slots, g.dofs, g.slots);
         ctx->launched();
         r->n_gshared += m;
      }
      TFEM_CUDA(cudaGetLastError());
      TFEM_CUDA(cudaStreamSynchronize(s));
      cudaFree(global);
      cudaFree(at);
   }
   r->warp_local = true;
}

} // namespace

tfem_restriction *restriction_from_map(tfem_ctx *ctx, int dim, int p, int64_t ne, int64_t ndofs,
                                       bool elem_major, uint32_t *gmap, ElemOrder order)
{
   auto *r = new tfem_restriction;
   r->ctx = ctx;
   r->dim = dim;
   r->p = p;
   r->nd = dim == 2 ? (p + 1) * (p + 1) : (p + 1) * (p + 1) * (p + 1);
   r->ne = ne;
   r->npos = order.n_pos(ne);
   r->ne_pad = round_up(r->npos, 64);
   r->ndofs = ndofs;
   r->elem_major = elem_major;
   r->gmap = gmap;
   r->order = order;
   const int64_t nslots = ne * r->nd;
   if (nslots >= (int64_t)INT32_MAX) invalid("restriction: more than 2^31-1 element slots on one device");
   const Layout L{elem_major, r->nd, ne, r->ne_pad, order};
   cudaStream_t s = ctx->stream;

   int32_t *counts = dalloc<int32_t>(ndofs), *flag = dalloc<int32_t>(ndofs);
   int32_t *scan = dalloc<int32_t>(ndofs), *rank = dalloc<int32_t>(ndofs);
   int8_t *bucket_of = dalloc<int8_t>(ndofs);
   TFEM_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * ndofs, s));
   TFEM_CUDA(cudaMemsetAsync(bucket_of, 0xff, ndofs, s));
   count_kernel<<<blocks_for(nslots), kThreads, 0, s>>>(gmap, L, counts);
   mark_exclusive_kernel<<<blocks_for(nslots), kThreads, 0, s>>>(gmap, L, counts);
   ctx->launched(2);
   TFEM_CUDA(cudaGetLastError());
   BucketPtrs bp{};
   const int cmax = 8; // conforming quads / hexes: 4 / 8; larger valences are rejected below
   int64_t covered = 0; // slots accounted for by exclusive DOFs and buckets
   for (int c = 1; c <= cmax; c++) {
      flag_count_kernel<<<blocks_for(ndofs), kThreads, 0, s>>>(counts, ndofs, c, flag);
      ctx->launched();
      exclusive_scan(ctx, flag, scan, ndofs);
      int32_t last_scan = 0, last_flag = 0;
      d2h(s, &last_scan, scan + ndofs - 1, 4);
      d2h(s, &last_flag, flag + ndofs - 1, 4);
      const int64_t n = static_cast<int64_t>(last_scan) + last_flag;
      covered += n * c;
      if (n == 0 || c == 1) continue;
      const int b = r->n_buckets++;
      auto &bk = r->buckets[b];
      bk.c = c;
      bk.n = n;
      bk.dofs = dalloc<int32_t>(n);
      bk.slots = dalloc<uint32_t>(n * c);
      rank_kernel<<<blocks_for(ndofs), kThreads, 0, s>>>(flag, scan, ndofs, b, bucket_of, rank,
                                                        bk.dofs);
      ctx->launched();
      bp.c[b] = c;
      bp.slots[b] = bk.slots;
      r->n_shared += n;
   }
   if (covered != nslots) {
      cudaFree(counts);
      cudaFree(flag);
      cudaFree(scan);
      cudaFree(rank);
      cudaFree(bucket_of);
      restriction_destroy(r);
      invalid("restriction: a DOF is shared by more than 8 elements");
   }
   TFEM_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * ndofs, s));
   // 3D only: in 2D (p >= 4) the element kernel's scattered stores cost
   // more than the scatter gains (measured -3 to -5 %)
   if (elem_major && r->dim == 3 && r->p >= 3) {
      const std::vector<uint16_t> perm = ev_perm(r->dim, r->p);
      r->evperm = dalloc<uint16_t>(r->nd);
      h2d(s, r->evperm, perm.data(), sizeof(uint16_t) * perm.size());
   }
   if (r->n_buckets > 0) {
      fill_slots_kernel<<<blocks_for(nslots), kThreads, 0, s>>>(gmap, L, bucket_of, rank, counts,
                                                               bp);
      ctx->launched();
      for (int b = 0; b < r->n_buckets; b++) {
         sort_rows_kernel<<<blocks_for(r->buckets[b].n), kThreads, 0, s>>>(
            r->buckets[b].slots, r->buckets[b].n, r->buckets[b].c, L);
         ctx->launched();
         if (r->evperm) {
            const int64_t m = r->buckets[b].n * r->buckets[b].c;
            remap_slots_kernel<<<blocks_for(m), kThreads, 0, s>>>(r->buckets[b].slots, m, r->nd,
                                                                  r->evperm);
            ctx->launched();
         }
         // element-major E-vector: rows in first-slot (element) order, so the
         // scatter's threads read neighbouring slots of the same elements
         if (elem_major) sort_rows_by_first_slot(ctx, r->buckets[b]);
      }
   }
   TFEM_CUDA(cudaGetLastError());
   TFEM_CUDA(cudaStreamSynchronize(s));
   cudaFree(counts);
   cudaFree(flag);
   cudaFree(scan);
   cudaFree(rank);
   cudaFree(bucket_of);
   if (order.pw == 8 && order.ph == 4 && !elem_major) build_warp_local(r, L);
   return r;
}

void restriction_mult_transpose(tfem_ctx *ctx, const tfem_restriction *r, const double *e,
                                double *l)
{
   const int64_t nslots = r->ne * r->nd;
   const Layout L{r->elem_major, r->nd, r->ne, r->ne_pad, r->order};
   exclusive_add_kernel<<<blocks_for(nslots), kThreads, 0, ctx->stream>>>(r->gmap, L, e, l);
   ctx->launched();
   if (r->n_shared > 0) {
      double *ev = const_cast<tfem_restriction *>(r)->ensure_evec();
      to_internal_kernel<<<blocks_for(nslots), kThreads, 0, ctx->stream>>>(L, r->evperm, e, ev);
      ctx->launched();
      scatter_shared(ctx, r, ev, nullptr, l, false, nullptr, nullptr, nullptr, false);
   }
   TFEM_CUDA(cudaGetLastError());
}

} // namespace tfem

using namespace tfem;

// Entry points used by capi.cu
namespace tfem {

tfem_restriction *restriction_cartesian(tfem_ctx *ctx, int dim, const int *n, int p)
{
   if (dim != 2 && dim != 3) invalid("restriction: dim must be 2 or 3");
   if (p < 1 || p > (dim == 3 ? kMaxP3D : kMaxP))
      invalid("build_h1_layout: order must be >= 1 (and <= 16 in 2D, 8 in 3D, on the device)");
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
   if (ndofs >= (int64_t)kDofMask) invalid("restriction: more than 2^30-1 DOFs on one device");
   const int nd = dim == 2 ? (p + 1) * (p + 1) : (p + 1) * (p + 1) * (p + 1);
   const ElemOrder order = elem_order_for(dim, p, true, n);
   const int64_t ne_pad = round_up(order.n_pos(ne), 64);
   if ((int64_t)nd * ne_pad >= (int64_t)UINT32_MAX) invalid("restriction: too many element slots");
   uint32_t *gmap = dalloc<uint32_t>(nd * ne_pad);
   TFEM_CUDA(cudaMemsetAsync(gmap, 0, sizeof(uint32_t) * nd * ne_pad, ctx->stream));
   const bool em = elem_major_layout(dim, p);
   if (dim == 2)
      layout2d_kernel<<<blocks_for(ne), kThreads, 0, ctx->stream>>>(
         n[0], n[1], p, Layout{em, nd, ne, ne_pad, order}, gmap);
   else
      layout3d_kernel<<<blocks_for(ne), kThreads, 0, ctx->stream>>>(n[0], n[1], n[2], p, gmap);
   ctx->launched();
   TFEM_CUDA(cudaGetLastError());
   tfem_restriction *r = restriction_from_map(ctx, dim, p, ne, ndofs, em, gmap, order);
   r->cartesian = true;
   for (int d = 0; d < dim; d++) r->n[d] = n[d];
   return r;
}

tfem_restriction *restriction_create(tfem_ctx *ctx, int dim, int p, int64_t ne, int64_t ndofs,
                                     const int32_t *elem_dofs)
{
   if (dim != 2 && dim != 3) invalid("restriction: dim must be 2 or 3");
   if (p < 1 || p > (dim == 3 ? kMaxP3D : kMaxP))
      invalid("restriction: order must be in [1, 16] (2D) / [1, 8] (3D)");
   if (ne < 1 || ndofs < 1) invalid("restriction: empty mesh");
   if (ndofs >= (int64_t)kDofMask) invalid("restriction: more than 2^30-1 DOFs on one device");
   const int nd = dim == 2 ? (p + 1) * (p + 1) : (p + 1) * (p + 1) * (p + 1);
   const int64_t ne_pad = round_up(ne, 64);
   int32_t *emap = dalloc<int32_t>(ne * nd);
   int *bad = dalloc<int>(1);
   h2d(ctx->stream, emap, elem_dofs, sizeof(int32_t) * ne * nd);
   TFEM_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
   uint32_t *gmap = dalloc<uint32_t>(nd * ne_pad);
   TFEM_CUDA(cudaMemsetAsync(gmap, 0, sizeof(uint32_t) * nd * ne_pad, ctx->stream));
   const Layout L{elem_major_layout(dim, p), nd, ne, ne_pad};
   transpose_in_kernel<<<blocks_for(ne * nd), kThreads, 0, ctx->stream>>>(emap, L, ndofs, gmap,
                                                                         bad);
   ctx->launched();
   int hbad = 0;
   d2h(ctx->stream, &hbad, bad, sizeof(int));
   cudaFree(emap);
   cudaFree(bad);
   if (hbad) {
      cudaFree(gmap);
      invalid("restriction: element DOF index out of range");
   }
   return restriction_from_map(ctx, dim, p, ne, ndofs, elem_major_layout(dim, p), gmap, ElemOrder{});
}

void restriction_destroy(tfem_restriction *r)
{
   if (!r) return;
   cudaFree(r->gmap);
   cudaFree(r->evperm);
   for (int b = 0; b < r->n_buckets; b++) {
      cudaFree(r->buckets[b].dofs);
      cudaFree(r->buckets[b].slots);
   }
   for (int b = 0; b < r->n_gbuckets; b++) {
      cudaFree(r->gbuckets[b].dofs);
      cudaFree(r->gbuckets[b].slots);
   }
   cudaFree(r->evec);
   delete r;
}

void restriction_elem_dofs(const tfem_restriction *r, int32_t *host)
{
   std::vector<uint32_t> g(static_cast<size_t>(r->nd) * r->ne_pad);
   d2h(r->ctx->stream, g.data(), r->gmap, sizeof(uint32_t) * g.size());
   const Layout L{r->elem_major, r->nd, r->ne, r->ne_pad, r->order};
   for (int64_t e = 0; e < r->ne; e++)
      for (int i = 0; i < r->nd; i++)
         host[e * r->nd + i] = static_cast<int32_t>(g[L.slot_e(i, e)] & kDofMask);
}

int64_t restriction_boundary_dofs(const tfem_restriction *r, int32_t *host)
{
   if (!r->cartesian) invalid("restriction_boundary_dofs: needs a Cartesian restriction");
   tfem_ctx *ctx = r->ctx;
   int32_t *mark = dalloc<int32_t>(r->ndofs);
   TFEM_CUDA(cudaMemsetAsync(mark, 0, sizeof(int32_t) * r->ndofs, ctx->stream));
   const Layout L{r->elem_major, r->nd, r->ne, r->ne_pad, r->order};
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
   const Layout L{r->elem_major, r->nd, r->ne, r->ne_pad, r->order};
   gather_kernel<<<blocks_for(r->ne * r->nd), kThreads, 0, ctx->stream>>>(r->gmap, L, l, e);
   ctx->launched();
   TFEM_CUDA(cudaGetLastError());
}

void restriction_assign_last(tfem_ctx *ctx, const tfem_restriction *r, const double *e,
                             double *l)
{
   const int64_t nslots = r->ne * r->nd;
   const Layout L{r->elem_major, r->nd, r->ne, r->ne_pad, r->order};
   assign_exclusive_kernel<<<blocks_for(nslots), kThreads, 0, ctx->stream>>>(r->gmap, L, e, l);
   ctx->launched();
   if (r->n_shared > 0) {
      double *ev = const_cast<tfem_restriction *>(r)->ensure_evec();
      to_internal_kernel<<<blocks_for(nslots), kThreads, 0, ctx->stream>>>(L, r->evperm, e, ev);
      ctx->launched();
      for (int b = 0; b < r->n_buckets; b++) {
         const auto &bk = r->buckets[b];
         assign_last_kernel<<<blocks_for(bk.n), kThreads, 0, ctx->stream>>>(bk.dofs, bk.slots,
                                                                          bk.n, bk.c, ev, l);
         ctx->launched();
      }
   }
   TFEM_CUDA(cudaGetLastError());
}

} // namespace tfem

double *tfem_restriction::ensure_evec()
{
   if (!evec) TFEM_CUDA(cudaMalloc(&evec, sizeof(double) * static_cast<size_t>(nd) * ne_pad));
   return evec;
}