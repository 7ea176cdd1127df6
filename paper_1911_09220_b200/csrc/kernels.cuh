// Shared definitions of the element kernels (apply2d_tma.cu, apply2d_hi.cu,
// apply3d_tma.cu, apply_grp.cu, apply2d_reg.cu) and their dispatch (apply.cu).
#pragma once

#include "common.cuh"

namespace tfem {

struct Tables {
   double B[kMaxQ][kMaxP + 1];
   double G[kMaxQ][kMaxP + 1];
};

struct ApplyArgs {
   Tables t;
   int64_t ne, ne_pad;
   int nd;
   const uint32_t *gmap;
   const double *qdata;
   const double *x;
   double *y;
   double *evec;
   const uint16_t *evperm; // E-vector slot order of element-major 3D maps (or null)
   int overwrite;
   const uint32_t *mask_in;
   const uint32_t *ess_out;
   const uint32_t *elem_ess; // optional: mask_in as a per-position slot word
   const uint32_t *notown; // DOFs owned by another rank: left out of the dot
   int warp_local;  // sum kWarpOwner/kWarpMember DOFs in-warp (else E-vector)
   int energy_dot;  // x . y = sum of element energies of the masked x + sum_ess x^2
                    // (single integrator, mask_in == ess_out, no notown; the
                    // scatter then adds only its essential DOFs' x^2)
   DotSink dot;     // fused x . y partials (CG's p . q)
   const int *done; // CG stop flag: skip the work once the solve has ended
};

using Launch = void (*)(const ApplyArgs &, cudaStream_t, unsigned);

struct KernelPick {
   Launch launch = nullptr;
   int elems_per_block = 1;
   int threads = 128;
   int persistent_blocks = 0; // > 0: grid = min(ceil(ne / elems_per_block), this)
   bool warp_reduce = false;  // can sum warp-local DOFs itself (ordered spaces)
   bool energy_dot = false;   // can take x . y as element energies
};

constexpr int kElemThreads2D = 128;

// The same arithmetic fed by a cp.async.bulk / mbarrier qdata pipeline
// (persistent blocks): 2D, p <= 3.
KernelPick pick_apply2d_tma(int p, int nq, int kind, bool exact, int sm_count);
// One element per warp with a bulk-copy qdata pipeline: 2D p >= 4.
KernelPick pick_apply2d_hi(int p, int nq, int kind, bool exact, int sm_count, bool colloc);
// One element per warp with a bulk-copy qdata pipeline: 3D, q^2 <= 32.
// colloc: B1d is exactly the identity (q = p+1 Gauss-Lobatto on the nodes).
KernelPick pick_apply3d_tma(int p, int nq, int kind, int sm_count, bool colloc);
// Thread-group-per-element kernels through shared memory: 2D p >= 4, 3D.
KernelPick pick_apply_grp(int dim, int p, int nq, int kind, bool exact);

constexpr __host__ __device__ int round32(int v) { return ((v + 31) / 32) * 32; }

// Elements per block of the group kernels so a block has ~256 threads.
constexpr __host__ __device__ int groups_for(int nt) { return nt >= 256 ? 1 : 256 / nt; }

} // namespace tfem
