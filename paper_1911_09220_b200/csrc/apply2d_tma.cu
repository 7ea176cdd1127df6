// K2, 2D p <= 3: a thread-per-element sum factorisation (every stage in
// registers) fed by an asynchronous bulk-copy pipeline (sm_90+
// cp.async.bulk + mbarrier; SASS UBLKCP, LDGSTS).
//
// Warp-specialised persistent kernel, one block per SM: kCompute computing
// warps (7 at p = 3, 11 at p = 2, 15 at p = 1: TileCfg) with one element per
// lane -- a tile is 32 kCompute consecutive element positions, that many
// 8 x 4 warp patches in ElemOrder -- and one producer warp.  A tile's
// qdata is streamed as Q "slices" (one per qy: the nc*Q planes (c, qy, qx),
// each a contiguous 1792 B run of the [(c*nqd+q)][ne_pad] layout) through a
// 4- or 5-deep ring of shared-memory stages, and the element map (D1^2 planes)
// through three buffers (the open tile's map is read again by its epilogue).
// The producer waits on a stage's "empty" mbarrier (one arrive per compute
// warp) before refilling it; compute warps wait on "full" and never on each
// other (no block barriers: with warps in lockstep every latency is exposed;
// see profiles/).  Each lane gathers the next tile's x into shared memory
// (LDGSTS) while it computes the current one.
//
// Epilogue per slot: exclusive DOFs go straight to y; warp-local DOFs
// (restriction.cu build_warp_local) are summed by the owner lane from its
// lower neighbours' slots, shuffled up 1 / 8 / 9 lanes, in ascending element
// order; the rest go to the E-vector for the scatter.  x . y (CG's p . q) is
// taken as the sum of element energies when the operator allows (EDOT).
//
// EXACT: the reference operation order, bit-identical to the CPU; otherwise
// fused multiply-adds and both gradient terms in one register block.
#include "async.cuh"
#include "kernels.cuh"

namespace tfem {

namespace {


// Compute warps per block: 7 at p = 3 (8 warps of 254 registers fill the
// register file); where ptxas needs fewer, more warps per SM (the register
// file is four 16K banks, one per scheduler): p = 2 eleven (168 registers,
// +5 % over 7), p = 1 fifteen (~120 registers, +12 %).
template <int P>
struct TileCfg {
   static constexpr int kCompute = P == 1 ? 15 : P == 2 ? 11 : 7;
   static constexpr int kTile = 32 * kCompute;        // elements per tile
   static constexpr int kBlock = 32 * (kCompute + 1); // + the producer warp
};

template <int P, int Q, int KIND, bool EXACT>
struct TileSmem {
   static constexpr int D1 = P + 1, ND = D1 * D1;
   static constexpr int NC = KIND == TFEM_MASS ? 1 : 3;
   static constexpr int SLICE = NC * Q; // planes per qy slice
   // p = 3 with FMA numerics: one x buffer (the next tile's x lands in the
   // open tile's columns once V is in registers) pays for a fifth slice
   // stage, +2.5 %; measured slower for p <= 2 and for the exact numerics.
   // Two map buffers instead of three cost 12-30 % (the prefetch then waits
   // for the next map).
   static constexpr bool kDeep = P == 3 && !EXACT;
   static constexpr int kStages = kDeep ? 5 : 4; // qdata slice ring
   static constexpr int kXb = kDeep ? 1 : 2;     // x buffers
   static constexpr int kMaps = 3; // the open tile's map stays until its epilogue
   double q[kStages][SLICE][TileCfg<P>::kTile];
   uint32_t gmap[kMaps][ND][TileCfg<P>::kTile];
   uint32_t gess[kMaps][TileCfg<P>::kTile];  // a.elem_ess words of the tile (when given)
   double xs[kXb][ND][TileCfg<P>::kTile];    // x of the open / next tile [i][lane]
   uint32_t essm[TileCfg<P>::kTile];         // per lane: slots whose DOF is essential (ess_out)
   uint64_t full[kStages];  // slice landed (tx count)
   uint64_t empty[kStages]; // slice consumed (TileCfg<P>::kCompute arrivals)
   uint64_t gfull[kMaps], gempty[kMaps];
   uint64_t xfull[kXb];     // a tile's gathers landed (TileCfg<P>::kTile lane arrivals)
};

// Issue qdata slice `k` of this block (tile lt = k / Q, qy = k % Q).
template <int P, int Q, int KIND, bool EXACT>
__device__ __forceinline__ void issue_slice(TileSmem<P, Q, KIND, EXACT> &sm, const ApplyArgs &a,
                                            int64_t ntiles, int64_t k)
{
   constexpr int NQD = Q * Q, SLICE = TileSmem<P, Q, KIND, EXACT>::SLICE;
   const int64_t lt = k / Q;
   const int qy = static_cast<int>(k % Q);
   const int64_t t = blockIdx.x + lt * gridDim.x;
   if (t >= ntiles) return;
   const int64_t e0 = t * TileCfg<P>::kTile;
   // whole tile runs except the last tile (ne_pad: multiple of 64)
   const int64_t avail = a.ne_pad - e0;
   const unsigned bytes = static_cast<unsigned>(avail < TileCfg<P>::kTile ? avail : TileCfg<P>::kTile) * 8u;
   constexpr int kStages = TileSmem<P, Q, KIND, EXACT>::kStages;
   const int s = static_cast<int>(k % kStages);
   mbar_expect_tx(&sm.full[s], bytes * SLICE);
#pragma unroll
   for (int j = 0; j < SLICE; j++) {
      const int c = j / Q, qx = j % Q;
      const int64_t plane = c * NQD + qy * Q + qx;
      bulk_g2s(&sm.q[s][j][0], a.qdata + plane * a.ne_pad + e0, bytes, &sm.full[s]);
   }
}

template <int P, int Q, int KIND, bool EXACT>
__device__ __forceinline__ void issue_gmap(TileSmem<P, Q, KIND, EXACT> &sm, const ApplyArgs &a,
                                           int64_t ntiles, int64_t lt)
{
   constexpr int ND = (P + 1) * (P + 1);
   const int64_t t = blockIdx.x + lt * gridDim.x;
   if (t >= ntiles) return;
   const int64_t e0 = t * TileCfg<P>::kTile;
   const int64_t avail = a.ne_pad - e0;
   const unsigned bytes = static_cast<unsigned>(avail < TileCfg<P>::kTile ? avail : TileCfg<P>::kTile) * 4u;
   const int b = static_cast<int>(lt % TileSmem<P, Q, KIND, EXACT>::kMaps);
   const unsigned ebytes = a.elem_ess ? bytes : 0u; // elem_ess: ne_pad words
   mbar_expect_tx(&sm.gfull[b], bytes * ND + ebytes);
#pragma unroll
   for (int i = 0; i < ND; i++) bulk_g2s(&sm.gmap[b][i][0], a.gmap + i * a.ne_pad + e0, bytes, &sm.gfull[b]);
   if (ebytes) bulk_g2s(&sm.gess[b][0], a.elem_ess + e0, ebytes, &sm.gfull[b]);
}

// One qy slice of the diffusion chain for the calling thread's element:
// d = T B^t / T G^t at (qx, qy), w = D d, then S = G^t w / B^t w over qx and
// v += S B / S G (reference order; FIRST starts the v sums with a product).
template <int P, int Q, bool EXACT, bool FIRST, bool EN>
__device__ __forceinline__ void diffusion_slice(const ApplyArgs &a, int qy, const double (&T1)[Q][P + 1],
                                                const double (&T2)[Q][P + 1],
                                                const double (*qs)[TileCfg<P>::kTile], int tid,
                                                double (&vx)[P + 1][P + 1],
                                                double (&vy)[P + 1][P + 1], double &en, bool live)
{
   constexpr int D1 = P + 1;
   double wx[Q], wy[Q];
#pragma unroll
   for (int qx = 0; qx < Q; qx++) {
      double dx = mul<EXACT>(T1[qx][0], a.t.B[qy][0]);
      double dy = mul<EXACT>(T2[qx][0], a.t.G[qy][0]);
#pragma unroll
      for (int b = 1; b < D1; b++) {
         dx = mac<EXACT>(dx, T1[qx][b], a.t.B[qy][b]);
         dy = mac<EXACT>(dy, T2[qx][b], a.t.G[qy][b]);
      }
      const double d0 = qs[0 * Q + qx][tid], d1 = qs[1 * Q + qx][tid], d2 = qs[2 * Q + qx][tid];
      wx[qx] = add<EXACT>(mul<EXACT>(d0, dx), mul<EXACT>(d1, dy));
      wy[qx] = add<EXACT>(mul<EXACT>(d1, dx), mul<EXACT>(d2, dy));
      if (EN && live) en = mac<EXACT>(mac<EXACT>(en, dx, wx[qx]), dy, wy[qx]); // grad u . D grad u
   }
#pragma unroll
   for (int i = 0; i < D1; i++) {
      double sx = mul<EXACT>(a.t.G[0][i], wx[0]);
      double sy = mul<EXACT>(a.t.B[0][i], wy[0]);
#pragma unroll
      for (int qx = 1; qx < Q; qx++) {
         sx = mac<EXACT>(sx, a.t.G[qx][i], wx[qx]);
         sy = mac<EXACT>(sy, a.t.B[qx][i], wy[qx]);
      }
#pragma unroll
      for (int b = 0; b < D1; b++) {
         if (FIRST) {
            vx[i][b] = mul<EXACT>(sx, a.t.B[qy][b]);
            vy[i][b] = mul<EXACT>(sy, a.t.G[qy][b]);
         } else {
            vx[i][b] = mac<EXACT>(vx[i][b], sx, a.t.B[qy][b]);
            vy[i][b] = mac<EXACT>(vy[i][b], sy, a.t.G[qy][b]);
         }
      }
   }
}

// FMA numerics: both terms go straight into R (R += S_x B + S_y G).
template <int P, int Q, bool FIRST, bool EN>
__device__ __forceinline__ void diffusion_slice_fused(const ApplyArgs &a, int qy,
                                                      const double (&T1)[Q][P + 1],
                                                      const double (&T2)[Q][P + 1],
                                                      const double (*qs)[TileCfg<P>::kTile], int tid,
                                                      double (&R)[P + 1][P + 1], double &en, bool live)
{
   constexpr int D1 = P + 1;
   double wx[Q], wy[Q];
#pragma unroll
   for (int qx = 0; qx < Q; qx++) {
      double dx = T1[qx][0] * a.t.B[qy][0];
      double dy = T2[qx][0] * a.t.G[qy][0];
#pragma unroll
      for (int b = 1; b < D1; b++) {
         dx = fma(T1[qx][b], a.t.B[qy][b], dx);
         dy = fma(T2[qx][b], a.t.G[qy][b], dy);
      }
      const double d0 = qs[0 * Q + qx][tid], d1 = qs[1 * Q + qx][tid], d2 = qs[2 * Q + qx][tid];
      wx[qx] = fma(d0, dx, d1 * dy);
      wy[qx] = fma(d1, dx, d2 * dy);
      if (EN && live) en = fma(dy, wy[qx], fma(dx, wx[qx], en));
   }
#pragma unroll
   for (int i = 0; i < D1; i++) {
      double sx = a.t.G[0][i] * wx[0];
      double sy = a.t.B[0][i] * wy[0];
#pragma unroll
      for (int qx = 1; qx < Q; qx++) {
         sx = fma(a.t.G[qx][i], wx[qx], sx);
         sy = fma(a.t.B[qx][i], wy[qx], sy);
      }
#pragma unroll
      for (int b = 0; b < D1; b++)
         R[i][b] = FIRST ? fma(sx, a.t.B[qy][b], sy * a.t.G[qy][b])
                         : fma(sx, a.t.B[qy][b], fma(sy, a.t.G[qy][b], R[i][b]));
   }
}

template <int P, int Q, bool EXACT, bool FIRST, bool EN>
__device__ __forceinline__ void mass_slice(const ApplyArgs &a, int qy, const double (&T)[Q][P + 1],
                                           const double (*qs)[TileCfg<P>::kTile], int tid,
                                           double (&R)[P + 1][P + 1], double &en, bool live)
{
   constexpr int D1 = P + 1;
   double w[Q];
#pragma unroll
   for (int qx = 0; qx < Q; qx++) {
      double u = mul<EXACT>(T[qx][0], a.t.B[qy][0]);
#pragma unroll
      for (int b = 1; b < D1; b++) u = mac<EXACT>(u, T[qx][b], a.t.B[qy][b]);
      w[qx] = mul<EXACT>(u, qs[qx][tid]);
      if (EN && live) en = mac<EXACT>(en, u, w[qx]);
   }
#pragma unroll
   for (int i = 0; i < D1; i++) {
      double s = mul<EXACT>(a.t.B[0][i], w[0]);
#pragma unroll
      for (int qx = 1; qx < Q; qx++) s = mac<EXACT>(s, a.t.B[qx][i], w[qx]);
#pragma unroll
      for (int b = 0; b < D1; b++)
         R[i][b] = FIRST ? mul<EXACT>(s, a.t.B[qy][b]) : mac<EXACT>(R[i][b], s, a.t.B[qy][b]);
   }
}

// EDOT: x . y as the sum of element energies (a.energy_dot; apply.cu).
template <int P, int Q, int KIND, bool EXACT, bool EDOT>
__global__ void __launch_bounds__(TileCfg<P>::kBlock, 1) apply2d_tma_kernel(const ApplyArgs a)
{
   using Smem = TileSmem<P, Q, KIND, EXACT>;
   constexpr int D1 = P + 1, ND = D1 * D1;
   constexpr int kStages = Smem::kStages;
   if (a.done && *a.done) return;
   extern __shared__ __align__(128) unsigned char smem_raw[];
   auto &sm = *reinterpret_cast<Smem *>(smem_raw);
   const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
   const int tid = threadIdx.x; // element slot inside the tile (compute warps)
   const int64_t ntiles = (a.ne + TileCfg<P>::kTile - 1) / TileCfg<P>::kTile;
   const int64_t my_tiles =
      blockIdx.x < ntiles ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
   if (threadIdx.x == 0) {
      for (int s = 0; s < kStages; s++) {
         mbar_init(&sm.full[s], 1);
         mbar_init(&sm.empty[s], TileCfg<P>::kCompute);
      }
      for (int b = 0; b < Smem::kMaps; b++) {
         mbar_init(&sm.gfull[b], 1);
         mbar_init(&sm.gempty[b], TileCfg<P>::kCompute);
      }
      for (int b = 0; b < Smem::kXb; b++) mbar_init(&sm.xfull[b], TileCfg<P>::kTile);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
   }
   __syncthreads();
   auto tile_elem = [&](int64_t lt) { return (blockIdx.x + lt * gridDim.x) * TileCfg<P>::kTile + tid; };
   double dot = 0.0;
   if (warp == TileCfg<P>::kCompute) {
      // ---------------------------------------------------------- producer
      // map(lt + 1) goes out before tile lt's slices (exact numerics gather
      // the next tile's x during tile lt).
      if (lane == 0) {
         int64_t k = 0;
         if (my_tiles > 0) issue_gmap<P, Q, KIND, EXACT>(sm, a, ntiles, 0);
         for (int64_t lt = 0; lt < my_tiles; lt++) {
            const int64_t nt = lt + 1;
            if (nt < my_tiles) {
               if (nt >= Smem::kMaps)
                  mbar_wait(&sm.gempty[nt % Smem::kMaps], static_cast<unsigned>((nt / Smem::kMaps - 1) & 1));
               issue_gmap<P, Q, KIND, EXACT>(sm, a, ntiles, nt);
            }
            for (int qy = 0; qy < Q; qy++, k++) {
               const int s = static_cast<int>(k % kStages);
               if (k >= kStages)
                  mbar_wait(&sm.empty[s], static_cast<unsigned>((k / kStages - 1) & 1));
               issue_slice<P, Q, KIND, EXACT>(sm, a, ntiles, k);
            }
         }
      }
      __syncwarp();
   } else {
   // ---------------------------------------------------------- consumers
   int64_t k = 0; // slice counter
   auto acquire = [&]() -> const double(*)[TileCfg<P>::kTile] {
      const int s = static_cast<int>(k % kStages);
      mbar_wait(&sm.full[s], static_cast<unsigned>((k / kStages) & 1));
      return sm.q[s];
   };
   auto release = [&]() {
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[k % kStages]);
      k++;
   };
   if (my_tiles > 0) { // gather of the first tile
      mbar_wait(&sm.gfull[0], 0u);
      if (tile_elem(0) < a.ne) {
#pragma unroll
         for (int i = 0; i < ND; i++)
            gather8(&sm.xs[0][i][tid], a.x + (sm.gmap[0][i][tid] & kDofMask));
      }
      gather_arrive(&sm.xfull[0]);
   }
   const bool ess_is_mask = a.ess_out == a.mask_in;

   for (int64_t lt = 0; lt < my_tiles; lt++) {
      const int64_t e = tile_elem(lt);
      const bool live = e < a.ne;
      const int gb = static_cast<int>(lt % Smem::kMaps);
      // one buffer: a lane's V is in registers before it gathers the next
      // tile into the same columns, and no arrival for tile lt + 1 precedes
      // the completion of tile lt's phase
      const int xb = static_cast<int>(lt % Smem::kXb), xn = static_cast<int>((lt + 1) % Smem::kXb);
      double *xs = &sm.xs[xb][0][0];
      // x: gathered one tile ahead (or in the prologue).  The map is read
      // again by the epilogue (no registers held across the qy loop).
      mbar_wait(&sm.xfull[xb], static_cast<unsigned>((lt / Smem::kXb) & 1));
      uint32_t essm = 0; // slots whose DOF is essential (ess_out)
      double V[D1][D1];
      if (a.elem_ess) { // mask_in as one word per position
         const uint32_t mw = live ? sm.gess[gb][tid] : 0u;
#pragma unroll
         for (int i = 0; i < ND; i++) {
            const double v = live ? xs[i * TileCfg<P>::kTile + tid] : 0.0;
            V[i % D1][i / D1] = (mw >> i) & 1u ? 0.0 : v;
         }
         if (ess_is_mask) {
            essm = mw;
         } else if (a.ess_out) {
#pragma unroll
            for (int i = 0; i < ND; i++)
               essm |= static_cast<uint32_t>(live && bit_set(a.ess_out, sm.gmap[gb][i][tid] & kDofMask)) << i;
         }
      } else {
#pragma unroll
         for (int i = 0; i < ND; i++) {
            const uint32_t d = sm.gmap[gb][i][tid] & kDofMask;
            double v = live ? xs[i * TileCfg<P>::kTile + tid] : 0.0;
            const bool m = a.mask_in && live && bit_set(a.mask_in, d);
            const bool es = ess_is_mask ? m : live && a.ess_out && bit_set(a.ess_out, d);
            essm |= static_cast<uint32_t>(es) << i;
            if (m) v = 0.0;
            V[i % D1][i / D1] = v;
         }
      }
      sm.essm[tid] = essm;
      // Gather of the next tile (issued after the x contraction, when V is
      // dead, to keep register pressure down).
      auto prefetch_next = [&]() {
         if (lt + 1 >= my_tiles) return;
         const int nb = static_cast<int>((lt + 1) % Smem::kMaps);
         mbar_wait(&sm.gfull[nb], static_cast<unsigned>(((lt + 1) / Smem::kMaps) & 1));
         if (tile_elem(lt + 1) < a.ne) {
#pragma unroll 4
            for (int i = 0; i < ND; i++)
               gather8(&sm.xs[xn][i][tid], a.x + (sm.gmap[nb][i][tid] & kDofMask));
         }
         gather_arrive(&sm.xfull[xn]);
      };
      double R[D1][D1];
      // EDOT: the element energies go straight into dot (live lanes)
      double &en = dot;
      if (KIND == TFEM_DIFFUSION) {
         double T1[Q][D1], T2[Q][D1];
#pragma unroll
         for (int qx = 0; qx < Q; qx++)
#pragma unroll
            for (int b = 0; b < D1; b++) {
               double s1 = mul<EXACT>(a.t.G[qx][0], V[0][b]);
               double s2 = mul<EXACT>(a.t.B[qx][0], V[0][b]);
#pragma unroll
               for (int kk = 1; kk < D1; kk++) {
                  s1 = mac<EXACT>(s1, a.t.G[qx][kk], V[kk][b]);
                  s2 = mac<EXACT>(s2, a.t.B[qx][kk], V[kk][b]);
               }
               T1[qx][b] = s1;
               T2[qx][b] = s2;
            }
         prefetch_next();
         if constexpr (EXACT) {
            double vx[D1][D1], vy[D1][D1];
#pragma unroll
            for (int qy = 0; qy < Q; qy++) { // unrolled: table indices stay immediates
               if (qy == 0) diffusion_slice<P, Q, EXACT, true, EDOT>(a, qy, T1, T2, acquire(), tid, vx, vy, en, live);
               else diffusion_slice<P, Q, EXACT, false, EDOT>(a, qy, T1, T2, acquire(), tid, vx, vy, en, live);
               release();
            }
#pragma unroll
            for (int i = 0; i < D1; i++)
#pragma unroll
               for (int b = 0; b < D1; b++) R[i][b] = add<EXACT>(vx[i][b], vy[i][b]);
         } else {
#pragma unroll
            for (int qy = 0; qy < Q; qy++) {
               if (qy == 0) diffusion_slice_fused<P, Q, true, EDOT>(a, qy, T1, T2, acquire(), tid, R, en, live);
               else diffusion_slice_fused<P, Q, false, EDOT>(a, qy, T1, T2, acquire(), tid, R, en, live);
               release();
            }
         }
      } else {
         double T[Q][D1];
#pragma unroll
         for (int qx = 0; qx < Q; qx++)
#pragma unroll
            for (int b = 0; b < D1; b++) {
               double s = mul<EXACT>(a.t.B[qx][0], V[0][b]);
#pragma unroll
               for (int kk = 1; kk < D1; kk++) s = mac<EXACT>(s, a.t.B[qx][kk], V[kk][b]);
               T[qx][b] = s;
            }
         prefetch_next();
#pragma unroll
         for (int qy = 0; qy < Q; qy++) {
            if (qy == 0) mass_slice<P, Q, EXACT, true, EDOT>(a, qy, T, acquire(), tid, R, en, live);
            else mass_slice<P, Q, EXACT, false, EDOT>(a, qy, T, acquire(), tid, R, en, live);
            release();
         }
      }
      // Epilogue.  Warp-local DOFs: the owner lane adds its lower
      // neighbours' slots (shuffled up 1 / 8 / 9 lanes; restriction.cu
      // warp_partners) in ascending element order -- the scatter's sum
      // without the E-vector.  x . y and essential values come from xs.
      const int pc = lane & 7, pr = lane >> 3; // lane's cell in the warp patch
      constexpr int p = P;
      double u9 = 0.0, u8a = 0.0, u1a = 0.0, u1b = 0.0, u8b = 0.0;
      double u1m[P > 1 ? P - 1 : 1] = {}, u8m[P > 1 ? P - 1 : 1] = {};
      if (a.warp_local) { // warp-uniform
         u9 = __shfl_up_sync(0xffffffffu, R[p][p], 9);
         u8a = __shfl_up_sync(0xffffffffu, R[0][p], 8);
         u1a = __shfl_up_sync(0xffffffffu, R[p][0], 1);
         u1b = __shfl_up_sync(0xffffffffu, R[p][p], 1);
         u8b = __shfl_up_sync(0xffffffffu, R[p][p], 8);
#pragma unroll
         for (int m = 1; m < P; m++) {
            u1m[m - 1] = __shfl_up_sync(0xffffffffu, R[p][m], 1);
            u8m[m - 1] = __shfl_up_sync(0xffffffffu, R[m][p], 8);
         }
      }
      if (live) {
#pragma unroll
         for (int i = 0; i < ND; i++) {
            const int ia = i % D1, ib = i / D1;
            const uint32_t g = sm.gmap[gb][i][tid];
            const uint32_t d = g & kDofMask;
            const uint32_t fl = g & kFlagMask;
            double r = R[ia][ib];
            if (fl == kExclusive || (fl == kWarpOwner && a.warp_local)) {
               // contributions in ascending element order: y = v0 (or
               // y_old + v0), then + v1 ... (the scatter's order)
               const double yo = a.overwrite ? 0.0 : a.y[d];
               double acc = 0.0;
               bool st = false;
               auto push = [&](bool present, double x) {
                  if (!present) return;
                  acc = st ? add<EXACT>(acc, x) : (a.overwrite ? x : add<EXACT>(yo, x));
                  st = true;
               };
               if (fl == kWarpOwner) { // present lower neighbours (warp_partners)
                  if (ia == 0 && ib == 0) {
                     push(pc >= 1 && pr >= 1, u9);
                     push(pr >= 1, u8a);
                     push(pc >= 1, u1a);
                  } else if (ia == 0 && ib == p) {
                     push(pc >= 1, u1b);
                  } else if (ia == p && ib == 0) {
                     push(pr >= 1, u8b);
                  } else if (ia == 0) {
                     push(pc >= 1, u1m[ib > 0 ? ib - 1 : 0]);
                  } else if (ib == 0) {
                     push(pr >= 1, u8m[ia > 0 ? ia - 1 : 0]);
                  }
               }
               push(true, r);
               r = acc;
               const bool es = (sm.essm[tid] >> i) & 1u;
               if (EDOT) {
                  // energy of the masked x, plus x_d^2 where y_d = x_d
                  if (es) {
                     r = __ldg(a.x + d);
                     dot = mac<EXACT>(dot, r, r);
                  }
               } else if (es || a.dot) {
                  const double xd = __ldg(a.x + d);
                  if (es) r = xd;
                  if (a.dot && !(a.notown && bit_set(a.notown, d))) dot = mac<EXACT>(dot, xd, r);
               }
               a.y[d] = r;
            } else if (fl == kWarpMember && a.warp_local) {
               // summed by the owner lane
            } else {
               a.evec[i * a.ne_pad + e] = r;
            }
         }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.gempty[gb]); // map buffer free again
   }
   } // consumers
   if (a.dot) {
      const double v[1] = {dot};
      emit<TileCfg<P>::kBlock, 1>(a.dot, v);
   }
}

// grid: min(tiles, persistent blocks) -- elem_blocks (apply.cu)
template <int P, int Q, int KIND, bool EXACT>
void launch(const ApplyArgs &a, cudaStream_t s, unsigned grid)
{
   const size_t smem = sizeof(TileSmem<P, Q, KIND, EXACT>);
   static_assert(sizeof(TileSmem<P, Q, KIND, EXACT>) <= 227 * 1024, "shared memory budget");
   if (a.energy_dot) {
      max_dynamic_smem((const void *)apply2d_tma_kernel<P, Q, KIND, EXACT, true>, smem);
      apply2d_tma_kernel<P, Q, KIND, EXACT, true><<<grid, TileCfg<P>::kBlock, smem, s>>>(a);
   } else {
      max_dynamic_smem((const void *)apply2d_tma_kernel<P, Q, KIND, EXACT, false>, smem);
      apply2d_tma_kernel<P, Q, KIND, EXACT, false><<<grid, TileCfg<P>::kBlock, smem, s>>>(a);
   }
}

template <int P, int KIND>
Launch pick_q(int nq, bool exact)
{
   if (nq == P + 2) return exact ? launch<P, P + 2, KIND, true> : launch<P, P + 2, KIND, false>;
   if (nq == P + 1) return exact ? launch<P, P + 1, KIND, true> : launch<P, P + 1, KIND, false>;
   return nullptr;
}

template <int KIND>
Launch pick_p(int p, int nq, bool exact)
{
   switch (p) {
   case 1: return pick_q<1, KIND>(nq, exact);
   case 2: return pick_q<2, KIND>(nq, exact);
   case 3: return pick_q<3, KIND>(nq, exact);
   }
   return nullptr;
}

} // namespace

// Grid: min(tiles, one block per SM) persistent blocks.
KernelPick pick_apply2d_tma(int p, int nq, int kind, bool exact, int sm_count)
{
   KernelPick k;
   k.launch = kind == TFEM_MASS ? pick_p<TFEM_MASS>(p, nq, exact)
                                : pick_p<TFEM_DIFFUSION>(p, nq, exact);
   k.elems_per_block = p == 1 ? TileCfg<1>::kTile : p == 2 ? TileCfg<2>::kTile : TileCfg<3>::kTile;
   k.threads = p == 1 ? TileCfg<1>::kBlock : p == 2 ? TileCfg<2>::kBlock : TileCfg<3>::kBlock;
   k.persistent_blocks = sm_count;
   k.warp_reduce = true;
   k.energy_dot = true;
   return k;
}

} // namespace tfem
