// K2, 3D with Q^2 <= 32 (BP1 / BP3 p <= 3, BP5 p <= 4): one element per
// warp, fed by a bulk-copy pipeline (cp.async.bulk + mbarrier, LDGSTS).
//
// Persistent block per SM: warps 0..kW-1 compute, warp kW is the producer.
// Warp w of block b takes elements e = (b kW + w) + k (grid kW), k = 0, 1, ..
// The producer streams each element's qdata -- contiguous nc q^3 doubles of
// the element-major [e][c][q] layout -- into the warp's own 2-slot ring
// (full / empty mbarriers per slot), so warps never wait on each other; a
// warp's intermediates live in its private shared memory (__syncwarp only).
// Each lane gathers the next element's x with LDGSTS while the warp
// contracts the current one.
//
// Per element (fused multiply-adds; 3D has no reference bits to match, same
// order as apply_grp.cu): x contracted into [c][b][qx], then one lane per
// (qx, qy) column contracts b, walks qz through the point factors and back,
// then qy and qx are contracted back into the D1^3 outputs.  Epilogue:
// exclusive DOFs to y, the rest to the E-vector (scatter).  EDOT: x . y as
// element energies (apply.cu).
#include "async.cuh"
#include "kernels.cuh"

namespace tfem {

namespace {

template <int P, int Q, int KIND>
struct alignas(16) Warp3 {
   static constexpr int D1 = P + 1, ND = D1 * D1 * D1, NQD = Q * Q * Q;
   static constexpr int NC = KIND == TFEM_MASS ? 1 : 6;
   static constexpr int kSlots = 2;
   double q[kSlots][NC * NQD];            // the element's point factors
   double V[2][ND];                       // x of the open / next element
   double TB[D1 * D1 * Q], TG[D1 * D1 * Q]; // [c][b][qx]
   double Px[D1 * Q * Q], Py[D1 * Q * Q], Pz[D1 * Q * Q]; // [c][qy][qx]
   uint64_t full[kSlots], empty[kSlots];
};

template <int P, int Q, int KIND>
struct Cfg3 {
   static constexpr size_t kWarpBytes = sizeof(Warp3<P, Q, KIND>);
   static constexpr int kW0 = static_cast<int>((200 * 1024) / kWarpBytes);
   static constexpr int kW = kW0 > 11 ? 11 : (kW0 < 1 ? 1 : kW0); // compute warps
   static constexpr int kBlock = 32 * (kW + 1);
   static constexpr size_t kSmem = kWarpBytes * kW;
};

template <int P, int Q, int KIND, bool EDOT>
__global__ void __launch_bounds__(Cfg3<P, Q, KIND>::kBlock, 1) apply3d_tma_kernel(const ApplyArgs a)
{
   using W = Warp3<P, Q, KIND>;
   constexpr int D1 = W::D1, ND = W::ND, NQD = W::NQD, NC = W::NC;
   constexpr int kW = Cfg3<P, Q, KIND>::kW, kBlock = Cfg3<P, Q, KIND>::kBlock;
   constexpr int kSlots = W::kSlots;
   constexpr int GPL = (ND + 31) / 32; // map entries per lane
   constexpr unsigned kQBytes = NC * NQD * 8;
   if (a.done && *a.done) return;
   extern __shared__ __align__(128) unsigned char smem_raw[];
   __shared__ double sB[Q][D1], sG[Q][D1];
   for (int j = threadIdx.x; j < Q * D1; j += blockDim.x) {
      sB[j / D1][j % D1] = a.t.B[j / D1][j % D1];
      sG[j / D1][j % D1] = a.t.G[j / D1][j % D1];
   }
   const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
   auto *ws = reinterpret_cast<W *>(smem_raw);
   if (threadIdx.x == 0) {
      for (int w = 0; w < kW; w++)
         for (int s = 0; s < kSlots; s++) {
            mbar_init(&ws[w].full[s], 1);
            mbar_init(&ws[w].empty[s], 1);
         }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
   }
   __syncthreads();
   const int64_t stride = (int64_t)gridDim.x * kW;
   auto elem = [&](int w, int64_t k) { return (int64_t)blockIdx.x * kW + w + k * stride; };
   double dot = 0.0;
   if (warp == kW) {
      // ---------------------------------------------------------- producer
      if (lane == 0) {
         for (int64_t k = 0;; k++) {
            bool any = false;
            for (int w = 0; w < kW; w++) {
               const int64_t e = elem(w, k);
               if (e >= a.ne) continue;
               any = true;
               const int s = static_cast<int>(k % kSlots);
               if (k >= kSlots)
                  mbar_wait(&ws[w].empty[s], static_cast<unsigned>((k / kSlots - 1) & 1));
               mbar_expect_tx(&ws[w].full[s], kQBytes);
               bulk_g2s(ws[w].q[s], a.qdata + e * (int64_t)(NC * NQD), kQBytes, &ws[w].full[s]);
            }
            if (!any) break;
         }
      }
      __syncwarp();
   } else {
      // ---------------------------------------------------------- consumer
      W &sm = ws[warp];
      const int qx = lane % Q, qy = lane / Q;
      uint32_t gcur[GPL], gnext[GPL];
      auto load_map = [&](int64_t e, uint32_t (&g)[GPL]) {
#pragma unroll
         for (int m = 0; m < GPL; m++) {
            const int i = lane + 32 * m;
            g[m] = (e < a.ne && i < ND) ? __ldg(a.gmap + e * ND + i) : 0u;
         }
      };
      auto prefetch_x = [&](int64_t e, const uint32_t (&g)[GPL], int buf) {
         if (e >= a.ne) return;
#pragma unroll
         for (int m = 0; m < GPL; m++) {
            const int i = lane + 32 * m;
            if (i < ND) gather8(&sm.V[buf][i], a.x + (g[m] & kDofMask));
         }
         cp_async_commit();
      };
      load_map(elem(warp, 0), gcur);
      prefetch_x(elem(warp, 0), gcur, 0);
      for (int64_t k = 0;; k++) {
         const int64_t e = elem(warp, k);
         if (e >= a.ne) break;
         const int vb = static_cast<int>(k & 1);
         cp_async_wait_all();
         // essential DOFs read as zero (masked gather)
         if (a.mask_in) {
#pragma unroll
            for (int m = 0; m < GPL; m++) {
               const int i = lane + 32 * m;
               if (i < ND && bit_set(a.mask_in, gcur[m] & kDofMask)) sm.V[vb][i] = 0.0;
            }
         }
         __syncwarp();
         const int64_t en = elem(warp, k + 1);
         load_map(en, gnext);
         const double *V = sm.V[vb];
         // contract a -> TB / TG [c][b][qx]
         for (int j = lane; j < D1 * D1 * Q; j += 32) {
            const int jx = j % Q, cb = j / Q;
            double sb = 0.0, sg = 0.0;
#pragma unroll
            for (int kk = 0; kk < D1; kk++) {
               const double v = V[cb * D1 + kk];
               sb = fma(sB[jx][kk], v, sb);
               if (KIND == TFEM_DIFFUSION) sg = fma(sG[jx][kk], v, sg);
            }
            sm.TB[j] = sb;
            sm.TG[j] = sg;
         }
         prefetch_x(en, gnext, vb ^ 1); // the other buffer is free
         __syncwarp();
         const int s = static_cast<int>(k % kSlots);
         mbar_wait(&sm.full[s], static_cast<unsigned>((k / kSlots) & 1));
         if (lane < Q * Q) {
            double UBB[D1], UBG[D1], UGB[D1];
#pragma unroll
            for (int c = 0; c < D1; c++) { // contract b
               double bb = 0.0, bg = 0.0, gb = 0.0;
#pragma unroll
               for (int b = 0; b < D1; b++) {
                  const double tb = sm.TB[(c * D1 + b) * Q + qx];
                  bb = fma(sB[qy][b], tb, bb);
                  if (KIND == TFEM_DIFFUSION) {
                     const double tg = sm.TG[(c * D1 + b) * Q + qx];
                     bg = fma(sG[qy][b], tb, bg);
                     gb = fma(sB[qy][b], tg, gb);
                  }
               }
               UBB[c] = bb;
               UBG[c] = bg;
               UGB[c] = gb;
            }
            double Px[D1], Py[D1], Pz[D1];
#pragma unroll
            for (int c = 0; c < D1; c++) Px[c] = Py[c] = Pz[c] = 0.0;
            const double *qd = sm.q[s];
#pragma unroll
            for (int qz = 0; qz < Q; qz++) { // contract c, point factors, back over qz
               const int q = qx + Q * (qy + Q * qz);
               if (KIND == TFEM_MASS) {
                  // (qz, c) are compile-time here: table operands come from
                  // the constant bank, not shared memory
                  double u = 0.0;
#pragma unroll
                  for (int c = 0; c < D1; c++) u = fma(a.t.B[qz][c], UBB[c], u);
                  const double w = u * qd[q];
                  if (EDOT) dot = fma(u, w, dot);
#pragma unroll
                  for (int c = 0; c < D1; c++) Px[c] = fma(a.t.B[qz][c], w, Px[c]);
               } else {
                  double ux = 0.0, uy = 0.0, uz = 0.0;
#pragma unroll
                  for (int c = 0; c < D1; c++) {
                     ux = fma(a.t.B[qz][c], UGB[c], ux);
                     uy = fma(a.t.B[qz][c], UBG[c], uy);
                     uz = fma(a.t.G[qz][c], UBB[c], uz);
                  }
                  const double D00 = qd[q], D01 = qd[NQD + q], D02 = qd[2 * NQD + q];
                  const double D11 = qd[3 * NQD + q], D12 = qd[4 * NQD + q], D22 = qd[5 * NQD + q];
                  const double wx = fma(D02, uz, fma(D01, uy, D00 * ux));
                  const double wy = fma(D12, uz, fma(D11, uy, D01 * ux));
                  const double wz = fma(D22, uz, fma(D12, uy, D02 * ux));
                  if (EDOT) dot = fma(uz, wz, fma(uy, wy, fma(ux, wx, dot)));
#pragma unroll
                  for (int c = 0; c < D1; c++) {
                     Px[c] = fma(a.t.B[qz][c], wx, Px[c]);
                     Py[c] = fma(a.t.B[qz][c], wy, Py[c]);
                     Pz[c] = fma(a.t.G[qz][c], wz, Pz[c]);
                  }
               }
            }
#pragma unroll
            for (int c = 0; c < D1; c++) {
               sm.Px[(c * Q + qy) * Q + qx] = Px[c];
               if (KIND == TFEM_DIFFUSION) {
                  sm.Py[(c * Q + qy) * Q + qx] = Py[c];
                  sm.Pz[(c * Q + qy) * Q + qx] = Pz[c];
               }
            }
         }
         __syncwarp();
         if (lane == 0) mbar_arrive(&sm.empty[s]); // point factors consumed
         // contract qy -> [c][b][qx] (x-gradient part in TB, y + z in TG)
         for (int j = lane; j < D1 * D1 * Q; j += 32) {
            const int jx = j % Q, cb = j / Q, b = cb % D1, c = cb / D1;
            double sx = 0.0, syz = 0.0;
#pragma unroll
            for (int y = 0; y < Q; y++) {
               const int o = (c * Q + y) * Q + jx;
               sx = fma(sB[y][b], sm.Px[o], sx);
               if (KIND == TFEM_DIFFUSION) {
                  syz = fma(sG[y][b], sm.Py[o], syz);
                  syz = fma(sB[y][b], sm.Pz[o], syz);
               }
            }
            sm.TB[j] = sx;
            sm.TG[j] = syz;
         }
         __syncwarp();
         // contract qx -> r(a, b, c) and the epilogue
#pragma unroll
         for (int m = 0; m < GPL; m++) {
            const int i = lane + 32 * m;
            if (i >= ND) continue;
            const int ia = i % D1, cb = i / D1;
            double r = 0.0;
#pragma unroll
            for (int x = 0; x < Q; x++) {
               if (KIND == TFEM_MASS) {
                  r = fma(sB[x][ia], sm.TB[cb * Q + x], r);
               } else {
                  r = fma(sG[x][ia], sm.TB[cb * Q + x], r);
                  r = fma(sB[x][ia], sm.TG[cb * Q + x], r);
               }
            }
            const uint32_t gg = gcur[m];
            if (is_exclusive(gg)) {
               const uint32_t d = gg & kDofMask;
               if (!a.overwrite) r += a.y[d];
               const bool es = a.ess_out && bit_set(a.ess_out, d);
               if (es) r = __ldg(a.x + d);
               a.y[d] = r;
               if (EDOT) {
                  if (es) dot = fma(r, r, dot);
               } else if (a.dot && !(a.notown && bit_set(a.notown, d))) {
                  dot = fma(__ldg(a.x + d), r, dot);
               }
            } else {
               a.evec[e * ND + i] = r;
            }
         }
         __syncwarp(); // TB / TG / P reused by the next element
#pragma unroll
         for (int m = 0; m < GPL; m++) gcur[m] = gnext[m];
      }
   }
   if (a.dot) {
      const double v[1] = {dot};
      emit<kBlock, 1>(a.dot, v);
   }
}

int g_sm3 = 0;

template <int P, int Q, int KIND>
void launch(const ApplyArgs &a, cudaStream_t s, unsigned /*blocks*/)
{
   using C = Cfg3<P, Q, KIND>;
   static_assert(C::kSmem <= 227 * 1024, "shared memory budget");
   static const bool once = [] {
      cudaFuncSetAttribute(apply3d_tma_kernel<P, Q, KIND, false>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem);
      cudaFuncSetAttribute(apply3d_tma_kernel<P, Q, KIND, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem);
      return true;
   }();
   (void)once;
   const int64_t nblk = (a.ne + C::kW - 1) / C::kW;
   const unsigned grid = static_cast<unsigned>(nblk < g_sm3 ? nblk : g_sm3);
   if (a.energy_dot)
      apply3d_tma_kernel<P, Q, KIND, true><<<grid, C::kBlock, C::kSmem, s>>>(a);
   else
      apply3d_tma_kernel<P, Q, KIND, false><<<grid, C::kBlock, C::kSmem, s>>>(a);
}

template <int P, int Q, int KIND>
KernelPick make()
{
   KernelPick k;
   // bulk copies need 16-byte sizes and element strides
   if constexpr ((Warp3<P, Q, KIND>::NC * Q * Q * Q) % 2 == 0) {
      k.launch = launch<P, Q, KIND>;
      k.elems_per_block = Cfg3<P, Q, KIND>::kW;
      k.threads = Cfg3<P, Q, KIND>::kBlock;
      k.persistent_blocks = g_sm3;
      k.energy_dot = true;
   }
   return k;
}

template <int KIND>
KernelPick pick_kind(int p, int nq)
{
   // Q^2 <= 32: one (qx, qy) column per lane
   switch (p) {
   case 1: return nq == 3 ? make<1, 3, KIND>() : nq == 2 ? make<1, 2, KIND>() : KernelPick{};
   case 2: return nq == 4 ? make<2, 4, KIND>() : nq == 3 ? make<2, 3, KIND>() : KernelPick{};
   case 3: return nq == 5 ? make<3, 5, KIND>() : nq == 4 ? make<3, 4, KIND>() : KernelPick{};
   case 4: return nq == 5 ? make<4, 5, KIND>() : KernelPick{};
   }
   return {};
}

} // namespace

KernelPick pick_apply3d_tma(int p, int nq, int kind, int sm_count)
{
   g_sm3 = sm_count;
   return kind == TFEM_MASS ? pick_kind<TFEM_MASS>(p, nq) : pick_kind<TFEM_DIFFUSION>(p, nq);
}

} // namespace tfem
