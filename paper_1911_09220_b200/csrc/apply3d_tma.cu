// K2, 3D with q <= 7 (BP1 / BP3 p <= 5, BP5 p <= 5): one group of
// EPW = max(1, 32 / Q^2) elements per warp (1 for Q >= 5, 2 for Q = 4, 3 for
// Q = 3; for Q^2 > 32 a lane walks several (qx, qy) columns), fed by a
// bulk-copy pipeline (cp.async.bulk + mbarrier, LDGSTS).
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

// Elements per warp: Q^2 <= 32 lanes per element in the column stage, so
// low orders pack several elements into one warp (p=1: 3, p=2: 2).
template <int Q>
constexpr int epw() { return 32 / (Q * Q) > 0 ? 32 / (Q * Q) : 1; }

// Row strides of TB / TG ([e][c][b][qx], row = Q + kPadT) and of the P
// planes ([e][c][qy][qx], plane = Q^2 + kPadP), padded against shared-memory
// bank conflicts of the row-wise stages (exhaustive search of the access
// patterns, 64-bit accesses in half-warp phases; measured slower at p = 5,
// q = 6, where the larger rows cost a warp of occupancy).
constexpr int pad_t3(int P, int Q)
{
   return (P == 2 && Q == 4) ? 3 : (P == 3 && Q == 4) ? 1 : (P == 4 && Q == 6) ? 1 : 0;
}
constexpr int pad_p3(int P, int Q)
{
   return (P == 2 && Q == 4) ? 4 : (P == 3 && Q == 4) ? 4 : (P == 4 && Q == 6) ? 2 : 0;
}

template <int P, int Q, int KIND>
struct alignas(16) Warp3 {
   static constexpr int D1 = P + 1, ND = D1 * D1 * D1, NQD = Q * Q * Q;
   static constexpr int NC = KIND == TFEM_MASS ? 1 : 6;
   static constexpr int EPW = epw<Q>();
   // q >= 8 (QG): the point factors are read from global memory in the
   // column stage (planes prefetched into registers) -- double-buffering
   // nc q^3 doubles per element in shared memory would leave too few warps
   // (and BP3 p = 5, q = 7: +15 % over the point-factor ring with three teams)
   static constexpr bool QG = Q >= 8 || (P == 5 && Q == 7 && KIND == TFEM_DIFFUSION);
   static constexpr int kSlots = QG ? 1 : 2;
   double q[kSlots][QG ? 1 : EPW * NC * NQD];         // the group's point factors
   // QG slab ring: each column thread's point factors of kSlab qz planes in
   // flight (cp.async, completion on sfull[slot]); thread-private entries
   // (q >= 9: +23 % at BP3 p = 7 over the register prefetch; at q = 8 the
   // register prefetch is 5 % faster with four teams, 8 % with six)
   static constexpr bool SLAB = QG && Q != 8;
   static constexpr int kSlab = SLAB ? 4 : 1;
   static constexpr int NTHq = 32 * ((Q * Q + 31) / 32 < 4 ? (Q * Q + 31) / 32 : 4);
   double slab[SLAB ? kSlab * NC * NTHq : 1]; // [slot][c][thread]
   uint64_t sfull[kSlab];
   double V[2][EPW * ND];                             // x of the open / next group
   static constexpr int kSt = Q + pad_t3(P, Q), kSp = Q * Q + pad_p3(P, Q); // padded strides
   static constexpr int kEt = D1 * D1 * kSt, kEp = D1 * kSp;                   // per element
   double TB[EPW * kEt], TG[EPW * kEt];                  // [e][c][b][qx]
   double Px[EPW * kEp], Py[EPW * kEp], Pz[EPW * kEp];   // [e][c][qy][qx]
   uint64_t full[kSlots], empty[kSlots];
   uint32_t gm[EPW * ND]; // the open group's map entries and essential flags
   uint8_t es[EPW * ND];  // (read by the epilogue)
};

template <int P, int Q, int KIND>
struct Cfg3 {
   // warps per element: two when neither the (p+1)^2 rows nor the q^2
   // columns fit one warp (p = 5, q = 6, 7): every stage is then one pass of
   // 64 threads, and a team's shared memory -- dominated by the element's
   // double-buffered point factors -- feeds twice the warps.  Measured (10M
   // DOFs): BP3 p=5 +17 %, BP5 p=5 +64 %; at p = 4, q = 6 (25 rows) one
   // warp per element stays faster (-7 % with teams: idle threads).
   // QG: one column per thread, ceil(q^2 / 32) warps per element (<= 4).
   static constexpr bool QG = Warp3<P, Q, KIND>::QG;
   static constexpr int WPE = QG ? ((Q * Q + 31) / 32 < 4 ? (Q * Q + 31) / 32 : 4)
                                 : (P + 1) * (P + 1) > 32 && Q * Q > 32 ? 2 : 1;
   static constexpr size_t kWarpBytes = sizeof(Warp3<P, Q, KIND>);
   // computing warps as shared memory allows: 224 KB (vs 200) is +9 % at
   // p = 4 (6 -> 7 warps), neutral where the 11-warp cap or the warp size binds
   static constexpr int kT0 = static_cast<int>((224 * 1024) / kWarpBytes); // teams by smem
   // Warps per block: 11 by default, 15 at p <= 2 with q <= p + 2 except
   // p = 2, q = 4, 13 at p = 3, q = 5 (what ptxas needs fits there).
   // Measured, ~10M DOFs (the register file is four 16K
   // banks, one per scheduler: 9-12 warps per block cap a thread at 168
   // registers, <= 8 warps at 255):
   //   QG q = 8 (BP3 p = 6, BP5 p = 7): four two-warp teams, 254 registers
   //     (p = 6: +14 % over the group kernel; 12 warps -7 %);
   //   QG BP3 p = 7: four three-warp teams (168 registers; two teams -12 %);
   //   QG BP3 p = 8: two four-warp teams (+2 % over three);
   //   QG BP5 p = 8: two three-warp teams (no spills, +29 % over three);
   //   QG BP3 p = 5 (q = 7): six two-warp teams, slab ring;
   //   BP5 p = 6, q = 7: three teams + producer (7 warps, no spills; +17 %
   //     over four teams with spills);
   //   BP5 p = 5: five teams (three: -16 %).
   static constexpr int kMaxW = QG ? (P == 8 && Q == 10 ? 8 : P == 8 && Q == 9 ? 6 : Q == 8 ? 8 : 12)
                              : (P == 6 && Q == 7 && KIND == TFEM_DIFFUSION) ? 6
                              : KIND != TFEM_DIFFUSION ? 11
                              : (Q <= 3) ? 15 : (P == 3 && Q == 5) ? 13 : 11;
   static constexpr int kT1 = kT0 * WPE > kMaxW ? kMaxW / WPE : kT0;
   static constexpr int kT = kT1 < 1 ? 1 : kT1;   // teams (elements in flight)
   static constexpr int kW = kT * WPE;            // compute warps
   static constexpr int kBlock = 32 * (kW + (QG ? 0 : 1)); // + the producer warp
   static constexpr size_t kSmem = kWarpBytes * kT;
};

// CO (collocated, BP5): q = p + 1 Gauss-Lobatto points on the Gauss-Lobatto
// nodes, so B1d = I exactly (quadrature.cpp:91-125, basis.cpp:53-58): every
// B contraction is a copy and is skipped -- half the FP64 work per element.
template <int P, int Q, int KIND, bool EDOT, bool CO>
__global__ void __launch_bounds__(Cfg3<P, Q, KIND>::kBlock, 1) apply3d_tma_kernel(const ApplyArgs a)
{
   static_assert(!CO || Q == P + 1, "collocation needs q = p + 1");
   using W = Warp3<P, Q, KIND>;
   constexpr int D1 = W::D1, ND = W::ND, NQD = W::NQD, NC = W::NC, EPW = W::EPW;
   constexpr int kW = Cfg3<P, Q, KIND>::kW, kBlock = Cfg3<P, Q, KIND>::kBlock;
   constexpr int kT = Cfg3<P, Q, KIND>::kT, WPE = Cfg3<P, Q, KIND>::WPE;
   constexpr int NTH = 32 * WPE;              // threads per team
   constexpr int kSlots = W::kSlots;
   constexpr int NT = D1 * D1 * Q;         // contraction outputs per element
   constexpr int kSt = W::kSt, kSp = W::kSp, kEt = W::kEt, kEp = W::kEp;
   constexpr int GPL = (EPW * ND + NTH - 1) / NTH; // map entries per thread
   // row-wise contractions (basis operands compile-time) when a team covers
   // the rows in one pass (or two at q <= 6 with one warp per element)
   constexpr int kRowMax = WPE > 1 ? NTH : (Q <= 6 ? 64 : 32);
   constexpr bool kRows1 = EPW * D1 * D1 <= kRowMax; // stages a and x
   constexpr bool kRows3 = EPW * Q * D1 <= kRowMax;  // stage y
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
      for (int w = 0; w < kT; w++) {
         for (int s = 0; s < kSlots; s++) {
            mbar_init(&ws[w].full[s], 1);
            mbar_init(&ws[w].empty[s], 1);
         }
         if constexpr (W::SLAB)
            for (int s = 0; s < W::kSlab; s++) mbar_init(&ws[w].sfull[s], Q * Q);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
   }
   __syncthreads();
   // team w of block b takes element groups g = (b kT + w) + k (grid kT);
   // group g is elements [g EPW, g EPW + EPW)
   const int64_t stride = (int64_t)gridDim.x * kT;
   auto group = [&](int w, int64_t k) { return (int64_t)blockIdx.x * kT + w + k * stride; };
   // a team: WPE warps on one element group; pt = thread in the team
   const int team = warp / WPE, pt = lane + 32 * (warp % WPE);
   auto team_sync = [&]() {
      if constexpr (WPE == 1) __syncwarp();
      else asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(NTH) : "memory");
   };
   auto count = [&](int64_t g) {
      const int64_t left = a.ne - g * EPW;
      return static_cast<int>(left < EPW ? (left > 0 ? left : 0) : EPW);
   };
   double dot = 0.0;
   if (!W::QG && warp == kW) {
      // ---------------------------------------------------------- producer
      if (lane == 0) {
         for (int64_t k = 0;; k++) {
            bool any = false;
            for (int w = 0; w < kT; w++) {
               const int64_t g = group(w, k);
               const int cnt = count(g);
               if (cnt == 0) continue;
               any = true;
               const int s = static_cast<int>(k % kSlots);
               if (k >= kSlots)
                  mbar_wait(&ws[w].empty[s], static_cast<unsigned>((k / kSlots - 1) & 1));
               mbar_expect_tx(&ws[w].full[s], kQBytes * cnt);
               bulk_g2s(ws[w].q[s], a.qdata + g * EPW * (int64_t)(NC * NQD), kQBytes * cnt,
                        &ws[w].full[s]);
            }
            if (!any) break;
         }
      }
      __syncwarp();
   } else {
      // ---------------------------------------------------------- consumer
      W &sm = ws[team];
      uint32_t gcur[GPL], gnext[GPL], gnn[GPL]; // map entries: this, next, next-but-one group
      uint32_t mcur[GPL], mnext[GPL]; // mask_in words of the map entries
      auto load_map = [&](int64_t g, uint32_t (&m_)[GPL]) {
         const int64_t lim = (int64_t)count(g) * ND;
#pragma unroll
         for (int m = 0; m < GPL; m++) {
            const int i = pt + NTH * m;
            m_[m] = i < lim ? __ldg(a.gmap + g * EPW * ND + i) : 0u;
         }
      };
      auto prefetch_x = [&](int64_t g, const uint32_t (&m_)[GPL], int buf) {
         const int64_t lim = (int64_t)count(g) * ND;
         if (lim == 0) return;
#pragma unroll
         for (int m = 0; m < GPL; m++) {
            const int i = pt + NTH * m;
            if (i < lim) gather8(&sm.V[buf][i], a.x + (m_[m] & kDofMask));
         }
         cp_async_commit();
      };
      // the mask words go out with the gather (tested a group later)
      auto load_mask = [&](int64_t g, const uint32_t (&m_)[GPL], uint32_t (&w_)[GPL]) {
         const int64_t lim = (int64_t)count(g) * ND;
#pragma unroll
         for (int m = 0; m < GPL; m++) {
            const int i = pt + NTH * m;
            w_[m] = a.mask_in && i < lim ? __ldg(a.mask_in + ((m_[m] & kDofMask) >> 5)) : 0u;
         }
      };
      load_map(group(team, 0), gcur);
      load_map(group(team, 1), gnext);
      prefetch_x(group(team, 0), gcur, 0);
      load_mask(group(team, 0), gcur, mcur);
      for (int64_t k = 0;; k++) {
         const int64_t g = group(team, k);
         const int cnt = count(g);
         if (cnt == 0) break;
         const int vb = static_cast<int>(k & 1);
         cp_async_wait_all();
         // essential DOFs read as zero (masked gather); map entries and
         // essential flags to shared memory for the epilogue
#pragma unroll
         for (int m = 0; m < GPL; m++) {
            const int i = pt + NTH * m;
            if (i >= cnt * ND) continue;
            const uint32_t d = gcur[m] & kDofMask;
            const bool mk = (mcur[m] >> (d & 31)) & 1u;
            if (mk) sm.V[vb][i] = 0.0;
            sm.gm[i] = gcur[m];
            sm.es[i] = (a.ess_out == a.mask_in ? mk : (a.ess_out && bit_set(a.ess_out, d))) ? 1 : 0;
         }
         team_sync();
         // SLAB: column thread pt's point factors of plane qz of this group go
         // to slot (k q + qz) % kSlab; the first kSlab - 1 planes now, so the
         // x stage below covers their latency
         auto slab_issue = [&](int qz) {
            if constexpr (W::SLAB) {
               const int64_t t = k * Q + qz;
               const int s = static_cast<int>(t % W::kSlab);
               double *dst = sm.slab + s * NC * W::NTHq + pt;
               const double *src = a.qdata + g * (int64_t)(NC * NQD) + pt + Q * Q * qz;
#pragma unroll
               for (int c = 0; c < NC; c++) gather8(dst + c * W::NTHq, src + c * NQD);
               gather_arrive(&sm.sfull[s]);
            }
         };
         if constexpr (W::SLAB) {
            if (pt < Q * Q)
#pragma unroll
               for (int qz = 0; qz < W::kSlab - 1; qz++) slab_issue(qz);
         }
         const int64_t gn = group(team, k + 1);
         load_map(group(team, k + 2), gnn); // two groups ahead: used a group later
         const double *V = sm.V[vb];
         // contract a -> TB / TG [e][c][b][qx]: a lane per (e, c, b) row, qx
         // unrolled (basis operands from the constant bank) when the rows
         // fit one pass of the warp; else a lane per output.  CO: TB = V,
         // only TG is formed.
         if constexpr (CO) {
            for (int it = pt; it < EPW * D1 * D1; it += NTH) {
               const int j = it / (D1 * D1), cb = it % (D1 * D1);
               double v[D1];
#pragma unroll
               for (int kk = 0; kk < D1; kk++) v[kk] = V[j * ND + cb * D1 + kk];
               double *TGo = sm.TG + j * kEt + cb * kSt;
#pragma unroll
               for (int jx = 0; jx < Q; jx++) {
                  double sg = 0.0;
#pragma unroll
                  for (int kk = 0; kk < D1; kk++) sg = fma(a.t.G[jx][kk], v[kk], sg);
                  TGo[jx] = sg;
               }
            }
         } else if constexpr (!kRows1) {
            for (int jj = pt; jj < EPW * NT; jj += NTH) {
               const int j = jj / NT, r = jj % NT, jx = r % Q, cb = r / Q;
               double sb = 0.0, sg = 0.0;
#pragma unroll
               for (int kk = 0; kk < D1; kk++) {
                  const double v = V[j * ND + cb * D1 + kk];
                  sb = fma(sB[jx][kk], v, sb);
                  if (KIND == TFEM_DIFFUSION) sg = fma(sG[jx][kk], v, sg);
               }
               sm.TB[j * kEt + cb * kSt + jx] = sb;
               sm.TG[j * kEt + cb * kSt + jx] = sg;
            }
         } else
         for (int it = pt; it < EPW * D1 * D1; it += NTH) {
            const int j = it / (D1 * D1), cb = it % (D1 * D1);
            double v[D1];
#pragma unroll
            for (int kk = 0; kk < D1; kk++) v[kk] = V[j * ND + cb * D1 + kk];
            double *TBo = sm.TB + j * kEt + cb * kSt, *TGo = sm.TG + j * kEt + cb * kSt;
#pragma unroll
            for (int jx = 0; jx < Q; jx++) {
               double sb = 0.0, sg = 0.0;
#pragma unroll
               for (int kk = 0; kk < D1; kk++) {
                  sb = fma(a.t.B[jx][kk], v[kk], sb);
                  if (KIND == TFEM_DIFFUSION) sg = fma(a.t.G[jx][kk], v[kk], sg);
               }
               TBo[jx] = sb;
               if (KIND == TFEM_DIFFUSION) TGo[jx] = sg;
            }
         }
         prefetch_x(gn, gnext, vb ^ 1); // the other buffer is free
         load_mask(gn, gnext, mnext);
         team_sync();
         const int s = static_cast<int>(k % kSlots);
         if constexpr (!W::QG) mbar_wait(&sm.full[s], static_cast<unsigned>((k / kSlots) & 1));
         // column stage: (element ej, qx, qy) columns over the lanes
         for (int cl = pt; cl < EPW * Q * Q; cl += NTH) {
            const int ej = cl / (Q * Q), col = cl % (Q * Q);
            const int qx = col % Q, qy = col / Q;
            const bool live = ej < cnt;
            const double *TB = sm.TB + ej * kEt, *TG = sm.TG + ej * kEt;
            // QG: the column's point factors, kR planes ahead of the qz walk
            // (the first ones issued before the b contraction)
            constexpr int kR = 3;
            double Dq[W::QG ? NC : 1][W::QG ? Q : 1];
            const double *qg = a.qdata + (g * EPW + (live ? ej : 0)) * (int64_t)(NC * NQD) + col;
            auto load_plane = [&](int qz) {
               if constexpr (W::QG && !W::SLAB) {
#pragma unroll
                  for (int c = 0; c < NC; c++) Dq[c][qz] = __ldg(qg + c * NQD + Q * Q * qz);
               }
            };
#pragma unroll
            for (int qz = 0; qz < kR && qz < Q; qz++) load_plane(qz);
            double UBB[D1], UBG[D1], UGB[D1];
            if constexpr (CO) {
               // UBB = V[c][qy][qx], UGB = TG[c][qy][qx], UBG = G_y V
               const double *Ve = V + ej * ND;
#pragma unroll
               for (int c = 0; c < D1; c++) {
                  UBB[c] = Ve[(c * D1 + qy) * D1 + qx];
                  if (KIND == TFEM_DIFFUSION) {
                     UGB[c] = TG[(c * D1 + qy) * kSt + qx];
                     double bg = 0.0;
#pragma unroll
                     for (int b = 0; b < D1; b++) bg = fma(sG[qy][b], Ve[(c * D1 + b) * D1 + qx], bg);
                     UBG[c] = bg;
                  }
               }
            } else
#pragma unroll
            for (int c = 0; c < D1; c++) { // contract b
               double bb = 0.0, bg = 0.0, gb = 0.0;
#pragma unroll
               for (int b = 0; b < D1; b++) {
                  const double tb = TB[(c * D1 + b) * kSt + qx];
                  bb = fma(sB[qy][b], tb, bb);
                  if (KIND == TFEM_DIFFUSION) {
                     const double tg = TG[(c * D1 + b) * kSt + qx];
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
            const double *qd = sm.q[s] + ej * NC * NQD;
            // point factor c at plane qz of this column
            auto D = [&](int c, int qz, int q) -> double {
               if constexpr (W::SLAB)
                  return sm.slab[((k * Q + qz) % W::kSlab) * NC * W::NTHq + c * W::NTHq + pt];
               else if constexpr (W::QG) return Dq[c][qz];
               else return qd[c * NQD + q];
            };
#pragma unroll
            for (int qz = 0; qz < Q; qz++) { // contract c, point factors, back over qz
               const int q = qx + Q * (qy + Q * qz);
               if constexpr (W::SLAB) {
                  if (qz + W::kSlab - 1 < Q) slab_issue(qz + W::kSlab - 1);
                  const int64_t t = k * Q + qz;
                  mbar_wait(&sm.sfull[t % W::kSlab], static_cast<unsigned>((t / W::kSlab) & 1));
               } else if (qz + kR < Q) {
                  load_plane(qz + kR);
               }
               // (qz, c) are compile-time here: table operands come from the
               // constant bank, not shared memory
               if (KIND == TFEM_MASS) {
                  double u = 0.0;
                  if constexpr (CO) {
                     u = UBB[qz];
                  } else {
#pragma unroll
                     for (int c = 0; c < D1; c++) u = fma(a.t.B[qz][c], UBB[c], u);
                  }
                  const double w = u * D(0, qz, q);
                  if (EDOT && live) dot = fma(u, w, dot);
                  if constexpr (CO) {
                     Px[qz] = w;
                  } else {
#pragma unroll
                     for (int c = 0; c < D1; c++) Px[c] = fma(a.t.B[qz][c], w, Px[c]);
                  }
               } else {
                  double ux = 0.0, uy = 0.0, uz = 0.0;
                  if constexpr (CO) {
                     ux = UGB[qz];
                     uy = UBG[qz];
#pragma unroll
                     for (int c = 0; c < D1; c++) uz = fma(a.t.G[qz][c], UBB[c], uz);
                  } else {
#pragma unroll
                     for (int c = 0; c < D1; c++) {
                        ux = fma(a.t.B[qz][c], UGB[c], ux);
                        uy = fma(a.t.B[qz][c], UBG[c], uy);
                        uz = fma(a.t.G[qz][c], UBB[c], uz);
                     }
                  }
                  const double D00 = D(0, qz, q), D01 = D(1, qz, q), D02 = D(2, qz, q);
                  const double D11 = D(3, qz, q), D12 = D(4, qz, q), D22 = D(5, qz, q);
                  const double wx = fma(D02, uz, fma(D01, uy, D00 * ux));
                  const double wy = fma(D12, uz, fma(D11, uy, D01 * ux));
                  const double wz = fma(D22, uz, fma(D12, uy, D02 * ux));
                  if (EDOT && live) dot = fma(uz, wz, fma(uy, wy, fma(ux, wx, dot)));
                  if constexpr (CO) {
                     Px[qz] = wx;
                     Py[qz] = wy;
#pragma unroll
                     for (int c = 0; c < D1; c++) Pz[c] = fma(a.t.G[qz][c], wz, Pz[c]);
                  } else {
#pragma unroll
                     for (int c = 0; c < D1; c++) {
                        Px[c] = fma(a.t.B[qz][c], wx, Px[c]);
                        Py[c] = fma(a.t.B[qz][c], wy, Py[c]);
                        Pz[c] = fma(a.t.G[qz][c], wz, Pz[c]);
                     }
                  }
               }
            }
            const int po = ej * kEp;
#pragma unroll
            for (int c = 0; c < D1; c++) {
               sm.Px[po + c * kSp + qy * Q + qx] = Px[c];
               if (KIND == TFEM_DIFFUSION) {
                  sm.Py[po + c * kSp + qy * Q + qx] = Py[c];
                  sm.Pz[po + c * kSp + qy * Q + qx] = Pz[c];
               }
            }
         }
         team_sync();
         if (!W::QG && pt == 0) mbar_arrive(&sm.empty[s]); // point factors consumed
         // contract qy -> [e][c][b][qx] (x-gradient part in TB, y + z in TG):
         // a lane per (e, c, qx), b unrolled (or a lane per output).  CO: TB
         // is Px itself (read in place below), TG = G_y Py + Pz.
         if constexpr (CO) {
            for (int it = pt; it < EPW * Q * D1; it += NTH) {
               const int j = it / (Q * D1), r = it % (Q * D1), jx = r % Q, c = r / Q;
               const int po = j * kEp + c * kSp + jx;
               if (KIND == TFEM_DIFFUSION) {
                  double py[Q];
#pragma unroll
                  for (int y = 0; y < Q; y++) py[y] = sm.Py[po + y * Q];
#pragma unroll
                  for (int b = 0; b < D1; b++) {
                     double syz = sm.Pz[po + b * Q];
#pragma unroll
                     for (int y = 0; y < Q; y++) syz = fma(a.t.G[y][b], py[y], syz);
                     sm.TG[j * kEt + (c * D1 + b) * kSt + jx] = syz;
                  }
               }
            }
         } else if constexpr (!kRows3) {
            for (int jj = pt; jj < EPW * NT; jj += NTH) {
               const int j = jj / NT, r = jj % NT, jx = r % Q, cb = r / Q, b = cb % D1, c = cb / D1;
               const int po = j * kEp;
               double sx = 0.0, syz = 0.0;
#pragma unroll
               for (int y = 0; y < Q; y++) {
                  const int o = po + c * kSp + y * Q + jx;
                  sx = fma(sB[y][b], sm.Px[o], sx);
                  if (KIND == TFEM_DIFFUSION) {
                     syz = fma(sG[y][b], sm.Py[o], syz);
                     syz = fma(sB[y][b], sm.Pz[o], syz);
                  }
               }
               sm.TB[j * kEt + cb * kSt + jx] = sx;
               sm.TG[j * kEt + cb * kSt + jx] = syz;
            }
         } else
         for (int it = pt; it < EPW * Q * D1; it += NTH) {
            const int j = it / (Q * D1), r = it % (Q * D1), jx = r % Q, c = r / Q;
            const int po = j * kEp + c * kSp + jx;
            double px[Q], py[Q], pz[Q];
#pragma unroll
            for (int y = 0; y < Q; y++) {
               px[y] = sm.Px[po + y * Q];
               if (KIND == TFEM_DIFFUSION) {
                  py[y] = sm.Py[po + y * Q];
                  pz[y] = sm.Pz[po + y * Q];
               }
            }
#pragma unroll
            for (int b = 0; b < D1; b++) {
               double sx = 0.0, syz = 0.0;
#pragma unroll
               for (int y = 0; y < Q; y++) {
                  sx = fma(a.t.B[y][b], px[y], sx);
                  if (KIND == TFEM_DIFFUSION) {
                     syz = fma(a.t.G[y][b], py[y], syz);
                     syz = fma(a.t.B[y][b], pz[y], syz);
                  }
               }
               const int o = j * kEt + (c * D1 + b) * kSt + jx;
               sm.TB[o] = sx;
               if (KIND == TFEM_DIFFUSION) sm.TG[o] = syz;
            }
         }
         team_sync();
         // one output slot: exclusive DOFs to y (essential: x), the rest to
         // the E-vector
         auto put = [&](int j, int i, double r) {
            const int64_t e = g * EPW + j;
            const uint32_t gg = sm.gm[j * ND + i];
            if (is_exclusive(gg)) {
               const uint32_t d = gg & kDofMask;
               if (!a.overwrite) r += a.y[d];
               const bool es = sm.es[j * ND + i] != 0;
               if (es) r = __ldg(a.x + d);
               a.y[d] = r;
               if (EDOT) {
                  if (es) dot = fma(r, r, dot);
               } else if (a.dot && !(a.notown && bit_set(a.notown, d))) {
                  dot = fma(__ldg(a.x + d), r, dot);
               }
            } else {
               a.evec[ev_em_p(a.evperm, ND, e, i)] = r;
            }
         };
         // contract qx -> r(a, b, c) and the epilogue: a lane per (e, c, b),
         // a unrolled (or a lane per output)
         constexpr int kA = kRows1 ? D1 : 1; // outputs per work item
         for (int it = pt; it < cnt * ND / kA; it += NTH) {
            const int j = it / (ND / kA), cb = kRows1 ? it % (D1 * D1) : (it % ND) / D1;
            double tb[Q], tg[Q];
#pragma unroll
            for (int x = 0; x < Q; x++) {
               // CO: TB[c][b][x] = Px[c][y = b][x]
               tb[x] = CO ? sm.Px[j * kEp + (cb / D1) * kSp + (cb % D1) * Q + x]
                          : sm.TB[j * kEt + cb * kSt + x];
               if (KIND == TFEM_DIFFUSION) tg[x] = sm.TG[j * kEt + cb * kSt + x];
            }
#pragma unroll
            for (int ka = 0; ka < kA; ka++) {
               const int ia = kRows1 ? ka : it % D1;
               double r = 0.0;
               if constexpr (CO) {
                  // r = G_x TB + TG[.., a] (B_x = I)
                  if (KIND == TFEM_MASS) {
                     r = kRows1 ? tb[ka] : tb[ia];
                  } else {
#pragma unroll
                     for (int x = 0; x < Q; x++) r = fma(kRows1 ? a.t.G[x][ka] : sG[x][ia], tb[x], r);
                     r += kRows1 ? tg[ka] : tg[ia];
                  }
               } else {
#pragma unroll
                  for (int x = 0; x < Q; x++) {
                     const double gx = kRows1 ? a.t.G[x][ka] : sG[x][ia];
                     const double bx = kRows1 ? a.t.B[x][ka] : sB[x][ia];
                     if (KIND == TFEM_MASS) {
                        r = fma(bx, tb[x], r);
                     } else {
                        r = fma(gx, tb[x], r);
                        r = fma(bx, tg[x], r);
                     }
                  }
               }
               put(j, cb * D1 + ia, r);
            }
         }
         team_sync(); // TB / TG / P reused by the next group
#pragma unroll
         for (int m = 0; m < GPL; m++) {
            gcur[m] = gnext[m];
            gnext[m] = gnn[m];
            mcur[m] = mnext[m];
         }
      }
   }
   if (a.dot) {
      const double v[1] = {dot};
      emit<kBlock, 1>(a.dot, v);
   }
}

// grid: min(blocks of kW warps, persistent blocks) -- elem_blocks (apply.cu)
template <int P, int Q, int KIND, bool CO>
void launch(const ApplyArgs &a, cudaStream_t s, unsigned grid)
{
   using C = Cfg3<P, Q, KIND>;
   static_assert(C::kSmem <= 227 * 1024, "shared memory budget");
   if (a.energy_dot) {
      max_dynamic_smem((const void *)apply3d_tma_kernel<P, Q, KIND, true, CO>, C::kSmem);
      apply3d_tma_kernel<P, Q, KIND, true, CO><<<grid, C::kBlock, C::kSmem, s>>>(a);
   } else {
      max_dynamic_smem((const void *)apply3d_tma_kernel<P, Q, KIND, false, CO>, C::kSmem);
      apply3d_tma_kernel<P, Q, KIND, false, CO><<<grid, C::kBlock, C::kSmem, s>>>(a);
   }
}

template <int P, int Q, int KIND>
KernelPick make(int sm_count, bool colloc)
{
   KernelPick k;
   // bulk copies need 16-byte sizes and element strides (QG: none)
   if constexpr (Warp3<P, Q, KIND>::QG || (Warp3<P, Q, KIND>::NC * Q * Q * Q) % 2 == 0) {
      if constexpr (Q == P + 1)
         k.launch = colloc ? launch<P, Q, KIND, true> : launch<P, Q, KIND, false>;
      else
         k.launch = launch<P, Q, KIND, false>;
      k.elems_per_block = Cfg3<P, Q, KIND>::kT * Warp3<P, Q, KIND>::EPW;
      k.threads = Cfg3<P, Q, KIND>::kBlock;
      k.persistent_blocks = sm_count;
      k.energy_dot = true;
   }
   return k;
}

template <int KIND>
KernelPick pick_kind(int p, int nq, int sm, bool co)
{
   // q <= 7 bulk-copies the point factors; q >= 8 reads them in the column
   // stage (QG)
   switch (p) {
   case 1: return nq == 3 ? make<1, 3, KIND>(sm, co) : nq == 2 ? make<1, 2, KIND>(sm, co) : KernelPick{};
   case 2: return nq == 4 ? make<2, 4, KIND>(sm, co) : nq == 3 ? make<2, 3, KIND>(sm, co) : KernelPick{};
   case 3: return nq == 5 ? make<3, 5, KIND>(sm, co) : nq == 4 ? make<3, 4, KIND>(sm, co) : KernelPick{};
   case 4: return nq == 5 ? make<4, 5, KIND>(sm, co) : nq == 6 ? make<4, 6, KIND>(sm, co) : KernelPick{};
   case 5: return nq == 6 ? make<5, 6, KIND>(sm, co) : nq == 7 ? make<5, 7, KIND>(sm, co) : KernelPick{};
   case 6: if (nq == 7) return make<6, 7, KIND>(sm, co); break; // BP5 p = 6
   }
   // q >= 8, diffusion (QG; measured against the group kernel at ~10M
   // DOFs: BP3 p = 6 +14 %, p = 7 +33 %, p = 8 +32 %, BP5 p = 7 +70 %,
   // p = 8 +38 %); mass stays on the group kernel
   if constexpr (KIND == TFEM_DIFFUSION) {
      if (p == 6 && nq == 8) return make<6, 8, KIND>(sm, co);
      if (p == 7 && nq == 9) return make<7, 9, KIND>(sm, co);
      if (p == 7 && nq == 8) return make<7, 8, KIND>(sm, co);   // BP5 p = 7
      if (p == 8 && nq == 9) return make<8, 9, KIND>(sm, co);   // BP5 p = 8
      if (p == 8 && nq == 10) return make<8, 10, KIND>(sm, co);
   }
   return {};
}

} // namespace

KernelPick pick_apply3d_tma(int p, int nq, int kind, int sm_count, bool colloc)
{
   return kind == TFEM_MASS ? pick_kind<TFEM_MASS>(p, nq, sm_count, colloc)
                            : pick_kind<TFEM_DIFFUSION>(p, nq, sm_count, colloc);
}

} // namespace tfem
