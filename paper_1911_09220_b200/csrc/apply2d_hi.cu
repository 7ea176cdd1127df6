// K2, 2D p >= 4: GRP elements per warp in lockstep, fed by a bulk-copy pipeline
// (cp.async.bulk + mbarrier, LDGSTS) -- the structure of apply3d_tma.cu with
// the contraction stages of apply_grp.cu's 2D kernel.
//
// Persistent block per SM: warps 0..kW-1 compute, warp kW is the producer,
// which streams the qdata of GRP consecutive elements (element-major
// [e][c][q], contiguous; GRP even, so every copy is whole 16-byte units) into
// the computing warp's own 2-slot ring.  The warp advances its GRP elements
// in lockstep: every lane carries GRP independent sum chains per stage (the
// single-element version was latency-bound on one chain per lane).  Each lane
// gathers the next slot's x with LDGSTS while the warp computes.
//
// Every output of every stage is one lane summing sequentially in the
// reference's order -- T = G V / B V (x), d = T B^t / T G^t (y) and the point
// factors, S = G^t W / B^t W (qx), r = S B + S G (qy) (tensor_kernels.cpp:
// 76-110) -- so EXACT is bit-identical to the CPU, like apply_grp.cu.
#include "async.cuh"
#include "kernels.cuh"

namespace tfem {

namespace {

// Row strides padded against shared-memory bank conflicts of the row-wise
// stages (64-bit accesses, half-warp phases; chosen by an exhaustive search
// of the stage access patterns).  qdata is padded per element only when an
// element's point factors are whole 16-byte units (even q), one bulk copy
// per element then (measured: +8 % at q = 8; the smaller copies of q = 6
// cost 20 %, q = 10 6 %).
constexpr int pad_q(int Q) { return Q == 8 ? 8 : 0; }
constexpr int pad_t(int P, int Q)
{
   return (P == 4 && Q == 6) ? 5 : (P == 5 && Q == 6) ? 3 : (P == 5 && Q == 7) ? 1
        : (P == 6 && Q == 7) ? 7 : (P == 7 && Q == 9) ? 1 : 0;
}
constexpr int pad_w(int P, int Q)
{
   return (P == 4 && Q == 6) ? 3 : (P == 5 && Q == 6) ? 3 : (P == 5 && Q == 7) ? 7
        : (P == 6 && Q == 7) ? 7 : (P == 6 && Q == 8) ? 1 : 0;
}
constexpr int pad_s(int P, int Q)
{
   return (P == 5 && Q == 6) ? 3 : (P == 6 && Q == 7) ? 7 : (P == 6 && Q == 8) ? 1 : 0;
}

template <int P, int Q, int KIND>
struct alignas(16) Warp2 {
   static constexpr int D1 = P + 1, ND = D1 * D1, NQD = Q * Q;
   static constexpr int NC = KIND == TFEM_MASS ? 1 : 3;
   // elements per slot, in lockstep: as many rows of the widest stage as
   // fit one warp, even (whole 16-byte qdata copies)
   static constexpr int kRow = D1 > Q ? D1 : Q;
   static constexpr int GRP = (32 / kRow) / 2 * 2 > 2 ? (32 / kRow) / 2 * 2 : 2;
   static constexpr int kSlots = 2;
   static constexpr int kQe = NC * NQD + ((NC * NQD) % 2 == 0 ? pad_q(Q) : 0); // element stride
   static constexpr bool kPerElem = kQe != NC * NQD; // one bulk copy per element
   static constexpr int kT = Q * D1 + pad_t(P, Q), kW2 = Q * Q + pad_w(P, Q), kS = D1 * Q + pad_s(P, Q);
   double q[kSlots][GRP * kQe];
   double V[2][GRP * ND];           // [e][a * D1 + b]
   // T is dead once W is formed, so S (written from W) reuses its storage:
   // the smaller per-warp footprint fits more computing warps per SM
   union {
      struct { double T1[GRP][kT], T2[GRP][kT]; }; // [e][qx][b]
      struct { double S1[GRP][kS], S2[GRP][kS]; }; // [e][a][qy]
   };
   double W1[GRP][kW2], W2[GRP][kW2]; // [e][qx][qy]
   uint32_t gm[GRP * ND];                   // the slot's map entries, for the epilogue
   uint8_t es[GRP * ND];                    // ... and their essential flags (ess_out)
   uint64_t full[kSlots], empty[kSlots];
};

template <int P, int Q, int KIND, bool EXACT, bool CO = false>
struct Cfg2 {
   static constexpr size_t kWarpBytes = sizeof(Warp2<P, Q, KIND>);
   // Latency-bound (ncu at p = 6: 2 warps per scheduler, 0.34 eligible):
   // as many computing warps as shared memory holds (224 KB: +2-7 % over
   // 200 KB at p = 5, 6, 8), up to what the registers allow -- 11 (170
   // registers), 15 (128) where ptxas needs no more (q = 6, p = 4, 5), and
   // in FMA numerics 13 at p = 7, q = 9 (+2.6 %; 126 registers -- 12 to 15
   // warps put four on one SMSP, so ptxas caps at 128; the bit-exact variant
   // needs 168).  12 warps at q = 7, p = 5 measured -2.3 %, at q = 9, p = 8
   // +-1 %: kept at 11 (tools/ab_wide.sh).
   static constexpr bool kDiff = KIND == TFEM_DIFFUSION;
   // BP5 p = 4 (collocated, 104-112 registers): 13 (+2.6 % at 10M, +1.9 % at
   // 200M DOFs; 15 -1 %)
   static constexpr int kMaxW = (kDiff && Q == 6 && (P == 4 || P == 5)) ? 15
                              : (kDiff && CO && P == 4 && Q == 5) ? 13
                              : (kDiff && CO && P == 7) ? 7 // BP5 p = 7: 255 registers, no spills: +2.5 %
                              : (kDiff && !EXACT && P == 7 && Q == 9) ? 13
                              : 11;
   static constexpr int kW0 = static_cast<int>((224 * 1024) / kWarpBytes);
   static constexpr int kW = kW0 > kMaxW ? kMaxW : (kW0 < 1 ? 1 : kW0);
   static constexpr int kBlock = 32 * (kW + 1);
   static constexpr size_t kSmem = kWarpBytes * kW;
};

// CO (collocated, BP5): q = p + 1 Gauss-Lobatto points on the nodes, B1d = I
// exactly: T2 = V, dx = T1, S2 = W2, vx = S1 (the B contractions are copies,
// so the stages read the source in place).  In EXACT numerics the skipped
// sums add only signed zeros, so results stay bit-identical up to the sign
// of a zero.
template <int P, int Q, int KIND, bool EXACT, bool EDOT, bool CO>
__global__ void __launch_bounds__(Cfg2<P, Q, KIND, EXACT, CO>::kBlock, 1) apply2d_hi_kernel(const ApplyArgs a)
{
   static_assert(!CO || Q == P + 1, "collocation needs q = p + 1");
   using W = Warp2<P, Q, KIND>;
   constexpr int D1 = W::D1, ND = W::ND, NQD = W::NQD, NC = W::NC, GRP = W::GRP;
   constexpr int kW = Cfg2<P, Q, KIND, EXACT, CO>::kW, kBlock = Cfg2<P, Q, KIND, EXACT, CO>::kBlock;
   constexpr int kSlots = W::kSlots;
   constexpr int GPL = (GRP * ND + 31) / 32;
   constexpr unsigned kQBytes = NC * NQD * 8;
   static_assert(GRP * D1 <= 32 && GRP * Q <= 32, "row-wise stages: one row per lane");
   if (a.done && *a.done) return;
   extern __shared__ __align__(128) unsigned char smem_raw[];
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
   auto group = [&](int w, int64_t k) { return (int64_t)blockIdx.x * kW + w + k * stride; };
   auto count = [&](int64_t g) {
      const int64_t left = a.ne - g * GRP;
      return static_cast<int>(left < GRP ? (left > 0 ? left : 0) : GRP);
   };
   double dot = 0.0;
   if (warp == kW) {
      // ---------------------------------------------------------- producer
      if (lane == 0) {
         for (int64_t k = 0;; k++) {
            bool any = false;
            for (int w = 0; w < kW; w++) {
               const int64_t g = group(w, k);
               const int cnt = count(g);
               if (cnt == 0) continue;
               any = true;
               const int s = static_cast<int>(k % kSlots);
               if (k >= kSlots)
                  mbar_wait(&ws[w].empty[s], static_cast<unsigned>((k / kSlots - 1) & 1));
               // a partial last pair still copies whole 16-byte units: the
               // padded qdata allocation (ne_pad) covers the tail
               if constexpr (W::kPerElem) {
                  mbar_expect_tx(&ws[w].full[s], kQBytes * cnt);
                  for (int e = 0; e < cnt; e++)
                     bulk_g2s(ws[w].q[s] + e * W::kQe, a.qdata + (g * GRP + e) * (int64_t)(NC * NQD),
                              kQBytes, &ws[w].full[s]);
               } else {
                  const unsigned bytes = (kQBytes * cnt + 15u) & ~15u;
                  mbar_expect_tx(&ws[w].full[s], bytes);
                  bulk_g2s(ws[w].q[s], a.qdata + g * GRP * (int64_t)(NC * NQD), bytes, &ws[w].full[s]);
               }
            }
            if (!any) break;
         }
      }
      __syncwarp();
   } else {
      // ---------------------------------------------------------- consumer
      W &sm = ws[warp];
      uint32_t gcur[GPL], gnext[GPL], gnn[GPL]; // map entries: this, next, next-but-one group
      uint32_t mcur[GPL], mnext[GPL]; // mask_in words of the map entries
      auto load_map = [&](int64_t g, uint32_t (&m_)[GPL]) {
         const int64_t lim = (int64_t)count(g) * ND;
#pragma unroll
         for (int m = 0; m < GPL; m++) {
            const int i = lane + 32 * m;
            m_[m] = i < lim ? __ldg(a.gmap + g * GRP * ND + i) : 0u;
         }
      };
      // V[e][a * D1 + b] = x[dofs[b * D1 + a]]
      auto vslot = [](int i) { const int e = i / ND, t = i % ND; return e * ND + (t % D1) * D1 + t / D1; };
      auto prefetch_x = [&](int64_t g, const uint32_t (&m_)[GPL], int buf) {
         const int64_t lim = (int64_t)count(g) * ND;
         if (lim == 0) return;
#pragma unroll
         for (int m = 0; m < GPL; m++) {
            const int i = lane + 32 * m;
            if (i < lim) gather8(&sm.V[buf][vslot(i)], a.x + (m_[m] & kDofMask));
         }
         cp_async_commit();
      };
      // the mask words go out with the gather (tested a group later)
      auto load_mask = [&](int64_t g, const uint32_t (&m_)[GPL], uint32_t (&w_)[GPL]) {
         const int64_t lim = (int64_t)count(g) * ND;
#pragma unroll
         for (int m = 0; m < GPL; m++) {
            const int i = lane + 32 * m;
            w_[m] = a.mask_in && i < lim ? __ldg(a.mask_in + ((m_[m] & kDofMask) >> 5)) : 0u;
         }
      };
      const bool ess_is_mask = a.ess_out == a.mask_in;
      load_map(group(warp, 0), gcur);
      load_map(group(warp, 1), gnext);
      prefetch_x(group(warp, 0), gcur, 0);
      load_mask(group(warp, 0), gcur, mcur);
      for (int64_t k = 0;; k++) {
         const int64_t g = group(warp, k);
         const int cnt = count(g);
         if (cnt == 0) break;
         const int vb = static_cast<int>(k & 1);
         cp_async_wait_all();
         // masked gather; the map entries and essential flags go to shared
         // memory for the epilogue (no global loads there)
#pragma unroll
         for (int m = 0; m < GPL; m++) {
            const int i = lane + 32 * m;
            if (i >= cnt * ND) continue;
            const uint32_t d = gcur[m] & kDofMask;
            const bool mk = (mcur[m] >> (d & 31)) & 1u;
            if (mk) sm.V[vb][vslot(i)] = 0.0;
            sm.gm[i] = gcur[m];
            sm.es[i] = (ess_is_mask ? mk : (a.ess_out && bit_set(a.ess_out, d))) ? 1 : 0;
         }
         __syncwarp();
         const int64_t gn = group(warp, k + 1);
         load_map(group(warp, k + 2), gnn); // two groups ahead: used a group later
         const int s = static_cast<int>(k % kSlots);
         mbar_wait(&sm.full[s], static_cast<unsigned>((k / kSlots) & 1));
         {
            const double *qs = sm.q[s];
            // Every stage is row-wise: a lane per (element, row) loads the
            // row once and runs the unrolled outputs along it with the basis
            // operands as compile-time constant-bank operands (the
            // per-output lane mapping was shared-memory bound).
            if (lane < GRP * D1 && !(CO && KIND == TFEM_MASS)) { // contract x: T[qx][b], a lane per (e, b)
               const int j = lane / D1, b = lane % D1;
               const double *V = sm.V[vb] + j * ND;
               double v[D1];
#pragma unroll
               for (int kk = 0; kk < D1; kk++) v[kk] = V[kk * D1 + b];
#pragma unroll
               for (int qx = 0; qx < Q; qx++) {
                  double s1 = mul<EXACT>(a.t.G[qx][0], v[0]);
                  double s2 = mul<EXACT>(a.t.B[qx][0], v[0]);
#pragma unroll
                  for (int kk = 1; kk < D1; kk++) {
                     if (KIND == TFEM_DIFFUSION) s1 = mac<EXACT>(s1, a.t.G[qx][kk], v[kk]);
                     if (!CO) s2 = mac<EXACT>(s2, a.t.B[qx][kk], v[kk]);
                  }
                  if (KIND == TFEM_DIFFUSION) sm.T1[j][qx * D1 + b] = s1;
                  if (!CO) sm.T2[j][qx * D1 + b] = s2; // CO: T2 = V in place
               }
            }
            prefetch_x(gn, gnext, vb ^ 1); // the other V buffer is free
            load_mask(gn, gnext, mnext);
            __syncwarp();
            if (lane < GRP * Q) { // contract y, point factors: W[qx][qy], a lane per (e, qx)
               const int j = lane / Q, qx = lane % Q;
               const double *qd = qs + j * W::kQe;
               const bool live = j < cnt;
               double t1[D1], t2[D1];
               const double *T2s = CO ? sm.V[vb] + j * ND : sm.T2[j]; // CO: T2 = V ([a D1 + b])
#pragma unroll
               for (int b = 0; b < D1; b++) {
                  if (KIND == TFEM_DIFFUSION) t1[b] = sm.T1[j][qx * D1 + b];
                  t2[b] = T2s[qx * D1 + b];
               }
#pragma unroll
               for (int qy = 0; qy < Q; qy++) {
                  const int t = qy * Q + qx;
                  if (KIND == TFEM_DIFFUSION) {
                     double dx = CO ? t1[qy] : mul<EXACT>(t1[0], a.t.B[qy][0]);
                     double dy = mul<EXACT>(t2[0], a.t.G[qy][0]);
#pragma unroll
                     for (int b = 1; b < D1; b++) {
                        if (!CO) dx = mac<EXACT>(dx, t1[b], a.t.B[qy][b]);
                        dy = mac<EXACT>(dy, t2[b], a.t.G[qy][b]);
                     }
                     const double d0 = qd[t], d1 = qd[NQD + t], d2 = qd[2 * NQD + t];
                     const double w1 = add<EXACT>(mul<EXACT>(d0, dx), mul<EXACT>(d1, dy));
                     const double w2 = add<EXACT>(mul<EXACT>(d1, dx), mul<EXACT>(d2, dy));
                     if (EDOT && live) dot = mac<EXACT>(mac<EXACT>(dot, dx, w1), dy, w2);
                     sm.W1[j][qx * Q + qy] = w1;
                     sm.W2[j][qx * Q + qy] = w2;
                  } else {
                     double u = CO ? t2[qy] : mul<EXACT>(t2[0], a.t.B[qy][0]);
#pragma unroll
                     for (int b = 1; b < D1; b++)
                        if (!CO) u = mac<EXACT>(u, t2[b], a.t.B[qy][b]);
                     const double w = mul<EXACT>(u, qd[t]);
                     if (EDOT && live) dot = mac<EXACT>(dot, u, w);
                     sm.W2[j][qx * Q + qy] = w;
                  }
               }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.empty[s]); // point factors consumed
            if (lane < GRP * Q && !(CO && KIND == TFEM_MASS)) { // contract qx: S[a][qy], a lane per (e, qy)
               const int j = lane / Q, qy = lane % Q;
               double w1[Q], w2[Q];
#pragma unroll
               for (int qx = 0; qx < Q; qx++) {
                  if (KIND == TFEM_DIFFUSION) w1[qx] = sm.W1[j][qx * Q + qy];
                  if (!CO) w2[qx] = sm.W2[j][qx * Q + qy];
               }
#pragma unroll
               for (int i = 0; i < D1; i++) {
                  if (KIND == TFEM_DIFFUSION) {
                     double s1 = mul<EXACT>(a.t.G[0][i], w1[0]);
                     double s2 = CO ? 0.0 : mul<EXACT>(a.t.B[0][i], w2[0]);
#pragma unroll
                     for (int qx = 1; qx < Q; qx++) {
                        s1 = mac<EXACT>(s1, a.t.G[qx][i], w1[qx]);
                        if (!CO) s2 = mac<EXACT>(s2, a.t.B[qx][i], w2[qx]);
                     }
                     sm.S1[j][i * Q + qy] = s1;
                     if (!CO) sm.S2[j][i * Q + qy] = s2; // CO: S2 = W2 in place
                  } else {
                     double sv = mul<EXACT>(a.t.B[0][i], w2[0]);
#pragma unroll
                     for (int qx = 1; qx < Q; qx++) sv = mac<EXACT>(sv, a.t.B[qx][i], w2[qx]);
                     sm.S2[j][i * Q + qy] = sv;
                  }
               }
            }
            __syncwarp();
            if (lane < cnt * D1) { // contract qy: r(a, b), a lane per (e, a); epilogue
               const int j = lane / D1, ia = lane % D1;
               double s1[Q], s2[Q];
               // CO: S2 = W2 ([qx = a][qy])
               const double *S2s = CO ? sm.W2[j] : sm.S2[j];
#pragma unroll
               for (int qy = 0; qy < Q; qy++) {
                  if (KIND == TFEM_DIFFUSION) s1[qy] = sm.S1[j][ia * Q + qy];
                  s2[qy] = S2s[ia * Q + qy];
               }
               const int64_t e = g * GRP + j;
#pragma unroll
               for (int b = 0; b < D1; b++) {
                  double rr;
                  if (KIND == TFEM_DIFFUSION) {
                     double vx = CO ? s1[b] : mul<EXACT>(s1[0], a.t.B[0][b]);
                     double vy = mul<EXACT>(s2[0], a.t.G[0][b]);
#pragma unroll
                     for (int qy = 1; qy < Q; qy++) {
                        if (!CO) vx = mac<EXACT>(vx, s1[qy], a.t.B[qy][b]);
                        vy = mac<EXACT>(vy, s2[qy], a.t.G[qy][b]);
                     }
                     rr = add<EXACT>(vx, vy);
                  } else if (CO) {
                     rr = s2[b];
                  } else {
                     rr = mul<EXACT>(s2[0], a.t.B[0][b]);
#pragma unroll
                     for (int qy = 1; qy < Q; qy++) rr = mac<EXACT>(rr, s2[qy], a.t.B[qy][b]);
                  }
                  const int t = ia + D1 * b;
                  const uint32_t gg = sm.gm[j * ND + t];
                  if (is_exclusive(gg)) {
                     const uint32_t d = gg & kDofMask;
                     if (!a.overwrite) rr = add<EXACT>(a.y[d], rr);
                     const bool es = sm.es[j * ND + t] != 0;
                     if (es) rr = __ldg(a.x + d);
                     a.y[d] = rr;
                     if (EDOT) {
                        if (es) dot = mac<EXACT>(dot, rr, rr);
                     } else if (a.dot && !(a.notown && bit_set(a.notown, d))) {
                        dot = mac<EXACT>(dot, __ldg(a.x + d), rr);
                     }
                  } else {
                     a.evec[ev_em_p(a.evperm, ND, e, t)] = rr;
                  }
               }
            }
            __syncwarp(); // T / W / S reused by the next slot
         }
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

// grid: min(blocks of kW groups, persistent blocks) -- elem_blocks (apply.cu)
template <int P, int Q, int KIND, bool EXACT, bool CO>
void launch(const ApplyArgs &a, cudaStream_t s, unsigned grid)
{
   using C = Cfg2<P, Q, KIND, EXACT, CO>;
   static_assert(C::kSmem <= 227 * 1024, "shared memory budget");
   if (a.energy_dot) {
      max_dynamic_smem((const void *)apply2d_hi_kernel<P, Q, KIND, EXACT, true, CO>, C::kSmem);
      apply2d_hi_kernel<P, Q, KIND, EXACT, true, CO><<<grid, C::kBlock, C::kSmem, s>>>(a);
   } else {
      max_dynamic_smem((const void *)apply2d_hi_kernel<P, Q, KIND, EXACT, false, CO>, C::kSmem);
      apply2d_hi_kernel<P, Q, KIND, EXACT, false, CO><<<grid, C::kBlock, C::kSmem, s>>>(a);
   }
}

template <int P, int Q, int KIND, bool EXACT>
Launch launcher(bool colloc)
{
   if constexpr (Q == P + 1)
      if (colloc) return launch<P, Q, KIND, EXACT, true>;
   return launch<P, Q, KIND, EXACT, false>;
}

template <int P, int Q, int KIND>
KernelPick make(bool exact, int sm_count, bool colloc)
{
   KernelPick k;
   k.launch = exact ? launcher<P, Q, KIND, true>(colloc) : launcher<P, Q, KIND, false>(colloc);
   int kw = exact ? Cfg2<P, Q, KIND, true>::kW : Cfg2<P, Q, KIND, false>::kW;
   int kb = exact ? Cfg2<P, Q, KIND, true>::kBlock : Cfg2<P, Q, KIND, false>::kBlock;
   if constexpr (Q == P + 1) {
      if (colloc) {
         kw = exact ? Cfg2<P, Q, KIND, true, true>::kW : Cfg2<P, Q, KIND, false, true>::kW;
         kb = exact ? Cfg2<P, Q, KIND, true, true>::kBlock : Cfg2<P, Q, KIND, false, true>::kBlock;
      }
   }
   k.elems_per_block = kw * Warp2<P, Q, KIND>::GRP;
   k.threads = kb;
   k.persistent_blocks = sm_count;
   k.energy_dot = true;
   return k;
}

template <int P, int KIND>
KernelPick pick_q(int nq, bool exact, int sm, bool co)
{
   if (nq == P + 2) return make<P, P + 2, KIND>(exact, sm, false);
   if (nq == P + 1) return make<P, P + 1, KIND>(exact, sm, co);
   return {};
}

template <int KIND>
KernelPick pick_p(int p, int nq, bool exact, int sm, bool co)
{
   switch (p) {
   case 4: return pick_q<4, KIND>(nq, exact, sm, co);
   case 5: return pick_q<5, KIND>(nq, exact, sm, co);
   case 6: return pick_q<6, KIND>(nq, exact, sm, co);
   case 7: return pick_q<7, KIND>(nq, exact, sm, co);
   case 8: return pick_q<8, KIND>(nq, exact, sm, co);
   }
   return {};
}

} // namespace

KernelPick pick_apply2d_hi(int p, int nq, int kind, bool exact, int sm_count, bool colloc)
{
   return kind == TFEM_MASS ? pick_p<TFEM_MASS>(p, nq, exact, sm_count, colloc)
                            : pick_p<TFEM_DIFFUSION>(p, nq, exact, sm_count, colloc);
}

} // namespace tfem
