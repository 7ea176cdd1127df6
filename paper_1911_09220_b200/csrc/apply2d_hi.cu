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

template <int P, int Q, int KIND>
struct alignas(16) Warp2 {
   static constexpr int D1 = P + 1, ND = D1 * D1, NQD = Q * Q;
   static constexpr int NC = KIND == TFEM_MASS ? 1 : 3;
   static constexpr int GRP = P <= 6 ? 4 : 2; // elements per slot, in lockstep
   static constexpr int kSlots = 2;
   double q[kSlots][GRP * NC * NQD];
   double V[2][GRP * ND];             // [e][a * D1 + b]
   double T1[GRP][Q * D1], T2[GRP][Q * D1]; // [e][qx][b]
   double W1[GRP][Q * Q], W2[GRP][Q * Q];   // [e][qx][qy]
   double S1[GRP][D1 * Q], S2[GRP][D1 * Q]; // [e][a][qy]
   uint32_t gm[GRP * ND];                   // the slot's map entries, for the epilogue
   uint8_t es[GRP * ND];                    // ... and their essential flags (ess_out)
   uint64_t full[kSlots], empty[kSlots];
};

template <int P, int Q, int KIND>
struct Cfg2 {
   static constexpr size_t kWarpBytes = sizeof(Warp2<P, Q, KIND>);
   static constexpr int kW0 = static_cast<int>((200 * 1024) / kWarpBytes);
   static constexpr int kW = kW0 > 11 ? 11 : (kW0 < 1 ? 1 : kW0);
   static constexpr int kBlock = 32 * (kW + 1);
   static constexpr size_t kSmem = kWarpBytes * kW;
};

template <int P, int Q, int KIND, bool EXACT, bool EDOT>
__global__ void __launch_bounds__(Cfg2<P, Q, KIND>::kBlock, 1) apply2d_hi_kernel(const ApplyArgs a)
{
   using W = Warp2<P, Q, KIND>;
   constexpr int D1 = W::D1, ND = W::ND, NQD = W::NQD, NC = W::NC, GRP = W::GRP;
   constexpr int kW = Cfg2<P, Q, KIND>::kW, kBlock = Cfg2<P, Q, KIND>::kBlock;
   constexpr int kSlots = W::kSlots;
   constexpr int GPL = (GRP * ND + 31) / 32;
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
               const unsigned bytes = (kQBytes * cnt + 15u) & ~15u;
               mbar_expect_tx(&ws[w].full[s], bytes);
               bulk_g2s(ws[w].q[s], a.qdata + g * GRP * (int64_t)(NC * NQD), bytes, &ws[w].full[s]);
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
            for (int t = lane; t < Q * D1; t += 32) { // contract x: [qx][b]
               const int qx = t / D1, b = t % D1;
#pragma unroll
               for (int j = 0; j < GRP; j++) {
                  const double *V = sm.V[vb] + j * ND;
                  double s1 = mul<EXACT>(sG[qx][0], V[b]);
                  double s2 = mul<EXACT>(sB[qx][0], V[b]);
#pragma unroll
                  for (int kk = 1; kk < D1; kk++) {
                     if (KIND == TFEM_DIFFUSION) s1 = mac<EXACT>(s1, sG[qx][kk], V[kk * D1 + b]);
                     s2 = mac<EXACT>(s2, sB[qx][kk], V[kk * D1 + b]);
                  }
                  sm.T1[j][t] = s1;
                  sm.T2[j][t] = s2;
               }
            }
            prefetch_x(gn, gnext, vb ^ 1); // the other V buffer is free
            load_mask(gn, gnext, mnext);
            __syncwarp();
            for (int t = lane; t < NQD; t += 32) { // contract y, point factors: [qx][qy]
               const int qx = t % Q, qy = t / Q;
#pragma unroll
               for (int j = 0; j < GRP; j++) {
                  const double *qd = qs + j * NC * NQD;
                  const bool live = j < cnt;
                  if (KIND == TFEM_DIFFUSION) {
                     double dx = mul<EXACT>(sm.T1[j][qx * D1], sB[qy][0]);
                     double dy = mul<EXACT>(sm.T2[j][qx * D1], sG[qy][0]);
#pragma unroll
                     for (int b = 1; b < D1; b++) {
                        dx = mac<EXACT>(dx, sm.T1[j][qx * D1 + b], sB[qy][b]);
                        dy = mac<EXACT>(dy, sm.T2[j][qx * D1 + b], sG[qy][b]);
                     }
                     const double d0 = qd[t], d1 = qd[NQD + t], d2 = qd[2 * NQD + t];
                     const double w1 = add<EXACT>(mul<EXACT>(d0, dx), mul<EXACT>(d1, dy));
                     const double w2 = add<EXACT>(mul<EXACT>(d1, dx), mul<EXACT>(d2, dy));
                     if (EDOT && live) dot = mac<EXACT>(mac<EXACT>(dot, dx, w1), dy, w2);
                     sm.W1[j][qx * Q + qy] = w1;
                     sm.W2[j][qx * Q + qy] = w2;
                  } else {
                     double u = mul<EXACT>(sm.T2[j][qx * D1], sB[qy][0]);
#pragma unroll
                     for (int b = 1; b < D1; b++) u = mac<EXACT>(u, sm.T2[j][qx * D1 + b], sB[qy][b]);
                     const double w = mul<EXACT>(u, qd[t]);
                     if (EDOT && live) dot = mac<EXACT>(dot, u, w);
                     sm.W2[j][qx * Q + qy] = w;
                  }
               }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.empty[s]); // point factors consumed
            for (int t = lane; t < D1 * Q; t += 32) { // contract qx: [a][qy]
               const int i = t / Q, qy = t % Q;
#pragma unroll
               for (int j = 0; j < GRP; j++) {
                  if (KIND == TFEM_DIFFUSION) {
                     double s1 = mul<EXACT>(sG[0][i], sm.W1[j][qy]);
                     double s2 = mul<EXACT>(sB[0][i], sm.W2[j][qy]);
#pragma unroll
                     for (int qx = 1; qx < Q; qx++) {
                        s1 = mac<EXACT>(s1, sG[qx][i], sm.W1[j][qx * Q + qy]);
                        s2 = mac<EXACT>(s2, sB[qx][i], sm.W2[j][qx * Q + qy]);
                     }
                     sm.S1[j][t] = s1;
                     sm.S2[j][t] = s2;
                  } else {
                     double sv = mul<EXACT>(sB[0][i], sm.W2[j][qy]);
#pragma unroll
                     for (int qx = 1; qx < Q; qx++) sv = mac<EXACT>(sv, sB[qx][i], sm.W2[j][qx * Q + qy]);
                     sm.S2[j][t] = sv;
                  }
               }
            }
            __syncwarp();
#pragma unroll
            for (int m = 0; m < (ND + 31) / 32; m++) { // contract qy: r(a, b)
               const int t = lane + 32 * m;
               if (t >= ND) continue;
               const int ia = t % D1, b = t / D1;
               double r[GRP];
#pragma unroll
               for (int j = 0; j < GRP; j++) {
                  if (KIND == TFEM_DIFFUSION) {
                     double vx = mul<EXACT>(sm.S1[j][ia * Q], sB[0][b]);
                     double vy = mul<EXACT>(sm.S2[j][ia * Q], sG[0][b]);
#pragma unroll
                     for (int qy = 1; qy < Q; qy++) {
                        vx = mac<EXACT>(vx, sm.S1[j][ia * Q + qy], sB[qy][b]);
                        vy = mac<EXACT>(vy, sm.S2[j][ia * Q + qy], sG[qy][b]);
                     }
                     r[j] = add<EXACT>(vx, vy);
                  } else {
                     double rv = mul<EXACT>(sm.S2[j][ia * Q], sB[0][b]);
#pragma unroll
                     for (int qy = 1; qy < Q; qy++) rv = mac<EXACT>(rv, sm.S2[j][ia * Q + qy], sB[qy][b]);
                     r[j] = rv;
                  }
               }
#pragma unroll
               for (int j = 0; j < GRP; j++) {
                  if (j >= cnt) continue;
                  const int64_t e = g * GRP + j;
                  double rr = r[j];
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
                     a.evec[ev_em(ND, a.ne_pad, e, t)] = rr;
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

int g_sm2 = 0;

template <int P, int Q, int KIND, bool EXACT>
void launch(const ApplyArgs &a, cudaStream_t s, unsigned /*blocks*/)
{
   using C = Cfg2<P, Q, KIND>;
   static_assert(C::kSmem <= 227 * 1024, "shared memory budget");
   static const bool once = [] {
      cudaFuncSetAttribute(apply2d_hi_kernel<P, Q, KIND, EXACT, false>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem);
      cudaFuncSetAttribute(apply2d_hi_kernel<P, Q, KIND, EXACT, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem);
      return true;
   }();
   (void)once;
   constexpr int GRP = Warp2<P, Q, KIND>::GRP;
   const int64_t groups = (a.ne + GRP - 1) / GRP;
   const int64_t nblk = (groups + C::kW - 1) / C::kW;
   const unsigned grid = static_cast<unsigned>(nblk < g_sm2 ? nblk : g_sm2);
   if (a.energy_dot)
      apply2d_hi_kernel<P, Q, KIND, EXACT, true><<<grid, C::kBlock, C::kSmem, s>>>(a);
   else
      apply2d_hi_kernel<P, Q, KIND, EXACT, false><<<grid, C::kBlock, C::kSmem, s>>>(a);
}

template <int P, int Q, int KIND>
KernelPick make(bool exact)
{
   KernelPick k;
   k.launch = exact ? launch<P, Q, KIND, true> : launch<P, Q, KIND, false>;
   k.elems_per_block = Cfg2<P, Q, KIND>::kW * Warp2<P, Q, KIND>::GRP;
   k.threads = Cfg2<P, Q, KIND>::kBlock;
   k.persistent_blocks = g_sm2;
   k.energy_dot = true;
   return k;
}

template <int P, int KIND>
KernelPick pick_q(int nq, bool exact)
{
   if (nq == P + 2) return make<P, P + 2, KIND>(exact);
   if (nq == P + 1) return make<P, P + 1, KIND>(exact);
   return {};
}

template <int KIND>
KernelPick pick_p(int p, int nq, bool exact)
{
   switch (p) {
   case 4: return pick_q<4, KIND>(nq, exact);
   case 5: return pick_q<5, KIND>(nq, exact);
   case 6: return pick_q<6, KIND>(nq, exact);
   case 7: return pick_q<7, KIND>(nq, exact);
   case 8: return pick_q<8, KIND>(nq, exact);
   }
   return {};
}

} // namespace

KernelPick pick_apply2d_hi(int p, int nq, int kind, bool exact, int sm_count)
{
   g_sm2 = sm_count;
   return kind == TFEM_MASS ? pick_p<TFEM_MASS>(p, nq, exact) : pick_p<TFEM_DIFFUSION>(p, nq, exact);
}

} // namespace tfem
