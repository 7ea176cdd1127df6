// K2, one element per thread group (NT = round32(q^2) threads), contractions
// staged through shared memory.
//
// 2D (p >= 4, where the register-resident kernel would spill): every stage
// assigns one output entry to one thread, which sums sequentially in the
// reference's order -- T = G V / B V (contract x), d = T B^t / T G^t
// (contract y), pointwise D, S = G^t W / B^t W (contract qx), r = S B + S G
// (contract qy) (tensor_kernels.cpp:76-110).  EXACT keeps it bit-identical.
//
// 3D: threads own (qx, qy) z-columns; the y/z contractions of a column stay
// in registers, x/y contractions go through shared memory.  Order: in x, y,
// z; out z, y, x (fused multiply-adds; 3D has no reference to match bits).
//
// Both read qdata element-major [e][c][q] (one coalesced row per component)
// and the element-major map [e][nd]; B1d/G1d are copied into shared memory
// once per block because the table indices differ across lanes.
#include "kernels.cuh"

namespace tfem {

namespace {

template <int P, int Q>
struct Smem2D {
   static constexpr int D1 = P + 1;
   double V[D1 * D1];         // V[a*D1 + b]
   double T1[Q * D1], T2[Q * D1]; // [qx][b]
   double W1[Q * Q], W2[Q * Q];   // [qx][qy]
   double S1[D1 * Q], S2[D1 * Q]; // [a][qy]
};

template <int P, int Q, int KIND, bool EXACT>
__global__ void apply2d_grp_kernel(const ApplyArgs a)
{
   constexpr int D1 = P + 1, ND = D1 * D1, NQD = Q * Q;
   constexpr int NT = round32(Q * Q);
   if (a.done && *a.done) return;
   __shared__ double sB[Q][D1], sG[Q][D1];
   extern __shared__ double smem_raw[];
   for (int j = threadIdx.x; j < Q * D1; j += blockDim.x) {
      sB[j / D1][j % D1] = a.t.B[j / D1][j % D1];
      sG[j / D1][j % D1] = a.t.G[j / D1][j % D1];
   }
   const int g = threadIdx.x / NT, t = threadIdx.x % NT;
   const int64_t e = blockIdx.x * (int64_t)(blockDim.x / NT) + g;
   const bool live = e < a.ne;
   auto &sm = reinterpret_cast<Smem2D<P, Q> *>(smem_raw)[g];
   uint32_t dof = 0;
   if (live && t < ND) {
      dof = __ldg(a.gmap + e * ND + t);
      const uint32_t d = dof & kDofMask;
      double v = __ldg(a.x + d);
      if (a.mask_in && bit_set(a.mask_in, d)) v = 0.0;
      sm.V[(t % D1) * D1 + t / D1] = v; // V(a, b) = x[dofs[b*D1 + a]]
   }
   __syncthreads();
   if (live && t < Q * D1) { // contract x: [qx][b]
      const int qx = t / D1, b = t % D1;
      double s1 = mul<EXACT>(sG[qx][0], sm.V[b]);
      double s2 = mul<EXACT>(sB[qx][0], sm.V[b]);
#pragma unroll
      for (int k = 1; k < D1; k++) {
         if (KIND == TFEM_DIFFUSION) s1 = mac<EXACT>(s1, sG[qx][k], sm.V[k * D1 + b]);
         s2 = mac<EXACT>(s2, sB[qx][k], sm.V[k * D1 + b]);
      }
      sm.T1[t] = s1;
      sm.T2[t] = s2;
   }
   __syncthreads();
   if (live && t < NQD) { // contract y and the point factors: [qx][qy]
      const int qx = t % Q, qy = t / Q;
      const double *qd = a.qdata + e * (int64_t)(KIND == TFEM_MASS ? 1 : 3) * NQD;
      if (KIND == TFEM_DIFFUSION) {
         double dx = mul<EXACT>(sm.T1[qx * D1], sB[qy][0]);
         double dy = mul<EXACT>(sm.T2[qx * D1], sG[qy][0]);
#pragma unroll
         for (int b = 1; b < D1; b++) {
            dx = mac<EXACT>(dx, sm.T1[qx * D1 + b], sB[qy][b]);
            dy = mac<EXACT>(dy, sm.T2[qx * D1 + b], sG[qy][b]);
         }
         const double d0 = __ldg(qd + t), d1 = __ldg(qd + NQD + t), d2 = __ldg(qd + 2 * NQD + t);
         sm.W1[qx * Q + qy] = add<EXACT>(mul<EXACT>(d0, dx), mul<EXACT>(d1, dy));
         sm.W2[qx * Q + qy] = add<EXACT>(mul<EXACT>(d1, dx), mul<EXACT>(d2, dy));
      } else {
         double u = mul<EXACT>(sm.T2[qx * D1], sB[qy][0]);
#pragma unroll
         for (int b = 1; b < D1; b++) u = mac<EXACT>(u, sm.T2[qx * D1 + b], sB[qy][b]);
         sm.W2[qx * Q + qy] = mul<EXACT>(u, __ldg(qd + t));
      }
   }
   __syncthreads();
   if (live && t < D1 * Q) { // contract qx: [a][qy]
      const int i = t / Q, qy = t % Q;
      if (KIND == TFEM_DIFFUSION) {
         double s1 = mul<EXACT>(sG[0][i], sm.W1[qy]);
         double s2 = mul<EXACT>(sB[0][i], sm.W2[qy]);
#pragma unroll
         for (int qx = 1; qx < Q; qx++) {
            s1 = mac<EXACT>(s1, sG[qx][i], sm.W1[qx * Q + qy]);
            s2 = mac<EXACT>(s2, sB[qx][i], sm.W2[qx * Q + qy]);
         }
         sm.S1[t] = s1;
         sm.S2[t] = s2;
      } else {
         double s = mul<EXACT>(sB[0][i], sm.W2[qy]);
#pragma unroll
         for (int qx = 1; qx < Q; qx++) s = mac<EXACT>(s, sB[qx][i], sm.W2[qx * Q + qy]);
         sm.S2[t] = s;
      }
   }
   __syncthreads();
   double dot = 0.0;
   if (live && t < ND) { // contract qy: r(a, b), out[b*D1 + a] = r(a, b)
      const int ia = t % D1, b = t / D1;
      double r;
      if (KIND == TFEM_DIFFUSION) {
         double vx = mul<EXACT>(sm.S1[ia * Q], sB[0][b]);
         double vy = mul<EXACT>(sm.S2[ia * Q], sG[0][b]);
#pragma unroll
         for (int qy = 1; qy < Q; qy++) {
            vx = mac<EXACT>(vx, sm.S1[ia * Q + qy], sB[qy][b]);
            vy = mac<EXACT>(vy, sm.S2[ia * Q + qy], sG[qy][b]);
         }
         r = add<EXACT>(vx, vy);
      } else {
         r = mul<EXACT>(sm.S2[ia * Q], sB[0][b]);
#pragma unroll
         for (int qy = 1; qy < Q; qy++) r = mac<EXACT>(r, sm.S2[ia * Q + qy], sB[qy][b]);
      }
      if (is_exclusive(dof)) {
         const uint32_t d = dof & kDofMask;
         if (!a.overwrite) r = add<EXACT>(a.y[d], r);
         if (a.ess_out && bit_set(a.ess_out, d)) r = __ldg(a.x + d);
         a.y[d] = r;
         if (a.dot && !(a.notown && bit_set(a.notown, d))) dot = mul<EXACT>(__ldg(a.x + d), r);
      } else {
         a.evec[ev_em_p(a.evperm, ND, e, t)] = r;
      }
   }
   if (a.dot) {
      const double v[1] = {dot};
      emit<NT * groups_for(NT), 1>(a.dot, v);
   }
}

template <int P, int Q>
struct Smem3D {
   static constexpr int D1 = P + 1;
   double TB[D1 * D1 * Q], TG[D1 * D1 * Q];   // [c][b][qx]
   // V is dead once TB / TG are formed, before the column stage writes the
   // P planes: they share storage (a smaller per-element footprint fits
   // more elements per SM at q >= 8)
   union {
      double V[D1 * D1 * D1];                                // [c][b][a]
      struct { double Px[D1 * Q * Q], Py[D1 * Q * Q], Pz[D1 * Q * Q]; }; // [c][qy][qx]
   };
};

template <int P, int Q, int KIND>
__global__ void apply3d_kernel(const ApplyArgs a)
{
   constexpr int D1 = P + 1, ND = D1 * D1 * D1, NQD = Q * Q * Q;
   constexpr int NT = round32(Q * Q);
   if (a.done && *a.done) return;
   __shared__ double sB[Q][D1], sG[Q][D1];
   extern __shared__ double smem_raw[];
   for (int j = threadIdx.x; j < Q * D1; j += blockDim.x) {
      sB[j / D1][j % D1] = a.t.B[j / D1][j % D1];
      sG[j / D1][j % D1] = a.t.G[j / D1][j % D1];
   }
   const int g = threadIdx.x / NT, t = threadIdx.x % NT;
   const int64_t e = blockIdx.x * (int64_t)(blockDim.x / NT) + g;
   const bool live = e < a.ne;
   auto &sm = reinterpret_cast<Smem3D<P, Q> *>(smem_raw)[g];
   const uint32_t *gm = a.gmap + e * ND;
   if (live) {
      for (int i = t; i < ND; i += NT) {
         const uint32_t d = __ldg(gm + i) & kDofMask;
         double v = __ldg(a.x + d);
         if (a.mask_in && bit_set(a.mask_in, d)) v = 0.0;
         sm.V[i] = v;
      }
   }
   __syncthreads();
   // The contractions between the column stage and the element's ends are
   // row-wise: a thread per row loads it once and runs the unrolled outputs
   // with the basis operands from the constant bank.
   if (live) { // contract a -> TB / TG [c][b][qx]: a thread per (c, b)
      for (int cb = t; cb < D1 * D1; cb += NT) {
         double v[D1];
#pragma unroll
         for (int k = 0; k < D1; k++) v[k] = sm.V[cb * D1 + k];
#pragma unroll
         for (int qx = 0; qx < Q; qx++) {
            double sb = 0.0, sg = 0.0;
#pragma unroll
            for (int k = 0; k < D1; k++) {
               sb = fma(a.t.B[qx][k], v[k], sb);
               if (KIND == TFEM_DIFFUSION) sg = fma(a.t.G[qx][k], v[k], sg);
            }
            sm.TB[cb * Q + qx] = sb;
            if (KIND == TFEM_DIFFUSION) sm.TG[cb * Q + qx] = sg;
         }
      }
   }
   __syncthreads();
   const int qx = t % Q, qy = t / Q;
   if (live && t < Q * Q) {
      // q >= 10: the column's point factors stream kR planes ahead of the qz
      // walk (issued before the b contraction), so their latency is not paid
      // at every qz step (measured p = 8: +8 %; p = 6, 7: neutral to -2 %,
      // so there each plane is loaded at its own step)
      constexpr int NCQ = KIND == TFEM_MASS ? 1 : 6;
      constexpr int kR = Q >= 10 ? 3 : 0;
      const double *qd = a.qdata + e * (int64_t)NCQ * NQD + qx + Q * qy;
      double Dq[NCQ][Q];
      auto load_plane = [&](int qz) {
#pragma unroll
         for (int c = 0; c < NCQ; c++) Dq[c][qz] = __ldg(qd + c * NQD + Q * Q * qz);
      };
#pragma unroll
      for (int qz = 0; qz < kR && qz < Q; qz++) load_plane(qz);
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
#pragma unroll
      for (int qz = 0; qz < Q; qz++) { // contract c, point factors, back over qz
         if (kR == 0) load_plane(qz);
         else if (qz + kR < Q) load_plane(qz + kR);
         if (KIND == TFEM_MASS) {
            double u = 0.0;
#pragma unroll
            for (int c = 0; c < D1; c++) u = fma(a.t.B[qz][c], UBB[c], u);
            const double w = u * Dq[0][qz];
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
            const double D00 = Dq[0][qz], D01 = Dq[1][qz], D02 = Dq[2][qz];
            const double D11 = Dq[3][qz], D12 = Dq[4][qz], D22 = Dq[5][qz];
            const double wx = fma(D02, uz, fma(D01, uy, D00 * ux));
            const double wy = fma(D12, uz, fma(D11, uy, D01 * ux));
            const double wz = fma(D22, uz, fma(D12, uy, D02 * ux));
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
   __syncthreads();
   // contract qy -> [c][b][qx] (x-gradient part in TB, rest in TG): a
   // thread per (c, qx)
   if (live) {
      for (int j = t; j < D1 * Q; j += NT) {
         const int jx = j % Q, c = j / Q;
         double px[Q], py[Q], pz[Q];
#pragma unroll
         for (int y = 0; y < Q; y++) {
            const int o = (c * Q + y) * Q + jx;
            px[y] = sm.Px[o];
            if (KIND == TFEM_DIFFUSION) {
               py[y] = sm.Py[o];
               pz[y] = sm.Pz[o];
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
            sm.TB[(c * D1 + b) * Q + jx] = sx;
            if (KIND == TFEM_DIFFUSION) sm.TG[(c * D1 + b) * Q + jx] = syz;
         }
      }
   }
   __syncthreads();
   double dot = 0.0;
   if (live) { // contract qx -> r(a, b, c): a thread per (c, b)
      for (int cb = t; cb < D1 * D1; cb += NT) {
         double tb[Q], tg[Q];
#pragma unroll
         for (int x = 0; x < Q; x++) {
            tb[x] = sm.TB[cb * Q + x];
            if (KIND == TFEM_DIFFUSION) tg[x] = sm.TG[cb * Q + x];
         }
#pragma unroll
         for (int ia = 0; ia < D1; ia++) {
            const int i = cb * D1 + ia;
            double r = 0.0;
#pragma unroll
            for (int x = 0; x < Q; x++) {
               if (KIND == TFEM_MASS) {
                  r = fma(a.t.B[x][ia], tb[x], r);
               } else {
                  r = fma(a.t.G[x][ia], tb[x], r);
                  r = fma(a.t.B[x][ia], tg[x], r);
               }
            }
            const uint32_t gg = __ldg(gm + i);
            if (is_exclusive(gg)) {
               const uint32_t d = gg & kDofMask;
               if (!a.overwrite) r += a.y[d];
               if (a.ess_out && bit_set(a.ess_out, d)) r = __ldg(a.x + d);
               a.y[d] = r;
               if (a.dot && !(a.notown && bit_set(a.notown, d))) dot = fma(__ldg(a.x + d), r, dot);
            } else {
               a.evec[ev_em_p(a.evperm, ND, e, i)] = r;
            }
         }
      }
   }
   if (a.dot) {
      const double v[1] = {dot};
      emit<NT * groups_for(NT), 1>(a.dot, v);
   }
}


template <int P, int Q, int KIND, bool EXACT>
void launch2d(const ApplyArgs &a, cudaStream_t s, unsigned blocks)
{
   constexpr int NT = round32(Q * Q), GR = groups_for(NT);
   const size_t smem = sizeof(Smem2D<P, Q>) * GR;
   if (smem > 48 * 1024) max_dynamic_smem((const void *)apply2d_grp_kernel<P, Q, KIND, EXACT>, smem);
   apply2d_grp_kernel<P, Q, KIND, EXACT><<<blocks, NT * GR, smem, s>>>(a);
}

template <int P, int Q, int KIND>
void launch3d(const ApplyArgs &a, cudaStream_t s, unsigned blocks)
{
   constexpr int NT = round32(Q * Q), GR = groups_for(NT);
   const size_t smem = sizeof(Smem3D<P, Q>) * GR;
   if (smem > 48 * 1024) max_dynamic_smem((const void *)apply3d_kernel<P, Q, KIND>, smem);
   apply3d_kernel<P, Q, KIND><<<blocks, NT * GR, smem, s>>>(a);
}

template <int P, int Q, int KIND>
KernelPick make2d(bool exact)
{
   KernelPick k;
   k.launch = exact ? launch2d<P, Q, KIND, true> : launch2d<P, Q, KIND, false>;
   k.elems_per_block = groups_for(round32(Q * Q));
   k.threads = round32(Q * Q) * k.elems_per_block;
   return k;
}

template <int P, int Q, int KIND>
KernelPick make3d()
{
   KernelPick k;
   k.launch = launch3d<P, Q, KIND>;
   k.elems_per_block = groups_for(round32(Q * Q));
   k.threads = round32(Q * Q) * k.elems_per_block;
   return k;
}

template <int P, int KIND>
KernelPick pick_q(int dim, int nq, bool exact)
{
   if (dim == 2) {
      if constexpr (P >= 4) { // lower orders use the register kernel
         if (nq == P + 2) return make2d<P, P + 2, KIND>(exact);
         if (nq == P + 1) return make2d<P, P + 1, KIND>(exact);
      }
   } else if constexpr (P <= kMaxP3D) {
      if (nq == P + 2) return make3d<P, P + 2, KIND>();
      if (nq == P + 1) return make3d<P, P + 1, KIND>();
   }
   return {};
}

template <int KIND>
KernelPick pick_p(int dim, int p, int nq, bool exact)
{
   switch (p) {
   case 1: return pick_q<1, KIND>(dim, nq, exact);
   case 2: return pick_q<2, KIND>(dim, nq, exact);
   case 3: return pick_q<3, KIND>(dim, nq, exact);
   case 4: return pick_q<4, KIND>(dim, nq, exact);
   case 5: return pick_q<5, KIND>(dim, nq, exact);
   case 6: return pick_q<6, KIND>(dim, nq, exact);
   case 7: return pick_q<7, KIND>(dim, nq, exact);
   case 8: return pick_q<8, KIND>(dim, nq, exact);
   // 2D p = 9..16: the generic shared-memory stages
   case 9: return pick_q<9, KIND>(dim, nq, exact);
   case 10: return pick_q<10, KIND>(dim, nq, exact);
   case 11: return pick_q<11, KIND>(dim, nq, exact);
   case 12: return pick_q<12, KIND>(dim, nq, exact);
   case 13: return pick_q<13, KIND>(dim, nq, exact);
   case 14: return pick_q<14, KIND>(dim, nq, exact);
   case 15: return pick_q<15, KIND>(dim, nq, exact);
   case 16: return pick_q<16, KIND>(dim, nq, exact);
   }
   return {};
}

} // namespace

KernelPick pick_apply_grp(int dim, int p, int nq, int kind, bool exact)
{
   return kind == TFEM_MASS ? pick_p<TFEM_MASS>(dim, p, nq, exact)
                            : pick_p<TFEM_DIFFUSION>(dim, p, nq, exact);
}

} // namespace tfem
