// K2, 2D low order: one thread per element, the whole sum-factorised chain
// in registers (forms.cpp:248-286, tensor_kernels.cpp:67-110).
//
// qdata planes [(c*nqd+q)][ne_pad] and the slot-major element map make every
// load a coalesced 256-byte warp access; B1d/G1d live in the kernel-parameter
// constant bank and are read as DMUL / DFMA operands (all indices are
// compile-time after unrolling, so the reads are warp-uniform).  EXACT=true
// evaluates every product and sum in the reference's order with unfused
// round-to-nearest operations -- bit-identical to the CPU reference;
// EXACT=false fuses multiply-adds.
#include "kernels.cuh"

namespace tfem {

namespace {

template <int P, int Q, int KIND, bool EXACT>
__global__ void __launch_bounds__(kElemThreads2D) apply2d_kernel(const ApplyArgs a)
{
   constexpr int D1 = P + 1;
   constexpr int ND = D1 * D1;
   constexpr int NQD = Q * Q;
   if (a.done && *a.done) return;
   const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
   double dot = 0.0;
   if (e < a.ne) {
      uint32_t dof[ND];
      double V[D1][D1]; // V[a][b] = x[dofs[b*D1 + a]] (forms.cpp:250-255)
#pragma unroll
      for (int i = 0; i < ND; i++) dof[i] = __ldg(a.gmap + i * a.ne_pad + e);
#pragma unroll
      for (int i = 0; i < ND; i++) {
         const uint32_t d = dof[i] & kDofMask;
         double v = __ldg(a.x + d);
         if (a.mask_in && bit_set(a.mask_in, d)) v = 0.0;
         V[i % D1][i / D1] = v;
      }
      const double *qd = a.qdata + e;
      const int64_t pl = a.ne_pad;
      double R[D1][D1]; // result r(a,b)
      if (KIND == TFEM_DIFFUSION) {
         // T1 = G V, T2 = B V (x contracted first; tensor_kernels.cpp:84-85)
         double T1[Q][D1], T2[Q][D1];
#pragma unroll
         for (int qx = 0; qx < Q; qx++)
#pragma unroll
            for (int b = 0; b < D1; b++) {
               double s1 = mul<EXACT>(a.t.G[qx][0], V[0][b]);
               double s2 = mul<EXACT>(a.t.B[qx][0], V[0][b]);
#pragma unroll
               for (int k = 1; k < D1; k++) {
                  s1 = mac<EXACT>(s1, a.t.G[qx][k], V[k][b]);
                  s2 = mac<EXACT>(s2, a.t.B[qx][k], V[k][b]);
               }
               T1[qx][b] = s1;
               T2[qx][b] = s2;
            }
         double vx[D1][D1], vy[D1][D1];
#pragma unroll
         for (int qy = 0; qy < Q; qy++) {
            double wx[Q], wy[Q];
#pragma unroll
            for (int qx = 0; qx < Q; qx++) {
               // dx = T1 B^t, dy = T2 G^t at (qx, qy) (mat_mult_nt)
               double dx = mul<EXACT>(T1[qx][0], a.t.B[qy][0]);
               double dy = mul<EXACT>(T2[qx][0], a.t.G[qy][0]);
#pragma unroll
               for (int b = 1; b < D1; b++) {
                  dx = mac<EXACT>(dx, T1[qx][b], a.t.B[qy][b]);
                  dy = mac<EXACT>(dy, T2[qx][b], a.t.G[qy][b]);
               }
               const int q = qy * Q + qx;
               const double d0 = __ldg(qd + (0 * NQD + q) * pl);
               const double d1 = __ldg(qd + (1 * NQD + q) * pl);
               const double d2 = __ldg(qd + (2 * NQD + q) * pl);
               // forms.cpp:274-275
               wx[qx] = add<EXACT>(mul<EXACT>(d0, dx), mul<EXACT>(d1, dy));
               wy[qx] = add<EXACT>(mul<EXACT>(d1, dx), mul<EXACT>(d2, dy));
            }
            // S = G^t Wx, B^t Wy over qx (mat_mult_tn), then += S B, S G over qy
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
                  if (qy == 0) {
                     vx[i][b] = mul<EXACT>(sx, a.t.B[0][b]);
                     vy[i][b] = mul<EXACT>(sy, a.t.G[0][b]);
                  } else {
                     vx[i][b] = mac<EXACT>(vx[i][b], sx, a.t.B[qy][b]);
                     vy[i][b] = mac<EXACT>(vy[i][b], sy, a.t.G[qy][b]);
                  }
               }
            }
         }
#pragma unroll
         for (int i = 0; i < D1; i++)
#pragma unroll
            for (int b = 0; b < D1; b++) R[i][b] = add<EXACT>(vx[i][b], vy[i][b]);
      } else {
         // mass: B V B^t, scale, B^t Q B (tensor_kernels.cpp:67-74, 89-97)
         double T[Q][D1];
#pragma unroll
         for (int qx = 0; qx < Q; qx++)
#pragma unroll
            for (int b = 0; b < D1; b++) {
               double s = mul<EXACT>(a.t.B[qx][0], V[0][b]);
#pragma unroll
               for (int k = 1; k < D1; k++) s = mac<EXACT>(s, a.t.B[qx][k], V[k][b]);
               T[qx][b] = s;
            }
#pragma unroll
         for (int qy = 0; qy < Q; qy++) {
            double w[Q];
#pragma unroll
            for (int qx = 0; qx < Q; qx++) {
               double u = mul<EXACT>(T[qx][0], a.t.B[qy][0]);
#pragma unroll
               for (int b = 1; b < D1; b++) u = mac<EXACT>(u, T[qx][b], a.t.B[qy][b]);
               w[qx] = mul<EXACT>(u, __ldg(qd + (qy * Q + qx) * pl));
            }
#pragma unroll
            for (int i = 0; i < D1; i++) {
               double s = mul<EXACT>(a.t.B[0][i], w[0]);
#pragma unroll
               for (int qx = 1; qx < Q; qx++) s = mac<EXACT>(s, a.t.B[qx][i], w[qx]);
#pragma unroll
               for (int b = 0; b < D1; b++)
                  R[i][b] = qy == 0 ? mul<EXACT>(s, a.t.B[0][b]) : mac<EXACT>(R[i][b], s, a.t.B[qy][b]);
            }
         }
      }
      // out[b*D1 + a] = r(a, b) (forms.cpp:281-286)
#pragma unroll
      for (int i = 0; i < ND; i++) {
         const uint32_t g = dof[i];
         double r = R[i % D1][i / D1];
         if (is_exclusive(g)) {
            const uint32_t d = g & kDofMask;
            if (!a.overwrite) r = add<EXACT>(a.y[d], r);
            if (a.ess_out && bit_set(a.ess_out, d)) r = __ldg(a.x + d);
            a.y[d] = r;
            if (a.dot && !(a.notown && bit_set(a.notown, d)))
               dot = mac<EXACT>(dot, __ldg(a.x + d), r);
         } else {
            a.evec[i * a.ne_pad + e] = r;
         }
      }
   }
   if (a.dot) {
      const double v[1] = {dot};
      emit<kElemThreads2D, 1>(a.dot, v);
   }
}


template <int P, int Q, int KIND, bool EXACT>
void launch2d(const ApplyArgs &a, cudaStream_t s, unsigned blocks)
{
   apply2d_kernel<P, Q, KIND, EXACT><<<blocks, kElemThreads2D, 0, s>>>(a);
}

template <int P, int KIND>
Launch pick_q(int nq, bool exact)
{
   if (nq == P + 2) return exact ? launch2d<P, P + 2, KIND, true> : launch2d<P, P + 2, KIND, false>;
   if (nq == P + 1) return exact ? launch2d<P, P + 1, KIND, true> : launch2d<P, P + 1, KIND, false>;
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

KernelPick pick_apply2d_reg(int p, int nq, int kind, bool exact)
{
   KernelPick k;
   k.launch = kind == TFEM_MASS ? pick_p<TFEM_MASS>(p, nq, exact)
                                : pick_p<TFEM_DIFFUSION>(p, nq, exact);
   k.elems_per_block = kElemThreads2D;
   k.threads = kElemThreads2D;
   return k;
}

} // namespace tfem
