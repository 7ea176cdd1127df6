// Diagnostics: the CUDA-core FP64 (DFMA) peak of this device, measured, for
// the FP64 side of the element kernels' roofline (bench.py "fp64").  Not on
// the reference path; no reference counterpart.
#include "kernels.cuh"

#include <algorithm>
#include <cmath>
#include <vector>

namespace tfem {

namespace {

constexpr int kChains = 8;   // independent DFMA chains per thread (hides the DFMA latency)
constexpr int kIters = 2048; // DFMAs per chain per launch

__global__ void __launch_bounds__(256) dfma_kernel(double *sink, double seed)
{
   double c[kChains];
#pragma unroll
   for (int i = 0; i < kChains; i++) c[i] = seed + 1e-3 * (threadIdx.x + i);
   const double m = 1.0 - 1e-12 * seed, k = 1e-9 * seed;
   for (int it = 0; it < kIters; it++) {
#pragma unroll
      for (int i = 0; i < kChains; i++) c[i] = fma(c[i], m, k);
   }
   double s = 0.0;
#pragma unroll
   for (int i = 0; i < kChains; i++) s += c[i];
   if (s == 123.456) sink[blockIdx.x] = s; // never true: keeps the chains live
}

// FP64 tensor-core (DMMA) throughput: mma.sync m8n8k4 f64, kChains
// independent accumulators per warp (north_star: DMMA only where it beats
// the CUDA-core DFMA path; this is the ceiling it would have).
__global__ void __launch_bounds__(256) dmma_kernel(double *sink, double seed)
{
   const int lane = threadIdx.x & 31;
   double a = seed + 1e-3 * lane, b = 1.0 - 1e-12 * seed;
   double c[kChains][2];
#pragma unroll
   for (int i = 0; i < kChains; i++) c[i][0] = c[i][1] = 1e-3 * i;
   for (int it = 0; it < kIters / 4; it++) {
#pragma unroll
      for (int i = 0; i < kChains; i++)
         asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                      : "+d"(c[i][0]), "+d"(c[i][1])
                      : "d"(a), "d"(b));
   }
   double s = 0.0;
#pragma unroll
   for (int i = 0; i < kChains; i++) s += c[i][0] + c[i][1];
   if (s == 123.456) sink[blockIdx.x] = s;
}

template <typename K>
double measure(tfem_ctx *ctx, K kernel, double flops_per_launch, unsigned grid)
{
   double *sink = nullptr;
   cuda_check(cudaMallocAsync(&sink, sizeof(double) * 64 * 1024, ctx->stream), "fp64_peak");
   cudaEvent_t e0, e1;
   cuda_check(cudaEventCreate(&e0), "fp64_peak");
   cuda_check(cudaEventCreate(&e1), "fp64_peak");
   kernel<<<grid, 256, 0, ctx->stream>>>(sink, 1.0); // warm-up
   ctx->launched();
   double best = 0.0;
   for (int rep = 0; rep < 5; rep++) {
      cuda_check(cudaEventRecord(e0, ctx->stream), "fp64_peak");
      for (int l = 0; l < 4; l++) kernel<<<grid, 256, 0, ctx->stream>>>(sink, 1.0 + rep);
      ctx->launched(4);
      cuda_check(cudaEventRecord(e1, ctx->stream), "fp64_peak");
      cuda_check(cudaEventSynchronize(e1), "fp64_peak");
      float ms = 0.f;
      cuda_check(cudaEventElapsedTime(&ms, e0, e1), "fp64_peak");
      const double tf = 4.0 * flops_per_launch / (ms * 1e-3) / 1e12;
      if (tf > best) best = tf;
   }
   cuda_check(cudaGetLastError(), "fp64_peak");
   cudaEventDestroy(e0);
   cudaEventDestroy(e1);
   cuda_check(cudaFreeAsync(sink, ctx->stream), "fp64_peak");
   return best;
}

// ----------------------------------------------------- contraction A/B
// The 1D sum-factorisation stage every element kernel is built from, at the
// 3D orders where DMMA could pay (north_star: DMMA only if it beats DFMA for
// the contraction at that order): per element, X [K = p+1][N = (p+1)^2]
// (the element's x as [a][bc]) -> Y1 = B X, Y2 = G X ([Q][N], B/G = q x
// (p+1)), the x stage of the forward pass.  Both variants run on shared-
// memory-resident elements (no HBM traffic: the compute ceiling alone),
// `kReps` passes over kElems elements per block; useful flops = 2 * 2 Q K N
// per element.
constexpr int kAbThreads = 256;
constexpr int kAbElems = 8; // elements resident per block
constexpr int kAbReps = 64; // passes over them per launch

template <int P>
struct AbDims {
   static constexpr int K = P + 1, N = K * K, Q = P + 2;
   static constexpr int Mp = (Q + 7) / 8 * 8, Kp = (K + 3) / 4 * 4, Np = (N + 7) / 8 * 8;
   static constexpr int S = Np + 4 + ((Np + 4) % 16 == 4 || (Np + 4) % 16 == 12 ? 0 : 4); // X row stride
};

template <int P>
__device__ void ab_fill(double *X, int e)
{
   using D = AbDims<P>;
   for (int j = threadIdx.x; j < D::Kp * D::S; j += blockDim.x) {
      const int k = j / D::S, n = j % D::S;
      X[j] = (k < D::K && n < D::N) ? 1.0 / (1.0 + k + 0.37 * n + 0.11 * e) : 0.0;
   }
}

// DFMA: a thread per column n, the column in registers, basis operands from
// the constant bank (compile-time indices) -- the element kernels' form.
template <int P>
__global__ void __launch_bounds__(kAbThreads) ab_dfma_kernel(const Tables t, double *out, double *sink)
{
   using D = AbDims<P>;
   extern __shared__ double ab_smem[];
   auto X = reinterpret_cast<double (*)[D::Kp * D::S]>(ab_smem);
   auto Y = reinterpret_cast<double (*)[2][D::Q * D::N]>(ab_smem + kAbElems * D::Kp * D::S);
   for (int e = 0; e < kAbElems; e++) ab_fill<P>(X[e], e + blockIdx.x);
   __syncthreads();
   for (int rep = 0; rep < kAbReps; rep++) {
      // (element, column) work items spread over the block
      for (int w = threadIdx.x; w < kAbElems * D::N; w += kAbThreads) {
         const int e = w / D::N, n = w % D::N;
         double x[D::K];
#pragma unroll
         for (int k = 0; k < D::K; k++) x[k] = X[e][k * D::S + n];
#pragma unroll
         for (int m = 0; m < D::Q; m++) {
            double y1 = 0.0, y2 = 0.0;
#pragma unroll
            for (int k = 0; k < D::K; k++) {
               y1 = fma(t.B[m][k], x[k], y1);
               y2 = fma(t.G[m][k], x[k], y2);
            }
            Y[e][0][m * D::N + n] = y1;
            Y[e][1][m * D::N + n] = y2;
         }
      }
      __syncthreads();
   }
   if (blockIdx.x == 0)
      for (int j = threadIdx.x; j < 2 * D::Q * D::N; j += blockDim.x) out[j] = Y[0][j / (D::Q * D::N)][j % (D::Q * D::N)];
   if (threadIdx.x == 0 && Y[kAbElems - 1][1][0] == 123.456) sink[blockIdx.x] = 1.0;
}

// DMMA: a warp per element, mma.sync m8n8k4 f64 tiles over the padded
// [Mp x Kp] basis and [Kp x Np] element; the basis fragments stay in
// registers, X fragments come from shared memory (row stride S = 4 mod 16
// doubles: conflict-free), Y tiles go back to shared memory.
template <int P>
__global__ void __launch_bounds__(kAbThreads) ab_dmma_kernel(const Tables t, double *out, double *sink)
{
   using D = AbDims<P>;
   constexpr int MT = D::Mp / 8, KT = D::Kp / 4, NT = D::Np / 8;
   extern __shared__ double ab_smem[];
   auto X = reinterpret_cast<double (*)[D::Kp * D::S]>(ab_smem);
   auto Y = reinterpret_cast<double (*)[2][D::Q * D::N]>(ab_smem + kAbElems * D::Kp * D::S);
   for (int e = 0; e < kAbElems; e++) ab_fill<P>(X[e], e + blockIdx.x);
   const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
   const int r = lane >> 2, c4 = lane & 3;
   double aB[MT][KT], aG[MT][KT];
#pragma unroll
   for (int mt = 0; mt < MT; mt++)
#pragma unroll
      for (int kt = 0; kt < KT; kt++) {
         const int m = mt * 8 + r, k = kt * 4 + c4;
         aB[mt][kt] = (m < D::Q && k < D::K) ? t.B[m][k] : 0.0;
         aG[mt][kt] = (m < D::Q && k < D::K) ? t.G[m][k] : 0.0;
      }
   __syncthreads();
   for (int rep = 0; rep < kAbReps; rep++) {
      for (int e = warp; e < kAbElems; e += kAbThreads / 32) {
         const double *Xe = X[e];
#pragma unroll
         for (int nt = 0; nt < NT; nt++) {
            double b[KT];
#pragma unroll
            for (int kt = 0; kt < KT; kt++) b[kt] = Xe[(kt * 4 + c4) * D::S + nt * 8 + r];
#pragma unroll
            for (int mt = 0; mt < MT; mt++) {
               double c1[2] = {0.0, 0.0}, c2[2] = {0.0, 0.0};
#pragma unroll
               for (int kt = 0; kt < KT; kt++) {
                  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                               : "+d"(c1[0]), "+d"(c1[1])
                               : "d"(aB[mt][kt]), "d"(b[kt]));
                  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                               : "+d"(c2[0]), "+d"(c2[1])
                               : "d"(aG[mt][kt]), "d"(b[kt]));
               }
               const int m = mt * 8 + r, n = nt * 8 + 2 * c4;
               if (m < D::Q) {
#pragma unroll
                  for (int h = 0; h < 2; h++)
                     if (n + h < D::N) {
                        Y[e][0][m * D::N + n + h] = c1[h];
                        Y[e][1][m * D::N + n + h] = c2[h];
                     }
               }
            }
         }
      }
      __syncthreads();
   }
   if (blockIdx.x == 0)
      for (int j = threadIdx.x; j < 2 * D::Q * D::N; j += blockDim.x) out[j] = Y[0][j / (D::Q * D::N)][j % (D::Q * D::N)];
   if (threadIdx.x == 0 && Y[kAbElems - 1][1][0] == 123.456) sink[blockIdx.x] = 1.0;
}

template <int P>
void contraction_ab_p(tfem_ctx *ctx, const Tables &t, double *res)
{
   using D = AbDims<P>;
   const unsigned grid = static_cast<unsigned>(ctx->sm_count) * 4u;
   const int ny = 2 * D::Q * D::N;
   double *buf = nullptr;
   cuda_check(cudaMallocAsync(&buf, sizeof(double) * (2 * ny + grid), ctx->stream), "contraction_ab");
   cudaEvent_t e0, e1;
   cuda_check(cudaEventCreate(&e0), "contraction_ab");
   cuda_check(cudaEventCreate(&e1), "contraction_ab");
   const double flops = 4.0 * D::Q * D::K * D::N * kAbElems * kAbReps * (double)grid;
   const size_t smem = sizeof(double) * kAbElems * (D::Kp * D::S + 2 * D::Q * D::N);
   max_dynamic_smem((const void *)ab_dfma_kernel<P>, smem);
   max_dynamic_smem((const void *)ab_dmma_kernel<P>, smem);
   auto time = [&](auto kern, double *out) {
      kern<<<grid, kAbThreads, smem, ctx->stream>>>(t, out, buf + 2 * ny); // warm-up
      ctx->launched();
      double best = 1e30;
      for (int rep = 0; rep < 5; rep++) {
         cuda_check(cudaEventRecord(e0, ctx->stream), "contraction_ab");
         kern<<<grid, kAbThreads, smem, ctx->stream>>>(t, out, buf + 2 * ny);
         ctx->launched();
         cuda_check(cudaEventRecord(e1, ctx->stream), "contraction_ab");
         cuda_check(cudaEventSynchronize(e1), "contraction_ab");
         float ms = 0.f;
         cuda_check(cudaEventElapsedTime(&ms, e0, e1), "contraction_ab");
         best = std::min(best, static_cast<double>(ms));
      }
      return best;
   };
   const double ms_f = time(ab_dfma_kernel<P>, buf);
   const double ms_m = time(ab_dmma_kernel<P>, buf + ny);
   std::vector<double> h(2 * ny);
   d2h(ctx->stream, h.data(), buf, sizeof(double) * h.size());
   double dmax = 0.0, ymax = 0.0;
   for (int j = 0; j < ny; j++) {
      dmax = std::max(dmax, std::abs(h[j] - h[ny + j]));
      ymax = std::max(ymax, std::abs(h[j]));
   }
   res[0] = flops / (ms_f * 1e-3) / 1e12;
   res[1] = flops / (ms_m * 1e-3) / 1e12;
   res[2] = dmax / std::max(ymax, 1e-300);
   res[3] = (double)D::Mp * D::Kp * D::Np / ((double)D::Q * D::K * D::N); // DMMA padding factor
   cuda_check(cudaGetLastError(), "contraction_ab");
   cudaEventDestroy(e0);
   cudaEventDestroy(e1);
   cuda_check(cudaFreeAsync(buf, ctx->stream), "contraction_ab");
}

} // namespace

void contraction_ab(tfem_ctx *ctx, int p, double *res)
{
   if (p < 2 || p > 8) invalid("contraction_ab: order must be in [2, 8]");
   // GLL-like synthetic tables (values only shape the arithmetic)
   Tables t{};
   for (int m = 0; m < p + 2; m++)
      for (int k = 0; k <= p; k++) {
         t.B[m][k] = 1.0 / (1.0 + m + 2.0 * k);
         t.G[m][k] = (m - k) / (3.0 + m + k);
      }
   switch (p) {
   case 2: return contraction_ab_p<2>(ctx, t, res);
   case 3: return contraction_ab_p<3>(ctx, t, res);
   case 4: return contraction_ab_p<4>(ctx, t, res);
   case 5: return contraction_ab_p<5>(ctx, t, res);
   case 6: return contraction_ab_p<6>(ctx, t, res);
   case 7: return contraction_ab_p<7>(ctx, t, res);
   case 8: return contraction_ab_p<8>(ctx, t, res);
   }
}

double dmma_peak_tflops(tfem_ctx *ctx)
{
   const unsigned grid = static_cast<unsigned>(ctx->sm_count) * 8u;
   // one m8n8k4 = 8 * 8 * 4 multiply-adds per warp = 512 flops
   const double flops = static_cast<double>(grid) * (256 / 32) * kChains * (kIters / 4) * 512.0;
   return measure(ctx, dmma_kernel, flops, grid);
}

double fp64_peak_tflops(tfem_ctx *ctx)
{
   double *sink = nullptr;
   cuda_check(cudaMallocAsync(&sink, sizeof(double) * 64 * 1024, ctx->stream), "fp64_peak");
   const unsigned grid = static_cast<unsigned>(ctx->sm_count) * 8u;
   cudaEvent_t e0, e1;
   cuda_check(cudaEventCreate(&e0), "fp64_peak");
   cuda_check(cudaEventCreate(&e1), "fp64_peak");
   dfma_kernel<<<grid, 256, 0, ctx->stream>>>(sink, 1.0); // warm-up
   ctx->launched();
   double best = 0.0;
   for (int rep = 0; rep < 5; rep++) {
      cuda_check(cudaEventRecord(e0, ctx->stream), "fp64_peak");
      for (int l = 0; l < 4; l++) dfma_kernel<<<grid, 256, 0, ctx->stream>>>(sink, 1.0 + rep);
      ctx->launched(4);
      cuda_check(cudaEventRecord(e1, ctx->stream), "fp64_peak");
      cuda_check(cudaEventSynchronize(e1), "fp64_peak");
      float ms = 0.f;
      cuda_check(cudaEventElapsedTime(&ms, e0, e1), "fp64_peak");
      const double flops = 4.0 * grid * 256.0 * kChains * kIters * 2.0;
      const double tf = flops / (ms * 1e-3) / 1e12;
      if (tf > best) best = tf;
   }
   cuda_check(cudaGetLastError(), "fp64_peak");
   cudaEventDestroy(e0);
   cudaEventDestroy(e1);
   cuda_check(cudaFreeAsync(sink, ctx->stream), "fp64_peak");
   return best;
}

} // namespace tfem
