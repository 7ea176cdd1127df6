// Diagnostics: the CUDA-core FP64 (DFMA) peak of this device, measured, for
// the FP64 side of the element kernels' roofline (bench.py "fp64").  Not on
// the reference path; no reference counterpart.
#include "kernels.cuh"

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

} // namespace

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
