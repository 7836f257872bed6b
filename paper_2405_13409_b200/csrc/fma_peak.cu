// FMA-throughput microbenchmark: the ALU roofline denominator for the FP64 solve kernels
// (independent FMA chains, >= 8 per thread, every SM).
#include "kernels.cuh"

namespace spoly {

template <typename T>
__global__ void __launch_bounds__(256) k_fma_peak(int iters, T a, T b, double* sink) {
  T x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = (T)(threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  T s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == (T)-1.2345) sink[0] = (double)s;  // never true; keeps the chains alive
}

void launch_fma_peak(int fp64, int iters, double* sink, int nsm, cudaStream_t st, int* blocks_out, int* threads_out,
                     int* flops_per_thread_iter) {
  const int threads = 256, blocks = nsm * 8;
  if (fp64)
    k_fma_peak<double><<<blocks, threads, 0, st>>>(iters, 0.999999, 1e-7, sink);
  else
    k_fma_peak<float><<<blocks, threads, 0, st>>>(iters, 0.999999f, 1e-7f, sink);
  *blocks_out = blocks;
  *threads_out = threads;
  *flops_per_thread_iter = 2 * 8 * 16;
}

}  // namespace spoly
