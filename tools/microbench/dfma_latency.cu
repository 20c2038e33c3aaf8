// FP64 pipe microbenchmark for sm_100a: dependent-chain latency and
// throughput of DFMA vs. the number of independent chains per thread and
// warps per SMSP.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dfma dfma_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void chain(double* out, long long* cyc, int iters, double a, double b) {
  double x[C];
#pragma unroll
  for (int k = 0; k < C; ++k) x[k] = threadIdx.x * 1e-3 + k;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int k = 0; k < C; ++k) x[k] = fma(x[k], a, b);
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < C; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int C>
void run(int warps_per_smsp, int sms) {
  const int threads = 128 * warps_per_smsp;  // 4 SMSPs
  const int iters = 4096;
  double* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(double) * sms * threads);
  cudaMalloc(&cyc, sizeof(long long) * sms);
  chain<C><<<sms, threads>>>(out, cyc, 16, 0.9999999, 1e-7);
  chain<C><<<sms, threads>>>(out, cyc, iters, 0.9999999, 1e-7);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  const double dfma_per_thread = 8.0 * iters * C;
  const double warp_dfma_per_smsp = dfma_per_thread * warps_per_smsp;
  printf("chains/thread %2d warps/SMSP %2d: %.2f cycles per dependent DFMA, %.3f warp-DFMA/clk/SMSP\n",
         C, warps_per_smsp, avg / (8.0 * iters), warp_dfma_per_smsp / avg);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {1, 2, 4, 8}) {
    run<1>(w, sms);
    run<2>(w, sms);
    run<4>(w, sms);
    run<8>(w, sms);
  }
  return 0;
}
