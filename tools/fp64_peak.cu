// FP64 roofline probe for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4)
// and DFMA issue-rate microbenchmarks. Prints one JSON object. Used once per pool to
// measure the FP64 denominators that MEASURED_PEAKS.json does not carry.
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void __launch_bounds__(256) dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int CHAINS>
__global__ void __launch_bounds__(256) dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-12, b = 0.999999;
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <typename K>
static float time_kernel(K kern, int grid, int block, double* out, int iters, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<grid, block>>>(out, iters);  // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    kern<<<grid, block>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 4096 * sizeof(double));
  const int iters = 20000;
  printf("{\"sms\": %d", sms);
  for (int bpsm : {1, 2, 4}) {
    for (int threads : {128, 256}) {
      const int grid = sms * bpsm;
      float ms = time_kernel(dmma_loop<8>, grid, threads, out, iters, 5);
      double fma = double(grid) * (threads / 32) * iters * 8.0 * 256.0;
      printf(", \"dmma_b%d_t%d_tflops\": %.3f", bpsm, threads, 2.0 * fma / (ms * 1e-3) / 1e12);
      float ms2 = time_kernel(dfma_loop<8>, grid, threads, out, iters, 5);
      double fma2 = double(grid) * threads * iters * 8.0;
      printf(", \"dfma_b%d_t%d_tflops\": %.3f", bpsm, threads, 2.0 * fma2 / (ms2 * 1e-3) / 1e12);
    }
  }
  printf(", \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
