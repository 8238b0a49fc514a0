// Dependent-chain latencies on sm_100a for the instructions on the panel leaf's per-column critical
// path (one warp, clock64 around N dependent operations); prints cycles per operation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_probe tools/lat_probe.cu && tools/lat_probe
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
constexpr int N = 2048;

__global__ void probe(double* out, long long* cyc, double seed) {
  __shared__ double sm[64];
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 64) sm[threadIdx.x] = seed + threadIdx.x;
  __syncthreads();
  double x = seed + lane * 1e-3, y = 1.0000001;
  long long t0, t1;
  int k = 0;
  // DFMA
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = fma(x, y, 1e-9);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[k] = t1 - t0;
  ++k;
  // DMUL
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x * y;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[k] = t1 - t0;
  ++k;
  // DADD
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x + y;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[k] = t1 - t0;
  ++k;
  // double division
  x = 1.5 + lane;
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N / 8; ++i) x = 1.0000001 / x + 0.5;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[k] = (t1 - t0) * 8;
  ++k;
  // shuffle (64-bit = 2 SHFL)
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1e-12;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[k] = t1 - t0;
  ++k;
  // redux max (u32)
  unsigned u = (unsigned)lane + (unsigned)x;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) u = __reduce_max_sync(0xffffffffu, u + lane) + 1u;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[k] = t1 - t0;
  ++k;
  // LDS chain (pointer chase through shared memory)
  int idx = lane;
  __shared__ int chase[64];
  if (threadIdx.x < 64) chase[threadIdx.x] = (threadIdx.x * 7 + 3) & 63;
  __syncthreads();
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) idx = chase[idx];
  t1 = clock64();
  if (threadIdx.x == 0) cyc[k] = t1 - t0;
  ++k;
  // __syncthreads with the whole CTA
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < N / 8; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) cyc[k] = (t1 - t0) * 8;
  ++k;
  // FP64 compare + select chain (the argmax step)
  double b = x;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) b = (b > y) ? b - 1e-9 : b + 1e-9;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[k] = t1 - t0;
  ++k;
  out[threadIdx.x] = x + u + idx + b;
}

__global__ void __cluster_dims__(8, 1, 1) cluster_probe(long long* cyc, int* sink) {
  __shared__ int v[32];
  cg::cluster_group cl = cg::this_cluster();
  v[threadIdx.x & 31] = threadIdx.x;
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = (t1 - t0) * (N / 256);
  // DSMEM dependent loads
  int* remote = cl.map_shared_rank(v, (cl.block_rank() + 1) % 8);
  int idx = threadIdx.x & 31;
  t0 = clock64();
  for (int i = 0; i < 256; ++i) idx = remote[idx & 31] & 31;
  t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[1] = (t1 - t0) * (N / 256);
  cl.sync();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = idx;
}

int main() {
  double* out;
  long long *cyc, h[16] = {0};
  int* sink;
  cudaMalloc(&out, 4096 * sizeof(double));
  cudaMalloc(&cyc, 16 * sizeof(long long));
  cudaMalloc(&sink, 8 * 512 * sizeof(int));
  const char* names[] = {"DFMA", "DMUL", "DADD", "double division", "64-bit shuffle + DADD", "REDUX.MAX u32 + IADD",
                         "LDS pointer chase", "__syncthreads (512 threads)", "DSETP + select + DADD"};
  for (int threads : {32, 512}) {
    for (int rep = 0; rep < 2; ++rep) probe<<<1, threads>>>(out, cyc, 1.25);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("threads per CTA = %d\n", threads);
    for (int k = 0; k < 9; ++k) printf("  %-32s %7.1f cycles\n", names[k], (double)h[k] / N);
  }
  for (int rep = 0; rep < 2; ++rep) cluster_probe<<<8, 512>>>(cyc, sink);
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  printf("cluster of 8 x 512 threads\n  %-32s %7.1f cycles\n  %-32s %7.1f cycles\n", "cluster.sync", (double)h[0] / N,
         "DSMEM dependent load", (double)h[1] / N);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
