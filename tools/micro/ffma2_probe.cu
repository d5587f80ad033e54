// FP32 FMA throughput probe: scalar FFMA vs packed FFMA2 (sm_100a), 8 independent chains
// per thread, 148*8 blocks of 256 threads.  Prints G FMA/s for each.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void scalar_k(float* out, float a, float b, int iters) {
  float x[8];
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], a, b);
  float s = 0; for (int j = 0; j < 8; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void packed_k(float* out, float a, float b, int iters) {
  float2 x[4];
  for (int j = 0; j < 4; ++j) x[j] = make_float2(threadIdx.x + j, threadIdx.x - j);
  const float2 A = make_float2(a, a), B = make_float2(b, b);
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = __ffma2_rn(x[j], A, B);
  float s = 0; for (int j = 0; j < 4; ++j) s += x[j].x + x[j].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* d; cudaMalloc(&d, 148 * 8 * 256 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0); scalar_k<<<148 * 8, 256>>>(d, 0.999f, 0.001f, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fmas = 148.0 * 8 * 256 * 8 * iters;
    printf("FFMA : %.1f G FMA/s\n", fmas / ms / 1e6);
    cudaEventRecord(e0); packed_k<<<148 * 8, 256>>>(d, 0.999f, 0.001f, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA2: %.1f G FMA/s\n", fmas / ms / 1e6);
  }
  return 0;
}
