#include <cstdio>
__global__ void kd(double* out, int iters) {
  double acc[8][2] = {};
  double x = threadIdx.x * 0.5, y = threadIdx.x * 0.25;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(acc[j][0]), "+d"(acc[j][1]) : "d"(x), "d"(y));
  }
  double s = 0;
  for (int j = 0; j < 8; ++j) s += acc[j][0] + acc[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void kf(double* out, int iters) {
  double acc[16] = {};
  double x = threadIdx.x * 0.5, y = threadIdx.x * 0.25;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = fma(x, y, acc[j]);
    x += 1e-9;
  }
  double s = 0;
  for (int j = 0; j < 16; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* o; cudaMalloc(&o, 148 * 8 * 1024 * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    int iters = 4096;
    cudaEventRecord(a); kd<<<148 * 4, 256>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double flops = 148.0 * 4 * 8 * iters * 8 * 512;  // warps*iters*8 mma*512 flop
    printf("DMMA: %.2f ms  %.1f TFLOP/s\n", ms, flops / ms / 1e9);
    cudaEventRecord(a); kf<<<148 * 4, 256>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    flops = 148.0 * 4 * 256 * iters * 16 * 2;
    printf("DFMA: %.2f ms  %.1f TFLOP/s\n", ms, flops / ms / 1e9);
  }
}
