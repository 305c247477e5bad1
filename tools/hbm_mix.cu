// HBM bandwidth by read:write mix (the practical roofline of a kernel that reads R bytes and writes
// W bytes, e.g. lm_kernel: 1.5 GB of xhat read, 3.3 GB of trace written at C4).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hbm_mix tools/hbm_mix.cu && tools/hbm_mix
// Each thread streams 16-byte vectors: every read vector is followed by `wpr` written vectors
// (streaming stores), grid = 148 x 8 CTAs of 256 threads, grid-stride; best of 10 (CUDA events).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void mix(const int4* __restrict__ src, int64_t nr, int4* __restrict__ dst, int64_t nw, int wpr) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (nr == 0) {  // write only
    for (; i < nw; i += stride) __stcs(dst + i, make_int4(1, 2, 3, static_cast<int>(i)));
    return;
  }
  int acc = 0;
  for (; i < nr; i += stride) {
    const int4 v = __ldcs(src + i);
    acc ^= v.x ^ v.w;
    for (int w = 0; w < wpr; ++w) {
      const int64_t j = i + w * nr;
      if (j < nw) __stcs(dst + j, v);
    }
  }
  if (acc == 0x7fffffff) dst[0] = make_int4(acc, 0, 0, 0);
}

int main() {
  const int64_t R = 1536ll << 20, W = 3072ll << 20;  // bytes
  int4 *s, *d;
  cudaMalloc(&s, R);
  cudaMalloc(&d, W);
  cudaMemset(s, 1, R);
  cudaMemset(d, 0, W);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct Case { const char* name; int64_t r, w; int wpr; } cases[] = {
      {"read only (1:0)", R, 0, 0}, {"write only (0:1)", 0, W, 0}, {"copy (1:1)", R, R, 1}, {"1:2 (lm_kernel mix)", R, W, 2},
  };
  for (auto& c : cases) {
    float best = 1e30f;
    for (int it = 0; it < 10; ++it) {
      cudaEventRecord(a);
      mix<<<148 * 8, 256>>>(s, c.r / 16, d, c.w / 16, c.wpr);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%-22s read %.2f GB write %.2f GB  %.3f ms  %.0f GB/s\n", c.name, c.r / 1e9, c.w / 1e9, best,
           (c.r + c.w) / 1e6 / best);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
