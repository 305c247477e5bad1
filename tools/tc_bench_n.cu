// tc_bench_n.cu -- microbenchmark: tcgen05.mma.kind::i8 cycles per instruction vs N (M = 128,
// K = 32), with one accumulator (dependent chain) or NACC rotating accumulators (bring-up tool).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include "../paper_2603_03065_b200/csrc/tc_common.cuh"
using namespace v3db;

__device__ __forceinline__ void mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}

// the whole warp runs the issue loop (operands warp-uniform); one elected lane issues each MMA
template <int N>
__global__ void __launch_bounds__(128, 1) mma_bench_warp(int nmma, int nacc, int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + 16384;
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < (16384 + 32768) / 16; i += 128) reinterpret_cast<uint4*>(smem)[i] = make_uint4(i, i, i, i);
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::mbar_fence_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc(&tslot, 512);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tslot;
  if (threadIdx.x < 32) {
    constexpr uint32_t idesc = tc::idesc_s8(128, N);
    const uint64_t da = tc::desc_sw128(tc::smem_u32(sA)), db = tc::desc_sw128(tc::smem_u32(sB));
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      for (int k = 0; k < nmma; ++k) {
        if (elect_one()) tc::mma_s8(tmem + (k % nacc) * N, da + 2 * (k & 3), db + 2 * (k & 3), idesc, k >= nacc);
        __syncwarp();
      }
      if (elect_one()) tc::mma_commit(&bar);
      __syncwarp();
      tc::mbar_wait(&bar, r & 1);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 512);
}

template <int N>
void run_warp(long long* d) {
  cudaFuncSetAttribute(mma_bench_warp<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024);
  for (int nacc : {1, 5}) {
    if (nacc * N > 512) continue;
    const int nmma = 40, reps = 200;
    mma_bench_warp<N><<<148, 128, 50 * 1024>>>(nmma, nacc, reps, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h = 0;
    cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("warp-issue A:smem N %3d nacc %d: %.1f cycles per MMA (%.1f floor) %s\n", N, nacc,
           (double)h / reps / nmma, 128.0 * N / 256, cudaGetErrorString(e));
  }
}

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) mma_bench(int nmma, int nacc, int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;             // 16 KB
  uint8_t* sB = smem + 16384;     // 32 KB
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < (16384 + 32768) / 16; i += 128) reinterpret_cast<uint4*>(smem)[i] = make_uint4(i, i, i, i);
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::mbar_fence_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc(&tslot, 512);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = tc::idesc_s8(128, N);
    const uint32_t aa = tc::smem_u32(sA), ba = tc::smem_u32(sB);
    const uint64_t da = tc::desc_sw128(aa), db = tc::desc_sw128(ba);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      for (int k = 0; k < nmma; ++k) {
        if constexpr (TS)
          mma_ts(tmem + (k % nacc) * N, tmem + 480 + 8 * (k & 3), db + 2 * (k & 3), idesc, k >= nacc);
        else
          tc::mma_s8(tmem + (k % nacc) * N, da + 2 * (k & 3), db + 2 * (k & 3), idesc, k >= nacc);
      }
      tc::mma_commit(&bar);
      tc::mbar_wait(&bar, r & 1);
    }
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 512);
}

template <int N, bool TS = false>
void run(long long* d) {
  cudaFuncSetAttribute(mma_bench<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024);
  for (int nacc : {1, 5}) {
    if (nacc * N > (TS ? 448 : 512)) continue;
    const int nmma = 40, reps = 200;
    mma_bench<N, TS><<<148, 128, 50 * 1024>>>(nmma, nacc, reps, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h = 0;
    cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%s N %3d nacc %d: %.1f cycles per MMA (%.1f floor) %s\n", TS ? "A:tmem" : "A:smem", N, nacc,
           (double)h / reps / nmma, 128.0 * N / 256, cudaGetErrorString(e));
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 148);
  run<16>(d);
  run<32>(d);
  run<64>(d);
  run<96>(d);
  run<128>(d);
  run<256>(d);
  run_warp<32>(d);
  run_warp<64>(d);
  run_warp<256>(d);
  run<32, true>(d);
  run<64, true>(d);
  run<256, true>(d);
  return 0;
}
