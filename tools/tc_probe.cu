// tc_probe.cu -- standalone bring-up probe for the hand-written tcgen05 int8 path (not part
// of libv3db).  C[128][N] = A[128][K] . B[N][K]^T, int8 x int8 -> int32, one CTA:
// operands written to shared memory by threads in the 128B-swizzled K-major layout,
// tcgen05.mma.kind::i8 into TMEM, commit -> mbarrier, tcgen05.ld back to registers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o tools/libtcprobe.so tools/tc_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// K-major, SWIZZLE_128B canonical layout: rows of 128 B, 8-row atoms of 1024 B (SBO).
__device__ __forceinline__ uint64_t sw128_kmajor_desc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
         (static_cast<uint64_t>(2) << 61);
}

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

template <int N, int K>
__global__ void __launch_bounds__(128) tc_probe_kernel(const int8_t* A, const int8_t* B, int32_t* C) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;                       // [128][K] as K/128 panels of [128][128]
  uint8_t* sB = smem + 128 * K;             // [N][K] as K/128 panels of [N][128]
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // swizzled stores: panel p (128 B of K), row r, 16-B chunk c -> p*rows*128 + r*128 + ((c ^ (r&7))*16)
  for (int e = tid; e < 128 * (K / 16); e += 128) {
    const int r = e / (K / 16), cc = e % (K / 16), p = cc / 8, c = cc % 8;
    const uint4 v = *reinterpret_cast<const uint4*>(A + r * K + cc * 16);
    *reinterpret_cast<uint4*>(sA + p * 128 * 128 + r * 128 + ((c ^ (r & 7)) * 16)) = v;
  }
  for (int e = tid; e < N * (K / 16); e += 128) {
    const int r = e / (K / 16), cc = e % (K / 16), p = cc / 8, c = cc % 8;
    const uint4 v = *reinterpret_cast<const uint4*>(B + r * K + cc * 16);
    *reinterpret_cast<uint4*>(sB + p * N * 128 + r * 128 + ((c ^ (r & 7)) * 16)) = v;
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(N < 32 ? 32 : N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;

  if (tid == 0) {
    constexpr uint32_t idesc = idesc_i8(128, N);
#pragma unroll
    for (int k = 0; k < K / 32; ++k) {
      const int p = k / 4, kk = (k % 4) * 32;
      const uint64_t ad = sw128_kmajor_desc(smem_u32(sA + p * 128 * 128) + kk);
      const uint64_t bd = sw128_kmajor_desc(smem_u32(sB + p * N * 128) + kk);
      const uint32_t acc = k > 0 ? 1u : 0u;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
          "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&mbar))
                 : "memory");
  }
  // wait for the MMA chain (phase 0)
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.b32 %0, 1, 0, P1;\n\t}\n"
          : "=r"(done)
          : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    const uint32_t addr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 16; ++j) C[row * N + c0 + j] = static_cast<int32_t>(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(N < 32 ? 32 : N));
}

extern "C" int tc_probe(const int8_t* A, const int8_t* B, int32_t* C, int N, int K) {
  cudaError_t e = cudaSuccess;
#define CASE(NN, KK)                                                                                      \
  if (N == NN && K == KK) {                                                                               \
    const int smem = 128 * KK + NN * KK;                                                                  \
    cudaFuncSetAttribute(tc_probe_kernel<NN, KK>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);     \
    tc_probe_kernel<NN, KK><<<1, 128, smem>>>(A, B, C);                                                   \
    e = cudaDeviceSynchronize();                                                                          \
    return e == cudaSuccess ? 0 : static_cast<int>(e);                                                    \
  }
  CASE(256, 128)
  CASE(128, 128)
  CASE(256, 256)
  CASE(64, 128)
  return -1;
}
