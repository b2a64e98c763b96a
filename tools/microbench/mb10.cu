// tcgen05.mma kind::i8 issue rate on B200 (one CTA, M = 128): cycles per MMA for A from shared memory (SS)
// or tensor memory (TS) and N = 16..256, K = 32 per instruction.  Decides the Ozaki tile shape (ozaki.cuh).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb10 mb10.cu && ./mb10
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFFu) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46);
}
template <int N, bool TS>
__global__ void k(long long* cyc, int iters) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t taddr;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su32(&taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar)));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = taddr;
  const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
  long long c0 = 0, c1 = 0;
  if (threadIdx.x == 0) {
    c0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t acc = (i & 7) ? 1u : 0u;
      const uint32_t d = t + (uint32_t)((i & 1) * N) + (TS ? 256u : 0u);   // accumulators after the A columns
      const uint64_t bd = desc(su32(sm) + 32768 + (uint32_t)((i & 3) * 256));
      if (TS) {
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
                     :: "r"(d), "r"(t + (uint32_t)((i & 7) * 8)), "l"(bd), "r"(idesc), "r"(acc));
      } else {
        const uint64_t ad = desc(su32(sm) + (uint32_t)((i & 3) * 256));
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                     :: "r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&bar)) : "memory");
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" :: "r"(su32(&bar)) : "memory");
    c1 = clock64();
    *cyc = c1 - c0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(t));
}
template <int N, bool TS>
void run(long long* d) {
  const int iters = 4096;
  cudaFuncSetAttribute(k<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<N, TS><<<1, 128, 64 * 1024>>>(d, iters);
  k<N, TS><<<1, 128, 64 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double c = (double)h / iters, mac = 128.0 * N * 32;
  printf("%s N=%3d: %.1f cycles/MMA, %.0f MAC/cycle (%s)\n", TS ? "TS" : "SS", N, c, mac / c, cudaGetErrorString(e));
}
int main() {
  long long* d;
  cudaMalloc(&d, 8);
  run<16, false>(d); run<32, false>(d); run<64, false>(d); run<128, false>(d); run<256, false>(d);
  run<16, true>(d); run<32, true>(d); run<64, true>(d); run<128, true>(d);
  return 0;
}
