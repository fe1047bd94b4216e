// tcgen05.mma rate with a CTA pair (cta_group::2, M = 256 over two SMs) vs one CTA
// (cta_group::1, M = 128), kind::tf32 MN-major (the dense forward's operands): does one
// M = 256 pair instruction cost what one M = 128 instruction costs (tcrate.cu: max(67, N/2)
// cycles), i.e. does the pair halve each SM's MMA time?  Operand values are garbage; the
// leader CTA issues NMMA back-to-back MMAs and commits; cycles per MMA are printed.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tcrate2 tcrate2.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r;
}

template <int PAIR>
__global__ void __cluster_dims__(2, 1, 1) rate(uint32_t idesc, int nmma, long long* out) {
  extern __shared__ __align__(1024) unsigned char dsm[];
  const uint32_t s0 = ((uint32_t)__cvta_generic_to_shared(dsm) + 1023u) & ~1023u;
  const uint32_t mbar = s0 + 196608, tptr = mbar + 16;
  const int tid = threadIdx.x, w = tid >> 5;
  const uint32_t rank = cluster_rank();
  if (w == 0) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" :: "r"(tptr) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" :: "r"(tptr) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mbar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t tmem;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(tmem) : "r"(tptr) : "memory");
  if (tid == 0 && (PAIR == 0 || rank == 0)) {
    const long long t0 = clock64();
    for (int i = 0; i < nmma; ++i) {
      const uint32_t b = s0 + (uint32_t)(i & 1) * 65536u;
      const uint64_t ad = desc(b, 4096, 512, 1), bd = desc(b + 16384, 4096, 512, 1);
      if (PAIR)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                     :: "r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(1u));
      else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                     :: "r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(1u));
    }
    const long long t1 = clock64();
    if (PAIR)
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(mbar) : "memory");
    else
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(mbar) : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                   : "=r"(ok) : "r"(mbar), "r"(0u) : "memory");
    const long long t2 = clock64();
    out[0] = t1 - t0; out[1] = t2 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (w == 0) {
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" :: "r"(tmem) : "memory");
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" :: "r"(tmem) : "memory");
  }
}

int main() {
  long long* d_out; cudaMalloc(&d_out, 16);
  long long h[2];
  cudaFuncSetAttribute(rate<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(rate<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int nmma = 4096;
  for (int pair = 0; pair < 2; ++pair)
    for (uint32_t n : {32u, 64u, 128u, 256u}) {
      const uint32_t mm = pair ? 256u : 128u;
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((n >> 3) << 17) |
                             ((mm >> 4) << 24);
      for (int rep = 0; rep < 2; ++rep) {
        if (pair) rate<1><<<2, 128, 200 * 1024>>>(idesc, nmma, d_out);
        else rate<0><<<2, 128, 200 * 1024>>>(idesc, nmma, d_out);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d_out, 16, cudaMemcpyDeviceToHost);
        if (rep == 1)
          printf("%s M=%3u N=%3u: issue %.1f cyc/MMA, complete %.1f cyc/MMA  %s\n", pair ? "cta_group::2" : "cta_group::1",
                 mm, n, (double)h[0] / nmma, (double)h[1] / nmma, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
      }
    }
  return 0;
}
