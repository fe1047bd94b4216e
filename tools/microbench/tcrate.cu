// tcgen05.mma issue/execution rate probe (round 2): one CTA issues NMMA back-to-back MMAs
// (M = 128, N = n, K = 8 for kind::tf32 / K = 16 for kind::f16) from shared memory into one
// TMEM accumulator, commits, waits; cycles per MMA = clock64 delta / NMMA.  Operand values
// are garbage (the rate is what is measured).  Layouts: K-major 128-B swizzle (layout 2) or
// MN-major 128-B swizzle with 32-B atoms (layout 1, the tf32 MN-major layout).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tcrate tcrate.cu
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

template <int KIND>   // 0 tf32, 1 f16
__global__ void rate(uint32_t idesc, uint32_t layout, uint32_t lbo, uint32_t sbo, int nmma, int nbufs, long long* out) {
  extern __shared__ __align__(1024) unsigned char dsm[];
  const uint32_t s0 = ((uint32_t)__cvta_generic_to_shared(dsm) + 1023u) & ~1023u;
  const uint32_t mbar = s0 + 196608, tptr = mbar + 16;
  const int tid = threadIdx.x, w = tid >> 5;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" :: "r"(tptr) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mbar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t tmem;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(tmem) : "r"(tptr) : "memory");
  if (tid == 0) {
    const long long t0 = clock64();
    for (int i = 0; i < nmma; ++i) {
      const uint32_t b = s0 + (uint32_t)(i & 7) * 16384u;           // A at b, B at b + 8 KB... (garbage values)
      const uint64_t ad = desc(b, lbo, sbo, layout), bd = desc(b + 8192, lbo, sbo, layout);
      if (KIND == 0)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                     :: "r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(1u));
      else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
                     :: "r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(1u));
    }
    const long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(mbar) : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                   : "=r"(ok) : "r"(mbar), "r"(0u) : "memory");
    const long long t2 = clock64();
    out[0] = t1 - t0; out[1] = t2 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" :: "r"(tmem) : "memory");
}

int main() {
  long long* d_out; cudaMalloc(&d_out, 16);
  long long h[2];
  cudaFuncSetAttribute(rate<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(rate<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int nmma = 4096;
  for (int kind = 0; kind < 2; ++kind)
    for (int major = 0; major < 2; ++major) {
      if (kind == 1 && major == 1) continue;
      for (uint32_t mm : {128u, 64u})
      for (uint32_t n : {32u, 64u, 128u, 256u}) {
        const uint32_t fmt = kind == 0 ? 2u : 1u;   // tf32 / bf16
        const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (major << 15) | (major << 16) | ((n >> 3) << 17) |
                               ((mm >> 4) << 24);
        const uint32_t layout = major ? 1u : 2u, lbo = major ? 4096u : 16u, sbo = major ? 512u : 1024u;
        for (int rep = 0; rep < 2; ++rep) {
          if (kind == 0) rate<0><<<1, 128, 200 * 1024>>>(idesc, layout, lbo, sbo, nmma, 8, d_out);
          else rate<1><<<1, 128, 200 * 1024>>>(idesc, layout, lbo, sbo, nmma, 8, d_out);
          cudaError_t e = cudaDeviceSynchronize();
          cudaMemcpy(h, d_out, 16, cudaMemcpyDeviceToHost);
          if (rep == 1)
            printf("%s %s M=%3u N=%3u: issue %.1f cyc/MMA, complete %.1f cyc/MMA  (A %u B + B %u B per MMA) %s\n",
                   kind == 0 ? "tf32" : "bf16", major ? "MN-major(B32)" : "K-major(SW128)", mm, n, (double)h[0] / nmma,
                   (double)h[1] / nmma, mm * 32u, n * 32u, cudaGetErrorString(e));
        }
      }
    }
  return 0;
}
