// tcgen05 kind::tf32 operand-layout probe (round 1): one M=128, N=32, K=8 MMA from shared
// memory into TMEM, read back with tcgen05.ld, compared with a host GEMM.
//   mode 0: A and B MN-major, 128-B swizzle (A atom g at g*1024, B one atom)
//   mode 1: A and B K-major, no swizzle (core matrices 8 rows x 16 B)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tcprobe tcprobe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

__global__ void probe(const float* A, const float* Bm, float* D, int mode, uint32_t lbo_a, uint32_t sbo_a,
                      uint32_t lbo_b, uint32_t sbo_b) {
  // A[128][8] (m, k), Bm[8][32] (k, n) row-major in global; D[128][32]
  __shared__ __align__(1024) unsigned char sm[8192 + 2048 + 64];
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t sA = sbase, sB = sbase + 8192, mbar = sbase + 8192 + 2048, tptr = mbar + 16;
  const int tid = threadIdx.x, w = tid >> 5;
  for (int e = tid; e < 128 * 8; e += blockDim.x) {
    const int mm = e / 8, k = e % 8;
    uint32_t off;
    if (mode == 0) { const int g = mm / 32, ml = mm % 32; off = g * 1024 + k * 128 + (((ml / 4) ^ k) << 4) + (ml % 4) * 4; }
    else if (mode == 2) { off = (mm / 4) * sbo_a + (k / 8) * lbo_a + (k % 8) * 16 + (mm % 4) * 4; }
    else { off = (mm / 8) * sbo_a + (k / 4) * lbo_a + (mm % 8) * 16 + (k % 4) * 4; }
    *reinterpret_cast<float*>(sm + off) = A[mm * 8 + k];
  }
  for (int e = tid; e < 8 * 32; e += blockDim.x) {
    const int k = e / 32, n = e % 32;
    uint32_t off;
    if (mode == 0) off = k * 128 + (((n / 4) ^ k) << 4) + (n % 4) * 4;
    else if (mode == 2) off = (n / 4) * sbo_b + (k / 8) * lbo_b + (k % 8) * 16 + (n % 4) * 4;
    else off = (n / 8) * sbo_b + (k / 4) * lbo_b + (n % 8) * 16 + (k % 4) * 4;
    *reinterpret_cast<float*>(sm + 8192 + off) = Bm[k * 32 + n];
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" :: "r"(tptr) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mbar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t tmem;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(tmem) : "r"(tptr) : "memory");
  const uint32_t major = mode == 1 ? 0u : 1u;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (major << 15) | (major << 16) | ((32u >> 3) << 17) |
                         ((128u >> 4) << 24);
  if (tid == 0) {
    const uint64_t ad = mode == 0 ? desc(sA, lbo_a, sbo_a, 2) : desc(sA, lbo_a, sbo_a, 0);
    const uint64_t bd = mode == 0 ? desc(sB, lbo_b, sbo_b, 2) : desc(sB, lbo_b, sbo_b, 0);   // modes 1, 2: no swizzle
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                 :: "r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(0u));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(mbar) : "memory");
  }
  uint32_t ok = 0;
  while (!ok) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                 : "=r"(ok) : "r"(mbar), "r"(0u) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (w < 4) {
    uint32_t v[32];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                   "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                   "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                 : "r"(tmem + ((uint32_t)(32 * w) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int row = 32 * w + (tid & 31);
    for (int n = 0; n < 32; ++n) D[row * 32 + n] = __uint_as_float(v[n]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" :: "r"(tmem) : "memory");
}

int main() {
  std::vector<float> A(128 * 8), Bm(8 * 32), ref(128 * 32), out(128 * 32);
  srand(1);
  for (auto& a : A) a = (float)(rand() % 7 - 3);
  for (auto& b : Bm) b = (float)(rand() % 5 - 2);
  for (int i = 0; i < 128; ++i)
    for (int n = 0; n < 32; ++n) { float s = 0; for (int k = 0; k < 8; ++k) s += A[i * 8 + k] * Bm[k * 32 + n]; ref[i * 32 + n] = s; }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, Bm.size() * 4); cudaMalloc(&dD, out.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, Bm.data(), Bm.size() * 4, cudaMemcpyHostToDevice);
  struct Cfg { int mode; uint32_t la, sa, lb, sb; const char* name; };
  Cfg cfgs[] = {
      {0, 1024, 4096, 1024, 1024, "MN sw128 lbo=1024 sbo=4096"},
      {0, 4096, 1024, 1024, 1024, "MN sw128 lbo=4096 sbo=1024 (swapped)"},
      {1, 128, 256, 128, 256, "K interleave lbo=128 sbo=256"},
      {1, 2048, 128, 512, 128, "K interleave lbo=2048 sbo=128"},
      {2, 4096, 128, 1024, 128, "MN interleave lbo=4096 sbo=128"},
      {2, 128, 256, 128, 256, "MN interleave lbo=128 sbo=256"},
  };
  for (auto& c : cfgs) {
    cudaMemset(dD, 0, out.size() * 4);
    probe<<<1, 128>>>(dA, dB, dD, c.mode, c.la, c.sa, c.lb, c.sb);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(out.data(), dD, out.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0; double maxerr = 0;
    for (size_t i = 0; i < out.size(); ++i) { double d = fabs(out[i] - ref[i]); if (d > 1e-3) ++bad; if (d > maxerr) maxerr = d; }
    printf("%-40s err=%s bad=%d/%zu maxerr=%g  D[0][0..3]=%g %g %g %g ref=%g %g %g %g\n", c.name, cudaGetErrorString(e), bad,
           out.size(), maxerr, out[0], out[1], out[2], out[3], ref[0], ref[1], ref[2], ref[3]);
  }
  return 0;
}
