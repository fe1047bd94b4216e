// tcgen05 kind::tf32 MN-major operand probe (round 2): A = Wd^T tile read straight from the
// dense layer's tiled [d][128] layout (MN-major: the 128 columns contiguous per feature) and
// B = xT [d][32] (MN-major: the 32 samples contiguous per feature), both loaded by TMA with
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B (CUTLASS: "for mn-major tf32 operands, SW128_32B is the
// only available smem layout"; descriptor layout type 1 = SWIZZLE_128B_BASE32B).  One CTA,
// D[128][32] = sum over K = 32 features (4 MMAs of K = 8), compared with a host GEMM.
// Also: does the MMA truncate or round fp32 inputs to tf32 (A = 1 + 3*2^-12, B = 1)?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tcprobe_mn tcprobe_mn.cu -lcuda
#include <cuda.h>
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

__global__ void probe(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB, float* D,
                      uint32_t lbo_a, uint32_t sbo_a, uint32_t kstep, uint32_t layout, int nk) {
  extern __shared__ __align__(1024) unsigned char dsm[];
  const uint32_t s0 = ((uint32_t)__cvta_generic_to_shared(dsm) + 1023u) & ~1023u;
  const uint32_t sA = s0, sB = s0 + 16384, mbar = s0 + 16384 + 4096, mbar2 = mbar + 8, tptr = mbar + 16;
  const int tid = threadIdx.x, w = tid >> 5;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" :: "r"(tptr) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mbar) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mbar2) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t tmem;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(tmem) : "r"(tptr) : "memory");
  if (tid == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(mbar), "r"(16384 + 4096) : "memory");
    for (int g = 0; g < 4; ++g)   // A: 4 column groups of 32 (128 B) x 32 features, group g at g*4096
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   :: "r"(sA + g * 4096), "l"(&tA), "r"(32 * g), "r"(0), "r"(mbar) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 :: "r"(sB), "l"(&tB), "r"(0), "r"(0), "r"(mbar) : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                   : "=r"(ok) : "r"(mbar), "r"(0u) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((32u >> 3) << 17) |
                           ((128u >> 4) << 24);
    for (int kb = 0; kb < nk; ++kb) {
      const uint64_t ad = desc(sA + kb * kstep, lbo_a, sbo_a, layout);
      const uint64_t bd = desc(sB + kb * kstep, 4096, sbo_a, layout);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                   :: "r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(kb > 0 ? 1u : 0u));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(mbar2) : "memory");
  }
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                 : "=r"(ok) : "r"(mbar2), "r"(0u) : "memory");
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

static void make_map(CUtensorMap* m, void* base, uint64_t inner, uint64_t rows, CUtensorMapSwizzle sw) {
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {inner * 4};
  cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("cuTensorMapEncodeTiled failed %d\n", (int)r); exit(1); }
}

int main() {
  const int K = 32;
  std::vector<float> A(K * 128), Bm(K * 32), ref(128 * 32), out(128 * 32);   // A[f][c], Bm[f][n] (MN-major)
  srand(1);
  for (auto& a : A) a = (float)(rand() % 7 - 3);
  for (auto& b : Bm) b = (float)(rand() % 5 - 2);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, Bm.size() * 4); cudaMalloc(&dD, out.size() * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  CUtensorMap tA, tB;
  struct Cfg { uint32_t lbo, sbo, kstep, layout; CUtensorMapSwizzle sw; const char* name; };
  Cfg cfgs[] = {
      {4096, 512, 1024, 1, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, "B32 lbo=4096 sbo=512"},
      {512, 4096, 1024, 1, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, "B32 lbo=512 sbo=4096"},
      {4096, 1024, 1024, 1, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, "B32 lbo=4096 sbo=1024"},
      {4096, 1024, 1024, 2, CU_TENSOR_MAP_SWIZZLE_128B, "SW128 lbo=4096 sbo=1024"},
  };
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {   // truncation probe: A = 1 + 3*2^-12 everywhere, B = 1 at feature 0 only
      for (auto& a : A) a = 1.0f + 3.0f / 4096.0f;
      for (int f = 0; f < K; ++f) for (int n = 0; n < 32; ++n) Bm[f * 32 + n] = f == 0 ? 1.0f : 0.0f;
    }
    for (int i = 0; i < 128; ++i)
      for (int n = 0; n < 32; ++n) {
        double s = 0;
        for (int f = 0; f < K; ++f) s += (double)A[f * 128 + i] * Bm[f * 32 + n];
        ref[i * 32 + n] = (float)s;
      }
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, Bm.data(), Bm.size() * 4, cudaMemcpyHostToDevice);
    for (auto& c : cfgs) {
      make_map(&tA, dA, 128, K, c.sw);
      make_map(&tB, dB, 32, K, c.sw);
      cudaMemset(dD, 0, out.size() * 4);
      probe<<<1, 128, 32768>>>(tA, tB, dD, c.lbo, c.sbo, c.kstep, c.layout, K / 8);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(out.data(), dD, out.size() * 4, cudaMemcpyDeviceToHost);
      int bad = 0; double maxerr = 0;
      for (size_t i = 0; i < out.size(); ++i) { double d = fabs(out[i] - ref[i]); if (d > 1e-3) ++bad; if (d > maxerr) maxerr = d; }
      printf("pass %d %-28s err=%s bad=%d/%zu maxerr=%g D[0][0..2]=%.9g %.9g %.9g ref=%.9g %.9g %.9g\n", pass, c.name,
             cudaGetErrorString(e), bad, out.size(), maxerr, out[0], out[1], out[2], ref[0], ref[1], ref[2]);
      if (e != cudaSuccess) return 1;
    }
  }
  printf("tf32 of 1+3*2^-12: truncate -> 1, round -> %.9g\n", 1.0 + 1.0 / 1024.0);
  return 0;
}
