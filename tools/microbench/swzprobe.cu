// Where does TMA put element (row f, col c) of a 32 x 32 fp32 box under
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B?  Prints the (f, c) found at each 16-B chunk of the
// first 8 rows, and checks the guess  byte = f*128 + ((4c) ^ ((f & 3) << 5)).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o swzprobe swzprobe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
__global__ void k(const __grid_constant__ CUtensorMap t, float* out) {
  __shared__ __align__(1024) float s[32 * 32];
  __shared__ __align__(8) unsigned long long bar;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(s), mb = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mb));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(mb), "r"(4096));
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 :: "r"(sb), "l"(&t), "r"(0), "r"(0), "r"(mb) : "memory");
    uint32_t ok = 0;
    while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(ok) : "r"(mb), "r"(0u) : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = s[i];
}
int main() {
  std::vector<float> a(32 * 32), o(1024);
  for (int f = 0; f < 32; ++f) for (int c = 0; c < 32; ++c) a[f * 32 + c] = f * 100 + c;
  float *da, *dout; cudaMalloc(&da, 4096); cudaMalloc(&dout, 4096);
  cudaMemcpy(da, a.data(), 4096, cudaMemcpyHostToDevice);
  CUtensorMap t; cuuint64_t dims[2] = {32, 32}, st[1] = {128}; cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
  cuTensorMapEncodeTiled(&t, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, da, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  k<<<1, 128>>>(t, dout); cudaDeviceSynchronize();
  cudaMemcpy(o.data(), dout, 4096, cudaMemcpyDeviceToHost);
  for (int r = 0; r < 8; ++r) { printf("row %d:", r); for (int ch = 0; ch < 8; ++ch) printf(" %4.0f", o[r * 32 + ch * 4]); printf("\n"); }
  int bad = 0;
  for (int f = 0; f < 32; ++f) for (int c = 0; c < 32; ++c) {
    const int byte = f * 128 + ((4 * c) ^ ((f & 3) << 5));
    if (o[byte / 4] != a[f * 32 + c]) ++bad;
  }
  printf("guess byte = f*128 + ((4c) ^ ((f & 3) << 5)): bad %d / 1024\n", bad);
  return 0;
}
