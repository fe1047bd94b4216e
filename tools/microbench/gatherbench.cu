// Async-gather microbenchmark (round 1): random 128-B rows of an L2-resident table
// [32768][64] fp32 (the hd layout: h line | dh line) gathered by
//   (a) ld.global.nc.v4 into registers (8 lanes per line),
//   (b) cp.async.cg 16 B (LDGSTS) into a per-warp smem ring, consumed with LDS,
//   (c) TMA cp.async.bulk.tensor.2d ... tile::gather4 (4 rows per instruction) into smem.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gatherbench gatherbench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

constexpr int ROWF = 64;   // floats per table row (256 B); we gather the first 128 B

__global__ void g_ldg(const int* __restrict__ idx, const float* __restrict__ tab, long nconn, float* out) {
  int lane = threadIdx.x & 31;
  long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * (long)blockDim.x) >> 5;
  float acc = 0.f;
  for (long r = warp; r * 32 < nconn; r += nw) {
    int c = __ldg(idx + r * 32 + lane);
    float4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { int ci = __shfl_sync(~0u, c, i * 4 + (lane >> 3));
      v[i] = __ldg(reinterpret_cast<const float4*>(tab + (long)ci * ROWF + 4 * (lane & 7))); }
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += v[i].x + v[i].y + v[i].z + v[i].w;
  }
  if (acc == 12345.f) out[0] = acc;
}

// (b) cp.async ring: each warp keeps D rows-of-32-connections in flight
template <int D>
__global__ void g_ldgsts(const int* __restrict__ idx, const float* __restrict__ tab, long nconn, float* out) {
  extern __shared__ float4 sm[];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float4* ring = sm + (size_t)wid * (D + 1) * 256;          // (D+1) slots x 32 lines x 8 float4
  long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * (long)blockDim.x) >> 5;
  long nrows = nconn / 32;
  float acc = 0.f;
  auto issue = [&](long r, int slot) {
    if (r < nrows) {
      int c = __ldg(idx + r * 32 + lane);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        int line = i * 4 + (lane >> 3);
        int ci = __shfl_sync(~0u, c, line);
        const float* src = tab + (long)ci * ROWF + 4 * (lane & 7);
        uint32_t dst = (uint32_t)__cvta_generic_to_shared(ring + slot * 256 + line * 8 + (lane & 7));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src));
      }
    }
    asm volatile("cp.async.commit_group;");
  };
  long r = warp; int it = 0;
#pragma unroll
  for (int d = 0; d < D; ++d) issue(r + d * nw, d);
  for (; r < nrows; r += nw, ++it) {
    issue(r + D * nw, (it + D) % (D + 1));
    asm volatile("cp.async.wait_group %0;" :: "n"(D));
    __syncwarp();
    const float4* slot = ring + (it % (D + 1)) * 256;
#pragma unroll
    for (int i = 0; i < 8; ++i) { float4 v = slot[(i * 4 + (lane >> 3)) * 8 + (lane & 7)]; acc += v.x + v.y + v.z + v.w; }
    __syncwarp();
  }
  asm volatile("cp.async.wait_group 0;");
  if (acc == 12345.f) out[0] = acc;
}

// (c) TMA gather4: one elected lane per warp issues 8 gather4 (32 rows x 128 B) per stage
template <int D>
__global__ void g_tma(const __grid_constant__ CUtensorMap tmap, const int* __restrict__ idx, long nconn, float* out) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  float4* ring = reinterpret_cast<float4*>(smraw) + (size_t)wid * (D + 1) * 256;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smraw + (size_t)nwb * (D + 1) * 4096) + wid * (D + 1);
  long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * (long)blockDim.x) >> 5;
  long nrows = nconn / 32;
  if (lane == 0)
    for (int s = 0; s <= D; ++s)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(bars + s)));
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncwarp();
  float acc = 0.f;
  uint32_t phase[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  auto issue = [&](long r, int slot) {
    if (r >= nrows) return;
    int c = __ldg(idx + r * 32 + lane);
    uint32_t bar = (uint32_t)__cvta_generic_to_shared(bars + slot);
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(bar), "r"(4096));
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      int r0 = __shfl_sync(~0u, c, 4 * g), r1 = __shfl_sync(~0u, c, 4 * g + 1);
      int r2 = __shfl_sync(~0u, c, 4 * g + 2), r3 = __shfl_sync(~0u, c, 4 * g + 3);
      if (lane == 0) {
        uint32_t dst = (uint32_t)__cvta_generic_to_shared(ring + slot * 256 + g * 32);
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                     :: "r"(dst), "l"(&tmap), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar) : "memory");
      }
    }
  };
  long r = warp; int it = 0;
  for (int d = 0; d < D; ++d) issue(r + d * nw, d);
  for (; r < nrows; r += nw, ++it) {
    issue(r + D * nw, (it + D) % (D + 1));
    int slot = it % (D + 1);
    uint32_t bar = (uint32_t)__cvta_generic_to_shared(bars + slot);
    uint32_t ph = (phase[0] >> slot) & 1;
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" :: "r"(bar), "r"(ph));
    phase[0] ^= (1u << slot);
    const float4* s = ring + slot * 256;
#pragma unroll
    for (int i = 0; i < 8; ++i) { float4 v = s[i * 32 + lane]; acc += v.x + v.y + v.z + v.w; }
    __syncwarp();
  }
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  const int m = 32768; const long L = 670091, k = 32, nconn = L * k;
  std::vector<int> hidx(nconn);
  uint64_t s = 88172645463325252ull;
  for (long i = 0; i < nconn; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; hidx[i] = (int)(s % m); }
  int* idx; float *tab, *out;
  CK(cudaMalloc(&idx, nconn * 4)); CK(cudaMemcpy(idx, hidx.data(), nconn * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&tab, (long)m * ROWF * 4)); CK(cudaMemset(tab, 0, (long)m * ROWF * 4)); CK(cudaMalloc(&out, 4));
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  auto timeit = [&](const char* name, auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    CK(cudaDeviceSynchronize()); CK(cudaGetLastError());
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) { CK(cudaEventRecord(e0)); launch(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms; }
    CK(cudaGetLastError());
    printf("%-34s %8.1f us  %8.1f GB/s\n", name, best * 1e3, nconn * 128.0 / (best * 1e-3) / 1e9);
  };
  for (int bps : {2, 4, 8}) { char nm[64]; snprintf(nm, 64, "ldg.v4 256thr x%d/SM", bps);
    timeit(nm, [&] { g_ldg<<<nsm * bps, 256>>>(idx, tab, nconn, out); }); }
  {
    auto f2 = g_ldgsts<2>; auto f4 = g_ldgsts<4>;
    for (int w : {8, 16}) {
      int sm2 = w * 3 * 4096, sm4 = w * 5 * 4096; char nm[64];
      if (sm2 <= 227 * 1024) CK(cudaFuncSetAttribute(f2, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2));
      if (sm4 <= 227 * 1024) CK(cudaFuncSetAttribute(f4, cudaFuncAttributeMaxDynamicSharedMemorySize, sm4));
      if (sm2 <= 227 * 1024) { snprintf(nm, 64, "ldgsts D=2 %d warps/CTA", w); timeit(nm, [&] { g_ldgsts<2><<<nsm, w * 32, sm2>>>(idx, tab, nconn, out); }); }
      if (sm4 <= 227 * 1024) { snprintf(nm, 64, "ldgsts D=4 %d warps/CTA", w); timeit(nm, [&] { g_ldgsts<4><<<nsm, w * 32, sm4>>>(idx, tab, nconn, out); }); }
    }
  }
  {
    CUtensorMap tmap;
    cuuint64_t dims[2] = {(cuuint64_t)ROWF, (cuuint64_t)m};
    cuuint64_t strides[1] = {(cuuint64_t)ROWF * 4};
    cuuint32_t box[2] = {32, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, tab, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("tensor map encode failed %d\n", (int)r); return 0; }
    auto f2 = g_tma<2>; auto f4 = g_tma<4>;
    for (int w : {4, 8, 16}) {
      int sm2 = w * 3 * 4096 + w * 3 * 8 + 64, sm4 = w * 5 * 4096 + w * 5 * 8 + 64; char nm[64];
      if (sm2 <= 227 * 1024) CK(cudaFuncSetAttribute(f2, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2));
      if (sm4 <= 227 * 1024) CK(cudaFuncSetAttribute(f4, cudaFuncAttributeMaxDynamicSharedMemorySize, sm4));
      if (sm2 <= 227 * 1024) { snprintf(nm, 64, "tma gather4 D=2 %d warps/CTA", w); timeit(nm, [&] { g_tma<2><<<nsm, w * 32, sm2>>>(tmap, idx, nconn, out); }); }
      if (sm4 <= 227 * 1024) { snprintf(nm, 64, "tma gather4 D=4 %d warps/CTA", w); timeit(nm, [&] { g_tma<4><<<nsm, w * 32, sm4>>>(tmap, idx, nconn, out); }); }
    }
  }
  return 0;
}
