// Microbenchmarks that fix the on-chip ceilings of the fixed fan-in hot path
// (SURVEY.md §7 step 0): random 128-B line gathers from an L2-resident hT[m][32],
// coalesced red.global.add.f32 / .v4.f32 into an L2-resident dhT[m][32], the
// combined gather+red pattern, bulk (TMA-engine) reductions, and an HBM stream.
// Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2bench l2bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ float ld_hint(const float* a, uint64_t p) {
  float v; asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(p)); return v; }
__device__ __forceinline__ void red_f32(float* a, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" :: "l"(a), "f"(v) : "memory"); }
__device__ __forceinline__ void red_v4(float* a, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory"); }

// one warp handles rows of 32 connections; lane = b
__global__ void k_gather(const int* __restrict__ idx, const float* __restrict__ hT, long nconn, float* out) {
  int lane = threadIdx.x & 31;
  long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  long nw = (gridDim.x * (long)blockDim.x) >> 5;
  uint64_t pl = pol_last();
  float acc = 0.f;
  for (long r = warp; r * 32 < nconn; r += nw) {
    int c = __ldg(idx + r * 32 + lane);
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) { int ci = __shfl_sync(~0u, c, i); v[i] = ld_hint(hT + (long)ci * 32 + lane, pl); }
#pragma unroll
    for (int i = 0; i < 32; ++i) acc += v[i];
  }
  if (acc == 12345.f) out[0] = acc;
}
__global__ void k_red(const int* __restrict__ idx, float* dhT, long nconn) {
  int lane = threadIdx.x & 31;
  long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  long nw = (gridDim.x * (long)blockDim.x) >> 5;
  for (long r = warp; r * 32 < nconn; r += nw) {
    int c = __ldg(idx + r * 32 + lane);
#pragma unroll
    for (int i = 0; i < 32; ++i) { int ci = __shfl_sync(~0u, c, i); red_f32(dhT + (long)ci * 32 + lane, 1.0f); }
  }
}
// lane l: line (l>>3) of each group of 4, floats 4*(l&7)..+3
__global__ void k_red4(const int* __restrict__ idx, float* dhT, long nconn) {
  int lane = threadIdx.x & 31;
  long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  long nw = (gridDim.x * (long)blockDim.x) >> 5;
  for (long r = warp; r * 32 < nconn; r += nw) {
    int c = __ldg(idx + r * 32 + lane);
#pragma unroll
    for (int i = 0; i < 8; ++i) { int ci = __shfl_sync(~0u, c, i * 4 + (lane >> 3));
      red_v4(dhT + (long)ci * 32 + 4 * (lane & 7), make_float4(1.f, 1.f, 1.f, 1.f)); }
  }
}
__global__ void k_gather4(const int* __restrict__ idx, const float* __restrict__ hT, long nconn, float* out) {
  int lane = threadIdx.x & 31;
  long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  long nw = (gridDim.x * (long)blockDim.x) >> 5;
  float acc = 0.f;
  for (long r = warp; r * 32 < nconn; r += nw) {
    int c = __ldg(idx + r * 32 + lane);
    float4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { int ci = __shfl_sync(~0u, c, i * 4 + (lane >> 3));
      v[i] = __ldg(reinterpret_cast<const float4*>(hT + (long)ci * 32 + 4 * (lane & 7))); }
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += v[i].x + v[i].y + v[i].z + v[i].w;
  }
  if (acc == 12345.f) out[0] = acc;
}
// gather + red (v4 both) — the fused-step on-chip pattern
__global__ void k_gr4(const int* __restrict__ idx, const float* __restrict__ hT, float* dhT, long nconn, float* out) {
  int lane = threadIdx.x & 31;
  long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  long nw = (gridDim.x * (long)blockDim.x) >> 5;
  float acc = 0.f;
  for (long r = warp; r * 32 < nconn; r += nw) {
    int c = __ldg(idx + r * 32 + lane);
    float4 v[8]; int cc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { cc[i] = __shfl_sync(~0u, c, i * 4 + (lane >> 3));
      v[i] = __ldg(reinterpret_cast<const float4*>(hT + (long)cc[i] * 32 + 4 * (lane & 7))); }
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += v[i].x + v[i].y + v[i].z + v[i].w;
    float s = __shfl_xor_sync(~0u, acc, 1) * 1e-30f;
#pragma unroll
    for (int i = 0; i < 8; ++i) red_v4(dhT + (long)cc[i] * 32 + 4 * (lane & 7), make_float4(s, s, s, s));
  }
  if (acc == 12345.f) out[0] = acc;
}
// gather + red (scalar, lane = b)
__global__ void k_gr1(const int* __restrict__ idx, const float* __restrict__ hT, float* dhT, long nconn, float* out) {
  int lane = threadIdx.x & 31;
  long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  long nw = (gridDim.x * (long)blockDim.x) >> 5;
  float acc = 0.f;
  for (long r = warp; r * 32 < nconn; r += nw) {
    int c = __ldg(idx + r * 32 + lane);
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) { int ci = __shfl_sync(~0u, c, i); v[i] = __ldg(hT + (long)ci * 32 + lane); }
#pragma unroll
    for (int i = 0; i < 32; ++i) acc += v[i];
    float s = acc * 1e-30f;
#pragma unroll
    for (int i = 0; i < 32; ++i) { int ci = __shfl_sync(~0u, c, i); red_f32(dhT + (long)ci * 32 + lane, s); }
  }
  if (acc == 12345.f) out[0] = acc;
}
// bulk reduce: each warp stages 32 lines (4 KB) in smem, lane i issues one 128-B cp.reduce.async.bulk
__global__ void k_bulkred(const int* __restrict__ idx, float* dhT, long nconn) {
  extern __shared__ float sm[];
  int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float* buf = sm + wib * 1024;
  long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  long nw = (gridDim.x * (long)blockDim.x) >> 5;
  for (long r = warp; r * 32 < nconn; r += nw) {
    int c = __ldg(idx + r * 32 + lane);
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 32; ++i) buf[i * 32 + lane] = 1.0f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    uint32_t s = (uint32_t)__cvta_generic_to_shared(buf + lane * 32);
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 128;"
                 :: "l"(dhT + (long)c * 32), "r"(s) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// gather (ld.v4 into registers) + bulk reduce: the contributions of a row go to a per-warp
// smem buffer (two buffers, alternating) and each lane issues one 128-B cp.reduce.async.bulk
// for its connection: the reductions leave through the TMA path, not the LSU -> L1 -> XBAR path
__global__ void k_gbulk(const int* __restrict__ idx, const float* __restrict__ hT, float* dhT, long nconn, float* out) {
  extern __shared__ float sm[];
  int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  long nw = (gridDim.x * (long)blockDim.x) >> 5;
  float acc = 0.f;
  int it = 0;
  for (long r = warp; r * 32 < nconn; r += nw, ++it) {
    float* buf = sm + (wib * 2 + (it & 1)) * 1024;
    int c = __ldg(idx + r * 32 + lane);
    float4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { int ci = __shfl_sync(~0u, c, i * 4 + (lane >> 3));
      v[i] = __ldg(reinterpret_cast<const float4*>(hT + (long)ci * 32 + 4 * (lane & 7))); }
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += v[i].x + v[i].y + v[i].z + v[i].w;
    float s = __shfl_xor_sync(~0u, acc, 1) * 1e-30f;
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");   // buffer it&1 free again
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 8; ++i)
      *reinterpret_cast<float4*>(buf + (i * 4 + (lane >> 3)) * 32 + 4 * (lane & 7)) = make_float4(s, s, s, s);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    uint32_t sa = (uint32_t)__cvta_generic_to_shared(buf + lane * 32);
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 128;"
                 :: "l"(dhT + (long)c * 32), "r"(sa) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (acc == 12345.f) out[0] = acc;
}
// gather + split reductions: lines of connection group gq < SPLIT go through red.v4 (LSU ->
// L1 -> XBAR), the others are staged in smem and leave through the TMA engine as one
// cp.reduce.async.bulk of 128 B each — two egress paths at once, if they are separate
template <int SPLIT>
__global__ void k_gsplit(const int* __restrict__ idx, const float* __restrict__ hT, float* dhT, long nconn, float* out) {
  extern __shared__ float sm[];
  int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, gq = lane >> 3, bq = lane & 7;
  long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  long nw = (gridDim.x * (long)blockDim.x) >> 5;
  float acc = 0.f;
  int it = 0;
  for (long r = warp; r * 32 < nconn; r += nw, ++it) {
    float* buf = sm + (wib * 2 + (it & 1)) * 1024;
    int c = __ldg(idx + r * 32 + lane);
    float4 v[8]; int cc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { cc[i] = __shfl_sync(~0u, c, i * 4 + gq);
      v[i] = __ldg(reinterpret_cast<const float4*>(hT + (long)cc[i] * 32 + 4 * bq)); }
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += v[i].x + v[i].y + v[i].z + v[i].w;
    float s = __shfl_xor_sync(~0u, acc, 1) * 1e-30f;
    if (gq < SPLIT) {
#pragma unroll
      for (int i = 0; i < 8; ++i) red_v4(dhT + (long)cc[i] * 32 + 4 * bq, make_float4(s, s, s, s));
    }
    if (SPLIT < 4) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncwarp();
      if (gq >= SPLIT) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          *reinterpret_cast<float4*>(buf + (i * 4 + gq) * 32 + 4 * bq) = make_float4(s, s, s, s);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if ((lane & 3) >= SPLIT) {      // connection `lane` has group lane & 3
        uint32_t sa = (uint32_t)__cvta_generic_to_shared(buf + lane * 32);
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 128;"
                     :: "l"(dhT + (long)c * 32), "r"(sa) : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (SPLIT < 4) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (acc == 12345.f) out[0] = acc;
}
__global__ void k_stream(const float4* __restrict__ a, long n4, float* out) {
  float acc = 0.f;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += gridDim.x * (long)blockDim.x) {
    float4 v = __ldg(a + i); acc += v.x + v.y + v.z + v.w; }
  if (acc == 12345.f) out[0] = acc;
}
__global__ void k_copy(const float4* __restrict__ a, float4* b, long n4) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += gridDim.x * (long)blockDim.x) b[i] = a[i];
}

int main(int argc, char** argv) {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("device %s SMs %d L2 %d MB clock %d\n", p.name, p.multiProcessorCount, p.l2CacheSize >> 20, p.clockRate);
  const int m = 32768;
  const long L = 670091, k = 32, nconn = L * k;
  std::vector<int> hidx(nconn);
  uint64_t s = 88172645463325252ull;
  for (long i = 0; i < nconn; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; hidx[i] = (int)(s % m); }
  int* idx; float *hT, *dhT, *out; float4 *big, *big2;
  CK(cudaMalloc(&idx, nconn * 4)); CK(cudaMemcpy(idx, hidx.data(), nconn * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&hT, (long)m * 32 * 4)); CK(cudaMalloc(&dhT, (long)m * 32 * 4)); CK(cudaMalloc(&out, 4));
  CK(cudaMemset(hT, 0, (long)m * 128)); CK(cudaMemset(dhT, 0, (long)m * 128));
  long nbig = 1L << 30; CK(cudaMalloc(&big, nbig)); CK(cudaMalloc(&big2, nbig)); CK(cudaMemset(big, 0, nbig));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  int nsm = p.multiProcessorCount;
  auto timeit = [&](const char* name, double bytes, auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
      CK(cudaEventRecord(e0)); launch(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
    }
    CK(cudaGetLastError());
    printf("%-28s %9.1f us  %8.1f GB/s\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9);
  };
  double gbytes = (double)nconn * 128;
  for (int bpsm : {4, 8, 16}) for (int tpb : {256}) {
    int grid = nsm * bpsm; char nm[64];
    snprintf(nm, 64, "gather f32 g=%d", grid);  timeit(nm, gbytes, [&] { k_gather<<<grid, tpb>>>(idx, hT, nconn, out); });
    snprintf(nm, 64, "gather v4 g=%d", grid);   timeit(nm, gbytes, [&] { k_gather4<<<grid, tpb>>>(idx, hT, nconn, out); });
    snprintf(nm, 64, "red f32 g=%d", grid);     timeit(nm, gbytes, [&] { k_red<<<grid, tpb>>>(idx, dhT, nconn); });
    snprintf(nm, 64, "red v4 g=%d", grid);      timeit(nm, gbytes, [&] { k_red4<<<grid, tpb>>>(idx, dhT, nconn); });
    snprintf(nm, 64, "gather+red f32 g=%d", grid); timeit(nm, 2 * gbytes, [&] { k_gr1<<<grid, tpb>>>(idx, hT, dhT, nconn, out); });
    snprintf(nm, 64, "gather+red v4 g=%d", grid);  timeit(nm, 2 * gbytes, [&] { k_gr4<<<grid, tpb>>>(idx, hT, dhT, nconn, out); });
    snprintf(nm, 64, "bulk red g=%d", grid);
    CK(cudaFuncSetAttribute(k_bulkred, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4096));
    timeit(nm, gbytes, [&] { k_bulkred<<<grid, tpb, 8 * 4096>>>(idx, dhT, nconn); });
    snprintf(nm, 64, "gather v4+bulk red g=%d", grid);
    CK(cudaFuncSetAttribute(k_gbulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 4096));
    timeit(nm, 2 * gbytes, [&] { k_gbulk<<<grid, tpb, 16 * 4096>>>(idx, hT, dhT, nconn, out); });
  }
  for (int bpsm : {4, 8}) {
    int grid = nsm * bpsm; char nm[64];
    CK(cudaFuncSetAttribute(k_gsplit<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 4096));
    CK(cudaFuncSetAttribute(k_gsplit<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 4096));
    CK(cudaFuncSetAttribute(k_gsplit<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 4096));
    CK(cudaFuncSetAttribute(k_gsplit<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 4096));
    CK(cudaFuncSetAttribute(k_gsplit<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 4096));
    snprintf(nm, 64, "gather+red split 4/4 LSU g=%d", grid);
    timeit(nm, 2 * gbytes, [&] { k_gsplit<4><<<grid, 256, 16 * 4096>>>(idx, hT, dhT, nconn, out); });
    snprintf(nm, 64, "gather+red split 3/4 LSU g=%d", grid);
    timeit(nm, 2 * gbytes, [&] { k_gsplit<3><<<grid, 256, 16 * 4096>>>(idx, hT, dhT, nconn, out); });
    snprintf(nm, 64, "gather+red split 2/4 LSU g=%d", grid);
    timeit(nm, 2 * gbytes, [&] { k_gsplit<2><<<grid, 256, 16 * 4096>>>(idx, hT, dhT, nconn, out); });
    snprintf(nm, 64, "gather+red split 1/4 LSU g=%d", grid);
    timeit(nm, 2 * gbytes, [&] { k_gsplit<1><<<grid, 256, 16 * 4096>>>(idx, hT, dhT, nconn, out); });
    snprintf(nm, 64, "gather+red split 0/4 LSU g=%d", grid);
    timeit(nm, 2 * gbytes, [&] { k_gsplit<0><<<grid, 256, 16 * 4096>>>(idx, hT, dhT, nconn, out); });
  }
  timeit("hbm read 1GiB", (double)nbig, [&] { k_stream<<<nsm * 8, 512>>>(big, nbig / 16, out); });
  timeit("hbm copy 1GiB", 2.0 * nbig, [&] { k_copy<<<nsm * 8, 512>>>(big, big2, nbig / 16); });
  return 0;
}
