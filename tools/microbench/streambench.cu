// DRAM access-pattern microbenchmark (round 1): the fused row kernel streams per label row
// 128 B from each of several arrays (W, idx, mW, vW, pos: structure of arrays), one warp per
// row, rows in 32-row blocks strided over warps; it also writes 3 of them back.  Compare:
//   (a) SoA, 5 arrays read + 3 written, 128 B per array per row (the current layout)
//   (b) AoS, one 640-B record per row (the same bytes, contiguous per row)
//   (c) plain sequential copy-like stream (float4 grid-stride) of the same bytes
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o streambench streambench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

// (a) SoA: 5 arrays of [L][32] floats; read all 5, write 3
__global__ void soa(const float* __restrict__ a0, const float* __restrict__ a1, float* a2, float* a3,
                    const float* __restrict__ a4, float* o0, long L, int blk_rows) {
  const int lane = threadIdx.x & 31;
  const long nw = (gridDim.x * (long)blockDim.x) >> 5;
  const long nblk = L / blk_rows;
  for (long b = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5; b < nblk; b += nw) {
    for (int i = 0; i < blk_rows; ++i) {
      const long r = (b * blk_rows + i) * 32 + lane;
      float x = a0[r] + a1[r] + a2[r] + a3[r] + a4[r];
      o0[r] = x; a2[r] = x * 0.5f; a3[r] = x * 0.25f;
    }
  }
}
// (b) AoS: record of 5 x 32 floats per row; read all, write 3 fields back
__global__ void aos(float* rec, long L, int blk_rows) {
  const int lane = threadIdx.x & 31;
  const long nw = (gridDim.x * (long)blockDim.x) >> 5;
  const long nblk = L / blk_rows;
  for (long b = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5; b < nblk; b += nw) {
    for (int i = 0; i < blk_rows; ++i) {
      float* r = rec + (b * blk_rows + i) * 160 + lane;
      float x = r[0] + r[32] + r[64] + r[96] + r[128];
      r[0] = x; r[64] = x * 0.5f; r[96] = x * 0.25f;
    }
  }
}
// (d) SoA with per-warp bulk async copies: each warp stages sub-blocks of R rows of all 5
// arrays (5 x R x 128 B) into a 2-stage smem ring with cp.async.bulk + mbarrier, reads them
// from smem, and writes 3 arrays back with plain stores.
template <int R>
__global__ void soa_bulk(const float* __restrict__ a0, const float* __restrict__ a1, float* a2, float* a3,
                         const float* __restrict__ a4, float* o0, long L) {
  extern __shared__ __align__(128) float sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float* ring = sm + (size_t)wid * 2 * 5 * R * 32;
  __shared__ __align__(8) unsigned long long bars[32][2];
  const long nw = (gridDim.x * (long)blockDim.x) >> 5;
  const long nsub = L / R;
  long sb = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  if (lane == 0) for (int s = 0; s < 2; ++s)
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"((unsigned)__cvta_generic_to_shared(&bars[wid][s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const float* src[5] = {a0, a1, a2, a3, a4};
  auto issue = [&](long sub, int stage) {
    if (sub >= nsub || lane != 0) return;
    unsigned bar = (unsigned)__cvta_generic_to_shared(&bars[wid][stage]);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(bar), "r"(5 * R * 128) : "memory");
    for (int a = 0; a < 5; ++a) {
      unsigned dst = (unsigned)__cvta_generic_to_shared(ring + (stage * 5 + a) * R * 32);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(dst), "l"(src[a] + sub * R * 32), "r"(R * 128), "r"(bar) : "memory");
    }
  };
  unsigned phase = 0;
  issue(sb, 0);
  int it = 0;
  for (; sb < nsub; sb += nw, ++it) {
    const int stage = it & 1;
    issue(sb + nw, stage ^ 1);
    unsigned bar = (unsigned)__cvta_generic_to_shared(&bars[wid][stage]);
    unsigned ph = (phase >> stage) & 1;
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" :: "r"(bar), "r"(ph) : "memory");
    phase ^= 1u << stage;
    const float* st = ring + stage * 5 * R * 32;
    for (int i = 0; i < R; ++i) {
      const long r = (sb * R + i) * 32 + lane;
      float x = st[0 * R * 32 + i * 32 + lane] + st[1 * R * 32 + i * 32 + lane] + st[2 * R * 32 + i * 32 + lane] +
                st[3 * R * 32 + i * 32 + lane] + st[4 * R * 32 + i * 32 + lane];
      o0[r] = x; a2[r] = x * 0.5f; a3[r] = x * 0.25f;
    }
    __syncwarp();
  }
}
__global__ void seq(const float4* __restrict__ a, float4* b, long n4r, long n4w) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4r; i += gridDim.x * (long)blockDim.x) {
    float4 v = a[i];
    if (i < n4w) b[i] = v;
  }
}

int main() {
  const long L = 670091 / 32 * 32;
  const size_t arr = (size_t)L * 32 * 4;
  float *a0, *a1, *a2, *a3, *a4, *o0, *rec;
  CK(cudaMalloc(&a0, arr)); CK(cudaMalloc(&a1, arr)); CK(cudaMalloc(&a2, arr)); CK(cudaMalloc(&a3, arr));
  CK(cudaMalloc(&a4, arr)); CK(cudaMalloc(&o0, arr)); CK(cudaMalloc(&rec, 5 * arr));
  CK(cudaMemset(a0, 0, arr)); CK(cudaMemset(a1, 0, arr)); CK(cudaMemset(a2, 0, arr)); CK(cudaMemset(a3, 0, arr));
  CK(cudaMemset(a4, 0, arr)); CK(cudaMemset(rec, 0, 5 * arr));
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const double bytes = 8.0 * arr;   // 5 reads + 3 writes
  auto timeit = [&](const char* name, auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) { CK(cudaEventRecord(e0)); launch(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms; }
    CK(cudaGetLastError());
    printf("%-40s %8.1f us  %8.1f GB/s\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9);
  };
  for (int warps_per_sm : {12, 24, 48}) for (int blk : {1, 32}) {
    char nm[80]; int threads = 128, grid = nsm * warps_per_sm / 4;
    snprintf(nm, 80, "SoA 5r+3w %dw/SM blk=%d", warps_per_sm, blk);
    timeit(nm, [&] { soa<<<grid, threads>>>(a0, a1, a2, a3, a4, o0, L, blk); });
    snprintf(nm, 80, "AoS 640B rec %dw/SM blk=%d", warps_per_sm, blk);
    timeit(nm, [&] { aos<<<grid, threads>>>(rec, L, blk); });
  }
  for (int warps_per_sm : {8, 12, 16}) {
    char nm[80]; int threads = 128, grid = nsm * warps_per_sm / 4;
    int sm8 = 4 * 2 * 5 * 8 * 32 * 4, sm4 = 4 * 2 * 5 * 4 * 32 * 4;
    CK(cudaFuncSetAttribute(soa_bulk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm8));
    CK(cudaFuncSetAttribute(soa_bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm4));
    snprintf(nm, 80, "SoA bulk R=8 %dw/SM", warps_per_sm);
    timeit(nm, [&] { soa_bulk<8><<<grid, threads, sm8>>>(a0, a1, a2, a3, a4, o0, L); });
    snprintf(nm, 80, "SoA bulk R=4 %dw/SM", warps_per_sm);
    timeit(nm, [&] { soa_bulk<4><<<grid, threads, sm4>>>(a0, a1, a2, a3, a4, o0, L); });
  }
  return 0;
}
