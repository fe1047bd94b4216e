// Die-locality microbenchmark (round 1): does placing the L2-resident h / dh lines on the
// gathering SM's own die raise the gather / red ceilings of the fused step's on-chip pattern?
//
// B200 = 2 dies x 74 SMs; L2 slices are split across the dies and a physical address maps to
// one die at ~2-KB granularity (B300_MICROARCH.md: "addr->die ~Bernoulli(0.5) @ 2KB-grain").
// 1. probe: one CTA per SM times dependent L2-hit loads to every 2-KB chunk of a 32-MB buffer;
//    near (same-die) and far chunks differ by ~30 cycles.
// 2. classify SMs and chunks into two dies (relative to SM 0's pattern).
// 3. build per-die copies of a 32768-line x 128-B table (16 lines per 2-KB chunk) and compare
//    random 128-B line gathers / red.v4 reductions (21.4 M lines, the Amazon-670K connection
//    count) from (a) a plain contiguous table, (b) the gathering SM's own-die copy, (c) the
//    other die's copy.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o diebench diebench.cu
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

constexpr int kChunk = 2048;                 // bytes
constexpr long kBuf = 128L << 20;            // probe / placement buffer
constexpr int kNCh = (int)(kBuf / kChunk);   // 65536 chunks
constexpr int kLines = 32768;                // table lines (m)
constexpr int kLinesPerChunk = kChunk / 128;

__device__ __forceinline__ unsigned smid() { unsigned r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }

// one CTA per SM (big smem), lane 0 times 8 dependent L2 loads per chunk (ld.cg bypasses L1)
__global__ void k_probe(const unsigned* __restrict__ buf, int nch, int stride_ch, float* lat, int* sm_of_block) {
  extern __shared__ char pad[];
  if (threadIdx.x != 0) return;
  const unsigned s = smid();
  sm_of_block[blockIdx.x] = (int)s;
  for (int c = 0; c < nch; c += stride_ch) {
    const unsigned* p = buf + (size_t)c * (kChunk / 4);
    unsigned x = 0;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(x) : "l"(p));   // warm into L2
    long long t0 = clock64();
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(x) : "l"(p + x));   // buffer is 0: p + x == p, but dependent
    long long t1 = clock64();
    lat[(size_t)blockIdx.x * nch + c] = (float)(t1 - t0) / 8.0f + (float)x;
  }
  (void)pad;
}

// gather: warp per 32 connections, lane (g = lane>>3, b = lane&7) loads 16 B of line 4i+g
// mode 0: plain table; 1: own-die copy; 2: other-die copy.  line address = chunk_base[die][c/16] + (c%16)*128
__global__ void k_gather(const int* __restrict__ idx, long nconn, const float* __restrict__ plain,
                         const char* __restrict__ base, const int* __restrict__ chunk_of, const int* __restrict__ sm_die,
                         int mode, float* out) {
  __shared__ int co[2][kLines / kLinesPerChunk];     // chunk index of line group c/16 in the die-d h copy
  for (int i = threadIdx.x; i < 2 * (kLines / kLinesPerChunk); i += blockDim.x) co[i / (kLines / kLinesPerChunk)][i % (kLines / kLinesPerChunk)] = chunk_of[i];
  __syncthreads();
  const int die = sm_die[smid()];
  const int use = mode == 1 ? die : 1 - die;
  const int lane = threadIdx.x & 31;
  long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * (long)blockDim.x) >> 5;
  float acc = 0.f;
  for (long r = warp; r * 32 < nconn; r += nw) {
    int c = __ldg(idx + r * 32 + lane);
    float4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int ci = __shfl_sync(~0u, c, i * 4 + (lane >> 3));
      const float* p = mode == 0 ? plain + (long)ci * 32
                                 : reinterpret_cast<const float*>(base + (long)co[use][ci / kLinesPerChunk] * kChunk + (ci % kLinesPerChunk) * 128);
      v[i] = __ldg(reinterpret_cast<const float4*>(p + 4 * (lane & 7)));
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += v[i].x + v[i].y + v[i].z + v[i].w;
  }
  if (acc == 12345.f) out[0] = acc;
}

__global__ void k_red(const int* __restrict__ idx, long nconn, float* plain, char* base,
                      const int* __restrict__ chunk_of, const int* __restrict__ sm_die, int mode, int gather_too,
                      const float* __restrict__ hplain, float* out) {
  constexpr int G = kLines / kLinesPerChunk;
  __shared__ int co[4][G];                           // [h die0, h die1, dh die0, dh die1]
  for (int i = threadIdx.x; i < 4 * G; i += blockDim.x) co[i / G][i % G] = chunk_of[i];
  __syncthreads();
  const int die = sm_die[smid()];
  const int use = mode == 1 ? die : 1 - die;
  const int lane = threadIdx.x & 31;
  long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * (long)blockDim.x) >> 5;
  float acc = 0.f;
  for (long r = warp; r * 32 < nconn; r += nw) {
    int c = __ldg(idx + r * 32 + lane);
    int cc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) cc[i] = __shfl_sync(~0u, c, i * 4 + (lane >> 3));
    if (gather_too) {
      float4 v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float* p = mode == 0 ? hplain + (long)cc[i] * 64
                                   : reinterpret_cast<const float*>(base + (long)co[use][cc[i] / kLinesPerChunk] * kChunk + (cc[i] % kLinesPerChunk) * 128);
        v[i] = __ldg(reinterpret_cast<const float4*>(p + 4 * (lane & 7)));
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) acc += v[i].x + v[i].y + v[i].z + v[i].w;
    }
    float s = __shfl_xor_sync(~0u, acc, 1) * 1e-30f + 1e-30f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float* p = mode == 0 ? plain + (long)cc[i] * (gather_too ? 64 : 32) + (gather_too ? 32 : 0)
                           : reinterpret_cast<float*>(base + (long)co[2 + use][cc[i] / kLinesPerChunk] * kChunk + (cc[i] % kLinesPerChunk) * 128);
      asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(p + 4 * (lane & 7)), "f"(s), "f"(s), "f"(s), "f"(s) : "memory");
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  const int nsm = p.multiProcessorCount;
  printf("device %s SMs %d\n", p.name, nsm);
  char* buf; CK(cudaMalloc(&buf, kBuf));
  CK(cudaMemset(buf, 0, kBuf));
  float* lat; int* smb; CK(cudaMalloc(&lat, (size_t)nsm * kNCh * 4)); CK(cudaMalloc(&smb, nsm * 4));
  const int pad = 200 * 1024;
  CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, pad));
  k_probe<<<nsm, 32, pad>>>(reinterpret_cast<unsigned*>(buf), kNCh, 1, lat, smb);
  CK(cudaDeviceSynchronize());
  std::vector<float> L((size_t)nsm * kNCh); std::vector<int> smofb(nsm);
  CK(cudaMemcpy(L.data(), lat, L.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(smofb.data(), smb, nsm * 4, cudaMemcpyDeviceToHost));
  // chunk labels relative to block 0's SM: near (< median) = die A
  std::vector<float> r0(L.begin(), L.begin() + kNCh), srt = r0;
  std::nth_element(srt.begin(), srt.begin() + kNCh / 2, srt.end());
  const float med = srt[kNCh / 2];
  std::vector<int> chdie(kNCh);
  double lo = 0, hi = 0; int nlo = 0, nhi = 0;
  for (int c = 0; c < kNCh; ++c) { chdie[c] = r0[c] < med ? 0 : 1; if (chdie[c]) { hi += r0[c]; ++nhi; } else { lo += r0[c]; ++nlo; } }
  printf("SM%d: chunk latency near %.1f (n=%d) far %.1f (n=%d) cycles\n", smofb[0], lo / nlo, nlo, hi / nhi, nhi);
  // SM die: mean latency to die-0 chunks below mean to die-1 chunks -> die 0
  std::vector<int> sm_die(256, 0); int n0 = 0;
  int consistent = 0;
  for (int b = 0; b < nsm; ++b) {
    double a0 = 0, a1 = 0; int c0 = 0, c1 = 0;
    for (int c = 0; c < kNCh; ++c) { if (chdie[c]) { a1 += L[(size_t)b * kNCh + c]; ++c1; } else { a0 += L[(size_t)b * kNCh + c]; ++c0; } }
    a0 /= c0; a1 /= c1;
    const int d = a0 < a1 ? 0 : 1;
    sm_die[smofb[b]] = d; n0 += d == 0;
    // agreement of this SM's per-chunk near/far with the chunk labels
    int agree = 0;
    for (int c = 0; c < kNCh; ++c) agree += ((L[(size_t)b * kNCh + c] < (a0 + a1) / 2) ? (d == 0 ? 0 : 1) : (d == 0 ? 1 : 0)) == chdie[c];
    consistent += agree > 0.95 * kNCh;
    if (b < 4 || b == nsm - 1) printf("  block %d sm %d: die %d, near %.1f far %.1f, label agreement %.3f\n", b, smofb[b], d,
                                      std::min(a0, a1), std::max(a0, a1), (double)agree / kNCh);
  }
  printf("SMs on die 0: %d, die 1: %d; SMs whose per-chunk pattern agrees >95%% with the labels: %d/%d\n", n0, nsm - n0, consistent, nsm);
  // per-die copies from disjoint chunks: [h die0, h die1, dh die0, dh die1], kLines/16 chunks each
  const int need = kLines / kLinesPerChunk;
  std::vector<int> off(4 * need);
  int k[2] = {0, 0};
  for (int c = 0; c < kNCh; ++c) {
    const int d = chdie[c];
    if (k[d] < 2 * need) { const int slot = k[d] < need ? d : 2 + d; off[slot * need + (k[d] % need)] = c; ++k[d]; }
  }
  if (k[0] < 2 * need || k[1] < 2 * need) { printf("not enough chunks per die\n"); return 1; }
  int* doff; int* dsm; CK(cudaMalloc(&doff, off.size() * 4)); CK(cudaMalloc(&dsm, 256 * 4));
  CK(cudaMemcpy(doff, off.data(), off.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dsm, sm_die.data(), 256 * 4, cudaMemcpyHostToDevice));
  // connections
  const long nconn = 670091L * 32;
  std::vector<int> hidx(nconn); uint64_t s = 88172645463325252ull;
  for (long i = 0; i < nconn; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; hidx[i] = (int)(s % kLines); }
  int* idx; CK(cudaMalloc(&idx, nconn * 4)); CK(cudaMemcpy(idx, hidx.data(), nconn * 4, cudaMemcpyHostToDevice));
  float *plain, *hd, *out; CK(cudaMalloc(&plain, (long)kLines * 128)); CK(cudaMalloc(&hd, (long)kLines * 256)); CK(cudaMalloc(&out, 4));
  CK(cudaMemset(plain, 0, (long)kLines * 128)); CK(cudaMemset(hd, 0, (long)kLines * 256));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  auto timeit = [&](const char* name, double bytes, auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
      CK(cudaEventRecord(e0)); launch(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); best = std::min(best, ms);
    }
    CK(cudaGetLastError());
    printf("%-34s %9.1f us  %8.1f GB/s\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9);
  };
  const double gb = (double)nconn * 128;
  const char* mname[3] = {"plain", "own-die copy", "other-die copy"};
  for (int bpsm : {4, 8}) {
    const int grid = nsm * bpsm;
    char nm[64];
    for (int mode = 0; mode < 3; ++mode) {
      snprintf(nm, 64, "gather %s g=%d", mname[mode], grid);
      timeit(nm, gb, [&] { k_gather<<<grid, 256>>>(idx, nconn, plain, buf, doff, dsm, mode, out); });
    }
    for (int mode = 0; mode < 3; ++mode) {
      snprintf(nm, 64, "red.v4 %s g=%d", mname[mode], grid);
      timeit(nm, gb, [&] { k_red<<<grid, 256>>>(idx, nconn, plain, buf, doff, dsm, mode, 0, hd, out); });
    }
    for (int mode = 0; mode < 3; ++mode) {
      snprintf(nm, 64, "gather+red %s g=%d", mname[mode], grid);
      timeit(nm, 2 * gb, [&] { k_red<<<grid, 256>>>(idx, nconn, hd, buf, doff, dsm, mode, 1, hd, out); });
    }
  }
  return 0;
}
