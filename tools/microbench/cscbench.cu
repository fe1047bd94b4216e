// The complete access pattern of one CSC-mode training step at Amazon-670K (VERDICT r1,
// next-round item 3): what the row pass and the column pass cost when they do nothing but
// move their bytes, for the hand-off variants of the pre-update weights W_old.
//
//   row pass (warp per label row, rows in label tiles):
//     state stream: read W, idx, mW, vW (128 B each, coalesced), write W, mW, vW;
//     gather the row's 32 h lines (128 B each, random, L2-resident hd);
//     hand-off  R0: write the g line only (no W_old)                       [floor]
//               R1: write g line + W_old line into the row's record          [built: record]
//               R2: write g line + scatter W_old to its CSC position pos[e]  [round-1 design]
//   column pass (warp per column, entries of one tile):
//     read the entry stream (4 B / entry, coalesced), gather one g line per entry;
//     W_old     C0: none (w = 1)                                            [floor]
//               C1: one 4-B load from the entry's record (random sector)    [built: record]
//               C2: coalesced read of wcsc in CSC order                     [round-1 design]
//   and the atomic design's pattern (gather + red.v4 line) for reference.
//
// Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cscbench cscbench.cu
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ float4 ldv4(const float* a) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a));
  return v;
}
__device__ __forceinline__ float ldna(const float* a) {
  float v; asm volatile("ld.global.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(a)); return v;
}
__device__ __forceinline__ int ldnai(const int* a) {
  int v; asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(a)); return v;
}
__device__ __forceinline__ void red_v4(float* a, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

// HAND: 0 = g line only, 1 = g + W_old line (record, 64 floats/row), 2 = g + scatter to pos; 3 = atomic red
template <int HAND>
__global__ void __launch_bounds__(256) k_row(float* W, const int* __restrict__ idx, float* mW, float* vW,
                                             const int* __restrict__ pos, float* wcsc, float* hd, float* rec,
                                             int64_t j0, int64_t j1, float* out) {
  const int lane = threadIdx.x & 31, gq = lane >> 3, bq = lane & 7;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  for (int64_t j = j0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); j < j1; j += nw) {
    const int64_t r = j * 32 + lane;
    float w = ldna(W + r), mw = ldna(mW + r), vw = ldna(vW + r);
    const int c = ldnai(idx + r);
    float4 hv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int cq = __shfl_sync(~0u, c, 4 * q + gq);
      hv[q] = ldv4(hd + (size_t)cq * 64 + 4 * bq);
    }
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += hv[q].x + hv[q].y + hv[q].z + hv[q].w;
    const float g = s * 1e-30f;
    if (HAND == 3) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int cq = __shfl_sync(~0u, c, 4 * q + gq);
        red_v4(hd + (size_t)cq * 64 + 32 + 4 * bq, make_float4(g, g, g, g));
      }
    } else {
      float* rr = rec + (j - j0) * (HAND == 1 ? 64 : 32);
      rr[lane] = g;
      if (HAND == 1) rr[32 + lane] = w;
      if (HAND == 2) wcsc[ldnai(pos + r)] = w;
    }
    w += g; mw += g; vw += g;
    W[r] = w; mW[r] = mw; vW[r] = vw;
    acc += s;
  }
  if (acc == 1234.5f) out[0] = acc;
}

// hybrid row pass: gather the row's h lines, red.v4 the contributions of the connections whose
// column is < split (the L1 -> XBAR egress path), write the record (g line + W_old line) for the
// column pass, which pulls the columns >= split (the XBAR -> L1 ingress path)
__global__ void __launch_bounds__(256) k_row_hyb(float* W, const int* __restrict__ idx, float* mW, float* vW,
                                                 float* hd, float* rec, int64_t j0, int64_t j1, int split, float* out) {
  const int lane = threadIdx.x & 31, gq = lane >> 3, bq = lane & 7;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  for (int64_t j = j0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); j < j1; j += nw) {
    const int64_t r = j * 32 + lane;
    float w = ldna(W + r), mw = ldna(mW + r), vw = ldna(vW + r);
    const int c = ldnai(idx + r);
    float4 hv[8]; int cq[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      cq[q] = __shfl_sync(~0u, c, 4 * q + gq);
      hv[q] = ldv4(hd + (size_t)cq[q] * 64 + 4 * bq);
    }
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += hv[q].x + hv[q].y + hv[q].z + hv[q].w;
    const float g = s * 1e-30f;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (cq[q] < split) red_v4(hd + (size_t)cq[q] * 64 + 32 + 4 * bq, make_float4(g, g, g, g));
    float* rr = rec + (j - j0) * 64;
    rr[lane] = g;
    rr[32 + lane] = w;
    w += g; mw += g; vw += g;
    W[r] = w; mW[r] = mw; vW[r] = vw;
    acc += s;
  }
  if (acc == 1234.5f) out[0] = acc;
}

// HAND: 0 = no W, 1 = W from the record (random sector), 2 = W coalesced from wcsc
template <int HAND>
__global__ void __launch_bounds__(256) k_col(const int* __restrict__ cp, const int* __restrict__ ent,
                                             const float* __restrict__ wcsc, const float* __restrict__ rec, int m,
                                             float* hd, int c_begin = 0) {
  const int lane = threadIdx.x & 31, gq = lane >> 3, bq = lane & 7;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int rs = HAND == 1 ? 64 : 32;
  for (int c = c_begin + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); c < m; c += nw) {
    const int p0 = cp[c], p1 = cp[c + 1];
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int p = p0; p < p1; p += 32) {
      const bool ok = p + lane < p1;
      const int e = ok ? ldnai(ent + p + lane) : 0;
      const int row = e >> 6, slot = e & 63;
      float4 gv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int rw = __shfl_sync(~0u, row, 4 * u + gq);
        gv[u] = (p + 4 * u + gq < p1) ? ldv4(rec + (size_t)rw * rs + 4 * bq) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      float wv = 1.0f;
      if (HAND == 1 && ok) wv = ldna(rec + (size_t)row * rs + 32 + slot);
      if (HAND == 2 && ok) wv = ldna(wcsc + p + lane);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float ww = __shfl_sync(~0u, wv, 4 * u + gq);
        acc.x += ww * gv[u].x; acc.y += ww * gv[u].y; acc.z += ww * gv[u].z; acc.w += ww * gv[u].w;
      }
    }
#pragma unroll
    for (int o = 8; o <= 16; o <<= 1) {
      acc.x += __shfl_xor_sync(~0u, acc.x, o); acc.y += __shfl_xor_sync(~0u, acc.y, o);
      acc.z += __shfl_xor_sync(~0u, acc.z, o); acc.w += __shfl_xor_sync(~0u, acc.w, o);
    }
    if (gq == 0) *reinterpret_cast<float4*>(hd + (size_t)c * 64 + 32 + 4 * bq) = acc;
  }
}

// ceilings of the pieces: random 128-B line gathers (ld.v4, 8 lanes per line) and random 4-B
// loads (one sector per lane), both driven by a coalesced index stream, many in flight per lane
template <bool LINES>
__global__ void __launch_bounds__(256) k_pieces(const int* __restrict__ ent, int64_t n, const float* __restrict__ rec,
                                                int rs, float* out) {
  const int lane = threadIdx.x & 31, gq = lane >> 3, bq = lane & 7;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b * 32 < n; b += nw) {
    const int e = ldnai(ent + b * 32 + lane);
    const int row = e >> 6, slot = e & 63;
    if (LINES) {
      float4 gv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) gv[u] = ldv4(rec + (size_t)__shfl_sync(~0u, row, 4 * u + gq) * rs + 4 * bq);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += gv[u].x + gv[u].y + gv[u].z + gv[u].w;
    } else {
      acc += ldna(rec + (size_t)row * rs + 32 + slot);
    }
  }
  if (acc == 1234.5f) out[0] = acc;
}

// SM egress: random 128-B line stores vs red.v4 lines (8 lanes per line, 4 lines per warp
// instruction) into an L2-resident buffer of `lines` lines, driven by the entry stream
template <bool RED>
__global__ void __launch_bounds__(256) k_egress(const int* __restrict__ ent, int64_t n, float* buf, int lines) {
  const int lane = threadIdx.x & 31, gq = lane >> 3, bq = lane & 7;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b * 32 < n; b += nw) {
    const int e = ldnai(ent + b * 32 + lane);
    const uint32_t ln = ((uint32_t)e * 2654435761u) % (uint32_t)lines;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      float* a = buf + (size_t)__shfl_sync(~0u, ln, 4 * u + gq) * 32 + 4 * bq;
      const float4 v = make_float4(1e-30f, 1e-30f, 1e-30f, 1e-30f);
      if (RED) red_v4(a, v);
      else asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
    }
  }
}

int main(int argc, char** argv) {
  CK(cudaSetDevice(0));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  const int nsm = p.multiProcessorCount;
  const int m = 32768;
  const int64_t L = 670091, k = 32, n = L * k;
  const int ntile = argc > 1 ? atoi(argv[1]) : 5;
  const int64_t tile = (L + ntile - 1) / ntile;
  printf("device %s, L=%lld m=%d k=%lld, %d label tiles of %lld rows\n", p.name, (long long)L, m, (long long)k, ntile,
         (long long)tile);
  // random distinct columns per row; CSC per tile: entries sorted by (tile, column, row)
  std::vector<int> hidx(n);
  uint64_t s = 88172645463325252ull;
  for (int64_t j = 0; j < L; ++j)
    for (int i = 0; i < 32; ++i) {
      int c;
      bool dup;
      do {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17; c = (int)(s % m);
        dup = false;
        for (int q = 0; q < i; ++q) dup |= hidx[j * 32 + q] == c;
      } while (dup);
      hidx[j * 32 + i] = c;
    }
  std::vector<int> cnt((size_t)ntile * m + 1, 0), hent(n), hpos(n);
  for (int64_t e = 0; e < n; ++e) cnt[(e / 32 / tile) * m + hidx[e] + 1]++;
  for (size_t q = 1; q < cnt.size(); ++q) cnt[q] += cnt[q - 1];
  std::vector<int> fill(cnt.begin(), cnt.end() - 1);
  for (int64_t e = 0; e < n; ++e) {
    const int64_t j = e / 32, t = j / tile;
    const int q = fill[t * m + hidx[e]]++;
    hent[q] = (int)(((j - t * tile) << 6) | (e & 31));
    hpos[e] = q;
  }
  int *idx, *cp, *ent, *pos; float *W, *mW, *vW, *hd, *rec, *wcsc, *out;
  CK(cudaMalloc(&idx, n * 4)); CK(cudaMalloc(&ent, n * 4)); CK(cudaMalloc(&pos, n * 4));
  CK(cudaMalloc(&cp, cnt.size() * 4));
  CK(cudaMemcpy(idx, hidx.data(), n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ent, hent.data(), n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(pos, hpos.data(), n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(cp, cnt.data(), cnt.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&W, n * 4)); CK(cudaMalloc(&mW, n * 4)); CK(cudaMalloc(&vW, n * 4)); CK(cudaMalloc(&wcsc, n * 4));
  CK(cudaMemset(W, 0, n * 4)); CK(cudaMemset(mW, 0, n * 4)); CK(cudaMemset(vW, 0, n * 4));
  CK(cudaMalloc(&hd, (size_t)m * 64 * 4)); CK(cudaMemset(hd, 0, (size_t)m * 256));
  CK(cudaMalloc(&rec, (size_t)tile * 64 * 4)); CK(cudaMemset(rec, 0, (size_t)tile * 256));
  CK(cudaMalloc(&out, 4));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const int grid_row = nsm * 8, grid_col = nsm * 8;
  auto timeit = [&](const char* name, auto launch) {
    for (int w = 0; w < 2; ++w) launch();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 7; ++r) {
      CK(cudaEventRecord(e0)); launch(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); best = std::min(best, ms);
    }
    CK(cudaGetLastError());
    printf("%-58s %8.1f us\n", name, best * 1e3);
  };
  auto rows = [&](int hand, int t) {
    const int64_t j0 = t * tile, j1 = std::min<int64_t>(L, j0 + tile);
    if (hand == 0) k_row<0><<<grid_row, 256>>>(W, idx, mW, vW, pos, wcsc, hd, rec, j0, j1, out);
    if (hand == 1) k_row<1><<<grid_row, 256>>>(W, idx, mW, vW, pos, wcsc, hd, rec, j0, j1, out);
    if (hand == 2) k_row<2><<<grid_row, 256>>>(W, idx, mW, vW, pos, wcsc, hd, rec, j0, j1, out);
    if (hand == 3) k_row<3><<<grid_row, 256>>>(W, idx, mW, vW, pos, wcsc, hd, rec, j0, j1, out);
  };
  auto cols = [&](int hand, int t) {
    if (hand == 0) k_col<0><<<grid_col, 256>>>(cp + (size_t)t * m, ent, wcsc, rec, m, hd);
    if (hand == 1) k_col<1><<<grid_col, 256>>>(cp + (size_t)t * m, ent, wcsc, rec, m, hd);
    if (hand == 2) k_col<2><<<grid_col, 256>>>(cp + (size_t)t * m, ent, wcsc, rec, m, hd);
  };
  for (int t = 0; t < 1; ++t) {
    const int64_t ne = std::min<int64_t>(n, tile * 32);     // the entries of one tile (CSC order)
    char nm[96];
    snprintf(nm, 96, "pieces: %lld random 128-B line gathers (x%d = all tiles)", (long long)ne, ntile);
    timeit(nm, [&] { for (int q = 0; q < ntile; ++q) k_pieces<true><<<grid_col, 256>>>(ent, ne, rec, 64, out); });
    snprintf(nm, 96, "pieces: %lld random 4-B loads (x%d = all tiles)", (long long)ne, ntile);
    timeit(nm, [&] { for (int q = 0; q < ntile; ++q) k_pieces<false><<<grid_col, 256>>>(ent, ne, rec, 64, out); });
  }
  {
    float* buf; const int lines4 = 32768, lines40 = 40 << 13;   // 4 MiB and 40 MiB
    CK(cudaMalloc(&buf, (size_t)lines40 * 128)); CK(cudaMemset(buf, 0, (size_t)lines40 * 128));
    const int64_t ne = std::min<int64_t>(n, tile * 32);
    char nm[96];
    for (int lines : {lines4, lines40}) {
      snprintf(nm, 96, "egress: %lld random line STORES into %d MiB (x%d)", (long long)ne, lines / 8192, ntile);
      timeit(nm, [&] { for (int q = 0; q < ntile; ++q) k_egress<false><<<grid_col, 256>>>(ent, ne, buf, lines); });
      snprintf(nm, 96, "egress: %lld random line REDs into %d MiB (x%d)", (long long)ne, lines / 8192, ntile);
      timeit(nm, [&] { for (int q = 0; q < ntile; ++q) k_egress<true><<<grid_col, 256>>>(ent, ne, buf, lines); });
    }
  }
  {
    // hybrid, sequential (row t; column t) vs software-pipelined on two streams (row t+1 || column t),
    // two record buffers; row grid gets RB CTAs/SM, the column grid CB CTAs/SM
    float* rec2; CK(cudaMalloc(&rec2, (size_t)tile * 64 * 4)); CK(cudaMemset(rec2, 0, (size_t)tile * 256));
    cudaStream_t s1, s2; CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    cudaEvent_t er[16], ec[16];
    for (int q = 0; q < 16; ++q) { CK(cudaEventCreateWithFlags(&er[q], cudaEventDisableTiming)); CK(cudaEventCreateWithFlags(&ec[q], cudaEventDisableTiming)); }
    for (double f : {0.0, 0.3, 0.45, 0.6, 1.0}) {
      const int split = (int)(f * m);
      for (int rb : {2, 4}) for (int cb : {2, 4}) {
        char nm[120];
        auto rowk = [&](int t, cudaStream_t st) {
          const int64_t j0 = t * tile, j1 = std::min<int64_t>(L, j0 + tile);
          k_row_hyb<<<nsm * rb, 256, 0, st>>>(W, idx, mW, vW, hd, (t & 1) ? rec2 : rec, j0, j1, split, out);
        };
        auto colk = [&](int t, cudaStream_t st) {
          k_col<1><<<nsm * cb, 256, 0, st>>>(cp + (size_t)t * m, ent, wcsc, (t & 1) ? rec2 : rec, m, hd, split);
        };
        if (rb == 4 && cb == 4) {
          snprintf(nm, 120, "hybrid f=%.2f sequential (row t; col t)", f);
          timeit(nm, [&] { for (int t = 0; t < ntile; ++t) { rowk(t, 0); if (split < m) colk(t, 0); } });
        }
        snprintf(nm, 120, "hybrid f=%.2f pipelined rows %d/SM || cols %d/SM", f, rb, cb);
        timeit(nm, [&] {
          CK(cudaEventRecord(er[15], 0)); CK(cudaStreamWaitEvent(s1, er[15])); CK(cudaStreamWaitEvent(s2, er[15]));
          for (int t = 0; t < ntile; ++t) {
            if (t >= 2) CK(cudaStreamWaitEvent(s1, ec[t - 2]));     // record buffer t&1 free again
            rowk(t, s1); CK(cudaEventRecord(er[t], s1));
            if (split < m) { CK(cudaStreamWaitEvent(s2, er[t])); colk(t, s2); }
            CK(cudaEventRecord(ec[t], s2));
          }
          CK(cudaEventRecord(er[14], s2)); CK(cudaStreamWaitEvent(0, er[14]));
          CK(cudaEventRecord(er[13], s1)); CK(cudaStreamWaitEvent(0, er[13]));
        });
      }
    }
  }
  timeit("atomic: row pass with gather + red.v4 (1 launch)", [&] { rows(3, 0); for (int t = 1; t < ntile; ++t) rows(3, t); });
  const char* rn[3] = {"R0 g line only", "R1 g + W_old line (record)", "R2 g + W_old scatter to pos[e]"};
  const char* cn[3] = {"C0 no W", "C1 W sector from the record", "C2 W coalesced (wcsc)"};
  for (int h = 0; h < 3; ++h) {
    char nm[96];
    snprintf(nm, 96, "row pass %s (all tiles)", rn[h]);
    timeit(nm, [&] { for (int t = 0; t < ntile; ++t) rows(h, t); });
  }
  for (int h = 0; h < 3; ++h) {
    char nm[96];
    snprintf(nm, 96, "column pass %s (all tiles)", cn[h]);
    timeit(nm, [&] { for (int t = 0; t < ntile; ++t) cols(h, t); });
  }
  for (int h = 0; h < 3; ++h) {
    char nm[96];
    snprintf(nm, 96, "row + column, %s / %s", rn[h], cn[h]);
    timeit(nm, [&] { for (int t = 0; t < ntile; ++t) { rows(h, t); cols(h, t); } });
  }
  return 0;
}
