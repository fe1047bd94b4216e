// ff_dense.cuh — sm_100a kernels of the intermediate layer of the proposed architecture
// (SURVEY §8(f) NEXT-2): features -> input dropout -> dense W_d (P:594-603,
// Fig. 2) -> ReLU (reading R18) -> the fixed fan-in layer.
//
// Layouts:
//   Wd, mWd, vWd, dWd  f32 tiled [ldw/128][d][128], ldw = m rounded up to 128 (the pad
//                      columns stay 0): element (f, c) at ((c/128)*d + f)*128 + c%128, so a
//                      CTA's 128-column tile over all features is one contiguous range of
//                      HBM;
//   bd, mbd, vbd, dbd  f32 [ldw];
//   xT  f32 [d][ldx], ldx = 32*nb: the dropped-out, scaled features, transposed so that
//       the 32 samples of one feature are one 128-B line (broadcast operand);
//   hd  the fixed fan-in layer's h|dh column lines [m][nb][64] (ff_kernels.cuh): the
//       forward writes h = ReLU(z) into the h half (and zeroes the dh half), the backward
//       reads the ReLU mask from the h half and dh from the dh half.  No tensor cores: at
//       the paper's B = 32 the layer is a 32-row GEMM whose backward + Adam is bound by
//       streaming Wd and its moments (24 B per weight), not by FMAs.
#pragma once
#include <cuda.h>   // CUtensorMap
#include <cstdio>
#include "ff_device.cuh"
#include "ff_kernels.cuh"   // cp.async helpers

namespace ff {

constexpr uint32_t kDomDropout = 3;

// streamed 16-B accesses of the dense layer's Adam state (no L1 allocation)
__device__ __forceinline__ float4 ld_na4(const float* a) {
  float4 v;
  asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a));
  return v;
}
__device__ __forceinline__ void st_na4(float* a, float4 v) {
  asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};"
               :: "l"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

// Input dropout (reading R25): xT[f][b] = x[b][f] * scale if word f of the
// Philox stream (ctr = (f/4, b, step, 3), key = seed) has (u >> 8) * 2^-24 >= p, else 0.
// train = 0: xT = x (inference, no dropout).  Samples B..ldx-1 are 0.  Thread per (b, f/4).
// xTlo (tensor-core forward, may be NULL): xT - (xT with the 13 low mantissa bits cleared),
// the exact lo part of the 3xTF32 split (k_dense_fwd_tma).
__global__ void k_dropout_T(const float* __restrict__ x, int B, int d, int ldx, float p, float scale, int train,
                            uint32_t step, uint32_t key0, uint32_t key1, float* __restrict__ xT,
                            const int64_t* __restrict__ t_auto, float* __restrict__ xTlo) {
  // the tensor-core forward is launched as this kernel's programmatic dependent: it may start
  // (TMEM/barrier set-up, the first Wd stages) now and waits (griddepcontrol.wait) before it
  // reads xT / xTlo
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // t_auto (FF_STEP_AUTO): the step key is the dense layer's device counter + 1, i.e. the
  // Adam step this forward belongs to (read before k_prep / k_step_t advance it)
  if (t_auto != nullptr) step = (uint32_t)(*t_auto + 1);
  const int nq = (d + 3) / 4;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)ldx * nq;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(e / nq), q = (int)(e % nq);
    U4 v{0u, 0u, 0u, 0u};
    if (train && b < B) v = philox((uint32_t)q, (uint32_t)b, step, kDomDropout, key0, key1);
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int f = 4 * q + w;
      if (f >= d) break;
      float val = 0.0f;
      if (b < B) {
        const float xv = x[(int64_t)b * d + f];
        if (!train) {
          val = xv;
        } else {
          const float unit = __fmul_rn((float)(word_of(v, w) >> 8), 1.0f / 16777216.0f);   // exact
          val = unit >= p ? __fmul_rn(xv, scale) : 0.0f;
        }
      }
      xT[(int64_t)f * ldx + b] = val;
      if (xTlo != nullptr) xTlo[(int64_t)f * ldx + b] = val - __uint_as_float(__float_as_uint(val) & 0xFFFFE000u);
    }
  }
}

// Forward: z[b][c] = bd[c] + sum_f xT[f][b] Wd[f][c], h = max(z, 0).  CTA = 256 threads ->
// 128 columns x 32 samples (chunk blockIdx.y).  The Wd tile (32 features x 128 columns,
// 16 KB) and the xT tile (32 x 32) of the next feature chunk are copied into a second
// shared-memory stage (cp.async) while the current chunk is computed, so the HBM latency of
// Wd hides behind the FMAs.  Warp w: lane -> 4 columns, samples 8(w&3)..+7, and the first
// (w < 4) or second (w >= 4) half of every chunk's features: a thread's 32 accumulators
// amortise each 16-B shared load of Wd over 8 samples (the kernel is bound by shared-memory
// wavefronts, not FMAs).  For B <= 32 the chunks are also split over two CTAs (gridDim.z =
// 2, for occupancy: one 32-sample chunk gives only m/128 CTAs).  Summation order, fixed:
// per CTA (bd + first halves) + second halves, f ascending within each; then CTA 0 + CTA 1.
#ifndef FF_DENSE_FCH
#define FF_DENSE_FCH 64
#endif
#ifndef FF_DENSE_SPLIT
#define FF_DENSE_SPLIT 1
#endif
constexpr int kDenseFwdThreads = 256, kDenseFch = FF_DENSE_FCH, kDenseFwdSplit = FF_DENSE_SPLIT;
constexpr int kDenseFwdSmem = 2 * kDenseFch * (128 + 32) * 4;
__device__ __forceinline__ void cp_async16_zfill(uint32_t dst, const float* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" :: "r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
}
__global__ void __launch_bounds__(kDenseFwdThreads) k_dense_fwd(const float* __restrict__ Wd,
                                                                const float* __restrict__ bd,
                                                                const float* __restrict__ xT, int d, int m, int ldw,
                                                                int ldx, int B, float* __restrict__ hd, int cstride,
                                                                int zero_dh, float* __restrict__ h_out,
                                                                float* __restrict__ zpart, unsigned* __restrict__ cnt) {
  extern __shared__ __align__(16) float dsm[];
  float* const wbuf = dsm;                                   // [2][kDenseFch][128]
  float* const xbuf = dsm + 2 * kDenseFch * 128;             // [2][kDenseFch][32]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, q2 = blockIdx.y;
  const int sg = w & 3, half = w >> 2;                       // samples 8sg..8sg+7; feature half
  const int ct = blockIdx.x * 128, c0 = ct + 4 * lane;
  const bool cok = c0 < ldw;
  // split over CTAs (gridDim.z = 2, B <= 32): CTA kz takes chunks [ch_lo, ch_hi); the two
  // partial sums meet in zpart and the second CTA to finish adds them (part 0 + part 1)
  const int nch_all = (d + kDenseFch - 1) / kDenseFch, kz = blockIdx.z;
  const int ch_lo = kz == 0 ? 0 : (nch_all + 1) / 2, ch_hi = gridDim.z == 1 || kz == 1 ? nch_all : (nch_all + 1) / 2;
  auto issue = [&](int ch) {
    const int f0 = ch * kDenseFch, stg = ch & 1;
    const uint32_t wdst = (uint32_t)__cvta_generic_to_shared(wbuf + stg * kDenseFch * 128);
    const uint32_t xdst = (uint32_t)__cvta_generic_to_shared(xbuf + stg * kDenseFch * 32);
#pragma unroll
    for (int u = 0; u < kDenseFch * 32 / kDenseFwdThreads; ++u) {   // kDenseFch rows x 32 float4
      const int e = u * kDenseFwdThreads + threadIdx.x, r = e >> 5, cq = (e & 31) * 4;
      const bool ok = f0 + r < d && ct + cq < ldw;
      cp_async16_zfill(wdst + (uint32_t)(r * 128 + cq) * 4u,
                       ok ? Wd + ((int64_t)blockIdx.x * d + f0 + r) * 128 + cq : Wd, ok);
    }
    static_assert(kDenseFch * 8 % kDenseFwdThreads == 0, "xT tile copy");
#pragma unroll
    for (int u = 0; u < kDenseFch * 8 / kDenseFwdThreads; ++u) {    // kDenseFch rows x 8 float4
      const int e = u * kDenseFwdThreads + threadIdx.x, r = e >> 3, s4 = (e & 7) * 4;
      const bool ok = f0 + r < d;
      cp_async16_zfill(xdst + (uint32_t)(r * 32 + s4) * 4u, ok ? xT + (int64_t)(f0 + r) * ldx + q2 * 32 + s4 : xT, ok);
    }
    cp_async_commit();
  };
  float4 bias4 = make_float4(0.f, 0.f, 0.f, 0.f);
  if (cok && half == 0 && kz == 0) bias4 = *reinterpret_cast<const float4*>(bd + c0);
  float2 acc[8][2];
#pragma unroll
  for (int s = 0; s < 8; ++s) { acc[s][0] = make_float2(bias4.x, bias4.y); acc[s][1] = make_float2(bias4.z, bias4.w); }
  if (ch_lo < ch_hi) issue(ch_lo);
  for (int ch = ch_lo; ch < ch_hi; ++ch) {
    if (ch + 1 < ch_hi) { issue(ch + 1); cp_async_wait<1>(); } else { cp_async_wait<0>(); }
    __syncthreads();
    const int nf = min(kDenseFch, d - ch * kDenseFch);
    const int r0 = half * (kDenseFch / 2), r1 = min(nf, r0 + kDenseFch / 2);
    const float* wt = wbuf + (ch & 1) * kDenseFch * 128 + 4 * lane;
    const float* xt = xbuf + (ch & 1) * kDenseFch * 32 + 8 * sg;
#pragma unroll 4
    for (int r = r0; r < r1; ++r) {
      const float4 w4 = *reinterpret_cast<const float4*>(wt + r * 128);
      const float4 xa = *reinterpret_cast<const float4*>(xt + r * 32);
      const float4 xb = *reinterpret_cast<const float4*>(xt + r * 32 + 4);
      const float xv[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        acc[s][0] = ffma2(bc2(xv[s]), make_float2(w4.x, w4.y), acc[s][0]);
        acc[s][1] = ffma2(bc2(xv[s]), make_float2(w4.z, w4.w), acc[s][1]);
      }
    }
    __syncthreads();                                         // stage ch & 1 is refilled next
  }
  // second-half warps hand their partial sums to the first-half warps (stage buffers reused)
  float* const part = dsm + (size_t)(w & 3) * 32 * 33;       // [lane][33] per sample group
  if (half == 1) {
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      part[lane * 33 + 4 * s + 0] = acc[s][0].x; part[lane * 33 + 4 * s + 1] = acc[s][0].y;
      part[lane * 33 + 4 * s + 2] = acc[s][1].x; part[lane * 33 + 4 * s + 3] = acc[s][1].y;
    }
  }
  __syncthreads();
  float zz[8][4];
  if (half == 0) {
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      zz[s][0] = __fadd_rn(acc[s][0].x, part[lane * 33 + 4 * s + 0]);
      zz[s][1] = __fadd_rn(acc[s][0].y, part[lane * 33 + 4 * s + 1]);
      zz[s][2] = __fadd_rn(acc[s][1].x, part[lane * 33 + 4 * s + 2]);
      zz[s][3] = __fadd_rn(acc[s][1].y, part[lane * 33 + 4 * s + 3]);
    }
  }
  if (gridDim.z > 1) {
    // zpart[kz][c][32 samples] (B <= 32 here); the last of the two CTAs of this tile combines
    __shared__ unsigned s_last;
    if (half == 0 && cok) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float* zp = zpart + ((int64_t)kz * ldw + c0 + u) * 32 + 8 * sg;
        __stcg(reinterpret_cast<float4*>(zp), make_float4(zz[0][u], zz[1][u], zz[2][u], zz[3][u]));
        __stcg(reinterpret_cast<float4*>(zp + 4), make_float4(zz[4][u], zz[5][u], zz[6][u], zz[7][u]));
      }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      s_last = atomicAdd(cnt + blockIdx.x, 1u) == 1u;
      if (s_last) cnt[blockIdx.x] = 0u;                      // ready for the next launch
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (half == 0 && cok) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float* z0p = zpart + ((int64_t)0 * ldw + c0 + u) * 32 + 8 * sg;
        const float* z1p = zpart + ((int64_t)1 * ldw + c0 + u) * 32 + 8 * sg;
        const float4 a0 = __ldcg(reinterpret_cast<const float4*>(z0p)), a1 = __ldcg(reinterpret_cast<const float4*>(z0p + 4));
        const float4 b0 = __ldcg(reinterpret_cast<const float4*>(z1p)), b1 = __ldcg(reinterpret_cast<const float4*>(z1p + 4));
        zz[0][u] = __fadd_rn(a0.x, b0.x); zz[1][u] = __fadd_rn(a0.y, b0.y);
        zz[2][u] = __fadd_rn(a0.z, b0.z); zz[3][u] = __fadd_rn(a0.w, b0.w);
        zz[4][u] = __fadd_rn(a1.x, b1.x); zz[5][u] = __fadd_rn(a1.y, b1.y);
        zz[6][u] = __fadd_rn(a1.z, b1.z); zz[7][u] = __fadd_rn(a1.w, b1.w);
      }
    }
  }
  if (half == 1 || !cok) return;
  float hv[8][4];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int b = q2 * 32 + 8 * sg + s;
    const bool valid = b < B;
    const float z0 = zz[s][0], z1 = zz[s][1], z2 = zz[s][2], z3 = zz[s][3];
    hv[s][0] = valid ? fmaxf(z0, 0.0f) : 0.0f;
    hv[s][1] = valid ? fmaxf(z1, 0.0f) : 0.0f;
    hv[s][2] = valid ? fmaxf(z2, 0.0f) : 0.0f;
    hv[s][3] = valid ? fmaxf(z3, 0.0f) : 0.0f;
    if (h_out != nullptr && valid) {
      float* hp = h_out + (int64_t)b * m + c0;
      if ((m & 3) == 0 && c0 + 3 < m) {                // 16-B aligned rows only
        *reinterpret_cast<float4*>(hp) = make_float4(hv[s][0], hv[s][1], hv[s][2], hv[s][3]);
      } else {
        for (int u = 0; u < 4 && c0 + u < m; ++u) hp[u] = hv[s][u];
      }
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int c = c0 + u;
    if (c >= m) break;
    float* line = hd + (int64_t)c * cstride + q2 * 64 + 8 * sg;
    *reinterpret_cast<float4*>(line) = make_float4(hv[0][u], hv[1][u], hv[2][u], hv[3][u]);
    *reinterpret_cast<float4*>(line + 4) = make_float4(hv[4][u], hv[5][u], hv[6][u], hv[7][u]);
    if (zero_dh) {
      *reinterpret_cast<float4*>(line + 32) = make_float4(0.f, 0.f, 0.f, 0.f);
      *reinterpret_cast<float4*>(line + 36) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
}

// ------------------------------------------------------------------ tensor-core forward
// The forward on the 5th-generation tensor cores (tcgen05, kind::tf32) for B <= 32, fed by
// TMA: per 128-column tile D[128 columns][32 samples] (fp32, in TMEM) = sum over 8-feature
// blocks of A[128][8] . B[8][32], A = Wd^T and B = xT read in place from their HBM layouts:
// both are MN-major (the tile's 128 columns, resp. the 32 samples, contiguous per feature),
// which kind::tf32 accepts only in the 128-B swizzle with 32-B atoms (descriptor layout 1,
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B; tools/microbench/tcprobe_mn.cu pins LBO = 4096 B
// between 32-column groups and SBO = 512 B between 4-feature groups).
// fp32 accuracy from 3xTF32: a = a_hi + a_lo exactly, a_hi = a with the 13 low mantissa bits
// cleared; a.b ~ a_hi.b_hi + a_hi.b_lo + a_lo.b_hi (the dropped a_lo.b_lo and the tf32
// truncation of the lo parts are <= ~2^-20 relative).  The tensor core itself truncates fp32
// operands to tf32 (tcprobe_mn: 1 + 3*2^-12 -> 1), so the raw TMA tiles ARE the hi operands;
// xT's lo is written once per forward by k_dropout_T, and Wd's lo per stage by four converter
// warps straight into TMEM (thread = A row = tile column: it reads its column's features from
// the swizzled raw tile, byte f*128 + ((4 c) ^ ((f & 3) << 5)) per tools/microbench/swzprobe.cu,
// and tcgen05.st's them into its TMEM lane), so A_lo never touches shared memory and its MMAs
// read A from TMEM.  Per 8-feature block two MMAs: A_hi . [x_hi | x_lo] (one N = 64 MMA: x_lo
// is the next 32-sample atom) and A_lo(TMEM) . x_hi (N = 32), into separate TMEM columns the
// epilogue sums in a fixed order (tools/microbench/tcrate.cu: an M = 128 MMA costs
// max(67, N / 2) cycles, so merging the x parts saves a third of the tensor time).
// Persistent, one CTA per SM over the column tiles, warp-specialised, no CTA barrier in the
// loop: warp 0 = TMA producer into a ring of kTmStages stages of kTmF = 64 features (A raw
// 32 KB + x hi/lo 16 KB); warps 2-5 = A-lo converters; warp 1 = MMA issuer (16 MMAs per stage,
// commit -> the stage's "empty" barrier); warps 6-9 = epilogue from one of two TMEM
// accumulator sets (the next tile's MMAs run while a tile's epilogue drains): bias, ReLU, h|dh
// lines through a per-warp shared-memory transpose (4 full 128-B lines per store instruction)
// and h_out.  Each column's result depends only on its own Wd column and xT, so column shards
// are bit-identical to the unsharded layer.  Measured steps (profiles/r02_dense_fwd_tma.txt):
// 32-feature stages with A_lo in shared memory 22.9 us, A_lo in TMEM 22.0, 64-feature stages
// 19.3 (per-stage barrier/commit overhead halved); the MMA issuer paces the pipeline.
#ifndef FF_TM_STAGES
#define FF_TM_STAGES 4
#endif
constexpr int kTmStages = FF_TM_STAGES;
#ifndef FF_TM_F
#define FF_TM_F 64
#endif
constexpr int kTmF = FF_TM_F;                                    // features per stage (32 or 64)
static_assert(kTmF == 32 || kTmF == 64, "stage features");
constexpr int kTmThreads = 320;                                  // 10 warps
constexpr uint32_t kTmG = kTmF * 128;                            // one 32-column group of the A tile (kTmF rows of 128 B)
constexpr uint32_t kTmA = 4 * kTmG, kTmX = kTmF * 32 * 4;        // A tile (kTmF f x 128 c), x tile (kTmF f x 32 b)
constexpr uint32_t kTmStage = kTmA + 2 * kTmX;                   // A raw | x hi | x lo (all TMA bytes)
constexpr uint32_t kTmEpi = 4 * 32 * 33 * 4;                     // epilogue transpose buffers
constexpr uint32_t kTmTileCols = 96;                             // TMEM columns per tile: [hi.hi | hi.lo] + lo.hi
constexpr uint32_t kTmLoCol = 2 * kTmTileCols;                   // TMEM: A-lo tiles (32 columns per stage) after the accumulators
constexpr uint32_t kTmAlloc = 512;
static_assert(kTmLoCol + kTmF * kTmStages <= kTmAlloc, "TMEM columns");
constexpr int kTmSmem = 1024 + kTmStages * kTmStage + kTmEpi + 256;

// shared-memory matrix descriptor (sm_100): start, LBO, SBO (16-B units), version 1, layout
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
// kind::tf32, D f32, A and B tf32 MN-major (bits 15, 16), M = 128, N = n
__host__ __device__ constexpr uint32_t tm_idesc(uint32_t n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}
// the same with A read from TMEM (A must be K-major there: lane = row, one column per K element)
__host__ __device__ constexpr uint32_t tm_idesc_ts(uint32_t n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}
template <uint32_t N>
__device__ __forceinline__ void tc_mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t accumulate) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
               :: "r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(tm_idesc_ts(N)), "r"(accumulate));
}
template <uint32_t N>
__device__ __forceinline__ void tc_mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
               :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(tm_idesc(N)), "r"(accumulate));
}
__device__ __forceinline__ void tc_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(mbar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t mbar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
               : "=r"(ok) : "r"(mbar), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) { while (!mbar_try_wait(mbar, parity)) {} }
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(mbar) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t mbar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               :: "r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(mbar) : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint32_t mbar) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
               :: "r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(mbar) : "memory");
}

#ifdef FF_TM_TRACE
__device__ long long g_tm_trace[5][96];   // block 0: TMA issue, landed, MMAs issued, -, slot free
#define TM_TR(r, i) do { if (blockIdx.x == 0 && (i) < 96) g_tm_trace[r][i] = clock64(); } while (0)
#else
#define TM_TR(r, i) do { } while (0)
#endif

// mW: Wd as a 3-D tensor {128 columns, d features, tiles} (box 32 x 32 x 1); mX / mXl: xT and
// its lo part {32 samples, d} (box 32 x 32).  Out-of-range features (d % 32 != 0) read as 0.
__global__ void __launch_bounds__(kTmThreads, 1) k_dense_fwd_tma(const __grid_constant__ CUtensorMap mW,
                                                                 const __grid_constant__ CUtensorMap mX,
                                                                 const __grid_constant__ CUtensorMap mXl,
                                                                 const float* __restrict__ bd, int d, int m, int B,
                                                                 float* __restrict__ hd, int cstride, int zero_dh,
                                                                 float* __restrict__ h_out) {
  extern __shared__ __align__(16) unsigned char tsm[];
  const uint32_t sbase = ((uint32_t)__cvta_generic_to_shared(tsm) + 1023u) & ~1023u;
  const uint32_t epi0 = sbase + kTmStages * kTmStage;
  const uint32_t bar0 = epi0 + kTmEpi;                            // full[S] | conv[S] | empty[S] | tfull[2] | tempty[2] | tmem
  auto full = [&](uint32_t s) { return bar0 + 8u * s; };
  auto conv = [&](uint32_t s) { return bar0 + 8u * (kTmStages + s); };
  auto empty = [&](uint32_t s) { return bar0 + 8u * (2 * kTmStages + s); };
  const uint32_t tfull0 = bar0 + 8u * (3 * kTmStages), tempty0 = tfull0 + 16, tptr_s = tempty0 + 16;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int ntiles = (m + 127) / 128, nst = (d + kTmF - 1) / kTmF;
  if (w == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(tptr_s), "n"(kTmAlloc) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    for (uint32_t s = 0; s < (uint32_t)kTmStages; ++s) { mbar_init(full(s), 1); mbar_init(conv(s), 4); mbar_init(empty(s), 1); }
    mbar_init(tfull0, 1); mbar_init(tfull0 + 8, 1); mbar_init(tempty0, 4); mbar_init(tempty0 + 8, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&mW) : "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&mX) : "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&mXl) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t tmem_d;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(tmem_d) : "r"(tptr_s) : "memory");

  if (w == 0) {                                                   // ===== TMA producer
    if (lane == 0) {
      // launched as k_dropout_T's programmatic dependent: the Wd loads of the first ring fill
      // are issued before griddepcontrol.wait (they do not depend on the dropout), the xT loads
      // after it
      uint32_t i = 0;
      bool x_ok = false;
      const uint32_t nfill = (uint32_t)min(kTmStages, nst * ((ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1));
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x)
        for (int st = 0; st < nst; ++st, ++i) {
          const uint32_t s = i % kTmStages;
          if (i >= (uint32_t)kTmStages) { mbar_wait(empty(s), ((i / kTmStages) - 1) & 1u); TM_TR(4, i - kTmStages); }
          TM_TR(0, i);
          const uint32_t stg = sbase + s * kTmStage;
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(full(s)), "r"(kTmStage) : "memory");
#pragma unroll
          for (int g = 0; g < 4; ++g) tma_load_3d(stg + (uint32_t)g * kTmG, &mW, 32 * g, kTmF * st, t, full(s));
          if (!x_ok && i + 1 < nfill) continue;                   // x of the first nfill stages after the wait
          if (!x_ok) {
            asm volatile("griddepcontrol.wait;" ::: "memory");
            x_ok = true;
            for (uint32_t k = 0; k < i; ++k) {                     // the earlier stages of the fill (x depends on the stage only)
              const uint32_t sk = k % kTmStages, stk = k % (uint32_t)nst;
              tma_load_2d(sbase + sk * kTmStage + kTmA, &mX, 0, kTmF * (int)stk, full(sk));
              tma_load_2d(sbase + sk * kTmStage + kTmA + kTmX, &mXl, 0, kTmF * (int)stk, full(sk));
            }
          }
          tma_load_2d(stg + kTmA, &mX, 0, kTmF * st, full(s));
          tma_load_2d(stg + kTmA + kTmX, &mXl, 0, kTmF * st, full(s));
        }
    }
  } else if (w == 1) {                                            // ===== MMA issuer
    if (lane == 0) {
      uint32_t i = 0;
      int tl = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
        const int acc = tl & 1;
        if (tl >= 2) mbar_wait(tempty0 + 8u * acc, (uint32_t)(((tl >> 1) - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dhh = tmem_d + kTmTileCols * (uint32_t)acc, dlh = dhh + 64;
        for (int st = 0; st < nst; ++st, ++i) {
          const uint32_t s = i % kTmStages, par = (i / kTmStages) & 1u;
          const uint32_t Ah = sbase + s * kTmStage, Xh = Ah + kTmA, Al = tmem_d + kTmLoCol + (uint32_t)kTmF * s;
          mbar_wait(full(s), par);
          mbar_wait(conv(s), par);
          TM_TR(2, i);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
          for (int kb = 0; kb < kTmF / 8; ++kb) {                 // 8 features = two 4-row groups = 1 KB
            const uint64_t xh = umma_desc(Xh + kb * 1024u, kTmX, 512, 1);
            const uint32_t accu = (st > 0 || kb > 0) ? 1u : 0u;
            tc_mma_tf32<64>(dhh, umma_desc(Ah + kb * 1024u, kTmG, 512, 1), xh, accu);   // [hi.hi | hi.lo]
            tc_mma_tf32_ts<32>(dlh, Al + 8u * kb, xh, accu);                              // lo.hi (A-lo in TMEM)
          }
          tc_commit(empty(s));
        }
        tc_commit(tfull0 + 8u * acc);
      }
    }
  } else if (w < 6) {                                             // ===== A-lo converters (128 threads)
    // thread = A row (tile column 32 q + lane, TMEM lane quarter q = w % 4): reads its column's
    // 32 features from the swizzled raw tile (byte f*128 + ((4 lane) ^ ((f & 3) << 5)) of
    // group q, tools/microbench/swzprobe.cu; conflict-free) and writes lo into its TMEM lane
    const int q = w & 3;
    uint32_t i = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x)
      for (int st = 0; st < nst; ++st, ++i) {
        const uint32_t s = i % kTmStages;
        mbar_wait(full(s), (i / kTmStages) & 1u);
        if (tid == 64) TM_TR(1, i);
        const uint32_t raw = sbase + s * kTmStage + (uint32_t)q * kTmG;
#pragma unroll
        for (int f0 = 0; f0 < kTmF; f0 += 32) {
          uint32_t lo[32];
#pragma unroll
          for (int f1 = 0; f1 < 32; ++f1) {
            const int f = f0 + f1;
            float v;
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(raw + (uint32_t)f * 128u + ((4u * lane) ^ ((uint32_t)(f & 3) << 5))));
            lo[f1] = __float_as_uint(v - __uint_as_float(__float_as_uint(v) & 0xFFFFE000u));
          }
          asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                       "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                       :: "r"(tmem_d + ((uint32_t)(32 * q) << 16) + kTmLoCol + (uint32_t)kTmF * s + (uint32_t)f0),
                          "r"(lo[0]), "r"(lo[1]), "r"(lo[2]), "r"(lo[3]), "r"(lo[4]), "r"(lo[5]), "r"(lo[6]), "r"(lo[7]),
                          "r"(lo[8]), "r"(lo[9]), "r"(lo[10]), "r"(lo[11]), "r"(lo[12]), "r"(lo[13]), "r"(lo[14]), "r"(lo[15]),
                          "r"(lo[16]), "r"(lo[17]), "r"(lo[18]), "r"(lo[19]), "r"(lo[20]), "r"(lo[21]), "r"(lo[22]), "r"(lo[23]),
                          "r"(lo[24]), "r"(lo[25]), "r"(lo[26]), "r"(lo[27]), "r"(lo[28]), "r"(lo[29]), "r"(lo[30]), "r"(lo[31])
                       : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(conv(s));
      }
  } else {                                                        // ===== epilogue (TMEM lane quarter w % 4)
    const int q = w & 3;
    const uint32_t ebuf = epi0 + (uint32_t)(w - 6) * (32u * 33u * 4u);
    int tl = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
      const int acc = tl & 1;
      mbar_wait(tfull0 + 8u * acc, (uint32_t)((tl >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float z[32];
#pragma unroll 1
      for (uint32_t sl = 0; sl < kTmTileCols / 32; ++sl) {         // hi.hi + hi.lo + lo.hi, in that order
        uint32_t v[32];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                     "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                       "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                       "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                     : "r"(tmem_d + ((uint32_t)(32 * q) << 16) + kTmTileCols * (uint32_t)acc + 32u * sl));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int s2 = 0; s2 < 32; ++s2) z[s2] = sl == 0 ? __uint_as_float(v[s2]) : z[s2] + __uint_as_float(v[s2]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty0 + 8u * acc);             // this accumulator set may be overwritten
      const int cbase = t * 128 + 32 * q, c = cbase + lane;       // TMEM lane = column
      const float bj = c < m ? bd[c] : 0.0f;
      float h[32];
#pragma unroll
      for (int s2 = 0; s2 < 32; ++s2) h[s2] = s2 < B ? fmaxf(z[s2] + bj, 0.0f) : 0.0f;
      if (h_out != nullptr && c < m) {
#pragma unroll
        for (int s2 = 0; s2 < 32; ++s2)
          if (s2 < B) h_out[(int64_t)s2 * m + c] = h[s2];
      }
      // transpose through shared memory: row = column (lane), 33-float pitch (conflict-free)
#pragma unroll
      for (int s2 = 0; s2 < 32; ++s2)
        asm volatile("st.shared.f32 [%0], %1;" :: "r"(ebuf + (uint32_t)(lane * 33 + s2) * 4u), "f"(h[s2]) : "memory");
      __syncwarp();
#pragma unroll
      for (int r = 0; r < 8; ++r) {                               // 4 lines per instruction, 8 lanes per line
        const int li = 4 * r + (lane >> 3), sg = lane & 7;
        float4 o;
        const uint32_t a = ebuf + (uint32_t)(li * 33 + 4 * sg) * 4u;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(o.x) : "r"(a) : "memory");
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(o.y) : "r"(a + 4) : "memory");
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(o.z) : "r"(a + 8) : "memory");
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(o.w) : "r"(a + 12) : "memory");
        const int cl = cbase + li;
        if (cl < m) {
          float* line = hd + (int64_t)cl * cstride + 4 * sg;
          *reinterpret_cast<float4*>(line) = o;
          if (zero_dh) *reinterpret_cast<float4*>(line + 32) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      __syncwarp();                                               // ebuf is rewritten by the next tile
    }
  }
#ifdef FF_TM_TRACE
  __syncthreads();
  if (blockIdx.x == 0 && tid == 0) {
    const long long t0 = g_tm_trace[0][0];
    const int n = min(96, nst * ((ntiles - 1) / (int)gridDim.x + 1));
    for (int i = 0; i < n; ++i)
      printf("TMTRACE %d issue %lld landed %lld mma %lld free %lld\n", i, g_tm_trace[0][i] - t0,
             g_tm_trace[1][i] - t0, g_tm_trace[2][i] - t0, i + kTmStages < n ? g_tm_trace[4][i] - t0 : -1ll);
  }
#endif
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem_d), "n"(kTmAlloc) : "memory");
}

// Backward + Adam: dz[b][c] = dh[b][c] * [h[b][c] > 0] (ReLU'(0) = 0, R26);
// dWd[f][c] = sum_b xT[f][b] dz[b][c] (b ascending), dbd[c] = sum_b dz[b][c]; then Adam
// (R6) over Wd and bd with those gradients.  This kernel streams 24 B per weight
// (read + write Wd, mWd, vWd) and is HBM-bound, so it is organised around keeping loads in
// flight: CTA = 256 threads -> 128 columns x a range of features, walked in blocks of 16
// features (lane -> 4 columns, warp w -> features 2w, 2w+1 of the block); the Adam operands
// of block i+1 are loaded into registers while block i is reduced and updated.  dz [32][128]
// (from the h|dh lines of hd) is staged in shared memory once per CTA (B <= 32; per block
// and 32-sample chunk otherwise), xT per block.  CTAs with blockIdx.y == 0 also do the
// bias (warp 0).  Gradients are stored to dWd/dbd when those are non-null.
constexpr int kDenseBwdThreads = 256, kDenseBwdBlk = 16;
__global__ void __launch_bounds__(kDenseBwdThreads, 2) k_dense_bwd_adam(
    float* __restrict__ Wd, float* __restrict__ mWd, float* __restrict__ vWd, float* __restrict__ bd,
    float* __restrict__ mbd, float* __restrict__ vbd, const float* __restrict__ xT, int d, int m, int ldw, int ldx,
    int nb, const float* __restrict__ hd, int cstride, AdamArgs adam, float* __restrict__ dWd,
    float* __restrict__ dbd, int rows_per_cta, const float* __restrict__ rbc) {
  adam.rbc1 = rbc[0]; adam.rbc2 = rbc[1];                         // this step's bias corrections (device t)
  __shared__ __align__(16) float dzs[32][128];
  __shared__ __align__(16) float xs[kDenseBwdBlk][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int ct = blockIdx.x * 128, c0 = ct + 4 * lane;
  const int f_lo = blockIdx.y * rows_per_cta, f_hi = min(d, f_lo + rows_per_cta);
  const int nblk = f_hi > f_lo ? (f_hi - f_lo + kDenseBwdBlk - 1) / kDenseBwdBlk : 0;
  const bool cok = c0 < ldw;
  const bool bias_cta = blockIdx.y == 0;
  auto stage_dz = [&](int q2) {
    if (threadIdx.x < 128) {   // thread t <-> column ct + t (32 h + 32 dh floats of its 256-B line)
      const int c = ct + threadIdx.x;
      const float* line = hd + (int64_t)c * cstride + q2 * 64;
#pragma unroll
      for (int s4 = 0; s4 < 32; s4 += 4) {
        float4 hv = make_float4(0.f, 0.f, 0.f, 0.f), gv = hv;
        if (c < m) { hv = *reinterpret_cast<const float4*>(line + s4); gv = *reinterpret_cast<const float4*>(line + 32 + s4); }
        dzs[s4 + 0][threadIdx.x] = hv.x > 0.0f ? gv.x : 0.0f;
        dzs[s4 + 1][threadIdx.x] = hv.y > 0.0f ? gv.y : 0.0f;
        dzs[s4 + 2][threadIdx.x] = hv.z > 0.0f ? gv.z : 0.0f;
        dzs[s4 + 3][threadIdx.x] = hv.w > 0.0f ? gv.w : 0.0f;
      }
    }
  };
  auto stage_x = [&](int fblk, int q2) {   // 16 rows x 8 float4, threads 128..255
    if (threadIdx.x >= 128) {
      const int e = threadIdx.x - 128, r = e >> 3, s4 = (e & 7) * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (fblk + r < f_hi) v = *reinterpret_cast<const float4*>(xT + (int64_t)(fblk + r) * ldx + q2 * 32 + s4);
      *reinterpret_cast<float4*>(&xs[r][s4]) = v;
    }
  };
  float4 P[2], Mo[2], Ve[2], Pn[2], Mn[2], Vn[2];
  auto load_ops = [&](int fblk, float4 (&p)[2], float4 (&mo)[2], float4 (&ve)[2]) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int f = fblk + 2 * w + r;
      p[r] = mo[r] = ve[r] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (cok && f < f_hi) {
        const int64_t o = ((int64_t)blockIdx.x * d + f) * 128 + 4 * lane;   // tiled layout
        p[r] = ld_na4(Wd + o); mo[r] = ld_na4(mWd + o); ve[r] = ld_na4(vWd + o);
      }
    }
  };
  if (nblk > 0) load_ops(f_lo, P, Mo, Ve);
  if (nb == 1) stage_dz(0);
  float db[4] = {0.f, 0.f, 0.f, 0.f};
  for (int bi = 0; bi < nblk; ++bi) {
    const int fblk = f_lo + bi * kDenseBwdBlk;
    if (bi + 1 < nblk) load_ops(fblk + kDenseBwdBlk, Pn, Mn, Vn);
    const bool do_bias = bias_cta && bi == 0 && w == 0;
    float2 acc[2][2];
#pragma unroll
    for (int r = 0; r < 2; ++r) { acc[r][0] = make_float2(0.f, 0.f); acc[r][1] = make_float2(0.f, 0.f); }
    for (int q2 = 0; q2 < nb; ++q2) {
      __syncthreads();                                   // previous block's readers are done
      if (nb > 1) stage_dz(q2);
      stage_x(fblk, q2);
      __syncthreads();
      if (!cok) continue;
#pragma unroll 4
      for (int b4 = 0; b4 < 32; b4 += 4) {
        float4 dz4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) dz4[u] = *reinterpret_cast<const float4*>(&dzs[b4 + u][4 * lane]);
        if (do_bias) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {   // b ascending
            db[0] = __fadd_rn(db[0], dz4[u].x); db[1] = __fadd_rn(db[1], dz4[u].y);
            db[2] = __fadd_rn(db[2], dz4[u].z); db[3] = __fadd_rn(db[3], dz4[u].w);
          }
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const float4 x4 = *reinterpret_cast<const float4*>(&xs[2 * w + r][b4]);
          const float xv[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {   // b = b4 + u ascending
            acc[r][0] = ffma2(bc2(xv[u]), make_float2(dz4[u].x, dz4[u].y), acc[r][0]);
            acc[r][1] = ffma2(bc2(xv[u]), make_float2(dz4[u].z, dz4[u].w), acc[r][1]);
          }
        }
      }
    }
    if (cok) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int f = fblk + 2 * w + r;
        if (f >= f_hi) continue;
        const int64_t o = ((int64_t)blockIdx.x * d + f) * 128 + 4 * lane;   // tiled layout
        const float4 g = make_float4(acc[r][0].x, acc[r][0].y, acc[r][1].x, acc[r][1].y);
        if (dWd != nullptr) *reinterpret_cast<float4*>(dWd + o) = g;
        adam_update(P[r].x, Mo[r].x, Ve[r].x, g.x, adam);
        adam_update(P[r].y, Mo[r].y, Ve[r].y, g.y, adam);
        adam_update(P[r].z, Mo[r].z, Ve[r].z, g.z, adam);
        adam_update(P[r].w, Mo[r].w, Ve[r].w, g.w, adam);
        st_na4(Wd + o, P[r]);
        st_na4(mWd + o, Mo[r]);
        st_na4(vWd + o, Ve[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) { P[r] = Pn[r]; Mo[r] = Mn[r]; Ve[r] = Vn[r]; }
  }
  if (bias_cta && w == 0 && cok && nblk > 0) {
    float4 p = *reinterpret_cast<const float4*>(bd + c0);
    float4 mo = *reinterpret_cast<const float4*>(mbd + c0);
    float4 ve = *reinterpret_cast<const float4*>(vbd + c0);
    if (dbd != nullptr) *reinterpret_cast<float4*>(dbd + c0) = make_float4(db[0], db[1], db[2], db[3]);
    adam_update(p.x, mo.x, ve.x, db[0], adam);
    adam_update(p.y, mo.y, ve.y, db[1], adam);
    adam_update(p.z, mo.z, ve.z, db[2], adam);
    adam_update(p.w, mo.w, ve.w, db[3], adam);
    *reinterpret_cast<float4*>(bd + c0) = p;
    *reinterpret_cast<float4*>(mbd + c0) = mo;
    *reinterpret_cast<float4*>(vbd + c0) = ve;
  }
}

// The same backward + Adam for B <= 32 (one 32-sample chunk).  Round 2: persistent — the
// (column tile, 16-feature block) work items, tile-major, are split into equal contiguous
// ranges over the resident CTAs (the round-1 grid of 256 x 3 CTAs ran 2.6 waves) — and fed by
// the TMA engine: a producer warp streams each block's Wd / mWd / vWd rows (3 x 8 KB,
// contiguous in the tiled layout) and its xT rows (2 KB) into a ring of kDenseBwdNS
// shared-memory stages with cp.async.bulk (one mbarrier per stage, complete_tx), and four
// compute warps — each 4 features x 128 columns, lane -> 4 columns, so every 16-B dz load
// serves 4 features — release a stage by arriving on its "empty" barrier.  A CTA restages the
// dz tile [32][128] when its range enters a new tile and updates the tile's bias right after
// the tile's first block.  Adam runs on packed fp32x2 ops (adam_update2, bit-identical);
// same arithmetic and order as k_dense_bwd_adam: bit-identical results.
#ifndef FF_BWD_NS
#define FF_BWD_NS 3
#endif
#ifndef FF_BWD_MINB
#define FF_BWD_MINB 2
#endif
constexpr int kDenseBwdNS = FF_BWD_NS;                               // stages
constexpr int kDenseBwdStage = (3 * kDenseBwdBlk * 128 + kDenseBwdBlk * 32) * 4;   // 26 KB
constexpr int kDenseBwd1Smem = 32 * 128 * 4 + kDenseBwdNS * kDenseBwdStage + 16 * kDenseBwdNS;
constexpr int kDenseBwd32Threads = 160, kDenseBwdFpw = 4;           // 4 compute warps + 1 TMA producer warp
static_assert(kDenseBwdFpw * 4 == kDenseBwdBlk, "features per warp");
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
__global__ void __launch_bounds__(kDenseBwd32Threads, FF_BWD_MINB) k_dense_bwd_adam_b32(
    float* __restrict__ Wd, float* __restrict__ mWd, float* __restrict__ vWd, float* __restrict__ bd,
    float* __restrict__ mbd, float* __restrict__ vbd, const float* __restrict__ xT, int d, int m, int ldx,
    const float* __restrict__ hd, int cstride, AdamArgs adam, float* __restrict__ dWd, float* __restrict__ dbd,
    int ntiles, const float* __restrict__ rbc) {
  adam.rbc1 = rbc[0]; adam.rbc2 = rbc[1];                         // this step's bias corrections (device t)
  extern __shared__ __align__(16) float bsm[];
  float (*dzs)[128] = reinterpret_cast<float (*)[128]>(bsm);        // [32][128]
  float* const stages = bsm + 32 * 128;
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(stages + kDenseBwdNS * (kDenseBwdStage / 4));
  auto full = [&](int s) { return bar0 + 8u * (uint32_t)s; };
  auto empty = [&](int s) { return bar0 + 8u * (uint32_t)(kDenseBwdNS + s); };
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nfb = (d + kDenseBwdBlk - 1) / kDenseBwdBlk;             // feature blocks per tile
  const int64_t nitems = (int64_t)ntiles * nfb;
  const int64_t it_lo = nitems * blockIdx.x / gridDim.x, it_hi = nitems * (blockIdx.x + 1) / gridDim.x;
  const int nblk = (int)(it_hi - it_lo);
  // stage layout (floats): P [16][128] | M [16][128] | V [16][128] | X [16][32]
  auto stage_ptr = [&](int s) { return stages + (size_t)s * (kDenseBwdStage / 4); };
  if (threadIdx.x == 0) {
    for (int s = 0; s < kDenseBwdNS; ++s) { mbar_init(full(s), 1); mbar_init(empty(s), 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (w == 4) {                                                      // ===== TMA producer warp
    if (lane == 0) {
      for (int bi = 0; bi < nblk; ++bi) {
        const int s = bi % kDenseBwdNS;
        if (bi >= kDenseBwdNS) mbar_wait(empty(s), (uint32_t)(((bi / kDenseBwdNS) - 1) & 1));
        const int64_t item = it_lo + bi;
        const int tile = (int)(item / nfb), fblk = (int)(item % nfb) * kDenseBwdBlk;
        const uint32_t rows = (uint32_t)min(kDenseBwdBlk, d - fblk);
        const uint32_t st = (uint32_t)__cvta_generic_to_shared(stage_ptr(s));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(full(s)), "r"(rows * (3u * 512u + 128u)) : "memory");
        const int64_t o = ((int64_t)tile * d + fblk) * 128;
        bulk_g2s(st, Wd + o, rows * 512u, full(s));
        bulk_g2s(st + 16u * 512u, mWd + o, rows * 512u, full(s));
        bulk_g2s(st + 32u * 512u, vWd + o, rows * 512u, full(s));
        bulk_g2s(st + 48u * 512u, xT + (int64_t)fblk * ldx, rows * 128u, full(s));
      }
    }
    return;
  }
  int cur_tile = -1;
  for (int bi = 0; bi < nblk; ++bi) {
    const int64_t item = it_lo + bi;
    const int tile = (int)(item / nfb), fblk = (int)(item % nfb) * kDenseBwdBlk;
    const int ct = tile * 128, c0 = ct + 4 * lane;
    if (tile != cur_tile) {                                          // dz tile: thread t <-> column ct + t
      asm volatile("bar.sync 1, 128;" ::: "memory");                 // the previous tile's readers are done
      {
        const int c = ct + threadIdx.x;
        const float* line = hd + (int64_t)c * cstride;
#pragma unroll
        for (int s4 = 0; s4 < 32; s4 += 4) {
          float4 hv = make_float4(0.f, 0.f, 0.f, 0.f), gv = hv;
          if (c < m) { hv = *reinterpret_cast<const float4*>(line + s4); gv = *reinterpret_cast<const float4*>(line + 32 + s4); }
          dzs[s4 + 0][threadIdx.x] = hv.x > 0.0f ? gv.x : 0.0f;
          dzs[s4 + 1][threadIdx.x] = hv.y > 0.0f ? gv.y : 0.0f;
          dzs[s4 + 2][threadIdx.x] = hv.z > 0.0f ? gv.z : 0.0f;
          dzs[s4 + 3][threadIdx.x] = hv.w > 0.0f ? gv.w : 0.0f;
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      cur_tile = tile;
    }
    const int s = bi % kDenseBwdNS;
    mbar_wait(full(s), (uint32_t)((bi / kDenseBwdNS) & 1));
    const float* st = stage_ptr(s);
    const bool do_bias = fblk == 0 && w == 0;
    float db[4] = {0.f, 0.f, 0.f, 0.f};
    float2 acc[kDenseBwdFpw][2];
#pragma unroll
    for (int r = 0; r < kDenseBwdFpw; ++r) { acc[r][0] = make_float2(0.f, 0.f); acc[r][1] = make_float2(0.f, 0.f); }
#pragma unroll 2
    for (int b4 = 0; b4 < 32; b4 += 4) {
      float4 dz4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) dz4[u] = *reinterpret_cast<const float4*>(&dzs[b4 + u][4 * lane]);
      if (do_bias) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {   // b ascending
          db[0] = __fadd_rn(db[0], dz4[u].x); db[1] = __fadd_rn(db[1], dz4[u].y);
          db[2] = __fadd_rn(db[2], dz4[u].z); db[3] = __fadd_rn(db[3], dz4[u].w);
        }
      }
#pragma unroll
      for (int r = 0; r < kDenseBwdFpw; ++r) {
        const float4 x4 = *reinterpret_cast<const float4*>(st + 48 * 128 + (kDenseBwdFpw * w + r) * 32 + b4);
        const float xv[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {   // b = b4 + u ascending
          acc[r][0] = ffma2(bc2(xv[u]), make_float2(dz4[u].x, dz4[u].y), acc[r][0]);
          acc[r][1] = ffma2(bc2(xv[u]), make_float2(dz4[u].z, dz4[u].w), acc[r][1]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kDenseBwdFpw; ++r) {
      const int rl = kDenseBwdFpw * w + r, f = fblk + rl;
      if (f >= d) continue;
      const int64_t o = ((int64_t)tile * d + f) * 128 + 4 * lane;
      const float4 P = *reinterpret_cast<const float4*>(st + rl * 128 + 4 * lane);
      const float4 Mo = *reinterpret_cast<const float4*>(st + 16 * 128 + rl * 128 + 4 * lane);
      const float4 Ve = *reinterpret_cast<const float4*>(st + 32 * 128 + rl * 128 + 4 * lane);
      if (dWd != nullptr) *reinterpret_cast<float4*>(dWd + o) = make_float4(acc[r][0].x, acc[r][0].y, acc[r][1].x, acc[r][1].y);
      float2 p0 = lo2(P), p1 = hi2(P), m0 = lo2(Mo), m1 = hi2(Mo), v0 = lo2(Ve), v1 = hi2(Ve);
      adam_update2(p0, m0, v0, acc[r][0], adam);
      adam_update2(p1, m1, v1, acc[r][1], adam);
      st_na4(Wd + o, make_float4(p0.x, p0.y, p1.x, p1.y));
      st_na4(mWd + o, make_float4(m0.x, m0.y, m1.x, m1.y));
      st_na4(vWd + o, make_float4(v0.x, v0.y, v1.x, v1.y));
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty(s));                            // this warp is done with stage s
    if (do_bias) {                                                   // the tile's bias, once (its first block)
      float4 p = *reinterpret_cast<const float4*>(bd + c0);
      float4 mo = *reinterpret_cast<const float4*>(mbd + c0);
      float4 ve = *reinterpret_cast<const float4*>(vbd + c0);
      if (dbd != nullptr) *reinterpret_cast<float4*>(dbd + c0) = make_float4(db[0], db[1], db[2], db[3]);
      adam_update(p.x, mo.x, ve.x, db[0], adam);
      adam_update(p.y, mo.y, ve.y, db[1], adam);
      adam_update(p.z, mo.z, ve.z, db[2], adam);
      adam_update(p.w, mo.w, ve.w, db[3], adam);
      *reinterpret_cast<float4*>(bd + c0) = p;
      *reinterpret_cast<float4*>(mbd + c0) = mo;
      *reinterpret_cast<float4*>(vbd + c0) = ve;
    }
  }
}

// dh [B][m] (user layout) -> the dh half of hd (standalone dense backward).  Grid
// ceil(m/32) x nb, 32x8 threads; samples >= B get 0.
__global__ void k_dh_in(const float* __restrict__ dh, int B, int m, int nb, float* __restrict__ hd) {
  __shared__ float t[32][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int c0 = blockIdx.x * 32, q2 = blockIdx.y;
  for (int r = ty; r < 32; r += 8) {
    const int b = q2 * 32 + r, c = c0 + tx;
    t[r][tx] = (b < B && c < m) ? dh[(int64_t)b * m + c] : 0.0f;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int c = c0 + r;
    if (c < m) hd[(int64_t)c * 64 * nb + q2 * 64 + 32 + tx] = t[tx][r];
  }
}

// Dense init (reading R27): Wd[f][c] = a * (2 * ((u >> 8) * 2^-24) - 1) in fp32, u = word c
// of the stream (ctr = (c/4, f, 0, 4), key = seed); pad columns and bd, moments = 0.
// Thread per (tile, feature, 4 columns), tiled layout.
__global__ void k_dense_init(float* __restrict__ Wd, int d, int m, int ldw, int col_begin, uint32_t key0, uint32_t key1,
                             float a) {
  const int64_t n4 = (int64_t)d * (ldw / 4);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n4; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / ((int64_t)d * 32);
    const int f = (int)((e / 32) % d), cq = (int)(e % 32);
    const int c = (int)t * 128 + 4 * cq;
    // global column g = col_begin + c + u draws word g % 4 of the block (g / 4, f, 0, 4) (R27):
    // a column shard reproduces its columns of the whole layer
    const uint32_t g0 = (uint32_t)(col_begin + c);
    const U4 v0 = philox(g0 / 4, (uint32_t)f, 0u, 4u, key0, key1);
    const U4 v1 = (g0 & 3u) ? philox(g0 / 4 + 1, (uint32_t)f, 0u, 4u, key0, key1) : v0;
    float out[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t g = g0 + (uint32_t)u;
      const uint32_t word = (g / 4 == g0 / 4) ? word_of(v0, (int)(g & 3u)) : word_of(v1, (int)(g & 3u));
      const float unit = __fmul_rn((float)(word >> 8), 1.0f / 16777216.0f);
      const float centered = __fsub_rn(__fmul_rn(2.0f, unit), 1.0f);
      out[u] = c + u < m ? __fmul_rn(a, centered) : 0.0f;
    }
    *reinterpret_cast<float4*>(Wd + e * 4) = make_float4(out[0], out[1], out[2], out[3]);
  }
}

// user [d][m] <-> tiled [ldw/128][d][128] (set/get_params, get_grads); pad columns untouched
__global__ void k_dense_retile(const float* __restrict__ src, float* __restrict__ dst, int d, int m, int to_tiled) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)d * m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int f = (int)(e / m), c = (int)(e % m);
    const int64_t t = ((int64_t)(c >> 7) * d + f) * 128 + (c & 127);
    if (to_tiled) dst[t] = src[e]; else dst[e] = src[t];
  }
}

}  // namespace ff
