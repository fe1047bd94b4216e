// ff_kernels.cuh — sm_100a kernels of the fixed fan-in (uniform sparsity) layer.
//
// Data layout in HBM: label-major W/idx/mW/vW [L][k] (one 128-B line
// per label row at k = 32), bias/mb/vb [L], the hidden batch transposed to hT[m][ldh]
// (ldh = 32*nb, nb = ceil(B/32); one 128-B line per h-column at B <= 32) and the dh
// accumulator, interleaved with it: hd[c][q2][0..32) = h[q2*32 + r][c] and
// hd[c][q2][32..64) = the dh accumulator of the same samples, so the dh line of a
// connection sits 128 B after its h line (one address serves gather and reduction).
// hd is 8 MiB at m = 32768, B = 32 and L2-resident.
//
// Thread mapping of the row kernels (one warp = one label row at a time):
//   lane = slot for the per-connection state (W, idx, moments: coalesced 128-B rows);
//   for the gathers lane = (gq = lane>>3, bq = lane&7): connection 4q+gq, samples 4bq..4bq+3,
//   so one warp instruction moves four 128-B hT lines (ld.v4) / dhT lines (red.v4).
#pragma once
#include "ff_device.cuh"
#include <cfloat>
#include <climits>

namespace ff {

enum : int { kErrLabelRange = 1, kErrNonFinite = 2, kErrIdxRange = 4, kErrIdxDup = 8 };
enum RowMode : int { kModeTrain = 0, kModeForward = 1, kModeBackward = 2 };

#ifndef FF_ROW_THREADS
#define FF_ROW_THREADS 256
#endif
#ifndef FF_ROW_MINB
#define FF_ROW_MINB 2
#endif
constexpr int kRowThreads = FF_ROW_THREADS;   // threads per CTA of the row kernels
constexpr int kRowMinBlocks = FF_ROW_MINB;    // __launch_bounds__ residency target
constexpr int kTopkMax = 8;

struct RowArgs {
  float* W; const int* idx; float* bias; float* mW; float* vW; float* mb; float* vb;
  float* dW; float* db;
  uint32_t* posmask;          // [nb][L] bit (b & 31) of word [b>>5][j]: is row_begin+j a positive of b
  float* hd;                  // [m][nb][64]: h line | dh line per column and 32-sample chunk
  float* gT;                  // CSC mode: one record per label row of the tile, rs floats each:
                              //   [q2*32 + r] = g[q2*32 + r][j] (gradient line of chunk q2),
                              //   [32*nb + i] = pre-update W[j][i] (0 if the row's gradient is all zero)
  int rs;                     // CSC mode: record stride in floats = 32*nb + 32*ceil(k/32)
  int64_t j_begin, j_end;     // label rows processed by this launch (a tile; multiple of 32)
  int br;                     // rows per warp block (32, 16, 8 or 4): smaller for small L
  int64_t L; int k; int B; int nb; int cstride;   // cstride = 64*nb floats per column
  float grad_scale;
  float* y_out;               // forward: y[B][L]
  const float* y_in;          // backward: y[B][L]
  float* loss;                // device scalar (zeroed by prep) or nullptr
  const float* rbc;           // train: device [rbc1, rbc2] of this step (written by k_prep), or nullptr
  int* err;
  AdamArgs adam;
  uint32_t check_finite;
  int sqh;                    // loss: 0 = BCE, 1 = squared hinge (exact zeros skipped)
  uint32_t split;             // CSC modes: columns c < split get their dh by red (hybrid), the rest by the pull
};

// Loss gradient of one score and its loss term (BCE or squared hinge).
__device__ __forceinline__ float loss_grad(float y, bool pos, float s, bool sqh, float* lterm) {
  if (sqh) return sqh_grad(y, pos, s, lterm);
  float e;
  const float g = bce_grad(y, pos, s, &e);
  *lterm = bce_loss_term(y, pos, e);
  return g;
}

__device__ __forceinline__ float comp(const float4& v, int e) {
  return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
}

// Block-wide sum of one float per thread, lane 0 of warp 0 adds it to *dst.
__device__ __forceinline__ void block_atomic_add(float v, float* dst) {
  __shared__ float part[32];
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) part[wid] = v;
  __syncthreads();
  if (wid == 0) {
    v = (lane < (int)(blockDim.x >> 5)) ? part[lane] : 0.0f;
    v = warp_sum(v);
    if (lane == 0 && v != 0.0f) atomicAdd(dst, v);
  }
}

// ---- shared pieces of the row kernels (forward / fused step / predict use the SAME
// arithmetic, so their scores are bit-identical: the top-K parity relies on it)

// Broadcast each connection's weight and hd column to the lanes that gather it: lane
// (gq, bq) handles connections s = 4q + gq, q < NG (the 8 lanes of equal gq read one
// 128-B line together, so register q must name the same connection on all of them).
// Columns stay raw 32-bit indices: the line address base + c * cfloats is then one
// IMAD.WIDE.U32 at the load.
template <int NG>
__device__ __forceinline__ void row_spread(float w, int c, int gq, float (&ws)[NG], uint32_t (&cs)[NG]) {
#pragma unroll
  for (int q = 0; q < NG; ++q) {
    ws[q] = __shfl_sync(kFull, w, 4 * q + gq);
    cs[q] = (uint32_t)__shfl_sync(kFull, c, 4 * q + gq);
  }
}
// k <= 64: lane owns slots lane (e = 0) and lane + 32 (e = 1); connection s = 4q + gq lives
// in register e = q / 8 of lane 4*(q%8) + gq.
template <int NG, int KPL>
__device__ __forceinline__ void row_spread_k(const float (&w)[KPL], const int (&c)[KPL], int gq, float (&ws)[NG],
                                             uint32_t (&cs)[NG]) {
#pragma unroll
  for (int q = 0; q < NG; ++q) {
    ws[q] = __shfl_sync(kFull, w[q / 8], 4 * (q % 8) + gq);
    cs[q] = (uint32_t)__shfl_sync(kFull, c[q / 8], 4 * (q % 8) + gq);
  }
}

// (as a byte offset c * (4 cfloats): one IMAD.WIDE.U32 with the base, instead of a float-index
// IMAD.WIDE followed by LEA + LEA.HI.X)
__device__ __forceinline__ const float* col_line(const float* hb, uint32_t c, uint32_t cfloats) {
  return reinterpret_cast<const float*>(reinterpret_cast<const char*>(hb) + (uint64_t)c * (4u * cfloats));
}
__device__ __forceinline__ float* col_line(float* hb, uint32_t c, uint32_t cfloats) {
  return reinterpret_cast<float*>(reinterpret_cast<char*>(hb) + (uint64_t)c * (4u * cfloats));
}

// Gather this lane's 16-B segment of each connection's 128-B h line (hb = the lane's
// segment in column 0 of the chunk).  FULL: k == 4*NG, every slot exists (no guards).
template <int NG, bool FULL>
__device__ __forceinline__ void row_gather(const float* hb, const uint32_t (&cs)[NG], uint32_t cfloats, int k, int gq,
                                           uint64_t pol, float4 (&hv)[NG]) {
#pragma unroll
  for (int q = 0; q < NG; ++q) {
    if (FULL) {
      hv[q] = ld_line4(col_line(hb, cs[q], cfloats), pol);
    } else {
      hv[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (4 * q + gq < k) hv[q] = ld_line4(col_line(hb, cs[q], cfloats), pol);
    }
  }
}

// The same gather without the L2 policy operand (hot loop of the pipelined kernel).
template <int NG>
__device__ __forceinline__ void row_gather_plain(const float* hb, const uint32_t (&cs)[NG], uint32_t cfloats,
                                                 float4 (&hv)[NG]) {
#pragma unroll
  for (int q = 0; q < NG; ++q) hv[q] = ld_line4_plain(col_line(hb, cs[q], cfloats));
}

// y for this lane's own sample lo + gq: per-lane FMAs over its connections, then a
// reduce-scatter over the four connection groups (xor 16, xor 8), + bias.
template <int NG>
__device__ __forceinline__ float row_score_own(const float (&ws)[NG], const float4 (&hv)[NG], int gq, float bj) {
  // packed FMAs in 4 independent chains (even / odd connections), then combined
  float2 y01a = make_float2(0.f, 0.f), y23a = make_float2(0.f, 0.f);
  float2 y01b = make_float2(0.f, 0.f), y23b = make_float2(0.f, 0.f);
#pragma unroll
  for (int q = 0; q < NG; q += 2) {
    y01a = ffma2(bc2(ws[q]), lo2(hv[q]), y01a);
    y23a = ffma2(bc2(ws[q]), hi2(hv[q]), y23a);
    if (q + 1 < NG) {
      y01b = ffma2(bc2(ws[q + 1]), lo2(hv[q + 1]), y01b);
      y23b = ffma2(bc2(ws[q + 1]), hi2(hv[q + 1]), y23b);
    }
  }
  const float4 yp = make_float4(y01a.x + y01b.x, y01a.y + y01b.y, y23a.x + y23b.x, y23a.y + y23b.y);
  const bool hi = gq & 2, odd = gq & 1;
  const float k0 = hi ? yp.z : yp.x, k1 = hi ? yp.w : yp.y;
  const float s0 = hi ? yp.x : yp.z, s1 = hi ? yp.y : yp.w;
  const float a0 = k0 + __shfl_xor_sync(kFull, s0, 16);
  const float a1 = k1 + __shfl_xor_sync(kFull, s1, 16);
  const float keep = odd ? a1 : a0, send = odd ? a0 : a1;
  return (keep + __shfl_xor_sync(kFull, send, 8)) + bj;
}

// Partial dW of connection q over this lane's 4 samples: (g0 h0 + g2 h2) + (g1 h1 + g3 h3)
// (two packed FMAs and one add); shared by every kernel so their dW are bit-identical.
__device__ __forceinline__ float dw_partial(const float4& g4, const float4& hv) {
  float2 t = ffma2(lo2(g4), lo2(hv), make_float2(0.f, 0.f));
  t = ffma2(hi2(g4), hi2(hv), t);
  return t.x + t.y;
}
// W[j][i] * g[b][j] for this lane's 4 samples (the Alg. 2 contributions of one connection).
__device__ __forceinline__ float4 dh_contrib(float w, const float4& g4) {
  const float2 a = fmul2(bc2(w), lo2(g4)), b = fmul2(bc2(w), hi2(g4));
  return make_float4(a.x, a.y, b.x, b.y);
}

// Reduce dwp[q] (partial dW of slot 4q+gq over this lane's 4 samples) over the 8 lanes of
// equal gq (transpose-reduce); return the total of slot `lane` (lane = slot layout).
template <int NG>
__device__ __forceinline__ float row_dw_slot(const float (&dwp)[NG], int lane) {
  const int bq = lane & 7;
  float v[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) v[q] = 0.0f;
#pragma unroll
  for (int q = 0; q < NG; ++q) v[q] = dwp[q];
  if (NG > 4) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const bool up = bq & 4;
      const float send = up ? v[q] : v[q + 4], keep = up ? v[q + 4] : v[q];
      v[q] = keep + __shfl_xor_sync(kFull, send, 4);
    }
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] += __shfl_xor_sync(kFull, v[q], 4);
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const bool up = bq & 2;
    const float send = up ? v[q] : v[q + 2], keep = up ? v[q + 2] : v[q];
    v[q] = keep + __shfl_xor_sync(kFull, send, 2);
  }
  {
    const bool up = bq & 1;
    const float send = up ? v[0] : v[1], keep = up ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(kFull, send, 1);
  }
  // lane (gq, bq) now holds slot 4*bq + gq
  return __shfl_sync(kFull, v[0], ((lane & 3) << 3) | ((lane >> 2) & (NG > 4 ? 7 : 3)));
}

// Bias gradient of one row over one 32-sample chunk: this lane's 4 samples
// (g0 + g1) + (g2 + g3), then a butterfly over the 8 lanes of equal gq (xor 1, 2, 4).
// IEEE addition is commutative, so every lane ends with the same bits; shared by every
// kernel so their db are bit-identical.
__device__ __forceinline__ float row_db_chunk(const float4& g4) {
  float p = (g4.x + g4.y) + (g4.z + g4.w);
  p += __shfl_xor_sync(kFull, p, 1);
  p += __shfl_xor_sync(kFull, p, 2);
  p += __shfl_xor_sync(kFull, p, 4);
  return p;
}

// dW of this lane's slots (lane, lane + 32 for k > 32).
template <int NG>
__device__ __forceinline__ void row_dw_slots(const float (&dwp)[NG], int lane, float (&gW)[(NG + 7) / 8]) {
  if constexpr (NG <= 8) {
    gW[0] = row_dw_slot<NG>(dwp, lane);
  } else {
    float lo[8], hi[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) { lo[q] = dwp[q]; hi[q] = dwp[q + 8]; }
    gW[0] = row_dw_slot<8>(lo, lane);
    gW[1] = row_dw_slot<8>(hi, lane);
  }
}

// The row kernel: forward (Alg. 1) for MODE forward; BCE gradient,
// Alg. 3 weight gradient, bias gradient and Alg. 2 input-gradient scatter
// for MODE backward; all of those plus Adam for MODE train — the
// fused step, in which y, g and dW live only in registers.
// Work split: a warp owns blocks of br consecutive label rows (32, or 16/8/4 when L is small) (persistent, strided over
// blocks) and walks their rows one at a time, prefetching the next row's state.  Per-label
// scalars (bias, its moments, the positive mask) are one coalesced vector per block
// (lane i <-> row i) and the bias Adam update runs once per block, vectorized.
// The Adam arguments of a training launch: the bias corrections of this step come from the
// device (k_prep advanced the device step counter t and wrote them), so a captured step
// replays with the right t.
__device__ __forceinline__ AdamArgs step_adam(const RowArgs& a) {
  AdamArgs ad = a.adam;
  if (a.rbc != nullptr) { ad.rbc1 = a.rbc[0]; ad.rbc2 = a.rbc[1]; }
  return ad;
}

// Programmatic dependent launch (the training step's kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): wait until the previous kernel of the
// stream has completed and its memory is visible, then let the next one be scheduled so its
// launch overlaps this kernel's tail.  Both are no-ops in a plain launch.
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <int MODE, bool STORE_GRADS, int NG, bool CSC, bool FULL>
__global__ void __launch_bounds__(kRowThreads, NG > 8 ? 1 : kRowMinBlocks) k_rows(RowArgs a) {
  pdl_begin();
  const AdamArgs adam = step_adam(a);
  constexpr int KPL = (NG + 7) / 8;                 // slots per lane (k <= 32 * KPL)
  const int lane = threadIdx.x & 31, gq = lane >> 3, bq = lane & 7;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t pol_s = policy_evict_first(), pol_l = policy_evict_last();
  const int k = FULL ? 4 * NG : a.k, nb = a.nb, B = a.B;
  const uint32_t cfl = (uint32_t)a.cstride;
  float* const hd_lane = a.hd + 4 * bq;            // this lane's segment, column 0, chunk 0
  const int br = a.br;
  const int64_t L = a.L, jb = a.j_begin, nblk = (a.j_end - jb + br - 1) / br;
  bool act[KPL];
#pragma unroll
  for (int e = 0; e < KPL; ++e) act[e] = lane + 32 * e < k;
  float loss_acc = 0.0f;

  float w_n[KPL], mw_n[KPL], vw_n[KPL];
  int c_n[KPL];
#pragma unroll
  for (int e = 0; e < KPL; ++e) { w_n[e] = mw_n[e] = vw_n[e] = 0.f; c_n[e] = 0; }
  auto prefetch_row = [&](int64_t jj) {
    const int64_t row = jj * k;
#pragma unroll
    for (int e = 0; e < KPL; ++e) {
      if (act[e]) {
        const int64_t r = row + lane + 32 * e;
        w_n[e] = ld_stream(a.W + r, pol_s);
        c_n[e] = ld_stream_ro(a.idx + r, pol_s);
        if (MODE == kModeTrain) { mw_n[e] = ld_stream(a.mW + r, pol_s); vw_n[e] = ld_stream(a.vW + r, pol_s); }
      }
    }
  };
  int64_t blk = global_warp();
  if (blk < nblk) prefetch_row(jb + blk * br);

  for (; blk < nblk; blk += nw) {
    const int64_t j0 = jb + blk * br;
    const int nl = (int)min((int64_t)br, a.j_end - j0);
    const bool lv = lane < nl;                  // lane i <-> row j0 + i for the block vectors
    float bias_v = 0.f, mb_v = 0.f, vb_v = 0.f, db_v = 0.f;
    uint32_t pm_v = 0u;
    if (lv) {
      if (MODE != kModeBackward) bias_v = ld_stream(a.bias + j0 + lane, pol_s);
      if (MODE == kModeTrain) { mb_v = ld_stream(a.mb + j0 + lane, pol_s); vb_v = ld_stream(a.vb + j0 + lane, pol_s); }
      if (MODE != kModeForward) pm_v = a.posmask[j0 + lane];
    }
    for (int i = 0; i < nl; ++i) {
      const int64_t j = j0 + i;
      float w[KPL], mw[KPL], vw[KPL];
      int c[KPL];
#pragma unroll
      for (int e = 0; e < KPL; ++e) { w[e] = w_n[e]; mw[e] = mw_n[e]; vw[e] = vw_n[e]; c[e] = c_n[e]; }
      if (i + 1 < nl) prefetch_row(j + 1);
      else if (blk + nw < nblk) prefetch_row(jb + (blk + nw) * br);
      const int64_t row = j * k;
      const float bj = __shfl_sync(kFull, bias_v, i);
      uint32_t pm = __shfl_sync(kFull, pm_v, i);

      float ws[NG]; uint32_t cs[NG];
      row_spread_k<NG, KPL>(w, c, gq, ws, cs);
      float dwp[NG];
#pragma unroll
      for (int q = 0; q < NG; ++q) dwp[q] = 0.0f;
      float dbr = 0.0f;                                // this row's bias gradient
      bool gany = false;                               // any nonzero gradient in this row

      for (int q2 = 0; q2 < nb; ++q2) {
        const int lo = q2 * 32 + 4 * bq;             // this lane's 4-sample segment
        const int b = lo + gq;                        // this lane's own sample
        float* hb = hd_lane + q2 * 64;                // h segment; its dh segment is +32 floats
        float4 hv[NG];
        row_gather<NG, FULL>(hb, cs, cfl, k, gq, pol_l, hv);
        float y;
        if (MODE != kModeBackward) {
          y = row_score_own<NG>(ws, hv, gq, bj);
          if (MODE == kModeForward) {
            if (b < B) a.y_out[(int64_t)b * L + j] = y;
            continue;
          }
        } else {
          y = (b < B) ? a.y_in[(int64_t)b * L + j] : 0.0f;
        }
        if (q2 > 0) {                                 // B > 32: masks of later chunks per row
          pm = a.posmask[(int64_t)q2 * L + j];
          if (lane == 0 && pm != 0u) a.posmask[(int64_t)q2 * L + j] = 0u;
        }
        const bool pos = (pm >> (4 * bq + gq)) & 1u;
        float lt;
        float g = loss_grad(y, pos, a.grad_scale, a.sqh != 0, &lt);
        if (b >= B) g = 0.0f;
        if (a.loss != nullptr && b < B) loss_acc += lt;
        gany |= __any_sync(kFull, g != 0.0f);
        if (a.check_finite && __any_sync(kFull, b < B && !isfinite(y)) && lane == 0) atomicOr(a.err, kErrNonFinite);
        float4 g4;
        g4.x = __shfl_sync(kFull, g, (0 << 3) | bq);
        g4.y = __shfl_sync(kFull, g, (1 << 3) | bq);
        g4.z = __shfl_sync(kFull, g, (2 << 3) | bq);
        g4.w = __shfl_sync(kFull, g, (3 << 3) | bq);
#pragma unroll
        for (int q = 0; q < NG; ++q) dwp[q] = q2 == 0 ? dw_partial(g4, hv[q]) : dwp[q] + dw_partial(g4, hv[q]);
        const float dbc = row_db_chunk(g4);
        dbr = q2 == 0 ? dbc : dbr + dbc;
        if (CSC) {
          // CSC mode: publish g[., j] (one 128-B line per chunk); dh is pulled later (k_dh_csc)
          st_hint(a.gT + (j - jb) * a.rs + q2 * 32 + 4 * bq + gq, g, pol_l);
          if (a.split != 0u) {                        // hybrid: columns < split by red
            const bool gnz = (g4.x != 0.0f) | (g4.y != 0.0f) | (g4.z != 0.0f) | (g4.w != 0.0f);
#pragma unroll
            for (int q = 0; q < NG; ++q) {
              if ((FULL || 4 * q + gq < k) && gnz && cs[q] < a.split)
                red_add4(col_line(hb, cs[q], cfl) + 32, dh_contrib(ws[q], g4), pol_l);
            }
          }
        } else {
          // Alg. 2 with the pre-update weights: dh[b][idx[j][i]] += W[j][i] g[b][j], skipping
          // this lane's reductions when its 4 gradients are exactly zero
          const bool gnz = (g4.x != 0.0f) | (g4.y != 0.0f) | (g4.z != 0.0f) | (g4.w != 0.0f);
#pragma unroll
          for (int q = 0; q < NG; ++q) {
            if ((FULL || 4 * q + gq < k) && gnz)
              red_add4(col_line(hb, cs[q], cfl) + 32, dh_contrib(ws[q], g4), pol_l);
          }
        }
      }
      if (MODE == kModeForward) continue;

      float gW[KPL];
      row_dw_slots<NG>(dwp, lane, gW);
      if (lane == i) db_v = dbr;                      // lane i <-> row j0 + i
#pragma unroll
      for (int e = 0; e < KPL; ++e) {
        if (!act[e]) continue;
        const int64_t r = row + lane + 32 * e;
        // pre-update W into the row's record for k_dh_csc (one coalesced line); 0 when the row's
        // gradient is all zero, so the column pass may skip the gather (w*g is exactly 0 anyway)
        if (CSC) a.gT[(j - jb) * a.rs + 32 * nb + lane + 32 * e] = gany ? w[e] : 0.0f;
        if (MODE == kModeBackward || STORE_GRADS) a.dW[r] = gW[e];
        if (MODE == kModeTrain) {
          adam_update(w[e], mw[e], vw[e], gW[e], adam);
          st_stream(a.W + r, w[e], pol_s);
          st_stream(a.mW + r, mw[e], pol_s);
          st_stream(a.vW + r, vw[e], pol_s);
        }
      }
    }
    if (MODE == kModeForward) continue;
    if (lv) {
      if (pm_v != 0u) a.posmask[j0 + lane] = 0u;      // self-clearing mask (chunk 0)
      if (MODE == kModeBackward || STORE_GRADS) a.db[j0 + lane] = db_v;
      if (MODE == kModeTrain) {                        // bias Adam, one row per lane
        adam_update(bias_v, mb_v, vb_v, db_v, adam);
        st_stream(a.bias + j0 + lane, bias_v, pol_s);
        st_stream(a.mb + j0 + lane, mb_v, pol_s);
        st_stream(a.vb + j0 + lane, vb_v, pol_s);
      }
    }
  }
  if (MODE != kModeForward && a.loss != nullptr) block_atomic_add(loss_acc * a.grad_scale, a.loss);
}

// ------------------------------------------------------------------ pipelined train step
// The fused training step of k_rows<train> for the hot configuration (k = 32 connections,
// B <= 32 samples), software-pipelined for memory-level parallelism.  The h-line gathers
// are staged through a per-warp shared-memory ring (cp.async.cg, 16 B per lane per
// connection, L2 -> smem without registers): while row X is computed, the gathers of the
// next D - 1 rows are in flight and the state of row X + D is being loaded.  In-flight
// data does not occupy registers (107-111 regs), so 16-24 warps fit per SM.  Each lane reads
// back exactly the 16-B slices it copied, so no cross-lane synchronisation is needed.
// Same arithmetic (the shared row_* helpers, same order) as k_rows: bit-identical results.
// Measured (Amazon-670K): CSC mode is latency/LSU-bound and prefers D = 2 with
// 6 CTAs/SM; atomic mode is bound by the L1->XBAR red path and is insensitive (D = 3, 4 CTAs).
// MODE: 0 = atomic dh, 1 = CSC pull, 2 = hybrid (columns < split by red, the rest pulled)
#ifndef FF_CSC_RING_D
#define FF_CSC_RING_D 2
#endif
#ifndef FF_CSC_RING_MINB
#define FF_CSC_RING_MINB 5
#endif
#ifndef FF_ATOM_RING_D
#define FF_ATOM_RING_D 3
#endif
#ifndef FF_ATOM_RING_MINB
#define FF_ATOM_RING_MINB 4
#endif
#ifndef FF_SQH_RING_D
#define FF_SQH_RING_D 2
#endif
#ifndef FF_SQH_RING_MINB
#define FF_SQH_RING_MINB 5
#endif
// MODE 3 = atomic dh with the squared hinge: the same code as MODE 0, tuned separately — with
// most reductions skipped the kernel is latency-bound and prefers 2 stages at 5 CTAs/SM
// (0.250 vs 0.265 ms at 100% skips), where the BCE step, bound by the reductions, does not care.
template <int MODE> struct RingCfg {
  static_assert((MODE == 1 ? FF_CSC_RING_D : MODE == 3 ? FF_SQH_RING_D : FF_ATOM_RING_D) >= 2, "ring depth D >= 2");
  static constexpr int D = MODE == 1 ? FF_CSC_RING_D : MODE == 3 ? FF_SQH_RING_D : FF_ATOM_RING_D;  // stages per warp
  static constexpr int kMinBlocks = MODE == 1 ? FF_CSC_RING_MINB : MODE == 3 ? FF_SQH_RING_MINB
                                                                              : FF_ATOM_RING_MINB;  // CTAs per SM
};
constexpr int kRingThreads = 128;
constexpr int kRingStageBytes = 8 * 32 * 16;            // 8 registers x 32 lanes x 16 B = 32 h lines
// MODE 3 (squared hinge) hands each row's weights / indices to the lanes through a transposed
// shared-memory area (two broadcast LDS.128 per 8 values instead of 8 shuffles): 3.5% faster
// there, where the kernel is issue/latency-bound, but 1-2% slower in the BCE (atomic, CSC)
// modes, so only MODE 3 uses it.
template <int MODE> __host__ __device__ constexpr bool ring_xpose() { return MODE == 3; }
// The CSC row pass (MODE 1) gathers its h lines straight into registers instead of through the
// ring (round 2): its rows only write a gradient line (no per-connection reductions), so the
// ring's 8 KB of shared-memory traffic per row was the larger cost — 0.564 vs 0.579 ms per CSC
// step at 5 CTAs/SM (atomic: 0.573 on the same box), parity green.
#ifndef FF_CSC_REG
#define FF_CSC_REG 1              // CSC row pass: 1 = h lines gathered straight into registers (no ring)
#endif
template <int MODE> __host__ __device__ constexpr bool ring_reg() { return MODE == 1 && FF_CSC_REG; }
constexpr int kRingXposeBytes = 256;                         // per stage: c[32] | w[32], transposed
template <int MODE>
constexpr int ring_smem() {
  return ring_reg<MODE>() ? 0 : (kRingThreads / 32) * RingCfg<MODE>::D * (kRingStageBytes + (ring_xpose<MODE>() ? kRingXposeBytes : 0));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const float* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }
__device__ __forceinline__ float4 lds4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
  return v;
}

// Opaque copy of a thread-constant value: ptxas cannot rematerialise an asm output, so the
// value stays in a register instead of being recomputed from %tid in every loop iteration
// (ncu source attribution: ~50 instructions per label row went to that in the ring kernel).
__device__ __forceinline__ int pin(int v) { asm volatile("" : "+r"(v)); return v; }
__device__ __forceinline__ uint32_t pin(uint32_t v) { asm volatile("" : "+r"(v)); return v; }
template <class T>
__device__ __forceinline__ T* pin(T* p) { asm volatile("" : "+l"(p)); return p; }

template <bool STORE_GRADS, int MODE>
__global__ void __launch_bounds__(kRingThreads, RingCfg<MODE>::kMinBlocks) k_train_ring(RowArgs a) {
  pdl_begin();
  const AdamArgs adam = step_adam(a);
  constexpr int NG = 8, D = RingCfg<MODE>::D;
  constexpr bool CSC = MODE == 1 || MODE == 2, HYB = MODE == 2;
  constexpr uint32_t kColFloats = 64;                   // hd column stride at nb = 1 (h | dh lines)
  extern __shared__ __align__(16) unsigned char ring_smem[];
  const int lane = pin((int)(threadIdx.x & 31)), gq = pin(lane >> 3), bq = pin(lane & 7);
  const int nwarp = (int)(((int64_t)gridDim.x * blockDim.x) >> 5);
  // this lane's slot of stage 0 of this warp's ring; slot of connection 4q + gq = + q * 512
  const uint32_t ring0 = pin((uint32_t)__cvta_generic_to_shared(ring_smem) +
                             (uint32_t)(threadIdx.x >> 5) * D * kRingStageBytes + (uint32_t)lane * 16u);
  const uint64_t pol_l = policy_evict_last();
  const int B = a.B;
  float* const hb = pin(a.hd + 4 * bq);
  float* const W = a.W; float* const mW = a.mW; float* const vW = a.vW;
  const int* const idx = a.idx;
  const float grad_scale = a.grad_scale;
  const bool want_loss = a.loss != nullptr, check = a.check_finite != 0, sqh = a.sqh != 0;
  const uint32_t split = a.split;
  const int64_t jb = a.j_begin, je = a.j_end;
  const int b = pin(4 * bq + gq);                       // this lane's own sample
  const bool bvalid = b < B;
  float loss_acc = 0.0f;

  // this warp's rows: the contiguous range [r_lo, r_hi) of the launch's rows (relative to
  // j_begin), walked one row at a time; the per-label vectors (bias, moments, positive mask)
  // are handled in blocks of 32 rows from r_lo (lane i <-> row block + i).  The cursor is the
  // row index alone (32-bit: L * k < 2^31).
  const uint32_t nrows = (uint32_t)(je - jb), jb32 = (uint32_t)jb;
  const uint32_t wq = (uint32_t)global_warp();
  const uint32_t r_lo = (uint32_t)(((uint64_t)nrows * wq) / (uint32_t)nwarp);
  const uint32_t r_hi = (uint32_t)(((uint64_t)nrows * (wq + 1)) / (uint32_t)nwarp);
  using Cur = uint32_t;
  auto adv = [&](Cur c) { return c + 1u; };
  auto live = [&](Cur c) { return c < r_hi; };
  auto row_of = [&](Cur c) { return jb32 + c; };
  auto i_of = [&](Cur c) { return (int)((c - r_lo) & 31u); };

  struct St { float w, mw, vw; int c; };
  auto load_st = [&](Cur cu, St& st) {
    if (live(cu)) {
      const uint32_t row = row_of(cu) * 32u + lane;
      st.w = ld_na(W + row);
      st.c = ld_na_ro(idx + row);
      st.mw = ld_na(mW + row);
      st.vw = ld_na(vW + row);
    }
  };
  struct Bv { float bias, mb, vb; uint32_t pm; };
  auto load_bv = [&](Cur cu, Bv& v) {                   // cu = the first row of a block
    v.bias = v.mb = v.vb = 0.0f; v.pm = 0u;
    if (live(cu) && (uint32_t)lane < r_hi - cu) {
      const uint32_t j = jb32 + cu + lane;
      v.bias = ld_na(a.bias + j); v.mb = ld_na(a.mb + j); v.vb = ld_na(a.vb + j); v.pm = a.posmask[j];
    }
  };
  constexpr bool XP = ring_xpose<MODE>();
  // (MODE 3) per stage a 256-B hand-off area: the row's indices and weights stored transposed,
  // so that lane (gq, bq) reads the 8 values of its connections 4q + gq as two LDS.128
  const uint32_t xbase = pin((uint32_t)__cvta_generic_to_shared(ring_smem) +
                             (uint32_t)((kRingThreads / 32) * D * kRingStageBytes) +
                             (uint32_t)(threadIdx.x >> 5) * D * (uint32_t)kRingXposeBytes);
  const uint32_t xslot = pin((uint32_t)(((lane & 3) * 8 + (lane >> 2)) * 4));
  auto xld8 = [&](uint32_t a, uint32_t (&v)[8]) {
    uint4 x0, x1;
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(x0.x), "=r"(x0.y), "=r"(x0.z), "=r"(x0.w) : "r"(a) : "memory");
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(x1.x), "=r"(x1.y), "=r"(x1.z), "=r"(x1.w) : "r"(a + 16u) : "memory");
    v[0] = x0.x; v[1] = x0.y; v[2] = x0.z; v[3] = x0.w; v[4] = x1.x; v[5] = x1.y; v[6] = x1.z; v[7] = x1.w;
  };
  constexpr bool REG = ring_reg<MODE>();
  // gathers of one row into ring stage `stg` (always commits a group, possibly empty)
  auto issue = [&](Cur cu, const St& st, uint32_t stg) {
    if (REG) return;                                    // gathered at compute time
    if (live(cu)) {
      const uint32_t dst = ring0 + stg * (uint32_t)kRingStageBytes;
      if constexpr (XP) {
        const uint32_t xa = xbase + stg * (uint32_t)kRingXposeBytes;
        __syncwarp();                                   // the stage's previous row is fully read
        asm volatile("st.shared.b32 [%0], %1;" :: "r"(xa + xslot), "r"(st.c) : "memory");
        asm volatile("st.shared.b32 [%0], %1;" :: "r"(xa + 128u + xslot), "r"(__float_as_uint(st.w)) : "memory");
        __syncwarp();
        uint32_t cc[8];
        xld8(xa + (uint32_t)gq * 32u, cc);
#pragma unroll
        for (int q = 0; q < NG; ++q) cp_async16(dst + (uint32_t)q * 512u, col_line(hb, cc[q], kColFloats));
      } else {
#pragma unroll
        for (int q = 0; q < NG; ++q) {
          const uint32_t c = (uint32_t)__shfl_sync(kFull, st.c, 4 * q + gq);
          cp_async16(dst + (uint32_t)q * 512u, col_line(hb, c, kColFloats));
        }
      }
    }
    cp_async_commit();
  };

  Cur X = r_lo;
  if (live(X)) {                                        // (no early return: block_atomic_add syncs)
  // rows X .. X+D-2 in flight before the loop; states of rows X .. X+D-1 loaded
  Cur q_cur[D];
  St q_st[D];
  q_cur[0] = X;
#pragma unroll
  for (int d = 1; d < D; ++d) q_cur[d] = adv(q_cur[d - 1]);
#pragma unroll
  for (int d = 0; d < D; ++d) load_st(q_cur[d], q_st[d]);
#pragma unroll
  for (int d = 0; d < D - 1; ++d) issue(q_cur[d], q_st[d], (uint32_t)d);
  Bv bv{}, bv_next{};
  load_bv(X, bv);
  float db_v = 0.0f;
  uint32_t stg = 0;                                     // ring stage of the row being computed

  while (true) {
    // issue the row D-1 ahead into the stage freed by the previous compute; load the state
    // of the row after it
    issue(q_cur[D - 1], q_st[D - 1], stg == 0 ? (uint32_t)(D - 1) : stg - 1);
    const Cur cu = q_cur[0];
    St st = q_st[0];
#pragma unroll
    for (int d = 0; d < D - 1; ++d) { q_cur[d] = q_cur[d + 1]; q_st[d] = q_st[d + 1]; }
    q_cur[D - 1] = adv(q_cur[D - 2]);
    load_st(q_cur[D - 1], q_st[D - 1]);
    if (live(q_cur[0]) && i_of(q_cur[0]) == 0) load_bv(q_cur[0], bv_next);

    float4 hv[NG];
    if constexpr (REG) {
#pragma unroll
      for (int q = 0; q < NG; ++q)
        hv[q] = ld_line4_plain(col_line(hb, (uint32_t)__shfl_sync(kFull, st.c, 4 * q + gq), kColFloats));
    } else {
      cp_async_wait<D - 1>();                           // this row's group is complete
      const uint32_t src = ring0 + stg * (uint32_t)kRingStageBytes;
#pragma unroll
      for (int q = 0; q < NG; ++q) hv[q] = lds4(src + (uint32_t)q * 512u);
    }
    float ws[NG];
    uint32_t cq[NG];                                    // (MODE 3) this row's columns of connections 4q + gq
    if constexpr (XP) {
      const uint32_t xa = xbase + stg * (uint32_t)kRingXposeBytes;
      uint32_t wq[8];
      xld8(xa + 128u + (uint32_t)gq * 32u, wq);
#pragma unroll
      for (int q = 0; q < NG; ++q) ws[q] = __uint_as_float(wq[q]);
      xld8(xa + (uint32_t)gq * 32u, cq);
    } else {
#pragma unroll
      for (int q = 0; q < NG; ++q) ws[q] = __shfl_sync(kFull, st.w, 4 * q + gq);
    }

    const uint32_t j = row_of(cu);
    const int i = i_of(cu);
    const float bj = __shfl_sync(kFull, bv.bias, i);
    const uint32_t pm = __shfl_sync(kFull, bv.pm, i);
    const float y = row_score_own<NG>(ws, hv, gq, bj);
    const bool pos_ = (pm >> b) & 1u;
    float lt = 0.0f;
    float g = loss_grad(y, pos_, grad_scale, sqh, &lt);
    if (!bvalid) g = 0.0f;
    if (want_loss && bvalid) loss_acc += lt;
    const bool gany = __any_sync(kFull, g != 0.0f);
    if (check && __any_sync(kFull, bvalid && !isfinite(y)) && lane == 0) atomicOr(a.err, kErrNonFinite);
    float4 g4;
    g4.x = __shfl_sync(kFull, g, (0 << 3) | bq);
    g4.y = __shfl_sync(kFull, g, (1 << 3) | bq);
    g4.z = __shfl_sync(kFull, g, (2 << 3) | bq);
    g4.w = __shfl_sync(kFull, g, (3 << 3) | bq);
    float dwp[NG];
#pragma unroll
    for (int q = 0; q < NG; ++q) dwp[q] = dw_partial(g4, hv[q]);
    if (CSC) {
      // the row's record: its gradient line and (at +32 floats) its pre-update weights, two
      // coalesced 128-B lines (0 weights when the row's gradient is all zero)
      float* const rec = a.gT + (size_t)(j - jb32) * (uint32_t)a.rs;
      st_hint(rec + b, g, pol_l);
      st_hint(rec + 32 + lane, gany ? st.w : 0.0f, pol_l);
      if (HYB) {                                         // hybrid: columns < split by red
        const bool gnz = (g4.x != 0.0f) | (g4.y != 0.0f) | (g4.z != 0.0f) | (g4.w != 0.0f);
#pragma unroll
        for (int q = 0; q < NG; ++q) {
          const uint32_t c = (uint32_t)__shfl_sync(kFull, st.c, 4 * q + gq);
          if (gnz && c < split) red_add4(col_line(hb, c, kColFloats) + 32, dh_contrib(ws[q], g4), pol_l);
        }
      }
    } else if (!sqh || gany) {                           // (squared hinge: an all-zero row reduces nothing)
      const bool gnz = (g4.x != 0.0f) | (g4.y != 0.0f) | (g4.z != 0.0f) | (g4.w != 0.0f);
#pragma unroll
      for (int q = 0; q < NG; ++q) {
        const uint32_t c = XP ? cq[q] : (uint32_t)__shfl_sync(kFull, st.c, 4 * q + gq);
        if (gnz) red_add4(col_line(hb, c, kColFloats) + 32, dh_contrib(ws[q], g4), pol_l);
      }
    }
    // implicit negative mining (squared hinge): a row whose gradient is exactly zero
    // for every sample has dW = db = 0 — the transpose-reduce is skipped (warp-uniform branch;
    // the same values up to the sign of zero, which Adam does not see)
    float gW = 0.0f, dbr = 0.0f;
    if (!sqh || gany) {
      gW = row_dw_slot<NG>(dwp, lane);
      dbr = row_db_chunk(g4);
    }
    if (lane == i) db_v = dbr;
    const uint32_t row = j * 32u + lane;
    if (STORE_GRADS) a.dW[row] = gW;
    adam_update(st.w, st.mw, st.vw, gW, adam);
    st_na(W + row, st.w);
    st_na(mW + row, st.mw);
    st_na(vW + row, st.vw);
    if (i == 31 || cu + 1u == r_hi) {                   // block done: vectorized bias update
      const uint32_t jl = jb32 + (cu - (uint32_t)i) + lane;
      if (lane <= i) {
        if (bv.pm != 0u) a.posmask[jl] = 0u;
        if (STORE_GRADS) a.db[jl] = db_v;
        float p = bv.bias, mo = bv.mb, ve = bv.vb;
        adam_update(p, mo, ve, db_v, adam);
        st_na(a.bias + jl, p);
        st_na(a.mb + jl, mo);
        st_na(a.vb + jl, ve);
      }
      db_v = 0.0f;
    }
    stg = stg + 1 == (uint32_t)D ? 0u : stg + 1;
    if (!live(q_cur[0])) break;
    if (i_of(q_cur[0]) == 0) bv = bv_next;
  }
  cp_async_wait<0>();
  }
  if (a.loss != nullptr) block_atomic_add(loss_acc * a.grad_scale, a.loss);
}

// ---------------------------------------------------------------------- CSC dh pull
// Alg. 2 as a gather over the transposed (CSC) index: for every column c,
//   dh[b][c] = sum_{p in col c} W_old[j_p][i_p] * g[b][j_p]
// with entries in (label tile, column, row) order — deterministic, no atomics.  The
// transposed index is split by label tile so that the records a launch gathers were
// written by the row launch just before it (L2-resident).  Entry p is the packed
// (row within the tile << 6) | slot; the row pass left, per row of the tile, one record of
// rs floats: the gradient line of each 32-sample chunk, then the row's pre-update weights.
// So the column pass reads the entry stream coalesced and, per entry, one 128-B gradient
// line plus the one 32-B sector holding W_old[j][i] — the hand-off of the pre-update
// weights costs the row pass one coalesced line per row instead of k scattered stores.
// Tile t covers col_ptr segments [t*m + c]; tile 0 writes the dh half of hd, later tiles
// accumulate into it.  Warp per column (grid-stride); lane (gq, bq) takes entry 4u + gq of
// each 32-entry batch and samples 4bq..4bq+3 (one 16-B slice of the 128-B g line).
// SKIPZ (squared hinge): a zero weight (a row whose gradient is all zero) skips the gather;
// the weight is then loaded before the gathers instead of beside them.
#ifndef FF_CSC_PLAIN
#define FF_CSC_PLAIN 1            // g-line gathers without the L2 policy operand (1% faster CSC step)
#endif
template <bool NB1, bool SKIPZ>
__global__ void __launch_bounds__(256) k_dh_csc(const int* __restrict__ col_ptr, const int* __restrict__ ent,
                                                const float* __restrict__ gT, int rs, int m, int nb_rt, int tile,
                                                float* __restrict__ hd, int c_begin) {
  pdl_begin();
  const int nb = NB1 ? 1 : nb_rt;
  const int lane = threadIdx.x & 31, gq = lane >> 3, bq = lane & 7;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const uint64_t pol_l = policy_evict_last();
  const int* cp = col_ptr + (int64_t)tile * m;
  const uint32_t rsu = (uint32_t)rs, woff = 32u * (uint32_t)nb;
  // one batch of up to 32 entries [p, p + 32) of a column ending at pend, for chunk q2:
  // returns the lane's 4-sample partial sums added to acc
  auto batch = [&](int er, bool ok, int p, int pend, int q2, float4& acc) {
    const bool tail = p + 32 > pend;
    const uint32_t rec = (uint32_t)er >> 6;
    const float* gb = gT + q2 * 32 + 4 * bq;
    float wv = 0.0f;
    if (SKIPZ && ok) wv = ld_na(gT + (size_t)rec * rsu + woff + ((uint32_t)er & 63u));
    float4 gv[8]; float ww[8];
    if (SKIPZ) {
#pragma unroll
      for (int u = 0; u < 8; ++u) ww[u] = __shfl_sync(kFull, wv, 4 * u + gq);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t grow = (uint32_t)__shfl_sync(kFull, (int)rec, 4 * u + gq);
      gv[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      const bool live = !tail || p + 4 * u + gq < pend;
#if FF_CSC_PLAIN
      if (live && (!SKIPZ || ww[u] != 0.0f)) gv[u] = ld_line4_plain(col_line(gb, grow, rsu));
#else
      if (live && (!SKIPZ || ww[u] != 0.0f)) gv[u] = ld_line4(col_line(gb, grow, rsu), pol_l);
#endif
    }
    if (!SKIPZ) {
      // issued after the gathers: the weight load and the gathers are in flight together
      if (ok) wv = ld_na(gT + (size_t)rec * rsu + woff + ((uint32_t)er & 63u));
#pragma unroll
      for (int u = 0; u < 8; ++u) ww[u] = __shfl_sync(kFull, wv, 4 * u + gq);
    }
    float2 a01 = lo2(acc), a23 = hi2(acc);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a01 = ffma2(bc2(ww[u]), lo2(gv[u]), a01);
      a23 = ffma2(bc2(ww[u]), hi2(gv[u]), a23);
    }
    acc = make_float4(a01.x, a01.y, a23.x, a23.y);
  };
  auto finish = [&](int c, int q2, float4 acc) {
#pragma unroll
    for (int o = 8; o <= 16; o <<= 1) {
      acc.x += __shfl_xor_sync(kFull, acc.x, o); acc.y += __shfl_xor_sync(kFull, acc.y, o);
      acc.z += __shfl_xor_sync(kFull, acc.z, o); acc.w += __shfl_xor_sync(kFull, acc.w, o);
    }
    if (gq == 0) {
      float4* dst = reinterpret_cast<float4*>(hd + (int64_t)c * 64 * nb + q2 * 64 + 32 + 4 * bq);
      if (tile > 0) {
        const float4 o = *dst;
        acc = make_float4(o.x + acc.x, o.y + acc.y, o.z + acc.z, o.w + acc.w);
      }
      *dst = acc;
    }
  };
  if (NB1) {
    // B <= 32: the entries of the next batch — in this column, or the first batch of the
    // warp's next column — are loaded while the current batch's gathers run, so the entry
    // stream's DRAM latency is not exposed once per batch.
    auto load_ent = [&](int p, int pend, int& er, bool& ok) {
      ok = p + lane < pend;
      er = ok ? ld_na_ro(ent + p + lane) : 0;
    };
    int c = c_begin + (int)global_warp();
    int p0 = 0, p1 = 0, er_n = 0;
    bool ok_n = false;
    if (c < m) { p0 = cp[c]; p1 = cp[c + 1]; load_ent(p0, p1, er_n, ok_n); }
    for (; c < m; c += nw) {
      const int cn = c + nw;
      int q0 = 0, q1 = 0;
      if (cn < m) { q0 = cp[cn]; q1 = cp[cn + 1]; }
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int p = p0; p < p1; p += 32) {
        const int er = er_n; const bool ok = ok_n;
        if (p + 32 < p1) load_ent(p + 32, p1, er_n, ok_n);        // next batch, same column
        else if (cn < m) load_ent(q0, q1, er_n, ok_n);            // first batch of the next column
        batch(er, ok, p, p1, 0, acc);
      }
      if (p0 == p1 && cn < m) load_ent(q0, q1, er_n, ok_n);        // empty column: prefetch here
      finish(c, 0, acc);
      p0 = q0; p1 = q1;
    }
    return;
  }
  for (int c = c_begin + (int)global_warp(); c < m; c += nw) {
    const int p0 = cp[c], p1 = cp[c + 1];
    for (int q2 = 0; q2 < nb; ++q2) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int p = p0; p < p1; p += 32) {
        const bool ok = p + lane < p1;
        const int er = ok ? ld_na_ro(ent + p + lane) : 0;
        batch(er, ok, p, p1, q2, acc);
      }
      finish(c, q2, acc);
    }
  }
}

// CSC build step 1: key = tile(row) * m + column, value = connection id e (row-major), so a
// stable radix sort by key yields entries in (tile, column, row) order.
__global__ void k_csc_keys(const int* __restrict__ idx, int64_t n, int k, int m, int64_t tile_rows,
                           int* __restrict__ keys, int* __restrict__ vals) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tile = (e / k) / tile_rows;
    keys[e] = (int)(tile * m + idx[e]);
    vals[e] = (int)e;
  }
}
// CSC build step 2: ent[p] = (row within its tile << 6) | slot of the p-th entry; col_ptr
// over the key space [0, nkeys] from the sorted keys (col_ptr[q] = first p with key >= q).
__global__ void k_csc_finish(const int* __restrict__ skeys, const int* __restrict__ svals, int64_t n, int k,
                             int64_t tile_rows, int nkeys, int* __restrict__ ent, int* __restrict__ col_ptr) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int e = svals[p];
    const int key = skeys[p];
    const int prev = p > 0 ? skeys[p - 1] : -1;
    const int j = e / k, i = e - j * k;
    ent[p] = (int)(((int64_t)j % tile_rows) << 6) | i;
    for (int c = prev + 1; c <= key; ++c) col_ptr[c] = (int)p;
    if (p == n - 1)
      for (int c = key + 1; c <= nkeys; ++c) col_ptr[c] = (int)n;
  }
  if (n == 0 && blockIdx.x == 0)
    for (int c = threadIdx.x; c <= nkeys; c += blockDim.x) col_ptr[c] = 0;
}

// ------------------------------------------------------------------------------ prep
// hd[c][q2][r] = h[q2*32 + r][c] (0 for samples >= B), hd[c][q2][32 + r] = 0 (dh
// accumulator), positives -> posmask bits, *loss = 0.  Grid: ceil(m/32) blocks of 32x8.
// VEC (m % 4 == 0, 16-B aligned h): 16-B loads of h rows and 16-B stores of the lines,
// through a conflict-free [32][33] shared tile (scalar smem accesses).
template <bool VEC>
__global__ void k_prep(const float* __restrict__ h, int B, int m, int nb, float* __restrict__ hd, int zero_dh,
                       const int* __restrict__ lbl_ptr, const int* __restrict__ lbl_ids,
                       uint32_t* __restrict__ posmask, int64_t L_local, int64_t row_begin,
                       int64_t L_global, float* loss, int* err, int64_t* t_dev, float* rbc, float beta1,
                       float beta2, int64_t* t2_dev, float* rbc2, float beta1d, float beta2d) {
  pdl_begin();
  __shared__ float t[32][33];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  if (t_dev != nullptr && blockIdx.x == 0 && tid == 0) {
    // training step: t <- t + 1 and the Adam bias corrections 1/(1 - beta^t) (fp64, R6/R7)
    const int64_t tn = *t_dev + 1;
    *t_dev = tn;
#ifndef FF_PREP_NOPOW
    rbc[0] = (float)(1.0 / (1.0 - pow((double)beta1, (double)tn)));
    rbc[1] = (float)(1.0 / (1.0 - pow((double)beta2, (double)tn)));
#else
    rbc[0] = 1.0f; rbc[1] = 1.0f;
#endif
  }
  if (t2_dev != nullptr && blockIdx.x == 0 && tid == 32) {
    // whole-architecture step: the dense layer's own counter (R28), after its dropout read it
    const int64_t tn = *t2_dev + 1;
    *t2_dev = tn;
    rbc2[0] = (float)(1.0 / (1.0 - pow((double)beta1d, (double)tn)));
    rbc2[1] = (float)(1.0 / (1.0 - pow((double)beta2d, (double)tn)));
  }
  const int c0 = blockIdx.x * 32;
  const int cstride = 64 * nb;
  if (h != nullptr) {
    for (int q2 = 0; q2 < nb; ++q2) {
      if (VEC) {
        const int r = tid >> 3, c4 = tid & 7, b = q2 * 32 + r, c = c0 + 4 * c4;
        const float4 v = (b < B && c < m) ? *reinterpret_cast<const float4*>(h + (int64_t)b * m + c)
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
        t[4 * c4][r] = v.x; t[4 * c4 + 1][r] = v.y; t[4 * c4 + 2][r] = v.z; t[4 * c4 + 3][r] = v.w;
        __syncthreads();
        const int cl = tid >> 3, q = tid & 7;
        if (c0 + cl < m) {
          float* line = hd + (int64_t)(c0 + cl) * cstride + q2 * 64;
          *reinterpret_cast<float4*>(line + 4 * q) = make_float4(t[cl][4 * q], t[cl][4 * q + 1], t[cl][4 * q + 2], t[cl][4 * q + 3]);
          if (zero_dh) *reinterpret_cast<float4*>(line + 32 + 4 * q) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      } else {
        for (int r = ty; r < 32; r += 8) {
          const int b = q2 * 32 + r, c = c0 + tx;
          t[r][tx] = (b < B && c < m) ? h[(int64_t)b * m + c] : 0.0f;
        }
        __syncthreads();
        for (int r = ty; r < 32; r += 8) {
          const int c = c0 + r;
          if (c < m) {
            float* line = hd + (int64_t)c * cstride + q2 * 64;
            line[tx] = t[tx][r];
            if (zero_dh) line[32 + tx] = 0.0f;
          }
        }
      }
      __syncthreads();
    }
  }
  if (lbl_ptr != nullptr) {
    const int lane = tx, wid = blockIdx.x * 8 + ty, nwarps = gridDim.x * 8;
    for (int b = wid; b < B; b += nwarps) {
      for (int q = lbl_ptr[b] + lane; q < lbl_ptr[b + 1]; q += 32) {
        const int64_t gid = lbl_ids[q];
        if (gid < 0 || gid >= L_global) { atomicOr(err, kErrLabelRange); continue; }
        const int64_t j = gid - row_begin;
        if (j >= 0 && j < L_local) atomicOr(posmask + (int64_t)(b >> 5) * L_local + j, 1u << (b & 31));
      }
    }
  }
  if (loss != nullptr && blockIdx.x == 0 && tx == 0 && ty == 0) *loss = 0.0f;
}

// dh[b][c] = hd[c][b/32][32 + b%32] for b < B.  Grid ceil(m/32) x nb, 32x8 threads; VEC as
// in k_prep (16-B line loads and 16-B dh row stores).
template <bool VEC>
__global__ void k_dh_out(const float* __restrict__ hd, int B, int m, int nb, float* __restrict__ dh) {
  pdl_begin();
  __shared__ float t[32][33];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  const int c0 = blockIdx.x * 32, q2 = blockIdx.y;
  if (VEC) {
    const int cl = tid >> 3, q = tid & 7;
    const float4 v = (c0 + cl < m) ? *reinterpret_cast<const float4*>(hd + (int64_t)(c0 + cl) * 64 * nb + q2 * 64 + 32 + 4 * q)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
    t[cl][4 * q] = v.x; t[cl][4 * q + 1] = v.y; t[cl][4 * q + 2] = v.z; t[cl][4 * q + 3] = v.w;
    __syncthreads();
    const int r = tid >> 3, c4 = tid & 7, b = q2 * 32 + r, c = c0 + 4 * c4;
    if (b < B && c < m)
      *reinterpret_cast<float4*>(dh + (int64_t)b * m + c) =
          make_float4(t[4 * c4][r], t[4 * c4 + 1][r], t[4 * c4 + 2][r], t[4 * c4 + 3][r]);
    return;
  }
  for (int r = ty; r < 32; r += 8) {
    const int c = c0 + r;
    t[r][tx] = (c < m) ? hd[(int64_t)c * 64 * nb + q2 * 64 + 32 + tx] : 0.0f;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int b = q2 * 32 + r, c = c0 + tx;
    if (b < B && c < m) dh[(int64_t)b * m + c] = t[tx][r];
  }
}

// ------------------------------------------------------------------------------ Adam
// The device step counter of the unfused path (adam_step): as in k_prep.
__global__ void k_step_t(int64_t* t_dev, float* rbc, float beta1, float beta2) {
  if (threadIdx.x == 0) {
    const int64_t tn = *t_dev + 1;
    *t_dev = tn;
    rbc[0] = (float)(1.0 / (1.0 - pow((double)beta1, (double)tn)));
    rbc[1] = (float)(1.0 / (1.0 - pow((double)beta2, (double)tn)));
  }
}

// Standalone Adam over W (with dW) and bias (with db).
__global__ void k_adam(float* __restrict__ W, float* __restrict__ mW, float* __restrict__ vW,
                       const float* __restrict__ dW, int64_t n, float* __restrict__ bias,
                       float* __restrict__ mb, float* __restrict__ vb, const float* __restrict__ db,
                       int64_t L, AdamArgs a, const float* rbc) {
  a.rbc1 = rbc[0]; a.rbc2 = rbc[1];                     // this step's bias corrections (k_step_t)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n + L; e += stride) {
    if (e < n) {
      float p = W[e], mo = mW[e], ve = vW[e];
      adam_update(p, mo, ve, dW[e], a);
      W[e] = p; mW[e] = mo; vW[e] = ve;
    } else {
      const int64_t j = e - n;
      float p = bias[j], mo = mb[j], ve = vb[j];
      adam_update(p, mo, ve, db[j], a);
      bias[j] = p; mb[j] = mo; vb[j] = ve;
    }
  }
}

// ------------------------------------------------------------------------------ init
// Uniform random connections: row j's slot i gets the i-th accepted draw of
// the init-idx stream (Lemire, rejecting duplicates); W[j][i] = a*(2*(u>>8)*2^-24 - 1) in
// fp32 from word i of the init-W stream (R17).  Also zeroes bias and the moments.
// Warp per row; lane owns slots lane and lane + 32 (k <= 64).
__global__ void k_init(float* __restrict__ W, int* __restrict__ idx, float* __restrict__ bias,
                       float* __restrict__ mW, float* __restrict__ vW, float* __restrict__ mb,
                       float* __restrict__ vb, int64_t L, int64_t row_begin, int m, int k,
                       uint32_t key0, uint32_t key1, float scale) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t thr = (uint32_t)(0x100000000ull % (uint64_t)m);
  for (int64_t j = global_warp(); j < L; j += nw) {
    const uint32_t grow = (uint32_t)(row_begin + j);
    int mine[2] = {-1, -1};
    int count = 0;
    for (uint32_t n = 0; count < k; ++n) {
      const U4 v = philox(n, grow, 0u, kDomInitIdx, key0, key1);
#pragma unroll
      for (int wi = 0; wi < 4; ++wi) {
        if (count < k) {
          const int cand = lemire_draw(word_of(v, wi), (uint32_t)m, thr);
          if (cand >= 0 && __ballot_sync(kFull, (lane < count && mine[0] == cand) ||
                                                  (lane + 32 < count && mine[1] == cand)) == 0u) {
            if (lane == (count & 31)) mine[count >> 5] = cand;
            ++count;
          }
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int slot = lane + 32 * e;
      if (slot < k) {
        const U4 v = philox((uint32_t)(slot >> 2), grow, 0u, kDomInitW, key0, key1);
        const uint32_t u = word_of(v, slot & 3);
        const float unit = __fmul_rn((float)(u >> 8), 1.0f / 16777216.0f);
        const float centered = __fsub_rn(__fmul_rn(2.0f, unit), 1.0f);
        const int64_t el = j * k + slot;
        idx[el] = mine[e];
        W[el] = __fmul_rn(scale, centered);
        mW[el] = 0.0f; vW[el] = 0.0f;
      }
    }
    if (lane == 0) { bias[j] = 0.0f; mb[j] = 0.0f; vb[j] = 0.0f; }
  }
}

// ---------------------------------------------------------------------- redistribution
// SET prune/regrow per row (R8-R14).  Warp per row, lane owns slots
// lane and lane + 32 (k <= 64): rank of (|W| bits, slot) among the row; the p lowest are
// pruned; the regrow stream (domain 2, counter (n, global row, step, 2)) yields candidates
// uniform on [0,m) that are accepted when not in the pre-call row set and not yet accepted;
// the q-th accepted index goes to the q-th pruned slot in ascending slot order; W = mW =
// vW = 0 there.
// K64: k in (32, 64] (a second slot per lane); otherwise k <= 32 and the second half is
// compiled out (the hot configuration k = 32: ~40% fewer instructions per row).
template <bool K64>
__global__ void k_redistribute(float* __restrict__ W, int* __restrict__ idx, float* __restrict__ mW,
                               float* __restrict__ vW, int64_t L, int64_t row_begin, int m, int k,
                               int p, uint32_t step, uint32_t key0, uint32_t key1) {
  // The p pruned slots are the p smallest (|W| bits, slot) keys of the row (R9), found by p
  // rounds of a warp min (redux.sync) + lowest-lane ballot: the same set as ranking every slot
  // against every other.  The next row's W and idx are loaded while this row is processed.
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t thr = (uint32_t)(0x100000000ull % (uint64_t)m);
  bool act[2];
  act[0] = lane < k;
  act[1] = K64 && lane + 32 < k;
  float w_n[2] = {0.0f, 0.0f}; int c_n[2] = {-1, -1};
  auto load = [&](int64_t jj) {
#pragma unroll
    for (int e = 0; e < 2; ++e)
      if (act[e]) { w_n[e] = ld_na(W + jj * k + lane + 32 * e); c_n[e] = idx[jj * k + lane + 32 * e]; }   // idx is written here: no .nc
  };
  int64_t j = global_warp();
  if (j < L) load(j);
  // the first Philox block (n = 0) of the warp's next 32 rows, one row per lane: draw words
  // for row j + i nw come from lane i by shuffle (usually all p draws come from it); further
  // blocks (n >= 1) are computed by the whole warp when a row needs them
  U4 pre{0u, 0u, 0u, 0u};
  int i_pre = 32;
  for (; j < L; j += nw) {
    if (i_pre == 32) {
      pre = philox(0u, (uint32_t)(row_begin + j + (int64_t)lane * nw), step, kDomRegrow, key0, key1);
      i_pre = 0;
    }
    const int src_lane = i_pre++;
    int c[2]; uint32_t key[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      c[e] = c_n[e];
      key[e] = act[e] ? (__float_as_uint(w_n[e]) & 0x7fffffffu) : 0xffffffffu;
    }
    if (j + nw < L) load(j + nw);
    uint32_t pm0 = 0u, pm1 = 0u;                       // pruned slots (bit = lane), halves e = 0, 1
    for (int r = 0; r < p; ++r) {
      const uint32_t kmin = __reduce_min_sync(kFull, min(key[0], key[1]));
      const uint32_t b0 = __ballot_sync(kFull, act[0] && key[0] == kmin);
      const uint32_t b1 = __ballot_sync(kFull, act[1] && key[1] == kmin);
      if (b0 != 0u) {                                   // lowest slot first (R9)
        const uint32_t bit = b0 & (0u - b0);
        pm0 |= bit;
        if (lane == __ffs(b0) - 1) key[0] = 0xffffffffu;
      } else {
        const uint32_t bit = b1 & (0u - b1);
        pm1 |= bit;
        if (lane == __ffs(b1) - 1) key[1] = 0xffffffffu;
      }
    }
    const bool pruned0 = (pm0 >> lane) & 1u, pruned1 = (pm1 >> lane) & 1u;
    const uint32_t grow = (uint32_t)(row_begin + j);
    // accepted draws: draw q is held by lane q & 31 in register q >> 5 (p <= 63 since p < k <= 64)
    int acc[2] = {-1, -1}, na = 0;
    for (uint32_t n = 0; na < p; ++n) {
      U4 v;
      if (n == 0) {
        v.x = __shfl_sync(kFull, pre.x, src_lane); v.y = __shfl_sync(kFull, pre.y, src_lane);
        v.z = __shfl_sync(kFull, pre.z, src_lane); v.w = __shfl_sync(kFull, pre.w, src_lane);
      } else {
        v = philox(n, grow, step, kDomRegrow, key0, key1);
      }
#pragma unroll
      for (int wi = 0; wi < 4; ++wi) {
        if (na < p) {
          const int cand = lemire_draw(word_of(v, wi), (uint32_t)m, thr);
          if (cand >= 0) {
            const bool taken = __ballot_sync(kFull, (act[0] && c[0] == cand) || (act[1] && c[1] == cand) ||
                                                    (lane < na && acc[0] == cand) ||
                                                    (lane + 32 < na && acc[1] == cand)) != 0u;
            if (!taken) {
              if (lane == (na & 31)) acc[na >> 5] = cand;
              ++na;
            }
          }
        }
      }
    }
    const int order0 = __popc(pm0 & ((1u << lane) - 1u));
    const int order1 = __popc(pm0) + __popc(pm1 & ((1u << lane) - 1u));
    const int a00 = __shfl_sync(kFull, acc[0], order0 & 31), a01 = __shfl_sync(kFull, acc[1], order0 & 31);
    const int a10 = __shfl_sync(kFull, acc[0], order1 & 31), a11 = __shfl_sync(kFull, acc[1], order1 & 31);
    const int new0 = order0 < 32 ? a00 : a01;
    const int new1 = order1 < 32 ? a10 : a11;
    if (pruned0) { const int64_t el = j * k + lane; idx[el] = new0; W[el] = 0.0f; mW[el] = 0.0f; vW[el] = 0.0f; }
    if (pruned1) { const int64_t el = j * k + lane + 32; idx[el] = new1; W[el] = 0.0f; mW[el] = 0.0f; vW[el] = 0.0f; }
  }
}

// The host entry point's loss output: one store into page-locked host memory (mapped,
// device-addressable), instead of a copy-engine D2H on the step's stream.
__global__ void k_store_scalar(const float* __restrict__ src, float* dst) {
  if (threadIdx.x == 0) { *dst = *src; __threadfence_system(); }
}

// Validation for set_params: idx in [0, m), distinct within each row (k <= 64).
__global__ void k_validate_idx(const int* __restrict__ idx, int64_t L, int m, int k, int* err) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = global_warp(); j < L; j += nw) {
    bool act[2]; int c[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      act[e] = lane + 32 * e < k;
      c[e] = act[e] ? idx[j * k + lane + 32 * e] : -1 - lane - 32 * e;   // distinct sentinels
      if (act[e] && (c[e] < 0 || c[e] >= m)) atomicOr(err, kErrIdxRange);
    }
    bool dup = false;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int cq0 = __shfl_sync(kFull, c[0], q), cq1 = __shfl_sync(kFull, c[1], q);
      dup |= act[0] && ((q != lane && cq0 == c[0]) || cq1 == c[0]);
      dup |= act[1] && ((q != lane && cq1 == c[1]) || cq0 == c[1]);
    }
    if (dup) atomicOr(err, kErrIdxDup);
  }
}

// ------------------------------------------------------------------------------ top-K
// Total order of the prediction: higher score first, then lower id.
__device__ __forceinline__ bool better(float s, int i, float t, int u) {
  return s > t || (s == t && i < u);
}
__device__ __forceinline__ void topk_insert(float (&ts)[kTopkMax], int (&ti)[kTopkMax], float s, int i) {
#pragma unroll
  for (int q = 0; q < kTopkMax; ++q) {
    if (better(s, i, ts[q], ti[q])) {
      const float s2 = ts[q]; const int i2 = ti[q];
      ts[q] = s; ti[q] = i; s = s2; i = i2;
    }
  }
}

// Insert only when the candidate beats the current K-th entry: after the first rows almost
// every row is rejected by this one comparison (the insertion network is ~70 instructions).
__device__ __forceinline__ void topk_consider(float (&ts)[kTopkMax], int (&ti)[kTopkMax], float s, int i) {
  if (better(s, i, ts[kTopkMax - 1], ti[kTopkMax - 1])) topk_insert(ts, ti, s, i);
}

// Fused forward + per-lane running top-K (y is never written).  For each 32-sample chunk
// q2 every lane owns sample q2*32 + 4*bq + gq; a block merges its warps' lists and writes
// candidates cand[blk][ldh][kTopkMax].
template <int NG, bool FULL>
__global__ void __launch_bounds__(kRowThreads) k_predict(const float* __restrict__ W, const int* __restrict__ idx,
                                                         const float* __restrict__ bias, const float* __restrict__ hd,
                                                         int64_t L, int k, int B, int nb, int64_t row_begin,
                                                         float* __restrict__ cand_s, int* __restrict__ cand_i,
                                                         int* __restrict__ err) {
  __shared__ float ss[kRowThreads / 32][32][kTopkMax];
  __shared__ int si[kRowThreads / 32][32][kTopkMax];
  const int lane = threadIdx.x & 31, gq = lane >> 3, bq = lane & 7, wid = threadIdx.x >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t pol_s = policy_evict_first(), pol_l = policy_evict_last();
  constexpr int KPL = (NG + 7) / 8;
  for (int q2 = 0; q2 < nb; ++q2) {
    const int lo = q2 * 32 + 4 * bq;
    const int b = lo + gq;
    const uint32_t cfl = 64u * (uint32_t)nb;
    const float* hb = hd + q2 * 64 + 4 * bq;
    float ts[kTopkMax]; int ti[kTopkMax];
#pragma unroll
    for (int q = 0; q < kTopkMax; ++q) { ts[q] = -INFINITY; ti[q] = INT_MAX; }
    int64_t j = global_warp();
    float w_n[KPL], bj_n = 0.f; int c_n[KPL];
    auto load = [&](int64_t jj) {
#pragma unroll
      for (int e = 0; e < KPL; ++e) {
        w_n[e] = 0.f; c_n[e] = 0;
        if (lane + 32 * e < k) {
          w_n[e] = ld_stream(W + jj * k + lane + 32 * e, pol_s);
          c_n[e] = ld_stream_ro(idx + jj * k + lane + 32 * e, pol_s);
        }
      }
      bj_n = ld_stream(bias + jj, pol_s);
    };
    if (j < L) load(j);
    for (; j < L; j += nw) {
      float w[KPL]; int c[KPL];
#pragma unroll
      for (int e = 0; e < KPL; ++e) { w[e] = w_n[e]; c[e] = c_n[e]; }
      const float bj = bj_n;
      const int64_t jn = j + nw;
      if (jn < L) load(jn);
      float ws[NG]; uint32_t cs[NG]; float4 hv[NG];
      row_spread_k<NG, KPL>(w, c, gq, ws, cs);
      row_gather<NG, FULL>(hb, cs, cfl, k, gq, pol_l, hv);
      const float y = row_score_own<NG>(ws, hv, gq, bj);
      if (err != nullptr && b < B && !isfinite(y)) atomicOr(err, kErrNonFinite);   // FF_FLAG_CHECK_FINITE (R15)
      if (b < B) topk_consider(ts, ti, y, (int)(row_begin + j));
    }
#pragma unroll
    for (int q = 0; q < kTopkMax; ++q) { ss[wid][lane][q] = ts[q]; si[wid][lane][q] = ti[q]; }
    __syncthreads();
    if (wid == 0) {
      for (int w2 = 1; w2 < (int)(blockDim.x >> 5); ++w2)
#pragma unroll
        for (int q = 0; q < kTopkMax; ++q) topk_insert(ts, ti, ss[w2][lane][q], si[w2][lane][q]);
      const int64_t base = ((int64_t)blockIdx.x * 32 * nb + b) * kTopkMax;
#pragma unroll
      for (int q = 0; q < kTopkMax; ++q) { cand_s[base + q] = ts[q]; cand_i[base + q] = ti[q]; }
    }
    __syncthreads();
  }
}

// Order-preserving int key of a score (atomicMax on floats of either sign) and its inverse.
__device__ __forceinline__ int score_key(float f) { const int i = __float_as_int(f); return i >= 0 ? i : i ^ 0x7FFFFFFF; }
__device__ __forceinline__ float key_score(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7FFFFFFF); }
constexpr int kKeyNegInf = (int)0x807FFFFF;                                   // score_key(-inf)
__global__ void k_fill_i32(int* __restrict__ p, int n, int v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

// Fused forward + running top-K for the hot configuration (k = 32, B <= 32), pipelined like
// k_train_ring: the h-line gathers of the next D - 1 rows are in flight (cp.async into a
// per-warp shared-memory ring) and the state (W, idx, bias) of row X + D is being loaded
// while row X is scored.  Same score arithmetic as k_predict / k_rows (row_score_own on the
// same operands): bit-identical y.  Warp w scores rows w, w + nwarp, ...; the block merges
// its warps' lists into cand[blk][32][kTopkMax] like k_predict.
#ifndef FF_PRED_RING_D
#define FF_PRED_RING_D 2
#endif
#ifndef FF_PRED_RING_THREADS
#define FF_PRED_RING_THREADS 128
#endif
#ifndef FF_PRED_XCH
#define FF_PRED_XCH 16u             // rows between threshold exchanges (power of 2)
#endif
#ifndef FF_PRED_FLUSH_EVERY
#define FF_PRED_FLUSH_EVERY 4u      // rows between candidate-buffer checks (1, 2, 4 or 8)
#endif
constexpr int kPredRingD = FF_PRED_RING_D;
constexpr int kPredRingThreads = FF_PRED_RING_THREADS;
constexpr int kPredRingSmem = (kPredRingThreads / 32) * kPredRingD * 8 * 32 * 16;
template <bool CHECK>                                    // FF_FLAG_CHECK_FINITE: report non-finite scores
__global__ void __launch_bounds__(kPredRingThreads) k_predict_ring(const float* __restrict__ W,
                                                                   const int* __restrict__ idx,
                                                                   const float* __restrict__ bias,
                                                                   const float* __restrict__ hd, int64_t L, int B,
                                                                   int nb, int q2, int64_t row_begin,
                                                                   float* __restrict__ cand_s,
                                                                   int* __restrict__ cand_i,
                                                                   int* __restrict__ gthr, int* __restrict__ err) {
  constexpr int NG = 8, D = kPredRingD;
  constexpr uint32_t kStage = 8 * 32 * 16;
  const uint32_t kColFloats = pin(64u * (uint32_t)nb);   // hd column stride; this launch scores line q2
  extern __shared__ __align__(16) unsigned char ring_smem[];
  // per-warp candidate buffer [slot][lane] while scoring (conflict-free), reused as the
  // block-merge lists [lane][q] at the end (same per-warp 1-KB regions)
  __shared__ float ss[kPredRingThreads / 32][32][kTopkMax];
  __shared__ int si[kPredRingThreads / 32][32][kTopkMax];
  const int lane = threadIdx.x & 31, gq = lane >> 3, bq = lane & 7, wid = threadIdx.x >> 5;
  float* const cbs = &ss[wid][0][0];
  int* const cbi = &si[wid][0][0];
  // thread constants pinned in registers (see pin()): the source lanes 4q + gq of the
  // per-connection shuffles, the ring slot, the h-line base and the state pointers
  const uint32_t nwarp = pin((uint32_t)(((int64_t)gridDim.x * blockDim.x) >> 5));
  const uint32_t ring0 = pin((uint32_t)__cvta_generic_to_shared(ring_smem) + (uint32_t)wid * D * kStage + (uint32_t)lane * 16u);
  const float* const hb = pin(hd + q2 * 64 + 4 * bq);
  const float* const Wp = pin(W);
  const int* const idxp = pin(idx);
  const float* const biasp = pin(bias);
  int sl[NG];
#pragma unroll
  for (int q = 0; q < NG; ++q) sl[q] = pin(4 * q + gq);
  const int b = q2 * 32 + 4 * bq + gq;                   // this lane's sample
  const uint32_t nrows = pin((uint32_t)L);
  float ts[kTopkMax]; int ti[kTopkMax];
#pragma unroll
  for (int q = 0; q < kTopkMax; ++q) { ts[q] = -INFINITY; ti[q] = INT_MAX; }
  float thr_s = -INFINITY; int thr_i = INT_MAX;        // the lane's current K-th best
  int ncand = 0;
  auto flush = [&]() {
    for (int q = 0; q < ncand; ++q) topk_consider(ts, ti, cbs[q * 32 + lane], cbi[q * 32 + lane]);
    ncand = 0;
    if (better(ts[kTopkMax - 1], ti[kTopkMax - 1], thr_s, thr_i)) { thr_s = ts[kTopkMax - 1]; thr_i = ti[kTopkMax - 1]; }
  };
  // Shared threshold per sample (gthr, an order-preserving int key): every 8 rows a lane
  // publishes the kTopkMax-th score of its running list and adopts the best one published by
  // any warp.  That score is the kTopkMax-th of some set of rows, so no row scoring below it
  // can be in the top K <= kTopkMax: skipping y < it is exact (y == it is kept — its id may
  // win the tie), and after the first rows almost no row reaches the candidate buffer.
  int* const gp = gthr + b;
  // (reading the shared value one exchange ahead, so that the load never stalls, measured
  // slower: the stale value lets more lanes publish, and the publishes contend on B words)
  auto exchange = [&]() {
    if (b < B) {
      const int g = *(volatile int*)gp;
      const float own = ts[kTopkMax - 1];
      if (own != -INFINITY && score_key(own) > g) atomicMax(gp, score_key(own));
      const float gs = key_score(g);
      if (gs > thr_s) { thr_s = gs; thr_i = INT_MAX; }
    }
  };
  uint32_t it = 0;

  struct St { float w, bj; int c; };
  auto load_st = [&](uint32_t j, St& st) {
    if (j < nrows) {
      st.w = ld_na(Wp + j * 32u + lane);
      st.c = ld_na_ro(idxp + j * 32u + lane);
      st.bj = ld_na(biasp + j);
    }
  };
  auto issue = [&](uint32_t j, const St& st, uint32_t stg) {
    if (j < nrows) {
      const uint32_t dst = ring0 + stg * kStage;
#pragma unroll
      for (int q = 0; q < NG; ++q) {
        const uint32_t c = (uint32_t)__shfl_sync(kFull, st.c, sl[q]);
        cp_async16(dst + (uint32_t)q * 512u, col_line(hb, c, kColFloats));
      }
    }
    cp_async_commit();
  };
  const uint32_t j0 = (uint32_t)global_warp();
  uint32_t qj[D];
  St qs[D];
#pragma unroll
  for (int d = 0; d < D; ++d) { qj[d] = j0 + (uint32_t)d * nwarp; qs[d] = St{0.f, 0.f, 0}; load_st(qj[d], qs[d]); }
#pragma unroll
  for (int d = 0; d < D - 1; ++d) issue(qj[d], qs[d], (uint32_t)d);
  uint32_t stg = 0;
  while (qj[0] < nrows) {
    issue(qj[D - 1], qs[D - 1], stg == 0 ? (uint32_t)(D - 1) : stg - 1);
    const uint32_t j = qj[0];
    const St st = qs[0];
#pragma unroll
    for (int d = 0; d < D - 1; ++d) { qj[d] = qj[d + 1]; qs[d] = qs[d + 1]; }
    qj[D - 1] = qj[D - 2] + nwarp;
    load_st(qj[D - 1], qs[D - 1]);
    cp_async_wait<D - 1>();
    float4 hv[NG];
    const uint32_t src = ring0 + stg * kStage;
#pragma unroll
    for (int q = 0; q < NG; ++q) hv[q] = lds4(src + (uint32_t)q * 512u);
    float ws[NG];
#pragma unroll
    for (int q = 0; q < NG; ++q) ws[q] = __shfl_sync(kFull, st.w, sl[q]);
    const float y = row_score_own<NG>(ws, hv, gq, st.bj);
    // candidates better than the lane's current K-th best are appended to its buffer (no
    // divergent insertion per row); a full buffer in any lane flushes the warp's buffers
    const int jid = (int)(row_begin + j);
    if (CHECK && b < B && !isfinite(y)) atomicOr(err, kErrNonFinite);              // FF_FLAG_CHECK_FINITE (R15)
    if (b < B && better(y, jid, thr_s, thr_i)) { cbs[ncand * 32 + lane] = y; cbi[ncand * 32 + lane] = jid; ++ncand; }
#if FF_PRED_FLUSH_EVERY == 1
    if (__any_sync(kFull, ncand == kTopkMax)) flush();
    if ((++it & (FF_PRED_XCH - 1u)) == 0) exchange();
#else
    // checked every FF_PRED_FLUSH_EVERY rows: a lane appends at most one candidate per row, so
    // a buffer holding more than kTopkMax - FF_PRED_FLUSH_EVERY is flushed before it can overflow
    if ((++it & (FF_PRED_FLUSH_EVERY - 1u)) == 0) {
      if (__any_sync(kFull, ncand > kTopkMax - FF_PRED_FLUSH_EVERY)) flush();
      if ((it & (FF_PRED_XCH - 1u)) == 0) exchange();
    }
#endif
    stg = stg + 1 == (uint32_t)D ? 0u : stg + 1;
  }
  cp_async_wait<0>();
  flush();
  __syncwarp();
#pragma unroll
  for (int q = 0; q < kTopkMax; ++q) { ss[wid][lane][q] = ts[q]; si[wid][lane][q] = ti[q]; }
  __syncthreads();
  if (wid == 0) {
    for (int w2 = 1; w2 < kPredRingThreads / 32; ++w2)
#pragma unroll
      for (int q = 0; q < kTopkMax; ++q) topk_insert(ts, ti, ss[w2][lane][q], si[w2][lane][q]);
    const int64_t base = ((int64_t)blockIdx.x * 32 * nb + b) * kTopkMax;
#pragma unroll
    for (int q = 0; q < kTopkMax; ++q) { cand_s[base + q] = ts[q]; cand_i[base + q] = ti[q]; }
  }
}

// The same fused forward + running top-K for k = 32, B <= 32 (per 32-sample line q2) with the
// h-line gathers loaded straight into registers (ld.global.v4) instead of through
// k_predict_ring's cp.async shared-memory ring, which moves every gathered byte through
// shared memory twice (the LDGSTS write and the LDS read: 8 KB per row, ~150 us per launch
// at 128 B/clock per SM); register gathers reach 19.9 TB/s vs 11-17.7 TB/s for LDGSTS
// (profiles/r01_gatherbench.txt).  Latency is hidden by occupancy (24 warps/SM at 80
// registers) with the next row's W/idx/bias prefetched.  Measured (profiles/r02_pred_reg.txt):
// 0.191 vs 0.213 ms at B = 32 (0.196 before the line address became one IMAD.WIDE.U32 of the
// column by the line's byte stride, instead of IMAD.WIDE + LEA + LEA.HI.X); a variant that also keeps the next row's 8 lines in flight
// (64 more registers, 16 warps/SM) took 0.27-0.30 ms, and one with the top-K lists in shared
// memory (64 registers, 32 warps/SM) 0.21-0.23 ms.  Same score arithmetic (row_score_own):
// bit-identical y.  Candidates go straight into the lane's register top-K list when they beat
// the lane's threshold (the max of its own K-th best and the per-sample shared threshold of
// k_predict_ring, exchanged every FF_PRED_XCH rows), which after the first rows is rare.
// Output: the block's merged lists in cand[blk][32 nb][kTopkMax], like the ring.
#ifndef FF_PRED_REG_THREADS
#define FF_PRED_REG_THREADS 128
#endif
#ifndef FF_PRED_REG_MINB
#define FF_PRED_REG_MINB 6
#endif
constexpr int kPredRegThreads = FF_PRED_REG_THREADS;
template <bool CHECK>
__global__ void __launch_bounds__(kPredRegThreads, FF_PRED_REG_MINB) k_predict_reg(const float* __restrict__ W,
                                                                                   const int* __restrict__ idx,
                                                                                   const float* __restrict__ bias,
                                                                                   const float* __restrict__ hd, int64_t L,
                                                                                   int B, int nb, int q2, int64_t row_begin,
                                                                                   float* __restrict__ cand_s,
                                                                                   int* __restrict__ cand_i,
                                                                                   int* __restrict__ gthr, int* __restrict__ err) {
  constexpr int NG = 8;
  __shared__ float ss[kPredRegThreads / 32][32][kTopkMax];
  __shared__ int si[kPredRegThreads / 32][32][kTopkMax];
  const int lane = threadIdx.x & 31, gq = lane >> 3, bq = lane & 7, wid = threadIdx.x >> 5;
  const uint32_t kColFloats = pin(64u * (uint32_t)nb);
  const uint32_t nwarp = pin((uint32_t)(((int64_t)gridDim.x * blockDim.x) >> 5));
  const float* const hb = pin(hd + q2 * 64 + 4 * bq);
  int sl[NG];
#pragma unroll
  for (int q = 0; q < NG; ++q) sl[q] = pin(4 * q + gq);
  const int b = q2 * 32 + 4 * bq + gq;
  const uint32_t nrows = pin((uint32_t)L);
  float ts[kTopkMax]; int ti[kTopkMax];
#pragma unroll
  for (int q = 0; q < kTopkMax; ++q) { ts[q] = -INFINITY; ti[q] = INT_MAX; }
  float thr_s = -INFINITY; int thr_i = INT_MAX;
  int* const gp = gthr + b;
  auto exchange = [&]() {
    if (b < B) {
      const int g = *(volatile int*)gp;
      const float own = ts[kTopkMax - 1];
      if (own != -INFINITY && score_key(own) > g) atomicMax(gp, score_key(own));
      const float gs = key_score(g);
      if (gs > thr_s) { thr_s = gs; thr_i = INT_MAX; }
    }
  };
  uint32_t j = (uint32_t)global_warp(), it = 0;
  float w = 0.f, bj = 0.f; int c = 0;
  if (j < nrows) { w = ld_na(W + j * 32u + lane); c = ld_na_ro(idx + j * 32u + lane); bj = ld_na(bias + j); }
  const char* const hbb = reinterpret_cast<const char*>(hb);
  const uint32_t cbytes = pin(4u * kColFloats);          // line address = one IMAD.WIDE.U32 per gather
  while (j < nrows) {
    float4 hv[NG];
#pragma unroll
    for (int q = 0; q < NG; ++q)
      hv[q] = ld_line4_plain(reinterpret_cast<const float*>(hbb + (uint64_t)(uint32_t)__shfl_sync(kFull, c, sl[q]) * cbytes));
    const uint32_t jn = j + nwarp;                       // the next row's state, in flight meanwhile
    float wn = 0.f, bjn = 0.f; int cn = 0;
    if (jn < nrows) { wn = ld_na(W + jn * 32u + lane); cn = ld_na_ro(idx + jn * 32u + lane); bjn = ld_na(bias + jn); }
    float ws[NG];
#pragma unroll
    for (int q = 0; q < NG; ++q) ws[q] = __shfl_sync(kFull, w, sl[q]);
    const float y = row_score_own<NG>(ws, hv, gq, bj);
    const int jid = (int)(row_begin + j);
    if (CHECK && b < B && !isfinite(y)) atomicOr(err, kErrNonFinite);              // FF_FLAG_CHECK_FINITE (R15)
    if (b < B && better(y, jid, thr_s, thr_i)) {
      topk_insert(ts, ti, y, jid);
      if (better(ts[kTopkMax - 1], ti[kTopkMax - 1], thr_s, thr_i)) { thr_s = ts[kTopkMax - 1]; thr_i = ti[kTopkMax - 1]; }
    }
    if ((++it & (FF_PRED_XCH - 1u)) == 0) exchange();
    j = jn; w = wn; c = cn; bj = bjn;
  }
#pragma unroll
  for (int q = 0; q < kTopkMax; ++q) { ss[wid][lane][q] = ts[q]; si[wid][lane][q] = ti[q]; }
  __syncthreads();
  if (wid == 0) {
    for (int w2 = 1; w2 < kPredRegThreads / 32; ++w2)
#pragma unroll
      for (int q = 0; q < kTopkMax; ++q) topk_insert(ts, ti, ss[w2][lane][q], si[w2][lane][q]);
    const int64_t base = ((int64_t)blockIdx.x * 32 * nb + b) * kTopkMax;
#pragma unroll
    for (int q = 0; q < kTopkMax; ++q) { cand_s[base + q] = ts[q]; cand_i[base + q] = ti[q]; }
  }
}

// Fused forward + top-K for large batches (B > 32, k = 32; NEXT-3): the batch is
// scored in chunks of 128 samples (4 hd lines per column; 16 MiB of h lines at m = 32768, so a
// chunk stays L2-resident while every row streams past it).  Per connection one warp
// instruction gathers four 128-B h lines (lane l: line l >> 3 of the chunk, 16-B segment
// l & 7), i.e. 512 B per instruction instead of the ring kernel's 128 B per 8 lanes.  The
// gathers are staged like k_train_ring's: a per-warp ring of D stages in shared memory
// (cp.async, no registers held), one stage = one connection group g (slots g + 4q, q < 8).
// The score of every sample is summed in exactly row_score_own's order — per group g two FMA
// chains (q even / odd) from 0, P_g = a + b, y = ((P_0 + P_2) + (P_1 + P_3)) + bias — so y is
// bit-identical to forward().
// Top-K: each lane owns 4 samples, with a register threshold per sample and a sorted
// kTopkMax list per (warp, sample) in an L2-resident scratch wl[warp][kTopkMax][128]; the
// block merges its warps' lists into cand[blk][b][kTopkMax] per chunk.  The host runs the
// kernel twice: over a prefix of the rows [0, r1) (thr = NULL), whose lists are merged into
// that prefix's exact top-K, then over [r1, L) with thr = that merged list: its K-th entry
// (score, id) starts every lane's threshold.  A row ranked below the K-th of a subset of the
// rows cannot be in the top K, so the skip is exact, and insertions (a dependent walk through
// the list) become rare; the final merge takes the second pass's lists plus the prefix list.
#ifndef FF_PREDW_THREADS
#define FF_PREDW_THREADS 256
#endif
#ifndef FF_PREDW_D
#define FF_PREDW_D 2
#endif
constexpr int kPredWThreads = FF_PREDW_THREADS, kPredWD = FF_PREDW_D;
constexpr int kPredWStage = 8 * 32 * 16;                                     // 8 connections x 512 B
#ifndef FF_PREDW_XPOSE
#define FF_PREDW_XPOSE 1
#endif
constexpr int kPredWSmem = (kPredWThreads / 32) * (kPredWD * kPredWStage + (FF_PREDW_XPOSE ? 3 * 128 : 0));
constexpr int kPredWListFloats = kTopkMax * 128;                             // per warp, per array
__global__ void __launch_bounds__(kPredWThreads) k_predict_wide(const float* __restrict__ W, const int* __restrict__ idx,
                                                                const float* __restrict__ bias,
                                                                const float* __restrict__ hd, int64_t r0, int64_t r1,
                                                                int B, int nb, int64_t row_begin,
                                                                const float* __restrict__ thr_s_in,
                                                                const int* __restrict__ thr_i_in, int K,
                                                                float* __restrict__ cand_s, int* __restrict__ cand_i,
                                                                float* __restrict__ wl_s, int* __restrict__ wl_i,
                                                                int* __restrict__ err) {
  constexpr int BC = 128, NW = kPredWThreads / 32, D = kPredWD;
  extern __shared__ __align__(16) unsigned char wide_smem[];
  float* const lst_s = wl_s + (int64_t)blockIdx.x * NW * kPredWListFloats;     // this block's [NW][kTopkMax][BC]
  int* const lst_i = wl_i + (int64_t)blockIdx.x * NW * kPredWListFloats;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float* const ws = lst_s + wid * kTopkMax * BC;
  int* const wi = lst_i + wid * kTopkMax * BC;
  const uint32_t ring0 = pin((uint32_t)__cvta_generic_to_shared(wide_smem) + (uint32_t)(wid * D * kPredWStage) +
                             (uint32_t)lane * 16u);
  const uint32_t nwarp = pin((uint32_t)(((int64_t)gridDim.x * blockDim.x) >> 5));
  const uint32_t nrows = pin((uint32_t)r1);
  const uint32_t cfl = pin(64u * (uint32_t)nb);            // floats per hd column
  const uint32_t j0 = (uint32_t)r0 + (uint32_t)global_warp();
  const int nchunk = (nb + 3) / 4;
  for (int ch = 0; ch < nchunk; ++ch) {
    const int q2 = ch * 4 + (lane >> 3);                    // this lane's line; samples 4 (lane & 7) + e
    const bool ok = q2 < nb;
    const float* const hb = hd + (ok ? q2 : 0) * 64 + 4 * (lane & 7);
    const int sb = q2 * 32 + 4 * (lane & 7);                // first sample of the lane
    const int s0 = (lane >> 3) * 32 + 4 * (lane & 7);       // its index within the chunk
    for (int t = threadIdx.x; t < NW * kTopkMax * BC; t += blockDim.x) { lst_s[t] = -INFINITY; lst_i[t] = INT_MAX; }
    __syncthreads();
    float thr_s[4]; int thr_i[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      thr_s[e] = -INFINITY; thr_i[e] = INT_MAX;
      if (thr_s_in && ok && sb + e < B) {
        thr_s[e] = thr_s_in[(int64_t)(sb + e) * kTopkMax + K - 1];
        thr_i[e] = thr_i_in[(int64_t)(sb + e) * kTopkMax + K - 1];
      }
    }
    // issue side: group (ji, gi) of the flat (row, group) sequence; ci = that row's idx lane
    uint32_t ji = j0; int gi = 0;
#if FF_PREDW_XPOSE
    // a row's indices / weights are handed to the lanes through shared memory, transposed so
    // that group g's eight slots g + 4q are one 32-B run ([g][q]): two broadcast LDS.128 per
    // group instead of eight shuffles.  Index rows alternate between two buffers by row parity.
    const uint32_t xp0 = (uint32_t)__cvta_generic_to_shared(wide_smem) + (uint32_t)(NW * D * kPredWStage) +
                         (uint32_t)(wid * 3 * 128);                 // cbuf[2][32] | wbuf[32] (ints/floats)
    const uint32_t xslot = (uint32_t)(((lane & 3) * 8 + (lane >> 2)) * 4);
    uint32_t ipar = 0;                                              // parity of row ji's index buffer
    auto sts32 = [](uint32_t a, uint32_t v) { asm volatile("st.shared.b32 [%0], %1;" :: "r"(a), "r"(v) : "memory"); };
    auto lds4u = [](uint32_t a) { uint4 v; asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory"); return v; };
    if (ji < nrows) sts32(xp0 + xslot, (uint32_t)ld_na_ro(idx + ji * 32u + lane));
    int ci_n = ji + nwarp < nrows ? ld_na_ro(idx + (ji + nwarp) * 32u + lane) : 0;
    __syncwarp();
    auto issue = [&](uint32_t stg) {
      if (ji < nrows) {
        const uint32_t dst = ring0 + stg * (uint32_t)kPredWStage;
        const uint32_t cb = xp0 + ipar * 128u + (uint32_t)gi * 32u;
        const uint4 c0 = lds4u(cb), c1 = lds4u(cb + 16u);
        const uint32_t cc[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (ok) cp_async16(dst + (uint32_t)q * 512u, col_line(hb, cc[q], cfl));   // lines >= nb: not gathered
      }
      cp_async_commit();
      if (++gi == 4) { gi = 0; ji += nwarp; ipar ^= 1u; }
    };
#else
    int ci = ji < nrows ? ld_na_ro(idx + ji * 32u + lane) : 0;
    int ci_n = ji + nwarp < nrows ? ld_na_ro(idx + (ji + nwarp) * 32u + lane) : 0;
    auto issue = [&](uint32_t stg) {
      if (ji < nrows) {
        const uint32_t dst = ring0 + stg * (uint32_t)kPredWStage;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t c = (uint32_t)__shfl_sync(kFull, ci, 4 * q + gi);
          if (ok) cp_async16(dst + (uint32_t)q * 512u, col_line(hb, c, cfl));    // lines >= nb: not gathered
        }
      }
      cp_async_commit();
      if (++gi == 4) {
        gi = 0; ji += nwarp; ci = ci_n;
        ci_n = ji + nwarp < nrows ? ld_na_ro(idx + (ji + nwarp) * 32u + lane) : 0;
      }
    };
#endif
#pragma unroll
    for (int d = 0; d < D - 1; ++d) issue((uint32_t)d);
    uint32_t stg = 0;
    float w_n = 0.f, b_n = 0.f;
    if (j0 < nrows) { w_n = ld_na(W + j0 * 32u + lane); b_n = ld_na(bias + j0); }
    for (uint32_t j = j0; j < nrows; j += nwarp) {
      const float wl = w_n, bj = b_n;
      if (j + nwarp < nrows) { w_n = ld_na(W + (j + nwarp) * 32u + lane); b_n = ld_na(bias + j + nwarp); }
#if FF_PREDW_XPOSE
      // this row's weights, and the next row's indices (issued during this row's last group)
      __syncwarp();                                        // the previous row's reads are done
      sts32(xp0 + 256u + xslot, __float_as_uint(wl));
      sts32(xp0 + (ipar ^ 1u) * 128u + xslot, (uint32_t)ci_n);   // (the issue side is on row j here, D <= 4)
      ci_n = j + 2u * nwarp < nrows ? ld_na_ro(idx + (j + 2u * nwarp) * 32u + lane) : 0;
      __syncwarp();
#endif
      float2 P[4][2];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        issue(stg == 0 ? (uint32_t)(D - 1) : stg - 1);        // the stage summed last iteration
        cp_async_wait<D - 1>();                               // this group's lines have landed
        const uint32_t src = ring0 + stg * (uint32_t)kPredWStage;
        float2 a0 = make_float2(0.f, 0.f), a1 = a0, b0 = a0, b1 = a0;
#if FF_PREDW_XPOSE
        const uint4 w0 = lds4u(xp0 + 256u + (uint32_t)g * 32u), w1 = lds4u(xp0 + 256u + (uint32_t)g * 32u + 16u);
        const uint32_t wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#endif
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 hv = lds4(src + (uint32_t)q * 512u);
#if FF_PREDW_XPOSE
          const float w = __uint_as_float(wv[q]);
#else
          const float w = __shfl_sync(kFull, wl, 4 * q + g);
#endif
          if (q & 1) { b0 = ffma2(bc2(w), lo2(hv), b0); b1 = ffma2(bc2(w), hi2(hv), b1); }
          else       { a0 = ffma2(bc2(w), lo2(hv), a0); a1 = ffma2(bc2(w), hi2(hv), a1); }
        }
        P[g][0] = make_float2(a0.x + b0.x, a0.y + b0.y);
        P[g][1] = make_float2(a1.x + b1.x, a1.y + b1.y);
        stg = stg + 1 == (uint32_t)D ? 0u : stg + 1;
      }
      const int jid = (int)(row_begin + j);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        auto el = [&](const float2& v) { return (e & 1) ? v.y : v.x; };
        const float y = ((el(P[0][e >> 1]) + el(P[2][e >> 1])) + (el(P[1][e >> 1]) + el(P[3][e >> 1]))) + bj;
        if (err != nullptr && ok && sb + e < B && !isfinite(y)) atomicOr(err, kErrNonFinite);   // (R15)
        if (ok && sb + e < B && better(y, jid, thr_s[e], thr_i[e])) {
          const int s = s0 + e;
          int r = kTopkMax - 1;
          while (r > 0 && better(y, jid, ws[(r - 1) * BC + s], wi[(r - 1) * BC + s])) {
            ws[r * BC + s] = ws[(r - 1) * BC + s]; wi[r * BC + s] = wi[(r - 1) * BC + s]; --r;
          }
          ws[r * BC + s] = y; wi[r * BC + s] = jid;
          const float ks = ws[(kTopkMax - 1) * BC + s]; const int ki = wi[(kTopkMax - 1) * BC + s];
          if (better(ks, ki, thr_s[e], thr_i[e])) { thr_s[e] = ks; thr_i[e] = ki; }
        }
      }
    }
    cp_async_wait<0>();
    __syncthreads();
    // block merge: thread t takes chunk samples t, t + blockDim, ...
    for (int s = threadIdx.x; s < BC; s += blockDim.x) {
      const int b = ch * BC + s;
      if (b >= 32 * nb) break;
      float ts[kTopkMax]; int ti[kTopkMax];
#pragma unroll
      for (int q = 0; q < kTopkMax; ++q) { ts[q] = lst_s[q * BC + s]; ti[q] = lst_i[q * BC + s]; }
      for (int w2 = 1; w2 < NW; ++w2)
#pragma unroll
        for (int q = 0; q < kTopkMax; ++q)
          topk_consider(ts, ti, lst_s[(w2 * kTopkMax + q) * BC + s], lst_i[(w2 * kTopkMax + q) * BC + s]);
      const int64_t base = ((int64_t)blockIdx.x * 32 * nb + b) * kTopkMax;
#pragma unroll
      for (int q = 0; q < kTopkMax; ++q) { cand_s[base + q] = ts[q]; cand_i[base + q] = ti[q]; }
    }
    __syncthreads();
  }
}

// Block per sample: merge `nlist` sorted candidate lists (first Kin entries used) into the
// top K.  Each thread keeps a running top-kTopkMax over lists tid, tid + blockDim, ...; each
// warp reduces its lanes by K rounds of arg-best + pop; warp 0 merges the warps' lists the
// same way.  Exact under the total order (score desc, id asc).
__device__ __forceinline__ void warp_topk_pop(float (&ts)[kTopkMax], int (&ti)[kTopkMax], int K, float* os, int* oi) {
  const int lane = threadIdx.x & 31;
  for (int r = 0; r < K; ++r) {
    float bs = ts[0]; int bi = ti[0];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const float s2 = __shfl_xor_sync(kFull, bs, o); const int i2 = __shfl_xor_sync(kFull, bi, o);
      if (better(s2, i2, bs, bi)) { bs = s2; bi = i2; }
    }
    if (lane == 0) { os[r] = bs; oi[r] = bi; }
    if (ti[0] == bi && ts[0] == bs && bi != INT_MAX) {
#pragma unroll
      for (int q = 0; q < kTopkMax - 1; ++q) { ts[q] = ts[q + 1]; ti[q] = ti[q + 1]; }
      ts[kTopkMax - 1] = -INFINITY; ti[kTopkMax - 1] = INT_MAX;
    }
  }
}
#ifndef FF_MERGE_THREADS
#define FF_MERGE_THREADS 1024
#endif
constexpr int kMergeThreads = FF_MERGE_THREADS;                  // <= 1024 (warp 0 merges <= 32 lists)
__global__ void __launch_bounds__(kMergeThreads) k_merge_topk_block(const float* __restrict__ in_s, const int* __restrict__ in_i,
                                                          int nlist, int64_t list_stride, int64_t sample_stride,
                                                          int Kin, int K, float* __restrict__ out_s,
                                                          int* __restrict__ out_i, int* __restrict__ reset_thr) {
  // the predict path's per-sample shared threshold is re-armed for the next call here (this
  // kernel runs after every kernel that read it)
  if (reset_thr != nullptr && threadIdx.x == 0) reset_thr[blockIdx.x] = kKeyNegInf;
  __shared__ float ws_s[kMergeThreads / 32][kTopkMax];
  __shared__ int ws_i[kMergeThreads / 32][kTopkMax];
  const int b = blockIdx.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwp = blockDim.x >> 5;
  float ts[kTopkMax]; int ti[kTopkMax];
#pragma unroll
  for (int q = 0; q < kTopkMax; ++q) { ts[q] = -INFINITY; ti[q] = INT_MAX; }
  for (int l = threadIdx.x; l < nlist; l += blockDim.x) {
    const int64_t base = (int64_t)l * list_stride + (int64_t)b * sample_stride;
    if (Kin == kTopkMax && (base & 3) == 0) {                // whole 8-entry lists: 16-B loads
      const float4 s0 = *reinterpret_cast<const float4*>(in_s + base), s1 = *reinterpret_cast<const float4*>(in_s + base + 4);
      const int4 i0 = *reinterpret_cast<const int4*>(in_i + base), i1 = *reinterpret_cast<const int4*>(in_i + base + 4);
      const float sv[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
      const int iv[8] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z, i1.w};
#pragma unroll
      for (int q = 0; q < 8; ++q) topk_consider(ts, ti, sv[q], iv[q]);
      continue;
    }
    for (int q = 0; q < Kin; ++q) {
      const float s = in_s[base + q]; const int i = in_i[base + q];
      if (!better(s, i, ts[kTopkMax - 1], ti[kTopkMax - 1])) break;   // lists are sorted
      topk_insert(ts, ti, s, i);
    }
  }
  warp_topk_pop(ts, ti, K, ws_s[wid], ws_i[wid]);
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int q = 0; q < kTopkMax; ++q) { ts[q] = -INFINITY; ti[q] = INT_MAX; }
    if (lane < nwp)
      for (int q = 0; q < K; ++q) topk_insert(ts, ti, ws_s[lane][q], ws_i[lane][q]);
    warp_topk_pop(ts, ti, K, out_s + (int64_t)b * K, out_i + (int64_t)b * K);
  }
}

// Warp per sample: merge `nlist` sorted lists of which the first Kin entries are used;
// list l of sample b starts at in + l*list_stride + b*sample_stride.  Output [B][K].
__global__ void k_merge_topk(const float* __restrict__ in_s, const int* __restrict__ in_i, int nlist,
                             int64_t list_stride, int64_t sample_stride, int Kin, int B, int K,
                             float* __restrict__ out_s, int* __restrict__ out_i) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int b = (int)global_warp(); b < B; b += nw) {
    float ts[kTopkMax]; int ti[kTopkMax];
#pragma unroll
    for (int q = 0; q < kTopkMax; ++q) { ts[q] = -INFINITY; ti[q] = INT_MAX; }
    for (int l = lane; l < nlist; l += 32) {
      const int64_t base = (int64_t)l * list_stride + (int64_t)b * sample_stride;
      for (int q = 0; q < Kin; ++q) topk_insert(ts, ti, in_s[base + q], in_i[base + q]);
    }
    for (int r = 0; r < K; ++r) {
      float bs = ts[0]; int bi = ti[0];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        const float s2 = __shfl_xor_sync(kFull, bs, o); const int i2 = __shfl_xor_sync(kFull, bi, o);
        if (better(s2, i2, bs, bi)) { bs = s2; bi = i2; }
      }
      if (lane == 0) { out_s[(int64_t)b * K + r] = bs; out_i[(int64_t)b * K + r] = bi; }
      if (ti[0] == bi && ts[0] == bs && bi != INT_MAX) {      // the owner pops its head
#pragma unroll
        for (int q = 0; q < kTopkMax - 1; ++q) { ts[q] = ts[q + 1]; ti[q] = ti[q + 1]; }
        ts[kTopkMax - 1] = -INFINITY; ti[kTopkMax - 1] = INT_MAX;
      }
    }
  }
}

// ---------------------------------------------------------------------- precision at K
// Eq. (1): hits[b] = |{q < K : ids[b][q] is a positive of b}|, and
// mean = (1/B) sum_b hits[b] / K (divided by K even with fewer than K positives, R16).
// One CTA; warp w takes samples w, w + 8, ...; lane q < K holds predicted id q and the
// warp walks the sample's positives (CSR) 32 at a time.  The mean is summed in a fixed
// order (per warp over its samples, then over warps), so it is deterministic.
__global__ void __launch_bounds__(256) k_precision_at_k(const int* __restrict__ ids, int B, int K,
                                                        const int* __restrict__ lbl_ptr, const int* __restrict__ lbl_ids,
                                                        int* __restrict__ hits, float* __restrict__ mean) {
  __shared__ float wsum[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float acc = 0.0f;
  for (int b = w; b < B; b += 8) {
    const int id = lane < K ? ids[(int64_t)b * K + lane] : -1;
    bool hit = false;
    for (int p = lbl_ptr[b]; p < lbl_ptr[b + 1]; p += 32) {
      const int n = min(32, lbl_ptr[b + 1] - p);
      const int pv = lane < n ? lbl_ids[p + lane] : -2;
      for (int t = 0; t < n; ++t) hit |= (__shfl_sync(kFull, pv, t) == id);
    }
    const int nh = __popc(__ballot_sync(kFull, hit && lane < K));
    if (lane == 0) {
      if (hits != nullptr) hits[b] = nh;
      acc = __fadd_rn(acc, __fdiv_rn((float)nh, (float)K));
    }
  }
  if (lane == 0) wsum[w] = acc;
  __syncthreads();
  if (threadIdx.x == 0 && mean != nullptr) {
    float t = 0.0f;
    for (int i = 0; i < 8; ++i) t = __fadd_rn(t, wsum[i]);
    *mean = B > 0 ? __fdiv_rn(t, (float)B) : 0.0f;
  }
}

// ---------------------------------------------------------------------- shortlist scoring
// Scores of explicit (sample, label) pairs — the "trivial matrix slicing" of P:1057-1059.
// One thread per pair.  score_one<NG> evaluates exactly the operation sequence the warp
// kernels perform for that pair (row_score_own): per connection group g = s mod 4 two fma
// chains over slots s = 4q + g (q even / odd, slots >= k contribute fma(0, 0, .)), their
// sum P_g, then ((P_0 + P_2) + (P_1 + P_3)) + bias — so the result is bit-identical to the
// forward / predict score of the same pair (IEEE addition is commutative).
template <int NG>
__device__ __forceinline__ float score_one(const float* __restrict__ Wj, const int* __restrict__ ij,
                                           const float* __restrict__ hrow, int k, float bj) {
  float P[4];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    float ca = 0.0f, cb = 0.0f;
#pragma unroll
    for (int q = 0; q < NG; q += 2) {
      const int s0 = 4 * q + g, s1 = 4 * (q + 1) + g;
      const float w0 = s0 < k ? Wj[s0] : 0.0f, h0 = s0 < k ? __ldg(hrow + ij[s0]) : 0.0f;
      ca = __fmaf_rn(w0, h0, ca);
      if (q + 1 < NG) {
        const float w1 = s1 < k ? Wj[s1] : 0.0f, h1 = s1 < k ? __ldg(hrow + ij[s1]) : 0.0f;
        cb = __fmaf_rn(w1, h1, cb);
      }
    }
    P[g] = __fadd_rn(ca, cb);
  }
  return __fadd_rn(__fadd_rn(__fadd_rn(P[0], P[2]), __fadd_rn(P[1], P[3])), bj);
}

// Warp per sample (grid-stride), lanes over its candidate entries.  Entries whose label is
// not in this shard's rows get +0 (shards' outputs sum to the full result); ids outside
// [0, L_global) set kErrLabelRange and get NaN.
template <int NG>
__global__ void __launch_bounds__(256) k_shortlist(const float* __restrict__ W, const int* __restrict__ idx,
                                                   const float* __restrict__ bias, const float* __restrict__ h,
                                                   int64_t m, int k, int64_t L, int64_t row_begin, int64_t L_global,
                                                   int B, const int* __restrict__ cand_ptr,
                                                   const int* __restrict__ cand_ids, float* __restrict__ scores,
                                                   int* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const int nw = (int)(((int64_t)gridDim.x * blockDim.x) >> 5);
  for (int b = (int)global_warp(); b < B; b += nw) {
    const int p0 = cand_ptr[b], p1 = cand_ptr[b + 1];
    const float* hrow = h + (int64_t)b * m;
    for (int p = p0 + lane; p < p1; p += 32) {
      const int gid = cand_ids[p];
      const int64_t j = (int64_t)gid - row_begin;
      float y = 0.0f;
      if (gid < 0 || gid >= L_global) {
        atomicOr(err, kErrLabelRange);
        y = __int_as_float(0x7fc00000);
      } else if (j >= 0 && j < L) {
        y = score_one<NG>(W + j * k, idx + j * k, hrow, k, bias[j]);
      }
      scores[p] = y;
    }
  }
}

}  // namespace ff
