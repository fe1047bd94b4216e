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
  int64_t L; int k; int B; int nb; int cstride;   // cstride = 64*nb floats per column
  float grad_scale;
  float* y_out;               // forward: y[B][L]
  const float* y_in;          // backward: y[B][L]
  float* loss;                // device scalar (zeroed by prep) or nullptr
  int* err;
  AdamArgs adam;
  uint32_t check_finite;
};

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

// Broadcast each connection's weight and hd column offset to the lanes that gather it:
// lane (gq, bq) handles connections s = 4q + gq, q < NG.
template <int NG>
__device__ __forceinline__ void row_spread(float w, int c, int cstride, int gq, float (&ws)[NG], uint32_t (&cs)[NG]) {
#pragma unroll
  for (int q = 0; q < NG; ++q) {
    ws[q] = __shfl_sync(kFull, w, 4 * q + gq);
    cs[q] = (uint32_t)__shfl_sync(kFull, c, 4 * q + gq) * (uint32_t)cstride;
  }
}

// Gather the 16-B segment [lo, lo+4) of each connection's 128-B h line of chunk `base`.
template <int NG>
__device__ __forceinline__ void row_gather(const float* hb, const uint32_t (&cs)[NG], int k, int gq,
                                           uint64_t pol, float4 (&hv)[NG]) {
#pragma unroll
  for (int q = 0; q < NG; ++q) {
    hv[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (4 * q + gq < k) hv[q] = ld_line4(hb + cs[q], pol);
  }
}

// y for this lane's own sample lo + gq: per-lane FMAs over its connections, then a
// reduce-scatter over the four connection groups (xor 16, xor 8), + bias.
template <int NG>
__device__ __forceinline__ float row_score_own(const float (&ws)[NG], const float4 (&hv)[NG], int gq, float bj) {
  float4 yp = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int q = 0; q < NG; ++q) {
    yp.x = fmaf(ws[q], hv[q].x, yp.x); yp.y = fmaf(ws[q], hv[q].y, yp.y);
    yp.z = fmaf(ws[q], hv[q].z, yp.z); yp.w = fmaf(ws[q], hv[q].w, yp.w);
  }
  const bool hi = gq & 2, odd = gq & 1;
  const float k0 = hi ? yp.z : yp.x, k1 = hi ? yp.w : yp.y;
  const float s0 = hi ? yp.x : yp.z, s1 = hi ? yp.y : yp.w;
  const float a0 = k0 + __shfl_xor_sync(kFull, s0, 16);
  const float a1 = k1 + __shfl_xor_sync(kFull, s1, 16);
  const float keep = odd ? a1 : a0, send = odd ? a0 : a1;
  return (keep + __shfl_xor_sync(kFull, send, 8)) + bj;
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

// The row kernel: forward (Alg. 1) for MODE forward; BCE gradient,
// Alg. 3 weight gradient, bias gradient and Alg. 2 input-gradient scatter
// for MODE backward; all of those plus Adam for MODE train — the
// fused step, in which y, g and dW live only in registers.
// Work split: a warp owns blocks of 32 consecutive label rows (persistent, strided over
// blocks) and walks their rows one at a time, prefetching the next row's state.  Per-label
// scalars (bias, its moments, the positive mask) are one coalesced vector per block
// (lane i <-> row i) and the bias Adam update runs once per block, vectorized.
template <int MODE, bool STORE_GRADS, int NG>
__global__ void __launch_bounds__(kRowThreads, kRowMinBlocks) k_rows(RowArgs a) {
  const int lane = threadIdx.x & 31, gq = lane >> 3, bq = lane & 7;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t pol_s = policy_evict_first(), pol_l = policy_evict_last();
  const int k = a.k, cstride = a.cstride, nb = a.nb, B = a.B;
  const int64_t L = a.L, nblk = (L + 31) >> 5;
  const bool act = lane < k;
  float loss_acc = 0.0f;

  float w_n = 0.f, mw_n = 0.f, vw_n = 0.f;
  int c_n = 0;
  auto prefetch_row = [&](int64_t jj) {
    const int64_t row = jj * k;
    if (act) {
      w_n = ld_stream(a.W + row + lane, pol_s);
      c_n = ld_stream_ro(a.idx + row + lane, pol_s);
      if (MODE == kModeTrain) { mw_n = ld_stream(a.mW + row + lane, pol_s); vw_n = ld_stream(a.vW + row + lane, pol_s); }
    }
  };
  int64_t blk = (((int64_t)blockIdx.x * blockDim.x) + threadIdx.x) >> 5;
  if (blk < nblk) prefetch_row(blk * 32);

  for (; blk < nblk; blk += nw) {
    const int64_t j0 = blk * 32;
    const int nl = (int)min((int64_t)32, L - j0);
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
      float w = w_n, mw = mw_n, vw = vw_n;
      const int c = c_n;
      if (i + 1 < nl) prefetch_row(j + 1);
      else if (blk + nw < nblk) prefetch_row((blk + nw) * 32);
      const int64_t row = j * k;
      const float bj = __shfl_sync(kFull, bias_v, i);
      uint32_t pm = __shfl_sync(kFull, pm_v, i);

      float ws[NG]; uint32_t cs[NG];
      row_spread<NG>(w, c, cstride, gq, ws, cs);
      float dwp[NG];
#pragma unroll
      for (int q = 0; q < NG; ++q) dwp[q] = 0.0f;
      float dbp = 0.0f;

      for (int q2 = 0; q2 < nb; ++q2) {
        const int lo = q2 * 32 + 4 * bq;             // this lane's 4-sample segment
        const int b = lo + gq;                        // this lane's own sample
        float* hb = a.hd + q2 * 64 + 4 * bq;          // h segment; its dh segment is +32 floats
        float4 hv[NG];
        row_gather<NG>(hb, cs, k, gq, pol_l, hv);
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
        float e;
        float g = bce_grad(y, pos, a.grad_scale, &e);
        if (b >= B) g = 0.0f;
        if (a.loss != nullptr && b < B) loss_acc += bce_loss_term(y, pos, e);
        if (a.check_finite && __any_sync(kFull, b < B && !isfinite(y)) && lane == 0) atomicOr(a.err, kErrNonFinite);
        dbp += g;
        float4 g4;
        g4.x = __shfl_sync(kFull, g, (0 << 3) | bq);
        g4.y = __shfl_sync(kFull, g, (1 << 3) | bq);
        g4.z = __shfl_sync(kFull, g, (2 << 3) | bq);
        g4.w = __shfl_sync(kFull, g, (3 << 3) | bq);
#pragma unroll
        for (int q = 0; q < NG; ++q) {
          float t = dwp[q];
          t = fmaf(g4.x, hv[q].x, t); t = fmaf(g4.y, hv[q].y, t);
          t = fmaf(g4.z, hv[q].z, t); t = fmaf(g4.w, hv[q].w, t);
          dwp[q] = t;
        }
        // Alg. 2 with the pre-update weights: dh[b][idx[j][i]] += W[j][i] g[b][j]
#pragma unroll
        for (int q = 0; q < NG; ++q) {
          if (4 * q + gq < k)
            red_add4(hb + cs[q] + 32, make_float4(ws[q] * g4.x, ws[q] * g4.y, ws[q] * g4.z, ws[q] * g4.w), pol_l);
        }
      }
      if (MODE == kModeForward) continue;

      const float gW = row_dw_slot<NG>(dwp, lane);
      const float db = warp_sum(dbp);
      if (lane == i) db_v = db;
      if (MODE == kModeBackward || STORE_GRADS) {
        if (act) a.dW[row + lane] = gW;
      }
      if (MODE == kModeTrain && act) {
        adam_update(w, mw, vw, gW, a.adam);
        st_stream(a.W + row + lane, w, pol_s);
        st_stream(a.mW + row + lane, mw, pol_s);
        st_stream(a.vW + row + lane, vw, pol_s);
      }
    }
    if (MODE == kModeForward) continue;
    if (lv) {
      if (pm_v != 0u) a.posmask[j0 + lane] = 0u;      // self-clearing mask (chunk 0)
      if (MODE == kModeBackward || STORE_GRADS) a.db[j0 + lane] = db_v;
      if (MODE == kModeTrain) {                        // bias Adam, one row per lane
        adam_update(bias_v, mb_v, vb_v, db_v, a.adam);
        st_stream(a.bias + j0 + lane, bias_v, pol_s);
        st_stream(a.mb + j0 + lane, mb_v, pol_s);
        st_stream(a.vb + j0 + lane, vb_v, pol_s);
      }
    }
  }
  if (MODE != kModeForward && a.loss != nullptr) block_atomic_add(loss_acc * a.grad_scale, a.loss);
}

// ------------------------------------------------------------------------------ prep
// hd[c][q2][r] = h[q2*32 + r][c] (0 for samples >= B), hd[c][q2][32 + r] = 0 (dh
// accumulator), positives -> posmask bits, *loss = 0.  Grid: ceil(m/32) blocks of 32x8.
__global__ void k_prep(const float* __restrict__ h, int B, int m, int nb, float* __restrict__ hd, int zero_dh,
                       const int* __restrict__ lbl_ptr, const int* __restrict__ lbl_ids,
                       uint32_t* __restrict__ posmask, int64_t L_local, int64_t row_begin,
                       int64_t L_global, float* loss, int* err) {
  __shared__ float t[32][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int c0 = blockIdx.x * 32;
  const int cstride = 64 * nb;
  if (h != nullptr) {
    for (int q2 = 0; q2 < nb; ++q2) {
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

// dh[b][c] = hd[c][b/32][32 + b%32] for b < B.  Grid ceil(m/32) x nb, 32x8 threads.
__global__ void k_dh_out(const float* __restrict__ hd, int B, int m, int nb, float* __restrict__ dh) {
  __shared__ float t[32][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int c0 = blockIdx.x * 32, q2 = blockIdx.y;
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
// Standalone Adam over W (with dW) and bias (with db).
__global__ void k_adam(float* __restrict__ W, float* __restrict__ mW, float* __restrict__ vW,
                       const float* __restrict__ dW, int64_t n, float* __restrict__ bias,
                       float* __restrict__ mb, float* __restrict__ vb, const float* __restrict__ db,
                       int64_t L, AdamArgs a) {
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
__global__ void k_init(float* __restrict__ W, int* __restrict__ idx, float* __restrict__ bias,
                       float* __restrict__ mW, float* __restrict__ vW, float* __restrict__ mb,
                       float* __restrict__ vb, int64_t L, int64_t row_begin, int m, int k,
                       uint32_t key0, uint32_t key1, float scale) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t thr = (uint32_t)(0x100000000ull % (uint64_t)m);
  for (int64_t j = (((int64_t)blockIdx.x * blockDim.x) + threadIdx.x) >> 5; j < L; j += nw) {
    const uint32_t grow = (uint32_t)(row_begin + j);
    int mine = -1, count = 0;
    for (uint32_t n = 0; count < k; ++n) {
      const U4 v = philox(n, grow, 0u, kDomInitIdx, key0, key1);
#pragma unroll
      for (int wi = 0; wi < 4; ++wi) {
        if (count < k) {
          const int cand = lemire_draw(word_of(v, wi), (uint32_t)m, thr);
          if (cand >= 0 && __ballot_sync(kFull, lane < count && mine == cand) == 0u) {
            if (lane == count) mine = cand;
            ++count;
          }
        }
      }
    }
    if (lane < k) {
      const U4 v = philox((uint32_t)(lane >> 2), grow, 0u, kDomInitW, key0, key1);
      const uint32_t u = word_of(v, lane & 3);
      const float unit = __fmul_rn((float)(u >> 8), 1.0f / 16777216.0f);
      const float centered = __fsub_rn(__fmul_rn(2.0f, unit), 1.0f);
      const int64_t e = j * k + lane;
      idx[e] = mine;
      W[e] = __fmul_rn(scale, centered);
      mW[e] = 0.0f; vW[e] = 0.0f;
    }
    if (lane == 0) { bias[j] = 0.0f; mb[j] = 0.0f; vb[j] = 0.0f; }
  }
}

// ---------------------------------------------------------------------- redistribution
// SET prune/regrow per row (R8-R14).  Warp per row, lane = slot:
// rank of (|W| bits, slot) among the row; the p lowest are pruned; the regrow stream
// (domain 2, counter (n, global row, step, 2)) yields candidates uniform on [0,m) that
// are accepted when not in the pre-call row set and not yet accepted; the q-th accepted
// index goes to the q-th pruned slot in ascending slot order; W = mW = vW = 0 there.
__global__ void k_redistribute(float* __restrict__ W, int* __restrict__ idx, float* __restrict__ mW,
                               float* __restrict__ vW, int64_t L, int64_t row_begin, int m, int k,
                               int p, uint32_t step, uint32_t key0, uint32_t key1) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t thr = (uint32_t)(0x100000000ull % (uint64_t)m);
  for (int64_t j = (((int64_t)blockIdx.x * blockDim.x) + threadIdx.x) >> 5; j < L; j += nw) {
    const int64_t e = j * k + lane;
    const bool act = lane < k;
    const float w = act ? W[e] : 0.0f;
    const int c = act ? idx[e] : -1;
    const uint32_t key = act ? (__float_as_uint(w) & 0x7fffffffu) : 0xffffffffu;
    int rank = 0;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const uint32_t kq = __shfl_sync(kFull, key, q);
      rank += (kq < key || (kq == key && q < lane)) ? 1 : 0;
    }
    const bool pruned = act && rank < p;
    const uint32_t pmask = __ballot_sync(kFull, pruned);
    const uint32_t grow = (uint32_t)(row_begin + j);
    int acc = -1, na = 0;
    for (uint32_t n = 0; na < p; ++n) {
      const U4 v = philox(n, grow, step, kDomRegrow, key0, key1);
#pragma unroll
      for (int wi = 0; wi < 4; ++wi) {
        if (na < p) {
          const int cand = lemire_draw(word_of(v, wi), (uint32_t)m, thr);
          if (cand >= 0) {
            const bool taken = __ballot_sync(kFull, (act && c == cand) || (lane < na && acc == cand)) != 0u;
            if (!taken) {
              if (lane == na) acc = cand;
              ++na;
            }
          }
        }
      }
    }
    const int order = __popc(pmask & ((1u << lane) - 1u));
    const int newc = __shfl_sync(kFull, acc, order & 31);
    if (pruned) { idx[e] = newc; W[e] = 0.0f; mW[e] = 0.0f; vW[e] = 0.0f; }
  }
}

// Validation for set_params: idx in [0, m), distinct within each row.
__global__ void k_validate_idx(const int* __restrict__ idx, int64_t L, int m, int k, int* err) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = (((int64_t)blockIdx.x * blockDim.x) + threadIdx.x) >> 5; j < L; j += nw) {
    const bool act = lane < k;
    const int c = act ? idx[j * k + lane] : -1 - lane;
    if (act && (c < 0 || c >= m)) atomicOr(err, kErrIdxRange);
    bool dup = false;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int cq = __shfl_sync(kFull, c, q);
      dup |= act && q != lane && q < k && cq == c;
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

// Fused forward + per-lane running top-K (y is never written).  For each 32-sample chunk
// q2 every lane owns sample q2*32 + 4*bq + gq; a block merges its warps' lists and writes
// candidates cand[blk][ldh][kTopkMax].
template <int NG>
__global__ void __launch_bounds__(kRowThreads) k_predict(const float* __restrict__ W, const int* __restrict__ idx,
                                                         const float* __restrict__ bias, const float* __restrict__ hd,
                                                         int64_t L, int k, int B, int nb, int64_t row_begin,
                                                         float* __restrict__ cand_s, int* __restrict__ cand_i) {
  __shared__ float ss[kRowThreads / 32][32][kTopkMax];
  __shared__ int si[kRowThreads / 32][32][kTopkMax];
  const int lane = threadIdx.x & 31, gq = lane >> 3, bq = lane & 7, wid = threadIdx.x >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t pol_s = policy_evict_first(), pol_l = policy_evict_last();
  const bool act = lane < k;
  for (int q2 = 0; q2 < nb; ++q2) {
    const int lo = q2 * 32 + 4 * bq;
    const int b = lo + gq;
    const int cstride = 64 * nb;
    const float* hb = hd + q2 * 64 + 4 * bq;
    float ts[kTopkMax]; int ti[kTopkMax];
#pragma unroll
    for (int q = 0; q < kTopkMax; ++q) { ts[q] = -INFINITY; ti[q] = INT_MAX; }
    int64_t j = (((int64_t)blockIdx.x * blockDim.x) + threadIdx.x) >> 5;
    float w_n = 0.f, bj_n = 0.f; int c_n = 0;
    if (j < L) {
      if (act) { w_n = ld_stream(W + j * k + lane, pol_s); c_n = ld_stream_ro(idx + j * k + lane, pol_s); }
      bj_n = ld_stream(bias + j, pol_s);
    }
    for (; j < L; j += nw) {
      const float w = w_n, bj = bj_n; const int c = c_n;
      const int64_t jn = j + nw;
      if (jn < L) {
        if (act) { w_n = ld_stream(W + jn * k + lane, pol_s); c_n = ld_stream_ro(idx + jn * k + lane, pol_s); }
        bj_n = ld_stream(bias + jn, pol_s);
      }
      float ws[NG]; uint32_t cs[NG]; float4 hv[NG];
      row_spread<NG>(w, c, cstride, gq, ws, cs);
      row_gather<NG>(hb, cs, k, gq, pol_l, hv);
      const float y = row_score_own<NG>(ws, hv, gq, bj);
      if (b < B) topk_insert(ts, ti, y, (int)(row_begin + j));
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

// Warp per sample: merge `nlist` sorted lists of which the first Kin entries are used;
// list l of sample b starts at in + l*list_stride + b*sample_stride.  Output [B][K].
__global__ void k_merge_topk(const float* __restrict__ in_s, const int* __restrict__ in_i, int nlist,
                             int64_t list_stride, int64_t sample_stride, int Kin, int B, int K,
                             float* __restrict__ out_s, int* __restrict__ out_i) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < B; b += nw) {
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

}  // namespace ff
