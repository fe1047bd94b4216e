// ff_device.cuh — device helpers of the fixed fan-in hot path (sm_100a).
// Citations: P:n = paper LaTeX line, S:n = SPEC line, Rn = DESIGN.md reading n.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ff {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------- Philox4x32-10
// Counter-based RNG of Salmon et al. (SC'11): 10 rounds of the Philox S-box with
// multipliers 0xD2511F53 / 0xCD9E8D57 and Weyl key increments 0x9E3779B9 / 0xBB67AE85.
// Counter (n, global row, step, domain), key (seed lo, seed hi) (R13).
struct U4 { uint32_t x, y, z, w; };

__device__ __forceinline__ U4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                     uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;   // bump for the next round (unused after the last)
  }
  return {c0, c1, c2, c3};
}

__device__ __forceinline__ uint32_t word_of(const U4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

// Uniform integer in [0, m) by multiply-shift with exact rejection (Lemire 2019):
// returns -1 when the low half falls below 2^32 mod m (the biased region).
__device__ __forceinline__ int lemire_draw(uint32_t u, uint32_t m, uint32_t thr) {
  const uint64_t x = (uint64_t)u * (uint64_t)m;
  return ((uint32_t)x < thr) ? -1 : (int)(x >> 32);
}

enum : uint32_t { kDomInitIdx = 0, kDomInitW = 1, kDomRegrow = 2 };

// ---------------------------------------------------------------- memory ops
// L2 policies: streamed state (W, idx, moments: read once per step) is evict_first so
// the L2-resident hT/dhT (4 MiB each at m = 32768, B = 32) is not displaced.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p;
}
__device__ __forceinline__ float ld_stream(const float* a, uint64_t pol) {
  float v; asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol)); return v;
}
__device__ __forceinline__ int ld_stream_ro(const int* a, uint64_t pol) {
  int v; asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol)); return v;
}
__device__ __forceinline__ void st_stream(float* a, float v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.f32 [%0], %1, %2;" :: "l"(a), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint(float* a, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" :: "l"(a), "f"(v), "l"(pol) : "memory");
}
// Plain (no L2 policy operand) variants for the hot loops: every `.L2::cache_hint` access
// costs two R2UR moves of the policy into a fresh uniform descriptor pair in SASS.
__device__ __forceinline__ float ld_na(const float* a) {
  float v; asm volatile("ld.global.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(a)); return v;
}
__device__ __forceinline__ int ld_na_ro(const int* a) {
  int v; asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(a)); return v;
}
__device__ __forceinline__ void st_na(float* a, float v) {
  asm volatile("st.global.L1::no_allocate.f32 [%0], %1;" :: "l"(a), "f"(v) : "memory");
}
__device__ __forceinline__ float4 ld_line4_plain(const float* a) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a));
  return v;
}
__device__ __forceinline__ void red_add4_plain(float* a, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};"
               :: "l"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
// one 16-B segment of an hT line (4 samples), L2-resident
__device__ __forceinline__ float4 ld_line4(const float* a, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a), "l"(pol));
  return v;
}
// fire-and-forget vector reduction into an L2-resident dhT line (Alg. 2's atomicAdd)
__device__ __forceinline__ void red_add4(float* a, float4 v, uint64_t pol) {
  asm volatile("red.global.add.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
               :: "l"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}

// ---------------------------------------------------------------- packed fp32x2 (sm_100)
// fma.rn.f32x2 / mul.rn.f32x2: two independent IEEE fp32 FMAs/MULs per instruction (FFMA2);
// each half rounds exactly like the scalar op.  A scalar operand broadcast into both halves
// folds into the instruction (no packing moves).
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 r;
  asm("{.reg .b64 a, b, c, d; mov.b64 a, {%2,%3}; mov.b64 b, {%4,%5}; mov.b64 c, {%6,%7};"
      " fma.rn.f32x2 d, a, b, c; mov.b64 {%0,%1}, d;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}
// The same FMA as a volatile asm: volatile asms keep their program order, so FMAs written
// after a batch of (volatile) line loads cannot be hoisted between them by the scheduler —
// otherwise the first FMA's wait on its load stalls the issue of the remaining loads.
__device__ __forceinline__ float2 ffma2_ordered(float2 a, float2 b, float2 c) {
  float2 r;
  asm volatile("{.reg .b64 a, b, c, d; mov.b64 a, {%2,%3}; mov.b64 b, {%4,%5}; mov.b64 c, {%6,%7};"
               " fma.rn.f32x2 d, a, b, c; mov.b64 {%0,%1}, d;}"
               : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 a, b, d; mov.b64 a, {%2,%3}; mov.b64 b, {%4,%5}; mul.rn.f32x2 d, a, b; mov.b64 {%0,%1}, d;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 a, b, d; mov.b64 a, {%2,%3}; mov.b64 b, {%4,%5}; add.rn.f32x2 d, a, b; mov.b64 {%0,%1}, d;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 a, b, d; mov.b64 a, {%2,%3}; mov.b64 b, {%4,%5}; sub.rn.f32x2 d, a, b; mov.b64 {%0,%1}, d;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 lo2(const float4& v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 hi2(const float4& v) { return make_float2(v.z, v.w); }
__device__ __forceinline__ float2 bc2(float s) { return make_float2(s, s); }

// ---------------------------------------------------------------- warp helpers
// This thread's global warp index, broadcast from lane 0 so that ptxas can prove it (and
// every loop bound derived from it) warp-uniform: without that it guards each later
// shuffle with a divergence check (UMOV + BRA.DIV, two extra issues per SHFL).
__device__ __forceinline__ int64_t global_warp() {
  return (int64_t)__shfl_sync(kFull, (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), 0);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// ---------------------------------------------------------------- loss / optimizer
// BCE-with-logits for one score y with target `pos`, in the cancellation-free
// split form (R5): with e = exp(-|y|), sigma(|y|) = 1/(1+e) and sigma(-|y|) = e/(1+e);
// g = s*sigma(y) for t = 0, -s*sigma(-y) for t = 1.  *e_out = e (reused by the loss term).
__device__ __forceinline__ float bce_grad(float y, bool pos, float s, float* e_out) {
  const float e = __expf(-fabsf(y));
  const float r = __fdividef(1.0f, 1.0f + e);
  const float er = e * r;
  const bool nonneg = y >= 0.0f;
  const float sig_y = nonneg ? r : er;       // sigma(y)
  const float sig_my = nonneg ? er : r;      // sigma(-y)
  *e_out = e;
  return pos ? -s * sig_my : s * sig_y;
}
// softplus(y) - t*y = max(y,0) - t*y + log1p(exp(-|y|)); e = exp(-|y|) in (0, 1].
// log1p(e) by __logf(1+e), or its 2-term series below 2^-10 (abs. error < 4e-7 per term).
__device__ __forceinline__ float bce_loss_term(float y, bool pos, float e) {
  const float l1p = e < 0.0009765625f ? e * (1.0f - 0.5f * e) : __logf(1.0f + e);
  return fmaxf(y, 0.0f) - (pos ? y : 0.0f) + l1p;
}

// Squared hinge with t' = +1 for positives, -1 for negatives:
// g = s * (-2 t' max(0, 1 - t' y)) — exactly zero when t' y >= 1 (the sign of 1 - t'y is
// exact in fp32 since t'y is); *lterm = max(0, 1 - t' y)^2.
__device__ __forceinline__ float sqh_grad(float y, bool pos, float s, float* lterm) {
  const float t = pos ? 1.0f : -1.0f;
  const float mg = fmaxf(0.0f, __fsub_rn(1.0f, t * y));
  *lterm = mg * mg;
  return s * (-2.0f * t * mg);
}

struct AdamArgs {
  float lr, beta1, beta2, one_minus_b1, one_minus_b2, rbc1, rbc2, eps;   // rbc = 1/(1 - beta^t)
};
// Adam (Kingma & Ba) with bias correction and eps outside the sqrt (R6):
// m = b1 m + (1-b1) q; v = b2 v + (1-b2) q^2; p -= lr (m/bc1) / (sqrt(v/bc2) + eps).
__device__ __forceinline__ void adam_update(float& p, float& mo, float& ve, float q, const AdamArgs& a) {
  mo = __fadd_rn(__fmul_rn(a.beta1, mo), __fmul_rn(a.one_minus_b1, q));
  ve = __fadd_rn(__fmul_rn(a.beta2, ve), __fmul_rn(a.one_minus_b2, __fmul_rn(q, q)));
  const float mhat = __fmul_rn(mo, a.rbc1);
  const float vhat = __fmul_rn(ve, a.rbc2);
  float sq;                                  // MUFU.SQRT, rel. error ~2^-23 (sqrt(0) = 0)
  asm("sqrt.approx.f32 %0, %1;" : "=f"(sq) : "f"(vhat));
  p = __fsub_rn(p, __fdividef(__fmul_rn(a.lr, mhat), __fadd_rn(sq, a.eps)));
}
// The same update for two parameters with packed fp32x2 ops (each half rounds exactly like
// the scalar op, so the results are bit-identical to two adam_update calls).
__device__ __forceinline__ void adam_update2(float2& p, float2& mo, float2& ve, float2 q, const AdamArgs& a) {
  mo = fadd2(fmul2(bc2(a.beta1), mo), fmul2(bc2(a.one_minus_b1), q));
  ve = fadd2(fmul2(bc2(a.beta2), ve), fmul2(bc2(a.one_minus_b2), fmul2(q, q)));
  const float2 mhat = fmul2(mo, bc2(a.rbc1));
  const float2 vhat = fmul2(ve, bc2(a.rbc2));
  float2 sq;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(sq.x) : "f"(vhat.x));
  asm("sqrt.approx.f32 %0, %1;" : "=f"(sq.y) : "f"(vhat.y));
  const float2 num = fmul2(bc2(a.lr), mhat), den = fadd2(sq, bc2(a.eps));
  p = fsub2(p, make_float2(__fdividef(num.x, den.x), __fdividef(num.y, den.y)));
}

}  // namespace ff
