// Round-1 experiment, NOT compiled: the tcgen05 dense forward with a cp.async.bulk raw ring
// (16-feature stages, kTcRaw deep) and converter warps that transpose + split hi/lo from
// shared memory.  Correct (tools/dense_fwd_check.py) but slower than the register-staged
// kernel in ff_dense.cuh: 29-30 us vs 23.9 us per launch at d = 512, m = 32768 for every
// (raw stages, operand buffers) in {(6,2), (4,3), (3,4)}; 37.6 us at 1 CTA per SM
// (tools/gpu_tcvar.sh).  Per-stage barrier and proxy-fence round trips of the converters
// dominate.  Finding kept from it: generic-proxy reads of a stage must be followed by
// fence.proxy.async before the mbarrier arrive that lets cp.async.bulk refill it; without
// the fence the refill overtook the reads at 2 CTAs per SM (h corrupted, max err 0.1).
// Next step: Wd stored K-major per column tile, TMA with 64-B swizzle so the
// raw tile IS the hi operand (tensor-core truncation) and only lo is computed in place.
// Needs umma_desc_kmajor, tc_mma_tf32, mbar_wait from ff_dense.cuh.
#ifndef FF_TC_RAW
#define FF_TC_RAW 6
#endif
#ifndef FF_TC_OPS
#define FF_TC_OPS 2
#endif
constexpr int kTcThreads = 256, kTcFch = 16;                       // converter threads; features per stage
constexpr int kTcRaw = FF_TC_RAW;                                  // raw (fp32, as in HBM) stages in flight
constexpr int kTcRawA = kTcFch * 128 * 4, kTcRawB = kTcFch * 32 * 4;               // 8 KB, 2 KB
constexpr int kTcAbytes = kTcFch * 128 * 4, kTcBbytes = kTcFch * 32 * 4;           // operand tiles: 8 KB, 2 KB
constexpr int kTcBuf = 2 * kTcAbytes + 2 * kTcBbytes;                              // hi/lo A, hi/lo B: 20 KB
constexpr int kTcNops = FF_TC_OPS;                                                 // operand buffers
constexpr int kTcOps = kTcNops * kTcBuf;
constexpr int kTcRawBytes = kTcRaw * (kTcRawA + kTcRawB);
constexpr int kTcBar = kTcOps + kTcRawBytes;                                       // barriers after the data
#ifndef FF_TC_EXTRA_SMEM
#define FF_TC_EXTRA_SMEM 0
#endif
constexpr int kTcSmem = kTcBar + 8 * (2 * kTcRaw + 2 * kTcNops) + 16 + 1024 + FF_TC_EXTRA_SMEM;   // + TMEM slot + align slack
static_assert(kTcFch == 16, "converter ownership assumes 16-feature stages");

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(mbar) : "memory");
}

__global__ void __launch_bounds__(kTcThreads + 64, 2) k_dense_fwd_tc(const float* __restrict__ Wd, const float* __restrict__ bd,
                                                                 const float* __restrict__ xT, int d, int m, int ldx,
                                                                 int B, float* __restrict__ hd, int cstride, int zero_dh,
                                                                 float* __restrict__ h_out) {
  // warps 0-7 convert, warp 8 issues the MMAs, warp 9 issues the bulk copies.  The 16-feature
  // slices of the Wd tile (16 rows x 512 B) and of xT (16 rows x 128 B, ldx = 32) are
  // contiguous in HBM: one cp.async.bulk each per stage into a kTcRaw-deep raw ring
  // (raw_full: expect_tx by the copy thread; raw_empty: 256 converter arrivals).  The
  // converters read a raw stage (4 strided scalars per 16-B K-major chunk, conflict-free),
  // split hi/lo into one of two operand buffers (op_full: 256 arrivals; op_empty: the MMAs'
  // tcgen05.commit).  No CTA-wide barrier in the stage loop; HBM latency is covered by the
  // raw ring (kTcRaw x 10 KB per CTA, 2 CTAs per SM), not by registers.
  extern __shared__ __align__(16) unsigned char tsm[];
  const uint32_t sbase = ((uint32_t)__cvta_generic_to_shared(tsm) + 1023u) & ~1023u;
  const uint32_t raw0 = sbase + kTcOps;                              // raw stage r: A at raw0 + r*(A+B), B after it
  const uint32_t bar = sbase + kTcBar;
  const uint32_t raw_full0 = bar, raw_empty0 = bar + 8 * kTcRaw;
  const uint32_t op_full0 = bar + 16 * kTcRaw, op_empty0 = op_full0 + 8 * kTcNops, tptr_s = op_empty0 + 8 * kTcNops;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int ct = blockIdx.x * 128;
  const int nst = (d + kTcFch - 1) / kTcFch;
  if (w == 0) {                                                      // TMEM: 32 columns (N = 32 fp32)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" :: "r"(tptr_s) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    for (int r = 0; r < kTcRaw; ++r) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(raw_full0 + 8u * r) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(raw_empty0 + 8u * r), "r"(kTcThreads) : "memory");
    }
    for (int b = 0; b < kTcNops; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(op_full0 + 8u * b), "r"(kTcThreads) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(op_empty0 + 8u * b) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t tmem_d;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(tmem_d) : "r"(tptr_s) : "memory");

  if (w == kTcThreads / 32 + 1) {                                    // ===== bulk-copy issuer
    if (lane == 0) {
      const float* const wt = Wd + (int64_t)blockIdx.x * d * 128;
      for (int st = 0; st < nst; ++st) {
        const int r = st % kTcRaw;
        if (st >= kTcRaw) mbar_wait(raw_empty0 + 8u * r, (uint32_t)((st / kTcRaw - 1) & 1));
        const int f0 = st * kTcFch, rows = min(kTcFch, d - f0);
        const uint32_t ba = (uint32_t)rows * 512u, bb = (uint32_t)rows * 128u;
        const uint32_t dst = raw0 + (uint32_t)r * (kTcRawA + kTcRawB);
        mbar_expect_tx(raw_full0 + 8u * r, ba + bb);
        bulk_g2s(dst, wt + (int64_t)f0 * 128, ba, raw_full0 + 8u * r);
        bulk_g2s(dst + kTcRawA, xT + (int64_t)f0 * ldx, bb, raw_full0 + 8u * r);
      }
    }
  } else if (w == kTcThreads / 32) {                                 // ===== MMA issuer
    if (lane == 0) {
      for (int st = 0; st < nst; ++st) {
        const int b = st % kTcNops;
        const uint32_t buf = sbase + (uint32_t)b * kTcBuf;
        const uint32_t A_hi = buf, A_lo = buf + kTcAbytes, B_hi = buf + 2 * kTcAbytes, B_lo = B_hi + kTcBbytes;
        mbar_wait(op_full0 + 8u * b, (uint32_t)((st / kTcNops) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int nkb = min(kTcFch / 8, (d - st * kTcFch + 7) / 8);
        for (int kb = 0; kb < nkb; ++kb) {
          const uint64_t ah = umma_desc_kmajor(A_hi + kb * 4096, 2048, 128), al = umma_desc_kmajor(A_lo + kb * 4096, 2048, 128);
          const uint64_t bh = umma_desc_kmajor(B_hi + kb * 1024, 512, 128), bl = umma_desc_kmajor(B_lo + kb * 1024, 512, 128);
          tc_mma_tf32(tmem_d, ah, bh, (st > 0 || kb > 0) ? 1u : 0u);
          tc_mma_tf32(tmem_d, ah, bl, 1u);
          tc_mma_tf32(tmem_d, al, bh, 1u);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     :: "r"(op_empty0 + 8u * b) : "memory");
      }
    }
  } else {                                                           // ===== converters
    // A: chunks e = u*256 + tid (u = 0, 1): column c = e & 127, K quad kq = e >> 7 (0..3);
    // B (threads < 128): sample tid & 31, K quad tid >> 5.  K-major core-matrix offsets as
    // in the descriptors: A chunk at kq*2048 + c*16, B chunk at kq*512 + b*16.
    auto split_store = [&](uint32_t hi_addr, uint32_t lo_addr, float4 v) {
      // hi = a with the 13 low mantissa bits cleared (exactly a tf32 value), lo = a - hi exactly;
      // the tensor core truncates lo to tf32 (<= 2^-21 |a|), a_lo.b_lo is dropped (<= 2^-20)
      const uint32_t h0 = __float_as_uint(v.x) & 0xFFFFE000u, h1 = __float_as_uint(v.y) & 0xFFFFE000u;
      const uint32_t h2 = __float_as_uint(v.z) & 0xFFFFE000u, h3 = __float_as_uint(v.w) & 0xFFFFE000u;
      const float l0 = v.x - __uint_as_float(h0), l1 = v.y - __uint_as_float(h1);
      const float l2 = v.z - __uint_as_float(h2), l3 = v.w - __uint_as_float(h3);
      asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(hi_addr), "r"(h0), "r"(h1), "r"(h2), "r"(h3) : "memory");
      asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" :: "r"(lo_addr), "f"(l0), "f"(l1), "f"(l2), "f"(l3) : "memory");
    };
    auto lds = [](uint32_t a) { float v; asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory"); return v; };
    const int c = tid & 127, kqa = tid >> 7;                         // A chunk u: K quad kqa + 2u
    const int bs = tid & 31, kqb = tid >> 5;                         // B chunk (tid < 128)
    for (int st = 0; st < nst; ++st) {
      const int r = st % kTcRaw, b = st % kTcNops;
      const int rows = min(kTcFch, d - st * kTcFch);
      const uint32_t ra = raw0 + (uint32_t)r * (kTcRawA + kTcRawB), rb = ra + kTcRawA;
      mbar_wait(raw_full0 + 8u * r, (uint32_t)((st / kTcRaw) & 1));
      float4 va[2], vb = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int f = 4 * (kqa + 2 * u);
        float t[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) t[i] = f + i < rows ? lds(ra + (uint32_t)(((f + i) * 128 + c) * 4)) : 0.0f;
        va[u] = make_float4(t[0], t[1], t[2], t[3]);
      }
      if (tid < 128) {
        const int f = 4 * kqb;
        float t[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) t[i] = f + i < rows ? lds(rb + (uint32_t)(((f + i) * 32 + bs) * 4)) : 0.0f;
        vb = make_float4(t[0], t[1], t[2], t[3]);
      }
      // the raw stage is refilled by the async proxy (cp.async.bulk) after these generic-proxy
      // reads: without this proxy fence the refill can overtake them (measured: corrupted h at
      // 2 CTAs per SM)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(raw_empty0 + 8u * r);                              // this raw stage may be refilled
      if (st >= kTcNops) mbar_wait(op_empty0 + 8u * b, (uint32_t)((st / kTcNops - 1) & 1));   // its MMAs are done
      const uint32_t buf = sbase + (uint32_t)b * kTcBuf;
      const uint32_t A_hi = buf, A_lo = buf + kTcAbytes, B_hi = buf + 2 * kTcAbytes, B_lo = B_hi + kTcBbytes;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const uint32_t off = (uint32_t)((kqa + 2 * u) * 2048 + c * 16);
        split_store(A_hi + off, A_lo + off, va[u]);
      }
      if (tid < 128) {
        const uint32_t off = (uint32_t)(kqb * 512 + bs * 16);
        split_store(B_hi + off, B_lo + off, vb);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic-proxy stores -> tensor core
      mbar_arrive(op_full0 + 8u * b);
    }
  }
  mbar_wait(op_empty0 + 8u * ((nst - 1) % kTcNops), (uint32_t)(((nst - 1) / kTcNops) & 1));   // all MMAs done
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (w < 4) {
    uint32_t v[32];
    const uint32_t taddr = tmem_d + ((uint32_t)(32 * w) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                   "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                   "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int c = ct + 32 * w + lane;                              // TMEM lane = column
    if (c < m) {
      const float bj = bd[c];
      float h[32];
#pragma unroll
      for (int s2 = 0; s2 < 32; ++s2) h[s2] = s2 < B ? fmaxf(__uint_as_float(v[s2]) + bj, 0.0f) : 0.0f;
      float* line = hd + (int64_t)c * cstride;
#pragma unroll
      for (int s4 = 0; s4 < 32; s4 += 4) {
        *reinterpret_cast<float4*>(line + s4) = make_float4(h[s4], h[s4 + 1], h[s4 + 2], h[s4 + 3]);
        if (zero_dh) *reinterpret_cast<float4*>(line + 32 + s4) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (h_out != nullptr) {
#pragma unroll
        for (int s2 = 0; s2 < 32; ++s2)
          if (s2 < B) h_out[(int64_t)s2 * m + c] = h[s2];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" :: "r"(tmem_d) : "memory");
}

