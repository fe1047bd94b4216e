// fixedfanin.cu — host side of the C ABI declared in include/fixedfanin.h: argument
// validation, workspace carving, kernel launches.  No device memory is allocated here
// (the caller owns the workspace) and no call synchronizes except set/get_params/check.
#include "fixedfanin.h"
#include "ff_kernels.cuh"
#include "ff_dense.cuh"
#include <cudaTypedefs.h>

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

using namespace ff;

namespace {

thread_local std::string g_err;
thread_local int32_t g_launches = 0;

ff_status fail(ff_status s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
ff_status fail(ff_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define FF_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) return fail(FF_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

#define FF_LAUNCHED()                                                                   \
  do {                                                                                  \
    ++g_launches;                                                                       \
    cudaError_t e_ = cudaGetLastError();                                                \
    if (e_ != cudaSuccess) return fail(FF_ERR_CUDA, "launch: %s", cudaGetErrorString(e_)); \
  } while (0)

constexpr size_t kAlign = 256;
constexpr int kMaxCandBlocks = 1024;    // predict grid cap (candidate buffer rows)
#ifndef FF_PRED_REG
#define FF_PRED_REG 1                    // B <= 96 predict: 1 = register gathers (k_predict_reg), 0 = cp.async ring
#endif
constexpr int kMaxWideWarps = 4096;     // wide predict: warps with a top-K list in the scratch
constexpr int kPredRingMaxLines = 3;    // predict: B <= 96 runs the ring kernel per 32-sample line

size_t up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct Layout {   // byte offsets into the workspace
  size_t W, idx, mW, vW, dW, bias, mb, vb, db, posmask, hd, cand_s, cand_i, pthr, wl_s, wl_i,
      h_stage, lbl_stage, dh_stage, scalars,
      ent, sort_keys2, gT, col_ptr, sort_keys, sort_tmp, sort_tmp_bytes,   // CSC mode only
      total;
};

int nb_of(int B) { return (B + 31) / 32; }

// CSC mode: one record per label row of a tile, rs floats: the row's gradient line per
// 32-sample chunk, then its pre-update weights (ceil(k/32) lines).
int csc_rec_stride(int max_batch, int k) { return 32 * nb_of(max_batch) + 32 * ((k + 31) / 32); }
// CSC mode label tile: the records of one tile (tile_rows * 4 rs B) stay L2-resident
// between the row launch that writes them and the column launch that gathers them.
#ifndef FF_CSC_TILE_MB
#define FF_CSC_TILE_MB 64
#endif
constexpr size_t kCscTileBytes = size_t(FF_CSC_TILE_MB) << 20;
size_t csc_tile_cap(const ff_config& c) {
  const size_t cap = kCscTileBytes / (4 * (size_t)csc_rec_stride(c.max_batch, c.k)) / 32 * 32;
  return std::max<size_t>(std::min<size_t>(cap, ((size_t)c.L_local + 31) / 32 * 32), 32);
}

Layout layout_of(const ff_config& c) {
  Layout o{};
  const size_t Lk = (size_t)c.L_local * (size_t)c.k, L = (size_t)c.L_local;
  const size_t nbm = (size_t)nb_of(c.max_batch), ldh = 32 * nbm, m = (size_t)c.m;
  const size_t nnz = c.max_nnz > 0 ? (size_t)c.max_nnz : 64 * (size_t)c.max_batch;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t r = off; off += up(bytes); return r; };
  o.W = take(4 * Lk); o.idx = take(4 * Lk); o.mW = take(4 * Lk); o.vW = take(4 * Lk); o.dW = take(4 * Lk);
  o.bias = take(4 * L); o.mb = take(4 * L); o.vb = take(4 * L); o.db = take(4 * L);
  o.posmask = take(4 * L * nbm);
  o.hd = take(8 * m * ldh);         // [m][nb][h 32 | dh 32]
  o.cand_s = take(4 * (size_t)kMaxCandBlocks * ldh * kTopkMax);
  o.cand_i = take(4 * (size_t)kMaxCandBlocks * ldh * kTopkMax);
  o.pthr = take(4 * ldh);                                            // predict ring: shared per-sample thresholds
  if (c.max_batch > 32 && c.k == 32) {                               // wide predict: per-warp top-K lists
    o.wl_s = take(4 * (size_t)kMaxWideWarps * kPredWListFloats);
    o.wl_i = take(4 * (size_t)kMaxWideWarps * kPredWListFloats);
  }
  o.h_stage = take(2 * 4 * (size_t)c.max_batch * m);                 // double-buffered (host entry point)
  o.lbl_stage = take(2 * 4 * ((size_t)c.max_batch + 1 + nnz));
  o.dh_stage = take(4 * (size_t)c.max_batch * m);
  o.scalars = take(kAlign);       // [0] int err, [1] float loss
  if (c.dh_mode != FF_DH_ATOMIC) {          // CSC and hybrid
    o.ent = take(4 * Lk); o.sort_keys2 = take(4 * Lk); o.sort_keys = take(4 * Lk);
    // tiles are >= cap/2 rows (create rounds the cap down to whole row-kernel waves, or keeps it)
    const size_t lt = csc_tile_cap(c), ntile = (2 * L + lt - 1) / lt + 1;
    o.gT = take(4 * lt * (size_t)csc_rec_stride(c.max_batch, c.k));      // records of one label tile
    o.col_ptr = take(4 * (std::max<size_t>(ntile, 1) * m + 1));
    o.sort_tmp_bytes = (size_t(8) << 20) + 2 * Lk;
    o.sort_tmp = take(o.sort_tmp_bytes);
  }
  o.total = off;
  return o;
}

ff_status validate(const ff_config* c) {
  if (!c) return fail(FF_ERR_ARG, "cfg is NULL");
  if (c->L_global < 1 || c->L_global >= (int64_t(1) << 31))
    return fail(FF_ERR_CONFIG, "L_global=%lld outside [1, 2^31)", (long long)c->L_global);
  if (c->row_begin < 0 || c->L_local < 0 || c->row_begin + c->L_local > c->L_global)
    return fail(FF_ERR_CONFIG, "shard rows [%lld, %lld) outside [0, L_global=%lld)", (long long)c->row_begin,
                (long long)(c->row_begin + c->L_local), (long long)c->L_global);
  if (c->m < 1) return fail(FF_ERR_CONFIG, "m=%d < 1", c->m);
  if (c->k < 1 || c->k > FF_MAX_FANIN || c->k > c->m)
    return fail(FF_ERR_CONFIG, "k=%d outside [1, min(m=%d, %d)]", c->k, c->m, FF_MAX_FANIN);
  if (c->max_batch < 1 || c->max_batch > FF_MAX_BATCH)
    return fail(FF_ERR_CONFIG, "max_batch=%d outside [1, %d]", c->max_batch, FF_MAX_BATCH);
  if (c->max_topk < 1 || c->max_topk > FF_MAX_TOPK)
    return fail(FF_ERR_CONFIG, "max_topk=%d outside [1, %d]", c->max_topk, FF_MAX_TOPK);
  if (c->max_nnz < 0) return fail(FF_ERR_CONFIG, "max_nnz < 0");
  if (c->dh_mode != FF_DH_ATOMIC && c->dh_mode != FF_DH_CSC && c->dh_mode != FF_DH_HYBRID)
    return fail(FF_ERR_CONFIG, "dh_mode=%d is not FF_DH_ATOMIC, FF_DH_CSC or FF_DH_HYBRID", c->dh_mode);
  if (!(c->hybrid_frac >= 0.0f && c->hybrid_frac <= 1.0f)) return fail(FF_ERR_CONFIG, "hybrid_frac outside [0, 1]");
  // the row kernels address W / idx / moments (and the CSC entries) with 32-bit connection
  // offsets j*k + i: every mode needs L_local*k < 2^31 (60 GB of state per shard at the limit)
  if (c->L_local * (int64_t)c->k >= (int64_t(1) << 31))
    return fail(FF_ERR_CONFIG, "L_local*k = %lld connections per shard >= 2^31 (shard the labels further)",
                (long long)(c->L_local * (int64_t)c->k));
  if (c->prune_frac < 0.0f || c->prune_frac >= 1.0f) return fail(FF_ERR_CONFIG, "prune_frac outside [0, 1)");
  if (c->loss != FF_LOSS_BCE && c->loss != FF_LOSS_SQH) return fail(FF_ERR_CONFIG, "loss=%d unknown", c->loss);
  if (c->beta1 < 0.0f || c->beta1 >= 1.0f || c->beta2 < 0.0f || c->beta2 >= 1.0f || c->eps < 0.0f)
    return fail(FF_ERR_CONFIG, "Adam hyper-parameters out of range");
  return FF_OK;
}

ff_config with_defaults(const ff_config& in) {
  ff_config c = in;
  if (c.beta1 == 0.0f) c.beta1 = 0.9f;
  if (c.beta2 == 0.0f) c.beta2 = 0.999f;
  if (c.eps == 0.0f) c.eps = 1e-8f;
  if (c.prune_frac == 0.0f) c.prune_frac = 0.1f;
  if (c.init_scale == 0.0f) c.init_scale = (float)(1.0 / std::sqrt((double)c.k));
  if (c.max_nnz == 0) c.max_nnz = 64 * c.max_batch;
  if (c.hybrid_frac == 0.0f) c.hybrid_frac = 0.5f;
  return c;
}

}  // namespace

struct ff_layer {
  ff_config cfg;
  Layout lay;
  char* ws;
  float *W, *mW, *vW, *dW, *bias, *mb, *vb, *db, *hd, *cand_s, *h_stage, *dh_stage, *wl_s;
  int *idx, *cand_i, *pthr, *wl_i, *lbl_stage, *err;
  int *ent, *col_ptr;               // CSC mode
  float* gT;
  int rs;                           // CSC mode: record stride (floats)
  int *sort_keys, *sort_keys2;
  void* sort_tmp;
  bool csc;                         // CSC or hybrid dh
  uint32_t split;                   // hybrid: columns [0, split) by red, [split, m) by the CSC pull; else 0
  int grid_csc;
  int64_t tile_rows;                // CSC mode: labels per tile (multiple of 32)
  int ntiles;
  float* loss_scratch;
  int64_t* t_dev;          // the authoritative Adam step counter (device; advanced by k_prep / k_step_t)
  float* rbc_dev;          // [2] bias corrections of the current step
  uint32_t* posmask;
  int64_t t;
  bool grads_valid;
  int grid_train, grid_fwd, grid_bwd, grid_pred, grid_rows, grid_ring, grid_pred_ring, grid_pred_wide, grid_pred_reg;
  int nsm;
  std::vector<cudaEvent_t> prof_ev;   // pairs (before, after) of the fused row kernel
  // host entry point: H2D copies on a library stream into one of two staging slots, so the
  // next step's copy overlaps this step's kernels
  cudaStream_t copy_st = nullptr;
  cudaEvent_t ev_ready[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};
  int stage_slot = 0;
  int prof_used = 0;
  bool prof_paused = false;
};

namespace {

int ring_mode(const ff_layer* l) {
  return !l->csc ? (l->cfg.loss == FF_LOSS_SQH ? 3 : 0) : l->split > 0 ? 2 : 1;
}

template <typename T>
T* at(char* base, size_t off) { return reinterpret_cast<T*>(base + off); }

// the dense layer's step counter, advanced by k_prep of a whole-architecture step
struct DenseT { int64_t* t; float* rbc; float beta1, beta2; };

#ifndef FF_STEP_PDL
#define FF_STEP_PDL 1            // launch the step's kernels as programmatic dependents (pdl_begin() in each)
#endif
// launch configuration with programmatic stream serialization: the kernel may be scheduled
// while its predecessor drains; it waits in pdl_begin() (griddepcontrol.wait) before touching
// any data
struct PdlCfg {
  cudaLaunchConfig_t c;
  cudaLaunchAttribute at[1];
  PdlCfg(dim3 g, dim3 b, size_t smem, cudaStream_t st) {
    c = {};
    c.gridDim = g; c.blockDim = b; c.dynamicSmemBytes = smem; c.stream = st;
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = FF_STEP_PDL;
    c.attrs = at; c.numAttrs = 1;
  }
};

ff_status launch_prep(ff_layer* l, const float* h, int B, bool zero_dh, const int* lbl_ptr,
                      const int* lbl_ids, float* loss, cudaStream_t st, bool step_t = false,
                      const DenseT* dt = nullptr) {
  const int nb = nb_of(B);
  dim3 grid((l->cfg.m + 31) / 32), block(32, 8);
  const bool vec = (l->cfg.m & 3) == 0 && (reinterpret_cast<uintptr_t>(h) & 15) == 0;
  PdlCfg pc(grid, block, 0, st);
  int zd = zero_dh ? 1 : 0;
  FF_CUDA(cudaLaunchKernelEx(&pc.c, vec ? k_prep<true> : k_prep<false>, h, B, l->cfg.m, nb, l->hd, zd, lbl_ptr, lbl_ids,
                             l->posmask, l->cfg.L_local, l->cfg.row_begin, l->cfg.L_global, loss, l->err,
                             step_t ? l->t_dev : (int64_t*)nullptr, l->rbc_dev, l->cfg.beta1, l->cfg.beta2,
                             dt ? dt->t : (int64_t*)nullptr, dt ? dt->rbc : (float*)nullptr, dt ? dt->beta1 : 0.0f,
                             dt ? dt->beta2 : 0.0f));
  ++g_launches;
  return FF_OK;
}

ff_status launch_dh_out(ff_layer* l, int B, float* dh, cudaStream_t st) {
  const int nb = nb_of(B);
  dim3 grid((l->cfg.m + 31) / 32, nb), block(32, 8);
  const bool vec = (l->cfg.m & 3) == 0 && (reinterpret_cast<uintptr_t>(dh) & 15) == 0;
  PdlCfg pc(grid, block, 0, st);
  const float* hdp = l->hd;
  FF_CUDA(cudaLaunchKernelEx(&pc.c, vec ? k_dh_out<true> : k_dh_out<false>, hdp, B, l->cfg.m, nb, dh));
  ++g_launches;
  return FF_OK;
}

AdamArgs adam_args(const ff_layer* l, float lr, int64_t t) {
  AdamArgs a;
  a.lr = lr;
  a.beta1 = l->cfg.beta1;
  a.beta2 = l->cfg.beta2;
  a.one_minus_b1 = 1.0f - l->cfg.beta1;
  a.one_minus_b2 = 1.0f - l->cfg.beta2;
  a.rbc1 = (float)(1.0 / (1.0 - std::pow((double)l->cfg.beta1, (double)t)));
  a.rbc2 = (float)(1.0 / (1.0 - std::pow((double)l->cfg.beta2, (double)t)));
  a.eps = l->cfg.eps;
  return a;
}

RowArgs row_args(ff_layer* l, int B) {
  RowArgs a{};
  a.W = l->W; a.idx = l->idx; a.bias = l->bias; a.mW = l->mW; a.vW = l->vW; a.mb = l->mb; a.vb = l->vb;
  a.dW = l->dW; a.db = l->db; a.posmask = l->posmask; a.hd = l->hd;
  a.L = l->cfg.L_local; a.k = l->cfg.k; a.B = B; a.nb = nb_of(B); a.cstride = 64 * a.nb;
  a.err = l->err;
  a.gT = l->gT; a.rs = l->rs;
  a.j_begin = 0; a.j_end = l->cfg.L_local;
  a.check_finite = (l->cfg.flags & FF_FLAG_CHECK_FINITE) ? 1u : 0u;
  a.sqh = l->cfg.loss == FF_LOSS_SQH ? 1 : 0;
  a.split = l->split;
  return a;
}

// Row kernels are specialized on NG = number of 4-connection groups a lane walks:
// 4 for k <= 16, 8 for k <= 32.
// FULL variants (k == 16 or k == 32: every slot of every group exists) drop the per-slot guards.
template <int MODE, bool SG, bool CSC>
const void* row_kernel_csc(int k) {
  if (k == 64) return (const void*)k_rows<MODE, SG, 16, CSC, true>;
  if (k == 32) return (const void*)k_rows<MODE, SG, 8, CSC, true>;
  if (k == 16) return (const void*)k_rows<MODE, SG, 4, CSC, true>;
  if (k > 32) return (const void*)k_rows<MODE, SG, 16, CSC, false>;
  return k < 16 ? (const void*)k_rows<MODE, SG, 4, CSC, false> : (const void*)k_rows<MODE, SG, 8, CSC, false>;
}
template <int MODE, bool SG>
const void* row_kernel(int k, bool csc) {
  return csc ? row_kernel_csc<MODE, SG, true>(k) : row_kernel_csc<MODE, SG, false>(k);
}
const void* predict_kernel(int k) {
  if (k == 64) return (const void*)k_predict<16, true>;
  if (k == 32) return (const void*)k_predict<8, true>;
  if (k == 16) return (const void*)k_predict<4, true>;
  if (k > 32) return (const void*)k_predict<16, false>;
  return k < 16 ? (const void*)k_predict<4, false> : (const void*)k_predict<8, false>;
}

// Pipelined fused step (k = 32, B <= 32): same arithmetic as k_rows<train>, more gathers in flight.
// ring kernel MODE: 0 atomic, 1 CSC, 2 hybrid
int ring_mode(const ff_layer* l);
const void* ring_kernel(bool sg, int mode) {
  if (sg) return mode == 3 ? (const void*)k_train_ring<true, 3> : mode == 2 ? (const void*)k_train_ring<true, 2>
               : mode == 1 ? (const void*)k_train_ring<true, 1> : (const void*)k_train_ring<true, 0>;
  return mode == 3 ? (const void*)k_train_ring<false, 3> : mode == 2 ? (const void*)k_train_ring<false, 2>
       : mode == 1 ? (const void*)k_train_ring<false, 1> : (const void*)k_train_ring<false, 0>;
}
int ring_smem_of(int mode) {
  return mode == 3 ? ring_smem<3>() : mode == 2 ? ring_smem<2>() : mode == 1 ? ring_smem<1>() : ring_smem<0>();
}

ff_status launch_rows(const void* fn, int grid, RowArgs& a, cudaStream_t st, int threads = kRowThreads, int smem = 0) {
  void* args[] = {&a};
  PdlCfg pc(dim3(grid), dim3(threads), (size_t)smem, st);
  FF_CUDA(cudaLaunchKernelExC(&pc.c, fn, args));
  ++g_launches;
  return FF_OK;
}

int occupancy_grid(const void* fn, int nsm, int threads, int smem = 0) {
  int per = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, (size_t)smem) != cudaSuccess || per < 1) per = 1;
  return nsm * per;
}

bool ptr_ok(const void* p, int64_t n) { return n == 0 || p != nullptr; }

// CSC mode: dh of one label tile = pull over the transposed index (after the row kernel
// published that tile's g lines and pre-update weights).
ff_status launch_dh_csc(ff_layer* l, int B, int tile, cudaStream_t st) {
  const bool skipz = l->cfg.loss == FF_LOSS_SQH;      // zero gradients are exact only for the squared hinge
  auto fn = B <= 32 ? (skipz ? k_dh_csc<true, true> : k_dh_csc<true, false>)
                    : (skipz ? k_dh_csc<false, true> : k_dh_csc<false, false>);
  PdlCfg pc(dim3(l->grid_csc), dim3(256), 0, st);
  const int* cp = l->col_ptr; const int* en = l->ent; const float* g = l->gT;
  int nbB = nb_of(B), sp = (int)l->split;
  FF_CUDA(cudaLaunchKernelEx(&pc.c, fn, cp, en, g, l->rs, l->cfg.m, nbB, tile, l->hd, sp));
  ++g_launches;
  return FF_OK;
}

// Rows per warp block: 32 unless that leaves resident warps idle (small L), then 16, 8 or 4
// so that every warp gets at least two blocks.
int block_rows(int64_t rows, int grid, int threads) {
  const int64_t warps = (int64_t)grid * (threads / 32);
  int br = 32;
  while (br > 4 && (rows + br - 1) / br < 2 * warps) br >>= 1;
  return br;
}

// One row-kernel launch, bracketed by a profiling event pair while profiling is on.
ff_status timed_rows(ff_layer* l, const void* fn, int grid, RowArgs& a, cudaStream_t st, int threads, int smem) {
  a.br = block_rows(a.j_end - a.j_begin, grid, threads);
  const bool timed = !l->prof_paused && 2 * (l->prof_used + 1) <= (int)l->prof_ev.size();
  if (timed) FF_CUDA(cudaEventRecord(l->prof_ev[2 * l->prof_used], st));
  ff_status s = launch_rows(fn, grid, a, st, threads, smem);
  if (s != FF_OK) return s;
  if (timed) FF_CUDA(cudaEventRecord(l->prof_ev[2 * l->prof_used++ + 1], st));
  return FF_OK;
}

// The row pass (+ the CSC column pass per label tile in CSC mode).
ff_status run_rows(ff_layer* l, const void* fn, int grid, RowArgs& a, int B, cudaStream_t st,
                   int threads = kRowThreads, int smem = 0) {
  if (!l->csc) {
    if (l->cfg.L_local == 0) return FF_OK;
    return timed_rows(l, fn, grid, a, st, threads, smem);
  }
  for (int t = 0; t < l->ntiles; ++t) {
    a.j_begin = (int64_t)t * l->tile_rows;
    a.j_end = std::min<int64_t>(a.j_begin + l->tile_rows, l->cfg.L_local);
    ff_status s = timed_rows(l, fn, grid, a, st, threads, smem);
    if (s != FF_OK) return s;
    if (B > 0) {
      s = launch_dh_csc(l, B, t, st);
      if (s != FF_OK) return s;
    }
  }

  return FF_OK;
}

// Rebuild the transposed (CSC) index of idx: stable radix sort of (column, connection id)
// pairs; the sort's ping-pong buffers borrow gT / wcsc / dW / ent_row, so it runs between
// steps only (create, set_params, redistribute) and invalidates stored gradients.
ff_status csc_rebuild(ff_layer* l, cudaStream_t st) {
  const int64_t n = l->cfg.L_local * l->cfg.k;
  int* keysA = l->sort_keys;
  int* keysB = l->sort_keys2;
  int* valsA = reinterpret_cast<int*>(l->dW);
  int* valsB = l->ent;
  const int nkeys = l->ntiles * l->cfg.m;
  int end_bit = 1;
  while ((1ll << end_bit) < (long long)nkeys) ++end_bit;
  if (n > 0) {
    k_csc_keys<<<l->nsm * 8, 256, 0, st>>>(l->idx, n, l->cfg.k, l->cfg.m, l->tile_rows, keysA, valsA);
    FF_LAUNCHED();
  }
  cub::DoubleBuffer<unsigned> dk(reinterpret_cast<unsigned*>(keysA), reinterpret_cast<unsigned*>(keysB));
  cub::DoubleBuffer<int> dv(valsA, valsB);
  if (n > 0) {
    size_t need = 0;
    FF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, need, dk, dv, (int)n, 0, end_bit, st));
    if (need > l->lay.sort_tmp_bytes)
      return fail(FF_ERR_CONFIG, "CSC sort needs %zu B of scratch > reserved %zu B", need, l->lay.sort_tmp_bytes);
    size_t have = l->lay.sort_tmp_bytes;
    FF_CUDA(cub::DeviceRadixSort::SortPairs(l->sort_tmp, have, dk, dv, (int)n, 0, end_bit, st));
    ++g_launches;
  }
  k_csc_finish<<<l->nsm * 8, 256, 0, st>>>(reinterpret_cast<const int*>(dk.Current()), dv.Current(), n, l->cfg.k,
                                           l->tile_rows, nkeys, l->ent, l->col_ptr);
  FF_LAUNCHED();
  l->grads_valid = false;
  return FF_OK;
}

// hd_ready: h is already in the h half of hd and (atomic mode) the dh half is zero (the
// model step's dense forward wrote them); dh then stays in hd (dh may be NULL).
// dh_optional (host entry point): dh == NULL skips only the [B][m] copy-out of dh.
ff_status train_step_impl(ff_layer* l, const float* h, int32_t B, const int32_t* lbl_ptr, const int32_t* lbl_ids,
                          float grad_scale, float lr, float* dh, float* loss, cudaStream_t st, bool hd_ready = false,
                          bool dh_optional = false, const DenseT* dt = nullptr) {
  if (B < 0 || B > l->cfg.max_batch) return fail(FF_ERR_ARG, "B=%d outside [0, max_batch=%d]", B, l->cfg.max_batch);
  if ((!hd_ready && (!ptr_ok(h, B) || (!dh_optional && !ptr_ok(dh, B)))) || lbl_ptr == nullptr)
    return fail(FF_ERR_ARG, "null h/dh/lbl_ptr");
  ff_status s = launch_prep(l, hd_ready ? nullptr : h, B, (!l->csc || l->split > 0) && !hd_ready, lbl_ptr, lbl_ids,
                            loss, st, true, dt);
  if (s != FF_OK) return s;
  l->t += 1;
  RowArgs a = row_args(l, B);
  a.grad_scale = grad_scale;
  a.loss = loss;
  a.adam = adam_args(l, lr, l->t);                // rbc1/rbc2 are replaced by the device's (a.rbc)
  a.rbc = l->rbc_dev;
  const bool sg = (l->cfg.flags & FF_FLAG_STORE_GRADS) != 0;
  const bool pipe = l->cfg.k == 32 && B <= 32 && !(l->cfg.flags & FF_FLAG_NO_PIPE);
  if (pipe) {
    const int rm = ring_mode(l);
    s = run_rows(l, ring_kernel(sg, rm), l->grid_ring, a, B, st, kRingThreads, ring_smem_of(rm));
  } else {
    const void* fn = sg ? row_kernel<kModeTrain, true>(l->cfg.k, l->csc) : row_kernel<kModeTrain, false>(l->cfg.k, l->csc);
    s = run_rows(l, fn, l->grid_train, a, B, st, kRowThreads);
  }
  if (s != FF_OK) return s;
  l->grads_valid = (l->cfg.flags & FF_FLAG_STORE_GRADS) != 0;
  if (B == 0 || dh == nullptr) return FF_OK;
  return launch_dh_out(l, B, dh, st);
}

// Top-K of the scores of h; hd_ready: h is already in the h half of hd (model predict).
ff_status predict_impl(ff_layer* l, const float* h, int32_t B, int32_t K, float* scores, int32_t* ids,
                       cudaStream_t st, bool hd_ready) {
  if (!l) return fail(FF_ERR_ARG, "layer is NULL");
  if (B < 0 || B > l->cfg.max_batch) return fail(FF_ERR_ARG, "B=%d outside [0, max_batch=%d]", B, l->cfg.max_batch);
  if (K < 1 || K > l->cfg.max_topk || K > l->cfg.L_local)
    return fail(FF_ERR_ARG, "K=%d outside [1, min(max_topk=%d, L_local=%lld)]", K, l->cfg.max_topk,
                (long long)l->cfg.L_local);
  if (B == 0) return FF_OK;
  if ((!h && !hd_ready) || !scores || !ids) return fail(FF_ERR_ARG, "null h/scores/ids");
  if (!hd_ready) {
    ff_status s = launch_prep(l, h, B, false, nullptr, nullptr, nullptr, st);
    if (s != FF_OK) return s;
  }
  const int nb = nb_of(B), ldh = 32 * nb;
  const float* W = l->W; const int* idx = l->idx; const float* bias = l->bias; const float* hd = l->hd;
  int64_t L = l->cfg.L_local, rb = l->cfg.row_begin; int k = l->cfg.k, BB = B, nbb = nb;
  float* cs = l->cand_s; int* ci = l->cand_i;
  int* perr = (l->cfg.flags & FF_FLAG_CHECK_FINITE) ? l->err : nullptr;     // NaN/inf scores reported (R15)
  int nlist = l->grid_pred;
  if (k == 32 && (nb == 1 || (nb <= kPredRingMaxLines && !(l->cfg.flags & FF_FLAG_NO_PIPE)))) {
    // hot configuration (B <= 32), and B <= 96: the pipelined kernel once per 32-sample line
    // (bit-identical scores; below 4 lines the wide kernel would leave lanes idle)
#if FF_PRED_REG
    nlist = l->grid_pred_reg;
#else
    nlist = l->grid_pred_ring;
#endif
    for (int q2 = 0; q2 < nb; ++q2) {
      int* gt = l->pthr;
      void* args[] = {&W, &idx, &bias, &hd, &L, &BB, &nbb, &q2, &rb, &cs, &ci, &gt, &perr};
#if FF_PRED_REG
      FF_CUDA(cudaLaunchKernel(perr ? (const void*)k_predict_reg<true> : (const void*)k_predict_reg<false>,
                               dim3(nlist), dim3(kPredRegThreads), args, 0, st));
#else
      FF_CUDA(cudaLaunchKernel(perr ? (const void*)k_predict_ring<true> : (const void*)k_predict_ring<false>, dim3(nlist),
                               dim3(kPredRingThreads), args, kPredRingSmem, st));
#endif
      if (q2 + 1 < nb) ++g_launches;
    }
  } else if (k == 32 && !(l->cfg.flags & FF_FLAG_NO_PIPE)) {   // large batch: chunked wide kernel (bit-identical)
    // pass 1 over a prefix of the rows, merged into its exact top-K (list slot g of cand);
    // pass 2 over the rest, thresholds from that list; the final merge takes g + 1 lists
    const int g = l->grid_pred_wide;
    const int64_t r1 = std::min<int64_t>(L, std::max<int64_t>(L / 32, (int64_t)g * (kPredWThreads / 32)));
    float* wls = l->wl_s; int* wli = l->wl_i;
    float* ps = cs + (int64_t)g * ldh * kTopkMax; int* pi = ci + (int64_t)g * ldh * kTopkMax;
    const float* no_s = nullptr; const int* no_i = nullptr;
    int64_t z = 0, Lw = L;
    int Kw = K;
    void* a1[] = {&W, &idx, &bias, &hd, &z, const_cast<int64_t*>(&r1), &BB, &nbb, &rb, &no_s, &no_i, &Kw, &cs, &ci, &wls, &wli, &perr};
    FF_CUDA(cudaLaunchKernel((const void*)k_predict_wide, dim3(g), dim3(kPredWThreads), a1, kPredWSmem, st));
    k_merge_topk_block<<<B, kMergeThreads, 0, st>>>(cs, ci, g, (int64_t)ldh * kTopkMax, kTopkMax, kTopkMax, kTopkMax,
                                                    ps, pi, nullptr);
    g_launches += 2;
    const float* ts_ = ps; const int* ti_ = pi;
    void* a2[] = {&W, &idx, &bias, &hd, const_cast<int64_t*>(&r1), &Lw, &BB, &nbb, &rb, &ts_, &ti_, &Kw, &cs, &ci, &wls, &wli, &perr};
    FF_CUDA(cudaLaunchKernel((const void*)k_predict_wide, dim3(g), dim3(kPredWThreads), a2, kPredWSmem, st));
    nlist = g + 1;
  } else {
    void* args[] = {&W, &idx, &bias, &hd, &L, &k, &BB, &nbb, &rb, &cs, &ci, &perr};
    FF_CUDA(cudaLaunchKernel(predict_kernel(l->cfg.k), dim3(l->grid_pred), dim3(kRowThreads), args, 0, st));
  }
  ++g_launches;
  k_merge_topk_block<<<B, kMergeThreads, 0, st>>>(l->cand_s, l->cand_i, nlist, (int64_t)ldh * kTopkMax, kTopkMax, kTopkMax, K,
                                                  scores, ids, l->pthr);         // also re-arms the ring's thresholds
  FF_LAUNCHED();
  return FF_OK;
}


// ============================================================ NEXT-2: the intermediate layer
struct DenseLayout {
  size_t Wd, mWd, vWd, dWd, bd, mbd, vbd, dbd, xT, xTlo, zpart, cnt, hd, x_stage, scal, total;
};
int ldw_of(int m) { return (m + 127) / 128 * 128; }   // Wd is stored in 128-column tiles
DenseLayout dense_layout_of(const ff_dense_config& c) {
  DenseLayout o{};
  const size_t dw = (size_t)c.d * (size_t)ldw_of(c.m), w = (size_t)ldw_of(c.m);
  const size_t nbm = (size_t)nb_of(c.max_batch), ldx = 32 * nbm;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t r = off; off += up(bytes); return r; };
  o.Wd = take(4 * dw); o.mWd = take(4 * dw); o.vWd = take(4 * dw);
  o.dWd = (c.flags & FF_FLAG_STORE_GRADS) ? take(4 * dw) : 0;
  o.bd = take(4 * w); o.mbd = take(4 * w); o.vbd = take(4 * w); o.dbd = take(4 * w);
  o.xT = take(4 * (size_t)c.d * ldx);
  o.xTlo = take(4 * (size_t)c.d * 32);                      // lo part of xT (tensor-core forward, B <= 32)
  o.zpart = take(2 * 4 * (size_t)ldw_of(c.m) * 32);        // split-feature forward partials (B <= 32)
  o.cnt = take(4 * (size_t)(ldw_of(c.m) / 128));
  o.hd = take(8 * (size_t)c.m * ldx);     // own h|dh lines for the standalone forward/backward
  o.x_stage = take(4 * (size_t)c.max_batch * (size_t)c.d);
  o.scal = take(kAlign);           // [0] int64 Adam t (device, authoritative), [8] float rbc[2]
  o.total = off;
  return o;
}
ff_status dense_validate(const ff_dense_config* c) {
  if (!c) return fail(FF_ERR_ARG, "cfg is NULL");
  if (c->d < 1 || c->m < 1) return fail(FF_ERR_CONFIG, "d=%d, m=%d must be >= 1", c->d, c->m);
  if ((int64_t)c->d * ldw_of(c->m) >= (int64_t(1) << 40)) return fail(FF_ERR_CONFIG, "d*m too large");
  if (c->max_batch < 1 || c->max_batch > FF_MAX_BATCH)
    return fail(FF_ERR_CONFIG, "max_batch=%d outside [1, %d]", c->max_batch, FF_MAX_BATCH);
  if (!(c->dropout >= 0.0f && c->dropout < 1.0f)) return fail(FF_ERR_CONFIG, "dropout outside [0, 1)");
  if (c->col_begin < 0 || c->m_global < 0 || (int64_t)c->col_begin + c->m > (c->m_global ? c->m_global : INT32_MAX))
    return fail(FF_ERR_CONFIG, "column shard [%d, %lld) outside [0, m_global=%d)", c->col_begin,
                (long long)c->col_begin + c->m, c->m_global);
  if (c->beta1 < 0.0f || c->beta1 >= 1.0f || c->beta2 < 0.0f || c->beta2 >= 1.0f || c->eps < 0.0f)
    return fail(FF_ERR_CONFIG, "Adam hyper-parameters out of range");
  return FF_OK;
}
ff_dense_config dense_defaults(const ff_dense_config& in) {
  ff_dense_config c = in;
  if (c.beta1 == 0.0f) c.beta1 = 0.9f;
  if (c.beta2 == 0.0f) c.beta2 = 0.999f;
  if (c.eps == 0.0f) c.eps = 1e-8f;
  if (c.m_global == 0) c.m_global = c.col_begin + c.m;
  if (c.init_scale == 0.0f) c.init_scale = (float)std::sqrt(6.0 / ((double)c.d + (double)c.m_global));
  return c;
}
AdamArgs adam_args_of(float beta1, float beta2, float eps, float lr, int64_t t) {
  AdamArgs a;
  a.lr = lr; a.beta1 = beta1; a.beta2 = beta2; a.one_minus_b1 = 1.0f - beta1; a.one_minus_b2 = 1.0f - beta2;
  a.rbc1 = (float)(1.0 / (1.0 - std::pow((double)beta1, (double)t)));
  a.rbc2 = (float)(1.0 / (1.0 - std::pow((double)beta2, (double)t)));
  a.eps = eps;
  return a;
}

}  // namespace

struct ff_dense {
  ff_dense_config cfg;
  DenseLayout lay;
  char* ws;
  float *Wd, *mWd, *vWd, *dWd, *bd, *mbd, *vbd, *dbd, *xT, *xTlo, *hd, *x_stage, *zpart;
  unsigned* cnt;
  CUtensorMap tmW, tmX, tmXl;   // TMA maps of Wd, xT and xTlo (k_dense_fwd_tma), encoded at create
  int ldw;
  int nsm;
  int grid_bwd32;       // resident CTAs of the persistent B <= 32 backward
  int64_t t;            // host mirror of *t_dev
  int64_t* t_dev;       // Adam step counter (R28), advanced on the device (CUDA-graph capturable)
  float* rbc_dev;       // [2] bias corrections of the current step
  int fwd_B;            // batch of the last training forward (-1: none since the last backward)
  bool grads_valid;
};

namespace {

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda link)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}
// Wd: {128 columns, d features, tiles} over the tiled layout [ldw/128][d][128]; xT, xTlo:
// {32 samples, d} (the B <= 32 layout, ldx = 32).  Box 32 x 32 (x 1); features >= d read 0.
const char* encode_dense_maps(ff_dense* n) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (enc == nullptr) return "cuTensorMapEncodeTiled unavailable";
  const cuuint64_t d = (cuuint64_t)n->cfg.d;
  const cuuint32_t es[3] = {1, 1, 1};
  {
    const cuuint64_t dims[3] = {128, d, (cuuint64_t)(n->ldw / 128)};
    const cuuint64_t strides[2] = {128 * 4, d * 128 * 4};
    const cuuint32_t box[3] = {32, (cuuint32_t)kTmF, 1};
    if (enc(&n->tmW, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, n->Wd, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS)
      return "Wd map";
  }
  const cuuint64_t dims[2] = {32, d};
  const cuuint64_t strides[1] = {32 * 4};
  const cuuint32_t box[2] = {32, (cuuint32_t)kTmF};
  if (enc(&n->tmX, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, n->xT, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
          CUDA_SUCCESS ||
      enc(&n->tmXl, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, n->xTlo, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
          CUDA_SUCCESS)
    return "xT map";
  return nullptr;
}

// dropout + forward into `hd` (the dense layer's own lines or a fixed fan-in layer's)
ff_status dense_forward_impl(ff_dense* n, const float* x, int B, uint64_t step, bool train, float* hd,
                             float* h_out, cudaStream_t st) {
  const int nb = nb_of(B), ldx = 32 * nb;
  const float p = n->cfg.dropout;
  const float scale = (float)(1.0f / (1.0f - p));
  {
    const int64_t work = (int64_t)ldx * ((n->cfg.d + 3) / 4);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 4096));
    k_dropout_T<<<grid, 256, 0, st>>>(x, B, n->cfg.d, ldx, p, scale, (train && p > 0.0f) ? 1 : 0, (uint32_t)step,
                                      (uint32_t)n->cfg.seed, (uint32_t)(n->cfg.seed >> 32), n->xT,
                                      step == FF_STEP_AUTO ? n->t_dev : nullptr, nb == 1 ? n->xTlo : nullptr);
    FF_LAUNCHED();
  }
  if (nb == 1 && !(n->cfg.flags & FF_FLAG_DENSE_SIMT)) {          // tensor cores (tcgen05 + TMA, 3xTF32)
    // persistent, one CTA per SM; a programmatic dependent of k_dropout_T (PDL): its set-up and
    // first Wd stages overlap the dropout kernel, its xT loads wait for it (griddepcontrol.wait)
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(std::min(n->ldw / 128, n->nsm));
    lc.blockDim = dim3(kTmThreads);
    lc.dynamicSmemBytes = kTmSmem;
    lc.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    const float* bdp = n->bd;
    int dd = n->cfg.d, mm = n->cfg.m, BB = B, cs = 64, zd = 1;
    FF_CUDA(cudaLaunchKernelEx(&lc, k_dense_fwd_tma, n->tmW, n->tmX, n->tmXl, bdp, dd, mm, BB, hd, cs, zd, h_out));
    ++g_launches;
    if (train) n->fwd_B = B;
    return FF_OK;
  }
  // B <= 32 and at least two feature chunks: split the features over two CTAs per column tile
  const int split = (nb == 1 && n->cfg.d >= 2 * kDenseFch) ? kDenseFwdSplit : 1;
  dim3 grid((n->ldw + 127) / 128, nb, split);
  k_dense_fwd<<<grid, kDenseFwdThreads, kDenseFwdSmem, st>>>(n->Wd, n->bd, n->xT, n->cfg.d, n->cfg.m, n->ldw, ldx, B, hd,
                                                             64 * nb, 1, h_out, n->zpart, n->cnt);
  FF_LAUNCHED();
  if (train) n->fwd_B = B;
  return FF_OK;
}

// backward + Adam from the h|dh lines of `hd` (t += 1)
// t_done: this step's k_prep already advanced the dense counter (whole-architecture step)
ff_status dense_backward_impl(ff_dense* n, int B, float lr, const float* hd, cudaStream_t st, bool t_done = false) {
  const int nb = nb_of(B), ldx = 32 * nb;
  n->t += 1;
  if (!t_done) {
    k_step_t<<<1, 32, 0, st>>>(n->t_dev, n->rbc_dev, n->cfg.beta1, n->cfg.beta2);
    FF_LAUNCHED();
  }
  const AdamArgs a = adam_args_of(n->cfg.beta1, n->cfg.beta2, n->cfg.eps, lr, n->t);   // rbc from the device
  const bool sg = (n->cfg.flags & FF_FLAG_STORE_GRADS) != 0;
  // feature ranges per column tile: about 4 CTAs per SM in total, whole 16-feature blocks
  const int gx = (n->ldw + 127) / 128;
  const int fq = std::max(1, std::min((n->cfg.d + kDenseBwdBlk - 1) / kDenseBwdBlk, (4 * n->nsm + gx - 1) / gx));
  const int rows = ((n->cfg.d + fq - 1) / fq + kDenseBwdBlk - 1) / kDenseBwdBlk * kDenseBwdBlk;
  dim3 grid(gx, (n->cfg.d + rows - 1) / rows);
  if (nb == 1)     // persistent: equal contiguous ranges of (tile, 16-feature block) items per resident CTA
    k_dense_bwd_adam_b32<<<std::min<int64_t>((int64_t)n->grid_bwd32, (int64_t)gx * ((n->cfg.d + kDenseBwdBlk - 1) / kDenseBwdBlk)),
                           kDenseBwd32Threads, kDenseBwd1Smem, st>>>(
        n->Wd, n->mWd, n->vWd, n->bd, n->mbd, n->vbd, n->xT, n->cfg.d, n->cfg.m, ldx, hd, 64 * nb, a,
        sg ? n->dWd : nullptr, sg ? n->dbd : nullptr, gx, n->rbc_dev);
  else
    k_dense_bwd_adam<<<grid, kDenseBwdThreads, 0, st>>>(n->Wd, n->mWd, n->vWd, n->bd, n->mbd, n->vbd, n->xT, n->cfg.d,
                                                        n->cfg.m, n->ldw, ldx, nb, hd, 64 * nb, a,
                                                        sg ? n->dWd : nullptr, sg ? n->dbd : nullptr, rows,
                                                        n->rbc_dev);
  FF_LAUNCHED();
  n->grads_valid = sg;
  n->fwd_B = -1;
  return FF_OK;
}

}  // namespace

extern "C" {

const char* fixedfanin_last_error(void) { return g_err.c_str(); }
int32_t fixedfanin_last_launch_count(void) { return g_launches; }

ff_status fixedfanin_workspace_size(const ff_config* cfg, size_t* bytes) {
  g_launches = 0;
  ff_status s = validate(cfg);
  if (s != FF_OK) return s;
  if (!bytes) return fail(FF_ERR_ARG, "bytes is NULL");
  *bytes = layout_of(with_defaults(*cfg)).total;
  return FF_OK;
}

ff_status fixedfanin_create(const ff_config* cfg, void* workspace, size_t bytes, ff_stream_t stream,
                            ff_layer** out) {
  g_launches = 0;
  ff_status s = validate(cfg);
  if (s != FF_OK) return s;
  if (!out || !workspace) return fail(FF_ERR_ARG, "out/workspace is NULL");
  if (reinterpret_cast<uintptr_t>(workspace) % kAlign) return fail(FF_ERR_ARG, "workspace not 256-B aligned");
  const ff_config c = with_defaults(*cfg);
  const Layout lay = layout_of(c);
  if (bytes < lay.total) return fail(FF_ERR_ARG, "workspace %zu B < required %zu B", bytes, lay.total);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  FF_CUDA(cudaGetLastError());
  ff_layer* l = new (std::nothrow) ff_layer();
  if (!l) return fail(FF_ERR_ARG, "host allocation failed");
  l->cfg = c; l->lay = lay;
  char* ws = static_cast<char*>(workspace);
  l->ws = ws;
  l->W = at<float>(ws, lay.W); l->idx = at<int>(ws, lay.idx); l->mW = at<float>(ws, lay.mW);
  l->vW = at<float>(ws, lay.vW); l->dW = at<float>(ws, lay.dW); l->bias = at<float>(ws, lay.bias);
  l->mb = at<float>(ws, lay.mb); l->vb = at<float>(ws, lay.vb); l->db = at<float>(ws, lay.db);
  l->posmask = at<uint32_t>(ws, lay.posmask); l->hd = at<float>(ws, lay.hd);
  l->cand_s = at<float>(ws, lay.cand_s); l->cand_i = at<int>(ws, lay.cand_i);
  l->pthr = at<int>(ws, lay.pthr);
  l->wl_s = lay.wl_s ? at<float>(ws, lay.wl_s) : nullptr; l->wl_i = lay.wl_i ? at<int>(ws, lay.wl_i) : nullptr;
  l->h_stage = at<float>(ws, lay.h_stage); l->lbl_stage = at<int>(ws, lay.lbl_stage);
  l->dh_stage = at<float>(ws, lay.dh_stage);
  l->err = at<int>(ws, lay.scalars); l->loss_scratch = at<float>(ws, lay.scalars + 4);
  l->t_dev = at<int64_t>(ws, lay.scalars + 8); l->rbc_dev = at<float>(ws, lay.scalars + 16);
  l->csc = c.dh_mode != FF_DH_ATOMIC;
  l->split = c.dh_mode == FF_DH_HYBRID
                 ? (uint32_t)std::min<double>(c.m, std::floor((double)c.hybrid_frac * (double)c.m + 0.5)) : 0u;
  if (l->csc) {
    l->ent = at<int>(ws, lay.ent); l->sort_keys2 = at<int>(ws, lay.sort_keys2);
    l->gT = at<float>(ws, lay.gT); l->col_ptr = at<int>(ws, lay.col_ptr); l->sort_tmp = ws + lay.sort_tmp;
    l->sort_keys = at<int>(ws, lay.sort_keys);
    l->rs = csc_rec_stride(c.max_batch, c.k);
  }
  l->t = 0; l->grads_valid = false;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&l->nsm, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) { delete l; return fail(FF_ERR_CUDA, "device query: %s", cudaGetErrorString(e)); }
  l->grid_train = occupancy_grid(row_kernel<kModeTrain, false>(c.k, l->csc), l->nsm, kRowThreads);
  l->grid_fwd = occupancy_grid(row_kernel<kModeForward, false>(c.k, false), l->nsm, kRowThreads);
  l->grid_bwd = occupancy_grid(row_kernel<kModeBackward, false>(c.k, l->csc), l->nsm, kRowThreads);
#ifndef FF_CSC_COL_CTAS
#define FF_CSC_COL_CTAS 0          // CSC column pass CTAs per SM (0: as many as fit)
#endif
  l->grid_csc = FF_CSC_COL_CTAS > 0 ? FF_CSC_COL_CTAS * l->nsm : occupancy_grid((const void*)k_dh_csc<true, false>, l->nsm, 256);
  for (int sg = 0; sg < 2; ++sg)
    for (int cs = 0; cs < 4; ++cs)
      if (cudaFuncSetAttribute(ring_kernel(sg, cs), cudaFuncAttributeMaxDynamicSharedMemorySize, ring_smem_of(cs)) !=
          cudaSuccess) {
        delete l;
        return fail(FF_ERR_CUDA, "pipelined kernel smem attribute");
      }
  l->grid_ring = occupancy_grid(ring_kernel(false, ring_mode(l)), l->nsm, kRingThreads, ring_smem_of(ring_mode(l)));
  if (l->csc) {
    // tile = a whole number of row-kernel "waves" (warps x 32 labels) within the L2 budget
    const int64_t cap = (int64_t)csc_tile_cap(c), wave = (int64_t)l->grid_train * (kRowThreads / 32) * 32;
    l->tile_rows = cap >= wave ? cap / wave * wave : cap;
    l->ntiles = (int)std::max<int64_t>(1, (c.L_local + l->tile_rows - 1) / l->tile_rows);
  }
  l->grid_pred = std::min(kMaxCandBlocks, occupancy_grid(predict_kernel(c.k), l->nsm, kRowThreads));
  if (cudaFuncSetAttribute((const void*)k_predict_ring<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kPredRingSmem) != cudaSuccess ||
      cudaFuncSetAttribute((const void*)k_predict_ring<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kPredRingSmem) != cudaSuccess) {
    delete l;
    return fail(FF_ERR_CUDA, "pipelined predict smem attribute");
  }
  l->grid_pred_ring =
      std::min(kMaxCandBlocks, occupancy_grid((const void*)k_predict_ring<false>, l->nsm, kPredRingThreads, kPredRingSmem));
#if FF_PRED_REG
  l->grid_pred_reg = std::min(kMaxCandBlocks, occupancy_grid((const void*)k_predict_reg<false>, l->nsm,
                                                             kPredRegThreads));
#endif
  if (cudaFuncSetAttribute((const void*)k_predict_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, kPredWSmem) !=
      cudaSuccess) {
    delete l;
    return fail(FF_ERR_CUDA, "wide predict smem attribute");
  }
  l->grid_pred_wide = std::min(std::min(kMaxCandBlocks - 1, kMaxWideWarps / (kPredWThreads / 32)),
                               occupancy_grid((const void*)k_predict_wide, l->nsm, kPredWThreads, kPredWSmem));
  l->grid_rows = l->nsm * 8;
  // zero everything that must start at zero (moments, masks, dW/db, dhT, scalars)
  e = cudaMemsetAsync(ws, 0, lay.total, st);
  if (e != cudaSuccess) { delete l; return fail(FF_ERR_CUDA, "memset: %s", cudaGetErrorString(e)); }
  {                                                    // predict thresholds start at score_key(-inf)
    const int n = 32 * nb_of(c.max_batch);
    k_fill_i32<<<(n + 255) / 256, 256, 0, st>>>(l->pthr, n, kKeyNegInf);
    ++g_launches;
  }
  if (c.L_local > 0) {
    k_init<<<l->grid_rows, 256, 0, st>>>(l->W, l->idx, l->bias, l->mW, l->vW, l->mb, l->vb, c.L_local, c.row_begin,
                                         c.m, c.k, (uint32_t)c.seed, (uint32_t)(c.seed >> 32), c.init_scale);
    ++g_launches;
    e = cudaGetLastError();
    if (e != cudaSuccess) { delete l; return fail(FF_ERR_CUDA, "init launch: %s", cudaGetErrorString(e)); }
  }
  if (l->csc) {
    ff_status s2 = csc_rebuild(l, st);
    if (s2 != FF_OK) { fixedfanin_destroy(l); return s2; }
  }
  *out = l;
  return FF_OK;
}

ff_status fixedfanin_destroy(ff_layer* l) {
  if (l) for (cudaEvent_t e : l->prof_ev) cudaEventDestroy(e);
  if (l) {
    for (int i = 0; i < 2; ++i) {
      if (l->ev_ready[i]) cudaEventDestroy(l->ev_ready[i]);
      if (l->ev_free[i]) cudaEventDestroy(l->ev_free[i]);
    }
    if (l->copy_st) cudaStreamDestroy(l->copy_st);

  }
  delete l;
  return FF_OK;
}

ff_status fixedfanin_set_params(ff_layer* l, const float* W, const int32_t* idx, const float* bias, const float* mW,
                                const float* vW, const float* mb, const float* vb, const int64_t* t,
                                ff_stream_t stream) {
  g_launches = 0;
  if (!l) return fail(FF_ERR_ARG, "layer is NULL");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t Lk = (size_t)l->cfg.L_local * l->cfg.k * 4, L4 = (size_t)l->cfg.L_local * 4;
  auto cp = [&](void* dst, const void* src, size_t n) -> cudaError_t {
    return (src && n) ? cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToDevice, st) : cudaSuccess;
  };
  FF_CUDA(cp(l->W, W, Lk)); FF_CUDA(cp(l->idx, idx, Lk)); FF_CUDA(cp(l->bias, bias, L4));
  FF_CUDA(cp(l->mW, mW, Lk)); FF_CUDA(cp(l->vW, vW, Lk)); FF_CUDA(cp(l->mb, mb, L4)); FF_CUDA(cp(l->vb, vb, L4));
  if (t) {
    l->t = *t;
    FF_CUDA(cudaMemcpyAsync(l->t_dev, &l->t, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    FF_CUDA(cudaStreamSynchronize(st));                 // &l->t is host memory read asynchronously
  }
  l->grads_valid = false;
  if (idx && l->cfg.L_local > 0) {
    FF_CUDA(cudaMemsetAsync(l->err, 0, sizeof(int), st));
    k_validate_idx<<<l->grid_rows, 256, 0, st>>>(l->idx, l->cfg.L_local, l->cfg.m, l->cfg.k, l->err);
    FF_LAUNCHED();
    int herr = 0;
    FF_CUDA(cudaMemcpyAsync(&herr, l->err, sizeof(int), cudaMemcpyDeviceToHost, st));
    FF_CUDA(cudaStreamSynchronize(st));
    if (herr & kErrIdxRange) return fail(FF_ERR_RANGE, "set_params: idx outside [0, m=%d)", l->cfg.m);
    if (herr & kErrIdxDup) return fail(FF_ERR_RANGE, "set_params: duplicate idx within a row");
    if (l->csc) {
      ff_status s2 = csc_rebuild(l, st);
      if (s2 != FF_OK) return s2;
    }
  }
  FF_CUDA(cudaStreamSynchronize(st));
  return FF_OK;
}

ff_status fixedfanin_get_params(ff_layer* l, float* W, int32_t* idx, float* bias, float* mW, float* vW, float* mb,
                                float* vb, int64_t* t, ff_stream_t stream) {
  g_launches = 0;
  if (!l) return fail(FF_ERR_ARG, "layer is NULL");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t Lk = (size_t)l->cfg.L_local * l->cfg.k * 4, L4 = (size_t)l->cfg.L_local * 4;
  auto cp = [&](void* dst, const void* src, size_t n) -> cudaError_t {
    return (dst && n) ? cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToDevice, st) : cudaSuccess;
  };
  FF_CUDA(cp(W, l->W, Lk)); FF_CUDA(cp(idx, l->idx, Lk)); FF_CUDA(cp(bias, l->bias, L4));
  FF_CUDA(cp(mW, l->mW, Lk)); FF_CUDA(cp(vW, l->vW, Lk)); FF_CUDA(cp(mb, l->mb, L4)); FF_CUDA(cp(vb, l->vb, L4));
  if (t) FF_CUDA(cudaMemcpyAsync(t, l->t_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FF_CUDA(cudaStreamSynchronize(st));
  if (t) l->t = *t;
  return FF_OK;
}

ff_status fixedfanin_forward(ff_layer* l, const float* h, int32_t B, float* y, ff_stream_t stream) {
  g_launches = 0;
  if (!l) return fail(FF_ERR_ARG, "layer is NULL");
  if (B < 0 || B > l->cfg.max_batch) return fail(FF_ERR_ARG, "B=%d outside [0, max_batch=%d]", B, l->cfg.max_batch);
  if (B == 0) return FF_OK;
  if (!h || (!y && l->cfg.L_local > 0)) return fail(FF_ERR_ARG, "null h/y");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  ff_status s = launch_prep(l, h, B, false, nullptr, nullptr, nullptr, st);
  if (s != FF_OK) return s;
  if (l->cfg.L_local == 0) return FF_OK;
  RowArgs a = row_args(l, B);
  a.y_out = y;
  a.br = block_rows(l->cfg.L_local, l->grid_fwd, kRowThreads);
  return launch_rows(row_kernel<kModeForward, false>(l->cfg.k, false), l->grid_fwd, a, st);
}

ff_status fixedfanin_backward(ff_layer* l, const float* h, const float* y, int32_t B, const int32_t* lbl_ptr,
                              const int32_t* lbl_ids, float grad_scale, float* dh, float* loss, ff_stream_t stream) {
  g_launches = 0;
  if (!l) return fail(FF_ERR_ARG, "layer is NULL");
  if (B < 0 || B > l->cfg.max_batch) return fail(FF_ERR_ARG, "B=%d outside [0, max_batch=%d]", B, l->cfg.max_batch);
  if (!ptr_ok(h, B) || !ptr_ok(dh, B) || lbl_ptr == nullptr || (B > 0 && l->cfg.L_local > 0 && !y))
    return fail(FF_ERR_ARG, "null h/y/dh/lbl_ptr");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  ff_status s = launch_prep(l, h, B, !l->csc || l->split > 0, lbl_ptr, lbl_ids, loss, st);
  if (s != FF_OK) return s;
  RowArgs a = row_args(l, B);
  a.y_in = y; a.grad_scale = grad_scale; a.loss = loss;
  s = run_rows(l, row_kernel<kModeBackward, false>(l->cfg.k, l->csc), l->grid_bwd, a, B, st);
  if (s != FF_OK) return s;
  l->grads_valid = true;
  if (B == 0) return FF_OK;
  return launch_dh_out(l, B, dh, st);
}

ff_status fixedfanin_get_grads(ff_layer* l, float* dW, float* db, ff_stream_t stream) {
  g_launches = 0;
  if (!l) return fail(FF_ERR_ARG, "layer is NULL");
  if (!l->grads_valid) return fail(FF_ERR_STATE, "no gradients: run backward (or train_step with FF_FLAG_STORE_GRADS)");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t Lk = (size_t)l->cfg.L_local * l->cfg.k * 4, L4 = (size_t)l->cfg.L_local * 4;
  if (dW && Lk) FF_CUDA(cudaMemcpyAsync(dW, l->dW, Lk, cudaMemcpyDeviceToDevice, st));
  if (db && L4) FF_CUDA(cudaMemcpyAsync(db, l->db, L4, cudaMemcpyDeviceToDevice, st));
  return FF_OK;
}

ff_status fixedfanin_adam_step(ff_layer* l, float lr, ff_stream_t stream) {
  g_launches = 0;
  if (!l) return fail(FF_ERR_ARG, "layer is NULL");
  if (!l->grads_valid) return fail(FF_ERR_STATE, "adam_step without a preceding backward");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  l->t += 1;
  const int64_t n = l->cfg.L_local * l->cfg.k;
  k_step_t<<<1, 32, 0, st>>>(l->t_dev, l->rbc_dev, l->cfg.beta1, l->cfg.beta2);
  FF_LAUNCHED();
  if (n > 0) {
    k_adam<<<l->nsm * 8, 256, 0, st>>>(l->W, l->mW, l->vW, l->dW, n, l->bias, l->mb, l->vb, l->db, l->cfg.L_local,
                                       adam_args(l, lr, l->t), l->rbc_dev);
    FF_LAUNCHED();
  }
  l->grads_valid = false;
  return FF_OK;
}

ff_status fixedfanin_train_step(ff_layer* l, const float* h, int32_t B, const int32_t* lbl_ptr,
                                const int32_t* lbl_ids, float grad_scale, float lr, float* dh, float* loss,
                                ff_stream_t stream) {
  g_launches = 0;
  if (!l) return fail(FF_ERR_ARG, "layer is NULL");
  return train_step_impl(l, h, B, lbl_ptr, lbl_ids, grad_scale, lr, dh, loss, reinterpret_cast<cudaStream_t>(stream));
}

ff_status fixedfanin_train_step_host(ff_layer* l, const float* h_host, int32_t B, const int32_t* lbl_ptr_host,
                                     const int32_t* lbl_ids_host, float grad_scale, float lr, float* dh_host,
                                     float* loss_host, ff_stream_t stream) {
  g_launches = 0;
  if (!l) return fail(FF_ERR_ARG, "layer is NULL");
  if (B < 0 || B > l->cfg.max_batch) return fail(FF_ERR_ARG, "B=%d outside [0, max_batch=%d]", B, l->cfg.max_batch);
  if (!lbl_ptr_host || (B > 0 && !h_host)) return fail(FF_ERR_ARG, "null host input");
  const int nnz = lbl_ptr_host[B];
  if (nnz < 0 || nnz > l->cfg.max_nnz) return fail(FF_ERR_ARG, "lbl_ptr[B]=%d outside [0, max_nnz=%d]", nnz, l->cfg.max_nnz);
  if (nnz > 0 && !lbl_ids_host) return fail(FF_ERR_ARG, "null lbl_ids_host");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (!l->copy_st) {
    FF_CUDA(cudaStreamCreateWithFlags(&l->copy_st, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      FF_CUDA(cudaEventCreateWithFlags(&l->ev_ready[i], cudaEventDisableTiming));
      FF_CUDA(cudaEventCreateWithFlags(&l->ev_free[i], cudaEventDisableTiming));
    }
  }
  // staging slot of this call: its previous user (two calls ago) must have finished reading it
  const int slot = l->stage_slot;
  l->stage_slot ^= 1;
  float* h_stage = l->h_stage + (size_t)slot * l->cfg.max_batch * l->cfg.m;
  int* lbl_stage = l->lbl_stage + (size_t)slot * ((size_t)l->cfg.max_batch + 1 + (size_t)l->cfg.max_nnz);
  const size_t hb = (size_t)B * l->cfg.m * 4;
  FF_CUDA(cudaStreamWaitEvent(l->copy_st, l->ev_free[slot], 0));
  if (hb) FF_CUDA(cudaMemcpyAsync(h_stage, h_host, hb, cudaMemcpyHostToDevice, l->copy_st));
  FF_CUDA(cudaMemcpyAsync(lbl_stage, lbl_ptr_host, 4 * (size_t)(B + 1), cudaMemcpyHostToDevice, l->copy_st));
  if (nnz) FF_CUDA(cudaMemcpyAsync(lbl_stage + B + 1, lbl_ids_host, 4 * (size_t)nnz, cudaMemcpyHostToDevice, l->copy_st));
  FF_CUDA(cudaEventRecord(l->ev_ready[slot], l->copy_st));
  FF_CUDA(cudaStreamWaitEvent(st, l->ev_ready[slot], 0));
  // dh is copied out to [B][m] only when the caller asks for it
  ff_status s = train_step_impl(l, h_stage, B, lbl_stage, lbl_stage + B + 1, grad_scale, lr,
                                dh_host ? l->dh_stage : nullptr, l->loss_scratch, st, false, true);
  int32_t launches = g_launches;
  if (s != FF_OK) return s;
  FF_CUDA(cudaEventRecord(l->ev_free[slot], st));
  if (loss_host) {
    // pinned (page-locked) host memory is device-addressable: one thread stores the loss
    // there right after the step's last kernel, with no copy-engine operation on `stream`
    cudaPointerAttributes pa{};
    const bool pinned = cudaPointerGetAttributes(&pa, loss_host) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
                        pa.devicePointer != nullptr;
    if (!pinned) cudaGetLastError();       // clear a pageable-pointer query error
    if (pinned) {
      k_store_scalar<<<1, 32, 0, st>>>(l->loss_scratch, static_cast<float*>(pa.devicePointer));
      FF_LAUNCHED();
      ++launches;
    } else {
      FF_CUDA(cudaMemcpyAsync(loss_host, l->loss_scratch, 4, cudaMemcpyDeviceToHost, st));
    }
  }
  if (dh_host && hb) FF_CUDA(cudaMemcpyAsync(dh_host, l->dh_stage, hb, cudaMemcpyDeviceToHost, st));
  g_launches = launches;
  return FF_OK;
}

ff_status fixedfanin_redistribute(ff_layer* l, uint64_t step, ff_stream_t stream) {
  g_launches = 0;
  if (!l) return fail(FF_ERR_ARG, "layer is NULL");
  const int p = (int)std::floor((double)l->cfg.prune_frac * (double)l->cfg.k);
  if (p < 1) return fail(FF_ERR_CONFIG, "prune count floor(%g*%d) = %d < 1", l->cfg.prune_frac, l->cfg.k, p);
  if (l->cfg.m - l->cfg.k < p) return fail(FF_ERR_CONFIG, "m - k = %d < prune count %d", l->cfg.m - l->cfg.k, p);
  // stored gradients belong to the pre-call connections (a regrown slot's dW would be applied
  // to a different column): invalidate them in every dh mode
  l->grads_valid = false;
  if (l->cfg.L_local == 0) return FF_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  (l->cfg.k > 32 ? k_redistribute<true> : k_redistribute<false>)<<<l->grid_rows, 256, 0, st>>>(l->W, l->idx, l->mW, l->vW, l->cfg.L_local, l->cfg.row_begin, l->cfg.m,
                                               l->cfg.k, p, (uint32_t)step, (uint32_t)l->cfg.seed,
                                               (uint32_t)(l->cfg.seed >> 32));
  FF_LAUNCHED();
  if (l->csc) return csc_rebuild(l, st);
  return FF_OK;
}

ff_status fixedfanin_predict_topk(ff_layer* l, const float* h, int32_t B, int32_t K, float* scores, int32_t* ids,
                                  ff_stream_t stream) {
  g_launches = 0;
  return predict_impl(l, h, B, K, scores, ids, reinterpret_cast<cudaStream_t>(stream), false);
}

ff_status fixedfanin_score_shortlist(ff_layer* l, const float* h, int32_t B, const int32_t* cand_ptr,
                                     const int32_t* cand_ids, float* scores, ff_stream_t stream) {
  g_launches = 0;
  if (!l) return fail(FF_ERR_ARG, "layer is NULL");
  if (B < 0) return fail(FF_ERR_ARG, "B=%d < 0", B);
  if (B == 0) return FF_OK;
  // cand_ids / scores are only dereferenced for existing entries (NULL allowed if cand_ptr[B] == 0)
  if (!h || !cand_ptr) return fail(FF_ERR_ARG, "null h/cand_ptr");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int k = l->cfg.k;
  // the same NG the warp kernels use for this k (predict_kernel / row_kernel_csc)
  const void* fn = k == 64 ? (const void*)k_shortlist<16> : k > 32 ? (const void*)k_shortlist<16>
                 : k == 32 ? (const void*)k_shortlist<8> : k <= 16 ? (const void*)k_shortlist<4>
                 : (const void*)k_shortlist<8>;
  {
    const float* W = l->W; const int* idx = l->idx; const float* bias = l->bias;
    int64_t m = l->cfg.m, L = l->cfg.L_local, rb = l->cfg.row_begin, Lg = l->cfg.L_global;
    int kk = k, BB = B;
    int* err = l->err;
    void* args[] = {&W, &idx, &bias, &h, &m, &kk, &L, &rb, &Lg, &BB, &cand_ptr, &cand_ids, &scores, &err};
    const int grid = std::max(1, std::min((B + 7) / 8, 8 * l->nsm));
    FF_CUDA(cudaLaunchKernel(fn, dim3(grid), dim3(256), args, 0, st));
    ++g_launches;
  }
  return FF_OK;
}

ff_status fixedfanin_precision_at_k(const int32_t* ids, int32_t B, int32_t K, const int32_t* lbl_ptr,
                                    const int32_t* lbl_ids, int32_t* hits, float* mean, ff_stream_t stream) {
  g_launches = 0;
  if (B < 0 || K < 1 || K > 32) return fail(FF_ERR_ARG, "B=%d / K=%d outside B >= 0, 1 <= K <= 32", B, K);
  if (!lbl_ptr || (B > 0 && !ids) || (!hits && !mean)) return fail(FF_ERR_ARG, "null ids/lbl_ptr, or no output");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  k_precision_at_k<<<1, 256, 0, st>>>(ids, B, K, lbl_ptr, lbl_ids, hits, mean);
  FF_LAUNCHED();
  return FF_OK;
}

ff_status fixedfanin_merge_topk(const float* in_s, const int32_t* in_i, int32_t P, int32_t B, int32_t K, float* out_s,
                                int32_t* out_i, ff_stream_t stream) {
  g_launches = 0;
  if (P < 1 || P > 1024 || B < 0 || K < 1 || K > FF_MAX_TOPK) return fail(FF_ERR_ARG, "bad P/B/K");
  if (B == 0) return FF_OK;
  if (!in_s || !in_i || !out_s || !out_i) return fail(FF_ERR_ARG, "null pointer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  k_merge_topk<<<(B + 7) / 8, 256, 0, st>>>(in_s, in_i, P, (int64_t)B * K, K, K, B, K, out_s, out_i);
  FF_LAUNCHED();
  return FF_OK;
}

ff_status fixedfanin_profile_begin(ff_layer* l, int32_t max_launches) {
  g_launches = 0;
  if (!l || max_launches < 1) return fail(FF_ERR_ARG, "layer NULL or max_launches < 1");
  for (cudaEvent_t e : l->prof_ev) cudaEventDestroy(e);
  l->prof_ev.assign(2 * (size_t)max_launches, nullptr);
  for (auto& e : l->prof_ev) FF_CUDA(cudaEventCreate(&e));
  l->prof_used = 0;
  l->prof_paused = false;
  return FF_OK;
}

ff_status fixedfanin_profile_pause(ff_layer* l, int32_t paused) {
  g_launches = 0;
  if (!l) return fail(FF_ERR_ARG, "layer is NULL");
  l->prof_paused = paused != 0;
  return FF_OK;
}

ff_status fixedfanin_profile_end(ff_layer* l, double* ms, int32_t* launches) {
  g_launches = 0;
  if (!l || !ms || !launches) return fail(FF_ERR_ARG, "null argument");
  double total = 0.0;
  if (l->prof_used > 0) FF_CUDA(cudaEventSynchronize(l->prof_ev[2 * l->prof_used - 1]));
  for (int i = 0; i < l->prof_used; ++i) {
    float t = 0.0f;
    FF_CUDA(cudaEventElapsedTime(&t, l->prof_ev[2 * i], l->prof_ev[2 * i + 1]));
    total += t;
  }
  *ms = total;
  *launches = l->prof_used;
  for (cudaEvent_t e : l->prof_ev) cudaEventDestroy(e);
  l->prof_ev.clear();
  l->prof_used = 0;
  return FF_OK;
}

ff_status fixedfanin_check(ff_layer* l, ff_stream_t stream) {
  g_launches = 0;
  if (!l) return fail(FF_ERR_ARG, "layer is NULL");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int herr = 0;
  FF_CUDA(cudaMemcpyAsync(&herr, l->err, sizeof(int), cudaMemcpyDeviceToHost, st));
  FF_CUDA(cudaStreamSynchronize(st));
  FF_CUDA(cudaGetLastError());
  if (herr) FF_CUDA(cudaMemsetAsync(l->err, 0, sizeof(int), st));
  if (herr & kErrLabelRange) return fail(FF_ERR_RANGE, "a label id was outside [0, L_global=%lld)", (long long)l->cfg.L_global);
  if (herr & kErrNonFinite) return fail(FF_ERR_NONFINITE, "non-finite score seen (FF_FLAG_CHECK_FINITE)");
  return FF_OK;
}


// ============================================================ NEXT-2: the intermediate layer
ff_status fixedfanin_dense_workspace_size(const ff_dense_config* cfg, size_t* bytes) {
  g_launches = 0;
  ff_status s = dense_validate(cfg);
  if (s != FF_OK) return s;
  if (!bytes) return fail(FF_ERR_ARG, "bytes is NULL");
  *bytes = dense_layout_of(dense_defaults(*cfg)).total;
  return FF_OK;
}

ff_status fixedfanin_dense_create(const ff_dense_config* cfg, void* workspace, size_t bytes, ff_stream_t stream,
                                  ff_dense** out) {
  g_launches = 0;
  ff_status s = dense_validate(cfg);
  if (s != FF_OK) return s;
  if (!out || !workspace) return fail(FF_ERR_ARG, "out/workspace is NULL");
  if (reinterpret_cast<uintptr_t>(workspace) % kAlign) return fail(FF_ERR_ARG, "workspace not 256-B aligned");
  const ff_dense_config c = dense_defaults(*cfg);
  const DenseLayout lay = dense_layout_of(c);
  if (bytes < lay.total) return fail(FF_ERR_ARG, "workspace %zu B < required %zu B", bytes, lay.total);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  FF_CUDA(cudaGetLastError());
  ff_dense* n = new (std::nothrow) ff_dense();
  if (!n) return fail(FF_ERR_ARG, "host allocation failed");
  n->cfg = c; n->lay = lay;
  char* ws = static_cast<char*>(workspace);
  n->ws = ws;
  n->Wd = at<float>(ws, lay.Wd); n->mWd = at<float>(ws, lay.mWd); n->vWd = at<float>(ws, lay.vWd);
  n->dWd = (c.flags & FF_FLAG_STORE_GRADS) ? at<float>(ws, lay.dWd) : nullptr;
  n->bd = at<float>(ws, lay.bd); n->mbd = at<float>(ws, lay.mbd); n->vbd = at<float>(ws, lay.vbd);
  n->dbd = at<float>(ws, lay.dbd);
  n->xT = at<float>(ws, lay.xT); n->xTlo = at<float>(ws, lay.xTlo); n->hd = at<float>(ws, lay.hd); n->x_stage = at<float>(ws, lay.x_stage);
  n->t_dev = at<int64_t>(ws, lay.scal); n->rbc_dev = at<float>(ws, lay.scal + 8);
  n->zpart = at<float>(ws, lay.zpart); n->cnt = at<unsigned>(ws, lay.cnt);
  n->ldw = ldw_of(c.m);
  n->t = 0; n->fwd_B = -1; n->grads_valid = false;
  {
    int dev = 0;
    cudaError_t e2 = cudaGetDevice(&dev);
    if (e2 == cudaSuccess) e2 = cudaDeviceGetAttribute(&n->nsm, cudaDevAttrMultiProcessorCount, dev);
    if (e2 != cudaSuccess) { delete n; return fail(FF_ERR_CUDA, "device query: %s", cudaGetErrorString(e2)); }
  }
  if (cudaFuncSetAttribute((const void*)k_dense_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, kDenseFwdSmem) !=
          cudaSuccess ||
      cudaFuncSetAttribute((const void*)k_dense_bwd_adam_b32, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kDenseBwd1Smem) != cudaSuccess ||
      cudaFuncSetAttribute((const void*)k_dense_fwd_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmSmem) !=
          cudaSuccess) {
    delete n;
    return fail(FF_ERR_CUDA, "dense forward smem attribute");
  }
  n->grid_bwd32 = occupancy_grid((const void*)k_dense_bwd_adam_b32, n->nsm, kDenseBwd32Threads, kDenseBwd1Smem);
  {
    // TMA maps (128-B swizzle with 32-B atoms: the MN-major tf32 operand layout, ff_dense.cuh)
    const char* why = encode_dense_maps(n);
    if (why) { delete n; return fail(FF_ERR_CUDA, "dense forward tensor maps: %s", why); }
  }
  cudaError_t e = cudaMemsetAsync(ws, 0, lay.total, st);
  if (e != cudaSuccess) { delete n; return fail(FF_ERR_CUDA, "memset: %s", cudaGetErrorString(e)); }
  const int64_t work = (int64_t)c.d * (n->ldw / 4);
  k_dense_init<<<(int)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 8192)), 256, 0, st>>>(
      n->Wd, c.d, c.m, n->ldw, c.col_begin, (uint32_t)c.seed, (uint32_t)(c.seed >> 32), c.init_scale);
  e = cudaGetLastError();
  if (e != cudaSuccess) { delete n; return fail(FF_ERR_CUDA, "init launch: %s", cudaGetErrorString(e)); }
  ++g_launches;
  *out = n;
  return FF_OK;
}

ff_status fixedfanin_dense_destroy(ff_dense* n) {
  delete n;
  return FF_OK;
}

ff_status fixedfanin_dense_set_params(ff_dense* n, const float* Wd, const float* bd, const float* mWd,
                                      const float* vWd, const float* mbd, const float* vbd, const int64_t* t,
                                      ff_stream_t stream) {
  g_launches = 0;
  if (!n) return fail(FF_ERR_ARG, "dense layer is NULL");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t m4 = 4 * (size_t)n->cfg.m;
  const int64_t dm = (int64_t)n->cfg.d * n->cfg.m;
  const int rg = (int)std::max<int64_t>(1, std::min<int64_t>((dm + 255) / 256, 8192));
  auto cp2 = [&](float* dst, const float* src) -> cudaError_t {   // [d][m] -> tiled
    if (!src) return cudaSuccess;
    k_dense_retile<<<rg, 256, 0, st>>>(src, dst, n->cfg.d, n->cfg.m, 1);
    return cudaGetLastError();
  };
  auto cp1 = [&](float* dst, const float* src) -> cudaError_t {
    return src ? cudaMemcpyAsync(dst, src, m4, cudaMemcpyDeviceToDevice, st) : cudaSuccess;
  };
  FF_CUDA(cp2(n->Wd, Wd)); FF_CUDA(cp2(n->mWd, mWd)); FF_CUDA(cp2(n->vWd, vWd));
  FF_CUDA(cp1(n->bd, bd)); FF_CUDA(cp1(n->mbd, mbd)); FF_CUDA(cp1(n->vbd, vbd));
  if (t) {
    n->t = *t;
    FF_CUDA(cudaMemcpyAsync(n->t_dev, &n->t, sizeof(int64_t), cudaMemcpyHostToDevice, st));
  }
  n->grads_valid = false;
  FF_CUDA(cudaStreamSynchronize(st));
  return FF_OK;
}

ff_status fixedfanin_dense_get_params(ff_dense* n, float* Wd, float* bd, float* mWd, float* vWd, float* mbd,
                                      float* vbd, int64_t* t, ff_stream_t stream) {
  g_launches = 0;
  if (!n) return fail(FF_ERR_ARG, "dense layer is NULL");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t m4 = 4 * (size_t)n->cfg.m;
  const int64_t dm = (int64_t)n->cfg.d * n->cfg.m;
  const int rg = (int)std::max<int64_t>(1, std::min<int64_t>((dm + 255) / 256, 8192));
  auto cp2 = [&](float* dst, const float* src) -> cudaError_t {   // tiled -> [d][m]
    if (!dst) return cudaSuccess;
    k_dense_retile<<<rg, 256, 0, st>>>(src, dst, n->cfg.d, n->cfg.m, 0);
    return cudaGetLastError();
  };
  auto cp1 = [&](float* dst, const float* src) -> cudaError_t {
    return dst ? cudaMemcpyAsync(dst, src, m4, cudaMemcpyDeviceToDevice, st) : cudaSuccess;
  };
  FF_CUDA(cp2(Wd, n->Wd)); FF_CUDA(cp2(mWd, n->mWd)); FF_CUDA(cp2(vWd, n->vWd));
  FF_CUDA(cp1(bd, n->bd)); FF_CUDA(cp1(mbd, n->mbd)); FF_CUDA(cp1(vbd, n->vbd));
  if (t) FF_CUDA(cudaMemcpyAsync(t, n->t_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FF_CUDA(cudaStreamSynchronize(st));
  if (t) n->t = *t;
  return FF_OK;
}

ff_status fixedfanin_dense_forward(ff_dense* n, const float* x, int32_t B, uint64_t step, int32_t train, float* h,
                                   ff_stream_t stream) {
  g_launches = 0;
  if (!n) return fail(FF_ERR_ARG, "dense layer is NULL");
  if (B < 0 || B > n->cfg.max_batch) return fail(FF_ERR_ARG, "B=%d outside [0, max_batch=%d]", B, n->cfg.max_batch);
  if (B == 0) return FF_OK;
  if (!x) return fail(FF_ERR_ARG, "null x");
  return dense_forward_impl(n, x, B, step, train != 0, n->hd, h, reinterpret_cast<cudaStream_t>(stream));
}

ff_status fixedfanin_dense_backward_adam(ff_dense* n, const float* dh, int32_t B, float lr, ff_stream_t stream) {
  g_launches = 0;
  if (!n) return fail(FF_ERR_ARG, "dense layer is NULL");
  if (n->fwd_B < 0) return fail(FF_ERR_STATE, "dense backward without a preceding training forward");
  if (B != n->fwd_B) return fail(FF_ERR_ARG, "B=%d differs from the forward's B=%d", B, n->fwd_B);
  if (B > 0 && !dh) return fail(FF_ERR_ARG, "null dh");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int nb = nb_of(B);
  if (B > 0) {
    dim3 grid((n->cfg.m + 31) / 32, nb), block(32, 8);
    k_dh_in<<<grid, block, 0, st>>>(dh, B, n->cfg.m, nb, n->hd);
    FF_LAUNCHED();
  }
  const int32_t pre = g_launches;
  ff_status s = dense_backward_impl(n, std::max(B, 1), lr, n->hd, st);
  g_launches += pre;
  return s;
}

ff_status fixedfanin_dense_get_grads(ff_dense* n, float* dWd, float* dbd, ff_stream_t stream) {
  g_launches = 0;
  if (!n) return fail(FF_ERR_ARG, "dense layer is NULL");
  if (!n->grads_valid) return fail(FF_ERR_STATE, "no gradients: create with FF_FLAG_STORE_GRADS and run a backward");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t m4 = 4 * (size_t)n->cfg.m;
  const int64_t dm = (int64_t)n->cfg.d * n->cfg.m;
  if (dWd) {
    k_dense_retile<<<(int)std::max<int64_t>(1, std::min<int64_t>((dm + 255) / 256, 8192)), 256, 0, st>>>(
        n->dWd, dWd, n->cfg.d, n->cfg.m, 0);
    FF_CUDA(cudaGetLastError());
  }
  if (dbd) FF_CUDA(cudaMemcpyAsync(dbd, n->dbd, m4, cudaMemcpyDeviceToDevice, st));
  return FF_OK;
}

ff_status fixedfanin_model_train_step(ff_dense* n, ff_layer* l, const float* x, int32_t B, uint64_t step,
                                      const int32_t* lbl_ptr, const int32_t* lbl_ids, float grad_scale, float lr,
                                      float* loss, ff_stream_t stream) {
  g_launches = 0;
  if (!n || !l) return fail(FF_ERR_ARG, "dense layer / layer is NULL");
  if (n->cfg.m != l->cfg.m) return fail(FF_ERR_CONFIG, "dense m=%d != layer m=%d", n->cfg.m, l->cfg.m);
  if (l->cfg.L_local != l->cfg.L_global)
    return fail(FF_ERR_CONFIG, "model step needs an unsharded layer (sharded: dense_forward, train_step, "
                               "all-reduce dh, dense_backward_adam)");
  if (B < 0 || B > n->cfg.max_batch || B > l->cfg.max_batch) return fail(FF_ERR_ARG, "B=%d outside max_batch", B);
  if (B == 0) return FF_OK;
  if (!x || !lbl_ptr) return fail(FF_ERR_ARG, "null x/lbl_ptr");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  ff_status s = dense_forward_impl(n, x, B, step, true, l->hd, nullptr, st);
  if (s != FF_OK) return s;
  int32_t nl = g_launches;
  const DenseT dt{n->t_dev, n->rbc_dev, n->cfg.beta1, n->cfg.beta2};
  s = train_step_impl(l, nullptr, B, lbl_ptr, lbl_ids, grad_scale, lr, nullptr, loss, st, true, false, &dt);
  if (s != FF_OK) return s;
  nl += g_launches;
  s = dense_backward_impl(n, B, lr, l->hd, st, true);
  g_launches += nl;
  return s;
}

ff_status fixedfanin_model_predict_topk(ff_dense* n, ff_layer* l, const float* x, int32_t B, int32_t K,
                                        float* scores, int32_t* ids, ff_stream_t stream) {
  g_launches = 0;
  if (!n || !l) return fail(FF_ERR_ARG, "dense layer / layer is NULL");
  if (n->cfg.m != l->cfg.m) return fail(FF_ERR_CONFIG, "dense m=%d != layer m=%d", n->cfg.m, l->cfg.m);
  if (B < 0 || B > n->cfg.max_batch || B > l->cfg.max_batch) return fail(FF_ERR_ARG, "B=%d outside max_batch", B);
  if (B == 0) return FF_OK;
  if (!x) return fail(FF_ERR_ARG, "null x");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  ff_status s = dense_forward_impl(n, x, B, 0, false, l->hd, nullptr, st);
  if (s != FF_OK) return s;
  const int32_t nl = g_launches;
  s = predict_impl(l, nullptr, B, K, scores, ids, st, true);
  g_launches += nl;
  return s;
}

}  // extern "C"
