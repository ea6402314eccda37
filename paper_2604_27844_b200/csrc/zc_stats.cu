// K1 — statistics + on-device codebook derivation.
//
// Reference: bf16.measure_sigma (bf16.py:88-103: np.std, ddof=0, over the
// finite elements in f64) feeding codec.codebook_for (codec.py:164-185) and
// derive_codebook / window_coverage / optimal_base_exponent (:74-161).
//
// stats_kernel: one 4096-element tile per CTA over the concatenation of up to
// kMaxSegments segments (the non-self chunks of an all-to-all, reference
// collectives._prepare_frames :230-242).  Per warp the shift K is the warp's
// first finite value; sums of d = x-K and d^2 are exact-ish in f64, so a
// constant buffer yields exactly M2 = 0 (the modal-fallback trigger).  Warp
// and CTA partials are merged with Chan's pairwise formula in a fixed order;
// finalize_kernel merges the CTA partials in a fixed tree, so the result is
// deterministic run to run.
//
// finalize_kernel derives the 7-entry window exactly like the reference
// (floor/ceil of log2(sigma) + BASE_EXPONENT_OFFSET, coverage comparison by
// erf, tie to floor, clamp base into [-126, 121]).  When sigma is 0 or no
// finite value exists, the finite values are all equal (or absent), so the
// exponent histogram has at most two non-empty bins -- the common finite
// exponent and 255 -- and the modal rule (first argmax) is evaluated from
// the counts without a histogram pass.
//
// hist_kernel + mode_kernel: the general modal fallback when a caller passes
// an explicit sigma that is 0 / negative / non-finite (reference codec.py:179-185
// over arbitrary data).
#include <cmath>
#include "zc_stats.cuh"

namespace zc {

__device__ void finalize_block(const Partial* parts, int64_t nparts, int64_t total_words,
                               uint8_t* book, double* result);

// Persistent: each CTA owns a contiguous run of tiles of the concatenated
// segments and keeps a kSStages-deep ring of 8 KB tiles in flight with TMA
// bulk copies; thread 0 issues, all threads accumulate.  The last CTA to
// finish merges every partial in a fixed order and derives the codebook.
constexpr int kSStages = 4;
constexpr int kSStageBytes = kTile * 2;

__device__ __forceinline__ void stats_issue(const uint16_t* x, const StatSegs& segs,
                                            int64_t tile, uint8_t* stage, uint64_t* bar) {
  const int s = find_seg(segs.tile_start, segs.nseg, tile);
  const uint16_t* xs = x + segs.x_off[s];
  const int64_t base = (tile - segs.tile_start[s]) * kTile;
  const int64_t valid = segs.n[s] - base;
  const uint32_t bytes = (uint32_t)((valid >= kTile ? kTile : valid) * 2) & ~15u;
  if (((reinterpret_cast<uintptr_t>(xs) & 15) == 0) && bytes > 0) {
    mbar_arrive_expect_tx(bar, bytes);
    tma_load_1d(stage, xs + base, bytes, bar);
  } else {
    mbar_arrive(bar);
  }
}

__global__ void __launch_bounds__(kThreads)
stats_kernel(const uint16_t* __restrict__ x, const StatSegs segs,
             Partial* __restrict__ out, unsigned* __restrict__ done, int64_t total_words,
             uint8_t* __restrict__ book, double* __restrict__ result,
             const int* __restrict__ need) {
  // fallback launch behind the certified pass: nothing to do when it decided
  if (need != nullptr && *need == 0) return;
  extern __shared__ __align__(128) uint8_t s_dyn[];
  uint8_t* ring = s_dyn;
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_dyn + kSStages * kSStageBytes);
  const int tid = threadIdx.x;
  const int64_t ntiles = segs.tile_start[segs.nseg];
  const int64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t i0 = blockIdx.x * per;
  const int64_t i1 = (i0 + per < ntiles) ? i0 + per : ntiles;
  if (tid == 0) {
    for (int k = 0; k < kSStages; ++k) mbar_init(bars + k, 1);
    fence_mbar_init();
    for (int k = 0; k < kSStages && i0 + k < i1; ++k)
      stats_issue(x, segs, i0 + k, ring + k * kSStageBytes, bars + k);
  }
  __syncthreads();
  StatAcc acc;
  for (int64_t i = i0; i < i1; ++i) {
    const int k = (int)(i - i0);
    const int st = k & (kSStages - 1);
    const int64_t tile = i;
    const int sg = find_seg(segs.tile_start, segs.nseg, tile);
    const uint16_t* xs = x + segs.x_off[sg];
    const int64_t base = (tile - segs.tile_start[sg]) * kTile;
    const int64_t tvalid = segs.n[sg] - base;
    const int tma_elems = ((reinterpret_cast<uintptr_t>(xs) & 15) == 0)
        ? (int)((((tvalid >= kTile ? kTile : tvalid) * 2) & ~15) / 2) : 0;
    mbar_wait_warp(bars + st, (uint32_t)((k / kSStages) & 1));
    const uint16_t* tw = reinterpret_cast<const uint16_t*>(ring + st * kSStageBytes);
    uint32_t w[8];
    uint32_t valid = 0xFFFFu;
    if (tid * kEPT + kEPT <= tma_elems) {
      const uint4 a = *reinterpret_cast<const uint4*>(tw + tid * kEPT);
      const uint4 b = *reinterpret_cast<const uint4*>(tw + tid * kEPT + 8);
      w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
      w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
    } else {
      const int64_t nvalid = tvalid - (int64_t)tid * kEPT;
      valid = nvalid >= kEPT ? 0xFFFFu : (nvalid > 0 ? ((1u << nvalid) - 1u) : 0u);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int e0 = tid * kEPT + 2 * j;
        uint32_t lo = 0, hi = 0;
        if (2 * j < nvalid) lo = (e0 < tma_elems) ? tw[e0] : xs[base + e0];
        if (2 * j + 1 < nvalid) hi = (e0 + 1 < tma_elems) ? tw[e0 + 1] : xs[base + e0 + 1];
        w[j] = lo | (hi << 16);
      }
    }
    acc.add16(w, valid);
    __syncthreads();                                   // stage free
    if (tid == 0 && i + kSStages < i1) {
      fence_proxy_async();
      stats_issue(x, segs, i + kSStages, ring + st * kSStageBytes, bars + st);
    }
  }
  stat_block_finish(acc, out + blockIdx.x);
  // the last CTA to finish merges every partial (fixed order) and derives the
  // codebook: no separate finalize launch
  __shared__ bool s_last;
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    finalize_block(out, gridDim.x, total_words, book, result);
    np_refine_near_flip(x, &segs, total_words, book, result, true);
  }
}

static size_t stats_dyn_smem() { return kSStages * kSStageBytes + kSStages * sizeof(uint64_t); }

static int stats_grid_cap() {
  static int caps[kMaxDevices];
  return per_device(caps, [] {
    cudaFuncSetAttribute(stats_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)stats_dyn_smem());
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stats_kernel, kThreads, stats_dyn_smem());
    return sms * (occ > 0 ? occ : 1);
  });
}

// Fixed-order merge of `nparts` partials by one kThreads-thread CTA (each
// thread a contiguous range, then a fixed binary tree), then the reference
// derivation.  result[0] = sigma (NaN when no finite value), result[1] =
// finite count, result[2] = path (1 analytic, 2 modal), book = 7 entries.
__device__ void finalize_block(const Partial* parts, int64_t nparts, int64_t total_words,
                               uint8_t* book, double* result) {
  __shared__ double f_n[kWarps], f_m[kWarps], f_q[kWarps];
  __shared__ int f_e[kWarps];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t per = (nparts + kThreads - 1) / kThreads;
  double na = 0.0, ma = 0.0, qa = 0.0;
  int e = -1;
  for (int64_t i = t * per; i < (t + 1) * per && i < nparts; ++i) {
    const double c = __ldcg(&parts[i].count), m = __ldcg(&parts[i].mean);
    const double q = __ldcg(&parts[i].m2), a = __ldcg(&parts[i].aux);
    chan_merge(na, ma, qa, c, m, q);
    if (e < 0) e = (int)a;
  }
  // fixed pairwise tree inside the warp (lane i absorbs lane i+o)
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double nb = __shfl_down_sync(0xffffffffu, na, o);
    const double mb = __shfl_down_sync(0xffffffffu, ma, o);
    const double qb = __shfl_down_sync(0xffffffffu, qa, o);
    const int eb = __shfl_down_sync(0xffffffffu, e, o);
    if ((lane & (2 * o - 1)) == 0) {
      chan_merge(na, ma, qa, nb, mb, qb);
      if (e < 0) e = eb;
    }
  }
  if (lane == 0) { f_n[warp] = na; f_m[warp] = ma; f_q[warp] = qa; f_e[warp] = e; }
  __syncthreads();
  if (t == 0) {
    double cn = 0.0, cm = 0.0, cq = 0.0;
    int ce = -1;
    for (int i = 0; i < kWarps; ++i) {
      chan_merge(cn, cm, cq, f_n[i], f_m[i], f_q[i]);
      if (ce < 0) ce = f_e[i];
    }
    finish_codebook(cn, cq, ce, total_words, book, result);
  }
}

__global__ void __launch_bounds__(kThreads)
finalize_kernel(const Partial* __restrict__ parts, int64_t nparts, int64_t total_words,
                uint8_t* __restrict__ book, double* __restrict__ result) {
  finalize_block(parts, nparts, total_words, book, result);
}


// No TMA ring and no block barrier here: with ~3 instructions per element the
// kernel is latency-bound on loads, and plain 16-B loads of two tiles per
// iteration (64 B in flight per thread, occupancy-sized grid) measured
// 5.87 TB/s vs 5.51 for a 4-stage TMA ring and 5.73 for four tiles.
__device__ __forceinline__ void sums_load16(const uint16_t* __restrict__ x, const StatSegs& segs,
                                            int64_t tile, int tid, uint32_t kw, uint32_t* w) {
  const int sg = find_seg(segs.tile_start, segs.nseg, tile);
  const uint16_t* xs = x + segs.x_off[sg];
  const int64_t base = (tile - segs.tile_start[sg]) * kTile + (int64_t)tid * kEPT;
  const int64_t nvalid = segs.n[sg] - base;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    uint32_t lo = kw, hi = kw;                             // d = 0 outside the segment
    if (2 * j < nvalid) lo = xs[base + 2 * j];
    if (2 * j + 1 < nvalid) hi = xs[base + 2 * j + 1];
    w[j] = lo | (hi << 16);
  }
}


__device__ __forceinline__ void ld_pair(const uint16_t* p, bool a32, uint4& a, uint4& b) {
  if (a32) {
    ld_stream_v8(p, a, b);
  } else {
    a = ld_stream_v4(p);
    b = ld_stream_v4(p + 8);
  }
}

__global__ void __launch_bounds__(kThreads)
sums_kernel(const uint16_t* __restrict__ x, const StatSegs segs, SumPartial* __restrict__ out,
                   unsigned* __restrict__ done, int64_t total, uint8_t* __restrict__ book,
                   double* __restrict__ result, int* __restrict__ need) {
  const int tid = threadIdx.x;
  const int64_t ntiles = segs.tile_start[segs.nseg];
  const int64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t i0 = blockIdx.x * per;
  const int64_t i1 = (i0 + per < ntiles) ? i0 + per : ntiles;
  uint32_t kw = x[segs.x_off[0]];
  if ((kw & 0x7F80u) == 0x7F80u) kw = 0;
  const uint32_t kpair = kw | (kw << 16);
  const uint64_t K2 = (uint64_t)(kpair & 0xFFFF0000u) << 32 | (uint64_t)(kpair << 16);
  // single aligned segment: every full tile is one 32-B load per thread
  // (two 16-B loads when the segment is only 16-B aligned)
  const uintptr_t xa = reinterpret_cast<uintptr_t>(x + segs.x_off[0]);
  const bool flat = segs.nseg == 1 && (xa & 15) == 0;
  const bool a32 = (xa & 31) == 0;
  const int64_t nfull = flat ? segs.n[0] / kTile : 0;
  const uint16_t* x0 = x + segs.x_off[0] + tid * kEPT;
  double s1 = 0.0, s2 = 0.0;
  int64_t i = i0;
  const int64_t fend = nfull < i1 ? nfull : i1;
  for (; i + 2 <= fend; i += 2) {
    uint4 a, b, c, d;
    ld_pair(x0 + i * kTile, a32, a, b);
    ld_pair(x0 + (i + 1) * kTile, a32, c, d);
    const uint32_t wa[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    const uint32_t wc[8] = {c.x, c.y, c.z, c.w, d.x, d.y, d.z, d.w};
    sums_acc16(wa, K2, s1, s2);
    sums_acc16(wc, K2, s1, s2);
  }
  for (; i < i1; ++i) {
    uint32_t w[8];
    if (i < nfull) {
      uint4 a, b;
      ld_pair(x0 + i * kTile, a32, a, b);
      w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
      w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
    } else {
      sums_load16(x, segs, i, tid, kw, w);
    }
    sums_acc16(w, K2, s1, s2);
  }
  __shared__ double b_1[kWarps], b_2[kWarps];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s1 += __shfl_down_sync(0xffffffffu, s1, o);
    s2 += __shfl_down_sync(0xffffffffu, s2, o);
  }
  if ((tid & 31) == 0) { b_1[tid >> 5] = s1; b_2[tid >> 5] = s2; }
  __syncthreads();
  __shared__ bool s_last;
  if (tid == 0) {
    double t1 = 0.0, t2 = 0.0;
    for (int k = 0; k < kWarps; ++k) { t1 += b_1[k]; t2 += b_2[k]; }
    out[blockIdx.x] = SumPartial{t1, t2};
    __threadfence();
    s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    certify_block(out, gridDim.x, total, book, result, need);
  }
}

static int sums_grid_cap() {
  static int caps[kMaxDevices];
  return per_device(caps, [] {
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sums_kernel, kThreads, 0);
    return sms * (occ > 0 ? occ : 1);
  });
}


__global__ void __launch_bounds__(kThreads)
hist_kernel(const uint16_t* __restrict__ x, const StatSegs segs, unsigned long long* __restrict__ hist) {
  __shared__ unsigned s_h[kWarps][256];
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < kWarps * 256; i += kThreads) (&s_h[0][0])[i] = 0;
  __syncthreads();
  const int64_t tile = blockIdx.x;
  const int seg = find_seg(segs.tile_start, segs.nseg, tile);
  const int64_t n = segs.n[seg];
  const uint16_t* xs = x + segs.x_off[seg];
  const int64_t base = (tile - segs.tile_start[seg]) * kTile + (int64_t)tid * kEPT;
  for (int k = 0; k < kEPT; ++k)
    if (base + k < n) atomicAdd(&s_h[warp][(xs[base + k] >> 7) & 0xFF], 1u);
  __syncthreads();
  unsigned v = 0;
  for (int i = 0; i < kWarps; ++i) v += s_h[i][tid];
  if (v) atomicAdd(hist + tid, (unsigned long long)v);
}

__global__ void mode_kernel(const unsigned long long* __restrict__ hist, int64_t total, uint8_t* book) {
  if (threadIdx.x != 0) return;
  int mode = 0;
  for (int i = 1; i < 256; ++i) if (hist[i] > hist[mode]) mode = i;   // first argmax
  const bool all_zero = (mode == 0) && ((int64_t)hist[0] == total);
  write_window(book, all_zero ? -6 : mode - 127 - 3);
}

// Workspace: [64] exact-pass counter, [68] certified-pass counter, [72] need
// flag, [128..) per-CTA partials (both passes; they run one after the other).
// exact != 0: result[0] must be the f64 statistic itself (measure_sigma);
// otherwise the certified pass decides the codebook and the exact kernel
// returns at once unless the certificate failed.
// Small inputs skip the certified pass: the exact kernel alone is one launch
// fewer, and its f64 work is negligible at this size.
constexpr int64_t kSmallExactTiles = 16;


// grid = kNpOwners / kThreads.  Runs only when the exact pass saw every
// element finite and sigma > 0 (and, behind the certificate, when it failed).
// grid = kNpOwners / kThreads (one owner block of 256 per CTA).
template <int kPass>
__global__ void __launch_bounds__(kThreads)
np_sigma_kernel(const uint16_t* __restrict__ x, const StatSegs segs, int64_t total,
                NpWs* __restrict__ w, unsigned* __restrict__ done, uint8_t* __restrict__ book,
                double* __restrict__ result) {
  if (total < 1 || !(__ldcg(result + 1) == (double)total) || !(__ldcg(result) > 0.0)) return;
  constexpr int kLv = 8;                              // log2(kThreads)
  static_assert((1 << kLv) == kThreads, "one owner index per thread");
  const int tid = threadIdx.x;
  const int t = (int)blockIdx.x * kThreads + tid;
  const double mean = kPass ? __ldcg(&w->mean) : 0.0;
  int64_t start = 0, n = total;
  int d = 0;
  bool owner = true;
  for (; d < kNpK; ++d) {
    if (n <= kNpLeaf) {
      owner = (t & ((1 << (kNpK - d)) - 1)) == 0;
      break;
    }
    const int64_t L = np_left(n);
    if ((t >> (kNpK - 1 - d)) & 1) {
      start += L;
      n -= L;
    } else {
      n = L;
    }
  }
  __shared__ double s_val[kThreads];
  __shared__ int8_t s_dep[kThreads];
  double mine = 0.0;
  if (owner) {
    NpCursor c;
    c.init(x, &segs, start, total);
    mine = np_subtree<kPass>(c, start, n, mean);
  }
  s_val[tid] = mine;
  s_dep[tid] = owner ? (int8_t)d : (int8_t)-1;
  w->depth[t] = s_dep[tid];
  __syncthreads();
  // node = left + right, bottom-up, in place at each node's leftmost index:
  // the CTA's 256 owner indices are one subtree (depth kNpK - 8), combined in
  // shared memory; the last CTA combines the CTAs' values above it
  for (int dd = kNpK - 1; dd >= kNpK - kLv; --dd) {
    const int step = 1 << (kNpK - dd);
    if ((tid & (step - 1)) == 0 && s_dep[tid] > dd)
      s_val[tid] = __dadd_rn(s_val[tid], s_val[tid + step / 2]);
    __syncthreads();
  }
  if (tid == 0) w->parts[t] = s_val[0];
  __shared__ bool s_last;
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int dd = kNpK - kLv - 1; dd >= 0; --dd) {
    for (int p = tid; p < (1 << dd); p += kThreads) {
      const int t0 = p << (kNpK - dd);
      if (__ldcg(&w->depth[t0]) > dd)
        w->parts[t0] = __dadd_rn(__ldcg(&w->parts[t0]),
                                 __ldcg(&w->parts[t0 + (1 << (kNpK - dd - 1))]));
    }
    __syncthreads();
  }
  if (tid == 0) {
    *done = 0;                                        // for the next pass / call
    const double v = __ddiv_rn(__dadd_rn(0.0, __ldcg(&w->parts[0])), (double)total);
    if (kPass == 0) {
      w->mean = v;
    } else {
      const double sigma = __dsqrt_rn(v);
      result[0] = sigma;
      if (isfinite(sigma) && sigma > 0.0) {
        write_window(book, derive_base(sigma));
        result[2] = 1.0;
      }
    }
  }
}

// both passes behind the exact statistic (result / book already hold its
// answer); `ws` is the caller's workspace (np area at kNpWsOff).  Run for
// the exact statistic (measure_sigma's flag): codebook_for's certified path
// and the speculative encoder keep the Chan pass, whose codebook is the
// reference's except within ~1e-15 relative of a flip threshold, without
// two extra launches per call.
cudaError_t launch_np_sigma(const uint16_t* x, const StatSegs& segs, int64_t total, void* ws,
                            unsigned* done, uint8_t* book, double* result, cudaStream_t st) {
  if (total < 1) return cudaSuccess;
  NpWs* w = reinterpret_cast<NpWs*>(reinterpret_cast<uint8_t*>(ws) + kNpWsOff);
  np_sigma_kernel<0><<<kNpOwners / kThreads, kThreads, 0, st>>>(x, segs, total, w, done, book,
                                                                result);
  np_sigma_kernel<1><<<kNpOwners / kThreads, kThreads, 0, st>>>(x, segs, total, w, done, book,
                                                                result);
  return cudaGetLastError();
}

cudaError_t launch_codebook_measured(const uint16_t* x, const StatSegs& segs, int64_t total,
                                     void* ws, uint8_t* book, double* result, int exact,
                                     cudaStream_t st, bool zeroed) {
  const int64_t ntiles = segs.tile_start[segs.nseg];
  const int asked = exact;            // measure_sigma's request: numpy's order too
  if (ntiles <= kSmallExactTiles) exact = 1;
  uint8_t* w8 = reinterpret_cast<uint8_t*>(ws);
  Partial* parts = reinterpret_cast<Partial*>(w8 + 128);
  const int cap = stats_grid_cap();
  const int64_t grid = ntiles < cap ? ntiles : cap;
  unsigned* done = reinterpret_cast<unsigned*>(w8 + 64);
  unsigned* done_sums = reinterpret_cast<unsigned*>(w8 + 68);
  int* need = reinterpret_cast<int*>(w8 + 72);
  if (grid > 0) {
    if (!zeroed) {   // else the caller cleared [64, 80) of ws in its own memset
      cudaError_t e = cudaMemsetAsync(done, 0, 16, st);
      if (e != cudaSuccess) return e;
    }
    if (!exact) {
      const int scap = sums_grid_cap();
      const int64_t sgrid = ntiles < scap ? ntiles : scap;
      sums_kernel<<<(unsigned)sgrid, kThreads, 0, st>>>(
          x, segs, reinterpret_cast<SumPartial*>(parts), done_sums, total, book, result, need);
    }
    stats_kernel<<<(unsigned)grid, kThreads, stats_dyn_smem(), st>>>(
        x, segs, parts, done, total, book, result, exact ? nullptr : need);
    // the reference's own summation order for sigma (all-finite inputs)
    if (asked == 1) {
      cudaError_t e = launch_np_sigma(x, segs, total, ws, reinterpret_cast<unsigned*>(w8 + 76),
                                      book, result, st);
      if (e != cudaSuccess) return e;
    }
  } else {
    finalize_kernel<<<1, kThreads, 0, st>>>(parts, 0, total, book, result);
  }
  return cudaGetLastError();
}

cudaError_t launch_codebook_modal(const uint16_t* x, const StatSegs& segs, int64_t total,
                                  void* ws, uint8_t* book, cudaStream_t st) {
  const int64_t ntiles = segs.tile_start[segs.nseg];
  unsigned long long* hist = reinterpret_cast<unsigned long long*>(reinterpret_cast<uint8_t*>(ws) + 128);
  cudaError_t e = cudaMemsetAsync(hist, 0, 256 * sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  if (ntiles > 0) hist_kernel<<<(unsigned)ntiles, kThreads, 0, st>>>(x, segs, hist);
  mode_kernel<<<1, 32, 0, st>>>(hist, total, book);
  return cudaGetLastError();
}

// ---- speculative encoder support (launch_encode_auto) -------------------------
// Guess for the speculative encoder: the analytic codebook of packed-fp32
// sums over a uniform element sample -- one 32-B sector (16 words) from every
// ZC_GTILESKIP-th 4096-word tile, i.e. 1/512 of the bytes by default, spread
// over the whole input so that no region is over-weighted (a tile sample
// would be fooled by a small cluster, e.g. the RMSNorm vectors at the end of
// a layer shard).  No certificate: a wrong guess only costs a re-encode.
// Sample density against the guess's latency (encode leg of the bench layer,
// scripts/exp/guess_time.py): every tile 153.8-154.2 us, every 2nd
// 152.2-152.8, every 4th 152.1-152.8; sigma of the 1/512 sample is within
// ~0.15 % for Gaussian data, so a guess off the certified book (a re-encode,
// ~140 us) needs sigma within ~0.2 % of a base flip: expected cost < 0.5 us.
#ifndef ZC_GSTRIDE
#define ZC_GSTRIDE 4096
#endif
#ifndef ZC_GTILESKIP
#define ZC_GTILESKIP 2
#endif
constexpr int kGuessStride = ZC_GSTRIDE;
constexpr int kGuessTileSkip = ZC_GTILESKIP;
static_assert(kTile % kGuessStride == 0, "probes per tile");
struct GuessPartial {
  double s1, s2, cnt;
};

__global__ void __launch_bounds__(kThreads)
guess_kernel(const uint16_t* __restrict__ x, const StatSegs segs, GuessPartial* __restrict__ parts,
             unsigned* __restrict__ done, uint8_t* __restrict__ guess) {
  grid_dep_launch();   // the encoder behind (PDL) may fill its rings meanwhile
  const int tid = threadIdx.x;
  const int64_t ntiles = segs.tile_start[segs.nseg];
  constexpr int kPerTile = kTile / kGuessStride;
  const int64_t nprobe = (ntiles + kGuessTileSkip - 1) / kGuessTileSkip * kPerTile;
  // shift word K (the first element; every thread reads the same one), read
  // after the first probe's load is in flight: both round trips overlap
  uint32_t kw = 0;
  uint64_t K2 = 0;
  bool have_k = false;
  auto read_k = [&] {
    kw = x[segs.x_off[0]];
    if ((kw & 0x7F80u) == 0x7F80u) kw = 0;
    K2 = sums_shift(kw);
    have_k = true;
  };
  double s1 = 0.0, s2 = 0.0, cnt = 0.0;
  for (int64_t p = (int64_t)blockIdx.x * kThreads + tid; p < nprobe; p += (int64_t)gridDim.x * kThreads) {
    const int64_t tile = p / kPerTile * kGuessTileSkip;
    const int sg = find_seg(segs.tile_start, segs.nseg, tile);
    const int64_t off = (tile - segs.tile_start[sg]) * kTile + (p % kPerTile) * kGuessStride;
    const int64_t nvalid = segs.n[sg] - off;
    const uint16_t* q = x + segs.x_off[sg] + off;
    uint32_t w[8];
    if (nvalid >= kEPT && (reinterpret_cast<uintptr_t>(q) & 31) == 0) {
      uint4 a, b;
      ld_stream_v8(q, a, b);
      if (!have_k) read_k();
      w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
      w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
    } else {
      if (!have_k) read_k();
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t lo = (2 * j < nvalid) ? q[2 * j] : kw;          // d = 0 outside
        const uint32_t hi = (2 * j + 1 < nvalid) ? q[2 * j + 1] : kw;
        w[j] = lo | (hi << 16);
      }
    }
    if (nvalid > 0) cnt += (double)(nvalid < kEPT ? nvalid : kEPT);
    sums_acc16(w, K2, s1, s2);
  }
  __shared__ double g_1[kWarps], g_2[kWarps], g_3[kWarps];
  __shared__ bool s_last;
  auto block_sum = [&](double& a1, double& a2, double& a3) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a1 += __shfl_down_sync(0xffffffffu, a1, o);
      a2 += __shfl_down_sync(0xffffffffu, a2, o);
      a3 += __shfl_down_sync(0xffffffffu, a3, o);
    }
    if ((tid & 31) == 0) { g_1[tid >> 5] = a1; g_2[tid >> 5] = a2; g_3[tid >> 5] = a3; }
    __syncthreads();
    if (tid == 0) {
      a1 = a2 = a3 = 0.0;
      for (int k = 0; k < kWarps; ++k) { a1 += g_1[k]; a2 += g_2[k]; a3 += g_3[k]; }
    }
  };
  block_sum(s1, s2, cnt);
  if (tid == 0) {
    parts[blockIdx.x] = GuessPartial{s1, s2, cnt};
    __threadfence();
    s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double a1 = 0.0, a2 = 0.0, a3 = 0.0;
  for (unsigned k = tid; k < gridDim.x; k += kThreads) {
    a1 += __ldcg(&parts[k].s1);
    a2 += __ldcg(&parts[k].s2);
    a3 += __ldcg(&parts[k].cnt);
  }
  __syncthreads();   // g_* reuse
  block_sum(a1, a2, a3);
  if (tid != 0) return;
  if (!have_k) read_k();
  const double m2 = a3 > 0.0 ? a2 - a1 * (a1 / a3) : 0.0;
  // degenerate sample (constant / non-finite): window around K's exponent
  const int base = (isfinite(m2) && m2 > 0.0) ? derive_base(sqrt(m2 / a3))
                                                : (int)((kw >> 7) & 0xFF) - 127 - 3;
  write_window(guess, base);
}

#ifdef ZC_EXP_FIXED_GUESS
__global__ void fixed_guess_kernel(uint8_t* guess) {
  grid_dep_launch();
  if (threadIdx.x == 0) write_window(guess, 116 - 127);
}
#endif
cudaError_t launch_guess(const uint16_t* x, const StatSegs& segs, void* parts, unsigned* done,
                         uint8_t* guess, cudaStream_t st) {
  const int64_t nprobe = (segs.tile_start[segs.nseg] + kGuessTileSkip - 1) / kGuessTileSkip *
                        (kTile / kGuessStride);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t grid = (nprobe + kThreads - 1) / kThreads;
  if (grid > 8 * sms) grid = 8 * sms;
#ifdef ZC_EXP_FIXED_GUESS   // experiment: the guess's cost (bench layer book)
  if (true) { fixed_guess_kernel<<<1, 32, 0, st>>>(guess); return cudaGetLastError(); }
#endif
  guess_kernel<<<(unsigned)grid, kThreads, 0, st>>>(x, segs,
                                                    reinterpret_cast<GuessPartial*>(parts), done,
                                                    guess);
  return cudaGetLastError();
}

// The exact f64 statistic over x, as a conditional launch behind the fused
// certificate (returns at once when *need == 0).  `grid_limit` caps the CTAs
// of this rarely-needed pass, so its no-op launch stays cheap.
cudaError_t launch_exact_if_needed(const uint16_t* x, const StatSegs& segs, int64_t total,
                                   Partial* parts, unsigned* done, uint8_t* book,
                                   double* result, const int* need, int grid_limit,
                                   cudaStream_t st) {
  const int64_t ntiles = segs.tile_start[segs.nseg];
  int64_t grid = stats_grid_cap();
  if (grid > grid_limit) grid = grid_limit;
  if (grid > ntiles) grid = ntiles;
  stats_kernel<<<(unsigned)grid, kThreads, stats_dyn_smem(), st>>>(
      x, segs, parts, done, total, book, result, need);
  return cudaGetLastError();
}


// Loads every kernel of this file now (cudaFuncGetAttributes forces a
// lazily loaded module function in): with CUDA_MODULE_LOADING=LAZY, the
// first launch of a kernel waits for the device, which deadlocks while a
// peer rank sharing the GPU spins on a flag this rank has yet to publish.
cudaError_t preload_stats() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, (const void*)finalize_kernel);
  cudaFuncGetAttributes(&a, (const void*)guess_kernel);
  cudaFuncGetAttributes(&a, (const void*)hist_kernel);
  cudaFuncGetAttributes(&a, (const void*)mode_kernel);
  cudaFuncGetAttributes(&a, (const void*)stats_kernel);
  cudaFuncGetAttributes(&a, (const void*)sums_kernel);
  cudaFuncGetAttributes(&a, (const void*)np_sigma_kernel<0>);
  cudaFuncGetAttributes(&a, (const void*)np_sigma_kernel<1>);
  stats_grid_cap();
  sums_grid_cap();
  return cudaGetLastError();
}

}  // namespace zc
