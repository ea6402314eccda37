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

// Persistent: each CTA strides over tiles (every `stride`-th tile: 1 for the
// exact statistic, >1 for the sampled guess of the speculative encoder).
__global__ void __launch_bounds__(kThreads)
stats_kernel(const uint16_t* __restrict__ x, const StatSegs segs, int64_t stride,
             Partial* __restrict__ out) {
  const int tid = threadIdx.x;
  const int64_t ntiles = segs.tile_start[segs.nseg];
  StatAcc acc;
  uint32_t w[8], nw[8];
  auto load = [&](int64_t tile, uint32_t* dst) {
    const int s = find_seg(segs.tile_start, segs.nseg, tile);
    const uint16_t* xs = x + segs.x_off[s];
    const int64_t base = (tile - segs.tile_start[s]) * kTile + (int64_t)tid * kEPT;
    const int64_t nvalid = segs.n[s] - base;
    if (nvalid >= kEPT && ((reinterpret_cast<uintptr_t>(xs) & 15) == 0)) {
      const uint4 a = ld_stream_v4(xs + base), b = ld_stream_v4(xs + base + 8);
      dst[0] = a.x; dst[1] = a.y; dst[2] = a.z; dst[3] = a.w;
      dst[4] = b.x; dst[5] = b.y; dst[6] = b.z; dst[7] = b.w;
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        // out-of-range elements become NaN words: excluded like non-finite
        const uint32_t lo = (2 * k < nvalid) ? xs[base + 2 * k] : 0x7FC0u;
        const uint32_t hi = (2 * k + 1 < nvalid) ? xs[base + 2 * k + 1] : 0x7FC0u;
        dst[k] = lo | (hi << 16);
      }
    }
  };
  int64_t i = blockIdx.x;
  if (i * stride < ntiles) load(i * stride, w);
  while (i * stride < ntiles) {
    const int64_t ni = i + gridDim.x;
    if (ni * stride < ntiles) load(ni * stride, nw);
    acc.add16(w, 0xFFFFu);
    i = ni;
#pragma unroll
    for (int k = 0; k < 8; ++k) w[k] = nw[k];
  }
  stat_block_finish(acc, out + blockIdx.x);
}

// --- host-identical codebook math (codec.py:74-161) ---------------------------
// BASE_EXPONENT_OFFSET = 0.5*log2(14 ln2 / 16383) (codec.py:59), bit-exact literal
constexpr double kBaseExponentOffset = -0x1.571514cbe4290p+2;
__device__ double window_coverage(double sigma, double x) {
  const double lo = exp2(x);
  const double hi = lo * 128.0;
  const double scale = sigma * sqrt(2.0);
  return erf(hi / scale) - erf(lo / scale);
}

__device__ int clamp_base(int b) { return b < -126 ? -126 : (b > 121 ? 121 : b); }

__device__ void write_window(uint8_t* book, int base) {
  const int first = clamp_base(base) + 127;
  for (int i = 0; i < 7; ++i) book[i] = (uint8_t)(first + i);
  book[7] = 0;
}

// Final reduction + derivation.  One CTA of 1024 threads; thread t merges a
// fixed contiguous range, then a fixed binary tree.  result[0] = sigma
// (NaN when no finite value), result[1] = finite count, result[2] = path
// (1 analytic, 2 modal), book = 7 entries.
__global__ void __launch_bounds__(1024)
finalize_kernel(const Partial* __restrict__ parts, int64_t nparts, int64_t total_words,
                uint8_t* __restrict__ book, double* __restrict__ result,
                const uint8_t* __restrict__ guess, int* __restrict__ mismatch) {
  __shared__ double s_n[1024], s_m[1024], s_q[1024];
  __shared__ int s_e[1024];
  const int t = threadIdx.x;
  const int64_t per = (nparts + 1023) / 1024;
  double na = 0.0, ma = 0.0, qa = 0.0;
  int e = -1;
  for (int64_t i = t * per; i < (t + 1) * per && i < nparts; ++i) {
    const Partial p = parts[i];
    chan_merge(na, ma, qa, p.count, p.mean, p.m2);
    if (e < 0) e = (int)p.aux;
  }
  s_n[t] = na; s_m[t] = ma; s_q[t] = qa; s_e[t] = e;
  __syncthreads();
  for (int s = 512; s > 0; s >>= 1) {
    if (t < s) {
      double a = s_n[t], b = s_m[t], c = s_q[t];
      chan_merge(a, b, c, s_n[t + s], s_m[t + s], s_q[t + s]);
      s_n[t] = a; s_m[t] = b; s_q[t] = c;
      if (s_e[t] < 0) s_e[t] = s_e[t + s];
    }
    __syncthreads();
  }
  if (t == 0) {
    const double cnt = s_n[0];
    const double sigma = cnt > 0.0 ? sqrt(s_q[0] / cnt) : nan("");
    result[0] = sigma;
    result[1] = cnt;
    if (cnt > 0.0 && isfinite(sigma) && sigma > 0.0) {
      // derive_codebook (codec.py:149-161)
      const double xo = log2(sigma) + kBaseExponentOffset;
      const double lo = floor(xo), hi = ceil(xo);
      const int base = (lo == hi || window_coverage(sigma, lo) >= window_coverage(sigma, hi))
                           ? (int)lo : (int)hi;
      write_window(book, base);
      result[2] = 1.0;
    } else {
      // modal fallback (codec.py:181-185) with the two possible bins
      const double c_nf = (double)total_words - cnt;
      int mode;
      if (cnt > 0.0 && cnt >= c_nf) mode = s_e[0];
      else if (total_words > 0) mode = 255;
      else mode = 0;
      const bool all_zero_exp = (mode == 0) && (cnt == (double)total_words);
      write_window(book, all_zero_exp ? -6 : mode - 127 - 3);
      result[2] = 2.0;
    }
    if (mismatch) {
      int diff = 0;
      for (int i = 0; i < 7; ++i) diff |= (book[i] != guess[i]);
      *mismatch = diff;
    }
  }
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

cudaError_t launch_codebook_measured(const uint16_t* x, const StatSegs& segs, int64_t total,
                                     void* ws, uint8_t* book, double* result, cudaStream_t st) {
  const int64_t ntiles = segs.tile_start[segs.nseg];
  Partial* parts = reinterpret_cast<Partial*>(reinterpret_cast<uint8_t*>(ws) + 128);
  static int grid_cap = 0;
  if (grid_cap == 0) {
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stats_kernel, kThreads, 0);
    grid_cap = sms * (occ > 0 ? occ : 1);
  }
  const int64_t grid = ntiles < grid_cap ? ntiles : grid_cap;
  if (grid > 0) stats_kernel<<<(unsigned)grid, kThreads, 0, st>>>(x, segs, 1, parts);
  finalize_kernel<<<1, 1024, 0, st>>>(parts, grid, total, book, result, nullptr, nullptr);
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

// Sampled guess for the speculative encoder: every `stride`-th tile.
cudaError_t launch_codebook_sampled(const uint16_t* x, const StatSegs& segs, int64_t stride,
                                    Partial* parts, uint8_t* book, double* result,
                                    cudaStream_t st) {
  const int64_t ntiles = segs.tile_start[segs.nseg];
  const int64_t sampled = (ntiles + stride - 1) / stride;
  static int grid_cap = 0;
  if (grid_cap == 0) {
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stats_kernel, kThreads, 0);
    grid_cap = sms * (occ > 0 ? occ : 1);
  }
  const int64_t grid = sampled < grid_cap ? sampled : grid_cap;
  stats_kernel<<<(unsigned)grid, kThreads, 0, st>>>(x, segs, stride, parts);
  finalize_kernel<<<1, 1024, 0, st>>>(parts, grid, 0, book, result, nullptr, nullptr);
  return cudaGetLastError();
}

// Exact codebook from per-CTA partials; flags a mismatch with `guess`.
cudaError_t launch_finalize(const Partial* parts, int64_t nparts, int64_t total, uint8_t* book,
                            double* result, const uint8_t* guess, int* mismatch,
                            cudaStream_t st) {
  finalize_kernel<<<1, 1024, 0, st>>>(parts, nparts, total, book, result, guess, mismatch);
  return cudaGetLastError();
}

}  // namespace zc
