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
#include "zc_common.cuh"

namespace zc {

struct Partial {   // 32 B per CTA
  double count;    // finite elements
  double mean;
  double m2;
  double aux;      // exponent of some finite element (or -1)
};

__device__ __forceinline__ void chan_merge(double& na, double& ma, double& m2a, double nb,
                                           double mb, double m2b) {
  if (nb == 0.0) return;
  if (na == 0.0) { na = nb; ma = mb; m2a = m2b; return; }
  const double n = na + nb;
  const double d = mb - ma;
  ma = ma + d * (nb / n);
  m2a = m2a + m2b + d * d * (na * nb / n);
  na = n;
}

// Persistent: each CTA strides over tiles, each thread keeps running f64
// sums of d = x - K (K = the first finite value the thread sees; non-finite
// words are replaced by K so they add exactly 0) and the per-thread
// (count, mean, M2) are Chan-merged once per CTA at the end.
__device__ __forceinline__ void chan_shfl(double& n, double& m, double& q, int o) {
  const double nb = __shfl_xor_sync(0xffffffffu, n, o);
  const double mb = __shfl_xor_sync(0xffffffffu, m, o);
  const double qb = __shfl_xor_sync(0xffffffffu, q, o);
  chan_merge(n, m, q, nb, mb, qb);
}

__global__ void __launch_bounds__(kThreads)
stats_kernel(const uint16_t* __restrict__ x, const StatSegs segs, Partial* __restrict__ out) {
  __shared__ double s_n[kWarps], s_m[kWarps], s_q[kWarps];
  __shared__ int s_e[kWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t ntiles = segs.tile_start[segs.nseg];

  bool have_k = false;
  uint32_t kword = 0;        // K as a bf16 word in the high half of an f32
  double K = 0.0, s1 = 0.0, s2 = 0.0;
  uint64_t cnt = 0;
  int kexp = -1;

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
  int64_t tile = blockIdx.x;
  if (tile < ntiles) load(tile, w);
  while (tile < ntiles) {
    const int64_t nt = tile + gridDim.x;
    if (nt < ntiles) load(nt, nw);
    // finite test per half: exponent field != 255 (bf16.py:100 np.isfinite);
    // bit 15 / bit 31 of v set iff the low / high word is finite
    uint32_t v[8], allfin = 0x80008000u;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      v[k] = (~w[k] & 0x7F807F80u) + 0x7F807F80u;
      allfin &= v[k];
    }
    if (allfin == 0x80008000u && have_k) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double lo = (double)__uint_as_float(w[k] << 16) - K;
        const double hi = (double)__uint_as_float(w[k] & 0xFFFF0000u) - K;
        s1 += lo;
        s2 = fma(lo, lo, s2);
        s1 += hi;
        s2 = fma(hi, hi, s2);
      }
      cnt += kEPT;
    } else {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint32_t word = (k & 1) ? (w[k >> 1] >> 16) : (w[k >> 1] & 0xFFFFu);
        const bool fin = (v[k >> 1] >> ((k & 1) ? 31 : 15)) & 1u;
        if (fin && !have_k) {
          have_k = true;
          kword = word;
          K = (double)__uint_as_float(word << 16);
          kexp = (word >> 7) & 0xFF;
        }
        if (fin) {
          const double d = (double)__uint_as_float(word << 16) - K;
          s1 += d;
          s2 = fma(d, d, s2);
          ++cnt;
        }
      }
    }
    tile = nt;
#pragma unroll
    for (int k = 0; k < 8; ++k) w[k] = nw[k];
  }
  (void)kword;
  // per-thread (count, mean, M2), then Chan merge: warp tree, then warps
  double c = (double)cnt, m = 0.0, q = 0.0;
  if (cnt > 0) {
    m = K + s1 / c;
    q = fmax(s2 - s1 * (s1 / c), 0.0);
  }
  int e = kexp;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    chan_shfl(c, m, q, o);
    const int eb = __shfl_xor_sync(0xffffffffu, e, o);
    e = (e < 0) ? eb : e;
  }
  if (lane == 0) { s_n[warp] = c; s_m[warp] = m; s_q[warp] = q; s_e[warp] = e; }
  __syncthreads();
  if (tid == 0) {
    double na = 0.0, ma = 0.0, qa = 0.0;
    int ea = -1;
    for (int i = 0; i < kWarps; ++i) {
      chan_merge(na, ma, qa, s_n[i], s_m[i], s_q[i]);
      if (ea < 0) ea = s_e[i];
    }
    out[blockIdx.x] = Partial{na, ma, qa, (double)ea};
  }
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
                uint8_t* __restrict__ book, double* __restrict__ result) {
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
  if (grid > 0) stats_kernel<<<(unsigned)grid, kThreads, 0, st>>>(x, segs, parts);
  finalize_kernel<<<1, 1024, 0, st>>>(parts, grid, total, book, result);
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

}  // namespace zc
