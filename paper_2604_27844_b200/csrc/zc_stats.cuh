// Shared f64 statistics accumulator (reference bf16.measure_sigma,
// bf16.py:88-103: np.std, ddof=0, over the finite elements in f64).
//
// Each thread keeps running sums of d = x - K (K = the first finite value it
// sees), so a constant buffer yields exactly M2 = 0 (the modal-fallback
// trigger, codec.py:179-185); per-thread (count, mean, M2) are Chan-merged
// in a fixed order.  Used by the stand-alone K1 kernel and fused into the
// encoder's TMA loop (speculative codebook path).
#pragma once
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

struct StatAcc {
  bool have_k = false;
  double K = 0.0, s1 = 0.0, s2 = 0.0;
  uint64_t cnt = 0;
  int kexp = -1;

  // 16 words packed in w[8]; `valid` masks elements inside the segment
  __device__ __forceinline__ void add16(const uint32_t* w, uint32_t valid) {
    // finite test per half: exponent field != 255 (bf16.py:100 np.isfinite);
    // bit 15 / bit 31 of v set iff the low / high word is finite
    uint32_t v[8], allfin = 0x80008000u;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      v[k] = (~w[k] & 0x7F807F80u) + 0x7F807F80u;
      allfin &= v[k];
    }
    if (allfin == 0x80008000u && have_k && valid == 0xFFFFu) {
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
        const bool fin = ((v[k >> 1] >> ((k & 1) ? 31 : 15)) & 1u) && ((valid >> k) & 1u);
        if (fin && !have_k) {
          have_k = true;
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
  }
};

__device__ __forceinline__ void chan_shfl(double& n, double& m, double& q, int o) {
  const double nb = __shfl_xor_sync(0xffffffffu, n, o);
  const double mb = __shfl_xor_sync(0xffffffffu, m, o);
  const double qb = __shfl_xor_sync(0xffffffffu, q, o);
  chan_merge(n, m, q, nb, mb, qb);
}

// CTA-wide fixed-order merge of every thread's accumulator; thread 0 writes
// *out.  Must be called by all threads of a kThreads-thread CTA.
__device__ __forceinline__ void stat_block_finish(const StatAcc& a, Partial* out) {
  __shared__ double s_n[kWarps], s_m[kWarps], s_q[kWarps];
  __shared__ int s_e[kWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double c = (double)a.cnt, m = 0.0, q = 0.0;
  if (a.cnt > 0) {
    m = a.K + a.s1 / c;
    q = fmax(a.s2 - a.s1 * (a.s1 / c), 0.0);
  }
  int e = a.kexp;
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
    *out = Partial{na, ma, qa, (double)ea};
  }
}

// ---- certified packed-fp32 statistic (see zc_stats.cu) -----------------------
struct SumPartial {
  double s1, s2;
};

__device__ __forceinline__ uint64_t f2_sub(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ double f2_sum(uint64_t v) {
  return (double)__uint_as_float((uint32_t)v) + (double)__uint_as_float((uint32_t)(v >> 32));
}

__device__ __forceinline__ void sums_acc16(const uint32_t* w, uint64_t K2, double& s1, double& s2) {
  uint64_t a1 = 0, a2 = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint64_t v = (uint64_t)(w[j] & 0xFFFF0000u) << 32 | (uint64_t)(w[j] << 16);
    const uint64_t d = f2_sub(v, K2);
    a1 = f2_add(a1, d);
    a2 = f2_fma(d, d, a2);
  }
  s1 += f2_sum(a1);
  s2 += f2_sum(a2);
}

// Unshifted form (K = 0): 4 ops per element pair instead of 5.  Exact
// inputs (bf16 is a subset of fp32), so the error bound above still holds;
// a large mean relative to sigma only makes the certificate fail more often
// (then the exact pass decides).  Used by the fused encoder.
__device__ __forceinline__ void sums_acc16_k0(const uint32_t* w, double& s1, double& s2) {
  uint64_t a1 = 0, a2 = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint64_t v = (uint64_t)(w[j] & 0xFFFF0000u) << 32 | (uint64_t)(w[j] << 16);
    a1 = f2_add(a1, v);
    a2 = f2_fma(v, v, a2);
  }
  s1 += f2_sum(a1);
  s2 += f2_sum(a2);
}

// Packed accumulation only (the caller flushes with f2_sum): the fused
// encoder chains two tiles' words, 16 terms per fp32 lane.
__device__ __forceinline__ void sums_chain16_k0(const uint32_t* w, uint64_t& a1, uint64_t& a2) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint64_t v = (uint64_t)(w[j] & 0xFFFF0000u) << 32 | (uint64_t)(w[j] << 16);
    a1 = f2_add(a1, v);
    a2 = f2_fma(v, v, a2);
  }
}

// Shift word pair of the certified statistic: K = the first element of the
// concatenation when finite, else 0, in both halves (d = x - K per element).
__device__ __forceinline__ uint64_t sums_shift(uint32_t kw) {
  const uint32_t kpair = kw | (kw << 16);
  return (uint64_t)(kpair & 0xFFFF0000u) << 32 | (uint64_t)(kpair << 16);
}

// CTA sum of (s1, s2) in a fixed order; thread 0 writes *out.
__device__ __forceinline__ void sums_block_finish(double s1, double s2, SumPartial* out) {
  __shared__ double b_1[kWarps], b_2[kWarps];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s1 += __shfl_down_sync(0xffffffffu, s1, o);
    s2 += __shfl_down_sync(0xffffffffu, s2, o);
  }
  const int tid = threadIdx.x;
  if ((tid & 31) == 0) { b_1[tid >> 5] = s1; b_2[tid >> 5] = s2; }
  __syncthreads();
  if (tid == 0) {
    double t1 = 0.0, t2 = 0.0;
    for (int k = 0; k < kWarps; ++k) { t1 += b_1[k]; t2 += b_2[k]; }
    *out = SumPartial{t1, t2};
  }
}

// --- host-identical codebook math (codec.py:74-161) ---------------------------
// BASE_EXPONENT_OFFSET = 0.5*log2(14 ln2 / 16383) (codec.py:59), bit-exact literal
constexpr double kBaseExponentOffset = -0x1.571514cbe4290p+2;
__device__ inline double window_coverage(double sigma, double x) {
  const double lo = exp2(x);
  const double hi = lo * 128.0;
  const double scale = sigma * sqrt(2.0);
  return erf(hi / scale) - erf(lo / scale);
}

__device__ inline int clamp_base(int b) { return b < -126 ? -126 : (b > 121 ? 121 : b); }

// derive_codebook (codec.py:149-161): floor/ceil of log2(sigma) + offset,
// larger coverage wins, tie to floor; clamped like write_window
// Coverage depends on sigma only through 2^x / sigma, so the floor/ceil
// choice depends only on frac(x_opt): floor below kFlipFrac, ceil above
// (swept against the reference's derive_codebook at 10^6 points per octave,
// no exception).  Away from the flip the erf evaluations are skipped -- they
// are a long serial f64 chain in a single thread at the end of the
// statistic kernels; within kFlipWindow of it the reference formula decides.
constexpr double kFlipFrac = 0.35891885782276935;
constexpr double kFlipWindow = 1e-4;
// Within kNpFlipFrac of the flip in frac(x_opt) (sigma within ~7e-9
// relative of a threshold) the f64 statistics re-derive the codebook from
// numpy's own sigma (np_refine_near_flip); `near` reports that case.
constexpr double kNpFlipFrac = 1e-8;
__device__ inline int derive_base(double sigma, bool* near = nullptr) {
  const double xo = log2(sigma) + kBaseExponentOffset;
  const double lo = floor(xo), hi = ceil(xo);
  const double fr = xo - lo;
  if (near != nullptr) *near = fabs(fr - kFlipFrac) < kNpFlipFrac;
  if (fabs(fr - kFlipFrac) > kFlipWindow) return clamp_base(fr < kFlipFrac ? (int)lo : (int)hi);
  const int base = (lo == hi || window_coverage(sigma, lo) >= window_coverage(sigma, hi))
                       ? (int)lo : (int)hi;
  return clamp_base(base);
}

__device__ inline void write_window(uint8_t* book, int base) {
  const int first = clamp_base(base) + 127;
  for (int i = 0; i < 7; ++i) book[i] = (uint8_t)(first + i);
  book[7] = 0;
}


// The reference derivation from merged statistics (count cn, M2 cq, first
// finite exponent ce): result[0] = sigma (NaN when no finite value),
// result[1] = finite count, result[2] = path (1 analytic, 2 modal).
__device__ inline void finish_codebook(double cn, double cq, int ce, int64_t total_words,
                                       uint8_t* book, double* result, bool* near = nullptr) {
  if (near != nullptr) *near = false;
  const double sigma = cn > 0.0 ? sqrt(cq / cn) : nan("");
  result[0] = sigma;
  result[1] = cn;
  if (cn > 0.0 && isfinite(sigma) && sigma > 0.0) {
    write_window(book, derive_base(sigma, near));
    result[2] = 1.0;
    if (near != nullptr) *near = *near && cn == (double)total_words;   // all finite
  } else {
    // modal fallback (codec.py:181-185): with sigma 0 or no finite value the
    // histogram has at most two bins, the common finite exponent and 255
    const double c_nf = (double)total_words - cn;
    int mode;
    if (cn > 0.0 && cn >= c_nf) mode = ce;
    else if (total_words > 0) mode = 255;
    else mode = 0;
    const bool all_zero_exp = (mode == 0) && (cn == (double)total_words);
    write_window(book, all_zero_exp ? -6 : mode - 127 - 3);
    result[2] = 2.0;
  }
}

// ---- certified fast statistic ------------------------------------------------
// Every element contributes d = x - K (K = the first element when finite, else
// 0; the same K everywhere, so partials merge by plain addition) to per-tile
// sums kept in packed fp32 (FADD2/FFMA2, at most 16 terms per lane), flushed
// to f64 once per tile (the fused encoder: once per tile pair).  A non-finite element poisons the sums (inf/NaN propagate),
// which routes the call to the exact f64 kernel.  Error bound (u = 2^-24):
// per element fl(x - K) = d(1+δ), |δ| <= u; 16-term fp32 chains add <= γ_16;
// f64 accumulation adds <= 2^-36 relative; with Q = Σd² (>= 0) and
// |S1| <= sqrt(N Q):  |ΔS2| <= 19u·Q, |ΔS1| <= 18u·Σ|d|, so
//   |ΔM2| = |ΔS2 - (2 S1 ΔS1 + ΔS1²)/N| <= 64u·Q + 2^-34·Q + N·2^-149
// (the last term: fp32 underflow of d², also in the bound on Q).  The codebook is certified when
// derive_base() agrees at both ends of sigma = sqrt((M2 ± Δ)/N), widened by
// 2^-40 for the reference's own f64 evaluation (np.std two-pass error); the
// reference's sigma lies in that interval and derive_base is monotone, so
// its codebook is this one.  Otherwise *need = 1 and the exact pass runs.
__device__ inline void certify_block(const SumPartial* parts, int64_t nparts, int64_t total,
                              uint8_t* book, double* result, int* need) {
  __shared__ double c_1[kWarps], c_2[kWarps];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t per = (nparts + kThreads - 1) / kThreads;
  double a1 = 0.0, a2 = 0.0;
  for (int64_t i = t * per; i < (t + 1) * per && i < nparts; ++i) {
    a1 += __ldcg(&parts[i].s1);
    a2 += __ldcg(&parts[i].s2);
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {   // fixed tree: lane i absorbs lane i+o
    const double b1 = __shfl_down_sync(0xffffffffu, a1, o);
    const double b2 = __shfl_down_sync(0xffffffffu, a2, o);
    if ((lane & (2 * o - 1)) == 0) { a1 += b1; a2 += b2; }
  }
  if (lane == 0) { c_1[warp] = a1; c_2[warp] = a2; }
  __syncthreads();
  if (t != 0) return;
  double S1 = 0.0, S2 = 0.0;
  for (int i = 0; i < kWarps; ++i) { S1 += c_1[i]; S2 += c_2[i]; }
  const double N = (double)total;
  int decided = 0;
  if (total > 0 && isfinite(S1) && isfinite(S2)) {
    const double m2 = S2 - S1 * (S1 / N);
    const double q = S2 * (1.0 + 0x1p-20);                 // >= true Q
    const double delta = (64.0 * 0x1p-24 + 0x1p-34) * q + N * 0x1p-149;
    if (m2 - delta > 0.0) {
      const double s_lo = sqrt((m2 - delta) / N) * (1.0 - 0x1p-40);
      const double s_hi = sqrt((m2 + delta) / N) * (1.0 + 0x1p-40);
      if (isfinite(s_hi)) {
        const int b = derive_base(s_lo);
        if (b == derive_base(s_hi)) {
          write_window(book, b);
          result[0] = sqrt(m2 / N);
          result[1] = N;
          result[2] = 3.0;                                   // analytic, certified
          decided = 1;
        }
      }
    }
  }
  *need = decided ? 0 : 1;
}

// ---- numpy-exact sigma (zc_stats.cu np_sigma_kernel) ---------------------------
// Workspace of the two passes: the mean of pass 0 and the subtree sums of the
// 2^kNpK owners of the pairwise tree's top levels.  It sits behind the
// encoder's run totals and speculative area (zc_encode.cu: 256 + 32 KB +
// 512 KB), in front of the encoder scratch.
constexpr int kNpK = 17;
constexpr int kNpOwners = 1 << kNpK;
struct NpWs {
  double mean;
  double pad[7];
  double parts[kNpOwners];
  int8_t depth[kNpOwners];       // owner's node depth, -1 = not an owner
};
constexpr int64_t kNpArea = ((int64_t)sizeof(NpWs) + 4095) / 4096 * 4096;
constexpr int64_t kNpWsOff = 256 + 8 * 4096 + 512 * 1024;

// ---- numpy-exact sigma ---------------------------------------------------------
// The reference's sigma is np.std over the finite values (bf16.py:103), i.e.
// numpy's _var: mean = (0.0 + S) / m, ret = (0.0 + Q) / m, sigma = sqrt(ret),
// with S = pairwise_sum(v), Q = pairwise_sum((v - mean)^2) and numpy's
// pairwise_sum (numpy/_core/src/umath/loops_utils.h.src, np.add.reduce of a
// contiguous 1-D float64 array in one inner-loop call): n < 8: 0.0 plus the
// elements in order; n <= 128: eight accumulators r[j] = a[j], r[j] += a[i+j]
// for i = 8, 16, .. < n - n % 8, ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then
// the remaining elements in order; n > 128: the sums of the halves split at
// n/2 - (n/2) % 8.  These kernels evaluate exactly that tree with IEEE
// round-to-nearest adds (no contraction), so sigma is bit-identical to the
// reference when every element is finite (the compacted array is then x
// itself); with non-finite elements the exact Chan pass's value stays.
// The tree's top kNpK levels are split over 2^kNpK threads: thread t owns
// the node reached by t's bits (MSB first) if t is that node's leftmost
// index; it evaluates its subtree depth first (explicit stack), and the last
// CTA combines the owners bottom-up (node = left + right).
constexpr int kNpLeaf = 128;

__device__ __forceinline__ int64_t np_left(int64_t n) {
  const int64_t n2 = n / 2;
  return n2 - n2 % 8;
}

// forward-only reader of the concatenated segments as float64 (segs ==
// nullptr: one segment of `total` elements at x)
struct NpCursor {
  const uint16_t* x;
  const StatSegs* segs;
  int s;
  int64_t hi;                       // concatenated end of segment s
  int64_t off;                      // element e of segment s is x[off + e]
  __device__ void init(const uint16_t* x_, const StatSegs* sg, int64_t e, int64_t total) {
    x = x_;
    segs = sg;
    s = 0;
    hi = sg ? sg->n[0] : total;
    off = sg ? sg->x_off[0] : 0;
    seek(e);
  }
  __device__ __forceinline__ void seek(int64_t e) {
    while (segs != nullptr && e >= hi && s + 1 < segs->nseg) {
      ++s;
      off = segs->x_off[s] - hi;
      hi += segs->n[s];
    }
  }
  __device__ __forceinline__ double val(int64_t e) {
    seek(e);
    return (double)__uint_as_float((uint32_t)x[off + e] << 16);
  }
  // elements e .. e + 7
  __device__ __forceinline__ void val8(int64_t e, double (&v)[8]) {
    seek(e);
    const uint16_t* p = x + off + e;
    if (e + 8 <= hi && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
      const uint4 q = __ldcg(reinterpret_cast<const uint4*>(p));
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        v[2 * j] = (double)__uint_as_float(w[j] << 16);
        v[2 * j + 1] = (double)__uint_as_float(w[j] & 0xFFFF0000u);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = val(e + j);
    }
  }
};

template <int kPass>
__device__ __forceinline__ double np_term(double v, double mean) {
  if (kPass == 0) return v;
  const double d = __dsub_rn(v, mean);
  return __dmul_rn(d, d);
}

template <int kPass>
__device__ double np_leaf(NpCursor& c, int64_t start, int64_t n, double mean) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, np_term<kPass>(c.val(start + i), mean));
    return r;
  }
  double r[8], v[8];
  c.val8(start, v);
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = np_term<kPass>(v[j], mean);
  int64_t i = 8;
  const int64_t lim = n - n % 8;
  for (; i < lim; i += 8) {
    c.val8(start + i, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], np_term<kPass>(v[j], mean));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, np_term<kPass>(c.val(start + i), mean));
  return res;
}

// pairwise_sum of [start, start + n): post-order walk with an explicit stack
template <int kPass, int kDepth = 32>
__device__ double np_subtree(NpCursor& c, int64_t start, int64_t n, double mean) {
  struct Fr {
    int64_t start, n;
    double lv;
    int st;                              // 0 new, 1 left pending, 2 right pending
  };
  Fr stk[kDepth];                        // depth <= log2(2^32 / 128) + 1 from the root
  int sp = 0;
  stk[sp++] = Fr{start, n, 0.0, 0};
  double ret = 0.0;
  bool have = false;                     // a finished child's value is in ret
  while (sp > 0) {
    Fr& f = stk[sp - 1];
    if (have) {
      if (f.st == 1) {                   // left done: keep it, descend right
        f.lv = ret;
        f.st = 2;
        have = false;
        const int64_t L = np_left(f.n);
        stk[sp++] = Fr{f.start + L, f.n - L, 0.0, 0};
      } else {                           // right done: left + right, up one level
        ret = __dadd_rn(f.lv, ret);
        --sp;
      }
      continue;
    }
    if (f.n <= kNpLeaf) {
      ret = np_leaf<kPass>(c, f.start, f.n, mean);
      --sp;
      have = true;
      continue;
    }
    f.st = 1;
    stk[sp++] = Fr{f.start, np_left(f.n), 0.0, 0};
  }
  return ret;
}

// numpy's sigma by ONE CTA of kThreads threads (thread t owns the node its
// 8 bits reach in the tree's top levels, as np_sigma_kernel with kNpK = 8),
// both passes, every thread returns the same value.  Only for the rare call
// whose sigma sits next to a flip threshold (np_refine_near_flip), so one SM
// streaming the input twice is acceptable.
template <int kDepth = 18>
__device__ __forceinline__ double np_block_sigma(const uint16_t* x, const StatSegs* segs,
                                                int64_t total) {
  constexpr int K = 8;
  static_assert((1 << K) == kThreads, "one owner index per thread");
  __shared__ double s_val[kThreads];
  __shared__ int8_t s_dep[kThreads];
  const int tid = threadIdx.x;
  int64_t start = 0, n = total;
  int d = 0;
  bool owner = true;
  for (; d < K; ++d) {
    if (n <= kNpLeaf) {
      owner = (tid & ((1 << (K - d)) - 1)) == 0;
      break;
    }
    const int64_t L = np_left(n);
    if ((tid >> (K - 1 - d)) & 1) {
      start += L;
      n -= L;
    } else {
      n = L;
    }
  }
  double v = 0.0;                          // pass 0: mean; pass 1: variance
  for (int pass = 0; pass < 2; ++pass) {
    double mine = 0.0;
    if (owner) {
      NpCursor c;                          // owners sit 8 levels down: 18 frames
      c.init(x, segs, start, total);       // cover 2^32 elements (stack < 1 KB)
      mine = pass ? np_subtree<1, kDepth>(c, start, n, v)
                  : np_subtree<0, kDepth>(c, start, n, 0.0);
    }
    __syncthreads();                       // previous pass's s_val[0] read by all
    s_val[tid] = mine;
    s_dep[tid] = owner ? (int8_t)d : (int8_t)-1;
    __syncthreads();
    for (int dd = K - 1; dd >= 0; --dd) {
      const int step = 1 << (K - dd);
      if ((tid & (step - 1)) == 0 && s_dep[tid] > dd)
        s_val[tid] = __dadd_rn(s_val[tid], s_val[tid + step / 2]);
      __syncthreads();
    }
    v = __ddiv_rn(__dadd_rn(0.0, s_val[0]), (double)total);
  }
  return __dsqrt_rn(v);
}

// Behind an f64 statistic whose codebook thread 0 just wrote (result =
// sigma, finite count, path): when every element is finite and sigma sits
// next to a flip threshold (derive_base's `near`), the whole CTA evaluates numpy's
// sigma and thread 0 re-derives the codebook from it -- the reference's
// codebook even in the last-ulp window where summation order decides.
// `book` / `result` may be shared memory; every thread of the CTA calls it.
// `segs` == nullptr: one segment of `total` elements.  Inlined (an ABI call
// would copy the segment table to the stack, and a kernel stack above the
// 1 KB default makes the driver grow and shrink local memory per launch).
template <int kDepth = 18>
__device__ __forceinline__ void np_refine_near_flip(const uint16_t* x, const StatSegs* segs,
                                                    int64_t total, uint8_t* book, double* result,
                                                    bool write_result) {
  __shared__ bool s_go;
  __syncthreads();
  if (threadIdx.x == 0) {
    const double s = result[0];
    bool near = false;
    if (total > 0 && result[1] == (double)total && isfinite(s) && s > 0.0) derive_base(s, &near);
    s_go = near;
  }
  __syncthreads();
  if (!s_go) return;
  const double s = np_block_sigma<kDepth>(x, segs, total);
  if (threadIdx.x == 0) {
    if (write_result) result[0] = s;
    write_window(book, derive_base(s));
  }
  __syncthreads();
}

}  // namespace zc
