// Shared f64 statistics accumulator (reference bf16.measure_sigma,
// bf16.py:88-103: np.std, ddof=0, over the finite elements in f64).
//
// Each thread keeps running sums of d = x - K (K = the first finite value it
// sees), so a constant buffer yields exactly M2 = 0 (the modal-fallback
// trigger, codec.py:179-185); per-thread (count, mean, M2) are Chan-merged
// in a fixed order.  Used by the stand-alone K1 kernel and fused into the
// encoder's TMA loop (speculative codebook path).
#pragma once
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

}  // namespace zc
