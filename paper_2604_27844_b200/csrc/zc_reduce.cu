// Fused decode + float32 reduction for the compressed reduce-scatter
// (reference collectives.zip_reduce_scatter / _reduce_chunks,
// collectives.py:137-144, :328-341; narrowing bf16.from_float32, bf16.py:53-66).
//
// One launch consumes every rank's contribution to this rank's shard in
// ascending rank order: frames (local receive buffers or a peer's HBM over
// NVLink) are decoded in registers -- the words never round-trip through
// HBM -- and raw word buffers (the self shard, or the uncompressed twin) are
// read directly.  A warp owns one 512-element group (the collectives' group
// size), a lane 16 consecutive elements: sign-mantissa bytes by one 16-B load,
// the three plane half-words, the group's escape base from group_index and a
// warp scan of the per-lane escape counts; the group's escape count is checked
// against group_index exactly like the decoder (reference
// CompressedChunk._check_consistency, codec.py:238-250).
//
// Float32 semantics are numpy's on x86 (the reference's arithmetic):
// acc = to_float32(chunk 0); acc += to_float32(chunk p) for p = 1..W-1 with
// round-to-nearest-even adds, no flush-to-zero; a NaN operand propagates
// quieted (the accumulator's when both are NaN, as numpy's SIMD loop body
// does), inf + -inf gives the x86 default NaN 0xFFC00000.  CUDA's own fadd
// would return the canonical 0x7FFFFFFF instead, so NaNs are handled
// explicitly.  The bf16 narrowing is the reference's RNE with the quiet bit
// forced on NaN (NOT __float2bfloat16_rn, which canonicalises NaN payloads).
#include "zc_common.cuh"

namespace zc {

// Header information for one source, filled by reduce_headers_kernel.
struct RedHdr {
  int64_t zc;
  const uint8_t* esc;      // zero-exponent section
  uint32_t tbl_lo, tbl_hi;
  int32_t err;
  int32_t pad;
};

__device__ __forceinline__ float add_x86(float a, float b) {
  const uint32_t ua = __float_as_uint(a), ub = __float_as_uint(b);
  if ((ua & 0x7FFFFFFFu) > 0x7F800000u) return __uint_as_float(ua | 0x00400000u);
  if ((ub & 0x7FFFFFFFu) > 0x7F800000u) return __uint_as_float(ub | 0x00400000u);
  const float r = __fadd_rn(a, b);
  return (r != r) ? __uint_as_float(0xFFC00000u) : r;   // inf + -inf
}

// bf16.from_float32 (bf16.py:53-66)
__device__ __forceinline__ uint32_t narrow_rne(float f) {
  const uint32_t u = __float_as_uint(f);
  if ((u & 0x7FFFFFFFu) > 0x7F800000u) return (u >> 16) | 0x0040u;
  return (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
}

// One thread per source: wait for a pulled frame (bounded), validate its
// header (reference parse order; collectives frame with 512-element groups).
__global__ void reduce_headers_kernel(const RedSrc* __restrict__ src, int W, int64_t n,
                                      RedHdr* __restrict__ hdr, int32_t* __restrict__ err,
                                      uint64_t epoch, int64_t timeout_ns) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= W) return;
  const RedSrc s = src[p];
  RedHdr h{};
  h.err = kOk;
  err[p] = 0x7F7F7F7F;
  if (!s.raw) {
    if (s.ready) {
      const uint64_t t0 = globaltimer_ns();
      while (ld_acquire_sys_u64(s.ready) < epoch) {
        if (timeout_ns > 0 && (int64_t)(globaltimer_ns() - t0) > timeout_ns) {
          h.err = kErrTimeout;
          break;
        }
        __nanosleep(256);
      }
    }
    if (h.err == kOk) {
      const HeaderInfo H = check_header(s.stat, n, s.dyn_len);
      h.err = H.err;
      if (h.err == kOk && H.gsl != 9) h.err = kErrGroupSize;
      if (h.err == kOk) {
        const Layout L = layout_of(n, 9);
        h.zc = H.zc;
        h.tbl_lo = H.tbl_lo;
        h.tbl_hi = H.tbl_hi;
        h.esc = s.dyn ? s.dyn : s.stat + L.off[5];
      }
    }
    if (h.err != kOk) err[p] = h.err;
  }
  hdr[p] = h;
}

__device__ __forceinline__ void load_words16(const uint16_t* p, int nv, uint32_t (&w)[8]) {
  if (nv == 16 && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
    const uint4 a = *reinterpret_cast<const uint4*>(p);
    const uint4 b = *reinterpret_cast<const uint4*>(p + 8);
    w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
    w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t lo = (2 * j < nv) ? p[2 * j] : 0u;
      const uint32_t hi = (2 * j + 1 < nv) ? p[2 * j + 1] : 0u;
      w[j] = lo | hi << 16;
    }
  }
}

// Decode the 16 words [e0, e0 + nv) of group g of a validated frame; the
// whole warp calls it (warp scan).  Returns the consistency error (lane 0).
__device__ __forceinline__ int32_t decode16(const uint8_t* __restrict__ frame, const RedHdr& h,
                                            const Layout& L, int64_t g, int64_t groups,
                                            int64_t e0, int nv, uint32_t (&w)[8]) {
  const int lane = threadIdx.x & 31;
  uint32_t S[4] = {0, 0, 0, 0};
  uint32_t p0 = 0, p1 = 0, p2 = 0;
  if (nv == 16) {
    const uint4 s = *reinterpret_cast<const uint4*>(frame + L.off[0] + e0);
    S[0] = s.x; S[1] = s.y; S[2] = s.z; S[3] = s.w;
    const int64_t pb = e0 >> 3;
    p0 = *reinterpret_cast<const uint16_t*>(frame + L.off[1] + pb);
    p1 = *reinterpret_cast<const uint16_t*>(frame + L.off[2] + pb);
    p2 = *reinterpret_cast<const uint16_t*>(frame + L.off[3] + pb);
  } else if (nv > 0) {
    for (int k = 0; k < nv; ++k) S[k >> 2] |= (uint32_t)frame[L.off[0] + e0 + k] << (8 * (k & 3));
    const int64_t pb = e0 >> 3;
    p0 = frame[L.off[1] + pb]; p1 = frame[L.off[2] + pb]; p2 = frame[L.off[3] + pb];
    if (nv > 8) {
      p0 |= (uint32_t)frame[L.off[1] + pb + 1] << 8;
      p1 |= (uint32_t)frame[L.off[2] + pb + 1] << 8;
      p2 |= (uint32_t)frame[L.off[3] + pb + 1] << 8;
    }
  }
  const uint32_t valid = nv >= 16 ? 0xFFFFu : (nv > 0 ? (1u << nv) - 1u : 0u);
  const uint32_t esc = ~(p0 | p1 | p2) & valid;
  const uint32_t cnt = __popc(esc);
  const uint32_t incl = warp_incl_scan(cnt);
  const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
  const uint32_t* gi = reinterpret_cast<const uint32_t*>(frame + L.off[4]);
  uint32_t gv = 0, gn = 0;
  if (lane == 0) {
    gv = gi[g];
    gn = (g + 1 < groups) ? gi[g + 1] : (uint32_t)h.zc;
  }
  gv = __shfl_sync(0xffffffffu, gv, 0);
  int32_t e = kOk;
  if (lane == 0) {
    if (g == 0 && gv != 0) e = kErrGroupIndex;
    if (gv + tot != gn) e = (g + 1 < groups) ? kErrGroupIndex : kErrZeroCount;
  }
  int64_t r = (int64_t)gv + (incl - cnt);
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const uint32_t c = ((p0 >> j) & 1u) | ((p1 >> j) & 1u) << 1 | ((p2 >> j) & 1u) << 2;
    uint32_t ex;
    if (c) {
      ex = prmt(h.tbl_lo, h.tbl_hi, c) & 0xFFu;
    } else {
      const int64_t q = r < h.zc ? r : (h.zc ? h.zc - 1 : 0);   // clamp: memory-safe when corrupt
      ex = (j < nv && h.zc) ? h.esc[q] : 0u;
      r += (j < nv) ? 1 : 0;
    }
    const uint32_t sm = (S[j >> 2] >> (8 * (j & 3))) & 0xFFu;
    const uint32_t word = (sm & 0x80u) << 8 | ex << 7 | (sm & 0x7Fu);
    w[j >> 1] |= word << (16 * (j & 1));
  }
  return e;
}

template <bool kF32>
__global__ void __launch_bounds__(256)
reduce_kernel(const RedSrc* __restrict__ src, const RedHdr* __restrict__ hdr, int W, int64_t n,
              void* __restrict__ out, int32_t* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t groups = (n + 511) >> 9;
  const Layout L = layout_of(n, 9);
  for (int64_t g = gw; g < groups; g += nw) {
    const int64_t e0 = g * 512 + lane * 16;
    const int64_t left = n - e0;
    const int nv = left >= 16 ? 16 : (left > 0 ? (int)left : 0);
    float acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0.f;
    for (int p = 0; p < W; ++p) {
      const RedSrc s = src[p];
      uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (s.raw) {
        if (nv > 0) load_words16(reinterpret_cast<const uint16_t*>(s.stat) + e0, nv, w);
      } else {
        const RedHdr h = hdr[p];
        if (h.err == kOk) {   // uniform across the warp
          const int32_t e = decode16(s.stat, h, L, g, groups, e0, nv, w);
          if (e != kOk) atomicMin(err + p, e);
        }
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float v = __uint_as_float(((w[j >> 1] >> (16 * (j & 1))) & 0xFFFFu) << 16);
        acc[j] = (p == 0) ? v : add_x86(acc[j], v);
      }
    }
    if (nv <= 0) continue;
    if (kF32) {
      float* o = reinterpret_cast<float*>(out) + e0;
      if (nv == 16 && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<float4*>(o + 4 * q) =
              make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
      } else {
        for (int j = 0; j < nv; ++j) o[j] = acc[j];
      }
    } else {
      uint32_t o[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = narrow_rne(acc[2 * j]) | narrow_rne(acc[2 * j + 1]) << 16;
      uint16_t* d = reinterpret_cast<uint16_t*>(out) + e0;
      if (nv == 16 && ((reinterpret_cast<uintptr_t>(d) & 31) == 0)) {
        st_v8(d, make_uint4(o[0], o[1], o[2], o[3]), make_uint4(o[4], o[5], o[6], o[7]));
      } else if (nv == 16 && ((reinterpret_cast<uintptr_t>(d) & 15) == 0)) {
        st_stream_v4(d, make_uint4(o[0], o[1], o[2], o[3]));
        st_stream_v4(d + 8, make_uint4(o[4], o[5], o[6], o[7]));
      } else {
        for (int j = 0; j < nv; ++j) d[j] = (uint16_t)(o[j >> 1] >> (16 * (j & 1)));
      }
    }
  }
}

// src / hdr are device arrays of W entries (hdr: scratch).  err_dev[W]
// receives 0x7F7F7F7F per source when valid.
struct RedSrcs {
  RedSrc s[kMaxSegments];
};

__global__ void store_srcs_kernel(const RedSrcs v, int W, RedSrc* __restrict__ dst) {
  const int i = threadIdx.x;
  if (i < W) dst[i] = v.s[i];
}

// Stages up to kMaxSegments sources from the host into device memory with
// one tiny kernel (kernel parameters: no host staging buffer, no sync,
// capturable in a CUDA graph).
cudaError_t store_srcs(const RedSrc* host, int W, RedSrc* dst, cudaStream_t st) {
  if (W < 1 || W > kMaxSegments) return cudaErrorInvalidValue;
  RedSrcs v{};
  for (int i = 0; i < W; ++i) v.s[i] = host[i];
  store_srcs_kernel<<<1, kMaxSegments, 0, st>>>(v, W, dst);
  return cudaGetLastError();
}

cudaError_t launch_reduce(const RedSrc* src_dev, void* hdr_scratch, int W, int64_t n, void* out,
                          int out_f32, int32_t* err_dev, uint64_t epoch, int64_t timeout_ns,
                          cudaStream_t st) {
  if (W < 1) return cudaErrorInvalidValue;
  RedHdr* hdr_dev = reinterpret_cast<RedHdr*>(hdr_scratch);
  reduce_headers_kernel<<<(W + 127) / 128, 128, 0, st>>>(src_dev, W, n, hdr_dev, err_dev, epoch,
                                                          timeout_ns);
  if (n < 1) return cudaGetLastError();
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t groups = (n + 511) >> 9;
  const int64_t want = (groups + 7) / 8;                // 8 warps per CTA
  const int64_t cap = (int64_t)sms * 8;
  const unsigned grid = (unsigned)(want < cap ? (want > 0 ? want : 1) : cap);
  if (out_f32)
    reduce_kernel<true><<<grid, 256, 0, st>>>(src_dev, hdr_dev, W, n, out, err_dev);
  else
    reduce_kernel<false><<<grid, 256, 0, st>>>(src_dev, hdr_dev, W, n, out, err_dev);
  return cudaGetLastError();
}

size_t reduce_hdr_bytes(int W) { return sizeof(RedHdr) * (size_t)(W > 0 ? W : 1); }
size_t red_src_bytes() { return sizeof(RedSrc); }


// Loads every kernel of this file now (cudaFuncGetAttributes forces a
// lazily loaded module function in): with CUDA_MODULE_LOADING=LAZY, the
// first launch of a kernel waits for the device, which deadlocks while a
// peer rank sharing the GPU spins on a flag this rank has yet to publish.
cudaError_t preload_reduce() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, (const void*)reduce_headers_kernel);
  cudaFuncGetAttributes(&a, (const void*)reduce_kernel<false>);
  cudaFuncGetAttributes(&a, (const void*)reduce_kernel<true>);
  cudaFuncGetAttributes(&a, (const void*)store_srcs_kernel);
  return cudaGetLastError();
}

}  // namespace zc
