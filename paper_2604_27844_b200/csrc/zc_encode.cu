// K2/K4 — single-pass frame encoder (reference codec.compress codec.py:264-305
// fused with container.serialize container.py:65-95).
//
// One CTA = one 4096-element tile (256 threads x 16 elements).  A launch
// covers one or more independent segments (the per-peer chunks of an
// all-to-all); every segment gets its own frame and its own
// decoupled look-back chain for the escape prefix.  Per element the work is
// integer only:
//   sign-mantissa byte  ((w>>8)&0x80)|(w&0x7F)       -> 1 B/elem, 16-B stores
//   code = LUT[exponent] via a 256-entry "spread" table whose entry carries
//   the three plane bits and the escape bit at bit positions 0/8/16/24, so
//   8 elements OR into one register whose bytes are plane0/1/2/escape bytes
//   group_index / escapes positioned by the look-back prefix.
// Bytes per element: 2 read + ~1.40 written (HBM bound, no tensor cores).
#include "zc_common.cuh"

namespace zc {

__device__ __forceinline__ void write_header_and_pads(uint8_t* frame, const Layout& L,
                                                      uint64_t zc, const uint8_t* book) {
  const int t = threadIdx.x;
  // header: "<4sBBBBQQ7sB6I" + zero pad to 128 (container.py:45-46, :82-85)
  if (t < 128) {
    uint8_t b = 0;
    if (t < 4) b = "ZCCL"[t];
    else if (t == 4) b = 1;                                  // version
    else if (t == 6) b = (uint8_t)L.gs_log2;
    else if (t >= 8 && t < 16) b = (uint8_t)(uint64_t(L.n) >> (8 * (t - 8)));
    else if (t >= 16 && t < 24) b = (uint8_t)(zc >> (8 * (t - 16)));
    else if (t >= 24 && t < 31) b = book[t - 24];
    else if (t == 31) b = book[0];
    else if (t >= 32 && t < 56) {
      int i = (t - 32) >> 2;
      b = (uint8_t)(uint32_t(L.off[i]) >> (8 * ((t - 32) & 3)));
    }
    frame[t] = b;
  }
  // zero pads behind every section
  const int64_t ends[6] = {L.off[0] + L.n, L.off[1] + L.plane_bytes, L.off[2] + L.plane_bytes,
                           L.off[3] + L.plane_bytes, L.off[4] + 4 * L.groups,
                           L.off[5] + (int64_t)zc};
  const int64_t lims[6] = {L.off[1], L.off[2], L.off[3], L.off[4], L.off[5],
                           L.off[5] + pad128((int64_t)zc)};
  for (int r = 0; r < 6; ++r) {
    int64_t p = ends[r] + t;
    if (p < lims[r]) frame[p] = 0;
  }
}

__global__ void __launch_bounds__(kThreads)
encode_kernel(const uint16_t* __restrict__ x, const EncodeSegs segs,
              const uint8_t* __restrict__ book, uint8_t* __restrict__ frames,
              uint64_t* __restrict__ status, unsigned* __restrict__ counter,
              uint64_t* __restrict__ frame_len) {
  __shared__ uint32_t s_lut[256];
  __shared__ __align__(16) uint8_t s_exp[kTile];     // per-thread exponent bytes
  __shared__ uint8_t s_esc[kTile];                   // compacted escapes of the tile
  __shared__ uint32_t s_warp[kWarps];
  __shared__ int64_t s_tile;
  __shared__ uint64_t s_excl;
  __shared__ uint8_t s_book[8];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = (int64_t)atomicAdd(counter, 1u);
  if (tid < 7) s_book[tid] = book[tid];
  __syncthreads();
  {
    // spread LUT (codec.py:131-138 encode_table), bit0/8/16 = code bits, bit24 = escape
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < 7; ++i) c = (s_book[i] == tid) ? uint32_t(i + 1) : c;
    s_lut[tid] = (c & 1u) | ((c >> 1) & 1u) << 8 | ((c >> 2) & 1u) << 16 | uint32_t(c == 0) << 24;
  }
  const int64_t tile = s_tile;
  const int seg = find_seg(segs.tile_start, segs.nseg, tile);
  const int64_t n = segs.n[seg];
  const Layout L = layout_of(n, segs.gs_log2);
  uint8_t* frame = frames + segs.frame_off[seg];
  const uint16_t* xs = x + segs.x_off[seg];
  const int64_t t_local = tile - segs.tile_start[seg];
  const int64_t base = t_local * kTile + (int64_t)tid * kEPT;
  const int64_t nvalid = n - base;  // may be <= 0
  const bool full = nvalid >= kEPT;
  __syncthreads();

  // ---- load 16 words (two 16-B loads on the aligned fast path) ----------
  uint32_t w[8];
  if (full && ((reinterpret_cast<uintptr_t>(xs) & 15) == 0)) {
    uint4 a = ld_stream_v4(xs + base), b = ld_stream_v4(xs + base + 8);
    w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
    w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint32_t lo = (2 * k < nvalid) ? xs[base + 2 * k] : 0u;
      uint32_t hi = (2 * k + 1 < nvalid) ? xs[base + 2 * k + 1] : 0u;
      w[k] = lo | (hi << 16);
    }
  }
  const uint32_t valid16 = full ? 0xFFFFu : (nvalid > 0 ? ((1u << nvalid) - 1u) : 0u);

  // ---- sign-mantissa bytes (codec.py:279) ---------------------------------
  uint32_t sm[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t p = prmt(w[2 * j], w[2 * j + 1], 0x6420);   // low byte of each word
    uint32_t q = prmt(w[2 * j], w[2 * j + 1], 0x7531);   // high byte (sign | e7..e1)
    sm[j] = (p & 0x7F7F7F7Fu) | (q & 0x80808080u);
  }
  // ---- exponent bytes (bf16.py:39-41) staged for the escape path ----------
  {
    uint32_t e[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) e[j] = prmt(w[2 * j] >> 7, w[2 * j + 1] >> 7, 0x6420);
    *reinterpret_cast<uint4*>(s_exp + tid * kEPT) = make_uint4(e[0], e[1], e[2], e[3]);
  }
  // ---- codes -> plane bytes + escape mask (codec.py:281-289) --------------
  uint32_t A = 0, B = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t wl = w[k >> 1];
    const uint32_t e = (k & 1) ? ((wl >> 23) & 0xFFu) : ((wl >> 7) & 0xFFu);
    A |= s_lut[e] << k;
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t wl = w[4 + (k >> 1)];
    const uint32_t e = (k & 1) ? ((wl >> 23) & 0xFFu) : ((wl >> 7) & 0xFFu);
    B |= s_lut[e] << k;
  }
  if (!full) {
    A &= (valid16 & 0xFFu) * 0x01010101u;
    B &= ((valid16 >> 8) & 0xFFu) * 0x01010101u;
  }
  const uint32_t p0 = prmt(A, B, 0x40), p1 = prmt(A, B, 0x51), p2 = prmt(A, B, 0x62);
  const uint32_t esc = prmt(A, B, 0x73) & 0xFFFFu;

  // ---- static-section stores ----------------------------------------------
  if (full) {
    st_stream_v4(frame + L.off[0] + base, make_uint4(sm[0], sm[1], sm[2], sm[3]));
    const int64_t pb = base >> 3;
    *reinterpret_cast<uint16_t*>(frame + L.off[1] + pb) = (uint16_t)p0;
    *reinterpret_cast<uint16_t*>(frame + L.off[2] + pb) = (uint16_t)p1;
    *reinterpret_cast<uint16_t*>(frame + L.off[3] + pb) = (uint16_t)p2;
  } else if (nvalid > 0) {
    for (int k = 0; k < nvalid; ++k) frame[L.off[0] + base + k] = (uint8_t)(sm[k >> 2] >> (8 * (k & 3)));
    const int64_t pb = base >> 3;
    frame[L.off[1] + pb] = (uint8_t)p0;
    frame[L.off[2] + pb] = (uint8_t)p1;
    frame[L.off[3] + pb] = (uint8_t)p2;
    if (nvalid > 8) {
      frame[L.off[1] + pb + 1] = (uint8_t)(p0 >> 8);
      frame[L.off[2] + pb + 1] = (uint8_t)(p1 >> 8);
      frame[L.off[3] + pb + 1] = (uint8_t)(p2 >> 8);
    }
  }

  // ---- tile-local exclusive scan of escape counts --------------------------
  const uint32_t cnt = __popc(esc);
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  uint32_t wbase = 0, agg = 0;
#pragma unroll
  for (int i = 0; i < kWarps; ++i) {
    uint32_t v = s_warp[i];
    wbase += (i < warp) ? v : 0u;
    agg += v;
  }
  const uint32_t lp = wbase + incl - cnt;   // escapes in the tile before this thread

  // ---- compact escapes into shared memory (codec.py:283-284) ---------------
  {
    uint32_t m = esc, pos = lp;
    while (m) {
      const int k = __ffs(m) - 1;
      m &= m - 1;
      s_esc[pos++] = s_exp[tid * kEPT + k];
    }
  }

  // ---- decoupled look-back: escapes before this tile in the segment ---------
  if (warp == 0) {
    uint64_t ex = lookback_warp(status, tile, segs.tile_start[seg], agg, 0);
    if (lane == 0) s_excl = ex;
  }
  __syncthreads();
  const uint64_t excl = s_excl;

  // ---- group index: exclusive escape prefix at every group start (:291-295)
  if (nvalid > 0) {
    uint32_t* gi = reinterpret_cast<uint32_t*>(frame + L.off[4]);
    const int gsl = segs.gs_log2;
    if (gsl >= 4) {
      if ((base & ((int64_t(1) << gsl) - 1)) == 0) gi[base >> gsl] = (uint32_t)(excl + lp);
    } else {
      const int gs = 1 << gsl;
      for (int j = 0; j < kEPT && j < nvalid; j += gs)
        gi[(base + j) >> gsl] = (uint32_t)(excl + lp + __popc(esc & ((1u << j) - 1u)));
    }
  }
  // ---- escapes out (dynamic section) ---------------------------------------
  {
    uint8_t* dst = frame + L.off[5] + excl;
    for (uint32_t i = tid; i < agg; i += kThreads) dst[i] = s_esc[i];
  }
  // ---- last tile of the segment: header, pads, frame length ---------------
  const int64_t ntiles_seg = segs.tile_start[seg + 1] - segs.tile_start[seg];
  if (t_local == ntiles_seg - 1) {
    const uint64_t zc = excl + agg;
    write_header_and_pads(frame, L, zc, s_book);
    if (tid == 0) frame_len[seg] = (uint64_t)L.off[5] + (uint64_t)pad128((int64_t)zc);
  }
}

cudaError_t launch_encode(const uint16_t* x, const EncodeSegs& segs, const uint8_t* book,
                          uint8_t* frames, void* ws, uint64_t* frame_len, cudaStream_t st) {
  const int64_t ntiles = segs.tile_start[segs.nseg];
  unsigned* counter = reinterpret_cast<unsigned*>(ws);
  uint64_t* status = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(ws) + 128);
  cudaError_t e = cudaMemsetAsync(ws, 0, 128 + 8 * ntiles, st);
  if (e != cudaSuccess) return e;
  encode_kernel<<<(unsigned)ntiles, kThreads, 0, st>>>(x, segs, book, frames, status, counter,
                                                      frame_len);
  return cudaGetLastError();
}

}  // namespace zc
