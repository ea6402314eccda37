// K3/K5 — frame decoder + validator (reference container.parse
// container.py:113-180 + codec.decompress codec.py:315-327 with
// CompressedChunk.check_structure / _check_consistency :210-250).
//
// One CTA = one 4096-element tile.  Every CTA re-validates the 128-B header
// of its segment (cheap, L2-resident) so that no host round trip is needed
// when the frame arrived over NCCL or sits in a peer's HBM (P2P pull).
// group_index makes every group independently decodable, so for group sizes
// up to the tile size there is no cross-tile dependence at all: each group
// checks gi[g] + escapes(g) == gi[g+1] (or zero_count for the last group),
// which is exactly the reference's consistency rule.  Groups larger than a
// tile are walked with the same decoupled look-back as the encoder, seeded
// with gi[g] at the group's first tile.
//
// Per element: codes come from a 256-entry byte->nibble spread table (one
// LDS per plane byte), a single PRMT turns 4 nibble codes into 4 exponent
// bytes (the 7-entry book + escape slot is an 8-byte PRMT table), escapes
// are expanded into a per-thread 16-byte shared-memory slot and OR-ed in,
// and words are reassembled with two LOP3s per pair.
#include "zc_common.cuh"

namespace zc {

struct HeaderInfo {
  int64_t n, zc;
  int gsl;
  uint32_t tbl_lo, tbl_hi;   // PRMT decode table: byte c = entries[c-1], byte 0 = 0
  int32_t err;
};

// Mirrors container.parse_header + parse offset/length checks, in order.
__device__ HeaderInfo check_header(const uint8_t* h, int64_t expect_n, int64_t dyn_len) {
  HeaderInfo r{};
  const uint64_t q0 = reinterpret_cast<const uint64_t*>(h)[0];
  const uint64_t n = reinterpret_cast<const uint64_t*>(h)[1];
  const uint64_t zc = reinterpret_cast<const uint64_t*>(h)[2];
  const uint64_t q3 = reinterpret_cast<const uint64_t*>(h)[3];
  const uint32_t* offs = reinterpret_cast<const uint32_t*>(h + 32);
  const uint32_t magic = (uint32_t)q0;
  const int version = (int)((q0 >> 32) & 0xFF), flags = (int)((q0 >> 40) & 0xFF);
  const int gsl = (int)((q0 >> 48) & 0xFF);
  r.err = kOk;
  if (magic != 0x4C43435Au) { r.err = kErrMagic; return r; }   // "ZCCL"
  if (version != 1) { r.err = kErrVersion; return r; }
  if (flags != 0) { r.err = kErrFlags; return r; }
  if (gsl > 30) { r.err = kErrGsLog2; return r; }
  if (n < 1) { r.err = kErrElementCount; return r; }
  if (zc > n) { r.err = kErrZeroCountHeader; return r; }
  uint8_t e[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) e[i] = (uint8_t)(q3 >> (8 * i));
  for (int i = 0; i < 7; ++i)
    for (int j = i + 1; j < 7; ++j)
      if (e[i] == e[j]) { r.err = kErrCodebookDistinct; return r; }
  if (e[7] != e[0]) { r.err = kErrCodebookBase; return r; }
  if (n > (uint64_t(1) << 40)) { r.err = kErrOffset0 + 1; return r; }
  const Layout L = layout_of((int64_t)n, gsl);
  for (int i = 0; i < 6; ++i)
    if ((int64_t)offs[i] != L.off[i]) { r.err = kErrOffset0 + i; return r; }
  if (dyn_len >= 0 && dyn_len != pad128((int64_t)zc)) { r.err = kErrFrameLength; return r; }
  if (expect_n >= 0 && (int64_t)n != expect_n) { r.err = kErrCountMismatch; return r; }
  r.n = (int64_t)n;
  r.zc = (int64_t)zc;
  r.gsl = gsl;
  r.tbl_lo = (uint32_t)e[0] << 8 | (uint32_t)e[1] << 16 | (uint32_t)e[2] << 24;
  r.tbl_hi = (uint32_t)e[3] | (uint32_t)e[4] << 8 | (uint32_t)e[5] << 16 | (uint32_t)e[6] << 24;
  return r;
}

__device__ __forceinline__ uint32_t reassemble2(uint32_t v) {
  // v = [s0, e0, s1, e1] -> two bf16 words (codec.py:308-312)
  return (v & 0x007F007Fu) | ((v >> 1) & 0x7F807F80u) | ((v << 8) & 0x80008000u);
}

__global__ void __launch_bounds__(kThreads)
decode_kernel(const DecodeSegs segs, uint16_t* __restrict__ out, int32_t* __restrict__ err,
              uint64_t* __restrict__ status, unsigned* __restrict__ counter, int write_out) {
  __shared__ uint32_t s_spread[256];
  __shared__ __align__(16) uint8_t s_dense[kTile];
  __shared__ uint32_t s_lp[kThreads + 1];
  __shared__ uint32_t s_warp[kWarps];
  __shared__ HeaderInfo s_hdr;
  __shared__ int64_t s_tile;
  __shared__ int64_t s_excl;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = (int64_t)atomicAdd(counter, 1u);
  {
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) v |= ((uint32_t(tid) >> k) & 1u) << (4 * k);
    s_spread[tid] = v;
  }
  __syncthreads();
  const int64_t tile = s_tile;
  const int seg = find_seg(segs.tile_start, segs.nseg, tile);
  const uint8_t* frame = segs.stat[seg];
  if (tid == 0) s_hdr = check_header(frame, segs.n[seg], segs.dyn_len[seg]);
  __syncthreads();
  const HeaderInfo H = s_hdr;
  if (H.err != kOk) {
    if (tid == 0) atomicMin(err + seg, H.err);
    return;
  }
  const int64_t n = H.n;
  const int gsl = H.gsl;
  const Layout L = layout_of(n, gsl);
  const uint8_t* dyn = segs.dyn[seg] ? segs.dyn[seg] : frame + L.off[5];
  const uint32_t* gi = reinterpret_cast<const uint32_t*>(frame + L.off[4]);
  const int64_t t_local = tile - segs.tile_start[seg];
  const int64_t tile_base = t_local * kTile;
  const int64_t base = tile_base + (int64_t)tid * kEPT;
  const int64_t nvalid = n - base;
  const bool full = nvalid >= kEPT;
  int32_t my_err = kOk;

  // ---- static-section loads -------------------------------------------------
  uint32_t S[4] = {0, 0, 0, 0};
  uint32_t p0 = 0, p1 = 0, p2 = 0;
  if (full) {
    const uint4 s = ld_stream_v4(frame + L.off[0] + base);
    S[0] = s.x; S[1] = s.y; S[2] = s.z; S[3] = s.w;
    const int64_t pb = base >> 3;
    p0 = *reinterpret_cast<const uint16_t*>(frame + L.off[1] + pb);
    p1 = *reinterpret_cast<const uint16_t*>(frame + L.off[2] + pb);
    p2 = *reinterpret_cast<const uint16_t*>(frame + L.off[3] + pb);
  } else if (nvalid > 0) {
    for (int k = 0; k < nvalid; ++k) S[k >> 2] |= (uint32_t)frame[L.off[0] + base + k] << (8 * (k & 3));
    const int64_t pb = base >> 3;
    p0 = frame[L.off[1] + pb]; p1 = frame[L.off[2] + pb]; p2 = frame[L.off[3] + pb];
    if (nvalid > 8) {
      p0 |= (uint32_t)frame[L.off[1] + pb + 1] << 8;
      p1 |= (uint32_t)frame[L.off[2] + pb + 1] << 8;
      p2 |= (uint32_t)frame[L.off[3] + pb + 1] << 8;
    }
  }
  const uint32_t valid16 = full ? 0xFFFFu : (nvalid > 0 ? ((1u << nvalid) - 1u) : 0u);
  const uint32_t esc = ~(p0 | p1 | p2) & valid16;

  // ---- tile-local scan of escape counts ------------------------------------
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
    const uint32_t v = s_warp[i];
    wbase += (i < warp) ? v : 0u;
    agg += v;
  }
  const uint32_t lp = wbase + incl - cnt;
  s_lp[tid] = lp;
  if (tid == kThreads - 1) s_lp[kThreads] = agg;

  // ---- escape base + consistency (codec.py:238-250) ------------------------
  int64_t ebase = 0;   // escapes before this thread's first element (segment-global)
  if (gsl > 12) {
    const int64_t g = tile_base >> gsl;
    const int64_t chain_first = segs.tile_start[seg] + ((g << gsl) / kTile);
    if (warp == 0) {
      const int64_t seed = (int64_t)gi[g];
      const uint64_t ex = lookback_warp(status, tile, chain_first, agg, (uint64_t)seed);
      if (lane == 0) s_excl = (int64_t)ex;
    }
    __syncthreads();
    ebase = s_excl + lp;
    const int64_t ntl = segs.tile_start[seg + 1] - segs.tile_start[seg];
    const bool last_of_group = (t_local == ntl - 1) || (((tile_base + kTile) >> gsl) != g);
    if (tid == 0) {
      if (t_local == 0 && gi[0] != 0) my_err = kErrGroupIndex;
      if (last_of_group) {
        const int64_t next = (g + 1 < L.groups) ? (int64_t)gi[g + 1] : H.zc;
        if (s_excl + (int64_t)agg != next) my_err = (g + 1 < L.groups) ? kErrGroupIndex : kErrZeroCount;
      }
    }
  } else {
    __syncthreads();   // s_lp complete
    if (nvalid > 0) {
      if (gsl >= 4) {
        const int64_t g = base >> gsl;
        const int gtid = (int)(((g << gsl) - tile_base) / kEPT);
        const int64_t gv = (int64_t)gi[g];
        ebase = gv + lp - s_lp[gtid];
        if (gtid == tid) {   // group start: check the whole group
          const int etid = gtid + (1 << (gsl - 4));
          const int64_t c = (int64_t)s_lp[etid < kThreads ? etid : kThreads] - lp;
          if (g == 0 && gv != 0) my_err = kErrGroupIndex;
          const int64_t next = (g + 1 < L.groups) ? (int64_t)gi[g + 1] : H.zc;
          if (gv + c != next) my_err = (g + 1 < L.groups) ? kErrGroupIndex : kErrZeroCount;
        }
      } else {
        const int gs = 1 << gsl;
        for (int j = 0; j < kEPT && j < nvalid; j += gs) {
          const int64_t g = (base + j) >> gsl;
          const int64_t gv = (int64_t)gi[g];
          const uint32_t gm = ((gs >= 32) ? 0xFFFFFFFFu : ((1u << gs) - 1u)) << j;
          const int64_t c = __popc(esc & gm);
          if (g == 0 && gv != 0) my_err = kErrGroupIndex;
          const int64_t next = (g + 1 < L.groups) ? (int64_t)gi[g + 1] : H.zc;
          if (gv + c != next) my_err = (g + 1 < L.groups) ? kErrGroupIndex : kErrZeroCount;
        }
      }
    }
  }

  // ---- exponents: codes -> PRMT table lookup -------------------------------
  uint32_t E[4];
  {
    const uint32_t lo = s_spread[p0 & 0xFF] | s_spread[p1 & 0xFF] << 1 | s_spread[p2 & 0xFF] << 2;
    const uint32_t hi = s_spread[(p0 >> 8) & 0xFF] | s_spread[(p1 >> 8) & 0xFF] << 1 |
                        s_spread[(p2 >> 8) & 0xFF] << 2;
    E[0] = prmt(H.tbl_lo, H.tbl_hi, lo);
    E[1] = prmt(H.tbl_lo, H.tbl_hi, lo >> 16);
    E[2] = prmt(H.tbl_lo, H.tbl_hi, hi);
    E[3] = prmt(H.tbl_lo, H.tbl_hi, hi >> 16);
  }
  // ---- escapes: expand into a dense per-thread slot ------------------------
  if (__syncthreads_or(esc != 0)) {
    uint8_t* slot = s_dense + tid * kEPT;
    *reinterpret_cast<uint4*>(slot) = make_uint4(0, 0, 0, 0);
    uint32_t m = esc;
    while (m) {
      const int k = __ffs(m) - 1;
      m &= m - 1;
      int64_t pos;
      if (gsl >= 4 || gsl > 12) {
        pos = ebase + __popc(esc & ((1u << k) - 1u));
      } else {
        const int64_t g = (base + k) >> gsl;
        const int j0 = (int)((g << gsl) - base);
        pos = (int64_t)gi[g] + __popc(esc & ((1u << k) - 1u)) - __popc(esc & ((1u << j0) - 1u));
      }
      uint8_t v = 0;
      if (pos < H.zc) {
        if (write_out) v = dyn[pos];
      } else {
        // out-of-range escape position: always accompanied by a failing group
        // check, which carries the field the reference names; lowest priority
        my_err = kErrZeroCount;
      }
      slot[k] = v;
    }
    const uint4 d = *reinterpret_cast<const uint4*>(slot);
    E[0] |= d.x; E[1] |= d.y; E[2] |= d.z; E[3] |= d.w;
  }
  if (my_err != kOk) atomicMin(err + seg, my_err);
  if (!write_out || nvalid <= 0) return;

  // ---- reassemble (codec.py:308-312) and store -----------------------------
  uint32_t o[8];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    o[2 * j] = reassemble2(prmt(S[j], E[j], 0x5140));
    o[2 * j + 1] = reassemble2(prmt(S[j], E[j], 0x7362));
  }
  uint16_t* dst = out + segs.out_off[seg] + base;
  if (full && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
    st_stream_v4(dst, make_uint4(o[0], o[1], o[2], o[3]));
    st_stream_v4(dst + 8, make_uint4(o[4], o[5], o[6], o[7]));
  } else {
    const int lim = full ? kEPT : (int)nvalid;
    for (int k = 0; k < lim; ++k) dst[k] = (uint16_t)(o[k >> 1] >> (16 * (k & 1)));
  }
}

cudaError_t launch_decode(const DecodeSegs& segs, uint16_t* out, int32_t* err, void* ws,
                          int write_out, cudaStream_t st) {
  const int64_t ntiles = segs.tile_start[segs.nseg];
  unsigned* counter = reinterpret_cast<unsigned*>(ws);
  uint64_t* status = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(ws) + 128);
  cudaError_t e = cudaMemsetAsync(ws, 0, 128 + 8 * ntiles, st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(err, 0x7F, sizeof(int32_t) * segs.nseg, st);
  if (e != cudaSuccess) return e;
  if (ntiles == 0) return cudaSuccess;
  decode_kernel<<<(unsigned)ntiles, kThreads, 0, st>>>(segs, out, err, status, counter, write_out);
  return cudaGetLastError();
}

}  // namespace zc
