// K3/K5 — frame decoder + validator (reference container.parse
// container.py:113-180 + codec.decompress codec.py:315-327 with
// CompressedChunk.check_structure / _check_consistency :210-250).
//
// Persistent kernel: each CTA claims 4096-element tiles from an atomic
// counter and prefetches the next tile's static-section bytes while decoding
// the current one.  The 128-B header of a segment is validated once per CTA
// per segment (so a frame that arrived over NCCL or sits in a peer's HBM
// needs no host round trip).  group_index makes every group independently
// decodable, so for group sizes up to the tile there is no cross-tile
// dependence: each group checks gi[g] + escapes(g) == gi[g+1] (zero_count for
// the last group) -- exactly the reference's consistency rule.  Groups larger
// than a tile are walked with the encoder's decoupled look-back, seeded with
// gi[g] at the group's first tile.
//
// Per element: codes come from a 256-entry byte->nibble spread table (one LDS
// per plane byte), one PRMT maps 4 nibble codes to 4 exponent bytes (the
// 7-entry book + escape slot is an 8-byte PRMT table), escapes are expanded
// into a per-thread 16-B shared slot and OR-ed in, and output words are built
// four at a time from (sm, exponent) byte vectors with two LOP3 and two PRMT.
#include <cstdlib>
#include "zc_common.cuh"

namespace zc {

struct StaticBits {
  uint4 s;                 // 16 sign-mantissa bytes
  uint32_t p0, p1, p2;     // 16 plane bits each
};

__device__ __forceinline__ void load_static(const uint8_t* frame, const Layout& L, int64_t base,
                                            int64_t nvalid, StaticBits& b) {
  b.s = make_uint4(0, 0, 0, 0);
  b.p0 = b.p1 = b.p2 = 0;
  if (nvalid >= kEPT) {
    b.s = ld_stream_v4(frame + L.off[0] + base);
    const int64_t pb = base >> 3;
    b.p0 = *reinterpret_cast<const uint16_t*>(frame + L.off[1] + pb);
    b.p1 = *reinterpret_cast<const uint16_t*>(frame + L.off[2] + pb);
    b.p2 = *reinterpret_cast<const uint16_t*>(frame + L.off[3] + pb);
  } else if (nvalid > 0) {
    uint32_t S[4] = {0, 0, 0, 0};
    for (int k = 0; k < nvalid; ++k) S[k >> 2] |= (uint32_t)frame[L.off[0] + base + k] << (8 * (k & 3));
    b.s = make_uint4(S[0], S[1], S[2], S[3]);
    const int64_t pb = base >> 3;
    b.p0 = frame[L.off[1] + pb]; b.p1 = frame[L.off[2] + pb]; b.p2 = frame[L.off[3] + pb];
    if (nvalid > 8) {
      b.p0 |= (uint32_t)frame[L.off[1] + pb + 1] << 8;
      b.p1 |= (uint32_t)frame[L.off[2] + pb + 1] << 8;
      b.p2 |= (uint32_t)frame[L.off[3] + pb + 1] << 8;
    }
  }
}

// 4 output words from 4 sign-mantissa bytes S and 4 exponent bytes E
// (codec.py:308-312): lo byte = e0<<7 | s&0x7F, hi byte = s&0x80 | e>>1.
__device__ __forceinline__ void reassemble4(uint32_t S, uint32_t E, uint32_t& o01, uint32_t& o23) {
  const uint32_t lo = bitsel(0x80808080u, E << 7, S);
  const uint32_t hi = bitsel(0x80808080u, S, E >> 1);
  o01 = prmt(lo, hi, 0x5140);
  o23 = prmt(lo, hi, 0x7362);
}

__global__ void __launch_bounds__(kThreads)
decode_lookback_kernel(const DecodeSegs segs, uint16_t* __restrict__ out, int32_t* __restrict__ err,
              uint64_t* __restrict__ status, unsigned* __restrict__ counter, int write_out) {
  __shared__ uint32_t s_spread[256];
  __shared__ __align__(16) uint8_t s_dense[kTile];
  __shared__ uint32_t s_lp[kThreads + 1];
  __shared__ __align__(16) uint32_t s_warp[kWarps];
  __shared__ HeaderInfo s_hdr;
  __shared__ int s_hdr_seg;
  __shared__ int64_t s_claim[2];
  __shared__ int64_t s_excl;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t ntiles = segs.tile_start[segs.nseg];
  if (tid == 0) {
    s_claim[0] = (int64_t)atomicAdd(counter, 1u);
    s_claim[1] = (int64_t)atomicAdd(counter, 1u);
    s_hdr_seg = -1;
  }
  {
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) v |= ((uint32_t(tid) >> k) & 1u) << (4 * k);
    s_spread[tid] = v;
  }
  __syncthreads();
  int64_t cur = s_claim[0], nxt = s_claim[1];

  // The static bytes of a tile can be prefetched before its header is checked
  // only when the layout is known: prefetch uses the caller's expected n and
  // the header's group size is only needed for gi, so layout offsets are
  // computed from the expected count (the header check rejects mismatches).
  auto layout_for = [&](int s) { return layout_of(segs.n[s], 0); };

  StaticBits cb;
  if (cur < ntiles) {
    const int s = find_seg(segs.tile_start, segs.nseg, cur);
    const int64_t base = (cur - segs.tile_start[s]) * kTile + (int64_t)tid * kEPT;
    load_static(segs.stat[s], layout_for(s), base, segs.n[s] - base, cb);
  }
  int it = 0;
  while (cur < ntiles) {
    StaticBits nb;
    if (nxt < ntiles) {
      const int s = find_seg(segs.tile_start, segs.nseg, nxt);
      const int64_t b2 = (nxt - segs.tile_start[s]) * kTile + (int64_t)tid * kEPT;
      load_static(segs.stat[s], layout_for(s), b2, segs.n[s] - b2, nb);
    }
    const int seg = find_seg(segs.tile_start, segs.nseg, cur);
    const uint8_t* frame = segs.stat[seg];
    if (seg != s_hdr_seg) {            // uniform: s_hdr_seg only changes between barriers
      __syncthreads();
      if (tid == 0) {
        s_hdr = check_header(frame, segs.n[seg], segs.dyn_len[seg]);
        s_hdr_seg = seg;
      }
      __syncthreads();
    }
    const HeaderInfo H = s_hdr;
    if (tid == 0) s_claim[it & 1] = (int64_t)atomicAdd(counter, 1u);
    if (H.err != kOk) {
      if (tid == 0) atomicMin(err + seg, H.err);
      __syncthreads();
      cur = nxt;
      nxt = s_claim[it & 1];
      cb = nb;
      ++it;
      __syncthreads();
      continue;
    }
    const int64_t n = H.n;
    const int gsl = H.gsl;
    const Layout L = layout_of(n, gsl);
    const uint8_t* dyn = segs.dyn[seg] ? segs.dyn[seg] : frame + L.off[5];
    const uint32_t* gi = reinterpret_cast<const uint32_t*>(frame + L.off[4]);
    const int64_t seg_t0 = segs.tile_start[seg];
    const int64_t t_local = cur - seg_t0;
    const int64_t tile_base = t_local * kTile;
    const int64_t base = tile_base + (int64_t)tid * kEPT;
    const int64_t nvalid = n - base;
    const bool full = nvalid >= kEPT;
    int32_t my_err = kOk;

    const uint32_t valid16 = full ? 0xFFFFu : (nvalid > 0 ? ((1u << nvalid) - 1u) : 0u);
    const uint32_t p0 = cb.p0, p1 = cb.p1, p2 = cb.p2;
    const uint32_t esc = ~(p0 | p1 | p2) & valid16;

    // ---- tile-local scan of escape counts --------------------------------
    const uint32_t cnt = __popc(esc);
    uint32_t incl = warp_incl_scan(cnt);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();                                     // (B)
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

    // ---- escape base + consistency (codec.py:238-250) ---------------------
    int64_t ebase = 0;
    if (gsl > 12) {
      const int64_t g = tile_base >> gsl;
      const int64_t chain_first = seg_t0 + ((g << gsl) / kTile);
      if (warp == 0) {
        const uint64_t ex = lookback_warp(status, cur, chain_first, agg, (uint64_t)gi[g]);
        if (lane == 0) s_excl = (int64_t)ex;
      }
      __syncthreads();                                   // (C)
      ebase = s_excl + lp;
      const int64_t ntl = segs.tile_start[seg + 1] - seg_t0;
      const bool last_of_group = (t_local == ntl - 1) || (((tile_base + kTile) >> gsl) != g);
      if (tid == 0) {
        if (t_local == 0 && gi[0] != 0) my_err = kErrGroupIndex;
        if (last_of_group) {
          const int64_t next = (g + 1 < L.groups) ? (int64_t)gi[g + 1] : H.zc;
          if (s_excl + (int64_t)agg != next)
            my_err = (g + 1 < L.groups) ? kErrGroupIndex : kErrZeroCount;
        }
      }
    } else {
      __syncthreads();                                   // (C) s_lp complete
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
            const uint32_t gm = ((1u << gs) - 1u) << j;
            const int64_t c = __popc(esc & gm);
            if (g == 0 && gv != 0) my_err = kErrGroupIndex;
            const int64_t next = (g + 1 < L.groups) ? (int64_t)gi[g + 1] : H.zc;
            if (gv + c != next) my_err = (g + 1 < L.groups) ? kErrGroupIndex : kErrZeroCount;
          }
        }
      }
    }

    // ---- exponents: codes -> PRMT table lookup ---------------------------
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
    // ---- escapes: expand into a dense per-thread slot ---------------------
    if (esc) {
      uint8_t* slot = s_dense + tid * kEPT;
      *reinterpret_cast<uint4*>(slot) = make_uint4(0, 0, 0, 0);
      uint32_t m = esc;
      while (m) {
        const int k = __ffs(m) - 1;
        m &= m - 1;
        int64_t pos;
        if (gsl >= 4) {
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
          // out-of-range escape position: always accompanied by a failing
          // group check, which carries the field the reference names
          my_err = kErrZeroCount;
        }
        slot[k] = v;
      }
      const uint4 d = *reinterpret_cast<const uint4*>(slot);
      E[0] |= d.x; E[1] |= d.y; E[2] |= d.z; E[3] |= d.w;
    }
    if (my_err != kOk) atomicMin(err + seg, my_err);

    // ---- reassemble (codec.py:308-312) and store --------------------------
    if (write_out && nvalid > 0) {
      uint32_t o[8];
      reassemble4(cb.s.x, E[0], o[0], o[1]);
      reassemble4(cb.s.y, E[1], o[2], o[3]);
      reassemble4(cb.s.z, E[2], o[4], o[5]);
      reassemble4(cb.s.w, E[3], o[6], o[7]);
      uint16_t* dst = out + segs.out_off[seg] + base;
      if (full && ((reinterpret_cast<uintptr_t>(dst) & 31) == 0)) {
        st_v8(dst, make_uint4(o[0], o[1], o[2], o[3]), make_uint4(o[4], o[5], o[6], o[7]));
      } else if (full && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
        st_stream_v4(dst, make_uint4(o[0], o[1], o[2], o[3]));
        st_stream_v4(dst + 8, make_uint4(o[4], o[5], o[6], o[7]));
      } else {
        const int lim = full ? kEPT : (int)nvalid;
        for (int k = 0; k < lim; ++k) dst[k] = (uint16_t)(o[k >> 1] >> (16 * (k & 1)));
      }
    }
    __syncthreads();                                     // (D) claim visible, smem reuse
    cur = nxt;
    nxt = s_claim[it & 1];
    cb = nb;
    ++it;
  }
}

// ============================================================================
// Ring decoder (group size <= tile, i.e. every tile starts a group — always
// the case for the collectives' 512).  Warp-specialised: warp 0 is the
// producer, warps 1..8 decode.  Each CTA owns a contiguous run of tiles of
// one segment.  For every tile the producer stages, with TMA bulk copies into
// a kStages ring: the 4 KB sign-mantissa slice, the three 512 B plane slices,
// the tile's group_index slice and the tile's escape bytes (their range is
// [gi[first group of tile], gi[first group of next tile]) — the producer
// warp fetches 32 tile boundaries at a time).  Consumers therefore never
// wait on global memory: every escape is read from shared memory at its
// tile-local rank, and consistency is checked as gi[g] == gi[tile] +
// escapes-before-g inside the tile plus gi[tile] + tile escapes ==
// gi[next tile] (zero_count after the last tile) — equivalent to the
// reference's diff(gi) == per-group escapes, gi[0] == 0, sum == zero_count.
// ============================================================================

#ifndef ZC_DSTAGES
#define ZC_DSTAGES 4
#endif
#ifndef ZC_DMINB
#define ZC_DMINB 3
#endif
#ifndef ZC_DCHUNK
#define ZC_DCHUNK 4
#endif
constexpr int kDStages = ZC_DSTAGES;
constexpr int kDChunk = ZC_DCHUNK;                  // tiles per dynamic claim
constexpr int kGiSlots = 264;                       // up to 257 gi entries (gs >= 16) + align
// Every escape byte of a tile is staged (a smaller slot with a global-memory
// overflow path measured 4 % slower: the extra select alone cost registers).
constexpr int kEscSlots = kTile + 32;
struct __align__(128) DStage {
  uint8_t sm[kTile];
  uint8_t pl[3][kTile / 8];
  uint32_t gi[kGiSlots];
  uint8_t esc[kEscSlots];
};
constexpr int kDStageBytes = sizeof(DStage);
#ifndef ZC_DGROUPS
#define ZC_DGROUPS 2
#endif
constexpr int kDGroups = ZC_DGROUPS;               // consumer groups of 4 warps
constexpr int kDThreads = 32 + 128 * kDGroups;

// Work is handed out dynamically in chunks of kDChunk tiles of one segment
// (an atomic counter, claimed one chunk ahead by the producer): HBM bandwidth
// is not shared evenly between SMs, and with static runs the CTAs finished
// between 79 and 150 us of a 150 us launch (scripts/exp/timeline.py).
struct DChunkPlan {
  int64_t chunk_start[kMaxSegments + 1];            // prefix of per-segment chunk counts
  int64_t chunk;                                    // tiles per claim (kDChunk; fewer for small inputs)
};

__device__ __forceinline__ uint32_t r16(uint64_t x) { return (uint32_t)((x + 15) & ~uint64_t(15)); }

// Dense-escape expansion (escape-heavy data): the thread's escape bytes are
// consecutive in the staged section, eb[0 .. popc(esc)).  For every nibble of
// esc (4 words) one unaligned 4-byte read (two aligned LDS.32 + PRMT) and one
// PRMT with the nibble's expand selector (s_xsel: byte j <- next escape byte
// when bit j is set, else a zero byte) OR the escape exponents into E.
__device__ __forceinline__ void expand_escapes(const uint8_t* eb, uint32_t esc, uint32_t* E,
                                               const uint32_t* s_xsel) {
  uint32_t o = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const uint32_t m4 = (esc >> (4 * q)) & 0xFu;
    if (m4) {
      const uintptr_t p = reinterpret_cast<uintptr_t>(eb + o);
      const uint32_t* pw = reinterpret_cast<const uint32_t*>(p & ~uintptr_t(3));
      const uint32_t src = prmt(pw[0], pw[1], 0x3210u + 0x1111u * (uint32_t)(p & 3));
      E[q] |= prmt(src, 0u, s_xsel[m4]);
      o += __popc(m4);
    }
  }
}

// kPull: segments are peer frames that become readable at different times
// (the peer-memory collectives).  Headers are validated lazily,
// when a CTA first touches a segment after its ready flag reached the epoch,
// and work is claimed per segment (one counter each, counter[1 + s]) from
// whichever segment is ready, starting at blockIdx % nseg: decoding of an
// early peer's frame never waits for a late one.
template <bool kPull>
__global__ void __launch_bounds__(kDThreads, ZC_DMINB)   // CTAs / SM (register cap)
decode_ring_kernel(const DecodeSegs segs, const DChunkPlan cp, uint16_t* __restrict__ out,
                   int32_t* __restrict__ err, unsigned* __restrict__ counter, int write_out) {
  extern __shared__ __align__(128) uint8_t s_dyn[];
  DStage* ring = reinterpret_cast<DStage*>(s_dyn);
  uint64_t* full = reinterpret_cast<uint64_t*>(s_dyn + kDStages * kDStageBytes);
  uint64_t* empty = full + kDStages;
  __shared__ __align__(16) uint32_t s_wsum[kDGroups][2][8];   // group x parity x virtual warp
  __shared__ HeaderInfo s_hdr[kMaxSegments];
  // what the pull-mode consumers need of a segment beyond its header, next
  // to it (written by the producer when it validates the segment)
  struct __align__(16) SegCons { const uint32_t* gi; uint16_t* out; int64_t groups; uint32_t flags; };
  __shared__ SegCons s_cons[kMaxSegments];
  auto fill_cons = [&](int s2, const HeaderInfo& h) {
    const Layout L = layout_of(h.n, h.gsl);
    uint16_t* o = out + segs.out_off[s2];
    const uint32_t f = (write_out && (reinterpret_cast<uintptr_t>(o) & 15) == 0 ? 1u : 0u) |
                       (write_out && (reinterpret_cast<uintptr_t>(o) & 31) == 0 ? 2u : 0u);
    s_cons[s2] = SegCons{reinterpret_cast<const uint32_t*>(segs.stat[s2] + L.off[4]), o, L.groups, f};
  };
  // per-stage metadata, one 16-B store / load: escape range start (lo),
  // length, offset of lo in the staged escape bytes, and tile (24 bits) |
  // segment (6) | group_index alignment shift (2); all ones = end marker
  struct __align__(16) StageMeta { uint32_t lo, cnt; int32_t esc_off; uint32_t tsg; };
  static_assert(kMaxSegments <= 64, "segment field");
  __shared__ StageMeta s_meta[kDStages];
  __shared__ uint32_t s_spread[256];
  __shared__ __align__(16) uint8_t s_slot[kDGroups * 128 * 32];
  __shared__ uint32_t s_xsel[16];                    // expand selectors (expand_escapes)

  const int tid = threadIdx.x;
  ZC_TL(0, 0);
  ZC_TL_SMID(2);
  if (tid >= 32 && tid < 32 + 256) {
    const int v = tid - 32;   // byte -> nibble spread: bit k -> bit 4k
    uint32_t sp = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) sp |= ((uint32_t(v) >> k) & 1u) << (4 * k);
    s_spread[v] = sp;
  }
  if (tid < 16) {
    const uint32_t m = tid;
    uint32_t sel = 0, c = 0;
    for (int j = 0; j < 4; ++j) {
      sel |= (((m >> j) & 1u) ? c++ : 4u) << (4 * j);
    }
    s_xsel[m] = sel;
  }
  if (!kPull && tid < segs.nseg) {   // every segment's header, validated once per CTA
    HeaderInfo h = check_header(segs.stat[tid], segs.n[tid], segs.dyn_len[tid]);
    // groups must fit one tile here (gi slices, per-tile escape bounds);
    // larger groups are the look-back decoder's (flags bit 1)
    if (h.err == kOk && h.gsl > 12) h.err = kErrGroupTooLarge;
    s_hdr[tid] = h;
    if (h.err != kOk && blockIdx.x == 0) atomicMin(err + tid, h.err);
  }
  if (tid == 0) {
    for (int i = 0; i < kDStages; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, kWarps / 2);             // the 4 warps of one consumer group
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t nchunks = cp.chunk_start[segs.nseg];

  if (tid < 32) {
    // ======================= producer warp ===============================
    const int lane = tid;
    int64_t k = 0;                                   // stages issued
    unsigned cl = 0;
    // pull mode bookkeeping (lane 0): segments exhausted / header-checked
    unsigned long long seg_done = 0, seg_checked = 0;
    const unsigned long long all_segs =
        segs.nseg >= 64 ? ~0ull : ((1ull << segs.nseg) - 1ull);
    int cur = segs.nseg ? (int)(blockIdx.x % (unsigned)segs.nseg) : 0;
    const uint64_t t_begin = kPull ? globaltimer_ns() : 0;
    // pull mode: the next chunk of the segment just selected is claimed
    // right away and used on the next iteration, so the claim's round trip
    // overlaps this chunk's issue (as the push path's one-ahead claim)
    int pend_seg = -1;
    unsigned pend = 0;
    if (!kPull && lane == 0) cl = atomicAdd(counter, 1u);
    int64_t c = (int64_t)__shfl_sync(0xffffffffu, cl, 0);
    while (true) {
      unsigned nx = 0;
      int seg = 0;
      if constexpr (kPull) {
        int sel = -1, stop = 0;
        unsigned sel_c = 0;
        if (lane == 0) {
          if (pend_seg >= 0) {
            if ((int64_t)pend < cp.chunk_start[pend_seg + 1] - cp.chunk_start[pend_seg]) {
              sel = pend_seg;
              sel_c = pend;
            } else {
              seg_done |= 1ull << pend_seg;
            }
            pend_seg = -1;
          }
          for (int i = 0; i < segs.nseg && sel < 0; ++i) {
            const int s2 = (cur + i) % segs.nseg;
            if ((seg_done >> s2) & 1ull) continue;
            if (!((seg_checked >> s2) & 1ull)) {
              if (segs.ready[s2] && ld_acquire_sys_u64(segs.ready[s2]) < segs.epoch) continue;
              // the peer's frame is complete: order the async-proxy (TMA)
              // reads below after the acquire
              asm volatile("fence.proxy.async;" ::: "memory");
              HeaderInfo h = check_header(segs.stat[s2], segs.n[s2], segs.dyn_len[s2]);
              if (h.err == kOk && h.gsl > 12) h.err = kErrGroupTooLarge;
              s_hdr[s2] = h;
              if (h.err == kOk) fill_cons(s2, h);
              seg_checked |= 1ull << s2;
              if (h.err != kOk) {
                atomicMin(err + s2, h.err);
                seg_done |= 1ull << s2;
                continue;
              }
            }
            const unsigned cc = atomicAdd(counter + 1 + s2, 1u);
            if ((int64_t)cc >= cp.chunk_start[s2 + 1] - cp.chunk_start[s2]) {
              seg_done |= 1ull << s2;
              continue;
            }
            sel = s2;
            sel_c = cc;
            cur = s2;
          }
          if (sel >= 0) {
            pend = atomicAdd(counter + 1 + sel, 1u);   // consumed next iteration
            pend_seg = sel;
          }
          if (sel < 0) {
            if (seg_done == all_segs) {
              stop = 1;
            } else if (segs.timeout_ns > 0 &&
                       (int64_t)(globaltimer_ns() - t_begin) > segs.timeout_ns) {
              for (int s2 = 0; s2 < segs.nseg; ++s2)
                if (!((seg_done >> s2) & 1ull)) atomicMin(err + s2, (int32_t)kErrTimeout);
              stop = 1;
            } else {
              __nanosleep(128);
            }
          }
        }
        stop = __shfl_sync(0xffffffffu, stop, 0);
        if (stop) break;
        sel = __shfl_sync(0xffffffffu, sel, 0);
        if (sel < 0) continue;
        seg = sel;
        c = cp.chunk_start[seg] + (int64_t)__shfl_sync(0xffffffffu, sel_c, 0);
        __syncwarp();                                  // s_hdr[seg] written by lane 0
      } else {
        if (c >= nchunks) break;
        if (lane == 0) nx = atomicAdd(counter, 1u);    // next claim overlaps this chunk
        while (seg + 1 < segs.nseg && c >= cp.chunk_start[seg + 1]) ++seg;
      }
      const HeaderInfo H = s_hdr[seg];
      if (H.err == kOk) {
        const int64_t n = H.n;
        const int gsl = H.gsl;
        const Layout L = layout_of(n, gsl);
        const uint8_t* frame = segs.stat[seg];
        const uint8_t* dyn = segs.dyn[seg] ? segs.dyn[seg] : frame + L.off[5];
        const uint32_t* gi = reinterpret_cast<const uint32_t*>(frame + L.off[4]);
        const int64_t gpt = int64_t(kTile) >> gsl;
        const bool stage_gi = gsl >= 4;              // slice fits kGiSlots
        const int64_t seg_tiles = segs.tile_start[seg + 1] - segs.tile_start[seg];
        const int64_t zcap = pad128(H.zc);
        const int64_t t0 = (c - cp.chunk_start[seg]) * cp.chunk;
        const int64_t t1 = (t0 + cp.chunk < seg_tiles) ? t0 + cp.chunk : seg_tiles;
        // escape-range bounds of the chunk's tiles: bound(t) = gi[first group of t]
        const int64_t tb = t0 + lane;
        uint32_t bnd = 0;
        if (lane <= t1 - t0) bnd = tb < seg_tiles ? gi[tb * gpt] : (uint32_t)H.zc;
        // lane j prepares tile t0 + j of the chunk (sizes, clamped escape
        // range, group_index slice) in parallel; then the tiles are issued
        // in order, tile j by lane j once its stage is free.  The lane-0
        // serial path per tile is only the wait, the stage metadata and the
        // bulk copies (~277 -> ~100 producer instructions per tile).
        const int64_t t = t0 + lane;
        const bool mine = t < t1;
        const int64_t lo = (int64_t)bnd;
        const int64_t hi = (int64_t)__shfl_down_sync(0xffffffffu, bnd, 1);
        const int64_t e0 = t * kTile;
        const int64_t valid = (n - e0) < kTile ? (n - e0) : kTile;
        const uint32_t b_sm = mine ? r16(valid) : 0u, b_pl = mine ? r16((valid + 7) >> 3) : 0u;
        // escapes: clamp into the section so a corrupt index stays memory-safe
        const int64_t clo = lo < 0 ? 0 : (lo > H.zc ? H.zc : lo);
        const int64_t chi = hi < clo ? clo : (hi > H.zc ? H.zc : hi);
        const uint8_t* esrc = dyn + clo;
        const uint8_t* eal = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(esrc) & ~uintptr_t(15));
        int64_t eb = (int64_t)r16((uint64_t)(chi - clo) + (uint64_t)(esrc - eal));
        if (eb > kEscSlots) eb = kEscSlots;
        if ((eal - dyn) + eb > zcap + 128) eb = 0;   // never read past the padded section
        // group_index slice [g0, g0 + ng] (+1 for the next tile's first entry)
        uint32_t b_gi = 0;
        const uint32_t* gsrc = gi;
        int32_t shift = 0;
        if (stage_gi && mine) {
          const int64_t g0 = t * gpt;
          int64_t ng = (valid + (int64_t(1) << gsl) - 1) >> gsl;
          if (g0 + ng < L.groups) ng += 1;
          const uint32_t* gp = gi + g0;
          gsrc = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(gp) & ~uintptr_t(15));
          shift = (int32_t)(gp - gsrc);
          b_gi = r16((uint64_t)(ng + shift) * 4);
        }
        const int ntl = (int)(t1 - t0);
        for (int jt = 0; jt < ntl; ++jt) {
          if (lane == jt) {
            const int64_t kk = k + jt;
            const int st = (int)(kk % kDStages);
            if (kk >= kDStages) mbar_wait(empty + st, (uint32_t)(((kk / kDStages) - 1) & 1));
            DStage& S = ring[st];
            s_meta[st] = StageMeta{(uint32_t)clo, (uint32_t)(chi - clo),
                                   (int32_t)(clo - (eal - dyn)),
                                   (uint32_t)t | (uint32_t)seg << 24 | (uint32_t)shift << 30};
            mbar_arrive_expect_tx(full + st, b_sm + 3 * b_pl + b_gi + (uint32_t)eb);
            tma_load_1d(S.sm, frame + L.off[0] + e0, b_sm, full + st);
            for (int b = 0; b < 3; ++b)
              tma_load_1d(S.pl[b], frame + L.off[1 + b] + (e0 >> 3), b_pl, full + st);
            if (b_gi) tma_load_1d(S.gi, gsrc, b_gi, full + st);
            if (eb) tma_load_1d(S.esc, eal, (uint32_t)eb, full + st);
          }
          __syncwarp();   // reconverge before the next shuffle (no BRA.DIV slow path)
        }
        k += ntl;
      }
      if (!kPull) c = (int64_t)__shfl_sync(0xffffffffu, nx, 0);
    }
    if (lane == 0) {                  // end markers: one for each consumer group
      for (int e = 0; e < kDGroups; ++e, ++k) {
        const int st = (int)(k % kDStages);
        if (k >= kDStages) mbar_wait(empty + st, (uint32_t)(((k / kDStages) - 1) & 1));
        s_meta[st].tsg = 0xFFFFFFFFu;
        mbar_arrive(full + st);
      }
    }
    return;
  }

  // ========================= consumer warps ==============================
  // kDGroups groups of 4 warps take stages in turn (group g: k = G i + g), so
  // a tile is decoded by 128 threads.  Lean path (gs = 512, full tile): each
  // lane owns 32 consecutive words -- half the per-word fixed cost of 16 --
  // and each half-warp one 512-word group (segmented scan over 16 lanes).
  // Other tiles: two passes of the 16-word logic over virtual threads
  // vct = 128 p + ct (virtual warp vw = 4 p + warp covers 512 words).
  // Mode A (gs <= 512): a virtual warp's 512 words start a group, so its
  // escape base is gi[first group of the warp] — no group-wide scan.  Mode B
  // (1024 <= gs <= 4096): groups span warps; one group-wide scan over the 8
  // virtual warps of the tile (named barrier per consumer group).
  const int ct0 = tid - 32;                          // 0..255
  const int grp = ct0 >> 7;                          // consumer group
  const int ct = ct0 & 127, lane = ct & 31, warp = ct >> 5;
  uint8_t* slot = s_slot + ct0 * 32;                 // 32 B per thread
  // per-segment state: push mode carries it across stages, reloaded when the
  // stage's segment changes; pull mode reloads it from shared memory every
  // stage (no loop-carried copies: the pull variant spilled them at the
  // 72-register cap; 4 peer frames 143.4 -> 139.7 us.  Reloading in push
  // mode too cost it 131.3 -> 137.4 us)
  int cseg = -1;
  uint32_t tbl_lo = 0, tbl_hi = 0;
  int64_t zc = 0, groups = 0;
  const uint32_t* gi = nullptr;
  uint16_t* out_seg = out;
  int64_t n = 0, gpt = 0;
  int gsl = 0;
  bool stage_gi = false, modeA = false, gs512 = false, out_aligned = false, out_a32 = false;
  for (int64_t i = 0;; ++i) {
    const int64_t k = (int64_t)kDGroups * i + grp;
    const int st = (int)(k % kDStages);
    mbar_wait_warp(full + st, (uint32_t)((k / kDStages) & 1));
    const StageMeta M = s_meta[st];
    if (M.tsg == 0xFFFFFFFFu) break;
    const int64_t t = M.tsg & 0xFFFFFFu;
    const int seg = (int)((M.tsg >> 24) & 63u);
    if (kPull) {                                     // uniform loads, every stage
      const HeaderInfo& H = s_hdr[seg];
      const SegCons& C = s_cons[seg];
      n = H.n;
      gsl = H.gsl;
      zc = H.zc;
      tbl_lo = H.tbl_lo;
      tbl_hi = H.tbl_hi;
      groups = C.groups;
      gi = C.gi;
      gpt = int64_t(kTile) >> gsl;
      stage_gi = gsl >= 4;
      modeA = gsl <= 9;
      gs512 = gsl == 9;
      out_seg = C.out;
      out_aligned = (C.flags & 1u) != 0;
      out_a32 = (C.flags & 2u) != 0;
    } else if (seg != cseg) {                        // uniform across the group
      cseg = seg;
      const HeaderInfo& H = s_hdr[seg];
      n = H.n;
      gsl = H.gsl;
      zc = H.zc;
      tbl_lo = H.tbl_lo;
      tbl_hi = H.tbl_hi;
      const Layout L = layout_of(n, gsl);
      groups = L.groups;
      gi = reinterpret_cast<const uint32_t*>(segs.stat[seg] + L.off[4]);
      gpt = int64_t(kTile) >> gsl;
      stage_gi = gsl >= 4;
      modeA = gsl <= 9;
      gs512 = gsl == 9;
      out_seg = out + segs.out_off[seg];
      out_aligned = ((reinterpret_cast<uintptr_t>(out_seg) & 15) == 0) && write_out;
      out_a32 = ((reinterpret_cast<uintptr_t>(out_seg) & 31) == 0) && write_out;
    }
    const DStage& S = ring[st];
    const int64_t tile_base = t * kTile;
    const int64_t lo = M.lo;
    const int32_t tcnt = (int32_t)M.cnt;
    const int32_t esc_off = M.esc_off;
    const int gshift = (int)(M.tsg >> 30);
    const uint8_t* esc_base = S.esc + esc_off;   // this tile's staged escapes
    int32_t my_err = kOk;
    if (gs512 && tile_base + kTile <= n) {
      // ---------------- lean path: gs = 512, full tile, 32 words / lane ------
      const int half = lane >> 4;
      const uint4 sa = *reinterpret_cast<const uint4*>(S.sm + ct * 32);
      const uint4 sb = *reinterpret_cast<const uint4*>(S.sm + ct * 32 + 16);
      const uint32_t p0 = *reinterpret_cast<const uint32_t*>(S.pl[0] + ct * 4);
      const uint32_t p1 = *reinterpret_cast<const uint32_t*>(S.pl[1] + ct * 4);
      const uint32_t p2 = *reinterpret_cast<const uint32_t*>(S.pl[2] + ct * 4);
      const uint32_t esc = ~(p0 | p1 | p2);
      const uint32_t cnt = __popc(esc);
      const uint32_t incl = half_incl_scan(cnt);
      const uint32_t htot = __shfl_sync(0xffffffffu, incl, lane | 15);
      const int gl = 2 * warp + half;                // group within the tile
      const uint32_t gwv = S.gi[gshift + gl];
      const int32_t rank0 = (int32_t)(gwv - (uint32_t)lo + incl - cnt);
      if ((lane & 15) == 0) {
        const int64_t g = t * 8 + gl;
        const bool has_next = g + 1 < groups;
        const uint32_t next = has_next ? S.gi[gshift + gl + 1] : (uint32_t)zc;
        if (g == 0 && gwv != 0) my_err = kErrGroupIndex;
        if (gwv + htot != next) my_err = has_next ? kErrGroupIndex : kErrZeroCount;
      }
      uint32_t E[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {                  // plane byte q: words 8q .. 8q+7
        const uint32_t sp = s_spread[(p0 >> (8 * q)) & 0xFF] |
                            s_spread[(p1 >> (8 * q)) & 0xFF] << 1 |
                            s_spread[(p2 >> (8 * q)) & 0xFF] << 2;
        E[2 * q] = prmt(tbl_lo, tbl_hi, sp);
        E[2 * q + 1] = prmt(tbl_lo, tbl_hi, sp >> 16);
      }
      // escape-heavy warps (>= 1/4 of their words) expand all lanes' escapes
      // with PRMT; sparse ones keep the per-escape slot loop
      const bool dense = __shfl_sync(0xffffffffu, incl, 15) + __shfl_sync(0xffffffffu, incl, 31) >=
                         256u;
      if (esc) {
        if (rank0 < 0 || rank0 + (int32_t)cnt > tcnt) {
          my_err = kErrZeroCount;     // accompanied by a failing index check
        } else if (dense) {
          expand_escapes(esc_base + rank0, esc, E, s_xsel);
        } else {
          *reinterpret_cast<uint4*>(slot) = make_uint4(0, 0, 0, 0);
          *reinterpret_cast<uint4*>(slot + 16) = make_uint4(0, 0, 0, 0);
          const uint8_t* eb = esc_base + rank0;
          uint32_t m = esc;
          while (m) {
            const int j = __ffs(m) - 1;
            m &= m - 1;
            slot[j] = *eb++;
          }
          const uint4 d0 = *reinterpret_cast<const uint4*>(slot);
          const uint4 d1 = *reinterpret_cast<const uint4*>(slot + 16);
          E[0] |= d0.x; E[1] |= d0.y; E[2] |= d0.z; E[3] |= d0.w;
          E[4] |= d1.x; E[5] |= d1.y; E[6] |= d1.z; E[7] |= d1.w;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + st);
      uint32_t o[16];
      reassemble4(sa.x, E[0], o[0], o[1]);
      reassemble4(sa.y, E[1], o[2], o[3]);
      reassemble4(sa.z, E[2], o[4], o[5]);
      reassemble4(sa.w, E[3], o[6], o[7]);
      reassemble4(sb.x, E[4], o[8], o[9]);
      reassemble4(sb.y, E[5], o[10], o[11]);
      reassemble4(sb.z, E[6], o[12], o[13]);
      reassemble4(sb.w, E[7], o[14], o[15]);
      uint16_t* dst = out_seg + (tile_base + ct * 32);
      if (out_a32) {
        st_v8(dst, make_uint4(o[0], o[1], o[2], o[3]), make_uint4(o[4], o[5], o[6], o[7]));
        st_v8(dst + 16, make_uint4(o[8], o[9], o[10], o[11]),
              make_uint4(o[12], o[13], o[14], o[15]));
      } else if (out_aligned) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          st_stream_v4(dst + 8 * q, make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]));
      } else if (write_out) {
#pragma unroll
        for (int j = 0; j < 32; ++j) dst[j] = (uint16_t)(o[j >> 1] >> (16 * (j & 1)));
      }
      if (my_err != kOk) atomicMin(err + seg, my_err);
      continue;
    }
    // ---------------- general path: two passes of 16 words / thread --------
    const int64_t rem = n - tile_base;                       // >= 1
    const int rem32 = rem >= kTile ? kTile : (int)rem;
    const int live_warps = (rem32 + 511) >> 9;
    const int64_t g0 = t * gpt;
    auto gi_at = [&](int64_t g) -> int64_t {   // g within this tile, or its first successor
      if (g >= groups) return zc;
      if (stage_gi) return (int64_t)S.gi[gshift + (int)(g - g0)];
      return (int64_t)gi[g];
    };
    uint4 sv[2];
    uint32_t escv[2], cntv[2], inclv[2], spv[2][2];
    int nvv[2];
    int32_t rank0v[2];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const int vct = 128 * p + ct;
      const int nv = rem32 - vct * kEPT >= kEPT ? kEPT : rem32 - vct * kEPT;   // may be <= 0
      const uint32_t valid16 = nv >= kEPT ? 0xFFFFu : (nv > 0 ? ((1u << nv) - 1u) : 0u);
      uint32_t p0 = 0, p1 = 0, p2 = 0;
      sv[p] = make_uint4(0, 0, 0, 0);
      if (nv > 0) {
        sv[p] = *reinterpret_cast<const uint4*>(S.sm + vct * kEPT);
        p0 = *reinterpret_cast<const uint16_t*>(S.pl[0] + vct * 2);
        p1 = *reinterpret_cast<const uint16_t*>(S.pl[1] + vct * 2);
        p2 = *reinterpret_cast<const uint16_t*>(S.pl[2] + vct * 2);
      }
      nvv[p] = nv;
      escv[p] = ~(p0 | p1 | p2) & valid16;
      cntv[p] = __popc(escv[p]);
      inclv[p] = warp_incl_scan(cntv[p]);
      spv[p][0] = s_spread[p0 & 0xFF] | s_spread[p1 & 0xFF] << 1 | s_spread[p2 & 0xFF] << 2;
      spv[p][1] = s_spread[(p0 >> 8) & 0xFF] | s_spread[(p1 >> 8) & 0xFF] << 1 |
                  s_spread[(p2 >> 8) & 0xFF] << 2;
    }
    if (modeA) {
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int vw = 4 * p + warp, vct = 128 * p + ct;
        const int64_t base = tile_base + (int64_t)vct * kEPT;
        const int nv = nvv[p];
        const uint32_t esc = escv[p], incl = inclv[p], wexcl = incl - cntv[p];
        if (gs512) {
          // one group per virtual warp, 32-bit math, staged slice
          const uint32_t wtot = __shfl_sync(0xffffffffu, incl, 31);
          const bool warp_live = vw < live_warps;
          const uint32_t gwv = warp_live ? S.gi[gshift + vw] : 0u;
          rank0v[p] = (int32_t)(gwv - (uint32_t)lo + wexcl);
          if (lane == 0 && warp_live) {
            const int64_t g = g0 + vw;
            const uint32_t next = (g + 1 < groups) ? S.gi[gshift + vw + 1] : (uint32_t)zc;
            if (g == 0 && gwv != 0) my_err = kErrGroupIndex;
            if (gwv + wtot != next) my_err = (g + 1 < groups) ? kErrGroupIndex : kErrZeroCount;
          }
        } else {
          const int64_t gw = (tile_base + vw * 512) >> gsl;     // warp's first group
          const bool warp_live = tile_base + vw * 512 < n;
          const int32_t wbase = warp_live ? (int32_t)(gi_at(gw) - lo) : 0;
          const int32_t rank0 = wbase + (int32_t)wexcl;
          rank0v[p] = rank0;
          const int tpg = gsl >= 4 ? 1 << (gsl - 4) : 1;          // threads per group
          const uint32_t gend = __shfl_sync(0xffffffffu, incl, (lane | (tpg - 1)) & 31);
          if (nv > 0) {
            if (gsl >= 4) {
              if ((lane & (tpg - 1)) == 0) {
                const int64_t g = base >> gsl;
                const int64_t c = (int64_t)(gend - wexcl);
                const int64_t gv = lo + rank0;           // == gi[g] when consistent
                if (g == 0 && gi_at(0) != 0) my_err = kErrGroupIndex;
                if (gi_at(g) != gv || gv + c != gi_at(g + 1))
                  my_err = (g + 1 < groups) ? kErrGroupIndex : kErrZeroCount;
              }
            } else {
              const int gs = 1 << gsl;
              int32_t r = rank0;
              for (int j = 0; j < kEPT && j < nv; j += gs) {
                const int64_t g = (base + j) >> gsl;
                const int64_t c = __popc(esc & (((1u << gs) - 1u) << j));
                if (g == 0 && gi_at(0) != 0) my_err = kErrGroupIndex;
                if (gi_at(g) != lo + r || lo + r + c != gi_at(g + 1))
                  my_err = (g + 1 < groups) ? kErrGroupIndex : kErrZeroCount;
                r += (int32_t)c;
              }
            }
          }
        }
      }
    } else {
      // mode B: group-wide scan of the 8 virtual warps' escape counts
      uint32_t* sw = s_wsum[grp][i & 1];
      if (lane == 31) {
        sw[warp] = inclv[0];
        sw[4 + warp] = inclv[1];
      }
      asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(128) : "memory");
      const uint32_t v = lane < 8 ? sw[lane] : 0u;
      const uint32_t vi = warp_incl_scan<8>(v);
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int vw = 4 * p + warp, vct = 128 * p + ct;
        const int64_t base = tile_base + (int64_t)vct * kEPT;
        const uint32_t wb = __shfl_sync(0xffffffffu, vi - v, vw);
        rank0v[p] = (int32_t)(wb + inclv[p] - cntv[p]);
        if (nvv[p] > 0 && (base & ((int64_t(1) << gsl) - 1)) == 0) {
          const int64_t g = base >> gsl;
          if (g == 0 && gi_at(0) != 0) my_err = kErrGroupIndex;
          if (gi_at(g) != lo + rank0v[p]) my_err = kErrGroupIndex;
        }
      }
      const uint32_t agg = __shfl_sync(0xffffffffu, vi, 7);
      if (ct == 0) {
        if ((int32_t)agg != tcnt) my_err = (g0 + gpt < groups) ? kErrGroupIndex : kErrZeroCount;
      }
    }
    // ---- exponents + escapes (staged bytes at their tile-local rank) --------
    uint32_t E[2][4];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      E[p][0] = prmt(tbl_lo, tbl_hi, spv[p][0]);
      E[p][1] = prmt(tbl_lo, tbl_hi, spv[p][0] >> 16);
      E[p][2] = prmt(tbl_lo, tbl_hi, spv[p][1]);
      E[p][3] = prmt(tbl_lo, tbl_hi, spv[p][1] >> 16);
      const uint32_t esc = escv[p];
      if (esc) {
        const int32_t rank0 = rank0v[p];
        if (rank0 < 0 || rank0 + (int32_t)cntv[p] > tcnt) {
          // escapes out of the staged range: always accompanied by a failing
          // index check, which carries the field the reference names
          my_err = kErrZeroCount;
        } else {
          uint8_t* sl = slot + 16 * p;
          *reinterpret_cast<uint4*>(sl) = make_uint4(0, 0, 0, 0);
          const uint8_t* eb = esc_base + rank0;
          uint32_t m = esc;
          while (m) {
            const int j = __ffs(m) - 1;
            m &= m - 1;
            sl[j] = *eb++;
          }
          const uint4 d = *reinterpret_cast<const uint4*>(sl);
          E[p][0] |= d.x; E[p][1] |= d.y; E[p][2] |= d.z; E[p][3] |= d.w;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + st);

    // ---- reassemble (codec.py:308-312) and store ---------------------------
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const int nv = nvv[p];
      if (write_out && nv > 0) {
        const int64_t base = tile_base + (int64_t)(128 * p + ct) * kEPT;
        uint32_t o0, o1, o2, o3, o4, o5, o6, o7;
        reassemble4(sv[p].x, E[p][0], o0, o1);
        reassemble4(sv[p].y, E[p][1], o2, o3);
        reassemble4(sv[p].z, E[p][2], o4, o5);
        reassemble4(sv[p].w, E[p][3], o6, o7);
        uint16_t* dst = out_seg + base;
        if (nv == kEPT && ((reinterpret_cast<uintptr_t>(dst) & 31) == 0)) {
          st_v8(dst, make_uint4(o0, o1, o2, o3), make_uint4(o4, o5, o6, o7));
        } else if (nv == kEPT && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
          st_stream_v4(dst, make_uint4(o0, o1, o2, o3));
          st_stream_v4(dst + 8, make_uint4(o4, o5, o6, o7));
        } else {
          const uint32_t ow[8] = {o0, o1, o2, o3, o4, o5, o6, o7};
#pragma unroll
          for (int j = 0; j < kEPT; ++j)
            if (j < nv) dst[j] = (uint16_t)(ow[j >> 1] >> (16 * (j & 1)));
        }
      }
    }
    if (my_err != kOk) atomicMin(err + seg, my_err);
  }
  ZC_TL(1, 32);
}

static int grid_cap(const void* fn, int threads, size_t dyn) {
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, dyn);
  return sms * (occ > 0 ? occ : 1);
}

// Error words (0x7F7F7F7F = ok) and the chunk counter in one launch instead of
// two memset nodes ahead of the ring decoder.
__global__ void decode_init_kernel(int32_t* __restrict__ err, int nseg, unsigned* __restrict__ counter) {
  const int t = threadIdx.x;
  if (t < nseg) err[t] = 0x7F7F7F7F;                // "no error" (atomicMin target)
  if (t <= nseg) counter[t] = 0u;                   // global claim + per-segment (pull) counters
}

cudaError_t launch_decode_small(const DecodeSegs&, uint16_t*, int32_t*, int, cudaStream_t);

// Frames of at most this many elements (every segment), known to use
// 512-element groups (flags bit 3), take the one-launch cluster decoder.
// Its 8 CTAs x 8 warps walk the groups with dependent global loads, so it
// stays latency-bound beyond ~2 groups per warp (64 Ki words); the ring
// decoder takes over there (bench.py --workload sweep).
static int64_t small_decode_max() {
  static const int64_t v = [] {
    const char* e = getenv("ZC_SMALL_DEC_MAX_WORDS");
    return e ? (int64_t)atoll(e) : (int64_t)65536;
  }();
  return v;
}

cudaError_t launch_decode(const DecodeSegs& segs, uint16_t* out, int32_t* err, void* ws,
                          int flags, cudaStream_t st) {
  if ((flags & 8) && !(flags & 2) && segs.nseg >= 1) {
    bool small = true;
    for (int s = 0; s < segs.nseg; ++s) small = small && segs.n[s] <= small_decode_max();
    if (small) return launch_decode_small(segs, out, err, flags, st);
  }
  // flags bit 0: write the words; bit 1: frames may use groups larger than a
  // tile (then the look-back decoder is used)
  const int write_out = flags & 1;
  const int any_large_groups = (flags >> 1) & 1;
  const int64_t ntiles = segs.tile_start[segs.nseg];
  cudaError_t e = cudaSuccess;
  if (ntiles == 0 || any_large_groups) {
    e = cudaMemsetAsync(err, 0x7F, sizeof(int32_t) * segs.nseg, st);
    if (e != cudaSuccess) return e;
  }
  if (ntiles == 0) return cudaSuccess;
  if (any_large_groups) {
    unsigned* counter = reinterpret_cast<unsigned*>(ws);
    uint64_t* status = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(ws) + 128);
    e = cudaMemsetAsync(ws, 0, 128 + 8 * ntiles, st);
    if (e != cudaSuccess) return e;
    static int caps[kMaxDevices];
    const int cap = per_device(caps, [] { return grid_cap((const void*)decode_lookback_kernel, kThreads, 0); });
    const unsigned grid = (unsigned)(ntiles < cap ? ntiles : cap);
    prof_mark(kProfDecode, false, st);
    decode_lookback_kernel<<<grid, kThreads, 0, st>>>(segs, out, err, status, counter, write_out);
    prof_mark(kProfDecode, true, st);
    return cudaGetLastError();
  }
  const size_t dyn = kDStages * kDStageBytes + 2 * kDStages * sizeof(uint64_t);
  const bool pull = (flags >> 2) & 1;
  static int caps2[kMaxDevices];
  const int cap2 = per_device(caps2, [dyn] {
    cudaFuncSetAttribute(decode_ring_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    cudaFuncSetAttribute(decode_ring_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    int c = grid_cap((const void*)decode_ring_kernel<false>, kDThreads, dyn);
    const int cp2 = grid_cap((const void*)decode_ring_kernel<true>, kDThreads, dyn);
    if (cp2 < c) c = cp2;
    if (const char* e = getenv("ZC_DECODE_CTAS_PER_SM")) {
      int dev = 0, sms = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const int want = sms * atoi(e);
      if (want > 0 && want < c) c = want;
    }
    return c;
  });
  DChunkPlan cp{};
  // inputs of at most one tile per CTA are spread one tile per CTA (a 1 MiB
  // message: 128 CTAs instead of 32; 26.8 against 30.3 us per codec step)
  const int64_t all_tiles = segs.tile_start[segs.nseg];
  cp.chunk = all_tiles <= cap2 ? 1 : kDChunk;
  for (int s = 0; s < segs.nseg; ++s) {
    const int64_t tiles = segs.tile_start[s + 1] - segs.tile_start[s];
    cp.chunk_start[s + 1] = cp.chunk_start[s] + (tiles + cp.chunk - 1) / cp.chunk;
  }
  const int64_t nchunks = cp.chunk_start[segs.nseg];
  const unsigned grid = (unsigned)(nchunks < cap2 ? nchunks : cap2);
  unsigned* counter = reinterpret_cast<unsigned*>(ws);
  decode_init_kernel<<<1, kMaxSegments + 32, 0, st>>>(err, segs.nseg, counter);
  prof_mark(kProfDecode, false, st);
  if (pull)
    decode_ring_kernel<true><<<grid, kDThreads, dyn, st>>>(segs, cp, out, err, counter, write_out);
  else
    decode_ring_kernel<false><<<grid, kDThreads, dyn, st>>>(segs, cp, out, err, counter, write_out);
  prof_mark(kProfDecode, true, st);
  return cudaGetLastError();
}




// ============================================================================
// Group random access (reference codec.decompress_group, codec.py:330-348):
// decode groups [g0, g1) of a frame whose structure was validated, reading
// only those groups' sign-mantissa / plane bytes and their escapes, which
// start at group_index[g] -- no earlier escape data is touched.  One CTA per
// group (grid-strided); a group is walked in 4096-element tiles with a block
// scan carrying the escape rank.  Escape positions are clamped into the
// section, so even an unvalidated frame stays memory-safe.
// ============================================================================
__global__ void __launch_bounds__(kThreads)
decode_groups_kernel(const uint8_t* __restrict__ frame, int64_t n, int gsl, int64_t g0,
                     int64_t g1, uint16_t* __restrict__ out) {
  __shared__ uint32_t s_warp[kWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Layout L = layout_of(n, gsl);
  const uint64_t zc = reinterpret_cast<const uint64_t*>(frame)[2];
  const uint8_t* e8 = reinterpret_cast<const uint8_t*>(frame) + 24;   // entries[0..6]
  const uint8_t* sm = frame + L.off[0];
  const uint8_t* pl0 = frame + L.off[1];
  const uint8_t* pl1 = frame + L.off[2];
  const uint8_t* pl2 = frame + L.off[3];
  const uint32_t* gi = reinterpret_cast<const uint32_t*>(frame + L.off[4]);
  const uint8_t* dyn = frame + L.off[5];
  const int64_t gs = int64_t(1) << gsl;
  for (int64_t g = g0 + blockIdx.x; g < g1; g += gridDim.x) {
    const int64_t s = g * gs;
    const int64_t e = (s + gs < n) ? s + gs : n;
    uint64_t run = gi[g];
    for (int64_t tb = s; tb < e; tb += kTile) {
      const int64_t base = tb + (int64_t)tid * kEPT;
      uint32_t esc = 0, code[kEPT];
#pragma unroll
      for (int j = 0; j < kEPT; ++j) {
        const int64_t k = base + j;
        uint32_t c = 0;
        if (k < e) {
          const int sh = (int)(k & 7);
          c = ((pl0[k >> 3] >> sh) & 1u) | ((pl1[k >> 3] >> sh) & 1u) << 1 |
              ((pl2[k >> 3] >> sh) & 1u) << 2;
          if (c == 0) esc |= 1u << j;
        }
        code[j] = c;
      }
      const uint32_t cnt = __popc(esc);
      const uint32_t incl = warp_incl_scan(cnt);
      if (lane == 31) s_warp[warp] = incl;
      __syncthreads();
      uint32_t wbase = 0, tot = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        wbase += (w < warp) ? s_warp[w] : 0u;
        tot += s_warp[w];
      }
      uint64_t pos = run + wbase + incl - cnt;
#pragma unroll
      for (int j = 0; j < kEPT; ++j) {
        const int64_t k = base + j;
        if (k < e) {
          uint32_t ex;
          if (code[j]) {
            ex = e8[code[j] - 1];
          } else {
            ex = pos < zc ? dyn[pos] : 0u;
            ++pos;
          }
          const uint32_t b = sm[k];
          out[k - g0 * gs] = (uint16_t)(((b & 0x80u) << 8) | (ex << 7) | (b & 0x7Fu));
        }
      }
      run += tot;
      __syncthreads();   // s_warp reuse
    }
  }
}

cudaError_t launch_decode_groups(const uint8_t* frame, int64_t n, int gsl, int64_t g0, int64_t g1,
                                 uint16_t* out, cudaStream_t st) {
  if (g1 <= g0) return cudaSuccess;
  const int64_t ng = g1 - g0;
  const unsigned grid = (unsigned)(ng < 4096 ? ng : 4096);
  decode_groups_kernel<<<grid, kThreads, 0, st>>>(frame, n, gsl, g0, g1, out);
  return cudaGetLastError();
}


// Loads every kernel of this file now (cudaFuncGetAttributes forces a
// lazily loaded module function in): with CUDA_MODULE_LOADING=LAZY, the
// first launch of a kernel waits for the device, which deadlocks while a
// peer rank sharing the GPU spins on a flag this rank has yet to publish.
cudaError_t preload_decode() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, (const void*)decode_groups_kernel);
  cudaFuncGetAttributes(&a, (const void*)decode_init_kernel);
  cudaFuncGetAttributes(&a, (const void*)decode_lookback_kernel);
  cudaFuncGetAttributes(&a, (const void*)decode_ring_kernel<false>);
  cudaFuncGetAttributes(&a, (const void*)decode_ring_kernel<true>);
  return cudaGetLastError();
}

}  // namespace zc

ZC_TL_EXPORT(zc_debug_timeline_dec)
