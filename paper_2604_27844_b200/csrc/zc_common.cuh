// Shared definitions for the ZipCCL B200 kernels (sm_100a).
//
// Frame layout (reference container.py:3-22, :45-95; codec.py:357-401):
//   [0,128)            header "<4sBBBBQQ7sB6I" (56 B) + zero pad
//   [off0, +n)         sign-mantissa bytes           ((w>>8)&0x80)|(w&0x7F)
//   [off1..off3)       three LSB-first code planes   ceil(n/8) B each
//   [off4, +4*groups)  u32 exclusive escape prefix per group (group_index)
//   [off5, +zc)        escaped raw exponent bytes, element order
// every section 128-aligned and zero padded; static part = [0, off5).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define ZC_HD __host__ __device__ __forceinline__

namespace zc {

constexpr int kAlign = 128;
constexpr int kHeaderBytes = 56;
constexpr int kMaxSegments = 64;

// Tile geometry shared by encode / decode / stats.
constexpr int kThreads = 256;               // 8 warps
constexpr int kEPT = 16;                    // elements per thread (two 16-B loads)
constexpr int kTile = kThreads * kEPT;      // 4096 elements per tile
constexpr int kWarps = kThreads / 32;

// Per-device cache of a host-side launch setting (occupancy caps; the
// MaxDynamicSharedMemorySize attribute is also set per device inside `init`).
// Thread ranks may drive several GPUs from one process.
constexpr int kMaxDevices = 64;
template <class F>
inline int per_device(int (&slot)[kMaxDevices], F init) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) return init();
  int v = __atomic_load_n(&slot[dev], __ATOMIC_ACQUIRE);
  if (v == 0) {
    v = init();
    __atomic_store_n(&slot[dev], v, __ATOMIC_RELEASE);
  }
  return v;
}

ZC_HD int64_t pad128(int64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct Layout {
  int64_t n;
  int gs_log2;
  int64_t off[6];   // sm, p0, p1, p2, gi, zero_exponents
  int64_t plane_bytes, groups;
};

// reference container.section_offsets (container.py:52-62)
ZC_HD Layout layout_of(int64_t n, int gs_log2) {
  Layout L;
  L.n = n;
  L.gs_log2 = gs_log2;
  L.plane_bytes = (n + 7) >> 3;
  L.groups = (n + (int64_t(1) << gs_log2) - 1) >> gs_log2;
  int64_t pos = pad128(kHeaderBytes);
  const int64_t sizes[5] = {n, L.plane_bytes, L.plane_bytes, L.plane_bytes, 4 * L.groups};
  for (int i = 0; i < 5; ++i) { L.off[i] = pos; pos += pad128(sizes[i]); }
  L.off[5] = pos;
  return L;
}

// Error codes, ordered like the reference's check order (container.parse_header
// :113-135, parse :138-180, CompressedChunk.check_structure/_check_consistency
// codec.py:210-250) so that atomicMin reports the field the reference names.
enum Err : int32_t {
  kOk = 0,
  kErrHeaderShort = 1,
  kErrMagic = 2,
  kErrVersion = 3,
  kErrFlags = 4,
  kErrGsLog2 = 5,
  kErrElementCount = 6,
  kErrZeroCountHeader = 7,
  kErrCodebookDistinct = 8,
  kErrCodebookBase = 9,
  kErrOffset0 = 10,   // .. kErrOffset0 + 5
  kErrFrameLength = 16,
  kErrGroupIndex = 17,
  kErrZeroCount = 18,
  kErrCountMismatch = 19,   // collectives: header element_count != expected
  kErrTimeout = 20,         // p2p: peer never signalled
  kErrGroupTooLarge = 21,   // ring decoder: gs > one tile (decode with large_groups)
  kErrGroupSize = 22,       // collectives' fused reduce: frames use 512-element groups
};

// ---- memory-ordering helpers (decoupled look-back, peer flags) -------------
// The look-back status word carries its payload in the same 64-bit word as
// its flag, so it needs coherence, not ordering: relaxed gpu-scope accesses
// (no L1 invalidation / fence per poll, unlike ld.acquire / st.release).
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Programmatic dependent launch (launch attribute ProgrammaticStreamSerialization):
// a dependent grid may be scheduled once every CTA of this grid has issued
// launch_dependents (or exited); grid_dep_wait blocks until the prerequisite
// grid has completed and its writes are visible.  Both are no-ops in a grid
// launched without the attribute.
__device__ __forceinline__ void grid_dep_launch() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void grid_dep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Read-once global loads (non-coherent path, no L1 allocation).  Not
// volatile: the compiler may batch and reorder them.
__device__ __forceinline__ uint4 ld_stream_v4(const void* p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
// Output stores are plain 16-B stores: an asm store with a memory clobber
// pinned every later shared-memory load behind it and cost the decoder 14%
// (measured: 4.66 -> 5.40 TB/s on the store-only ring).
__device__ __forceinline__ void st_stream_v4(void* p, uint4 v) {
  *reinterpret_cast<uint4*>(p) = v;
}
// 32-B vector accesses (sm_100 LDG/STG.256).  When each lane owns 32
// contiguous bytes, one 256-bit store per lane instead of two 128-bit ones
// writes whole lines per instruction: 4.82 -> 5.88 TB/s on the store-ring
// micro-benchmark (scripts/exp/store_ring.cu; the decoder itself gains ~1%,
// its consumers' latency dominates).  p must be 32-B aligned.  Not volatile,
// no memory clobber (see st_stream_v4).
__device__ __forceinline__ void st_v8(void* p, uint4 a, uint4 b) {
  asm("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a.x), "r"(a.y),
      "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w));
}
__device__ __forceinline__ void ld_stream_v8(const void* p, uint4& a, uint4& b) {
  asm("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
      : "l"(p));
}

// Inclusive scan over the first `Lanes` lanes of a warp (all 32 lanes must
// call it).  shfl.up's lane-valid predicate guards the add: one SHFL + one
// predicated IADD per step, no lane compare / select.
template <int Lanes = 32>
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
#pragma unroll
  for (int o = 1; o < Lanes; o <<= 1)
    asm volatile("{ .reg .u32 t; .reg .pred p;\n\t"
                 "shfl.sync.up.b32 t|p, %0, %1, 0, -1;\n\t"
                 "@p add.u32 %0, %0, t; }"
                 : "+r"(v) : "r"(o));
  return v;
}

// Inclusive scan within each 16-lane half of a warp (segment mask 0x1000).
__device__ __forceinline__ uint32_t half_incl_scan(uint32_t v) {
#pragma unroll
  for (int o = 1; o < 16; o <<= 1)
    asm volatile("{ .reg .u32 t; .reg .pred p;\n\t"
                 "shfl.sync.up.b32 t|p, %0, %1, 0x1000, -1;\n\t"
                 "@p add.u32 %0, %0, t; }"
                 : "+r"(v) : "r"(o));
  return v;
}

// (a & m) | (b & ~m) as one LOP3
__device__ __forceinline__ uint32_t bitsel(uint32_t m, uint32_t a, uint32_t b) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xCA;" : "=r"(d) : "r"(m), "r"(a), "r"(b));
  return d;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

// ---- TMA bulk copies + mbarriers (sm_90+ async proxy, used as the B200 ring) --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n ZC_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra ZC_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// Warp-converged wait: lanes can leave the try_wait loop on different
// iterations; without reconverging, every following warp shuffle takes the
// BRA.DIV / WARPSYNC.COLLECTIVE slow path (measured: 17% of decode issue).
__device__ __forceinline__ void mbar_wait_warp(uint64_t* bar, uint32_t parity) {
  mbar_wait(bar, parity);
  __syncwarp();
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`.
// dst, src 16-B aligned; bytes a multiple of 16.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// Tile-status word for the decoupled look-back: flag in the top two bits,
// inclusive/aggregate escape count in the low 62.
constexpr uint64_t kFlagAgg = uint64_t(1) << 62;
constexpr uint64_t kFlagInc = uint64_t(2) << 62;
constexpr uint64_t kValMask = (uint64_t(1) << 62) - 1;

// Warp 0 of a tile computes the exclusive prefix of `agg` over the tiles
// [chain_first, tile) of its chain, publishing aggregate then inclusive.
// `seed` is the prefix at the chain start (0 for encode, group_index for
// decode chains).  Each lane inspects kLookbackPerLane predecessors, so one
// L2 round trip covers a 256-tile window: the inclusive-prefix frontier then
// advances 256 tiles per round trip instead of 32, which is what lets the
// single-pass encoder keep up with HBM on B200 (a 32-wide window caps it at
// ~0.45 G elements/ms).  Caller guarantees lower tile ids were claimed
// earlier (atomic tile counter), so waiting cannot deadlock.
constexpr int kLookbackPerLane = 8;

template <int V = kLookbackPerLane>
__device__ __forceinline__ uint64_t lookback_warp(uint64_t* status, int64_t tile,
                                                  int64_t chain_first, uint64_t agg,
                                                  uint64_t seed) {
  const int lane = threadIdx.x & 31;
  if (tile == chain_first) {
    if (lane == 0) st_relaxed_u64(status + tile, kFlagInc | ((seed + agg) & kValMask));
    return seed;
  }
  if (lane == 0) st_relaxed_u64(status + tile, kFlagAgg | (agg & kValMask));
  uint64_t excl = 0;
  int64_t p = tile - 1;   // newest predecessor not yet accounted for
  while (true) {
    // lane l covers predecessors p - l*V - v, v = 0..V-1 (newest first)
    uint64_t s[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int64_t q = p - (int64_t)lane * V - v;
      s[v] = (q >= chain_first) ? ld_relaxed_u64(status + q) : kFlagInc;
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int64_t q = p - (int64_t)lane * V - v;
      while ((s[v] >> 62) == 0) s[v] = ld_relaxed_u64(status + q);
    }
    // per lane: sum up to and including its newest inclusive entry
    uint64_t part = 0;
    bool hit = false;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      if (!hit) {
        part += s[v] & kValMask;   // out-of-chain slots carry value 0
        hit = (s[v] & kFlagInc) != 0;
      }
    }
    const unsigned inc_mask = __ballot_sync(0xffffffffu, hit);
    const int first = inc_mask ? __ffs(inc_mask) - 1 : 32;
    uint64_t v = (lane <= first) ? part : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (inc_mask) break;
    p -= 32 * V;
  }
  if (lane == 0) st_relaxed_u64(status + tile, kFlagInc | ((excl + agg) & kValMask));
  return excl;
}

// Segment tables passed by value (A2A per-peer batching).
struct EncodeSegs {
  int nseg;
  int gs_log2;
  int64_t tile_start[kMaxSegments + 1];   // prefix of per-segment tile counts
  int64_t x_off[kMaxSegments];            // element offset into x
  int64_t n[kMaxSegments];                // elements (>= 1)
  int64_t frame_off[kMaxSegments];        // byte offset of frame in frames
};

struct StatSegs {
  int nseg;
  int64_t tile_start[kMaxSegments + 1];
  int64_t x_off[kMaxSegments];
  int64_t n[kMaxSegments];
};

struct DecodeSegs {
  int nseg;
  int64_t tile_start[kMaxSegments + 1];
  const uint8_t* stat[kMaxSegments];      // frame start (header)
  const uint8_t* dyn[kMaxSegments];       // zero-exponent section start (null: in place)
  int64_t dyn_len[kMaxSegments];          // bytes available in dyn (-1 unknown)
  int64_t n[kMaxSegments];                // expected element count
  int64_t out_off[kMaxSegments];          // element offset into out
  // pull mode (peer frames decoded behind arrival, decode_ring_kernel<true>):
  // segment s may be staged once *ready[s] >= epoch (null: ready now)
  const uint64_t* ready[kMaxSegments];
  uint64_t epoch;
  int64_t timeout_ns;                     // 0: wait forever
};

struct HeaderInfo {
  int64_t n, zc;
  int gsl;
  uint32_t tbl_lo, tbl_hi;   // PRMT decode table: byte c = entries[c-1], byte 0 = 0
  int32_t err;
};

// Mirrors container.parse_header + parse offset/length checks, in order.
__device__ __forceinline__ HeaderInfo check_header(const uint8_t* h, int64_t expect_n, int64_t dyn_len) {
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

// One contribution to the fused reduce-scatter (zc_reduce.cu): a frame
// (local, a split design-2 receive buffer, or a peer's HBM) or raw words.
struct RedSrc {
  const uint8_t* stat;     // frame start, or the raw words when raw != 0
  const uint8_t* dyn;      // zero-exponent section (null: in place)
  int64_t dyn_len;         // bytes in dyn (-1 unknown)
  const uint64_t* ready;   // pull: wait until *ready >= epoch (null: ready)
  int32_t raw;
  int32_t pad;
};

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Kernel timing hooks (zc_profile_enable / zc_profile_read in the C-ABI):
// when enabled, CUDA events are recorded on the launching stream right
// before and after the pass-1 encoder and the decoder launches.  No-ops
// otherwise (and never enable them while a stream is being captured).
enum ProfTag { kProfEncode = 0, kProfDecode = 1, kProfTags = 2 };

// Per-CTA %globaltimer stamps for load-balance experiments; compiled only
// into the -DZC_TIMELINE debug library (scripts/exp/timeline.py).  One copy
// per translation unit (no -rdc), read by zc_debug_timeline_{enc,dec}.
#ifdef ZC_TIMELINE
constexpr int kTlSlots = 10, kTlCtas = 8192;
static __device__ unsigned long long zc_tl[kTlSlots][kTlCtas];
#define ZC_TL_EXPORT(name)                                                   \
  extern "C" int name(unsigned long long* host) {                            \
    return (int)cudaMemcpyFromSymbol(host, zc::zc_tl, sizeof(zc::zc_tl));     \
  }
#define ZC_TL(slot, thread)                                                  \
  do {                                                                       \
    if (threadIdx.x == (thread) && blockIdx.x < kTlCtas) {                   \
      unsigned long long t_;                                                 \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                 \
      zc_tl[slot][blockIdx.x] = t_;                                          \
    }                                                                        \
  } while (0)
#define ZC_TL_SMID(slot)                                                     \
  do {                                                                       \
    if (threadIdx.x == 0 && blockIdx.x < kTlCtas) {                          \
      unsigned s_;                                                           \
      asm volatile("mov.u32 %0, %%smid;" : "=r"(s_));                         \
      zc_tl[slot][blockIdx.x] = s_;                                          \
    }                                                                        \
  } while (0)
#else
#define ZC_TL(slot, thread) do {} while (0)
#define ZC_TL_SMID(slot) do {} while (0)
#define ZC_TL_EXPORT(name)
#endif
void prof_mark(int tag, bool end, cudaStream_t st);

__device__ __forceinline__ int find_seg(const int64_t* tile_start, int nseg, int64_t tile) {
  int s = 0;
  while (s + 1 < nseg && tile >= tile_start[s + 1]) ++s;
  return s;
}

}  // namespace zc
