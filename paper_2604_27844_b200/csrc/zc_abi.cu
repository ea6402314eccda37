// C-ABI entry points of libzipccl_b200.so (declared in include/zipccl_b200.h).
// Plain pointers and sizes only; all device work is enqueued on the caller's
// stream and nothing here synchronises.
#include <cstring>
#include <mutex>
#include <vector>
#include <nvtx3/nvToolsExt.h>

#include "zc_common.cuh"
#include "zc_stats.cuh"

namespace zc {
cudaError_t launch_codebook_measured(const uint16_t*, const StatSegs&, int64_t, void*, uint8_t*,
                                     double*, int, cudaStream_t, bool zeroed = false);
cudaError_t launch_codebook_modal(const uint16_t*, const StatSegs&, int64_t, void*, uint8_t*,
                                  cudaStream_t);
cudaError_t launch_encode(const uint16_t*, const EncodeSegs&, const uint8_t*, uint8_t*, void*,
                          uint64_t*, cudaStream_t, bool zeroed = false);
cudaError_t launch_decode(const DecodeSegs&, uint16_t*, int32_t*, void*, int, cudaStream_t);
cudaError_t launch_decode_groups(const uint8_t*, int64_t, int, int64_t, int64_t, uint16_t*,
                                 cudaStream_t);
int64_t encode_workspace_bytes(int64_t ntiles);
cudaError_t launch_encode_auto(const uint16_t*, const EncodeSegs&, const StatSegs&, int64_t,
                               uint8_t*, void*, uint64_t*, uint8_t*, double*, int, cudaStream_t);
}  // namespace zc

using namespace zc;

namespace zc {
namespace {
struct ProfState {
  std::mutex m;
  bool on = false;
  std::vector<cudaEvent_t> ev[kProfTags];   // begin/end pairs
  size_t used[kProfTags] = {0, 0};
};
ProfState g_prof;
constexpr size_t kProfMaxPairs = 4096;
}  // namespace

void prof_mark(int tag, bool end, cudaStream_t st) {
  if (!g_prof.on) return;
  std::lock_guard<std::mutex> lk(g_prof.m);
  if (!g_prof.on || tag < 0 || tag >= kProfTags) return;
  auto& v = g_prof.ev[tag];
  size_t& u = g_prof.used[tag];
  if (u >= kProfMaxPairs) return;
  const size_t i = 2 * u + (end ? 1 : 0);
  while (v.size() <= i) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    v.push_back(e);
  }
  cudaEventRecord(v[i], st);
  if (end) ++u;
}
}  // namespace zc

namespace {
constexpr int kStatusBadArg = -1;
constexpr int kStatusWorkspace = -2;
constexpr int kStatusTooLarge = -3;

int64_t tiles_of(int64_t n) { return (n + kTile - 1) / kTile; }

int status_of(cudaError_t e) { return e == cudaSuccess ? 0 : (int)e; }

struct Range {   // NVTX range around each codec entry point (header-only NVTX v3)
  explicit Range(const char* name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
};
}  // namespace


extern "C" {

int zc_abi_version(void) { return 2; }

int zc_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(g_prof.m);
  g_prof.on = on != 0;
  if (g_prof.on)
    for (int t = 0; t < kProfTags; ++t) g_prof.used[t] = 0;
  return 0;
}

int zc_profile_read(int tag, float* ms, int cap) {
  if (tag < 0 || tag >= kProfTags || (!ms && cap > 0)) return kStatusBadArg;
  std::lock_guard<std::mutex> lk(g_prof.m);
  const size_t n = g_prof.used[tag] < (size_t)cap ? g_prof.used[tag] : (size_t)cap;
  for (size_t i = 0; i < n; ++i) {
    cudaEvent_t a = g_prof.ev[tag][2 * i], b = g_prof.ev[tag][2 * i + 1];
    cudaError_t e = cudaEventSynchronize(b);
    if (e == cudaSuccess) e = cudaEventElapsedTime(ms + i, a, b);
    if (e != cudaSuccess) return (int)e;
  }
  return (int)n;
}

int zc_tile_elements(void) { return kTile; }

int zc_max_segments(void) { return kMaxSegments; }

const char* zc_status_string(int status) {
  switch (status) {
    case 0: return "ok";
    case kStatusBadArg: return "invalid argument";
    case kStatusWorkspace: return "workspace too small";
    case kStatusTooLarge: return "frame exceeds the u32 section-offset range";
    default: return status > 0 ? cudaGetErrorString((cudaError_t)status) : "unknown status";
  }
}

int64_t zc_static_bytes(int64_t n, int gs_log2) {
  if (n < 1 || gs_log2 < 0 || gs_log2 > 30) return -1;
  return layout_of(n, gs_log2).off[5];
}

int64_t zc_max_frame_bytes(int64_t n, int gs_log2) {
  if (n < 1 || gs_log2 < 0 || gs_log2 > 30) return -1;
  return layout_of(n, gs_log2).off[5] + pad128(n);
}

int64_t zc_workspace_bytes(int64_t total_elems, int nseg) {
  if (total_elems < 0 || nseg < 0) return -1;
  const int64_t tiles = total_elems / kTile + nseg + 1;
  const int64_t a = 128 + 32 * tiles + 4096;
  const int64_t b = encode_workspace_bytes(tiles);
  return a > b ? a : b;
}

int zc_codebook_measured(const uint16_t* x, const int64_t* seg_off, const int64_t* seg_n, int nseg,
                         void* ws, int64_t ws_bytes, uint8_t* book_dev, double* result_dev,
                         int flags, cudaStream_t stream) {
  Range nvtx_range("zc_codebook_measured");
  if (nseg < 0 || nseg > kMaxSegments || !book_dev || !result_dev || !ws) return kStatusBadArg;
  StatSegs s{};
  int k = 0;
  int64_t total = 0;
  s.tile_start[0] = 0;
  for (int i = 0; i < nseg; ++i) {
    if (seg_n[i] < 0) return kStatusBadArg;
    if (seg_n[i] == 0) continue;
    s.x_off[k] = seg_off[i];
    s.n[k] = seg_n[i];
    s.tile_start[k + 1] = s.tile_start[k] + tiles_of(seg_n[i]);
    total += seg_n[i];
    ++k;
  }
  s.nseg = k;
  if (k > 0 && !x) return kStatusBadArg;
  // (the numpy-order sigma passes use the area at kNpWsOff)
  if (128 + 32 * s.tile_start[k] > ws_bytes || kNpWsOff + kNpArea > ws_bytes)
    return kStatusWorkspace;
  return status_of(launch_codebook_measured(x, s, total, ws, book_dev, result_dev, flags & 1,
                                            stream));
}

int zc_codebook_modal(const uint16_t* x, const int64_t* seg_off, const int64_t* seg_n, int nseg,
                      void* ws, int64_t ws_bytes, uint8_t* book_dev, cudaStream_t stream) {
  Range nvtx_range("zc_codebook_modal");
  if (nseg < 0 || nseg > kMaxSegments || !book_dev || !ws) return kStatusBadArg;
  StatSegs s{};
  int k = 0;
  int64_t total = 0;
  for (int i = 0; i < nseg; ++i) {
    if (seg_n[i] < 0) return kStatusBadArg;
    if (seg_n[i] == 0) continue;
    s.x_off[k] = seg_off[i];
    s.n[k] = seg_n[i];
    s.tile_start[k + 1] = s.tile_start[k] + tiles_of(seg_n[i]);
    total += seg_n[i];
    ++k;
  }
  s.nseg = k;
  if (k > 0 && !x) return kStatusBadArg;
  if (128 + 2048 > ws_bytes) return kStatusWorkspace;
  return status_of(launch_codebook_modal(x, s, total, ws, book_dev, stream));
}

int zc_encode(const uint16_t* x, const int64_t* seg_off, const int64_t* seg_n,
              const int64_t* frame_off, int nseg, const uint8_t* book_dev, int gs_log2,
              uint8_t* frames, void* ws, int64_t ws_bytes, uint64_t* frame_len_dev,
              cudaStream_t stream) {
  Range nvtx_range("zc_encode");
  if (nseg < 1 || nseg > kMaxSegments || !x || !book_dev || !frames || !ws || !frame_len_dev)
    return kStatusBadArg;
  if (gs_log2 < 0 || gs_log2 > 30) return kStatusBadArg;
  EncodeSegs s{};
  s.nseg = nseg;
  s.gs_log2 = gs_log2;
  s.tile_start[0] = 0;
  for (int i = 0; i < nseg; ++i) {
    if (seg_n[i] < 1 || seg_off[i] < 0 || frame_off[i] < 0) return kStatusBadArg;
    if ((reinterpret_cast<uintptr_t>(frames + frame_off[i]) & (kAlign - 1)) != 0) return kStatusBadArg;
    if (layout_of(seg_n[i], gs_log2).off[5] > int64_t(0xFFFFFFFF)) return kStatusTooLarge;
    s.x_off[i] = seg_off[i];
    s.n[i] = seg_n[i];
    s.frame_off[i] = frame_off[i];
    s.tile_start[i + 1] = s.tile_start[i] + tiles_of(seg_n[i]);
  }
  if (encode_workspace_bytes(s.tile_start[nseg]) > ws_bytes) return kStatusWorkspace;
  return status_of(launch_encode(x, s, book_dev, frames, ws, frame_len_dev, stream));
}

int zc_encode_measured(const uint16_t* x, const int64_t* seg_off, const int64_t* seg_n,
                       const int64_t* frame_off, int nseg, int gs_log2, uint8_t* frames, void* ws,
                       int64_t ws_bytes, uint64_t* frame_len_dev, uint8_t* book_dev,
                       double* result_dev, int flags, cudaStream_t stream) {
  Range nvtx_range("zc_encode_measured");
  if (nseg < 1 || nseg > kMaxSegments || !x || !book_dev || !result_dev || !frames || !ws ||
      !frame_len_dev)
    return kStatusBadArg;
  if (gs_log2 < 0 || gs_log2 > 30) return kStatusBadArg;
  EncodeSegs s{};
  StatSegs ss{};
  s.nseg = nseg;
  ss.nseg = nseg;
  s.gs_log2 = gs_log2;
  int64_t total = 0;
  for (int i = 0; i < nseg; ++i) {
    if (seg_n[i] < 1 || seg_off[i] < 0 || frame_off[i] < 0) return kStatusBadArg;
    if ((reinterpret_cast<uintptr_t>(frames + frame_off[i]) & (kAlign - 1)) != 0) return kStatusBadArg;
    if (layout_of(seg_n[i], gs_log2).off[5] > int64_t(0xFFFFFFFF)) return kStatusTooLarge;
    s.x_off[i] = ss.x_off[i] = seg_off[i];
    s.n[i] = ss.n[i] = seg_n[i];
    s.frame_off[i] = frame_off[i];
    s.tile_start[i + 1] = ss.tile_start[i + 1] = s.tile_start[i] + tiles_of(seg_n[i]);
    total += seg_n[i];
  }
  if (encode_workspace_bytes(s.tile_start[nseg]) > ws_bytes ||
      128 + 32 * s.tile_start[nseg] > ws_bytes)
    return kStatusWorkspace;
  return status_of(launch_encode_auto(x, s, ss, total, frames, ws, frame_len_dev, book_dev,
                                      result_dev, flags & 1, stream));
}

int zc_decode(const uint8_t* const* stat, const uint8_t* const* dyn, const int64_t* dyn_len,
              const int64_t* n, const int64_t* out_off, int nseg, uint16_t* out, int32_t* err_dev,
              void* ws, int64_t ws_bytes, int write_out, cudaStream_t stream) {
  Range nvtx_range("zc_decode");
  if (nseg < 1 || nseg > kMaxSegments || !stat || !dyn || !n || !err_dev || !ws) return kStatusBadArg;
  if ((write_out & 1) && (!out || !out_off)) return kStatusBadArg;
  DecodeSegs s{};
  s.nseg = nseg;
  s.tile_start[0] = 0;
  for (int i = 0; i < nseg; ++i) {
    if (n[i] < 1 || !stat[i]) return kStatusBadArg;
    if ((reinterpret_cast<uintptr_t>(stat[i]) & 15) != 0) return kStatusBadArg;
    s.stat[i] = stat[i];
    s.dyn[i] = dyn[i];   // null: dynamic section follows the static part in place
    s.dyn_len[i] = dyn_len ? dyn_len[i] : -1;
    s.n[i] = n[i];
    s.out_off[i] = out_off ? out_off[i] : 0;
    s.tile_start[i + 1] = s.tile_start[i] + tiles_of(n[i]);
  }
  if (128 + 8 * s.tile_start[nseg] > ws_bytes) return kStatusWorkspace;
  // bits 0, 1, 3 (write / large groups / 512-element groups); pull mode is
  // the collectives' own
  return status_of(launch_decode(s, out, err_dev, ws, write_out & 11, stream));
}

int zc_decode_when_ready(const uint8_t* const* stat, const int64_t* n, const int64_t* out_off,
                         const uint64_t* const* ready, int nseg, uint64_t epoch,
                         int64_t timeout_ns, uint16_t* out, int32_t* err_dev, void* ws,
                         int64_t ws_bytes, cudaStream_t stream) {
  Range nvtx_range("zc_decode_when_ready");
  if (nseg < 1 || nseg > kMaxSegments || !stat || !n || !ready || !out || !err_dev || !ws)
    return kStatusBadArg;
  DecodeSegs s{};
  s.nseg = nseg;
  s.epoch = epoch;
  s.timeout_ns = timeout_ns;
  s.tile_start[0] = 0;
  for (int i = 0; i < nseg; ++i) {
    if (n[i] < 1 || !stat[i] || (reinterpret_cast<uintptr_t>(stat[i]) & 15) != 0) return kStatusBadArg;
    s.stat[i] = stat[i];
    s.dyn[i] = nullptr;
    s.dyn_len[i] = -1;
    s.n[i] = n[i];
    s.out_off[i] = out_off ? out_off[i] : 0;
    s.ready[i] = ready[i];
    s.tile_start[i + 1] = s.tile_start[i] + tiles_of(n[i]);
  }
  if (128 + 8 * s.tile_start[nseg] + 256 > ws_bytes) return kStatusWorkspace;
  // bit 0 write, bit 2 pull mode (the ring decoder; frames of <= 4096-element groups)
  return status_of(launch_decode(s, out, err_dev, ws, 1 | 4, stream));
}

int zc_decode_groups(const uint8_t* frame, int64_t n, int gs_log2, int64_t g0, int64_t g1,
                     uint16_t* out, cudaStream_t stream) {
  Range nvtx_range("zc_decode_groups");
  if (!frame || !out || n < 1 || gs_log2 < 0 || gs_log2 > 30) return kStatusBadArg;
  if ((reinterpret_cast<uintptr_t>(frame) & 7) != 0) return kStatusBadArg;
  const int64_t groups = (n + (int64_t(1) << gs_log2) - 1) >> gs_log2;
  if (g0 < 0 || g1 < g0 || g1 > groups) return kStatusBadArg;
  return status_of(launch_decode_groups(frame, n, gs_log2, g0, g1, out, stream));
}

}  // extern "C"
