// Native compressed collectives: communicator + the two data planes.
//
// Replaces the reference's collectives over its transport seam
// (collectives.py:203-341, transport.py:559-623) with C++ over NCCL / CUDA
// peer memory, exported through the C-ABI (include/zipccl_b200.h):
//
// * peer-memory plane ("p2p", the product on one NVLink/NVSwitch node):
//   every rank owns a symmetric buffer (two frame slots alternating by
//   epoch + a flag area) that its peers map (CUDA IPC, or plain pointers for
//   in-process ranks).  A call encodes into the slot, publishes
//   ready[me] = epoch in every peer's flag area with system-scope release
//   stores, and decodes the peers' frames STRAIGHT OUT OF THEIR HBM: the
//   decoder's producer warp claims work from whichever peer's frame is ready
//   (decode_ring_kernel<true>), so the NVLink transfer IS the decode and a
//   late peer never holds up the others.  No host round trip, no metadata
//   exchange: element counts are checked against each frame's header.
// * message plane ("msg", the reference's protocols over NCCL; in-process
//   ranks run the same code over a device-copy transport): the all-gather
//   exchanges one u64 per rank (element count + frame length packed) and
//   then the frames; the all-to-all runs design 1 (16 B of metadata per peer,
//   then frames) or design 2 (static sections pre-sized from recv_counts,
//   u64 dynamic sizes, dynamic sections) exactly as collectives.py:245-325,
//   so TrafficStats match the reference's size law.  With ZC_PIPELINE the
//   frames move in W-1 ring steps and each peer is decoded on a side stream
//   as soon as its step lands.
// * reduce-scatter: the all-to-all of shard frames followed by ONE fused
//   decode + fp32-reduce kernel (zc_reduce.cu) -- on the p2p plane it reads
//   every peer's frame for this shard over NVLink.
// * raw twins (ncclAllGather, grouped send/recv, raw all-to-all + the same
//   reduce kernel) for the adaptive switch and the baselines.
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "zc_common.cuh"

namespace zc {
cudaError_t launch_encode(const uint16_t*, const EncodeSegs&, const uint8_t*, uint8_t*, void*,
                          uint64_t*, cudaStream_t, bool zeroed = false);
cudaError_t launch_encode_auto(const uint16_t*, const EncodeSegs&, const StatSegs&, int64_t,
                               uint8_t*, void*, uint64_t*, uint8_t*, double*, int, cudaStream_t);
cudaError_t launch_decode(const DecodeSegs&, uint16_t*, int32_t*, void*, int, cudaStream_t);
cudaError_t launch_reduce(const RedSrc*, void*, int, int64_t, void*, int, int32_t*, uint64_t,
                          int64_t, cudaStream_t);
cudaError_t store_srcs(const RedSrc*, int, RedSrc*, cudaStream_t);
size_t reduce_hdr_bytes(int W);
cudaError_t preload_encode();
cudaError_t preload_decode();
cudaError_t preload_stats();
cudaError_t preload_reduce();
cudaError_t preload_estimate();
cudaError_t preload_small();
}  // namespace zc

extern "C" int64_t zc_workspace_bytes(int64_t total_elems, int nseg);

using namespace zc;

namespace {

// NVTX range around every collective call (host enqueue side): a profiler
// timeline shows each rank's encode / publish / decode launches under the
// collective that issued them (SURVEY §5 tracing).  Header-only NVTX v3.
struct Range {
  explicit Range(const char* name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
};

constexpr int kStatusBadArg = -1;
constexpr int kStatusProtocol = -4;    // sizes / counts disagree (ProtocolError)
constexpr int kStatusCapacity = -5;    // p2p slot too small for this all-to-all
constexpr int kStatusTransport = -6;   // NCCL failure, in-process rendezvous timeout
constexpr int kStatusCollective = -7;  // a peer's frame is unusable (CollectiveError, peer)

constexpr int64_t kFlagBytes = 4096;   // ready[64] | done[64] | stats | pad
constexpr int64_t kReadyOff = 0, kDoneOff = 512, kStatsOff = 1024;
// device-side wait bound for peer flags (ZC_TIMEOUT_MS overrides 30 s)
int64_t timeout_ns() {
  static const int64_t v = [] {
    const char* e = getenv("ZC_TIMEOUT_MS");
    return e ? (int64_t)atoll(e) * 1000000ll : 30ll * 1000 * 1000 * 1000;
  }();
  return v;
}
#define kTimeoutNs timeout_ns()
bool debug_on() {
  static const bool v = getenv("ZC_DEBUG") != nullptr;
  return v;
}

// flags
[[maybe_unused]] constexpr int kPlaneP2P = 1;   // the default plane (header ZC_PLANE_P2P)
constexpr int kPlaneMsg = 2, kA2AD1 = 4, kCheckCounts = 8, kPipeline = 16;

int64_t pad128h(int64_t x) { return (x + 127) / 128 * 128; }
int64_t tiles_of(int64_t n) { return (n + kTile - 1) / kTile; }
int64_t static_of(int64_t n) { return layout_of(n, 9).off[5]; }
int64_t maxframe_of(int64_t n) { return layout_of(n, 9).off[5] + pad128h(n); }

// ---- grow-only device buffer --------------------------------------------------
struct Buf {
  void* p = nullptr;
  int64_t cap = 0;
  // grows (after draining `st`: the old block may still be in use by it)
  cudaError_t need(int64_t bytes, cudaStream_t st) {
    if (bytes <= cap) return cudaSuccess;
    if (p) {
      cudaStreamSynchronize(st);
      cudaFree(p);
      p = nullptr;
      cap = 0;
    }
    int64_t c = std::max<int64_t>(bytes, 1 << 20);
    c = (c + (1 << 20) - 1) / (1 << 20) * (1 << 20);
    cudaError_t e = cudaMalloc(&p, (size_t)c);
    if (e != cudaSuccess) { p = nullptr; return e; }
    cap = c;
    return cudaSuccess;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
  void release() { if (p) cudaFree(p); p = nullptr; cap = 0; }
};

// ---- in-process rendezvous (thread ranks) --------------------------------------
struct Hub {
  explicit Hub(int w) : world(w), box(w, nullptr) {}
  int world;
  std::mutex m;
  std::condition_variable cv;
  std::vector<const void*> box;
  int arrived = 0, readers = 0;
  uint64_t gen = 0;
  bool draining = false, aborted = false;

  // Every rank deposits `mine` and receives everybody's; the box is not
  // reused until every rank has copied it.  false on timeout / abort.
  bool exchange(int rank, const void* mine, std::vector<const void*>& all) {
    std::unique_lock<std::mutex> lk(m);
    const auto deadline = std::chrono::steady_clock::now() + std::chrono::seconds(60);
    while (draining && !aborted)
      if (cv.wait_until(lk, deadline) == std::cv_status::timeout) { aborted = true; cv.notify_all(); }
    if (aborted) return false;
    box[rank] = mine;
    const uint64_t g = gen;
    if (++arrived == world) {
      draining = true;
      readers = world;
      ++gen;
      cv.notify_all();
    } else {
      while (gen == g && !aborted)
        if (cv.wait_until(lk, deadline) == std::cv_status::timeout) { aborted = true; cv.notify_all(); }
      if (aborted) return false;
    }
    all = box;
    if (--readers == 0) {
      draining = false;
      arrived = 0;
      cv.notify_all();
    }
    return true;
  }
  void abort() {
    std::lock_guard<std::mutex> lk(m);
    aborted = true;
    cv.notify_all();
  }
};

// One message of the message plane.
struct Msg {
  int peer;
  const void* ptr;   // send source / receive destination
  int64_t bytes;
};

}  // namespace

struct zc_comm {
  int rank = 0, world = 1, device = 0;
  ncclComm_t nccl = nullptr;
  std::shared_ptr<Hub> hub;
  bool shared_device = false;
  bool p2p = false;
  // peer memory
  uint8_t* sym = nullptr;
  int64_t slot_bytes = 0;
  std::vector<uint8_t*> peer_sym;
  std::vector<void*> opened;
  uint64_t epoch = 0;
  // scratch
  Buf ws, sendbuf, recvbuf, small, srcs;
  uint64_t* pinned = nullptr;             // host, 4 x 64 u64 (size read-back)
  cudaEvent_t ev_post = nullptr, ev_copied = nullptr;
  cudaStream_t side = nullptr;
  std::vector<cudaEvent_t> step_ev;
  uint64_t host_bytes = 0, host_msgs = 0;
  std::string last_error;
  int last_peer = -1;

  int fail(int status, const std::string& msg, int peer = -1) {
    last_error = msg;
    last_peer = peer;
    return status;
  }
  uint8_t* flags() const { return sym; }
  uint64_t* ready_local() const { return reinterpret_cast<uint64_t*>(sym + kReadyOff); }
  uint64_t* done_local() const { return reinterpret_cast<uint64_t*>(sym + kDoneOff); }
  uint64_t* dstats() const { return reinterpret_cast<uint64_t*>(sym + kStatsOff); }
  uint8_t* slot_of(int r, uint64_t e) const {
    return peer_sym[r] + kFlagBytes + (int64_t)(e & 1) * slot_bytes;
  }
};

namespace {

// ---------------------------------------------------------------------------
// small kernels of the p2p plane

struct PeerFlagPtrs {
  uint64_t* p[kMaxSegments];
};

// ready/done publication: zero the invalidated frame headers, account the
// bytes peers will pull, release-store `epoch` into slot `me` of every peer's
// flag array.
__global__ void publish_kernel(PeerFlagPtrs targets, int world, int me, uint64_t epoch,
                               const uint64_t* __restrict__ flen, int nflen, int64_t mult,
                               int64_t extra_bytes, uint64_t* __restrict__ stats, PeerFlagPtrs zap,
                               int nzap) {
  const int t = threadIdx.x;
  if (t < nzap) {
    uint4* h = reinterpret_cast<uint4*>(zap.p[t]);
    for (int i = 0; i < 8; ++i) h[i] = make_uint4(0, 0, 0, 0);
  }
  if (t == 0 && stats) {
    uint64_t b = 0;
    for (int i = 0; i < nflen; ++i) b += flen[i];
    b = b * (uint64_t)mult + (uint64_t)extra_bytes;
    stats[0] += b;
    stats[1] += (uint64_t)(world - 1);
  }
  __syncthreads();
  __threadfence_system();
  if (t < world && t != me && targets.p[t]) st_release_sys_u64(targets.p[t] + me, epoch);
}

// wait until flags[p] >= epoch for every p != me (bounded; err[p] = timeout)
__global__ void wait_flags_kernel(const uint64_t* flags, int world, int me, uint64_t epoch,
                                  int64_t timeout_ns, int32_t* err) {
  const int p = threadIdx.x;
  if (p >= world || p == me) return;
  const uint64_t t0 = globaltimer_ns();
  while (ld_acquire_sys_u64(flags + p) < epoch) {
    if (timeout_ns > 0 && (int64_t)(globaltimer_ns() - t0) > timeout_ns) {
      if (err) atomicMin(err + p, (int32_t)kErrTimeout);
      return;
    }
    __nanosleep(200);
  }
}

// err_dev[rank] from the decoder's per-segment words (+ self = ok), then the
// done publication (so a peer may reuse its slot).
__global__ void finish_kernel(const int32_t* __restrict__ seg_err, PeerFlagPtrs seg_rank,
                              int nseg, int32_t* __restrict__ err, int world, int me,
                              PeerFlagPtrs done_targets, uint64_t epoch) {
  const int t = threadIdx.x;
  if (err && t < world) {
    int32_t v = 0x7F7F7F7F;
    for (int i = 0; i < nseg; ++i)
      if ((int)(intptr_t)seg_rank.p[i] == t) v = seg_err[i];
    if (err[t] != v && t != me) err[t] = v < err[t] ? v : err[t];
    if (t == me) err[t] = 0x7F7F7F7F;
  }
  if (done_targets.p[0] || world > 1) {
    __syncthreads();
    __threadfence_system();
    if (t < world && t != me && done_targets.p[t]) st_release_sys_u64(done_targets.p[t] + me, epoch);
  }
}

__global__ void init_err_kernel(int32_t* err, int n) {
  const int t = threadIdx.x;
  if (t < n) err[t] = 0x7F7F7F7F;
}

// per-rank error words from a message-plane decode (segment i = rank seg_rank[i])
__global__ void map_err_kernel(const int32_t* __restrict__ seg_err, PeerFlagPtrs seg_rank,
                               int nseg, int32_t* __restrict__ err, int world) {
  const int t = threadIdx.x;
  if (t >= world) return;
  int32_t v = err[t];
  for (int i = 0; i < nseg; ++i)
    if ((int)(intptr_t)seg_rank.p[i] == t && seg_err[i] < v) v = seg_err[i];
  err[t] = v;
}

// ---------------------------------------------------------------------------
// message-plane transport: NCCL, or device copies between in-process ranks

struct Post {
  const std::vector<Msg>* sends;
  const void* send1;       // all-gather source
  int64_t bytes1;
  cudaEvent_t ev;
};

int check_nccl(zc_comm* c, ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return 0;
  return c->fail(kStatusTransport, std::string(what) + ": " + ncclGetErrorString(r));
}

int t_allgather(zc_comm* c, const void* send, void* recv, int64_t bytes, cudaStream_t st) {
  if (c->world == 1 || bytes == 0) {
    if (bytes && send != recv) cudaMemcpyAsync(recv, send, (size_t)bytes, cudaMemcpyDefault, st);
    return 0;
  }
  if (c->nccl)
    return check_nccl(c, ncclAllGather(send, recv, (size_t)bytes, ncclUint8, c->nccl, st),
                      "ncclAllGather");
  Post mine{nullptr, send, bytes, c->ev_post};
  cudaEventRecord(c->ev_post, st);
  std::vector<const void*> all;
  if (!c->hub->exchange(c->rank, &mine, all)) return c->fail(kStatusTransport, "rendezvous timed out");
  int status = 0;
  for (int p = 0; p < c->world; ++p) {
    const Post* q = reinterpret_cast<const Post*>(all[p]);
    if (q->bytes1 != bytes) {
      status = c->fail(kStatusProtocol, "all-gather size mismatch with rank " + std::to_string(p), p);
      continue;
    }
    if (p != c->rank) cudaStreamWaitEvent(st, q->ev, 0);
    uint8_t* dst = reinterpret_cast<uint8_t*>(recv) + (int64_t)p * bytes;
    if (q->send1 != dst) cudaMemcpyAsync(dst, q->send1, (size_t)bytes, cudaMemcpyDefault, st);
  }
  cudaEventRecord(c->ev_copied, st);
  // the event handle travels by value (a peer may leave before we read)
  if (!c->hub->exchange(c->rank, reinterpret_cast<const void*>(c->ev_copied), all))
    return c->fail(kStatusTransport, "rendezvous timed out");
  for (int p = 0; p < c->world; ++p)
    if (p != c->rank) cudaStreamWaitEvent(st, reinterpret_cast<cudaEvent_t>(const_cast<void*>(all[p])), 0);
  return status;
}

// Grouped point-to-point: sends/recvs of exact sizes (recv sizes are the
// receiver's expectation).  The in-process transport checks both sides and
// reports a disagreement as a protocol error naming `label`; NCCL cannot.
int t_exchange(zc_comm* c, const std::vector<Msg>& sends, const std::vector<Msg>& recvs,
               cudaStream_t st, const char* label) {
  if (c->nccl) {
    ncclGroupStart();
    for (const Msg& m : sends)
      if (m.bytes) ncclSend(m.ptr, (size_t)m.bytes, ncclUint8, m.peer, c->nccl, st);
    for (const Msg& m : recvs)
      if (m.bytes) ncclRecv(const_cast<void*>(m.ptr), (size_t)m.bytes, ncclUint8, m.peer, c->nccl, st);
    return check_nccl(c, ncclGroupEnd(), "ncclSend/ncclRecv");
  }
  Post mine{&sends, nullptr, 0, c->ev_post};
  cudaEventRecord(c->ev_post, st);
  std::vector<const void*> all;
  if (!c->hub->exchange(c->rank, &mine, all)) return c->fail(kStatusTransport, "rendezvous timed out");
  int status = 0;
  for (int p = 0; p < c->world; ++p) {
    if (p == c->rank) continue;
    const Post* q = reinterpret_cast<const Post*>(all[p]);
    const Msg* src = nullptr;
    for (const Msg& m : *q->sends)
      if (m.peer == c->rank && m.bytes) src = &m;
    const Msg* dst = nullptr;
    for (const Msg& m : recvs)
      if (m.peer == p && m.bytes) dst = &m;
    const int64_t got = src ? src->bytes : 0, want = dst ? dst->bytes : 0;
    if (got != want) {
      if (!status)
        status = c->fail(kStatusProtocol, std::string(label) + " from rank " + std::to_string(p) +
                                              " is " + std::to_string(got) + " bytes, expected " +
                                              std::to_string(want), p);
      continue;
    }
    if (!want) continue;
    cudaStreamWaitEvent(st, q->ev, 0);
    cudaMemcpyAsync(const_cast<void*>(dst->ptr), src->ptr, (size_t)want, cudaMemcpyDefault, st);
  }
  cudaEventRecord(c->ev_copied, st);
  // the event handle travels by value (a peer may leave before we read)
  if (!c->hub->exchange(c->rank, reinterpret_cast<const void*>(c->ev_copied), all))
    return c->fail(kStatusTransport, "rendezvous timed out");
  for (int p = 0; p < c->world; ++p)
    if (p != c->rank) cudaStreamWaitEvent(st, reinterpret_cast<cudaEvent_t>(const_cast<void*>(all[p])), 0);
  return status;
}

// u64 per peer (exchange_sizes, transport.py:607-623); host result; syncs st.
int t_sizes(zc_comm* c, const std::vector<uint64_t>& out_vals, int words_per_peer,
            std::vector<uint64_t>& in_vals, cudaStream_t st, const char* label) {
  const int W = c->world, k = words_per_peer;
  cudaError_t e = c->small.need((int64_t)16 * W * k + 256, st);
  if (e != cudaSuccess) return (int)e;
  uint64_t* sbuf = c->small.as<uint64_t>();
  uint64_t* rbuf = sbuf + W * k;
  for (int i = 0; i < W * k; ++i) c->pinned[i] = out_vals[i];
  cudaMemcpyAsync(sbuf, c->pinned, sizeof(uint64_t) * W * k, cudaMemcpyHostToDevice, st);
  // the self entries too, so the read-back below copies initialised memory only
  cudaMemcpyAsync(rbuf + c->rank * k, sbuf + c->rank * k, sizeof(uint64_t) * k,
                  cudaMemcpyDeviceToDevice, st);
  std::vector<Msg> s, r;
  for (int p = 0; p < W; ++p) {
    if (p == c->rank) continue;
    s.push_back({p, sbuf + p * k, 8 * k});
    r.push_back({p, rbuf + p * k, 8 * k});
  }
  int rc = t_exchange(c, s, r, st, label);
  if (rc) return rc;
  cudaMemcpyAsync(c->pinned + 128, rbuf, sizeof(uint64_t) * W * k, cudaMemcpyDeviceToHost, st);
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return (int)e;
  in_vals.assign(c->pinned + 128, c->pinned + 128 + W * k);
  for (int j = 0; j < k; ++j) in_vals[c->rank * k + j] = out_vals[c->rank * k + j];
  c->host_bytes += (uint64_t)8 * k * (W - 1);
  c->host_msgs += (uint64_t)(W - 1);
  return 0;
}

// ---------------------------------------------------------------------------
// encode helpers

// frames of segments (x_off[i], n[i]) at frames + frame_off[i]; measured
// codebook over all of them unless book is given.
int encode_segments(zc_comm* c, const uint16_t* x, const std::vector<int64_t>& xo,
                    const std::vector<int64_t>& nn, const std::vector<int64_t>& fo,
                    uint8_t* frames, const uint8_t* book, uint64_t* flen, cudaStream_t st) {
  const int nseg = (int)nn.size();
  if (nseg == 0) return 0;
  if (nseg > kMaxSegments) return c->fail(kStatusBadArg, "too many segments");
  EncodeSegs s{};
  StatSegs ss{};
  s.nseg = ss.nseg = nseg;
  s.gs_log2 = 9;
  int64_t total = 0;
  for (int i = 0; i < nseg; ++i) {
    if (static_of(nn[i]) > int64_t(0xFFFFFFFF))
      return c->fail(-3, "frame exceeds the u32 section-offset range");
    s.x_off[i] = ss.x_off[i] = xo[i];
    s.n[i] = ss.n[i] = nn[i];
    s.frame_off[i] = fo[i];
    s.tile_start[i + 1] = ss.tile_start[i + 1] = s.tile_start[i] + tiles_of(nn[i]);
    total += nn[i];
  }
  cudaError_t e = c->ws.need(zc_workspace_bytes(total, nseg) + 4096, st);
  if (e != cudaSuccess) return (int)e;
  uint8_t* w = c->ws.as<uint8_t>();
  if (book) {
    e = launch_encode(x, s, book, frames, w + 4096, flen, st);
  } else {
    uint8_t* bk = w;                                   // book[8] + result[3]
    double* res = reinterpret_cast<double*>(w + 64);
    e = launch_encode_auto(x, s, ss, total, frames, w + 4096, flen, bk, res, 1, st);
  }
  return (int)e;
}

int cuda_status(cudaError_t e) { return e == cudaSuccess ? 0 : (int)e; }

// the per-call scratch layout in c->small (after the size exchange area)
struct Scratch {
  uint64_t* flen;      // [64]
  int32_t* seg_err;    // [64]
};
Scratch scratch_of(zc_comm* c) {
  uint8_t* b = c->small.as<uint8_t>() + 8192;
  return {reinterpret_cast<uint64_t*>(b), reinterpret_cast<int32_t*>(b + 512)};
}
int need_small(zc_comm* c, cudaStream_t st) {
  return cuda_status(c->small.need(8192 + 4096, st));
}

PeerFlagPtrs flag_targets(zc_comm* c, int64_t off) {
  PeerFlagPtrs t{};
  for (int p = 0; p < c->world && p < kMaxSegments; ++p)
    t.p[p] = (p == c->rank) ? nullptr : reinterpret_cast<uint64_t*>(c->peer_sym[p] + off);
  return t;
}

// ---------------------------------------------------------------------------
// peer-memory plane

int p2p_begin(zc_comm* c, int32_t* err, cudaStream_t st, uint64_t& e) {
  e = ++c->epoch;
  if (debug_on()) fprintf(stderr, "[zc] rank %d p2p epoch %llu shared %d\n", c->rank, (unsigned long long)e, (int)c->shared_device);
  if (err) init_err_kernel<<<1, 64, 0, st>>>(err, c->world);
  if (e >= 3)   // the slot of epoch e - 2 must have been read by every peer
    wait_flags_kernel<<<1, 64, 0, st>>>(c->done_local(), c->world, c->rank, e - 2, kTimeoutNs, err);
  return cuda_status(cudaGetLastError());
}

// Ranks sharing one GPU (in-process test groups) must never spin on the
// device for each other: a spinning kernel can starve the peer's encoder of
// SMs, and any lazily loaded kernel waits for the device.  They meet on the
// host instead, after each one's publication has executed; the device-side
// waits that follow then find their flags set.
int p2p_host_meet(zc_comm* c, cudaStream_t st) {
  if (!c->shared_device || !c->hub) return 0;
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return (int)e;
  std::vector<const void*> all;
  if (!c->hub->exchange(c->rank, nullptr, all)) return c->fail(kStatusTransport, "rendezvous timed out");
  return 0;
}

int p2p_decode(zc_comm* c, const std::vector<int>& peers, const std::vector<int64_t>& stat_off,
               const std::vector<int64_t>& counts, const std::vector<int64_t>& out_off,
               uint16_t* out, int32_t* err, uint64_t e, cudaStream_t st) {
  Scratch sc = scratch_of(c);
  PeerFlagPtrs seg_rank{};
  const int nseg = (int)peers.size();
  int rc = p2p_host_meet(c, st);
  if (rc) return rc;
  if (nseg) {
    DecodeSegs s{};
    s.nseg = nseg;
    s.epoch = e;
    s.timeout_ns = kTimeoutNs;
    for (int i = 0; i < nseg; ++i) {
      const int p = peers[i];
      s.stat[i] = c->slot_of(p, e) + stat_off[i];
      s.dyn[i] = nullptr;
      s.dyn_len[i] = -1;
      s.n[i] = counts[i];
      s.out_off[i] = out_off[i];
      s.ready[i] = c->ready_local() + p;
      s.tile_start[i + 1] = s.tile_start[i] + tiles_of(counts[i]);
      seg_rank.p[i] = reinterpret_cast<uint64_t*>((intptr_t)p);
    }
    int64_t total = 0;
    for (auto v : counts) total += v;
    cudaError_t ce = c->ws.need(zc_workspace_bytes(total, nseg) + 4096, st);
    if (ce != cudaSuccess) return (int)ce;
    ce = launch_decode(s, out, sc.seg_err, c->ws.p, 1 | 4 | 8, st);
    if (ce != cudaSuccess) return (int)ce;
  }
  finish_kernel<<<1, 64, 0, st>>>(sc.seg_err, seg_rank, nseg, err, c->world, c->rank,
                                  flag_targets(c, kDoneOff), e);
  if (debug_on()) fprintf(stderr, "[zc] rank %d decode enqueued (%d segs)\n", c->rank, nseg);
  return cuda_status(cudaGetLastError());
}


int p2p_grow(zc_comm* c, int64_t need, cudaStream_t st);

int p2p_allgather(zc_comm* c, const uint16_t* x, int64_t n, uint16_t* out, const uint8_t* book,
                  int32_t* err, cudaStream_t st) {
  const int W = c->world, me = c->rank;
  if (maxframe_of(n) > c->slot_bytes) {
    int rc = p2p_grow(c, maxframe_of(n), st);
    if (rc) return rc;
  }
  int rc = need_small(c, st);
  if (rc) return rc;
  uint64_t e = 0;
  if ((rc = p2p_begin(c, err, st, e))) return rc;
  Scratch sc = scratch_of(c);
  if ((rc = encode_segments(c, x, {0}, {n}, {0}, c->slot_of(me, e), book, sc.flen, st))) return rc;
  PeerFlagPtrs zap{};
  // the peers pull F bytes each; flags: ready + done, 8 B per peer each
  publish_kernel<<<1, 64, 0, st>>>(flag_targets(c, kReadyOff), W, me, e, sc.flen, 1, W - 1,
                                   16 * (W - 1), c->dstats(), zap, 0);
  cudaMemcpyAsync(out + (int64_t)me * n, x, sizeof(uint16_t) * n, cudaMemcpyDeviceToDevice, st);
  std::vector<int> peers;
  std::vector<int64_t> so, cn, oo;
  for (int p = 0; p < W; ++p) {
    if (p == me) continue;
    peers.push_back(p);
    so.push_back(0);
    cn.push_back(n);
    oo.push_back((int64_t)p * n);
  }
  return p2p_decode(c, peers, so, cn, oo, out, err, e, st);
}

// All-to-all frames live in fixed per-destination regions of the sender's
// slot (region q = slot + q * region), so a receiver locates its frame from
// the sender's rank alone -- no offset exchange, no host round trip.  A pair
// whose frame cannot fit is skipped by both sides (both see the same count)
// and reported as kStatusCapacity after the protocol completed.
int64_t region_of(const zc_comm* c) { return (c->slot_bytes / c->world) / 128 * 128; }

int p2p_alltoall_encode(zc_comm* c, const uint16_t* x, const int64_t* sc_, const int64_t* rc,
                        const uint8_t* book, uint64_t e, cudaStream_t st, bool& overflow,
                        int64_t& flen_count) {
  const int W = c->world, me = c->rank;
  const int64_t region = region_of(c);
  std::vector<int64_t> xo, nn, fo;
  PeerFlagPtrs zap{};
  int nzap = 0;
  int64_t off = 0;
  overflow = false;
  for (int q = 0; q < W; ++q) {
    const int64_t cnt = sc_[q];
    if (q != me) {
      const bool fits = cnt > 0 && maxframe_of(cnt) <= region;
      if (cnt > 0 && !fits) overflow = true;
      if (rc[q] > 0 && maxframe_of(rc[q]) > region) overflow = true;
      if (fits) {
        xo.push_back(off);
        nn.push_back(cnt);
        fo.push_back((int64_t)q * region);
      } else {
        zap.p[nzap++] = reinterpret_cast<uint64_t*>(c->slot_of(me, e) + (int64_t)q * region);
      }
    }
    off += cnt;
  }
  Scratch s = scratch_of(c);
  int rc2 = encode_segments(c, x, xo, nn, fo, c->slot_of(me, e), book, s.flen, st);
  if (rc2) return rc2;
  flen_count = (int64_t)nn.size();
  if (debug_on()) fprintf(stderr, "[zc] rank %d a2a encoded, publishing epoch %llu\n", me, (unsigned long long)e);
  publish_kernel<<<1, 64, 0, st>>>(flag_targets(c, kReadyOff), W, me, e, s.flen, (int)nn.size(),
                                   1, 16 * (W - 1), c->dstats(), zap, nzap);
  if (debug_on()) fprintf(stderr, "[zc] rank %d published\n", me);
  return cuda_status(cudaGetLastError());
}

int p2p_alltoall(zc_comm* c, const uint16_t* x, const int64_t* sc_, const int64_t* rc,
                 uint16_t* out, const uint8_t* book, int32_t* err, cudaStream_t st) {
  const int W = c->world, me = c->rank;
  int rc0 = need_small(c, st);
  if (rc0) return rc0;
  uint64_t e = 0;
  if ((rc0 = p2p_begin(c, err, st, e))) return rc0;
  bool overflow = false;
  int64_t nf = 0;
  if ((rc0 = p2p_alltoall_encode(c, x, sc_, rc, book, e, st, overflow, nf))) return rc0;
  const int64_t region = region_of(c);
  int64_t xoff = 0, ooff = 0;
  std::vector<int> peers;
  std::vector<int64_t> so, cn, oo;
  for (int p = 0; p < W; ++p) {
    if (p == me) {
      if (sc_[p])
        cudaMemcpyAsync(out + ooff, x + xoff, sizeof(uint16_t) * sc_[p], cudaMemcpyDeviceToDevice, st);
    } else if (rc[p] > 0 && maxframe_of(rc[p]) <= region) {
      peers.push_back(p);
      so.push_back((int64_t)me * region);
      cn.push_back(rc[p]);
      oo.push_back(ooff);
    }
    xoff += sc_[p];
    ooff += (p == me) ? sc_[p] : rc[p];
  }
  rc0 = p2p_decode(c, peers, so, cn, oo, out, err, e, st);
  if (rc0) return rc0;
  if (overflow)
    return c->fail(kStatusCapacity, "all-to-all frame exceeds the peer-memory region of " +
                                        std::to_string(region) + " bytes; reserve a larger "
                                        "workspace (zc_comm_reserve)");
  return 0;
}

int p2p_reduce_scatter(zc_comm* c, const uint16_t* x, int64_t shard, void* out, int f32,
                       const uint8_t* book, int32_t* err, cudaStream_t st) {
  const int W = c->world, me = c->rank;
  if ((int64_t)W * (maxframe_of(shard) + 128) > c->slot_bytes) {
    int rc = p2p_grow(c, (int64_t)W * (maxframe_of(shard) + 128), st);
    if (rc) return rc;
  }
  int rc0 = need_small(c, st);
  if (rc0) return rc0;
  uint64_t e = 0;
  if ((rc0 = p2p_begin(c, err, st, e))) return rc0;
  std::vector<int64_t> cnt(W, shard);
  bool overflow = false;
  int64_t nf = 0;
  if ((rc0 = p2p_alltoall_encode(c, x, cnt.data(), cnt.data(), book, e, st, overflow, nf))) return rc0;
  if ((rc0 = p2p_host_meet(c, st))) return rc0;
  const int64_t region = region_of(c);
  std::vector<RedSrc> src(W);
  for (int p = 0; p < W; ++p) {
    RedSrc r{};
    if (p == me) {
      r.stat = reinterpret_cast<const uint8_t*>(x + (int64_t)me * shard);
      r.raw = 1;
    } else {
      r.stat = c->slot_of(p, e) + (int64_t)me * region;
      r.dyn_len = -1;
      r.ready = c->ready_local() + p;
    }
    src[p] = r;
  }
  cudaError_t ce = c->srcs.need((int64_t)(sizeof(RedSrc) + 64) * W + 4096, st);
  if (ce != cudaSuccess) return (int)ce;
  RedSrc* sd = c->srcs.as<RedSrc>();
  void* hdr = c->srcs.as<uint8_t>() + sizeof(RedSrc) * W + 256;
  if ((ce = store_srcs(src.data(), W, sd, st)) != cudaSuccess) return (int)ce;
  // err[] of the reduce is indexed by rank already
  int32_t* e_out = err ? err : scratch_of(c).seg_err;
  if ((ce = launch_reduce(sd, hdr, W, shard, out, f32, e_out, e, kTimeoutNs, st)) != cudaSuccess)
    return (int)ce;
  PeerFlagPtrs none{};
  finish_kernel<<<1, 64, 0, st>>>(nullptr, none, 0, nullptr, W, me, flag_targets(c, kDoneOff), e);
  return cuda_status(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// message plane

__global__ void pack_size_kernel(const uint64_t* flen, int64_t n, uint64_t* out) {
  if (threadIdx.x == 0) out[0] = (uint64_t)n | ((flen[0] / 128) << 32);
}

int decode_local(zc_comm* c, const std::vector<int>& ranks, const std::vector<const uint8_t*>& stat,
                 const std::vector<const uint8_t*>& dyn, const std::vector<int64_t>& dyn_len,
                 const std::vector<int64_t>& counts, const std::vector<int64_t>& out_off,
                 uint16_t* out, int32_t* err, int32_t* seg_err, cudaStream_t st) {
  const int nseg = (int)ranks.size();
  if (!nseg) return 0;
  DecodeSegs s{};
  s.nseg = nseg;
  PeerFlagPtrs sr{};
  int64_t total = 0;
  for (int i = 0; i < nseg; ++i) {
    s.stat[i] = stat[i];
    s.dyn[i] = dyn[i];
    s.dyn_len[i] = dyn_len[i];
    s.n[i] = counts[i];
    s.out_off[i] = out_off[i];
    s.tile_start[i + 1] = s.tile_start[i] + tiles_of(counts[i]);
    sr.p[i] = reinterpret_cast<uint64_t*>((intptr_t)ranks[i]);
    total += counts[i];
  }
  cudaError_t ce = c->ws.need(zc_workspace_bytes(total, nseg) + 4096, st);
  if (ce != cudaSuccess) return (int)ce;
  ce = launch_decode(s, out, seg_err, c->ws.p, 1 | 8, st);
  if (ce != cudaSuccess) return (int)ce;
  if (err) map_err_kernel<<<1, 64, 0, st>>>(seg_err, sr, nseg, err, c->world);
  return cuda_status(cudaGetLastError());
}

int msg_allgather(zc_comm* c, const uint16_t* x, int64_t n, uint16_t* out, const uint8_t* book,
                  int32_t* err, int flags, cudaStream_t st) {
  const int W = c->world, me = c->rank;
  int rc = need_small(c, st);
  if (rc) return rc;
  Scratch s = scratch_of(c);
  if (err) init_err_kernel<<<1, 64, 0, st>>>(err, W);
  cudaError_t ce = c->sendbuf.need(maxframe_of(n), st);
  if (ce != cudaSuccess) return (int)ce;
  if ((rc = encode_segments(c, x, {0}, {n}, {0}, c->sendbuf.as<uint8_t>(), book, s.flen, st))) return rc;
  // size phase: one u64 per rank = element count | frame length / 128 << 32
  // (the reference's exchange_sizes of the frame length, collectives.py:215)
  uint64_t* packed = c->small.as<uint64_t>() + 512;
  pack_size_kernel<<<1, 32, 0, st>>>(s.flen, n, packed);
  if ((rc = t_allgather(c, packed, packed + 1, 8, st))) return rc;
  cudaMemcpyAsync(c->pinned, packed + 1, 8 * W, cudaMemcpyDeviceToHost, st);
  if ((ce = cudaStreamSynchronize(st)) != cudaSuccess) return (int)ce;
  std::vector<int64_t> len(W);
  for (int p = 0; p < W; ++p) {
    const int64_t np = (int64_t)(c->pinned[p] & 0xFFFFFFFFull);
    len[p] = (int64_t)(c->pinned[p] >> 32) * 128;
    if (np != n)
      return c->fail(kStatusCollective, "frame holds " + std::to_string(np) +
                                            " elements, expected " + std::to_string(n), p);
  }
  c->host_bytes += (uint64_t)(8 + len[me]) * (W - 1);
  c->host_msgs += (uint64_t)2 * (W - 1);
  std::vector<int64_t> roff(W + 1, 0);
  for (int p = 0; p < W; ++p) roff[p + 1] = roff[p] + (p == me ? 0 : len[p]);
  if ((ce = c->recvbuf.need(roff[W] + 128, st)) != cudaSuccess) return (int)ce;
  uint8_t* rb = c->recvbuf.as<uint8_t>();
  const uint8_t* mine = c->sendbuf.as<uint8_t>();
  cudaMemcpyAsync(out + (int64_t)me * n, x, sizeof(uint16_t) * n, cudaMemcpyDeviceToDevice, st);
  if (!(flags & kPipeline)) {
    std::vector<Msg> sends, recvs;
    for (int p = 0; p < W; ++p) {
      if (p == me) continue;
      sends.push_back({p, mine, len[me]});
      recvs.push_back({p, rb + roff[p], len[p]});
    }
    if ((rc = t_exchange(c, sends, recvs, st, "frame"))) return rc;
    std::vector<int> ranks;
    std::vector<const uint8_t*> stp, dyn;
    std::vector<int64_t> dl, cn, oo;
    for (int p = 0; p < W; ++p) {
      if (p == me) continue;
      ranks.push_back(p);
      stp.push_back(rb + roff[p]);
      dyn.push_back(nullptr);
      dl.push_back(len[p] - static_of(n));
      cn.push_back(n);
      oo.push_back((int64_t)p * n);
    }
    return decode_local(c, ranks, stp, dyn, dl, cn, oo, out, err, s.seg_err, st);
  }
  // pipelined: W-1 ring steps; peer (me - k) is decoded on the side stream
  // as soon as step k landed, while step k + 1 moves
  if ((int)c->step_ev.size() < W) {
    for (int i = (int)c->step_ev.size(); i < W; ++i) {
      cudaEvent_t ev;
      cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      c->step_ev.push_back(ev);
    }
  }
  cudaEventRecord(c->step_ev[0], st);
  cudaStreamWaitEvent(c->side, c->step_ev[0], 0);   // the side stream follows st's history
  for (int k = 1; k < W; ++k) {
    const int to = (me + k) % W, from = (me - k + W) % W;
    std::vector<Msg> sends{{to, mine, len[me]}}, recvs{{from, rb + roff[from], len[from]}};
    if ((rc = t_exchange(c, sends, recvs, st, "frame"))) return rc;
    cudaEventRecord(c->step_ev[k], st);
    cudaStreamWaitEvent(c->side, c->step_ev[k], 0);
    if ((rc = decode_local(c, {from}, {rb + roff[from]}, {nullptr}, {len[from] - static_of(n)},
                           {n}, {(int64_t)from * n}, out, err, s.seg_err + 2 * k, c->side)))
      return rc;
  }
  cudaEventRecord(c->step_ev[0], c->side);
  cudaStreamWaitEvent(st, c->step_ev[0], 0);
  return 0;
}

// Exchange of all-to-all frames (design 1 or 2) into c->recvbuf; returns per
// peer the static / dynamic pointers of the received frame.
struct Recv {
  std::vector<const uint8_t*> stat, dyn;
  std::vector<int64_t> dyn_len;
};

int msg_a2a_exchange(zc_comm* c, const uint16_t* x, const int64_t* sc_, const int64_t* rc,
                     const uint8_t* book, int flags, cudaStream_t st, Recv& R) {
  const int W = c->world, me = c->rank;
  int rc0 = need_small(c, st);
  if (rc0) return rc0;
  Scratch s = scratch_of(c);
  const bool d1 = flags & kA2AD1;
  // counts check first: design 1 always (its metadata), design 2 on request
  std::vector<int64_t> fo(W, 0);
  int64_t pos = 0;
  std::vector<int64_t> xo, nn, fof;
  std::vector<int> seg_peer;
  int64_t off = 0;
  for (int q = 0; q < W; ++q) {
    if (q != me && sc_[q] > 0) {
      fo[q] = pos;
      xo.push_back(off);
      nn.push_back(sc_[q]);
      fof.push_back(pos);
      seg_peer.push_back(q);
      pos += maxframe_of(sc_[q]);
    }
    off += sc_[q];
  }
  if (!d1 && (flags & kCheckCounts)) {
    std::vector<uint64_t> o(W), in;
    for (int q = 0; q < W; ++q) o[q] = (uint64_t)sc_[q];
    if ((rc0 = t_sizes(c, o, 1, in, st, "count"))) return rc0;
    for (int p = 0; p < W; ++p)
      if (p != me && (int64_t)in[p] != rc[p]) {
        const int64_t got = in[p] ? static_of((int64_t)in[p]) : 0;
        const int64_t want = rc[p] ? static_of(rc[p]) : 0;
        return c->fail(kStatusProtocol, "static section from rank " + std::to_string(p) + " is " +
                                            std::to_string(got) + " bytes, expected " +
                                            std::to_string(want), p);
      }
  }
  cudaError_t ce = c->sendbuf.need(pos + 128, st);
  if (ce != cudaSuccess) return (int)ce;
  uint8_t* sb = c->sendbuf.as<uint8_t>();
  if ((rc0 = encode_segments(c, x, xo, nn, fof, sb, book, s.flen, st))) return rc0;
  if (!nn.empty())
    cudaMemcpyAsync(c->pinned + 192, s.flen, 8 * nn.size(), cudaMemcpyDeviceToHost, st);
  if ((ce = cudaStreamSynchronize(st)) != cudaSuccess) return (int)ce;
  std::vector<int64_t> flen(W, 0);
  for (size_t i = 0; i < seg_peer.size(); ++i) flen[seg_peer[i]] = (int64_t)c->pinned[192 + i];
  R.stat.assign(W, nullptr);
  R.dyn.assign(W, nullptr);
  R.dyn_len.assign(W, 0);
  if (d1) {
    // metadata: (count, frame bytes) per peer, 16 B (collectives.py:255-266)
    std::vector<uint64_t> o(2 * W), in;
    for (int q = 0; q < W; ++q) { o[2 * q] = (uint64_t)sc_[q]; o[2 * q + 1] = (uint64_t)flen[q]; }
    if ((rc0 = t_sizes(c, o, 2, in, st, "metadata"))) return rc0;
    std::vector<int64_t> got(W, 0), roff(W + 1, 0);
    for (int p = 0; p < W; ++p) {
      if (p == me) continue;
      if ((int64_t)in[2 * p] != rc[p])
        return c->fail(kStatusProtocol, "rank " + std::to_string(p) + " will send " +
                                            std::to_string(in[2 * p]) + " elements, rank " +
                                            std::to_string(me) + " expected " +
                                            std::to_string(rc[p]), p);
      got[p] = (int64_t)in[2 * p + 1];
      if (rc[p] == 0 && got[p])
        return c->fail(kStatusCollective, "expected an empty frame, got " +
                                              std::to_string(got[p]) + " bytes", p);
      if (rc[p] > 0 && (got[p] < static_of(rc[p]) || got[p] % 128))
        return c->fail(kStatusCollective, "frame length " + std::to_string(got[p]) +
                                              " cannot hold " + std::to_string(rc[p]) +
                                              " elements", p);
    }
    for (int p = 0; p < W; ++p) roff[p + 1] = roff[p] + got[p];
    if ((ce = c->recvbuf.need(roff[W] + 128, st)) != cudaSuccess) return (int)ce;
    uint8_t* rb = c->recvbuf.as<uint8_t>();
    std::vector<Msg> sends, recvs;
    for (int p = 0; p < W; ++p) {
      if (p == me) continue;
      if (flen[p]) sends.push_back({p, sb + fo[p], flen[p]});
      if (got[p]) recvs.push_back({p, rb + roff[p], got[p]});
      R.stat[p] = rb + roff[p];
      R.dyn_len[p] = rc[p] ? got[p] - static_of(rc[p]) : 0;
    }
    c->host_bytes += (uint64_t)[&] { int64_t t = 0; for (auto v : flen) t += v; return t; }();
    c->host_msgs += (uint64_t)(W - 1);
    return t_exchange(c, sends, recvs, st, "frame");
  }
  // design 2: statics pre-sized from recv_counts, no metadata first
  std::vector<int64_t> sin(W, 0), soff(W + 1, 0);
  for (int p = 0; p < W; ++p) sin[p] = (p != me && rc[p] > 0) ? static_of(rc[p]) : 0;
  for (int p = 0; p < W; ++p) soff[p + 1] = soff[p] + sin[p];
  std::vector<Msg> sends, recvs;
  for (int p = 0; p < W; ++p) {
    if (p == me) continue;
    if (flen[p]) sends.push_back({p, sb + fo[p], static_of(sc_[p])});
    if (sin[p]) recvs.push_back({p, nullptr, sin[p]});
  }
  // the receive buffer holds statics then dynamics; sized for the statics now
  int64_t dyn_cap_guess = 0;
  for (int p = 0; p < W; ++p) dyn_cap_guess += (p != me && rc[p] > 0) ? pad128h(rc[p]) : 0;
  if ((ce = c->recvbuf.need(soff[W] + dyn_cap_guess + 256, st)) != cudaSuccess) return (int)ce;
  uint8_t* rb = c->recvbuf.as<uint8_t>();
  for (auto& m : recvs) m.ptr = rb + soff[m.peer];
  int64_t sent = 0;
  for (int p = 0; p < W; ++p)
    if (p != me && flen[p]) sent += static_of(sc_[p]);
  if ((rc0 = t_exchange(c, sends, recvs, st, "static section"))) return rc0;
  std::vector<uint64_t> o(W, 0), in;
  for (int q = 0; q < W; ++q) o[q] = (q != me && flen[q]) ? (uint64_t)(flen[q] - static_of(sc_[q])) : 0;
  if ((rc0 = t_sizes(c, o, 1, in, st, "dynamic size"))) return rc0;
  std::vector<int64_t> doff(W + 1, 0);
  for (int p = 0; p < W; ++p) {
    const int64_t d = (p != me && rc[p] > 0) ? (int64_t)in[p] : 0;
    if (d % 128)
      return c->fail(kStatusCollective, "dynamic section of " + std::to_string(d) +
                                            " bytes is not 128-aligned", p);
    if (d > pad128h(rc[p]) + 128)
      return c->fail(kStatusCollective, "dynamic section of " + std::to_string(d) +
                                            " bytes exceeds the frame bound", p);
    doff[p + 1] = doff[p] + d;
  }
  std::vector<Msg> ds, dr;
  for (int p = 0; p < W; ++p) {
    if (p == me) continue;
    if (o[p]) ds.push_back({p, sb + fo[p] + static_of(sc_[p]), (int64_t)o[p]});
    const int64_t d = doff[p + 1] - doff[p];
    if (d) dr.push_back({p, rb + soff[W] + doff[p], d});
    sent += (int64_t)o[p];
    R.stat[p] = rb + soff[p];
    R.dyn[p] = d ? rb + soff[W] + doff[p] : rb + soff[p];
    R.dyn_len[p] = d;
  }
  c->host_bytes += (uint64_t)sent;
  c->host_msgs += (uint64_t)2 * (W - 1);
  return t_exchange(c, ds, dr, st, "dynamic section");
}

int msg_alltoall(zc_comm* c, const uint16_t* x, const int64_t* sc_, const int64_t* rc,
                 uint16_t* out, const uint8_t* book, int32_t* err, int flags, cudaStream_t st) {
  const int W = c->world, me = c->rank;
  if (err) init_err_kernel<<<1, 64, 0, st>>>(err, W);
  Recv R;
  int rc0 = msg_a2a_exchange(c, x, sc_, rc, book, flags, st, R);
  if (rc0) return rc0;
  std::vector<int> ranks;
  std::vector<const uint8_t*> stp, dyn;
  std::vector<int64_t> dl, cn, oo;
  int64_t xoff = 0, ooff = 0;
  for (int p = 0; p < W; ++p) {
    if (p == me) {
      if (sc_[p])
        cudaMemcpyAsync(out + ooff, x + xoff, sizeof(uint16_t) * sc_[p], cudaMemcpyDeviceToDevice, st);
    } else if (rc[p] > 0) {
      ranks.push_back(p);
      stp.push_back(R.stat[p]);
      dyn.push_back(R.dyn[p]);
      dl.push_back(R.dyn_len[p]);
      cn.push_back(rc[p]);
      oo.push_back(ooff);
    }
    xoff += sc_[p];
    ooff += (p == me) ? sc_[p] : rc[p];
  }
  return decode_local(c, ranks, stp, dyn, dl, cn, oo, out, err, scratch_of(c).seg_err, st);
}

int reduce_from(zc_comm* c, const std::vector<RedSrc>& src, int64_t shard, void* out, int f32,
                int32_t* err, cudaStream_t st) {
  const int W = c->world;
  cudaError_t ce = c->srcs.need((int64_t)(sizeof(RedSrc) + 64) * W + 4096, st);
  if (ce != cudaSuccess) return (int)ce;
  RedSrc* sd = c->srcs.as<RedSrc>();
  void* hdr = c->srcs.as<uint8_t>() + sizeof(RedSrc) * W + 256;
  if ((ce = store_srcs(src.data(), W, sd, st)) != cudaSuccess) return (int)ce;
  int32_t* e_out = err ? err : scratch_of(c).seg_err;
  return cuda_status(launch_reduce(sd, hdr, W, shard, out, f32, e_out, 0, 0, st));
}

int msg_reduce_scatter(zc_comm* c, const uint16_t* x, int64_t shard, void* out, int f32,
                       const uint8_t* book, int32_t* err, int flags, cudaStream_t st) {
  const int W = c->world, me = c->rank;
  std::vector<int64_t> cnt(W, shard);
  Recv R;
  int rc0 = msg_a2a_exchange(c, x, cnt.data(), cnt.data(), book, flags, st, R);
  if (rc0) return rc0;
  std::vector<RedSrc> src(W);
  for (int p = 0; p < W; ++p) {
    RedSrc r{};
    if (p == me) {
      r.stat = reinterpret_cast<const uint8_t*>(x + (int64_t)me * shard);
      r.raw = 1;
    } else {
      r.stat = R.stat[p];
      r.dyn = R.dyn[p];
      r.dyn_len = R.dyn_len[p];
    }
    src[p] = r;
  }
  return reduce_from(c, src, shard, out, f32, err, st);
}

// ---- raw twins --------------------------------------------------------------------

int raw_alltoall_into(zc_comm* c, const uint16_t* x, const int64_t* sc_, const int64_t* rc,
                      uint16_t* out, int flags, cudaStream_t st) {
  const int W = c->world, me = c->rank;
  if (flags & kCheckCounts) {
    std::vector<uint64_t> o(W), in;
    for (int q = 0; q < W; ++q) o[q] = (uint64_t)sc_[q];
    int rc0 = t_sizes(c, o, 1, in, st, "count");
    if (rc0) return rc0;
    for (int p = 0; p < W; ++p)
      if (p != me && (int64_t)in[p] != rc[p])
        return c->fail(kStatusProtocol, "rank " + std::to_string(p) + " will send " +
                                            std::to_string(in[p]) + " elements, rank " +
                                            std::to_string(me) + " expected " +
                                            std::to_string(rc[p]), p);
  }
  std::vector<Msg> sends, recvs;
  int64_t xoff = 0, ooff = 0, sent = 0;
  for (int p = 0; p < W; ++p) {
    if (p == me) {
      if (sc_[p])
        cudaMemcpyAsync(out + ooff, x + xoff, sizeof(uint16_t) * sc_[p], cudaMemcpyDeviceToDevice, st);
    } else {
      if (sc_[p]) sends.push_back({p, x + xoff, 2 * sc_[p]});
      if (rc[p]) recvs.push_back({p, out + ooff, 2 * rc[p]});
      sent += 2 * sc_[p];
    }
    xoff += sc_[p];
    ooff += (p == me) ? sc_[p] : rc[p];
  }
  c->host_bytes += (uint64_t)sent;
  c->host_msgs += (uint64_t)(W - 1);
  return t_exchange(c, sends, recvs, st, "message");
}

// ---- symmetric workspace ------------------------------------------------------------

int p2p_setup(zc_comm* c, int64_t slot_bytes, cudaStream_t st);

// Collective growth: every rank calls it in the same call (the trigger is a
// function of arguments equal on every rank).  Quiesce (local stream, then
// every rank) so nobody still reads the old buffers, then re-create.
int p2p_grow(zc_comm* c, int64_t need, cudaStream_t st) {
  int rc = need_small(c, st);
  if (rc) return rc;
  uint64_t* v = c->small.as<uint64_t>() + 768;
  cudaMemcpyAsync(v, &need, 8, cudaMemcpyHostToDevice, st);
  cudaStreamSynchronize(st);
  if ((rc = t_allgather(c, v, v + 1, 8, st))) return rc;
  cudaMemcpyAsync(c->pinned + 64, v + 1, 8 * c->world, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  int64_t mx = need;
  for (int p = 0; p < c->world; ++p) mx = std::max<int64_t>(mx, (int64_t)c->pinned[64 + p]);
  cudaDeviceSynchronize();
  return p2p_setup(c, std::max<int64_t>(mx, 2 * c->slot_bytes), st);
}

void p2p_teardown(zc_comm* c) {
  for (void* p : c->opened) cudaIpcCloseMemHandle(p);
  c->opened.clear();
  if (c->sym) cudaFree(c->sym);
  c->sym = nullptr;
  c->peer_sym.clear();
}

// (Re)creates the symmetric buffer and maps every peer's.  Collective.
int p2p_setup(zc_comm* c, int64_t slot_bytes, cudaStream_t st) {
  const int W = c->world;
  slot_bytes = (slot_bytes + (1 << 20) - 1) / (1 << 20) * (1 << 20);
  // every rank must be past its last use of the old buffers
  if (c->sym) {
    cudaDeviceSynchronize();
    uint64_t* v = c->small.as<uint64_t>() + 768;
    int rc = t_allgather(c, v, v + 1, 8, st);   // barrier
    if (rc) return rc;
    cudaStreamSynchronize(st);
    p2p_teardown(c);
  }
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&c->sym), (size_t)(kFlagBytes + 2 * slot_bytes));
  if (e != cudaSuccess) { c->sym = nullptr; return (int)e; }
  cudaMemset(c->sym, 0, (size_t)kFlagBytes);
  cudaDeviceSynchronize();
  c->slot_bytes = slot_bytes;
  c->epoch = 0;
  c->peer_sym.assign(W, nullptr);
  c->peer_sym[c->rank] = c->sym;
  int ok = 1;
  if (c->hub) {
    struct P { uint8_t* base; int dev; } mine{c->sym, c->device};
    std::vector<const void*> all;
    if (!c->hub->exchange(c->rank, &mine, all)) return c->fail(kStatusTransport, "rendezvous timed out");
    c->shared_device = false;
    for (int p = 0; p < W; ++p) {
      const P* q = reinterpret_cast<const P*>(all[p]);
      c->peer_sym[p] = q->base;
      if (p != c->rank && q->dev == c->device) c->shared_device = true;
      if (p != c->rank && q->dev != c->device) {
        cudaError_t pe = cudaDeviceEnablePeerAccess(q->dev, 0);
        if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) ok = 0;
        cudaGetLastError();
      }
    }
    std::vector<const void*> again;
    if (!c->hub->exchange(c->rank, &mine, again)) return c->fail(kStatusTransport, "rendezvous timed out");
  } else if (W > 1) {
    // IPC handles all-gathered over NCCL
    cudaIpcMemHandle_t h;
    e = cudaIpcGetMemHandle(&h, c->sym);
    if (e != cudaSuccess) { ok = 0; cudaGetLastError(); memset(&h, 0, sizeof(h)); }
    const int hb = (int)sizeof(cudaIpcMemHandle_t);
    cudaError_t ce = c->small.need(8192 + 4096 + (int64_t)(W + 1) * hb + 256, st);
    if (ce != cudaSuccess) return (int)ce;
    uint8_t* d = c->small.as<uint8_t>() + 12288;
    cudaMemcpyAsync(d, &h, hb, cudaMemcpyHostToDevice, st);
    int rc = t_allgather(c, d, d + hb, hb, st);
    if (rc) return rc;
    std::vector<uint8_t> all((size_t)W * hb);
    cudaMemcpyAsync(all.data(), d + hb, (size_t)W * hb, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    for (int p = 0; p < W && ok; ++p) {
      if (p == c->rank) continue;
      cudaIpcMemHandle_t ph;
      memcpy(&ph, all.data() + (size_t)p * hb, hb);
      void* ptr = nullptr;
      cudaError_t oe = cudaIpcOpenMemHandle(&ptr, ph, cudaIpcMemLazyEnablePeerAccess);
      if (oe != cudaSuccess) { ok = 0; cudaGetLastError(); break; }
      c->opened.push_back(ptr);
      c->peer_sym[p] = reinterpret_cast<uint8_t*>(ptr);
    }
    // every rank must have mapped every peer
    uint64_t* v = c->small.as<uint64_t>() + 768;
    const uint64_t okv = (uint64_t)ok;
    cudaMemcpyAsync(v, &okv, 8, cudaMemcpyHostToDevice, st);
    if ((rc = t_allgather(c, v, v + 1, 8, st))) return rc;
    cudaMemcpyAsync(c->pinned + 64, v + 1, 8 * W, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    for (int p = 0; p < W; ++p) ok &= (int)(c->pinned[64 + p] & 1);
  }
  c->p2p = ok && W <= kMaxSegments;
  return 0;
}

}  // namespace

// ============================================================================
// C-ABI
extern "C" {

int zc_nccl_id_bytes(void) { return (int)sizeof(ncclUniqueId); }

int zc_nccl_get_id(void* id_out) {
  if (!id_out) return kStatusBadArg;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return kStatusTransport;
  memcpy(id_out, &id, sizeof(id));
  return 0;
}

static int comm_common_init(zc_comm* c, int64_t slot_bytes) {
  cudaGetDevice(&c->device);
  // every kernel a collective may launch is loaded before any rank can spin
  preload_encode();
  preload_decode();
  preload_stats();
  preload_reduce();
  preload_estimate();
  preload_small();
  {
    cudaFuncAttributes a;
    const void* ks[] = {(const void*)publish_kernel, (const void*)wait_flags_kernel,
                        (const void*)finish_kernel, (const void*)init_err_kernel,
                        (const void*)map_err_kernel, (const void*)pack_size_kernel};
    for (const void* k : ks) cudaFuncGetAttributes(&a, k);
  }
  cudaEventCreateWithFlags(&c->ev_post, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_copied, cudaEventDisableTiming);
  cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking);
  cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&c->pinned), 8 * 512);
  if (e != cudaSuccess) return (int)e;
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  int rc = need_small(c, st);
  if (!rc) rc = p2p_setup(c, slot_bytes > 0 ? slot_bytes : (int64_t)1 << 28, st);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  return rc;
}

int zc_comm_init(zc_comm** out, const void* nccl_id, int rank, int world, int64_t slot_bytes,
                 int flags) {
  if (!out || !nccl_id || world < 1 || rank < 0 || rank >= world) return kStatusBadArg;
  zc_comm* c = new zc_comm();
  c->rank = rank;
  c->world = world;
  ncclUniqueId id;
  memcpy(&id, nccl_id, sizeof(id));
  if (ncclCommInitRank(&c->nccl, world, id, rank) != ncclSuccess) {
    delete c;
    return kStatusTransport;
  }
  int rc = comm_common_init(c, slot_bytes);
  if (flags & 1) c->p2p = false;   // ZC_COMM_NO_P2P
  *out = c;
  return rc;
}

// `world` communicators for in-process ranks (one host thread each);
// comms[i] is rank i on devices[i] (or the current device when null).  The
// caller's threads then drive them concurrently, like NCCL ranks.
int zc_comm_init_local(zc_comm** comms, int world, const int* devices, int64_t slot_bytes,
                       int flags) {
  if (!comms || world < 1 || world > kMaxSegments) return kStatusBadArg;
  auto hub = std::make_shared<Hub>(world);
  int cur = 0;
  cudaGetDevice(&cur);
  std::vector<zc_comm*> cs(world);
  for (int r = 0; r < world; ++r) {
    zc_comm* c = new zc_comm();
    c->rank = r;
    c->world = world;
    c->hub = hub;
    cs[r] = c;
    comms[r] = c;
  }
  // setup is collective over the hub: one thread per rank
  std::vector<int> rcs(world, 0);
  std::vector<std::thread*> th;
  for (int r = 0; r < world; ++r) {
    th.push_back(new std::thread([&, r] {
      cudaSetDevice(devices ? devices[r] : cur);
      rcs[r] = comm_common_init(cs[r], slot_bytes);
      if (flags & 1) cs[r]->p2p = false;
    }));
  }
  for (auto* t : th) { t->join(); delete t; }
  cudaSetDevice(cur);
  for (int r = 0; r < world; ++r)
    if (rcs[r]) return rcs[r];
  return 0;
}

int zc_comm_destroy(zc_comm* c) {
  if (!c) return 0;
  cudaDeviceSynchronize();
  p2p_teardown(c);
  c->ws.release(); c->sendbuf.release(); c->recvbuf.release(); c->small.release(); c->srcs.release();
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->ev_post) cudaEventDestroy(c->ev_post);
  if (c->ev_copied) cudaEventDestroy(c->ev_copied);
  for (auto ev : c->step_ev) cudaEventDestroy(ev);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->nccl) ncclCommDestroy(c->nccl);
  delete c;
  return 0;
}

int zc_comm_abort(zc_comm* c) {
  if (c && c->hub) c->hub->abort();
  return 0;
}

int zc_comm_info(zc_comm* c, int* info) {
  if (!c || !info) return kStatusBadArg;
  info[0] = c->rank;
  info[1] = c->world;
  info[2] = c->p2p ? 1 : 0;
  info[3] = c->shared_device ? 1 : 0;
  info[4] = c->nccl ? 1 : 0;
  return 0;
}

const char* zc_comm_last_error(zc_comm* c, int* peer) {
  if (!c) return "null communicator";
  if (peer) *peer = c->last_peer;
  return c->last_error.c_str();
}

int zc_comm_stats(zc_comm* c, uint64_t* bytes_sent, uint64_t* messages) {
  if (!c) return kStatusBadArg;
  uint64_t d[2] = {0, 0};
  if (c->sym) {
    cudaDeviceSynchronize();
    cudaMemcpy(d, c->dstats(), 16, cudaMemcpyDeviceToHost);
  }
  if (bytes_sent) *bytes_sent = c->host_bytes + d[0];
  if (messages) *messages = c->host_msgs + d[1];
  return 0;
}

int zc_comm_reserve(zc_comm* c, int64_t slot_bytes, void* stream) {
  if (!c) return kStatusBadArg;
  if (slot_bytes <= c->slot_bytes) return 0;
  return p2p_grow(c, slot_bytes, reinterpret_cast<cudaStream_t>(stream));
}

// The peer-memory plane is the default when the communicator has it
// (ZC_PLANE_P2P only names it); ZC_PLANE_MSG forces the message plane.
static bool use_p2p(zc_comm* c, int flags) {
  if (flags & kPlaneMsg) return false;
  return c->p2p;
}

int zc_allgather(zc_comm* c, const uint16_t* x, int64_t n, uint16_t* out, const uint8_t* book_dev,
                 int32_t* err_dev, int flags, void* stream) {
  Range nvtx_range("zc_allgather");
  if (!c || n < 1 || !x || !out) return kStatusBadArg;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  c->last_error.clear();
  c->last_peer = -1;
  if (c->world == 1) {
    if (err_dev) init_err_kernel<<<1, 64, 0, st>>>(err_dev, 1);
    return cuda_status(cudaMemcpyAsync(out, x, sizeof(uint16_t) * n, cudaMemcpyDeviceToDevice, st));
  }
  if (use_p2p(c, flags)) return p2p_allgather(c, x, n, out, book_dev, err_dev, st);
  return msg_allgather(c, x, n, out, book_dev, err_dev, flags, st);
}

int zc_allgather_raw(zc_comm* c, const uint16_t* x, int64_t n, uint16_t* out, void* stream) {
  Range nvtx_range("zc_allgather_raw");
  if (!c || n < 0 || (n && (!x || !out))) return kStatusBadArg;
  c->host_bytes += (uint64_t)(2 * n) * (c->world - 1);
  c->host_msgs += (uint64_t)(c->world - 1);
  return t_allgather(c, x, out, 2 * n, reinterpret_cast<cudaStream_t>(stream));
}

int zc_alltoall(zc_comm* c, const uint16_t* x, const int64_t* send_counts,
                const int64_t* recv_counts, uint16_t* out, const uint8_t* book_dev,
                int32_t* err_dev, int flags, void* stream) {
  Range nvtx_range("zc_alltoall");
  if (!c || !send_counts || !recv_counts) return kStatusBadArg;
  for (int p = 0; p < c->world; ++p)
    if (send_counts[p] < 0 || recv_counts[p] < 0) return kStatusBadArg;
  if (send_counts[c->rank] != recv_counts[c->rank]) return kStatusBadArg;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  c->last_error.clear();
  c->last_peer = -1;
  if (c->world == 1) {
    if (err_dev) init_err_kernel<<<1, 64, 0, st>>>(err_dev, 1);
    if (send_counts[0])
      cudaMemcpyAsync(out, x, sizeof(uint16_t) * send_counts[0], cudaMemcpyDeviceToDevice, st);
    return cuda_status(cudaGetLastError());
  }
  if (use_p2p(c, flags) && !(flags & kA2AD1))
    return p2p_alltoall(c, x, send_counts, recv_counts, out, book_dev, err_dev, st);
  return msg_alltoall(c, x, send_counts, recv_counts, out, book_dev, err_dev, flags, st);
}

int zc_alltoall_raw(zc_comm* c, const uint16_t* x, const int64_t* send_counts,
                    const int64_t* recv_counts, uint16_t* out, int flags, void* stream) {
  Range nvtx_range("zc_alltoall_raw");
  if (!c || !send_counts || !recv_counts) return kStatusBadArg;
  if (send_counts[c->rank] != recv_counts[c->rank]) return kStatusBadArg;
  c->last_error.clear();
  return raw_alltoall_into(c, x, send_counts, recv_counts, out, flags,
                           reinterpret_cast<cudaStream_t>(stream));
}

int zc_reduce_scatter(zc_comm* c, const uint16_t* x, int64_t shard, void* out, int out_f32,
                      const uint8_t* book_dev, int32_t* err_dev, int flags, void* stream) {
  Range nvtx_range("zc_reduce_scatter");
  if (!c || shard < 1 || !x || !out) return kStatusBadArg;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  c->last_error.clear();
  c->last_peer = -1;
  if (c->world == 1) {
    std::vector<RedSrc> src(1);
    src[0].stat = reinterpret_cast<const uint8_t*>(x);
    src[0].raw = 1;
    return reduce_from(c, src, shard, out, out_f32, err_dev, st);
  }
  if (use_p2p(c, flags) && !(flags & kA2AD1))
    return p2p_reduce_scatter(c, x, shard, out, out_f32, book_dev, err_dev, st);
  return msg_reduce_scatter(c, x, shard, out, out_f32, book_dev, err_dev, flags, st);
}

int zc_reduce_scatter_raw(zc_comm* c, const uint16_t* x, int64_t shard, void* out, int out_f32,
                          int32_t* err_dev, void* stream) {
  Range nvtx_range("zc_reduce_scatter_raw");
  if (!c || shard < 1 || !x || !out) return kStatusBadArg;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int W = c->world, me = c->rank;
  c->last_error.clear();
  cudaError_t ce = c->recvbuf.need(2 * shard * W + 256, st);
  if (ce != cudaSuccess) return (int)ce;
  uint16_t* rb = c->recvbuf.as<uint16_t>();
  std::vector<int64_t> cnt(W, shard);
  // rank-order contributions: rb[p * shard ..] = rank p's shard `me`
  std::vector<int64_t> sc2(W, shard);
  int rc = 0;
  if (W > 1) {
    rc = raw_alltoall_into(c, x, sc2.data(), cnt.data(), rb, 0, st);
    if (rc) return rc;
  }
  std::vector<RedSrc> src(W);
  for (int p = 0; p < W; ++p) {
    src[p].stat = reinterpret_cast<const uint8_t*>(p == me ? x + (int64_t)me * shard
                                                           : rb + (int64_t)p * shard);
    src[p].raw = 1;
  }
  return reduce_from(c, src, shard, out, out_f32, err_dev, st);
}

// Fused decode + fp32 reduction over arbitrary sources (the generic
// reduce-scatter of the Python layer; W unbounded): src_dev is a device
// array of W RedSrc-compatible records (see zc_red_src_bytes), hdr_scratch
// >= zc_reduce_scratch_bytes(W) bytes of device memory.
int zc_reduce_frames(const void* src_dev, int W, int64_t n, void* out, int out_f32,
                     void* hdr_scratch, int32_t* err_dev, void* stream) {
  if (!src_dev || W < 1 || n < 0 || !out || !hdr_scratch || !err_dev) return kStatusBadArg;
  return cuda_status(launch_reduce(reinterpret_cast<const RedSrc*>(src_dev), hdr_scratch, W, n, out,
                                   out_f32, err_dev, 0, 0, reinterpret_cast<cudaStream_t>(stream)));
}

int64_t zc_reduce_scratch_bytes(int W) { return (int64_t)reduce_hdr_bytes(W); }
int zc_red_src_bytes(void) { return (int)sizeof(RedSrc); }

}  // extern "C"
