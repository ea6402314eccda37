// Peer memory plumbing for the pull-decode collectives over NVLink.
//
// Each rank exports its symmetric workspace (frames + flag array) with a CUDA
// IPC handle; peers map it and decode frames straight out of the owner's HBM
// (K5 fused pull-decode).  Readiness is signalled device-side: the owner
// writes `epoch` into its slot of every peer's flag array with a system-scope
// release store after its encode kernel; a consumer kernel waits with
// system-scope acquire loads (bounded by %globaltimer) before decoding.
// This replaces the reference's send/recv transport seam
// (transport.Communicator, transport.py:559-623) for the data path.
#include <cstring>
#include "zc_common.cuh"

namespace zc {

struct PeerPtrs {
  uint64_t* flags[kMaxSegments];
};

__global__ void signal_kernel(PeerPtrs peers, int world, int me, uint64_t epoch) {
  const int p = threadIdx.x;
  __threadfence_system();
  if (p < world && p != me) st_release_sys_u64(peers.flags[p] + me, epoch);
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void wait_kernel(const uint64_t* flags, int world, int me, uint64_t epoch,
                            int64_t timeout_ns, int32_t* err) {
  const int p = threadIdx.x;
  if (p >= world || p == me) return;
  const uint64_t t0 = globaltimer();
  while (ld_acquire_sys_u64(flags + p) < epoch) {
    if (timeout_ns > 0 && (int64_t)(globaltimer() - t0) > timeout_ns) {
      if (err) atomicMin(err, (int32_t)kErrTimeout);
      return;
    }
    __nanosleep(200);
  }
}

}  // namespace zc

using namespace zc;

extern "C" {

int zc_ipc_handle_bytes(void) { return (int)sizeof(cudaIpcMemHandle_t); }

int zc_ipc_get_handle(void* dev_ptr, void* handle_out) {
  if (!dev_ptr || !handle_out) return -1;
  cudaError_t e = cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handle_out), dev_ptr);
  return e == cudaSuccess ? 0 : (int)e;
}

int zc_ipc_open_handle(const void* handle, void** dev_ptr_out) {
  if (!handle || !dev_ptr_out) return -1;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? 0 : (int)e;
}

int zc_ipc_close_handle(void* dev_ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  return e == cudaSuccess ? 0 : (int)e;
}

int zc_alloc(int64_t bytes, void** dev_ptr_out) {
  if (bytes <= 0 || !dev_ptr_out) return -1;
  cudaError_t e = cudaMalloc(dev_ptr_out, (size_t)bytes);
  if (e != cudaSuccess) return (int)e;
  e = cudaMemset(*dev_ptr_out, 0, (size_t)bytes);
  return e == cudaSuccess ? 0 : (int)e;
}

int zc_free(void* dev_ptr) {
  cudaError_t e = cudaFree(dev_ptr);
  return e == cudaSuccess ? 0 : (int)e;
}

int zc_signal_peers(void* const* peer_flags, int world, int my_rank, uint64_t epoch,
                    void* stream) {
  if (world < 1 || world > kMaxSegments || !peer_flags) return -1;
  PeerPtrs p{};
  for (int i = 0; i < world; ++i) p.flags[i] = reinterpret_cast<uint64_t*>(peer_flags[i]);
  signal_kernel<<<1, 64, 0, reinterpret_cast<cudaStream_t>(stream)>>>(p, world, my_rank, epoch);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

int zc_wait_signals(const void* flags, int world, int my_rank, uint64_t epoch, int64_t timeout_ns,
                    int32_t* err_dev, void* stream) {
  if (world < 1 || world > kMaxSegments || !flags) return -1;
  wait_kernel<<<1, 64, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const uint64_t*>(flags), world, my_rank, epoch, timeout_ns, err_dev);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

}  // extern "C"
