// Micro-benchmark: the decoder's TMA-ring read side (sm + 3 planes + a few
// escape bytes per 4096-element tile, ~5.7 KB) with different output-store
// schemes for the 8 KB of words per tile.  Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2604_27844_b200/csrc
//        scripts/exp/store_ring.cu -o scripts/exp/store_ring
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "zc_common.cuh"

using namespace zc;

#ifndef RT
#define RT 4096
#endif
#ifndef RST
#define RST 4
#endif
constexpr int kSt = RST;
constexpr int kRT = RT;                              // elements per ring tile
struct __align__(128) Stage {
  uint8_t sm[kRT];
  uint8_t pl[3][kRT / 8];
  uint8_t esc[128];
};

__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(ssrc)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int V>
__global__ void __launch_bounds__(288) ring(const uint8_t* __restrict__ sm, const uint8_t* __restrict__ pl,
                                            uint16_t* __restrict__ out, int64_t ntiles, int64_t per) {
  extern __shared__ __align__(128) uint8_t s_dyn[];
  Stage* S = reinterpret_cast<Stage*>(s_dyn);
  uint64_t* full = reinterpret_cast<uint64_t*>(s_dyn + kSt * sizeof(Stage));
  uint64_t* empty = full + kSt;
  uint8_t* obuf = reinterpret_cast<uint8_t*>(empty + kSt) + 64;   // 8 warps x 2 x 1 KB (V>=2)
  obuf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(obuf) + 127) & ~uintptr_t(127));
  const int tid = threadIdx.x;
  const int64_t t0 = blockIdx.x * per;
  int64_t t1 = t0 + per;
  if (t1 > ntiles) t1 = ntiles;
  if (tid == 0) {
    for (int i = 0; i < kSt; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 8); }
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t n = ntiles * kRT;
  if (tid < 32) {
    if (tid == 0) {
      for (int64_t t = t0; t < t1; ++t) {
        const int64_t k = t - t0;
        const int st = (int)(k % kSt);
        if (k >= kSt) mbar_wait(empty + st, (uint32_t)(((k / kSt) - 1) & 1));
        mbar_arrive_expect_tx(full + st, kRT + 3 * (kRT / 8) + 96);
        tma_load_1d(S[st].sm, sm + t * kRT, kRT, full + st);
        for (int b = 0; b < 3; ++b)
          tma_load_1d(S[st].pl[b], pl + b * (n / 8) + t * (kRT / 8), kRT / 8, full + st);
        tma_load_1d(S[st].esc, sm + ((t * 96) % (n - 128)) / 16 * 16, 96, full + st);
      }
    }
    return;
  }
  const int ct = tid - 32, lane = ct & 31, warp = ct >> 5;
  uint8_t* wb = obuf + warp * 2048;
  for (int64_t t = t0; t < t1; ++t) {
    const int64_t k = t - t0;
    const int st = (int)(k % kSt);
    mbar_wait_warp(full + st, (uint32_t)((k / kSt) & 1));
    if (kRT == 8192) {   // 32 elements per thread: two 16-B sm loads, 64 B out
      const uint4 s0 = *reinterpret_cast<const uint4*>(S[st].sm + ct * 32);
      const uint4 s1 = *reinterpret_cast<const uint4*>(S[st].sm + ct * 32 + 16);
      const uint32_t q0 = *reinterpret_cast<const uint32_t*>(S[st].pl[0] + ct * 4);
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + st);
      uint8_t* ob = reinterpret_cast<uint8_t*>(out) + t * (2 * kRT) + ct * 64;
      const uint4 a = make_uint4(s0.x ^ q0, s0.y, s0.z, s0.w), b = make_uint4(s1.x, s1.y ^ q0, s1.z, s1.w);
      asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(ob),
                   "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w) : "memory");
      asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(ob + 32),
                   "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w), "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w) : "memory");
      continue;
    }
    const uint4 sv = *reinterpret_cast<const uint4*>(S[st].sm + ct * 16);
    const uint32_t p0 = *reinterpret_cast<const uint16_t*>(S[st].pl[0] + ct * 2);
    const uint32_t p1 = *reinterpret_cast<const uint16_t*>(S[st].pl[1] + ct * 2);
    const uint32_t p2 = *reinterpret_cast<const uint16_t*>(S[st].pl[2] + ct * 2);
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + st);
    const uint32_t m = p0 ^ p1 ^ p2;
    const uint4 a = make_uint4(sv.x ^ m, sv.y, sv.z, sv.w);
    const uint4 b = make_uint4(sv.w, sv.z ^ m, sv.y, sv.x);
    uint8_t* ob = reinterpret_cast<uint8_t*>(out) + t * (2 * kTile);
    if (V == 0) {          // current decoder: lane owns 32 contiguous bytes
      *reinterpret_cast<uint4*>(ob + ct * 32) = a;
      *reinterpret_cast<uint4*>(ob + ct * 32 + 16) = b;
    } else if (V == 1) {   // coalesced (ceiling; wrong order, same bytes)
      *reinterpret_cast<uint4*>(ob + warp * 1024 + lane * 16) = a;
      *reinterpret_cast<uint4*>(ob + warp * 1024 + 512 + lane * 16) = b;
    } else if (V == 2) {   // per-warp smem + 1 KB bulk store, double buffered
      uint8_t* buf = wb + (k & 1) * 1024;
      if (lane == 0) bulk_wait_read<1>();
      __syncwarp();
      *reinterpret_cast<uint4*>(buf + lane * 32) = a;
      *reinterpret_cast<uint4*>(buf + lane * 32 + 16) = b;
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) { bulk_store(ob + warp * 1024, buf, 1024); bulk_commit(); }
    } else if (V == 3) {   // per-warp smem transpose, coalesced STG
      uint8_t* buf = wb;
      *reinterpret_cast<uint4*>(buf + lane * 32) = a;
      *reinterpret_cast<uint4*>(buf + lane * 32 + 16) = b;
      __syncwarp();
      const uint4 c = *reinterpret_cast<const uint4*>(buf + lane * 16);
      const uint4 d = *reinterpret_cast<const uint4*>(buf + 512 + lane * 16);
      __syncwarp();
      *reinterpret_cast<uint4*>(ob + warp * 1024 + lane * 16) = c;
      *reinterpret_cast<uint4*>(ob + warp * 1024 + 512 + lane * 16) = d;
    } else if (V == 4) {   // streaming (evict-first) stores, lane-owned 32 B
      __stcs(reinterpret_cast<uint4*>(ob + ct * 32), a);
      __stcs(reinterpret_cast<uint4*>(ob + ct * 32 + 16), b);
    } else if (V == 5) {   // one 32-B vector store (sm_100 st.global.v8.b32)
      asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(ob + ct * 32),
                   "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
                   : "memory");
    }
  }
  if (V == 2 && lane == 0) bulk_wait_all();
}

template <int V>
float run(const uint8_t* sm, const uint8_t* pl, uint16_t* out, int64_t ntiles, int ctas_per_sm) {
  size_t dyn = kSt * sizeof(Stage) + 2 * kSt * 8 + 64 + 128 + 8 * 2048;
  cudaFuncSetAttribute(ring<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ring<V>, 288, dyn);
  if (ctas_per_sm > occ) ctas_per_sm = occ;
  const int grid0 = 148 * ctas_per_sm;
  const int64_t per = (ntiles + grid0 - 1) / grid0;
  const int grid = (int)((ntiles + per - 1) / per);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) ring<V><<<grid, 288, dyn>>>(sm, pl, out, ntiles, per);
  cudaEventRecord(a);
  const int it = 20;
  for (int i = 0; i < it; ++i) ring<V><<<grid, 288, dyn>>>(sm, pl, out, ntiles, per);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
  const double bytes = (double)ntiles * (kRT + 3 * kRT / 8 + 96 + 2 * kRT);
  printf("V%d occ=%d ctas/sm=%d grid=%d: %.1f us  %.0f GB/s\n", V, occ, ctas_per_sm, grid,
         1e3 * ms / it, bytes / (ms / it * 1e-3) / 1e9);
  return ms / it;
}

int main() {
  const int64_t n = 218112000;
  const int64_t ntiles = n / kRT;
  uint8_t *sm, *pl;
  uint16_t* out;
  cudaMalloc(&sm, n);
  cudaMalloc(&pl, 3 * n / 8 + 4096);
  cudaMalloc(&out, 2 * n);
  cudaMemset(sm, 1, n);
  cudaMemset(pl, 2, 3 * n / 8);
  for (int c : {2, 3, 4}) run<5>(sm, pl, out, ntiles, c);
  return 0;
}
