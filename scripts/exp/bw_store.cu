// Store-path probe: write-only bandwidth vs threads per SM and store width,
// and a TMA bulk-store (smem -> global) variant.  436 MB written per launch.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void st128(uint4* out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(out + i, make_uint4((uint32_t)i, 1, 2, 3));
}
__global__ void st256(uint4* out, size_t n2) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t a = (uint32_t)i;
    asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(out + 2 * i), "r"(a) : "memory");
  }
}
// one warp per CTA slice: fill an 8 KB smem tile, bulk-store it, ring of 4
__global__ void sttma(uint8_t* out, size_t tiles) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int t = threadIdx.x;
  int slot = 0;
  for (size_t k = blockIdx.x; k < tiles; k += gridDim.x, slot = (slot + 1) & 3) {
    if (t == 0) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
    __syncthreads();
    uint4* s = reinterpret_cast<uint4*>(sm + slot * 8192);
    for (int i = t; i < 512; i += blockDim.x) s[i] = make_uint4((uint32_t)k, i, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (t == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 8192;" ::"l"(out + k * 8192),
                   "r"((uint32_t)__cvta_generic_to_shared(sm + slot * 8192)) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
int main() {
  const size_t W = 436224000;
  uint8_t* out; cudaMalloc(&out, W + 65536);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch) {
    for (int it = 0; it < 3; ++it) launch();
    cudaEventRecord(a);
    for (int it = 0; it < 10; ++it) launch();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
    printf("%-28s %7.1f us %6.0f GB/s  %s\n", name, ms * 1e3, W / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  char nm[64];
  for (int thr : {256, 512, 1024, 2048}) {
    snprintf(nm, 64, "st128 %d thr/SM", thr);
    run(nm, [&] { st128<<<sms * (thr / 256), 256>>>((uint4*)out, W / 16); });
    snprintf(nm, 64, "st256 %d thr/SM", thr);
    run(nm, [&] { st256<<<sms * (thr / 256), 256>>>((uint4*)out, W / 32); });
  }
  cudaFuncSetAttribute(sttma, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  for (int per : {1, 2, 4, 6}) {
    snprintf(nm, 64, "tma-store %d CTA/SM", per);
    run(nm, [&] { sttma<<<sms * per, 128, 32768>>>(out, W / 8192); });
  }
  return 0;
}
