// HBM bandwidth for a read/write byte mix (the codec kernels' traffic shape):
// each CTA streams its share of R read bytes and W written bytes with 16-B
// vector accesses.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 bw_mix.cu -o bw_mix
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void mix(const uint4* __restrict__ in, size_t nr, uint4* __restrict__ out, size_t nw) {
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nt = (size_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  const size_t n = nr > nw ? nr : nw;
  for (size_t i = tid; i < n; i += nt) {
    if (i < nr) { uint4 v = __ldcs(in + i); acc ^= v.x ^ v.y ^ v.z ^ v.w; }
    if (i < nw) __stcs(out + i, make_uint4(acc, (uint32_t)i, 0, 0));
  }
  if (acc == 0x12345678u) out[0].x = acc;
}
int main() {
  const size_t R = 436224000, Ws[] = {0, 306247808, 436224000, 2 * 436224000ul};
  uint4 *in, *out;
  cudaMalloc(&in, 2 * R); cudaMalloc(&out, 2 * R);
  cudaMemset(in, 1, 2 * R);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (size_t rr : {R, (size_t)306247808}) for (size_t W : Ws) for (int per : {4, 8}) {
    const size_t nr = rr / 16, nw = W / 16;
    for (int it = 0; it < 3; ++it) mix<<<sms * per, 256>>>(in, nr, out, nw);
    cudaEventRecord(a);
    for (int it = 0; it < 10; ++it) mix<<<sms * per, 256>>>(in, nr, out, nw);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
    printf("read %zu MB write %zu MB ctas/SM %d: %.1f us  %.0f GB/s\n", rr >> 20, W >> 20, per, ms * 1e3, (rr + W) / ms / 1e6);
  }
  return 0;
}
