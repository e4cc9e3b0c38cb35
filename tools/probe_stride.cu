// Probe: time to touch one 16-byte gram every S bytes of a 16 GiB buffer
// (the access pattern of a sampled q-gram filter).  Tools only.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int U>
__global__ void k_stride(const uint8_t* __restrict__ p, size_t nsamp, size_t S, uint32_t* out) {
  uint32_t acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < nsamp; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; u++) v[u] = __ldcs(reinterpret_cast<const uint4*>(p + (i + u * stride) * S));
#pragma unroll
    for (int u = 0; u < U; u++) acc ^= v[u].x ^ v[u].w;
  }
  for (; i < nsamp; i += stride) { uint4 v = *reinterpret_cast<const uint4*>(p + i * S); acc ^= v.x; }
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  size_t n = (size_t)16 << 30;
  uint8_t* d; uint32_t* o;
  cudaMalloc(&d, n); cudaMalloc(&o, 4); cudaMemset(d, 0x5a, n);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (size_t S : {16, 32, 64, 128, 256, 512, 1024, 4096}) {
    size_t ns = n / S;
    for (int bpsm : {8, 16}) {
      auto run = [&] { k_stride<4><<<nsm * bpsm, 256>>>(d, ns, S, o); };
      for (int w = 0; w < 3; w++) run();
      cudaEventRecord(a);
      for (int r = 0; r < 10; r++) run();
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
      printf("S=%5zu blk/SM=%2d  %8.3f ms  text-equiv %9.1f GB/s  samples %8.2f G/s\n", S, bpsm, ms,
             n / (ms * 1e-3) / 1e9, ns / (ms * 1e-3) / 1e9);
    }
  }
  return 0;
}
