// Bandwidth probe: read-only streaming over a large buffer with (a) LDG.128
// grid-stride loads and (b) TMA 1D bulk copies into a shared-memory ring.
// Calibrates the practical read ceiling for the scan kernels (not product code).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int U>
__global__ void k_ldg(const uint4* __restrict__ p, size_t n16, uint32_t* out) {
  uint32_t acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; u++) v[u] = __ldcs(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; u++) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n16; i += stride) { uint4 v = p[i]; acc ^= v.x ^ v.y ^ v.z ^ v.w; }
  if (acc == 0x12345678) out[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}"
               :: "r"(smem_u32(b)), "r"(parity) : "memory");
}

template <int STAGES, int TILE>
__global__ void __launch_bounds__(256) k_tma(const uint8_t* __restrict__ p, size_t ntiles, uint32_t* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* bars = (uint64_t*)(sm + STAGES * TILE);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; s++) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  size_t t0 = blockIdx.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; s++) {
      size_t t = t0 + (size_t)s * gridDim.x;
      if (t < ntiles) { mbar_expect_tx(&bars[s], TILE); bulk_g2s(sm + s * TILE, p + t * TILE, TILE, &bars[s]); }
    }
  }
  uint32_t acc = 0;
  int it = 0;
  for (size_t t = t0; t < ntiles; t += gridDim.x, it++) {
    int s = it % STAGES;
    mbar_wait(&bars[s], (it / STAGES) & 1);
    const uint4* q = (const uint4*)(sm + s * TILE);
#pragma unroll 4
    for (int k = threadIdx.x; k < TILE / 16; k += 256) { uint4 v = q[k]; acc ^= v.x ^ v.y ^ v.z ^ v.w; }
    __syncthreads();
    if (threadIdx.x == 0) {
      size_t tn = t + (size_t)STAGES * gridDim.x;
      if (tn < ntiles) { mbar_expect_tx(&bars[s], TILE); bulk_g2s(sm + s * TILE, p + tn * TILE, TILE, &bars[s]); }
    }
  }
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  size_t n = (size_t)16 << 30;
  uint8_t* d; uint32_t* o;
  CK(cudaMalloc(&d, n)); CK(cudaMalloc(&o, 4));
  CK(cudaMemset(d, 0x5a, n));
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  auto rep = [&](const char* name, auto launch) {
    for (int w = 0; w < 3; w++) launch();
    cudaEventRecord(a);
    for (int r = 0; r < 10; r++) launch();
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("%-40s %8.3f ms  %8.1f GB/s  err=%s\n", name, ms / 10, n / (ms / 10 * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  for (int bpsm : {4, 8, 16}) {
    char nm[64]; snprintf(nm, 64, "ldg U=4 256thr %d blk/SM", bpsm);
    rep(nm, [&] { k_ldg<4><<<nsm * bpsm, 256>>>((const uint4*)d, n / 16, o); });
    snprintf(nm, 64, "ldg U=8 256thr %d blk/SM", bpsm);
    rep(nm, [&] { k_ldg<8><<<nsm * bpsm, 256>>>((const uint4*)d, n / 16, o); });
  }
  {
    constexpr int ST = 4, TL = 16384; size_t smem = ST * TL + 64;
    cudaFuncSetAttribute(k_tma<ST, TL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int bpsm : {2, 3}) { char nm[64]; snprintf(nm, 64, "tma 4x16K %d blk/SM", bpsm);
      rep(nm, [&] { k_tma<ST, TL><<<nsm * bpsm, 256, smem>>>(d, n / TL, o); }); }
  }
  {
    constexpr int ST = 3, TL = 32768; size_t smem = ST * TL + 64;
    cudaFuncSetAttribute(k_tma<ST, TL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int bpsm : {1, 2}) { char nm[64]; snprintf(nm, 64, "tma 3x32K %d blk/SM", bpsm);
      rep(nm, [&] { k_tma<ST, TL><<<nsm * bpsm, 256, smem>>>(d, n / TL, o); }); }
  }
  {
    constexpr int ST = 6, TL = 8192; size_t smem = ST * TL + 64;
    cudaFuncSetAttribute(k_tma<ST, TL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int bpsm : {2, 4}) { char nm[64]; snprintf(nm, 64, "tma 6x8K %d blk/SM", bpsm);
      rep(nm, [&] { k_tma<ST, TL><<<nsm * bpsm, 256, smem>>>(d, n / TL, o); }); }
  }
  // copy reference
  uint8_t* d2; CK(cudaMalloc(&d2, n / 2));
  rep("memcpy D2D 8GiB (r+w counted as n)", [&] { cudaMemcpyAsync(d2, d, n / 2, cudaMemcpyDeviceToDevice); });
  return 0;
}
