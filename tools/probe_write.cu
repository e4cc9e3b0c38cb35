// Write-bandwidth probe: int64 position-like streams written with 8-byte
// (256 B/warp) and 16-byte (512 B/warp) coalesced stores, default and
// streaming (.cs) cache hints.  Calibrates the ceiling of position output
// (expand_kernel); not product code.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int VEC, bool CS>
__global__ void k_write(int64_t* __restrict__ out, size_t n, int64_t base) {
  const size_t stride = (size_t)gridDim.x * blockDim.x * VEC;
  for (size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * VEC; i < n; i += stride) {
    if (VEC == 2) {
      longlong2 v = make_longlong2(base + i, base + i + 1);
      if (CS) __stcs(reinterpret_cast<longlong2*>(out + i), v);
      else *reinterpret_cast<longlong2*>(out + i) = v;
    } else {
      if (CS) __stcs(out + i, base + (int64_t)i);
      else out[i] = base + (int64_t)i;
    }
  }
}

template <int VEC, bool CS>
float run(int64_t* d, size_t n, int grid) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_write<VEC, CS><<<grid, 256>>>(d, n, 7);
  cudaEventRecord(a);
  for (int r = 0; r < 10; r++) k_write<VEC, CS><<<grid, 256>>>(d, n, r);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return n * 8.0 * 10 / (ms * 1e-3) / 1e9;
}

int main() {
  const size_t n = (size_t)2 << 30 >> 3 << 2;  // 8 GiB of int64
  int64_t* d;
  if (cudaMalloc(&d, n * 8) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int mult : {4, 8, 16, 32}) {
    const int grid = nsm * mult;
    printf("grid %5d  v1 %7.0f  v1.cs %7.0f  v2 %7.0f  v2.cs %7.0f GB/s\n", grid, run<1, false>(d, n, grid),
           run<1, true>(d, n, grid), run<2, false>(d, n, grid), run<2, true>(d, n, grid));
  }
  cudaFree(d);
  return 0;
}
