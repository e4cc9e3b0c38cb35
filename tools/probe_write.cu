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

// region-per-warp: each warp writes whole 16 KB runs (2048 int64), 256 B per
// store instruction -- the dense-segment output pattern of expand_kernel
__global__ void k_region(int64_t* __restrict__ out, size_t nseg, int64_t base) {
  const int lane = threadIdx.x & 31;
  const size_t w0 = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t g = w0; g < nseg; g += nw) {
    int64_t* d = out + g * 2048 + 5;  // odd offset: runs are not 256-B aligned in expand either
    for (int i = lane; i < 2048 - 5; i += 32) d[i] = base + (int64_t)(g * 2048 + i);
  }
}
// region-per-warp variants: run start offset OFF (int64 elements), 16-byte
// vector stores over the 16-B aligned body (VEC 2), streaming hint (CS)
template <int OFF, int VEC, bool CS>
__global__ void k_region_v(int64_t* __restrict__ out, size_t nseg, int64_t base) {
  const int lane = threadIdx.x & 31;
  const size_t w0 = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t g = w0; g < nseg; g += nw) {
    int64_t* d = out + g * 2048 + OFF;
    const int len = 2048 - 5;
    const int64_t v0 = base + (int64_t)(g * 2048);
    if (VEC == 1) {
      for (int i = lane; i < len; i += 32) {
        if (CS) __stcs(d + i, v0 + i); else d[i] = v0 + i;
      }
    } else {
      const int head = (int)(((uintptr_t)d >> 3) & 1);  // 0 or 1 element to reach 16-B alignment
      if (lane == 0 && head) d[0] = v0;
      const int body = (len - head) / 2;
      longlong2* dv = reinterpret_cast<longlong2*>(d + head);
      for (int i = lane; i < body; i += 32) {
        const longlong2 v = make_longlong2(v0 + head + 2 * i, v0 + head + 2 * i + 1);
        if (CS) __stcs(dv + i, v); else dv[i] = v;
      }
      if (lane == 0 && head + 2 * body < len) d[len - 1] = v0 + len - 1;
    }
  }
}
template <int OFF, int VEC, bool CS>
float run_region_v(int64_t* d, size_t n, int grid, int block) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const size_t nseg = n / 2048 - 1;
  k_region_v<OFF, VEC, CS><<<grid, block>>>(d, nseg, 7);
  cudaEventRecord(a);
  for (int r = 0; r < 10; r++) k_region_v<OFF, VEC, CS><<<grid, block>>>(d, nseg, r);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return nseg * (2048 - 5) * 8.0 * 10 / (ms * 1e-3) / 1e9;
}

// region-per-warp, each warp starting at a rotated point of its run (de-
// correlates which DRAM channels the warps hit at the same moment)
__global__ void k_region_rot(int64_t* __restrict__ out, size_t nseg, int64_t base, int rmul) {
  const int lane = threadIdx.x & 31;
  const size_t w0 = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  const int len = 2048 - 5;
  for (size_t g = w0; g < nseg; g += nw) {
    int64_t* d = out + g * 2048 + 5;
    const int rot = (int)((g * (size_t)rmul) % (size_t)len) & ~31;
    for (int i = lane; i < len; i += 32) {
      int j = i + rot;
      if (j >= len) j -= len;
      d[j] = base + (int64_t)(g * 2048 + j);
    }
  }
}
float run_region_rot(int64_t* d, size_t n, int grid, int block, int rmul) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const size_t nseg = n / 2048 - 1;
  k_region_rot<<<grid, block>>>(d, nseg, 7, rmul);
  cudaEventRecord(a);
  for (int r = 0; r < 10; r++) k_region_rot<<<grid, block>>>(d, nseg, r, rmul);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return nseg * (2048 - 5) * 8.0 * 10 / (ms * 1e-3) / 1e9;
}

// region-per-warp through TMA bulk stores: the warp fills a 16 KB smem buffer
// (double-buffered) and one lane issues cp.async.bulk.global.shared for the
// 16-B aligned body; head/tail elements are plain stores
__global__ void __launch_bounds__(128) k_region_tma(int64_t* __restrict__ out, size_t nseg, int64_t base, int off) {
  extern __shared__ __align__(128) int64_t sbuf[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t w0 = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  const int len = 2048 - 5;
  int buf = 0;
  for (size_t g = w0; g < nseg; g += nw, buf ^= 1) {
    int64_t* d = out + g * 2048 + off;
    const int64_t v0 = base + (int64_t)(g * 2048);
    const int head = (int)(((uintptr_t)d >> 3) & 1);
    const int body = (len - head) & ~1;
    int64_t* sb = sbuf + (warp * 2 + buf) * 2048;
    // the bulk copy that read this buffer two iterations ago must be done
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
    for (int i = lane; i < body; i += 32) sb[i] = v0 + head + i;
    if (lane == 0 && head) d[0] = v0;
    if (lane == 0 && head + body < len) d[len - 1] = v0 + len - 1;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d + head),
                   "r"((uint32_t)__cvta_generic_to_shared(sb)), "r"((uint32_t)(body * 8))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
float run_region_tma(int64_t* d, size_t n, int grid, int off) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const size_t nseg = n / 2048 - 1;
  const size_t smem = 4 * 2 * 2048 * 8;
  cudaFuncSetAttribute(k_region_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_region_tma<<<grid, 128, smem>>>(d, nseg, 7, off);
  cudaEventRecord(a);
  for (int r = 0; r < 10; r++) k_region_tma<<<grid, 128, smem>>>(d, nseg, r, off);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("  (tma err: %s)\n", cudaGetErrorString(cudaGetLastError()));
  return nseg * (2048 - 5) * 8.0 * 10 / (ms * 1e-3) / 1e9;
}

// region-per-CTA of S consecutive 16 KB runs: the whole block writes S*2048
// int64 at a time (a CTA expanding S consecutive dense segments)
template <int S>
__global__ void k_region_cta_s(int64_t* __restrict__ out, size_t nreg, int64_t base) {
  for (size_t g = blockIdx.x; g < nreg; g += gridDim.x) {
    int64_t* d = out + g * 2048 * S + 5;
    for (int i = threadIdx.x; i < 2048 * S - 5; i += blockDim.x) d[i] = base + (int64_t)(g * 2048 * S + i);
  }
}
template <int S>
float run_region_cta_s(int64_t* d, size_t n, int grid, int block) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const size_t nreg = n / (2048 * S) - 1;
  k_region_cta_s<S><<<grid, block>>>(d, nreg, 7);
  cudaEventRecord(a);
  for (int r = 0; r < 10; r++) k_region_cta_s<S><<<grid, block>>>(d, nreg, r);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return nreg * (2048.0 * S - 5) * 8.0 * 10 / (ms * 1e-3) / 1e9;
}

// region-per-CTA: the whole block writes one 16 KB run at a time
__global__ void k_region_cta(int64_t* __restrict__ out, size_t nseg, int64_t base) {
  for (size_t g = blockIdx.x; g < nseg; g += gridDim.x) {
    int64_t* d = out + g * 2048 + 5;
    for (int i = threadIdx.x; i < 2048 - 5; i += blockDim.x) d[i] = base + (int64_t)(g * 2048 + i);
  }
}
float run_region_cta(int64_t* d, size_t n, int grid, int block) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const size_t nseg = n / 2048;
  k_region_cta<<<grid, block>>>(d, nseg, 7);
  cudaEventRecord(a);
  for (int r = 0; r < 10; r++) k_region_cta<<<grid, block>>>(d, nseg, r);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return nseg * (2048 - 5) * 8.0 * 10 / (ms * 1e-3) / 1e9;
}
float run_region(int64_t* d, size_t n, int grid, int block) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const size_t nseg = n / 2048;
  k_region<<<grid, block>>>(d, nseg, 7);
  cudaEventRecord(a);
  for (int r = 0; r < 10; r++) k_region<<<grid, block>>>(d, nseg, r);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return nseg * (2048 - 5) * 8.0 * 10 / (ms * 1e-3) / 1e9;
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
  for (int mult : {4, 8, 16}) printf("region-per-warp grid %5d x 128: %7.0f GB/s\n", nsm * mult, run_region(d, n, nsm * mult, 128));
  for (int mult : {2, 4}) printf("region-per-warp grid %5d x 512: %7.0f GB/s\n", nsm * mult, run_region(d, n, nsm * mult, 512));
  for (int mult : {4, 8, 16}) printf("region-per-CTA grid %5d x 128: %7.0f GB/s\n", nsm * mult, run_region_cta(d, n, nsm * mult, 128));
  for (int mult : {2, 4}) printf("region-per-CTA grid %5d x 512: %7.0f GB/s\n", nsm * mult, run_region_cta(d, n, nsm * mult, 512));
  for (int mult : {4, 8}) {
    const int g = nsm * mult;
    printf("region-per-warp x256 grid %5d: off5 v1 %7.0f | off0 v1 %7.0f | off5 v2 %7.0f | off0 v2 %7.0f | off5 v2.cs %7.0f | off5 v1.cs %7.0f GB/s\n", g,
           run_region_v<5, 1, false>(d, n, g, 256), run_region_v<0, 1, false>(d, n, g, 256),
           run_region_v<5, 2, false>(d, n, g, 256), run_region_v<0, 2, false>(d, n, g, 256),
           run_region_v<5, 2, true>(d, n, g, 256), run_region_v<5, 1, true>(d, n, g, 256));
  }
  for (int mult : {1, 2, 3}) {
    const int g = nsm * mult;
    printf("region-per-warp TMA bulk store grid %5d x 128: off5 %7.0f | off0 %7.0f GB/s\n", g,
           run_region_tma(d, n, g, 5), run_region_tma(d, n, g, 0));
  }
  cudaFree(d);
  return 0;
}
