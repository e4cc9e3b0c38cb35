// Write-pattern probe for expand_kernel (tools only): int64 outputs of
// variable-size segments written (W) by a warp per segment, (C) by a CTA per
// segment, (O) output-partitioned -- 256-element chunks per warp, grid-stride
// -- and (O8) 2048-element chunks per 8-warp CTA.  Segment sizes uniform in
// [lo, hi]; offsets = exclusive prefix.  Reports GB/s of output written.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) k_warp(int64_t* __restrict__ out, const int64_t* __restrict__ off, int nseg) {
  const int lane = threadIdx.x & 31;
  const int W = gridDim.x * 8;
  for (int g = blockIdx.x * 8 + (threadIdx.x >> 5); g < nseg; g += W) {
    const int64_t o = off[g];
    const int sz = (int)(off[g + 1] - o);
    int64_t* d = out + o;
#pragma unroll 4
    for (int i = lane; i < sz; i += 32) d[i] = (int64_t)g * 2048 + i;
  }
}
// warp per segment, rows aligned to the output's 256-byte lines
__global__ void __launch_bounds__(256) k_warp_al(int64_t* __restrict__ out, const int64_t* __restrict__ off, int nseg) {
  const int lane = threadIdx.x & 31;
  const int W = gridDim.x * 8;
  for (int g = blockIdx.x * 8 + (threadIdx.x >> 5); g < nseg; g += W) {
    const int64_t o = off[g];
    const unsigned sz = (unsigned)(off[g + 1] - o);
    int64_t* d = out + o;
    const unsigned head = (unsigned)(o & 31);
    const unsigned nrows = (head + sz + 31) >> 5;
#pragma unroll 4
    for (unsigned r = 0; r < nrows; r++) {
      const unsigned i = 32 * r + lane - head;
      if (i < sz) d[i] = (int64_t)g * 2048 + i;
    }
  }
}
// warp per segment, aligned rows, plus the real kernel's reads: a 256-byte
// bitmap and a 24-byte queue entry per segment, prefetched one segment ahead
__global__ void __launch_bounds__(256) k_warp_al_rd(int64_t* __restrict__ out, const int64_t* __restrict__ off, int nseg,
                                                    const uint2* __restrict__ bm) {
  const int lane = threadIdx.x & 31;
  const int W = gridDim.x * 8;
  int g = blockIdx.x * 8 + (threadIdx.x >> 5);
  uint2 x = g < nseg ? bm[(size_t)g * 32 + lane] : make_uint2(0, 0);
  for (; g < nseg; g += W) {
    const uint2 nx = g + W < nseg ? bm[(size_t)(g + W) * 32 + lane] : make_uint2(0, 0);
    const int64_t o = off[g];
    const unsigned sz = (unsigned)(off[g + 1] - o);
    int64_t* d = out + o;
    const unsigned head = (unsigned)(o & 31);
    const unsigned nrows = (head + sz + 31) >> 5;
    const int64_t v0 = (int64_t)g * 2048 + (x.x ^ x.y);
#pragma unroll 4
    for (unsigned r = 0; r < nrows; r++) {
      const unsigned i = 32 * r + lane - head;
      if (i < sz) d[i] = v0 + i;
    }
    x = nx;
  }
}
// CTA per segment, aligned rows, warp w on rows w, w + 8, ...
__global__ void __launch_bounds__(256) k_cta_al(int64_t* __restrict__ out, const int64_t* __restrict__ off, int nseg) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int g = blockIdx.x; g < nseg; g += gridDim.x) {
    const int64_t o = off[g];
    const unsigned sz = (unsigned)(off[g + 1] - o);
    int64_t* d = out + o;
    const unsigned head = (unsigned)(o & 31);
    const unsigned nrows = (head + sz + 31) >> 5;
#pragma unroll 4
    for (unsigned r = warp; r < nrows; r += 8) {
      const unsigned i = 32 * r + lane - head;
      if (i < sz) d[i] = (int64_t)g * 2048 + i;
    }
  }
}
__global__ void __launch_bounds__(256) k_cta(int64_t* __restrict__ out, const int64_t* __restrict__ off, int nseg) {
  for (int g = blockIdx.x; g < nseg; g += gridDim.x) {
    const int64_t o = off[g];
    const int sz = (int)(off[g + 1] - o);
    int64_t* d = out + o;
#pragma unroll 4
    for (int i = threadIdx.x; i < sz; i += 256) d[i] = (int64_t)g * 2048 + i;
  }
}
// output-partitioned: chunk of CH elements per warp, chunks grid-stride by warp
template <int CH>
__global__ void __launch_bounds__(256) k_out(int64_t* __restrict__ out, int64_t total) {
  const int lane = threadIdx.x & 31;
  const int64_t W = (int64_t)gridDim.x * 8;
  const int64_t nch = (total + CH - 1) / CH;
  for (int64_t c = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); c < nch; c += W) {
    int64_t* d = out + c * CH;
    const int64_t lim = total - c * CH < CH ? total - c * CH : CH;
#pragma unroll
    for (int j = 0; j < CH / 32; j++)
      if (lane + 32 * j < lim) d[lane + 32 * j] = c * CH + lane + 32 * j;
  }
}
// output-partitioned, CTA-wide chunk of 8 * CH elements, warp w writes rows w, w + 8, ...
template <int CH>
__global__ void __launch_bounds__(256) k_out_cta(int64_t* __restrict__ out, int64_t total) {
  const int64_t nch = (total + 8 * CH - 1) / (8 * CH);
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
    int64_t* d = out + c * 8 * CH;
    const int64_t lim = total - c * 8 * CH < 8 * CH ? total - c * 8 * CH : 8 * CH;
#pragma unroll
    for (int j = 0; j < CH / 32; j++)
      if (threadIdx.x + 256 * j < lim) d[threadIdx.x + 256 * j] = c * 8 * CH + threadIdx.x + 256 * j;
  }
}

template <class F>
static double timeit(F f, double bytes) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaEventRecord(a);
  for (int r = 0; r < 5; r++) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return bytes * 5 / (ms * 1e-3) / 1e9;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int64_t cap = (int64_t)256 << 20;  // 2 GiB of int64
  int64_t* out;
  cudaMalloc(&out, cap * 8);
  for (auto range : {std::pair<int, int>{2030, 2048}, {1000, 2048}, {400, 640}, {40, 200}}) {
    std::vector<int64_t> off(1, 0);
    srand(7);
    while (off.back() + range.second < cap) off.push_back(off.back() + range.first + rand() % (range.second - range.first + 1));
    const int nseg = (int)off.size() - 1;
    const int64_t total = off.back();
    int64_t* d_off;
    cudaMalloc(&d_off, off.size() * 8);
    cudaMemcpy(d_off, off.data(), off.size() * 8, cudaMemcpyHostToDevice);
    const double bytes = total * 8.0;
    uint2* d_bm;
    cudaMalloc(&d_bm, (size_t)nseg * 256);
    cudaMemset(d_bm, 0x55, (size_t)nseg * 256);
    printf("sizes %d..%d (%d segments):\n", range.first, range.second, nseg);
    for (int mult : {1, 2, 4, 5, 8}) {
      const int g = nsm * mult;
      printf("  grid %4d: warp/seg aligned %6.0f  +reads %6.0f  cta/seg aligned %6.0f |", g,
             timeit([&] { k_warp_al<<<g, 256>>>(out, d_off, nseg); }, bytes),
             timeit([&] { k_warp_al_rd<<<g, 256>>>(out, d_off, nseg, d_bm); }, bytes),
             timeit([&] { k_cta_al<<<g, 256>>>(out, d_off, nseg); }, bytes));
      printf(" warp/seg %6.0f  cta/seg %6.0f  out256/warp %6.0f  out1024/warp %6.0f  out2048/cta %6.0f out8192/cta %6.0f GB/s\n",
             timeit([&] { k_warp<<<g, 256>>>(out, d_off, nseg); }, bytes),
             timeit([&] { k_cta<<<g, 256>>>(out, d_off, nseg); }, bytes),
             timeit([&] { k_out<256><<<g, 256>>>(out, total); }, bytes),
             timeit([&] { k_out<1024><<<g, 256>>>(out, total); }, bytes),
             timeit([&] { k_out_cta<256><<<g, 256>>>(out, total); }, bytes),
             timeit([&] { k_out_cta<1024><<<g, 256>>>(out, total); }, bytes));
    }
    cudaFree(d_off);
    cudaFree(d_bm);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
