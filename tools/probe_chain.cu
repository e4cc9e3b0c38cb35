// Floor of a 3-kernel chain (scan -> offsets -> expand shapes) on B200 (tools only).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_chain tools/probe_chain.cu
#include <cuda_runtime.h>
#include <cstdio>

__global__ void __launch_bounds__(544) ka(int* x, int trig) {
  if (trig) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) atomicAdd(x, 1);
}
__global__ void __launch_bounds__(512) kb(int* x, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) atomicAdd(x + 1, 1);
}
__global__ void __launch_bounds__(128) kc(int* x, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) atomicAdd(x + 2, 1);
}
__global__ void kall(int* x) {  // one kernel doing the three steps with grid barriers
  if (threadIdx.x == 0) atomicAdd(x, 1);
}

template <class K, class... A>
static void launch(K k, int grid, int block, cudaStream_t st, bool pdl, A... a) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, a...);
}

int main() {
  int* x;
  cudaMalloc(&x, 64);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int R = 2000;
  for (int mode = 0; mode < 6; mode++) {
    // 0: A only; 1: A,B,C plain; 2: A,B,C PDL; 3: PDL + early trigger; 4: A,B PDL; 5: graph of mode 3
    auto chain = [&]() {
      const bool pdl = mode >= 2;
      launch(ka, 296, 544, st, false, x, mode == 3 || mode == 5 ? 1 : 0);
      if (mode >= 1) launch(kb, mode == 4 ? 8 : 8, 512, st, pdl, x, pdl ? 1 : 0);
      if (mode >= 1 && mode != 4) launch(kc, 592, 128, st, pdl, x, pdl ? 1 : 0);
    };
    cudaGraphExec_t ge = nullptr;
    if (mode == 5) {
      cudaGraph_t g;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
      for (int i = 0; i < 100; i++) chain();
      cudaStreamEndCapture(st, &g);
      cudaGraphInstantiate(&ge, g, 0);
    }
    for (int w = 0; w < 50; w++) chain();
    cudaEventRecord(e0, st);
    if (mode == 5)
      for (int i = 0; i < R / 100; i++) cudaGraphLaunch(ge, st);
    else
      for (int i = 0; i < R; i++) chain();
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("mode %d: %.2f us per chain (%s)\n", mode, 1e3 * ms / R,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
