// pdl_probe.cu -- per-kernel cost of a dependent chain of small kernels in one CUDA graph,
// with and without programmatic dependent launch (griddepcontrol.wait / launch_dependents at
// the top of each kernel, cudaLaunchAttributeProgrammaticStreamSerialization on the launch).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pdl_probe tools/pdl_probe.cu
//   tools/pdl_probe
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

template <bool PDL>
__global__ void k_axpy(int n, const float* __restrict__ x, float* __restrict__ y) {
  if (PDL) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) y[i] = 0.5f * y[i] + x[i];
}

template <bool PDL>
int run(int n, int grid, int chain, float* x, float* y, cudaStream_t s, float* ms) {
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  for (int i = 0; i < chain; ++i) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = PDL ? 1 : 0;
    CK(cudaLaunchKernelEx(&cfg, k_axpy<PDL>, n, (const float*)(i & 1 ? y : x), i & 1 ? x : y));
  }
  CK(cudaStreamEndCapture(s, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) CK(cudaGraphLaunch(ge, s));
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0, s);
    CK(cudaGraphLaunch(ge, s));
    cudaEventRecord(e1, s);
    CK(cudaEventSynchronize(e1));
    float t;
    cudaEventElapsedTime(&t, e0, e1);
    if (t < best) best = t;
  }
  *ms = best;
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  return 0;
}

int main() {
  const int chain = 400;
  float *x, *y;
  CK(cudaMalloc(&x, 64 << 20));
  CK(cudaMalloc(&y, 64 << 20));
  CK(cudaMemset(x, 0, 64 << 20));
  CK(cudaMemset(y, 0, 64 << 20));
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  int ns[] = {256, 32768, 262144, 1048576, 4194304};
  for (int n : ns)
    for (int grid : {1, 148, 592, 1184}) {
      if (grid * 256 > 4 * n && grid > 1) continue;
      float a, b;
      if (run<false>(n, grid, chain, x, y, s, &a) || run<true>(n, grid, chain, x, y, s, &b)) return 1;
      printf("n %8d grid %5d: plain %7.2f us/kernel  pdl %7.2f us/kernel  (%.2f us saved)\n", n, grid,
             a * 1e3f / chain, b * 1e3f / chain, (a - b) * 1e3f / chain);
    }
  return 0;
}
