#include <cstdio>
#include <cuda_runtime.h>
__global__ void spin(int n, float* x) { float a = 0; for (int i = 0; i < n; ++i) a = a * 0.999f + 1; if (a == 0) x[0] = a; }
int main() {
  cudaStream_t s; cudaStreamCreate(&s);
  float* x; cudaMalloc(&x, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  cudaEventRecord(a, s);
  spin<<<1, 32, 0, s>>>(1000000, x);
  cudaEventRecord(b, s);
  cudaError_t e = cudaStreamEndCapture(s, &g);
  printf("end capture: %s\n", cudaGetErrorString(e));
  e = cudaGraphInstantiate(&ge, g, 0); printf("inst: %s\n", cudaGetErrorString(e));
  for (int r = 0; r < 3; ++r) {
    e = cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    float ms = -1; e = cudaEventElapsedTime(&ms, a, b);
    printf("replay %d: %s %.3f ms\n", r, cudaGetErrorString(e), ms);
  }
  return 0;
}
