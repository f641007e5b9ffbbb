// Probe: per-node overhead of a captured chain of small kernels (one stream; and
// two streams with the panel/side dependency pattern of the engine).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void tiny(int* p, int v) { if (threadIdx.x == 0 && blockIdx.x == 0) p[0] += v; }
int main() {
  int* d; cudaMalloc(&d, 64);
  cudaStream_t s, s2, cap; cudaStreamCreate(&s); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking);
  cudaEvent_t ev[4]; for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  for (int mode = 0; mode < 2; ++mode) {
    const int N = 256;
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < N; ++i) {
      if (mode == 1 && i >= 2) cudaStreamWaitEvent(cap, ev[i & 1], 0);
      tiny<<<8, 256, 0, cap>>>(d, 1);
      if (mode == 1) {
        cudaEventRecord(ev[2], cap);
        cudaStreamWaitEvent(s2, ev[2], 0);
        tiny<<<64, 256, 0, s2>>>(d + 4, 1);
        tiny<<<64, 256, 0, s2>>>(d + 8, 1);
        cudaEventRecord(ev[i & 1], s2);
      }
    }
    if (mode == 1) cudaStreamWaitEvent(cap, ev[(N - 1) & 1], 0);
    cudaStreamEndCapture(cap, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a, s); cudaGraphLaunch(ge, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("mode %d: %d chain kernels in %.1f us -> %.2f us per main-stream kernel (%s)\n", mode, N, best * 1e3,
           best * 1e3 / N, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
