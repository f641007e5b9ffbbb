// Probe: instruction-fetch rate of straight-line code (cold i-cache) vs a warm loop.
#include <cstdio>
#include <cuda_runtime.h>
template <int N>
__device__ __forceinline__ void body(unsigned& a, unsigned& b, unsigned& c, unsigned& d) {
  // 16 independent chains (a..d used as inputs only by their own chain)
  unsigned x[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) x[q] = a + q;
#pragma unroll
  for (int i = 0; i < N / 4; ++i)
#pragma unroll
    for (int q = 0; q < 16; ++q) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[q]) : "r"(b), "r"(c));
#pragma unroll
  for (int q = 0; q < 16; ++q) d += x[q];
}
template <int N, int REP>
__global__ void k(unsigned* out, long long* clk) {
  unsigned a = threadIdx.x, b = a + 1, c = a + 2, d = a + 3;
  long long t0 = clock64();
#pragma unroll 1
  for (int r = 0; r < REP; ++r) body<N>(a, b, c, d);
  long long t1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  out[threadIdx.x + blockIdx.x * blockDim.x] = a + b + c + d;
}
template <int N, int REP>
void run(int threads, const char* name) {
  unsigned* o; long long* c; cudaMalloc(&o, 4 * 1024); cudaMalloc(&c, 8 * 16);
  long long h = 0;
  for (int it = 0; it < 3; ++it) {
    k<N, REP><<<1, threads>>>(o, c);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  }
  const double instr = double(N) * 4 * REP;
  printf("%-26s warps %2d: %8lld cycles, %.3f warp-instr/cycle per warp, code %.1f KB\n", name, threads / 32, h,
         instr / h, N * 4 * 16 / 1024.0);
  cudaFree(o); cudaFree(c);
}
int main() {
  run<64, 512>(32, "loop 256 IMAD");
  run<64, 512>(256, "loop 256 IMAD");
  run<512, 64>(32, "loop 2048 IMAD");
  run<2048, 16>(32, "loop 8192 IMAD");
  run<8192, 4>(32, "straight 32768 IADD x4");
  run<8192, 4>(256, "straight 32768 IADD x4");
  run<8192, 1>(32, "straight 32768 IADD");
  run<8192, 1>(256, "straight 32768 IADD");
  return 0;
}
