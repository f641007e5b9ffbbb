// Probe: straight-line code throughput (i-cache) and DFMA issue rate with 8 warps.
#include <cstdio>
#include <cuda_runtime.h>
template <int N>
__device__ __forceinline__ void body(double& a, double& b, double& c, double& d, double x) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    asm volatile("fma.rn.f64 %0, %0, %4, %4;\n fma.rn.f64 %1, %1, %4, %4;\n fma.rn.f64 %2, %2, %4, %4;\n fma.rn.f64 %3, %3, %4, %4;\n"
                 : "+d"(a), "+d"(b), "+d"(c), "+d"(d) : "d"(x));
  }
}
template <int N, int REP>
__global__ void k(double* out, long long* clk, double x) {
  double a = threadIdx.x, b = a + 1, c = a + 2, d = a + 3;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int r = 0; r < REP; ++r) body<N>(a, b, c, d, x);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  out[threadIdx.x + blockIdx.x * blockDim.x] = a + b + c + d;
}
template <int N, int REP>
void run(int threads, const char* name) {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8 * 16);
  long long h = 0;
  for (int it = 0; it < 3; ++it) {
    k<N, REP><<<1, threads>>>(o, c, 1.0000001);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  }
  const double instr = double(N) * 4 * REP;  // DFMA per thread
  printf("%-28s threads %4d: %8lld cycles, %.2f cycles per DFMA per warp-slot (%.1f DFMA/clk/SM)\n", name, threads, h,
         h / instr, instr * threads / h);
  cudaFree(o); cudaFree(c);
}
int main() {
  run<8, 256>(32, "loop body 32 DFMA");
  run<8, 256>(256, "loop body 32 DFMA");
  run<8, 256>(1024, "loop body 32 DFMA");
  run<2048, 1>(32, "straight 8192 DFMA");
  run<2048, 1>(256, "straight 8192 DFMA");
  run<2048, 1>(1024, "straight 8192 DFMA");
  run<2048, 4>(256, "straight 8192 DFMA x4");
  return 0;
}
