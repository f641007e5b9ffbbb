// Probe: per-step latency of the top-block LU dependency chain (one warp).
#include <cstdio>
#include <cuda_runtime.h>
template <int VAR>
__global__ void k(double* io, long long* clk, int kbe, double* urinv) {
  int jf = 32;
  const int lane = threadIdx.x & 31;
  double v[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) v[c] = io[lane * 32 + c] + (c == lane ? 64.0 : 0.0);
  __syncwarp();
  long long t0 = clock64();
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    if (VAR == 3 && j >= kbe) break;
    const double pj = __shfl_sync(0xffffffffu, v[j], j);
    double rinv;
    if (VAR == 0) rinv = __drcp_rn(pj);
    else rinv = 1.0 / pj;
    if (VAR == 2) {  // chain only: update just the next column
      if (lane > j) {
        const double l = v[j] * rinv;
        v[j] = l;
        if (j + 1 < 32) v[j + 1] = fma(-l, __shfl_sync(0xffffffffu, v[j + 1], j), v[j + 1]);
      }
    } else {
      double pr[32];
#pragma unroll
      for (int c = j + 1; c < 32; ++c) pr[c] = __shfl_sync(0xffffffffu, v[c], j);
      if (VAR == 3 && lane == j) urinv[j] = rinv;
      if (lane > j && (VAR != 3 || lane < kbe)) {
        const double l = v[j] * rinv;
        v[j] = l;
        if (VAR == 3 && !(fabs(l) <= 1.0) && jf == 32) jf = j;
#pragma unroll
        for (int c = j + 1; c < 32; ++c) v[c] = fma(-l, pr[c], v[c]);
      }
    }
  }
  long long t1 = clock64();
#pragma unroll
  for (int c = 0; c < 32; ++c) io[lane * 32 + c] = v[c];
  if (lane == 0) clk[0] = t1 - t0 + jf * 0;
  if (jf == 7) io[0] = 1.0;
}
template <int VAR>
void run(const char* name) {
  double* io; long long* c; cudaMalloc(&io, 8 * 1024); cudaMalloc(&c, 8);
  cudaMemset(io, 0, 8 * 1024);
  long long h = 0;
  double* ur; cudaMalloc(&ur, 8 * 32);
  for (int i = 0; i < 3; ++i) { k<VAR><<<1, 32>>>(io, c, 32, ur); cudaDeviceSynchronize(); }
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-30s %lld cycles (%.0f per step)\n", name, h, h / 32.0);
}
int main() {
  run<0>("full step, __drcp_rn");
  run<1>("full step, 1/x");
  run<3>("full step + guards/jf/urinv");
  return 0;
}
