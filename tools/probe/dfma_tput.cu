// Probe: FP64 FMA issue throughput (independent chains) and the shifting-window
// elimination step (panel2's shift_update) in isolation, 256 threads / SM.
#include <cstdio>
__global__ void tput(double* out, long long* cyc, int n) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double y = 1.0000001;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], y, 1e-300);
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void shift(double* out, long long* cyc, int n) {
  __shared__ __align__(16) double ub[32 * 34];
  for (int e = threadIdx.x; e < 32 * 34; e += blockDim.x) ub[e] = 1e-3 * e;
  __syncthreads();
  double w[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) w[c] = threadIdx.x + c;
  long long t0 = clock64();
  for (int it = 0; it < n; ++it)
    for (int j = 0; j < 32; ++j) {
      const double l = w[0] * ub[j * 34 + 33];
      const double2* p2 = reinterpret_cast<const double2*>(ub + j * 34);
#pragma unroll
      for (int c2 = 0; c2 < 16; ++c2) {
        const double2 u = p2[c2];
        if (c2 > 0) w[2 * c2 - 1] = fma(-l, u.x, w[2 * c2]);
        w[2 * c2] = fma(-l, u.y, w[2 * c2 + 1]);
      }
      w[31] = l;
    }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < 32; ++c) s += w[c];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024 * 148); cudaMalloc(&c, 8 * 256);
  for (int nt : {32, 128, 256, 512}) {
    tput<<<1, nt>>>(o, c, 4096);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    const double warp_instr = 4096.0 * 16 * (nt / 32);
    printf("dfma tput threads %3d: %.2f cycles per warp-DFMA per SM (%.1f lanes/clk/SM)\n", nt, h / warp_instr,
           32.0 * warp_instr / h);
  }
  for (int nt : {32, 256}) {
    shift<<<1, nt>>>(o, c, 64);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("shift step threads %3d: %.1f cycles per step\n", nt, h / (64.0 * 32));
  }
  return 0;
}
