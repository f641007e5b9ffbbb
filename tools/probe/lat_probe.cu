// Probe: dependent-chain latencies (cycles) of FP64 ops, shuffles, smem, barriers on sm_100a.
#include <cstdio>
__global__ void lat(double* out, long long* cyc, double x0, int n) {
  double x = x0 + threadIdx.x * 1e-30, y = 1.0000001;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-300);
  t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0) / n;
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x * y;
  t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0) / n;
  // drcp chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __drcp_rn(x) + 1e-300;
  t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0) / n;
  // shfl chain (double)
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1e-300;
  t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0) / n;
  // redux chain
  unsigned u = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) u = __reduce_max_sync(0xffffffffu, u) + 1u;
  t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0) / n;
  // syncthreads loop
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64(); if (threadIdx.x == 0) cyc[5] = (t1 - t0) / n;
  // FFMA chain (float) reference
  float f = x0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) f = fmaf(f, 1.0000001f, 1e-30f);
  t1 = clock64(); if (threadIdx.x == 0) cyc[6] = (t1 - t0) / n;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + 1e-300;
  t1 = clock64(); if (threadIdx.x == 0) cyc[7] = (t1 - t0) / n;
  out[threadIdx.x] = x + f + u;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8 * 16);
  for (int nt : {32, 256}) {
    lat<<<1, nt>>>(o, c, 1.0, 4096);
    long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    printf("threads %d: dfma %lld dmul %lld drcp+dadd %lld shfl+dadd %lld redux+iadd %lld syncthreads %lld ffma %lld dadd %lld\n",
           nt, h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
  }
  return 0;
}
