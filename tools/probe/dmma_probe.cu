// Probe: verify mma.sync m16n8k4/k8/k16 f64 fragment layouts on sm_100a and
// measure a DMMA-only throughput loop (registers only) to bound the FP64 tensor peak.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma_k4(double* c, const double* a, double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(b));
}
__device__ __forceinline__ void mma_k8(double* c, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

// A row-major 16x4 in gmem, B 4x8 (k-major), C 16x8 row-major
__global__ void layout_k4(const double* A, const double* B, double* C) {
  int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a[2] = {A[(g)*4 + t], A[(g + 8) * 4 + t]};
  double b = B[t * 8 + g];
  double c[4] = {0, 0, 0, 0};
  mma_k4(c, a, b);
  C[g * 8 + 2 * t] = c[0]; C[g * 8 + 2 * t + 1] = c[1];
  C[(g + 8) * 8 + 2 * t] = c[2]; C[(g + 8) * 8 + 2 * t + 1] = c[3];
}
// k8: a[v0 + 2 v1] = A[g + 8 v0][t + 4 v1], b[v] = B[t + 4 v][g]
__global__ void layout_k8(const double* A, const double* B, double* C) {
  int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a[4] = {A[g * 8 + t], A[(g + 8) * 8 + t], A[g * 8 + t + 4], A[(g + 8) * 8 + t + 4]};
  double b[2] = {B[t * 8 + g], B[(t + 4) * 8 + g]};
  double c[4] = {0, 0, 0, 0};
  mma_k8(c, a, b);
  C[g * 8 + 2 * t] = c[0]; C[g * 8 + 2 * t + 1] = c[1];
  C[(g + 8) * 8 + 2 * t] = c[2]; C[(g + 8) * 8 + 2 * t + 1] = c[3];
}

template <int KIND>
__global__ void tput(double* out, int iters) {
  double c[8][4];
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  double a[4] = {1.0 + threadIdx.x * 1e-9, 1.0, 1.0, 1.0}, b[2] = {1e-9, 1e-9};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 4) mma_k4(c[i], a, b[0]); else mma_k8(c[i], a, b);
    }
  }
  double s = 0; for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.0) out[0] = s;
}
__global__ void tput_dfma(double* out, int iters) {
  double c[16];
  for (int i = 0; i < 16; ++i) c[i] = threadIdx.x;
  double a = 1.0000001, b = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0; for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double hA[128], hB[64], hC[128], *dA, *dB, *dC;
  srand(1);
  for (int i = 0; i < 128; ++i) hA[i] = rand() % 7 - 3;
  for (int i = 0; i < 64; ++i) hB[i] = rand() % 5 - 2;
  cudaMalloc(&dA, 1024); cudaMalloc(&dB, 1024); cudaMalloc(&dC, 1024);
  cudaMemcpy(dA, hA, 1024, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, 512, cudaMemcpyHostToDevice);
  for (int K : {4, 8}) {
    if (K == 4) layout_k4<<<1, 32>>>(dA, dB, dC); else layout_k8<<<1, 32>>>(dA, dB, dC);
    cudaMemcpy(hC, dC, 1024, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < 16; ++m) for (int n = 0; n < 8; ++n) {
      double r = 0; for (int k = 0; k < K; ++k) r += hA[m * K + k] * hB[k * 8 + n];
      if (r != hC[m * 8 + n]) ++bad;
    }
    printf("layout k%d: %s (%d bad)\n", K, bad ? "MISMATCH" : "ok", bad);
  }
  int dev; cudaGetDevice(&dev); cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int sms = p.multiProcessorCount;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    for (int warps : {4, 8, 16}) {
      float ms;
      cudaEventRecord(e0); tput<4><<<sms * 2, warps * 32>>>(dC, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double fl = double(sms) * 2 * warps * iters * 8 * 1024.0;
      printf("dmma k4 warps/cta=%d: %.2f TFLOP/s\n", warps, fl / ms / 1e9);
      cudaEventRecord(e0); tput<8><<<sms * 2, warps * 32>>>(dC, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("dmma k8 warps/cta=%d: %.2f TFLOP/s\n", warps, 2 * fl / ms / 1e9);
      cudaEventRecord(e0); tput_dfma<<<sms * 2, warps * 32>>>(dC, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("dfma warps/cta=%d: %.2f TFLOP/s\n", warps, double(sms) * 2 * warps * 32 * iters * 16 * 2.0 / ms / 1e9);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
