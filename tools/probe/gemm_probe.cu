// Probe: descriptor GEMM throughput (C -= A B, FP64 DMMA) vs shape.
#include "../../paper_1302_5995_b200/csrc/k_gemm.cu"
#include <cstdio>
#include <vector>
using namespace dtnb;
int main() {
  gemm_init();
  struct Case { int m, n, k; };
  for (int upd = 0; upd < 2; ++upd)
  for (Case cs : {Case{2044, 2044, 1020}, Case{4096, 4096, 2048}, Case{8188, 4096, 8188}, Case{1916, 2044, 128}}) {
    const size_t ldA = (cs.m + 7) / 8 * 8, ldB = (cs.k + 1) / 2 * 2, ldC = (cs.m + 1) / 2 * 2;
    double *A, *B, *C;
    cudaMalloc(&A, ldA * cs.k * 8); cudaMalloc(&B, ldB * cs.n * 8); cudaMalloc(&C, ldC * cs.n * 8);
    cudaMemset(A, 0, ldA * cs.k * 8); cudaMemset(B, 0, ldB * cs.n * 8); cudaMemset(C, 0, ldC * cs.n * 8);
    GemmDesc d{A, B, C, cs.m, cs.n, cs.k, int(ldA), int(ldB), int(ldC)};
    GemmDesc* dd; cudaMalloc(&dd, sizeof(d)); cudaMemcpy(dd, &d, sizeof(d), cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      if (upd) launch_gemm_desc(dd, 1, gemm_tiles(cs.m, cs.n), cs.k, -1.0, 1.0, 0, true);
      else launch_gemm_desc(dd, 1, gemm_tiles(cs.m, cs.n), cs.k, 1.0, 0.0, 0, true);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (r > 0 && ms < best) best = ms;
    }
    printf("%s m %5d n %5d k %5d: %.3f ms  %.2f TF/s (%s)\n", upd ? "C-=AB" : "C=AB ", cs.m, cs.n, cs.k, best, 2.0 * cs.m * cs.n * double(cs.k) / (best * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(dd);
  }
  return 0;
}
