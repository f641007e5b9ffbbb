// Probe: TMA-staged large-tile GEMM (k_tma.cu) vs the cp.async kernels (k_gemm.cu):
// results on random data (max |diff| relative to |C|) and throughput per shape.
#include "../../paper_1302_5995_b200/csrc/k_gemm.cu"
#include "../../paper_1302_5995_b200/csrc/k_tma.cu"
#include <cstdio>
#include <random>
#include <vector>
#include <cmath>
using namespace dtnb;
int main() {
  gemm_init();
  printf("tma init: %s, enabled %d\n", cudaGetErrorString(gemm_tma_init()), int(gemm_tma_enabled()));
  struct Case { int m, n, k; };
  for (int upd = 0; upd < 2; ++upd)
  for (Case cs : {Case{1000, 777, 70}, Case{1916, 2044, 128}, Case{2044, 2044, 1020}, Case{4096, 4096, 2048}, Case{8188, 4096, 8188}, Case{16380, 16380, 510}}) {
    const size_t ldA = (cs.m + 7) / 8 * 8, ldB = (cs.k + 1) / 2 * 2, ldC = (cs.m + 1) / 2 * 2;
    double *A, *B, *C, *C2, *C0;
    cudaMalloc(&A, ldA * cs.k * 8); cudaMalloc(&B, ldB * cs.n * 8); cudaMalloc(&C, ldC * cs.n * 8);
    cudaMalloc(&C2, ldC * cs.n * 8); cudaMalloc(&C0, ldC * cs.n * 8);
    std::mt19937_64 rng(7);
    auto fill = [&](double* dptr, size_t cnt) {
      std::vector<double> h(cnt);
      for (auto& x : h) x = double(rng() >> 11) * 0x1.0p-53 - 0.5;
      cudaMemcpy(dptr, h.data(), cnt * 8, cudaMemcpyHostToDevice);
    };
    fill(A, ldA * cs.k); fill(B, ldB * cs.n); fill(C0, ldC * cs.n);
    GemmDesc d{A, B, C, cs.m, cs.n, cs.k, int(ldA), int(ldB), int(ldC)};
    GemmDesc d2 = d; d2.C = C2;
    GemmDesc* dd; cudaMalloc(&dd, 2 * sizeof(d));
    cudaMemcpy(dd, &d, sizeof(d), cudaMemcpyHostToDevice); cudaMemcpy(dd + 1, &d2, sizeof(d), cudaMemcpyHostToDevice);
    std::vector<CUtensorMap> maps; std::vector<char> ok;
    tma_encode_descs(&d2, 1, maps, ok);
    CUtensorMap* dm; cudaMalloc(&dm, maps.size() * sizeof(CUtensorMap));
    cudaMemcpy(dm, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice);
    const double al = upd ? -1.0 : 1.0, be = upd ? 1.0 : 0.0;
    const int tiles = gemm_tiles(cs.m, cs.n);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best[2] = {1e9f, 1e9f};
    for (int which = 0; which < 2; ++which)
      for (int r = 0; r < 5; ++r) {
        cudaMemcpy(which ? C2 : C, C0, ldC * cs.n * 8, cudaMemcpyDeviceToDevice);
        cudaEventRecord(e0);
        if (which == 0) launch_gemm_desc(dd, 1, tiles, cs.k, al, be, 0, true, true);
        else if (ok[0]) launch_gemm_tma(dd + 1, dm, 1, tiles, al, be, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best[which]) best[which] = ms;
      }
    std::vector<double> h1(ldC * cs.n), h2(ldC * cs.n);
    cudaMemcpy(h1.data(), C, h1.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2.data(), C2, h2.size() * 8, cudaMemcpyDeviceToHost);
    double md = 0, mx = 0;
    for (int c = 0; c < cs.n; ++c) for (int r = 0; r < cs.m; ++r) {
      md = std::fmax(md, std::fabs(h1[r + c * ldC] - h2[r + c * ldC])); mx = std::fmax(mx, std::fabs(h1[r + c * ldC])); }
    const double fl = 2.0 * cs.m * cs.n * double(cs.k);
    printf("%s m %5d n %5d k %5d ok %d: cp.async %.3f ms %.2f TF/s | TMA %.3f ms %.2f TF/s | max diff %.2e (|C| %.2e) %s\n",
           upd ? "C-=AB" : "C=AB ", cs.m, cs.n, cs.k, int(ok[0]), best[0], fl / best[0] / 1e9, best[1], fl / best[1] / 1e9, md, mx,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(C2); cudaFree(C0); cudaFree(dd); cudaFree(dm);
  }
  return 0;
}
