// Probe: device time of the batched block substitution kernel vs shape.
#define TS_PROFILE
#include "../../paper_1302_5995_b200/csrc/k_misc.cu"
#include <cstdio>
#include <vector>
#include <random>
using namespace dtnb;
int main() {
  misc_init();
  struct Case { int bk, ncols, count; };
  for (Case cs : {Case{128, 128, 16}, Case{128, 2044, 1}, Case{128, 2044, 2}, Case{64, 256, 256}, Case{128, 1020, 8}}) {
    const int ld = 2048 + 128;
    std::vector<double> hU(size_t(ld) * 128);
    std::mt19937_64 rng(1);
    for (size_t i = 0; i < hU.size(); ++i) hU[i] = double(rng() >> 11) * 0x1.0p-53 - 0.5;
    for (int i = 0; i < 128; ++i) hU[i + size_t(i) * ld] += 8.0;
    double *dU, *dY;
    cudaMalloc(&dU, hU.size() * 8);
    cudaMalloc(&dY, size_t(ld) * cs.ncols * cs.count * 8);
    cudaMemcpy(dU, hU.data(), hU.size() * 8, cudaMemcpyHostToDevice);
    cudaMemset(dY, 0, size_t(ld) * cs.ncols * cs.count * 8);
    std::vector<TrsmDesc> hd;
    for (int i = 0; i < cs.count; ++i) hd.push_back(TrsmDesc{dU, dY + size_t(ld) * cs.ncols * i, ld, ld, cs.bk, cs.ncols});
    TrsmDesc* dd; cudaMalloc(&dd, hd.size() * sizeof(TrsmDesc));
    cudaMemcpy(dd, hd.data(), hd.size() * sizeof(TrsmDesc), cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(e0);
      launch_trsm_batched(dd, cs.count, cs.ncols, cs.bk, false, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (r > 0 && ms < best) best = ms;
    }
    printf("bk %3d ncols %5d count %4d: %.1f us  (%s)\n", cs.bk, cs.ncols, cs.count, best * 1e3, cudaGetErrorString(cudaGetLastError()));
    long long c[16]; cudaMemcpyFromSymbol(c, g_ts_clk, sizeof(c));
    printf("   load %lld |", c[1] - c[0]);
    for (int i = 2; i < 10; ++i) printf(" %lld", c[i] - c[i - 1]);
    printf(" | end %lld\n", c[15] - c[9]);
    cudaFree(dU); cudaFree(dY); cudaFree(dd);
  }
  return 0;
}
