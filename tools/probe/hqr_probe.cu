// Probe: sketch-QR kernels (hqr_kernel / hqr1_kernel / hqrb_kernel) on random tall
// matrices of the structured-merge shapes; device time per launch, orthogonality and
// factorization residuals checked on the host. HQRB_PROFILE: per-phase clocks.
#include "../../paper_1302_5995_b200/csrc/k_struct.cu"
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
using namespace dtnb;
int main(int argc, char** argv) {
  struct_init();
  for (int C : {1, 2, 4, 8, 16})
    for (int kb : {60, 100, 120, 200}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(C * 64);
      cfg.blockDim = dim3(256);
      cfg.dynamicSmemBytes = size_t(kb) * 1024;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = C;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int nclus = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&nclus, C > 1 ? (void*)hqrb_kernel<true> : (void*)hqrb_kernel<false>, &cfg);
      printf("cluster %2d smem %3d KB: max active clusters %d (%s)\n", C, kb, nclus, cudaGetErrorString(e));
    }
  const bool piv = getenv("PIV") != nullptr;
  const int shapes_t[][4] = {{64, 254, 64, 4}, {16, 510, 152, 4}, {8, 510, 152, 4}, {4, 1022, 80, 4}};
  const int shapes_p[][4] = {{128, 64, 64, 16}, {64, 49, 49, 16}, {8, 73, 73, 16}, {4, 89, 89, 16}};
  for (auto& sh : piv ? shapes_p : shapes_t) {
    const int count = sh[0], m = sh[1], n = sh[2], p = sh[3], nc = n + p, ld = m + 2;
    std::vector<double> hY(size_t(ld) * nc * count);
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<double> U(-1, 1);
    // low-rank-ish: Y = A B with decaying spectrum + noise
    for (int q = 0; q < count; ++q)
      for (int j = 0; j < nc; ++j)
        for (int i = 0; i < m; ++i) {
          double s = 0;
          for (int k = 0; k < 8; ++k) s += std::pow(0.2, k) * std::sin(0.1 * (k + 1) * (i + 1) + 0.37 * j * (k + 1));
          hY[size_t(q) * ld * nc + i + size_t(j) * ld] = s + 1e-6 * U(rng);
        }
    double *dY, *dY0, *dQ, *dstat, *deps;
    cudaMalloc(&dY, hY.size() * 8);
    cudaMalloc(&dY0, hY.size() * 8);
    cudaMalloc(&dQ, size_t(ld) * n * count * 8);
    cudaMalloc(&dstat, 2 * count * 8);
    cudaMalloc(&deps, 8);
    double eps = 1e-10;
    cudaMemcpy(deps, &eps, 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dY0, hY.data(), hY.size() * 8, cudaMemcpyHostToDevice);
    std::vector<QrDesc> hd(count);
    for (int q = 0; q < count; ++q)
      hd[q] = QrDesc{dY + size_t(q) * ld * nc, dQ + size_t(q) * ld * n, dstat + 2 * q, nullptr, ld, ld, m, n, p, 0, 0, 0};
    QrDesc* dd;
    cudaMalloc(&dd, count * sizeof(QrDesc));
    cudaMemcpy(dd, hd.data(), count * sizeof(QrDesc), cudaMemcpyHostToDevice);
    {
      const char* mode = getenv("DTN_HQR_BLOCKED") ? getenv("DTN_HQR_BLOCKED") : "1";
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      float best = 1e9;
      for (int r = 0; r < 5; ++r) {
        cudaMemcpy(dY, dY0, hY.size() * 8, cudaMemcpyDeviceToDevice);
        cudaEventRecord(e0);
        cudaError_t err = launch_hqr(dd, count, m, nc, deps, 0, piv);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) {
          printf("launch error %s\n", cudaGetErrorString(err));
          return 1;
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
      }
      std::vector<double> hQ(size_t(ld) * n), hs(2);
      cudaMemcpy(hQ.data(), dQ, hQ.size() * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(hs.data(), dstat, 16, cudaMemcpyDeviceToHost);
      double orth = 0, resid = 0, ynrm = 0;
      for (int a = 0; a < n; ++a)
        for (int b = 0; b <= a; ++b) {
          double s = 0;
          for (int i = 0; i < m; ++i) s += hQ[i + size_t(a) * ld] * hQ[i + size_t(b) * ld];
          orth = std::max(orth, std::fabs(s - (a == b)));
        }
      for (int j = 0; j < n; ++j) {  // |(I - Q Q^T) y_j|
        std::vector<double> c(n, 0.0);
        for (int a = 0; a < n; ++a)
          for (int i = 0; i < m; ++i) c[a] += hQ[i + size_t(a) * ld] * hY[i + size_t(j) * ld];
        for (int i = 0; i < m; ++i) {
          double r = hY[i + size_t(j) * ld];
          for (int a = 0; a < n; ++a) r -= hQ[i + size_t(a) * ld] * c[a];
          resid = std::max(resid, std::fabs(r));
          ynrm = std::max(ynrm, std::fabs(hY[i + size_t(j) * ld]));
        }
      }
      printf("count %3d m %4d n %3d: %s %.1f us  |Q^TQ - I| %.2e  |(I-QQ^T)Y|/|Y| %.2e  rank %g tail %.2e\n", count, m, n,
             mode[0] == '0' ? "unblocked" : "blocked  ", best * 1e3, orth, resid / ynrm, hs[0], hs[1]);
#ifdef HQRB_PROFILE
      cudaMemcpy(dY, dY0, hY.size() * 8, cudaMemcpyDeviceToDevice);
      { long long z[16] = {0}; cudaMemcpyToSymbol(g_hqrb_clk, z, sizeof(z)); }
      launch_hqr(dd, count, m, nc, deps, 0, piv);
      cudaDeviceSynchronize();
      long long h[16];
      cudaMemcpyFromSymbol(h, g_hqrb_clk, sizeof(h));
      {
        std::vector<unsigned long long> t(2 * 2048);
        cudaMemcpyFromSymbol(t.data(), g_hqrb_t, t.size() * 8);
        unsigned long long s0 = ~0ull, s1 = 0, e0 = ~0ull, e1 = 0;
        int nb = 0;
        for (int b = 0; b < 2048; ++b)
          if (t[2 * b]) { ++nb; s0 = std::min(s0, t[2*b]); s1 = std::max(s1, t[2*b]); e0 = std::min(e0, t[2*b+1]); e1 = std::max(e1, t[2*b+1]); }
        printf("   blocks %d: start spread %.1f us, end spread %.1f us, span %.1f us\n", nb, (s1 - s0) * 1e-3, (e1 - e0) * 1e-3, (e1 - s0) * 1e-3);
        std::vector<unsigned long long> z(2 * 2048, 0);
        cudaMemcpyToSymbol(g_hqrb_t, z.data(), z.size() * 8);
      }
      printf("   clk: panel-steps %lld  W+reduce %lld  dlarft %lld  update %lld  probe %lld  Q %lld | piv: load %lld argmax %lld swap %lld refl+upd %lld Q %lld\n", h[1], h[2], h[3], h[4],
             h[5], h[6], h[7], h[8], h[9], h[10], h[11]);
#endif
    }
  }
  return 0;
}
