// Probe: device time of one panel launch (kb = 32) vs rows / cluster size.
#define DTN_PANEL_PROFILE
#include "../../paper_1302_5995_b200/csrc/k_blocked.cu"
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
using namespace dtnb;
int main() {
  {
    cudaFuncAttributes fb;
    printf("getattr panel2<true,1>: %s\n", cudaGetErrorString(cudaFuncGetAttributes(&fb, panel2_kernel<true, 1>)));
    printf("  regs %d\n", fb.numRegs);
    printf("set nonport panel2<true,1>: %s\n", cudaGetErrorString(cudaFuncSetAttribute(panel2_kernel<true, 1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)));
    printf("set nonport panel2<true,2>: %s\n", cudaGetErrorString(cudaFuncSetAttribute(panel2_kernel<true, 2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)));
    printf("set dyn panel2<false,1>: %s\n", cudaGetErrorString(cudaFuncSetAttribute(panel2_kernel<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(panel_dyn_smem(1)))));
    cudaError_t e = blocked_init();
    printf("blocked_init: %s\n", cudaGetErrorString(e));
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, panel2_kernel<false, 1>);
    printf("panel2<false,1>: regs %d static smem %zu max dyn %d maxthreads %d\n", fa.numRegs, fa.sharedSizeBytes,
           fa.maxDynamicSharedSizeBytes, fa.maxThreadsPerBlock);
    cudaFuncGetAttributes(&fa, panel_kernel<false, 1>);
    printf("panel<false,1>: regs %d static smem %zu max dyn %d maxthreads %d\n", fa.numRegs, fa.sharedSizeBytes,
           fa.maxDynamicSharedSizeBytes, fa.maxThreadsPerBlock);
  }
  for (int kbv : {32})
  for (int rows : {256, 512, 1024, 2048, 4096}) {
    const int n = rows, ld = (n + 7) / 8 * 8;
    NodeDev nd{};
    nd.kind = 2; nd.ni = n; nd.nb = 0; nd.total = n; nd.ncols = n; nd.ld = nd.ldm = ld; nd.a = nd.b = -1;
    NodeDev* dn; int* dl; double* da; double* db; int* dp; double* ds;
    cudaMalloc(&dn, sizeof(nd)); cudaMalloc(&dl, 4); cudaMalloc(&da, sizeof(double) * ld * 64);
    cudaMalloc(&db, sizeof(double) * ld * 64); cudaMalloc(&dp, 4 * (n + 200)); cudaMalloc(&ds, 16);
    int zero = 0;
    cudaMemcpy(dn, &nd, sizeof(nd), cudaMemcpyHostToDevice); cudaMemcpy(dl, &zero, 4, cudaMemcpyHostToDevice);
    std::vector<double> h(size_t(ld) * 64);
    std::mt19937_64 rng(1);
    for (auto& x : h) x = double(rng() >> 11) * 0x1.0p-53 - 0.5;
    cudaMemcpy(db, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    KernelArgs a{dn, nullptr, nullptr, 0, 0, da, dp, ds};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9, tot = 0; int reps = 20;
    for (int r = 0; r < reps + 2; ++r) {
      cudaMemcpy(da, db, h.size() * 8, cudaMemcpyDeviceToDevice);
      cudaEventRecord(e0);
      cudaError_t err = launch_panel(a, dl, 1, n, 0, kbv, 0, false);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      if (err != cudaSuccess) { printf("err %s\n", cudaGetErrorString(err)); return 1; }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 2) { best = ms < best ? ms : best; tot += ms; }
    }
    { long long q[16]; cudaMemcpyFromSymbol(q, g_p2_clk, sizeof(q));
      printf("  pivoted loop (per step, avg over the last launch x reps): argmax+publish %lld sync %lld cta-argmax+push %lld mbar-wait %lld cluster-argmax+rcp %lld update %lld\n",
             q[9] / (32 * (reps + 2)), q[10] / (32 * (reps + 2)), q[11] / (32 * (reps + 2)), q[12] / (32 * (reps + 2)), q[13] / (32 * (reps + 2)), q[14] / (32 * (reps + 2)));
      long long z[16] = {0}; cudaMemcpyToSymbol(g_p2_clk, z, sizeof(z)); }
    int rpt, cs; panel_shape(n, &rpt, &cs);
    printf("rpt %d kb %2d rows %5d csize %2d: best %.1f us, mean %.1f us (%.2f us/column)\n", rpt, kbv, n, cs, best * 1e3, tot / reps * 1e3,
           best * 1e3 / kbv);
  {
      long long h[256];
      cudaMemcpyFromSymbol(h, g_panel_clk, sizeof(h));
      printf("phases: redux | publish | barrier | pivot-decide | rcp | update | rotate | next\n");
      for (int j = 0; j < 32; j += 4) {
        printf("col %2d:", j);
        for (int q = 1; q < 8; ++q) printf(" %5lld", h[j*8+q]-h[j*8+q-1]);
        printf(" %5lld\n", j < 31 ? h[(j+1)*8]-h[j*8+7] : 0LL);
      }
    }
  
  }
  // diagonally dominant panels: the no-interchange fast path succeeds
  for (int rows : {256, 512, 1024, 2048, 4096}) {
    const int n = rows, ld = (n + 7) / 8 * 8;
    NodeDev nd{};
    nd.kind = 2; nd.ni = n; nd.nb = 0; nd.total = n; nd.ncols = n; nd.ld = nd.ldm = ld; nd.a = nd.b = -1;
    NodeDev* dn; int* dl; double* da; double* db; int* dp; double* ds;
    cudaMalloc(&dn, sizeof(nd)); cudaMalloc(&dl, 4); cudaMalloc(&da, sizeof(double) * ld * 32);
    cudaMalloc(&db, sizeof(double) * ld * 32); cudaMalloc(&dp, 4 * (n + 300)); cudaMalloc(&ds, 16);
    int zero = 0;
    cudaMemcpy(dn, &nd, sizeof(nd), cudaMemcpyHostToDevice); cudaMemcpy(dl, &zero, 4, cudaMemcpyHostToDevice);
    std::vector<double> h(size_t(ld) * 32);
    std::mt19937_64 rng(1);
    for (auto& x : h) x = double(rng() >> 11) * 0x1.0p-53 - 0.5;
    for (int i = 0; i < 32; ++i) h[i + size_t(i) * ld] = 4.0 * n;
    cudaMemcpy(db, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    KernelArgs a{dn, nullptr, nullptr, 0, 0, da, dp, ds};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < 12; ++r) {
      cudaMemcpy(da, db, h.size() * 8, cudaMemcpyDeviceToDevice);
      cudaEventRecord(e0);
      launch_panel(a, dl, 1, n, 0, 32, 0, false);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 2) best = ms < best ? ms : best;
    }
    int piv[32]; cudaMemcpy(piv, dp, sizeof(piv), cudaMemcpyDeviceToHost);
    int moved = 0; for (int i = 0; i < 32; ++i) moved += piv[i] != i;
    { long long q[16]; cudaMemcpyFromSymbol(q, g_p2_clk, sizeof(q));
      printf("  p2 clk: load %lld save %lld topLU %lld ubsync %lld subst %lld check %lld final %lld tail %lld\n", q[1]-q[0], q[2]-q[1], q[3]-q[2], q[4]-q[3], q[5]-q[4], q[6]-q[5], q[7]-q[6], q[8]-q[7]); }
    long long pc[8]; cudaMemcpyFromSymbol(pc, g_pro_clk, sizeof(pc));
    printf("diag-dominant rows %5d: best %.1f us (rows moved %d) %s | start->save %lld topLU %lld subst %lld check %lld\n", n, best * 1e3, moved,
           cudaGetErrorString(cudaGetLastError()), pc[4] - pc[3], pc[5] - pc[4], pc[6] - pc[5], pc[7] - pc[6]);
  }
  // fused prologue: panel(32) after panel(0), with and without the prologue
  for (int rows : {256, 512, 1024, 2048, 4096}) {
    const int n = rows, ld = (n + 7) / 8 * 8;
    NodeDev nd{};
    nd.kind = 2; nd.ni = n; nd.nb = 0; nd.total = n; nd.ncols = n; nd.ld = nd.ldm = ld; nd.a = nd.b = -1;
    NodeDev* dn; int* dl; double* da; double* db; int* dp; double* ds;
    cudaMalloc(&dn, sizeof(nd)); cudaMalloc(&dl, 4); cudaMalloc(&da, sizeof(double) * ld * 64);
    cudaMalloc(&db, sizeof(double) * ld * 64); cudaMalloc(&dp, 4 * (n + 300)); cudaMalloc(&ds, 16);
    int zero = 0;
    cudaMemcpy(dn, &nd, sizeof(nd), cudaMemcpyHostToDevice); cudaMemcpy(dl, &zero, 4, cudaMemcpyHostToDevice);
    std::vector<double> h(size_t(ld) * 64);
    std::mt19937_64 rng(1);
    for (auto& x : h) x = double(rng() >> 11) * 0x1.0p-53 - 0.5;
    const bool dd = getenv("PROBE_DIAG") != nullptr;  // diagonally dominant: the fast path succeeds
    if (dd) for (int i = 0; i < 64; ++i) h[i + size_t(i) * ld] = 4.0 * n;
    cudaMemcpy(db, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    KernelArgs a{dn, nullptr, nullptr, 0, 0, da, dp, ds};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int fused = 0; fused < 2; ++fused) {
      float best = 1e9;
      for (int r = 0; r < 12; ++r) {
        cudaMemcpy(da, db, h.size() * 8, cudaMemcpyDeviceToDevice);
        launch_panel(a, dl, 1, n, 0, 32, 0, false);
        cudaEventRecord(e0);
        cudaError_t err = launch_panel(a, dl, 1, n - 32, 32, 32, 0, fused);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        if (err != cudaSuccess) { printf("err %s\n", cudaGetErrorString(err)); return 1; }
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (r >= 2) best = ms < best ? ms : best;
      }
      { long long q[16]; cudaMemcpyFromSymbol(q, g_p2_clk, sizeof(q));
        printf("  p2 clk: load+prologue %lld save %lld topLU %lld ubsync %lld subst %lld check %lld final %lld tail %lld\n", q[1]-q[0], q[2]-q[1], q[3]-q[2], q[4]-q[3], q[5]-q[4], q[6]-q[5], q[7]-q[6], q[8]-q[7]);
        long long w[16]; cudaMemcpyFromSymbol(w, g_p2b_clk, sizeof(w));
        printf("  last thread of the last CTA: load+prologue %lld save %lld (wait for top LU) %lld ubsync %lld subst %lld check %lld final %lld tail %lld | vs thread 0: start %+lld end %+lld\n", w[1]-w[0], w[2]-w[1], w[3]-w[2], w[4]-w[3], w[5]-w[4], w[6]-w[5], w[7]-w[6], w[8]-w[7], w[0]-q[0], w[8]-q[8]); }
      long long pc[8];
      cudaMemcpyFromSymbol(pc, g_pro_clk, sizeof(pc));
      printf("rows %5d panel(k0=32) fused=%d%s: best %.1f us  prologue clk: loads %lld solve %lld update %lld | save %lld topLU %lld subst %lld check %lld\n", n,
             fused, dd ? " diag" : "", best * 1e3, pc[1] - pc[0], pc[2] - pc[1], pc[3] - pc[2], pc[4] - pc[3], pc[5] - pc[4], pc[6] - pc[5], pc[7] - pc[6]);
    }
  }
  // empty-ish launch overhead reference
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
}
