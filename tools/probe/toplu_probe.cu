// Probe: the no-interchange top-block LU of a 32 x 32 panel by ONE warp (panel2's fast
// path), variants: (a) smem publish + __syncwarp + broadcast loads (panel2), (b) the
// pivot row broadcast by shuffles, (c) (a) without the multiplier stores.
#include <cstdio>
#include <type_traits>
constexpr int PKB = 32, PLD = 34;
template <int W>
__device__ __forceinline__ void shift_w(double (&w)[PKB], double l, const double* __restrict__ prow) {
  const double2* p2 = reinterpret_cast<const double2*>(prow);
#pragma unroll
  for (int c2 = 0; c2 < W / 2; ++c2) {
    const double2 u = p2[c2];
    if (c2 > 0) w[2 * c2 - 1] = fma(-l, u.x, w[2 * c2]);
    w[2 * c2] = fma(-l, u.y, w[2 * c2 + 1]);
  }
  w[W - 1] = 0.0;
}
template <int V>
__global__ void toplu(double* M, long long* cyc, int reps) {
  __shared__ __align__(16) double ub[PKB * PLD];
  __shared__ double urinv[PKB];
  const int lane = threadIdx.x;
  double v[PKB];
  long long tot = 0;
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int c = 0; c < PKB; ++c) v[c] = (lane == c ? 64.0 : 0.0) + 1e-3 * ((lane * 7 + c * 3) % 11);
    __syncwarp();
    const long long t0 = clock64();
    double rnext = __drcp_rn(v[0]);
    auto chunk = [&](auto Wc) {
      constexpr int W = decltype(Wc)::value;
      const int j0 = PKB - W, j1 = j0 + 8;
      for (int j = j0; j < j1; ++j) {
        if constexpr (V == 1) {
          double u[W];
#pragma unroll
          for (int c = 0; c < W; ++c) u[c] = __shfl_sync(0xffffffffu, v[c], j);
          const double ri = __shfl_sync(0xffffffffu, rnext, j);
          if (lane > j) {
            const double l = v[0] * ri;
            M[lane + j * 64] = l;
#pragma unroll
            for (int c = 1; c < W; ++c) v[c - 1] = fma(-l, u[c], v[c]);
            v[W - 1] = 0.0;
            rnext = __drcp_rn(v[0]);
          }
        } else {
          if (lane == j) {
#pragma unroll
            for (int c = 0; c < W; c += 2) *reinterpret_cast<double2*>(ub + j * PLD + c) = make_double2(v[c], v[c + 1]);
            urinv[j] = rnext;
          }
          __syncwarp();
          if (lane > j) {
            const double l = v[0] * urinv[j];
            if (V == 0) M[lane + j * 64] = l;
            shift_w<W>(v, l, ub + j * PLD);
            rnext = __drcp_rn(v[0]);
          }
        }
      }
    };
    long long ta = clock64();
    chunk(std::integral_constant<int, 32>{});
    long long tb = clock64();
    chunk(std::integral_constant<int, 24>{});
    long long tc = clock64();
    chunk(std::integral_constant<int, 16>{});
    long long td = clock64();
    chunk(std::integral_constant<int, 8>{});
    __syncwarp();
    long long te = clock64();
    tot += te - t0;
    if (lane == 0 && r == reps - 1) { cyc[8 + 4 * V] = tb - ta; cyc[9 + 4 * V] = tc - tb; cyc[10 + 4 * V] = td - tc; cyc[11 + 4 * V] = te - td; }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < PKB; ++c) s += v[c];
  M[4096 + lane] = s;
  if (lane == 0) cyc[V] = tot / reps;
}
int main() {
  double* M;
  long long* c;
  cudaMalloc(&M, 8 * 8192);
  cudaMalloc(&c, 8 * 32);
  toplu<0><<<1, 32>>>(M, c, 20);
  toplu<1><<<1, 32>>>(M, c, 20);
  toplu<2><<<1, 32>>>(M, c, 20);
  long long h[32];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  for (int v = 0; v < 3; ++v) printf("variant %d chunks (8 steps each, W=32/24/16/8): %lld %lld %lld %lld\n", v, h[8 + 4 * v], h[9 + 4 * v], h[10 + 4 * v], h[11 + 4 * v]);
  printf("top LU 32x32, one warp: smem %lld cycles, shuffles %lld, smem without stores %lld (%s)\n", h[0], h[1], h[2],
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
