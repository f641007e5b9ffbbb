// FP64 tensor-core GEMM (DMMA: mma.sync m16n8k4 .f64) for the merge
// trailing updates, the root-inverse triangular sweeps and the batched solve.
// CTA tile BM x BN, K staged through shared memory in BK chunks with a
// two-stage cp.async pipeline; 8 warps, each owning a WM x WN accumulator
// tile in registers (FP64 has no tcgen05/TMEM path on sm_100a).
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "common.cuh"

namespace dtnb {

constexpr int GBM = 128, GBN = 64, GWM = 32, GWN = 32;
constexpr int GTHREADS = (GBM / GWM) * (GBN / GWN) * 32;  // 256
constexpr int GPA = 4;                                    // A smem row pad (bank-conflict free frags)
// B smem leading dim: == 4 mod 16 (bank-conflict-free fragments), >= BK
template <int BK>
constexpr int gemm_ldb() { return BK <= 16 ? 20 : BK + 4; }

template <int BK>
struct GemmSmem {
  double a[2][BK][GBM + GPA];
  double b[2][GBN][gemm_ldb<BK>()];
};

// One BM x BN tile of C = alpha*A*B + beta*C (any alpha, beta; (-1, 1) is UPD):
// UPD (C -= A*B) preloads the C tile into the accumulators before the K loop
// (its latency overlaps the first A/B stage) and feeds -A to the DMMA, so the
// epilogue is a plain store. Requires 16-byte aligned B columns.
// AT (two-source A, the HBS apply's leaf steps): the first ka columns of A
// come from A stored row-major (A(r, c) = A[c + r lda]: the vectors X read
// transposed, no transpose pass), the rest from the column-major A2 (lda2);
// ka must be a multiple of BK.
template <int BK, bool A16 = true, bool UPD = false, bool TC = false, bool AT = false>
__device__ __forceinline__ void gemm_tile(const double* __restrict__ A, int lda, const double* __restrict__ B,
                                          int ldb, double* C, int ldc, int m, int n, int k, int tm, int tn,
                                          double alpha, double beta, GemmSmem<BK>& sm,
                                          const double* __restrict__ A2 = nullptr, int lda2 = 0, int ka = 0,
                                          int ka_valid = 0) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int wm0 = (warp % (GBM / GWM)) * GWM, wn0 = (warp / (GBM / GWM)) * GWN;
  const int row0 = tm * GBM, col0 = tn * GBN;
  const int KT = (k + BK - 1) / BK;

  auto load = [&](int stage, int kt) {
    const int kb0 = kt * BK;
    // A: BK columns x GBM rows, 2-double chunks along rows (1-double chunks
    // when A's columns are only 8-byte aligned)
    if (AT && kb0 < ka) {
      // row-major source: BK consecutive k of one row per BK threads (coalesced),
      // columns >= ka_valid of the first segment are zero (odd leaf sizes)
      constexpr int ACH = BK * GBM;
#pragma unroll
      for (int c = tid; c < ACH; c += GTHREADS) {
        const int rr = c / BK, kk = c % BK;
        const int gr = row0 + rr, gc = kb0 + kk;
        const bool ok = gc < ka_valid && gr < m;
        cp_async8(&sm.a[stage][kk][rr], ok ? A + gc + (long long)gr * lda : A, ok ? 8 : 0);
      }
    } else if (AT) {
      constexpr int ACH = BK * GBM / 2;
#pragma unroll
      for (int c = tid; c < ACH; c += GTHREADS) {
        const int kk = c / (GBM / 2), rr = (c % (GBM / 2)) * 2;
        const int gr = row0 + rr, gc = kb0 + kk;
        int bytes = 0;
        const double* src = A2;
        if (gc < k && gr < m) {
          bytes = (m - gr) >= 2 ? 16 : 8;
          src = A2 + gr + (long long)(gc - ka) * lda2;
        }
        cp_async16(&sm.a[stage][kk][rr], src, bytes);
      }
    } else if constexpr (A16) {
      constexpr int ACH = BK * GBM / 2;
#pragma unroll
      for (int c = tid; c < ACH; c += GTHREADS) {
        const int kk = c / (GBM / 2), rr = (c % (GBM / 2)) * 2;
        const int gr = row0 + rr, gc = kb0 + kk;
        int bytes = 0;
        const double* src = A;
        if (gc < k && gr < m) {
          bytes = (m - gr) >= 2 ? 16 : 8;
          src = A + gr + (long long)gc * lda;
        }
        cp_async16(&sm.a[stage][kk][rr], src, bytes);
      }
    } else {
      constexpr int ACH = BK * GBM;
#pragma unroll
      for (int c = tid; c < ACH; c += GTHREADS) {
        const int kk = c / GBM, rr = c % GBM;
        const int gr = row0 + rr, gc = kb0 + kk;
        const bool ok = gc < k && gr < m;
        cp_async8(&sm.a[stage][kk][rr], ok ? A + gr + (long long)gc * lda : A, ok ? 8 : 0);
      }
    }
    // B: GBN columns x BK rows, 2-double chunks along k
    constexpr int BCH = GBN * BK / 2;
#pragma unroll
    for (int c = tid; c < BCH; c += GTHREADS) {
      const int nn = c / (BK / 2), kp = (c % (BK / 2)) * 2;
      const int gk = kb0 + kp, gc = col0 + nn;
      int bytes = 0;
      const double* src = B;
      if (gc < n && gk < k) {
        bytes = (k - gk) >= 2 ? 16 : 8;
        src = B + gk + (long long)gc * ldb;
      }
      cp_async16(&sm.b[stage][nn][kp], src, bytes);
    }
    cp_async_commit();
  };

  double acc[GWM / 16][GWN / 8][4];
  if (KT > 0) load(0, 0);
#pragma unroll
  for (int i = 0; i < GWM / 16; ++i)
#pragma unroll
    for (int j = 0; j < GWN / 8; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        double x = 0.0;
        if constexpr (UPD) {
          const int r = row0 + wm0 + i * 16 + g + 8 * (v >> 1);
          const int c = col0 + wn0 + j * 8 + 2 * tig + (v & 1);
          if (r < m && c < n) x = C[r + (long long)c * ldc];
        }
        acc[i][j][v] = x;
      }
  for (int kt = 0; kt < KT; ++kt) {
    if (kt + 1 < KT) {
      load((kt + 1) & 1, kt + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int s = kt & 1;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      double af[GWM / 16][2], bf[GWN / 8];
#pragma unroll
      for (int i = 0; i < GWM / 16; ++i) {
        af[i][0] = sm.a[s][ks * 4 + tig][wm0 + i * 16 + g];
        af[i][1] = sm.a[s][ks * 4 + tig][wm0 + i * 16 + g + 8];
        if constexpr (UPD) {
          af[i][0] = -af[i][0];
          af[i][1] = -af[i][1];
        }
      }
#pragma unroll
      for (int j = 0; j < GWN / 8; ++j) bf[j] = sm.b[s][wn0 + j * 8 + g][ks * 4 + tig];
#pragma unroll
      for (int i = 0; i < GWM / 16; ++i)
#pragma unroll
        for (int j = 0; j < GWN / 8; ++j) mma_f64_m16n8k4(acc[i][j], af[i][0], af[i][1], bf[j]);
    }
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < GWM / 16; ++i) {
#pragma unroll
    for (int j = 0; j < GWN / 8; ++j) {
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int r = row0 + wm0 + i * 16 + g + 8 * (v >> 1);
        const int c = col0 + wn0 + j * 8 + 2 * tig + (v & 1);
        if (r < m && c < n) {
          // TC: C is stored transposed (element (r, c) at C[c + r * ldc])
          double* p = TC ? C + c + (long long)r * ldc : C + r + (long long)c * ldc;
          if constexpr (UPD) *p = acc[i][j][v];
          else *p = beta == 0.0 ? alpha * acc[i][j][v] : fma(alpha, acc[i][j][v], beta * *p);
        }
      }
    }
  }
}

template <int BK, bool UPD, bool A16, bool TC = false>
__global__ void __launch_bounds__(GTHREADS, 2) gemm_desc_kernel(const GemmDesc* __restrict__ descs, double alpha,
                                                             double beta) {
  extern __shared__ __align__(16) unsigned char gsm_raw[];
  GemmSmem<BK>& sm = *reinterpret_cast<GemmSmem<BK>*>(gsm_raw);
  const GemmDesc d = descs[blockIdx.y];
  const int tiles_m = (d.m + GBM - 1) / GBM, tiles_n = (d.n + GBN - 1) / GBN;
  const int t = blockIdx.x;
  if (t >= tiles_m * tiles_n) return;
  // B columns are always 16-byte aligned; A only when the launcher says so
  gemm_tile<BK, A16, UPD, TC>(d.A, d.lda, d.B, d.ldb, d.C, d.ldc, d.m, d.n, d.k, t % tiles_m, t / tiles_m, alpha,
                              beta, sm);
}

// Two-source A (see gemm_tile AT), C stored transposed or not.
template <int BK, bool TC>
__global__ void __launch_bounds__(GTHREADS) gemm_desc2_kernel(const GemmDesc2* __restrict__ descs) {
  extern __shared__ __align__(16) unsigned char gsm_raw[];
  GemmSmem<BK>& sm = *reinterpret_cast<GemmSmem<BK>*>(gsm_raw);
  const GemmDesc2 d = descs[blockIdx.y];
  const int tiles_m = (d.m + GBM - 1) / GBM, tiles_n = (d.n + GBN - 1) / GBN;
  const int t = blockIdx.x;
  if (t >= tiles_m * tiles_n) return;
  gemm_tile<BK, true, false, TC, true>(d.A, d.lda, d.B, d.ldb, d.C, d.ldc, d.m, d.n, d.k, t % tiles_m, t / tiles_m,
                                       1.0, 0.0, sm, d.A2, d.lda2, d.ka, d.ka_valid);
}

// ---- large-tile variant: 128 x 128 CTA tile, 8 warps of 64 x 32 (16 DMMA per
// k-step per warp: fragment loads per DMMA drop from 1 to 0.75), three-stage
// cp.async pipeline. For large GEMMs (Schur complements, root inverse, solve).
constexpr int XBM = 128, XBN = 128, XBK = 16, XST = 3, XWM = 64, XWN = 32;
constexpr int XLDB = XBK + 4;
struct GemmSmemX {
  double a[XST][XBK][XBM + GPA];
  double b[XST][XBN][XLDB];
};

template <bool UPD>
__global__ void __launch_bounds__(GTHREADS, 1) gemm_big_kernel(const GemmDesc* __restrict__ descs, double alpha,
                                                              double beta) {
  extern __shared__ __align__(16) unsigned char gsm_raw[];
  GemmSmemX& sm = *reinterpret_cast<GemmSmemX*>(gsm_raw);
  const GemmDesc d = descs[blockIdx.y];
  const int m = d.m, n = d.n, k = d.k;
  const int tiles_m = (m + XBM - 1) / XBM, tiles_n = (n + XBN - 1) / XBN;
  if (int(blockIdx.x) >= tiles_m * tiles_n) return;
  const int row0 = (blockIdx.x % tiles_m) * XBM, col0 = (blockIdx.x / tiles_m) * XBN;
  const double* A = d.A;
  const double* B = d.B;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int wm0 = (warp % (XBM / XWM)) * XWM, wn0 = (warp / (XBM / XWM)) * XWN;
  const int KT = (k + XBK - 1) / XBK;
  auto load = [&](int stage, int kt) {
    const int kb0 = kt * XBK;
#pragma unroll
    for (int c = tid; c < XBK * XBM / 2; c += GTHREADS) {  // A: 16-byte chunks along rows
      const int kk = c / (XBM / 2), rr = (c % (XBM / 2)) * 2;
      const int gr = row0 + rr, gc = kb0 + kk;
      int bytes = 0;
      const double* src = A;
      if (gc < k && gr < m) {
        bytes = (m - gr) >= 2 ? 16 : 8;
        src = A + gr + (long long)gc * d.lda;
      }
      cp_async16(&sm.a[stage][kk][rr], src, bytes);
    }
#pragma unroll
    for (int c = tid; c < XBN * XBK / 2; c += GTHREADS) {  // B: 16-byte chunks along k
      const int nn = c / (XBK / 2), kp = (c % (XBK / 2)) * 2;
      const int gk = kb0 + kp, gc = col0 + nn;
      int bytes = 0;
      const double* src = B;
      if (gc < n && gk < k) {
        bytes = (k - gk) >= 2 ? 16 : 8;
        src = B + gk + (long long)gc * d.ldb;
      }
      cp_async16(&sm.b[stage][nn][kp], src, bytes);
    }
  };
  double acc[XWM / 16][XWN / 8][4];
  if (KT > 0) load(0, 0);
  cp_async_commit();
  if (KT > 1) load(1, 1);
  cp_async_commit();
#pragma unroll
  for (int i = 0; i < XWM / 16; ++i)
#pragma unroll
    for (int j = 0; j < XWN / 8; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        double x = 0.0;
        if constexpr (UPD) {
          const int r = row0 + wm0 + i * 16 + g + 8 * (v >> 1);
          const int c = col0 + wn0 + j * 8 + 2 * tig + (v & 1);
          if (r < m && c < n) x = d.C[r + (long long)c * d.ldc];
        }
        acc[i][j][v] = x;
      }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<1>();  // stage kt has landed (kt + 1 may still be in flight)
    __syncthreads();     // ... for every thread, and stage (kt + 2) % 3 is free
    if (kt + 2 < KT) load((kt + 2) % XST, kt + 2);
    cp_async_commit();
    const int s = kt % XST;
#pragma unroll
    for (int ks = 0; ks < XBK / 4; ++ks) {
      double af[XWM / 16][2], bf[XWN / 8];
#pragma unroll
      for (int i = 0; i < XWM / 16; ++i) {
        af[i][0] = sm.a[s][ks * 4 + tig][wm0 + i * 16 + g];
        af[i][1] = sm.a[s][ks * 4 + tig][wm0 + i * 16 + g + 8];
        if constexpr (UPD) {
          af[i][0] = -af[i][0];
          af[i][1] = -af[i][1];
        }
      }
#pragma unroll
      for (int j = 0; j < XWN / 8; ++j) bf[j] = sm.b[s][wn0 + j * 8 + g][ks * 4 + tig];
#pragma unroll
      for (int i = 0; i < XWM / 16; ++i)
#pragma unroll
        for (int j = 0; j < XWN / 8; ++j) mma_f64_m16n8k4(acc[i][j], af[i][0], af[i][1], bf[j]);
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int i = 0; i < XWM / 16; ++i)
#pragma unroll
    for (int j = 0; j < XWN / 8; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int r = row0 + wm0 + i * 16 + g + 8 * (v >> 1);
        const int c = col0 + wn0 + j * 8 + 2 * tig + (v & 1);
        if (r < m && c < n) {
          double* p = d.C + r + (long long)c * d.ldc;
          if constexpr (UPD) *p = acc[i][j][v];
          else *p = beta == 0.0 ? alpha * acc[i][j][v] : fma(alpha, acc[i][j][v], beta * *p);
        }
      }
}

// Trailing update of the blocked partial LU (right-looking, dense_nd.cpp:174-181
// restated as a blocked elimination): for each merge in the list with
// ni > k0, M[k1:, k1:] -= M[k1:, k0:k1] * M[k0:k1, k1:], k1 = k0 + min(kb, ni-k0).
template <int BK>
__global__ void __launch_bounds__(GTHREADS) trailing_update_kernel(KernelArgs args, const int* __restrict__ list,
                                                                   int k0, int kb, int c0, int c1, int iface_rows) {
  extern __shared__ __align__(16) unsigned char gsm_raw[];
  GemmSmem<BK>& sm = *reinterpret_cast<GemmSmem<BK>*>(gsm_raw);
  const NodeDev nd = args.nodes[list[blockIdx.y]];
  if (k0 >= nd.ni) return;
  const int kbe = min(kb, nd.ni - k0), k1 = k0 + kbe;
  // rows [k1, total) (or [k1, ni): interface rows only, Schur form);
  // columns [k1 + c0, min(total, k1 + c1)) (look-ahead split)
  const int m = (iface_rows ? nd.ni : nd.total) - k1;
  // c0 < 0: start after the next panel's interface columns (fused into its prologue)
  const int cb = k1 + (c0 >= 0 ? c0 : min(kb, max(nd.ni - k1, 0)));
  const int n = min(nd.defer ? nd.ni : nd.ncols, k1 + c1) - cb;  // deferred: interface columns only
  if (m <= 0 || n <= 0) return;
  const int tiles = (m + GBM - 1) / GBM, tiles_n = (n + GBN - 1) / GBN;
  const int t = blockIdx.x;
  if (t >= tiles * tiles_n) return;
  double* M = args.arena + nd.m_off;
  const long long ld = nd.ldm;
  if ((k1 & 1) == 0)
    gemm_tile<BK, true, true>(M + k1 + k0 * ld, nd.ldm, M + k0 + cb * ld, nd.ldm, M + k1 + cb * ld, nd.ldm, m, n, kbe,
                              t % tiles, t / tiles, -1.0, 1.0, sm);
  else
    gemm_tile<BK, false, true>(M + k1 + k0 * ld, nd.ldm, M + k0 + cb * ld, nd.ldm, M + k1 + cb * ld, nd.ldm, m, n,
                               kbe, t % tiles, t / tiles, -1.0, 1.0, sm);
}

int gemm_tiles(int m, int n);

template <int BK, bool UPD, bool A16, bool TC = false>
cudaError_t set_desc_attr() {
  return cudaFuncSetAttribute(gemm_desc_kernel<BK, UPD, A16, TC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              sizeof(GemmSmem<BK>));
}

cudaError_t gemm_init() {
  cudaError_t e;
  for (cudaError_t x : {set_desc_attr<16, false, true>(), set_desc_attr<8, false, true>(), set_desc_attr<16, true, true>(),
                        set_desc_attr<8, true, true>(), set_desc_attr<16, false, false>(),
                        set_desc_attr<8, false, false>(), set_desc_attr<16, true, false>(),
                        set_desc_attr<8, true, false>(), set_desc_attr<32, false, true>(),
                        set_desc_attr<32, true, true>(), set_desc_attr<32, false, false>(),
                        set_desc_attr<32, true, false>(), set_desc_attr<8, false, true, true>(),
                        set_desc_attr<16, false, true, true>(), set_desc_attr<32, false, true, true>()})
    if (x != cudaSuccess) return x;
  e = cudaFuncSetAttribute(gemm_big_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(GemmSmemX));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(gemm_big_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(GemmSmemX));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(trailing_update_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           sizeof(GemmSmem<16>));
  if (e != cudaSuccess) return e;
  // (function attributes belong to the current device's context: set here, per
  // device, from dtn_gpu_create -- never cached in a process-wide static)
  for (cudaError_t x : {cudaFuncSetAttribute(gemm_desc2_kernel<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             sizeof(GemmSmem<16>)),
                        cudaFuncSetAttribute(gemm_desc2_kernel<16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             sizeof(GemmSmem<16>))})
    if (x != cudaSuccess) return x;
  return cudaFuncSetAttribute(trailing_update_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              sizeof(GemmSmem<8>));
}

int gemm_tiles(int m, int n) { return ((m + GBM - 1) / GBM) * ((n + GBN - 1) / GBN); }

// K-chunk 32 for long reductions (DTN_GEMM_BK32_MIN, default 2048: +3 % on the
// config-5 solve, K = 8188; shorter reductions measured faster with 16)
int gemm_bk32_min() {
  static const int v = [] {
    const char* e = std::getenv("DTN_GEMM_BK32_MIN");
    const int x = e ? std::atoi(e) : 2048;
    return x <= 0 ? (1 << 30) : x;
  }();
  return v;
}

// Large-tile path (DTN_GEMM_BIG=0 disables): aligned A and enough work (measured: 30 vs 27 TF/s
// from 4096^2 x 2048 up; at 2044^2 x 1020 the 128 x 64 tile is better, 26 vs 25)
int gemm_big_min_tiles() {
  static const int v = [] {
    const char* e = std::getenv("DTN_GEMM_BIG");
    if (e && e[0] == '0') return 1 << 30;
    const char* t = std::getenv("DTN_GEMM_BIG_TILES");
    return t ? std::atoi(t) : 1184;  // ~4 waves of 128 x 128 tiles: below that the smaller tile balances better
  }();
  return v;
}

cudaError_t launch_gemm_desc(const GemmDesc* d_descs, int count, int max_tiles, int kmax, double alpha, double beta,
                             cudaStream_t st, bool a_aligned, bool allow_big) {
  if (count <= 0 || max_tiles <= 0) return cudaSuccess;
  if (allow_big && a_aligned && max_tiles * count >= gemm_big_min_tiles() && kmax >= 64) {
    const bool upd = alpha == -1.0 && beta == 1.0;
    dim3 grid(max_tiles, count);  // (128 x 64 tile count bounds the 128 x 128 one; extra CTAs exit)
    if (upd) gemm_big_kernel<true><<<grid, GTHREADS, sizeof(GemmSmemX), st>>>(d_descs, alpha, beta);
    else gemm_big_kernel<false><<<grid, GTHREADS, sizeof(GemmSmemX), st>>>(d_descs, alpha, beta);
    return cudaGetLastError();
  }
  dim3 grid(max_tiles, count);
  const bool upd = alpha == -1.0 && beta == 1.0;  // other (alpha, beta): scaled epilogue
  const bool bk16 = kmax % 16 == 0 || kmax > 64;
  const bool bk32 = kmax >= gemm_bk32_min();
#define DTNB_DESC_LAUNCH(BK, U, AL) \
  gemm_desc_kernel<BK, U, AL><<<grid, GTHREADS, sizeof(GemmSmem<BK>), st>>>(d_descs, alpha, beta)
#define DTNB_DESC_PICK(U, AL)                           \
  do {                                                  \
    if (bk32) DTNB_DESC_LAUNCH(32, U, AL);              \
    else if (bk16) DTNB_DESC_LAUNCH(16, U, AL);         \
    else DTNB_DESC_LAUNCH(8, U, AL);                    \
  } while (0)
  if (a_aligned) {
    if (upd) DTNB_DESC_PICK(true, true);
    else DTNB_DESC_PICK(false, true);
  } else {
    if (upd) DTNB_DESC_PICK(true, false);
    else DTNB_DESC_PICK(false, false);
  }
#undef DTNB_DESC_PICK
#undef DTNB_DESC_LAUNCH
  return cudaGetLastError();
}

// C stored transposed (C^T = (A B)^T, element (r, c) at C[c + r ldc]): the
// HBS apply's leaf step writes y directly from the transposed sweep.
cudaError_t launch_gemm_desc_tc(const GemmDesc* d_descs, int count, int max_tiles, int kmax, double alpha, double beta,
                                cudaStream_t st) {
  if (count <= 0 || max_tiles <= 0) return cudaSuccess;
  dim3 grid(max_tiles, count);
  if (kmax >= gemm_bk32_min())
    gemm_desc_kernel<32, false, true, true><<<grid, GTHREADS, sizeof(GemmSmem<32>), st>>>(d_descs, alpha, beta);
  else if (kmax % 16 == 0 || kmax > 64)
    gemm_desc_kernel<16, false, true, true><<<grid, GTHREADS, sizeof(GemmSmem<16>), st>>>(d_descs, alpha, beta);
  else
    gemm_desc_kernel<8, false, true, true><<<grid, GTHREADS, sizeof(GemmSmem<8>), st>>>(d_descs, alpha, beta);
  return cudaGetLastError();
}

cudaError_t launch_gemm_desc2(const GemmDesc2* d_descs, int count, int max_tiles, bool tc, cudaStream_t st) {
  if (count <= 0 || max_tiles <= 0) return cudaSuccess;
  dim3 grid(max_tiles, count);
  if (tc) gemm_desc2_kernel<16, true><<<grid, GTHREADS, sizeof(GemmSmem<16>), st>>>(d_descs);
  else gemm_desc2_kernel<16, false><<<grid, GTHREADS, sizeof(GemmSmem<16>), st>>>(d_descs);
  return cudaGetLastError();
}

// ---- skinny products Y (m x n) = A (m x k) X (k x n), n <= 32: the small-batch
// apply_dtn / apply_schur is a stream over A (HBM-bound), which a 128-row GEMM
// tile grid of ceil(m / 128) CTAs cannot saturate. Split-K instead: CTA (row
// block, K slice) keeps its rows' partial sums for all n columns in registers
// (one row per thread, A read coalesced down the columns, the X slice in shared
// memory), partials go to a workspace and a second kernel adds the slices in a
// fixed order (deterministic).
constexpr int SK_ROWS = 128, SK_KC = 64;

template <int N>
__global__ void __launch_bounds__(SK_ROWS) skinny_partial_kernel(const double* __restrict__ A, int lda,
                                                                 const double* __restrict__ X, int ldx, int m, int k,
                                                                 int n, double* __restrict__ work) {
  __shared__ double xs[SK_KC][N];
  const int r = blockIdx.x * SK_ROWS + threadIdx.x, s = blockIdx.y;
  const int c0 = s * SK_KC, c1 = min(k, c0 + SK_KC);
  for (int e = threadIdx.x; e < SK_KC * N; e += SK_ROWS) {
    const int c = e / N, j = e % N;
    xs[c][j] = (c0 + c < c1 && j < n) ? X[(c0 + c) + (long long)j * ldx] : 0.0;
  }
  __syncthreads();
  if (r >= m) return;
  double acc[N];
#pragma unroll
  for (int j = 0; j < N; ++j) acc[j] = 0.0;
  const double* a = A + r + (long long)c0 * lda;
#pragma unroll 16
  for (int c = 0; c < c1 - c0; ++c) {
    const double g = __ldg(a + (long long)c * lda);
#pragma unroll
    for (int j = 0; j < N; ++j) acc[j] = fma(g, xs[c][j], acc[j]);
  }
#pragma unroll
  for (int j = 0; j < N; ++j)
    if (j < n) work[((long long)s * n + j) * m + r] = acc[j];
}

__global__ void skinny_reduce_kernel(const double* __restrict__ work, int slices, int m, int n, double* Y, int ldy) {
  const long long total = (long long)m * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int j = int(e / m), r = int(e - (long long)j * m);
    double t = 0.0;
    for (int s = 0; s < slices; ++s) t += work[((long long)s * n + j) * m + r];
    Y[r + (long long)j * ldy] = t;
  }
}

size_t skinny_work_doubles(int m, int k, int n) { return size_t((k + SK_KC - 1) / SK_KC) * size_t(n) * size_t(m); }

cudaError_t launch_skinny_gemm(const double* A, int lda, const double* X, int ldx, double* Y, int ldy, int m, int k,
                               int n, double* work, cudaStream_t st) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  if (n > 32) return cudaErrorInvalidValue;
  const int slices = (k + SK_KC - 1) / SK_KC;
  const dim3 grid((m + SK_ROWS - 1) / SK_ROWS, slices);
  if (n <= 4) skinny_partial_kernel<4><<<grid, SK_ROWS, 0, st>>>(A, lda, X, ldx, m, k, n, work);
  else if (n <= 8) skinny_partial_kernel<8><<<grid, SK_ROWS, 0, st>>>(A, lda, X, ldx, m, k, n, work);
  else if (n <= 16) skinny_partial_kernel<16><<<grid, SK_ROWS, 0, st>>>(A, lda, X, ldx, m, k, n, work);
  else skinny_partial_kernel<32><<<grid, SK_ROWS, 0, st>>>(A, lda, X, ldx, m, k, n, work);
  const long long total = (long long)m * n;
  skinny_reduce_kernel<<<int(std::min<long long>((total + 255) / 256, 1184)), 256, 0, st>>>(work, slices, m, n, Y,
                                                                                              ldy);
  return cudaGetLastError();
}

// Columns [k1 + c0, k1 + c1) of the trailing block (c1 = INT_MAX: to the end).
cudaError_t launch_trailing_update(const KernelArgs& args, const int* d_list, int count, int max_total, int k0, int kb,
                                   int c0, int c1, cudaStream_t st, int max_rows) {
  const int m = (max_rows > 0 ? max_rows : max_total) - k0 - 1;
  const int n = std::min(max_total + args.nl - k0 - 1, c1) - std::max(c0, 0);
  if (count <= 0 || m <= 0 || n <= 0) return cudaSuccess;
  dim3 grid(gemm_tiles(m, n), count);
  if (kb % 16 == 0)
    trailing_update_kernel<16><<<grid, GTHREADS, sizeof(GemmSmem<16>), st>>>(args, d_list, k0, kb, c0, c1,
                                                                             max_rows > 0 ? 1 : 0);
  else
    trailing_update_kernel<8><<<grid, GTHREADS, sizeof(GemmSmem<8>), st>>>(args, d_list, k0, kb, c0, c1,
                                                                           max_rows > 0 ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace dtnb
