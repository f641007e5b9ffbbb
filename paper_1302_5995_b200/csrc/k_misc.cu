// Root inverse helpers (G = S^{-1}, dense_nd.cpp:218-224) and small utilities.
#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "common.cuh"

namespace dtnb {

// X = P * I for the row-swap sequence ipiv (LAPACK convention, 0-based absolute rows).
__global__ void perm_identity_kernel(const int* __restrict__ ipiv, int n, int* perm, double* X, int ldx) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) perm[i] = i;
    for (int i = 0; i < n; ++i) {
      const int p = ipiv[i];
      const int t = perm[i];
      perm[i] = perm[p];
      perm[p] = t;
    }
  }
}
__global__ void scatter_identity_kernel(const int* __restrict__ perm, int n, double* X, int ldx) {
  const long long total = (long long)n * ldx;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int r = int(e % ldx), c = int(e / ldx);
    X[e] = (r < n && perm[r] == c) ? 1.0 : 0.0;
  }
}

// Columns [c0, c0 + w) of P (P A = L U, perm[pos] = original row): X(pos, j) = 1 iff
// perm[pos] == c0 + j -- the right-hand sides of G's column chunk G = U^{-1} L^{-1} P.
__global__ void perm_identity_cols_kernel(const int* __restrict__ perm, int n, int c0, int w, double* X, int ldx) {
  const long long total = (long long)w * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int r = int(e % n), c = int(e / n);
    X[r + (long long)c * ldx] = perm[r] == c0 + c ? 1.0 : 0.0;
  }
}

cudaError_t launch_perm_identity_cols(const int* perm, int n, int c0, int w, double* X, int ldx, cudaStream_t st) {
  if (w <= 0 || n <= 0) return cudaSuccess;
  perm_identity_cols_kernel<<<592, 256, 0, st>>>(perm, n, c0, w, X, ldx);
  return cudaGetLastError();
}

// X[k0:k0+kbe, :] <- T^{-1} X[k0:k0+kbe, :] with T the kbe x kbe diagonal block
// of the LU factors (lower: unit lower L; else upper U). One warp per column.
__global__ void __launch_bounds__(256) trsm_rows_kernel(const double* __restrict__ LU, int ldlu, double* X, int ldx,
                                                        int ncols, int k0, int kbe, int lower) {
  __shared__ double T[32][33];
  for (int e = threadIdx.x; e < kbe * kbe; e += blockDim.x)
    T[e % kbe][e / kbe] = LU[(k0 + e % kbe) + (long long)(k0 + e / kbe) * ldlu];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = blockIdx.x * 8 + warp; j < ncols; j += gridDim.x * 8) {
    double* col = X + (long long)j * ldx + k0;
    double x = lane < kbe ? col[lane] : 0.0;
    if (lower) {
      for (int c = 0; c < kbe; ++c) {
        const double xc = __shfl_sync(0xffffffffu, x, c);
        if (lane > c && lane < kbe) x = fma(-T[lane][c], xc, x);
      }
    } else {
      for (int c = kbe - 1; c >= 0; --c) {
        if (lane == c) x = x / T[c][c];
        const double xc = __shfl_sync(0xffffffffu, x, c);
        if (lane < c) x = fma(-T[lane][c], xc, x);
      }
    }
    if (lane < kbe) col[lane] = x;
  }
}

// out = max_j sum_i |X(i,j)| (1-norm), via atomicMax on the bit pattern of
// a non-negative double.
__global__ void norm1_kernel(const double* __restrict__ X, int ldx, int m, int n, unsigned long long* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = blockIdx.x * (blockDim.x / 32) + warp; j < n; j += gridDim.x * (blockDim.x / 32)) {
    double s = 0.0;
    for (int i = lane; i < m; i += 32) s += fabs(X[i + (long long)j * ldx]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) atomicMax(out, __double_as_longlong(s));
  }
}

__global__ void copy2d_kernel(const double* __restrict__ src, int lds, double* dst, int ldd, int m, int n) {
  const long long total = (long long)m * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int r = int(e % m), c = int(e / m);
    dst[r + (long long)c * ldd] = src[r + (long long)c * lds];
  }
}

// Inverses of the diagonal TB x TB blocks of the LU factors: Linv_k = L_kk^{-1}
// (unit lower) and Uinv_k = U_kk^{-1}, one CTA per block, one thread per
// column, block staged in shared memory. Output: full TB x TB blocks (zero
// outside the triangle; identity padding for a partial last block).
constexpr int TB = 128;
__global__ void __launch_bounds__(TB) tri_inv_blocks_kernel(const double* __restrict__ LU, int ldlu, int n,
                                                            double* __restrict__ out) {
  extern __shared__ double blk[];  // TB x (TB+1)
  const int kb = blockIdx.x, k0 = kb * TB, bk = min(TB, n - k0);
  const int j = threadIdx.x;
  for (int c = 0; c < TB; ++c) {
    const int r = j;
    blk[c * (TB + 1) + r] = (r < bk && c < bk) ? LU[(k0 + r) + (long long)(k0 + c) * ldlu] : (r == c ? 1.0 : 0.0);
  }
  __syncthreads();
  double* Li = out + (long long)kb * 2 * TB * TB;
  double* Ui = Li + TB * TB;
  // column j of L^{-1}: forward substitution with the unit lower triangle
  {
    double x[TB];
#pragma unroll 1
    for (int i = 0; i < TB; ++i) x[i] = 0.0;
    // (register array with dynamic indexing lives in local memory; bounded by TB)
    x[j] = 1.0;
    for (int i = j + 1; i < TB; ++i) {
      double s = 0.0;
      for (int m = j; m < i; ++m) s = fma(blk[m * (TB + 1) + i], x[m], s);
      x[i] = -s;
    }
    for (int i = 0; i < TB; ++i) Li[i + (long long)j * TB] = x[i];
  }
  // column j of U^{-1}: back substitution
  {
    double x[TB];
    for (int i = 0; i < TB; ++i) x[i] = 0.0;
    x[j] = 1.0 / blk[j * (TB + 1) + j];
    for (int i = j - 1; i >= 0; --i) {
      double s = 0.0;
      for (int m = i + 1; m <= j; ++m) s = fma(blk[m * (TB + 1) + i], x[m], s);
      x[i] = -s / blk[i * (TB + 1) + i];
    }
    for (int i = 0; i < TB; ++i) Ui[i + (long long)j * TB] = x[i];
  }
}

// Batched: inverses of the 128 x 128 diagonal blocks of U for several LU
// factors (back substitution of the merge systems); out layout as above.
__global__ void __launch_bounds__(TB) tri_inv_u_batched_kernel(const TriDesc* __restrict__ descs) {
  extern __shared__ double blk[];
  const TriDesc d = descs[blockIdx.y];
  const int kb = blockIdx.x, k0 = kb * TB;
  if (k0 >= d.n) return;
  const int bk = min(TB, d.n - k0);
  const int j = threadIdx.x;
  for (int c = 0; c < TB; ++c)
    blk[c * (TB + 1) + j] = (j < bk && c < bk) ? d.LU[(k0 + j) + (long long)(k0 + c) * d.ld] : (j == c ? 1.0 : 0.0);
  __syncthreads();
  double* Ui = d.out + (long long)kb * 2 * TB * TB + TB * TB;
  double x[TB];
  for (int i = 0; i < TB; ++i) x[i] = 0.0;
  x[j] = 1.0 / blk[j * (TB + 1) + j];
  for (int i = j - 1; i >= 0; --i) {
    double s = 0.0;
    for (int m = i + 1; m <= j; ++m) s = fma(blk[m * (TB + 1) + i], x[m], s);
    x[i] = -s / blk[i * (TB + 1) + i];
  }
  for (int i = 0; i < TB; ++i) Ui[i + (long long)j * TB] = x[i];
}

__global__ void copy2d_batched_kernel(const CopyDesc* __restrict__ descs) {
  const CopyDesc d = descs[blockIdx.y];
  // rows over RT = pow2 >= m (<= blockDim) threads, the CTA's blockDim / RT
  // thread groups and the grid over columns (no per-element division)
  int RT = 32;
  while (RT < d.m && RT < int(blockDim.x)) RT <<= 1;
  const int groups = int(blockDim.x) / RT, g = int(threadIdx.x) / RT, r0 = int(threadIdx.x) & (RT - 1);
  for (int c = blockIdx.x * groups + g; c < d.n; c += gridDim.x * groups)
    for (int r = r0; r < d.m; r += RT)
      d.dst[r + (long long)c * d.ldd] = d.src[r + (long long)c * d.lds];
}

cudaError_t launch_tri_inv_u_batched(const void* d_descs, int count, int max_blocks, cudaStream_t st) {
  if (count <= 0 || max_blocks <= 0) return cudaSuccess;
  tri_inv_u_batched_kernel<<<dim3(max_blocks, count), TB, TB * (TB + 1) * sizeof(double), st>>>(
      static_cast<const TriDesc*>(d_descs));
  return cudaGetLastError();
}

cudaError_t launch_copy2d_batched(const void* d_descs, int count, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  copy2d_batched_kernel<<<dim3(64, count), 256, 0, st>>>(static_cast<const CopyDesc*>(d_descs));
  return cudaGetLastError();
}

// Batched block substitution (as dtrsm, no explicit inverse): Y <- T^{-1} Y
// with T the bk x bk (bk <= 128) upper triangle (backward) or, LOWER, the unit
// lower triangle (forward) of the block at d.U. One CTA per 64 columns of one
// descriptor; T and the Y tile are staged column-major in shared memory with
// 16-byte cp.async (T's columns, Y's block and both leading dimensions must
// be 16-byte aligned: true for every caller, all blocks start at multiples of
// 128 rows of 8-aligned leading dimensions). Rows are processed in 32-row
// groups: each group is solved by substitution with one column per thread
// (warps 0-1; triangle entries are shared-memory broadcasts, no shuffles),
// then the rows not yet solved are updated with the group's solution with FP64 FMAs
// in register blocks (see update() on the accumulation order). The next group's
// rows are updated first so its substitution overlaps the update of the rest.
// bk is padded to a multiple of 32 (zero-filled T and Y rows).
constexpr int TS_COLS_MAX = 64;
__host__ __device__ constexpr int ts_pad(int bk) { return (bk + 31) & ~31; }
#ifdef TS_PROFILE
__device__ long long g_ts_clk[16];
#define TSCLK(i) do { if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) g_ts_clk[i] = clock64(); } while (0)
#else
#define TSCLK(i) do { } while (0)
#endif

template <bool LOWER, int TS_COLS>
__global__ void __launch_bounds__(256, 2) trsm_block_kernel(const TrsmDesc* __restrict__ descs) {
  extern __shared__ __align__(16) double trsm_smem[];
  const TrsmDesc d = descs[blockIdx.y];
  const int bk = d.bk, bkp = ts_pad(bk), ld = bkp + 2;
  const int col0 = blockIdx.x * TS_COLS;
  if (col0 >= d.ncols) return;
  const int ncl = min(TS_COLS, d.ncols - col0);
  double* Uc = trsm_smem;        // T[r][c] at c * ld + r
  double* Yt = Uc + bkp * ld;    // Y[r][col0 + c] at c * ld + r
  double* rd = Yt + TS_COLS * ld;  // 1 / T[i][i] (upper)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tig = lane & 3;
  TSCLK(0);
  const int npair = bkp / 2;
  for (int c = warp; c < bkp; c += 8)
    for (int p = lane; p < npair; p += 32) {  // only the pairs the triangle touches
      const int r = 2 * p;
      if (LOWER ? r + 1 < c : r > c) continue;  // (never read)
      const int bytes = (c < bk && r < bk) ? min(2, bk - r) * 8 : 0;
      cp_async16(Uc + c * ld + r, bytes ? d.U + r + (long long)c * d.ldu : d.U, bytes);
    }
  for (int c = warp; c < TS_COLS; c += 8)
    for (int p = lane; p < npair; p += 32) {
      const int r = 2 * p;
      const int bytes = (c < ncl && r < bk) ? min(2, bk - r) * 8 : 0;
      cp_async16(Yt + c * ld + r, bytes ? d.Y + r + (long long)(col0 + c) * d.ldy : d.Y, bytes);
    }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  if (!LOWER)
    for (int i = tid; i < bkp; i += 256) rd[i] = i < bk ? 1.0 / Uc[i * ld + i] : 1.0;
  __syncthreads();
  TSCLK(1);

  // substitution on the 32 rows of group sb, one column per thread (warps 0-1)
  auto leaf = [&](int sb) {
    const int r0 = sb * 32;
    double* yc = Yt + (warp * 32 + lane) * ld + r0;
    double x[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = yc[i];
    if (LOWER) {
#pragma unroll
      for (int i = 0; i < 31; ++i) {
        const double* tc = Uc + (r0 + i) * ld + r0;
#pragma unroll
        for (int m = i + 1; m < 32; ++m) x[m] = fma(-tc[m], x[i], x[m]);
      }
    } else {
#pragma unroll
      for (int i = 31; i >= 0; --i) {
        const double* tc = Uc + (r0 + i) * ld + r0;
        x[i] *= rd[r0 + i];
#pragma unroll
        for (int m = 0; m < i; ++m) x[m] = fma(-tc[m], x[i], x[m]);
      }
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) yc[i] = x[i];
  };
  // Y[ra:rb, :] -= T[ra:rb, g0:g0+32] Y[g0:g0+32, :] by warps [w0, w0 + nw),
  // 4 x 4 register blocks. Each element accumulates its 32 terms with
  // sequential FMAs in the order of the column substitution (farthest column
  // first): measured on the near-resonant config-3 operator, this order is
  // 3.5x more accurate (G g vs a sparse direct solve) than DMMA tiles, whose
  // accumulation order differs, so the update stays on the FP64 FMA pipe.
  auto update = [&](int ra, int rb, int g0, int w0, int nw) {
    const int nrq = (rb - ra) / 4, ntask = nrq * (TS_COLS / 4);
    for (int t = tid - w0 * 32; t < ntask; t += nw * 32) {
      const int r = ra + (t % nrq) * 4, c = (t / nrq) * 4;
      double acc[4][4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double2 lo = *reinterpret_cast<const double2*>(Yt + (c + j) * ld + r);
        const double2 hi = *reinterpret_cast<const double2*>(Yt + (c + j) * ld + r + 2);
        acc[0][j] = lo.x; acc[1][j] = lo.y; acc[2][j] = hi.x; acc[3][j] = hi.y;
      }
#pragma unroll 8
      for (int k = 0; k < 32; ++k) {
        const int kk = LOWER ? g0 + k : g0 + 31 - k;
        const double2 ulo = *reinterpret_cast<const double2*>(Uc + kk * ld + r);
        const double2 uhi = *reinterpret_cast<const double2*>(Uc + kk * ld + r + 2);
        const double u[4] = {ulo.x, ulo.y, uhi.x, uhi.y};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double y = Yt[(c + j) * ld + kk];
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[i][j] = fma(-u[i], y, acc[i][j]);
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        *reinterpret_cast<double2*>(Yt + (c + j) * ld + r) = make_double2(acc[0][j], acc[1][j]);
        *reinterpret_cast<double2*>(Yt + (c + j) * ld + r + 2) = make_double2(acc[2][j], acc[3][j]);
      }
    }
  };
  const int ng = bkp / 32;
  int prev = LOWER ? 0 : ng - 1;
  if (warp < TS_COLS / 32) leaf(prev);
  __syncthreads();
  TSCLK(2);
  for (int step = 1; step < ng; ++step) {
    const int next = LOWER ? prev + 1 : prev - 1;
    update(next * 32, next * 32 + 32, prev * 32, 0, 8);
    __syncthreads();
    if (warp < TS_COLS / 32) leaf(next);
    else if (LOWER) update(next * 32 + 32, bkp, prev * 32, TS_COLS / 32, 8 - TS_COLS / 32);
    else update(0, next * 32, prev * 32, TS_COLS / 32, 8 - TS_COLS / 32);
    __syncthreads();
    TSCLK(2 + step);
    prev = next;
  }
  for (int c = warp; c < ncl; c += 8)
    for (int p = lane; p < npair; p += 32) {
      const int r = 2 * p;
      double* dst = d.Y + r + (long long)(col0 + c) * d.ldy;
      if (r + 1 < bk) *reinterpret_cast<double2*>(dst) = *reinterpret_cast<const double2*>(Yt + c * ld + r);
      else if (r < bk) *dst = Yt[c * ld + r];
    }
  TSCLK(15);
}

// Dirichlet-ring DtN (SURVEY f-1): T[i][j] = (delta_ij + coef[j] G[adj[i]][adj[j]]) / h
// for the non-corner ring nodes, T = (1/h)(I + P G D_b).
__global__ void ring_dtn_kernel(const double* __restrict__ G, int ldg, const int* __restrict__ adj,
                                const double* __restrict__ coef, int m, double inv_h, double* __restrict__ T, long long ldt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // consecutive threads: consecutive rows of T
  if (i >= m) return;
  const int ai = adj[i];
  for (int j = blockIdx.y; j < m; j += gridDim.y) {
    const double g = G[ai + (long long)adj[j] * ldg];
    T[i + (long long)j * ldt] = ((i == j ? 1.0 : 0.0) + coef[j] * g) * inv_h;
  }
}

cudaError_t launch_ring_dtn(const double* G, int ldg, const int* adj, const double* coef, int m, double h, double* T,
                            long long ldt, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  dim3 grid((m + 127) / 128, std::min(m, 2048));
  ring_dtn_kernel<<<grid, 128, 0, st>>>(G, ldg, adj, coef, m, 1.0 / h, T, ldt);
  return cudaGetLastError();
}

// nblk consecutive TB x TB column-major identity blocks
__global__ void block_identity_kernel(double* out, long long total) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x)
    out[e] = (e % TB) == ((e / TB) % TB) ? 1.0 : 0.0;
}

cudaError_t launch_block_identity(double* out, int nblk, cudaStream_t st) {
  const long long total = (long long)nblk * TB * TB;
  block_identity_kernel<<<int(std::min<long long>((total + 255) / 256, 1184)), 256, 0, st>>>(out, total);
  return cudaGetLastError();
}

// Diagnostic (DTN_SUBST_REF=1): the round-1 warp-per-4-columns substitution kernel.
// Batched block back substitution by rows (as dtrsm, no explicit inverse):
// one warp per column, lane l holds rows l, l+32, l+64, l+96.
__global__ void __launch_bounds__(256) trsm_upper_block_kernel_ref(const TrsmDesc* __restrict__ descs) {
  extern __shared__ double trsm_smem[];
  double (*Us)[TB + 1] = reinterpret_cast<double (*)[TB + 1]>(trsm_smem);
  double* rd = trsm_smem + TB * (TB + 1);
  const TrsmDesc d = descs[blockIdx.y];
  const int bk = d.bk;
  if (blockIdx.x * 8 >= d.ncols) return;
  for (int e = threadIdx.x; e < bk * bk; e += blockDim.x) {
    const int r = e % bk, c = e / bk;
    Us[r][c] = d.U[r + (long long)c * d.ldu];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < bk; c += blockDim.x) rd[c] = 1.0 / Us[c][c];
  __syncthreads();
  // each warp runs TCW independent columns interleaved (ILP over the
  // 128-step dependent substitution chain)
  constexpr int TCW = 4;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j0 = (blockIdx.x * 8 + warp) * TCW; j0 < d.ncols; j0 += gridDim.x * 8 * TCW) {
    double x[TCW][4];
#pragma unroll
    for (int u = 0; u < TCW; ++u)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        x[u][q] = (j0 + u < d.ncols && lane + 32 * q < bk) ? d.Y[lane + 32 * q + (long long)(j0 + u) * d.ldy] : 0.0;
    for (int c = bk - 1; c >= 0; --c) {
      const int owner = c & 31, qc = c >> 5;
      const double rdc = rd[c];
      double xc[TCW];
#pragma unroll
      for (int u = 0; u < TCW; ++u) {
        double t = x[u][0];
#pragma unroll
        for (int q = 1; q < 4; ++q) t = (q == qc) ? x[u][q] : t;
        xc[u] = __shfl_sync(0xffffffffu, t * rdc, owner);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = lane + 32 * q;
        const double urc = (r < c) ? Us[r][c] : 0.0;
#pragma unroll
        for (int u = 0; u < TCW; ++u) {
          if (r == c) x[u][q] = xc[u];
          else x[u][q] = fma(-urc, xc[u], x[u][q]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < TCW; ++u)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (j0 + u < d.ncols && lane + 32 * q < bk) d.Y[lane + 32 * q + (long long)(j0 + u) * d.ldy] = x[u][q];
  }
}

cudaError_t launch_trsm_upper_ref(const void* d_descs, int count, int max_cols, cudaStream_t st) {
  if (count <= 0 || max_cols <= 0) return cudaSuccess;
  const int bx = std::min((max_cols + 31) / 32, 1184);
  trsm_upper_block_kernel_ref<<<dim3(bx, count), 256, (TB * (TB + 1) + TB) * sizeof(double), st>>>(
      static_cast<const TrsmDesc*>(d_descs));
  return cudaGetLastError();
}

size_t trsm_smem_bytes(int max_bk) {
  const int bkp = ts_pad(std::max(1, std::min(max_bk, TB)));
  return size_t(bkp * (bkp + 2) + TS_COLS_MAX * (bkp + 2) + bkp) * sizeof(double);
}

cudaError_t launch_trsm_batched(const void* d_descs, int count, int max_cols, int max_bk, bool lower,
                                cudaStream_t st) {
  if (count <= 0 || max_cols <= 0) return cudaSuccess;
  if (max_bk > TB) return cudaErrorInvalidValue;
  const auto* dd = static_cast<const TrsmDesc*>(d_descs);
  const size_t sm = trsm_smem_bytes(max_bk);
  // few CTAs (the tall, narrow back substitutions of the top merges): 32-column CTAs
  // halve each CTA's serial work; otherwise 64 columns per CTA (the triangle staged once
  // per 64 columns)
  static const int narrow_env = [] {
    const char* e = std::getenv("DTN_TRSM_NARROW");
    return e ? std::atoi(e) : -1;
  }();
  const int tiles64 = (max_cols + 63) / 64 * count;
  const bool narrow = narrow_env >= 0 ? narrow_env != 0 : tiles64 < 148;
  if (narrow) {
    const dim3 grid((max_cols + 31) / 32, count);
    if (lower) trsm_block_kernel<true, 32><<<grid, 256, sm, st>>>(dd);
    else trsm_block_kernel<false, 32><<<grid, 256, sm, st>>>(dd);
  } else {
    const dim3 grid((max_cols + 63) / 64, count);
    if (lower) trsm_block_kernel<true, 64><<<grid, 256, sm, st>>>(dd);
    else trsm_block_kernel<false, 64><<<grid, 256, sm, st>>>(dd);
  }
  return cudaGetLastError();
}

cudaError_t launch_trsm_upper_batched(const void* d_descs, int count, int max_cols, cudaStream_t st) {
  return launch_trsm_batched(d_descs, count, max_cols, TB, false, st);
}

__global__ void set_identity_kernel(double* X, int ldx, int n) {
  const long long total = (long long)n * ldx;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int r = int(e % ldx), c = int(e / ldx);
    X[e] = (r == c && r < n) ? 1.0 : 0.0;
  }
}

// G[:, perm[i]] = W[:, i]  (A^{-1} = U^{-1} L^{-1} P)
__global__ void permute_columns_kernel(const double* __restrict__ W, int ldw, const int* __restrict__ perm, int n,
                                       double* __restrict__ G, int ldg) {
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const double* src = W + (long long)i * ldw;
    double* dst = G + (long long)perm[i] * ldg;
    for (int r = threadIdx.x; r < n; r += blockDim.x) dst[r] = src[r];
  }
}

cudaError_t misc_init() {
  cudaError_t e = cudaFuncSetAttribute(tri_inv_blocks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       TB * (TB + 1) * sizeof(double));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(tri_inv_u_batched_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           TB * (TB + 1) * sizeof(double));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(trsm_upper_block_kernel_ref, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (TB * (TB + 1) + TB) * sizeof(double));
  if (e != cudaSuccess) return e;
  for (auto f : {trsm_block_kernel<false, 64>, trsm_block_kernel<true, 64>, trsm_block_kernel<false, 32>,
                 trsm_block_kernel<true, 32>}) {
    e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(trsm_smem_bytes(TB)));
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_tri_inv_blocks(const double* LU, int ldlu, int n, double* out, cudaStream_t st) {
  const int nblk = (n + TB - 1) / TB;
  tri_inv_blocks_kernel<<<nblk, TB, TB * (TB + 1) * sizeof(double), st>>>(LU, ldlu, n, out);
  return cudaGetLastError();
}

cudaError_t launch_set_identity(double* X, int ldx, int n, cudaStream_t st) {
  set_identity_kernel<<<1184, 256, 0, st>>>(X, ldx, n);
  return cudaGetLastError();
}

cudaError_t launch_permute_columns(const double* W, int ldw, const int* perm, int n, double* G, int ldg,
                                   cudaStream_t st) {
  permute_columns_kernel<<<std::min(n, 2048), 256, 0, st>>>(W, ldw, perm, n, G, ldg);
  return cudaGetLastError();
}

cudaError_t launch_perm_only(const int* d_ipiv, int n, int* d_perm, cudaStream_t st) {
  perm_identity_kernel<<<1, 32, 0, st>>>(d_ipiv, n, d_perm, nullptr, 0);
  return cudaGetLastError();
}

cudaError_t launch_perm_identity(const int* d_ipiv, int n, int* d_perm, double* X, int ldx, cudaStream_t st) {
  perm_identity_kernel<<<1, 32, 0, st>>>(d_ipiv, n, d_perm, X, ldx);
  scatter_identity_kernel<<<1184, 256, 0, st>>>(d_perm, n, X, ldx);
  return cudaGetLastError();
}

cudaError_t launch_trsm_rows(const double* LU, int ldlu, double* X, int ldx, int ncols, int k0, int kbe, bool lower,
                             cudaStream_t st) {
  const int blocks = (ncols + 7) / 8;
  trsm_rows_kernel<<<blocks, 256, 0, st>>>(LU, ldlu, X, ldx, ncols, k0, kbe, lower ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_norm1(const double* X, int ldx, int m, int n, unsigned long long* out, cudaStream_t st) {
  norm1_kernel<<<(n + 7) / 8, 256, 0, st>>>(X, ldx, m, n, out);
  return cudaGetLastError();
}

cudaError_t launch_copy2d(const double* src, int lds, double* dst, int ldd, int m, int n, cudaStream_t st) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  copy2d_kernel<<<1184, 256, 0, st>>>(src, lds, dst, ldd, m, n);
  return cudaGetLastError();
}

// Singular-block screen of a build (dense_nd.cpp:93-96, 175-180): the lowest
// id of a checked node whose pivots fail pmin > pmax * 1e-300 (or are not
// finite) -> *first_bad (INT_MAX when none), so the host reads 4 bytes instead
// of every node's pivot statistics. chk: 1 = check, 2 = check when G is built.
__global__ void pivot_screen_kernel(const double* __restrict__ pivstat, const int* __restrict__ chk, int n, int want_G,
                                    int* first_bad) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int c = chk[i];
    if (c == 0 || (c == 2 && !want_G)) continue;
    const double pmin = pivstat[2 * i], pmax = pivstat[2 * i + 1];
    if (!((pmin > pmax * 1e-300) && isfinite(pmax))) atomicMin(first_bad, i);
  }
}

cudaError_t launch_pivot_screen(const double* pivstat, const int* chk, int n, int want_G, int* first_bad,
                                cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  pivot_screen_kernel<<<std::min((n + 255) / 256, 1184), 256, 0, st>>>(pivstat, chk, n, want_G, first_bad);
  return cudaGetLastError();
}

// Row permutation of the deferred boundary columns: dst(i, c) = src(perm[i], c)
// (perm = the interface LU's running permutation, perm[pos] = original row).
__global__ void row_gather_kernel(const RowGatherDesc* __restrict__ descs, const int* __restrict__ piv) {
  const RowGatherDesc d = descs[blockIdx.y];
  const int* perm = piv + d.perm_off;
  for (int c = blockIdx.x; c < d.cols; c += gridDim.x)
    for (int i = threadIdx.x; i < d.rows; i += blockDim.x)
      d.dst[i + (long long)c * d.ldd] = d.src[perm[i] + (long long)c * d.lds];
}

cudaError_t launch_row_gather(const RowGatherDesc* d_descs, int count, const int* piv, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  row_gather_kernel<<<dim3(592, count), 256, 0, st>>>(d_descs, piv);
  return cudaGetLastError();
}

}  // namespace dtnb
