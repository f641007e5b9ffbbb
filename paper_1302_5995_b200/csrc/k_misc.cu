// Root inverse helpers (G = S^{-1}, dense_nd.cpp:218-224) and small utilities.
#include <algorithm>
#include <cfloat>

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
  const long long total = (long long)d.m * d.n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int r = int(e % d.m), c = int(e / d.m);
    d.dst[r + (long long)c * d.ldd] = d.src[r + (long long)c * d.lds];
  }
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

// Batched block back substitution by rows (as dtrsm, no explicit inverse):
// one warp per column, lane l holds rows l, l+32, l+64, l+96.
__global__ void __launch_bounds__(256) trsm_upper_block_kernel(const TrsmDesc* __restrict__ descs) {
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

cudaError_t launch_trsm_upper_batched(const void* d_descs, int count, int max_cols, cudaStream_t st) {
  if (count <= 0 || max_cols <= 0) return cudaSuccess;
  const int bx = std::min((max_cols + 31) / 32, 1184);
  trsm_upper_block_kernel<<<dim3(bx, count), 256, (TB * (TB + 1) + TB) * sizeof(double), st>>>(
      static_cast<const TrsmDesc*>(d_descs));
  return cudaGetLastError();
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
  return cudaFuncSetAttribute(trsm_upper_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (TB * (TB + 1) + TB) * sizeof(double));
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

}  // namespace dtnb
