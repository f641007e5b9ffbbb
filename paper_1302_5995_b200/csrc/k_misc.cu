// Root inverse helpers (G = S^{-1}, dense_nd.cpp:218-224) and small utilities.
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
