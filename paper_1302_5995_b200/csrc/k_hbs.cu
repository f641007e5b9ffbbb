// Kernels of the HBS (hierarchically block separable) compression and apply
// (hbs.cpp:61-232 restated for the GPU, see hbs.cu): batched transposes,
// a batched cyclic Jacobi eigensolver for the per-node Gram matrices, the
// rank selection, column gathers and the zero-padded repacking of factors.
// The contractions themselves run on the DMMA GEMM (k_gemm.cu).
#include <algorithm>
#include <cfloat>
#include <cstdint>

#include "common.cuh"
#include "hbs.hpp"

namespace dtnb {

// ---- dst (n x m) = src (m x n)^T, batched; 32 x 32 tiles through shared memory
__global__ void __launch_bounds__(256) transpose_batched_kernel(const TransDesc* __restrict__ descs) {
  __shared__ double tile[32][33];
  const TransDesc d = descs[blockIdx.y];
  const int tm = (d.m + 31) / 32, tn = (d.n + 31) / 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int t = blockIdx.x; t < tm * tn; t += gridDim.x) {
    const int r0 = (t % tm) * 32, c0 = (t / tm) * 32;
#pragma unroll
    for (int k = 0; k < 32; k += 8) {
      const int r = r0 + tx, c = c0 + ty + k;
      tile[ty + k][tx] = (r < d.m && c < d.n) ? d.src[r + (long long)c * d.lds] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 32; k += 8) {
      const int c = c0 + tx, r = r0 + ty + k;  // dst row c, column r
      if (c < d.n && r < d.m) d.dst[c + (long long)r * d.ldd] = tile[tx][ty + k];
    }
    __syncthreads();
  }
}

cudaError_t launch_transpose_batched(const TransDesc* d_descs, int count, int max_tiles, cudaStream_t st) {
  if (count <= 0 || max_tiles <= 0) return cudaSuccess;
  transpose_batched_kernel<<<dim3(std::min(max_tiles, 1184), count), 256, 0, st>>>(d_descs);
  return cudaGetLastError();
}

// ---- symmetric eigen-decomposition A = V diag(lambda) V^T by the cyclic
// Jacobi method, parallel (round-robin) ordering: each round rotates s/2
// disjoint (p, q) pairs, a sweep is s-1 rounds. One CTA per matrix; A (and V
// when both fit) live in shared memory with an odd leading dimension,
// otherwise in global memory (L2). A rotation is skipped when
// |a_pq| <= tol * sqrt(|a_pp a_qq|) (rel: Demmel-Veselic relative accuracy,
// used on the graded second-pass Gram matrices) or <= tol * max|a_ii| (not rel),
// tol = max(s, 16) * DBL_EPSILON.
// On exit the diagonal of desc.A holds lambda and desc.V the eigenvectors.
constexpr int JT = 512;
constexpr int JMAXP = 512;  // max pairs (s <= 1024)

__global__ void __launch_bounds__(JT) jacobi_eig_kernel(const EigDesc* __restrict__ descs, int max_sweeps,
                                                       int smem_doubles, int rel, int min_s) {
  extern __shared__ __align__(16) double jsm[];
  __shared__ double cs_[JMAXP], sn_[JMAXP];
  __shared__ int pp_[JMAXP], qq_[JMAXP];
  __shared__ int rotated;
  __shared__ double amax;
  const EigDesc d = descs[blockIdx.x];
  const int s = d.s, tid = threadIdx.x;
  if (s <= 0 || s < min_s) return;
  const int ls = s | 1;
  const long long need = (long long)s * ls;
  double* A = d.A;
  long long lda = d.lda;
  double* V = d.V;
  long long ldv = d.ldv;
  const bool a_sm = need <= smem_doubles, v_sm = 2 * need <= smem_doubles;
  if (a_sm) {
    A = jsm;
    lda = ls;
    for (long long e = tid; e < (long long)s * s; e += JT) {
      const int r = int(e % s), c = int(e / s);
      A[r + c * lda] = d.A[r + c * d.lda];
    }
  }
  if (v_sm) {
    V = jsm + need;
    ldv = ls;
  }
  for (long long e = tid; e < (long long)s * s; e += JT) {
    const int r = int(e % s), c = int(e / s);
    V[r + c * ldv] = r == c ? 1.0 : 0.0;
  }
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int i = 0; i < s; ++i) m = fmax(m, fabs(A[i + i * lda]));
    amax = m;
  }
  __syncthreads();
  const double tol = DBL_EPSILON * double(max(s, 16));  // dimension-scaled stopping rule (as LAPACK dgesvj)
  const double abs_tol = tol * amax;
  const int n2 = s + (s & 1), np = n2 / 2;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int r = 0; r < n2 - 1; ++r) {
      for (int i = tid; i < np; i += JT) {
        int a, b;
        if (i == 0) {
          a = r;
          b = n2 - 1;
        } else {
          a = (r + i) % (n2 - 1);
          b = (r - i + n2 - 1) % (n2 - 1);
        }
        const int p = min(a, b), q = max(a, b);
        double c = 1.0, sg = 0.0;
        if (q < s) {
          const double app = A[p + p * lda], aqq = A[q + q * lda], apq = A[p + q * lda];
          const double thr = rel ? tol * sqrt(fabs(app * aqq)) : abs_tol;
          if (apq != 0.0 && fabs(apq) > thr) {
            const double tau = (aqq - app) / (2.0 * apq);
            double t;
            if (fabs(tau) > 1e150) t = 0.5 / tau;
            else t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            sg = t * c;
            rotated = 1;
          }
        }
        cs_[i] = c;
        sn_[i] = sg;
        pp_[i] = p;
        qq_[i] = q;
      }
      __syncthreads();
      // rows p, q <- J^T (rows)
      for (int w = tid; w < np * s; w += JT) {
        const int i = w / s, j = w - i * s;
        const double sg = sn_[i];
        if (sg != 0.0) {
          const double c = cs_[i];
          const int p = pp_[i], q = qq_[i];
          const double x = A[p + j * lda], y = A[q + j * lda];
          A[p + j * lda] = c * x - sg * y;
          A[q + j * lda] = sg * x + c * y;
        }
      }
      __syncthreads();
      // columns p, q <- (A J), V <- V J
      for (int w = tid; w < np * s; w += JT) {
        const int i = w / s, j = w - i * s;
        const double sg = sn_[i];
        if (sg != 0.0) {
          const double c = cs_[i];
          const int p = pp_[i], q = qq_[i];
          const double x = A[j + p * lda], y = A[j + q * lda];
          A[j + p * lda] = c * x - sg * y;
          A[j + q * lda] = sg * x + c * y;
          const double vx = V[j + p * ldv], vy = V[j + q * ldv];
          V[j + p * ldv] = c * vx - sg * vy;
          V[j + q * ldv] = sg * vx + c * vy;
        }
      }
      __syncthreads();
    }
    if (!rotated) break;
    __syncthreads();
  }
  if (a_sm)
    for (int i = tid; i < s; i += JT) d.A[i + (long long)i * d.lda] = A[i + i * lda];
  if (v_sm)
    for (long long e = tid; e < (long long)s * s; e += JT) {
      const int r = int(e % s), c = int(e / s);
      d.V[r + c * d.ldv] = V[r + c * ldv];
    }
}

int jacobi_smem_doubles() { return 200 * 1024 / 8; }

// ---- the same Jacobi eigensolver for s <= 2 * JPMAXP, with A stored as its
// packed upper triangle in shared memory (s <= 236 fits: the top-level Gram
// matrices of the compressed operators, k_left + k_right <= ~200) and one
// fused update per round: every 2 x 2 block (pair i, pair j), i <= j, becomes
// T_i A_ij T_j^T in one pass (no separate row and column passes), V <- V T^T
// in the same phase -- 2 barriers per round instead of 3 and half the A
// traffic. Rotations are computed exactly as in jacobi_eig_kernel. floor > 0
// (relative to max a_ii): a pair whose diagonal entries are both below it is
// left alone -- both directions are far below the truncation level
// (sigma < 1e-2 eps sigma_0), so neither the eps-rank nor the retained basis
// depends on rotations among them, and the relative rule would otherwise
// chase rounding noise there for every sweep.
constexpr int JPMAXP = 128;
constexpr int kPackedMaxS = 236;  // 236 * 237 / 2 doubles = 218.5 KB

__device__ __forceinline__ int jp_idx(int r, int c) {  // packed upper triangle, r <= c
  return c * (c + 1) / 2 + r;
}

template <int NT>
__global__ void __launch_bounds__(NT) jacobi_eig_packed_kernel(const EigDesc* __restrict__ descs, int max_sweeps,
                                                              int smem_doubles, int rel, double floor_rel) {
  extern __shared__ __align__(16) double jsm[];
  __shared__ double cs_[JPMAXP], sn_[JPMAXP];
  __shared__ int pp_[JPMAXP], qq_[JPMAXP];
  __shared__ int rotated;
  __shared__ double amax;
  const EigDesc d = descs[blockIdx.x];
  const int s = d.s, tid = threadIdx.x;
  if (s <= 0 || s > kPackedMaxS) return;
  double* P = jsm;
  const int npk = s * (s + 1) / 2;
  const int ls = s | 1;
  const bool v_sm = (long long)npk + (long long)s * ls <= smem_doubles;
  double* V = v_sm ? jsm + npk : d.V;
  const long long ldv = v_sm ? ls : d.ldv;
  for (int e = tid; e < s * s; e += NT) {
    const int r = e % s, c = e / s;
    if (r <= c) P[jp_idx(r, c)] = d.A[r + (long long)c * d.lda];
    V[r + c * ldv] = r == c ? 1.0 : 0.0;
  }
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int i = 0; i < s; ++i) m = fmax(m, fabs(P[jp_idx(i, i)]));
    amax = m;
  }
  __syncthreads();
  const double tol = DBL_EPSILON * double(max(s, 16));  // dimension-scaled stopping rule (as LAPACK dgesvj)
  const double abs_tol = tol * amax;
  const double flo = floor_rel * amax;
  const int n2 = s + (s & 1), np = n2 / 2;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int r = 0; r < n2 - 1; ++r) {
      // 1. rotations of this round's disjoint pairs
      for (int i = tid; i < np; i += NT) {
        int a, b;
        if (i == 0) {
          a = r;
          b = n2 - 1;
        } else {
          a = (r + i) % (n2 - 1);
          b = (r - i + n2 - 1) % (n2 - 1);
        }
        const int p = min(a, b), q = max(a, b);
        double c = 1.0, sg = 0.0;
        if (q < s) {
          const double app = P[jp_idx(p, p)], aqq = P[jp_idx(q, q)], apq = P[jp_idx(p, q)];
          // pairs entirely below the truncation level (both diagonals < 4 eps^2 a_max)
          // only need their eigenvalues to 1e-8 relative (the eps-rank decision), not
          // to machine precision: a 1e-4 relative rule there
          const bool sub = flo > 0.0 && fabs(app) < 4e4 * flo && fabs(aqq) < 4e4 * flo;
          const double thr = rel ? (sub ? 1e-4 : tol) * sqrt(fabs(app * aqq)) : abs_tol;
          const bool below = flo > 0.0 && fabs(app) < flo && fabs(aqq) < flo;
          if (!below && apq != 0.0 && fabs(apq) > thr) {
            const double tau = (aqq - app) / (2.0 * apq);
            double t;
            if (fabs(tau) > 1e150) t = 0.5 / tau;
            else t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            sg = t * c;
            rotated = 1;
          }
        }
        cs_[i] = c;
        sn_[i] = sg;
        pp_[i] = p;
        qq_[i] = q;
      }
      __syncthreads();
      // 2. A <- T A T^T block by block (i <= j), V <- V T^T
      const int nblk = np * (np + 1) / 2;
      for (int w = tid; w < nblk; w += NT) {
        // w = j (j + 1) / 2 + i, i <= j (block pair enumeration without the i > j half)
        int j = int((sqrtf(8.0f * float(w) + 1.0f) - 1.0f) * 0.5f);
        while ((j + 1) * (j + 2) / 2 <= w) ++j;
        while (j * (j + 1) / 2 > w) --j;
        const int i = w - j * (j + 1) / 2;
        const double si = sn_[i], sj = sn_[j];
        if (si == 0.0 && sj == 0.0) continue;
        const double ci = cs_[i], cj = cs_[j];
        const int a = pp_[i], b = qq_[i];
        if (i == j) {  // b < s (a rotation)
          const double app = P[jp_idx(a, a)], aqq = P[jp_idx(b, b)], apq = P[jp_idx(a, b)];
          const double t1 = ci * app - si * apq, t2 = ci * apq - si * aqq;  // row a of T A
          const double t3 = si * app + ci * apq, t4 = si * apq + ci * aqq;  // row b of T A
          P[jp_idx(a, a)] = ci * t1 - si * t2;
          P[jp_idx(b, b)] = si * t3 + ci * t4;
          P[jp_idx(a, b)] = 0.0;
          continue;
        }
        const int e = pp_[j], f = qq_[j];
        const bool bv = b < s, fv = f < s;  // dummy partner index n2-1 == s (odd s)
        const double xae = P[a <= e ? jp_idx(a, e) : jp_idx(e, a)];
        const double xaf = fv ? P[a <= f ? jp_idx(a, f) : jp_idx(f, a)] : 0.0;
        const double xbe = bv ? P[b <= e ? jp_idx(b, e) : jp_idx(e, b)] : 0.0;
        const double xbf = (bv && fv) ? P[b <= f ? jp_idx(b, f) : jp_idx(f, b)] : 0.0;
        // rows: a' = c_i a - s_i b, b' = s_i a + c_i b
        const double rae = ci * xae - si * xbe, raf = ci * xaf - si * xbf;
        const double rbe = si * xae + ci * xbe, rbf = si * xaf + ci * xbf;
        // columns: e' = c_j e - s_j f, f' = s_j e + c_j f
        P[a <= e ? jp_idx(a, e) : jp_idx(e, a)] = cj * rae - sj * raf;
        if (fv) P[a <= f ? jp_idx(a, f) : jp_idx(f, a)] = sj * rae + cj * raf;
        if (bv) P[b <= e ? jp_idx(b, e) : jp_idx(e, b)] = cj * rbe - sj * rbf;
        if (bv && fv) P[b <= f ? jp_idx(b, f) : jp_idx(f, b)] = sj * rbe + cj * rbf;
      }
      for (int w = tid; w < np * s; w += NT) {
        const int i = w / s, j = w - i * s;
        const double sg = sn_[i];
        if (sg != 0.0) {
          const double c = cs_[i];
          const int p = pp_[i], q = qq_[i];
          const double vx = V[j + p * ldv], vy = V[j + q * ldv];
          V[j + p * ldv] = c * vx - sg * vy;
          V[j + q * ldv] = sg * vx + c * vy;
        }
      }
      __syncthreads();
    }
    if (!rotated) break;
    __syncthreads();
  }
  for (int i = tid; i < s; i += NT) d.A[i + (long long)i * d.lda] = P[jp_idx(i, i)];
  if (v_sm)
    for (int e = tid; e < s * s; e += NT) {
      const int r = e % s, c = e / s;
      d.V[r + (long long)c * d.ldv] = V[r + c * ldv];
    }
}

int jacobi_packed_smem_doubles() { return 220 * 1024 / 8; }

// Per-device kernel attributes (called from dtn_gpu_create for every context's
// device: attributes belong to the current device's context).
cudaError_t hbs_kernels_init() {
  cudaError_t e = cudaFuncSetAttribute(jacobi_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       jacobi_smem_doubles() * 8);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(jacobi_eig_packed_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              jacobi_packed_smem_doubles() * 8);
}

cudaError_t launch_jacobi_eig(const EigDesc* d_descs, int count, int max_sweeps, bool rel, double floor_rel,
                              int max_s, cudaStream_t st) {
  if (count <= 0 || max_s <= 0) return cudaSuccess;
  // s <= 236: packed kernel, shared memory sized for this batch's largest block (the
  // packed triangle, plus V when it fits) so that two CTAs share an SM at the low tree
  // levels (256-thread CTAs measured slower: the rounds are latency-bound); larger
  // blocks: the general kernel
  const int sp = std::min(max_s, kPackedMaxS);
  const long long npk = (long long)sp * (sp + 1) / 2, withv = npk + (long long)sp * (sp | 1);
  const int smem = int(std::min<long long>(withv <= jacobi_packed_smem_doubles() ? withv : npk,
                                           jacobi_packed_smem_doubles()));
  jacobi_eig_packed_kernel<1024><<<count, 1024, size_t(smem) * 8, st>>>(d_descs, max_sweeps, smem, rel ? 1 : 0,
                                                                       floor_rel);
  if (max_s > kPackedMaxS)
    jacobi_eig_kernel<<<count, JT, size_t(jacobi_smem_doubles()) * 8, st>>>(d_descs, max_sweeps, jacobi_smem_doubles(),
                                                                          rel ? 1 : 0, kPackedMaxS + 1);
  return cudaGetLastError();
}

// ---- rank selection (hbs.cpp:33-40 svd_rank): sigma_i = sqrt(max(lambda_i, 0)),
// sorted descending (ties: lower index first); rank = #{sigma_i > eps sigma_0},
// 0 when sigma_0 <= 0. One CTA per descriptor.
__global__ void __launch_bounds__(256) hbs_select_kernel(const SelDesc* __restrict__ descs, double eps) {
  const SelDesc d = descs[blockIdx.x];
  const int s = d.s;
  __shared__ double top;
  __shared__ int cnt;
  if (threadIdx.x == 0) {
    top = 0.0;
    cnt = 0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < s; i += blockDim.x) {
    const double li = d.lam[(long long)i * d.stride];
    int pos = 0;
    for (int j = 0; j < s; ++j) {
      const double lj = d.lam[(long long)j * d.stride];
      pos += (lj > li || (lj == li && j < i)) ? 1 : 0;
    }
    d.order[pos] = i;
    d.sigma[pos] = sqrt(fmax(li, 0.0));
    if (pos == 0) top = sqrt(fmax(li, 0.0));
  }
  __syncthreads();
  const double cut = eps * top;
  for (int i = threadIdx.x; i < s; i += blockDim.x)
    if (top > 0.0 && d.sigma[i] > cut) atomicAdd(&cnt, 1);
  __syncthreads();
  if (threadIdx.x == 0) *d.rank = cnt;
}

cudaError_t launch_hbs_select(const SelDesc* d_descs, int count, double eps, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  hbs_select_kernel<<<count, 256, 0, st>>>(d_descs, eps);
  return cudaGetLastError();
}

// ---- dst(:, j) = src(:, order[j]), j < k
__global__ void gather_cols_kernel(const GatherDesc* __restrict__ descs) {
  const GatherDesc d = descs[blockIdx.y];
  const long long total = (long long)d.rows * d.k;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int r = int(e % d.rows), j = int(e / d.rows);
    d.dst[r + (long long)j * d.ldd] = d.src[r + (long long)d.order[j] * d.lds];
  }
}

cudaError_t launch_gather_cols(const GatherDesc* d_descs, int count, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  gather_cols_kernel<<<dim3(32, count), 256, 0, st>>>(d_descs);
  return cudaGetLastError();
}

// ---- repack with zero padding (and optional transpose): dst(i, j) =
// src(rmap(i), cmap(j)) (trans: src(cmap(j), rmap(i))), 0 where a map is -1;
// map(i) = i for i < x1, x1 + (i - xp1) for xp1 <= i < xp1 + x2, else -1
__device__ __forceinline__ int pack_map(int i, int x1, int xp1, int x2) {
  if (i < x1) return i;
  if (i >= xp1 && i < xp1 + x2) return x1 + (i - xp1);
  return -1;
}

__global__ void pack_kernel(const PackDesc* __restrict__ descs) {
  const PackDesc d = descs[blockIdx.y];
  const long long total = (long long)d.rp * d.cp;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int i = int(e % d.rp), j = int(e / d.rp);
    const int ri = pack_map(i, d.r1, d.rp1, d.r2), cj = pack_map(j, d.c1, d.cp1, d.c2);
    double v = 0.0;
    if (ri >= 0 && cj >= 0) v = d.trans ? d.src[cj + (long long)ri * d.lds] : d.src[ri + (long long)cj * d.lds];
    d.dst[i + (long long)j * d.ldd] = v;
  }
}

cudaError_t launch_pack(const PackDesc* d_descs, int count, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  pack_kernel<<<dim3(32, count), 256, 0, st>>>(d_descs);
  return cudaGetLastError();
}

// ---- zero m x n blocks
__global__ void zero_blocks_kernel(const ZeroDesc* __restrict__ descs) {
  const ZeroDesc d = descs[blockIdx.y];
  const long long total = (long long)d.m * d.n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int r = int(e % d.m), c = int(e / d.m);
    d.p[r + (long long)c * d.ld] = 0.0;
  }
}

cudaError_t launch_zero_blocks(const ZeroDesc* d_descs, int count, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  zero_blocks_kernel<<<dim3(32, count), 256, 0, st>>>(d_descs);
  return cudaGetLastError();
}

// ---- dst(m x n) += src(m x n), batched (Dtilde = B + diag(Dhat_l, Dhat_r), hbs_ops.cpp:172-176)
__global__ void add_blocks_kernel(const AddDesc* __restrict__ descs) {
  const AddDesc d = descs[blockIdx.y];
  const long long total = (long long)d.m * d.n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int r = int(e % d.m), c = int(e / d.m);
    d.dst[r + (long long)c * d.ldd] += d.src[r + (long long)c * d.lds];
  }
}

// base[e] = sum_{s < slices} base[e + s stride], e < count (the K-slices of a split product)
__global__ void __launch_bounds__(256) sum_slices_kernel(double* base, long long stride, int slices, long long count) {
  for (long long e = blockIdx.x * 256LL + threadIdx.x; e < count; e += (long long)gridDim.x * 256) {
    double t = base[e];
    for (int q = 1; q < slices; ++q) t += base[e + q * stride];
    base[e] = t;
  }
}

cudaError_t launch_sum_slices(double* base, long long stride, int slices, long long count, cudaStream_t st) {
  if (count <= 0 || slices <= 1) return cudaSuccess;
  const long long blocks = std::min<long long>((count + 255) / 256, 148 * 8);
  sum_slices_kernel<<<unsigned(blocks), 256, 0, st>>>(base, stride, slices, count);
  return cudaGetLastError();
}

cudaError_t launch_add_blocks(const AddDesc* d_descs, int count, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  add_blocks_kernel<<<dim3(32, count), 256, 0, st>>>(d_descs);
  return cudaGetLastError();
}

// ---- in-place inverse of small dense blocks (the checked inverses of
// invert_hbs, hbs_ops.cpp:148-201): Gauss-Jordan with partial (row) pivoting,
// one CTA per matrix, the matrix in shared memory (odd leading dimension)
// when it fits, else in place in global memory (L2-resident at these sizes).
// Step k: argmax |a_ik| over i >= k (lowest index on ties), swap rows k and p,
// then one fused rank-1 sweep a_ij -= a_ik a_kj / a_kk over the whole matrix
// with the pivot row/column replaced in place; the recorded row interchanges
// become column interchanges of the inverse at the end. A zero or non-finite
// pivot marks the block singular (*info = k + 1) and stops.
constexpr int GJT = 512;
constexpr int GJ_SMEM_MAX = 160;  // s <= 160: 160 * 161 doubles = 206 KB

// SM: every block of the launch fits in shared memory (the matrix addressed as shared,
// not through generic pointers); else every block is inverted in place in global memory
template <bool SM>
__global__ void __launch_bounds__(GJT) gj_inverse_kernel(const InvDesc* __restrict__ descs) {
  extern __shared__ __align__(16) double gsm[];
  __shared__ double rv[GJT / 32];
  __shared__ int ri[GJT / 32];
  __shared__ int piv_row;
  __shared__ int bad;
  const InvDesc d = descs[blockIdx.x];
  const int s = d.s;
  if (s <= 0) {
    if (threadIdx.x == 0) *d.info = 0;
    return;
  }
  constexpr bool in_smem = SM;
  const int lda = in_smem ? (s | 1) : d.lda;
  double* A = in_smem ? gsm : d.A;
  double* rowk = in_smem ? gsm + (long long)lda * s : gsm;  // s doubles
  double* colk = rowk + s;                                  // s doubles
  int* perm = reinterpret_cast<int*>(colk + s);             // s ints
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (in_smem)
    for (int e = tid; e < s * s; e += GJT) A[(e % s) + (e / s) * lda] = d.A[(e % s) + (long long)(e / s) * d.lda];
  if (tid == 0) bad = 0;
  __syncthreads();
  __shared__ double s_piv;
  for (int k = 0; k < s; ++k) {
    // 1. pivot: argmax |a_ik|, i >= k (warp 0; lowest index on ties, NaN ranks highest)
    if (warp == 0) {
      double bv = -1.0;
      int bi = s;
      for (int i = k + lane; i < s; i += 32) {
        double v = fabs(A[i + (long long)k * lda]);
        if (v != v) v = INFINITY;
        if (v > bv) {
          bv = v;
          bi = i;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (lane == 0) {
        const double pv = bi < s ? A[bi + (long long)k * lda] : 0.0;
        if (bi >= s || pv == 0.0 || !isfinite(pv)) bad = k + 1;
        piv_row = bi;
        perm[k] = bi;
        s_piv = pv;
      }
    }
    __syncthreads();
    if (bad) break;
    // 2. swap rows k and p (column by column), the scaled pivot row and the pivot
    //    column, all from the values before the swap
    const int p = piv_row;
    const double rp = 1.0 / s_piv;
    for (int x = tid; x < s; x += GJT) {
      double* cj = A + (long long)x * lda;
      const double ak = cj[k], ap = cj[p];
      if (p != k) {
        cj[k] = ap;
        cj[p] = ak;
      }
      rowk[x] = (x == k ? 1.0 : ap) * rp;  // new row k = old row p
      // pivot column after the swap: rows k and p from thread k's own (pre-swap)
      // reads of column k, every other row unaffected by the swap
      if (x == k) {
        colk[k] = s_piv;
        if (p != k) colk[p] = ak;
      } else if (x != p) {
        colk[x] = A[x + (long long)k * lda];
      }
    }
    __syncthreads();
    // 3. rank-1 sweep: warp w owns columns w, w + 16, ..., lanes own rows (no division
    //    per entry); a_kj <- rowk_j, a_ik <- -colk_i rowk_k, a_ij -= colk_i rowk_j
    for (int j = warp; j < s; j += GJT / 32) {
      double* cj = A + (long long)j * lda;
      const double rj = rowk[j];
      const bool jk = j == k;
      for (int i = lane; i < s; i += 32) {
        const double a = jk ? 0.0 : cj[i];
        cj[i] = i == k ? rj : fma(-colk[i], rj, a);
      }
    }
    __syncthreads();
  }
  if (bad) {
    if (tid == 0) *d.info = bad;
    return;
  }
  // 5. undo the interchanges on the columns, last first
  for (int k = s - 1; k >= 0; --k) {
    const int p = perm[k];
    if (p != k)
      for (int i = tid; i < s; i += GJT) {
        const double t = A[i + (long long)k * lda];
        A[i + (long long)k * lda] = A[i + (long long)p * lda];
        A[i + (long long)p * lda] = t;
      }
    __syncthreads();
  }
  if (in_smem)
    for (int e = tid; e < s * s; e += GJT) d.A[(e % s) + (long long)(e / s) * d.lda] = A[(e % s) + (e / s) * lda];
  if (tid == 0) *d.info = 0;
}

cudaError_t launch_gj_inverse(const InvDesc* d_descs, int count, int max_s, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const int sm = std::min(max_s, GJ_SMEM_MAX);
  // shared: the matrix (when it fits) + pivot row/column + permutation
  const size_t bytes = size_t((sm | 1)) * sm * 8 + size_t(max_s) * 20 + 64;
  if (bytes > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(gj_inverse_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
    if (e != cudaSuccess) return e;
  }
  if (max_s <= GJ_SMEM_MAX) gj_inverse_kernel<true><<<count, GJT, bytes, st>>>(d_descs);
  else gj_inverse_kernel<false><<<count, GJT, size_t(max_s) * 20 + 64, st>>>(d_descs);
  return cudaGetLastError();
}

}  // namespace dtnb
