// Compressed-engine kernels (K5: structured merges, build_root_accel,
// accel_nd.cpp:434-628, 667-689; paper Sec. 6 Steps 1-3) on the B200.
//
// A structured box keeps its S dense in HBM (CCW order) together with rank-ell
// factors of the two off-diagonal blocks of its [J; K] split (J = the edge its
// next merge eliminates, arc_boundary accel_nd.cpp:46-88):
//   S[J, K] ~= L_jk R_jk,  L_jk = Q1,              R_jk^T = S[J, :]^T Q1
//   S[K, J] ~= L_kj R_kj,  L_kj = S[:, J] Q2,      R_kj^T = Q2
// with Q1, Q2 orthonormal bases of randomized range-finder sketches
// Y1 = S[J, K] Omega and Y2 = S[K, J]^T Omega (compress_box / lowrank_from_dense,
// accel_nd.cpp:93-130, lowrank.cpp:27-36; the sketch replaces the truncated SVD).
// Merging two structured boxes a | b (interface J = J_a u J_b):
//   Step 1  the reduced interface system [[M_jj, Z], [W, 0]], Z = blockdiag(L_jk),
//           W = blockdiag(R_kj), is factored with the blocked partial-pivot LU of the
//           dense path (interface pivots only); its Schur complement is
//           C = -W M_jj^{-1} Z ((ra + rb) x (ra + rb))          sgather_red_kernel
//   Step 2  the low-rank products: T = -L_k C with L_k = blockdiag(L_kj) in the
//           parent's boundary order                             factor_gather_kernel
//   Step 3  S_parent = M_kk - T R_k, M_kk the children's kept blocks plus the
//           junction couplings (accel_nd.cpp:518-549)           kk_gather_kernel
// then the parent's own factors for its next merge (omega_kernel, hqr_kernel and
// four descriptor GEMMs, see engine.cu).
#include <algorithm>
#include <cstdint>

#include <cooperative_groups.h>

#include "common.cuh"

namespace dtnb {

namespace cg = cooperative_groups;
constexpr int SG_COLS = 8;

// Reduced interface system of a structured merge (ldm x total, total = ni + ra + rb):
// rows/columns [J_a (jn_a); J_b (jn_b); factor columns (ra + rb)].
__global__ void __launch_bounds__(256) sgather_red_kernel(KernelArgs args, const int* __restrict__ list) {
  const NodeDev nd = args.nodes[list[blockIdx.y]];
  const int j0c = blockIdx.x * SG_COLS;
  if (j0c >= nd.total) return;
  const NodeDev ca = args.nodes[nd.a], cb = args.nodes[nd.b];
  const double* A = args.arena + ca.s_off;
  const double* B = args.arena + cb.s_off;
  const double* Q1a = args.arena + ca.q1_off;
  const double* Q2a = args.arena + ca.q2_off;
  const double* Q1b = args.arena + cb.q1_off;
  const double* Q2b = args.arena + cb.q2_off;
  double* M = args.arena + nd.m_off;
  const PosDev* pos = args.pos + nd.pos_off;
  const int ni = nd.ni, ja = ca.jn, ra = ca.ell;
  for (int jj = 0; jj < SG_COLS; ++jj) {
    const int j = j0c + jj;
    if (j >= nd.total) break;
    double* col = M + (long long)j * nd.ldm;
    if (j < ni) {  // interface column
      const PosDev pj = pos[j];
      const double* colA = pj.src >= 0 ? A + (long long)pj.src * ca.ld : nullptr;
      const double* colB = pj.src < 0 ? B + (long long)(-pj.src - 1) * cb.ld : nullptr;
      for (int i = threadIdx.x; i < ni; i += blockDim.x) {
        const PosDev pi = pos[i];
        double v = 0.0;
        if (pi.src >= 0 && colA) v = colA[pi.src];
        else if (pi.src < 0 && colB) v = colB[-pi.src - 1];
        else if (pi.partner == j) v = args.stencil[pi.dir * args.nu + pi.gid];
        col[i] = v;
      }
      for (int c = threadIdx.x; c < nd.sys_nb; c += blockDim.x) {  // W = blockdiag(Q2_a^T, Q2_b^T)
        double v = 0.0;
        if (c < ra && j < ja) v = Q2a[j + (long long)c * ca.ldq];
        else if (c >= ra && j >= ja) v = Q2b[(j - ja) + (long long)(c - ra) * cb.ldq];
        col[ni + c] = v;
      }
    } else {  // factor column: Z = blockdiag(Q1_a, Q1_b), zero block below
      const int c = j - ni;
      for (int i = threadIdx.x; i < nd.total; i += blockDim.x) {
        double v = 0.0;
        if (i < ja) {
          if (c < ra) v = Q1a[i + (long long)c * ca.ldq];
        } else if (i < ni) {
          if (c >= ra) v = Q1b[(i - ja) + (long long)(c - ra) * cb.ldq];
        }
        col[i] = v;
      }
    }
  }
}

// The kept block M_kk of a structured merge into the parent's S (ld), in the
// parent's CCW order: the children's S entries plus the junction couplings
// (the boundary rows of merge_two's assembly, dense_nd.cpp:135-165).
__global__ void __launch_bounds__(256) kk_gather_kernel(KernelArgs args, const int* __restrict__ list) {
  const NodeDev nd = args.nodes[list[blockIdx.y]];
  const int q0 = blockIdx.x * SG_COLS;
  if (q0 >= nd.nb) return;
  const NodeDev ca = args.nodes[nd.a], cb = args.nodes[nd.b];
  const double* A = args.arena + ca.s_off;
  const double* B = args.arena + cb.s_off;
  double* S = args.arena + nd.s_off;
  const PosDev* pos = args.pos + nd.pos_off + nd.ni;
  for (int qq = 0; qq < SG_COLS; ++qq) {
    const int q = q0 + qq;
    if (q >= nd.nb) break;
    const PosDev pq = pos[q];
    const double* colA = pq.src >= 0 ? A + (long long)pq.src * ca.ld : nullptr;
    const double* colB = pq.src < 0 ? B + (long long)(-pq.src - 1) * cb.ld : nullptr;
    for (int p = threadIdx.x; p < nd.nb; p += blockDim.x) {
      const PosDev pp = pos[p];
      double v = 0.0;
      if (pp.src >= 0 && colA) v = colA[pp.src];
      else if (pp.src < 0 && colB) v = colB[-pp.src - 1];
      else if (pp.partner == nd.ni + q) v = args.stencil[pp.dir * args.nu + pp.gid];
      S[p + (long long)q * nd.ld] = v;
    }
  }
}

// L_k = blockdiag(L_kj) (nb x r, ldg) and R_k = blockdiag(R_jk) (r x nb, ldr) in the
// parent's boundary order (the children's J rows never reach the parent).
__global__ void __launch_bounds__(256) factor_gather_kernel(KernelArgs args, const int* __restrict__ list) {
  const NodeDev nd = args.nodes[list[blockIdx.y]];
  const NodeDev ca = args.nodes[nd.a], cb = args.nodes[nd.b];
  const int nb = nd.nb, r = nd.sys_nb, ra = ca.ell;
  const long long tot = (long long)nb * r;
  const PosDev* pos = args.pos + nd.pos_off + nd.ni;
  double* Lk = args.arena + nd.lkg_off;
  double* Rk = args.arena + nd.rkg_off;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    {  // L_k, column-major walk (coalesced stores)
      const int p = int(e % nb), c = int(e / nb);
      const int src = pos[p].src;
      double v = 0.0;
      if (src >= 0) {
        if (c < ra) v = args.arena[ca.lk_off + src + (long long)c * ca.ldf];
      } else if (c >= ra) {
        v = args.arena[cb.lk_off + (-src - 1) + (long long)(c - ra) * cb.ldf];
      }
      Lk[p + (long long)c * nd.ldg] = v;
    }
    {  // R_k (r x nb), column-major walk
      const int c = int(e % r), p = int(e / r);
      const int src = pos[p].src;
      double v = 0.0;
      if (src >= 0) {
        if (c < ra) v = args.arena[ca.rt_off + src + (long long)c * ca.ldf];
      } else if (c >= ra) {
        v = args.arena[cb.rt_off + (-src - 1) + (long long)(c - ra) * cb.ldf];
      }
      Rk[c + (long long)p * nd.ldr] = v;
    }
  }
}

// Sketch matrix Omega (nb x ell, ldf) of a structured box: uniform[-1, 1) from a
// counter-based hash of (row, column) -- identical on every run -- with the J rows
// zero, so that Y1 = S[J, :] Omega = S[J, K] Omega[K, :] and likewise Y2.
__device__ __forceinline__ double hash_uniform(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  x ^= x >> 31;
  return double(x >> 11) * 0x1.0p-52 - 1.0;
}

__global__ void __launch_bounds__(256) omega_kernel(KernelArgs args, const int* __restrict__ list) {
  const NodeDev nd = args.nodes[list[blockIdx.y]];
  const long long tot = (long long)nd.nb * (nd.ell + kProbes);
  double* Om = args.arena + nd.om_off;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int p = int(e % nd.nb), c = int(e / nd.nb);
    const bool in_j = p >= nd.j0 && p < nd.j0 + nd.jn;
    Om[p + (long long)c * nd.ldf] = in_j ? 0.0 : hash_uniform((unsigned long long)p * 0x100000001B3ull + c);
  }
}

// Householder QR of the first n columns of Y (m x (n + p)) and the explicit
// Q = H_0 ... H_{n-1} [I; 0] (m x n) (LAPACK dgeqr2 / dorg2r conventions:
// H = I - tau v v^T, v_c = 1, beta = -sign(alpha) ||x||), one thread-block
// cluster of C CTAs per matrix: CTA r owns rows [r R, (r + 1) R) and keeps them in
// shared memory when they fit (SM) -- the column loop then never touches HBM/L2
// except through the cluster's DSMEM reductions. Per column: partial norms (one
// cluster barrier: the pivot column's norm and alpha), then partial dot products
// of the reflector with every trailing column (a second barrier), each CTA
// summing the C partials in rank order so every CTA computes bit-identical
// reflectors. Reduction buffers alternate by column parity (a CTA can run at most
// one barrier ahead of the slowest reader). The reflectors are applied to the p
// probe columns too: their rows n..m-1 then hold (I - Q Q^T) y, the randomized
// range finder's a-posteriori estimate (Halko, Martinsson & Tropp 2011, Sec. 4.3).
// stat[1] = max_probe |(I - Q Q^T) y| / scale, stat[0] = #{|R_ii| > eps scale},
// relative to the box operator's scale max_i |S_ii| sqrt(k / 3) (the expected
// norm of S applied to a k-vector of uniform[-1, 1] entries, S diagonally dominant).
constexpr int QR_THREADS = 256, QR_WARPS = QR_THREADS / 32, QR_MAXC = 16, QR_MAXN = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct QrShared {
  double a[2][2];              // [parity][0: partial sum of squares, 1: alpha (owner)]
  double w[2][QR_MAXN + 8];    // [parity] partial dot products
  double tau[QR_MAXN], rdiag[QR_MAXN];
  double red[QR_WARPS];
};

// CL = false: a single CTA per matrix (C == 1), plain block barriers and shared memory
template <bool SM, bool CL>
__global__ void __launch_bounds__(QR_THREADS) hqr_cluster_kernel(const QrDesc* __restrict__ descs,
                                                                 const double* eps_ptr, int C) {
  extern __shared__ __align__(16) double qdyn[];
  __shared__ QrShared sh;
  struct Sync {
    __device__ void sync() const {
      if constexpr (CL) cg::this_cluster().sync();
      else __syncthreads();
    }
    __device__ double* map(double* p, int q) const {
      if constexpr (CL) return cg::this_cluster().map_shared_rank(p, q);
      else return p;
    }
  } cl;
  const int rank = CL ? int(cg::this_cluster().block_rank()) : 0;
  const QrDesc d = descs[blockIdx.x / C];
  const int m = d.m, n = d.n, nc = d.n + d.p;
  const int R = (m + C - 1) / C, r0 = rank * R, r1 = min(m, r0 + R), nr = max(r1 - r0, 0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // local rows: shared memory (ld = R) or the matrix itself
  double* Yl = SM ? qdyn : d.Y + r0;
  const long long ldl = SM ? R : d.ldy;
  if (SM) {
    for (int j = 0; j < nc; ++j)
      for (int i = tid; i < nr; i += QR_THREADS) Yl[i + j * ldl] = d.Y[r0 + i + (long long)j * d.ldy];
    __syncthreads();
  }
  auto remote_sum = [&](double* base) {  // sum over ranks, fixed order
    double t = 0.0;
    for (int q = 0; q < C; ++q) t += *cl.map(base, q);
    return t;
  };
  for (int c = 0; c < n; ++c) {
    const int par = c & 1;
    double* yc = Yl + (long long)c * ldl;
    // rows of this CTA strictly below the diagonal: [max(c + 1, r0), r1)
    const int lo = max(c + 1 - r0, 0);
    double ss = 0.0;
    for (int i = lo + tid; i < nr; i += QR_THREADS) ss = fma(yc[i], yc[i], ss);
    ss = warp_sum(ss);
    if (lane == 0) sh.red[warp] = ss;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < QR_WARPS; ++w) t += sh.red[w];
      sh.a[par][0] = t;
      sh.a[par][1] = (c >= r0 && c < r1) ? yc[c - r0] : 0.0;
    }
    cl.sync();
    const double sst = remote_sum(&sh.a[par][0]);
    const double alpha = *cl.map(&sh.a[par][1], c / R);
    double beta, tc, scal;
    if (sst == 0.0) {
      beta = alpha;
      tc = 0.0;
      scal = 0.0;
    } else {
      beta = -copysign(sqrt(fma(alpha, alpha, sst)), alpha);
      tc = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    for (int i = lo + tid; i < nr; i += QR_THREADS) yc[i] *= scal;  // v below the diagonal
    const bool own = c >= r0 && c < r1;
    if (own && tid == 0) yc[c - r0] = beta;
    if (tid == 0) {
      sh.tau[c] = tc;
      sh.rdiag[c] = beta;
    }
    __syncthreads();
    // partial dots v^T y_j over the local rows (v_c = 1 on the owner's row c)
    const int lv = max(c - r0, 0);  // first local row of the reflector
    for (int j = c + 1 + warp; j < nc; j += QR_WARPS) {
      const double* yj = Yl + (long long)j * ldl;
      double s = 0.0;
      for (int i = lv + lane; i < nr; i += 32) s = fma((own && i == c - r0) ? 1.0 : yc[i], yj[i], s);
      s = warp_sum(s);
      if (lane == 0) sh.w[par][j] = s;
    }
    cl.sync();
    if (tc != 0.0) {
      for (int j = c + 1 + warp; j < nc; j += QR_WARPS) {
        const double wj = remote_sum(&sh.w[par][j]) * tc;
        double* yj = Yl + (long long)j * ldl;
        for (int i = lv + lane; i < nr; i += 32) yj[i] = fma(-wj, (own && i == c - r0) ? 1.0 : yc[i], yj[i]);
      }
    }
    __syncthreads();
  }
  // range-finder check: |(I - Q Q^T) y_probe|^2 = sum of the probe columns' rows >= n
  double pres = 0.0;
  {
    const int lo = max(n - r0, 0);
    for (int q = 0; q < d.p; ++q) {
      const double* yq = Yl + (long long)(n + q) * ldl;
      double ss = 0.0;
      for (int i = lo + tid; i < nr; i += QR_THREADS) ss = fma(yq[i], yq[i], ss);
      ss = warp_sum(ss);
      if (lane == 0) sh.red[warp] = ss;
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < QR_WARPS; ++w) t += sh.red[w];
        sh.w[q & 1][QR_MAXN + (q >> 1)] = t;
      }
      __syncthreads();
    }
    cl.sync();
    for (int q = 0; q < d.p; ++q) pres = fmax(pres, sqrt(remote_sum(&sh.w[q & 1][QR_MAXN + (q >> 1)])));
    cl.sync();  // (the partial buffers are reused below)
  }
  // Q = H_0 ... H_{n-1} [I; 0] on the local rows, backward accumulation
  double* Q = d.Q + r0;
  const long long ldq = d.ldq;
  for (int j = 0; j < n; ++j)
    for (int i = tid; i < nr; i += QR_THREADS) Q[i + j * ldq] = (r0 + i == j) ? 1.0 : 0.0;
  __syncthreads();
  for (int c = n - 1; c >= 0; --c) {
    const int par = c & 1;
    const double tc = sh.tau[c];
    const double* yc = Yl + (long long)c * ldl;
    const bool own = c >= r0 && c < r1;
    const int lv = max(c - r0, 0);
    for (int j = c + warp; j < n; j += QR_WARPS) {
      const double* qj = Q + (long long)j * ldq;
      double s = 0.0;
      for (int i = lv + lane; i < nr; i += 32) s = fma((own && i == c - r0) ? 1.0 : yc[i], qj[i], s);
      s = warp_sum(s);
      if (lane == 0) sh.w[par][j] = s;
    }
    cl.sync();
    if (tc != 0.0) {
      for (int j = c + warp; j < n; j += QR_WARPS) {
        const double wj = remote_sum(&sh.w[par][j]) * tc;
        double* qj = Q + (long long)j * ldq;
        for (int i = lv + lane; i < nr; i += 32) qj[i] = fma(-wj, (own && i == c - r0) ? 1.0 : yc[i], qj[i]);
      }
    }
    __syncthreads();
  }
  if (rank == 0 && d.stat) {
    double dmax = 0.0;
    for (int i = tid; i < d.nbs; i += QR_THREADS) dmax = fmax(dmax, fabs(d.S[i + (long long)i * d.lds]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    if (lane == 0) sh.red[warp] = dmax;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < QR_WARPS; ++w) t = fmax(t, sh.red[w]);
      const double eps = *eps_ptr, scale = t * sqrt(double(d.k) / 3.0);
      int rk = 0;
      for (int i = 0; i < n; ++i)
        if (fabs(sh.rdiag[i]) > eps * scale) ++rk;
      d.stat[0] = double(rk);
      d.stat[1] = scale > 0.0 ? pres / scale : 0.0;
    }
  }
  cl.sync();  // no CTA leaves while others may still read its shared memory
}

cudaError_t launch_sgather_red(const KernelArgs& args, const int* d_list, int count, int max_total, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  dim3 grid((max_total + SG_COLS - 1) / SG_COLS, count);
  sgather_red_kernel<<<grid, 256, 0, st>>>(args, d_list);
  return cudaGetLastError();
}

cudaError_t launch_kk_gather(const KernelArgs& args, const int* d_list, int count, int max_nb, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  dim3 grid((max_nb + SG_COLS - 1) / SG_COLS, count);
  kk_gather_kernel<<<grid, 256, 0, st>>>(args, d_list);
  return cudaGetLastError();
}

cudaError_t launch_factor_gather(const KernelArgs& args, const int* d_list, int count, long long max_elems,
                                 cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  dim3 grid(unsigned(std::min<long long>((max_elems + 255) / 256, 1184)), count);
  factor_gather_kernel<<<grid, 256, 0, st>>>(args, d_list);
  return cudaGetLastError();
}

cudaError_t launch_omega(const KernelArgs& args, const int* d_list, int count, long long max_elems, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  dim3 grid(unsigned(std::min<long long>((max_elems + 255) / 256, 1184)), count);
  omega_kernel<<<grid, 256, 0, st>>>(args, d_list);
  return cudaGetLastError();
}

// cluster size for an m x nc matrix: the smallest C whose row blocks fit in shared memory
// (<= 200 KB), else 16 CTAs working on the matrix in global memory (L1/L2-resident)
static int qr_cluster(int m, int nc, bool* smem) {
  for (int C = 1; C <= QR_MAXC; C *= 2) {
    const long long R = (m + C - 1) / C;
    if (R * nc * 8 <= 200 * 1024) {
      *smem = true;
      return C;
    }
  }
  *smem = false;
  return QR_MAXC;
}

cudaError_t struct_init() {
  for (auto f : {hqr_cluster_kernel<true, true>, hqr_cluster_kernel<false, true>, hqr_cluster_kernel<true, false>}) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_hqr(const QrDesc* d_descs, int count, int max_m, int max_nc, const double* d_eps, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  if (max_nc > QR_MAXN) return cudaErrorInvalidValue;
  bool sm = false;
  const int C = qr_cluster(max_m, max_nc, &sm);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(count * C);
  cfg.blockDim = dim3(QR_THREADS);
  cfg.stream = st;
  cfg.dynamicSmemBytes = sm ? size_t((max_m + C - 1) / C) * max_nc * 8 : 0;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (sm && C == 1) {
    cfg.numAttrs = 0;
    return cudaLaunchKernelEx(&cfg, hqr_cluster_kernel<true, false>, d_descs, d_eps, C);
  }
  if (sm) return cudaLaunchKernelEx(&cfg, hqr_cluster_kernel<true, true>, d_descs, d_eps, C);
  return cudaLaunchKernelEx(&cfg, hqr_cluster_kernel<false, true>, d_descs, d_eps, C);
}

}  // namespace dtnb
